import json, torch, sys
sys.path.insert(0, '.')
from paper_1804_07531_b200 import rsvd
c = rsvd.Context(0)
t, g = c.probe_peaks()
print(json.dumps({"dmma_fp64_tflops": t, "hbm_read_gbs": g, "sms": c.sm_count, "gpu": torch.cuda.get_device_name(0)}))
