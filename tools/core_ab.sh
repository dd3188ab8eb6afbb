for c in 0 1; do echo "CROSS=$c"; RSVD_GCL_CROSS=$c python tools/core_probe.py 70 140 250 500 2>&1 | grep -v Warn; done
