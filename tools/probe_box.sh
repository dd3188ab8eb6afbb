free -g; nproc; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))"; lscpu | head -20; df -h /tmp /dev/shm | cat
python - <<'PY'
import numpy as np, time
a=np.random.rand(4096,200000); x=np.random.rand(200000,120)
t=time.perf_counter(); y=a@x; t1=time.perf_counter()-t
t=time.perf_counter(); z=a.T@y; t2=time.perf_counter()-t
print('gemm A@X GF/s', 2*4096*200000*120/t1/1e9, 'AT@Y', 2*4096*200000*120/t2/1e9)
PY
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 blas | head
