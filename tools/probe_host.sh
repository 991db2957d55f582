nproc; free -g; lscpu | head -20; nvidia-smi -L
python - <<'PY'
import time, numpy as np, torch, os
print("cpu_count", os.cpu_count(), "torch threads", torch.get_num_threads())
a=np.random.rand(128,1024).astype(np.float32); b=np.random.rand(1024,262144).astype(np.float32)
for i in range(3):
    t=time.perf_counter(); c=a@b; dt=time.perf_counter()-t
    print("np sgemm 128x1024x262144 %.3f s  %.1f GF/s"%(dt, 2*128*1024*262144/dt/1e9))
bt=torch.from_numpy(b.T.copy()); at=torch.from_numpy(a)
for i in range(3):
    t=time.perf_counter(); c=at@bt.T; dt=time.perf_counter()-t
    print("torch sgemm %.3f s  %.1f GF/s"%(dt, 2*128*1024*262144/dt/1e9))
PY
