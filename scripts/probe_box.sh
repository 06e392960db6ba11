set -x
free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1; nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv
numactl -H 2>/dev/null | head -20
ulimit -l
python - <<'PY'
import torch, time
xs=[]
tot=0
for i in range(12):
    try:
        t0=time.time()
        x=torch.empty(10*2**30, dtype=torch.uint8, pin_memory=True)
        xs.append(x); tot+=10
        print("pinned GB", tot, "alloc s", round(time.time()-t0,2), flush=True)
    except Exception as e:
        print("fail at", tot, e); break
del xs
print(torch.cuda.mem_get_info())
PY
