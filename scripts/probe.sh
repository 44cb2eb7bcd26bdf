nvidia-smi; free -g; nproc; lscpu | head -25; cat /proc/meminfo | head -5; ulimit -l
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
n = 1<<30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device='cuda')
s = torch.cuda.Stream()
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
    e1.synchronize(); print("H2D GB/s", n/e0.elapsed_time(e1)/1e6)
    with torch.cuda.stream(s):
        e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
    e1.synchronize(); print("D2H GB/s", n/e0.elapsed_time(e1)/1e6)
t=time.time(); big = torch.empty(40<<30, dtype=torch.uint8, pin_memory=True); print("pin 40GiB s", time.time()-t)
PY
