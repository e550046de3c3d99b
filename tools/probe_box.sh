nvidia-smi; free -g; nproc; lscpu | head -20; df -h /dev/shm; ulimit -l
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for gb in [1, 4]:
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device='cuda')
    for _ in range(2):
        torch.cuda.synchronize(); t=time.time(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1=time.time()-t
        t=time.time(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2=time.time()-t
    print(f"{gb}GiB H2D {n/t1/1e9:.1f} GB/s D2H {n/t2/1e9:.1f} GB/s")
    s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2=torch.empty(n, dtype=torch.uint8, device='cuda')
    torch.cuda.synchronize(); t=time.time()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t3=time.time()-t
    print(f"{gb}GiB bidir {2*n/t3/1e9:.1f} GB/s total")
t=time.time(); x = torch.empty(32<<30, dtype=torch.uint8, pin_memory=True); print("pin 32GiB s", time.time()-t)
PY
