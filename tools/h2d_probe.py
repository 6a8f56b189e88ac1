"""Pinned host <-> device copy bandwidth (the e2e ceiling of decode_host) and the PCIe link state."""
import torch, time
x = torch.empty(2048*1024*1024//4, dtype=torch.float32, pin_memory=True)
d = torch.empty_like(x, device="cuda")
for sz_mb in (16, 64, 256, 2048):
    n = sz_mb*1024*1024//4
    for _ in range(2): d[:n].copy_(x[:n], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(3): d[:n].copy_(x[:n], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(sz_mb, "MiB H2D", 3*n*4/ (e0.elapsed_time(e1)/1e3)/1e9, "GB/s")
# D2H
y = torch.empty(256*1024*1024, dtype=torch.uint8, pin_memory=True)
dy = torch.empty_like(y, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y.copy_(dy, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H 256MiB", y.numel()/(e0.elapsed_time(e1)/1e3)/1e9)
import subprocess; print(subprocess.run(r"nvidia-smi -q | grep -A3 -i 'PCIe Generation\|Link Width'", shell=True, capture_output=True, text=True).stdout)
