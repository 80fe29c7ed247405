"""Practical HBM bandwidth on this GPU: torch.sum over 8 GB (read only) and copy_ (read + write).
  python tools/hbm_read_bw.py
(B200 here: read 6.53 TB/s, copy 6.67 TB/s: the roofline denominators in MEASURED_PEAKS.json are
what a streaming kernel can reach.)"""
import torch, time
x = torch.empty(2*1024**3, dtype=torch.float32, device='cuda').uniform_()   # 8 GB
for _ in range(3): s = x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): s = x.sum()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("torch.sum read GB/s", x.numel()*4/ms/1e6)
y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("copy (r+w) GB/s", 2*x.numel()*4/ms/1e6)
