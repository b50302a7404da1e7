"""PCIe copy bandwidth probe (pinned host <-> device), H2D, D2H and both at once."""
import time
import torch

n = 805306368
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_in.copy_(h_in, non_blocking=True); h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    return time.perf_counter() - t0
h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
bb = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  both {2*n/bb/1e9:.1f} GB/s total ({bb*1e3:.1f} ms)")

# two streams per direction (halves), to see whether one copy engine per
# direction is the limit
s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
def both4():
    with torch.cuda.stream(s1): d_in[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s3): d_in[half:].copy_(h_in[half:], non_blocking=True)
    with torch.cuda.stream(s2): h_out[:half].copy_(d_out[:half], non_blocking=True)
    with torch.cuda.stream(s4): h_out[half:].copy_(d_out[half:], non_blocking=True)
b4 = min(t(both4) for _ in range(3))
def h2d2():
    with torch.cuda.stream(s1): d_in[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s3): d_in[half:].copy_(h_in[half:], non_blocking=True)
h2 = min(t(h2d2) for _ in range(3))
bb = min(t(both) for _ in range(3))
print(f"both, 1 stream each way {bb*1e3:.1f} ms; 2 streams each way {b4*1e3:.1f} ms; H2D on 2 streams {n/h2/1e9:.1f} GB/s")
