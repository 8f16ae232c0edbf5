"""PCIe copy rates on the GPU box: H2D / D2H alone and concurrently (pinned)."""
import time
import torch

n = 1 << 26
h_in = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
h_out = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
d_in = torch.empty(4 * n, dtype=torch.float64, device="cuda")
d_out = torch.empty(3 * n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s1):
        for q in range(4):
            d_in[q * n:(q + 1) * n].copy_(h_in[q], non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for q in range(3):
            h_out[q].copy_(d_out[q * n:(q + 1) * n], non_blocking=True)


for name, fns in (("h2d", [h2d]), ("d2h", [d2h]), ("both", [h2d, d2h])):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in fns:
            f()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    gb = (32 * n if h2d in fns else 0) / 1e9, (24 * n if d2h in fns else 0) / 1e9
    print(f"{name}: {dt*1e3:.1f} ms  h2d {gb[0]/dt:.1f} GB/s  d2h {gb[1]/dt:.1f} GB/s")
