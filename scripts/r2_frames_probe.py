"""e2e frames pipeline probe (c4): frame period against the PCIe floor, for several frame counts."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
wl = CF.c4_large_uniform(n, seed=0)
sim = E.Simulation(E.SimulationParams(**dict(wl.params, record_forces=False)))
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (wl.x, wl.y, wl.z, wl.d)]
outs = [[torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in range(3)] for _ in range(2)]
sim.run_frames([pin] * 2, outs, iterations=1, first_iteration=0)
# copy-only floors
dev = torch.empty(4 * n, dtype=torch.float64, device="cuda")
hin = torch.from_numpy(np.concatenate([a for a in pin]))
hin = hin.pin_memory()
hout = torch.empty(3 * n, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
for both in (False, True):
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            dev.copy_(hin, non_blocking=True)
        if both:
            with torch.cuda.stream(s2):
                hout.copy_(dev[:3 * n], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print("copy floor both=%s: %.1f ms per frame (H2D %.1f GB/s)" % (both, dt * 1e3, 32 * n / dt / 1e9))
for frames in (10, 20, 40):
    t0 = time.perf_counter()
    sim.run_frames([pin] * frames, [outs[f % 2] for f in range(frames)], iterations=1, first_iteration=10)
    dt = time.perf_counter() - t0
    print("frames %d: %.1f ms per frame -> %.4g agent-it/s" % (frames, dt / frames * 1e3, n * frames / dt))
