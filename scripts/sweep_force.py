"""Sweep force-kernel build variants x internal bin geometry on one workload.

Usage (on the GPU box):
    python scripts/sweep_force.py --config c4 --n 67108864 --libs variants/*.so --bins 1x1 2x1 2x2 3x1
Prints one JSON line per (lib, bins) with ms/step and force-kernel ms.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import numpy as np
    import torch

    import paper_2301_06984_b200 as E
    d = np.load(args.cache)
    byz, bx = (int(v) for v in args.bin.split("x"))
    prm = json.loads(str(d["params"]))
    prm.update(record_forces=False, bins_per_box=byz, bins_per_box_x=bx)
    sim = E.Simulation(E.SimulationParams(**prm))
    mask = d["mask"] if d["mask"].size else None
    sim.add_agents(d["x"], d["y"], d["z"], d["d"], behaviour_mask=mask)
    sim.simulate(args.warmup)
    sim.synchronize()
    r0 = sim.report()
    sim.reset_timers(True)
    st = torch.cuda.ExternalStream(sim.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    sim.simulate(args.steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    fms, fl = sim.force_kernel_time()
    r1 = sim.report()
    n = r1.final_agent_count
    print(json.dumps({"lib": os.path.basename(os.environ.get("ABSIM_GPU_LIB", "default")), "bins": args.bin,
                      "lpa": os.environ.get("ABSIM_LPA", "default"),
                      "n": n, "ms_per_step": ms, "force_ms": fms / max(fl, 1),
                      "agent_it_per_s": n / (ms / 1e3),
                      "evals_per_agent": (r1.force_evaluations - r0.force_evaluations) / (n * args.steps)}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--libs", nargs="*", default=[])
    ap.add_argument("--bins", nargs="*", default=["2x1"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cache", default="/tmp/sweep_wl.npz")
    ap.add_argument("--lpas", nargs="*", default=[""])
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--bin", default="2x1")
    args = ap.parse_args()
    if args.child:
        return child(args)
    import numpy as np
    import bench
    t0 = time.time()
    wl = bench._workload(args.config, args.n)
    np.savez(args.cache, x=wl.x, y=wl.y, z=wl.z, d=wl.d,
             mask=wl.mask if wl.mask is not None else np.zeros(0, np.uint8),
             params=json.dumps(wl.params))
    print(f"# workload {wl.name} n={wl.n} generated in {time.time() - t0:.1f}s", flush=True)
    libs = args.libs or [""]
    for lib in libs:
        for b, lpa in [(b, q) for b in args.bins for q in args.lpas]:
            env = dict(os.environ)
            if lpa:
                env["ABSIM_LPA"] = lpa
            if lib:
                env["ABSIM_GPU_LIB"] = os.path.abspath(lib)
            subprocess.run([sys.executable, __file__, "--child", "--bin", b, "--cache", args.cache,
                            "--steps", str(args.steps), "--warmup", str(args.warmup)], env=env, timeout=900)


if __name__ == "__main__":
    main()
