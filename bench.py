"""bench.py — agent-iterations/s of the mechanical step on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE configs[3] ("c4"): 2^26 agents, uniform cube
at 12 mean neighbours, lognormal(ln 10, 0.1) diameters, dt 0.01 — the
largest single-GPU config and the one the north-star roofline target is
stated on. Inputs (2.5 GB of state) are far larger than L2 (126 MB), so no
explicit flush is needed between steps. `--config c1|c2|c3|c4` picks another.

One "step" = one full iteration (grid rebuild + radius query + repulsion +
displacement [+ staticness / behaviours / commit for c2/c3]).

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified absim engine with all host threads) on a bounded sample of
the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-iterations/sec for the mechanical step; achieved fraction of HBM roofline"
UNIT = "agent-iterations/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# initial population of each config at its default size (what the GPU arm's
# config reports as agents_per_gpu), without generating it
FULL_AGENTS = {"c1": 131_072, "c2": 16 ** 3, "c3": 1 << 23, "c4": 1 << 26, "c5": 10_000_000,
               "rclust": 1 << 22, "rprolif": 32768}


def _workload(name, n=None, seed=0):
    from paper_2301_06984_b200 import configs as CF
    if name == "c1":
        return CF.c1_relaxation(n or 131_072, seed)
    if name == "c2":
        return CF.c2_proliferation(side=16 if n is None else round(n ** (1 / 3)), seed=seed)
    if name == "c3":
        return CF.c3_spheroid(n or (1 << 23), seed)
    if name == "c5":
        return CF.c5_sir(n or 10_000_000, seed)
    if name == "rclust":  # the reference's own clustering benchmark (models::Cohere)
        return CF.ref_clustering(n or (1 << 22), seed=42 + seed)
    if name == "rprolif":  # the reference's own proliferation benchmark (models::GrowDivide)
        return CF.ref_proliferation(n or 32768)
    return CF.c4_large_uniform(n or (1 << 26), seed)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(k)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=None)
    return dist, world, rank, local


CPU_SAMPLE = {"c1": 131_072, "c2": None, "c3": 1 << 21, "c4": 1 << 22, "c5": 1 << 21, "rclust": 1 << 18,
              "rprolif": 4096}
CPU_STEPS = {"c1": 800, "c2": 60, "c3": 80, "c4": 30, "c5": 10, "rclust": 10, "rprolif": 18}
REF_BUILDERS = {"ref_clustering": "clustering", "ref_proliferation": "proliferation"}


ENV_IDS = {"uniform_grid": 0, "brute_force": 1, "kdtree": 2}


def _ref_sim(wl_name, sample_n, threads, env="uniform_grid"):
    """The reference engine (oracle/_ref, unmodified absim) on a bounded
    sample of the workload; falls back to the C port if it is not built."""
    from oracle import oracle as O
    wl = _workload(wl_name, sample_n, seed=0)
    prm = wl.params
    p = O.OracleParams(seed=prm.get("seed", 0), dt=prm.get("simulation_time_step", 0.1),
                       detect_static=prm.get("detect_static_agents", False),
                       model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8),
                       sorting_frequency=prm.get("sorting_frequency", 0), threads=threads, domains=0,
                       fixed_box=prm.get("fixed_box_length", 0.0), env=ENV_IDS[env])
    try:
        if prm.get("model", 0) == 4:  # SIR: periodic cube as ghost images over the reference engine
            return O.RefSirSim(p, wl.x, wl.y, wl.z), "reference", threads, wl
        if wl.name in REF_BUILDERS:  # the reference's own population builder and models
            return O.RefSim.builtin(p, REF_BUILDERS[wl.name], wl.n), "reference", threads, wl
        return O.RefSim(p, wl.x, wl.y, wl.z, wl.d, wl.mask), "reference", threads, wl
    except (FileNotFoundError, OSError):
        p.threads = 1
        s = O.PortSim(p, wl.x, wl.y, wl.z, wl.d, wl.mask)
        if wl.tags is not None:
            s.set_tags(wl.tags)
            s.set_rng_counters(wl.rng_counters)
        return s, "port", 1, wl


BRUTE_SAMPLE, BRUTE_STEPS = 16384, 4  # O(N^2) reference: a smaller bounded sample


def cpu_baseline(wl_name, steps=None, threads=None, env="uniform_grid"):
    """Reference CPU throughput on a bounded sample (population built untimed)."""
    threads = threads or os.cpu_count()
    brute = env == "brute_force"
    steps = steps or (BRUTE_STEPS if brute else CPU_STEPS[wl_name])
    sim, kind, cores, wl = _ref_sim(wl_name, BRUTE_SAMPLE if brute else CPU_SAMPLE[wl_name], threads, env)
    agent_its = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        agent_its += sim.counts()["agents"]
        sim.simulate(1)
    wall = time.perf_counter() - t0
    return {"value": agent_its / wall, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{wl.name} shape from {wl.n} agents x {steps} iterations "
                      f"({agent_its} agent-iterations, same density and distributions), {wall:.1f} s of CPU wall time"}


def _workload_config(args, wl_name, n, world):
    """The workload keys of a bench line, identical for the GPU and reference arms."""
    state_mb = int(n) * 128 / 1e6  # positions (2 x 32 B) + uid, flags, partners, keys, fp32 copies
    if state_mb > 4 * 126:
        l2 = f"state {state_mb / 1e3:.1f} GB per GPU >> 126 MB L2, no flush"
    else:
        l2 = (f"state {state_mb:.0f} MB per GPU does not exceed the 126 MB L2 by much: every iteration reads the "
              f"state the previous one wrote (the simulation's own data flow), no flush between iterations")
    return {"workload": wl_name, "agents_per_gpu": int(n), "global_agents": int(n) * world,
            "parallelism": "single" if world == 1 else f"replicas{world}", "environment": args.env,
            "l2": l2}


def run_reference(args):
    """--impl reference: each step is one iteration of the unmodified reference
    (oracle/_ref, all host cores) on the SAME population the GPU arm simulates
    at N=1 (config.agents_per_gpu equal: c4 = 2^26 agents, ~8 s per iteration
    on 16 cores, so the driver's 5 + 20 iterations take ~4 min; the population
    build is untimed). Under torchrun (N>1) rank 0 alone runs one GPU's share.
    --ref-sample N times a smaller sample of the same shape instead."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count()
    brute = args.env == "brute_force"
    n = BRUTE_SAMPLE if brute else (args.ref_sample or args.n or FULL_AGENTS[args.config])
    if args.config == "c2":
        n = None  # the proliferation run starts from its 16^3 lattice
    t_build = time.perf_counter()
    sim, kind, cores, wl = _ref_sim(args.config, n, threads, args.env)
    t_build = time.perf_counter() - t_build
    for _ in range(args.warmup):
        sim.simulate(1)
    agent_its = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        agent_its += sim.counts()["agents"]
        sim.simulate(1)
    wall = time.perf_counter() - t0
    v = agent_its / wall
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            # the GPU arm's workload keys, with the population this run actually timed
            "config": _workload_config(args, wl.name, wl.n, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{wl.name} at {wl.n} agents (the GPU arm's N=1 population"
                                       f"{'' if wl.n == FULL_AGENTS.get(args.config, wl.n) else ': a bounded sample'}), "
                                       f"{args.steps} timed iterations after {args.warmup} warm-up; "
                                       f"population built in {t_build:.1f} s (untimed)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.gpus > 1:
        line["config"]["note"] = f"reference on rank 0 of {args.gpus}: one GPU's share of the weak-scaling run"
    print(json.dumps(line))


def _slab_workload(n_per, world, rank, seed=0):
    """Weak-scaling c4 (configs[3]): world * n_per agents uniform in one cube at
    12 mean neighbours; rank r generates the agents of its z-slab (uids
    r * n_per + i), lognormal(ln 10, 0.1) diameters from rng_word."""
    import numpy as np
    from paper_2301_06984_b200 import configs as CF
    L = (n_per * world / CF.DENSITY) ** (1.0 / 3.0)
    uid = np.arange(n_per, dtype=np.uint64) + np.uint64(rank * n_per)
    x = CF.u01(CF.rng_word(seed, uid, 0)) * L
    y = CF.u01(CF.rng_word(seed, uid, 1)) * L
    z = (rank + CF.u01(CF.rng_word(seed, uid, 2))) * (L / world)
    u1 = 1.0 - CF.u01(CF.rng_word(seed, uid, 4))
    u2 = CF.u01(CF.rng_word(seed, uid, 5))
    d = np.exp(math.log(10.0) + 0.1 * (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)))
    return x, y, z, d, uid, L


def _decomposed_workload(args, world, rank):
    """(x, y, z, d, mask, uid, uid_count, params, name, scaling, per-rank
    nominal agents) of this rank's slab. c4 weak: 2^26 agents per GPU in one
    cube; c4 strong: 2^26 in total; c3 (strong): the 2^23-agent spheroid split
    into equal-count slabs (distributed.balanced_bounds, the device driver's
    own edges)."""
    import numpy as np
    from paper_2301_06984_b200 import distributed as D
    if args.config == "c3":
        wl = _workload("c3", args.n, args.seed)
        st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=wl.mask, balanced=True)
        prm = dict(wl.params)
        return (st["x"], st["y"], st["z"], st["d"], st["beh"], st["uid"], wl.n, prm, wl.name, "strong",
                wl.n / world)
    strong = args.scaling == "strong"
    total = args.n or (1 << 26)
    n_per = total // world if strong else total
    x, y, z, d, uid, L = _slab_workload(n_per, world, rank, args.seed)
    prm = dict(seed=args.seed, simulation_time_step=0.01)
    return (x, y, z, d, None, uid, n_per * world, prm, "c4_large_uniform", "strong" if strong else "weak", n_per)


def run_decomposed(args, dist, world, rank, local):
    """N GPUs: the library's slab decomposition (csrc/decomp.cuh) over NCCL."""
    import torch

    import paper_2301_06984_b200 as E
    from paper_2301_06984_b200 import distributed as D
    x, y, z, d, mask, uid, uid_count, prm, name, scaling, n_nominal = _decomposed_workload(args, world, rank)
    n_per = len(x)
    prm = dict(prm, record_forces=False, bins_per_box=args.bins, bins_per_box_x=args.bins_x,
               capacity=int(max(n_per, n_nominal) * 1.3) + 1024)
    sim = E.Simulation(E.SimulationParams(**prm), device=local)
    sim.add_agents(x, y, z, d, behaviour_mask=mask, uid=uid, uid_count=uid_count)
    dec = D.DeviceSlabDecomposition(sim, dist, rank, world, transport="nccl",
                                    cap=int(0.06 * n_per) + (1 << 20))
    dec.simulate(args.warmup)
    stream = torch.cuda.ExternalStream(sim.stream)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = sim.report().kernel_launches
    sim.reset_timers(True)
    with Clocks(local) as clk:
        e0.record(stream)
        dec.simulate(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    force_ms, force_launches = sim.force_kernel_time()
    sim.reset_timers(False)
    launches = torch.tensor([float(sim.report().kernel_launches - l0)], device="cuda")
    dist.all_reduce(launches)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    owned = torch.tensor([float(dec.info()[1])], device="cuda")
    dist.all_reduce(owned)
    total = float(owned.item())
    value = total * args.steps / (ms_max / 1e3)
    evals_per_agent_step = dec.totals()[0] / max(1.0, total * (args.steps + args.warmup))

    # end to end per rank through the public API with HOST buffers: upload the
    # rank's slab from page-locked memory, one decomposed iteration (bounds
    # all-reduce, migration + halo over NCCL), positions back to page-locked
    # memory; wall time between barriers, max over ranks
    e2e = None
    if not args.no_e2e:
        import numpy as np
        pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (x, y, z, d, uid)]
        outp = [torch.empty(int(n_per * 1.3), dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
        e2e_steps = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        n_e = 0
        it = args.warmup + args.steps
        for k in range(e2e_steps):
            sim.add_agents(*pin[:4], behaviour_mask=mask, uid=pin[4], uid_count=uid_count)
            sim.set_iteration(it + k)
            dec.simulate(1)
            n_e = sim.positions(*outp)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": uid_count * e2e_steps / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": uid_count * 40, "d2h_bytes_per_step": n_e * 24 * world,
               "steps": e2e_steps, "timing": "wall clock between barriers, max over ranks",
               "path": "per rank: abs_gpu_upload (pinned) -> decomposed iteration -> abs_gpu_download (pinned)"}
    if rank == 0:
        hbm, peak_src = _peaks()
        bpa = 134 if args.config == "c3" else 128
        step_bytes = bpa * (total / world) * args.steps
        # rank 0's k_force (owned agents + ghosts stepped as candidates only):
        # 56 B per owned agent per launch over its CUDA-event average
        avg_force_ms = force_ms / max(1, force_launches)
        achieved = 56 * sim.agent_count() / (avg_force_ms / 1e3) / 1e9 if avg_force_ms > 0 else 0.0
        roofline = {"bound": "hbm", "kernel": "k_force", "achieved": achieved, "peak": hbm, "peak_source": peak_src,
                    "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                    "algorithmic_bytes_per_launch": 56 * sim.agent_count(), "avg_launch_ms": avg_force_ms,
                    "rank": 0}
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{name} ({scaling} scaling)", "agents_per_gpu": int(n_nominal),
                       "global_agents": int(total),
                       "parallelism": f"slab{world} (equal-count z slabs, NCCL halo + migration, library-driven)",
                       "l2": f"state {int(n_nominal) * 128 / 1e9:.2f} GB per GPU against the 126 MB L2, no flush"},
            "roofline": roofline,
            "step_roofline": {"bytes_per_agent_iteration": bpa, "unit": "GB/s",
                              "achieved_per_gpu": step_bytes / (ms_max / 1e3) / 1e9,
                              "frac": step_bytes / (ms_max / 1e3) / 1e9 / hbm},
            "clocks": clk.summary(),
            "force_evaluations_per_agent_step": evals_per_agent_step,
            "e2e": e2e, "gpu_launches": int(launches.item()),
            "gpu_launches_note": "all ranks: engine kernels + export/import/compaction",
        }))


def run_gpu(args):
    import numpy as np
    import torch

    import paper_2301_06984_b200 as E

    dist, world, rank, local = _dist() if int(os.environ.get("WORLD_SIZE", "1")) > 1 else (None, 1, 0, 0)
    torch.cuda.set_device(local)
    if world > 1 or args.decompose:
        if args.config not in ("c4", "c3"):
            raise SystemExit("the multi-GPU bench decomposes configs c4 (weak or strong) and c3 (strong)")
        if dist is None:
            import torch.distributed as dist0
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist0.init_process_group("nccl", rank=0, world_size=1)
            dist = dist0
        run_decomposed(args, dist, world, rank, local)
        dist.barrier()
        dist.destroy_process_group()
        return
    wl = _workload(args.config, args.n, seed=args.seed + rank)
    prm = dict(wl.params)
    prm["record_forces"] = False
    prm["environment"] = args.env
    prm["bins_per_box"] = args.bins
    prm["bins_per_box_x"] = args.bins_x
    prm["neighbor_list"] = args.lists != "off"
    prm["neighbor_skin"] = args.skin
    if wl.params.get("model") == E.MODEL_PROLIFERATION:
        prm["capacity"] = 5 * wl.n * 2 ** 9
    if wl.params.get("model") == E.MODEL_GROW_DIVIDE:  # doubles every 3 iterations
        prm["capacity"] = 3 * wl.n * 2 ** ((args.warmup + args.steps + 8) // 3)
    sim = E.Simulation(E.SimulationParams(**prm), device=local)
    sim.add_agents(wl.x, wl.y, wl.z, wl.d, behaviour_mask=wl.mask)
    if wl.tags is not None:
        sim.set_agent_ext(wl.tags, wl.rng_counters)
    stream = torch.cuda.ExternalStream(sim.stream)

    sim.simulate(args.warmup)
    sim.synchronize()
    r0 = sim.report()
    sim.reset_timers(False)  # the headline window records no per-iteration phase events
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        sim.simulate(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    r1 = sim.report()
    # the dominant kernel's average launch time: a few more iterations with the
    # per-launch CUDA events on (they cost launch-bound configs ~10-15 %)
    kr = max(1, min(args.steps, 5))
    sim.reset_timers(True)
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    sim.simulate(kr)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_r = e2.elapsed_time(e3)
    force_ms, force_launches = sim.force_kernel_time()
    lists = sim.list_stats()
    sim.reset_timers(False)
    r2 = sim.report()
    # the device sums every iteration's agent count at its start (exact for
    # growing populations, as the reference arm's per-step sum)
    agent_its = r1.agent_iterations - r0.agent_iterations
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        a = torch.tensor([float(agent_its)], device="cuda")
        dist.all_reduce(a)
        agent_its = float(a.item())
    value = agent_its / (ms_max / 1e3)

    # end to end through the public API with HOST buffers: every step uploads
    # the step's input state (x, y, z, d) from page-locked host memory, runs the
    # iteration and reads the resulting positions back into page-locked memory
    e2e = None
    sir_model = wl.params.get("model") == E.MODEL_SIR
    if not args.no_e2e and rank == 0:
        pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (wl.x, wl.y, wl.z, wl.d)]
        mask = None if wl.mask is None else torch.from_numpy(wl.mask).pin_memory().numpy()
        outp = [torch.empty(wl.n, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
        # a host-driven loop continues the step numbering after each upload
        # (set_iteration), so periodic work (sorting_frequency) keeps its cadence
        it = sim.iteration
        ext = None
        if wl.tags is not None:  # per-agent tags / stream counters travel with the state
            ext = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (wl.tags, wl.rng_counters)]
        sim.add_agents(*pin, behaviour_mask=mask)
        if ext:
            sim.set_agent_ext(*ext)
        sim.set_iteration(it)
        sim.simulate(1)
        sim.positions(*outp)
        e2e_steps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            sim.add_agents(*pin, behaviour_mask=mask)
            if ext:
                sim.set_agent_ext(*ext)
            sim.set_iteration(it + 1 + k)
            sim.simulate(1)
            n_e = sim.positions(*outp)
        dt = time.perf_counter() - t0
        seq = {"value": wl.n * e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": wl.n * (32 + (1 if wl.mask is not None else 0) + (12 if ext else 0)),
               "d2h_bytes_per_step": n_e * 24, "steps": e2e_steps,
               "path": "abs_gpu_upload (pinned host) -> abs_gpu_simulate(1) -> abs_gpu_download (pinned host)"}
        e2e = seq
        if mask is None and ext is None and not sir_model:
            # the same per-step work through abs_gpu_run_frames: every frame
            # uploads its inputs from page-locked memory, runs one iteration
            # and downloads the positions, with the next frame's H2D and the
            # previous frame's D2H overlapping this frame's compute
            frames = max(5, min(args.steps, 20))
            outs = [outp, [torch.empty(wl.n, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]]
            it2 = it + 1 + e2e_steps
            sim.run_frames([pin] * 2, outs, iterations=1, first_iteration=it2)  # staging allocated untimed
            it2 += 2
            t0 = time.perf_counter()
            counts = sim.run_frames([pin] * frames, [outs[f % 2] for f in range(frames)], iterations=1,
                                    first_iteration=it2)
            dt = time.perf_counter() - t0
            e2e = {"value": wl.n * frames / dt, "unit": UNIT, "h2d_bytes_per_step": wl.n * 32,
                   "d2h_bytes_per_step": counts[-1] * 24, "steps": frames,
                   "path": "abs_gpu_run_frames: per step H2D x,y,z,d (pinned) -> ingest -> 1 iteration -> "
                           "D2H x,y,z (pinned); copies of neighbouring steps overlap on two copy streams",
                   "sequential": seq}
            # how a caller runs the config itself: one upload, K iterations on the device, one download
            # (the copies amortise over the run; reported beside the per-step figure, not instead of it;
            # constant populations only: the pinned output arrays hold the initial agent count)
            if not wl.params.get("model"):
                t0 = time.perf_counter()
                sim.add_agents(*pin, behaviour_mask=mask)
                sim.set_iteration(0)
                sim.simulate(args.steps)
                n_w = sim.positions(*outp)
                dt = time.perf_counter() - t0
                e2e["whole_run"] = {"value": wl.n * args.steps / dt, "unit": UNIT, "steps": args.steps,
                                    "h2d_bytes": wl.n * 32, "d2h_bytes": n_w * 24,
                                    "path": "abs_gpu_upload (pinned host) once -> abs_gpu_simulate(steps) -> "
                                            "abs_gpu_download (pinned host) once"}

    hbm, peak_src = _peaks()
    n_agents = (r1.final_agent_count + r2.final_agent_count) // 2  # during the kernel-event pass
    avg_force_ms = force_ms / max(1, force_launches)
    sir = wl.params.get("model") == E.MODEL_SIR
    # k_force: read {x,y,z,d} 32 B + write {x,y,z} 24 B per agent;
    # k_sir (config 5): read {x,y,z,state} 28 B + write {x,y,z,state} 28 B
    force_bytes = 56 * n_agents
    achieved = force_bytes / (avg_force_ms / 1e3) / 1e9 if avg_force_ms > 0 else 0.0
    step_bytes = wl.bytes_per_agent_iteration * agent_its / max(1, world)
    step_achieved = step_bytes / (ms / 1e3) / 1e9
    traffic = None
    issue = None
    tp = os.path.join(ROOT, "profiles", "force_traffic.json")
    kernel_name = "k_sir" if sir else ("k_force_list" if lists["list_steps"] else "k_force")
    if os.path.exists(tp):  # ncu --set full figures of the same workload, per kernel (profiles/r2/)
        try:
            with open(tp) as f:
                tt = json.load(f).get(args.config, {})
            if tt.get("agents") == n_agents and kernel_name in tt:
                tk = tt[kernel_name]
                traffic = tk.get("dram_bytes_per_launch")
                issue = {k: tk[k] for k in ("issue_active_pct", "warps_active_pct", "l1_hit_pct", "l2_hit_pct",
                                            "warp_instructions_per_agent", "kernels") if k in tk}
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _workload_config(args, wl.name, wl.n, world),
        "device_knobs": {"bins_per_box": [args.bins_x, args.bins, args.bins], "lists": args.lists, "skin": args.skin},
        # k_force_list = the list step's force work, k_list_scan + k_list_forces, timed as one event pair
        "roofline": {"bound": "hbm", "kernel": kernel_name,
                     "achieved": achieved, "peak": hbm,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "algorithmic_bytes_per_launch": force_bytes,
                     "avg_launch_ms": avg_force_ms, "force_share_of_step": force_ms / ms_r,
                     "timing": f"CUDA events around each launch over {kr} further iterations",
                     # the binding limit is instruction issue / load latency, not HBM: the same
                     # capture's issue-slot utilisation (profiles/force_traffic.json)
                     "ncu_issue": issue},
        "step_roofline": {"bytes_per_agent_iteration": wl.bytes_per_agent_iteration,
                          "achieved": step_achieved, "frac": step_achieved / hbm, "unit": "GB/s"},
        "clocks": clk.summary(),
        "gpu_launches": int(r1.kernel_launches - r0.kernel_launches),
        "force_evaluations_per_agent_step": (r1.force_evaluations - r0.force_evaluations) / max(1, agent_its / world),
        "lists": lists,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        # c2 grows from its 16^3 lattice: the reference runs the same iterations as the GPU arm
        # (warm-up + timed steps; 200 iterations reach ~2.1 M agents, ~10 s on 16 cores)
        c2_steps = (args.warmup + args.steps) if args.config == "c2" else None
        line["cpu_baseline"] = cpu_baseline(args.config, steps=c2_steps, env=args.env)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "rclust", "rprolif"])
    ap.add_argument("--agents", "--n", dest="n", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--bins", type=int, default=0, help="sub-bins per box edge along y, z (0 = auto)")
    ap.add_argument("--bins-x", type=int, default=0, help="sub-bins per box edge along x (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--lists", default="auto", choices=["auto", "off"],
                    help="neighbour lists between environment rebuilds (DESIGN.md §4b)")
    ap.add_argument("--skin", type=float, default=0.0, help="neighbour-list skin (0 = auto)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="--impl reference: time a bounded sample of this many agents instead of the full population")
    ap.add_argument("--decompose", action="store_true", help="use the slab decomposition even at N=1")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="c4 under torchrun: 2^26 agents per GPU (weak) or in total (strong)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--env", default="uniform_grid", choices=["uniform_grid", "brute_force", "kdtree"],
                    help="EnvironmentKind (params.hpp:9); brute_force / kdtree = the comparison baselines")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
