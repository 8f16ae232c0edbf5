"""Debug: 2-rank device decomposition of config 2 with uid invariant checks
after every phase (simulate / commit / drop_ghosts)."""
import os
import sys
import tempfile

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def check(sim, what, rank, it):
    a = sim.agents()
    r = sim.report()
    u = a["uid"]
    bad = (u >= r.uid_count).sum()
    dup = len(u) - len(np.unique(u))
    if bad or dup:
        print(f"rank {rank} it {it} after {what}: n={len(u)} uid_count={r.uid_count} bad={bad} dup={dup} "
              f"sample={u[:8]} flags={a['flags'][:8]}", flush=True)
        return False
    return True


def worker(rank, world, port):
    import torch
    import torch.distributed as dist
    import paper_2301_06984_b200 as E
    from paper_2301_06984_b200 import configs as CF
    from paper_2301_06984_b200 import distributed as D
    from paper_2301_06984_b200 import _native as N
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    wl = CF.c2_proliferation(side=6, seed=0)
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=np.ones(wl.n, np.uint8))
    sim = E.Simulation(E.SimulationParams(**wl.params), device=0)
    sim.add_agents(st["x"], st["y"], st["z"], st["d"], behaviour_mask=st["beh"], uid=st["uid"], uid_count=wl.n)
    dec = D.DeviceSlabDecomposition(sim, dist, rank, world, transport="host", cap=1 << 14)
    ok = True
    for it in range(50):
        import paper_2301_06984_b200.distributed as DD
        # replicate step() with checks
        b = sim.local_bounds()
        red = dec._allreduce(np.concatenate([-b[:3], b[3:]]), dist.ReduceOp.MAX)
        g = D.global_grid(np.concatenate([-red[:3], red[3:]]), dec.fixed_box_length)
        L = D.layer_bounds(int(g.dims[2]), world)
        lo, hi = L[rank], L[rank + 1]
        n_lo, n_hi = dec._export(g, lo, hi, 0)
        got_lo, got_hi = dec._exchange(n_lo, n_hi)
        dec._import("recv_lo", got_lo, False)
        dec._import("recv_hi", got_hi, False)
        ok = ok and check(sim, "migrate", rank, it)
        n_lo, n_hi = dec._export(g, lo, hi, 1)
        got_lo, got_hi = dec._exchange(n_lo, n_hi)
        dec._import("recv_lo", got_lo, True)
        dec._import("recv_hi", got_hi, True)
        ok = ok and check(sim, "halo", rank, it)
        grid, dims = g.as_override()
        sim.set_grid_override(grid, dims)
        r0 = sim.report()
        sim.simulate(1)
        ok = ok and check(sim, "simulate", rank, it)
        dec._commit_additions()
        r1 = sim.report()
        ok = ok and check(sim, f"commit (staged->added {r1.agents_added - r0.agents_added})", rank, it)
        N.check(N.load().abs_gpu_drop_ghosts(sim._ctx), sim._ctx)
        ok = ok and check(sim, "drop_ghosts", rank, it)
        if not ok:
            break
    print(f"rank {rank} done ok={ok} n={sim.report().final_agent_count} uid_count={sim.report().uid_count}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(2, port), nprocs=2, join=True)
