import sys, threading, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'scripts'); sys.path.insert(0, 'tests')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF, distributed as D
from oracle import oracle as O
from debug_dist_threads import FakeDist
wl = CF.c3_spheroid(3000, seed=2)
world = 2; fd = FakeDist(world); res = {}
orc = O.PortSim(O.OracleParams(seed=2, dt=0.01, detect_static=True, model=2, mp=wl.params["model_params"]), wl.x, wl.y, wl.z, wl.d, wl.mask)
bar = threading.Barrier(world)
def run(rank):
    threading.current_thread().rank = rank
    torch.cuda.set_device(0)
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank, mask=wl.mask)
    sim = E.Simulation(E.SimulationParams(**wl.params), device=0)
    sim.add_agents(st["x"], st["y"], st["z"], st["d"], behaviour_mask=st["beh"], uid=st["uid"], uid_count=wl.n)
    dec = D.DeviceSlabDecomposition(sim, fd, rank, world, transport="host", cap=1 << 14)
    for s in range(5):
        dec.step()
        res[(rank, s)] = sim.agents()
        bar.wait()
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
mask = wl.mask
for s in range(5):
    orc.simulate(1)
    o = orc.dump(); oi = np.argsort(o["uid"])
    g = {k: np.concatenate([res[(r, s)][k] for r in range(world)]) for k in ("uid", "x", "flags")}
    gi = np.argsort(g["uid"])
    same_uid = np.array_equal(g["uid"][gi], o["uid"][oi])
    dx = np.abs(g["x"][gi] - o["x"][oi]) if same_uid else None
    bad = np.nonzero(dx > 1e-9 * np.maximum(1, np.abs(o["x"][oi])))[0] if same_uid else []
    print("step", s, "n", len(g["uid"]), "uids ok", same_uid, "bad", len(bad), "driven among bad", int(mask[o["uid"][oi][bad].astype(int)].sum()) if len(bad) else 0,
          "flags eq", np.array_equal(g["flags"][gi], o["flags"][oi]) if same_uid else None, flush=True)
    if len(bad): print("  sample uids", o["uid"][oi][bad][:8], "g", g["x"][gi][bad][:3], "o", o["x"][oi][bad][:3])
