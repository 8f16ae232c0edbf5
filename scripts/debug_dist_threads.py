"""Two ranks as threads in one process (in-process collectives) — debugging aid."""
import sys, threading, numpy as np, torch
sys.path.insert(0, '.')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF, distributed as D

class FakeDist:
    class ReduceOp:
        MAX, SUM = "max", "sum"
    def __init__(self, world):
        self.world = world; self.bar = threading.Barrier(world); self.buf = {}; self.lock = threading.Lock()
    def all_reduce(self, t, op):
        me = threading.current_thread().rank
        with self.lock: self.buf[("ar", me)] = t.clone()
        self.bar.wait()
        vals = [self.buf[("ar", r)] for r in range(self.world)]
        res = vals[0].clone()
        for v in vals[1:]: res = torch.maximum(res, v) if op == "max" else res + v
        self.bar.wait(); t.copy_(res)
    class _Op:
        def wait(self): pass
    def isend(self, t, p):
        me = threading.current_thread().rank
        with self.lock: self.buf.setdefault(("p2p", me, p), []).append(t.clone())
        return FakeDist._Op()
    def irecv(self, t, p):
        me = threading.current_thread().rank
        d = self
        class R:
            def wait(self_):
                while True:
                    with d.lock:
                        q = d.buf.get(("p2p", p, me))
                        if q: t.copy_(q.pop(0)); return
        return R()

wl = CF.c1_relaxation(3000, seed=1)
world = 2; fd = FakeDist(world); out = {}
def run(rank):
    threading.current_thread().rank = rank
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank)
    eng = D.GpuRankEngine(E.SimulationParams(**wl.params), device=0)
    dec = D.SlabDecomposition(eng, fd, rank, world, st, uid_count=wl.n)
    for s in range(6):
        dec.step()
        print("rank", rank, "step", s, "owned", len(dec.state["x"]), flush=True)
    out[rank] = dec.state
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
print("done", {r: len(v["x"]) for r, v in out.items()})
