"""Does a concurrent nvidia-smi sampler stall a launch-bound run?"""
import os
import subprocess
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF


def run(sampler):
    wl = CF.ref_proliferation(32768)
    sim = E.Simulation(E.SimulationParams(**dict(wl.params, capacity=3 * wl.n * 2 ** 7)))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    sim.set_agent_ext(wl.tags, wl.rng_counters)
    sim.simulate(3)
    sim.synchronize()
    p = None
    if sampler:
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                             stdout=subprocess.DEVNULL)
        time.sleep(0.3)
    st = torch.cuda.ExternalStream(sim.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    sim.simulate(10)
    e1.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if p:
        p.terminate()
        p.wait()
    print(f"sampler={sampler} events {e0.elapsed_time(e1):.2f} ms wall {wall*1e3:.2f} ms n={sim.report().final_agent_count}",
          flush=True)


for s in (False, True, False, True):
    run(s)
