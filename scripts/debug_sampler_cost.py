"""Timing perturbation of clock samplers: none / nvidia-smi process / NVML thread."""
import os
import subprocess
import sys
import threading
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF


class NvmlSampler:
    def __init__(self, idx=0, period=0.1):
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        self.period, self.samples, self.stop = period, [], threading.Event()

    def __enter__(self):
        self.t = threading.Thread(target=self.loop, daemon=True)
        self.t.start()
        time.sleep(0.05)
        return self

    def loop(self):
        while not self.stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((sm, rs))
            self.stop.wait(self.period)

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()


def make(kind):
    if kind == "c4":
        wl = CF.c4_large_uniform(1 << 24, 0)
        sim = E.Simulation(E.SimulationParams(**dict(wl.params, record_forces=False)))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    else:
        wl = CF.ref_proliferation(32768)
        sim = E.Simulation(E.SimulationParams(**dict(wl.params, capacity=3 * wl.n * 2 ** 7)))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
        sim.set_agent_ext(wl.tags, wl.rng_counters)
    sim.simulate(3)
    sim.synchronize()
    return sim


def timed(sim, steps):
    st = torch.cuda.ExternalStream(sim.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sim.simulate(steps)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for kind, steps in (("rprolif", 10), ("c4", 10)):
    for mode in ("none", "smi", "nvml", "none", "smi", "nvml"):
        sim = make(kind)
        if mode == "smi":
            p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                                  "clocks_event_reasons.active", "--format=csv,noheader", "-lms", "100"],
                                 stdout=subprocess.DEVNULL)
            time.sleep(0.3)
            ms = timed(sim, steps)
            p.terminate()
            p.wait()
        elif mode == "nvml":
            with NvmlSampler() as s:
                ms = timed(sim, steps)
        else:
            ms = timed(sim, steps)
        print(f"{kind} {mode:5s} {ms:9.3f} ms", flush=True)
        del sim
