"""Newton-iteration device time with and without per-kernel-class event
timing (KScope), to bound the profiling overhead inside bench.py's timed
region (the bench's Newton cycle: the first timestep's solving iterations)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from dataclasses import replace
from paper_1811_11992_b200 import configs, _native as N
from paper_1811_11992_b200.newton import Simulator
import bench

case = configs.config("c4")
case = replace(case, solver=replace(case.solver, precond="mcilu"))
grid, pack, wells, streams, state = configs.build_case(case)
sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
cyc = bench.NewtonCycle(sim, case.schedule.dt_init)
for _ in range(5):
    cyc.step()
for prof in (0, 1, 0, 1):
    N.check(sim.ctx.L.isc_set_profiling(sim.ctx.h, prof), "p")
    cyc.j = 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        cyc.step()
    e1.record()
    torch.cuda.synchronize()
    print("profiling", prof, "ms/step", e0.elapsed_time(e1) / 10, flush=True)
