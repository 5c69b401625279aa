import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1811_11992_b200 import configs
from paper_1811_11992_b200.assembly import Workspace, assemble
from paper_1811_11992_b200.linsolve import BlockSolver
from paper_1811_11992_b200.newton import Simulator
case = configs.config("c4")
from dataclasses import replace
case = replace(case, solver=replace(case.solver, precond="mcilu"))
grid, pack, wells, streams, state = configs.build_case(case)
sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
cyc = bench.NewtonCycle(sim, case.schedule.dt_init)
host_states = []
for _ in range(5):
    cur = cyc.work if cyc.j % 5 else cyc.init
    host_states.append(cur.to_host()); cyc.step()
ws = Workspace(grid, pack, None, wells=wells, streams=streams, precond="mcilu")
solver = BlockSolver(grid, ws, tol=case.solver.linear_tol, maxiter=case.solver.linear_max, precond="mcilu")
from types import SimpleNamespace
hs = [SimpleNamespace(**{k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy() for k, v in h.items()}) for h in host_states]
accn_h = torch.from_numpy(np.ascontiguousarray(sim.accn.t().cpu().numpy())).pin_memory().numpy()
capped = sim.capped.copy(); dt = case.schedule.dt_init
ta = ts = 0.0
for rep in range(3):
    for j in range(5):
        t0 = time.perf_counter()
        blocks = assemble(grid, pack, ws, wells, streams, hs[j], accn_h, dt, dt, capped, freeze_upwind=j + 1 > 5)
        t1 = time.perf_counter()
        du, dbhp, _ = solver.solve(blocks)
        t2 = time.perf_counter()
        if rep: ta += t1 - t0; ts += t2 - t1
print(f"e2e per step: assemble {ta/10*1e3:.2f} ms, solve {ts/10*1e3:.2f} ms, total {(ta+ts)/10*1e3:.2f} ms")
ctx = ws.ctx
import ctypes
st = ctx.stage_times() if hasattr(ctx, 'stage_times') else None
print('stage times (cumulative)', st)
