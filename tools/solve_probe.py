"""Drop-in API timing split: assemble(host State) / BlockSolver.solve -> host du (C4 cycle)."""
import sys, time, numpy as np, torch, ctypes
sys.path.insert(0, '.')
exec(open('tools/e2e_probe.py').read().split("ta = ts = 0.0")[0])
from paper_1811_11992_b200 import _native as N
ctx = None
t_solve = t_dl = t_asm = 0.0
for rep in range(3):
    for j in range(5):
        t0 = time.perf_counter()
        blocks = assemble(grid, pack, ws, wells, streams, hs[j], accn_h, dt, dt, capped, freeze_upwind=j + 1 > 5)
        t1 = time.perf_counter()
        du, dbhp, _ = solver.solve(blocks)
        t2 = t3 = time.perf_counter()
        if rep: t_asm += t1 - t0; t_solve += t2 - t1; t_dl += t3 - t2
print(f"assemble {t_asm/10*1e3:.2f}  solve (host du) {t_solve/10*1e3:.2f} ms")
