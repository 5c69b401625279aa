"""Time spent inside the two C-ABI calls vs the whole drop-in step (C4 cycle, host arrays)."""
import sys, time
sys.path.insert(0, '.')
exec(open('tools/e2e_probe.py').read().split("ta = ts = 0.0")[0])
ctx = ws.bind(wells, streams)
acc = {"a": 0.0, "s": 0.0}
L = ctx.L
class Wrap:
    def __init__(self, lib): self._lib = lib
    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if name in ("isc_assemble_host", "isc_solve_host"):
            key = "a" if name == "isc_assemble_host" else "s"
            def timed(*args):
                t0 = time.perf_counter(); r = fn(*args); acc[key] += time.perf_counter() - t0; return r
            return timed
        return fn
ctx.L = Wrap(L)
tot = 0.0
for rep in range(3):
    for j in range(5):
        if rep == 1 and j == 0: acc["a"] = acc["s"] = 0.0; tot = 0.0
        t0 = time.perf_counter()
        blocks = assemble(grid, pack, ws, wells, streams, hs[j], accn_h, dt, dt, capped, freeze_upwind=j + 1 > 5)
        du, dbhp, _ = solver.solve(blocks)
        tot += time.perf_counter() - t0
print(f"per step: total {tot/10*1e3:.2f} ms, in isc_assemble_host {acc['a']/10*1e3:.2f}, in isc_solve_host {acc['s']/10*1e3:.2f}, python {(tot-acc['a']-acc['s'])/10*1e3:.3f} ms")
