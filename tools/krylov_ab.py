"""A/B of the Krylov method on the mcilu red-eliminated system: BiCGSTAB vs
GMRES(m) on C4 Newton systems (perturbed states, as tests/test_gpu_fullsize)
and on the C1-C3 decks — iterations, solve time, and agreement of du."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_11992_b200 import _native as N, configs
from paper_1811_11992_b200.device import DeviceContext, state_to_device
from tests.golden_states import perturb


def run(name, tol):
    case = configs.config(name)
    grid, pack, wells, streams, state = configs.build_case(case)
    ctx = DeviceContext(grid, pack, wells, streams, "mcilu")
    zero = torch.zeros(9, grid.ncell, dtype=torch.float64, device=ctx.device)
    ctx.assemble(state_to_device(state, ctx.device), state.bhp, zero, 1.0, 0.0,
                 np.zeros(len(wells), bool), False)
    accn = ctx.copy_out(1, 9).t().contiguous().cpu().numpy()
    for seed in (23, 5):
        st, acc = perturb(state, accn, seed)
        d_st = state_to_device(st, ctx.device)
        d_acc = torch.from_numpy(np.ascontiguousarray(acc.T)).to(ctx.device)
        res = {}
        for kry, m in (("bicgstab", 0), ("gmres", 10), ("gmres", 20), ("gmres", 30)):
            ctx.set_krylov(kry, m)
            ts = []
            for rep in range(3):
                ctx.assemble(d_st, st.bhp, d_acc, 2e-3, 2e-3, np.zeros(len(wells), bool), False)
                du = ctx.empty(9, grid.ncell)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                try:
                    dbhp, it = ctx.solve(tol, 400, du)
                except Exception as e:   # noqa
                    print(name, seed, kry, m, "FAILED", e, flush=True)
                    it = -1
                    break
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            if it < 0:
                continue
            res[(kry, m)] = du.cpu().numpy()
            ref = res[("bicgstab", 0)]
            rel = np.linalg.norm(res[(kry, m)] - ref) / np.linalg.norm(ref)
            print(f"{name} seed {seed} {kry:8s} m={m:2d} iters {it:3d} solve {min(ts)*1e3:8.2f} ms"
                  f"  |du-du_bicg|/|du| {rel:.2e}", flush=True)
    ctx.close()


for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    run(name, 1e-5)
