"""C5-type synthetic system (seeded BSR of BASELINE configs[4]) at a reduced nz:
BiCGSTAB iterations and solve time per preconditioner (mcilu / ras / bjacobi / none).
    python tools/c5_precond_probe.py [nz]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_11992_b200 import _native as N
from paper_1811_11992_b200.device import DeviceContext
from paper_1811_11992_b200.grid import build_grid
from paper_1811_11992_b200.model import load_pack

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 40
grid = build_grid(400, 400, nz, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
pack = load_pack("tube3_pack", grid.phi_ref)
for pre in sys.argv[2:] or ["mcilu", "ras", "bjacobi", "none"]:
    ctx = DeviceContext(grid, pack, (), (), pre)
    N.check(ctx.L.isc_synth_system(ctx.h, 7), "synth")
    bc, bcol, it = ctypes.c_int64(-1), ctypes.c_int32(-1), ctypes.c_int32(0)
    N.check(ctx.L.isc_decouple(ctx.h, ctypes.byref(bc), ctypes.byref(bcol)), "decouple")
    du = torch.empty(9, grid.ncell, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        torch.cuda.synchronize()
        e0.record()
        st = ctx.L.isc_solve(ctx.h, 1e-8, 1000, N.ptr(du), N.VP(0), ctypes.byref(it),
                             ctypes.byref(bc), ctypes.byref(bcol))
        e1.record()
        torch.cuda.synchronize()
        print(f"{pre:8s} nz={nz} rows={grid.ncell} status={st} iters={it.value} "
              f"solve_ms={e0.elapsed_time(e1):.1f}", flush=True)
    ctx.close()
    del du
    torch.cuda.empty_cache()
