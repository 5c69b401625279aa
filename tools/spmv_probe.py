import sys, json
sys.path.insert(0, '.')
import torch, numpy as np
from paper_1811_11992_b200 import _native as N
from paper_1811_11992_b200.grid import build_grid
from paper_1811_11992_b200.model import load_pack
from paper_1811_11992_b200.device import DeviceContext
import ctypes
def run(nx, ny, nz, steps=20):
    grid = build_grid(nx, ny, nz, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    pack = load_pack("tube3_pack", grid.phi_ref)
    ctx = DeviceContext(grid, pack, (), (), "none")
    N.check(ctx.L.isc_synth_system(ctx.h, 7), "synth")
    bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
    N.check(ctx.L.isc_decouple(ctx.h, ctypes.byref(bc), ctypes.byref(bcol)), "decouple")
    x = torch.randn(9, grid.ncell, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): ctx.L.isc_spmv(ctx.h, N.ptr(x), N.ptr(y))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): ctx.L.isc_spmv(ctx.h, N.ptr(x), N.ptr(y))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nbytes = 8 * (162 * grid.nconn + 18 * grid.ncell)
    ctx.close()
    return ms, nbytes / ms / 1e6
for dims in [(400, 400, 50), (399, 400, 50)]:
    print(dims, run(*dims))
