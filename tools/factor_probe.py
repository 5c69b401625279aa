"""Time the multicolour factorisation alone on a decoupled C4 system
(isc_precond_setup, repeated; A/B builds of the factor kernel)."""
import ctypes
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1811_11992_b200 import _native as N, configs
from paper_1811_11992_b200.device import DeviceContext, state_to_device

case = configs.config("c4")
grid, pack, wells, streams, state = configs.build_case(case)
ctx = DeviceContext(grid, pack, wells, streams, "mcilu")
zero = torch.zeros(9, grid.ncell, dtype=torch.float64, device=ctx.device)
ctx.assemble(state_to_device(state, ctx.device), state.bhp, zero, 2e-3, 2e-3,
             np.zeros(len(wells), bool), False)
bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
N.check(ctx.L.isc_decouple(ctx.h, ctypes.byref(bc), ctypes.byref(bcol)), "decouple")
for _ in range(2):
    ctx.L.isc_precond_setup(ctx.h, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ctx.L.isc_precond_setup(ctx.h, None)
e1.record()
torch.cuda.synchronize()
print("factor ms", e0.elapsed_time(e1) / 10, "form", ctx.decoupled_form)
