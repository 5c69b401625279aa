import sys, numpy as np
sys.path.insert(0, '.')
from tests.helpers import case_objects
from tests.golden_states import random_state_like_reference
from paper_1811_11992_b200.assembly import Workspace, assemble
from paper_1811_11992_b200.device import soa_from_rows, state_to_device
c = case_objects("c4")
st, accn = random_state_like_reference(c, 43)
capped = np.zeros(len(c.wells), dtype=bool)
ws_d = Workspace(c.grid, c.pack, None, wells=c.wells, streams=c.streams, precond="mcilu")
ctx = ws_d.bind(c.wells, c.streams)
wout_d = ctx.assemble(state_to_device(st, ctx.device), st.bhp, soa_from_rows(accn, ctx.device), 2e-3, 2e-3, capped, False)
r0 = ctx.copy_out(0, 9).cpu().numpy()
import torch
d0 = torch.empty(1); 
ws_h = Workspace(c.grid, c.pack, None, wells=c.wells, streams=c.streams, precond="mcilu")
for rep in range(5):
    assemble(c.grid, c.pack, ws_h, c.wells, c.streams, st, accn, 2e-3, 2e-3, capped)
    r1 = ws_h.ctx.copy_out(0, 9).cpu().numpy()
    print(rep, "resid equal:", np.array_equal(r0, r1), "wout equal:", np.array_equal(ws_h.last_wout, wout_d))
# full blocks once
ws_d._invalidate(); ws_h._invalidate()
print("diag equal:", np.array_equal(ws_d.diag, ws_h.diag), "offd equal:", np.array_equal(ws_d.offd, ws_h.offd))
