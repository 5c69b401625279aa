import numpy as np, sys
sys.path.insert(0, '.')
from tests.helpers import case_objects, golden, state_from
from paper_1811_11992_b200.assembly import Workspace, assemble
g = golden("asm_small3d.npz"); gn = golden("numjac_small3d.npz")
c = case_objects("small3d")
ws = Workspace(c.grid, c.pack, None, wells=c.wells, streams=c.streams, precond="ras")
dt = float(g["dt"])
assemble(c.grid, c.pack, ws, c.wells, c.streams, state_from(g), g["accn"], dt, dt, g["capped"], jacobian="numeric")
for name in ("diag", "offd"):
    a, b, an = ws.__getattr__(name), gn[name], g[name]
    e = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    idx = np.unravel_index(np.argmax(e), e.shape)
    print(name, idx, "gpu", a[idx], "ref", b[idx], "analytic", an[idx], "err", e[idx])
    # per column u max error
    ax = tuple(range(e.ndim - 1))
    print("  per-column max", np.array2string(e.max(axis=ax), precision=2))
    et = np.abs(an - b) / np.maximum(1.0, np.abs(an))
    print("  ref FD vs analytic per column", np.array2string(et.max(axis=ax), precision=2))
    print("  count > 1e-8:", int((e > 1e-8).sum()), "of", e.size)
