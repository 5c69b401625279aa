"""The drop-in boundary exercised inside the UNMODIFIED reference driver.

The reference package (`iscsim`, installed unmodified into baseline/_ref —
`pip install --no-deps --target baseline/_ref <reference pkg>`, DESIGN.md §7;
git-ignored, it travels to the GPU box with the snapshot) runs its own
`Simulator.advance()` (newton.py:373-431) on the C2 deck at LINEAR_TOL 1e-10
with exactly the monkey-patch INTEGRATION.md §2 gives a maintainer:
`iscsim.newton.Workspace`, `.assemble` and `.BlockSolver` replaced by this
package's device-backed versions (the driver looks them up at call time,
newton.py:224-234, 276-279, 304). Its step sequence, Newton counts, Krylov
counts and final fields must equal the pure reference run frozen in
traj_c2_1e-10.npz; the reference's own numpy code computes the norm, the
update, the capped-injector logic and the audit around our kernels.
Skipped when baseline/_ref is absent.
"""

import importlib
import os
import sys
import tempfile

import numpy as np
import pytest

from tests.helpers import GOLDEN, golden

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _reference():
    if not os.path.isdir(os.path.join(REF, "iscsim")):
        pytest.skip("the reference is not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_iscsim_"))
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        return importlib.import_module("iscsim.newton"), importlib.import_module("iscsim.deck")
    except ImportError as exc:   # e.g. numba missing
        pytest.skip(f"reference not importable: {exc}")


@pytest.mark.parametrize("precond", ["ras", "mcilu"])
def test_reference_driver_with_device_hot_path(precond):
    nw, deck_mod = _reference()
    from paper_1811_11992_b200 import assembly as gpu_asm, configs, errors
    from paper_1811_11992_b200 import linsolve as gpu_ls
    # the exceptions the device path raises are the reference's own classes
    import iscsim.errors as ref_errors
    assert errors.SingularCellBlock is ref_errors.SingularCellBlock

    with open(os.path.join(GOLDEN, "c2_deck_1e-10.txt")) as fh:
        deck = deck_mod.parse_deck(fh.read())
    phi = configs.config("c2").rock_arrays()[3]   # per-cell porosity
    saved = {k: getattr(nw, k) for k in ("build_grid", "Workspace", "assemble", "BlockSolver")}

    def build_grid(spec, rock):
        g = saved["build_grid"](spec, rock)
        g.phi_ref[:] = phi
        return g

    def block_solver(grid, ws, tol, maxiter, precond):   # newton.py:229-234 call
        # "mcilu": the north star's multicolour block-ILU(0) in place of the
        # deck's PRECOND ras (LINEAR_TOL 1e-10: same Newton sequence)
        return gpu_ls.BlockSolver(grid, ws, tol, maxiter,
                                  "mcilu" if use_mcilu else precond)

    use_mcilu = precond == "mcilu"

    iters = []
    orig_solve = gpu_ls.BlockSolver.solve

    def counting(self, blocks):
        du, dbhp, it = orig_solve(self, blocks)
        iters.append(it)
        return du, dbhp, it

    try:
        nw.build_grid = build_grid
        nw.Workspace = gpu_asm.Workspace
        nw.assemble = gpu_asm.assemble
        nw.BlockSolver = block_solver
        gpu_ls.BlockSolver.solve = counting
        sim = nw.Simulator(deck, threads=1)
        sim.advance()
    finally:
        for k, v in saved.items():
            setattr(nw, k, v)
        gpu_ls.BlockSolver.solve = orig_solve

    g = golden("traj_c2_1e-10.npz")
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves) for s in sim.steps])
    ref = g["steps"]
    assert rec.shape[0] == ref.shape[0]
    np.testing.assert_array_equal(rec[:, 2], ref[:, 2])        # Newton per step
    np.testing.assert_array_equal(rec[:, 4], ref[:, 4])        # solves per step
    np.testing.assert_allclose(rec[:, :2], ref[:, :2], rtol=1e-12)
    if precond == "ras":   # the reference's own preconditioner: its Krylov counts
        assert np.all(np.abs(rec[:, 3] - ref[:, 3]) <= rec[:, 4]), (rec[:, 3], ref[:, 3])
    for f in ("p", "t", "sw", "sg"):
        a, b = np.asarray(getattr(sim.state, f)), g["final_" + f]
        assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)) <= 1e-6, f
    np.testing.assert_allclose(sim.state.bhp, g["final_bhp"], rtol=1e-6)
    np.testing.assert_allclose(sim.cumulative_imbalance(), float(g["cum_imbalance"]),
                               rtol=1e-6, atol=1e-12)
    assert len(iters) == int(ref[:, 4].sum())
