"""Seeded perturbed states shared by the golden generator and the tests."""

import numpy as np


def perturb(state, accn, seed):
    """Seeded, bounded, physically admissible state around `state`.

    Works on the reference's State and on ours (same field names); the
    reference run in tests/golden/make_golden.py and the tests call this
    same function, so both sides see bit-identical inputs.
    """
    rng = np.random.default_rng(seed)
    st = state.copy()
    n = st.p.shape[0]
    st.p = st.p + rng.normal(0.0, 20.0, n)
    st.t = st.t + rng.uniform(0.0, 400.0, n)
    st.sw = rng.uniform(0.1, 0.4, n)
    st.sg = rng.uniform(0.01, 0.3, n)
    st.x = np.clip(st.x + rng.normal(0.0, 0.05, st.x.shape), 0.0, 1.0)
    st.y = np.clip(st.y + rng.normal(0.0, 0.05, st.y.shape), 0.0, 1.0)
    st.cc = rng.uniform(0.0, 0.2, n)
    st.bhp = st.bhp + rng.normal(0.0, 5.0, st.bhp.shape)
    accn = accn * (1.0 + rng.normal(0.0, 1e-3, accn.shape))
    return st, accn


def random_state_like_reference(c, seed):
    """perturb() applied to the initial state and its accumulation snapshot
    (newton.py:246-252) computed with the oracle — what the reference did."""
    from oracle import isc_oracle as O
    ws = O.Workspace(c.grid, c.pack)
    zero = np.zeros((c.grid.ncell, c.pack.nequ))
    O.assemble(c.grid, O.Model(c.pack), ws, c.wells, c.streams, c.state, zero, 1.0, 0.0,
               np.zeros(len(c.wells), dtype=bool))
    return perturb(c.state, ws.acc.copy(), seed)


# Constructed 2-cell systems (nx=2): decoupled A = [[I, B], [C, I]] with a 2x2
# integer coupling in unknowns 0..1, rhs b there and 0 elsewhere. Found by a
# search over small integer matrices; each drives the reference's BiCGSTAB
# (linsolve.py:481-578, precond none) through one restart branch:
BREAKDOWN_CASES = {
    # (only cases whose branch sequence is the same under serial, reversed
    # and pairwise dot-product order, so the device's reduction order cannot
    # change the outcome)
    # restart after an exact rho = 0 (iteration 2), then converges
    "rho_restart_ok": ([[2, -1], [0, 1]], [[-2, -1], [-2, 0]], [2, -1, 0, 0]),
    # restart after r^.v = 0 (iteration 2), then converges
    "den_restart_ok": ([[-2, 0], [1, -1]], [[-2, 1], [0, -1]], [0, 0, 0, -1]),
    # omega = 0 detected at iteration 3, restart, converges (t.s cancels to an
    # exact 0 only in the reference's serial dot order: ROUNDING_DEPENDENT)
    "omega_restart_ok": ([[-2, 1], [-1, -2]], [[0, -2], [-1, -1]], [0, 1, -1, -1]),
    # r^.v = 0 twice: Breakdown (denominator) after the restart
    "den_den_breakdown": ([[-2, 1], [1, -2]], [[0, -1], [0, -2]], [1, 0, 1, 0]),
    # rho = 0 twice: Breakdown (scalar)
    "rho_rho_breakdown": ([[-1, -1], [2, 0]], [[1, 0], [-2, -1]], [0, 0, 2, 2]),
    # rho = 0, restart, omega = 0: Breakdown (scalar)
    "rho_omega_breakdown": ([[2, -1], [2, -2]], [[-2, -2], [-2, -2]], [0, 1, 0, 0]),
    # t.t = 0 twice: Breakdown (stagnation)
    "tt_tt_breakdown": ([[0, 0], [-1, 2]], [[-1, 1], [2, 1]], [0, 2, 2, 0]),
    # omega = 0, restart, then r^.v = 0: Breakdown (denominator)
    "omega_den_breakdown": ([[0, 0], [-2, 1]], [[2, -1], [-2, 1]], [-1, 2, -1, 2]),
    # rho = 0, restart, then t.t = 0: Breakdown (stagnation)
    "rho_tt_breakdown": ([[-1, 1], [0, 0]], [[1, 1], [2, 0]], [0, 2, 0, 0]),
}


def breakdown_system(case):
    """(diag, offd, resid) of a BREAKDOWN_CASES entry in the reference layout."""
    bm, cm, b = (np.asarray(v, dtype=np.float64) for v in case)
    diag = np.tile(np.eye(9), (2, 1, 1))
    offd = np.zeros((1, 2, 9, 9))
    offd[0, 0, :2, :2] = bm
    offd[0, 1, :2, :2] = cm
    resid = np.zeros((2, 9))
    resid[0, :2], resid[1, :2] = -b[:2], -b[2:]
    return diag, offd, resid

# cases whose branch needs the reference's serial dot order (an exact zero
# from cancelling rounded values): bit-exact in the oracle, which sums in that
# order; a device reduction in another order legitimately misses the zero
ROUNDING_DEPENDENT = ("omega_restart_ok",)
