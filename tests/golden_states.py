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
