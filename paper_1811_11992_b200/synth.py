"""Seeded synthetic 7-point block systems (BASELINE config 5 microbench).

"diagonally dominant fp64 blocks with off-diagonals drawn N(0,0.1)·|diag|"
(BASELINE.json configs[4]), made concrete as in SURVEY §8(d):
diagonal blocks N(0,1) with each diagonal entry replaced by its row's
|.|-sum + 1; off-diagonal block entries N(0,0.1)·|d_rr| of the owning row;
residual N(0,1). The solver decouples and solves J·du = -resid.

Values come from a counter-based generator (splitmix64 + Box-Muller) keyed
by (row cell, direction, r, u), so the *same* matrix can be produced on the
host (this numpy version: small parity cases, the reference's BlockSolver in
tests/golden) and directly in HBM by the device generator
``isc_synth_system`` (csrc/synth.cu) at 16 M block rows.

Direction order of a row's six couplings: -z, -y, -x, +x, +y, +z (the
reference's ascending-connection gather order, _kernels.py:828-854).
"""

from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
STREAM_DIAG, STREAM_OFFD, STREAM_RHS = 0, 1, 2
_STREAM_SHIFT = 40


def _mix(x: np.ndarray) -> np.ndarray:
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def _u01(seed: int, key: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = _mix(np.uint64(seed) * _GOLD + key.astype(np.uint64))
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    key = (np.uint64(stream) << np.uint64(_STREAM_SHIFT)) + idx.astype(np.uint64) * np.uint64(2)
    u1 = _u01(seed, key)
    u2 = _u01(seed, key + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def synth_system(grid, nu: int = 9, seed: int = 7):
    """(diag (n,nu,nu), offd (m,2,nu,nu), resid (n,nu)) in the reference layout."""
    n, m = grid.ncell, grid.nconn
    b2 = nu * nu
    diag = normal(seed, STREAM_DIAG, np.arange(n * b2, dtype=np.int64)).reshape(n, nu, nu)
    rs = np.abs(diag).sum(axis=2)
    idx = np.arange(nu)
    diag[:, idx, idx] = rs + 1.0
    dmag = np.abs(diag[:, idx, idx])
    ca = np.asarray(grid.conn_a, dtype=np.int64)
    cb = np.asarray(grid.conn_b, dtype=np.int64)
    d_ab = _direction(grid, ca, cb)
    d_ba = 5 - d_ab
    e = np.arange(b2, dtype=np.int64)
    key_ab = (ca * 6 + d_ab)[:, None] * b2 + e[None, :]
    key_ba = (cb * 6 + d_ba)[:, None] * b2 + e[None, :]
    offd = np.empty((m, 2, nu, nu))
    offd[:, 0] = (0.1 * normal(seed, STREAM_OFFD, key_ab)).reshape(m, nu, nu) * dmag[ca][:, :, None]
    offd[:, 1] = (0.1 * normal(seed, STREAM_OFFD, key_ba)).reshape(m, nu, nu) * dmag[cb][:, :, None]
    resid = normal(seed, STREAM_RHS, np.arange(n * nu, dtype=np.int64)).reshape(n, nu)
    return diag, offd, resid


def _direction(grid, ca, cb):
    """+x/+y/+z code (3/4/5) of conn_b relative to conn_a from (i, j, k)."""
    nx, ny = grid.nx, grid.ny
    ia, ja, ka = ca % nx, (ca // nx) % ny, ca // (nx * ny)
    ib, jb, kb = cb % nx, (cb // nx) % ny, cb // (nx * ny)
    return np.where(ib != ia, 3, np.where(jb != ja, 4, 5)).astype(np.int64)
