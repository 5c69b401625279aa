"""Structured Cartesian grid: geometry, connection list, slab partition.

Vectorised restatement of the reference's grid.py so that multi-million cell
grids build in seconds (the reference's per-cell Python loops take ~40 s at
2 M cells). Results are bit-identical to the reference:

* cells x-fastest, ``c = i + nx*(j + ny*k)``, depth increasing downward
  (grid.py:1-8, 49-57, 80-93);
* connections in (k, j, i) x (+x, +y, +z) order with ``conn_a < conn_b`` and
  harmonic geometric factors ``harm(A*k_a/h_a, A*k_b/h_b)`` and thermal
  factors ``harm(A/h_a, A/h_b)`` (grid.py:95-124);
* ``partition`` slabs along the longest axis, remainder to the leading slabs,
  halo = neighbour cells owned elsewhere (grid.py:148-186).

The GPU kernels never use the connection list for the 7-point structure
(neighbours are implicit in the (i, j, k) index); it is kept so the drop-in
surface exposes the same ``Grid`` attributes as the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np

AXIS_X, AXIS_Y, AXIS_Z = 0, 1, 2


@dataclass(frozen=True, eq=False)
class Grid:
    """Same fields as the reference's Grid (grid.py:20-57)."""

    nx: int
    ny: int
    nz: int
    dx: np.ndarray
    dy: np.ndarray
    dz: np.ndarray
    depth: np.ndarray
    volume: np.ndarray
    kx: np.ndarray
    ky: np.ndarray
    kz: np.ndarray
    phi_ref: np.ndarray
    area_z: np.ndarray
    conn_a: np.ndarray
    conn_b: np.ndarray
    conn_geom: np.ndarray
    conn_therm: np.ndarray
    conn_axis: np.ndarray

    @property
    def ncell(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def nconn(self) -> int:
        return self.conn_a.shape[0]

    def cell_index(self, i: int, j: int, k: int) -> int:
        return i + self.nx * (j + self.ny * k)

    def cell_ijk(self, cell: int) -> Tuple[int, int, int]:
        return (cell % self.nx, (cell // self.nx) % self.ny,
                cell // (self.nx * self.ny))


def _harmonic(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """2ab/(a+b), zero when either side is non-positive (grid.py:60-64)."""
    out = np.zeros_like(a)
    ok = (a > 0.0) & (b > 0.0)
    aa, bb = a[ok], b[ok]
    out[ok] = 2.0 * aa * bb / (aa + bb)
    return out


def _axis(v, n: int) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64).ravel()
    if a.size == 1:
        a = np.full(n, float(a[0]))
    if a.size != n:
        raise ValueError(f"axis sizes: expected 1 or {n} values, got {a.size}")
    return a


def _cellwise(v, n: int) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64).ravel()
    if a.size == 1:
        a = np.full(n, float(a[0]))
    if a.size != n:
        raise ValueError(f"cell property: expected 1 or {n} values, got {a.size}")
    return np.ascontiguousarray(a)


def build_grid(nx: int, ny: int, nz: int, dx, dy, dz, permx, permy, permz,
               phi_ref, depth_top: float = 0.0) -> Grid:
    """Geometry and connection list (grid.py:67-135), vectorised."""
    n = nx * ny * nz
    dx, dy, dz = _axis(dx, nx), _axis(dy, ny), _axis(dz, nz)
    kx, ky, kz = _cellwise(permx, n), _cellwise(permy, n), _cellwise(permz, n)
    phi = _cellwise(phi_ref, n)

    z_top = depth_top + np.concatenate(([0.0], np.cumsum(dz)[:-1]))
    z_center = z_top + 0.5 * dz
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    depth = z_center[kk]
    dxi, dyj, dzk = dx[ii], dy[jj], dz[kk]
    volume = dxi * dyj * dzk
    area_z = dxi * dyj

    cell = np.arange(n, dtype=np.int64)
    has = np.stack([ii + 1 < nx, jj + 1 < ny, kk + 1 < nz], axis=1)
    nbr = np.stack([cell + 1, cell + nx, cell + nx * ny], axis=1)
    # per-axis face area and half-cell lengths on both sides
    ii1 = np.minimum(ii + 1, nx - 1)
    jj1 = np.minimum(jj + 1, ny - 1)
    kk1 = np.minimum(kk + 1, nz - 1)
    area = np.stack([dyj * dzk, dxi * dzk, dxi * dyj], axis=1)
    ha = np.stack([dxi, dyj, dzk], axis=1)
    hb = np.stack([dx[ii1], dy[jj1], dz[kk1]], axis=1)
    nb_safe = np.where(has, nbr, cell[:, None])
    ka = np.stack([kx, ky, kz], axis=1)
    kb = np.stack([kx[nb_safe[:, 0]], ky[nb_safe[:, 1]], kz[nb_safe[:, 2]]], axis=1)

    mask = has.ravel()
    conn_a = np.repeat(cell, 3)[mask].astype(np.int32)
    conn_b = nbr.ravel()[mask].astype(np.int32)
    A = area.ravel()[mask]
    Ha, Hb = ha.ravel()[mask], hb.ravel()[mask]
    Ka, Kb = ka.ravel()[mask], kb.ravel()[mask]
    conn_geom = _harmonic(A * Ka / Ha, A * Kb / Hb)
    conn_therm = _harmonic(A / Ha, A / Hb)
    conn_axis = np.tile(np.array([AXIS_X, AXIS_Y, AXIS_Z], dtype=np.int8), n)[mask]
    return Grid(nx=nx, ny=ny, nz=nz, dx=dx, dy=dy, dz=dz, depth=depth, volume=volume,
                kx=kx, ky=ky, kz=kz, phi_ref=phi, area_z=area_z,
                conn_a=conn_a, conn_b=conn_b, conn_geom=conn_geom,
                conn_therm=conn_therm, conn_axis=conn_axis)


@dataclass(frozen=True, eq=False)
class Partition:
    """Slab decomposition with halos (grid.py:138-145)."""

    nsub: int
    axis: int
    bounds: Tuple[Tuple[int, int], ...]   # [lo, hi) slab range along `axis`
    owner: np.ndarray

    @property
    def cells(self) -> Tuple[np.ndarray, ...]:
        return tuple(np.flatnonzero(self.owner == s).astype(np.int32)
                     for s in range(self.nsub))


def slab_bounds(n_axis: int, p: int) -> Tuple[Tuple[int, int], ...]:
    """Slab sizes differ by at most one; leading slabs take the remainder."""
    base, extra = divmod(n_axis, p)
    out, pos = [], 0
    for s in range(p):
        size = base + (1 if s < extra else 0)
        out.append((pos, pos + size))
        pos += size
    return tuple(out)


def partition(grid, p: int) -> Partition:
    """Slab partition along the longest axis (grid.py:148-186).

    The first maximum wins ties (``np.argmax``), exactly as the reference.
    Halo cells of slab s are the adjacent planes of its neighbours, which is
    what the reference's connection scan yields on a 7-point grid.
    """
    if p < 1:
        raise ValueError("thread count must be >= 1")
    dims = (grid.nx, grid.ny, grid.nz)
    axis = int(np.argmax(dims))
    bounds = slab_bounds(dims[axis], p)
    slab_of = np.empty(dims[axis], dtype=np.int32)
    for s, (lo, hi) in enumerate(bounds):
        slab_of[lo:hi] = s
    c = np.arange(grid.ncell)
    ijk = (c % grid.nx, (c // grid.nx) % grid.ny, c // (grid.nx * grid.ny))
    owner = slab_of[ijk[axis]]
    return Partition(nsub=p, axis=axis, bounds=bounds, owner=owner)


def heat_loss_coefficients(grid, config=None):
    """Per-cell top/bottom face area and loss constants (grid.py:189-206)."""
    area = np.zeros(grid.ncell)
    if config is None:
        return area, 0.0, 1.0, 0.0
    nxny = grid.nx * grid.ny
    k = np.arange(grid.ncell) // nxny
    faces = (k == 0).astype(np.float64) + (k == grid.nz - 1).astype(np.float64)
    area = faces * grid.area_z
    return area, config.k_ob, config.distance, config.rho
