"""z-slab decomposition over GPUs.

Each rank owns a contiguous range of z-planes (remainder to the leading
ranks, e.g. C4 on 8 GPUs -> 7,7,6,6,6,6,6,6 planes) and builds a *local*
problem: its planes plus one ghost plane towards each neighbouring rank.
Everything per cell stays rank-local; what crosses GPUs is

  * the one-plane halo of the state before each assembly and of p-hat,
    s-hat and x before each SpMV (NCCL send/recv over NVLink, or the
    in-process hub for single-GPU validation);
  * the BiCGSTAB dot products, the Newton norm and the audit sums
    (all-reduced packed scalars).

Ghost rows carry no equation (the library masks them). Cells are coloured by
their global plane index (``grid.k_offset``), and the owner ranks' boundary
blocks are copied into the ghost planes before the multicolour factorisation,
so the preconditioner — and the BiCGSTAB iteration — is the single-GPU one
whatever the rank count.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .configs import Case, InitialState, initial_state
from .grid import build_grid, slab_bounds
from .model import load_pack
from .wells import build_streams, build_wells


@dataclass
class SlabPiece:
    """One rank's local problem."""

    rank: int
    nranks: int
    k0: int                 # first owned global plane
    k1: int                 # one past the last owned global plane
    g_lo: int               # ghost planes below (0/1)
    g_hi: int               # ghost planes above (0/1)
    grid: object
    pack: object
    wells: tuple
    streams: tuple
    state: InitialState
    well_ids: tuple         # global indices of this rank's wells

    @property
    def kw_lo(self) -> int:
        return self.g_lo

    @property
    def kw_hi(self) -> int:
        return self.g_lo + (self.k1 - self.k0)

    @property
    def owned_cells(self) -> np.ndarray:
        """Local indices of the owned cells (natural order)."""
        nxny = self.grid.nx * self.grid.ny
        return np.arange(self.kw_lo * nxny, self.kw_hi * nxny)


def split_case(case: Case, nranks: int, rank: int, rock=None) -> SlabPiece:
    """Local problem of `rank` (owned z-planes + ghosts) cut from `case`."""
    nx, ny, nz = case.nx, case.ny, case.nz
    nxny = nx * ny
    k0, k1 = slab_bounds(nz, nranks)[rank]
    g_lo = 1 if k0 > 0 else 0
    g_hi = 1 if k1 < nz else 0
    ka, kb = k0 - g_lo, k1 + g_hi
    kx, ky, kz, phi = rock if rock is not None else case.rock_arrays()
    sl = slice(ka * nxny, kb * nxny)
    dz = np.broadcast_to(np.asarray(case.d[2], dtype=np.float64), (nz,))
    # global cell-centre depths, sliced (bit-identical to the global grid)
    z_top = 0.0 + np.concatenate(([0.0], np.cumsum(dz)[:-1]))
    zc = z_top + 0.5 * dz
    g = build_grid(nx, ny, kb - ka, case.d[0], case.d[1], dz[ka:kb], kx[sl], ky[sl], kz[sl],
                   phi[sl])
    depth = np.repeat(zc[ka:kb], nxny)
    g = replace(g, depth=depth)
    # global index of local plane 0: the device colours cells by the global
    # (i + j + k) parity, so neighbouring ranks agree on red/black
    object.__setattr__(g, "k_offset", ka)
    pack = load_pack(case.pack, g.phi_ref)
    mine = [w for w, s in enumerate(case.wells) if k0 <= s.k - 1 < k1]
    specs = [replace(case.wells[w], k=case.wells[w].k - ka) for w in mine]
    wells = build_wells(specs, g)
    streams = build_streams(pack, wells)
    state = initial_state(case, g, wells)
    return SlabPiece(rank, nranks, k0, k1, g_lo, g_hi, g, pack, tuple(wells), tuple(streams),
                     state, tuple(mine))


def attach_hub(ctx, hub, piece: SlabPiece):
    N.check(ctx.L.isc_comm_hub(ctx.h, hub, piece.rank, piece.g_lo, piece.g_hi, piece.kw_lo,
                               piece.kw_hi), "isc_comm_hub")


def attach_nccl(ctx, uid: bytes, piece: SlabPiece):
    buf = ctypes.create_string_buffer(uid, 128)
    N.check(ctx.L.isc_comm_nccl(ctx.h, buf, piece.rank, piece.nranks, piece.g_lo, piece.g_hi,
                                piece.kw_lo, piece.kw_hi), "isc_comm_nccl")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    N.check(N.lib().isc_nccl_unique_id(buf), "isc_nccl_unique_id")
    return buf.raw


class Hub:
    """In-process transport: one context + host thread per emulated rank."""

    def __init__(self, nranks: int):
        self.h = N.lib().isc_hub_create(nranks)
        self.nranks = nranks

    def close(self):
        if self.h:
            N.lib().isc_hub_destroy(self.h)
            self.h = None

    def run(self, fn, args_per_rank: Sequence):
        """fn(*args) on one thread per rank (ctypes releases the GIL)."""
        out: List = [None] * self.nranks
        err: List = [None] * self.nranks

        def body(r):
            try:
                out[r] = fn(*args_per_rank[r])
            except BaseException as exc:  # surfaced below
                err[r] = exc

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.nranks)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out
