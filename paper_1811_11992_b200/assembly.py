"""Drop-in ``Workspace`` / ``assemble`` backed by the sm_100a kernels.

Same call signature and side effects as the reference's
``assemble(grid, pack, ws, wells, streams, state, accn, dt, t_new, capped,
jacobian="analytic", freeze_upwind=False) -> List[WellBlock]``
(assembly.py:561-598): the residual, the block Jacobian (diagonal blocks and
per-connection ``offd``), accumulation, reaction sources, ``yfull`` and the
persistent upwind flags land in ``ws``; ``PoreSpaceExhausted`` is raised
for a coke-filled cell (assembly.py:548-552).

``ws`` keeps everything in HBM. The reference-layout arrays
(``ws.resid`` (n,9), ``ws.diag`` (n,9,9), ``ws.offd`` (m,2,9,9), ``ws.acc``,
``ws.src``, ``ws.yfull``) are materialised lazily, on first access after an
assembly, as numpy arrays (drop-in consumers such as ``scaled_norm`` or a
report writer read them); the GPU Newton driver never touches them.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np
import torch

from . import _native as N
from .device import DeviceContext, soa_from_rows, state_to_device

NU = 9


@dataclass
class WellBlock:
    """One well's residual row and couplings (assembly.py:348-363)."""

    cells: np.ndarray
    resid: float
    dwdb: float
    wrow: np.ndarray
    bcol: np.ndarray
    phase_rates: np.ndarray
    comp_rates: np.ndarray


def blocks_from_wout(wells, wout) -> List[WellBlock]:
    out = []
    for w, well in enumerate(wells):
        o = wout[w]
        out.append(WellBlock(
            cells=np.array([p.cell for p in well.perfs], dtype=np.int64),
            resid=float(o[0]), dwdb=float(o[1]), wrow=o[2:2 + NU].reshape(1, NU).copy(),
            bcol=o[2 + NU:2 + 2 * NU].reshape(1, NU).copy(),
            phase_rates=o[2 + 2 * NU:5 + 2 * NU].reshape(1, 3).copy(),
            comp_rates=o[5 + 2 * NU:5 + 3 * NU].reshape(1, NU).copy()))
    return out


def wout_from_blocks(blocks) -> np.ndarray:
    wout = np.zeros((len(blocks), N.WELL_OUT))
    for w, b in enumerate(blocks):
        wout[w, 0], wout[w, 1] = b.resid, b.dwdb
        wout[w, 2:2 + NU] = np.asarray(b.wrow).reshape(-1)[:NU]
        wout[w, 2 + NU:2 + 2 * NU] = np.asarray(b.bcol).reshape(-1)[:NU]
        wout[w, 2 + 2 * NU:5 + 2 * NU] = np.asarray(b.phase_rates).reshape(-1)[:3]
        wout[w, 5 + 2 * NU:5 + 3 * NU] = np.asarray(b.comp_rates).reshape(-1)[:NU]
    return wout


class Workspace:
    """Device-resident workspace; constructor mirrors assembly.py:287.

    ``Workspace(grid, pack, deck_or_None, wells=..., streams=...)``: the
    reference builds wells/streams separately and passes them to
    ``assemble``; the native context needs them at creation, so they are
    bound here (or at the first ``assemble`` call if omitted).
    """

    _LAZY = ("resid", "diag", "offd", "acc", "src", "yfull", "upw")

    def __init__(self, grid, pack, deck=None, wells=None, streams=None, precond="ras"):
        self.grid, self.pack = grid, pack
        self.heat_loss = getattr(deck, "heat_loss", None) if deck is not None else None
        self.precond = precond
        self.ctx = None
        if wells is not None:
            self.bind(wells, streams)
        self._fresh = set()
        self._cache = {}

    def bind(self, wells, streams):
        if self.ctx is None:
            self.ctx = DeviceContext(self.grid, self.pack, wells, streams, self.precond,
                                     self.heat_loss)
        return self.ctx

    @property
    def device(self):
        return self.ctx.device

    def _invalidate(self):
        self._cache.clear()

    def __getattr__(self, name):
        if name in Workspace._LAZY:
            cache = self.__dict__.get("_cache")
            if cache is None or self.__dict__.get("ctx") is None:
                raise AttributeError(name)
            if name not in cache:
                self._materialise(name)
            return cache[name]
        raise AttributeError(name)

    def _materialise(self, name):
        ctx, n = self.ctx, self.grid.ncell
        if name in ("resid", "diag", "offd"):
            m = self.grid.nconn
            d = ctx.empty(n, NU, NU)
            o = ctx.empty(m, 2, NU, NU)
            r = ctx.empty(n, NU)
            N.check(ctx.L.isc_export_system(ctx.h, N.ptr(d), N.ptr(o), N.ptr(r)),
                    "isc_export_system")
            self._cache.update(diag=d.cpu().numpy(), offd=o.cpu().numpy(), resid=r.cpu().numpy())
        elif name in ("acc", "src"):
            t = ctx.copy_out(1 if name == "acc" else 2, NU)
            self._cache[name] = t.t().contiguous().cpu().numpy()
        elif name == "yfull":
            self._cache[name] = ctx.copy_out(3, 5).t().contiguous().cpu().numpy()
        elif name == "upw":
            flags = ctx.copy_out(5, 9, dtype=torch.int8).cpu().numpy().reshape(3, 3, n)
            ca = np.asarray(self.grid.conn_a, dtype=np.int64)
            ax = np.asarray(self.grid.conn_axis, dtype=np.int64)
            self._cache[name] = flags[ax, :, ca].astype(np.int8)


def assemble(grid, pack, ws, wells, streams, state, accn, dt, t_new, capped,
             jacobian="analytic", freeze_upwind=False) -> List[WellBlock]:
    """Residual and Jacobian at ``state`` (assembly.py:561-598); with
    ``jacobian == "numeric"`` every block is then replaced by the
    finite-difference Jacobian (assembly.py:593-597, 843-939) on the device."""
    ctx = ws.bind(wells, streams)
    ws._invalidate()
    if isinstance(getattr(state, "p", None), np.ndarray) and not isinstance(accn, torch.Tensor):
        # reference-layout host arrays: staged + transposed inside the library
        wout = ctx.assemble_host(state, accn, dt, t_new, capped, freeze_upwind)
    else:
        u = getattr(state, "u", state)
        d_state = u if isinstance(u, torch.Tensor) else state_to_device(state, ctx.device)
        d_accn = accn if isinstance(accn, torch.Tensor) else soa_from_rows(accn, ctx.device)
        bhp = np.asarray(state.bhp, dtype=np.float64)
        wout = ctx.assemble(d_state, bhp, d_accn, dt, t_new, capped, freeze_upwind)
    if jacobian == "numeric":
        wout = ctx.numeric_jacobian()
    ws.last_wout = wout
    return blocks_from_wout(wells, wout)


def check_jacobian(grid, pack, ws, wells, streams, state, accn, dt, t_new, capped) -> float:
    """Worst |analytic - numeric| / max(1, |analytic|) over the diagonal,
    off-diagonal and well blocks (assembly.py:942-982); ``ws`` is left holding
    the analytic system, as in the reference."""
    blocks = assemble(grid, pack, ws, wells, streams, state, accn, dt, t_new, capped)
    diag_a, offd_a = ws.diag.copy(), ws.offd.copy()
    ctx = ws.bind(wells, streams)
    ws._invalidate()
    nblocks = blocks_from_wout(wells, ctx.numeric_jacobian())

    def scaled(a, b):
        return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(a)))) if a.size else 0.0

    worst = max(scaled(diag_a, ws.diag), scaled(offd_a, ws.offd))
    for b, nb in zip(blocks, nblocks):
        worst = max(worst, scaled(b.wrow, nb.wrow), scaled(b.bcol, nb.bcol),
                    abs(b.dwdb - nb.dwdb) / max(1.0, abs(b.dwdb)))
    # restore the analytic system (the reference copies its blocks back)
    assemble(grid, pack, ws, wells, streams, state, accn, dt, t_new, capped)
    return worst
