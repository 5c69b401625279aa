"""Drop-in ``BlockSolver`` backed by the sm_100a kernels.

``BlockSolver(grid, ws, tol, maxiter, precond).solve(blocks) -> (du, dbhp,
iters)`` as in linsolve.py:317-479: well Schur elimination, Gauss-Jordan
decoupling of every block row, the subdomain block ILU(0) (``bjacobi``:
non-overlapping slabs, ``ras``: one-plane overlap with restriction; slab
count min(64, max(1, n // 2048)) along the longest axis, natural order)
and right-preconditioned BiCGSTAB with the reference's single restart,
breakdown thresholds and tolerances. ``precond="mcilu"`` selects the north
star's multicolour block-ILU(0) instead, solved on the red-eliminated system
(same stopping test on the full residual), with the
reference's BiCGSTAB or, ``krylov="gmres"``, restarted GMRES(``restart``).
Raises ``SingularCellBlock``,
``Breakdown`` and ``MaxIterations`` like the reference. ``du`` is returned
as a numpy (n, 9) array for drop-in callers; ``solve_device`` keeps it in
HBM as a (9, n) tensor for the GPU Newton driver.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .assembly import Workspace, wout_from_blocks

NU = 9


class BlockSolver:
    def __init__(self, grid, ws: Workspace, tol: float = 1e-5, maxiter: int = 200,
                 precond: str = "ras", krylov: str = "bicgstab", restart: int = 30):
        if precond not in ("none", "bjacobi", "ras", "mcilu"):
            raise ValueError(f"unknown preconditioner {precond!r}")
        if krylov not in N.KRYLOV:
            raise ValueError(f"unknown Krylov method {krylov!r}")
        self.krylov, self.restart = krylov, restart
        self.grid, self.ws, self.tol, self.maxiter, self.precond = grid, ws, tol, maxiter, precond
        ws.precond = precond
        if ws.ctx is not None:
            ws.ctx.set_precond(precond)
        self._du = None

    def _ctx(self):
        if self.ws.ctx is None:
            raise RuntimeError("assemble() must run before solve()")
        self.ws.ctx.set_precond(self.precond)
        if getattr(self.ws.ctx, "krylov", "bicgstab") != self.krylov:
            self.ws.ctx.set_krylov(self.krylov, self.restart)
        return self.ws.ctx

    def solve_device(self, blocks=None):
        ctx = self._ctx()
        if blocks is not None and ctx.nw:
            ctx.set_wells_out(wout_from_blocks(blocks))
        if self._du is None or self._du.shape[1] != self.grid.ncell:
            self._du = ctx.empty(NU, self.grid.ncell)
        self.ws._invalidate()   # diag/offd are overwritten by the decoupling
        dbhp, iters = ctx.solve(self.tol, self.maxiter, self._du)
        return self._du, dbhp, iters

    def solve(self, blocks):
        """Drop-in: du as a host (n, 9) array like the reference."""
        ctx = self._ctx()
        if blocks is not None and ctx.nw:
            ctx.set_wells_out(wout_from_blocks(blocks))
        self.ws._invalidate()
        return ctx.solve_host(self.tol, self.maxiter)


def load_system(ws: Workspace, diag, offd, resid, blocks=()):
    """Hand a reference-layout system (numpy or torch) to the device context."""
    ctx = ws.ctx
    dev = ctx.device
    d = torch.as_tensor(np.ascontiguousarray(diag), dtype=torch.float64).to(dev)
    o = torch.as_tensor(np.ascontiguousarray(offd), dtype=torch.float64).to(dev)
    r = torch.as_tensor(np.ascontiguousarray(resid), dtype=torch.float64).to(dev)
    wout = wout_from_blocks(blocks) if blocks else np.zeros((1, N.WELL_OUT))
    N.check(ctx.L.isc_import_system(ctx.h, N.ptr(d), N.ptr(o), N.ptr(r), N.ptr(wout)),
            "isc_import_system")
    ws._invalidate()
