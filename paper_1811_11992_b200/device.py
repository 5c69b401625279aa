"""Device context: one ``isc_ctx`` per (grid, pack, wells) and its buffers.

Owns the C-ABI handle (model constants, static grid factors, per-cell
records, the assembled/decoupled 7-point block system, preconditioner
factors, Krylov vectors — all in HBM) and issues every call on torch's
current CUDA stream so torch-side copies and library kernels are ordered.
Buffers handed across the boundary are torch CUDA tensors owned here;
the library never frees them.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .model import RK_TREF

DARCY_CONST = 1.0623e-14 * 144.0 / (1.0e-3 * 0.2248089431 / 10.76391042 / 86400.0)  # units.py:24
NU = 9
NF = 5


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def face_arrays(grid):
    """(gd, td, conn_id) of shape (3, n): per owner cell and +axis face.

    gd = DARCY_CONST * conn_geom exactly as the reference Workspace
    (assembly.py:320-323); conn_id is the reference's connection index.
    """
    n = grid.ncell
    ca = np.asarray(grid.conn_a, dtype=np.int64)
    axis = np.asarray(grid.conn_axis, dtype=np.int64)
    gd = np.zeros((3, n))
    td = np.zeros((3, n))
    cid = np.full((3, n), -1, dtype=np.int64)
    gd[axis, ca] = DARCY_CONST * np.asarray(grid.conn_geom, dtype=np.float64)
    td[axis, ca] = np.asarray(grid.conn_therm, dtype=np.float64)
    cid[axis, ca] = np.arange(ca.shape[0], dtype=np.int64)
    return gd, td, cid


def heat_loss_area(grid, heat_loss):
    if heat_loss is None:
        return None, 0.0, 1.0, 0.0, 0.0
    nxny = grid.nx * grid.ny
    k = np.arange(grid.ncell) // nxny
    faces = (k == 0).astype(np.float64) + (k == grid.nz - 1).astype(np.float64)
    return (faces * np.asarray(grid.area_z), heat_loss.k_ob, heat_loss.distance, heat_loss.rho,
            heat_loss.t_initial)


class DeviceContext:
    """The native context for one discrete problem."""

    def __init__(self, grid, pack, wells: Sequence, streams: Sequence, precond: str = "ras",
                 heat_loss=None, device: Optional[torch.device] = None,
                 own_stream: bool = False):
        if not torch.cuda.is_available():
            raise N.NativeLibraryMissing("no CUDA device: the product path has no CPU fallback")
        self.L = N.lib()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.grid, self.pack = grid, pack
        self.wells, self.streams = tuple(wells), tuple(streams)
        self.n = grid.ncell
        self.nw = len(self.wells)
        self.precond = precond
        self.krylov = "bicgstab"
        keep = self._keep = {}

        def hold(name, a, dtype=np.float64):
            keep[name] = _c(a, dtype)
            return N.ptr(keep[name])

        md = N.ModelDesc(
            nco=pack.nco, ncg=pack.ncg, heavy=pack.heavy, nreac=len(pack.law_codes),
            nswt=len(pack.swt_s), nslt=len(pack.slt_s),
            liq=hold("liq", pack.liq), gasp=hold("gasp", pack.gasp), kv=hold("kv", pack.kv),
            rockp=hold("rockp", pack.rockp), swt_s=hold("swt_s", pack.swt_s),
            swt_krw=hold("swt_krw", pack.swt_krw), swt_krow=hold("swt_krow", pack.swt_krow),
            swt_pcow=hold("swt_pcow", pack.swt_pcow), slt_s=hold("slt_s", pack.slt_s),
            slt_krg=hold("slt_krg", pack.slt_krg), slt_krog=hold("slt_krog", pack.slt_krog),
            slt_pcog=hold("slt_pcog", pack.slt_pcog),
            law=hold("law", pack.law_codes, np.int64), rcoef=hold("rcoef", pack.rcoef),
            nmat=hold("nmat", pack.nmat), fuel=hold("fuel", pack.fuel_idx, np.int64),
            ox=hold("ox", pack.ox_idx, np.int64), ccmax=float(pack.ccmax))
        gd, td, cid = face_arrays(grid)
        hl_area, hl_kob, hl_d, hl_rho, hl_tini = heat_loss_area(grid, heat_loss)
        gdesc = N.GridDesc(
            nx=grid.nx, ny=grid.ny, nz=grid.nz, depth=hold("depth", grid.depth),
            volume=hold("volume", grid.volume), phi_ref=hold("phi_ref", pack.phi_ref),
            gd=hold("gd", gd), td=hold("td", td), conn_id=hold("cid", cid, np.int64),
            hl_area=hold("hl", hl_area) if hl_area is not None else N.VP(0),
            hl_kob=hl_kob, hl_d=hl_d, hl_rho=hl_rho, hl_tini=hl_tini,
            k_offset=int(getattr(grid, "k_offset", 0)))
        wd = (N.WellDesc * max(1, self.nw))()
        for w, (well, stream) in enumerate(zip(self.wells, self.streams)):
            d = wd[w]
            perf = well.perfs[0]
            if len(well.perfs) != 1:
                raise NotImplementedError("multi-perforation wells (reference builds one)")
            d.cell, d.kind, d.control = perf.cell, well.kind, well.control
            d.target, d.wi, d.z_bh = well.target, perf.wi, perf.z_bh
            d.pinjmax, d.heat_rate, d.heat_stop = well.pinjmax, well.heat_rate, well.heat_stop
            if stream is not None:
                for a in range(NF):
                    d.s_yfull[a] = float(stream.yfull[a])
                for j in range(2):
                    d.s_yinj[j] = float(stream.yinj[j])
                d.s_tinj, d.s_mu, d.s_h, d.s_mbar = stream.tinj, stream.mu, stream.h, stream.mbar
        h = N.VP()
        st = self.L.isc_create(ctypes.byref(md), ctypes.byref(gdesc), self.nw, wd,
                               N.PRECOND[precond], ctypes.byref(h))
        N.check(st, "isc_create")
        self.h = h
        if not own_stream:   # order library work after torch's pending copies
            N.check(self.L.isc_set_stream(self.h, N.VP(torch.cuda.current_stream().cuda_stream)),
                    "isc_set_stream")
        self.wout = np.zeros((max(1, self.nw), N.WELL_OUT))

    def close(self):
        if getattr(self, "h", None):
            self.L.isc_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- small helpers --------------------------------------------------------
    def set_precond(self, precond: str):
        if precond != self.precond:
            N.check(self.L.isc_set_precond(self.h, N.PRECOND[precond]), "isc_set_precond")
            self.precond = precond

    def set_krylov(self, krylov: str = "bicgstab", restart: int = 0):
        """Krylov method of the mcilu red-eliminated solve: the reference's
        BiCGSTAB (default) or restarted GMRES(restart) (isc_set_krylov)."""
        N.check(self.L.isc_set_krylov(self.h, N.KRYLOV[krylov], int(restart)), "isc_set_krylov")
        self.krylov = krylov

    @property
    def decoupled_form(self) -> str:
        """Form of the decoupled system: "none", "explicit" (D^-1 B_d blocks,
        as the reference) or "compact" (mcilu: raw flux rows + D^-1[:, :6])."""
        return ("none", "explicit", "compact")[self.L.isc_decoupled_form(self.h)]

    @property
    def condensed(self) -> bool:
        """The current multicolour factorisation is the condensed form
        (6-component red-eliminated iteration, csrc/compact.cu)."""
        return bool(self.L.isc_condensed(self.h))

    def empty(self, *shape, dtype=torch.float64):
        return torch.empty(*shape, dtype=dtype, device=self.device)

    def copy_out(self, what: int, rows: int, dtype=torch.float64):
        out = self.empty(rows, self.n, dtype=dtype)
        N.check(self.L.isc_copy_out(self.h, what, N.ptr(out)), "isc_copy_out")
        return out

    def launch_count(self) -> int:
        return int(self.L.isc_launch_count(self.h))

    def stage_times(self):
        out = np.zeros(4)
        self.L.isc_stage_times(self.h, N.ptr(out))
        return out

    # -- hot path ---------------------------------------------------------------
    def assemble(self, d_state, bhp, d_accn, dt, t_new, capped, freeze):
        """isc_assemble; returns the (nw, 32) well outputs (host)."""
        bhp = _c(bhp if self.nw else np.zeros(1))
        cap = np.ascontiguousarray(np.asarray(capped if self.nw else [0], dtype=np.uint8))
        bad = ctypes.c_int64(-1)
        st = self.L.isc_assemble(self.h, N.ptr(d_state), N.ptr(bhp), N.ptr(d_accn), float(dt), float(t_new),
                N.ptr(cap), int(bool(freeze)), N.ptr(self.wout), ctypes.byref(bad))
        N.check(st, "isc_assemble", bad_cell=bad.value)
        return self.wout[:self.nw].copy()

    def numeric_jacobian(self):
        """isc_numeric_jacobian: finite-difference blocks at the inputs of the
        last assemble (assembly.py:843-939); returns the well outputs."""
        bad = ctypes.c_int64(-1)
        st = self.L.isc_numeric_jacobian(self.h, N.ptr(self.wout), ctypes.byref(bad))
        N.check(st, "isc_numeric_jacobian", bad_cell=bad.value)
        return self.wout[:self.nw].copy()

    def assemble_host(self, state, accn, dt, t_new, capped, freeze):
        """isc_assemble_host: the reference's State arrays and accn (n, 9) on
        the host; copies + transposes happen in the library."""
        arrs = [_c(getattr(state, f)) for f in ("p", "x", "y", "t", "sw", "sg", "cc")]
        accn = _c(accn)
        bhp = _c(state.bhp if self.nw else np.zeros(1))
        cap = np.ascontiguousarray(np.asarray(capped if self.nw else [0], dtype=np.uint8))
        bad = ctypes.c_int64(-1)
        st = self.L.isc_assemble_host(self.h, *[N.ptr(a) for a in arrs], N.ptr(bhp), N.ptr(accn),
                                      float(dt), float(t_new), N.ptr(cap), int(bool(freeze)),
                                      N.ptr(self.wout), ctypes.byref(bad))
        N.check(st, "isc_assemble_host", bad_cell=bad.value)
        return self.wout[:self.nw].copy()

    def solve_host(self, tol, maxiter):
        """isc_solve_host -> (du (n, 9) numpy, dbhp, iters).

        du lands in one of two pinned host buffers used in turn (the caller
        consumes it before the next-but-one solve, as the Newton loop does)."""
        dbhp = np.zeros(max(1, self.nw))
        it = ctypes.c_int32(0)
        bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
        if not hasattr(self, "_du_pool"):
            self._du_pool = [torch.empty(self.n, NU, dtype=torch.float64).pin_memory()
                             for _ in range(2)]
            self._du_turn = 0
        buf = self._du_pool[self._du_turn]
        self._du_turn ^= 1
        st = self.L.isc_solve_host(self.h, float(tol), int(maxiter), N.ptr(buf), N.ptr(dbhp),
                                   ctypes.byref(it), ctypes.byref(bc), ctypes.byref(bcol))
        N.check(st, "isc_solve", bad_cell=bc.value, bad_col=bcol.value)
        return buf.numpy(), dbhp[:self.nw], int(it.value)

    def solve(self, tol, maxiter, d_du):
        dbhp = np.zeros(max(1, self.nw))
        it = ctypes.c_int32(0)
        bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
        st = self.L.isc_solve(self.h, float(tol), int(maxiter), N.ptr(d_du), N.ptr(dbhp),
                              ctypes.byref(it), ctypes.byref(bc), ctypes.byref(bcol))
        N.check(st, "isc_solve", bad_cell=bc.value, bad_col=bcol.value)
        return dbhp[:self.nw], int(it.value)

    def set_wells_out(self, wout: np.ndarray):
        if self.nw:
            buf = _c(wout).reshape(self.nw, N.WELL_OUT)
            N.check(self.L.isc_set_wells_out(self.h, N.ptr(buf)), "isc_set_wells_out")

    def newton_update(self, d_state, d_du, eps):
        N.check(self.L.isc_newton_update(self.h, N.ptr(d_state), N.ptr(d_du), float(eps)),
                "isc_newton_update")

    def scaled_norm_cells(self, d_accn, dt) -> float:
        out = ctypes.c_double(0.0)
        N.check(self.L.isc_scaled_norm(self.h, N.ptr(d_accn), float(dt), ctypes.byref(out)),
                "isc_scaled_norm")
        return out.value

    def allreduce_host(self, vals, op: str = "sum"):
        """Sum / max of a few host doubles over the ranks of the z-slab
        decomposition (identity on a single GPU)."""
        buf = np.ascontiguousarray(np.asarray(vals, dtype=np.float64).reshape(-1))
        N.check(self.L.isc_comm_allreduce_host(self.h, N.ptr(buf), buf.size,
                                               1 if op == "max" else 0), "allreduce")
        return buf

    def synchronize(self):
        N.check(self.L.isc_synchronize(self.h), "isc_synchronize")

    def audit_sums(self, d_accn):
        out = np.zeros(3 * (NF + 1))
        N.check(self.L.isc_audit_sums(self.h, N.ptr(d_accn), N.ptr(out)), "isc_audit_sums")
        return out.reshape(3, NF + 1)


def state_to_device(state, device) -> torch.Tensor:
    """Reference-layout State (numpy) -> SoA (9, n) device tensor."""
    cols = [np.asarray(state.p)[None], np.asarray(state.x).T, np.asarray(state.y).T,
            np.asarray(state.t)[None], np.asarray(state.sw)[None], np.asarray(state.sg)[None],
            np.asarray(state.cc)[None]]
    soa = np.ascontiguousarray(np.concatenate(cols, axis=0), dtype=np.float64)
    return torch.from_numpy(soa).to(device)


def soa_from_rows(a, device) -> torch.Tensor:
    """(n, k) host array -> (k, n) device tensor."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).to(device)
