"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference simulator's Newton hot path (iscsim,
arxiv 1811.11992): the per-cell/per-connection kernels run in the plain-C
library ``oracle/_build/libisc_oracle.so`` (isc_oracle.c); the drivers
below restate the reference's Python layers (assembly.py, linsolve.py,
newton.py) with numpy. Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs may import this module; the product never does.

Inputs are duck-typed: the reference's own Grid/ModelPack/Well objects work
as well as ours (paper_1811_11992_b200.grid/model/wells), which is how the
golden tests pin this oracle to the reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libisc_oracle.so")

DARCY_CONST = 1.0623e-14 * 144.0 / (1.0e-3 * 0.2248089431 / 10.76391042 / 86400.0)  # units.py:18-24
RANKINE_OFFSET = 459.67
R_GAS_DENSITY = 10.7316
GASP_TCR, GASP_PC = 1, 2
INJECTOR, CTRL_BHP = 0, 0
SUBDOMAIN_CELLS, MAX_SUBDOMAINS = 2048, 64          # linsolve.py:34-35
BREAKDOWN_EPS = 1e-30                               # linsolve.py:37
FREEZE_UPWIND_AFTER, FAST_ITERS = 5, 4              # newton.py:56-60
GROWTH_FACTOR, CUT_FACTOR, TIME_EPS = 2.0, 0.5, 1e-9


# condensed multicolour form: flux rows CR_ of a block; primary / secondary
# unknowns (p, x_1, y_1, T, S_w, S_g) / (x_2, y_2, C_c) for nco = ncg = 2
CR_ = 6
COND_P = [0, 1, 3, 5, 6, 7]
COND_S = [2, 4, 8]


class OracleError(Exception):
    pass


# error classes named as the reference's (errors.py:43-88); tests compare names
class PoreSpaceExhausted(OracleError): pass
class SingularCellBlock(OracleError): pass
class Breakdown(OracleError): pass
class MaxIterations(OracleError): pass
class DivergedResidual(OracleError): pass
class DegenerateTemperature(OracleError): pass
class SimulationStalled(OracleError): pass


_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.orc_dot.restype = ctypes.c_double
        _lib.orc_z_factor_mix.restype = ctypes.c_double
        _lib.orc_cubic_largest_root.restype = ctypes.c_double
        _lib.orc_ilu_factor.restype = ctypes.c_int64
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


class _OrcModel(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int64) for f in ("nco", "ncg", "heavy", "nreac", "nswt", "nslt")]
                + [(f, ctypes.c_void_p) for f in (
                    "liq", "gasp", "kv", "rockp", "swt_s", "swt_krw", "swt_krow", "swt_pcow",
                    "slt_s", "slt_krg", "slt_krog", "slt_pcog", "law", "rcoef", "nmat",
                    "fuel", "ox")]
                + [("ccmax", ctypes.c_double)])


class Model:
    """Pack constants pinned in contiguous arrays for the C side."""

    def __init__(self, pack):
        self.pack = pack
        self.keep = {}
        for f in ("liq", "gasp", "kv", "rockp", "swt_s", "swt_krw", "swt_krow", "swt_pcow",
                  "slt_s", "slt_krg", "slt_krog", "slt_pcog", "rcoef", "nmat"):
            self.keep[f] = _c(getattr(pack, f))
        for f in ("law_codes", "fuel_idx", "ox_idx"):
            self.keep[f] = _c(getattr(pack, f), np.int64)
        k = self.keep
        self.s = _OrcModel(
            nco=pack.nco, ncg=pack.ncg, heavy=pack.heavy, nreac=k["law_codes"].shape[0],
            nswt=k["swt_s"].shape[0], nslt=k["slt_s"].shape[0],
            liq=_p(k["liq"]), gasp=_p(k["gasp"]), kv=_p(k["kv"]), rockp=_p(k["rockp"]),
            swt_s=_p(k["swt_s"]), swt_krw=_p(k["swt_krw"]), swt_krow=_p(k["swt_krow"]),
            swt_pcow=_p(k["swt_pcow"]), slt_s=_p(k["slt_s"]), slt_krg=_p(k["slt_krg"]),
            slt_krog=_p(k["slt_krog"]), slt_pcog=_p(k["slt_pcog"]), law=_p(k["law_codes"]),
            rcoef=_p(k["rcoef"]), nmat=_p(k["nmat"]), fuel=_p(k["fuel_idx"]),
            ox=_p(k["ox_idx"]), ccmax=float(pack.ccmax))
        self.phi_ref = _c(pack.phi_ref)


def z_factor_mix(w, tcrit_r, pcrit, p, t):
    """_props.py:107-150 through the C restatement: (z, dzdp, dzdt, dzdw)."""
    w, tc, pc = _c(w), _c(tcrit_r), _c(pcrit)
    dzdw = np.zeros(w.shape[0])
    dzdp, dzdt = ctypes.c_double(), ctypes.c_double()
    z = lib().orc_z_factor_mix(ctypes.c_int(w.shape[0]), _p(w), _p(tc), _p(pc),
                               ctypes.c_double(p), ctypes.c_double(t), _p(dzdw),
                               ctypes.byref(dzdp), ctypes.byref(dzdt))
    return z, dzdp.value, dzdt.value, dzdw


# ---------------------------------------------------------------- workspace

class Workspace:
    """Same arrays as the reference's Workspace (assembly.py:284-345)."""

    def __init__(self, grid, pack, heat_loss=None):
        n, m, nu, nf = grid.ncell, grid.nconn, pack.nequ, pack.nfull
        z = np.zeros
        self.pot, self.dpot = z((n, 3)), z((n, 3, nu))
        self.beta, self.dbeta = z((n, 3)), z((n, 3, nu))
        self.hph, self.dhph = z((n, 3)), z((n, 3, nu))
        self.yfull, self.dyfull = z((n, nf)), z((n, nf, nu))
        self.gam, self.dgam = z((n, 3)), z((n, 3, nu))
        self.pcv, self.dpcv = z((n, 2)), z((n, 2))
        self.kr3, self.dkr3 = z((n, 3)), z((n, 3, 2))
        self.ktd = z((n, 1 + nu))
        self.acc, self.dacc = z((n, nu)), z((n, nu, nu))
        self.src, self.dsrc = z((n, nu)), z((n, nu, nu))
        self.ok = np.zeros(n, dtype=np.uint8)
        self.flux, self.dfa, self.dfb = z((m, nu)), z((m, nu, nu)), z((m, nu, nu))
        self.resid, self.diag, self.offd = z((n, nu)), z((n, nu, nu)), z((m, 2, nu, nu))
        self.upw = np.zeros((m, 3), dtype=np.int8)
        self.gd = DARCY_CONST * _c(grid.conn_geom)
        self.td = _c(grid.conn_therm)
        cells = np.concatenate([grid.conn_a, grid.conn_b])
        ics = np.concatenate([np.arange(m), np.arange(m)]).astype(np.int64)
        sides = np.concatenate([np.zeros(m, np.int8), np.ones(m, np.int8)])
        order = np.lexsort((ics, cells))
        self.adj_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(cells, minlength=n), out=self.adj_ptr[1:])
        self.adj_ids = ics[order]
        self.adj_sides = sides[order]
        self.hl_area = np.zeros(n)
        self.hl_kob, self.hl_d, self.hl_rho, self.hl_tini = 0.0, 1.0, 0.0, 0.0
        if heat_loss is not None:
            nxny = grid.nx * grid.ny
            k = np.arange(n) // nxny
            faces = (k == 0).astype(np.float64) + (k == grid.nz - 1).astype(np.float64)
            self.hl_area = faces * grid.area_z
            self.hl_kob, self.hl_d = heat_loss.k_ob, heat_loss.distance
            self.hl_rho, self.hl_tini = heat_loss.rho, heat_loss.t_initial


@dataclass
class WellBlock:
    """assembly.py:348-363"""

    cells: np.ndarray
    resid: float
    dwdb: float
    wrow: np.ndarray
    bcol: np.ndarray
    phase_rates: np.ndarray
    comp_rates: np.ndarray


def cell_pass(model: Model, ws: Workspace, state):
    L = lib()
    n = state.p.shape[0]
    st = [_c(state.p), _c(state.t), _c(state.sw), _c(state.sg), _c(state.x), _c(state.y),
          _c(state.cc)]
    L.orc_cell_pass(ctypes.byref(model.s), ctypes.c_int64(n), *[_p(a) for a in st],
                    _p(model.phi_ref),
                    *[_p(getattr(ws, f)) for f in (
                        "pot", "dpot", "beta", "dbeta", "hph", "dhph", "yfull", "dyfull", "gam",
                        "dgam", "pcv", "dpcv", "kr3", "dkr3", "ktd", "acc", "dacc", "src",
                        "dsrc", "ok")])
    if not ws.ok.all():
        raise PoreSpaceExhausted(f"coke fills the pore volume in cell {int(np.argmin(ws.ok))}")


def _perf_producer(pack, ws, c, x_c, bhp, wi, dz):
    """assembly.py:370-418"""
    nu, nco, nf, row_e = pack.nequ, pack.nco, pack.nfull, pack.row_energy
    rows, drows, brows = np.zeros(nu), np.zeros((nu, nu)), np.zeros(nu)
    qph, dq_sum, dq_sum_db = np.zeros(3), np.zeros(nu), 0.0
    yf, dyf = ws.yfull[c], ws.dyfull[c]
    for a in range(3):
        dd = bhp - ws.pot[c, a] - ws.gam[c, a] * dz
        ddd = -ws.dpot[c, a] - dz * ws.dgam[c, a]
        cwi = DARCY_CONST * wi
        q = cwi * ws.beta[c, a] * dd
        dq = cwi * (ws.dbeta[c, a] * dd + ws.beta[c, a] * ddd)
        dq_db = cwi * ws.beta[c, a]
        qph[a] = q
        dq_sum += dq
        dq_sum_db += dq_db
        if a == 0:
            rows[0] += q
            drows[0] += dq
            brows[0] += dq_db
        elif a == 1:
            rows[1:1 + nco] += q * x_c
            drows[1:1 + nco] += np.outer(x_c, dq)
            for i in range(nco):
                drows[1 + i, 1 + i] += q
            brows[1:1 + nco] += dq_db * x_c
        else:
            rows[:nf] += q * yf
            drows[:nf] += np.outer(yf, dq) + q * dyf
            brows[:nf] += dq_db * yf
        rows[row_e] += q * ws.hph[c, a]
        drows[row_e] += dq * ws.hph[c, a] + q * ws.dhph[c, a]
        brows[row_e] += dq_db * ws.hph[c, a]
    return rows, drows, brows, qph, dq_sum, dq_sum_db


def _perf_injector(pack, ws, c, stream, bhp, wi, dz):
    """assembly.py:421-471"""
    nu, nco, ncg, row_e = pack.nequ, pack.nco, pack.ncg, pack.row_energy
    ct = 1 + nco + ncg
    csw, csg = ct + 1, ct + 2
    lam = ws.kr3[c, 0] + ws.kr3[c, 1] + ws.kr3[c, 2]
    dlam = np.zeros(nu)
    dlam[csw] = ws.dkr3[c, 0, 0] + ws.dkr3[c, 1, 0]
    dlam[csg] = ws.dkr3[c, 1, 1] + ws.dkr3[c, 2, 1]
    pg, dpg = ws.pot[c, 2], ws.dpot[c, 2]
    z, dzdp, _dzdt, _ = z_factor_mix(stream.yfull, pack.gasp[:, GASP_TCR],
                                     pack.gasp[:, GASP_PC], pg, stream.tinj)
    trs = stream.tinj + RANKINE_OFFSET
    rho = pg / (z * R_GAS_DENSITY * trs)
    drho_dpg = rho * (1.0 / pg - dzdp / z)
    gam = rho * stream.mbar / 144.0
    dgam_dpg = drho_dpg * stream.mbar / 144.0
    dd = bhp - pg - gam * dz
    ddd = -dpg * (1.0 + dz * dgam_dpg)
    cwi = DARCY_CONST * wi
    mob = rho * lam / stream.mu
    dmob = (drho_dpg * dpg * lam + rho * dlam) / stream.mu
    q = cwi * mob * dd
    dq = cwi * (dmob * dd + mob * ddd)
    dq_db = cwi * mob
    rows, drows, brows = np.zeros(nu), np.zeros((nu, nu)), np.zeros(nu)
    rows[1 + nco:1 + nco + ncg] = q * stream.yinj
    drows[1 + nco:1 + nco + ncg] = np.outer(stream.yinj, dq)
    brows[1 + nco:1 + nco + ncg] = dq_db * stream.yinj
    rows[row_e] = q * stream.h
    drows[row_e] = dq * stream.h
    brows[row_e] = dq_db * stream.h
    return rows, drows, brows, np.array([0.0, 0.0, q]), dq, dq_db


def well_pass(pack, grid, ws, wells, streams, state, capped, t_new):
    """assembly.py:474-527"""
    blocks: List[WellBlock] = []
    nu, row_e = pack.nequ, pack.row_energy
    for wix, well in enumerate(wells):
        bhp = state.bhp[wix]
        nperf = len(well.perfs)
        wrow, bcol = np.zeros((nperf, nu)), np.zeros((nperf, nu))
        phase_rates, comp_rates = np.zeros((nperf, 3)), np.zeros((nperf, nu))
        qsum = dqsum_db = 0.0
        heater_on = well.heat_rate != 0.0 and t_new <= well.heat_stop
        for pix, perf in enumerate(well.perfs):
            c = perf.cell
            dz = perf.z_bh - grid.depth[c]
            if well.kind == INJECTOR:
                rows, drows, brows, qph, dqs, dqs_db = _perf_injector(
                    pack, ws, c, streams[wix], bhp, perf.wi, dz)
            else:
                rows, drows, brows, qph, dqs, dqs_db = _perf_producer(
                    pack, ws, c, state.x[c], bhp, perf.wi, dz)
            ws.resid[c] -= rows
            ws.diag[c] -= drows
            bcol[pix] = -brows
            wrow[pix] = dqs
            phase_rates[pix] = qph
            comp_rates[pix] = rows
            qsum += qph.sum()
            dqsum_db += dqs_db
            if heater_on:
                ws.resid[c, row_e] -= well.heat_rate
                comp_rates[pix, row_e] += well.heat_rate
        if well.control == CTRL_BHP:
            resid_w, dwdb = bhp - well.target, 1.0
            wrow[:] = 0.0
        elif capped[wix]:
            resid_w, dwdb = bhp - well.pinjmax, 1.0
            wrow[:] = 0.0
        else:
            resid_w, dwdb = qsum - well.target, dqsum_db
        blocks.append(WellBlock(
            cells=np.array([p.cell for p in well.perfs], dtype=np.int64), resid=resid_w,
            dwdb=dwdb, wrow=wrow, bcol=bcol, phase_rates=phase_rates, comp_rates=comp_rates))
    return blocks


def assemble(grid, model: Model, ws: Workspace, wells, streams, state, accn, dt, t_new,
             capped, freeze_upwind=False, jacobian="analytic"):
    """assembly.py:561-598."""
    L = lib()
    pack = model.pack
    n, m, nu = grid.ncell, grid.nconn, pack.nequ
    cell_pass(model, ws, state)
    t_state = _c(state.t)
    L.orc_compose_pass(ctypes.c_int64(pack.nco), ctypes.c_int64(pack.ncg), ctypes.c_int64(n),
                       _p(ws.resid), _p(ws.diag), _p(ws.acc), _p(ws.dacc), _p(ws.src),
                       _p(ws.dsrc), _p(_c(accn)), _p(_c(grid.volume)), ctypes.c_double(dt),
                       _p(t_state), _p(ws.hl_area), ctypes.c_double(ws.hl_kob),
                       ctypes.c_double(ws.hl_d), ctypes.c_double(ws.hl_rho),
                       ctypes.c_double(ws.hl_tini))
    L.orc_conn_pass(ctypes.c_int64(pack.nco), ctypes.c_int64(pack.ncg), ctypes.c_int64(m),
                    _p(_c(grid.conn_a, np.int32)), _p(_c(grid.conn_b, np.int32)), _p(ws.gd),
                    _p(ws.td), _p(_c(grid.depth)), _p(t_state), _p(_c(state.x)),
                    *[_p(getattr(ws, f)) for f in ("pot", "dpot", "beta", "dbeta", "hph",
                                                   "dhph", "yfull", "dyfull", "gam", "dgam",
                                                   "ktd")],
                    _p(ws.upw), ctypes.c_int(1 if freeze_upwind else 0), _p(ws.flux),
                    _p(ws.dfa), _p(ws.dfb))
    L.orc_gather_pass(ctypes.c_int64(n), ctypes.c_int64(nu), _p(ws.adj_ptr), _p(ws.adj_ids),
                      _p(ws.adj_sides), _p(ws.flux), _p(ws.dfa), _p(ws.dfb), _p(ws.resid),
                      _p(ws.diag), _p(ws.offd))
    blocks = well_pass(pack, grid, ws, wells, streams, state, capped, t_new)
    if jacobian == "numeric":
        numeric_jacobian(grid, model, ws, wells, streams, state, accn, dt, t_new, capped,
                         blocks, freeze_upwind)
    return blocks


# ------------------------------------------------ numeric (FD) Jacobian

FD_REL_STEP, FD_PRESSURE_FLOOR, FD_UNIT_FLOOR = 1e-6, 1e-3, 5e-5   # assembly.py:33-35
_CELL_FIELDS = ("pot", "dpot", "beta", "dbeta", "hph", "dhph", "yfull", "dyfull", "gam",
                "dgam", "pcv", "dpcv", "kr3", "dkr3", "ktd", "acc", "dacc", "src", "dsrc")
_CONN_FIELDS = ("pot", "dpot", "beta", "dbeta", "hph", "dhph", "yfull", "dyfull", "gam",
                "dgam", "ktd")


class _Probe:
    """One-cell scratch (assembly.py:605-630 _CellBufs) plus two-cell staging
    arrays for single-connection conn_eval calls."""

    def __init__(self, ws):
        for f in _CELL_FIELDS:
            setattr(self, f, np.zeros((1,) + getattr(ws, f).shape[1:]))
        self.ok = np.zeros(1, dtype=np.uint8)
        self.pair = {f: np.zeros((2,) + getattr(ws, f).shape[1:]) for f in _CONN_FIELDS}
        nu = ws.acc.shape[1]
        self.flux = np.zeros((1, nu))
        self.dfa, self.dfb = np.zeros((1, nu, nu)), np.zeros((1, nu, nu))
        self.ca, self.cb = np.zeros(1, np.int32), np.ones(1, np.int32)


class _Shadow:
    """assembly.py:633-667: index [c] of any field resolves to the probe."""

    def __init__(self, probe):
        self._p = probe

    def __getattr__(self, f):
        arr = getattr(self._p, f)[0]

        class _One:
            def __getitem__(self, key):
                if isinstance(key, tuple):
                    return arr[key[1:]] if len(key) > 1 else arr
                return arr
        return _One()


def _eval_cell(model, probe, scal, phi_ref_c):
    """assembly.py:670-684"""
    one = lambda v: np.array([v], dtype=np.float64)   # noqa: E731
    lib().orc_cell_pass(ctypes.byref(model.s), ctypes.c_int64(1), _p(one(scal["p"])),
                        _p(one(scal["t"])), _p(one(scal["sw"])), _p(one(scal["sg"])),
                        _p(_c(scal["x"][None, :])), _p(_c(scal["y"][None, :])),
                        _p(one(scal["cc"])), _p(one(phi_ref_c)),
                        *[_p(getattr(probe, f)) for f in _CELL_FIELDS], _p(probe.ok))
    if not probe.ok[0]:
        raise PoreSpaceExhausted("coke fills the pore volume at a probed state")


def _cell_unknowns(state, c, pack):
    """assembly.py:687-699"""
    vals = np.empty(pack.nequ)
    vals[0] = state.p[c]
    vals[1:1 + pack.nco] = state.x[c]
    vals[1 + pack.nco:1 + pack.nco + pack.ncg] = state.y[c]
    ct = 1 + pack.nco + pack.ncg
    vals[ct], vals[ct + 1], vals[ct + 2], vals[ct + 3] = (state.t[c], state.sw[c],
                                                          state.sg[c], state.cc[c])
    return vals


def _apply_unknown(scal, u, val, pack):
    """assembly.py:702-719"""
    ct = 1 + pack.nco + pack.ncg
    if u == 0:
        scal["p"] = val
    elif u < 1 + pack.nco:
        scal["x"][u - 1] = val
    elif u < ct:
        scal["y"][u - 1 - pack.nco] = val
    elif u == ct:
        scal["t"] = val
    elif u == ct + 1:
        scal["sw"] = val
    elif u == ct + 2:
        scal["sg"] = val
    else:
        scal["cc"] = val


def _conn_probe(model, probe, ws, grid, state, ic, scal, side_a, freeze):
    """conn_eval of connection ic with the probed cell on side a (side_a) or
    b, the other side from the unperturbed workspace (assembly.py:757-790)."""
    pack = model.pack
    a, b = int(grid.conn_a[ic]), int(grid.conn_b[ic])
    other = b if side_a else a
    slot_p, slot_o = (0, 1) if side_a else (1, 0)
    for f in _CONN_FIELDS:
        probe.pair[f][slot_p] = getattr(probe, f)[0]
        probe.pair[f][slot_o] = getattr(ws, f)[other]
    t2 = np.empty(2)
    x2 = np.empty((2, pack.nco))
    t2[slot_p], t2[slot_o] = scal["t"], state.t[other]
    x2[slot_p], x2[slot_o] = scal["x"], state.x[other]
    depth2 = np.array([grid.depth[a], grid.depth[b]], dtype=np.float64)
    upw = ws.upw[ic:ic + 1].copy()          # probes never store upstream flags
    lib().orc_conn_pass(ctypes.c_int64(pack.nco), ctypes.c_int64(pack.ncg), ctypes.c_int64(1),
                        _p(probe.ca), _p(probe.cb), _p(ws.gd[ic:ic + 1].copy()),
                        _p(ws.td[ic:ic + 1].copy()), _p(depth2), _p(t2), _p(x2),
                        *[_p(probe.pair[f]) for f in _CONN_FIELDS], _p(upw),
                        ctypes.c_int(1 if freeze else 0), _p(probe.flux), _p(probe.dfa),
                        _p(probe.dfb))
    return probe.flux[0].copy()


def _probe_rows(grid, model, ws, wells, streams, state, accn, dt, c, scal, probe, conn_rows,
                freeze):
    """assembly.py:722-804: rows of cell c and of its neighbours at a probe."""
    pack = model.pack
    row_e = pack.row_energy
    row_os, row_gs = row_e + 1, row_e + 2
    _eval_cell(model, probe, scal, model.phi_ref[c])
    vdt = grid.volume[c] / dt
    rows = vdt * (probe.acc[0] - accn[c]) - grid.volume[c] * probe.src[0]
    rows[row_os] = probe.acc[0, row_os]
    rows[row_gs] = probe.acc[0, row_gs]
    if ws.hl_area[c] > 0.0:
        rows[row_e] += ws.hl_area[c] * ws.hl_kob * ((scal["t"] - ws.hl_tini) / ws.hl_d
                                                    - ws.hl_rho)
    for slot, k in enumerate(range(ws.adj_ptr[c], ws.adj_ptr[c + 1])):
        ic = int(ws.adj_ids[k])
        if ws.adj_sides[k] == 0:
            flux = _conn_probe(model, probe, ws, grid, state, ic, scal, True, freeze)
            rows += flux
            conn_rows[slot] = -flux
        else:
            flux = _conn_probe(model, probe, ws, grid, state, ic, scal, False, freeze)
            rows -= flux
            conn_rows[slot] = flux.copy()
    shadow = _Shadow(probe)
    fw_parts = {}
    for wix, well in enumerate(wells):
        for perf in well.perfs:
            if perf.cell != c:
                continue
            dz = perf.z_bh - grid.depth[c]
            if well.kind == INJECTOR:
                prow, _, _, qph, _, _ = _perf_injector(pack, shadow, c, streams[wix],
                                                       state.bhp[wix], perf.wi, dz)
            else:
                prow, _, _, qph, _, _ = _perf_producer(pack, shadow, c, scal["x"],
                                                       state.bhp[wix], perf.wi, dz)
            rows -= prow
            fw_parts[wix] = fw_parts.get(wix, 0.0) + qph.sum()
    return rows, fw_parts


def _fd_points(pack, base, u, sw, sg):
    """assembly.py:807-840"""
    ct = 1 + pack.nco + pack.ncg
    v = base[u]
    if u == 0:
        h = max(FD_REL_STEP * abs(v), FD_PRESSURE_FLOOR)
        return v + h, v - h
    h = max(FD_REL_STEP * abs(v), FD_UNIT_FLOOR)
    if u == ct:
        return v + h, v - h
    if u == ct + 1 or u == ct + 2:
        if v - h < 0.0:
            return v + h, v
        if 1.0 - sw - sg - h < 0.0:
            return v, v - h
        return v + h, v - h
    if u == ct + 3:
        if v - h < 0.0:
            return v + h, v
        return v + h, v - h
    if v - h < 0.0:
        return v + h, v
    if v + h > 1.0:
        return v, v - h
    return v + h, v - h


def numeric_jacobian(grid, model, ws, wells, streams, state, accn, dt, t_new, capped, blocks,
                     freeze=False):
    """assembly.py:843-939: every Jacobian block by finite differences."""
    pack = model.pack
    nu = pack.nequ
    probe = _Probe(ws)
    rate_wells = {wix for wix, w in enumerate(wells)
                  if w.control != CTRL_BHP and not capped[wix]}
    perf_lookup = {}
    for wix, well in enumerate(wells):
        for pix, perf in enumerate(well.perfs):
            perf_lookup.setdefault(perf.cell, []).append((wix, pix))
    for c in range(grid.ncell):
        base = _cell_unknowns(state, c, pack)
        nadj = int(ws.adj_ptr[c + 1] - ws.adj_ptr[c])
        rows_cp = [np.zeros(nu) for _ in range(nadj)]
        rows_cm = [np.zeros(nu) for _ in range(nadj)]
        for u in range(nu):
            vp, vm = _fd_points(pack, base, u, state.sw[c], state.sg[c])
            scal = {"p": state.p[c], "t": state.t[c], "sw": state.sw[c], "sg": state.sg[c],
                    "cc": state.cc[c], "x": np.array(state.x[c], dtype=np.float64),
                    "y": np.array(state.y[c], dtype=np.float64)}
            _apply_unknown(scal, u, vp, pack)
            rows_p, fw_p = _probe_rows(grid, model, ws, wells, streams, state, accn, dt, c,
                                       scal, probe, rows_cp, freeze)
            _apply_unknown(scal, u, vm, pack)
            rows_m, fw_m = _probe_rows(grid, model, ws, wells, streams, state, accn, dt, c,
                                       scal, probe, rows_cm, freeze)
            inv2h = 1.0 / (vp - vm)
            ws.diag[c][:, u] = (rows_p - rows_m) * inv2h
            for slot, k in enumerate(range(ws.adj_ptr[c], ws.adj_ptr[c + 1])):
                ic = ws.adj_ids[k]
                side = 1 if ws.adj_sides[k] == 0 else 0
                ws.offd[ic, side][:, u] = (rows_cp[slot] - rows_cm[slot]) * inv2h
            for wix, pix in perf_lookup.get(c, ()):
                if wix in rate_wells:
                    blocks[wix].wrow[pix, u] = (fw_p.get(wix, 0.0) - fw_m.get(wix, 0.0)) * inv2h
                else:
                    blocks[wix].wrow[pix, u] = 0.0
    # bhp columns (assembly.py:903-939)
    for wix, well in enumerate(wells):
        h = max(FD_REL_STEP * abs(state.bhp[wix]), FD_PRESSURE_FLOOR)
        for pix, perf in enumerate(well.perfs):
            c = perf.cell
            dz = perf.z_bh - grid.depth[c]
            outs = []
            for bhp in (state.bhp[wix] + h, state.bhp[wix] - h):
                if well.kind == INJECTOR:
                    prow, _, _, qph, _, _ = _perf_injector(pack, ws, c, streams[wix], bhp,
                                                           perf.wi, dz)
                else:
                    prow, _, _, qph, _, _ = _perf_producer(pack, ws, c, state.x[c], bhp,
                                                           perf.wi, dz)
                outs.append((prow, qph.sum()))
            blocks[wix].bcol[pix] = -(outs[0][0] - outs[1][0]) * (0.5 / h)
        if well.control == CTRL_BHP or capped[wix]:
            blocks[wix].dwdb = 1.0
        else:
            dq = 0.0
            for pix, perf in enumerate(well.perfs):
                c = perf.cell
                dz = perf.z_bh - grid.depth[c]
                qs = []
                for bhp in (state.bhp[wix] + h, state.bhp[wix] - h):
                    if well.kind == INJECTOR:
                        _, _, _, qph, _, _ = _perf_injector(pack, ws, c, streams[wix], bhp,
                                                            perf.wi, dz)
                    else:
                        _, _, _, qph, _, _ = _perf_producer(pack, ws, c, state.x[c], bhp,
                                                            perf.wi, dz)
                    qs.append(qph.sum())
                dq += (qs[0] - qs[1]) * 0.5 / h
            blocks[wix].dwdb = dq


def check_jacobian(grid, model, ws, wells, streams, state, accn, dt, t_new, capped):
    """assembly.py:942-982: worst |analytic - numeric| / max(1, |analytic|)."""
    blocks = assemble(grid, model, ws, wells, streams, state, accn, dt, t_new, capped)
    diag_a, offd_a = ws.diag.copy(), ws.offd.copy()
    wrow_a = [b.wrow.copy() for b in blocks]
    bcol_a = [b.bcol.copy() for b in blocks]
    dwdb_a = [b.dwdb for b in blocks]
    numeric_jacobian(grid, model, ws, wells, streams, state, accn, dt, t_new, capped, blocks)

    def scaled(a, n):
        return np.max(np.abs(a - n) / np.maximum(1.0, np.abs(a))) if a.size else 0.0

    worst = max(scaled(diag_a, ws.diag), scaled(offd_a, ws.offd))
    for wix, b in enumerate(blocks):
        worst = max(worst, scaled(wrow_a[wix], b.wrow), scaled(bcol_a[wix], b.bcol),
                    abs(dwdb_a[wix] - b.dwdb) / max(1.0, abs(dwdb_a[wix])))
    ws.diag[:] = diag_a
    ws.offd[:] = offd_a
    for wix, b in enumerate(blocks):
        b.wrow[:] = wrow_a[wix]
        b.bcol[:] = bcol_a[wix]
        b.dwdb = dwdb_a[wix]
    return worst


# ------------------------------------------------------------ linear solver

def subdomain_count(ncell: int) -> int:
    """linsolve.py:40-42"""
    return min(MAX_SUBDOMAINS, max(1, ncell // SUBDOMAIN_CELLS))


def partition_cells(grid, p):
    """grid.py:148-186: owned cells and halo cells per slab."""
    dims = (grid.nx, grid.ny, grid.nz)
    axis = int(np.argmax(dims))
    base, extra = divmod(dims[axis], p)
    slab_of = np.repeat(np.arange(p), [base + (1 if s < extra else 0) for s in range(p)])
    c = np.arange(grid.ncell)
    ijk = (c % grid.nx, (c // grid.nx) % grid.ny, c // (grid.nx * grid.ny))
    owner = slab_of[ijk[axis]]
    cells = [np.flatnonzero(owner == s).astype(np.int64) for s in range(p)]
    ca, cb = np.asarray(grid.conn_a, np.int64), np.asarray(grid.conn_b, np.int64)
    sa, sb = owner[ca], owner[cb]
    cut = sa != sb
    halos = []
    for s in range(p):
        h = np.concatenate([cb[cut & (sa == s)], ca[cut & (sb == s)]])
        halos.append(np.unique(h).astype(np.int64))
    return cells, halos


class _Subdomain:
    """linsolve.py:262-298"""

    def __init__(self, grid, owned, ext):
        self.cells = ext
        self.owned = owned
        self.owned_pos = np.searchsorted(ext, owned)
        in_ext = np.zeros(grid.ncell, dtype=bool)
        in_ext[ext] = True
        mask = in_ext[grid.conn_a] & in_ext[grid.conn_b]
        ics = np.nonzero(mask)[0].astype(np.int64)
        la = np.searchsorted(ext, grid.conn_a[ics])
        lb = np.searchsorted(ext, grid.conn_b[ics])
        n = ext.shape[0]
        lo_c = np.where(la > lb, la, lb)
        lo_j = np.where(la > lb, lb, la)
        lo_sd = np.where(la > lb, 0, 1).astype(np.int8)
        order = np.lexsort((lo_j, lo_c))
        self.low_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(lo_c, minlength=n), out=self.low_ptr[1:])
        self.low_j = _c(lo_j[order], np.int64)
        self.low_ic = _c(ics[order], np.int64)
        self.low_sd = _c(lo_sd[order], np.int8)
        up_c, up_j, up_sd = lo_j, lo_c, (1 - lo_sd).astype(np.int8)
        order = np.lexsort((up_j, up_c))
        self.up_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(up_c, minlength=n), out=self.up_ptr[1:])
        self.up_j = _c(up_j[order], np.int64)
        self.up_ic = _c(ics[order], np.int64)
        self.up_sd = _c(up_sd[order], np.int8)


class BlockSolver:
    """linsolve.py:317-578 (BiCGSTAB with none / bjacobi / ras), plus
    ``mcilu``: the north star's multicolour (red-black) block ILU(0) of the
    decoupled system as the right preconditioner of the same BiCGSTAB (the
    reference has no such preconditioner; this restates the algorithm the
    device solves in red-eliminated form, so its iteration
    counts and solutions have a CPU checker)."""

    def __init__(self, grid, ws, tol=1e-5, maxiter=200, precond="ras", threads=1):
        if precond not in ("none", "bjacobi", "ras", "mcilu"):
            raise ValueError(f"unknown preconditioner {precond!r}")
        # threads > 1: the independent subdomains' factor / apply calls run on a
        # thread pool (ctypes releases the GIL). Each subdomain writes only its
        # own slots and owned rows, so results are bit-identical to the
        # reference's serial loop (linsolve.py:398-421); used by bench.py's CPU arm.
        self._pool = None
        if threads > 1:
            from concurrent.futures import ThreadPoolExecutor
            self._pool = ThreadPoolExecutor(max_workers=threads)
        self.grid, self.ws, self.tol, self.maxiter, self.precond = grid, ws, tol, maxiter, precond
        self.nu = ws.resid.shape[1]
        n = grid.ncell
        self.invs = np.zeros((n, self.nu, self.nu))
        self.flags = np.zeros(n, dtype=np.int64)
        self.other = _c(np.where(ws.adj_sides == 0, grid.conn_b[ws.adj_ids],
                                 grid.conn_a[ws.adj_ids]), np.int64)
        self.subs: List[_Subdomain] = []
        if precond == "mcilu":
            i, j, k = (np.arange(n) % grid.nx, (np.arange(n) // grid.nx) % grid.ny,
                       np.arange(n) // (grid.nx * grid.ny))
            self.black = ((i + j + k) % 2) == 1
        elif precond != "none":
            owned_l, halos = partition_cells(grid, subdomain_count(n))
            for owned, halo in zip(owned_l, halos):
                ext = np.union1d(owned, halo).astype(np.int64) if (
                    precond == "ras" and halo.size) else owned
                self.subs.append(_Subdomain(grid, owned, ext))
            self._uinv = [np.zeros((s.cells.shape[0], self.nu, self.nu)) for s in self.subs]
            self._lblk = [np.zeros((s.low_j.shape[0], self.nu, self.nu)) for s in self.subs]
            self._zloc = [np.zeros((s.cells.shape[0], self.nu)) for s in self.subs]

    def _eliminate_wells(self, blocks, rhs):
        """linsolve.py:362-394 (single perforation: no extra blocks)."""
        elims = []
        for b in blocks:
            if b.dwdb == 0.0 or not np.isfinite(b.dwdb):
                raise SingularCellBlock("well equation has a zero bhp derivative")
            inv_d = 1.0 / b.dwdb
            for p in range(b.cells.shape[0]):
                c = b.cells[p]
                rhs[c] += b.bcol[p] * (b.resid * inv_d)
                for q in range(b.cells.shape[0]):
                    upd = np.outer(b.bcol[p], b.wrow[q]) * inv_d
                    if b.cells[q] != c:
                        raise NotImplementedError("multi-perforation wells")
                    self.ws.diag[c] -= upd
            elims.append((b.cells, b.wrow.copy(), b.dwdb, b.resid))
        return elims

    def _mc_factor(self):
        """Red-black block ILU(0) of the decoupled A (diagonal blocks taken as
        I, as stored after decoupling): U_b = I - sum_r A_br A_rb per black
        cell (the fill-in of the 7-point pattern stays on the block diagonal)."""
        ws, g = self.ws, self.grid
        a, b = np.asarray(g.conn_a, np.int64), np.asarray(g.conn_b, np.int64)
        ub = np.tile(np.eye(self.nu), (g.ncell, 1, 1))
        blk_a = self.black[a]   # connection's black end is a (else b)
        prod_a = np.einsum("cij,cjk->cik", ws.offd[:, 0], ws.offd[:, 1])   # A_ab A_ba
        prod_b = np.einsum("cij,cjk->cik", ws.offd[:, 1], ws.offd[:, 0])   # A_ba A_ab
        np.subtract.at(ub, a[blk_a], prod_a[blk_a])
        np.subtract.at(ub, b[~blk_a], prod_b[~blk_a])
        try:
            self._ubinv = np.linalg.inv(ub[self.black])
        except np.linalg.LinAlgError as exc:
            raise SingularCellBlock(f"multicolour ILU(0) pivot block is singular: {exc}")

    def _mc_apply(self, r, z):
        """z = U^-1 L^-1 r: z_r = r_r; w_b = r_b - A_br z_r; z_b = U_b^-1 w_b;
        z_r = r_r - A_rb z_b."""
        ws, g = self.ws, self.grid
        a, b = np.asarray(g.conn_a, np.int64), np.asarray(g.conn_b, np.int64)
        blk_a = self.black[a]
        red_c = np.where(blk_a, b, a)
        blk_c = np.where(blk_a, a, b)
        a_br = np.where(blk_a[:, None, None], ws.offd[:, 0], ws.offd[:, 1])
        a_rb = np.where(blk_a[:, None, None], ws.offd[:, 1], ws.offd[:, 0])
        w = r.copy()
        np.subtract.at(w, blk_c, np.einsum("cij,cj->ci", a_br, r[red_c]))
        z[:] = r
        z[self.black] = np.einsum("cij,cj->ci", self._ubinv, w[self.black])
        np.subtract.at(z, red_c, np.einsum("cij,cj->ci", a_rb, z[blk_c]))

    def _factor(self):
        if self.precond == "mcilu":
            self._mc_factor()
            return
        ws = self.ws

        def one(s):
            sub = self.subs[s]
            return lib().orc_ilu_factor(
                ctypes.c_int64(self.nu), _p(ws.diag), _p(ws.offd),
                ctypes.c_int64(sub.cells.shape[0]), _p(sub.cells), _p(sub.low_ptr),
                _p(sub.low_j), _p(sub.low_ic), _p(sub.low_sd), _p(self._uinv[s]),
                _p(self._lblk[s]))

        idx = range(len(self.subs))
        bads = list(self._pool.map(one, idx)) if self._pool else [one(s) for s in idx]
        for s, bad in enumerate(bads):   # first failing subdomain, as the serial loop
            if bad >= 0:
                raise SingularCellBlock(
                    f"ILU(0) pivot failed in cell {int(self.subs[s].cells[bad])}")

    def _apply_precond(self, r, z):
        if self.precond == "none":
            z[:] = r
            return
        if self.precond == "mcilu":
            self._mc_apply(r, z)
            return
        z[:] = 0.0
        r = _c(r)

        def one(s):
            sub = self.subs[s]
            lib().orc_ilu_apply(
                ctypes.c_int64(self.nu), _p(r), ctypes.c_int64(sub.cells.shape[0]),
                _p(sub.cells), _p(sub.low_ptr), _p(sub.low_j), _p(self._lblk[s]),
                _p(sub.up_ptr), _p(sub.up_j), _p(sub.up_ic), _p(sub.up_sd), _p(self.ws.offd),
                _p(self._uinv[s]), _p(self._zloc[s]))

        if self._pool:
            list(self._pool.map(one, range(len(self.subs))))
        else:
            for s in range(len(self.subs)):
                one(s)
        for s, sub in enumerate(self.subs):
            z[sub.owned] = self._zloc[s][sub.owned_pos]

    def _matvec(self, v, out):
        ws = self.ws
        lib().orc_matvec(ctypes.c_int64(v.shape[0]), ctypes.c_int64(self.nu), _p(ws.diag),
                         _p(ws.offd), _p(ws.adj_ptr), _p(ws.adj_ids), _p(ws.adj_sides),
                         _p(self.other), _p(_c(v)), _p(out))

    @staticmethod
    def _dot(a, b):
        a, b = _c(a), _c(b)
        return lib().orc_dot(ctypes.c_int64(a.size), _p(a), _p(b))

    def solve(self, blocks):
        """linsolve.py:438-479"""
        ws = self.ws
        rhs = -ws.resid
        elims = self._eliminate_wells(blocks, rhs)
        self.flags[:] = 0
        # mcilu: the local rows' block of every cell before decoupling (the
        # condensed form below needs D[6:, :] after the well fold)
        dloc = None
        if self.precond == "mcilu" and not np.any(ws.offd[:, :, CR_:, :] != 0.0):
            dloc = ws.diag[:, CR_:, :].copy()   # (an assembled system's structure)
        lib().orc_decouple_pass(ctypes.c_int64(rhs.shape[0]), ctypes.c_int64(self.nu),
                                _p(ws.diag), _p(rhs), _p(ws.offd), _p(ws.adj_ptr),
                                _p(ws.adj_ids), _p(ws.adj_sides), _p(self.invs), _p(self.flags))
        if self.flags.any():
            cell = int(np.argmax(self.flags > 0))
            raise SingularCellBlock(
                f"diagonal block of cell {cell} is singular at column {int(self.flags[cell] - 1)}")
        if self.precond != "none":
            self._factor()
        cond = self._cond_setup(dloc) if dloc is not None and self.condensed else None
        du, iters = self._cond_solve(rhs, cond) if cond is not None else self._bicgstab(rhs)
        dbhp = np.zeros(len(elims))
        for w, (cells, wrow, dwdb, resid) in enumerate(elims):
            s = resid
            for p in range(cells.shape[0]):
                s += float(wrow[p] @ du[cells[p]])
            dbhp[w] = -s / dwdb
        return du, dbhp, iters

    # ------------------------------------------------------------------
    # Condensed multicolour solve (the device's mcilu default, compact.cu
    # "condensed form"; no reference counterpart). With the decoupled blocks
    # A = D^-1 B of an assembled system (rows >= CR_ of B are zero) the
    # red-eliminated system S9 x_b = g_b (S9 = I - A_br A_rb, g_b = b_b -
    # A_br b_r) has x_b - g_b in range(E_b), E = [I; E_S] over the primary
    # unknowns P, E_S = -D[CR_:, S]^-1 D[CR_:, P] from the local rows. So
    # x_b = g_b + E_b w with the 6-component system
    #     S6 w = h,  S6 = P S9 E,  h = P (g_b - S9 g_b)
    # solved by the same BiCGSTAB (linsolve.py:481-578 control flow) from
    # w = 0, right-preconditioned by the diagonal blocks of S6 (the ILU(0)
    # pivot blocks restricted to P), stopping on ||r6|| / ||b|| with b the
    # full decoupled rhs. Then x_r = b_r - A_rb x_b.
    condensed = True

    def _cond_setup(self, dloc):
        ws, g = self.ws, self.grid
        black = self.black
        m = dloc[black][:, :, COND_S]            # (nb, 3, 3)
        r = dloc[black][:, :, COND_P]            # (nb, 3, 6)
        try:
            es = -np.linalg.solve(m, r)
        except np.linalg.LinAlgError:
            return None
        if not np.all(np.isfinite(es)):
            return None
        nb = int(black.sum())
        e = np.zeros((nb, self.nu, CR_))
        e[:, COND_P, :] = np.eye(CR_)[None]
        e[:, COND_S, :] = es
        a, b = np.asarray(g.conn_a, np.int64), np.asarray(g.conn_b, np.int64)
        blk_a = black[a]
        red_c = np.where(blk_a, b, a)
        blk_c = np.where(blk_a, a, b)
        a_br = np.where(blk_a[:, None, None], ws.offd[:, 0], ws.offd[:, 1])
        a_rb = np.where(blk_a[:, None, None], ws.offd[:, 1], ws.offd[:, 0])
        bpos = np.full(g.ncell, -1, dtype=np.int64)
        bpos[black] = np.arange(nb)

        def s9(xb):   # (nb, 9) -> S9 xb
            z = np.zeros((g.ncell, self.nu))
            z[black] = xb
            y = np.zeros((g.ncell, self.nu))
            np.add.at(y, red_c, np.einsum("cij,cj->ci", a_rb, z[blk_c]))   # A_rb xb
            out = z.copy()
            np.subtract.at(out, blk_c, np.einsum("cij,cj->ci", a_br, y[red_c]))
            return out[black]

        # diagonal blocks of S6: P (I - sum_r A_br A_rb) E (the red neighbours' paths)
        d9 = np.tile(np.eye(self.nu), (nb, 1, 1))
        prod = np.einsum("cij,cjk->cik", a_br, a_rb)   # A_br(r) A_rb(r) per connection
        np.subtract.at(d9, bpos[blk_c], prod)
        u6 = np.einsum("cpi,cij,cjq->cpq", np.eye(self.nu)[COND_P][None].repeat(nb, 0), d9, e)
        try:
            u6inv = np.linalg.inv(u6)
        except np.linalg.LinAlgError as exc:
            raise SingularCellBlock(f"multicolour ILU(0) pivot block is singular: {exc}")
        return dict(e=e, s9=s9, u6inv=u6inv, red_c=red_c, blk_c=blk_c, a_rb=a_rb, a_br=a_br,
                    nb=nb)

    def _cond_solve(self, bfull, C):
        black, e, s9, nb = self.black, C["e"], C["s9"], C["nb"]
        red_c, blk_c, a_rb, a_br = C["red_c"], C["blk_c"], C["a_rb"], C["a_br"]
        # g_b = b_b - A_br b_r
        gfull = bfull.copy()
        np.subtract.at(gfull, blk_c, np.einsum("cij,cj->ci", a_br, bfull[red_c]))
        g9 = gfull[black]
        h = (g9 - s9(g9))[:, COND_P]

        def op(w):   # S6 w (flat)
            w = w.reshape(nb, CR_)
            return s9(np.einsum("cij,cj->ci", e, w))[:, COND_P].ravel()

        def prec(v):
            return np.einsum("cij,cj->ci", C["u6inv"], v.reshape(nb, CR_)).ravel()

        w, it = self._bicgstab_op(h.ravel(), op, prec, np.sqrt(self._dot(bfull, bfull)))
        xb = g9 + np.einsum("cij,cj->ci", e, w.reshape(nb, CR_))
        x = bfull.copy()
        x[black] = xb
        xz = np.zeros_like(bfull)
        xz[black] = xb
        np.subtract.at(x, red_c, np.einsum("cij,cj->ci", a_rb, xz[blk_c]))
        return x, it

    def _bicgstab_op(self, b, op, prec, nb):
        """_bicgstab's control flow (linsolve.py:481-578) on an operator with
        a right preconditioner; the tolerance base nb is given (the full
        system's ||b||)."""
        x = np.zeros_like(b)
        if nb == 0.0:
            return x, 0
        r, rhat = b.copy(), b.copy()
        p, v = np.zeros_like(b), np.zeros_like(b)
        rho_old = alpha = omega = 1.0
        restarted, it, first = False, 0, True

        def restart():
            r = b - op(x)
            return r, r.copy()

        while it < self.maxiter:
            it += 1
            rho = self._dot(rhat, r)
            if abs(rho) < BREAKDOWN_EPS * nb * nb or (not first and omega == 0.0):
                if restarted:
                    raise Breakdown(f"BiCGSTAB scalar breakdown at iteration {it}")
                r, rhat = restart()
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                rho = self._dot(rhat, r)
                if abs(rho) < BREAKDOWN_EPS * nb * nb:
                    raise Breakdown("BiCGSTAB restart found a null residual")
            if first:
                p[:] = r
                first = False
            else:
                beta = (rho / rho_old) * (alpha / omega)
                p = r + beta * (p - omega * v)
            phat = prec(p)
            v = op(phat)
            den = self._dot(rhat, v)
            if abs(den) < BREAKDOWN_EPS * nb * nb:
                if restarted:
                    raise Breakdown(f"BiCGSTAB denominator breakdown at iteration {it}")
                r, rhat = restart()
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                continue
            alpha = rho / den
            s = r - alpha * v
            if np.sqrt(self._dot(s, s)) / nb <= self.tol:
                x += alpha * phat
                return x, it
            shat = prec(s)
            t = op(shat)
            tt = self._dot(t, t)
            if tt == 0.0:
                if restarted:
                    raise Breakdown("BiCGSTAB stagnated (t = 0)")
                r, rhat = restart()
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                continue
            omega = self._dot(t, s) / tt
            x += alpha * phat + omega * shat
            r = s - omega * t
            if np.sqrt(self._dot(r, r)) / nb <= self.tol:
                return x, it
            rho_old = rho
        raise MaxIterations(f"BiCGSTAB did not converge in {self.maxiter} iterations")

    def _restart(self, b, x, t):
        self._matvec(x, t)
        r = b - t
        return r, r.copy()

    def _bicgstab(self, b):
        """linsolve.py:481-578"""
        x = np.zeros_like(b)
        nb = np.sqrt(self._dot(b, b))
        if nb == 0.0:
            return x, 0
        r, rhat = b.copy(), b.copy()
        p, v = np.zeros_like(b), np.zeros_like(b)
        phat, shat, t = np.zeros_like(b), np.zeros_like(b), np.zeros_like(b)
        rho_old = alpha = omega = 1.0
        restarted, it, first = False, 0, True
        while it < self.maxiter:
            it += 1
            rho = self._dot(rhat, r)
            if abs(rho) < BREAKDOWN_EPS * nb * nb or (not first and omega == 0.0):
                if restarted:
                    raise Breakdown(f"BiCGSTAB scalar breakdown at iteration {it}")
                r, rhat = self._restart(b, x, t)
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                rho = self._dot(rhat, r)
                if abs(rho) < BREAKDOWN_EPS * nb * nb:
                    raise Breakdown("BiCGSTAB restart found a null residual")
            if first:
                p[:] = r
                first = False
            else:
                beta = (rho / rho_old) * (alpha / omega)
                p = r + beta * (p - omega * v)
            self._apply_precond(p, phat)
            self._matvec(phat, v)
            den = self._dot(rhat, v)
            if abs(den) < BREAKDOWN_EPS * nb * nb:
                if restarted:
                    raise Breakdown(f"BiCGSTAB denominator breakdown at iteration {it}")
                r, rhat = self._restart(b, x, t)
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                continue
            alpha = rho / den
            s = r - alpha * v
            if np.sqrt(self._dot(s, s)) / nb <= self.tol:
                x += alpha * phat
                return x, it
            self._apply_precond(s, shat)
            self._matvec(shat, t)
            tt = self._dot(t, t)
            if tt == 0.0:
                if restarted:
                    raise Breakdown("BiCGSTAB stagnated (t = 0)")
                r, rhat = self._restart(b, x, t)
                p[:] = 0.0
                v[:] = 0.0
                rho_old = alpha = omega = 1.0
                first, restarted = True, True
                continue
            omega = self._dot(t, s) / tt
            x += alpha * phat + omega * shat
            r = s - omega * t
            if np.sqrt(self._dot(r, r)) / nb <= self.tol:
                return x, it
            rho_old = rho
        raise MaxIterations(f"BiCGSTAB did not converge in {self.maxiter} iterations")


# ------------------------------------------------------------ Newton driver

def _damp_array(old, raw, eps):
    """newton.py:80-89"""
    out = raw.copy()
    neg = raw < 0.0
    if np.any(neg):
        out[neg] = np.sqrt(eps * np.maximum(old[neg], 0.0))
    halve = ~neg & (raw < eps) & (old >= eps)
    if np.any(halve):
        out[halve] = 0.5 * old[halve]
    return out


def apply_update(state, du, dbhp, nco, ncg, eps):
    """newton.py:92-121"""
    new = state.copy()
    ct = 1 + nco + ncg
    new.p += du[:, 0]
    new.x = np.clip(new.x + du[:, 1:1 + nco], 0.0, 1.0)
    new.y = np.clip(new.y + du[:, 1 + nco:ct], 0.0, 1.0)
    new.t = np.maximum(new.t + du[:, ct], -459.0)
    new.cc = np.maximum(new.cc + du[:, ct + 3], 0.0)
    so_old = 1.0 - state.sw - state.sg
    sw = _damp_array(state.sw, state.sw + du[:, ct + 1], eps)
    sg = _damp_array(state.sg, state.sg + du[:, ct + 2], eps)
    so = _damp_array(so_old, 1.0 - sw - sg, eps)
    sg = 1.0 - sw - so
    neg = sg < 0.0
    if np.any(neg):
        sg[neg] = _damp_array(state.sg, sg, eps)[neg]
    sw = np.clip(sw, 0.0, 1.0)
    sg = np.clip(sg, 0.0, 1.0 - sw)
    new.sw, new.sg = sw, sg
    new.bhp = state.bhp + dbhp
    return new


def scaled_norm(ws, accn, volume, dt, blocks, wells, capped, row_os, row_gs):
    """newton.py:124-144"""
    scale = (volume / dt)[:, None] * np.maximum(1.0, np.abs(accn))
    scale[:, row_os] = 1.0
    scale[:, row_gs] = 1.0
    norm = float(np.max(np.abs(ws.resid) / scale))
    for w, (well, blk) in enumerate(zip(wells, blocks)):
        target = well.pinjmax if capped[w] else well.target
        norm = max(norm, abs(blk.resid) / max(1.0, abs(target)))
    return norm


def desired_capped(wells, capped, state, blocks):
    """newton.py:147-168"""
    want = capped.copy()
    for w, well in enumerate(wells):
        if well.kind != INJECTOR or well.control == CTRL_BHP:
            continue
        if not math.isfinite(well.pinjmax):
            continue
        if capped[w]:
            if float(np.sum(blocks[w].phase_rates)) > well.target:
                want[w] = False
        elif state.bhp[w] > well.pinjmax:
            want[w] = True
    return want


@dataclass
class StepRecord:
    time: float
    dt: float
    newton: int
    linear: int
    solves: int
    balance: float


class Simulator:
    """newton.py:214-437 restated over the oracle kernels.

    Built from explicit pieces (grid, pack, wells, streams, initial state,
    schedule, solver settings) instead of a deck.
    """

    def __init__(self, grid, pack, wells, streams, state, schedule, solver, heat_loss=None,
                 jacobian="analytic", threads=1):
        self.jacobian = jacobian   # newton.py:228
        self.grid, self.pack, self.wells, self.streams = grid, pack, tuple(wells), streams
        self.schedule, self.solver_cfg = schedule, solver
        self.model = Model(pack)
        self.ws = Workspace(grid, pack, heat_loss)
        self.solver = BlockSolver(grid, self.ws, tol=solver.linear_tol,
                                  maxiter=solver.linear_max, precond=solver.precond,
                                  threads=threads)
        self.state = state.copy()
        self.capped = np.zeros(len(self.wells), dtype=bool)
        self.time = 0.0
        self.blocks: List[WellBlock] = []
        zero = np.zeros((grid.ncell, pack.nequ))
        self.blocks = assemble(grid, self.model, self.ws, self.wells, self.streams, self.state,
                               zero, 1.0, 0.0, self.capped)
        self.accn = self.ws.acc.copy()
        self.steps: List[StepRecord] = []
        self.cum_imbalance = np.zeros(pack.nfull + 1)
        self.cum_throughput = np.zeros(pack.nfull + 1)
        self.cum_rates = np.zeros((len(self.wells), 3))
        self.work_seconds = 0.0
        self.newton_iterations = 0      # assemble+solve iterations (bench accounting)

    def newton_step(self, state, dt, t_new, capped):
        """newton.py:254-310"""
        import time as _time
        pack, grid, cfg = self.pack, self.grid, self.solver_cfg
        work, capped = state, capped.copy()
        lin_total = solves = growths = 0
        prev = math.inf
        for it in range(1, cfg.newton_max + 1):
            t0 = _time.perf_counter()
            blocks = assemble(grid, self.model, self.ws, self.wells, self.streams, work,
                              self.accn, dt, t_new, capped,
                              freeze_upwind=(it > FREEZE_UPWIND_AFTER), jacobian=self.jacobian)
            self.work_seconds += _time.perf_counter() - t0
            norm = scaled_norm(self.ws, self.accn, grid.volume, dt, blocks, self.wells, capped,
                               pack.row_energy + 1, pack.row_energy + 2)
            if not math.isfinite(norm) or norm > prev:
                growths += 1
                if growths >= 3:
                    raise DivergedResidual(f"residual grew {growths} consecutive iterations")
            else:
                growths = 0
            if math.isfinite(norm):
                prev = norm
            want = desired_capped(self.wells, capped, work, blocks)
            if not np.array_equal(want, capped):
                capped = want
                continue
            if norm <= cfg.newton_tol:
                self.blocks = blocks
                return work, True, it, lin_total, solves, capped
            if it == cfg.newton_max:
                break
            t0 = _time.perf_counter()
            du, dbhp, iters = self.solver.solve(blocks)
            self.work_seconds += _time.perf_counter() - t0
            lin_total += iters
            solves += 1
            work = apply_update(work, du, dbhp, pack.nco, pack.ncg, cfg.eps)
        return state, False, cfg.newton_max, lin_total, solves, capped

    def report_times(self):
        s = self.schedule
        times = set(t for t in s.report_times if 0.0 <= t <= s.t_end + TIME_EPS)
        if s.report_interval:
            nrep = int(math.floor(s.t_end / s.report_interval + TIME_EPS))
            times.update(k * s.report_interval for k in range(1, nrep + 1))
        times.add(s.t_end)
        return sorted(times)

    def forced_times(self):
        """newton.py:312-323"""
        s = self.schedule
        times = set(rt for rt in self.report_times() if rt > TIME_EPS)
        for well in self.wells:
            if well.heat_rate and 0.0 < well.heat_stop < s.t_end:
                times.add(well.heat_stop)
        times.add(s.t_end)
        return sorted(times)

    def audit_step(self, dt):
        """newton.py:339-366"""
        pack, vol = self.pack, self.grid.volume
        rows = list(range(pack.nfull)) + [pack.nequ - 1]
        worst = 0.0
        for k, r in enumerate(rows):
            dacc = float(np.dot(vol, self.ws.acc[:, r] - self.accn[:, r]))
            reac = float(np.dot(vol, self.ws.src[:, r]))
            wellq = wellabs = 0.0
            for blk in self.blocks:
                q = float(np.sum(blk.comp_rates[:, r]))
                wellq += q
                wellabs += abs(q)
            imb = dacc - dt * (reac + wellq)
            scale = max(1.0, float(np.dot(vol, np.abs(self.ws.acc[:, r]))))
            worst = max(worst, abs(imb) / scale)
            self.cum_imbalance[k] += imb
            self.cum_throughput[k] += dt * (wellabs + abs(reac))
        return worst

    def advance(self, log_cb=None):
        """newton.py:373-431 (report callbacks omitted: no frames written)."""
        s = self.schedule
        dtc, dt_min, dt_max = s.dt_init, s.dt_min, s.dt_max
        forced = self.forced_times()
        while self.time < s.t_end - TIME_EPS:
            dt = min(dtc, dt_max)
            for ft in forced:
                if ft > self.time + TIME_EPS:
                    dt = min(dt, ft - self.time)
                    break
            t_new = self.time + dt
            for ft in forced:
                if abs(t_new - ft) <= TIME_EPS:
                    t_new = ft
                    break
            dt = t_new - self.time
            try:
                state, ok, iters, lin, solves, capped = self.newton_step(
                    self.state, dt, t_new, self.capped)
                reason = "" if ok else "newton iteration limit"
            except (DivergedResidual, SingularCellBlock, Breakdown, MaxIterations,
                    PoreSpaceExhausted, DegenerateTemperature) as exc:
                if not self.steps and isinstance(exc, PoreSpaceExhausted):
                    raise
                ok, iters, lin, solves = False, 0, 0, 0
                reason = f"{type(exc).__name__}: {exc}"
            if not ok:
                if log_cb:
                    log_cb(f"t={self.time:g} dt={dt:g} rejected ({reason})")
                if dt <= dt_min * (1.0 + 1e-9):
                    raise SimulationStalled(f"timestep {dt:g} failed ({reason})")
                dtc = max(dt * CUT_FACTOR, dt_min)
                continue
            self.state, self.capped, self.time = state, capped, t_new
            balance = self.audit_step(dt)
            self.accn = self.ws.acc.copy()
            for w, blk in enumerate(self.blocks):
                self.cum_rates[w] += dt * blk.phase_rates.sum(axis=0)
            self.steps.append(StepRecord(time=t_new, dt=dt, newton=iters, linear=lin,
                                         solves=solves, balance=balance))
            if log_cb:
                log_cb(f"t={t_new:g} dt={dt:g} newton={iters} linear={lin}")
            if iters <= FAST_ITERS:
                dtc = min(dtc * GROWTH_FACTOR, dt_max)

    def totals(self):
        return (len(self.steps), sum(s.newton for s in self.steps),
                sum(s.linear for s in self.steps))

    def cumulative_imbalance(self):
        return float(np.max(np.abs(self.cum_imbalance) / np.maximum(1.0, self.cum_throughput)))
