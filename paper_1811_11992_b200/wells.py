"""Peaceman wells (setup only) and injector stream constants.

Same ``Well``/``Perforation``/``WellStream`` fields as the reference
(wells.py:36-54, assembly.py:222-231) so the drop-in ``assemble`` accepts
either. One perforation per well, as in the reference (wells.py:134-137).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from .model import (GASP_AVG, GASP_BVG, GASP_CPG1, GASP_CPG2, GASP_CPG3,
                    GASP_CPG4, GASP_M, RK_TREF)

INJECTOR, PRODUCER = 0, 1                              # wells.py:32
CTRL_BHP, CTRL_RATE_GAS, CTRL_RATE_TOTAL = 0, 1, 2     # wells.py:33
SCF_PER_LBMOL = 379.3                                  # units.py:30
RANKINE_OFFSET = 459.67


@dataclass(frozen=True)
class Perforation:
    cell: int
    wi: float
    z_bh: float


@dataclass(frozen=True, eq=False)
class Well:
    name: str
    kind: int
    control: int
    target: float
    perfs: Tuple[Perforation, ...]
    yinj: Optional[np.ndarray]
    tinj: float
    pinjmax: float
    heat_rate: float
    heat_stop: float


@dataclass(frozen=True)
class WellSpec:
    """Deck-level description of one well (the *WELL section's fields)."""

    name: str
    kind: str                       # "injector" | "producer"
    i: int
    j: int
    k: int                          # 1-based
    control: str = "bhp"            # "bhp" | "rate_gas" | "rate_total"
    bhp: Optional[float] = None
    rate: Optional[float] = None
    rate_conditions: str = "standard"
    wi: Optional[float] = None
    radius: Optional[float] = None
    skin: float = 0.0
    yinj: Optional[Tuple[float, ...]] = None
    tinj: Optional[float] = None
    pinjmax: Optional[float] = None
    heat_rate: float = 0.0
    heat_stop: float = 0.0
    zbh: Optional[float] = None


def equivalent_radius(dx: float, dy: float, kx: float, ky: float) -> float:
    """Peaceman anisotropic r_e (wells.py:57-61)."""
    r = ky / kx
    return (0.28 * math.sqrt(math.sqrt(r) * dx * dx + math.sqrt(1.0 / r) * dy * dy)
            / (r ** 0.25 + (1.0 / r) ** 0.25))


def well_index(dx, dy, h3, k11, k22, rw, skin) -> float:
    """Vertical-well Peaceman index (wells.py:64-77)."""
    if k11 <= 0.0 or k22 <= 0.0:
        raise ValueError("well cell needs positive horizontal permeability")
    if rw <= 0.0:
        raise ValueError("well radius must be positive")
    re = equivalent_radius(dx, dy, k11, k22)
    denom = math.log(re / rw) + skin
    if denom <= 0.0:
        raise ValueError(f"well index denominator ln(re/rw)+skin = {denom} is not positive")
    return 2.0 * math.pi * h3 * math.sqrt(k11 * k22) / denom


def gas_rate_to_molar(rate_ft3_per_hr: float) -> float:
    """Standard-condition ft³/hr to lbmol/day (wells.py:80-82)."""
    return rate_ft3_per_hr * 24.0 / SCF_PER_LBMOL


def build_wells(specs: Sequence[WellSpec], grid) -> Tuple[Well, ...]:
    """Runtime wells on the grid (wells.py:107-142)."""
    out = []
    for spec in specs:
        i, j, k = spec.i - 1, spec.j - 1, spec.k - 1
        cell = grid.cell_index(i, j, k)
        if spec.wi is not None:
            wi = float(spec.wi)
        else:
            wi = well_index(float(grid.dx[i]), float(grid.dy[j]), float(grid.dz[k]),
                            float(grid.kx[cell]), float(grid.ky[cell]),
                            float(spec.radius), float(spec.skin))
        z_bh = float(spec.zbh) if spec.zbh is not None else float(grid.depth[cell])
        kind = INJECTOR if spec.kind == "injector" else PRODUCER
        if spec.control == "bhp":
            control, target = CTRL_BHP, float(spec.bhp)
        elif spec.control == "rate_gas":
            control = CTRL_RATE_GAS
            target = (gas_rate_to_molar(spec.rate) if spec.rate_conditions == "standard"
                      else float(spec.rate))
        else:
            control, target = CTRL_RATE_TOTAL, float(spec.rate)
        out.append(Well(
            name=spec.name, kind=kind, control=control, target=target,
            perfs=(Perforation(cell=cell, wi=wi, z_bh=z_bh),),
            yinj=np.asarray(spec.yinj, dtype=np.float64) if spec.yinj else None,
            tinj=float(spec.tinj) if spec.tinj is not None else 0.0,
            pinjmax=float(spec.pinjmax) if spec.pinjmax is not None else math.inf,
            heat_rate=float(spec.heat_rate), heat_stop=float(spec.heat_stop)))
    return tuple(out)


@dataclass(frozen=True)
class WellStream:
    """Injected-gas constants (assembly.py:222-231)."""

    yfull: np.ndarray
    yinj: np.ndarray
    tinj: float
    mu: float
    h: float
    mbar: float


def build_streams(pack, wells) -> Tuple[Optional[WellStream], ...]:
    """Stream viscosity/enthalpy/molar mass at T_inj (assembly.py:234-277).

    Integer powers are written the way numba lowers ``t ** 3``/``t ** 4`` in
    the reference's gas_enthalpy (_props.py:181-191).
    """
    out = []
    t_ref = float(pack.rockp[RK_TREF])
    for well in wells:
        if well.kind != INJECTOR or well.yinj is None:
            out.append(None)
            continue
        yinj = np.asarray(well.yinj, dtype=np.float64)
        yfull = np.zeros(pack.nfull)
        yfull[1 + pack.nco:] = yinj
        wsum = musum = h = mbar = 0.0
        t = well.tinj
        tr = t + RANKINE_OFFSET
        for j in range(pack.ncg):
            if yinj[j] <= 0.0:
                continue
            g = pack.gasp[1 + pack.nco + j]
            m = float(g[GASP_M])
            sq = math.sqrt(m)
            mu_c = float(g[GASP_AVG]) * tr ** float(g[GASP_BVG])
            c1, c2, c3, c4 = (float(g[GASP_CPG1]), float(g[GASP_CPG2]),
                              float(g[GASP_CPG3]), float(g[GASP_CPG4]))
            t3, r3 = t * (t * t), t_ref * (t_ref * t_ref)
            t4, r4 = (t * t) * (t * t), (t_ref * t_ref) * (t_ref * t_ref)
            h_c = (c1 * (t - t_ref) + c2 / 2.0 * (t * t - t_ref * t_ref)
                   + c3 / 3.0 * (t3 - r3) + c4 / 4.0 * (t4 - r4))
            wsum += yinj[j] * sq
            musum += yinj[j] * mu_c * sq
            h += yinj[j] * h_c
            mbar += yinj[j] * m
        if wsum <= 0.0:
            raise ValueError(f"well {well.name}: injected composition has no gas content")
        out.append(WellStream(yfull=yfull, yinj=yinj, tinj=well.tinj,
                              mu=musum / wsum, h=h, mbar=mbar))
    return tuple(out)
