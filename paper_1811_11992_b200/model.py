"""Flattened fluid/rock/reaction constants (the reference's ``ModelPack``).

Same attribute names and array layouts as the reference's ``ModelPack``
(assembly.py:42-81) so either object can be handed to the drop-in
``assemble``. The column constants restate _kernels.py:48-63.

The packs used by the benchmark configurations are stored as JSON under
``data/`` (exported once from the reference's own ``build_pack`` by
``tools/export_pack.py``); ``phi_ref`` is per cell and supplied by the grid.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, replace
from typing import Tuple

import numpy as np

# liq table columns (rows: water then oils) — _kernels.py:48-51
LIQ_RHO_REF, LIQ_CP, LIQ_CT1, LIQ_CT2, LIQ_CPT = 0, 1, 2, 3, 4
LIQ_AVISC, LIQ_BVISC, LIQ_HVR, LIQ_EV, LIQ_TCRIT_F = 5, 6, 7, 8, 9
NLIQ = 10
# gas-capable table columns (rows: water, oils, gases) — _kernels.py:53-56
GASP_M, GASP_TCR, GASP_PC, GASP_AVG, GASP_BVG = 0, 1, 2, 3, 4
GASP_CPG1, GASP_CPG2, GASP_CPG3, GASP_CPG4 = 5, 6, 7, 8
NGASP = 9
# rock/solver scalars — _kernels.py:58-63
RK_CPOR, RK_CTPOR, RK_CPTPOR, RK_MODE = 0, 1, 2, 3
RK_CP1, RK_CP2, RK_COKE_CP, RK_RHO_COKE = 4, 5, 6, 7
RK_KTW, RK_KTO, RK_KTG, RK_KTR, RK_KTC = 8, 9, 10, 11, 12
RK_PREF, RK_TREF, RK_EPS_PER, RK_KROCW = 13, 14, 15, 16
NRK = 17

LAW_GAS_OIL, LAW_GAS_SOLID, LAW_CRACKING = 0, 1, 2  # _props.py:240-242

DATA_DIR = os.path.join(os.path.dirname(__file__), "data")


@dataclass(frozen=True)
class ModelPack:
    """Kernel-ready constants; mirrors assembly.py:42-81 field for field."""

    nco: int
    ncg: int
    heavy: int
    liq: np.ndarray
    gasp: np.ndarray
    kv: np.ndarray
    rockp: np.ndarray
    phi_ref: np.ndarray
    swt_s: np.ndarray
    swt_krw: np.ndarray
    swt_krow: np.ndarray
    swt_pcow: np.ndarray
    slt_s: np.ndarray
    slt_krg: np.ndarray
    slt_krog: np.ndarray
    slt_pcog: np.ndarray
    law_codes: np.ndarray
    rcoef: np.ndarray
    nmat: np.ndarray
    fuel_idx: np.ndarray
    ox_idx: np.ndarray
    ccmax: float
    names: Tuple[str, ...]

    @property
    def nfull(self) -> int:
        return 1 + self.nco + self.ncg

    @property
    def nequ(self) -> int:
        return self.nco + self.ncg + 5

    @property
    def row_energy(self) -> int:
        return 1 + self.nco + self.ncg

    @property
    def t_ref(self) -> float:
        return float(self.rockp[RK_TREF])


_FLOAT_FIELDS = ("liq", "gasp", "kv", "rockp", "swt_s", "swt_krw", "swt_krow",
                 "swt_pcow", "slt_s", "slt_krg", "slt_krog", "slt_pcog",
                 "rcoef", "nmat")
_INT_FIELDS = ("law_codes", "fuel_idx", "ox_idx")


def pack_to_dict(pack) -> dict:
    """Serialise any ModelPack-like object (reference or ours) to JSON data."""
    out = {"nco": int(pack.nco), "ncg": int(pack.ncg), "heavy": int(pack.heavy),
           "ccmax": float(pack.ccmax), "names": list(pack.names)}
    for f in _FLOAT_FIELDS:
        a = np.asarray(getattr(pack, f), dtype=np.float64)
        out[f] = {"shape": list(a.shape), "data": [float(v) for v in a.ravel()]}
    for f in _INT_FIELDS:
        a = np.asarray(getattr(pack, f), dtype=np.int64)
        out[f] = {"shape": list(a.shape), "data": [int(v) for v in a.ravel()]}
    return out


def pack_from_dict(d: dict, phi_ref: np.ndarray) -> ModelPack:
    kw = {}
    for f in _FLOAT_FIELDS:
        kw[f] = np.asarray(d[f]["data"], dtype=np.float64).reshape(d[f]["shape"])
    for f in _INT_FIELDS:
        kw[f] = np.asarray(d[f]["data"], dtype=np.int64).reshape(d[f]["shape"])
    ccmax = d["ccmax"]
    return ModelPack(
        nco=int(d["nco"]), ncg=int(d["ncg"]), heavy=int(d["heavy"]),
        phi_ref=np.ascontiguousarray(phi_ref, dtype=np.float64),
        ccmax=float(ccmax) if ccmax is not None else float("inf"),
        names=tuple(d["names"]), **kw)


def load_pack(name: str, phi_ref: np.ndarray) -> ModelPack:
    """Load a stored pack (``data/<name>.json``) bound to per-cell phi_ref."""
    with open(os.path.join(DATA_DIR, name + ".json"), encoding="utf-8") as fh:
        return pack_from_dict(json.load(fh), phi_ref)


def with_phi(pack: ModelPack, phi_ref: np.ndarray) -> ModelPack:
    return replace(pack, phi_ref=np.ascontiguousarray(phi_ref, dtype=np.float64))
