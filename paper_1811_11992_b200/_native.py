"""ctypes binding of the C-ABI in include/iscgpu.h.

The library is loaded from ``paper_1811_11992_b200/_lib/libiscgpu.so``
(built in-tree by ``paper_1811_11992_b200.build``). There is no fallback:
if the library or a CUDA device is missing every entry point raises
NativeLibraryMissing / RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (Breakdown, MaxIterations, NativeLibraryMissing, PoreSpaceExhausted,
                     SingularCellBlock)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libiscgpu.so")

ISC_OK, ISC_PSE, ISC_SINGULAR, ISC_BREAKDOWN, ISC_MAXIT = 0, 1, 2, 3, 4
PRECOND = {"none": 0, "bjacobi": 1, "ras": 2, "mcilu": 3}
KRYLOV = {"bicgstab": 0, "gmres": 1}
WELL_OUT = 32
NREC = 85

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
VP = ctypes.c_void_p


class ModelDesc(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int64) for f in ("nco", "ncg", "heavy", "nreac", "nswt", "nslt")]
                + [(f, VP) for f in ("liq", "gasp", "kv", "rockp", "swt_s", "swt_krw",
                                     "swt_krow", "swt_pcow", "slt_s", "slt_krg", "slt_krog",
                                     "slt_pcog", "law", "rcoef", "nmat", "fuel", "ox")]
                + [("ccmax", ctypes.c_double)])


class GridDesc(ctypes.Structure):
    _fields_ = ([("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32)]
                + [(f, VP) for f in ("depth", "volume", "phi_ref", "gd", "td", "conn_id",
                                     "hl_area")]
                + [(f, ctypes.c_double) for f in ("hl_kob", "hl_d", "hl_rho", "hl_tini")]
                + [("k_offset", ctypes.c_int32)])


class WellDesc(ctypes.Structure):
    _fields_ = [("cell", ctypes.c_int64), ("kind", ctypes.c_int32), ("control", ctypes.c_int32),
                ("target", ctypes.c_double), ("wi", ctypes.c_double), ("z_bh", ctypes.c_double),
                ("pinjmax", ctypes.c_double), ("heat_rate", ctypes.c_double),
                ("heat_stop", ctypes.c_double), ("s_yfull", ctypes.c_double * 5),
                ("s_yinj", ctypes.c_double * 2), ("s_tinj", ctypes.c_double),
                ("s_mu", ctypes.c_double), ("s_h", ctypes.c_double), ("s_mbar", ctypes.c_double)]


_SIGS = {
    "isc_create": (ctypes.c_int, [ctypes.POINTER(ModelDesc), ctypes.POINTER(GridDesc),
                                  ctypes.c_int32, ctypes.POINTER(WellDesc), ctypes.c_int32,
                                  ctypes.POINTER(VP)]),
    "isc_destroy": (ctypes.c_int, [VP]),
    "isc_last_error": (ctypes.c_char_p, []),
    "isc_block_size": (ctypes.c_int, []),
    "isc_assemble": (ctypes.c_int, [VP, VP, VP, VP, ctypes.c_double, ctypes.c_double, VP,
                                    ctypes.c_int32, VP, c_int64_p]),
    "isc_assemble_host": (ctypes.c_int, [VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, ctypes.c_double,
                                         ctypes.c_double, VP, ctypes.c_int32, VP, c_int64_p]),
    "isc_download_du": (ctypes.c_int, [VP, VP]),
    "isc_numeric_jacobian": (ctypes.c_int, [VP, VP, c_int64_p]),
    "isc_copy_out": (ctypes.c_int, [VP, ctypes.c_int32, VP]),
    "isc_export_system": (ctypes.c_int, [VP, VP, VP, VP]),
    "isc_import_system": (ctypes.c_int, [VP, VP, VP, VP, VP]),
    "isc_set_wells_out": (ctypes.c_int, [VP, VP]),
    "isc_set_precond": (ctypes.c_int, [VP, ctypes.c_int32]),
    "isc_set_krylov": (ctypes.c_int, [VP, ctypes.c_int32, ctypes.c_int32]),
    "isc_decoupled_form": (ctypes.c_int, [VP]),
    "isc_condensed": (ctypes.c_int, [VP]),
    "isc_synth_system": (ctypes.c_int, [VP, ctypes.c_uint64]),
    "isc_synth_system_slab": (ctypes.c_int, [VP, ctypes.c_uint64, ctypes.c_int32]),
    "isc_solve": (ctypes.c_int, [VP, ctypes.c_double, ctypes.c_int32, VP, VP,
                                 ctypes.POINTER(ctypes.c_int32), c_int64_p,
                                 ctypes.POINTER(ctypes.c_int32)]),
    "isc_solve_host": (ctypes.c_int, [VP, ctypes.c_double, ctypes.c_int32, VP, VP,
                                      ctypes.POINTER(ctypes.c_int32), c_int64_p,
                                      ctypes.POINTER(ctypes.c_int32)]),
    "isc_decouple": (ctypes.c_int, [VP, c_int64_p, ctypes.POINTER(ctypes.c_int32)]),
    "isc_precond_setup": (ctypes.c_int, [VP, c_int64_p]),
    "isc_spmv": (ctypes.c_int, [VP, VP, VP]),
    "isc_precond_apply": (ctypes.c_int, [VP, VP, VP]),
    "isc_copy_rhs": (ctypes.c_int, [VP, VP]),
    "isc_set_rhs": (ctypes.c_int, [VP, VP]),
    "isc_newton_update": (ctypes.c_int, [VP, VP, VP, ctypes.c_double]),
    "isc_scaled_norm": (ctypes.c_int, [VP, VP, ctypes.c_double, c_double_p]),
    "isc_audit_sums": (ctypes.c_int, [VP, VP, VP]),
    "isc_comm_nccl": (ctypes.c_int, [VP, VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "isc_nccl_unique_id": (ctypes.c_int, [VP]),
    "isc_comm_is_nccl": (ctypes.c_int, [VP]),
    "isc_hub_create": (VP, [ctypes.c_int32]),
    "isc_hub_destroy": (ctypes.c_int, [VP]),
    "isc_comm_hub": (ctypes.c_int, [VP, VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.c_int32, ctypes.c_int32]),
    "isc_comm_allreduce_host": (ctypes.c_int, [VP, VP, ctypes.c_int32, ctypes.c_int32]),
    "isc_stream": (VP, [VP]),
    "isc_set_stream": (ctypes.c_int, [VP, VP]),
    "isc_synchronize": (ctypes.c_int, [VP]),
    "isc_launch_count": (ctypes.c_int64, [VP]),
    "isc_stage_times": (ctypes.c_int, [VP, VP]),
    "isc_set_profiling": (ctypes.c_int, [VP, ctypes.c_int32]),
    "isc_kernel_times": (ctypes.c_int, [VP, VP, VP, ctypes.c_int32]),
    "isc_format_double": (ctypes.c_int, [ctypes.c_double, ctypes.c_char_p]),
    "isc_format_cells": (ctypes.c_int, [ctypes.c_double, ctypes.c_int64, VP, VP, VP, VP, VP,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, VP,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, VP,
                                        ctypes.c_int32, VP, c_int64_p]),
    "isc_free": (None, [VP]),
}

_lib = None


def lib():
    """Load the sm_100a library (raises NativeLibraryMissing, never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is not built; run `python -m paper_1811_11992_b200.build`")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover
        raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols():
    return sorted(_SIGS)


def last_error() -> str:
    return lib().isc_last_error().decode(errors="replace")


def check(status: int, what: str = "", bad_cell=None, bad_col=None):
    """Map a C status to the reference's exception classes (errors.py:43-88)."""
    if status == ISC_OK:
        return
    msg = last_error()
    if status == ISC_PSE:
        raise PoreSpaceExhausted(f"coke fills the pore volume in cell {bad_cell}")
    if status == ISC_SINGULAR:
        if bad_cell is not None and bad_cell >= 0:
            raise SingularCellBlock(
                f"diagonal block of cell {bad_cell} is singular at column {bad_col}")
        raise SingularCellBlock(msg or what)
    if status == ISC_BREAKDOWN:
        raise Breakdown(msg)
    if status == ISC_MAXIT:
        raise MaxIterations(msg)
    raise RuntimeError(f"{what}: iscgpu status {status}: {msg}")


def ptr(a) -> VP:
    """Device or host data pointer of a torch tensor / numpy array."""
    if a is None:
        return VP(0)
    if isinstance(a, np.ndarray):
        return VP(a.ctypes.data)
    return VP(a.data_ptr())
