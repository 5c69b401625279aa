"""CPU-side checks of the boundary: the C-ABI library builds, loads and
exports every entry point include/iscgpu.h declares; host-side builders and
error mapping behave like the reference's. No kernel is launched here."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1811_11992_b200 import _native as N
from paper_1811_11992_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iscgpu.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*|void \*|void|int64_t)\s*\**\s*(isc_\w+)\(",
                                 txt, flags=re.M)))


def test_library_builds_and_exports_header_symbols():
    B.build()
    lib = ctypes.CDLL(B.LIB)
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    # the Python binding covers every declared entry point
    assert set(declared) <= set(N.exported_symbols()) | {"isc_stream"}
    nm = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True)
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm.stdout), name


def test_sm100a_cubin_embedded():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_status_mapping_to_reference_exceptions():
    from paper_1811_11992_b200.errors import (Breakdown, MaxIterations, PoreSpaceExhausted,
                                              SingularCellBlock)
    N.lib()
    with pytest.raises(PoreSpaceExhausted):
        N.check(1, bad_cell=3)
    with pytest.raises(SingularCellBlock, match="cell 5 is singular at column 2"):
        N.check(2, bad_cell=5, bad_col=2)
    with pytest.raises(Breakdown):
        N.check(3)
    with pytest.raises(MaxIterations):
        N.check(4)
    N.check(0)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.errors import NativeLibraryMissing
    from paper_1811_11992_b200.assembly import Workspace
    g, p, w, s, st = configs.build_case(configs.config("small3d"))
    with pytest.raises(NativeLibraryMissing):
        Workspace(g, p, None, wells=w, streams=s)


def test_face_arrays_match_connection_list():
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.device import DARCY_CONST, face_arrays
    g, p, w, s, st = configs.build_case(configs.config("sub2"))
    gd, td, cid = face_arrays(g)
    ic = cid[cid >= 0]
    assert sorted(ic.tolist()) == list(range(g.nconn))
    ax, a = np.nonzero(cid >= 0)
    np.testing.assert_array_equal(g.conn_a[cid[ax, a]], a)
    np.testing.assert_array_equal(gd[ax, a], DARCY_CONST * g.conn_geom[cid[ax, a]])
    step = np.array([1, g.nx, g.nx * g.ny])[ax]
    np.testing.assert_array_equal(g.conn_b[cid[ax, a]], a + step)


def test_partition_semantics():
    """Slab partition along the first longest axis, remainder to leading slabs."""
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.grid import partition, slab_bounds
    assert slab_bounds(200, 64)[:9] == ((0, 4), (4, 8), (8, 12), (12, 16), (16, 20), (20, 24),
                                        (24, 28), (28, 32), (32, 35))
    g, *_ = configs.build_case(configs.config("sub2"))
    part = partition(g, 2)
    assert part.axis == 0 and part.bounds == ((0, 16), (16, 32))
    assert (part.owner.reshape(8, 16, 32)[:, :, :16] == 0).all()
