"""Report frames (report.py:50-149): the native cells.csv
formatter against the reference writer's own bytes (tests/golden/
report_frames.npz, made by running iscsim.report.write_frame) and against
Python's repr. Host-only code in the library: runs without a GPU."""

import os

import numpy as np
import pytest

from paper_1811_11992_b200.report import (ReportFrame, ReportSink, format_cells, format_float,
                                          write_frame)
from tests.helpers import golden


def _frame(g, k):
    oil, vap, wells = (tuple(s.split("|")) if s else () for s in g[k + "names"])
    return ReportFrame(time=float(g[k + "time"]), p=g[k + "p"], t=g[k + "t"], sw=g[k + "sw"],
                       so=g[k + "so"], sg=g[k + "sg"], x=g[k + "x"], y=g[k + "y"], cc=g[k + "cc"],
                       oil_names=oil, vap_names=vap, well_names=wells, bhp=g[k + "bhp"],
                       rates=g[k + "rates"], cum=g[k + "cum"])


def test_frames_byte_identical_with_reference_writer(tmp_path):
    g = golden("report_frames.npz")
    with ReportSink(str(tmp_path)) as sink:
        write_frame(_frame(g, "f1_"), sink)
        write_frame(_frame(g, "f2_"), sink)
    for name in ("cells", "wells"):
        got = (tmp_path / f"{name}.csv").read_bytes()
        assert got == bytes(g[name + "_csv"]), name


def test_repr_of_random_doubles():
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2 ** 63, size=40000, dtype=np.uint64)
    vals = np.concatenate([bits.view(np.float64), -bits[:5000].view(np.float64),
                           rng.normal(size=20000) * 10.0 ** rng.integers(-30, 30, 20000)])
    for v in vals:
        assert format_float(v) == repr(float(v))


def test_threaded_rows_are_ordered():
    g = golden("report_frames.npz")
    f = _frame(g, "f1_")
    one = format_cells(f, threads=1)
    many = format_cells(f, threads=16)
    assert one == many
    ref = "".join(",".join([repr(float(f.time)), str(c)] + [repr(float(v)) for v in (
        f.p[c], f.t[c], f.sw[c], 1.0 - f.sw[c] - f.sg[c], f.sg[c], *f.x[c], *f.y[c], f.cc[c])])
        + "\n" for c in range(f.p.shape[0]))
    assert one == ref.encode()
