"""Shared test helpers: golden fixtures and seeded cases (no reference needed)."""

import os
from dataclasses import replace
from types import SimpleNamespace

import numpy as np

from paper_1811_11992_b200 import configs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def case_objects(name, **solver_overrides):
    case = configs.config(name)
    if solver_overrides:
        case = replace(case, solver=replace(case.solver, **solver_overrides))
    grid, pack, wells, streams, state = configs.build_case(case)
    return SimpleNamespace(case=case, grid=grid, pack=pack, wells=wells, streams=streams,
                           state=state)


def state_from(g, prefix="st_"):
    return configs.InitialState(*(np.array(g[prefix + f]) for f in
                                  ("p", "t", "sw", "sg", "x", "y", "cc", "bhp")))


def row_scaled_err(a, b):
    """max |a-b| / max(|b|, max|b| over the block row), rows = last-but-one axis."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    rowmax = np.max(np.abs(b), axis=-1, keepdims=True)
    scale = np.maximum(np.abs(b), rowmax)
    scale = np.where(scale == 0.0, 1.0, scale)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def scaled_resid_err(a, b, accn, volume, dt, row_os, row_gs):
    """Residual difference in the scaled_norm metric (newton.py:124-144)."""
    scale = (volume / dt)[:, None] * np.maximum(1.0, np.abs(accn))
    scale[:, row_os] = 1.0
    scale[:, row_gs] = 1.0
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / scale))
