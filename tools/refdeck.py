"""Reference-side harness (runs only where /root/reference exists).

Turns one of our ``configs.Case`` objects into a deck for the reference
simulator ``iscsim``: the fluid, rock-property and relperm sections come
from the reference's own ``decks/tube.deck`` with the light-oil oxidation
reaction removed; grid, per-cell permeability, init, wells, schedule and
solver sections are written from the Case. Per-cell porosity cannot be
expressed in a deck (deck.py:424-429, grid.py:78), so ``run_reference``
patches ``grid.phi_ref`` the way SURVEY Appendix B.3 describes.

Used by tools/export_pack.py and tests/golden/make_golden.py; never by the
product, the GPU tests, smoke() or bench.py.
"""

from __future__ import annotations

import os
import re
import sys
from typing import Dict, List

import numpy as np

REF_SRC = "/root/reference/pkg/src"
TUBE_DECK = "/root/reference/pkg/decks/tube.deck"


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_iscgpu")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import iscsim  # noqa: F401
    import iscsim.newton  # noqa: F401
    return iscsim


def _sections(text: str) -> Dict[str, List[List[str]]]:
    """Section name -> list of sections (each a list of raw body lines)."""
    out: Dict[str, List[List[str]]] = {}
    cur = None
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].rstrip()
        if not line.strip():
            continue
        if line.startswith("*"):
            cur = []
            out.setdefault(line[1:].strip(), []).append(cur)
        elif cur is not None:
            cur.append(line.strip())
    return out


def _drop_light_oil_oxidation(lines: List[str]) -> List[str]:
    """Remove the RATE block whose STOICH consumes LO with O2 (gas-oil law)."""
    blocks, head = [], []
    for ln in lines:
        if ln.startswith("RATE"):
            blocks.append([ln])
        elif blocks:
            blocks[-1].append(ln)
        else:
            head.append(ln)
    keep = []
    for b in blocks:
        toks = [ln.split() for ln in b]
        is_gas_oil = any(t[0] == "LAW" and t[1] == "gas-oil" for t in toks)
        eats_lo = any(t[0] == "STOICH" and t[1] == "LO" and float(t[2]) < 0 for t in toks)
        if is_gas_oil and eats_lo:
            continue
        keep.extend(b)
    tail = [ln for ln in head]
    # CCMAX / TOL rows live after the last block in tube.deck: they were
    # appended to the last block above; nothing else to restore.
    return tail + keep


def _fmt(v) -> str:
    return repr(float(v))


def case_to_deck(case) -> str:
    from paper_1811_11992_b200.wells import WellSpec  # noqa: F401

    tube = _sections(open(TUBE_DECK, encoding="utf-8").read())
    kx, ky, kz, _phi = case.rock_arrays()
    out = ["*GRID", f"NX {case.nx}", f"NY {case.ny}", f"NZ {case.nz}",
           f"DX {_fmt(case.d[0])}", f"DY {_fmt(case.d[1])}", f"DZ {_fmt(case.d[2])}",
           "DEPTH_TOP 0.0", ""]
    out.append("*ROCK")
    for key, arr in (("PERMX", kx), ("PERMY", ky), ("PERMZ", kz)):
        if np.all(arr == arr[0]):
            out.append(f"{key} {_fmt(arr[0])}")
        else:
            out.append(key + " " + " ".join(_fmt(v) for v in arr))
    out.append("POROSITY 0.3")
    for ln in tube["ROCK"][0]:
        if ln.split()[0] not in ("PERMX", "PERMY", "PERMZ", "POROSITY", "HEATLOSS"):
            out.append(ln)
    hl = getattr(case, "heat_loss", None)
    if hl is not None:
        out.append(f"HEATLOSS {_fmt(hl.k_ob)} {_fmt(hl.distance)} {_fmt(hl.rho)} "
                   f"{_fmt(hl.t_initial)}")
    out.append("")
    for sec in ("COMPONENTS", "KVALUES", "DENSITY", "VISCOSITY", "ENTHALPY"):
        out.append("*" + sec)
        out.extend(tube[sec][0])
        out.append("")
    out.append("*REACTIONS")
    out.extend(_drop_light_oil_oxidation(tube["REACTIONS"][0]))
    out.append("")
    for sec in ("RELPERM-SWT", "RELPERM-SLT"):
        out.append("*" + sec)
        out.extend(tube[sec][0])
        out.append("")
    ini = case.init
    out += ["*INIT", f"PRES {_fmt(ini.p)}", f"TEMP {_fmt(ini.t)}", f"SW {_fmt(ini.s_w)}",
            f"SO {_fmt(1.0 - ini.s_w - ini.s_g)}", f"SG {_fmt(ini.s_g)}",
            "XOIL " + " ".join(_fmt(v) for v in ini.x),
            "YGAS " + " ".join(_fmt(v) for v in ini.y), f"CC {_fmt(ini.c_c)}", ""]
    for w in case.wells:
        out += ["*WELL", f"NAME {w.name}", f"TYPE {w.kind}", f"CELL {w.i} {w.j} {w.k}"]
        if w.wi is not None:
            out.append(f"WI {_fmt(w.wi)}")
        else:
            out.append(f"RADIUS {_fmt(w.radius)}")
            out.append(f"SKIN {_fmt(w.skin)}")
        if w.control == "bhp":
            out.append(f"BHP {_fmt(w.bhp)}")
        elif w.control == "rate_gas":
            out.append(f"RATE {_fmt(w.rate)}")
            out.append(f"RATE_CONDITIONS {w.rate_conditions}")
        else:
            out.append(f"RATE_TOTAL {_fmt(w.rate)}")
        if w.yinj:
            out.append("YINJ " + " ".join(_fmt(v) for v in w.yinj))
        if w.tinj is not None:
            out.append(f"TINJ {_fmt(w.tinj)}")
        if w.pinjmax is not None:
            out.append(f"PINJMAX {_fmt(w.pinjmax)}")
        if w.heat_rate:
            out.append(f"HEAT_RATE {_fmt(w.heat_rate)}")
            out.append(f"HEAT_STOP {_fmt(w.heat_stop)}")
        out.append("")
    s = case.schedule
    out += ["*SCHEDULE", f"END {_fmt(s.t_end)}"]
    if s.report_interval:
        out.append(f"REPORT_INTERVAL {_fmt(s.report_interval)}")
    out += [f"DTINIT {_fmt(s.dt_init)}", f"DTMIN {_fmt(s.dt_min)}", f"DTMAX {_fmt(s.dt_max)}", ""]
    v = case.solver
    out += ["*SOLVER", f"NEWTON_TOL {_fmt(v.newton_tol)}", f"NEWTON_MAX {v.newton_max}",
            f"LINEAR_TOL {_fmt(v.linear_tol)}", f"LINEAR_MAX {v.linear_max}", "THREADS 1",
            f"PRECOND {v.precond}", f"EPS {_fmt(v.eps)}", "JACOBIAN analytic", ""]
    return "\n".join(out)


def reference_simulator(case, threads: int = 1, jacobian=None):
    """Reference ``Simulator`` for a case with the per-cell porosity patch."""
    import_reference()
    import iscsim.newton as nw
    from iscsim.deck import parse_deck

    deck = parse_deck(case_to_deck(case))
    _kx, _ky, _kz, phi = case.rock_arrays()
    orig = nw.build_grid

    def patched(spec, rock):
        g = orig(spec, rock)
        g.phi_ref[:] = phi
        return g

    nw.build_grid = patched
    try:
        sim = nw.Simulator(deck, threads=threads, jacobian=jacobian)
    finally:
        nw.build_grid = orig
    return sim
