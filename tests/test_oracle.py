"""Pin the CPU oracle to the reference (CPU only, no GPU).

The oracle (oracle/isc_oracle.{c,py}) is the checker for every GPU parity
test, so it is itself checked against:
  * the reference's own 31 scalar property goldens (pkg/tests/goldens.py);
  * fixtures produced by running the reference in this container
    (tests/golden/make_golden.py): cell-pass outputs, the assembled system,
    well blocks, decoupled BiCGSTAB solutions for every preconditioner, a
    2-subdomain RAS case, the synthetic microbench and full C1/C2 runs.
Our grid/pack/well builders feed the oracle, so these tests also pin the
product's host-side builders bit for bit.
"""

import copy
import ctypes
import json
import math
import os

from dataclasses import replace

import numpy as np
import pytest

from oracle import isc_oracle as O
from paper_1811_11992_b200 import wells as W
from paper_1811_11992_b200.synth import synth_system
from tests.helpers import GOLDEN, case_objects, golden, state_from

KV = {"H2O": (1.7202e6, 0.0, 0.0, -6869.59, -376.64),
      "LO": (1.4546e5, 0.0, 0.0, -4458.73, -387.78),
      "HO": (2.7454e5, 0.0, 0.0, -8424.83, -205.69)}
CPG = {"H2O": (7.613, 8.616e-4, 0.0, 0.0), "LO": (-1.89, 0.1275, -3.9e-5, 4.6e-9),
       "HO": (-8.14, 0.549, -1.68e-4, 1.98e-8), "O2": (6.713, -4.883e-7, 1.287e-6, -4.36e-10),
       "IR": (7.44, -0.0018, 1.975e-6, -4.78e-10)}
M = {"H2O": 18.0, "LO": 156.7, "HO": 675.0, "O2": 32.0, "IR": 40.8}
GVISC = {"H2O": (8.822e-6, 1.116), "LO": (2.166e-6, 0.943), "HO": (3.926e-6, 1.102),
         "O2": (2.196e-4, 0.721), "IR": (2.127e-4, 0.702)}
MIX = ("H2O", "LO", "HO", "O2", "IR")
MIX_Y = (0.05, 0.02, 0.01, 0.20, 0.72)


def _arr(*v):
    return np.asarray(v, dtype=np.float64)


def _call(fn, *args, nout=3):
    out = np.zeros(nout)
    conv = []
    for a in args:
        if isinstance(a, np.ndarray):
            conv.append(a.ctypes.data_as(ctypes.c_void_p))
        elif isinstance(a, int):
            conv.append(ctypes.c_int64(a))
        else:
            conv.append(ctypes.c_double(a))
    getattr(O.lib(), fn)(*conv, out.ctypes.data_as(ctypes.c_void_p))
    return out


def _kval(name, p, t):
    return _call("orc_props_k_value", _arr(*KV[name]), p, t)[0]


def _rho_liq(c, p, t):
    return _call("orc_props_liquid_density", _arr(*c, 14.7, 77.0), p, t)[0]


def _h(name, t):
    return _call("orc_props_gas_enthalpy", _arr(*CPG[name]), 77.0, t, nout=2)[0]


def _hv(hvr, ev, tc, t):
    return _call("orc_props_vaporization_enthalpy", hvr, ev, tc, t, nout=2)[0]


def _z(ys, tc_f, pc, p, t):
    z, _, _, _ = O.z_factor_mix(np.asarray(ys), np.asarray(tc_f) + 459.67, np.asarray(pc), p, t)
    return z


def _props_values():
    v = {}
    v["k_w_2014_100"] = _kval("H2O", 2014.7, 100.0)
    v["k_lo_500_300"] = _kval("LO", 500.0, 300.0)
    v["k_ho_500_300"] = _kval("HO", 500.0, 300.0)
    v["k_allterms_800_250"] = _call("orc_props_k_value", _arr(1e3, 1e-2, 0.5, -4000.0, -300.0),
                                    800.0, 250.0)[0]
    v["z_o2_65_200"] = _z([1.0], [-181.77], [730.0], 65.0, 200.0)
    zt = _z([0.21, 0.79], [-181.0, -232.0], [730.0, 500.0], 2014.7, 100.0)
    v["z_tubegas_2014_100"] = zt
    v["rho_g_tube_init"] = 2014.7 / (zt * 10.7316 * (100.0 + 459.67))
    v["rho_w_tube_2514_150"] = _rho_liq((3.466, 3e-6, 1.2e-4, 0.0, 0.0), 2514.7, 150.0)
    rlo = _rho_liq((0.3195, 5e-6, 2.839e-4, 0.0, 0.0), 2014.7, 100.0)
    rho = _rho_liq((0.0914, 5e-6, 1.496e-4, 0.0, 0.0), 2014.7, 100.0)
    v["rho_lo_tube_init"], v["rho_ho_tube_init"] = rlo, rho
    v["rho_o_tube_init"] = 1.0 / (0.744 / rlo + 0.256 / rho)
    v["mu_w_100"] = _call("orc_props_liquid_viscosity", 4.7352e-3, 2728.2, 100.0, nout=2)[0]
    mlo = _call("orc_props_liquid_viscosity", 4.02e-4, 6121.6, 200.0, nout=2)[0]
    v["mu_o_tube_200"] = math.exp(0.3 * math.log(mlo) + 0.7 * math.log(mlo))
    mus = [_call("orc_props_gas_component_viscosity", *GVISC[c], 300.0, nout=2)[0] for c in MIX]
    sq = [math.sqrt(M[c]) for c in MIX]
    v["mu_g_tube_300"] = (sum(y * m * s for y, m, s in zip(MIX_Y, mus, sq))
                          / sum(y * s for y, s in zip(MIX_Y, sq)))
    v["h_gw_177"] = _h("H2O", 177.0)
    v["h_g_tube_400"] = sum(y * _h(c, 400.0) for y, c in zip(MIX_Y, MIX))
    v["hvap_ho_300"] = _hv(12198.0, 0.38, 1138.0, 300.0)
    v["h_o_tube_300"] = (0.744 * (_h("LO", 300.0) - _hv(1917.0, 0.38, 651.7, 300.0))
                         + 0.256 * (_h("HO", 300.0) - _hv(12198.0, 0.38, 1138.0, 300.0)))
    v["u_coke_177"] = 4.06 * (177.0 - 77.0)
    v["u_rock_tube_300"] = 35.0 * (300.0 - 77.0)
    hw = _h("H2O", 100.0) - _hv(1657.0, 0.38, 705.7, 100.0)
    v["u_w_tube_init"] = hw - 2014.7 / _rho_liq((3.466, 3e-6, 1.2e-4, 0.0, 0.0), 2014.7, 100.0)
    por = lambda mode: _call("orc_props_porosity", _arr(0.4142, 5e-6, 0.0, 0.0, 14.7, 77.0),
                             mode, 2064.7, 100.0)[0]
    v["phi_tube_linear"] = por(0)
    v["phi_tube_nonlinear"] = por(1)
    v["phif_tube_linear"] = por(0) - 0.05 / 57.2
    v["arr_tube_r4_600"] = _call("orc_props_arrhenius", 1.00008e4, 25200.0, 600.0, nout=2)[0]
    v["arr_tube_r1_500"] = _call("orc_props_arrhenius", 7.248e11, 59450.0, 500.0, nout=2)[0]
    v["stone2_spec"] = _call("orc_props_stone2", _arr(1.0, 0.5, 0.1, 0.4, 0.2), nout=5)[0]
    v["re_iso_16_4"] = W.equivalent_radius(16.4, 16.4, 1.0, 1.0)
    v["wi_field_inj"] = W.well_index(16.4, 16.42857142857143, 7.0, 4000.0, 4000.0, 0.5, 0.0)
    v["molar_rate_tube_inj"] = W.gas_rate_to_molar(0.554)
    v["molar_rate_field_inj"] = W.gas_rate_to_molar(115000.0)
    return v


def test_property_goldens():
    """The reference's 31 scalar goldens; its oracle uses independent routes
    (bisection cubic root, adaptive Simpson), hence 1e-10 relative."""
    gold = json.load(open(os.path.join(GOLDEN, "props_goldens.json")))["goldens"]
    vals = _props_values()
    assert set(vals) == set(gold)
    for k, g in gold.items():
        assert abs(vals[k] - g) <= 1e-10 * max(1.0, abs(g)), (k, vals[k], g)


def test_cubic_root_branches():
    """Both Cardano branches polish to a machine-level residual (_props.py:68-104)."""
    for a, b in ((0.5, 0.05), (0.05, 0.01), (1e-4, 1e-5), (2.0, 0.2)):
        z = O.lib().orc_cubic_largest_root(ctypes.c_double(a), ctypes.c_double(b))
        g = z ** 3 - z ** 2 + (a - b - b * b) * z - a * b
        assert abs(g) < 1e-13
        roots = np.roots([1.0, -1.0, a - b - b * b, -a * b])
        assert abs(z - max(r.real for r in roots if abs(r.imag) < 1e-9)) < 1e-10


def _oracle_assemble(c, st, accn, dt, t_new, capped, freeze=False, ws=None):
    model = O.Model(c.pack)
    ws = ws or O.Workspace(c.grid, c.pack)
    blocks = O.assemble(c.grid, model, ws, c.wells, c.streams, st, accn, dt, t_new, capped,
                        freeze_upwind=freeze)
    return ws, blocks


def test_assembly_bitexact_vs_reference():
    """cell_pass / compose / conn / gather / wells reproduce the reference bit for bit."""
    g = golden("asm_small3d.npz")
    c = case_objects("small3d")
    st = state_from(g)
    ws, blocks = _oracle_assemble(c, st, g["accn"], float(g["dt"]), float(g["t_new"]),
                                  g["capped"])
    for f in ("pot", "dpot", "beta", "dbeta", "hph", "dhph", "yfull", "dyfull", "gam", "dgam",
              "pcv", "dpcv", "kr3", "dkr3", "ktd", "acc", "dacc", "src", "dsrc", "resid",
              "diag", "offd", "upw"):
        np.testing.assert_array_equal(getattr(ws, f), g[f], err_msg=f)
    for k in ("resid", "dwdb"):
        np.testing.assert_array_equal([getattr(b, k) for b in blocks], g["w_" + k])
    for k in ("wrow", "bcol", "phase_rates", "comp_rates"):
        np.testing.assert_array_equal(np.stack([getattr(b, k) for b in blocks]), g["w_" + k])
    # frozen upwinding at a second state reuses the stored flags
    st2 = state_from(g, "st2_")
    ws, blocks2 = _oracle_assemble(c, st2, g["accn2"], float(g["dt"]), float(g["t_new"]),
                                   g["capped"], freeze=True, ws=ws)
    for f in ("resid", "diag", "offd"):
        np.testing.assert_array_equal(getattr(ws, f), g[f + "2"], err_msg=f)


def test_numeric_jacobian_bitexact_vs_reference():
    """The finite-difference Jacobian (assembly.py:843-939) — probes, one-sided
    steps at the box edges, neighbour rows, well wrow/bcol/dwdb — and
    check_jacobian (942-982) reproduce the reference bit for bit."""
    g = golden("asm_small3d.npz")
    gn = golden("numjac_small3d.npz")
    c = case_objects("small3d")
    model = O.Model(c.pack)
    ws = O.Workspace(c.grid, c.pack)
    dt, t_new = float(g["dt"]), float(g["t_new"])
    st = state_from(g)
    blocks = O.assemble(c.grid, model, ws, c.wells, c.streams, st, g["accn"], dt, t_new,
                        g["capped"], jacobian="numeric")
    for f in ("resid", "diag", "offd", "upw"):
        np.testing.assert_array_equal(getattr(ws, f), gn[f], err_msg=f)
    for k in ("resid", "dwdb"):
        np.testing.assert_array_equal([getattr(b, k) for b in blocks], gn["w_" + k])
    for k in ("wrow", "bcol"):
        np.testing.assert_array_equal(np.stack([getattr(b, k) for b in blocks]), gn["w_" + k])
    st2 = state_from(g, "st2_")
    blocks2 = O.assemble(c.grid, model, ws, c.wells, c.streams, st2, g["accn2"], dt, t_new,
                         g["capped"], jacobian="numeric", freeze_upwind=True)
    for f in ("resid", "diag", "offd"):
        np.testing.assert_array_equal(getattr(ws, f), gn[f + "2"], err_msg=f)
    for k in ("wrow", "bcol"):
        np.testing.assert_array_equal(np.stack([getattr(b, k) for b in blocks2]),
                                      gn["w2_" + k])
    worst = O.check_jacobian(c.grid, model, O.Workspace(c.grid, c.pack), c.wells, c.streams,
                             st, g["accn"], dt, t_new, g["capped"])
    assert worst == float(gn["check"])


@pytest.mark.parametrize("precond", ["none", "bjacobi", "ras"])
def test_solve_bitexact_vs_reference(precond):
    g = golden("asm_small3d.npz")
    s = golden("solve_small3d.npz")
    c = case_objects("small3d")
    ws, blocks = _oracle_assemble(c, state_from(g), g["accn"], float(g["dt"]),
                                  float(g["t_new"]), g["capped"])
    du, dbhp, it = O.BlockSolver(c.grid, ws, tol=1e-10, maxiter=1000,
                                 precond=precond).solve(blocks)
    assert it == int(s[precond + "_iters"])
    np.testing.assert_array_equal(du, s[precond + "_du"])
    np.testing.assert_array_equal(dbhp, s[precond + "_dbhp"])


def test_two_subdomain_ras_vs_reference():
    """32x16x8: two x-slab subdomains, RAS halos (linsolve.py:338-358)."""
    from tests.golden_states import random_state_like_reference
    s = golden("solve_sub2.npz")
    c = case_objects("sub2")
    st, accn = random_state_like_reference(c, int(s["seed"]))
    ws, blocks = _oracle_assemble(c, st, accn, 2e-3, 2e-3, np.zeros(len(c.wells), bool))
    np.testing.assert_array_equal(np.abs(ws.resid).max(axis=0), s["resid_absmax"])
    for pc in ("none", "bjacobi", "ras"):
        d0, o0 = ws.diag.copy(), ws.offd.copy()
        du, dbhp, it = O.BlockSolver(c.grid, ws, tol=1e-10, maxiter=1000,
                                     precond=pc).solve(blocks)
        ws.diag[:], ws.offd[:] = d0, o0
        assert it == int(s[pc + "_iters"]), pc
        if pc == "ras":
            np.testing.assert_array_equal(du, s["ras_du"])
            np.testing.assert_array_equal(dbhp, s["ras_dbhp"])


def test_synthetic_microbench_vs_reference():
    from paper_1811_11992_b200.grid import build_grid
    from types import SimpleNamespace
    s = golden("synth_16.npz")
    grid = build_grid(16, 16, 16, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    diag, offd, resid = synth_system(grid, 9, seed=7)
    np.testing.assert_array_equal(diag[:3], s["diag_probe"])
    np.testing.assert_array_equal(offd[:3], s["offd_probe"])
    ws = O.Workspace(grid, SimpleNamespace(nequ=9, nfull=5))
    for pc in ("none", "bjacobi", "ras"):
        ws.diag, ws.offd, ws.resid = diag.copy(), offd.copy(), resid
        du, _, it = O.BlockSolver(grid, ws, tol=1e-8, maxiter=1000, precond=pc).solve([])
        assert it == int(s[pc + "_iters"]), pc
        if pc == "ras":
            np.testing.assert_array_equal(du, s["ras_du"])


def test_numeric_jacobian_run_prefix_vs_reference():
    """JACOBIAN numeric mode (newton.py:228,278): the first 4 steps of the
    reference's C1 run reproduced exactly (the Python-driven FD oracle is too
    slow for the whole run here; the GPU test runs all 50 steps)."""
    g = golden("traj_c1_1e-10_numeric.npz")
    c = case_objects("c1", linear_tol=1e-10)
    k = 4
    sched = replace(c.case.schedule, t_end=float(g["steps"][k - 1, 0]))
    sim = O.Simulator(c.grid, c.pack, c.wells, c.streams, c.state, sched, c.case.solver,
                      jacobian="numeric")
    sim.advance()
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves) for s in sim.steps])
    np.testing.assert_array_equal(rec, g["steps"][:k, :5])


@pytest.mark.parametrize("name,tol", [("c1", 1e-10), ("c1", 1e-5), ("c2", 1e-10),
                                      ("c2hl", 1e-10), ("c2cap", 1e-10), ("c2rate", 1e-10)])
def test_trajectory_vs_reference(name, tol):
    """Whole runs: step/Newton/linear sequences equal, fields bit-identical
    (c2hl: overburden heat loss, _kernels.py:821-825; c2cap: injector capped
    and released, newton.py:147-168, assembly.py:515-516, with Newton-limit
    step cuts; c2rate: total-rate producer, assembly.py:518-520)."""
    g = golden(f"traj_{name}_{tol:.0e}.npz")
    c = case_objects(name, linear_tol=tol)
    sim = O.Simulator(c.grid, c.pack, c.wells, c.streams, c.state, c.case.schedule,
                      c.case.solver, heat_loss=c.case.heat_loss)
    sim.advance()
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves, s.balance)
                    for s in sim.steps])
    np.testing.assert_array_equal(rec[:, :5], g["steps"][:, :5])
    np.testing.assert_allclose(rec[:, 5], g["steps"][:, 5], rtol=0, atol=1e-12)
    for f in ("p", "t", "sw", "sg", "x", "y", "cc", "bhp"):
        np.testing.assert_array_equal(getattr(sim.state, f), g["final_" + f], err_msg=f)


@pytest.mark.parametrize("name", sorted(__import__("tests.golden_states", fromlist=["x"])
                                        .BREAKDOWN_CASES))
def test_bicgstab_restart_and_breakdown_vs_reference(name):
    """BiCGSTAB's single restart and its Breakdown exits (linsolve.py:497-575)
    on the constructed 2-cell systems: same iteration count and solution, or
    the same Breakdown message, as the reference (bicgstab_breakdown.npz)."""
    from types import SimpleNamespace
    from paper_1811_11992_b200.grid import build_grid
    from tests.golden_states import BREAKDOWN_CASES, breakdown_system
    g = golden("bicgstab_breakdown.npz")
    grid = build_grid(2, 1, 1, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    diag, offd, resid = breakdown_system(BREAKDOWN_CASES[name])
    ws = O.Workspace(grid, SimpleNamespace(nequ=9, nfull=5))
    ws.diag, ws.offd, ws.resid = diag, offd, resid
    status = str(g[name + "_status"])
    if status == "ok":
        du, _, it = O.BlockSolver(grid, ws, tol=1e-10, maxiter=50, precond="none").solve([])
        assert it == int(g[name + "_iters"])
        np.testing.assert_array_equal(du, g[name + "_du"])
    else:
        with pytest.raises(O.Breakdown) as exc:
            O.BlockSolver(grid, ws, tol=1e-10, maxiter=50, precond="none").solve([])
        assert "Breakdown: " + str(exc.value) == status


@pytest.mark.parametrize("nx", [4, 5])
def test_oracle_mcilu_is_red_black_ilu0(nx):
    """The oracle's multicolour block ILU(0) (checker for the device's mcilu)
    equals the red-black block ILU(0) computed densely."""
    from paper_1811_11992_b200.grid import build_grid
    from types import SimpleNamespace
    grid = build_grid(nx, 3, 3, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    n = grid.ncell
    diag, offd, _ = synth_system(grid, 9, seed=5)
    # decoupled system: identity diagonal blocks, D^-1 B off the diagonal
    inv = np.linalg.inv(diag)
    a, b = grid.conn_a, grid.conn_b
    off = np.stack([inv[a] @ offd[:, 0], inv[b] @ offd[:, 1]], axis=1)
    ws = O.Workspace(grid, SimpleNamespace(nequ=9, nfull=5))
    ws.offd = off
    bs = O.BlockSolver(grid, ws, precond="mcilu")
    bs._factor()
    A = np.zeros((9 * n, 9 * n))
    for c in range(n):
        A[9 * c:9 * c + 9, 9 * c:9 * c + 9] = np.eye(9)
    for ic in range(grid.nconn):
        A[9 * a[ic]:9 * a[ic] + 9, 9 * b[ic]:9 * b[ic] + 9] = off[ic, 0]
        A[9 * b[ic]:9 * b[ic] + 9, 9 * a[ic]:9 * a[ic] + 9] = off[ic, 1]
    red = np.flatnonzero(~bs.black)
    blk = np.flatnonzero(bs.black)
    perm = np.concatenate([np.arange(9 * c, 9 * c + 9) for c in np.concatenate([red, blk])])
    Ap = A[np.ix_(perm, perm)]
    nr = red.size
    Arb, Abr = Ap[:9 * nr, 9 * nr:], Ap[9 * nr:, :9 * nr]
    Ub = np.eye(9 * blk.size)
    for q in range(blk.size):
        sl = slice(9 * q, 9 * q + 9)
        Ub[sl, sl] = np.eye(9) - Abr[sl] @ Arb[:, sl]
    L = np.block([[np.eye(9 * nr), np.zeros_like(Arb)], [Abr, np.eye(9 * blk.size)]])
    U = np.block([[np.eye(9 * nr), Arb], [np.zeros_like(Abr), Ub]])
    r = np.random.default_rng(1).normal(size=(n, 9))
    z = np.zeros_like(r)
    bs._apply_precond(r, z)
    zp = np.linalg.solve(U, np.linalg.solve(L, r.reshape(-1)[perm]))
    zr = np.empty_like(zp)
    zr[perm] = zp
    np.testing.assert_allclose(z.reshape(-1), zr, rtol=1e-11, atol=1e-13)


def test_oracle_mcilu_solve_agrees_with_reference_solution():
    """BiCGSTAB with the multicolour preconditioner reaches the reference's
    solution of the same system (LINEAR_TOL 1e-10 makes it solver-independent)."""
    g = golden("asm_small3d.npz")
    s = golden("solve_small3d.npz")
    c = case_objects("small3d")
    ws, blocks = _oracle_assemble(c, state_from(g), g["accn"], float(g["dt"]),
                                  float(g["t_new"]), g["capped"])
    du, dbhp, it = O.BlockSolver(c.grid, ws, tol=1e-10, maxiter=1000,
                                 precond="mcilu").solve(blocks)
    ref = s["ras_du"]
    assert np.linalg.norm(du - ref) <= 1e-8 * np.linalg.norm(ref)
    assert int(s["ras_iters"]) <= it < int(s["none_iters"])


def test_oracle_condensed_mcilu_algebra_and_solution():
    """The condensed multicolour solve (oracle _cond_setup/_cond_solve, the
    checker of the device's default mcilu form, csrc/compact.cu): on the
    reference-assembled small3d system (local rows 6..8 carry no flux)
    (1) S9 (E w) = E (S6 w) for random w -- the red-eliminated 9-component
    operator maps range(E) into itself, so x_b = g_b + E_b w is exact;
    (2) U6 is S6's block diagonal; (3) the condensed du solves the full
    decoupled system to the tolerance and equals the 9-component solve's
    (LINEAR_TOL 1e-10) to 1e-8."""
    g = golden("asm_small3d.npz")
    c = case_objects("small3d")
    ws, blocks = _oracle_assemble(c, state_from(g), g["accn"], float(g["dt"]),
                                  float(g["t_new"]), g["capped"])
    assert not np.any(ws.offd[:, :, O.CR_:, :] != 0.0)
    ref_ws = copy.deepcopy(ws)
    bs = O.BlockSolver(c.grid, ws, tol=1e-10, maxiter=1000, precond="mcilu")
    rhs = -ws.resid
    bs._eliminate_wells(blocks, rhs)
    dloc = ws.diag[:, O.CR_:, :].copy()
    import ctypes
    O.lib().orc_decouple_pass(ctypes.c_int64(rhs.shape[0]), ctypes.c_int64(9), O._p(ws.diag),
                              O._p(rhs), O._p(ws.offd), O._p(ws.adj_ptr), O._p(ws.adj_ids),
                              O._p(ws.adj_sides), O._p(bs.invs), O._p(bs.flags))
    C = bs._cond_setup(dloc)
    assert C is not None
    nb, e = C["nb"], C["e"]
    w = np.random.default_rng(7).normal(size=(nb, O.CR_))
    ew = np.einsum("cij,cj->ci", e, w)
    s9ew = C["s9"](ew)
    s6w = s9ew[:, O.COND_P]
    np.testing.assert_allclose(s9ew, np.einsum("cij,cj->ci", e, s6w), rtol=1e-12, atol=1e-12)
    # block diagonal: S6 applied to a single black cell's unit vectors
    q = nb // 2
    for u in range(O.CR_):
        wu = np.zeros((nb, O.CR_))
        wu[q, u] = 1.0
        col = C["s9"](np.einsum("cij,cj->ci", e, wu))[q, O.COND_P]
        np.testing.assert_allclose(np.linalg.inv(C["u6inv"][q])[:, u], col, rtol=1e-10,
                                   atol=1e-12)
    # solutions
    du6, _, it6 = O.BlockSolver(c.grid, copy.deepcopy(ref_ws), tol=1e-10, maxiter=1000,
                                precond="mcilu").solve(blocks)
    saved = O.BlockSolver.condensed
    try:
        O.BlockSolver.condensed = False
        du9, _, it9 = O.BlockSolver(c.grid, copy.deepcopy(ref_ws), tol=1e-10, maxiter=1000,
                                    precond="mcilu").solve(blocks)
    finally:
        O.BlockSolver.condensed = saved
    assert np.linalg.norm(du6 - du9) <= 1e-8 * np.linalg.norm(du9)
    assert it6 <= it9 + 1
