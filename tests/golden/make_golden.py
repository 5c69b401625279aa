"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Runs only in a container that has /root/reference (read-only) and numba:
    python tests/golden/make_golden.py
Everything written here is produced by the reference's own public objects
(iscsim.assembly.assemble, iscsim.linsolve.BlockSolver, iscsim.newton.Simulator)
on seeded inputs that our side regenerates bit-identically
(paper_1811_11992_b200.configs / synth). Fixture files:

  props_goldens.json   the reference's 31 scalar goldens (pkg/tests/goldens.py)
  asm_small3d.npz      state -> cell_pass outputs, resid/diag/offd, wells (8x6x4)
  solve_small3d.npz    decoupled BiCGSTAB du/dbhp/iters for none/bjacobi/ras
  solve_sub2.npz       32x16x8 grid (2 RAS subdomains): iters + du for each precond
  synth_16.npz         synthetic 16^3 system: iters for each precond, du (ras)
  traj_<case>_<tol>.npz  full runs: per-step records and final fields
  numjac_small3d.npz   assemble(jacobian="numeric") blocks (free and frozen upwind)
                       and check_jacobian's worst discrepancy
  report_frames.npz    two frames (inputs) and the reference writer's cells.csv /
                       wells.csv bytes (report.py write_frame)

    python tests/golden/make_golden.py [name ...]   # regenerate only some
"""

import json
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tools.refdeck import import_reference, reference_simulator  # noqa: E402
from paper_1811_11992_b200 import configs  # noqa: E402
from paper_1811_11992_b200.synth import synth_system  # noqa: E402

import_reference()
import iscsim.assembly as A  # noqa: E402
import iscsim.linsolve as L  # noqa: E402
from iscsim.grid import build_grid as ref_build_grid  # noqa: E402
from iscsim.deck import GridSpec, RockSpec  # noqa: E402


def random_state(sim, seed):
    from tests.golden_states import perturb
    return perturb(sim.state, sim.accn, seed)


def state_dict(st, prefix="st_"):
    return {prefix + f: np.asarray(getattr(st, f)) for f in
            ("p", "t", "sw", "sg", "x", "y", "cc", "bhp")}


def blocks_dict(blocks, prefix="w_"):
    out = {}
    for key in ("resid", "dwdb"):
        out[prefix + key] = np.array([getattr(b, key) for b in blocks])
    for key in ("wrow", "bcol", "phase_rates", "comp_rates"):
        out[prefix + key] = np.stack([getattr(b, key) for b in blocks])
    return out


CELL_FIELDS = ("pot", "dpot", "beta", "dbeta", "hph", "dhph", "yfull", "dyfull", "gam",
               "dgam", "pcv", "dpcv", "kr3", "dkr3", "ktd", "acc", "dacc", "src", "dsrc")


def solve_all(sim, blocks, tol, precs=("none", "bjacobi", "ras")):
    out = {}
    d0, o0 = sim.ws.diag.copy(), sim.ws.offd.copy()
    for pc in precs:
        bs = L.BlockSolver(sim.grid, sim.ws, tol=tol, maxiter=1000, precond=pc)
        du, dbhp, it = bs.solve(blocks)
        sim.ws.diag[:] = d0
        sim.ws.offd[:] = o0
        out[f"{pc}_du"], out[f"{pc}_dbhp"], out[f"{pc}_iters"] = du, dbhp, np.array(it)
    return out


def make_props():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ref_goldens", "/root/reference/pkg/tests/goldens.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)  # the reference's own golden file
    GOLDENS = mod.GOLDENS
    with open(os.path.join(HERE, "props_goldens.json"), "w") as fh:
        json.dump({"source": "/root/reference/pkg/tests/goldens.py", "goldens": GOLDENS},
                  fh, indent=1)


def make_asm_small3d():
    sim = reference_simulator(configs.config("small3d"))
    st, accn = random_state(sim, 5)
    dt = t_new = 2e-3
    blocks = A.assemble(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams, st, accn, dt,
                        t_new, sim.capped)
    out = {"dt": np.array(dt), "t_new": np.array(t_new), "accn": accn,
           "capped": sim.capped.copy(), **state_dict(st)}
    for f in CELL_FIELDS + ("resid", "diag", "offd", "upw"):
        out[f] = getattr(sim.ws, f).copy()
    out.update(blocks_dict(blocks))
    sol = solve_all(sim, blocks, 1e-10)
    # second assembly with frozen upwinding at a perturbed state (newton.py:279)
    st2, accn2 = random_state(sim, 6)
    blocks2 = A.assemble(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams, st2, accn2, dt,
                         t_new, sim.capped, freeze_upwind=True)
    out.update(state_dict(st2, "st2_"))
    out["accn2"] = accn2
    for f in ("resid", "diag", "offd"):
        out[f + "2"] = getattr(sim.ws, f).copy()
    out.update(blocks_dict(blocks2, "w2_"))
    np.savez_compressed(os.path.join(HERE, "asm_small3d.npz"), **out)
    np.savez_compressed(os.path.join(HERE, "solve_small3d.npz"), **sol)


def make_solve_sub2():
    sim = reference_simulator(configs.config("sub2"))
    st, accn = random_state(sim, 11)
    blocks = A.assemble(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams, st, accn, 2e-3,
                        2e-3, sim.capped)
    sol = solve_all(sim, blocks, 1e-10)
    keep = {k: v for k, v in sol.items() if k.endswith("iters") or k.startswith("ras")}
    keep["resid_absmax"] = np.abs(sim.ws.resid).max(axis=0)
    np.savez_compressed(os.path.join(HERE, "solve_sub2.npz"), seed=np.array(11), **keep)


def make_synth():
    nx = ny = nz = 16
    n = nx * ny * nz
    ones = (1.0,) * n
    grid = ref_build_grid(GridSpec(nx, ny, nz, (1.0,) * nx, (1.0,) * ny, (1.0,) * nz),
                          RockSpec(ones, ones, ones, 0.3))
    diag, offd, resid = synth_system(grid, 9, seed=7)
    from types import SimpleNamespace
    m = grid.nconn
    cells = np.concatenate([grid.conn_a, grid.conn_b])
    ics = np.concatenate([np.arange(m), np.arange(m)]).astype(np.int64)
    sides = np.concatenate([np.zeros(m, np.int8), np.ones(m, np.int8)])
    order = np.lexsort((ics, cells))
    ws = SimpleNamespace(diag=diag.copy(), offd=offd.copy(), resid=resid)
    ws.adj_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cells, minlength=n), out=ws.adj_ptr[1:])
    ws.adj_ids, ws.adj_sides = ics[order], sides[order]
    out = {}
    for pc in ("none", "bjacobi", "ras"):
        ws.diag[:] = diag
        ws.offd[:] = offd
        du, _, it = L.BlockSolver(grid, ws, tol=1e-8, maxiter=1000, precond=pc).solve([])
        out[pc + "_iters"] = np.array(it)
        if pc == "ras":
            out["ras_du"] = du
    out["diag_probe"] = diag[:3].copy()
    out["offd_probe"] = offd[:3].copy()
    np.savez_compressed(os.path.join(HERE, "synth_16.npz"), **out)


def make_numjac_small3d():
    """The reference's finite-difference Jacobian (assembly.py:843-939) and
    its analytic-vs-numeric check (assembly.py:942-982) at the seeded states
    of asm_small3d.npz."""
    sim = reference_simulator(configs.config("small3d"))
    st, accn = random_state(sim, 5)
    dt = t_new = 2e-3
    out = {}
    blocks = A.assemble(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams, st, accn, dt,
                        t_new, sim.capped, jacobian="numeric")
    for f in ("resid", "diag", "offd", "upw"):
        out[f] = getattr(sim.ws, f).copy()
    out.update(blocks_dict(blocks))
    # frozen upwinding at the second state (flags left by the first call)
    st2, accn2 = random_state(sim, 6)
    blocks2 = A.assemble(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams, st2, accn2, dt,
                         t_new, sim.capped, jacobian="numeric", freeze_upwind=True)
    for f in ("resid", "diag", "offd"):
        out[f + "2"] = getattr(sim.ws, f).copy()
    out.update(blocks_dict(blocks2, "w2_"))
    out["check"] = np.array(A.check_jacobian(sim.grid, sim.pack, sim.ws, sim.wells, sim.streams,
                                             st, accn, dt, t_new, sim.capped))
    np.savez_compressed(os.path.join(HERE, "numjac_small3d.npz"), **out)
    print("check_jacobian", float(out["check"]))


def make_report_frames():
    """report.py:115-149 on two frames: a C2 run's accepted state after 3 steps
    (real values) and a synthetic frame of formatting edge cases (integers,
    1e16 / 1e-5 thresholds, subnormals, huge, -0.0, nan, inf)."""
    import tempfile
    import iscsim.report as R
    case = configs.config("c2")
    case = replace(case, schedule=replace(case.schedule, t_end=3 * case.schedule.dt_init))
    sim = reference_simulator(case)
    sim.advance()
    f1 = R.capture_frame(sim, sim.time)
    n = 64
    rng = np.random.default_rng(3)
    edge = np.array([0.0, -0.0, 1.0, 123.0, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5, 1.2e-5,
                     5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, np.nan, np.inf,
                     -np.inf, 0.1, 1 / 3, 2014.7, -459.67, 1e22, 1e-7, 12345678901234567.0,
                     0.30000000000000004])
    vals = np.concatenate([edge, rng.normal(size=8 * n) * 10.0 ** rng.integers(-20, 20, 8 * n)])
    take = lambda k: vals[(np.arange(n) * 7 + k) % vals.size].copy()   # noqa: E731
    f2 = R.ReportFrame(time=1e-5, p=take(0), t=take(1), sw=take(2), so=1.0 - take(2) - take(3),
                       sg=take(3), x=np.stack([take(4), take(5)], 1),
                       y=np.stack([take(6 + a) for a in range(5)], 1), cc=take(11),
                       oil_names=f1.oil_names, vap_names=f1.vap_names,
                       well_names=("INJ", "PROD"), bhp=take(12)[:2],
                       rates=np.stack([take(13)[:3], take(14)[:3]]),
                       cum=np.stack([take(15)[:3], take(16)[:3]]))
    out = {}
    with tempfile.TemporaryDirectory() as d:
        with R.ReportSink(d) as sink:
            R.write_frame(f1, sink)
            R.write_frame(f2, sink)
        for name in ("cells", "wells"):
            with open(os.path.join(d, name + ".csv"), "rb") as fh:
                out[name + "_csv"] = np.frombuffer(fh.read(), dtype=np.uint8)
    for k, f in (("f1_", f1), ("f2_", f2)):
        for fld in ("time", "p", "t", "sw", "so", "sg", "x", "y", "cc", "bhp", "rates", "cum"):
            out[k + fld] = np.asarray(getattr(f, fld))
        out[k + "names"] = np.array(["|".join(f.oil_names), "|".join(f.vap_names),
                                     "|".join(f.well_names)])
    np.savez_compressed(os.path.join(HERE, "report_frames.npz"), **out)


def make_traj_c3():
    """BASELINE configs[2]: 60x60x20 (72k cells), 20 timesteps, LINEAR_TOL 1e-10."""
    make_traj("c3", 1e-10)


def make_traj_c4_sample():
    """BASELINE configs[3] (200x200x50, 2 M cells, 5 timesteps) at the deck's
    LINEAR_TOL 1e-5 with the reference's RAS: per-step records and a seeded
    sample of 4096 cells of the final fields (the full fields would be 150 MB)."""
    case = configs.config("c4")
    sim = reference_simulator(case, threads=min(16, os.cpu_count() or 4))
    sim.advance()
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves, s.balance)
                    for s in sim.steps])
    rng = np.random.default_rng(99)
    idx = np.sort(rng.choice(sim.grid.ncell, 4096, replace=False))
    out = {"steps": rec, "cum_imbalance": np.array(sim.cumulative_imbalance()),
           "sample_idx": idx, "final_bhp": np.asarray(sim.state.bhp)}
    for f in ("p", "t", "sw", "sg", "cc"):
        a = np.asarray(getattr(sim.state, f))
        out["sample_" + f] = a[idx]
        out["norm_" + f] = np.array(np.linalg.norm(a))
    np.savez_compressed(os.path.join(HERE, "traj_c4_sample.npz"), **out)
    print("c4", sim.totals())


def make_traj_c4_1e10():
    """BASELINE configs[3] at LINEAR_TOL 1e-10 (the north star's field bar
    needs it on both sides): per-step records, per-solve Krylov
    counts, the field norms and a seeded 16384-cell sample of the final p, T,
    Sw, Sg, C_c (the full fields would be 80 MB)."""
    case = configs.config("c4")
    case = replace(case, solver=replace(case.solver, linear_tol=1e-10))
    sim = reference_simulator(case, threads=min(16, os.cpu_count() or 4))
    iters = []
    orig = L.BlockSolver.solve

    def counting(self, blocks):
        du, dbhp, it = orig(self, blocks)
        iters.append(it)
        return du, dbhp, it

    L.BlockSolver.solve = counting
    try:
        sim.advance()
    finally:
        L.BlockSolver.solve = orig
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves, s.balance)
                    for s in sim.steps])
    rng = np.random.default_rng(4242)
    idx = np.sort(rng.choice(sim.grid.ncell, 16384, replace=False))
    out = {"steps": rec, "cum_imbalance": np.array(sim.cumulative_imbalance()),
           "solve_iters": np.array(iters), "sample_idx": idx,
           "final_bhp": np.asarray(sim.state.bhp)}
    for f in ("p", "t", "sw", "sg", "cc"):
        a = np.asarray(getattr(sim.state, f))
        out["sample_" + f] = a[idx]
        out["norm_" + f] = np.array(np.linalg.norm(a))
    np.savez_compressed(os.path.join(HERE, "traj_c4_1e-10_sample.npz"), **out)
    print("c4 1e-10", sim.totals(), iters)


def make_traj_variants():
    """C2 with heat loss, with a capping/releasing injector, with a
    rate-controlled producer (configs.config docstring), LINEAR_TOL 1e-10."""
    for name in ("c2hl", "c2cap", "c2rate"):
        make_traj(name, 1e-10)


def make_bicgstab_breakdown():
    """The reference's BiCGSTAB restart / breakdown branches on the constructed
    2-cell systems of tests/golden_states.BREAKDOWN_CASES."""
    from types import SimpleNamespace
    from tests.golden_states import BREAKDOWN_CASES, breakdown_system
    from iscsim.errors import Breakdown
    grid = ref_build_grid(GridSpec(2, 1, 1, (1.0, 1.0), (1.0,), (1.0,)),
                          RockSpec((1.0, 1.0), (1.0, 1.0), (1.0, 1.0), 0.3))
    out = {}
    for name, case in BREAKDOWN_CASES.items():
        diag, offd, resid = breakdown_system(case)
        ws = SimpleNamespace(diag=diag, offd=offd, resid=resid,
                             adj_ptr=np.array([0, 1, 2], np.int64),
                             adj_ids=np.array([0, 0], np.int64),
                             adj_sides=np.array([0, 1], np.int8))
        try:
            du, _, it = L.BlockSolver(grid, ws, tol=1e-10, maxiter=50, precond="none").solve([])
            out[name + "_status"] = np.array("ok")
            out[name + "_iters"] = np.array(it)
            out[name + "_du"] = du
        except Breakdown as exc:
            out[name + "_status"] = np.array("Breakdown: " + str(exc))
        print(name, out[name + "_status"], out.get(name + "_iters"))
    np.savez_compressed(os.path.join(HERE, "bicgstab_breakdown.npz"), **out)


def make_c2_deck():
    """The reference deck text of config C2 at LINEAR_TOL 1e-10 (tools/refdeck.py:
    the reference's tube.deck fluid with the case's grid, rock, wells and
    schedule), for the drop-in test that runs the unmodified reference driver
    with the device path patched in (tests/test_gpu_dropin_reference.py)."""
    from tools.refdeck import case_to_deck
    case = configs.config("c2")
    case = replace(case, solver=replace(case.solver, linear_tol=1e-10))
    with open(os.path.join(HERE, "c2_deck_1e-10.txt"), "w") as fh:
        fh.write(case_to_deck(case))


def make_traj_numeric():
    """C1 run in JACOBIAN numeric mode (newton.py:228, 278)."""
    make_traj("c1", 1e-10, jacobian="numeric")


def make_traj(name, ltol, jacobian=None):
    case = configs.config(name)
    case = replace(case, solver=replace(case.solver, linear_tol=ltol))
    sim = reference_simulator(case, threads=min(16, os.cpu_count() or 4), jacobian=jacobian)
    sim.advance()
    rec = np.array([(s.time, s.dt, s.newton, s.linear, s.solves, s.balance)
                    for s in sim.steps])
    out = {"steps": rec, "cum_imbalance": np.array(sim.cumulative_imbalance()),
           **state_dict(sim.state, "final_")}
    tag = "" if jacobian is None else f"_{jacobian}"
    np.savez_compressed(os.path.join(HERE, f"traj_{name}_{ltol:.0e}{tag}.npz"), **out)
    print(name, ltol, sim.totals())


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()["make_" + name]()
        sys.exit(0)
    make_props()
    make_asm_small3d()
    make_solve_sub2()
    make_synth()
    make_numjac_small3d()
    make_traj_numeric()
    make_report_frames()
    make_traj("c1", 1e-10)
    make_traj("c1", 1e-5)
    make_traj("c2", 1e-10)
    make_traj("c2", 1e-5)
    make_traj_c3()
    make_traj_variants()
    make_bicgstab_breakdown()
    make_c2_deck()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
