"""Benchmark: cell·Newton-iterations per second on the B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE configs[3], the 2 M-cell case the north star quotes its
roofline bar on): C4 = 200x200x50 grid, seeded log-normal permeability and
uniform porosity, 4 air injectors + 4 producers, deck-default solver
(LINEAR_TOL 1e-5, LINEAR_MAX 200). One *step* = one solving Newton iteration
of the C4 run's first timestep (dt = 2e-3 d), taken in the order the run
takes them: step j runs iteration (j mod 5) + 1 of that timestep, and every
5th step starts again from the initial state (the reference's C4 first
timestep is 6 residual evaluations / 5 solves, traj_c4_sample.npz; the
sixth evaluation only confirms convergence). So every timed iteration
solves a real Newton correction — from the large first residual down to the
last correction before convergence — instead of re-solving a converged
state. An iteration = newton.py:275-309's loop body: assemble (cell + face
+ wells; upwinding frozen after iteration 5), scaled norm, capped-injector
check, well Schur fold + Gauss-Jordan decoupling, preconditioner setup,
preconditioned BiCGSTAB to LINEAR_TOL, damped update. The preconditioner is
the north star's multicolour block-ILU(0) (--precond mcilu, default); the
reference's own RAS subdomain block-ILU(0) is measured on the same workload
and reported under "ras_exact". ``value`` = cells x steps / device time
(inputs resident in HBM); ``e2e`` = the same iterations through the drop-in
API (assemble/BlockSolver.solve) with each iteration's state and the
accumulation copied from pinned host memory and du read back every step.
The system (9 GB) is far larger than L2, so no flush is needed.

``--impl reference`` times the reference algorithm's CPU implementation (the
plain-C/numpy oracle port of the reference's RAS block-ILU(0) BiCGSTAB, all
host threads: OpenMP in the cell/face/decoupling loops the reference runs
with prange, its independent RAS subdomains factored and applied on a thread
pool) on the same workload: the full C4 grid, the same iteration cycle.
Multi-GPU (torchrun): the C4 grid is z-slab decomposed over the ranks
(strong scaling; NCCL halo per half pass and all-reduced Krylov scalars; the
multicolour preconditioner includes the cross-rank terms, so BiCGSTAB takes
the single-GPU iterations); device time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell·Newton-iters/sec (assemble+decouple+solve)"
UNIT = "cell-iters/s"
KCLASS = ["cell", "face", "wells", "decouple", "ilu_factor", "ilu_apply", "spmv", "other"]
# solving Newton iterations of the C4 first timestep (the reference's run:
# 6 residual evaluations, 5 solves, 22 BiCGSTAB iterations with its RAS at
# LINEAR_TOL 1e-5 — tests/golden/traj_c4_sample.npz)
CYCLE = 5
REF_STEP1 = {"newton": 6, "solves": 5, "bicgstab_iters": 22, "precond": "ras"}


def workload(cfg_name, case):
    dt = case.schedule.dt_init
    return {"workload": f"{cfg_name.upper()} {case.nx}x{case.ny}x{case.nz} ({case.ncell} cells, "
                        f"{len(case.wells)} wells): the {CYCLE} solving Newton iterations of the "
                        f"first timestep (dt={dt} d) in run order, restarting from the initial "
                        f"state every {CYCLE} steps; iteration = assemble + scaled norm + "
                        f"decouple + precond setup + BiCGSTAB to LINEAR_TOL + damped update",
            "linear_tol": case.solver.linear_tol,
            "l2": "inputs larger than L2 (system ~9 GB), no flush"}


class NewtonCycle:
    """Bench step j = solving Newton iteration (j mod CYCLE) + 1 of the first
    timestep, restarting from the initial state every CYCLE steps."""

    def __init__(self, sim, dt):
        self.sim, self.dt, self.j = sim, dt, 0
        self.init = sim.state.copy()
        self.work = sim.state.copy()
        self.capped = sim.capped.copy()

    def step(self):
        it = self.j % CYCLE + 1
        if it == 1:
            self.work.u.copy_(self.init.u)
            self.work.bhp = self.init.bhp.copy()
            self.capped = self.sim.capped.copy()
        self.j += 1
        return self.sim.newton_iteration(self.work, self.dt, self.dt, self.capped, it)[1]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4",
                    help="c4 (headline, BASELINE configs[3]) or c5 (configs[4] linear-solver "
                         "microbench)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="c5 under torchrun: strong = 400x400x100 split over the ranks, weak = "
                         "400x400x(100*ranks)")
    ap.add_argument("--precond", default="mcilu",
                    help="GPU preconditioner for the headline: mcilu (north_star's multicolour "
                         "block-ILU(0), default) or the reference's ras / bjacobi / none")
    ap.add_argument("--no-ras", action="store_true",
                    help="skip the secondary measurement with the reference's exact RAS")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spmv", action="store_true")
    return ap.parse_args()


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) < 7:
                continue
            for k, nm in enumerate(names):
                if s[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def ilu_bytes(ctx_counts, n, m):
    """Algorithmic bytes of one RAS ILU(0) apply: matrix data streamed once
    (U^-1 per slot, L blocks per lower link, A blocks per upper link),
    the input read and output written once per slot / cell."""
    nslots, nlow, nup = ctx_counts
    return 8 * (81 * (nslots + nlow + nup) + 9 * nslots + 9 * n)


def ilu_structure_counts(grid):
    """(slots, lower links, upper links) of the reference's RAS partition."""
    nsub = min(64, max(1, grid.ncell // 2048))
    dims = [grid.nx, grid.ny, grid.nz]
    axis = int(np.argmax(dims))
    base, extra = divmod(dims[axis], nsub)
    slots = links = 0
    pos = 0
    for s in range(nsub):
        size = base + (1 if s < extra else 0)
        lo, hi = pos, pos + size
        if nsub > 1:
            lo, hi = max(0, lo - 1), min(dims[axis], hi + 1)
        w = list(dims)
        w[axis] = hi - lo
        slots += w[0] * w[1] * w[2]
        links += (w[0] - 1) * w[1] * w[2] + w[0] * (w[1] - 1) * w[2] + w[0] * w[1] * (w[2] - 1)
        pos += size
    return slots, links, links


def ncu_traffic(kernel_class, precond):
    """DRAM bytes (read + write) per launch of a kernel class from the latest
    committed `ncu --set full` capture (profiles/r*/ncu_traffic.json, made by
    tools/ncu_summary.py on the C4 mcilu bench); None when not captured."""
    import glob
    if precond != "mcilu":
        return None, None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")))
    if not files:
        return None, None
    with open(files[-1]) as fh:
        d = json.load(fh)
    if kernel_class not in d:
        return None, None
    return float(d[kernel_class]["dram_bytes"]), os.path.relpath(files[-1], ROOT)


def algorithmic_bytes(grid, nw, precond="ras", form="explicit"):
    """Compulsory bytes per launch of each kernel class."""
    n, m = grid.ncell, grid.nconn
    out = {
        # SURVEY §8(d) assembly 8(111n + 164m), split by kernel: the cell pass
        # reads state, phi_ref, accn, V, depth (21 n) and writes resid + the
        # diagonal blocks (90 n); the face passes read gd + td (2 m) and write
        # both off-diagonal blocks of every connection (162 m)
        "cell": 8 * 111 * n,
        "face": 8 * 164 * m,
        "decouple": 8 * (99 * n + 324 * m),
        "spmv": 8 * (162 * m + 18 * n),
        "ilu_apply": ilu_bytes(ilu_structure_counts(grid), n, m),
    }
    if precond == "mcilu":
        # red-eliminated BiCGSTAB (capi.cu bicgstab_schur), per product S U_b^-1:
        # red pass w_r = -B_rb z_b: the red rows' blocks (81 m), z_b read once
        # (9 n/2), w_r written (9 n/2)
        out["ilu_apply"] = 8 * (81 * m + 9 * n)
        # black pass v_b = z_b + B_br w_r: the black rows' blocks (81 m), w_r and
        # z_b read (9 n), v_b written (9 n/2), one dot operand (9 n/2)
        out["spmv"] = 8 * (81 * m + 18 * n)
        # k_mc_factor: the black rows' blocks and the red neighbours' blocks
        # pointing back (81 m each), U_b^-1 out (81 n/2)
        out["mc_factor"] = 8 * (162 * m + 40.5 * n)
        if form == "compact":
            # compact operator (csrc/compact.cu)
            # red pass y_r = B_rb z_b: 54 per red block of which 49 are loaded (the
            # component rows' coke column is structurally zero and skipped while
            # the assembly saw no nonzero there), z_b gathered (9 n/2), y written
            # (6 n/2); black pass v_b = z_b - D_b^-1[:, :6] B'_br y: 36
            # per black block, D_b^-1[:, :6] (54 n/2), y gathered (6 n/2), z_b,
            # v_b and the dot operand (3 x 9 n/2)
            out["ilu_apply"] = 8 * (49 * m + 7.5 * n)
            out["spmv"] = 8 * (36 * m + 43.5 * n)
            # k_decouple_compact_t with the well Schur fold: diag and resid in,
            # D^-1[:, :6] and rhs out
            out["decouple"] = 8 * (81 * n + 9 * n + 54 * n + 9 * n)
            # k_mc_factor_compact per black cell: B_bd and B_back flux rows
            # (54 m each colour), D^-1[:, :6] of both colours (27 n each), the red
            # neighbours' b (9 n/2), B' out (36 m), U_b^-1 out (81 n/2), g_b out
            # twice (9 n)
            out["mc_factor"] = 8 * (144 * m + 54 * n + 4.5 * n + 40.5 * n + 9 * n)
        if form == "condensed":
            # condensed form (csrc/compact.cu: 6-component iteration)
            # red pass y_r = sum_d Bc_rd w: 36 per red block, w gathered (6 n/2),
            # y written (6 n/2); black pass v = z - Dc_b^-1 sum_d B'_bd y: 36 per
            # black block, Dc_b^-1 (36 n/2), y gathered, z read, v written and the
            # dot operand (4 x 6 n/2)
            out["ilu_apply"] = 8 * (36 * m + 6 * n)
            out["spmv"] = 8 * (36 * m + 30 * n)
            # + k_cond_es: the local rows of the black cells' diagonal blocks in
            # (27 n/2), E_S out (18 n/2)
            out["decouple"] = 8 * (81 * n + 9 * n + 54 * n + 9 * n + 22.5 * n)
            # k_mc_factor_cond_t (condensed form): B_bd and B_back flux rows (54 m each),
            # D^-1[:, :6] of both colours (54 n), the red neighbours' b (4.5 n),
            # E_S (9 n), B' out (36 m), U6^-1 out (18 n), g_b (4.5 n); the Bc
            # blocks are formed with the raw red pass on g (k_cc_red_bc)
            out["mc_factor"] = 8 * (144 * m + 90 * n)
    return out


# ------------------------------------------------------------------ ours

def measure_device(case, steps, warmup, world):
    """Device-resident Newton-cycle steps of `case` -> (ms, iters, sim)."""
    import torch
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.newton import Simulator
    grid, pack, wells, streams, state = configs.build_case(case)
    sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
    cyc = NewtonCycle(sim, case.schedule.dt_init)
    for _ in range(warmup):
        cyc.step()
    cyc.j = 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    e0.record()
    for _ in range(steps):
        its.append(cyc.step())
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), float(np.mean(its)), sim


def run_ours(args, rank, world, local):
    """Device-resident Newton iterations; under torchrun the global case is
    z-slab decomposed over the ranks (NCCL halos + all-reduces, strong
    scaling), single GPU otherwise."""
    import torch
    from paper_1811_11992_b200 import configs, _native as N
    from paper_1811_11992_b200.assembly import Workspace, assemble
    from paper_1811_11992_b200.linsolve import BlockSolver
    from paper_1811_11992_b200.newton import Simulator

    torch.cuda.set_device(local)
    case = configs.config(args.config)
    if args.precond:
        from dataclasses import replace
        case = replace(case, solver=replace(case.solver, precond=args.precond))
    n_global = case.ncell
    dist_note = "single GPU"
    if world > 1:
        import torch.distributed as dist
        from paper_1811_11992_b200.distributed import attach_nccl, nccl_unique_id, split_case
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if case.solver.precond not in ("mcilu", "none"):
            from dataclasses import replace
            case = replace(case, solver=replace(case.solver, precond="mcilu"))
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        piece = split_case(case, world, rank)
        grid, pack, wells, streams, state = (piece.grid, piece.pack, piece.wells, piece.streams,
                                             piece.state)
        sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver,
                        comm_setup=lambda ctx: attach_nccl(ctx, uid[0], piece))
        dist_note = (f"z-slab x{world} (planes {piece.k0}-{piece.k1 - 1} on rank {rank}; NCCL "
                     f"halo per half pass + all-reduced Krylov scalars; mcilu with cross-rank "
                     f"boundary blocks)")
    else:
        grid, pack, wells, streams, state = configs.build_case(case)
        sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
    n = grid.ncell
    ctx = sim.ctx
    dt = case.schedule.dt_init
    cyc = NewtonCycle(sim, dt)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # one pass over the cycle, untimed: the iterates (for the e2e leg) and the
    # per-iteration Krylov counts; then the warm-up steps
    host_states, host_u, cycle_iters = [], [], []
    for _ in range(CYCLE):
        cur = cyc.work if cyc.j % CYCLE else cyc.init
        if world == 1:
            host_states.append(cur.to_host())
        else:
            host_u.append((cur.u.cpu().pin_memory(), cur.bhp.copy()))
        cycle_iters.append(cyc.step())
    for _ in range(args.warmup):
        cyc.step()
    cyc.j = 0
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    N.check(ctx.L.isc_set_profiling(ctx.h, 1), "profiling")
    ms8, cnt8 = np.zeros(8), np.zeros(8, dtype=np.int64)
    ctx.L.isc_kernel_times(ctx.h, N.ptr(ms8), N.ptr(cnt8), 1)
    l0 = ctx.launch_count()
    st0 = ctx.stage_times()
    its = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record()
    for _ in range(args.steps):
        its.append(cyc.step())
    ev1.record()
    barrier()
    dev_ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - l0
    stage_ms = (ctx.stage_times() - st0) / max(1, args.steps)
    ctx.L.isc_kernel_times(ctx.h, N.ptr(ms8), N.ptr(cnt8), 1)
    N.check(ctx.L.isc_set_profiling(ctx.h, 0), "profiling")
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())

    e2e_steps = max(CYCLE, min(args.steps, 2 * CYCLE))
    if world == 1:
        # ---- e2e through the drop-in API with host buffers ---------------
        # the same iterations: iterate j's host State (pinned) and the host
        # accumulation go in, du comes back to the host every step
        ws = Workspace(grid, pack, None, wells=wells, streams=streams,
                       precond=case.solver.precond)
        solver = BlockSolver(grid, ws, tol=case.solver.linear_tol,
                             maxiter=case.solver.linear_max, precond=case.solver.precond)
        from types import SimpleNamespace
        hstates = [SimpleNamespace(**{k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
                                      .numpy() for k, v in hs.items()}) for hs in host_states]
        accn_h = torch.from_numpy(
            np.ascontiguousarray(sim.accn.t().cpu().numpy())).pin_memory().numpy()
        bi = (sum(a.nbytes for a in vars(hstates[0]).values()) + accn_h.nbytes)
        capped = sim.capped.copy()

        def e2e_step(j):
            it = j % CYCLE + 1
            blocks = assemble(grid, pack, ws, wells, streams, hstates[it - 1], accn_h, dt, dt,
                              capped, freeze_upwind=it > 5)
            return solver.solve(blocks)

        for j in range(CYCLE):
            du, dbhp, _ = e2e_step(j)
        barrier()
        t0 = time.perf_counter()
        for j in range(e2e_steps):
            du, dbhp, _ = e2e_step(j)
        barrier()
        e2e_s = time.perf_counter() - t0
        bo = du.nbytes + dbhp.nbytes
        path = ("assembly.assemble(host State of iterate j, host accn) + "
                "linsolve.BlockSolver.solve -> host du")
        ws.ctx.close()
    else:
        # ---- e2e per rank: iterate j's slab state H2D from pinned host, the
        # iteration, the updated state D2H, every step ----------------------
        h_out = torch.empty_like(host_u[0][0]).pin_memory()
        bi = bo = h_out.numel() * 8
        barrier()
        t0 = time.perf_counter()
        for j in range(e2e_steps):
            it = j % CYCLE + 1
            cyc.work.u.copy_(host_u[it - 1][0], non_blocking=True)
            cyc.work.bhp = host_u[it - 1][1].copy()
            sim.newton_iteration(cyc.work, dt, dt, sim.capped.copy(), it)
            h_out.copy_(cyc.work.u, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        barrier()
        t = torch.tensor([time.perf_counter() - t0], device="cuda")
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        path = ("newton.Simulator.newton_iteration per rank: iterate j's slab state H2D from "
                "pinned host, updated state D2H, every step")
    e2e = {"value": n_global * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(bi),
           "d2h_bytes_per_step": int(bo), "path": path}

    value = n_global * args.steps / (dev_ms / 1e3)
    cfg = workload(args.config, case)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded: log-normal perm, uniform porosity; BASELINE configs[3])",
           "config": cfg,
           "algorithm": {"precond": case.solver.precond,
                         "note": ("multicolour (red-black) block-ILU(0) per north_star; the "
                                  "reference's exact RAS on the GPU is reported in ras_exact")
                         if case.solver.precond == "mcilu" else "reference preconditioner",
                         "bicgstab_iters_per_step": float(np.mean(its)),
                         "bicgstab_iters_per_cycle_iteration": cycle_iters,
                         "reference_first_timestep": REF_STEP1,
                         "parallelism": dist_note},
           "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
           # timers per stage, CUDA events, ms per Newton iteration
           "stage_ms": {"assemble": float(stage_ms[0]), "decouple": float(stage_ms[1]),
                        "precond_setup": float(stage_ms[2]), "krylov": float(stage_ms[3])}}
    # ---- roofline of the dominant kernel class ----------------------------
    hbm, peak_src = peaks()
    algo = algorithmic_bytes(grid, len(wells), case.solver.precond,
                             "condensed" if sim.ctx.condensed else sim.ctx.decoupled_form)
    ktimes = {KCLASS[i]: {"ms": float(ms8[i]), "launches": int(cnt8[i])} for i in range(8)}
    classes = {"ilu_apply": ("ilu_apply",), "spmv": ("spmv",), "decouple": ("decouple",),
               "cell": ("cell",), "face": ("face",)}
    if case.solver.precond == "mcilu":   # red pass / black pass of S U_b^-1
        classes = {"red_pass": ("ilu_apply",), "black_pass": ("spmv",),
                   "decouple": ("decouple",), "cell": ("cell",), "face": ("face",),
                   "mc_factor": ("ilu_factor",)}
        algo = dict(algo, red_pass=algo["ilu_apply"], black_pass=algo["spmv"])
    rows = {}
    for key, parts in classes.items():
        ms = sum(ktimes[p]["ms"] for p in parts)
        nl = ktimes[parts[0]]["launches"]
        if nl == 0 or ms <= 0:
            continue
        per = ms / nl
        ach = algo[key] / (per / 1e3) / 1e9
        rows[key] = {"avg_ms": per, "launches": nl, "share": ms / dev_ms,
                     "algorithmic_bytes": algo[key], "achieved_gbs": ach, "frac": ach / hbm}
    dom = max(rows, key=lambda k: rows[k]["share"])
    traffic, tsrc = ncu_traffic(dom, case.solver.precond)
    out["roofline"] = {"kernel": dom, "bound": "hbm", "achieved": rows[dom]["achieved_gbs"],
                       "peak": hbm, "unit": "GB/s", "frac": rows[dom]["achieved_gbs"] / hbm,
                       # north_star quotes the ~8 TB/s HBM3e spec
                       "frac_of_8tbs_spec": rows[dom]["achieved_gbs"] / 8000.0,
                       "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
                       "kernels": rows, "kernel_ms": ktimes}
    return out, sim


# ------------------------------------------------------ SpMV microbench

def run_spmv_c5(steps=20):
    """BASELINE configs[4]: 400x400x100 synthetic BSR (16 M block rows),
    decoupled; SpMV achieved HBM GB/s (CUDA events, inputs >> L2)."""
    import torch
    from paper_1811_11992_b200 import _native as N
    from paper_1811_11992_b200.grid import build_grid
    from paper_1811_11992_b200.model import load_pack
    from paper_1811_11992_b200.device import DeviceContext
    free, _ = torch.cuda.mem_get_info()
    nx, ny, nz = 400, 400, 100
    if free < 120e9:
        nz = max(10, int(100 * free / 140e9))
    grid = build_grid(nx, ny, nz, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    pack = load_pack("tube3_pack", grid.phi_ref)
    ctx = DeviceContext(grid, pack, (), (), "mcilu")
    N.check(ctx.L.isc_synth_system(ctx.h, 7), "synth")
    import ctypes
    bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    N.check(ctx.L.isc_decouple(ctx.h, ctypes.byref(bc), ctypes.byref(bcol)), "decouple")
    e1.record()
    torch.cuda.synchronize()
    dec_ms = e0.elapsed_time(e1)
    x = torch.randn(9, grid.ncell, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        N.check(ctx.L.isc_spmv(ctx.h, N.ptr(x), N.ptr(y)), "spmv")
    torch.cuda.synchronize()
    # isc_spmv (natural-order C-ABI) also permutes x in / y out; time the
    # SpMV kernel itself with CUDA events around its launches
    ms8, cnt8 = np.zeros(8), np.zeros(8, dtype=np.int64)
    N.check(ctx.L.isc_set_profiling(ctx.h, 1), "profiling")
    ctx.L.isc_kernel_times(ctx.h, N.ptr(ms8), N.ptr(cnt8), 1)
    for _ in range(steps):
        ctx.L.isc_spmv(ctx.h, N.ptr(x), N.ptr(y))
    ctx.L.isc_kernel_times(ctx.h, N.ptr(ms8), N.ptr(cnt8), 1)
    N.check(ctx.L.isc_set_profiling(ctx.h, 0), "profiling")
    ms = ms8[6] / max(1, cnt8[6])
    nbytes = 8 * (162 * grid.nconn + 18 * grid.ncell)
    hbm, src = peaks()
    # BASELINE configs[4] solve: multicolour ILU(0) + BiCGSTAB to 1e-8 on the
    # decoupled system (factorisation + Krylov; decoupling timed above)
    du = torch.empty_like(x)
    it = ctypes.c_int32(0)
    e0.record()
    st = ctx.L.isc_solve(ctx.h, 1e-8, 1000, N.ptr(du), N.VP(0), ctypes.byref(it),
                         ctypes.byref(bc), ctypes.byref(bcol))
    e1.record()
    torch.cuda.synchronize()
    N.check(st, "c5 solve")
    solve_ms = e0.elapsed_time(e1)
    ctx.close()
    del x, y, du
    torch.cuda.empty_cache()
    return {"grid": f"{nx}x{ny}x{nz}", "block_rows": grid.ncell, "ms": ms,
            "algorithmic_bytes": nbytes, "achieved_gbs": nbytes / ms / 1e6,
            "frac": nbytes / ms / 1e6 / hbm, "peak": hbm, "peak_source": src,
            "solve": {"precond": "mcilu", "tol": 1e-8, "bicgstab_iters": int(it.value),
                      "decouple_ms": dec_ms, "factor_plus_krylov_ms": solve_ms,
                      "block_rows_per_s": grid.ncell / ((dec_ms + solve_ms) / 1e3)}}


def run_c5(args, rank, world, local):
    """BASELINE configs[4]: seeded synthetic 7-point BSR (400x400x100, 16 M
    block rows; weak scaling: 400x400x(100*ranks)), Gauss-Jordan decoupled
    once, then every step = multicolour ILU(0) setup + BiCGSTAB to 1e-8.
    Under torchrun each rank generates its z-slab rows of the global system
    (isc_synth_system_slab, keyed by global cell index) and the solve runs
    over NCCL (halo per half pass, all-reduced Krylov scalars)."""
    import ctypes
    import torch
    from dataclasses import replace
    from paper_1811_11992_b200 import configs, _native as N
    from paper_1811_11992_b200.device import DeviceContext
    torch.cuda.set_device(local)
    case = configs.config("c5")
    if args.scaling == "weak" and world > 1:
        case = replace(case, nz=case.nz * world)
    n_global = case.ncell
    if world > 1:
        import torch.distributed as dist
        from paper_1811_11992_b200.distributed import attach_nccl, nccl_unique_id, split_case
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        piece = split_case(case, world, rank)
        grid, pack = piece.grid, piece.pack
        ctx = DeviceContext(grid, pack, (), (), "mcilu")
        attach_nccl(ctx, uid[0], piece)
        note = f"z-slab x{world} ({args.scaling}), planes {piece.k0}-{piece.k1 - 1} on rank {rank}"
    else:
        grid, pack, _, _, _ = configs.build_case(case)
        ctx = DeviceContext(grid, pack, (), (), "mcilu")
        note = "single GPU"

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    N.check(ctx.L.isc_synth_system_slab(ctx.h, 7, case.nz), "synth")
    bc, bcol = ctypes.c_int64(-1), ctypes.c_int32(-1)
    it = ctypes.c_int32(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    N.check(ctx.L.isc_decouple(ctx.h, ctypes.byref(bc), ctypes.byref(bcol)), "decouple")
    e1.record()
    barrier()
    dec_ms = e0.elapsed_time(e1)
    du = ctx.empty(9, grid.ncell)

    def step():
        N.check(ctx.L.isc_precond_setup(ctx.h, ctypes.byref(bc)), "setup")
        N.check(ctx.L.isc_solve(ctx.h, case.solver.linear_tol, case.solver.linear_max,
                                N.ptr(du), N.VP(0), ctypes.byref(it), ctypes.byref(bc),
                                ctypes.byref(bcol)), "c5 solve")
        return it.value

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count()
    its = []
    e0.record()
    for _ in range(args.steps):
        its.append(step())
    e1.record()
    barrier()
    dev_ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    # host-buffer leg: a new decoupled rhs from pinned host memory per solve
    # (isc_set_rhs), du back to pinned host memory
    rhs = ctx.empty(9, grid.ncell)
    N.check(ctx.L.isc_copy_rhs(ctx.h, N.ptr(rhs)), "rhs")
    h_rhs = rhs.cpu().pin_memory()
    h_du = torch.empty_like(h_rhs).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        rhs.copy_(h_rhs, non_blocking=True)
        N.check(ctx.L.isc_set_rhs(ctx.h, N.ptr(rhs)), "set rhs")
        step()
        h_du.copy_(du, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_ms, e2e_s, dec_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_s, dec_ms = (float(v) for v in t.tolist())
    ctx.close()
    unit = "block-rows/s"
    out = {"metric": "block-rows/s (multicolour ILU(0) setup + BiCGSTAB to 1e-8, decoupled "
                     "7-point BSR)",
           "value": n_global * args.steps / (dev_ms / 1e3), "unit": unit, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
           "higher_is_better": True, "scaling": args.scaling if world > 1 else "strong",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded BSR of BASELINE configs[4], keyed by global cell index)",
           "config": {"workload": f"C5 {case.nx}x{case.ny}x{case.nz} ({n_global} block rows), "
                                  f"decoupled once ({dec_ms:.1f} ms), step = mcilu setup + "
                                  f"BiCGSTAB to {case.solver.linear_tol}",
                      "l2": "inputs larger than L2 (system ~72 GB per 16 M rows), no flush"},
           "algorithm": {"precond": "mcilu", "bicgstab_iters": its, "parallelism": note},
           "e2e": {"value": n_global * e2e_steps / e2e_s, "unit": unit,
                   "h2d_bytes_per_step": int(h_rhs.numel() * 8 * world),
                   "d2h_bytes_per_step": int(h_du.numel() * 8 * world),
                   "path": "isc_set_rhs (pinned host rhs) + isc_precond_setup + isc_solve -> "
                           "pinned host du"},
           "gpu_launches": int(launches), "clocks": clk, "decouple_ms": dec_ms}
    return out


# --------------------------------------------------------- CPU oracle arm

def run_oracle(steps, warmup, config="c4", budget_s=None):
    """The reference algorithm on the host: the oracle port (plain C with
    OpenMP where the reference uses prange, numpy drivers, the reference's
    RAS subdomain block-ILU(0) with its independent subdomains on a thread
    pool) stepping the same Newton-iteration cycle of the same full-size case.
    ``budget_s`` (cpu_baseline leg) stops after the first step past the budget."""
    ncpu = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(ncpu)
    from oracle import isc_oracle as O
    from paper_1811_11992_b200 import configs
    case = configs.config(config)
    grid, pack, wells, streams, state = configs.build_case(case)
    sim = O.Simulator(grid, pack, wells, streams, state, case.schedule, case.solver,
                      threads=ncpu)
    solver = sim.solver
    dt = case.schedule.dt_init
    init = sim.state.copy()
    cur = {"st": init.copy(), "j": 0, "capped": np.zeros(len(wells), dtype=bool)}

    def step():
        """newton.py:275-309 loop body for solving iteration (j mod CYCLE) + 1."""
        it = cur["j"] % CYCLE + 1
        if it == 1:
            cur["st"] = init.copy()
        st = cur["st"]
        blocks = O.assemble(grid, sim.model, sim.ws, sim.wells, sim.streams, st, sim.accn, dt,
                            dt, cur["capped"], freeze_upwind=it > 5)
        O.scaled_norm(sim.ws, sim.accn, grid.volume, dt, blocks, sim.wells, cur["capped"],
                      pack.row_energy + 1, pack.row_energy + 2)
        O.desired_capped(sim.wells, cur["capped"], st, blocks)
        du, dbhp, iters = solver.solve(blocks)
        cur["st"] = O.apply_update(st, du, dbhp, pack.nco, pack.ncg, case.solver.eps)
        cur["j"] += 1
        return iters

    for _ in range(warmup):
        step()
    cur["j"] = 0
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        its.append(step())
        if budget_s and time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    done = len(its)
    return {"value": grid.ncell * done / el, "unit": UNIT, "cores": ncpu, "kind": "port",
            "sample": f"{config.upper()} full grid ({grid.ncell} cells), {done} Newton "
                      f"iterations of the first-timestep cycle (assemble + norm + decouple + "
                      f"RAS block-ILU(0) + BiCGSTAB to {case.solver.linear_tol} + update), "
                      f"oracle/ C+numpy port of the reference, OpenMP + "
                      f"{ncpu}-thread subdomain pool",
            "seconds": el, "steps": done, "bicgstab_iters": its, "case": case}


def run_oracle_c5(steps, warmup):
    """Reference arm of the C5 microbench: the reference's solver (oracle
    port: RAS block-ILU(0) on its subdomain thread pool, BiCGSTAB to 1e-8) on
    a bounded C5 sample (the host-side generator's 200x200x10 system, the
    reference's layout), decoupled once; step = factorisation + BiCGSTAB."""
    ncpu = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(ncpu)
    import ctypes
    from types import SimpleNamespace
    from oracle import isc_oracle as O
    from paper_1811_11992_b200.grid import build_grid
    from paper_1811_11992_b200.synth import synth_system
    grid = build_grid(200, 200, 10, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.3)
    diag, offd, resid = synth_system(grid, 9, seed=7)
    ws = O.Workspace(grid, SimpleNamespace(nequ=9, nfull=5))
    ws.diag, ws.offd, ws.resid = diag, offd, resid
    bs = O.BlockSolver(grid, ws, tol=1e-8, maxiter=1000, precond="ras", threads=ncpu)
    rhs = -resid
    O.lib().orc_decouple_pass(ctypes.c_int64(grid.ncell), ctypes.c_int64(9), O._p(ws.diag),
                              O._p(rhs), O._p(ws.offd), O._p(ws.adj_ptr), O._p(ws.adj_ids),
                              O._p(ws.adj_sides), O._p(bs.invs), O._p(bs.flags))

    def step():
        bs._factor()
        return bs._bicgstab(rhs)[1]

    for _ in range(warmup):
        step()
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        its.append(step())
    el = time.perf_counter() - t0
    return {"value": grid.ncell * steps / el, "unit": "block-rows/s", "cores": ncpu,
            "kind": "port", "seconds": el, "bicgstab_iters": its,
            "sample": f"C5 sample {grid.nx}x{grid.ny}x{grid.nz} ({grid.ncell} block rows): RAS "
                      f"block-ILU(0) setup + BiCGSTAB to 1e-8, oracle/ C+numpy port, OpenMP + "
                      f"{ncpu}-thread subdomain pool"}


def run_timesteps(config="c4", nsteps=2):
    """whole timesteps of the C4 run through newton.Simulator.advance
    (multicolour solve): Newton counts two ways (residual evaluations, solves),
    BiCGSTAB iterations, wall time (the driver's host logic included)."""
    import time as _t
    import torch
    from dataclasses import replace
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.newton import Simulator
    case = configs.config(config)
    case = replace(case, solver=replace(case.solver, precond="mcilu"),
                   schedule=replace(case.schedule, t_end=nsteps * case.schedule.dt_init))
    grid, pack, wells, streams, state = configs.build_case(case)
    sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    sim.advance()
    torch.cuda.synchronize()
    wall = _t.perf_counter() - t0
    out = {"config": config, "precond": "mcilu",
           "steps": [{"time": s.time, "dt": s.dt, "newton": s.newton, "solves": s.solves,
                      "linear": s.linear} for s in sim.steps],
           "wall_s": wall, "cumulative_imbalance": float(sim.cumulative_imbalance())}
    sim.ctx.close()
    return out


def run_numjac(config="c4", reps=3):
    """JACOBIAN numeric (assembly.py:843-939) at the C4 initial
    state — 2 probes x 9 unknowns per cell, each a full cell_eval + six face
    fluxes — timed with CUDA events after one analytic assemble."""
    import torch
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.device import DeviceContext, state_to_device
    case = configs.config(config)
    grid, pack, wells, streams, state = configs.build_case(case)
    ctx = DeviceContext(grid, pack, wells, streams, "none")
    d_state = state_to_device(state, ctx.device)
    zero = torch.zeros(9, grid.ncell, dtype=torch.float64, device=ctx.device)
    ctx.assemble(d_state, state.bhp, zero, 1.0, 0.0, np.zeros(len(wells), bool), False)
    acc = ctx.copy_out(1, 9).clone()
    ctx.assemble(d_state, state.bhp, acc, 2e-3, 2e-3, np.zeros(len(wells), bool), False)
    ctx.numeric_jacobian()   # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ctx.numeric_jacobian()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ctx.close()
    return {"config": config, "cells": grid.ncell, "ms": ms,
            "cells_per_s": grid.ncell / (ms / 1e3),
            "probes_per_s": 18 * grid.ncell / (ms / 1e3)}


def run_report(config="c4"):
    """one report frame of the C4 state — device->host capture
    (state + yfull) and the native repr-identical cells.csv formatter."""
    import time as _t
    import torch
    from paper_1811_11992_b200 import configs
    from paper_1811_11992_b200.newton import Simulator
    from paper_1811_11992_b200.report import capture_frame, format_cells
    case = configs.config(config)
    grid, pack, wells, streams, state = configs.build_case(case)
    sim = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    frame = capture_frame(sim, 0.002)
    t1 = _t.perf_counter()
    text = format_cells(frame)
    t2 = _t.perf_counter()
    sim.ctx.close()
    return {"config": config, "cells": grid.ncell, "capture_ms": (t1 - t0) * 1e3,
            "format_ms": (t2 - t1) * 1e3, "bytes": len(text),
            "format_mb_per_s": len(text) / (t2 - t1) / 1e6, "threads": min(64, os.cpu_count() or 1)}


def main():
    args = parse()
    rank, world, local = dist_setup(args.gpus)
    if world > 1:
        # NCCL's init lines (ranks, transports, NVLS) on stderr: the JSON line
        # stays alone on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        if rank != 0:
            return
        if args.config == "c5":
            res = run_oracle_c5(args.steps, args.warmup)
            line = {"metric": "block-rows/s (multicolour ILU(0) setup + BiCGSTAB to 1e-8, "
                              "decoupled 7-point BSR)",
                    "value": res["value"], "unit": res["unit"], "n_gpus": args.gpus,
                    "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": res["seconds"] * 1e3 / max(1, args.steps),
                    "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                    "dtype": "f64", "data": "synthetic (seeded BSR of BASELINE configs[4])",
                    "impl": "reference", "config": {"workload": res["sample"]},
                    "algorithm": {"precond": "ras", "bicgstab_iters": res["bicgstab_iters"]},
                    "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind",
                                                         "sample")},
                    "e2e": {"value": res["value"], "unit": res["unit"], "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line))
            return
        res = run_oracle(args.steps, args.warmup, args.config)
        case = res["case"]
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": res["seconds"] * 1e3 / max(1, res["steps"]),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (seeded: log-normal perm, uniform porosity; BASELINE "
                        "configs[3])",
                "impl": "reference", "config": workload(args.config, case),
                "algorithm": {"precond": case.solver.precond,
                              "note": "the reference's own algorithm (RAS subdomain "
                                      "block-ILU(0), serial-order dots) on the host cores",
                              "bicgstab_iters_per_step": float(np.mean(res["bicgstab_iters"])),
                              "bicgstab_iters": res["bicgstab_iters"]},
                "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    if args.config == "c5":
        out = run_c5(args, rank, world, local)
        if rank == 0:
            print(json.dumps(out))
        return
    out, sim = run_ours(args, rank, world, local)
    sim.ctx.close()
    del sim
    if rank == 0 and world == 1 and not args.no_ras and args.precond != "ras":
        # the reference's own preconditioner (exact RAS block-ILU(0)), same workload
        from dataclasses import replace
        from paper_1811_11992_b200 import configs
        case = configs.config(args.config)
        case = replace(case, solver=replace(case.solver, precond="ras"))
        ms, its, s2 = measure_device(case, max(2, args.steps // 2), 1, world)
        n = case.ncell
        out["ras_exact"] = {"value": n * max(2, args.steps // 2) / (ms / 1e3), "unit": UNIT,
                            "ms_per_step": ms / max(2, args.steps // 2),
                            "bicgstab_iters_per_step": its,
                            "note": "reference's RAS subdomain block-ILU(0), natural order, "
                                    "level-scheduled (same BiCGSTAB iteration counts as the "
                                    "reference)"}
        s2.ctx.close()
        del s2
    if rank == 0 and world == 1:
        if not args.no_spmv:
            try:
                out["spmv_c5"] = run_spmv_c5()
            except Exception as exc:  # report, never hide
                out["spmv_c5"] = {"error": repr(exc)}
        if not args.no_spmv:
            try:
                out["timesteps_c4"] = run_timesteps(args.config)
            except Exception as exc:  # report, never hide
                out["timesteps_c4"] = {"error": repr(exc)}
        if not args.no_spmv:
            try:
                out["numeric_jacobian_c4"] = run_numjac(args.config)
            except Exception as exc:  # report, never hide
                out["numeric_jacobian_c4"] = {"error": repr(exc)}
        if not args.no_spmv:
            try:
                out["report_frame_c4"] = run_report(args.config)
            except Exception as exc:  # report, never hide
                out["report_frame_c4"] = {"error": repr(exc)}
        if not args.no_cpu_baseline:
            cb = run_oracle(steps=CYCLE, warmup=0, config=args.config, budget_s=20.0)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
