"""GPU Newton driver: the reference ``Simulator`` with a device-resident state.

Control flow restates newton.py:183-437 verbatim — check-first Newton
iterations with upwind freezing after iteration 5, divergence guard,
capped-injector switching, adaptive timestep with cuts on the reference's
exception set, forced times, conservation audit — while every per-cell
array stays in HBM: the state is a (9, n) SoA tensor, ``apply_update``
and the cell part of ``scaled_norm`` and ``audit_step`` run as kernels
(SURVEY §8(f) #1), and only per-well scalars cross PCIe each iteration.
"""

from __future__ import annotations

import math
import time as _time
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np
import torch

from .assembly import WellBlock, blocks_from_wout
from .device import DeviceContext, state_to_device
from .errors import (Breakdown, DegenerateTemperature, DivergedResidual, MaxIterations,
                     PoreSpaceExhausted, SimulationStalled, SingularCellBlock)
from .wells import CTRL_BHP, INJECTOR

GROWTH_FACTOR = 2.0
CUT_FACTOR = 0.5
FAST_ITERS = 4
FREEZE_UPWIND_AFTER = 5
_TIME_EPS = 1e-9
NU = 9


@dataclass
class DeviceState:
    """(9, n) SoA cell unknowns on the GPU + host bhp per well."""

    u: torch.Tensor
    bhp: np.ndarray

    def copy(self) -> "DeviceState":
        return DeviceState(self.u.clone(), self.bhp.copy())

    def to_host(self):
        """numpy views in the reference's State field layout."""
        a = self.u.cpu().numpy()
        return dict(p=a[0].copy(), x=a[1:3].T.copy(), y=a[3:5].T.copy(), t=a[5].copy(),
                    sw=a[6].copy(), sg=a[7].copy(), cc=a[8].copy(), bhp=self.bhp.copy())


@dataclass
class StepRecord:
    time: float
    dt: float
    newton: int
    linear: int
    solves: int
    balance: float


class TimestepController:
    """newton.py:183-211"""

    def __init__(self, dt, dt_min, dt_max):
        self.dt, self.dt_min, self.dt_max = dt, dt_min, dt_max

    def propose(self, t, forced):
        dt = min(self.dt, self.dt_max)
        for ft in forced:
            if ft > t + _TIME_EPS:
                dt = min(dt, ft - t)
                break
        return dt

    def on_success(self, iters):
        if iters <= FAST_ITERS:
            self.dt = min(self.dt * GROWTH_FACTOR, self.dt_max)

    def on_failure(self, attempted, t, reason):
        if attempted <= self.dt_min * (1.0 + 1e-9):
            raise SimulationStalled(
                f"timestep {attempted:g} at t={t:g} failed ({reason}) and is already at the "
                f"minimum {self.dt_min:g}")
        self.dt = max(attempted * CUT_FACTOR, self.dt_min)


def desired_capped(wells, capped, bhp, blocks):
    """newton.py:147-168"""
    want = capped.copy()
    for w, well in enumerate(wells):
        if well.kind != INJECTOR or well.control == CTRL_BHP:
            continue
        if not math.isfinite(well.pinjmax):
            continue
        if capped[w]:
            if float(np.sum(blocks[w].phase_rates)) > well.target:
                want[w] = False
        elif bhp[w] > well.pinjmax:
            want[w] = True
    return want


class Simulator:
    """Device-resident mirror of the reference ``Simulator`` (newton.py:214-437)."""

    def __init__(self, grid, pack, wells, streams, state, schedule, solver, heat_loss=None,
                 comm_setup=None, own_stream: bool = False, jacobian: str = "analytic"):
        self.grid, self.pack = grid, pack
        self.wells, self.streams = tuple(wells), tuple(streams)
        self.schedule, self.solver_cfg = schedule, solver
        self.jacobian = jacobian   # "numeric": FD blocks every iteration (newton.py:228,278)
        self.ctx = DeviceContext(grid, pack, self.wells, self.streams, solver.precond, heat_loss,
                                 own_stream=own_stream)
        if getattr(solver, "krylov", "bicgstab") != "bicgstab":
            self.ctx.set_krylov(solver.krylov, getattr(solver, "gmres_restart", 0))
        if comm_setup is not None:   # z-slab rank: window + NCCL/hub transport
            comm_setup(self.ctx)
        dev = self.ctx.device
        self.own_stream = own_stream
        self.state = DeviceState(state_to_device(state, dev), np.asarray(state.bhp, dtype=float))
        self.capped = np.zeros(len(self.wells), dtype=bool)
        self.time = 0.0
        self.du = self.ctx.empty(NU, grid.ncell)
        zero = torch.zeros(NU, grid.ncell, dtype=torch.float64, device=dev)
        self._torch_sync()
        self.blocks: List[WellBlock] = self._assemble(self.state, zero, 1.0, 0.0, self.capped,
                                                      False, analytic=True)
        self.accn = self.ctx.copy_out(1, NU)
        self.steps: List[StepRecord] = []
        self.cum_rates = np.zeros((len(self.wells), 3))
        self.cum_imbalance = np.zeros(pack.nfull + 1)
        self.cum_throughput = np.zeros(pack.nfull + 1)
        self.work_seconds = 0.0
        self.assemble_calls = 0
        self.solve_calls = 0

    # -- device operations ------------------------------------------------------
    def _torch_sync(self):
        """Library on its own stream: wait for torch-side producers first."""
        if self.own_stream:
            torch.cuda.current_stream().synchronize()

    def _assemble(self, st: DeviceState, accn, dt, t_new, capped, freeze, analytic=False):
        wout = self.ctx.assemble(st.u, st.bhp, accn, dt, t_new, capped, freeze)
        if self.jacobian == "numeric" and not analytic:
            wout = self.ctx.numeric_jacobian()
        return blocks_from_wout(self.wells, wout)

    def scaled_norm(self, blocks, dt, capped) -> float:
        """newton.py:124-144: cell rows on the device, well rows on the host."""
        norm = self.ctx.scaled_norm_cells(self.accn, dt)   # max over ranks
        wn = 0.0
        for w, (well, blk) in enumerate(zip(self.wells, blocks)):
            target = well.pinjmax if capped[w] else well.target
            wn = max(wn, abs(blk.resid) / max(1.0, abs(target)))
        wn = float(self.ctx.allreduce_host([wn], "max")[0])   # wells live on their owner rank
        return max(norm, wn)

    def newton_iteration(self, work: DeviceState, dt, t_new, capped, it: int = 1):
        """One solving Newton iteration — the body of newton_step's loop
        (newton.py:275-309) for an iteration that does not converge: assemble
        (upwinding frozen after iteration 5), scaled norm, capped-injector
        check, solve, damped update. The benchmark's unit of work; returns
        (scaled norm, BiCGSTAB iterations)."""
        cfg = self.solver_cfg
        blocks = self._assemble(work, self.accn, dt, t_new, capped, it > FREEZE_UPWIND_AFTER)
        norm = self.scaled_norm(blocks, dt, capped)
        desired_capped(self.wells, capped, work.bhp, blocks)
        dbhp, iters = self.ctx.solve(cfg.linear_tol, cfg.linear_max, self.du)
        self.ctx.newton_update(work.u, self.du, cfg.eps)
        work.bhp = work.bhp + dbhp
        return norm, iters

    def newton_step(self, state: DeviceState, dt: float, t_new: float, capped: np.ndarray):
        """newton.py:254-310"""
        cfg = self.solver_cfg
        work = state.copy()
        self._torch_sync()
        capped = capped.copy()
        lin_total = solves = growths = 0
        prev = math.inf
        for it in range(1, cfg.newton_max + 1):
            t0 = _time.perf_counter()
            blocks = self._assemble(work, self.accn, dt, t_new, capped,
                                    it > FREEZE_UPWIND_AFTER)
            self.assemble_calls += 1
            self.work_seconds += _time.perf_counter() - t0
            norm = self.scaled_norm(blocks, dt, capped)
            if not math.isfinite(norm) or norm > prev:
                growths += 1
                if growths >= 3:
                    raise DivergedResidual(
                        f"residual grew {growths} consecutive iterations (now {norm:g}) "
                        f"at t={t_new:g}")
            else:
                growths = 0
            if math.isfinite(norm):
                prev = norm
            want = desired_capped(self.wells, capped, work.bhp, blocks)
            switched = float(not np.array_equal(want, capped))
            if self.ctx.allreduce_host([switched], "max")[0] > 0.0:   # collective decision
                capped = want
                continue
            if norm <= cfg.newton_tol:
                self.blocks = blocks
                return work, True, it, lin_total, solves, capped
            if it == cfg.newton_max:
                break
            t0 = _time.perf_counter()
            dbhp, iters = self.ctx.solve(cfg.linear_tol, cfg.linear_max, self.du)
            self.work_seconds += _time.perf_counter() - t0
            self.solve_calls += 1
            lin_total += iters
            solves += 1
            self.ctx.newton_update(work.u, self.du, cfg.eps)
            work.bhp = work.bhp + dbhp
        return state, False, cfg.newton_max, lin_total, solves, capped

    def report_times(self):
        s = self.schedule
        times = set(t for t in s.report_times if 0.0 <= t <= s.t_end + _TIME_EPS)
        if s.report_interval:
            nrep = int(math.floor(s.t_end / s.report_interval + _TIME_EPS))
            times.update(k * s.report_interval for k in range(1, nrep + 1))
        times.add(s.t_end)
        return sorted(times)

    def forced_times(self):
        s = self.schedule
        times = set(rt for rt in self.report_times() if rt > _TIME_EPS)
        for well in self.wells:
            if well.heat_rate and 0.0 < well.heat_stop < s.t_end:
                times.add(well.heat_stop)
        times.add(s.t_end)
        return sorted(times)

    def audit_step(self, dt: float) -> float:
        """newton.py:339-366 with the per-cell sums reduced on the device."""
        nf = self.pack.nfull
        rows = list(range(nf)) + [self.pack.nequ - 1]
        sums = self.ctx.audit_sums(self.accn)
        worst = 0.0
        wq = np.zeros((2, len(rows)))
        for k, r in enumerate(rows):
            for blk in self.blocks:
                q = float(np.sum(blk.comp_rates[:, r]))
                wq[0, k] += q
                wq[1, k] += abs(q)
        wq = self.ctx.allreduce_host(wq, "sum").reshape(2, len(rows))
        for k, r in enumerate(rows):
            dacc, reac, absacc = sums[0, k], sums[1, k], sums[2, k]
            wellq, wellabs = wq[0, k], wq[1, k]
            imb = dacc - dt * (reac + wellq)
            worst = max(worst, abs(imb) / max(1.0, absacc))
            self.cum_imbalance[k] += imb
            self.cum_throughput[k] += dt * (wellabs + abs(reac))
        return worst

    def advance(self, log_cb: Optional[Callable[[str], None]] = None) -> None:
        """newton.py:373-431 (report frames are out of scope)."""
        s = self.schedule
        ctrl = TimestepController(s.dt_init, s.dt_min, s.dt_max)
        forced = self.forced_times()
        while self.time < s.t_end - _TIME_EPS:
            dt = ctrl.propose(self.time, forced)
            t_new = self.time + dt
            for ft in forced:
                if abs(t_new - ft) <= _TIME_EPS:
                    t_new = ft
                    break
            dt = t_new - self.time
            try:
                state, ok, iters, lin, solves, capped = self.newton_step(
                    self.state, dt, t_new, self.capped)
                reason = "" if ok else "newton iteration limit"
            except (DivergedResidual, SingularCellBlock, Breakdown, MaxIterations,
                    PoreSpaceExhausted, DegenerateTemperature) as exc:
                if not self.steps and isinstance(exc, PoreSpaceExhausted):
                    raise
                ok, iters, lin, solves = False, 0, 0, 0
                reason = f"{type(exc).__name__}: {exc}"
            if not ok:
                if log_cb:
                    log_cb(f"t={self.time:<12.6g} dt={dt:<10.4g} rejected ({reason})")
                ctrl.on_failure(dt, self.time, reason or "no convergence")
                continue
            self.state, self.capped, self.time = state, capped, t_new
            balance = self.audit_step(dt)
            self.accn = self.ctx.copy_out(1, NU)
            for w, blk in enumerate(self.blocks):
                self.cum_rates[w] += dt * blk.phase_rates.sum(axis=0)
            self.steps.append(StepRecord(time=t_new, dt=dt, newton=iters, linear=lin,
                                         solves=solves, balance=balance))
            if log_cb:
                log_cb(f"t={t_new:<12.6g} dt={dt:<10.4g} newton={iters:<3d} linear={lin}")
            ctrl.on_success(iters)

    def totals(self):
        return (len(self.steps), sum(s.newton for s in self.steps),
                sum(s.linear for s in self.steps))

    def cumulative_imbalance(self) -> float:
        return float(np.max(np.abs(self.cum_imbalance) / np.maximum(1.0, self.cum_throughput)))
