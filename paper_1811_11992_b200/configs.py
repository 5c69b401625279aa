"""The BASELINE.json configurations as seeded synthetic cases.

BASELINE.json leaves several inputs open (SURVEY §7 hard part 8); the
choices made here are used identically on the reference side (the golden
generator writes them into decks) and on ours:

* fluid: the reference's ``tube.deck`` fluid with the light-oil oxidation
  reaction removed -> 3 reactions (heavy-oil oxidation, cracking, coke burn);
  stored as ``data/tube3_pack.json`` (exported from the reference's
  ``build_pack`` by tools/export_pack.py);
* initial state p 2014.7 psi, T 68 °F, Sw 0.2, So 0.799, Sg 0.001
  (BASELINE's Sg = 0 raises SingularCellBlock at t = 0 on the reference),
  x = (0.744, 0.256), y = (0.21, 0.79), C_c = 0;
* heterogeneous cases: PERMX = PERMY = exp(N(ln 500, 1.0)), PERMZ = 0.1·PERMX,
  phi_ref ~ U(0.25, 0.35) drawn in that order from ``default_rng(seed)``;
* fixed timestep (DTINIT = DTMAX = dt) with the heater stop and report
  interval on multiples of dt so every case takes exactly ``nsteps`` steps.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional, Tuple

import numpy as np

from .grid import build_grid
from .model import load_pack
from .wells import WellSpec, build_streams, build_wells, CTRL_BHP

CM_IN_FT = 0.03280839895013123


@dataclass(frozen=True)
class Schedule:
    t_end: float
    dt_init: float
    dt_min: float
    dt_max: float
    report_interval: Optional[float] = None
    report_times: Tuple[float, ...] = ()


@dataclass(frozen=True)
class SolverSettings:
    newton_tol: float = 1e-4
    newton_max: int = 15
    linear_tol: float = 1e-5
    linear_max: int = 200
    precond: str = "ras"
    eps: float = 1e-4
    krylov: str = "bicgstab"   # mcilu only: "gmres" = restarted GMRES(gmres_restart)
    gmres_restart: int = 30


@dataclass(frozen=True)
class InitSpec:
    p: float = 2014.7
    t: float = 68.0
    s_w: float = 0.2
    s_g: float = 0.001
    x: Tuple[float, ...] = (0.744, 0.256)
    y: Tuple[float, ...] = (0.21, 0.79)
    c_c: float = 0.0


@dataclass(frozen=True)
class HeatLoss:
    """Overburden heat loss (deck.py:131-135 ``HeatLossSpec``, the *ROCK
    ``HEATLOSS kob d rho tini`` row); applied on the top and bottom layers
    (grid.py:189-206, _kernels.py:821-825)."""

    k_ob: float
    distance: float
    rho: float
    t_initial: float


@dataclass(frozen=True)
class Case:
    name: str
    nx: int
    ny: int
    nz: int
    d: Tuple[float, float, float]
    wells: Tuple[WellSpec, ...]
    schedule: Schedule
    solver: SolverSettings = SolverSettings()
    init: InitSpec = InitSpec()
    seed: Optional[int] = None          # None: homogeneous rock
    perm: float = 1000.0                # homogeneous perm (md)
    phi: float = 0.3                    # homogeneous porosity
    pack: str = "tube3_pack"
    nsteps: int = 0
    heat_loss: Optional[HeatLoss] = None

    @property
    def ncell(self) -> int:
        return self.nx * self.ny * self.nz

    def rock_arrays(self):
        """(permx, permy, permz, phi) per cell, seeded as documented above."""
        n = self.ncell
        if self.seed is None:
            k = np.full(n, self.perm)
            return k, k.copy(), k.copy(), np.full(n, self.phi)
        rng = np.random.default_rng(self.seed)
        kh = np.exp(rng.normal(np.log(500.0), 1.0, n))
        phi = rng.uniform(0.25, 0.35, n)
        return kh, kh.copy(), 0.1 * kh, phi


def _fixed_schedule(nsteps: int, dt: float) -> Schedule:
    return Schedule(t_end=nsteps * dt, dt_init=dt, dt_min=1e-7, dt_max=dt,
                    report_interval=nsteps * dt)


def _air_injector(name, i, j, k, rate, heat_rate=0.0, heat_stop=0.0, wi=None,
                  radius=None, tinj=68.0):
    return WellSpec(name=name, kind="injector", i=i, j=j, k=k, control="rate_gas",
                    rate=rate, rate_conditions="standard", wi=wi, radius=radius,
                    yinj=(0.21, 0.79), tinj=tinj, pinjmax=10000.0,
                    heat_rate=heat_rate, heat_stop=heat_stop)


def _bhp_producer(name, i, j, k, bhp=2014.7, wi=None, radius=None):
    return WellSpec(name=name, kind="producer", i=i, j=j, k=k, control="bhp",
                    bhp=bhp, wi=wi, radius=radius)


def config(name: str, **overrides) -> Case:
    """C1..C4 of BASELINE.json (+ a small 3D case for tests).

    C2 variants that switch on the reference's less common branches:

    * ``c2hl``   — overburden heat loss with the reference deck's own row
      (decks/heatloss.deck:23, ``HEATLOSS 24.0 50.0 42.0 100.0``);
    * ``c2cap``  — injector pressure cap 2450 psi: the injector caps and is
      released again inside Newton iterations (newton.py:147-168), steps fail
      on the Newton limit and are cut, and the run ends capped
      (the well equation ``bhp - pinjmax``, assembly.py:515-516);
    * ``c2rate`` — the producer on total-rate control (``RATE_TOTAL -10``
      lbmol/day, the ``qsum - target`` equation, assembly.py:518-520).
    """
    if name in ("c2hl", "c2cap", "c2rate"):
        base = config("c2")
        if name == "c2hl":
            case = replace(base, name=name, heat_loss=HeatLoss(24.0, 50.0, 42.0, 100.0))
        elif name == "c2cap":
            inj, prod = base.wells
            case = replace(base, name=name, wells=(replace(inj, pinjmax=2450.0), prod))
        else:
            inj, prod = base.wells
            case = replace(base, name=name,
                           wells=(inj, replace(prod, control="rate_total", rate=-10.0, bhp=None)))
        return _apply_overrides(case, overrides)
    if name == "c5":
        # BASELINE configs[4]: the linear-solver microbench grid (400x400x100,
        # 16 M block rows). Only the grid matters: the system is the seeded
        # synthetic BSR of synth.py / isc_synth_system(_slab), decoupled and
        # solved with the multicolour ILU(0) + BiCGSTAB to 1e-8.
        case = Case(name="c5", nx=400, ny=400, nz=100, d=(1.0, 1.0, 1.0), wells=(),
                    schedule=_fixed_schedule(1, 1.0),
                    solver=SolverSettings(linear_tol=1e-8, linear_max=1000, precond="mcilu"),
                    perm=1.0, phi=0.3, nsteps=1)
        return _apply_overrides(case, overrides)
    if name == "c1":
        nsteps, dt = 50, 5e-4
        case = Case(
            name="c1", nx=100, ny=1, nz=1, d=(CM_IN_FT,) * 3,
            wells=(_air_injector("INJ", 1, 1, 1, 0.0230, heat_rate=30.0,
                                 heat_stop=0.02, wi=1.0, tinj=70.0),
                   _bhp_producer("PROD", 100, 1, 1, wi=1.0)),
            schedule=_fixed_schedule(nsteps, dt), perm=1000.0, phi=0.3, nsteps=nsteps)
    elif name in ("c2", "c3", "small3d", "sub2"):
        nx, ny, nz = {"c2": (20, 20, 5), "c3": (60, 60, 20), "small3d": (8, 6, 4),
                      "sub2": (32, 16, 8)}[name]
        nsteps, dt = 20, 2e-3
        case = Case(
            name=name, nx=nx, ny=ny, nz=nz, d=(10.0, 10.0, 2.0),
            wells=(_air_injector("INJ", 1, 1, nz, 5000.0, heat_rate=2.0e6,
                                 heat_stop=0.01, radius=0.25),
                   _bhp_producer("PROD", nx, ny, nz, radius=0.25)),
            schedule=_fixed_schedule(nsteps, dt), seed=1234, nsteps=nsteps)
    elif name == "c4":
        nx, ny, nz = 200, 200, 50
        nsteps, dt = 5, 2e-3
        wells = []
        for w, j in enumerate((25, 75, 125, 175)):
            wells.append(_air_injector(f"INJ{w}", 1, j, nz, 5000.0, heat_rate=2.0e6,
                                       heat_stop=0.01, radius=0.25))
            wells.append(_bhp_producer(f"PROD{w}", nx, j, nz, radius=0.25))
        case = Case(name="c4", nx=nx, ny=ny, nz=nz, d=(10.0, 10.0, 2.0),
                    wells=tuple(wells), schedule=_fixed_schedule(nsteps, dt),
                    seed=1234, nsteps=nsteps)
    else:
        raise KeyError(f"unknown config {name!r}")
    return _apply_overrides(case, overrides)


def _apply_overrides(case: Case, overrides) -> Case:
    solver = overrides.pop("solver", None)
    if solver is not None:
        case = replace(case, solver=solver)
    if overrides:
        case = replace(case, **overrides)
    return case


@dataclass
class InitialState:
    """Primary unknowns (assembly.py:179-196 ``State``)."""

    p: np.ndarray
    t: np.ndarray
    sw: np.ndarray
    sg: np.ndarray
    x: np.ndarray
    y: np.ndarray
    cc: np.ndarray
    bhp: np.ndarray

    def copy(self) -> "InitialState":
        return InitialState(*(np.array(getattr(self, f)) for f in
                              ("p", "t", "sw", "sg", "x", "y", "cc", "bhp")))


def initial_state(case: Case, grid, wells) -> InitialState:
    """Uniform initial conditions, rate-well bhp at reservoir p (assembly.py:199-215)."""
    n = grid.ncell
    ini = case.init
    bhp = np.array([w.target if w.control == CTRL_BHP else ini.p for w in wells],
                   dtype=np.float64)
    return InitialState(
        p=np.full(n, ini.p), t=np.full(n, ini.t), sw=np.full(n, ini.s_w),
        sg=np.full(n, ini.s_g),
        x=np.tile(np.asarray(ini.x, dtype=np.float64), (n, 1)),
        y=np.tile(np.asarray(ini.y, dtype=np.float64), (n, 1)),
        cc=np.full(n, ini.c_c), bhp=bhp)


def build_case(case: Case):
    """(grid, pack, wells, streams, state) for a case, no reference needed."""
    kx, ky, kz, phi = case.rock_arrays()
    grid = build_grid(case.nx, case.ny, case.nz, case.d[0], case.d[1], case.d[2],
                      kx, ky, kz, phi)
    pack = load_pack(case.pack, grid.phi_ref)
    wells = build_wells(case.wells, grid)
    streams = build_streams(pack, wells)
    state = initial_state(case, grid, wells)
    return grid, pack, wells, streams, state
