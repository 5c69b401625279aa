"""Multi-rank z-slab decomposition validated on ONE GPU.

Several contexts (one per emulated rank, each with its own stream and host
thread) exchange halos and all-reduce Krylov scalars through the in-process
hub transport — the same library code path the NCCL transport drives on a
multi-GPU node, minus the transport itself. Compared against the
single-context solve of the whole grid:
  * the assembled residual of every owned cell is bit-identical;
  * du agrees to the Krylov tolerance and BiCGSTAB takes the single-GPU
    number of iterations (±1: reductions are summed per rank);
  * short Newton runs reproduce the single-GPU Newton sequence and fields.
"""

import ctypes

import numpy as np
import pytest
import torch

from paper_1811_11992_b200 import _native as N
from paper_1811_11992_b200 import configs
from paper_1811_11992_b200.device import DeviceContext, soa_from_rows, state_to_device
from paper_1811_11992_b200.distributed import Hub, attach_hub, split_case
from tests.golden_states import random_state_like_reference
from tests.helpers import case_objects

pytestmark = pytest.mark.gpu


def _slice_state(st, accn, piece, nxny):
    ka = piece.k0 - piece.g_lo
    kb = piece.k1 + piece.g_hi
    sl = slice(ka * nxny, kb * nxny)
    loc = configs.InitialState(st.p[sl].copy(), st.t[sl].copy(), st.sw[sl].copy(),
                               st.sg[sl].copy(), st.x[sl].copy(), st.y[sl].copy(),
                               st.cc[sl].copy(), st.bhp[list(piece.well_ids)].copy())
    return loc, accn[sl].copy()


def _single(c, st, accn, precond, tol, krylov="bicgstab"):
    ctx = DeviceContext(c.grid, c.pack, c.wells, c.streams, precond)
    ctx.set_krylov(krylov)
    wout = ctx.assemble(state_to_device(st, ctx.device), st.bhp, soa_from_rows(accn, ctx.device),
                        2e-3, 2e-3, np.zeros(len(c.wells), bool), False)
    resid = ctx.copy_out(0, 9).cpu().numpy()
    du = ctx.empty(9, c.grid.ncell)
    dbhp, it = ctx.solve(tol, 1000, du)
    out = (resid, du.cpu().numpy(), dbhp, it, wout)
    ctx.close()
    return out


@pytest.mark.parametrize("nranks,krylov", [(2, "bicgstab"), (3, "bicgstab"),
                                           (5, "bicgstab"),   # 5: ranks with one owned plane
                                           (2, "gmres"), (3, "gmres")])
def test_slab_assembly_and_solve_match_single_gpu(nranks, krylov):
    c = case_objects("sub2")
    st, accn = random_state_like_reference(c, 31)
    nxny = c.grid.nx * c.grid.ny
    ref_resid, ref_du, ref_dbhp, ref_it, ref_wout = _single(c, st, accn, "mcilu", 1e-10, krylov)

    hub = Hub(nranks)
    pieces = [split_case(c.case, nranks, r) for r in range(nranks)]
    ctxs = []
    for p in pieces:
        ctx = DeviceContext(p.grid, p.pack, p.wells, p.streams, "mcilu", own_stream=True)
        ctx.set_krylov(krylov)
        attach_hub(ctx, hub.h, p)
        ctxs.append(ctx)
    inputs = []
    for p, ctx in zip(pieces, ctxs):
        lst, lacc = _slice_state(st, accn, p, nxny)
        inputs.append((ctx, p, state_to_device(lst, ctx.device), lst.bhp,
                       soa_from_rows(lacc, ctx.device)))
    torch.cuda.synchronize()

    def rank_work(ctx, p, d_st, bhp, d_acc):
        wout = ctx.assemble(d_st, bhp, d_acc, 2e-3, 2e-3, np.zeros(len(p.wells), bool), False)
        resid = ctx.copy_out(0, 9).cpu().numpy()
        du = ctx.empty(9, p.grid.ncell)
        dbhp, it = ctx.solve(1e-10, 1000, du)
        ctx.synchronize()
        # the condensed form runs on the slabs too (compact.cu: ghost-plane
        # E_S and boundary Bc), under BiCGSTAB and GMRES
        assert ctx.condensed
        return resid, du.cpu().numpy(), dbhp, it, wout

    outs = hub.run(rank_work, inputs)
    its = set()
    for p, (resid, du, dbhp, it, wout) in zip(pieces, outs):
        own = p.owned_cells
        glob = own + (p.k0 - p.g_lo) * nxny
        np.testing.assert_array_equal(resid[:, own], ref_resid[:, glob])
        scale = np.linalg.norm(ref_du)
        assert np.linalg.norm(du[:, own] - ref_du[:, glob]) <= 1e-7 * scale
        for w_loc, w_glob in enumerate(p.well_ids):
            np.testing.assert_array_equal(wout[w_loc], ref_wout[w_glob])
            assert abs(dbhp[w_loc] - ref_dbhp[w_glob]) <= 1e-6 * max(1.0, abs(ref_dbhp[w_glob]))
        its.add(it)
    assert len(its) == 1           # every rank ran the same Krylov iterations
    # the red-eliminated solve with the owner ranks' boundary blocks in the
    # factor is the single-GPU iteration (up to the order of the reductions)
    assert abs(its.pop() - ref_it) <= 1, (ref_it,)
    for ctx in ctxs:
        ctx.close()
    hub.close()


@pytest.mark.parametrize("name,nsteps", [("c2", 4), ("c3", 6)])
def test_slab_newton_run_matches_single_gpu(name, nsteps):
    """C2 (20x20x5) / C3 (60x60x20, BASELINE's "1 and 2 GPUs" case) split over
    2 emulated ranks: timesteps with LINEAR_TOL 1e-10 give the single-GPU
    Newton counts and fields."""
    from dataclasses import replace
    from paper_1811_11992_b200.newton import Simulator
    case = configs.config(name)
    case = replace(case, solver=replace(case.solver, linear_tol=1e-10, precond="mcilu"),
                   schedule=replace(case.schedule, t_end=nsteps * case.schedule.dt_init))
    grid, pack, wells, streams, state = configs.build_case(case)
    ref = Simulator(grid, pack, wells, streams, state, case.schedule, case.solver)
    ref.advance()
    ref_state = ref.state.to_host()
    ref_newton = [s.newton for s in ref.steps]

    nranks = 2
    hub = Hub(nranks)
    pieces = [split_case(case, nranks, r) for r in range(nranks)]

    def rank_run(p):
        sim = Simulator(p.grid, p.pack, p.wells, p.streams, p.state, case.schedule, case.solver,
                        comm_setup=lambda ctx: attach_hub(ctx, hub.h, p), own_stream=True)
        sim.advance()
        sim.ctx.synchronize()
        return [s.newton for s in sim.steps], sim.state.to_host(), sim.cumulative_imbalance()

    outs = hub.run(rank_run, [(p,) for p in pieces])
    nxny = grid.nx * grid.ny
    for p, (newton, st, imb) in zip(pieces, outs):
        assert newton == ref_newton
        own = p.owned_cells
        glob = own + (p.k0 - p.g_lo) * nxny
        for f in ("p", "t", "sw", "sg"):
            a, b = st[f][own], ref_state[f][glob]
            assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)) <= 1e-6, f
        np.testing.assert_allclose(imb, ref.cumulative_imbalance(), rtol=1e-6, atol=1e-12)
    hub.close()


def test_allreduce_max_propagates_nan_from_one_rank():
    """The Newton norm's max over ranks keeps a NaN that only one rank sees
    (the reference's scaled_norm is NaN then and counts as growth,
    newton.py:284-289); sums propagate it too."""
    c = case_objects("sub2")
    nranks = 2
    hub = Hub(nranks)
    pieces = [split_case(c.case, nranks, r) for r in range(nranks)]
    ctxs = []
    for p in pieces:
        cx = DeviceContext(p.grid, p.pack, p.wells, p.streams, "mcilu", own_stream=True)
        attach_hub(cx, hub.h, p)
        ctxs.append(cx)

    def work(cx, r):
        mx = cx.allreduce_host([float("nan") if r == 1 else 3.0, 1.0 + r], "max")
        sm = cx.allreduce_host([float("nan") if r == 0 else 2.0, 1.0], "sum")
        return mx, sm

    res = hub.run(work, [(cx, r) for r, cx in enumerate(ctxs)])
    for mx, sm in res:
        assert np.isnan(mx[0]) and mx[1] == 2.0
        assert np.isnan(sm[0]) and sm[1] == 2.0
    for cx in ctxs:
        cx.close()
    hub.close()


def _export(ctx, grid):
    d = ctx.empty(grid.ncell, 9, 9)
    o = ctx.empty(grid.nconn, 2, 9, 9)
    r = ctx.empty(grid.ncell, 9)
    N.check(ctx.L.isc_export_system(ctx.h, N.ptr(d), N.ptr(o), N.ptr(r)), "export")
    return d.cpu().numpy(), o.cpu().numpy(), r.cpu().numpy()


@pytest.mark.parametrize("nranks", [2, 3])
def test_c5_slab_generator_and_solve_match_single_gpu(nranks):
    """BASELINE configs[4] on z-slabs: isc_synth_system_slab keys every value
    by the global cell index, so each rank holds exactly its rows of the
    single-GPU system (bit for bit), and the slab mcilu solve to 1e-8 takes
    the single-GPU BiCGSTAB iterations (+-1) and du (C5 grid scaled down)."""
    import ctypes
    case = configs.config("c5", nx=8, ny=6, nz=10)
    grid, pack, wells, streams, _ = configs.build_case(case)
    ctx = DeviceContext(grid, pack, (), (), "mcilu")
    N.check(ctx.L.isc_synth_system(ctx.h, 7), "synth")
    gd, go, gr = _export(ctx, grid)
    du1 = ctx.empty(9, grid.ncell)
    dbhp, it1 = ctx.solve(1e-8, 1000, du1)
    du1 = du1.cpu().numpy()
    ctx.close()
    gidx = {(int(a), int(b)): ic for ic, (a, b) in enumerate(zip(grid.conn_a, grid.conn_b))}
    nxny = grid.nx * grid.ny
    hub = Hub(nranks)
    pieces = [split_case(case, nranks, r) for r in range(nranks)]
    ctxs = []
    for p in pieces:
        cx = DeviceContext(p.grid, p.pack, (), (), "mcilu", own_stream=True)
        attach_hub(cx, hub.h, p)
        ctxs.append(cx)

    def rank_work(cx, p):
        N.check(cx.L.isc_synth_system_slab(cx.h, 7, case.nz), "synth slab")
        sysl = _export(cx, p.grid)
        du = cx.empty(9, p.grid.ncell)
        _, it = cx.solve(1e-8, 1000, du)
        cx.synchronize()
        return sysl, du.cpu().numpy(), it

    res = hub.run(rank_work, [(cx, p) for cx, p in zip(ctxs, pieces)])
    for p, ((ld, lo, lr), du, it) in zip(pieces, res):
        off = (p.k0 - p.g_lo) * nxny
        own = p.owned_cells
        np.testing.assert_array_equal(ld[own], gd[own + off])
        np.testing.assert_array_equal(lr[own], gr[own + off])
        ownset = set((own + off).tolist())
        for icl, (a, b) in enumerate(zip(p.grid.conn_a, p.grid.conn_b)):
            ga, gb = int(a) + off, int(b) + off
            ic = gidx[(ga, gb)]
            if ga in ownset:
                np.testing.assert_array_equal(lo[icl, 0], go[ic, 0])
            if gb in ownset:
                np.testing.assert_array_equal(lo[icl, 1], go[ic, 1])
        assert abs(it - it1) <= 1, (it, it1)
        ref = du1[:, own + off]
        assert np.linalg.norm(du[:, own] - ref) <= 1e-6 * np.linalg.norm(ref)
    for cx in ctxs:
        cx.close()
    hub.close()


def test_nccl_transport_one_rank(monkeypatch):
    """The NCCL transport itself on one GPU: a one-rank communicator
    (ISC_NCCL_SINGLE=1 makes the library create and use it; the
    dlopen binding of torch's NCCL, `ncclCommInitRank`, the packed
    `ncclAllReduce` of the Krylov scalars, the Newton norm and the host
    all-reduce) under the slab code path of the library — assembly, solve and
    norm equal the plain single-context run, and a NaN norm stays NaN through
    the reduction (NCCL's max alone would drop it). The halo send/recv needs
    a second GPU and stays with the hub tests above."""
    from paper_1811_11992_b200.distributed import attach_nccl, nccl_unique_id
    c = case_objects("sub2")
    st, accn = random_state_like_reference(c, 37)
    ref_resid, ref_du, ref_dbhp, ref_it, ref_wout = _single(c, st, accn, "mcilu", 1e-10)
    piece = split_case(c.case, 1, 0)
    assert piece.g_lo == 0 and piece.g_hi == 0 and piece.grid.ncell == c.grid.ncell
    ctx = DeviceContext(piece.grid, piece.pack, piece.wells, piece.streams, "mcilu")
    monkeypatch.setenv("ISC_NCCL_SINGLE", "1")
    attach_nccl(ctx, nccl_unique_id(), piece)
    assert N.lib().isc_comm_is_nccl(ctx.h) == 1
    d_accn = soa_from_rows(accn, ctx.device)
    wout = ctx.assemble(state_to_device(st, ctx.device), st.bhp, d_accn, 2e-3, 2e-3,
                        np.zeros(len(c.wells), bool), False)
    np.testing.assert_array_equal(ctx.copy_out(0, 9).cpu().numpy(), ref_resid)
    np.testing.assert_array_equal(wout, ref_wout)
    norm = ctx.scaled_norm_cells(d_accn, 2e-3)
    assert np.isfinite(norm) and norm > 0.0
    du = ctx.empty(9, c.grid.ncell)
    dbhp, it = ctx.solve(1e-10, 1000, du)
    assert abs(it - ref_it) <= 1
    a = du.cpu().numpy()
    assert np.linalg.norm(a - ref_du) <= 1e-8 * np.linalg.norm(ref_du)
    np.testing.assert_allclose(dbhp, ref_dbhp, rtol=1e-7)
    # a NaN residual on this rank survives the rank reduction
    bad = accn.copy()
    bad[3, 2] = np.nan
    ctx.assemble(state_to_device(st, ctx.device), st.bhp, soa_from_rows(bad, ctx.device), 2e-3,
                 2e-3, np.zeros(len(c.wells), bool), False)
    assert np.isnan(ctx.scaled_norm_cells(soa_from_rows(bad, ctx.device), 2e-3))
    ctx.close()
