"""CPU (gloo, world_size 2) checks of the z-slab decomposition logic.

Each process builds its slab (owned planes + ghost planes) with
`distributed.split_case`, assembles it with the CPU oracle, exchanges
boundary planes with its neighbour through torch.distributed (gloo) and
applies the assembled operator. Owned rows must equal the single-process
result: residual rows bit for bit, operator rows of A x to rounding, and
an all-reduced dot product. This is the algorithm the GPU ranks run with
NCCL (csrc/comm.cuh); the GPU hub tests cover the device kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_11992_b200 import configs
from paper_1811_11992_b200.distributed import split_case


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global(case):
    from oracle import isc_oracle as O
    from tests.golden_states import perturb
    grid, pack, wells, streams, state = configs.build_case(case)
    ws = O.Workspace(grid, pack)
    zero = np.zeros((grid.ncell, pack.nequ))
    O.assemble(grid, O.Model(pack), ws, wells, streams, state, zero, 1.0, 0.0,
               np.zeros(len(wells), bool))
    st, accn = perturb(state, ws.acc.copy(), 41)
    blocks = O.assemble(grid, O.Model(pack), ws, wells, streams, st, accn, 2e-3, 2e-3,
                        np.zeros(len(wells), bool))
    return grid, st, accn, ws, blocks


def _matvec(ws, grid, x):
    from oracle import isc_oracle as O
    other = np.where(ws.adj_sides == 0, grid.conn_b[ws.adj_ids],
                     grid.conn_a[ws.adj_ids]).astype(np.int64)
    out = np.zeros_like(x)
    import ctypes
    O.lib().orc_matvec(ctypes.c_int64(x.shape[0]), ctypes.c_int64(9), O._p(ws.diag),
                       O._p(ws.offd), O._p(ws.adj_ptr), O._p(ws.adj_ids), O._p(ws.adj_sides),
                       O._p(other), O._p(np.ascontiguousarray(x)), O._p(out))
    return out


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import isc_oracle as O
        case = configs.config("sub2")
        grid, st, accn, gws, gblocks = _global(case)
        piece = split_case(case, world, rank)
        nxny = grid.nx * grid.ny
        ka = piece.k0 - piece.g_lo
        sl = slice(ka * nxny, (piece.k1 + piece.g_hi) * nxny)
        lst = configs.InitialState(st.p[sl], st.t[sl], st.sw[sl], st.sg[sl], st.x[sl], st.y[sl],
                                   st.cc[sl], st.bhp[list(piece.well_ids)])
        lws = O.Workspace(piece.grid, piece.pack)
        lblocks = O.assemble(piece.grid, O.Model(piece.pack), lws, piece.wells, piece.streams,
                             lst, accn[sl], 2e-3, 2e-3, np.zeros(len(piece.wells), bool))
        own = piece.owned_cells
        glob = own + ka * nxny
        # 1) owned residual / diagonal rows are bit-identical to the global assembly
        np.testing.assert_array_equal(lws.resid[own], gws.resid[glob])
        np.testing.assert_array_equal(lws.diag[own], gws.diag[glob])
        for wl, wg in enumerate(piece.well_ids):
            assert lblocks[wl].resid == gblocks[wg].resid
        # 2) distributed operator: owned x + halo planes from the neighbours
        rng = np.random.default_rng(5)
        xg = rng.normal(size=(grid.ncell, 9))
        x = np.zeros((piece.grid.ncell, 9))
        x[own] = xg[glob]
        lo_plane, hi_plane = piece.kw_lo, piece.kw_hi - 1
        reqs = []
        recv_lo = torch.zeros(nxny * 9, dtype=torch.float64)
        recv_hi = torch.zeros(nxny * 9, dtype=torch.float64)
        if piece.g_lo:
            send = torch.from_numpy(x[lo_plane * nxny:(lo_plane + 1) * nxny].ravel().copy())
            reqs += [dist.isend(send, rank - 1), dist.irecv(recv_lo, rank - 1)]
        if piece.g_hi:
            send = torch.from_numpy(x[hi_plane * nxny:(hi_plane + 1) * nxny].ravel().copy())
            reqs += [dist.isend(send, rank + 1), dist.irecv(recv_hi, rank + 1)]
        for r in reqs:
            r.wait()
        if piece.g_lo:
            x[0:nxny] = recv_lo.numpy().reshape(nxny, 9)
        if piece.g_hi:
            k = piece.kw_hi
            x[k * nxny:(k + 1) * nxny] = recv_hi.numpy().reshape(nxny, 9)
        y = _matvec(lws, piece.grid, x)
        yg = _matvec(gws, grid, xg)
        np.testing.assert_allclose(y[own], yg[glob], rtol=1e-13, atol=1e-9)
        # 3) all-reduced dot product of owned rows == global dot
        d = torch.tensor([float(np.sum(y[own] * x[own]))], dtype=torch.float64)
        dist.all_reduce(d)
        np.testing.assert_allclose(d.item(), float(np.sum(yg * xg)), rtol=1e-12)
        dist.destroy_process_group()
    except BaseException as exc:  # report to the parent
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def test_split_case_tiles_the_grid():
    case = configs.config("sub2")
    grid, *_ = configs.build_case(case)
    nxny = grid.nx * grid.ny
    for world in (1, 2, 3):
        owned, wells = [], []
        for r in range(world):
            p = split_case(case, world, r)
            ka = p.k0 - p.g_lo
            owned.append(p.owned_cells + ka * nxny)
            wells += list(p.well_ids)
            np.testing.assert_array_equal(p.grid.depth, grid.depth[ka * nxny:ka * nxny +
                                                                   p.grid.ncell])
            np.testing.assert_array_equal(p.grid.phi_ref, grid.phi_ref[ka * nxny:ka * nxny +
                                                                       p.grid.ncell])
        np.testing.assert_array_equal(np.concatenate(owned), np.arange(grid.ncell))
        assert sorted(wells) == list(range(len(case.wells)))


@pytest.mark.timeout(300)
def test_two_rank_gloo_slab_operator():
    world = 2
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
