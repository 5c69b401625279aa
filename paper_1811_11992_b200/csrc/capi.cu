// C-ABI (include/iscgpu.h): context creation, assembly, decoupling,
// preconditioner setup, solve, Newton bookkeeping and report entry points.
// One translation unit: the kernel files (*.cu) and the host runtime pieces
// (runtime.cuh, ilu_build.cuh, comm_runtime.cuh, krylov.cuh) are included.
#include "runtime.cuh"
#include "ilu_build.cuh"

// --------------------------------------------------------------- create

extern "C" const char* isc_last_error(void) { return g_err.c_str(); }
extern "C" int isc_block_size(void) { return NU; }

extern "C" int isc_create(const isc_model_desc* md, const isc_grid_desc* gdsc, int32_t nwells,
                          const isc_well_desc* wells, int32_t precond, isc_ctx** out) {
  if (!md || !gdsc || !out) { g_err = "null argument"; return ISC_BAD_ARGUMENT; }
  if (md->nco != NCO || md->ncg != NCG) {
    g_err = "library compiled for nco=2, ncg=2 (block size 9)";
    return ISC_UNSUPPORTED;
  }
  if (md->nreac > MAXREAC || md->nswt > MAXTAB || md->nslt > MAXTAB || md->nswt < 1 ||
      md->nslt < 1) {
    g_err = "model tables exceed compiled limits";
    return ISC_UNSUPPORTED;
  }
  if (precond < 0 || precond > 3) { g_err = "unknown preconditioner"; return ISC_BAD_ARGUMENT; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_err = "no CUDA device";
    return ISC_CUDA_ERROR;
  }
  isc_ctx* ctx = new isc_ctx();
  ctx->precond = precond;
  {
    const char* e = std::getenv("ISC_MCILU_FULL");   // A/B switch for the full-system form
    ctx->mc_schur = !(e && e[0] == '1');
    const char* e2 = std::getenv("ISC_COMPACT");
    ctx->compact_ok = !(e2 && e2[0] == '0');
    const char* e3 = std::getenv("ISC_COND");
    ctx->cond_ok = !(e3 && e3[0] == '0');
  }
  Dims& g = ctx->g;
  g.nx = gdsc->nx; g.ny = gdsc->ny; g.nz = gdsc->nz;
  g.nxny = (int64_t)g.nx * g.ny;
  g.n = g.nxny * g.nz;
  g.colored = (g.nx % 2 == 0) ? 1 : 0;
  g.half = g.n / 2;
  g.kpar = gdsc->k_offset & 1;
  ctx->k_offset = gdsc->k_offset;
  g.tw_lo = 0;
  g.tw_hi = g.half;
  g.ph = g.nxny / 2;
  g.kw_lo = 0;
  g.kw_hi = g.nz;
  const int64_t n = g.n;
  // model
  Model& M = ctx->M;
  std::memset(&M, 0, sizeof(M));
  std::memcpy(M.liq, md->liq, sizeof(M.liq));
  std::memcpy(M.gasp, md->gasp, sizeof(M.gasp));
  std::memcpy(M.kv, md->kv, sizeof(M.kv));
  std::memcpy(M.rockp, md->rockp, sizeof(M.rockp));
  for (int i = 0; i < md->nswt; ++i) {
    M.swt_s[i] = md->swt_s[i]; M.swt_krw[i] = md->swt_krw[i];
    M.swt_krow[i] = md->swt_krow[i]; M.swt_pcow[i] = md->swt_pcow[i];
  }
  for (int i = 0; i < md->nslt; ++i) {
    M.slt_s[i] = md->slt_s[i]; M.slt_krg[i] = md->slt_krg[i];
    M.slt_krog[i] = md->slt_krog[i]; M.slt_pcog[i] = md->slt_pcog[i];
  }
  M.nreac = (int)md->nreac; M.nswt = (int)md->nswt; M.nslt = (int)md->nslt;
  M.heavy = (int)md->heavy; M.ccmax = md->ccmax;
  for (int q = 0; q < md->nreac; ++q) {
    for (int k = 0; k < 3; ++k) M.rcoef[q][k] = md->rcoef[q * 3 + k];
    for (int a = 0; a <= NF; ++a) M.nmat[a][q] = md->nmat[a * md->nreac + q];
    M.law[q] = (int)md->law[q]; M.fuel[q] = (int)md->fuel[q]; M.ox[q] = (int)md->ox[q];
  }
  CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  for (auto& e : ctx->chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
  for (auto& e : ctx->cell_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : ctx->face_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : ctx->halo_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
  // static grid arrays
  ALLOC(ctx->depth, n * 8); ALLOC(ctx->vol, n * 8); ALLOC(ctx->phi_ref, n * 8);
  ALLOC(ctx->gd, 3 * n * 8); ALLOC(ctx->td, 3 * n * 8); ALLOC(ctx->conn_id, 3 * n * 8);
  {
    // per-cell static arrays in storage order (common.cuh: colour-blocked)
    std::vector<int64_t> pos(n);
    for (int64_t c = 0; c < n; ++c) pos[c] = pos_of(g, c);
    std::vector<double> tmp((size_t)3 * n);
    auto put = [&](double* dst, const double* src, int rows) -> int {
      for (int r = 0; r < rows; ++r)
        for (int64_t c = 0; c < n; ++c) tmp[(size_t)r * n + pos[c]] = src[(size_t)r * n + c];
      return cudaMemcpy(dst, tmp.data(), (size_t)rows * n * 8, cudaMemcpyHostToDevice) ==
                     cudaSuccess ? 0 : ISC_CUDA_ERROR;
    };
    if (put(ctx->depth, gdsc->depth, 1) || put(ctx->vol, gdsc->volume, 1) ||
        put(ctx->phi_ref, gdsc->phi_ref, 1) || put(ctx->gd, gdsc->gd, 3) ||
        put(ctx->td, gdsc->td, 3)) {
      g_err = "static array upload failed";
      return ISC_CUDA_ERROR;
    }
    CK(cudaMemcpy(ctx->conn_id, gdsc->conn_id, 3 * n * 8, cudaMemcpyHostToDevice));
    if (gdsc->hl_area) {
      ALLOC(ctx->hl_area, n * 8);
      if (put(ctx->hl_area, gdsc->hl_area, 1)) return ISC_CUDA_ERROR;
    }
  }
  ALLOC(ctx->st_c, (size_t)NU * n * 8);
  ALLOC(ctx->stage, (size_t)2 * NU * n * 8);
  ALLOC(ctx->accn_c, (size_t)NU * n * 8);
  ctx->hl_kob = gdsc->hl_kob; ctx->hl_d = gdsc->hl_d; ctx->hl_rho = gdsc->hl_rho;
  ctx->hl_tini = gdsc->hl_tini;
  // wells
  ctx->nw = nwells;
  if (nwells > 0) {
    std::vector<WellDev> wd(nwells);
    for (int w = 0; w < nwells; ++w) {
      const isc_well_desc& s = wells[w];
      WellDev& d = wd[w];
      if (s.cell < 0 || s.cell >= n) { g_err = "well cell out of range"; return ISC_BAD_ARGUMENT; }
      d.cell = s.cell; d.kind = s.kind; d.control = s.control; d.target = s.target;
      d.wi = s.wi; d.z_bh = s.z_bh; d.pinjmax = s.pinjmax; d.heat_rate = s.heat_rate;
      d.heat_stop = s.heat_stop;
      for (int a = 0; a < NF; ++a) d.s_yfull[a] = s.s_yfull[a];
      for (int j = 0; j < NCG; ++j) d.s_yinj[j] = s.s_yinj[j];
      d.s_tinj = s.s_tinj; d.s_mu = s.s_mu; d.s_h = s.s_h; d.s_mbar = s.s_mbar;
      ctx->wcell_h.push_back(s.cell);
      ctx->wpos_h.push_back(pos_of(g, s.cell));
      d.cell = pos_of(g, s.cell);
    }
    ALLOC(ctx->wells_d, nwells * sizeof(WellDev));
    CK(cudaMemcpy(ctx->wells_d, wd.data(), nwells * sizeof(WellDev), cudaMemcpyHostToDevice));
    ALLOC(ctx->wcell_d, nwells * 8);
    CK(cudaMemcpy(ctx->wcell_d, ctx->wpos_h.data(), nwells * 8, cudaMemcpyHostToDevice));
  }
  ALLOC(ctx->wout_d, std::max(1, nwells) * WOUT * 8);
  CK(cudaMallocHost(&ctx->wout_h, std::max(1, nwells) * WOUT * 8));
  ALLOC(ctx->bhp_d, std::max(1, nwells) * 8);
  ALLOC(ctx->capped_d, std::max(1, nwells));
  // assembly buffers
  ALLOC(ctx->rec, (size_t)NREC * n * 8);
  ALLOC(ctx->cmid, (size_t)NMID * n * 8);
  ALLOC(ctx->fbuf, (size_t)3 * ROW_OS * n * 8);
  ALLOC(ctx->acc, (size_t)NU * n * 8);
  ALLOC(ctx->src, (size_t)NU * n * 8);
  ALLOC(ctx->resid, (size_t)NU * n * 8);
  ALLOC(ctx->diag, (size_t)NB * n * 8);
  ALLOC(ctx->offd, (size_t)NDIR * NB * n * 8);
  ALLOC(ctx->upw, (size_t)9 * n);
  CK(cudaMemset(ctx->upw, 0, (size_t)9 * n));
  ALLOC(ctx->bad_d, 8);
  ALLOC(ctx->ticket_d, 4);
  ALLOC(ctx->wdu_d, std::max(1, nwells) * NU * 8);
  CK(cudaMallocHost(&ctx->wdu_h, std::max(1, nwells) * NU * 8));
  CK(cudaMemset(ctx->ticket_d, 0, 4));
  CK(cudaMallocHost(&ctx->bad_h, 16));   // [0] bad cell (cell pass / decoupling), [1] factor status
  // solver vectors
  double** vecs[] = {&ctx->rhs, &ctx->xk, &ctx->rk, &ctx->rhat, &ctx->pk,
                     &ctx->vk, &ctx->phat, &ctx->shat, &ctx->sk, &ctx->tk};
  for (double** v : vecs) ALLOC(*v, (size_t)NU * n * 8);
  ALLOC(ctx->sc, S_NSCAL * 8);
  CK(cudaMallocHost(&ctx->sc_h, S_NSCAL * 8));
  ctx->npartial = std::max<int64_t>((int64_t)RED_BLOCKS * std::max(3 * (NF + 1), GM_MAXV + 1),
                                    ((int64_t)grid1d(n, 32) + 2) * NU * 3);
  ALLOC(ctx->partial2, (int64_t)FIN_BLOCKS * 3 * 8);
  ALLOC(ctx->partial, ctx->npartial * 8);
  ALLOC(ctx->flags, n * 4);
  ALLOC(ctx->fail_d, 4);
  ALLOC(ctx->ccnz_d, 4);
  CK(cudaMemset(ctx->ccnz_d, 0xff, 4));
  if (precond == ISC_PRECOND_BJACOBI || precond == ISC_PRECOND_RAS) {
    int s = build_ilu(ctx);
    if (s) return s;
  } else if (precond == ISC_PRECOND_MCILU) {
    ALLOC(ctx->mc_uinv, (size_t)NB * n * 8);
  }
  *out = ctx;
  return ISC_OK;
}

extern "C" int isc_destroy(isc_ctx* ctx) {
  if (!ctx) return ISC_OK;
  cudaStreamSynchronize(ctx->stream);
  void* ptrs[] = {ctx->depth, ctx->vol, ctx->phi_ref, ctx->gd, ctx->td, ctx->hl_area,
                  ctx->conn_id, ctx->wells_d, ctx->wcell_d, ctx->wout_d, ctx->bhp_d,
                  ctx->capped_d, ctx->rec, ctx->acc, ctx->src, ctx->resid, ctx->diag,
                  ctx->offd, ctx->upw, ctx->bad_d, ctx->ticket_d, ctx->wdu_d, ctx->rhs, ctx->xk, ctx->rk, ctx->rhat,
                  ctx->pk, ctx->vk, ctx->phat, ctx->shat, ctx->sk, ctx->tk, ctx->sc,
                  ctx->partial, ctx->partial2, ctx->fbuf, ctx->flags, ctx->fail_d, ctx->ccnz_d, ctx->st_c, ctx->accn_c, ctx->stage,
                  ctx->halo_send_lo, ctx->halo_send_hi, ctx->halo_recv_lo, ctx->halo_recv_hi,
                  ctx->gm_V, ctx->gm_h, ctx->cbp, ctx->cmid, ctx->ces, ctx->cbc, ctx->cg9,
                  ctx->ch6, ctx->cfail_d};
  if (ctx->comm.nccl && nccl_api().CommDestroy) nccl_api().CommDestroy(ctx->comm.nccl);
  free_ilu(ctx);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->wout_h) cudaFreeHost(ctx->wout_h);
  if (ctx->bad_h) cudaFreeHost(ctx->bad_h);
  if (ctx->cfail_h) cudaFreeHost(ctx->cfail_h);
  if (ctx->wdu_h) cudaFreeHost(ctx->wdu_h);
  if (ctx->sc_h) cudaFreeHost(ctx->sc_h);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (auto& e : ctx->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  for (auto& e : ctx->cell_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->face_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->halo_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return ISC_OK;
}

extern "C" void* isc_stream(isc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
extern "C" int isc_set_stream(isc_ctx* ctx, void* stream) {
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return ISC_OK;
}
extern "C" int isc_synchronize(isc_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}
extern "C" int64_t isc_launch_count(isc_ctx* ctx) { return ctx ? ctx->launches : 0; }
extern "C" int isc_stage_times(isc_ctx* ctx, double* out4) {
  STAGE(sync_stream(ctx));
  for (int i = 0; i < 4; ++i) out4[i] = ctx->stage_ms[i];
  return ISC_OK;
}
extern "C" int isc_set_profiling(isc_ctx* ctx, int32_t on) {
  CK(cudaStreamSynchronize(ctx->stream));
  kflush(ctx);
  ctx->profiling = on != 0;
  return ISC_OK;
}
extern "C" int isc_kernel_times(isc_ctx* ctx, double* ms8, int64_t* count8, int32_t reset) {
  CK(cudaStreamSynchronize(ctx->stream));
  kflush(ctx);
  for (int i = 0; i < 8; ++i) {
    ms8[i] = ctx->kern_ms[i];
    count8[i] = ctx->kern_n[i];
    if (reset) { ctx->kern_ms[i] = 0; ctx->kern_n[i] = 0; }
  }
  return ISC_OK;
}


// ------------------------------------------------------------- assemble

// face evaluation over lower cells [c0, c1), axes axis_lo .. axis_lo+naxes-1
static void launch_face_eval(const FaceArgs2& F2, int64_t c0, int64_t c1, int axis_lo, int naxes,
                             cudaStream_t st) {
  const int blocks = grid1d(c1 - c0, 32);
  k_face_eval_light<<<blocks, dim3(32, naxes), 0, st>>>(F2, c0, c1, axis_lo);
  k_face_eval_energy<<<blocks, dim3(32, naxes), 0, st>>>(F2, c0, c1, axis_lo);
}

// the cell pass over positions [A.c_begin, A.c_end): properties, gas phase,
// then the reaction / accumulation rows (fewer live values per kernel;
// assemble.cu)
static void launch_cell(isc_ctx* ctx, CellArgs A, cudaStream_t st) {
  const int blocks = grid1d(A.c_end - A.c_begin, 128);
  A.mid = ctx->cmid;
  k_cell_props<<<blocks, 128, 0, st>>>(ctx->M, A);
  k_cell_gas<<<blocks, 128, 0, st>>>(ctx->M, A);
  k_cell_rows<<<blocks, 128, 0, st>>>(ctx->M, A);
  ctx->launches += 2;
}

extern "C" int isc_assemble(isc_ctx* ctx, const double* d_state, const double* h_bhp,
                            const double* d_accn, double dt, double t_new,
                            const uint8_t* h_capped, int32_t freeze, double* h_wells_out,
                            int64_t* bad_cell) {
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  ctx->assembled = false;
  // set by isc_assemble_host when it ran these passes while staging
  const bool cell_pre = ctx->cell_pre, face_pre = ctx->face_pre, gather_pre = ctx->gather_pre;
  ctx->cell_pre = ctx->face_pre = ctx->gather_pre = false;
  STAGE(stage_begin(ctx, 0));
  if (ctx->nw > 0) {
    CK(cudaMemcpyAsync(ctx->bhp_d, h_bhp, ctx->nw * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->capped_d, h_capped, ctx->nw, cudaMemcpyHostToDevice, st));
  }
  if (!cell_pre) CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  if (d_state) {   // NULL: state/accn already staged by isc_assemble_host
    k_to_pos<double><<<grid1d(n, 256), 256, 0, st>>>(ctx->g, NU, d_state, ctx->st_c);
    k_to_pos<double><<<grid1d(n, 256), 256, 0, st>>>(ctx->g, NU, d_accn, ctx->accn_c);
    ctx->launches += 2;
  }
  d_state = ctx->st_c;
  d_accn = ctx->accn_c;
  {
    int hs = halo_exchange(ctx, ctx->st_c, NU);   // ghost planes of the state (multi-GPU)
    if (hs) return hs;
  }
  CellArgs A{ctx->g, d_state, ctx->phi_ref, ctx->vol, ctx->hl_area, ctx->hl_kob, ctx->hl_d,
             ctx->hl_rho, ctx->hl_tini, d_accn, dt, ctx->rec, ctx->acc, ctx->src,
             ctx->resid, ctx->diag, ctx->bad_d, 0, n};
  if (!cell_pre) {
    KScope ks(ctx, KT_CELL);
    launch_cell(ctx, A, st);
  }
  LAUNCH_CHECK();
  // the pore-space test (assembly.py:548-552) is read back with the well
  // outputs at the end -- one synchronisation per assembly; on failure the
  // face and well passes ran on the failed state and their results are
  // discarded with the status (the upwind flags they wrote are rewritten by
  // the retried step's first, unfrozen iterations, newton.py:279)
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  FaceArgs F{ctx->g, d_state, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, freeze,
             ctx->resid, ctx->diag, ctx->offd, ctx->ccnz_d};
  {
    KScope ks(ctx, KT_FACE);
    FaceArgs2 F2{F, ctx->fbuf};
    if (!face_pre) {
      CK(cudaMemsetAsync(ctx->ccnz_d, 0, 4, st));   // set by k_face_eval* on a nonzero
      launch_face_eval(F2, 0, n, 0, 3, st);
    }
    if (!gather_pre) {
      const int64_t c0 = (int64_t)ctx->g.kw_lo * ctx->g.nxny, c1 = (int64_t)ctx->g.kw_hi * ctx->g.nxny;
      k_face_gather<<<grid1d(c1 - c0, 32), dim3(32, ROW_OS), 0, st>>>(F2, c0, c1);
      ++ctx->launches;
    }
  }
  LAUNCH_CHECK();
  if (ctx->nw > 0) {
    KScope ks(ctx, KT_WELLS);
    k_wells<<<1, 32, 0, st>>>(ctx->M, ctx->g, ctx->nw, ctx->wells_d, d_state, ctx->bhp_d,
                              ctx->capped_d, ctx->rec, ctx->depth, t_new, ctx->resid,
                              ctx->diag, ctx->wout_d);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(ctx->wout_h, ctx->wout_d, ctx->nw * WOUT * 8, cudaMemcpyDeviceToHost, st));
  }
  STAGE(stage_end(ctx, 0));
  STAGE(sync_stream(ctx));
  {
    // all ranks of a z-slab run take the same branch
    double flag = *ctx->bad_h != ~0ULL ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
    if (as) return as;
    if (flag > 0.0) {
      if (bad_cell) *bad_cell = *ctx->bad_h != ~0ULL ? (int64_t)*ctx->bad_h : -1;
      g_err = "coke fills the pore volume";
      return ISC_PORE_SPACE_EXHAUSTED;
    }
  }
  if (ctx->nw > 0 && h_wells_out) std::memcpy(h_wells_out, ctx->wout_h, ctx->nw * WOUT * 8);
  ctx->decoupled = false;
  ctx->compact = false;
  ctx->factored = false;
  ctx->offd_rows = ROW_OS;   // rows ROW_OS.. of the off-diagonal blocks were not written
  ctx->assembled = true;
  ctx->asm_dt = dt;
  ctx->asm_freeze = freeze;
  return ISC_OK;
}

extern "C" int isc_numeric_jacobian(isc_ctx* ctx, double* h_wells_out, int64_t* bad_cell) {
  if (!ctx->assembled || ctx->decoupled) {
    g_err = "isc_numeric_jacobian needs the system of the last isc_assemble";
    return ISC_BAD_ARGUMENT;
  }
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  CellArgs A{ctx->g, ctx->st_c, ctx->phi_ref, ctx->vol, ctx->hl_area, ctx->hl_kob, ctx->hl_d,
             ctx->hl_rho, ctx->hl_tini, ctx->accn_c, ctx->asm_dt, nullptr, nullptr, nullptr,
             nullptr, nullptr, ctx->bad_d, 0, n};
  NumJacArgs J{A, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, ctx->asm_freeze,
               ctx->diag, ctx->offd, ctx->nw, ctx->wells_d, ctx->bhp_d, ctx->capped_d,
               ctx->wout_d, ctx->bad_d};
  k_numjac<<<grid1d(n, 32), dim3(32, NU), 0, st>>>(ctx->M, J);
  LAUNCH_CHECK();
  if (ctx->nw > 0) {
    k_numjac_wells<<<1, 32, 0, st>>>(ctx->M, ctx->g, ctx->nw, ctx->wells_d, ctx->st_c,
                                     ctx->bhp_d, ctx->capped_d, ctx->rec, ctx->depth,
                                     ctx->wout_d);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(ctx->wout_h, ctx->wout_d, ctx->nw * WOUT * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ctx->offd_rows = NU;   // every row of every block written
  // finite-difference blocks can carry coke-column entries in every row: the
  // compact form's coke-column skip (k_cc_red, k_face_gather) must not apply
  CK(cudaMemsetAsync(ctx->ccnz_d, 0xff, 4, st));
  double flag = *ctx->bad_h != ~0ULL ? 1.0 : 0.0;
  int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
  if (as) return as;
  if (flag > 0.0) {
    if (bad_cell) *bad_cell = *ctx->bad_h != ~0ULL ? (int64_t)*ctx->bad_h : -1;
    g_err = "coke fills the pore volume at a probed state";
    return ISC_PORE_SPACE_EXHAUSTED;
  }
  if (ctx->nw > 0 && h_wells_out) std::memcpy(h_wells_out, ctx->wout_h, ctx->nw * WOUT * 8);
  return ISC_OK;
}

// Reference-layout host inputs (State arrays p, x (n,nco), y (n,ncg), t, sw,
// sg, cc and accn (n, NU)): one H2D copy each into a staging buffer, the
// SoA/storage-order transpose on the device, then isc_assemble.
extern "C" int isc_assemble_host(isc_ctx* ctx, const double* h_p, const double* h_x,
                                 const double* h_y, const double* h_t, const double* h_sw,
                                 const double* h_sg, const double* h_cc, const double* h_bhp,
                                 const double* h_accn, double dt, double t_new,
                                 const uint8_t* h_capped, int32_t freeze, double* h_wells_out,
                                 int64_t* bad_cell) {
  const int64_t n = ctx->g.n;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  double* sg = ctx->stage;
  const double* rest[4] = {h_t, h_sw, h_sg, h_cc};
  // Copies of plane chunks on the copy stream, each chunk's transpose and
  // cell pass on the main stream as soon as it lands: the PCIe transfer
  // overlaps the cell kernel (one chunk on z-slabs, whose cell pass needs
  // the halo exchange of the whole state first).
  const bool pipe = !ctx->comm.active();
  static const int nq_max = [] {   // plane chunks of the staged copy (ISC_H2D_CHUNKS, 1..32)
    const char* e = std::getenv("ISC_H2D_CHUNKS");
    const int v = e ? std::atoi(e) : 13;
    return std::max(1, std::min(30, v));
  }();
  static const int first_planes = [] {   // planes of the first chunk (ISC_H2D_FIRST)
    const char* e = std::getenv("ISC_H2D_FIRST");
    return std::max(1, e ? std::atoi(e) : 2);
  }();
  // chunk bounds: a thin first chunk (the compute starts as soon as it has
  // landed), the remaining planes in nq - 1 equal chunks (every chunk costs
  // the ramp and tail of its ~10 kernels)
  int kb[34];
  int nq = 1;
  kb[0] = 0;
  kb[1] = g.nz;
  if (pipe && nq_max > 1 && g.nz > first_planes) {
    const int nrest = std::min(nq_max - 1, g.nz - first_planes);
    nq = 1 + nrest;
    kb[1] = first_planes;
    for (int q = 1; q <= nrest; ++q)
      kb[1 + q] = first_planes + (int)((int64_t)(g.nz - first_planes) * q / nrest);
  }
  int64_t gathered = 0;   // positions whose faces are all evaluated and gathered
  // Alternate chunks run on two compute streams so that one chunk's kernels
  // fill the ramps and tails of the other's (ten dependent kernels per chunk
  // otherwise drain the GPU at every boundary). Chunk q's face evaluation
  // reads the records of chunk q - 1's last plane (cell_ev[q - 1]) and its
  // gather the blocks chunk q - 1's faces wrote (face_ev[q - 1]); everything
  // else a chunk touches lies in its own planes. The per-kernel-class timers
  // record on the main stream only: one stream while profiling.
  static const bool two_env = [] {
    const char* e = std::getenv("ISC_H2D_TWO_STREAMS");
    return !e || std::atoi(e) != 0;
  }();
  const bool two = pipe && two_env && !ctx->profiling && nq > 2;
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  CK(cudaEventRecord(ctx->chunk_ev[0], st));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->chunk_ev[0], 0));   // stage buffer free
  if (two) CK(cudaStreamWaitEvent(ctx->stream2, ctx->chunk_ev[0], 0));
  CellArgs A{g, ctx->st_c, ctx->phi_ref, ctx->vol, ctx->hl_area, ctx->hl_kob, ctx->hl_d,
             ctx->hl_rho, ctx->hl_tini, ctx->accn_c, dt, ctx->rec, ctx->acc, ctx->src,
             ctx->resid, ctx->diag, ctx->bad_d, 0, n};
  FaceArgs F{g, ctx->st_c, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, freeze,
             ctx->resid, ctx->diag, ctx->offd, ctx->ccnz_d};
  FaceArgs2 F2{F, ctx->fbuf};
  if (pipe) CK(cudaMemsetAsync(ctx->ccnz_d, 0, 4, st));
  if (two) {   // stream2's first kernels follow the two flag resets
    CK(cudaEventRecord(ctx->face_ev[31], st));
    CK(cudaStreamWaitEvent(ctx->stream2, ctx->face_ev[31], 0));
  }
  cudaStream_t st_main = st;
  for (int q = 0; q < nq; ++q) {
    st = two && (q & 1) ? ctx->stream2 : st_main;
    const int64_t k0 = kb[q], k1 = kb[q + 1];
    const int64_t c0 = k0 * g.nxny, c1 = k1 * g.nxny, cnt = c1 - c0;
    const size_t b = (size_t)cnt * 8;
    cudaStream_t cs = ctx->cstream;
    CK(cudaMemcpyAsync(sg + c0, h_p + c0, b, cudaMemcpyHostToDevice, cs));
    CK(cudaMemcpyAsync(sg + n + c0 * NCO, h_x + c0 * NCO, b * NCO, cudaMemcpyHostToDevice, cs));
    CK(cudaMemcpyAsync(sg + (1 + NCO) * n + c0 * NCG, h_y + c0 * NCG, b * NCG,
                       cudaMemcpyHostToDevice, cs));
    for (int r = 0; r < 4; ++r)
      CK(cudaMemcpyAsync(sg + (1 + NCO + NCG + r) * n + c0, rest[r] + c0, b,
                         cudaMemcpyHostToDevice, cs));
    CK(cudaMemcpyAsync(sg + (size_t)(CT + 4) * n + c0 * NU, h_accn + c0 * NU, b * NU,
                       cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->chunk_ev[q], cs));
    CK(cudaStreamWaitEvent(st, ctx->chunk_ev[q], 0));
    k_stage_state<<<grid1d(cnt, 256), 256, 0, st>>>(g, sg, ctx->st_c, ctx->accn_c, c0, c1);
    ++ctx->launches;
    if (pipe) {   // planes [k0, k1) occupy positions [c0, c1) in both storage orders
      A.c_begin = c0;
      A.c_end = c1;
      {
        KScope ks(ctx, KT_CELL);
        launch_cell(ctx, A, st);
      }
      if (two) {
        CK(cudaEventRecord(ctx->cell_ev[q], st));
        if (q > 0) CK(cudaStreamWaitEvent(st, ctx->cell_ev[q - 1], 0));
      }
      KScope ks(ctx, KT_FACE);
      // all three axes of the planes whose upper neighbours' records now
      // exist: the last plane of the previous chunk up to this chunk's last
      // but one (one launch per row class, the axes share the record loads)
      const int64_t z0 = std::max<int64_t>(0, (k0 - 1) * g.nxny), z1 = (k1 - 1) * g.nxny;
      if (z1 > z0) {
        launch_face_eval(F2, z0, z1, 0, 3, st);
        ctx->launches += 2;
      }
      if (two) {
        CK(cudaEventRecord(ctx->face_ev[q], st));
        if (q > 0) CK(cudaStreamWaitEvent(st, ctx->face_ev[q - 1], 0));
      }
      // every face of the planes below k1 - 1 is now evaluated: gather them
      // while the next chunk is still on the bus
      if (z1 > gathered) {
        k_face_gather<<<grid1d(z1 - gathered, 32), dim3(32, ROW_OS), 0, st>>>(F2, gathered, z1);
        ++ctx->launches;
        gathered = z1;
      }
    }
  }
  st = st_main;
  if (two) {   // join: the main stream continues after both streams' last chunks
    CK(cudaEventRecord(ctx->face_ev[30], ctx->stream2));
    CK(cudaStreamWaitEvent(st, ctx->face_ev[30], 0));
  }
  if (pipe) {   // the top plane's faces (+z: boundary, zero blocks), the last planes' gather
    KScope ks(ctx, KT_FACE);
    const int64_t z0 = (int64_t)(g.nz - 1) * g.nxny;
    launch_face_eval(F2, z0, n, 0, 3, st);
    k_face_gather<<<grid1d(n - gathered, 32), dim3(32, ROW_OS), 0, st>>>(F2, gathered, n);
    ctx->launches += 2;
  }
  LAUNCH_CHECK();
  ctx->cell_pre = pipe;
  ctx->face_pre = pipe;
  ctx->gather_pre = pipe;
  return isc_assemble(ctx, nullptr, h_bhp, nullptr, dt, t_new, h_capped, freeze, h_wells_out,
                      bad_cell);
}

// du of the last isc_solve as a host (n, NU) array in natural cell order
extern "C" int isc_download_du(isc_ctx* ctx, double* h_du) {
  const int64_t n = ctx->g.n;
  k_unstage_rows<<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, ctx->xk, ctx->stage, 0, n);
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(h_du, ctx->stage, (size_t)n * NU * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

extern "C" int isc_copy_out(isc_ctx* ctx, int32_t what, void* d_dst) {
  const int64_t n = ctx->g.n;
  const void* src = nullptr;
  size_t bytes = 0;
  switch (what) {
    case 0: src = ctx->resid; bytes = (size_t)NU * n * 8; break;
    case 1: src = ctx->acc; bytes = (size_t)NU * n * 8; break;
    case 2: src = ctx->src; bytes = (size_t)NU * n * 8; break;
    case 3: src = ctx->rec + (size_t)R_Y * n; bytes = (size_t)NF * n * 8; break;
    case 4: src = ctx->rec; bytes = (size_t)NREC * n * 8; break;
    case 5: src = ctx->upw; bytes = (size_t)9 * n; break;
    default: g_err = "unknown array"; return ISC_BAD_ARGUMENT;
  }
  // back to natural cell order
  if (what == 5) {
    k_from_pos<int8_t><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, 9, (const int8_t*)src,
                                                                (int8_t*)d_dst);
  } else {
    const int rows = (int)(bytes / 8 / n);
    k_from_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, rows, (const double*)src,
                                                                (double*)d_dst);
  }
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

extern "C" int isc_export_system(isc_ctx* ctx, double* d_diag, double* d_offd, double* d_resid) {
  k_export_system<<<grid1d(ctx->g.n, 128), 128, 0, ctx->stream>>>(
      ctx->g, ctx->conn_id, ctx->diag, ctx->offd, ctx->resid, d_diag, d_offd, d_resid,
      ctx->offd_rows);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

extern "C" int isc_import_system(isc_ctx* ctx, const double* d_diag, const double* d_offd,
                                 const double* d_resid, const double* h_wells_out) {
  CK(cudaMemsetAsync(ctx->ccnz_d, 0xff, 4, ctx->stream));   // imported blocks: full rows
  k_import_system<<<grid1d(ctx->g.n, 128), 128, 0, ctx->stream>>>(
      ctx->g, ctx->conn_id, d_diag, d_offd, d_resid, ctx->diag, ctx->offd, ctx->resid);
  LAUNCH_CHECK();
  if (ctx->nw > 0 && h_wells_out) {
    std::memcpy(ctx->wout_h, h_wells_out, ctx->nw * WOUT * 8);
    CK(cudaMemcpyAsync(ctx->wout_d, ctx->wout_h, ctx->nw * WOUT * 8, cudaMemcpyHostToDevice,
                       ctx->stream));
  }
  // flux-only off-diagonal rows (an assembled system's structure): the
  // multicolour solve may use the compact form
  int rows = NU;
  if (ctx->g.colored) {
    CK(cudaMemsetAsync(ctx->fail_d, 0, 4, ctx->stream));
    k_flux_rows_only<<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g, ctx->offd,
                                                                      ctx->fail_d);
    LAUNCH_CHECK();
    int nz = 1;
    CK(cudaMemcpyAsync(&nz, ctx->fail_d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (nz == 0) rows = ROW_OS;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->decoupled = ctx->factored = false;
  ctx->compact = false;
  ctx->offd_rows = rows;
  ctx->assembled = false;
  return ISC_OK;
}

extern "C" int isc_set_wells_out(isc_ctx* ctx, const double* h_wells_out) {
  if (ctx->nw == 0) return ISC_OK;
  std::memcpy(ctx->wout_h, h_wells_out, ctx->nw * WOUT * 8);
  CK(cudaMemcpyAsync(ctx->wout_d, ctx->wout_h, ctx->nw * WOUT * 8, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

static void free_ilu(isc_ctx* ctx) {
  void* ptrs[] = {ctx->lvl_ptr_d, (void*)ctx->ilu.cell, (void*)ctx->ilu.owned,
                  (void*)ctx->ilu.lo, (void*)ctx->ilu.up, ctx->ilu.lblk, ctx->ilu.uinv,
                  ctx->ilu.zs};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  ctx->ilu = IluDev{};
  if (ctx->mc_uinv) cudaFree(ctx->mc_uinv);
  ctx->mc_uinv = nullptr;
  ctx->lvl_ptr_d = nullptr;
  ctx->nlev = 0;
}

extern "C" int isc_set_precond(isc_ctx* ctx, int32_t precond) {
  if (precond < 0 || precond > 3) { g_err = "unknown preconditioner"; return ISC_BAD_ARGUMENT; }
  if (precond == ctx->precond) return ISC_OK;
  if (ctx->compact && ctx->decoupled) {
    g_err = "system decoupled in the multicolour compact form: assemble again first";
    return ISC_UNSUPPORTED;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  free_ilu(ctx);
  ctx->precond = precond;
  ctx->factored = false;
  if (precond == ISC_PRECOND_BJACOBI || precond == ISC_PRECOND_RAS) return build_ilu(ctx);
  if (precond == ISC_PRECOND_MCILU) ALLOC(ctx->mc_uinv, (size_t)NB * ctx->g.n * 8);
  return ISC_OK;
}

extern "C" int isc_synth_system_slab(isc_ctx* ctx, uint64_t seed, int32_t nz_global) {
  if (nz_global <= 0) nz_global = ctx->k_offset + ctx->g.nz;
  if (ctx->k_offset < 0 || ctx->k_offset + ctx->g.nz > nz_global) {
    g_err = "isc_synth_system_slab: local planes outside the global grid";
    return ISC_BAD_ARGUMENT;
  }
  k_synth<<<grid1d(ctx->g.n, 128), 128, 0, ctx->stream>>>(ctx->g, seed, ctx->k_offset, nz_global,
                                                          ctx->diag, ctx->offd, ctx->resid);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->decoupled = ctx->factored = false;
  ctx->compact = false;
  ctx->offd_rows = NU;
  ctx->assembled = false;
  return ISC_OK;
}

extern "C" int isc_synth_system(isc_ctx* ctx, uint64_t seed) {
  return isc_synth_system_slab(ctx, seed, 0);
}

// ------------------------------------------------------------- decouple

// Decoupling in two halves: decouple_enqueue launches the well Schur fold and
// the Gauss-Jordan pass and queues the read-back of the first singular cell;
// decouple_check (after a synchronisation) reports it. isc_solve queues the
// preconditioner setup in between, so the two share one synchronisation.
// v[u*n + pos[w]] for every well w and row u -> out[w*NU + u]
__global__ void k_gather_rows(int64_t n, const double* __restrict__ v,
                              const int64_t* __restrict__ pos, int nw, double* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= nw * NU) return;
  const int w = t / NU, u = t - w * NU;
  out[t] = v[(int64_t)u * n + pos[w]];
}

// condensed-form buffers (lazy; false when the device has no room: the
// 9-component compact form is used instead)
static bool cond_alloc(isc_ctx* ctx) {
  if (ctx->ces) return true;
  const size_t half = (size_t)ctx->g.half, n = (size_t)ctx->g.n;
  if (cudaMalloc(&ctx->ces, (size_t)NCS * CR * half * 8) != cudaSuccess ||
      cudaMalloc(&ctx->cbc, (size_t)NDIR * CR * CR * half * 8) != cudaSuccess ||
      cudaMalloc(&ctx->cg9, (size_t)NU * n * 8) != cudaSuccess ||
      cudaMalloc(&ctx->ch6, (size_t)CR * n * 8) != cudaSuccess ||
      cudaMalloc(&ctx->cfail_d, 4) != cudaSuccess ||
      cudaMallocHost(&ctx->cfail_h, 4) != cudaSuccess) {
    cudaGetLastError();
    for (void* p : {(void*)ctx->ces, (void*)ctx->cbc, (void*)ctx->cg9, (void*)ctx->ch6,
                    (void*)ctx->cfail_d})
      if (p) cudaFree(p);
    if (ctx->cfail_h) cudaFreeHost(ctx->cfail_h);
    ctx->ces = ctx->cbc = ctx->cg9 = ctx->ch6 = nullptr;
    ctx->cfail_d = ctx->cfail_h = nullptr;
    ctx->cond_ok = false;
    return false;
  }
  return true;
}

static int decouple_enqueue(isc_ctx* ctx, int64_t* bad_cell, int32_t* bad_col) {
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  // well equations with a zero / non-finite bhp derivative (linsolve.py:372-375);
  // wout_h is current (isc_assemble / isc_numeric_jacobian / isc_set_wells_out)
  {
    double wbad = 0.0;
    if (ctx->nw > 0) {
      for (int w = 0; w < ctx->nw; ++w) {
        const double dwdb = ctx->wout_h[w * WOUT + 1];
        if (dwdb == 0.0 || !std::isfinite(dwdb)) wbad = 1.0;
      }
    }
    int as = isc_comm_allreduce_host(ctx, &wbad, 1, 1);
    if (as) return as;
    if (wbad > 0.0) {
      if (bad_cell) *bad_cell = -1;
      if (bad_col) *bad_col = -1;
      g_err = "well equation has a zero bhp derivative";
      return ISC_SINGULAR_CELL_BLOCK;
    }
  }
  STAGE(stage_begin(ctx, 1));
  {
  KScope ks(ctx, KT_DECOUPLE);
  // compact form: the red-eliminated multicolour solve of an assembled
  // system (compact.cu)
  ctx->compact = ctx->compact_ok && ctx->precond == ISC_PRECOND_MCILU && ctx->g.colored &&
                 ctx->mc_schur && ctx->offd_rows == ROW_OS;
  if (ctx->compact && !ctx->cbp &&
      cudaMalloc(&ctx->cbp, (size_t)NDIR * CR * CR * ctx->g.half * 8) != cudaSuccess) {
    cudaGetLastError();
    ctx->cbp = nullptr;
    ctx->compact = false;   // no room for B': the explicit form
  }
  if (!ctx->compact) {   // (the compact decoupling folds the wells itself)
    k_rhs_schur<<<grid1d(n, 256), 256, 0, st>>>(ctx->g, ctx->resid, ctx->rhs, ctx->diag, ctx->nw,
                                                ctx->wcell_d, ctx->wout_d, WOUT);
    LAUNCH_CHECK();
  } else if (ctx->comm.active()) {
    k_zero_ghost_rows<<<RED_BLOCKS, 256, 0, st>>>(ctx->g, NU, ctx->rhs);
    LAUNCH_CHECK();
  }
  CK(cudaMemsetAsync(ctx->flags, 0, n * 4, st));
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  if (ctx->compact) {
    const int64_t owned = (int64_t)(ctx->g.kw_hi - ctx->g.kw_lo) * ctx->g.nxny;
    // condensed form (BiCGSTAB): E_S of the black cells from the local rows,
    // formed by the decoupling of the owned planes and, on z-slabs, by
    // k_cond_es for the ghost planes (whose local rows the assembly evaluated
    // here too; the decoupling leaves the local rows' slots in place)
    ctx->cond_es = ctx->cond_ok && cond_alloc(ctx);
    if (ctx->cond_es) CK(cudaMemsetAsync(ctx->cfail_d, 0, 4, st));
    CK(cudaFuncSetAttribute(k_decouple_compact_t, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            DCT_SMEM));
    k_decouple_compact_t<<<grid1d(owned, DCT_THREADS), DCT_THREADS, DCT_SMEM, st>>>(
        ctx->g, ctx->diag, ctx->rhs, ctx->flags, ctx->bad_d, ctx->resid, ctx->nw, ctx->wcell_d,
        ctx->wout_d, WOUT, ctx->cond_es ? ctx->ces : nullptr, ctx->cfail_d);
    if (ctx->cond_es) {
      const Dims& g0 = ctx->g;
      for (int side = 0; side < 2; ++side) {   // ghost planes [0, kw_lo), [kw_hi, nz)
        Dims ga = g0;
        ga.tw_lo = side == 0 ? 0 : (int64_t)g0.kw_hi * g0.ph;
        ga.tw_hi = side == 0 ? (int64_t)g0.kw_lo * g0.ph : g0.half;
        if (ga.tw_hi > ga.tw_lo)
          k_cond_es<<<grid1d(ga.tw_hi - ga.tw_lo, 256), 256, 0, st>>>(ga, ctx->diag, ctx->ces,
                                                                      ctx->cfail_d);
      }
      CK(cudaMemcpyAsync(ctx->cfail_h, ctx->cfail_d, 4, cudaMemcpyDeviceToHost, st));
    }
  } else {
    ctx->cond_es = false;
    // once per process (thread-safe static init: hub ranks share the process)
    static const cudaError_t attr = cudaFuncSetAttribute(
        k_decouple_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(WsSmem));
    CK(attr);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t owned = (int64_t)(ctx->g.kw_hi - ctx->g.kw_lo) * ctx->g.nxny;
    const int64_t groups = (owned + WS_CELLS - 1) / WS_CELLS;
    const int grid = (int)std::min<int64_t>(groups, (int64_t)sms * WS_BLOCKS_PER_SM);
    k_decouple_ws<<<grid, WS_THREADS, sizeof(WsSmem), st>>>(ctx->g, ctx->diag, ctx->offd,
                                                           ctx->rhs, ctx->flags, ctx->bad_d,
                                                           ctx->offd_rows);
  }
  LAUNCH_CHECK();
  if (!ctx->compact) ctx->offd_rows = NU;   // the decoupled blocks are dense
  }
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  STAGE(stage_end(ctx, 1));
  return ISC_OK;
}

static int decouple_check(isc_ctx* ctx, int64_t* bad_cell, int32_t* bad_col) {
  if (ctx->cond_es && ctx->comm.active()) {   // every rank takes the same form
    double f = *ctx->cfail_h ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &f, 1, 1);
    if (as) return as;
    *ctx->cfail_h = f > 0.0 ? 1 : 0;
  }
  {
    double flag = *ctx->bad_h != ~0ULL ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
    if (as) return as;
    if (flag > 0.0 && *ctx->bad_h == ~0ULL) {
      if (bad_cell) *bad_cell = -1;
      if (bad_col) *bad_col = -1;
      g_err = "diagonal block is singular on another rank";
      return ISC_SINGULAR_CELL_BLOCK;
    }
  }
  if (*ctx->bad_h != ~0ULL) {
    const int64_t c = (int64_t)*ctx->bad_h;
    int flag = 0;
    CK(cudaMemcpy(&flag, ctx->flags + c, 4, cudaMemcpyDeviceToHost));
    if (bad_cell) *bad_cell = c;
    if (bad_col) *bad_col = flag - 1;
    g_err = "diagonal block is singular";
    return ISC_SINGULAR_CELL_BLOCK;
  }
  ctx->decoupled = true;
  return ISC_OK;
}

extern "C" int isc_decouple(isc_ctx* ctx, int64_t* bad_cell, int32_t* bad_col) {
  STAGE(decouple_enqueue(ctx, bad_cell, bad_col));
  STAGE(sync_stream(ctx));
  return decouple_check(ctx, bad_cell, bad_col);
}

extern "C" int isc_copy_rhs(isc_ctx* ctx, double* d_dst) {
  k_from_pos<double><<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, ctx->rhs, d_dst);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

// Replace the decoupled right-hand side (natural order, SoA (9, n)) of a
// decoupled system; the next isc_solve refactors (the multicolour setup also
// forms the reduced right-hand side from it).
extern "C" int isc_set_rhs(isc_ctx* ctx, const double* d_src) {
  if (!ctx->decoupled) {
    g_err = "isc_set_rhs needs a decoupled system";
    return ISC_BAD_ARGUMENT;
  }
  k_to_pos<double><<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, d_src, ctx->rhs);
  LAUNCH_CHECK();
  ctx->factored = false;
  return ISC_OK;
}

// Preconditioner setup in two halves as the decoupling: precond_enqueue
// launches the factorisation and queues the read-back of its status,
// precond_check reports it after a synchronisation.
static int precond_enqueue(isc_ctx* ctx) {
  ctx->cond = false;
  if (ctx->precond == ISC_PRECOND_NONE) return ISC_OK;
  cudaStream_t st = ctx->stream;
  STAGE(stage_begin(ctx, 2));
  CK(cudaMemsetAsync(ctx->fail_d, 0x7f, 4, st));
  Dims g = ctx->g;
  IluDev L = ctx->ilu;
  const double* offd = ctx->offd;
  const int64_t* lp = ctx->lvl_ptr_d;
  int nlev = ctx->nlev;
  int* fail = ctx->fail_d;
  {
  KScope ks(ctx, KT_ILU_FACTOR);
  if (ctx->precond == ISC_PRECOND_MCILU) {
    const int64_t nblack = ctx->g.colored ? ctx->g.n - ctx->g.half : ctx->g.n;
    // Schur path on slabs: bring the owner ranks' decoupled blocks of the
    // boundary planes into the ghost planes (the -z blocks of our lowest owned
    // plane go down, the +z blocks of our highest go up), so U_b — and with it
    // the Krylov iteration — is the single-GPU one
    const int cross = (ctx->g.colored && ctx->comm.active()) ? 1 : 0;
    if (cross) {
      if (halo_exchange(ctx, ctx->offd + (int64_t)DZM * NB * ctx->g.n, NB)) return ISC_CUDA_ERROR;
      if (halo_exchange(ctx, ctx->offd + (int64_t)DZP * NB * ctx->g.n, NB)) return ISC_CUDA_ERROR;
      // compact form: the owner's D^-1[:, :CR] of the ghost planes as well
      if (ctx->compact && halo_exchange(ctx, ctx->diag, CR * NU)) return ISC_CUDA_ERROR;
    }
    if (ctx->compact) {
      // the reduced rhs g_b is formed on the way (red neighbours' b: halo on slabs)
      if (cross && halo_exchange(ctx, ctx->rhs, NU)) return ISC_CUDA_ERROR;
      // condensed form when the decoupling's E_S are usable (checked after
      // its synchronisation; isc_solve refactors in the 9-component form
      // otherwise)
      ctx->cond = ctx->cond_es && !(ctx->cfail_h && *ctx->cfail_h && ctx->decoupled);
      const int fblocks = grid1d(ctx->g.tw_hi - ctx->g.tw_lo, MCFC_CELLS);
      // ISC_MCF_T=0: the cooperative (shared-memory) kernel instead of the
      // thread-per-cell one (same values; tests compare them)
      const char* mcf_env = std::getenv("ISC_MCF_T");
      const bool factor_t = !mcf_env || std::atoi(mcf_env) != 0;
      if (ctx->cond && factor_t) {
        k_mc_factor_cond_t<<<grid1d(ctx->g.tw_hi - ctx->g.tw_lo, MCFT_THREADS), MCFT_THREADS, 0,
                             st>>>(ctx->g, ctx->offd, ctx->diag, ctx->mc_uinv, ctx->cbp,
                                   ctx->fail_d, ctx->rhs, ctx->cg9, ctx->ces);
      } else if (ctx->cond) {
        CK(cudaFuncSetAttribute(k_mc_factor_compact<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(McfcSmem)));
        k_mc_factor_compact<true><<<fblocks, dim3(MCFC_CELLS, NU), sizeof(McfcSmem), st>>>(
            ctx->g, ctx->offd, ctx->diag, ctx->mc_uinv, ctx->cbp, ctx->fail_d, ctx->rhs,
            ctx->cg9, nullptr, ctx->ces);
      } else {
        CK(cudaFuncSetAttribute(k_mc_factor_compact<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(McfcSmem)));
        k_mc_factor_compact<false><<<fblocks, dim3(MCFC_CELLS, NU), sizeof(McfcSmem), st>>>(
            ctx->g, ctx->offd, ctx->diag, ctx->mc_uinv, ctx->cbp, ctx->fail_d, ctx->rhs, ctx->rk,
            ctx->rhat, nullptr);
      }
      ctx->gb_fresh = true;
    } else
      k_mc_factor<<<grid1d(nblack, 32), dim3(32, NU), 0, st>>>(ctx->g, ctx->offd, ctx->mc_uinv,
                                                              ctx->fail_d, cross);
    CK(cudaGetLastError());
  } else {
  CK(cudaFuncSetAttribute(k_ilu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(FactorSmem)));
  k_ilu_factor<<<ctx->nsub * ILCF, dim3(IL_SLOTS, NU), sizeof(FactorSmem), st>>>(g, L, offd, lp,
                                                                               nlev, fail);
  CK(cudaGetLastError());
  }
  }
  ++ctx->launches;
  CK(cudaMemcpyAsync(ctx->bad_h + 1, ctx->fail_d, 4, cudaMemcpyDeviceToHost, st));
  STAGE(stage_end(ctx, 2));
  return ISC_OK;
}

static int precond_check(isc_ctx* ctx, int64_t* bad_cell) {
  if (ctx->precond == ISC_PRECOND_NONE) { ctx->factored = true; return ISC_OK; }
  int fail_h = 0;
  std::memcpy(&fail_h, ctx->bad_h + 1, 4);
  {
    double flag = fail_h != 0x7f7f7f7f ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
    if (as) return as;
    if (flag > 0.0) fail_h = 1;
  }
  if (fail_h != 0x7f7f7f7f) {
    if (bad_cell) *bad_cell = -1;
    g_err = "ILU(0) pivot failed";
    return ISC_SINGULAR_CELL_BLOCK;
  }
  ctx->factored = true;
  return ISC_OK;
}

extern "C" int isc_precond_setup(isc_ctx* ctx, int64_t* bad_cell) {
  STAGE(precond_enqueue(ctx));
  STAGE(sync_stream(ctx));
  return precond_check(ctx, bad_cell);
}

static int precond_apply(isc_ctx* ctx, const double* r, double* z) {
  const int64_t len = (int64_t)NU * ctx->g.n;
  if (ctx->precond == ISC_PRECOND_NONE) {
    CK(cudaMemcpyAsync(z, r, len * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return ISC_OK;
  }
  Dims g = ctx->g;
  if (ctx->precond == ISC_PRECOND_MCILU) {
    KScope ks(ctx, KT_ILU_APPLY);
    const int b1 = grid1d(g.colored ? g.n - g.half : g.n, 32);
    const int b2 = grid1d(g.colored ? g.half : g.n, 32);
    k_mc_apply<1><<<b1, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, ctx->mc_uinv, r, z);
    k_mc_apply<2><<<b2, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, ctx->mc_uinv, r, z);
    ctx->launches += 2;
    CK(cudaGetLastError());
    return ISC_OK;
  }
  IluDev L = ctx->ilu;
  const double* offd = ctx->offd;
  const int64_t* lp = ctx->lvl_ptr_d;
  int nlev = ctx->nlev;
  KScope ks(ctx, KT_ILU_APPLY);
  k_ilu_apply<<<ctx->nsub * ILC, dim3(IL_SLOTS, NU), 0, ctx->stream>>>(g, L, offd, lp, nlev, r, z);
  CK(cudaGetLastError());
  ++ctx->launches;
  return ISC_OK;
}

template <int K>
static int spmv(isc_ctx* ctx, const double* x, double* y, const double* w0, const double* w1,
                int* nblocks) {
  const int blocks = grid1d(ctx->g.n, 32);
  KScope ks(ctx, KT_SPMV);
  k_spmv<K><<<blocks, dim3(32, NU), 0, ctx->stream>>>(ctx->g, ctx->offd, x, y, w0, w1,
                                                      ctx->partial);
  LAUNCH_CHECK();
  if (nblocks) *nblocks = blocks * NU;   // per-warp partials
  return ISC_OK;
}

extern "C" int isc_spmv(isc_ctx* ctx, const double* d_x, double* d_y) {
  const int64_t n = ctx->g.n;
  k_to_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, d_x, ctx->sk);
  if (ctx->compact) {   // y = x + sum_d (D^-1 B_d) x, one pass per colour
    const Dims& g = ctx->g;
    const int blocks = grid1d(g.tw_hi - g.tw_lo, 32);
    KScope ks(ctx, KT_SPMV);
    k_cc_spmv<0><<<blocks, dim3(32, CR), 0, ctx->stream>>>(
        g, ctx->offd, ctx->diag, ctx->sk, ctx->sk, ctx->tk, nullptr, nullptr, nullptr, nullptr, 0, 0);
    k_cc_spmv<1><<<blocks, dim3(32, CR), 0, ctx->stream>>>(
        g, ctx->offd, ctx->diag, ctx->sk, ctx->sk, ctx->tk, nullptr, nullptr, nullptr, nullptr, 0, 0);
    LAUNCH_CHECK();
  } else {
    int s = spmv<0>(ctx, ctx->sk, ctx->tk, nullptr, nullptr, nullptr);
    if (s) return s;
  }
  k_from_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, ctx->tk, d_y);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

extern "C" int isc_precond_apply(isc_ctx* ctx, const double* d_r, double* d_z) {
  const int64_t n = ctx->g.n;
  if (ctx->compact) {
    g_err = "the compact multicolour form applies its preconditioner inside the reduced solve";
    return ISC_UNSUPPORTED;
  }
  k_to_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, d_r, ctx->sk);
  int s = precond_apply(ctx, ctx->sk, ctx->tk);
  if (s) return s;
  k_from_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, ctx->tk, d_z);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

// phat = M^-1 p and v = A phat (+ K partial dots of v) for the colour-blocked
// multicolour preconditioner; returns the number of partial slots.
template <int K>
static int mc_apply_spmv(isc_ctx* ctx, const double* p, double* phat, double* v,
                         const double* w0, const double* w1, int* nparts) {
  const Dims& g = ctx->g;
  const int b1 = grid1d(g.n - g.half, 32), b2 = grid1d(g.half, 32);
  {
    KScope ks(ctx, KT_ILU_APPLY);
    k_mc_apply<1><<<b1, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, ctx->mc_uinv, p, phat);
    k_mc_red<K><<<b2, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, p, phat, v, w0, w1,
                                                     ctx->partial, b2 + b1);
  }
  {
    KScope ks(ctx, KT_SPMV);
    k_mc_black_spmv<K><<<b1, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, phat, v, w0, w1,
                                                            ctx->partial, b2 + b1, b2, nullptr);
  }
  ctx->launches += 3;
  CK(cudaGetLastError());
  *nparts = (b1 + b2) * NU;   // per-warp partials
  return ISC_OK;
}

#include "comm_runtime.cuh"
#include "krylov.cuh"

extern "C" int isc_decoupled_form(const isc_ctx* ctx) {
  return !ctx->decoupled ? 0 : (ctx->compact ? 2 : 1);
}

extern "C" int isc_condensed(const isc_ctx* ctx) { return ctx->cond ? 1 : 0; }

extern "C" int isc_set_krylov(isc_ctx* ctx, int32_t krylov, int32_t restart) {
  if (krylov != ISC_KRYLOV_BICGSTAB && krylov != ISC_KRYLOV_GMRES) {
    g_err = "unknown Krylov method";
    return ISC_BAD_ARGUMENT;
  }
  if (restart < 0 || restart > GM_MAXV - 1) {
    g_err = "GMRES restart length out of range (1..31, 0 = default)";
    return ISC_BAD_ARGUMENT;
  }
  ctx->krylov = krylov;
  if (restart > 0) ctx->gm_m = restart;
  return ISC_OK;
}

extern "C" int isc_solve(isc_ctx* ctx, double tol, int32_t maxiter, double* d_du, double* h_dbhp,
                         int32_t* iters, int64_t* bad_cell, int32_t* bad_col) {
  // decoupling and preconditioner setup queued back to back, one
  // synchronisation, then their checks in the reference's order
  // (SingularCellBlock from the decoupling first, linsolve.py:458-463)
  const bool dec = !ctx->decoupled, fac = !ctx->factored;
  if (dec) {   // (a decoupled system was checked by its isc_decouple)
    int s = decouple_enqueue(ctx, bad_cell, bad_col);
    if (s) return s;
  }
  if (fac) STAGE(precond_enqueue(ctx));
  if (dec || fac) STAGE(sync_stream(ctx));
  if (dec) {
    int s = decouple_check(ctx, bad_cell, bad_col);
    if (s) return s;
  }
  if (fac && ctx->cond && *ctx->cfail_h) {
    // a cell's local rows cannot be condensed: the 9-component compact form
    STAGE(precond_enqueue(ctx));
    STAGE(sync_stream(ctx));
  }
  if (fac) {
    int s = precond_check(ctx, bad_cell);
    if (s) {
      if (bad_col) *bad_col = -1;
      return s;
    }
  }
  int it = 0;
  STAGE(stage_begin(ctx, 3));
  const bool schur = ctx->mc_schur && ctx->precond == ISC_PRECOND_MCILU &&
                     ctx->g.colored;
  int status = !schur ? bicgstab(ctx, tol, maxiter, &it)
               : ctx->krylov == ISC_KRYLOV_GMRES ? gmres_schur(ctx, tol, maxiter, &it)
                                                 : bicgstab_schur(ctx, tol, maxiter, &it);
  STAGE(stage_end(ctx, 3));
  if (iters) *iters = it;
  if (status) return status;
  const int64_t n = ctx->g.n;
  if (d_du) {
    k_from_pos<double><<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, ctx->xk, d_du);
    LAUNCH_CHECK();
  }
  // bhp back-substitution dbhp = -(r_w + wrow . du_c) / dwdb (linsolve.py:473-478):
  // the perforated cells' du gathered in one launch, read back with the final
  // synchronisation
  const bool wells = ctx->nw > 0 && h_dbhp;
  if (wells) {
    k_gather_rows<<<1, 32 * ((ctx->nw * NU + 31) / 32), 0, ctx->stream>>>(
        n, ctx->xk, ctx->wcell_d, ctx->nw, ctx->wdu_d);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(ctx->wdu_h, ctx->wdu_d, (size_t)ctx->nw * NU * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (wells) {
    for (int w = 0; w < ctx->nw; ++w) {
      const double* duc = ctx->wdu_h + (size_t)w * NU;
      const double* o = ctx->wout_h + w * WOUT;
      double dotv = 0.0;
      for (int u = 0; u < NU; ++u) dotv += o[2 + u] * duc[u];
      const double s = o[0] + dotv;
      h_dbhp[w] = -s / o[1];
    }
  }
  return ISC_OK;
}

// isc_solve with du delivered to the host (n, NU) array h_du (natural cell
// order; pinned memory for an asynchronous copy): on the condensed
// single-GPU path the solve's last kernels (red back-substitution, x_b = g_b
// + E_b w, transpose) run per plane chunk and each chunk's copy overlaps the
// next chunk's kernels; otherwise isc_solve + isc_download_du.
extern "C" int isc_solve_host(isc_ctx* ctx, double tol, int32_t maxiter, double* h_du,
                              double* h_dbhp, int32_t* iters, int64_t* bad_cell,
                              int32_t* bad_col) {
  ctx->h_du = h_du;
  ctx->h_du_queued = false;
  const int s = isc_solve(ctx, tol, maxiter, nullptr, h_dbhp, iters, bad_cell, bad_col);
  ctx->h_du = nullptr;
  const bool queued = ctx->h_du_queued;
  ctx->h_du_queued = false;
  if (queued) CK(cudaStreamSynchronize(ctx->cstream));
  if (s) return s;
  return queued ? ISC_OK : isc_download_du(ctx, h_du);
}

// -------------------------------------------------------------- Newton

extern "C" int isc_newton_update(isc_ctx* ctx, double* d_state, const double* d_du, double eps) {
  k_newton_update<<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g.n, d_state, d_du, eps);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

extern "C" int isc_scaled_norm(isc_ctx* ctx, const double* d_accn, double dt, double* norm) {
  k_to_pos<double><<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, d_accn, ctx->accn_c);
  k_norm_partial<<<RED_BLOCKS, 256, 0, ctx->stream>>>(ctx->g, ctx->resid, ctx->accn_c, ctx->vol,
                                                     dt, ctx->partial);
  LAUNCH_CHECK();
  std::vector<double> part(RED_BLOCKS);
  CK(cudaMemcpyAsync(part.data(), ctx->partial, RED_BLOCKS * 8, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double m = 0.0;
  bool nan = false;
  for (double v : part) {
    if (v != v) nan = true;
    m = std::max(m, v);
  }
  *norm = nan ? NAN : m;
  return isc_comm_allreduce_host(ctx, norm, 1, 1);
}

extern "C" int isc_audit_sums(isc_ctx* ctx, const double* d_accn, double* h_out) {
  constexpr int NR = NF + 1;
  k_to_pos<double><<<grid1d(ctx->g.n, 256), 256, 0, ctx->stream>>>(ctx->g, NU, d_accn, ctx->accn_c);
  k_audit_partial<<<RED_BLOCKS, 256, 0, ctx->stream>>>(ctx->g, ctx->acc, ctx->accn_c, ctx->src,
                                                      ctx->vol, ctx->partial);
  LAUNCH_CHECK();
  std::vector<double> part((size_t)3 * NR * RED_BLOCKS);
  CK(cudaMemcpyAsync(part.data(), ctx->partial, part.size() * 8, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < 3 * NR; ++k) {
    double s = 0.0;
    for (int b = 0; b < RED_BLOCKS; ++b) s += part[(size_t)k * RED_BLOCKS + b];
    h_out[k] = s;
  }
  return isc_comm_allreduce_host(ctx, h_out, 3 * NR, 0);
}

// ------------------------------------------------------------- reports

extern "C" int isc_format_double(double v, char* out32) { return py_repr_double(v, out32); }

extern "C" int isc_format_cells(double time, int64_t n, const double* p, const double* t,
                                const double* sw, const double* sg, const double* x,
                                int64_t x_cell_stride, int64_t x_comp_stride, int32_t nco,
                                const double* y, int64_t y_cell_stride, int64_t y_comp_stride,
                                int32_t nf, const double* cc, int32_t threads, char** out,
                                int64_t* len) {
  if (n < 0 || nco < 0 || nf < 0 || !out || !len) {
    g_err = "isc_format_cells: bad arguments";
    return ISC_BAD_ARGUMENT;
  }
  FrameCells F{time, n, p, t, sw, sg, cc, x, x_cell_stride, x_comp_stride, nco,
               y, y_cell_stride, y_comp_stride, nf};
  std::string s;
  try {
    s = format_cells(F, threads);
  } catch (const std::exception& e) {
    g_err = std::string("isc_format_cells: ") + e.what();
    return ISC_BAD_ARGUMENT;
  }
  char* buf = (char*)std::malloc(s.size() + 1);
  if (!buf) { g_err = "isc_format_cells: out of host memory"; return ISC_BAD_ARGUMENT; }
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  *out = buf;
  *len = (int64_t)s.size();
  return ISC_OK;
}

extern "C" void isc_free(void* p) { std::free(p); }
