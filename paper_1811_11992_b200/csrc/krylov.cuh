// Krylov drivers of the host runtime: BiCGSTAB on the full decoupled system
// (none / bjacobi / ras, linsolve.py:481-578), the device-driven BiCGSTAB and
// restarted GMRES(m) on the red-eliminated multicolour system (mcilu). Part
// of the capi.cu translation unit.
#pragma once
// ------------------------------------------------------------- BiCGSTAB

struct Kry {
  isc_ctx* ctx;
  int64_t len;
  const double* stop = nullptr;   // device-driven iterations: S_STOP guard of the sums
  int vgrid() const { return RED_BLOCKS; }
  // fixed-order sums: one block for RED_BLOCKS partials, two stages for the
  // per-warp partials of the stencil passes
  template <int K>
  void finalize(int nparts, int s0, int s1, int post) {
    if (nparts <= RED_BLOCKS) {
      k_finalize<K><<<1, 256, 0, ctx->stream>>>(ctx->partial, nparts, ctx->sc, s0, s1, s1,
                                                stop, post);
      ++ctx->launches;
      return;
    }
    k_partial_sum_fin<K><<<FIN_BLOCKS, 256, 0, ctx->stream>>>(
        ctx->partial, nparts, ctx->partial2, ctx->sc, s0, s1, stop, post, ctx->ticket_d);
    ++ctx->launches;
  }
  // post: the device-driven iteration's scalar step that needs these sums
  // (POST_DEN / _SS / _END), fused into the sum on one GPU; after the
  // all-reduce as its own kernel on z-slabs
  int post_step(int post) {
    if (post == POST_NONE || !ctx->comm.active()) return 0;
    if (post == POST_DEN) k_bicg_den<<<1, 1, 0, ctx->stream>>>(ctx->sc);
    else if (post == POST_SS) k_bicg_ss<<<1, 1, 0, ctx->stream>>>(ctx->sc);
    else k_bicg_end<<<1, 1, 0, ctx->stream>>>(ctx->sc);
    ++ctx->launches;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  }
  int finalize1(int nparts, int s0, int post = POST_NONE) {
    finalize<1>(nparts, s0, s0, ctx->comm.active() ? POST_NONE : post);
    if (cudaGetLastError() != cudaSuccess) return ISC_CUDA_ERROR;
    const int s = allreduce_dev(ctx, ctx->sc + s0, 1);
    return s ? s : post_step(post);
  }
  int finalize2(int nparts, int s0, int s1, int post = POST_NONE) {   // s1 == s0 + 1
    finalize<2>(nparts, s0, s1, ctx->comm.active() ? POST_NONE : post);
    if (cudaGetLastError() != cudaSuccess) return ISC_CUDA_ERROR;
    const int s = allreduce_dev(ctx, ctx->sc + s0, 2);
    return s ? s : post_step(post);
  }
  int dot(const double* a, const double* b, int slot) {
    k_dots<1><<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(len, a, b, nullptr, nullptr, nullptr,
                                                          nullptr, ctx->partial);
    ++ctx->launches;
    return finalize1(RED_BLOCKS, slot);
  }
  int read_scalars() {
    if (cudaMemcpyAsync(ctx->sc_h, ctx->sc, S_NSCAL * 8, cudaMemcpyDeviceToHost, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      g_err = "scalar readback failed";
      return ISC_CUDA_ERROR;
    }
    kflush(ctx);
    return 0;
  }
  int set(int slot, double v) {
    ctx->sc_h[slot] = v;   // host staging; pushed by push()
    return 0;
  }
  int push() {
    return cudaMemcpyAsync(ctx->sc, ctx->sc_h, S_NSCAL * 8, cudaMemcpyHostToDevice, ctx->stream) ==
                   cudaSuccess ? 0 : ISC_CUDA_ERROR;
  }
};

#define TRY(x) do { int s_ = (x); if (s_) return s_; } while (0)

// linsolve.py:481-578 with b = ctx->rhs, solution in ctx->xk
static int bicgstab(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  const int64_t len = (int64_t)NU * ctx->g.n;
  cudaStream_t st = ctx->stream;
  Kry K{ctx, len};
  double *b = ctx->rhs, *x = ctx->xk, *r = ctx->rk, *rhat = ctx->rhat, *p = ctx->pk,
         *v = ctx->vk, *phat = ctx->phat, *shat = ctx->shat, *s = ctx->sk, *t = ctx->tk;
  CK(cudaMemsetAsync(x, 0, len * 8, st));
  TRY(K.dot(b, b, S_BB));
  TRY(K.read_scalars());
  const double nb = std::sqrt(ctx->sc_h[S_BB]);
  *iters = 0;
  if (nb == 0.0) return ISC_OK;
  const double brk = 1e-30 * nb * nb;
  const bool mc_fused = ctx->precond == ISC_PRECOND_MCILU && ctx->g.colored &&
                        !ctx->comm.active();
  CK(cudaMemsetAsync(t, 0, len * 8, st));   // ghost rows of SpMV outputs stay zero
  CK(cudaMemcpyAsync(r, b, len * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(rhat, b, len * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(p, 0, len * 8, st));
  CK(cudaMemsetAsync(v, 0, len * 8, st));
  double* sh = ctx->sc_h;
  for (int i = 0; i < S_NSCAL; ++i) sh[i] = 0.0;
  sh[S_RHO_OLD] = 1.0; sh[S_ALPHA] = 1.0; sh[S_OMEGA] = 1.0; sh[S_FIRST] = 1.0;
  sh[S_BB] = nb * nb;
  bool restarted = false, first = true;
  int it = 0;
  // rho = rhat . r  (kept in S_RHO_NEW between iterations)
  TRY(K.push());
  TRY(K.dot(rhat, r, S_RHO_NEW));
  TRY(K.read_scalars());
  auto restart = [&]() -> int {
    // r = b - A x; rhat = r; p = v = 0; scalars reset (linsolve.py:509-519)
    if (halo_exchange(ctx, x, NU)) return ISC_CUDA_ERROR;
    if (spmv<0>(ctx, x, t, nullptr, nullptr, nullptr)) return ISC_CUDA_ERROR;
    k_sub<<<RED_BLOCKS, RED_THREADS, 0, st>>>(len, b, t, r);
    ++ctx->launches;
    if (cudaMemcpyAsync(rhat, r, len * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return ISC_CUDA_ERROR;
    cudaMemsetAsync(p, 0, len * 8, st);
    cudaMemsetAsync(v, 0, len * 8, st);
    sh[S_RHO_OLD] = 1.0; sh[S_ALPHA] = 1.0; sh[S_OMEGA] = 1.0;
    first = true;
    restarted = true;
    return 0;
  };
  while (it < maxiter) {
    ++it;
    double rho = sh[S_RHO_NEW];
    const double omega = sh[S_OMEGA];
    if (std::fabs(rho) < brk || (!first && omega == 0.0)) {
      if (restarted) { g_err = "BiCGSTAB scalar breakdown at iteration " + std::to_string(it); *iters = it; return ISC_BREAKDOWN; }
      TRY(restart());
      TRY(K.push());
      TRY(K.dot(rhat, r, S_RHO_NEW));
      TRY(K.read_scalars());
      rho = sh[S_RHO_NEW];
      if (std::fabs(rho) < brk) { g_err = "BiCGSTAB restart found a null residual"; *iters = it; return ISC_BREAKDOWN; }
    }
    sh[S_RHO] = rho;
    sh[S_FIRST] = first ? 1.0 : 0.0;
    first = false;
    TRY(K.push());
    k_update_p<<<RED_BLOCKS, RED_THREADS, 0, st>>>(len, r, p, v, ctx->sc);
    ++ctx->launches;
    int nb1 = 0;
    if (mc_fused) {
      TRY(mc_apply_spmv<1>(ctx, p, phat, v, rhat, nullptr, &nb1));
    } else {
      TRY(precond_apply(ctx, p, phat));
      TRY(halo_exchange(ctx, phat, NU));
      TRY(spmv<1>(ctx, phat, v, rhat, nullptr, &nb1));
    }
    TRY(K.finalize1(nb1, S_DEN));
    // speculative s = r - alpha v, ||s||^2 (used only if den is not a breakdown)
    k_update_s<<<RED_BLOCKS, RED_THREADS, 0, st>>>(len, r, v, s, ctx->sc, ctx->partial);
    ++ctx->launches;
    TRY(K.finalize1(RED_BLOCKS, S_SS));
    TRY(K.read_scalars());
    const double den = sh[S_DEN];
    if (std::fabs(den) < brk) {
      if (restarted) { g_err = "BiCGSTAB denominator breakdown at iteration " + std::to_string(it); *iters = it; return ISC_BREAKDOWN; }
      TRY(restart());
      TRY(K.push());
      TRY(K.dot(rhat, r, S_RHO_NEW));
      TRY(K.read_scalars());
      continue;
    }
    sh[S_ALPHA] = rho / den;
    if (std::sqrt(sh[S_SS]) / nb <= tol) {
      TRY(K.push());
      k_axpy_alpha<<<RED_BLOCKS, RED_THREADS, 0, st>>>(len, x, phat, ctx->sc);
      ++ctx->launches;
      *iters = it;
      CK(cudaStreamSynchronize(st));
      return ISC_OK;
    }
    TRY(K.push());
    int nb2 = 0;
    if (mc_fused) {
      TRY(mc_apply_spmv<2>(ctx, s, shat, t, nullptr, s, &nb2));
    } else {
      TRY(precond_apply(ctx, s, shat));
      TRY(halo_exchange(ctx, shat, NU));
      TRY(spmv<2>(ctx, shat, t, nullptr, s, &nb2));
    }
    TRY(K.finalize2(nb2, S_TT, S_TS));
    k_update_xr<<<RED_BLOCKS, RED_THREADS, 0, st>>>(len, x, phat, shat, r, s, t, rhat, ctx->sc,
                                                     ctx->partial);
    ++ctx->launches;
    TRY(K.finalize2(RED_BLOCKS, S_RR, S_RHO_NEW));
    TRY(K.read_scalars());
    const double tt = sh[S_TT];
    if (tt == 0.0) {
      if (restarted) { g_err = "BiCGSTAB stagnated (t = 0)"; *iters = it; return ISC_BREAKDOWN; }
      TRY(restart());
      TRY(K.push());
      TRY(K.dot(rhat, r, S_RHO_NEW));
      TRY(K.read_scalars());
      continue;
    }
    sh[S_OMEGA] = sh[S_TS] / tt;
    if (std::sqrt(sh[S_RR]) / nb <= tol) { *iters = it; return ISC_OK; }
    sh[S_RHO_OLD] = rho;
  }
  *iters = it;
  g_err = "BiCGSTAB did not converge";
  return ISC_MAX_ITERATIONS;
}

// Half passes of the red-eliminated product, explicit decoupled blocks or
// the compact form (compact.cu); `blocks` covers g's [tw_lo, tw_hi)
static void sc_rhs_launch(isc_ctx* ctx, const Dims& g, int blocks, const double* b, double* o1,
                          double* o2) {
  if (ctx->compact)
    k_cc_rhs<<<blocks, dim3(32, CR), 0, ctx->stream>>>(
        g, ctx->offd, ctx->diag, b, b, o1, o2, nullptr, nullptr, nullptr, 0, 0);
  else
    k_sc_rhs<<<blocks, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, b, o1, o2);
}
static void sc_red_launch(isc_ctx* ctx, const Dims& g, int blocks, double* z,
                          const double* stop = nullptr) {
  if (ctx->compact)
    k_cc_red<<<blocks, dim3(32, CR), 0, ctx->stream>>>(g, ctx->offd, ctx->ccnz_d, z, stop);
  else
    k_sc_red<<<blocks, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, z, stop);
}
static void sc_xred_launch(isc_ctx* ctx, const Dims& g, int blocks, const double* b, double* x) {
  if (ctx->compact)
    k_cc_xred<<<blocks, dim3(32, CR), 0, ctx->stream>>>(
        g, ctx->offd, ctx->diag, x, b, x, nullptr, nullptr, nullptr, nullptr, 0, 0);
  else
    k_sc_xred<<<blocks, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, b, x);
}
// black pass with K dot products; per-warp partial slots: stride x rows_per_block()
template <int K>
static void sc_black_launch(isc_ctx* ctx, const Dims& g, int blocks, const double* z, double* v,
                            const double* w0, const double* w1, int stride, int slot0,
                            const double* stop = nullptr) {
  if (ctx->compact)
    k_cc_black<K><<<blocks, dim3(32, CR), 0, ctx->stream>>>(g, ctx->cbp, ctx->diag, z, v, w0, w1,
                                                            ctx->partial, stride, slot0, stop);
  else
    k_mc_black_spmv<K><<<blocks, dim3(32, NU), 0, ctx->stream>>>(g, ctx->offd, z, v, w0, w1,
                                                                ctx->partial, stride, slot0,
                                                                stop);
}
static int sc_warps(const isc_ctx* ctx) { return ctx->compact ? CR : NU; }

// BiCGSTAB on the red-eliminated system S x_b = g_b with the multicolour
// preconditioner acting as block-Jacobi U_b (solver.cu "Schur complement"
// section): same preconditioner and the same stopping test on the full
// system's residual (its red rows vanish identically), the Krylov vectors
// on the black half, each product reading every off-diagonal block once.
// Control flow as bicgstab() / linsolve.py:481-578.
//
// NC = CR: the condensed form (compact.cu): the same iteration on S6 w = h
// (6-component vectors, Bc / B' / Dc^-1 passes, U6^-1), started at x_b = g_b,
// and x_b = g_b + E_b w at the end.
template <int NC>
static int bicgstab_schur_t(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  constexpr bool cnd = NC == CR;
  const int64_t len = (int64_t)NU * ctx->g.n;      // the full decoupled rhs b
  const int64_t lenv = (int64_t)NC * ctx->g.n;     // Krylov vectors (black positions used)
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  Kry K{ctx, len};
  double *b = ctx->rhs, *x = ctx->xk, *r = ctx->rk, *rhat = ctx->rhat, *p = ctx->pk,
         *v = ctx->vk, *phat = ctx->phat, *shat = ctx->shat, *s = ctx->sk, *t = ctx->tk;
  const double* uinv = ctx->mc_uinv;
  const int bh = grid1d(g.tw_hi - g.tw_lo, 32);   // blocks of a half pass (owned planes)
  CK(cudaMemsetAsync(x, 0, lenv * 8, st));
  *iters = 0;
  // control state first (the dots below write their slots after this push);
  // ||b||, the breakdown threshold and r^.r are formed on the device, so the
  // first chunk of iterations is queued without a host round trip
  double* sh = ctx->sc_h;
  for (int i = 0; i < S_NSCAL; ++i) sh[i] = 0.0;
  sh[S_RHO_OLD] = 1.0; sh[S_ALPHA] = 1.0; sh[S_OMEGA] = 1.0; sh[S_FIRST] = 1.0;
  sh[S_STOP] = STOP_RUN;
  sh[S_MAXIT] = (double)maxiter;
  sh[S_TOL] = tol;
  TRY(K.push());
  TRY(K.dot(b, b, S_BB));   // ||b|| of the full decoupled rhs (the reference's tolerance base)
  // p, v and t need no clearing: p and v are read only after the first
  // iteration wrote them (S_FIRST), t only where the black pass wrote it
  if (cnd) {
    // h = Dc_b^-1 sum_d B'_bd y_r(g_b): the raw red pass on g_b (y into its
    // red positions), then the black pass's product part, into r, rhat, ch6
    // (timed with the vector kernels: the half-pass classes keep the
    // iteration's products only)
    KScope ks(ctx, KT_VEC);
    if (ctx->gb_fresh) {
      ctx->gb_fresh = false;
      // (slabs: g_b of the ghost planes' black cells, then their red cells' y)
      TRY(halo_exchange(ctx, ctx->cg9, NU));
      k_cc_red_bc<<<bh, dim3(32, CR), 0, st>>>(g, ctx->offd, ctx->ccnz_d, ctx->ces, ctx->cg9,
                                               ctx->cbc);
      TRY(halo_exchange(ctx, ctx->cg9, CR));
      k_cc6_black<0, true><<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbp, ctx->diag, ctx->cg9, r,
                                                        nullptr, nullptr, ctx->partial, 0, 0,
                                                        nullptr, rhat, ctx->ch6);
      ctx->launches += 2;
    } else {
      CK(cudaMemcpyAsync(r, ctx->ch6, lenv * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(rhat, ctx->ch6, lenv * 8, cudaMemcpyDeviceToDevice, st));
    }
  } else if (ctx->compact && ctx->gb_fresh) {
    ctx->gb_fresh = false;   // g_b already in r and rhat (k_mc_factor_compact)
  } else {
    TRY(halo_exchange(ctx, b, NU));   // slabs: red neighbours on other ranks
    {
      KScope ks(ctx, KT_SPMV);
      sc_rhs_launch(ctx, g, bh, b, r, rhat);   // g_b
    }
    ++ctx->launches;
  }
  bool restarted = false, first = true;
  int it = 0;
  // One half pass over the owned planes. On slabs the planes next to the
  // ghost planes wait for the halo exchange of their input, the interior
  // runs while it is in flight (red: z_b in, w_r out; black: w_r in, v_b and
  // the dot partials out, partial slots interior | low | high).
  const bool slab = ctx->comm.active();
  auto plane_dims = [&](int64_t k0, int64_t k1) {
    Dims d = g;
    d.tw_lo = k0 * g.ph;
    d.tw_hi = k1 * g.ph;
    return d;
  };
  const int64_t klo = g.kw_lo, khi = g.kw_hi;
  const bool split = slab && khi - klo >= 3;
  const Dims gi = plane_dims(klo + 1, khi - 1), gl = plane_dims(klo, klo + 1),
             gh = plane_dims(khi - 1, khi);
  const int bi = split ? grid1d(gi.tw_hi - gi.tw_lo, 32) : 0;
  const int bl1 = split ? grid1d(gl.tw_hi - gl.tw_lo, 32) : 0;
  const int bh1 = split ? grid1d(gh.tw_hi - gh.tw_lo, 32) : 0;
  const int bparts = split ? bi + bl1 + bh1 : bh;   // black-pass partial slots (blocks)
  auto red_launch = [&](const Dims& d, int blocks, double* z, const double* stop) {
    if (cnd)
      k_cc6_red<<<blocks, dim3(32, CR), 0, st>>>(d, ctx->cbc, z, stop);
    else
      sc_red_launch(ctx, d, blocks, z, stop);
  };
  auto red_pass = [&](double* z, const double* stop) -> int {
    if (!split) {
      TRY(halo_exchange(ctx, z, NC));
      red_launch(g, bh, z, stop);
      ++ctx->launches;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    TRY(halo_start(ctx, z, NC));
    red_launch(gi, bi, z, stop);
    TRY(halo_finish(ctx, z, NC));
    red_launch(gl, bl1, z, stop);
    red_launch(gh, bh1, z, stop);
    ctx->launches += 3;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto black_pass = [&](int K, double* z, double* vout, const double* w0,
                        const double* w1, const double* stop) -> int {
    auto launch = [&](const Dims& d, int blocks, int slot0) {
      if (cnd) {
        if (K == 1)
          k_cc6_black<1, false><<<blocks, dim3(32, CR), 0, st>>>(
              d, ctx->cbp, ctx->diag, z, vout, w0, w1, ctx->partial, bparts, slot0, stop,
              nullptr, nullptr);
        else
          k_cc6_black<2, false><<<blocks, dim3(32, CR), 0, st>>>(
              d, ctx->cbp, ctx->diag, z, vout, w0, w1, ctx->partial, bparts, slot0, stop,
              nullptr, nullptr);
        return;
      }
      if (K == 1)
        sc_black_launch<1>(ctx, d, blocks, z, vout, w0, w1, bparts, slot0, stop);
      else
        sc_black_launch<2>(ctx, d, blocks, z, vout, w0, w1, bparts, slot0, stop);
    };
    if (!split) {
      TRY(halo_exchange(ctx, z, cnd ? CR : NU));
      launch(g, bh, 0);
      ++ctx->launches;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    TRY(halo_start(ctx, z, cnd ? CR : NU));
    launch(gi, bi, 0);
    TRY(halo_finish(ctx, z, cnd ? CR : NU));
    launch(gl, bl1, bi);
    launch(gh, bh1, bi + bl1);
    ctx->launches += 3;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto dot_b = [&](const double* a, const double* c, int slot) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_dot<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, a, c, ctx->partial);
    ++ctx->launches;
    return K.finalize1(RED_BLOCKS, slot);
  };
  auto finish = [&]() -> int {   // x_r = b_r - B_rb x_b
    if (cnd && ctx->h_du && !ctx->comm.active() && x == ctx->xk) {
      // du goes to the host (isc_solve_host): the same kernels per plane
      // chunk, each chunk's transpose + copy (copy stream) under the next
      // chunk's kernels. A red cell reads w of the black cells one plane
      // below and above it, so chunk q + 1's back-substitution runs before
      // chunk q's x_b overwrites w.
      KScope ks(ctx, KT_VEC);
      const int nq = std::min(6, g.nz);
      auto gq_of = [&](int q) {
        Dims gq = g;
        gq.tw_lo = (int64_t)(g.nz * (int64_t)q / nq) * g.ph;
        gq.tw_hi = (int64_t)(g.nz * (int64_t)(q + 1) / nq) * g.ph;
        return gq;
      };
      auto xred_q = [&](int q) {
        const Dims gq = gq_of(q);
        k_cc6_xred<<<grid1d(gq.tw_hi - gq.tw_lo, 32), dim3(32, CR), 0, st>>>(gq, ctx->cbc, ctx->diag,
                                                                             ctx->cg9, b, x);
      };
      xred_q(0);
      for (int q = 0; q < nq; ++q) {
        if (q + 1 < nq) xred_q(q + 1);
        const Dims gq = gq_of(q);
        const int64_t cnt = gq.tw_hi - gq.tw_lo;
        k_cond_expand<<<(int)std::min<int64_t>(RED_BLOCKS, grid1d(cnt, RED_THREADS)), RED_THREADS, 0,
                        st>>>(gq, ctx->ces, ctx->cg9, x);
        const int64_t c0 = 2 * gq.tw_lo, c1 = 2 * gq.tw_hi;   // the chunk's planes, both colours
        k_unstage_rows<<<grid1d(c1 - c0, 256), 256, 0, st>>>(g, x, ctx->stage, c0, c1);
        if (cudaEventRecord(ctx->chunk_ev[q], st) != cudaSuccess) return ISC_CUDA_ERROR;
        if (cudaStreamWaitEvent(ctx->cstream, ctx->chunk_ev[q], 0) != cudaSuccess) return ISC_CUDA_ERROR;
        if (cudaMemcpyAsync(ctx->h_du + c0 * NU, ctx->stage + c0 * NU, (size_t)(c1 - c0) * NU * 8,
                            cudaMemcpyDeviceToHost, ctx->cstream) != cudaSuccess)
          return ISC_CUDA_ERROR;
        ctx->launches += 3;
      }
      ctx->h_du_queued = true;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    if (cnd) {   // x_r from w and y_r(g), then x_b = g_b + E_b w
      if (halo_exchange(ctx, x, CR)) return ISC_CUDA_ERROR;
      KScope ks(ctx, KT_VEC);
      k_cc6_xred<<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbc, ctx->diag, ctx->cg9, b, x);
      k_cond_expand<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, ctx->ces, ctx->cg9, x);
      ctx->launches += 2;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    if (halo_exchange(ctx, x, NU)) return ISC_CUDA_ERROR;
    KScope ks(ctx, KT_SPMV);
    sc_xred_launch(ctx, g, bh, b, x);
    ++ctx->launches;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  TRY(dot_b(rhat, r, S_RHO_NEW));
  k_bicg_init<<<1, 1, 0, st>>>(ctx->sc);   // S_NB, S_BRK; ||b|| = 0 stops at once
  ++ctx->launches;
  auto restart = [&]() -> int {
    // r_b = g_b - S x_b; rhat = r; p = v = 0 (linsolve.py:509-519)
    {
      KScope ks(ctx, KT_SPMV);
      if (red_pass(x, nullptr)) return ISC_CUDA_ERROR;   // red part of x: scratch
      if (black_pass(1, x, t, rhat, nullptr, nullptr)) return ISC_CUDA_ERROR;
      if (!cnd) sc_rhs_launch(ctx, g, bh, b, v, shat);   // g_b (scratch)
    }
    k_sc_sub<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, cnd ? ctx->ch6 : v, t, r, rhat);
    ctx->launches += 4;
    cudaMemsetAsync(p, 0, lenv * 8, st);
    cudaMemsetAsync(v, 0, lenv * 8, st);
    sh[S_RHO_OLD] = 1.0; sh[S_ALPHA] = 1.0; sh[S_OMEGA] = 1.0;
    first = true;
    restarted = true;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  // Device-driven iterations: the scalar logic runs in k_bicg_* between the
  // vector kernels and every kernel returns at once after S_STOP is set, so
  // chunks of iterations are enqueued without a host round trip (the
  // host-driven form synchronised twice per iteration). The first chunk is
  // sized from the previous solve's count, then two at a time. The host
  // handles each stop code exactly as linsolve.py:500-578 branches.
  // (After a stop, the skipped finalize kernels leave their slots alone but
  // a multi-rank all-reduce still sums them again; only slots the next
  // restart or iteration recomputes are affected.)
  double* stop = ctx->sc + S_STOP;
  K.stop = stop;
  auto enqueue_iteration = [&]() -> int {
    k_bicg_top<<<1, 1, 0, st>>>(ctx->sc);
    {
      KScope ks(ctx, KT_VEC);
      k_sc_update_p<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, p, v, uinv, phat, ctx->sc, stop);
    }
    {
      KScope ks(ctx, KT_ILU_APPLY);
      TRY(red_pass(phat, stop));
    }
    {
      KScope ks(ctx, KT_SPMV);
      TRY(black_pass(1, phat, v, rhat, nullptr, stop));
    }
    CK(cudaGetLastError());
    TRY(K.finalize1(bparts * sc_warps(ctx), S_DEN, POST_DEN));
    {
      KScope ks(ctx, KT_VEC);
      k_sc_update_s<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, v, s, uinv, shat, ctx->sc,
                                                        ctx->partial, stop);
    }
    TRY(K.finalize1(RED_BLOCKS, S_SS, POST_SS));
    {
      KScope ks(ctx, KT_ILU_APPLY);
      TRY(red_pass(shat, stop));
    }
    {
      KScope ks(ctx, KT_SPMV);
      TRY(black_pass(2, shat, t, nullptr, s, stop));
    }
    CK(cudaGetLastError());
    TRY(K.finalize2(bparts * sc_warps(ctx), S_TT, S_TS));
    {
      KScope ks(ctx, KT_VEC);
      k_sc_update_xr<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, x, phat, shat, r, s, t, rhat,
                                                         ctx->sc, ctx->partial, stop);
    }
    TRY(K.finalize2(RED_BLOCKS, S_RR, S_RHO_NEW, POST_END));
    ctx->launches += 4;   // 3 vector updates + k_bicg_top (passes, sums and steps count themselves)
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  // a restart by the host: device state -> sh, restart, new rho, state -> HBM
  auto host_restart = [&]() -> int {
    sh[S_STOP] = STOP_RUN;
    K.stop = nullptr;
    TRY(K.push());
    TRY(restart());
    sh[S_FIRST] = 1.0;
    TRY(K.push());
    TRY(dot_b(rhat, r, S_RHO_NEW));
    TRY(K.read_scalars());
    K.stop = stop;
    return 0;
  };
  int chunk = std::max(1, std::min(16, ctx->bicg_last_iters > 0 ? ctx->bicg_last_iters - 1 : 4));
  for (;;) {
    for (int c = 0; c < chunk; ++c) TRY(enqueue_iteration());
    TRY(K.read_scalars());
    chunk = 2;
    const int code = (int)sh[S_STOP];
    it = (int)sh[S_IT];
    if (code == STOP_RUN) continue;
    *iters = it;
    if (code == STOP_ZERO) {   // b = 0: x = 0 (linsolve.py:486-487)
      sh[S_STOP] = STOP_RUN;
      return K.push();
    }
    ctx->bicg_last_iters = it;
    const double brk = sh[S_BRK];
    if (code == STOP_CONV_S) {   // ||s|| / ||b|| <= tol: x += alpha phat (linsolve.py:550-552)
      sh[S_STOP] = STOP_RUN;
      TRY(K.push());
      k_sc_axpy_alpha<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, x, phat, ctx->sc);
      ++ctx->launches;
      TRY(finish());
      CK(cudaStreamSynchronize(st));
      return ISC_OK;
    }
    if (code == STOP_CONV) {
      sh[S_STOP] = STOP_RUN;
      TRY(K.push());
      TRY(finish());
      return ISC_OK;
    }
    if (code == STOP_MAXIT) {
      sh[S_STOP] = STOP_RUN;
      TRY(K.push());
      g_err = "BiCGSTAB did not converge";
      return ISC_MAX_ITERATIONS;
    }
    if (restarted) {
      sh[S_STOP] = STOP_RUN;
      TRY(K.push());
      g_err = code == STOP_TOP ? "BiCGSTAB scalar breakdown at iteration " + std::to_string(it)
            : code == STOP_DEN ? "BiCGSTAB denominator breakdown at iteration " + std::to_string(it)
                               : std::string("BiCGSTAB stagnated (t = 0)");
      return ISC_BREAKDOWN;
    }
    TRY(host_restart());   // the single restart from the current iterate
    if (code == STOP_TOP) {
      // restart at the loop head: the same iteration continues with the new
      // rho (linsolve.py:509-522) -- the next k_bicg_top counts it again
      if (std::fabs(sh[S_RHO_NEW]) < brk) {
        g_err = "BiCGSTAB restart found a null residual";
        return ISC_BREAKDOWN;
      }
      sh[S_IT] = it - 1;
      TRY(K.push());
    }
    chunk = 1;
  }
}
static int bicgstab_schur(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  return ctx->cond ? bicgstab_schur_t<CR>(ctx, tol, maxiter, iters)
                   : bicgstab_schur_t<NU>(ctx, tol, maxiter, iters);
}

// Restarted right-preconditioned GMRES(m) on the red-eliminated system
// S x_b = g_b with U_b block-Jacobi (the north star's "BiCGSTAB/GMRES";
// optional, isc_set_krylov). Arnoldi with classical Gram-Schmidt and one
// reorthogonalisation (CGS2): two fused multi-dots and two multi-axpys per
// step, the second one also giving ||w||; the Hessenberg column goes to the
// host once per step for the Givens rotations. One product S U_b^-1 per
// iteration (BiCGSTAB: two). Stopping test as bicgstab_schur: ||r|| / ||b||
// of the full system (the Givens residual estimate within a cycle, the true
// reduced residual at each restart).
// NC = CR: the condensed form (as bicgstab_schur_t): S6 w = h from w = 0,
// x_b = g_b + E_b w at the end.
template <int NC>
static int gmres_schur_t(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  constexpr bool cnd = NC == CR;
  const int64_t len9 = (int64_t)NU * ctx->g.n;   // the full decoupled rhs b
  const int64_t len = (int64_t)NC * ctx->g.n;    // Krylov vectors and basis stride
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  Kry K{ctx, len9};
  const int m = std::max(1, std::min(ctx->gm_m, GM_MAXV - 1));
  if (!ctx->gm_V) {
    if (cudaMalloc(&ctx->gm_V, (size_t)GM_MAXV * len9 * 8) != cudaSuccess ||
        cudaMalloc(&ctx->gm_h, (size_t)4 * (GM_MAXV + 1) * 8) != cudaSuccess) {
      cudaGetLastError();
      g_err = "cannot allocate the GMRES basis";
      return ISC_CUDA_ERROR;
    }
  }
  double *b = ctx->rhs, *x = ctx->xk, *r = ctx->rk, *z = ctx->phat, *t = ctx->tk,
         *gb = ctx->shat, *u = ctx->sk;
  double* V = ctx->gm_V;
  double *h1 = ctx->gm_h, *h2 = h1 + (GM_MAXV + 1), *yd = h2 + (GM_MAXV + 1);
  const double* uinv = ctx->mc_uinv;
  const int bh = grid1d(g.tw_hi - g.tw_lo, 32);
  CK(cudaMemsetAsync(x, 0, len * 8, st));
  TRY(K.dot(b, b, S_BB));
  TRY(K.read_scalars());
  const double nb = std::sqrt(ctx->sc_h[S_BB]);
  *iters = 0;
  if (nb == 0.0) return ISC_OK;
  if (cnd) {   // h into r and gb (as bicgstab_schur_t)
    KScope ks(ctx, KT_VEC);
    if (ctx->gb_fresh) {
      ctx->gb_fresh = false;
      TRY(halo_exchange(ctx, ctx->cg9, NU));
      k_cc_red_bc<<<bh, dim3(32, CR), 0, st>>>(g, ctx->offd, ctx->ccnz_d, ctx->ces, ctx->cg9,
                                               ctx->cbc);
      TRY(halo_exchange(ctx, ctx->cg9, CR));
      k_cc6_black<0, true><<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbp, ctx->diag, ctx->cg9, r,
                                                        nullptr, nullptr, ctx->partial, 0, 0,
                                                        nullptr, gb, ctx->ch6);
      ctx->launches += 2;
    } else {
      CK(cudaMemcpyAsync(r, ctx->ch6, len * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(gb, ctx->ch6, len * 8, cudaMemcpyDeviceToDevice, st));
    }
  } else if (ctx->compact && ctx->gb_fresh) {   // g_b from the factorisation
    ctx->gb_fresh = false;
    CK(cudaMemcpyAsync(gb, r, len * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    TRY(halo_exchange(ctx, b, NU));
    {
      KScope ks(ctx, KT_SPMV);
      sc_rhs_launch(ctx, g, bh, b, r, gb);   // r = g_b (x_b = 0)
    }
    ++ctx->launches;
  }
  auto matvec = [&](double* zz, double* out) -> int {   // out = S zz (zz: black in, red scratch)
    {
      KScope ks(ctx, KT_ILU_APPLY);
      TRY(halo_exchange(ctx, zz, NC));
      if (cnd)
        k_cc6_red<<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbc, zz, nullptr);
      else
        sc_red_launch(ctx, g, bh, zz);
    }
    {
      KScope ks(ctx, KT_SPMV);
      TRY(halo_exchange(ctx, zz, cnd ? CR : NU));
      if (cnd)
        k_cc6_black<1, false><<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbp, ctx->diag, zz, out, zz,
                                                           nullptr, ctx->partial, bh, 0, nullptr,
                                                           nullptr, nullptr);
      else
        sc_black_launch<1>(ctx, g, bh, zz, out, zz, nullptr, bh, 0);
    }
    ctx->launches += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto norm2_into = [&](const double* a, int slot) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_dot<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, a, a, ctx->partial);
    ++ctx->launches;
    return K.finalize1(RED_BLOCKS, slot);
  };
  auto multidot = [&](int nv, const double* w, double* hout) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_multidot<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, nv, w, ctx->partial);
    k_sum_partials<<<GM_MAXV + 1, 32, 0, st>>>(ctx->partial, RED_BLOCKS, GM_MAXV + 1, hout);
    ctx->launches += 2;
    if (cudaGetLastError() != cudaSuccess) return ISC_CUDA_ERROR;
    return allreduce_dev(ctx, hout, GM_MAXV + 1);
  };
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gv(m + 1), hc(2 * (GM_MAXV + 1)),
      y(m);
  int it = 0;
  TRY(norm2_into(r, S_RR));
  TRY(K.read_scalars());
  double beta = std::sqrt(ctx->sc_h[S_RR]);
  for (;;) {
    if (beta / nb <= tol) break;
    if (it >= maxiter) {
      *iters = it;
      g_err = "GMRES did not converge";
      return ISC_MAX_ITERATIONS;
    }
    {
      KScope ks(ctx, KT_VEC);
      k_sc_scale<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, ctx->sc + S_RR, V);   // v0 = r / beta
    }
    ++ctx->launches;
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int j = 0;
    double res = beta;
    for (; j < m && it < maxiter; ++j) {
      ++it;
      double* vj = V + (int64_t)j * len;
      double* w = V + (int64_t)(j + 1) * len;
      {
        KScope ks(ctx, KT_VEC);
        k_sc_precond<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, vj, uinv, z);
      }
      ++ctx->launches;
      TRY(matvec(z, w));
      TRY(multidot(j + 1, w, h1));
      {
        KScope ks(ctx, KT_VEC);
        k_sc_multiaxpy<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j + 1, h1, 1.0, w, 0,
                                                               nullptr);
      }
      ++ctx->launches;
      TRY(multidot(j + 1, w, h2));
      {
        KScope ks(ctx, KT_VEC);
        k_sc_multiaxpy<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j + 1, h2, 1.0, w, 0,
                                                               ctx->partial);
      }
      ++ctx->launches;
      TRY(K.finalize1(RED_BLOCKS, S_TT));   // ||w||^2 after CGS2
      CK(cudaMemcpyAsync(hc.data(), h1, 2 * (GM_MAXV + 1) * 8, cudaMemcpyDeviceToHost, st));
      TRY(K.read_scalars());
      double* col = &H[(size_t)j * (m + 1)];
      for (int i = 0; i <= j; ++i) col[i] = hc[i] + hc[GM_MAXV + 1 + i];
      const double hn = std::sqrt(ctx->sc_h[S_TT]);
      col[j + 1] = hn;
      if (!std::isfinite(hn)) {
        *iters = it;
        g_err = "GMRES breakdown (non-finite Arnoldi vector)";
        return ISC_BREAKDOWN;
      }
      if (hn > 0.0) {
        KScope ks(ctx, KT_VEC);
        k_sc_scale<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, w, ctx->sc + S_TT, w);
        ++ctx->launches;
      }
      for (int i = 0; i < j; ++i) {
        const double a = cs[i] * col[i] + sn[i] * col[i + 1];
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
        col[i] = a;
      }
      const double rr = std::hypot(col[j], col[j + 1]);
      if (rr == 0.0) {
        *iters = it;
        g_err = "GMRES breakdown (singular Hessenberg)";
        return ISC_BREAKDOWN;
      }
      cs[j] = col[j] / rr;
      sn[j] = col[j + 1] / rr;
      col[j] = rr;
      col[j + 1] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      res = std::fabs(gv[j + 1]);
      if (res / nb <= tol || hn == 0.0) { ++j; break; }
    }
    // y = R^-1 g; x_b += U_b^-1 (V y)
    for (int i = j - 1; i >= 0; --i) {
      double a = gv[i];
      for (int k = i + 1; k < j; ++k) a -= H[(size_t)k * (m + 1) + i] * y[k];
      y[i] = a / H[(size_t)i * (m + 1) + i];
    }
    CK(cudaMemcpyAsync(yd, y.data(), j * 8, cudaMemcpyHostToDevice, st));
    {
      KScope ks(ctx, KT_VEC);
      k_sc_multiaxpy<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j, yd, -1.0, u, 1,
                                                             nullptr);
      k_sc_precond<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, u, uinv, z);
      k_sc_add<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, z, x);
    }
    ctx->launches += 3;
    if (res / nb <= tol) break;
    // restart: r_b = g_b - S x_b
    CK(cudaMemcpyAsync(u, x, len * 8, cudaMemcpyDeviceToDevice, st));
    TRY(matvec(u, t));
    k_sc_sub<NC><<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, gb, t, r, z);
    ++ctx->launches;
    TRY(norm2_into(r, S_RR));
    TRY(K.read_scalars());
    beta = std::sqrt(ctx->sc_h[S_RR]);
  }
  if (cnd) {   // x_r from w and y_r(g), then x_b = g_b + E_b w
    TRY(halo_exchange(ctx, x, CR));
    KScope ks(ctx, KT_VEC);
    k_cc6_xred<<<bh, dim3(32, CR), 0, st>>>(g, ctx->cbc, ctx->diag, ctx->cg9, b, x);
    k_cond_expand<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, ctx->ces, ctx->cg9, x);
    ctx->launches += 2;
    *iters = it;
    CK(cudaStreamSynchronize(st));
    return ISC_OK;
  }
  // x_r = b_r - B_rb x_b
  TRY(halo_exchange(ctx, x, NU));
  {
    KScope ks(ctx, KT_SPMV);
    sc_xred_launch(ctx, g, bh, b, x);
  }
  ++ctx->launches;
  *iters = it;
  CK(cudaStreamSynchronize(st));
  return ISC_OK;
}
static int gmres_schur(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  return ctx->cond ? gmres_schur_t<CR>(ctx, tol, maxiter, iters)
                   : gmres_schur_t<NU>(ctx, tol, maxiter, iters);
}

// 0: not decoupled, 1: explicit decoupled blocks, 2: compact form (compact.cu)
