// Numeric (finite-difference) Jacobian on the device: the reference's
// JACOBIAN numeric mode and the FD half of --check-jacobian
// (assembly.py:601-939).
//
//   k_numjac        one thread per (cell, unknown u): the two probe states of
//                   _fd_points (807-840), cell_eval + compose at each
//                   (_probe_rows 722-804, values only: CellSinkProbe keeps
//                   the record fields and rows in registers), the six faces'
//                   flux rows against the neighbours' unperturbed records in
//                   the reference's adjacency order, the cell's perforation
//                   rows, then column u of the cell's diagonal block, of the
//                   six neighbours' blocks pointing back at the cell and the
//                   well rows (wrow) — (rows+ - rows-) / (v+ - v-).
//   k_numjac_wells  one thread: each well's bhp column (bcol) and dwdb from
//                   central probes of bhp (903-939).
//
// Runs after the analytic assemble at the same inputs (residuals and well
// residuals stay the analytic pass's); every column of every block it owns is
// overwritten, so the off-diagonal rows ROW_OS.. become data (zeros).
// (included by capi.cu after assemble.cu)

namespace isc {

constexpr double FD_REL_STEP = 1e-6, FD_PRESSURE_FLOOR = 1e-3, FD_UNIT_FLOOR = 5e-5;

// probe values (v+, v-) for unknown u (assembly.py:807-840)
__device__ __forceinline__ void fd_points(int u, const double (&base)[NU], double sw, double sg,
                                          double& vp, double& vm) {
  const double v = base[u];
  if (u == 0) {
    const double h = fmax(FD_REL_STEP * fabs(v), FD_PRESSURE_FLOOR);
    vp = v + h; vm = v - h;
    return;
  }
  const double h = fmax(FD_REL_STEP * fabs(v), FD_UNIT_FLOOR);
  vp = v + h; vm = v - h;
  if (u == CT) return;
  if (u == CSW || u == CSG) {
    if (v - h < 0.0) { vp = v + h; vm = v; }
    else if (1.0 - sw - sg - h < 0.0) { vp = v; vm = v - h; }
    return;
  }
  if (u == CCC) {
    if (v - h < 0.0) { vp = v + h; vm = v; }
    return;
  }
  if (v - h < 0.0) { vp = v + h; vm = v; }
  else if (v + h > 1.0) { vp = v; vm = v - h; }
}

// Flux rows of one connection, values only, in conn_eval's per-row
// accumulation order (_kernels.py:677-771; face_row without partials).
template <class RA, class RB>
__device__ __forceinline__ void face_flux_values(const RA& A_, const RB& B_, const double* xa,
                                                 const double* xb, double ta, double tb,
                                                 double za, double zb, double gd, double td,
                                                 const int8_t* upw, int64_t upw_stride,
                                                 int64_t a_pos, int freeze, double (&flux)[NU]) {
#pragma unroll
  for (int r = 0; r < NU; ++r) flux[r] = 0.0;
#pragma unroll
  for (int al = 0; al < 3; ++al) {
    const double phi_a = A_.f(R_POT + al) - A_.f(R_GAM + al) * za;
    const double phi_b = B_.f(R_POT + al) - B_.f(R_GAM + al) * zb;
    const double dphi = phi_a - phi_b;
    const bool up_a = freeze ? upw[al * upw_stride + a_pos] == 1 : dphi >= 0.0;
    const double conv = gd * dphi;
    const double b_up = up_a ? A_.f(R_BETA + al) : B_.f(R_BETA + al);
    if (al == 0) {
      const double val = b_up * 1.0;
      flux[0] += conv * val;
    } else if (al == 1) {
#pragma unroll
      for (int m = 0; m < NCO; ++m) {
        const double val = b_up * (up_a ? xa[m] : xb[m]);
        flux[1 + m] += conv * val;
      }
    } else {
#pragma unroll
      for (int m = 0; m < NF; ++m) {
        const double val = b_up * (up_a ? A_.f(R_Y + m) : B_.f(R_Y + m));
        flux[m] += conv * val;
      }
    }
    const double val = b_up * (up_a ? A_.f(R_HPH + al) : B_.f(R_HPH + al));
    flux[ROW_E] += conv * val;
  }
  double hm, dh_a, dh_b;
  harmonic_pair(A_.f(R_KT), B_.f(R_KT), hm, dh_a, dh_b);
  if (hm > 0.0 || dh_a != 0.0 || dh_b != 0.0) flux[ROW_E] += td * hm * (ta - tb);
}

// Perforation rows and total rate at bhp, values only (assembly.py:370-471;
// k_wells without partials). V is the cell's record accessor.
template <class R>
__device__ __forceinline__ void perf_values(const Model& M, const WellDev& W, const R& V,
                                            const double* x_c, double bh, double dz,
                                            double (&rows)[NU], double& qsum) {
#pragma unroll
  for (int r = 0; r < NU; ++r) rows[r] = 0.0;
  const double cwi = DARCY_CONST * W.wi;
  double qph[3] = {0.0, 0.0, 0.0};
  if (W.kind == 0) {
    const double lam = V.f(R_LAM);
    const double pg = V.f(R_POT + 2);
    double dzdw[NF], dzdp, dzdt;
    const double zf = z_factor_mix<NF>(W.s_yfull, M.gasp, pg, W.s_tinj, dzdw, dzdp, dzdt);
    const double trs = W.s_tinj + RANKINE;
    const double rho = pg / (zf * R_GAS * trs);
    const double gam = rho * W.s_mbar / 144.0;
    const double dd = bh - pg - gam * dz;
    const double mob = rho * lam / W.s_mu;
    const double q = cwi * mob * dd;
#pragma unroll
    for (int j = 0; j < NCG; ++j) rows[1 + NCO + j] = q * W.s_yinj[j];
    rows[ROW_E] = q * W.s_h;
    qph[2] = q;
  } else {
#pragma unroll
    for (int al = 0; al < 3; ++al) {
      const double beta = V.f(R_BETA + al);
      const double dd = bh - V.f(R_POT + al) - V.f(R_GAM + al) * dz;
      const double q = cwi * beta * dd;
      qph[al] = q;
      if (al == 0) {
        rows[0] += q;
      } else if (al == 1) {
#pragma unroll
        for (int i = 0; i < NCO; ++i) rows[1 + i] += q * x_c[i];
      } else {
#pragma unroll
        for (int m = 0; m < NF; ++m) rows[m] += q * V.f(R_Y + m);
      }
      rows[ROW_E] += q * V.f(R_HPH + al);
    }
  }
  qsum = qph[0] + qph[1] + qph[2];
}

struct NumJacArgs {
  CellArgs A;                      // cell_eval inputs (st, phi_ref, vol, accn, dt, heat loss)
  const double* __restrict__ rec;  // unperturbed records of the analytic pass
  const double* __restrict__ depth;
  const double* __restrict__ gd;
  const double* __restrict__ td;
  const int8_t* __restrict__ upw;
  int freeze;
  double* __restrict__ diag;
  double* __restrict__ offd;
  int nw;
  const WellDev* __restrict__ wells;
  const double* __restrict__ bhp;
  const uint8_t* __restrict__ capped;
  double* wout;
  unsigned long long* bad;
};

// grid (ceil(n/32)), block (32, NU): threadIdx.y = unknown u
#ifndef NJ_MINB
#define NJ_MINB 3   // C4 FD Jacobian: 30.3 / 27.6 / 22.9 / 23.3 ms at 1..4
#endif
__global__ void __launch_bounds__(32 * NU, NJ_MINB) k_numjac(const Model M, const NumJacArgs J) {
  const Dims& g = J.A.g;
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int u = threadIdx.y;
  if (c >= n) return;
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double base[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) base[q] = J.A.st[q * n + c];
  double vp, vm;
  fd_points(u, base, base[CSW], base[CSG], vp, vm);
  double up[NU], um[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) { up[q] = base[q]; um[q] = base[q]; }
#pragma unroll
  for (int q = 0; q < NU; ++q)
    if (q == u) { up[q] = vp; um[q] = vm; }
  CellSinkProbe P, Q;
  cell_eval(M, J.A, c, up, P);
  cell_eval(M, J.A, c, um, Q);
  if (P.failed || Q.failed) {   // PoreSpaceExhausted at a probed state (assembly.py:682-684)
    atomicMin(J.bad, (unsigned long long)cell);
    return;
  }
  const double inv2h = 1.0 / (vp - vm);
  double rp[NU], rm[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) { rp[r] = P.rows[r]; rm[r] = Q.rows[r]; }
  const double xp[NCO] = {up[1], up[2]}, xm[NCO] = {um[1], um[2]};
  static_assert(NCO == 2, "probe x arrays");
#pragma unroll 1
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) {   // boundary: the cell's own block column is zero
#pragma unroll
      for (int r = 0; r < NU; ++r) J.offd[(int64_t)((d * NU + r) * NU + u) * n + c] = 0.0;
      continue;
    }
    const bool c_is_a = d >= DXP;
    const int axis = c_is_a ? d - DXP : 2 - d;
    const int64_t a = c_is_a ? c : nb;
    const CellView NB{J.rec, n, nb};
    const double xnb[NCO] = {J.A.st[1 * n + nb], J.A.st[2 * n + nb]};
    const double tnb = J.A.st[CT * n + nb];
    const double zc = J.depth[c], znb = J.depth[nb];
    const double gdv = J.gd[axis * n + a], tdv = J.td[axis * n + a];
    const int8_t* upw = J.upw + (int64_t)axis * 3 * n;
    double fp[NU], fm[NU];
    if (c_is_a) {
      face_flux_values(P, NB, xp, xnb, up[CT], tnb, zc, znb, gdv, tdv, upw, n, a, J.freeze, fp);
      face_flux_values(Q, NB, xm, xnb, um[CT], tnb, zc, znb, gdv, tdv, upw, n, a, J.freeze, fm);
    } else {
      face_flux_values(NB, P, xnb, xp, tnb, up[CT], znb, zc, gdv, tdv, upw, n, a, J.freeze, fp);
      face_flux_values(NB, Q, xnb, xm, tnb, um[CT], znb, zc, gdv, tdv, upw, n, a, J.freeze, fm);
    }
    const int od = opposite(d);
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      double col;
      if (c_is_a) {   // neighbour is side b: its row is -flux
        rp[r] += fp[r];
        rm[r] += fm[r];
        col = (-fp[r] - -fm[r]) * inv2h;
      } else {        // neighbour is side a: its row is +flux
        rp[r] -= fp[r];
        rm[r] -= fm[r];
        col = (fp[r] - fm[r]) * inv2h;
      }
      J.offd[(int64_t)((od * NU + r) * NU + u) * n + nb] = col;
    }
  }
  for (int w = 0; w < J.nw; ++w) {
    const WellDev W = J.wells[w];
    if (W.cell != c) continue;
    const double dz = W.z_bh - J.depth[c];
    double prow[NU], qp, qm;
    perf_values(M, W, P, xp, J.bhp[w], dz, prow, qp);
#pragma unroll
    for (int r = 0; r < NU; ++r) rp[r] -= prow[r];
    perf_values(M, W, Q, xm, J.bhp[w], dz, prow, qm);
#pragma unroll
    for (int r = 0; r < NU; ++r) rm[r] -= prow[r];
    const bool rate = W.control != 0 && !J.capped[w];
    J.wout[(int64_t)w * WOUT + 2 + u] = rate ? ((0.0 + qp) - (0.0 + qm)) * inv2h : 0.0;
  }
#pragma unroll
  for (int r = 0; r < NU; ++r) J.diag[(int64_t)(r * NU + u) * n + c] = (rp[r] - rm[r]) * inv2h;
}

// bhp columns and dwdb (assembly.py:903-939), one thread, wells in order
__global__ void k_numjac_wells(const Model M, Dims g, int nw, const WellDev* __restrict__ wells,
                               const double* __restrict__ st, const double* __restrict__ bhp,
                               const uint8_t* __restrict__ capped,
                               const double* __restrict__ rec, const double* __restrict__ depth,
                               double* wout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t n = g.n;
  for (int w = 0; w < nw; ++w) {
    const WellDev W = wells[w];
    const int64_t c = W.cell;
    const CellView V{rec, n, c};
    const double b0 = bhp[w];
    const double h = fmax(FD_REL_STEP * fabs(b0), FD_PRESSURE_FLOOR);
    const double dz = W.z_bh - depth[c];
    const double x_c[NCO] = {st[1 * n + c], st[2 * n + c]};
    double rp[NU], rm[NU], qp, qm;
    perf_values(M, W, V, x_c, b0 + h, dz, rp, qp);
    perf_values(M, W, V, x_c, b0 - h, dz, rm, qm);
    double* o = wout + (int64_t)w * WOUT;
    const double inv2h = 0.5 / h;
#pragma unroll
    for (int r = 0; r < NU; ++r) o[2 + NU + r] = -(rp[r] - rm[r]) * inv2h;
    if (W.control == 0 || capped[w]) o[1] = 1.0;
    else o[1] = 0.0 + (qp - qm) * 0.5 / h;
  }
}

}  // namespace isc
