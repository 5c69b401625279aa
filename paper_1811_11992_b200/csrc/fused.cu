// Fused face assembly + well Schur fold + Gauss-Jordan decoupling.
//
// The drop-in path (isc_assemble -> isc_solve) writes the assembled
// block rows to HBM (k_face), reads them back to decouple (k_decouple) and
// writes them again. Here the six faces' derivative columns are computed
// straight into the registers of the threads that own those columns of the
// augmented block row [D | B_-z .. B_+z | rhs] (9 x 64), the diagonal block
// is reduced from the per-face own-derivatives through shared memory in the
// reference's gather order, and the row is decoupled in place: only the
// decoupled off-diagonal blocks, the rhs and the residual reach HBM.
//
// Well terms and the Schur fold are additive updates of the cell-local
// diagonal block / residual (assembly.py:500-510, linsolve.py:378-386) and
// are applied before the faces (k_wells on the cell parts, k_schur_pre).
// Same arithmetic per term as k_face / k_decouple; only the summation order
// of the well and face contributions differs (rounding level).
#include "common.cuh"
#include "record.cuh"

namespace isc {

// single column u of the record partials (CellView gives dense 9-vectors)
struct ColView {
  const double* __restrict__ rec;
  int64_t n, c;
  __device__ __forceinline__ double f(int k) const { return rec[(int64_t)k * n + c]; }
  __device__ __forceinline__ double dpot(int al, int u) const {
    if (u == 0) return 1.0;
    if (al == 0 && u == CSW) return f(R_DPOT0_SW);
    if (al == 2 && u == CSG) return f(R_DPOT2_SG);
    return 0.0;
  }
  __device__ __forceinline__ double dgam(int al, int u) const {
    if (al == 2) return f(R_DGAM2 + u);
    if (al == 0) return u == 0 ? f(R_DGAM0_P) : (u == CT ? f(R_DGAM0_T) : 0.0);
    if (u == 0) return f(R_DGAM1_P);
    if (u == CT) return f(R_DGAM1_T);
    if (u >= 1 && u <= NCO) return f(R_DGAM1_X + u - 1);
    return 0.0;
  }
  __device__ __forceinline__ double dbeta(int al, int u) const {
    if (al == 2) return f(R_DBETA2 + u);
    if (al == 0) {
      if (u == 0) return f(R_DBETA0_P);
      if (u == CT) return f(R_DBETA0_T);
      if (u == CSW) return f(R_DBETA0_SW);
      return 0.0;
    }
    if (u == 0) return f(R_DBETA1_P);
    if (u == CT) return f(R_DBETA1_T);
    if (u == CSW) return f(R_DBETA1_SW);
    if (u == CSG) return f(R_DBETA1_SG);
    if (u >= 1 && u <= NCO) return f(R_DBETA1_X + u - 1);
    return 0.0;
  }
  __device__ __forceinline__ double dhph(int al, int u) const {
    if (al == 2) return f(R_DHPH2 + u);
    if (al == 0) return u == CT ? f(R_DHPH0_T) : 0.0;
    if (u == CT) return f(R_DHPH1_T);
    if (u >= 1 && u <= NCO) return f(R_DHPH1_X + u - 1);
    return 0.0;
  }
  __device__ __forceinline__ double dyfull(int m, int u) const {
    if (m == 0) {
      if (u == 0) return f(R_DY0_P);
      if (u == CT) return f(R_DY0_T);
      if (u == CSW) return f(R_DY0_SW);
      return 0.0;
    }
    if (m < 1 + NCO) {
      const int i = m - 1;
      if (u == 0) return f(R_DYO + 4 * i);
      if (u == CT) return f(R_DYO + 4 * i + 1);
      if (u == 1 + i) return f(R_DYO + 4 * i + 2);
      if (u == CSW || u == CSG) return f(R_DYO + 4 * i + 3);
      return 0.0;
    }
    return u == m ? 1.0 : 0.0;
  }
  __device__ __forceinline__ double dkt(int u) const {
    if (u == 0) return f(R_KT + 1);
    if (u == CT) return f(R_KT + 2);
    if (u == CSW) return f(R_KT + 3);
    if (u == CSG) return f(R_KT + 4);
    if (u == CCC) return f(R_KT + 5);
    return 0.0;
  }
};

// Column u of both derivative blocks of one connection (a = lower cell) for
// all rows, and (with_flux) the flux vector. Accumulation order per element
// follows conn_eval (_kernels.py:677-771): phases in order, the component
// row of each phase, then its energy term, conduction last.
__device__ __forceinline__ void face_cols(const int u, const ColView& A_, const ColView& B_,
                                          const double* __restrict__ st, int64_t n, int64_t a,
                                          int64_t b, double za, double zb, double gd, double td,
                                          int8_t* upw, int64_t upw_stride, int freeze,
                                          bool write_upw, bool with_flux, double* flux,
                                          double* dfa, double* dfb) {
#pragma unroll
  for (int r = 0; r < NU; ++r) { flux[r] = 0.0; dfa[r] = 0.0; dfb[r] = 0.0; }
#pragma unroll
  for (int al = 0; al < 3; ++al) {
    const double phi_a = A_.f(R_POT + al) - A_.f(R_GAM + al) * za;
    const double phi_b = B_.f(R_POT + al) - B_.f(R_GAM + al) * zb;
    const double dphi = phi_a - phi_b;
    bool up_a;
    if (freeze) {
      up_a = upw[al * upw_stride + a] == 1;
    } else {
      up_a = dphi >= 0.0;
      if (write_upw) upw[al * upw_stride + a] = up_a ? 1 : 0;
    }
    const ColView& U = up_a ? A_ : B_;
    const int64_t cu = up_a ? a : b;
    const double b_up = U.f(R_BETA + al);
    const double conv = gd * dphi;
    const double ga = A_.dpot(al, u) - za * A_.dgam(al, u);
    const double gb = B_.dpot(al, u) - zb * B_.dgam(al, u);
    const double dbu = U.dbeta(al, u);
    double* dtgt = up_a ? dfa : dfb;
    // component rows of this phase
    const int m0 = al == 0 ? 0 : (al == 1 ? 1 : 0);
    const int m1 = al == 0 ? 1 : (al == 1 ? 1 + NCO : NF);
#pragma unroll
    for (int row = 0; row < NF; ++row) {
      if (row < m0 || row >= m1) continue;
      double w_up;
      if (al == 0) w_up = 1.0;
      else if (al == 1) w_up = st[(int64_t)row * n + cu];
      else w_up = U.f(R_Y + row);
      const double val = b_up * w_up;
      if (with_flux) flux[row] += conv * val;
      if (val != 0.0) {
        dfa[row] += gd * val * ga;
        dfb[row] -= gd * val * gb;
      }
      double dv = dbu * w_up;
      if (al == 1 && u == row) dv += b_up;              // d(x_m)/d x_m
      else if (al == 2) dv += b_up * U.dyfull(row, u);
      if (dv != 0.0) dtgt[row] += conv * dv;
    }
    // energy row
    const double h_up = U.f(R_HPH + al);
    const double val = b_up * h_up;
    if (with_flux) flux[ROW_E] += conv * val;
    if (val != 0.0) {
      dfa[ROW_E] += gd * val * ga;
      dfb[ROW_E] -= gd * val * gb;
    }
    const double dv = dbu * h_up + b_up * U.dhph(al, u);
    if (dv != 0.0) dtgt[ROW_E] += conv * dv;
  }
  double hm, dh_a, dh_b;
  harmonic_pair(A_.f(R_KT), B_.f(R_KT), hm, dh_a, dh_b);
  if (hm > 0.0 || dh_a != 0.0 || dh_b != 0.0) {
    const double dt_ab = st[CT * n + a] - st[CT * n + b];
    if (with_flux) flux[ROW_E] += td * hm * dt_ab;
    if (u == CT) { dfa[ROW_E] += td * hm; dfb[ROW_E] -= td * hm; }
    if (dt_ab != 0.0) {
      dfa[ROW_E] += td * dt_ab * dh_a * A_.dkt(u);
      dfb[ROW_E] += td * dt_ab * dh_b * B_.dkt(u);
    }
  }
}

// diag -= bcol wrow^T / dwdb on the well cells; schur[w] = bcol (r_w / dwdb)
// (linsolve.py:378-386); one thread per well, wells in order.
__global__ void k_schur_pre(Dims g, int nw, const int64_t* __restrict__ wcell,
                            const double* __restrict__ wout, int wstride, double* diag,
                            double* schur) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t n = g.n;
  for (int w = 0; w < nw; ++w) {
    const int64_t c = wcell[w];
    const double* o = wout + (int64_t)w * wstride;
    const double resid_w = o[0], dwdb = o[1];
    const double* wrow = o + 2;
    const double* bcol = o + 2 + NU;
    const double inv_d = 1.0 / dwdb;
    for (int r = 0; r < NU; ++r) {
      schur[w * NU + r] = bcol[r] * (resid_w * inv_d);
      for (int u = 0; u < NU; ++u) diag[(int64_t)(r * NU + u) * n + c] -= bcol[r] * wrow[u] * inv_d;
    }
  }
}

constexpr int FD_CELLS = 8;   // cells per CTA; 64 column threads per cell

struct FusedSmem {
  double own[NDIR][NU][NU][FD_CELLS];   // signed own-derivative column u, row r
  double flux[NDIR][NU][FD_CELLS];      // signed face flux rows
  double colk[NU][FD_CELLS];
  double cmax[NU][FD_CELLS];
  int piv[FD_CELLS];
  int failc[FD_CELLS];
};

struct FusedArgs {
  FaceArgs F;                            // st, rec, depth, gd, td, upw, freeze, resid (out), diag (cell part, in)
  const double* __restrict__ resid_cell; // cell part + wells (in)
  double* rhs;                           // decoupled rhs (out)
  int nw;
  const int64_t* __restrict__ wcell;
  const double* __restrict__ schur;
  int* flags;
  unsigned long long* bad;
};

__global__ void __launch_bounds__(FD_CELLS * 64) k_face_dc(const FusedArgs P) {
  extern __shared__ __align__(16) unsigned char dsm[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(dsm);
  const FaceArgs& F = P.F;
  const int64_t n = F.g.n;
  const int cl = threadIdx.x % FD_CELLS, j = threadIdx.x / FD_CELLS;   // cell lane, column
  const int64_t c = (int64_t)blockIdx.x * FD_CELLS + cl;
  const bool live = c < n;
  int i = 0, jj = 0, k = 0;
  const int64_t cell = live ? locate(F.g, c, i, jj, k) : 0;
  double a[NU];   // this thread's column of the augmented block row
  // ---- phase 1: faces -> off-diagonal columns (+ own-derivative columns to smem)
  if (j >= NU && j < NU + NDIR * NU) {
    const int d = (j - NU) / NU, u = (j - NU) % NU;
    const int64_t nb = live ? nb_pos(F.g, cell, i, jj, k, d) : -1;
    double own[NU], fl[NU];
    if (nb >= 0) {
      const bool c_is_a = d >= DXP;
      const int64_t fa = c_is_a ? c : nb, fb = c_is_a ? nb : c;
      const int axis = c_is_a ? d - DXP : 2 - d;
      const ColView Av{F.rec, n, fa}, Bv{F.rec, n, fb};
      double dfa[NU], dfb[NU];
      face_cols(u, Av, Bv, F.st, n, fa, fb, F.depth[fa], F.depth[fb], F.gd[axis * n + fa],
                F.td[axis * n + fa], F.upw + (int64_t)axis * 3 * n, n, F.freeze,
                c_is_a && u == 0, u == 0, fl, dfa, dfb);
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        own[r] = c_is_a ? dfa[r] : -dfb[r];
        a[r] = c_is_a ? dfb[r] : -dfa[r];
        fl[r] = c_is_a ? fl[r] : -fl[r];
      }
    } else {
#pragma unroll
      for (int r = 0; r < NU; ++r) { own[r] = 0.0; a[r] = 0.0; fl[r] = 0.0; }
    }
#pragma unroll
    for (int r = 0; r < NU; ++r) S.own[d][u][r][cl] = own[r];
    if (u == 0) {
#pragma unroll
      for (int r = 0; r < NU; ++r) S.flux[d][r][cl] = fl[r];
    }
  }
  if (j == 0) S.failc[cl] = NU;
  __syncthreads();
  // ---- phase 2: diagonal columns and rhs in the reference's gather order
  if (j < NU) {
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      double v = live ? F.diag[(int64_t)(r * NU + j) * n + c] : (r == j ? 1.0 : 0.0);
#pragma unroll
      for (int d = 0; d < NDIR; ++d) v += S.own[d][j][r][cl];
      a[r] = v;
    }
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < NU; ++r) m = fmax(m, fabs(a[r]));
    S.cmax[j][cl] = m;
  } else if (j == NU + NDIR * NU) {
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      double res = live ? P.resid_cell[(int64_t)r * n + c] : 0.0;
#pragma unroll
      for (int d = 0; d < NDIR; ++d) res += S.flux[d][r][cl];
      if (live) F.resid[(int64_t)r * n + c] = res;
      a[r] = -res;
    }
    for (int w = 0; w < P.nw; ++w)
      if (live && P.wcell[w] == c) {
#pragma unroll
        for (int r = 0; r < NU; ++r) a[r] += P.schur[w * NU + r];
      }
  }
  __syncthreads();
  double amax = 0.0;
#pragma unroll
  for (int u = 0; u < NU; ++u) amax = fmax(amax, S.cmax[u][cl]);
  const double tol = 1e-13 * amax;
  // ---- phase 3: Gauss-Jordan with partial pivoting (linsolve.py:70-119)
#pragma unroll
  for (int kk = 0; kk < NU; ++kk) {
    if (j == kk) {
      int piv = kk;
      double pv = fabs(a[kk]);
#pragma unroll
      for (int r = kk + 1; r < NU; ++r) {
        const double v = fabs(a[r]);
        if (v > pv) { pv = v; piv = r; }
      }
      if (pv <= tol || amax == 0.0) atomicMin(&S.failc[cl], amax == 0.0 ? 0 : kk);
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double v = a[r];
        if (r == kk) {
#pragma unroll
          for (int q = kk + 1; q < NU; ++q) if (q == piv) v = a[q];
        } else if (r == piv) {
          v = a[kk];
        }
        S.colk[r][cl] = v;
      }
      S.piv[cl] = piv;
    }
    __syncthreads();
    const int piv = S.piv[cl];
    if (piv != kk) {
      const double t0 = a[kk];
#pragma unroll
      for (int q = kk + 1; q < NU; ++q)
        if (q == piv) { a[kk] = a[q]; a[q] = t0; }
    }
    const double dinv = 1.0 / S.colk[kk][cl];
    a[kk] *= dinv;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      if (r == kk) continue;
      const double f = S.colk[r][cl];
      if (f != 0.0) a[r] -= f * a[kk];
    }
    __syncthreads();
  }
  if (!live) return;
  if (j == 0 && S.failc[cl] < NU) {
    P.flags[cell] = S.failc[cl] + 1;
    atomicMin(P.bad, (unsigned long long)cell);
  }
  if (j >= NU && j < NU + NDIR * NU) {
    const int d = (j - NU) / NU, u = (j - NU) % NU;
#pragma unroll
    for (int r = 0; r < NU; ++r) F.offd[(int64_t)((d * NU + r) * NU + u) * n + c] = a[r];
  } else if (j == NU + NDIR * NU) {
#pragma unroll
    for (int r = 0; r < NU; ++r) P.rhs[(int64_t)r * n + c] = a[r];
  }
}

}  // namespace isc
