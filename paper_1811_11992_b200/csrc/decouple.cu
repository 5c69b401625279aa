// Well Schur fold + block Gauss-Jordan decoupling of every block row.
//
// Restates linsolve.py:362-394 (well elimination, single perforation) and
// linsolve.py:70-152 (GJ with partial pivoting, pivot tolerance
// 1e-13*max|D|, D^-1 applied to the row's rhs and off-diagonal blocks).
//
// Kernels: k_decouple_ws (default; warp-specialised, below) and k_decouple3
// (the same arithmetic one phase after the other, -DDECOUPLE_WS=0). Loads and
// stores of a warp are consecutive cells of one column -> coalesced. The
// decoupled diagonal (D^-1 D, identity up to rounding; the reference stores
// it, Appendix A.11) is not written: SpMV/ILU use an exact identity.
#include "common.cuh"

namespace isc {

// rhs = -resid, then fold each well's bhp unknown into its perforated cell.
__global__ void k_rhs_schur(Dims g, const double* __restrict__ resid, double* rhs, double* diag,
                            int nw, const int64_t* __restrict__ wcell,
                            const double* __restrict__ wout, int wstride) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (!owned_k(g, plane_of(g, c))) {   // ghost rows (z-slabs) carry no equation
#pragma unroll
    for (int r = 0; r < NU; ++r) rhs[r * n + c] = 0.0;
    return;
  }
#pragma unroll
  for (int r = 0; r < NU; ++r) rhs[r * n + c] = -resid[r * n + c];
  for (int w = 0; w < nw; ++w) {
    if (wcell[w] != c) continue;
    const double* o = wout + (int64_t)w * wstride;
    const double resid_w = o[0], dwdb = o[1];
    const double* wrow = o + 2;
    const double* bcol = o + 2 + NU;
    const double inv_d = 1.0 / dwdb;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      rhs[r * n + c] += bcol[r] * (resid_w * inv_d);
#pragma unroll
      for (int u = 0; u < NU; ++u) diag[(int64_t)(r * NU + u) * n + c] -= bcol[r] * wrow[u] * inv_d;
    }
  }
}

// k_decouple_ws: D^-1 first, then D^-1 x [B_-z .. B_+z | rhs] -- exactly
// the reference's order of operations (_gj_inverse on [D | I], then _mm/_mv
// with sequential k sums, linsolve.py:130-152) -- in a warp-specialised
// persistent pipeline. Per CTA, 9 "inverse" warps run Gauss-Jordan on [D | I] for groups
// of 32 cells (warp u owns column u of every cell in the group; one named
// barrier per pivot step, the pivot column double-buffered) and hand D^-1
// over in a double-buffered shared tile; 8 "product" warps stream the 55
// columns [B_-z .. B_+z | rhs] of the previous group through D^-1. The
// Gauss-Jordan latency (a dependent chain of 9 steps) hides behind the
// product warps' HBM stream instead of stalling it.
constexpr int WS_CELLS = 32;
constexpr int WS_GJ_WARPS = NU;          // 288 threads
#ifndef WS_B_WARPS
#define WS_B_WARPS 8
#endif
constexpr int WS_THREADS = 32 * (WS_GJ_WARPS + WS_B_WARPS);   // 544
#ifndef WS_BLOCKS_PER_SM
#define WS_BLOCKS_PER_SM 2
#endif
enum { WS_BAR_GJ = 1, WS_BAR_READY = 2, WS_BAR_FREE = 4 };   // READY/FREE + buffer

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

struct WsSmem {
  double inv[2][NU][NU][WS_CELLS];   // D^-1 (row, col, cell), double-buffered
  double colk[2][NU][WS_CELLS];      // pivot column of the current step
  double cmax[NU][WS_CELLS];
  int piv[2][WS_CELLS];
  int failc[WS_CELLS];
  unsigned char ghost[2][WS_CELLS];
};

__global__ void __launch_bounds__(WS_THREADS, WS_BLOCKS_PER_SM) k_decouple_ws(
    Dims g, const double* __restrict__ diag, double* offd, double* rhs, int* flags,
    unsigned long long* bad, int offd_rows) {
  extern __shared__ __align__(16) unsigned char ws_raw[];
  WsSmem& S = *reinterpret_cast<WsSmem*>(ws_raw);
  const int64_t n = g.n;
  // owned planes only (ghost rows carry no equation; the factor takes the
  // owner ranks' boundary blocks): positions [p0, p1)
  const int64_t p0 = (int64_t)g.kw_lo * g.nxny, p1 = (int64_t)g.kw_hi * g.nxny;
  const int64_t ngroups = (p1 - p0 + WS_CELLS - 1) / WS_CELLS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb_threads = 32 * (WS_GJ_WARPS + WS_B_WARPS);
  if (warp < WS_GJ_WARPS) {
    // ------------------------------------------------ inverse warps
    const int u = warp, cl = lane;
    int i = 0;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++i) {
      const int buf = i & 1;
      const int64_t c = p0 + grp * WS_CELLS + cl;
      const bool live = c < p1;
      double a[NU], e[NU];
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        a[r] = live ? diag[(int64_t)(r * NU + u) * n + c] : (r == u ? 1.0 : 0.0);
        e[r] = (r == u) ? 1.0 : 0.0;
      }
      double m = 0.0;
#pragma unroll
      for (int r = 0; r < NU; ++r) m = fmax(m, fabs(a[r]));
      S.cmax[u][cl] = m;
      if (u == 0) S.failc[cl] = NU;
      named_sync(WS_BAR_GJ, 32 * WS_GJ_WARPS);
      double amax = 0.0;
#pragma unroll
      for (int q = 0; q < NU; ++q) amax = fmax(amax, S.cmax[q][cl]);
      const double tol = 1e-13 * amax;
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int kb = k & 1;
        if (u == k) {
          int piv = k;
          double pv = fabs(a[k]);
#pragma unroll
          for (int r = k + 1; r < NU; ++r) {
            const double v = fabs(a[r]);
            if (v > pv) { pv = v; piv = r; }
          }
          if (pv <= tol || amax == 0.0) S.failc[cl] = min(S.failc[cl], amax == 0.0 ? 0 : k);
#pragma unroll
          for (int r = 0; r < NU; ++r) {
            double v = a[r];
            if (r == k) {
#pragma unroll
              for (int q = k + 1; q < NU; ++q) if (q == piv) v = a[q];
            } else if (r == piv) {
              v = a[k];
            }
            S.colk[kb][r][cl] = v;
          }
          S.piv[kb][cl] = piv;
        }
        named_sync(WS_BAR_GJ, 32 * WS_GJ_WARPS);
        const int piv = S.piv[kb][cl];
        if (piv != k) {
          const double t0 = a[k], t1 = e[k];
#pragma unroll
          for (int q = k + 1; q < NU; ++q)
            if (q == piv) { a[k] = a[q]; e[k] = e[q]; a[q] = t0; e[q] = t1; }
        }
        const double dinv = 1.0 / S.colk[kb][k][cl];
        a[k] *= dinv;
        e[k] *= dinv;
#pragma unroll
        for (int r = 0; r < NU; ++r) {
          if (r == k) continue;
          const double f = S.colk[kb][r][cl];
          if (f != 0.0) { a[r] -= f * a[k]; e[r] -= f * e[k]; }
        }
      }
      // hand the inverse over once the product warps released this buffer
      if (i >= 2) named_sync(WS_BAR_FREE + buf, nb_threads);
#pragma unroll
      for (int r = 0; r < NU; ++r) S.inv[buf][r][u][cl] = e[r];
      if (u == 0) {
        bool gh = false;
        if (live) {
          gh = !owned_k(g, plane_of(g, c));
          const int fc = S.failc[cl];
          if (!gh && fc < NU) {
            const int64_t cell = cell_of(g, c);
            flags[cell] = fc + 1;
            atomicMin(bad, (unsigned long long)cell);
          }
        }
        S.ghost[buf][cl] = gh ? 1 : 0;
      }
      named_arrive(WS_BAR_READY + buf, nb_threads);
    }
  } else {
    // ------------------------------------------------ product warps
    const int t = threadIdx.x - 32 * WS_GJ_WARPS;   // 0..32*WS_B_WARPS-1
    const int cl = t & 31, col0 = t >> 5;          // cell, first column
    constexpr int NCOLB = NDIR * NU + 1;           // 55
    int i = 0;
    const int64_t mine = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++i) {
      const int buf = i & 1;
      const int64_t c = p0 + grp * WS_CELLS + cl;
      named_sync(WS_BAR_READY + buf, nb_threads);
      if (c < p1) {
        const bool gh = S.ghost[buf][cl] != 0;
#pragma unroll 1
        for (int col = col0; col < NCOLB; col += WS_B_WARPS) {
          double* base;
          int64_t stride;
          int kin;
          if (col < NDIR * NU) {
            const int d = col / NU, uu = col % NU;
            base = offd + (int64_t)(d * NB + uu) * n + c;
            stride = (int64_t)NU * n;
            kin = offd_rows;
          } else {
            base = rhs + c;
            stride = n;
            kin = NU;
            if (gh) {   // ghost rows carry no equation
#pragma unroll
              for (int r = 0; r < NU; ++r) base[r * stride] = 0.0;
              continue;
            }
          }
          double v[NU];
#pragma unroll
          for (int r = 0; r < NU; ++r) v[r] = r < kin ? base[r * stride] : 0.0;
#pragma unroll
          for (int r = 0; r < NU; ++r) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < NU; ++k)
              if (k < kin) s += S.inv[buf][r][k][cl] * v[k];
            base[r * stride] = s;
          }
        }
      }
      if (i + 2 < mine) named_arrive(WS_BAR_FREE + buf, nb_threads);
    }
  }
}

}  // namespace isc
