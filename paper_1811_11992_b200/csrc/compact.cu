// Compact decoupled operator for the multicolour (mcilu) solve.
//
// The reference decouples every block row explicitly, B_d <- D^-1 B_d
// (linsolve.py:130-152), and the bjacobi/ras paths here do the same
// (k_decouple_ws). For the red-eliminated multicolour solve the decoupled
// blocks are only ever applied to vectors, and an assembled off-diagonal
// block has structurally zero rows ROW_OS..8 (constraint and coke rows carry
// no flux). So
//     (D^-1 B_d) x = D^-1[:, :CR] (B_d[:CR, :] x),   CR = ROW_OS = 6,
// and the operator is kept as the raw flux rows of B_d (54 values per
// direction) plus the first CR columns of D^-1 (54 values per cell, stored
// over the diagonal block). The decoupling (k_decouple_compact_t) no longer
// reads and rewrites the 7.8 GB of off-diagonal blocks at C4: it inverts the
// diagonal blocks (same Gauss-Jordan, pivot rule and failure reporting as
// k_decouple_ws) and decouples the rhs. The factorisation keeps the 6x6
// blocks B'_bd = B_bd[:CR, :] D_nb^-1[:, :CR] of the black cells, so the
// product S z_b of the Krylov iteration is
//     y_r = B_rb z_b (raw rows, k_cc_red),  v_b = z_b - D_b^-1[:, :CR] B'_br y
//     (k_cc_black)
// — 6x54 + 6x36 + 54 = 594 matrix values per red/black cell pair against
// 2 x 6 x 81 = 972 for the explicit blocks. The operator is the same matrix;
// only the rounding of its products differs from the explicit form (which the
// mcilu iterates never matched bit for bit anyway: a different
// preconditioner from the reference's RAS).
//
//   dinv[(q*CR + r)*n + p]          q < 9, r < CR        (over diag)
//   offd rows r < CR as assembled (undecoupled)
//   bp[((d*CR + q)*CR + s)*half + t] t-th black cell, B'_bd (ctx->cbp)
#include "common.cuh"

namespace isc {

constexpr int CR = ROW_OS;   // flux rows of an assembled off-diagonal block
// condensed form (below): primary / secondary unknowns of a cell
constexpr int NCS = NU - CR;   // secondary unknowns per cell (3)
__host__ __device__ constexpr int cprim(int p) {   // p-th primary unknown
  return p + (p >= NCO ? 1 : 0) + (p >= NCO + NCG - 1 ? 1 : 0);
}
__host__ __device__ constexpr int csec(int i) {    // i-th secondary unknown
  return i == 0 ? NCO : (i == 1 ? NCO + NCG : CCC);
}
static_assert(cprim(CR - 1) == CSG && csec(NCS - 1) == CCC, "condensed unknown split");

// cp.async (LDGSTS): global -> shared without register staging
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef DCT_THREADS
#define DCT_THREADS 128
#endif
#ifndef DCT_UNIFORM_SWAP
#define DCT_UNIFORM_SWAP 1
#endif
// opaque selects: a plain `q == piv ? x : y` chain over an unrolled register
// array is folded back into a dynamically indexed (local-memory) array
__device__ __forceinline__ double sel_d(bool p, double x, double y) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r) : "d"(x), "d"(y), "r"((unsigned)p));
  return r;
}
__device__ __forceinline__ int sel_i(bool p, int x, int y) {
  int r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
      : "=r"(r) : "r"(x), "r"(y), "r"((unsigned)p));
  return r;
}
// E_S of the cell at storage position c from its diagonal block's local rows
// (Gauss-Jordan with partial pivoting on [D[CR:, S] | D[CR:, P]]); false when
// a pivot is below 1e-12 of max|D[CR:, S]| or not finite (the form is then
// not used for this system).
template <class L>
__device__ __forceinline__ bool cond_es_from(L ld, double (&es)[NCS][CR]) {
  double m[NCS][NCS + CR];
  double mmax = 0.0;
#pragma unroll
  for (int i = 0; i < NCS; ++i) {
#pragma unroll
    for (int j = 0; j < NCS; ++j) {
      m[i][j] = ld(CR + i, csec(j));
      mmax = fmax(mmax, fabs(m[i][j]));
    }
#pragma unroll
    for (int p = 0; p < CR; ++p) m[i][NCS + p] = ld(CR + i, cprim(p));
  }
  bool ok = mmax > 0.0 && mmax < INFINITY;
#pragma unroll
  for (int k = 0; k < NCS; ++k) {
    int piv = k;
    double pv = fabs(m[k][k]);
#pragma unroll
    for (int r = k + 1; r < NCS; ++r)
      if (fabs(m[r][k]) > pv) { pv = fabs(m[r][k]); piv = r; }
    ok = ok && pv > 1e-12 * mmax;
#pragma unroll
    for (int r = k + 1; r < NCS; ++r) {
      if (r != piv) continue;
#pragma unroll
      for (int j = 0; j < NCS + CR; ++j) {
        const double t = m[k][j];
        m[k][j] = m[r][j];
        m[r][j] = t;
      }
    }
    const double dv = 1.0 / m[k][k];
#pragma unroll
    for (int j = 0; j < NCS + CR; ++j) m[k][j] *= dv;
#pragma unroll
    for (int r = 0; r < NCS; ++r) {
      if (r == k) continue;
      const double f = m[r][k];
#pragma unroll
      for (int j = 0; j < NCS + CR; ++j) m[r][j] -= f * m[k][j];
    }
  }
#pragma unroll
  for (int i = 0; i < NCS; ++i)
#pragma unroll
    for (int p = 0; p < CR; ++p) {
      es[i][p] = -m[i][NCS + p];
      ok = ok && isfinite(es[i][p]);
    }
  return ok;
}
__device__ __forceinline__ bool cond_es(const double* __restrict__ diag, int64_t n, int64_t c,
                                        double (&es)[NCS][CR]) {
  return cond_es_from([&](int r, int u) { return diag[(int64_t)(r * NU + u) * n + c]; }, es);
}

// D^-1 of every owned cell and rhs <- D^-1 rhs, one thread per cell with the
// block held in registers: in-place Gauss-Jordan (once column k is
// eliminated its slot holds column perm[k] of the inverse, where perm tracks
// the row interchanges) with the reference's pivot rule (partial pivoting,
// failure below 1e-13 max|D|, _gj_inverse linsolve.py:70-119), scaling by the
// reciprocal and elimination order; no shared memory and no barriers.
// The well Schur fold (linsolve.py:362-394; k_rhs_schur for the other forms)
// is applied on the way in: rhs = -resid, and a perforated cell's block and
// rhs take the well's bhp column (the local rows' slots are written back:
// the condensed form reads them).
__global__ void __launch_bounds__(DCT_THREADS) k_decouple_compact_t(
    Dims g, double* diag, double* rhs, int* flags, unsigned long long* bad,
    const double* __restrict__ resid, int nw, const int64_t* __restrict__ wcell,
    const double* __restrict__ wout, int wstride, double* __restrict__ es, int* cfail) {
  const int64_t n = g.n;
  const int64_t p0 = (int64_t)g.kw_lo * g.nxny, p1 = (int64_t)g.kw_hi * g.nxny;
  const int64_t c = p0 + (int64_t)blockIdx.x * DCT_THREADS + threadIdx.x;
  if (c >= p1) return;
  double a[NU][NU];   // a[r][j]: row r, slot j
#pragma unroll
  for (int r = 0; r < NU; ++r)
#pragma unroll
    for (int j = 0; j < NU; ++j) a[r][j] = diag[(int64_t)(r * NU + j) * n + c];
  {
    double rv[NU];
#pragma unroll
    for (int r = 0; r < NU; ++r) rv[r] = -resid[(int64_t)r * n + c];
    for (int w = 0; w < nw; ++w) {
      if (wcell[w] != c) continue;
      const double* o = wout + (int64_t)w * wstride;
      const double resid_w = o[0], dwdb = o[1];
      const double* wrow = o + 2;
      const double* bcol = o + 2 + NU;
      const double inv_d = 1.0 / dwdb;
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        rv[r] += bcol[r] * (resid_w * inv_d);
#pragma unroll
        for (int u = 0; u < NU; ++u) a[r][u] -= bcol[r] * wrow[u] * inv_d;
      }
#pragma unroll
      for (int r = CR; r < NU; ++r)
#pragma unroll
        for (int u = 0; u < NU; ++u) diag[(int64_t)(r * NU + u) * n + c] = a[r][u];
    }
#pragma unroll
    for (int r = 0; r < NU; ++r) rhs[(int64_t)r * n + c] = rv[r];
  }
  if (es) {   // condensed form: E_S of a black cell (warp-uniform colour)
    const int64_t rem = c - (int64_t)plane_of(g, c) * g.nxny;
    if (rem >= g.ph) {
      double e[NCS][CR];
      if (!cond_es_from([&](int r, int u) { return a[r][u]; }, e)) atomicOr(cfail, 1);
      const int64_t tb = c - g.ph * (int64_t)(plane_of(g, c) + 1);
#pragma unroll
      for (int i = 0; i < NCS; ++i)
#pragma unroll
        for (int p = 0; p < CR; ++p) es[(int64_t)(i * CR + p) * g.half + tb] = e[i][p];
    }
  }
  double amax = 0.0;
#pragma unroll
  for (int r = 0; r < NU; ++r)
#pragma unroll
    for (int j = 0; j < NU; ++j) amax = fmax(amax, fabs(a[r][j]));
  const double tol = 1e-13 * amax;
  int perm[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) perm[r] = r;
  int failc = NU;
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    int piv = k;
    double pv = fabs(a[k][k]);
#pragma unroll
    for (int r = k + 1; r < NU; ++r) {
      const double v = fabs(a[r][k]);
      if (v > pv) { pv = v; piv = r; }
    }
    if (pv <= tol || amax == 0.0) failc = amax == 0.0 ? 0 : min(failc, k);
#if DCT_UNIFORM_SWAP
    // No interchange anywhere in the warp (about every other step on the C4
    // blocks): the select chain over the candidate rows is skipped -- a
    // warp-uniform branch around it, the values are untouched either way.
    // (A vote per candidate row, or a plain register swap of the row a
    // uniform warp picked, makes the compiler move the block to local memory.)
    if (!__all_sync(__activemask(), piv == k))
#endif
    {
#pragma unroll
      for (int q = k + 1; q < NU; ++q) {
        const bool sw = q == piv;
#pragma unroll
        for (int j = 0; j < NU; ++j) {
          const double t = a[k][j];
          a[k][j] = sel_d(sw, a[q][j], t);
          a[q][j] = sel_d(sw, t, a[q][j]);
        }
        const int t = perm[k];
        perm[k] = sel_i(sw, perm[q], t);
        perm[q] = sel_i(sw, t, perm[q]);
      }
    }
    const double dv = 1.0 / a[k][k];
    // row k: the pivot slot becomes column perm[k] of the inverse (1 * dv)
#pragma unroll
    for (int j = 0; j < NU; ++j) a[k][j] = (j == k ? 1.0 : a[k][j]) * dv;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      if (r == k) continue;
      const double f = a[r][k];
      if (f != 0.0) {
#pragma unroll
        for (int j = 0; j < NU; ++j) a[r][j] = (j == k ? 0.0 : a[r][j]) - f * a[k][j];
      }
    }
  }
  const bool gh = !owned_k(g, plane_of(g, c));
  if (!gh && failc < NU) {
    const int64_t cell = cell_of(g, c);
    flags[cell] = failc + 1;
    atomicMin(bad, (unsigned long long)cell);
  }
  // D^-1[:, :CR] over the diagonal block: slot j is inverse column perm[j]
#pragma unroll
  for (int j = 0; j < NU; ++j) {
    const int col = perm[j];
    if (col < CR) {
#pragma unroll
      for (int r = 0; r < NU; ++r) diag[(int64_t)(r * CR + col) * n + c] = a[r][j];
    }
  }
  // rhs row u: sequential k sum as the reference's _mv. The inverse's
  // columns are un-permuted through this thread's shared-memory slot (a
  // dynamically indexed store; selecting slot iperm[k] for each (u, k) from
  // registers took 648 double selects)
  extern __shared__ double dct_inv[];   // [NB][DCT_THREADS]
  double* mine = dct_inv + threadIdx.x;
#pragma unroll
  for (int j = 0; j < NU; ++j) {
    const int col = perm[j];
#pragma unroll
    for (int u = 0; u < NU; ++u) mine[(u * NU + col) * DCT_THREADS] = a[u][j];
  }
  double rv[NU];
#pragma unroll
  for (int k = 0; k < NU; ++k) rv[k] = rhs[(int64_t)k * n + c];
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NU; ++k) s += mine[(u * NU + k) * DCT_THREADS] * rv[k];
    rhs[(int64_t)u * n + c] = gh ? 0.0 : s;
  }
}
constexpr int DCT_SMEM = NB * DCT_THREADS * 8;

// z-slabs: the ghost planes' rows of v carry no equation (zero), planes
// [0, kw_lo) and [kw_hi, nz)
__global__ void k_zero_ghost_rows(Dims g, int rows, double* v) {
  const int64_t lo = (int64_t)g.kw_lo * g.nxny, hi = (int64_t)(g.nz - g.kw_hi) * g.nxny;
  const int64_t m = lo + hi;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / m);
    const int64_t q = t - (int64_t)r * m;
    const int64_t c = q < lo ? q : (int64_t)g.kw_hi * g.nxny + (q - lo);
    v[(int64_t)r * g.n + c] = 0.0;
  }
}

// One half pass of the compact operator over the owned cells of one colour
// (thread (cell lane, flux row r < CR), then output rows q = y, y + CR):
//   out_q = base_q + SIGN * sum_r dinv[q][r] * (sum_d B_d[r, :] src(nb))
// red pass   (COL 0, SIGN -1, no base):  z_r = -B_rb z_b
// black pass (COL 1, SIGN +1, base z):   v_b = z_b + B_br z_r  (+ dots, K)
// rhs        (COL 1, SIGN -1, base b):   g_b = b_b - B_br b_r  (out, out2)
// x_red      (COL 0, SIGN -1, base b):   x_r = b_r - B_rb x_b
// full SpMV  (both colours, SIGN +1, base x): y = x + sum_d (D^-1 B_d) x
// K = 1: per-warp partials of out . w0; K = 2: out . out and out . w1,
// stored partial[k*stride + slot*CR + y].
#ifndef CP_MINB
#define CP_MINB 4
#endif
template <int COL, int SIGN, bool BASE, int K>
__device__ __forceinline__ void cpass(
    const Dims& g, const double* __restrict__ offd, const double* __restrict__ dinv,
    const double* __restrict__ src, const double* __restrict__ base, double* __restrict__ out,
    double* __restrict__ out2, const double* __restrict__ w0, const double* __restrict__ w1,
    double* partial, int stride, int slot0) {
  __shared__ double ts[CR][32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  const bool live = t < g.tw_hi;
  int64_t c = 0;
  int k = 0;
  double acc[K > 0 ? K : 1];
#pragma unroll
  for (int q = 0; q < (K > 0 ? K : 1); ++q) acc[q] = 0.0;
  if (live) {
    c = colour_pos(g, COL, t);
    int i, j;
    const int64_t cell = locate(g, c, i, j, k);
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
      double tt = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) tt += blk[(int64_t)u * n] * src[(int64_t)u * n + nb];
      s += tt;
    }
    ts[r][ls] = s;
  }
  __syncthreads();
  if (live) {
    const bool own = owned_k(g, k);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = r + h * CR;
      if (q >= NU) break;
      double wd = 0.0;
      if (K == 1) wd = w0[(int64_t)q * n + c];
      if (K == 2) wd = w1[(int64_t)q * n + c];
      double m = 0.0;
#pragma unroll
      for (int rr = 0; rr < CR; ++rr) m += dinv[(int64_t)(q * CR + rr) * n + c] * ts[rr][ls];
      const double v = BASE ? (SIGN > 0 ? base[(int64_t)q * n + c] + m : base[(int64_t)q * n + c] - m)
                            : (SIGN > 0 ? m : -m);
      out[(int64_t)q * n + c] = v;
      if (out2) out2[(int64_t)q * n + c] = v;
      if (own) {
        if (K == 1) acc[0] += v * wd;
        if (K == 2) { acc[0] += v * v; acc[K - 1] += v * wd; }
      }
    }
  }
  if (K > 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double x = acc[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (ls == 0)
        partial[(int64_t)q * stride * CR + (int64_t)(slot0 + blockIdx.x) * CR + r] = x;
    }
  }
}

// the passes as separately named kernels (profiles, ncu -k)
#define CP_ARGS                                                                              \
  Dims g, const double* __restrict__ offd, const double* __restrict__ dinv,                 \
      const double* __restrict__ src, const double* __restrict__ base, double* __restrict__ out, \
      double* __restrict__ out2, const double* __restrict__ w0, const double* __restrict__ w1,   \
      double *partial, int stride, int slot0
#define CP_PASS offd, dinv, src, base, out, out2, w0, w1, partial, stride, slot0
__global__ void __launch_bounds__(32 * CR, CP_MINB) k_cc_rhs(CP_ARGS) {
  cpass<1, -1, true, 0>(g, CP_PASS);
}
__global__ void __launch_bounds__(32 * CR, CP_MINB) k_cc_xred(CP_ARGS) {
  cpass<0, -1, true, 0>(g, CP_PASS);
}
template <int COL>
__global__ void __launch_bounds__(32 * CR, CP_MINB) k_cc_spmv(CP_ARGS) {
  cpass<COL, 1, true, 0>(g, CP_PASS);
}

// The product S z_b of the Krylov iteration, in two half passes that need
// no D^-1 on the red side:
//   red pass   y_r = sum_d B_rd[:CR, :] z_b(nb)                 (CR rows)
//   black pass v_b = z_b - D_b^-1[:, :CR] sum_d B'_bd y(nb),
//              B'_bd = B_bd[:CR, :] D_nb^-1[:, :CR]   (CR x CR, from the factorisation)
// since (D_b^-1 B_bd)(D_r^-1 B_rd') = D_b^-1[:, :CR] B'_bd B_rd'[:CR, :].
// Per product 6x54 + 6x36 + 54 matrix values per cell pair instead of
// 2 x (6x54 + 54). y lives in rows 0..CR-1 of z's red positions.
#ifndef CC_MINB
#define CC_MINB 6   // C4 sweep 3..6: 0.402/0.420 -> 0.396/0.407 ms (red/black) at 6
#endif
// ccnz: 0 while every component row (< ROW_E) of the blocks has a zero coke
// column (the face evaluation clears it per assembly and sets it on a
// nonzero; imports and other writers set it) -- those 5 of the 54 row values
// are then not loaded (adding their zero products changes no bit for a
// finite z; a non-finite coke entry of z would make the full product NaN
// (0 * inf) where the skip leaves the row finite -- the Krylov vectors'
// norms, summed over all components, still turn non-finite in that case, so
// BiCGSTAB's breakdown / tolerance tests see it one dot product later).
__global__ void __launch_bounds__(32 * CR, CC_MINB) k_cc_red(Dims g, const double* __restrict__ offd,
                                                             const int* __restrict__ ccnz,
                                                             double* __restrict__ z,
                                                             const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  if (t >= g.tw_hi) return;
  const bool skip_cc = r < ROW_E && *ccnz == 0;   // warp-uniform (one row per warp)
  const int64_t c = colour_pos(g, 0, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (u == CCC && skip_cc) continue;
      tt += blk[(int64_t)u * n] * z[(int64_t)u * n + nb];
    }
    s += tt;
  }
  z[(int64_t)r * n + c] = s;
}

// K = 1: per-warp partials of v . w0; K = 2: v . v and v . w1
// (partial[k*stride*CR + slot*CR + y])
template <int K>
__global__ void __launch_bounds__(32 * CR, CC_MINB) k_cc_black(
    Dims g, const double* __restrict__ bp, const double* __restrict__ dinv,
    const double* __restrict__ z, double* __restrict__ v, const double* __restrict__ w0,
    const double* __restrict__ w1, double* partial, int stride, int slot0, const double* stop) {
  if (stopped(stop)) return;   // block-uniform: before the barrier
  __shared__ double ts[CR][32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  const bool live = t < g.tw_hi;
  int64_t c = 0;
  int k = 0;
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  if (live) {
    c = colour_pos(g, 1, t);
    int i, j;
    const int64_t cell = locate(g, c, i, j, k);
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = bp + (int64_t)((d * CR + r) * CR) * g.half + t;
      double tt = 0.0;
#pragma unroll
      for (int e = 0; e < CR; ++e) tt += blk[(int64_t)e * g.half] * z[(int64_t)e * n + nb];
      s += tt;
    }
    ts[r][ls] = s;
  }
  __syncthreads();
  if (live) {
    const bool own = owned_k(g, k);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = r + h * CR;
      if (q >= NU) break;
      const double wd = K == 1 ? w0[(int64_t)q * n + c] : w1[(int64_t)q * n + c];
      double m = 0.0;
#pragma unroll
      for (int rr = 0; rr < CR; ++rr) m += dinv[(int64_t)(q * CR + rr) * n + c] * ts[rr][ls];
      const double val = z[(int64_t)q * n + c] - m;
      v[(int64_t)q * n + c] = val;
      if (own) {
        if (K == 1) acc[0] += val * wd;
        if (K == 2) { acc[0] += val * val; acc[K - 1] += val * wd; }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double x = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (ls == 0) partial[(int64_t)q * stride * CR + (int64_t)(slot0 + blockIdx.x) * CR + r] = x;
  }
}

// U_b = I - D_b^-1 sum_d B_bd D_nb^-1 B_nb,back (the multicolour ILU(0)
// pivot block, k_mc_factor's product with the decoupled blocks formed on the
// fly), then its Gauss-Jordan inverse; B'_bd = B_bd[:CR, :] D_nb^-1[:, :CR]
// is kept for the black passes (bp[((d*CR + q)*CR + s)*half + t]). With
// g1 != nullptr the reduced rhs g_b = b_b - D_b^-1[:, :CR] sum_d B_bd b_r(nb)
// is formed on the way (the blocks are in shared memory anyway) and written
// to g1 and g2. Thread (black cell lane, column u).
#ifndef MCFC_CELLS
#define MCFC_CELLS 32   // black cells per CTA (thread (cell lane, column u): 288 threads)
#endif
#ifndef MCFC_MINB
#define MCFC_MINB 2     // two CTAs per SM: the double-buffered stages take ~99 KB of smem each (16 cells at 3 or 4 per SM: no faster)
#endif
// The products use fused multiply-adds (fma(); the translation unit is
// compiled --fmad=false for the assembly's reference operation order, which
// this preconditioner -- no reference counterpart -- does not need).
// Direction tiles are double-buffered with cp.async (LDGSTS: global -> shared
// without register staging): the loads of direction d+1 -- B_bd rows, the red
// neighbour's D^-1[:, :CR] and back block rows, its b -- are in flight while
// direction d is multiplied, so the six directions' HBM round trips overlap
// the products instead of alternating with them (round 1: one exposed round
// trip per tile and 2.8 TB/s).
struct McfcStage {
  double b[CR][NU][MCFC_CELLS];      // B_bd flux rows of the black cell
  double d[NU][CR][MCFC_CELLS];      // D_nb^-1[:, :CR] of the red neighbour
  double o[CR][NU][MCFC_CELLS];      // B_nb,back flux rows (the red neighbour's block pointing back)
  double r[NU][MCFC_CELLS];          // b(nb): the red neighbour's decoupled rhs
};
struct McfcSmem {
  McfcStage st[2];
  double bpsh[CR][CR][MCFC_CELLS];   // B'_bd = B_bd[:CR, :] D_nb^-1[:, :CR]
  double colk[NU][MCFC_CELLS];
  int pivs[MCFC_CELLS];
};

// COND: the condensed form (see "condensed form" below): U6 = I - Dc_b^-1
// sum_d B'_bd Bc_nb,back = I - Dc_b^-1 Q E_b (Q = sum_d B'_bd B_nb,back[:CR, :]
// as above, E_b from es), its 6 x 6 inverse in uinv; g_b (9 rows) to g1
// only. (The Bc blocks themselves are formed by k_cc_red_bc.)
template <bool COND>
__global__ void __launch_bounds__(MCFC_CELLS * NU, MCFC_MINB) k_mc_factor_compact(
    Dims g, const double* __restrict__ offd, const double* __restrict__ dinv,
    double* __restrict__ uinv, double* __restrict__ bp, int* fail, const double* __restrict__ b,
    double* __restrict__ g1, double* __restrict__ g2, const double* __restrict__ es) {
  constexpr int NC = COND ? CR : NU;   // order of the pivot block
  extern __shared__ __align__(16) unsigned char mcfc_raw[];
  McfcSmem& S = *reinterpret_cast<McfcSmem*>(mcfc_raw);
  auto& bpsh = S.bpsh;
  auto& colk = S.colk;
  auto& pivs = S.pivs;
  const int64_t n = g.n;
  const int ls = threadIdx.x, u = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * MCFC_CELLS + ls;
  const bool in = t < g.tw_hi;
  const int64_t c = in ? colour_pos(g, 1, t) : 0;
  int i = 0, j = 0, k = 0;
  const int64_t cell = in ? locate(g, c, i, j, k) : 0;
  const bool live = in && owned_k(g, k);
  int64_t nbs[NDIR];
#pragma unroll
  for (int d = 0; d < NDIR; ++d) nbs[d] = live ? nb_pos(g, cell, i, j, k, d) : -1;
  auto nb_of = [&](int d) -> int64_t { return nbs[d]; };
  // issue direction d's tiles into stage s (6 + 6 + 6 B_bd / D^-1 / back
  // values per thread, b(nb)[u] by every thread)
  auto issue = [&](int d, int sidx) {
    const int64_t nb = nb_of(d);
    if (nb < 0) return;
    McfcStage& T = S.st[sidx];
#pragma unroll
    for (int e = 0; e < CR; ++e) {
      const int idx = u * CR + e;   // 0..53
      const int br = idx / NU, bu = idx % NU;
      cp_async8(&T.b[br][bu][ls], offd + (int64_t)((d * NU + br) * NU + bu) * n + c);
      const int dq = idx / CR, dr = idx % CR;
      cp_async8(&T.d[dq][dr][ls], dinv + (int64_t)(dq * CR + dr) * n + nb);
      cp_async8(&T.o[e][u][ls], offd + (int64_t)((opposite(d) * NU + e) * NU + u) * n + nb);
    }
    if (g1) cp_async8(&T.r[u][ls], b + (int64_t)u * n + nb);
  };
  // Register-blocked products (the smem pipe bounds this kernel): thread
  // u = 3 tq + tc owns the 2x2 block B'[2tq.., 2tc..] and the 2x3 block
  // Q[2tq.., 3tc..]; each entry is summed in the same order as a plain loop
  double grow[2] = {0.0, 0.0};   // (sum_d B_bd b_r(nb))[2tq + qq], by the tc == 0 threads
  constexpr int QW = 3;
  double qacc[2][QW];            // Q[2tq + qq][3 tc + uu] = sum_d B'_bd B_back[:CR, :]
#pragma unroll
  for (int qq = 0; qq < 2; ++qq)
#pragma unroll
    for (int uu = 0; uu < QW; ++uu) qacc[qq][uu] = 0.0;
  const int tq = u / 3, tc = u - 3 * (u / 3);
  issue(0, 0);
  cp_async_commit();
#pragma unroll 1
  for (int d = 0; d < NDIR; ++d) {
    if (d + 1 < NDIR) issue(d + 1, (d + 1) & 1);
    cp_async_commit();   // (possibly empty group: keeps the wait count uniform)
    cp_async_wait<1>();
    __syncthreads();
    const McfcStage& T = S.st[d & 1];
    const int64_t nb = nb_of(d);
    if (nb >= 0) {
      double brow[2][NU];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int a = 0; a < NU; ++a) brow[qq][a] = T.b[2 * tq + qq][a][ls];
      if (g1 && tc == 0) {
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          double sr = 0.0;
#pragma unroll
          for (int a = 0; a < NU; ++a) sr = fma(brow[qq][a], T.r[a][ls], sr);
          grow[qq] += sr;
        }
      }
      // B'_bd = B_bd[:CR, :] D_nb^-1[:, :CR]; kept for the black passes
#pragma unroll
      for (int ss = 0; ss < 2; ++ss) {
        double dcol[NU];
#pragma unroll
        for (int a = 0; a < NU; ++a) dcol[a] = T.d[a][2 * tc + ss][ls];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          double sb = 0.0;
#pragma unroll
          for (int a = 0; a < NU; ++a) sb = fma(brow[qq][a], dcol[a], sb);
          const int q = 2 * tq + qq, s2 = 2 * tc + ss;
          bpsh[q][s2][ls] = sb;
          bp[(int64_t)((d * CR + q) * CR + s2) * g.half + t] = sb;
        }
      }
    }
    __syncthreads();
    if (nb >= 0) {   // Q[2tq.., 3tc..] += B'_bd[2tq.., :] B_back[:CR, 3tc..]
      double bpr[2][CR];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int r = 0; r < CR; ++r) bpr[qq][r] = bpsh[2 * tq + qq][r][ls];
#pragma unroll
      for (int uu = 0; uu < QW; ++uu) {
        double ocol[CR];
#pragma unroll
        for (int r = 0; r < CR; ++r) ocol[r] = T.o[r][3 * tc + uu][ls];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          double sq = 0.0;
#pragma unroll
          for (int r = 0; r < CR; ++r) sq = fma(bpr[qq][r], ocol[r], sq);
          qacc[qq][uu] += sq;
        }
      }
    }
    __syncthreads();   // stage d & 1 is refilled by the next iteration's issue
  }
  // Q and grow back to the column-per-thread layout of the Gauss-Jordan:
  // qcol[q] = Q[q][u]
  double qcol[CR];
  {
    double (*qsh)[NU][MCFC_CELLS] = reinterpret_cast<double (*)[NU][MCFC_CELLS]>(&S.st[1].o[0][0][0]);
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
#pragma unroll
      for (int uu = 0; uu < QW; ++uu) qsh[2 * tq + qq][QW * tc + uu][ls] = qacc[qq][uu];
    if (tc == 0) {
      colk[2 * tq][ls] = grow[0];
      colk[2 * tq + 1][ls] = grow[1];
    }
    __syncthreads();
    if (!COND) {
#pragma unroll
      for (int q = 0; q < CR; ++q) qcol[q] = qsh[q][u][ls];
    } else {   // column u < 6 of Q E_b = Q[:, P[u]] + sum_i Q[:, S[i]] E_b[i][u]
      double e[NCS];
#pragma unroll
      for (int ii = 0; ii < NCS; ++ii)
        e[ii] = live && u < CR ? es[(int64_t)(ii * CR + u) * g.half + t] : 0.0;
      const int pu = u < CR ? u + (u >= NCO ? 1 : 0) + (u >= NCO + NCG - 1 ? 1 : 0) : 0;
#pragma unroll
      for (int q = 0; q < CR; ++q) {
        double v = qsh[q][pu][ls];
#pragma unroll
        for (int ii = 0; ii < NCS; ++ii) v = fma(qsh[q][csec(ii)][ls], e[ii], v);
        qcol[q] = v;
      }
    }
  }
  cp_async_wait<0>();
  auto& dsh = S.st[0].d;
  // U[:, u] = e_u - D_b^-1[:, :CR] Q[:, u]  (condensed: rows P of D_b^-1)
  if (in) {
#pragma unroll
    for (int e = 0; e < CR; ++e) {
      const int idx = u * CR + e;
      dsh[idx / CR][idx % CR][ls] = dinv[(int64_t)idx * n + c];
    }
  }
  __syncthreads();
  if (g1 && live) {
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < CR; ++r) m = fma(dsh[u][r][ls], colk[r][ls], m);
    const double gv = b[(int64_t)u * n + c] - m;
    g1[(int64_t)u * n + c] = gv;
    if (g2) g2[(int64_t)u * n + c] = gv;
  }
  double ucol[NC], icol[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int pq = COND ? q + (q >= NCO ? 1 : 0) + (q >= NCO + NCG - 1 ? 1 : 0) : q;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < CR; ++r) s = fma(dsh[pq][r][ls], qcol[r], s);
    ucol[q] = (q == u ? 1.0 : 0.0) - s;
    icol[q] = (q == u) ? 1.0 : 0.0;
  }
  {
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < NC; ++r) m = fmax(m, fabs(ucol[r]));
    S.st[1].b[0][u][ls] = m;
  }
  __syncthreads();
  double amax = 0.0;
#pragma unroll
  for (int q = 0; q < NC; ++q) amax = fmax(amax, S.st[1].b[0][q][ls]);
  const double tol = 1e-13 * amax;
  __syncthreads();
#pragma unroll
  for (int kk = 0; kk < NC; ++kk) {
    if (u == kk) {
      int piv = kk;
      double pv = fabs(ucol[kk]);
#pragma unroll
      for (int r = kk + 1; r < NC; ++r) {
        const double v = fabs(ucol[r]);
        if (v > pv) { pv = v; piv = r; }
      }
      if (live && (pv <= tol || amax == 0.0)) atomicMin(fail, 1);
#pragma unroll
      for (int r = 0; r < NC; ++r) {
        double v = ucol[r];
        if (r == kk) {
#pragma unroll
          for (int q = kk + 1; q < NC; ++q) if (q == piv) v = ucol[q];
        } else if (r == piv) {
          v = ucol[kk];
        }
        colk[r][ls] = v;
      }
      pivs[ls] = piv;
    }
    __syncthreads();
    const int piv = pivs[ls];
    if (piv != kk) {
      const double t0 = ucol[kk], t1 = icol[kk];
#pragma unroll
      for (int q = kk + 1; q < NC; ++q)
        if (q == piv) { ucol[kk] = ucol[q]; icol[kk] = icol[q]; ucol[q] = t0; icol[q] = t1; }
    }
    const double dv = 1.0 / colk[kk][ls];
    ucol[kk] *= dv;
    icol[kk] *= dv;
#pragma unroll
    for (int r = 0; r < NC; ++r) {
      if (r == kk) continue;
      const double f = colk[r][ls];
      if (f != 0.0) { ucol[r] = fma(-f, ucol[kk], ucol[r]); icol[r] = fma(-f, icol[kk], icol[r]); }
    }
    __syncthreads();
  }
  if (live && u < NC) {
#pragma unroll
    for (int r = 0; r < NC; ++r) uinv[(int64_t)(r * NC + u) * n + c] = icol[r];
  }
}

// The condensed factorisation with one thread per black cell and everything
// in registers (no shared memory, no barriers): Q (6 x 9), the direction's
// B' (6 x 6) and the streamed rows / columns of the tiles. Per direction the
// thread streams column a of B_bd[:CR, :] with row a of the red neighbour's
// D^-1[:, :CR] (36 fused multiply-adds per 12 loads), then column u of the
// back block (36 per 6 loads); the sums run in the cooperative kernel's
// order (each B' and per-direction Q entry a chain over the inner index from
// zero), so the two kernels give the same values. Then U6 = I - Dc_b^-1 Q E_b
// and its Gauss-Jordan inverse on [U6 | I] (row interchanges by opaque
// selects, as k_decouple_compact_t).
#ifndef MCFT_THREADS
#define MCFT_THREADS 64
#endif
#ifndef MCFT_MINB
#define MCFT_MINB 4   // C4 sweep 3..8 (64 threads): 3-4 best (222 registers, no spills)
#endif
#ifndef MCFT_UA
#define MCFT_UA 9   // unroll of the streamed loops = loads in flight per thread (C4: 9/3 best; 9/9 spills)
#endif
#ifndef MCFT_UU
#define MCFT_UU 3
#endif
constexpr int kMcftUA = MCFT_UA, kMcftUU = MCFT_UU;
#ifndef MCFT_QSMEM
#define MCFT_QSMEM 1   // Q in shared memory (one slot per thread): registers for more resident warps
#endif
__global__ void __launch_bounds__(MCFT_THREADS, MCFT_MINB) k_mc_factor_cond_t(
    Dims g, const double* __restrict__ offd, const double* __restrict__ dinv,
    double* __restrict__ uinv, double* __restrict__ bp, int* fail, const double* __restrict__ b,
    double* __restrict__ g1, const double* __restrict__ es) {
  const int64_t n = g.n;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * MCFT_THREADS + threadIdx.x;
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 1, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  if (!owned_k(g, k)) return;
#if MCFT_QSMEM
  __shared__ double Qs[CR * NU][MCFT_THREADS];
#define QREF(q, u) Qs[(q) * NU + (u)][threadIdx.x]
#else
  double Qr[CR][NU];
#define QREF(q, u) Qr[q][u]
#endif
  double grow[CR];
#pragma unroll
  for (int q = 0; q < CR; ++q) {
    grow[q] = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) QREF(q, u) = 0.0;
  }
#pragma unroll 1
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* Bd = offd + (int64_t)d * NB * n + c;              // B_bd[q][a] at (q*NU + a)*n
    const double* Dn = dinv + nb;                                    // D_nb^-1[a][s] at (a*CR + s)*n
    const double* Bk = offd + (int64_t)opposite(d) * NB * n + nb;    // B_back[r][u] at (r*NU + u)*n
    double Bp[CR][CR], sr[CR];
#pragma unroll
    for (int q = 0; q < CR; ++q) {
      sr[q] = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < CR; ++s2) Bp[q][s2] = 0.0;
    }
#pragma unroll(kMcftUA)
    for (int a = 0; a < NU; ++a) {
      double bc[CR], dr[CR];
#pragma unroll
      for (int q = 0; q < CR; ++q) bc[q] = Bd[(int64_t)(q * NU + a) * n];
#pragma unroll
      for (int s2 = 0; s2 < CR; ++s2) dr[s2] = Dn[(int64_t)(a * CR + s2) * n];
      const double ra = b[(int64_t)a * n + nb];
#pragma unroll
      for (int q = 0; q < CR; ++q) {
        sr[q] = fma(bc[q], ra, sr[q]);
#pragma unroll
        for (int s2 = 0; s2 < CR; ++s2) Bp[q][s2] = fma(bc[q], dr[s2], Bp[q][s2]);
      }
    }
#pragma unroll
    for (int q = 0; q < CR; ++q) {
      grow[q] += sr[q];
#pragma unroll
      for (int s2 = 0; s2 < CR; ++s2)
        bp[(int64_t)((d * CR + q) * CR + s2) * g.half + t] = Bp[q][s2];
    }
#pragma unroll(kMcftUU)
    for (int u = 0; u < NU; ++u) {
      double oc[CR];
#pragma unroll
      for (int r = 0; r < CR; ++r) oc[r] = Bk[(int64_t)(r * NU + u) * n];
#pragma unroll
      for (int q = 0; q < CR; ++q) {
        double sq = 0.0;
#pragma unroll
        for (int r = 0; r < CR; ++r) sq = fma(Bp[q][r], oc[r], sq);
        QREF(q, u) += sq;
      }
    }
  }
  // QE = Q E_b: column u of the primary unknowns plus the secondary columns through E_S
  double QE[CR][CR];
  {
    double e[NCS][CR];
#pragma unroll
    for (int ii = 0; ii < NCS; ++ii)
#pragma unroll
      for (int u = 0; u < CR; ++u) e[ii][u] = es[(int64_t)(ii * CR + u) * g.half + t];
#pragma unroll
    for (int q = 0; q < CR; ++q)
#pragma unroll
      for (int u = 0; u < CR; ++u) {
        double v = QREF(q, cprim(u));
#pragma unroll
        for (int ii = 0; ii < NCS; ++ii) v = fma(QREF(q, csec(ii)), e[ii][u], v);
        QE[q][u] = v;
      }
  }
#undef QREF
  // rows of D_b^-1[:, :CR]: g_b = b_b - D_b^-1[:, :CR] grow (all nine), and
  // U6 = I - Dc_b^-1 QE from the primary rows
  double a[CR][CR];
#pragma unroll
  for (int q9 = 0; q9 < NU; ++q9) {
    double dr[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) dr[r] = dinv[(int64_t)(q9 * CR + r) * n + c];
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < CR; ++r) m = fma(dr[r], grow[r], m);
    g1[(int64_t)q9 * n + c] = b[(int64_t)q9 * n + c] - m;
    const bool prim = q9 != csec(0) && q9 != csec(1) && q9 != csec(2);
    if (prim) {
      const int q = q9 - (q9 > csec(0) ? 1 : 0) - (q9 > csec(1) ? 1 : 0);
#pragma unroll
      for (int u = 0; u < CR; ++u) {
        double s2 = 0.0;
#pragma unroll
        for (int r = 0; r < CR; ++r) s2 = fma(dr[r], QE[r][u], s2);
        a[q][u] = (q == u ? 1.0 : 0.0) - s2;
      }
    }
  }
  // in-place Gauss-Jordan (slot j ends as column perm[j] of the inverse):
  // the cooperative kernel's pivot rule and operations
  double amax = 0.0;
#pragma unroll
  for (int r = 0; r < CR; ++r)
#pragma unroll
    for (int u = 0; u < CR; ++u) amax = fmax(amax, fabs(a[r][u]));
  const double tol = 1e-13 * amax;
  bool bad = false;
  int perm[CR];
#pragma unroll
  for (int r = 0; r < CR; ++r) perm[r] = r;
#pragma unroll
  for (int kk = 0; kk < CR; ++kk) {
    int piv = kk;
    double pv = fabs(a[kk][kk]);
#pragma unroll
    for (int r = kk + 1; r < CR; ++r) {
      const double v = fabs(a[r][kk]);
      if (v > pv) { pv = v; piv = r; }
    }
    bad = bad || pv <= tol || amax == 0.0;
#pragma unroll
    for (int q = kk + 1; q < CR; ++q) {
      const bool sw = q == piv;
#pragma unroll
      for (int u = 0; u < CR; ++u) {
        const double x = a[kk][u];
        a[kk][u] = sel_d(sw, a[q][u], x);
        a[q][u] = sel_d(sw, x, a[q][u]);
      }
      const int x = perm[kk];
      perm[kk] = sel_i(sw, perm[q], x);
      perm[q] = sel_i(sw, x, perm[q]);
    }
    const double dv = 1.0 / a[kk][kk];
#pragma unroll
    for (int u = 0; u < CR; ++u) a[kk][u] = (u == kk ? 1.0 : a[kk][u]) * dv;
#pragma unroll
    for (int r = 0; r < CR; ++r) {
      if (r == kk) continue;
      const double f = a[r][kk];
      if (f != 0.0) {
#pragma unroll
        for (int u = 0; u < CR; ++u) a[r][u] = fma(-f, a[kk][u], u == kk ? 0.0 : a[r][u]);
      }
    }
  }
  if (bad) atomicMin(fail, 1);
#pragma unroll
  for (int u = 0; u < CR; ++u) {
    double* dst = uinv + (int64_t)perm[u] * n + c;
#pragma unroll
    for (int r = 0; r < CR; ++r) dst[(int64_t)(r * CR) * n] = a[r][u];
  }
}

// ------------------------------------------------------ condensed form
//
// The local rows ROW_OS.. of an assembled system (the oil and gas mole-
// fraction sums and the coke balance) have no flux: D[CR:, :] x_c = b[CR:]
// involves the cell's own unknowns only. They fix the secondary unknowns
// S = (last x, last y, C_c) of every cell in terms of the six primary ones
// P = (p, x_1, y_1, T, S_w, S_g):  x_S = E_S x_P + ...,  E_S = -D[CR:, S]^-1
// D[CR:, P]  (3 x 6 per cell). With E = [I; E_S] (9 x 6):
//   D^-1[:, :CR] = E Dc^-1,  Dc^-1 = D^-1[P, :CR]   (D E = [D[:CR,:] E; 0]),
// so the decoupled red-eliminated operator S9 z = z - D_b^-1[:, :CR] sum_d
// B'_bd y(z) (k_cc_black) maps z - range(E_b) into range(E_b), and its
// solution is x_b = g_b + E_b w with the 6-component
//   S6 w = w - Dc_b^-1 sum_d B'_bd sum_d' Bc_rd' w(nb) = h,
//   h = Dc_b^-1 sum_d B'_bd y_r(g),  Bc_rd = B_rd[:CR, :] E_b (6 x 6),
// y_r(g) the raw red pass on the reduced rhs g. BiCGSTAB with the
// multicolour preconditioner then runs on S6 (block-Jacobi U6 = I -
// Dc_b^-1 sum_d B'_bd Bc_r,back, the same ILU(0) pivot restricted to P):
// 6 x 36 + 6 x 36 + 36 matrix values per red/black pair and product instead
// of 6 x 49 + 6 x 36 + 54, 6-component Krylov vectors and a 36-value U6^-1
// instead of 81. It starts at x_b = g_b (w = 0) instead of 0, one product
// (for h) before the first iteration; on C2/C3 that start saves one
// iteration at LINEAR_TOL 1e-5 and 1e-10. Stopping test
// ||r6|| / ||b|| (r9 = E r6: the constraint rows' components of the full
// residual are left out of the norm).

// E_S of the black cells of g's [tw_lo, tw_hi) into es[(i*CR + p)*half + t];
// *fail = 1 when a cell's local block is not usable. The decoupling forms the
// owned cells' E_S from its registers; this kernel covers the ghost planes
// of a z-slab (their diagonal blocks are assembled here but not decoupled;
// the local rows' slots are never overwritten).
__global__ void k_cond_es(Dims g, const double* __restrict__ diag, double* __restrict__ es,
                          int* fail) {
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 1, t);
  double e[NCS][CR];
  if (!cond_es(diag, g.n, c, e)) atomicOr(fail, 1);
#pragma unroll
  for (int i = 0; i < NCS; ++i)
#pragma unroll
    for (int p = 0; p < CR; ++p) es[(int64_t)(i * CR + p) * g.half + t] = e[i][p];
}

// Red pass of S6: y_r = sum_d Bc_rd w(nb) (thread (red cell, row r < CR));
// Bc stored per red cell index t: cbc[((d*CR + r)*CR + p)*half + t]
__global__ void __launch_bounds__(32 * CR, CC_MINB) k_cc6_red(Dims g, const double* __restrict__ cbc,
                                                              double* __restrict__ z,
                                                              const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 0, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = cbc + (int64_t)((d * CR + r) * CR) * g.half + t;
    double tt = 0.0;
#pragma unroll
    for (int p = 0; p < CR; ++p) tt += blk[(int64_t)p * g.half] * z[(int64_t)p * n + nb];
    s += tt;
  }
  z[(int64_t)r * n + c] = s;
}

// Black pass of S6 (H = false): v_b = z_b - Dc_b^-1 sum_d B'_bd y(nb), with
// K dot products as k_cc_black; H = true: the rhs h = Dc_b^-1 sum_d B'_bd
// y(nb) into v, out2 and out3 (no dots).
template <int K, bool H>
__global__ void __launch_bounds__(32 * CR, CC_MINB) k_cc6_black(
    Dims g, const double* __restrict__ bp, const double* __restrict__ dinv,
    const double* __restrict__ z, double* __restrict__ v, const double* __restrict__ w0,
    const double* __restrict__ w1, double* partial, int stride, int slot0, const double* stop,
    double* __restrict__ out2, double* __restrict__ out3) {
  if (stopped(stop)) return;   // block-uniform: before the barrier
  __shared__ double ts[CR][32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  const bool live = t < g.tw_hi;
  int64_t c = 0;
  double acc[K > 0 ? K : 1];
#pragma unroll
  for (int q = 0; q < (K > 0 ? K : 1); ++q) acc[q] = 0.0;
  if (live) {
    c = colour_pos(g, 1, t);
    int i, j, k;
    const int64_t cell = locate(g, c, i, j, k);
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = bp + (int64_t)((d * CR + r) * CR) * g.half + t;
      double tt = 0.0;
#pragma unroll
      for (int e = 0; e < CR; ++e) tt += blk[(int64_t)e * g.half] * z[(int64_t)e * n + nb];
      s += tt;
    }
    ts[r][ls] = s;
  }
  __syncthreads();
  if (live) {
    const int q = r;   // output row q of Dc^-1 = D^-1[P[q], :CR]
    const int pq = q + (q >= NCO ? 1 : 0) + (q >= NCO + NCG - 1 ? 1 : 0);
    double m = 0.0;
#pragma unroll
    for (int rr = 0; rr < CR; ++rr) m += dinv[(int64_t)(pq * CR + rr) * n + c] * ts[rr][ls];
    if (H) {
      v[(int64_t)q * n + c] = m;
      out2[(int64_t)q * n + c] = m;
      out3[(int64_t)q * n + c] = m;
    } else {
      const double val = z[(int64_t)q * n + c] - m;
      v[(int64_t)q * n + c] = val;
      const double wd = K == 1 ? w0[(int64_t)q * n + c] : (K == 2 ? w1[(int64_t)q * n + c] : 0.0);
      if (K == 1) acc[0] += val * wd;
      if (K == 2) { acc[0] += val * val; acc[K - 1] += val * wd; }
    }
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double x = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (ls == 0) partial[(int64_t)q * stride * CR + (int64_t)(slot0 + blockIdx.x) * CR + r] = x;
  }
}

// The raw red pass on the reduced rhs g (y_r = sum_d B_rd[:CR, :] g(nb), as
// k_cc_red, for h) fused with forming the condensed red blocks
//   Bc_rd[q][p] = B_rd[q][P[p]] + sum_i B_rd[q][S[i]] E_nb[i][p]
// from the same block loads and the black neighbours' E_S (k_cond_es covers
// ghost planes, so on z-slabs the boundary planes' blocks towards the ghost
// planes come out here too). Thread (red cell, row q), owned planes.
__global__ void __launch_bounds__(32 * CR, CC_MINB) k_cc_red_bc(Dims g, const double* __restrict__ offd,
                                                                const int* __restrict__ ccnz,
                                                                const double* __restrict__ es,
                                                                double* __restrict__ z,
                                                                double* __restrict__ cbc) {
  const int64_t n = g.n;
  const int ls = threadIdx.x, q = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  if (t >= g.tw_hi) return;
  const bool skip_cc = q < ROW_E && *ccnz == 0;   // warp-uniform (one row per warp)
  const int64_t c = colour_pos(g, 0, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = offd + (int64_t)((d * NU + q) * NU) * n + c;
    double bv[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) bv[u] = (u == CCC && skip_cc) ? 0.0 : blk[(int64_t)u * n];
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (u == CCC && skip_cc) continue;
      tt += bv[u] * z[(int64_t)u * n + nb];
    }
    s += tt;
    const int64_t tb = nb - g.ph * (int64_t)(plane_of(g, nb) + 1);   // black index of nb
#pragma unroll
    for (int p = 0; p < CR; ++p) {
      double v = bv[cprim(p)];
#pragma unroll
      for (int ii = 0; ii < NCS; ++ii)
        v += bv[csec(ii)] * es[(int64_t)(ii * CR + p) * g.half + tb];
      cbc[(int64_t)((d * CR + q) * CR + p) * g.half + t] = v;
    }
  }
  z[(int64_t)q * n + c] = s;
}

// x_r = b_r - D_r^-1[:, :CR] (y_r(g) + sum_d Bc_rd w(nb)) -- the red
// back-substitution b_r - B_rb x_b with x_b = g_b + E_b w, from the raw red
// pass on g (kept in g's red positions by k_cc_red_bc) and the 6x6 Bc blocks
// instead of the 6x9 raw ones. Thread (red cell, row r < CR), then output
// rows q = r, r + CR as k_cc_xred.
__global__ void __launch_bounds__(32 * CR, CP_MINB) k_cc6_xred(Dims g, const double* __restrict__ cbc,
                                                               const double* __restrict__ dinv,
                                                               const double* __restrict__ yg,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ x) {
  __shared__ double ts[CR][32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;
  const bool live = t < g.tw_hi;
  int64_t c = 0;
  if (live) {
    c = colour_pos(g, 0, t);
    int i, j, k;
    const int64_t cell = locate(g, c, i, j, k);
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = cbc + (int64_t)((d * CR + r) * CR) * g.half + t;
      double tt = 0.0;
#pragma unroll
      for (int p = 0; p < CR; ++p) tt += blk[(int64_t)p * g.half] * x[(int64_t)p * n + nb];
      s += tt;
    }
    ts[r][ls] = yg[(int64_t)r * n + c] + s;
  }
  __syncthreads();
  if (live) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = r + h * CR;
      if (q >= NU) break;
      double m = 0.0;
#pragma unroll
      for (int rr = 0; rr < CR; ++rr) m += dinv[(int64_t)(q * CR + rr) * n + c] * ts[rr][ls];
      x[(int64_t)q * n + c] = b[(int64_t)q * n + c] - m;
    }
  }
}

// x_b = g_b + E_b w_b (9 rows out of the 6-component w in rows 0..CR-1 of x)
__global__ void k_cond_expand(Dims g, const double* __restrict__ es,
                              const double* __restrict__ gb, double* __restrict__ x) {
  const int64_t n = g.n;
  for (int64_t t = g.tw_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.tw_hi;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = colour_pos(g, 1, t);
    double w[CR];
#pragma unroll
    for (int p = 0; p < CR; ++p) w[p] = x[(int64_t)p * n + c];
#pragma unroll
    for (int p = 0; p < CR; ++p)
      x[(int64_t)cprim(p) * n + c] = gb[(int64_t)cprim(p) * n + c] + w[p];
#pragma unroll
    for (int i = 0; i < NCS; ++i) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < CR; ++p) s += es[(int64_t)(i * CR + p) * g.half + t] * w[p];
      x[(int64_t)csec(i) * n + c] = gb[(int64_t)csec(i) * n + c] + s;
    }
  }
}

// An imported system qualifies for the compact form when every
// off-diagonal block of an existing connection has zero rows CR..8 (the
// structure an assembled system has): *flag = 1 otherwise.
__global__ void k_flux_rows_only(Dims g, const double* __restrict__ offd, int* flag) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  bool nz = false;
  for (int d = 0; d < NDIR; ++d) {
    if (nb_pos(g, cell, i, j, k, d) < 0) continue;
    for (int r = CR; r < NU; ++r)
#pragma unroll
      for (int u = 0; u < NU; ++u) nz |= offd[(int64_t)((d * NU + r) * NU + u) * n + c] != 0.0;
  }
  if (nz) atomicOr(flag, 1);
}

}  // namespace isc
