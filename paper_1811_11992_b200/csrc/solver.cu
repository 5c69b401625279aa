// Decoupled-system operators: 7-point BSR SpMV, fused Krylov vector updates
// with deterministic dot products, and the reference's subdomain block
// ILU(0) (bjacobi / RAS) run as a level-scheduled wavefront.
//
// Vectors are SoA v[r*n + c]. The decoupled diagonal block is the identity
// (decouple.cu), so  y = x + sum_d B_d x_{nb_d}  (linsolve.py:159-177).
#include <cooperative_groups.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace isc {

// Blocks per SM for the bandwidth-bound stencil passes: fewer resident blocks
// but more registers per thread keeps more independent loads in flight per
// warp, which is what these streams need (C4 sweep 2..7: 3 best for the
// multicolour passes, 4 for the full SpMV; profiles/r1/minb_sweep.md).
#ifndef MC_MINB
#define MC_MINB 3
#endif
#ifndef SPMV_MINB
#define SPMV_MINB 4
#endif


constexpr int RED_BLOCKS = 148 * 8;   // fixed partition -> deterministic sums
constexpr int FIN_BLOCKS = 148;       // first stage of the two-stage partial sums
constexpr int RED_THREADS = 256;

// Krylov scalar slots in device memory (host mirror reads them)
enum {
  S_RHO = 0, S_RHO_OLD, S_ALPHA, S_OMEGA, S_DEN, S_SS, S_TT, S_TS, S_RR, S_RHO_NEW, S_BB,
  S_FIRST,
  // device-driven BiCGSTAB (bicgstab_schur): control state kept in HBM
  S_STOP, S_IT, S_MAXIT, S_NB, S_TOL, S_BRK,
  S_NSCAL
};
// S_STOP codes: why the device-driven iteration stopped (0 = running)
enum { STOP_RUN = 0, STOP_TOP = 1, STOP_DEN = 2, STOP_CONV_S = 3, STOP_TT = 4, STOP_CONV = 5,
       STOP_MAXIT = 6, STOP_ZERO = 7 };

// every kernel of a device-driven iteration returns at once when `stop`
// (nullable: host-driven callers) holds a nonzero code
__device__ __forceinline__ bool stopped(const double* stop) { return stop && *stop != 0.0; }

// scalar steps of the device-driven BiCGSTAB (linsolve.py:500-575), run by
// one thread after the dot product they need (k_bicg_* or fused into the
// fixed-order sum that produced it, k_finalize's `post`)
enum { POST_NONE = 0, POST_DEN = 1, POST_SS = 2, POST_END = 3 };
__device__ __forceinline__ void bicg_den(double* sc) {   // after r^.v: denominator test, alpha
  if (sc[S_STOP] != 0.0) return;
  const double den = sc[S_DEN];
  if (fabs(den) < sc[S_BRK]) { sc[S_STOP] = STOP_DEN; return; }
  sc[S_ALPHA] = sc[S_RHO] / den;
}
__device__ __forceinline__ void bicg_ss(double* sc) {    // after ||s||: early convergence
  if (sc[S_STOP] != 0.0) return;
  if (sqrt(sc[S_SS]) / sc[S_NB] <= sc[S_TOL]) sc[S_STOP] = STOP_CONV_S;
}
__device__ __forceinline__ void bicg_end(double* sc) {   // after t.t, t.s, ||r||, r^.r
  if (sc[S_STOP] != 0.0) return;
  const double tt = sc[S_TT];
  if (tt == 0.0) { sc[S_STOP] = STOP_TT; return; }
  sc[S_OMEGA] = sc[S_TS] / tt;
  if (sqrt(sc[S_RR]) / sc[S_NB] <= sc[S_TOL]) { sc[S_STOP] = STOP_CONV; return; }
  sc[S_RHO_OLD] = sc[S_RHO];
  sc[S_FIRST] = 0.0;
}

template <int K>
__device__ __forceinline__ void block_reduce_store(double (&v)[K], double* partial) {
  __shared__ double sh[K][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane2 = tid & 31, wid2 = tid >> 5;
  (void)lane; (void)wid;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane2 == 0) sh[k][wid2] = x;
  }
  __syncthreads();
  const int nwarps = (blockDim.x * blockDim.y) >> 5;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += sh[k][w];
      partial[k * gridDim.x + blockIdx.x] = s;
    }
  }
}

// per-warp partials, no block barrier: lane 0 of warp y (block = 32 x NU)
// stores partial[k*stride + slot*NU + y]. A block-wide reduction would make
// every warp of the stencil passes wait for the block's slowest one, which
// costs ~30 % of their bandwidth (tools/layout_probe.cu).
template <int K>
__device__ __forceinline__ void warp_store_at(double (&v)[K], double* partial, int64_t stride,
                                              int64_t slot) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (threadIdx.x == 0) partial[(int64_t)k * stride + slot * NU + threadIdx.y] = x;
  }
}

// first stage of a two-stage fixed-order sum: block b reduces the contiguous
// chunk b of each of the K partial arrays into out[k*gridDim.x + b]
template <int K>
__global__ void __launch_bounds__(256) k_partial_sum(const double* __restrict__ partial,
                                                     int64_t nparts, double* __restrict__ out,
                                                     const double* stop) {
  if (stopped(stop)) return;
  __shared__ double sh[K][8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t chunk = (nparts + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < nparts ? lo + chunk : nparts;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int64_t i = lo + t; i < hi; i += 256) s += partial[(int64_t)k * nparts + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) sh[k][w] = s;
  }
  __syncthreads();
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i) s += sh[k][i];
      out[(int64_t)k * gridDim.x + blockIdx.x] = s;
    }
  }
}

// sum the per-block partials in fixed order into sc[slot_k] (256 threads)
template <int K>
__device__ __forceinline__ void finalize_block(const double* __restrict__ partial, int nparts,
                                               double* sc, int s0, int s1, int post) {
  const int slots[2] = {s0, s1};
  __shared__ double sh[K][8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int i = t; i < nparts; i += 256) s += partial[(int64_t)k * nparts + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) sh[k][w] = s;
  }
  __syncthreads();
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i) s += sh[k][i];
      sc[slots[k]] = s;
    }
    if (post == POST_DEN) bicg_den(sc);
    else if (post == POST_SS) bicg_ss(sc);
    else if (post == POST_END) bicg_end(sc);
  }
}
template <int K>
__global__ void __launch_bounds__(256) k_finalize(const double* __restrict__ partial, int nparts,
                                                  double* sc, int s0, int s1, int s2,
                                                  const double* stop, int post) {
  if (stopped(stop)) return;
  finalize_block<K>(partial, nparts, sc, s0, s1, post);
}

// both stages of the fixed-order sum in one launch: the last block to finish
// its chunk (ticket) runs the second stage over out[] exactly as k_finalize
// would, then resets the ticket
template <int K>
__global__ void __launch_bounds__(256) k_partial_sum_fin(const double* __restrict__ partial,
                                                         int64_t nparts, double* out, double* sc,
                                                         int s0, int s1, const double* stop,
                                                         int post, unsigned* ticket) {
  if (stopped(stop)) return;
  __shared__ double sh[K][8];
  __shared__ bool last;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t chunk = (nparts + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < nparts ? lo + chunk : nparts;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int64_t i = lo + t; i < hi; i += 256) s += partial[(int64_t)k * nparts + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) sh[k][w] = s;
  }
  __syncthreads();
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i) s += sh[k][i];
      out[(int64_t)k * gridDim.x + blockIdx.x] = s;
    }
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_block<K>(out, gridDim.x, sc, s0, s1, post);
  if (t == 0) *ticket = 0u;
}

// partial dot products of up to 3 vector pairs over len entries
template <int K>
__global__ void __launch_bounds__(RED_THREADS) k_dots(int64_t len, const double* a0, const double* b0,
                                                      const double* a1, const double* b1,
                                                      const double* a2, const double* b2,
                                                      double* partial) {
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc[0] += a0[i] * b0[i];
    if (K > 1) acc[K > 1 ? 1 : 0] += a1[i] * b1[i];
    if (K > 2) acc[K > 2 ? 2 : 0] += a2[i] * b2[i];
  }
  block_reduce_store<K>(acc, partial);
}

// ------------------------------------------------------------------- SpMV
// y = x + sum_d B_d x_nb ; optional fused partial dots of y with (w0, w1):
// grid (ceil(n/32)), block (32, NU): thread (c, r).
template <int K>
__global__ void __launch_bounds__(32 * NU, SPMV_MINB) k_spmv(Dims g, const double* __restrict__ offd,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y,
                                                  const double* __restrict__ w0,
                                                  const double* __restrict__ w1,
                                                  double* partial) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int r = threadIdx.y;
  constexpr int KK = K > 0 ? K : 1;
  double acc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) acc[k] = 0.0;
  bool own = false;
  int64_t cell = 0;
  int i = 0, j = 0, k = 0;
  if (c < n) {
    cell = locate(g, c, i, j, k);
    own = owned_k(g, k);
  }
  if (own) {   // ghost rows carry no equation (multi-GPU slabs)
    double s = x[r * n + c];
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) t += __ldg(blk + (int64_t)u * n) * __ldg(x + (int64_t)u * n + nb);
      s += t;
    }
    y[r * n + c] = s;
    // K == 1: (y . w0) ; K == 2: (y . y, y . w1)
    if (K == 1) acc[0] = s * w0[r * n + c];
    if (K == 2) { acc[0] = s * s; acc[K > 1 ? 1 : 0] = s * w1[r * n + c]; }
  }
  if (K > 0) warp_store_at<KK>(acc, partial, (int64_t)gridDim.x * NU, blockIdx.x);
}

// --------------------------------------------------------- vector kernels
// p = r + beta (p - omega v),  beta = (rho/rho_old)(alpha/omega); or p = r
__global__ void k_update_p(int64_t len, const double* __restrict__ r, double* __restrict__ p,
                           const double* __restrict__ v, const double* __restrict__ sc) {
  const bool first = sc[S_FIRST] != 0.0;
  const double beta = (sc[S_RHO] / sc[S_RHO_OLD]) * (sc[S_ALPHA] / sc[S_OMEGA]);
  const double omega = sc[S_OMEGA];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = first ? r[i] : r[i] + beta * (p[i] - omega * v[i]);
}

// alpha = rho/den; s = r - alpha v; partial s.s
__global__ void __launch_bounds__(RED_THREADS) k_update_s(int64_t len, const double* __restrict__ r,
                                                          const double* __restrict__ v,
                                                          double* __restrict__ s, double* sc,
                                                          double* partial) {
  const double alpha = sc[S_RHO] / sc[S_DEN];
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double si = r[i] - alpha * v[i];
    s[i] = si;
    acc[0] += si * si;
  }
  block_reduce_store<1>(acc, partial);
}

__global__ void k_store_alpha(double* sc) { sc[S_ALPHA] = sc[S_RHO] / sc[S_DEN]; }

// x += alpha phat
__global__ void k_axpy_alpha(int64_t len, double* __restrict__ x, const double* __restrict__ ph,
                             const double* __restrict__ sc) {
  const double alpha = sc[S_ALPHA];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] += alpha * ph[i];
}

// omega = ts/tt; x += alpha phat + omega shat; r = s - omega t; partial r.r, rhat.r
__global__ void __launch_bounds__(RED_THREADS) k_update_xr(int64_t len, double* __restrict__ x,
                                                           const double* __restrict__ ph,
                                                           const double* __restrict__ sh_,
                                                           double* __restrict__ r,
                                                           const double* __restrict__ s,
                                                           const double* __restrict__ t,
                                                           const double* __restrict__ rhat,
                                                           const double* sc, double* partial) {
  const double tt = sc[S_TT];
  double acc[2] = {0.0, 0.0};
  if (tt != 0.0) {
    const double alpha = sc[S_ALPHA];
    const double omega = sc[S_TS] / tt;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x) {
      x[i] += alpha * ph[i] + omega * sh_[i];
      const double ri = s[i] - omega * t[i];
      r[i] = ri;
      acc[0] += ri * ri;
      acc[1] += rhat[i] * ri;
    }
  }
  block_reduce_store<2>(acc, partial);
}

__global__ void k_sub(int64_t len, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// --------------------------------------------------- subdomain ILU(0)
//
// Slots: every (subdomain, extended cell) pair, numbered level-major where
// the level of a cell inside its subdomain box is (i-x0)+(j-y0)+(k-z0);
// cells of one level depend only on the previous level (natural-order
// ILU(0) on a 7-point stencil == block D-ILU, linsolve.py:206-259).
struct IluDev {
  int64_t nslots;
  const int64_t* __restrict__ cell;    // global cell of a slot
  const int8_t* __restrict__ owned;    // slot owns its cell (RAS restriction)
  const int64_t* __restrict__ lo;      // [3*nslots] lower neighbour slots (-z,-y,-x) or -1
  const int64_t* __restrict__ up;      // [3*nslots] upper neighbour slots (+x,+y,+z) or -1
  double* lblk;                        // [(q*NB + e)*nslots + s]  A_cj U_jj^-1
  double* uinv;                        // [e*nslots + s]
  double* zs;                          // [r*nslots + s] local solution
  double* aup;                         // [(q*NB + e)*nslots + s]  upper blocks, slot order
};

#ifndef IL_SLOTS_N
#define IL_SLOTS_N 32
#endif
constexpr int IL_SLOTS = IL_SLOTS_N;   // slots per tile (CTA = IL_SLOTS x NU threads)

// U = I - sum_j (A_cj U_j^-1) A_jc ; uinv = U^-1 (GJ, partial pivoting)
// Thread (slot, column u). The three lower blocks A_cj are staged through
// shared memory (one scattered column per thread instead of 81 loads), the
// matching A_jc columns stay in registers and are also written out in slot
// order as the upper block of slot j (coalesced reads in the apply sweep).
struct FactorSmem {
  double ash[3][NU][NU][IL_SLOTS];   // A_cj (q, row, col) for the tile
  double lsh[NU][NU][IL_SLOTS];      // one lblk (row, col) for the tile
  double colk[2 * NU][IL_SLOTS];
  int pivs[IL_SLOTS];
};

__device__ void ilu_factor_tile(const Dims& g, const IluDev& L, const double* __restrict__ offd,
                                int64_t s0, int64_t s1, int* fail, FactorSmem& S) {
  auto& ash = S.ash;
  auto& lsh = S.lsh;
  auto& colk = S.colk;
  auto& pivs = S.pivs;
  const int64_t n = g.n;
  const int ls = threadIdx.x, u = threadIdx.y;   // slot lane, owned column
  const int64_t s = s0 + ls;
  const bool live = s < s1;
  const int64_t ns = L.nslots;
  const int64_t c = live ? L.cell[s] : 0;
  const int dlo[3] = {DZM, DYM, DXM};
  // independent of the previous level: neighbour slots, A_cj and A_jc columns
  int64_t sj[3];
  double ajc[3][NU];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    sj[q] = live ? L.lo[q * ns + s] : -1;
    if (sj[q] >= 0) {
      const double* Acj = offd + (int64_t)(dlo[q] * NB + u) * n + c;
#pragma unroll
      for (int r = 0; r < NU; ++r) ash[q][r][u][ls] = Acj[(int64_t)(r * NU) * n];
      const int64_t cj = L.cell[sj[q]];
      const double* Ajc = offd + (int64_t)(opposite(dlo[q]) * NB + u) * n + cj;
#pragma unroll
      for (int k = 0; k < NU; ++k) ajc[q][k] = Ajc[(int64_t)(k * NU) * n];
      // upper block of slot j towards this slot (q' = 2 - q: +z, +y, +x order)
#pragma unroll
      for (int k = 0; k < NU; ++k) L.aup[(int64_t)((2 - q) * NB + k * NU + u) * ns + sj[q]] = ajc[q][k];
    } else {
#pragma unroll
      for (int k = 0; k < NU; ++k) ajc[q][k] = 0.0;
    }
  }
  // own column u of U (starts at the identity: decoupled diagonal)
  double ucol[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) ucol[r] = (r == u) ? 1.0 : 0.0;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    // lblk[:, u] = A_cj * Uinv_j[:, u]
    double lc[NU];
#pragma unroll
    for (int r = 0; r < NU; ++r) lc[r] = 0.0;
    if (sj[q] >= 0) {
      double uj[NU];
#pragma unroll
      for (int k = 0; k < NU; ++k) uj[k] = __ldcg(L.uinv + (int64_t)(k * NU + u) * ns + sj[q]);
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < NU; ++k) t += ash[q][r][k][ls] * uj[k];
        lc[r] = t;
      }
#pragma unroll
      for (int r = 0; r < NU; ++r) L.lblk[(int64_t)(q * NB + r * NU + u) * ns + s] = lc[r];
    }
#pragma unroll
    for (int r = 0; r < NU; ++r) lsh[r][u][ls] = lc[r];
    __syncthreads();
    if (sj[q] >= 0) {
      // U[:, u] -= lblk * A_jc[:, u]
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < NU; ++k) t += lsh[r][k][ls] * ajc[q][k];
        ucol[r] -= t;
      }
    }
    __syncthreads();
  }
  // Gauss-Jordan inverse of U; thread owns column u of U and column u of inv
  double icol[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) icol[r] = (r == u) ? 1.0 : 0.0;
  // tolerance 1e-13 * max|U|
  {
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < NU; ++r) m = fmax(m, fabs(ucol[r]));
    lsh[0][u][ls] = m;
  }
  __syncthreads();
  double amax = 0.0;
#pragma unroll
  for (int k = 0; k < NU; ++k) amax = fmax(amax, lsh[0][k][ls]);
  const double tol = 1e-13 * amax;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    if (u == k) {
      int piv = k;
      double pv = fabs(ucol[k]);
#pragma unroll
      for (int r = k + 1; r < NU; ++r) {
        const double v = fabs(ucol[r]);
        if (v > pv) { pv = v; piv = r; }
      }
      if ((pv <= tol || amax == 0.0) && live) atomicMin(fail, 1);
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double v = ucol[r];
        if (r == k) {
#pragma unroll
          for (int q2 = k + 1; q2 < NU; ++q2) if (q2 == piv) v = ucol[q2];
        } else if (r == piv) {
          v = ucol[k];
        }
        colk[r][ls] = v;
      }
      pivs[ls] = piv;
    }
    __syncthreads();
    const int piv = pivs[ls];
    if (piv != k) {
      double t0 = ucol[k], t1 = icol[k];
#pragma unroll
      for (int q2 = k + 1; q2 < NU; ++q2)
        if (q2 == piv) { ucol[k] = ucol[q2]; icol[k] = icol[q2]; ucol[q2] = t0; icol[q2] = t1; }
    }
    const double dinv = 1.0 / colk[k][ls];
    ucol[k] *= dinv;
    icol[k] *= dinv;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      if (r == k) continue;
      const double f = colk[r][ls];
      if (f != 0.0) {
        ucol[r] -= f * ucol[k];
        icol[r] -= f * icol[k];
      }
    }
    __syncthreads();
  }
  if (live) {
#pragma unroll
    for (int r = 0; r < NU; ++r) L.uinv[(int64_t)(r * NU + u) * ns + s] = icol[r];
  }
}

// One thread-block cluster per subdomain (subdomains are independent):
// levels are separated by a cluster barrier (release/acquire at cluster
// scope) instead of a grid-wide sync, and values produced by other CTAs of
// the cluster are read through L2 (__ldcg).
#ifndef ILC_APPLY
#define ILC_APPLY 4
#endif
constexpr int ILC = ILC_APPLY;    // CTAs per cluster (apply; 64 clusters stay resident)
#ifndef ILCF_FACTOR
#define ILCF_FACTOR 4
#endif
constexpr int ILCF = ILCF_FACTOR;   // CTAs per cluster (factor: 2 CTAs/SM -> one resident wave)

#ifndef ILF_MINB
#define ILF_MINB 1   // C4 RAS factorisation 45.3 -> 32.8 ms (no spills)
#endif
#ifndef ILA_MINB
#define ILA_MINB 2
#endif
__global__ void __cluster_dims__(ILCF, 1, 1) __launch_bounds__(IL_SLOTS * NU, ILF_MINB)
    k_ilu_factor(Dims g, IluDev L, const double* offd, const int64_t* __restrict__ sub_ptr,
                 int nlev, int* fail) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char dsm[];
  FactorSmem& S = *reinterpret_cast<FactorSmem*>(dsm);
  const int sub = blockIdx.x / ILCF, crank = blockIdx.x % ILCF;
  const int64_t* lp = sub_ptr + (int64_t)sub * (nlev + 1);
  for (int lev = 0; lev < nlev; ++lev) {
    const int64_t b = lp[lev], e = lp[lev + 1];
    for (int64_t s0 = b + (int64_t)crank * IL_SLOTS; s0 < e; s0 += (int64_t)ILCF * IL_SLOTS)
      ilu_factor_tile(g, L, offd, s0, e, fail, S);
    cluster.sync();
  }
}

// forward then backward sweep; z_out (global, SoA) gets the owned slots
__global__ void __cluster_dims__(ILC, 1, 1) __launch_bounds__(IL_SLOTS * NU, ILA_MINB)
    k_ilu_apply(Dims g, IluDev L, const double* offd, const int64_t* __restrict__ sub_ptr,
                int nlev, const double* __restrict__ rin, double* __restrict__ zout) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double wsh[NU][IL_SLOTS];
  const int64_t n = g.n, ns = L.nslots;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int sub = blockIdx.x / ILC, crank = blockIdx.x % ILC;
  const int64_t* lp = sub_ptr + (int64_t)sub * (nlev + 1);
  // forward: z_c = r_c - sum_j lblk_cj z_j   (lower j in order -z,-y,-x)
  for (int lev = 0; lev < nlev; ++lev) {
    const int64_t b = lp[lev], e = lp[lev + 1];
    for (int64_t s = b + (int64_t)crank * IL_SLOTS + ls; s < e; s += (int64_t)ILC * IL_SLOTS) {
      // every load of the slot issued before the first use (the level's
      // latency is one round trip, not one per neighbour)
      const int64_t c = L.cell[s];
      int64_t sj[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) sj[q] = L.lo[q * ns + s];
      double lb[3][NU], zn[3][NU];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int64_t jj = sj[q] >= 0 ? sj[q] : s;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          lb[q][u] = L.lblk[(int64_t)(q * NB + r * NU + u) * ns + s];
          zn[q][u] = __ldcg(L.zs + (int64_t)u * ns + jj);
        }
      }
      double z = rin[r * n + c];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (sj[q] < 0) continue;
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < NU; ++u) t += lb[q][u] * zn[q][u];
        z -= t;
      }
      L.zs[(int64_t)r * ns + s] = z;
    }
    cluster.sync();
  }
  // backward: z_c = U_c^-1 (z_c - sum_j A_cj z_j)   (upper j in order +x,+y,+z)
  for (int lev = nlev - 1; lev >= 0; --lev) {
    const int64_t b = lp[lev], e = lp[lev + 1];
    for (int64_t s0 = b + (int64_t)crank * IL_SLOTS; s0 < e; s0 += (int64_t)ILC * IL_SLOTS) {
      const int64_t s = s0 + ls;
      const bool live = s < e;
      double w = 0.0;
      int64_t c = 0;
      if (live) {
        c = L.cell[s];
        int64_t sj[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) sj[q] = L.up[q * ns + s];
        double ab[3][NU], zn[3][NU];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int64_t jj = sj[q] >= 0 ? sj[q] : s;
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            ab[q][u] = L.aup[(int64_t)(q * NB + r * NU + u) * ns + s];
            zn[q][u] = __ldcg(L.zs + (int64_t)u * ns + jj);
          }
        }
        w = __ldcg(L.zs + (int64_t)r * ns + s);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (sj[q] < 0) continue;
          double t = 0.0;
#pragma unroll
          for (int u = 0; u < NU; ++u) t += ab[q][u] * zn[q][u];
          w -= t;
        }
      }
      wsh[r][ls] = w;
      __syncthreads();
      if (live) {
        double z = 0.0;
#pragma unroll
        for (int u = 0; u < NU; ++u) z += L.uinv[(int64_t)(r * NU + u) * ns + s] * wsh[u][ls];
        L.zs[(int64_t)r * ns + s] = z;
        if (L.owned[s]) zout[r * n + c] = z;
      }
      __syncthreads();
    }
    cluster.sync();
  }
}

// ------------------------------------------- multicolour block ILU(0)
// Red-black ordering (red: i+j+k even) of the decoupled system A = I + sum B_d.
// Red rows have no lower neighbours, so U_red = I and L_black,red = A; the
// black pivots are U_b = I - sum_d B_bd B_{nb,-d}. Apply (M = LU):
//   pass 1 (black):  z_b = U_b^-1 (r_b - sum_d B_bd r_nb)
//   pass 2 (red):    z_r = r_r - sum_d B_rd z_nb
// Every pass is fully parallel (no wavefront); BASELINE north_star's
// "multicolour block-ILU(0)".

__device__ __forceinline__ bool is_black(const Dims& g, int i, int j, int k) {
  return ((i + j + k + g.kpar) & 1) != 0;
}

// thread (cell lane, column u); black cells only do work
#ifndef MCF_MINB
#define MCF_MINB 3   // C4 sweep 2..5: 3.4 -> 2.5 ms at 3
#endif
__global__ void __launch_bounds__(32 * NU, MCF_MINB) k_mc_factor(Dims g, const double* __restrict__ offd,
                                                          double* __restrict__ uinv, int* fail,
                                                          int cross) {
  __shared__ double bsh[NU][NU][32];   // B_bd (row, col) of the current direction
  __shared__ double colk[NU][32];
  __shared__ int pivs[32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, u = threadIdx.y;
  const int64_t t = (int64_t)blockIdx.x * 32 + ls;   // t-th black cell when colour-blocked
  const bool in = t < (g.colored ? g.half : n);
  const int64_t c = g.colored ? (in ? colour_pos(g, 1, t) : 0) : t;
  int i = 0, j = 0, k = 0;
  const int64_t cell = in ? locate(g, c, i, j, k) : 0;
  const bool live = in && is_black(g, i, j, k) && owned_k(g, k);
  double ucol[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) ucol[r] = (r == u) ? 1.0 : 0.0;
#pragma unroll 1
  for (int d = 0; d < NDIR; ++d) {
    int64_t nb = live ? nb_pos(g, cell, i, j, k, d) : -1;
    // slabs: a ghost-plane neighbour's block pointing back at this cell is the
    // owner rank's (exchanged after decoupling) when cross != 0; otherwise the
    // factor is rank-local
    if (!cross && ((d == DZM && !owned_k(g, k - 1)) || (d == DZP && !owned_k(g, k + 1)))) nb = -1;
    if (nb >= 0) {
      const double* B = offd + (int64_t)(d * NB + u) * n + c;
#pragma unroll
      for (int r = 0; r < NU; ++r) bsh[r][u][ls] = B[(int64_t)(r * NU) * n];
    }
    __syncthreads();
    if (nb >= 0) {
      const double* Bo = offd + (int64_t)(opposite(d) * NB + u) * n + nb;   // column u
      double bc[NU];
#pragma unroll
      for (int q = 0; q < NU; ++q) bc[q] = Bo[(int64_t)(q * NU) * n];
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NU; ++q) t += bsh[r][q][ls] * bc[q];
        ucol[r] -= t;
      }
    }
    __syncthreads();
  }
  // Gauss-Jordan inverse (partial pivoting, tolerance 1e-13 max|U|)
  double icol[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) icol[r] = (r == u) ? 1.0 : 0.0;
  {
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < NU; ++r) m = fmax(m, fabs(ucol[r]));
    bsh[0][u][ls] = m;
  }
  __syncthreads();
  double amax = 0.0;
#pragma unroll
  for (int q = 0; q < NU; ++q) amax = fmax(amax, bsh[0][q][ls]);
  const double tol = 1e-13 * amax;
  __syncthreads();
#pragma unroll
  for (int kk = 0; kk < NU; ++kk) {
    if (u == kk) {
      int piv = kk;
      double pv = fabs(ucol[kk]);
#pragma unroll
      for (int r = kk + 1; r < NU; ++r) {
        const double v = fabs(ucol[r]);
        if (v > pv) { pv = v; piv = r; }
      }
      if (live && (pv <= tol || amax == 0.0)) atomicMin(fail, 1);
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        double v = ucol[r];
        if (r == kk) {
#pragma unroll
          for (int q = kk + 1; q < NU; ++q) if (q == piv) v = ucol[q];
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
      double t0 = ucol[kk], t1 = icol[kk];
#pragma unroll
      for (int q = kk + 1; q < NU; ++q)
        if (q == piv) { ucol[kk] = ucol[q]; icol[kk] = icol[q]; ucol[q] = t0; icol[q] = t1; }
    }
    const double dinv = 1.0 / colk[kk][ls];
    ucol[kk] *= dinv;
    icol[kk] *= dinv;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      if (r == kk) continue;
      const double f = colk[r][ls];
      if (f != 0.0) { ucol[r] -= f * ucol[kk]; icol[r] -= f * icol[kk]; }
    }
    __syncthreads();
  }
  if (live) {
#pragma unroll
    for (int r = 0; r < NU; ++r) uinv[(int64_t)(r * NU + u) * n + c] = icol[r];
  }
}

// pass 1 (black rows) / pass 2 (red rows); thread (cell lane, row r)
template <int PASS>
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_mc_apply(Dims g, const double* __restrict__ offd,
                                                      const double* __restrict__ uinv,
                                                      const double* __restrict__ rin,
                                                      double* __restrict__ z) {
  __shared__ double wsh[NU][32];
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  // colour-blocked storage: pass 1 covers the black cells, pass 2 the red cells
  const int64_t t = (int64_t)blockIdx.x * 32 + ls;
  const bool in = t < (g.colored ? g.half : n);
  const int64_t c = g.colored ? (in ? colour_pos(g, PASS == 1 ? 1 : 0, t) : 0) : t;
  int i = 0, j = 0, k = 0;
  const int64_t cell = in ? locate(g, c, i, j, k) : 0;
  const bool live = in && (is_black(g, i, j, k) == (PASS == 1)) && owned_k(g, k);
  double w = 0.0;
  if (live) {
    // pass 1 reads red neighbours of r (z_red = r_red); pass 2 the black z
    const double* src = PASS == 1 ? rin : z;
    w = rin[r * n + c];
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      if ((d == DZM && !owned_k(g, k - 1)) || (d == DZP && !owned_k(g, k + 1))) continue;
      const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) t += blk[(int64_t)u * n] * src[(int64_t)u * n + nb];
      w -= t;
    }
  }
  if (PASS == 2) {
    if (live) z[r * n + c] = w;
    return;
  }
  wsh[r][ls] = w;
  __syncthreads();
  if (live) {
    double zz = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) zz += uinv[(int64_t)(r * NU + u) * n + c] * wsh[u][ls];
    z[r * n + c] = zz;
  }
}

// ------------------------- multicolour preconditioner fused with the SpMV
// BiCGSTAB needs phat = M^-1 p and v = A phat. With M = LU in red-black
// order, the red rows of A M^-1 p equal p_r exactly (red rows of A are
// I_r + B_rb and z_r = p_r - B_rb z_b), so only the black rows of the
// product are formed:  v_r = p_r,  v_b = z_b + B_br z_r.
// Three passes read each colour's blocks 1.5x instead of 2x+1x.

template <int K>
__device__ __forceinline__ void block_reduce_store_at(double (&v)[K], double* partial,
                                                      int stride, int slot) {
  __shared__ double sh[K][32];
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sh[k][wid] = x;
  }
  __syncthreads();
  const int nwarps = (blockDim.x * blockDim.y) >> 5;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += sh[k][w];
      partial[(int64_t)k * stride + slot] = s;
    }
  }
}

// pass 2 (red rows): z_r = p_r - sum B_rd z_b, v_r = p_r, partial dots of v_r
// K == 1: v.w0 ; K == 2: (v.v, v.w1)
template <int K>
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_mc_red(Dims g, const double* __restrict__ offd,
                                                    const double* __restrict__ pin,
                                                    double* __restrict__ z, double* __restrict__ v,
                                                    const double* __restrict__ w0,
                                                    const double* __restrict__ w1,
                                                    double* partial, int stride) {
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = (int64_t)blockIdx.x * 32 + ls;   // t-th red cell (colour-blocked storage)
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  if (t < g.half) {
    const int64_t c = colour_pos(g, 0, t);
    int i, j, k;
    const int64_t cell = locate(g, c, i, j, k);
    const double pr = pin[r * n + c];
    double w = pr;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) t += blk[(int64_t)u * n] * z[(int64_t)u * n + nb];
      w -= t;
    }
    z[r * n + c] = w;
    v[r * n + c] = pr;
    if (K == 1) acc[0] = pr * w0[r * n + c];
    if (K == 2) { acc[0] = pr * pr; acc[K - 1] = pr * w1[r * n + c]; }
  }
  warp_store_at<K>(acc, partial, (int64_t)stride * NU, blockIdx.x);
}

// black rows of the product: v_b = z_b + sum B_bd z_r, partial dots of v_b
template <int K>
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_mc_black_spmv(Dims g, const double* __restrict__ offd,
                                                           const double* __restrict__ z,
                                                           double* __restrict__ v,
                                                           const double* __restrict__ w0,
                                                           const double* __restrict__ w1,
                                                           double* partial, int stride,
                                                           int slot0, const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;   // t-th black cell (owned)
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  if (t < g.tw_hi) {
    const int64_t c = colour_pos(g, 1, t);
    int i, j, k;
    const int64_t cell = locate(g, c, i, j, k);
    double s = z[r * n + c];
    // the dot operand is loaded up front, in flight with the block stream
    const double wdot = K == 1 ? w0[r * n + c] : (K == 2 ? w1[r * n + c] : 0.0);
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int64_t nb = nb_pos(g, cell, i, j, k, d);
      if (nb < 0) continue;
      const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) t += blk[(int64_t)u * n] * z[(int64_t)u * n + nb];
      s += t;
    }
    v[r * n + c] = s;
    if (owned_k(g, k)) {   // ghost planes (slabs) stay out of the sums
      if (K == 1) acc[0] = s * wdot;
      if (K == 2) { acc[0] = s * s; acc[K - 1] = s * wdot; }
    }
  }
  warp_store_at<K>(acc, partial, (int64_t)stride * NU, slot0 + blockIdx.x);
}

// ------------------------- red-eliminated (Schur complement) BiCGSTAB
// With the decoupled diagonal blocks equal to I, red-black ordering gives
//   [ I     B_rb ] [x_r]   [b_r]        S x_b = g_b,  S = I - B_br B_rb,
//   [ B_br  I    ] [x_b] = [b_b]   <=>  g_b = b_b - B_br b_r,
//                                        x_r = b_r - B_rb x_b.
// The multicolour block-ILU(0) M = LU (U_b = I - blockdiag(B_br B_rb)) acts
// on this system as block-Jacobi with U_b: A M^-1 = L diag(I, S U_b^-1) L^-1,
// so right-preconditioned BiCGSTAB on (S, U_b) is BiCGSTAB with the same
// preconditioner with the red residual eliminated exactly. Its residual
// equals the full system's (red rows vanish identically), so the reference's
// stopping test ||r|| / ||b|| is unchanged. One product z_b = U_b^-1 p_b,
// w_r = -B_rb z_b, v_b = z_b + B_br w_r reads each off-diagonal block once
// (the full-system fused product reads the black ones twice), and every
// Krylov vector lives on the black half only.

// red pass: z_r = -sum_d B_rd z_b(nb)  (z holds z_b at black positions)
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_sc_red(Dims g, const double* __restrict__ offd,
                                                              double* __restrict__ z,
                                                              const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;   // owned planes only
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 0, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double w = 0.0;
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) tt += blk[(int64_t)u * n] * z[(int64_t)u * n + nb];
    w -= tt;
  }
  z[r * n + c] = w;
}

// red pass of the back-substitution: x_r = b_r - sum_d B_rd x_b(nb)
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_sc_xred(Dims g, const double* __restrict__ offd,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ x) {
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;   // owned planes only
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 0, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double w = b[r * n + c];
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) tt += blk[(int64_t)u * n] * x[(int64_t)u * n + nb];
    w -= tt;
  }
  x[r * n + c] = w;
}

// reduced right-hand side: g_b = b_b - sum_d B_bd b_r(nb), written to r and
// rhat (black positions); partial g.g
__global__ void __launch_bounds__(32 * NU, MC_MINB) k_sc_rhs(Dims g, const double* __restrict__ offd,
                                                              const double* __restrict__ b,
                                                              double* __restrict__ r_,
                                                              double* __restrict__ rhat) {
  const int64_t n = g.n;
  const int ls = threadIdx.x, r = threadIdx.y;
  const int64_t t = g.tw_lo + (int64_t)blockIdx.x * 32 + ls;   // owned planes only
  if (t >= g.tw_hi) return;
  const int64_t c = colour_pos(g, 1, t);
  int i, j, k;
  const int64_t cell = locate(g, c, i, j, k);
  double w = b[r * n + c];
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(g, cell, i, j, k, d);
    if (nb < 0) continue;
    const double* blk = offd + (int64_t)((d * NU + r) * NU) * n + c;
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) tt += blk[(int64_t)u * n] * b[(int64_t)u * n + nb];
    w -= tt;
  }
  r_[r * n + c] = w;
  rhat[r * n + c] = w;
}

// black-half vector kernels: thread per black cell (all NC rows: 9, or 6 in
// the condensed form, compact.cu), fixed grid and block-order partial sums
// (deterministic)
#ifndef VEC_MINB
#define VEC_MINB 4   // caps the U_b^-1 products at 64 registers (255 unbounded)
#endif
#define SC_LOOP(t)                                                                            \
  for (int64_t t = g.tw_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.tw_hi;    \
       t += (int64_t)gridDim.x * blockDim.x)

// p_b = r_b (first) or r_b + beta (p_b - omega v_b); z_b = U_b^-1 p_b
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_update_p(Dims g, const double* __restrict__ r,
                                                             double* __restrict__ p,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ uinv,
                                                             double* __restrict__ z,
                                                             const double* __restrict__ sc,
                                                             const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const bool first = sc[S_FIRST] != 0.0;
  const double beta = (sc[S_RHO] / sc[S_RHO_OLD]) * (sc[S_ALPHA] / sc[S_OMEGA]);
  const double omega = sc[S_OMEGA];
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) {   // ghost plane (slabs): filled by the halo exchange
#pragma unroll
      for (int q = 0; q < NC; ++q) { p[q * n + c] = 0.0; z[q * n + c] = 0.0; }
      continue;
    }
    double pv[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t i = q * n + c;
      pv[q] = first ? r[i] : r[i] + beta * (p[i] - omega * v[i]);
      p[i] = pv[q];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double zz = 0.0;
#pragma unroll
      for (int u = 0; u < NC; ++u) zz += uinv[(int64_t)(q * NC + u) * n + c] * pv[u];
      z[q * n + c] = zz;
    }
  }
}

// alpha = rho/den; s_b = r_b - alpha v_b; partial s.s; shat_b = U_b^-1 s_b
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_update_s(Dims g, const double* __restrict__ r,
                                                             const double* __restrict__ v,
                                                             double* __restrict__ s,
                                                             const double* __restrict__ uinv,
                                                             double* __restrict__ sh,
                                                             const double* __restrict__ sc,
                                                             double* partial, const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const double alpha = sc[S_RHO] / sc[S_DEN];
  double acc[1] = {0.0};
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) {   // ghost plane (slabs): filled by the halo exchange
#pragma unroll
      for (int q = 0; q < NC; ++q) { s[q * n + c] = 0.0; sh[q * n + c] = 0.0; }
      continue;
    }
    const bool own = true;
    double sv[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t i = q * n + c;
      sv[q] = r[i] - alpha * v[i];
      s[i] = sv[q];
      if (own) acc[0] += sv[q] * sv[q];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double zz = 0.0;
#pragma unroll
      for (int u = 0; u < NC; ++u) zz += uinv[(int64_t)(q * NC + u) * n + c] * sv[u];
      sh[q * n + c] = zz;
    }
  }
  block_reduce_store<1>(acc, partial);
}

// omega = ts/tt; x_b += alpha phat_b + omega shat_b; r_b = s_b - omega t_b;
// partial r.r, rhat.r
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_update_xr(Dims g, double* __restrict__ x,
                                                              const double* __restrict__ ph,
                                                              const double* __restrict__ sh_,
                                                              double* __restrict__ r,
                                                              const double* __restrict__ s,
                                                              const double* __restrict__ t_,
                                                              const double* __restrict__ rhat,
                                                              const double* sc, double* partial,
                                                              const double* stop) {
  if (stopped(stop)) return;
  const int64_t n = g.n;
  const double tt = sc[S_TT];
  double acc[2] = {0.0, 0.0};
  if (tt != 0.0) {
    const double alpha = sc[S_ALPHA];
    const double omega = sc[S_TS] / tt;
    SC_LOOP(t) {
      const int64_t c = colour_pos(g, 1, t);
      const bool own = owned_k(g, plane_of(g, c));
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const int64_t i = q * n + c;
        x[i] += alpha * ph[i] + omega * sh_[i];
        const double ri = s[i] - omega * t_[i];
        r[i] = ri;
        if (own) {
          acc[0] += ri * ri;
          acc[1] += rhat[i] * ri;
        }
      }
    }
  }
  block_reduce_store<2>(acc, partial);
}

// Device-driven BiCGSTAB control (one thread each): the scalar logic of
// linsolve.py:500-575 evaluated in HBM between the vector kernels, so a
// chunk of iterations runs without a host round trip. Any exit -- a
// breakdown test, the tolerance, the iteration limit -- only sets S_STOP;
// the host reads it after the chunk and runs the branch (restart, Breakdown,
// MaxIterations, final update) exactly as the host-driven loop does.
__global__ void k_bicg_init(double* sc) {    // ||b||, breakdown threshold 1e-30 ||b||^2
  const double nb = sqrt(sc[S_BB]);
  sc[S_NB] = nb;
  sc[S_BRK] = 1e-30 * nb * nb;
  if (nb == 0.0) sc[S_STOP] = STOP_ZERO;
}
__global__ void k_bicg_top(double* sc) {     // loop head: it += 1; rho / omega tests
  if (sc[S_STOP] != 0.0) return;
  if (sc[S_IT] >= sc[S_MAXIT]) { sc[S_STOP] = STOP_MAXIT; return; }
  sc[S_IT] += 1.0;
  const double rho = sc[S_RHO_NEW];
  if (fabs(rho) < sc[S_BRK] || (sc[S_FIRST] == 0.0 && sc[S_OMEGA] == 0.0)) {
    sc[S_STOP] = STOP_TOP;
    return;
  }
  sc[S_RHO] = rho;
}
__global__ void k_bicg_den(double* sc) { bicg_den(sc); }
__global__ void k_bicg_ss(double* sc) { bicg_ss(sc); }
__global__ void k_bicg_end(double* sc) { bicg_end(sc); }

// black-half helpers: x_b += alpha phat_b;  out_b = a_b - b_b;  dot over black rows
template <int NC>
__global__ void k_sc_axpy_alpha(Dims g, double* __restrict__ x, const double* __restrict__ ph,
                                const double* __restrict__ sc) {
  const int64_t n = g.n;
  const double alpha = sc[S_ALPHA];
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
#pragma unroll
    for (int q = 0; q < NC; ++q) x[q * n + c] += alpha * ph[q * n + c];
  }
}

template <int NC>
__global__ void k_sc_sub(Dims g, const double* __restrict__ a, const double* __restrict__ b,
                         double* __restrict__ out, double* __restrict__ out2) {
  const int64_t n = g.n;
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const double v = a[q * n + c] - b[q * n + c];
      out[q * n + c] = v;
      if (out2) out2[q * n + c] = v;
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_dot(Dims g, const double* __restrict__ a,
                                                        const double* __restrict__ b,
                                                        double* partial) {
  const int64_t n = g.n;
  double acc[1] = {0.0};
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) continue;
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[0] += a[q * n + c] * b[q * n + c];
  }
  block_reduce_store<1>(acc, partial);
}

// ------------------------------------------------ GMRES on the reduced system
// Right-preconditioned restarted GMRES on S x_b = g_b with U_b block-Jacobi
// (the north star's "BiCGSTAB/GMRES"): Arnoldi with classical Gram-Schmidt
// and one reorthogonalisation (CGS2). Vectors are black-half, full-length
// storage (9n, black positions used), the basis V packed with stride vs.
constexpr int GM_MAXV = 32;   // basis vectors held (restart length GM_MAXV - 1)

// z_b = U_b^-1 v_b
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_precond(Dims g,
                                                                      const double* __restrict__ v,
                                                                      const double* __restrict__ uinv,
                                                                      double* __restrict__ z) {
  const int64_t n = g.n;
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) {   // ghost plane (slabs): filled by the halo exchange
#pragma unroll
      for (int q = 0; q < NC; ++q) z[q * n + c] = 0.0;
      continue;
    }
    double pv[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) pv[q] = v[q * n + c];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double zz = 0.0;
#pragma unroll
      for (int u = 0; u < NC; ++u) zz += uinv[(int64_t)(q * NC + u) * n + c] * pv[u];
      z[q * n + c] = zz;
    }
  }
}

// per-block partials of h_i = V_i . w (i < nv) and, when w2 == nullptr, of
// w . w in slot nv; partial[i * gridDim.x + block] (fixed order, owned rows)
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, 2) k_sc_multidot(Dims g, const double* __restrict__ V,
                                                                int64_t vs, int nv,
                                                                const double* __restrict__ w,
                                                                double* partial) {
  const int64_t n = g.n;
  double acc[GM_MAXV + 1];
#pragma unroll
  for (int i = 0; i <= GM_MAXV; ++i) acc[i] = 0.0;
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) continue;
#pragma unroll 1
    for (int q = 0; q < NC; ++q) {
      const double wq = w[q * n + c];
#pragma unroll
      for (int i = 0; i < GM_MAXV; ++i)
        if (i < nv) acc[i] += V[(int64_t)i * vs + q * n + c] * wq;
      acc[GM_MAXV] += wq * wq;
    }
  }
  __shared__ double sh[GM_MAXV + 1][RED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i <= GM_MAXV; ++i) {
    double x = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sh[i][wid] = x;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= GM_MAXV; i += blockDim.x) {
    double x = 0.0;
    for (int k = 0; k < RED_THREADS / 32; ++k) x += sh[i][k];
    partial[(int64_t)i * gridDim.x + blockIdx.x] = x;
  }
}

// out[i] = sum_b partial[i * nparts + b] in fixed order (i < nout); one warp per value
__global__ void k_sum_partials(const double* __restrict__ partial, int nparts, int nout,
                               double* out) {
  const int i = blockIdx.x;
  if (i >= nout) return;
  double x = 0.0;
  for (int b = threadIdx.x; b < nparts; b += 32) x += partial[(int64_t)i * nparts + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  if (threadIdx.x == 0) out[i] = x;
}

// w = (zero ? 0 : w) - sum_{i<nv} h_i V_i over owned black rows; partial w.w
// (when partial != nullptr)
template <int NC>
__global__ void __launch_bounds__(RED_THREADS, VEC_MINB) k_sc_multiaxpy(Dims g, const double* __restrict__ V,
                                                                        int64_t vs, int nv,
                                                                        const double* __restrict__ h,
                                                                        double hsign,
                                                                        double* __restrict__ w,
                                                                        int zero, double* partial) {
  const int64_t n = g.n;
  __shared__ double hs[GM_MAXV];
  for (int i = threadIdx.x; i < GM_MAXV; i += blockDim.x) hs[i] = i < nv ? hsign * h[i] : 0.0;
  __syncthreads();
  double acc[1] = {0.0};
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
    if (!owned_k(g, plane_of(g, c))) {
#pragma unroll
      for (int q = 0; q < NC; ++q) w[q * n + c] = 0.0;
      continue;
    }
#pragma unroll 1
    for (int q = 0; q < NC; ++q) {
      double x = zero ? 0.0 : w[q * n + c];
      for (int i = 0; i < nv; ++i) x -= hs[i] * V[(int64_t)i * vs + q * n + c];
      w[q * n + c] = x;
      acc[0] += x * x;
    }
  }
  if (partial) block_reduce_store<1>(acc, partial);
}

// out = w / sqrt(nn[0]) (owned black rows)
template <int NC>
__global__ void k_sc_scale(Dims g, const double* __restrict__ w, const double* __restrict__ nn,
                           double* __restrict__ out) {
  const int64_t n = g.n;
  const double inv = 1.0 / sqrt(nn[0]);
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
#pragma unroll
    for (int q = 0; q < NC; ++q) out[q * n + c] = w[q * n + c] * inv;
  }
}

// x_b += z_b
template <int NC>
__global__ void k_sc_add(Dims g, const double* __restrict__ z, double* __restrict__ x) {
  const int64_t n = g.n;
  SC_LOOP(t) {
    const int64_t c = colour_pos(g, 1, t);
#pragma unroll
    for (int q = 0; q < NC; ++q) x[q * n + c] += z[q * n + c];
  }
}

}  // namespace isc
