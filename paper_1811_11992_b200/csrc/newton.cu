// Device-resident Newton bookkeeping: damped update, scaled residual norm,
// conservation audit sums, and the synthetic microbench generator.
#include "common.cuh"

namespace isc {

// numpy's maximum / minimum propagate NaN from either operand; CUDA's fmax /
// fmin return the other operand instead, so NaN-carrying updates would turn
// into finite states and hide divergence from the norm check
__device__ __forceinline__ double np_maximum(double a, double b) {
  return (a != a || b != b) ? a + b : fmax(a, b);
}
__device__ __forceinline__ double np_minimum(double a, double b) {
  return (a != a || b != b) ? a + b : fmin(a, b);
}

// newton.py:80-89 (_damp_array), one element; comparisons with NaN are
// false, so a NaN raw value passes through as in numpy
__device__ __forceinline__ double damp(double old, double raw, double eps) {
  if (raw < 0.0) return sqrt(eps * np_maximum(old, 0.0));
  if (raw < eps && old >= eps) return 0.5 * old;
  return raw;
}

// np.clip(v, lo, hi) == minimum(maximum(v, lo), hi), NaN-propagating
__device__ __forceinline__ double clip(double v, double lo, double hi) {
  return np_minimum(np_maximum(v, lo), hi);
}

// newton.py:92-121; state and du SoA in unknown order
__global__ void k_newton_update(int64_t n, double* __restrict__ st, const double* __restrict__ du,
                                double eps) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  st[c] = st[c] + du[c];
#pragma unroll
  for (int i = 1; i < CT; ++i) st[i * n + c] = clip(st[i * n + c] + du[i * n + c], 0.0, 1.0);
  st[CT * n + c] = np_maximum(st[CT * n + c] + du[CT * n + c], -459.0);
  st[CCC * n + c] = np_maximum(st[CCC * n + c] + du[CCC * n + c], 0.0);
  const double sw0 = st[CSW * n + c], sg0 = st[CSG * n + c];
  const double so_old = 1.0 - sw0 - sg0;
  const double sw = damp(sw0, sw0 + du[CSW * n + c], eps);
  double sg = damp(sg0, sg0 + du[CSG * n + c], eps);
  const double so = damp(so_old, 1.0 - sw - sg, eps);
  sg = 1.0 - sw - so;
  if (sg < 0.0) sg = damp(sg0, sg, eps);
  const double swc = clip(sw, 0.0, 1.0);
  st[CSW * n + c] = swc;
  st[CSG * n + c] = clip(sg, 0.0, 1.0 - swc);
}

// partial maxima of |resid| / scale (newton.py:124-144), mass/energy/coke rows
// scaled by (V/dt) max(1, |accn|), constraint rows by 1
__global__ void __launch_bounds__(256) k_norm_partial(Dims g, const double* __restrict__ resid,
                                                      const double* __restrict__ accn,
                                                      const double* __restrict__ vol, double dt,
                                                      double* partial) {
  const int64_t n = g.n;
  double m = 0.0;
  bool nan = false;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (g.kw_lo > 0 || g.kw_hi < g.nz) {
      if (!owned_k(g, plane_of(g, c))) continue;
    }
    const double vdt = vol[c] / dt;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      const double sc = (r == ROW_OS || r == ROW_GS) ? 1.0 : vdt * fmax(1.0, fabs(accn[r * n + c]));
      const double v = fabs(resid[r * n + c]) / sc;
      if (v != v) nan = true;
      m = fmax(m, v);
    }
  }
  if (nan) m = __longlong_as_double(0x7ff8000000000000ULL);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_down_sync(0xffffffffu, m, o);
    m = (other != other || m != m) ? __longlong_as_double(0x7ff8000000000000ULL) : fmax(m, other);
  }
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = sh[0];
    for (int w = 1; w < 8; ++w) r = (sh[w] != sh[w] || r != r) ? sh[w] + r : fmax(r, sh[w]);
    partial[blockIdx.x] = r;
  }
}

// audit sums per row r in rows[]: sum V(acc-accn), sum V src, sum V|acc|
// (newton.py:339-366); rows = 0..NF-1 and the coke row
__global__ void __launch_bounds__(256) k_audit_partial(Dims g, const double* __restrict__ acc,
                                                       const double* __restrict__ accn,
                                                       const double* __restrict__ src,
                                                       const double* __restrict__ vol,
                                                       double* partial) {
  const int64_t n = g.n;
  constexpr int NR = NF + 1;
  double s[3 * NR];
#pragma unroll
  for (int k = 0; k < 3 * NR; ++k) s[k] = 0.0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (g.kw_lo > 0 || g.kw_hi < g.nz) {
      if (!owned_k(g, plane_of(g, c))) continue;
    }
    const double v = vol[c];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int r = k < NF ? k : ROW_CK;
      const double a = acc[r * n + c];
      s[k] += v * (a - accn[r * n + c]);
      s[NR + k] += v * src[r * n + c];
      s[2 * NR + k] += v * fabs(a);
    }
  }
  __shared__ double sh[3 * NR][8];
#pragma unroll
  for (int k = 0; k < 3 * NR; ++k) {
    double x = s[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 3 * NR; ++k) {
      double x = 0.0;
      for (int w = 0; w < 8; ++w) x += sh[k][w];
      partial[(int64_t)k * gridDim.x + blockIdx.x] = x;
    }
  }
}

// ------------------------------------------------ synthetic microbench
// Device twin of paper_1811_11992_b200/synth.py (counter-based generator).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double u01(uint64_t seed, uint64_t key) {
  const uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ULL + key);
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double snormal(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t key = (stream << 40) + idx * 2ULL;
  const double a = u01(seed, key), b = u01(seed, key + 1ULL);
  return sqrt(-2.0 * log(a)) * cos(6.283185307179586 * b);
}

// On a z-slab (k_offset > 0 or nz < nz_global) every value is keyed by the
// cell's GLOBAL index and the z-faces by the global grid's boundary, so each
// rank generates exactly its rows of the single-GPU system.
__global__ void k_synth(Dims g, uint64_t seed, int k_offset, int nz_global, double* diag,
                        double* offd, double* resid) {
  const int64_t n = g.n;
  const int64_t cl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // local natural cell
  if (cl >= n) return;
  const int64_t c = cl + (int64_t)k_offset * g.nxny;                   // global cell (RNG key)
  const int64_t pc = pos_of(g, cl);
  double dmag[NU];
#pragma unroll
  for (int r = 0; r < NU; ++r) {
    double v[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = snormal(seed, 0, (uint64_t)(c * NB + r * NU + u));
    // numpy pairwise row sum of 9 |entries| (8-way unrolled block + tail)
    const double rs = ((fabs(v[0]) + fabs(v[1])) + (fabs(v[2]) + fabs(v[3]))) +
                      ((fabs(v[4]) + fabs(v[5])) + (fabs(v[6]) + fabs(v[7]))) + fabs(v[8]);
    v[r] = rs + 1.0;
    dmag[r] = fabs(v[r]);
#pragma unroll
    for (int u = 0; u < NU; ++u) diag[(int64_t)(r * NU + u) * n + pc] = v[u];
    resid[(int64_t)r * n + pc] = snormal(seed, 2, (uint64_t)(c * NU + r));
  }
  int i, j, k;
  cell_ijk(g, cl, i, j, k);
  const int kg = k + k_offset;
  for (int d = 0; d < NDIR; ++d) {
    const bool has = d == DZM ? kg > 0
                   : d == DZP ? kg + 1 < nz_global
                              : neighbour(g, cl, i, j, k, d) >= 0;
#pragma unroll
    for (int r = 0; r < NU; ++r)
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const double v = has ? 0.1 * snormal(seed, 1, (uint64_t)((c * NDIR + d) * NB + r * NU + u)) * dmag[r]
                             : 0.0;
        offd[(int64_t)((d * NU + r) * NU + u) * n + pc] = v;
      }
  }
}

}  // namespace isc
