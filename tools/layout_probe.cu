// Probe: SpMV bandwidth with the strided SoA offd layout vs a 32-cell tiled
// layout (all 486 coefficients of a 32-cell tile contiguous).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NU = 9;
struct G { int nx, ny, nz; int64_t n, nxny; };
__device__ __forceinline__ int64_t nbr(const G& g, int64_t c, int i, int j, int k, int d) {
  switch (d) {
    case 0: return k > 0 ? c - g.nxny : -1;
    case 1: return j > 0 ? c - g.nx : -1;
    case 2: return i > 0 ? c - 1 : -1;
    case 3: return i + 1 < g.nx ? c + 1 : -1;
    case 4: return j + 1 < g.ny ? c + g.nx : -1;
    default: return k + 1 < g.nz ? c + g.nxny : -1;
  }
}
// colour-blocked storage: p = colour*half + (c>>1)
template <int OWN>
__global__ void __launch_bounds__(288) spmv_col(G g, const double* __restrict__ offd,
                                            const double* __restrict__ x, double* __restrict__ y) {
  const int64_t n = g.n, half = n / 2;
  const int64_t p = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int r = threadIdx.y;
  if (p >= n) return;
  const int col = p >= half;
  const int64_t c0 = 2 * (p - col * half);
  uint32_t cc = (uint32_t)c0;
  int k = cc / (uint32_t)g.nxny; uint32_t rem = cc - k * (uint32_t)g.nxny;
  int j = rem / g.nx, i = rem - j * g.nx;
  int64_t c = c0;
  if (((i + j + k) & 1) != col) { c = c0 + 1; ++i; }
  if (OWN && (k < 1 || k >= g.nz - 1)) return;
  double s = x[r * n + p];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int64_t nb0 = nbr(g, c, i, j, k, d);
    if (nb0 < 0) continue;
    const int64_t nb = (int64_t)(col ^ 1) * half + (nb0 >> 1);
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int e = (d * NU + r) * NU + u;
      t += __ldg(offd + (int64_t)e * n + p) * __ldg(x + (int64_t)u * n + nb);
    }
    s += t;
  }
  y[r * n + p] = s;
}
template <int OWN>
double runc(G g, const double* offd, const double* x, double* y) {
  dim3 blk(32, 9); unsigned grid = (unsigned)((g.n + 31) / 32);
  for (int w = 0; w < 3; ++w) spmv_col<OWN><<<grid, blk>>>(g, offd, x, y);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int w = 0; w < 10; ++w) spmv_col<OWN><<<grid, blk>>>(g, offd, x, y);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}
// MODE 0: global colour blocking p = col*half + (c>>1)
// MODE 1: plane colour blocking p = k*nxny + col*nxny/2 + (q>>1)
// RED: 1 -> only red rows processed (one thread per red cell)
template <int MODE, int RED, int RDX = 0>
__global__ void __launch_bounds__(288) spmv_m(G g, const double* __restrict__ offd,
                                            const double* __restrict__ x, double* __restrict__ y,
                                            double* partial = nullptr) {
  __shared__ double shr[9];
  __shared__ unsigned cnt;
  if (RDX == 3) { if (threadIdx.x == 0 && threadIdx.y == 0) cnt = 0; __syncthreads(); }
  const int64_t n = g.n, half = n / 2, ph = g.nxny / 2;
  int64_t t = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int r = threadIdx.y;
  const bool inr = t < (RED ? half : n);
  if (!RDX && !inr) return;
  int64_t p = 0;
  double accd = 0.0;
  if (inr) {
  if (MODE == 0) p = t;
  else if (MODE == 2) { const int hr = g.nx / 2; p = RED ? (t / hr) * g.nx + (t % hr) : t; }
  else if (RED) { const int64_t kk = t / ph; p = kk * g.nxny + (t - kk * ph); }
  else p = t;
  int col, i, j, k; int64_t c;
  if (MODE == 0) {
    col = p >= half;
    const int64_t c0 = 2 * (p - col * half);
    uint32_t cc = (uint32_t)c0;
    k = cc / (uint32_t)g.nxny; uint32_t rem = cc - k * (uint32_t)g.nxny;
    j = rem / g.nx; i = rem - j * g.nx; c = c0;
    if (((i + j + k) & 1) != col) { c = c0 + 1; ++i; }
  } else if (MODE == 2) {
    const uint32_t row = (uint32_t)p / (uint32_t)g.nx, rr = (uint32_t)p - row * g.nx;
    k = row / g.ny; j = row - k * g.ny;
    col = rr >= (uint32_t)g.nx / 2; i = 2 * (rr - col * g.nx / 2);
    if (((i + j + k) & 1) != col) ++i;
    c = (int64_t)k * g.nxny + j * g.nx + i;
  } else {
    k = (uint32_t)p / (uint32_t)g.nxny; uint32_t rem = (uint32_t)p - k * (uint32_t)g.nxny;
    col = rem >= ph; const uint32_t q0 = 2 * (rem - col * ph);
    j = q0 / g.nx; i = q0 - j * g.nx;
    if (((i + j + k) & 1) != col) ++i;
    c = (int64_t)k * g.nxny + j * g.nx + i;
  }
  double s = x[r * n + p];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int64_t nb0 = nbr(g, c, i, j, k, d);
    if (nb0 < 0) continue;
    int64_t nb;
    if (MODE == 0) nb = (int64_t)(col ^ 1) * half + (nb0 >> 1);
    else if (MODE == 2) {
      const int64_t rown = nb0 / g.nx;
      nb = rown * g.nx + (col ^ 1) * (g.nx / 2) + ((nb0 - rown * g.nx) >> 1);
    } else {
      const int kn = d == 0 ? k - 1 : (d == 5 ? k + 1 : k);
      const int64_t qn = nb0 - (int64_t)kn * g.nxny;
      nb = (int64_t)kn * g.nxny + (col ^ 1) * ph + (qn >> 1);
    }
    double tt = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int e = (d * NU + r) * NU + u;
      tt += __ldg(offd + (int64_t)e * n + p) * __ldg(x + (int64_t)u * n + nb);
    }
    s += tt;
  }
  y[r * n + p] = s;
  accd = s * x[r * n + p + 1];
  }
  if (RDX == 1) {
    for (int o = 16; o > 0; o >>= 1) accd += __shfl_down_sync(0xffffffffu, accd, o);
    if (threadIdx.x == 0) shr[threadIdx.y] = accd;
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      double q = 0; for (int w = 0; w < 9; ++w) q += shr[w];
      partial[blockIdx.x] = q;
    }
  } else if (RDX == 3) {   // last warp of the block sums in fixed order
    for (int o = 16; o > 0; o >>= 1) accd += __shfl_down_sync(0xffffffffu, accd, o);
    if (threadIdx.x == 0) {
      shr[threadIdx.y] = accd;
      __threadfence_block();
      const unsigned done = atomicAdd(&cnt, 1u);
      if (done == 8) {
        __threadfence_block();
        double q = 0; for (int w = 0; w < 9; ++w) q += ((volatile double*)shr)[w];
        partial[blockIdx.x] = q;
      }
    }
  } else if (RDX == 2) {   // per-warp partials, no barrier
    for (int o = 16; o > 0; o >>= 1) accd += __shfl_down_sync(0xffffffffu, accd, o);
    if (threadIdx.x == 0) partial[blockIdx.x * 9 + threadIdx.y] = accd;
  }
}
template <int MODE, int RED, int RDX = 0>
double runm(G g, const double* offd, const double* x, double* y) {
  dim3 blk(32, 9); unsigned grid = (unsigned)(((RED ? g.n / 2 : g.n) + 31) / 32);
  static double* part = nullptr;
  if (!part) cudaMalloc(&part, sizeof(double) * 9 * (g.n / 32 + 1));
  for (int w = 0; w < 3; ++w) spmv_m<MODE, RED, RDX><<<grid, blk>>>(g, offd, x, y, part);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int w = 0; w < 10; ++w) spmv_m<MODE, RED, RDX><<<grid, blk>>>(g, offd, x, y, part);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}
template <int TILE>
__global__ void __launch_bounds__(288) spmv(G g, const double* __restrict__ offd,
                                            const double* __restrict__ x, double* __restrict__ y) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int r = threadIdx.y;
  if (c >= n) return;
  const uint32_t cc = (uint32_t)c;
  const int k = cc / (uint32_t)g.nxny; const uint32_t rem = cc - k * (uint32_t)g.nxny;
  const int j = rem / g.nx, i = rem - j * g.nx;
  double s = x[r * n + c];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int64_t nb = nbr(g, c, i, j, k, d);
    if (nb < 0) continue;
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int e = (d * NU + r) * NU + u;
      const double a = TILE == 0 ? __ldg(offd + (int64_t)e * n + c)
                                 : __ldg(offd + ((c / TILE) * 486 + e) * TILE + (c % TILE));
      t += a * __ldg(x + (int64_t)u * n + nb);
    }
    s += t;
  }
  y[r * n + c] = s;
}
template <int TILE>
double run(G g, const double* offd, const double* x, double* y) {
  dim3 blk(32, 9); unsigned grid = (unsigned)((g.n + 31) / 32);
  for (int w = 0; w < 3; ++w) spmv<TILE><<<grid, blk>>>(g, offd, x, y);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int w = 0; w < 10; ++w) spmv<TILE><<<grid, blk>>>(g, offd, x, y);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}
__global__ void fill(double* a, int64_t len, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    a[i] = (double)(z >> 11) * 0x1.0p-53 - 0.5;
  }
}
int main(int argc, char** argv) {
  G g{400, 400, 50, 0, 0};
  if (argc == 4) { g.nx = atoi(argv[1]); g.ny = atoi(argv[2]); g.nz = atoi(argv[3]); } g.nxny = (int64_t)g.nx * g.ny; g.n = g.nxny * g.nz;
  double *offd, *x, *y;
  cudaMalloc(&offd, sizeof(double) * 486 * g.n);
  cudaMalloc(&x, sizeof(double) * 9 * g.n); cudaMalloc(&y, sizeof(double) * 9 * g.n);
  cudaMemset(offd, 0, sizeof(double) * 486 * g.n); cudaMemset(x, 0, sizeof(double) * 9 * g.n);
  double z0 = run<0>(g, offd, x, y);
  printf("zeros strided %.3f ms\n", z0);
  fill<<<148 * 8, 256>>>(offd, 486 * g.n, 1); fill<<<148 * 8, 256>>>(x, 9 * g.n, 2);
  const int64_t m = 3 * g.n - g.nxny - g.nx * g.nz - g.ny * g.nz;
  const double bytes = 8.0 * (162.0 * m + 18.0 * g.n);
  double t0 = run<0>(g, offd, x, y), t1 = run<32>(g, offd, x, y), t2 = run<64>(g, offd, x, y);
  printf("strided %.3f ms %.0f GB/s\n", t0, bytes / t0 / 1e6);
  printf("tile32  %.3f ms %.0f GB/s\n", t1, bytes / t1 / 1e6);
  printf("tile64  %.3f ms %.0f GB/s\n", t2, bytes / t2 / 1e6);
  double t3 = runc<0>(g, offd, x, y);
  printf("colour  %.3f ms %.0f GB/s\n", t3, bytes / t3 / 1e6);
  double m00 = runm<0, 0>(g, offd, x, y), m10 = runm<1, 0>(g, offd, x, y);
  double m01 = runm<0, 1>(g, offd, x, y), m11 = runm<1, 1>(g, offd, x, y);
  printf("global-colour full %.3f ms %.0f GB/s\n", m00, bytes / m00 / 1e6);
  printf("plane-colour  full %.3f ms %.0f GB/s\n", m10, bytes / m10 / 1e6);
  printf("global-colour red  %.3f ms %.0f GB/s\n", m01, bytes / 2 / m01 / 1e6);
  printf("plane-colour  red  %.3f ms %.0f GB/s\n", m11, bytes / 2 / m11 / 1e6);
  double m20 = runm<2, 0>(g, offd, x, y), m21 = runm<2, 1>(g, offd, x, y);
  printf("row-colour    full %.3f ms %.0f GB/s\n", m20, bytes / m20 / 1e6);
  printf("row-colour    red  %.3f ms %.0f GB/s\n", m21, bytes / 2 / m21 / 1e6);
  double r1 = runm<1, 1, 1>(g, offd, x, y), r2 = runm<1, 1, 2>(g, offd, x, y);
  printf("plane red + block-reduce %.3f ms %.0f GB/s\n", r1, bytes / 2 / r1 / 1e6);
  printf("plane red + warp-partial %.3f ms %.0f GB/s\n", r2, bytes / 2 / r2 / 1e6);
  double r3 = runm<1, 1, 3>(g, offd, x, y);
  printf("plane red + last-warp    %.3f ms %.0f GB/s\n", r3, bytes / 2 / r3 / 1e6);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
