// Shared definitions for the sm_100a Newton hot path (fp64 throughout).
//
// Per-cell unknown (column) order and residual (row) order follow the
// reference (_kernels.py:11-16):
//   columns  p, x_0..x_{nco-1}, y_0..y_{ncg-1}, T, S_w, S_g, C_c
//   rows     F_W, F_O[..], F_G[..], F_E, F_OS, F_GS, F_Coke
// The library is compiled for the reference's benchmark fluid
// (nco = 2 oils, ncg = 2 gases, block size 9); other compositions are
// rejected at context creation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace isc {

constexpr int NCO = 2;
constexpr int NCG = 2;
constexpr int NF = 1 + NCO + NCG;   // full gas composition entries
constexpr int NU = NCO + NCG + 5;   // block size (9)
constexpr int CT = 1 + NCO + NCG;   // T column / energy row
constexpr int CSW = CT + 1, CSG = CT + 2, CCC = CT + 3;
constexpr int ROW_E = CT, ROW_OS = CT + 1, ROW_GS = CT + 2, ROW_CK = CT + 3;
constexpr int NB = NU * NU;         // 81 entries per block
constexpr int NDIR = 6;             // -z, -y, -x, +x, +y, +z
constexpr int MAXREAC = 4;
constexpr int MAXTAB = 32;

constexpr double RANKINE = 459.67;
constexpr double R_GAS = 10.7316;
constexpr double R_ARR = 1.9859;
constexpr double PSI_PER_FT = 1.0 / 144.0;

// Flattened model constants, passed by value as a kernel parameter (lands in
// the constant bank; every thread reads the same words).  Layout mirrors the
// reference ModelPack tables (assembly.py:42-68, _kernels.py:48-63).
struct Model {
  double liq[1 + NCO][10];
  double gasp[NF][9];
  double kv[1 + NCO][5];
  double rockp[17];
  double swt_s[MAXTAB], swt_krw[MAXTAB], swt_krow[MAXTAB], swt_pcow[MAXTAB];
  double slt_s[MAXTAB], slt_krg[MAXTAB], slt_krog[MAXTAB], slt_pcog[MAXTAB];
  double rcoef[MAXREAC][3];
  double nmat[NF + 1][MAXREAC];
  int law[MAXREAC], fuel[MAXREAC], ox[MAXREAC];
  int nreac, nswt, nslt, heavy;
  double ccmax;
};

enum { L_RHO = 0, L_CP, L_CT1, L_CT2, L_CPT, L_AVISC, L_BVISC, L_HVR, L_EV, L_TCF };
enum { G_M = 0, G_TCR, G_PC, G_AVG, G_BVG, G_CPG1, G_CPG2, G_CPG3, G_CPG4 };
enum {
  RK_CPOR = 0, RK_CTPOR, RK_CPTPOR, RK_MODE, RK_CP1, RK_CP2, RK_COKE_CP, RK_RHO_COKE,
  RK_KTW, RK_KTO, RK_KTG, RK_KTR, RK_KTC, RK_PREF, RK_TREF, RK_EPS_PER, RK_KROCW
};

// Structured grid geometry (x fastest: c = i + nx*(j + ny*k)).
//
// Storage order of every per-cell array in HBM ("position" p): when nx is
// even the cells are colour-blocked plane by plane: plane k occupies
// positions [k*nxny, (k+1)*nxny), its red cells (i+j+k even) first, then
// its black cells, each in natural order:
//   p = k*nxny + colour*ph + (q >> 1),   q = in-plane index, ph = nxny/2
//     = (c >> 1) + ph*(k + colour).
// Each colour's rows of a plane are contiguous, so the multicolour ILU
// passes and any single-colour sweep stream full 32 B sectors, while the
// working set of a sweep stays within three neighbouring planes (a
// whole-array red/black split streams 11 % slower on B200: tools/
// layout_probe.cu). Neighbours of a cell all have the other colour, so their
// positions follow from (c ± stride) >> 1. With odd nx the natural order is
// used (colored = 0).
struct Dims {
  int nx, ny, nz;
  int64_t n;       // nx*ny*nz
  int64_t nxny;
  int colored;     // 1: colour-blocked storage
  int64_t half;    // n/2 (cells of each colour) when colored
  int64_t ph;      // nxny/2 (cells of each colour in one plane) when colored
  int kpar;        // parity of the global index of local plane 0 (z-slabs)
  // z-slab decomposition (multi-GPU): this context holds planes [0, nz) of
  // which [kw_lo, kw_hi) are owned; the rest are one-plane ghost copies of
  // the neighbouring ranks' cells. Single GPU: kw_lo = 0, kw_hi = nz.
  int kw_lo, kw_hi;
  // owned range of the per-colour index t (colour-blocked storage: planes
  // [kw_lo, kw_hi) hold t in [kw_lo*ph, kw_hi*ph)); single GPU: [0, half)
  int64_t tw_lo, tw_hi;
};

__host__ __device__ __forceinline__ bool owned_k(const Dims& g, int k) {
  return k >= g.kw_lo && k < g.kw_hi;
}

__host__ __device__ __forceinline__ void cell_ijk(const Dims& g, int64_t c, int& i, int& j,
                                                  int& k) {
  if (g.n < (int64_t)0x7fffffff) {
    const uint32_t cc = (uint32_t)c, nx = (uint32_t)g.nx, nxny = (uint32_t)g.nxny;
    const uint32_t kk = cc / nxny, rem = cc - kk * nxny;
    k = (int)kk;
    j = (int)(rem / nx);
    i = (int)(rem - (uint32_t)j * nx);
  } else {
    k = (int)(c / g.nxny);
    const int64_t rem = c - (int64_t)k * g.nxny;
    j = (int)(rem / g.nx);
    i = (int)(rem - (int64_t)j * g.nx);
  }
}

__host__ __device__ __forceinline__ int64_t pos_of(const Dims& g, int64_t c) {
  if (!g.colored) return c;
  int i, j, k;
  cell_ijk(g, c, i, j, k);
  return (c >> 1) + g.ph * (int64_t)(k + ((i + j + k + g.kpar) & 1));
}

// cell index and (i, j, k) of storage position p (one decomposition)
__host__ __device__ __forceinline__ int64_t locate(const Dims& g, int64_t p, int& i, int& j,
                                                   int& k) {
  if (!g.colored) {
    cell_ijk(g, p, i, j, k);
    return p;
  }
  int64_t rem;
  if (g.n < (int64_t)0x7fffffff) {
    const uint32_t kk = (uint32_t)p / (uint32_t)g.nxny;
    k = (int)kk;
    rem = (uint32_t)p - kk * (uint32_t)g.nxny;
  } else {
    k = (int)(p / g.nxny);
    rem = p - (int64_t)k * g.nxny;
  }
  const int col = rem >= g.ph ? 1 : 0;
  const uint32_t q0 = 2u * (uint32_t)(rem - col * g.ph);
  j = (int)(q0 / (uint32_t)g.nx);
  i = (int)(q0 - (uint32_t)j * (uint32_t)g.nx);
  i += (((i + j + k + g.kpar) & 1) != col) ? 1 : 0;
  return (int64_t)k * g.nxny + (int64_t)j * g.nx + i;
}

__host__ __device__ __forceinline__ int64_t cell_of(const Dims& g, int64_t p) {
  int i, j, k;
  return locate(g, p, i, j, k);
}

// z-plane of storage position p (planes are contiguous in both orders)
__host__ __device__ __forceinline__ int plane_of(const Dims& g, int64_t p) {
  if (g.n < (int64_t)0x7fffffff) return (int)((uint32_t)p / (uint32_t)g.nxny);
  return (int)(p / g.nxny);
}

// storage position of the t-th cell of colour col (0 <= t < half)
__host__ __device__ __forceinline__ int64_t colour_pos(const Dims& g, int col, int64_t t) {
  int64_t kk;
  if (g.n < (int64_t)0x7fffffff) kk = (uint32_t)t / (uint32_t)g.ph;
  else kk = t / g.ph;
  return kk * g.nxny + (int64_t)col * g.ph + (t - kk * g.ph);
}

// Direction d of a neighbour, in the reference's gather order
// (ascending connection index seen from a cell, _kernels.py:828-854).
enum { DZM = 0, DYM = 1, DXM = 2, DXP = 3, DYP = 4, DZP = 5 };

__host__ __device__ inline int opposite(int d) { return 5 - d; }
__device__ __forceinline__ int64_t neighbour(const Dims& g, int64_t c, int i, int j, int k, int d);

// storage position of the neighbour of cell c (at position p) in direction
// d, or -1 at the boundary
__device__ __forceinline__ int64_t nb_pos(const Dims& g, int64_t c, int i, int j, int k, int d) {
  const int64_t nb = neighbour(g, c, i, j, k, d);
  if (nb < 0 || !g.colored) return nb;
  const int kn = k + (d == DZM ? -1 : (d == DZP ? 1 : 0));
  return (nb >> 1) + g.ph * (int64_t)(kn + (((i + j + k + g.kpar) & 1) ^ 1));
}

// neighbour of cell c in direction d, or -1 at the boundary
__device__ __forceinline__ int64_t neighbour(const Dims& g, int64_t c, int i, int j, int k, int d) {
  switch (d) {
    case DZM: return k > 0 ? c - g.nxny : -1;
    case DYM: return j > 0 ? c - g.nx : -1;
    case DXM: return i > 0 ? c - 1 : -1;
    case DXP: return i + 1 < g.nx ? c + 1 : -1;
    case DYP: return j + 1 < g.ny ? c + g.nx : -1;
    default:  return k + 1 < g.nz ? c + g.nxny : -1;
  }
}

}  // namespace isc
