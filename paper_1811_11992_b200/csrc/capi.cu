// C-ABI (include/iscgpu.h) and the host-side runtime: context/buffer
// ownership, subdomain/level structure of the ILU(0) preconditioner, and the
// BiCGSTAB control flow of the reference (linsolve.py:481-578) driving the
// device kernels. Single translation unit: the kernel files are included.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/iscgpu.h"
#include "assemble.cu"
#include "decouple.cu"
#include "fused.cu"
#include "comm.cuh"
#include "newton.cu"
#include "numjac.cu"
#include "report.cuh"
#include "solver.cu"
#include "compact.cu"

#ifndef FACE_SPLIT
#define FACE_SPLIT 1   // k_face_eval as light rows + energy row kernels
#endif
#ifndef CELL_SPLIT
#define CELL_SPLIT 1   // cell pass as k_cell_props + k_cell_rows
#endif

#ifndef MC_SCHUR
#define MC_SCHUR 1   // mcilu on the red-eliminated system (0: full-system fused form)
#endif

using namespace isc;

static thread_local std::string g_err;

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      return ISC_CUDA_ERROR;                                                        \
    }                                                                               \
  } while (0)

#define LAUNCH_CHECK()                                                              \
  do {                                                                              \
    ++ctx->launches;                                                                \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) {                                                        \
      g_err = std::string("kernel launch: ") + cudaGetErrorString(e_);             \
      return ISC_CUDA_ERROR;                                                        \
    }                                                                               \
  } while (0)

struct isc_ctx {
  Dims g{};
  Model M{};
  int k_offset = 0;                        // global index of local plane 0 (z-slabs)
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t cstream = nullptr;          // host->device staging copies (isc_assemble_host)
  cudaEvent_t chunk_ev[8] = {};
  cudaEvent_t halo_ev[2] = {};             // halo planes packed / landed
  bool cell_pre = false;                   // k_cell already ran (pipelined host staging)
  bool face_pre = false;                   // k_face_eval too
  bool mc_schur = true;   // mcilu: red-eliminated BiCGSTAB (ISC_MCILU_FULL=1: full system)
  int krylov = ISC_KRYLOV_BICGSTAB;   // mcilu red-eliminated system: BiCGSTAB or GMRES(m)
  int gm_m = 30;                      // GMRES restart length (<= GM_MAXV - 1)
  int bicg_last_iters = 0;            // previous red-eliminated BiCGSTAB count (chunk size)
  double* gm_V = nullptr;             // GMRES basis, gm_m + 1 full-length vectors (lazy)
  double* gm_h = nullptr;             // GMRES device scalars: h (2 x GM_MAXV+1), y
  int64_t launches = 0;
  // static grid data
  double *depth = nullptr, *vol = nullptr, *phi_ref = nullptr, *gd = nullptr, *td = nullptr,
         *hl_area = nullptr;
  double hl_kob = 0, hl_d = 1, hl_rho = 0, hl_tini = 0;
  int64_t* conn_id = nullptr;
  // wells
  int nw = 0;
  WellDev* wells_d = nullptr;
  int64_t* wcell_d = nullptr;
  std::vector<int64_t> wcell_h;   // natural cell of each well
  std::vector<int64_t> wpos_h;    // its storage position
  double *st_c = nullptr, *accn_c = nullptr;   // state / accn in storage order
  double* stage = nullptr;                      // host-layout staging (18 n doubles)
  double* wout_d = nullptr;
  double* wout_h = nullptr;   // pinned
  double* bhp_d = nullptr;
  uint8_t* capped_d = nullptr;
  // assembly buffers
  double *rec = nullptr, *acc = nullptr, *src = nullptr, *resid = nullptr, *diag = nullptr,
         *offd = nullptr;
  int8_t* upw = nullptr;
  unsigned long long* bad_d = nullptr;
  unsigned long long* bad_h = nullptr;   // pinned
  // solver
  int precond = ISC_PRECOND_RAS;
  bool decoupled = false, factored = false;
  int offd_rows = NU;   // rows of offd holding data (ROW_OS after an un-decoupled assembly)
  bool compact = false;   // decoupled in compact form (compact.cu): diag = D^-1[:, :CR], offd raw
  bool compact_ok = true; // ISC_COMPACT=0 disables the compact form (A/B switch)
  double* cmid = nullptr; // split cell pass: property values for k_cell_rows (NMID x n)
  double* cbp = nullptr;  // compact form: B'_bd = B_bd[:6, :] D_nb^-1[:, :6] of black cells
  bool gb_fresh = false;  // compact form: the factorisation left g_b in rk / rhat
  bool assembled = false;   // the last assembly was isc_assemble (inputs kept for FD)
  double asm_dt = 0.0;
  int asm_freeze = 0;
  double *rhs = nullptr, *xk = nullptr, *rk = nullptr, *rhat = nullptr, *pk = nullptr,
         *vk = nullptr, *phat = nullptr, *shat = nullptr, *sk = nullptr, *tk = nullptr;
  double* sc = nullptr;
  double* sc_h = nullptr;   // pinned
  double* partial = nullptr;
  double* partial2 = nullptr;   // second stage of the fixed-order sums
  double* fbuf = nullptr;       // face fluxes of the face-centric assembly (3*ROW_OS x n)
  int64_t npartial = 0;
  int* flags = nullptr;
  int* fail_d = nullptr;
  int* ccnz_d = nullptr;   // != 0: a flux row < ROW_E has a coke column entry (k_cc_red reads it)
  // ILU
  IluDev ilu{};
  int64_t* lvl_ptr_d = nullptr;
  int nlev = 0;
  int nsub = 1;
  double* schur = nullptr;        // per-well Schur rhs terms (fused path)
  int64_t dc_bad_cell = -1;       // singular block found by the fused decoupling
  int dc_bad_col = -1;
  double* mc_uinv = nullptr;   // multicolour ILU: U_b^-1 of black cells
  // multi-GPU z-slab decomposition
  Comm comm;
  double *halo_send_lo = nullptr, *halo_send_hi = nullptr, *halo_recv_lo = nullptr,
         *halo_recv_hi = nullptr;
  // timing
  cudaEvent_t ev[8] = {};
  double stage_ms[4] = {0, 0, 0, 0};
  // per-kernel-class device time (CUDA events), enabled by isc_set_profiling
  bool profiling = false;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  struct Pending { int kind; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  double kern_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t kern_n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

// kernel classes for isc_kernel_times
enum { KT_CELL = 0, KT_FACE, KT_WELLS, KT_DECOUPLE, KT_ILU_FACTOR, KT_ILU_APPLY, KT_SPMV, KT_VEC };

static cudaEvent_t pool_event(isc_ctx* ctx) {
  if (ctx->pool_used == ctx->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->pool.push_back(e);
  }
  return ctx->pool[ctx->pool_used++];
}
struct KScope {
  isc_ctx* ctx;
  int kind;
  cudaEvent_t a = nullptr;
  KScope(isc_ctx* c, int k) : ctx(c), kind(k) {
    if (ctx->profiling) {
      a = pool_event(ctx);
      cudaEventRecord(a, ctx->stream);
    }
  }
  ~KScope() {
    if (ctx->profiling) {
      cudaEvent_t b = pool_event(ctx);
      cudaEventRecord(b, ctx->stream);
      ctx->pending.push_back({kind, a, b});
    }
  }
};
// after a stream synchronisation: fold finished event pairs into the totals
static void kflush(isc_ctx* ctx) {
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      ctx->kern_ms[p.kind] += ms;
      ctx->kern_n[p.kind] += 1;
    }
  }
  ctx->pending.clear();
  ctx->pool_used = 0;
}

static int dev_alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes > 0 ? bytes : 8);
  if (e != cudaSuccess) {
    g_err = std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e);
    return ISC_CUDA_ERROR;
  }
  return ISC_OK;
}
#define ALLOC(ptr, bytes)                                            \
  do {                                                               \
    int s_ = dev_alloc((void**)&(ptr), (size_t)(bytes));             \
    if (s_) return s_;                                               \
  } while (0)

static int grid1d(int64_t n, int t) { return (int)((n + t - 1) / t); }
static void free_ilu(isc_ctx* ctx);
static int halo_exchange(isc_ctx* ctx, double* v, int rows);
static int allreduce_dev(isc_ctx* ctx, double* d, int count);
extern "C" int isc_comm_allreduce_host(isc_ctx* ctx, double* vals, int32_t count, int32_t op);

// ------------------------------------------------------ ILU structure
// Subdomains exactly as the reference: count min(64, max(1, n // 2048))
// (linsolve.py:34-42), slabs along the first longest axis with the
// remainder on the leading slabs (grid.py:148-166); RAS extends each slab
// by its one-plane halo (linsolve.py:341-345), bjacobi does not.
static int build_ilu(isc_ctx* ctx) {
  const Dims& g = ctx->g;
  const int64_t n = g.n;
  const int nsub = (int)std::min<int64_t>(64, std::max<int64_t>(1, n / 2048));
  const int dims[3] = {g.nx, g.ny, g.nz};
  int axis = 0;
  for (int a = 1; a < 3; ++a)
    if (dims[a] > dims[axis]) axis = a;
  const int na = dims[axis];
  const int base = na / nsub, extra = na % nsub;
  struct Box { int lo[3], hi[3], olo, ohi; };
  std::vector<Box> boxes;
  int pos = 0;
  for (int s = 0; s < nsub; ++s) {
    const int size = base + (s < extra ? 1 : 0);
    Box b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = 0; b.hi[a] = dims[a]; }
    b.olo = pos;
    b.ohi = pos + size;
    b.lo[axis] = pos;
    b.hi[axis] = pos + size;
    if (ctx->precond == ISC_PRECOND_RAS && nsub > 1) {
      b.lo[axis] = std::max(0, pos - 1);
      b.hi[axis] = std::min(na, pos + size + 1);
    }
    pos += size;
    boxes.push_back(b);
  }
  // slots: subdomain-major, level-major inside a subdomain box; the level
  // of a cell is (i-x0)+(j-y0)+(k-z0) (its dependencies sit one level lower)
  int maxlev = 0;
  for (auto& b : boxes)
    maxlev = std::max(maxlev, (b.hi[0] - b.lo[0] - 1) + (b.hi[1] - b.lo[1] - 1) + (b.hi[2] - b.lo[2] - 1));
  const int nlev = maxlev + 1;
  std::vector<int64_t> lvl_ptr((size_t)nsub * (nlev + 1), 0);
  int64_t total = 0;
  for (int s = 0; s < nsub; ++s) {
    const Box& b = boxes[s];
    std::vector<int64_t> cnt(nlev, 0);
    for (int k = b.lo[2]; k < b.hi[2]; ++k)
      for (int j = b.lo[1]; j < b.hi[1]; ++j)
        for (int i = b.lo[0]; i < b.hi[0]; ++i) cnt[(i - b.lo[0]) + (j - b.lo[1]) + (k - b.lo[2])]++;
    int64_t* lp = lvl_ptr.data() + (size_t)s * (nlev + 1);
    lp[0] = total;
    for (int l = 0; l < nlev; ++l) lp[l + 1] = lp[l] + cnt[l];
    total = lp[nlev];
  }
  const int64_t ns = total;
  std::vector<int64_t> cell(ns), lo(3 * ns, -1), up(3 * ns, -1);
  std::vector<int8_t> owned(ns, 0);
  for (int sidx = 0; sidx < nsub; ++sidx) {
    const Box& b = boxes[sidx];
    std::vector<int64_t> fill(lvl_ptr.begin() + (size_t)sidx * (nlev + 1),
                              lvl_ptr.begin() + (size_t)sidx * (nlev + 1) + nlev);
    const int wx = b.hi[0] - b.lo[0], wy = b.hi[1] - b.lo[1], wz = b.hi[2] - b.lo[2];
    std::vector<int64_t> slot((size_t)wx * wy * wz);
    for (int k = b.lo[2]; k < b.hi[2]; ++k)
      for (int j = b.lo[1]; j < b.hi[1]; ++j)
        for (int i = b.lo[0]; i < b.hi[0]; ++i) {
          const int li = i - b.lo[0], lj = j - b.lo[1], lk = k - b.lo[2];
          const int64_t s = fill[li + lj + lk]++;
          slot[((size_t)lk * wy + lj) * wx + li] = s;
          cell[s] = pos_of(g, i + (int64_t)g.nx * (j + (int64_t)g.ny * k));
          const int ijk[3] = {i, j, k};
          owned[s] = (ijk[axis] >= b.olo && ijk[axis] < b.ohi) ? 1 : 0;
        }
    for (int lk = 0; lk < wz; ++lk)
      for (int lj = 0; lj < wy; ++lj)
        for (int li = 0; li < wx; ++li) {
          const int64_t s = slot[((size_t)lk * wy + lj) * wx + li];
          auto at = [&](int a, int bb, int c) { return slot[((size_t)c * wy + bb) * wx + a]; };
          // lower in ascending neighbour index: -z, -y, -x
          if (lk > 0) lo[0 * ns + s] = at(li, lj, lk - 1);
          if (lj > 0) lo[1 * ns + s] = at(li, lj - 1, lk);
          if (li > 0) lo[2 * ns + s] = at(li - 1, lj, lk);
          // upper ascending: +x, +y, +z
          if (li + 1 < wx) up[0 * ns + s] = at(li + 1, lj, lk);
          if (lj + 1 < wy) up[1 * ns + s] = at(li, lj + 1, lk);
          if (lk + 1 < wz) up[2 * ns + s] = at(li, lj, lk + 1);
        }
  }
  ctx->nsub = nsub;
  int64_t *cell_d, *lo_d, *up_d;
  int8_t* owned_d;
  ALLOC(cell_d, ns * 8);
  ALLOC(lo_d, 3 * ns * 8);
  ALLOC(up_d, 3 * ns * 8);
  ALLOC(owned_d, ns);
  ALLOC(ctx->lvl_ptr_d, lvl_ptr.size() * 8);
  CK(cudaMemcpy(cell_d, cell.data(), ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lo_d, lo.data(), 3 * ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(up_d, up.data(), 3 * ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(owned_d, owned.data(), ns, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->lvl_ptr_d, lvl_ptr.data(), lvl_ptr.size() * 8, cudaMemcpyHostToDevice));
  double *lblk, *uinv, *zs, *aup;
  ALLOC(aup, (size_t)3 * NB * ns * 8);
  ALLOC(lblk, (size_t)3 * NB * ns * 8);
  ALLOC(uinv, (size_t)NB * ns * 8);
  ALLOC(zs, (size_t)NU * ns * 8);
  ctx->ilu = IluDev{ns, cell_d, owned_d, lo_d, up_d, lblk, uinv, zs, aup};
  ctx->nlev = nlev;
  return ISC_OK;
}

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
  ALLOC(ctx->schur, std::max(1, nwells) * NU * 8);
  ALLOC(ctx->capped_d, std::max(1, nwells));
  // assembly buffers
  ALLOC(ctx->rec, (size_t)NREC * n * 8);
  if (CELL_SPLIT) ALLOC(ctx->cmid, (size_t)NMID * n * 8);
  ALLOC(ctx->fbuf, (size_t)3 * ROW_OS * n * 8);
  ALLOC(ctx->acc, (size_t)NU * n * 8);
  ALLOC(ctx->src, (size_t)NU * n * 8);
  ALLOC(ctx->resid, (size_t)NU * n * 8);
  ALLOC(ctx->diag, (size_t)NB * n * 8);
  ALLOC(ctx->offd, (size_t)NDIR * NB * n * 8);
  ALLOC(ctx->upw, (size_t)9 * n);
  CK(cudaMemset(ctx->upw, 0, (size_t)9 * n));
  ALLOC(ctx->bad_d, 8);
  CK(cudaMallocHost(&ctx->bad_h, 8));
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
                  ctx->offd, ctx->upw, ctx->bad_d, ctx->rhs, ctx->xk, ctx->rk, ctx->rhat,
                  ctx->pk, ctx->vk, ctx->phat, ctx->shat, ctx->sk, ctx->tk, ctx->sc,
                  ctx->partial, ctx->partial2, ctx->fbuf, ctx->flags, ctx->fail_d, ctx->ccnz_d, ctx->schur, ctx->st_c, ctx->accn_c, ctx->stage,
                  ctx->halo_send_lo, ctx->halo_send_hi, ctx->halo_recv_lo, ctx->halo_recv_hi,
                  ctx->gm_V, ctx->gm_h, ctx->cbp, ctx->cmid};
  if (ctx->comm.nccl && nccl_api().CommDestroy) nccl_api().CommDestroy(ctx->comm.nccl);
  free_ilu(ctx);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->wout_h) cudaFreeHost(ctx->wout_h);
  if (ctx->bad_h) cudaFreeHost(ctx->bad_h);
  if (ctx->sc_h) cudaFreeHost(ctx->sc_h);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (auto& e : ctx->chunk_ev)
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

static int stage_begin(isc_ctx* ctx, int st) {
  CK(cudaEventRecord(ctx->ev[2 * st], ctx->stream));
  return ISC_OK;
}
static int stage_end(isc_ctx* ctx, int st) {
  CK(cudaEventRecord(ctx->ev[2 * st + 1], ctx->stream));
  CK(cudaEventSynchronize(ctx->ev[2 * st + 1]));
  kflush(ctx);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev[2 * st], ctx->ev[2 * st + 1]));
  ctx->stage_ms[st] += ms;
  return ISC_OK;
}
#define STAGE(call) do { int s_ = (call); if (s_) return s_; } while (0)

// ------------------------------------------------------------- assemble

// face evaluation over lower cells [c0, c1), axes axis_lo .. axis_lo+naxes-1
static void launch_face_eval(const FaceArgs2& F2, int64_t c0, int64_t c1, int axis_lo, int naxes,
                             cudaStream_t st) {
  const int blocks = grid1d(c1 - c0, 32);
  if (FACE_SPLIT) {
    k_face_eval_light<<<dim3(blocks, ROW_E), dim3(32, naxes), 0, st>>>(F2, c0, c1, axis_lo);
    k_face_eval_energy<<<blocks, dim3(32, naxes), 0, st>>>(F2, c0, c1, axis_lo);
  } else {
    k_face_eval<<<dim3(blocks, ROW_OS), dim3(32, naxes), 0, st>>>(F2, c0, c1, axis_lo);
  }
}

// the cell pass over positions [A.c_begin, A.c_end): one kernel, or the
// property and row halves (fewer live values per kernel; assemble.cu)
static void launch_cell(isc_ctx* ctx, CellArgs A, cudaStream_t st) {
  const int blocks = grid1d(A.c_end - A.c_begin, 128);
  if (CELL_SPLIT) {
    A.mid = ctx->cmid;
    k_cell_props<<<blocks, 128, 0, st>>>(ctx->M, A);
    if (CELL_GAS_SPLIT) {
      k_cell_gas<<<blocks, 128, 0, st>>>(ctx->M, A);
      ++ctx->launches;
    }
    k_cell_rows<<<blocks, 128, 0, st>>>(ctx->M, A);
    ++ctx->launches;
  } else {
    k_cell<<<blocks, 128, 0, st>>>(ctx->M, A);
  }
}

extern "C" int isc_assemble(isc_ctx* ctx, const double* d_state, const double* h_bhp,
                            const double* d_accn, double dt, double t_new,
                            const uint8_t* h_capped, int32_t freeze, double* h_wells_out,
                            int64_t* bad_cell) {
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  ctx->assembled = false;
  // set by isc_assemble_host when it ran these passes while staging
  const bool cell_pre = ctx->cell_pre, face_pre = ctx->face_pre;
  ctx->cell_pre = ctx->face_pre = false;
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
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  {
    // all ranks of a z-slab run take the same branch
    double flag = *ctx->bad_h != ~0ULL ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
    if (as) return as;
    if (flag > 0.0) {
      if (bad_cell) *bad_cell = *ctx->bad_h != ~0ULL ? (int64_t)*ctx->bad_h : -1;
      g_err = "coke fills the pore volume";
      STAGE(stage_end(ctx, 0));
      return ISC_PORE_SPACE_EXHAUSTED;
    }
  }
  FaceArgs F{ctx->g, d_state, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, freeze,
             ctx->resid, ctx->diag, ctx->offd, ctx->ccnz_d};
#ifndef FACE_CENTRIC
#define FACE_CENTRIC 1
#endif
  {
    KScope ks(ctx, KT_FACE);
    if (FACE_CENTRIC) {
      FaceArgs2 F2{F, ctx->fbuf};
      if (!face_pre) {
        CK(cudaMemsetAsync(ctx->ccnz_d, 0, 4, st));   // set by k_face_eval* on a nonzero
        launch_face_eval(F2, 0, n, 0, 3, st);
      }
      k_face_gather<<<grid1d((int64_t)(ctx->g.kw_hi - ctx->g.kw_lo) * ctx->g.nxny, 32),
                      dim3(32, ROW_OS), 0, st>>>(F2);
      ++ctx->launches;
    } else {
      CK(cudaMemsetAsync(ctx->ccnz_d, 0xff, 4, st));   // two-sided kernel: not tracked
      k_face<<<grid1d(n, 32), dim3(32, NU), 0, st>>>(F);
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
  STAGE(stage_end(ctx, 0));   // synchronises
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

// Fast path: assemble + well Schur fold + decoupling fused (fused.cu). The
// un-decoupled diagonal/off-diagonal blocks are never written; a singular
// block is reported by the following isc_solve, as the reference raises it
// inside BlockSolver.solve (linsolve.py:458-463).
extern "C" int isc_assemble_decoupled(isc_ctx* ctx, const double* d_state, const double* h_bhp,
                                      const double* d_accn, double dt, double t_new,
                                      const uint8_t* h_capped, int32_t freeze,
                                      double* h_wells_out, int64_t* bad_cell) {
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  STAGE(stage_begin(ctx, 0));
  if (ctx->nw > 0) {
    CK(cudaMemcpyAsync(ctx->bhp_d, h_bhp, ctx->nw * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->capped_d, h_capped, ctx->nw, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
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
  { KScope ks(ctx, KT_CELL); launch_cell(ctx, A, st); }
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  {
    // all ranks of a z-slab run take the same branch
    double flag = *ctx->bad_h != ~0ULL ? 1.0 : 0.0;
    int as = isc_comm_allreduce_host(ctx, &flag, 1, 1);
    if (as) return as;
    if (flag > 0.0) {
      if (bad_cell) *bad_cell = *ctx->bad_h != ~0ULL ? (int64_t)*ctx->bad_h : -1;
      g_err = "coke fills the pore volume";
      STAGE(stage_end(ctx, 0));
      return ISC_PORE_SPACE_EXHAUSTED;
    }
  }
  if (ctx->nw > 0) {
    KScope ks(ctx, KT_WELLS);
    k_wells<<<1, 32, 0, st>>>(ctx->M, ctx->g, ctx->nw, ctx->wells_d, d_state, ctx->bhp_d,
                              ctx->capped_d, ctx->rec, ctx->depth, t_new, ctx->resid,
                              ctx->diag, ctx->wout_d);
    LAUNCH_CHECK();
    k_schur_pre<<<1, 32, 0, st>>>(ctx->g, ctx->nw, ctx->wcell_d, ctx->wout_d, WOUT, ctx->diag,
                                  ctx->schur);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(ctx->wout_h, ctx->wout_d, ctx->nw * WOUT * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemsetAsync(ctx->flags, 0, n * 4, st));
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  {
    KScope ks(ctx, KT_FACE);
    FaceArgs F{ctx->g, d_state, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, freeze,
               ctx->resid, ctx->diag, ctx->offd, ctx->ccnz_d};
    CK(cudaMemsetAsync(ctx->ccnz_d, 0xff, 4, st));   // decoupled (dense) blocks
    FusedArgs P{F, ctx->resid, ctx->rhs, ctx->nw, ctx->wcell_d, ctx->schur, ctx->flags,
                ctx->bad_d};
    CK(cudaFuncSetAttribute(k_face_dc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(FusedSmem)));
    k_face_dc<<<grid1d(n, FD_CELLS), FD_CELLS * 64, sizeof(FusedSmem), st>>>(P);
    LAUNCH_CHECK();
  }
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  STAGE(stage_end(ctx, 0));   // synchronises
  if (ctx->nw > 0 && h_wells_out) std::memcpy(h_wells_out, ctx->wout_h, ctx->nw * WOUT * 8);
  ctx->dc_bad_cell = -1;
  ctx->dc_bad_col = -1;
  if (*ctx->bad_h != ~0ULL) {
    const int64_t c = (int64_t)*ctx->bad_h;
    int flag = 0;
    CK(cudaMemcpy(&flag, ctx->flags + c, 4, cudaMemcpyDeviceToHost));
    ctx->dc_bad_cell = c;
    ctx->dc_bad_col = flag - 1;
  }
  ctx->compact = false;
  ctx->decoupled = true;
  ctx->factored = false;
  ctx->offd_rows = NU;
  ctx->assembled = false;
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
  const int nq = pipe ? std::min(8, g.nz) : 1;
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
  CK(cudaEventRecord(ctx->chunk_ev[0], st));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->chunk_ev[0], 0));   // stage buffer free
  CellArgs A{g, ctx->st_c, ctx->phi_ref, ctx->vol, ctx->hl_area, ctx->hl_kob, ctx->hl_d,
             ctx->hl_rho, ctx->hl_tini, ctx->accn_c, dt, ctx->rec, ctx->acc, ctx->src,
             ctx->resid, ctx->diag, ctx->bad_d, 0, n};
  FaceArgs F{g, ctx->st_c, ctx->rec, ctx->depth, ctx->gd, ctx->td, ctx->upw, freeze,
             ctx->resid, ctx->diag, ctx->offd, ctx->ccnz_d};
  FaceArgs2 F2{F, ctx->fbuf};
  if (pipe && FACE_CENTRIC) CK(cudaMemsetAsync(ctx->ccnz_d, 0, 4, st));
  for (int q = 0; q < nq; ++q) {
    const int64_t k0 = (int64_t)g.nz * q / nq, k1 = (int64_t)g.nz * (q + 1) / nq;
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
      KScope ks(ctx, KT_FACE);
      // x/y faces of this chunk's cells; z faces of the plane below it and of
      // all but its last plane (their upper records now exist)
      launch_face_eval(F2, c0, c1, 0, 2, st);
      const int64_t z0 = std::max<int64_t>(0, (k0 - 1) * g.nxny), z1 = (k1 - 1) * g.nxny;
      if (z1 > z0)
        launch_face_eval(F2, z0, z1, 2, 1, st);
      ctx->launches += 3;
    }
  }
  if (pipe) {   // z faces of the top plane (boundary: zero blocks)
    KScope ks(ctx, KT_FACE);
    const int64_t z0 = (int64_t)(g.nz - 1) * g.nxny;
    launch_face_eval(F2, z0, n, 2, 1, st);
    ++ctx->launches;
  }
  LAUNCH_CHECK();
  ctx->cell_pre = pipe;
  ctx->face_pre = pipe && FACE_CENTRIC;
  return isc_assemble(ctx, nullptr, h_bhp, nullptr, dt, t_new, h_capped, freeze, h_wells_out,
                      bad_cell);
}

// du of the last isc_solve as a host (n, NU) array in natural cell order
extern "C" int isc_download_du(isc_ctx* ctx, double* h_du) {
  const int64_t n = ctx->g.n;
  k_unstage_rows<<<grid1d(n, 256), 256, 0, ctx->stream>>>(ctx->g, ctx->xk, ctx->stage);
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

extern "C" int isc_decouple(isc_ctx* ctx, int64_t* bad_cell, int32_t* bad_col) {
  const int64_t n = ctx->g.n;
  cudaStream_t st = ctx->stream;
  // well equations with a zero / non-finite bhp derivative (linsolve.py:372-375)
  {
    double wbad = 0.0;
    if (ctx->nw > 0) {
      CK(cudaMemcpyAsync(ctx->wout_h, ctx->wout_d, ctx->nw * WOUT * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
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
  k_rhs_schur<<<grid1d(n, 256), 256, 0, st>>>(ctx->g, ctx->resid, ctx->rhs, ctx->diag, ctx->nw,
                                              ctx->wcell_d, ctx->wout_d, WOUT);
  LAUNCH_CHECK();
  CK(cudaMemsetAsync(ctx->flags, 0, n * 4, st));
  CK(cudaMemsetAsync(ctx->bad_d, 0xff, 8, st));
#ifndef DECOUPLE_WS
#define DECOUPLE_WS 1
#endif
  // compact form: the red-eliminated multicolour solve of an assembled
  // system (compact.cu)
  ctx->compact = ctx->compact_ok && ctx->precond == ISC_PRECOND_MCILU && ctx->g.colored &&
                 ctx->mc_schur && MC_SCHUR && ctx->offd_rows == ROW_OS;
  if (ctx->compact && !ctx->cbp &&
      cudaMalloc(&ctx->cbp, (size_t)NDIR * CR * CR * ctx->g.half * 8) != cudaSuccess) {
    cudaGetLastError();
    ctx->cbp = nullptr;
    ctx->compact = false;   // no room for B': the explicit form
  }
  if (ctx->compact) {
    const int64_t owned = (int64_t)(ctx->g.kw_hi - ctx->g.kw_lo) * ctx->g.nxny;
#ifndef DCC_THREAD
#define DCC_THREAD 1   // thread per cell (k_decouple_compact_t); 0: thread per column
#endif
    if (DCC_THREAD)
      k_decouple_compact_t<<<grid1d(owned, DCT_THREADS), DCT_THREADS, 0, st>>>(
          ctx->g, ctx->diag, ctx->rhs, ctx->flags, ctx->bad_d);
    else
      k_decouple_compact<<<grid1d(owned, 32), dim3(32, NU), 0, st>>>(ctx->g, ctx->diag, ctx->rhs,
                                                                    ctx->flags, ctx->bad_d);
  } else if (DECOUPLE_WS) {
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
  } else {
    k_decouple3<<<grid1d(n, DC3_CELLS), DC3_THREADS, 0, st>>>(ctx->g, ctx->diag, ctx->offd,
                                                               ctx->rhs, ctx->flags, ctx->bad_d,
                                                               ctx->offd_rows);
  }
  LAUNCH_CHECK();
  if (!ctx->compact) ctx->offd_rows = NU;   // the decoupled blocks are dense
  }
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->bad_d, 8, cudaMemcpyDeviceToHost, st));
  STAGE(stage_end(ctx, 1));
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
  ctx->dc_bad_cell = -1;
  return ISC_OK;
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

extern "C" int isc_precond_setup(isc_ctx* ctx, int64_t* bad_cell) {
  if (ctx->precond == ISC_PRECOND_NONE) { ctx->factored = true; return ISC_OK; }
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
      CK(cudaFuncSetAttribute(k_mc_factor_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(McfcSmem)));
      k_mc_factor_compact<<<grid1d(ctx->g.tw_hi - ctx->g.tw_lo, 32), dim3(32, NU),
                            sizeof(McfcSmem), st>>>(
          ctx->g, ctx->offd, ctx->diag, ctx->mc_uinv, ctx->cbp, ctx->fail_d, ctx->rhs, ctx->rk,
          ctx->rhat);
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
  int fail_h = 0;
  CK(cudaMemcpyAsync(ctx->bad_h, ctx->fail_d, 4, cudaMemcpyDeviceToHost, st));
  STAGE(stage_end(ctx, 2));
  std::memcpy(&fail_h, ctx->bad_h, 4);
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

// ------------------------------------------------- multi-GPU z-slab comm

static int setup_window(isc_ctx* ctx, int32_t rank, int32_t nranks, int32_t has_lo,
                        int32_t has_hi, int32_t kw_lo, int32_t kw_hi) {
  if (kw_lo < 0 || kw_hi > ctx->g.nz || kw_lo >= kw_hi || (has_lo && kw_lo < 1) ||
      (has_hi && kw_hi > ctx->g.nz - 1)) {
    g_err = "bad owned plane window";
    return ISC_BAD_ARGUMENT;
  }
  if (ctx->precond == ISC_PRECOND_RAS || ctx->precond == ISC_PRECOND_BJACOBI) {
    g_err = "multi-rank solves use mcilu or none (rank-local block-Jacobi of the multicolour ILU)";
    return ISC_UNSUPPORTED;
  }
  ctx->g.kw_lo = kw_lo;
  ctx->g.kw_hi = kw_hi;
  ctx->g.tw_lo = ctx->g.colored ? (int64_t)kw_lo * ctx->g.ph : 0;
  ctx->g.tw_hi = ctx->g.colored ? (int64_t)kw_hi * ctx->g.ph : ctx->g.half;
  ctx->comm.rank = rank;
  ctx->comm.nranks = nranks;
  ctx->comm.has_lo = has_lo != 0;
  ctx->comm.has_hi = has_hi != 0;
  // one plane of up to NB rows (vectors: NU; boundary blocks for the factor: NB)
  const size_t bytes = (size_t)NB * ctx->g.nxny * 8;
  if (!ctx->halo_send_lo) {
    ALLOC(ctx->halo_send_lo, bytes);
    ALLOC(ctx->halo_send_hi, bytes);
    ALLOC(ctx->halo_recv_lo, bytes);
    ALLOC(ctx->halo_recv_hi, bytes);
  }
  return ISC_OK;
}

extern "C" int isc_comm_nccl(isc_ctx* ctx, const void* unique_id, int32_t rank, int32_t nranks,
                             int32_t has_lo, int32_t has_hi, int32_t kw_lo, int32_t kw_hi) {
  int s = setup_window(ctx, rank, nranks, has_lo, has_hi, kw_lo, kw_hi);
  if (s) return s;
  if (nranks > 1) {
    NcclApi& api = nccl_api();
    if (!api.ok) { g_err = "libnccl.so.2 not available in this process"; return ISC_UNSUPPORTED; }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    const int r = api.CommInitRank(&ctx->comm.nccl, nranks, id, rank);
    if (r != ncclSuccess_) {
      g_err = std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "");
      return ISC_CUDA_ERROR;
    }
  }
  return ISC_OK;
}

extern "C" int isc_nccl_unique_id(void* out128) {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_err = "libnccl.so.2 not found"; return ISC_UNSUPPORTED; }
  auto fn = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
  if (!fn) { g_err = "ncclGetUniqueId not found"; return ISC_UNSUPPORTED; }
  ncclUniqueId id;
  if (fn(&id) != ncclSuccess_) { g_err = "ncclGetUniqueId failed"; return ISC_CUDA_ERROR; }
  std::memcpy(out128, &id, sizeof(id));
  return ISC_OK;
}

extern "C" void* isc_hub_create(int32_t nranks) {
  Hub* h = new Hub();
  h->nranks = nranks;
  h->send_lo.assign(nranks, nullptr);
  h->send_hi.assign(nranks, nullptr);
  h->ready.assign(nranks, nullptr);
  h->red.assign((size_t)nranks * 64, 0.0);
  return h;
}
extern "C" int isc_hub_destroy(void* hub) {
  delete (Hub*)hub;
  return ISC_OK;
}

extern "C" int isc_comm_hub(isc_ctx* ctx, void* hub, int32_t rank, int32_t has_lo, int32_t has_hi,
                            int32_t kw_lo, int32_t kw_hi) {
  Hub* h = (Hub*)hub;
  int s = setup_window(ctx, rank, h->nranks, has_lo, has_hi, kw_lo, kw_hi);
  if (s) return s;
  ctx->comm.hub = h;
  h->send_lo[rank] = ctx->halo_send_lo;
  h->send_hi[rank] = ctx->halo_send_hi;
  CK(cudaEventCreateWithFlags(&h->ready[rank], cudaEventDisableTiming));
  return ISC_OK;
}

// one-plane halo of a storage-order vector (rows x n)
// Halo exchange in two halves so that work not touching the ghost planes
// can run in between: halo_start packs the boundary planes on the main
// stream; halo_finish moves them on the copy stream (NCCL send/recv, or
// device copies between hub contexts), unpacks into the ghost planes there
// and makes the main stream wait for it.
static int halo_start(isc_ctx* ctx, double* v, int rows) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  const int64_t cnt = (int64_t)rows * g.nxny;
  const int bl = grid1d(cnt, 256);
  if (cm.has_lo) k_pack_plane<<<bl, 256, 0, st>>>(g, rows, g.kw_lo, v, ctx->halo_send_lo);
  if (cm.has_hi) k_pack_plane<<<bl, 256, 0, st>>>(g, rows, g.kw_hi - 1, v, ctx->halo_send_hi);
  ctx->launches += (cm.has_lo ? 1 : 0) + (cm.has_hi ? 1 : 0);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->halo_ev[0], st));
  return ISC_OK;
}

static int halo_finish(isc_ctx* ctx, double* v, int rows) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream, cs = ctx->cstream;
  const int64_t cnt = (int64_t)rows * g.nxny;
  const int bl = grid1d(cnt, 256);
  CK(cudaStreamWaitEvent(cs, ctx->halo_ev[0], 0));
  if (cm.nccl) {
    NcclApi& api = nccl_api();
    api.GroupStart();
    if (cm.has_lo) {
      api.Send(ctx->halo_send_lo, cnt, ncclFloat64_, cm.rank - 1, cm.nccl, cs);
      api.Recv(ctx->halo_recv_lo, cnt, ncclFloat64_, cm.rank - 1, cm.nccl, cs);
    }
    if (cm.has_hi) {
      api.Send(ctx->halo_send_hi, cnt, ncclFloat64_, cm.rank + 1, cm.nccl, cs);
      api.Recv(ctx->halo_recv_hi, cnt, ncclFloat64_, cm.rank + 1, cm.nccl, cs);
    }
    const int r = api.GroupEnd();
    if (r != ncclSuccess_) { g_err = "NCCL halo exchange failed"; return ISC_CUDA_ERROR; }
  } else if (cm.hub) {
    Hub* h = cm.hub;
    CK(cudaEventRecord(h->ready[cm.rank], cs));   // after the pack (cs waited for it)
    h->barrier();
    if (cm.has_lo) {
      CK(cudaStreamWaitEvent(cs, h->ready[cm.rank - 1], 0));
      CK(cudaMemcpyAsync(ctx->halo_recv_lo, h->send_hi[cm.rank - 1], cnt * 8,
                         cudaMemcpyDeviceToDevice, cs));
    }
    if (cm.has_hi) {
      CK(cudaStreamWaitEvent(cs, h->ready[cm.rank + 1], 0));
      CK(cudaMemcpyAsync(ctx->halo_recv_hi, h->send_lo[cm.rank + 1], cnt * 8,
                         cudaMemcpyDeviceToDevice, cs));
    }
    CK(cudaStreamSynchronize(cs));
    h->barrier();   // neighbours may now reuse their send buffers
  }
  if (cm.has_lo) k_unpack_plane<<<bl, 256, 0, cs>>>(g, rows, g.kw_lo - 1, ctx->halo_recv_lo, v);
  if (cm.has_hi) k_unpack_plane<<<bl, 256, 0, cs>>>(g, rows, g.kw_hi, ctx->halo_recv_hi, v);
  ctx->launches += (cm.has_lo ? 1 : 0) + (cm.has_hi ? 1 : 0);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->halo_ev[1], cs));
  CK(cudaStreamWaitEvent(st, ctx->halo_ev[1], 0));
  return ISC_OK;
}

static int halo_exchange(isc_ctx* ctx, double* v, int rows) {
  int s = halo_start(ctx, v, rows);
  if (s) return s;
  return halo_finish(ctx, v, rows);
}

// sum `count` consecutive device scalars over the ranks (in place)
static int allreduce_dev(isc_ctx* ctx, double* d, int count) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  if (cm.nccl) {
    const int r = nccl_api().AllReduce(d, d, count, ncclFloat64_, ncclSum_, cm.nccl, ctx->stream);
    if (r != ncclSuccess_) { g_err = "NCCL allreduce failed"; return ISC_CUDA_ERROR; }
    return ISC_OK;
  }
  Hub* h = cm.hub;
  double loc[64];
  CK(cudaMemcpyAsync(loc, d, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::memcpy(&h->red[(size_t)cm.rank * 64], loc, count * 8);
  h->barrier();
  for (int i = 0; i < count; ++i) {
    double s = 0.0;
    for (int q = 0; q < h->nranks; ++q) s += h->red[(size_t)q * 64 + i];   // rank order
    loc[i] = s;
  }
  h->barrier();
  CK(cudaMemcpyAsync(d, loc, count * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

// host-side reductions over ranks: op 0 sum, 1 max (NaN propagates)
extern "C" int isc_comm_allreduce_host(isc_ctx* ctx, double* vals, int32_t count, int32_t op) {
  Comm& cm = ctx->comm;
  if (!cm.active() || count <= 0) return ISC_OK;
  if (count > 64) { g_err = "too many values"; return ISC_BAD_ARGUMENT; }
  if (cm.nccl) {
    // NCCL's max on doubles drops NaN (fmax semantics), so a NaN norm on one
    // rank would vanish behind the others' finite values. For op max the
    // values go as (NaN -> +inf, NaN flag) pairs in one reduction and NaN is
    // restored wherever any rank had one (the hub path below propagates it).
    double buf[128];
    const int len = op ? 2 * count : count;
    for (int i = 0; i < count; ++i) {
      const bool nan = vals[i] != vals[i];
      buf[i] = (op && nan) ? INFINITY : vals[i];
      if (op) buf[count + i] = nan ? 1.0 : 0.0;
    }
    double* d = ctx->partial;   // scratch
    CK(cudaMemcpyAsync(d, buf, len * 8, cudaMemcpyHostToDevice, ctx->stream));
    const int r = nccl_api().AllReduce(d, d, len, ncclFloat64_, op ? ncclMax_ : ncclSum_,
                                       cm.nccl, ctx->stream);
    if (r != ncclSuccess_) { g_err = "NCCL allreduce failed"; return ISC_CUDA_ERROR; }
    CK(cudaMemcpyAsync(buf, d, len * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < count; ++i) vals[i] = (op && buf[count + i] > 0.0) ? NAN : buf[i];
    return ISC_OK;
  }
  Hub* h = cm.hub;
  std::memcpy(&h->red[(size_t)cm.rank * 64], vals, count * 8);
  h->barrier();
  for (int i = 0; i < count; ++i) {
    double s = op ? h->red[i] : 0.0;
    for (int q = op ? 1 : 0; q < h->nranks; ++q) {
      const double v = h->red[(size_t)q * 64 + i];
      s = op ? ((v != v || s != s) ? v + s : std::max(s, v)) : s + v;
    }
    vals[i] = s;
  }
  h->barrier();
  return ISC_OK;
}

// ------------------------------------------------------------- BiCGSTAB

struct Kry {
  isc_ctx* ctx;
  int64_t len;
  const double* stop = nullptr;   // device-driven iterations: S_STOP guard of the sums
  int vgrid() const { return RED_BLOCKS; }
  // fixed-order sums: one block for RED_BLOCKS partials, two stages for the
  // per-warp partials of the stencil passes
  template <int K>
  void finalize(int nparts, int s0, int s1) {
    if (nparts <= RED_BLOCKS) {
      k_finalize<K><<<1, 256, 0, ctx->stream>>>(ctx->partial, nparts, ctx->sc, s0, s1, s1,
                                                stop);
      ++ctx->launches;
      return;
    }
    k_partial_sum<K><<<FIN_BLOCKS, 256, 0, ctx->stream>>>(ctx->partial, nparts, ctx->partial2,
                                                          stop);
    k_finalize<K><<<1, 256, 0, ctx->stream>>>(ctx->partial2, FIN_BLOCKS, ctx->sc, s0, s1, s1,
                                              stop);
    ctx->launches += 2;
  }
  int finalize1(int nparts, int s0) {
    finalize<1>(nparts, s0, s0);
    if (cudaGetLastError() != cudaSuccess) return ISC_CUDA_ERROR;
    return allreduce_dev(ctx, ctx->sc + s0, 1);
  }
  int finalize2(int nparts, int s0, int s1) {   // s1 == s0 + 1
    finalize<2>(nparts, s0, s1);
    if (cudaGetLastError() != cudaSuccess) return ISC_CUDA_ERROR;
    return allreduce_dev(ctx, ctx->sc + s0, 2);
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
static int bicgstab_schur(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  const int64_t len = (int64_t)NU * ctx->g.n;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  Kry K{ctx, len};
  double *b = ctx->rhs, *x = ctx->xk, *r = ctx->rk, *rhat = ctx->rhat, *p = ctx->pk,
         *v = ctx->vk, *phat = ctx->phat, *shat = ctx->shat, *s = ctx->sk, *t = ctx->tk;
  const double* uinv = ctx->mc_uinv;
  const int bh = grid1d(g.tw_hi - g.tw_lo, 32);   // blocks of a half pass (owned planes)
  CK(cudaMemsetAsync(x, 0, len * 8, st));
  TRY(K.dot(b, b, S_BB));   // ||b|| of the full decoupled rhs (the reference's tolerance base)
  TRY(K.read_scalars());
  const double nb = std::sqrt(ctx->sc_h[S_BB]);
  *iters = 0;
  if (nb == 0.0) return ISC_OK;
  const double brk = 1e-30 * nb * nb;
  // p, v and t need no clearing: p and v are read only after the first
  // iteration wrote them (S_FIRST), t only where the black pass wrote it
  if (ctx->compact && ctx->gb_fresh) {
    ctx->gb_fresh = false;   // g_b already in r and rhat (k_mc_factor_compact)
  } else {
    TRY(halo_exchange(ctx, b, NU));   // slabs: red neighbours on other ranks
    {
      KScope ks(ctx, KT_SPMV);
      sc_rhs_launch(ctx, g, bh, b, r, rhat);   // g_b
    }
    ++ctx->launches;
  }
  double* sh = ctx->sc_h;
  for (int i = 0; i < S_NSCAL; ++i) sh[i] = 0.0;
  sh[S_RHO_OLD] = 1.0; sh[S_ALPHA] = 1.0; sh[S_OMEGA] = 1.0; sh[S_FIRST] = 1.0;
  sh[S_BB] = nb * nb;
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
  auto red_pass = [&](double* z, const double* stop) -> int {
    if (!split) {
      TRY(halo_exchange(ctx, z, NU));
      sc_red_launch(ctx, g, bh, z, stop);
      ++ctx->launches;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    TRY(halo_start(ctx, z, NU));
    sc_red_launch(ctx, gi, bi, z, stop);
    TRY(halo_finish(ctx, z, NU));
    sc_red_launch(ctx, gl, bl1, z, stop);
    sc_red_launch(ctx, gh, bh1, z, stop);
    ctx->launches += 3;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto black_pass = [&](int K, double* z, double* vout, const double* w0,
                        const double* w1, const double* stop) -> int {
    auto launch = [&](const Dims& d, int blocks, int slot0) {
      if (K == 1)
        sc_black_launch<1>(ctx, d, blocks, z, vout, w0, w1, bparts, slot0, stop);
      else
        sc_black_launch<2>(ctx, d, blocks, z, vout, w0, w1, bparts, slot0, stop);
    };
    if (!split) {
      TRY(halo_exchange(ctx, z, NU));
      launch(g, bh, 0);
      ++ctx->launches;
      return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
    }
    TRY(halo_start(ctx, z, NU));
    launch(gi, bi, 0);
    TRY(halo_finish(ctx, z, NU));
    launch(gl, bl1, bi);
    launch(gh, bh1, bi + bl1);
    ctx->launches += 3;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto dot_b = [&](const double* a, const double* c, int slot) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_dot<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, a, c, ctx->partial);
    ++ctx->launches;
    return K.finalize1(RED_BLOCKS, slot);
  };
  auto finish = [&]() -> int {   // x_r = b_r - B_rb x_b
    if (halo_exchange(ctx, x, NU)) return ISC_CUDA_ERROR;
    KScope ks(ctx, KT_SPMV);
    sc_xred_launch(ctx, g, bh, b, x);
    ++ctx->launches;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  TRY(K.push());
  TRY(dot_b(rhat, r, S_RHO_NEW));
  TRY(K.read_scalars());
  auto restart = [&]() -> int {
    // r_b = g_b - S x_b; rhat = r; p = v = 0 (linsolve.py:509-519)
    {
      KScope ks(ctx, KT_SPMV);
      if (red_pass(x, nullptr)) return ISC_CUDA_ERROR;   // red part of x: scratch
      if (black_pass(1, x, t, rhat, nullptr, nullptr)) return ISC_CUDA_ERROR;
      sc_rhs_launch(ctx, g, bh, b, v, shat);   // g_b (scratch)
    }
    k_sc_sub<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, v, t, r, rhat);
    ctx->launches += 4;
    cudaMemsetAsync(p, 0, len * 8, st);
    cudaMemsetAsync(v, 0, len * 8, st);
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
  sh[S_STOP] = STOP_RUN;
  sh[S_IT] = 0.0;
  sh[S_MAXIT] = (double)maxiter;
  sh[S_NB] = nb;
  sh[S_TOL] = tol;
  sh[S_BRK] = brk;
  TRY(K.push());
  auto enqueue_iteration = [&]() -> int {
    k_bicg_top<<<1, 1, 0, st>>>(ctx->sc);
    {
      KScope ks(ctx, KT_VEC);
      k_sc_update_p<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, p, v, uinv, phat, ctx->sc, stop);
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
    TRY(K.finalize1(bparts * sc_warps(ctx), S_DEN));
    k_bicg_den<<<1, 1, 0, st>>>(ctx->sc);
    {
      KScope ks(ctx, KT_VEC);
      k_sc_update_s<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, v, s, uinv, shat, ctx->sc,
                                                        ctx->partial, stop);
    }
    TRY(K.finalize1(RED_BLOCKS, S_SS));
    k_bicg_ss<<<1, 1, 0, st>>>(ctx->sc);
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
      k_sc_update_xr<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, x, phat, shat, r, s, t, rhat,
                                                         ctx->sc, ctx->partial, stop);
    }
    TRY(K.finalize2(RED_BLOCKS, S_RR, S_RHO_NEW));
    k_bicg_end<<<1, 1, 0, st>>>(ctx->sc);
    ctx->launches += 7;   // 3 vector updates + 4 control kernels (passes and sums count themselves)
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
    ctx->bicg_last_iters = it;
    if (code == STOP_CONV_S) {   // ||s|| / ||b|| <= tol: x += alpha phat (linsolve.py:550-552)
      sh[S_STOP] = STOP_RUN;
      TRY(K.push());
      k_sc_axpy_alpha<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, x, phat, ctx->sc);
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

// Restarted right-preconditioned GMRES(m) on the red-eliminated system
// S x_b = g_b with U_b block-Jacobi (the north star's "BiCGSTAB/GMRES";
// optional, isc_set_krylov). Arnoldi with classical Gram-Schmidt and one
// reorthogonalisation (CGS2): two fused multi-dots and two multi-axpys per
// step, the second one also giving ||w||; the Hessenberg column goes to the
// host once per step for the Givens rotations. One product S U_b^-1 per
// iteration (BiCGSTAB: two). Stopping test as bicgstab_schur: ||r|| / ||b||
// of the full system (the Givens residual estimate within a cycle, the true
// reduced residual at each restart).
static int gmres_schur(isc_ctx* ctx, double tol, int maxiter, int* iters) {
  const int64_t len = (int64_t)NU * ctx->g.n;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  Kry K{ctx, len};
  const int m = std::max(1, std::min(ctx->gm_m, GM_MAXV - 1));
  if (!ctx->gm_V) {
    if (cudaMalloc(&ctx->gm_V, (size_t)GM_MAXV * len * 8) != cudaSuccess ||
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
  if (ctx->compact && ctx->gb_fresh) {   // g_b from the factorisation
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
      TRY(halo_exchange(ctx, zz, NU));
      sc_red_launch(ctx, g, bh, zz);
    }
    {
      KScope ks(ctx, KT_SPMV);
      TRY(halo_exchange(ctx, zz, NU));
      sc_black_launch<1>(ctx, g, bh, zz, out, zz, nullptr, bh, 0);
    }
    ctx->launches += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : ISC_CUDA_ERROR;
  };
  auto norm2_into = [&](const double* a, int slot) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_dot<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, a, a, ctx->partial);
    ++ctx->launches;
    return K.finalize1(RED_BLOCKS, slot);
  };
  auto multidot = [&](int nv, const double* w, double* hout) -> int {
    KScope ks(ctx, KT_VEC);
    k_sc_multidot<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, nv, w, ctx->partial);
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
      k_sc_scale<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, r, ctx->sc + S_RR, V);   // v0 = r / beta
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
        k_sc_precond<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, vj, uinv, z);
      }
      ++ctx->launches;
      TRY(matvec(z, w));
      TRY(multidot(j + 1, w, h1));
      {
        KScope ks(ctx, KT_VEC);
        k_sc_multiaxpy<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j + 1, h1, 1.0, w, 0,
                                                           nullptr);
      }
      ++ctx->launches;
      TRY(multidot(j + 1, w, h2));
      {
        KScope ks(ctx, KT_VEC);
        k_sc_multiaxpy<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j + 1, h2, 1.0, w, 0,
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
        k_sc_scale<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, w, ctx->sc + S_TT, w);
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
      k_sc_multiaxpy<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, V, len, j, yd, -1.0, u, 1, nullptr);
      k_sc_precond<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, u, uinv, z);
      k_sc_add<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, z, x);
    }
    ctx->launches += 3;
    if (res / nb <= tol) break;
    // restart: r_b = g_b - S x_b
    CK(cudaMemcpyAsync(u, x, len * 8, cudaMemcpyDeviceToDevice, st));
    TRY(matvec(u, t));
    k_sc_sub<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, gb, t, r, z);
    ++ctx->launches;
    TRY(norm2_into(r, S_RR));
    TRY(K.read_scalars());
    beta = std::sqrt(ctx->sc_h[S_RR]);
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

// 0: not decoupled, 1: explicit decoupled blocks, 2: compact form (compact.cu)
extern "C" int isc_decoupled_form(const isc_ctx* ctx) {
  return !ctx->decoupled ? 0 : (ctx->compact ? 2 : 1);
}

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
  if (!ctx->decoupled) {
    int s = isc_decouple(ctx, bad_cell, bad_col);
    if (s) return s;
  } else {
    double wbad = 0.0;
    for (int w = 0; w < ctx->nw; ++w) {
      const double dwdb = ctx->wout_h[w * WOUT + 1];
      if (dwdb == 0.0 || !std::isfinite(dwdb)) wbad = 1.0;
    }
    double flags2[2] = {wbad, ctx->dc_bad_cell >= 0 ? 1.0 : 0.0};
    {
      int as = isc_comm_allreduce_host(ctx, flags2, 2, 1);
      if (as) return as;
    }
    if (flags2[0] > 0.0) {
      if (bad_cell) *bad_cell = -1;
      if (bad_col) *bad_col = -1;
      g_err = "well equation has a zero bhp derivative";
      return ISC_SINGULAR_CELL_BLOCK;
    }
    if (flags2[1] > 0.0 && ctx->dc_bad_cell < 0) {
      if (bad_cell) *bad_cell = -1;
      if (bad_col) *bad_col = -1;
      g_err = "diagonal block is singular on another rank";
      return ISC_SINGULAR_CELL_BLOCK;
    }
    if (ctx->dc_bad_cell >= 0) {
      if (bad_cell) *bad_cell = ctx->dc_bad_cell;
      if (bad_col) *bad_col = ctx->dc_bad_col;
      g_err = "diagonal block is singular";
      return ISC_SINGULAR_CELL_BLOCK;
    }
  }
  if (!ctx->factored) {
    int s = isc_precond_setup(ctx, bad_cell);
    if (s) {
      if (bad_col) *bad_col = -1;
      return s;
    }
  }
  int it = 0;
  STAGE(stage_begin(ctx, 3));
  const bool schur = MC_SCHUR && ctx->mc_schur && ctx->precond == ISC_PRECOND_MCILU &&
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
  // bhp back-substitution dbhp = -(r_w + wrow . du_c) / dwdb (linsolve.py:473-478)
  if (ctx->nw > 0 && h_dbhp) {
    std::vector<double> duc(NU);
    for (int w = 0; w < ctx->nw; ++w) {
      const int64_t c = ctx->wpos_h[w];
      for (int u = 0; u < NU; ++u)
        CK(cudaMemcpyAsync(&duc[u], ctx->xk + (int64_t)u * n + c, 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      const double* o = ctx->wout_h + w * WOUT;
      double dotv = 0.0;
      for (int u = 0; u < NU; ++u) dotv += o[2 + u] * duc[u];
      const double s = o[0] + dotv;
      h_dbhp[w] = -s / o[1];
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
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
