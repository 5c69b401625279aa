// Host runtime shared by the C-ABI translation unit (capi.cu): the context
// (isc_ctx: device buffers, streams, the z-slab window), error reporting, the
// per-kernel-class CUDA-event timers and the stage timers.
#pragma once
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
#include "comm.cuh"
#include "newton.cu"
#include "numjac.cu"
#include "report.cuh"
#include "solver.cu"
#include "compact.cu"

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
  cudaEvent_t chunk_ev[32] = {};
  cudaStream_t stream2 = nullptr;          // second compute stream of the staged assembly (alternate chunks)
  cudaEvent_t cell_ev[32] = {}, face_ev[32] = {};   // chunk q's cell pass / face evaluation done
  cudaEvent_t halo_ev[2] = {};             // halo planes packed / landed
  bool cell_pre = false;                   // k_cell already ran (pipelined host staging)
  bool face_pre = false;                   // k_face_eval too
  bool gather_pre = false;                 // and k_face_gather
  double* h_du = nullptr;                  // isc_solve_host: du streamed to this host array by the solve
  bool h_du_queued = false;                // ... its copies are on cstream
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
  // condensed form (compact.cu): the Krylov iteration on 6-component vectors
  bool cond_ok = true;    // ISC_COND=0 disables (A/B switch)
  bool cond_es = false;   // E_S of the black cells computed by the last decoupling
  bool cond = false;      // the current factorisation is the condensed one
  double* ces = nullptr;  // E_S (NCS*CR x half)
  double* cbc = nullptr;  // Bc_rd of the red cells (NDIR*CR*CR x half)
  double* cg9 = nullptr;  // reduced rhs g_b (9 x n), kept for x_b = g_b + E_b w
  double* ch6 = nullptr;  // condensed rhs h (CR x n)
  int* cfail_d = nullptr;
  int* cfail_h = nullptr;  // pinned
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
  unsigned* ticket_d = nullptr; // last-block ticket of k_partial_sum_fin (zero between launches)
  double *wdu_d = nullptr, *wdu_h = nullptr;   // du of the perforated cells (dbhp)
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
  std::vector<Pending> pending;         // kernel-class event pairs (profiling)
  std::vector<Pending> stage_pending;   // stage event pairs (always; no sync to take them)
  cudaEvent_t stage_open[4] = {};
  bool stage_is_open[4] = {false, false, false, false};
  int stages_open = 0;                  // begun, not yet ended (their events stay reserved)
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
// fold the finished event pairs into the totals (pairs whose end event has
// not completed yet stay pending; the pool is recycled once none is left)
static void kflush(isc_ctx* ctx) {
  auto fold = [&](std::vector<isc_ctx::Pending>& v, double* ms_out, int64_t* n_out) {
    size_t keep = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      if (cudaEventQuery(v[i].b) != cudaSuccess) {
        cudaGetLastError();   // cudaErrorNotReady is not an error here
        v[keep++] = v[i];
        continue;
      }
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, v[i].a, v[i].b) == cudaSuccess) {
        ms_out[v[i].kind] += ms;
        if (n_out) n_out[v[i].kind] += 1;
      }
    }
    v.resize(keep);
  };
  fold(ctx->pending, ctx->kern_ms, ctx->kern_n);
  fold(ctx->stage_pending, ctx->stage_ms, nullptr);
  if (ctx->pending.empty() && ctx->stage_pending.empty() && ctx->stages_open == 0)
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

// stage timers (assemble / decouple / preconditioner setup / Krylov): event
// pairs on the stream, folded at the next synchronisation -- taking a time
// never adds one
static int stage_begin(isc_ctx* ctx, int st) {
  ctx->stage_open[st] = pool_event(ctx);
  if (!ctx->stage_is_open[st]) ++ctx->stages_open;   // (an error path may skip an end)
  ctx->stage_is_open[st] = true;
  CK(cudaEventRecord(ctx->stage_open[st], ctx->stream));
  return ISC_OK;
}
static int stage_end(isc_ctx* ctx, int st) {
  cudaEvent_t b = pool_event(ctx);
  CK(cudaEventRecord(b, ctx->stream));
  ctx->stage_pending.push_back({st, ctx->stage_open[st], b});
  if (ctx->stage_is_open[st]) --ctx->stages_open;
  ctx->stage_is_open[st] = false;
  return ISC_OK;
}
// synchronise the context's stream and fold the timers
static int sync_stream(isc_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  kflush(ctx);
  return ISC_OK;
}
#define STAGE(call) do { int s_ = (call); if (s_) return s_; } while (0)
