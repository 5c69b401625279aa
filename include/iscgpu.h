/*
 * iscgpu — C-ABI of the B200 (sm_100a) Newton hot path for the fully
 * implicit in-situ combustion simulator of arxiv 1811.11992 (reference
 * package `iscsim`, Python + numba).
 *
 * One shared library (paper_1811_11992_b200/_lib/libiscgpu.so), plain
 * pointers and sizes, no torch types. Pointers named d_* are device (HBM)
 * pointers; h_* are host pointers. Vectors and states are structure-of-arrays
 * over cells: v[u*n + c] with u in the reference's unknown order
 * [p, x_0..x_{nco-1}, y_0..y_{ncg-1}, T, S_w, S_g, C_c] (_kernels.py:11-16).
 * Every call returns an isc_status; ISC_OK == 0.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/iscsim):
 *   isc_assemble        assembly.assemble            assembly.py:561-598
 *                       (cell_pass/compose_pass/conn_pass/gather_pass,
 *                        _kernels.py:613-854; _well_pass assembly.py:474-527)
 *   isc_export_system   Workspace.resid/diag/offd    assembly.py:315-317
 *   isc_import_system   (caller-provided ws arrays for BlockSolver.solve)
 *   isc_solve           BlockSolver.solve            linsolve.py:438-479
 *                       (_eliminate_wells 362-394, _decouple_pass 126-152,
 *                        _factor 398-408, _bicgstab 481-578)
 *   isc_spmv            BlockSolver._matvec          linsolve.py:425-434
 *   isc_precond_apply   BlockSolver._apply_precond   linsolve.py:410-421
 *   isc_newton_update   newton.apply_update          newton.py:92-121
 *   isc_scaled_norm     newton.scaled_norm (cells)   newton.py:124-144
 *   isc_audit_sums      Simulator.audit_step (sums)  newton.py:339-366
 *   isc_synth_system    (BASELINE config 5 generator; paper_1811_11992_b200/synth.py)
 *   isc_numeric_jacobian assembly._numeric_jacobian  assembly.py:843-939
 *   isc_format_cells    report.write_frame (cells)   report.py:115-149
 *   isc_format_double   report._fmt (repr(float))    report.py:76-77
 *   isc_comm_nccl / isc_comm_hub   z-slab multi-GPU transport (the reference
 *                       has no multi-GPU path)
 */
#ifndef ISCGPU_H
#define ISCGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ISC_OK = 0,
  ISC_PORE_SPACE_EXHAUSTED = 1, /* errors.PoreSpaceExhausted  (assembly.py:548-552) */
  ISC_SINGULAR_CELL_BLOCK = 2,  /* errors.SingularCellBlock   (linsolve.py:372-375,405-408,458-463) */
  ISC_BREAKDOWN = 3,            /* errors.Breakdown           (linsolve.py:503-569) */
  ISC_MAX_ITERATIONS = 4,       /* errors.MaxIterations       (linsolve.py:576-578) */
  ISC_BAD_ARGUMENT = 10,
  ISC_CUDA_ERROR = 11,
  ISC_UNSUPPORTED = 12
} isc_status;

/* none / bjacobi / ras reproduce the reference (linsolve.py:322-358); mcilu is
 * the red-black multicolour block ILU(0) of BASELINE's north_star, solved on
 * the red-eliminated system (same stopping test on the full residual). */
typedef enum {
  ISC_PRECOND_NONE = 0, ISC_PRECOND_BJACOBI = 1, ISC_PRECOND_RAS = 2, ISC_PRECOND_MCILU = 3
} isc_precond;

/* Krylov method on the mcilu red-eliminated system: the reference's
 * BiCGSTAB control flow (default; linsolve.py:481-578) or restarted
 * right-preconditioned GMRES(m) (north_star "BiCGSTAB/GMRES"; same
 * preconditioner, same stopping test ||r||/||b|| <= tol). Other
 * preconditioners always run BiCGSTAB. */
typedef enum { ISC_KRYLOV_BICGSTAB = 0, ISC_KRYLOV_GMRES = 1 } isc_krylov;

typedef struct isc_ctx isc_ctx;

/* Flattened model constants: the reference's ModelPack (assembly.py:42-68),
 * host pointers to row-major float64 / int64 arrays. */
typedef struct {
  int64_t nco, ncg, heavy, nreac, nswt, nslt;
  const double *liq;   /* (1+nco, 10) */
  const double *gasp;  /* (nfull, 9)  */
  const double *kv;    /* (1+nco, 5)  */
  const double *rockp; /* (17)        */
  const double *swt_s, *swt_krw, *swt_krow, *swt_pcow; /* (nswt) */
  const double *slt_s, *slt_krg, *slt_krog, *slt_pcog; /* (nslt) */
  const int64_t *law;  /* (nreac) */
  const double *rcoef; /* (nreac, 3) */
  const double *nmat;  /* (nfull+1, nreac) */
  const int64_t *fuel, *ox; /* (nreac) */
  double ccmax;
} isc_model_desc;

/* Structured grid (grid.py:20-57). Per-cell host arrays of length n;
 * gd/td are (3, n): Darcy factor DARCY_CONST*conn_geom and thermal factor
 * of the +x/+y/+z face owned by each cell (0 where no face); conn_id (3, n)
 * the reference's connection index of that face or -1; hl_area may be NULL. */
typedef struct {
  int32_t nx, ny, nz;
  const double *depth, *volume, *phi_ref;
  const double *gd, *td;
  const int64_t *conn_id;
  const double *hl_area;
  double hl_kob, hl_d, hl_rho, hl_tini;
  int32_t k_offset; /* global index of local plane 0 (z-slabs; 0 otherwise): the
                     * red/black colour is (i + j + k_global) & 1 on every rank */
} isc_grid_desc;

/* One single-perforation well (wells.py:36-54) and its injector stream
 * constants (assembly.py:222-231; zeros for producers). */
typedef struct {
  int64_t cell;
  int32_t kind;    /* 0 injector, 1 producer */
  int32_t control; /* 0 bhp, 1 rate_gas, 2 rate_total */
  double target, wi, z_bh, pinjmax, heat_rate, heat_stop;
  double s_yfull[5], s_yinj[2], s_tinj, s_mu, s_h, s_mbar;
} isc_well_desc;

/* Per-well assembly output, ISC_WELL_OUT doubles per well:
 * [resid, dwdb, wrow(9), bcol(9), phase_rates(3), comp_rates(9)]
 * (WellBlock, assembly.py:348-363). */
#define ISC_WELL_OUT 32
#define ISC_NREC 85

int isc_create(const isc_model_desc *model, const isc_grid_desc *grid, int32_t nwells,
               const isc_well_desc *wells, int32_t precond, isc_ctx **out);
int isc_destroy(isc_ctx *ctx);
const char *isc_last_error(void);
int isc_block_size(void); /* 9 */

/* Residual + analytic Jacobian at d_state (SoA 9 x n). h_bhp/h_capped: nwells.
 * d_accn SoA 9 x n. freeze: reuse stored upwind flags (newton.py:279).
 * h_wells_out receives nwells*ISC_WELL_OUT doubles. On
 * ISC_PORE_SPACE_EXHAUSTED *bad_cell is the lowest such cell. */
int isc_assemble(isc_ctx *ctx, const double *d_state, const double *h_bhp, const double *d_accn,
                 double dt, double t_new, const uint8_t *h_capped, int32_t freeze,
                 double *h_wells_out, int64_t *bad_cell);

/* isc_assemble with the reference's host layout (assembly.py:179-196 State
 * arrays and accn (n, 9)); d_state == NULL in isc_assemble means "already
 * staged by this call". Pinned host arrays give full PCIe bandwidth. */
int isc_assemble_host(isc_ctx *ctx, const double *h_p, const double *h_x, const double *h_y,
                      const double *h_t, const double *h_sw, const double *h_sg,
                      const double *h_cc, const double *h_bhp, const double *h_accn, double dt,
                      double t_new, const uint8_t *h_capped, int32_t freeze,
                      double *h_wells_out, int64_t *bad_cell);
/* du of the last isc_solve (called with d_du == NULL) as host (n, 9). */
int isc_download_du(isc_ctx *ctx, double *h_du);

/* JACOBIAN numeric (assembly.py:593-597, 843-939; replaces the reference's
 * _numeric_jacobian): every Jacobian block and the well rows (wrow), bhp
 * columns (bcol) and dwdb of the last isc_assemble / isc_assemble_host are
 * replaced by central finite differences at the same inputs (probe points of
 * _fd_points, assembly.py:807-840); residuals keep the analytic pass's values.
 * h_wells_out as in isc_assemble. ISC_PORE_SPACE_EXHAUSTED if a probed state
 * exhausts the pore space (assembly.py:682-684), *bad_cell = lowest cell. */
int isc_numeric_jacobian(isc_ctx *ctx, double *h_wells_out, int64_t *bad_cell);

/* Copy an internal per-cell array to d_dst: 0 resid (9 x n), 1 acc (9 x n),
 * 2 src (9 x n), 3 yfull (5 x n), 4 record (ISC_NREC x n), 5 upwind flags
 * int8 (3 axes x 3 phases x n). */
int isc_copy_out(isc_ctx *ctx, int32_t what, void *d_dst);

/* Assembled (pre-decoupling) system in the reference layout:
 * diag (n,9,9), offd (m,2,9,9), resid (n,9). */
int isc_export_system(isc_ctx *ctx, double *d_diag, double *d_offd, double *d_resid);
/* Load a caller's system (reference layout) + well outputs for isc_solve. */
int isc_import_system(isc_ctx *ctx, const double *d_diag, const double *d_offd,
                      const double *d_resid, const double *h_wells_out);
/* Replace the well outputs used by the next isc_solve (WellBlock data). */
int isc_set_wells_out(isc_ctx *ctx, const double *h_wells_out);
/* Switch preconditioner (rebuilds the subdomain/level structure). */
int isc_set_precond(isc_ctx *ctx, int32_t precond);
/* Form of the decoupled system held by the context: 0 not decoupled,
 * 1 explicit D^-1 B_d blocks (the reference's, linsolve.py:130-152),
 * 2 compact (mcilu on an assembled system: raw flux rows of B_d and
 * D^-1[:, :6], the same operator). */
int isc_decoupled_form(const isc_ctx *ctx);
/* 1 when the current multicolour factorisation is the condensed one (the
 * red-eliminated BiCGSTAB / GMRES on 6-component vectors after eliminating
 * each cell's local constraint rows, compact.cu; ISC_COND != 0), else 0. No reference counterpart (an internal form of
 * linsolve.BlockSolver.solve, linsolve.py:438-479). */
int isc_condensed(const isc_ctx *ctx);
/* Select the Krylov method (isc_krylov); restart = GMRES restart length
 * 1..31 (0 keeps the current, default 30). No reference counterpart: an
 * extension of linsolve.BlockSolver's solve (linsolve.py:481-578). */
int isc_set_krylov(isc_ctx *ctx, int32_t krylov, int32_t restart);
/* Generate the seeded synthetic system of BASELINE config 5 in place. */
int isc_synth_system(isc_ctx *ctx, uint64_t seed);

/* Same, for a z-slab context (grid k_offset = global index of local plane 0)
 * of a global grid with nz_global planes: every value is keyed by the global
 * cell index and z-faces follow the global boundary, so each rank holds its
 * rows of the single-GPU system bit for bit. nz_global <= 0: k_offset + nz. */
int isc_synth_system_slab(isc_ctx *ctx, uint64_t seed, int32_t nz_global);

/* Well Schur fold, GJ decoupling, preconditioner setup and BiCGSTAB on the
 * current system; d_du (SoA 9 x n) receives the cell update, h_dbhp the
 * nwells bhp updates. Status 2/3/4 as the reference's exceptions; for
 * status 2, *bad_cell/*bad_col identify the block (-1 when not a cell). */
int isc_solve(isc_ctx *ctx, double tol, int32_t maxiter, double *d_du, double *h_dbhp,
              int32_t *iters, int64_t *bad_cell, int32_t *bad_col);

/* isc_solve delivering du as the reference's BlockSolver.solve does
 * (linsolve.py:396-479: a host (n, 9) array in natural cell order; pinned
 * memory for an asynchronous copy). On the single-GPU condensed path the
 * solve's last kernels run per plane chunk with each chunk's copy under the
 * next chunk's kernels; otherwise isc_solve(d_du = NULL) + isc_download_du. */
int isc_solve_host(isc_ctx *ctx, double tol, int32_t maxiter, double *h_du, double *h_dbhp,
                   int32_t *iters, int64_t *bad_cell, int32_t *bad_col);
/* Decouple only (tests): leaves D^-1-scaled blocks/rhs inside the context
 * (the compact form for mcilu on an assembled system: isc_decoupled_form). */
int isc_decouple(isc_ctx *ctx, int64_t *bad_cell, int32_t *bad_col);
int isc_precond_setup(isc_ctx *ctx, int64_t *bad_cell);
int isc_spmv(isc_ctx *ctx, const double *d_x, double *d_y);
int isc_precond_apply(isc_ctx *ctx, const double *d_r, double *d_z);
/* decoupled rhs (after isc_decouple) -> d_dst (9 x n) */
int isc_copy_rhs(isc_ctx *ctx, double *d_dst);

/* Replace the decoupled right-hand side of a decoupled system (natural order,
 * SoA (9, n) device array); the next isc_solve refactors. Used by the C5
 * microbench's host-buffer leg (a new rhs per solve). */
int isc_set_rhs(isc_ctx *ctx, const double *d_src);

int isc_newton_update(isc_ctx *ctx, double *d_state, const double *d_du, double eps);
int isc_scaled_norm(isc_ctx *ctx, const double *d_accn, double dt, double *norm);
/* out[3*(nfull+1)]: per audited row sum V(acc-accn), sum V src, sum V|acc| */
int isc_audit_sums(isc_ctx *ctx, const double *d_accn, double *h_out);

/* ---- multi-GPU z-slab decomposition ----------------------
 * The context's grid holds the owned planes [kw_lo, kw_hi) plus one ghost
 * plane towards each neighbouring rank (has_lo / has_hi). Halos of the state
 * (before assembly) and of p-hat / s-hat / x (before each SpMV) and the
 * Krylov dot products / norms / audit sums cross ranks; the preconditioner is
 * rank-local (block-Jacobi across ranks of the multicolour ILU). NCCL: one
 * process per GPU, unique_id = 128-byte ncclUniqueId (e.g. broadcast by
 * torch.distributed). Hub: several contexts in one process, one host thread
 * per rank (single-GPU validation of the multi-rank algorithm). */
int isc_comm_nccl(isc_ctx *ctx, const void *unique_id, int32_t rank, int32_t nranks,
                  int32_t has_lo, int32_t has_hi, int32_t kw_lo, int32_t kw_hi);
int isc_nccl_unique_id(void *out128);   /* ncclGetUniqueId on the calling rank */
/* 1 when the context reduces / exchanges through an NCCL communicator (nranks > 1, or one
 * rank with ISC_NCCL_SINGLE=1 in the environment of isc_comm_nccl: transport check on one GPU) */
int isc_comm_is_nccl(isc_ctx *ctx);
void *isc_hub_create(int32_t nranks);
int isc_hub_destroy(void *hub);
int isc_comm_hub(isc_ctx *ctx, void *hub, int32_t rank, int32_t has_lo, int32_t has_hi,
                 int32_t kw_lo, int32_t kw_hi);
/* op 0 = sum, 1 = max, over ranks, in place on count (<= 64) host doubles */
int isc_comm_allreduce_host(isc_ctx *ctx, double *vals, int32_t count, int32_t op);

/* Stream used by every call (torch can wait on it); device sync helper. */
void *isc_stream(isc_ctx *ctx);
/* Issue all work on a caller's stream (e.g. torch's current stream); NULL
 * restores the context's own stream. */
int isc_set_stream(isc_ctx *ctx, void *stream);
int isc_synchronize(isc_ctx *ctx);
/* Kernel launches issued by this context since creation (bench accounting). */
int64_t isc_launch_count(isc_ctx *ctx);
/* Cumulative device milliseconds per stage measured with CUDA events:
 * out[0] assemble, [1] decouple, [2] precond setup, [3] krylov. */
int isc_stage_times(isc_ctx *ctx, double *out4);
/* Per-kernel-class device time from CUDA events recorded around every
 * launch while profiling is on: classes 0 cell, 1 face, 2 wells,
 * 3 decouple (rhs+Schur+GJ), 4 ILU factor, 5 ILU apply, 6 SpMV, 7 other. */
int isc_set_profiling(isc_ctx *ctx, int32_t on);
int isc_kernel_times(isc_ctx *ctx, double *ms8, int64_t *count8, int32_t reset);

/* ---- report frames (report.py:50-149), host only ----
 * Python repr(float(v)) of v: the shortest round-trip string, CPython's
 * layout rules (report.py:76-77 _fmt). out32 >= 32 bytes; returns length. */
int isc_format_double(double v, char *out32);
/* The cells.csv rows of one frame (report.py:131-138), byte-identical with
 * the reference's writer: "time,cell,p,T,S_w,S_o,S_g,x_*,y_*,C_c" per cell,
 * S_o = 1.0 - S_w - S_g. x[c*x_cell_stride + i*x_comp_stride] (i < nco),
 * y likewise (nf entries, the full gas composition). Formatted on `threads`
 * host threads; *out is malloc'ed (release with isc_free), *len bytes. */
int isc_format_cells(double time, int64_t n, const double *p, const double *t,
                     const double *sw, const double *sg, const double *x,
                     int64_t x_cell_stride, int64_t x_comp_stride, int32_t nco,
                     const double *y, int64_t y_cell_stride, int64_t y_comp_stride, int32_t nf,
                     const double *cc, int32_t threads, char **out, int64_t *len);
void isc_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* ISCGPU_H */
