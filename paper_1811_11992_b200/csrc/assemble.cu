// Residual + analytic Jacobian assembly on sm_100a (fp64).
//
//   k_cell   one thread per cell: porosity, phase properties, modified-PER
//            K-values, RK Z-factor, mobilities, enthalpies, accumulation,
//            constraint rows, Arrhenius reactions and the cell-local
//            (V/dt)(acc-accn) - V*src composition (+ heat loss).
//            Restates _kernels.py:66-610 and 797-825.
//   k_face   one thread per (cell, residual row): the cell's six faces in
//            the reference's fixed gather order (-z,-y,-x,+x,+y,+z), each
//            face's flux row and both derivative rows (_kernels.py:642-771),
//            accumulated into the diagonal block row / residual and written
//            as the off-diagonal block rows (_kernels.py:828-854).
//   k_wells  Peaceman perforation rows, bhp column, heater and the well
//            equation (assembly.py:370-527), one thread, wells in order.
//
// Device layout (SoA, cell index fastest so every warp access coalesces):
//   state  st[u*n + c]            (u in unknown order)
//   resid  resid[r*n + c]
//   diag   diag[(r*NU + u)*n + c]
//   offd   offd[((d*NU + r)*NU + u)*n + c]   block (row c, column nb_d(c))
//   rec    rec[f*n + c]            (record.cuh)
// Compiled with --fmad=false so the arithmetic follows the reference's
// unfused operation order (parity bar: 1e-10 row-scaled).
#include "common.cuh"
#include "props.cuh"
#include "record.cuh"

namespace isc {

// -------------------------------------------------------------------- cell

struct CellArgs {
  Dims g;
  const double* __restrict__ st;
  const double* __restrict__ phi_ref;
  const double* __restrict__ vol;
  const double* __restrict__ hl_area;  // nullable
  double hl_kob, hl_d, hl_rho, hl_tini;
  const double* __restrict__ accn;     // SoA NU x n
  double dt;
  double* __restrict__ rec;
  double* __restrict__ acc;            // SoA NU x n
  double* __restrict__ src;            // SoA NU x n
  double* __restrict__ resid;
  double* __restrict__ diag;
  unsigned long long* bad;             // min index of a pore-space-exhausted cell
  int64_t c_begin, c_end;              // positions handled by k_cell (pipelined staging)
  double* __restrict__ mid = nullptr;  // NMID x n: property values for k_cell_rows (split pass)
};

// Where one cell evaluation's outputs go. The analytic pass stores them in
// the workspace arrays; a finite-difference probe keeps the record fields
// and residual rows in registers and drops every analytic partial (dead code
// after inlining).
struct CellSinkGlobal {
  static constexpr bool kMidOut = false, kUnroll = false, kSplitGas = false;
  const CellArgs& A;
  int64_t n, c;
  __device__ double& rec(int f) { return A.rec[(int64_t)f * n + c]; }
  __device__ void acc(int r, double v) { A.acc[r * n + c] = v; }
  __device__ void src(int r, double v) { A.src[r * n + c] = v; }
  __device__ void diag(int r, int u, double v) { A.diag[(int64_t)(r * NU + u) * n + c] = v; }
  __device__ void resid(int r, double v) { A.resid[r * n + c] = v; }
  __device__ void fail() { atomicMin(A.bad, (unsigned long long)cell_of(A.g, c)); }
};

#ifndef PROBE_UNROLL
#define PROBE_UNROLL true   // numeric Jacobian at C4: 72 -> 30.5 ms unrolled
#endif
struct CellSinkProbe {
  static constexpr bool kMidOut = false, kUnroll = PROBE_UNROLL, kSplitGas = false;
  double v[NREC];      // record fields at the probed state
  double rows[NU];     // residual rows of the cell part (compose)
  bool failed = false;
  __device__ double& rec(int f) { return v[f]; }
  __device__ void acc(int, double) {}
  __device__ void src(int, double) {}
  __device__ void diag(int, int, double) {}
  __device__ void resid(int r, double x) { rows[r] = x; }
  __device__ void fail() { failed = true; }
  __device__ double f(int k) const { return v[k]; }   // record accessor (flux, wells)
};

// The property half of the split cell pass: the record and the values the
// reaction / accumulation rows need (A.mid), nothing else.
struct CellSinkProps {
  static constexpr bool kMidOut = true, kUnroll = false, kSplitGas = true;   // the gas phase runs in k_cell_gas
  const CellArgs& A;
  int64_t n, c;
  __device__ double& rec(int f) { return A.rec[(int64_t)f * n + c]; }
  __device__ void mid(int f, double v) { A.mid[(int64_t)f * n + c] = v; }
  __device__ void acc(int, double) {}
  __device__ void src(int, double) {}
  __device__ void diag(int, int, double) {}
  __device__ void resid(int, double) {}
  __device__ void fail() { atomicMin(A.bad, (unsigned long long)cell_of(A.g, c)); }
};

// dyfull (NF x NU) with its structure (_kernels.py:220-252): the water row
// has d/dp, d/dT, d/dSw; oil row i has d/dp, d/dT, d/dx_i, d/dSw, d/dSg (the
// last two non-zero for the heaviest oil only); gas row a is the unit vector
// of its own column. 13 stored values instead of 45, so the cell kernel keeps
// them in registers; dy(a, u) and nz(a, u) fold at compile time in unrolled
// loops, and the sums skip the structural zeros (the reference adds +-0).
struct DyFull {
  double w[3];
  double o[NCO][5];
  __device__ __forceinline__ double operator()(int a, int u) const {
    if (a == 0) return u == 0 ? w[0] : (u == CT ? w[1] : (u == CSW ? w[2] : 0.0));
    if (a < 1 + NCO) {
      const int i = a - 1;
      return u == 0 ? o[i][0]
                    : (u == CT ? o[i][1]
                               : (u == 1 + i ? o[i][2]
                                             : (u == CSW ? o[i][3] : (u == CSG ? o[i][4] : 0.0))));
    }
    return u == a ? 1.0 : 0.0;
  }
  __host__ __device__ static constexpr bool nz(int a, int u) {
    return a == 0 ? (u == 0 || u == CT || u == CSW)
                  : (a < 1 + NCO ? (u == 0 || u == CT || u == a || u == CSW || u == CSG)
                                 : u == a);
  }
};

// Values of the property pass that the reaction / accumulation rows use
// besides the record: stored per cell by k_cell_props for k_cell_rows
// (mid[f*n + c]), or kept in registers when one thread does both (probes).
enum MidField {
  MI_PHI, MI_DPHI_P, MI_DPHI_T, MI_PHIF, MI_DPHIF_CC, MI_PCOG, MI_RO, MI_DRO_P, MI_DRO_T,
  MI_DRO_X, MI_RG = MI_DRO_X + NCO, MI_DRG, MI_RW = MI_DRG + NU, MI_DRW_P, MI_DRW_T, MI_UW,
  MI_DUW_P, MI_DUW_T, MI_UO, MI_DUO_P, MI_DUO_T, MI_UG, MI_DUG, NMID = MI_DUG + NU
};
struct CellMid {   // register form
  double v[NMID];
  DyFull dyf;
  double yf[NF], dpcog, hli[NCO];
};

// Reactions, accumulation rows and the cell-local composition of one cell
// (_kernels.py:430-608, 797-825) from the property pass's values m.
template <class S, bool kUnroll = false>
__device__ __forceinline__ void cell_rows(const Model& M, const CellArgs& A, int64_t c,
                                          const double (&u_)[NU], const CellMid& m, S& s) {
  const int64_t n = A.g.n;
  const double* rk = M.rockp;
  const double p = u_[0], t = u_[CT], sw = u_[CSW], sg = u_[CSG], cc = u_[CCC];
  double x[NCO], y[NCG];
#pragma unroll
  for (int i = 0; i < NCO; ++i) x[i] = u_[1 + i];
#pragma unroll
  for (int j = 0; j < NCG; ++j) y[j] = u_[1 + NCO + j];
  const double so = 1.0 - sw - sg;
  const double t_ref = rk[RK_TREF];
  const double phi = m.v[MI_PHI], dphi_p = m.v[MI_DPHI_P], dphi_t = m.v[MI_DPHI_T];
  const double phif = m.v[MI_PHIF], dphif_cc = m.v[MI_DPHIF_CC];
  const double pcog = m.v[MI_PCOG], dpcog = m.dpcog;
  const double ro = m.v[MI_RO], dro_p = m.v[MI_DRO_P], dro_t = m.v[MI_DRO_T], ro2 = ro * ro;
  double dro_x[NCO], hli[NCO];
#pragma unroll
  for (int i = 0; i < NCO; ++i) { dro_x[i] = m.v[MI_DRO_X + i]; hli[i] = m.hli[i]; }
  const double rg = m.v[MI_RG];
  double drg[NU], dug[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) { drg[u] = m.v[MI_DRG + u]; dug[u] = m.v[MI_DUG + u]; }
  const double rw = m.v[MI_RW], drw_p = m.v[MI_DRW_P], drw_t = m.v[MI_DRW_T];
  const double uw = m.v[MI_UW], duw_p = m.v[MI_DUW_P], duw_t = m.v[MI_DUW_T];
  const double uo = m.v[MI_UO], duo_p = m.v[MI_DUO_P], duo_t = m.v[MI_DUO_T];
  const double ug = m.v[MI_UG];
  const DyFull dyf = m.dyf;
  double yf[NF];
#pragma unroll
  for (int a = 0; a < NF; ++a) yf[a] = m.yf[a];

  // reactions first (_kernels.py:537-608): r and d r / d u per reaction
  double rr_v[MAXREAC], rr_d[MAXREAC][NU];
  bool rr_on[MAXREAC];
  {
    const double pg = p + pcog;
    const double ccr = cc > 0.0 ? cc : 0.0;
auto react = [&](const int q) {
      rr_on[q] = false;
      rr_v[q] = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) rr_d[q][u] = 0.0;
      if (q >= M.nreac) return;
      double dpp[NU], dfm[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) { dpp[u] = 0.0; dfm[u] = 0.0; }
      const int oxi = M.ox[q];
      double pp = 0.0;
      if (oxi >= 0) {
        double y_ox = 0.0;
#pragma unroll
        for (int a = 0; a < NF; ++a) if (a == oxi) y_ox = yf[a];
        pp = y_ox * pg;
        if (pp > 0.0) {
#pragma unroll
          for (int a = 0; a < NF; ++a)
            if (a == oxi) {
#pragma unroll
              for (int u = 0; u < NU; ++u) dpp[u] = dyf(a, u) * pg;
            }
          dpp[0] += y_ox;
          dpp[CSG] += y_ox * dpcog;
        } else {
          pp = 0.0;
        }
      }
      const int fui = M.fuel[q];
      double fm = 0.0;
      if (fui >= 0) {
        double xf = 0.0;
#pragma unroll
        for (int i = 0; i < NCO; ++i) if (i == fui) xf = x[i];
        fm = phif * so * ro * xf;
        if (fm > 0.0) {
          const double base = so * ro * xf;
          dfm[0] = dphi_p * base + phif * so * dro_p * xf;
          dfm[CT] = dphi_t * base + phif * so * dro_t * xf;
          dfm[CSW] = -phif * ro * xf;
          dfm[CSG] = -phif * ro * xf;
          dfm[CCC] = dphif_cc * base;
#pragma unroll
          for (int i = 0; i < NCO; ++i) dfm[1 + i] = phif * so * dro_x[i] * xf;
#pragma unroll
          for (int i = 0; i < NCO; ++i) if (i == fui) dfm[1 + i] += phif * so * ro;
        } else {
          fm = 0.0;
        }
      }
      double o[5];
      reaction_rate_one(M.law[q], M.rcoef[q][0], M.rcoef[q][1], t, pp, fm, ccr, M.ccmax, o);
      if (o[0] == 0.0 && o[1] == 0.0 && o[2] == 0.0 && o[3] == 0.0 && o[4] == 0.0) return;
      rr_on[q] = true;
      rr_v[q] = o[0];
#pragma unroll
      for (int u = 0; u < NU; ++u) rr_d[q][u] = o[2] * dpp[u] + o[3] * dfm[u];
      rr_d[q][CT] += o[1];
      if (o[4] != 0.0 && cc >= 0.0) rr_d[q][CCC] += o[4];
        };
    if constexpr (kUnroll) {
#pragma unroll
      for (int q = 0; q < MAXREAC; ++q) react(q);
    } else {
#pragma unroll 1
      for (int q = 0; q < MAXREAC; ++q) react(q);
    }
  }

  // accumulation rows + composition, row by row (_kernels.py:430-535, 797-825)
  const double mw_g = rg * sg;
  const double vol = A.vol[c];
  const double vdt = vol / A.dt;
  double ur, dur_t;
  ur = rk[RK_CP1] * (t - t_ref) + 0.5 * rk[RK_CP2] * (t * t - t_ref * t_ref);   // _props.py:208-213
  dur_t = rk[RK_CP1] + rk[RK_CP2] * t;
  const double uc = rk[RK_COKE_CP] * (t - t_ref);
  const double duc_t = rk[RK_COKE_CP];
  const double hl = A.hl_area ? A.hl_area[c] : 0.0;

auto row = [&](const int r) {
    double accr, dacc[NU];
    if (r == 0) {
      const double a_w = rw * sw + mw_g * yf[0];
      accr = phif * a_w;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double d = (drg[u] * sg * yf[0] + mw_g * dyf(0, u));
        if (u == 0) d += drw_p * sw;
        else if (u == CT) d += drw_t * sw;
        else if (u == CSW) d += rw;
        if (u == CSG) d += rg * yf[0];
        dacc[u] = phif * d;
      }
      dacc[0] += dphi_p * a_w;
      dacc[CT] += dphi_t * a_w;
      dacc[CCC] += dphif_cc * a_w;
    } else if (r < 1 + NCO) {
      const int i = r - 1;
      const double a_i = ro * so * x[i] + mw_g * yf[r];
      accr = phif * a_i;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double d = drg[u] * sg * yf[r] + mw_g * dyf(r, u);
        if (u == 0) d += dro_p * so * x[i];
        else if (u == CT) d += dro_t * so * x[i];
        else if (u == CSW || u == CSG) d += -ro * x[i] + (u == CSG ? rg * yf[r] : 0.0);
        if (1 <= u && u < 1 + NCO) {
          d += dro_x[u - 1] * so * x[i];
          if (u - 1 == i) d += ro * so;
        }
        dacc[u] = phif * d;
      }
      dacc[0] += dphi_p * a_i;
      dacc[CT] += dphi_t * a_i;
      dacc[CCC] += dphif_cc * a_i;
    } else if (r < NF) {
      const int j = r - 1 - NCO;
      const double a_j = mw_g * y[j];
      accr = phif * a_j;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double d = drg[u] * sg * y[j];
        if (u == CSG) d += rg * y[j];
        if (u == 1 + NCO + j) d += mw_g;
        dacc[u] = phif * d;
      }
      dacc[0] += dphi_p * a_j;
      dacc[CT] += dphi_t * a_j;
      dacc[CCC] += dphif_cc * a_j;
    } else if (r == ROW_E) {
      const double a_e = rw * sw * uw + ro * so * uo + mw_g * ug;
      accr = phif * a_e + (1.0 - phi) * ur + cc * uc;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double d = drg[u] * sg * ug + mw_g * dug[u];
        if (u == 0) {
          d += drw_p * sw * uw + rw * sw * duw_p;
          d += dro_p * so * uo + ro * so * duo_p;
        } else if (u == CT) {
          d += drw_t * sw * uw + rw * sw * duw_t;
          d += dro_t * so * uo + ro * so * duo_t;
        } else if (u == CSW) {
          d += rw * uw - ro * uo;
        }
        if (u == CSG) d += -ro * uo + rg * ug;
        if (1 <= u && u < 1 + NCO) {
          const double duo_xi = hli[u - 1] + p * dro_x[u - 1] / ro2;
          d += dro_x[u - 1] * so * uo + ro * so * duo_xi;
        }
        dacc[u] = phif * d;
      }
      dacc[0] += dphi_p * a_e - dphi_p * ur;
      dacc[CT] += dphi_t * a_e - dphi_t * ur + (1.0 - phi) * dur_t + cc * duc_t;
      dacc[CCC] += dphif_cc * a_e + uc;
    } else if (r == ROW_OS) {
      double sx = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) dacc[u] = 0.0;
#pragma unroll
      for (int i = 0; i < NCO; ++i) { sx += x[i]; dacc[1 + i] = 1.0; }
      accr = sx - 1.0;
    } else if (r == ROW_GS) {
      double sy = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) dacc[u] = 0.0;
#pragma unroll
      for (int a = 0; a < NF; ++a) {
        sy += yf[a];
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (DyFull::nz(a, u)) dacc[u] += dyf(a, u);
      }
      accr = sy - 1.0;
    } else {  // coke
#pragma unroll
      for (int u = 0; u < NU; ++u) dacc[u] = 0.0;
      dacc[CCC] = 1.0;
      accr = cc;
    }
    // reaction source row r (stoichiometric row: nmat row r for r < NF,
    // nmat row NF for the coke row, heats for the energy row)
    double srcr = 0.0, dsrc[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) dsrc[u] = 0.0;
    if (r < NF || r == ROW_CK || r == ROW_E) {
#pragma unroll
      for (int q = 0; q < MAXREAC; ++q) {
        if (!rr_on[q]) continue;
        const double s = r < NF ? M.nmat[r][q] : (r == ROW_CK ? M.nmat[NF][q] : M.rcoef[q][2]);
        if (s != 0.0) {
          srcr += s * rr_v[q];
#pragma unroll
          for (int u = 0; u < NU; ++u) dsrc[u] += s * rr_d[q][u];
        }
      }
    }
    s.acc(r, accr);
    s.src(r, srcr);
    double res;
    if (r == ROW_OS || r == ROW_GS) {
      res = accr;
#pragma unroll
      for (int u = 0; u < NU; ++u) s.diag(r, u, dacc[u]);
    } else {
      res = vdt * (accr - A.accn[r * n + c]) - vol * srcr;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double dv = vdt * dacc[u] - vol * dsrc[u];
        if (r == ROW_E && u == ROW_E && hl > 0.0) dv += hl * A.hl_kob / A.hl_d;
        s.diag(r, u, dv);
      }
    }
    if (r == ROW_E && hl > 0.0) res += hl * A.hl_kob * ((t - A.hl_tini) / A.hl_d - A.hl_rho);
    s.resid(r, res);
    };
  if constexpr (kUnroll) {
#pragma unroll
    for (int r = 0; r < NU; ++r) row(r);
  } else {
#pragma unroll 1
    for (int r = 0; r < NU; ++r) row(r);
  }
}

// gas phase (_kernels.py:254-328): density, molar mass, viscosity and
// enthalpy of the gas with their partials
struct GasPhase {
  double rg, drg[NU], mgbar, dmg[NU], mug, dmug[NU], hg, dhg[NU], ug, dug[NU];
};
__device__ __forceinline__ void gas_phase(const Model& M, double p, double t, double t_ref,
                                          const double (&yf)[NF], const DyFull& dyf,
                                          GasPhase& G) {
  double dzdw[NF], dz_p, dz_t;
  const double z = z_factor_mix<NF>(yf, M.gasp, p, t, dzdw, dz_p, dz_t);
  double dz[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) dz[u] = 0.0;
  dz[0] = dz_p;
  dz[CT] += dz_t;
#pragma unroll
  for (int a = 0; a < NF; ++a)
    if (dzdw[a] != 0.0) {
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (DyFull::nz(a, u)) dz[u] += dzdw[a] * dyf(a, u);
    }
  const double tr = t + RANKINE;
  const double rg = p / (z * R_GAS * tr);
  double drg[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) drg[u] = -rg * dz[u] / z;
  drg[0] += rg / p;
  drg[CT] -= rg / tr;
  double mgbar = 0.0, dmg[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) dmg[u] = 0.0;
#pragma unroll
  for (int a = 0; a < NF; ++a) {
    mgbar += yf[a] * M.gasp[a][G_M];
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (DyFull::nz(a, u)) dmg[u] += M.gasp[a][G_M] * dyf(a, u);
  }
  double wsum = 0.0, musum = 0.0, dmusum_t = 0.0, sqm[NF], muc[NF];
#pragma unroll
  for (int a = 0; a < NF; ++a) {
    sqm[a] = sqrt(M.gasp[a][G_M]);
    double m_c, dm_c;
    gas_component_viscosity(M.gasp[a][G_AVG], M.gasp[a][G_BVG], t, m_c, dm_c);
    muc[a] = m_c;
    wsum += yf[a] * sqm[a];
    musum += yf[a] * m_c * sqm[a];
    dmusum_t += yf[a] * dm_c * sqm[a];
  }
  double dmug[NU], mug;
#pragma unroll
  for (int u = 0; u < NU; ++u) dmug[u] = 0.0;
  if (wsum > 1e-30) {
    mug = musum / wsum;
    dmug[CT] += dmusum_t / wsum;
#pragma unroll
    for (int a = 0; a < NF; ++a) {
      double dmy = sqm[a] * (muc[a] - mug) / wsum;
      if (dmy != 0.0) {
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (DyFull::nz(a, u)) dmug[u] += dmy * dyf(a, u);
      }
    }
  } else {
    mug = 1.0;
  }
  double hg = 0.0, dhg[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) dhg[u] = 0.0;
#pragma unroll
  for (int a = 0; a < NF; ++a) {
    double h_c, dh_c;
    gas_enthalpy(M.gasp[a], t_ref, t, h_c, dh_c);
    hg += yf[a] * h_c;
    dhg[CT] += yf[a] * dh_c;
    if (h_c != 0.0) {
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (DyFull::nz(a, u)) dhg[u] += h_c * dyf(a, u);
    }
  }
  const double ug = hg - p / rg;
  double dug[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) dug[u] = dhg[u] + p * drg[u] / (rg * rg);
  dug[0] -= 1.0 / rg;

  G.rg = rg; G.mgbar = mgbar; G.mug = mug; G.hg = hg; G.ug = ug;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    G.drg[u] = drg[u]; G.dmg[u] = dmg[u]; G.dmug[u] = dmug[u]; G.dhg[u] = dhg[u]; G.dug[u] = dug[u];
  }
}

// cell_eval + compose for the cell at position c with unknowns u_
// (_kernels.py:66-610, 797-825); inputs other than the unknowns from A.
template <class S>
__device__ __forceinline__ void cell_eval(const Model& M, const CellArgs& A, int64_t c,
                                          const double (&u_)[NU], S& s) {
  const int64_t n = A.g.n;
  const double* rk = M.rockp;
  const double p = u_[0], t = u_[CT], sw = u_[CSW], sg = u_[CSG], cc = u_[CCC];
  double x[NCO], y[NCG];
#pragma unroll
  for (int i = 0; i < NCO; ++i) x[i] = u_[1 + i];
#pragma unroll
  for (int j = 0; j < NCG; ++j) y[j] = u_[1 + NCO + j];
  const double so = 1.0 - sw - sg;

  // porosity and fluid porosity (_kernels.py:121-134)
  double phi, dphi_p, dphi_t;
  porosity(A.phi_ref[c], rk, p, t, phi, dphi_p, dphi_t);
  const double rho_coke = rk[RK_RHO_COKE];
  double phif, dphif_cc;
  if (rho_coke > 0.0 && isfinite(rho_coke)) { phif = phi - cc / rho_coke; dphif_cc = -1.0 / rho_coke; }
  else { phif = phi; dphif_cc = 0.0; }
  if constexpr (S::kMidOut) s.mid(MI_PHIF, phif);   // k_cell_rows skips failed cells
  if (phif <= 0.0) { s.fail(); return; }
  const double t_ref = rk[RK_TREF], eps_per = rk[RK_EPS_PER];
#define REC(f) s.rec(f)

  // water (_kernels.py:139-156)
  double rw, drw_p, drw_t, muw, dmuw_t, hgw, dhgw_t, hvw, dhvw_t;
  liquid_density(M.liq[0], rk[RK_PREF], t_ref, p, t, rw, drw_p, drw_t);
  liquid_viscosity(M.liq[0][L_AVISC], M.liq[0][L_BVISC], t, muw, dmuw_t);
  gas_enthalpy(M.gasp[0], t_ref, t, hgw, dhgw_t);
  vaporization_enthalpy(M.liq[0][L_HVR], M.liq[0][L_EV], M.liq[0][L_TCF], t, hvw, dhvw_t);
  const double hw = hgw - hvw, dhw_t = dhgw_t - dhvw_t;
  const double uw = hw - p / rw;
  const double duw_p = -1.0 / rw + p * drw_p / (rw * rw);
  const double duw_t = dhw_t + p * drw_t / (rw * rw);

  // oil (_kernels.py:158-218)
  double rho_i[NCO], drho_i_p[NCO], drho_i_t[NCO], mu_i[NCO], dmu_i_t[NCO], hli[NCO], dhli_t[NCO];
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
    liquid_density(M.liq[1 + i], rk[RK_PREF], t_ref, p, t, rho_i[i], drho_i_p[i], drho_i_t[i]);
    liquid_viscosity(M.liq[1 + i][L_AVISC], M.liq[1 + i][L_BVISC], t, mu_i[i], dmu_i_t[i]);
    double hg_i, dhg_i, hv_i, dhv_i;
    gas_enthalpy(M.gasp[1 + i], t_ref, t, hg_i, dhg_i);
    vaporization_enthalpy(M.liq[1 + i][L_HVR], M.liq[1 + i][L_EV], M.liq[1 + i][L_TCF], t, hv_i, dhv_i);
    hli[i] = hg_i - hv_i;
    dhli_t[i] = dhg_i - dhv_i;
  }
  double inv_ro = 0.0, dinv_p = 0.0, dinv_t = 0.0;
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
    inv_ro += x[i] / rho_i[i];
    dinv_p -= x[i] * drho_i_p[i] / (rho_i[i] * rho_i[i]);
    dinv_t -= x[i] * drho_i_t[i] / (rho_i[i] * rho_i[i]);
  }
  if (inv_ro < 1e-12) { inv_ro = 1e-12; dinv_p = 0.0; dinv_t = 0.0; }
  const double ro = 1.0 / inv_ro, ro2 = ro * ro;
  const double dro_p = -ro2 * dinv_p, dro_t = -ro2 * dinv_t;
  double lnmu = 0.0, dlnmu_t = 0.0;
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
    lnmu += x[i] * log(mu_i[i]);
    dlnmu_t += x[i] * dmu_i_t[i] / mu_i[i];
  }
  const double muo = exp(lnmu), dmuo_t = muo * dlnmu_t;
  double ho = 0.0, dho_t = 0.0;
#pragma unroll
  for (int i = 0; i < NCO; ++i) { ho += x[i] * hli[i]; dho_t += x[i] * dhli_t[i]; }
  const double uo = ho - p / ro;
  const double duo_p = -1.0 / ro + p * dro_p / ro2;
  const double duo_t = dho_t + p * dro_t / ro2;
  double dro_x[NCO];
#pragma unroll
  for (int i = 0; i < NCO; ++i) dro_x[i] = -ro2 / rho_i[i];

  // K-values -> yfull, dyfull (_kernels.py:220-252)
  double yf[NF];
  DyFull dyf;
#pragma unroll
  for (int i = 0; i < NCO; ++i)
#pragma unroll
    for (int q = 0; q < 5; ++q) dyf.o[i][q] = 0.0;
  {
    double kw, dkw_p, dkw_t, fw, dfw_s;
    k_value(M.kv[0], p, t, kw, dkw_p, dkw_t);
    per_factor(sw, eps_per, fw, dfw_s);
    yf[0] = fw * kw;
    dyf.w[0] = fw * dkw_p;
    dyf.w[1] = fw * dkw_t;
    dyf.w[2] = dfw_s * kw;
    double fo_h, dfo_h;
    per_factor(so, eps_per, fo_h, dfo_h);
#pragma unroll
    for (int i = 0; i < NCO; ++i) {
      double ki, dki_p, dki_t;
      k_value(M.kv[1 + i], p, t, ki, dki_p, dki_t);
      const int cr = 1 + i;
      if (i == M.heavy) {
        yf[cr] = fo_h * ki * x[i];
        dyf.o[i][0] = fo_h * dki_p * x[i];
        dyf.o[i][1] = fo_h * dki_t * x[i];
        dyf.o[i][2] = fo_h * ki;
        dyf.o[i][3] = -dfo_h * ki * x[i];
        dyf.o[i][4] = -dfo_h * ki * x[i];
      } else {
        yf[cr] = ki * x[i];
        dyf.o[i][0] = dki_p * x[i];
        dyf.o[i][1] = dki_t * x[i];
        dyf.o[i][2] = ki;
      }
    }
#pragma unroll
    for (int j = 0; j < NCG; ++j) {
      yf[1 + NCO + j] = y[j];
    }
  }
  // record: yfull and its structural partials
#pragma unroll
  for (int a = 0; a < NF; ++a) REC(R_Y + a) = yf[a];
  REC(R_DY0_P) = dyf.w[0];
  REC(R_DY0_T) = dyf.w[1];
  REC(R_DY0_SW) = dyf.w[2];
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
    REC(R_DYO + 4 * i + 0) = dyf.o[i][0];
    REC(R_DYO + 4 * i + 1) = dyf.o[i][1];
    REC(R_DYO + 4 * i + 2) = dyf.o[i][2];
    REC(R_DYO + 4 * i + 3) = dyf.o[i][3];
  }

  // gas phase (_kernels.py:254-328); the split property pass leaves it to k_cell_gas
  GasPhase G;
  if constexpr (!S::kSplitGas) gas_phase(M, p, t, t_ref, yf, dyf, G);
  const double rg = G.rg, mgbar = G.mgbar, mug = G.mug, hg = G.hg, ug = G.ug;
  const double (&drg)[NU] = G.drg;
  const double (&dmg)[NU] = G.dmg;
  const double (&dmug)[NU] = G.dmug;
  const double (&dhg)[NU] = G.dhg;
  const double (&dug)[NU] = G.dug;

  // relperm + capillary pressure (_kernels.py:330-353)
  double krw, dkrw, krow, dkrow, pcow, dpcow, krg, dkrg, krog, dkrog, pcog, dpcog, s2[5];
  interp1(M.nswt, M.swt_s, M.swt_krw, sw, krw, dkrw);
  interp1(M.nswt, M.swt_s, M.swt_krow, sw, krow, dkrow);
  interp1(M.nswt, M.swt_s, M.swt_pcow, sw, pcow, dpcow);
  interp1(M.nslt, M.slt_s, M.slt_krg, sg, krg, dkrg);
  interp1(M.nslt, M.slt_s, M.slt_krog, sg, krog, dkrog);
  interp1(M.nslt, M.slt_s, M.slt_pcog, sg, pcog, dpcog);
  stone2(rk[RK_KROCW], krow, krw, krog, krg, s2);
  const double kro = s2[0];
  const double dkro_sw = s2[1] * dkrow + s2[2] * dkrw;
  const double dkro_sg = s2[3] * dkrog + s2[4] * dkrg;
  REC(R_LAM) = krw + kro + krg;                  // assembly.py:434-437
  REC(R_DLAM_SW) = dkrw + dkro_sw;
  REC(R_DLAM_SG) = dkro_sg + dkrg;

  // specific weights (_kernels.py:355-373)
  const double m_w = M.gasp[0][G_M];
  REC(R_GAM + 0) = rw * m_w * PSI_PER_FT;
  REC(R_DGAM0_P) = drw_p * m_w * PSI_PER_FT;
  REC(R_DGAM0_T) = drw_t * m_w * PSI_PER_FT;
  double mobar = 0.0;
#pragma unroll
  for (int i = 0; i < NCO; ++i) mobar += x[i] * M.gasp[1 + i][G_M];
  REC(R_GAM + 1) = ro * mobar * PSI_PER_FT;
  REC(R_DGAM1_P) = dro_p * mobar * PSI_PER_FT;
  REC(R_DGAM1_T) = dro_t * mobar * PSI_PER_FT;
#pragma unroll
  for (int i = 0; i < NCO; ++i)
    REC(R_DGAM1_X + i) = (dro_x[i] * mobar + ro * M.gasp[1 + i][G_M]) * PSI_PER_FT;
  if constexpr (!S::kSplitGas) {
#pragma unroll
    for (int u = 0; u < NU; ++u) REC(R_DGAM2 + u) = (drg[u] * mgbar + rg * dmg[u]) * PSI_PER_FT;
    REC(R_GAM + 2) = rg * mgbar * PSI_PER_FT;
  }

  // phase pressures (_kernels.py:375-385)
  REC(R_POT + 0) = p - pcow;
  REC(R_POT + 1) = p;
  REC(R_POT + 2) = p + pcog;
  REC(R_DPOT0_SW) = -dpcow;
  REC(R_DPOT2_SG) = dpcog;

  // mobility-density products (_kernels.py:387-408)
  REC(R_BETA + 0) = rw * krw / muw;
  {
    double b0p = 0.0, b0t = 0.0, b0s = 0.0;
    if (krw > 0.0 || dkrw != 0.0) {
      b0p = drw_p * krw / muw;
      b0t = (drw_t * krw - rw * krw * dmuw_t / muw) / muw;
      b0s = rw * dkrw / muw;
    }
    REC(R_DBETA0_P) = b0p; REC(R_DBETA0_T) = b0t; REC(R_DBETA0_SW) = b0s;
  }
  REC(R_BETA + 1) = ro * kro / muo;
  {
    double b1p = 0.0, b1t = 0.0, b1w = 0.0, b1g = 0.0, b1x[NCO];
#pragma unroll
    for (int i = 0; i < NCO; ++i) b1x[i] = 0.0;
    if (kro > 0.0 || dkro_sw != 0.0 || dkro_sg != 0.0) {
      b1p = dro_p * kro / muo;
      b1t = (dro_t * kro - ro * kro * dmuo_t / muo) / muo;
      b1w = ro * dkro_sw / muo;
      b1g = ro * dkro_sg / muo;
#pragma unroll
      for (int i = 0; i < NCO; ++i) {
        double dmuo_xi = muo * log(mu_i[i]);
        b1x[i] = (dro_x[i] * kro - ro * kro * dmuo_xi / muo) / muo;
      }
    }
    REC(R_DBETA1_P) = b1p; REC(R_DBETA1_T) = b1t; REC(R_DBETA1_SW) = b1w; REC(R_DBETA1_SG) = b1g;
#pragma unroll
    for (int i = 0; i < NCO; ++i) REC(R_DBETA1_X + i) = b1x[i];
  }
  if constexpr (!S::kSplitGas) {
  {
    const bool on = krg > 0.0 || dkrg != 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      double v = 0.0;
      if (on) {
        v = (drg[u] * krg - rg * krg * dmug[u] / mug) / mug;
        if (u == CSG) v += rg * dkrg / mug;
      }
      REC(R_DBETA2 + u) = v;
    }
  }
  REC(R_BETA + 2) = rg * krg / mug;
  }

  // phase enthalpies (_kernels.py:410-419)
  REC(R_HPH + 0) = hw;
  REC(R_DHPH0_T) = dhw_t;
  REC(R_HPH + 1) = ho;
  REC(R_DHPH1_T) = dho_t;
#pragma unroll
  for (int i = 0; i < NCO; ++i) REC(R_DHPH1_X + i) = hli[i];
  if constexpr (!S::kSplitGas) {
    REC(R_HPH + 2) = hg;
#pragma unroll
    for (int u = 0; u < NU; ++u) REC(R_DHPH2 + u) = dhg[u];
  }

  // thermal conductivity (_kernels.py:421-428)
  {
    const double br = sw * rk[RK_KTW] + so * rk[RK_KTO] + sg * rk[RK_KTG];
    REC(R_KT + 0) = phif * br + (1.0 - phi) * rk[RK_KTR] + cc * rk[RK_KTC];
    REC(R_KT + 1) = dphi_p * br - dphi_p * rk[RK_KTR];
    REC(R_KT + 2) = dphi_t * br - dphi_t * rk[RK_KTR];
    REC(R_KT + 3) = phif * (rk[RK_KTW] - rk[RK_KTO]);
    REC(R_KT + 4) = phif * (rk[RK_KTG] - rk[RK_KTO]);
    REC(R_KT + 5) = dphif_cc * br + rk[RK_KTC];
  }
#undef REC

  // the reaction / accumulation rows (cell_rows) from the property values
  if constexpr (S::kMidOut) {
    s.mid(MI_PHI, phi); s.mid(MI_DPHI_P, dphi_p); s.mid(MI_DPHI_T, dphi_t);
    s.mid(MI_PHIF, phif); s.mid(MI_DPHIF_CC, dphif_cc); s.mid(MI_PCOG, pcog);
    s.mid(MI_RO, ro); s.mid(MI_DRO_P, dro_p); s.mid(MI_DRO_T, dro_t);
#pragma unroll
    for (int i = 0; i < NCO; ++i) s.mid(MI_DRO_X + i, dro_x[i]);
    if constexpr (!S::kSplitGas) {
      s.mid(MI_RG, rg);
#pragma unroll
      for (int u = 0; u < NU; ++u) s.mid(MI_DRG + u, drg[u]);
    }
    s.mid(MI_RW, rw); s.mid(MI_DRW_P, drw_p); s.mid(MI_DRW_T, drw_t);
    s.mid(MI_UW, uw); s.mid(MI_DUW_P, duw_p); s.mid(MI_DUW_T, duw_t);
    s.mid(MI_UO, uo); s.mid(MI_DUO_P, duo_p); s.mid(MI_DUO_T, duo_t);
    if constexpr (!S::kSplitGas) {
      s.mid(MI_UG, ug);
#pragma unroll
      for (int u = 0; u < NU; ++u) s.mid(MI_DUG + u, dug[u]);
    }
  } else {
    CellMid m;
    m.v[MI_PHI] = phi; m.v[MI_DPHI_P] = dphi_p; m.v[MI_DPHI_T] = dphi_t;
    m.v[MI_PHIF] = phif; m.v[MI_DPHIF_CC] = dphif_cc; m.v[MI_PCOG] = pcog;
    m.v[MI_RO] = ro; m.v[MI_DRO_P] = dro_p; m.v[MI_DRO_T] = dro_t;
#pragma unroll
    for (int i = 0; i < NCO; ++i) { m.v[MI_DRO_X + i] = dro_x[i]; m.hli[i] = hli[i]; }
    m.v[MI_RG] = rg;
#pragma unroll
    for (int u = 0; u < NU; ++u) { m.v[MI_DRG + u] = drg[u]; m.v[MI_DUG + u] = dug[u]; }
    m.v[MI_RW] = rw; m.v[MI_DRW_P] = drw_p; m.v[MI_DRW_T] = drw_t;
    m.v[MI_UW] = uw; m.v[MI_DUW_P] = duw_p; m.v[MI_DUW_T] = duw_t;
    m.v[MI_UO] = uo; m.v[MI_DUO_P] = duo_p; m.v[MI_DUO_T] = duo_t;
    m.v[MI_UG] = ug;
    m.dyf = dyf;
#pragma unroll
    for (int a = 0; a < NF; ++a) m.yf[a] = yf[a];
    m.dpcog = dpcog;
    cell_rows<S, S::kUnroll>(M, A, c, u_, m, s);
  }
}

// The cell pass in three kernels with fewer live values each: the
// properties (record + A.mid), the gas phase, then the reaction /
// accumulation rows (cell_rows over the stored values).
#ifndef CELLP_MINB
#define CELLP_MINB 7   // C4 sweep 4..12 (rows at 2): 8 best before the gas split, 6-7 after
#endif
#ifndef CELLR_MINB
#define CELLR_MINB 2   // C4 sweep 1..6 (props at 8): 1-2 best (255 registers, 128 B spilled)
#endif
#ifndef CELLR_UNROLL
#define CELLR_UNROLL true
#endif
__global__ void __launch_bounds__(128, CELLP_MINB) k_cell_props(const Model M, const CellArgs A) {
  const int64_t n = A.g.n;
  const int64_t c = A.c_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.c_end) return;
  double u_[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) u_[u] = A.st[u * n + c];
  CellSinkProps s{A, n, c};
  cell_eval(M, A, c, u_, s);
}

// the gas phase of the split cell pass: record fields of the gas and the
// values the rows need (after k_cell_props: yfull / dyfull from the record)
#ifndef CELLG_MINB
#define CELLG_MINB 4   // C4 sweep 2..8: 4 best
#endif
__global__ void __launch_bounds__(128, CELLG_MINB) k_cell_gas(const Model M, const CellArgs A) {
  const int64_t n = A.g.n;
  const int64_t c = A.c_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.c_end) return;
  const double p = A.st[c], t = A.st[CT * n + c], sg = A.st[CSG * n + c];
  double* rec = A.rec + c;
  double yf[NF];
#pragma unroll
  for (int a = 0; a < NF; ++a) yf[a] = rec[(int64_t)(R_Y + a) * n];
  DyFull dyf;
  dyf.w[0] = rec[(int64_t)R_DY0_P * n];
  dyf.w[1] = rec[(int64_t)R_DY0_T * n];
  dyf.w[2] = rec[(int64_t)R_DY0_SW * n];
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) dyf.o[i][q] = rec[(int64_t)(R_DYO + 4 * i + q) * n];
    dyf.o[i][4] = i == M.heavy ? dyf.o[i][3] : 0.0;
  }
  GasPhase G;
  gas_phase(M, p, t, M.rockp[RK_TREF], yf, dyf, G);
  double krg, dkrg;
  interp1(M.nslt, M.slt_s, M.slt_krg, sg, krg, dkrg);
#define REC(f) rec[(int64_t)(f) * n]
#pragma unroll
  for (int u = 0; u < NU; ++u) REC(R_DGAM2 + u) = (G.drg[u] * G.mgbar + G.rg * G.dmg[u]) * PSI_PER_FT;
  REC(R_GAM + 2) = G.rg * G.mgbar * PSI_PER_FT;
  {
    const bool on = krg > 0.0 || dkrg != 0.0;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      double v = 0.0;
      if (on) {
        v = (G.drg[u] * krg - G.rg * krg * G.dmug[u] / G.mug) / G.mug;
        if (u == CSG) v += G.rg * dkrg / G.mug;
      }
      REC(R_DBETA2 + u) = v;
    }
  }
  REC(R_BETA + 2) = G.rg * krg / G.mug;
  REC(R_HPH + 2) = G.hg;
#pragma unroll
  for (int u = 0; u < NU; ++u) REC(R_DHPH2 + u) = G.dhg[u];
#undef REC
  double* mid = A.mid + c;
  mid[(int64_t)MI_RG * n] = G.rg;
  mid[(int64_t)MI_UG * n] = G.ug;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    mid[(int64_t)(MI_DRG + u) * n] = G.drg[u];
    mid[(int64_t)(MI_DUG + u) * n] = G.dug[u];
  }
}

__global__ void __launch_bounds__(128, CELLR_MINB) k_cell_rows(const Model M, const CellArgs A) {
  const int64_t n = A.g.n;
  const int64_t c = A.c_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.c_end) return;
  if (A.mid[(int64_t)MI_PHIF * n + c] <= 0.0) return;   // pore space exhausted (reported)
  double u_[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) u_[u] = A.st[u * n + c];
  CellMid m;
#pragma unroll
  for (int f = 0; f < NMID; ++f) m.v[f] = A.mid[(int64_t)f * n + c];
  const double* rec = A.rec + c;
#pragma unroll
  for (int a = 0; a < NF; ++a) m.yf[a] = rec[(int64_t)(R_Y + a) * n];
  m.dyf.w[0] = rec[(int64_t)R_DY0_P * n];
  m.dyf.w[1] = rec[(int64_t)R_DY0_T * n];
  m.dyf.w[2] = rec[(int64_t)R_DY0_SW * n];
#pragma unroll
  for (int i = 0; i < NCO; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) m.dyf.o[i][q] = rec[(int64_t)(R_DYO + 4 * i + q) * n];
    m.dyf.o[i][4] = i == M.heavy ? m.dyf.o[i][3] : 0.0;   // d/dSg == d/dSw (heaviest oil)
    m.hli[i] = rec[(int64_t)(R_DHPH1_X + i) * n];
  }
  m.dpcog = rec[(int64_t)R_DPOT2_SG * n];
  CellSinkGlobal s{A, n, c};
  cell_rows<CellSinkGlobal, CELLR_UNROLL>(M, A, c, u_, m, s);
}

// -------------------------------------------------------------------- face

struct FaceArgs {
  Dims g;
  const double* __restrict__ st;
  const double* __restrict__ rec;
  const double* __restrict__ depth;
  const double* __restrict__ gd;   // [axis*n + a] Darcy factor of the +axis face of a
  const double* __restrict__ td;   // [axis*n + a] thermal factor
  int8_t* upw;                     // [(axis*3 + phase)*n + a]
  int freeze;
  double* __restrict__ resid;
  double* __restrict__ diag;
  double* __restrict__ offd;
  int* ccnz;   // set to 1 when a flux row < ROW_E gets a nonzero coke-column entry
};

// dense 9-vectors of a cell's record partials
struct CellView {
  const double* __restrict__ rec;
  int64_t n, c;
  __device__ double f(int k) const { return rec[(int64_t)k * n + c]; }
  __device__ void dpot(int al, double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    v[0] = 1.0;
    if (al == 0) v[CSW] = f(R_DPOT0_SW);
    if (al == 2) v[CSG] = f(R_DPOT2_SG);
  }
  __device__ void dgam(int al, double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    if (al == 0) { v[0] = f(R_DGAM0_P); v[CT] = f(R_DGAM0_T); }
    else if (al == 1) {
      v[0] = f(R_DGAM1_P); v[CT] = f(R_DGAM1_T);
#pragma unroll
      for (int i = 0; i < NCO; ++i) v[1 + i] = f(R_DGAM1_X + i);
    } else {
#pragma unroll
      for (int u = 0; u < NU; ++u) v[u] = f(R_DGAM2 + u);
    }
  }
  __device__ void dbeta(int al, double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    if (al == 0) { v[0] = f(R_DBETA0_P); v[CT] = f(R_DBETA0_T); v[CSW] = f(R_DBETA0_SW); }
    else if (al == 1) {
      v[0] = f(R_DBETA1_P); v[CT] = f(R_DBETA1_T); v[CSW] = f(R_DBETA1_SW); v[CSG] = f(R_DBETA1_SG);
#pragma unroll
      for (int i = 0; i < NCO; ++i) v[1 + i] = f(R_DBETA1_X + i);
    } else {
#pragma unroll
      for (int u = 0; u < NU; ++u) v[u] = f(R_DBETA2 + u);
    }
  }
  __device__ void dhph(int al, double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    if (al == 0) v[CT] = f(R_DHPH0_T);
    else if (al == 1) {
      v[CT] = f(R_DHPH1_T);
#pragma unroll
      for (int i = 0; i < NCO; ++i) v[1 + i] = f(R_DHPH1_X + i);
    } else {
#pragma unroll
      for (int u = 0; u < NU; ++u) v[u] = f(R_DHPH2 + u);
    }
  }
  __device__ void dyfull(int m, double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    if (m == 0) { v[0] = f(R_DY0_P); v[CT] = f(R_DY0_T); v[CSW] = f(R_DY0_SW); }
    else if (m < 1 + NCO) {
      // m is a run-time row: compare-and-select keeps v in registers
      const int i = m - 1;
      v[0] = f(R_DYO + 4 * i); v[CT] = f(R_DYO + 4 * i + 1);
      const double dx = f(R_DYO + 4 * i + 2);
#pragma unroll
      for (int q = 0; q < NCO; ++q)
        if (q == i) v[1 + q] = dx;
      const double s = f(R_DYO + 4 * i + 3);
      v[CSW] = s; v[CSG] = s;
    } else {
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (u == m) v[u] = 1.0;   // gas m: unit partial at its own column
    }
  }
  __device__ void dkt(double* v) const {
#pragma unroll
    for (int u = 0; u < NU; ++u) v[u] = 0.0;
    v[0] = f(R_KT + 1); v[CT] = f(R_KT + 2); v[CSW] = f(R_KT + 3); v[CSG] = f(R_KT + 4);
    v[CCC] = f(R_KT + 5);
  }
};

// Structurally non-zero columns of the per-phase partials (record.cuh). The
// reference accumulates dense 9-vectors; terms whose partials are literal
// zeros only add +-0 and are skipped here at compile time (the phase loop is
// unrolled), which also keeps the face kernel's registers in check.
__host__ __device__ constexpr unsigned colbit(int u) { return 1u << u; }
constexpr unsigned XCOLS = ((1u << NCO) - 1u) << 1;   // oil x columns
constexpr unsigned ALLCOLS = (1u << NU) - 1u;
__host__ __device__ constexpr unsigned m_dpot(int al) {
  return al == 0 ? colbit(0) | colbit(CSW) : (al == 1 ? colbit(0) : colbit(0) | colbit(CSG));
}
__host__ __device__ constexpr unsigned m_dgam(int al) {
  return al == 0 ? colbit(0) | colbit(CT) : (al == 1 ? colbit(0) | colbit(CT) | XCOLS : ALLCOLS);
}
__host__ __device__ constexpr unsigned m_dbeta(int al) {
  return al == 0 ? colbit(0) | colbit(CT) | colbit(CSW)
                 : (al == 1 ? colbit(0) | colbit(CT) | colbit(CSW) | colbit(CSG) | XCOLS : ALLCOLS);
}
__host__ __device__ constexpr unsigned m_dhph(int al) {
  return al == 0 ? colbit(CT) : (al == 1 ? colbit(CT) | XCOLS : ALLCOLS);
}
constexpr unsigned M_DKT = colbit(0) | colbit(CT) | colbit(CSW) | colbit(CSG) | colbit(CCC);

// Row `row` of one connection's flux and derivative blocks (a = lower cell).
// Follows conn_eval's accumulation order exactly (_kernels.py:677-771).
template <int row>
__device__ __forceinline__ void face_row(const CellView& A_, const CellView& B_,
                                         const double* __restrict__ st, int64_t n, int64_t a,
                                         int64_t b, double za, double zb, double gd, double td,
                                         int8_t* upw, int64_t upw_stride, int freeze,
                                         bool write_upw, double& flux, double* dfa, double* dfb) {
  flux = 0.0;
#pragma unroll
  for (int u = 0; u < NU; ++u) { dfa[u] = 0.0; dfb[u] = 0.0; }
  if (row == ROW_OS || row == ROW_GS || row == ROW_CK) return;
  double v1[NU], v2[NU];
#pragma unroll
  for (int al = 0; al < 3; ++al) {
    // does this phase touch this row?
    const bool comp_row = (al == 0 && row == 0) || (al == 1 && row >= 1 && row < 1 + NCO) ||
                          (al == 2 && row < NF);
    const bool energy = row == ROW_E;
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
    if (!comp_row && !energy) continue;
    const CellView& U = up_a ? A_ : B_;
    const double b_up = U.f(R_BETA + al);
    const double conv = gd * dphi;
    double w_up, val;
    int m = 0;
    if (comp_row) {
      if (al == 0) w_up = 1.0;
      else if (al == 1) { m = row - 1; w_up = st[(1 + m) * n + (up_a ? a : b)]; }
      else { m = row; w_up = U.f(R_Y + m); }
    } else {
      w_up = U.f(R_HPH + al);   // energy: h_up
    }
    val = b_up * w_up;
    flux += conv * val;
    if (val != 0.0) {
      const unsigned mpg = m_dpot(al) | m_dgam(al);
      A_.dpot(al, v1); A_.dgam(al, v2);
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (mpg & colbit(u)) dfa[u] += gd * val * (v1[u] - za * v2[u]);
      B_.dpot(al, v1); B_.dgam(al, v2);
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (mpg & colbit(u)) dfb[u] -= gd * val * (v1[u] - zb * v2[u]);
    }
    const double beta_up = U.f(R_BETA + al);
    U.dbeta(al, v1);
    if (comp_row) {
      if (al == 2) U.dyfull(m, v2);
      const unsigned mb = al == 2 ? ALLCOLS : (m_dbeta(al) | (al == 1 ? XCOLS : 0u));
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if (!(mb & colbit(u))) continue;
        double dv = v1[u] * w_up;
        if (al == 1 && u == 1 + m) dv += beta_up;
        else if (al == 2) dv += beta_up * v2[u];
        if (dv != 0.0) {   // upstream side (no pointer select: stays in registers)
          if (up_a) dfa[u] += conv * dv;
          else dfb[u] += conv * dv;
        }
      }
    } else {
      U.dhph(al, v2);
      const unsigned mh = m_dbeta(al) | m_dhph(al);
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if (!(mh & colbit(u))) continue;
        double dv = v1[u] * w_up + beta_up * v2[u];
        if (dv != 0.0) {
          if (up_a) dfa[u] += conv * dv;
          else dfb[u] += conv * dv;
        }
      }
    }
  }
  if (row == ROW_E) {
    double hm, dh_a, dh_b;
    harmonic_pair(A_.f(R_KT), B_.f(R_KT), hm, dh_a, dh_b);
    if (hm > 0.0 || dh_a != 0.0 || dh_b != 0.0) {
      const double dt_ab = st[CT * n + a] - st[CT * n + b];
      flux += td * hm * dt_ab;
      dfa[CT] += td * hm;
      dfb[CT] -= td * hm;
      if (dt_ab != 0.0) {
        A_.dkt(v1);
        B_.dkt(v2);
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          if (!(M_DKT & colbit(u))) continue;
          dfa[u] += td * dt_ab * dh_a * v1[u];
          dfb[u] += td * dt_ab * dh_b * v2[u];
        }
      }
    }
  }
}

// ------------------------------------------------------- face-centric pair
//
// Each face is evaluated once:
//   k_face_eval_*  thread per (lower cell a, axis) -- the five light rows in
//                  one thread (_light), the energy row in another (_energy):
//                  per row the flux and both derivative rows of face (a,
//                  a+axis); writes
//                  offd[a][+axis] row = dfb, offd[b][-axis] row = -dfa and
//                  the flux into fbuf[(axis*ROW_OS + row)*n + a]; zero rows
//                  for boundary blocks.
//   k_face_gather  thread per (cell, row < ROW_OS): the reference's gather
//                  (_kernels.py:828-854) in its fixed order; the diagonal
//                  contribution of each face is read back as minus the
//                  neighbour's block pointing at the cell (-(-dfa) = dfa for
//                  side a, -dfb for side b: the same values and order as the
//                  two-sided kernel).
struct FaceArgs2 {
  FaceArgs F;
  double* __restrict__ fbuf;   // (3 * ROW_OS) x n face fluxes
};

template <int ROW>
__device__ __forceinline__ void face_eval_row(const FaceArgs2& A2, int64_t c, int64_t cell, int i,
                                              int j, int k, int axis) {
  const FaceArgs& F = A2.F;
  const int64_t n = F.g.n;
  const int dp = DXP + axis, dm = opposite(dp);
  const bool has_lo = (axis == 0 ? i > 0 : (axis == 1 ? j > 0 : k > 0));
  if (!has_lo) {   // no face below: the cell's -axis block row is zero
    double* orow = F.offd + (int64_t)((dm * NU + ROW) * NU) * n + c;
#pragma unroll
    for (int u = 0; u < NU; ++u) orow[(int64_t)u * n] = 0.0;
  }
  const int64_t nb = nb_pos(F.g, cell, i, j, k, dp);
  double* orow_a = F.offd + (int64_t)((dp * NU + ROW) * NU) * n + c;
  if (nb < 0) {
#pragma unroll
    for (int u = 0; u < NU; ++u) orow_a[(int64_t)u * n] = 0.0;
    return;
  }
  const CellView Av{F.rec, n, c}, Bv{F.rec, n, nb};
  double flux, dfa[NU], dfb[NU];
  face_row<ROW>(Av, Bv, F.st, n, c, nb, F.depth[c], F.depth[nb], F.gd[axis * n + c],
                F.td[axis * n + c], F.upw + (int64_t)axis * 3 * n, n, F.freeze, ROW == 0, flux,
                dfa, dfb);
  double* orow_b = F.offd + (int64_t)((dm * NU + ROW) * NU) * n + nb;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    orow_a[(int64_t)u * n] = dfb[u];
    orow_b[(int64_t)u * n] = -dfa[u];
  }
  // the component rows' coke column is zero for an assembled system (no
  // flux term depends on C_c); k_cc_red skips its loads while none is set
  if (ROW < ROW_E && (dfa[CCC] != 0.0 || dfb[CCC] != 0.0)) *F.ccnz = 1;
  A2.fbuf[(int64_t)(axis * ROW_OS + ROW) * n + c] = flux;
}

// The light rows (0..4) and the energy row (5, every phase) as separate
// kernels so that each gets its own register budget / occupancy. A thread
// evaluates all five light rows of its face: the rows share the phase
// potentials, the upwind choice and the upstream partials, which stay in
// registers across the inlined rows (same expressions, so the same values as
// the earlier thread per (face, row): face pair 3.70 -> 3.52 ms at C4).
#ifndef FEVL_MINB
#define FEVL_MINB 5   // C4: 128 registers, 5 CTAs per SM (4: 132 registers, no gain; 6-7: spills, none)
#endif
#ifndef FEVE_MINB
#define FEVE_MINB 5   // C4 sweep 4..8: face pair 4.06 -> 3.97 ms at 5
#endif
__global__ void __launch_bounds__(32 * 3, FEVL_MINB) k_face_eval_light(const FaceArgs2 A2,
                                                                       int64_t c_begin,
                                                                       int64_t c_end, int axis_lo) {
  const int64_t c = c_begin + (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (c >= c_end) return;
  const int axis = axis_lo + threadIdx.y;
  int i, j, k;
  const int64_t cell = locate(A2.F.g, c, i, j, k);
  face_eval_row<0>(A2, c, cell, i, j, k, axis);
  face_eval_row<1>(A2, c, cell, i, j, k, axis);
  face_eval_row<2>(A2, c, cell, i, j, k, axis);
  face_eval_row<3>(A2, c, cell, i, j, k, axis);
  face_eval_row<4>(A2, c, cell, i, j, k, axis);
}
__global__ void __launch_bounds__(32 * 3, FEVE_MINB) k_face_eval_energy(const FaceArgs2 A2,
                                                                        int64_t c_begin,
                                                                        int64_t c_end, int axis_lo) {
  const int64_t c = c_begin + (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (c >= c_end) return;
  const int axis = axis_lo + threadIdx.y;
  int i, j, k;
  const int64_t cell = locate(A2.F.g, c, i, j, k);
  face_eval_row<ROW_E>(A2, c, cell, i, j, k, axis);
}

// grid (ceil(owned cells / 32)); block (32, ROW_OS). Owned planes only:
// ghost rows (z-slabs) carry no equation.
#ifndef FG_MINB
#define FG_MINB 4   // C4 sweep 1..8: 4 (85 registers) best; without a minimum the compiler capped at 64
#endif
__global__ void __launch_bounds__(32 * ROW_OS, FG_MINB) k_face_gather(const FaceArgs2 A2,
                                                                      int64_t c_begin,
                                                                      int64_t c_end) {
  const FaceArgs& F = A2.F;
  const int64_t n = F.g.n;
  const int64_t c = c_begin + (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int row = threadIdx.y;
  if (c >= c_end) return;
  int i, j, k;
  const int64_t cell = locate(F.g, c, i, j, k);
  double res = F.resid[row * n + c];
  // the face evaluation of this assembly found the component rows' coke
  // column zero: those back-block loads are skipped (warp-uniform)
  const bool skip_cc = row < ROW_E && *F.ccnz == 0;
  double drow[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) drow[u] = F.diag[(int64_t)(row * NU + u) * n + c];
#pragma unroll
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = nb_pos(F.g, cell, i, j, k, d);
    if (nb < 0) continue;
    const bool c_is_a = d >= DXP;
    const int axis = c_is_a ? d - DXP : 2 - d;
    const double flux = A2.fbuf[(int64_t)(axis * ROW_OS + row) * n + (c_is_a ? c : nb)];
    if (c_is_a) res += flux;
    else res -= flux;
    const double* back = F.offd + (int64_t)((opposite(d) * NU + row) * NU) * n + nb;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (u == CCC && skip_cc) continue;
      drow[u] += -back[(int64_t)u * n];
    }
  }
  F.resid[row * n + c] = res;
#pragma unroll
  for (int u = 0; u < NU; ++u) F.diag[(int64_t)(row * NU + u) * n + c] = drow[u];
}

// ------------------------------------------------------------------- wells

// Per-well device record (host mirror in csrc/capi.cu / include/iscgpu.h)
struct WellDev {
  int64_t cell;
  int kind, control;           // INJECTOR 0 / PRODUCER 1; CTRL_BHP 0, rate 1/2
  double target, wi, z_bh, pinjmax, heat_rate, heat_stop;
  double s_yfull[NF], s_yinj[NCG], s_tinj, s_mu, s_h, s_mbar;
};
// output per well: resid, dwdb, wrow[NU], bcol[NU], phase_rates[3], comp_rates[NU]
constexpr int WOUT = 2 + NU + NU + 3 + NU;
constexpr double DARCY_CONST = 1.0623e-14 * 144.0 / (1.0e-3 * 0.2248089431 / 10.76391042 / 86400.0);

__global__ void k_wells(const Model M, Dims g, int nw, const WellDev* __restrict__ wells,
                        const double* __restrict__ st, const double* __restrict__ bhp,
                        const uint8_t* __restrict__ capped, const double* __restrict__ rec,
                        const double* __restrict__ depth, double t_new,
                        double* resid, double* diag, double* wout) {
  // one thread per well evaluates its perforation (independent of the other
  // wells); the cell rows are then applied by one thread in well order, the
  // reference's sequence of updates (wells sharing a cell stay bit-exact)
  constexpr int WB = 32;
  __shared__ double s_rows[WB][NU], s_drows[WB][NU][NU], s_heat[WB];
  __shared__ int64_t s_cell[WB];
  const int64_t n = g.n;
  for (int base = 0; base < nw; base += WB) {
  const int w = base + threadIdx.x;
  const int tw = threadIdx.x;
  if (w < nw) {
    const WellDev W = wells[w];
    const int64_t c = W.cell;
    const CellView V{rec, n, c};
    const double dz = W.z_bh - depth[c];
    const double bh = bhp[w];
    double rows[NU], drows[NU][NU], brows[NU], qph[3], dqs[NU], dqs_db = 0.0;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      rows[r] = 0.0; brows[r] = 0.0; dqs[r] = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) drows[r][u] = 0.0;
    }
    qph[0] = qph[1] = qph[2] = 0.0;
    const double cwi = DARCY_CONST * W.wi;
    if (W.kind == 0) {
      // injector (assembly.py:421-471)
      const double lam = V.f(R_LAM);
      double dlam[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) dlam[u] = 0.0;
      dlam[CSW] = V.f(R_DLAM_SW);
      dlam[CSG] = V.f(R_DLAM_SG);
      const double pg = V.f(R_POT + 2);
      double dpg[NU];
      V.dpot(2, dpg);
      double dzdw[NF], dzdp, dzdt;
      const double zf = z_factor_mix<NF>(W.s_yfull, M.gasp, pg, W.s_tinj, dzdw, dzdp, dzdt);
      const double trs = W.s_tinj + RANKINE;
      const double rho = pg / (zf * R_GAS * trs);
      const double drho_dpg = rho * (1.0 / pg - dzdp / zf);
      const double gam = rho * W.s_mbar / 144.0;
      const double dgam_dpg = drho_dpg * W.s_mbar / 144.0;
      const double dd = bh - pg - gam * dz;
      const double mob = rho * lam / W.s_mu;
      const double q = cwi * mob * dd;
      double dq[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const double ddd = -dpg[u] * (1.0 + dz * dgam_dpg);
        const double dmob = (drho_dpg * dpg[u] * lam + rho * dlam[u]) / W.s_mu;
        dq[u] = cwi * (dmob * dd + mob * ddd);
      }
      const double dq_db = cwi * mob;
#pragma unroll
      for (int j = 0; j < NCG; ++j) {
        rows[1 + NCO + j] = q * W.s_yinj[j];
#pragma unroll
        for (int u = 0; u < NU; ++u) drows[1 + NCO + j][u] = W.s_yinj[j] * dq[u];
        brows[1 + NCO + j] = dq_db * W.s_yinj[j];
      }
      rows[ROW_E] = q * W.s_h;
#pragma unroll
      for (int u = 0; u < NU; ++u) drows[ROW_E][u] = dq[u] * W.s_h;
      brows[ROW_E] = dq_db * W.s_h;
      qph[2] = q;
#pragma unroll
      for (int u = 0; u < NU; ++u) dqs[u] = dq[u];
      dqs_db = dq_db;
    } else {
      // producer (assembly.py:370-418)
      double x_c[NCO];
#pragma unroll
      for (int i = 0; i < NCO; ++i) x_c[i] = st[(1 + i) * n + c];
      for (int al = 0; al < 3; ++al) {
        double v1[NU], v2[NU], v3[NU];
        V.dpot(al, v1);
        V.dgam(al, v2);
        V.dbeta(al, v3);
        const double beta = V.f(R_BETA + al);
        const double dd = bh - V.f(R_POT + al) - V.f(R_GAM + al) * dz;
        const double q = cwi * beta * dd;
        double dq[NU];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const double ddd = -v1[u] - dz * v2[u];
          dq[u] = cwi * (v3[u] * dd + beta * ddd);
        }
        const double dq_db = cwi * beta;
        qph[al] = q;
#pragma unroll
        for (int u = 0; u < NU; ++u) dqs[u] += dq[u];
        dqs_db += dq_db;
        if (al == 0) {
          rows[0] += q;
#pragma unroll
          for (int u = 0; u < NU; ++u) drows[0][u] += dq[u];
          brows[0] += dq_db;
        } else if (al == 1) {
#pragma unroll
          for (int i = 0; i < NCO; ++i) {
            rows[1 + i] += q * x_c[i];
#pragma unroll
            for (int u = 0; u < NU; ++u) drows[1 + i][u] += x_c[i] * dq[u];
            drows[1 + i][1 + i] += q;
            brows[1 + i] += dq_db * x_c[i];
          }
        } else {
          for (int m = 0; m < NF; ++m) {
            const double yfm = V.f(R_Y + m);
            double dy[NU];
            V.dyfull(m, dy);
            rows[m] += q * yfm;
#pragma unroll
            for (int u = 0; u < NU; ++u) drows[m][u] += yfm * dq[u] + q * dy[u];
            brows[m] += dq_db * yfm;
          }
        }
        const double h = V.f(R_HPH + al);
        double dh[NU];
        V.dhph(al, dh);
        rows[ROW_E] += q * h;
#pragma unroll
        for (int u = 0; u < NU; ++u) drows[ROW_E][u] += dq[u] * h + q * dh[u];
        brows[ROW_E] += dq_db * h;
      }
    }
    double* o = wout + (int64_t)w * WOUT;
    const bool heater = W.heat_rate != 0.0 && t_new <= W.heat_stop;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
      s_rows[tw][r] = rows[r];
#pragma unroll
      for (int u = 0; u < NU; ++u) s_drows[tw][r][u] = drows[r][u];
      o[2 + NU + r] = -brows[r];                       // bcol
      o[2 + 2 * NU + 3 + r] = rows[r];                 // comp_rates
    }
    s_cell[tw] = c;
    s_heat[tw] = 0.0;
    if (heater) {
      s_heat[tw] = W.heat_rate;
      o[2 + 2 * NU + 3 + ROW_E] += W.heat_rate;
    }
    o[2 + 2 * NU + 0] = qph[0];
    o[2 + 2 * NU + 1] = qph[1];
    o[2 + 2 * NU + 2] = qph[2];
    const double qsum = qph[0] + qph[1] + qph[2];
    double resid_w, dwdb;
    bool zero_row = false;
    if (W.control == 0) { resid_w = bh - W.target; dwdb = 1.0; zero_row = true; }
    else if (capped[w]) { resid_w = bh - W.pinjmax; dwdb = 1.0; zero_row = true; }
    else { resid_w = qsum - W.target; dwdb = dqs_db; }
    o[0] = resid_w;
    o[1] = dwdb;
#pragma unroll
    for (int u = 0; u < NU; ++u) o[2 + u] = zero_row ? 0.0 : dqs[u];   // wrow
  }
  __syncthreads();
  // apply the rows: lane e owns matrix/residual entry e of the perforated
  // cell and walks the wells in order, so every address sees the reference's
  // sequence of updates (wells sharing a cell included; the heater after its
  // well's rows) while the 90 entries proceed in parallel (one thread walking
  // them all serialised 8 x 90 dependent read-modify-writes)
  const int nq = min(WB, nw - base);
  for (int e = threadIdx.x; e < NB + NU; e += blockDim.x) {
    for (int q = 0; q < nq; ++q) {
      const int64_t c = s_cell[q];
      if (e < NB) {
        diag[(int64_t)e * n + c] -= s_drows[q][e / NU][e % NU];
      } else {
        const int r = e - NB;
        resid[r * n + c] -= s_rows[q][r];
        if (r == ROW_E && s_heat[q] != 0.0) resid[ROW_E * n + c] -= s_heat[q];
      }
    }
  }
  __syncthreads();
  }
}

// --------------------------------------------------- layout conversion

// internal (SoA) -> reference layout diag (n,NU,NU), offd (m,2,NU,NU), resid (n,NU)
// conn_id[axis*n + a] = connection index of a's +axis face, or -1.
__global__ void k_export_system(Dims g, const int64_t* __restrict__ conn_id,
                                const double* __restrict__ diag, const double* __restrict__ offd,
                                const double* __restrict__ resid, double* rdiag, double* roffd,
                                double* rresid, int offd_rows) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // natural cell
  if (c >= n) return;
  const int64_t pc = pos_of(g, c);
  for (int e = 0; e < NB; ++e) rdiag[c * NB + e] = diag[(int64_t)e * n + pc];
  for (int r = 0; r < NU; ++r) rresid[c * NU + r] = resid[(int64_t)r * n + pc];
  int i, j, k;
  cell_ijk(g, c, i, j, k);
  for (int axis = 0; axis < 3; ++axis) {
    const int64_t ic = conn_id[axis * n + c];
    if (ic < 0) continue;
    const int dplus = DXP + axis;
    const int64_t nbp = nb_pos(g, c, i, j, k, dplus);
    const int dminus = opposite(dplus);
    for (int e = 0; e < NB; ++e) {
      const bool live = e / NU < offd_rows;   // rows >= offd_rows are structural zeros
      roffd[(ic * 2 + 0) * NB + e] = live ? offd[(int64_t)(dplus * NB + e) * n + pc] : 0.0;
      roffd[(ic * 2 + 1) * NB + e] = live ? offd[(int64_t)(dminus * NB + e) * n + nbp] : 0.0;
    }
  }
}

// reference layout -> internal (used when a caller hands us its own ws arrays)
__global__ void k_import_system(Dims g, const int64_t* __restrict__ conn_id,
                                const double* __restrict__ rdiag, const double* __restrict__ roffd,
                                const double* __restrict__ rresid, double* diag, double* offd,
                                double* resid) {
  const int64_t n = g.n;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // natural cell
  if (c >= n) return;
  const int64_t pc = pos_of(g, c);
  for (int e = 0; e < NB; ++e) diag[(int64_t)e * n + pc] = rdiag[c * NB + e];
  if (resid)
    for (int r = 0; r < NU; ++r) resid[(int64_t)r * n + pc] = rresid[c * NU + r];
  int i, j, k;
  cell_ijk(g, c, i, j, k);
  for (int d = 0; d < NDIR; ++d) {
    const int64_t nb = neighbour(g, c, i, j, k, d);
    if (nb < 0) {
      for (int e = 0; e < NB; ++e) offd[(int64_t)(d * NB + e) * n + pc] = 0.0;
      continue;
    }
    int64_t ic;
    int side;
    if (d >= DXP) { ic = conn_id[(d - DXP) * n + c]; side = 0; }
    else { ic = conn_id[(2 - d) * n + nb]; side = 1; }
    for (int e = 0; e < NB; ++e) offd[(int64_t)(d * NB + e) * n + pc] = roffd[(ic * 2 + side) * NB + e];
  }
}

// host-layout state (the reference's State arrays + accn (n, NU)) staged in
// one device buffer -> SoA state / accn in storage order
__global__ void k_stage_state(Dims g, const double* __restrict__ stage, double* __restrict__ st,
                              double* __restrict__ accn, int64_t c0, int64_t c1) {
  const int64_t n = g.n;
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // natural cell
  if (c >= c1) return;
  const int64_t p = pos_of(g, c);
  const double* sp = stage;
  const double* sx = stage + n;
  const double* sy = sx + NCO * n;
  const double* rest = sy + NCG * n;          // t, sw, sg, cc
  const double* sa = rest + 4 * n;            // accn (n, NU)
  st[p] = sp[c];
#pragma unroll
  for (int i = 0; i < NCO; ++i) st[(int64_t)(1 + i) * n + p] = sx[c * NCO + i];
#pragma unroll
  for (int j = 0; j < NCG; ++j) st[(int64_t)(1 + NCO + j) * n + p] = sy[c * NCG + j];
#pragma unroll
  for (int q = 0; q < 4; ++q) st[(int64_t)(CT + q) * n + p] = rest[q * n + c];
  if (accn)
#pragma unroll
    for (int r = 0; r < NU; ++r) accn[(int64_t)r * n + p] = sa[c * NU + r];
}

// SoA (storage order) -> AoS (n, NU) natural order, for a host download
__global__ void k_unstage_rows(Dims g, const double* __restrict__ v, double* __restrict__ out,
                               int64_t c0, int64_t c1) {
  const int64_t n = g.n;
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int64_t p = pos_of(g, c);
#pragma unroll
  for (int r = 0; r < NU; ++r) out[c * NU + r] = v[(int64_t)r * n + p];
}

// natural-order SoA (rows x n) <-> storage positions
template <typename T>
__global__ void k_to_pos(Dims g, int rows, const T* __restrict__ src, T* __restrict__ dst) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int64_t p = pos_of(g, c);
  for (int r = 0; r < rows; ++r) dst[(int64_t)r * g.n + p] = src[(int64_t)r * g.n + c];
}
template <typename T>
__global__ void k_from_pos(Dims g, int rows, const T* __restrict__ src, T* __restrict__ dst) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int64_t p = pos_of(g, c);
  for (int r = 0; r < rows; ++r) dst[(int64_t)r * g.n + c] = src[(int64_t)r * g.n + p];
}

}  // namespace isc
