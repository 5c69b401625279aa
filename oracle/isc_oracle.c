/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference simulator's Newton hot path
 * (iscsim, arxiv 1811.11992). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product (paper_1811_11992_b200) never links or calls it.
 *
 * Layouts follow the reference's numpy arrays exactly (row-major AoS):
 *   per cell  pot (3) dpot (3,nu) beta (3) dbeta (3,nu) hph (3) dhph (3,nu)
 *             yfull (nf) dyfull (nf,nu) gam (3) dgam (3,nu) pcv (2) dpcv (2)
 *             kr3 (3) dkr3 (3,2) ktd (1+nu) acc (nu) dacc (nu,nu) src (nu)
 *             dsrc (nu,nu)
 *   per conn  flux (nu) dfa (nu,nu) dfb (nu,nu) upw (3) int8
 *   system    resid (n,nu) diag (n,nu,nu) offd (m,2,nu,nu)
 *
 * Arithmetic mirrors the reference operation by operation (no FMA
 * contraction: build with -ffp-contract=off), integer powers are expanded
 * the way numba lowers `x ** <int literal>` (square-and-multiply), and the
 * transcendental calls go to the same glibc libm numba calls, so on the same
 * host the oracle reproduces the reference bit for bit in most entries.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/iscsim/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RANKINE 459.67          /* _props.py:19 */
#define R_GAS 10.7316           /* _props.py:20 */
#define R_ARR 1.9859            /* _props.py:21 */
#define PSI_PER_FT (1.0 / 144.0) /* _kernels.py:46 */

/* column indices of the flattened tables, _kernels.py:48-63 */
enum { L_RHO = 0, L_CP, L_CT1, L_CT2, L_CPT, L_AVISC, L_BVISC, L_HVR, L_EV, L_TCF, NLIQ };
enum { G_M = 0, G_TCR, G_PC, G_AVG, G_BVG, G_CPG1, G_CPG2, G_CPG3, G_CPG4, NGASP };
enum {
  RK_CPOR = 0, RK_CTPOR, RK_CPTPOR, RK_MODE, RK_CP1, RK_CP2, RK_COKE_CP,
  RK_RHO_COKE, RK_KTW, RK_KTO, RK_KTG, RK_KTR, RK_KTC, RK_PREF, RK_TREF,
  RK_EPS_PER, RK_KROCW, NRK
};

#define MAXNU 24
#define MAXNF 20

typedef struct {
  int64_t nco, ncg, heavy, nreac, nswt, nslt;
  const double *liq, *gasp, *kv, *rockp;
  const double *swt_s, *swt_krw, *swt_krow, *swt_pcow;
  const double *slt_s, *slt_krg, *slt_krog, *slt_pcog;
  const int64_t *law;
  const double *rcoef, *nmat;
  const int64_t *fuel, *ox;
  double ccmax;
} OrcModel;

static inline double ipow3(double t) { return t * (t * t); }
static inline double ipow4(double t) { double s = t * t; return s * s; }
static inline double ipow5(double t) { double s = t * t; return t * (s * s); }

/* ---------------------------------------------------------------- _props.py */

/* _props.py:24-41 */
static void k_value(double kv1, double kv2, double kv3, double kv4, double kv5,
                    double p, double t, double *k, double *dkdp, double *dkdt) {
  double pref = kv1 / p + kv2 * p + kv3;
  double dpref = -kv1 / (p * p) + kv2;
  if (pref == 0.0 && dpref == 0.0) { *k = 0.0; *dkdp = 0.0; *dkdt = 0.0; return; }
  double tdiff = t - kv5;
  double e = exp(kv4 / tdiff);
  *k = pref * e;
  *dkdp = dpref * e;
  *dkdt = -(*k) * kv4 / (tdiff * tdiff);
}

/* _props.py:44-50 */
static void per_factor(double s, double eps, double *f, double *dfds) {
  double den = s + eps;
  *f = s / den;
  *dfds = eps / (den * den);
}

/* _props.py:53-65 */
static void liquid_density(double rho_ref, double cp, double ct1, double ct2, double cpt,
                           double p_ref, double t_ref, double p, double t,
                           double *rho, double *drdp, double *drdt) {
  double dp = p - p_ref, dt = t - t_ref;
  double expo = cp * dp - ct1 * dt - 0.5 * ct2 * dt * dt + cpt * dp * dt;
  *rho = rho_ref * exp(expo);
  *drdp = *rho * (cp + cpt * dt);
  *drdt = *rho * (-ct1 - ct2 * dt + cpt * dp);
}

/* _props.py:68-104 */
double orc_cubic_largest_root(double a, double b) {
  double c1 = a - b - b * b;
  double c0 = -a * b;
  double p = c1 - 1.0 / 3.0;
  double q = -2.0 / 27.0 + c1 / 3.0 + c0;
  double disc = 0.25 * q * q + p * p * p / 27.0;
  double z;
  if (disc >= 0.0) {
    double s = sqrt(disc);
    double u = -0.5 * q + s, v = -0.5 * q - s;
    double cu = copysign(pow(fabs(u), 1.0 / 3.0), u);
    double cv = copysign(pow(fabs(v), 1.0 / 3.0), v);
    z = cu + cv + 1.0 / 3.0;
  } else {
    double rp = sqrt(-p / 3.0);
    double arg = 3.0 * q / (2.0 * p * rp);
    if (arg > 1.0) arg = 1.0;
    else if (arg < -1.0) arg = -1.0;
    double theta = acos(arg) / 3.0;
    z = 2.0 * rp * cos(theta) + 1.0 / 3.0;
  }
  for (int it = 0; it < 3; ++it) {
    double g = ((z - 1.0) * z + c1) * z + c0;
    double gp = (3.0 * z - 2.0) * z + c1;
    if (gp == 0.0) break;
    z -= g / gp;
  }
  return z;
}

/* _props.py:107-150; w, tcrit_r, pcrit have length n; fills dzdw */
double orc_z_factor_mix(int n, const double *w, const double *tcrit_r, const double *pcrit,
                        double p, double t, double *dzdw, double *dzdp, double *dzdt) {
  double tr = t + RANKINE;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < n; ++i) {
    double ti = tcrit_r[i];
    double bi = ti / pcrit[i];
    a += w[i] * ti * sqrt(bi);
    b += w[i] * bi;
  }
  if (a <= 0.0 || b <= 0.0) {
    for (int i = 0; i < n; ++i) dzdw[i] = 0.0;
    *dzdp = 0.0; *dzdt = 0.0;
    return 1.0;
  }
  double coef_a = 0.427480 * p * pow(a, 1.5) * pow(b, 0.25) / pow(tr, 2.5);
  double coef_b = 0.086640 * p * b / tr;
  double z = orc_cubic_largest_root(coef_a, coef_b);
  double gp = (3.0 * z - 2.0) * z + (coef_a - coef_b - coef_b * coef_b);
  if (fabs(gp) < 1e-30) gp = 1e-30;
  double dzda = -(z - coef_b) / gp;
  double dzdb = -((-1.0 - 2.0 * coef_b) * z - coef_a) / gp;
  double da_dp = coef_a / p, db_dp = coef_b / p;
  double da_dtr = -2.5 * coef_a / tr, db_dtr = -coef_b / tr;
  *dzdp = dzda * da_dp + dzdb * db_dp;
  *dzdt = dzda * da_dtr + dzdb * db_dtr;
  for (int i = 0; i < n; ++i) {
    double ti = tcrit_r[i];
    double bi = ti / pcrit[i];
    double dai = ti * sqrt(bi);
    double da_dw = 1.5 * coef_a / a * dai + 0.25 * coef_a / b * bi;
    double db_dw = coef_b / b * bi;
    dzdw[i] = dzda * da_dw + dzdb * db_dw;
  }
  return z;
}

/* _props.py:163-169 */
static void liquid_viscosity(double av, double bv, double t, double *mu, double *dmu) {
  double tr = t + RANKINE;
  *mu = av * exp(bv / tr);
  *dmu = -(*mu) * bv / (tr * tr);
}

/* _props.py:172-178 */
static void gas_component_viscosity(double av, double bv, double t, double *mu, double *dmu) {
  double tr = t + RANKINE;
  *mu = av * pow(tr, bv);
  *dmu = *mu * bv / tr;
}

/* _props.py:181-191 */
static void gas_enthalpy(double c1, double c2, double c3, double c4, double t_ref, double t,
                         double *h, double *dh) {
  *h = c1 * (t - t_ref) + c2 / 2.0 * (t * t - t_ref * t_ref) +
       c3 / 3.0 * (ipow3(t) - ipow3(t_ref)) + c4 / 4.0 * (ipow4(t) - ipow4(t_ref));
  *dh = c1 + c2 * t + c3 * t * t + c4 * ipow3(t);
}

/* _props.py:194-205 */
static void vaporization_enthalpy(double hvr, double ev, double tcrit, double t,
                                  double *h, double *dh) {
  if (t >= tcrit || hvr == 0.0) { *h = 0.0; *dh = 0.0; return; }
  double dt = tcrit - t;
  *h = hvr * pow(dt, ev);
  *dh = -ev * hvr * pow(dt, ev - 1.0);
}

/* _props.py:216-228 */
static void porosity(double phi_ref, double cpor, double ctpor, double cptpor, double p_ref,
                     double t_ref, int nonlinear, double p, double t,
                     double *phi, double *dp_, double *dt_) {
  double dp = p - p_ref, dt = t - t_ref;
  double ctot = cpor * dp - ctpor * dt + cptpor * dp * dt;
  double dc_dp = cpor + cptpor * dt;
  double dc_dt = -ctpor + cptpor * dp;
  if (nonlinear) {
    *phi = phi_ref * exp(ctot);
    *dp_ = *phi * dc_dp; *dt_ = *phi * dc_dt;
    return;
  }
  *phi = phi_ref * (1.0 + ctot);
  *dp_ = phi_ref * dc_dp; *dt_ = phi_ref * dc_dt;
}

/* _props.py:231-237 */
static void arrhenius(double freq, double ea, double t, double *k, double *dk) {
  double tr = t + RANKINE;
  *k = freq * exp(-ea / (R_ARR * tr));
  *dk = *k * ea / (R_ARR * tr * tr);
}

/* _props.py:245-268; out = r, dT, dpp, dfm, dcc */
static void reaction_rate_one(int64_t law, double a, double ea, double t, double pp,
                              double fm, double cc, double ccmax, double *o) {
  double k, dk;
  arrhenius(a, ea, t, &k, &dk);
  if (law == 0) { o[0] = k * pp * fm; o[1] = dk * pp * fm; o[2] = k * fm; o[3] = k * pp; o[4] = 0.0; return; }
  if (law == 1) { o[0] = k * pp * cc; o[1] = dk * pp * cc; o[2] = k * cc; o[3] = 0.0; o[4] = k * pp; return; }
  double ratio = cc / ccmax;
  double lim = 1.0 - ipow5(ratio);
  if (lim <= 0.0) { o[0] = o[1] = o[2] = o[3] = o[4] = 0.0; return; }
  double dlim = -5.0 * ipow4(ratio) / ccmax;
  o[0] = k * fm * lim; o[1] = dk * fm * lim; o[2] = 0.0; o[3] = k * lim; o[4] = k * fm * dlim;
}

/* _props.py:271-291; o = kro, d_krow, d_krw, d_krog, d_krg */
static void stone2(double krocw, double krow, double krw, double krog, double krg, double *o) {
  o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
  if (krocw <= 0.0) return;
  double fo = krow / krocw + krw;
  double fg = krog / krocw + krg;
  double raw = krocw * (fo * fg - krw - krg);
  if (raw <= 0.0) return;
  if (raw >= 1.0) { o[0] = 1.0; return; }
  o[0] = raw; o[1] = fg; o[2] = krocw * (fg - 1.0); o[3] = fo; o[4] = krocw * (fo - 1.0);
}

/* _props.py:294-315 */
static void interp1(int64_t n, const double *xs, const double *ys, double x, double *y, double *dy) {
  if (x <= xs[0]) { *y = ys[0]; *dy = 0.0; return; }
  if (x >= xs[n - 1]) { *y = ys[n - 1]; *dy = 0.0; return; }
  int64_t lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) / 2;
    if (xs[mid] <= x) lo = mid; else hi = mid;
  }
  double slope = (ys[lo + 1] - ys[lo]) / (xs[lo + 1] - xs[lo]);
  *y = ys[lo] + slope * (x - xs[lo]);
  *dy = slope;
}

/* _props.py:318-327 */
static void harmonic_pair(double a, double b, double *h, double *da, double *db) {
  double s = a + b;
  if (a <= 0.0 || b <= 0.0 || s <= 0.0) { *h = 0.0; *da = 0.0; *db = 0.0; return; }
  *h = 2.0 * a * b / s;
  *da = 2.0 * b * b / (s * s);
  *db = 2.0 * a * a / (s * s);
}

/* scalar entry points for the property goldens (tests only) */
void orc_props_k_value(const double *kv, double p, double t, double *out) {
  k_value(kv[0], kv[1], kv[2], kv[3], kv[4], p, t, &out[0], &out[1], &out[2]);
}
void orc_props_liquid_density(const double *c, double p, double t, double *out) {
  liquid_density(c[0], c[1], c[2], c[3], c[4], c[5], c[6], p, t, &out[0], &out[1], &out[2]);
}
void orc_props_liquid_viscosity(double a, double b, double t, double *out) { liquid_viscosity(a, b, t, &out[0], &out[1]); }
void orc_props_gas_component_viscosity(double a, double b, double t, double *out) { gas_component_viscosity(a, b, t, &out[0], &out[1]); }
void orc_props_gas_enthalpy(const double *c, double t_ref, double t, double *out) { gas_enthalpy(c[0], c[1], c[2], c[3], t_ref, t, &out[0], &out[1]); }
void orc_props_vaporization_enthalpy(double hvr, double ev, double tc, double t, double *out) { vaporization_enthalpy(hvr, ev, tc, t, &out[0], &out[1]); }
void orc_props_porosity(const double *c, int nonlinear, double p, double t, double *out) {
  porosity(c[0], c[1], c[2], c[3], c[4], c[5], nonlinear, p, t, &out[0], &out[1], &out[2]);
}
void orc_props_arrhenius(double a, double ea, double t, double *out) { arrhenius(a, ea, t, &out[0], &out[1]); }
void orc_props_stone2(const double *c, double *out) { stone2(c[0], c[1], c[2], c[3], c[4], out); }
void orc_props_reaction_rate(int64_t law, double a, double ea, double t, double pp, double fm,
                             double cc, double ccmax, double *out) {
  reaction_rate_one(law, a, ea, t, pp, fm, cc, ccmax, out);
}

/* ------------------------------------------------------------- _kernels.py */

typedef struct {
  double *pot, *dpot, *beta, *dbeta, *hph, *dhph, *yfull, *dyfull;
  double *gam, *dgam, *pcv, *dpcv, *kr3, *dkr3, *ktd;
  double *acc, *dacc, *src, *dsrc;
} CellOut;

/* _kernels.py:66-610 — one cell; returns 1 (ok) or 0 (pore space exhausted). */
static int cell_eval(const OrcModel *M, double p, double t, double sw, double sg,
                     const double *x, const double *y, double cc, double phi_ref_c,
                     const CellOut *O) {
  const int nco = (int)M->nco, ncg = (int)M->ncg;
  const int nf = 1 + nco + ncg, nu = nco + ncg + 5;
  const int ct = 1 + nco + ncg, csw = ct + 1, csg = ct + 2, ccc = ct + 3;
  const int row_e = ct, row_os = ct + 1, row_gs = ct + 2, row_ck = ct + 3;
  const double *liq = M->liq, *gasp = M->gasp, *kv = M->kv, *rk = M->rockp;
  double so = 1.0 - sw - sg;
#define LQ(r, c) liq[(r) * NLIQ + (c)]
#define GP(r, c) gasp[(r) * NGASP + (c)]
#define D2(a, r, u) a[(r) * nu + (u)]

  memset(O->acc, 0, sizeof(double) * nu);
  memset(O->src, 0, sizeof(double) * nu);
  memset(O->dacc, 0, sizeof(double) * nu * nu);
  memset(O->dsrc, 0, sizeof(double) * nu * nu);
  memset(O->pot, 0, sizeof(double) * 3);
  memset(O->beta, 0, sizeof(double) * 3);
  memset(O->hph, 0, sizeof(double) * 3);
  memset(O->gam, 0, sizeof(double) * 3);
  memset(O->kr3, 0, sizeof(double) * 3);
  memset(O->dpot, 0, sizeof(double) * 3 * nu);
  memset(O->dbeta, 0, sizeof(double) * 3 * nu);
  memset(O->dhph, 0, sizeof(double) * 3 * nu);
  memset(O->dgam, 0, sizeof(double) * 3 * nu);
  memset(O->dkr3, 0, sizeof(double) * 6);
  memset(O->yfull, 0, sizeof(double) * nf);
  memset(O->dyfull, 0, sizeof(double) * nf * nu);
  memset(O->ktd, 0, sizeof(double) * (nu + 1));

  double phi, dphi_p, dphi_t;
  porosity(phi_ref_c, rk[RK_CPOR], rk[RK_CTPOR], rk[RK_CPTPOR], rk[RK_PREF], rk[RK_TREF],
           rk[RK_MODE] != 0.0, p, t, &phi, &dphi_p, &dphi_t);
  double rho_coke = rk[RK_RHO_COKE];
  double phif, dphif_cc;
  if (rho_coke > 0.0 && isfinite(rho_coke)) { phif = phi - cc / rho_coke; dphif_cc = -1.0 / rho_coke; }
  else { phif = phi; dphif_cc = 0.0; }
  if (phif <= 0.0) return 0;
  double t_ref = rk[RK_TREF], eps_per = rk[RK_EPS_PER];

  /* water phase, _kernels.py:139-156 */
  double rw, drw_p, drw_t, muw, dmuw_t, hgw, dhgw_t, hvw, dhvw_t;
  liquid_density(LQ(0, L_RHO), LQ(0, L_CP), LQ(0, L_CT1), LQ(0, L_CT2), LQ(0, L_CPT),
                 rk[RK_PREF], t_ref, p, t, &rw, &drw_p, &drw_t);
  liquid_viscosity(LQ(0, L_AVISC), LQ(0, L_BVISC), t, &muw, &dmuw_t);
  gas_enthalpy(GP(0, G_CPG1), GP(0, G_CPG2), GP(0, G_CPG3), GP(0, G_CPG4), t_ref, t, &hgw, &dhgw_t);
  vaporization_enthalpy(LQ(0, L_HVR), LQ(0, L_EV), LQ(0, L_TCF), t, &hvw, &dhvw_t);
  double hw = hgw - hvw, dhw_t = dhgw_t - dhvw_t;
  double uw = hw - p / rw;
  double duw_p = -1.0 / rw + p * drw_p / (rw * rw);
  double duw_t = dhw_t + p * drw_t / (rw * rw);

  /* oil phase, _kernels.py:158-218 */
  double rho_i[MAXNF], drho_i_p[MAXNF], drho_i_t[MAXNF], mu_i[MAXNF], dmu_i_t[MAXNF];
  double hli[MAXNF], dhli_t[MAXNF];
  for (int i = 0; i < nco; ++i) {
    int r = i + 1;
    liquid_density(LQ(r, L_RHO), LQ(r, L_CP), LQ(r, L_CT1), LQ(r, L_CT2), LQ(r, L_CPT),
                   rk[RK_PREF], t_ref, p, t, &rho_i[i], &drho_i_p[i], &drho_i_t[i]);
    liquid_viscosity(LQ(r, L_AVISC), LQ(r, L_BVISC), t, &mu_i[i], &dmu_i_t[i]);
    double hg_i, dhg_i, hv_i, dhv_i;
    gas_enthalpy(GP(r, G_CPG1), GP(r, G_CPG2), GP(r, G_CPG3), GP(r, G_CPG4), t_ref, t, &hg_i, &dhg_i);
    vaporization_enthalpy(LQ(r, L_HVR), LQ(r, L_EV), LQ(r, L_TCF), t, &hv_i, &dhv_i);
    hli[i] = hg_i - hv_i;
    dhli_t[i] = dhg_i - dhv_i;
  }
  double inv_ro = 0.0, dinv_p = 0.0, dinv_t = 0.0;
  for (int i = 0; i < nco; ++i) {
    inv_ro += x[i] / rho_i[i];
    dinv_p -= x[i] * drho_i_p[i] / (rho_i[i] * rho_i[i]);
    dinv_t -= x[i] * drho_i_t[i] / (rho_i[i] * rho_i[i]);
  }
  if (inv_ro < 1e-12) { inv_ro = 1e-12; dinv_p = 0.0; dinv_t = 0.0; }
  double ro = 1.0 / inv_ro, ro2 = ro * ro;
  double dro_p = -ro2 * dinv_p, dro_t = -ro2 * dinv_t;
  double lnmu = 0.0, dlnmu_t = 0.0;
  for (int i = 0; i < nco; ++i) {
    lnmu += x[i] * log(mu_i[i]);
    dlnmu_t += x[i] * dmu_i_t[i] / mu_i[i];
  }
  double muo = exp(lnmu), dmuo_t = muo * dlnmu_t;
  double ho = 0.0, dho_t = 0.0;
  for (int i = 0; i < nco; ++i) { ho += x[i] * hli[i]; dho_t += x[i] * dhli_t[i]; }
  double uo = ho - p / ro;
  double duo_p = -1.0 / ro + p * dro_p / ro2;
  double duo_t = dho_t + p * dro_t / ro2;

  /* K-values and yfull, _kernels.py:220-252 */
  double *yfull = O->yfull, *dyfull = O->dyfull;
  double kw, dkw_p, dkw_t, fw, dfw_s;
  k_value(kv[0], kv[1], kv[2], kv[3], kv[4], p, t, &kw, &dkw_p, &dkw_t);
  per_factor(sw, eps_per, &fw, &dfw_s);
  yfull[0] = fw * kw;
  D2(dyfull, 0, 0) = fw * dkw_p;
  D2(dyfull, 0, ct) = fw * dkw_t;
  D2(dyfull, 0, csw) = dfw_s * kw;
  double fo_h, dfo_h;
  per_factor(so, eps_per, &fo_h, &dfo_h);
  for (int i = 0; i < nco; ++i) {
    const double *kr = kv + (1 + i) * 5;
    double ki, dki_p, dki_t;
    k_value(kr[0], kr[1], kr[2], kr[3], kr[4], p, t, &ki, &dki_p, &dki_t);
    int c = 1 + i;
    if (i == M->heavy) {
      yfull[c] = fo_h * ki * x[i];
      D2(dyfull, c, 0) = fo_h * dki_p * x[i];
      D2(dyfull, c, ct) = fo_h * dki_t * x[i];
      D2(dyfull, c, 1 + i) = fo_h * ki;
      D2(dyfull, c, csw) = -dfo_h * ki * x[i];
      D2(dyfull, c, csg) = -dfo_h * ki * x[i];
    } else {
      yfull[c] = ki * x[i];
      D2(dyfull, c, 0) = dki_p * x[i];
      D2(dyfull, c, ct) = dki_t * x[i];
      D2(dyfull, c, 1 + i) = ki;
    }
  }
  for (int j = 0; j < ncg; ++j) {
    int c = 1 + nco + j;
    yfull[c] = y[j];
    D2(dyfull, c, 1 + nco + j) = 1.0;
  }

  /* gas phase, _kernels.py:254-328 */
  double tcr[MAXNF], pcr[MAXNF], dzdw[MAXNF];
  for (int c = 0; c < nf; ++c) { tcr[c] = GP(c, G_TCR); pcr[c] = GP(c, G_PC); }
  double dz_p, dz_t;
  double z = orc_z_factor_mix(nf, yfull, tcr, pcr, p, t, dzdw, &dz_p, &dz_t);
  double dz[MAXNU];
  for (int u = 0; u < nu; ++u) dz[u] = 0.0;
  dz[0] = dz_p;
  dz[ct] += dz_t;
  for (int c = 0; c < nf; ++c)
    if (dzdw[c] != 0.0)
      for (int u = 0; u < nu; ++u) dz[u] += dzdw[c] * D2(dyfull, c, u);
  double tr = t + RANKINE;
  double rg = p / (z * R_GAS * tr);
  double drg[MAXNU];
  for (int u = 0; u < nu; ++u) drg[u] = -rg * dz[u] / z;
  drg[0] += rg / p;
  drg[ct] -= rg / tr;
  double mgbar = 0.0, dmg[MAXNU];
  for (int u = 0; u < nu; ++u) dmg[u] = 0.0;
  for (int c = 0; c < nf; ++c) {
    mgbar += yfull[c] * GP(c, G_M);
    for (int u = 0; u < nu; ++u) dmg[u] += GP(c, G_M) * D2(dyfull, c, u);
  }
  double wsum = 0.0, musum = 0.0, dmusum_t = 0.0, sqm[MAXNF], muc[MAXNF];
  for (int c = 0; c < nf; ++c) {
    sqm[c] = sqrt(GP(c, G_M));
    double m_c, dm_c;
    gas_component_viscosity(GP(c, G_AVG), GP(c, G_BVG), t, &m_c, &dm_c);
    muc[c] = m_c;
    wsum += yfull[c] * sqm[c];
    musum += yfull[c] * m_c * sqm[c];
    dmusum_t += yfull[c] * dm_c * sqm[c];
  }
  double dmug[MAXNU], mug;
  for (int u = 0; u < nu; ++u) dmug[u] = 0.0;
  if (wsum > 1e-30) {
    mug = musum / wsum;
    dmug[ct] += dmusum_t / wsum;
    for (int c = 0; c < nf; ++c) {
      double dmy = sqm[c] * (muc[c] - mug) / wsum;
      if (dmy != 0.0)
        for (int u = 0; u < nu; ++u) dmug[u] += dmy * D2(dyfull, c, u);
    }
  } else {
    mug = 1.0;
  }
  double hg = 0.0, dhg[MAXNU];
  for (int u = 0; u < nu; ++u) dhg[u] = 0.0;
  for (int c = 0; c < nf; ++c) {
    double h_c, dh_c;
    gas_enthalpy(GP(c, G_CPG1), GP(c, G_CPG2), GP(c, G_CPG3), GP(c, G_CPG4), t_ref, t, &h_c, &dh_c);
    hg += yfull[c] * h_c;
    dhg[ct] += yfull[c] * dh_c;
    if (h_c != 0.0)
      for (int u = 0; u < nu; ++u) dhg[u] += h_c * D2(dyfull, c, u);
  }
  double ug = hg - p / rg, dug[MAXNU];
  for (int u = 0; u < nu; ++u) dug[u] = dhg[u] + p * drg[u] / (rg * rg);
  dug[0] -= 1.0 / rg;

  /* relperm and capillary pressure, _kernels.py:330-353 */
  double krw, dkrw, krow, dkrow, pcow, dpcow, krg, dkrg, krog, dkrog, pcog, dpcog, st[5];
  interp1(M->nswt, M->swt_s, M->swt_krw, sw, &krw, &dkrw);
  interp1(M->nswt, M->swt_s, M->swt_krow, sw, &krow, &dkrow);
  interp1(M->nswt, M->swt_s, M->swt_pcow, sw, &pcow, &dpcow);
  interp1(M->nslt, M->slt_s, M->slt_krg, sg, &krg, &dkrg);
  interp1(M->nslt, M->slt_s, M->slt_krog, sg, &krog, &dkrog);
  interp1(M->nslt, M->slt_s, M->slt_pcog, sg, &pcog, &dpcog);
  stone2(rk[RK_KROCW], krow, krw, krog, krg, st);
  double kro = st[0];
  double dkro_sw = st[1] * dkrow + st[2] * dkrw;
  double dkro_sg = st[3] * dkrog + st[4] * dkrg;
  O->kr3[0] = krw; O->kr3[1] = kro; O->kr3[2] = krg;
  O->dkr3[0] = dkrw; O->dkr3[2] = dkro_sw; O->dkr3[3] = dkro_sg; O->dkr3[5] = dkrg;
  O->pcv[0] = pcow; O->pcv[1] = pcog;
  O->dpcv[0] = dpcow; O->dpcv[1] = dpcog;

  /* specific weights, _kernels.py:355-373 */
  double *gam = O->gam, *dgam = O->dgam;
  double m_w = GP(0, G_M);
  gam[0] = rw * m_w * PSI_PER_FT;
  D2(dgam, 0, 0) = drw_p * m_w * PSI_PER_FT;
  D2(dgam, 0, ct) = drw_t * m_w * PSI_PER_FT;
  double mobar = 0.0;
  for (int i = 0; i < nco; ++i) mobar += x[i] * GP(1 + i, G_M);
  gam[1] = ro * mobar * PSI_PER_FT;
  D2(dgam, 1, 0) = dro_p * mobar * PSI_PER_FT;
  D2(dgam, 1, ct) = dro_t * mobar * PSI_PER_FT;
  for (int i = 0; i < nco; ++i) {
    double dro_xi = -ro2 / rho_i[i];
    D2(dgam, 1, 1 + i) = (dro_xi * mobar + ro * GP(1 + i, G_M)) * PSI_PER_FT;
  }
  for (int u = 0; u < nu; ++u) D2(dgam, 2, u) = (drg[u] * mgbar + rg * dmg[u]) * PSI_PER_FT;
  gam[2] = rg * mgbar * PSI_PER_FT;

  /* phase pressures, _kernels.py:375-385 */
  double *pot = O->pot, *dpot = O->dpot;
  pot[0] = p - pcow; D2(dpot, 0, 0) = 1.0; D2(dpot, 0, csw) = -dpcow;
  pot[1] = p; D2(dpot, 1, 0) = 1.0;
  pot[2] = p + pcog; D2(dpot, 2, 0) = 1.0; D2(dpot, 2, csg) = dpcog;

  /* mobility-density products, _kernels.py:387-408 */
  double *beta = O->beta, *dbeta = O->dbeta;
  beta[0] = rw * krw / muw;
  if (krw > 0.0 || dkrw != 0.0) {
    D2(dbeta, 0, 0) = drw_p * krw / muw;
    D2(dbeta, 0, ct) = (drw_t * krw - rw * krw * dmuw_t / muw) / muw;
    D2(dbeta, 0, csw) = rw * dkrw / muw;
  }
  beta[1] = ro * kro / muo;
  if (kro > 0.0 || dkro_sw != 0.0 || dkro_sg != 0.0) {
    D2(dbeta, 1, 0) = dro_p * kro / muo;
    D2(dbeta, 1, ct) = (dro_t * kro - ro * kro * dmuo_t / muo) / muo;
    D2(dbeta, 1, csw) = ro * dkro_sw / muo;
    D2(dbeta, 1, csg) = ro * dkro_sg / muo;
    for (int i = 0; i < nco; ++i) {
      double dro_xi = -ro2 / rho_i[i];
      double dmuo_xi = muo * log(mu_i[i]);
      D2(dbeta, 1, 1 + i) = (dro_xi * kro - ro * kro * dmuo_xi / muo) / muo;
    }
  }
  if (krg > 0.0 || dkrg != 0.0) {
    for (int u = 0; u < nu; ++u) D2(dbeta, 2, u) = (drg[u] * krg - rg * krg * dmug[u] / mug) / mug;
    D2(dbeta, 2, csg) += rg * dkrg / mug;
  }
  beta[2] = rg * krg / mug;

  /* phase enthalpies, _kernels.py:410-419 */
  double *hph = O->hph, *dhph = O->dhph;
  hph[0] = hw; D2(dhph, 0, ct) = dhw_t;
  hph[1] = ho; D2(dhph, 1, ct) = dho_t;
  for (int i = 0; i < nco; ++i) D2(dhph, 1, 1 + i) = hli[i];
  hph[2] = hg;
  for (int u = 0; u < nu; ++u) D2(dhph, 2, u) = dhg[u];

  /* conductivity, _kernels.py:421-428 */
  double *ktd = O->ktd;
  double br = sw * rk[RK_KTW] + so * rk[RK_KTO] + sg * rk[RK_KTG];
  ktd[0] = phif * br + (1.0 - phi) * rk[RK_KTR] + cc * rk[RK_KTC];
  ktd[1 + 0] = dphi_p * br - dphi_p * rk[RK_KTR];
  ktd[1 + ct] = dphi_t * br - dphi_t * rk[RK_KTR];
  ktd[1 + csw] = phif * (rk[RK_KTW] - rk[RK_KTO]);
  ktd[1 + csg] = phif * (rk[RK_KTG] - rk[RK_KTO]);
  ktd[1 + ccc] = dphif_cc * br + rk[RK_KTC];

  /* accumulation, _kernels.py:430-518 */
  double *acc = O->acc, *dacc = O->dacc;
  double mw_g = rg * sg;
  double a_w = rw * sw + mw_g * yfull[0];
  acc[0] = phif * a_w;
  for (int u = 0; u < nu; ++u) {
    double d = (drg[u] * sg * yfull[0] + mw_g * D2(dyfull, 0, u));
    if (u == 0) d += drw_p * sw;
    else if (u == ct) d += drw_t * sw;
    else if (u == csw) d += rw;
    if (u == csg) d += rg * yfull[0];
    D2(dacc, 0, u) = phif * d;
  }
  D2(dacc, 0, 0) += dphi_p * a_w;
  D2(dacc, 0, ct) += dphi_t * a_w;
  D2(dacc, 0, ccc) += dphif_cc * a_w;
  for (int i = 0; i < nco; ++i) {
    int c = 1 + i;
    double a_i = ro * so * x[i] + mw_g * yfull[c];
    acc[c] = phif * a_i;
    for (int u = 0; u < nu; ++u) {
      double d = drg[u] * sg * yfull[c] + mw_g * D2(dyfull, c, u);
      if (u == 0) d += dro_p * so * x[i];
      else if (u == ct) d += dro_t * so * x[i];
      else if (u == csw || u == csg) d += -ro * x[i] + (u == csg ? rg * yfull[c] : 0.0);
      if (1 <= u && u < 1 + nco) {
        double dro_xi = -ro2 / rho_i[u - 1];
        d += dro_xi * so * x[i];
        if (u - 1 == i) d += ro * so;
      }
      D2(dacc, c, u) = phif * d;
    }
    D2(dacc, c, 0) += dphi_p * a_i;
    D2(dacc, c, ct) += dphi_t * a_i;
    D2(dacc, c, ccc) += dphif_cc * a_i;
  }
  for (int j = 0; j < ncg; ++j) {
    int c = 1 + nco + j;
    double a_j = mw_g * y[j];
    acc[c] = phif * a_j;
    for (int u = 0; u < nu; ++u) {
      double d = drg[u] * sg * y[j];
      if (u == csg) d += rg * y[j];
      if (u == 1 + nco + j) d += mw_g;
      D2(dacc, c, u) = phif * d;
    }
    D2(dacc, c, 0) += dphi_p * a_j;
    D2(dacc, c, ct) += dphi_t * a_j;
    D2(dacc, c, ccc) += dphif_cc * a_j;
  }
  /* energy */
  double ur = rk[RK_CP1] * (t - t_ref) + 0.5 * rk[RK_CP2] * (t * t - t_ref * t_ref);
  double dur_t = rk[RK_CP1] + rk[RK_CP2] * t; /* _props.py:208-213 */
  double uc = rk[RK_COKE_CP] * (t - t_ref);
  double duc_t = rk[RK_COKE_CP];
  double a_e = rw * sw * uw + ro * so * uo + mw_g * ug;
  acc[row_e] = phif * a_e + (1.0 - phi) * ur + cc * uc;
  for (int u = 0; u < nu; ++u) {
    double d = drg[u] * sg * ug + mw_g * dug[u];
    if (u == 0) {
      d += drw_p * sw * uw + rw * sw * duw_p;
      d += dro_p * so * uo + ro * so * duo_p;
    } else if (u == ct) {
      d += drw_t * sw * uw + rw * sw * duw_t;
      d += dro_t * so * uo + ro * so * duo_t;
    } else if (u == csw) {
      d += rw * uw - ro * uo;
    }
    if (u == csg) d += -ro * uo + rg * ug;
    if (1 <= u && u < 1 + nco) {
      int i = u - 1;
      double dro_xi = -ro2 / rho_i[i];
      double duo_xi = hli[i] + p * dro_xi / ro2;
      d += dro_xi * so * uo + ro * so * duo_xi;
    }
    D2(dacc, row_e, u) = phif * d;
  }
  D2(dacc, row_e, 0) += dphi_p * a_e - dphi_p * ur;
  D2(dacc, row_e, ct) += dphi_t * a_e - dphi_t * ur + (1.0 - phi) * dur_t + cc * duc_t;
  D2(dacc, row_e, ccc) += dphif_cc * a_e + uc;
  /* constraints, _kernels.py:520-531 */
  double sx = 0.0;
  for (int i = 0; i < nco; ++i) { sx += x[i]; D2(dacc, row_os, 1 + i) = 1.0; }
  acc[row_os] = sx - 1.0;
  double sy = 0.0;
  for (int c = 0; c < nf; ++c) {
    sy += yfull[c];
    for (int u = 0; u < nu; ++u) D2(dacc, row_gs, u) += D2(dyfull, c, u);
  }
  acc[row_gs] = sy - 1.0;
  acc[row_ck] = cc;
  D2(dacc, row_ck, ccc) = 1.0;

  /* reactions, _kernels.py:537-608 */
  double *src = O->src, *dsrc = O->dsrc;
  int nreac = (int)M->nreac;
  if (nreac > 0) {
    double pg = p + pcog;
    double ccr = cc > 0.0 ? cc : 0.0;
    double dpp[MAXNU], dfm[MAXNU], dr[MAXNU];
    for (int rr = 0; rr < nreac; ++rr) {
      int64_t oxi = M->ox[rr];
      for (int u = 0; u < nu; ++u) { dpp[u] = 0.0; dfm[u] = 0.0; }
      double pp = 0.0;
      if (oxi >= 0) {
        double y_ox = yfull[oxi];
        pp = y_ox * pg;
        if (pp > 0.0) {
          for (int u = 0; u < nu; ++u) dpp[u] = D2(dyfull, oxi, u) * pg;
          dpp[0] += y_ox;
          dpp[csg] += y_ox * dpcog;
        } else {
          pp = 0.0;
        }
      }
      int64_t fui = M->fuel[rr];
      double fm = 0.0;
      if (fui >= 0) {
        double xf = x[fui];
        fm = phif * so * ro * xf;
        if (fm > 0.0) {
          double base = so * ro * xf;
          dfm[0] = dphi_p * base + phif * so * dro_p * xf;
          dfm[ct] = dphi_t * base + phif * so * dro_t * xf;
          dfm[csw] = -phif * ro * xf;
          dfm[csg] = -phif * ro * xf;
          dfm[ccc] = dphif_cc * base;
          for (int i = 0; i < nco; ++i) {
            double dro_xi = -ro2 / rho_i[i];
            dfm[1 + i] = phif * so * dro_xi * xf;
          }
          dfm[1 + fui] += phif * so * ro;
        } else {
          fm = 0.0;
        }
      }
      double o[5];
      reaction_rate_one(M->law[rr], M->rcoef[rr * 3 + 0], M->rcoef[rr * 3 + 1], t, pp, fm, ccr,
                        M->ccmax, o);
      double r = o[0], dr_t = o[1], dr_pp = o[2], dr_fm = o[3], dr_cc = o[4];
      if (r == 0.0 && dr_t == 0.0 && dr_pp == 0.0 && dr_fm == 0.0 && dr_cc == 0.0) continue;
      for (int u = 0; u < nu; ++u) dr[u] = dr_pp * dpp[u] + dr_fm * dfm[u];
      dr[ct] += dr_t;
      if (dr_cc != 0.0 && cc >= 0.0) dr[ccc] += dr_cc;
      for (int c = 0; c < nf; ++c) {
        double s = M->nmat[c * nreac + rr];
        if (s != 0.0) {
          src[c] += s * r;
          for (int u = 0; u < nu; ++u) D2(dsrc, c, u) += s * dr[u];
        }
      }
      double s_ck = M->nmat[nf * nreac + rr];
      if (s_ck != 0.0) {
        src[row_ck] += s_ck * r;
        for (int u = 0; u < nu; ++u) D2(dsrc, row_ck, u) += s_ck * dr[u];
      }
      double h_r = M->rcoef[rr * 3 + 2];
      if (h_r != 0.0) {
        src[row_e] += h_r * r;
        for (int u = 0; u < nu; ++u) D2(dsrc, row_e, u) += h_r * dr[u];
      }
    }
  }
  return 1;
#undef LQ
#undef GP
#undef D2
}

/* _kernels.py:613-639 (prange over cells) */
void orc_cell_pass(const OrcModel *M, int64_t n, const double *p, const double *t,
                   const double *sw, const double *sg, const double *x, const double *y,
                   const double *cc, const double *phi_ref,
                   double *pot, double *dpot, double *beta, double *dbeta, double *hph,
                   double *dhph, double *yfull, double *dyfull, double *gam, double *dgam,
                   double *pcv, double *dpcv, double *kr3, double *dkr3, double *ktd,
                   double *acc, double *dacc, double *src, double *dsrc, uint8_t *ok) {
  const int64_t nco = M->nco, ncg = M->ncg, nf = 1 + nco + ncg, nu = nco + ncg + 5;
#pragma omp parallel for schedule(static) if (n > 256)
  for (int64_t c = 0; c < n; ++c) {
    CellOut O = {pot + 3 * c, dpot + 3 * nu * c, beta + 3 * c, dbeta + 3 * nu * c,
                 hph + 3 * c, dhph + 3 * nu * c, yfull + nf * c, dyfull + nf * nu * c,
                 gam + 3 * c, dgam + 3 * nu * c, pcv + 2 * c, dpcv + 2 * c, kr3 + 3 * c,
                 dkr3 + 6 * c, ktd + (nu + 1) * c, acc + nu * c, dacc + nu * nu * c,
                 src + nu * c, dsrc + nu * nu * c};
    ok[c] = (uint8_t)cell_eval(M, p[c], t[c], sw[c], sg[c], x + nco * c, y + ncg * c, cc[c],
                               phi_ref[c], &O);
  }
}

/* _kernels.py:797-825 */
void orc_compose_pass(int64_t nco, int64_t ncg, int64_t n, double *resid, double *diag,
                      const double *acc, const double *dacc, const double *src,
                      const double *dsrc, const double *accn, const double *vol, double dt,
                      const double *t_state, const double *hl_area, double hl_kob, double hl_d,
                      double hl_rho, double hl_tini) {
  const int64_t nu = nco + ncg + 5, row_e = 1 + nco + ncg, row_os = row_e + 1, row_gs = row_e + 2;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double vdt = vol[c] / dt;
    for (int64_t r = 0; r < nu; ++r) {
      int64_t i = c * nu + r;
      if (r == row_os || r == row_gs) {
        resid[i] = acc[i];
        for (int64_t u = 0; u < nu; ++u) diag[i * nu + u] = dacc[i * nu + u];
      } else {
        resid[i] = vdt * (acc[i] - accn[i]) - vol[c] * src[i];
        for (int64_t u = 0; u < nu; ++u)
          diag[i * nu + u] = vdt * dacc[i * nu + u] - vol[c] * dsrc[i * nu + u];
      }
    }
    if (hl_area[c] > 0.0) {
      resid[c * nu + row_e] += hl_area[c] * hl_kob * ((t_state[c] - hl_tini) / hl_d - hl_rho);
      diag[(c * nu + row_e) * nu + row_e] += hl_area[c] * hl_kob / hl_d;
    }
  }
}

/* _kernels.py:642-771 — one connection */
static void conn_eval(int nco, int ncg, double gd, double td, double za, double zb, double ta,
                      double tb, const double *potA, const double *dpotA, const double *betaA,
                      const double *dbetaA, const double *hphA, const double *dhphA,
                      const double *yfullA, const double *dyfullA, const double *xA,
                      const double *gamA, const double *dgamA, const double *ktA,
                      const double *potB, const double *dpotB, const double *betaB,
                      const double *dbetaB, const double *hphB, const double *dhphB,
                      const double *yfullB, const double *dyfullB, const double *xB,
                      const double *gamB, const double *dgamB, const double *ktB, int8_t *upw,
                      int freeze, double *flux, double *dfa, double *dfb) {
  const int nf = 1 + nco + ncg, nu = nco + ncg + 5, ct = 1 + nco + ncg, row_e = ct;
#define D2(a, r, u) a[(r) * nu + (u)]
  memset(flux, 0, sizeof(double) * nu);
  memset(dfa, 0, sizeof(double) * nu * nu);
  memset(dfb, 0, sizeof(double) * nu * nu);
  for (int al = 0; al < 3; ++al) {
    double phi_a = potA[al] - gamA[al] * za;
    double phi_b = potB[al] - gamB[al] * zb;
    double dphi = phi_a - phi_b;
    int up_a;
    if (freeze) up_a = upw[al] == 1;
    else { up_a = dphi >= 0.0; upw[al] = up_a ? 1 : 0; }
    double b_up = up_a ? betaA[al] : betaB[al];
    double conv = gd * dphi;
    int ncomp = al == 0 ? 1 : (al == 1 ? nco : nf);
    for (int m = 0; m < ncomp; ++m) {
      int row;
      double w_up;
      if (al == 0) { row = 0; w_up = 1.0; }
      else if (al == 1) { row = 1 + m; w_up = up_a ? xA[m] : xB[m]; }
      else { row = m; w_up = up_a ? yfullA[m] : yfullB[m]; }
      double val = b_up * w_up;
      double f = conv * val;
      flux[row] += f;
      if (val != 0.0) {
        for (int u = 0; u < nu; ++u) {
          D2(dfa, row, u) += gd * val * (D2(dpotA, al, u) - za * D2(dgamA, al, u));
          D2(dfb, row, u) -= gd * val * (D2(dpotB, al, u) - zb * D2(dgamB, al, u));
        }
      }
      if (up_a) {
        for (int u = 0; u < nu; ++u) {
          double dv = D2(dbetaA, al, u) * w_up;
          if (al == 1 && u == 1 + m) dv += betaA[al];
          else if (al == 2) dv += betaA[al] * D2(dyfullA, m, u);
          if (dv != 0.0) D2(dfa, row, u) += conv * dv;
        }
      } else {
        for (int u = 0; u < nu; ++u) {
          double dv = D2(dbetaB, al, u) * w_up;
          if (al == 1 && u == 1 + m) dv += betaB[al];
          else if (al == 2) dv += betaB[al] * D2(dyfullB, m, u);
          if (dv != 0.0) D2(dfb, row, u) += conv * dv;
        }
      }
    }
    double h_up = up_a ? hphA[al] : hphB[al];
    double val = b_up * h_up;
    flux[row_e] += conv * val;
    if (val != 0.0) {
      for (int u = 0; u < nu; ++u) {
        D2(dfa, row_e, u) += gd * val * (D2(dpotA, al, u) - za * D2(dgamA, al, u));
        D2(dfb, row_e, u) -= gd * val * (D2(dpotB, al, u) - zb * D2(dgamB, al, u));
      }
    }
    if (up_a) {
      for (int u = 0; u < nu; ++u) {
        double dv = D2(dbetaA, al, u) * h_up + betaA[al] * D2(dhphA, al, u);
        if (dv != 0.0) D2(dfa, row_e, u) += conv * dv;
      }
    } else {
      for (int u = 0; u < nu; ++u) {
        double dv = D2(dbetaB, al, u) * h_up + betaB[al] * D2(dhphB, al, u);
        if (dv != 0.0) D2(dfb, row_e, u) += conv * dv;
      }
    }
  }
  double hm, dh_a, dh_b;
  harmonic_pair(ktA[0], ktB[0], &hm, &dh_a, &dh_b);
  if (hm > 0.0 || dh_a != 0.0 || dh_b != 0.0) {
    double dt_ab = ta - tb;
    flux[row_e] += td * hm * dt_ab;
    D2(dfa, row_e, ct) += td * hm;
    D2(dfb, row_e, ct) -= td * hm;
    if (dt_ab != 0.0) {
      for (int u = 0; u < nu; ++u) {
        D2(dfa, row_e, u) += td * dt_ab * dh_a * ktA[1 + u];
        D2(dfb, row_e, u) += td * dt_ab * dh_b * ktB[1 + u];
      }
    }
  }
#undef D2
}

/* _kernels.py:774-794 */
void orc_conn_pass(int64_t nco, int64_t ncg, int64_t m, const int32_t *ca, const int32_t *cb,
                   const double *gd, const double *td, const double *depth, const double *t_state,
                   const double *x_state, const double *pot, const double *dpot,
                   const double *beta, const double *dbeta, const double *hph, const double *dhph,
                   const double *yfull, const double *dyfull, const double *gam,
                   const double *dgam, const double *ktd, int8_t *upw, int freeze, double *flux,
                   double *dfa, double *dfb) {
  const int64_t nf = 1 + nco + ncg, nu = nco + ncg + 5;
#pragma omp parallel for schedule(static) if (m > 256)
  for (int64_t ic = 0; ic < m; ++ic) {
    int64_t a = ca[ic], b = cb[ic];
    conn_eval((int)nco, (int)ncg, gd[ic], td[ic], depth[a], depth[b], t_state[a], t_state[b],
              pot + 3 * a, dpot + 3 * nu * a, beta + 3 * a, dbeta + 3 * nu * a, hph + 3 * a,
              dhph + 3 * nu * a, yfull + nf * a, dyfull + nf * nu * a, x_state + nco * a,
              gam + 3 * a, dgam + 3 * nu * a, ktd + (nu + 1) * a,
              pot + 3 * b, dpot + 3 * nu * b, beta + 3 * b, dbeta + 3 * nu * b, hph + 3 * b,
              dhph + 3 * nu * b, yfull + nf * b, dyfull + nf * nu * b, x_state + nco * b,
              gam + 3 * b, dgam + 3 * nu * b, ktd + (nu + 1) * b, upw + 3 * ic, freeze,
              flux + nu * ic, dfa + nu * nu * ic, dfb + nu * nu * ic);
  }
}

/* _kernels.py:828-854 */
void orc_gather_pass(int64_t n, int64_t nu, const int64_t *ptr, const int64_t *ids,
                     const int8_t *sides, const double *flux, const double *dfa,
                     const double *dfb, double *resid, double *diag, double *offd) {
  const int64_t b2 = nu * nu;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    for (int64_t k = ptr[c]; k < ptr[c + 1]; ++k) {
      int64_t ic = ids[k];
      if (sides[k] == 0) {
        for (int64_t r = 0; r < nu; ++r) {
          resid[c * nu + r] += flux[ic * nu + r];
          for (int64_t u = 0; u < nu; ++u) {
            diag[c * b2 + r * nu + u] += dfa[ic * b2 + r * nu + u];
            offd[(ic * 2 + 0) * b2 + r * nu + u] = dfb[ic * b2 + r * nu + u];
          }
        }
      } else {
        for (int64_t r = 0; r < nu; ++r) {
          resid[c * nu + r] -= flux[ic * nu + r];
          for (int64_t u = 0; u < nu; ++u) {
            diag[c * b2 + r * nu + u] -= dfb[ic * b2 + r * nu + u];
            offd[(ic * 2 + 1) * b2 + r * nu + u] = -dfa[ic * b2 + r * nu + u];
          }
        }
      }
    }
  }
}

/* ------------------------------------------------------------- linsolve.py */

/* linsolve.py:49-57 */
static void mm(int n, const double *a, const double *b, double *out) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += a[i * n + k] * b[k * n + j];
      out[i * n + j] = s;
    }
}
/* linsolve.py:60-67 */
static void mv(int n, const double *a, const double *v, double *out) {
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += a[i * n + k] * v[k];
    out[i] = s;
  }
}

/* linsolve.py:70-119 — a is destroyed; returns -1 or the failing column */
static int gj_inverse(int n, double *a, double *inv) {
  double amax = 0.0;
  for (int i = 0; i < n * n; ++i) { double v = fabs(a[i]); if (v > amax) amax = v; }
  if (amax == 0.0) return 0;
  double tol = 1e-13 * amax;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[i * n + j] = i == j ? 1.0 : 0.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    double pv = fabs(a[col * n + col]);
    for (int r = col + 1; r < n; ++r) {
      double v = fabs(a[r * n + col]);
      if (v > pv) { pv = v; piv = r; }
    }
    if (pv <= tol) return col;
    if (piv != col)
      for (int j = 0; j < n; ++j) {
        double tmp = a[col * n + j]; a[col * n + j] = a[piv * n + j]; a[piv * n + j] = tmp;
        tmp = inv[col * n + j]; inv[col * n + j] = inv[piv * n + j]; inv[piv * n + j] = tmp;
      }
    double d = 1.0 / a[col * n + col];
    for (int j = 0; j < n; ++j) { a[col * n + j] *= d; inv[col * n + j] *= d; }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      double f = a[r * n + col];
      if (f != 0.0)
        for (int j = 0; j < n; ++j) {
          a[r * n + j] -= f * a[col * n + j];
          inv[r * n + j] -= f * inv[col * n + j];
        }
    }
  }
  return -1;
}

/* linsolve.py:126-152 */
void orc_decouple_pass(int64_t n, int64_t nu, double *diag, double *rhs, double *offd,
                       const int64_t *ptr, const int64_t *ids, const int8_t *sides,
                       double *invs, int64_t *flags) {
  const int64_t b2 = nu * nu;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double work[MAXNU * MAXNU], tmp[MAXNU * MAXNU];
    double *inv = invs + c * b2;
    memcpy(work, diag + c * b2, sizeof(double) * b2);
    int bad = gj_inverse((int)nu, work, inv);
    if (bad >= 0) { flags[c] = bad + 1; continue; }
    mv((int)nu, inv, rhs + c * nu, tmp);
    memcpy(rhs + c * nu, tmp, sizeof(double) * nu);
    mm((int)nu, inv, diag + c * b2, tmp);
    memcpy(diag + c * b2, tmp, sizeof(double) * b2);
    for (int64_t k = ptr[c]; k < ptr[c + 1]; ++k) {
      double *blk = offd + (ids[k] * 2 + (sides[k] == 0 ? 0 : 1)) * b2;
      mm((int)nu, inv, blk, tmp);
      memcpy(blk, tmp, sizeof(double) * b2);
    }
  }
}

/* linsolve.py:159-177 */
void orc_matvec(int64_t n, int64_t nu, const double *diag, const double *offd,
                const int64_t *ptr, const int64_t *ids, const int8_t *sides,
                const int64_t *other, const double *v, double *out) {
  const int64_t b2 = nu * nu;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    for (int64_t r = 0; r < nu; ++r) {
      double s = 0.0;
      for (int64_t u = 0; u < nu; ++u) s += diag[c * b2 + r * nu + u] * v[c * nu + u];
      out[c * nu + r] = s;
    }
    for (int64_t k = ptr[c]; k < ptr[c + 1]; ++k) {
      const double *blk = offd + (ids[k] * 2 + (sides[k] == 0 ? 0 : 1)) * b2;
      const double *vo = v + other[k] * nu;
      for (int64_t r = 0; r < nu; ++r) {
        double s = 0.0;
        for (int64_t u = 0; u < nu; ++u) s += blk[r * nu + u] * vo[u];
        out[c * nu + r] += s;
      }
    }
  }
}

/* linsolve.py:193-199 (serial, fixed order) */
double orc_dot(int64_t len, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += a[i] * b[i];
  return s;
}

/* linsolve.py:206-232 */
int64_t orc_ilu_factor(int64_t nu, const double *diag, const double *offd, int64_t next,
                       const int64_t *cells, const int64_t *low_ptr, const int64_t *low_j,
                       const int64_t *low_ic, const int8_t *low_sd, double *uinv,
                       double *lblk) {
  const int64_t b2 = nu * nu;
  double ucc[MAXNU * MAXNU], work[MAXNU * MAXNU];
  for (int64_t lc = 0; lc < next; ++lc) {
    memcpy(ucc, diag + cells[lc] * b2, sizeof(double) * b2);
    for (int64_t k = low_ptr[lc]; k < low_ptr[lc + 1]; ++k) {
      int64_t lj = low_j[k], ic = low_ic[k];
      const double *a_cj = offd + (ic * 2 + (low_sd[k] == 0 ? 0 : 1)) * b2;
      const double *a_jc = offd + (ic * 2 + (low_sd[k] == 0 ? 1 : 0)) * b2;
      mm((int)nu, a_cj, uinv + lj * b2, lblk + k * b2);
      mm((int)nu, lblk + k * b2, a_jc, work);
      for (int64_t i = 0; i < b2; ++i) ucc[i] -= work[i];
    }
    if (gj_inverse((int)nu, ucc, uinv + lc * b2) >= 0) return lc;
  }
  return -1;
}

/* linsolve.py:235-259 */
void orc_ilu_apply(int64_t nu, const double *r, int64_t next, const int64_t *cells,
                   const int64_t *low_ptr, const int64_t *low_j, const double *lblk,
                   const int64_t *up_ptr, const int64_t *up_j, const int64_t *up_ic,
                   const int8_t *up_sd, const double *offd, const double *uinv, double *zloc) {
  const int64_t b2 = nu * nu;
  double tmp[MAXNU], cp[MAXNU];
  for (int64_t lc = 0; lc < next; ++lc) {
    int64_t g = cells[lc];
    for (int64_t u = 0; u < nu; ++u) zloc[lc * nu + u] = r[g * nu + u];
    for (int64_t k = low_ptr[lc]; k < low_ptr[lc + 1]; ++k) {
      mv((int)nu, lblk + k * b2, zloc + low_j[k] * nu, tmp);
      for (int64_t u = 0; u < nu; ++u) zloc[lc * nu + u] -= tmp[u];
    }
  }
  for (int64_t lc = next - 1; lc >= 0; --lc) {
    for (int64_t k = up_ptr[lc]; k < up_ptr[lc + 1]; ++k) {
      const double *blk = offd + (up_ic[k] * 2 + (up_sd[k] == 0 ? 0 : 1)) * b2;
      mv((int)nu, blk, zloc + up_j[k] * nu, tmp);
      for (int64_t u = 0; u < nu; ++u) zloc[lc * nu + u] -= tmp[u];
    }
    memcpy(cp, zloc + lc * nu, sizeof(double) * nu);
    mv((int)nu, uinv + lc * b2, cp, tmp);
    memcpy(zloc + lc * nu, tmp, sizeof(double) * nu);
  }
}

int orc_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
