// Device scalar property kernels: every correlation with its analytic
// partials, one-to-one with the reference's _props.py (cited per function).
// Integer powers are expanded the way numba lowers `x ** <int literal>`
// (square-and-multiply) so the CUDA results track the reference closely.
#pragma once
#include "common.cuh"

namespace isc {

__device__ __forceinline__ double ipow3(double t) { return t * (t * t); }
__device__ __forceinline__ double ipow4(double t) { double s = t * t; return s * s; }
__device__ __forceinline__ double ipow5(double t) { double s = t * t; return t * (s * s); }

// _props.py:24-41  K = (kv1/p + kv2 p + kv3) exp(kv4/(T - kv5))
__device__ __forceinline__ void k_value(const double* kv, double p, double t, double& k,
                                        double& dkdp, double& dkdt) {
  double pref = kv[0] / p + kv[1] * p + kv[2];
  double dpref = -kv[0] / (p * p) + kv[1];
  if (pref == 0.0 && dpref == 0.0) { k = 0.0; dkdp = 0.0; dkdt = 0.0; return; }
  double tdiff = t - kv[4];
  double e = exp(kv[3] / tdiff);
  k = pref * e;
  dkdp = dpref * e;
  dkdt = -k * kv[3] / (tdiff * tdiff);
}

// _props.py:44-50  S/(S+eps)
__device__ __forceinline__ void per_factor(double s, double eps, double& f, double& dfds) {
  double den = s + eps;
  f = s / den;
  dfds = eps / (den * den);
}

// _props.py:53-65
__device__ __forceinline__ void liquid_density(const double* lq, double p_ref, double t_ref,
                                               double p, double t, double& rho, double& drdp,
                                               double& drdt) {
  double dp = p - p_ref, dt = t - t_ref;
  double expo = lq[L_CP] * dp - lq[L_CT1] * dt - 0.5 * lq[L_CT2] * dt * dt + lq[L_CPT] * dp * dt;
  rho = lq[L_RHO] * exp(expo);
  drdp = rho * (lq[L_CP] + lq[L_CPT] * dt);
  drdt = rho * (-lq[L_CT1] - lq[L_CT2] * dt + lq[L_CPT] * dp);
}

// _props.py:68-104  largest real root of Z^3 - Z^2 + (A-B-B^2)Z - AB
__device__ __forceinline__ double cubic_largest_root(double a, double b) {
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
    arg = arg > 1.0 ? 1.0 : (arg < -1.0 ? -1.0 : arg);
    double theta = acos(arg) / 3.0;
    z = 2.0 * rp * cos(theta) + 1.0 / 3.0;
  }
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    double g = ((z - 1.0) * z + c1) * z + c0;
    double gp = (3.0 * z - 2.0) * z + c1;
    if (gp == 0.0) break;
    z -= g / gp;
  }
  return z;
}

// _props.py:107-150  RK Z factor of a mixture, partials in p, T and weights.
// w/tcr/pcr have NW entries; dzdw filled.
template <int NW>
__device__ __forceinline__ double z_factor_mix(const double* w, const double (*gasp)[9], double p,
                                               double t, double* dzdw, double& dzdp,
                                               double& dzdt) {
  double tr = t + RANKINE;
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    double ti = gasp[i][G_TCR];
    double bi = ti / gasp[i][G_PC];
    a += w[i] * ti * sqrt(bi);
    b += w[i] * bi;
  }
  if (a <= 0.0 || b <= 0.0) {
#pragma unroll
    for (int i = 0; i < NW; ++i) dzdw[i] = 0.0;
    dzdp = 0.0; dzdt = 0.0;
    return 1.0;
  }
  double coef_a = 0.427480 * p * pow(a, 1.5) * pow(b, 0.25) / pow(tr, 2.5);
  double coef_b = 0.086640 * p * b / tr;
  double z = cubic_largest_root(coef_a, coef_b);
  double gp = (3.0 * z - 2.0) * z + (coef_a - coef_b - coef_b * coef_b);
  if (fabs(gp) < 1e-30) gp = 1e-30;
  double dzda = -(z - coef_b) / gp;
  double dzdb = -((-1.0 - 2.0 * coef_b) * z - coef_a) / gp;
  dzdp = dzda * (coef_a / p) + dzdb * (coef_b / p);
  dzdt = dzda * (-2.5 * coef_a / tr) + dzdb * (-coef_b / tr);
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    double ti = gasp[i][G_TCR];
    double bi = ti / gasp[i][G_PC];
    double dai = ti * sqrt(bi);
    double da_dw = 1.5 * coef_a / a * dai + 0.25 * coef_a / b * bi;
    double db_dw = coef_b / b * bi;
    dzdw[i] = dzda * da_dw + dzdb * db_dw;
  }
  return z;
}

// _props.py:163-169
__device__ __forceinline__ void liquid_viscosity(double av, double bv, double t, double& mu,
                                                 double& dmu) {
  double tr = t + RANKINE;
  mu = av * exp(bv / tr);
  dmu = -mu * bv / (tr * tr);
}

// _props.py:172-178
__device__ __forceinline__ void gas_component_viscosity(double av, double bv, double t,
                                                        double& mu, double& dmu) {
  double tr = t + RANKINE;
  mu = av * pow(tr, bv);
  dmu = mu * bv / tr;
}

// _props.py:181-191
__device__ __forceinline__ void gas_enthalpy(const double* g, double t_ref, double t, double& h,
                                             double& dh) {
  h = g[G_CPG1] * (t - t_ref) + g[G_CPG2] / 2.0 * (t * t - t_ref * t_ref) +
      g[G_CPG3] / 3.0 * (ipow3(t) - ipow3(t_ref)) + g[G_CPG4] / 4.0 * (ipow4(t) - ipow4(t_ref));
  dh = g[G_CPG1] + g[G_CPG2] * t + g[G_CPG3] * t * t + g[G_CPG4] * ipow3(t);
}

// _props.py:194-205 (Heaviside(0) = 0)
__device__ __forceinline__ void vaporization_enthalpy(double hvr, double ev, double tcrit,
                                                      double t, double& h, double& dh) {
  if (t >= tcrit || hvr == 0.0) { h = 0.0; dh = 0.0; return; }
  double dt = tcrit - t;
  h = hvr * pow(dt, ev);
  dh = -ev * hvr * pow(dt, ev - 1.0);
}

// _props.py:216-228
__device__ __forceinline__ void porosity(double phi_ref, const double* rk, double p, double t,
                                         double& phi, double& dp_, double& dt_) {
  double dp = p - rk[RK_PREF], dt = t - rk[RK_TREF];
  double ctot = rk[RK_CPOR] * dp - rk[RK_CTPOR] * dt + rk[RK_CPTPOR] * dp * dt;
  double dc_dp = rk[RK_CPOR] + rk[RK_CPTPOR] * dt;
  double dc_dt = -rk[RK_CTPOR] + rk[RK_CPTPOR] * dp;
  if (rk[RK_MODE] != 0.0) {
    phi = phi_ref * exp(ctot);
    dp_ = phi * dc_dp;
    dt_ = phi * dc_dt;
  } else {
    phi = phi_ref * (1.0 + ctot);
    dp_ = phi_ref * dc_dp;
    dt_ = phi_ref * dc_dt;
  }
}

// _props.py:231-237
__device__ __forceinline__ void arrhenius(double freq, double ea, double t, double& k,
                                          double& dk) {
  double tr = t + RANKINE;
  k = freq * exp(-ea / (R_ARR * tr));
  dk = k * ea / (R_ARR * tr * tr);
}

// _props.py:245-268; o = r, dT, dpp, dfm, dcc
__device__ __forceinline__ void reaction_rate_one(int law, double a, double ea, double t,
                                                  double pp, double fm, double cc, double ccmax,
                                                  double* o) {
  double k, dk;
  arrhenius(a, ea, t, k, dk);
  if (law == 0) { o[0] = k * pp * fm; o[1] = dk * pp * fm; o[2] = k * fm; o[3] = k * pp; o[4] = 0.0; return; }
  if (law == 1) { o[0] = k * pp * cc; o[1] = dk * pp * cc; o[2] = k * cc; o[3] = 0.0; o[4] = k * pp; return; }
  double ratio = cc / ccmax;
  double lim = 1.0 - ipow5(ratio);
  if (lim <= 0.0) { o[0] = o[1] = o[2] = o[3] = o[4] = 0.0; return; }
  double dlim = -5.0 * ipow4(ratio) / ccmax;
  o[0] = k * fm * lim; o[1] = dk * fm * lim; o[2] = 0.0; o[3] = k * lim; o[4] = k * fm * dlim;
}

// _props.py:271-291; o = kro, d/dkrow, d/dkrw, d/dkrog, d/dkrg
__device__ __forceinline__ void stone2(double krocw, double krow, double krw, double krog,
                                       double krg, double* o) {
  o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
  if (krocw <= 0.0) return;
  double fo = krow / krocw + krw;
  double fg = krog / krocw + krg;
  double raw = krocw * (fo * fg - krw - krg);
  if (raw <= 0.0) return;
  if (raw >= 1.0) { o[0] = 1.0; return; }
  o[0] = raw; o[1] = fg; o[2] = krocw * (fg - 1.0); o[3] = fo; o[4] = krocw * (fo - 1.0);
}

// _props.py:294-315 piecewise-linear with end clamp
__device__ __forceinline__ void interp1(int n, const double* xs, const double* ys, double x,
                                        double& y, double& dy) {
  if (x <= xs[0]) { y = ys[0]; dy = 0.0; return; }
  if (x >= xs[n - 1]) { y = ys[n - 1]; dy = 0.0; return; }
  int lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (xs[mid] <= x) lo = mid; else hi = mid;
  }
  double slope = (ys[lo + 1] - ys[lo]) / (xs[lo + 1] - xs[lo]);
  y = ys[lo] + slope * (x - xs[lo]);
  dy = slope;
}

// _props.py:318-327
__device__ __forceinline__ void harmonic_pair(double a, double b, double& h, double& da,
                                              double& db) {
  double s = a + b;
  if (a <= 0.0 || b <= 0.0 || s <= 0.0) { h = 0.0; da = 0.0; db = 0.0; return; }
  h = 2.0 * a * b / s;
  da = 2.0 * b * b / (s * s);
  db = 2.0 * a * a / (s * s);
}

}  // namespace isc
