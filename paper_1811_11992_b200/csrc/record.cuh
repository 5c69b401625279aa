// Per-cell property record written by the cell kernel and read by the face
// kernel (SoA: field f of cell c lives at rec[f*n + c]).
//
// The reference keeps 180 dense values per cell for the connection pass
// (pot, dpot, beta, dbeta, hph, dhph, yfull, dyfull, gam, dgam, ktd;
// assembly.py:292-306). Most of those partials are structurally zero
// (_kernels.py:220-428): only the entries below are stored, 85
// doubles per cell, and the face kernel rebuilds dense 9-vectors in registers
// with literal zeros elsewhere.
#pragma once
#include "common.cuh"

namespace isc {

enum RecField : int {
  R_POT = 0,                 // pot[3]  (phase pressures; gravity applied per face)
  R_DPOT0_SW = 3,            // dpot[0][csw] = -dpcow
  R_DPOT2_SG = 4,            // dpot[2][csg] = dpcog    (dpot[a][p] == 1)
  R_GAM = 5,                 // gam[3]
  R_DGAM0_P = 8, R_DGAM0_T = 9,
  R_DGAM1_P = 10, R_DGAM1_T = 11, R_DGAM1_X = 12,          // + NCO
  R_DGAM2 = 12 + NCO,                                      // dense NU
  R_BETA = R_DGAM2 + NU,                                   // beta[3]
  R_DBETA0_P = R_BETA + 3, R_DBETA0_T, R_DBETA0_SW,
  R_DBETA1_P, R_DBETA1_T, R_DBETA1_SW, R_DBETA1_SG, R_DBETA1_X,  // + NCO
  R_DBETA2 = R_DBETA1_X + NCO,                             // dense NU
  R_HPH = R_DBETA2 + NU,                                   // hph[3]
  R_DHPH0_T = R_HPH + 3,
  R_DHPH1_T, R_DHPH1_X,                                    // + NCO
  R_DHPH2 = R_DHPH1_X + NCO,                               // dense NU
  R_Y = R_DHPH2 + NU,                                      // yfull[NF]
  R_DY0_P = R_Y + NF, R_DY0_T, R_DY0_SW,                   // water row of dyfull
  R_DYO = R_DY0_SW + 1,                                    // per oil: P, T, X, S (4 each)
  R_KT = R_DYO + 4 * NCO,                                  // ktd[0], d/dp, d/dT, d/dSw, d/dSg, d/dCc
  R_LAM = R_KT + 6, R_DLAM_SW, R_DLAM_SG,                  // total relperm (injector wells)
  NREC
};

static_assert(NREC == 85, "record layout");

}  // namespace isc
