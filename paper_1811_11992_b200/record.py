"""Python mirror of csrc/record.cuh: expand the device per-cell record into
the reference's dense cell-pass arrays (pot/dpot/... of assembly.py:292-306).
Used by parity tests and diagnostics only."""

import numpy as np

NCO, NCG = 2, 2
NF, NU = 1 + NCO + NCG, NCO + NCG + 5
CT = 1 + NCO + NCG
CSW, CSG, CCC = CT + 1, CT + 2, CT + 3

R_POT, R_DPOT0_SW, R_DPOT2_SG, R_GAM = 0, 3, 4, 5
R_DGAM0_P, R_DGAM0_T, R_DGAM1_P, R_DGAM1_T, R_DGAM1_X = 8, 9, 10, 11, 12
R_DGAM2 = 12 + NCO
R_BETA = R_DGAM2 + NU
R_DBETA0 = R_BETA + 3                 # p, T, Sw
R_DBETA1 = R_DBETA0 + 3               # p, T, Sw, Sg, x..
R_DBETA2 = R_DBETA1 + 4 + NCO
R_HPH = R_DBETA2 + NU
R_DHPH0_T = R_HPH + 3
R_DHPH1 = R_DHPH0_T + 1               # T, x..
R_DHPH2 = R_DHPH1 + 1 + NCO
R_Y = R_DHPH2 + NU
R_DY0 = R_Y + NF                      # p, T, Sw
R_DYO = R_DY0 + 3                     # per oil p, T, x, s
R_KT = R_DYO + 4 * NCO
R_LAM = R_KT + 6
NREC = R_LAM + 3
assert NREC == 85


def expand(rec: np.ndarray) -> dict:
    """rec (85, n) -> dict of dense reference-layout arrays."""
    n = rec.shape[1]
    z = np.zeros
    pot, dpot = rec[R_POT:R_POT + 3].T.copy(), z((n, 3, NU))
    dpot[:, :, 0] = 1.0
    dpot[:, 0, CSW] = rec[R_DPOT0_SW]
    dpot[:, 2, CSG] = rec[R_DPOT2_SG]
    gam, dgam = rec[R_GAM:R_GAM + 3].T.copy(), z((n, 3, NU))
    dgam[:, 0, 0], dgam[:, 0, CT] = rec[R_DGAM0_P], rec[R_DGAM0_T]
    dgam[:, 1, 0], dgam[:, 1, CT] = rec[R_DGAM1_P], rec[R_DGAM1_T]
    for i in range(NCO):
        dgam[:, 1, 1 + i] = rec[R_DGAM1_X + i]
    dgam[:, 2, :] = rec[R_DGAM2:R_DGAM2 + NU].T
    beta, dbeta = rec[R_BETA:R_BETA + 3].T.copy(), z((n, 3, NU))
    dbeta[:, 0, 0], dbeta[:, 0, CT], dbeta[:, 0, CSW] = rec[R_DBETA0:R_DBETA0 + 3]
    dbeta[:, 1, 0], dbeta[:, 1, CT] = rec[R_DBETA1], rec[R_DBETA1 + 1]
    dbeta[:, 1, CSW], dbeta[:, 1, CSG] = rec[R_DBETA1 + 2], rec[R_DBETA1 + 3]
    for i in range(NCO):
        dbeta[:, 1, 1 + i] = rec[R_DBETA1 + 4 + i]
    dbeta[:, 2, :] = rec[R_DBETA2:R_DBETA2 + NU].T
    hph, dhph = rec[R_HPH:R_HPH + 3].T.copy(), z((n, 3, NU))
    dhph[:, 0, CT] = rec[R_DHPH0_T]
    dhph[:, 1, CT] = rec[R_DHPH1]
    for i in range(NCO):
        dhph[:, 1, 1 + i] = rec[R_DHPH1 + 1 + i]
    dhph[:, 2, :] = rec[R_DHPH2:R_DHPH2 + NU].T
    yfull, dyfull = rec[R_Y:R_Y + NF].T.copy(), z((n, NF, NU))
    dyfull[:, 0, 0], dyfull[:, 0, CT], dyfull[:, 0, CSW] = rec[R_DY0:R_DY0 + 3]
    for i in range(NCO):
        b = R_DYO + 4 * i
        dyfull[:, 1 + i, 0], dyfull[:, 1 + i, CT] = rec[b], rec[b + 1]
        dyfull[:, 1 + i, 1 + i] = rec[b + 2]
        dyfull[:, 1 + i, CSW] = rec[b + 3]
        dyfull[:, 1 + i, CSG] = rec[b + 3]
    for j in range(NCG):
        dyfull[:, 1 + NCO + j, 1 + NCO + j] = 1.0
    ktd = z((n, 1 + NU))
    ktd[:, 0] = rec[R_KT]
    ktd[:, 1 + 0], ktd[:, 1 + CT] = rec[R_KT + 1], rec[R_KT + 2]
    ktd[:, 1 + CSW], ktd[:, 1 + CSG], ktd[:, 1 + CCC] = rec[R_KT + 3], rec[R_KT + 4], rec[R_KT + 5]
    return dict(pot=pot, dpot=dpot, gam=gam, dgam=dgam, beta=beta, dbeta=dbeta, hph=hph,
                dhph=dhph, yfull=yfull, dyfull=dyfull, ktd=ktd)
