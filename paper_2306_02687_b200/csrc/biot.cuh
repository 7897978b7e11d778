// Device finite-strain material point (BASELINE config 2, parity unpinned):
// 2-D polar decomposition F = R U, Biot strain U - I through the small-strain
// packed update (J2 radial return / elastic, materials.hpp:138-214), first
// Piola-Kirchhoff stress P = R T and its consistent tangent A = dP/dF.
// Same formulation as the CPU checker's update_biot; the device forms the
// three reciprocals it needs (1/ρ, 1/|s_tr|, 1/(3μ+h)) once and multiplies,
// and may contract a*b+c into FMA — ulp-level differences that the 1e-10
// parity tolerance covers.
// Components are ordered (F00, F01, F10, F11).
#pragma once

#include "device_common.cuh"
#include "material.cuh"

namespace fe2 {

struct BiotOut {
  double P[4];
  double A[16];  // A[r][s] = dP_r / dF_s (only with the tangent)
  double ep0, ep1, ep2, ep3, eq;
  bool plastic;
};

template <bool kTangent>
__device__ __forceinline__ void update_biot(const MatDev& m, double ep0, double ep1, double ep2, double ep3,
                                            double eq, double F0, double F1, double F2, double F3, BiotOut& o) {
  const double num = F2 - F1, den = F0 + F3;
  const double rho2 = num * num + den * den;
  const double inv_rho = dev::rsqrt_fast(rho2);
  const double c = den * inv_rho, s = num * inv_rho;
  const double U00 = c * F0 + s * F2, U01 = c * F1 + s * F3;
  const double U10 = -s * F0 + c * F2, U11 = -s * F1 + c * F3;
  // update4 on the Biot strain e = (U00 - 1, U11 - 1, 0, (U01 + U10) / 2)
  const double lam = m.lam, mu = m.mu, two_mu = 2.0 * mu;
  const double x0 = (U00 - 1.0) - ep0, x1 = (U11 - 1.0) - ep1, x2 = 0.0 - ep2, x3 = 0.5 * (U01 + U10) - ep3;
  const double lt = lam * (x0 + x1 + x2);
  const double t0 = lt + two_mu * x0, t1 = lt + two_mu * x1, t2 = lt + two_mu * x2, t3 = two_mu * x3;
  const double p = (t0 + t1 + t2) * (1.0 / 3.0);
  const double d0 = t0 - p, d1 = t1 - p, d2 = t2 - p, d3 = t3;
  const double ss = d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * d3 * d3;
  const double inv_ns = ss > 0.0 ? dev::rsqrt_fast(ss) : 0.0;
  const double q_tr = sqrt(1.5) * (ss * inv_ns);
  const double f = (m.kind == 1) ? q_tr - (m.sy0 + m.h * eq) : 0.0;
  const bool plastic = (m.kind == 1) && !(f <= 0.0);
  double T00 = t0, T11 = t1, T01 = t3;
  // tangent sub-block D[i][j], i, j in {0 (11), 1 (22), 3 (12)} of the packed 4x4
  double D00 = lam + two_mu, D01 = lam, D03 = 0.0, D10 = lam, D11 = lam + two_mu, D13 = 0.0;
  double D30 = 0.0, D31 = 0.0, D33 = two_mu;
  o.ep0 = ep0;
  o.ep1 = ep1;
  o.ep2 = ep2;
  o.ep3 = ep3;
  o.eq = eq;
  if (plastic) {
    const double dlam = f * m.inv_denom;                  // f / (3 mu + h)
    const double inv_q = 0.81649658092772603273 * inv_ns;  // 1 / q_tr = sqrt(2/3) / |s_tr|
    const double r0 = d0 * inv_q, r1 = d1 * inv_q, r2 = d2 * inv_q, r3 = d3 * inv_q;
    const double cs = 3.0 * mu * dlam;
    T00 = t0 - cs * r0;
    T11 = t1 - cs * r1;
    T01 = t3 - cs * r3;
    const double ce = 1.5 * dlam;
    o.ep0 = ep0 + ce * r0;
    o.ep1 = ep1 + ce * r1;
    o.ep2 = ep2 + ce * r2;
    o.ep3 = ep3 + ce * r3;
    o.eq = eq + dlam;
    if (kTangent) {
      const double n0 = d0 * inv_ns, n1 = d1 * inv_ns, n3 = d3 * inv_ns;
      const double c1 = 6.0 * mu * mu * dlam * inv_q;
      const double c2 = 6.0 * mu * mu * (m.inv_denom - dlam * inv_q);
      const double m3 = 2.0 * n3;
      D00 = (D00 - c1 * (2.0 / 3.0)) - c2 * (n0 * n0);
      D01 = (D01 - c1 * (-1.0 / 3.0)) - c2 * (n0 * n1);
      D03 = (D03 - c1 * 0.0) - c2 * (n0 * m3);
      D10 = (D10 - c1 * (-1.0 / 3.0)) - c2 * (n1 * n0);
      D11 = (D11 - c1 * (2.0 / 3.0)) - c2 * (n1 * n1);
      D13 = (D13 - c1 * 0.0) - c2 * (n1 * m3);
      D30 = (D30 - c1 * 0.0) - c2 * (n3 * n0);
      D31 = (D31 - c1 * 0.0) - c2 * (n3 * n1);
      D33 = (D33 - c1 * 1.0) - c2 * (n3 * m3);
    }
  }
  o.plastic = plastic;
  o.P[0] = c * T00 - s * T01;
  o.P[1] = c * T01 - s * T11;
  o.P[2] = s * T00 + c * T01;
  o.P[3] = s * T01 + c * T11;
  if (!kTangent) return;
  // dθ/dF and R J T, J = [[0,-1],[1,0]]
  const double inv_rho2 = inv_rho * inv_rho;
  const double g[4] = {-num * inv_rho2, -den * inv_rho2, den * inv_rho2, -num * inv_rho2};
  const double RJT00 = -s * T00 - c * T01, RJT01 = -s * T01 - c * T11;
  const double RJT10 = c * T00 - s * T01, RJT11 = c * T01 - s * T11;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double dth = g[k];
    const double dF0 = k == 0 ? 1.0 : 0.0, dF1 = k == 1 ? 1.0 : 0.0, dF2 = k == 2 ? 1.0 : 0.0,
                 dF3 = k == 3 ? 1.0 : 0.0;
    // dU = -J U dθ + R^T dF
    const double dU00 = U10 * dth + (c * dF0 + s * dF2);
    const double dU01 = U11 * dth + (c * dF1 + s * dF3);
    const double dU10 = -U00 * dth + (-s * dF0 + c * dF2);
    const double dU11 = -U01 * dth + (-s * dF1 + c * dF3);
    const double e0 = dU00, e1 = dU11, e3 = 0.5 * (dU01 + dU10);
    const double dT00 = D00 * e0 + D01 * e1 + D03 * e3;
    const double dT11 = D10 * e0 + D11 * e1 + D13 * e3;
    const double dT01 = D30 * e0 + D31 * e1 + D33 * e3;
    o.A[0 * 4 + k] = RJT00 * dth + (c * dT00 - s * dT01);
    o.A[1 * 4 + k] = RJT01 * dth + (c * dT01 - s * dT11);
    o.A[2 * 4 + k] = RJT10 * dth + (s * dT00 + c * dT01);
    o.A[3 * 4 + k] = RJT11 * dth + (s * dT01 + c * dT11);
  }
}

}  // namespace fe2
