// Device material point: plane-strain J2 with linear isotropic hardening and
// isotropic elasticity, on packed 4-tensors (11, 22, 33, 12-tensor) and the
// engineering-Voigt facade. Arithmetic follows the reference
// (/root/reference/proj/include/fe2rom/materials.hpp):
//   trial_state :162-169, update4(J2) :205-214, finish_return :173-185,
//   radial_return_tangent4 :138-154, elastic_result :187-195,
//   condense_tangent :305-314, update_material :317-325.
#pragma once

#include <cuda_runtime.h>

namespace fe2 {

struct MatDev {
  int kind;  // 0 elastic, 1 J2 linear, 2 power law, 3 strain-hardening creep
  double lam, mu, sy0, h;
  double inv_denom;  // 1 / (3 mu + h)
  double E;          // Young's modulus (power law / creep)
  double N;          // power law: sy(e) = sy0 (1 + E e / sy0)^N          (materials.hpp:51-65)
  double A, cn, cm;  // creep: deq/dt = (q/A)^(n/(m+1)) ((m+1) eq)^(m/(m+1)) (:67-76)
  double dt;         // creep: time of one load increment (PathStep::dt)
};

// Outputs of one update: condensed stress (3), symmetric condensed tangent
// as 6 unique entries (C00, C01, C02, C11, C12, C22), new history.
struct MatOut {
  double s0, s1, s2;
  double c00, c01, c02, c11, c12, c22;
  double ep0, ep1, ep2, ep3, eq, s33;
  bool plastic;
};

__host__ __device__ inline MatDev make_mat(int kind, double E, double nu, double sy0, double h) {
  MatDev m;
  m.kind = kind;
  m.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  m.mu = 0.5 * E / (1.0 + nu);
  m.sy0 = sy0;
  m.h = h;
  m.inv_denom = 1.0 / (3.0 * m.mu + h);
  m.E = E;
  m.N = 0.0;
  m.A = m.cn = m.cm = 0.0;
  m.dt = 1.0;
  return m;
}

// power law (kind 2): p = {sy0, N}; creep (kind 3): p = {A, n, m, dt}
__host__ __device__ inline MatDev make_mat_general(int kind, double E, double nu, const double* p) {
  MatDev m = make_mat(kind, E, nu, kind == 2 ? p[0] : 0.0, 0.0);
  if (kind == 2) m.N = p[1];
  if (kind == 3) {
    m.A = p[0];
    m.cn = p[1];
    m.cm = p[2];
    m.dt = p[3];
  }
  return m;
}

// update_material(mat, {ep, eq}, eps3) — eps3 engineering Voigt.
__device__ __forceinline__ MatOut update_material(const MatDev& m, double ep0, double ep1, double ep2,
                                                  double ep3, double eq, double e11, double e22, double g12) {
  const double lam = m.lam, mu = m.mu;
  const double two_mu = 2.0 * mu;
  // elastic strain (strain4_from_voigt: e33 = 0, e12 = g12 / 2)
  const double x0 = e11 - ep0, x1 = e22 - ep1, x2 = 0.0 - ep2, x3 = 0.5 * g12 - ep3;
  const double lt = lam * (x0 + x1 + x2);
  const double t0 = lt + two_mu * x0, t1 = lt + two_mu * x1, t2 = lt + two_mu * x2, t3 = two_mu * x3;
  const double p = (t0 + t1 + t2) / 3.0;
  const double d0 = t0 - p, d1 = t1 - p, d2 = t2 - p, d3 = t3;
  const double ss = d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * d3 * d3;
  const double ns = sqrt(ss);
  const double q_tr = sqrt(1.5) * ns;
  MatOut o;
  const double f = (m.kind == 1) ? q_tr - (m.sy0 + m.h * eq) : 0.0;
  if (m.kind != 1 || f <= 0.0) {
    o.s0 = t0;
    o.s1 = t1;
    o.s2 = t3;
    o.c00 = lam + two_mu;
    o.c01 = lam;
    o.c02 = 0.0;
    o.c11 = lam + two_mu;
    o.c12 = 0.0;
    o.c22 = mu;  // 0.5 * (2 mu)
    o.ep0 = ep0;
    o.ep1 = ep1;
    o.ep2 = ep2;
    o.ep3 = ep3;
    o.eq = eq;
    o.s33 = t2;
    o.plastic = false;
    return o;
  }
  const double denom = 3.0 * mu + m.h;
  const double dlam = f / denom;
  const double inv_q = 1.0 / q_tr;
  const double r0 = d0 * inv_q, r1 = d1 * inv_q, r2 = d2 * inv_q, r3 = d3 * inv_q;  // s_tr / q_tr
  const double cs = 3.0 * mu * dlam;
  o.s0 = t0 - cs * r0;
  o.s1 = t1 - cs * r1;
  o.s2 = t3 - cs * r3;
  const double ce = 1.5 * dlam;
  o.ep0 = ep0 + ce * r0;
  o.ep1 = ep1 + ce * r1;
  o.ep2 = ep2 + ce * r2;
  o.ep3 = ep3 + ce * r3;
  o.eq = eq + dlam;
  o.s33 = t2 - cs * r2;
  const double inv_n = 1.0 / ns;
  const double n0 = d0 * inv_n, n1 = d1 * inv_n, n3 = d3 * inv_n;
  const double mu2 = 6.0 * mu * mu;
  const double c1 = mu2 * dlam * inv_q;
  const double c2 = mu2 * (1.0 / denom - dlam * inv_q);
  o.c00 = (lam + two_mu - c1 * (2.0 / 3.0)) - c2 * (n0 * n0);
  o.c01 = (lam + c1 * (1.0 / 3.0)) - c2 * (n0 * n1);
  o.c02 = -c2 * (n0 * n3);
  o.c11 = (lam + two_mu - c1 * (2.0 / 3.0)) - c2 * (n1 * n1);
  o.c12 = -c2 * (n1 * n3);
  o.c22 = 0.5 * ((two_mu - c1) - c2 * (n3 * (2.0 * n3)));
  o.plastic = true;
  return o;
}

// Power-law and creep return maps (materials.hpp:216-292): the same
// safeguarded scalar Newton iterations as the reference, then finish_return
// (:173-185) with dlam and d(dlam)/d(q_tr). ok = false when the iteration
// does not converge (the reference's ErrorCode::material).
__device__ inline MatOut update_material_general(const MatDev& m, double ep0, double ep1, double ep2, double ep3,
                                                 double eq, double e11, double e22, double g12, bool& ok) {
  const double lam = m.lam, mu = m.mu;
  const double two_mu = 2.0 * mu;
  const double x0 = e11 - ep0, x1 = e22 - ep1, x2 = 0.0 - ep2, x3 = 0.5 * g12 - ep3;
  const double lt = lam * (x0 + x1 + x2);
  const double t0 = lt + two_mu * x0, t1 = lt + two_mu * x1, t2 = lt + two_mu * x2, t3 = two_mu * x3;
  const double p = (t0 + t1 + t2) / 3.0;
  const double d0 = t0 - p, d1 = t1 - p, d2 = t2 - p, d3 = t3;
  const double ns = sqrt(d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * d3 * d3);
  const double q_tr = sqrt(1.5) * ns;
  ok = true;
  bool plastic = false;
  double dlam = 0.0, kq = 0.0;
  if (m.kind == 2) {
    auto sy = [&](double e) { return m.sy0 * pow(1.0 + m.E * e / m.sy0, m.N); };
    auto sy_slope = [&](double e) { return m.E * m.N * pow(1.0 + m.E * e / m.sy0, m.N - 1.0); };
    const double f_tr = q_tr - sy(eq);
    if (!(f_tr <= 0.0)) {
      double lo = 0.0, hi = f_tr / (3.0 * mu), x = hi * 0.5;
      const double tol = 1e-12 * fmax(m.sy0, q_tr);
      bool conv = false;
      for (int it = 0; it < 50; ++it) {
        const double gx = q_tr - 3.0 * mu * x - sy(eq + x);
        if (fabs(gx) <= tol) {
          conv = true;
          break;
        }
        if (gx > 0.0) lo = x;
        else hi = x;
        double next = x + gx / (3.0 * mu + sy_slope(eq + x));
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        x = next;
      }
      ok = conv;
      plastic = true;
      dlam = x;
      kq = 1.0 / (3.0 * mu + sy_slope(eq + x));
    }
  } else if (m.kind == 3) {
    if (!(m.dt > 0.0)) {
      ok = false;
    } else if (q_tr > 1e-14 * m.E) {
      const double p1 = m.cn / (m.cm + 1.0), p2 = m.cm / (m.cm + 1.0), eq_floor = 1e-12;
      auto hard = [&](double e) { return pow((m.cm + 1.0) * fmax(e, eq_floor), p2); };
      auto hard_slope = [&](double e) {
        return e <= eq_floor ? 0.0 : p2 * (m.cm + 1.0) * pow((m.cm + 1.0) * e, p2 - 1.0);
      };
      auto rate_q = [&](double q) { return pow(q / m.A, p1); };
      auto rate_q_slope = [&](double q) { return p1 / m.A * pow(q / m.A, p1 - 1.0); };
      double lo = 0.0, hi = q_tr / (3.0 * mu);
      if (hi - m.dt * rate_q(q_tr - 3.0 * mu * hi) * hard(eq + hi) < 0.0) ok = false;  // bracket failure
      double x = 0.5 * hi, Rp = 1.0;
      const double tol = 1e-14 * fmax(1.0, hi);
      bool conv = false;
      for (int it = 0; ok && it < 200; ++it) {
        const double q = q_tr - 3.0 * mu * x;
        const double e = eq + x;
        const double Rx = x - m.dt * rate_q(q) * hard(e);
        Rp = 1.0 + 3.0 * mu * m.dt * rate_q_slope(q) * hard(e) - m.dt * rate_q(q) * hard_slope(e);
        if (fabs(Rx) <= tol) {
          conv = true;
          break;
        }
        if (Rx < 0.0) lo = x;
        else hi = x;
        double next = (Rp > 0.0) ? x - Rx / Rp : 0.5 * (lo + hi);
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        x = next;
      }
      ok = ok && conv;
      if (ok && x > 0.0) {
        plastic = true;
        dlam = x;
        kq = m.dt * rate_q_slope(q_tr - 3.0 * mu * x) * hard(eq + x) / Rp;
      }
    }
  }
  MatOut o;
  if (!plastic) {
    o.s0 = t0;
    o.s1 = t1;
    o.s2 = t3;
    o.c00 = lam + two_mu;
    o.c01 = lam;
    o.c02 = 0.0;
    o.c11 = lam + two_mu;
    o.c12 = 0.0;
    o.c22 = mu;
    o.ep0 = ep0;
    o.ep1 = ep1;
    o.ep2 = ep2;
    o.ep3 = ep3;
    o.eq = eq;
    o.s33 = t2;
    o.plastic = false;
    return o;
  }
  const double r0 = d0 / q_tr, r1 = d1 / q_tr, r2 = d2 / q_tr, r3 = d3 / q_tr;
  const double cs = 3.0 * mu * dlam;
  o.s0 = t0 - cs * r0;
  o.s1 = t1 - cs * r1;
  o.s2 = t3 - cs * r3;
  const double ce = 1.5 * dlam;
  o.ep0 = ep0 + ce * r0;
  o.ep1 = ep1 + ce * r1;
  o.ep2 = ep2 + ce * r2;
  o.ep3 = ep3 + ce * r3;
  o.eq = eq + dlam;
  o.s33 = t2 - cs * r2;
  const double n0 = d0 / ns, n1 = d1 / ns, n3 = d3 / ns;
  const double mu2 = 6.0 * mu * mu;
  const double c1 = mu2 * dlam / q_tr;
  const double c2 = mu2 * (kq - dlam / q_tr);
  o.c00 = (lam + two_mu - c1 * (2.0 / 3.0)) - c2 * (n0 * n0);
  o.c01 = (lam + c1 * (1.0 / 3.0)) - c2 * (n0 * n1);
  o.c02 = -c2 * (n0 * n3);
  o.c11 = (lam + two_mu - c1 * (2.0 / 3.0)) - c2 * (n1 * n1);
  o.c12 = -c2 * (n1 * n3);
  o.c22 = 0.5 * ((two_mu - c1) - c2 * (n3 * (2.0 * n3)));
  o.plastic = true;
  return o;
}

// Any material kind: the closed-form path for elastic / J2, the iterative
// return maps otherwise.
__device__ __forceinline__ MatOut update_material_any(const MatDev& m, double ep0, double ep1, double ep2,
                                                      double ep3, double eq, double e11, double e22, double g12,
                                                      bool& ok) {
  ok = true;
  if (m.kind <= 1) return update_material(m, ep0, ep1, ep2, ep3, eq, e11, e22, g12);
  return update_material_general(m, ep0, ep1, ep2, ep3, eq, e11, e22, g12, ok);
}

}  // namespace fe2
