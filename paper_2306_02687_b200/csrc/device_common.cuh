// Device helpers shared by the hyper-ROM kernels: TMA bulk copies and
// mbarriers, the FP64 tensor-core MMA, warp reductions, reference-rounded
// updates, fast reciprocals, and the J2 elastic trial / radial-return
// corrections (materials.hpp:138-214).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "material.cuh"

namespace fe2 {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok)
               : "r"(smem_u32(bar)), "r"(parity)
               : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// D(8x8) += A(8x4) B(4x8) on the FP64 tensor cores (SASS DMMA.8x8x4).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2*(lane%4)+{0,1}].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x + a*y rounded as the reference's `u_free + alpha * du` (no contraction).
__device__ __forceinline__ double axpy_rn(double x, double a, double y) { return __dadd_rn(x, __dmul_rn(a, y)); }
// E_prev + (E_tgt - E_prev) * target, as run_trajectory (rve.hpp:465).
__device__ __forceinline__ double lerp_rn(double e0, double e1, double t) {
  return __dadd_rn(e0, __dmul_rn(__dsub_rn(e1, e0), t));
}
__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}

__device__ __forceinline__ int tri(int i) { return i * (i + 1) / 2; }  // packed lower row offset

struct Trial {
  double t0, t1, t2, t3;  // trial stress (packed 4)
  double d0, d1, d2, d3;  // trial deviator
  double ss, inv_ns, q_tr, f;  // |s_tr|^2, 1/|s_tr|, sqrt(3/2)|s_tr|, yield function
};

// trial_state (materials.hpp:162-169) and f = q_tr - (sy0 + h eq) (:208)
__device__ __forceinline__ Trial trial_state(const MatDev& m, double ep0, double ep1, double ep2, double ep3,
                                             double eq, double e11, double e22, double g12) {
  Trial T;
  const double two_mu = 2.0 * m.mu;
  const double x0 = e11 - ep0, x1 = e22 - ep1, x2 = 0.0 - ep2, x3 = 0.5 * g12 - ep3;
  const double lt = m.lam * (x0 + x1 + x2);
  T.t0 = lt + two_mu * x0;
  T.t1 = lt + two_mu * x1;
  T.t2 = lt + two_mu * x2;
  T.t3 = two_mu * x3;
  const double p = (T.t0 + T.t1 + T.t2) * (1.0 / 3.0);
  T.d0 = T.t0 - p;
  T.d1 = T.t1 - p;
  T.d2 = T.t2 - p;
  T.d3 = T.t3;
  T.ss = T.d0 * T.d0 + T.d1 * T.d1 + T.d2 * T.d2 + 2.0 * T.d3 * T.d3;
  // |s_tr| and its reciprocal from one MUFU rsqrt seed (no IEEE sqrt sequence)
  T.inv_ns = T.ss > 0.0 ? rsqrt_fast(T.ss) : 0.0;
  T.q_tr = 1.2247448713915890491 * (T.ss * T.inv_ns);  // sqrt(3/2) |s_tr|
  T.f = T.q_tr - (m.sy0 + m.h * eq);
  return T;
}

struct Corr {
  double dc00, dc01, dc02, dc11, dc12, dc22;  // ΔC = C - C_e (condensed)
  double ds0, ds1, ds2;                       // Δσ = σ - σ_tr (11, 22, 12)
};

// finish_return + radial_return_tangent4 (materials.hpp:138-154, :173-185) as corrections
__device__ __forceinline__ Corr radial_return(const MatDev& m, const Trial& T) {
  Corr c;
  const double mu = m.mu;
  const double dlam = T.f * m.inv_denom;
  const double inv_q = 0.81649658092772603273 * T.inv_ns;  // 1/q_tr = sqrt(2/3) / |s_tr|
  const double cs = 3.0 * mu * dlam * inv_q;
  c.ds0 = -cs * T.d0;
  c.ds1 = -cs * T.d1;
  c.ds2 = -cs * T.d3;
  const double inv_n = T.inv_ns;
  const double n0 = T.d0 * inv_n, n1 = T.d1 * inv_n, n3 = T.d3 * inv_n;
  const double mu2 = 6.0 * mu * mu;
  const double c1 = mu2 * dlam * inv_q;
  const double c2 = mu2 * (m.inv_denom - dlam * inv_q);
  c.dc00 = -c1 * (2.0 / 3.0) - c2 * (n0 * n0);
  c.dc01 = c1 * (1.0 / 3.0) - c2 * (n0 * n1);
  c.dc02 = -c2 * (n0 * n3);
  c.dc11 = -c1 * (2.0 / 3.0) - c2 * (n1 * n1);
  c.dc12 = -c2 * (n1 * n3);
  c.dc22 = -0.5 * c1 - c2 * (n3 * n3);
  return c;
}

// The scalar return of an iterative material (the history-carrying points of
// a power-law or creep model) on the trial state T: the reference's
// safeguarded Newton iterations, power law materials.hpp:216-244 (plastic iff
// f_tr > 0), strain-hardening creep :246-292 (inelastic iff the solve gives
// dlam > 0; dt = the sub-step's time, PathStep::dt x its fraction,
// rve.hpp:466). q_tr is formed as the reference does, sqrt(3/2) sqrt(|s_tr|²).
// Out: dlam, kq = d(dlam)/d(q_tr); ok = false when the iteration does not
// converge, the creep bracket fails or dt <= 0 (ErrorCode::material).
struct GenRet {
  double dlam, kq;
  bool plastic, ok;
};
// inlined into the GEN kernels (a call frame spilled 0.3-0.9 KB per thread around the call;
// inlined: +4-6% at n = 64, equal at n = 24)
static __device__ __forceinline__ GenRet general_return(const MatDev& m, double ss, double eq, double dt) {
  GenRet g{0.0, 0.0, false, true};
  const double mu = m.mu;
  const double q_tr = 1.2247448713915890491 * sqrt(ss);
  if (m.kind == 2) {
    // sy(e) = sy0 b^N with b = 1 + E e / sy0, and sy'(e) = E N b^(N-1) = sy(e) N E / (sy0 b):
    // one pow per iteration for both (the reference evaluates two)
    auto sy = [&](double e) { return m.sy0 * pow(1.0 + m.E * e / m.sy0, m.N); };
    auto slope_of = [&](double e, double s) { return s * (m.N * m.E) / (m.sy0 + m.E * e); };
    const double f_tr = q_tr - sy(eq);
    if (f_tr <= 0.0) return g;
    double lo = 0.0, hi = f_tr / (3.0 * mu), x = hi * 0.5;
    const double tol = 1e-12 * fmax(m.sy0, q_tr);
    bool conv = false;
    for (int it = 0; it < 50; ++it) {
      const double s = sy(eq + x);
      const double gx = q_tr - 3.0 * mu * x - s;
      if (fabs(gx) <= tol) {
        conv = true;
        break;
      }
      if (gx > 0.0) lo = x;
      else hi = x;
      double next = x + gx / (3.0 * mu + slope_of(eq + x, s));
      if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
      x = next;
    }
    g.ok = conv;
    g.plastic = true;
    g.dlam = x;
    g.kq = 1.0 / (3.0 * mu + slope_of(eq + x, sy(eq + x)));
    return g;
  }
  // creep (kind 3)
  if (!(dt > 0.0)) {
    g.ok = false;
    return g;
  }
  if (!(q_tr > 1e-14 * m.E)) return g;
  const double p1 = m.cn / (m.cm + 1.0), p2 = m.cm / (m.cm + 1.0), eq_floor = 1e-12;
  auto hard = [&](double e) { return pow((m.cm + 1.0) * fmax(e, eq_floor), p2); };
  auto rate_q = [&](double q) { return pow(q / m.A, p1); };
  double lo = 0.0, hi = q_tr / (3.0 * mu);
  if (hi - dt * rate_q(q_tr - 3.0 * mu * hi) * hard(eq + hi) < 0.0) {  // bracket failure
    g.ok = false;
    return g;
  }
  double x = 0.5 * hi, Rp = 1.0;
  const double tol = 1e-14 * fmax(1.0, hi);
  bool conv = false;
  for (int it = 0; it < 200; ++it) {
    const double q = q_tr - 3.0 * mu * x;
    const double e = eq + x;
    // F = (q/A)^p1 ((m+1) e)^p2 once per iteration: the slopes are F p1 / q and F p2 / e
    // ((q/A)^(p1-1) p1 / A and p2 (m+1) ((m+1) e)^(p2-1) of the reference, :262-265)
    const double rq = rate_q(q), hd = hard(e), F = rq * hd;
    const double Rx = x - dt * F;
    Rp = 1.0 + 3.0 * mu * dt * (F * p1 / q) - (e <= eq_floor ? 0.0 : dt * (F * p2 / e));
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
  g.ok = conv;
  if (conv && x > 0.0) {
    g.plastic = true;
    g.dlam = x;
    const double q = q_tr - 3.0 * mu * x;
    g.kq = dt * (p1 / m.A * pow(q / m.A, p1 - 1.0)) * hard(eq + x) / Rp;
  }
  return g;
}

// radial_return with a given multiplier and sensitivity (iterative materials)
__device__ __forceinline__ Corr radial_return_gen(const MatDev& m, const Trial& T, double dlam, double kq) {
  Corr c;
  const double mu = m.mu;
  const double inv_q = 0.81649658092772603273 * T.inv_ns;
  const double cs = 3.0 * mu * dlam * inv_q;
  c.ds0 = -cs * T.d0;
  c.ds1 = -cs * T.d1;
  c.ds2 = -cs * T.d3;
  const double inv_n = T.inv_ns;
  const double n0 = T.d0 * inv_n, n1 = T.d1 * inv_n, n3 = T.d3 * inv_n;
  const double mu2 = 6.0 * mu * mu;
  const double c1 = mu2 * dlam * inv_q;
  const double c2 = mu2 * (kq - dlam * inv_q);
  c.dc00 = -c1 * (2.0 / 3.0) - c2 * (n0 * n0);
  c.dc01 = c1 * (1.0 / 3.0) - c2 * (n0 * n1);
  c.dc02 = -c2 * (n0 * n3);
  c.dc11 = -c1 * (2.0 / 3.0) - c2 * (n1 * n1);
  c.dc12 = -c2 * (n1 * n3);
  c.dc22 = -0.5 * c1 - c2 * (n3 * n3);
  return c;
}

}  // namespace dev
}  // namespace fe2
