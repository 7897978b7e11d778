// B200 (sm_100a) kernels of the hyper-ROM engine.
//
// Decomposition used on the device (exact algebra):
//   σ_q = C_e ε_q − S(εp_q) + Δσ_q ,  C_q = C_e + ΔC_q ,  ε_q = E + G_q α
// where Δσ_q, ΔC_q are the radial-return corrections (zero at elastic
// points). Summed with the cubature weights:
//   r    = K_e α + K_aE,e E − b_p + Σ_plastic w G_q^T Δσ_q
//   K_aa = K_e + Σ_plastic w G_q^T ΔC_q G_q
//   K_aE = K_aE,e + Σ_plastic w G_q^T ΔC_q ,   C_EE = C_EE,e + Σ_plastic w ΔC_q
//   Σraw = K_aE,e^T α + C_EE,e E − s_p + Σ_plastic w Δσ_q
// with K_e, K_aE,e, C_EE,e constant over the model (host, once) and
// b_p = Σ w G^T S(εp), s_p = Σ w S(εp) constant over an increment (kept
// per point, updated by the commit kernel from the plastic increments only).
//
//  K2+K3  k_newton_round — one warp per macro point; the J2 cubature rows G_q
//         stream through shared memory in 32-point chunks (TMA bulk copies,
//         mbarrier double buffering) shared by the CTA's points. Per chunk:
//         lane = cubature point: ε_q, elastic trial and yield test from the
//         HBM history (prefetched a chunk ahead); plastic points are
//         compacted (ballot/popc) and only they are contracted on the FP64
//         tensor cores (mma.sync m8n8k4 f64 = DMMA) over the flattened
//         (point, strain-row) index. The warp then runs the reduced Newton /
//         line-search state machine of micro_newton (rve.hpp:285-346):
//         Cholesky of K_aa in shared memory, step, Armijo test, and at
//         convergence the static condensation C = (C_EE − K_Ea K_aa^-1 K_aE)/V
//         (homogenize, rve.hpp:350-392). K_aa never touches HBM.
//  K1     k_commit — recomputes the update at the converged (E, α), writes the
//         history SoA stream (commit-after-acceptance, rve.hpp:283-284, :480)
//         and folds the plastic-strain increments into b_p, s_p.
#include <cstdio>

#include "hrom_kernels.cuh"

namespace fe2 {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// D(8x8) += A(8x4) B(4x8), fp64 tensor core. Fragments: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = D[lane/4][2*(lane%4) + {0,1}].
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
__device__ __forceinline__ int warp_sum_i(int v) {
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

// Cholesky of the lower triangle of sK (row stride ld) in place; lane i owns
// row i (n <= 32). Returns false if K is not positive definite.
__device__ bool warp_cholesky(double* sK, int ld, int n, int lane) {
  for (int j = 0; j < n; ++j) {
    __syncwarp();
    const double d = sK[j * ld + j];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    const double inv = 1.0 / ljj;
    __syncwarp();
    if (lane == j) sK[j * ld + j] = ljj;
    if (lane > j && lane < n) sK[lane * ld + j] *= inv;
    __syncwarp();
    if (lane > j && lane < n) {
      const double lij = sK[lane * ld + j];
      for (int k = j + 1; k <= lane; ++k) sK[lane * ld + k] -= lij * sK[k * ld + j];
    }
  }
  __syncwarp();
  return true;
}

// Solve L L^T x = b; lane i holds b_i in, x_i out (n <= 32).
__device__ double warp_chol_solve(const double* sK, int ld, int n, int lane, double b) {
  double x = b;
  for (int j = 0; j < n; ++j) {
    const double yj = __shfl_sync(0xffffffffu, x, j) / sK[j * ld + j];
    if (lane == j) x = yj;
    if (lane > j && lane < n) x -= sK[lane * ld + j] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {
    const double xj = __shfl_sync(0xffffffffu, x, j) / sK[j * ld + j];
    if (lane == j) x = xj;
    if (lane < j) x -= sK[j * ld + lane] * xj;
  }
  return x;
}

// Elastic trial state of update4 (materials.hpp:162-169) and the yield test
// (:208-210); the plastic branch returns the radial-return corrections
// Δσ = σ − σ_tr (condensed) and ΔC = C − C_e (6 unique).
struct Trial {
  double t0, t1, t2, t3;  // trial stress (packed 4)
  double d0, d1, d2, d3;  // trial deviator
  double ss, q_tr, f;
};

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
  const double p = (T.t0 + T.t1 + T.t2) / 3.0;
  T.d0 = T.t0 - p;
  T.d1 = T.t1 - p;
  T.d2 = T.t2 - p;
  T.d3 = T.t3;
  T.ss = T.d0 * T.d0 + T.d1 * T.d1 + T.d2 * T.d2 + 2.0 * T.d3 * T.d3;
  T.q_tr = sqrt(1.5) * sqrt(T.ss);
  T.f = T.q_tr - (m.sy0 + m.h * eq);
  return T;
}

struct Corr {
  double dc00, dc01, dc02, dc11, dc12, dc22;  // ΔC
  double ds0, ds1, ds2;                       // Δσ (11, 22, 12)
};

__device__ __forceinline__ Corr radial_return(const MatDev& m, const Trial& T) {
  Corr c;
  const double mu = m.mu;
  const double denom = 3.0 * mu + m.h;
  const double dlam = T.f / denom;
  const double inv_q = 1.0 / T.q_tr;
  const double cs = 3.0 * mu * dlam * inv_q;
  c.ds0 = -cs * T.d0;
  c.ds1 = -cs * T.d1;
  c.ds2 = -cs * T.d3;
  const double inv_n = 1.0 / sqrt(T.ss);
  const double n0 = T.d0 * inv_n, n1 = T.d1 * inv_n, n3 = T.d3 * inv_n;
  const double mu2 = 6.0 * mu * mu;
  const double c1 = mu2 * dlam * inv_q;
  const double c2 = mu2 * (1.0 / denom - dlam * inv_q);
  c.dc00 = -c1 * (2.0 / 3.0) - c2 * (n0 * n0);
  c.dc01 = c1 * (1.0 / 3.0) - c2 * (n0 * n1);
  c.dc02 = -c2 * (n0 * n3);
  c.dc11 = -c1 * (2.0 / 3.0) - c2 * (n1 * n1);
  c.dc12 = -c2 * (n1 * n3);
  c.dc22 = -0.5 * c1 - c2 * (n3 * n3);
  return c;
}

constexpr int kW = 8;  // warps (= macro points) per CTA in the round kernel

template <int NP>
struct RoundLayout {
  static constexpr int S = 3 * NP + 1;
  static constexpr int kSlots = kQC * 9 + kQC * 3 + kQC;  // ΔC rows, Δσ, point index (as doubles)
  static constexpr int kUnion = (kSlots > NP * (NP + 1)) ? kSlots : NP * (NP + 1);
  static constexpr int WS = NP /*alpha_ev*/ + NP /*r*/ + 3 * NP /*KaE*/ + kUnion;
  static constexpr size_t gbuf = static_cast<size_t>(kQC) * S;
  static constexpr size_t bytes = (2 * gbuf + static_cast<size_t>(kW) * WS) * sizeof(double) + 16;
};

// Commit one point's history at (E, α) from global G (one warp; used for the
// converged sub-steps of bisected increments), folding the plastic-strain
// increments into b_p, s_p.
template <int NP>
__device__ void warp_commit_point(const ModelDev& M, const PointsDev& D, int64_t p, const double* sAl, double E0,
                                  double E1, double E2, int lane) {
  constexpr int S = 3 * NP + 1;
  const int64_t PK = D.P * static_cast<int64_t>(M.K2p);
  double* H = D.hist + p * M.K2p;
  const MatDev& m = M.mat2;
  double bacc = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int q0 = 0; q0 < M.K2; q0 += 32) {
    const int q = q0 + lane;
    double w0 = 0.0, w1 = 0.0, w2v = 0.0;
    if (q < M.K2) {
      const double* Gq = M.G2 + static_cast<size_t>(q) * S;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
      for (int a = 0; a < NP; ++a) {
        const double al = sAl[a];
        e0 += Gq[a] * al;
        e1 += Gq[NP + a] * al;
        e2 += Gq[2 * NP + a] * al;
      }
      const MatOut o = update_material(m, H[q], H[PK + q], H[2 * PK + q], H[3 * PK + q], H[4 * PK + q],
                                       E0 + e0, E1 + e1, E2 + e2);
      const double x0 = o.ep0 - H[q], x1 = o.ep1 - H[PK + q], x2 = o.ep2 - H[2 * PK + q],
                   x3 = o.ep3 - H[3 * PK + q];
      const double lt = m.lam * (x0 + x1 + x2), wq = M.w2[q];
      w0 = wq * (lt + 2.0 * m.mu * x0);
      w1 = wq * (lt + 2.0 * m.mu * x1);
      w2v = wq * (2.0 * m.mu * x3);
      if (o.plastic) {
        H[q] = o.ep0;
        H[PK + q] = o.ep1;
        H[2 * PK + q] = o.ep2;
        H[3 * PK + q] = o.ep3;
        H[4 * PK + q] = o.eq;
      }
    }
    s0 += w0;
    s1 += w1;
    s2 += w2v;
    for (int l = 0; l < 32; ++l) {
      const double a0 = __shfl_sync(0xffffffffu, w0, l), a1 = __shfl_sync(0xffffffffu, w1, l),
                   a2 = __shfl_sync(0xffffffffu, w2v, l);
      const int ql = q0 + l;
      if (ql < M.K2 && lane < NP) {
        const double* Gq = M.G2 + static_cast<size_t>(ql) * S;
        bacc += Gq[lane] * a0 + Gq[NP + lane] * a1 + Gq[2 * NP + lane] * a2;
      }
    }
  }
  if (lane < NP) D.bp[p * NP + lane] += bacc;
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    D.sp[p * 4 + 0] += s0;
    D.sp[p * 4 + 1] += s1;
    D.sp[p * 4 + 2] += s2;
  }
}

template <int NT>
__global__ void __launch_bounds__(kW * 32, 2) k_newton_round(RoundArgs A) {
  constexpr int NP = 8 * NT;
  constexpr int NTP = NT * (NT + 1) / 2;
  using L = RoundLayout<NP>;
  constexpr int S = L::S;
  constexpr int LD = NP + 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* Gbuf0 = reinterpret_cast<double*>(smem_raw);
  double* Gbuf1 = Gbuf0 + L::gbuf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wbase = Gbuf1 + L::gbuf + static_cast<size_t>(warp) * L::WS;
  double* sA = wbase;        // α at the evaluation point
  double* sV = sA + NP;      // residual r
  double* sKaE = sV + NP;    // K_aE [NP][3]
  double* sU = sKaE + 3 * NP;
  double* sDC = sU;                                   // [32][9] w ΔC rows of the plastic slots
  double* sDS = sU + kQC * 9;                         // [32][3] w Δσ
  int* sQ = reinterpret_cast<int*>(sU + kQC * 12);    // [32]    chunk-local cubature index
  double* sK = sU;                                    // K_aa lower [NP][NP+1] (after the chunk loop)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Gbuf1 + L::gbuf + static_cast<size_t>(kW) * L::WS);

  const ModelDev& M = A.M;
  const PointsDev& D = A.D;
  const MatDev& mt = M.mat2;
  const int nch = M.nchunks;
  constexpr uint32_t kChunkBytes = kQC * S * sizeof(double);

  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2 && c < nch; ++c) {
      mbar_expect_tx(&mbar[c], kChunkBytes);
      tma_load_1d(c ? Gbuf1 : Gbuf0, M.G2 + static_cast<size_t>(c) * kQC * S, kChunkBytes, &mbar[c]);
    }
  }

  const int idx = blockIdx.x * kW + warp;
  const bool valid = idx < A.n_active;
  const int64_t p = valid ? A.active[idx] : 0;
  double E0 = 0.0, E1 = 0.0, E2 = 0.0;
  if (valid) {
    E0 = D.E_ev[p * 3 + 0];
    E1 = D.E_ev[p * 3 + 1];
    E2 = D.E_ev[p * 3 + 2];
    for (int a = lane; a < NP; a += 32) sA[a] = D.alpha_ev[p * NP + a];
  }
  __syncwarp();

  double acc[NTP][2];
  double kae[NT][3];
  double rr[NT];
#pragma unroll
  for (int t = 0; t < NTP; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    rr[t] = 0.0;
    kae[t][0] = kae[t][1] = kae[t][2] = 0.0;
  }
  // lane-partial plastic corrections of C_EE and Σraw
  double c00 = 0.0, c01 = 0.0, c02 = 0.0, c11 = 0.0, c12 = 0.0, c22 = 0.0, ds0 = 0.0, ds1 = 0.0, ds2 = 0.0;

  const int64_t PK = D.P * static_cast<int64_t>(M.K2p);
  const double* H0 = D.hist + p * M.K2p;
  double h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0;
  if (valid) {
    h0 = H0[lane];
    h1 = H0[PK + lane];
    h2 = H0[2 * PK + lane];
    h3 = H0[3 * PK + lane];
    h4 = H0[4 * PK + lane];
  }
  const int m = lane & 3, col = lane >> 2;
  int qo[3], io[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    qo[s] = (4 * s + m) / 3;
    io[s] = (4 * s + m) % 3;
  }

  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    const double* Gb = buf ? Gbuf1 : Gbuf0;
    mbar_wait(&mbar[buf], (c >> 1) & 1);
    if (valid) {
      const int q = c * kQC + lane;
      // ---- lane = cubature point: strain, elastic trial, yield test
      const double* Gq = Gb + lane * S;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll 8
      for (int a = 0; a < NP; ++a) {
        const double al = sA[a];
        e0 += Gq[a] * al;
        e1 += Gq[NP + a] * al;
        e2 += Gq[2 * NP + a] * al;
      }
      const Trial T = trial_state(mt, h0, h1, h2, h3, h4, E0 + e0, E1 + e1, E2 + e2);
      const bool plastic = (T.f > 0.0) && (q < M.K2);
      const unsigned bal = __ballot_sync(0xffffffffu, plastic);
      const int np = __popc(bal);
      if (plastic) {
        const Corr cr = radial_return(mt, T);
        const double wq = M.w2[q];
        const int slot = __popc(bal & ((1u << lane) - 1u));
        const double w00 = wq * cr.dc00, w01 = wq * cr.dc01, w02 = wq * cr.dc02;
        const double w11 = wq * cr.dc11, w12 = wq * cr.dc12, w22 = wq * cr.dc22;
        double* dc = sDC + slot * 9;
        dc[0] = w00;
        dc[1] = w01;
        dc[2] = w02;
        dc[3] = w01;
        dc[4] = w11;
        dc[5] = w12;
        dc[6] = w02;
        dc[7] = w12;
        dc[8] = w22;
        const double f0 = wq * cr.ds0, f1 = wq * cr.ds1, f2 = wq * cr.ds2;
        sDS[slot * 3 + 0] = f0;
        sDS[slot * 3 + 1] = f1;
        sDS[slot * 3 + 2] = f2;
        sQ[slot] = lane;
        c00 += w00;
        c01 += w01;
        c02 += w02;
        c11 += w11;
        c12 += w12;
        c22 += w22;
        ds0 += f0;
        ds1 += f1;
        ds2 += f2;
      }
      // zero the slots that round the plastic count up to a multiple of 4
      const int np4 = (np + 3) & ~3;
      if (lane >= np && lane < np4) {
#pragma unroll
        for (int e = 0; e < 9; ++e) sDC[lane * 9 + e] = 0.0;
        sDS[lane * 3 + 0] = sDS[lane * 3 + 1] = sDS[lane * 3 + 2] = 0.0;
        sQ[lane] = 0;
      }
      if (c + 1 < nch) {  // prefetch the next chunk's history
        const int qn = q + kQC;
        h0 = H0[qn];
        h1 = H0[PK + qn];
        h2 = H0[2 * PK + qn];
        h3 = H0[3 * PK + qn];
        h4 = H0[4 * PK + qn];
      }
      __syncwarp();
      // ---- plastic contraction on DMMA: k = 3 slot + i, four k per k-step
      const int ng = np4 >> 2;
#pragma unroll 1
      for (int g = 0; g < ng; ++g) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const int slot = 4 * g + qo[s];
          const int i = io[s];
          const double* wc = sDC + slot * 9 + i * 3;
          const double k0 = wc[0], k1 = wc[1], k2 = wc[2];
          const double ws = sDS[slot * 3 + i];
          const double* gp = Gb + sQ[slot] * S + col;
          double Af[NT], Bf[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double g0 = gp[t * 8], g1 = gp[NP + t * 8], g2 = gp[2 * NP + t * 8];
            Af[t] = (i == 0) ? g0 : ((i == 1) ? g1 : g2);
            Bf[t] = k0 * g0 + k1 * g1 + k2 * g2;
            kae[t][s] += Bf[t];
            rr[t] += ws * Af[t];
          }
          int ti = 0;
#pragma unroll
          for (int t1 = 0; t1 < NT; ++t1)
#pragma unroll
            for (int t2 = t1; t2 < NT; ++t2) {
              dmma(acc[ti][0], acc[ti][1], Af[t1], Bf[t2]);
              ++ti;
            }
        }
      }
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + 2 < nch) {
      fence_proxy_async();
      mbar_expect_tx(&mbar[buf], kChunkBytes);
      tma_load_1d(buf ? Gbuf1 : Gbuf0, M.G2 + static_cast<size_t>(c + 2) * kQC * S, kChunkBytes, &mbar[buf]);
    }
  }
  if (!valid) return;

  // ---- reductions: r and K_aE corrections over the four k-lanes of each column
  const int n = M.n;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    double v = rr[t];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    double ki[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int s = (i - (m % 3) + 3) % 3;  // slot s holds strain row (s + m) mod 3
      double x = (s == 0) ? kae[t][0] : ((s == 1) ? kae[t][1] : kae[t][2]);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      ki[i] = x;
    }
    if (m == 0) {
      const int a = t * 8 + col;
      sV[a] = v;
      sKaE[a * 3 + 0] = ki[0];
      sKaE[a * 3 + 1] = ki[1];
      sKaE[a * 3 + 2] = ki[2];
    }
  }
  __syncwarp();
  // K_aa corrections -> lower triangle of sK (slots are dead now)
  {
    const int r_ = lane >> 2, c_ = 2 * (lane & 3);
    int ti = 0;
#pragma unroll
    for (int t1 = 0; t1 < NT; ++t1)
#pragma unroll
      for (int t2 = t1; t2 < NT; ++t2) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = t1 * 8 + r_, cl = t2 * 8 + c_ + e;
          if (t1 < t2)
            sK[cl * LD + row] = acc[ti][e];
          else if (row >= cl)
            sK[row * LD + cl] = acc[ti][e];
        }
        ++ti;
      }
  }
  c00 = warp_sum(c00);
  c01 = warp_sum(c01);
  c02 = warp_sum(c02);
  c11 = warp_sum(c11);
  c12 = warp_sum(c12);
  c22 = warp_sum(c22);
  ds0 = warp_sum(ds0);
  ds1 = warp_sum(ds1);
  ds2 = warp_sum(ds2);
  __syncwarp();
  // ---- elastic predictor part (constant K_e, K_aE,e, C_EE,e) and b_p, s_p
  double sa0 = 0.0, sa1 = 0.0, sa2 = 0.0;
  if (lane < n) {
    const int a = lane;
    const double* ke = M.KaEe + a * 3;
    double s = 0.0;
    for (int b = 0; b < n; ++b) {
      const double kab = M.Ke[b * NP + a];  // K_e symmetric: coalesced column read
      s += kab * sA[b];
      if (b <= a) sK[a * LD + b] += kab;
    }
    s += ke[0] * E0 + ke[1] * E1 + ke[2] * E2;
    sV[a] += s - D.bp[p * NP + a];
    sKaE[a * 3 + 0] += ke[0];
    sKaE[a * 3 + 1] += ke[1];
    sKaE[a * 3 + 2] += ke[2];
    sa0 = ke[0] * sA[a];
    sa1 = ke[1] * sA[a];
    sa2 = ke[2] * sA[a];
  }
  sa0 = warp_sum(sa0);
  sa1 = warp_sum(sa1);
  sa2 = warp_sum(sa2);
  const double* ce = M.CEEe;
  const double* spp = D.sp + p * 4;
  const double s0 = ds0 + sa0 + (ce[0] * E0 + ce[1] * E1 + ce[2] * E2) - spp[0];
  const double s1 = ds1 + sa1 + (ce[3] * E0 + ce[4] * E1 + ce[5] * E2) - spp[1];
  const double s2 = ds2 + sa2 + (ce[6] * E0 + ce[7] * E1 + ce[8] * E2) - spp[2];
  const double ce00 = ce[0] + c00, ce01 = ce[1] + c01, ce02 = ce[2] + c02;
  const double ce11 = ce[4] + c11, ce12 = ce[5] + c12, ce22 = ce[8] + c22;
  __syncwarp();

  if (A.dbg) {  // assembly dump for parity tests (r, K full, KaE, C_EE, S_raw)
    double* o = A.dbg + static_cast<size_t>(idx) * (n + n * n + 3 * n + 12);
    for (int a = lane; a < n; a += 32) o[a] = sV[a];
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      o[n + e] = (j <= i) ? sK[i * LD + j] : sK[j * LD + i];
    }
    for (int e = lane; e < 3 * n; e += 32) o[n + n * n + e] = sKaE[e];
    if (lane == 0) {
      double* cc = o + n + n * n + 3 * n;
      cc[0] = ce00;
      cc[1] = ce01;
      cc[2] = ce02;
      cc[3] = ce01;
      cc[4] = ce11;
      cc[5] = ce12;
      cc[6] = ce02;
      cc[7] = ce12;
      cc[8] = ce22;
      cc[9] = s0;
      cc[10] = s1;
      cc[11] = s2;
    }
    return;
  }

  // ---- reduced Newton state machine (micro_newton, rve.hpp:300-342)
  const double rl = (lane < n) ? sV[lane] : 0.0;
  const double rn = sqrt(warp_sum(rl * rl));
  const double srn = sqrt(s0 * s0 + s1 * s1 + s2 * s2);
  PointState st = D.st[p];
  double* al = D.alpha + p * NP;
  double* aev = D.alpha_ev + p * NP;
  double* dal = D.dalpha + p * NP;
  const NewtonCfg& cfg = A.cfg;
  auto fail = [&](int code) {
    st.err = code;
    st.phase = kFailed;
    st.rn_last = rn;
    if (lane == 0) {
      A.O.status[p] = code;
      A.O.iters[p] = st.iters;
      A.O.res[p] = rn;
      for (int i = 0; i < 3; ++i) A.O.sigma[p * 3 + i] = qnan();
      for (int i = 0; i < 9; ++i) A.O.C[p * 9 + i] = qnan();
    }
  };
  constexpr int kSolver = 1 + 4;  // 1 + ErrorCode::solver
  for (int pass = 0; pass < 2; ++pass) {
    if (st.mode == kNewton) {
      if (st.it == 0) st.ref = fmax(fmax(rn, srn), 1e-30);
      if (rn <= cfg.tol * st.ref) {
        st.iters += st.it;
        st.rn_last = rn;
        const double target = fmin(1.0, st.done + st.frac);
        if (target >= 1.0 - 1e-12) {
          if (!warp_cholesky(sK, LD, n, lane)) {
            fail(kSolver);
            break;
          }
          // condensation: X = L^-1 K_aE, C = (C_EE - X^T X) / V
          double x0 = (lane < n) ? sKaE[lane * 3 + 0] : 0.0;
          double x1 = (lane < n) ? sKaE[lane * 3 + 1] : 0.0;
          double x2 = (lane < n) ? sKaE[lane * 3 + 2] : 0.0;
          for (int j = 0; j < n; ++j) {
            const double ljj = sK[j * LD + j];
            const double y0 = __shfl_sync(0xffffffffu, x0, j) / ljj;
            const double y1 = __shfl_sync(0xffffffffu, x1, j) / ljj;
            const double y2 = __shfl_sync(0xffffffffu, x2, j) / ljj;
            if (lane == j) {
              x0 = y0;
              x1 = y1;
              x2 = y2;
            } else if (lane > j && lane < n) {
              const double l = sK[lane * LD + j];
              x0 -= l * y0;
              x1 -= l * y1;
              x2 -= l * y2;
            }
          }
          const double q00 = warp_sum(x0 * x0), q01 = warp_sum(x0 * x1), q02 = warp_sum(x0 * x2);
          const double q11 = warp_sum(x1 * x1), q12 = warp_sum(x1 * x2), q22 = warp_sum(x2 * x2);
          if (lane == 0) {
            const double V = M.volume;
            double* Cp = A.O.C + p * 9;
            Cp[0] = (ce00 - q00) / V;
            Cp[1] = (ce01 - q01) / V;
            Cp[2] = (ce02 - q02) / V;
            Cp[3] = (ce01 - q01) / V;
            Cp[4] = (ce11 - q11) / V;
            Cp[5] = (ce12 - q12) / V;
            Cp[6] = (ce02 - q02) / V;
            Cp[7] = (ce12 - q12) / V;
            Cp[8] = (ce22 - q22) / V;
            A.O.sigma[p * 3 + 0] = s0 / V;
            A.O.sigma[p * 3 + 1] = s1 / V;
            A.O.sigma[p * 3 + 2] = s2 / V;
            A.O.res[p] = rn;
            A.O.iters[p] = st.iters;
            A.O.status[p] = 0;
          }
          st.phase = kDone;
        } else {
          // converged sub-step of a bisected increment: commit, then the next one
          warp_commit_point<NP>(M, D, p, sA, E0, E1, E2, lane);
          for (int a = lane; a < NP; a += 32) D.alpha_c[p * NP + a] = sA[a];
          st.done = target;
          const double nt = fmin(1.0, st.done + st.frac);
          if (lane == 0)
            for (int i = 0; i < 3; ++i) D.E_ev[p * 3 + i] = lerp_rn(D.E_prev[p * 3 + i], D.E_tgt[p * 3 + i], nt);
          st.it = 0;
          st.mode = kNewton;
        }
        break;
      }
      if (st.it == cfg.max_iter) {
        st.iters += cfg.max_iter;
        st.rn_last = rn;
        if (++st.bis > cfg.max_bis) {
          fail(kSolver);
          break;
        }
        st.frac *= 0.5;
        const double nt = fmin(1.0, st.done + st.frac);
        if (lane == 0)
          for (int i = 0; i < 3; ++i) D.E_ev[p * 3 + i] = lerp_rn(D.E_prev[p * 3 + i], D.E_tgt[p * 3 + i], nt);
        for (int a = lane; a < NP; a += 32) {
          const double ac = D.alpha_c[p * NP + a];
          al[a] = ac;
          aev[a] = ac;
        }
        st.it = 0;
        st.mode = kNewton;
        break;
      }
      // Newton step: K Δα = -r
      if (!warp_cholesky(sK, LD, n, lane)) {
        fail(kSolver);
        break;
      }
      const double du = warp_chol_solve(sK, LD, n, lane, -rl);
      if (lane < NP) {
        dal[lane] = (lane < n) ? du : 0.0;
        aev[lane] = (lane < n) ? axpy_rn(al[lane], 1.0, du) : 0.0;
      }
      st.rn_it = rn;
      st.a = 1.0;
      st.ls = 0;
      st.best_rn = __longlong_as_double(0x7ff0000000000000ll);
      st.best_a = 1.0;
      st.mode = kLineSearch;
      break;
    } else {
      // backtracking line search on the residual norm (rve.hpp:327-341)
      const double trial = rn;
      if (trial < st.best_rn) {
        st.best_rn = trial;
        st.best_a = st.a;
      }
      const bool armijo = trial <= (1.0 - 1e-4 * st.a) * st.rn_it;
      if (armijo || st.ls == 7) {
        st.it += 1;
        if (st.best_a == st.a) {  // the accepted iterate is this evaluation point
          if (lane < NP) al[lane] = sA[lane];
          st.mode = kNewton;
          continue;  // reuse this assembly as the new iterate's
        }
        if (lane < NP) {
          const double nv = (lane < n) ? axpy_rn(al[lane], st.best_a, dal[lane]) : 0.0;
          al[lane] = nv;
          aev[lane] = nv;
        }
        st.mode = kNewton;
        break;
      }
      st.ls += 1;
      st.a *= 0.5;
      if (lane < NP) aev[lane] = (lane < n) ? axpy_rn(al[lane], st.a, dal[lane]) : 0.0;
      break;
    }
  }
  __syncwarp();
  if (lane == 0) {
    D.st[p] = st;
    if (st.phase == kActive) A.next_active[atomicAdd(A.n_next, 1)] = static_cast<int>(p);
  }
}

// ---------------------------------------------------------------------------
// K1: history commit at the converged (E, α) of every finished point, plus
// the b_p, s_p update from the plastic-strain increments. HBM stream: read
// εp(4), eq; write εp(4), eq — 80 B per J2 cubature point (σ33 is write-only
// in the reference, materials.hpp:181/:193, and is recomputed on readback).
// G chunks arrive by TMA bulk copies (double buffered); each warp owns kCPPW
// points and prefetches their next-chunk history while it computes.
constexpr int kCW = 8;    // warps per commit CTA
constexpr int kCPPW = 2;  // points per warp

template <int NP>
struct CommitLayout {
  static constexpr int S = 3 * NP + 1;
  static constexpr size_t gbuf = static_cast<size_t>(kQC) * S;
  static constexpr size_t bytes = (2 * gbuf + static_cast<size_t>(kCW) * (kCPPW * NP + kQC * 3)) * sizeof(double) + 16;
};

template <int NP>
__global__ void __launch_bounds__(kCW * 32, 2) k_commit(ModelDev M, PointsDev D, Outputs O) {
  using L = CommitLayout<NP>;
  constexpr int S = L::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* Gbuf0 = reinterpret_cast<double*>(smem_raw);
  double* Gbuf1 = Gbuf0 + L::gbuf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sAl = Gbuf1 + L::gbuf + static_cast<size_t>(warp) * (kCPPW * NP + kQC * 3);  // [kCPPW][NP]
  double* sWw = sAl + kCPPW * NP;                                                        // [32][3]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Gbuf1 + L::gbuf + static_cast<size_t>(kCW) * (kCPPW * NP + kQC * 3));
  const int nch = M.nchunks;
  constexpr uint32_t kChunkBytes = kQC * S * sizeof(double);
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2 && c < nch; ++c) {
      mbar_expect_tx(&mbar[c], kChunkBytes);
      tma_load_1d(c ? Gbuf1 : Gbuf0, M.G2 + static_cast<size_t>(c) * kQC * S, kChunkBytes, &mbar[c]);
    }
  }
  const int64_t p_base = (static_cast<int64_t>(blockIdx.x) * kCW + warp) * kCPPW;
  const int64_t PK = D.P * static_cast<int64_t>(M.K2p);
  const MatDev& mt = M.mat2;
  bool live[kCPPW];
  double Ep[kCPPW][3], hv[kCPPW][5], bacc[kCPPW], sacc[kCPPW][3];
  int pc[kCPPW];
#pragma unroll
  for (int k = 0; k < kCPPW; ++k) {
    const int64_t p = p_base + k;
    live[k] = p < D.P && D.st[p].phase == kDone;
    pc[k] = 0;
    bacc[k] = 0.0;
    sacc[k][0] = sacc[k][1] = sacc[k][2] = 0.0;
    Ep[k][0] = Ep[k][1] = Ep[k][2] = 0.0;
    hv[k][0] = hv[k][1] = hv[k][2] = hv[k][3] = hv[k][4] = 0.0;
    if (live[k]) {
      Ep[k][0] = D.E_ev[p * 3 + 0];
      Ep[k][1] = D.E_ev[p * 3 + 1];
      Ep[k][2] = D.E_ev[p * 3 + 2];
      for (int a = lane; a < NP; a += 32) sAl[k * NP + a] = D.alpha_ev[p * NP + a];
      const double* H = D.hist + p * M.K2p + lane;
      hv[k][0] = H[0];
      hv[k][1] = H[PK];
      hv[k][2] = H[2 * PK];
      hv[k][3] = H[3 * PK];
      hv[k][4] = H[4 * PK];
    }
  }
  __syncwarp();
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    const double* Gb = buf ? Gbuf1 : Gbuf0;
    mbar_wait(&mbar[buf], (c >> 1) & 1);
    const int q = c * kQC + lane;
    const bool real = q < M.K2;
    const double wq = M.w2[q];
    const double* Gq = Gb + lane * S;
#pragma unroll
    for (int k = 0; k < kCPPW; ++k) {
      if (!live[k]) continue;
      const int64_t p = p_base + k;
      const double* a = sAl + k * NP;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll 8
      for (int j = 0; j < NP; ++j) {
        const double al = a[j];
        e0 += Gq[j] * al;
        e1 += Gq[NP + j] * al;
        e2 += Gq[2 * NP + j] * al;
      }
      const MatOut o = update_material(mt, hv[k][0], hv[k][1], hv[k][2], hv[k][3], hv[k][4], Ep[k][0] + e0,
                                       Ep[k][1] + e1, Ep[k][2] + e2);
      const bool pl = real && o.plastic;
      double w0 = 0.0, w1 = 0.0, w2 = 0.0;  // w S(Δεp): change of the plastic-strain load
      if (pl) {
        const double x0 = o.ep0 - hv[k][0], x1 = o.ep1 - hv[k][1], x2 = o.ep2 - hv[k][2], x3 = o.ep3 - hv[k][3];
        const double lt = mt.lam * (x0 + x1 + x2);
        w0 = wq * (lt + 2.0 * mt.mu * x0);
        w1 = wq * (lt + 2.0 * mt.mu * x1);
        w2 = wq * (2.0 * mt.mu * x3);
      }
      double* H = D.hist + p * M.K2p + q;
      if (c + 1 < nch) {  // prefetch this point's next chunk
        hv[k][0] = H[kQC];
        hv[k][1] = H[PK + kQC];
        hv[k][2] = H[2 * PK + kQC];
        hv[k][3] = H[3 * PK + kQC];
        hv[k][4] = H[4 * PK + kQC];
      }
      if (pl) {  // elastic points keep their history bit for bit
        H[0] = o.ep0;
        H[PK] = o.ep1;
        H[2 * PK] = o.ep2;
        H[3 * PK] = o.ep3;
        H[4 * PK] = o.eq;
      }
      if (D.flags && real) D.flags[p * M.K2p + q] = o.plastic ? 1 : 0;
      sacc[k][0] += w0;
      sacc[k][1] += w1;
      sacc[k][2] += w2;
      const unsigned bal = __ballot_sync(0xffffffffu, pl);
      pc[k] += __popc(bal);
      if (bal) {  // b_p[a] += Σ_plastic q  G_q[:, a] . w S(Δεp_q)   (lane = mode a)
        sWw[lane * 3 + 0] = w0;
        sWw[lane * 3 + 1] = w1;
        sWw[lane * 3 + 2] = w2;
        __syncwarp();
        if (lane < NP) {
          unsigned bits = bal;
          double b = 0.0;
          while (bits) {
            const int l = __ffs(bits) - 1;
            bits &= bits - 1;
            const double* gl = Gb + l * S + lane;
            b += gl[0] * sWw[l * 3 + 0] + gl[NP] * sWw[l * 3 + 1] + gl[2 * NP] * sWw[l * 3 + 2];
          }
          bacc[k] += b;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + 2 < nch) {
      fence_proxy_async();
      mbar_expect_tx(&mbar[buf], kChunkBytes);
      tma_load_1d(buf ? Gbuf1 : Gbuf0, M.G2 + static_cast<size_t>(c + 2) * kQC * S, kChunkBytes, &mbar[buf]);
    }
  }
#pragma unroll
  for (int k = 0; k < kCPPW; ++k) {
    const int64_t p = p_base + k;
    if (!live[k]) continue;
    if (lane == 0 && O.pcount) O.pcount[p] = pc[k];
    for (int a = lane; a < NP; a += 32) D.alpha_c[p * NP + a] = D.alpha_ev[p * NP + a];
    if (lane < NP) D.bp[p * NP + lane] += bacc[k];
    const double t0 = warp_sum(sacc[k][0]), t1 = warp_sum(sacc[k][1]), t2 = warp_sum(sacc[k][2]);
    if (lane == 0) {
      D.sp[p * 4 + 0] += t0;
      D.sp[p * 4 + 1] += t1;
      D.sp[p * 4 + 2] += t2;
    }
  }
}

// Start of an increment: path point, sub-step bookkeeping, warm start
// α = α_committed (run_trajectory, rve.hpp:459-472), active list.
template <int NP>
__global__ void k_begin_increment(PointsDev D, Outputs O, const double* dE, int* active, int* n_active) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= D.P) return;
  PointState st = D.st[p];
  for (int i = 0; i < 3; ++i) {
    D.E_prev[p * 3 + i] = D.E_tgt[p * 3 + i];
    D.E_tgt[p * 3 + i] = dE[p * 3 + i];
  }
  if (O.pcount) O.pcount[p] = 0;
  if (st.phase == kFailed) {  // a point whose trajectory already failed stays failed
    O.status[p] = st.err;
    O.iters[p] = 0;
    O.res[p] = qnan();
    for (int i = 0; i < 3; ++i) O.sigma[p * 3 + i] = qnan();
    for (int i = 0; i < 9; ++i) O.C[p * 9 + i] = qnan();
    return;
  }
  for (int i = 0; i < 3; ++i) D.E_ev[p * 3 + i] = lerp_rn(D.E_prev[p * 3 + i], D.E_tgt[p * 3 + i], 1.0);
  for (int a = 0; a < NP; ++a) {
    const double ac = D.alpha_c[p * NP + a];
    D.alpha[p * NP + a] = ac;
    D.alpha_ev[p * NP + a] = ac;
  }
  st.done = 0.0;
  st.frac = 1.0;
  st.bis = 0;
  st.iters = 0;
  st.it = 0;
  st.ls = 0;
  st.mode = kNewton;
  st.phase = kActive;
  st.err = 0;
  D.st[p] = st;
  active[atomicAdd(n_active, 1)] = static_cast<int>(p);
}

__global__ void k_material_batch(MatDev m, int64_t N, const double* eps, const double* st_in, double* sigma,
                                 double* C, double* st_out, uint8_t* plastic) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double s[5] = {0, 0, 0, 0, 0};
  if (st_in)
    for (int c = 0; c < 5; ++c) s[c] = st_in[i * 6 + c];
  const MatOut o = update_material(m, s[0], s[1], s[2], s[3], s[4], eps[i * 3], eps[i * 3 + 1], eps[i * 3 + 2]);
  sigma[i * 3 + 0] = o.s0;
  sigma[i * 3 + 1] = o.s1;
  sigma[i * 3 + 2] = o.s2;
  double* c9 = C + i * 9;
  c9[0] = o.c00;
  c9[1] = o.c01;
  c9[2] = o.c02;
  c9[3] = o.c01;
  c9[4] = o.c11;
  c9[5] = o.c12;
  c9[6] = o.c02;
  c9[7] = o.c12;
  c9[8] = o.c22;
  if (st_out) {
    double* so = st_out + i * 6;
    so[0] = o.ep0;
    so[1] = o.ep1;
    so[2] = o.ep2;
    so[3] = o.ep3;
    so[4] = o.eq;
    so[5] = o.s33;
  }
  if (plastic) plastic[i] = o.plastic ? 1 : 0;
}

template <int NT>
void launch_round_nt(const RoundArgs& a, cudaStream_t s) {
  constexpr int NP = 8 * NT;
  const size_t smem = RoundLayout<NP>::bytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_newton_round<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  const int grid = (a.n_active + kW - 1) / kW;
  k_newton_round<NT><<<grid, kW * 32, smem, s>>>(a);
}

template <int NP>
void launch_commit_np(const ModelDev& M, const PointsDev& D, const Outputs& O, cudaStream_t s) {
  const size_t smem = CommitLayout<NP>::bytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_commit<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  const int64_t per_cta = kCW * kCPPW;
  const int64_t grid = (D.P + per_cta - 1) / per_cta;
  k_commit<NP><<<static_cast<unsigned>(grid), kCW * 32, smem, s>>>(M, D, O);
}

}  // namespace

size_t newton_round_smem(int NP) {
  switch (NP) {
    case 8: return RoundLayout<8>::bytes;
    case 16: return RoundLayout<16>::bytes;
    case 24: return RoundLayout<24>::bytes;
    case 32: return RoundLayout<32>::bytes;
    default: return 0;
  }
}

void launch_newton_round(const RoundArgs& a, cudaStream_t s) {
  switch (a.M.NP) {
    case 8: launch_round_nt<1>(a, s); break;
    case 16: launch_round_nt<2>(a, s); break;
    case 24: launch_round_nt<3>(a, s); break;
    case 32: launch_round_nt<4>(a, s); break;
    default: break;
  }
}

void launch_commit(const ModelDev& M, const PointsDev& D, const Outputs& O, cudaStream_t s) {
  switch (M.NP) {
    case 8: launch_commit_np<8>(M, D, O, s); break;
    case 16: launch_commit_np<16>(M, D, O, s); break;
    case 24: launch_commit_np<24>(M, D, O, s); break;
    case 32: launch_commit_np<32>(M, D, O, s); break;
    default: break;
  }
}

void launch_begin_increment(const ModelDev& M, const PointsDev& D, const Outputs& O, const double* dE,
                            int* active, int* n_active, cudaStream_t s) {
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((D.P + threads - 1) / threads);
  switch (M.NP) {
    case 8: k_begin_increment<8><<<grid, threads, 0, s>>>(D, O, dE, active, n_active); break;
    case 16: k_begin_increment<16><<<grid, threads, 0, s>>>(D, O, dE, active, n_active); break;
    case 24: k_begin_increment<24><<<grid, threads, 0, s>>>(D, O, dE, active, n_active); break;
    case 32: k_begin_increment<32><<<grid, threads, 0, s>>>(D, O, dE, active, n_active); break;
    default: break;
  }
}

void launch_material_batch(const MatDev& m, int64_t N, const double* eps, const double* st_in, double* sigma,
                           double* C, double* st_out, uint8_t* plastic, cudaStream_t s) {
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((N + threads - 1) / threads);
  k_material_batch<<<grid, threads, 0, s>>>(m, N, eps, st_in, sigma, C, st_out, plastic);
}

}  // namespace fe2
