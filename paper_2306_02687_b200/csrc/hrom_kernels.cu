// B200 (sm_100a) kernels of the hyper-ROM engine.
//
//  K2+K3  k_newton_round  — one warp per macro point. The J2 cubature rows
//         G_q (3 x NP) stream through shared memory in 32-point chunks by
//         TMA bulk copies (cp.async.bulk + mbarrier, double buffered) and are
//         shared by the W points of the CTA. Per chunk each lane runs the
//         constitutive update of one cubature point (HBM history stream,
//         prefetched one chunk ahead), then the warp contracts
//           K_aa += Σ_q G_q^T (w C_q) G_q        on FP64 tensor cores
//                                                 (mma.sync m8n8k4 f64 = DMMA)
//           K_aE += Σ_q G_q^T (w C_q),  r += Σ_q G_q^T (w σ_q)   (DFMA)
//         over the flattened (q, strain-row) index in k-steps of 4. The
//         elastic-inclusion cubature points are linear, so their part is a
//         precomputed constant (K_inc, K_aE_inc, C_EE_inc) added once. The
//         same warp then runs the reduced Newton / line-search state machine
//         of micro_newton (rve.hpp:285-346): Cholesky of K_aa in shared memory
//         with warp shuffles, the step, the Armijo test, and at convergence
//         the static condensation C = (C_EE - K_Ea K_aa^-1 K_aE)/V
//         (homogenize, rve.hpp:350-392) — K_aa never touches HBM.
//  K1     k_commit        — recomputes the constitutive update at the
//         converged (E, α) and writes the history (commit-after-acceptance,
//         rve.hpp:283-284, :480): a coalesced SoA stream, HBM bound.
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

// Cholesky of the lower triangle of sK (row stride ld) in place; lane i owns
// row i (n <= 32). Returns false if K is not positive definite.
__device__ bool warp_cholesky(double* sK, int ld, int n, int lane) {
  for (int j = 0; j < n; ++j) {
    __syncwarp();
    const double d = sK[j * ld + j];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    __syncwarp();
    if (lane == j) sK[j * ld + j] = ljj;
    if (lane > j && lane < n) sK[lane * ld + j] = sK[lane * ld + j] / ljj;
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

constexpr int kW = 8;  // warps (= macro points) per CTA in the round kernel

template <int NP>
struct RoundLayout {
  static constexpr int S = 3 * NP + 1;
  static constexpr int kUnion = (kQC * 12 > NP * (NP + 1)) ? kQC * 12 : NP * (NP + 1);
  static constexpr int WS = NP /*alpha_ev*/ + NP /*r*/ + 3 * NP /*KaE*/ + kUnion;
  static constexpr size_t gbuf = static_cast<size_t>(kQC) * S;
  static constexpr size_t bytes = (2 * gbuf + static_cast<size_t>(kW) * WS) * sizeof(double) + 16;
};

// Recompute the constitutive update at (E, α) for all J2 cubature points of
// point p and write its history (one warp). Used for bisected sub-steps.
template <int NP>
__device__ void warp_commit_point(const ModelDev& M, const PointsDev& D, int64_t p, const double* sAl, double E0,
                                  double E1, double E2, int lane) {
  constexpr int S = 3 * NP + 1;
  const int64_t PK = D.P * static_cast<int64_t>(M.K2p);
  double* H = D.hist + p * M.K2p;
  for (int q = lane; q < M.K2; q += 32) {
    const double* Gq = M.G2 + static_cast<size_t>(q) * S;
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    for (int a = 0; a < NP; ++a) {
      const double al = sAl[a];
      e0 += Gq[a] * al;
      e1 += Gq[NP + a] * al;
      e2 += Gq[2 * NP + a] * al;
    }
    const MatOut o = update_material(M.mat2, H[q], H[PK + q], H[2 * PK + q], H[3 * PK + q],
                                     H[4 * PK + q], E0 + e0, E1 + e1, E2 + e2);
    H[q] = o.ep0;
    H[PK + q] = o.ep1;
    H[2 * PK + q] = o.ep2;
    H[3 * PK + q] = o.ep3;
    H[4 * PK + q] = o.eq;
    H[5 * PK + q] = o.s33;
  }
}

template <int NT>
__global__ void __launch_bounds__(kW * 32, 1) k_newton_round(RoundArgs A) {
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
  double* sWC = sU;             // w C_q rows  [32][9]   (material phase)
  double* sWS = sU + kQC * 9;   // w σ_q       [32][3]
  double* sK = sU;              // K_aa lower  [NP][NP+1] (after the chunk loop)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Gbuf1 + L::gbuf + static_cast<size_t>(kW) * L::WS);

  const ModelDev& M = A.M;
  const PointsDev& D = A.D;
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
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  double ce00 = 0.0, ce01 = 0.0, ce02 = 0.0, ce11 = 0.0, ce12 = 0.0, ce22 = 0.0;
  int pc = 0;

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
      // ---- material phase: lane = cubature point
      {
        const double* Gq = Gb + lane * S;
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll 8
        for (int a = 0; a < NP; ++a) {
          const double al = sA[a];
          e0 += Gq[a] * al;
          e1 += Gq[NP + a] * al;
          e2 += Gq[2 * NP + a] * al;
        }
        const MatOut o = update_material(M.mat2, h0, h1, h2, h3, h4, E0 + e0, E1 + e1, E2 + e2);
        const double wq = M.w2[q];
        double* wc = sWC + lane * 9;
        const double w00 = wq * o.c00, w01 = wq * o.c01, w02 = wq * o.c02;
        const double w11 = wq * o.c11, w12 = wq * o.c12, w22 = wq * o.c22;
        wc[0] = w00;
        wc[1] = w01;
        wc[2] = w02;
        wc[3] = w01;
        wc[4] = w11;
        wc[5] = w12;
        wc[6] = w02;
        wc[7] = w12;
        wc[8] = w22;
        const double f0 = wq * o.s0, f1 = wq * o.s1, f2 = wq * o.s2;
        sWS[lane * 3 + 0] = f0;
        sWS[lane * 3 + 1] = f1;
        sWS[lane * 3 + 2] = f2;
        s0 += f0;
        s1 += f1;
        s2 += f2;
        ce00 += w00;
        ce01 += w01;
        ce02 += w02;
        ce11 += w11;
        ce12 += w12;
        ce22 += w22;
        pc += (o.plastic && q < M.K2) ? 1 : 0;
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
      // ---- contraction phase: k = 3 q_local + i, four k per DMMA k-step
#pragma unroll 1
      for (int c3 = 0; c3 < (kQC * 3) / 12; ++c3) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const int ql = 4 * c3 + qo[s];
          const int i = io[s];
          const double* wc = sWC + ql * 9 + i * 3;
          const double c0 = wc[0], c1 = wc[1], c2 = wc[2];
          const double ws = sWS[ql * 3 + i];
          const double* g = Gb + ql * S + col;
          double Af[NT], Bf[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double g0 = g[t * 8], g1 = g[NP + t * 8], g2 = g[2 * NP + t * 8];
            Af[t] = (i == 0) ? g0 : ((i == 1) ? g1 : g2);
            Bf[t] = c0 * g0 + c1 * g1 + c2 * g2;
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

  // ---- reductions: r and K_aE over the four k-lanes of each column
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
  // K tiles -> lower triangle of sK
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
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  ce00 = warp_sum(ce00);
  ce01 = warp_sum(ce01);
  ce02 = warp_sum(ce02);
  ce11 = warp_sum(ce11);
  ce12 = warp_sum(ce12);
  ce22 = warp_sum(ce22);
  pc = warp_sum_i(pc);
  __syncwarp();
  // ---- constant elastic-inclusion part: σ_q = C_e (E + G_q α) is linear
  double sa0 = 0.0, sa1 = 0.0, sa2 = 0.0;
  for (int a = lane; a < n; a += 32) {
    const double* kr = M.Kinc + a * NP;
    double s = 0.0;
    for (int b = 0; b < n; ++b) s += kr[b] * sA[b];
    const double* ke = M.KaEinc + a * 3;
    s += ke[0] * E0 + ke[1] * E1 + ke[2] * E2;
    sV[a] += s;
    for (int b = 0; b <= a; ++b) sK[a * LD + b] += kr[b];
    sKaE[a * 3 + 0] += ke[0];
    sKaE[a * 3 + 1] += ke[1];
    sKaE[a * 3 + 2] += ke[2];
    sa0 += ke[0] * sA[a];
    sa1 += ke[1] * sA[a];
    sa2 += ke[2] * sA[a];
  }
  sa0 = warp_sum(sa0);
  sa1 = warp_sum(sa1);
  sa2 = warp_sum(sa2);
  const double* ci = M.CEEinc;
  s0 += sa0 + (ci[0] * E0 + ci[1] * E1 + ci[2] * E2);
  s1 += sa1 + (ci[3] * E0 + ci[4] * E1 + ci[5] * E2);
  s2 += sa2 + (ci[6] * E0 + ci[7] * E1 + ci[8] * E2);
  ce00 += ci[0];
  ce01 += ci[1];
  ce02 += ci[2];
  ce11 += ci[4];
  ce12 += ci[5];
  ce22 += ci[8];
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
      for (int i = 0; i < 3; ++i) A.O.sigma[p * 3 + i] = __longlong_as_double(0x7ff8000000000000ll);
      for (int i = 0; i < 9; ++i) A.O.C[p * 9 + i] = __longlong_as_double(0x7ff8000000000000ll);
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
// K1: history commit at the converged (E, α) of every finished point.
constexpr int kCommitWarps = 8;
constexpr int kCommitPPW = 4;  // points per warp

template <int NP>
__global__ void __launch_bounds__(kCommitWarps * 32) k_commit(ModelDev M, PointsDev D, Outputs O) {
  constexpr int S = 3 * NP + 1;
  constexpr int TS = kQC + 1;  // transposed row stride
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sG = reinterpret_cast<double*>(smem_raw);              // [3*NP][TS]
  double* sAl = sG + 3 * NP * TS;                                 // [warps][PPW][NP]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p_base = (static_cast<int64_t>(blockIdx.x) * kCommitWarps + warp) * kCommitPPW;
  const int64_t PK = D.P * static_cast<int64_t>(M.K2p);
  bool live[kCommitPPW];
  double Ep[kCommitPPW][3];
  int pc[kCommitPPW];
#pragma unroll
  for (int k = 0; k < kCommitPPW; ++k) {
    const int64_t p = p_base + k;
    live[k] = p < D.P && D.st[p].phase == kDone;
    pc[k] = 0;
    Ep[k][0] = Ep[k][1] = Ep[k][2] = 0.0;
    if (live[k]) {
      Ep[k][0] = D.E_ev[p * 3 + 0];
      Ep[k][1] = D.E_ev[p * 3 + 1];
      Ep[k][2] = D.E_ev[p * 3 + 2];
      for (int a = lane; a < NP; a += 32) sAl[(warp * kCommitPPW + k) * NP + a] = D.alpha_ev[p * NP + a];
    }
  }
  for (int c = 0; c < M.nchunks; ++c) {
    __syncthreads();
    for (int e = threadIdx.x; e < kQC * 3 * NP; e += blockDim.x) {
      const int ql = e / (3 * NP), j = e - ql * (3 * NP);
      sG[j * TS + ql] = M.G2[static_cast<size_t>(c * kQC + ql) * S + j];
    }
    __syncthreads();
    const int q = c * kQC + lane;
    const bool real = q < M.K2;
    const MatDev mt = M.mat2;
#pragma unroll
    for (int k = 0; k < kCommitPPW; ++k) {
      if (!live[k]) continue;
      const int64_t p = p_base + k;
      const double* a = sAl + (warp * kCommitPPW + k) * NP;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll 8
      for (int j = 0; j < NP; ++j) {
        const double al = a[j];
        e0 += sG[j * TS + lane] * al;
        e1 += sG[(NP + j) * TS + lane] * al;
        e2 += sG[(2 * NP + j) * TS + lane] * al;
      }
      double* H = D.hist + p * M.K2p + q;
      const MatOut o = update_material(mt, H[0], H[PK], H[2 * PK], H[3 * PK], H[4 * PK], Ep[k][0] + e0,
                                       Ep[k][1] + e1, Ep[k][2] + e2);
      if (real) {
        H[0] = o.ep0;
        H[PK] = o.ep1;
        H[2 * PK] = o.ep2;
        H[3 * PK] = o.ep3;
        H[4 * PK] = o.eq;
        H[5 * PK] = o.s33;
        if (D.flags) D.flags[p * M.K2p + q] = o.plastic ? 1 : 0;
      }
      pc[k] += __popc(__ballot_sync(0xffffffffu, real && o.plastic));
    }
  }
#pragma unroll
  for (int k = 0; k < kCommitPPW; ++k) {
    const int64_t p = p_base + k;
    if (!live[k]) continue;
    if (lane == 0 && O.pcount) O.pcount[p] = pc[k];
    for (int a = lane; a < NP; a += 32) D.alpha_c[p * NP + a] = D.alpha_ev[p * NP + a];
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
    O.res[p] = __longlong_as_double(0x7ff8000000000000ll);
    for (int i = 0; i < 3; ++i) O.sigma[p * 3 + i] = __longlong_as_double(0x7ff8000000000000ll);
    for (int i = 0; i < 9; ++i) O.C[p * 9 + i] = __longlong_as_double(0x7ff8000000000000ll);
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
  const size_t smem = (3 * NP * (kQC + 1) + kCommitWarps * kCommitPPW * NP) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_commit<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  const int64_t per_cta = kCommitWarps * kCommitPPW;
  const int64_t grid = (D.P + per_cta - 1) / per_cta;
  k_commit<NP><<<static_cast<unsigned>(grid), kCommitWarps * 32, smem, s>>>(M, D, O);
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
