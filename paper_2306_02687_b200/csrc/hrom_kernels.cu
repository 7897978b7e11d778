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
// per point; accepting a state moves them by that pass's plastic parts).
//
// k_increment — ONE persistent launch per load increment. Each warp owns a
// macro point at a time (work queue) and drives it through the whole
// increment of run_trajectory (rve.hpp:459-491): assembly passes and the
// reduced Newton / line-search state machine of micro_newton
// (rve.hpp:285-346), bisected sub-steps (:473-478), the static condensation
// C = (C_EE − K_Ea K_aa^-1 K_aE)/V of homogenize (:350-392), and the
// commit-after-acceptance of the history (:283-284, :480).
//  - G rows: the whole J2 operator resident in shared memory when it fits
//    (RES, 8 warps), else a ring of 32-point chunks filled by TMA bulk copies
//    (cp.async.bulk + mbarrier) that all warps consume in the same cyclic
//    order (the last warp to release a stage refills it; no CTA barrier).
//  - Assembly pass: lane = cubature point (ε_q, elastic trial, yield test on
//    the history loaded one chunk ahead); plastic points are compacted
//    (ballot/popc) and only they are contracted on the FP64 tensor cores
//    (mma.sync m8n8k4 f64 = DMMA). K_aa stays in shared memory. The pass also
//    writes the candidate history of its state into the point's non-committed
//    buffer (double-buffered history).
//  - Accepting a converged state flips the point's buffer bit, stores α_c and
//    moves b_p, s_p by the pass's plastic corrections — no commit pass.
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"
#include "hrom_kernels.cuh"

namespace fe2 {

namespace {

using namespace dev;  // TMA / mbarrier, DMMA, warp reductions, fast reciprocals (device_common.cuh)

// D(8x8) += A(8x4) B(4x8) without `volatile`: the compiler may hoist the next
// k-step's fragment loads above it (measured faster in this kernel's loops).
__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ int tri_(int i) { return i * (i + 1) / 2; }

// Left-looking Cholesky of the packed lower triangle sK (row i at i(i+1)/2)
// in place; lane i owns row i (n <= 32). sInv[j] = 1 / L_jj. False if not SPD.
// Look-ahead by one column: while column j's pivot goes through shuffle ->
// rsqrt -> scale, each lane already forms the dot product of column j+1 over
// the final entries k < j; only the k = j term waits for the new column.
__device__ bool warp_cholesky(double* sK, double* sInv, int n, int lane) {
  const bool act = lane < n;
  const double* ri = sK + tri_(act ? lane : 0);
  double s = act ? ri[0] : 0.0;  // K_ij - sum_{k<j} L_ik L_jk for column j = 0
  for (int j = 0; j < n; ++j) {
    double part = 0.0;  // sum_{k<j} L_ik L_{j+1,k}
    if (act && lane > j && j + 1 < n) {
      const double* rn = sK + tri_(j + 1);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int k = 0;
      for (; k + 3 < j; k += 4) {
        a0 += ri[k] * rn[k];
        a1 += ri[k + 1] * rn[k + 1];
        a2 += ri[k + 2] * rn[k + 2];
        a3 += ri[k + 3] * rn[k + 3];
      }
      if (k < j) a0 += ri[k] * rn[k];
      if (k + 1 < j) a1 += ri[k + 1] * rn[k + 1];
      if (k + 2 < j) a2 += ri[k + 2] * rn[k + 2];
      part = (a0 + a1) + (a2 + a3);
    }
    const double d = __shfl_sync(0xffffffffu, s, j);
    if (!(d > 0.0)) return false;
    const double inv = rsqrt_fast(d);
    const double lij = s * inv;
    if (lane == j) {
      sK[tri_(j) + j] = d * inv;
      sInv[j] = inv;
    } else if (act && lane > j) {
      sK[tri_(lane) + j] = lij;
    }
    const double lnj = __shfl_sync(0xffffffffu, lij, (j + 1) & 31);  // L_{j+1,j}
    if (act && lane > j && j + 1 < n) s = ri[j + 1] - (part + lij * lnj);
    __syncwarp();
  }
  return true;
}

// Blocked right-looking Cholesky of the same packed lower sK (used at NT = 4):
// per 8-column block b, (1) the 8 x 8 diagonal block on lanes 0-7 in registers
// (lane r = block row, column broadcast by shuffles), (2) the rows below solved
// against it, one lane per row in registers, (3) the lower block tiles of the
// trailing matrix updated on the FP64 tensor cores, D = A - L_t1 L_t2ᵀ as two
// DMMA m8n8k4 k-steps per tile. Pad rows (>= n) stay zero. sInv[j] = 1 / L_jj.
template <int NT>
__device__ bool warp_cholesky_blk(double* sK, double* sInv, int n, int lane) {
#pragma unroll
  for (int b = 0; b < NT; ++b) {
    const int c0 = 8 * b;
    if (c0 >= n) break;
    {  // (1) diagonal block
      const int r = lane & 7, row = c0 + r;
      const bool vr = lane < 8 && row < n;
      const double* rk = sK + tri_(vr ? row : 0) + c0;
      double a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = (vr && k <= r) ? rk[k] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (c0 + k < n) {
          const double d = __shfl_sync(0xffffffffu, a[k], k);
          if (!(d > 0.0)) return false;
          const double inv = rsqrt_fast(d);
          if (r == k) a[k] = d * inv;
          else if (r > k) a[k] *= inv;
          if (lane == k) sInv[c0 + k] = inv;
#pragma unroll
          for (int kk = k + 1; kk < 8; ++kk) {
            const double lk = __shfl_sync(0xffffffffu, a[k], kk);  // L(c0 + kk, c0 + k)
            if (r >= kk) a[kk] -= a[k] * lk;
          }
        }
      }
      if (vr) {
        double* wk = sK + tri_(row) + c0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k <= r) wk[k] = a[k];
      }
    }
    __syncwarp();
    {  // (2) rows below the block (the block is full: c0 + 8 <= row < n)
      const int row = c0 + 8 + lane;
      if (row < n) {
        double* xr = sK + tri_(row) + c0;
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = xr[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double* lk = sK + tri_(c0 + k) + c0;  // row c0 + k of the diagonal block (broadcast)
          double v = x[k];
#pragma unroll
          for (int m = 0; m < k; ++m) v -= x[m] * lk[m];
          x[k] = v * sInv[c0 + k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) xr[k] = x[k];
      }
    }
    __syncwarp();
    // (3) trailing lower block tiles (t1 >= t2 > b)
    const int fr = lane >> 2, fk = lane & 3;  // fragment row / k-lane
#pragma unroll
    for (int t1 = b + 1; t1 < NT; ++t1) {
      if (8 * t1 >= n) break;
#pragma unroll
      for (int t2 = b + 1; t2 <= t1; ++t2) {
        const int row = 8 * t1 + fr, col0 = 8 * t2 + 2 * fk;
        double* drow = sK + tri_(row);
        double d0 = (row >= col0) ? drow[col0] : 0.0;
        double d1 = (row >= col0 + 1) ? drow[col0 + 1] : 0.0;
        const double* la = sK + tri_(8 * t1 + fr) + c0 + fk;  // A = -L[8 t1 + r][c0 + k]
        const double* lb = sK + tri_(8 * t2 + fr) + c0 + fk;  // B[k][c] = L[8 t2 + c][c0 + k]
        dmma(d0, d1, -la[0], lb[0]);
        dmma(d0, d1, -la[4], lb[4]);
        if (row >= col0) drow[col0] = d0;
        if (row >= col0 + 1) drow[col0 + 1] = d1;
      }
    }
    __syncwarp();
  }
  return true;
}

// Solve L L^T x = b (packed L); lane i holds b_i in, x_i out (n <= 32).
__device__ double warp_chol_solve(const double* sK, const double* sInv, int n, int lane, double b) {
  double x = b;
  const double* ri = sK + tri_(lane < n ? lane : 0);
  for (int j = 0; j < n; ++j) {
    const double yj = __shfl_sync(0xffffffffu, x, j) * sInv[j];
    if (lane == j) x = yj;
    if (lane > j && lane < n) x -= ri[j] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {
    const double xj = __shfl_sync(0xffffffffu, x, j) * sInv[j];
    if (lane == j) x = xj;
    if (lane < j) x -= sK[tri_(j) + lane] * xj;
  }
  return x;
}

#ifndef FE2_KW
#define FE2_KW 16
#endif
#ifndef FE2_MONO_KW
#define FE2_MONO_KW 12
#endif
#ifndef FE2_STAGES
#define FE2_STAGES 6
#endif
#ifndef FE2_MINB
#define FE2_MINB 1
#endif
#ifndef FE2_KWRES
#define FE2_KWRES 12
#endif
#ifndef FE2_GROUP_UNROLL
#define FE2_GROUP_UNROLL 1
#endif
constexpr int kGroupUnroll = FE2_GROUP_UNROLL;  // plastic-group loop unroll (tuning)
// warps per CTA of the streamed-G ring increment kernel: 16 (128 registers) for NP = 8;
// 12 (168 registers, no spills) for NP = 16 / 24 (n = 16: +19% at K = 1,000, +17% at K = 4,000
// over 8 warps); NP = 32 spills 216 B at 168 registers and keeps 8 warps with 255 (the
// 16-warp builds spilled 0.5-1.1 KB per thread from NP = 16 on)
#ifndef FE2_KW_WIDE
#define FE2_KW_WIDE 8
#endif
#ifndef FE2_KW_MID
#define FE2_KW_MID 12
#endif
constexpr int kw_for(int NT) { return NT == 1 ? FE2_KW : (NT <= 3 ? FE2_KW_MID : FE2_KW_WIDE); }
// warps per CTA when the whole G2 is resident in shared memory: 12 (168 registers, the
// warp-uniform Newton state in shared memory, WarpSt) — measured +12% over 8 warps with
// 255 registers at n = 24; NP = 32 spills at 168 registers and keeps 8
// ... and 16 warps (128 registers; 12 / 64 B of spills) for NP = 8 / 16: +6-11% at K = 100, +6% at K = 400
#ifndef FE2_KWRES_SMALL
#define FE2_KWRES_SMALL 16
#endif
constexpr int kwres_for(int NT) { return NT == 4 ? 8 : (NT <= 2 ? FE2_KWRES_SMALL : FE2_KWRES); }
// warps per CTA of the monolithic iteration (ring-streamed G): 16 at NP = 8 (128 registers), 12
// above (168 registers: the 16-warp builds spilled 64-320 B; measured +10% at n = 24, +2% at
// n = 32, and 16 warps 7% faster at n = 12)
constexpr int mono_kw(int NT) { return NT == 1 ? 16 : FE2_MONO_KW; }
constexpr int kMaxStages = FE2_STAGES;  // G-chunk ring depth (shared by the CTA), at most

template <int NP, int W>
struct IncLayout {
  // G2 record of a cubature point: rows at R1 / R2 (see g2_row_offset) then
  // [w | 0]; S/2 odd keeps the lane-per-point 128-bit row loads conflict-free
  static constexpr int R1 = g2_row_offset(NP, 1), R2 = g2_row_offset(NP, 2);
  static constexpr int S = R2 + NP + 2;
  static constexpr int chunk = kQC * S;                      // doubles per ring stage
  static constexpr int kSlots = kQC * 6 + kQC * 3 + kQC;     // w ΔC (6 unique), w Δσ, point index
  static constexpr int kTri = NP * (NP + 1) / 2;              // packed lower K_aa
  static constexpr int kUnion = (kSlots > kTri) ? kSlots : kTri;
  static constexpr int kState = 40;                     // WarpSt (warp-uniform Newton / pass state)
  // per-warp scratch (doubles), even so that every warp's α vector stays 16-B aligned
  static constexpr int WS = (6 * NP + 3 * NP + kUnion + kState + 1) & ~1;
  // ring depth: as deep as the 227 KB shared-memory budget allows (<= kMaxStages)
  static constexpr long kBudget = 227L * 1024 - 512 - static_cast<long>(W) * WS * 8;
  static constexpr int kFit = static_cast<int>(kBudget / (static_cast<long>(chunk) * 8));
  static constexpr int ST = kFit < 2 ? 2 : (kFit > kMaxStages ? kMaxStages : kFit);
  static constexpr size_t ring_bytes = static_cast<size_t>(ST) * chunk * sizeof(double);
  // control block: full[ST] (u64) | cnt[ST] (int) | ctrl (u64)
  static constexpr int kCntOff = ST * 8;
  static constexpr int kCtrlOff = ((kCntOff + ST * 4 + 7) / 8) * 8;
  static constexpr size_t bytes = ring_bytes + static_cast<size_t>(W) * WS * sizeof(double) + kCtrlOff + 8;
  // resident variant: the whole G2 (nch chunks) in shared memory, no ring
  static constexpr size_t res_bytes(int nch) {
    return static_cast<size_t>(nch) * chunk * sizeof(double) + static_cast<size_t>(W) * WS * sizeof(double) + kCtrlOff + 8;
  }
};

// Shared-memory ring of G chunks. ctrl packs {working warps (hi 32), issued
// positions (lo 32)} so that a refill can only be issued while some warp
// still works, and an idle warp knows exactly which positions will arrive.
struct Ring {
  double* buf;
  uint64_t* full;
  int* cnt;
  unsigned long long* ctrl;
  const double* G2;
  int nch;
  int chunk;           // doubles per stage
  volatile int* tr;    // watchdog trace slot of this warp (or null)
  int stages;          // ring depth
  int nwarps;          // warps consuming the ring
  bool res;            // G2 fully resident: no waits, no refills
};

__device__ __forceinline__ void trace(const Ring& R, int seq, int code) {
  if (R.tr && (threadIdx.x & 31) == 0) {
    R.tr[0] = seq;
    R.tr[1] = code;
    R.tr[2] = static_cast<int>(*reinterpret_cast<volatile unsigned long long*>(R.ctrl) & 0xffffffffull);
    R.tr[3] = static_cast<int>(*reinterpret_cast<volatile unsigned long long*>(R.ctrl) >> 32);
    __threadfence_system();
  }
}

__device__ __forceinline__ const double* ring_wait(const Ring& R, int seq) {
  if (R.res) return R.buf + static_cast<size_t>(seq % R.nch) * R.chunk;
  const int s = seq % R.stages;
  trace(R, seq, 1);
  mbar_wait(&R.full[s], static_cast<uint32_t>((seq / R.stages) & 1));
  trace(R, seq, 2);
  return R.buf + static_cast<size_t>(s) * R.chunk;
}

__device__ __forceinline__ void ring_release(const Ring& R, int seq, int lane) {
  __syncwarp();
  if (R.res) return;
  if (lane == 0) {
    const int s = seq % R.stages;
    __threadfence_block();
    if (atomicAdd(&R.cnt[s], 1) == R.nwarps - 1) {
      R.cnt[s] = 0;
      const int nxt = seq + R.stages;
      unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(R.ctrl);
      bool issue = false;
      while ((old >> 32) > 0) {
        const unsigned long long lo = old & 0xffffffffull;
        const unsigned long long nw = (old & 0xffffffff00000000ull) | (lo > static_cast<unsigned>(nxt + 1) ? lo : static_cast<unsigned>(nxt + 1));
        const unsigned long long got = atomicCAS(R.ctrl, old, nw);
        if (got == old) {
          issue = true;
          break;
        }
        old = got;
      }
      if (issue) {
        const uint32_t bytes = static_cast<uint32_t>(R.chunk * sizeof(double));
        fence_proxy_async();
        mbar_expect_tx(&R.full[s], bytes);
        tma_load_1d(R.buf + static_cast<size_t>(s) * R.chunk, R.G2 + static_cast<size_t>(nxt % R.nch) * R.chunk,
                    bytes, &R.full[s]);
      }
    }
  }
  __syncwarp();
}

// A warp without more points keeps consuming (so the ring keeps turning for
// the others) until no warp works and every issued position was consumed.
__device__ void ring_drain(const Ring& R, int seq, int lane) {
  if (R.res) return;
  if (lane == 0) atomicAdd(R.ctrl, 0xffffffff00000000ull);  // working -= 1 (mod 2^64)
  __syncwarp();
  trace(R, seq, 4);
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(R.ctrl, 0ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    const int issued = static_cast<int>(c & 0xffffffffull);
    const unsigned working = static_cast<unsigned>(c >> 32);
    if (seq < issued) {
      ring_wait(R, seq);
      ring_release(R, seq, lane);
      ++seq;
      continue;
    }
    if (working == 0) break;
    __nanosleep(64);
  }
  trace(R, seq, 5);
}

// Warp-uniform state of the point a warp is driving, kept in the warp's shared
// scratch instead of registers: the outputs of the last assembly pass (written
// once per pass), the point's macro strains (written once per point) and the
// micro_newton / run_trajectory state machine, parked here across each assembly
// pass. Every lane stores its own identical copy and nothing is read-modify-
// written in shared memory, so lanes need not run converged. Keeping this out
// of the register file lets the chunk loop run at <= 168 registers (12 warps).
struct WarpSt {
  double s0, s1, s2, ce00, ce01, ce02, ce11, ce12, ce22, dsp0, dsp1, dsp2;  // pass outputs
  double a, rn_it, best_rn, best_a, ref, done, frac;                        // Newton / line search
  double E0, E1, E2, Ep0, Ep1, Ep2, Et0, Et1, Et2;                          // macro strain
  int mode, it, ls, iters, bis, err, np_last, k_linear;
  int merr, pad_;  // iterative materials: some return map of the last pass failed (ErrorCode::material)
  unsigned cnt[4];  // assemblies, commits, plastic evaluations, plastic points of accepted states (lane 0)
};
static_assert(sizeof(WarpSt) <= 40 * sizeof(double), "WarpSt exceeds IncLayout::kState");

// Phase timeline of lane 0 of every warp (tuning builds only: -DFE2_INC_PROF; the
// last warp to finish prints the sums): 0 strain GEMV (incl. ring wait), 1 trial /
// yield / candidate history / slots, 2 DMMA contraction, 3 pass tail (reductions,
// K_aa scatter, elastic predictor), 4 factorisation, 5 rest of the Newton state
// machine (solves, condensation, commit, work queue).
#ifdef FE2_INC_PROF
__device__ unsigned long long g_inc_prof[7];
#define INC_T(k)                                              \
  do {                                                        \
    if (lane == 0) {                                          \
      const long long t_ = clock64();                         \
      prof[k] += static_cast<unsigned long long>(t_ - t_prof); \
      t_prof = t_;                                            \
    }                                                         \
  } while (0)
#else
#define INC_T(k) \
  do {           \
  } while (0)
#endif

// RES: the whole projected operator G2 sits in shared memory for the kernel's
// lifetime (loaded once by TMA): warps never wait on each other for G chunks.
// Otherwise G2 streams through the CTA-shared ring (W warps, ST stages).
// GEN: the history-carrying points follow an iterative material (power law /
// creep, general_return) instead of the closed-form J2 return.
template <int NT, int W, bool RES, bool MONO = false, bool GEN = false>
__global__ void __launch_bounds__(W * 32, RES ? 1 : FE2_MINB) k_increment(IncArgs A) {
  constexpr int NP = 8 * NT;
  constexpr int NTP = NT * (NT + 1) / 2;
  using L = IncLayout<NP, W>;
  constexpr int S = L::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef FE2_INC_PROF
  unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
  long long t_prof = clock64();
#endif
  const size_t ring_bytes = RES ? static_cast<size_t>(A.M.nchunks) * L::chunk * sizeof(double) : L::ring_bytes;
  double* ring_buf = reinterpret_cast<double*>(smem_raw);
  double* wbase = reinterpret_cast<double*>(smem_raw + ring_bytes) + static_cast<size_t>(warp) * L::WS;
  unsigned char* ctrl_base = smem_raw + ring_bytes + static_cast<size_t>(W) * L::WS * sizeof(double);
  uint64_t* full = reinterpret_cast<uint64_t*>(ctrl_base);
  int* cnt = reinterpret_cast<int*>(ctrl_base + L::kCntOff);
  unsigned long long* ctrl = reinterpret_cast<unsigned long long*>(ctrl_base + L::kCtrlOff);

  double* sAev = wbase;          // α at the evaluation point
  double* sAl = sAev + NP;       // α, current Newton iterate
  double* sDA = sAl + NP;        // Δα
  double* sV = sDA + NP;         // residual r
  double* sInv = sV + NP;        // 1 / L_jj
  double* sRp = sInv + NP;       // plastic part of r (Σ_plastic w G^T Δσ) of the last pass
  double* sKaE = sRp + NP;       // K_aE [NP][3]
  double* sU = sKaE + 3 * NP;
  double* sDC = sU;                                 // [32][6] w ΔC (00 01 02 11 12 22) of the plastic slots
  double* sDS = sU + kQC * 6;                       // [32][3] w Δσ of the plastic slots
  int* sQ = reinterpret_cast<int*>(sU + kQC * 9);   // [32]    chunk-local cubature index
  double* sK = sU;                                  // K_aa packed lower (after an assembly pass)

  const ModelDev& M = A.M;
  const PointsDev& D = A.D;
  const MatDev& mt = M.mat2;
  const int nch = M.nchunks;
  const Ring R{ring_buf, full, cnt, ctrl, M.G2, nch, L::chunk,
               A.trace ? A.trace + (static_cast<size_t>(blockIdx.x) * W + warp) * 4 : nullptr, L::ST, W, RES};

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::ST; ++s) {
      mbar_init(&full[s], 1);
      cnt[s] = 0;
    }
    *ctrl = (static_cast<unsigned long long>(W) << 32) | static_cast<unsigned long long>(L::ST);
  }
  if (threadIdx.x == 0) fence_mbar_init();
  __syncthreads();
  if (RES) {  // the whole operator, once: nch bulk copies on one barrier
    if (threadIdx.x == 0) {
      const uint32_t bytes = static_cast<uint32_t>(L::chunk * sizeof(double));
      mbar_expect_tx(&full[0], bytes * static_cast<uint32_t>(nch));
      for (int c = 0; c < nch; ++c)
        tma_load_1d(ring_buf + static_cast<size_t>(c) * L::chunk, M.G2 + static_cast<size_t>(c) * L::chunk, bytes,
                    &full[0]);
    }
    mbar_wait(&full[0], 0);
  } else if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(L::chunk * sizeof(double));
    for (int s = 0; s < L::ST; ++s) {
      mbar_expect_tx(&full[s], bytes);
      tma_load_1d(ring_buf + static_cast<size_t>(s) * L::chunk, M.G2 + static_cast<size_t>(s % nch) * L::chunk,
                  bytes, &full[s]);
    }
  }

  const int m = lane & 3, col = lane >> 2;
  int seq = 0;
  WarpSt* const W_ = reinterpret_cast<WarpSt*>(wbase + L::WS - L::kState);
  // counters: lane 0's private copies in the warp state (only lane 0 updates / reads them)
  unsigned* const cnt_ = W_->cnt;
  if (lane == 0) cnt_[0] = cnt_[1] = cnt_[2] = cnt_[3] = 0;

  // outputs of an assembly pass (warp-uniform after the reductions)
  double &s0 = W_->s0, &s1 = W_->s1, &s2 = W_->s2, &ce00 = W_->ce00, &ce01 = W_->ce01, &ce02 = W_->ce02;
  double &ce11 = W_->ce11, &ce12 = W_->ce12, &ce22 = W_->ce22;
  double &dsp0 = W_->dsp0, &dsp1 = W_->dsp1, &dsp2 = W_->dsp2;  // plastic parts of Σraw (for the commit)
  int& np_last = W_->np_last;   // plastic points of the last pass
  int& k_linear = W_->k_linear;  // the last assembly had no plastic point (K_aa == K_e)
  s0 = s1 = s2 = ce00 = ce01 = ce02 = ce11 = ce12 = ce22 = dsp0 = dsp1 = dsp2 = 0.0;
  np_last = k_linear = 0;
  const bool dbg = A.dbg != nullptr;
  const int n = M.n;

  // ------------------------------------------------ per-lane history loads
  // Lane = cubature point: its (εp, eq) come from the point's committed buffer
  // by coalesced 8-B loads (256 B per warp and component), one chunk ahead; at
  // the end of a pass the first chunk of the predicted next pass (same point,
  // or the next point after the final acceptance) is loaded so it arrives
  // during the Newton phase. The lane that reads a history entry is the lane
  // that wrote its candidate, so program order covers read-after-write.
  double nh0 = 0.0, nh1 = 0.0, nh2 = 0.0, nh3 = 0.0, nh4 = 0.0;  // chunk 0 of point pf_p
  int64_t pf_p = -1;
  auto hbase = [&](int64_t p) -> const double* {  // committed buffer of point p, this lane
    return D.hist + (D.st[p].pad[0] ? D.hist_alt : 0) + p * nch * (5 * kQC) + lane;
  };
  auto hload = [&](const double* base, int c, double& a0, double& a1, double& a2, double& a3, double& a4) {
    const double* b = base + c * (5 * kQC);
    a0 = b[0];
    a1 = b[kQC];
    a2 = b[2 * kQC];
    a3 = b[3 * kQC];
    a4 = b[4 * kQC];
  };

  // ---------------------------------------------------------------- passes
  auto assembly_pass = [&](int64_t p, double E0, double E1, double E2, int64_t pred) {
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
    double c00 = 0.0, c01 = 0.0, c02 = 0.0, c11 = 0.0, c12 = 0.0, c22 = 0.0, ds0 = 0.0, ds1 = 0.0, ds2 = 0.0;
    int np_tot = 0;
    bool merr = false;  // GEN: a return map of this pass failed
    // GEN creep: the time of this sub-step, PathStep::dt x (target - done) (rve.hpp:466)
    const double dt_sub = GEN ? mt.dt * (fmin(1.0, W_->done + W_->frac) - W_->done) : 0.0;
    const bool cur = D.st[p].pad[0] != 0;  // committed buffer; the candidate goes to the other one
    double* hcand = D.hist + (cur ? 0 : D.hist_alt) + p * nch * (5 * kQC) + lane;
    uint8_t* fcand = D.flags ? D.flags + (cur ? 0 : D.flags_alt) + p * M.K2p : nullptr;
    double x0, x1, x2, x3, x4;  // history of the next chunk
    const double* hcur = D.hist + (cur ? D.hist_alt : 0) + p * nch * (5 * kQC) + lane;
    if (pf_p == p) {
      x0 = nh0;
      x1 = nh1;
      x2 = nh2;
      x3 = nh3;
      x4 = nh4;
    } else {
      hload(hcur, 0, x0, x1, x2, x3, x4);
    }
    pf_p = -1;
    INC_T(5);
    for (int c = 0; c < nch; ++c) {
      const double h0 = x0, h1 = x1, h2 = x2, h3 = x3, h4 = x4;
      if (c + 1 < nch) {
        hload(hcur, c + 1, x0, x1, x2, x3, x4);
      } else if (pred >= 0) {
        hload(pred == p ? hcur : hbase(pred), 0, nh0, nh1, nh2, nh3, nh4);
        pf_p = pred;
      }
      const double* Gb = RES ? R.buf + static_cast<size_t>(c) * L::chunk : ring_wait(R, seq);
      const int q = c * kQC + lane;
      // lane = cubature point: strain, elastic trial, yield test
      const double* Gq = Gb + lane * S;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0;
      {  // ε = G_q α with 128-bit shared loads (rows are 16-B aligned, S even)
        const double2* g0v = reinterpret_cast<const double2*>(Gq);
        const double2* g1v = reinterpret_cast<const double2*>(Gq + L::R1);
        const double2* g2v = reinterpret_cast<const double2*>(Gq + L::R2);
        const double2* av = reinterpret_cast<const double2*>(sAev);
#pragma unroll 4
        for (int a = 0; a < NP / 2; ++a) {
          const double2 al = av[a], x0 = g0v[a], x1 = g1v[a], x2 = g2v[a];
          e0 += x0.x * al.x;
          f0 += x0.y * al.y;
          e1 += x1.x * al.x;
          f1 += x1.y * al.y;
          e2 += x2.x * al.x;
          f2 += x2.y * al.y;
        }
      }
      INC_T(0);
      const Trial T = trial_state(mt, h0, h1, h2, h3, h4, E0 + (e0 + f0), E1 + (e1 + f1), E2 + (e2 + f2));
      bool plastic;
      double dlam_g = 0.0, kq_g = 0.0;
      if constexpr (GEN) {
        plastic = false;
        if (q < M.K2) {
          const GenRet g = general_return(mt, T.ss, h4, dt_sub);
          plastic = g.plastic;
          dlam_g = g.dlam;
          kq_g = g.kq;
          merr = merr || !g.ok;
        }
      } else {
        plastic = (T.f > 0.0) && (q < M.K2);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, plastic);
      const int np = __popc(bal);
      np_tot += np;
      {  // candidate history of this state (finish_return, materials.hpp:173-185): written every
         // pass into the non-committed buffer, adopted by a flip if the state is accepted
        double n0 = h0, n1 = h1, n2 = h2, n3 = h3, n4 = h4;
        if (plastic) {
          const double dlam = GEN ? dlam_g : T.f * mt.inv_denom;
          const double ce = 1.5 * dlam * (0.81649658092772603273 * T.inv_ns);
          n0 = h0 + ce * T.d0;
          n1 = h1 + ce * T.d1;
          n2 = h2 + ce * T.d2;
          n3 = h3 + ce * T.d3;
          n4 = h4 + dlam;
        }
        double* Hd = hcand + c * (5 * kQC);
        Hd[0] = n0;
        Hd[kQC] = n1;
        Hd[2 * kQC] = n2;
        Hd[3 * kQC] = n3;
        Hd[4 * kQC] = n4;
        if (fcand && q < M.K2) fcand[q] = plastic ? 1 : 0;
      }
      if (plastic) {
        const Corr cr = GEN ? radial_return_gen(mt, T, dlam_g, kq_g) : radial_return(mt, T);
        const double wq = Gq[L::R2 + NP];  // cubature weight rides in the record's pad
        const int slot = __popc(bal & ((1u << lane) - 1u));
        const double w00 = wq * cr.dc00, w01 = wq * cr.dc01, w02 = wq * cr.dc02;
        const double w11 = wq * cr.dc11, w12 = wq * cr.dc12, w22 = wq * cr.dc22;
        double* dc = sDC + slot * 6;
        dc[0] = w00;
        dc[1] = w01;
        dc[2] = w02;
        dc[3] = w11;
        dc[4] = w12;
        dc[5] = w22;
        const double g0 = wq * cr.ds0, g1 = wq * cr.ds1, g2 = wq * cr.ds2;
        sDS[slot * 3 + 0] = g0;
        sDS[slot * 3 + 1] = g1;
        sDS[slot * 3 + 2] = g2;
        sQ[slot] = lane;
        c00 += w00;
        c01 += w01;
        c02 += w02;
        c11 += w11;
        c12 += w12;
        c22 += w22;
        ds0 += g0;
        ds1 += g1;
        ds2 += g2;
      }
      const int np4 = (np + 3) & ~3;  // zero the slots that round np up to a multiple of 4
      if (lane >= np && lane < np4) {
#pragma unroll
        for (int e = 0; e < 6; ++e) sDC[lane * 6 + e] = 0.0;
        sDS[lane * 3 + 0] = sDS[lane * 3 + 1] = sDS[lane * 3 + 2] = 0.0;
        sQ[lane] = 0;
      }
      __syncwarp();
      INC_T(1);
      // plastic contraction on DMMA. A group = 4 plastic slots; k-lane m owns slot 4g + m
      // and the k-step i (0..2) contracts strain row i of the four slots: the lane loads
      // its slot's three G rows ONCE per group (each element once, no re-loads per
      // row), forms the three rows of B = (w ΔC) G in registers and feeds A = G row i.
      const int ng = np4 >> 2;
#pragma unroll kGroupUnroll
      for (int g = 0; g < ng; ++g) {
        const int slot = 4 * g + m;
        const double* wc = sDC + slot * 6;  // w ΔC: 00 01 02 11 12 22
        const double w00 = wc[0], w01 = wc[1], w02 = wc[2], w11 = wc[3], w12 = wc[4], w22 = wc[5];
        const double ws0 = sDS[slot * 3 + 0], ws1 = sDS[slot * 3 + 1], ws2 = sDS[slot * 3 + 2];
        const double* gp = Gb + sQ[slot] * S + col;
        double G0[NT], G1[NT], G2[NT], B0[NT], B1[NT], B2[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          G0[t] = gp[t * 8];
          G1[t] = gp[L::R1 + t * 8];
          G2[t] = gp[L::R2 + t * 8];
          B0[t] = w00 * G0[t] + w01 * G1[t] + w02 * G2[t];
          B1[t] = w01 * G0[t] + w11 * G1[t] + w12 * G2[t];
          B2[t] = w02 * G0[t] + w12 * G1[t] + w22 * G2[t];
          kae[t][0] += B0[t];
          kae[t][1] += B1[t];
          kae[t][2] += B2[t];
          rr[t] += ws0 * G0[t] + ws1 * G1[t] + ws2 * G2[t];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {  // k-step i: row i of the four slots
          int ti = 0;
#pragma unroll
          for (int t1 = 0; t1 < NT; ++t1)
#pragma unroll
            for (int t2 = t1; t2 < NT; ++t2) {
              const double a_ = i == 0 ? G0[t1] : (i == 1 ? G1[t1] : G2[t1]);
              const double b_ = i == 0 ? B0[t2] : (i == 1 ? B1[t2] : B2[t2]);
              dmma_nv(acc[ti][0], acc[ti][1], a_, b_);
              ++ti;
            }
        }
      }
      INC_T(2);
      ring_release(R, seq, lane);
      ++seq;
    }
    // reductions: r and K_aE corrections over the four k-lanes of each column
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double v = rr[t];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      double ki[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {  // kae[t][i]: strain row i of this lane's slots
        double x = kae[t][i];
        x += __shfl_xor_sync(0xffffffffu, x, 1);
        x += __shfl_xor_sync(0xffffffffu, x, 2);
        ki[i] = x;
      }
      if (m == 0) {
        const int a = t * 8 + col;
        sV[a] = v;
        sRp[a] = v;
        sKaE[a * 3 + 0] = ki[0];
        sKaE[a * 3 + 1] = ki[1];
        sKaE[a * 3 + 2] = ki[2];
      }
    }
    __syncwarp();
    {  // K_aa corrections -> lower triangle of sK (slots are dead now)
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
              sK[tri_(cl) + row] = acc[ti][e];
            else if (row >= cl)
              sK[tri_(row) + cl] = acc[ti][e];
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
    // elastic predictor part (constant K_e, K_aE,e, C_EE,e) and b_p, s_p
    double sa0 = 0.0, sa1 = 0.0, sa2 = 0.0;
    if (lane < n) {
      const int a = lane;
      const double* ke = M.KaEe + a * 3;
      double sx = 0.0, sy = 0.0;
      double* ka = sK + tri_(a);
      int b = 0;
      for (; b + 1 < n; b += 2) {
        const double k0 = M.Ke[b * NP + a], k1 = M.Ke[(b + 1) * NP + a];  // symmetric: coalesced reads
        sx += k0 * sAev[b];
        sy += k1 * sAev[b + 1];
        if (b <= a) ka[b] += k0;
        if (b + 1 <= a) ka[b + 1] += k1;
      }
      if (b < n) {
        const double k0 = M.Ke[b * NP + a];
        sx += k0 * sAev[b];
        if (b <= a) ka[b] += k0;
      }
      const double sr = (sx + sy) + (ke[0] * E0 + ke[1] * E1 + ke[2] * E2);
      sV[a] += sr - D.bp[p * NP + a];
      sKaE[a * 3 + 0] += ke[0];
      sKaE[a * 3 + 1] += ke[1];
      sKaE[a * 3 + 2] += ke[2];
      sa0 = ke[0] * sAev[a];
      sa1 = ke[1] * sAev[a];
      sa2 = ke[2] * sAev[a];
    }
    sa0 = warp_sum(sa0);
    sa1 = warp_sum(sa1);
    sa2 = warp_sum(sa2);
    const double* ce = M.CEEe;
    const double* spp = D.sp + p * 4;
    s0 = ds0 + sa0 + (ce[0] * E0 + ce[1] * E1 + ce[2] * E2) - spp[0];
    s1 = ds1 + sa1 + (ce[3] * E0 + ce[4] * E1 + ce[5] * E2) - spp[1];
    s2 = ds2 + sa2 + (ce[6] * E0 + ce[7] * E1 + ce[8] * E2) - spp[2];
    ce00 = ce[0] + c00;
    ce01 = ce[1] + c01;
    ce02 = ce[2] + c02;
    ce11 = ce[4] + c11;
    ce12 = ce[5] + c12;
    ce22 = ce[8] + c22;
    dsp0 = ds0;
    dsp1 = ds1;
    dsp2 = ds2;
    np_last = np_tot;
    k_linear = (np_tot == 0) ? 1 : 0;
    if constexpr (GEN) W_->merr = __any_sync(0xffffffffu, merr) ? 1 : 0;
    if (lane == 0) {
      cnt_[2] += static_cast<unsigned>(np_tot);
      cnt_[0] += 1;
    }
    __syncwarp();
    INC_T(3);
  };

  // Factor K_aa. With no plastic point in the assembly K_aa == K_e exactly,
  // whose factor was computed once on the host.
  auto factor = [&]() -> bool {
    INC_T(5);
    if (k_linear) {
      for (int e = lane; e < tri_(n); e += 32) sK[e] = M.Le[e];  // packed lower, coalesced
      if (lane < n) sInv[lane] = M.LeInv[lane];
      __syncwarp();
      INC_T(4);
      return true;
    }
    // blocked (DMMA trailing updates) for four 8-column blocks with G resident: +5% at n = 32,
    // K = 600; the left-looking form was measured faster at n <= 24 (1-2%) and in the
    // ring-streamed kernel (3% at n = 32, K = 4,000)
    bool ok;
    if constexpr (NT == 4 && RES) ok = warp_cholesky_blk<NT>(sK, sInv, n, lane);
    else ok = warp_cholesky(sK, sInv, n, lane);
    INC_T(4);
    return ok;
  };

  // Accept the state of the last assembly pass: its candidate history (already
  // in the other buffer) becomes the committed one, and the committed
  // plastic-strain loads move by the pass's plastic corrections
  // (w S(Δεp) = -w Δσ for the deviatoric return): b_p -= r_plastic, s_p -= Σ w Δσ.
  auto commit_point = [&](int64_t p) -> int {
    for (int a = lane; a < NP; a += 32) {
      D.alpha_c[p * NP + a] = sAev[a];
      D.bp[p * NP + a] -= sRp[a];
    }
    if (lane == 0) {
      D.sp[p * 4 + 0] -= dsp0;
      D.sp[p * 4 + 1] -= dsp1;
      D.sp[p * 4 + 2] -= dsp2;
      D.st[p].pad[0] ^= 1;
    }
    if (lane == 0) {
      cnt_[1] += 1;
      cnt_[3] += static_cast<unsigned>(np_last);
    }
    __syncwarp();
    return np_last;
  };

  const NewtonCfg& cfg = A.cfg;
  constexpr int kSolver = 1 + 4;    // 1 + ErrorCode::solver
  constexpr int kMaterial = 1 + 3;  // 1 + ErrorCode::material

  // Every large piece (assembly pass, factorization, acceptance) has exactly
  // one call site below, so each is inlined once: the kernel's instruction
  // footprint stays small enough that warps in different phases do not
  // thrash the instruction cache.
  // (dbg: assembly dump for parity tests — r, K full, KaE, C_EE, S_raw)
  auto dump = [&]() {
    double* o = A.dbg;
    for (int a = lane; a < n; a += 32) o[a] = sV[a];
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      o[n + e] = (j <= i) ? sK[tri_(i) + j] : sK[tri_(j) + i];
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
  };

  // Monolithic scheme ("micro problems advance one Newton
  // iteration per macro iteration sharing the same consistent linearization"):
  // one reduced iteration of point p at the macro strain E of this macro
  // iterate. The linearised micro equation K Δα = -(r + K_aE ΔE) is
  // condensed: the macro code receives Σ~ = (Σ_raw - K_Eα K^-1 r) / V and
  // C = (C_EE - K_Eα K^-1 K_aE) / V, and the next call moves α by
  // -(K^-1 r + K^-1 K_aE ΔE) once ΔE is known. No commit (launch_mono_commit).
  auto mono_point = [&](int64_t p, double E0, double E1, double E2) {
    double* rec = A.mono + p * mono_stride(NP);
    const double* z = rec;
    double* tail = rec + 6 * NP;
    if (A.mono_first) {
      for (int b = lane; b < NP; b += 32) sAev[b] = D.alpha_c[p * NP + b];
    } else {
      const double d0 = E0 - tail[0], d1 = E1 - tail[1], d2 = E2 - tail[2];
      for (int b = lane; b < NP; b += 32)
        sAev[b] = (b < n) ? rec[5 * NP + b] - (z[b] + z[NP + b] * d0 + z[2 * NP + b] * d1 + z[3 * NP + b] * d2)
                          : 0.0;
    }
    __syncwarp();
    assembly_pass(p, E0, E1, E2, -1);
    const double rl = (lane < n) ? sV[lane] : 0.0;
    const double rn = sqrt(warp_sum(rl * rl));
    // micro scale: max(|r| at the step's first iteration, |Σ_raw| now) — E moves during a monolithic step
    const double r_first = A.mono_first ? rn : tail[6];
    const double ref = fmax(fmax(r_first, sqrt(s0 * s0 + s1 * s1 + s2 * s2)), 1e-30);
    if (!factor()) {  // fatal for the point: mono_commit skips it, later iterations report it
      if (lane == 0) {
        A.O.status[p] = kSolver;
        A.O.iters[p] = 1;
        A.O.res[p] = rn / ref;
        D.st[p].err = kSolver;
      }
      __syncwarp();
      return;
    }
    const double k0 = (lane < n) ? sKaE[lane * 3 + 0] : 0.0;
    const double k1 = (lane < n) ? sKaE[lane * 3 + 1] : 0.0;
    const double k2 = (lane < n) ? sKaE[lane * 3 + 2] : 0.0;
    const double zr = warp_chol_solve(sK, sInv, n, lane, rl);
    const double z0 = warp_chol_solve(sK, sInv, n, lane, k0);
    const double z1 = warp_chol_solve(sK, sInv, n, lane, k1);
    const double z2 = warp_chol_solve(sK, sInv, n, lane, k2);
    const double t0 = warp_sum(k0 * zr), t1 = warp_sum(k1 * zr), t2 = warp_sum(k2 * zr);
    const double q00 = warp_sum(k0 * z0), q11 = warp_sum(k1 * z1), q22 = warp_sum(k2 * z2);
    const double q01 = 0.5 * (warp_sum(k0 * z1) + warp_sum(k1 * z0));
    const double q02 = 0.5 * (warp_sum(k0 * z2) + warp_sum(k2 * z0));
    const double q12 = 0.5 * (warp_sum(k1 * z2) + warp_sum(k2 * z1));
    if (lane < NP) {
      rec[lane] = zr;
      rec[NP + lane] = z0;
      rec[2 * NP + lane] = z1;
      rec[3 * NP + lane] = z2;
      rec[4 * NP + lane] = sRp[lane];
      rec[5 * NP + lane] = sAev[lane];
    }
    if (lane == 0) {
      const double V = M.volume;
      double* Cp = A.O.C + p * 9;
      Cp[0] = (ce00 - q00) / V;
      Cp[1] = (ce01 - q01) / V;
      Cp[2] = (ce02 - q02) / V;
      Cp[3] = Cp[1];
      Cp[4] = (ce11 - q11) / V;
      Cp[5] = (ce12 - q12) / V;
      Cp[6] = Cp[2];
      Cp[7] = Cp[5];
      Cp[8] = (ce22 - q22) / V;
      A.O.sigma[p * 3 + 0] = (s0 - t0) / V;
      A.O.sigma[p * 3 + 1] = (s1 - t1) / V;
      A.O.sigma[p * 3 + 2] = (s2 - t2) / V;
      A.O.res[p] = rn / ref;
      A.O.iters[p] = 1;
      A.O.status[p] = 0;
      if (A.O.pcount) A.O.pcount[p] = np_last;
      tail[0] = E0;
      tail[1] = E1;
      tail[2] = E2;
      tail[3] = dsp0;
      tail[4] = dsp1;
      tail[5] = dsp2;
      tail[6] = r_first;
    }
    __syncwarp();
  };

  // ------------------------------------------------------------ point loop
  auto grab = [&]() -> int64_t {
    if (dbg) return (blockIdx.x == 0 && warp == 0 && seq == 0) ? A.dbg_point : D.P;
    int v = 0;
    if (lane == 0) v = atomicAdd(A.work, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  int64_t p_next = grab();
  while (p_next < D.P) {
    const int64_t p = p_next;
    p_next = -1;
    double &Ep0 = W_->Ep0, &Ep1 = W_->Ep1, &Ep2 = W_->Ep2, &Et0 = W_->Et0, &Et1 = W_->Et1, &Et2 = W_->Et2;
    Ep0 = dbg ? 0.0 : D.E_c[p * 3 + 0];
    Ep1 = dbg ? 0.0 : D.E_c[p * 3 + 1];
    Ep2 = dbg ? 0.0 : D.E_c[p * 3 + 2];
    Et0 = dbg ? A.dbg_E[0] : A.dE[p * 3 + 0];
    Et1 = dbg ? A.dbg_E[1] : A.dE[p * 3 + 1];
    Et2 = dbg ? A.dbg_E[2] : A.dE[p * 3 + 2];
    const int dead = dbg ? 0 : D.st[p].err;
    auto write_fail = [&](int code, int iters, double rn) {
      if (lane == 0) {
        A.O.status[p] = code;
        A.O.iters[p] = iters;
        A.O.res[p] = rn;
        for (int i = 0; i < 3; ++i) A.O.sigma[p * 3 + i] = qnan();
        for (int i = 0; i < 9; ++i) A.O.C[p * 9 + i] = qnan();
        if (A.O.pcount) A.O.pcount[p] = 0;
      }
    };
    if (dead) {  // a point whose trajectory already failed stays failed
      write_fail(dead, 0, qnan());
      if (lane == 0) {
        D.E_c[p * 3 + 0] = Et0;
        D.E_c[p * 3 + 1] = Et1;
        D.E_c[p * 3 + 2] = Et2;
      }
      p_next = grab();
      continue;
    }
    if constexpr (MONO) {
      mono_point(p, Et0, Et1, Et2);
      p_next = grab();
      continue;
    }
    // warm start α = α_committed, E = E_prev + (E_k - E_prev) * 1 (rve.hpp:465-472)
    for (int a = lane; a < NP; a += 32) {
      const double ac = dbg ? ((a < n) ? A.dbg_alpha[a] : 0.0) : D.alpha_c[p * NP + a];
      sAev[a] = ac;
      sAl[a] = ac;
    }
    double E0 = lerp_rn(Ep0, Et0, 1.0), E1 = lerp_rn(Ep1, Et1, 1.0), E2 = lerp_rn(Ep2, Et2, 1.0);
    __syncwarp();
    int mode = 0, it = 0, ls = 0, iters = 0, bis = 0;
    double a = 1.0, rn_it = 0.0, best_rn = 0.0, best_a = 1.0, ref = 0.0, done = 0.0, frac = 1.0;
    int err = 0;
    while (true) {
      // park the Newton state in shared memory across the pass: the registers are
      // free for the chunk loop (each lane stores its own, warp-uniform copy; no
      // read-modify-write of shared state, so convergence does not matter)
      W_->E0 = E0, W_->E1 = E1, W_->E2 = E2;
      W_->mode = mode, W_->it = it, W_->ls = ls, W_->iters = iters, W_->bis = bis, W_->err = err;
      W_->a = a, W_->rn_it = rn_it, W_->best_rn = best_rn, W_->best_a = best_a, W_->ref = ref;
      W_->done = done, W_->frac = frac;
      assembly_pass(p, E0, E1, E2, dbg ? -1 : p);
      {  // volatile reloads: the compiler may not forward the parked values in registers
        const volatile WarpSt* V = W_;
        E0 = V->E0, E1 = V->E1, E2 = V->E2;
        mode = V->mode, it = V->it, ls = V->ls, iters = V->iters, bis = V->bis, err = V->err;
        a = V->a, rn_it = V->rn_it, best_rn = V->best_rn, best_a = V->best_a, ref = V->ref;
        done = V->done, frac = V->frac;
      }
      if (dbg) {
        dump();
        break;
      }
      if constexpr (GEN) {
        // a failed return map throws out of micro_newton and run_trajectory
        // (materials.hpp:244, :287): the point's trajectory ends here
        if (W_->merr) {
          err = kMaterial;
          write_fail(err, iters, qnan());
          break;
        }
      }
      const double rl = (lane < n) ? sV[lane] : 0.0;
      const double rn = sqrt(warp_sum(rl * rl));
      const double srn = sqrt(s0 * s0 + s1 * s1 + s2 * s2);
      // 0: assemble again, 1: final commit, 2: sub-step commit, 3: failed
      int action = 0;
      for (int pass = 0; pass < 2; ++pass) {
        if (mode == 0) {  // Newton iterate (micro_newton, rve.hpp:300-342)
          if (it == 0) ref = fmax(fmax(rn, srn), 1e-30);
          const bool conv = rn <= cfg.tol * ref;
          const double target = fmin(1.0, done + frac);
          const bool final_commit = conv && target >= 1.0 - 1e-12;
          const bool newton_step = !conv && it != cfg.max_iter;
          // the one factorization site: Newton step or final condensation
          if ((final_commit || newton_step) && !factor()) {
            if (conv) iters += it;
            err = kSolver;
            write_fail(err, iters, rn);
            action = 3;
            break;
          }
          if (conv) {
            iters += it;
            if (final_commit) {
              // condensation: X = L^-1 K_aE, C = (C_EE - X^T X) / V
              double x0 = (lane < n) ? sKaE[lane * 3 + 0] : 0.0;
              double x1 = (lane < n) ? sKaE[lane * 3 + 1] : 0.0;
              double x2 = (lane < n) ? sKaE[lane * 3 + 2] : 0.0;
              for (int j = 0; j < n; ++j) {
                const double inv = sInv[j];
                const double y0 = __shfl_sync(0xffffffffu, x0, j) * inv;
                const double y1 = __shfl_sync(0xffffffffu, x1, j) * inv;
                const double y2 = __shfl_sync(0xffffffffu, x2, j) * inv;
                if (lane == j) {
                  x0 = y0;
                  x1 = y1;
                  x2 = y2;
                } else if (lane > j && lane < n) {
                  const double l = sK[tri_(lane) + j];
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
                A.O.iters[p] = iters;
                A.O.status[p] = 0;
              }
              action = 1;
            } else {
              action = 2;
              done = target;
            }
            break;
          }
          if (it == cfg.max_iter) {  // not converged: bisect the load step (rve.hpp:473-478)
            iters += cfg.max_iter;
            if (++bis > cfg.max_bis) {
              err = kSolver;
              write_fail(err, iters, rn);
              action = 3;
              break;
            }
            frac *= 0.5;
            const double nt = fmin(1.0, done + frac);
            E0 = lerp_rn(Ep0, Et0, nt);
            E1 = lerp_rn(Ep1, Et1, nt);
            E2 = lerp_rn(Ep2, Et2, nt);
            for (int b = lane; b < NP; b += 32) {
              const double ac = D.alpha_c[p * NP + b];
              sAl[b] = ac;
              sAev[b] = ac;
            }
            it = 0;
            mode = 0;
            action = 0;
            break;
          }
          // Newton step: K Δα = -r (factor computed above)
          const double du = warp_chol_solve(sK, sInv, n, lane, -rl);
          if (lane < NP) {
            sDA[lane] = (lane < n) ? du : 0.0;
            sAev[lane] = (lane < n) ? axpy_rn(sAl[lane], 1.0, du) : 0.0;
          }
          rn_it = rn;
          a = 1.0;
          ls = 0;
          best_rn = __longlong_as_double(0x7ff0000000000000ll);
          best_a = 1.0;
          mode = 1;
          action = 0;
          break;
        } else {  // backtracking line search on the residual norm (rve.hpp:327-341)
          const double trial = rn;
          if (trial < best_rn) {
            best_rn = trial;
            best_a = a;
          }
          const bool armijo = trial <= (1.0 - 1e-4 * a) * rn_it;
          if (armijo || ls == 7) {
            it += 1;
            mode = 0;
            if (best_a == a) {  // the accepted iterate is this evaluation point
              if (lane < NP) sAl[lane] = sAev[lane];
              __syncwarp();
              continue;  // reuse this assembly as the new iterate's
            }
            if (lane < NP) {
              const double nv = (lane < n) ? axpy_rn(sAl[lane], best_a, sDA[lane]) : 0.0;
              sAl[lane] = nv;
              sAev[lane] = nv;
            }
            action = 0;
            break;
          }
          ls += 1;
          a *= 0.5;
          if (lane < NP) sAev[lane] = (lane < n) ? axpy_rn(sAl[lane], a, sDA[lane]) : 0.0;
          action = 0;
          break;
        }
      }
      __syncwarp();
      if (action == 0) continue;
      if (action == 3) break;
      // the one commit site: final (the next point's first history chunks are
      // requested right away) or a converged sub-step
      const int pc = commit_point(p);
      if (action == 1) {
        if (lane == 0 && A.O.pcount) A.O.pcount[p] = pc;
        p_next = grab();
        if (p_next < D.P) {
          hload(hbase(p_next), 0, nh0, nh1, nh2, nh3, nh4);
          pf_p = p_next;
        }
        break;
      }
      // converged sub-step: the next one starts from the new committed state
      // (the chunk prefetched during the pass came from the old buffer)
      pf_p = -1;
      const double nt = fmin(1.0, done + frac);
      E0 = lerp_rn(Ep0, Et0, nt);
      E1 = lerp_rn(Ep1, Et1, nt);
      E2 = lerp_rn(Ep2, Et2, nt);
      if (lane < NP) sAl[lane] = sAev[lane];
      __syncwarp();
      it = 0;
      mode = 0;
    }
    if (dbg) break;
    if (lane == 0) {
      if (err) D.st[p].err = err;
      D.E_c[p * 3 + 0] = Et0;
      D.E_c[p * 3 + 1] = Et1;
      D.E_c[p * 3 + 2] = Et2;
    }
    if (p_next < 0) p_next = grab();
  }
  ring_drain(R, seq, lane);
#ifdef FE2_INC_PROF
  INC_T(5);
  if (lane == 0) {
    for (int k = 0; k < 6; ++k) atomicAdd(&g_inc_prof[k], prof[k]);
    __threadfence();
    if (atomicAdd(&g_inc_prof[6], 1ull) == static_cast<unsigned long long>(gridDim.x) * W - 1) {
      unsigned long long s_ = 0;
      for (int k = 0; k < 6; ++k) s_ += g_inc_prof[k];
      printf("FE2_INC_PROF NT=%d W=%d cycles%%: gemv %.1f material %.1f dmma %.1f pass-tail %.1f factor %.1f "
             "newton %.1f (total %llu warp-cycles)\n",
             NT, W, 100.0 * g_inc_prof[0] / s_, 100.0 * g_inc_prof[1] / s_, 100.0 * g_inc_prof[2] / s_,
             100.0 * g_inc_prof[3] / s_, 100.0 * g_inc_prof[4] / s_, 100.0 * g_inc_prof[5] / s_, s_);
      for (int k = 0; k < 7; ++k) g_inc_prof[k] = 0;
    }
  }
#endif
  if (A.cnt && lane == 0) {
    atomicAdd(&A.cnt->assemblies, static_cast<unsigned long long>(cnt_[0]));
    atomicAdd(&A.cnt->commits, static_cast<unsigned long long>(cnt_[1]));
    atomicAdd(&A.cnt->plastic_evals, static_cast<unsigned long long>(cnt_[2]));
    atomicAdd(&A.cnt->commit_plastic, static_cast<unsigned long long>(cnt_[3]));
  }
}

__global__ void k_material_batch(MatDev m, int64_t N, const double* eps, const double* st_in, double* sigma,
                                 double* C, double* st_out, uint8_t* plastic, int* err) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double s[5] = {0, 0, 0, 0, 0};
  if (st_in)
    for (int c = 0; c < 5; ++c) s[c] = st_in[i * 6 + c];
  bool ok = true;
  const MatOut o =
      update_material_any(m, s[0], s[1], s[2], s[3], s[4], eps[i * 3], eps[i * 3 + 1], eps[i * 3 + 2], ok);
  if (!ok && err) atomicExch(err, 1);
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

constexpr size_t kMaxDynSmem = 227 * 1024;

template <int NT, int W, bool RES, bool MONO = false, bool GEN = false>
void launch_inc_variant(const IncArgs& a, int num_sms, cudaStream_t s, size_t smem) {
  auto kern = k_increment<NT, W, RES, MONO, GEN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMaxDynSmem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = static_cast<int64_t>(num_sms) * per_sm;
  const int64_t need = (a.D.P + W - 1) / W;
  if (a.dbg) grid = 1;
  else if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<static_cast<unsigned>(grid), W * 32, smem, s>>>(a);
}

bool resident_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("FE2_NO_RESIDENT");
    return e && *e && *e != '0';
  }();
  return off;
}

template <int NT, bool GEN>
void launch_inc_nt(const IncArgs& a, int num_sms, cudaStream_t s) {
  constexpr int NP = 8 * NT;
  constexpr int WR = kwres_for(NT);
  const size_t res = IncLayout<NP, WR>::res_bytes(a.M.nchunks);
  if (res <= kMaxDynSmem && !resident_disabled())
    launch_inc_variant<NT, WR, true, false, GEN>(a, num_sms, s, res);
  else
    launch_inc_variant<NT, kw_for(NT), false, false, GEN>(a, num_sms, s, IncLayout<NP, kw_for(NT)>::bytes);
}

}  // namespace

size_t increment_smem(int NP) {
  switch (NP) {
    case 8: return IncLayout<8, kw_for(1)>::bytes;
    case 16: return IncLayout<16, kw_for(2)>::bytes;
    case 24: return IncLayout<24, kw_for(3)>::bytes;
    case 32: return IncLayout<32, kw_for(4)>::bytes;
    default: return 0;
  }
}

__global__ void k_mono_commit(PointsDev D, int NP, const double* __restrict__ mono) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= D.P || D.st[p].err) return;
  const double* rec = mono + p * mono_stride(NP);
  for (int a = 0; a < NP; ++a) {
    D.alpha_c[p * NP + a] = rec[5 * NP + a];
    D.bp[p * NP + a] -= rec[4 * NP + a];
  }
  for (int i = 0; i < 3; ++i) {
    D.E_c[p * 3 + i] = rec[6 * NP + i];
    D.sp[p * 4 + i] -= rec[6 * NP + 3 + i];
  }
  D.st[p].pad[0] ^= 1;
}

void launch_mono_commit(const PointsDev& D, int NP, const double* mono, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((D.P + 127) / 128);
  k_mono_commit<<<grid, 128, 0, s>>>(D, NP, mono);
}

// the monolithic iteration: G resident in shared memory when it fits (as launch_inc_nt), else the ring
template <int NT>
void launch_mono_nt(const IncArgs& a, int num_sms, cudaStream_t s) {
  constexpr int NP = 8 * NT;
  constexpr int WR = kwres_for(NT);
  const size_t res = IncLayout<NP, WR>::res_bytes(a.M.nchunks);
  if (res <= kMaxDynSmem && !resident_disabled())
    launch_inc_variant<NT, WR, true, true>(a, num_sms, s, res);
  else
    launch_inc_variant<NT, mono_kw(NT), false, true>(a, num_sms, s, IncLayout<NP, mono_kw(NT)>::bytes);
}

void launch_increment_mono(const IncArgs& a, int num_sms, cudaStream_t s) {
  switch (a.M.NP) {
    case 8: launch_mono_nt<1>(a, num_sms, s); break;
    case 16: launch_mono_nt<2>(a, num_sms, s); break;
    case 24: launch_mono_nt<3>(a, num_sms, s); break;
    case 32: launch_mono_nt<4>(a, num_sms, s); break;
    default: break;
  }
}

void launch_increment(const IncArgs& a, int num_sms, cudaStream_t s) {
  const bool gen = a.M.mat2.kind >= 2;  // power-law / creep history points
  switch (a.M.NP) {
    case 8: gen ? launch_inc_nt<1, true>(a, num_sms, s) : launch_inc_nt<1, false>(a, num_sms, s); break;
    case 16: gen ? launch_inc_nt<2, true>(a, num_sms, s) : launch_inc_nt<2, false>(a, num_sms, s); break;
    case 24: gen ? launch_inc_nt<3, true>(a, num_sms, s) : launch_inc_nt<3, false>(a, num_sms, s); break;
    case 32: gen ? launch_inc_nt<4, true>(a, num_sms, s) : launch_inc_nt<4, false>(a, num_sms, s); break;
    default: break;
  }
}

void launch_material_batch(const MatDev& m, int64_t N, const double* eps, const double* st_in, double* sigma,
                           double* C, double* st_out, uint8_t* plastic, int* err, cudaStream_t s) {
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((N + threads - 1) / threads);
  k_material_batch<<<grid, threads, 0, s>>>(m, N, eps, st_in, sigma, C, st_out, plastic, err);
}

}  // namespace fe2
