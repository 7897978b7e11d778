// B200 (sm_100a) finite-strain (Biot stress) hyper-ROM increment kernel —
// BASELINE config 2, parity unpinned (the CPU checker's fs_* functions are the
// checker; the reference has no finite-strain code).
//
// The kinematics are nonlinear at every cubature point (the rotation R of
// F = R U enters P = R T even where the material is elastic), so there is no
// elastic-predictor shortcut: every assembly contracts ALL K points,
//   r    = Σ_q G_q^T w P_q             K_aa = Σ_q G_q^T (w A_q) G_q
//   K_aF = Σ_q G_q^T w A_q             K_Fa = Σ_q (w A_q) G_q
//   C_FF = Σ_q w A_q                   P_raw = Σ_q w P_q
// with G_q the 4-row displacement-gradient operator (F_q = I + H + G_q α).
// The k-dimension of one cubature point is exactly 4 = the k of the FP64
// tensor-core MMA m8n8k4, so each point is one k-step: A-fragment = G_q^T
// (8-mode tile), B-fragment = (w A_q G_q) tile, computed in registers from
// G_q and the point's w A_q; an extra B tile [w A_q | w P_q | 0] yields K_aF
// and r from the same A-fragments. K_aa is not symmetric (plastic flow is not
// coaxial with the stretch), so Newton and the condensation use a warp LU
// with partial pivoting (fs_newton / fs_condense of the oracle).
//
// Structure as k_increment (hrom_kernels.cu): one persistent launch per
// increment, one warp per macro point from a work queue, G chunks through a
// TMA shared-memory ring shared by the CTA, history (J2 chunks only) through
// a per-warp TMA stream; every pass is a full assembly (a line-search trial
// that is accepted is reused as the next iterate's assembly, as the oracle's
// re-assembly at the same α would give the same numbers).
#include <cstdio>

#include "biot.cuh"
#include "device_common.cuh"
#include "hrom_kernels.cuh"

namespace fe2 {

namespace {

using namespace dev;

#ifndef FE2_FS_KW
#define FE2_FS_KW 8
#endif
#ifndef FE2_FS_STAGES
#define FE2_FS_STAGES 4
#endif
constexpr int kFW = FE2_FS_KW;  // warps per CTA
constexpr int kFHS = 2;         // per-warp history ring depth
constexpr int kSl = 21;         // slot stride: w A (16) | w P (4) | pad — conflict-free 64-bit lane stores

template <int NP>
struct FsLayout {
  // [G row 0..3 (RS each: NP + 4 pad) | w | 0]: RS ≡ 4 or 12 mod 16 doubles puts the
  // four k-lanes' A-fragment rows of a point on distinct banks, S ≡ 2 mod 16 keeps
  // the lanes' 128-bit row loads of the deformation step conflict-free
  static constexpr int RS = NP + 4;
  static constexpr int S = 4 * RS + 2;
  static constexpr int chunk = kQC * S;
  static constexpr int kSlots = kQC * kSl;
  static constexpr int LDK = NP + 1;                    // K_aa / LU row stride
  static constexpr int kKm = NP * LDK;
  static constexpr int kUnion = kSlots > kKm ? kSlots : kKm;
  static constexpr int kHist = kFHS * 5 * kQC;
  // α_eval, α, Δα, r, K_aF [NP][4], K_Fa [4][NP], C_FF|P_raw [20] (+4 pad), pivots [NP] (int), 1/U_jj [NP]
  static constexpr int WS = 4 * NP + 4 * NP + 4 * NP + 24 + NP / 2 + NP + kUnion + kHist;
  static constexpr long kBudget = 227L * 1024 - 512 - static_cast<long>(kFW) * WS * 8;
  static constexpr int kFit = static_cast<int>(kBudget / (static_cast<long>(chunk) * 8));
  static constexpr int ST = kFit < 2 ? 2 : (kFit > FE2_FS_STAGES ? FE2_FS_STAGES : kFit);
  static constexpr size_t ring_bytes = static_cast<size_t>(ST) * chunk * sizeof(double);
  static constexpr int kHbarOff = ST * 8;
  static constexpr int kCntOff = kHbarOff + kFW * kFHS * 8;
  static constexpr int kCtrlOff = ((kCntOff + ST * 4 + 7) / 8) * 8;
  static constexpr size_t bytes = ring_bytes + static_cast<size_t>(kFW) * WS * sizeof(double) + kCtrlOff + 8;
};

// Shared G-chunk ring (same protocol as hrom_kernels.cu: the last warp to
// release a stage refills it; ctrl = {working warps, issued positions}).
struct FsRing {
  double* buf;
  uint64_t* full;
  int* cnt;
  unsigned long long* ctrl;
  const double* G;
  int nch;
  int chunk;
  int stages;
  volatile int* tr;
};

__device__ __forceinline__ void fs_trace(const FsRing& R, int seq, int code) {
  if (R.tr && (threadIdx.x & 31) == 0) {
    R.tr[0] = seq;
    R.tr[1] = code;
    R.tr[2] = static_cast<int>(*reinterpret_cast<volatile unsigned long long*>(R.ctrl) & 0xffffffffull);
    R.tr[3] = static_cast<int>(*reinterpret_cast<volatile unsigned long long*>(R.ctrl) >> 32);
    __threadfence_system();
  }
}

__device__ __forceinline__ const double* fs_ring_wait(const FsRing& R, int seq) {
  const int s = seq % R.stages;
  fs_trace(R, seq, 1);
  mbar_wait(&R.full[s], static_cast<uint32_t>((seq / R.stages) & 1));
  fs_trace(R, seq, 2);
  return R.buf + static_cast<size_t>(s) * R.chunk;
}

__device__ __forceinline__ void fs_ring_release(const FsRing& R, int seq, int lane) {
  __syncwarp();
  if (lane == 0) {
    const int s = seq % R.stages;
    __threadfence_block();
    if (atomicAdd(&R.cnt[s], 1) == kFW - 1) {
      R.cnt[s] = 0;
      const int nxt = seq + R.stages;
      unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(R.ctrl);
      bool issue = false;
      while ((old >> 32) > 0) {
        const unsigned long long lo = old & 0xffffffffull;
        const unsigned long long want = static_cast<unsigned>(nxt + 1);
        const unsigned long long nw = (old & 0xffffffff00000000ull) | (lo > want ? lo : want);
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
        tma_load_1d(R.buf + static_cast<size_t>(s) * R.chunk, R.G + static_cast<size_t>(nxt % R.nch) * R.chunk,
                    bytes, &R.full[s]);
      }
    }
  }
  __syncwarp();
}

__device__ void fs_ring_drain(const FsRing& R, int seq, int lane) {
  if (lane == 0) atomicAdd(R.ctrl, 0xffffffff00000000ull);  // working -= 1
  __syncwarp();
  fs_trace(R, seq, 4);
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(R.ctrl, 0ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    const int issued = static_cast<int>(c & 0xffffffffull);
    const unsigned working = static_cast<unsigned>(c >> 32);
    if (seq < issued) {
      fs_ring_wait(R, seq);
      fs_ring_release(R, seq, lane);
      ++seq;
      continue;
    }
    if (working == 0) break;
    __nanosleep(64);
  }
  fs_trace(R, seq, 5);
}

// D += A B on the FP64 tensor pipe (m8n8k4). Not volatile: only the data
// dependences order it, so independent shared loads can be scheduled around it.
__device__ __forceinline__ void mma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// LU with partial pivoting of the n x n matrix in sA (row stride lda), lane i
// owning row i (n <= 32); multipliers stored below the diagonal, pivot rows
// in piv (first maximal |a_ij|, as the oracle's Lu::factor). False if singular.
__device__ bool warp_lu(double* sA, int lda, int* piv, double* inv_diag, int n, int lane) {
  for (int j = 0; j < n; ++j) {
    double v = (lane >= j && lane < n) ? fabs(sA[lane * lda + j]) : -1.0;
    int idx = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    if (!(v > 0.0)) return false;
    if (lane == 0) piv[j] = idx;
    if (idx != j)
      for (int k = lane; k < n; k += 32) {
        const double t = sA[j * lda + k];
        sA[j * lda + k] = sA[idx * lda + k];
        sA[idx * lda + k] = t;
      }
    __syncwarp();
    const double inv = 1.0 / sA[j * lda + j];
    if (lane == 0) inv_diag[j] = inv;
    if (lane > j && lane < n) {
      double* ri = sA + lane * lda;
      const double* rj = sA + j * lda;
      const double l = ri[j] * inv;
      ri[j] = l;
#pragma unroll 4
      for (int k = j + 1; k < n; ++k) ri[k] -= l * rj[k];
    }
    __syncwarp();
  }
  return true;
}

// Solve A x = b with the factors of warp_lu; lane i holds b_i in, x_i out.
__device__ double warp_lu_solve(const double* sA, int lda, const int* piv, const double* inv_diag, int n, int lane,
                                double b) {
  double y = b;
  for (int j = 0; j < n; ++j) {
    const int p = piv[j];
    if (p != j) {
      const double yj = __shfl_sync(0xffffffffu, y, j), yp = __shfl_sync(0xffffffffu, y, p);
      if (lane == j) y = yp;
      else if (lane == p) y = yj;
    }
  }
  for (int j = 0; j < n; ++j) {  // unit lower
    const double yj = __shfl_sync(0xffffffffu, y, j);
    if (lane > j && lane < n) y -= sA[lane * lda + j] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {
    double xj = 0.0;
    if (lane == j) y = y * inv_diag[j];
    xj = __shfl_sync(0xffffffffu, y, j);
    if (lane < j) y -= sA[lane * lda + j] * xj;
  }
  return lane < n ? y : 0.0;
}

template <int NT>
__global__ void __launch_bounds__(kFW * 32, 1) k_increment_fs(IncArgs A) {
  constexpr int NP = 8 * NT;
  using L = FsLayout<NP>;
  constexpr int S = L::S;
  constexpr int LDK = L::LDK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring_buf = reinterpret_cast<double*>(smem_raw);
  double* wbase = reinterpret_cast<double*>(smem_raw + L::ring_bytes) + static_cast<size_t>(warp) * L::WS;
  unsigned char* ctrl_base = smem_raw + L::ring_bytes + static_cast<size_t>(kFW) * L::WS * sizeof(double);
  uint64_t* full = reinterpret_cast<uint64_t*>(ctrl_base);
  uint64_t* hbar = reinterpret_cast<uint64_t*>(ctrl_base + L::kHbarOff) + warp * kFHS;
  int* cnt = reinterpret_cast<int*>(ctrl_base + L::kCntOff);
  unsigned long long* ctrl = reinterpret_cast<unsigned long long*>(ctrl_base + L::kCtrlOff);

  double* sAev = wbase;             // α at the evaluation point
  double* sAl = sAev + NP;          // α, current Newton iterate
  double* sDA = sAl + NP;           // Δα
  double* sV = sDA + NP;            // r
  double* sKaF = sV + NP;           // [NP][4]
  double* sKFa = sKaF + 4 * NP;     // [4][NP]
  double* sCP = sKFa + 4 * NP;      // C_FF (16) | P_raw (4)
  int* sPiv = reinterpret_cast<int*>(sCP + 24);
  double* sInvD = sCP + 24 + NP / 2;  // 1 / U_jj of the LU (pivots use the first NP/2 doubles)
  double* sU = sInvD + NP;
  double* sSlot = sU;               // [32][kSl] per-point w A | w P (assembly pass)
  double* sK = sU;                  // [NP][LDK] K_aa / LU factors (after the pass)
  double* hb = sU + L::kUnion;      // [kFHS][5][32] history stages

  const ModelDev& M = A.M;
  const PointsDev& D = A.D;
  const int nch = M.nchunks, nchh = M.nch_hist;
  const FsRing R{ring_buf, full, cnt, ctrl, M.G2, nch, L::chunk, L::ST,
                 A.trace ? A.trace + (static_cast<size_t>(blockIdx.x) * kFW + warp) * 4 : nullptr};

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::ST; ++s) {
      mbar_init(&full[s], 1);
      cnt[s] = 0;
    }
    *ctrl = (static_cast<unsigned long long>(kFW) << 32) | static_cast<unsigned long long>(L::ST);
  }
  if (lane == 0)
    for (int s = 0; s < kFHS; ++s) mbar_init(&hbar[s], 1);
  if (lane == 0) fence_mbar_init();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(L::chunk * sizeof(double));
    for (int s = 0; s < L::ST; ++s) {
      mbar_expect_tx(&full[s], bytes);
      tma_load_1d(ring_buf + static_cast<size_t>(s) * L::chunk, M.G2 + static_cast<size_t>(s % nch) * L::chunk,
                  bytes, &full[s]);
    }
  }

  const int m = lane & 3, col = lane >> 2;
  int seq = 0;
  unsigned long long n_asm = 0, n_com = 0, n_pl = 0, n_cpl = 0;
  int np_last = 0;  // plastic points of the last assembly pass
  const int n = M.n;
  const double volume = M.volume;
  auto valid = [&](int c) -> int {  // real cubature points of chunk c
    const int v = c < nchh ? M.K2 - c * kQC : M.K_el - (c - nchh) * kQC;
    return v < kQC ? v : kQC;
  };

  // ------------------------------------------------ per-warp history stream
  int h_iss = 0, h_con = 0;
  int64_t pf_p = -1;
  int pf_n = 0;
  const int h_first = nchh < kFHS ? nchh : kFHS;
  auto h_issue = [&](int64_t p, int c) {
    const int s = h_iss % kFHS;
    if (lane == 0) {
      const double* base = D.hist + (D.st[p].pad[0] ? D.hist_alt : 0);  // the committed buffer of p
      fence_proxy_async();
      mbar_expect_tx(&hbar[s], 5 * kQC * sizeof(double));
      tma_load_1d(hb + s * 5 * kQC, base + (p * nchh + c) * (5 * kQC), 5 * kQC * sizeof(double), &hbar[s]);
    }
    ++h_iss;
  };
  auto h_take = [&]() -> const double* {
    const int s = h_con % kFHS;
    mbar_wait(&hbar[s], static_cast<uint32_t>((h_con / kFHS) & 1));
    ++h_con;
    return hb + s * 5 * kQC;
  };
  auto h_begin = [&](int64_t p, bool after_write) {
    if (pf_p != p) {
      while (h_con < h_iss) h_take();
      __syncwarp();
      pf_n = 0;
    }
    if (after_write && pf_n == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    }
    for (int c = pf_n; c < h_first; ++c) h_issue(p, c);
    pf_p = -1;
    pf_n = 0;
  };
  auto h_prefetch = [&](int64_t p) {  // first chunks of point p's next pass, discarding stale ones
    while (h_con < h_iss) h_take();
    __syncwarp();
    for (int c = 0; c < h_first; ++c) h_issue(p, c);
    pf_p = p;
    pf_n = h_first;
  };
  auto h_next = [&](int64_t p, int c, int64_t pred) {
    const int nc = c + kFHS;
    if (nc < nchh) {
      h_issue(p, nc);
    } else if (pred >= 0 && nc - nchh < h_first && pf_n == nc - nchh && (pf_p == pred || pf_n == 0)) {
      h_issue(pred, nc - nchh);
      pf_p = pred;
      ++pf_n;
    }
  };
  // lane's history (εp, eq) of chunk c (zero for the elastic chunks)
  auto h_read = [&](int64_t p, int c, int64_t pred, double* h) {
    if (c < nchh) {
      const double* Hs = h_take();
#pragma unroll
      for (int i = 0; i < 5; ++i) h[i] = Hs[i * kQC + lane];
      __syncwarp();
      h_next(p, c, pred);
    } else {
#pragma unroll
      for (int i = 0; i < 5; ++i) h[i] = 0.0;
    }
  };
  // F_q = I + H + G_q α_eval for the lane's cubature point of the chunk in Gb
  auto deformation = [&](const double* Gb, double H0, double H1, double H2, double H3, double* F) {
    const double* Gq = Gb + lane * S;
    double a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
    const double2* av = reinterpret_cast<const double2*>(sAev);
#pragma unroll 4
    for (int k = 0; k < NP / 2; ++k) {
      const double2 al = av[k];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double2 x = reinterpret_cast<const double2*>(Gq + r * L::RS)[k];
        a[r] += x.x * al.x;
        b[r] += x.y * al.y;
      }
    }
    F[0] = (1.0 + H0) + (a[0] + b[0]);
    F[1] = (0.0 + H1) + (a[1] + b[1]);
    F[2] = (0.0 + H2) + (a[2] + b[2]);
    F[3] = (1.0 + H3) + (a[3] + b[3]);
  };

  // ---------------------------------------------------------------- passes
  auto assembly_pass = [&](int64_t p, double H0, double H1, double H2, double H3, int64_t pred, bool after_write) {
    double acc[NT][NT][2];
    double kx[NT][2];
    double kfa[NT];
    double c20 = 0.0;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      kx[i][0] = kx[i][1] = 0.0;
      kfa[i] = 0.0;
    }
    // candidate history of this state, written into the non-committed buffer;
    // accepting the state flips st[p].pad[0] (no separate commit pass)
    const bool cur = D.st[p].pad[0] != 0;
    double* hcand = D.hist + (cur ? 0 : D.hist_alt) + p * nchh * (5 * kQC) + lane;
    uint8_t* fcand = D.flags ? D.flags + (cur ? 0 : D.flags_alt) + p * M.K2p : nullptr;
    int np_tot = 0;
    h_begin(p, after_write);
    for (int c = 0; c < nch; ++c) {
      double h[5];
      h_read(p, c, pred, h);
      const double* Gb = fs_ring_wait(R, seq);
      const int nv = valid(c);
      double F[4];
      deformation(Gb, H0, H1, H2, H3, F);
      const double wq = Gb[lane * S + 4 * L::RS];
      BiotOut o;
      update_biot<true>(c < nchh ? M.mat2 : M.matE, h[0], h[1], h[2], h[3], h[4], F[0], F[1], F[2], F[3], o);
      const int npc = __popc(__ballot_sync(0xffffffffu, o.plastic && lane < nv));
      n_pl += static_cast<unsigned long long>(npc);
      np_tot += npc;
      if (c < nchh) {  // J2 chunk: candidate εp, eq (pads keep theirs)
        const bool real = lane < nv;
        double* Hd = hcand + c * (5 * kQC);
        Hd[0] = real ? o.ep0 : h[0];
        Hd[kQC] = real ? o.ep1 : h[1];
        Hd[2 * kQC] = real ? o.ep2 : h[2];
        Hd[3 * kQC] = real ? o.ep3 : h[3];
        Hd[4 * kQC] = real ? o.eq : h[4];
        if (fcand && real) fcand[c * kQC + lane] = o.plastic ? 1 : 0;
      }
      double* sl = sSlot + lane * kSl;
#pragma unroll
      for (int e = 0; e < 16; ++e) sl[e] = wq * o.A[e];
#pragma unroll
      for (int e = 0; e < 4; ++e) sl[16 + e] = wq * o.P[e];
      __syncwarp();
      if (lane < 20) {  // C_FF | P_raw partial sums of the chunk (fixed order, 4 chains)
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
        for (int q = 0; q < kQC; q += 4) {
          t0 += sSlot[q * kSl + lane];
          t1 += sSlot[(q + 1) * kSl + lane];
          t2 += sSlot[(q + 2) * kSl + lane];
          t3 += sSlot[(q + 3) * kSl + lane];
        }
        c20 += (t0 + t1) + (t2 + t3);
      }
      // one MMA k-step per cubature point: A = G_q^T tile, B = (w A_q G_q) tile.
      // Software-pipelined: the shared-memory operands of point q+1 are loaded
      // before the MMAs of point q issue, so their latency hides behind them.
      const int bidx = col < 4 ? m * 4 + col : 16 + m;
      const bool bon = col <= 4;
      double pg[NT][4], pa[NT], pw[4], pb;
      auto load_q = [&](int q) {
        const double* g = Gb + q * S + col;
        const double* sq = sSlot + q * kSl;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
#pragma unroll
          for (int r = 0; r < 4; ++r) pg[t][r] = g[r * L::RS + t * 8];
          pa[t] = g[m * L::RS + t * 8];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) pw[r] = sq[m * 4 + r];
        pb = bon ? sq[bidx] : 0.0;
      };
      load_q(0);
#pragma unroll 1
      for (int q = 0; q < nv; ++q) {
        double Af[NT], Bf[NT];
        const double bx = pb;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          Af[t] = pa[t];
          Bf[t] = pw[0] * pg[t][0] + pw[1] * pg[t][1] + pw[2] * pg[t][2] + pw[3] * pg[t][3];
          kfa[t] += Bf[t];
        }
        load_q(q + 1 < nv ? q + 1 : q);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
#pragma unroll
          for (int j = 0; j < NT; ++j) mma_f64(acc[i][j][0], acc[i][j][1], Af[i], Bf[j]);
          mma_f64(kx[i][0], kx[i][1], Af[i], bx);
        }
      }
      fs_ring_release(R, seq, lane);
      ++seq;
    }
    // K_aa (full), K_aF | r, K_Fa, C_FF | P_raw to shared memory (slots are dead now)
    {
      const int r_ = lane >> 2, c_ = 2 * (lane & 3);
#pragma unroll
      for (int i = 0; i < NT; ++i) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) sK[(i * 8 + r_) * LDK + j * 8 + c_ + e] = acc[i][j][e];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = c_ + e, row = i * 8 + r_;
          if (cc < 4) sKaF[row * 4 + cc] = kx[i][e];
          else if (cc == 4) sV[row] = kx[i][e];
        }
        sKFa[m * NP + i * 8 + col] = kfa[i];
      }
      if (lane < 20) sCP[lane] = c20;
    }
    np_last = np_tot;
    ++n_asm;
    __syncwarp();
  };

  // accept the state of the last assembly pass: its candidate history becomes
  // the committed one (flip), α_c, plastic count
  auto commit_point = [&](int64_t p) -> int {
    for (int a = lane; a < NP; a += 32) D.alpha_c[p * NP + a] = sAev[a];
    if (lane == 0) D.st[p].pad[0] ^= 1;
    ++n_com;
    n_cpl += static_cast<unsigned long long>(np_last);
    __syncwarp();
    return np_last;
  };

  const NewtonCfg& cfg = A.cfg;
  constexpr int kSolver = 1 + 4;  // 1 + ErrorCode::solver

  // One call site each for the assembly pass, the LU and the acceptance
  // (small instruction footprint); the debug dump runs through the same loop.
  const bool dbg = A.dbg != nullptr;  // assembly dump: r, K_aa, K_aF, K_Fa, C_FF, P_raw
  auto dump = [&]() {
    double* o = A.dbg;
    for (int a = lane; a < n; a += 32) o[a] = sV[a];
    for (int e = lane; e < n * n; e += 32) o[n + e] = sK[(e / n) * LDK + e % n];
    for (int e = lane; e < 4 * n; e += 32) o[n + n * n + e] = sKaF[(e / 4) * 4 + e % 4];
    for (int e = lane; e < 4 * n; e += 32) o[n + n * n + 4 * n + e] = sKFa[(e / n) * NP + e % n];
    if (lane < 20) o[n + n * n + 8 * n + lane] = sCP[lane];
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
    double Hp[4], Ht[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Hp[i] = dbg ? 0.0 : D.E_c[p * 4 + i];
      Ht[i] = dbg ? A.dbg_E[i] : A.dE[p * 4 + i];
    }
    const int dead = dbg ? 0 : D.st[p].err;
    auto write_fail = [&](int code, int iters, double rn) {
      if (lane == 0) {
        A.O.status[p] = code;
        A.O.iters[p] = iters;
        A.O.res[p] = rn;
        for (int i = 0; i < 4; ++i) A.O.sigma[p * 4 + i] = qnan();
        for (int i = 0; i < 16; ++i) A.O.C[p * 16 + i] = qnan();
        if (A.O.pcount) A.O.pcount[p] = 0;
      }
    };
    if (dead) {
      write_fail(dead, 0, qnan());
      if (lane == 0)
        for (int i = 0; i < 4; ++i) D.E_c[p * 4 + i] = Ht[i];
      p_next = grab();
      continue;
    }
    bool after_write = false;
    for (int a = lane; a < NP; a += 32) {
      const double ac = dbg ? ((a < n) ? A.dbg_alpha[a] : 0.0) : D.alpha_c[p * NP + a];
      sAev[a] = ac;
      sAl[a] = ac;
    }
    double H[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) H[i] = lerp_rn(Hp[i], Ht[i], 1.0);
    __syncwarp();
    int mode = 0, it = 0, ls = 0, iters = 0, bis = 0;
    double a = 1.0, rn_it = 0.0, best_rn = 0.0, best_a = 1.0, ref = 0.0, done = 0.0, frac = 1.0;
    int err = 0;
    while (true) {
      assembly_pass(p, H[0], H[1], H[2], H[3], dbg ? -1 : p, after_write);
      after_write = false;
      if (dbg) {
        dump();
        break;
      }
      const double rl = (lane < n) ? sV[lane] : 0.0;
      const double rn = sqrt(warp_sum(rl * rl));
      const double pr0 = sCP[16], pr1 = sCP[17], pr2 = sCP[18], pr3 = sCP[19];
      const double prn = sqrt(pr0 * pr0 + pr1 * pr1 + pr2 * pr2 + pr3 * pr3);
      int action = 0;  // 0: assemble again, 1: final commit, 2: sub-step commit, 3: failed
      for (int pass = 0; pass < 2; ++pass) {
        if (mode == 0) {  // Newton iterate (fs_newton)
          if (it == 0) ref = fmax(fmax(rn, prn), 1e-30);
          const bool conv = rn <= cfg.tol * ref;
          const double target = fmin(1.0, done + frac);
          const bool final_commit = conv && target >= 1.0 - 1e-12;
          const bool newton_step = !conv && it != cfg.max_iter;
          // the one LU site: Newton step or final condensation
          if ((final_commit || newton_step) && !warp_lu(sK, LDK, sPiv, sInvD, n, lane)) {
            if (conv) iters += it;
            err = kSolver;
            write_fail(err, iters, rn);
            action = 3;
            break;
          }
          if (conv) {
            iters += it;
            if (final_commit) {
              // condensation (fs_condense): Y = K^-1 (-K_aF), A_M = (C_FF + K_Fa Y) / V
              double y[4];
#pragma unroll
              for (int s = 0; s < 4; ++s)
                y[s] = warp_lu_solve(sK, LDK, sPiv, sInvD, n, lane, (lane < n) ? -sKaF[lane * 4 + s] : 0.0);
              double out16[16];
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const double kf = (lane < n) ? sKFa[r * NP + lane] : 0.0;
#pragma unroll
                for (int s = 0; s < 4; ++s) out16[r * 4 + s] = warp_sum(kf * y[s]);
              }
              if (lane == 0) {
                double* Cp = A.O.C + p * 16;
#pragma unroll
                for (int e = 0; e < 16; ++e) Cp[e] = (sCP[e] + out16[e]) / volume;
                A.O.sigma[p * 4 + 0] = pr0 / volume;
                A.O.sigma[p * 4 + 1] = pr1 / volume;
                A.O.sigma[p * 4 + 2] = pr2 / volume;
                A.O.sigma[p * 4 + 3] = pr3 / volume;
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
          if (it == cfg.max_iter) {  // not converged: bisect the load step
            iters += cfg.max_iter;
            if (++bis > cfg.max_bis) {
              err = kSolver;
              write_fail(err, iters, rn);
              action = 3;
              break;
            }
            frac *= 0.5;
            const double nt = fmin(1.0, done + frac);
#pragma unroll
            for (int i = 0; i < 4; ++i) H[i] = lerp_rn(Hp[i], Ht[i], nt);
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
          // Newton step: K Δα = -r (LU factors computed above)
          const double du = warp_lu_solve(sK, LDK, sPiv, sInvD, n, lane, -rl);
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
        } else {  // backtracking line search on the residual norm
          const double trial = rn;
          if (trial < best_rn) {
            best_rn = trial;
            best_a = a;
          }
          const bool armijo = trial <= (1.0 - 1e-4 * a) * rn_it;
          if (armijo || ls == 7) {
            it += 1;
            mode = 0;
            if (best_a == a) {  // the accepted iterate is this evaluation point: reuse its assembly
              if (lane < NP) sAl[lane] = sAev[lane];
              __syncwarp();
              continue;
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
      // the one commit site: final (the next point's history is requested right
      // away) or a converged sub-step (stale prefetches dropped; fence before
      // the async-proxy reads of the buffer just written by generic stores)
      const int pc = commit_point(p);
      if (action == 1) {
        if (lane == 0 && A.O.pcount) A.O.pcount[p] = pc;
        p_next = grab();
        if (p_next < D.P && nchh > 0) h_prefetch(p_next);
        break;
      }
      pf_p = -1;
      after_write = true;
      const double nt = fmin(1.0, done + frac);
#pragma unroll
      for (int i = 0; i < 4; ++i) H[i] = lerp_rn(Hp[i], Ht[i], nt);
      if (lane < NP) sAl[lane] = sAev[lane];
      __syncwarp();
      it = 0;
      mode = 0;
    }
    if (dbg) break;
    if (lane == 0) {
      if (err) D.st[p].err = err;
      for (int i = 0; i < 4; ++i) D.E_c[p * 4 + i] = Ht[i];
    }
    if (p_next < 0) p_next = grab();
  }
  while (h_con < h_iss) h_take();
  fs_ring_drain(R, seq, lane);
  if (A.cnt && lane == 0) {
    atomicAdd(&A.cnt->assemblies, n_asm);
    atomicAdd(&A.cnt->commits, n_com);
    atomicAdd(&A.cnt->plastic_evals, n_pl);
    atomicAdd(&A.cnt->commit_plastic, n_cpl);
  }
}

template <int NT>
void launch_fs_nt(const IncArgs& a, int num_sms, cudaStream_t s) {
  constexpr int NP = 8 * NT;
  const size_t smem = FsLayout<NP>::bytes;
  // per launch: the opt-in is per device context (a handle may live on any device) and cheap
  cudaFuncSetAttribute(k_increment_fs<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_increment_fs<NT>, kFW * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = static_cast<int64_t>(num_sms) * per_sm;
  const int64_t need = (a.D.P + kFW - 1) / kFW;
  if (a.dbg) grid = 1;
  else if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k_increment_fs<NT><<<static_cast<unsigned>(grid), kFW * 32, smem, s>>>(a);
}

}  // namespace

size_t increment_fs_smem(int NP) {
  switch (NP) {
    case 8: return FsLayout<8>::bytes;
    case 16: return FsLayout<16>::bytes;
    case 24: return FsLayout<24>::bytes;
    case 32: return FsLayout<32>::bytes;
    default: return 0;
  }
}

void launch_increment_fs(const IncArgs& a, int num_sms, cudaStream_t s) {
  switch (a.M.NP) {
    case 8: launch_fs_nt<1>(a, num_sms, s); break;
    case 16: launch_fs_nt<2>(a, num_sms, s); break;
    case 24: launch_fs_nt<3>(a, num_sms, s); break;
    case 32: launch_fs_nt<4>(a, num_sms, s); break;
    default: break;
  }
}

}  // namespace fe2
