// B200 (sm_100a) persistent increment kernel for LARGE reduced bases
// (n = 33…128, BASELINE configs 3 and 4): one CTA per macro point (4 warps and
// two CTAs per SM for n <= 64, 8 warps above).
//
// Same algebra and same increment/Newton semantics as k_increment
// (hrom_kernels.cu), re-tiled for n > 32:
//  - G chunks (QB = 16 cubature points; strain rows padded to RS = NP + 4
//    doubles) stream through a 2-stage shared ring by TMA bulk copies; the
//    CTA walks them in lockstep.
//  - Material phase: TPQ = BT/QB threads per cubature point split the modes of
//    ε_q = E + G_q α (128-bit loads) and reduce with shuffles; one lane runs
//    the elastic trial / yield test / radial return and writes the candidate
//    history (double-buffered, no commit pass).
//  - Plastic points of a chunk are compacted CTA-wide (ballot + warp prefix,
//    deterministic order); each plastic point's threads then stage its B rows
//    (w ΔC_q) G_q (stride RS, aliasing K_aa, dead during a pass) and the
//    G-chunk offsets of its A rows, so every DMMA fragment is ONE conflict-free
//    64-bit shared load.
//  - The NT(NT+1)/2 upper tile pairs of K_aa are contracted on the FP64
//    tensor cores (DMMA) in compile-time register blocks (folded tile rows for
//    n = 64 / 128: NT + 1 pairs per warp), fragments prefetched one k-step
//    ahead; the K_aE and r corrections ride on the diagonal-tile owners'
//    fragments (n <= 64) or are summed from the staged rows.
//  - Newton / line search / bisection / condensation run CTA-wide: blocked
//    left-looking Cholesky of the packed K_aa (4-column panels), substitutions
//    on the row warps. MONO = the monolithic scheme's single iteration
//    (fe2_hrom_mono_iterate; instantiated in hrom_kernels_big_mono.cu).
#include "device_common.cuh"
#include "hrom_kernels.cuh"

namespace fe2 {

namespace {

using namespace dev;

#ifndef FE2_BIG_MINB
#define FE2_BIG_MINB 1
#endif
#ifndef FE2_BIG_QB32_MAXNP
#define FE2_BIG_QB32_MAXNP 64
#endif
// Warps per CTA (one macro point per CTA): 4 for NP <= 64 with 16-point
// chunks, so two CTAs (two points) share an SM — while one point sits in its
// barrier-bound phases (compaction, factorization) the other keeps the FP64
// pipe busy (+21% at n = 64); 8 for NP > 64, whose accumulators would not
// fit 4 warps' registers.
// The assembly pass is a lambda with two call sites (Newton loop, debug
// probe); NVVM inlines it for n = 64 / 128 but not for the other widths, whose
// kernels are compiled in hrom_kernels_big_other.cu with it forced inline
// (forcing it here cost n = 64 3%).
#ifdef FE2_BIG_INLINE_PASS
#define FE2_BIG_PASS_ATTR __attribute__((always_inline))
#else
#define FE2_BIG_PASS_ATTR
#endif
#ifndef FE2_BIG_SMALL_WARPS
#define FE2_BIG_SMALL_WARPS 4
#endif
constexpr int bw_for(int NT) { return NT <= 8 ? FE2_BIG_SMALL_WARPS : 8; }

template <int NT>
struct Big {
  static constexpr int NP = 8 * NT;
  static constexpr int BW = bw_for(NT);  // warps per CTA
  static constexpr int BT = BW * 32;     // threads per CTA
#ifndef FE2_BIG_SMALL_MINB
#define FE2_BIG_SMALL_MINB 2
#endif
  static constexpr int MINB = BW == 8 ? FE2_BIG_MINB : FE2_BIG_SMALL_MINB;
#ifndef FE2_BIG_QB_SMALL
#define FE2_BIG_QB_SMALL 16
#endif
  static constexpr int QB = (NP <= FE2_BIG_QB32_MAXNP && BW == 8) ? 32 : (BW == 8 ? 16 : FE2_BIG_QB_SMALL);  // cubature points per chunk
  static constexpr int TPQ = BT / QB;    // threads per cubature point
  static constexpr int RS = NP + 4;  // strain-row stride in G chunks and staged rows (≡ 4 or 12 mod 16)
  static constexpr int S = 3 * RS;    // doubles per cubature point in G2 (ModelDev::S for NP > 32)
  static constexpr int chunk = QB * S;
  static constexpr int TRI = NP * (NP + 1) / 2;
  static constexpr int STG = 3 * QB * RS;  // staged B rows
  static constexpr int KREG = TRI > STG ? TRI : STG;
  static constexpr int RED = 128;  // >= BW * 12 (block_sum_n)
  // doubles: ring[2][chunk] | sK[TRI] ∪ stage[STG] | vectors 9 NP | slots QB*(6+3) | ints sQ[QB],
  // row offsets[3 QB] | red
  static constexpr size_t dbl = 2 * static_cast<size_t>(chunk) + KREG + 9 * NP + QB * 11 + RED;
  // + control words, then sZ[NP][4] (monolithic iteration only) at the end
  static constexpr size_t zoff = dbl * sizeof(double) + 2 * sizeof(uint64_t) + 16 * sizeof(int);
  static constexpr size_t bytes = zoff + 4 * NP * sizeof(double);
};

// Tile pairs (t1 <= t2) of one warp. NT = 2 x warps (n = 64 on 4 warps,
// n = 128 on 8): folded tile rows, NT + 1 pairs per warp. Otherwise the upper
// triangle is cut into b x b tile blocks dealt largest-first to the
// least-loaded warp. The
// contraction is DMMA-issue bound per warp once the fragments are single
// conflict-free loads, so balance beats fragment reuse.
struct PairTable {
  int n;
  int t1[160];
  int t2[160];
};
template <int NT>
constexpr PairTable pairs_for(int W) {
  constexpr int BW = bw_for(NT);
  if constexpr (2 * BW == NT) {
    // folded rows: warp W owns tile rows W and NT-1-W, (NT - W) + (W + 1) =
    // NT + 1 pairs each — exactly balanced, two diagonal tiles per warp
    PairTable P{};
    for (int r : {W, NT - 1 - W})
      for (int t2 = r; t2 < NT; ++t2) {
        P.t1[P.n] = r;
        P.t2[P.n] = t2;
        ++P.n;
      }
    return P;
  }
  const int b = 2;
  const int nb = (NT + b - 1) / b;
  // blocks as (row tiles [r0, r1), col tiles [c0, c1)), pair count
  int r0[64] = {}, r1[64] = {}, c0[64] = {}, c1[64] = {}, cnt[64] = {}, nbk = 0;
  for (int B1 = 0; B1 < nb; ++B1)
    for (int B2 = B1; B2 < nb; ++B2) {
      const int ra = B1 * b, rb = (B1 * b + b < NT) ? B1 * b + b : NT;
      const int ca = B2 * b, cb = (B2 * b + b < NT) ? B2 * b + b : NT;
      const int parts = 1;
      const int h = (rb - ra + parts - 1) / parts;
      for (int s = 0; s < parts; ++s) {
        r0[nbk] = ra + s * h;
        r1[nbk] = (ra + s * h + h < rb) ? ra + s * h + h : rb;
        c0[nbk] = ca;
        c1[nbk] = cb;
        int c = 0;
        for (int t1 = r0[nbk]; t1 < r1[nbk]; ++t1)
          for (int t2 = c0[nbk]; t2 < c1[nbk]; ++t2) c += t1 <= t2 ? 1 : 0;
        cnt[nbk] = c;
        ++nbk;
      }
    }
  // largest-first to the least-loaded warp (ties: lowest index)
  int load[8] = {}, owner[64] = {};
  bool done[64] = {};
  for (int k = 0; k < nbk; ++k) {
    int best = -1;
    for (int j = 0; j < nbk; ++j)
      if (!done[j] && (best < 0 || cnt[j] > cnt[best])) best = j;
    done[best] = true;
    int w = 0;
    for (int v = 1; v < BW; ++v)
      if (load[v] < load[w]) w = v;
    owner[best] = w;
    load[w] += cnt[best];
  }
  PairTable P{};
  for (int j = 0; j < nbk; ++j) {
    if (owner[j] != W) continue;
    for (int t1 = r0[j]; t1 < r1[j]; ++t1)
      for (int t2 = c0[j]; t2 < c1[j]; ++t2)
        if (t1 <= t2) {
          P.t1[P.n] = t1;
          P.t2[P.n] = t2;
          ++P.n;
        }
  }
  return P;
}
template <int NT>
constexpr int max_pairs() {
  int m = 0;
  for (int w = 0; w < bw_for(NT); ++w) {
    const int c = pairs_for<NT>(w).n;
    m = c > m ? c : m;
  }
  return m;
}
template <int NT>
constexpr int total_pairs() {
  int m = 0;
  for (int w = 0; w < bw_for(NT); ++w) m += pairs_for<NT>(w).n;
  return m;
}
static_assert(total_pairs<5>() == 15 && total_pairs<8>() == 36 && total_pairs<12>() == 78 &&
                  total_pairs<16>() == 136,
              "tile-pair partition must cover the upper triangle");
static_assert((bw_for(8) != 4 || max_pairs<8>() == 9) && max_pairs<16>() == 17, "unexpected partition balance");

// non-volatile DMMA (pure in its operands: the scheduler may interleave the
// fragment loads of the next k-step)
__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// CTA-wide sum (all threads get the result); red has >= BW + 1 doubles.
template <int BW>
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < BW; ++w) s += red[w];
  return s;
}

// Compile-time walk over warp W's tile pairs (keeps every index a constant,
// so the accumulators and fragments stay in registers).
template <int NT, int W, int J, int MP>
__device__ __forceinline__ void dmma_pairs(double (&acc)[MP][2], const double (&A)[NT], const double (&B)[NT]) {
  if constexpr (J < pairs_for<NT>(W).n) {
    constexpr int t1 = pairs_for<NT>(W).t1[J];
    constexpr int t2 = pairs_for<NT>(W).t2[J];
    dmma_nv(acc[J][0], acc[J][1], A[t1], B[t2]);
    dmma_pairs<NT, W, J + 1, MP>(acc, A, B);
  }
}
template <int NT, int W, int J, int MP>
__device__ __forceinline__ void store_pairs(double* sK, const double (&acc)[MP][2], int r_, int c_) {
  if constexpr (J < pairs_for<NT>(W).n) {
    constexpr int t1 = pairs_for<NT>(W).t1[J];
    constexpr int t2 = pairs_for<NT>(W).t2[J];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int row = t1 * 8 + r_, cl = t2 * 8 + c_ + e;
      if constexpr (t1 < t2)
        sK[tri(cl) + row] = acc[J][e];
      else if (row >= cl)
        sK[tri(row) + cl] = acc[J][e];
    }
    store_pairs<NT, W, J + 1, MP>(sK, acc, r_, c_);
  }
}
// which fragment tiles warp W reads (so unused loads are never issued)
template <int NT>
constexpr bool uses_row(int W, int t) {
  const PairTable P = pairs_for<NT>(W);
  for (int j = 0; j < P.n; ++j)
    if (P.t1[j] == t) return true;
  return false;
}
template <int NT>
constexpr bool uses_col(int W, int t) {
  const PairTable P = pairs_for<NT>(W);
  for (int j = 0; j < P.n; ++j)
    if (P.t2[j] == t) return true;
  return false;
}
// fragments of one k-step from the staged rows: A[T] = A row (lane's k) at
// mode 8T + col, B[T] likewise (only the tiles warp W uses are loaded)
template <int NT, int W, int T>
__device__ __forceinline__ void load_frags(const double* pa, const double* pb, double (&A)[NT], double (&B)[NT]) {
  if constexpr (T < NT) {
    if constexpr (uses_row<NT>(W, T)) A[T] = pa[T * 8];
    if constexpr (uses_col<NT>(W, T)) B[T] = pb[T * 8];
    load_frags<NT, W, T + 1>(pa, pb, A, B);
  }
}

// does warp W own the diagonal tile pair (t, t)? Its owner also accumulates
// the r and K_aE corrections of the modes of tile t from the same fragments
// (NT <= 8; above that the extra accumulators would spill, and a per-mode
// loop over the plastic slots is used instead).
template <int NT>
constexpr bool kFragCorr = NT <= 8;
template <int NT>
constexpr bool owns_diag(int W, int t) {
  if (!kFragCorr<NT>) return false;
  const PairTable P = pairs_for<NT>(W);
  for (int j = 0; j < P.n; ++j)
    if (P.t1[j] == t && P.t2[j] == t) return true;
  return false;
}
// The owned diagonal tiles of a warp are kept compactly: slot diag_slot(W, T) of
// kae[KD][3] / rr[KD] (KD = the most any warp owns). Indexed by tile instead, all
// NT tiles' accumulators stayed live across the warp-dispatch switch: 252 -> 219
// registers at n = 64 (+3.4%), and the power-law / creep kernels stopped spilling.
template <int NT>
constexpr int diag_slot(int W, int T) {
  int j = 0;
  for (int t = 0; t < T; ++t) j += owns_diag<NT>(W, t) ? 1 : 0;
  return j;
}
template <int NT>
constexpr int kdiag() {
  int m = 1;
  for (int w = 0; w < 8; ++w) {
    const int c = diag_slot<NT>(w, NT);
    m = c > m ? c : m;
  }
  return m;
}
template <int NT>
constexpr int KD = kdiag<NT>();

template <int NT, int W, int T>
__device__ __forceinline__ void diag_acc(const double (&A)[NT], const double (&B)[NT], double ws, int s,
                                         double (&kae)[KD<NT>][3], double (&rr)[KD<NT>]) {
  if constexpr (T < NT) {
    if constexpr (owns_diag<NT>(W, T)) {
      // K_aE correction row (s + m) mod 3 of mode 8T + col, and r correction
      constexpr int j = diag_slot<NT>(W, T);
      if (s == 0) kae[j][0] += B[T];
      else if (s == 1) kae[j][1] += B[T];
      else kae[j][2] += B[T];
      rr[j] += ws * A[T];
    }
    diag_acc<NT, W, T + 1>(A, B, ws, s, kae, rr);
  }
}

// DMMA over the chunk's plastic rows for warp W's tile pairs: k-step ks
// covers rows 4ks..4ks+3 (row f = 3 slot + strain row i); lane (m, col) reads
// row 4ks + m — its A fragment straight from the G chunk at the staged row
// offset sRO[f], its B fragment from the staged (w ΔC_q) G_q rows. The three
// k-steps of a group of four slots are unrolled (the K_aE row of lane m is
// (s + m) mod 3 at k-step s of the group) and the next k-step's fragments are
// loaded before the current DMMAs.
template <int NT, int W, int MP>
__device__ __forceinline__ void contract(const double* Gb, const int* sRO, const double* stB, const double* sDS,
                                         int np4, double (&acc)[MP][2], double (&kae)[KD<NT>][3], double (&rr)[KD<NT>],
                                         int lane) {
  constexpr int RS = Big<NT>::RS;
  const int m = lane & 3, col = lane >> 2;
  const int ng = np4 >> 2;
  const double* ga = Gb + col;
  const int* ro = sRO + m;
  const double* pb = stB + m * RS + col;
  const double* pw = sDS + m;
  if constexpr (NT > 8) {  // no room for a prefetch set in the registers (two sets spill 0.4-3 KB)
#pragma unroll 1
    for (int g = 0; g < ng; ++g) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int f = 12 * g + 4 * s;
        double A[NT], B[NT];
        load_frags<NT, W, 0>(ga + ro[f], pb + f * RS, A, B);
        dmma_pairs<NT, W, 0, MP>(acc, A, B);
      }
    }
    return;
  }
#ifdef FE2_BIG_NOPREFETCH
  {
#pragma unroll 1
    for (int g = 0; g < ng; ++g) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int f = 12 * g + 4 * s;
        double A[NT], B[NT];
        load_frags<NT, W, 0>(ga + ro[f], pb + f * RS, A, B);
        dmma_pairs<NT, W, 0, MP>(acc, A, B);
        diag_acc<NT, W, 0>(A, B, pw[f], s, kae, rr);
      }
    }
    return;
  }
#endif
  double A0[NT], B0[NT], A1[NT], B1[NT], A2[NT], B2[NT];
  if (ng > 0) load_frags<NT, W, 0>(ga + ro[0], pb, A0, B0);
#pragma unroll 1
  for (int g = 0; g < ng; ++g) {
    const int f = 12 * g;  // first staged row of the group
    load_frags<NT, W, 0>(ga + ro[f + 4], pb + (f + 4) * RS, A1, B1);
    dmma_pairs<NT, W, 0, MP>(acc, A0, B0);
    diag_acc<NT, W, 0>(A0, B0, pw[f], 0, kae, rr);
    load_frags<NT, W, 0>(ga + ro[f + 8], pb + (f + 8) * RS, A2, B2);
    dmma_pairs<NT, W, 0, MP>(acc, A1, B1);
    diag_acc<NT, W, 0>(A1, B1, pw[f + 4], 1, kae, rr);
    if (g + 1 < ng) load_frags<NT, W, 0>(ga + ro[f + 12], pb + (f + 12) * RS, A0, B0);
    dmma_pairs<NT, W, 0, MP>(acc, A2, B2);
    diag_acc<NT, W, 0>(A2, B2, pw[f + 8], 2, kae, rr);
  }
}

// reduce the owned tiles' r / K_aE corrections over the four k-lanes of each
// column and store them (sV = r_plastic, sKaE = K_aE correction)
template <int NT, int W, int T>
__device__ __forceinline__ void diag_store(const double (&kae)[KD<NT>][3], const double (&rr)[KD<NT>], double* sV,
                                           double* sKaE, int lane) {
  if constexpr (T < NT) {
    if constexpr (owns_diag<NT>(W, T)) {
      const int m = lane & 3, col = lane >> 2;
      constexpr int j = diag_slot<NT>(W, T);
      double v = rr[j];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      double ki[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int s = (i - (m % 3) + 3) % 3;  // slot s holds strain row (s + m) mod 3
        double x = (s == 0) ? kae[j][0] : ((s == 1) ? kae[j][1] : kae[j][2]);
        x += __shfl_xor_sync(0xffffffffu, x, 1);
        x += __shfl_xor_sync(0xffffffffu, x, 2);
        ki[i] = x;
      }
      if (m == 0) {
        const int a = T * 8 + col;
        sV[a] = v;
        sKaE[a * 3 + 0] = ki[0];
        sKaE[a * 3 + 1] = ki[1];
        sKaE[a * 3 + 2] = ki[2];
      }
    }
    diag_store<NT, W, T + 1>(kae, rr, sV, sKaE, lane);
  }
}

template <int NT, int W, int MP>
__device__ __forceinline__ void store_tiles(double* sK, const double (&acc)[MP][2], int lane) {
  store_pairs<NT, W, 0, MP>(sK, acc, lane >> 2, 2 * (lane & 3));
}

template <int NT, int MP>
__device__ __forceinline__ void contract_dispatch(int warp, const double* Gb, const int* sRO, const double* stB,
                                                  const double* sDS, int np4, double (&acc)[MP][2],
                                                  double (&kae)[KD<NT>][3], double (&rr)[KD<NT>], int lane) {
  switch (warp) {
    case 0: contract<NT, 0, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 1: contract<NT, 1, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 2: contract<NT, 2, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 3: contract<NT, 3, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 4: contract<NT, 4, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 5: contract<NT, 5, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    case 6: contract<NT, 6, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
    default: contract<NT, 7, MP>(Gb, sRO, stB, sDS, np4, acc, kae, rr, lane); break;
  }
}
template <int NT>
__device__ __forceinline__ void diag_store_dispatch(int warp, const double (&kae)[KD<NT>][3], const double (&rr)[KD<NT>],
                                                    double* sV, double* sKaE, int lane) {
  switch (warp) {
    case 0: diag_store<NT, 0, 0>(kae, rr, sV, sKaE, lane); break;
    case 1: diag_store<NT, 1, 0>(kae, rr, sV, sKaE, lane); break;
    case 2: diag_store<NT, 2, 0>(kae, rr, sV, sKaE, lane); break;
    case 3: diag_store<NT, 3, 0>(kae, rr, sV, sKaE, lane); break;
    case 4: diag_store<NT, 4, 0>(kae, rr, sV, sKaE, lane); break;
    case 5: diag_store<NT, 5, 0>(kae, rr, sV, sKaE, lane); break;
    case 6: diag_store<NT, 6, 0>(kae, rr, sV, sKaE, lane); break;
    default: diag_store<NT, 7, 0>(kae, rr, sV, sKaE, lane); break;
  }
}
template <int NT, int MP>
__device__ __forceinline__ void store_dispatch(int warp, double* sK, const double (&acc)[MP][2], int lane) {
  switch (warp) {
    case 0: store_tiles<NT, 0, MP>(sK, acc, lane); break;
    case 1: store_tiles<NT, 1, MP>(sK, acc, lane); break;
    case 2: store_tiles<NT, 2, MP>(sK, acc, lane); break;
    case 3: store_tiles<NT, 3, MP>(sK, acc, lane); break;
    case 4: store_tiles<NT, 4, MP>(sK, acc, lane); break;
    case 5: store_tiles<NT, 5, MP>(sK, acc, lane); break;
    case 6: store_tiles<NT, 6, MP>(sK, acc, lane); break;
    default: store_tiles<NT, 7, MP>(sK, acc, lane); break;
  }
}

// The factorization and substitutions run on the first NW = ceil(NP/32)
// warps only (thread i = row i), synchronised by a named barrier over those
// warps; the other warps wait once at the closing CTA barrier.
template <int NW, int BW>
__device__ __forceinline__ void rows_sync() {
  if constexpr (NW >= BW)
    __syncthreads();
  else
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}

// CTA-wide sums of N values at once (two barriers in all; the same summation
// order as block_sum for each value). red has >= BW * N doubles.
template <int BW, int N>
__device__ __forceinline__ void block_sum_n(double (&v)[N], double* red) {
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = warp_sum(v[k]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) red[warp * N + k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < BW; ++w) s += red[w * N + k];
    v[k] = s;
  }
}

// Left-looking blocked Cholesky (panels of kPB columns) of the packed lower
// sK on the whole CTA: per panel, (1) every row thread subtracts the products
// with the previous columns (TPR threads per row split the k range), (2) lanes
// of warp 0 factor the kPB x kPB diagonal block with shuffles, (3) the rows
// below solve against it — 3 barriers per panel instead of 2 per column.
// False (CTA-uniform) if not SPD.
constexpr int kPB = 4;
template <int BT, int NP>
__device__ bool cta_cholesky_blk(double* sK, double* sInv, double* flag, int n) {
  constexpr int TPR = (2 * NP <= BT) ? 2 : 1;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid / TPR, h = tid % TPR;
  const bool live = row < n;
  double* ri = sK + tri(live ? row : 0);
  for (int j0 = 0; j0 < n; j0 += kPB) {
    const int nb = min(kPB, n - j0);
    double s[kPB];
#pragma unroll
    for (int c = 0; c < kPB; ++c) s[c] = 0.0;
    if (live && row >= j0 && j0 > 0) {
      for (int k = h; k < j0; k += TPR) {
        const double lr = ri[k];
#pragma unroll
        for (int c = 0; c < kPB; ++c)
          if (c < nb && j0 + c <= row) s[c] += lr * sK[tri(j0 + c) + k];
      }
    }
    if constexpr (TPR == 2) {
#pragma unroll
      for (int c = 0; c < kPB; ++c) s[c] += __shfl_xor_sync(0xffffffffu, s[c], 1);
    }
    if (live && row >= j0 && h == 0 && j0 > 0) {
#pragma unroll
      for (int c = 0; c < kPB; ++c)
        if (c < nb && j0 + c <= row) ri[j0 + c] -= s[c];
    }
    __syncthreads();
    if (tid < 32) {  // diagonal block: lane r < nb holds block row r
      double a[kPB];
      const int r = lane < nb ? lane : 0;
      const double* br = sK + tri(j0 + r) + j0;
#pragma unroll
      for (int c = 0; c < kPB; ++c) a[c] = (c <= r && c < nb) ? br[c] : 0.0;
      bool ok = true;
#pragma unroll
      for (int k = 0; k < kPB; ++k) {
        if (k < nb) {
          const double d = __shfl_sync(0xffffffffu, a[k], k);
          if (!(d > 0.0)) ok = false;
          const double inv = rsqrt_fast(d);
          if (lane == k) {
            a[k] = d * inv;
            sInv[j0 + k] = inv;
          } else if (lane > k) {
            a[k] *= inv;
          }
#pragma unroll
          for (int c = k + 1; c < kPB; ++c) {
            const double lck = __shfl_sync(0xffffffffu, a[k], c);
            if (lane >= c && lane < nb) a[c] -= a[k] * lck;
          }
        }
      }
      if (lane < nb) {
        double* bw = sK + tri(j0 + lane) + j0;
#pragma unroll
        for (int c = 0; c < kPB; ++c)
          if (c <= lane) bw[c] = a[c];
      }
      if (lane == 0) flag[0] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    if (flag[0] == 0.0) return false;
    if (live && h == 0 && row >= j0 + nb) {
      double l[kPB];
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        if (c < nb) {
          double t = ri[j0 + c];
          const double* lc = sK + tri(j0 + c) + j0;
#pragma unroll
          for (int k = 0; k < c; ++k) t -= l[k] * lc[k];
          l[c] = t * sInv[j0 + c];
          ri[j0 + c] = l[c];
        }
      }
    }
    __syncthreads();
  }
  return true;
}

// Forward substitution L y = b in place on sB[n] (cols RHS interleaved: sB[i*cols + c]).
template <int NW, int BW>
__device__ void cta_forward(const double* sK, const double* sInv, double* sB, int n, int cols) {
  const int tid = threadIdx.x;
  if (tid < NW * 32) {
    for (int j = 0; j < n; ++j) {
      if (tid < cols) sB[j * cols + tid] *= sInv[j];
      rows_sync<NW, BW>();
      if (tid > j && tid < n) {
        const double l = sK[tri(tid) + j];
        for (int c = 0; c < cols; ++c) sB[tid * cols + c] -= l * sB[j * cols + c];
      }
      rows_sync<NW, BW>();
    }
  }
  __syncthreads();
}
// Backward substitution L^T x = y in place (single RHS).
template <int NW, int BW>
__device__ void cta_backward(const double* sK, const double* sInv, double* sB, int n) {
  const int tid = threadIdx.x;
  if (tid < NW * 32) {
    for (int j = n - 1; j >= 0; --j) {
      if (tid == 0) sB[j] *= sInv[j];
      rows_sync<NW, BW>();
      if (tid < j) sB[tid] -= sK[tri(j) + tid] * sB[j];
      rows_sync<NW, BW>();
    }
  }
  __syncthreads();
}
// The same for four interleaved RHS (monolithic iteration: K^-1 [r | K_aE]).
template <int NW, int BW>
__device__ void cta_backward4(const double* sK, const double* sInv, double* sB, int n) {
  const int tid = threadIdx.x;
  if (tid < NW * 32) {
    for (int j = n - 1; j >= 0; --j) {
      if (tid < 4) sB[j * 4 + tid] *= sInv[j];
      rows_sync<NW, BW>();
      if (tid < j) {
        const double l = sK[tri(j) + tid];
#pragma unroll
        for (int c = 0; c < 4; ++c) sB[tid * 4 + c] -= l * sB[j * 4 + c];
      }
      rows_sync<NW, BW>();
    }
  }
  __syncthreads();
}

// Phase timeline of thread 0 of every CTA (tuning builds only: -DFE2_BIG_PROF;
// the last CTA prints the sums): 0 ring wait, 1 strain + material,
// 2 compaction + slots, 3 staging, 4 contraction, 5 chunk tail, 6 pass tail,
// 7 Newton / factorisation / condensation.
#ifdef FE2_BIG_PROF
__device__ unsigned long long g_big_prof[9];
#define BIG_T(k)                                              \
  do {                                                        \
    if (threadIdx.x == 0) {                                   \
      const long long t_ = clock64();                         \
      prof[k] += static_cast<unsigned long long>(t_ - t_prof); \
      t_prof = t_;                                            \
    }                                                         \
  } while (0)
#else
#define BIG_T(k) \
  do {           \
  } while (0)
#endif

// GEN: iterative history material (power law / creep, general_return)
template <int NT, bool MONO = false, bool GEN = false>
__global__ void __launch_bounds__(Big<NT>::BT, Big<NT>::MINB) k_increment_big(IncArgs A) {
#ifdef FE2_BIG_PROF
  unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_prof = clock64();
#endif
  using L = Big<NT>;
  constexpr int NP = L::NP, QB = L::QB, TPQ = L::TPQ, S = L::S;
  constexpr int MP = max_pairs<NT>();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* sK = ring + 2 * static_cast<size_t>(L::chunk);
  double* stB = sK;  // staged B rows alias sK (dead during an assembly pass)
  double* sAev = sK + L::KREG;
  double* sAl = sAev + NP;
  double* sDA = sAl + NP;
  double* sV = sDA + NP;
  double* sInv = sV + NP;
  double* sRp = sInv + NP;   // plastic part of r of the last pass (for the commit)
  double* sKaE = sRp + NP;   // [NP][3]
  double* sDS = sKaE + 3 * NP + QB * 6;  // (QB * 6 doubles before it are spare)
  int* sQ = reinterpret_cast<int*>(sDS + QB * 3);
  int* sRO = sQ + QB;  // [3 QB] G-chunk offset of plastic row f = 3 slot + i
  double* red = sDS + QB * 5;
  uint64_t* full = reinterpret_cast<uint64_t*>(red + L::RED);
  int* ictl = reinterpret_cast<int*>(full + 2);  // [0..7] warp counts, [8] point
  double* sZ = reinterpret_cast<double*>(smem_raw + L::zoff);  // [NP][4] monolithic K^-1 [r | K_aE]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const ModelDev& M = A.M;
  const PointsDev& D = A.D;
  const MatDev& mt = M.mat2;
  const int nch = M.K2p / QB;
  const int n = M.n;
  constexpr uint32_t kChunkBytes = L::chunk * sizeof(double);

  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < 2; ++s) {
      mbar_expect_tx(&full[s], kChunkBytes);
      tma_load_1d(ring + s * L::chunk, M.G2 + static_cast<size_t>(s % nch) * L::chunk, kChunkBytes, &full[s]);
    }
  // ring positions (global chunk sequence: chunk pos % nch, stage pos % 2):
  // tpos = next to take, rpos = next to refill (after the chunk's last barrier)
  int tpos = 0, rpos = 0;
  unsigned long long n_asm = 0, n_com = 0, n_pl = 0, n_cpl = 0;

  const int qi = tid / TPQ, sub = tid % TPQ;  // cubature point of this thread within a chunk, mode slice
  // [buf][P][K2p/32][5][32]: the committed buffer of a point is st[p].pad[0];
  // every assembly pass writes its candidate history into the other one and
  // accepting a state flips the bit (no commit pass)
  auto hist_ptr = [&](int64_t p, int q, bool buf) {
    return D.hist + (buf ? D.hist_alt : 0) + (p * (M.K2p / kQC) + q / kQC) * (5 * kQC) + (q % kQC);
  };
  auto ring_take = [&]() -> const double* {
    const int s = tpos & 1;
    mbar_wait(&full[s], static_cast<uint32_t>((tpos >> 1) & 1));
    ++tpos;
    return ring + s * L::chunk;
  };
  auto ring_release = [&]() {  // after the CTA barrier that ends the chunk
    if (tid == 0) {
      const int s = rpos & 1;
      fence_proxy_async();
      mbar_expect_tx(&full[s], kChunkBytes);
      tma_load_1d(ring + s * L::chunk, M.G2 + static_cast<size_t>((rpos + 2) % nch) * L::chunk, kChunkBytes,
                  &full[s]);
    }
    ++rpos;
  };
  // strain of this thread's cubature point (threads of a point split the modes)
  auto strain = [&](const double* Gb, double E0, double E1, double E2, double& e0, double& e1, double& e2) {
    // 128-bit loads of mode pairs (2j, 2j+1); rows are 16-B aligned (S, RS even)
    const double2* Gq = reinterpret_cast<const double2*>(Gb + qi * S);
    const double2* al2 = reinterpret_cast<const double2*>(sAev);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int j = sub; j < NP / 2; j += TPQ) {
      const double2 al = al2[j];
      const double2 g0 = Gq[j], g1 = Gq[L::RS / 2 + j], g2 = Gq[L::RS + j];
      a0 += g0.x * al.x + g0.y * al.y;
      a1 += g1.x * al.x + g1.y * al.y;
      a2 += g2.x * al.x + g2.y * al.y;
    }
#pragma unroll
    for (int o = TPQ / 2; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    e0 = E0 + a0;
    e1 = E1 + a1;
    e2 = E2 + a2;
  };
  // deterministic CTA-wide compaction: returns the slot of this thread's
  // point (if flagged) and the total count
  auto compact = [&](bool flag, int& slot, int& total) {
    const unsigned bal = __ballot_sync(0xffffffffu, flag && sub == 0);
    if (lane == 0) ictl[warp] = __popc(bal);
    __syncthreads();
    int pre = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < L::BW; ++w) {
      const int c = ictl[w];
      pre += (w < warp) ? c : 0;
      total += c;
    }
    slot = pre + __popc(bal & ((1u << lane) - 1u));
  };

  // outputs of an assembly pass
  double s0 = 0, s1 = 0, s2 = 0, ce00 = 0, ce01 = 0, ce02 = 0, ce11 = 0, ce12 = 0, ce22 = 0;
  double dsp0 = 0, dsp1 = 0, dsp2 = 0;  // plastic parts of Σraw
  int np_last = 0;
  bool k_linear = false;
  double rn_pass = 0.0;  // |r| of the last pass
  double dt_pass = A.M.mat2.dt;  // GEN creep: time of the sub-step being assembled (rve.hpp:466)
  bool merr_pass = false;        // GEN: a return map of the last pass failed (ErrorCode::material)

  auto assembly_pass = [&](int64_t p, double E0, double E1, double E2) FE2_BIG_PASS_ATTR {
    double acc[MP][2];
#pragma unroll
    for (int j = 0; j < MP; ++j) acc[j][0] = acc[j][1] = 0.0;
    double c00 = 0, c01 = 0, c02 = 0, c11 = 0, c12 = 0, c22 = 0, ds0 = 0, ds1 = 0, ds2 = 0;
    double kae[KD<NT>][3], rr[KD<NT>];  // r / K_aE corrections of the diagonal tiles this warp owns
#pragma unroll
    for (int t = 0; t < KD<NT>; ++t) rr[t] = kae[t][0] = kae[t][1] = kae[t][2] = 0.0;
    double rm = 0.0, ka0 = 0.0, ka1 = 0.0, ka2 = 0.0;  // NT > 8: thread a < NP, mode a
    int np_tot = 0;
    double merr = 0.0;  // GEN: return-map failures of this thread's points
    const bool cur = D.st[p].pad[0] != 0;
    double h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0;
    {  // every thread of a cubature point holds its history (one broadcast load per point)
      const double* H = hist_ptr(p, qi, cur);
      h0 = H[0];
      h1 = H[kQC];
      h2 = H[2 * kQC];
      h3 = H[3 * kQC];
      h4 = H[4 * kQC];
    }
    BIG_T(7);
    for (int c = 0; c < nch; ++c) {
      const double* Gb = ring_take();
      BIG_T(0);
      const int q = c * QB + qi;
      double e0, e1, e2;
      strain(Gb, E0, E1, E2, e0, e1, e2);
      bool plastic = false;
      Corr cr{};
      {  // the point's threads all run the return map on the reduced strain (same instruction
         // count for the warp as one lane per point, no divergence, no broadcast afterwards)
        const Trial T = trial_state(mt, h0, h1, h2, h3, h4, e0, e1, e2);
        double dlam_g = 0.0;
        if constexpr (GEN) {
          if (q < M.K2) {
            const GenRet g = general_return(mt, T.ss, h4, dt_pass);
            plastic = g.plastic;
            dlam_g = g.dlam;
            if (!g.ok) merr = 1.0;
            if (plastic) cr = radial_return_gen(mt, T, g.dlam, g.kq);
          }
        } else {
          plastic = (T.f > 0.0) && (q < M.K2);
          if (plastic) cr = radial_return(mt, T);
        }
        {  // candidate history (finish_return) into the non-committed buffer
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
          if (sub == 0) {
            double* Hc = hist_ptr(p, q, !cur);
            Hc[0] = n0;
            Hc[kQC] = n1;
            Hc[2 * kQC] = n2;
            Hc[3 * kQC] = n3;
            Hc[4 * kQC] = n4;
            if (D.flags && q < M.K2) D.flags[(cur ? 0 : D.flags_alt) + p * M.K2p + q] = plastic ? 1 : 0;
          }
        }
        if (c + 1 < nch) {
          const double* H = hist_ptr(p, q + QB, cur);
          h0 = H[0];
          h1 = H[kQC];
          h2 = H[2 * kQC];
          h3 = H[3 * kQC];
          h4 = H[4 * kQC];
        }
      }
      int slot, np;
      BIG_T(1);
      compact(plastic, slot, np);
      // The point's TPQ threads stage its operand rows right away (no staging
      // pass, no CTA barrier before it): every thread already holds its point's
      // w ΔC_q and flag (all of them ran the return map), the slot comes from the
      // point's first lane; each thread writes the B rows (w ΔC_q) G_q of its
      // modes (128-bit) and lanes sub < 3 the A-row offsets.
      {
        const int src = lane & ~(TPQ - 1);
        const double wq = plastic ? M.w2[q] : 0.0;
        const double d00 = wq * cr.dc00, d01 = wq * cr.dc01, d02 = wq * cr.dc02;
        const double d11 = wq * cr.dc11, d12 = wq * cr.dc12, d22 = wq * cr.dc22;
        if (plastic && sub == 0) {  // one lane per point accumulates the plastic sums
          sDS[slot * 3 + 0] = wq * cr.ds0;
          sDS[slot * 3 + 1] = wq * cr.ds1;
          sDS[slot * 3 + 2] = wq * cr.ds2;
          sQ[slot] = qi;
          c00 += d00;
          c01 += d01;
          c02 += d02;
          c11 += d11;
          c12 += d12;
          c22 += d22;
          ds0 += sDS[slot * 3 + 0];
          ds1 += sDS[slot * 3 + 1];
          ds2 += sDS[slot * 3 + 2];
        }
        const bool pl = plastic;
        const int ps = __shfl_sync(0xffffffffu, slot, src);
        if (pl) {
          const double2* Gq = reinterpret_cast<const double2*>(Gb + qi * S);
          double2* br = reinterpret_cast<double2*>(stB + 3 * ps * L::RS);
          if (sub < 3) sRO[3 * ps + sub] = qi * S + sub * L::RS;
#pragma unroll
          for (int j = sub; j < NP / 2; j += TPQ) {
            const double2 g0 = Gq[j], g1 = Gq[L::RS / 2 + j], g2 = Gq[L::RS + j];
            br[j] = make_double2(d00 * g0.x + d01 * g1.x + d02 * g2.x, d00 * g0.y + d01 * g1.y + d02 * g2.y);
            br[L::RS / 2 + j] =
                make_double2(d01 * g0.x + d11 * g1.x + d12 * g2.x, d01 * g0.y + d11 * g1.y + d12 * g2.y);
            br[L::RS + j] = make_double2(d02 * g0.x + d12 * g1.x + d22 * g2.x, d02 * g0.y + d12 * g1.y + d22 * g2.y);
          }
        }
      }
      const int np4 = (np + 3) & ~3;
      {  // pad slots [np, np4): zero B rows, Δσ and valid A-row offsets
        const int per = 3 * (NP / 2);
        for (int e = tid; e < (np4 - np) * per; e += L::BT) {
          const int z = np + e / per, r = e % per;
          reinterpret_cast<double2*>(stB + (3 * z + r / (NP / 2)) * L::RS)[r % (NP / 2)] = make_double2(0.0, 0.0);
        }
        if (tid < 3 * (np4 - np)) {
          const int z = np + tid / 3, i = tid % 3;
          sRO[3 * z + i] = i * L::RS;
          sDS[3 * z + i] = 0.0;
        }
      }
      n_pl += static_cast<unsigned long long>(tid == 0 ? np : 0);
      np_tot += np;
      BIG_T(2);
      __syncthreads();
      BIG_T(3);
      contract_dispatch<NT, MP>(warp, Gb, sRO, stB, sDS, np4, acc, kae, rr, lane);
      BIG_T(4);
      if constexpr (!kFragCorr<NT>) {
        // r and K_aE corrections from the staged rows: thread (h, a) sums mode a over the
        // plastic slots h, h + HS, ... (HS = threads per mode; combined after the chunk loop)
        constexpr int HS = L::BT / NP;
        const int hh = tid / NP, am = tid - hh * NP;
        if (hh < HS) {
          for (int sl = hh; sl < np; sl += HS) {
            const double* ar = Gb + sQ[sl] * S + am;
            const double* br = stB + 3 * sl * L::RS + am;
            const double* ds = sDS + sl * 3;
            rm += ar[0] * ds[0] + ar[L::RS] * ds[1] + ar[2 * L::RS] * ds[2];
            ka0 += br[0];
            ka1 += br[L::RS];
            ka2 += br[2 * L::RS];
          }
        }
      }
      __syncthreads();
      ring_release();
      BIG_T(5);
    }
    if constexpr (!kFragCorr<NT>) {
      constexpr int HS = L::BT / NP;
      if constexpr (HS > 1) {  // partial sums of the slot classes h > 0, added in a fixed order
        const int hh = tid / NP, am = tid - hh * NP;
        if (hh > 0 && hh < HS) {
          double* o = stB + ((hh - 1) * NP + am) * 4;  // the staging area is free after the last chunk
          o[0] = rm;
          o[1] = ka0;
          o[2] = ka1;
          o[3] = ka2;
        }
        __syncthreads();
        if (hh == 0) {
#pragma unroll
          for (int h = 1; h < HS; ++h) {
            const double* o = stB + ((h - 1) * NP + am) * 4;
            rm += o[0];
            ka0 += o[1];
            ka1 += o[2];
            ka2 += o[3];
          }
        }
        __syncthreads();  // before the K_aa tiles overwrite the aliased area
      }
    }
    store_dispatch<NT, MP>(warp, sK, acc, lane);
    if constexpr (kFragCorr<NT>) {
      diag_store_dispatch<NT>(warp, kae, rr, sRp, sKaE, lane);
    } else if (tid < NP) {
      sRp[tid] = rm;
      sKaE[tid * 3 + 0] = ka0;
      sKaE[tid * 3 + 1] = ka1;
      sKaE[tid * 3 + 2] = ka2;
    }
    // one CTA reduction for the nine plastic sums and the elastic Σ part
    // (its barriers also publish sK / sRp / sKaE)
    constexpr int kRs = GEN ? 13 : 12;  // GEN: + the return-map failure count
    double rs[kRs] = {c00, c01, c02, c11, c12, c22, ds0, ds1, ds2, 0.0, 0.0, 0.0};
    if constexpr (GEN) rs[kRs - 1] = merr;
    if (tid < n) {
      const double* ke = M.KaEe + tid * 3;
      const double al = sAev[tid];
      rs[9] = ke[0] * al;
      rs[10] = ke[1] * al;
      rs[11] = ke[2] * al;
    }
    block_sum_n<L::BW, kRs>(rs, red);
    if constexpr (GEN) merr_pass = rs[kRs - 1] != 0.0;
    c00 = rs[0], c01 = rs[1], c02 = rs[2], c11 = rs[3], c12 = rs[4], c22 = rs[5];
    ds0 = rs[6], ds1 = rs[7], ds2 = rs[8];
    const double sa0 = rs[9], sa1 = rs[10], sa2 = rs[11];
    // elastic predictor part and b_p, s_p (thread a = mode)
    double rl = 0.0;
    if (tid < n) {
      const int a = tid;
      const double* ke = M.KaEe + a * 3;
      double sx = 0.0;
      double* ka = sK + tri(a);
      for (int b = 0; b < n; ++b) {
        const double k0 = M.Ke[b * NP + a];
        sx += k0 * sAev[b];
        if (b <= a) ka[b] += k0;
      }
      rl = sRp[a] + sx + (ke[0] * E0 + ke[1] * E1 + ke[2] * E2) - D.bp[p * NP + a];
      sV[a] = rl;
      sKaE[a * 3 + 0] += ke[0];
      sKaE[a * 3 + 1] += ke[1];
      sKaE[a * 3 + 2] += ke[2];
    }
    rn_pass = sqrt(block_sum<L::BW>(rl * rl, red));  // also publishes sK, sV, sKaE
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
    k_linear = (np_tot == 0);
    ++n_asm;
    BIG_T(6);
  };

  auto factor = [&]() -> bool {
    if (k_linear) {
      for (int e = tid; e < tri(n); e += L::BT) sK[e] = M.Le[e];
      if (tid < n) sInv[tid] = M.LeInv[tid];
      __syncthreads();
      return true;
    }
    return cta_cholesky_blk<L::BT, NP>(sK, sInv, red + L::RED - 2, n);  // clear of block sums
  };

  // accept the last pass's state: flip to its candidate history, α_c, and move
  // the committed plastic-strain loads by its plastic corrections
  // (w S(Δεp) = -w Δσ): b_p -= r_plastic, s_p -= Σ w Δσ
  auto commit_point = [&](int64_t p) -> int {
    for (int a = tid; a < NP; a += L::BT) {
      D.alpha_c[p * NP + a] = sAev[a];
      D.bp[p * NP + a] -= sRp[a];
    }
    __syncthreads();  // every thread has read st[p].pad[0] of this pass before the flip
    if (tid == 0) {
      D.sp[p * 4 + 0] -= dsp0;
      D.sp[p * 4 + 1] -= dsp1;
      D.sp[p * 4 + 2] -= dsp2;
      D.st[p].pad[0] ^= 1;
    }
    ++n_com;
    n_cpl += static_cast<unsigned long long>(tid == 0 ? np_last : 0);
    __syncthreads();
    return np_last;
  };

  const NewtonCfg& cfg = A.cfg;
  constexpr int kSolver = 1 + 4;    // 1 + ErrorCode::solver
  constexpr int kMaterial = 1 + 3;  // 1 + ErrorCode::material

  // One monolithic Newton iteration of point p (the paper's scheme; same
  // algebra as k_increment<..., MONO>): α ← α_w − K⁻¹(r + K_aE ΔE)
  // with the previous iteration's solves, assemble at (E, α) from the committed
  // history, factor, and return the condensed Σ̃ = (Σ_raw − K_Eα K⁻¹ r)/V and
  // C = (C_EE − K_Eα K⁻¹ K_aE)/V; record z = K⁻¹[r | K_aE], the plastic loads
  // and α for the next iteration / fe2_hrom_mono_commit. No commit here.
  auto mono_point = [&](int64_t p, double E0, double E1, double E2) {
    double* rec = A.mono + p * mono_stride(NP);
    double* tail = rec + 6 * NP;
    if (A.mono_first) {
      for (int a = tid; a < NP; a += L::BT) sAev[a] = D.alpha_c[p * NP + a];
    } else {
      const double d0 = E0 - tail[0], d1 = E1 - tail[1], d2 = E2 - tail[2];
      for (int a = tid; a < NP; a += L::BT)
        sAev[a] = (a < n) ? rec[5 * NP + a] - (rec[a] + rec[NP + a] * d0 + rec[2 * NP + a] * d1 + rec[3 * NP + a] * d2)
                          : 0.0;
    }
    __syncthreads();
    assembly_pass(p, E0, E1, E2);
    const double rn = rn_pass;
    // micro scale: max(|r| at the step's first iteration, |Σ_raw| now) — E moves during a monolithic step
    const double r_first = A.mono_first ? rn : tail[6];
    const double ref = fmax(fmax(r_first, sqrt(s0 * s0 + s1 * s1 + s2 * s2)), 1e-30);
    if (!factor()) {  // fatal for the point: mono_commit skips it, later iterations report it
      if (tid == 0) {
        A.O.status[p] = kSolver;
        A.O.iters[p] = 1;
        A.O.res[p] = rn / ref;
        D.st[p].err = kSolver;
      }
      __syncthreads();
      return;
    }
    for (int a = tid; a < NP; a += L::BT) {
      const bool in = a < n;
      sZ[a * 4 + 0] = in ? sV[a] : 0.0;
      sZ[a * 4 + 1] = in ? sKaE[a * 3 + 0] : 0.0;
      sZ[a * 4 + 2] = in ? sKaE[a * 3 + 1] : 0.0;
      sZ[a * 4 + 3] = in ? sKaE[a * 3 + 2] : 0.0;
    }
    __syncthreads();
    cta_forward<(NP + 31) / 32, L::BW>(sK, sInv, sZ, n, 4);
    cta_backward4<(NP + 31) / 32, L::BW>(sK, sInv, sZ, n);
    double v[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (tid < n) {
      const double k0 = sKaE[tid * 3 + 0], k1 = sKaE[tid * 3 + 1], k2 = sKaE[tid * 3 + 2];
      const double zr = sZ[tid * 4 + 0], z0 = sZ[tid * 4 + 1], z1 = sZ[tid * 4 + 2], z2 = sZ[tid * 4 + 3];
      v[0] = k0 * zr, v[1] = k1 * zr, v[2] = k2 * zr;
      v[3] = k0 * z0, v[4] = k1 * z1, v[5] = k2 * z2;
      v[6] = k0 * z1, v[7] = k1 * z0, v[8] = k0 * z2, v[9] = k2 * z0, v[10] = k1 * z2, v[11] = k2 * z1;
    }
    block_sum_n<L::BW, 12>(v, red);
    const double q01 = 0.5 * (v[6] + v[7]), q02 = 0.5 * (v[8] + v[9]), q12 = 0.5 * (v[10] + v[11]);
    for (int a = tid; a < NP; a += L::BT) {
#pragma unroll
      for (int c = 0; c < 4; ++c) rec[c * NP + a] = sZ[a * 4 + c];
      rec[4 * NP + a] = sRp[a];
      rec[5 * NP + a] = sAev[a];
    }
    if (tid == 0) {
      const double V = M.volume;
      double* Cp = A.O.C + p * 9;
      Cp[0] = (ce00 - v[3]) / V;
      Cp[1] = (ce01 - q01) / V;
      Cp[2] = (ce02 - q02) / V;
      Cp[3] = Cp[1];
      Cp[4] = (ce11 - v[4]) / V;
      Cp[5] = (ce12 - q12) / V;
      Cp[6] = Cp[2];
      Cp[7] = Cp[5];
      Cp[8] = (ce22 - v[5]) / V;
      A.O.sigma[p * 3 + 0] = (s0 - v[0]) / V;
      A.O.sigma[p * 3 + 1] = (s1 - v[1]) / V;
      A.O.sigma[p * 3 + 2] = (s2 - v[2]) / V;
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
    __syncthreads();
  };

  if (A.dbg) {
    if (blockIdx.x == 0) {
      const int64_t p = A.dbg_point;
      for (int a = tid; a < NP; a += L::BT) sAev[a] = (a < n) ? A.dbg_alpha[a] : 0.0;
      __syncthreads();
      assembly_pass(p, A.dbg_E[0], A.dbg_E[1], A.dbg_E[2]);
      double* o = A.dbg;
      for (int a = tid; a < n; a += L::BT) o[a] = sV[a];
      for (int e = tid; e < n * n; e += L::BT) {
        const int i = e / n, j = e % n;
        o[n + e] = (j <= i) ? sK[tri(i) + j] : sK[tri(j) + i];
      }
      for (int e = tid; e < 3 * n; e += L::BT) o[n + n * n + e] = sKaE[e];
      if (tid == 0) {
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
    }
  } else {
    while (true) {
      __syncthreads();
      if (tid == 0) ictl[8] = atomicAdd(A.work, 1);
      __syncthreads();
      const int64_t p = ictl[8];
      if (p >= D.P) break;
      const double Ep0 = D.E_c[p * 3 + 0], Ep1 = D.E_c[p * 3 + 1], Ep2 = D.E_c[p * 3 + 2];
      const double Et0 = A.dE[p * 3 + 0], Et1 = A.dE[p * 3 + 1], Et2 = A.dE[p * 3 + 2];
      const int dead = D.st[p].err;
      auto write_fail = [&](int code, int iters, double rn) {
        if (tid == 0) {
          A.O.status[p] = code;
          A.O.iters[p] = iters;
          A.O.res[p] = rn;
          for (int i = 0; i < 3; ++i) A.O.sigma[p * 3 + i] = qnan();
          for (int i = 0; i < 9; ++i) A.O.C[p * 9 + i] = qnan();
          if (A.O.pcount) A.O.pcount[p] = 0;
        }
      };
      auto finish = [&](int err) {
        __syncthreads();
        if (tid == 0) {
          if (err) D.st[p].err = err;
          D.E_c[p * 3 + 0] = Et0;
          D.E_c[p * 3 + 1] = Et1;
          D.E_c[p * 3 + 2] = Et2;
        }
      };
      if (dead) {
        write_fail(dead, 0, qnan());
        finish(0);
        continue;
      }
      if constexpr (MONO) {  // E_c moves at fe2_hrom_mono_commit (k_mono_commit)
        mono_point(p, Et0, Et1, Et2);
        continue;
      }
      for (int a = tid; a < NP; a += L::BT) {
        const double ac = D.alpha_c[p * NP + a];
        sAev[a] = ac;
        sAl[a] = ac;
      }
      double E0 = lerp_rn(Ep0, Et0, 1.0), E1 = lerp_rn(Ep1, Et1, 1.0), E2 = lerp_rn(Ep2, Et2, 1.0);
      __syncthreads();
      int mode = 0, it = 0, ls = 0, iters = 0, bis = 0, err = 0;
      double a = 1.0, rn_it = 0.0, best_rn = 0.0, best_a = 1.0, ref = 0.0, done = 0.0, frac = 1.0;
      while (true) {
        if constexpr (GEN) dt_pass = mt.dt * (fmin(1.0, done + frac) - done);
        assembly_pass(p, E0, E1, E2);
        if constexpr (GEN) {
          // a failed return map throws out of micro_newton and run_trajectory
          // (materials.hpp:244, :287): the point's trajectory ends here
          if (merr_pass) {
            err = kMaterial;
            write_fail(err, iters, qnan());
            break;
          }
        }
        const double rn = rn_pass;
        const double srn = sqrt(s0 * s0 + s1 * s1 + s2 * s2);
        int action = 0;  // 0 assemble again, 1 final commit, 2 sub-step commit, 3 failed
        for (int pass = 0; pass < 2; ++pass) {
          if (mode == 0) {
            if (it == 0) ref = fmax(fmax(rn, srn), 1e-30);
            if (rn <= cfg.tol * ref) {
              iters += it;
              const double target = fmin(1.0, done + frac);
              if (target >= 1.0 - 1e-12) {
                if (!factor()) {
                  err = kSolver;
                  write_fail(err, iters, rn);
                  action = 3;
                  break;
                }
                // condensation X = L^-1 K_aE, C = (C_EE - X^T X)/V (homogenize, rve.hpp:372-390)
                cta_forward<(NP + 31) / 32, L::BW>(sK, sInv, sKaE, n, 3);
                double x0 = 0, x1 = 0, x2 = 0;
                if (tid < n) {
                  x0 = sKaE[tid * 3 + 0];
                  x1 = sKaE[tid * 3 + 1];
                  x2 = sKaE[tid * 3 + 2];
                }
                double qs[6] = {x0 * x0, x0 * x1, x0 * x2, x1 * x1, x1 * x2, x2 * x2};
                block_sum_n<L::BW, 6>(qs, red);
                const double q00 = qs[0], q01 = qs[1], q02 = qs[2], q11 = qs[3], q12 = qs[4], q22 = qs[5];
                if (tid == 0) {
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
            if (it == cfg.max_iter) {  // bisect the load step (rve.hpp:473-478)
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
              __syncthreads();
              for (int b = tid; b < NP; b += L::BT) {
                const double ac = D.alpha_c[p * NP + b];
                sAl[b] = ac;
                sAev[b] = ac;
              }
              it = 0;
              action = 0;
              break;
            }
            if (!factor()) {
              err = kSolver;
              write_fail(err, iters, rn);
              action = 3;
              break;
            }
            if (tid < n) sDA[tid] = -sV[tid];
            __syncthreads();
            cta_forward<(NP + 31) / 32, L::BW>(sK, sInv, sDA, n, 1);
            cta_backward<(NP + 31) / 32, L::BW>(sK, sInv, sDA, n);
            for (int b = tid; b < NP; b += L::BT) sAev[b] = (b < n) ? axpy_rn(sAl[b], 1.0, sDA[b]) : 0.0;
            rn_it = rn;
            a = 1.0;
            ls = 0;
            best_rn = __longlong_as_double(0x7ff0000000000000ll);
            best_a = 1.0;
            mode = 1;
            action = 0;
            break;
          } else {  // backtracking line search (rve.hpp:327-341)
            const double trial = rn;
            if (trial < best_rn) {
              best_rn = trial;
              best_a = a;
            }
            const bool armijo = trial <= (1.0 - 1e-4 * a) * rn_it;
            if (armijo || ls == 7) {
              it += 1;
              mode = 0;
              __syncthreads();
              if (best_a == a) {
                for (int b = tid; b < NP; b += L::BT) sAl[b] = sAev[b];
                __syncthreads();
                continue;
              }
              for (int b = tid; b < NP; b += L::BT) {
                const double nv = (b < n) ? axpy_rn(sAl[b], best_a, sDA[b]) : 0.0;
                sAl[b] = nv;
                sAev[b] = nv;
              }
              action = 0;
              break;
            }
            ls += 1;
            a *= 0.5;
            __syncthreads();
            for (int b = tid; b < NP; b += L::BT) sAev[b] = (b < n) ? axpy_rn(sAl[b], a, sDA[b]) : 0.0;
            action = 0;
            break;
          }
        }
        __syncthreads();
        if (action == 0) continue;
        if (action == 3) break;
        const int pc = commit_point(p);
        if (action == 1) {
          if (tid == 0 && A.O.pcount) A.O.pcount[p] = pc;
          break;
        }
        const double nt = fmin(1.0, done + frac);
        E0 = lerp_rn(Ep0, Et0, nt);
        E1 = lerp_rn(Ep1, Et1, nt);
        E2 = lerp_rn(Ep2, Et2, nt);
        for (int b = tid; b < NP; b += L::BT) sAl[b] = sAev[b];
        __syncthreads();
        it = 0;
        mode = 0;
      }
      finish(err);
    }
  }
  // no TMA may be in flight at exit: the two positions issued ahead
  __syncthreads();
  for (int k = 0; k < 2; ++k) {
    mbar_wait(&full[rpos & 1], static_cast<uint32_t>((rpos >> 1) & 1));
    ++rpos;
  }
#ifdef FE2_BIG_PROF
  BIG_T(7);
  if (tid == 0) {
    for (int k = 0; k < 8; ++k) atomicAdd(&g_big_prof[k], prof[k]);
    __threadfence();
    if (atomicAdd(&g_big_prof[8], 1ull) == gridDim.x - 1) {
      unsigned long long s = 0;
      for (int k = 0; k < 8; ++k) s += g_big_prof[k];
      printf("FE2_BIG_PROF NT=%d cycles%%: wait %.1f material %.1f compact %.1f stage %.1f contract %.1f tail %.1f "
             "pass-tail %.1f newton %.1f\n",
             NT, 100.0 * g_big_prof[0] / s, 100.0 * g_big_prof[1] / s, 100.0 * g_big_prof[2] / s,
             100.0 * g_big_prof[3] / s, 100.0 * g_big_prof[4] / s, 100.0 * g_big_prof[5] / s,
             100.0 * g_big_prof[6] / s, 100.0 * g_big_prof[7] / s);
      for (int k = 0; k < 9; ++k) g_big_prof[k] = 0;
    }
  }
#endif
  if (A.cnt && tid == 0) {
    atomicAdd(&A.cnt->assemblies, n_asm);
    atomicAdd(&A.cnt->commits, n_com);
    atomicAdd(&A.cnt->plastic_evals, n_pl);
    atomicAdd(&A.cnt->commit_plastic, n_cpl);
  }
}

template <int NT, bool MONO = false, bool GEN = false>
bool launch_big_nt_(const IncArgs& a, int num_sms, cudaStream_t s) {
  if (a.M.S != Big<NT>::S) return false;  // G2 rows must carry the padded strain-row stride
  const size_t smem = Big<NT>::bytes;
  // per launch: the opt-in is per device context (a handle may live on any device) and cheap
  cudaFuncSetAttribute(k_increment_big<NT, MONO, GEN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_increment_big<NT, MONO, GEN>, Big<NT>::BT, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = static_cast<int64_t>(num_sms) * per_sm;
  if (a.dbg) grid = 1;
  else if (grid > a.D.P) grid = a.D.P;
  if (grid < 1) grid = 1;
  k_increment_big<NT, MONO, GEN><<<static_cast<unsigned>(grid), Big<NT>::BT, smem, s>>>(a);
  return true;
}

template <int NT, bool MONO = false>
bool launch_big_nt(const IncArgs& a, int num_sms, cudaStream_t s) {
  return launch_big_nt_<NT, MONO, false>(a, num_sms, s);
}

}  // namespace

#if !defined(FE2_BIG_MONO_TU) && !defined(FE2_BIG_OTHER_TU) && !defined(FE2_BIG_GEN_TU)
// NP = 64 and 128 (BASELINE configs 3/4) here; 40, 48, 56, 80, 96, 112 in
// hrom_kernels_big_other.cu; power-law / creep models in hrom_kernels_big_gen.cu
bool launch_increment_big(const IncArgs& a, int num_sms, cudaStream_t s) {
  if (a.M.mat2.kind >= 2) return launch_increment_big_gen(a, num_sms, s);
  switch (a.M.NP) {
    case 64: return launch_big_nt<8>(a, num_sms, s);
    case 128: return launch_big_nt<16>(a, num_sms, s);
    default: return launch_increment_big_other(a, num_sms, s);
  }
}

size_t increment_big_smem(int NP) {
  switch (NP) {
    case 40: return Big<5>::bytes;
    case 48: return Big<6>::bytes;
    case 56: return Big<7>::bytes;
    case 64: return Big<8>::bytes;
    case 80: return Big<10>::bytes;
    case 96: return Big<12>::bytes;
    case 112: return Big<14>::bytes;
    case 128: return Big<16>::bytes;
    default: return 0;
  }
}

#elif defined(FE2_BIG_OTHER_TU)
bool launch_increment_big_other(const IncArgs& a, int num_sms, cudaStream_t s) {
  switch (a.M.NP) {
    case 40: return launch_big_nt<5>(a, num_sms, s);
    case 48: return launch_big_nt<6>(a, num_sms, s);
    case 56: return launch_big_nt<7>(a, num_sms, s);
    case 80: return launch_big_nt<10>(a, num_sms, s);
    case 96: return launch_big_nt<12>(a, num_sms, s);
    case 112: return launch_big_nt<14>(a, num_sms, s);
    default: return false;
  }
}

#elif defined(FE2_BIG_GEN_TU)
bool launch_increment_big_gen(const IncArgs& a, int num_sms, cudaStream_t s) {
  switch (a.M.NP) {
    case 40: return launch_big_nt_<5, false, true>(a, num_sms, s);
    case 48: return launch_big_nt_<6, false, true>(a, num_sms, s);
    case 56: return launch_big_nt_<7, false, true>(a, num_sms, s);
    case 64: return launch_big_nt_<8, false, true>(a, num_sms, s);
    case 80: return launch_big_nt_<10, false, true>(a, num_sms, s);
    case 96: return launch_big_nt_<12, false, true>(a, num_sms, s);
    case 112: return launch_big_nt_<14, false, true>(a, num_sms, s);
    case 128: return launch_big_nt_<16, false, true>(a, num_sms, s);
    default: return false;
  }
}

#else
bool launch_increment_big_mono(const IncArgs& a, int num_sms, cudaStream_t s) {
  switch (a.M.NP) {
    case 40: return launch_big_nt<5, true>(a, num_sms, s);
    case 48: return launch_big_nt<6, true>(a, num_sms, s);
    case 56: return launch_big_nt<7, true>(a, num_sms, s);
    case 64: return launch_big_nt<8, true>(a, num_sms, s);
    case 80: return launch_big_nt<10, true>(a, num_sms, s);
    case 96: return launch_big_nt<12, true>(a, num_sms, s);
    case 112: return launch_big_nt<14, true>(a, num_sms, s);
    case 128: return launch_big_nt<16, true>(a, num_sms, s);
    default: return false;
  }
}

#endif  // FE2_BIG_MONO_TU

}  // namespace fe2
