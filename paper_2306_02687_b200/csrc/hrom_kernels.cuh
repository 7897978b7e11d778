// Device side of the B200 hyper-ROM engine: data layout and the launchers of
// the persistent per-increment kernel (assembly + Newton + condensation +
// commit, fused) and of the batched material update. See DESIGN.md for the
// layout and rooflines.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "material.cuh"

namespace fe2 {

constexpr int kQC = 32;  // cubature points per chunk (one per lane in the material phase)

// Per-point persistent record: only the trajectory-failure code survives
// between increments (run_trajectory throws and the point stops, rve.hpp:474).
struct PointState {
  int err;  // 0 alive, else 1 + ErrorCode
  int pad[3];
};

// Offset of strain row i (0..2) in a cubature point's G2 record for the
// warp-per-point kernel (NP <= 32). For NP ≡ 0 mod 16 the rows are padded to
// NP + 4 doubles so the three rows of a point start on distinct bank groups
// (rows NP apart would all collide: a 4-way conflict on the DMMA A-fragment
// loads; +26% at n = 16, +9-12% at n = 32); NP ≡ 8 mod 16 keeps rows NP
// apart (padding them to NP + 4 measured 5-10% slower at n = 8 and 24).
constexpr int g2_row_stride(int NP) { return NP % 16 == 0 ? NP + 4 : NP; }
constexpr int g2_row_offset(int NP, int i) { return i * g2_row_stride(NP); }

struct ModelDev {
  int n;        // modes
  int NP;       // modes padded to a multiple of 8 (DMMA tile)
  int S;        // doubles per cubature point in G2: g2_row_offset(NP, 2) + NP + 2 (NP <= 32: rows at
                // g2_row_offset, [w | 0] last) or 3*(NP + 4) (NP > 32: rows padded to NP + 4, k_increment_big)
  int K2;       // J2 cubature points
  int K2p;      // padded to a multiple of kQC
  int nchunks;  // K2p / kQC
  const double* G2;       // [K2p][S]   projected operator rows (zero padded)
  const double* w2;       // [K2p]      cubature weights (0 on pads)
  const double* Ke;       // [NP][NP]   Σ_{all q} w G^T C_e G   (elastic predictor stiffness)
  const double* KaEe;     // [NP][3]    Σ_{all q} w G^T C_e
  const double* Le;       // [NP][NP+1] Cholesky factor of K_e (lower), used when no point is plastic
  const double* LeInv;    // [NP]       1 / diag(Le)
  double CEEe[9];         //            Σ_{all q} w C_e
  double inv_denom;       // 1 / (3 mu + h) of the J2 material
  double volume;
  MatDev mat2;            // the (single) J2 material of the history-carrying points
  // finite strain (kinematics 1): G2 is the 4-row gradient operator with rows
  // [4 x (NP + 4) | w | 0] (S = 4 (NP + 4) + 2), J2 chunks [0, nch_hist) then elastic chunks
  int nch_hist;           // chunks carrying history (J2 points, = K2p / kQC)
  int K_el;               // elastic cubature points (chunks nch_hist .. nchunks-1)
  MatDev matE;            // the (single) elastic material of the finite-strain model
};

struct PointsDev {
  int64_t P;
  double* hist;     // [P][K2p/32][5][32]: per (point, 32-point chunk) one 1,280-B block of SoA
                    // eps_p(4), eq — one bulk copy per chunk, coalesced lane stores
                    // (sigma33 is write-only in the reference and recomputed on readback)
  double* alpha_c;  // [P][NP] committed reduced coordinates
  double* E_c;      // [P][4]  committed macro strain (3) / displacement gradient H (4)
  double* bp;       // [P][NP] Σ_{J2 q} w G_q^T S(eps_p,q)  (committed plastic-strain load)
  double* sp;       // [P][4]  Σ_{J2 q} w S(eps_p,q)
  PointState* st;   // .pad[0] = which history buffer is committed (small-n kernel)
  uint8_t* flags;   // [P][K2p] plastic flags of the last commit (optional)
  // small-n kernel (k_increment): double-buffered history. Every assembly pass
  // writes its candidate history into the non-committed buffer; accepting a
  // converged state flips st[p].pad[0] (no separate commit pass). Offsets in
  // elements from hist / flags to the second buffer (0 = single buffer).
  int64_t hist_alt;
  int64_t flags_alt;
};

struct Outputs {
  double* sigma;  // [P][3]  (finite strain: P_M [P][4])
  double* C;      // [P][9]  (finite strain: A_M [P][16])
  double* res;    // [P]
  int* iters;     // [P]
  int* status;    // [P]
  int* pcount;    // [P]
};

struct NewtonCfg {
  double tol;
  int max_iter;
  int max_bis;
};

// Device counters of one launch (for the roofline): assembly passes, commit
// passes, J2 points that were plastic in assembly passes.
struct IncCounters {
  unsigned long long assemblies;
  unsigned long long commits;
  unsigned long long plastic_evals;
  unsigned long long commit_plastic;  // plastic J2 points of the accepted states
};

struct IncArgs {
  ModelDev M;
  PointsDev D;
  Outputs O;
  NewtonCfg cfg;
  const double* dE;    // [P][3] this increment's path point (finite strain: H [P][4])
  int* work;           // work-queue counter (zeroed before launch)
  IncCounters* cnt;    // optional
  // debug: one assembly of point dbg_point at (dbg_alpha, dbg_E), dumped to dbg
  double* dbg;
  const double* dbg_alpha;
  const double* dbg_E;
  int64_t dbg_point;
  // watchdog trace (mapped pinned host memory, FE2_TRACE=1): per warp
  // {ring position, state code, point, stage-counter snapshot}
  volatile int* trace;
  // monolithic iteration (k_increment<..., MONO>): per-point working record
  // [P][mono_stride(NP)], see mono_stride; mono_first = first iteration of a step
  double* mono;
  int mono_first;
};

// Per-point record of the monolithic scheme: z[4][NP] (K^-1 r, K^-1 K_aE),
// r_plastic[NP], α_w[NP] (the evaluation point), E[3], Σ_plastic[3], ref, pad.
constexpr int mono_stride(int NP) { return 6 * NP + 8; }

// host launchers (hrom_kernels.cu: NP <= 32, one warp per point;
// hrom_kernels_big.cu: NP in {40,48,56,64,80,96,112,128}, one CTA per point)
void launch_increment(const IncArgs& a, int num_sms, cudaStream_t s);
// one monolithic Newton iteration for every point (no commit), NP <= 32
void launch_increment_mono(const IncArgs& a, int num_sms, cudaStream_t s);
// adopt the last monolithic iterate of every live point as its committed state
void launch_mono_commit(const PointsDev& D, int NP, const double* mono, cudaStream_t s);
bool launch_increment_big(const IncArgs& a, int num_sms, cudaStream_t s);
bool launch_increment_big_other(const IncArgs& a, int num_sms, cudaStream_t s);  // NP not 64 / 128
bool launch_increment_big_gen(const IncArgs& a, int num_sms, cudaStream_t s);    // power-law / creep models
// one monolithic Newton iteration for every point, NP in the launch_increment_big set
bool launch_increment_big_mono(const IncArgs& a, int num_sms, cudaStream_t s);
size_t increment_big_smem(int NP);
void launch_material_batch(const MatDev& m, int64_t N, const double* eps, const double* st_in, double* sigma,
                           double* C, double* st_out, uint8_t* plastic, int* err, cudaStream_t s);
size_t increment_smem(int NP);
// batched constitutive update on SoA device buffers (material_soa.cu)
void launch_material_soa(const MatDev& m, int64_t N, const double* eps, const double* hin, double* sig, double* C6,
                         double* hout, uint8_t* plastic, int num_sms, cudaStream_t s);
// finite-strain (Biot) path, hrom_kernels_fs.cu: NP <= 32, one warp per point
void launch_increment_fs(const IncArgs& a, int num_sms, cudaStream_t s);
size_t increment_fs_smem(int NP);

}  // namespace fe2
