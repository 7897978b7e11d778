// Device side of the B200 hyper-ROM engine: data layout, the fused
// assemble + Newton-step round (K2+K3), the history commit (K1) and the
// batched material update. See DESIGN.md for the layout and rooflines.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "material.cuh"

namespace fe2 {

constexpr int kQC = 32;  // cubature points per chunk (one per lane in the material phase)

enum Phase : int { kActive = 0, kDone = 1, kFailed = 2 };
enum Mode : int { kNewton = 0, kLineSearch = 1 };

// Per-point Newton / increment state (one 96-byte record per macro point).
struct PointState {
  double a;        // current line-search step
  double rn_it;    // residual norm at the current iterate
  double best_rn;  // best line-search residual so far
  double best_a;   // its step
  double ref;      // convergence reference (fixed at it = 0)
  double done;     // fraction of the increment committed (run_trajectory)
  double frac;     // current sub-step fraction
  double rn_last;  // last residual norm
  int mode, it, ls, iters, bis, phase, err, pad;
};

struct ModelDev {
  int n;        // modes
  int NP;       // modes padded to a multiple of 8 (DMMA tile)
  int S;        // doubles per cubature point in G2 (3*NP + 1, odd: bank-conflict free rows)
  int K2;       // J2 cubature points
  int K2p;      // padded to a multiple of kQC
  int nchunks;  // K2p / kQC
  const double* G2;       // [K2p][S]   projected operator rows (zero padded)
  const double* w2;       // [K2p]      cubature weights (0 on pads)
  const double* Ke;       // [NP][NP]   Σ_{all q} w G^T C_e G   (elastic predictor stiffness)
  const double* KaEe;     // [NP][3]    Σ_{all q} w G^T C_e
  double CEEe[9];         //            Σ_{all q} w C_e
  double volume;
  MatDev mat2;            // the (single) J2 material of the history-carrying points
};

struct PointsDev {
  int64_t P;
  double* hist;  // 5 SoA components [5][P][K2p]: eps_p(4), eq (sigma33 is recomputed on readback)
  double* alpha_c;
  double* alpha;
  double* alpha_ev;
  double* dalpha;  // [P][NP] each
  double* E_prev;
  double* E_tgt;
  double* E_ev;  // [P][3] each
  double* bp;     // [P][NP]  Σ_{J2 q} w G_q^T S(eps_p,q)  (committed plastic-strain load)
  double* sp;     // [P][4]   Σ_{J2 q} w S(eps_p,q)
  PointState* st;
  uint8_t* flags;  // [P][K2p] plastic flags of the last commit (optional)
};

struct Outputs {
  double* sigma;  // [P][3]
  double* C;      // [P][9]
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

struct RoundArgs {
  ModelDev M;
  PointsDev D;
  Outputs O;
  NewtonCfg cfg;
  const int* active;
  int n_active;
  int* next_active;
  int* n_next;
  double* dbg;  // debug assembly dump (r, K, KaE, CEE, Sraw) or nullptr
};

// host launchers (hrom_kernels.cu)
void launch_newton_round(const RoundArgs& a, cudaStream_t s);
void launch_commit(const ModelDev& M, const PointsDev& D, const Outputs& O, cudaStream_t s);
void launch_begin_increment(const ModelDev& M, const PointsDev& D, const Outputs& O, const double* dE,
                            int* active, int* n_active, cudaStream_t s);
void launch_material_batch(const MatDev& m, int64_t N, const double* eps, const double* st_in, double* sigma,
                           double* C, double* st_out, uint8_t* plastic, cudaStream_t s);
size_t newton_round_smem(int NP);

}  // namespace fe2
