/*
 * fe2rom CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain C++20 restatement (no Eigen) of the reference arithmetic of
 * arXiv 2306.02687's `fe2rom` library (/root/reference/proj/include/fe2rom),
 * composed into the reduced (hyper-ROM) form the SPEC contracts
 * `reduced_newton` and `hyper_assemble`
 * describe. It is the checker for the B200 path, never the thing measured
 * or shipped: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * Parity status:
 *   - material point (J2 linear hardening + elastic): PINNED by the
 *     reference's own known-answer tests (test_materials.cpp:49-118,210-271),
 *     ported in tests/test_oracle_kat.py;
 *   - HF micro Newton / homogenize semantics: PINNED by the reference KATs of
 *     test_rve.cpp:44-62, 82-100, 132-195, ported on the dense HF restatement;
 *   - hyper-ROM level (random Φ, random cubature): the reference has no code
 *     for it, so it is anchored by the bridge test (full basis + full
 *     cubature == HF) — "parity unpinned" beyond that bridge.
 *
 * Every entry point returns 0 on success, else 1 + the reference ErrorCode
 * ordinal (common.hpp:26-37); orc_last_error() gives the message.
 */
#ifndef FE2ROM_ORACLE_H
#define FE2ROM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* material kinds (materials.hpp:37-76): 0 = ElasticParams {E, nu},
 * 1 = J2LinearParams {E, nu, sy0, h}, 2 = PowerLawParams {E, nu, sy0, N},
 * 3 = CreepParams {E, nu, A, n, m, dt} (dt: time of one load increment,
 * PathStep::dt; bisected sub-steps use their fraction of it). */
typedef struct {
  int kind;
  double p[6];
} orc_material_t;

const char* orc_last_error(void);

/* ---- Rng (common.hpp:56-88) ------------------------------------------- */
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void* rng);
uint64_t orc_rng_next_u64(void* rng);
double orc_rng_uniform(void* rng);
double orc_rng_uniform_ab(void* rng, double a, double b);
int orc_rng_uniform_int(void* rng, int n);
double orc_rng_normal(void* rng);

/* ---- material point: update_material (materials.hpp:317-325) ---------- */
/* state6 = (eps_p[4] packed 11,22,33,12-tensor, eq, sigma33) */
int orc_update_material(const orc_material_t* mat, const double* state_in6, const double* eps3,
                        double* sigma3, double* C9, double* state_out6, int* plastic);
/* packed 4-component update (update4, materials.hpp:333-348) */
int orc_update4(const orc_material_t* mat, const double* state_in6, const double* eps4,
                double* sigma4, double* D16, double* state_out6);

/* ---- RVE mesh (mesh.hpp:171-352) --------------------------------------- */
typedef struct orc_mesh_s* orc_mesh_t;
/* geometry: 0 = RveGeometry::default_cell(subdiv); 1 = empty cell (homogeneous) */
int orc_mesh_build(int geometry, int subdivisions, orc_mesh_t* out);
void orc_mesh_free(orc_mesh_t m);
int orc_mesh_counts(orc_mesh_t m, int* n_nodes, int* n_elements, double* area);
/* nodes: xy[2*n_nodes]; elements: conn[6*n_el], mat[n_el] */
int orc_mesh_arrays(orc_mesh_t m, double* xy, int* conn, int* mat);
/* B (3x12, row-major) and w = (1/6) detJ at integration point ip = 3e+g (rve.hpp:167-185) */
int orc_mesh_ip(orc_mesh_t m, int ip, double* B36, double* w, int* element);

/* ---- HF dense restatement of micro_newton / homogenize (rve.hpp:285-392),
 *      linear BC (rve.hpp:84-92), strain-driven trajectory (rve.hpp:448-494) */
typedef struct {
  double tol;   /* MicroOptions::tol (1e-8)  */
  int max_iter; /* MicroOptions::max_iter (30) */
  int max_bisections; /* TrajectoryOptions::max_bisections (4) */
} orc_newton_opts_t;

/* Run a strain path E[n_steps][3] on the HF RVE (materials by element id).
 * Per step outputs: sigma[3], C[9], iterations, converged flag.
 * u_fluct_inf (optional, per step): max |u - E.x| over all DOFs.
 * snapshots (optional) [n_steps][n_dofs]: the converged fluctuation u - E.x
 * of each step (SnapshotRecorder x_u, rve.hpp:486-490). */
int orc_hf_trajectory(orc_mesh_t m, const orc_material_t* mats, int n_mats, int n_steps,
                      const double* E, const orc_newton_opts_t* opts, double* sigma, double* C,
                      int* iterations, double* u_fluct_inf, double* res_hist_last, double* snapshots);

/* ---- hyper-ROM model (offline stage): Φ, cubature rule, G_q ------------
 * Φ: Gaussian (Rng) on free DOFs, Householder thin QR, zero rows on the
 * linear-BC boundary. Cubature: K distinct IPs by partial Fisher-Yates with
 * uniform_int, weights U[0.5,1.5]·area/K. G_q = B_q Φ[dofs(el(q)), :].
 * K == 0 selects the full rule (all IPs, own weights); n == 0 selects the
 * identity basis on free DOFs (the SPEC.md:591 bridge). */
typedef struct orc_model_s* orc_model_t;
int orc_model_build(int subdivisions, int n, int K, uint64_t seed, orc_model_t* out);
int orc_model_build_on_mesh(orc_mesh_t mesh, int n, int K, uint64_t seed, orc_model_t* out);
void orc_model_free(orc_model_t m);
/* sizes: n modes, K cubature points, n_free, volume */
int orc_model_sizes(orc_model_t m, int* n, int* K, int* n_free, double* volume);
/* G[K][3][n], w[K], ip_id[K], mat_id[K] (0 = J2 matrix, 1 = elastic inclusion) */
int orc_model_arrays(orc_model_t m, double* G, double* w, int* ip_id, int* mat_id);
/* Φ restricted to free DOFs: phi[n_free][n] */
int orc_model_phi(orc_model_t m, double* phi);

/* ---- seeded macro strain paths (per-point streams keyed by point index) */
/* kind 0: BASELINE config-0 uniaxial rotated path; kind 1: config-1 reversal.
 * E[P][n_incr][3] for global points p0 .. p0+P-1. */
int orc_paths(int kind, uint64_t seed, int64_t p0, int64_t P, int n_incr, double* E);

/* ---- the hyper-ROM online path (the oracle for the GPU kernels) -------- */
typedef struct orc_hrom_s* orc_hrom_t;
int orc_hrom_create(int n, int K, const double* G, const double* w, const int* mat_id,
                    const orc_material_t* mats, int n_mats, double volume, orc_hrom_t* out);
void orc_hrom_free(orc_hrom_t h);

typedef struct {
  double* sigma;         /* [P][n_incr][3]  macro stress Σ                */
  double* C;             /* [P][n_incr][9]  condensed macro tangent       */
  int* iters;            /* [P][n_incr]     Newton iterations (all solves of the increment) */
  int* plastic_count;    /* [P][n_incr]     # cubature points with f > 0 at commit */
  double* res_norm;      /* [P][n_incr]     final reduced residual norm  */
  int* status;           /* [P][n_incr]     0 ok, else 1+ErrorCode        */
  int* bisections;       /* [P][n_incr]     load-step bisections used     */
  uint8_t* plastic_flags;/* optional [P][n_incr][K]                       */
  double* alpha;         /* optional [P][n] final committed α             */
  double* state;         /* optional [P][K][6] final committed history    */
} orc_hrom_out_t;

/* Run P independent macro points (global ids p0..) through n_incr increments
 * E[P][n_incr][3] from the virgin state, n_threads std::threads in the
 * reference parallel_for pattern (common.hpp:109-132). */
int orc_hrom_run(orc_hrom_t h, int64_t P, int n_incr, const double* E,
                 const orc_newton_opts_t* opts, int n_threads, orc_hrom_out_t* out);

/* One assembly (hyper_assemble) at (α, E) from a given per-point history
 * state[K][6]: r[n], K[n][n], KaE[n][3], C_EE[9], S_raw[3]; state_out[K][6]
 * (nullable) = the updated history of that assembly. */
int orc_hrom_assemble(orc_hrom_t h, const double* alpha, const double* E, const double* state,
                      double* r, double* Kaa, double* KaE, double* C_EE, double* S_raw,
                      int* plastic_count, double* state_out);

/* ---- finite strain, Biot stress (BASELINE config 2) — PARITY UNPINNED:
 * the reference has no finite-strain code. Components ordered (F00, F01,
 * F10, F11); P = R T(U - I); A = dP/dF row-major 4x4. */
int orc_update_biot(const orc_material_t* mat, const double* state_in6, const double* F4, double* P4, double* A16,
                    double* state_out6, int* plastic);
/* 4-row displacement-gradient operator G4[K][4][n] of orc_model_build(subdivisions, n, K, seed) */
int orc_model_g4(int subdivisions, int n, int K, uint64_t seed, double* G4);
/* config-2 paths: H[P][n_incr][4] (F = I + H), det(I + H_end) > 0.8 */
int orc_paths_fs(uint64_t seed, int64_t p0, int64_t P, int n_incr, double* H);
typedef struct orc_hrom_fs_s* orc_hrom_fs_t;
int orc_hrom_fs_create(int n, int K, const double* G4, const double* w, const int* mat_id, const orc_material_t* mats,
                       int n_mats, double volume, orc_hrom_fs_t* out);
void orc_hrom_fs_free(orc_hrom_fs_t h);
/* outputs as orc_hrom_out_t with sigma -> P_M [P][n_incr][4], C -> A_M [P][n_incr][16] */
int orc_hrom_fs_run(orc_hrom_fs_t h, int64_t P, int n_incr, const double* H, const orc_newton_opts_t* opts,
                    int n_threads, orc_hrom_out_t* out);
int orc_hrom_fs_assemble(orc_hrom_fs_t h, const double* alpha, const double* H, const double* state, double* r,
                         double* Kaa, double* KaF, double* KFa, double* CFF, double* P_raw, int* plastic_count);

#ifdef __cplusplus
}
#endif
#endif
