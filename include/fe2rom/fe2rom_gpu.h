/*
 * fe2rom_gpu.h — C ABI of the B200 hyper-ROM macro-Gauss-point engine.
 *
 * Drop-in boundary for the online hot path of the monolithic hyper-ROM FE²
 * scheme (arXiv 2306.02687): the batched evaluation of hyper-reduced RVE
 * models at every macro Gauss point. Each entry point replaces a reference
 * interface (paths relative to /root/reference/proj/include/fe2rom/):
 *
 *   fe2_material_update_batch  <- update_material        materials.hpp:317-325
 *                                 (batched; update4 elastic / J2 / power law / creep :199-292)
 *   fe2_hrom_create            <- build_rve_problem      rve.hpp:167-185, in the
 *                                 reduced form of SPEC.md:351-359 (G_q = B_q Φ,
 *                                 cubature weights), materials by id (:158-162)
 *   fe2_hrom_alloc_points      <- std::vector<MaterialState>(n_ips)  rve.hpp:450,
 *                                 run_trajectory's virgin states, one set per point
 *   fe2_hrom_solve_increment   <- one path step of run_trajectory rve.hpp:459-491:
 *                                 set_macro_strain + micro_newton (:285-346, reduced:
 *                                 SPEC.md:289-297) + homogenize (:350-392) + the
 *                                 commit of states (:480), with load-step bisection
 *                                 (:473-478), for every point of the batch
 *   fe2_hrom_read_state        <- MicroResult::states / MaterialState   rve.hpp:207,
 *                                 materials.hpp:102-106
 *   fe2_last_error             <- fe2rom::Error::what()  common.hpp:39-46
 *   fe2_hrom_create_fs         <- (no reference counterpart: finite-strain Biot
 *                                 variant of BASELINE config 2, SURVEY.md §8 a15;
 *                                 parity unpinned, checked against oracle fs_*)
 *
 * Conventions
 *   - Strain is engineering Voigt (E11, E22, g12), stress (S11, S22, S12)
 *     (rve.hpp:13-19, materials.hpp:21). C is row-major 3x3.
 *   - History per cubature point is MaterialState = (eps_p[4] packed
 *     11,22,33,12-tensor, eq, sigma33): 6 doubles (materials.hpp:102-106).
 *   - Return codes: 0 = OK, else 1 + the reference ErrorCode ordinal
 *     (common.hpp:26-37): 1 config, 2 geometry, 3 mesh, 4 material,
 *     5 solver, 6 numeric, 7 rank, 8 bc, 9 io, 10 provenance. No exception
 *     crosses the ABI. Per-point Newton failure is reported in status[]
 *     with the same codes (run_trajectory throws ErrorCode::solver after
 *     max_bisections, rve.hpp:474-476).
 *   - The caller owns host arrays; the library owns device buffers. A handle
 *     is bound to one device and is not thread-safe. Multi-GPU = one handle
 *     per device (one process per GPU); points are sharded, never split.
 *   - Finite-strain handles (fe2_hrom_create_fs) take the macro displacement
 *     gradient H = F - I as (H00, H01, H10, H11) in place of E, return the
 *     first Piola-Kirchhoff stress P_M[4] in place of sigma and the tangent
 *     A_M = dP_M/dF row-major 4x4 in place of C; everything else is shared.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with code 6 (numeric) and a message.
 */
#ifndef FE2ROM_GPU_H
#define FE2ROM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Material parameters (materials.hpp:37-76, validate :80-98).
 * kind 0: ElasticParams  p = {E, nu}
 * kind 1: J2LinearParams p = {E, nu, sigma_y0, hardening}
 * kind 2: PowerLawParams p = {E, nu, sigma_y0, N}          sy(e) = sy0 (1 + E e / sy0)^N
 * kind 3: CreepParams    p = {E, nu, A, n, m, dt}          deq/dt = (q/A)^(n/(m+1)) ((m+1) eq)^(m/(m+1));
 *                        dt = time of one load increment (PathStep::dt; bisected sub-steps use their share)
 * The small-strain hyper-ROM engine (fe2_hrom_create; one inelastic material per
 * model), fe2_material_update_batch and the HF solver (fe2_hf_*) carry all four;
 * the finite-strain engine, the monolithic iteration and the SoA update carry 0/1. */
typedef struct {
  int kind;
  double p[6];
} fe2_material_t;

/* MicroOptions (rve.hpp:195-200) + TrajectoryOptions::max_bisections (:439-443) */
typedef struct {
  double tol;         /* default 1e-8 */
  int max_iter;       /* default 30   */
  int max_bisections; /* default 4    */
} fe2_newton_opts_t;

typedef struct fe2_hrom_s* fe2_hrom_t;

const char* fe2_last_error(void);
/* library version string, e.g. "fe2rom-b200 0.1 sm_100a" */
const char* fe2_version(void);
/* number of usable CUDA devices (0 on a host without GPU) */
int fe2_device_count(void);

/* ---- batched material point: update_material over N points on the GPU.
 * eps[N*3], state_in[N*6] (may be NULL = virgin), outputs sigma[N*3],
 * C[N*9], state_out[N*6] (nullable), plastic[N] (nullable). Host buffers. */
int fe2_material_update_batch(int device, const fe2_material_t* mat, int64_t N, const double* eps,
                              const double* state_in, double* sigma, double* C, double* state_out,
                              uint8_t* plastic);

/* ---- batched material point on DEVICE structure-of-arrays buffers (the
 * HBM-bound constitutive update; SURVEY §8(b) fe2_material_update_batch with
 * SoA history). eps[3][N] (E11, E22, g12), hist_in[5][N] (eps_p 11,22,33,12,
 * eq; NULL = virgin) -> sigma[3][N], C6[6][N] (C00 C01 C02 C11 C12 C22 of the
 * symmetric condensed tangent), hist_out[6][N] (eps_p[4], eq, sigma33;
 * nullable), plastic[N] (nullable). Asynchronous on `stream` (cudaStream_t). */
int fe2_material_update_soa_device(int device, const fe2_material_t* mat, int64_t N, const double* d_eps,
                                   const double* d_hist_in, double* d_sigma, double* d_C6, double* d_hist_out,
                                   uint8_t* d_plastic, void* stream);

/* ---- hyper-ROM model on one device.
 * G[K][3][n] host, w[K], mat_id[K] (index into mats), volume = RVE area. */
int fe2_hrom_create(int device, int n, int K, const double* G, const double* w, const int* mat_id,
                    const fe2_material_t* mats, int n_mats, double volume, fe2_hrom_t* out);
void fe2_hrom_destroy(fe2_hrom_t h);

/* ---- finite-strain (Biot stress) hyper-ROM model (BASELINE config 2).
 * G4[K][4][n] is the displacement-gradient operator (rows dux/dX, dux/dY,
 * duy/dX, duy/dY; fe2_model_g4), n <= 32, at most one J2 and one elastic
 * material. Solve calls then take H[P*4] and return P_M[P*4], A_M[P*16]. */
int fe2_hrom_create_fs(int device, int n, int K, const double* G4, const double* w, const int* mat_id,
                       const fe2_material_t* mats, int n_mats, double volume, fe2_hrom_t* out);
/* 0 = small strain (fe2_hrom_create), 1 = finite strain (fe2_hrom_create_fs) */
int fe2_hrom_kinematics(fe2_hrom_t h, int* kinematics);
/* finite-strain assembly of a point's committed history at (α, H): r[n],
 * Kaa[n*n], KaF[n*4], KFa[4*n], C_FF[16], P_raw[4] (host) */
int fe2_hrom_fs_assemble_point(fe2_hrom_t h, int64_t point, const double* alpha, const double* H, double* r,
                               double* Kaa, double* KaF, double* KFa, double* C_FF, double* P_raw);

/* Allocate P >= 1 macro points in the virgin state (α = 0, MaterialState{}).
 * P = 0 is ErrorCode::config; a batch that does not fit in HBM is
 * ErrorCode::numeric and leaves the handle usable for a smaller P.
 * keep_flags != 0 also keeps per-(point, cubature point) plastic flags of
 * the last commit (P*K bytes) for parity checks. */
int fe2_hrom_alloc_points(fe2_hrom_t h, int64_t P, int keep_flags);
/* Return the allocated points to the virgin state (no reallocation). */
int fe2_hrom_reset_points(fe2_hrom_t h);
/* Device pointers of the handle's own output buffers (filled by every
 * fe2_hrom_solve_increment call), e.g. to all-gather them over NCCL. */
int fe2_hrom_output_ptrs(fe2_hrom_t h, double** d_sigma, double** d_C, int** d_iters, int** d_plastic_count,
                         double** d_res_norm, int** d_status);

/* One load increment for all P points: E[P*3] is the path point of this
 * increment (the previous one is remembered; the first starts from 0).
 * Host buffers; every output is nullable. iters[P] counts all Newton
 * iterations of the increment (bisected sub-steps included). */
int fe2_hrom_solve_increment(fe2_hrom_t h, const double* E, const fe2_newton_opts_t* opts,
                             double* sigma, double* C, int* iters, int* plastic_count,
                             double* res_norm, int* status);

/* Asynchronous form of fe2_hrom_solve_increment (same arguments, host
 * buffers — pin them, cudaHostAlloc, for the copies to overlap): returns once
 * the increment is queued. Inputs are staged and outputs produced in two
 * alternating device buffers, and each increment's outputs are copied to the
 * host on a second stream while the next increment computes. E must stay
 * unchanged and the outputs are only valid until / after fe2_hrom_wait
 * (the copies run asynchronously). Increments are applied in call order. */
int fe2_hrom_solve_increment_async(fe2_hrom_t h, const double* E, const fe2_newton_opts_t* opts,
                                   double* sigma, double* C, int* iters, int* plastic_count,
                                   double* res_norm, int* status);
/* Wait for every queued asynchronous increment and output copy. */
int fe2_hrom_wait(fe2_hrom_t h);

/* Same, on DEVICE buffers already resident in HBM (E, outputs), ordered on
 * `stream` (cudaStream_t, NULL = the handle's stream). The call returns
 * after the increment is complete on `stream`. */
int fe2_hrom_solve_increment_device(fe2_hrom_t h, const double* d_E, const fe2_newton_opts_t* opts,
                                    double* d_sigma, double* d_C, int* d_iters, int* d_plastic_count,
                                    double* d_res_norm, int* d_status, void* stream);

/* ---- multi-GPU exchange of the monolithic scheme ----
 * Points are sharded in contiguous blocks over the ranks of one box, one
 * handle per device; the engines never communicate during assembly,
 * factorisation or condensation. After an increment (or monolithic macro
 * iteration) every rank needs every point's condensed response, so the only
 * collective is an NCCL all-gather of per-point records over NVLink, plus a
 * max all-reduce of two flags for lockstep termination.
 * libnccl.so.2 is dlopen'ed at first use (no link-time dependency).
 *   fe2_nccl_get_unique_id: rank 0 creates the 128-byte id, the caller
 *     broadcasts it (MPI, torch.distributed, a file ...);
 *   fe2_nccl_comm_init / _destroy: one communicator per rank and device.
 *   fe2_hrom_gather_layout: every rank's point count P_r over comm (one
 *     all-gather of an int64, host-synchronising; the handle caches it, and
 *     fe2_hrom_gather computes it on first use). The gathered buffer holds
 *     world blocks of P_max = max_r P_r rows; rank r's points are rows
 *     [r*P_max, r*P_max + P_r) and the rest of its block is padding
 *     (status -1, NaN values). counts[world] is nullable.
 * fe2_hrom_gather packs this rank's records
 *   {Σ (nc) | C_macro (nt) | ‖r‖ | status} — nc, nt = 3, 9 small strain
 *   (14 doubles per point), 4, 16 finite strain (P_M, A_M) —
 * from the given device outputs of the last increment / monolithic iterate
 * (NULL = the handle's own buffers, fe2_hrom_output_ptrs) into its block of
 * d_all, all-gathers in place into d_all [world][P_max][nc + nt + 2]
 * (device, doubles) and max-reduces flags[0] = "some point failed"
 * (status > 0) and flags[1] = "some point has ‖r‖ > res_tol" (the
 * monolithic iteration's termination test; pass +inf to ignore). With
 * flags != NULL (host int[2]) the call synchronises the handle's stream and
 * returns the flags; with NULL it stays asynchronous on the stream.
 * Replaces nothing in the reference (its RVE solves run in one process,
 * SPEC.md:247, :511); the records are what fe2.macro_step consumes
 * (SPEC.md:474-481). Errors: ErrorCode::rank for NCCL failures. */
int fe2_nccl_get_unique_id(void* id128);
int fe2_nccl_comm_init(int device, int nranks, int rank, const void* id128, void** comm);
int fe2_nccl_comm_destroy(void* comm);
int fe2_hrom_gather_layout(fe2_hrom_t h, void* comm, int64_t* P_max, int64_t* counts);
int fe2_hrom_gather(fe2_hrom_t h, void* comm, const double* d_sigma, const double* d_C, const double* d_res_norm,
                    const int* d_status, double res_tol, double* d_all, int* flags);

/* Committed state readback (host): alpha[P*n], state[P*K*6] in the caller's
 * cubature order (elastic-material points report eps_p = 0, eq = 0 and the
 * sigma33 of their last commit), flags[P*K] (needs keep_flags). Nullable. */
int fe2_hrom_read_state(fe2_hrom_t h, double* alpha, double* state, uint8_t* flags);

/* One hyper-assembly of point 0's committed history at a
 * given (α, E): r[n], Kaa[n*n], KaE[n*3], C_EE[9], S_raw[3] (host). */
int fe2_hrom_assemble_point(fe2_hrom_t h, int64_t point, const double* alpha, const double* E,
                            double* r, double* Kaa, double* KaE, double* C_EE, double* S_raw);

/* Save / return to the committed state of every point (history, α, loads,
 * previous path point, failure codes): a macro Newton iteration that does not
 * converge is undone by fe2_hrom_restore (the micro commit of the reference's
 * nested scheme happens only when the macro step is accepted). */
int fe2_hrom_snapshot(fe2_hrom_t h);
int fe2_hrom_restore(fe2_hrom_t h);

/* Mixed control for every point (rve.hpp:496-571 mixed_control_step, the
 * consumer pattern of the uniaxial-tension calibration): strain
 * components with control[p*3+j] != 0 are prescribed (E_prescribed), the others
 * are driven so the conjugate macro stresses reach sigma_target, by an outer
 * Newton on the condensed tangent (complete pivoting) — every outer iteration
 * re-solves the active points from their committed state. Converged when
 * |Σ_u - target_u| <= tol (max(1e-12, |target|) + 1e-3) (reference defaults
 * tol 1e-10, max_iter 25). E[P*3]: in the committed macro strains, out the
 * converged ones; the engine is left at the accepted state (committed).
 * status 0 or 1 + ErrorCode (solver: no convergence in max_iter or singular J;
 * the micro solve's code if it failed). Small-strain handles. */
int fe2_hrom_mixed_step(fe2_hrom_t h, const int* control, const double* E_prescribed, const double* sigma_target,
                        double tol, int max_iter, const fe2_newton_opts_t* micro, double* E, double* sigma,
                        double* C, int* outer_iters, int* status);

typedef struct {
  int64_t points;
  int n, K, K_j2;
  int64_t kernel_launches;   /* own kernels launched since create */
  int64_t increments;        /* increments solved (one persistent launch each) */
  int64_t assemblies;        /* (point, hyper-assembly pass) pairs since create */
  int64_t commits;           /* (point, history-commit pass) pairs since create */
  int64_t plastic_evals;     /* (point, J2 cubature point) found plastic in assembly passes */
  /* CUDA-event kernel timing (only while fe2_hrom_set_timing is on) */
  double kernel_ms;          /* summed duration of the increment kernels */
  int64_t timed_launches, timed_assemblies, timed_commits, timed_plastic_evals;
  int64_t timed_commit_plastic; /* J2 points written by commit passes in timed launches */
} fe2_hrom_stats_t;
int fe2_hrom_stats(fe2_hrom_t h, fe2_hrom_stats_t* out);
/* zero every counter of fe2_hrom_stats */
int fe2_hrom_reset_stats(fe2_hrom_t h);
/* enable per-launch CUDA-event timing inside solve_increment */
int fe2_hrom_set_timing(fe2_hrom_t h, int on);
/* order all later work of the handle on `stream` (cudaStream_t; NULL = own). NULL is also the
 * legacy default stream's handle: a caller working on the default stream (e.g. torch's
 * current_stream() without a stream context) gets the handle's non-blocking stream and must
 * synchronise with it (fe2_hrom_wait), or pass a stream of its own. */
int fe2_hrom_set_stream(fe2_hrom_t h, void* stream);

/* ---- macro FE driver of the two-scale beam (the caller
 * of the hot path; SPEC.md:455-518 fe2.macro_step / solve_program, nested
 * variant): plane-strain L x H strip of Tri6 pairs (build_beam_mesh,
 * mesh.hpp:133-169), left edge clamped, vertical tip displacement U on the
 * x = L edge, reaction R. Each macro Newton iteration runs converged micro
 * solves for all macro Gauss points (one engine increment from the committed
 * state, fe2_hrom_restore) and assembles the tangent from C_macro; accepted
 * steps commit (fe2_hrom_snapshot). Program: n_load steps to u_max, then
 * unloading in the same steps until R changes sign (U_residual = linear zero
 * crossing; NaN if none within max_unload steps). Host code; the engine
 * holds fe2_macro_points() points. A finite-strain engine (fe2_hrom_create_fs)
 * makes it a total-Lagrangian FE² run: H = F - I from the 4-row gradient
 * operator, f_int = sum w Bg^T P, K = sum w Bg^T A Bg (LU). */
typedef struct {
  double length, height;      /* beam L x H (desk default 4 x 1) */
  int nx, ny;                 /* cells along x / y, two Tri6 each (desk: 8 x 2 = 32 elements) */
  double u_max;               /* peak tip displacement */
  int n_load;                 /* load steps to u_max */
  int max_unload;             /* unload steps at most */
  double tol;                 /* macro residual tolerance relative to max(|f_int|, largest accepted |f_int|) (1e-6) */
  int max_iter;               /* macro Newton iterations per step (20) */
  int max_bisections;         /* macro step bisections (4) */
  fe2_newton_opts_t micro;    /* micro Newton options (monolithic: micro.tol = the joint micro tolerance) */
  int scheme;                 /* 0 = nested (converged micro solves per macro iteration), 1 = monolithic */
} fe2_macro_config_t;
int fe2_macro_points(const fe2_macro_config_t* cfg, int64_t* n_points);
/* per macro Gauss point: B[36] (3 x 12 strain operator), w, element (nullable) */
int fe2_macro_gauss(const fe2_macro_config_t* cfg, double* B, double* w, int* elem);
/* rows[k] = (U, R, macro iterations of the step, cumulative micro iterations, wall ms) */
int fe2_macro_run(const fe2_macro_config_t* cfg, fe2_hrom_t engine, double* rows, int max_rows, int* n_rows,
                  double* u_residual);
/* The same program with full-field RVEs at the macro points (HF FE², nested;
 * the reference the hyper-ROM curves are compared with):
 * hf holds fe2_macro_points() points (fe2_hf_alloc_points). */
typedef struct fe2_hf_s* fe2_hf_t;
int fe2_macro_run_hf(const fe2_macro_config_t* cfg, fe2_hf_t hf, double* rows, int max_rows, int* n_rows,
                     double* u_residual);

/* ---- monolithic scheme (SPEC.md:474-481 HF_monolithic / hyper-ROM): the
 * micro problems advance ONE reduced Newton iteration per macro iteration,
 * sharing the macro linearisation. Small-strain handles, any supported n
 * (warp-per-point kernel for n <= 32, CTA-per-point kernel above).
 *   fe2_hrom_mono_begin     start a macro step from the committed state
 *                           (α = α_committed; history candidates discarded)
 *   fe2_hrom_mono_iterate   for every point at this macro iterate's E[P*3]:
 *                           α -= K^-1 (r + K_aE ΔE) with the previous iteration's
 *                           factors (ΔE = change of E since then), assemble at
 *                           (E, α), factor, and return the condensed stress
 *                           Σ~ = (Σ_raw - K_Eα K^-1 r)/V, C = (C_EE - K_Eα K^-1 K_aE)/V,
 *                           rel_res = |r| / max(|r| at the step's first
 *                           iteration, |Σ_raw| now, 1e-30), plastic counts and
 *                           status (5 = solver: singular K_αα)
 *   fe2_hrom_mono_commit    adopt the last iterate (α, history) as committed
 * The caller accepts a step when its macro residual and every rel_res are
 * below tolerance (fe2_macro_run with scheme = 1). */
int fe2_hrom_mono_begin(fe2_hrom_t h);
int fe2_hrom_mono_iterate(fe2_hrom_t h, const double* E, double* sigma, double* C, double* rel_res,
                          int* plastic_count, int* status);
/* The same on device buffers (E[P*3] in HBM; NULL outputs = the handle's own,
 * fe2_hrom_output_ptrs), asynchronous on `stream` (NULL = the handle's). */
int fe2_hrom_mono_iterate_device(fe2_hrom_t h, const double* d_E, double* d_sigma, double* d_C, double* d_rel_res,
                                 int* d_plastic_count, int* d_status, void* stream);
int fe2_hrom_mono_commit(fe2_hrom_t h);

/* ---- Empirical Cubature Method (SPEC.md:333-369
 * hyper.ecm_select), host only: U[m][k] = orthonormal integrand modes at the m
 * integration points (e.g. left singular vectors of the force snapshots),
 * w_full[m] = the full-rule weights. A constant column is appended (volume
 * exactness). Greedy max-correlation selection with least-squares re-fit and
 * removal of non-positive weights; stops at rel_residual <= tol or m_target
 * points (at most k + 1). ids/weights need min(m_target, k + 1) entries;
 * returned ids ascending, weights > 0. */
int fe2_ecm_select(const double* U, const double* w_full, int m, int k, int m_target, double tol, int* ids,
                   double* weights, int* m_out, double* rel_residual);

/* ---- offline stage (host only, no GPU): seeded hyper-ROM model and paths
 * matching BASELINE.json configs. */
typedef struct fe2_model_s* fe2_model_t;
/* default_cell(subdivisions) RVE (mesh.hpp:185-191, :218-352), linear BC,
 * n random orthonormal modes, K random cubature points (K = 0: the full rule,
 * every integration point with its own quadrature weight — ECM training). */
int fe2_model_build(int subdivisions, int n, int K, uint64_t seed, fe2_model_t* out);
/* The same on an RVE read from a plain-text mesh in the reference's format
 * (write_mesh / read_mesh, mesh.hpp:413-489: "fe2rom-mesh 1", nodes, Tri6
 * elements with material ids 0 = matrix / 1 = inclusion, node sets); the
 * linear BC acts on the nodes of the mesh's bounding box. */
int fe2_model_build_from_mesh(const char* path, int n, int K, uint64_t seed, fe2_model_t* out);
/* Write the default_cell(subdivisions) RVE in that format (bit-exact %.17g). */
int fe2_mesh_write(int subdivisions, const char* path);
void fe2_model_free(fe2_model_t m);
int fe2_model_sizes(fe2_model_t m, int* n, int* K, int* n_free, double* volume);
int fe2_model_arrays(fe2_model_t m, double* G, double* w, int* ip_id, int* mat_id);
/* G4[K][4][n]: the displacement-gradient operator of the same Φ and cubature */
int fe2_model_g4(fe2_model_t m, double* G4);
/* The same with a given basis (e.g. fe2_pod_basis) instead of the seeded Φ:
 * basis[n][n_dofs] column-major over ALL DOFs (mode j at basis + j * n_dofs,
 * the reference ReducedBasis::V); boundary rows are ignored.
 * mesh_path NULL selects default_cell(subdivisions). */
int fe2_model_build_basis(int subdivisions, const char* mesh_path, const double* basis, int n, int K, uint64_t seed,
                          fe2_model_t* out);

/* ---- high-fidelity RVE solve and POD basis ----------
 * fe2_hf_* is the full-field micro problem on the device: per-element
 * material update + element stiffness kernel, deterministic gather of the
 * free stiffness's lower band (free DOFs in reverse Cuthill-McKee order),
 * band Cholesky + substitutions on one CTA per system (the reference's
 * sparse SimplicialLDLT, rve.hpp:295-325). Replaces
 * micro_newton + homogenize + run_trajectory with SnapshotRecorder
 * (rve.hpp:285-392, :397-494; linear BC). */
/* RVE = default_cell(subdivisions) or mesh_path; materials indexed by the
 * element material id. */
int fe2_hf_create(int device, int subdivisions, const char* mesh_path, const fe2_material_t* materials, int n_materials,
                  fe2_hf_t* out);
void fe2_hf_destroy(fe2_hf_t h);
int fe2_hf_sizes(fe2_hf_t h, int* n_dofs, int* n_free, int* n_ips, double* volume);
/* run_trajectory from the virgin state along E[n_steps][3] (bisection,
 * warm start = committed solution + affine increment, rve.hpp:459-471).
 * Per step: sigma[3], C[9] (homogenize), Newton iterations (all attempts),
 * max |u - E.x|, last residual norm; snapshots (nullable) [n_steps][n_dofs]
 * = the converged fluctuation field u - E.x (the x_u column, rve.hpp:486-490).
 * Non-convergence after max_bisections -> solver error. */
int fe2_hf_trajectory(fe2_hf_t h, int n_steps, const double* E, const fe2_newton_opts_t* opts, double* sigma,
                      double* C, int* iterations, double* u_fluct_inf, double* res_last, double* snapshots);
/* A batch of independent trajectories (the POD training set):
 * trajectory t follows E[t][n_steps][3] from the virgin state; outputs as
 * fe2_hf_trajectory at offset t (sigma[t][k][3], C[t][k][9], iterations[t][k],
 * u_fluct_inf / res_last[t][k], snapshots[t][k][n_dofs]); status[t] = 0 or
 * 1 + ErrorCode of a failed trajectory (its later rows are unspecified).
 * Trajectories run concurrently (up to FE2_HF_WORKERS, default 64: one
 * stream and host thread each, one CTA per band factorisation). */
int fe2_hf_trajectories(fe2_hf_t h, int n_traj, int n_steps, const double* E, const fe2_newton_opts_t* opts,
                        double* sigma, double* C, int* iterations, double* u_fluct_inf, double* res_last,
                        double* snapshots, int* status);
/* Half bandwidth of the free stiffness in the device's band ordering. */
int fe2_hf_band(fe2_hf_t h, int* half_bandwidth);
/* HF engine of an FE² run (SPEC.md:474-477 HF_nested): P macro points, each
 * an RVE with its own committed state (virgin at allocation). One call = one
 * path step of run_trajectory for every point from its committed state
 * (bisection, warm start); Σ[P*3], C[P*9] (homogenize), iterations, status
 * (0, or 1 + ErrorCode when the point's step failed — it keeps its state).
 * snapshot / restore save and return to the committed states (deferred
 * commits, fe2_macro_run_hf). Points are solved concurrently (as fe2_hf_trajectories). */
int fe2_hf_alloc_points(fe2_hf_t h, int64_t P);
int fe2_hf_points(fe2_hf_t h, int64_t* P);
int fe2_hf_solve_increment(fe2_hf_t h, const double* E, const fe2_newton_opts_t* opts, double* sigma, double* C,
                           int* iters, int* status);
int fe2_hf_snapshot(fe2_hf_t h);
/* HF_monolithic: one condensed full-field Newton iteration of
 * every point per call — the fluctuation moves by the previous iteration's
 * linearisation, w <- w - K^-1 (r + K_fE dE), the point is assembled at (E, w)
 * from its committed states, and Σ~ = (Σ_raw - K_Ef K^-1 r)/V,
 * C = (C_EE - K_Ef K^-1 K_fE)/V and the relative micro residual
 * |r| / max(|r_first|, |reactions|) are returned (status 0 or 1 + ErrorCode).
 * begin starts a step from the committed state; commit adopts the last iterate.
 * The same algebra as fe2_hrom_mono_* on the full field (Φ = identity). */
int fe2_hf_mono_begin(fe2_hf_t h);
int fe2_hf_mono_iterate(fe2_hf_t h, const double* E, double* sigma, double* C, double* rel_res, int* status);
int fe2_hf_mono_commit(fe2_hf_t h);
int fe2_hf_restore(fe2_hf_t h);
/* build_elastic_modes: fluctuation responses of the
 * elastic RVE (every material's elastic part) to unit macro strains
 * (1,0,0),(0,1,0),(0,0,1), orthonormalised (Gram-Schmidt, twice); modes whose
 * remaining norm is <= 1e-10 |E.x| are dropped (homogeneous RVE -> 0 modes).
 * modes[3][n_dofs] column-major; *count = modes kept. */
int fe2_hf_elastic_modes(fe2_hf_t h, double* modes, int* count);
/* pod: V = [elastic | leading left singular vectors of X
 * deflated against the elastic modes], re-orthonormalised. X[n_cols][n_rows]
 * and elastic[n_elastic][n_rows] column-major; V[n_target][n_rows]. Deflated
 * singular values (descending, n_cols of them) go to singular_values; a POD
 * mode's largest-magnitude entry is positive. Deflated rank counts singular
 * values > 1e-10 |X|_F; n_target > n_elastic + rank -> rank error with
 * *max_modes = n_elastic + rank. SVD on the device (cuSOLVER gesvd). */
int fe2_pod_basis(int device, const double* X, int64_t n_rows, int n_cols, const double* elastic, int n_elastic,
                  int n_target, double* V, double* singular_values, int* max_modes);

/* path kind 0 = config-0 uniaxial rotated, 1 = config-1 reversal:
 * E[P][n_incr][3]; kind 2 = config-2 finite strain: H[P][n_incr][4]
 * (F = I + (k/n_incr) H_end, H_end ~ U[-0.08, 0.08]^4 with det F > 0.8),
 * for global points p0..p0+P-1 */
int fe2_paths(int kind, uint64_t seed, int64_t p0, int64_t P, int n_incr, double* E);

#ifdef __cplusplus
}
#endif
#endif
