// fe2rom/hrom_gpu.hpp — header-only C++ mirror of the reference fe2rom
// interface over the B200 C ABI (fe2rom_gpu.h). Eigen-free, so a caller of
// /root/reference/proj/include/fe2rom can switch the per-macro-point RVE
// solve to the GPU batch without other dependencies.
//
// Reference names kept (paths relative to /root/reference/proj/include/fe2rom/):
//   ElasticParams, J2LinearParams, PowerLawParams,
//   CreepParams, Material                          materials.hpp:37-78
//   MaterialState (eps_p[4], eq, sigma33)          materials.hpp:102-106
//   MicroOptions {tol, max_iter}                   rve.hpp:195-200
//   TrajectoryOptions {micro, max_bisections}      rve.hpp:439-443
//   HomogenizedResponse {sigma, tangent}           rve.hpp:37-40
//   Error / ErrorCode                              common.hpp:26-52
//   update_material (batched)                      materials.hpp:317-325
// HyperRomBatch::solve_increment is run_trajectory's per-step body
// (rve.hpp:459-491) — micro_newton + homogenize + commit — for a batch of
// macro Gauss points with a hyper-reduced RVE model.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <variant>
#include <cmath>
#include <vector>

#include "fe2rom/fe2rom_gpu.h"

namespace fe2rom::gpu {

enum class ErrorCode { config, geometry, mesh, material, solver, numeric, rank, bc, io, provenance };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode c, const std::string& what) : std::runtime_error(what), code_(c) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

inline void check(int rc) {
  if (rc != 0) throw Error(static_cast<ErrorCode>(rc - 1), fe2_last_error());
}

using Voigt3 = std::array<double, 3>;  // (e11, e22, g12) / (s11, s22, s12)
using Mat3 = std::array<double, 9>;    // row-major

struct ElasticParams {
  double E = 1.0;
  double nu = 0.3;
};
struct J2LinearParams {
  ElasticParams elastic;
  double sigma_y0 = 0.01;
  double hardening = 0.016;
};
struct PowerLawParams {  // materials.hpp:51-65
  double E = 1.0;
  double nu = 0.3;
  double sigma_y0 = 0.01;
  double N = 0.1;
};
struct CreepParams {  // materials.hpp:67-76; dt = time of one load increment
  double E = 1.0;
  double nu = 0.14;
  double A = 22.09;
  double n = 1.06;
  double m = -0.56;
  double dt = 1.0;
};
using Material = std::variant<ElasticParams, J2LinearParams, PowerLawParams, CreepParams>;

struct MaterialState {
  std::array<double, 4> eps_p{0, 0, 0, 0};
  double eq = 0.0;
  double sigma33 = 0.0;
};

struct MicroOptions {
  double tol = 1e-8;
  int max_iter = 30;
};
struct TrajectoryOptions {
  MicroOptions micro;
  int max_bisections = 4;
};

struct HomogenizedResponse {
  Voigt3 sigma{};
  Mat3 tangent{};
  int iterations = 0;      // all Newton iterations of the increment
  int plastic_points = 0;  // cubature points with f > 0 at the commit
  double residual = 0.0;
  int status = 0;          // 0 or 1 + ErrorCode
};

inline fe2_material_t to_c(const Material& m) {
  fe2_material_t c{};
  if (auto* e = std::get_if<ElasticParams>(&m)) {
    c.kind = 0;
    c.p[0] = e->E;
    c.p[1] = e->nu;
  } else if (auto* j = std::get_if<J2LinearParams>(&m)) {
    c.kind = 1;
    c.p[0] = j->elastic.E;
    c.p[1] = j->elastic.nu;
    c.p[2] = j->sigma_y0;
    c.p[3] = j->hardening;
  } else if (auto* pl = std::get_if<PowerLawParams>(&m)) {
    c.kind = 2;
    c.p[0] = pl->E;
    c.p[1] = pl->nu;
    c.p[2] = pl->sigma_y0;
    c.p[3] = pl->N;
  } else {
    const auto& cr = std::get<CreepParams>(m);
    c.kind = 3;
    c.p[0] = cr.E;
    c.p[1] = cr.nu;
    c.p[2] = cr.A;
    c.p[3] = cr.n;
    c.p[4] = cr.m;
    c.p[5] = cr.dt;
  }
  return c;
}

struct MaterialResult {
  Voigt3 sigma{};
  Mat3 tangent{};
  MaterialState state;
  bool plastic = false;
};

// Batched update_material on the device (materials.hpp:317-325).
inline std::vector<MaterialResult> update_material(const Material& mat, const std::vector<MaterialState>& s0,
                                                   const std::vector<Voigt3>& eps, int device = 0) {
  const int64_t N = static_cast<int64_t>(eps.size());
  std::vector<double> e(3 * N), st(6 * N), sig(3 * N), C(9 * N), so(6 * N);
  std::vector<uint8_t> pl(N);
  for (int64_t i = 0; i < N; ++i) {
    for (int c = 0; c < 3; ++c) e[3 * i + c] = eps[i][c];
    const MaterialState& s = s0.empty() ? MaterialState{} : s0[i];
    for (int c = 0; c < 4; ++c) st[6 * i + c] = s.eps_p[c];
    st[6 * i + 4] = s.eq;
    st[6 * i + 5] = s.sigma33;
  }
  const fe2_material_t m = to_c(mat);
  check(fe2_material_update_batch(device, &m, N, e.data(), st.data(), sig.data(), C.data(), so.data(), pl.data()));
  std::vector<MaterialResult> out(N);
  for (int64_t i = 0; i < N; ++i) {
    for (int c = 0; c < 3; ++c) out[i].sigma[c] = sig[3 * i + c];
    for (int c = 0; c < 9; ++c) out[i].tangent[c] = C[9 * i + c];
    for (int c = 0; c < 4; ++c) out[i].state.eps_p[c] = so[6 * i + c];
    out[i].state.eq = so[6 * i + 4];
    out[i].state.sigma33 = so[6 * i + 5];
    out[i].plastic = pl[i] != 0;
  }
  return out;
}

// A batch of macro Gauss points sharing one hyper-reduced RVE model on one
// device: G[K][3][n] (G_q = B_q Φ), cubature weights, material per point.
class HyperRomBatch {
 public:
  HyperRomBatch(int device, int n, int K, const std::vector<double>& G, const std::vector<double>& w,
                const std::vector<int>& mat_id, const std::vector<Material>& materials, double volume)
      : n_(n), K_(K) {
    std::vector<fe2_material_t> mc;
    for (const auto& m : materials) mc.push_back(to_c(m));
    check(fe2_hrom_create(device, n, K, G.data(), w.data(), mat_id.data(), mc.data(), static_cast<int>(mc.size()),
                          volume, &h_));
  }
  ~HyperRomBatch() { fe2_hrom_destroy(h_); }
  HyperRomBatch(const HyperRomBatch&) = delete;
  HyperRomBatch& operator=(const HyperRomBatch&) = delete;

  // virgin states (std::vector<MaterialState>(n_ips), rve.hpp:450) for P points
  void alloc_points(int64_t P, bool keep_flags = false) {
    check(fe2_hrom_alloc_points(h_, P, keep_flags ? 1 : 0));
    P_ = P;
  }

  // one path step for every point: E[p] is this increment's macro strain
  std::vector<HomogenizedResponse> solve_increment(const std::vector<Voigt3>& E, const TrajectoryOptions& o = {}) {
    if (static_cast<int64_t>(E.size()) != P_) throw Error(ErrorCode::config, "one macro strain per point");
    std::vector<double> e(3 * P_), sig(3 * P_), C(9 * P_), res(P_);
    std::vector<int> it(P_), pc(P_), st(P_);
    for (int64_t p = 0; p < P_; ++p)
      for (int c = 0; c < 3; ++c) e[3 * p + c] = E[p][c];
    const fe2_newton_opts_t opts{o.micro.tol, o.micro.max_iter, o.max_bisections};
    check(fe2_hrom_solve_increment(h_, e.data(), &opts, sig.data(), C.data(), it.data(), pc.data(), res.data(),
                                   st.data()));
    std::vector<HomogenizedResponse> out(P_);
    for (int64_t p = 0; p < P_; ++p) {
      for (int c = 0; c < 3; ++c) out[p].sigma[c] = sig[3 * p + c];
      for (int c = 0; c < 9; ++c) out[p].tangent[c] = C[9 * p + c];
      out[p].iterations = it[p];
      out[p].plastic_points = pc[p];
      out[p].residual = res[p];
      out[p].status = st[p];
    }
    return out;
  }

  // committed MaterialState of every cubature point of point p
  std::vector<MaterialState> states(int64_t p) const {
    std::vector<double> a(static_cast<size_t>(P_) * n_), s(static_cast<size_t>(P_) * K_ * 6);
    check(fe2_hrom_read_state(h_, a.data(), s.data(), nullptr));
    std::vector<MaterialState> out(K_);
    for (int q = 0; q < K_; ++q) {
      const double* x = s.data() + (static_cast<size_t>(p) * K_ + q) * 6;
      for (int c = 0; c < 4; ++c) out[q].eps_p[c] = x[c];
      out[q].eq = x[4];
      out[q].sigma33 = x[5];
    }
    return out;
  }

  fe2_hrom_t handle() const { return h_; }

  // Multi-GPU exchange (one batch per rank and device, any P per rank):
  // all-gather every rank's {Σ (3) | C_macro (9) | ‖r‖ | status} records of
  // the last increment into the device buffer d_all [world][P_max][14]
  // (P_max from gather_layout; padding rows have status -1); returns true if
  // a point failed on any rank. See fe2_hrom_gather.
  bool gather(void* nccl_comm, double* d_all) {
    int flags[2] = {0, 0};
    check(fe2_hrom_gather(h_, nccl_comm, nullptr, nullptr, nullptr, nullptr, HUGE_VAL, d_all, flags));
    return flags[0] != 0;
  }
  // Rows per rank block of the gathered buffer (max point count over the ranks).
  int64_t gather_layout(void* nccl_comm, std::vector<int64_t>* counts = nullptr) {
    int64_t p_max = 0;
    std::vector<int64_t> c(64);
    check(fe2_hrom_gather_layout(h_, nccl_comm, &p_max, c.data()));
    if (counts) *counts = c;
    return p_max;
  }

 private:
  fe2_hrom_t h_ = nullptr;
  int n_ = 0, K_ = 0;
  int64_t P_ = 0;
};

// One NCCL communicator per rank and device (fe2_nccl_comm_init); rank 0
// creates the id with unique_id() and the caller broadcasts its 128 bytes.
class NcclComm {
 public:
  using Id = std::array<unsigned char, 128>;
  static Id unique_id() {
    Id id{};
    check(fe2_nccl_get_unique_id(id.data()));
    return id;
  }
  NcclComm(int device, int nranks, int rank, const Id& id) { check(fe2_nccl_comm_init(device, nranks, rank, id.data(), &c_)); }
  ~NcclComm() { fe2_nccl_comm_destroy(c_); }
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  void* get() const { return c_; }

 private:
  void* c_ = nullptr;
};

// Finite-strain (Biot stress) response of one macro point: first
// Piola-Kirchhoff stress P (F00, F01, F10, F11) and A = dP/dF row-major.
struct FiniteStrainResponse {
  std::array<double, 4> P{};
  std::array<double, 16> A{};
  int iterations = 0;
  int plastic_points = 0;
  double residual = 0.0;
  int status = 0;
};

// BASELINE config 2: G4[K][4][n] displacement-gradient operator (n <= 32);
// each increment takes H = F - I per point. No reference counterpart.
class FiniteStrainBatch {
 public:
  FiniteStrainBatch(int device, int n, int K, const std::vector<double>& G4, const std::vector<double>& w,
                    const std::vector<int>& mat_id, const std::vector<Material>& materials, double volume) {
    std::vector<fe2_material_t> mc;
    for (const auto& m : materials) mc.push_back(to_c(m));
    check(fe2_hrom_create_fs(device, n, K, G4.data(), w.data(), mat_id.data(), mc.data(),
                             static_cast<int>(mc.size()), volume, &h_));
  }
  ~FiniteStrainBatch() { fe2_hrom_destroy(h_); }
  FiniteStrainBatch(const FiniteStrainBatch&) = delete;
  FiniteStrainBatch& operator=(const FiniteStrainBatch&) = delete;

  void alloc_points(int64_t P) {
    check(fe2_hrom_alloc_points(h_, P, 0));
    P_ = P;
  }

  std::vector<FiniteStrainResponse> solve_increment(const std::vector<std::array<double, 4>>& H,
                                                    const TrajectoryOptions& o = {}) {
    if (static_cast<int64_t>(H.size()) != P_) throw Error(ErrorCode::config, "one displacement gradient per point");
    std::vector<double> h(4 * P_), Pm(4 * P_), A(16 * P_), res(P_);
    std::vector<int> it(P_), pc(P_), st(P_);
    for (int64_t p = 0; p < P_; ++p)
      for (int c = 0; c < 4; ++c) h[4 * p + c] = H[p][c];
    const fe2_newton_opts_t opts{o.micro.tol, o.micro.max_iter, o.max_bisections};
    check(fe2_hrom_solve_increment(h_, h.data(), &opts, Pm.data(), A.data(), it.data(), pc.data(), res.data(),
                                   st.data()));
    std::vector<FiniteStrainResponse> out(P_);
    for (int64_t p = 0; p < P_; ++p) {
      for (int c = 0; c < 4; ++c) out[p].P[c] = Pm[4 * p + c];
      for (int c = 0; c < 16; ++c) out[p].A[c] = A[16 * p + c];
      out[p].iterations = it[p];
      out[p].plastic_points = pc[p];
      out[p].residual = res[p];
      out[p].status = st[p];
    }
    return out;
  }

  fe2_hrom_t handle() const { return h_; }

 private:
  fe2_hrom_t h_ = nullptr;
  int64_t P_ = 0;
};

}  // namespace fe2rom::gpu
