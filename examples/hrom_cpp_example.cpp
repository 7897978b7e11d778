// Minimal C++ caller of the B200 engine through the reference-style wrapper:
// builds the config-0 hyper-ROM model (offline stage of the library), runs a
// few increments for a handful of macro points and prints Σ and C_macro.
#include <cstdio>
#include <vector>

#include "fe2rom/hrom_gpu.hpp"

int main(int argc, char** argv) {
  const int P = argc > 1 ? std::atoi(argv[1]) : 4, n_incr = 5;
  fe2_model_t m = nullptr;
  fe2rom::gpu::check(fe2_model_build(33, 12, 200, 0, &m));
  int n = 0, K = 0, nf = 0;
  double vol = 0.0;
  fe2rom::gpu::check(fe2_model_sizes(m, &n, &K, &nf, &vol));
  std::vector<double> G(static_cast<size_t>(K) * 3 * n), w(K);
  std::vector<int> ip(K), mat(K);
  fe2rom::gpu::check(fe2_model_arrays(m, G.data(), w.data(), ip.data(), mat.data()));
  fe2_model_free(m);
  std::vector<double> E(static_cast<size_t>(P) * n_incr * 3);
  fe2rom::gpu::check(fe2_paths(0, 0, 0, P, n_incr, E.data()));
  try {
    fe2rom::gpu::HyperRomBatch batch(0, n, K, G, w, mat,
                                     {fe2rom::gpu::J2LinearParams{}, fe2rom::gpu::ElasticParams{10.0, 0.3}}, vol);
    batch.alloc_points(P);
    for (int k = 0; k < n_incr; ++k) {
      std::vector<fe2rom::gpu::Voigt3> Ek(P);
      for (int p = 0; p < P; ++p)
        for (int c = 0; c < 3; ++c) Ek[p][c] = E[(static_cast<size_t>(p) * n_incr + k) * 3 + c];
      const auto r = batch.solve_increment(Ek);
      std::printf("increment %d point 0: sigma = (%.6e, %.6e, %.6e) C11 = %.6e iters = %d plastic = %d\n", k + 1,
                  r[0].sigma[0], r[0].sigma[1], r[0].sigma[2], r[0].tangent[0], r[0].iterations,
                  r[0].plastic_points);
      for (int p = 0; p < P; ++p) {  // machine-readable: every point, full precision
        std::printf("R %d %d %d", k, p, r[p].iterations);
        for (int c = 0; c < 3; ++c) std::printf(" %.17g", r[p].sigma[c]);
        for (int c = 0; c < 9; ++c) std::printf(" %.17g", r[p].tangent[c]);
        std::printf("\n");
      }
    }
    // finite strain (config 2 kinematics) on the same model: G4 and H = F - I paths
    fe2_model_t m4 = nullptr;
    fe2rom::gpu::check(fe2_model_build(33, 12, 200, 0, &m4));
    std::vector<double> G4(static_cast<size_t>(K) * 4 * n), H(static_cast<size_t>(P) * n_incr * 4);
    fe2rom::gpu::check(fe2_model_g4(m4, G4.data()));
    fe2_model_free(m4);
    fe2rom::gpu::check(fe2_paths(2, 0, 0, P, n_incr, H.data()));
    fe2rom::gpu::FiniteStrainBatch fs(0, n, K, G4, w, mat,
                                      {fe2rom::gpu::J2LinearParams{}, fe2rom::gpu::ElasticParams{10.0, 0.3}}, vol);
    fs.alloc_points(P);
    for (int k = 0; k < n_incr; ++k) {
      std::vector<std::array<double, 4>> Hk(P);
      for (int p = 0; p < P; ++p)
        for (int c = 0; c < 4; ++c) Hk[p][c] = H[(static_cast<size_t>(p) * n_incr + k) * 4 + c];
      const auto r = fs.solve_increment(Hk);
      std::printf("finite-strain increment %d point 0: P = (%.6e, %.6e, %.6e, %.6e) A00 = %.6e iters = %d\n", k + 1,
                  r[0].P[0], r[0].P[1], r[0].P[2], r[0].P[3], r[0].A[0], r[0].iterations);
      for (int p = 0; p < P; ++p) {
        std::printf("F %d %d %d", k, p, r[p].iterations);
        for (int c = 0; c < 4; ++c) std::printf(" %.17g", r[p].P[c]);
        for (int c = 0; c < 16; ++c) std::printf(" %.17g", r[p].A[c]);
        std::printf("\n");
      }
    }
  } catch (const fe2rom::gpu::Error& e) {
    std::printf("fe2rom::gpu::Error code=%d: %s\n", static_cast<int>(e.code()), e.what());
    return e.code() == fe2rom::gpu::ErrorCode::numeric ? 2 : 1;
  }
  return 0;
}
