// Golden-fixture generator: runs the REFERENCE's own code
// (/root/reference/proj/include/fe2rom/{common,materials,mesh,rve}.hpp, compiled unmodified
// against the Eigen-API shim in oracle/refshim) on seeded inputs and writes .npy fixtures.
//
// TEST INFRASTRUCTURE ONLY. Built into oracle/_ref/ by `make -C oracle ref` (needs
// /root/reference, i.e. only in the build container); its outputs are committed under
// tests/golden/ by oracle/make_golden.py, which is the only caller.
//
// Fixtures (all float64 unless noted):
//   mat_<name>.npy        [N, 27]: eps(3) | state_in(6: eps_p 4, eq, sigma33) | sigma(3) |
//                         C(9, row-major) | state_out(6)      update_material (materials.hpp:317-325)
//   mesh<s>_xy.npy        [n_nodes, 2]                        build_rve_mesh(default_cell(s)) (mesh.hpp:218-352)
//   mesh<s>_conn.npy      int32 [n_el, 7]: 6 nodes | material id
//   mesh<s>_ip.npy        [n_ips, 37]: B (3x12 row-major) | weight        build_rve_problem (rve.hpp:167-185)
//   mesh<s>_meta.npy      [3]: area, n_free (linear BC), volume
//   mesh<s>_text.txt      the mesh in the reference's text format (write_mesh, mesh.hpp:413-431)
//   hf_<case>.npy         [steps, 1 + 3 + 9]: iterations | sigma | C_hom   run_trajectory semantics
//                         (rve.hpp:448-494) with micro_newton (:285-346) + homogenize (:350-392)
//   hf_<case>_states.npy  [n_ips, 6] committed states returned by run_trajectory itself
//   hf_<case>_xu.npy      [steps, n_dofs] its SnapshotRecorder columns (rve.hpp:485-489)
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "fe2rom/rve.hpp"

using namespace fe2rom;

namespace {

std::string g_out;

void write_npy(const std::string& name, const char* descr, const void* data, size_t elem, std::vector<long> shape) {
  std::string sh = "(";
  for (size_t i = 0; i < shape.size(); ++i) sh += std::to_string(shape[i]) + (shape.size() == 1 || i + 1 < shape.size() ? "," : "");
  sh += ")";
  std::string hdr = std::string("{'descr': '") + descr + "', 'fortran_order': False, 'shape': " + sh + ", }";
  const size_t base = 10 + hdr.size() + 1;
  hdr += std::string((64 - base % 64) % 64, ' ') + "\n";
  FILE* f = std::fopen((g_out + "/" + name).c_str(), "wb");
  if (!f) fail(ErrorCode::io, "cannot write " + name);
  const unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  std::fwrite(magic, 1, 8, f);
  const unsigned short hl = static_cast<unsigned short>(hdr.size());
  std::fwrite(&hl, 2, 1, f);
  std::fwrite(hdr.data(), 1, hdr.size(), f);
  long n = 1;
  for (long s : shape) n *= s;
  std::fwrite(data, elem, static_cast<size_t>(n), f);
  std::fclose(f);
}
void write_f64(const std::string& name, const std::vector<double>& v, std::vector<long> shape) {
  write_npy(name, "<f8", v.data(), 8, std::move(shape));
}

std::vector<Material> desk_materials(int matrix_kind) {
  // the reference's desk RVE (test_rve.cpp:9-17): J2 matrix + stiff elastic inclusions;
  // matrix_kind 1/2 swaps the matrix for the power-law / creep model (materials.hpp:51-76)
  Material matrix = J2LinearParams{{1.0, 0.3}, 0.01, 0.016};
  if (matrix_kind == 1) matrix = PowerLawParams{1.0, 0.3, 0.01, 0.1};
  if (matrix_kind == 2) matrix = CreepParams{};
  return {matrix, Material(ElasticParams{10.0, 0.3})};
}

void push_state(std::vector<double>& row, const MaterialState& s) {
  for (int i = 0; i < 4; ++i) row.push_back(s.eps_p[i]);
  row.push_back(s.eq);
  row.push_back(s.sigma33);
}

// update_material on N seeded (state, strain) pairs. States come from 0-3 committed random
// pre-strain steps of the same model, so they are reachable histories (deviatoric eps_p,
// eq consistent with it); the final strain is scaled so both branches occur.
void materials_fixture(const std::string& name, const Material& mat, double dt, int N, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<double> out;
  out.reserve(static_cast<size_t>(N) * 27);
  for (int c = 0; c < N; ++c) {
    MaterialState s;
    const int pre = rng.uniform_int(4);
    for (int k = 0; k < pre; ++k) {
      const Voigt3 e(rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(-0.05, 0.05));
      s = update_material(mat, s, e, dt).state;
    }
    const double scale = rng.uniform() < 0.3 ? 0.004 : 1.0;
    const Voigt3 eps(scale * rng.uniform(-0.03, 0.03), scale * rng.uniform(-0.03, 0.03),
                     scale * rng.uniform(-0.05, 0.05));
    const MaterialResult r = update_material(mat, s, eps, dt);
    std::vector<double> row;
    for (int i = 0; i < 3; ++i) row.push_back(eps[i]);
    push_state(row, s);
    for (int i = 0; i < 3; ++i) row.push_back(r.sigma[i]);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) row.push_back(r.tangent(i, j));
    push_state(row, r.state);
    out.insert(out.end(), row.begin(), row.end());
  }
  write_f64("mat_" + name + ".npy", out, {N, 27});
}

void mesh_fixture(int s) {
  const RveProblem p = build_rve_problem(build_rve_mesh(RveGeometry::default_cell(s)), desk_materials(0));
  std::vector<double> xy;
  for (const auto& nd : p.mesh.nodes) {
    xy.push_back(nd.x);
    xy.push_back(nd.y);
  }
  std::vector<int> conn;
  for (const auto& el : p.mesh.elements) {
    for (int a = 0; a < 6; ++a) conn.push_back(el.nodes[a]);
    conn.push_back(el.material_id);
  }
  std::vector<double> ip;
  for (const auto& d : p.ips) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 12; ++j) ip.push_back(d.B(i, j));
    ip.push_back(d.weight);
  }
  const DofMap dm = apply_macro_strain(p.mesh, MacroStrain(), BcKind::linear);
  const std::string pre = "mesh" + std::to_string(s) + "_";
  write_f64(pre + "xy.npy", xy, {p.mesh.n_nodes(), 2});
  write_npy(pre + "conn.npy", "<i4", conn.data(), 4, {p.mesh.n_elements(), 7});
  write_f64(pre + "ip.npy", ip, {p.n_ips(), 37});
  write_f64(pre + "meta.npy", {p.mesh.area, static_cast<double>(dm.n_free), p.volume}, {3});
  std::ofstream os(g_out + "/" + pre + "text.txt", std::ios::binary);  // write_mesh (mesh.hpp:413-431)
  write_mesh(p.mesh, os);
}

// One trajectory, two ways: (1) the per-step loop of run_trajectory (rve.hpp:459-491:
// bisection, warm start, commit) calling the reference's micro_newton and homogenize to
// record iterations, Sigma and C_hom per step; (2) run_trajectory itself, whose committed
// states and snapshot columns must equal (1)'s.
void hf_fixture(const std::string& name, int s, int matrix_kind, const std::vector<Voigt3>& E_path, double dt,
                int max_iter) {
  const RveProblem p = build_rve_problem(build_rve_mesh(RveGeometry::default_cell(s)), desk_materials(matrix_kind));
  TrajectoryOptions topts;
  topts.micro.max_iter = max_iter;
  std::vector<PathStep> path;
  for (const auto& e : E_path) path.push_back({MacroStrain(e), dt});

  std::vector<double> rows;
  std::vector<double> xu_loop;
  std::vector<MaterialState> states(p.n_ips());
  DofMap dm = apply_macro_strain(p.mesh, MacroStrain(), BcKind::linear);
  Vec u_free = Vec::Zero(dm.n_free);
  MacroStrain E_prev, E_committed;
  for (std::size_t k = 0; k < path.size(); ++k) {
    double done = 0.0, frac = 1.0;
    int bisections = 0, iters = 0;
    while (done < 1.0 - 1e-12) {
      const double target = std::min(1.0, done + frac);
      MacroStrain E(Voigt3(E_prev.voigt + (path[k].E.voigt - E_prev.voigt) * target));
      set_macro_strain(dm, p.mesh, E);
      MicroOptions mo = topts.micro;
      mo.dt = path[k].dt * (target - done);
      const Vec u_start =
          u_free + affine_free_start(p.mesh, dm, MacroStrain(Voigt3(E.voigt - E_committed.voigt)));
      auto res = micro_newton(p, dm, states, u_start, mo);
      iters += res.iterations;
      if (!res.converged) {
        require(++bisections <= topts.max_bisections, ErrorCode::solver, "fixture path " + name + " failed at step " + std::to_string(k));
        frac *= 0.5;
        continue;
      }
      states = res.states;
      for (int i = 0; i < dm.n_total(); ++i)
        if (dm.dofs[i].kind == DofKind::free) u_free[dm.dofs[i].free_index] = res.u_full[i];
      E_committed = E;
      done = target;
      if (done >= 1.0 - 1e-12) {
        const HomogenizedResponse h = homogenize(p, dm, res);
        rows.push_back(iters);
        for (int i = 0; i < 3; ++i) rows.push_back(h.sigma[i]);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) rows.push_back(h.tangent(i, j));
        const Vec w = res.u_full - affine_field(p.mesh, E);
        for (int i = 0; i < w.size(); ++i) xu_loop.push_back(w[i]);
      }
    }
    E_prev = path[k].E;
  }

  SnapshotRecorder rec;
  const auto final_states = run_trajectory(p, BcKind::linear, path, std::vector<MaterialState>(p.n_ips()), &rec, topts);
  const Mat X = rec.matrix();
  std::vector<double> xu, st;
  for (int c = 0; c < X.cols(); ++c)
    for (int i = 0; i < X.rows(); ++i) xu.push_back(X(i, c));
  require(xu == xu_loop, ErrorCode::numeric, "run_trajectory snapshots differ from the per-step loop");
  for (std::size_t i = 0; i < final_states.size(); ++i) {
    require(final_states[i].eq == states[i].eq, ErrorCode::numeric, "run_trajectory states differ");
    std::vector<double> row;
    push_state(row, final_states[i]);
    st.insert(st.end(), row.begin(), row.end());
  }
  write_f64("hf_" + name + ".npy", rows, {static_cast<long>(path.size()), 13});
  write_f64("hf_" + name + "_states.npy", st, {p.n_ips(), 6});
  write_f64("hf_" + name + "_xu.npy", xu, {static_cast<long>(path.size()), p.mesh.n_dofs()});
}

std::vector<Voigt3> uniaxial_path(double s, double theta, int n) {  // config-0 shape
  std::vector<Voigt3> v;
  const double c = std::cos(theta), sn = std::sin(theta);
  for (int k = 1; k <= n; ++k) {
    const double f = 0.05 * s * k / n;
    v.emplace_back(f * c * c, f * sn * sn, f * 2.0 * sn * c);
  }
  return v;
}
std::vector<Voigt3> reversal_path(double a, double b, int n) {  // config-1 shape: load, then back to 0
  std::vector<Voigt3> v;
  for (int k = 1; k <= n; ++k) {
    const double f = k <= n / 2 ? double(k) / (n / 2) : double(n - k) / (n / 2);
    v.emplace_back(f * a, 0.0, f * 2.0 * b);
  }
  return v;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_golden OUT_DIR [--big]\n");
    return 2;
  }
  g_out = argv[1];
  const bool big = argc > 2 && std::strcmp(argv[2], "--big") == 0;
  try {
    if (big) {  // default_cell(33): hashed by make_golden.py, not committed
      mesh_fixture(33);
      return 0;
    }
    const int N = 512;
    materials_fixture("j2", J2LinearParams{{1.0, 0.3}, 0.01, 0.016}, 1.0, N, 101);
    materials_fixture("elastic", ElasticParams{10.0, 0.3}, 1.0, N, 102);
    materials_fixture("powerlaw", PowerLawParams{1.0, 0.3, 0.01, 0.1}, 1.0, N, 103);
    materials_fixture("creep", CreepParams{}, 0.05, N, 104);
    for (int s : {6, 8}) mesh_fixture(s);
    hf_fixture("c6_uniaxial", 6, 0, uniaxial_path(1.2, 0.4, 10), 0.1, 30);
    hf_fixture("c6_reversal", 6, 0, reversal_path(0.03, -0.015, 12), 1.0 / 12, 30);
    hf_fixture("c6_bisect", 6, 0, {Voigt3(0.03, -0.01, 0.02), Voigt3(0.05, -0.02, 0.04)}, 0.5, 5);
    hf_fixture("c8_uniaxial", 8, 0, uniaxial_path(0.9, 1.1, 8), 0.125, 30);
    hf_fixture("c6_powerlaw", 6, 1, uniaxial_path(1.0, 0.2, 8), 0.125, 30);
    hf_fixture("c6_creep", 6, 2, uniaxial_path(1.0, 0.7, 8), 0.125, 30);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_golden: %s\n", e.what());
    return 1;
  }
  return 0;
}
