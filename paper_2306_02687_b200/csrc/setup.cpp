// Offline stage of the hyper-ROM model (host C++, no GPU): the unit-cell RVE
// mesh, the per-integration-point strain operators, a seeded orthonormal
// fluctuation basis Φ, a seeded cubature rule, and the projected operators
// G_q = B_q Φ that the device kernels contract. This is the input generator
// for BASELINE.json's configs; the online path never calls back into it.
//
// Reference behaviour followed (paths relative to
// /root/reference/proj/include/fe2rom/):
//   RveGeometry::default_cell           mesh.hpp:185-191
//   build_rve_mesh (snap, mid-edge, pore) mesh.hpp:218-352
//   tri6 gradients / shape_eval          mesh.hpp:67-115 ; tri3 rule :33-38
//   linear BC (boundary DOFs fixed)      rve.hpp:84-92 ; free numbering :122-124
//   IpData weight = w_g * detJ           rve.hpp:178-181
//   Rng (mt19937_64, uniform, normal)    common.hpp:56-88
// Seeded choices the reference leaves open (Φ, cubature, paths) are the
// DESIGN.md "Inputs" decisions; tests/test_setup.py checks this builder
// against the independent CPU oracle bit for bit.
#include "fe2rom/fe2rom_gpu.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "common.hpp"
#include "rve.hpp"

namespace fe2 {

namespace {

class SeededStream {  // common.hpp:56-88
 public:
  explicit SeededStream(std::uint64_t seed) : mt_(seed) {}
  double unit() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }
  double in(double lo, double hi) { return lo + (hi - lo) * unit(); }
  int below(int n) { return std::min(n - 1, static_cast<int>(unit() * n)); }
  double gauss() {
    if (cached_) {
      cached_ = false;
      return spare_;
    }
    double u1 = unit();
    while (u1 <= 1e-300) u1 = unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * std::numbers::pi * unit();
    spare_ = rad * std::sin(ang);
    cached_ = true;
    return rad * std::cos(ang);
  }

 private:
  std::mt19937_64 mt_;
  double spare_ = 0.0;
  bool cached_ = false;
};

constexpr std::uint64_t kPhiStream = 0x243F6A8885A308D3ull;
constexpr std::uint64_t kRuleStream = 0x13198A2E03707344ull;
constexpr std::uint64_t kPathStream = 0xA4093822299F31D0ull;

std::uint64_t mix64(std::uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Disc {
  double cx, cy, rad;
  double distance(double x, double y) const { return std::hypot(x - cx, y - cy); }
};

struct Cell {  // unit-cell mesh
  std::vector<double> x, y;           // nodes
  std::vector<std::array<int, 6>> tri;
  std::vector<int> phase;             // 0 matrix, 1 inclusion
  std::vector<char> on_boundary;      // node lies on the cell boundary
  double area = 0.0;
};

// Element strain operator at reference point (xi, eta): returns detJ and
// writes the 3x12 operator rows (dN/dx, dN/dy interleaved per node).
double strain_operator(const Cell& c, const std::array<int, 6>& t, double xi, double eta, double Bop[3][12]) {
  const double l1 = 1.0 - xi - eta, l2 = xi, l3 = eta;
  const double g[6][2] = {{-(4.0 * l1 - 1.0), -(4.0 * l1 - 1.0)},
                          {4.0 * l2 - 1.0, 0.0},
                          {0.0, 4.0 * l3 - 1.0},
                          {4.0 * (l1 - l2), -4.0 * l2},
                          {4.0 * l3, 4.0 * l2},
                          {-4.0 * l3, 4.0 * (l1 - l3)}};
  double j00 = 0.0, j01 = 0.0, j10 = 0.0, j11 = 0.0;
  for (int a = 0; a < 6; ++a) {
    j00 += g[a][0] * c.x[t[a]];
    j01 += g[a][0] * c.y[t[a]];
    j10 += g[a][1] * c.x[t[a]];
    j11 += g[a][1] * c.y[t[a]];
  }
  const double det = j00 * j11 - j01 * j10;
  if (!(det > 0.0)) throw Failure(Code::mesh, "inverted element (detJ <= 0)");
  const double k00 = j11 / det, k01 = -j01 / det, k10 = -j10 / det, k11 = j00 / det;
  std::memset(Bop, 0, sizeof(double) * 36);
  for (int a = 0; a < 6; ++a) {
    const double dx = k00 * g[a][0] + k01 * g[a][1];
    const double dy = k10 * g[a][0] + k11 * g[a][1];
    Bop[0][2 * a] = dx;
    Bop[1][2 * a + 1] = dy;
    Bop[2][2 * a] = dy;
    Bop[2][2 * a + 1] = dx;
  }
  return det;
}

constexpr double kGauss[3][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0}};
constexpr double kGaussW = 1.0 / 6.0;

Cell mesh_default_cell(int sub) {
  if (sub < 2) throw Failure(Code::config, "rve subdivisions must be >= 2");
  const std::vector<Disc> incl = {{0.3, 0.3, 0.2}, {0.7, 0.65, 0.2}};
  const Disc pore{0.65, 0.25, 0.15};
  std::vector<Disc> discs = incl;
  discs.push_back(pore);
  const double margin = 0.5 / sub;
  for (const auto& d : discs) {
    const bool inside = d.cx - d.rad > margin && d.cx + d.rad < 1.0 - margin && d.cy - d.rad > margin &&
                        d.cy + d.rad < 1.0 - margin;
    if (!inside) throw Failure(Code::geometry, "inclusion/pore not inside unit cell");
  }
  const int g = 2 * sub + 1;
  const int nn = g * g;
  std::vector<double> px(nn), py(nn);
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      px[j * g + i] = i / (g - 1.0);
      py[j * g + i] = j / (g - 1.0);
    }
  const double band = 0.3 / sub;
  std::vector<int> snapped(nn, -1);
  auto project = [&](int id, const Disc& d) {
    const double r = d.distance(px[id], py[id]);
    if (r > 1e-12) {
      px[id] = d.cx + (px[id] - d.cx) * d.rad / r;
      py[id] = d.cy + (py[id] - d.cy) * d.rad / r;
    }
  };
  for (int j = 2; j < g - 1; j += 2)
    for (int i = 2; i < g - 1; i += 2) {
      const int id = j * g + i;
      int pick = -1, near = 0;
      double gap_best = band;
      for (int c = 0; c < (int)discs.size(); ++c) {
        const double gap = std::abs(discs[c].distance(px[id], py[id]) - discs[c].rad);
        near += gap < band;
        if (gap < gap_best) {
          gap_best = gap;
          pick = c;
        }
      }
      if (near > 1 || pick < 0) continue;
      project(id, discs[pick]);
      snapped[id] = pick;
    }
  auto midpoint = [&](int mid, int a, int b) {
    px[mid] = 0.5 * (px[a] + px[b]);
    py[mid] = 0.5 * (py[a] + py[b]);
    if (snapped[a] >= 0 && snapped[a] == snapped[b]) project(mid, discs[snapped[a]]);
  };
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      const int oi = i & 1, oj = j & 1;
      if (oi && !oj) midpoint(j * g + i, j * g + i - 1, j * g + i + 1);
      if (!oi && oj) midpoint(j * g + i, (j - 1) * g + i, (j + 1) * g + i);
      if (oi && oj) midpoint(j * g + i, (j - 1) * g + i - 1, (j + 1) * g + i + 1);
    }
  Cell cell;
  std::vector<int> renum(nn, -1);
  for (int j = 0; j < sub; ++j)
    for (int i = 0; i < sub; ++i) {
      const int b = (2 * j) * g + 2 * i;  // lower-left corner
      const std::array<std::array<int, 6>, 2> pair = {{
          {b, b + 2, b + 2 * g + 2, b + 1, b + g + 2, b + g + 1},
          {b, b + 2 * g + 2, b + 2 * g, b + g + 1, b + 2 * g + 1, b + g},
      }};
      for (const auto& t : pair) {
        const double cx = (px[t[0]] + px[t[1]] + px[t[2]]) / 3.0;
        const double cy = (py[t[0]] + py[t[1]] + py[t[2]]) / 3.0;
        if (pore.distance(cx, cy) < pore.rad) continue;
        int ph = 0;
        for (const auto& d : incl)
          if (d.distance(cx, cy) < d.rad) {
            ph = 1;
            break;
          }
        std::array<int, 6> loc;
        for (int a = 0; a < 6; ++a) {
          if (renum[t[a]] < 0) {
            renum[t[a]] = (int)cell.x.size();
            cell.x.push_back(px[t[a]]);
            cell.y.push_back(py[t[a]]);
          }
          loc[a] = renum[t[a]];
        }
        cell.tri.push_back(loc);
        cell.phase.push_back(ph);
      }
    }
  if (cell.tri.empty()) throw Failure(Code::mesh, "meshing produced no elements");
  cell.on_boundary.assign(cell.x.size(), 0);
  for (size_t k = 0; k < cell.x.size(); ++k) {
    const double x = cell.x[k], y = cell.y[k];
    cell.on_boundary[k] = std::abs(x) < 1e-12 || std::abs(x - 1.0) < 1e-12 || std::abs(y) < 1e-12 ||
                          std::abs(y - 1.0) < 1e-12;
  }
  double area = 0.0;
  double Bop[3][12];
  for (const auto& t : cell.tri) {
    double a = 0.0;
    for (int q = 0; q < 3; ++q) a += kGaussW * strain_operator(cell, t, kGauss[q][0], kGauss[q][1], Bop);
    area += a;
  }
  cell.area = area;
  return cell;
}

// Orthonormal basis by Householder reflections: Q = H_0 ... H_{n-1} [I; 0].
void orthonormalise(std::vector<double>& A, int m, int n) {
  std::vector<double> refl;        // packed reflectors
  std::vector<size_t> off(n + 1, 0);
  std::vector<double> beta(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double ss = 0.0;
    for (int i = j; i < m; ++i) ss += A[(size_t)i * n + j] * A[(size_t)i * n + j];
    const double len = std::sqrt(ss);
    const double shift = A[(size_t)j * n + j] >= 0.0 ? -len : len;
    off[j] = refl.size();
    for (int i = j; i < m; ++i) refl.push_back(A[(size_t)i * n + j]);
    double* v = refl.data() + off[j];
    v[0] = v[0] - shift;
    double vv = 0.0;
    for (int i = 0; i < m - j; ++i) vv += v[i] * v[i];
    if (vv > 0.0) {
      beta[j] = 2.0 / vv;
      for (int c = j; c < n; ++c) {
        double dot = 0.0;
        for (int i = j; i < m; ++i) dot += v[i - j] * A[(size_t)i * n + c];
        const double s = beta[j] * dot;
        for (int i = j; i < m; ++i) A[(size_t)i * n + c] = A[(size_t)i * n + c] - s * v[i - j];
      }
    }
  }
  off[n] = refl.size();
  std::vector<double> Q((size_t)m * n, 0.0);
  for (int j = 0; j < n; ++j) Q[(size_t)j * n + j] = 1.0;
  for (int j = n - 1; j >= 0; --j) {
    if (beta[j] == 0.0) continue;
    const double* v = refl.data() + off[j];
    for (int c = 0; c < n; ++c) {
      double dot = 0.0;
      for (int i = j; i < m; ++i) dot += v[i - j] * Q[(size_t)i * n + c];
      const double s = beta[j] * dot;
      for (int i = j; i < m; ++i) Q[(size_t)i * n + c] = Q[(size_t)i * n + c] - s * v[i - j];
    }
  }
  A.swap(Q);
}

}  // namespace

struct Model {
  int n = 0, K = 0, n_free = 0;
  double volume = 0.0;
  std::vector<double> G, w;
  std::vector<double> G4;  // [K][4][n] displacement-gradient operator (finite strain)
  std::vector<int> ip, mat;
};

// Plain-text mesh in the reference's format (write_mesh / read_mesh,
// mesh.hpp:413-489): "fe2rom-mesh 1", nodes "id x y" (%.17g, bit-exact
// round trip), elements "e material n0..n5", node sets. The linear-BC
// boundary of a read mesh is the nodes on its bounding box.
void finish_cell(Cell& cell) {
  double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
  for (size_t k = 0; k < cell.x.size(); ++k) {
    x0 = std::min(x0, cell.x[k]);
    x1 = std::max(x1, cell.x[k]);
    y0 = std::min(y0, cell.y[k]);
    y1 = std::max(y1, cell.y[k]);
  }
  const double tol = 1e-12 * std::max(1.0, std::max(x1 - x0, y1 - y0));
  cell.on_boundary.assign(cell.x.size(), 0);
  for (size_t k = 0; k < cell.x.size(); ++k)
    cell.on_boundary[k] = std::abs(cell.x[k] - x0) < tol || std::abs(cell.x[k] - x1) < tol ||
                          std::abs(cell.y[k] - y0) < tol || std::abs(cell.y[k] - y1) < tol;
  double area = 0.0, Bop[3][12];
  for (const auto& t : cell.tri) {  // per-element sums first, as mesh_default_cell (compute_area)
    double ae = 0.0;
    for (int q = 0; q < 3; ++q) ae += kGaussW * strain_operator(cell, t, kGauss[q][0], kGauss[q][1], Bop);
    area += ae;
  }
  cell.area = area;
}

void mesh_write(const Cell& cell, std::FILE* f) {
  std::fprintf(f, "fe2rom-mesh 1\nnodes %zu\n", cell.x.size());
  for (size_t k = 0; k < cell.x.size(); ++k) std::fprintf(f, "%zu %.17g %.17g\n", k, cell.x[k], cell.y[k]);
  std::fprintf(f, "elements %zu\n", cell.tri.size());
  for (size_t e = 0; e < cell.tri.size(); ++e) {
    std::fprintf(f, "%zu %d", e, cell.phase[e]);
    for (int a = 0; a < 6; ++a) std::fprintf(f, " %d", cell.tri[e][a]);
    std::fprintf(f, "\n");
  }
  // node sets of the unit cell (build_rve_mesh, mesh.hpp:344-347), in std::map order
  std::map<std::string, std::vector<int>> sets;
  for (size_t k = 0; k < cell.x.size(); ++k) {
    if (std::abs(cell.x[k]) < 1e-12) sets["left"].push_back(static_cast<int>(k));
    if (std::abs(cell.x[k] - 1.0) < 1e-12) sets["right"].push_back(static_cast<int>(k));
    if (std::abs(cell.y[k]) < 1e-12) sets["bottom"].push_back(static_cast<int>(k));
    if (std::abs(cell.y[k] - 1.0) < 1e-12) sets["top"].push_back(static_cast<int>(k));
  }
  for (const auto& [name, ids] : sets) {
    std::fprintf(f, "set %s %zu\n", name.c_str(), ids.size());
    for (size_t i = 0; i < ids.size(); ++i) std::fprintf(f, "%d%c", ids[i], i + 1 < ids.size() ? ' ' : '\n');
  }
}

Cell mesh_read(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  check(is.good(), Code::io, "cannot open mesh file: " + path);
  std::string magic, key;
  int version = 0, count = 0;
  is >> magic >> version;
  check(magic == "fe2rom-mesh" && version == 1, Code::io, "not a fe2rom mesh file");
  is >> key >> count;
  check(key == "nodes" && count >= 0, Code::io, "malformed mesh file (nodes)");
  Cell cell;
  cell.x.resize(count);
  cell.y.resize(count);
  for (int i = 0; i < count; ++i) {
    int id = -1;
    is >> id >> cell.x[i] >> cell.y[i];
    check(is.good() && id == i, Code::io, "node ids must be dense");
  }
  is >> key >> count;
  check(key == "elements" && count >= 0, Code::io, "malformed mesh file (elements)");
  cell.tri.resize(count);
  cell.phase.resize(count);
  for (int e = 0; e < count; ++e) {
    int id = -1;
    is >> id >> cell.phase[e];
    for (int a = 0; a < 6; ++a) {
      is >> cell.tri[e][a];
      check(cell.tri[e][a] >= 0 && cell.tri[e][a] < static_cast<int>(cell.x.size()), Code::io,
            "element references missing node");
    }
    check(is.good(), Code::io, "malformed mesh file (element)");
  }
  check(!cell.tri.empty(), Code::mesh, "mesh has no elements");
  finish_cell(cell);  // node sets are not needed: the linear BC acts on the bounding box
  return cell;
}

Model build_model_on(const Cell& cell, int n, int K, std::uint64_t seed, const double* basis = nullptr);

Model build_model(int sub, int n, int K, std::uint64_t seed) { return build_model_on(mesh_default_cell(sub), n, K, seed); }

// basis: optional Φ over all DOFs, column-major (mode j at basis + j * 2 n_nodes),
// e.g. a POD basis (fe2_pod_basis); its boundary rows are ignored (linear BC).
// Without it Φ is the seeded orthonormal basis.
Model build_model_on(const Cell& cell, int n, int K, std::uint64_t seed, const double* basis) {
  const int n_nodes = (int)cell.x.size();
  const int n_ip = 3 * (int)cell.tri.size();
  std::vector<int> dof_free(2 * n_nodes, -1);
  int nf = 0;
  for (int d = 0; d < 2 * n_nodes; ++d)
    if (!cell.on_boundary[d / 2]) dof_free[d] = nf++;
  if (n < 1 || n > nf) throw Failure(Code::config, "mode count out of range");
  const bool full_rule = K == 0;  // all integration points with their own weights (training / ECM)
  if (full_rule) K = n_ip;
  if (K < 1 || K > n_ip) throw Failure(Code::config, "cubature size out of range");

  std::vector<double> phi((size_t)nf * n);
  if (basis) {
    for (int d = 0; d < 2 * n_nodes; ++d)
      if (dof_free[d] >= 0)
        for (int j = 0; j < n; ++j) phi[(size_t)dof_free[d] * n + j] = basis[(size_t)j * 2 * n_nodes + d];
  } else {
    SeededStream s(seed ^ kPhiStream);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < nf; ++i) phi[(size_t)i * n + j] = s.gauss();
    orthonormalise(phi, nf, n);
  }
  Model md;
  md.n = n;
  md.K = K;
  md.n_free = nf;
  md.volume = cell.area;
  if (full_rule) {
    for (int i = 0; i < n_ip; ++i) {
      const auto& t = cell.tri[i / 3];
      double Bq[3][12];
      const double det = strain_operator(cell, t, kGauss[i % 3][0], kGauss[i % 3][1], Bq);
      md.ip.push_back(i);
      md.w.push_back(kGaussW * det);
    }
  } else {
    SeededStream s(seed ^ kRuleStream);
    std::vector<int> perm(n_ip);
    for (int i = 0; i < n_ip; ++i) perm[i] = i;
    for (int i = 0; i < K; ++i) std::swap(perm[i], perm[i + s.below(n_ip - i)]);
    const double unit_w = cell.area / K;
    md.ip.assign(perm.begin(), perm.begin() + K);
    for (int i = 0; i < K; ++i) md.w.push_back(s.in(0.5, 1.5) * unit_w);
  }
  md.G.assign((size_t)K * 3 * n, 0.0);
  md.G4.assign((size_t)K * 4 * n, 0.0);
  md.mat.resize(K);
  double Bop[3][12];
  for (int q = 0; q < K; ++q) {
    const int e = md.ip[q] / 3, gp = md.ip[q] % 3;
    const auto& t = cell.tri[e];
    md.mat[q] = cell.phase[e];
    strain_operator(cell, t, kGauss[gp][0], kGauss[gp][1], Bop);
    int rows[12];
    for (int d = 0; d < 12; ++d) rows[d] = dof_free[2 * t[d / 2] + d % 2];
    double* Gq = md.G.data() + (size_t)q * 3 * n;
    for (int i = 0; i < 3; ++i)
      for (int a = 0; a < n; ++a) {
        double acc = 0.0;
        for (int d = 0; d < 12; ++d)
          if (rows[d] >= 0) acc += Bop[i][d] * phi[(size_t)rows[d] * n + a];
        Gq[i * n + a] = acc;
      }
    // gradient rows (dux/dX, dux/dY, duy/dX, duy/dY) from the same dN/dx, dN/dy
    double Bg[4][12] = {};
    for (int a = 0; a < 6; ++a) {
      Bg[0][2 * a] = Bop[0][2 * a];
      Bg[1][2 * a] = Bop[2][2 * a];
      Bg[2][2 * a + 1] = Bop[2][2 * a + 1];
      Bg[3][2 * a + 1] = Bop[1][2 * a + 1];
    }
    double* G4q = md.G4.data() + (size_t)q * 4 * n;
    for (int i = 0; i < 4; ++i)
      for (int a = 0; a < n; ++a) {
        double acc = 0.0;
        for (int d = 0; d < 12; ++d)
          if (rows[d] >= 0) acc += Bg[i][d] * phi[(size_t)rows[d] * n + a];
        G4q[i * n + a] = acc;
      }
  }
  return md;
}

void make_paths(int kind, std::uint64_t seed, std::int64_t p0, std::int64_t P, int n_incr, double* E) {
  for (std::int64_t k = 0; k < P; ++k) {
    const std::uint64_t p = static_cast<std::uint64_t>(p0 + k);
    SeededStream s(mix64(seed ^ kPathStream) ^ mix64(p));
    double end[3];
    double* out = E + (size_t)k * n_incr * 3;
    if (kind == 0) {  // config 0: uniaxial E11 = 0.05 scaled by s, rotated by theta
      const double scale = s.in(0.5, 1.5);
      const double th = s.in(0.0, std::numbers::pi);
      const double c = std::cos(th), sn = std::sin(th);
      const double e = 0.05 * scale;
      end[0] = e * (c * c);
      end[1] = e * (sn * sn);
      end[2] = e * (2.0 * sn * c);
      for (int i = 1; i <= n_incr; ++i) {
        const double f = static_cast<double>(i) / n_incr;
        for (int c3 = 0; c3 < 3; ++c3) out[(i - 1) * 3 + c3] = end[c3] * f;
      }
    } else if (kind == 1) {  // config 1: bending-like (E11, 2 E12), reversed halfway
      const double a = s.in(-0.03, 0.03);
      const double b = s.in(-0.02, 0.02);
      end[0] = a;
      end[1] = 0.0;
      end[2] = 2.0 * b;
      const int half = n_incr / 2;
      for (int i = 1; i <= n_incr; ++i) {
        const double f = i <= half ? static_cast<double>(i) / half : static_cast<double>(n_incr - i) / half;
        for (int c3 = 0; c3 < 3; ++c3) out[(i - 1) * 3 + c3] = end[c3] * f;
      }
    } else if (kind == 2) {  // config 2: F = I + (i / n_incr) H, H ~ U[-0.08, 0.08]^4, det(I + H) > 0.8
      double H[4];
      do {
        for (double& h : H) h = s.in(-0.08, 0.08);
      } while (!((1.0 + H[0]) * (1.0 + H[3]) - H[1] * H[2] > 0.8));
      double* out4 = E + (size_t)k * n_incr * 4;
      for (int i = 1; i <= n_incr; ++i) {
        const double f = static_cast<double>(i) / n_incr;
        for (int c4 = 0; c4 < 4; ++c4) out4[(i - 1) * 4 + c4] = H[c4] * f;
      }
    } else {
      throw Failure(Code::config, "unknown path kind");
    }
  }
}


Cell load_cell(int subdivisions, const char* mesh_path) {
  return mesh_path ? mesh_read(mesh_path) : mesh_default_cell(subdivisions);
}

RveData rve_data(int subdivisions, const char* mesh_path) {
  const Cell cell = load_cell(subdivisions, mesh_path);
  RveData r;
  r.n_nodes = (int)cell.x.size();
  r.n_el = (int)cell.tri.size();
  r.x = cell.x;
  r.y = cell.y;
  r.volume = cell.area;
  r.phase = cell.phase;
  r.free_index.assign(2 * r.n_nodes, -1);
  for (int d = 0; d < 2 * r.n_nodes; ++d)
    if (!cell.on_boundary[d / 2]) r.free_index[d] = r.n_free++;
  r.conn.resize((size_t)6 * r.n_el);
  r.B.resize((size_t)36 * 3 * r.n_el);
  r.w.resize((size_t)3 * r.n_el);
  for (int e = 0; e < r.n_el; ++e) {
    for (int a = 0; a < 6; ++a) r.conn[(size_t)6 * e + a] = cell.tri[e][a];
    for (int g = 0; g < 3; ++g) {
      double Bq[3][12];
      const double det = strain_operator(cell, cell.tri[e], kGauss[g][0], kGauss[g][1], Bq);
      std::memcpy(r.B.data() + (size_t)36 * (3 * e + g), Bq, sizeof(Bq));
      r.w[3 * e + g] = kGaussW * det;
    }
  }
  return r;
}

int orthonormalize_columns(std::vector<double>& A, std::int64_t rows, int cols, const std::vector<double>& drop_tol) {
  int kept = 0;
  for (int j = 0; j < cols; ++j) {
    double* v = A.data() + (size_t)j * rows;
    double nrm = 0.0;
    for (int pass = 0; pass < 2; ++pass)
      for (int c = 0; c < kept; ++c) {
        const double* q = A.data() + (size_t)c * rows;
        double dot = 0.0;
        for (std::int64_t i = 0; i < rows; ++i) dot += q[i] * v[i];
        for (std::int64_t i = 0; i < rows; ++i) v[i] -= dot * q[i];
      }
    for (std::int64_t i = 0; i < rows; ++i) nrm += v[i] * v[i];
    nrm = std::sqrt(nrm);
    if (!(nrm > drop_tol[j])) continue;
    double* dst = A.data() + (size_t)kept * rows;
    for (std::int64_t i = 0; i < rows; ++i) dst[i] = v[i] / nrm;
    ++kept;
  }
  A.resize((size_t)kept * rows);
  return kept;
}

}  // namespace fe2

struct fe2_model_s {
  fe2::Model m;
};

extern "C" {

int fe2_model_build(int subdivisions, int n, int K, uint64_t seed, fe2_model_t* out) {
  return fe2::guard([&] { *out = new fe2_model_s{fe2::build_model(subdivisions, n, K, seed)}; });
}
int fe2_model_build_from_mesh(const char* path, int n, int K, uint64_t seed, fe2_model_t* out) {
  return fe2::guard([&] {
    fe2::check(path && out, fe2::Code::config, "bad arguments");
    *out = new fe2_model_s{fe2::build_model_on(fe2::mesh_read(path), n, K, seed)};
  });
}
int fe2_model_build_basis(int subdivisions, const char* mesh_path, const double* basis, int n, int K, uint64_t seed,
                          fe2_model_t* out) {
  return fe2::guard([&] {
    fe2::check(basis && out && n >= 1, fe2::Code::config, "bad arguments");
    *out = new fe2_model_s{fe2::build_model_on(fe2::load_cell(subdivisions, mesh_path), n, K, seed, basis)};
  });
}
int fe2_mesh_write(int subdivisions, const char* path) {
  return fe2::guard([&] {
    fe2::check(path != nullptr, fe2::Code::config, "bad arguments");
    std::FILE* f = std::fopen(path, "wb");
    fe2::check(f != nullptr, fe2::Code::io, std::string("cannot open for write: ") + path);
    fe2::mesh_write(fe2::mesh_default_cell(subdivisions), f);
    std::fclose(f);
  });
}
void fe2_model_free(fe2_model_t m) { delete m; }
int fe2_model_sizes(fe2_model_t m, int* n, int* K, int* n_free, double* volume) {
  return fe2::guard([&] {
    fe2::check(m != nullptr, fe2::Code::config, "null model");
    if (n) *n = m->m.n;
    if (K) *K = m->m.K;
    if (n_free) *n_free = m->m.n_free;
    if (volume) *volume = m->m.volume;
  });
}
int fe2_model_arrays(fe2_model_t m, double* G, double* w, int* ip_id, int* mat_id) {
  return fe2::guard([&] {
    fe2::check(m != nullptr, fe2::Code::config, "null model");
    if (G) std::memcpy(G, m->m.G.data(), m->m.G.size() * sizeof(double));
    if (w) std::memcpy(w, m->m.w.data(), m->m.w.size() * sizeof(double));
    if (ip_id) std::memcpy(ip_id, m->m.ip.data(), m->m.ip.size() * sizeof(int));
    if (mat_id) std::memcpy(mat_id, m->m.mat.data(), m->m.mat.size() * sizeof(int));
  });
}
int fe2_model_g4(fe2_model_t m, double* G4) {
  return fe2::guard([&] {
    fe2::check(m != nullptr && G4 != nullptr, fe2::Code::config, "null model or output");
    std::memcpy(G4, m->m.G4.data(), m->m.G4.size() * sizeof(double));
  });
}
int fe2_paths(int kind, uint64_t seed, int64_t p0, int64_t P, int n_incr, double* E) {
  return fe2::guard([&] {
    fe2::check(P >= 0 && n_incr >= 1 && E != nullptr, fe2::Code::config, "bad path arguments");
    fe2::make_paths(kind, seed, p0, P, n_incr, E);
  });
}

}  // extern "C"
