// fe2rom CPU ORACLE — TEST INFRASTRUCTURE ONLY (see fe2rom_oracle.h).
//
// Plain C++20 restatement of the reference arithmetic, each function citing
// the reference file:line it follows (paths relative to
// /root/reference/proj/include/fe2rom/). Built -O3 with no -march (the
// reference's Release defaults, proj/CMakeLists.txt:7-9), so no FMA
// contraction: every product and sum is rounded the way the reference's
// scalar code rounds it.
#include "fe2rom_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <mutex>
#include <numbers>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------------------
// Errors (common.hpp:26-52)
enum class ErrorCode { config, geometry, mesh, material, solver, numeric, rank, bc, io, provenance };

struct Error : std::runtime_error {
  Error(ErrorCode c, const std::string& w) : std::runtime_error(w), code(c) {}
  ErrorCode code;
};
[[noreturn]] inline void fail(ErrorCode c, const std::string& m) { throw Error(c, m); }
inline void require(bool ok, ErrorCode c, const std::string& m) {
  if (!ok) fail(c, m);
}

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return 1 + static_cast<int>(e.code);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1 + static_cast<int>(ErrorCode::numeric);
  }
}

// ---------------------------------------------------------------------------
// Rng (common.hpp:56-88): mt19937_64, (u64 >> 11) * 2^-53, Box-Muller with
// cached spare (cos first, then sin).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t next_u64() { return gen_(); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  int uniform_int(int n) { return std::min(n - 1, static_cast<int>(uniform() * n)); }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * std::numbers::pi * uniform();
    spare_ = r * std::sin(t);
    have_spare_ = true;
    return r * std::cos(t);
  }

 private:
  std::mt19937_64 gen_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

// ---------------------------------------------------------------------------
// Materials (materials.hpp). Packed 4-tensors (11, 22, 33, 12-tensor).
struct State {
  double ep[4] = {0, 0, 0, 0};
  double eq = 0.0;
  double s33 = 0.0;
};

struct Mat {
  int kind = 0;  // 0 elastic, 1 J2 linear, 2 power law, 3 strain-hardening creep
  double E = 1.0, nu = 0.3, sy0 = 0.01, h = 0.016;
  double N = 0.1;                               // power law (materials.hpp:51-65)
  double A = 22.09, n = 1.06, m = -0.56, dt = 1.0;  // creep (:67-76); dt = PathStep::dt
  double lambda() const { return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)); }  // :49
  double mu() const { return 0.5 * E / (1.0 + nu); }                          // :50
  double yield_stress(double eq) const { return sy0 * std::pow(1.0 + E * eq / sy0, N); }      // :59-61
  double yield_slope(double eq) const { return E * N * std::pow(1.0 + E * eq / sy0, N - 1.0); }  // :62-64
};

inline Mat to_mat(const orc_material_t& m) {
  Mat r;
  r.kind = m.kind;
  r.E = m.p[0];
  r.nu = m.p[1];
  if (m.kind == 1) {
    r.sy0 = m.p[2];
    r.h = m.p[3];
  } else if (m.kind == 2) {
    r.sy0 = m.p[2];
    r.N = m.p[3];
  } else if (m.kind == 3) {
    r.A = m.p[2];
    r.n = m.p[3];
    r.m = m.p[4];
    r.dt = m.p[5];
  }
  // validate (materials.hpp:80-98)
  require(m.kind >= 0 && m.kind <= 3, ErrorCode::config, "unsupported material kind");
  require(r.E > 0.0 && r.nu >= 0.0 && r.nu < 0.5, ErrorCode::config, "invalid elastic parameters");
  if (m.kind == 1)
    require(r.sy0 > 0.0 && r.h >= 0.0, ErrorCode::config, "invalid J2 parameters");
  if (m.kind == 2)
    require(r.sy0 > 0.0 && r.N > 0.0 && r.N < 1.0, ErrorCode::config, "invalid power-law parameters");
  if (m.kind == 3)
    require(r.A > 0.0 && r.n > 0.0 && r.m > -1.0, ErrorCode::config, "invalid creep parameters");
  return r;
}

inline double trace4(const double* v) { return v[0] + v[1] + v[2]; }  // :19
inline void dev4(const double* v, double* o) {                        // :21-24
  const double p = trace4(v) / 3.0;
  o[0] = v[0] - p;
  o[1] = v[1] - p;
  o[2] = v[2] - p;
  o[3] = v[3];
}
inline double contract4(const double* a, const double* b) {  // :26-28
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + 2.0 * a[3] * b[3];
}
inline double norm4(const double* v) { return std::sqrt(contract4(v, v)); }  // :30

struct Result4 {
  double sigma[4];
  double D[4][4];
  State state;
  bool plastic = false;
};

inline void elastic_tangent4(double l, double mu, double D[4][4]) {  // :122-128
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) D[i][j] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D[i][j] = l;
  for (int i = 0; i < 4; ++i) D[i][i] += 2.0 * mu;
}

inline void elastic_stress4(double l, double mu, const double* e, double* s) {  // :130-134
  const double lt = l * trace4(e);
  s[0] = lt + 2.0 * mu * e[0];
  s[1] = lt + 2.0 * mu * e[1];
  s[2] = lt + 2.0 * mu * e[2];
  s[3] = 2.0 * mu * e[3];
}

// update4 for ElasticParams (:199-203), J2LinearParams (:205-214),
// PowerLawParams (:216-244) and CreepParams (:246-292), with
// trial_state (:162-169), elastic_result (:187-195), finish_return (:173-185)
// and radial_return_tangent4 (:138-154).
inline Result4 update4(const Mat& m, const State& s0, const double* eps) {
  const double l = m.lambda(), mu = m.mu();
  Result4 out;
  double ee[4], sig_tr[4], s_tr[4];
  for (int i = 0; i < 4; ++i) ee[i] = eps[i] - s0.ep[i];
  elastic_stress4(l, mu, ee, sig_tr);
  dev4(sig_tr, s_tr);
  const double q_tr = std::sqrt(1.5) * norm4(s_tr);
  bool plastic = false;
  double dlam = 0.0, dlam_dqtr = 0.0;
  if (m.kind == 1) {  // closed form (:205-214)
    const double f = q_tr - (m.sy0 + m.h * s0.eq);
    plastic = !(f <= 0.0);
    const double denom = 3.0 * mu + m.h;
    dlam = f / denom;
    dlam_dqtr = 1.0 / denom;
  } else if (m.kind == 2) {  // power law: safeguarded Newton on g (:216-244)
    const double f_tr = q_tr - m.yield_stress(s0.eq);
    if (!(f_tr <= 0.0)) {
      auto g = [&](double x) { return q_tr - 3.0 * mu * x - m.yield_stress(s0.eq + x); };
      double lo = 0.0, hi = f_tr / (3.0 * mu), x = hi * 0.5;
      const double tol = 1e-12 * std::max(m.sy0, q_tr);
      bool converged = false;
      for (int it = 0; it < 50; ++it) {
        const double gx = g(x);
        if (std::abs(gx) <= tol) {
          converged = true;
          break;
        }
        if (gx > 0.0) lo = x;
        else hi = x;
        const double slope = 3.0 * mu + m.yield_slope(s0.eq + x);
        double next = x + gx / slope;
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        x = next;
      }
      require(converged, ErrorCode::material, "power-law return map did not converge");
      plastic = true;
      dlam = x;
      dlam_dqtr = 1.0 / (3.0 * mu + m.yield_slope(s0.eq + x));
    }
  } else if (m.kind == 3) {  // strain-hardening creep: safeguarded Newton on R (:246-292)
    require(m.dt > 0.0, ErrorCode::material, "creep update needs dt > 0");
    if (q_tr > 1e-14 * m.E) {
      const double p1 = m.n / (m.m + 1.0), p2 = m.m / (m.m + 1.0), eq_floor = 1e-12;
      auto hard = [&](double e) { return std::pow((m.m + 1.0) * std::max(e, eq_floor), p2); };
      auto hard_slope = [&](double e) {
        if (e <= eq_floor) return 0.0;
        return p2 * (m.m + 1.0) * std::pow((m.m + 1.0) * e, p2 - 1.0);
      };
      auto rate_q = [&](double q) { return std::pow(q / m.A, p1); };
      auto rate_q_slope = [&](double q) { return p1 / m.A * std::pow(q / m.A, p1 - 1.0); };
      auto R = [&](double x) { return x - m.dt * rate_q(q_tr - 3.0 * mu * x) * hard(s0.eq + x); };
      double lo = 0.0, hi = q_tr / (3.0 * mu);
      require(!(R(hi) < 0.0), ErrorCode::material, "creep return bracket failure");
      double x = 0.5 * hi;
      const double tol = 1e-14 * std::max(1.0, hi);
      bool converged = false;
      double Rp = 1.0;
      for (int it = 0; it < 200; ++it) {
        const double q = q_tr - 3.0 * mu * x;
        const double e = s0.eq + x;
        const double Rx = x - m.dt * rate_q(q) * hard(e);
        Rp = 1.0 + 3.0 * mu * m.dt * rate_q_slope(q) * hard(e) - m.dt * rate_q(q) * hard_slope(e);
        if (std::abs(Rx) <= tol) {
          converged = true;
          break;
        }
        if (Rx < 0.0) lo = x;
        else hi = x;
        double next = (Rp > 0.0) ? x - Rx / Rp : 0.5 * (lo + hi);
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        x = next;
      }
      require(converged, ErrorCode::material, "creep return map did not converge");
      if (x > 0.0) {
        plastic = true;
        dlam = x;
        dlam_dqtr = m.dt * rate_q_slope(q_tr - 3.0 * mu * x) * hard(s0.eq + x) / Rp;
      }
    }
  }
  if (!plastic) {
    for (int i = 0; i < 4; ++i) out.sigma[i] = sig_tr[i];
    elastic_tangent4(l, mu, out.D);
    out.state = s0;
    out.state.s33 = sig_tr[2];
    out.plastic = false;
    return out;
  }
  double dir[4];
  for (int i = 0; i < 4; ++i) dir[i] = s_tr[i] / q_tr;
  const double c_sig = 3.0 * mu * dlam;
  for (int i = 0; i < 4; ++i) out.sigma[i] = sig_tr[i] - c_sig * dir[i];
  out.state = s0;
  const double c_ep = 1.5 * dlam;
  for (int i = 0; i < 4; ++i) out.state.ep[i] = s0.ep[i] + c_ep * dir[i];
  out.state.eq = s0.eq + dlam;
  out.state.s33 = out.sigma[2];
  const double ns = norm4(s_tr);
  double n_unit[4];
  for (int i = 0; i < 4; ++i) n_unit[i] = s_tr[i] / ns;
  elastic_tangent4(l, mu, out.D);
  static const double pdev[4][4] = {{2.0 / 3.0, -1.0 / 3.0, -1.0 / 3.0, 0.0},
                                    {-1.0 / 3.0, 2.0 / 3.0, -1.0 / 3.0, 0.0},
                                    {-1.0 / 3.0, -1.0 / 3.0, 2.0 / 3.0, 0.0},
                                    {0.0, 0.0, 0.0, 1.0}};
  const double c1 = 6.0 * mu * mu * dlam / q_tr;
  const double c2 = 6.0 * mu * mu * (dlam_dqtr - dlam / q_tr);
  const double n_dbl[4] = {n_unit[0], n_unit[1], n_unit[2], 2.0 * n_unit[3]};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out.D[i][j] -= c1 * pdev[i][j];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out.D[i][j] -= c2 * (n_unit[i] * n_dbl[j]);
  out.plastic = true;
  return out;
}

struct Result3 {
  double sigma[3];
  double C[3][3];
  State state;
  bool plastic;
};

// update_material (:317-325): strain4_from_voigt (:35) + condense_tangent (:305-314)
inline Result3 update_material(const Mat& m, const State& s0, const double* e3) {
  const double e4[4] = {e3[0], e3[1], 0.0, 0.5 * e3[2]};
  const Result4 r4 = update4(m, s0, e4);
  Result3 out;
  out.sigma[0] = r4.sigma[0];
  out.sigma[1] = r4.sigma[1];
  out.sigma[2] = r4.sigma[3];
  static const int rows[3] = {0, 1, 3};
  for (int i = 0; i < 3; ++i) {
    out.C[i][0] = r4.D[rows[i]][0];
    out.C[i][1] = r4.D[rows[i]][1];
    out.C[i][2] = 0.5 * r4.D[rows[i]][3];
  }
  out.state = r4.state;
  out.plastic = r4.plastic;
  return out;
}

// ---------------------------------------------------------------------------
// Mesh (mesh.hpp)
struct Node {
  double x, y;
};
struct Element {
  std::array<int, 6> nodes;
  int mat;
};
struct Circle {
  double x, y, r;
  double dist(double px, double py) const { return std::hypot(px - x, py - y); }  // :174
  bool contains(double px, double py) const { return dist(px, py) < r; }         // :175
};

struct Mesh {
  std::vector<Node> nodes;
  std::vector<Element> elements;
  std::vector<int> left, right, bottom, top;
  double area = 0.0;
  int n_nodes() const { return (int)nodes.size(); }
  int n_el() const { return (int)elements.size(); }
  int n_dofs() const { return 2 * n_nodes(); }
  int n_ips() const { return 3 * n_el(); }
};

static const double kQP[3][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0}};
static const double kQW = 1.0 / 6.0;  // tri3 (mesh.hpp:33-38)

inline void tri6_shape_grad(double xi, double eta, double d[6][2]) {  // :67-77
  const double l1 = 1.0 - xi - eta, l2 = xi, l3 = eta;
  d[0][0] = -(4.0 * l1 - 1.0);
  d[0][1] = -(4.0 * l1 - 1.0);
  d[1][0] = 4.0 * l2 - 1.0;
  d[1][1] = 0.0;
  d[2][0] = 0.0;
  d[2][1] = 4.0 * l3 - 1.0;
  d[3][0] = 4.0 * (l1 - l2);
  d[3][1] = -4.0 * l2;
  d[4][0] = 4.0 * l3;
  d[4][1] = 4.0 * l2;
  d[5][0] = -4.0 * l3;
  d[5][1] = 4.0 * (l1 - l3);
}

// shape_eval (:85-115): B (3x12, col 2a = x, 2a+1 = y), detJ > 0.
inline double shape_eval(const Mesh& mesh, const Element& el, double xi, double eta, double B[3][12]) {
  double dN[6][2];
  tri6_shape_grad(xi, eta, dN);
  double J00 = 0, J01 = 0, J10 = 0, J11 = 0;
  for (int a = 0; a < 6; ++a) {
    const Node& nd = mesh.nodes[el.nodes[a]];
    J00 += dN[a][0] * nd.x;
    J01 += dN[a][0] * nd.y;
    J10 += dN[a][1] * nd.x;
    J11 += dN[a][1] * nd.y;
  }
  const double detJ = J00 * J11 - J01 * J10;
  require(detJ > 0.0, ErrorCode::mesh, "inverted element (detJ <= 0)");
  const double i00 = J11 / detJ, i01 = -J01 / detJ, i10 = -J10 / detJ, i11 = J00 / detJ;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 12; ++c) B[r][c] = 0.0;
  for (int a = 0; a < 6; ++a) {
    const double dNdx = i00 * dN[a][0] + i01 * dN[a][1];
    const double dNdy = i10 * dN[a][0] + i11 * dN[a][1];
    B[0][2 * a] = dNdx;
    B[1][2 * a + 1] = dNdy;
    B[2][2 * a] = dNdy;
    B[2][2 * a + 1] = dNdx;
  }
  return detJ;
}

inline double compute_area(const Mesh& mesh) {  // :117-129
  double a = 0.0;
  double B[3][12];
  for (const auto& el : mesh.elements) {
    double ea = 0.0;
    for (int g = 0; g < 3; ++g) ea += kQW * shape_eval(mesh, el, kQP[g][0], kQP[g][1], B);
    a += ea;
  }
  return a;
}

struct Geometry {
  std::vector<Circle> inclusions;
  std::optional<Circle> pore;
  int subdivisions = 12;
};

inline Geometry default_cell(int subdivisions) {  // :185-191
  Geometry g;
  g.inclusions = {{0.3, 0.3, 0.2}, {0.7, 0.65, 0.2}};
  g.pore = Circle{0.65, 0.25, 0.15};
  g.subdivisions = subdivisions;
  return g;
}

inline void validate_geometry(const Geometry& geo) {  // :196-210
  std::vector<Circle> all = geo.inclusions;
  if (geo.pore) all.push_back(*geo.pore);
  const double wall_margin = 0.5 / geo.subdivisions;
  for (const auto& c : all) {
    require(c.r > 0.0, ErrorCode::geometry, "circle radius must be positive");
    const bool inside = c.x - c.r > wall_margin && c.x + c.r < 1.0 - wall_margin &&
                        c.y - c.r > wall_margin && c.y + c.r < 1.0 - wall_margin;
    require(inside, ErrorCode::geometry, "inclusion/pore not inside unit cell");
  }
  for (std::size_t a = 0; a < all.size(); ++a)
    for (std::size_t b = a + 1; b < all.size(); ++b)
      require(all[a].dist(all[b].x, all[b].y) > all[a].r + all[b].r, ErrorCode::geometry,
              "overlapping inclusions/pore");
}

// build_rve_mesh (:218-352)
inline Mesh build_rve_mesh(const Geometry& geo) {
  require(geo.subdivisions >= 2, ErrorCode::config, "rve subdivisions must be >= 2");
  validate_geometry(geo);
  const int n = geo.subdivisions;
  const int g = 2 * n + 1;
  auto gid = [g](int i, int j) { return j * g + i; };
  std::vector<double> px(g * g), py(g * g);
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      px[gid(i, j)] = i / (g - 1.0);
      py[gid(i, j)] = j / (g - 1.0);
    }
  std::vector<Circle> circles = geo.inclusions;
  if (geo.pore) circles.push_back(*geo.pore);

  const double band = 0.3 / n;
  std::vector<signed char> on_circle(g * g, -1);
  for (int j = 0; j < g; j += 2) {
    for (int i = 0; i < g; i += 2) {
      if (i == 0 || j == 0 || i == g - 1 || j == g - 1) continue;
      const int id = gid(i, j);
      int best = -1, claims = 0;
      double best_gap = band;
      for (std::size_t c = 0; c < circles.size(); ++c) {
        const double gap = std::abs(circles[c].dist(px[id], py[id]) - circles[c].r);
        if (gap < band) ++claims;
        if (gap < best_gap) {
          best_gap = gap;
          best = (int)c;
        }
      }
      if (claims > 1) continue;
      if (best >= 0) {
        const Circle& c = circles[best];
        const double d = c.dist(px[id], py[id]);
        if (d > 1e-12) {
          px[id] = c.x + (px[id] - c.x) * c.r / d;
          py[id] = c.y + (py[id] - c.y) * c.r / d;
        }
        on_circle[id] = (signed char)best;
      }
    }
  }
  auto place_mid = [&](int mid, int a, int b) {
    px[mid] = 0.5 * (px[a] + px[b]);
    py[mid] = 0.5 * (py[a] + py[b]);
    if (on_circle[a] >= 0 && on_circle[a] == on_circle[b]) {
      const Circle& c = circles[on_circle[a]];
      const double d = c.dist(px[mid], py[mid]);
      if (d > 1e-12) {
        px[mid] = c.x + (px[mid] - c.x) * c.r / d;
        py[mid] = c.y + (py[mid] - c.y) * c.r / d;
      }
    }
  };
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      const bool mi = (i % 2 == 1), mj = (j % 2 == 1);
      if (mi && !mj) place_mid(gid(i, j), gid(i - 1, j), gid(i + 1, j));
      if (!mi && mj) place_mid(gid(i, j), gid(i, j - 1), gid(i, j + 1));
      if (mi && mj) place_mid(gid(i, j), gid(i - 1, j - 1), gid(i + 1, j + 1));
    }
  auto material_of = [&](double cx, double cy) -> int {
    if (geo.pore && geo.pore->contains(cx, cy)) return -1;
    for (std::size_t c = 0; c < geo.inclusions.size(); ++c)
      if (geo.inclusions[c].contains(cx, cy)) return 1;
    return 0;
  };
  std::vector<std::array<int, 6>> raw;
  std::vector<int> raw_mat;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int i0 = 2 * i, j0 = 2 * j;
      const std::array<std::array<int, 6>, 2> tris = {{
          {gid(i0, j0), gid(i0 + 2, j0), gid(i0 + 2, j0 + 2), gid(i0 + 1, j0), gid(i0 + 2, j0 + 1),
           gid(i0 + 1, j0 + 1)},
          {gid(i0, j0), gid(i0 + 2, j0 + 2), gid(i0, j0 + 2), gid(i0 + 1, j0 + 1), gid(i0 + 1, j0 + 2),
           gid(i0, j0 + 1)},
      }};
      for (const auto& t : tris) {
        const double cx = (px[t[0]] + px[t[1]] + px[t[2]]) / 3.0;
        const double cy = (py[t[0]] + py[t[1]] + py[t[2]]) / 3.0;
        const int mat = material_of(cx, cy);
        if (mat < 0) continue;
        raw.push_back(t);
        raw_mat.push_back(mat);
      }
    }
  require(!raw.empty(), ErrorCode::mesh, "meshing produced no elements");
  std::vector<int> remap(g * g, -1);
  Mesh mesh;
  for (std::size_t e = 0; e < raw.size(); ++e) {
    Element el;
    el.mat = raw_mat[e];
    for (int a = 0; a < 6; ++a) {
      const int old = raw[e][a];
      if (remap[old] < 0) {
        remap[old] = mesh.n_nodes();
        mesh.nodes.push_back({px[old], py[old]});
      }
      el.nodes[a] = remap[old];
    }
    mesh.elements.push_back(el);
  }
  const double tol = 1e-12;
  for (int id = 0; id < mesh.n_nodes(); ++id) {
    const Node& nd = mesh.nodes[id];
    if (std::abs(nd.x) < tol) mesh.left.push_back(id);
    if (std::abs(nd.x - 1.0) < tol) mesh.right.push_back(id);
    if (std::abs(nd.y) < tol) mesh.bottom.push_back(id);
    if (std::abs(nd.y - 1.0) < tol) mesh.top.push_back(id);
  }
  mesh.area = compute_area(mesh);
  return mesh;
}

// Linear-BC DOF partition (rve.hpp:84-92, :122-131): free_index[dof] or -1.
struct DofMap {
  std::vector<int> free_index;
  int n_free = 0;
};
inline DofMap linear_bc(const Mesh& mesh) {
  DofMap dm;
  dm.free_index.assign(mesh.n_dofs(), 0);
  std::vector<char> fixed(mesh.n_dofs(), 0);
  for (const auto* set : {&mesh.left, &mesh.right, &mesh.bottom, &mesh.top})
    for (int nd : *set) fixed[2 * nd] = fixed[2 * nd + 1] = 1;
  for (int i = 0; i < mesh.n_dofs(); ++i) dm.free_index[i] = fixed[i] ? -1 : dm.n_free++;
  return dm;
}

// ---------------------------------------------------------------------------
// Dense SPD solve (the reduced system is dense n x n; the HF
// bridge uses it in place of SimplicialLDLT, rve.hpp:318-325).
struct Chol {
  int n = 0;
  std::vector<double> L;
  bool factor(const std::vector<double>& A, int n_) {
    n = n_;
    L.assign((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j) {
      double d = A[(size_t)j * n + j];
      for (int k = 0; k < j; ++k) d -= L[(size_t)j * n + k] * L[(size_t)j * n + k];
      if (!(d > 0.0)) return false;
      const double ljj = std::sqrt(d);
      L[(size_t)j * n + j] = ljj;
      for (int i = j + 1; i < n; ++i) {
        double s = A[(size_t)i * n + j];
        for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
        L[(size_t)i * n + j] = s / ljj;
      }
    }
    return true;
  }
  void solve(const double* b, double* x) const {
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) {
      double s = b[i];
      for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * y[k];
      y[i] = s / L[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= L[(size_t)k * n + i] * x[k];
      x[i] = s / L[(size_t)i * n + i];
    }
  }
};

inline double norm2(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

// ---------------------------------------------------------------------------
// HF dense micro problem (rve.hpp:220-392), linear BC only.
struct HfProblem {
  Mesh mesh;
  std::vector<Mat> mats;
  DofMap dm;
  std::vector<std::array<double, 36>> B;  // per ip
  std::vector<double> w;                   // per ip
  double volume = 0.0;
  double dt_scale = 1.0;  // fraction of the increment's dt (bisected sub-steps, rve.hpp:466)
};

inline HfProblem build_hf(const Mesh& mesh, const std::vector<Mat>& mats) {  // rve.hpp:167-185
  HfProblem p;
  p.mesh = mesh;
  p.mats = mats;
  p.dm = linear_bc(mesh);
  for (int e = 0; e < mesh.n_el(); ++e) {
    require(mesh.elements[e].mat >= 0 && mesh.elements[e].mat < (int)mats.size(), ErrorCode::config,
            "element material id out of range");
    for (int g = 0; g < 3; ++g) {
      double B[3][12];
      const double detJ = shape_eval(mesh, mesh.elements[e], kQP[g][0], kQP[g][1], B);
      std::array<double, 36> b;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 12; ++c) b[r * 12 + c] = B[r][c];
      p.B.push_back(b);
      p.w.push_back(kQW * detJ);
    }
  }
  p.volume = mesh.area;
  return p;
}

inline void affine_field(const Mesh& mesh, const double* E, std::vector<double>& u) {  // rve.hpp:43-51
  u.assign(mesh.n_dofs(), 0.0);
  const double e11 = E[0], e22 = E[1], e12 = 0.5 * E[2];
  for (int id = 0; id < mesh.n_nodes(); ++id) {
    u[2 * id] = e11 * mesh.nodes[id].x + e12 * mesh.nodes[id].y;
    u[2 * id + 1] = e12 * mesh.nodes[id].x + e22 * mesh.nodes[id].y;
  }
}

struct HfSolve {
  bool converged = false;
  int iterations = 0;
  std::vector<double> res_hist;
  std::vector<double> u_full;
  std::vector<State> states;
  std::vector<std::array<double, 3>> sigma;
  std::vector<std::array<double, 9>> C;
  std::vector<double> K;  // converged free stiffness (dense)
};

// assemble_micro (rve.hpp:220-262), dense.
inline void hf_assemble(const HfProblem& p, const std::vector<double>& u_full,
                        const std::vector<State>& s0, bool with_K, HfSolve& scratch,
                        std::vector<double>& f_full, std::vector<double>& K) {
  const int nf = p.dm.n_free;
  f_full.assign(p.mesh.n_dofs(), 0.0);
  if (with_K) K.assign((size_t)nf * nf, 0.0);
  for (int e = 0; e < p.mesh.n_el(); ++e) {
    const auto& el = p.mesh.elements[e];
    double u_el[12], f_el[12] = {0}, k_el[12][12] = {{0}};
    for (int a = 0; a < 6; ++a) {
      u_el[2 * a] = u_full[2 * el.nodes[a]];
      u_el[2 * a + 1] = u_full[2 * el.nodes[a] + 1];
    }
    for (int g = 0; g < 3; ++g) {
      const int ip = 3 * e + g;
      const double* B = p.B[ip].data();
      const double wq = p.w[ip];
      double eps[3];
      for (int r = 0; r < 3; ++r) {
        double s = 0.0;
        for (int c = 0; c < 12; ++c) s += B[r * 12 + c] * u_el[c];
        eps[r] = s;
      }
      Mat mat = p.mats[el.mat];
      mat.dt *= p.dt_scale;
      const Result3 res = update_material(mat, s0[ip], eps);
      scratch.states[ip] = res.state;
      for (int i = 0; i < 3; ++i) scratch.sigma[ip][i] = res.sigma[i];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) scratch.C[ip][3 * i + j] = res.C[i][j];
      for (int a = 0; a < 12; ++a) {
        double s = 0.0;
        for (int i = 0; i < 3; ++i) s += B[i * 12 + a] * res.sigma[i];
        f_el[a] += s * wq;
      }
      if (with_K) {
        double CB[3][12];
        for (int i = 0; i < 3; ++i)
          for (int b = 0; b < 12; ++b) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j) s += res.C[i][j] * B[j * 12 + b];
            CB[i][b] = s;
          }
        for (int a = 0; a < 12; ++a)
          for (int b = 0; b < 12; ++b) {
            double s = 0.0;
            for (int i = 0; i < 3; ++i) s += B[i * 12 + a] * CB[i][b];
            k_el[a][b] += s * wq;
          }
      }
    }
    for (int a = 0; a < 12; ++a) {
      const int ga = 2 * el.nodes[a / 2] + a % 2;
      f_full[ga] += f_el[a];
      if (!with_K) continue;
      const int fa = p.dm.free_index[ga];
      if (fa < 0) continue;
      for (int b = 0; b < 12; ++b) {
        const int gb = 2 * el.nodes[b / 2] + b % 2;
        const int fb = p.dm.free_index[gb];
        if (fb < 0) continue;
        K[(size_t)fa * nf + fb] += k_el[a][b];
      }
    }
  }
}

// micro_newton (rve.hpp:285-346) with fixed values u = E.x on the boundary.
inline HfSolve hf_newton(const HfProblem& p, const double* E, const std::vector<State>& s0,
                         const std::vector<double>& u_free_init, double tol, int max_iter) {
  const int nf = p.dm.n_free, nd = p.mesh.n_dofs();
  HfSolve r;
  r.states.resize(p.mesh.n_ips());
  r.sigma.resize(p.mesh.n_ips());
  r.C.resize(p.mesh.n_ips());
  std::vector<double> aff;
  affine_field(p.mesh, E, aff);
  auto expand = [&](const std::vector<double>& uf) {
    std::vector<double> u(nd);
    for (int i = 0; i < nd; ++i) u[i] = p.dm.free_index[i] >= 0 ? uf[p.dm.free_index[i]] : aff[i];
    return u;
  };
  auto reduce = [&](const std::vector<double>& f) {
    std::vector<double> rr(nf, 0.0);
    for (int i = 0; i < nd; ++i)
      if (p.dm.free_index[i] >= 0) rr[p.dm.free_index[i]] += f[i];
    return rr;
  };
  std::vector<double> u_free = u_free_init;
  std::vector<double> f_full, K, Kd;
  double ref = 0.0;
  for (int it = 0; it <= max_iter; ++it) {
    r.u_full = expand(u_free);
    hf_assemble(p, r.u_full, s0, true, r, f_full, K);
    const std::vector<double> res = reduce(f_full);
    const double rn = norm2(res.data(), nf);
    r.res_hist.push_back(rn);
    if (it == 0) {
      double s = 0.0;
      for (int i = 0; i < nd; ++i)
        if (p.dm.free_index[i] < 0) s += f_full[i] * f_full[i];
      ref = std::max({rn, std::sqrt(s), 1e-30});
    }
    if (rn <= tol * ref) {
      r.converged = true;
      r.iterations = it;
      r.K = K;
      return r;
    }
    if (it == max_iter) break;
    Chol ch;
    require(ch.factor(K, nf), ErrorCode::solver, "micro stiffness factorization failed");
    std::vector<double> mres(nf), du(nf);
    for (int i = 0; i < nf; ++i) mres[i] = -res[i];
    ch.solve(mres.data(), du.data());
    double alpha = 1.0, best_alpha = 1.0, best_rn = std::numeric_limits<double>::infinity();
    HfSolve tmp;
    tmp.states.resize(p.mesh.n_ips());
    tmp.sigma.resize(p.mesh.n_ips());
    tmp.C.resize(p.mesh.n_ips());
    for (int ls = 0; ls < 8; ++ls) {
      std::vector<double> ut(nf);
      for (int i = 0; i < nf; ++i) ut[i] = u_free[i] + alpha * du[i];
      hf_assemble(p, expand(ut), s0, false, tmp, f_full, Kd);
      const std::vector<double> rt = reduce(f_full);
      const double trial = norm2(rt.data(), nf);
      if (trial < best_rn) {
        best_rn = trial;
        best_alpha = alpha;
      }
      if (trial <= (1.0 - 1e-4 * alpha) * rn) break;
      alpha *= 0.5;
    }
    for (int i = 0; i < nf; ++i) u_free[i] = u_free[i] + best_alpha * du[i];
  }
  r.converged = false;
  r.iterations = max_iter;
  return r;
}

// homogenize (rve.hpp:350-392)
inline void hf_homogenize(const HfProblem& p, const HfSolve& m, double* sigma, double* C) {
  require(m.converged, ErrorCode::solver, "homogenize requires a converged micro state");
  const int nf = p.dm.n_free, nd = p.mesh.n_dofs();
  double s[3] = {0, 0, 0};
  for (int ip = 0; ip < p.mesh.n_ips(); ++ip)
    for (int i = 0; i < 3; ++i) s[i] += p.w[ip] * m.sigma[ip][i];
  for (int i = 0; i < 3; ++i) sigma[i] = s[i] / p.volume;
  std::vector<double> rhs_full((size_t)nd * 3, 0.0);
  double c_avg[9] = {0};
  for (int ip = 0; ip < p.mesh.n_ips(); ++ip) {
    const auto& el = p.mesh.elements[ip / 3];
    const double* B = p.B[ip].data();
    for (int a = 0; a < 12; ++a) {
      const int ga = 2 * el.nodes[a / 2] + a % 2;
      for (int j = 0; j < 3; ++j) {
        double t = 0.0;
        for (int i = 0; i < 3; ++i) t += B[i * 12 + a] * m.C[ip][3 * i + j];
        rhs_full[(size_t)ga * 3 + j] += t * p.w[ip];
      }
    }
    for (int k = 0; k < 9; ++k) c_avg[k] += p.w[ip] * m.C[ip][k];
  }
  Chol ch;
  require(ch.factor(m.K, nf), ErrorCode::solver, "homogenize: singular converged stiffness");
  double c_hom[9];
  for (int k = 0; k < 9; ++k) c_hom[k] = c_avg[k];
  for (int j = 0; j < 3; ++j) {
    std::vector<double> rhs(nf, 0.0), h(nf);
    for (int i = 0; i < nd; ++i)
      if (p.dm.free_index[i] >= 0) rhs[p.dm.free_index[i]] += rhs_full[(size_t)i * 3 + j];
    for (int i = 0; i < nf; ++i) rhs[i] = -rhs[i];
    ch.solve(rhs.data(), h.data());
    std::vector<double> h_full(nd, 0.0);
    for (int i = 0; i < nd; ++i)
      if (p.dm.free_index[i] >= 0) h_full[i] = h[p.dm.free_index[i]];
    for (int ip = 0; ip < p.mesh.n_ips(); ++ip) {
      const auto& el = p.mesh.elements[ip / 3];
      const double* B = p.B[ip].data();
      double he[12];
      for (int a = 0; a < 6; ++a) {
        he[2 * a] = h_full[2 * el.nodes[a]];
        he[2 * a + 1] = h_full[2 * el.nodes[a] + 1];
      }
      double bh[3];
      for (int r = 0; r < 3; ++r) {
        double t = 0.0;
        for (int c = 0; c < 12; ++c) t += B[r * 12 + c] * he[c];
        bh[r] = t;
      }
      for (int i = 0; i < 3; ++i) {
        double t = 0.0;
        for (int k = 0; k < 3; ++k) t += m.C[ip][3 * i + k] * bh[k];
        c_hom[3 * i + j] += p.w[ip] * t;
      }
    }
  }
  for (int k = 0; k < 9; ++k) C[k] = c_hom[k] / p.volume;
}

// ---------------------------------------------------------------------------
// Hyper-ROM model (offline): Φ, cubature, G_q. Decisions pinned in DESIGN.md.
constexpr std::uint64_t kSeedPhi = 0x243F6A8885A308D3ull;
constexpr std::uint64_t kSeedCub = 0x13198A2E03707344ull;
constexpr std::uint64_t kSeedPath = 0xA4093822299F31D0ull;

inline std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline std::uint64_t path_seed(std::uint64_t seed, std::int64_t p) {
  return splitmix64(seed ^ kSeedPath) ^ splitmix64(static_cast<std::uint64_t>(p));
}

struct Model {
  int n = 0, K = 0, n_free = 0;
  double volume = 0.0;
  std::vector<double> phi;  // [n_free][n]
  std::vector<double> G;    // [K][3][n]
  std::vector<double> w;
  std::vector<int> ip, mat;
};

// Householder thin QR, Q = H_0 ... H_{n-1} [I; 0] (rows m, cols n), in place.
inline void thin_q(std::vector<double>& A, int m, int n) {
  std::vector<std::vector<double>> V(n);
  std::vector<double> tau(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double nx = 0.0;
    for (int i = j; i < m; ++i) nx += A[(size_t)i * n + j] * A[(size_t)i * n + j];
    nx = std::sqrt(nx);
    const double x0 = A[(size_t)j * n + j];
    const double alpha = x0 >= 0.0 ? -nx : nx;
    std::vector<double> v(m - j);
    for (int i = j; i < m; ++i) v[i - j] = A[(size_t)i * n + j];
    v[0] = v[0] - alpha;
    double vn = 0.0;
    for (double t : v) vn += t * t;
    if (vn > 0.0) {
      tau[j] = 2.0 / vn;
      for (int c = j; c < n; ++c) {
        double s = 0.0;
        for (int i = j; i < m; ++i) s += v[i - j] * A[(size_t)i * n + c];
        const double ts = tau[j] * s;
        for (int i = j; i < m; ++i) A[(size_t)i * n + c] = A[(size_t)i * n + c] - ts * v[i - j];
      }
    }
    V[j] = std::move(v);
  }
  std::vector<double> Q((size_t)m * n, 0.0);
  for (int j = 0; j < n; ++j) Q[(size_t)j * n + j] = 1.0;
  for (int j = n - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    const auto& v = V[j];
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int i = j; i < m; ++i) s += v[i - j] * Q[(size_t)i * n + c];
      const double ts = tau[j] * s;
      for (int i = j; i < m; ++i) Q[(size_t)i * n + c] = Q[(size_t)i * n + c] - ts * v[i - j];
    }
  }
  A.swap(Q);
}

inline Model build_model(const Mesh& mesh, int n, int K, std::uint64_t seed) {
  HfProblem hf = build_hf(mesh, {Mat{}, Mat{}});  // B and w only; materials irrelevant here
  const int nf = hf.dm.n_free;
  const int n_ips = mesh.n_ips();
  Model md;
  md.n_free = nf;
  md.volume = mesh.area;
  if (n == 0) {  // identity basis on free DOFs (bridge)
    n = nf;
    md.phi.assign((size_t)nf * n, 0.0);
    for (int i = 0; i < nf; ++i) md.phi[(size_t)i * n + i] = 1.0;
  } else {
    require(n >= 1 && n <= nf, ErrorCode::config, "mode count out of range");
    md.phi.assign((size_t)nf * n, 0.0);
    Rng rng(seed ^ kSeedPhi);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < nf; ++i) md.phi[(size_t)i * n + j] = rng.normal();
    thin_q(md.phi, nf, n);
  }
  md.n = n;
  if (K == 0) {  // full rule, own weights
    K = n_ips;
    for (int q = 0; q < n_ips; ++q) {
      md.ip.push_back(q);
      md.w.push_back(hf.w[q]);
    }
  } else {
    require(K >= 1 && K <= n_ips, ErrorCode::config, "cubature size out of range");
    Rng rng(seed ^ kSeedCub);
    std::vector<int> ids(n_ips);
    for (int i = 0; i < n_ips; ++i) ids[i] = i;
    for (int i = 0; i < K; ++i) {
      const int j = i + rng.uniform_int(n_ips - i);
      std::swap(ids[i], ids[j]);
    }
    const double scale = mesh.area / K;
    for (int i = 0; i < K; ++i) {
      md.ip.push_back(ids[i]);
      md.w.push_back(rng.uniform(0.5, 1.5) * scale);
    }
  }
  md.K = K;
  md.G.assign((size_t)K * 3 * n, 0.0);
  for (int q = 0; q < K; ++q) {
    const int ip = md.ip[q];
    const auto& el = mesh.elements[ip / 3];
    md.mat.push_back(el.mat);
    const double* B = hf.B[ip].data();
    int fidx[12];
    for (int d = 0; d < 12; ++d) fidx[d] = hf.dm.free_index[2 * el.nodes[d / 2] + d % 2];
    for (int i = 0; i < 3; ++i)
      for (int a = 0; a < n; ++a) {
        double s = 0.0;
        for (int d = 0; d < 12; ++d)
          if (fidx[d] >= 0) s += B[i * 12 + d] * md.phi[(size_t)fidx[d] * n + a];
        md.G[((size_t)q * 3 + i) * n + a] = s;
      }
  }
  return md;
}

// Seeded macro strain paths (BASELINE.json configs 0 and 1).
inline void make_path(int kind, std::uint64_t seed, std::int64_t p, int n_incr, double* E) {
  Rng rng(path_seed(seed, p));
  if (kind == 0) {
    const double s = rng.uniform(0.5, 1.5);
    const double th = rng.uniform(0.0, std::numbers::pi);
    const double c = std::cos(th), sn = std::sin(th);
    const double e = 0.05 * s;
    const double end[3] = {e * (c * c), e * (sn * sn), e * (2.0 * sn * c)};
    for (int k = 1; k <= n_incr; ++k) {
      const double f = static_cast<double>(k) / n_incr;
      for (int i = 0; i < 3; ++i) E[(k - 1) * 3 + i] = end[i] * f;
    }
  } else if (kind == 1) {
    const double a = rng.uniform(-0.03, 0.03);
    const double b = rng.uniform(-0.02, 0.02);
    const double end[3] = {a, 0.0, 2.0 * b};
    const int half = n_incr / 2;
    for (int k = 1; k <= n_incr; ++k) {
      const double f = k <= half ? static_cast<double>(k) / half : static_cast<double>(n_incr - k) / half;
      for (int i = 0; i < 3; ++i) E[(k - 1) * 3 + i] = end[i] * f;
    }
  } else {
    fail(ErrorCode::config, "unknown path kind");
  }
}

// ---------------------------------------------------------------------------
// Hyper-ROM online path: hyper_assemble + reduced Newton
// mirroring micro_newton (rve.hpp:285-346) + condensation mirroring
// homogenize (rve.hpp:350-392) + increments mirroring run_trajectory
// (rve.hpp:448-494).
struct Hrom {
  int n = 0, K = 0;
  std::vector<double> G, w;
  std::vector<int> mat;
  std::vector<Mat> mats;
  double volume = 0.0;
};

struct Assembly {
  std::vector<double> r, Kaa, KaE;
  double C_EE[9], S_raw[3];
  std::vector<State> states;
  std::vector<uint8_t> plastic;
  int plastic_count = 0;
  double rn = 0.0;
};

// ε_q = E + G_q α (decision 6) ; update_material ; weighted sums.
// dt_scale: the fraction of the increment a (bisected) sub-step covers; a creep
// material integrates over PathStep::dt x dt_scale (rve.hpp:466, MicroOptions::dt)
inline void hrom_assemble(const Hrom& h, const double* alpha, const double* E,
                          const std::vector<State>& s0, bool with_K, Assembly& A, double dt_scale = 1.0) {
  const int n = h.n;
  A.r.assign(n, 0.0);
  if (with_K) {
    A.Kaa.assign((size_t)n * n, 0.0);
    A.KaE.assign((size_t)n * 3, 0.0);
  }
  for (int k = 0; k < 9; ++k) A.C_EE[k] = 0.0;
  for (int i = 0; i < 3; ++i) A.S_raw[i] = 0.0;
  A.states.resize(h.K);
  A.plastic.assign(h.K, 0);
  A.plastic_count = 0;
  std::vector<double> H((size_t)3 * n);
  for (int q = 0; q < h.K; ++q) {
    const double* Gq = h.G.data() + (size_t)q * 3 * n;
    double eps[3];
    for (int i = 0; i < 3; ++i) {
      double s = 0.0;
      for (int a = 0; a < n; ++a) s += Gq[i * n + a] * alpha[a];
      eps[i] = E[i] + s;
    }
    Mat mq = h.mats[h.mat[q]];
    mq.dt *= dt_scale;
    const Result3 res = update_material(mq, s0[q], eps);
    A.states[q] = res.state;
    A.plastic[q] = res.plastic ? 1 : 0;
    A.plastic_count += res.plastic ? 1 : 0;
    const double wq = h.w[q];
    double f[3];
    for (int i = 0; i < 3; ++i) {
      f[i] = wq * res.sigma[i];
      A.S_raw[i] += f[i];
    }
    for (int a = 0; a < n; ++a) A.r[a] += Gq[a] * f[0] + Gq[n + a] * f[1] + Gq[2 * n + a] * f[2];
    if (!with_K) continue;
    double wC[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        wC[i][j] = wq * res.C[i][j];
        A.C_EE[3 * i + j] += wC[i][j];
      }
    for (int i = 0; i < 3; ++i)
      for (int b = 0; b < n; ++b) H[i * n + b] = wC[i][0] * Gq[b] + wC[i][1] * Gq[n + b] + wC[i][2] * Gq[2 * n + b];
    for (int a = 0; a < n; ++a) {
      for (int j = 0; j < 3; ++j)
        A.KaE[a * 3 + j] += Gq[a] * wC[0][j] + Gq[n + a] * wC[1][j] + Gq[2 * n + a] * wC[2][j];
      double* Krow = A.Kaa.data() + (size_t)a * n;
      const double g0 = Gq[a], g1 = Gq[n + a], g2 = Gq[2 * n + a];
      for (int b = 0; b < n; ++b) Krow[b] += g0 * H[b] + g1 * H[n + b] + g2 * H[2 * n + b];
    }
  }
  A.rn = norm2(A.r.data(), n);
}

struct PointResult {
  bool converged = false;
  int iterations = 0;
  double rn = 0.0;
  std::vector<double> alpha;
  Assembly A;  // assembly at the converged iterate
};

inline PointResult hrom_newton(const Hrom& h, const std::vector<double>& alpha0, const double* E,
                               const std::vector<State>& s0, double tol, int max_iter, double dt_scale = 1.0) {
  const int n = h.n;
  PointResult pr;
  std::vector<double> alpha = alpha0, du(n), mres(n), trial_alpha(n);
  Assembly& A = pr.A;
  Assembly T;
  double ref = 0.0;
  for (int it = 0; it <= max_iter; ++it) {
    hrom_assemble(h, alpha.data(), E, s0, true, A, dt_scale);
    const double rn = A.rn;
    if (it == 0) ref = std::max({rn, norm2(A.S_raw, 3), 1e-30});
    if (rn <= tol * ref) {
      pr.converged = true;
      pr.iterations = it;
      pr.rn = rn;
      pr.alpha = alpha;
      return pr;
    }
    if (it == max_iter) {
      pr.rn = rn;
      break;
    }
    Chol ch;
    require(ch.factor(A.Kaa, n), ErrorCode::solver, "reduced stiffness factorization failed");
    for (int i = 0; i < n; ++i) mres[i] = -A.r[i];
    ch.solve(mres.data(), du.data());
    double a = 1.0, best_a = 1.0, best_rn = std::numeric_limits<double>::infinity();
    for (int ls = 0; ls < 8; ++ls) {
      for (int i = 0; i < n; ++i) trial_alpha[i] = alpha[i] + a * du[i];
      hrom_assemble(h, trial_alpha.data(), E, s0, false, T, dt_scale);
      const double trial = T.rn;
      if (trial < best_rn) {
        best_rn = trial;
        best_a = a;
      }
      if (trial <= (1.0 - 1e-4 * a) * rn) break;
      a *= 0.5;
    }
    for (int i = 0; i < n; ++i) alpha[i] = alpha[i] + best_a * du[i];
  }
  pr.converged = false;
  pr.iterations = max_iter;
  pr.alpha = alpha;
  return pr;
}

// condensation: C = (C_EE - K_Eα K_αα^-1 K_αE) / V via 3 sensitivity solves
// h_j = K^-1 (-K_αE e_j) (homogenize, rve.hpp:372-390); Σ = Σ_raw / V.
inline void hrom_condense(const Hrom& h, const Assembly& A, double* sigma, double* C) {
  const int n = h.n;
  for (int i = 0; i < 3; ++i) sigma[i] = A.S_raw[i] / h.volume;
  Chol ch;
  require(ch.factor(A.Kaa, n), ErrorCode::solver, "condensation: singular reduced stiffness");
  double c[9];
  for (int k = 0; k < 9; ++k) c[k] = A.C_EE[k];
  std::vector<double> rhs(n), hj(n);
  for (int j = 0; j < 3; ++j) {
    for (int a = 0; a < n; ++a) rhs[a] = -A.KaE[a * 3 + j];
    ch.solve(rhs.data(), hj.data());
    for (int i = 0; i < 3; ++i) {
      double t = 0.0;
      for (int a = 0; a < n; ++a) t += A.KaE[a * 3 + i] * hj[a];
      c[3 * i + j] += t;
    }
  }
  for (int k = 0; k < 9; ++k) C[k] = c[k] / h.volume;
}

template <class Fn>
void parallel_for(std::int64_t n, int n_threads, Fn&& fn) {  // common.hpp:109-132 (cyclic)
  if (n_threads <= 1 || n <= 1) {
    for (std::int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  n_threads = (int)std::min<std::int64_t>(n_threads, n);
  std::vector<std::thread> pool;
  std::exception_ptr first_error;
  std::mutex mx;
  for (int t = 0; t < n_threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (std::int64_t i = t; i < n; i += n_threads) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mx);
        if (!first_error) first_error = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (first_error) std::rethrow_exception(first_error);
}

inline void hrom_point_trajectory(const Hrom& h, std::int64_t pi, int n_incr, const double* Ep,
                                  double tol, int max_iter, int max_bis, orc_hrom_out_t* out) {
  const int n = h.n, K = h.K;
  std::vector<double> alpha_c(n, 0.0);
  std::vector<State> states(K);
  double E_prev[3] = {0, 0, 0};
  bool dead = false;
  int dead_code = 0;  // the error that ended the trajectory, reported for every later increment
  for (int k = 0; k < n_incr; ++k) {
    const std::int64_t o = pi * n_incr + k;
    const double* Ek = Ep + 3 * k;
    int iters = 0, bis = 0, status = 0;
    double sig[3] = {NAN, NAN, NAN}, C[9];
    for (double& c : C) c = NAN;
    double rn = NAN;
    int pc = 0;
    if (!dead) {
      double done = 0.0, frac = 1.0;
      while (done < 1.0 - 1e-12) {
        const double target = std::min(1.0, done + frac);
        double E[3];
        for (int i = 0; i < 3; ++i) E[i] = E_prev[i] + (Ek[i] - E_prev[i]) * target;
        PointResult pr;
        try {
          pr = hrom_newton(h, alpha_c, E, states, tol, max_iter, target - done);
        } catch (const Error& e) {
          status = 1 + (int)e.code;
          dead = true;
          break;
        }
        iters += pr.iterations;
        rn = pr.rn;
        if (!pr.converged) {
          if (++bis > max_bis) {
            status = 1 + (int)ErrorCode::solver;
            dead = true;
            break;
          }
          frac *= 0.5;
          continue;
        }
        try {
          hrom_condense(h, pr.A, sig, C);
        } catch (const Error& e) {
          status = 1 + (int)e.code;
          dead = true;
          break;
        }
        states = pr.A.states;
        alpha_c = pr.alpha;
        pc = pr.A.plastic_count;
        done = target;
        if (out->plastic_flags)
          std::memcpy(out->plastic_flags + (size_t)o * K, pr.A.plastic.data(), (size_t)K);
      }
    } else {
      status = dead_code;
    }
    if (dead && !dead_code) dead_code = status;
    if (status != 0) {  // run_trajectory throws: no response for this increment
      for (double& s : sig) s = NAN;
      for (double& c : C) c = NAN;
    }
    if (out->sigma) std::memcpy(out->sigma + o * 3, sig, sizeof sig);
    if (out->C) std::memcpy(out->C + o * 9, C, sizeof C);
    if (out->iters) out->iters[o] = iters;
    if (out->plastic_count) out->plastic_count[o] = pc;
    if (out->res_norm) out->res_norm[o] = rn;
    if (out->status) out->status[o] = status;
    if (out->bisections) out->bisections[o] = bis;
    for (int i = 0; i < 3; ++i) E_prev[i] = Ek[i];
  }
  if (out->alpha) std::memcpy(out->alpha + pi * n, alpha_c.data(), sizeof(double) * n);
  if (out->state)
    for (int q = 0; q < K; ++q) {
      double* s = out->state + ((size_t)pi * K + q) * 6;
      for (int c = 0; c < 4; ++c) s[c] = states[q].ep[c];
      s[4] = states[q].eq;
      s[5] = states[q].s33;
    }
}

// ---------------------------------------------------------------------------
// Finite strain, Biot stress (BASELINE config 2). PARITY UNPINNED: the
// reference contains no finite-strain code (SPEC.md:8 declares it out of
// scope; the paper's biot_stress section is absent from PAPER.md:19-20), so
// this is our formulation, checked only for self-consistency (FD tangents,
// objectivity, small-strain limit) in tests/test_oracle_fs.py:
//   F = R U (2-D polar decomposition: R = rotation by θ = atan2(F10-F01, F00+F11),
//   cos θ and sin θ formed directly as (F00+F11)/ρ, (F10-F01)/ρ),
//   Biot strain U - I -> the pinned small-strain update4 (J2 / elastic) gives
//   the Biot stress T, P = R T (first Piola-Kirchhoff), A = dP/dF closed form.
// Components are ordered (F00, F01, F10, F11) = (dx/dX, dx/dY, dy/dX, dy/dY).
struct FsResult {
  double P[4];
  double A[16];  // A[r][s] = dP_r / dF_s
  State state;
  bool plastic;
};

inline FsResult update_biot(const Mat& m, const State& s0, const double* F) {
  const double num = F[2] - F[1], den = F[0] + F[3];
  const double rho2 = num * num + den * den;
  const double rho = std::sqrt(rho2);
  const double c = den / rho, s = num / rho;  // R(θ), θ = atan2(num, den)
  // U = R^T F
  const double U00 = c * F[0] + s * F[2], U01 = c * F[1] + s * F[3];
  const double U10 = -s * F[0] + c * F[2], U11 = -s * F[1] + c * F[3];
  const double e4[4] = {U00 - 1.0, U11 - 1.0, 0.0, 0.5 * (U01 + U10)};
  const Result4 r4 = update4(m, s0, e4);
  const double T00 = r4.sigma[0], T11 = r4.sigma[1], T01 = r4.sigma[3];
  FsResult out;
  out.P[0] = c * T00 - s * T01;
  out.P[1] = c * T01 - s * T11;
  out.P[2] = s * T00 + c * T01;
  out.P[3] = s * T01 + c * T11;
  out.state = r4.state;
  out.plastic = r4.plastic;
  const double g[4] = {-num / rho2, -den / rho2, den / rho2, -num / rho2};  // dθ/dF
  // R J T with J = [[0,-1],[1,0]]: (RJ) = [[-s,-c],[c,-s]]
  const double RJT00 = -s * T00 - c * T01, RJT01 = -s * T01 - c * T11;
  const double RJT10 = c * T00 - s * T01, RJT11 = c * T01 - s * T11;
  for (int k = 0; k < 4; ++k) {
    const double dth = g[k];
    double dF[4] = {0, 0, 0, 0};
    dF[k] = 1.0;
    // dU = -J U dθ + R^T dF,   -J U = [[U10, U11], [-U00, -U01]]
    const double dU00 = U10 * dth + (c * dF[0] + s * dF[2]);
    const double dU01 = U11 * dth + (c * dF[1] + s * dF[3]);
    const double dU10 = -U00 * dth + (-s * dF[0] + c * dF[2]);
    const double dU11 = -U01 * dth + (-s * dF[1] + c * dF[3]);
    const double de[4] = {dU00, dU11, 0.0, 0.5 * (dU01 + dU10)};
    double dT[4];
    for (int i = 0; i < 4; ++i) {
      double t = 0.0;
      for (int j = 0; j < 4; ++j) t += r4.D[i][j] * de[j];
      dT[i] = t;
    }
    const double d00 = dT[0], d11 = dT[1], d01 = dT[3];
    out.A[0 * 4 + k] = RJT00 * dth + (c * d00 - s * d01);
    out.A[1 * 4 + k] = RJT01 * dth + (c * d01 - s * d11);
    out.A[2 * 4 + k] = RJT10 * dth + (s * d00 + c * d01);
    out.A[3 * 4 + k] = RJT11 * dth + (s * d01 + c * d11);
  }
  return out;
}

// Dense LU with partial pivoting (the finite-strain K_aa is not symmetric).
struct Lu {
  int n = 0;
  std::vector<double> a;
  std::vector<int> piv;
  bool factor(const std::vector<double>& A, int n_) {
    n = n_;
    a = A;
    piv.resize(n);
    for (int j = 0; j < n; ++j) {
      int p = j;
      double best = std::abs(a[(size_t)j * n + j]);
      for (int i = j + 1; i < n; ++i)
        if (std::abs(a[(size_t)i * n + j]) > best) {
          best = std::abs(a[(size_t)i * n + j]);
          p = i;
        }
      if (!(best > 0.0)) return false;
      piv[j] = p;
      if (p != j)
        for (int k = 0; k < n; ++k) std::swap(a[(size_t)j * n + k], a[(size_t)p * n + k]);
      const double inv = 1.0 / a[(size_t)j * n + j];
      for (int i = j + 1; i < n; ++i) {
        const double l = a[(size_t)i * n + j] * inv;
        a[(size_t)i * n + j] = l;
        for (int k = j + 1; k < n; ++k) a[(size_t)i * n + k] -= l * a[(size_t)j * n + k];
      }
    }
    return true;
  }
  void solve(const double* b, double* x) const {
    std::vector<double> y(b, b + n);
    for (int j = 0; j < n; ++j) std::swap(y[j], y[piv[j]]);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) y[i] -= a[(size_t)i * n + k] * y[k];
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= a[(size_t)i * n + k] * x[k];
      x[i] = s / a[(size_t)i * n + i];
    }
  }
};

// 4-row displacement-gradient operator at an IP from the strain operator B
// (mesh.hpp:106-113): rows (dwx/dX, dwx/dY, dwy/dX, dwy/dY).
inline void grad_operator(const double* B, double Bg[4][12]) {
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 12; ++c) Bg[r][c] = 0.0;
  for (int a = 0; a < 6; ++a) {
    Bg[0][2 * a] = B[0 * 12 + 2 * a];          // dN/dX
    Bg[1][2 * a] = B[2 * 12 + 2 * a];          // dN/dY
    Bg[2][2 * a + 1] = B[2 * 12 + 2 * a + 1];  // dN/dX
    Bg[3][2 * a + 1] = B[1 * 12 + 2 * a + 1];  // dN/dY
  }
}

// G4_q = Bg_q Φ[dofs(el(q))] for the cubature of a built model (same Φ, ids, weights).
inline std::vector<double> build_g4(const Mesh& mesh, const Model& md) {
  HfProblem hf = build_hf(mesh, {Mat{}, Mat{}});
  const int n = md.n;
  std::vector<double> G4((size_t)md.K * 4 * n, 0.0);
  for (int q = 0; q < md.K; ++q) {
    const int ip = md.ip[q];
    const auto& el = mesh.elements[ip / 3];
    double Bg[4][12];
    grad_operator(hf.B[ip].data(), Bg);
    int fidx[12];
    for (int d = 0; d < 12; ++d) fidx[d] = hf.dm.free_index[2 * el.nodes[d / 2] + d % 2];
    for (int r = 0; r < 4; ++r)
      for (int a = 0; a < n; ++a) {
        double s = 0.0;
        for (int d = 0; d < 12; ++d)
          if (fidx[d] >= 0) s += Bg[r][d] * md.phi[(size_t)fidx[d] * n + a];
        G4[((size_t)q * 4 + r) * n + a] = s;
      }
  }
  return G4;
}

// config-2 paths: H ~ U[-0.08, 0.08]^4 (H00, H01, H10, H11), redrawn until
// det(I + H) > 0.8; increments H_k = (k / n_incr) H.
inline void make_path_fs(std::uint64_t seed, std::int64_t p, int n_incr, double* Hout) {
  Rng rng(path_seed(seed, p));
  double H[4];
  while (true) {
    for (double& h : H) h = rng.uniform(-0.08, 0.08);
    const double det = (1.0 + H[0]) * (1.0 + H[3]) - H[1] * H[2];
    if (det > 0.8) break;
  }
  for (int k = 1; k <= n_incr; ++k) {
    const double f = static_cast<double>(k) / n_incr;
    for (int i = 0; i < 4; ++i) Hout[(k - 1) * 4 + i] = H[i] * f;
  }
}

struct HromFs {
  int n = 0, K = 0;
  std::vector<double> G;  // [K][4][n]
  std::vector<double> w;
  std::vector<int> mat;
  std::vector<Mat> mats;
  double volume = 0.0;
};

struct AssemblyFs {
  std::vector<double> r, Kaa, KaF, KFa;  // n, n*n, n*4, 4*n
  double CFF[16], P_raw[4];
  std::vector<State> states;
  std::vector<uint8_t> plastic;
  int plastic_count = 0;
  double rn = 0.0;
};

// F_q = I + H + G4_q α ; P, A per point ; weighted sums.
inline void fs_assemble(const HromFs& h, const double* alpha, const double* H, const std::vector<State>& s0,
                        bool with_K, AssemblyFs& A) {
  const int n = h.n;
  A.r.assign(n, 0.0);
  if (with_K) {
    A.Kaa.assign((size_t)n * n, 0.0);
    A.KaF.assign((size_t)n * 4, 0.0);
    A.KFa.assign((size_t)4 * n, 0.0);
  }
  for (double& v : A.CFF) v = 0.0;
  for (double& v : A.P_raw) v = 0.0;
  A.states.resize(h.K);
  A.plastic.assign(h.K, 0);
  A.plastic_count = 0;
  const double I4[4] = {1.0, 0.0, 0.0, 1.0};
  std::vector<double> Hq((size_t)4 * n);
  for (int q = 0; q < h.K; ++q) {
    const double* Gq = h.G.data() + (size_t)q * 4 * n;
    double F[4];
    for (int r = 0; r < 4; ++r) {
      double s = 0.0;
      for (int a = 0; a < n; ++a) s += Gq[r * n + a] * alpha[a];
      F[r] = (I4[r] + H[r]) + s;
    }
    const FsResult res = update_biot(h.mats[h.mat[q]], s0[q], F);
    A.states[q] = res.state;
    A.plastic[q] = res.plastic ? 1 : 0;
    A.plastic_count += res.plastic ? 1 : 0;
    const double wq = h.w[q];
    double wP[4];
    for (int r = 0; r < 4; ++r) {
      wP[r] = wq * res.P[r];
      A.P_raw[r] += wP[r];
    }
    for (int a = 0; a < n; ++a)
      A.r[a] += Gq[a] * wP[0] + Gq[n + a] * wP[1] + Gq[2 * n + a] * wP[2] + Gq[3 * n + a] * wP[3];
    if (!with_K) continue;
    double wA[4][4];
    for (int r = 0; r < 4; ++r)
      for (int s = 0; s < 4; ++s) {
        wA[r][s] = wq * res.A[r * 4 + s];
        A.CFF[r * 4 + s] += wA[r][s];
      }
    for (int r = 0; r < 4; ++r)  // Hq = wA G_q (4 x n)
      for (int b = 0; b < n; ++b)
        Hq[r * n + b] = wA[r][0] * Gq[b] + wA[r][1] * Gq[n + b] + wA[r][2] * Gq[2 * n + b] + wA[r][3] * Gq[3 * n + b];
    for (int r = 0; r < 4; ++r)
      for (int b = 0; b < n; ++b) A.KFa[r * n + b] += Hq[r * n + b];
    for (int a = 0; a < n; ++a) {
      const double g0 = Gq[a], g1 = Gq[n + a], g2 = Gq[2 * n + a], g3 = Gq[3 * n + a];
      for (int s = 0; s < 4; ++s) A.KaF[a * 4 + s] += g0 * wA[0][s] + g1 * wA[1][s] + g2 * wA[2][s] + g3 * wA[3][s];
      double* Krow = A.Kaa.data() + (size_t)a * n;
      for (int b = 0; b < n; ++b) Krow[b] += g0 * Hq[b] + g1 * Hq[n + b] + g2 * Hq[2 * n + b] + g3 * Hq[3 * n + b];
    }
  }
  A.rn = norm2(A.r.data(), n);
}

struct PointResultFs {
  bool converged = false;
  int iterations = 0;
  double rn = 0.0;
  std::vector<double> alpha;
  AssemblyFs A;
};

inline PointResultFs fs_newton(const HromFs& h, const std::vector<double>& alpha0, const double* H,
                               const std::vector<State>& s0, double tol, int max_iter) {
  const int n = h.n;
  PointResultFs pr;
  std::vector<double> alpha = alpha0, du(n), mres(n), ta(n);
  AssemblyFs& A = pr.A;
  AssemblyFs T;
  double ref = 0.0;
  for (int it = 0; it <= max_iter; ++it) {
    fs_assemble(h, alpha.data(), H, s0, true, A);
    const double rn = A.rn;
    if (it == 0) ref = std::max({rn, norm2(A.P_raw, 4), 1e-30});
    if (rn <= tol * ref) {
      pr.converged = true;
      pr.iterations = it;
      pr.rn = rn;
      pr.alpha = alpha;
      return pr;
    }
    if (it == max_iter) {
      pr.rn = rn;
      break;
    }
    Lu lu;
    require(lu.factor(A.Kaa, n), ErrorCode::solver, "reduced stiffness factorization failed");
    for (int i = 0; i < n; ++i) mres[i] = -A.r[i];
    lu.solve(mres.data(), du.data());
    double a = 1.0, best_a = 1.0, best_rn = std::numeric_limits<double>::infinity();
    for (int ls = 0; ls < 8; ++ls) {
      for (int i = 0; i < n; ++i) ta[i] = alpha[i] + a * du[i];
      fs_assemble(h, ta.data(), H, s0, false, T);
      if (T.rn < best_rn) {
        best_rn = T.rn;
        best_a = a;
      }
      if (T.rn <= (1.0 - 1e-4 * a) * rn) break;
      a *= 0.5;
    }
    for (int i = 0; i < n; ++i) alpha[i] = alpha[i] + best_a * du[i];
  }
  pr.converged = false;
  pr.iterations = max_iter;
  pr.alpha = alpha;
  return pr;
}

// A_M = (C_FF - K_Fa K_aa^-1 K_aF) / V ; P_M = P_raw / V
inline void fs_condense(const HromFs& h, const AssemblyFs& A, double* P, double* AM) {
  const int n = h.n;
  for (int r = 0; r < 4; ++r) P[r] = A.P_raw[r] / h.volume;
  Lu lu;
  require(lu.factor(A.Kaa, n), ErrorCode::solver, "condensation: singular reduced stiffness");
  double c[16];
  for (int k = 0; k < 16; ++k) c[k] = A.CFF[k];
  std::vector<double> rhs(n), y(n);
  for (int s = 0; s < 4; ++s) {
    for (int a = 0; a < n; ++a) rhs[a] = -A.KaF[a * 4 + s];
    lu.solve(rhs.data(), y.data());
    for (int r = 0; r < 4; ++r) {
      double t = 0.0;
      for (int a = 0; a < n; ++a) t += A.KFa[r * n + a] * y[a];
      c[r * 4 + s] += t;
    }
  }
  for (int k = 0; k < 16; ++k) AM[k] = c[k] / h.volume;
}

inline void fs_point_trajectory(const HromFs& h, std::int64_t pi, int n_incr, const double* Hp, double tol,
                                int max_iter, int max_bis, orc_hrom_out_t* out) {
  const int n = h.n, K = h.K;
  std::vector<double> alpha_c(n, 0.0);
  std::vector<State> states(K);
  double H_prev[4] = {0, 0, 0, 0};
  bool dead = false;
  int dead_code = 0;  // the error that ended the trajectory, reported for every later increment
  for (int k = 0; k < n_incr; ++k) {
    const std::int64_t o = pi * n_incr + k;
    const double* Hk = Hp + 4 * k;
    int iters = 0, bis = 0, status = 0, pc = 0;
    double P[4], AM[16], rn = NAN;
    for (double& v : P) v = NAN;
    for (double& v : AM) v = NAN;
    if (!dead) {
      double done = 0.0, frac = 1.0;
      while (done < 1.0 - 1e-12) {
        const double target = std::min(1.0, done + frac);
        double H[4];
        for (int i = 0; i < 4; ++i) H[i] = H_prev[i] + (Hk[i] - H_prev[i]) * target;
        PointResultFs pr;
        try {
          pr = fs_newton(h, alpha_c, H, states, tol, max_iter);
        } catch (const Error& e) {
          status = 1 + (int)e.code;
          dead = true;
          break;
        }
        iters += pr.iterations;
        rn = pr.rn;
        if (!pr.converged) {
          if (++bis > max_bis) {
            status = 1 + (int)ErrorCode::solver;
            dead = true;
            break;
          }
          frac *= 0.5;
          continue;
        }
        try {
          fs_condense(h, pr.A, P, AM);
        } catch (const Error& e) {
          status = 1 + (int)e.code;
          dead = true;
          break;
        }
        states = pr.A.states;
        alpha_c = pr.alpha;
        pc = pr.A.plastic_count;
        if (out->plastic_flags)
          std::memcpy(out->plastic_flags + (size_t)o * K, pr.A.plastic.data(), (size_t)K);
        done = target;
      }
    } else {
      status = dead_code;
    }
    if (dead && !dead_code) dead_code = status;
    if (status != 0) {
      for (double& v : P) v = NAN;
      for (double& v : AM) v = NAN;
    }
    if (out->sigma) std::memcpy(out->sigma + o * 4, P, sizeof P);
    if (out->C) std::memcpy(out->C + o * 16, AM, sizeof AM);
    if (out->iters) out->iters[o] = iters;
    if (out->plastic_count) out->plastic_count[o] = pc;
    if (out->res_norm) out->res_norm[o] = rn;
    if (out->status) out->status[o] = status;
    if (out->bisections) out->bisections[o] = bis;
    for (int i = 0; i < 4; ++i) H_prev[i] = Hk[i];
  }
  if (out->alpha) std::memcpy(out->alpha + pi * n, alpha_c.data(), sizeof(double) * n);
  if (out->state)
    for (int q = 0; q < K; ++q) {
      double* s = out->state + ((size_t)pi * K + q) * 6;
      for (int c = 0; c < 4; ++c) s[c] = states[q].ep[c];
      s[4] = states[q].eq;
      s[5] = states[q].s33;
    }
}

}  // namespace orc

// ===========================================================================
// C ABI
using namespace orc;

struct orc_mesh_s {
  Mesh mesh;
};
struct orc_model_s {
  Model model;
};
struct orc_hrom_s {
  Hrom h;
};

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

void* orc_rng_new(uint64_t seed) { return new Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t orc_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double orc_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
double orc_rng_uniform_ab(void* r, double a, double b) { return static_cast<Rng*>(r)->uniform(a, b); }
int orc_rng_uniform_int(void* r, int n) { return static_cast<Rng*>(r)->uniform_int(n); }
double orc_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }

static State unpack_state(const double* s) {
  State st;
  if (s) {
    for (int c = 0; c < 4; ++c) st.ep[c] = s[c];
    st.eq = s[4];
    st.s33 = s[5];
  }
  return st;
}
static void pack_state(const State& st, double* s) {
  for (int c = 0; c < 4; ++c) s[c] = st.ep[c];
  s[4] = st.eq;
  s[5] = st.s33;
}

int orc_update_material(const orc_material_t* mat, const double* state_in6, const double* eps3,
                        double* sigma3, double* C9, double* state_out6, int* plastic) {
  return guarded([&] {
    const Mat m = to_mat(*mat);
    const Result3 r = update_material(m, unpack_state(state_in6), eps3);
    for (int i = 0; i < 3; ++i) sigma3[i] = r.sigma[i];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) C9[3 * i + j] = r.C[i][j];
    if (state_out6) pack_state(r.state, state_out6);
    if (plastic) *plastic = r.plastic ? 1 : 0;
  });
}

int orc_update4(const orc_material_t* mat, const double* state_in6, const double* eps4, double* sigma4,
                double* D16, double* state_out6) {
  return guarded([&] {
    const Mat m = to_mat(*mat);
    const Result4 r = update4(m, unpack_state(state_in6), eps4);
    for (int i = 0; i < 4; ++i) sigma4[i] = r.sigma[i];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) D16[4 * i + j] = r.D[i][j];
    if (state_out6) pack_state(r.state, state_out6);
  });
}

int orc_mesh_build(int geometry, int subdivisions, orc_mesh_t* out) {
  return guarded([&] {
    Geometry geo;
    if (geometry == 0)
      geo = default_cell(subdivisions);
    else
      geo.subdivisions = subdivisions;
    *out = new orc_mesh_s{build_rve_mesh(geo)};
  });
}
void orc_mesh_free(orc_mesh_t m) { delete m; }
int orc_mesh_counts(orc_mesh_t m, int* nn, int* ne, double* area) {
  *nn = m->mesh.n_nodes();
  *ne = m->mesh.n_el();
  *area = m->mesh.area;
  return 0;
}
int orc_mesh_arrays(orc_mesh_t m, double* xy, int* conn, int* mat) {
  for (int i = 0; i < m->mesh.n_nodes(); ++i) {
    xy[2 * i] = m->mesh.nodes[i].x;
    xy[2 * i + 1] = m->mesh.nodes[i].y;
  }
  for (int e = 0; e < m->mesh.n_el(); ++e) {
    for (int a = 0; a < 6; ++a) conn[6 * e + a] = m->mesh.elements[e].nodes[a];
    mat[e] = m->mesh.elements[e].mat;
  }
  return 0;
}
int orc_mesh_ip(orc_mesh_t m, int ip, double* B36, double* w, int* element) {
  return guarded([&] {
    require(ip >= 0 && ip < m->mesh.n_ips(), ErrorCode::config, "ip out of range");
    double B[3][12];
    const int e = ip / 3, g = ip % 3;
    const double detJ = shape_eval(m->mesh, m->mesh.elements[e], kQP[g][0], kQP[g][1], B);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 12; ++c) B36[r * 12 + c] = B[r][c];
    *w = kQW * detJ;
    *element = e;
  });
}

int orc_hf_trajectory(orc_mesh_t m, const orc_material_t* mats, int n_mats, int n_steps, const double* E,
                      const orc_newton_opts_t* opts, double* sigma, double* C, int* iterations,
                      double* u_fluct_inf, double* res_last, double* snapshots) {
  return guarded([&] {
    std::vector<Mat> ms;
    for (int i = 0; i < n_mats; ++i) ms.push_back(to_mat(mats[i]));
    HfProblem p = build_hf(m->mesh, ms);
    const int nf = p.dm.n_free;
    std::vector<State> states(p.mesh.n_ips());
    std::vector<double> u_free(nf, 0.0);
    double E_prev[3] = {0, 0, 0}, E_comm[3] = {0, 0, 0};
    for (int k = 0; k < n_steps; ++k) {
      double done = 0.0, frac = 1.0;
      int bis = 0, its = 0;
      while (done < 1.0 - 1e-12) {
        const double target = std::min(1.0, done + frac);
        double Ev[3], dE[3];
        for (int i = 0; i < 3; ++i) Ev[i] = E_prev[i] + (E[3 * k + i] - E_prev[i]) * target;
        for (int i = 0; i < 3; ++i) dE[i] = Ev[i] - E_comm[i];
        std::vector<double> aff;
        affine_field(p.mesh, dE, aff);
        std::vector<double> u0(nf);
        for (int i = 0; i < p.mesh.n_dofs(); ++i)
          if (p.dm.free_index[i] >= 0) u0[p.dm.free_index[i]] = u_free[p.dm.free_index[i]] + aff[i];
        p.dt_scale = target - done;
        HfSolve r = hf_newton(p, Ev, states, u0, opts->tol, opts->max_iter);
        its += r.iterations;
        if (!r.converged) {
          require(++bis <= opts->max_bisections, ErrorCode::solver, "micro trajectory failed after max bisections");
          frac *= 0.5;
          continue;
        }
        states = r.states;
        for (int i = 0; i < p.mesh.n_dofs(); ++i)
          if (p.dm.free_index[i] >= 0) u_free[p.dm.free_index[i]] = r.u_full[i];
        for (int i = 0; i < 3; ++i) E_comm[i] = Ev[i];
        done = target;
        if (done >= 1.0 - 1e-12) {
          hf_homogenize(p, r, sigma + 3 * k, C + 9 * k);
          if (u_fluct_inf) {
            std::vector<double> aff2;
            affine_field(p.mesh, Ev, aff2);
            double mx = 0.0;
            for (int i = 0; i < p.mesh.n_dofs(); ++i) mx = std::max(mx, std::abs(r.u_full[i] - aff2[i]));
            u_fluct_inf[k] = mx;
          }
          if (snapshots) {  // SnapshotRecorder x_u column, rve.hpp:486-490
            std::vector<double> aff3;
            affine_field(p.mesh, Ev, aff3);
            for (int i = 0; i < p.mesh.n_dofs(); ++i)
              snapshots[(size_t)k * p.mesh.n_dofs() + i] = r.u_full[i] - aff3[i];
          }
          if (res_last) res_last[k] = r.res_hist.back();
        }
      }
      iterations[k] = its;
      for (int i = 0; i < 3; ++i) E_prev[i] = E[3 * k + i];
    }
  });
}

int orc_model_build_on_mesh(orc_mesh_t mesh, int n, int K, uint64_t seed, orc_model_t* out) {
  return guarded([&] { *out = new orc_model_s{build_model(mesh->mesh, n, K, seed)}; });
}
int orc_model_build(int subdivisions, int n, int K, uint64_t seed, orc_model_t* out) {
  return guarded([&] {
    const Mesh mesh = build_rve_mesh(default_cell(subdivisions));
    *out = new orc_model_s{build_model(mesh, n, K, seed)};
  });
}
void orc_model_free(orc_model_t m) { delete m; }
int orc_model_sizes(orc_model_t m, int* n, int* K, int* n_free, double* volume) {
  *n = m->model.n;
  *K = m->model.K;
  *n_free = m->model.n_free;
  *volume = m->model.volume;
  return 0;
}
int orc_model_arrays(orc_model_t m, double* G, double* w, int* ip_id, int* mat_id) {
  const Model& md = m->model;
  if (G) std::memcpy(G, md.G.data(), md.G.size() * sizeof(double));
  if (w) std::memcpy(w, md.w.data(), md.w.size() * sizeof(double));
  if (ip_id) std::memcpy(ip_id, md.ip.data(), md.ip.size() * sizeof(int));
  if (mat_id) std::memcpy(mat_id, md.mat.data(), md.mat.size() * sizeof(int));
  return 0;
}
int orc_model_phi(orc_model_t m, double* phi) {
  std::memcpy(phi, m->model.phi.data(), m->model.phi.size() * sizeof(double));
  return 0;
}

int orc_paths(int kind, uint64_t seed, int64_t p0, int64_t P, int n_incr, double* E) {
  return guarded([&] {
    for (int64_t p = 0; p < P; ++p) make_path(kind, seed, p0 + p, n_incr, E + (size_t)p * n_incr * 3);
  });
}

int orc_hrom_create(int n, int K, const double* G, const double* w, const int* mat_id,
                    const orc_material_t* mats, int n_mats, double volume, orc_hrom_t* out) {
  return guarded([&] {
    require(n >= 1 && K >= 1, ErrorCode::config, "n and K must be positive");
    auto* h = new orc_hrom_s;
    h->h.n = n;
    h->h.K = K;
    h->h.G.assign(G, G + (size_t)K * 3 * n);
    h->h.w.assign(w, w + K);
    h->h.mat.assign(mat_id, mat_id + K);
    for (int i = 0; i < n_mats; ++i) h->h.mats.push_back(to_mat(mats[i]));
    for (int q = 0; q < K; ++q)
      if (mat_id[q] < 0 || mat_id[q] >= n_mats) {
        delete h;
        fail(ErrorCode::config, "cubature material id out of range");
      }
    h->h.volume = volume;
    *out = h;
  });
}
void orc_hrom_free(orc_hrom_t h) { delete h; }

int orc_hrom_run(orc_hrom_t h, int64_t P, int n_incr, const double* E, const orc_newton_opts_t* opts,
                 int n_threads, orc_hrom_out_t* out) {
  return guarded([&] {
    parallel_for(P, n_threads, [&](int64_t p) {
      hrom_point_trajectory(h->h, p, n_incr, E + (size_t)p * n_incr * 3, opts->tol, opts->max_iter,
                            opts->max_bisections, out);
    });
  });
}

int orc_hrom_assemble(orc_hrom_t h, const double* alpha, const double* E, const double* state, double* r,
                      double* Kaa, double* KaE, double* C_EE, double* S_raw, int* plastic_count, double* state_out) {
  return guarded([&] {
    std::vector<State> s0(h->h.K);
    if (state)
      for (int q = 0; q < h->h.K; ++q) s0[q] = unpack_state(state + (size_t)q * 6);
    Assembly A;
    hrom_assemble(h->h, alpha, E, s0, true, A);
    std::memcpy(r, A.r.data(), sizeof(double) * h->h.n);
    std::memcpy(Kaa, A.Kaa.data(), sizeof(double) * h->h.n * h->h.n);
    std::memcpy(KaE, A.KaE.data(), sizeof(double) * h->h.n * 3);
    std::memcpy(C_EE, A.C_EE, sizeof A.C_EE);
    std::memcpy(S_raw, A.S_raw, sizeof A.S_raw);
    if (plastic_count) *plastic_count = A.plastic_count;
    if (state_out)
      for (int q = 0; q < h->h.K; ++q) pack_state(A.states[q], state_out + (size_t)q * 6);
  });
}

// ---- finite strain (config 2; parity unpinned, see update_biot)
struct orc_hrom_fs_s {
  HromFs h;
};

int orc_update_biot(const orc_material_t* mat, const double* state_in6, const double* F4, double* P4, double* A16,
                    double* state_out6, int* plastic) {
  return guarded([&] {
    const Mat m = to_mat(*mat);
    const FsResult r = update_biot(m, unpack_state(state_in6), F4);
    std::memcpy(P4, r.P, sizeof r.P);
    std::memcpy(A16, r.A, sizeof r.A);
    if (state_out6) pack_state(r.state, state_out6);
    if (plastic) *plastic = r.plastic ? 1 : 0;
  });
}

int orc_model_g4(int subdivisions, int n, int K, uint64_t seed, double* G4) {
  return guarded([&] {
    const Mesh mesh = build_rve_mesh(default_cell(subdivisions));
    const Model md = build_model(mesh, n, K, seed);
    const std::vector<double> g = build_g4(mesh, md);
    std::memcpy(G4, g.data(), g.size() * sizeof(double));
  });
}

int orc_paths_fs(uint64_t seed, int64_t p0, int64_t P, int n_incr, double* H) {
  return guarded([&] {
    for (int64_t p = 0; p < P; ++p) make_path_fs(seed, p0 + p, n_incr, H + (size_t)p * n_incr * 4);
  });
}

int orc_hrom_fs_create(int n, int K, const double* G4, const double* w, const int* mat_id, const orc_material_t* mats,
                       int n_mats, double volume, orc_hrom_fs_t* out) {
  return guarded([&] {
    require(n >= 1 && K >= 1, ErrorCode::config, "n and K must be positive");
    auto* h = new orc_hrom_fs_s;
    h->h.n = n;
    h->h.K = K;
    h->h.G.assign(G4, G4 + (size_t)K * 4 * n);
    h->h.w.assign(w, w + K);
    h->h.mat.assign(mat_id, mat_id + K);
    for (int i = 0; i < n_mats; ++i) h->h.mats.push_back(to_mat(mats[i]));
    h->h.volume = volume;
    *out = h;
  });
}
void orc_hrom_fs_free(orc_hrom_fs_t h) { delete h; }

int orc_hrom_fs_run(orc_hrom_fs_t h, int64_t P, int n_incr, const double* H, const orc_newton_opts_t* opts,
                    int n_threads, orc_hrom_out_t* out) {
  return guarded([&] {
    parallel_for(P, n_threads, [&](int64_t p) {
      fs_point_trajectory(h->h, p, n_incr, H + (size_t)p * n_incr * 4, opts->tol, opts->max_iter,
                          opts->max_bisections, out);
    });
  });
}

int orc_hrom_fs_assemble(orc_hrom_fs_t h, const double* alpha, const double* H, const double* state, double* r,
                         double* Kaa, double* KaF, double* KFa, double* CFF, double* P_raw, int* plastic_count) {
  return guarded([&] {
    std::vector<State> s0(h->h.K);
    if (state)
      for (int q = 0; q < h->h.K; ++q) s0[q] = unpack_state(state + (size_t)q * 6);
    AssemblyFs A;
    fs_assemble(h->h, alpha, H, s0, true, A);
    const int n = h->h.n;
    std::memcpy(r, A.r.data(), sizeof(double) * n);
    std::memcpy(Kaa, A.Kaa.data(), sizeof(double) * n * n);
    std::memcpy(KaF, A.KaF.data(), sizeof(double) * n * 4);
    std::memcpy(KFa, A.KFa.data(), sizeof(double) * 4 * n);
    std::memcpy(CFF, A.CFF, sizeof A.CFF);
    std::memcpy(P_raw, A.P_raw, sizeof A.P_raw);
    if (plastic_count) *plastic_count = A.plastic_count;
  });
}

}  // extern "C"
