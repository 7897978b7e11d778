// Macro FE driver of the two-scale beam (the caller of
// the hot path): SPEC.md:455-518 fe2.macro_step / solve_program in the nested
// variant — every macro Newton iteration runs fully converged micro solves
// (one engine increment for all macro Gauss points) and assembles the macro
// tangent from their condensed C_macro; the micro history is committed only
// when the macro step converges (engine snapshot / restore). scheme = 1 runs
// the monolithic variant instead (SPEC.md:474-481 and its DESIGN DECISION:
// single-iteration-coupled Newton, micro condensed every iteration): each
// macro iteration advances every micro problem by ONE reduced Newton iteration
// (fe2_hrom_mono_iterate) and assembles the macro residual / tangent from the
// condensed stress and tangent; a step is accepted when the macro residual AND
// every micro residual are below tolerance (fe2_hrom_mono_commit).
//
// Macro problem (SPEC "desk" defaults): plane strain L x H strip of
// structured Tri6 pairs (build_beam_mesh, mesh.hpp:133-169), left edge
// clamped, a vertical displacement U prescribed on the tip edge (x = L),
// reaction R = sum of the tip nodes' vertical internal forces. Load program:
// n_load steps to u_max, then unloading in the same steps until R changes
// sign; the residual displacement U_res is the linear zero crossing
// (solve_program). Host code only; the micro solves run on the device.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"

namespace fe2 {

namespace {

struct Beam {
  std::vector<double> x, y;
  std::vector<std::array<int, 6>> tri;
  std::vector<int> left, tip;
  // per macro Gauss point (3 per element): strain operator B (3 x 12, row-major), weight
  std::vector<std::array<double, 36>> B;
  std::vector<double> w;
  std::vector<int> elem;
};

constexpr double kGp[3][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0}};

// Tri6 strain operator at (xi, eta) (shape_eval, mesh.hpp:85-115); returns detJ.
double tri6_B(const Beam& m, const std::array<int, 6>& t, double xi, double eta, double* Bop) {
  const double l1 = 1.0 - xi - eta, l2 = xi, l3 = eta;
  const double g[6][2] = {{-(4.0 * l1 - 1.0), -(4.0 * l1 - 1.0)},
                          {4.0 * l2 - 1.0, 0.0},
                          {0.0, 4.0 * l3 - 1.0},
                          {4.0 * (l1 - l2), -4.0 * l2},
                          {4.0 * l3, 4.0 * l2},
                          {-4.0 * l3, 4.0 * (l1 - l3)}};
  double j00 = 0.0, j01 = 0.0, j10 = 0.0, j11 = 0.0;
  for (int a = 0; a < 6; ++a) {
    j00 += g[a][0] * m.x[t[a]];
    j01 += g[a][0] * m.y[t[a]];
    j10 += g[a][1] * m.x[t[a]];
    j11 += g[a][1] * m.y[t[a]];
  }
  const double det = j00 * j11 - j01 * j10;
  check(det > 0.0, Code::mesh, "inverted macro element (detJ <= 0)");
  const double k00 = j11 / det, k01 = -j01 / det, k10 = -j10 / det, k11 = j00 / det;
  std::memset(Bop, 0, sizeof(double) * 36);
  for (int a = 0; a < 6; ++a) {
    const double dx = k00 * g[a][0] + k01 * g[a][1];
    const double dy = k10 * g[a][0] + k11 * g[a][1];
    Bop[0 * 12 + 2 * a] = dx;
    Bop[1 * 12 + 2 * a + 1] = dy;
    Bop[2 * 12 + 2 * a] = dy;
    Bop[2 * 12 + 2 * a + 1] = dx;
  }
  return det;
}

// build_beam_mesh (mesh.hpp:133-169): nodes on a (2nx+1) x (2ny+1) grid,
// per cell the lower-right (A,B,C) and upper-left (A,C,D) Tri6.
Beam build_beam(double L, double H, int nx, int ny) {
  check(L > 0.0 && H > 0.0, Code::config, "beam dimensions must be positive");
  check(nx >= 1 && ny >= 1, Code::config, "beam subdivisions must be >= 1");
  Beam m;
  const int gx = 2 * nx + 1, gy = 2 * ny + 1;
  auto gid = [gx](int i, int j) { return j * gx + i; };
  for (int j = 0; j < gy; ++j)
    for (int i = 0; i < gx; ++i) {
      m.x.push_back(L * i / (gx - 1.0));
      m.y.push_back(H * j / (gy - 1.0));
    }
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int i0 = 2 * i, j0 = 2 * j;
      m.tri.push_back({gid(i0, j0), gid(i0 + 2, j0), gid(i0 + 2, j0 + 2), gid(i0 + 1, j0), gid(i0 + 2, j0 + 1),
                       gid(i0 + 1, j0 + 1)});
      m.tri.push_back({gid(i0, j0), gid(i0 + 2, j0 + 2), gid(i0, j0 + 2), gid(i0 + 1, j0 + 1), gid(i0 + 1, j0 + 2),
                       gid(i0, j0 + 1)});
    }
  for (int j = 0; j < gy; ++j) {
    m.left.push_back(gid(0, j));
    m.tip.push_back(gid(gx - 1, j));
  }
  for (size_t e = 0; e < m.tri.size(); ++e)
    for (int g = 0; g < 3; ++g) {
      std::array<double, 36> B{};
      const double det = tri6_B(m, m.tri[e], kGp[g][0], kGp[g][1], B.data());
      m.B.push_back(B);
      m.w.push_back(det / 6.0);
      m.elem.push_back(static_cast<int>(e));
    }
  return m;
}

// dense Cholesky solve of the SPD free-DOF block (macro tangent from the
// symmetric condensed C_macro); false if not positive definite
bool chol_solve(std::vector<double>& A, int n, std::vector<double>& b) {
  for (int j = 0; j < n; ++j) {
    double d = A[static_cast<size_t>(j) * n + j];
    for (int k = 0; k < j; ++k) d -= A[static_cast<size_t>(j) * n + k] * A[static_cast<size_t>(j) * n + k];
    if (!(d > 0.0)) return false;
    const double l = std::sqrt(d);
    A[static_cast<size_t>(j) * n + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double s = A[static_cast<size_t>(i) * n + j];
      for (int k = 0; k < j; ++k) s -= A[static_cast<size_t>(i) * n + k] * A[static_cast<size_t>(j) * n + k];
      A[static_cast<size_t>(i) * n + j] = s / l;
    }
  }
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= A[static_cast<size_t>(i) * n + k] * b[k];
    b[i] = s / A[static_cast<size_t>(i) * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= A[static_cast<size_t>(k) * n + i] * b[k];
    b[i] = s / A[static_cast<size_t>(i) * n + i];
  }
  return true;
}

// dense LU solve with partial pivoting (finite-strain macro tangent: A = dP/dF is
// not symmetric); false if singular
bool lu_solve(std::vector<double>& A, int n, std::vector<double>& b) {
  for (int j = 0; j < n; ++j) {
    int p = j;
    double best = std::abs(A[static_cast<size_t>(j) * n + j]);
    for (int i = j + 1; i < n; ++i)
      if (std::abs(A[static_cast<size_t>(i) * n + j]) > best) {
        best = std::abs(A[static_cast<size_t>(i) * n + j]);
        p = i;
      }
    if (!(best > 0.0)) return false;
    if (p != j) {
      for (int k = 0; k < n; ++k) std::swap(A[static_cast<size_t>(j) * n + k], A[static_cast<size_t>(p) * n + k]);
      std::swap(b[j], b[p]);
    }
    const double inv = 1.0 / A[static_cast<size_t>(j) * n + j];
    for (int i = j + 1; i < n; ++i) {
      const double l = A[static_cast<size_t>(i) * n + j] * inv;
      if (l == 0.0) continue;
      for (int k = j + 1; k < n; ++k) A[static_cast<size_t>(i) * n + k] -= l * A[static_cast<size_t>(j) * n + k];
      b[i] -= l * b[j];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= A[static_cast<size_t>(i) * n + k] * b[k];
    b[i] = s / A[static_cast<size_t>(i) * n + i];
  }
  return true;
}

void engine_check(int rc) {
  if (rc != 0) throw Failure(static_cast<Code>(rc - 1), std::string("engine: ") + fe2_last_error());
}

}  // namespace

}  // namespace fe2

using namespace fe2;

extern "C" {

int fe2_macro_points(const fe2_macro_config_t* cfg, int64_t* n_points) {
  return guard([&] {
    check(cfg && n_points, Code::config, "bad arguments");
    const Beam m = build_beam(cfg->length, cfg->height, cfg->nx, cfg->ny);
    *n_points = static_cast<int64_t>(m.w.size());
  });
}

int fe2_macro_gauss(const fe2_macro_config_t* cfg, double* B, double* w, int* elem) {
  return guard([&] {
    check(cfg != nullptr, Code::config, "bad arguments");
    const Beam m = build_beam(cfg->length, cfg->height, cfg->nx, cfg->ny);
    for (size_t g = 0; g < m.w.size(); ++g) {
      if (B) std::memcpy(B + g * 36, m.B[g].data(), 36 * sizeof(double));
      if (w) w[g] = m.w[g];
      if (elem) elem[g] = m.elem[g];
    }
  });
}

}  // extern "C"

namespace {

// The load program on either micro backend: a hyper-ROM engine (engine) or
// full-field HF RVEs (hf), nested or monolithic (cfg->scheme).
void macro_program(const fe2_macro_config_t* cfg, fe2_hrom_t engine, fe2_hf_t hf, double* rows, int max_rows,
                   int* n_rows, double* u_residual) {
  {
    check(cfg && (engine || hf) && rows && n_rows && max_rows > 0, Code::config, "bad arguments");
    check(cfg->n_load >= 1 && cfg->max_iter >= 1 && cfg->tol > 0.0, Code::config, "invalid macro options");
    int kin = 0;
    if (engine) engine_check(fe2_hrom_kinematics(engine, &kin));
    const Beam m = build_beam(cfg->length, cfg->height, cfg->nx, cfg->ny);
    const int P = static_cast<int>(m.w.size());
    // per-Gauss-point operator: small strain (E11, E22, g12) = B u; finite strain
    // (total Lagrangian) H = F - I = (dux/dX, dux/dY, duy/dX, duy/dY) = Bg u
    const int nr = kin ? 4 : 3;
    std::vector<double> Op(static_cast<size_t>(P) * nr * 12, 0.0);
    for (int g = 0; g < P; ++g) {
      double* o = Op.data() + static_cast<size_t>(g) * nr * 12;
      const double* B = m.B[g].data();
      if (!kin) {
        std::memcpy(o, B, 36 * sizeof(double));
      } else {
        for (int a = 0; a < 6; ++a) {
          o[0 * 12 + 2 * a] = B[0 * 12 + 2 * a];          // dN/dx
          o[1 * 12 + 2 * a] = B[2 * 12 + 2 * a];          // dN/dy
          o[2 * 12 + 2 * a + 1] = B[2 * 12 + 2 * a + 1];  // dN/dx
          o[3 * 12 + 2 * a + 1] = B[1 * 12 + 2 * a + 1];  // dN/dy
        }
      }
    }
    int64_t held = 0;
    if (engine) {
      fe2_hrom_stats_t est{};
      engine_check(fe2_hrom_stats(engine, &est));
      held = est.points;
    } else {
      engine_check(fe2_hf_points(hf, &held));
    }
    check(held == P, Code::config, "engine must hold one point per macro Gauss point (fe2_macro_points)");
    const int nd = 2 * static_cast<int>(m.x.size());
    // DOF roles: fixed (left: x, y), prescribed (tip: y), free (others)
    std::vector<int> role(nd, 0);  // 0 free, 1 fixed at 0, 2 prescribed U
    for (int nd_ : m.left) role[2 * nd_] = role[2 * nd_ + 1] = 1;
    for (int nd_ : m.tip) role[2 * nd_ + 1] = 2;
    std::vector<int> fidx(nd, -1);
    int nf = 0;
    for (int d = 0; d < nd; ++d)
      if (role[d] == 0) fidx[d] = nf++;

    std::vector<double> u(nd, 0.0), E(nr * P), sig(nr * P), C(nr * nr * P), res(P), fint(nd), Kff, rhs;
    std::vector<int> it(P), pc(P), st(P);
    const fe2_newton_opts_t mopt = cfg->micro;
    auto dofs = [&](int e, int d) { return 2 * m.tri[e][d / 2] + d % 2; };

    // one trial micro solve at displacement u from the committed state; false if any point failed
    long long micro_total = 0;
    double fscale = 0.0;  // largest |f_int| of an accepted step: the residual's absolute floor near R = 0
    const bool mono = cfg->scheme == 1;
    check(cfg->scheme == 0 || cfg->scheme == 1, Code::config, "scheme must be 0 (nested) or 1 (monolithic)");
    check(!mono || kin == 0, Code::config, "the monolithic scheme runs on small-strain handles");
    bool micro_ok = true;  // monolithic: every point's micro residual below micro.tol
    auto micro_solve = [&]() -> bool {
      for (int g = 0; g < P; ++g) {
        const int e = m.elem[g];
        const double* o = Op.data() + static_cast<size_t>(g) * nr * 12;
        for (int i = 0; i < nr; ++i) {
          double s = 0.0;
          for (int d = 0; d < 12; ++d) s += o[i * 12 + d] * u[dofs(e, d)];
          E[nr * g + i] = s;
        }
      }
      if (mono) {  // one micro iteration per point, condensed stress and tangent
        engine_check(engine ? fe2_hrom_mono_iterate(engine, E.data(), sig.data(), C.data(), res.data(), pc.data(),
                                                    st.data())
                            : fe2_hf_mono_iterate(hf, E.data(), sig.data(), C.data(), res.data(), st.data()));
        micro_ok = true;
        for (int g = 0; g < P; ++g) {
          if (st[g] != 0) return false;
          micro_total += 1;
          micro_ok = micro_ok && res[g] <= mopt.tol;
        }
      } else if (hf) {
        engine_check(fe2_hf_restore(hf));
        engine_check(fe2_hf_solve_increment(hf, E.data(), &mopt, sig.data(), C.data(), it.data(), st.data()));
        for (int g = 0; g < P; ++g) {
          if (st[g] != 0) return false;
          micro_total += it[g];
        }
      } else {
        engine_check(fe2_hrom_restore(engine));
        engine_check(fe2_hrom_solve_increment(engine, E.data(), &mopt, sig.data(), C.data(), it.data(), pc.data(),
                                              res.data(), st.data()));
        for (int g = 0; g < P; ++g) {
          if (st[g] != 0) return false;
          micro_total += it[g];
        }
      }
      std::fill(fint.begin(), fint.end(), 0.0);
      for (int g = 0; g < P; ++g) {
        const int e = m.elem[g];
        const double* o = Op.data() + static_cast<size_t>(g) * nr * 12;
        for (int d = 0; d < 12; ++d) {
          double s = 0.0;
          for (int i = 0; i < nr; ++i) s += o[i * 12 + d] * sig[nr * g + i];
          fint[dofs(e, d)] += m.w[g] * s;
        }
      }
      return true;
    };
    // K_ff = Σ_g w B_gᵀ C_g B_g over the free DOFs
    auto assemble_K = [&](const std::vector<double>& Cc) {
        Kff.assign(static_cast<size_t>(nf) * nf, 0.0);
        for (int g = 0; g < P; ++g) {
          const int e = m.elem[g];
          const double* o = Op.data() + static_cast<size_t>(g) * nr * 12;
          const double* Cg = Cc.data() + static_cast<size_t>(g) * nr * nr;
          double CB[4][12];
          for (int i = 0; i < nr; ++i)
            for (int d = 0; d < 12; ++d) {
              double s = 0.0;
              for (int j = 0; j < nr; ++j) s += Cg[i * nr + j] * o[j * 12 + d];
              CB[i][d] = s;
            }
          for (int a = 0; a < 12; ++a) {
            const int fa = fidx[dofs(e, a)];
            if (fa < 0) continue;
            for (int b = 0; b < 12; ++b) {
              const int fb = fidx[dofs(e, b)];
              if (fb < 0) continue;
              double s = 0.0;
              for (int i = 0; i < nr; ++i) s += o[i * 12 + a] * CB[i][b];
              Kff[static_cast<size_t>(fa) * nf + fb] += m.w[g] * s;
            }
          }
        }
    };
    auto solve_K = [&]() {
      if (kin)
        check(lu_solve(Kff, nf, rhs), Code::solver, "finite-strain macro tangent is singular");
      else
        check(chol_solve(Kff, nf, rhs), Code::solver, "macro tangent is not positive definite");
    };
    // Step predictor: the prescribed tip increment ΔU spread over the free DOFs
    // with the tangent of the last accepted state, Δu_f = -K_ff⁻¹ K_fp ΔU
    // (keeps the first iterate of a plastic step near the solution).
    std::vector<double> C_acc;
    auto predict = [&](double U) {
      const double dU = U - u[2 * m.tip[0] + 1];
      if (dU == 0.0 || C_acc.empty()) return;
      std::vector<double> du(nd, 0.0), fp(nd, 0.0);
      for (int nd_ : m.tip) du[2 * nd_ + 1] = dU;
      for (int g = 0; g < P; ++g) {
        const int e = m.elem[g];
        const double* o = Op.data() + static_cast<size_t>(g) * nr * 12;
        const double* Cg = C_acc.data() + static_cast<size_t>(g) * nr * nr;
        double eg[4] = {0, 0, 0, 0}, sg[4] = {0, 0, 0, 0};
        for (int i = 0; i < nr; ++i)
          for (int d = 0; d < 12; ++d) eg[i] += o[i * 12 + d] * du[dofs(e, d)];
        for (int i = 0; i < nr; ++i)
          for (int j = 0; j < nr; ++j) sg[i] += Cg[i * nr + j] * eg[j];
        for (int d = 0; d < 12; ++d) {
          double t = 0.0;
          for (int i = 0; i < nr; ++i) t += o[i * 12 + d] * sg[i];
          fp[dofs(e, d)] += m.w[g] * t;
        }
      }
      assemble_K(C_acc);
      rhs.assign(nf, 0.0);
      for (int d = 0; d < nd; ++d)
        if (fidx[d] >= 0) rhs[fidx[d]] = -fp[d];
      solve_K();
      for (int d = 0; d < nd; ++d)
        if (fidx[d] >= 0) u[d] += rhs[fidx[d]];
    };
    // macro Newton for a prescribed tip displacement; returns iterations or -1
    auto macro_step = [&](double U) -> int {
      predict(U);
      for (int nd_ : m.tip) u[2 * nd_ + 1] = U;
      if (mono) engine_check(engine ? fe2_hrom_mono_begin(engine) : fe2_hf_mono_begin(hf));
      for (int k = 0; k <= cfg->max_iter; ++k) {
        if (!micro_solve()) return -1;
        double rn = 0.0, fn = 0.0;
        for (int d = 0; d < nd; ++d) {
          fn += fint[d] * fint[d];
          if (role[d] == 0) rn += fint[d] * fint[d];
        }
        rn = std::sqrt(rn);
        fn = std::sqrt(fn);
        if (rn <= cfg->tol * std::max(std::max(fn, fscale), 1e-30) && micro_ok) return k;
        if (k == cfg->max_iter) return -1;
        assemble_K(C);
        rhs.assign(nf, 0.0);
        for (int d = 0; d < nd; ++d)
          if (fidx[d] >= 0) rhs[fidx[d]] = -fint[d];
        solve_K();
        for (int d = 0; d < nd; ++d)
          if (fidx[d] >= 0) u[d] += rhs[fidx[d]];
      }
      return -1;
    };

    const auto t0 = std::chrono::steady_clock::now();
    if (engine) {
      engine_check(fe2_hrom_reset_points(engine));
      engine_check(fe2_hrom_snapshot(engine));  // committed: virgin state
    } else {
      engine_check(fe2_hf_alloc_points(hf, P));
      engine_check(fe2_hf_snapshot(hf));
    }
    // tangent of the virgin state (u = 0) for the first step's predictor
    if (mono) engine_check(engine ? fe2_hrom_mono_begin(engine) : fe2_hf_mono_begin(hf));
    check(micro_solve(), Code::solver, "micro solve at the virgin state failed");
    C_acc = C;
    micro_total = 0;
    int nrow = 0;
    double U_done = 0.0;
    std::vector<double> u_done = u;
    auto reaction = [&]() {
      double R = 0.0;
      for (int nd_ : m.tip) R += fint[2 * nd_ + 1];
      return R;
    };
    // advance the committed state to displacement U_target by (bisected) macro steps
    auto advance = [&](double U_target) {
      double frac = 1.0;
      int bis = 0;
      const double U0 = U_done;
      double done = 0.0;
      int iters_sum = 0;
      while (done < 1.0 - 1e-12) {
        const double target = std::min(1.0, done + frac);
        const double U = U0 + (U_target - U0) * target;
        const int k = macro_step(U);
        if (k < 0) {
          u = u_done;  // back to the last converged displacement field
          check(++bis <= cfg->max_bisections, Code::solver, "macro step did not converge after bisection");
          frac *= 0.5;
          continue;
        }
        iters_sum += k;
        // accept: the micro states are committed
        engine_check(mono ? (engine ? fe2_hrom_mono_commit(engine) : fe2_hf_mono_commit(hf))
                          : (hf ? fe2_hf_snapshot(hf) : fe2_hrom_snapshot(engine)));
        {
          double fn = 0.0;
          for (int d = 0; d < nd; ++d) fn += fint[d] * fint[d];
          fscale = std::max(fscale, std::sqrt(fn));
        }
        u_done = u;
        U_done = U;
        C_acc = C;
        done = target;
      }
      check(nrow < max_rows, Code::config, "curve buffer too small");
      double* r = rows + 5 * static_cast<size_t>(nrow++);
      r[0] = U_done;
      r[1] = reaction();
      r[2] = iters_sum;
      r[3] = static_cast<double>(micro_total);
      r[4] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    const double dU = cfg->u_max / cfg->n_load;
    for (int k = 1; k <= cfg->n_load; ++k) advance(dU * k);
    // unload in the same steps until the reaction changes sign
    double ures = std::nan("");
    for (int k = 0; k < cfg->max_unload; ++k) {
      const double R_prev = rows[5 * (nrow - 1) + 1], U_prev = rows[5 * (nrow - 1)];
      advance(U_done - dU);
      const double R = rows[5 * (nrow - 1) + 1], U = rows[5 * (nrow - 1)];
      if ((R_prev > 0.0) != (R > 0.0)) {
        ures = U_prev + (U - U_prev) * (R_prev / (R_prev - R));
        break;
      }
    }
    *n_rows = nrow;
    if (u_residual) *u_residual = ures;
  }
}

}  // namespace

extern "C" {

int fe2_macro_run(const fe2_macro_config_t* cfg, fe2_hrom_t engine, double* rows, int max_rows, int* n_rows,
                  double* u_residual) {
  return guard([&] {
    check(engine != nullptr, Code::config, "null engine");
    macro_program(cfg, engine, nullptr, rows, max_rows, n_rows, u_residual);
  });
}

// Batched mixed control (rve.hpp:496-571 mixed_control_step, one step for every point of
// the engine): prescribed strain components where control[p*3 + j] != 0, the others
// driven so that the conjugate macro stresses hit sigma_target, by an outer Newton with
// the condensed tangent — each outer iteration re-solves every still-active point from
// its committed state (fe2_hrom_restore + one increment), J = C[u][u] with complete
// pivoting (Eigen fullPivLu), converged when |Σ_u - target_u| <= tol (max(1e-12,
// |target|) + 1e-3). E[P*3] in: the committed macro strains (start of the unknown
// components), out: the converged ones; sigma / C / outer_iters / status per point.
int fe2_hrom_mixed_step(fe2_hrom_t h, const int* control, const double* E_prescribed, const double* sigma_target,
                        double tol, int max_iter, const fe2_newton_opts_t* micro, double* E, double* sigma,
                        double* C, int* outer_iters, int* status) {
  return guard([&] {
    check(h && control && E_prescribed && sigma_target && micro && E, Code::config, "bad arguments");
    check(tol > 0.0 && max_iter >= 0, Code::config, "invalid mixed-control options");
    int kin = 0;
    engine_check(fe2_hrom_kinematics(h, &kin));
    check(kin == 0, Code::config, "mixed control runs on small-strain handles");
    fe2_hrom_stats_t st{};
    engine_check(fe2_hrom_stats(h, &st));
    const int64_t P = st.points;
    check(P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    std::vector<double> Ew(E, E + 3 * P), sg(3 * P), Cm(9 * P), res(P);
    std::vector<int> it(P), pc(P), stt(P), active(P, 1), iters(P, 0), code(P, 0);
    for (int64_t p = 0; p < P; ++p)
      for (int j = 0; j < 3; ++j)
        if (control[3 * p + j]) Ew[3 * p + j] = E_prescribed[3 * p + j];
    engine_check(fe2_hrom_snapshot(h));  // the committed state every outer iteration starts from
    for (int k = 0; k <= max_iter; ++k) {
      engine_check(fe2_hrom_restore(h));
      engine_check(fe2_hrom_solve_increment(h, Ew.data(), micro, sg.data(), Cm.data(), it.data(), pc.data(),
                                            res.data(), stt.data()));
      int n_active = 0;
      for (int64_t p = 0; p < P; ++p) {
        if (!active[p]) continue;
        iters[p] = k;
        if (stt[p] != 0) {  // the micro solve failed (mixed_control_step throws, rve.hpp:547)
          code[p] = stt[p];
          active[p] = 0;
          continue;
        }
        int u[3], nu = 0;
        for (int j = 0; j < 3; ++j)
          if (!control[3 * p + j]) u[nu++] = j;
        if (nu == 0) {
          active[p] = 0;
          continue;
        }
        const double* tg = sigma_target + 3 * p;
        const double scale = std::max(1e-12, std::sqrt(tg[0] * tg[0] + tg[1] * tg[1] + tg[2] * tg[2])) + 1e-3;
        double r[3], rn = 0.0;
        for (int a = 0; a < nu; ++a) {
          r[a] = sg[3 * p + u[a]] - tg[u[a]];
          rn += r[a] * r[a];
        }
        if (std::sqrt(rn) <= tol * scale) {
          active[p] = 0;
          continue;
        }
        if (k == max_iter) {  // "mixed control did not converge" (rve.hpp:559)
          code[p] = 1 + static_cast<int>(Code::solver);
          active[p] = 0;
          continue;
        }
        // J dE = -r with complete pivoting
        double J[3][3], b[3];
        int cp[3] = {0, 1, 2};
        for (int a = 0; a < nu; ++a) {
          b[a] = -r[a];
          for (int c = 0; c < nu; ++c) J[a][c] = Cm[9 * p + 3 * u[a] + u[c]];
        }
        bool sing = false;
        for (int c = 0; c < nu && !sing; ++c) {
          int pr = c, pcn = c;
          double best = -1.0;
          for (int i = c; i < nu; ++i)
            for (int jj = c; jj < nu; ++jj)
              if (std::abs(J[i][jj]) > best) {
                best = std::abs(J[i][jj]);
                pr = i;
                pcn = jj;
              }
          if (!(best > 0.0)) {
            sing = true;
            break;
          }
          for (int jj = 0; jj < nu; ++jj) std::swap(J[c][jj], J[pr][jj]);
          std::swap(b[c], b[pr]);
          for (int i = 0; i < nu; ++i) std::swap(J[i][c], J[i][pcn]);
          std::swap(cp[c], cp[pcn]);
          for (int i = c + 1; i < nu; ++i) {
            const double l = J[i][c] / J[c][c];
            for (int jj = c; jj < nu; ++jj) J[i][jj] -= l * J[c][jj];
            b[i] -= l * b[c];
          }
        }
        if (sing) {
          code[p] = 1 + static_cast<int>(Code::solver);
          active[p] = 0;
          continue;
        }
        double x[3];
        for (int i = nu - 1; i >= 0; --i) {
          double s = b[i];
          for (int jj = i + 1; jj < nu; ++jj) s -= J[i][jj] * x[jj];
          x[i] = s / J[i][i];
        }
        for (int a = 0; a < nu; ++a) Ew[3 * p + u[cp[a]]] += x[a];
        ++n_active;
      }
      if (n_active == 0) break;
    }
    std::memcpy(E, Ew.data(), sizeof(double) * 3 * P);
    if (sigma) std::memcpy(sigma, sg.data(), sizeof(double) * 3 * P);
    if (C) std::memcpy(C, Cm.data(), sizeof(double) * 9 * P);
    if (outer_iters) std::memcpy(outer_iters, iters.data(), sizeof(int) * P);
    if (status) std::memcpy(status, code.data(), sizeof(int) * P);
  });
}

int fe2_macro_run_hf(const fe2_macro_config_t* cfg, fe2_hf_t hf, double* rows, int max_rows, int* n_rows,
                     double* u_residual) {
  return guard([&] {
    check(hf != nullptr, Code::config, "null HF handle");
    macro_program(cfg, nullptr, hf, rows, max_rows, n_rows, u_residual);
  });
}

}  // extern "C"
