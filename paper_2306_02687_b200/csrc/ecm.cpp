// Empirical Cubature Method (SPEC.md:333-369 hyper.ecm_select):
// from an orthonormal basis U (m integration points x k integrand modes,
// evaluated per point) select m~ points and strictly positive weights w with
// U_Z^T w = b, b = U^T w_full (the full-rule integrals of every mode), and a
// constant column appended so that sum(w) = |Omega| (volume exactness).
// Greedy selection by largest positive correlation of U[q,:] with the current
// residual (lowest index on ties), least-squares re-fit on the selected set
// after every addition, and removal of points whose weight turns non-positive
// (the original ECM; SPEC DESIGN DECISIONS). Offline, host, deterministic.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"

namespace fe2 {

namespace {

// min || A x - b || for A (k x z, column-major), z <= k, by Householder QR.
// Returns false if A is rank deficient.
bool least_squares(std::vector<double> A, int k, int z, std::vector<double> b, std::vector<double>& x) {
  for (int j = 0; j < z; ++j) {
    double* a = A.data() + static_cast<size_t>(j) * k;
    double nrm = 0.0;
    for (int i = j; i < k; ++i) nrm += a[i] * a[i];
    nrm = std::sqrt(nrm);
    if (!(nrm > 0.0)) return false;
    const double alpha = a[j] > 0.0 ? -nrm : nrm;
    std::vector<double> v(a + j, a + k);
    v[0] -= alpha;
    double vv = 0.0;
    for (double t : v) vv += t * t;
    if (vv > 0.0) {
      const double beta = 2.0 / vv;
      for (int c = j; c < z; ++c) {
        double* ac = A.data() + static_cast<size_t>(c) * k;
        double s = 0.0;
        for (int i = j; i < k; ++i) s += v[i - j] * ac[i];
        s *= beta;
        for (int i = j; i < k; ++i) ac[i] -= s * v[i - j];
      }
      double s = 0.0;
      for (int i = j; i < k; ++i) s += v[i - j] * b[i];
      s *= beta;
      for (int i = j; i < k; ++i) b[i] -= s * v[i - j];
    }
    if (std::abs(A[static_cast<size_t>(j) * k + j]) <= 1e-13 * nrm) return false;
  }
  x.assign(z, 0.0);
  for (int j = z - 1; j >= 0; --j) {
    double s = b[j];
    for (int c = j + 1; c < z; ++c) s -= A[static_cast<size_t>(c) * k + j] * x[c];
    x[j] = s / A[static_cast<size_t>(j) * k + j];
  }
  return true;
}

}  // namespace

}  // namespace fe2

using namespace fe2;

extern "C" {

int fe2_ecm_select(const double* U, const double* w_full, int m, int k, int m_target, double tol, int* ids,
                   double* weights, int* m_out, double* rel_residual) {
  return guard([&] {
    check(U && w_full && ids && weights && m_out && m >= 1 && k >= 0 && m_target >= 1 && tol >= 0.0,
          Code::config, "bad ECM arguments");
    // basis with the constant column (volume exactness), scaled like the modes
    const int ke = k + 1;
    std::vector<double> Ue(static_cast<size_t>(m) * ke);
    double cscale = 0.0;
    for (int q = 0; q < m; ++q)
      for (int j = 0; j < k; ++j) cscale = std::max(cscale, std::abs(U[static_cast<size_t>(q) * k + j]));
    if (!(cscale > 0.0)) cscale = 1.0 / std::sqrt(static_cast<double>(m));
    for (int q = 0; q < m; ++q) {
      for (int j = 0; j < k; ++j) Ue[static_cast<size_t>(q) * ke + j] = U[static_cast<size_t>(q) * k + j];
      Ue[static_cast<size_t>(q) * ke + k] = cscale;
    }
    std::vector<double> b(ke, 0.0), rn(m, 0.0);
    for (int q = 0; q < m; ++q) {
      check(w_full[q] > 0.0, Code::config, "full-rule weights must be positive");
      double s = 0.0;
      for (int j = 0; j < ke; ++j) {
        const double u = Ue[static_cast<size_t>(q) * ke + j];
        b[j] += w_full[q] * u;
        s += u * u;
      }
      rn[q] = std::sqrt(s);
    }
    double bn = 0.0;
    for (double t : b) bn += t * t;
    bn = std::sqrt(bn);
    check(bn > 0.0, Code::numeric, "all integrals vanish");
    std::vector<int> Z;
    std::vector<double> w, r = b;
    std::vector<char> in(m, 0);
    auto residual = [&]() {
      double s = 0.0;
      for (double t : r) s += t * t;
      return std::sqrt(s) / bn;
    };
    auto refit = [&]() -> bool {
      while (!Z.empty()) {
        const int z = static_cast<int>(Z.size());
        std::vector<double> A(static_cast<size_t>(ke) * z);
        for (int c = 0; c < z; ++c)
          for (int j = 0; j < ke; ++j) A[static_cast<size_t>(c) * ke + j] = Ue[static_cast<size_t>(Z[c]) * ke + j];
        if (!least_squares(A, ke, z, b, w)) return false;
        // drop non-positive weights and re-fit (ECM)
        std::vector<int> keep;
        for (int c = 0; c < z; ++c)
          if (w[c] > 0.0) keep.push_back(Z[c]);
          else in[Z[c]] = 0;
        if (static_cast<int>(keep.size()) == z) break;
        Z.swap(keep);
      }
      r = b;
      for (size_t c = 0; c < Z.size(); ++c)
        for (int j = 0; j < ke; ++j) r[j] -= w[c] * Ue[static_cast<size_t>(Z[c]) * ke + j];
      return true;
    };
    int guard_iters = 0;
    while (static_cast<int>(Z.size()) < std::min(m_target, ke) && residual() > tol && guard_iters++ < 4 * m + 16) {
      int best = -1;
      double bc = 0.0;
      for (int q = 0; q < m; ++q) {
        if (in[q] || !(rn[q] > 0.0)) continue;
        double c = 0.0;
        for (int j = 0; j < ke; ++j) c += Ue[static_cast<size_t>(q) * ke + j] * r[j];
        c /= rn[q];
        if (c > bc) {
          bc = c;
          best = q;
        }
      }
      if (best < 0) break;  // no point correlates positively with the residual
      Z.push_back(best);
      in[best] = 1;
      if (!refit()) {  // dependent on the selected set: drop it again
        in[best] = 0;
        Z.pop_back();
        rn[best] = 0.0;  // never reconsider
        refit();
      }
    }
    check(!Z.empty(), Code::numeric, "ECM selected no point");
    std::vector<int> order(Z.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int c) { return Z[a] < Z[c]; });
    for (size_t i = 0; i < order.size(); ++i) {
      ids[i] = Z[order[i]];
      weights[i] = w[order[i]];
    }
    *m_out = static_cast<int>(Z.size());
    if (rel_residual) *rel_residual = residual();
  });
}

}  // extern "C"
