// High-fidelity RVE solve on the device and the POD basis built from its
// snapshots (SURVEY §8(f) rank 2 — the offline stage that replaces the seeded
// Φ with physical modes).
//
// Reference behaviour followed (paths relative to
// /root/reference/proj/include/fe2rom/ unless noted):
//   assemble_micro                      rve.hpp:220-262
//   micro_newton (8-halving Armijo LS)   rve.hpp:285-346
//   homogenize (3 sensitivity solves)    rve.hpp:350-392
//   run_trajectory + SnapshotRecorder    rve.hpp:397-494 (x_u = u - E.x per step)
//   build_elastic_modes, pod
//
// Device layout: the material update, strains and element stiffness run in
// k_hf_element (one CTA per Tri6 element, 144 threads = its 12x12 entries);
// k_hf_gather sums the element vectors/matrices into the residual and the
// dense free stiffness with ONE thread per DOF walking its element incidences
// in ascending element order — the reference's assembly order, no atomics,
// bit-reproducible. The dense SPD factorisation/solves and the SVD are
// cuSOLVER (dlopen'ed at first use so the hot-path library does not pull in
// cuSOLVER/cuBLAS at load). Host code keeps the Newton control flow, norms
// and the homogenisation sums (a few thousand integration points).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"
#include "host_util.cuh"
#include "material.cuh"
#include "rve.hpp"

namespace fe2 {

namespace {

// ---------------------------------------------------------------------------
// cuSOLVER, resolved at first use.
struct Cusolver {
  decltype(&cusolverDnCreate) create = nullptr;
  decltype(&cusolverDnDestroy) destroy = nullptr;
  decltype(&cusolverDnSetStream) set_stream = nullptr;
  decltype(&cusolverDnDpotrf_bufferSize) potrf_ws = nullptr;
  decltype(&cusolverDnDpotrf) potrf = nullptr;
  decltype(&cusolverDnDpotrs) potrs = nullptr;
  decltype(&cusolverDnDgesvd_bufferSize) gesvd_ws = nullptr;
  decltype(&cusolverDnDgesvd) gesvd = nullptr;
  std::string err;

  static const Cusolver& get() {
    static const Cusolver s = load();
    check(s.err.empty(), Code::solver, s.err);
    return s;
  }

 private:
  static Cusolver load() {
    Cusolver s;
    void* lib = nullptr;
    for (const char* name : {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11", "libcusolver.so"})
      if ((lib = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!lib) {
      s.err = "cannot load cuSOLVER (libcusolver.so.11)";
      return s;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn && s.err.empty()) s.err = std::string("cuSOLVER symbol missing: ") + name;
    };
    sym(s.create, "cusolverDnCreate");
    sym(s.destroy, "cusolverDnDestroy");
    sym(s.set_stream, "cusolverDnSetStream");
    sym(s.potrf_ws, "cusolverDnDpotrf_bufferSize");
    sym(s.potrf, "cusolverDnDpotrf");
    sym(s.potrs, "cusolverDnDpotrs");
    sym(s.gesvd_ws, "cusolverDnDgesvd_bufferSize");
    sym(s.gesvd, "cusolverDnDgesvd");
    return s;
  }
};

void sol_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS)
    throw Failure(Code::solver, std::string("cuSOLVER ") + what + " failed (status " + std::to_string(int(st)) + ")");
}

constexpr int kMaxMats = 8;
struct MatTable {
  MatDev m[kMaxMats];
};

// ---------------------------------------------------------------------------
// Kernels

// One CTA per element: strains + material update at its 3 integration points
// (threads 0-2), element force (threads 0-11) and, with_K, the 12x12 element
// stiffness (thread t = entry (t / 12, t % 12)). Arithmetic order follows
// assemble_micro (rve.hpp:233-256): eps = B u_el, f_a += (B^T sigma)_a w,
// k_ab += (B^T (C B))_ab w over the points in order.
__global__ void __launch_bounds__(144) k_hf_element(int n_el, const int* __restrict__ conn,
                                                    const int* __restrict__ phase, MatTable mats,
                                                    const double* __restrict__ B, const double* __restrict__ w,
                                                    const double* __restrict__ u, const double* __restrict__ st0,
                                                    int with_K, double* __restrict__ f_el, double* __restrict__ k_el,
                                                    double* __restrict__ st_out, double* __restrict__ sig_out,
                                                    double* __restrict__ C_out, int* __restrict__ err) {
  const int e = blockIdx.x, t = threadIdx.x;
  if (e >= n_el) return;
  __shared__ double sB[3][36], sS[3][3], sC[3][9], sW[3];
  for (int i = t; i < 108; i += blockDim.x) sB[i / 36][i % 36] = B[(size_t)108 * e + i];
  __syncthreads();
  if (t < 3) {
    const int ip = 3 * e + t;
    double ue[12];
    for (int a = 0; a < 6; ++a) {
      const int nd = conn[6 * e + a];
      ue[2 * a] = u[2 * nd];
      ue[2 * a + 1] = u[2 * nd + 1];
    }
    double eps[3];
    for (int r = 0; r < 3; ++r) {
      double s = 0.0;
      for (int c = 0; c < 12; ++c) s += sB[t][r * 12 + c] * ue[c];
      eps[r] = s;
    }
    const double* s0 = st0 + (size_t)6 * ip;
    bool ok = true;
    const MatOut o =
        update_material_any(mats.m[phase[e]], s0[0], s0[1], s0[2], s0[3], s0[4], eps[0], eps[1], eps[2], ok);
    if (!ok) atomicExch(err, 1);
    sS[t][0] = o.s0;
    sS[t][1] = o.s1;
    sS[t][2] = o.s2;
    const double Cf[9] = {o.c00, o.c01, o.c02, o.c01, o.c11, o.c12, o.c02, o.c12, o.c22};
    for (int k = 0; k < 9; ++k) sC[t][k] = Cf[k];
    sW[t] = w[ip];
    if (with_K) {
      double* so = st_out + (size_t)6 * ip;
      so[0] = o.ep0;
      so[1] = o.ep1;
      so[2] = o.ep2;
      so[3] = o.ep3;
      so[4] = o.eq;
      so[5] = o.s33;
      sig_out[3 * ip] = o.s0;
      sig_out[3 * ip + 1] = o.s1;
      sig_out[3 * ip + 2] = o.s2;
      for (int k = 0; k < 9; ++k) C_out[(size_t)9 * ip + k] = Cf[k];
    }
  }
  __syncthreads();
  if (t < 12) {
    double f = 0.0;
    for (int g = 0; g < 3; ++g) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) s += sB[g][i * 12 + t] * sS[g][i];
      f += s * sW[g];
    }
    f_el[(size_t)12 * e + t] = f;
  }
  if (with_K) {
    const int a = t / 12, b = t % 12;
    double k = 0.0;
    for (int g = 0; g < 3; ++g) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) {
        double cb = 0.0;
        for (int j = 0; j < 3; ++j) cb += sC[g][3 * i + j] * sB[g][j * 12 + b];
        s += sB[g][i * 12 + a] * cb;
      }
      k += s * sW[g];
    }
    k_el[(size_t)144 * e + t] = k;
  }
}

// One thread per DOF: residual entry and (free DOF, with_K) its stiffness
// row, summed over the DOF's element incidences in ascending element order.
__global__ void k_hf_gather(int nd, const int* __restrict__ inc_ptr, const int* __restrict__ inc,
                            const int* __restrict__ conn, const int* __restrict__ free_index, int nf,
                            const double* __restrict__ f_el, const double* __restrict__ k_el, int with_K,
                            double* __restrict__ f_full, double* __restrict__ K) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const int p0 = inc_ptr[d], p1 = inc_ptr[d + 1];
  double f = 0.0;
  for (int p = p0; p < p1; ++p) f += f_el[inc[p]];
  f_full[d] = f;
  const int fa = free_index[d];
  if (!with_K || fa < 0) return;
  double* row = K + (size_t)fa * nf;
  for (int p = p0; p < p1; ++p) {
    const int e = inc[p] / 12, a = inc[p] % 12;
    const double* ke = k_el + (size_t)144 * e + 12 * a;
    for (int b = 0; b < 12; ++b) {
      const int fb = free_index[2 * conn[6 * e + b / 2] + b % 2];
      if (fb >= 0) row[fb] += ke[b];
    }
  }
}

double norm2(const double* v, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

}  // namespace

}  // namespace fe2

using namespace fe2;

struct fe2_hf_s {
  int device = 0;
  RveData r;
  MatTable mats{}, mats_el{};
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t sol = nullptr;
  int *d_conn = nullptr, *d_phase = nullptr, *d_free = nullptr, *d_inc_ptr = nullptr, *d_inc = nullptr;
  int* d_info = nullptr;
  int* d_err = nullptr;  // set by k_hf_element when a return map fails
  double *d_B = nullptr, *d_w = nullptr, *d_u = nullptr, *d_st0 = nullptr, *d_st1 = nullptr;
  double *d_fel = nullptr, *d_kel = nullptr, *d_f = nullptr, *d_K = nullptr, *d_sig = nullptr, *d_C = nullptr;
  double *d_rhs = nullptr, *d_work = nullptr;
  int lwork = 0;
  bool factored = false;  // d_K holds the Cholesky factor of the last assembled stiffness
  double* st_comm = nullptr;  // committed states the assembly reads (d_st0, or a point's block)
  // macro-point batch (fe2_hf_alloc_points): per point committed states on the
  // device, committed free displacements / strains on the host; snapshot copies
  int64_t P = 0;
  double *d_pst = nullptr, *d_pst_snap = nullptr;
  std::vector<double> pu, pu_snap, pE, pE_snap;  // [P][nf], [P][6] = (E_prev, E_comm)

  int nd() const { return r.n_dofs(); }
  int nf() const { return r.n_free; }

  ~fe2_hf_s() {
    if (sol) Cusolver::get().destroy(sol);
    if (stream) cudaStreamDestroy(stream);
    for (int* p : {d_conn, d_phase, d_free, d_inc_ptr, d_inc, d_info, d_err})
      if (p) cudaFree(p);
    for (double* p : {d_B, d_w, d_u, d_st0, d_st1, d_fel, d_kel, d_f, d_K, d_sig, d_C, d_rhs, d_work, d_pst, d_pst_snap})
      if (p) cudaFree(p);
  }

  void affine(const double* E, std::vector<double>& u) const {  // affine_field, rve.hpp:43-51
    u.assign(nd(), 0.0);
    const double e11 = E[0], e22 = E[1], e12 = 0.5 * E[2];
    for (int id = 0; id < r.n_nodes; ++id) {
      u[2 * id] = e11 * r.x[id] + e12 * r.y[id];
      u[2 * id + 1] = e12 * r.x[id] + e22 * r.y[id];
    }
  }

  // assemble_micro at u_full from the committed states (d_st0); with_K also
  // keeps the trial states, stresses and tangents of every point.
  void assemble(const std::vector<double>& u_full, bool with_K, const MatTable& mt, std::vector<double>& f_full) {
    CK(cudaMemcpyAsync(d_u, u_full.data(), sizeof(double) * nd(), cudaMemcpyHostToDevice, stream));
    if (with_K) CK(cudaMemsetAsync(d_K, 0, sizeof(double) * nf() * nf(), stream));
    k_hf_element<<<r.n_el, 144, 0, stream>>>(r.n_el, d_conn, d_phase, mt, d_B, d_w, d_u, st_comm, with_K ? 1 : 0,
                                             d_fel, d_kel, d_st1, d_sig, d_C, d_err);
    CK(cudaGetLastError());
    k_hf_gather<<<(nd() + 127) / 128, 128, 0, stream>>>(nd(), d_inc_ptr, d_inc, d_conn, d_free, nf(), d_fel, d_kel,
                                                        with_K ? 1 : 0, d_f, d_K);
    CK(cudaGetLastError());
    f_full.resize(nd());
    CK(cudaMemcpyAsync(f_full.data(), d_f, sizeof(double) * nd(), cudaMemcpyDeviceToHost, stream));
    int err = 0;
    CK(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check(err == 0, Code::material, "material return map did not converge");
    if (with_K) factored = false;
  }

  void factor(const char* what) {
    const Cusolver& cs = Cusolver::get();
    // d_K is row-major; cuSOLVER's column-major UPPER triangle is its row-major lower one
    sol_check(cs.potrf(sol, CUBLAS_FILL_MODE_UPPER, nf(), d_K, nf(), d_work, lwork, d_info), "potrf");
    int info = 0;
    CK(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check(info == 0, Code::solver, what);
    factored = true;
  }

  // x = K^-1 b for nrhs column-major right-hand sides (in place on host b)
  void solve(std::vector<double>& b, int nrhs) {
    const Cusolver& cs = Cusolver::get();
    CK(cudaMemcpyAsync(d_rhs, b.data(), sizeof(double) * nf() * nrhs, cudaMemcpyHostToDevice, stream));
    sol_check(cs.potrs(sol, CUBLAS_FILL_MODE_UPPER, nf(), nrhs, d_K, nf(), d_rhs, nf(), d_info), "potrs");
    CK(cudaMemcpyAsync(b.data(), d_rhs, sizeof(double) * nf() * nrhs, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }

  struct Newton {
    bool converged = false;
    int iterations = 0;
    double res_last = 0.0;
    std::vector<double> u_full;
  };

  // micro_newton (rve.hpp:285-346): boundary DOFs fixed to E.x, reference
  // force = max(|r_0|, |boundary reactions_0|, 1e-30), 8-halving Armijo line
  // search keeping the best trial. On convergence d_st1 / d_sig / d_C / d_K
  // hold the converged states, stresses, tangents and (unfactored) stiffness.
  Newton newton(const double* E, std::vector<double> u_free, double tol, int max_iter, const MatTable& mt) {
    const int n = nf(), N = nd();
    Newton out;
    std::vector<double> aff;
    affine(E, aff);
    auto expand = [&](const std::vector<double>& uf, std::vector<double>& u) {
      u.resize(N);
      for (int i = 0; i < N; ++i) u[i] = r.free_index[i] >= 0 ? uf[r.free_index[i]] : aff[i];
    };
    auto reduce = [&](const std::vector<double>& f, std::vector<double>& rr) {
      rr.assign(n, 0.0);
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) rr[r.free_index[i]] += f[i];
    };
    std::vector<double> f_full, res, du(n), ut(n), u_trial, rt;
    double ref = 0.0;
    for (int it = 0; it <= max_iter; ++it) {
      expand(u_free, out.u_full);
      assemble(out.u_full, true, mt, f_full);
      reduce(f_full, res);
      const double rn = norm2(res.data(), n);
      out.res_last = rn;
      if (it == 0) {
        double s = 0.0;
        for (int i = 0; i < N; ++i)
          if (r.free_index[i] < 0) s += f_full[i] * f_full[i];
        ref = std::max({rn, std::sqrt(s), 1e-30});
      }
      if (rn <= tol * ref) {
        out.converged = true;
        out.iterations = it;
        return out;
      }
      if (it == max_iter) break;
      factor("micro stiffness factorization failed");
      for (int i = 0; i < n; ++i) du[i] = -res[i];
      solve(du, 1);
      double alpha = 1.0, best_alpha = 1.0, best_rn = std::numeric_limits<double>::infinity();
      for (int ls = 0; ls < 8; ++ls) {
        for (int i = 0; i < n; ++i) ut[i] = u_free[i] + alpha * du[i];
        expand(ut, u_trial);
        assemble(u_trial, false, mt, f_full);
        reduce(f_full, rt);
        const double trial = norm2(rt.data(), n);
        if (trial < best_rn) {
          best_rn = trial;
          best_alpha = alpha;
        }
        if (trial <= (1.0 - 1e-4 * alpha) * rn) break;
        alpha *= 0.5;
      }
      for (int i = 0; i < n; ++i) u_free[i] = u_free[i] + best_alpha * du[i];
    }
    out.converged = false;
    out.iterations = max_iter;
    return out;
  }

  // homogenize (rve.hpp:350-392) at the converged state of the last newton().
  void homogenize(double* sigma, double* C) {
    const int n = nf(), N = nd(), nip = r.n_ips();
    std::vector<double> sg((size_t)3 * nip), Cq((size_t)9 * nip);
    CK(cudaMemcpyAsync(sg.data(), d_sig, sizeof(double) * sg.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(Cq.data(), d_C, sizeof(double) * Cq.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    double s[3] = {0, 0, 0};
    for (int ip = 0; ip < nip; ++ip)
      for (int i = 0; i < 3; ++i) s[i] += r.w[ip] * sg[3 * ip + i];
    for (int i = 0; i < 3; ++i) sigma[i] = s[i] / r.volume;
    std::vector<double> rhs_full((size_t)N * 3, 0.0);
    double c_avg[9] = {0};
    for (int ip = 0; ip < nip; ++ip) {
      const int* el = r.conn.data() + 6 * (ip / 3);
      const double* B = r.B.data() + (size_t)36 * ip;
      const double* Cp = Cq.data() + (size_t)9 * ip;
      for (int a = 0; a < 12; ++a) {
        const int ga = 2 * el[a / 2] + a % 2;
        for (int j = 0; j < 3; ++j) {
          double t = 0.0;
          for (int i = 0; i < 3; ++i) t += B[i * 12 + a] * Cp[3 * i + j];
          rhs_full[(size_t)ga * 3 + j] += t * r.w[ip];
        }
      }
      for (int k = 0; k < 9; ++k) c_avg[k] += r.w[ip] * Cp[k];
    }
    if (!factored) factor("homogenize: singular converged stiffness");
    std::vector<double> h((size_t)n * 3, 0.0);
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) h[(size_t)j * n + r.free_index[i]] += rhs_full[(size_t)i * 3 + j];
    for (double& v : h) v = -v;
    solve(h, 3);
    double c_hom[9];
    for (int k = 0; k < 9; ++k) c_hom[k] = c_avg[k];
    std::vector<double> h_full(N);
    for (int j = 0; j < 3; ++j) {
      for (int i = 0; i < N; ++i) h_full[i] = r.free_index[i] >= 0 ? h[(size_t)j * n + r.free_index[i]] : 0.0;
      for (int ip = 0; ip < nip; ++ip) {
        const int* el = r.conn.data() + 6 * (ip / 3);
        const double* B = r.B.data() + (size_t)36 * ip;
        const double* Cp = Cq.data() + (size_t)9 * ip;
        double he[12];
        for (int a = 0; a < 6; ++a) {
          he[2 * a] = h_full[2 * el[a]];
          he[2 * a + 1] = h_full[2 * el[a] + 1];
        }
        double bh[3];
        for (int q = 0; q < 3; ++q) {
          double t = 0.0;
          for (int c = 0; c < 12; ++c) t += B[q * 12 + c] * he[c];
          bh[q] = t;
        }
        for (int i = 0; i < 3; ++i) {
          double t = 0.0;
          for (int k = 0; k < 3; ++k) t += Cp[3 * i + k] * bh[k];
          c_hom[3 * i + j] += r.w[ip] * t;
        }
      }
    }
    for (int k = 0; k < 9; ++k) C[k] = c_hom[k] / r.volume;
  }

  // One path step of run_trajectory (rve.hpp:459-491) from the committed
  // state (st_comm on the device, u_free, E_comm) towards E_target, E_prev
  // being the previous path point: warm start = committed solution + affine
  // increment, bisection on non-convergence (throws ErrorCode::solver after
  // max_bisections). On success the committed state has advanced; the last
  // converged Newton result is returned (its d_sig / d_C / d_K are current).
  Newton increment(const double* E_prev, const double* E_target, std::vector<double>& u_free, double* E_comm,
                   double tol, int max_iter, int max_bisections, const MatTable& mt, int& its) {
    const int N = nd();
    std::vector<double> aff, u0(nf());
    double done = 0.0, frac = 1.0;
    int bis = 0;
    its = 0;
    Newton res;
    while (done < 1.0 - 1e-12) {
      const double target = std::min(1.0, done + frac);
      double Ev[3], dE[3];
      for (int i = 0; i < 3; ++i) Ev[i] = E_prev[i] + (E_target[i] - E_prev[i]) * target;
      for (int i = 0; i < 3; ++i) dE[i] = Ev[i] - E_comm[i];
      affine(dE, aff);
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) u0[r.free_index[i]] = u_free[r.free_index[i]] + aff[i];
      MatTable ms = mt;  // creep: the sub-step's fraction of the increment's dt (rve.hpp:466)
      for (MatDev& md : ms.m) md.dt *= target - done;
      res = newton(Ev, u0, tol, max_iter, ms);
      its += res.iterations;
      if (!res.converged) {
        check(++bis <= max_bisections, Code::solver, "micro trajectory failed after max bisections");
        frac *= 0.5;
        continue;
      }
      CK(cudaMemcpyAsync(st_comm, d_st1, sizeof(double) * 6 * r.n_ips(), cudaMemcpyDeviceToDevice, stream));
      for (int i = 0; i < N; ++i)
        if (r.free_index[i] >= 0) u_free[r.free_index[i]] = res.u_full[i];
      for (int i = 0; i < 3; ++i) E_comm[i] = Ev[i];
      done = target;
    }
    return res;
  }

  // run_trajectory (rve.hpp:448-494) from the virgin state.
  void trajectory(int n_steps, const double* E, double tol, int max_iter, int max_bisections, const MatTable& mt,
                  double* sigma, double* C, int* iterations, double* u_fluct_inf, double* res_last, double* snaps) {
    const int n = nf(), N = nd();
    st_comm = d_st0;
    CK(cudaMemsetAsync(d_st0, 0, sizeof(double) * 6 * r.n_ips(), stream));
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), stream));
    std::vector<double> u_free(n, 0.0), aff;
    double E_prev[3] = {0, 0, 0}, E_comm[3] = {0, 0, 0};
    for (int k = 0; k < n_steps; ++k) {
      int its = 0;
      const Newton res = increment(E_prev, E + 3 * k, u_free, E_comm, tol, max_iter, max_bisections, mt, its);
      if (sigma || C) {
        double s3[3], c9[9];
        homogenize(s3, c9);
        if (sigma) std::memcpy(sigma + 3 * k, s3, sizeof(s3));
        if (C) std::memcpy(C + 9 * k, c9, sizeof(c9));
      }
      affine(E_comm, aff);
      double mx = 0.0;
      for (int i = 0; i < N; ++i) {
        const double wv = res.u_full[i] - aff[i];
        mx = std::max(mx, std::abs(wv));
        if (snaps) snaps[(size_t)k * N + i] = wv;
      }
      if (u_fluct_inf) u_fluct_inf[k] = mx;
      if (res_last) res_last[k] = res.res_last;
      if (iterations) iterations[k] = its;
      for (int i = 0; i < 3; ++i) E_prev[i] = E[3 * k + i];
    }
    CK(cudaStreamSynchronize(stream));
  }

  // A batch of P macro points, each an RVE with its own committed state
  // (the HF engine of an FE² run, SPEC.md:474-477 HF_nested). One increment
  // per call for every point; a point whose step fails keeps its committed
  // state and reports status 1 + ErrorCode.
  void alloc_points(int64_t n_points) {
    dfree(d_pst);
    dfree(d_pst_snap);
    P = n_points;
    d_pst = dalloc<double>(static_cast<size_t>(P) * 6 * r.n_ips());
    d_pst_snap = dalloc<double>(static_cast<size_t>(P) * 6 * r.n_ips());
    CK(cudaMemsetAsync(d_pst, 0, sizeof(double) * P * 6 * r.n_ips(), stream));
    CK(cudaMemsetAsync(d_pst_snap, 0, sizeof(double) * P * 6 * r.n_ips(), stream));
    pu.assign(static_cast<size_t>(P) * nf(), 0.0);
    pE.assign(static_cast<size_t>(P) * 6, 0.0);
    pu_snap = pu;
    pE_snap = pE;
    CK(cudaStreamSynchronize(stream));
  }

  void solve_points(const double* E, double tol, int max_iter, int max_bisections, double* sigma, double* C,
                    int* iters, int* status) {
    const int n = nf();
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), stream));
    std::vector<double> u_free(n);
    for (int64_t p = 0; p < P; ++p) {
      st_comm = d_pst + static_cast<size_t>(p) * 6 * r.n_ips();
      double* Ep = pE.data() + 6 * p;  // (E_prev, E_comm)
      std::copy(pu.begin() + p * n, pu.begin() + (p + 1) * n, u_free.begin());
      double E_comm[3] = {Ep[3], Ep[4], Ep[5]};
      int its = 0, code = 0;
      const size_t sb = sizeof(double) * 6 * r.n_ips();
      CK(cudaMemcpyAsync(d_st0, st_comm, sb, cudaMemcpyDeviceToDevice, stream));  // backup for a failed step
      try {
        increment(Ep, E + 3 * p, u_free, E_comm, tol, max_iter, max_bisections, mats, its);
        double s3[3], c9[9];
        homogenize(s3, c9);
        if (sigma) std::memcpy(sigma + 3 * p, s3, sizeof(s3));
        if (C) std::memcpy(C + 9 * p, c9, sizeof(c9));
        std::copy(u_free.begin(), u_free.end(), pu.begin() + p * n);
        for (int i = 0; i < 3; ++i) {
          Ep[i] = E[3 * p + i];
          Ep[3 + i] = E_comm[i];
        }
      } catch (const Failure& f) {
        code = 1 + static_cast<int>(f.code);
        CK(cudaMemsetAsync(d_err, 0, sizeof(int), stream));
        // a failed bisection may have committed sub-steps: return to the call's start
        CK(cudaMemcpyAsync(st_comm, d_st0, sb, cudaMemcpyDeviceToDevice, stream));
      }
      if (iters) iters[p] = its;
      if (status) status[p] = code;
    }
    st_comm = d_st0;
    CK(cudaStreamSynchronize(stream));
  }
};

extern "C" {

int fe2_hf_create(int device, int subdivisions, const char* mesh_path, const fe2_material_t* materials, int n_materials,
                  fe2_hf_t* out) {
  return guard([&] {
    check(out && materials && n_materials >= 1 && n_materials <= kMaxMats, Code::config, "bad HF arguments");
    *out = nullptr;
    auto h = std::make_unique<fe2_hf_s>();
    for (int i = 0; i < n_materials; ++i) {
      h->mats.m[i] = to_dev(materials[i]);
      fe2_material_t el = materials[i];
      el.kind = 0;  // the elastic part (build_elastic_modes)
      h->mats_el.m[i] = to_dev(el);
    }
    h->r = rve_data(subdivisions, mesh_path);
    const RveData& r = h->r;
    for (int e = 0; e < r.n_el; ++e)
      check(r.phase[e] >= 0 && r.phase[e] < n_materials, Code::config, "element material id out of range");
    check(r.n_free >= 1, Code::mesh, "RVE has no free DOF");
    require_device(device);
    h->device = device;
    const Cusolver& cs = Cusolver::get();
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    sol_check(cs.create(&h->sol), "create");
    sol_check(cs.set_stream(h->sol, h->stream), "set stream");
    // per-DOF element incidences in ascending element order (CSR)
    const int N = r.n_dofs(), n = r.n_free;
    std::vector<int> cnt(N + 1, 0), inc;
    for (int e = 0; e < r.n_el; ++e)
      for (int a = 0; a < 12; ++a) ++cnt[2 * r.conn[6 * e + a / 2] + a % 2 + 1];
    for (int d = 0; d < N; ++d) cnt[d + 1] += cnt[d];
    inc.resize(cnt[N]);
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < r.n_el; ++e)
      for (int a = 0; a < 12; ++a) inc[pos[2 * r.conn[6 * e + a / 2] + a % 2]++] = 12 * e + a;
    auto up_i = [&](int*& d, const std::vector<int>& v) {
      d = dalloc<int>(v.size());
      CK(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    };
    auto up_d = [&](double*& d, const std::vector<double>& v) {
      d = dalloc<double>(v.size());
      CK(cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
    };
    up_i(h->d_conn, r.conn);
    up_i(h->d_phase, r.phase);
    up_i(h->d_free, r.free_index);
    up_i(h->d_inc_ptr, cnt);
    up_i(h->d_inc, inc);
    up_d(h->d_B, r.B);
    up_d(h->d_w, r.w);
    h->d_info = dalloc<int>(1);
    h->d_err = dalloc<int>(1);
    CK(cudaMemset(h->d_err, 0, sizeof(int)));
    h->d_u = dalloc<double>(N);
    h->d_f = dalloc<double>(N);
    h->d_st0 = dalloc<double>((size_t)6 * r.n_ips());
    h->d_st1 = dalloc<double>((size_t)6 * r.n_ips());
    h->d_sig = dalloc<double>((size_t)3 * r.n_ips());
    h->d_C = dalloc<double>((size_t)9 * r.n_ips());
    h->d_fel = dalloc<double>((size_t)12 * r.n_el);
    h->d_kel = dalloc<double>((size_t)144 * r.n_el);
    h->d_K = dalloc<double>((size_t)n * n);
    h->d_rhs = dalloc<double>((size_t)3 * n);
    sol_check(cs.potrf_ws(h->sol, CUBLAS_FILL_MODE_UPPER, n, h->d_K, n, &h->lwork), "potrf workspace");
    h->d_work = dalloc<double>(std::max(1, h->lwork));
    *out = h.release();
  });
}

void fe2_hf_destroy(fe2_hf_t h) {
  if (!h) return;
  cudaSetDevice(h->device);
  delete h;
}

int fe2_hf_sizes(fe2_hf_t h, int* n_dofs, int* n_free, int* n_ips, double* volume) {
  return guard([&] {
    check(h != nullptr, Code::config, "null HF handle");
    if (n_dofs) *n_dofs = h->nd();
    if (n_free) *n_free = h->nf();
    if (n_ips) *n_ips = h->r.n_ips();
    if (volume) *volume = h->r.volume;
  });
}

int fe2_hf_trajectory(fe2_hf_t h, int n_steps, const double* E, const fe2_newton_opts_t* opts, double* sigma,
                      double* C, int* iterations, double* u_fluct_inf, double* res_last, double* snapshots) {
  return guard([&] {
    check(h && E && opts && n_steps >= 0, Code::config, "bad HF trajectory arguments");
    check(opts->tol > 0.0 && opts->max_iter >= 1 && opts->max_bisections >= 0, Code::config, "bad Newton options");
    CK(cudaSetDevice(h->device));
    h->trajectory(n_steps, E, opts->tol, opts->max_iter, opts->max_bisections, h->mats, sigma, C, iterations,
                  u_fluct_inf, res_last, snapshots);
  });
}

int fe2_hf_alloc_points(fe2_hf_t h, int64_t P) {
  return guard([&] {
    check(h != nullptr && P >= 1, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    h->alloc_points(P);
  });
}

int fe2_hf_solve_increment(fe2_hf_t h, const double* E, const fe2_newton_opts_t* opts, double* sigma, double* C,
                           int* iters, int* status) {
  return guard([&] {
    check(h && E && opts, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    check(opts->tol > 0.0 && opts->max_iter >= 1 && opts->max_bisections >= 0, Code::config, "bad Newton options");
    CK(cudaSetDevice(h->device));
    h->solve_points(E, opts->tol, opts->max_iter, opts->max_bisections, sigma, C, iters, status);
  });
}

int fe2_hf_snapshot(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(h->d_pst_snap, h->d_pst, sizeof(double) * h->P * 6 * h->r.n_ips(), cudaMemcpyDeviceToDevice,
                       h->stream));
    h->pu_snap = h->pu;
    h->pE_snap = h->pE;
    CK(cudaStreamSynchronize(h->stream));
  });
}

int fe2_hf_restore(fe2_hf_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hf_alloc_points)");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(h->d_pst, h->d_pst_snap, sizeof(double) * h->P * 6 * h->r.n_ips(), cudaMemcpyDeviceToDevice,
                       h->stream));
    h->pu = h->pu_snap;
    h->pE = h->pE_snap;
    CK(cudaStreamSynchronize(h->stream));
  });
}

int fe2_hf_points(fe2_hf_t h, int64_t* P) {
  return guard([&] {
    check(h != nullptr && P != nullptr, Code::config, "bad arguments");
    *P = h->P;
  });
}

int fe2_hf_elastic_modes(fe2_hf_t h, double* modes, int* count) {
  return guard([&] {
    check(h && modes && count, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    const int N = h->nd();
    std::vector<double> A((size_t)3 * N), drop(3);
    for (int j = 0; j < 3; ++j) {
      double E[3] = {0, 0, 0};
      E[j] = 1.0;
      int its = 0;
      h->trajectory(1, E, 1e-10, 10, 0, h->mats_el, nullptr, nullptr, &its, nullptr, nullptr, A.data() + (size_t)j * N);
      std::vector<double> aff;
      h->affine(E, aff);
      drop[j] = 1e-10 * norm2(aff.data(), aff.size());
    }
    *count = orthonormalize_columns(A, N, 3, drop);
    std::memset(modes, 0, sizeof(double) * 3 * N);
    std::memcpy(modes, A.data(), sizeof(double) * A.size());
  });
}

int fe2_pod_basis(int device, const double* X, int64_t n_rows, int n_cols, const double* elastic, int n_elastic,
                  int n_target, double* V, double* singular_values, int* max_modes) {
  return guard([&] {
    check(X && V && n_rows >= 1 && n_cols >= 1 && n_elastic >= 0 && (n_elastic == 0 || elastic), Code::config,
          "bad POD arguments");
    check(n_target >= std::max(1, n_elastic) && n_target <= n_rows, Code::config, "POD target out of range");
    check(n_rows * static_cast<int64_t>(n_cols) < (int64_t(1) << 31), Code::config, "snapshot matrix too large");
    const size_t R = static_cast<size_t>(n_rows), M = static_cast<size_t>(n_cols);
    // elastic modes, orthonormalised
    std::vector<double> Em(elastic, elastic + R * n_elastic);
    const int ne = orthonormalize_columns(Em, n_rows, n_elastic, std::vector<double>(n_elastic, 1e-10));
    check(ne == n_elastic, Code::config, "elastic modes are linearly dependent");
    // deflation against the elastic span (classical Gram-Schmidt, twice)
    std::vector<double> D(X, X + R * M);
    const double xnorm = norm2(X, R * M);
    for (int pass = 0; pass < 2; ++pass)
      for (size_t c = 0; c < M; ++c) {
        double* d = D.data() + c * R;
        for (int j = 0; j < ne; ++j) {
          const double* q = Em.data() + static_cast<size_t>(j) * R;
          double dot = 0.0;
          for (size_t i = 0; i < R; ++i) dot += q[i] * d[i];
          for (size_t i = 0; i < R; ++i) d[i] -= dot * q[i];
        }
      }
    // SVD of the deflated snapshots on the device (gesvd needs rows >= cols:
    // otherwise factor D^T and read the left vectors from its VT)
    require_device(device);
    const Cusolver& cs = Cusolver::get();
    cusolverDnHandle_t sol = nullptr;
    sol_check(cs.create(&sol), "create");
    const bool tall = R >= M;
    const int m = tall ? n_rows : n_cols, n = tall ? n_cols : static_cast<int>(n_rows);
    std::vector<double> A(R * M);
    if (tall) A = D;
    else
      for (size_t c = 0; c < M; ++c)
        for (size_t i = 0; i < R; ++i) A[c + i * M] = D[i + c * R];
    double *dA = nullptr, *dS = nullptr, *dU = nullptr, *dW = nullptr, *dRw = nullptr;
    int* dInfo = nullptr;
    int lw = 0, info = 0;
    std::vector<double> S(n), Uh;
    try {
      dA = dalloc<double>(A.size());
      dS = dalloc<double>(n);
      dU = dalloc<double>(static_cast<size_t>(tall ? m : n) * n);
      dRw = dalloc<double>(n);
      dInfo = dalloc<int>(1);
      CK(cudaMemcpy(dA, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
      sol_check(cs.gesvd_ws(sol, m, n, &lw), "gesvd workspace");
      dW = dalloc<double>(std::max(1, lw));
      if (tall)
        sol_check(cs.gesvd(sol, 'S', 'N', m, n, dA, m, dS, dU, m, nullptr, n, dW, lw, dRw, dInfo), "gesvd");
      else
        sol_check(cs.gesvd(sol, 'N', 'S', m, n, dA, m, dS, nullptr, m, dU, n, dW, lw, dRw, dInfo), "gesvd");
      CK(cudaMemcpy(&info, dInfo, sizeof(int), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(S.data(), dS, sizeof(double) * n, cudaMemcpyDeviceToHost));
      Uh.resize(static_cast<size_t>(tall ? m : n) * n);
      CK(cudaMemcpy(Uh.data(), dU, sizeof(double) * Uh.size(), cudaMemcpyDeviceToHost));
    } catch (...) {
      for (double* p : {dA, dS, dU, dW, dRw}) dfree(p);
      dfree(dInfo);
      cs.destroy(sol);
      throw;
    }
    for (double* p : {dA, dS, dU, dW, dRw}) dfree(p);
    dfree(dInfo);
    cs.destroy(sol);
    check(info == 0, Code::solver, "SVD did not converge");
    const int ns = std::min<int64_t>(n_rows, n_cols);  // == n
    if (singular_values)
      for (int i = 0; i < n_cols; ++i) singular_values[i] = i < ns ? S[i] : 0.0;
    int rank = 0;
    while (rank < ns && S[rank] > 1e-10 * xnorm) ++rank;
    if (max_modes) *max_modes = ne + rank;
    const int k = n_target - ne;
    check(k <= rank, Code::rank,
          "POD: requested " + std::to_string(n_target) + " modes, at most " + std::to_string(ne + rank) + " usable");
    // left singular vector i: column i of U (tall) or row i of VT (n x n, wide)
    std::vector<double> Vh(R * n_target);
    std::copy(Em.begin(), Em.end(), Vh.begin());
    for (int i = 0; i < k; ++i) {
      double* v = Vh.data() + static_cast<size_t>(ne + i) * R;
      for (size_t r = 0; r < R; ++r) v[r] = tall ? Uh[r + static_cast<size_t>(i) * m] : Uh[i + r * static_cast<size_t>(n)];
    }
    const int kept = orthonormalize_columns(Vh, n_rows, n_target, std::vector<double>(n_target, 1e-8));
    check(kept == n_target, Code::numeric, "POD basis lost rank in re-orthonormalisation");
    for (int j = ne; j < n_target; ++j) {  // sign: largest-magnitude entry positive (lowest index on ties)
      double* v = Vh.data() + static_cast<size_t>(j) * R;
      size_t im = 0;
      for (size_t r = 1; r < R; ++r)
        if (std::abs(v[r]) > std::abs(v[im])) im = r;
      if (v[im] < 0.0)
        for (size_t r = 0; r < R; ++r) v[r] = -v[r];
    }
    std::memcpy(V, Vh.data(), sizeof(double) * Vh.size());
  });
}

}  // extern "C"
