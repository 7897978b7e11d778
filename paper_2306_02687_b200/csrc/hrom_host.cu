// Host driver of the B200 hyper-ROM engine behind the C ABI
// (include/fe2rom/fe2rom_gpu.h). Owns the device model (projected operator
// rows, weights, elastic-predictor constants), the per-point SoA state in
// HBM, and the increment loop: one persistent kernel launch per increment
// (assembly + Newton + condensation + commit fused, see hrom_kernels.cu).
// One handle per device; no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"
#include "hrom_kernels.cuh"
#include "host_util.cuh"

namespace fe2 {

namespace {
thread_local std::string g_last_error;

}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace fe2

using namespace fe2;

struct fe2_hrom_s {
  int device = 0, num_sms = 148;
  cudaStream_t stream = nullptr;  // work stream (own, or the caller's)
  cudaStream_t own_stream = nullptr;
  int kin = 0;  // 0 small strain (E, sigma, C), 1 finite strain (H, P, A)
  int n = 0, NP = 0, S = 0, K = 0, K2 = 0, K2p = 0, Kel = 0, Kelp = 0;
  double volume = 0.0;
  MatDev matE{};  // finite strain: the elastic material
  std::vector<int> j2_idx, el_idx;  // original cubature indices
  std::vector<double> G, w;         // host copy (caller order)
  std::vector<MatDev> qmat;         // per original cubature point
  MatDev mat2{};
  double CEEe[9] = {0};
  // device model
  double *G2 = nullptr, *w2 = nullptr, *Ke = nullptr, *KaEe = nullptr, *Le = nullptr, *LeInv = nullptr;
  // device points
  int64_t P = 0;
  bool keep_flags = false;
  double *hist = nullptr, *alpha_c = nullptr, *E_c = nullptr, *bp = nullptr, *sp = nullptr;
  PointState* st = nullptr;
  uint8_t* flags = nullptr;
  int* work = nullptr;              // work-queue counter
  double* mono = nullptr;           // monolithic scheme: per-point working records (mono_stride)
  bool mono_first = true;           // the next fe2_hrom_mono_iterate starts a step
  IncCounters* cnt = nullptr;       // device counters of a launch
  IncCounters* h_cnt = nullptr;     // pinned copy
  // asynchronous host-buffer increments (fe2_hrom_solve_increment_async):
  // double-buffered device inputs/outputs, output copies on a second stream
  struct AsyncBuf {
    double *dE = nullptr, *sig = nullptr, *C = nullptr, *res = nullptr;
    int *it = nullptr, *pc = nullptr, *st = nullptr;
    cudaEvent_t done = nullptr, copied = nullptr;
    bool used = false;
  } abuf[2];
  int acur = 0;
  int64_t async_pending = 0;  // launches since the last fe2_hrom_wait
  cudaStream_t copy_stream = nullptr;
  IncCounters* cnt_async = nullptr;  // device accumulator of async launches
  // staging for the host-buffer API and default outputs
  double *dE = nullptr, *o_sigma = nullptr, *o_C = nullptr, *o_res = nullptr;
  int *o_iters = nullptr, *o_status = nullptr, *o_pc = nullptr;
  // multi-GPU exchange (fe2_hrom_gather): layout over the last communicator, device
  // scratch for the point counts and the two reduced flags, pinned flag readback
  ExchangeLayout xlayout{};
  int64_t* x_scratch = nullptr;
  int* x_flags = nullptr;
  int* h_xflags = nullptr;
  // stats
  bool timing = false;
  fe2_hrom_stats_t stats{};
  cudaEvent_t ev[2] = {nullptr, nullptr};

  int ncomp() const { return kin ? 4 : 3; }   // macro input / stress components
  // every increment kernel double-buffers the history (no commit pass)
  int nbuf() const { return 2; }
  int ntan() const { return kin ? 16 : 9; }    // macro tangent entries
  ModelDev model() const {
    ModelDev M{};
    M.n = n;
    M.NP = NP;
    M.S = S;
    M.K2 = K2;
    M.K2p = K2p;
    M.nchunks = (K2p + Kelp) / kQC;
    M.nch_hist = K2p / kQC;
    M.K_el = Kel;
    M.matE = matE;
    M.G2 = G2;
    M.w2 = w2;
    M.Ke = Ke;
    M.KaEe = KaEe;
    M.Le = Le;
    M.LeInv = LeInv;
    M.inv_denom = mat2.inv_denom;
    std::memcpy(M.CEEe, CEEe, sizeof CEEe);
    M.volume = volume;
    M.mat2 = mat2;
    return M;
  }
  PointsDev points() const {
    PointsDev D{};
    D.P = P;
    D.hist = hist;
    D.alpha_c = alpha_c;
    D.E_c = E_c;
    D.bp = bp;
    D.sp = sp;
    D.st = st;
    D.flags = flags;
    D.hist_alt = nbuf() == 2 ? static_cast<int64_t>(P) * K2p * 5 : 0;
    D.flags_alt = (nbuf() == 2 && flags) ? static_cast<int64_t>(P) * K2p : 0;
    return D;
  }
  // snapshot of the committed point state (fe2_hrom_snapshot / _restore)
  unsigned char* snap = nullptr;
  size_t snap_bytes = 0;
  struct Part {
    void* p;
    size_t bytes;
  };
  std::vector<Part> state_parts() const {
    std::vector<Part> v = {{hist, static_cast<size_t>(nbuf()) * P * K2p * 5 * sizeof(double)},
                           {alpha_c, static_cast<size_t>(P) * NP * sizeof(double)},
                           {bp, static_cast<size_t>(P) * NP * sizeof(double)},
                           {E_c, static_cast<size_t>(P) * ncomp() * sizeof(double)},
                           {sp, static_cast<size_t>(P) * 4 * sizeof(double)},
                           {st, static_cast<size_t>(P) * sizeof(PointState)}};
    if (flags) v.push_back({flags, static_cast<size_t>(nbuf()) * P * K2p});
    return v;
  }
  void free_async() {
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    for (auto& b : abuf) {
      dfree(b.dE);
      dfree(b.sig);
      dfree(b.C);
      dfree(b.res);
      dfree(b.it);
      dfree(b.pc);
      dfree(b.st);
      if (b.done) cudaEventDestroy(b.done);
      if (b.copied) cudaEventDestroy(b.copied);
      b = AsyncBuf{};
    }
    acur = 0;
  }
  void free_points() {
    free_async();
    dfree(mono);
    mono_first = true;
    dfree(snap);
    snap_bytes = 0;
    dfree(hist);
    dfree(alpha_c);
    dfree(E_c);
    dfree(bp);
    dfree(sp);
    dfree(st);
    dfree(flags);
    dfree(dE);
    dfree(o_sigma);
    dfree(o_C);
    dfree(o_res);
    dfree(o_iters);
    dfree(o_status);
    dfree(o_pc);
    P = 0;
  }
  void zero_points(cudaStream_t s) {
    CK(cudaMemsetAsync(hist, 0, static_cast<size_t>(nbuf()) * P * K2p * 5 * sizeof(double), s));
    const size_t an = static_cast<size_t>(P) * NP * sizeof(double);
    CK(cudaMemsetAsync(alpha_c, 0, an, s));
    CK(cudaMemsetAsync(bp, 0, an, s));
    CK(cudaMemsetAsync(E_c, 0, P * ncomp() * sizeof(double), s));
    CK(cudaMemsetAsync(sp, 0, P * 4 * sizeof(double), s));
    CK(cudaMemsetAsync(st, 0, P * sizeof(PointState), s));
    if (flags) CK(cudaMemsetAsync(flags, 0, static_cast<size_t>(nbuf()) * P * K2p, s));
  }
  ~fe2_hrom_s() {
    cudaSetDevice(device);
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    free_points();
    dfree(cnt_async);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    dfree(G2);
    dfree(w2);
    dfree(Ke);
    dfree(KaEe);
    dfree(Le);
    dfree(LeInv);
    dfree(work);
    dfree(cnt);
    dfree(x_scratch);
    dfree(x_flags);
    if (h_xflags) cudaFreeHost(h_xflags);
    if (h_cnt) cudaFreeHost(h_cnt);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
};

namespace {

void launch_any(fe2_hrom_t h, const IncArgs& a, int num_sms, cudaStream_t s) {
  if (h->kin == 1)
    launch_increment_fs(a, num_sms, s);
  else if (a.M.NP <= 32)
    launch_increment(a, num_sms, s);
  else
    check(launch_increment_big(a, num_sms, s), Code::config, "unsupported mode count");
}

struct Eps3 {
  double v[3];
};
// committed strain eps_q = E_c + G_q alpha_c of point p (host, readback only)
Eps3 strain_at(fe2_hrom_t h, int64_t p, int q, const double* ac, const double* Ec) {
  const int n = h->n, NP = h->NP;
  const double* Gq = h->G.data() + static_cast<size_t>(q) * 3 * n;
  Eps3 e;
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int a = 0; a < n; ++a) s += Gq[i * n + a] * ac[p * NP + a];
    e.v[i] = Ec[p * 3 + i] + s;
  }
  return e;
}

// finite strain: Biot strain (U00 - 1, U11 - 1) of the committed F_q = I + H_c + G4_q alpha_c
Eps3 biot_strain_at(fe2_hrom_t h, int64_t p, int q, const double* ac, const double* Hc) {
  const int n = h->n, NP = h->NP;
  const double* Gq = h->G.data() + static_cast<size_t>(q) * 4 * n;
  const double I4[4] = {1.0, 0.0, 0.0, 1.0};
  double F[4];
  for (int i = 0; i < 4; ++i) {
    double s = 0.0;
    for (int a = 0; a < n; ++a) s += Gq[i * n + a] * ac[p * NP + a];
    F[i] = (I4[i] + Hc[p * 4 + i]) + s;
  }
  const double num = F[2] - F[1], den = F[0] + F[3];
  const double rho = std::sqrt(num * num + den * den);
  const double c = den / rho, sn = num / rho;
  Eps3 e;
  e.v[0] = (c * F[0] + sn * F[2]) - 1.0;
  e.v[1] = (-sn * F[1] + c * F[3]) - 1.0;
  e.v[2] = 0.0;
  return e;
}

NewtonCfg make_cfg(const fe2_newton_opts_t* opts) {
  NewtonCfg cfg{1e-8, 30, 4};
  if (opts) {
    cfg.tol = opts->tol;
    cfg.max_iter = opts->max_iter;
    cfg.max_bis = opts->max_bisections;
  }
  check(cfg.tol > 0.0 && cfg.max_iter >= 0 && cfg.max_bis >= 0, Code::config, "invalid Newton options");
  return cfg;
}

// Watchdog (debug aid, FE2_TRACE=<seconds>): the persistent kernel writes its
// per-warp ring position and state into mapped pinned host memory; if the
// launch does not finish in time the trace is printed and the process exits
// instead of hanging the device.
struct Watchdog {
  int* host = nullptr;
  int* dev = nullptr;
  int slots = 0;
  double seconds = 0.0;
  explicit Watchdog(int num_sms) {
    const char* env = std::getenv("FE2_TRACE");
    if (!env || !*env) return;
    seconds = std::atof(env);
    if (seconds <= 0.0) seconds = 60.0;
    slots = num_sms * 4 * 8;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&host), slots * 4 * sizeof(int), cudaHostAllocMapped));
    std::memset(host, 0xff, slots * 4 * sizeof(int));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
  }
  ~Watchdog() {
    if (host) cudaFreeHost(host);
  }
  void wait(cudaStream_t s, const char* what) {
    if (!host) return;
    const auto t0 = std::chrono::steady_clock::now();
    while (cudaStreamQuery(s) == cudaErrorNotReady) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > seconds) {
        std::fprintf(stderr, "[fe2 watchdog] %s did not finish in %.0f s; warp {pos, state, issued, working}:\n",
                     what, seconds);
        for (int i = 0; i < slots; ++i)
          if (host[4 * i] != -1)
            std::fprintf(stderr, "  cta %d warp %d: %d %d %d %d\n", i / 8, i % 8, host[4 * i], host[4 * i + 1],
                         host[4 * i + 2], host[4 * i + 3]);
        std::fflush(stderr);
        std::_Exit(3);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
};

// One increment on device buffers: a single persistent kernel launch.
void run_increment(fe2_hrom_t h, const double* d_E, const NewtonCfg& cfg, const Outputs& O, cudaStream_t s) {
  check(h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
  IncArgs a{};
  a.M = h->model();
  a.D = h->points();
  a.O = O;
  a.cfg = cfg;
  a.dE = d_E;
  a.work = h->work;
  a.cnt = h->cnt;
  CK(cudaMemsetAsync(h->work, 0, sizeof(int), s));
  CK(cudaMemsetAsync(h->cnt, 0, sizeof(IncCounters), s));
  Watchdog wd(h->num_sms);
  a.trace = wd.dev;
  if (h->timing) CK(cudaEventRecord(h->ev[0], s));
  launch_any(h, a, h->num_sms, s);
  CK(cudaGetLastError());
  if (h->timing) CK(cudaEventRecord(h->ev[1], s));
  wd.wait(s, "k_increment");
  CK(cudaMemcpyAsync(h->h_cnt, h->cnt, sizeof(IncCounters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const IncCounters c = *h->h_cnt;
  h->stats.kernel_launches += 1;
  h->stats.increments += 1;
  h->stats.assemblies += static_cast<int64_t>(c.assemblies);
  h->stats.commits += static_cast<int64_t>(c.commits);
  h->stats.plastic_evals += static_cast<int64_t>(c.plastic_evals);
  if (h->timing) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    h->stats.kernel_ms += ms;
    h->stats.timed_launches += 1;
    h->stats.timed_assemblies += static_cast<int64_t>(c.assemblies);
    h->stats.timed_commits += static_cast<int64_t>(c.commits);
    h->stats.timed_plastic_evals += static_cast<int64_t>(c.plastic_evals);
    h->stats.timed_commit_plastic += static_cast<int64_t>(c.commit_plastic);
  }
}

}  // namespace

extern "C" {

const char* fe2_last_error(void) { return fe2::g_last_error.c_str(); }

const char* fe2_version(void) { return "fe2rom-b200 0.2 sm_100a"; }

int fe2_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int fe2_material_update_batch(int device, const fe2_material_t* mat, int64_t N, const double* eps,
                              const double* state_in, double* sigma, double* C, double* state_out,
                              uint8_t* plastic) {
  return guard([&] {
    check(mat && eps && sigma && C && N >= 0, Code::config, "bad arguments");
    const MatDev m = to_dev(*mat);
    require_device(device);
    if (N == 0) return;
    double *d_eps = dalloc<double>(N * 3), *d_in = state_in ? dalloc<double>(N * 6) : nullptr;
    double *d_sig = dalloc<double>(N * 3), *d_C = dalloc<double>(N * 9);
    double* d_out = state_out ? dalloc<double>(N * 6) : nullptr;
    uint8_t* d_pl = plastic ? dalloc<uint8_t>(N) : nullptr;
    int* d_err = dalloc<int>(1);
    CK(cudaMemset(d_err, 0, sizeof(int)));
    CK(cudaMemcpy(d_eps, eps, N * 3 * sizeof(double), cudaMemcpyHostToDevice));
    if (state_in) CK(cudaMemcpy(d_in, state_in, N * 6 * sizeof(double), cudaMemcpyHostToDevice));
    launch_material_batch(m, N, d_eps, d_in, d_sig, d_C, d_out, d_pl, d_err, nullptr);
    CK(cudaGetLastError());
    int err = 0;
    CK(cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    dfree(d_err);
    CK(cudaMemcpy(sigma, d_sig, N * 3 * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(C, d_C, N * 9 * sizeof(double), cudaMemcpyDeviceToHost));
    if (state_out) CK(cudaMemcpy(state_out, d_out, N * 6 * sizeof(double), cudaMemcpyDeviceToHost));
    if (plastic) CK(cudaMemcpy(plastic, d_pl, N, cudaMemcpyDeviceToHost));
    dfree(d_eps);
    dfree(d_in);
    dfree(d_sig);
    dfree(d_C);
    dfree(d_out);
    dfree(d_pl);
    check(err == 0, Code::material, m.kind == 2 ? "power-law return map did not converge"
                                                : "creep return map did not converge (or dt <= 0)");
  });
}

int fe2_material_update_soa_device(int device, const fe2_material_t* mat, int64_t N, const double* d_eps,
                                   const double* d_hist_in, double* d_sigma, double* d_C6, double* d_hist_out,
                                   uint8_t* d_plastic, void* stream) {
  return guard([&] {
    check(mat && d_eps && d_sigma && d_C6 && N >= 0, Code::config, "bad arguments");
    const MatDev m = to_dev(*mat);
    check(m.kind <= 1, Code::config, "the SoA device update supports elastic and J2 materials");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw Failure(Code::numeric, "no CUDA device available: the B200 engine has no CPU fallback");
    check(device >= 0 && device < count, Code::config, "device index out of range");
    CK(cudaSetDevice(device));
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    launch_material_soa(m, N, d_eps, d_hist_in, d_sigma, d_C6, d_hist_out, d_plastic, sms,
                        static_cast<cudaStream_t>(stream));
    CK(cudaGetLastError());
  });
}

int fe2_hrom_create(int device, int n, int K, const double* G, const double* w, const int* mat_id,
                    const fe2_material_t* mats, int n_mats, double volume, fe2_hrom_t* out) {
  return guard([&] {
    check(out != nullptr, Code::config, "null output handle");
    *out = nullptr;
    check(n >= 1 && K >= 1 && G && w && mat_id && mats && n_mats >= 1, Code::config, "bad model arguments");
    check(n <= 128, Code::config, "this build supports n <= 128 modes");
    check(volume > 0.0, Code::config, "RVE volume must be positive");
    std::vector<MatDev> md;  // any kind: J2 closed form, power law / creep by their return maps
    for (int i = 0; i < n_mats; ++i) md.push_back(to_dev(mats[i]));
    require_device(device);
    auto h = new fe2_hrom_s;
    try {
      h->device = device;
      CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
      h->n = n;
      // DMMA tiles of 8; the one-CTA-per-point path uses 16-point chunks above
      // 64 modes, whose mode split needs NP a multiple of 16
      h->NP = (n + 7) / 8 * 8;
      if (h->NP > 64) h->NP = (n + 15) / 16 * 16;
      // G2 record of a cubature point: rows G0 | G1 | G2 at g2_row_offset(NP, i)
      // then [w, 0] for the warp-per-point kernel (the three rows on distinct
      // bank groups); for the CTA-per-point kernel (NP > 32) each
      // strain row is padded to RG = NP + 4 doubles (≡ 4 or 12 mod 16), S =
      // 3 RG, so its DMMA A fragments read the rows of consecutive cubature
      // points conflict-free straight from the G chunk (weight in row 0's pad).
      const int RG = h->NP + 4;  // NP > 32
      h->S = h->NP > 32 ? 3 * RG : g2_row_offset(h->NP, 2) + h->NP + 2;
      h->K = K;
      h->volume = volume;
      h->G.assign(G, G + static_cast<size_t>(K) * 3 * n);
      h->w.assign(w, w + K);
      int j2_mat = -1;
      for (int q = 0; q < K; ++q) {
        check(mat_id[q] >= 0 && mat_id[q] < n_mats, Code::config, "cubature material id out of range");
        check(w[q] > 0.0, Code::config, "cubature weights must be positive");
        h->qmat.push_back(md[mat_id[q]]);
        if (md[mat_id[q]].kind >= 1) {  // history-carrying (J2, power law or creep)
          check(j2_mat < 0 || j2_mat == mat_id[q], Code::config,
                "this build supports one inelastic (J2 / power-law / creep) material per model");
          j2_mat = mat_id[q];
          h->j2_idx.push_back(q);
        } else {
          h->el_idx.push_back(q);
        }
      }
      h->mat2 = j2_mat >= 0 ? md[j2_mat] : make_mat(1, 1.0, 0.3, 1.0, 0.0);
      h->K2 = static_cast<int>(h->j2_idx.size());
      h->K2p = std::max(kQC, (h->K2 + kQC - 1) / kQC * kQC);
      const int NP = h->NP, S = h->S;
      std::vector<double> G2(static_cast<size_t>(h->K2p) * S, 0.0), w2(h->K2p, 0.0);
      for (int q2 = 0; q2 < h->K2; ++q2) {
        const int q = h->j2_idx[q2];
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < n; ++a)
            G2[static_cast<size_t>(q2) * S + (NP > 32 ? i * RG : g2_row_offset(NP, i)) + a] =
                G[(static_cast<size_t>(q) * 3 + i) * n + a];
        w2[q2] = w[q];
        // the weight also rides in a pad (row 0's for NP > 32, the record's last two doubles otherwise)
        G2[static_cast<size_t>(q2) * S + (NP > 32 ? NP : S - 2)] = w[q];
      }
      // elastic predictor over ALL cubature points (J2 points with the J2
      // material's C_e): K_e = Σ w G^T C_e G, K_aE,e = Σ w G^T C_e, C_EE,e = Σ w C_e.
      // The device adds only the plastic corrections ΔC_q of plastic points.
      std::vector<double> Ke(static_cast<size_t>(NP) * NP, 0.0), KaEe(static_cast<size_t>(NP) * 3, 0.0);
      for (int q = 0; q < K; ++q) {
        const MatDev& m = h->qmat[q];
        const double Ce[3][3] = {{m.lam + 2.0 * m.mu, m.lam, 0.0}, {m.lam, m.lam + 2.0 * m.mu, 0.0}, {0.0, 0.0, m.mu}};
        const double* Gq = G + static_cast<size_t>(q) * 3 * n;
        const double wq = w[q];
        double wC[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            wC[i][j] = wq * Ce[i][j];
            h->CEEe[3 * i + j] += wC[i][j];
          }
        for (int a = 0; a < n; ++a) {
          for (int j = 0; j < 3; ++j)
            KaEe[a * 3 + j] += Gq[a] * wC[0][j] + Gq[n + a] * wC[1][j] + Gq[2 * n + a] * wC[2][j];
          for (int b = 0; b < n; ++b) {
            double s = 0.0;
            for (int i = 0; i < 3; ++i)
              s += Gq[i * n + a] * (wC[i][0] * Gq[b] + wC[i][1] * Gq[n + b] + wC[i][2] * Gq[2 * n + b]);
            Ke[static_cast<size_t>(a) * NP + b] += s;
          }
        }
      }
      for (int a = 0; a < n; ++a)  // exact symmetry
        for (int b = 0; b < a; ++b) {
          const double v = 0.5 * (Ke[static_cast<size_t>(a) * NP + b] + Ke[static_cast<size_t>(b) * NP + a]);
          Ke[static_cast<size_t>(a) * NP + b] = Ke[static_cast<size_t>(b) * NP + a] = v;
        }
      // Cholesky factor of K_e in the kernel's packed-lower layout (row i at
      // i(i+1)/2): the device reuses it whenever an assembly has no plastic point.
      auto tri = [](int i) { return i * (i + 1) / 2; };
      std::vector<double> Le(static_cast<size_t>(tri(NP)), 0.0), LeInv(NP, 0.0);
      for (int j = 0; j < n; ++j) {
        double d = Ke[static_cast<size_t>(j) * NP + j];
        for (int k = 0; k < j; ++k) d -= Le[tri(j) + k] * Le[tri(j) + k];
        check(d > 0.0, Code::solver, "elastic reduced stiffness K_e is not positive definite");
        const double ljj = std::sqrt(d);
        Le[tri(j) + j] = ljj;
        LeInv[j] = 1.0 / ljj;
        for (int i = j + 1; i < n; ++i) {
          double s = Ke[static_cast<size_t>(i) * NP + j];
          for (int k = 0; k < j; ++k) s -= Le[tri(i) + k] * Le[tri(j) + k];
          Le[tri(i) + j] = s / ljj;
        }
      }
      h->Le = dalloc<double>(Le.size());
      h->LeInv = dalloc<double>(LeInv.size());
      CK(cudaMemcpy(h->Le, Le.data(), Le.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->LeInv, LeInv.data(), LeInv.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
      h->stream = h->own_stream;
      for (auto& e : h->ev) CK(cudaEventCreate(&e));
      h->G2 = dalloc<double>(G2.size());
      h->w2 = dalloc<double>(w2.size());
      h->Ke = dalloc<double>(Ke.size());
      h->KaEe = dalloc<double>(KaEe.size());
      h->work = dalloc<int>(1);
      h->cnt = dalloc<IncCounters>(1);
      CK(cudaMallocHost(&h->h_cnt, sizeof(IncCounters)));
      CK(cudaMemcpy(h->G2, G2.data(), G2.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->w2, w2.data(), w2.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->Ke, Ke.data(), Ke.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->KaEe, KaEe.data(), KaEe.size() * sizeof(double), cudaMemcpyHostToDevice));
      h->stats.n = n;
      h->stats.K = K;
      h->stats.K_j2 = h->K2;
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void fe2_hrom_destroy(fe2_hrom_t h) { delete h; }

int fe2_hrom_alloc_points(fe2_hrom_t h, int64_t P, int keep_flags) {
  return guard([&] {
    check(h != nullptr && P >= 1, Code::config, "bad arguments");
    check(P < (int64_t(1) << 31), Code::config, "at most 2^31-1 points per device");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamSynchronize(h->stream));
    h->free_points();
    h->hist = dalloc<double>(static_cast<size_t>(h->nbuf()) * P * h->K2p * 5);
    h->alpha_c = dalloc<double>(static_cast<size_t>(P) * h->NP);
    h->bp = dalloc<double>(static_cast<size_t>(P) * h->NP);
    h->E_c = dalloc<double>(P * h->ncomp());
    h->sp = dalloc<double>(P * 4);
    h->st = dalloc<PointState>(P);
    h->keep_flags = keep_flags != 0;
    if (h->keep_flags) h->flags = dalloc<uint8_t>(static_cast<size_t>(h->nbuf()) * P * h->K2p);
    h->dE = dalloc<double>(P * h->ncomp());
    h->o_sigma = dalloc<double>(P * h->ncomp());
    h->o_C = dalloc<double>(P * h->ntan());
    h->o_res = dalloc<double>(P);
    h->o_iters = dalloc<int>(P);
    h->o_status = dalloc<int>(P);
    h->o_pc = dalloc<int>(P);
    h->P = P;
    h->zero_points(h->stream);
    CK(cudaStreamSynchronize(h->stream));
    h->stats.points = P;
  });
}

int fe2_hrom_reset_points(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    CK(cudaSetDevice(h->device));
    h->zero_points(h->stream);
    h->mono_first = true;  // a pending monolithic iterate belongs to the discarded state
  });
}

int fe2_hrom_output_ptrs(fe2_hrom_t h, double** d_sigma, double** d_C, int** d_iters, int** d_pc, double** d_res,
                         int** d_status) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    if (d_sigma) *d_sigma = h->o_sigma;
    if (d_C) *d_C = h->o_C;
    if (d_iters) *d_iters = h->o_iters;
    if (d_pc) *d_pc = h->o_pc;
    if (d_res) *d_res = h->o_res;
    if (d_status) *d_status = h->o_status;
  });
}

int fe2_hrom_solve_increment_device(fe2_hrom_t h, const double* d_E, const fe2_newton_opts_t* opts, double* d_sigma,
                                    double* d_C, int* d_iters, int* d_pc, double* d_res, int* d_status,
                                    void* stream) {
  return guard([&] {
    check(h != nullptr && d_E != nullptr, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    Outputs O{d_sigma ? d_sigma : h->o_sigma, d_C ? d_C : h->o_C, d_res ? d_res : h->o_res,
              d_iters ? d_iters : h->o_iters, d_status ? d_status : h->o_status, d_pc ? d_pc : h->o_pc};
    run_increment(h, d_E, make_cfg(opts), O, stream ? static_cast<cudaStream_t>(stream) : h->stream);
  });
}

int fe2_hrom_mono_begin(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    check(h->kin == 0, Code::config, "the monolithic iteration needs a small-strain handle");
    check(h->mat2.kind <= 1, Code::config,
          "the monolithic iteration supports J2 / elastic models (power law / creep: fe2_hrom_solve_increment)");
    h->mono_first = true;
  });
}

namespace {
// One monolithic iteration of every point at the macro iterate d_E (device), outputs into O.
void mono_launch(fe2_hrom_t h, const double* d_E, const Outputs& O, cudaStream_t s) {
  check(h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
  check(h->kin == 0, Code::config, "the monolithic iteration needs a small-strain handle");
  check(h->mat2.kind <= 1, Code::config,
        "the monolithic iteration supports J2 / elastic models (power law / creep: fe2_hrom_solve_increment)");
  const int64_t P = h->P;
  if (!h->mono) {
    h->mono = dalloc<double>(static_cast<size_t>(P) * mono_stride(h->NP));
    CK(cudaMemsetAsync(h->mono, 0, static_cast<size_t>(P) * mono_stride(h->NP) * sizeof(double), s));
  }
  IncArgs a{};
  a.M = h->model();
  a.D = h->points();
  a.O = O;
  a.cfg = NewtonCfg{1e-8, 1, 0};
  a.dE = d_E;
  a.work = h->work;
  a.cnt = h->cnt;
  a.mono = h->mono;
  a.mono_first = h->mono_first ? 1 : 0;
  CK(cudaMemsetAsync(h->work, 0, sizeof(int), s));
  CK(cudaMemsetAsync(h->cnt, 0, sizeof(IncCounters), s));
  if (h->timing) CK(cudaEventRecord(h->ev[0], s));
  if (h->NP <= 32)
    launch_increment_mono(a, h->num_sms, s);
  else
    check(launch_increment_big_mono(a, h->num_sms, s), Code::config, "unsupported mode count");
  CK(cudaGetLastError());
  if (h->timing) {  // timing builds the stats synchronously (counters + events)
    CK(cudaEventRecord(h->ev[1], s));
    CK(cudaMemcpyAsync(h->h_cnt, h->cnt, sizeof(IncCounters), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    const IncCounters c = *h->h_cnt;
    h->stats.kernel_ms += ms;
    h->stats.timed_launches += 1;
    h->stats.timed_assemblies += static_cast<int64_t>(c.assemblies);
    h->stats.timed_plastic_evals += static_cast<int64_t>(c.plastic_evals);
  }
  h->stats.kernel_launches += 1;
  h->mono_first = false;
}
}  // namespace

int fe2_hrom_mono_iterate(fe2_hrom_t h, const double* E, double* sigma, double* C, double* rel_res,
                          int* plastic_count, int* status) {
  return guard([&] {
    check(h != nullptr && E != nullptr, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    CK(cudaSetDevice(h->device));
    const int64_t P = h->P;
    cudaStream_t s = h->stream;
    CK(cudaMemcpyAsync(h->dE, E, P * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    mono_launch(h, h->dE, Outputs{h->o_sigma, h->o_C, h->o_res, h->o_iters, h->o_status, h->o_pc}, s);
    if (sigma) CK(cudaMemcpyAsync(sigma, h->o_sigma, P * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (C) CK(cudaMemcpyAsync(C, h->o_C, P * 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (rel_res) CK(cudaMemcpyAsync(rel_res, h->o_res, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (plastic_count) CK(cudaMemcpyAsync(plastic_count, h->o_pc, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (status) CK(cudaMemcpyAsync(status, h->o_status, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int fe2_hrom_mono_iterate_device(fe2_hrom_t h, const double* d_E, double* d_sigma, double* d_C, double* d_rel_res,
                                 int* d_plastic_count, int* d_status, void* stream) {
  return guard([&] {
    check(h != nullptr && d_E != nullptr, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    mono_launch(h, d_E,
                Outputs{d_sigma ? d_sigma : h->o_sigma, d_C ? d_C : h->o_C, d_rel_res ? d_rel_res : h->o_res,
                        h->o_iters, d_status ? d_status : h->o_status, d_plastic_count ? d_plastic_count : h->o_pc},
                s);
  });
}

int fe2_hrom_mono_commit(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    check(h->mono != nullptr && !h->mono_first, Code::config, "fe2_hrom_mono_commit needs a monolithic iterate");
    CK(cudaSetDevice(h->device));
    launch_mono_commit(h->points(), h->NP, h->mono, h->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    h->mono_first = true;
  });
}

int fe2_hrom_solve_increment(fe2_hrom_t h, const double* E, const fe2_newton_opts_t* opts, double* sigma, double* C,
                             int* iters, int* plastic_count, double* res_norm, int* status) {
  return guard([&] {
    check(h != nullptr && E != nullptr, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    CK(cudaSetDevice(h->device));
    const NewtonCfg cfg = make_cfg(opts);
    const int64_t P = h->P;
    cudaStream_t s = h->stream;
    CK(cudaMemcpyAsync(h->dE, E, P * h->ncomp() * sizeof(double), cudaMemcpyHostToDevice, s));
    Outputs O{h->o_sigma, h->o_C, h->o_res, h->o_iters, h->o_status, h->o_pc};
    run_increment(h, h->dE, cfg, O, s);
    if (sigma) CK(cudaMemcpyAsync(sigma, h->o_sigma, P * h->ncomp() * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (C) CK(cudaMemcpyAsync(C, h->o_C, P * h->ntan() * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (iters) CK(cudaMemcpyAsync(iters, h->o_iters, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (plastic_count) CK(cudaMemcpyAsync(plastic_count, h->o_pc, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (res_norm) CK(cudaMemcpyAsync(res_norm, h->o_res, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (status) CK(cudaMemcpyAsync(status, h->o_status, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int fe2_hrom_solve_increment_async(fe2_hrom_t h, const double* E, const fe2_newton_opts_t* opts, double* sigma,
                                   double* C, int* iters, int* plastic_count, double* res_norm, int* status) {
  return guard([&] {
    check(h != nullptr && E != nullptr, Code::config, "bad arguments");
    check(h->P > 0, Code::config, "no points allocated (fe2_hrom_alloc_points)");
    CK(cudaSetDevice(h->device));
    const NewtonCfg cfg = make_cfg(opts);
    const int64_t P = h->P;
    const int nc = h->ncomp(), nt = h->ntan();
    cudaStream_t s = h->stream;
    if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    if (!h->cnt_async) {
      h->cnt_async = dalloc<IncCounters>(1);
      CK(cudaMemset(h->cnt_async, 0, sizeof(IncCounters)));
    }
    auto& b = h->abuf[h->acur];
    if (!b.dE) {
      b.dE = dalloc<double>(P * nc);
      b.sig = dalloc<double>(P * nc);
      b.C = dalloc<double>(P * nt);
      b.res = dalloc<double>(P);
      b.it = dalloc<int>(P);
      b.pc = dalloc<int>(P);
      b.st = dalloc<int>(P);
      CK(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&b.copied, cudaEventDisableTiming));
    }
    if (b.used) CK(cudaStreamWaitEvent(s, b.copied, 0));  // its previous outputs have left the device
    CK(cudaMemcpyAsync(b.dE, E, P * nc * sizeof(double), cudaMemcpyHostToDevice, s));
    IncArgs a{};
    a.M = h->model();
    a.D = h->points();
    a.O = Outputs{b.sig, b.C, b.res, b.it, b.st, b.pc};
    a.cfg = cfg;
    a.dE = b.dE;
    a.work = h->work;
    a.cnt = h->cnt_async;  // accumulates until fe2_hrom_wait
    CK(cudaMemsetAsync(h->work, 0, sizeof(int), s));
    launch_any(h, a, h->num_sms, s);
    CK(cudaGetLastError());
    CK(cudaEventRecord(b.done, s));
    // the outputs of this increment go to the host on the copy stream while the next one computes
    cudaStream_t c = h->copy_stream;
    CK(cudaStreamWaitEvent(c, b.done, 0));
    if (sigma) CK(cudaMemcpyAsync(sigma, b.sig, P * nc * sizeof(double), cudaMemcpyDeviceToHost, c));
    if (C) CK(cudaMemcpyAsync(C, b.C, P * nt * sizeof(double), cudaMemcpyDeviceToHost, c));
    if (iters) CK(cudaMemcpyAsync(iters, b.it, P * sizeof(int), cudaMemcpyDeviceToHost, c));
    if (plastic_count) CK(cudaMemcpyAsync(plastic_count, b.pc, P * sizeof(int), cudaMemcpyDeviceToHost, c));
    if (res_norm) CK(cudaMemcpyAsync(res_norm, b.res, P * sizeof(double), cudaMemcpyDeviceToHost, c));
    if (status) CK(cudaMemcpyAsync(status, b.st, P * sizeof(int), cudaMemcpyDeviceToHost, c));
    CK(cudaEventRecord(b.copied, c));
    b.used = true;
    h->acur ^= 1;
    h->async_pending += 1;
    h->stats.kernel_launches += 1;
    h->stats.increments += 1;
  });
}

int fe2_hrom_wait(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamSynchronize(h->stream));
    if (h->copy_stream) CK(cudaStreamSynchronize(h->copy_stream));
    if (h->async_pending > 0 && h->cnt_async) {
      IncCounters c{};
      CK(cudaMemcpy(&c, h->cnt_async, sizeof(IncCounters), cudaMemcpyDeviceToHost));
      CK(cudaMemset(h->cnt_async, 0, sizeof(IncCounters)));
      h->stats.assemblies += static_cast<int64_t>(c.assemblies);
      h->stats.commits += static_cast<int64_t>(c.commits);
      h->stats.plastic_evals += static_cast<int64_t>(c.plastic_evals);
      h->async_pending = 0;
    }
  });
}

int fe2_hrom_read_state(fe2_hrom_t h, double* alpha, double* state, uint8_t* flags) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    check(!flags || h->keep_flags, Code::config, "plastic flags were not kept (alloc_points keep_flags=0)");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamSynchronize(h->stream));
    const int64_t P = h->P;
    const int n = h->n, NP = h->NP, K = h->K, K2p = h->K2p;
    std::vector<double> ac(static_cast<size_t>(P) * NP);
    CK(cudaMemcpy(ac.data(), h->alpha_c, ac.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (alpha)
      for (int64_t p = 0; p < P; ++p)
        for (int a = 0; a < n; ++a) alpha[p * n + a] = ac[p * NP + a];
    // committed history buffer per point (double-buffered small-n kernel)
    std::vector<PointState> pst(static_cast<size_t>(P));
    CK(cudaMemcpy(pst.data(), h->st, pst.size() * sizeof(PointState), cudaMemcpyDeviceToHost));
    auto curbuf = [&](int64_t p) { return (h->nbuf() == 2 && pst[p].pad[0]) ? 1 : 0; };
    if (state) {
      std::vector<double> hs(static_cast<size_t>(h->nbuf()) * P * K2p * 5), Ec(static_cast<size_t>(P) * h->ncomp());
      CK(cudaMemcpy(hs.data(), h->hist, hs.size() * sizeof(double), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(Ec.data(), h->E_c, Ec.size() * sizeof(double), cudaMemcpyDeviceToHost));
      auto hidx = [&](int64_t p, int q2, int comp) {  // [buf][P][K2p/32][5][32]
        return static_cast<size_t>(curbuf(p)) * P * K2p * 5 +
               (static_cast<size_t>(p) * (K2p / kQC) + q2 / kQC) * (5 * kQC) + comp * kQC + q2 % kQC;
      };
      for (int64_t p = 0; p < P && h->kin == 1; ++p) {
        // finite strain: sigma33 of the Biot stress from the committed U - I and eps_p
        for (int q = 0; q < K; ++q) {
          double* s = state + (static_cast<size_t>(p) * K + q) * 6;
          for (int c = 0; c < 5; ++c) s[c] = 0.0;
        }
        for (int q2 = 0; q2 < h->K2; ++q2) {
          const int q = h->j2_idx[q2];
          double* s = state + (static_cast<size_t>(p) * K + q) * 6;
          for (int c = 0; c < 5; ++c) s[c] = hs[hidx(p, q2, c)];
        }
        for (int q = 0; q < K; ++q) {
          const Eps3 e = biot_strain_at(h, p, q, ac.data(), Ec.data());
          double* s = state + (static_cast<size_t>(p) * K + q) * 6;
          const MatDev& m = h->qmat[q];
          s[5] = m.lam * ((e.v[0] - s[0]) + (e.v[1] - s[1]) + (0.0 - s[2])) + 2.0 * m.mu * (0.0 - s[2]);
        }
      }
      for (int64_t p = 0; p < P && h->kin == 0; ++p) {
        // sigma33 is write-only in the reference (materials.hpp:181, :193): it is
        // not kept in HBM but recomputed here from the committed strain and eps_p,
        // sigma33 = lam tr(eps - eps_p) + 2 mu (0 - eps_p,33).
        for (int q = 0; q < K; ++q) {
          const Eps3 e = strain_at(h, p, q, ac.data(), Ec.data());
          double* s = state + (static_cast<size_t>(p) * K + q) * 6;
          for (int c = 0; c < 5; ++c) s[c] = 0.0;
          s[5] = h->qmat[q].lam * (e.v[0] + e.v[1]);
        }
        for (int q2 = 0; q2 < h->K2; ++q2) {
          const int q = h->j2_idx[q2];
          double* s = state + (static_cast<size_t>(p) * K + q) * 6;
          for (int c = 0; c < 5; ++c) s[c] = hs[hidx(p, q2, c)];
          const MatDev& m = h->mat2;
          const Eps3 e = strain_at(h, p, q, ac.data(), Ec.data());
          s[5] = m.lam * ((e.v[0] - s[0]) + (e.v[1] - s[1]) + (0.0 - s[2])) + 2.0 * m.mu * (0.0 - s[2]);
        }
      }
    }
    if (flags) {
      std::vector<uint8_t> fl(static_cast<size_t>(h->nbuf()) * P * K2p);
      CK(cudaMemcpy(fl.data(), h->flags, fl.size(), cudaMemcpyDeviceToHost));
      std::memset(flags, 0, static_cast<size_t>(P) * K);
      for (int64_t p = 0; p < P; ++p) {
        const size_t off = static_cast<size_t>(curbuf(p)) * P * K2p;
        for (int q2 = 0; q2 < h->K2; ++q2) flags[static_cast<size_t>(p) * K + h->j2_idx[q2]] = fl[off + p * K2p + q2];
      }
    }
  });
}

int fe2_hrom_assemble_point(fe2_hrom_t h, int64_t point, const double* alpha, const double* E, double* r,
                            double* Kaa, double* KaE, double* C_EE, double* S_raw) {
  return guard([&] {
    check(h != nullptr && h->P > 0 && point >= 0 && point < h->P, Code::config, "bad point");
    check(h->kin == 0, Code::config, "finite-strain handle: use fe2_hrom_fs_assemble_point");
    check(alpha && E && r && Kaa && KaE && C_EE && S_raw, Code::config, "null buffer");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const int n = h->n;
    const size_t dn = static_cast<size_t>(n) + n * n + 3 * n + 12;
    double* dbg = dalloc<double>(dn + n + 3);
    CK(cudaMemcpyAsync(dbg + dn, alpha, n * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dbg + dn + n, E, 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    IncArgs a{};
    a.M = h->model();
    a.D = h->points();
    a.O = Outputs{h->o_sigma, h->o_C, h->o_res, h->o_iters, h->o_status, h->o_pc};
    a.cfg = NewtonCfg{1e-8, 30, 4};
    a.work = h->work;
    a.dbg = dbg;
    a.dbg_alpha = dbg + dn;
    a.dbg_E = dbg + dn + n;
    a.dbg_point = point;
    Watchdog wd(h->num_sms);
    a.trace = wd.dev;
    launch_any(h, a, h->num_sms, s);
    h->stats.kernel_launches += 1;
    CK(cudaGetLastError());
    wd.wait(s, "k_increment (assembly dump)");
    std::vector<double> o(dn);
    CK(cudaMemcpyAsync(o.data(), dbg, dn * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(dbg);
    std::memcpy(r, o.data(), n * sizeof(double));
    std::memcpy(Kaa, o.data() + n, static_cast<size_t>(n) * n * sizeof(double));
    std::memcpy(KaE, o.data() + n + n * n, 3 * n * sizeof(double));
    std::memcpy(C_EE, o.data() + n + n * n + 3 * n, 9 * sizeof(double));
    std::memcpy(S_raw, o.data() + n + n * n + 3 * n + 9, 3 * sizeof(double));
  });
}

int fe2_hrom_snapshot(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    CK(cudaSetDevice(h->device));
    const auto parts = h->state_parts();
    size_t total = 0;
    for (const auto& pt : parts) total += (pt.bytes + 255) / 256 * 256;
    if (h->snap_bytes != total) {
      dfree(h->snap);
      h->snap = dalloc<unsigned char>(total);
      h->snap_bytes = total;
    }
    size_t off = 0;
    for (const auto& pt : parts) {
      CK(cudaMemcpyAsync(h->snap + off, pt.p, pt.bytes, cudaMemcpyDeviceToDevice, h->stream));
      off += (pt.bytes + 255) / 256 * 256;
    }
    CK(cudaStreamSynchronize(h->stream));
  });
}

int fe2_hrom_restore(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    check(h->snap != nullptr, Code::config, "no snapshot (fe2_hrom_snapshot)");
    CK(cudaSetDevice(h->device));
    size_t off = 0;
    for (const auto& pt : h->state_parts()) {
      CK(cudaMemcpyAsync(pt.p, h->snap + off, pt.bytes, cudaMemcpyDeviceToDevice, h->stream));
      off += (pt.bytes + 255) / 256 * 256;
    }
    CK(cudaStreamSynchronize(h->stream));
    h->mono_first = true;  // a pending monolithic iterate belongs to the replaced state
  });
}

int fe2_hrom_stats(fe2_hrom_t h, fe2_hrom_stats_t* out) {
  return guard([&] {
    check(h && out, Code::config, "bad arguments");
    *out = h->stats;
  });
}

int fe2_hrom_reset_stats(fe2_hrom_t h) {
  return guard([&] {
    check(h != nullptr, Code::config, "bad arguments");
    const fe2_hrom_stats_t keep = h->stats;
    h->stats = fe2_hrom_stats_t{};
    h->stats.points = keep.points;
    h->stats.n = keep.n;
    h->stats.K = keep.K;
    h->stats.K_j2 = keep.K_j2;
  });
}

namespace {
void ensure_layout(fe2_hrom_t h, void* comm) {
  if (!h->x_scratch) {
    h->x_scratch = dalloc<int64_t>(kMaxRanks);
    h->x_flags = dalloc<int>(2);
    CK(cudaMallocHost(&h->h_xflags, 2 * sizeof(int)));
  }
  if (h->xlayout.comm != comm || h->xlayout.P_local != h->P)
    exchange_layout(h->device, h->stream, comm, h->P, h->x_scratch, &h->xlayout);
}
}  // namespace

int fe2_hrom_gather_layout(fe2_hrom_t h, void* comm, int64_t* P_max, int64_t* counts) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    check(comm != nullptr, Code::config, "null NCCL communicator");
    CK(cudaSetDevice(h->device));
    h->xlayout.comm = nullptr;  // always re-exchange the counts here
    ensure_layout(h, comm);
    if (P_max) *P_max = h->xlayout.P_max;
    if (counts)
      for (int r = 0; r < h->xlayout.world; ++r) counts[r] = h->xlayout.counts[r];
  });
}

int fe2_hrom_gather(fe2_hrom_t h, void* comm, const double* d_sigma, const double* d_C, const double* d_res_norm,
                    const int* d_status, double res_tol, double* d_all, int* flags) {
  return guard([&] {
    check(h != nullptr && h->P > 0, Code::config, "no points allocated");
    check(comm != nullptr, Code::config, "null NCCL communicator");
    CK(cudaSetDevice(h->device));
    ensure_layout(h, comm);
    exchange_records(h->device, h->stream, h->xlayout, h->ncomp(), h->ntan(), d_sigma ? d_sigma : h->o_sigma,
                     d_C ? d_C : h->o_C, d_res_norm ? d_res_norm : h->o_res, d_status ? d_status : h->o_status,
                     res_tol, d_all, h->x_flags, h->h_xflags, flags);
  });
}

int fe2_hrom_set_stream(fe2_hrom_t h, void* stream) {
  return guard([&] {
    check(h != nullptr, Code::config, "bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamSynchronize(h->stream));
    h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  });
}

int fe2_hrom_set_timing(fe2_hrom_t h, int on) {
  return guard([&] {
    check(h != nullptr, Code::config, "bad arguments");
    h->timing = on != 0;
  });
}

int fe2_hrom_create_fs(int device, int n, int K, const double* G4, const double* w, const int* mat_id,
                       const fe2_material_t* mats, int n_mats, double volume, fe2_hrom_t* out) {
  return guard([&] {
    check(out != nullptr, Code::config, "null output handle");
    *out = nullptr;
    check(n >= 1 && K >= 1 && G4 && w && mat_id && mats && n_mats >= 1, Code::config, "bad model arguments");
    check(n <= 32, Code::config, "the finite-strain path supports n <= 32 modes");
    check(volume > 0.0, Code::config, "RVE volume must be positive");
    std::vector<MatDev> md;
    for (int i = 0; i < n_mats; ++i) {
      md.push_back(to_dev(mats[i]));
      require_engine_material(md.back());
    }
    require_device(device);
    auto h = new fe2_hrom_s;
    try {
      h->kin = 1;
      h->device = device;
      CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
      h->n = n;
      h->NP = (n + 7) / 8 * 8;
      h->S = 4 * (h->NP + 4) + 2;  // rows padded to NP + 4 (FsLayout: conflict-free A fragments)
      h->K = K;
      h->volume = volume;
      h->G.assign(G4, G4 + static_cast<size_t>(K) * 4 * n);
      h->w.assign(w, w + K);
      int j2_mat = -1, el_mat = -1;
      for (int q = 0; q < K; ++q) {
        check(mat_id[q] >= 0 && mat_id[q] < n_mats, Code::config, "cubature material id out of range");
        check(w[q] > 0.0, Code::config, "cubature weights must be positive");
        h->qmat.push_back(md[mat_id[q]]);
        if (md[mat_id[q]].kind == 1) {
          check(j2_mat < 0 || j2_mat == mat_id[q], Code::config, "this build supports one J2 material per model");
          j2_mat = mat_id[q];
          h->j2_idx.push_back(q);
        } else {
          check(el_mat < 0 || el_mat == mat_id[q], Code::config,
                "the finite-strain path supports one elastic material per model");
          el_mat = mat_id[q];
          h->el_idx.push_back(q);
        }
      }
      h->mat2 = j2_mat >= 0 ? md[j2_mat] : make_mat(1, 1.0, 0.3, 1.0, 0.0);
      h->matE = el_mat >= 0 ? md[el_mat] : make_mat(0, 1.0, 0.3, 0.0, 0.0);
      h->K2 = static_cast<int>(h->j2_idx.size());
      h->K2p = (h->K2 + kQC - 1) / kQC * kQC;
      h->Kel = static_cast<int>(h->el_idx.size());
      h->Kelp = (h->Kel + kQC - 1) / kQC * kQC;
      const int NP = h->NP, S = h->S;
      // rows [G4 row 0..3 (NP + 4 each) | w | 0]: J2 points (padded to K2p), then elastic points
      const int RG = NP + 4;
      std::vector<double> G2(static_cast<size_t>(h->K2p + h->Kelp) * S, 0.0);
      auto put = [&](int slot, int q) {
        for (int i = 0; i < 4; ++i)
          for (int a = 0; a < n; ++a)
            G2[static_cast<size_t>(slot) * S + i * RG + a] = G4[(static_cast<size_t>(q) * 4 + i) * n + a];
        G2[static_cast<size_t>(slot) * S + 4 * RG] = w[q];
      };
      for (int q2 = 0; q2 < h->K2; ++q2) put(q2, h->j2_idx[q2]);
      for (int e = 0; e < h->Kel; ++e) put(h->K2p + e, h->el_idx[e]);
      CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
      h->stream = h->own_stream;
      for (auto& e : h->ev) CK(cudaEventCreate(&e));
      h->G2 = dalloc<double>(G2.size());
      h->work = dalloc<int>(1);
      h->cnt = dalloc<IncCounters>(1);
      CK(cudaMallocHost(&h->h_cnt, sizeof(IncCounters)));
      CK(cudaMemcpy(h->G2, G2.data(), G2.size() * sizeof(double), cudaMemcpyHostToDevice));
      h->stats.n = n;
      h->stats.K = K;
      h->stats.K_j2 = h->K2;
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int fe2_hrom_kinematics(fe2_hrom_t h, int* kinematics) {
  return guard([&] {
    check(h != nullptr && kinematics != nullptr, Code::config, "bad arguments");
    *kinematics = h->kin;
  });
}

int fe2_hrom_fs_assemble_point(fe2_hrom_t h, int64_t point, const double* alpha, const double* H, double* r,
                               double* Kaa, double* KaF, double* KFa, double* C_FF, double* P_raw) {
  return guard([&] {
    check(h != nullptr && h->P > 0 && point >= 0 && point < h->P, Code::config, "bad point");
    check(h->kin == 1, Code::config, "small-strain handle: use fe2_hrom_assemble_point");
    check(alpha && H && r && Kaa && KaF && KFa && C_FF && P_raw, Code::config, "null buffer");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const int n = h->n;
    const size_t dn = static_cast<size_t>(n) + n * n + 8 * n + 20;
    double* dbg = dalloc<double>(dn + n + 4);
    CK(cudaMemcpyAsync(dbg + dn, alpha, n * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dbg + dn + n, H, 4 * sizeof(double), cudaMemcpyHostToDevice, s));
    IncArgs a{};
    a.M = h->model();
    a.D = h->points();
    a.O = Outputs{h->o_sigma, h->o_C, h->o_res, h->o_iters, h->o_status, h->o_pc};
    a.cfg = NewtonCfg{1e-8, 30, 4};
    a.work = h->work;
    a.dbg = dbg;
    a.dbg_alpha = dbg + dn;
    a.dbg_E = dbg + dn + n;
    a.dbg_point = point;
    Watchdog wd(h->num_sms);
    a.trace = wd.dev;
    launch_any(h, a, h->num_sms, s);
    h->stats.kernel_launches += 1;
    CK(cudaGetLastError());
    wd.wait(s, "k_increment_fs (assembly dump)");
    std::vector<double> o(dn);
    CK(cudaMemcpyAsync(o.data(), dbg, dn * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(dbg);
    const double* src = o.data();
    std::memcpy(r, src, n * sizeof(double));
    std::memcpy(Kaa, src + n, static_cast<size_t>(n) * n * sizeof(double));
    std::memcpy(KaF, src + n + n * n, 4 * n * sizeof(double));
    std::memcpy(KFa, src + n + n * n + 4 * n, 4 * n * sizeof(double));
    std::memcpy(C_FF, src + n + n * n + 8 * n, 16 * sizeof(double));
    std::memcpy(P_raw, src + n + n * n + 8 * n + 16, 4 * sizeof(double));
  });
}

}  // extern "C"
