// Host-side helpers shared by the C-ABI translation units (internal).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "common.hpp"
#include "fe2rom/fe2rom_gpu.h"
#include "material.cuh"

namespace fe2 {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure(Code::numeric, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class T>
inline T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  const cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();  // not sticky: clear it so later launch checks do not report it
    throw Failure(Code::numeric, std::string("device allocation of ") + std::to_string(count * sizeof(T)) +
                                     " bytes failed: " + cudaGetErrorString(e));
  }
  return static_cast<T*>(p);
}
template <class T>
inline void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

inline void require_device(int device) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Failure(Code::numeric, "no CUDA device available: the B200 engine has no CPU fallback");
  check(device >= 0 && device < count, Code::config, "device index out of range");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  check(prop.major == 10, Code::numeric, std::string("the engine is built for sm_100a (B200); found ") + prop.name);
  CK(cudaSetDevice(device));
}

inline MatDev to_dev(const fe2_material_t& m) {  // validate, materials.hpp:80-98
  check(m.kind >= 0 && m.kind <= 3, Code::config, "unsupported material kind");
  const double E = m.p[0], nu = m.p[1];
  check(E > 0.0 && nu >= 0.0 && nu < 0.5, Code::config, "invalid elastic parameters");
  if (m.kind == 1) check(m.p[2] > 0.0 && m.p[3] >= 0.0, Code::config, "invalid J2 parameters");
  if (m.kind == 2)
    check(m.p[2] > 0.0 && m.p[3] > 0.0 && m.p[3] < 1.0, Code::config, "invalid power-law parameters");
  if (m.kind == 3) check(m.p[2] > 0.0 && m.p[3] > 0.0 && m.p[4] > -1.0, Code::config, "invalid creep parameters");
  if (m.kind >= 2) return make_mat_general(m.kind, E, nu, m.p + 2);
  return make_mat(m.kind, E, nu, m.kind == 1 ? m.p[2] : 0.0, m.kind == 1 ? m.p[3] : 0.0);
}

// The finite-strain (Biot) engine carries closed-form J2 / elastic points only.
inline void require_engine_material(const MatDev& m) {
  check(m.kind <= 1, Code::config,
        "the finite-strain hyper-ROM engine supports elastic and J2 materials; power-law / creep run "
        "through the small-strain engine, fe2_material_update_batch and the HF solver");
}

// exchange.cu: the block layout over a communicator (every rank's point count; the
// gathered buffer holds world blocks of P_max rows), then per exchange: pack the per-point
// records {Σ | C | ‖r‖ | status} into this rank's block of d_all (padding rows status -1),
// NCCL all-gather in place, max-reduce {some point failed, some point above res_tol}.
constexpr int kMaxRanks = 64;
struct ExchangeLayout {
  void* comm = nullptr;
  int world = 0, rank = 0;
  int64_t P_local = 0, P_max = 0, P_total = 0;
  int64_t counts[kMaxRanks] = {};
};
void exchange_layout(int device, cudaStream_t stream, void* comm, int64_t P, int64_t* d_scratch, ExchangeLayout* out);
void exchange_records(int device, cudaStream_t stream, const ExchangeLayout& L, int nc, int nt,
                      const double* d_sigma, const double* d_C, const double* d_res, const int* d_status,
                      double res_tol, double* d_all, int* d_flags, int* h_flags, int* flags_host);

}  // namespace fe2
