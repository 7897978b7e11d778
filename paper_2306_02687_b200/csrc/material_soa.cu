// Batched constitutive update on structure-of-arrays device buffers — the
// HBM-bound form of update_material (materials.hpp:317-325) over a batch of
// material points (SURVEY §8(b) fe2_material_update_batch with SoA history).
//
// Per point: read ε (3) and the history εp (4), eq (5 x 8 B) = 64 B; write
// σ (3), the 6 unique entries of the symmetric C (materials.hpp:305-314
// condense_tangent), the new history εp, eq, σ33 (6) and the plastic flag
// = 121 B. Each thread owns two adjacent points: every array moves as 16-B
// vectors (coalesced 512-B warp transactions), with streaming cache hints
// (each byte is touched once). Grid: a multiple of the SM count, grid-stride.
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>

#include "hrom_kernels.cuh"

namespace fe2 {

namespace {

__device__ __forceinline__ double2 ld2(const double* p, int64_t i) { return __ldcs(reinterpret_cast<const double2*>(p + i)); }
__device__ __forceinline__ void st2(double* p, int64_t i, double a, double b) {
  __stcs(reinterpret_cast<double2*>(p + i), make_double2(a, b));
}

// Scalar variant: odd N or component arrays not 16-B aligned.
__global__ void __launch_bounds__(256) k_material_soa1(MatDev m, int64_t N, const double* __restrict__ eps,
                                                       const double* __restrict__ hin, double* __restrict__ sig,
                                                       double* __restrict__ C6, double* __restrict__ hout,
                                                       uint8_t* __restrict__ plastic) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
    double h[5] = {0, 0, 0, 0, 0};
    if (hin)
      for (int c = 0; c < 5; ++c) h[c] = __ldcs(hin + c * N + i);
    const MatOut a = update_material(m, h[0], h[1], h[2], h[3], h[4], __ldcs(eps + i), __ldcs(eps + N + i),
                                     __ldcs(eps + 2 * N + i));
    __stcs(sig + i, a.s0);
    __stcs(sig + N + i, a.s1);
    __stcs(sig + 2 * N + i, a.s2);
    const double c[6] = {a.c00, a.c01, a.c02, a.c11, a.c12, a.c22};
    for (int k = 0; k < 6; ++k) __stcs(C6 + k * N + i, c[k]);
    if (hout) {
      const double o[6] = {a.ep0, a.ep1, a.ep2, a.ep3, a.eq, a.s33};
      for (int k = 0; k < 6; ++k) __stcs(hout + k * N + i, o[k]);
    }
    if (plastic) plastic[i] = a.plastic ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256) k_material_soa(MatDev m, int64_t N, const double* __restrict__ eps,
                                                      const double* __restrict__ hin, double* __restrict__ sig,
                                                      double* __restrict__ C6, double* __restrict__ hout,
                                                      uint8_t* __restrict__ plastic) {
  const int64_t pairs = N / 2;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < pairs; t += stride) {
    const int64_t i = 2 * t;
    const double2 e0 = ld2(eps, i), e1 = ld2(eps, N + i), e2 = ld2(eps, 2 * N + i);
    double2 h0 = make_double2(0.0, 0.0), h1 = h0, h2 = h0, h3 = h0, h4 = h0;
    if (hin) {
      h0 = ld2(hin, i);
      h1 = ld2(hin, N + i);
      h2 = ld2(hin, 2 * N + i);
      h3 = ld2(hin, 3 * N + i);
      h4 = ld2(hin, 4 * N + i);
    }
    const MatOut a = update_material(m, h0.x, h1.x, h2.x, h3.x, h4.x, e0.x, e1.x, e2.x);
    const MatOut b = update_material(m, h0.y, h1.y, h2.y, h3.y, h4.y, e0.y, e1.y, e2.y);
    st2(sig, i, a.s0, b.s0);
    st2(sig, N + i, a.s1, b.s1);
    st2(sig, 2 * N + i, a.s2, b.s2);
    st2(C6, i, a.c00, b.c00);
    st2(C6, N + i, a.c01, b.c01);
    st2(C6, 2 * N + i, a.c02, b.c02);
    st2(C6, 3 * N + i, a.c11, b.c11);
    st2(C6, 4 * N + i, a.c12, b.c12);
    st2(C6, 5 * N + i, a.c22, b.c22);
    if (hout) {
      st2(hout, i, a.ep0, b.ep0);
      st2(hout, N + i, a.ep1, b.ep1);
      st2(hout, 2 * N + i, a.ep2, b.ep2);
      st2(hout, 3 * N + i, a.ep3, b.ep3);
      st2(hout, 4 * N + i, a.eq, b.eq);
      st2(hout, 5 * N + i, a.s33, b.s33);
    }
    if (plastic)
      *reinterpret_cast<uchar2*>(plastic + i) = make_uchar2(a.plastic ? 1 : 0, b.plastic ? 1 : 0);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

void launch_material_soa(const MatDev& m, int64_t N, const double* eps, const double* hin, double* sig, double* C6,
                         double* hout, uint8_t* plastic, int num_sms, cudaStream_t s) {
  if (N <= 0) return;
  static const int threads = [] {
    const char* e = std::getenv("FE2_SOA_THREADS");
    const int v = e ? std::atoi(e) : 256;
    return (v == 64 || v == 128 || v == 256) ? v : 256;
  }();
  static const int gridmul = [] {
    const char* e = std::getenv("FE2_SOA_GRIDMUL");
    const int v = e ? std::atoi(e) : 128;
    return v >= 1 && v <= 4096 ? v : 128;
  }();
  const bool vec = (N % 2 == 0) && aligned16(eps) && (!hin || aligned16(hin)) && aligned16(sig) && aligned16(C6) &&
                   (!hout || aligned16(hout)) && (!plastic || (reinterpret_cast<uintptr_t>(plastic) & 1u) == 0);
  const int64_t work = vec ? N / 2 : N;
  int64_t grid = static_cast<int64_t>(num_sms) * gridmul;  // CTAs per SM in the grid (grid-stride). Measured on 2^25 points: 8 -> 0.87, 32 -> 0.95,
  // 128 -> 0.98 of the HBM copy peak, 512+ (one pair per thread) -> 0.93 (FE2_SOA_GRIDMUL / FE2_SOA_THREADS: tuning)
  const int64_t need = (work + threads - 1) / threads;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  if (vec)
    k_material_soa<<<static_cast<unsigned>(grid), threads, 0, s>>>(m, N, eps, hin, sig, C6, hout, plastic);
  else
    k_material_soa1<<<static_cast<unsigned>(grid), threads, 0, s>>>(m, N, eps, hin, sig, C6, hout, plastic);
}

}  // namespace fe2
