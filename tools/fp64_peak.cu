// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64),
// DFMA, and a mix of both, to establish the roofline denominators the
// hyper-ROM assembly is measured against (BASELINE.md §2 "not yet measured").
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters) {
  double acc[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters) {
  double acc[CH];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[threadIdx.x] = s;
}

// one DMMA + R DFMA per inner step: do the two pipes overlap?
template <int CH, int R>
__global__ void k_mix(double* out, int iters) {
  double acc[CH][2], f[CH * R];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
  for (int c = 0; c < CH * R; ++c) f[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      dmma(acc[c][0], acc[c][1], a, b);
#pragma unroll
      for (int r = 0; r < R; ++r) f[c * R + r] = fma(f[c * R + r], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int c = 0; c < CH * R; ++c) s += f[c];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  const int iters = 4096;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int wpb : {4, 8, 16}) {
    const int threads = 32 * wpb, blocks = sms * 2;
    float ms = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * wpb;
    printf(", \"dmma_tflops_w%d\": %.2f", wpb, flops / ms / 1e9);
    ms = timeit([&] { k_dfma<8><<<blocks, threads>>>(out, iters); });
    flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_tflops_w%d\": %.2f", wpb, flops / ms / 1e9);
  }
  {
    const int threads = 32 * 8, blocks = sms * 2;
    float ms = timeit([&] { k_mix<4, 4><<<blocks, threads>>>(out, iters); });
    double dm = 2.0 * 256.0 * 4 * iters * (double)blocks * 8;
    double df = 2.0 * 16 * iters * (double)blocks * threads;
    printf(", \"mix_1dmma_4dfma_ms\": %.4f, \"mix_dmma_part_tflops\": %.2f, \"mix_dfma_part_tflops\": %.2f",
           ms, dm / ms / 1e9, df / ms / 1e9);
    ms = timeit([&] { k_mix<4, 8><<<blocks, threads>>>(out, iters); });
    dm = 2.0 * 256.0 * 4 * iters * (double)blocks * 8;
    df = 2.0 * 32 * iters * (double)blocks * threads;
    printf(", \"mix_1dmma_8dfma_ms\": %.4f, \"mix8_dmma_part_tflops\": %.2f, \"mix8_dfma_part_tflops\": %.2f",
           ms, dm / ms / 1e9, df / ms / 1e9);
    ms = timeit([&] { k_dmma<4><<<blocks, threads>>>(out, iters); });
    printf(", \"dmma4_alone_ms\": %.4f", ms);
  }
  printf("}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
