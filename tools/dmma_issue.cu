// DMMA issue-rate probe (sm_100a): how fast ONE warp per SM sub-partition can
// drive the FP64 tensor pipe, with and without shared-memory fragment loads,
// and the dependent-chain latency of DMMA.m8n8k4. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_issue tools/dmma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// CH independent accumulators, constant operands
template <int CH>
__global__ void k_const(double* out, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 9 accumulators fed like contract2: per k-step 2 A + 8 B fragments from shared
// memory (lane-dependent addresses), next k-step's set loaded before the DMMAs
__global__ void k_loads(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[9][2];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c][0] = acc[c][1] = 0.0;
  double A0[2], B0[8], A1[2], B1[8];
  const double* base = sm + (lane & 3) * 68 + (lane >> 2);
#pragma unroll
  for (int t = 0; t < 2; ++t) A0[t] = base[t * 8];
#pragma unroll
  for (int t = 0; t < 8; ++t) B0[t] = base[1024 + t * 8];
  for (int i = 0; i < iters; i += 2) {
    const double* p1 = base + ((i + 1) & 7) * 272;
#pragma unroll
    for (int t = 0; t < 2; ++t) A1[t] = p1[t * 8];
#pragma unroll
    for (int t = 0; t < 8; ++t) B1[t] = p1[1024 + t * 8];
    dmma(acc[0][0], acc[0][1], A0[0], B0[0]);
#pragma unroll
    for (int t = 0; t < 8; ++t) dmma(acc[1 + t][0], acc[1 + t][1], A0[1], B0[t]);
    const double* p2 = base + ((i + 2) & 7) * 272;
#pragma unroll
    for (int t = 0; t < 2; ++t) A0[t] = p2[t * 8];
#pragma unroll
    for (int t = 0; t < 8; ++t) B0[t] = p2[1024 + t * 8];
    dmma(acc[0][0], acc[0][1], A1[0], B1[0]);
#pragma unroll
    for (int t = 0; t < 8; ++t) dmma(acc[1 + t][0], acc[1 + t][1], A1[1], B1[t]);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 9; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warps 0-3 drive DMMA (9 accumulators), warps 4-7 run DFMA chains of width CH
// (CH = 0: idle) on the same sub-partitions: DMMA throughput under FP64 traffic
template <int CH>
__global__ void k_roles(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp < 4) {
    double acc[9][2];
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 9; ++c) dmma(acc[c][0], acc[c][1], a, b);
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) s += acc[c][0] + acc[c][1];
  } else if (CH > 0) {
    double f[CH > 0 ? CH : 1];
#pragma unroll
    for (int c = 0; c < CH; ++c) f[c] = c;
    const double a = 0.999, b = 1e-3;
    for (int i = 0; i < iters * 9; ++i) {
#pragma unroll
      for (int c = 0; c < CH; ++c) f[c] = fma(f[c], a, b);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) s += f[c];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int iters = 8192;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int wps : {1, 2}) {  // warps per SM sub-partition
    const int threads = 128 * wps;
    float ms = timeit([&] { k_const<9><<<sms, threads>>>(out, iters); });
    double fl = 2.0 * 256 * 9 * iters * (double)sms * threads / 32;
    printf(", \"const9_wps%d_tflops\": %.2f", wps, fl / ms / 1e9);
    ms = timeit([&] { k_loads<<<sms, threads>>>(out, iters); });
    printf(", \"loads9_wps%d_tflops\": %.2f", wps, fl / ms / 1e9);
  }
  for (int ch : {1, 2, 4}) {
    const int threads = 128;
    float ms = 0;
    if (ch == 1) ms = timeit([&] { k_const<1><<<sms, threads>>>(out, iters); });
    if (ch == 2) ms = timeit([&] { k_const<2><<<sms, threads>>>(out, iters); });
    if (ch == 4) ms = timeit([&] { k_const<4><<<sms, threads>>>(out, iters); });
    // cycles per DMMA of one warp (one warp per sub-partition)
    const double cyc = ms * 1e-3 * clk * 1e3 / ((double)iters * ch);
    printf(", \"chain%d_cycles_per_dmma\": %.1f", ch, cyc);
  }
  {
    const double fl = 2.0 * 256 * 9 * iters * (double)sms * 4;
    float ms = timeit([&] { k_roles<0><<<sms, 256>>>(out, iters); });
    printf(", \"roles_dfma0_tflops\": %.2f", fl / ms / 1e9);
    ms = timeit([&] { k_roles<1><<<sms, 256>>>(out, iters); });
    printf(", \"roles_dfma1chain_tflops\": %.2f", fl / ms / 1e9);
    ms = timeit([&] { k_roles<4><<<sms, 256>>>(out, iters); });
    printf(", \"roles_dfma4chain_tflops\": %.2f", fl / ms / 1e9);
  }
  printf("}\n");
  return 0;
}
