// fma_peak.cu -- FP32 pipe microbenchmark on B200 (sm_100a): FFMA vs FFMA2 throughput.
// Used to derive the "alu" roofline denominator measured on the box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak tools/fma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 16;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) ffma_kernel(float* out, float a, float b) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  const float m = a + threadIdx.x * 1e-9f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fmaf(acc[c], m, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float a, float b) {
  float2 acc[kChains / 2];
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) acc[c] = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
  const float2 m = make_float2(a + threadIdx.x * 1e-9f, a);
  const float2 bb = make_float2(b, b);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) acc[c] = __ffma2_rn(acc[c], m, bb);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) s += acc[c].x + acc[c].y;
  if (s == 12345.678f) out[0] = s;
}

template <class K>
double run(K kern, const char* name, int blocks) {
  float* d;
  cudaMalloc(&d, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(d, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) kern<<<blocks, 256>>>(d, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fma = (double)blocks * 256 * kIters * kChains * reps;
  double tflops = 2 * fma / (ms * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", name, blocks,
         tflops, ms / reps);
  cudaFree(d);
  return tflops;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {8, 32}) {
    run(ffma_kernel, "ffma", sms * mult);
    run(ffma2_kernel, "ffma2", sms * mult);
  }
  return 0;
}
