// vote_micro.cu -- isolates the K3 inner loop (no TMA, no epilogue) to find where FP32-pipe
// cycles go.  Variants (template flags):
//   LDS    : k values re-read from shared memory every iteration (as K3) vs kept in registers
//   COUNT  : sign-bit counting (LEA.HI) after each chain vs a plain float accumulation
//   CPT    : cells per thread
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o vote_micro tools/vote_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kTile = 256;

__device__ __forceinline__ void add_sign(unsigned& acc, float v) {
  asm("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(__float_as_uint(v) >> 31));
}

template <int CPT, bool LDS, bool COUNT>
__global__ void __launch_bounds__(256, 2) loop_kernel(float* out, int reps) {
  __shared__ __align__(16) float sK[9][kTile];
  for (int e = threadIdx.x; e < 9 * kTile; e += blockDim.x)
    (&sK[0][0])[e] = 1e-3f * (float)((e * 7919) % 1000) - 0.5f;
  __syncthreads();
  float phi[CPT][9], init[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    init[c] = -0.3f - 0.01f * c - threadIdx.x * 1e-6f;
#pragma unroll
    for (int j = 0; j < 9; ++j) phi[c][j] = 0.1f * (j + 1) + 0.001f * c + threadIdx.x * 1e-7f;
  }
  unsigned neg[CPT];
  float facc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) { neg[c] = 0; facc[c] = 0.f; }
  float4 kr[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) kr[j] = *reinterpret_cast<const float4*>(&sK[j][4 * (threadIdx.x & 7)]);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int i = 0; i < kTile; i += 4) {
      float4 kk[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        if (LDS) kk[j] = *reinterpret_cast<const float4*>(&sK[j][i]);
        else { kk[j] = kr[j]; kr[j].x += 1e-7f; }
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        float2 lo = make_float2(init[c], init[c]), hi = lo;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          const float2 f2 = make_float2(phi[c][j], phi[c][j]);
          lo = __ffma2_rn(f2, make_float2(kk[j].x, kk[j].y), lo);
          hi = __ffma2_rn(f2, make_float2(kk[j].z, kk[j].w), hi);
        }
        if (COUNT) {
          add_sign(neg[c], lo.x); add_sign(neg[c], lo.y);
          add_sign(neg[c], hi.x); add_sign(neg[c], hi.y);
        } else {
          facc[c] += lo.x + lo.y + hi.x + hi.y;
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CPT; ++c) s += (float)neg[c] + facc[c];
  if (s == 1234.5f) out[0] = s;
}

template <int CPT, bool LDS, bool COUNT>
void run(const char* name, int sms) {
  float* d;
  cudaMalloc(&d, 4);
  const int reps = 64, blocks = sms * 2 * 8;
  loop_kernel<CPT, LDS, COUNT><<<blocks, 256>>>(d, 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop_kernel<CPT, LDS, COUNT><<<blocks, 256>>>(d, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double pairs = (double)blocks * 256 * reps * kTile * CPT;
  printf("{\"variant\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"err\": \"%s\"}\n", name,
         pairs * 18 / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, true, true>("cpt4 lds count (K3)", sms);
  run<4, false, true>("cpt4 regs count", sms);
  run<4, true, false>("cpt4 lds nocount", sms);
  run<4, false, false>("cpt4 regs nocount", sms);
  run<2, true, true>("cpt2 lds count", sms);
  run<6, true, true>("cpt6 lds count", sms);
  run<8, true, true>("cpt8 lds count", sms);
  return 0;
}
