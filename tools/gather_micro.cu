// Microbenchmark: random row gathers from an L2-resident table with cp.async (the K3-CT gather
// pattern), rows of 64 B (4 lanes x 16 B) vs 32 B (2 lanes x 16 B).  Each warp gathers stages of
// 256 rows into its own shared-memory ring, kStages commit groups in flight.  Reports rows/s and
// bytes/s over the whole GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather_micro tools/gather_micro.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>


template <int ROWB, int kStages, int kRowsPerStage>
__global__ void gather(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ idx,
                       int64_t nidx, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * kStages * kRowsPerStage * ROWB;
  constexpr int kLanesPerRow = ROWB / 16, kRowsPerInst = 32 / kLanesPerRow;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, nwt = (int64_t)gridDim.x * nw;
  int64_t pos = gw * 4096 % nidx;
  for (int it = 0; it < iters; ++it) {
    uint8_t* st = ring + (size_t)(it % kStages) * kRowsPerStage * ROWB;
    for (int j = 0; j < kRowsPerStage / kRowsPerInst; ++j) {
      const int r = j * kRowsPerInst + lane / kLanesPerRow, c = lane % kLanesPerRow;
      const uint32_t ix = __ldg(idx + (pos + r) % nidx);
      const uint8_t* src = tab + (size_t)ix * ROWB + c * 16;
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(st + r * ROWB + c * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
    pos = (pos + nwt * kRowsPerStage) % nidx;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (lane == 0) atomicAdd(sink, (unsigned long long)ring[lane]);
}

int main() {
  const int64_t nrows = 1 << 20;
  const int64_t nidx = 1 << 24;
  std::vector<uint32_t> h(nidx);
  std::mt19937 g(1);
  for (auto& v : h) v = g() % nrows;
  uint8_t* tab;
  uint32_t* idx;
  unsigned long long* sink;
  cudaMalloc(&tab, nrows * 64);
  cudaMemset(tab, 1, nrows * 64);
  cudaMalloc(&idx, nidx * 4);
  cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 200;
  auto run = [&](auto kern, int warps, int stages, int rps, int rowb) {
    const size_t smem = (size_t)warps * stages * rps * rowb;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int it2 = iters * 128 / rps;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<148, warps * 32, smem>>>(tab, idx, nidx, it2, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double rows = 148.0 * warps * it2 * rps;
      if (rep == 2)
        printf("warps %2d stages %2d rows/stage %3d row %2d B (smem %3zu KB): %.3f ms  %.2f Grows/s  %.2f TB/s  (%s)\n",
               warps, stages, rps, rowb, smem >> 10, ms, rows / ms / 1e6, rows * rowb / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(gather<64, 6, 128>, 4, 6, 128, 64);
  run(gather<64, 6, 64>, 8, 6, 64, 64);
  run(gather<64, 3, 64>, 16, 3, 64, 64);
  run(gather<64, 6, 32>, 16, 6, 32, 64);
  run(gather<64, 4, 32>, 24, 4, 32, 64);
  run(gather<64, 3, 32>, 32, 3, 32, 64);
  run(gather<32, 6, 32>, 32, 6, 32, 32);
  return 0;
}
