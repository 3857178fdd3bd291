// Microbenchmark: latency of tcgen05.commit -> mbarrier completion as seen by (a) the committing
// thread and (b) another warp waiting on the barrier, with and without a preceding MMA, and the
// mbarrier arrive -> try_wait wake latency between two warps.  One CTA, clock64 deltas.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/commit_lat tools/commit_lat.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2506_11547_b200/csrc/rv_tc_ptx.h"
using namespace rv::tcx;

__global__ void k(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t a[128 * 64];
  __shared__ __align__(1024) uint8_t b[256 * 64];
  __shared__ uint64_t bar0, bar1, bar2, bar3;
  __shared__ uint32_t tbase;
  __shared__ long long t_commit, t_seen;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) a[i] = 0;
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) b[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { bar_init(&bar0, 1); bar_init(&bar1, 1); bar_init(&bar2, 1); bar_init(&bar3, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  long long s_self = 0, s_mma = 0, s_other = 0, s_wake = 0, s_issue = 0, s_issue4 = 0, s_mma4 = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t par = it & 1;
    // (a) commit with nothing pending, waited by the committing thread
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      mma_commit(&bar0);
      bar_wait(&bar0, par);
      s_self += clock64() - t0;
      // (b) one M128 N256 K16 MMA then commit, waited by the issuing thread
      t0 = clock64();
      mma_f16_i(tmem, smem_desc(su32(a), 128, 512), smem_desc(su32(b), 128, 512), idesc_f16(256), 0);
      mma_f16_i(tmem, smem_desc(su32(a) + 256, 128, 512), smem_desc(su32(b) + 256, 128, 512), idesc_f16(256), 1);
      const long long t1 = clock64();
      mma_commit(&bar1);
      bar_wait(&bar1, par);
      s_mma += clock64() - t0;
      s_issue += t1 - t0;
      // (b2) the same as four back-to-back stages (8 MMAs, one commit each), issue and drain
      t0 = clock64();
      for (int q = 0; q < 4; ++q) {
        mma_f16_i(tmem + (q & 1) * 256, smem_desc(su32(a), 128, 512), smem_desc(su32(b), 128, 512), idesc_f16(256), 0);
        mma_f16_i(tmem + (q & 1) * 256, smem_desc(su32(a) + 256, 128, 512), smem_desc(su32(b) + 256, 128, 512), idesc_f16(256), 1);
        mma_commit(&bar3);
      }
      const long long t2 = clock64();
      bar_wait(&bar3, par);  // bar3 counts 4 commits per phase
      s_issue4 += t2 - t0;
      s_mma4 += clock64() - t0;
    }
    __syncthreads();
    // (c) commit by thread 0, seen by warp 1 (wake after completion); (d) plain arrive -> warp 1
    if (threadIdx.x == 0) { t_commit = clock64(); mma_commit(&bar2); }
    if (warp == 1) {
      bar_wait(&bar2, par);
      if (lane == 0) s_other += clock64() - *(volatile long long*)&t_commit;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = s_self / iters; out[1] = s_mma / iters; out[3] = s_issue / iters; out[4] = s_issue4 / iters; out[5] = s_mma4 / iters; }
  if (threadIdx.x == 32) out[2] = s_other / iters;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)); }
}

int main() {
  long long* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  k<<<1, 64>>>(d, 2000);
  long long h[8] = {0};
  cudaError_t e = cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("err=%s commit(nothing pending)->own wait: %lld clk; 2 MMA(M128 N256 K16)+commit->own wait: %lld clk; commit->other warp wake: %lld clk\n",
         cudaGetErrorString(e), h[0], h[1], h[2]);
  printf("issue of 2 MMAs: %lld clk; 4 stages (8 MMAs + 4 commits): issue %lld clk, issue+drain %lld clk\n", h[3], h[4], h[5]);
  return 0;
}
