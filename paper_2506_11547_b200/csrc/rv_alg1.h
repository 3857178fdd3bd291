// rv_alg1.h -- launcher of the paper's Algorithm 1 on the GPU (rv_alg1.cu, NEXT-4 baseline).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace rv {

// acc: DEVICE u32 [B^3], zeroed by the caller; cs / sn: DEVICE [J] cos / sin(alpha_j / 2);
// bad: DEVICE first row that cannot be normalised (init UINT64_MAX); best: DEVICE packed
// (count << 32 | ~lin) of the fullest bin (init 0).
void launch_alg1(const float* x, const float* y, int64_t n, int32_t B, int32_t J,
                 const double* cs, const double* sn, uint32_t* acc, unsigned long long* bad,
                 unsigned long long* best, cudaStream_t s);

}  // namespace rv
