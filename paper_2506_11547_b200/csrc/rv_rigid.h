// rv_rigid.h -- launchers of the rigid-pose front end (rv_rigid.cu, NEXT-3).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace rv {

// CTAs of the pair kernels for n points (pairs i < j)
int64_t pairs_ctas(int64_t n);
// K9 pass 1: per-CTA kept counts (cta_cnt[pairs_ctas]) and their prefix (cta_off[+1], the
// total at cta_off[pairs_ctas])
void launch_pairs_count(const float* x, const float* y, int64_t n, double mu_t, int32_t* cta_cnt,
                        int64_t* cta_off, cudaStream_t s);
// K9 pass 2: the kept pairs in pair order (m, n fp32 [k][3]; ij int32 [k][2], may be null)
void launch_pairs_write(const float* x, const float* y, int64_t n, double mu_t,
                        const int64_t* cta_off, float* m_out, float* n_out, int32_t* ij_out,
                        cudaStream_t s);
// K10: translation vote with rotation R (row-major double[9]); acc: u32 [Bt^3], zero on entry
// and on return; bins: int64 [n] scratch; best: packed (count << 32 | ~lin), init 0; sums:
// double[3] of the winning bin's candidates, init 0
void launch_translation(const float* x, const float* y, int64_t n, const double* R, double lo,
                        double inv, int64_t Bt, uint32_t* acc, int64_t* bins,
                        unsigned long long* best, double* sums, cudaStream_t s);

}  // namespace rv
