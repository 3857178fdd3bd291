// rv_alg1.cu -- NEXT-4: the paper's own Algorithm 1 on the B200, as a same-box
// baseline for the exact certified vote.
//
// Every correspondence's quaternion circle q(alpha) = q_b1 cos(alpha/2) + q_b2 sin(alpha/2)
// is sampled at J angles alpha_j = -pi + 2 pi j / J; each sample is taken to the
// half sphere q3 <= 0, projected, binned on the B^3 grid of [-1, 1]^3 (Alg. 1 line 1)
// and adds one vote; the winner is the fullest bin (ties -> lowest lin) and its centre's
// rotation.  Readings R13-R15.
//
// Precision: the bin of a sample is an integer decided by floating point, so this kernel and
// the oracle (or_alg1_bins) take it in the same arithmetic: fp64, every operation explicitly
// rounded (__dmul_rn / __dadd_rn / __ddiv_rn / __dsqrt_rn: no FMA contraction) in the
// oracle's order, and cos / sin of alpha_j / 2 from a host-computed (libm) table.
//
// B200 mapping: one thread per correspondence, J samples in registers; consecutive samples
// of one circle that land in the same bin are merged into one atomicAdd (the count is the
// same); the 187 MB accumulator (B = 360) lives in HBM / L2.  The argmax is a grid-stride
// pass with a packed (count << 32 | ~lin) 64-bit atomicMax.
#include <cstdint>
#include <cuda_runtime.h>

#include "rv_alg1.h"

namespace rv {

namespace {

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
  c[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
  c[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}
// x / |x| (false: zero-length or non-finite)
__device__ __forceinline__ bool normalize3(const float* v, double* out) {
  const double a0 = v[0], a1 = v[1], a2 = v[2];
  const double na = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)),
                                         __dmul_rn(a2, a2)));
  if (!(na > 0.0) || !isfinite(na)) return false;
  out[0] = __ddiv_rn(a0, na);
  out[1] = __ddiv_rn(a1, na);
  out[2] = __ddiv_rn(a2, na);
  return true;
}

// q_b1, q_b2 of the circle of a -> b (R13: half-angle identities, perpendicular
// axis when a x b = 0)
__device__ void circle_basis(const double* a, const double* b, double* qb1, double* qb2) {
  double d = dot3(a, b);
  if (d > 1.0) d = 1.0;
  if (d < -1.0) d = -1.0;
  const double ch = __dsqrt_rn(__ddiv_rn(__dadd_rn(1.0, d), 2.0));
  const double sh = __dsqrt_rn(__ddiv_rn(__dsub_rn(1.0, d), 2.0));
  double c[3];
  cross3(a, b, c);
  double nc = __dsqrt_rn(dot3(c, c));
  if (nc == 0.0) {
    int k = 0;
    for (int t = 1; t < 3; ++t)
      if (fabs(a[t]) < fabs(a[k])) k = t;
    double e[3] = {0.0, 0.0, 0.0};
    e[k] = 1.0;
    cross3(a, e, c);
    nc = __dsqrt_rn(dot3(c, c));
  }
  qb1[0] = ch;
  for (int t = 0; t < 3; ++t) qb1[1 + t] = __dmul_rn(sh, __ddiv_rn(c[t], nc));
  const double* v = qb1 + 1;
  qb2[0] = -dot3(b, v);
  double bxv[3];
  cross3(b, v, bxv);
  for (int t = 0; t < 3; ++t) qb2[1 + t] = __dadd_rn(__dmul_rn(qb1[0], b[t]), bxv[t]);
}

}  // namespace

__global__ void __launch_bounds__(256) rv_alg1_vote_kernel(const float* __restrict__ x,
                                                           const float* __restrict__ y, int64_t n,
                                                           int32_t B, int32_t J,
                                                           const double* __restrict__ cs,
                                                           const double* __restrict__ sn,
                                                           uint32_t* acc,
                                                           unsigned long long* bad) {
  const double hb = (double)B / 2.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[3], b[3];
    if (!normalize3(x + 3 * i, a) || !normalize3(y + 3 * i, b)) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    double qb1[4], qb2[4];
    circle_basis(a, b, qb1, qb2);
    int64_t run_lin = -1;
    uint32_t run = 0;
    for (int32_t j = 0; j < J; ++j) {
      const double c = cs[j], s = sn[j];
      double q[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) q[t] = __dadd_rn(__dmul_rn(qb1[t], c), __dmul_rn(qb2[t], s));
      if (q[3] > 0.0) {
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] = -q[t];
      }
      const double den = __dsub_rn(1.0, q[3]);
      int64_t idx[3];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const double pt = __ddiv_rn(q[t], den);
        int64_t v = (int64_t)floor(__dmul_rn(__dadd_rn(pt, 1.0), hb));
        v = v < 0 ? 0 : (v > B - 1 ? B - 1 : v);
        idx[t] = v;
      }
      const int64_t lin = (idx[0] * B + idx[1]) * B + idx[2];
      if (lin == run_lin) {
        ++run;
      } else {
        if (run) atomicAdd(&acc[run_lin], run);
        run_lin = lin;
        run = 1;
      }
    }
    if (run) atomicAdd(&acc[run_lin], run);
  }
}

__global__ void __launch_bounds__(256) rv_alg1_argmax_kernel(const uint32_t* __restrict__ acc,
                                                             int64_t m,
                                                             unsigned long long* best) {
  unsigned long long k = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = ((unsigned long long)acc[e] << 32) |
                                 (unsigned long long)(0xffffffffu - (uint32_t)e);
    k = v > k ? v : k;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_down_sync(0xffffffffu, k, o);
    k = t > k ? t : k;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(best, k);
}

void launch_alg1(const float* x, const float* y, int64_t n, int32_t B, int32_t J,
                 const double* cs, const double* sn, uint32_t* acc, unsigned long long* bad,
                 unsigned long long* best, cudaStream_t s) {
  const int64_t m = (int64_t)B * B * B;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  rv_alg1_vote_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, y, n, B, J, cs, sn, acc, bad);
  rv_alg1_argmax_kernel<<<148 * 8, 256, 0, s>>>(acc, m, best);
}

}  // namespace rv
