// rv_rigid.cu -- NEXT-3: the rigid-pose front end of the paper.
//
//  K9  pairs: every i < j (lexicographic) gives m = x_i - x_j, n = y_i - y_j (fp64, exact for
//      fp32 inputs), kept iff both are non-zero and |‖m‖ - ‖n‖| <= mu_t (the rotation-invariant
//      length check).  Kept pairs are written in pair order (count per CTA, one-CTA
//      scan, ordered write with warp ballots), as fp32 -- the rotation vote's input format --
//      so the list is deterministic and equals the oracle's (or_rigid_pairs) exactly: the keep
//      decision is an integer decided by floating point, taken here in the oracle's fp64
//      arithmetic with every operation explicitly rounded.
//  K10 translation vote: t_i = y_i - R(q) x_i (fp64, same rounding discipline) is
//      binned on [lo, hi)^3 at `step` ([-5,5]^3 at 0.025, 400^3 bins); the fullest bin
//      (ties -> lowest lin) is found by a packed atomicMax over the touched bins only, its
//      candidates' mean is summed, and the touched bins are cleared again, so the 256 MB
//      accumulator is zeroed once per context, not per call.
#include <cstdint>
#include <cuda_runtime.h>

#include "rv_rigid.h"

namespace rv {

namespace {

constexpr int kPairThreads = 256;
constexpr int kPairRounds = 16;  // pairs per CTA = 4096

// pairs before row i of the strict upper triangle of an n x n matrix
__device__ __forceinline__ int64_t row_off(int64_t i, int64_t n) { return i * n - i * (i + 1) / 2; }

// (i, j) of the k-th pair (lexicographic)
__device__ __forceinline__ void pair_of(int64_t k, int64_t n, int64_t* pi, int64_t* pj) {
  int64_t lo = 0, hi = n - 1;  // last i with row_off(i) <= k
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_off(mid, n) <= k) lo = mid; else hi = mid;
  }
  *pi = lo;
  *pj = lo + 1 + (k - row_off(lo, n));
}

__device__ __forceinline__ bool keep_pair(const float* __restrict__ x, const float* __restrict__ y,
                                          int64_t i, int64_t j, double mu_t, double* m,
                                          double* d) {
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    m[t] = __dsub_rn((double)x[3 * i + t], (double)x[3 * j + t]);
    d[t] = __dsub_rn((double)y[3 * i + t], (double)y[3 * j + t]);
  }
  const double lm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[0], m[0]), __dmul_rn(m[1], m[1])),
                                         __dmul_rn(m[2], m[2])));
  const double ld = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                         __dmul_rn(d[2], d[2])));
  return lm > 0.0 && ld > 0.0 && fabs(__dsub_rn(lm, ld)) <= mu_t;
}

}  // namespace

__global__ void __launch_bounds__(kPairThreads) rv_pairs_count(const float* __restrict__ x,
                                                               const float* __restrict__ y,
                                                               int64_t n, double mu_t,
                                                               int32_t* cta_cnt) {
  const int64_t total = n * (n - 1) / 2;
  const int64_t k0 = (int64_t)blockIdx.x * kPairThreads * kPairRounds;
  int c = 0;
  for (int r = 0; r < kPairRounds; ++r) {
    const int64_t k = k0 + (int64_t)r * kPairThreads + threadIdx.x;
    if (k >= total) break;
    int64_t i, j;
    pair_of(k, n, &i, &j);
    double m[3], d[3];
    c += keep_pair(x, y, i, j, mu_t, m, d) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  __shared__ int ws[kPairThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kPairThreads / 32; ++w) t += ws[w];
    cta_cnt[blockIdx.x] = t;
  }
}

// exclusive prefix of the CTA counts (one CTA); off[nb] = total
__global__ void __launch_bounds__(1024) rv_pairs_scan(const int32_t* __restrict__ cnt, int64_t nb,
                                                      int64_t* off) {
  __shared__ int64_t sh[1024];
  const int t = threadIdx.x;
  const int64_t i0 = nb * t / 1024, i1 = nb * (t + 1) / 1024;
  int64_t s = 0;
  for (int64_t i = i0; i < i1; ++i) s += cnt[i];
  sh[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += v;
    __syncthreads();
  }
  int64_t e = sh[t] - s;
  for (int64_t i = i0; i < i1; ++i) {
    off[i] = e;
    e += cnt[i];
  }
  if (t == 1023) off[nb] = sh[1023];
}

__global__ void __launch_bounds__(kPairThreads) rv_pairs_write(const float* __restrict__ x,
                                                               const float* __restrict__ y,
                                                               int64_t n, double mu_t,
                                                               const int64_t* __restrict__ off,
                                                               float* m_out, float* n_out,
                                                               int32_t* ij_out) {
  const int64_t total = n * (n - 1) / 2;
  const int64_t k0 = (int64_t)blockIdx.x * kPairThreads * kPairRounds;
  __shared__ int ws[kPairThreads / 32];
  int64_t base = off[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < kPairRounds; ++r) {
    const int64_t k = k0 + (int64_t)r * kPairThreads + threadIdx.x;
    bool keep = false;
    int64_t i = 0, j = 0;
    double m[3], d[3];
    if (k < total) {
      pair_of(k, n, &i, &j);
      keep = keep_pair(x, y, i, j, mu_t, m, d);
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) ws[warp] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < kPairThreads / 32; ++w) {
      if (w < warp) before += ws[w];
      tot += ws[w];
    }
    __syncthreads();
    if (keep) {
      const int64_t pos = base + before + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        m_out[3 * pos + t] = __double2float_rn(m[t]);
        n_out[3 * pos + t] = __double2float_rn(d[t]);
      }
      if (ij_out) {
        ij_out[2 * pos] = (int32_t)i;
        ij_out[2 * pos + 1] = (int32_t)j;
      }
    }
    base += tot;
  }
}

// ---- K10 translation vote ------------------------------------------------------------------
struct TransArgs {
  double R[9];
  double lo, inv;
  int64_t Bt;
};

__device__ __forceinline__ int64_t trans_bin(const float* __restrict__ x,
                                             const float* __restrict__ y, int64_t i,
                                             const TransArgs& A, double* t) {
  const double a[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  int64_t idx[3];
  bool ok = true;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double ra = __dadd_rn(__dadd_rn(__dmul_rn(A.R[3 * r], a[0]), __dmul_rn(A.R[3 * r + 1], a[1])),
                                __dmul_rn(A.R[3 * r + 2], a[2]));
    t[r] = __dsub_rn((double)y[3 * i + r], ra);
    const double f = floor(__dmul_rn(__dsub_rn(t[r], A.lo), A.inv));
    if (!(f >= 0.0) || !(f < (double)A.Bt)) ok = false;
    idx[r] = ok ? (int64_t)f : 0;
  }
  return ok ? (idx[0] * A.Bt + idx[1]) * A.Bt + idx[2] : -1;
}

__global__ void rv_trans_vote(const float* __restrict__ x, const float* __restrict__ y, int64_t n,
                              TransArgs A, uint32_t* acc, int64_t* bins) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t[3];
    const int64_t b = trans_bin(x, y, i, A, t);
    bins[i] = b;
    if (b >= 0) atomicAdd(&acc[b], 1u);
  }
}

__global__ void rv_trans_max(const int64_t* __restrict__ bins, int64_t n,
                             const uint32_t* __restrict__ acc, unsigned long long* best) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = bins[i];
    if (b < 0) continue;
    atomicMax(best, ((unsigned long long)acc[b] << 32) |
                        (unsigned long long)(0xffffffffu - (uint32_t)b));
  }
}

__global__ void rv_trans_sum(const float* __restrict__ x, const float* __restrict__ y, int64_t n,
                             TransArgs A, const int64_t* __restrict__ bins,
                             const unsigned long long* __restrict__ best, uint32_t* acc,
                             double* sums) {
  const int64_t win = (int64_t)(0xffffffffu - (uint32_t)(*best & 0xffffffffu));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = bins[i];
    if (b < 0) continue;
    if (b == win) {
      double t[3];
      trans_bin(x, y, i, A, t);
      atomicAdd(&sums[0], t[0]);
      atomicAdd(&sums[1], t[1]);
      atomicAdd(&sums[2], t[2]);
    }
  }
}

__global__ void rv_trans_clear(const int64_t* __restrict__ bins, int64_t n, uint32_t* acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (bins[i] >= 0) acc[bins[i]] = 0u;
}

// ---- launchers -----------------------------------------------------------------------------
int64_t pairs_ctas(int64_t n) {
  const int64_t total = n * (n - 1) / 2;
  return (total + (int64_t)kPairThreads * kPairRounds - 1) / ((int64_t)kPairThreads * kPairRounds);
}

void launch_pairs_count(const float* x, const float* y, int64_t n, double mu_t, int32_t* cta_cnt,
                        int64_t* cta_off, cudaStream_t s) {
  const int64_t nb = pairs_ctas(n);
  if (nb > 0) rv_pairs_count<<<(unsigned)nb, kPairThreads, 0, s>>>(x, y, n, mu_t, cta_cnt);
  rv_pairs_scan<<<1, 1024, 0, s>>>(cta_cnt, nb, cta_off);
}

void launch_pairs_write(const float* x, const float* y, int64_t n, double mu_t,
                        const int64_t* cta_off, float* m_out, float* n_out, int32_t* ij_out,
                        cudaStream_t s) {
  const int64_t nb = pairs_ctas(n);
  if (nb > 0)
    rv_pairs_write<<<(unsigned)nb, kPairThreads, 0, s>>>(x, y, n, mu_t, cta_off, m_out, n_out,
                                                         ij_out);
}

void launch_translation(const float* x, const float* y, int64_t n, const double* R, double lo,
                        double inv, int64_t Bt, uint32_t* acc, int64_t* bins,
                        unsigned long long* best, double* sums, cudaStream_t s) {
  TransArgs A;
  for (int e = 0; e < 9; ++e) A.R[e] = R[e];
  A.lo = lo;
  A.inv = inv;
  A.Bt = Bt;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  rv_trans_vote<<<(unsigned)blocks, 256, 0, s>>>(x, y, n, A, acc, bins);
  rv_trans_max<<<(unsigned)blocks, 256, 0, s>>>(bins, n, acc, best);
  rv_trans_sum<<<(unsigned)blocks, 256, 0, s>>>(x, y, n, A, bins, best, acc, sums);
  rv_trans_clear<<<(unsigned)blocks, 256, 0, s>>>(bins, n, acc);
}

}  // namespace rv
