// rv_dive.cuh -- the dive's device steps (the host planner's rules, rv_plan.cpp), shared by the
// per-level loop's kernels (rv_dplan.cu) and the one-pass solve's fused dive-level planner
// (rv_cull.cu): the 27-neighbourhood of a pick, the ordered children of a neighbourhood, and the
// pick itself (max excess UB - n (1 - t) / 2, blocks away from NEXT-2's exclusion balls first,
// centres inside the ball first, ties -> lowest lin).  Every function is CTA-wide (any blockDim
// that is a multiple of 32, <= 1024).
#pragma once
#include <cstdint>

#include "rv_geom.h"

namespace rv {

// the 27-neighbourhood of (i,j,k) at resolution B, candidates only, ascending lin: the offsets
// (a,b,c) in lexicographic order give ascending lin
__device__ __forceinline__ int dive_neighbourhood(int32_t B, uint32_t lin, uint32_t out[27]) {
  int32_t i, j, k;
  lin_to_ijk(lin, B, i, j, k);
  int m = 0;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b)
      for (int c = -1; c <= 1; ++c) {
        const int32_t ni = i + a, nj = j + b, nk = k + c;
        if (ni < 0 || nj < 0 || nk < 0 || ni >= B || nj >= B || nk >= B) continue;
        if (is_candidate(B, ni, nj, nk)) out[m++] = ijk_to_lin(ni, nj, nk, B);
      }
  return m;
}

// CTA-wide ordered compaction: this thread's position among the threads with keep == true (in
// thread order); *total = the CTA's count.  wsum: shared int[32].
__device__ __forceinline__ int dive_cta_rank(bool keep, int* total, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) before += wsum[w];
    tot += wsum[w];
  }
  __syncthreads();
  *total = tot;
  return before + __popc(bal & ((1u << lane) - 1u));
}

// the candidate children (Bc = f Bp) of the neighbourhood of `pick`, in (parent, a, b, c) order,
// written to out[0 .. min(count, cap)); returns the count (every thread).  par: shared
// uint32[27]; sh: shared int[34].
__device__ __forceinline__ int dive_children_cta(uint32_t pick, int32_t Bp, int32_t f,
                                                 uint32_t* out, int32_t cap, const Excl& ex,
                                                 bool finest, uint32_t* par, int* sh) {
  if (threadIdx.x == 0) sh[32] = dive_neighbourhood(Bp, pick, par);
  __syncthreads();
  const int f3 = f * f * f, total = sh[32] * f3;
  const int32_t Bc = Bp * f;
  int base = 0;
  for (int e0 = 0; e0 < total; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    bool keep = false;
    uint32_t lin = 0;
    if (e < total) {
      int32_t i, j, k;
      lin_to_ijk(par[e / f3], Bp, i, j, k);
      const int r = e % f3, a = r / (f * f), b = (r / f) % f, c = r % f;
      const int32_t ci = f * i + a, cj = f * j + b, ck = f * k + c;
      lin = ijk_to_lin(ci, cj, ck, Bc);
      keep = is_candidate(Bc, ci, cj, ck) && !excl_dropped(ex, Bc, lin, finest);
    }
    int tot;
    const int pos = dive_cta_rank(keep, &tot, sh);
    if (keep && base + pos < cap) out[base + pos] = lin;
    base += tot;
  }
  return base < cap ? base : cap;
}

// the dive's pick over a list (lins, a) of m blocks at resolution B (n correspondences); returns
// it to every thread.  sh: shared DiveKey[33].
struct DiveKey {
  int32_t valid, rank;
  double x;
  uint32_t lin;
};
__device__ __forceinline__ bool dive_better(const DiveKey& a, const DiveKey& b) {
  if (!b.valid) return a.valid != 0;
  if (!a.valid) return false;
  if (a.rank != b.rank) return a.rank > b.rank;
  if (a.x != b.x) return a.x > b.x;
  return a.lin < b.lin;
}
__device__ __forceinline__ DiveKey dive_shfl(const DiveKey& k, int o) {
  DiveKey r;
  r.valid = __shfl_down_sync(0xffffffffu, k.valid, o);
  r.rank = __shfl_down_sync(0xffffffffu, k.rank, o);
  r.x = __shfl_down_sync(0xffffffffu, k.x, o);
  r.lin = __shfl_down_sync(0xffffffffu, k.lin, o);
  return r;
}
__device__ __forceinline__ uint32_t dive_pick_cta(const uint32_t* __restrict__ lins,
                                                  const uint32_t* __restrict__ a, int m, int32_t B,
                                                  double eps, double n, const Excl& ex,
                                                  DiveKey* sh) {
  DiveKey best{0, 0, -1e300, 0u};
  for (int e = threadIdx.x; e < m; e += blockDim.x) {
    const uint32_t lin = lins[e];
    int32_t i, j, k;
    lin_to_ijk(lin, B, i, j, k);
    DiveKey c;
    c.valid = 1;
    c.rank = 2 * excl_rank(ex, B, lin) + (centre_inside(B, lin) ? 1 : 0);
    c.x = (double)a[e] - n * (1.0 - bound_threshold(B, i, j, k, eps)) * 0.5;
    c.lin = lin;
    if (dive_better(c, best)) best = c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const DiveKey other = dive_shfl(best, o);
    if (dive_better(other, best)) best = other;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) sh[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    DiveKey b = sh[0];
    for (int w = 1; w < nw; ++w)
      if (dive_better(sh[w], b)) b = sh[w];
    sh[32] = b;
  }
  __syncthreads();
  const uint32_t r = sh[32].lin;
  __syncthreads();
  return r;
}

}  // namespace rv
