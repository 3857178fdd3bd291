// rv_dplan.cu -- the certified coarse-to-fine level loop of a BATCHED solve, on the device.
//
// The host planner (rv_plan.cpp) decides, level by level, which blocks to vote; for one large
// problem that is cheap, but a batch of thousands of small problems would spend its time in
// per-problem host work and transfers.  These kernels take the same decisions for every
// problem at once (one CTA per problem), so the host only sequences the phases and reads back
// per-phase totals (to size the next launch).  The decisions reproduce rv_plan.cpp exactly:
//   dive:  children of the 27-neighbourhood of the pick (neighbours in ascending lin, children
//          in (a,b,c) order); pick = max excess UB - n*bg (centre inside the ball first, ties
//          -> lowest lin); at the finest level lb* = max cnt_b;
//   BnB:   parents with UB >= lb*, their candidate children in parent order;
//   final: L = max lo; recheck the blocks with hi >= L and hi != lo; winner = max exact count,
//          ties -> lowest lin.
// Ordered compaction inside a CTA uses warp ballots + a CTA-wide exclusive scan.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rotvote.h"
#include "rv_dplan.h"
#include "rv_geom.h"

namespace rv {

namespace {

constexpr int kDpThreads = 256;

// CTA-wide ordered compaction helper: returns this thread's output position among the
// threads with keep == true (in thread order) and writes the CTA total to *total.
__device__ __forceinline__ int cta_rank(bool keep, int* total, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0, tot = 0;
  for (int w = 0; w < kDpThreads / 32; ++w) {
    if (w < warp) before += wsum[w];
    tot += wsum[w];
  }
  __syncthreads();
  *total = tot;
  return before + __popc(bal & ((1u << lane) - 1u));
}

// the 27-neighbourhood of (i,j,k) at resolution B, candidates only, ascending lin: the offsets
// (a,b,c) in lexicographic order give ascending lin
__device__ int neighbourhood(int32_t B, uint32_t lin, uint32_t out[27]) {
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

}  // namespace

// Dive children: parents = neighbourhood of the pick at level resolution Bp (pick[p], or
// idx_list[pick_idx[p]] when idx_list is given: the level-0 argmax indexes the grid list);
// children at Bc = f*Bp written (in order) to out + p*cap; cnt[p] = number written.
__global__ void __launch_bounds__(kDpThreads) dp_dive_children(const uint32_t* __restrict__ pick,
                                                               const int32_t* __restrict__ pick_idx,
                                                               const uint32_t* __restrict__ idx_list,
                                                               int32_t Bp, int32_t f,
                                                               uint32_t* out, int32_t cap,
                                                               int32_t* cnt) {
  const int p = blockIdx.x;
  __shared__ uint32_t par[27];
  __shared__ int npar, wsum[kDpThreads / 32];
  if (threadIdx.x == 0)
    npar = neighbourhood(Bp, idx_list ? idx_list[pick_idx[p]] : pick[p], par);
  __syncthreads();
  const int f3 = f * f * f, total = npar * f3;
  const int32_t Bc = Bp * f;
  int base = 0;
  for (int e0 = 0; e0 < total; e0 += kDpThreads) {
    const int e = e0 + threadIdx.x;
    bool keep = false;
    uint32_t lin = 0;
    if (e < total) {
      int32_t i, j, k;
      lin_to_ijk(par[e / f3], Bp, i, j, k);
      const int r = e % f3, a = r / (f * f), b = (r / f) % f, c = r % f;
      const int32_t ci = f * i + a, cj = f * j + b, ck = f * k + c;
      keep = is_candidate(Bc, ci, cj, ck);
      lin = ijk_to_lin(ci, cj, ck, Bc);
    }
    int tot;
    const int pos = cta_rank(keep, &tot, wsum);
    if (keep && base + pos < cap) out[(int64_t)p * cap + base + pos] = lin;
    base += tot;
  }
  if (threadIdx.x == 0) cnt[p] = base < cap ? base : cap;
}

// Dive pick over the problem's list (lins, a) of cnt[p] blocks at list + off[p].
__global__ void __launch_bounds__(kDpThreads) dp_dive_pick(const uint32_t* __restrict__ lins,
                                                           const uint32_t* __restrict__ a,
                                                           const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ cnt,
                                                           int32_t B, double eps,
                                                           const int64_t* __restrict__ rows,
                                                           uint32_t* pick) {
  const int p = blockIdx.x;
  const double n = (double)(rows[p + 1] - rows[p]);
  const int64_t o = off[p];
  const int m = cnt[p];
  int best = -1, bin = 0;
  double bx = -1e300;
  uint32_t blin = 0;
  for (int e = threadIdx.x; e < m; e += blockDim.x) {
    const uint32_t lin = lins[o + e];
    int32_t i, j, k;
    lin_to_ijk(lin, B, i, j, k);
    const int in = centre_inside(B, lin) ? 1 : 0;
    const double t = bound_threshold(B, i, j, k, eps);
    const double x = (double)a[o + e] - n * (1.0 - t) * 0.5;
    if (best < 0 || in > bin || (in == bin && (x > bx || (x == bx && lin < blin)))) {
      best = e; bin = in; bx = x; blin = lin;
    }
  }
  __shared__ int sb[kDpThreads], si[kDpThreads];
  __shared__ double sx[kDpThreads];
  __shared__ uint32_t sl[kDpThreads];
  sb[threadIdx.x] = best; si[threadIdx.x] = bin; sx[threadIdx.x] = bx; sl[threadIdx.x] = blin;
  __syncthreads();
  for (int w = kDpThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const int o2 = threadIdx.x + w;
      if (sb[o2] >= 0) {
        const int t = threadIdx.x;
        const bool take = sb[t] < 0 || si[o2] > si[t] ||
                          (si[o2] == si[t] && (sx[o2] > sx[t] || (sx[o2] == sx[t] && sl[o2] < sl[t])));
        if (take) { sb[t] = sb[o2]; si[t] = si[o2]; sx[t] = sx[o2]; sl[t] = sl[o2]; }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) pick[p] = sl[0];
}

// lb*[p] = max cnt_b over the problem's list
__global__ void __launch_bounds__(kDpThreads) dp_max_lo(const uint32_t* __restrict__ b,
                                                        const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ cnt,
                                                        int64_t* lb) {
  const int p = blockIdx.x;
  uint32_t mx = 0;
  for (int e = threadIdx.x; e < cnt[p]; e += blockDim.x) mx = max(mx, b[off[p] + e]);
  for (int s = 16; s > 0; s >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, s));
  __shared__ uint32_t w[kDpThreads / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int i = 0; i < kDpThreads / 32; ++i) r = max(r, w[i]);
    lb[p] = r;
  }
}

// BnB children of the parents with UB >= lb[p].  Parent list of problem p: lins + poff[p]
// (or the shared grid list when shared != 0) with counts ub + uoff[p], pcnt[p] entries.
// count pass (out == nullptr): ccnt[p] = number of candidate children; write pass: children
// in parent order at out + coff[p].
__global__ void __launch_bounds__(kDpThreads) dp_bnb_children(
    const uint32_t* __restrict__ lins, const int64_t* __restrict__ poff,
    const uint32_t* __restrict__ ub, const int64_t* __restrict__ uoff,
    const int32_t* __restrict__ pcnt, int64_t shared_m, const int64_t* __restrict__ lb,
    int32_t Bp, int32_t f, uint32_t* out, const int64_t* __restrict__ coff, int32_t* ccnt) {
  const int p = blockIdx.x;
  __shared__ int wsum[kDpThreads / 32];
  __shared__ uint32_t sp[kDpThreads];  // survivors of the current parent chunk, in order
  const int64_t po = shared_m ? 0 : poff[p];
  const int64_t uo = shared_m ? (int64_t)p * shared_m : uoff[p];
  const int m = shared_m ? (int)shared_m : pcnt[p];
  const int f3 = f * f * f;
  const int32_t Bc = Bp * f;
  const int64_t L = lb[p];
  int base = 0;
  for (int c0 = 0; c0 < m; c0 += kDpThreads) {
    // 1. the chunk's survivors (UB >= lb*), compacted in parent order
    const int par = c0 + threadIdx.x;
    const bool surv = par < m && (int64_t)ub[uo + par] >= L;
    int ns;
    const int spos = cta_rank(surv, &ns, wsum);
    if (surv) sp[spos] = lins[po + par];
    __syncthreads();
    // 2. their candidate children, (parent, a, b, c) order
    for (int e0 = 0; e0 < ns * f3; e0 += kDpThreads) {
      const int e = e0 + threadIdx.x;
      bool keep = false;
      uint32_t lin = 0;
      if (e < ns * f3) {
        int32_t i, j, k;
        lin_to_ijk(sp[e / f3], Bp, i, j, k);
        const int r = e % f3, a = r / (f * f), b = (r / f) % f, c = r % f;
        const int32_t ci = f * i + a, cj = f * j + b, ck = f * k + c;
        keep = is_candidate(Bc, ci, cj, ck);
        lin = ijk_to_lin(ci, cj, ck, Bc);
      }
      int tot;
      const int pos = cta_rank(keep, &tot, wsum);
      if (out && keep) out[coff[p] + base + pos] = lin;
      base += tot;
    }
    __syncthreads();  // sp is rewritten by the next chunk
  }
  if (!out && threadIdx.x == 0) ccnt[p] = base;
}

// Finest level: L[p] = max lo; recheck set = blocks with hi >= L and hi != lo (count pass /
// ordered write of their list positions at rlist + roff[p]).
__global__ void __launch_bounds__(kDpThreads) dp_recheck_set(
    const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo,
    const int64_t* __restrict__ off, const int32_t* __restrict__ cnt, int32_t* rcnt,
    const int64_t* __restrict__ roff, int32_t* rlist) {
  const int p = blockIdx.x;
  __shared__ int wsum[kDpThreads / 32];
  __shared__ uint32_t Ls;
  uint32_t mx = 0;
  for (int e = threadIdx.x; e < cnt[p]; e += blockDim.x) mx = max(mx, lo[off[p] + e]);
  for (int s = 16; s > 0; s >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, s));
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = (int)mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int i = 0; i < kDpThreads / 32; ++i) r = max(r, (uint32_t)wsum[i]);
    Ls = r;
  }
  __syncthreads();
  const uint32_t L = Ls;
  int base = 0;
  for (int e0 = 0; e0 < cnt[p]; e0 += kDpThreads) {
    const int e = e0 + threadIdx.x;
    const bool keep = e < cnt[p] && hi[off[p] + e] >= L && hi[off[p] + e] != lo[off[p] + e];
    int tot;
    const int pos = cta_rank(keep, &tot, wsum);
    if (rlist && keep) rlist[roff[p] + base + pos] = e;
    base += tot;
  }
  if (!rlist && threadIdx.x == 0) rcnt[p] = base;
}

// Gather the lins of the recheck list (positions rlist) into rlins (same layout).
__global__ void dp_gather(const uint32_t* __restrict__ lins, const int64_t* __restrict__ off,
                          const int64_t* __restrict__ roff, const int32_t* __restrict__ rcnt,
                          const int32_t* __restrict__ rlist, uint32_t* rlins) {
  const int p = blockIdx.x;
  for (int e = threadIdx.x; e < rcnt[p]; e += blockDim.x)
    rlins[roff[p] + e] = lins[off[p] + rlist[roff[p] + e]];
}

// Winner per problem: exact count = lo where lo == hi, the rechecked count where rechecked;
// max, ties -> lowest lin.  res[p] = {lin, votes, n_tied}.
__global__ void __launch_bounds__(kDpThreads) dp_finalize(
    const uint32_t* __restrict__ lins, const uint32_t* __restrict__ hi,
    const uint32_t* __restrict__ lo, const int64_t* __restrict__ off,
    const int32_t* __restrict__ cnt, const uint32_t* __restrict__ ex,
    const int64_t* __restrict__ roff, const int32_t* __restrict__ rcnt,
    const int32_t* __restrict__ rlist, int32_t* res) {
  const int p = blockIdx.x;
  __shared__ int64_t best[kDpThreads];
  __shared__ uint32_t blin[kDpThreads];
  __shared__ int32_t ties[kDpThreads];
  int64_t b = -1;
  uint32_t bl = 0xffffffffu;
  int32_t t = 0;
  auto offer = [&](int64_t v, uint32_t lin) {
    if (v > b) { b = v; bl = lin; t = 1; }
    else if (v == b) { ++t; if (lin < bl) bl = lin; }
  };
  for (int e = threadIdx.x; e < cnt[p]; e += blockDim.x)
    if (hi[off[p] + e] == lo[off[p] + e]) offer(lo[off[p] + e], lins[off[p] + e]);
  for (int e = threadIdx.x; e < rcnt[p]; e += blockDim.x)
    offer(ex[roff[p] + e], lins[off[p] + rlist[roff[p] + e]]);
  best[threadIdx.x] = b; blin[threadIdx.x] = bl; ties[threadIdx.x] = t;
  __syncthreads();
  for (int w = kDpThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const int o = threadIdx.x + w, s = threadIdx.x;
      if (best[o] > best[s]) { best[s] = best[o]; blin[s] = blin[o]; ties[s] = ties[o]; }
      else if (best[o] == best[s] && best[o] >= 0) {
        ties[s] += ties[o];
        if (blin[o] < blin[s]) blin[s] = blin[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    res[3 * p] = (int32_t)blin[0];
    res[3 * p + 1] = (int32_t)(best[0] < 0 ? 0 : best[0]);
    res[3 * p + 2] = ties[0];
  }
}

// --- launchers ------------------------------------------------------------------------------
void dp_launch_dive_children(const uint32_t* pick, const int32_t* pick_idx,
                             const uint32_t* idx_list, int32_t Bp, int32_t f, uint32_t* out,
                             int32_t cap, int32_t* cnt, int32_t P, cudaStream_t s) {
  dp_dive_children<<<P, kDpThreads, 0, s>>>(pick, pick_idx, idx_list, Bp, f, out, cap, cnt);
}
void dp_launch_dive_pick(const uint32_t* lins, const uint32_t* a, const int64_t* off,
                         const int32_t* cnt, int32_t B, double eps, const int64_t* rows,
                         uint32_t* pick, int32_t P, cudaStream_t s) {
  dp_dive_pick<<<P, kDpThreads, 0, s>>>(lins, a, off, cnt, B, eps, rows, pick);
}
void dp_launch_max_lo(const uint32_t* b, const int64_t* off, const int32_t* cnt, int64_t* lb,
                      int32_t P, cudaStream_t s) {
  dp_max_lo<<<P, kDpThreads, 0, s>>>(b, off, cnt, lb);
}
void dp_launch_bnb_children(const uint32_t* lins, const int64_t* poff, const uint32_t* ub,
                            const int64_t* uoff, const int32_t* pcnt, int64_t shared_m,
                            const int64_t* lb, int32_t Bp, int32_t f, uint32_t* out,
                            const int64_t* coff, int32_t* ccnt, int32_t P, cudaStream_t s) {
  dp_bnb_children<<<P, kDpThreads, 0, s>>>(lins, poff, ub, uoff, pcnt, shared_m, lb, Bp, f, out,
                                           coff, ccnt);
}
void dp_launch_recheck_set(const uint32_t* hi, const uint32_t* lo, const int64_t* off,
                           const int32_t* cnt, int32_t* rcnt, const int64_t* roff, int32_t* rlist,
                           int32_t P, cudaStream_t s) {
  dp_recheck_set<<<P, kDpThreads, 0, s>>>(hi, lo, off, cnt, rcnt, roff, rlist);
}
void dp_launch_gather(const uint32_t* lins, const int64_t* off, const int64_t* roff,
                      const int32_t* rcnt, const int32_t* rlist, uint32_t* rlins, int32_t P,
                      cudaStream_t s) {
  dp_gather<<<P, 128, 0, s>>>(lins, off, roff, rcnt, rlist, rlins);
}
void dp_launch_finalize(const uint32_t* lins, const uint32_t* hi, const uint32_t* lo,
                        const int64_t* off, const int32_t* cnt, const uint32_t* ex,
                        const int64_t* roff, const int32_t* rcnt, const int32_t* rlist,
                        int32_t* res, int32_t P, cudaStream_t s) {
  dp_finalize<<<P, kDpThreads, 0, s>>>(lins, hi, lo, off, cnt, ex, roff, rcnt, rlist, res);
}

}  // namespace rv
