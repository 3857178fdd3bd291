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
//   BnB:   parents with UB >= lb*, their candidate children;
//   final: L = max lo; recheck the blocks with hi >= L and hi != lo; winner = max exact count,
//          ties -> lowest lin (a packed 64-bit atomicMax of (count, ~lin)).
// The dive's lists are built per problem (one CTA, ordered compaction by warp ballots + a
// CTA-wide scan); the BnB and final-level kernels are flat (one thread per list entry of all
// problems, per-problem atomic slot allocation).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rotvote.h"
#include "rv_dive.cuh"
#include "rv_dplan.h"
#include "rv_geom.h"

namespace rv {

namespace {

constexpr int kDpThreads = 256;

// (the dive helpers: rv_dive.cuh)

}  // namespace

// Dive children: parents = neighbourhood of the pick at level resolution Bp (pick[p], or
// idx_list[pick_idx[p]] when idx_list is given: the level-0 argmax indexes the grid list);
// children at Bc = f*Bp written (in order) to out + p*cap; cnt[p] = number written.
__global__ void __launch_bounds__(kDpThreads) dp_dive_children(const uint32_t* __restrict__ pick,
                                                               const int32_t* __restrict__ pick_idx,
                                                               const uint32_t* __restrict__ idx_list,
                                                               int32_t Bp, int32_t f,
                                                               uint32_t* out, int32_t cap,
                                                               int32_t* cnt,
                                                               const int32_t* __restrict__ active,
                                                               Excl ex, int32_t finest) {
  const int p = blockIdx.x;
  if (active && !active[p]) {  // re-dive: this problem did not trigger it
    if (threadIdx.x == 0) cnt[p] = 0;
    return;
  }
  __shared__ uint32_t par[27];
  __shared__ int sh[34];
  const uint32_t pk = idx_list ? idx_list[pick_idx[p]] : pick[p];
  const int c = dive_children_cta(pk, Bp, f, out + (int64_t)p * cap, cap, ex, finest != 0, par, sh);
  if (threadIdx.x == 0) cnt[p] = c;
}

// Dive pick over the problem's list (lins, a) of cnt[p] blocks at list + off[p].
__global__ void __launch_bounds__(kDpThreads) dp_dive_pick(const uint32_t* __restrict__ lins,
                                                           const uint32_t* __restrict__ a,
                                                           const int64_t* __restrict__ off,
                                                           const int32_t* __restrict__ cnt,
                                                           int32_t B, double eps,
                                                           const int64_t* __restrict__ rows,
                                                           uint32_t* pick, Excl ex) {
  const int p = blockIdx.x;
  __shared__ DiveKey sh[33];
  const int64_t o = off[p];
  const uint32_t pk = dive_pick_cta(lins + o, a + o, cnt[p], B, eps,
                                    (double)(rows[p + 1] - rows[p]), ex, sh);
  if (threadIdx.x == 0) pick[p] = pk;
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

// ---- flat list kernels: one thread per list entry of all problems ----------------------------
// A level's list of problem p holds act_off[p+1] - act_off[p] entries stored from cap[p]
// (capacity layout: a problem's children are bounded by its parents x f^3).  The order of
// the entries inside a problem's list is not deterministic (atomic slot allocation) and
// never matters: every decision is a max with ties broken by the lowest lin.
__device__ __forceinline__ int find_problem(const int64_t* __restrict__ act_off, int32_t P,
                                            int64_t g) {
  int lo = 0, hi = P;  // last p with act_off[p] <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (act_off[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// BnB: candidate children (Bc = f*Bp) of the parents with UB >= lb[p], appended to problem
// p's child region ccap[p] (count ccnt[p], zeroed by the caller); their count slots are
// zeroed here.  shared_lins: the parents' lins are plins[e] (the level-0 grid shared by all
// problems), else plins[pcap[p] + e].
__global__ void dp_bnb_expand(const uint32_t* __restrict__ plins, int32_t shared_lins,
                              const int64_t* __restrict__ act_off, const int64_t* __restrict__ pcap,
                              const uint32_t* __restrict__ pub, const int64_t* __restrict__ lb,
                              int32_t P, int32_t Bp, int32_t f, const int64_t* __restrict__ ccap,
                              uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                              int32_t* err, Own own, Excl ex, int32_t finest, TailScan ts) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < ts.zero_n;
       b += (int64_t)gridDim.x * blockDim.x)
    ts.zero_buf[b] = 0;
  const int64_t total = act_off[P];
  const int32_t Bc = Bp * f;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    // shared level-0 parents: every problem has act_off[1] of them (no search needed)
    const int p = shared_lins ? (int)(g / act_off[1]) : find_problem(act_off, P, g);
    const int64_t e = g - act_off[p], idx = pcap[p] + e;
    if ((int64_t)pub[idx] < lb[p]) continue;
    int32_t i, j, k;
    lin_to_ijk(shared_lins ? plins[e] : plins[idx], Bp, i, j, k);
    if (own.lut) {  // another rank's subtree: the owner of its level-0 ancestor's group expands it
      const int32_t r = Bp / own.B0;
      const int32_t grp = own.lut[ijk_to_lin(i / r, j / r, k / r, own.B0)];
      if (grp < own.lo || grp >= own.hi) continue;
    }
    auto kept = [&](int32_t ci, int32_t cj, int32_t ck) {
      return is_candidate(Bc, ci, cj, ck) &&
             !excl_dropped(ex, Bc, ijk_to_lin(ci, cj, ck, Bc), finest != 0);
    };
    int c = 0;
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b)
        for (int d = 0; d < f; ++d) c += kept(f * i + a, f * j + b, f * k + d) ? 1 : 0;
    if (c == 0) continue;
    int64_t w = ccap[p] + atomicAdd(&ccnt[p], c);
    if (w + c > ccap[p + 1]) {  // invariant: children <= parents x f^3 (never expected)
      atomicOr(err, 1);
      continue;
    }
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b)
        for (int d = 0; d < f; ++d) {
          const int32_t ci = f * i + a, cj = f * j + b, ck = f * k + d;
          if (!kept(ci, cj, ck)) continue;
          clins[w] = ijk_to_lin(ci, cj, ck, Bc);
          ca[w] = 0;
          cb[w] = 0;
          ++w;
        }
  }
  if (ts.done) {  // the one-problem scan, by the last CTA to finish (see TailScan)
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(ts.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      volatile int32_t* vc = ccnt;
      int32_t c = vc[0];
      if (ts.rc.flags) {  // re-dive trigger (R18), once per problem
        const int32_t fl = (!ts.rc.done[0] && ts.rc.pcnt[0] > 0 && c >= 16384 &&
                            2 * (int64_t)c > (int64_t)ts.rc.pcnt[0] * ts.rc.f3) ? 1 : 0;
        ts.rc.flags[0] = fl;
        if (fl) {
          ts.rc.done[0] = 1;
          atomicOr(ts.rc.any, ts.rc.any_bit);
        }
      }
      if (ts.op.err && *reinterpret_cast<volatile int32_t*>(ts.op.err)) {  // abandon the level
        c = 0;
        ccnt[0] = 0;
      }
      const int64_t nb = (int64_t)c * ts.f3;
      ts.act[0] = 0;
      ts.act[1] = c;
      if (ts.next_base) {
        ts.next_base[0] = 0;
        ts.next_base[1] = ts.op.cap_lim > 0 && nb > ts.op.cap_lim ? ts.op.cap_lim : nb;
      }
      *ts.total = c;
      if (ts.phase) *ts.phase = ts.phase_add ? *ts.phase + c : c;
      if (ts.zero_next) *ts.zero_next = 0;
      *ts.done = 0;
    }
  }
}

// finest level, pass 1: Lmax[p] = max lo (zeroed by the caller); one atomic per (warp, problem)
__global__ void dp_final_max(const int64_t* __restrict__ act_off, const int64_t* __restrict__ cap,
                             const uint32_t* __restrict__ lo, int32_t P, uint32_t* Lmax) {
  const int64_t total = act_off[P];
  const int lane = threadIdx.x & 31;
  // warp-uniform loop: lanes past the end run with valid == false (whole-warp reductions)
  for (int64_t g0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); g0 < total;
       g0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = g0 + lane;
    const bool valid = g < total;
    const int p = valid ? find_problem(act_off, P, g) : -1;
    const uint32_t v = valid ? lo[cap[p] + g - act_off[p]] : 0u;
    const uint32_t grp = __match_any_sync(0xffffffffu, p);
    const uint32_t mx = __reduce_max_sync(grp, v);
    if (valid && lane == __ffs(grp) - 1) atomicMax(&Lmax[p], mx);
  }
}

__device__ __forceinline__ unsigned long long win_key(uint32_t votes, uint32_t lin) {
  return ((unsigned long long)votes << 32) | (unsigned long long)(0xffffffffu - lin);
}

// finest level, pass 2: blocks with hi == lo offer their (exact) count to best[p] (one
// atomic per (warp, problem)); blocks with hi >= Lmax[p], hi != lo go to the recheck list of
// problem p (region act_off[p], count rcnt[p]; both zeroed by the caller)
__global__ void dp_final_split(const int64_t* __restrict__ act_off, const int64_t* __restrict__ cap,
                               const uint32_t* __restrict__ lins, const uint32_t* __restrict__ hi,
                               const uint32_t* __restrict__ lo, const uint32_t* __restrict__ Lmax,
                               int32_t P, unsigned long long* best, uint32_t* rlins,
                               int32_t* rcnt) {
  const int64_t total = act_off[P];
  const int lane = threadIdx.x & 31;
  // warp-uniform loop: lanes past the end run with valid == false (whole-warp reductions)
  for (int64_t g0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); g0 < total;
       g0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = g0 + lane;
    const bool valid = g < total;
    const int p = valid ? find_problem(act_off, P, g) : -1;
    uint32_t h = 0, l = 0, lin = 0;
    if (valid) {
      const int64_t idx = cap[p] + g - act_off[p];
      h = hi[idx];
      l = lo[idx];
      lin = lins[idx];
    }
    const bool exact = valid && h == l;
    const uint32_t grp = __match_any_sync(0xffffffffu, p);
    const uint32_t vmax = __reduce_max_sync(grp, exact ? l : 0u);
    const uint32_t lmin = __reduce_min_sync(grp, (exact && l == vmax) ? lin : 0xffffffffu);
    const uint32_t any = __ballot_sync(0xffffffffu, exact) & grp;
    if (any && lane == __ffs(grp) - 1) atomicMax(&best[p], win_key(vmax, lmin));
    if (valid && !exact && h >= Lmax[p]) rlins[act_off[p] + atomicAdd(&rcnt[p], 1)] = lin;
  }
}

// finest level, pass 3 (after the exact recheck): rechecked blocks offer their exact counts
__global__ void dp_final_rechecked(const int64_t* __restrict__ act_off,
                                   const int32_t* __restrict__ rcnt,
                                   const uint32_t* __restrict__ rlins,
                                   const uint32_t* __restrict__ ex, int32_t P,
                                   unsigned long long* best) {
  const int64_t total = act_off[P];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int p = find_problem(act_off, P, g);
    if (g - act_off[p] >= rcnt[p]) continue;
    atomicMax(&best[p], win_key(ex[g], rlins[g]));
  }
}

// finest level, pass 4: ties[p] = exact-known blocks with the winning count (zeroed by the
// caller).  Blocks neither exact nor rechecked have hi < Lmax <= the best count.
__global__ void dp_final_ties(const int64_t* __restrict__ act_off, const int64_t* __restrict__ cap,
                              const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo,
                              const int32_t* __restrict__ rcnt, const uint32_t* __restrict__ ex,
                              int32_t P, const unsigned long long* __restrict__ best,
                              int32_t* ties) {
  const int64_t total = act_off[P];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < 2 * total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = g < total ? g : g - total;
    const int p = find_problem(act_off, P, h);
    const uint32_t bv = (uint32_t)(best[p] >> 32);
    if (g < total) {
      const int64_t idx = cap[p] + h - act_off[p];
      if (hi[idx] == lo[idx] && lo[idx] == bv) atomicAdd(&ties[p], 1);
    } else if (h - act_off[p] < rcnt[p] && ex[h] == bv) {
      atomicAdd(&ties[p], 1);
    }
  }
}

// ---- device-built vote decomposition ---------------------------------------------------------
namespace {
__host__ __device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }
constexpr int kPlanThreads = 1024;
constexpr int64_t kExactChunk = 1 << 12;  // = build_exact_items (the final level has few blocks: the CTAs come from the correspondences)

// correspondence chunks of a problem with nt tiles: ct = ceil(nt / min(nch, nt)) tiles each,
// ceil(nt / ct) of them non-empty (the host builder's loop `for t0 < nt; t0 += ct`)
__device__ __forceinline__ void tc_chunks(int64_t nt, int64_t nch_all, int64_t* ct, int64_t* nc) {
  const int64_t nch = i64min(nch_all, nt);
  *ct = (nt + nch - 1) / nch;
  *nc = (nt + *ct - 1) / *ct;
}

__device__ __forceinline__ int64_t list_m(const DpList& L, int p) {
  return L.cnt ? (int64_t)L.cnt[p] : L.shared_m;
}

// CTA-wide exclusive scan of one int64 per thread (kPlanThreads threads): warp shuffles,
// then the warp totals scanned by warp 0 -- two barriers
__device__ int64_t cta_scan_excl(int64_t v, int64_t* sh, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;  // warp inclusive total
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < kPlanThreads / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sh[32 + lane] = w;  // inclusive prefix of the warp totals
  }
  __syncthreads();
  const int64_t before = warp > 0 ? sh[32 + warp - 1] : 0;
  *total = sh[32 + kPlanThreads / 32 - 1];
  __syncthreads();  // sh is reused by the next call
  return before + x - v;
}

// CTA-wide max of one int64 per thread
__device__ int64_t cta_max(int64_t v, int64_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = i64max(v, __shfl_down_sync(0xffffffffu, v, o));
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  int64_t r = sh[0];
  for (int w = 1; w < kPlanThreads / 32; ++w) r = i64max(r, sh[w]);
  __syncthreads();
  return r;
}
}  // namespace

__global__ void __launch_bounds__(kPlanThreads) dp_items_plan(
    DpList L, const int64_t* __restrict__ rows, const int64_t* __restrict__ koffs, int32_t P,
    int32_t B, double eps, int mode, int32_t slots, VoteSeg* segs, int64_t* item_off,
    int64_t* ablk_off, int32_t* counts, uint32_t* bits0, int64_t bits_m0) {
  __shared__ int64_t sh[kPlanThreads];
  __shared__ int64_t s_cbs, s_tmax;
  __shared__ int32_t s_nch;
  const int t = threadIdx.x;
  const int cpb = mode == 1 ? kTcM / 2 : kTcM;
  // this thread's contiguous range of problems
  const int p0 = (int)((int64_t)P * t / kPlanThreads), p1 = (int)((int64_t)P * (t + 1) / kPlanThreads);
  int64_t cbs = 0, tmax = 0;
  for (int p = p0; p < p1; ++p) {
    const int64_t m = list_m(L, p), n = rows[p + 1] - rows[p];
    if (m == 0 || n == 0) continue;
    cbs += (m + cpb - 1) / cpb;
    tmax = i64max(tmax, (n + kTcN - 1) / kTcN);
  }
  int64_t tot;
  cta_scan_excl(cbs, sh, &tot);
  if (t == 0) s_cbs = tot;
  const int64_t tmx = cta_max(tmax, sh);
  if (t == 0) s_tmax = tmx;
  __syncthreads();
  {
    // correspondence chunks per item: fill whole waves of the persistent kernel's CTAs (the
    // host rule: best score, >= 4 waves preferred; up to 64 waves).  Thread t scores the chunk
    // counts t+1, t+1+kPlanThreads, ...; the CTA keeps the best score, smallest count.
    const int64_t cb_all = s_cbs, tm = s_tmax;
    double my_s = -1e300;
    int64_t my_n = 1;
    if (mode != 2 && cb_all > 0) {
      const int64_t min_tiles = i64min(tm, 8);
      const int64_t max_nch = i64max(1, tm / i64max(1, min_tiles));
      for (int64_t nch = 1 + t; nch <= max_nch; nch += kPlanThreads) {
        const double waves = (double)(cb_all * nch) / slots;
        if (waves > 64.0 && nch > 1) break;
        const double eff = waves / ceil(waves);
        const double score = eff - (waves < 4.0 ? 0.5 * (4.0 - waves) / 4.0 : 0.0);
        if (score > my_s + 1e-9) { my_s = score; my_n = nch; }
      }
    }
    __shared__ double ss[kPlanThreads / 32];
    double m = my_s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_down_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    if ((t & 31) == 0) ss[t >> 5] = m;
    __syncthreads();
    double top = ss[0];
    for (int w = 1; w < kPlanThreads / 32; ++w) top = ss[w] > top ? ss[w] : top;
    // smallest chunk count whose score is within 1e-9 of the best
    const int64_t cand = (my_s > top - 1e-9) ? my_n : INT64_MAX;
    const int64_t best_n = -cta_max(-cand, sh);
    if (t == 0) s_nch = (int32_t)(best_n == INT64_MAX ? 1 : best_n);
  }
  __syncthreads();
  const int64_t nch_all = s_nch;
  // per-problem item / A-block counts, their offsets, and the segments
  int64_t ni = 0, na = 0;
  for (int p = p0; p < p1; ++p) {
    const int64_t m = list_m(L, p), n = rows[p + 1] - rows[p];
    if (m == 0 || n == 0) continue;
    if (mode == 2) {
      ni += (m + kExactCells - 1) / kExactCells * ((n + kExactChunk - 1) / kExactChunk);
    } else {
      const int64_t cb = (m + cpb - 1) / cpb, nt = (n + kTcN - 1) / kTcN;
      int64_t ct, nc;
      tc_chunks(nt, nch_all, &ct, &nc);
      ni += cb * nc;
      if (!L.shared || p == 0) na += cb;
    }
  }
  int64_t ti, ta;
  int64_t ei = cta_scan_excl(ni, sh, &ti);
  int64_t ea = cta_scan_excl(na, sh, &ta);
  for (int p = p0; p < p1; ++p) {
    item_off[p] = ei;
    ablk_off[p] = L.shared ? 0 : ea;
    const int64_t m = list_m(L, p), n = rows[p + 1] - rows[p];
    if (m > 0 && n > 0) {
      if (mode == 2) {
        ei += (m + kExactCells - 1) / kExactCells * ((n + kExactChunk - 1) / kExactChunk);
      } else {
        const int64_t cb = (m + cpb - 1) / cpb, nt = (n + kTcN - 1) / kTcN;
        int64_t ct, nc;
        tc_chunks(nt, nch_all, &ct, &nc);
        ei += cb * nc;
        if (!L.shared || p == 0) ea += cb;
      }
    }
    VoteSeg sg;
    const int64_t b = L.shared ? (int64_t)p * L.shared_m : L.base[p];
    sg.lins = L.shared ? L.lins : L.lins + b;
    sg.cnt_a = L.ca + b;
    sg.cnt_b = L.cb + b;
    sg.koff = koffs[p];
    sg.row = rows[p];
    sg.n = (int32_t)n;
    sg.B = B;
    sg.eps = eps;
    // level-0 pass bitmasks (K3-TC BITS; the list is the shared level-0 grid): rows of m0
    // blocks x wpc words, problem p from m0 * toffs[p] / 32
    sg.wpc = (int32_t)((koffs[p + 1] - koffs[p]) / 32);
    // (a rank's slice of a one-problem grid starts at row base[0] of the grid)
    sg.bits = bits0 ? bits0 + bits_m0 * (koffs[p] / 32) + (L.shared ? 0 : b) * sg.wpc : nullptr;
    sg.k12 = nullptr;
    sg.pad_ = 0;
    segs[p] = sg;
  }
  if (t == 0) {
    item_off[P] = ti;
    ablk_off[P] = L.shared ? 0 : ta;
    counts[0] = (int32_t)ti;
    counts[1] = (int32_t)ta;
    counts[2] = (int32_t)nch_all;
  }
}

__global__ void dp_items_write(DpList L, const int64_t* __restrict__ rows, int32_t P, int mode,
                               const int64_t* __restrict__ item_off,
                               const int64_t* __restrict__ ablk_off,
                               const int32_t* __restrict__ counts, VoteItem* items,
                               ABlock* ablocks, int64_t max_items, int64_t max_ablocks,
                               int32_t* err) {
  int64_t n_items = counts[0], n_ab = counts[1];
  const int64_t nch_all = counts[2];
  const int cpb = mode == 1 ? kTcM / 2 : kTcM;
  if (n_items > max_items || n_ab > max_ablocks) {  // invariant: the host's bound holds
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(err, 2);
    n_items = 0;
    n_ab = 0;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_items; g += stride) {
    const int p = find_problem(item_off, P, g);
    const int64_t local = g - item_off[p];
    const int64_t m = list_m(L, p), n = rows[p + 1] - rows[p];
    VoteItem it;
    it.seg = p;
    if (mode == 2) {
      const int64_t nc = (n + kExactChunk - 1) / kExactChunk;
      const int64_t cg = local / nc, c = local % nc;
      it.cell0 = (int32_t)(cg * kExactCells);
      it.ncell = (int32_t)i64min(kExactCells, m - cg * kExactCells);
      it.i0 = (int32_t)(c * kExactChunk);
      it.ni = (int32_t)i64min(kExactChunk, n - c * kExactChunk);
      it.ablk = 0;
    } else {
      const int64_t cb = (m + cpb - 1) / cpb, per = (m + cb - 1) / cb;
      const int64_t nt = (n + kTcN - 1) / kTcN;
      int64_t ct, nch;
      tc_chunks(nt, nch_all, &ct, &nch);
      const int64_t b = local % cb, c = local / cb;  // chunk-major (see build_tc_items)
      const int64_t c0 = b * per, t0 = c * ct;
      it.cell0 = (int32_t)c0;
      it.ncell = (int32_t)i64max(0, i64min(per, m - c0));
      it.i0 = (int32_t)(t0 * kTcN);
      it.ni = (int32_t)(i64max(0, i64min(ct, nt - t0)) * kTcN);
      it.ablk = (int32_t)(ablk_off[p] + b);
    }
    if (it.ncell < 1 || it.ncell > cpb || it.ni < 1) atomicOr(err, 4);  // invariant
    items[g] = it;
  }
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_ab; g += stride) {
    const int p = L.shared ? 0 : find_problem(ablk_off, P, g);
    const int64_t local = g - (L.shared ? 0 : ablk_off[p]);
    const int64_t m = list_m(L, p);
    const int64_t cb = (m + cpb - 1) / cpb, per = (m + cb - 1) / cb;
    ABlock a;
    a.seg = p;
    a.cell0 = (int32_t)(local * per);
    a.ncell = (int32_t)i64max(0, i64min(per, m - local * per));
    a.pad = 0;
    ablocks[g] = a;
  }
}

__global__ void __launch_bounds__(kPlanThreads) dp_scan(int32_t* cnt, int32_t P,
                                                        int64_t f3, int64_t* act,
                                                        int64_t* next_base, int64_t* total,
                                                        RediveCheck rc, OnePass op) {
  __shared__ int64_t sh[kPlanThreads];
  __shared__ int32_t s_abort;
  const int t = threadIdx.x;
  const int p0 = (int)((int64_t)P * t / kPlanThreads), p1 = (int)((int64_t)P * (t + 1) / kPlanThreads);
  for (int p = p0; p < p1; ++p) {
    if (rc.flags) {  // re-dive trigger (R18), once per problem
      const int32_t fl = (!rc.done[p] && rc.pcnt[p] > 0 && cnt[p] >= 16384 &&
                          2 * (int64_t)cnt[p] > (int64_t)rc.pcnt[p] * rc.f3) ? 1 : 0;
      rc.flags[p] = fl;
      if (fl) {
        rc.done[p] = 1;
        atomicOr(rc.any, rc.any_bit);
      }
    }
  }
  // one-pass solve: a raised error word (capacity, or the re-dive the one-pass loop does not
  // take) empties this level, so every later launch has nothing to do; the host redoes the solve
  if (t == 0) s_abort = op.err ? *reinterpret_cast<volatile int32_t*>(op.err) : 0;
  __syncthreads();
  const bool abort = s_abort != 0;
  int64_t v = 0;
  for (int p = p0; p < p1; ++p) {
    if (abort) cnt[p] = 0;
    v += cnt[p];
  }
  int64_t tot;
  int64_t e = cta_scan_excl(v, sh, &tot);
  auto clamp = [&](int64_t b) { return op.cap_lim > 0 && b > op.cap_lim ? op.cap_lim : b; };
  for (int p = p0; p < p1; ++p) {
    act[p] = e;
    if (next_base) next_base[p] = clamp(e * f3);
    e += cnt[p];
  }
  if (t == 0) {
    act[P] = tot;
    if (next_base) next_base[P] = clamp(tot * f3);
    *total = tot;
  }
}

// ---- one problem sharded over ranks: ordered (deterministic) lists -------------------------
// Every rank must hold the identical list to vote a contiguous slice of it, so the children
// are placed by a prefix over the parents instead of by atomics: count, scan, write.

// pcnt[g] = candidate children of parent g if it survives (UB >= lb), else 0
__global__ void dp_expand_count(const uint32_t* __restrict__ plins, int32_t shared_lins,
                                const int64_t* __restrict__ act_off,
                                const int64_t* __restrict__ pcap, const uint32_t* __restrict__ pub,
                                const int64_t* __restrict__ lb, int32_t P, int32_t Bp, int32_t f,
                                int32_t* pcnt) {
  const int64_t total = act_off[P];
  const int32_t Bc = Bp * f;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int p = find_problem(act_off, P, g);
    const int64_t e = g - act_off[p], idx = pcap[p] + e;
    int c = 0;
    if ((int64_t)pub[idx] >= lb[p]) {
      int32_t i, j, k;
      lin_to_ijk(shared_lins ? plins[e] : plins[idx], Bp, i, j, k);
      for (int a = 0; a < f; ++a)
        for (int b = 0; b < f; ++b)
          for (int d = 0; d < f; ++d) c += is_candidate(Bc, f * i + a, f * j + b, f * k + d) ? 1 : 0;
    }
    pcnt[g] = c;
  }
}

// exclusive prefix of v[0..n) into off[0..n] (one CTA)
__global__ void __launch_bounds__(kPlanThreads) dp_scan_i32(const int32_t* __restrict__ v,
                                                            const int64_t* __restrict__ n_dev,
                                                            int64_t* off) {
  __shared__ int64_t sh[kPlanThreads];
  const int64_t n = *n_dev;
  const int t = threadIdx.x;
  const int64_t i0 = n * t / kPlanThreads, i1 = n * (t + 1) / kPlanThreads;
  int64_t sum = 0;
  for (int64_t i = i0; i < i1; ++i) sum += v[i];
  int64_t tot;
  int64_t e = cta_scan_excl(sum, sh, &tot);
  for (int64_t i = i0; i < i1; ++i) {
    off[i] = e;
    e += v[i];
  }
  if (t == 0) off[n] = tot;
}

// children of parent g at ccap[p] + (off[g] - off[act_off[p]]), (a,b,c) order; count slots
// zeroed; ccnt[p] from the offsets
__global__ void dp_expand_write(const uint32_t* __restrict__ plins, int32_t shared_lins,
                                const int64_t* __restrict__ act_off,
                                const int64_t* __restrict__ pcap, const int32_t* __restrict__ pcnt,
                                const int64_t* __restrict__ off, int32_t P, int32_t Bp, int32_t f,
                                const int64_t* __restrict__ ccap, uint32_t* clins, uint32_t* ca,
                                uint32_t* cb, int32_t* ccnt) {
  const int64_t total = act_off[P];
  const int32_t Bc = Bp * f;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int p = find_problem(act_off, P, g);
    if (g == act_off[p]) ccnt[p] = (int32_t)(off[act_off[p + 1]] - off[act_off[p]]);
    if (pcnt[g] == 0) continue;
    const int64_t e = g - act_off[p], idx = pcap[p] + e;
    int32_t i, j, k;
    lin_to_ijk(shared_lins ? plins[e] : plins[idx], Bp, i, j, k);
    int64_t w = ccap[p] + off[g] - off[act_off[p]];
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b)
        for (int d = 0; d < f; ++d) {
          const int32_t ci = f * i + a, cj = f * j + b, ck = f * k + d;
          if (!is_candidate(Bc, ci, cj, ck)) continue;
          clins[w] = ijk_to_lin(ci, cj, ck, Bc);
          ca[w] = 0;
          cb[w] = 0;
          ++w;
        }
  }
}

// the slice [r * chunk, min((r + 1) * chunk, cnt[0])) of a one-problem list: base_out[0],
// cnt_out[0] (base_out[1] = base_out[0] + cnt_out[0] for the flat kernels' act layout)
__global__ void dp_slice(const int64_t* __restrict__ base, const int32_t* __restrict__ cnt,
                         int64_t shared_m, int64_t r0, int64_t chunk, int64_t* base_out,
                         int32_t* cnt_out) {
  const int64_t m = cnt ? (int64_t)cnt[0] : shared_m;
  const int64_t c = i64max(0, i64min(chunk, m - r0));
  base_out[0] = (base ? base[0] : 0) + r0;
  base_out[1] = base_out[0] + c;
  cnt_out[0] = (int32_t)c;
}

// lb[p] = max(lb[p], lb2[p])
__global__ void dp_lb_max(int64_t* lb, const int64_t* __restrict__ lb2, int32_t P) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x)
    if (lb2[p] > lb[p]) lb[p] = lb2[p];
}

// --- launchers ------------------------------------------------------------------------------
void dp_launch_dive_children(const uint32_t* pick, const int32_t* pick_idx,
                             const uint32_t* idx_list, int32_t Bp, int32_t f, uint32_t* out,
                             int32_t cap, int32_t* cnt, int32_t P, cudaStream_t s,
                             const int32_t* active, const Excl& ex, bool finest) {
  dp_dive_children<<<P, kDpThreads, 0, s>>>(pick, pick_idx, idx_list, Bp, f, out, cap, cnt,
                                            active, ex, finest ? 1 : 0);
}
void dp_launch_lb_max(int64_t* lb, const int64_t* lb2, int32_t P, cudaStream_t s) {
  dp_lb_max<<<(P + 255) / 256, 256, 0, s>>>(lb, lb2, P);
}
void dp_launch_dive_pick(const uint32_t* lins, const uint32_t* a, const int64_t* off,
                         const int32_t* cnt, int32_t B, double eps, const int64_t* rows,
                         uint32_t* pick, int32_t P, cudaStream_t s, const Excl& ex) {
  dp_dive_pick<<<P, kDpThreads, 0, s>>>(lins, a, off, cnt, B, eps, rows, pick, ex);
}
void dp_launch_max_lo(const uint32_t* b, const int64_t* off, const int32_t* cnt, int64_t* lb,
                      int32_t P, cudaStream_t s) {
  dp_max_lo<<<P, kDpThreads, 0, s>>>(b, off, cnt, lb);
}
void dp_launch_items(const DpList& L, const int64_t* rows, const int64_t* koffs, int32_t P,
                     int32_t B, double eps, int mode, int32_t slots, VoteSeg* segs,
                     int64_t* item_off, int64_t* ablk_off, int32_t* counts, VoteItem* items,
                     ABlock* ablocks, int64_t max_items, int64_t max_ablocks, int32_t* err,
                     cudaStream_t s, uint32_t* bits0, int64_t bits_m0) {
  dp_items_plan<<<1, kPlanThreads, 0, s>>>(L, rows, koffs, P, B, eps, mode, slots, segs, item_off,
                                          ablk_off, counts, bits0, bits_m0);
  dp_items_write<<<148 * 4, 256, 0, s>>>(L, rows, P, mode, item_off, ablk_off, counts, items,
                                         ablocks, max_items, max_ablocks, err);
}

void dp_items_bound(int mode, int64_t entries, int32_t P, int64_t nmax, int32_t slots,
                    int64_t* max_items, int64_t* max_ablocks) {
  if (mode == 2) {
    *max_items = std::max<int64_t>(1, entries * ((nmax + kExactChunk - 1) / kExactChunk));
    *max_ablocks = 1;
    return;
  }
  const int cpb = mode == 1 ? kTcM / 2 : kTcM;
  const int64_t cbs = entries / cpb + P + 1;  // sum of ceil(m_p / cpb)
  *max_items = std::max<int64_t>(cbs, (int64_t)64 * slots + cbs);
  *max_ablocks = cbs;
}

void dp_launch_scan(int32_t* cnt, int32_t P, int64_t f3, int64_t* act, int64_t* next_base,
                    int64_t* total, cudaStream_t s, const RediveCheck* rc, const OnePass* op) {
  dp_scan<<<1, kPlanThreads, 0, s>>>(cnt, P, f3, act, next_base, total,
                                    rc ? *rc : RediveCheck{nullptr, 0, nullptr, nullptr, nullptr, 1},
                                    op ? *op : OnePass{nullptr, 0});
}

namespace {
inline unsigned flat_grid(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}
}  // namespace

void dp_launch_bnb_expand(const uint32_t* plins, bool shared_lins, const int64_t* act_off,
                          const int64_t* pcap, const uint32_t* pub, const int64_t* lb, int32_t P,
                          int64_t total, int32_t Bp, int32_t f, const int64_t* ccap,
                          uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                          int32_t* err, cudaStream_t s, const Own& own, const Excl& ex,
                          bool finest, const TailScan& ts) {
  dp_bnb_expand<<<flat_grid(total), 256, 0, s>>>(plins, shared_lins ? 1 : 0, act_off, pcap, pub,
                                                 lb, P, Bp, f, ccap, clins, ca, cb, ccnt, err, own,
                                                 ex, finest ? 1 : 0, ts);
}

// ---- one problem over ranks, each searching the subtrees it owns (the one-pass sharded solve)
// slot r of (best, ties) = rank r's finest-level winner key and its tie count; the merge takes the
// largest key and sums the ties of the ranks whose winning count equals it
__global__ void dp_merge_rank_winners(const unsigned long long* __restrict__ best_r,
                                      const int32_t* __restrict__ ties_r, int32_t W,
                                      unsigned long long* best, int32_t* ties) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long b = 0;
  for (int r = 0; r < W; ++r) b = best_r[r] > b ? best_r[r] : b;
  int32_t t = 0;
  for (int r = 0; r < W; ++r)
    if (best_r[r] && (best_r[r] >> 32) == (b >> 32)) t += ties_r[r];
  *best = b;
  *ties = t;
}
void dp_launch_merge_rank_winners(const unsigned long long* best_r, const int32_t* ties_r,
                                  int32_t W, unsigned long long* best, int32_t* ties,
                                  cudaStream_t s) {
  dp_merge_rank_winners<<<1, 32, 0, s>>>(best_r, ties_r, W, best, ties);
}
__global__ void dp_add_i32(int32_t* dst, const int32_t* __restrict__ src) { *dst += *src; }
void dp_launch_add_i32(int32_t* dst, const int32_t* src, cudaStream_t s) {
  dp_add_i32<<<1, 1, 0, s>>>(dst, src);
}
void dp_launch_expand_ordered(const uint32_t* plins, bool shared_lins, const int64_t* act_off,
                              const int64_t* pcap, const uint32_t* pub, const int64_t* lb,
                              int32_t P, int64_t total, int32_t Bp, int32_t f, const int64_t* ccap,
                              uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                              int32_t* pcnt, int64_t* off, cudaStream_t s) {
  dp_expand_count<<<flat_grid(total), 256, 0, s>>>(plins, shared_lins ? 1 : 0, act_off, pcap, pub,
                                                   lb, P, Bp, f, pcnt);
  dp_scan_i32<<<1, kPlanThreads, 0, s>>>(pcnt, act_off + P, off);
  dp_expand_write<<<flat_grid(total), 256, 0, s>>>(plins, shared_lins ? 1 : 0, act_off, pcap,
                                                   pcnt, off, P, Bp, f, ccap, clins, ca, cb, ccnt);
}
void dp_launch_slice(const int64_t* base, const int32_t* cnt, int64_t shared_m, int64_t r0,
                     int64_t chunk, int64_t* base_out, int32_t* cnt_out, cudaStream_t s) {
  dp_slice<<<1, 1, 0, s>>>(base, cnt, shared_m, r0, chunk, base_out, cnt_out);
}
void dp_launch_final_max(const int64_t* act_off, const int64_t* cap, const uint32_t* lo, int32_t P,
                         int64_t total, uint32_t* Lmax, cudaStream_t s) {
  dp_final_max<<<flat_grid(total), 256, 0, s>>>(act_off, cap, lo, P, Lmax);
}
void dp_launch_final_split(const int64_t* act_off, const int64_t* cap, const uint32_t* lins,
                           const uint32_t* hi, const uint32_t* lo, const uint32_t* Lmax, int32_t P,
                           int64_t total, unsigned long long* best, uint32_t* rlins, int32_t* rcnt,
                           cudaStream_t s) {
  dp_final_split<<<flat_grid(total), 256, 0, s>>>(act_off, cap, lins, hi, lo, Lmax, P, best, rlins,
                                                  rcnt);
}
void dp_launch_final_rechecked(const int64_t* act_off, const int32_t* rcnt, const uint32_t* rlins,
                               const uint32_t* ex, int32_t P, int64_t total,
                               unsigned long long* best, cudaStream_t s) {
  dp_final_rechecked<<<flat_grid(total), 256, 0, s>>>(act_off, rcnt, rlins, ex, P, best);
}
void dp_launch_final_ties(const int64_t* act_off, const int64_t* cap, const uint32_t* hi,
                          const uint32_t* lo, const int32_t* rcnt, const uint32_t* ex, int32_t P,
                          int64_t total, const unsigned long long* best, int32_t* ties,
                          cudaStream_t s) {
  dp_final_ties<<<flat_grid(2 * total), 256, 0, s>>>(act_off, cap, hi, lo, rcnt, ex, P, best, ties);
}

}  // namespace rv
