// rv_dplan.h -- launchers of the device-resident batched level loop (rv_dplan.cu).
// Per-problem lists live in flat device arrays: problem p's list starts at off[p] and has
// cnt[p] entries; counts arrays use the same layout as the lists they belong to.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

#include "rv_kernels.h"

namespace rv {

// A level's per-problem block lists on the device: problem p's list is lins + base[p]
// (shared: every problem's list is lins[0 .. shared_m)), cnt[p] entries (cnt == nullptr:
// shared_m each); its counts live at ca / cb + base[p].
struct DpList {
  const uint32_t* lins;
  int32_t shared;
  int64_t shared_m;
  const int64_t* base;
  const int32_t* cnt;
  uint32_t* ca;
  uint32_t* cb;
};

// Device-built vote decomposition (same rules as build_tc_items / build_exact_items):
// mode 0 = K3-TC bound (<= kTcM cells per item), 1 = K3-TC final (kTcM/2), 2 = K5 exact
// (one cell per item, 8192-correspondence chunks).  Writes segs[P] (koffs: the TC table
// offsets for modes 0/1, the K table offsets for mode 2), items, ablocks and
// counts = {n_items, n_ablocks, chunks}; item_off / ablk_off: scratch [P+1].  The caller
// sizes items / ablocks from a bound (dp_items_bound).  bits0 (mode 0 on the level-0 grid, or
// a rank's slice of a one-problem grid): the segments carry the level-0 pass bitmasks K3-TC
// writes (rv_cull.cu), bits_m0 rows per problem.
// err: invariant violations are OR-ed in (1 child capacity, 2 item bound, 4 item shape); the
// host checks the word once at the end of the solve (there are no silent out-of-bounds writes).
void dp_launch_items(const DpList& L, const int64_t* rows, const int64_t* koffs, int32_t P,
                     int32_t B, double eps, int mode, int32_t slots, VoteSeg* segs,
                     int64_t* item_off, int64_t* ablk_off, int32_t* counts, VoteItem* items,
                     ABlock* ablocks, int64_t max_items, int64_t max_ablocks, int32_t* err,
                     cudaStream_t s, uint32_t* bits0 = nullptr, int64_t bits_m0 = 0);
// items / ablocks needed for at most `entries` list entries over P problems of <= nmax rows
void dp_items_bound(int mode, int64_t entries, int32_t P, int64_t nmax, int32_t slots,
                    int64_t* max_items, int64_t* max_ablocks);
// The re-dive trigger (R18) evaluated by the scan: flags[p] = !done[p] && pcnt[p] > 0 &&
// cnt[p] >= 16384 && 2 cnt[p] > pcnt[p] * f3 (then done[p] = 1, *any |= 1)
struct RediveCheck {
  const int32_t* pcnt;
  int64_t f3;
  int32_t* done;
  int32_t* flags;
  int32_t* any;
  int32_t any_bit;  // OR-ed into *any when a problem triggers
};
// One-pass single solve (no host round trip per level): err = the solve's error word -- when it
// is nonzero the scan empties the level (counts and offsets 0), so the rest of the solve does
// nothing and the host redoes it with per-level round trips; cap_lim > 0 clamps next_base to
// the fixed capacity of the next level's arrays (one problem: its region is [0, cap_lim)).
struct OnePass {
  int32_t* err;
  int64_t cap_lim;
};
// act[p] = exclusive prefix of cnt (act[P] = total, also written to *total); next_base[p] =
// act[p] * f3 (optional); rc: also evaluate the re-dive trigger
void dp_launch_scan(int32_t* cnt, int32_t P, int64_t f3, int64_t* act, int64_t* next_base,
                    int64_t* total, cudaStream_t s, const RediveCheck* rc = nullptr,
                    const OnePass* op = nullptr);

// dive: candidate children (Bc = f*Bp) of the 27-neighbourhood of the pick (pick[p], or
// idx_list[pick_idx[p]] if idx_list != nullptr), at out + p*cap
// (active != nullptr: problems with active[p] == 0 get an empty list -- the re-dive)
void dp_launch_dive_children(const uint32_t* pick, const int32_t* pick_idx,
                             const uint32_t* idx_list, int32_t Bp, int32_t f, uint32_t* out,
                             int32_t cap, int32_t* cnt, int32_t P, cudaStream_t s,
                             const int32_t* active = nullptr, const Excl& ex = Excl(),
                             bool finest = false);
// lb[p] = max(lb[p], lb2[p])
void dp_launch_lb_max(int64_t* lb, const int64_t* lb2, int32_t P, cudaStream_t s);
// dive: pick[p] = the list's max-excess block (planner key)
void dp_launch_dive_pick(const uint32_t* lins, const uint32_t* a, const int64_t* off,
                         const int32_t* cnt, int32_t B, double eps, const int64_t* rows,
                         uint32_t* pick, int32_t P, cudaStream_t s, const Excl& ex = Excl());
// lb[p] = max cnt_b of the list
void dp_launch_max_lo(const uint32_t* b, const int64_t* off, const int32_t* cnt, int64_t* lb,
                      int32_t P, cudaStream_t s);
// Subtree ownership of a one-problem search over ranks: a block belongs to the rank owning the
// ancestor group of its level-0 (resolution B0) ancestor, lut[B0 lin] = group, owned groups
// [lo, hi).  lut == nullptr: everything.
struct Own {
  const int32_t* lut = nullptr;
  int32_t B0 = 0;
  int64_t lo = 0, hi = 0;
};
// One problem (P == 1): the level's scan run by the expansion's last CTA (no separate launch):
// act = {0, c}, next_base = {0, min(c f3, cap_lim)}, *total = c, the phase slot, the re-dive check
// and the one-pass error word as dp_scan does (c = *ccnt, 0 when the word is raised).  done: a
// zeroed counter the last CTA resets.
struct TailScan {
  uint32_t* done = nullptr;   // nullptr: no tail scan
  int64_t f3 = 1;
  int64_t* act = nullptr;
  int64_t* next_base = nullptr;
  int64_t* total = nullptr;
  int32_t* phase = nullptr;    // the phase slot: = c, or += c when phase_add (ranks' subtrees)
  int32_t phase_add = 0;
  int32_t* zero_next = nullptr;  // a count to zero after the re-dive check (the next level's)
  int32_t* zero_buf = nullptr;   // zeroed by the whole grid first (the cull bucket counters)
  int64_t zero_n = 0;
  RediveCheck rc{nullptr, 0, nullptr, nullptr, nullptr, 1};
  OnePass op{nullptr, 0};
};
// best = max_r best_r, ties = sum of ties_r over the ranks whose count equals best's (one thread)
void dp_launch_merge_rank_winners(const unsigned long long* best_r, const int32_t* ties_r,
                                  int32_t W, unsigned long long* best, int32_t* ties,
                                  cudaStream_t s);
// *dst += *src (one thread: per-rank phase counts summed in order)
void dp_launch_add_i32(int32_t* dst, const int32_t* src, cudaStream_t s);
// Flat list kernels (one thread per entry; entries of problem p: act_off[p]..act_off[p+1]
// stored from cap[p]).  BnB expand: candidate children of parents with UB >= lb[p] into the
// child region ccap[p] (ccnt zeroed by the caller; the children's count slots are zeroed).
void dp_launch_bnb_expand(const uint32_t* plins, bool shared_lins, const int64_t* act_off,
                          const int64_t* pcap, const uint32_t* pub, const int64_t* lb, int32_t P,
                          int64_t total, int32_t Bp, int32_t f, const int64_t* ccap,
                          uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                          int32_t* err, cudaStream_t s, const Own& own = Own(),
                          const Excl& ex = Excl(), bool finest = false,
                          const TailScan& ts = TailScan());
// Ordered BnB expansion (one problem sharded over ranks: every rank builds the identical
// list): per-parent child counts into pcnt[total parents], their prefix into off[total + 1],
// then the children in parent order.
void dp_launch_expand_ordered(const uint32_t* plins, bool shared_lins, const int64_t* act_off,
                              const int64_t* pcap, const uint32_t* pub, const int64_t* lb,
                              int32_t P, int64_t total, int32_t Bp, int32_t f, const int64_t* ccap,
                              uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                              int32_t* pcnt, int64_t* off, cudaStream_t s);
// rank slice of a one-problem list: entries [r0, r0 + chunk) clipped to its length (cnt[0],
// or shared_m when cnt == nullptr); base_out[2] = {start, end}, cnt_out[0] = length
void dp_launch_slice(const int64_t* base, const int32_t* cnt, int64_t shared_m, int64_t r0,
                     int64_t chunk, int64_t* base_out, int32_t* cnt_out, cudaStream_t s);
// finest level: Lmax[p] = max lo; split into exact-known (offered to best[p], a packed
// (count << 32 | ~lin) max) and recheck lists (rlins at act_off[p], rcnt[p]); after the
// exact recheck (counts ex, same layout as rlins) the rechecked offer theirs; ties counted.
void dp_launch_final_max(const int64_t* act_off, const int64_t* cap, const uint32_t* lo, int32_t P,
                         int64_t total, uint32_t* Lmax, cudaStream_t s);
void dp_launch_final_split(const int64_t* act_off, const int64_t* cap, const uint32_t* lins,
                           const uint32_t* hi, const uint32_t* lo, const uint32_t* Lmax, int32_t P,
                           int64_t total, unsigned long long* best, uint32_t* rlins, int32_t* rcnt,
                           cudaStream_t s);
void dp_launch_final_rechecked(const int64_t* act_off, const int32_t* rcnt, const uint32_t* rlins,
                               const uint32_t* ex, int32_t P, int64_t total,
                               unsigned long long* best, cudaStream_t s);
void dp_launch_final_ties(const int64_t* act_off, const int64_t* cap, const uint32_t* hi,
                          const uint32_t* lo, const int32_t* rcnt, const uint32_t* ex, int32_t P,
                          int64_t total, const unsigned long long* best, int32_t* ties,
                          cudaStream_t s);


// Item planner of K3-C for a level's per-problem lists: the entries bucketed by (problem,
// level-0 ancestor) (lut0: level-0 lin at resolution B0 -> bitmask row, -1 if not a
// candidate), items of <= 32 blocks of a bucket x ranges of the ancestor's index list (l0cnt:
// the list lengths = level-0 counts, lofs: their row offsets; ~8 items per resident warp);
// segs[p] get the problem's k12 rows.  Scratch sizes: act P+1, acnt P*m0, aoff / ioff P*m0+1, tanc / tslot / cidx T,
// phi 12 T floats, counts 2, work 1 (T = the level's total entries).
struct CullScratch {
  int64_t* act;
  int32_t* acnt;
  int64_t* aoff;
  int64_t* ioff;
  int32_t* tanc;
  int32_t* tslot;
  int32_t* cidx;
  float* phi;
  int32_t* counts;
  int32_t* work;
  uint8_t* tphi;    // K3-CT: the blocks' 64-byte fp16-split rows (nullptr: FP32 K3-C only)
  float tc_guard;   // the guard of those rows' thresholds (guard + the TC error margin)
  int32_t ct_na;    // K3-CT: A blocks of 128 rows per item (1 or 2)
};
// A dive level of the one-pass solve folded into the small planner's CTA (one launch instead of
// pick + children + zeroing + phase copy + planning): pick over the previous dive level's list
// (prev_lins / prev_a / prev_off[0] / prev_cnt[0] at resolution pickB; prev_lins == nullptr:
// the level-0 start grid_list[l0idx[0]]), the ordered children of its neighbourhood at
// Bc = f Bp into out (cap, count *out_cnt, also *phase), their count slots ca / cb (cb may be
// null) zeroed.  The planner then plans the new list (L must describe out / out_cnt / ca / cb).
struct DiveStep {
  int32_t on = 0;
  const uint32_t* prev_lins = nullptr;
  const uint32_t* prev_a = nullptr;
  const int64_t* prev_off = nullptr;
  const int32_t* prev_cnt = nullptr;
  int32_t pickB = 0;
  const int32_t* l0idx = nullptr;
  const uint32_t* grid_list = nullptr;
  uint32_t* pick_out = nullptr;
  Excl ex;
  int32_t finest = 0;
  int32_t Bp = 0, f = 0, cap = 0;
  uint32_t* out = nullptr;
  int32_t* out_cnt = nullptr;
  uint32_t* ca = nullptr;
  uint32_t* cb = nullptr;
  int32_t* phase = nullptr;
};
// returns the number of kernels it launched (one CTA does everything for small levels)
// own_lo .. own_hi: the level-0 rows (ancestors) this rank votes (blocks of other ancestors
// are left at zero for the count all-reduce).  pre_act: the lists' prefix (act[0..P]) already
// on the device and the bucket counters (P * m0) already zeroed -- the one-problem branch and
// bound, whose expansion does both (TailScan) -- so the act launch is skipped
int launch_cull_items(const DpList& L, const int64_t* rows, const int64_t* toffs, int32_t P,
                      int32_t B, int32_t B0, const int32_t* lut0, int64_t m0,
                      const uint32_t* l0cnt, const int64_t* lofs, const float* k12, double eps,
                      int mode, float guard, int num_sms, const CullScratch& cs, VoteSeg* segs,
                      CullItem* items, int64_t entries_bound, int64_t max_items, int32_t* err,
                      cudaStream_t s, int64_t own_lo = 0, int64_t own_hi = INT64_MAX,
                      const DiveStep* dive = nullptr, const int64_t* pre_act = nullptr);
// items needed for at most `entries` list entries
int64_t cull_items_bound(int64_t entries, int num_sms);

}  // namespace rv
