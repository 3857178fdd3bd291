// rv_dplan.h -- launchers of the device-resident batched level loop (rv_dplan.cu).
// Per-problem lists live in flat device arrays: problem p's list starts at off[p] and has
// cnt[p] entries; counts arrays use the same layout as the lists they belong to.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace rv {

// dive: candidate children (Bc = f*Bp) of the 27-neighbourhood of the pick (pick[p], or
// idx_list[pick_idx[p]] if idx_list != nullptr), at out + p*cap
void dp_launch_dive_children(const uint32_t* pick, const int32_t* pick_idx,
                             const uint32_t* idx_list, int32_t Bp, int32_t f, uint32_t* out,
                             int32_t cap, int32_t* cnt, int32_t P, cudaStream_t s);
// dive: pick[p] = the list's max-excess block (planner key)
void dp_launch_dive_pick(const uint32_t* lins, const uint32_t* a, const int64_t* off,
                         const int32_t* cnt, int32_t B, double eps, const int64_t* rows,
                         uint32_t* pick, int32_t P, cudaStream_t s);
// lb[p] = max cnt_b of the list
void dp_launch_max_lo(const uint32_t* b, const int64_t* off, const int32_t* cnt, int64_t* lb,
                      int32_t P, cudaStream_t s);
// Flat list kernels (one thread per entry; entries of problem p: act_off[p]..act_off[p+1]
// stored from cap[p]).  BnB expand: candidate children of parents with UB >= lb[p] into the
// child region ccap[p] (ccnt zeroed by the caller; the children's count slots are zeroed).
void dp_launch_bnb_expand(const uint32_t* plins, bool shared_lins, const int64_t* act_off,
                          const int64_t* pcap, const uint32_t* pub, const int64_t* lb, int32_t P,
                          int64_t total, int32_t Bp, int32_t f, const int64_t* ccap,
                          uint32_t* clins, uint32_t* ca, uint32_t* cb, int32_t* ccnt,
                          cudaStream_t s);
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

}  // namespace rv
