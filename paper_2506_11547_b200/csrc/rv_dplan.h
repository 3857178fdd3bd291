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
// BnB children of parents with UB >= lb[p] (count pass: out == nullptr -> ccnt; write pass
// at out + coff[p]); shared_m > 0: every problem's parents are the shared list lins[0..m)
// with UBs at ub + p*shared_m
void dp_launch_bnb_children(const uint32_t* lins, const int64_t* poff, const uint32_t* ub,
                            const int64_t* uoff, const int32_t* pcnt, int64_t shared_m,
                            const int64_t* lb, int32_t Bp, int32_t f, uint32_t* out,
                            const int64_t* coff, int32_t* ccnt, int32_t P, cudaStream_t s);
// finest level: recheck set (count pass rlist == nullptr -> rcnt; write pass: positions)
void dp_launch_recheck_set(const uint32_t* hi, const uint32_t* lo, const int64_t* off,
                           const int32_t* cnt, int32_t* rcnt, const int64_t* roff, int32_t* rlist,
                           int32_t P, cudaStream_t s);
void dp_launch_gather(const uint32_t* lins, const int64_t* off, const int64_t* roff,
                      const int32_t* rcnt, const int32_t* rlist, uint32_t* rlins, int32_t P,
                      cudaStream_t s);
// res[3p..3p+2] = {winner lin, votes, n_tied}
void dp_launch_finalize(const uint32_t* lins, const uint32_t* hi, const uint32_t* lo,
                        const int64_t* off, const int32_t* cnt, const uint32_t* ex,
                        const int64_t* roff, const int32_t* rcnt, const int32_t* rlist,
                        int32_t* res, int32_t P, cudaStream_t s);

}  // namespace rv
