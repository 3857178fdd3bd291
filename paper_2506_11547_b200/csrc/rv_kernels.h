// rv_kernels.h -- device-side descriptors and launchers of librotvote's sm_100a kernels.
#pragma once
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

#include "rv_geom.h"

namespace rv {

// Kernel attributes (the dynamic shared-memory opt-in) are per device: a launcher sets them the
// first time it runs on each device of the process.  Racing threads may both set them
// (idempotent).
inline bool first_launch_on_device(std::atomic<uint64_t>& done) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return false;
  return true;
}
inline void mark_device_done(std::atomic<uint64_t>& done) {
  int d = 0;
  cudaGetDevice(&d);
  done.fetch_or(1ull << (d & 63), std::memory_order_release);
}


#ifndef RV_CPT
#define RV_CPT 4
#endif
#ifndef RV_TILE
#define RV_TILE 256
#endif
#ifndef RV_STAGES
#define RV_STAGES 4
#endif
#ifndef RV_VOTERS
#define RV_VOTERS 256
#endif
#ifndef RV_MINB
#define RV_MINB 2
#endif
#ifndef RV_PIPE
#define RV_PIPE 0   // 0: thread 0 refills a stage after a block barrier; 1: producer warp + mbarriers
#endif
#ifndef RV_TC_COUNT_ALU_ONLY
#define RV_TC_COUNT_ALU_ONLY 1
#endif
#ifndef RV_COUNT_ASM
#define RV_COUNT_ASM 1
#endif
constexpr int kVoteThreads = RV_VOTERS;            // K3 voting threads (+1 producer warp)
constexpr int kVoteMinBlocks = RV_MINB;            // K3 CTAs per SM the registers are sized for
constexpr int kProducerThreads = RV_PIPE ? 32 : 0; // dedicated TMA producer warp
constexpr int kCellsPerThread = RV_CPT;            // K3 register blocking (cells per thread)
constexpr int kCellsPerBlock = kVoteThreads * kCellsPerThread;
constexpr int kTile = RV_TILE;                     // correspondences per TMA stage
constexpr int kStages = RV_STAGES;
#ifndef RV_TC_N
#define RV_TC_N 256
#endif
constexpr int kTcN = RV_TC_N;                      // K3-TC: correspondences per tile (MMA N)
constexpr int kTcAcc = 512 / kTcN;                 // K3-TC: TMEM accumulator buffers (512 columns)
constexpr int kTcM = 128;                          // K3-TC: cells per CTA (MMA M, TMEM lanes)
constexpr int kTcStages = 7;                       // K3-TC: 16 KB tiles in flight (also pins 1 CTA/SM)
constexpr int kRefThreads = 256;                   // K6/K7 block
#ifndef RV_REF_ROWS
#define RV_REF_ROWS 4096
#endif
constexpr int kRefRowsPerItem = RV_REF_ROWS;       // K6 rows per block (multiple of 32)

// One problem's block list for a vote launch.
struct VoteSeg {
  const uint32_t* lins;  // DEVICE block indices (lin at resolution B)
  uint32_t* cnt_a;       // DEVICE counts (indexed like lins)
  uint32_t* cnt_b;       // DEVICE second counts (RV_MODE_FINAL) or nullptr
  int64_t koff;          // offset of the problem's rows in the 9-row K table (multiple of 4)
  int64_t row;           // offset of the problem's rows in x, y
  int32_t n;             // correspondences of the problem
  int32_t B;             // grid resolution of lins
  double eps;            // inlier angle
  // ancestor culling (rv_cull.cu): the level-0 pass bitmasks of the problem (row r = level-0
  // block r, wpc words per row, bit i%32 of word i/32 = correspondence i passed that block's
  // bound test) and its 48-byte K rows; K3-TC with bits != nullptr writes the bitmasks
  uint32_t* bits;
  const float* k12;      // [n_pad][12] fp32: the 9 entries of K1, then 3 zeros
  int32_t wpc;           // words per bitmask row (= the problem's padded rows / 32)
  int32_t pad_;
};

// K3-C work item: the ncell (<= 32) blocks at bucket positions [pos0, pos0 + ncell) of the
// level's bucket order (phi rows and list indices there), all of problem seg and one level-0
// ancestor, against the entries [e0, e0 + ne) of that ancestor's index list (a range of
// its row in the compacted level-0 lists).
struct CullItem {
  int32_t seg, pos0, ncell, ne;
  int64_t e0;
};
constexpr int kCullMaxCells = 32;    // blocks per K3-C item

// One thread block of work: blocks [cell0, cell0+ncell) of segment seg against
// correspondences [i0, i0+ni) of it (i0, ni multiples of 4; rows >= n are zero padding).
// ablk (K3-TC only): the item's block of the A-operand table (launch_vote_tc).
struct VoteItem {
  int32_t seg, cell0, ncell, i0, ni, ablk;
};
constexpr int kExactCells = 8;  // blocks per K5 item (each K row read once for all of them)

// K3-TC A-operand block: rows of cells [cell0, cell0+ncell) of segment seg (8 KB in the table).
struct ABlock {
  int32_t seg, cell0, ncell, pad;
};

// One problem of a refinement launch.
struct RefSeg {
  int64_t row;           // offset of the problem's rows in x, y
  int64_t mask_word;     // offset of the problem's mask in the mask buffer (words)
  int32_t n;
  int32_t item_begin, item_end;  // its K6 items
  int32_t pad;
  double tau;            // cos(eps)
};
struct RefItem {
  int32_t seg, r0, nr;   // rows [r0, r0+nr) of the problem, r0 % 32 == 0
};

// K1: normalise + 9-entry K table (fp64 -> fp32), zero padding to pad4(n) per problem.
// koffs[P+1] DEVICE padded offsets, rows[P+1] DEVICE row offsets.  bad: DEVICE int64,
// atomicMin of the first row that cannot be normalised (init to INT64_MAX).
void launch_setup(const float* x, const float* y, const int64_t* rows, const int64_t* koffs,
                  int32_t P, int64_t total_pad, float* k9, int64_t stride,
                  unsigned long long* bad, cudaStream_t s);

// K3: fp32 FFMA2 vote over TMA-staged K tiles.  mode RV_MODE_BOUND / RV_MODE_FINAL;
// groups in {1, 2, 4}: a CTA covers kCellsPerBlock / groups cells.
void launch_vote(int mode, int groups, const float* k9, int64_t stride, const VoteSeg* segs,
                 const VoteItem* items, int32_t n_items, float guard, cudaStream_t s);

// K1-TC: fp16-split correspondence table for the tensor-core vote (64 B per row,
// interleaved K-major layout, each problem padded to a multiple of kTcN rows).
// k12 != nullptr: also the 48-byte fp32 K rows of the culled vote ([toffs rows][12], the same
// fp64 -> fp32 rounding as K1); tab_rm != nullptr: the table's rows again, row-major (64 B each,
// contiguous: K3-CT's gather source).
// K1 fused into K1-TC for one problem (P == 1, rows 0 .. n): also K1's fp32 table (k9 [9][stride],
// rows g < n_pad, zero padding) and its data check (bad); k9 == nullptr: K1-TC alone
struct K9Out {
  float* k9 = nullptr;
  int64_t stride = 0, n_pad = 0;
  unsigned long long* bad = nullptr;
};
void launch_setup_tc(const float* x, const float* y, const int64_t* rows, const int64_t* toffs,
                     int32_t P, int64_t total_pad, uint8_t* tab, cudaStream_t s,
                     float* k12 = nullptr, uint8_t* tab_rm = nullptr, const K9Out& k9o = K9Out());

// K3-TC: BOUND-mode vote on tcgen05 (items: ncell <= kTcM, i0/ni multiples of kTcN, koff
// in table rows); final_mode: RV_MODE_FINAL counts at tau -/+ guard (items: ncell <= kTcM/2).
// Two launches: K2-TC writes the A-operand table (8 KB per ABlock, kTcABlockBytes) into
// atab, then the persistent vote kernel (item.ablk selects its A block).  dump != nullptr
// writes the raw scores S' = s - t instead of counting (test hook):
// dump[cell * dump_ld + correspondence].
constexpr int64_t kTcABlockBytes = 128 * 64;
// counts_dev != nullptr: {n_items, n_ablocks} are read on the device (device-built items;
// the host arguments are ignored and the grids are fixed).
void launch_vote_tc(const uint8_t* tab, uint8_t* atab, const ABlock* ablocks, int32_t n_ablocks,
                    const VoteSeg* segs, const VoteItem* items, int32_t n_items, float guard,
                    float* dump, int64_t dump_ld, cudaStream_t s, bool final_mode = false,
                    const int32_t* counts_dev = nullptr, bool emit_bits = false);

// K3-C (rv_cull.cu): the culled vote.  mode RV_MODE_BOUND / RV_MODE_FINAL; counts_dev[0] =
// item count (device); work counter: zeroed by the item planner; pairs: += evaluated pairs.
// phi / cidx: the planner's bucket-order block rows and list indices; lidx: the level-0 index
// lists (cull_compact).
void launch_vote_cull(int mode, const VoteSeg* segs, const CullItem* items,
                      const int32_t* counts_dev, int32_t* work, unsigned long long* pairs,
                      const float* phi, const int32_t* cidx, const uint32_t* lidx, float guard,
                      int num_sms, cudaStream_t s);
// K3-CT (rv_cull.cu): the culled vote on the tensor cores (same items and planner as K3-C;
// needs the planner's fp16-split block rows tphi).  tab: the K1-TC table, pad_row: a padding
// row of it (score -1).
void launch_vote_cull_tc(int mode, const VoteSeg* segs, const CullItem* items,
                         const int32_t* counts_dev, const uint8_t* tab, int64_t pad_row,
                         const uint8_t* tphi, const int32_t* cidx, const uint32_t* lidx,
                         unsigned long long* pairs, int num_sms, cudaStream_t s,
                         int32_t* work,  // the planner's zeroed work counter
                         bool static_order = false);  // rv_config.ct_sched == 1
// Level-0 index lists: row offsets lofs[P*m0 + 1] (exclusive prefix of the level-0 counts, each
// padded to a multiple of 4; lofs[P*m0] = the total), then the compaction of the K3-TC bitmasks
// (bits0: problem p's rows from m0 * toffs[p] / 32, (toffs[p+1] - toffs[p]) / 32 words each).
// Ancestor groups (K3-CT): list row g of a problem is the union of the level-0 rows
// gmem[goff[g] .. goff[g+1]), G rows per problem; goff == nullptr: one row per level-0 row.
struct CullGroups {
  const int32_t* goff = nullptr;
  const int32_t* gmem = nullptr;
  int64_t G = 0;
};
void launch_cull_rows(const uint32_t* l0cnt, int32_t P, int64_t m0, int64_t* lofs,
                      cudaStream_t s, const CullGroups& gr = CullGroups());
// (any order within a row; fill: scratch [P*m0] int32; rows [row_lo, row_hi) only: the rows
// this rank voted at level 0)
void launch_cull_compact(const uint32_t* bits0, const int64_t* toffs, int32_t P, int64_t m0,
                         int64_t wpc_max, const int64_t* lofs, int32_t* fill, uint32_t* lidx,
                         cudaStream_t s, int64_t row_lo = 0, int64_t row_hi = INT64_MAX,
                         const CullGroups& gr = CullGroups(), int64_t cap = 0,
                         int32_t* err = nullptr);
// (cap > 0: lists longer than cap entries in total raise bit 16 of *err and write nothing)
// L2 prefetch of [p, p + bytes) (cp.async.bulk.prefetch.L2, 16 KB per request)
void launch_l2_prefetch(const void* p, int64_t bytes, cudaStream_t s);


// K4 (batched): level-0 reductions, one CTA per problem.  argmax: the dive's start index per
// problem (planner key, see rv_plan_feed_l0_start).  survivors: outc != nullptr counts the
// blocks with UB >= lb[j] of problem problems[j]; otherwise writes their indices ascending at
// out + off[j].
void launch_l0_argmax(const uint32_t* cnt, int64_t m0, const uint32_t* lins, int32_t B,
                      const double* bg, const int64_t* rows, int32_t P, int32_t* out,
                      cudaStream_t s, const Excl& ex = Excl());
void launch_l0_survivors(const uint32_t* cnt, int64_t m0, const int32_t* problems,
                         const int64_t* lb, const int64_t* off, int32_t J, int32_t* outc,
                         int32_t* out, cudaStream_t s);

// K5: exact counts (fp32 vote + fp64 recheck of |s32 - tau| < guard).  items: one block
// per (block, correspondence chunk), ncell == 1.
// n_dev != nullptr: the item count is read on the device (n_items ignored; fixed grid).
void launch_exact(const float* k9, int64_t stride, const float* x, const float* y,
                  const VoteSeg* segs, const VoteItem* items, int32_t n_items, float guard,
                  cudaStream_t s, const int32_t* n_dev = nullptr);

// K6: fp64 inlier test at qs[seg] + partial sums of K over inliers (+ mask words).
void launch_inliers(const float* x, const float* y, const RefSeg* segs, const RefItem* items,
                    int32_t n_items, const double* qs, uint32_t* masks, double* partials,
                    cudaStream_t s);

// K7: per problem, reduce the partials in fixed order; mode 0: top-eigenvector refinement
// step (cyclic Jacobi, fp64) updating qs/flags; mode 1: write the inlier count only.
void launch_eig(const RefSeg* segs, int32_t P, const double* partials, double* qs,
                int32_t* flags, uint32_t* ninl, int mode, cudaStream_t s);

// K6+K7 fused for one problem (cooperative launch, grid-wide barriers between the passes):
// `rounds` refinement rounds from q0 (HOST-independent: q0 != nullptr DEVICE double[4], else the
// centre of the winner decoded from *best at resolution B), then the final mask / count.
// Writes q[4], *flags (RV_REFINED | RV_DEGENERATE), *ninl, mask (DEVICE, may be null).
// partials: DEVICE double [ceil(n / kRefRowsPerItem) * 10].
constexpr int kRefine1MaxCtas = 148 * 8;
struct Refine1Args {
  const float* x;
  const float* y;
  int64_t n;
  const float* k9;       // K1's fp32 table [9][stride] of this problem
  int64_t stride;
  double tau;            // cos(eps)
  float guard;           // fp32 screening band (>= 2.7e-6, R10)
  int32_t rounds;
  const unsigned long long* best;
  int32_t B;
  const double* q0;
  double* partials;
  double* q;
  int32_t* flags;
  uint32_t* ninl;
  uint32_t* mask;
  uint32_t* bar;         // DEVICE grid-barrier counter, zeroed by launch_refine1
};
cudaError_t launch_refine1(const Refine1Args& a, int num_sms, cudaStream_t s);
// qs[4p..] = canonical centre rotation of the winner packed in best[p] at resolution B
void launch_decode_q0(const unsigned long long* best, int32_t P, int32_t B, double* qs,
                      cudaStream_t s);
// pairs dst[k][0..1] = (v0[k], v1[k]), k < n, in one launch
struct SetList {
  static constexpr int kMax = 16;
  int64_t* dst[kMax];
  int64_t v0[kMax], v1[kMax];
  int32_t n = 0;
  bool add(int64_t* d, int64_t a, int64_t b) {
    if (n >= kMax) return false;
    dst[n] = d; v0[n] = a; v1[n] = b; ++n;
    return true;
  }
};
void launch_set_consts(const SetList& l, cudaStream_t s);
// d[0] = v0, d[1] = v1 (one thread)
void launch_set_i64x2(int64_t* d, int64_t v0, int64_t v1, cudaStream_t s);

}  // namespace rv
