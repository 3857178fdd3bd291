/* ============================================================================
 * rotvote_plan.h -- host-side search planner of librotvote (pure C++, no CUDA).
 *
 * The planner is the level loop of the certified coarse-to-fine search
 * (reading R6).  It decides which blocks of
 * which grid level are voted next and digests their counts; it never counts
 * anything itself.  rot_vote_solve drives it with the GPU kernels; the tests
 * drive it with counts from the CPU oracle and, for multi-rank checks, shard
 * each request with rv_shard_range across gloo ranks.  Every rank that feeds
 * identical counts holds an identical planner state.
 *
 * Request protocol:  while (rv_plan_request(p, &B, &mode, &m, &lins)) {
 *     count the m blocks `lins` of the B^3 grid in `mode` (rotvote.h RV_MODE_*)
 *     rv_plan_feed(p, cnt_a, cnt_b);            // cnt_b only for RV_MODE_FINAL
 *   }  rv_plan_get_result(p, &res);
 * Semantics of the counts per mode are those of rot_vote_count_cells.
 * ========================================================================== */
#ifndef ROTVOTE_PLAN_H_
#define ROTVOTE_PLAN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rv_plan rv_plan;

typedef struct {
  uint32_t lin;          /* winning block at the finest resolution */
  int32_t  B;            /* finest resolution */
  uint32_t votes;        /* its exact count */
  int32_t  n_tied;       /* finest blocks with the same count */
  uint32_t lb_star;      /* lower bound used for pruning */
  int32_t  n_rechecked;  /* blocks sent to RV_MODE_EXACT */
  uint64_t pair_votes;   /* sum over requests of m * n */
  uint64_t cells_evaluated;
  int32_t  n_phases;
  int64_t  cells_per_phase[16];
} rv_plan_result;

/* chain[chain_len] nested resolutions (each divides the next, 1 <= B <= 1625); levels in
 * [0, chain_len] (0 -> min(5, chain_len)); n >= 1 correspondences; eps in (0, pi);
 * guard >= 0.  Returns 0 or -1 (invalid) and sets *out. */
int  rv_plan_create(const int32_t* chain, int32_t chain_len, int32_t levels, int64_t n,
                    double eps, double guard, rv_plan** out);
/* NEXT-2 (several rotations): the same search restricted to the finest blocks whose centre
 * rotation is more than rho (rotation angle, radians, in [0, pi]) from each of the n_excl
 * rotations excl_q (HOST double[n_excl][4], scalar-first, normalised here): a finest block is
 * excluded iff |q_c . q_e| >= cos(rho/2); a coarser block is skipped only when all of it is
 * (angle(q_c, q_e) + r(c) <= rho).  With everything excluded the result has votes = 0 and
 * n_tied = 0.  Returns 0 or -1. */
int  rv_plan_create_ex(const int32_t* chain, int32_t chain_len, int32_t levels, int64_t n,
                       double eps, double guard, const double* excl_q, int32_t n_excl,
                       double rho, rv_plan** out);
void rv_plan_destroy(rv_plan* p);

/* 1 if a request is pending (outputs set; lins valid until the next feed), 0 when done. */
int  rv_plan_request(const rv_plan* p, int32_t* B, int32_t* mode, int64_t* m,
                     const uint32_t** lins);
/* 1 if the pending request is the complete candidate list of its grid (level 0, or the
 * exhaustive scan), i.e. identical to rv_grid_candidates(B); 0 otherwise. */
int  rv_plan_request_is_full_grid(const rv_plan* p);
/* Level 0 reduced by the caller (batched solves keep level-0 counts on the device).
 * rv_plan_feed_l0_start replaces rv_plan_feed for a level-0 RV_MODE_BOUND request: `start` is
 * the index (into that request) of the dive's first block, the one rv_plan_feed would pick --
 * max excess UB - n*bg[e] with bg = rv_plan_l0_background, blocks with their centre inside the
 * ball first, ties -> lowest index.  After the dive the plan has no request and
 * rv_plan_needs_l0_survivors returns 1 with the pruning bound; the caller then passes the
 * indices of the level-0 blocks with UB >= lb_star (ascending) to rv_plan_feed_l0_survivors.
 * All return 0 / -1 (wrong state or index). */
int  rv_plan_feed_l0_start(rv_plan* p, int64_t start);
int  rv_plan_needs_l0_survivors(const rv_plan* p, int64_t* lb_star);
int  rv_plan_feed_l0_survivors(rv_plan* p, const int32_t* idx, int64_t k);
/* The cached per-candidate background (1 - cos(min(pi, eps + r(c))))/2 of the full grid B, in
 * rv_grid_candidates order (HOST, valid for the process lifetime); NULL when not cached. */
const double* rv_plan_l0_background(int32_t B, double eps, int64_t* m);

/* Feed the counts of the pending request (HOST arrays of m entries).  0 or -1. */
int  rv_plan_feed(rv_plan* p, const uint32_t* cnt_a, const uint32_t* cnt_b);
/* 0 when done and *out filled, -1 while requests are pending. */
int  rv_plan_get_result(const rv_plan* p, rv_plan_result* out);

/* Contiguous shard of a request of m blocks for `rank` of `world`:
 * [m*rank/world, m*(rank+1)/world). */
void rv_shard_range(int64_t m, int32_t rank, int32_t world, int64_t* begin, int64_t* end);

/* Candidate blocks (meeting the closed unit ball) of the B^3 grid in ascending linear
 * index; writes min(count, cap) entries to out (may be NULL) and returns the count. */
int64_t rv_grid_candidates(int32_t B, uint32_t* out, int64_t cap);

/* Ancestor groups of a culled solve: the level-0 blocks of the B0 grid (rows in
 * rv_grid_candidates(B0) order, m0 of them) with equal (i / gi, j / gj, k / gk) form a group,
 * numbered by first appearance in row order; a group's list is the union of its members'.
 * Writes (each may be NULL) group_of[m0] (row -> group), goff[G + 1] and gmem[m0] (the rows of
 * group g, ascending, are gmem[goff[g] .. goff[g+1])).  Returns G, or -1 for B0 outside
 * [1, 1625] or a group extent < 1. */
int64_t rv_cull_groups(int32_t B0, int32_t gi, int32_t gj, int32_t gk, int32_t* group_of,
                       int32_t* goff, int32_t* gmem);
/* The multi-rank partition of one culled problem: slice[world + 1] = level-0
 * row boundaries (rank r votes rows slice[r] .. slice[r+1] with their pass bitmasks), each cut at
 * the first row at or after ceil(m0 r / world) where a new run of whole groups starts, so no
 * group straddles two slices; gslice[world + 1] = group boundaries (rank r owns groups
 * gslice[r] .. gslice[r+1], those whose first member is in its slice, and votes every finer
 * block whose level-0 ancestor is in one of them).  0, or -1 on invalid arguments. */
int rv_cull_partition(int32_t B0, int32_t gi, int32_t gj, int32_t gk, int32_t world,
                      int64_t* slice, int64_t* gslice);

#ifdef __cplusplus
}
#endif
#endif /* ROTVOTE_PLAN_H_ */
