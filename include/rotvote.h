/* ============================================================================
 * rotvote.h -- C-ABI of librotvote, the B200 (sm_100a) rotation-voting hot path
 * of arXiv 2506.11547 "Linearly Solving Robust Rotation Estimation".
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX source); S:n =
 * SPEC.md line n; "R#" = a reading listed in DESIGN.md §Readings.
 *
 * What the library computes:
 *   Given N correspondences (x_i, y_i), find the block c of the paper's
 *   stereographic accumulator grid (the cube [-1,1]^3 cut into B^3 blocks,
 *   Alg. 1 line 1; B = 2/epsilon_grid = 360 at the paper's default
 *   epsilon = 1/180) whose centre rotation q_c = P'(p_c) is
 *   crossed by the most quaternion circles, i.e.
 *       count(c) = #{ i : y_i^T R(q_c) x_i >= cos(eps) }      (R1, R2)
 *   maximised over every block meeting the unit ball (hemisphere + equator,
 *   P:409-411), ties -> lowest linear index (R7); then refine linearly on the
 *   inlier set (Q q = 0 in least squares, computed as the top
 *   eigenvector of sum_i M_i, Horn P:125-150, M_i of Appendix A).
 *   The search is a certified coarse-to-fine branch and bound (R6) whose result
 *   equals the exhaustive scan for every `levels`.
 *
 * Conventions
 *   - quaternions are scalar-first [q0,q1,q2,q3], returned as the
 *     hemisphere representative q3 <= 0 (tie rule S:361-369).
 *   - x, y: contiguous row-major [n][3] float32 (any nonzero length: rows are
 *     normalised).  DEVICE pointers on the context's device unless a
 *     function says HOST.
 *   - every call is ordered on cfg.stream and returns after its results are
 *     written (host-synchronous).  One context per host thread / stream.
 *   - return value: RV_OK (0) or a negative RV_E* code; the message is in
 *     rot_vote_last_error(ctx).  No C++ exception crosses the ABI.
 *   - multi-GPU (world > 1): every rank calls every entry point collectively
 *     with identical arguments (its own device replica of x, y) and receives
 *     identical results.
 * ========================================================================== */
#ifndef ROTVOTE_H_
#define ROTVOTE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---------------------------------------------------------- */
#define RV_OK        0
#define RV_EINVAL   -1  /* null pointer, n < 2, n > max_n, eps not in (0,pi),
                           levels not in [0, chain_len], bad chain, rank/world mismatch */
#define RV_EDATA    -2  /* a non-finite or zero-length x_i / y_i (cannot normalise) */
#define RV_ECUDA    -3  /* CUDA runtime failure */
#define RV_ENCCL    -4  /* NCCL failure (or libnccl.so.2 not loadable when world > 1) */
#define RV_ENOMEM   -5  /* workspace allocation failed */

/* ---- result flags ------------------------------------------------------------ */
#define RV_REFINED     1  /* at least one refinement round succeeded */
#define RV_DEGENERATE  2  /* a round had < 2 inliers or eigengap <= 1e-12*|lambda1|;
                             q is the last good estimate (q_c* if round 1 failed) */
#define RV_RECHECKED   4  /* the final level needed the fp64 near-threshold recheck */
#define RV_RETRIED     8  /* the one-pass solve hit a fixed capacity or the re-dive trigger (R18)
                             and was redone by the per-level loop (same result, slower) */

#define RV_MAX_CHAIN   8
#define RV_MAX_PHASES 16

/* Opaque context: owns every device workspace, pinned staging buffer, the
 * CUDA stream binding and (world > 1) the NCCL communicator. */
typedef struct rv_ctx rv_ctx;

typedef struct {
  int32_t device;        /* CUDA ordinal of this rank's GPU */
  int32_t rank;          /* 0 for a single GPU */
  int32_t world;         /* 1 for a single GPU; > 1: NCCL over NVLink, cells sharded */
  const void* nccl_id;   /* HOST, 128-byte ncclUniqueId from rot_vote_get_unique_id on rank 0,
                            broadcast by the caller; required when world > 1.  With world == 1 a
                            non-NULL id creates a 1-rank communicator and takes the NCCL path. */
  int64_t max_n;         /* workspace sizing: solve with n > max_n -> RV_EINVAL
                            (batched: total correspondences) */
  int32_t max_problems;  /* batched sizing (>= 1) */
  int32_t chain_len;     /* 0 -> default chain {5,15,45,90,180,360} */
  int32_t chain[RV_MAX_CHAIN]; /* nested grid resolutions, each divides the next; the last is
                            the paper's accumulator resolution B = 2/epsilon_grid */
  int32_t refine_rounds; /* linear refinement rounds (R8); 2 */
  float   guard;         /* fp32 guard band on the vote statistic (R10); 1e-5 */
  void*   stream;        /* cudaStream_t to order all work on (NULL = legacy default) */
  int32_t emulate_world; /* test hook: > 1 evaluates the cell shards of that many ranks one after
                            another on this GPU (loopback); 0/1 = off.  Requires world == 1. */
  int32_t tensor_vote;   /* 1: bound-level votes on the tensor cores (K3-TC, tcgen05, fp16-split
                            operands, fp32 accumulation); 0: FP32-pipe FFMA2 vote everywhere */
  int32_t cull;          /* 1 (needs tensor_vote): ancestor culling -- level 0 writes each block's
                            pass bitmask, every finer level votes its blocks only against the
                            correspondences that passed the bound test of a level-0 block of
                            their ancestor's group (K3-CT on the tensor cores; 2: K3-C on the
                            FP32 pipe over per-ancestor lists; the certified argument is in
                            DESIGN.md §5).  Same result; applies to the device level loop when
                            the bitmasks fit (<= 4 GiB).  0: off.  Other values -> RV_EINVAL. */
  int32_t planner;       /* 0: the level loop runs on the device (default; a single problem on one
                            GPU runs it in one pass: one host round trip per solve); 1: the host
                            planner (rv_plan.cpp) drives every level -- the reference the GPU tests
                            compare the device loop against; 2: the device loop with one host round
                            trip per branch-and-bound level (the one-pass solve's fallback).  Same
                            result.  Other values -> RV_EINVAL. */
  int32_t ct_sched;      /* K3-CT item scheduling: 0 (default) = big levels take their items
                            dynamically from a work counter (a scheduler warp per CTA), small ones
                            in the static order b, b + grid, ...; 1 = always the static order.
                            Same counts (integer sums); 1 exists so the tests can compare the
                            two orders.  Other values -> RV_EINVAL. */
} rv_config;

typedef struct {
  double   q[4];          /* refined rotation, scalar-first, q3 <= 0 */
  double   q_cell[4];     /* rotation of the winning block centre (before refinement) */
  uint32_t votes;         /* exact count of the winning block */
  uint32_t n_inliers;     /* |{i : s_i(q) >= cos(eps)}| at the returned q (popcount of the mask) */
  int32_t  cell[3];       /* winning block (i,j,k) at the finest resolution */
  int32_t  flags;         /* RV_REFINED | RV_DEGENERATE | RV_RECHECKED */
  int32_t  B;             /* finest resolution */
  int32_t  n_tied;        /* finest blocks sharing the winning count */
  uint64_t pair_votes;    /* sum over levels of n x blocks: every (correspondence, block) pair the
                             search decides (a culled pair is decided by its ancestor's test) */
  uint64_t cells_evaluated;
  uint32_t lb_star;       /* certified lower bound used for pruning */
  int32_t  n_phases;      /* entries used in cells_per_phase */
  int64_t  cells_per_phase[RV_MAX_PHASES];
  float    ms;            /* device time of the solve on cfg.stream (CUDA events) */
  int32_t  n_rechecked;   /* blocks that needed the fp64 near-threshold recheck */
  float    vote_ms;       /* summed device time of the K3 vote launches (CUDA events on cfg.stream) */
  int32_t  launches;      /* kernels this call launched (all of librotvote's own) */
  uint64_t vote_pairs;    /* (correspondence, block) pairs voted by K3 / K3-TC on this rank, padding
                             excluded */
  int32_t  vote_launches; /* K3 / K3-TC launches on this rank */
  int32_t  cull_launches; /* culled-vote launches (K3-CT or K3-C) on this rank */
  uint64_t cull_pairs;    /* (correspondence, block) pairs the culled vote evaluated on this rank */
  float    cull_ms;       /* summed device time of the culled-vote launches (CUDA events on
                             cfg.stream) */
  int32_t  cull_tc_launches; /* of cull_launches: on the tensor cores (K3-CT) */
  int32_t  host_syncs;    /* host waits on the device inside the call (one-pass solve: 1) */
  /* device time per phase (CUDA events on cfg.stream; one-pass single solves, else 0):
   * a1 setup, level 0 (vote + culling lists + dive start), the dive, the branch-and-bound
   * levels, the finest level (a5 recheck + winner), a6 refinement */
  float    t_setup_ms, t_level0_ms, t_dive_ms, t_bnb_ms, t_final_ms, t_refine_ms;
} rv_result;

/* ---- lifetime ------------------------------------------------------------------ */

/* Fill *cfg with the defaults: device 0, rank 0, world 1, max_n 1<<20, max_problems 1,
 * default chain, refine_rounds 2, guard 1e-5, stream NULL, tensor_vote 1, cull 1. */
void rot_vote_default_config(rv_config* cfg);

/* Create a context.  Allocates the K table for cfg->max_n correspondences, the streams, events
 * and pinned staging on cfg->device; world > 1 initialises NCCL (ncclCommInitRank, collective
 * across ranks).  The level workspace (block lists, pass bitmasks, culling lists, item tables)
 * is owned by the context too but sized by the first solve of a given (n, eps, chain) and kept:
 * that solve allocates (RV_ENOMEM if it cannot), later solves of the same or a smaller size do
 * not, and a one-pass solve whose fixed capacities prove too small is redone by the per-level
 * loop (rv_result.flags & RV_RETRIED) with the capacities grown for the next call.  Deviation
 * from SURVEY 8(b) "solve does not allocate": true from the second solve of a size on.
 * *out = NULL on failure.  Errors: RV_EINVAL, RV_ECUDA, RV_ENCCL, RV_ENOMEM. */
int rot_vote_create(const rv_config* cfg, rv_ctx** out);

/* Release everything the context owns.  NULL is a no-op. */
void rot_vote_destroy(rv_ctx* ctx);

/* Last error message of this context ("" if none); valid until the next call. */
const char* rot_vote_last_error(const rv_ctx* ctx);

/* Write a fresh 128-byte ncclUniqueId into id_out (HOST).  Call on rank 0 only.
 * Returns RV_ENCCL when libnccl.so.2 cannot be loaded. */
int rot_vote_get_unique_id(void* id_out);

/* ---- the hot path ----------------------------------------------------------------- */

/* Solve one problem (BASELINE north_star rot_vote_solve(x, y, N, eps, levels)).
 *   x, y   DEVICE [n][3] float32, caller-owned, unchanged.
 *   n      2 <= n <= max_n.
 *   eps    inlier angle in radians (double), 0 < eps < pi (R1): i is an inlier of q iff
 *          angle(R(q) x_i, y_i) <= eps, i.e. s_i(q) >= cos(eps) evaluated in double.
 *   levels number of chain levels used, the last `levels` entries of the chain;
 *          0 -> min(5, chain_len); 1 = exhaustive scan of the finest grid.
 *          The result does not depend on it (certified search, R6).
 *   out    HOST, filled on success.
 *   inlier_mask DEVICE uint32[ceil(n/32)] (bit i%32 of word i/32 = inlier i, LSB
 *          first) at the returned q, or NULL.
 * Errors: RV_EINVAL, RV_EDATA, RV_ECUDA, RV_ENCCL, RV_ENOMEM. */
int rot_vote_solve(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                   int32_t levels, rv_result* out, uint32_t* inlier_mask);

/* Same as rot_vote_solve but x, y are HOST pointers and inlier_mask (if not NULL) is a
 * HOST buffer: the copies to and from the device are part of the call (end-to-end API). */
int rot_vote_solve_host(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                        int32_t levels, rv_result* out, uint32_t* inlier_mask);

/* Solve P independent problems (BASELINE config 5).  Problem p is rows
 * [offsets[p], offsets[p+1]) of x, y (DEVICE).  offsets: HOST int64[P+1], offsets[0] = 0,
 * each problem has >= 2 rows, offsets[P] <= max_n, P <= max_problems.
 * out: HOST rv_result[P].  masks: DEVICE, problem p's mask at word offset
 * sum_{r<p} ceil(n_r/32), or NULL.
 * world > 1: problems are sharded in contiguous ranges across ranks (no per-level
 * collectives); the rv_result array is all-gathered so every rank returns all P results;
 * each rank writes the masks of its own problems only. */
int rot_vote_solve_batched(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets,
                           int32_t P, double eps, int32_t levels, rv_result* out, uint32_t* masks);

/* ---- the individual steps, exposed for parity tests ---------- */

/* a1 (K1 rv_setup): normalise x_i, y_i and write the 9 independent entries of the traceless
 * 4x4 form K_i with y^T R(q) x = q^T K_i q (= Appendix-A M):
 *   k_out[j*n + i], j = 0..8 -> K00, K11, K22, K01, K02, K03, K12, K13, K23
 *   (K33 = -(K00+K11+K22) since tr K_i = 0).  k_out: DEVICE float32[9*n].
 * Computed in fp64 and rounded once to fp32.  Errors: RV_EDATA on a bad row. */
int rot_vote_setup(rv_ctx* ctx, const float* x, const float* y, int64_t n, float* k_out);

#define RV_MODE_BOUND 0  /* cnt_a = #{i : s32_i(q_c) >= cos(min(pi, eps + r(c))) - guard} (R6) */
#define RV_MODE_FINAL 1  /* cnt_a = #{s32 >= cos(eps) - guard}, cnt_b = #{s32 >= cos(eps) + guard} */
#define RV_MODE_EXACT 2  /* cnt_a = #{i : s_i(q_c) >= cos(eps)} exactly: fp32 vote with an fp64
                            recheck of every pair within the guard band (K5) */
#define RV_MODE_BOUND_TC 3 /* RV_MODE_BOUND evaluated by K3-TC (context with tensor_vote = 1):
                              cnt_a = #{s_tc >= cos(min(pi, eps + r(c))) - guard - 1.5e-5}, the extra
                              1.5e-5 covering the worst-case error of the fp16-split MMA */
#define RV_MODE_FINAL_TC 4 /* RV_MODE_FINAL evaluated by K3-TC: cnt_a = #{s_tc >= cos(eps) - guard
                              - 1.5e-5}, cnt_b = #{s_tc >= cos(eps) + guard + 1.5e-5} */

/* a2-a5 (K3 rv_vote, K5 rv_recheck): vote m blocks of the B^3 grid.
 *   lins   DEVICE uint32[m], block (i,j,k) -> (i*B + j)*B + k.
 *   cnt_a  DEVICE uint32[m]; cnt_b DEVICE uint32[m] (RV_MODE_FINAL only, else may be NULL).
 * s32 is the fp32 contraction phi(q_c) . k_i of the 9-entry forms. */
int rot_vote_count_cells(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t B,
                         const uint32_t* lins, int64_t m, double eps, int32_t mode,
                         uint32_t* cnt_a, uint32_t* cnt_b);
/* rot_vote_count_cells maps modes to kernels literally (BOUND/FINAL: K3 on the FP32 pipe;
 * BOUND_TC/FINAL_TC: K3-TC).  The solve with tensor_vote = 1 sends its bound and final levels
 * to K3-TC: the planner only needs cnt_b <= exact <= cnt_a, which the wider band keeps. */

/* Ancestor culling (K3-CT / K3-C), for parity tests: vote the full level-0 grid
 * at resolution B0 with K3-TC (bound mode) writing the pass bitmasks, then count the m blocks
 * `lins` (resolution B, B % B0 == 0, any order) against their level-0 ancestors'
 * correspondences only (K3-CT: the union U over the ancestor's group; K3-C: L(anc)):
 *   BOUND: cnt_a = #{i in U : s_i(q_c) >= cos(min(pi, eps + r(c))) - guard'}
 *   FINAL: cnt_a / cnt_b at cos(eps) -/+ guard' (as RV_MODE_FINAL), over U
 * with L(a) = {i : s_tc_i(q_a) >= cos(min(pi, eps + r(a))) - guard - 1.5e-5}; guard' = the
 * vote's own guard (K3-CT: guard + 1.5e-5, fp16-split scores; K3-C: guard, FP32 scores).
 * Every exact voter of a block is in L(anc) ⊆ U, so the counts stay within the guard band of
 * the exact ones.
 * bits_out: DEVICE uint32[m0][ceil(n/256)*8] copy of the level-0 bitmasks (row = the block's
 * index in the ascending candidate list of B0, bit i%32 of word i/32 = i in L), or NULL.
 * Needs tensor_vote = 1 and cull = 1; 1 <= B0 <= 90. */
int rot_vote_count_cells_culled(rv_ctx* ctx, const float* x, const float* y, int64_t n,
                                int32_t B0, int32_t B, const uint32_t* lins, int64_t m,
                                double eps, int32_t mode, uint32_t* cnt_a, uint32_t* cnt_b,
                                uint32_t* bits_out);

/* Test hook for K3-TC's arithmetic: the raw tensor-core scores S' = s_tc - t of m blocks
 * (t = the RV_MODE_BOUND_TC threshold, guard included) against every correspondence.  out: DEVICE float
 * [m][ld] with ld = n rounded up to 256; columns >= n hold -1 (padding rows).  Needs a
 * context created with tensor_vote = 1. */
int rot_vote_debug_tc_scores(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t B,
                             const uint32_t* lins, int64_t m, double eps, float* out);

/* a6 (K6 rv_inliers + K7 rv_eig4): `rounds` rounds of linear refinement from q0 (HOST
 * double[4]); writes q_out (HOST double[4], canonical), flags (HOST, RV_REFINED /
 * RV_DEGENERATE), n_inliers (HOST) and the mask at q_out (DEVICE, may be NULL).  Inlier
 * decisions are made in fp64. q0 need not be normalised; rounds = 0 only evaluates the
 * mask at the (normalised, hemisphere-canonical) q0. */
int rot_vote_refine(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                    const double* q0, int32_t rounds, double* q_out, int32_t* flags,
                    uint32_t* n_inliers, uint32_t* mask);

/* ---- NEXT-2: several rotations -----------------------------------------------
 * Up to K peaks, greedily (reading R16): peak 1 is rot_vote_solve's winner; peak k is the
 * fullest finest block whose centre rotation is more than rho (rotation angle, radians, in
 * [0, pi]) from every earlier peak's centre (|q_c . q_j| < cos(rho/2)), ties -> lowest lin,
 * found by the same certified search with the earlier peaks' balls excluded (blocks entirely
 * inside a ball are skipped, finest blocks tested exactly).  Each peak is refined on its own
 * inliers.  out: HOST rv_result[K]; *n_found peaks are written (fewer than K when every
 * remaining block is suppressed).  Block counts voted for one peak are reused by the next.
 * Runs the host planner (sharded over ranks like rot_vote_solve).  No masks.
 * Errors: as rot_vote_solve; RV_EINVAL for K outside [1, 64] or rho outside [0, pi]. */
int rot_vote_solve_multi(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                         int32_t levels, int32_t K, double rho, rv_result* out,
                         int32_t* n_found);

/* ---- NEXT-3: rigid pose front end ---------------------------------------------
 * Points x, y (DEVICE [n][3] fp32, y = R x + t for inliers).  Pairs i < j give m = x_i - x_j,
 * n = y_i - y_j, kept iff |‖m‖ - ‖n‖| <= mu_t (rotation-invariant length check, P:563-573;
 * reading R17); the kept pairs are the correspondences of a rotation vote (rot_vote_solve at
 * eps / levels), and with its rotation R* every point votes t_i = y_i - R* x_i on the grid
 * [t_lo, t_hi)^3 at t_step ([-5,5]^3, 0.025); t = the fullest bin's centre (ties ->
 * lowest lin), t_mean = the mean of its candidates.  The context needs max_n >= the number of
 * kept pairs (RV_EINVAL otherwise, with the count in the message).  pair_ij: DEVICE int32
 * [pair_cap][2] receiving the kept pairs' (i, j) in pair order (may be NULL). */
typedef struct {
  double   q[4];          /* rotation (rot_vote_solve on the pairs, refined) */
  double   t[3];          /* translation: centre of the fullest bin */
  double   t_mean[3];     /* mean of that bin's candidates */
  uint32_t rot_votes;     /* the rotation's vote count (pairs) */
  uint32_t rot_inliers;   /* pairs within eps of the refined rotation */
  uint32_t t_votes;       /* candidates in the translation bin */
  int32_t  t_cell[3];
  int32_t  pad_;
  int64_t  pairs_total;   /* n (n - 1) / 2 */
  int64_t  pairs_kept;
  float    ms, pairs_ms, rot_ms, trans_ms;  /* device times (CUDA events) */
} rv_rigid_result;

int rot_vote_rigid(rv_ctx* ctx, const float* x, const float* y, int64_t n, double mu_t,
                   double eps, int32_t levels, double t_lo, double t_hi, double t_step,
                   rv_rigid_result* out, int32_t* pair_ij, int64_t pair_cap);

/* The translation vote alone, for a given rotation q (HOST double[4], scalar-first):
 * lin / votes / t / t_mean as in rot_vote_rigid (HOST outputs).  RV_EDATA when no candidate
 * falls inside the grid. */
int rot_vote_translation(rv_ctx* ctx, const float* x, const float* y, int64_t n,
                         const double* q, double t_lo, double t_hi, double t_step,
                         int64_t* lin, uint32_t* votes, double* t, double* t_mean);

/* ---- NEXT-4: the paper's Algorithm 1 as a same-box baseline ------------------
 * Every correspondence's quaternion circle is sampled at J angles
 * alpha_j = -pi + 2 pi j / J (Alg. 1 line 2), each sample taken to the half sphere q3 <= 0,
 * projected and binned on the B^3 grid of [-1,1]^3 (Alg. 1 line 1; B = the chain's
 * finest resolution, 360 by default); every sample adds one vote (Alg. 1 line 8).
 * Result: the fullest bin (ties -> lowest lin), its votes and its centre's rotation (Alg. 1
 * line 11; no refinement).  The bins are decided in fp64 with every operation rounded
 * explicitly, so the accumulator equals the oracle's (or_alg1_bins) exactly.
 * x, y: DEVICE [n][3] fp32.  acc_out: DEVICE u32 [B^3] copy of the accumulator (may be NULL).
 * The context owns the accumulator (4 B^3 bytes, allocated on first use).
 * Errors: RV_EINVAL (n < 1, J < 1, n > max_n), RV_EDATA (zero / non-finite vector),
 * RV_ENOMEM, RV_ECUDA. */
typedef struct {
  double   q[4];        /* rotation of the winning block's centre (hemisphere-canonical) */
  uint32_t votes;       /* its accumulator count (samples) */
  int32_t  cell[3];     /* (i, j, k) at resolution B */
  int32_t  B, J;
  uint64_t samples;     /* n * J */
  float    ms;          /* device time of the call (CUDA events) */
  float    vote_ms;     /* device time of the sampling / scatter kernel */
} rv_alg1_result;

int rot_vote_alg1(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t J,
                  rv_alg1_result* out, uint32_t* acc_out);

#ifdef __cplusplus
}
#endif
#endif /* ROTVOTE_H_ */
