// rv_host_plan.cpp -- the paths that drive the host planner (rv_plan.cpp): host-built vote
// items, one planner request sharded over ranks, the single solve with the host planner,
// several rotations (NEXT-2), rigid pose (NEXT-3) and the batched host-planner requests.
#include "rv_ctx.h"

namespace rvi {

// ---- work decomposition ---------------------------------------------------------------------

// Vote items for segments given as (n_cells, n_corr) pairs.  The CTA shape (groups G: a CTA
// covers kCellsPerBlock/G cells) is chosen to waste the fewest thread slots; the
// correspondence chunk gives >= ~8 waves of equal-cost CTAs while keeping each CTA above
// ~1M pair votes so its prologue (cell rotations, thresholds, first TMA) stays negligible.
int build_vote_items(const std::vector<int64_t>& ncell, const std::vector<int64_t>& ncorr,
                     int slots, std::vector<rv::VoteItem>& items, int force_groups = 0) {
  items.clear();
  // G = 1 unless a smaller CTA saves more than 5% of the thread slots
  int groups = 1;
  int64_t pad1 = 0;
  for (size_t s = 0; s < ncell.size(); ++s)
    pad1 += (ncell[s] + rv::kCellsPerBlock - 1) / rv::kCellsPerBlock * rv::kCellsPerBlock;
  int64_t best_pad = pad1;
  for (int G : {2, 4}) {
    const int64_t cpb = rv::kCellsPerBlock / G;
    int64_t padded = 0;
    for (size_t s = 0; s < ncell.size(); ++s) padded += (ncell[s] + cpb - 1) / cpb * cpb;
    if (padded < best_pad && (double)padded < 0.95 * (double)pad1) { best_pad = padded; groups = G; }
  }
  if (force_groups == 1 || force_groups == 2 || force_groups == 4) groups = force_groups;
  const int64_t cpb = rv::kCellsPerBlock / groups;
  // correspondence chunks: one chunk count per launch, picked so the CTA count fills whole
  // waves (items / slots just below an integer), with 4..64 waves and CTAs of >= 2^20 pair
  // slots (their prologue -- cell rotations, thresholds, first TMA -- stays negligible)
  int64_t cbs = 0, nmax = 0;
  for (size_t s = 0; s < ncell.size(); ++s) {
    if (ncell[s] == 0 || ncorr[s] == 0) continue;
    cbs += (ncell[s] + cpb - 1) / cpb;
    nmax = std::max<int64_t>(nmax, pad4(ncorr[s]));
  }
  if (cbs == 0) return groups;
  const int64_t min_chunk = std::min<int64_t>(nmax, std::max<int64_t>(256, (1 << 20) / cpb));
  const int64_t max_nch = std::max<int64_t>(1, nmax / min_chunk);
  int64_t best_nch = 1;
  double best_eff = -1;
  for (int64_t nch = 1; nch <= max_nch; ++nch) {
    const int64_t items_n = cbs * nch;
    const double waves = (double)items_n / slots;
    if (waves > 64.0 && nch > 1) break;
    const double eff = waves / std::ceil(waves);
    // prefer >= 4 waves (dynamic balance), then the fullest last wave
    const double score = eff - (waves < 4.0 ? 0.5 * (4.0 - waves) / 4.0 : 0.0);
    if (score > best_eff + 1e-9) { best_eff = score; best_nch = nch; }
  }
  for (size_t s = 0; s < ncell.size(); ++s) {
    const int64_t n4 = pad4(ncorr[s]);
    if (ncell[s] == 0 || n4 == 0) continue;
    const int64_t cb = (ncell[s] + cpb - 1) / cpb;
    const int64_t per = (ncell[s] + cb - 1) / cb;  // balanced cells per CTA
    const int64_t nch = std::min<int64_t>(best_nch, std::max<int64_t>(1, n4 / 4));
    const int64_t chunk = (n4 / 4 + nch - 1) / nch * 4;  // balanced, multiple of 4
    for (int64_t b = 0; b < cb; ++b) {
      const int64_t c0 = b * per, nc = std::min(per, ncell[s] - c0);
      if (nc <= 0) continue;
      for (int64_t i0 = 0; i0 < n4; i0 += chunk)
        items.push_back({(int32_t)s, (int32_t)c0, (int32_t)nc, (int32_t)i0,
                         (int32_t)std::min(chunk, n4 - i0)});
    }
  }
  return groups;
}

// K3-TC items: <= cpb cells (kTcM, or kTcM/2 rows-pairs in FINAL mode) x a correspondence
// chunk of whole kTcN tiles; chunk count chosen, as for K3, to fill whole waves of the
// persistent kernel's CTAs.  ablocks: the distinct A-operand blocks (K2-TC); a segment whose
// block list equals the previous segment's (same seg_key, same cell count -- the shared
// level-0 grid of a batch) reuses its blocks.
void build_tc_items(const std::vector<int64_t>& ncell, const std::vector<int64_t>& ncorr,
                    int slots, std::vector<rv::VoteItem>& items, std::vector<rv::ABlock>& ablocks,
                    int64_t cpb, const std::vector<const void*>* seg_key) {
  items.clear();
  ablocks.clear();
  int64_t cbs = 0, tmax = 0;
  for (size_t s = 0; s < ncell.size(); ++s) {
    if (ncell[s] == 0 || ncorr[s] == 0) continue;
    cbs += (ncell[s] + cpb - 1) / cpb;
    tmax = std::max<int64_t>(tmax, (ncorr[s] + rv::kTcN - 1) / rv::kTcN);
  }
  if (cbs == 0) return;
  const int64_t min_tiles = std::min<int64_t>(tmax, 8);
  const int64_t max_nch = std::max<int64_t>(1, tmax / std::max<int64_t>(1, min_tiles));
  int64_t best_nch = 1;
  double best = -1;
  for (int64_t nch = 1; nch <= max_nch; ++nch) {
    const double waves = (double)(cbs * nch) / slots;
    if (waves > 64.0 && nch > 1) break;
    const double eff = waves / std::ceil(waves);
    const double score = eff - (waves < 4.0 ? 0.5 * (4.0 - waves) / 4.0 : 0.0);
    if (score > best + 1e-9) { best = score; best_nch = nch; }
  }
  int64_t last = -1;
  int32_t last_base = 0;
  std::vector<int32_t> seg_base(ncell.size(), 0);
  for (size_t s = 0; s < ncell.size(); ++s) {
    if (ncell[s] == 0 || ncorr[s] == 0) continue;
    const int64_t cb = (ncell[s] + cpb - 1) / cpb;
    const int64_t per = (ncell[s] + cb - 1) / cb;
    if (seg_key && last >= 0 && (*seg_key)[s] == (*seg_key)[last] && ncell[s] == ncell[last]) {
      seg_base[s] = last_base;
    } else {
      seg_base[s] = (int32_t)ablocks.size();
      for (int64_t b = 0; b < cb; ++b) {
        const int64_t c0 = b * per, nc = std::min(per, ncell[s] - c0);
        if (nc > 0) ablocks.push_back({(int32_t)s, (int32_t)c0, (int32_t)nc, 0});
      }
    }
    last = (int64_t)s;
    last_base = seg_base[s];
  }
  // chunk-major order: the CTAs running at the same time share one correspondence chunk,
  // whose tiles then stay in L2 (block-major order spreads them over the whole table)
  for (int64_t c = 0; c < best_nch; ++c)
    for (size_t s = 0; s < ncell.size(); ++s) {
      if (ncell[s] == 0 || ncorr[s] == 0) continue;
      const int64_t nt = (ncorr[s] + rv::kTcN - 1) / rv::kTcN;
      const int64_t nch = std::min<int64_t>(best_nch, nt);
      if (c >= nch) continue;
      const int64_t ct = (nt + nch - 1) / nch;  // tiles per chunk
      const int64_t t0 = c * ct;
      if (t0 >= nt) continue;
      const int64_t cb = (ncell[s] + cpb - 1) / cpb;
      const int64_t per = (ncell[s] + cb - 1) / cb;
      for (int64_t b = 0; b < cb; ++b) {
        const int64_t c0 = b * per, nc = std::min(per, ncell[s] - c0);
        if (nc <= 0) continue;
        items.push_back({(int32_t)s, (int32_t)c0, (int32_t)nc, (int32_t)(t0 * rv::kTcN),
                         (int32_t)(std::min(ct, nt - t0) * rv::kTcN), seg_base[s] + (int32_t)b});
      }
    }
}

void build_exact_items(const std::vector<int64_t>& ncell, const std::vector<int64_t>& ncorr,
                       std::vector<rv::VoteItem>& items) {
  items.clear();
  const int64_t chunk = 1 << 12;  // ~250 items per block group at N = 1e6: one wave
  for (size_t s = 0; s < ncell.size(); ++s)
    for (int64_t c = 0; c < ncell[s]; c += rv::kExactCells)
      for (int64_t i0 = 0; i0 < ncorr[s]; i0 += chunk)
        items.push_back({(int32_t)s, (int32_t)c,
                         (int32_t)std::min<int64_t>(rv::kExactCells, ncell[s] - c), (int32_t)i0,
                         (int32_t)std::min(chunk, ncorr[s] - i0)});
}

// K2-TC + K3-TC over the items already in ctx->vitems (segments in ctx->vsegs).  The block
// list goes through a pageable copy (staged on the call).  Asynchronous.
int launch_tc(rv_ctx* ctx, const std::vector<rv::ABlock>& ab, int32_t n_items, bool fin,
              float* dump, int64_t ld) {
  if (ab.empty() || n_items <= 0) return RV_OK;
  RV_CUDA(ctx->ablk.ensure(ab.size()), "allocating A blocks");
  RV_CUDA(ctx->atab.ensure(ab.size() * (size_t)rv::kTcABlockBytes), "allocating A table");
  RV_CUDA(cudaMemcpyAsync(ctx->ablk.p, ab.data(), ab.size() * sizeof(rv::ABlock),
                          cudaMemcpyHostToDevice, ctx->stream), "H2D");
  rv::launch_vote_tc(ctx->tctab.p, ctx->atab.p, ctx->ablk.p, (int32_t)ab.size(), ctx->vsegs.p,
                     ctx->vitems.p, n_items, ctx->cfg.guard + kTcExtraGuard, dump, ld,
                     ctx->stream, fin);
  ctx->launches += 1;  // K2-TC (the vote launch is counted by the caller)
  return RV_OK;
}

// ---- one planner request (single problem), sharded over ranks --------------------------------
// Counts land in cnt_a/cnt_b (HOST, m entries each).
// auto_tc: RV_MODE_BOUND / RV_MODE_FINAL go to K3-TC when the context has tensor_vote (the
// solve); false keeps the explicit mode -> kernel mapping of rot_vote_count_cells.
int eval_request(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps, int32_t B,
                 int32_t mode, int64_t m, const uint32_t* lins, uint32_t* cnt_a, uint32_t* cnt_b,
                 bool auto_tc) {
  const int W = ctx->effective_world();
  const int64_t chunk = (m + W - 1) / W;
  const int64_t per_rank = 2 * chunk;  // [a | b]
  // ranks evaluated by this process
  int r_lo = 0, r_hi = W;
  const bool nccl_path = ctx->comm != nullptr;  // world > 1, or world 1 with an NCCL id
  if (nccl_path) { r_lo = ctx->cfg.rank; r_hi = r_lo + 1; }
  const int nr = r_hi - r_lo;

  RV_CUDA(ctx->lins.ensure(std::max<int64_t>(1, chunk * nr)), "allocating block list");
  // gathered counts [W][2*chunk] + (world>1) local [2*chunk]
  const size_t cnt_need = (size_t)per_rank * W + (nccl_path ? per_rank : 0) + 1;
  RV_CUDA(ctx->cnt.ensure(cnt_need), "allocating counts");
  uint32_t* gathered = ctx->cnt.p;
  uint32_t* local = nccl_path ? ctx->cnt.p + per_rank * W : nullptr;

  std::vector<int64_t> ncell, ncorr;
  std::vector<rv::VoteSeg> segs;
  for (int r = r_lo; r < r_hi; ++r) {
    int64_t b, e;
    rv_shard_range(m, r, W, &b, &e);
    rv::VoteSeg sg{};
    sg.lins = ctx->lins.p + (int64_t)(r - r_lo) * chunk;
    uint32_t* tgt = local ? local : gathered + (int64_t)r * per_rank;
    sg.cnt_a = tgt;
    sg.cnt_b = tgt + chunk;
    sg.koff = 0;
    sg.row = 0;
    sg.n = (int32_t)n;
    sg.B = B;
    sg.eps = eps;
    segs.push_back(sg);
    ncell.push_back(e - b);
    ncorr.push_back(n);
  }
  std::vector<rv::VoteItem> items;
  std::vector<rv::ABlock> ablocks;
  int groups = 1;
  const bool tc_auto = auto_tc && ctx->tc_on;
  const bool tc_final = mode == RV_MODE_FINAL_TC || (mode == RV_MODE_FINAL && tc_auto);
  const bool use_tc = tc_final || mode == RV_MODE_BOUND_TC || (mode == RV_MODE_BOUND && tc_auto);
  if ((mode == RV_MODE_BOUND_TC || mode == RV_MODE_FINAL_TC) && !ctx->tc_on)
    return ctx->fail(RV_EINVAL, "the _TC modes need a context created with tensor_vote = 1");
  if (use_tc) {
    for (rv::VoteSeg& sg : segs) sg.koff = ctx->tc_toff[0];
    build_tc_items(ncell, ncorr, ctx->num_sms, items, ablocks, tc_final ? rv::kTcM / 2 : rv::kTcM);
  } else if (mode == RV_MODE_EXACT) {
    build_exact_items(ncell, ncorr, items);
  } else {
    groups = build_vote_items(ncell, ncorr, ctx->num_sms * ctx->vote_blocks_per_sm, items,
                              ctx->force_groups);
  }

  RV_CUDA(ctx->vsegs.ensure(segs.size()), "allocating segments");
  RV_CUDA(ctx->vitems.ensure(std::max<size_t>(1, items.size())), "allocating items");
  RV_CUDA(ctx->up.ensure(chunk * nr * 4 + segs.size() * sizeof(rv::VoteSeg) +
                         items.size() * sizeof(rv::VoteItem) + 4096),
          "allocating staging");
  RV_CUDA(ctx->down.ensure(per_rank * W * 4 + 256), "allocating staging");
  ctx->up.reset();
  uint32_t* hl = ctx->up.take<uint32_t>(std::max<int64_t>(1, chunk * nr));
  for (int r = r_lo; r < r_hi; ++r) {
    int64_t b, e;
    rv_shard_range(m, r, W, &b, &e);
    std::memcpy(hl + (int64_t)(r - r_lo) * chunk, lins + b, (e - b) * 4);
  }
  rv::VoteSeg* hs = ctx->up.take<rv::VoteSeg>(segs.size());
  std::memcpy(hs, segs.data(), segs.size() * sizeof(rv::VoteSeg));
  rv::VoteItem* hi = ctx->up.take<rv::VoteItem>(std::max<size_t>(1, items.size()));
  if (!items.empty()) std::memcpy(hi, items.data(), items.size() * sizeof(rv::VoteItem));

  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaMemcpyAsync(ctx->lins.p, hl, chunk * nr * 4, cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->vsegs.p, hs, segs.size() * sizeof(rv::VoteSeg),
                          cudaMemcpyHostToDevice, s), "H2D");
  if (!items.empty())
    RV_CUDA(cudaMemcpyAsync(ctx->vitems.p, hi, items.size() * sizeof(rv::VoteItem),
                            cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemsetAsync(local ? local : gathered, 0,
                          (local ? per_rank : per_rank * W) * sizeof(uint32_t), s), "memset");
  if (mode == RV_MODE_EXACT) {
    rv::launch_exact(ctx->k9.p, ctx->stride, x, y, ctx->vsegs.p, ctx->vitems.p,
                     (int32_t)items.size(), ctx->cfg.guard, s);
  } else {
    RV_CUDA(cudaEventRecord(ctx->evv0, s), "event");
    if (use_tc)
      {
        if (int rc = launch_tc(ctx, ablocks, (int32_t)items.size(), tc_final)) return rc;
      }
    else
      rv::launch_vote(mode, groups, ctx->k9.p, ctx->stride, ctx->vsegs.p, ctx->vitems.p,
                      (int32_t)items.size(), ctx->cfg.guard, s);
    RV_CUDA(cudaEventRecord(ctx->evv1, s), "event");
    for (int64_t c : ncell) ctx->vote_pairs += (uint64_t)c * (uint64_t)n;
    ctx->vote_launches += 1;
  }
  ctx->launches += items.empty() ? 0 : 1;
  RV_CUDA(cudaGetLastError(), "launching the vote kernel");
  if (nccl_path) {
    ncclResult_t nr_ = nccl().AllGather(local, gathered, (size_t)per_rank, ncclUint32, ctx->comm, s);
    if (nr_ != ncclSuccess)
      return ctx->fail(RV_ENCCL, "ncclAllGather: %s", nccl().GetErrorString(nr_));
  }
  ctx->down.reset();
  uint32_t* hc = ctx->down.take<uint32_t>(per_rank * W);
  RV_CUDA(cudaMemcpyAsync(hc, gathered, per_rank * W * 4, cudaMemcpyDeviceToHost, s), "D2H");
  ctx->mark("  launched");
  RV_SYNC(cudaStreamSynchronize(s), "vote");
  ctx->mark("  synced");
  if (mode != RV_MODE_EXACT && !items.empty()) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->evv0, ctx->evv1);
    ctx->vote_ms += ms;
  }
  for (int r = 0; r < W; ++r) {
    int64_t b, e;
    rv_shard_range(m, r, W, &b, &e);
    std::memcpy(cnt_a + b, hc + (int64_t)r * per_rank, (e - b) * 4);
    if (cnt_b) std::memcpy(cnt_b + b, hc + (int64_t)r * per_rank + chunk, (e - b) * 4);
  }
  return RV_OK;
}

// Block counts already voted in this call, keyed by (mode, B, lin): a later search over the
// same input (the next peak of rot_vote_solve_multi) votes only the blocks it has not seen.
using CountCache = std::unordered_map<uint64_t, std::pair<uint32_t, uint32_t>>;

// Drive a host planner to completion: every request voted (sharded over ranks) by
// eval_request; with a cache only the uncached blocks are voted.
int run_host_plan(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                  rv_plan* plan, rv_plan_result* pr, CountCache* cache) {
  std::vector<uint32_t> ca, cb, ml, ma, mb;
  std::vector<int64_t> mi;
  int32_t B, mode;
  int64_t m;
  const uint32_t* lins;
  while (rv_plan_request(plan, &B, &mode, &m, &lins)) {
    ca.assign(m, 0);
    cb.assign(m, 0);
    if (!cache) {
      if (int rc = eval_request(ctx, x, y, n, eps, B, mode, m, lins, ca.data(), cb.data()))
        return rc;
    } else {
      ml.clear();
      mi.clear();
      for (int64_t e = 0; e < m; ++e) {
        const uint64_t key = ((uint64_t)mode << 56) | ((uint64_t)B << 32) | lins[e];
        auto it = cache->find(key);
        if (it != cache->end()) {
          ca[e] = it->second.first;
          cb[e] = it->second.second;
        } else {
          ml.push_back(lins[e]);
          mi.push_back(e);
        }
      }
      if (!ml.empty()) {
        ma.assign(ml.size(), 0);
        mb.assign(ml.size(), 0);
        if (int rc = eval_request(ctx, x, y, n, eps, B, mode, (int64_t)ml.size(), ml.data(),
                                  ma.data(), mb.data()))
          return rc;
        for (size_t q = 0; q < ml.size(); ++q) {
          ca[mi[q]] = ma[q];
          cb[mi[q]] = mb[q];
          cache->emplace(((uint64_t)mode << 56) | ((uint64_t)B << 32) | ml[q],
                         std::make_pair(ma[q], mb[q]));
        }
      }
    }
    if (rv_plan_feed(plan, ca.data(), cb.data()) != 0)
      return ctx->fail(RV_ECUDA, "internal: planner rejected counts");
    ctx->mark("  fed");
  }
  rv_plan_get_result(plan, pr);
  return RV_OK;
}

int solve_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps, int32_t levels,
               rv_result* out, uint32_t* mask) {
  if (int rc = validate_common(ctx, x, y, eps, levels)) return rc;
  if (!out) return ctx->fail(RV_EINVAL, "out must be non-null");
  if (n < 2) return ctx->fail(RV_EINVAL, "n must be >= 2 (got %lld)", (long long)n);
  if (n > ctx->cfg.max_n)
    return ctx->fail(RV_EINVAL, "n = %lld exceeds max_n = %lld", (long long)n,
                     (long long)ctx->cfg.max_n);
  // the device-resident level loop with P = 1 (no per-level host work; over several ranks each
  // level's votes are sharded, see solve_batched_dplan).  The host planner below remains for
  // RV_HOST_PLAN=1 and the configurations the device loop does not take (levels == 1).
  const int32_t lev = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
  if (dplan_applies(ctx, lev, ctx->chain[ctx->chain.size() - lev], eps)) {
    const int64_t offs1[2] = {0, n};
    return solve_batched_impl(ctx, x, y, offs1, 1, eps, levels, out, mask);
  }
  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaEventRecord(ctx->ev0, s), "event");
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  if (int rc = check_bad(ctx)) return rc;

  Trace tr;
  ctx->trace = tr.on ? &tr : nullptr;
  ctx->mark("setup");
  rv_plan* plan = nullptr;
  if (rv_plan_create(ctx->chain.data(), (int32_t)ctx->chain.size(), levels, n, eps,
                     (double)ctx->cfg.guard, &plan) != 0)
    return ctx->fail(RV_EINVAL, "invalid search plan");
  ctx->mark("plan");
  rv_plan_result pr{};
  int rc = run_host_plan(ctx, x, y, n, eps, plan, &pr, nullptr);
  rv_plan_destroy(plan);
  if (rc) return rc;

  fill_result(pr, out);
  int32_t fl = 0;
  uint32_t ni = 0;
  const int32_t pid = 0;
  const int64_t mw = 0;
  rc = run_refine(ctx, x, y, offs, 1, &pid, eps, out->q_cell, ctx->cfg.refine_rounds, &mw, mask,
                  out->q, &fl, &ni);
  ctx->mark("refine");
  ctx->trace = nullptr;
  if (rc) return rc;
  out->flags |= fl;
  out->n_inliers = ni;
  RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  RV_SYNC(cudaEventSynchronize(ctx->ev1), "event");
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  out->ms = ms;
  ctx->fill_counters(*out);
  return RV_OK;
}


// ---- NEXT-2: several rotations (greedy peaks with suppression, reading R16) --------------------
int solve_multi_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                     int32_t levels, int32_t K, double rho, rv_result* out, int32_t* n_found) {
  if (int rc = validate_common(ctx, x, y, eps, levels)) return rc;
  if (!out || !n_found) return ctx->fail(RV_EINVAL, "out and n_found must be non-null");
  if (K < 1 || K > 64) return ctx->fail(RV_EINVAL, "K must lie in [1, 64], got %d", K);
  if (!(rho >= 0.0) || !(rho <= 3.141592653589793))
    return ctx->fail(RV_EINVAL, "rho must lie in [0, pi], got %g", rho);
  if (n < 2 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  *n_found = 0;
  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaEventRecord(ctx->ev0, s), "event");
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  CountCache cache;
  std::vector<double> excl;  // earlier peaks' block-centre rotations
  int32_t found = 0;
  // one GPU: every peak is a one-pass device solve with the earlier peaks' balls excluded
  // (rv_geom.h excl_dropped / excl_rank: the host planner's rules); a solve the one-pass loop
  // hands back (capacity, re-dive) runs on the host planner below
  const int32_t lev = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
  const std::vector<int32_t> ch(ctx->chain.end() - lev, ctx->chain.end());
  const bool dev = one_pass_applies(ctx, 1) && ctx->effective_world() == 1 && !ctx->comm &&
                   dplan_applies(ctx, lev, ch[0], eps);
  float dev_ms = 0;
  bool setup_done = false;  // (each one-pass solve runs its own setup)
  bool l0_ok = false;       // the last one-pass solve completed: its setup and level 0 are valid
  for (int32_t k = 0; k < K; ++k) {
    if (dev) {
      std::vector<double> eq(excl);
      for (int32_t e = 0; e < k; ++e) {
        double* q = eq.data() + 4 * e;
        const double nq = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        for (int c = 0; c < 4; ++c) q[c] /= nq;
      }
      RV_CUDA(ctx->excl_q.ensure(std::max<size_t>(4, eq.size())), "allocating");
      if (k > 0)
        RV_CUDA(cudaMemcpyAsync(ctx->excl_q.p, eq.data(), eq.size() * 8, cudaMemcpyHostToDevice, s),
                "H2D");
      const rv::Excl ex{ctx->excl_q.p, k, rho, std::cos(rho / 2.0)};
      rv_result r{};
      bool redo = false;
      ctx->reuse_l0 = l0_ok;  // the previous peak ran one pass on this input
      const int rc1 = solve_one_pass(ctx, x, y, n, eps, ch, &r, nullptr, &redo, &ex);
      ctx->reuse_l0 = false;
      if (rc1) return rc1;
      l0_ok = !redo;
      if (!redo) {
        dev_ms += r.ms;
        if (r.votes == 0 && r.n_tied == 0) break;  // every block suppressed
        out[k] = r;
        excl.insert(excl.end(), r.q_cell, r.q_cell + 4);
        ++found;
        continue;
      }
    }
    if (!setup_done && !dev) {
      if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
      if (int rc = check_bad(ctx)) return rc;
      setup_done = true;
    }
    rv_plan* plan = nullptr;
    if (rv_plan_create_ex(ctx->chain.data(), (int32_t)ctx->chain.size(), levels, n, eps,
                          (double)ctx->cfg.guard, excl.data(), k, rho, &plan) != 0)
      return ctx->fail(RV_EINVAL, "invalid search plan");
    rv_plan_result pr{};
    int rc = run_host_plan(ctx, x, y, n, eps, plan, &pr, &cache);
    rv_plan_destroy(plan);
    if (rc) return rc;
    if (pr.votes == 0 && pr.n_tied == 0) break;  // every block suppressed
    rv_result& r = out[k];
    fill_result(pr, &r);
    int32_t fl = 0;
    uint32_t ni = 0;
    const int32_t pid = 0;
    const int64_t mw = 0;
    rc = run_refine(ctx, x, y, offs, 1, &pid, eps, r.q_cell, ctx->cfg.refine_rounds, &mw,
                    nullptr, r.q, &fl, &ni);
    if (rc) return rc;
    r.flags |= fl;
    r.n_inliers = ni;
    excl.insert(excl.end(), r.q_cell, r.q_cell + 4);
    ++found;
  }
  RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  RV_SYNC(cudaEventSynchronize(ctx->ev1), "event");
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  cudaGetLastError();
  for (int32_t k = 0; k < found; ++k) {
    out[k].ms = ms;
    ctx->fill_counters(out[k]);
  }
  *n_found = found;
  (void)dev_ms;
  return RV_OK;
}

// ---- NEXT-3: rigid pose front end ----------------------------------------------------------
// R(q) of P:955-961, row-major, each entry evaluated left to right (the translation bins are

void quat_to_R_rowmajor(const double* q, double* R) {
  const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
  R[0] = q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3;
  R[1] = 2.0 * (q1 * q2 - q0 * q3);
  R[2] = 2.0 * (q1 * q3 + q0 * q2);
  R[3] = 2.0 * (q1 * q2 + q0 * q3);
  R[4] = q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3;
  R[5] = 2.0 * (q2 * q3 - q0 * q1);
  R[6] = 2.0 * (q1 * q3 - q0 * q2);
  R[7] = 2.0 * (q2 * q3 + q0 * q1);
  R[8] = q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3;
}

int translation_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, const double* q,
                     double lo, double hi, double step, int64_t* lin, uint32_t* votes, double* t,
                     double* t_mean) {
  if (!x || !y || !q || !lin || !votes || !t || !t_mean)
    return ctx->fail(RV_EINVAL, "null argument");
  if (n < 1 || !(step > 0.0) || !(hi > lo)) return ctx->fail(RV_EINVAL, "bad translation grid");
  const double inv = 1.0 / step;
  const int64_t Bt = (int64_t)std::llround((hi - lo) * inv);
  if (Bt < 1 || Bt > 1024) return ctx->fail(RV_EINVAL, "translation grid of %lld bins per axis", (long long)Bt);
  const int64_t m = Bt * Bt * Bt;
  cudaStream_t s = ctx->stream;
  if (ctx->rg_acc_m != m) {
    RV_CUDA(ctx->rg_acc.ensure(m), "allocating the translation accumulator");
    RV_CUDA(cudaMemsetAsync(ctx->rg_acc.p, 0, m * 4, s), "memset");  // kept zero afterwards
    ctx->rg_acc_m = m;
  }
  RV_CUDA(ctx->rg_bins.ensure(n), "allocating");
  RV_CUDA(ctx->rg_best.ensure(1), "allocating");
  RV_CUDA(ctx->rg_sums.ensure(3), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->rg_best.p, 0, 8, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->rg_sums.p, 0, 24, s), "memset");
  double R[9];
  quat_to_R_rowmajor(q, R);
  rv::launch_translation(x, y, n, R, lo, inv, Bt, ctx->rg_acc.p, ctx->rg_bins.p, ctx->rg_best.p,
                         ctx->rg_sums.p, s);
  ctx->launches += 4;
  RV_CUDA(cudaGetLastError(), "launching the translation vote");
  unsigned long long hb = 0;
  double hs[3];
  RV_CUDA(cudaMemcpyAsync(&hb, ctx->rg_best.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hs, ctx->rg_sums.p, 24, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "translation vote");
  if (hb == 0) return ctx->fail(RV_EDATA, "no translation candidate inside the grid");
  const int64_t L = (int64_t)(0xffffffffu - (uint32_t)(hb & 0xffffffffu));
  *lin = L;
  *votes = (uint32_t)(hb >> 32);
  const int64_t id[3] = {L / (Bt * Bt), (L / Bt) % Bt, L % Bt};
  for (int r = 0; r < 3; ++r) {
    t[r] = lo + ((double)id[r] + 0.5) * step;
    t_mean[r] = hs[r] / (double)*votes;
  }
  return RV_OK;
}

int rigid_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double mu_t, double eps,
               int32_t levels, double lo, double hi, double step, rv_rigid_result* out,
               int32_t* pair_ij, int64_t pair_cap) {
  if (!x || !y || !out) return ctx->fail(RV_EINVAL, "x, y and out must be non-null");
  if (n < 2 || n > (1 << 20)) return ctx->fail(RV_EINVAL, "n must lie in [2, 2^20]");
  if (!(mu_t >= 0.0)) return ctx->fail(RV_EINVAL, "mu_t must be >= 0");
  cudaStream_t s = ctx->stream;
  std::memset(out, 0, sizeof(*out));
  cudaEvent_t e[4];
  for (auto& v : e) RV_CUDA(cudaEventCreate(&v), "event");
  struct Ev { cudaEvent_t* e; ~Ev() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); } } guard_ev{e};
  RV_CUDA(cudaEventRecord(e[0], s), "event");
  // K9: the kept pairs, in pair order
  const int64_t nb = rv::pairs_ctas(n);
  RV_CUDA(ctx->rg_cnt.ensure(std::max<int64_t>(1, nb)), "allocating");
  RV_CUDA(ctx->rg_off.ensure(nb + 1), "allocating");
  rv::launch_pairs_count(x, y, n, mu_t, ctx->rg_cnt.p, ctx->rg_off.p, s);
  int64_t kept = 0;
  RV_CUDA(cudaMemcpyAsync(&kept, ctx->rg_off.p + nb, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "pair count");
  out->pairs_total = n * (n - 1) / 2;
  out->pairs_kept = kept;
  if (kept < 2) return ctx->fail(RV_EDATA, "only %lld pairs pass the length check", (long long)kept);
  if (kept > ctx->cfg.max_n)
    return ctx->fail(RV_EINVAL, "%lld pairs pass the length check but max_n = %lld",
                     (long long)kept, (long long)ctx->cfg.max_n);
  RV_CUDA(ctx->rg_m.ensure(3 * kept), "allocating pairs");
  RV_CUDA(ctx->rg_n.ensure(3 * kept), "allocating pairs");
  rv::launch_pairs_write(x, y, n, mu_t, ctx->rg_off.p, ctx->rg_m.p, ctx->rg_n.p,
                         (pair_ij && pair_cap >= kept) ? pair_ij : nullptr, s);
  ctx->launches += 3;
  RV_CUDA(cudaGetLastError(), "launching the pair kernels");
  RV_CUDA(cudaEventRecord(e[1], s), "event");
  // the rotation vote on the pairs
  rv_result rot{};
  if (int rc = solve_impl(ctx, ctx->rg_m.p, ctx->rg_n.p, kept, eps, levels, &rot, nullptr))
    return rc;
  RV_CUDA(cudaEventRecord(e[2], s), "event");
  // K10: the translation vote with the refined rotation
  int64_t lin = 0;
  if (int rc = translation_impl(ctx, x, y, n, rot.q, lo, hi, step, &lin, &out->t_votes, out->t,
                                out->t_mean))
    return rc;
  RV_CUDA(cudaEventRecord(e[3], s), "event");
  RV_SYNC(cudaEventSynchronize(e[3]), "event");
  const int64_t Bt = (int64_t)std::llround((hi - lo) / step);
  out->t_cell[0] = (int32_t)(lin / (Bt * Bt));
  out->t_cell[1] = (int32_t)((lin / Bt) % Bt);
  out->t_cell[2] = (int32_t)(lin % Bt);
  std::memcpy(out->q, rot.q, sizeof(out->q));
  out->rot_votes = rot.votes;
  out->rot_inliers = rot.n_inliers;
  cudaEventElapsedTime(&out->ms, e[0], e[3]);
  cudaEventElapsedTime(&out->pairs_ms, e[0], e[1]);
  cudaEventElapsedTime(&out->rot_ms, e[1], e[2]);
  cudaEventElapsedTime(&out->trans_ms, e[2], e[3]);
  return RV_OK;
}

// ---- batched: one launch per mode covers every active problem's request ----------------------
// (BatchReq: rv_ctx.h)

// keep_dev != nullptr: the cnt_a counts stay on the device (copied to keep_dev, request order)
// and nothing is read back (level 0 of a batched solve, reduced by the K4 kernels).
int eval_batch(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode,
               const std::vector<BatchReq>& reqs, std::vector<std::vector<uint32_t>>& ca,
               std::vector<std::vector<uint32_t>>& cb, uint32_t* keep_dev) {
  if (reqs.empty()) return RV_OK;
  int64_t total = 0, upload = 0;
  for (const BatchReq& r : reqs) {
    total += r.m;
    if (!r.full_grid) upload += r.m;
  }
  for (const BatchReq& r : reqs)
    if (r.full_grid && (ctx->grid_list_B != r.B || ctx->grid_list_m != r.m)) {
      RV_CUDA(ctx->grid_list.ensure(r.m), "allocating grid list");
      RV_CUDA(cudaMemcpy(ctx->grid_list.p, r.lins, r.m * 4, cudaMemcpyHostToDevice), "H2D grid");
      ctx->grid_list_B = r.B;
      ctx->grid_list_m = r.m;
    }
  RV_CUDA(ctx->lins.ensure(std::max<int64_t>(1, upload)), "allocating block list");
  RV_CUDA(ctx->cnt.ensure(2 * total), "allocating counts");
  std::vector<int64_t> ncell, ncorr;
  std::vector<rv::VoteSeg> segs;
  int64_t off = 0, uoff = 0;
  for (const BatchReq& r : reqs) {
    rv::VoteSeg sg{};
    sg.lins = r.full_grid ? ctx->grid_list.p : ctx->lins.p + uoff;
    if (!r.full_grid) uoff += r.m;
    sg.cnt_a = ctx->cnt.p + off;
    sg.cnt_b = ctx->cnt.p + total + off;
    sg.koff = koff[r.prob];
    sg.row = rows[r.prob];
    sg.n = (int32_t)(rows[r.prob + 1] - rows[r.prob]);
    sg.B = r.B;
    sg.eps = eps;
    segs.push_back(sg);
    ncell.push_back(r.m);
    ncorr.push_back(sg.n);
    off += r.m;
  }
  std::vector<rv::VoteItem> items;
  std::vector<rv::ABlock> ablocks;
  int groups = 1;
  const bool tc_final = mode == RV_MODE_FINAL && ctx->tc_on;
  const bool use_tc = tc_final || (mode == RV_MODE_BOUND && ctx->tc_on);
  if (use_tc) {
    for (size_t q = 0; q < reqs.size(); ++q) segs[q].koff = ctx->tc_toff[reqs[q].prob];
    std::vector<const void*> keys(segs.size());
    for (size_t q = 0; q < segs.size(); ++q) keys[q] = segs[q].lins;
    build_tc_items(ncell, ncorr, ctx->num_sms, items, ablocks, tc_final ? rv::kTcM / 2 : rv::kTcM,
                   &keys);
  } else if (mode == RV_MODE_EXACT) {
    build_exact_items(ncell, ncorr, items);
  } else {
    groups = build_vote_items(ncell, ncorr, ctx->num_sms * ctx->vote_blocks_per_sm, items,
                              ctx->force_groups);
  }
  RV_CUDA(ctx->vsegs.ensure(segs.size()), "allocating segments");
  RV_CUDA(ctx->vitems.ensure(std::max<size_t>(1, items.size())), "allocating items");
  RV_CUDA(ctx->up.ensure(upload * 4 + segs.size() * sizeof(rv::VoteSeg) +
                         items.size() * sizeof(rv::VoteItem) + 4096), "allocating staging");
  RV_CUDA(ctx->down.ensure(2 * total * 4 + 256), "allocating staging");
  ctx->up.reset();
  uint32_t* hl = ctx->up.take<uint32_t>(std::max<int64_t>(1, upload));
  off = 0;
  for (const BatchReq& r : reqs) {
    if (r.full_grid) continue;
    std::memcpy(hl + off, r.lins, r.m * 4);
    off += r.m;
  }
  rv::VoteSeg* hs = ctx->up.take<rv::VoteSeg>(segs.size());
  std::memcpy(hs, segs.data(), segs.size() * sizeof(rv::VoteSeg));
  rv::VoteItem* hi = ctx->up.take<rv::VoteItem>(std::max<size_t>(1, items.size()));
  if (!items.empty()) std::memcpy(hi, items.data(), items.size() * sizeof(rv::VoteItem));
  cudaStream_t s = ctx->stream;
  if (upload > 0)
    RV_CUDA(cudaMemcpyAsync(ctx->lins.p, hl, upload * 4, cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->vsegs.p, hs, segs.size() * sizeof(rv::VoteSeg),
                          cudaMemcpyHostToDevice, s), "H2D");
  if (!items.empty())
    RV_CUDA(cudaMemcpyAsync(ctx->vitems.p, hi, items.size() * sizeof(rv::VoteItem),
                            cudaMemcpyHostToDevice, s), "H2D");
  const int64_t ncnt = (mode == RV_MODE_FINAL ? 2 : 1) * total;  // cnt_b only in FINAL mode
  RV_CUDA(cudaMemsetAsync(ctx->cnt.p, 0, ncnt * 4, s), "memset");
  if (mode == RV_MODE_EXACT) {
    rv::launch_exact(ctx->k9.p, ctx->stride, x, y, ctx->vsegs.p, ctx->vitems.p,
                     (int32_t)items.size(), ctx->cfg.guard, s);
  } else {
    RV_CUDA(cudaEventRecord(ctx->evv0, s), "event");
    if (use_tc)
      {
        if (int rc = launch_tc(ctx, ablocks, (int32_t)items.size(), tc_final)) return rc;
      }
    else
      rv::launch_vote(mode, groups, ctx->k9.p, ctx->stride, ctx->vsegs.p, ctx->vitems.p,
                      (int32_t)items.size(), ctx->cfg.guard, s);
    RV_CUDA(cudaEventRecord(ctx->evv1, s), "event");
    for (size_t q = 0; q < ncell.size(); ++q) ctx->vote_pairs += (uint64_t)ncell[q] * ncorr[q];
    ctx->vote_launches += 1;
  }
  ctx->launches += items.empty() ? 0 : 1;
  RV_CUDA(cudaGetLastError(), "launching the vote kernel");
  if (keep_dev) {
    RV_CUDA(cudaMemcpyAsync(keep_dev, ctx->cnt.p, total * 4, cudaMemcpyDeviceToDevice, s), "D2D");
    RV_SYNC(cudaStreamSynchronize(s), "batched vote");
    if (mode != RV_MODE_EXACT && !items.empty()) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ctx->evv0, ctx->evv1);
      ctx->vote_ms += ms;
    }
    return RV_OK;
  }
  ctx->down.reset();
  uint32_t* hc = ctx->down.take<uint32_t>(2 * total);
  RV_CUDA(cudaMemcpyAsync(hc, ctx->cnt.p, ncnt * 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "batched vote");
  if (mode != RV_MODE_EXACT && !items.empty()) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->evv0, ctx->evv1);
    ctx->vote_ms += ms;
  }
  off = 0;
  for (const BatchReq& r : reqs) {
    ca[r.prob].assign(hc + off, hc + off + r.m);
    if (mode == RV_MODE_FINAL) cb[r.prob].assign(hc + total + off, hc + total + off + r.m);
    off += r.m;
  }
  return RV_OK;
}

// ---- batched: the level loop on the device (rv_dplan.cu) --------------------------------------
// Vote per-problem block lists that already live on the device: problem p's list is
// dlins + hoff[p] (hcnt[p] blocks), its counts land at dca / dcb + hoff[p]; span = the extent
// of the count arrays to clear.  Asynchronous; the small host arrays go through pageable
// copies (staged by the driver on the call), so nothing host-side needs to outlive it.
int vote_lists(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode, int32_t B,
               const uint32_t* dlins, const std::vector<int64_t>& hoff,
               const std::vector<int32_t>& hcnt, int64_t span, uint32_t* dca, uint32_t* dcb) {
  const int32_t PL = (int32_t)hcnt.size();
  const bool use_tc = ctx->tc_on && mode != RV_MODE_EXACT;
  const bool tc_final = use_tc && mode == RV_MODE_FINAL;
  std::vector<int64_t> ncell, ncorr;
  std::vector<rv::VoteSeg> segs;
  for (int32_t p = 0; p < PL; ++p) {
    if (hcnt[p] == 0) continue;
    rv::VoteSeg sg{};
    sg.lins = dlins + hoff[p];
    sg.cnt_a = dca + hoff[p];
    sg.cnt_b = dcb + hoff[p];
    sg.koff = use_tc ? ctx->tc_toff[p] : koff[p];
    sg.row = rows[p];
    sg.n = (int32_t)(rows[p + 1] - rows[p]);
    sg.B = B;
    sg.eps = eps;
    segs.push_back(sg);
    ncell.push_back(hcnt[p]);
    ncorr.push_back(sg.n);
  }
  if (segs.empty()) return RV_OK;
  std::vector<rv::VoteItem> items;
  std::vector<rv::ABlock> ablocks;
  int groups = 1;
  if (use_tc)
    build_tc_items(ncell, ncorr, ctx->num_sms, items, ablocks, tc_final ? rv::kTcM / 2 : rv::kTcM);
  else if (mode == RV_MODE_EXACT)
    build_exact_items(ncell, ncorr, items);
  else
    groups = build_vote_items(ncell, ncorr, ctx->num_sms * ctx->vote_blocks_per_sm, items,
                              ctx->force_groups);
  if (items.empty()) return RV_OK;
  RV_CUDA(ctx->vsegs.ensure(segs.size()), "allocating segments");
  RV_CUDA(ctx->vitems.ensure(items.size()), "allocating items");
  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaMemcpyAsync(ctx->vsegs.p, segs.data(), segs.size() * sizeof(rv::VoteSeg),
                          cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->vitems.p, items.data(), items.size() * sizeof(rv::VoteItem),
                          cudaMemcpyHostToDevice, s), "H2D");
  if (span > 0) {  // span 0: the caller's list kernel zeroed the count slots
    RV_CUDA(cudaMemsetAsync(dca, 0, span * 4, s), "memset");
    if (mode == RV_MODE_FINAL) RV_CUDA(cudaMemsetAsync(dcb, 0, span * 4, s), "memset");
  }
  if (mode == RV_MODE_EXACT) {
    rv::launch_exact(ctx->k9.p, ctx->stride, x, y, ctx->vsegs.p, ctx->vitems.p,
                     (int32_t)items.size(), ctx->cfg.guard, s);
  } else {
    ctx->collect_vote_ms();
    RV_CUDA(cudaEventRecord(ctx->evv0, s), "event");
    if (use_tc)
      {
        if (int rc = launch_tc(ctx, ablocks, (int32_t)items.size(), tc_final)) return rc;
      }
    else
      rv::launch_vote(mode, groups, ctx->k9.p, ctx->stride, ctx->vsegs.p, ctx->vitems.p,
                      (int32_t)items.size(), ctx->cfg.guard, s);
    RV_CUDA(cudaEventRecord(ctx->evv1, s), "event");
    ctx->vote_pending = true;
    for (size_t q = 0; q < ncell.size(); ++q) ctx->vote_pairs += (uint64_t)ncell[q] * ncorr[q];
    ctx->vote_launches += 1;
  }
  ctx->launches += 1;
  RV_CUDA(cudaGetLastError(), "launching the vote kernel");
  return RV_OK;
}

}  // namespace rvi
