// rv_level_loop.cpp -- the certified level loop on the device (rv_dplan.cu) for P problems,
// ancestor culling (rv_cull.cu), the sharded one-problem levels, and the batched entry.
#include "rv_ctx.h"

#include <functional>

namespace rvi {

// Culling state for a level 0 at B0 (grid_host holds its m0 candidates): the lin -> row table,
// the pair counter (zeroed), the bitmask geometry.
int cull_prepare(rv_ctx* ctx, int32_t B0, int64_t m0, int32_t PL) {
  if (ctx->lut0_B != B0) {
    std::vector<int32_t> lut((size_t)B0 * B0 * B0, -1);
    for (int64_t a = 0; a < m0; ++a) lut[ctx->grid_host[a]] = (int32_t)a;
    RV_CUDA(ctx->lut0.ensure(lut.size()), "allocating");
    RV_CUDA(cudaMemcpy(ctx->lut0.p, lut.data(), lut.size() * 4, cudaMemcpyHostToDevice), "H2D lut");
    // ancestor groups (rotvote_plan.h rv_cull_groups): level-0 blocks with equal
    // (i / gi, j / gj, k / gk), numbered in row order
    const int32_t* gs = ctx->cull_gshape;
    const int64_t G = rv_cull_groups(B0, gs[0], gs[1], gs[2], nullptr, nullptr, nullptr);
    if (G < 1) return ctx->fail(RV_EINVAL, "invalid ancestor group shape");
    std::vector<int32_t> g_of((size_t)m0), go((size_t)G + 1), gm((size_t)m0);
    rv_cull_groups(B0, gs[0], gs[1], gs[2], g_of.data(), go.data(), gm.data());
    std::vector<int32_t> lg((size_t)B0 * B0 * B0, -1);
    for (int64_t a = 0; a < m0; ++a) lg[ctx->grid_host[a]] = g_of[a];
    RV_CUDA(ctx->lutg.ensure(lg.size()), "allocating");
    RV_CUDA(ctx->goff.ensure(go.size()), "allocating");
    RV_CUDA(ctx->gmem.ensure(gm.size()), "allocating");
    RV_CUDA(cudaMemcpy(ctx->lutg.p, lg.data(), lg.size() * 4, cudaMemcpyHostToDevice), "H2D lut");
    RV_CUDA(cudaMemcpy(ctx->goff.p, go.data(), go.size() * 4, cudaMemcpyHostToDevice), "H2D lut");
    RV_CUDA(cudaMemcpy(ctx->gmem.p, gm.data(), gm.size() * 4, cudaMemcpyHostToDevice), "H2D lut");
    ctx->cull_G_grouped = G;
    ctx->lut0_B = B0;
    ctx->cull_s.clear();  // recomputed below for this B0
  }
  {
    const int W = ctx->effective_world();
    if ((int64_t)ctx->cull_s.size() != W + 1) {
      // rotvote_plan.h rv_cull_partition: level-0 slices of whole groups, owned group ranges
      ctx->cull_s.assign(W + 1, 0);
      ctx->cull_g.assign(W + 1, 0);
      const int32_t* gs = ctx->cull_gshape;
      if (rv_cull_partition(B0, gs[0], gs[1], gs[2], W, ctx->cull_s.data(), ctx->cull_g.data()))
        return ctx->fail(RV_EINVAL, "invalid culling partition");
    }
  }
  // group unions for K3-CT (with per-ancestor lists an item would fill a quarter of its 128
  // rows); a split problem (ctx->split_one) uses the slab-aligned slices above, a rank's share
  // of a batch runs like a one-rank batch
  ctx->cull_grouped = ctx->cull_tc;
  ctx->cull_G = ctx->cull_grouped ? ctx->cull_G_grouped : m0;
  RV_CUDA(ctx->c_pairs.ensure(1), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->c_pairs.p, 0, 8, ctx->stream), "memset");
  RV_CUDA(ctx->dp_err.ensure(1), "allocating");
  int64_t wmax = 0;
  for (int32_t p = 0; p < PL; ++p)
    wmax = std::max<int64_t>(wmax, (ctx->tc_toff[p + 1] - ctx->tc_toff[p]) / 32);
  ctx->cull_B0 = B0;
  ctx->cull_m0 = m0;
  ctx->cull_wpc_max = wmax;
  return RV_OK;
}

// After the level-0 vote wrote the bitmasks: the index lists L(a) (row offsets, one read of
// their total, the compaction), and ctx->cull_ready.  Culling is skipped (the solve goes on
// unculled) when the lists would exceed 2^29 entries or a quarter of the level-0 pairs (then
// the ancestor lists cut too little for the gather to pay).
int cull_build_lists(rv_ctx* ctx, int32_t PL, int64_t m0, const uint32_t* l0cnt,
                     bool force) {
  cudaStream_t s = ctx->stream;
  rv::CullGroups gr;
  if (ctx->cull_grouped) gr = rv::CullGroups{ctx->goff.p, ctx->gmem.p, ctx->cull_G};
  const int64_t NB = (int64_t)PL * ctx->cull_G;
  RV_CUDA(ctx->c_lofs.ensure(NB + 1), "allocating");
  rv::launch_cull_rows(l0cnt, PL, m0, ctx->c_lofs.p, s, gr);
  ctx->launches += 1;
  ctx->down.reset();
  int64_t* ht = ctx->down.take<int64_t>(1);
  RV_CUDA(cudaMemcpyAsync(ht, ctx->c_lofs.p + NB, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "level-0 lists");
  const int64_t total = *ht;
  const double pairs0 = (double)m0 * (double)(ctx->tc_toff[PL] - ctx->tc_toff[0]);
  ctx->cull_ready = false;
  if (total > ((int64_t)1 << 29) || (!force && (double)total > 0.25 * pairs0)) return RV_OK;
  RV_CUDA(ctx->c_lidx.ensure(total + 4), "allocating level-0 lists");
  RV_CUDA(ctx->c_fill.ensure(NB), "allocating");
  int64_t row_lo = 0, row_hi = NB;
  if (ctx->comm && ctx->split_one) {  // this rank's level-0 slice / groups
    if (ctx->cull_grouped) {
      row_lo = ctx->cull_g[ctx->cfg.rank];
      row_hi = ctx->cull_g[ctx->cfg.rank + 1];
    } else {
      const int64_t c0 = (m0 + ctx->cfg.world - 1) / ctx->cfg.world;
      row_lo = (int64_t)ctx->cfg.rank * c0;
      row_hi = std::min<int64_t>(m0, row_lo + c0);
    }
  }
  rv::launch_cull_compact(ctx->cbits.p, ctx->toffs.p, PL, m0, ctx->cull_wpc_max, ctx->c_lofs.p,
                          ctx->c_fill.p, ctx->c_lidx.p, s, row_lo, row_hi, gr);
  ctx->launches += 1;
  // list lengths: the level-0 counts, or the union sizes the compaction counted
  ctx->cull_l0cnt = ctx->cull_grouped ? reinterpret_cast<const uint32_t*>(ctx->c_fill.p) : l0cnt;
  ctx->cull_ready = true;
  ctx->ct_prefetched = false;
  return RV_OK;
}

// true when the device level loop applies: >= 2 levels and a cached level-0 background
bool dplan_applies(rv_ctx* ctx, int32_t levels_eff, int32_t B0, double eps) {
  if (levels_eff < 2 || ctx->host_plan) return false;
  int64_t mbg = 0;
  return rv_plan_l0_background(B0, eps, &mbg) != nullptr && mbg > 0;
}

// Vote one level of per-problem device lists (rv::DpList).  K3-TC and K5: the items are
// built on the device (dp_launch_items) and the kernels read their counts there -- no host
// round trip.  FP32 K3 (tensor_vote = 0): the counts and bases are read back and the items
// built on the host (vote_lists).  The caller has zeroed the count slots.
// emit_bits (level 0 of a culled solve): K3-TC also writes the level-0 pass bitmasks.  Once
// they exist (ctx->cull_ready), BOUND / FINAL levels go to K3-C (rv_cull.cu), items planned on
// the device.
int vote_level(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode, int32_t B,
               const rv::DpList& Ld, int32_t PL, int64_t entries_bound, int64_t nmax,
               bool emit_bits, const rv::DiveStep* dive) {
  cudaStream_t s = ctx->stream;
  if (ctx->cull_ready && mode != RV_MODE_EXACT) {
    const int64_t eb = std::max<int64_t>(1, entries_bound);
    const int64_t nb = (int64_t)PL * ctx->cull_G;  // buckets: (problem, list row)
    const int64_t mi = rv::cull_items_bound(eb, ctx->num_sms);
    RV_CUDA(ctx->c_act.ensure(PL + 1), "allocating");
    RV_CUDA(ctx->c_acnt.ensure(nb), "allocating");
    RV_CUDA(ctx->c_aoff.ensure(nb + 1), "allocating");
    RV_CUDA(ctx->c_ioff.ensure(nb + 1), "allocating");
    RV_CUDA(ctx->c_tanc.ensure(eb), "allocating");
    RV_CUDA(ctx->c_tslot.ensure(eb), "allocating");
    const int64_t npos = eb + 7 * nb + 16;  // bucket positions are padded to multiples of 8
    RV_CUDA(ctx->c_cidx.ensure(npos), "allocating");
    if (!ctx->cull_grouped) RV_CUDA(ctx->c_phi.ensure(npos * 12), "allocating");  // K3-C only
    // (+256 rows: K3-CT's A tiles read up to 2 x 128 rows from an item's first)
    if (ctx->cull_grouped) RV_CUDA(ctx->c_tphi.ensure((npos * 2 + 256) * 64), "allocating");
    RV_CUDA(ctx->c_icnt.ensure(2), "allocating");
    RV_CUDA(ctx->c_work.ensure(1), "allocating");
    RV_CUDA(ctx->vsegs.ensure(PL), "allocating segments");
    RV_CUDA(ctx->c_items.ensure(mi), "allocating K3-C items");
    const rv::CullScratch cs{ctx->c_act.p, ctx->c_acnt.p, ctx->c_aoff.p, ctx->c_ioff.p,
                             ctx->c_tanc.p, ctx->c_tslot.p, ctx->c_cidx.p, ctx->c_phi.p,
                             ctx->c_icnt.p, ctx->c_work.p,
                             ctx->cull_grouped ? ctx->c_tphi.p : nullptr,
                             ctx->cfg.guard + kTcExtraGuard, ctx->cull_na};
    const int nl = rv::launch_cull_items(Ld, ctx->rows.p, ctx->toffs.p, PL, B, ctx->cull_B0,
                                         ctx->cull_grouped ? ctx->lutg.p : ctx->lut0.p,
                                         ctx->cull_G, ctx->cull_l0cnt,
                                         ctx->c_lofs.p, ctx->k12.p, eps, mode, ctx->cfg.guard,
                                         ctx->num_sms, cs, ctx->vsegs.p, ctx->c_items.p, eb, mi,
                                         ctx->dp_err.p, s, ctx->cull_own_lo, ctx->cull_own_hi,
                                         dive, ctx->cull_pre_act);
    if (nl < 0) return ctx->fail(RV_ECUDA, "internal: a folded dive level needs the small planner");
    ctx->launches += nl;
#ifndef RV_CT_PREFETCH
#define RV_CT_PREFETCH 0  // measured: no gain (K3-CT 0.843 vs 0.844 ms), +25 us
#endif
    if (RV_CT_PREFETCH && ctx->cull_grouped && !ctx->ct_prefetched) {  // first culled level
      rv::launch_l2_prefetch(ctx->tctab_rm.p, (ctx->tc_toff.back() + 8) * 64, s);
      ctx->launches += 1;
      ctx->ct_prefetched = true;
    }
    cudaEvent_t e0, e1;
    RV_CUDA(ctx->cev_pair(&e0, &e1), "event");
    RV_CUDA(ctx->record(e0, s), "event");
    if (ctx->cull_grouped)  // K3-CT
      rv::launch_vote_cull_tc(mode, ctx->vsegs.p, ctx->c_items.p, ctx->c_icnt.p, ctx->tctab_rm.p,
                              ctx->tc_toff.back(), ctx->c_tphi.p, ctx->c_cidx.p, ctx->c_lidx.p,
                              ctx->c_pairs.p, ctx->num_sms, s,
                              ctx->c_work.p, ctx->cfg.ct_sched == 1);
    else
      rv::launch_vote_cull(mode, ctx->vsegs.p, ctx->c_items.p, ctx->c_icnt.p, ctx->c_work.p,
                           ctx->c_pairs.p, ctx->c_phi.p, ctx->c_cidx.p, ctx->c_lidx.p,
                           ctx->cfg.guard, ctx->num_sms, s);
    RV_CUDA(ctx->record(e1, s), "event");
    ctx->launches += 1;
    ctx->cull_launches += 1;
    ctx->cull_tc_launches += ctx->cull_grouped ? 1 : 0;
    RV_CUDA(cudaGetLastError(), "launching the culled vote");
    return RV_OK;
  }
  if (ctx->tc_on || mode == RV_MODE_EXACT) {
    const int im = mode == RV_MODE_EXACT ? 2 : mode == RV_MODE_FINAL ? 1 : 0;
    int64_t mi = 0, ma = 0;
    rv::dp_items_bound(im, entries_bound, PL, nmax, ctx->num_sms, &mi, &ma);
    RV_CUDA(ctx->vsegs.ensure(PL), "allocating segments");
    RV_CUDA(ctx->vitems.ensure(mi), "allocating items");
    RV_CUDA(ctx->ablk.ensure(ma), "allocating A blocks");
    if (im != 2) RV_CUDA(ctx->atab.ensure(ma * (size_t)rv::kTcABlockBytes), "allocating A table");
    RV_CUDA(ctx->dp_ioff.ensure(PL + 1), "allocating");
    RV_CUDA(ctx->dp_aoff.ensure(PL + 1), "allocating");
    RV_CUDA(ctx->dp_icnt.ensure(4), "allocating");
    rv::dp_launch_items(Ld, ctx->rows.p, im == 2 ? ctx->koffs.p : ctx->toffs.p, PL, B, eps, im,
                        ctx->num_sms, ctx->vsegs.p, ctx->dp_ioff.p, ctx->dp_aoff.p, ctx->dp_icnt.p,
                        ctx->vitems.p, ctx->ablk.p, mi, ma, ctx->dp_err.p, s,
                        emit_bits ? ctx->cbits.p : nullptr, ctx->cull_m0);
    ctx->launches += 2;
    if (im == 2) {
      rv::launch_exact(ctx->k9.p, ctx->stride, x, y, ctx->vsegs.p, ctx->vitems.p, 0,
                       ctx->cfg.guard, s, ctx->dp_icnt.p);
      ctx->launches += 1;
    } else {
      cudaEvent_t e0, e1;
      RV_CUDA(ctx->ev_pair(&e0, &e1), "event");
      RV_CUDA(ctx->record(e0, s), "event");
      rv::launch_vote_tc(ctx->tctab.p, ctx->atab.p, ctx->ablk.p, 0, ctx->vsegs.p, ctx->vitems.p, 0,
                         ctx->cfg.guard + kTcExtraGuard, nullptr, 0, s, im == 1, ctx->dp_icnt.p,
                         emit_bits);
      RV_CUDA(ctx->record(e1, s), "event");
      ctx->launches += 2;
      ctx->vote_launches += 1;
    }
    RV_CUDA(cudaGetLastError(), "launching a batched vote");
    return RV_OK;
  }
  // FP32 path: host-built items from the read-back counts
  std::vector<int32_t> hcnt(PL);
  std::vector<int64_t> hoff(PL + 1);
  RV_CUDA(cudaMemcpyAsync(hcnt.data(), Ld.cnt, PL * 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hoff.data(), Ld.base, (PL + 1) * 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "batched level");
  ctx->collect_vote_ms();
  return vote_lists(ctx, x, y, rows, koff, eps, mode, B, Ld.lins, hoff, hcnt, 0, Ld.ca, Ld.cb);
}

// One level of a ONE-problem list sharded over ranks: rank r votes the entries
// [r * chunk, (r + 1) * chunk) and one in-place ncclAllGather per count array assembles the
// level (the count arrays hold >= W * chunk entries from 0).  The loopback emulation
// (emulate_world) votes every rank's slice here, one launch sequence per slice.
int vote_level_sharded(rv_ctx* ctx, const float* x, const float* y,
                       const std::vector<int64_t>& rows, const std::vector<int64_t>& koff,
                       double eps, int32_t mode, int32_t B, const rv::DpList& Ld, int64_t chunk,
                       int64_t nmax, bool emit_bits = false) {
  cudaStream_t s = ctx->stream;
  const bool nccl_path = ctx->comm != nullptr;
  const int W = ctx->effective_world();
  const int r_lo = nccl_path ? ctx->cfg.rank : 0, r_hi = nccl_path ? r_lo + 1 : W;
  RV_CUDA(ctx->dp_sbase.ensure(2), "allocating");
  RV_CUDA(ctx->dp_scnt.ensure(1), "allocating");
  for (int r = r_lo; r < r_hi; ++r) {
    rv::dp_launch_slice(Ld.shared ? nullptr : Ld.base, Ld.cnt, Ld.shared_m, (int64_t)r * chunk, chunk,
                        ctx->dp_sbase.p, ctx->dp_scnt.p, s);
    ctx->launches += 1;
    const rv::DpList Ls{Ld.lins, 0, 0, ctx->dp_sbase.p, ctx->dp_scnt.p, Ld.ca, Ld.cb};
    if (int rc = vote_level(ctx, x, y, rows, koff, eps, mode, B, Ls, 1, chunk, nmax, emit_bits))
      return rc;
  }
  if (nccl_path) {
    const size_t off = (size_t)ctx->cfg.rank * chunk;
    for (int a = 0; a < (mode == RV_MODE_FINAL ? 2 : 1); ++a) {
      uint32_t* buf = a == 0 ? Ld.ca : Ld.cb;
      ncclResult_t nr = nccl().AllGather(buf + off, buf, (size_t)chunk, ncclUint32, ctx->comm, s);
      if (nr != ncclSuccess)
        return ctx->fail(RV_ENCCL, "ncclAllGather: %s", nccl().GetErrorString(nr));
    }
  }
  return RV_OK;
}

// Level 0 of a culled ONE-problem solve over ranks: rank r votes (with the pass bitmasks) the
// i-slab-aligned rows [cull_s[r], cull_s[r+1]) of the shared level-0 list, so every group of
// the rank's culled levels has all its members' bitmasks here; one in-place ncclAllReduce(sum)
// assembles the counts (the slices are disjoint and the array was zeroed).  Loopback: every
// rank's slice in turn.
int vote_level0_slabs(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
                      const std::vector<int64_t>& koff, double eps, int32_t B0, const rv::DpList& Ld,
                      int64_t m0, int64_t nmax) {
  cudaStream_t s = ctx->stream;
  const bool nccl_path = ctx->comm != nullptr;
  const int W = ctx->effective_world();
  const int r_lo = nccl_path ? ctx->cfg.rank : 0, r_hi = nccl_path ? r_lo + 1 : W;
  RV_CUDA(ctx->dp_sbase.ensure(2), "allocating");
  RV_CUDA(ctx->dp_scnt.ensure(1), "allocating");
  for (int r = r_lo; r < r_hi; ++r) {
    const int64_t r0 = ctx->cull_s[r], len = ctx->cull_s[r + 1] - r0;
    if (len <= 0) continue;
    rv::dp_launch_slice(nullptr, Ld.cnt, Ld.shared_m, r0, len, ctx->dp_sbase.p, ctx->dp_scnt.p, s);
    ctx->launches += 1;
    const rv::DpList Ls{Ld.lins, 0, 0, ctx->dp_sbase.p, ctx->dp_scnt.p, Ld.ca, Ld.cb};
    if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, Ls, 1, len, nmax, true))
      return rc;
  }
  if (nccl_path) {
    ncclResult_t nr = nccl().AllReduce(Ld.ca, Ld.ca, (size_t)m0, ncclUint32, ncclSum, ctx->comm, s);
    if (nr != ncclSuccess) return ctx->fail(RV_ENCCL, "ncclAllReduce: %s", nccl().GetErrorString(nr));
  }
  return RV_OK;
}

// A culled level of a ONE-problem list over ranks: rank r votes the blocks whose level-0
// ancestor is one of the rows it voted (and compacted) at level 0, [r c0, (r+1) c0); the other
// blocks' counts stay zero and one in-place ncclAllReduce(sum) per count array assembles the
// level (each block is voted by exactly one rank).  Loopback: every rank's share in turn.
int vote_level_owned(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
                     const std::vector<int64_t>& koff, double eps, int32_t mode, int32_t B,
                     const rv::DpList& Ld, int64_t entries, int64_t nmax) {
  const bool nccl_path = ctx->comm != nullptr;
  const int W = ctx->effective_world();
  const int r_lo = nccl_path ? ctx->cfg.rank : 0, r_hi = nccl_path ? r_lo + 1 : W;
  const int64_t c0 = (ctx->cull_G + W - 1) / W;
  for (int r = r_lo; r < r_hi; ++r) {
    if (ctx->cull_grouped) {  // the groups whose members this rank voted at level 0
      ctx->cull_own_lo = ctx->cull_g[r];
      ctx->cull_own_hi = ctx->cull_g[r + 1];
    } else {
      ctx->cull_own_lo = (int64_t)r * c0;
      ctx->cull_own_hi = std::min<int64_t>(ctx->cull_G, (int64_t)(r + 1) * c0);
    }
    int rc = vote_level(ctx, x, y, rows, koff, eps, mode, B, Ld, 1, entries, nmax);
    ctx->cull_own_lo = 0;
    ctx->cull_own_hi = INT64_MAX;
    if (rc) return rc;
  }
  if (nccl_path) {
    for (int a = 0; a < (mode == RV_MODE_FINAL ? 2 : 1); ++a) {
      uint32_t* buf = a == 0 ? Ld.ca : Ld.cb;
      ncclResult_t nr = nccl().AllReduce(buf, buf, (size_t)entries, ncclUint32, ncclSum, ctx->comm,
                                         ctx->stream);
      if (nr != ncclSuccess)
        return ctx->fail(RV_ENCCL, "ncclAllReduce: %s", nccl().GetErrorString(nr));
    }
  }
  return RV_OK;
}

// The certified search of rv_plan.cpp for PL problems at once, every decision on the device
// (rv_dplan.cu).  Host round trips: one per branch-and-bound level (the size of the next
// child region) and one at the end; with K3-TC the items are built on the device.
// ch = the `levels` resolutions searched (ch.size() >= 2).  Fills res[p].
// before_sync (optional) enqueues more work (the refinement) between the finalize kernels and
// the one final wait; the data check of run_setup (ctx->bad) is read back with the finalize.
int solve_batched_dplan(rv_ctx* ctx, const float* x, const float* y,
                        const std::vector<int64_t>& rows, const std::vector<int64_t>& koff,
                        int32_t PL, double eps, const std::vector<int32_t>& ch,
                        std::vector<rv_plan_result>& res, Trace& tr,
                        const std::function<int()>& before_sync) {
  const int L = (int)ch.size();
  cudaStream_t s = ctx->stream;
  int64_t nmax = 0;
  for (int32_t p = 0; p < PL; ++p) nmax = std::max<int64_t>(nmax, rows[p + 1] - rows[p]);
  // one problem on several ranks: every level's list is built identically on every rank
  // (ordered expansion) and its votes are sharded (vote_level_sharded)
  const int W = ctx->effective_world();
  const bool shard = ctx->split_one;
  if (shard && PL != 1) return ctx->fail(RV_ECUDA, "internal: a split solve has one problem");
  const int64_t slack = shard ? W : 0;  // count arrays hold W * ceil(m / W) >= m entries
  std::vector<int64_t> phase_chunk;       // per phase: the shard chunk (0: not sharded)
  auto vote = [&](int32_t mode, int32_t B, const rv::DpList& Ld, int64_t entries) -> int {
    if (!shard) return vote_level(ctx, x, y, rows, koff, eps, mode, B, Ld, PL, entries, nmax);
    if (ctx->cull_ready)  // culled levels: sharded by ancestor ownership
      return vote_level_owned(ctx, x, y, rows, koff, eps, mode, B, Ld, entries, nmax);
    return vote_level_sharded(ctx, x, y, rows, koff, eps, mode, B, Ld, (entries + W - 1) / W, nmax);
  };
  // per-phase block counts, kept on the device and read once at the end
  const int max_ph = 3 * L + 1;
  RV_CUDA(ctx->dp_phase.ensure((size_t)max_ph * PL), "allocating");
  int nph = 0;
  std::vector<char> ph_optional;  // re-dive phases: absent for problems that did not re-dive
  auto keep_phase = [&](const int32_t* dcnt, bool optional = false) -> int {
    RV_CUDA(cudaMemcpyAsync(ctx->dp_phase.p + (size_t)nph * PL, dcnt, PL * 4,
                            cudaMemcpyDeviceToDevice, s), "D2D");
    ++nph;
    ph_optional.push_back(optional ? 1 : 0);
    return RV_OK;
  };
  ctx->ev_reset();
  RV_CUDA(ctx->dp_err.ensure(1), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->dp_err.p, 0, 4, s), "memset");
  // ---- level 0: every problem votes the full candidate grid; counts stay on the device
  const int32_t B0 = ch[0];
  const int64_t m0 = rv_grid_candidates(B0, nullptr, 0);
  if (ctx->grid_host_B != B0) {
    ctx->grid_host.resize(m0);
    rv_grid_candidates(B0, ctx->grid_host.data(), m0);
    ctx->grid_host_B = B0;
  }
  int64_t mbg = 0;
  const double* bgh = rv_plan_l0_background(B0, eps, &mbg);
  if (!bgh || mbg != m0) return ctx->fail(RV_ECUDA, "internal: level-0 background unavailable");
  RV_CUDA(ctx->l0cnt.ensure((size_t)PL * m0 + slack), "allocating level-0 counts");
  if (ctx->l0bg_B != B0 || ctx->l0bg_eps != eps || ctx->l0bg.cap < (size_t)m0) {
    RV_CUDA(ctx->l0bg.ensure(m0), "allocating");
    RV_CUDA(cudaMemcpy(ctx->l0bg.p, bgh, m0 * sizeof(double), cudaMemcpyHostToDevice),
            "H2D background");
    ctx->l0bg_B = B0;
    ctx->l0bg_eps = eps;
  }
  if (ctx->grid_list_B != B0 || ctx->grid_list_m != m0) {
    RV_CUDA(ctx->grid_list.ensure(m0), "allocating grid list");
    RV_CUDA(cudaMemcpy(ctx->grid_list.p, ctx->grid_host.data(), m0 * 4, cudaMemcpyHostToDevice),
            "H2D grid");
    ctx->grid_list_B = B0;
    ctx->grid_list_m = m0;
  }
  // ancestor culling: level 0 writes the pass bitmasks (every rank votes all of level 0, so
  // every rank holds every ancestor's list); bitmasks capped at 4 GiB
  ctx->cull_ready = false;
  const int64_t tpad = ctx->tc_on ? ctx->tc_toff.back() : 0;
  const bool cull = ctx->cull_on && (int64_t)ctx->tc_toff.size() == PL + 1 &&
                    nmax >= ctx->cull_min_n && (int64_t)PL * m0 <= ((int64_t)1 << 22) &&
                    (double)m0 * (double)(tpad / 32) * 4.0 <= 4294967296.0;
  if (cull) {
    RV_CUDA(ctx->cbits.ensure((size_t)m0 * (size_t)(tpad / 32)), "allocating level-0 bitmasks");
    if (int rc = cull_prepare(ctx, B0, m0, PL)) return rc;
  }
  bool culled = false;  // the finer levels run K3-C (the lists were built)
  if (cull) {
    RV_CUDA(cudaMemsetAsync(ctx->l0cnt.p, 0, ((size_t)PL * m0 + slack) * 4, s), "memset");
    const rv::DpList l0{ctx->grid_list.p, 1, m0, nullptr, nullptr, ctx->l0cnt.p, ctx->l0cnt.p};
    if (shard && ctx->cull_grouped) {  // slab-aligned slices (whole groups per rank)
      if (int rc = vote_level0_slabs(ctx, x, y, rows, koff, eps, B0, l0, m0, nmax)) return rc;
    } else if (shard) {  // each rank votes (and later compacts) its slice of level 0
      if (int rc = vote_level_sharded(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, l0,
                                      (m0 + W - 1) / W, nmax, true))
        return rc;
    } else if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, l0, PL, PL * m0,
                                   nmax, true)) {
      return rc;
    }
    if (int rc = cull_build_lists(ctx, PL, m0, ctx->l0cnt.p)) return rc;
    culled = ctx->cull_ready;
  } else if (ctx->tc_on || shard) {
    RV_CUDA(cudaMemsetAsync(ctx->l0cnt.p, 0, ((size_t)PL * m0 + slack) * 4, s), "memset");
    const rv::DpList l0{ctx->grid_list.p, 1, m0, nullptr, nullptr, ctx->l0cnt.p, ctx->l0cnt.p};
    if (int rc = vote(RV_MODE_BOUND, B0, l0, PL * m0)) return rc;
  } else {
    std::vector<BatchReq> g0(PL);
    for (int32_t p = 0; p < PL; ++p) g0[p] = {p, B0, RV_MODE_BOUND, m0, ctx->grid_host.data(), true};
    std::vector<std::vector<uint32_t>> unused;
    if (int rc = eval_batch(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, g0, unused, unused,
                            ctx->l0cnt.p))
      return rc;
  }
  RV_CUDA(ctx->l0idx.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_pick.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_lb.ensure(PL), "allocating");
  rv::launch_l0_argmax(ctx->l0cnt.p, m0, ctx->grid_list.p, B0, ctx->l0bg.p, ctx->rows.p, PL,
                       ctx->l0idx.p, s);
  ctx->launches += 1;
  tr.mark("  level 0");
  std::vector<int64_t> hbase(PL + 1);
  // ---- dive: the 27-neighbourhood of the pick, level by level; lb* at the finest level
  for (int l = 1; l < L; ++l) {
    const int32_t Bp = ch[l - 1], f = ch[l] / ch[l - 1], cap = 27 * f * f * f;
    const size_t span = (size_t)PL * cap + slack;
    RV_CUDA(ctx->dp_lins[0].ensure(span), "allocating");
    RV_CUDA(ctx->dp_ca[0].ensure(span), "allocating");
    RV_CUDA(ctx->dp_cb[0].ensure(span), "allocating");
    RV_CUDA(ctx->dp_cnt[0].ensure(PL), "allocating");
    RV_CUDA(ctx->dp_off[0].ensure(PL + 1), "allocating");
    for (int32_t p = 0; p <= PL; ++p) hbase[p] = (int64_t)p * cap;
    RV_CUDA(cudaMemcpyAsync(ctx->dp_off[0].p, hbase.data(), (PL + 1) * 8, cudaMemcpyHostToDevice, s),
            "H2D");
    rv::dp_launch_dive_children(ctx->dp_pick.p, ctx->l0idx.p, l == 1 ? ctx->grid_list.p : nullptr,
                                Bp, f, ctx->dp_lins[0].p, cap, ctx->dp_cnt[0].p, PL, s);
    const int32_t mode = l == L - 1 ? RV_MODE_FINAL : RV_MODE_BOUND;
    RV_CUDA(cudaMemsetAsync(ctx->dp_ca[0].p, 0, span * 4, s), "memset");
    if (mode == RV_MODE_FINAL) RV_CUDA(cudaMemsetAsync(ctx->dp_cb[0].p, 0, span * 4, s), "memset");
    ctx->launches += 1;
    if (int rc = keep_phase(ctx->dp_cnt[0].p)) return rc;
    const rv::DpList dl{ctx->dp_lins[0].p, 0, 0, ctx->dp_off[0].p, ctx->dp_cnt[0].p,
                        ctx->dp_ca[0].p, ctx->dp_cb[0].p};
    if (int rc = vote(mode, ch[l], dl, (int64_t)PL * cap)) return rc;
    phase_chunk.push_back(shard ? ((int64_t)cap + W - 1) / W : 0);
    if (mode == RV_MODE_BOUND)
      rv::dp_launch_dive_pick(ctx->dp_lins[0].p, ctx->dp_ca[0].p, ctx->dp_off[0].p,
                              ctx->dp_cnt[0].p, ch[l], eps, ctx->rows.p, ctx->dp_pick.p, PL, s);
    else
      rv::dp_launch_max_lo(ctx->dp_cb[0].p, ctx->dp_off[0].p, ctx->dp_cnt[0].p, ctx->dp_lb.p, PL, s);
    ctx->launches += 1;
    tr.mark("  dive level");
  }
  // ---- branch and bound from the level-0 survivors (UB >= lb*).  A list of problem p has
  // act[p+1] - act[p] entries stored from base[p]; its children get the capacity region
  // act[p] * f^3 .. act[p+1] * f^3 (parents x f^3).  Lists alternate between sets 0 and 1;
  // their offsets live in rings (act: 2, base: 3), so a level's parents' offsets survive the
  // scan of its children -- the re-dive (R18) needs them.
  //   parents' act of level l = dp_actr[l & 1]   (the scan writes the children's into the other)
  //   children's base of level l = dp_bring[l % 3], parents' = dp_bring[(l - 1) % 3]
  for (int r = 0; r < 2; ++r) RV_CUDA(ctx->dp_actr[r].ensure(PL + 1), "allocating");
  for (int r = 0; r < 3; ++r) RV_CUDA(ctx->dp_bring[r].ensure(PL + 1), "allocating");
  RV_CUDA(ctx->dp_tot.ensure(1), "allocating");
  RV_CUDA(ctx->down.ensure(256), "allocating staging");
  RV_CUDA(ctx->dp_rdone.ensure(PL), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->dp_rdone.p, 0, PL * 4, s), "memset");
  for (int32_t p = 0; p <= PL; ++p) hbase[p] = (int64_t)p * m0;  // level 0: act == base
  RV_CUDA(cudaMemcpyAsync(ctx->dp_actr[1].p, hbase.data(), (PL + 1) * 8, cudaMemcpyHostToDevice, s),
          "H2D");
  int64_t ptotal = (int64_t)PL * m0;
  const uint32_t* plins = ctx->grid_list.p;
  const uint32_t* pub = ctx->l0cnt.p;
  bool shared = true;
  int cur = -1;
  {
    // children base of BnB level 1: act * f^3
    const int32_t f = ch[1] / ch[0];
    const int64_t f3 = (int64_t)f * f * f;
    for (int32_t p = 0; p <= PL; ++p) hbase[p] = (int64_t)p * m0 * f3;
    RV_CUDA(cudaMemcpyAsync(ctx->dp_bring[1].p, hbase.data(), (PL + 1) * 8, cudaMemcpyHostToDevice,
                            s), "H2D");
  }
  for (int l = 1; l < L; ++l) {
    const int nb = cur == 1 ? 0 : 1;  // level 1 -> set 1 (set 0 still holds the dive lists)
    const int32_t Bp = ch[l - 1], f = ch[l] / ch[l - 1];
    const int64_t f3 = (int64_t)f * f * f;
    const int64_t cap_total = std::max<int64_t>(1, ptotal * f3) + slack;
    int64_t* pact = ctx->dp_actr[l & 1].p;          // parents' act
    int64_t* cact = ctx->dp_actr[(l + 1) & 1].p;    // children's act (written by the scan)
    int64_t* cbase = ctx->dp_bring[l % 3].p;        // children's base
    int64_t* pbase = shared ? pact : ctx->dp_bring[(l + 2) % 3].p;  // parents' base
    int64_t* nbase = ctx->dp_bring[(l + 1) % 3].p;  // grandchildren's base (scan output)
    RV_CUDA(ctx->dp_lins[nb].ensure(cap_total), "allocating");
    RV_CUDA(ctx->dp_ca[nb].ensure(cap_total), "allocating");
    RV_CUDA(ctx->dp_cb[nb].ensure(cap_total), "allocating");
    RV_CUDA(ctx->dp_cnt[nb].ensure(PL), "allocating");
    if (shard) {
      RV_CUDA(ctx->dp_pcnt.ensure(std::max<int64_t>(1, ptotal)), "allocating");
      RV_CUDA(ctx->dp_poff.ensure(ptotal + 1), "allocating");
    }
    auto expand = [&]() {
      RV_CUDA(cudaMemsetAsync(ctx->dp_cnt[nb].p, 0, PL * 4, s), "memset");
      if (shard) {  // identical list on every rank: children placed by a prefix over parents
        rv::dp_launch_expand_ordered(plins, shared, pact, pbase, pub, ctx->dp_lb.p, PL, ptotal, Bp,
                                     f, cbase, ctx->dp_lins[nb].p, ctx->dp_ca[nb].p,
                                     ctx->dp_cb[nb].p, ctx->dp_cnt[nb].p, ctx->dp_pcnt.p,
                                     ctx->dp_poff.p, s);
        ctx->launches += 3;
      } else {
        rv::dp_launch_bnb_expand(plins, shared, pact, pbase, pub, ctx->dp_lb.p, PL, ptotal, Bp, f,
                                 cbase, ctx->dp_lins[nb].p, ctx->dp_ca[nb].p, ctx->dp_cb[nb].p,
                                 ctx->dp_cnt[nb].p, ctx->dp_err.p, s);
        ctx->launches += 1;
      }
      return RV_OK;
    };
    int64_t nf3 = 1;
    if (l + 1 < L) {
      const int64_t nf = ch[l + 1] / ch[l];
      nf3 = nf * nf * nf;
    }
    // the children's act offsets and the grandchildren's base, and (level >= 2) the re-dive
    // trigger (R18, as rv_plan.cpp: a problem whose level keeps >= 16384 blocks and more than
    // half of all possible children dives again from its best-excess parent block, once per
    // problem); then the total and the trigger on the host
    RV_CUDA(ctx->dp_rflag.ensure(PL), "allocating");
    RV_CUDA(ctx->dp_rany.ensure(1), "allocating");
    auto scan_and_read = [&](int64_t* total, int32_t* any) -> int {
      rv::RediveCheck chk{cur >= 0 ? ctx->dp_cnt[cur].p : nullptr, f3, ctx->dp_rdone.p,
                          ctx->dp_rflag.p, ctx->dp_rany.p, 1};
      if (any) RV_CUDA(cudaMemsetAsync(ctx->dp_rany.p, 0, 4, s), "memset");
      rv::dp_launch_scan(ctx->dp_cnt[nb].p, PL, nf3, cact, nbase, ctx->dp_tot.p, s,
                         any ? &chk : nullptr);
      ctx->launches += 1;
      ctx->down.reset();
      int64_t* ht = ctx->down.take<int64_t>(1);
      int32_t* ha = ctx->down.take<int32_t>(1);
      RV_CUDA(cudaMemcpyAsync(ht, ctx->dp_tot.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
      if (any) RV_CUDA(cudaMemcpyAsync(ha, ctx->dp_rany.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
      RV_SYNC(cudaStreamSynchronize(s), "batched level");
      ctx->collect_vote_ms();
      *total = *ht;
      if (any) *any = *ha;
      return RV_OK;
    };
    if (int rc = expand()) return rc;
    int64_t ctotal = 0;
    int32_t any = 0;
    if (int rc = scan_and_read(&ctotal, l >= 2 ? &any : nullptr)) return rc;
    {
      if (any) {
        RV_CUDA(ctx->dp_lb2.ensure(PL), "allocating");
        rv::dp_launch_dive_pick(ctx->dp_lins[cur].p, ctx->dp_ca[cur].p, pbase, ctx->dp_cnt[cur].p,
                                ch[l - 1], eps, ctx->rows.p, ctx->dp_pick.p, PL, s);
        ctx->launches += 1;
        for (int lv = l; lv < L; ++lv) {
          const int32_t rf = ch[lv] / ch[lv - 1], rcap = 27 * rf * rf * rf;
          const size_t rspan = (size_t)PL * rcap + slack;
          RV_CUDA(ctx->dp_lins[2].ensure(rspan), "allocating");
          RV_CUDA(ctx->dp_ca[2].ensure(rspan), "allocating");
          RV_CUDA(ctx->dp_cb[2].ensure(rspan), "allocating");
          RV_CUDA(ctx->dp_cnt[2].ensure(PL), "allocating");
          RV_CUDA(ctx->dp_off[2].ensure(PL + 1), "allocating");
          for (int32_t p = 0; p <= PL; ++p) hbase[p] = (int64_t)p * rcap;
          RV_CUDA(cudaMemcpyAsync(ctx->dp_off[2].p, hbase.data(), (PL + 1) * 8,
                                  cudaMemcpyHostToDevice, s), "H2D");
          rv::dp_launch_dive_children(ctx->dp_pick.p, nullptr, nullptr, ch[lv - 1], rf,
                                      ctx->dp_lins[2].p, rcap, ctx->dp_cnt[2].p, PL, s,
                                      ctx->dp_rflag.p);
          const int32_t rmode = lv == L - 1 ? RV_MODE_FINAL : RV_MODE_BOUND;
          RV_CUDA(cudaMemsetAsync(ctx->dp_ca[2].p, 0, rspan * 4, s), "memset");
          if (rmode == RV_MODE_FINAL)
            RV_CUDA(cudaMemsetAsync(ctx->dp_cb[2].p, 0, rspan * 4, s), "memset");
          ctx->launches += 1;
          if (int rc = keep_phase(ctx->dp_cnt[2].p, true)) return rc;
          const rv::DpList rl{ctx->dp_lins[2].p, 0, 0, ctx->dp_off[2].p, ctx->dp_cnt[2].p,
                              ctx->dp_ca[2].p, ctx->dp_cb[2].p};
          if (int rc = vote(rmode, ch[lv], rl, (int64_t)PL * rcap)) return rc;
          phase_chunk.push_back(shard ? ((int64_t)rcap + W - 1) / W : 0);
          if (rmode == RV_MODE_BOUND) {
            rv::dp_launch_dive_pick(ctx->dp_lins[2].p, ctx->dp_ca[2].p, ctx->dp_off[2].p,
                                    ctx->dp_cnt[2].p, ch[lv], eps, ctx->rows.p, ctx->dp_pick.p,
                                    PL, s);
          } else {
            rv::dp_launch_max_lo(ctx->dp_cb[2].p, ctx->dp_off[2].p, ctx->dp_cnt[2].p,
                                 ctx->dp_lb2.p, PL, s);
            rv::dp_launch_lb_max(ctx->dp_lb.p, ctx->dp_lb2.p, PL, s);
            ctx->launches += 1;
          }
          ctx->launches += 1;
        }
        // level l again, with the raised lb* (the parents' offsets are intact in the rings)
        if (int rc = expand()) return rc;
        if (int rc = scan_and_read(&ctotal, nullptr)) return rc;
        tr.mark("  re-dive");
      }
    }
    if (int rc = keep_phase(ctx->dp_cnt[nb].p)) return rc;
    const int32_t mode = l == L - 1 ? RV_MODE_FINAL : RV_MODE_BOUND;
    const rv::DpList cl{ctx->dp_lins[nb].p, 0, 0, cbase, ctx->dp_cnt[nb].p, ctx->dp_ca[nb].p,
                        ctx->dp_cb[nb].p};
    if (int rc = vote(mode, ch[l], cl, ctotal)) return rc;
    phase_chunk.push_back(shard ? (ctotal + W - 1) / W : 0);
    ptotal = ctotal;
    plins = ctx->dp_lins[nb].p;
    pub = ctx->dp_ca[nb].p;
    shared = false;
    cur = nb;
    tr.mark("  bnb level");
  }
  // ---- finest level: max lo, exact-known blocks, recheck of hi >= max lo, hi != lo; winner
  // (the last scan, at level L-1, wrote the final list's act into dp_actr[L & 1]; its base is
  // the ring's dp_bring[(L - 1) % 3])
  const int64_t ftotal = ptotal;
  const uint32_t* flins = ctx->dp_lins[cur].p;
  const uint32_t* fhi = ctx->dp_ca[cur].p;
  const uint32_t* flo = ctx->dp_cb[cur].p;
  const int64_t* fcap = ctx->dp_bring[(L - 1) % 3].p;
  int64_t* fact = ctx->dp_actr[L & 1].p;
  RV_CUDA(ctx->dp_rcnt.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_lmax.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_best.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_ties.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_rlins.ensure(std::max<int64_t>(1, ftotal)), "allocating");
  RV_CUDA(ctx->dp_ex.ensure(std::max<int64_t>(1, ftotal)), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->dp_rcnt.p, 0, PL * 4, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->dp_lmax.p, 0, PL * 4, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->dp_best.p, 0, PL * 8, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->dp_ties.p, 0, PL * 4, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->dp_ex.p, 0, std::max<int64_t>(1, ftotal) * 4, s), "memset");
  rv::dp_launch_final_max(fact, fcap, flo, PL, ftotal, ctx->dp_lmax.p, s);
  rv::dp_launch_final_split(fact, fcap, flins, fhi, flo, ctx->dp_lmax.p, PL, ftotal,
                            ctx->dp_best.p, ctx->dp_rlins.p, ctx->dp_rcnt.p, s);
  ctx->launches += 2;
  if (int rc = keep_phase(ctx->dp_rcnt.p)) return rc;
  const rv::DpList rl{ctx->dp_rlins.p, 0, 0, fact, ctx->dp_rcnt.p, ctx->dp_ex.p,
                      ctx->dp_ex.p};
  if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_EXACT, ch[L - 1], rl, PL, ftotal,
                          nmax))
    return rc;
  rv::dp_launch_final_rechecked(fact, ctx->dp_rcnt.p, ctx->dp_rlins.p, ctx->dp_ex.p, PL,
                                ftotal, ctx->dp_best.p, s);
  rv::dp_launch_final_ties(fact, fcap, fhi, flo, ctx->dp_rcnt.p, ctx->dp_ex.p, PL, ftotal,
                           ctx->dp_best.p, ctx->dp_ties.p, s);
  ctx->launches += 2;
  RV_CUDA(cudaGetLastError(), "launching the level loop");
  // (its own staging: the refinement enqueued by before_sync stages through ctx->down)
  RV_CUDA(ctx->down2.ensure((size_t)PL * 24 + (size_t)nph * PL * 4 + 2048), "allocating staging");
  ctx->down2.reset();
  unsigned long long* hbest = ctx->down2.take<unsigned long long>(PL);
  int32_t* hties = ctx->down2.take<int32_t>(PL);
  int64_t* hlb = ctx->down2.take<int64_t>(PL);
  int32_t* hph = ctx->down2.take<int32_t>((size_t)nph * PL);
  int32_t* herr = ctx->down2.take<int32_t>(1);
  unsigned long long* hcp = ctx->down2.take<unsigned long long>(1);
  unsigned long long* hbad = ctx->down2.take<unsigned long long>(1);
  RV_CUDA(cudaMemcpyAsync(herr, ctx->dp_err.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hbad, ctx->bad.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (culled) RV_CUDA(cudaMemcpyAsync(hcp, ctx->c_pairs.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hbest, ctx->dp_best.p, 8 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hties, ctx->dp_ties.p, 4 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hlb, ctx->dp_lb.p, 8 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hph, ctx->dp_phase.p, 4 * (size_t)nph * PL, cudaMemcpyDeviceToHost, s),
          "D2H");
  if (before_sync)
    if (int rc = before_sync()) return rc;
  RV_SYNC(cudaStreamSynchronize(s), "batched finalize");
  ctx->collect_vote_ms();
  ctx->ev_collect();
  ctx->cev_collect();
  ctx->cull_ready = false;
  if (culled) ctx->cull_pairs += *hcp;
  if (*hbad != ~0ull)
    return ctx->fail(RV_EDATA, "correspondence row %llu has a zero-length or non-finite vector",
                     *hbad);
  if (*herr != 0)
    return ctx->fail(RV_ECUDA, "internal: device level-loop invariant violated (code %d)", *herr);
  tr.mark("  finalize");
  res.assign(PL, rv_plan_result{});
  uint64_t tc_pairs = 0;
  for (int32_t p = 0; p < PL; ++p) {
    rv_plan_result& r = res[p];
    const uint64_t n = (uint64_t)(rows[p + 1] - rows[p]);
    r.votes = (uint32_t)(hbest[p] >> 32);
    r.lin = hbest[p] ? 0xffffffffu - (uint32_t)(hbest[p] & 0xffffffffu) : 0u;
    r.B = ch[L - 1];
    r.n_tied = hties[p];
    r.lb_star = (uint32_t)hlb[p];
    const int32_t nre = hph[(size_t)(nph - 1) * PL + p];
    r.n_rechecked = nre;
    // phases: level 0, the dive, BnB, and the recheck when non-empty
    auto add = [&](int64_t c) {
      r.pair_votes += (uint64_t)c * n;
      r.cells_evaluated += (uint64_t)c;
      if (r.n_phases < 16) r.cells_per_phase[r.n_phases++] = c;
    };
    add(m0);
    for (int ph = 0; ph + 1 < nph; ++ph) {
      const int64_t c = hph[(size_t)ph * PL + p];
      if (ph_optional[ph] && c == 0) continue;  // this problem did not re-dive
      add(c);
    }
    if (nre > 0) add(nre);
    if (culled) {  // K3-TC voted level 0 only (this rank's slice); K3-C counts its own pairs
      if (shard && ctx->comm) {
        const int64_t c0 = (m0 + W - 1) / W;
        tc_pairs += (uint64_t)std::max<int64_t>(0, std::min<int64_t>(c0, m0 - (int64_t)ctx->cfg.rank * c0)) * n;
      } else {
        tc_pairs += (uint64_t)m0 * n;
      }
    } else if (cull) {  // level 0 unsharded, the finer levels on K3-TC (sharded if W > 1)
      tc_pairs += (uint64_t)m0 * n;
      for (int ph = 0; ph + 1 < nph; ++ph) {
        const int64_t c = hph[(size_t)ph * PL + p];
        const int64_t mine = !shard || !ctx->comm ? c
            : std::max<int64_t>(0, std::min<int64_t>(phase_chunk[ph], c - (int64_t)ctx->cfg.rank * phase_chunk[ph]));
        tc_pairs += (uint64_t)mine * n;
      }
    } else if (!shard || !ctx->comm) {
      tc_pairs += (r.pair_votes - (uint64_t)nre * n);
    } else {  // this rank's slices only: level 0, then the dive and BnB phases
      const int64_t c0 = (m0 + W - 1) / W;
      auto mine = [&](int64_t m, int64_t c) {
        return (uint64_t)std::max<int64_t>(0, std::min<int64_t>(c, m - (int64_t)ctx->cfg.rank * c));
      };
      tc_pairs += mine(m0, c0) * n;
      for (int ph = 0; ph + 1 < nph; ++ph)
        tc_pairs += mine(hph[(size_t)ph * PL + p], phase_chunk[ph]) * n;
    }
  }
  if (ctx->tc_on) ctx->vote_pairs += tc_pairs;
  return RV_OK;
}

// ---- the one-pass single solve ------------------------------------------------------------------
// One problem on one GPU: the whole certified search -- setup, level 0 with its culling lists,
// the dive, every branch-and-bound level, the finest level with its exact recheck, and the
// refinement -- is enqueued without a single host round trip; the host reads everything back
// once at the end.  What the per-level loop (solve_batched_dplan) learns from its round trips is
// replaced by data-independent capacities: the level lists hold up to ctx->op_cap blocks
// (min with the grid's candidate count), the culling lists up to a quarter of the level-0 pairs
// (the per-level loop's own culling limit), the exact recheck up to kOnePassRecheck blocks.  A
// device-side violation (a longer list, or the re-dive trigger R18, which this loop does not
// take) raises the solve's error word; the level scans then empty every later level, and the
// host redoes the solve with the per-level loop (rv_result.flags |= RV_RETRIED).  Every decision
// is the per-level loop's, so both give the same result.
// capacities start small (a first solve allocates little) and grow 8x (level lists, up to
// kOnePassCapMax blocks) or 2x (culling lists, up to a quarter of the level-0 pairs) after a
// solve that outgrew them; the grown sizes stay with the context
constexpr int64_t kOnePassCapMax = (int64_t)1 << 22;
constexpr int64_t kOnePassRecheck = 4096;

bool one_pass_applies(rv_ctx* ctx, int32_t P) {
  if (P != 1 || ctx->cfg.planner != 0 || !ctx->tc_on) return false;
  const bool sharded = ctx->effective_world() > 1 || ctx->comm != nullptr;
  // over ranks: the subtree ownership needs the grouped (K3-CT) culling
  return !sharded || (ctx->cull_on && ctx->cull_tc);
}

#ifndef RV_OP_CHECK
#define RV_OP_CHECK 0  // debug builds: wait and check after each phase of a one-pass solve
#endif
#if RV_OP_CHECK
#define OP_CHECK(what)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = ctx->capturing ? cudaSuccess : cudaStreamSynchronize(s);            \
    if (e_ != cudaSuccess) return ctx->fail(RV_ECUDA, "one-pass %s: %s", what, cudaGetErrorString(e_)); \
    int32_t w_ = 0;                                                                      \
    if (!ctx->capturing && ctx->dp_err.p) cudaMemcpy(&w_, ctx->dp_err.p, 4, cudaMemcpyDeviceToHost); \
    if (w_) fprintf(stderr, "[rv] one-pass %s: error word %d\n", what, w_);             \
  } while (0)
#else
#define OP_CHECK(what) do { } while (0)
#endif

// The read-back slots of a one-pass solve in ctx->grb (pinned)
struct OnePassRB {
  unsigned long long *best, *cp, *bad;
  int32_t *ties, *err, *fl, *ph;
  int64_t* lb;
  double* q;
  uint32_t* ni;
  explicit OnePassRB(char* g) {
    best = reinterpret_cast<unsigned long long*>(g);
    cp = best + 1;
    bad = best + 2;
    lb = reinterpret_cast<int64_t*>(g + 24);
    q = reinterpret_cast<double*>(g + 32);
    ties = reinterpret_cast<int32_t*>(g + 64);
    err = ties + 1;
    fl = ties + 2;
    ni = reinterpret_cast<uint32_t*>(ties + 3);
    ph = ties + 4;  // up to 3 L + 1 phase counts
  }
};

// Enqueue the whole solve on ctx->stream (no host wait), read-backs into ctx->grb; fills the
// host values the result needs (hv).  Every size and launch shape is a function of (n, eps, ch)
// and the context only, which is what makes the sequence graph-capturable.
int enqueue_one_pass(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                     const std::vector<int32_t>& ch, uint32_t* mask, rv_ctx::OnePassHost& hv,
                     const rv::Excl& ex) {
  const int L = (int)ch.size();
  // one problem over W ranks (one_pass_applies: grouped culling): level 0 in slabs and the dive's
  // blocks by owner, each with one all-reduce of fixed size; the branch and bound split into the
  // subtrees of the owned level-0 groups, searched by each rank on its own (no collective); the
  // ranks' winners merged at the end.  Loopback (emulate_world): every rank in turn.
  const int W = ctx->effective_world();
  const bool sharded = W > 1;
  const bool nccl_path = ctx->comm != nullptr;
  const int r_lo = nccl_path ? ctx->cfg.rank : 0, r_hi = nccl_path ? r_lo + 1 : W;
  // the flat kernels loop over the device's own totals; their grids only need to fill the GPU
  auto flat_hint = [&](int64_t m) { return std::min<int64_t>(m, (int64_t)ctx->num_sms * 2 * 256); };
  cudaStream_t s = ctx->stream;
  const int32_t PL = 1;
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> rows(offs, offs + 2), koff;
  cudaEvent_t* ph = ctx->ph;
  const int32_t B0 = ch[0];
  const int64_t m0 = rv_grid_candidates(B0, nullptr, 0);
  // pinned staging for every host-built upload of the solve (it is not reused before the final
  // sync): run_setup's offsets, the level-0 background, the dive / BnB offsets
  RV_CUDA(ctx->up.ensure((size_t)m0 * 8 + 65536), "allocating staging");
  RV_CUDA(ctx->record(ph[0], s), "event");
  nvtxRangePushA("rv.setup");
  // every offset pair of the solve in one launch: rows, K / TC table offsets, the dive levels'
  // list offsets (one pair per level), the branch and bound's first act / base
  {
    RV_CUDA(ctx->rows.ensure(2), "allocating offsets");
    RV_CUDA(ctx->koffs.ensure(2), "allocating offsets");
    RV_CUDA(ctx->toffs.ensure(2), "allocating offsets");
    RV_CUDA(ctx->dp_off[0].ensure(2 * (size_t)L), "allocating");
    for (int r = 0; r < 2; ++r) RV_CUDA(ctx->dp_actr[r].ensure(2), "allocating");
    for (int r = 0; r < 3; ++r) RV_CUDA(ctx->dp_bring[r].ensure(2), "allocating");
    rv::SetList sl;
    sl.add(ctx->rows.p, 0, n);
    sl.add(ctx->koffs.p, 0, pad4(n));
    sl.add(ctx->toffs.p, 0, (n + rv::kTcN - 1) / rv::kTcN * rv::kTcN);
    for (int l = 1; l < L; ++l) {
      const int64_t f = ch[l] / ch[l - 1];
      sl.add(ctx->dp_off[0].p + 2 * l, 0, 27 * f * f * f);
    }
    if (!sharded) {  // (the branch and bound's rings start here; per rank when sharded)
      const int64_t f = ch[1] / ch[0];
      sl.add(ctx->dp_actr[1].p, 0, m0);
      sl.add(ctx->dp_bring[1].p, 0,
             std::min<int64_t>(m0 * f * f * f,
                               std::min<int64_t>(ctx->op_cap, (int64_t)ch[1] * ch[1] * ch[1])));
    }
    OP_CHECK("before the offsets");
    rv::launch_set_consts(sl, s);
    ctx->launches += 1;
    OP_CHECK("offsets");
  }
  // (ctx->reuse_l0: the previous solve of this call had the same input -- NEXT-2's next peak --
  // so the K tables, level 0's counts and the culling lists are still valid)
  const bool reuse_l0 = ctx->reuse_l0;
  if (reuse_l0) koff.assign({0, pad4(n)});
  else if (int rc = run_setup(ctx, x, y, offs, 1, koff, true)) return rc;
  nvtxRangePop();
  RV_CUDA(ctx->record(ph[1], s), "event");
  OP_CHECK("setup");
  auto upload_i64 = [&](int64_t* dst, std::initializer_list<int64_t> v) -> int {
    rv::launch_set_i64x2(dst, *v.begin(), *(v.begin() + 1), s);  // kernel arguments, see run_setup
    ctx->launches += 1;
    return RV_OK;
  };
  int64_t nmax = n;
  RV_CUDA(ctx->dp_phase.ensure((size_t)(3 * L + 1)), "allocating");
  int nph = 0;
  auto keep_phase = [&](const int32_t* dcnt) -> int {
    RV_CUDA(cudaMemcpyAsync(ctx->dp_phase.p + nph, dcnt, 4, cudaMemcpyDeviceToDevice, s), "D2D");
    ++nph;
    return RV_OK;
  };
  ctx->ev_reset();
  RV_CUDA(ctx->dp_err.ensure(1), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->dp_err.p, 0, 4, s), "memset");
  // ---- level 0 (every block of the grid), with the culling lists
  nvtxRangePushA("rv.level0");
  if (ctx->grid_host_B != B0) {
    ctx->grid_host.resize(m0);
    rv_grid_candidates(B0, ctx->grid_host.data(), m0);
    ctx->grid_host_B = B0;
  }
  int64_t mbg = 0;
  const double* bgh = rv_plan_l0_background(B0, eps, &mbg);
  if (!bgh || mbg != m0) return ctx->fail(RV_ECUDA, "internal: level-0 background unavailable");
  RV_CUDA(ctx->l0cnt.ensure((size_t)m0), "allocating level-0 counts");
  if (ctx->l0bg_B != B0 || ctx->l0bg_eps != eps || ctx->l0bg.cap < (size_t)m0) {
    RV_CUDA(ctx->l0bg.ensure(m0), "allocating");
    double* h = ctx->up.take<double>(m0);
    std::memcpy(h, bgh, m0 * sizeof(double));
    RV_CUDA(cudaMemcpyAsync(ctx->l0bg.p, h, m0 * sizeof(double), cudaMemcpyHostToDevice, s),
            "H2D background");
    ctx->l0bg_B = B0;
    ctx->l0bg_eps = eps;
  }
  if (ctx->grid_list_B != B0 || ctx->grid_list_m != m0) {
    RV_CUDA(ctx->grid_list.ensure(m0), "allocating grid list");
    RV_CUDA(cudaMemcpy(ctx->grid_list.p, ctx->grid_host.data(), m0 * 4, cudaMemcpyHostToDevice),
            "H2D grid");
    ctx->grid_list_B = B0;
    ctx->grid_list_m = m0;
  }
  ctx->cull_ready = false;
  const int64_t tpad = ctx->tc_toff.back();
  const bool cull = ctx->cull_on && (double)m0 * (double)(tpad / 32) * 4.0 <= 4294967296.0;
  const rv::DpList l0{ctx->grid_list.p, 1, m0, nullptr, nullptr, ctx->l0cnt.p, ctx->l0cnt.p};
  if (reuse_l0) {
    if (cull) {
      ctx->cull_l0cnt = reinterpret_cast<const uint32_t*>(ctx->c_fill.p);
      ctx->cull_ready = true;
    }
  } else if (cull) {
    RV_CUDA(cudaMemsetAsync(ctx->l0cnt.p, 0, (size_t)m0 * 4, s), "memset");
    RV_CUDA(ctx->cbits.ensure((size_t)m0 * (size_t)(tpad / 32)), "allocating level-0 bitmasks");
    if (int rc = cull_prepare(ctx, B0, m0, PL)) return rc;
    if (sharded) {  // this rank's slab (i-slab aligned: whole groups), counts all-reduced
      if (int rc = vote_level0_slabs(ctx, x, y, rows, koff, eps, B0, l0, m0, nmax)) return rc;
    } else if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, l0, PL, m0, nmax,
                                   true)) {
      return rc;
    }
    // the lists: row offsets, then the compaction into a fixed capacity (an eighth of the
    // level-0 pairs; cfg4's lists fill 3%: longer lists raise the error word and the per-level
    // loop, which reads their length back, redoes the solve)
    rv::CullGroups gr;
    if (ctx->cull_grouped) gr = rv::CullGroups{ctx->goff.p, ctx->gmem.p, ctx->cull_G};
    const int64_t NB = ctx->cull_G;
    const int64_t lcap = std::min<int64_t>((int64_t)1 << 29, (m0 * tpad) >> ctx->op_lshift) + 4 * NB;
    RV_CUDA(ctx->c_lofs.ensure(NB + 1), "allocating");
    RV_CUDA(ctx->c_lidx.ensure(lcap + 4), "allocating level-0 lists");
    RV_CUDA(ctx->c_fill.ensure(NB), "allocating");
    rv::launch_cull_rows(ctx->l0cnt.p, PL, m0, ctx->c_lofs.p, s, gr);
    // (a rank compacts the lists of its own groups; loopback: all)
    const int64_t row_lo = nccl_path && sharded ? ctx->cull_g[ctx->cfg.rank] : 0;
    const int64_t row_hi = nccl_path && sharded ? ctx->cull_g[ctx->cfg.rank + 1] : NB;
    rv::launch_cull_compact(ctx->cbits.p, ctx->toffs.p, PL, m0, ctx->cull_wpc_max, ctx->c_lofs.p,
                            ctx->c_fill.p, ctx->c_lidx.p, s, row_lo, row_hi, gr, lcap,
                            ctx->dp_err.p);
    ctx->launches += 2;
    // list lengths = the compaction's fill counters (also per ancestor, where they equal the
    // level-0 counts): a compaction that overflowed wrote nothing and leaves them 0, so no
    // later vote reads an unwritten list before the error word ends the solve
    ctx->cull_l0cnt = reinterpret_cast<const uint32_t*>(ctx->c_fill.p);
    ctx->cull_ready = true;
  } else {
    RV_CUDA(cudaMemsetAsync(ctx->l0cnt.p, 0, (size_t)m0 * 4, s), "memset");
    if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, l0, PL, m0, nmax))
      return rc;
  }
  RV_CUDA(ctx->l0idx.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_pick.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_lb.ensure(PL), "allocating");
  rv::launch_l0_argmax(ctx->l0cnt.p, m0, ctx->grid_list.p, B0, ctx->l0bg.p, ctx->rows.p, PL,
                       ctx->l0idx.p, s, ex);
  ctx->launches += 1;
  nvtxRangePop();
  RV_CUDA(ctx->record(ph[2], s), "event");
  OP_CHECK("level0");
  // ---- dive (fixed sizes: the 27-neighbourhood's children)
  // the dive's list buffers at the largest level's size up front: a folded level picks from the
  // previous level's list in place, so nothing may reallocate them between two dive levels
  {
    int64_t capmax = 1;
    for (int l = 1; l < L; ++l) {
      const int64_t f = ch[l] / ch[l - 1];
      capmax = std::max<int64_t>(capmax, 27 * f * f * f);
    }
    RV_CUDA(ctx->dp_lins[0].ensure(capmax), "allocating");
    RV_CUDA(ctx->dp_ca[0].ensure(capmax), "allocating");
    RV_CUDA(ctx->dp_cb[0].ensure(capmax), "allocating");
  }
  nvtxRangePushA("rv.dive");
  for (int l = 1; l < L; ++l) {
    const int32_t Bp = ch[l - 1], f = ch[l] / ch[l - 1], cap = 27 * f * f * f;
    RV_CUDA(ctx->dp_lins[0].ensure(cap), "allocating");
    RV_CUDA(ctx->dp_ca[0].ensure(cap), "allocating");
    RV_CUDA(ctx->dp_cb[0].ensure(cap), "allocating");
    RV_CUDA(ctx->dp_cnt[0].ensure(PL), "allocating");
    int64_t* doff = ctx->dp_off[0].p + 2 * l;  // {0, cap}, written at the start
    const int32_t mode = l == L - 1 ? RV_MODE_FINAL : RV_MODE_BOUND;
    const rv::DpList dl{ctx->dp_lins[0].p, 0, 0, doff, ctx->dp_cnt[0].p,
                        ctx->dp_ca[0].p, ctx->dp_cb[0].p};
    // one rank, culled, a small level: the pick (over the previous dive level), the children,
    // their zeroed counts and the phase count run inside the one-CTA planner (rv_dplan.h
    // DiveStep) -- one launch instead of five
    const bool fold = !sharded && ctx->cull_ready && cap <= 8192 && ctx->cull_G <= (1 << 14);
    if (fold) {
      rv::DiveStep d;
      d.on = 1;
      if (l > 1) {
        d.prev_lins = ctx->dp_lins[0].p;
        d.prev_a = ctx->dp_ca[0].p;
        d.prev_off = ctx->dp_off[0].p + 2 * (l - 1);
        d.prev_cnt = ctx->dp_cnt[0].p;
        d.pickB = ch[l - 1];
      }
      d.l0idx = ctx->l0idx.p;
      d.grid_list = ctx->grid_list.p;
      d.pick_out = ctx->dp_pick.p;
      d.ex = ex;
      d.finest = l == L - 1;
      d.Bp = Bp;
      d.f = f;
      d.cap = cap;
      d.out = ctx->dp_lins[0].p;
      d.out_cnt = ctx->dp_cnt[0].p;
      d.ca = ctx->dp_ca[0].p;
      d.cb = mode == RV_MODE_FINAL ? ctx->dp_cb[0].p : nullptr;
      d.phase = ctx->dp_phase.p + nph;
      ++nph;
      if (int rc = vote_level(ctx, x, y, rows, koff, eps, mode, ch[l], dl, PL, cap, nmax, false, &d))
        return rc;
      if (mode == RV_MODE_FINAL) {
        rv::dp_launch_max_lo(ctx->dp_cb[0].p, doff, ctx->dp_cnt[0].p, ctx->dp_lb.p, PL, s);
        ctx->launches += 1;
      }
      OP_CHECK("dive level (folded)");
#if RV_OP_CHECK
      if (!ctx->capturing) {
        int32_t c_ = 0;
        int64_t lb_ = 0;
        uint32_t pk_ = 0, a_[4] = {0, 0, 0, 0};
        cudaMemcpy(&c_, ctx->dp_cnt[0].p, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&pk_, ctx->dp_pick.p, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(a_, ctx->dp_ca[0].p, 16, cudaMemcpyDeviceToHost);
        if (mode == RV_MODE_FINAL) cudaMemcpy(&lb_, ctx->dp_lb.p, 8, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[rv] dive level %d: pick %u, %d blocks, counts %u %u %u %u, lb %lld\n", l,
                pk_, c_, a_[0], a_[1], a_[2], a_[3], (long long)lb_);
      }
#endif
      continue;
    }
    if (l > 1)  // the previous level's pick (a folded level picks by itself)
      rv::dp_launch_dive_pick(ctx->dp_lins[0].p, ctx->dp_ca[0].p, ctx->dp_off[0].p + 2 * (l - 1),
                              ctx->dp_cnt[0].p, ch[l - 1], eps, ctx->rows.p, ctx->dp_pick.p, PL, s,
                              ex);
    rv::dp_launch_dive_children(ctx->dp_pick.p, ctx->l0idx.p, l == 1 ? ctx->grid_list.p : nullptr,
                                Bp, f, ctx->dp_lins[0].p, cap, ctx->dp_cnt[0].p, PL, s, nullptr,
                                ex, l == L - 1);
    RV_CUDA(cudaMemsetAsync(ctx->dp_ca[0].p, 0, (size_t)cap * 4, s), "memset");
    if (mode == RV_MODE_FINAL) RV_CUDA(cudaMemsetAsync(ctx->dp_cb[0].p, 0, (size_t)cap * 4, s), "memset");
    ctx->launches += l > 1 ? 2 : 1;
    if (int rc = keep_phase(ctx->dp_cnt[0].p)) return rc;
    if (sharded) {  // each block voted by its owner, counts all-reduced (fixed size cap)
      if (int rc = vote_level_owned(ctx, x, y, rows, koff, eps, mode, ch[l], dl, cap, nmax))
        return rc;
    } else if (int rc = vote_level(ctx, x, y, rows, koff, eps, mode, ch[l], dl, PL, cap, nmax)) {
      return rc;
    }
    if (mode == RV_MODE_FINAL) {
      rv::dp_launch_max_lo(ctx->dp_cb[0].p, doff, ctx->dp_cnt[0].p, ctx->dp_lb.p, PL, s);
      ctx->launches += 1;
    }
  }
  nvtxRangePop();
  RV_CUDA(ctx->record(ph[3], s), "event");
  OP_CHECK("dive");
  // ---- branch and bound from the level-0 survivors: lists alternate between sets 0 and 1 at
  // fixed capacities; offsets in the rings as in the per-level loop
  nvtxRangePushA("rv.bnb");
  std::vector<int64_t> capl(L, 0);
  for (int l = 1; l < L; ++l)
    capl[l] = std::min<int64_t>(ctx->op_cap, (int64_t)ch[l] * ch[l] * ch[l]);  // (B^3 >= candidates;
                                                                              // counting them costs ms)
  for (int r = 0; r < 2; ++r) RV_CUDA(ctx->dp_actr[r].ensure(PL + 1), "allocating");
  for (int r = 0; r < 3; ++r) RV_CUDA(ctx->dp_bring[r].ensure(PL + 1), "allocating");
  RV_CUDA(ctx->dp_tot.ensure(1), "allocating");
  RV_CUDA(ctx->dp_rdone.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_rflag.ensure(PL), "allocating");
  const int64_t fcapn = capl[L - 1];
  RV_CUDA(ctx->dp_rcnt.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_lmax.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_best.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_ties.ensure(PL), "allocating");
  RV_CUDA(ctx->dp_rlins.ensure(fcapn), "allocating");
  RV_CUDA(ctx->dp_ex.ensure(fcapn), "allocating");
  // per-rank winners (sharded): slots r of best_r / ties_r
  RV_CUDA(ctx->dp_best_r.ensure((size_t)W), "allocating");
  RV_CUDA(ctx->dp_ties_r.ensure((size_t)W), "allocating");
  const int ph_bnb = nph;  // the branch-and-bound phases (and the recheck) are summed over ranks
  if (sharded)
    RV_CUDA(cudaMemsetAsync(ctx->dp_phase.p + ph_bnb, 0, (size_t)L * 4, s), "memset");
  for (int rk = r_lo; rk < r_hi; ++rk) {
    rv::Own own;
    if (sharded) {
      own = rv::Own{ctx->lutg.p, B0, ctx->cull_g[rk], ctx->cull_g[rk + 1]};
      ctx->cull_own_lo = own.lo;
      ctx->cull_own_hi = own.hi;
    }
    int nphr = ph_bnb;
    auto keep_phase_r = [&](const int32_t* dcnt) -> int {
      if (!sharded) {
        ++nphr;
        return keep_phase(dcnt);
      }
      rv::dp_launch_add_i32(ctx->dp_phase.p + nphr, dcnt, s);
      ctx->launches += 1;
      ++nphr;
      return RV_OK;
    };
    RV_CUDA(cudaMemsetAsync(ctx->dp_rdone.p, 0, PL * 4, s), "memset");
    if (sharded) {  // (one rank: written with the solve's other offsets at the start)
      if (int rc = upload_i64(ctx->dp_actr[1].p, {0, m0})) return rc;
      const int64_t f = ch[1] / ch[0];
      if (int rc = upload_i64(ctx->dp_bring[1].p, {0, std::min<int64_t>(m0 * f * f * f, capl[1])}))
        return rc;
    }
    const uint32_t* plins = ctx->grid_list.p;
    const uint32_t* pub = ctx->l0cnt.p;
    bool shared = true;
    int cur = -1;
    for (int l = 1; l < L; ++l) {
      const int nb = cur == 1 ? 0 : 1;
      const int32_t Bp = ch[l - 1], f = ch[l] / ch[l - 1];
      const int64_t f3 = (int64_t)f * f * f;
      int64_t* pact = ctx->dp_actr[l & 1].p;
      int64_t* cact = ctx->dp_actr[(l + 1) & 1].p;
      int64_t* cbase = ctx->dp_bring[l % 3].p;
      int64_t* pbase = shared ? pact : ctx->dp_bring[(l + 2) % 3].p;
      int64_t* nbase = ctx->dp_bring[(l + 1) % 3].p;
      RV_CUDA(ctx->dp_lins[nb].ensure(capl[l]), "allocating");
      RV_CUDA(ctx->dp_ca[nb].ensure(capl[l]), "allocating");
      RV_CUDA(ctx->dp_cb[nb].ensure(capl[l]), "allocating");
      RV_CUDA(ctx->dp_cnt[nb].ensure(PL), "allocating");
      // (level 1: zeroed here; a deeper level's count by the previous level's tail scan)
      if (l == 1) RV_CUDA(cudaMemsetAsync(ctx->dp_cnt[nb].p, 0, PL * 4, s), "memset");
      int64_t nf3 = 1;
      if (l + 1 < L) {
        const int64_t nf = ch[l + 1] / ch[l];
        nf3 = nf * nf * nf;
      }
      // The level's scan runs in the expansion's last CTA (one problem: rv_dplan.h TailScan).
      // Re-dive trigger (R18): not taken here -- it raises the error word (bit 8) and the solve
      // is redone by the per-level loop, which takes it (sharded: on the rank's own subtrees)
      rv::TailScan ts;
      ts.done = reinterpret_cast<uint32_t*>(ctx->dp_tdone.p);
      ts.f3 = nf3;
      ts.act = cact;
      ts.next_base = nbase;
      ts.total = ctx->dp_tot.p;
      ts.phase = ctx->dp_phase.p + nphr;
      ts.phase_add = sharded ? 1 : 0;
      ts.zero_next = l + 1 < L ? ctx->dp_cnt[nb ^ 1].p : nullptr;
      if (l >= 2)
        ts.rc = rv::RediveCheck{ctx->dp_cnt[cur].p, f3, ctx->dp_rdone.p, ctx->dp_rflag.p,
                                ctx->dp_err.p, 8};
      ts.op = rv::OnePass{ctx->dp_err.p, l + 1 < L ? capl[l + 1] : 0};
      if (ctx->cull_ready) {  // the level's cull bucket counters and list prefix (= cact)
        RV_CUDA(ctx->c_acnt.ensure((size_t)PL * ctx->cull_G), "allocating");
        ts.zero_buf = ctx->c_acnt.p;
        ts.zero_n = (int64_t)PL * ctx->cull_G;
      }
      // (only level 1's parents -- the shared level-0 grid -- span other ranks' groups)
      rv::dp_launch_bnb_expand(plins, shared, pact, pbase, pub, ctx->dp_lb.p, PL,
                               flat_hint(shared ? m0 : capl[l - 1]), Bp, f, cbase,
                               ctx->dp_lins[nb].p, ctx->dp_ca[nb].p, ctx->dp_cb[nb].p,
                               ctx->dp_cnt[nb].p, ctx->dp_err.p, s,
                               shared ? own : rv::Own(), ex, l == L - 1, ts);
      ctx->launches += 1;
      ++nphr;
      if (!sharded) ++nph;  // (keep_phase's slot; one rank: nph == nphr)
      const int32_t mode = l == L - 1 ? RV_MODE_FINAL : RV_MODE_BOUND;
      const rv::DpList cl{ctx->dp_lins[nb].p, 0, 0, cbase, ctx->dp_cnt[nb].p, ctx->dp_ca[nb].p,
                          ctx->dp_cb[nb].p};
      ctx->cull_pre_act = ctx->cull_ready ? cact : nullptr;
      const int vrc = vote_level(ctx, x, y, rows, koff, eps, mode, ch[l], cl, PL, capl[l], nmax);
      ctx->cull_pre_act = nullptr;
      if (vrc) return vrc;
      plins = ctx->dp_lins[nb].p;
      pub = ctx->dp_ca[nb].p;
      shared = false;
      cur = nb;
    }
    if (rk == r_lo) RV_CUDA(ctx->record(ph[4], s), "event");
    // ---- finest level: max lo, exact-known blocks, the fp64 recheck, winner, ties (sharded:
    // over the rank's subtrees; its max lo <= the global one, so it rechecks a superset)
    const uint32_t* flins = ctx->dp_lins[cur].p;
    const uint32_t* fhi = ctx->dp_ca[cur].p;
    const uint32_t* flo = ctx->dp_cb[cur].p;
    const int64_t* fcap = ctx->dp_bring[(L - 1) % 3].p;
    int64_t* fact = ctx->dp_actr[L & 1].p;
    RV_CUDA(cudaMemsetAsync(ctx->dp_rcnt.p, 0, PL * 4, s), "memset");
    RV_CUDA(cudaMemsetAsync(ctx->dp_lmax.p, 0, PL * 4, s), "memset");
    RV_CUDA(cudaMemsetAsync(ctx->dp_best.p, 0, PL * 8, s), "memset");
    RV_CUDA(cudaMemsetAsync(ctx->dp_ties.p, 0, PL * 4, s), "memset");
    RV_CUDA(cudaMemsetAsync(ctx->dp_ex.p, 0, (size_t)kOnePassRecheck * 4, s), "memset");
    rv::dp_launch_final_max(fact, fcap, flo, PL, flat_hint(fcapn), ctx->dp_lmax.p, s);
    rv::dp_launch_final_split(fact, fcap, flins, fhi, flo, ctx->dp_lmax.p, PL, flat_hint(fcapn),
                              ctx->dp_best.p, ctx->dp_rlins.p, ctx->dp_rcnt.p, s);
    ctx->launches += 2;
    if (int rc = keep_phase_r(ctx->dp_rcnt.p)) return rc;
    // (a recheck list longer than kOnePassRecheck blocks exceeds the items' bound: error word)
    const rv::DpList rl{ctx->dp_rlins.p, 0, 0, fact, ctx->dp_rcnt.p, ctx->dp_ex.p, ctx->dp_ex.p};
    if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_EXACT, ch[L - 1], rl, PL,
                            kOnePassRecheck, nmax))
      return rc;
    rv::dp_launch_final_rechecked(fact, ctx->dp_rcnt.p, ctx->dp_rlins.p, ctx->dp_ex.p, PL,
                                  kOnePassRecheck, ctx->dp_best.p, s);
    rv::dp_launch_final_ties(fact, fcap, fhi, flo, ctx->dp_rcnt.p, ctx->dp_ex.p, PL,
                             flat_hint(fcapn), ctx->dp_best.p, ctx->dp_ties.p, s);
    ctx->launches += 2;
    if (sharded) {
      RV_CUDA(cudaMemcpyAsync(ctx->dp_best_r.p + rk, ctx->dp_best.p, 8, cudaMemcpyDeviceToDevice, s),
              "D2D");
      RV_CUDA(cudaMemcpyAsync(ctx->dp_ties_r.p + rk, ctx->dp_ties.p, 4, cudaMemcpyDeviceToDevice, s),
              "D2D");
    }
    if (rk + 1 == r_hi) nph = nphr;
  }
  ctx->cull_own_lo = 0;
  ctx->cull_own_hi = INT64_MAX;
  if (sharded) {
    if (nccl_path) {  // the ranks' winners, summed phases, and the error word on every rank
      const int rk = ctx->cfg.rank;
      ncclResult_t nr = nccl().AllGather(ctx->dp_best_r.p + rk, ctx->dp_best_r.p, 1, ncclUint64,
                                         ctx->comm, s);
      if (nr == ncclSuccess)
        nr = nccl().AllGather(ctx->dp_ties_r.p + rk, ctx->dp_ties_r.p, 1, ncclInt32, ctx->comm, s);
      if (nr == ncclSuccess)
        nr = nccl().AllReduce(ctx->dp_phase.p + ph_bnb, ctx->dp_phase.p + ph_bnb, (size_t)L,
                              ncclInt32, ncclSum, ctx->comm, s);
      if (nr == ncclSuccess)
        nr = nccl().AllReduce(ctx->dp_err.p, ctx->dp_err.p, 1, ncclInt32, ncclMax, ctx->comm, s);
      if (nr != ncclSuccess)
        return ctx->fail(RV_ENCCL, "one-pass collectives: %s", nccl().GetErrorString(nr));
    }
    rv::dp_launch_merge_rank_winners(ctx->dp_best_r.p, ctx->dp_ties_r.p, W, ctx->dp_best.p,
                                     ctx->dp_ties.p, s);
    ctx->launches += 1;
  }
  nvtxRangePop();
  RV_CUDA(ctx->record(ph[5], s), "event");
  OP_CHECK("bnb+final");
  // ---- refinement from the winner (decoded on the device), K6 + K7 in one cooperative launch
  nvtxRangePushA("rv.refine");
  RV_CUDA(ctx->partials.ensure((size_t)((n + rv::kRefRowsPerItem - 1) / rv::kRefRowsPerItem) * 10),
          "allocating");
  RV_CUDA(ctx->qs.ensure(4), "allocating");
  RV_CUDA(ctx->flags.ensure(1), "allocating");
  RV_CUDA(ctx->ninl.ensure(2), "allocating");  // [1]: the refinement's grid-barrier counter
  rv::Refine1Args ra{x, y, n, ctx->k9.p, ctx->stride, std::cos(eps), ctx->cfg.guard,
                     ctx->cfg.refine_rounds, ctx->dp_best.p, ch[L - 1], nullptr,
                     ctx->partials.p, ctx->qs.p, ctx->flags.p, ctx->ninl.p, mask,
                     reinterpret_cast<uint32_t*>(ctx->ninl.p + 1)};
  RV_CUDA(rv::launch_refine1(ra, ctx->num_sms, s), "launching the refinement");
  ctx->launches += 1;
  nvtxRangePop();
  RV_CUDA(ctx->record(ph[6], s), "event");
  OP_CHECK("refine");
  // ---- the one read-back (into the pinned block; the host reads it after one wait)
  OnePassRB rb(ctx->grb);
  if (nph > 3 * L + 1) return ctx->fail(RV_ECUDA, "internal: phase slots");
  RV_CUDA(cudaMemcpyAsync(rb.err, ctx->dp_err.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.bad, ctx->bad.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (cull) RV_CUDA(cudaMemcpyAsync(rb.cp, ctx->c_pairs.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.best, ctx->dp_best.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.ties, ctx->dp_ties.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.lb, ctx->dp_lb.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.ph, ctx->dp_phase.p, 4 * (size_t)nph, cudaMemcpyDeviceToHost, s),
          "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.q, ctx->qs.p, 32, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.fl, ctx->flags.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(rb.ni, ctx->ninl.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  hv.m0 = m0;
  hv.nph = nph;
  hv.cull = cull;
  return RV_OK;
}

// Key of a one-pass enqueue: everything its launch sequence depends on
static void one_pass_key(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                         const std::vector<int32_t>& ch, const uint32_t* mask, uint64_t k[8]) {
  uint64_t e;
  std::memcpy(&e, &eps, 8);
  k[0] = (uint64_t)(uintptr_t)x;
  k[1] = (uint64_t)(uintptr_t)y;
  k[2] = (uint64_t)n;
  k[3] = e;
  k[4] = (uint64_t)(uintptr_t)mask;
  k[5] = ((uint64_t)ch.size() << 32) | (uint64_t)(uint32_t)ch[0];
  k[6] = (uint64_t)(uintptr_t)ctx->stream;
  k[7] = 0;
  for (int32_t b : ch) k[7] = k[7] * 1009u + (uint64_t)b;
}

int solve_one_pass(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                   const std::vector<int32_t>& ch, rv_result* out, uint32_t* mask, bool* redo,
                   const rv::Excl* excl) {
  *redo = false;
  const rv::Excl ex = excl ? *excl : rv::Excl();
  const bool graphs = ctx->graphs_on && ex.n == 0;  // (the exclusions are not in the key)
  cudaStream_t s = ctx->stream;
  uint64_t key[8];
  one_pass_key(ctx, x, y, n, eps, ch, mask, key);
  const bool same_as_last = ctx->lastkey_ok && std::memcmp(key, ctx->lastkey, sizeof(key)) == 0;
  const bool replay = graphs && ctx->gexec && ctx->gkey_ok &&
                      std::memcmp(key, ctx->gkey, sizeof(key)) == 0 &&
                      ctx->gepoch == g_realloc_epoch.load();
  rv_ctx::OnePassHost hv;
  ctx->ev_reset();
  ctx->cevn = 0;
  if (replay) {
    RV_CUDA(cudaEventRecord(ctx->gfork, s), "event");
    RV_CUDA(cudaStreamWaitEvent(ctx->gstream, ctx->gfork, 0), "fork");
    RV_CUDA(cudaGraphLaunch(ctx->gexec, ctx->gstream), "launching the solve graph");
    RV_CUDA(cudaEventRecord(ctx->ev1, ctx->gstream), "event");
    RV_CUDA(cudaEventRecord(ctx->gjoin, ctx->gstream), "event");
    RV_CUDA(cudaStreamWaitEvent(s, ctx->gjoin, 0), "join");
    hv = ctx->ghost;
    ctx->launches = hv.launches;
    ctx->vote_launches = hv.vote_launches;
    ctx->cull_launches = hv.cull_launches;
    ctx->cull_tc_launches = hv.cull_tc_launches;
    ctx->evn = hv.evn;
    ctx->cevn = hv.cevn;
  } else if (graphs && same_as_last && ctx->gstream) {
    // capture this enqueue (the previous solve with the same key ran it directly, so the
    // workspace is sized and every one-time kernel attribute is set)
    if (ctx->gexec) {
      cudaGraphExecDestroy(ctx->gexec);
      ctx->gexec = nullptr;
      ctx->gkey_ok = false;
    }
    RV_CUDA(cudaEventRecord(ctx->gfork, s), "event");
    RV_CUDA(cudaStreamWaitEvent(ctx->gstream, ctx->gfork, 0), "fork");
    ctx->stream = ctx->gstream;
    cudaGraph_t g = nullptr;
    // A workspace buffer reallocated while capturing leaves the nodes captured before it with
    // the freed pointer (nothing runs during a capture, so -- unlike a direct enqueue -- the
    // earlier kernels have not finished with it): such a graph must never be launched.  It
    // happens when the previous solve grew a capacity (overflow / retry), so the capture is
    // discarded and this solve runs directly; the next one captures.
    const uint64_t epoch0 = g_realloc_epoch.load();
    const int64_t c_l = ctx->launches, c_v = ctx->vote_launches, c_c = ctx->cull_launches,
                  c_t = ctx->cull_tc_launches;
    cudaError_t ce = cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeRelaxed);
    int rc = RV_OK;
    if (ce == cudaSuccess) {
      ctx->capturing = true;
      rc = enqueue_one_pass(ctx, x, y, n, eps, ch, mask, hv, ex);
      ctx->capturing = false;
      cudaError_t ee = cudaStreamEndCapture(ctx->gstream, &g);
      if (ce == cudaSuccess) ce = ee;
    }
    ctx->stream = s;
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce == cudaSuccess && g_realloc_epoch.load() != epoch0) {
      cudaGraphDestroy(g);
      ctx->launches = c_l;
      ctx->vote_launches = c_v;
      ctx->cull_launches = c_c;
      ctx->cull_tc_launches = c_t;
      ctx->lastkey_ok = false;  // (run directly below; the solve after this one captures)
      return solve_one_pass(ctx, x, y, n, eps, ch, out, mask, redo, excl);
    }
    cudaGraphExec_t ge = nullptr;
    if (ce == cudaSuccess) ce = cudaGraphInstantiateWithFlags(&ge, g, 0);
    if (g) cudaGraphDestroy(g);
    if (ce != cudaSuccess) {  // not capturable here: run directly from now on
      cudaGetLastError();
      ctx->graphs_on = false;
      ctx->stream = s;
      return solve_one_pass(ctx, x, y, n, eps, ch, out, mask, redo, excl);
    }
    ctx->gexec = ge;
    std::memcpy(ctx->gkey, key, sizeof(key));
    ctx->gkey_ok = true;
    ctx->gepoch = g_realloc_epoch.load();
    hv.launches = ctx->launches;
    hv.vote_launches = ctx->vote_launches;
    hv.cull_launches = ctx->cull_launches;
    hv.cull_tc_launches = ctx->cull_tc_launches;
    hv.evn = ctx->evn;
    hv.cevn = ctx->cevn;
    ctx->ghost = hv;
    RV_CUDA(cudaGraphLaunch(ctx->gexec, ctx->gstream), "launching the solve graph");
    RV_CUDA(cudaEventRecord(ctx->ev1, ctx->gstream), "event");
    RV_CUDA(cudaEventRecord(ctx->gjoin, ctx->gstream), "event");
    RV_CUDA(cudaStreamWaitEvent(s, ctx->gjoin, 0), "join");
  } else {
    if (int rc = enqueue_one_pass(ctx, x, y, n, eps, ch, mask, hv, ex)) return rc;
    RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  }
  std::memcpy(ctx->lastkey, key, sizeof(key));
  ctx->lastkey_ok = ex.n == 0;
  RV_SYNC(cudaEventSynchronize(ctx->ev1), "one-pass solve");
  ctx->collect_vote_ms();
  ctx->ev_collect();
  ctx->cev_collect();
  ctx->cull_ready = false;
  OnePassRB rb(ctx->grb);
  const int64_t m0 = hv.m0;
  const int nph = hv.nph;
  const int L = (int)ch.size();
  cudaEvent_t* ph = ctx->ph;
  if (*rb.bad != ~0ull)
    return ctx->fail(RV_EDATA, "correspondence row %llu has a zero-length or non-finite vector",
                     *rb.bad);
  if (*rb.err != 0) {  // a capacity or the re-dive: the per-level loop redoes the solve
    *redo = true;
    ctx->lastkey_ok = false;  // (capacities may grow: the next solve sizes the workspace directly)
    ctx->redo_reason = *rb.err;
    if ((*rb.err & 16) && ctx->op_lshift > 2) --ctx->op_lshift;  // culling lists
    if ((*rb.err & 3) && ctx->op_cap < kOnePassCapMax)             // level lists / items
      ctx->op_cap = std::min<int64_t>(kOnePassCapMax, ctx->op_cap * 8);
    return RV_OK;
  }
  // ---- the result (as solve_batched_dplan + fill_result + run_refine)
  rv_plan_result r{};
  r.votes = (uint32_t)(*rb.best >> 32);
  r.lin = *rb.best ? 0xffffffffu - (uint32_t)(*rb.best & 0xffffffffu) : 0u;
  r.B = ch[L - 1];
  r.n_tied = *rb.ties;
  r.lb_star = (uint32_t)*rb.lb;
  const int32_t nre = rb.ph[nph - 1];
  r.n_rechecked = nre;
  auto add = [&](int64_t c) {
    r.pair_votes += (uint64_t)c * (uint64_t)n;
    r.cells_evaluated += (uint64_t)c;
    if (r.n_phases < 16) r.cells_per_phase[r.n_phases++] = c;
  };
  add(m0);
  for (int p = 0; p + 1 < nph; ++p) add(rb.ph[p]);
  if (nre > 0) add(nre);
  fill_result(r, out);
  // no successful round keeps q0: the host's block centre (as the per-level loop returns it;
  // the device-decoded copy can differ in the last bit)
  if (*rb.fl & RV_REFINED) std::memcpy(out->q, rb.q, 32);
  else std::memcpy(out->q, out->q_cell, 32);
  out->flags |= *rb.fl;
  out->n_inliers = *rb.ni;
  if (hv.cull) {
    ctx->cull_pairs += *rb.cp;
    ctx->vote_pairs += (uint64_t)m0 * (uint64_t)n;
  } else {
    ctx->vote_pairs += r.pair_votes - (uint64_t)nre * (uint64_t)n;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, ph[0], ctx->ev1);
  out->ms = ms;
  float* tp[6] = {&out->t_setup_ms, &out->t_level0_ms, &out->t_dive_ms, &out->t_bnb_ms,
                  &out->t_final_ms, &out->t_refine_ms};
  for (int k = 0; k < 6; ++k) cudaEventElapsedTime(tp[k], ph[k], ph[k + 1]);
  cudaGetLastError();  // (a failed timing query must not surface in a later launch check)
  return RV_OK;
}

int solve_batched_impl(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets,
                       int32_t P, double eps, int32_t levels, rv_result* out, uint32_t* masks) {
  if (int rc = validate_common(ctx, x, y, eps, levels)) return rc;
  if (!offsets || !out) return ctx->fail(RV_EINVAL, "offsets and out must be non-null");
  if (P < 1 || P > ctx->cfg.max_problems)
    return ctx->fail(RV_EINVAL, "P = %d outside [1, max_problems = %d]", P, ctx->cfg.max_problems);
  if (offsets[0] != 0) return ctx->fail(RV_EINVAL, "offsets[0] must be 0");
  for (int32_t p = 0; p < P; ++p)
    if (offsets[p + 1] - offsets[p] < 2)
      return ctx->fail(RV_EINVAL, "problem %d has fewer than 2 correspondences", p);
  if (offsets[P] > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "total rows exceed max_n");
  cudaStream_t s = ctx->stream;
  {
    const int32_t lev = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
    const std::vector<int32_t> ch(ctx->chain.end() - lev, ctx->chain.end());
    if (one_pass_applies(ctx, P) && dplan_applies(ctx, lev, ch[0], eps)) {
      bool redo = false;
      if (int rc = solve_one_pass(ctx, x, y, offsets[1], eps, ch, out, masks, &redo)) return rc;
      if (!redo) {
        out->launches = ctx->launches;
        ctx->fill_counters(*out);
        return RV_OK;
      }
      const int32_t hs = ctx->host_syncs;
      ctx->reset_counters();  // the per-level loop below redoes the solve
      ctx->host_syncs = hs;
      ctx->retried = true;
    }
  }
  RV_CUDA(cudaEventRecord(ctx->ev0, s), "event");
  const int W = ctx->cfg.world;
  int64_t pb, pe;
  rv_shard_range(P, ctx->cfg.rank, W, &pb, &pe);
  // one problem on several ranks: every rank runs it, each level's votes sharded over the
  // ranks (solve_batched_dplan); no result gather
  const int32_t lev_eff = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
  const bool one_sharded = P == 1 && W > 1 &&
                           dplan_applies(ctx, lev_eff, ctx->chain[ctx->chain.size() - lev_eff], eps);
  if (one_sharded) { pb = 0; pe = 1; }
  // the one-problem split (real ranks or the loopback emulation) is decided from the caller's P
  // here, never from this rank's local share
  ctx->split_one = P == 1 && ctx->effective_world() > 1 &&
                   dplan_applies(ctx, lev_eff, ctx->chain[ctx->chain.size() - lev_eff], eps);
  const int32_t PL = (int32_t)(pe - pb);
  std::vector<rv_result> local(PL);
  Trace tr;
  if (PL > 0) {
    std::vector<int64_t> rows(offsets + pb, offsets + pe + 1), koff;
    const int32_t lev = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
    const std::vector<int32_t> ch(ctx->chain.end() - lev, ctx->chain.end());
    const bool dev_loop = dplan_applies(ctx, lev, ch[0], eps);
    // the culling rows only when solve_batched_dplan can cull this batch (P x m0 buckets)
    bool cull_rows = dev_loop;
    if (dev_loop && PL > 1) {
      if (ctx->grid_host_B != ch[0]) {
        const int64_t m = rv_grid_candidates(ch[0], nullptr, 0);
        ctx->grid_host.resize(m);
        rv_grid_candidates(ch[0], ctx->grid_host.data(), m);
        ctx->grid_host_B = ch[0];
      }
      cull_rows = (int64_t)PL * (int64_t)ctx->grid_host.size() <= ((int64_t)1 << 22);
    }
    if (int rc = run_setup(ctx, x, y, rows.data(), PL, koff, false, cull_rows)) return rc;
    // the device loop reads the data check back with its finalize (no round trip here)
    if (!dev_loop)
      if (int rc = check_bad(ctx)) return rc;
    tr.mark("setup");
    int rc = RV_OK;
    std::vector<rv_plan_result> pres(PL);
    std::vector<int64_t> mw_dev(PL);
    RefineOut ro;
    if (dev_loop) {
      // the refinement starts from the winners decoded on the device and is enqueued before
      // the finalize's wait: one host round trip for the finalize and the refinement
      {
        int64_t w = 0;
        for (int64_t p = 0; p < pb; ++p) w += (offsets[p + 1] - offsets[p] + 31) / 32;
        for (int32_t p = 0; p < PL; ++p) {
          mw_dev[p] = w;
          w += (rows[p + 1] - rows[p] + 31) / 32;
        }
      }
      auto refine_hook = [&]() -> int {
        RV_CUDA(ctx->qs.ensure((size_t)PL * 4), "allocating");
        rv::launch_decode_q0(ctx->dp_best.p, PL, ch.back(), ctx->qs.p, ctx->stream);
        ctx->launches += 1;
        return enqueue_refine(ctx, x, y, rows.data(), PL, eps, ctx->cfg.refine_rounds,
                              mw_dev.data(), masks, ro);
      };
      rc = solve_batched_dplan(ctx, x, y, rows, koff, PL, eps, ch, pres, tr, refine_hook);
      if (rc) return rc;
    } else {
      std::vector<rv_plan*> plans(PL, nullptr);
      parallel_for(PL, [&](int64_t p) {
        rv_plan_create(ctx->chain.data(), (int32_t)ctx->chain.size(), levels,
                       rows[p + 1] - rows[p], eps, (double)ctx->cfg.guard, &plans[p]);
      });
      for (int32_t p = 0; p < PL && !rc; ++p)
        if (!plans[p]) rc = ctx->fail(RV_EINVAL, "invalid search plan");
      tr.mark("plans created");
      std::vector<std::vector<uint32_t>> ca(PL), cb(PL);
      bool l0_on_device = false;
      int64_t m0 = 0;
      while (!rc) {
        std::vector<BatchReq> by_mode[3];
        bool any = false;
        for (int32_t p = 0; p < PL; ++p) {
          BatchReq r;
          r.prob = p;
          if (rv_plan_request(plans[p], &r.B, &r.mode, &r.m, &r.lins)) {
            r.full_grid = rv_plan_request_is_full_grid(plans[p]) != 0;
            by_mode[r.mode].push_back(r);
            any = true;
          }
        }
        if (!any) break;
        tr.mark("requests gathered");
        // level 0 of a batch (every problem, same full grid, bound mode): reduce on the device
        const std::vector<BatchReq>& g0 = by_mode[RV_MODE_BOUND];
        bool l0_reduce = PL >= 2 && (int64_t)g0.size() == PL && !by_mode[1].size() &&
                         !by_mode[2].size();
        for (const BatchReq& r : g0) l0_reduce = l0_reduce && r.full_grid && r.m == g0[0].m;
        if (l0_reduce) {
          int64_t mbg = 0;
          const double* bgh = rv_plan_l0_background(g0[0].B, eps, &mbg);
          l0_reduce = bgh && mbg == g0[0].m;
          if (l0_reduce) {
            m0 = g0[0].m;
            RV_CUDA(ctx->l0cnt.ensure((size_t)PL * m0), "allocating level-0 counts");
            if (ctx->l0bg_B != g0[0].B || ctx->l0bg_eps != eps || ctx->l0bg.cap < (size_t)m0) {
              RV_CUDA(ctx->l0bg.ensure(m0), "allocating");
              RV_CUDA(cudaMemcpy(ctx->l0bg.p, bgh, m0 * sizeof(double), cudaMemcpyHostToDevice),
                      "H2D background");
              ctx->l0bg_B = g0[0].B;
              ctx->l0bg_eps = eps;
            }
            rc = eval_batch(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, g0, ca, cb, ctx->l0cnt.p);
            if (rc) break;
            RV_CUDA(ctx->l0idx.ensure(PL), "allocating");
            rv::launch_l0_argmax(ctx->l0cnt.p, m0, ctx->grid_list.p, g0[0].B, ctx->l0bg.p,
                                 ctx->rows.p, PL, ctx->l0idx.p, ctx->stream);
            ctx->launches += 1;
            std::vector<int32_t> start(PL);
            RV_CUDA(cudaMemcpyAsync(start.data(), ctx->l0idx.p, PL * 4, cudaMemcpyDeviceToHost,
                                    ctx->stream), "D2H");
            RV_SYNC(cudaStreamSynchronize(ctx->stream), "level-0 argmax");
            std::vector<int> bad(PL, 0);
            parallel_for(PL, [&](int64_t p) { bad[p] = rv_plan_feed_l0_start(plans[p], start[p]); });
            for (int b : bad)
              if (b) rc = ctx->fail(RV_ECUDA, "internal: planner rejected the level-0 start");
            l0_on_device = true;
            tr.mark("  level 0 on device");
            continue;
          }
        }
        for (int md = 0; md < 3 && !rc; ++md) {
          if (by_mode[md].empty()) continue;
          rc = eval_batch(ctx, x, y, rows, koff, eps, md, by_mode[md], ca, cb);
          if (rc) break;
          tr.mark(md == 0 ? "  eval bound" : md == 1 ? "  eval final" : "  eval exact");
          const std::vector<BatchReq>& grp = by_mode[md];
          std::vector<int> bad(grp.size(), 0);
          parallel_for((int64_t)grp.size(), [&](int64_t q) {
            const BatchReq& r = grp[q];
            bad[q] = rv_plan_feed(plans[r.prob], ca[r.prob].data(), cb[r.prob].data()) != 0;
          });
          for (int b : bad)
            if (b) rc = ctx->fail(RV_ECUDA, "internal: planner rejected counts");
          tr.mark("  feed");
        }
        if (rc || !l0_on_device) continue;
        // plans whose dive ended: compact their level-0 survivors (UB >= lb*) on the device
        std::vector<int32_t> need;
        std::vector<int64_t> lbs;
        for (int32_t p = 0; p < PL; ++p) {
          int64_t lb = 0;
          if (rv_plan_needs_l0_survivors(plans[p], &lb)) {
            need.push_back(p);
            lbs.push_back(lb);
          }
        }
        if (need.empty()) continue;
        const int32_t J = (int32_t)need.size();
        RV_CUDA(ctx->l0idx.ensure(2 * (size_t)J + 1), "allocating");
        RV_CUDA(ctx->l0aux.ensure(2 * (size_t)J + 1), "allocating");
        int32_t* dprob = ctx->l0idx.p;
        int32_t* dcnt = ctx->l0idx.p + J;
        int64_t* dlb = ctx->l0aux.p;
        int64_t* doff = ctx->l0aux.p + J;
        RV_CUDA(cudaMemcpyAsync(dprob, need.data(), J * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        RV_CUDA(cudaMemcpyAsync(dlb, lbs.data(), J * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        rv::launch_l0_survivors(ctx->l0cnt.p, m0, dprob, dlb, nullptr, J, dcnt, nullptr, ctx->stream);
        std::vector<int32_t> k(J);
        RV_CUDA(cudaMemcpyAsync(k.data(), dcnt, J * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        RV_SYNC(cudaStreamSynchronize(ctx->stream), "level-0 survivors");
        std::vector<int64_t> offv(J + 1, 0);
        for (int32_t j = 0; j < J; ++j) offv[j + 1] = offv[j] + k[j];
        DevBuf<int32_t>& surv = ctx->l0surv;
        RV_CUDA(surv.ensure(std::max<int64_t>(1, offv[J])), "allocating");
        RV_CUDA(cudaMemcpyAsync(doff, offv.data(), J * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        rv::launch_l0_survivors(ctx->l0cnt.p, m0, dprob, dlb, doff, J, nullptr, surv.p, ctx->stream);
        ctx->launches += 2;
        std::vector<int32_t> idx(std::max<int64_t>(1, offv[J]));
        RV_CUDA(cudaMemcpyAsync(idx.data(), surv.p, offv[J] * 4, cudaMemcpyDeviceToHost, ctx->stream),
                "D2H");
        RV_SYNC(cudaStreamSynchronize(ctx->stream), "level-0 survivors");
        std::vector<int> bad(J, 0);
        parallel_for(J, [&](int64_t j) {
          bad[j] = rv_plan_feed_l0_survivors(plans[need[j]], idx.data() + offv[j], k[j]);
        });
        for (int b : bad)
          if (b) rc = ctx->fail(RV_ECUDA, "internal: planner rejected the level-0 survivors");
        tr.mark("  level-0 survivors");
      }
      if (!rc)
        for (int32_t p = 0; p < PL; ++p) rv_plan_get_result(plans[p], &pres[p]);
      for (rv_plan* pl : plans) rv_plan_destroy(pl);
      if (rc) return rc;
    }
    std::vector<double> q0((size_t)PL * 4), qf((size_t)PL * 4);
    std::vector<int32_t> fl(PL), ids(PL);
    std::vector<uint32_t> ni(PL);
    std::vector<int64_t> mw(PL);
    {
      int64_t w = 0;
      for (int64_t p = 0; p < pb; ++p) w += (offsets[p + 1] - offsets[p] + 31) / 32;
      for (int32_t p = 0; p < PL; ++p) {
        fill_result(pres[p], &local[p]);
        std::memcpy(&q0[4 * p], local[p].q_cell, 32);
        ids[p] = p;
        mw[p] = w;
        w += (rows[p + 1] - rows[p] + 31) / 32;
      }
    }
    tr.mark("results");
    if (dev_loop) {  // read back with the finalize; no successful round keeps the host's q0
      for (int32_t p = 0; p < PL; ++p) {
        fl[p] = ro.flags[p] & (RV_REFINED | RV_DEGENERATE);
        ni[p] = ro.ninl[p];
        if (fl[p] & RV_REFINED) std::memcpy(&qf[4 * p], ro.q + 4 * p, 32);
        else std::memcpy(&qf[4 * p], &q0[4 * p], 32);
      }
    } else {
      // rows are absolute: refine over the local offsets table
      rc = run_refine(ctx, x, y, rows.data(), PL, ids.data(), eps, q0.data(),
                      ctx->cfg.refine_rounds, mw.data(), masks, qf.data(), fl.data(), ni.data());
      if (rc) return rc;
    }
    tr.mark("refine");
    for (int32_t p = 0; p < PL; ++p) {
      std::memcpy(local[p].q, &qf[4 * p], 32);
      local[p].flags |= fl[p];
      local[p].n_inliers = ni[p];
    }
  }
  RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  RV_SYNC(cudaEventSynchronize(ctx->ev1), "event");
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  for (rv_result& r : local) {
    r.ms = ms;
    ctx->fill_counters(r);
  }
  if (!ctx->comm || one_sharded) {
    std::memcpy(out, local.data(), (size_t)P * sizeof(rv_result));
    return RV_OK;
  }
  // all-gather the per-rank result slices (fixed-size slots of ceil(P/W) results)
  const int64_t chunk = (P + W - 1) / W;
  const size_t slot = (size_t)chunk * sizeof(rv_result);
  RV_CUDA(ctx->gather.ensure(slot * (W + 1)), "allocating");
  RV_CUDA(ctx->up.ensure(slot + 256), "allocating staging");
  RV_CUDA(ctx->down.ensure(slot * W + 256), "allocating staging");
  ctx->up.reset();
  char* hu = ctx->up.take<char>(slot);
  std::memset(hu, 0, slot);
  if (PL > 0) std::memcpy(hu, local.data(), (size_t)PL * sizeof(rv_result));
  char* mine = ctx->gather.p + slot * W;
  RV_CUDA(cudaMemcpyAsync(mine, hu, slot, cudaMemcpyHostToDevice, s), "H2D");
  ncclResult_t nr = nccl().AllGather(mine, ctx->gather.p, slot, ncclChar, ctx->comm, s);
  if (nr != ncclSuccess) return ctx->fail(RV_ENCCL, "ncclAllGather: %s", nccl().GetErrorString(nr));
  ctx->down.reset();
  char* hd = ctx->down.take<char>(slot * W);
  RV_CUDA(cudaMemcpyAsync(hd, ctx->gather.p, slot * W, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "gather");
  for (int r = 0; r < W; ++r) {
    int64_t b, e;
    rv_shard_range(P, r, W, &b, &e);
    std::memcpy(out + b, hd + slot * r, (size_t)(e - b) * sizeof(rv_result));
  }
  return RV_OK;
}

}  // namespace rvi
