// rv_api.cpp -- the C-ABI of librotvote (include/rotvote.h): validation, context lifetime,
// result assembly and the entry points (the steps live in rv_setup.cpp, rv_host_plan.cpp and
// rv_level_loop.cpp).
#include "rv_ctx.h"

namespace rvi {

void canonicalize(double q[4]) {
  bool flip;
  if (q[3] < -1e-15) flip = false;
  else if (q[3] > 1e-15) flip = true;
  else {
    flip = false;
    for (int a = 0; a < 3; ++a)
      if (q[a] != 0.0) { flip = q[a] < 0.0; break; }
  }
  if (flip)
    for (int a = 0; a < 4; ++a) q[a] = -q[a];
}

void canonical_cell_quat(int32_t B, uint32_t lin, double q[4]) {
  int32_t i, j, k;
  rv::lin_to_ijk(lin, B, i, j, k);
  rv::cell_quat(B, i, j, k, q);
  canonicalize(q);
}

int validate_common(rv_ctx* ctx, const void* x, const void* y, double eps, int32_t levels) {
  if (!ctx) return RV_EINVAL;
  if (!x || !y) return ctx->fail(RV_EINVAL, "x and y must be non-null");
  if (!(eps > 0.0) || !(eps < 3.141592653589793))
    return ctx->fail(RV_EINVAL, "eps must lie in (0, pi), got %g", eps);
  if (levels < 0 || levels > (int32_t)ctx->chain.size())
    return ctx->fail(RV_EINVAL, "levels must lie in [0, %d], got %d", (int)ctx->chain.size(), levels);
  return RV_OK;
}

void fill_result(const rv_plan_result& pr, rv_result* out) {
  std::memset(out, 0, sizeof(*out));
  out->votes = pr.votes;
  int32_t i, j, k;
  rv::lin_to_ijk(pr.lin, pr.B, i, j, k);
  out->cell[0] = i; out->cell[1] = j; out->cell[2] = k;
  out->B = pr.B;
  out->n_tied = pr.n_tied;
  out->pair_votes = pr.pair_votes;
  out->cells_evaluated = pr.cells_evaluated;
  out->lb_star = pr.lb_star;
  out->n_rechecked = pr.n_rechecked;
  out->n_phases = std::min(pr.n_phases, (int32_t)RV_MAX_PHASES);
  for (int p = 0; p < out->n_phases; ++p) out->cells_per_phase[p] = pr.cells_per_phase[p];
  if (pr.n_rechecked > 0) out->flags |= RV_RECHECKED;
  canonical_cell_quat(pr.B, pr.lin, out->q_cell);
}

}  // namespace rvi

using namespace rvi;

// =============================================================================================
extern "C" {

void rot_vote_default_config(rv_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->device = 0;
  cfg->rank = 0;
  cfg->world = 1;
  cfg->nccl_id = nullptr;
  cfg->max_n = 1 << 20;
  cfg->max_problems = 1;
  cfg->chain_len = 0;
  cfg->refine_rounds = 2;
  cfg->guard = 1e-5f;
  cfg->stream = nullptr;
  cfg->emulate_world = 0;
  cfg->tensor_vote = 1;
  cfg->cull = 1;
}

int rot_vote_get_unique_id(void* id_out) {
  if (!id_out) return RV_EINVAL;
  NcclApi& a = nccl();
  if (!a.ok) return RV_ENCCL;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return RV_ENCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return RV_OK;
}

int rot_vote_create(const rv_config* cfg, rv_ctx** out) {
  if (!out) return RV_EINVAL;
  *out = nullptr;
  if (!cfg) return RV_EINVAL;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return RV_EINVAL;
  if (cfg->world > 1 && (!cfg->nccl_id || cfg->emulate_world > 1)) return RV_EINVAL;
  if (cfg->nccl_id && cfg->emulate_world > 1) return RV_EINVAL;
  if (cfg->max_n < 2 || cfg->max_n > ((int64_t)1 << 31) - 4096) return RV_EINVAL;
  if (cfg->max_problems < 1 || cfg->refine_rounds < 0 || !(cfg->guard >= 0.0f)) return RV_EINVAL;
  if (cfg->chain_len < 0 || cfg->chain_len > RV_MAX_CHAIN) return RV_EINVAL;
  if (cfg->cull < 0 || cfg->cull > 2 || cfg->planner < 0 || cfg->planner > 2) return RV_EINVAL;
  if (cfg->ct_sched < 0 || cfg->ct_sched > 1) return RV_EINVAL;
  rv_ctx* ctx = new rv_ctx();
  ctx->cfg = *cfg;
  if (cfg->chain_len == 0) ctx->chain.assign(kDefaultChain, kDefaultChain + 6);
  else ctx->chain.assign(cfg->chain, cfg->chain + cfg->chain_len);
  for (size_t l = 0; l < ctx->chain.size(); ++l) {
    if (ctx->chain[l] < 1 || ctx->chain[l] > 1625 ||
        (l > 0 && ctx->chain[l] % ctx->chain[l - 1] != 0)) {
      delete ctx;
      return RV_EINVAL;
    }
  }
  ctx->stream = (cudaStream_t)cfg->stream;
  ctx->tc_on = cfg->tensor_vote != 0;
  ctx->cull_on = ctx->tc_on && cfg->cull != 0;
  ctx->cull_tc = cfg->cull != 2;
  ctx->host_plan = cfg->planner == 1;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->evv0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->evv1);
  for (int k = 0; k < 8 && e == cudaSuccess; ++k) e = cudaEventCreate(&ctx->ph[k]);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->gfork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->gjoin, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&ctx->grb), 4096);
  if (e == cudaSuccess) {
    ctx->stride = pad4(cfg->max_n) + 64;
    e = ctx->k9.ensure((size_t)9 * ctx->stride);
  }
  if (e == cudaSuccess) e = ctx->bad.ensure(1);
  if (e == cudaSuccess) e = ctx->dp_tdone.ensure(1);  // tail-scan counter: zero between launches
  if (e == cudaSuccess) e = cudaMemset(ctx->dp_tdone.p, 0, ctx->dp_tdone.cap * 4);
  if (e == cudaSuccess) e = ctx->up.ensure(1 << 20);
  if (e == cudaSuccess) e = ctx->down.ensure(1 << 20);
  if (e != cudaSuccess) {
    int code = e == cudaErrorMemoryAllocation ? RV_ENOMEM : RV_ECUDA;
    rot_vote_destroy(ctx);
    return code;
  }
  if (cfg->nccl_id) {  // world > 1, or a 1-rank communicator (exercises the NCCL path)
    NcclApi& a = nccl();
    if (!a.ok) {
      rot_vote_destroy(ctx);
      return RV_ENCCL;
    }
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    if (a.CommInitRank(&ctx->comm, cfg->world, id, cfg->rank) != ncclSuccess) {
      ctx->comm = nullptr;
      rot_vote_destroy(ctx);
      return RV_ENCCL;
    }
  }
  *out = ctx;
  return RV_OK;
}

void rot_vote_destroy(rv_ctx* ctx) {
  if (!ctx) return;
  if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
  ctx->tctab.release(); ctx->tctab_rm.release(); ctx->toffs.release();
  ctx->k9.release(); ctx->lins.release(); ctx->cnt.release(); ctx->vsegs.release();
  ctx->vitems.release(); ctx->rsegs.release(); ctx->ritems.release(); ctx->partials.release();
  ctx->qs.release(); ctx->flags.release(); ctx->ninl.release(); ctx->rows.release();
  ctx->koffs.release(); ctx->bad.release(); ctx->dp_tdone.release(); ctx->hx.release(); ctx->hy.release();
  ctx->hmask.release(); ctx->gather.release(); ctx->grid_list.release();
  ctx->l0cnt.release(); ctx->l0bg.release(); ctx->l0idx.release(); ctx->l0aux.release();
  ctx->l0surv.release(); ctx->atab.release(); ctx->ablk.release();
  for (int b = 0; b < 3; ++b) {
    ctx->dp_lins[b].release(); ctx->dp_ca[b].release(); ctx->dp_cb[b].release();
    ctx->dp_off[b].release(); ctx->dp_cnt[b].release();
  }
  ctx->dp_lb2.release();
  for (int b = 0; b < 2; ++b) ctx->dp_actr[b].release();
  for (int b = 0; b < 3; ++b) ctx->dp_bring[b].release();
  ctx->dp_rflag.release(); ctx->dp_rany.release(); ctx->dp_rdone.release();
  ctx->dp_lb.release(); ctx->dp_rcnt.release(); ctx->dp_ties.release();
  ctx->dp_pick.release(); ctx->dp_rlins.release(); ctx->dp_ex.release(); ctx->dp_lmax.release();
  ctx->rg_m.release(); ctx->rg_n.release(); ctx->rg_cnt.release(); ctx->rg_off.release();
  ctx->rg_bins.release(); ctx->rg_acc.release(); ctx->rg_best.release(); ctx->rg_sums.release();
  ctx->dp_best.release(); ctx->dp_best_r.release(); ctx->dp_ties_r.release(); ctx->excl_q.release(); ctx->a1_acc.release(); ctx->a1_tab.release(); ctx->a1_best.release(); ctx->dp_ioff.release(); ctx->dp_aoff.release(); ctx->dp_tot.release();
  ctx->dp_icnt.release(); ctx->dp_phase.release(); ctx->dp_err.release();
  ctx->dp_pcnt.release(); ctx->dp_scnt.release(); ctx->dp_poff.release(); ctx->dp_sbase.release();
  ctx->cbits.release(); ctx->k12.release(); ctx->lut0.release(); ctx->lutg.release(); ctx->goff.release(); ctx->gmem.release(); ctx->lut0_B = 0; ctx->c_act.release();
  ctx->c_lofs.release(); ctx->c_lidx.release(); ctx->c_fill.release();
  ctx->c_ioff.release(); ctx->c_aoff.release(); ctx->c_acnt.release(); ctx->c_tanc.release();
  ctx->c_tslot.release(); ctx->c_cidx.release(); ctx->c_phi.release(); ctx->c_icnt.release();
  ctx->c_tphi.release();
  ctx->c_work.release(); ctx->c_items.release(); ctx->c_pairs.release();
  for (cudaEvent_t e : ctx->cevs) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->evs) cudaEventDestroy(e);
  ctx->up.release(); ctx->down.release(); ctx->up2.release(); ctx->down2.release();
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evv0) cudaEventDestroy(ctx->evv0);
  if (ctx->evv1) cudaEventDestroy(ctx->evv1);
  for (cudaEvent_t e : ctx->ph)
    if (e) cudaEventDestroy(e);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->gfork) cudaEventDestroy(ctx->gfork);
  if (ctx->gjoin) cudaEventDestroy(ctx->gjoin);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->grb) cudaFreeHost(ctx->grb);
  delete ctx;
}

const char* rot_vote_last_error(const rv_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

int rot_vote_solve(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                   int32_t levels, rv_result* out, uint32_t* inlier_mask) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  ctx->reset_counters();
  return solve_impl(ctx, x, y, n, eps, levels, out, inlier_mask);
}

int rot_vote_solve_host(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                        int32_t levels, rv_result* out, uint32_t* inlier_mask) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  ctx->reset_counters();
  if (int rc = validate_common(ctx, x, y, eps, levels)) return rc;
  if (n < 2 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  RV_CUDA(ctx->hx.ensure(3 * n), "allocating");
  RV_CUDA(ctx->hy.ensure(3 * n), "allocating");
  const int64_t words = (n + 31) / 32;
  if (inlier_mask) RV_CUDA(ctx->hmask.ensure(words), "allocating");
  RV_CUDA(cudaMemcpyAsync(ctx->hx.p, x, 12 * n, cudaMemcpyHostToDevice, ctx->stream), "H2D x");
  RV_CUDA(cudaMemcpyAsync(ctx->hy.p, y, 12 * n, cudaMemcpyHostToDevice, ctx->stream), "H2D y");
  int rc = solve_impl(ctx, ctx->hx.p, ctx->hy.p, n, eps, levels, out,
                      inlier_mask ? ctx->hmask.p : nullptr);
  if (rc) return rc;
  if (inlier_mask) {
    RV_CUDA(cudaMemcpyAsync(inlier_mask, ctx->hmask.p, words * 4, cudaMemcpyDeviceToHost,
                            ctx->stream), "D2H mask");
    RV_CUDA(cudaStreamSynchronize(ctx->stream), "D2H mask");
  }
  return RV_OK;
}

int rot_vote_solve_batched(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets,
                           int32_t P, double eps, int32_t levels, rv_result* out, uint32_t* masks) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  ctx->reset_counters();
  return solve_batched_impl(ctx, x, y, offsets, P, eps, levels, out, masks);
}

int rot_vote_setup(rv_ctx* ctx, const float* x, const float* y, int64_t n, float* k_out) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (!x || !y || !k_out) return ctx->fail(RV_EINVAL, "null pointer");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  for (int j = 0; j < 9; ++j)
    RV_CUDA(cudaMemcpyAsync(k_out + (int64_t)j * n, ctx->k9.p + (int64_t)j * ctx->stride, n * 4,
                            cudaMemcpyDeviceToDevice, ctx->stream), "copy K");
  return check_bad(ctx);
}

int rot_vote_count_cells(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t B,
                         const uint32_t* lins, int64_t m, double eps, int32_t mode, uint32_t* cnt_a,
                         uint32_t* cnt_b) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (int rc = validate_common(ctx, x, y, eps, 0)) return rc;
  if (!lins || !cnt_a || ((mode == RV_MODE_FINAL || mode == RV_MODE_FINAL_TC) && !cnt_b) || m < 0)
    return ctx->fail(RV_EINVAL, "null pointer");
  if (mode < RV_MODE_BOUND || mode > RV_MODE_FINAL_TC) return ctx->fail(RV_EINVAL, "bad mode");
  if (B < 1 || B > 1625) return ctx->fail(RV_EINVAL, "bad B");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  if (m == 0) return RV_OK;
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  if (int rc = check_bad(ctx)) return rc;
  std::vector<uint32_t> hl(m), ha(m), hb(m);
  RV_CUDA(cudaMemcpyAsync(hl.data(), lins, m * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  RV_CUDA(cudaStreamSynchronize(ctx->stream), "D2H");
  if (int rc = eval_request(ctx, x, y, n, eps, B, mode, m, hl.data(), ha.data(), hb.data(),
                            /*auto_tc=*/false))
    return rc;
  RV_CUDA(cudaMemcpyAsync(cnt_a, ha.data(), m * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  if (mode == RV_MODE_FINAL || mode == RV_MODE_FINAL_TC)
    RV_CUDA(cudaMemcpyAsync(cnt_b, hb.data(), m * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  RV_CUDA(cudaStreamSynchronize(ctx->stream), "H2D");
  return RV_OK;
}

int rot_vote_count_cells_culled(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t B0,
                                int32_t B, const uint32_t* lins, int64_t m, double eps,
                                int32_t mode, uint32_t* cnt_a, uint32_t* cnt_b, uint32_t* bits_out) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (int rc = validate_common(ctx, x, y, eps, 0)) return rc;
  if (!ctx->cull_on) return ctx->fail(RV_EINVAL, "needs a context created with tensor_vote = 1, cull = 1");
  if (!lins || !cnt_a || (mode == RV_MODE_FINAL && !cnt_b) || m < 0)
    return ctx->fail(RV_EINVAL, "null pointer");
  if (mode != RV_MODE_BOUND && mode != RV_MODE_FINAL) return ctx->fail(RV_EINVAL, "bad mode");
  if (B0 < 1 || B0 > 90 || B < B0 || B > 1625 || B % B0 != 0) return ctx->fail(RV_EINVAL, "bad B0 / B");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  cudaStream_t s = ctx->stream;
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  ctx->reset_counters();
  ctx->split_one = false;  // a one-rank step: this rank compacts every list
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  if (int rc = check_bad(ctx)) return rc;
  const int64_t m0 = rv_grid_candidates(B0, nullptr, 0);
  if (ctx->grid_host_B != B0) {
    ctx->grid_host.resize(m0);
    rv_grid_candidates(B0, ctx->grid_host.data(), m0);
    ctx->grid_host_B = B0;
  }
  RV_CUDA(ctx->grid_list.ensure(m0), "allocating grid list");
  RV_CUDA(cudaMemcpy(ctx->grid_list.p, ctx->grid_host.data(), m0 * 4, cudaMemcpyHostToDevice), "H2D");
  ctx->grid_list_B = B0;
  ctx->grid_list_m = m0;
  const int64_t wpc = ctx->tc_toff[1] / 32;
  RV_CUDA(ctx->cbits.ensure((size_t)m0 * wpc), "allocating level-0 bitmasks");
  RV_CUDA(ctx->l0cnt.ensure(m0), "allocating");
  RV_CUDA(cudaMemsetAsync(ctx->l0cnt.p, 0, m0 * 4, s), "memset");
  if (int rc = cull_prepare(ctx, B0, m0, 1)) return rc;
  RV_CUDA(cudaMemsetAsync(ctx->dp_err.p, 0, 4, s), "memset");
  const std::vector<int64_t> rows{0, n};
  ctx->cull_ready = false;
  const rv::DpList l0{ctx->grid_list.p, 1, m0, nullptr, nullptr, ctx->l0cnt.p, ctx->l0cnt.p};
  if (int rc = vote_level(ctx, x, y, rows, koff, eps, RV_MODE_BOUND, B0, l0, 1, m0, n, true))
    return rc;
  if (int rc = cull_build_lists(ctx, 1, m0, ctx->l0cnt.p, true)) return rc;
  if (m > 0 && !ctx->cull_ready) return ctx->fail(RV_ENOMEM, "level-0 lists exceed 2^29 entries");
  if (m > 0) {
    RV_CUDA(ctx->dp_sbase.ensure(2), "allocating");
    RV_CUDA(ctx->dp_scnt.ensure(1), "allocating");
    const int64_t hb[2] = {0, m};
    const int32_t hc = (int32_t)m;
    RV_CUDA(cudaMemcpyAsync(ctx->dp_sbase.p, hb, 16, cudaMemcpyHostToDevice, s), "H2D");
    RV_CUDA(cudaMemcpyAsync(ctx->dp_scnt.p, &hc, 4, cudaMemcpyHostToDevice, s), "H2D");
    RV_CUDA(cudaMemsetAsync(cnt_a, 0, m * 4, s), "memset");
    if (mode == RV_MODE_FINAL) RV_CUDA(cudaMemsetAsync(cnt_b, 0, m * 4, s), "memset");
    const rv::DpList Ld{lins, 0, 0, ctx->dp_sbase.p, ctx->dp_scnt.p, cnt_a,
                        mode == RV_MODE_FINAL ? cnt_b : cnt_a};
    int rc = vote_level(ctx, x, y, rows, koff, eps, mode, B, Ld, 1, m, n);
    ctx->cull_ready = false;
    if (rc) return rc;
  }
  if (bits_out)
    RV_CUDA(cudaMemcpyAsync(bits_out, ctx->cbits.p, (size_t)m0 * wpc * 4, cudaMemcpyDeviceToDevice, s),
            "D2D");
  int32_t herr = 0;
  RV_CUDA(cudaMemcpyAsync(&herr, ctx->dp_err.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaStreamSynchronize(s), "culled vote");
  if (herr) return ctx->fail(RV_ECUDA, "internal: culled item planner invariant violated (code %d)", herr);
  return RV_OK;
}

int rot_vote_debug_tc_scores(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t B,
                             const uint32_t* lins, int64_t m, double eps, float* out) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (int rc = validate_common(ctx, x, y, eps, 0)) return rc;
  if (!ctx->tc_on) return ctx->fail(RV_EINVAL, "needs a context created with tensor_vote = 1");
  if (!lins || !out || m < 1 || B < 1 || B > 1625) return ctx->fail(RV_EINVAL, "bad arguments");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  const int64_t offs[2] = {0, n};
  std::vector<int64_t> koff;
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  if (int rc = check_bad(ctx)) return rc;
  const int64_t ld = (n + rv::kTcN - 1) / rv::kTcN * rv::kTcN;
  rv::VoteSeg sg{};
  sg.lins = lins;
  sg.cnt_a = nullptr;
  sg.cnt_b = nullptr;
  sg.koff = 0;
  sg.row = 0;
  sg.n = (int32_t)n;
  sg.B = B;
  sg.eps = eps;
  std::vector<rv::VoteItem> items;
  std::vector<rv::ABlock> ablocks;
  build_tc_items({m}, {n}, ctx->num_sms, items, ablocks);
  RV_CUDA(ctx->vsegs.ensure(1), "allocating");
  RV_CUDA(ctx->vitems.ensure(items.size()), "allocating");
  RV_CUDA(cudaMemcpy(ctx->vsegs.p, &sg, sizeof(sg), cudaMemcpyHostToDevice), "H2D");
  RV_CUDA(cudaMemcpy(ctx->vitems.p, items.data(), items.size() * sizeof(rv::VoteItem),
                     cudaMemcpyHostToDevice), "H2D");
  if (int rc = launch_tc(ctx, ablocks, (int32_t)items.size(), false, out, ld)) return rc;
  RV_CUDA(cudaGetLastError(), "launching K3-TC");
  RV_CUDA(cudaStreamSynchronize(ctx->stream), "K3-TC");
  return RV_OK;
}

int rot_vote_solve_multi(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                         int32_t levels, int32_t K, double rho, rv_result* out,
                         int32_t* n_found) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  ctx->reset_counters();
  return solve_multi_impl(ctx, x, y, n, eps, levels, K, rho, out, n_found);
}

int rot_vote_rigid(rv_ctx* ctx, const float* x, const float* y, int64_t n, double mu_t,
                   double eps, int32_t levels, double t_lo, double t_hi, double t_step,
                   rv_rigid_result* out, int32_t* pair_ij, int64_t pair_cap) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  ctx->reset_counters();
  return rigid_impl(ctx, x, y, n, mu_t, eps, levels, t_lo, t_hi, t_step, out, pair_ij, pair_cap);
}

int rot_vote_translation(rv_ctx* ctx, const float* x, const float* y, int64_t n,
                         const double* q, double t_lo, double t_hi, double t_step,
                         int64_t* lin, uint32_t* votes, double* t, double* t_mean) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  return translation_impl(ctx, x, y, n, q, t_lo, t_hi, t_step, lin, votes, t, t_mean);
}

int rot_vote_alg1(rv_ctx* ctx, const float* x, const float* y, int64_t n, int32_t J,
                  rv_alg1_result* out, uint32_t* acc_out) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (!x || !y || !out) return ctx->fail(RV_EINVAL, "x, y and out must be non-null");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  if (J < 1 || J > (1 << 20)) return ctx->fail(RV_EINVAL, "J must lie in [1, 2^20]");
  const int32_t B = ctx->chain.back();
  const int64_t m = (int64_t)B * B * B;
  cudaStream_t s = ctx->stream;
  RV_CUDA(ctx->a1_acc.ensure(m), "allocating the Algorithm-1 accumulator");
  RV_CUDA(ctx->a1_best.ensure(2), "allocating");
  if (ctx->a1_J != J) {
    // alpha_j = -pi + 2 pi j / J  (Alg. 1 line 2), the half angles' cos / sin in libm double
    std::vector<double> tab(2 * (size_t)J);
    const double pi = 3.14159265358979323846;
    for (int32_t j = 0; j < J; ++j) {
      const double half = (-pi + 2.0 * pi * (double)j / (double)J) / 2.0;
      tab[j] = std::cos(half);
      tab[J + j] = std::sin(half);
    }
    RV_CUDA(ctx->a1_tab.ensure(2 * (size_t)J), "allocating");
    RV_CUDA(cudaMemcpy(ctx->a1_tab.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), "H2D");
    ctx->a1_J = J;
  }
  cudaEvent_t e2, e3;
  RV_CUDA(cudaEventCreate(&e2), "event");
  RV_CUDA(cudaEventCreate(&e3), "event");
  RV_CUDA(cudaEventRecord(ctx->ev0, s), "event");
  RV_CUDA(cudaMemsetAsync(ctx->a1_acc.p, 0, m * 4, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->a1_best.p, 0, 8, s), "memset");
  RV_CUDA(cudaMemsetAsync(ctx->a1_best.p + 1, 0xff, 8, s), "memset");
  RV_CUDA(cudaEventRecord(e2, s), "event");
  rv::launch_alg1(x, y, n, B, J, ctx->a1_tab.p, ctx->a1_tab.p + J, ctx->a1_acc.p,
                  ctx->a1_best.p + 1, ctx->a1_best.p, s);
  RV_CUDA(cudaGetLastError(), "launching Algorithm 1");
  RV_CUDA(cudaEventRecord(e3, s), "event");
  if (acc_out)
    RV_CUDA(cudaMemcpyAsync(acc_out, ctx->a1_acc.p, m * 4, cudaMemcpyDeviceToDevice, s), "D2D");
  unsigned long long hb[2];
  RV_CUDA(cudaMemcpyAsync(hb, ctx->a1_best.p, 16, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  RV_CUDA(cudaStreamSynchronize(s), "Algorithm 1");
  float ms = 0, vms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  cudaEventElapsedTime(&vms, e2, e3);
  cudaEventDestroy(e2);
  cudaEventDestroy(e3);
  if (hb[1] != ~0ull)
    return ctx->fail(RV_EDATA, "correspondence row %llu has a zero-length or non-finite vector",
                     hb[1]);
  std::memset(out, 0, sizeof(*out));
  const uint32_t lin = 0xffffffffu - (uint32_t)(hb[0] & 0xffffffffu);
  out->votes = (uint32_t)(hb[0] >> 32);
  int32_t i, j, k;
  rv::lin_to_ijk(lin, B, i, j, k);
  out->cell[0] = i; out->cell[1] = j; out->cell[2] = k;
  canonical_cell_quat(B, lin, out->q);
  out->B = B;
  out->J = J;
  out->samples = (uint64_t)n * (uint64_t)J;
  out->ms = ms;
  out->vote_ms = vms;
  return RV_OK;
}

int rot_vote_refine(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                    const double* q0, int32_t rounds, double* q_out, int32_t* flags,
                    uint32_t* n_inliers, uint32_t* mask) {
  if (!ctx) return RV_EINVAL;
  ctx->err.clear();
  cudaSetDevice(ctx->cfg.device);
  if (int rc = validate_common(ctx, x, y, eps, 0)) return rc;
  if (!q0 || !q_out || rounds < 0) return ctx->fail(RV_EINVAL, "bad arguments");
  if (n < 1 || n > ctx->cfg.max_n) return ctx->fail(RV_EINVAL, "n out of range");
  double q[4];
  const double nq = std::sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
  if (!(nq > 0.0)) return ctx->fail(RV_EINVAL, "q0 must be nonzero");
  for (int a = 0; a < 4; ++a) q[a] = q0[a] / nq;
  canonicalize(q);
  const int64_t offs[2] = {0, n};
  const int32_t pid = 0;
  const int64_t mw = 0;
  int32_t fl = 0;
  uint32_t ni = 0;
  if (int rc = run_refine(ctx, x, y, offs, 1, &pid, eps, q, rounds, &mw, mask, q_out, &fl, &ni))
    return rc;
  if (flags) *flags = fl;
  if (n_inliers) *n_inliers = ni;
  return RV_OK;
}

}  // extern "C"

