// rv_setup.cpp -- a1 (K1 / K1-TC setup launches and the data check) and a6 (the linear
// refinement, K6 / K7) for P problems.
#include "rv_ctx.h"

namespace rvi {

// ---- K1 for P problems ----------------------------------------------------------------------
int run_setup(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
              std::vector<int64_t>& koff_out, bool dev_offsets, bool cull_rows) {
  koff_out.assign(P + 1, 0);
  for (int32_t p = 0; p < P; ++p) koff_out[p + 1] = koff_out[p] + pad4(offsets[p + 1] - offsets[p]);
  const int64_t total = koff_out[P];
  if (total > ctx->stride) {
    ctx->stride = pad4(total);
    RV_CUDA(ctx->k9.ensure((size_t)9 * ctx->stride), "allocating K table");
  }
  RV_CUDA(ctx->rows.ensure(P + 1), "allocating offsets");
  RV_CUDA(ctx->koffs.ensure(P + 1), "allocating offsets");
  RV_CUDA(ctx->bad.ensure(1), "allocating flag");
  RV_CUDA(ctx->up.ensure(3 * (P + 1) * sizeof(int64_t) + 2048), "allocating staging");
  ctx->up.reset();
  if (dev_offsets) {
    // one problem: the caller wrote rows / koffs / toffs with launch_set_consts (the offsets
    // as kernel arguments, graph-capturable)
  } else {
    int64_t* hrows = ctx->up.take<int64_t>(P + 1);
    int64_t* hk = ctx->up.take<int64_t>(P + 1);
    std::memcpy(hrows, offsets, (P + 1) * sizeof(int64_t));
    std::memcpy(hk, koff_out.data(), (P + 1) * sizeof(int64_t));
    RV_CUDA(cudaMemcpyAsync(ctx->rows.p, hrows, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
            "copying offsets");
    RV_CUDA(cudaMemcpyAsync(ctx->koffs.p, hk, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
            "copying offsets");
  }
  RV_CUDA(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), ctx->stream), "memset");
  // one problem with the tensor-core tables: K1 runs inside K1-TC (x, y read once)
  const bool fused = ctx->tc_on && P == 1;
  if (!fused) {
    rv::launch_setup(x, y, ctx->rows.p, ctx->koffs.p, P, total, ctx->k9.p, ctx->stride, ctx->bad.p,
                     ctx->stream);
    ctx->launches += 1;
  }
  if (ctx->tc_on) {
    std::vector<int64_t> toff(P + 1, 0);
    for (int32_t p = 0; p < P; ++p) {
      const int64_t np = offsets[p + 1] - offsets[p];
      toff[p + 1] = toff[p] + (np + rv::kTcN - 1) / rv::kTcN * rv::kTcN;
    }
    // + one group of 8 padding rows after the last problem (K3-CT gathers it for padding)
    RV_CUDA(ctx->tctab.ensure((size_t)(toff[P] + 8) * 64), "allocating K3-TC table");
    RV_CUDA(ctx->toffs.ensure(P + 1), "allocating offsets");
    if (dev_offsets) {
      // (written by the caller, see above)
    } else {
      int64_t* ht = ctx->up.take<int64_t>(P + 1);  // staging sized for it above
      std::memcpy(ht, toff.data(), (P + 1) * sizeof(int64_t));
      RV_CUDA(cudaMemcpyAsync(ctx->toffs.p, ht, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
              "copying offsets");
    }
    // the culled levels' rows: K3-CT's fp16-split row-major copy, or K3-C's fp32 rows (the
    // culled path cull_prepare will pick: K3-CT unless RV_CULL_TC=0 or a multi-rank batch)
    const bool ct = cull_rows && ctx->cull_on && ctx->cull_tc;
    const bool k3c = cull_rows && ctx->cull_on && !ct;
    if (k3c) RV_CUDA(ctx->k12.ensure((size_t)(toff[P] + 8) * 12), "allocating K3-C rows");
    if (ct) RV_CUDA(ctx->tctab_rm.ensure((size_t)(toff[P] + 8) * 64), "allocating K3-CT rows");
    rv::K9Out k9o;
    if (fused) k9o = rv::K9Out{ctx->k9.p, ctx->stride, total, ctx->bad.p};
    rv::launch_setup_tc(x, y, ctx->rows.p, ctx->toffs.p, P, toff[P] + 8, ctx->tctab.p, ctx->stream,
                        k3c ? ctx->k12.p : nullptr, ct ? ctx->tctab_rm.p : nullptr, k9o);
    ctx->launches += 1;
    ctx->tc_toff = toff;
  }
  RV_CUDA(cudaGetLastError(), "launching rv_setup");
  return RV_OK;
}

int check_bad(rv_ctx* ctx) {
  unsigned long long b = 0;
  RV_CUDA(cudaMemcpyAsync(&b, ctx->bad.p, sizeof(b), cudaMemcpyDeviceToHost, ctx->stream),
          "reading data flag");
  RV_SYNC(cudaStreamSynchronize(ctx->stream), "rv_setup");
  if (b != ~0ull)
    return ctx->fail(RV_EDATA, "correspondence row %llu has a zero-length or non-finite vector", b);
  return RV_OK;
}

// ---- refinement (K6/K7) for P problems --------------------------------------------------------
// qs0: HOST [P][4] start rotations; writes q/flags/ninl (HOST) and masks (DEVICE, optional).
int run_refine(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
               const int32_t* prob_ids /* which problems (indices into offsets) */, double eps,
               const double* qs0, int32_t rounds, const int64_t* mask_words, uint32_t* masks,
               double* q_out, int32_t* flags_out, uint32_t* ninl_out) {
  std::vector<rv::RefSeg> segs(P);
  std::vector<rv::RefItem> items;
  const double tau = std::cos(eps);
  for (int32_t s = 0; s < P; ++s) {
    const int32_t p = prob_ids ? prob_ids[s] : s;
    const int64_t n = offsets[p + 1] - offsets[p];
    segs[s].row = offsets[p];
    segs[s].mask_word = mask_words ? mask_words[s] : 0;
    segs[s].n = (int32_t)n;
    segs[s].tau = tau;
    segs[s].pad = 0;
    segs[s].item_begin = (int32_t)items.size();
    for (int64_t r0 = 0; r0 < n; r0 += rv::kRefRowsPerItem)
      items.push_back({s, (int32_t)r0, (int32_t)std::min<int64_t>(rv::kRefRowsPerItem, n - r0)});
    segs[s].item_end = (int32_t)items.size();
  }
  RV_CUDA(ctx->rsegs.ensure(P), "allocating");
  RV_CUDA(ctx->ritems.ensure(items.size()), "allocating");
  RV_CUDA(ctx->partials.ensure(items.size() * 10), "allocating");
  RV_CUDA(ctx->qs.ensure((size_t)P * 4), "allocating");
  RV_CUDA(ctx->flags.ensure(P), "allocating");
  RV_CUDA(ctx->ninl.ensure(P), "allocating");
  RV_CUDA(ctx->up.ensure(P * sizeof(rv::RefSeg) + items.size() * sizeof(rv::RefItem) + P * 32 + 4096),
          "allocating staging");
  RV_CUDA(ctx->down.ensure(P * (32 + 8) + 4096), "allocating staging");
  ctx->up.reset();
  rv::RefSeg* hs = ctx->up.take<rv::RefSeg>(P);
  std::memcpy(hs, segs.data(), P * sizeof(rv::RefSeg));
  rv::RefItem* hi = ctx->up.take<rv::RefItem>(items.size());
  std::memcpy(hi, items.data(), items.size() * sizeof(rv::RefItem));
  double* hq = ctx->up.take<double>((size_t)P * 4);
  std::memcpy(hq, qs0, (size_t)P * 4 * sizeof(double));
  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaMemcpyAsync(ctx->rsegs.p, hs, P * sizeof(rv::RefSeg), cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->ritems.p, hi, items.size() * sizeof(rv::RefItem),
                          cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->qs.p, hq, (size_t)P * 32, cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemsetAsync(ctx->flags.p, 0, P * sizeof(int32_t), s), "memset");
  for (int r = 0; r < rounds; ++r) {
    rv::launch_inliers(x, y, ctx->rsegs.p, ctx->ritems.p, (int32_t)items.size(), ctx->qs.p, nullptr,
                       ctx->partials.p, s);
    rv::launch_eig(ctx->rsegs.p, P, ctx->partials.p, ctx->qs.p, ctx->flags.p, ctx->ninl.p, 0, s);
  }
  rv::launch_inliers(x, y, ctx->rsegs.p, ctx->ritems.p, (int32_t)items.size(), ctx->qs.p, masks,
                     ctx->partials.p, s);
  rv::launch_eig(ctx->rsegs.p, P, ctx->partials.p, ctx->qs.p, ctx->flags.p, ctx->ninl.p, 1, s);
  ctx->launches += 2 * rounds + 2;
  RV_CUDA(cudaGetLastError(), "launching refinement");
  ctx->down.reset();
  double* dq = ctx->down.take<double>((size_t)P * 4);
  int32_t* df = ctx->down.take<int32_t>(P);
  uint32_t* dn = ctx->down.take<uint32_t>(P);
  RV_CUDA(cudaMemcpyAsync(dq, ctx->qs.p, (size_t)P * 32, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(df, ctx->flags.p, P * 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(dn, ctx->ninl.p, P * 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_SYNC(cudaStreamSynchronize(s), "refinement");
  std::memcpy(q_out, dq, (size_t)P * 32);
  for (int32_t p = 0; p < P; ++p) flags_out[p] = df[p] & (RV_REFINED | RV_DEGENERATE);
  std::memcpy(ninl_out, dn, P * 4);
  return RV_OK;
}

// The refinement of P problems enqueued without a wait: q0 already in ctx->qs (device), the
// segment / item tables through ctx->up2 and the outputs into ctx->down (pinned; valid after the
// caller's next wait).  Same launches and arithmetic as run_refine.
int enqueue_refine(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
                   double eps, int32_t rounds, const int64_t* mask_words, uint32_t* masks,
                   RefineOut& out) {
  std::vector<rv::RefSeg> segs(P);
  std::vector<rv::RefItem> items;
  const double tau = std::cos(eps);
  for (int32_t p = 0; p < P; ++p) {
    const int64_t n = offsets[p + 1] - offsets[p];
    segs[p].row = offsets[p];
    segs[p].mask_word = mask_words ? mask_words[p] : 0;
    segs[p].n = (int32_t)n;
    segs[p].tau = tau;
    segs[p].pad = 0;
    segs[p].item_begin = (int32_t)items.size();
    for (int64_t r0 = 0; r0 < n; r0 += rv::kRefRowsPerItem)
      items.push_back({p, (int32_t)r0, (int32_t)std::min<int64_t>(rv::kRefRowsPerItem, n - r0)});
    segs[p].item_end = (int32_t)items.size();
  }
  RV_CUDA(ctx->rsegs.ensure(P), "allocating");
  RV_CUDA(ctx->ritems.ensure(items.size()), "allocating");
  RV_CUDA(ctx->partials.ensure(items.size() * 10), "allocating");
  RV_CUDA(ctx->flags.ensure(P), "allocating");
  RV_CUDA(ctx->ninl.ensure(P), "allocating");
  RV_CUDA(ctx->up2.ensure(P * sizeof(rv::RefSeg) + items.size() * sizeof(rv::RefItem) + 4096),
          "allocating staging");
  RV_CUDA(ctx->down.ensure(P * (32 + 8) + 4096), "allocating staging");
  ctx->up2.reset();
  rv::RefSeg* hs = ctx->up2.take<rv::RefSeg>(P);
  std::memcpy(hs, segs.data(), P * sizeof(rv::RefSeg));
  rv::RefItem* hi = ctx->up2.take<rv::RefItem>(items.size());
  std::memcpy(hi, items.data(), items.size() * sizeof(rv::RefItem));
  cudaStream_t s = ctx->stream;
  RV_CUDA(cudaMemcpyAsync(ctx->rsegs.p, hs, P * sizeof(rv::RefSeg), cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemcpyAsync(ctx->ritems.p, hi, items.size() * sizeof(rv::RefItem),
                          cudaMemcpyHostToDevice, s), "H2D");
  RV_CUDA(cudaMemsetAsync(ctx->flags.p, 0, P * sizeof(int32_t), s), "memset");
  for (int r = 0; r < rounds; ++r) {
    rv::launch_inliers(x, y, ctx->rsegs.p, ctx->ritems.p, (int32_t)items.size(), ctx->qs.p, nullptr,
                       ctx->partials.p, s);
    rv::launch_eig(ctx->rsegs.p, P, ctx->partials.p, ctx->qs.p, ctx->flags.p, ctx->ninl.p, 0, s);
  }
  rv::launch_inliers(x, y, ctx->rsegs.p, ctx->ritems.p, (int32_t)items.size(), ctx->qs.p, masks,
                     ctx->partials.p, s);
  rv::launch_eig(ctx->rsegs.p, P, ctx->partials.p, ctx->qs.p, ctx->flags.p, ctx->ninl.p, 1, s);
  ctx->launches += 2 * rounds + 2;
  RV_CUDA(cudaGetLastError(), "launching refinement");
  ctx->down.reset();
  out.q = ctx->down.take<double>((size_t)P * 4);
  out.flags = ctx->down.take<int32_t>(P);
  out.ninl = ctx->down.take<uint32_t>(P);
  RV_CUDA(cudaMemcpyAsync(out.q, ctx->qs.p, (size_t)P * 32, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(out.flags, ctx->flags.p, P * 4, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(out.ninl, ctx->ninl.p, P * 4, cudaMemcpyDeviceToHost, s), "D2H");
  return RV_OK;
}

}  // namespace rvi
