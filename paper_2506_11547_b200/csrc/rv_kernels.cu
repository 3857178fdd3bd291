// rv_kernels.cu -- librotvote's hand-written sm_100a kernels.
//
//   K1 rv_setup    a1  normalise + 9-entry traceless quadratic form K_i (fp64 -> fp32 SoA)
//   K3 rv_vote     a3  (cells x 9)·(9 x N) contraction on the FP32 pipe (FFMA2), thresholded
//                      and counted in registers; K tiles staged in shared memory by the TMA
//                      bulk-copy engine (cp.async.bulk + mbarrier), reused by 1024 blocks
//   K5 rv_exact    a5  exact count: fp32 vote + fp64 recheck inside the guard band
//   K6 rv_inliers  a6  fp64 inlier test, ballot -> mask words, partial sums of K over inliers
//   K7 rv_eig      a6  fixed-order reduction + 4x4 cyclic Jacobi (fp64), top eigenvector
//
// Citations: P:n = PAPER.md line n.  The vote statistic s_i(q) = y^T R(q) x = q^T K_i q
// (Appendix A) with K_i traceless, so 9 numbers per correspondence suffice:
//   s = phi(q) . k,  phi = [q0²-q3², q1²-q3², q2²-q3², 2q0q1, 2q0q2, 2q0q3, 2q1q2, 2q1q3, 2q2q3].
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "../../include/rotvote.h"
#include "rv_geom.h"
#include "rv_kernels.h"

namespace rv {

// ------------------------------------------------------------------------------------------
// K1 setup
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rv_setup_kernel(const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       const int64_t* __restrict__ rows,
                                                       const int64_t* __restrict__ koffs,
                                                       int32_t P, int64_t total_pad,
                                                       float* __restrict__ k9, int64_t stride,
                                                       unsigned long long* bad) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total_pad;
       g += (int64_t)gridDim.x * blockDim.x) {
    // problem containing padded index g (binary search over koffs)
    int32_t lo = 0, hi = P;
    while (hi - lo > 1) {
      int32_t mid = (lo + hi) >> 1;
      if (koffs[mid] <= g) lo = mid; else hi = mid;
    }
    const int64_t i = g - koffs[lo];
    const int64_t n = rows[lo + 1] - rows[lo];
    double k[9];
    if (i < n) {
      const int64_t r = rows[lo] + i;
      double a[3] = {x[3 * r], x[3 * r + 1], x[3 * r + 2]};
      double b[3] = {y[3 * r], y[3 * r + 1], y[3 * r + 2]};
      double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      double nb = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
      if (!(na > 0.0) || !(nb > 0.0) || !isfinite(na) || !isfinite(nb)) {
        atomicMin(bad, (unsigned long long)r);
        na = nb = 1.0;
      }
      const double ia = 1.0 / na, ib = 1.0 / nb;
#pragma unroll
      for (int c = 0; c < 3; ++c) { a[c] *= ia; b[c] *= ib; }
      k9_of(a, b, k);
    } else {
#pragma unroll
      for (int j = 0; j < 9; ++j) k[j] = 0.0;  // padding: s = 0 for every q
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) k9[j * stride + g] = (float)k[j];
  }
}

void launch_setup(const float* x, const float* y, const int64_t* rows, const int64_t* koffs,
                  int32_t P, int64_t total_pad, float* k9, int64_t stride,
                  unsigned long long* bad, cudaStream_t s) {
  int64_t blocks = (total_pad + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  rv_setup_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, y, rows, koffs, P, total_pad, k9, stride,
                                                   bad);
}

// ------------------------------------------------------------------------------------------
// TMA bulk-copy + mbarrier helpers (PTX, sm_90+ / sm_100a)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ uint32_t sign_bit(float v) { return __float_as_uint(v) >> 31; }

// ------------------------------------------------------------------------------------------
// K3 vote
// ------------------------------------------------------------------------------------------
// Warp-specialised CTA: warps 0..7 vote, warp 8 is the TMA producer.  Each voting thread owns
// kCellsPerThread blocks (cells): phi(q_c) and the threshold live in registers; one FFMA2
// (scalar-broadcast phi operand) evaluates a cell against two correspondences.  The voters
// form G groups; group g handles the 4-correspondence chunks g, g+G, ... of every tile, so a
// CTA covers 1024/G cells (G > 1 keeps the thread slots full when a level has few cells).
// K tiles (9 rows x kTile correspondences) arrive by cp.async.bulk into a kStages ring with
// full/empty mbarriers; voters never block one another.  The threshold is folded into the
// FMA chain's initial value, the count is the sign bit (cnt = processed - #negatives), and
// the counts leave the CTA with one atomicAdd per cell.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// acc += sign bit of v; an opaque add keeps NVVM from re-associating the running sum into a
// tree whose last add lands on the FMA pipe (IMAD); ptxas fuses shift+add into LEA.HI (ALU).
__device__ __forceinline__ void add_sign(uint32_t& acc, float v) {
  asm("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(__float_as_uint(v) >> 31));
}

template <int MODE, int G>
__global__ void __launch_bounds__(kVoteThreads + kProducerThreads, kVoteMinBlocks)
    rv_vote_kernel(const float* __restrict__ k9, int64_t stride, const VoteSeg* __restrict__ segs,
                   const VoteItem* __restrict__ items, float guard) {
  constexpr int TPG = kVoteThreads / G;               // voting threads per group
  constexpr int CPB = TPG * kCellsPerThread;          // cells per CTA
  __shared__ __align__(128) float sK[kStages][9][kTile];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  static_assert(2 * kVoteThreads * kCellsPerThread <= kStages * 9 * kTile, "red aliases sK");
  uint32_t* red = reinterpret_cast<uint32_t*>(&sK[0][0][0]);  // epilogue only (G > 1)

  const VoteItem it = items[blockIdx.x];
  const VoteSeg& sg = segs[it.seg];
  const int tid = threadIdx.x;
  const int ntiles = (it.ni + kTile - 1) / kTile;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kVoteThreads / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const float* kbase = k9 + sg.koff + it.i0;
  auto issue = [&](int t) {  // TMA bulk copies of tile t (9 rows) into stage t % kStages
    const int st = t % kStages;
    const int cnt = min(kTile, it.ni - t * kTile);
    const uint32_t bytes = (uint32_t)cnt * 4u;
    mbar_expect_tx(&full[st], bytes * 9u);
#pragma unroll
    for (int j = 0; j < 9; ++j)
      tma_bulk_g2s(&sK[st][j][0], kbase + j * stride + (int64_t)t * kTile, bytes, &full[st]);
  };

  // ---------------- producer (RV_PIPE == 1: a dedicated warp) ----------------
  if (kProducerThreads > 0 && tid >= kVoteThreads) {
    if (tid == kVoteThreads)
      for (int t = 0; t < ntiles; ++t) {
        if (t >= kStages) mbar_wait(&empty[t % kStages], (uint32_t)(((t / kStages) - 1) & 1));
        issue(t);
      }
  }
  if (kProducerThreads == 0 && tid == 0)
    for (int t = 0; t < kStages && t < ntiles; ++t) issue(t);

  // ---------------- voters ----------------
  const int g = tid / TPG;           // group of this voter
  const int local = tid % TPG;
  const bool voter = tid < kVoteThreads;
  float phi[kCellsPerThread][9];
  float init[kCellsPerThread];
  uint32_t neg_a[kCellsPerThread], neg_b[kCellsPerThread];
  const float two_g = 2.0f * guard;
  {
    const int32_t B = sg.B;
    const double tau = cos(sg.eps);
#pragma unroll
    for (int c = 0; c < kCellsPerThread; ++c) {
      int e = local + c * TPG;
      if (e >= it.ncell || !voter) e = 0;  // inactive slot: recompute cell 0, never stored
      const uint32_t lin = sg.lins[it.cell0 + e];
      int32_t i, j, k;
      lin_to_ijk(lin, B, i, j, k);
      double q[4], f[9];
      cell_quat(B, i, j, k, q);
      phi9(q, f);
#pragma unroll
      for (int t = 0; t < 9; ++t) phi[c][t] = (float)f[t];
      double thr = (MODE == RV_MODE_BOUND) ? bound_threshold(B, i, j, k, sg.eps) - guard
                                           : tau - guard;
      init[c] = (float)(-thr);
      neg_a[c] = neg_b[c] = 0;
    }
  }
  if (voter) {
    const int lane = tid & 31;
    for (int t = 0; t < ntiles; ++t) {
      const int st = t % kStages;
      mbar_wait(&full[st], (uint32_t)((t / kStages) & 1));
      const int cnt = min(kTile, it.ni - t * kTile);
      const float* sk = &sK[st][0][0];
#pragma unroll 1
      for (int i = 4 * g; i < cnt; i += 4 * G) {
        float4 kk[9];
#pragma unroll
        for (int j = 0; j < 9; ++j) kk[j] = *reinterpret_cast<const float4*>(sk + j * kTile + i);
#pragma unroll
        for (int c = 0; c < kCellsPerThread; ++c) {
          const float2 i2 = make_float2(init[c], init[c]);
          float2 lo = i2, hi = i2;
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            const float2 f2 = make_float2(phi[c][j], phi[c][j]);
            lo = __ffma2_rn(f2, make_float2(kk[j].x, kk[j].y), lo);
            hi = __ffma2_rn(f2, make_float2(kk[j].z, kk[j].w), hi);
          }
#if RV_COUNT_ASM
          add_sign(neg_a[c], lo.x);
          add_sign(neg_a[c], lo.y);
          add_sign(neg_a[c], hi.x);
          add_sign(neg_a[c], hi.y);
          if (MODE == RV_MODE_FINAL) {
            add_sign(neg_b[c], lo.x - two_g);
            add_sign(neg_b[c], lo.y - two_g);
            add_sign(neg_b[c], hi.x - two_g);
            add_sign(neg_b[c], hi.y - two_g);
          }
#else
          neg_a[c] += sign_bit(lo.x) + sign_bit(lo.y) + sign_bit(hi.x) + sign_bit(hi.y);
          if (MODE == RV_MODE_FINAL)
            neg_b[c] += sign_bit(lo.x - two_g) + sign_bit(lo.y - two_g) + sign_bit(hi.x - two_g) +
                        sign_bit(hi.y - two_g);
#endif
        }
      }
      if (kProducerThreads > 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      } else {
        __syncthreads();  // stage st fully consumed by every voter
        if (tid == 0 && t + kStages < ntiles) issue(t + kStages);
      }
    }
  }

  // epilogue: counts = processed - negatives - zero-padding rows that counted as >= 0
  const int valid = max(0, min(it.ni, sg.n - it.i0));
  const uint32_t pad = (uint32_t)(it.ni - valid);
  if (G == 1) {
    if (tid < kVoteThreads) {
#pragma unroll
      for (int c = 0; c < kCellsPerThread; ++c) {
        const int e = local + c * TPG;
        if (e >= it.ncell) continue;
        uint32_t ca = (uint32_t)it.ni - neg_a[c] - (sign_bit(init[c]) ? 0u : pad);
        atomicAdd(&sg.cnt_a[it.cell0 + e], ca);
        if (MODE == RV_MODE_FINAL) {
          uint32_t cb = (uint32_t)it.ni - neg_b[c] - (sign_bit(init[c] - two_g) ? 0u : pad);
          atomicAdd(&sg.cnt_b[it.cell0 + e], cb);
        }
      }
    }
  } else {
    __syncthreads();  // every tile consumed: sK is free to hold the per-group partial counts
    if (tid < kVoteThreads) {
#pragma unroll
      for (int c = 0; c < kCellsPerThread; ++c) {
        const int e = local + c * TPG;
        red[g * CPB + e] = neg_a[c];
        if (MODE == RV_MODE_FINAL) red[G * CPB + g * CPB + e] = neg_b[c];
      }
    }
    __syncthreads();
    if (tid < TPG) {
#pragma unroll
      for (int c = 0; c < kCellsPerThread; ++c) {
        const int e = local + c * TPG;
        if (e >= it.ncell) continue;
        uint32_t na = 0, nb = 0;
#pragma unroll
        for (int q = 0; q < G; ++q) {
          na += red[q * CPB + e];
          if (MODE == RV_MODE_FINAL) nb += red[G * CPB + q * CPB + e];
        }
        uint32_t ca = (uint32_t)it.ni - na - (sign_bit(init[c]) ? 0u : pad);
        atomicAdd(&sg.cnt_a[it.cell0 + e], ca);
        if (MODE == RV_MODE_FINAL) {
          uint32_t cb = (uint32_t)it.ni - nb - (sign_bit(init[c] - two_g) ? 0u : pad);
          atomicAdd(&sg.cnt_b[it.cell0 + e], cb);
        }
      }
    }
  }
}

template <int MODE, int G>
static void launch_vote_t(const float* k9, int64_t stride, const VoteSeg* segs,
                          const VoteItem* items, int32_t n_items, float guard, cudaStream_t s) {
  rv_vote_kernel<MODE, G><<<n_items, kVoteThreads + kProducerThreads, 0, s>>>(k9, stride, segs,
                                                                             items, guard);
}

void launch_vote(int mode, int groups, const float* k9, int64_t stride, const VoteSeg* segs,
                 const VoteItem* items, int32_t n_items, float guard, cudaStream_t s) {
  if (n_items <= 0) return;
  if (mode == RV_MODE_BOUND) {
    if (groups == 4) launch_vote_t<RV_MODE_BOUND, 4>(k9, stride, segs, items, n_items, guard, s);
    else if (groups == 2) launch_vote_t<RV_MODE_BOUND, 2>(k9, stride, segs, items, n_items, guard, s);
    else launch_vote_t<RV_MODE_BOUND, 1>(k9, stride, segs, items, n_items, guard, s);
  } else {
    if (groups == 4) launch_vote_t<RV_MODE_FINAL, 4>(k9, stride, segs, items, n_items, guard, s);
    else if (groups == 2) launch_vote_t<RV_MODE_FINAL, 2>(k9, stride, segs, items, n_items, guard, s);
    else launch_vote_t<RV_MODE_FINAL, 1>(k9, stride, segs, items, n_items, guard, s);
  }
}

// ------------------------------------------------------------------------------------------
// K5 exact count
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 2) rv_exact_kernel(const float* __restrict__ k9,
                                                       int64_t stride,
                                                       const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       const VoteSeg* __restrict__ segs,
                                                       const VoteItem* __restrict__ items,
                                                       int32_t n_items,
                                                       const int32_t* __restrict__ n_dev,
                                                       float guard) {
  // n_dev: the item count lives on the device (device-built items; fixed grid)
  // An item is up to kExactCells blocks x a range of correspondences: each correspondence's K
  // row is read once for all of them (the final level's few blocks used to re-stream the table
  // once per block).
  const int32_t n = n_dev ? *n_dev : n_items;
  __shared__ float sf32[kExactCells][9];
  __shared__ double sf64[kExactCells][9];
  __shared__ uint32_t ws[kExactCells][8];
  __shared__ double s_tau;
  for (int32_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
  const VoteItem it = items[idx];
  const VoteSeg& sg = segs[it.seg];
  const int nc = it.ncell < 1 ? 1 : (it.ncell > kExactCells ? kExactCells : it.ncell);
  if (threadIdx.x == 32) s_tau = cos(sg.eps);
  if ((int)threadIdx.x < nc) {
    const uint32_t lin = sg.lins[it.cell0 + threadIdx.x];
    int32_t ci, cj, ck;
    lin_to_ijk(lin, sg.B, ci, cj, ck);
    double q[4], f64[9];
    cell_quat(sg.B, ci, cj, ck, q);
    phi9(q, f64);
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      sf64[threadIdx.x][t] = f64[t];
      sf32[threadIdx.x][t] = (float)f64[t];
    }
  }
  __syncthreads();
  const double tau_it = s_tau;
  const float init = (float)(-tau_it);

  uint32_t cnt[kExactCells];
#pragma unroll
  for (int c = 0; c < kExactCells; ++c) cnt[c] = 0u;
  const int end = min(it.i0 + it.ni, sg.n);
  for (int i = it.i0 + threadIdx.x; i < end; i += blockDim.x) {
    float kv[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) kv[t] = k9[t * stride + sg.koff + i];
    uint32_t near = 0u;  // blocks whose fp32 score is inside the guard band
#pragma unroll
    for (int c = 0; c < kExactCells; ++c) {
      if (c < nc) {
        float s = init;
#pragma unroll
        for (int t = 0; t < 9; ++t) s = fmaf(sf32[c][t], kv[t], s);
        if (fabsf(s) < guard) near |= 1u << c;
        else cnt[c] += s >= 0.0f ? 1u : 0u;
      }
    }
    if (near) {  // decide those in fp64 from the raw inputs
      const int64_t r = sg.row + i;
      double a[3] = {x[3 * r], x[3 * r + 1], x[3 * r + 2]};
      double b[3] = {y[3 * r], y[3 * r + 1], y[3 * r + 2]};
      const double ia = 1.0 / sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      const double ib = 1.0 / sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
#pragma unroll
      for (int u = 0; u < 3; ++u) { a[u] *= ia; b[u] *= ib; }
      double k[9];
      k9_of(a, b, k);
      uint32_t pass = 0u;
#pragma unroll 1
      for (int c = 0; c < kExactCells; ++c) {
        if (!(near >> c & 1u)) continue;
        double s64 = 0.0;
#pragma unroll
        for (int t = 0; t < 9; ++t) s64 = fma(sf64[c][t], k[t], s64);
        pass |= (s64 >= tau_it ? 1u : 0u) << c;
      }
#pragma unroll
      for (int c = 0; c < kExactCells; ++c) cnt[c] += pass >> c & 1u;  // (cnt stays in registers)
    }
  }
  // block reduction per block of the item
#pragma unroll
  for (int c = 0; c < kExactCells; ++c) {
    uint32_t v = cnt[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ws[c][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < nc) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[threadIdx.x][w];
    atomicAdd(&sg.cnt_a[it.cell0 + threadIdx.x], t);
  }
  __syncthreads();  // ws / sf* are rewritten by the next item
  }
}

void launch_exact(const float* k9, int64_t stride, const float* x, const float* y,
                  const VoteSeg* segs, const VoteItem* items, int32_t n_items, float guard,
                  cudaStream_t s, const int32_t* n_dev) {
  if (n_dev) {
    rv_exact_kernel<<<148 * 8, 256, 0, s>>>(k9, stride, x, y, segs, items, 0, n_dev, guard);
    return;
  }
  if (n_items <= 0) return;
  rv_exact_kernel<<<n_items, 256, 0, s>>>(k9, stride, x, y, segs, items, n_items, nullptr, guard);
}

// ------------------------------------------------------------------------------------------
// K6 inliers + partial sums
// ------------------------------------------------------------------------------------------
// K_i of row r in fp64 from the raw fp32 row (normalised in fp64), one compiled copy shared by
// K6 and the fused refinement so both produce the same bits
__device__ __noinline__ void ref_row_k(const float* __restrict__ x, const float* __restrict__ y,
                                       int64_t r, double k[9]) {
  double a[3] = {x[3 * r], x[3 * r + 1], x[3 * r + 2]};
  double b[3] = {y[3 * r], y[3 * r + 1], y[3 * r + 2]};
  const double ia = 1.0 / sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
  const double ib = 1.0 / sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
#pragma unroll
  for (int c = 0; c < 3; ++c) { a[c] *= ia; b[c] *= ib; }
  k9_of(a, b, k);
}

__global__ void __launch_bounds__(kRefThreads) rv_inliers_kernel(
    const float* __restrict__ x, const float* __restrict__ y, const RefSeg* __restrict__ segs,
    const RefItem* __restrict__ items, const double* __restrict__ qs, uint32_t* masks,
    double* __restrict__ partials) {
  const RefItem it = items[blockIdx.x];
  const RefSeg& sg = segs[it.seg];
  double q[4] = {qs[4 * it.seg], qs[4 * it.seg + 1], qs[4 * it.seg + 2], qs[4 * it.seg + 3]};
  double f[9];
  phi9(q, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.0;
  const int end = it.r0 + it.nr;
  for (int base = it.r0 + warp * 32; base < end; base += kRefThreads) {
    const int i = base + lane;
    bool in = false;
    double k[9];
    if (i < end && i < sg.n) {
      ref_row_k(x, y, sg.row + i, k);
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 9; ++t) s = fma(f[t], k[t], s);
      in = s >= sg.tau;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    if (masks && lane == 0 && base < sg.n) masks[sg.mask_word + (base >> 5)] = bal;
    if (in) {
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[t] += k[t];
      acc[9] += 1.0;
    }
  }
  // fixed-order reduction: warp butterfly, then warps in order
#pragma unroll
  for (int t = 0; t < 10; ++t)
    for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_down_sync(0xffffffffu, acc[t], o);
  __shared__ double ws[kRefThreads / 32][10];
  if (lane == 0)
#pragma unroll
    for (int t = 0; t < 10; ++t) ws[warp][t] = acc[t];
  __syncthreads();
  if (threadIdx.x < 10) {
    double s = 0.0;
    for (int w = 0; w < kRefThreads / 32; ++w) s += ws[w][threadIdx.x];
    partials[(int64_t)blockIdx.x * 10 + threadIdx.x] = s;
  }
}

void launch_inliers(const float* x, const float* y, const RefSeg* segs, const RefItem* items,
                    int32_t n_items, const double* qs, uint32_t* masks, double* partials,
                    cudaStream_t s) {
  if (n_items <= 0) return;
  rv_inliers_kernel<<<n_items, kRefThreads, 0, s>>>(x, y, segs, items, qs, masks, partials);
}

// ------------------------------------------------------------------------------------------
// K7 reduction + 4x4 symmetric eigen-solver (cyclic Jacobi, fp64)
// ------------------------------------------------------------------------------------------
constexpr int32_t kStop = 1 << 8;  // internal: a round failed, later rounds keep q

// Jacobi rotation (p, q) of A (similarity) and V (accumulated), given c, s
__device__ __forceinline__ void jrot(double A[4][4], double V[4][4], int p, int q, double c,
                                     double s) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double akp = A[k][p], akq = A[k][q];
    A[k][p] = c * akp - s * akq;
    A[k][q] = s * akp + c * akq;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double apk = A[p][k], aqk = A[q][k];
    A[p][k] = c * apk - s * aqk;
    A[q][k] = s * apk + c * aqk;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double vkp = V[k][p], vkq = V[k][q];
    V[k][p] = c * vkp - s * vkq;
    V[k][q] = s * vkp + c * vkq;
  }
}
// rotation zeroing A[p][q]: tan(2 phi) = 2 apq / (aqq - app), t = tan phi in the stable form
// sign(d) apq / (|d| + sqrt(d^2 + apq^2)), d = (aqq - app) / 2 (one sqrt, one division)
__device__ __forceinline__ void jparams(double app, double aqq, double apq, double& c, double& s) {
  const double d = 0.5 * (aqq - app);
  const double t = copysign(1.0, d) * apq / (fabs(d) + sqrt(d * d + apq * apq));
  c = rsqrt(1.0 + t * t);
  s = t * c;
}

// 4x4 symmetric eigen-decomposition by Jacobi sweeps in the parallel (round-robin) order: each
// sweep is three rounds of two disjoint rotations, (0,1)(2,3), (0,2)(1,3), (0,3)(1,2), whose
// parameters are computed side by side (the serial solve's latency is the point: it runs on one
// thread between two grid-wide passes).  Stops when the off-diagonal mass is below 1e-32 of the
// diagonal's (relative 1e-16).
__device__ void jacobi4(double A[4][4], double V[4][4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) V[r][c] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, diag = 0.0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      diag += A[r][r] * A[r][r];
#pragma unroll
      for (int c = r + 1; c < 4; ++c) off += A[r][c] * A[r][c];
    }
    if (off == 0.0 || off <= 1e-32 * diag) break;
#pragma unroll
    for (int rd = 0; rd < 3; ++rd) {
      const int p1 = 0, q1 = rd + 1;                        // (0,1) (0,2) (0,3)
      const int p2 = rd == 0 ? 2 : 1, q2 = rd == 2 ? 2 : 3;  // (2,3) (1,3) (1,2)
      double c1 = 1.0, s1 = 0.0, c2 = 1.0, s2 = 0.0;
      const bool r1 = A[p1][q1] != 0.0, r2 = A[p2][q2] != 0.0;
      if (r1) jparams(A[p1][p1], A[q1][q1], A[p1][q1], c1, s1);
      if (r2) jparams(A[p2][p2], A[q2][q2], A[p2][q2], c2, s2);
      if (r1) jrot(A, V, p1, q1, c1, s1);
      if (r2) jrot(A, V, p2, q2, c2, s2);
    }
  }
}

// One refinement step from the inlier sums S (9 entries of sum K_i, count): flags | RV_REFINED and
// q <- the hemisphere-canonical top eigenvector, or flags | RV_DEGENERATE | kStop (fewer than 2
// inliers, or eigengap <= 1e-12 |lambda1|: q kept, later rounds skipped, reading R8)
__device__ __noinline__ int32_t eig_update(const double S[10], int32_t fl, double* q) {
  const double count = S[9];
  if (fl & kStop) return fl;
  if (count < 2.0) return fl | RV_DEGENERATE | kStop;
  // S = sum K_i over inliers; K33 = -(K00 + K11 + K22) by tracelessness
  double A[4][4] = {{S[0], S[3], S[4], S[5]},
                    {S[3], S[1], S[6], S[7]},
                    {S[4], S[6], S[2], S[8]},
                    {S[5], S[7], S[8], -(S[0] + S[1] + S[2])}};
  double V[4][4];
  jacobi4(A, V);
  // the largest eigenvalue and its column, selected with constant indices only (a dynamic
  // index would put A and V in local memory for the whole solve)
  double d[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) d[r] = A[r][r];
  int i0 = 0;
  double l1 = d[0];
#pragma unroll
  for (int r = 1; r < 4; ++r)
    if (d[r] > l1) { l1 = d[r]; i0 = r; }
  double l2 = -1e300;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (r != i0 && d[r] > l2) l2 = d[r];
  if (l1 - l2 <= 1e-12 * fabs(l1)) return fl | RV_DEGENERATE | kStop;
  double v[4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
    v[a] = i0 == 0 ? V[a][0] : i0 == 1 ? V[a][1] : i0 == 2 ? V[a][2] : V[a][3];
  const double nv = rsqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
  // hemisphere representative: q3 < 0; |q3| <= 1e-15 -> first nonzero of q0..q2 positive
  bool flip;
  if (v[3] * nv < -1e-15) flip = false;
  else if (v[3] * nv > 1e-15) flip = true;
  else {
    flip = false;
    for (int a = 0; a < 3; ++a)
      if (v[a] != 0.0) { flip = v[a] < 0.0; break; }
  }
  const double sgn = flip ? -nv : nv;
  for (int a = 0; a < 4; ++a) q[a] = v[a] * sgn;
  return fl | RV_REFINED;
}

// One warp per problem (8 per CTA; per_cta: one CTA per problem, for small batches, so the
// partials of a 1e6-row problem are summed by 256 threads): the lanes sum the problem's K6
// partials in a fixed order, lane 0 solves.
__global__ void __launch_bounds__(256) rv_eig_kernel(const RefSeg* __restrict__ segs,
                                                     const double* __restrict__ partials,
                                                     double* qs, int32_t* flags, uint32_t* ninl,
                                                     int mode, int32_t P, int per_cta) {
  const int lane = threadIdx.x & 31;
  const int p = per_cta ? blockIdx.x : blockIdx.x * 8 + (threadIdx.x >> 5);
  if (p >= P) return;
  const RefSeg& sg = segs[p];
  double S[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) S[t] = 0.0;
  const int t0 = per_cta ? (int)threadIdx.x : lane, tn = per_cta ? (int)blockDim.x : 32;
  for (int itm = sg.item_begin + t0; itm < sg.item_end; itm += tn)
#pragma unroll
    for (int t = 0; t < 10; ++t) S[t] += partials[(int64_t)itm * 10 + t];
#pragma unroll
  for (int t = 0; t < 10; ++t)
    for (int o = 16; o > 0; o >>= 1) S[t] += __shfl_down_sync(0xffffffffu, S[t], o);
  if (per_cta) {  // the warps' sums in warp order
    __shared__ double ws[8][10];
    if (lane == 0)
#pragma unroll
      for (int t = 0; t < 10; ++t) ws[threadIdx.x >> 5][t] = S[t];
    __syncthreads();
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += ws[w][t];
      S[t] = v;
    }
  } else if (lane != 0) {
    return;
  }
  const double count = S[9];
  if (mode == 1) {
    ninl[p] = (uint32_t)count;
    return;
  }
  flags[p] = eig_update(S, flags[p], qs + 4 * p);
}

void launch_eig(const RefSeg* segs, int32_t P, const double* partials, double* qs, int32_t* flags,
                uint32_t* ninl, int mode, cudaStream_t s) {
  if (P <= 0) return;
  if (P <= 148)
    rv_eig_kernel<<<P, 256, 0, s>>>(segs, partials, qs, flags, ninl, mode, P, 1);
  else
    rv_eig_kernel<<<(P + 7) / 8, 256, 0, s>>>(segs, partials, qs, flags, ninl, mode, P, 0);
}


// ------------------------------------------------------------------------------------------
// K6+K7 fused for ONE problem (the one-pass single solve): the rounds of R8 and the final mask in
// one cooperative launch (grid-wide barriers instead of launch boundaries).  q0 is the winner's
// block centre decoded on the device from the winner key (count << 32 | ~lin), so the solve needs
// no host round trip between the vote and the refinement.  The inlier test screens every row
// with the fp32 K table of K1 against cos(eps) -/+ guard (|s32 - s| <= 2.7e-6 < guard, DESIGN R10)
// and decides the rows inside the band in fp64 from x, y exactly as K6 does; the inliers' fp64
// K_i are summed in a fixed order (warp butterflies, CTA partials in block order).
// ------------------------------------------------------------------------------------------
#ifndef RV_R1_TRACE
#define RV_R1_TRACE 0  // tuning builds: %globaltimer stamps of CTA 0 (rv_r1_trace_copy)
#endif
#if RV_R1_TRACE
__device__ unsigned long long g_r1_trace[32];
__device__ __forceinline__ void r1_stamp(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x == 0 && threadIdx.x == 0 && k < 32) g_r1_trace[k] = t;
}
extern "C" int rv_r1_trace_copy(unsigned long long* h) {
  return (int)cudaMemcpyFromSymbol(h, g_r1_trace, sizeof(g_r1_trace));
}
#else
__device__ __forceinline__ void r1_stamp(int) {}
#endif
constexpr int kR1Threads = kRefThreads;  // K6's decomposition (see below)
static_assert(kRefRowsPerItem % kRefThreads == 0, "K6 items are whole rounds of rows");

// Grid-wide barrier of a cooperative launch (all CTAs co-resident): thread 0 of each CTA
// arrives on a counter and polls it with relaxed loads and a short sleep; one fence after.  (The
// cooperative-groups barrier polls with L1-invalidating acquire loads, and a CTA sharing its SM
// with the one doing the serial eigen step slowed that step ~5x.)
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    atomicAdd(bar, 1u);
    const uint32_t target = gen * gridDim.x;
    uint32_t v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v < target) __nanosleep(32);
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kR1Threads) rv_refine1_kernel(Refine1Args a) {
  uint32_t gen = 0;  // grid barriers passed (a.bar counts arrivals; zeroed before the launch)
  __shared__ double ws[kR1Threads / 32][10];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double q[4] = {0.0, 0.0, 0.0, -1.0};
    if (a.q0) {
      const double nq = sqrt(a.q0[0] * a.q0[0] + a.q0[1] * a.q0[1] + a.q0[2] * a.q0[2] +
                             a.q0[3] * a.q0[3]);
      for (int c = 0; c < 4; ++c) q[c] = a.q0[c] / nq;
    } else {
      const unsigned long long key = *a.best;
      if (key) {  // (no winner only when the solve was abandoned; the host redoes it)
        const uint32_t lin = 0xffffffffu - (uint32_t)(key & 0xffffffffull);
        int32_t i, j, k;
        lin_to_ijk(lin, a.B, i, j, k);
        cell_quat(a.B, i, j, k, q);
      }
    }
    bool flip;  // hemisphere representative (R9), as the host's canonicalize
    if (q[3] < -1e-15) flip = false;
    else if (q[3] > 1e-15) flip = true;
    else {
      flip = false;
      for (int c = 0; c < 3; ++c)
        if (q[c] != 0.0) { flip = q[c] < 0.0; break; }
    }
    for (int c = 0; c < 4; ++c) a.q[c] = flip ? -q[c] : q[c];
    *a.flags = 0;
  }
  r1_stamp(0);
  grid_barrier(a.bar, gen);
  r1_stamp(1);
  const float t_hi = (float)(a.tau + (double)a.guard), t_lo = (float)(a.tau - (double)a.guard);
  // K6's decomposition exactly (items of kRefRowsPerItem rows, warp w takes rows w*32 + lane +
  // 256 j of an item, per-item partials reduced as K6 does, summed as K7 does), so q, the mask
  // and the count are bit-identical to the K6 / K7 launches
  const int64_t n_items = (a.n + kRefRowsPerItem - 1) / kRefRowsPerItem;
  for (int r = 0; r <= a.rounds; ++r) {
    const bool last = r == a.rounds;
    double q[4];
    for (int c = 0; c < 4; ++c) q[c] = reinterpret_cast<volatile double*>(a.q)[c];
    double f[9];
    phi9(q, f);
    float f32[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) f32[t] = (float)f[t];
    for (int64_t itm = blockIdx.x; itm < n_items; itm += gridDim.x) {
      const int64_t r0 = itm * kRefRowsPerItem;
      const int64_t end = r0 + kRefRowsPerItem < a.n ? r0 + kRefRowsPerItem : a.n;
      double acc[10];
#pragma unroll
      for (int t = 0; t < 10; ++t) acc[t] = 0.0;
      // pass A: the fp32 screen of the thread's kRowsPT rows (rows r0 + warp*32 + lane + 256 j),
      // every K-table load issued up front; pass B: the decisions and the sums in K6's order
      constexpr int kRowsPT = kRefRowsPerItem / kR1Threads;
      float s32[kRowsPT];
#pragma unroll
      for (int jr = 0; jr < kRowsPT; ++jr) {
        const int64_t i = r0 + warp * 32 + lane + (int64_t)jr * kR1Threads;
        float v = 0.0f;
        if (i < end) {
#pragma unroll
          for (int t = 0; t < 9; ++t) v = fmaf(f32[t], __ldg(a.k9 + t * a.stride + i), v);
        }
        s32[jr] = v;
      }
#pragma unroll
      for (int jr = 0; jr < kRowsPT; ++jr) {
        const int64_t base = r0 + warp * 32 + (int64_t)jr * kR1Threads;
        if (base >= end) break;  // warp-uniform
        const int64_t i = base + lane;
        bool in = false, band = false;
        if (i < end) {
          in = s32[jr] >= t_hi;
          band = !in && s32[jr] >= t_lo;
        }
        double k[9];
        if (in || band) {  // fp64 K_i from the raw row (the sums, and the band's decision), as K6
          ref_row_k(a.x, a.y, i, k);
          if (band) {
            double sd = 0.0;
#pragma unroll
            for (int t = 0; t < 9; ++t) sd = fma(f[t], k[t], sd);
            in = sd >= a.tau;
          }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        if (last && a.mask && lane == 0) a.mask[base >> 5] = bal;
        if (in) {
#pragma unroll
          for (int t = 0; t < 9; ++t) acc[t] += k[t];
          acc[9] += 1.0;
        }
      }
#pragma unroll
      for (int t = 0; t < 10; ++t)
        for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_down_sync(0xffffffffu, acc[t], o);
      if (lane == 0)
#pragma unroll
        for (int t = 0; t < 10; ++t) ws[warp][t] = acc[t];
      __syncthreads();
      if (threadIdx.x < 10) {
        double v = 0.0;
        for (int w = 0; w < kR1Threads / 32; ++w) v += ws[w][threadIdx.x];
        __stcg(a.partials + itm * 10 + threadIdx.x, v);
      }
      __syncthreads();
    }
    r1_stamp(2 + 4 * r);
    grid_barrier(a.bar, gen);
    r1_stamp(3 + 4 * r);
    if (blockIdx.x == 0) {  // K7's per-CTA sum: thread t takes items t, t + 256, ...
      double S[10];
#pragma unroll
      for (int t = 0; t < 10; ++t) S[t] = 0.0;
      for (int64_t b = threadIdx.x; b < n_items; b += kR1Threads)
#pragma unroll
        for (int t = 0; t < 10; ++t) S[t] += __ldcg(a.partials + b * 10 + t);
      r1_stamp(16 + 4 * r);
#pragma unroll
      for (int t = 0; t < 10; ++t)
        for (int o = 16; o > 0; o >>= 1) S[t] += __shfl_down_sync(0xffffffffu, S[t], o);
      if (lane == 0)
#pragma unroll
        for (int t = 0; t < 10; ++t) ws[warp][t] = S[t];
      r1_stamp(17 + 4 * r);
      __syncthreads();
      r1_stamp(18 + 4 * r);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < 10; ++t) {
          double v = 0.0;
          for (int w = 0; w < kR1Threads / 32; ++w) v += ws[w][t];
          S[t] = v;
        }
        if (last) *a.ninl = (uint32_t)S[9];
        else *a.flags = eig_update(S, *a.flags, a.q);
      }
    }
    r1_stamp(4 + 4 * r);
    grid_barrier(a.bar, gen);
    r1_stamp(5 + 4 * r);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.flags &= (RV_REFINED | RV_DEGENERATE);
}

// the refinement's start of P problems: q0[p] = the hemisphere-canonical centre rotation of the
// winner packed in best[p] (count << 32 | ~lin) at resolution B (the host's canonical_cell_quat)
__global__ void rv_decode_q0_kernel(const unsigned long long* __restrict__ best, int32_t P,
                                    int32_t B, double* qs) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    double q[4] = {0.0, 0.0, 0.0, -1.0};
    const unsigned long long key = best[p];
    if (key) {
      const uint32_t lin = 0xffffffffu - (uint32_t)(key & 0xffffffffull);
      int32_t i, j, k;
      lin_to_ijk(lin, B, i, j, k);
      cell_quat(B, i, j, k, q);
    }
    bool flip;
    if (q[3] < -1e-15) flip = false;
    else if (q[3] > 1e-15) flip = true;
    else {
      flip = false;
      for (int c = 0; c < 3; ++c)
        if (q[c] != 0.0) { flip = q[c] < 0.0; break; }
    }
    for (int c = 0; c < 4; ++c) qs[4 * p + c] = flip ? -q[c] : q[c];
  }
}
void launch_decode_q0(const unsigned long long* best, int32_t P, int32_t B, double* qs,
                      cudaStream_t s) {
  rv_decode_q0_kernel<<<(P + 255) / 256, 256, 0, s>>>(best, P, B, qs);
}

// up to kSetMax int64 pairs into device memory in one launch (a one-pass solve's offset tables,
// carried by the kernel's arguments)
__global__ void rv_set_consts_kernel(SetList l) {
  const int t = threadIdx.x;
  if (t < l.n) {
    l.dst[t][0] = l.v0[t];
    l.dst[t][1] = l.v1[t];
  }
}
void launch_set_consts(const SetList& l, cudaStream_t s) {
  if (l.n > 0) rv_set_consts_kernel<<<1, 32, 0, s>>>(l);
}

// two int64 constants into device memory as a kernel (a one-pass solve's offsets: a captured
// graph then carries them in its kernel arguments instead of pointing at host staging)
__global__ void rv_set_i64x2_kernel(int64_t* d, int64_t v0, int64_t v1) {
  d[0] = v0;
  d[1] = v1;
}
void launch_set_i64x2(int64_t* d, int64_t v0, int64_t v1, cudaStream_t s) {
  rv_set_i64x2_kernel<<<1, 1, 0, s>>>(d, v0, v1);
}

cudaError_t launch_refine1(const Refine1Args& a, int num_sms, cudaStream_t s) {
  static int per_sm[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (per_sm[dev] == 0) {
    int b = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rv_refine1_kernel, kR1Threads, 0);
    if (e != cudaSuccess) return e;
    per_sm[dev] = b < 1 ? 1 : (b > 4 ? 4 : b);
  }
  const int grid = num_sms * per_sm[dev];
  if (grid > kRefine1MaxCtas) return cudaErrorInvalidConfiguration;
  Refine1Args args = a;
  cudaError_t e = cudaMemsetAsync(args.bar, 0, 4, s);
  if (e != cudaSuccess) return e;
  void* kargs[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)rv_refine1_kernel, dim3(grid), dim3(kR1Threads),
                                     kargs, 0, s);
}
}  // namespace rv

namespace rv {

// ------------------------------------------------------------------------------------------
// K4 (batched): level-0 reductions on the device, one CTA per problem.  cnt is [P][m0] (the
// level-0 UB counts of every problem against the shared candidate list lins[m0]).
// ------------------------------------------------------------------------------------------
// dive start: max excess UB - n*bg[e], blocks with their centre inside the ball first, ties ->
// lowest index (the same key, in the same double arithmetic, as the host planner)
__global__ void __launch_bounds__(256) rv_l0_argmax_kernel(const uint32_t* __restrict__ cnt,
                                                           int64_t m0,
                                                           const uint32_t* __restrict__ lins,
                                                           int32_t B, const double* __restrict__ bg,
                                                           const int64_t* __restrict__ rows,
                                                           int32_t* out, Excl ex) {
  const int p = blockIdx.x;
  const double n = (double)(rows[p + 1] - rows[p]);
  const uint32_t* c = cnt + (int64_t)p * m0;
  int best = -1, bin = 0;
  double bx = -1e300;
  for (int e = threadIdx.x; e < m0; e += blockDim.x) {
    // (NEXT-2: blocks away from the exclusion balls first)
    const int in = 2 * excl_rank(ex, B, lins[e]) + (centre_inside(B, lins[e]) ? 1 : 0);
    const double x = (double)c[e] - n * bg[e];
    if (best < 0 || in > bin || (in == bin && (x > bx || (x == bx && e < best)))) {
      best = e; bin = in; bx = x;
    }
  }
  __shared__ int sb[256], si[256];
  __shared__ double sx[256];
  sb[threadIdx.x] = best; si[threadIdx.x] = bin; sx[threadIdx.x] = bx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const int o = threadIdx.x + w;
      const int b2 = sb[o];
      if (b2 >= 0) {
        const int b1 = sb[threadIdx.x];
        const bool take = b1 < 0 || si[o] > si[threadIdx.x] ||
                          (si[o] == si[threadIdx.x] &&
                           (sx[o] > sx[threadIdx.x] || (sx[o] == sx[threadIdx.x] && b2 < b1)));
        if (take) { sb[threadIdx.x] = b2; si[threadIdx.x] = si[o]; sx[threadIdx.x] = sx[o]; }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[p] = sb[0];
}

// survivors (UB >= lb) of the listed problems: count pass (outc != nullptr) or compaction pass
// (ascending indices at out + off[j]); problems[j], lb[j] per listed problem j = blockIdx.x
__global__ void __launch_bounds__(256) rv_l0_survivors_kernel(const uint32_t* __restrict__ cnt,
                                                              int64_t m0,
                                                              const int32_t* __restrict__ problems,
                                                              const int64_t* __restrict__ lb,
                                                              const int64_t* __restrict__ off,
                                                              int32_t* outc, int32_t* out) {
  const int j = blockIdx.x;
  const uint32_t* c = cnt + (int64_t)problems[j] * m0;
  const int64_t L = lb[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int wsum[8];
  int base = 0;
  for (int64_t e0 = 0; e0 < m0; e0 += blockDim.x) {
    const int64_t e = e0 + threadIdx.x;
    const bool keep = e < m0 && (int64_t)c[e] >= L;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    if (out && keep) out[off[j] + base + before + __popc(bal & ((1u << lane) - 1u))] = (int32_t)e;
    base += total;
    __syncthreads();
  }
  if (outc && threadIdx.x == 0) outc[j] = base;
}

void launch_l0_argmax(const uint32_t* cnt, int64_t m0, const uint32_t* lins, int32_t B,
                      const double* bg, const int64_t* rows, int32_t P, int32_t* out,
                      cudaStream_t s, const Excl& ex) {
  if (P > 0) rv_l0_argmax_kernel<<<P, 256, 0, s>>>(cnt, m0, lins, B, bg, rows, out, ex);
}

void launch_l0_survivors(const uint32_t* cnt, int64_t m0, const int32_t* problems,
                         const int64_t* lb, const int64_t* off, int32_t J, int32_t* outc,
                         int32_t* out, cudaStream_t s) {
  if (J > 0)
    rv_l0_survivors_kernel<<<J, 256, 0, s>>>(cnt, m0, problems, lb, off, outc, out);
}

}  // namespace rv
