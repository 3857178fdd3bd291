// rv_vote_tc.cu -- K3-TC: the vote contraction on the 5th-generation tensor cores (tcgen05).
//
// SURVEY §8(f) NEXT-1.  For a CTA of 128 cells and a stream of 256-correspondence tiles the
// scores S'[c][i] = phi(q_c) . k_i - t_c are one (128 x 32) . (32 x 256) fp16 MMA with fp32
// accumulation, split so the products stay fp32-grade:
//   k   = k_hi + k_lo,  phi = phi_hi + phi_lo  (fp16 each),
//   S' ~= k_hi.phi_hi + k_hi.phi_lo + k_lo.phi_hi + 1.(-t_hi) + 1.(-t_lo)
// laid out along K = 32:  A row (cell) = [phi_hi | phi_lo | phi_hi | -t_hi, -t_lo, -1, 0, 0]
//                         B row (corr) = [k_hi   | k_hi   | k_lo   |  1,     1,    p, 0, 0]
// with p = 0 for a correspondence and p = 1 for a padding row (S' = -1: never counted).
// The count is then the sign bit of the accumulator, read from TMEM by the epilogue warps
// (tcgen05.ld 32x32b: TMEM lane = cell, column = correspondence), so the SM's integer pipes do
// one instruction per pair instead of the FP32 pipe's 9-FMA contraction.
//
// Two kernels per vote: K2-TC writes the A operand of every distinct block of <= 128 cells
// (8 KB each, fp64 cell rotation + threshold, one thread per row; a block shared by several
// problems -- the level-0 grid of a batch -- is built once), then the persistent vote kernel,
// one CTA per SM looping over work items.  CTA roles: warp 0 lane 0 = TMA producer (per item
// its A block into one of two A buffers, then one 16 KB cp.async.bulk per correspondence tile
// into a ring of kTcStages), warp 1 = TMEM allocator + single-thread MMA issuer
// (2 x tcgen05.mma K=16 per tile, accumulators double-buffered in 2 x 256 TMEM columns),
// warps 2..9 = epilogue (warp w reads TMEM lanes 32*(w%4).. (its cells); the two warps of a
// lane quarter take alternate tiles -- accumulator 0 / 1 -- so one warp's TMEM loads overlap
// the other's count -- and counts sign bits).
// Completion flows through mbarriers: full[s] / afull[a] (TMA tx), empty[s] / aempty[a]
// (tcgen05.commit), tfull[b] (tcgen05.commit), tempty[b] (the 8 epilogue warps).
#include <cstdint>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/rotvote.h"
#include "rv_geom.h"
#include "rv_kernels.h"
#include "rv_tc_ptx.h"

namespace rv {

namespace {

using namespace tcx;  // mbarriers, bulk copies, descriptors, tcgen05 (rv_tc_ptx.h)

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate) {
  mma_f16_n<kTcN>(d_tmem, adesc, bdesc, accumulate);
}
#define RV_LD32 RV_TCX_LD32

// Sign-bit counting on two pipes: acc += bits >> 31 fuses to LEA.HI (ALU pipe);
// acc += hi32(bits * 2) is IMAD.HI (FMA pipe) when the 2 is a runtime register.
// (volatile: tcgen05.ld destinations may only be read after tcgen05.wait::ld, so the counts
// must not be hoisted above it)
__device__ __forceinline__ void add_sign_alu(uint32_t& acc, uint32_t bits) {
  asm volatile("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(bits >> 31));
}
__device__ __forceinline__ void add_sign_fma(uint32_t& acc, uint32_t bits, uint32_t two) {
#if RV_TC_COUNT_ALU_ONLY
  (void)two;
  asm volatile("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(bits >> 31));
#else
  asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(bits), "r"(two));
#endif
}

// byte offset of element (row, col) in the interleaved K-major layout of 32 fp16 columns:
// 8-row groups of 512 B, each holding four 8x(8 fp16) core matrices of 128 B.
__device__ __forceinline__ uint32_t il_off(int row, int col) {
  return (uint32_t)((row >> 3) * 512 + (col >> 3) * 128 + (row & 7) * 16 + (col & 7) * 2);
}

}  // namespace

// ------------------------------------------------------------------------------------------
// K1-TC: the fp16-split correspondence table, 64 B per correspondence, interleaved layout,
// each problem padded to a multiple of kTcN rows (padding rows score -1).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rv_setup_tc_kernel(const float* __restrict__ x,
                                                          const float* __restrict__ y,
                                                          const int64_t* __restrict__ rows,
                                                          const int64_t* __restrict__ toffs,
                                                          int32_t P, int64_t total_pad,
                                                          uint8_t* __restrict__ tab,
                                                          float* __restrict__ k12,
                                                          uint8_t* __restrict__ tab_rm,
                                                          K9Out k9o) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total_pad;
       g += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = P;
    while (hi - lo > 1) {
      int32_t mid = (lo + hi) >> 1;
      if (toffs[mid] <= g) lo = mid; else hi = mid;
    }
    const int64_t i = g - toffs[lo];
    const int64_t n = rows[lo + 1] - rows[lo];
    __half v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = __float2half_rn(0.0f);
    if (i < n) {
      const int64_t r = rows[lo] + i;
      double a[3] = {x[3 * r], x[3 * r + 1], x[3 * r + 2]};
      double b[3] = {y[3 * r], y[3 * r + 1], y[3 * r + 2]};
      double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      double nb = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
      if (k9o.k9 && (!(na > 0.0) || !(nb > 0.0) || !isfinite(na) || !isfinite(nb))) {
        atomicMin(k9o.bad, (unsigned long long)r);  // K1's data check (one problem)
        na = nb = 1.0;
      }
      const double ia = 1.0 / na, ib = 1.0 / nb;
#pragma unroll
      for (int c = 0; c < 3; ++c) { a[c] *= ia; b[c] *= ib; }
      double k[9];
      k9_of(a, b, k);
      if (k9o.k9)  // K1's fp32 table of the one problem (K1 fused: x, y read once)
#pragma unroll
        for (int j = 0; j < 9; ++j) k9o.k9[j * k9o.stride + g] = (float)k[j];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const __half h = __double2half(k[j]);
        const __half l = __double2half(k[j] - (double)__half2float(h));
        v[j] = h;
        v[9 + j] = h;
        v[18 + j] = l;
      }
      v[27] = __float2half_rn(1.0f);
      v[28] = __float2half_rn(1.0f);
      if (k12) {  // the culled vote's rows: K1's fp64 -> fp32 rounding
        float4* kr = reinterpret_cast<float4*>(k12 + g * 12);
        kr[0] = make_float4((float)k[0], (float)k[1], (float)k[2], (float)k[3]);
        kr[1] = make_float4((float)k[4], (float)k[5], (float)k[6], (float)k[7]);
        kr[2] = make_float4((float)k[8], 0.0f, 0.0f, 0.0f);
      }
    } else {
      if (k9o.k9 && g < k9o.n_pad)  // K1's zero padding (s = 0 for every q)
#pragma unroll
        for (int j = 0; j < 9; ++j) k9o.k9[j * k9o.stride + g] = 0.0f;
      v[29] = __float2half_rn(1.0f);  // padding row: S' = -1
      if (k12) {
        float4* kr = reinterpret_cast<float4*>(k12 + g * 12);
        kr[0] = kr[1] = kr[2] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    }
    // row g of the whole table: group g>>3, 4 chunks of 16 B (+ the row-major copy K3-CT
    // gathers: a row's 64 B contiguous, two whole 32-byte sectors)
    uint8_t* rowp = tab + (g >> 3) * 512 + (g & 7) * 16;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      uint4 w;
      __half* hw = reinterpret_cast<__half*>(&w);
#pragma unroll
      for (int e = 0; e < 8; ++e) hw[e] = v[ch * 8 + e];
      *reinterpret_cast<uint4*>(rowp + ch * 128) = w;
      if (tab_rm) *reinterpret_cast<uint4*>(tab_rm + g * 64 + ch * 16) = w;
    }
  }
}

void launch_setup_tc(const float* x, const float* y, const int64_t* rows, const int64_t* toffs,
                     int32_t P, int64_t total_pad, uint8_t* tab, cudaStream_t s, float* k12,
                     uint8_t* tab_rm, const K9Out& k9o) {
  int64_t blocks = (total_pad + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  rv_setup_tc_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, y, rows, toffs, P, total_pad, tab, k12,
                                                       tab_rm, k9o);
}

// ------------------------------------------------------------------------------------------
// K3-TC
// ------------------------------------------------------------------------------------------
#ifndef RV_TC_EPI_WARPS
#define RV_TC_EPI_WARPS 8
#endif
#ifndef RV_TC_PINGPONG
#define RV_TC_PINGPONG 1  // the two warps of a lane quarter take alternate tiles (0: split columns)
#endif
constexpr int kTcEpiWarps = RV_TC_EPI_WARPS;  // multiple of 4 (one lane quarter per SMSP)
[[maybe_unused]] constexpr int kTcSplit = kTcEpiWarps / 4;  // warps per lane quarter
#ifndef RV_TC_ABUFS
#define RV_TC_ABUFS 2
#endif
constexpr int kTcABufs = RV_TC_ABUFS;  // A-operand buffers (items of lookahead for its TMA)
// Warp roles: an SMSP's issue arbiter prefers the highest warp id among its eligible warps, so
// the two issuing warps (their loops answer the pipeline's barriers) take the highest ids and the
// epilogue warps the lowest (RV_TC_ROLES=0: the old order, producer 0 / MMA 1 / epilogue 2.., A/B)
#ifndef RV_TC_ROLES
#define RV_TC_ROLES 1
#endif
constexpr int kTcEpi0 = RV_TC_ROLES ? 0 : 2;                      // first epilogue warp
constexpr int kTcProdW = RV_TC_ROLES ? RV_TC_EPI_WARPS : 0;       // the TMA producer
constexpr int kTcMmaW = kTcProdW + 1;                             // the MMA issuer
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;  // producer, MMA, epilogue warps
constexpr int kTcAccCols = kTcAcc * kTcN;  // = 512: the whole TMEM
constexpr uint32_t kTileBytes = kTcN * 64;  // 16 KB at N = 256

static_assert(!RV_TC_PINGPONG || (kTcAcc == 2 && kTcEpiWarps == 8),
              "ping-pong epilogue: two accumulators, one warp pair per TMEM lane quarter");
static_assert(RV_TC_PINGPONG || kTcN == 256, "bitmask emission needs the ping-pong epilogue");

struct __align__(1024) TcSmem {
  uint8_t b[kTcStages][kTileBytes];  // correspondence tiles
  uint8_t a[kTcABufs][128 * 64];     // A operand (128 rows x 32 fp16), kTcABufs buffers
  uint64_t full[kTcStages], empty[kTcStages], tfull[kTcAcc], tempty[kTcAcc], afull[kTcABufs],
      aempty[kTcABufs];
  uint32_t tmem_base;
};

// K2-TC: the A operand of every ABlock -- per row (cell, or cell x threshold in FIN mode)
// [phi_hi | phi_lo | phi_hi | -t_hi, -t_lo, -1, 0, 0] in the interleaved K-major layout, one
// thread per row.  Rows past the block's cells are zero (they score 0 and are not counted).
template <bool FIN>
__global__ void __launch_bounds__(128) rv_tc_atab_kernel(const VoteSeg* __restrict__ segs,
                                                         const ABlock* __restrict__ ablocks,
                                                         int32_t n_ablocks,
                                                         const int32_t* __restrict__ counts_dev,
                                                         float guard, uint8_t* __restrict__ atab) {
  const int32_t nab = counts_dev ? counts_dev[1] : n_ablocks;
  for (int32_t bi = blockIdx.x; bi < nab; bi += gridDim.x) {
  const ABlock ab = ablocks[bi];
  const VoteSeg& sg = segs[ab.seg];
  const int m = threadIdx.x;  // A row
  const int cell = FIN ? (m >> 1) : m;
  __half v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = __float2half_rn(0.0f);
  if (cell < ab.ncell) {
    const uint32_t lin = sg.lins[ab.cell0 + cell];
    int32_t i, j, k;
    lin_to_ijk(lin, sg.B, i, j, k);
    double q[4], f[9];
    cell_quat(sg.B, i, j, k, q);
    phi9(q, f);
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const __half h = __double2half(f[t]);
      const __half l = __double2half(f[t] - (double)__half2float(h));
      v[t] = h;
      v[9 + t] = l;
      v[18 + t] = h;
    }
    const double thr = FIN ? cos(sg.eps) + ((m & 1) ? guard : -guard)
                           : bound_threshold(sg.B, i, j, k, sg.eps) - guard;
    const __half th = __double2half(-thr);
    const __half tl = __double2half(-thr - (double)__half2float(th));
    v[27] = th;
    v[28] = tl;
    v[29] = __float2half_rn(-1.0f);
  }
  uint8_t* blk = atab + (int64_t)bi * kTcABlockBytes;
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint4 w;
    __half* hw = reinterpret_cast<__half*>(&w);
#pragma unroll
    for (int e = 0; e < 8; ++e) hw[e] = v[ch * 8 + e];
    *reinterpret_cast<uint4*>(blk + il_off(m, ch * 8)) = w;
  }
  }
}

// Persistent: CTA b processes items b, b + gridDim.x, ...; every role walks the same item
// sequence, and the tile / accumulator / A-buffer rings run on across item boundaries, so the
// prologue (TMEM allocation, barriers) is paid once per SM instead of once per item.
//   warp 0 lane 0   TMA producer: per item its 8 KB A block (K2-TC table) into the free A
//                   buffer, then one 16 KB cp.async.bulk per correspondence tile
//   warp 1 lane 0   MMA issuer: 2 x tcgen05.mma K=16 per tile into accumulator gt % 2
//   warps 2..9      epilogue: tcgen05.ld the accumulator, count sign bits, one atomic per
//                   (cell, item)
// FIN: RV_MODE_FINAL -- two A rows per cell (TMEM lanes 2c, 2c+1) carry the thresholds
//      tau - g' (cnt_a) and tau + g' (cnt_b), so an item covers kTcM/2 cells.
// ABL (ablation, tuning only): bit0 skip the count, bit1 skip the MMAs, bit2 skip the TMA
// BITS: also write each cell's pass bitmask (seg.bits, ancestor culling, rv_cull.cu): bit e of
//       word (i0 + 256 t) / 32 + 4 rr + q = score >= 0 for that column
template <bool DUMP, int ABL = 0, bool FIN = false, bool BITS = false>
__global__ void __launch_bounds__(kTcThreads, 1)
    rv_vote_tc_kernel(const uint8_t* __restrict__ tab, const uint8_t* __restrict__ atab,
                      const VoteSeg* __restrict__ segs, const VoteItem* __restrict__ items,
                      int32_t n_items_host, const int32_t* __restrict__ counts_dev, float guard,
                      float* dump, int64_t dump_ld) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int32_t n_items =
      counts_dev ? __shfl_sync(0xffffffffu, counts_dev[0], 0) : n_items_host;  // (warp-uniform)
  TcSmem& sm = *reinterpret_cast<TcSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue (once per CTA): TMEM, barriers ----
  if (warp == kTcMmaW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&sm.tmem_base)),
                 "r"(kTcAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      bar_init(&sm.full[s], 1);
      bar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < kTcAcc; ++b) {
      bar_init(&sm.tfull[b], 1);
      bar_init(&sm.tempty[b], RV_TC_PINGPONG ? kTcEpiWarps / 2 : kTcEpiWarps);
    }
    for (int b = 0; b < kTcABufs; ++b) {
      bar_init(&sm.afull[b], 1);
      bar_init(&sm.aempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  // The two issuing warps walk their loops whole, with warp-uniform values (item fields broadcast
  // from lane 0), and one elected lane issues: the bulk-copy and tcgen05 operands then live in
  // uniform registers.  (Issued from inside `if (lane == 0)`, ptxas moved every operand through
  // an ELECT / R2UR loop per instruction: ~90 dependent instructions per tile in the MMA warp.)
  if (warp == kTcProdW) {
    // ---------------- TMA producer ----------------
    uint32_t gt = 0, gi = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++gi) {
      const VoteItem it = items[idx];
      const int it_ablk = __shfl_sync(0xffffffffu, it.ablk, 0);
      const int it_ni = __shfl_sync(0xffffffffu, it.ni, 0);
      const int64_t row0 = __shfl_sync(0xffffffffu, segs[it.seg].koff + it.i0, 0);
      const uint32_t ab = gi % kTcABufs;
      if (gi >= (uint32_t)kTcABufs) bar_wait(&sm.aempty[ab], ((gi / kTcABufs) - 1) & 1);
      if (elect_one()) {
        bar_expect_tx(&sm.afull[ab], (uint32_t)kTcABlockBytes);
        bulk_g2s(sm.a[ab], atab + (int64_t)it_ablk * kTcABlockBytes, (uint32_t)kTcABlockBytes,
                 &sm.afull[ab]);
      }
      __syncwarp();
      const uint8_t* src = tab + row0 * 64;
      const int ntiles = it_ni / kTcN;  // it.i0, it.ni are multiples of kTcN
      for (int t = 0; t < ntiles; ++t, ++gt) {
        const uint32_t s = gt % kTcStages;
        if (gt >= (uint32_t)kTcStages) bar_wait(&sm.empty[s], ((gt / kTcStages) - 1) & 1);
        if (elect_one()) {
          if (ABL & 4) {
            bar_arrive(&sm.full[s]);
          } else {
            bar_expect_tx(&sm.full[s], kTileBytes);
            bulk_g2s(sm.b[s], src + (int64_t)t * kTileBytes, kTileBytes, &sm.full[s]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kTcMmaW) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t dhi = smem_desc_hi(512);
    const uint32_t blo0 = smem_desc_lo(su32(sm.b[0]), 128);
    const uint32_t alo0 = smem_desc_lo(su32(sm.a[0]), 128);
    uint32_t gt = 0, gi = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++gi) {
      const int ntiles = __shfl_sync(0xffffffffu, items[idx].ni, 0) / kTcN;
      const uint32_t ab = gi % kTcABufs;
      bar_wait(&sm.afull[ab], (gi / kTcABufs) & 1);
      const uint32_t alo = alo0 + ab * (uint32_t)(sizeof(sm.a[0]) >> 4);
      for (int t = 0; t < ntiles; ++t, ++gt) {
        const uint32_t s = gt % kTcStages, b = gt % kTcAcc;
        bar_wait(&sm.full[s], (gt / kTcStages) & 1);
        if (gt >= (uint32_t)kTcAcc) bar_wait(&sm.tempty[b], ((gt / kTcAcc) - 1) & 1);
        tc_fence_after();
        const uint32_t blo = blo0 + s * (uint32_t)(sizeof(sm.b[0]) >> 4);
        if (elect_one()) {
          if (!(ABL & 2)) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
              mma_f16(tmem + b * kTcN, desc64(alo + 16 * k, dhi), desc64(blo + 16 * k, dhi),
                      (uint32_t)k);
          }
          mma_commit(&sm.empty[s]);  // smem slot free once these MMAs completed
          mma_commit(&sm.tfull[b]);  // accumulator b ready
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&sm.aempty[ab]);  // A buffer free once the item's MMAs completed
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: count sign bits (warps 2..9) ----------------
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const int half = (warp - kTcEpi0) >> 2;     // accumulator (ping-pong) / column half
    const int m = 32 * (warp & 3) + lane;       // TMEM lane = A row
    const int cell = FIN ? (m >> 1) : m;
    const uint32_t two = guard > -1.0f ? 2u : 3u;  // a runtime 2 (keeps IMAD.HI)
    uint32_t gt = 0;
#if RV_TC_PINGPONG
    // the warp pair (w, w + 4) of a lane quarter takes alternate tiles: warp half h counts the
    // tiles in accumulator h (all 256 columns, two rounds of 128), so one warp's TMEM loads
    // overlap the other warp's count
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const VoteItem it = items[idx];
      const int ntiles = it.ni / kTcN;
      uint32_t n0 = 0, n1 = 0, n2 = 0, n3 = 0, n4 = 0, n5 = 0, n6 = 0, n7 = 0, mine = 0;
      // BITS: this cell's bitmask row for the item's columns (hoisted out of the tile loop)
      uint32_t* brow = nullptr;
      if (BITS && cell < it.ncell) {
        const VoteSeg& sg = segs[it.seg];
        brow = sg.bits + (int64_t)(it.cell0 + cell) * sg.wpc + (it.i0 >> 5);
      }
      // this warp's tiles of the item: global tile index g = gt + t with g % 2 == half
      const uint32_t acc_addr = lane_addr + (uint32_t)(half * kTcN);
      for (int t = (half - (int)(gt & 1)) & 1; t < ntiles; t += 2) {
        const uint32_t g = gt + (uint32_t)t;
        bar_wait(&sm.tfull[half], (g >> 1) & 1);
        tc_fence_after();
        ++mine;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          uint32_t r[4][32];
#pragma unroll
          for (int q = 0; q < 4; ++q) RV_LD32(r[q], acc_addr + (uint32_t)(rr * 128 + 32 * q));
          tmem_wait_ld();
          if (rr == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.tempty[half]);
          }
          if (BITS) {
            // sign bits -> one word per 32 columns (shf funnel: w = w << 1 | sign, column 31
            // first, so bit e = column e); count = columns - negatives; store the pass words
            uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int e = 31; e >= 0; --e)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                asm volatile("shf.l.clamp.b32 %0, %1, %0, 1;" : "+r"(w[q]) : "r"(r[q][e]));
            n0 += __popc(w[0]);
            n1 += __popc(w[1]);
            n2 += __popc(w[2]);
            n3 += __popc(w[3]);
            if (brow)
              *reinterpret_cast<uint4*>(brow + t * (kTcN >> 5) + rr * 4) =
                  make_uint4(~w[0], ~w[1], ~w[2], ~w[3]);
          } else if (DUMP) {
            if (cell < it.ncell) {
              float* drow = dump + (int64_t)(it.cell0 + cell) * dump_ld + it.i0 + (int64_t)t * kTcN + rr * 128;
#pragma unroll
              for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int e = 0; e < 32; ++e) drow[32 * q + e] = __uint_as_float(r[q][e]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int e = 0; e < 32; e += 8) {
                add_sign_alu(n0, r[q][e]);
                add_sign_fma(n1, r[q][e + 1], two);
                add_sign_alu(n2, r[q][e + 2]);
                add_sign_fma(n3, r[q][e + 3], two);
                add_sign_alu(n4, r[q][e + 4]);
                add_sign_fma(n5, r[q][e + 5], two);
                add_sign_alu(n6, r[q][e + 6]);
                add_sign_fma(n7, r[q][e + 7], two);
              }
          }
        }
      }
      gt += (uint32_t)ntiles;
      if (!DUMP && cell < it.ncell && mine > 0) {
        const VoteSeg& sg = segs[it.seg];
        const uint32_t neg = (n0 + n1) + (n2 + n3) + (n4 + n5) + (n6 + n7);
        const uint32_t cnt = mine * (uint32_t)kTcN - neg;  // its tiles' columns
        atomicAdd(FIN && (m & 1) ? &sg.cnt_b[it.cell0 + cell] : &sg.cnt_a[it.cell0 + cell], cnt);
      }
    }
#else
    constexpr int kLd = kTcN / kTcSplit / 32;  // tcgen05.ld x32 per warp per tile
    const int col0 = half * (kTcN / kTcSplit);
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const VoteItem it = items[idx];
      const int ntiles = it.ni / kTcN;
      uint32_t n0 = 0, n1 = 0, n2 = 0, n3 = 0, n4 = 0, n5 = 0, n6 = 0, n7 = 0;
      for (int t = 0; t < ntiles; ++t, ++gt) {
        const uint32_t b = gt % kTcAcc;
        bar_wait(&sm.tfull[b], (gt / kTcAcc) & 1);
        tc_fence_after();
        // this warp's part of accumulator b -> registers, then hand the buffer back to the
        // MMA issuer before counting (the count overlaps the next MMAs)
        uint32_t r[kLd][32];
#pragma unroll
        for (int q = 0; q < kLd; ++q) RV_LD32(r[q], lane_addr + (uint32_t)(b * kTcN + col0 + 32 * q));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(&sm.tempty[b]);
        if (ABL & 1) {
          n0 += r[0][0] ^ r[kLd - 1][31];
        } else if (DUMP) {
          if (cell < it.ncell) {
            float* drow = dump + (int64_t)(it.cell0 + cell) * dump_ld + it.i0 + (int64_t)t * kTcN + col0;
#pragma unroll
            for (int q = 0; q < kLd; ++q)
#pragma unroll
              for (int e = 0; e < 32; ++e) drow[32 * q + e] = __uint_as_float(r[q][e]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < kLd; ++q)
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              add_sign_alu(n0, r[q][e]);
              add_sign_fma(n1, r[q][e + 1], two);
              add_sign_alu(n2, r[q][e + 2]);
              add_sign_fma(n3, r[q][e + 3], two);
              add_sign_alu(n4, r[q][e + 4]);
              add_sign_fma(n5, r[q][e + 5], two);
              add_sign_alu(n6, r[q][e + 6]);
              add_sign_fma(n7, r[q][e + 7], two);
            }
        }
      }
      if (!DUMP && cell < it.ncell) {
        // rows of the chunk: real correspondences score phi.k - t; padding rows score -1
        const VoteSeg& sg = segs[it.seg];
        const uint32_t neg = (n0 + n1) + (n2 + n3) + (n4 + n5) + (n6 + n7);
        const uint32_t cnt = (uint32_t)(it.ni / kTcSplit) - neg;  // its share of the columns
        atomicAdd(FIN && (m & 1) ? &sg.cnt_b[it.cell0 + cell] : &sg.cnt_a[it.cell0 + cell], cnt);
      }
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTcMmaW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTcAccCols));
  }
}

size_t tc_smem_bytes() { return sizeof(TcSmem) + 1024; }

void launch_vote_tc(const uint8_t* tab, uint8_t* atab, const ABlock* ablocks, int32_t n_ablocks,
                    const VoteSeg* segs, const VoteItem* items, int32_t n_items, float guard,
                    float* dump, int64_t dump_ld, cudaStream_t s, bool final_mode,
                    const int32_t* counts_dev, bool emit_bits) {
  if (!counts_dev && (n_items <= 0 || n_ablocks <= 0)) return;
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  const int agrid = counts_dev ? sms * 8 : n_ablocks;
  if (final_mode)
    rv_tc_atab_kernel<true><<<agrid, 128, 0, s>>>(segs, ablocks, n_ablocks, counts_dev, guard, atab);
  else
    rv_tc_atab_kernel<false><<<agrid, 128, 0, s>>>(segs, ablocks, n_ablocks, counts_dev, guard, atab);
  // persistent: one CTA per SM
  const int grid = counts_dev ? sms : (n_items < sms ? n_items : sms);
  static std::atomic<uint64_t> attr_done{0};
  if (first_launch_on_device(attr_done)) {
    cudaFuncSetAttribute(rv_vote_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tc_smem_bytes());
    cudaFuncSetAttribute(rv_vote_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tc_smem_bytes());
    cudaFuncSetAttribute(rv_vote_tc_kernel<false, 0, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes());
    cudaFuncSetAttribute(rv_vote_tc_kernel<false, 0, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes());
    mark_device_done(attr_done);
  }
  if (emit_bits && !final_mode && !dump) {
    rv_vote_tc_kernel<false, 0, false, true><<<grid, kTcThreads, tc_smem_bytes(), s>>>(
        tab, atab, segs, items, n_items, counts_dev, guard, nullptr, 0);
    return;
  }
  if (final_mode) {
    rv_vote_tc_kernel<false, 0, true><<<grid, kTcThreads, tc_smem_bytes(), s>>>(
        tab, atab, segs, items, n_items, counts_dev, guard, nullptr, 0);
    return;
  }
  // tuning builds only (-DRV_TC_ABLATE=1..7 skips pipeline stages: WRONG counts); the product
  // library is compiled without it
#ifdef RV_TC_ABLATE
  constexpr int abl = RV_TC_ABLATE;
#else
  constexpr int abl = 0;
#endif
  if (dump)
    rv_vote_tc_kernel<true><<<grid, kTcThreads, tc_smem_bytes(), s>>>(tab, atab, segs, items,
                                                                         n_items, counts_dev, guard, dump, dump_ld);
  else if (abl != 0) {
#define RV_ABL_CASE(A)                                                                           \
  case A:                                                                                        \
    cudaFuncSetAttribute(rv_vote_tc_kernel<false, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)tc_smem_bytes());                                                  \
    rv_vote_tc_kernel<false, A><<<grid, kTcThreads, tc_smem_bytes(), s>>>(tab, atab, segs, items, \
                                                                 n_items, counts_dev, guard, nullptr, 0);    \
    break;
    switch (abl) { RV_ABL_CASE(1) RV_ABL_CASE(2) RV_ABL_CASE(3) RV_ABL_CASE(4) RV_ABL_CASE(5)
                   RV_ABL_CASE(6) RV_ABL_CASE(7) default: break; }
#undef RV_ABL_CASE
  } else
    rv_vote_tc_kernel<false><<<grid, kTcThreads, tc_smem_bytes(), s>>>(tab, atab, segs, items,
                                                                          n_items, counts_dev, guard, nullptr, 0);
}

}  // namespace rv
