// rv_api.cpp -- the C-ABI of librotvote (include/rotvote.h): validation, workspace, the
// level loop that drives the host planner (rv_plan.cpp) with the sm_100a kernels
// (rv_kernels.cu), multi-GPU cell sharding over NCCL, refinement and result assembly.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>  // types only; the library is dlopen'ed (libnccl.so.2) when world > 1

#include "../../include/rotvote.h"
#include "../../include/rotvote_plan.h"
#include "rv_geom.h"
#include "rv_alg1.h"
#include "rv_dplan.h"
#include "rv_rigid.h"
#include "rv_kernels.h"

namespace {

const int32_t kDefaultChain[6] = {5, 15, 45, 90, 180, 360};
// Extra guard for K3-TC bound counts: worst-case |S'_tc - (s - t)| of the fp16-split MMA
// (split remainders <= 3 * 2^-22 * sum|k phi| <= 2.9e-6, threshold split 2.4e-7, fp32
// accumulation of 32 exact products <= 32 * 2^-24 * 5 = 9.5e-6) < 1.3e-5; measured 3.7e-7.
const float kTcExtraGuard = 1.5e-5f;

// ---- NCCL, loaded at run time -------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.AllReduce && a.CommDestroy &&
           a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

// ---- growable buffers ------------------------------------------------------------------------
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    size_t want = std::max<size_t>(n, cap * 3 / 2 + 64);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// pinned host staging used as a bump allocator within one synchronous step
struct Staging {
  char* p = nullptr;
  size_t cap = 0, used = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    size_t want = std::max<size_t>(n, cap * 3 / 2 + 4096);
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void reset() { used = 0; }
  template <class T>
  T* take(size_t n) {  // caller ensured capacity
    size_t off = (used + 255) & ~(size_t)255;
    used = off + n * sizeof(T);
    return reinterpret_cast<T*>(p + off);
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

inline int64_t pad4(int64_t n) { return (n + 3) & ~(int64_t)3; }

// RV_TRACE=1: host-side phase timings of batched solves on stderr (tuning aid)
struct Trace {
  bool on = getenv("RV_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[rv] %-28s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// Host-side parallel loop for the per-problem planner work of batched solves (planners are
// independent objects; each index is touched by exactly one thread).  RV_HOST_THREADS caps it.
template <class F>
void parallel_for(int64_t n, F f) {
  static const int hw = [] {
    int t = (int)std::thread::hardware_concurrency();
    if (const char* e = getenv("RV_HOST_THREADS")) t = atoi(e);
    return std::max(1, std::min(t, 32));
  }();
  const int T = (int)std::min<int64_t>(hw, (n + 63) / 64);
  if (T <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) f(i);
    });
  for (std::thread& x : th) x.join();
}

}  // namespace

struct rv_ctx {
  rv_config cfg{};
  std::vector<int32_t> chain;
  cudaStream_t stream = nullptr;
  std::string err;
  int num_sms = 148;
  int vote_blocks_per_sm = rv::kVoteMinBlocks;
#ifdef RV_VOTE_GROUPS
  int force_groups = RV_VOTE_GROUPS;  // tuning builds: force the FP32 K3 CTA shape (1|2|4)
#else
  int force_groups = 0;
#endif
  ncclComm_t comm = nullptr;

  DevBuf<float> k9;              // [9][stride]
  int64_t stride = 0;
  DevBuf<uint8_t> tctab;         // K3-TC table, 64 B per (padded) row
  DevBuf<uint8_t> tctab_rm;      // its rows row-major (K3-CT's gather source)
  DevBuf<int64_t> toffs;         // per-problem row offsets in tctab
  bool tc_on = false;            // cfg.tensor_vote: BOUND levels on tcgen05
  std::vector<int64_t> tc_toff;  // host copy of toffs for the current setup
  DevBuf<uint32_t> lins, cnt;    // request blocks, counts (gathered layout)
  DevBuf<rv::VoteSeg> vsegs;
  DevBuf<rv::VoteItem> vitems;
  DevBuf<rv::RefSeg> rsegs;
  DevBuf<rv::RefItem> ritems;
  DevBuf<double> partials, qs;
  DevBuf<int32_t> flags;
  DevBuf<uint32_t> ninl;
  DevBuf<int64_t> rows, koffs;
  DevBuf<unsigned long long> bad;
  DevBuf<float> hx, hy;          // device copies for rot_vote_solve_host
  DevBuf<uint32_t> hmask;
  DevBuf<char> gather;           // batched result all-gather
  DevBuf<uint32_t> grid_list;    // device copy of one grid's full candidate list (batched L0)
  DevBuf<uint32_t> l0cnt;        // batched level-0 counts kept on the device [P][m0]
  DevBuf<double> l0bg;           // device copy of the level-0 background table
  int32_t l0bg_B = 0;
  double l0bg_eps = 0;
  DevBuf<int32_t> l0idx;         // K4 outputs / survivor indices
  DevBuf<int64_t> l0aux;         // lb / offsets for K4
  int32_t grid_list_B = 0;
  int64_t grid_list_m = 0;
  std::vector<uint32_t> grid_host;  // candidate list of grid_host_B (host)
  int32_t grid_host_B = 0;
  // device-resident batched level loop (rv_dplan.cu): ping-pong block lists + counts, the
  // per-problem offsets/counts/picks/bounds, the recheck lists and the winners
  // sets 0 / 1: ping-pong level lists; set 2: the re-dive's lists
  DevBuf<uint32_t> dp_lins[3], dp_ca[3], dp_cb[3];
  DevBuf<int64_t> dp_off[3], dp_lb, dp_lb2, dp_actr[2], dp_bring[3];
  DevBuf<int32_t> dp_cnt[3], dp_rcnt, dp_ties, dp_rflag, dp_rany, dp_rdone;
  DevBuf<uint32_t> dp_pick, dp_rlins, dp_ex, dp_lmax;
  DevBuf<unsigned long long> dp_best;
  DevBuf<float> rg_m, rg_n;         // NEXT-3: kept pairs
  DevBuf<int32_t> rg_cnt;
  DevBuf<int64_t> rg_off, rg_bins;
  DevBuf<uint32_t> rg_acc;          // translation accumulator (zero between calls)
  int64_t rg_acc_m = 0;
  DevBuf<unsigned long long> rg_best;
  DevBuf<double> rg_sums;
  DevBuf<uint32_t> a1_acc;          // NEXT-4: the Algorithm-1 accumulator (B^3)
  DevBuf<double> a1_tab;            // cos / sin(alpha_j / 2)
  DevBuf<unsigned long long> a1_best;
  int32_t a1_J = 0;
  DevBuf<int64_t> dp_ioff, dp_aoff, dp_tot;
  DevBuf<int32_t> dp_icnt, dp_phase, dp_err, dp_pcnt, dp_scnt;
  DevBuf<int64_t> dp_poff, dp_sbase;
  // event pairs around the batched vote launches (read after the final sync)
  std::vector<cudaEvent_t> evs;
  size_t evn = 0;
  void ev_reset() { evn = 0; }
  cudaError_t ev_pair(cudaEvent_t* a, cudaEvent_t* b) {
    while (evs.size() < evn + 2) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      evs.push_back(e);
    }
    *a = evs[evn];
    *b = evs[evn + 1];
    evn += 2;
    return cudaSuccess;
  }
  void ev_collect() {
    for (size_t i = 0; i + 1 < evn; i += 2) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, evs[i], evs[i + 1]) == cudaSuccess) vote_ms += ms;
    }
    evn = 0;
  }
  // ancestor culling (rv_cull.cu): level-0 pass bitmasks, the K3-C rows, the level-0 lin ->
  // bitmask row table, the K3-C item planner's scratch, and its own event pairs
  bool cull_on = false;          // cfg.cull (with tensor_vote)
  bool cull_ready = false;       // this solve's level-0 bitmasks are written: levels >= 1 cull
  bool ct_prefetched = false;    // K3-CT's gather table was prefetched into L2 this solve
  int64_t cull_min_n = 0;        // cull only problems of >= this many correspondences (the
                                 // largest of a batch)
  int32_t cull_B0 = 0;
  int64_t cull_m0 = 0, cull_wpc_max = 0;
  DevBuf<uint32_t> cbits;        // level-0 pass bitmasks (K3-TC)
  DevBuf<int64_t> c_lofs;        // level-0 index lists: row offsets
  DevBuf<uint32_t> c_lidx;       //   and the lists
  DevBuf<int32_t> c_fill;        //   compaction fill counters
  const uint32_t* cull_l0cnt = nullptr;  // the level-0 counts (= list lengths) of this solve
  int64_t cull_own_lo = 0, cull_own_hi = INT64_MAX;  // level-0 rows a K3-C launch votes
  DevBuf<float> k12;
  DevBuf<int32_t> lut0;
  int32_t lut0_B = 0;
  // K3-CT ancestor groups (2 x 2 x 1 neighbouring level-0 blocks share one union list):
  // lutg = level-0 lin -> group, gmem[goff[g] .. goff[g+1]) = its level-0 rows
  DevBuf<int32_t> lutg, goff, gmem;
  int64_t cull_G = 0, cull_G_grouped = 0;
  bool cull_grouped = false;     // this solve's lists are group unions (K3-CT)
#ifndef RV_CT_NA
#define RV_CT_NA 1  // 2 (2x2x2 groups, M = 256 per gathered stage): measured slower, 1.12 vs 0.86 ms
#endif
  // K3-CT: items of up to cull_na x 128 block rows (one gathered stage feeds cull_na MMAs) over
  // the union lists of ancestor groups of cull_gshape level-0 blocks -- 2 x (2 x 2 x 2) by
  // default: up to 216 children of 8 ancestors at f = 3 share each gathered row
  int32_t cull_na = RV_CT_NA;
  int32_t cull_gshape[3] = {RV_CT_NA == 2 ? 2 : 1, 2, 2};  // ancestor group extent (i, j, k)
  // several ranks: level 0 is sliced at (i, j/2) row-pair boundaries (a group never straddles
  // two slices); rank r votes level-0 rows [cull_s[r], cull_s[r+1]) and owns the groups
  // [cull_g[r], cull_g[r+1]) (those whose first member is in its slice)
  std::vector<int64_t> cull_s, cull_g;
  DevBuf<int64_t> c_act, c_aoff, c_ioff;
  DevBuf<int32_t> c_acnt, c_tanc, c_tslot, c_cidx, c_icnt, c_work;
  DevBuf<float> c_phi;
  DevBuf<uint8_t> c_tphi;        // K3-CT block rows (fp16 split)
  bool cull_tc = true;           // culled levels on the tensor cores (K3-CT, group lists);
                                 // cfg.cull == 2: the FP32 K3-C on per-ancestor lists
  DevBuf<rv::CullItem> c_items;
  DevBuf<unsigned long long> c_pairs;
  std::vector<cudaEvent_t> cevs;
  size_t cevn = 0;
  cudaError_t cev_pair(cudaEvent_t* a, cudaEvent_t* b) {
    while (cevs.size() < cevn + 2) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      cevs.push_back(e);
    }
    *a = cevs[cevn];
    *b = cevs[cevn + 1];
    cevn += 2;
    return cudaSuccess;
  }
  void cev_collect() {
    for (size_t i = 0; i + 1 < cevn; i += 2) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, cevs[i], cevs[i + 1]) == cudaSuccess) cull_ms += ms;
    }
    cevn = 0;
  }
  DevBuf<int32_t> l0surv;        // host-planner batched path: level-0 survivor indices
  DevBuf<uint8_t> atab;          // K3-TC A-operand blocks (K2-TC)
  DevBuf<rv::ABlock> ablk;
  bool vote_pending = false;     // evv0/evv1 bracket a vote launch not yet accounted
  void collect_vote_ms() {
    if (!vote_pending) return;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, evv0, evv1) == cudaSuccess) vote_ms += ms;
    vote_pending = false;
  }
  Staging up, down;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evv0 = nullptr, evv1 = nullptr;
  // per-call counters reported in rv_result
  float vote_ms = 0, cull_ms = 0;
  uint64_t vote_pairs = 0, cull_pairs = 0;
  int32_t launches = 0, vote_launches = 0, cull_launches = 0, cull_tc_launches = 0;
  void reset_counters() {
    vote_ms = 0; vote_pairs = 0; launches = 0; vote_launches = 0; vote_pending = false;
    cull_ms = 0; cull_pairs = 0; cull_launches = 0; cull_tc_launches = 0; cevn = 0;
  }
  template <class R>
  void fill_counters(R& r) const {
    r.vote_ms = vote_ms;
    r.vote_pairs = vote_pairs;
    r.launches = launches;
    r.vote_launches = vote_launches;
    r.cull_ms = cull_ms;
    r.cull_pairs = cull_pairs;
    r.cull_launches = cull_launches;
    r.cull_tc_launches = cull_tc_launches;
  }
  Trace* trace = nullptr;  // RV_TRACE=1: host phase timings
  void mark(const char* what) {
    if (trace) trace->mark(what);
  }

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? RV_ENOMEM : RV_ECUDA, "%s: %s", what,
                cudaGetErrorString(e));
  }
  // this call runs ONE problem whose levels are sharded over the ranks (or the loopback
  // emulation of that); set by solve_batched_impl from the caller's problem count -- a rank's
  // local share of a batch (one problem when P is in [W, 2W)) is never split
  bool split_one = false;
  bool host_plan = false;  // cfg.planner == 1: the host planner drives every level
  int effective_world() const {
    if (cfg.world > 1) return cfg.world;
    return cfg.emulate_world > 1 ? cfg.emulate_world : 1;
  }
};

#define RV_CUDA(call, what)                               \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return ctx->cuda_fail(e_, what); \
  } while (0)

namespace {

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
                    int64_t cpb = rv::kTcM, const std::vector<const void*>* seg_key = nullptr) {
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
              float* dump = nullptr, int64_t ld = 0) {
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

// ---- K1 for P problems ----------------------------------------------------------------------
int run_setup(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
              std::vector<int64_t>& koff_out) {
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
  int64_t* hrows = ctx->up.take<int64_t>(P + 1);
  int64_t* hk = ctx->up.take<int64_t>(P + 1);
  std::memcpy(hrows, offsets, (P + 1) * sizeof(int64_t));
  std::memcpy(hk, koff_out.data(), (P + 1) * sizeof(int64_t));
  RV_CUDA(cudaMemcpyAsync(ctx->rows.p, hrows, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
          "copying offsets");
  RV_CUDA(cudaMemcpyAsync(ctx->koffs.p, hk, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
          "copying offsets");
  RV_CUDA(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), ctx->stream), "memset");
  rv::launch_setup(x, y, ctx->rows.p, ctx->koffs.p, P, total, ctx->k9.p, ctx->stride, ctx->bad.p,
                   ctx->stream);
  ctx->launches += 1;
  if (ctx->tc_on) {
    std::vector<int64_t> toff(P + 1, 0);
    for (int32_t p = 0; p < P; ++p) {
      const int64_t np = offsets[p + 1] - offsets[p];
      toff[p + 1] = toff[p] + (np + rv::kTcN - 1) / rv::kTcN * rv::kTcN;
    }
    // + one group of 8 padding rows after the last problem (K3-CT gathers it for padding)
    RV_CUDA(ctx->tctab.ensure((size_t)(toff[P] + 8) * 64), "allocating K3-TC table");
    RV_CUDA(ctx->toffs.ensure(P + 1), "allocating offsets");
    int64_t* ht = ctx->up.take<int64_t>(P + 1);  // staging sized for it above
    std::memcpy(ht, toff.data(), (P + 1) * sizeof(int64_t));
    RV_CUDA(cudaMemcpyAsync(ctx->toffs.p, ht, (P + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
            "copying offsets");
    // the culled levels' rows: K3-CT's fp16-split row-major copy, or K3-C's fp32 rows (the
    // culled path cull_prepare will pick: K3-CT unless RV_CULL_TC=0 or a multi-rank batch)
    const bool ct = ctx->cull_on && ctx->cull_tc;
    const bool k3c = ctx->cull_on && !ct;
    if (k3c) RV_CUDA(ctx->k12.ensure((size_t)(toff[P] + 8) * 12), "allocating K3-C rows");
    if (ct) RV_CUDA(ctx->tctab_rm.ensure((size_t)(toff[P] + 8) * 64), "allocating K3-CT rows");
    rv::launch_setup_tc(x, y, ctx->rows.p, ctx->toffs.p, P, toff[P] + 8, ctx->tctab.p, ctx->stream,
                        k3c ? ctx->k12.p : nullptr, ct ? ctx->tctab_rm.p : nullptr);
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
  RV_CUDA(cudaStreamSynchronize(ctx->stream), "rv_setup");
  if (b != ~0ull)
    return ctx->fail(RV_EDATA, "correspondence row %llu has a zero-length or non-finite vector", b);
  return RV_OK;
}

// ---- one planner request (single problem), sharded over ranks --------------------------------
// Counts land in cnt_a/cnt_b (HOST, m entries each).
// auto_tc: RV_MODE_BOUND / RV_MODE_FINAL go to K3-TC when the context has tensor_vote (the
// solve); false keeps the explicit mode -> kernel mapping of rot_vote_count_cells.
int eval_request(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps, int32_t B,
                 int32_t mode, int64_t m, const uint32_t* lins, uint32_t* cnt_a, uint32_t* cnt_b,
                 bool auto_tc = true) {
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
  RV_CUDA(cudaStreamSynchronize(s), "vote");
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
  RV_CUDA(cudaStreamSynchronize(s), "refinement");
  std::memcpy(q_out, dq, (size_t)P * 32);
  for (int32_t p = 0; p < P; ++p) flags_out[p] = df[p] & (RV_REFINED | RV_DEGENERATE);
  std::memcpy(ninl_out, dn, P * 4);
  return RV_OK;
}

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

int solve_batched_impl(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets,
                       int32_t P, double eps, int32_t levels, rv_result* out, uint32_t* masks);
bool dplan_applies(rv_ctx* ctx, int32_t levels_eff, int32_t B0, double eps);

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
  RV_CUDA(cudaEventSynchronize(ctx->ev1), "event");
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
  if (int rc = run_setup(ctx, x, y, offs, 1, koff)) return rc;
  if (int rc = check_bad(ctx)) return rc;
  CountCache cache;
  std::vector<double> excl;  // earlier peaks' block-centre rotations
  int32_t found = 0;
  for (int32_t k = 0; k < K; ++k) {
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
  RV_CUDA(cudaEventSynchronize(ctx->ev1), "event");
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  for (int32_t k = 0; k < found; ++k) {
    out[k].ms = ms;
    ctx->fill_counters(out[k]);
  }
  *n_found = found;
  return RV_OK;
}

// ---- NEXT-3: rigid pose front end ----------------------------------------------------------
// R(q) of P:955-961, row-major, each entry evaluated left to right (the translation bins are
// integers decided on these values, so the order is part of the definition)
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
  RV_CUDA(cudaStreamSynchronize(s), "translation vote");
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
  RV_CUDA(cudaStreamSynchronize(s), "pair count");
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
  RV_CUDA(cudaEventSynchronize(e[3]), "event");
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
struct BatchReq {
  int32_t prob;        // local problem index
  int32_t B, mode;
  int64_t m;
  const uint32_t* lins;
  bool full_grid;      // the complete candidate list of B: served from one device copy
};

// keep_dev != nullptr: the cnt_a counts stay on the device (copied to keep_dev, request order)
// and nothing is read back (level 0 of a batched solve, reduced by the K4 kernels).
int eval_batch(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode,
               const std::vector<BatchReq>& reqs, std::vector<std::vector<uint32_t>>& ca,
               std::vector<std::vector<uint32_t>>& cb, uint32_t* keep_dev = nullptr) {
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
    RV_CUDA(cudaStreamSynchronize(s), "batched vote");
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
  RV_CUDA(cudaStreamSynchronize(s), "batched vote");
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
                     bool force = false) {
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
  RV_CUDA(cudaStreamSynchronize(s), "level-0 lists");
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
               bool emit_bits = false) {
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
    RV_CUDA(ctx->c_phi.ensure(npos * 12), "allocating");
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
    ctx->launches += rv::launch_cull_items(Ld, ctx->rows.p, ctx->toffs.p, PL, B, ctx->cull_B0,
                                           ctx->cull_grouped ? ctx->lutg.p : ctx->lut0.p,
                                           ctx->cull_G, ctx->cull_l0cnt,
                                           ctx->c_lofs.p, ctx->k12.p, eps, mode, ctx->cfg.guard,
                                           ctx->num_sms, cs, ctx->vsegs.p, ctx->c_items.p, eb, mi,
                                           ctx->dp_err.p, s, ctx->cull_own_lo, ctx->cull_own_hi);
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
    RV_CUDA(cudaEventRecord(e0, s), "event");
    if (ctx->cull_grouped)  // K3-CT
      rv::launch_vote_cull_tc(mode, ctx->vsegs.p, ctx->c_items.p, ctx->c_icnt.p, ctx->tctab_rm.p,
                              ctx->tc_toff.back(), ctx->c_tphi.p, ctx->c_cidx.p, ctx->c_lidx.p,
                              ctx->c_pairs.p, ctx->num_sms, s,
                              ctx->c_work.p);
    else
      rv::launch_vote_cull(mode, ctx->vsegs.p, ctx->c_items.p, ctx->c_icnt.p, ctx->c_work.p,
                           ctx->c_pairs.p, ctx->c_phi.p, ctx->c_cidx.p, ctx->c_lidx.p,
                           ctx->cfg.guard, ctx->num_sms, s);
    RV_CUDA(cudaEventRecord(e1, s), "event");
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
      RV_CUDA(cudaEventRecord(e0, s), "event");
      rv::launch_vote_tc(ctx->tctab.p, ctx->atab.p, ctx->ablk.p, 0, ctx->vsegs.p, ctx->vitems.p, 0,
                         ctx->cfg.guard + kTcExtraGuard, nullptr, 0, s, im == 1, ctx->dp_icnt.p,
                         emit_bits);
      RV_CUDA(cudaEventRecord(e1, s), "event");
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
  RV_CUDA(cudaStreamSynchronize(s), "batched level");
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
int solve_batched_dplan(rv_ctx* ctx, const float* x, const float* y,
                        const std::vector<int64_t>& rows, const std::vector<int64_t>& koff,
                        int32_t PL, double eps, const std::vector<int32_t>& ch,
                        std::vector<rv_plan_result>& res, Trace& tr) {
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
                          ctx->dp_rflag.p, ctx->dp_rany.p};
      if (any) RV_CUDA(cudaMemsetAsync(ctx->dp_rany.p, 0, 4, s), "memset");
      rv::dp_launch_scan(ctx->dp_cnt[nb].p, PL, nf3, cact, nbase, ctx->dp_tot.p, s,
                         any ? &chk : nullptr);
      ctx->launches += 1;
      ctx->down.reset();
      int64_t* ht = ctx->down.take<int64_t>(1);
      int32_t* ha = ctx->down.take<int32_t>(1);
      RV_CUDA(cudaMemcpyAsync(ht, ctx->dp_tot.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
      if (any) RV_CUDA(cudaMemcpyAsync(ha, ctx->dp_rany.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
      RV_CUDA(cudaStreamSynchronize(s), "batched level");
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
  RV_CUDA(ctx->down.ensure((size_t)PL * 24 + (size_t)nph * PL * 4 + 2048), "allocating staging");
  ctx->down.reset();
  unsigned long long* hbest = ctx->down.take<unsigned long long>(PL);
  int32_t* hties = ctx->down.take<int32_t>(PL);
  int64_t* hlb = ctx->down.take<int64_t>(PL);
  int32_t* hph = ctx->down.take<int32_t>((size_t)nph * PL);
  int32_t* herr = ctx->down.take<int32_t>(1);
  unsigned long long* hcp = ctx->down.take<unsigned long long>(1);
  RV_CUDA(cudaMemcpyAsync(herr, ctx->dp_err.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
  if (culled) RV_CUDA(cudaMemcpyAsync(hcp, ctx->c_pairs.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hbest, ctx->dp_best.p, 8 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hties, ctx->dp_ties.p, 4 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hlb, ctx->dp_lb.p, 8 * (size_t)PL, cudaMemcpyDeviceToHost, s), "D2H");
  RV_CUDA(cudaMemcpyAsync(hph, ctx->dp_phase.p, 4 * (size_t)nph * PL, cudaMemcpyDeviceToHost, s),
          "D2H");
  RV_CUDA(cudaStreamSynchronize(s), "batched finalize");
  ctx->collect_vote_ms();
  ctx->ev_collect();
  ctx->cev_collect();
  ctx->cull_ready = false;
  if (culled) ctx->cull_pairs += *hcp;
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
    if (int rc = run_setup(ctx, x, y, rows.data(), PL, koff)) return rc;
    if (int rc = check_bad(ctx)) return rc;
    tr.mark("setup");
    int rc = RV_OK;
    const int32_t lev = levels == 0 ? std::min<int32_t>(5, (int32_t)ctx->chain.size()) : levels;
    const std::vector<int32_t> ch(ctx->chain.end() - lev, ctx->chain.end());
    std::vector<rv_plan_result> pres(PL);
    if (dplan_applies(ctx, lev, ch[0], eps)) {
      rc = solve_batched_dplan(ctx, x, y, rows, koff, PL, eps, ch, pres, tr);
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
            RV_CUDA(cudaStreamSynchronize(ctx->stream), "level-0 argmax");
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
        RV_CUDA(cudaStreamSynchronize(ctx->stream), "level-0 survivors");
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
        RV_CUDA(cudaStreamSynchronize(ctx->stream), "level-0 survivors");
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
    // rows are absolute: refine over the local offsets table
    rc = run_refine(ctx, x, y, rows.data(), PL, ids.data(), eps, q0.data(), ctx->cfg.refine_rounds,
                    mw.data(), masks, qf.data(), fl.data(), ni.data());
    if (rc) return rc;
    tr.mark("refine");
    for (int32_t p = 0; p < PL; ++p) {
      std::memcpy(local[p].q, &qf[4 * p], 32);
      local[p].flags |= fl[p];
      local[p].n_inliers = ni[p];
    }
  }
  RV_CUDA(cudaEventRecord(ctx->ev1, s), "event");
  RV_CUDA(cudaEventSynchronize(ctx->ev1), "event");
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
  RV_CUDA(cudaStreamSynchronize(s), "gather");
  for (int r = 0; r < W; ++r) {
    int64_t b, e;
    rv_shard_range(P, r, W, &b, &e);
    std::memcpy(out + b, hd + slot * r, (size_t)(e - b) * sizeof(rv_result));
  }
  return RV_OK;
}

}  // namespace

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
  if (cfg->cull < 0 || cfg->cull > 2 || cfg->planner < 0 || cfg->planner > 1) return RV_EINVAL;
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
  if (e == cudaSuccess) {
    ctx->stride = pad4(cfg->max_n) + 64;
    e = ctx->k9.ensure((size_t)9 * ctx->stride);
  }
  if (e == cudaSuccess) e = ctx->bad.ensure(1);
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
  ctx->koffs.release(); ctx->bad.release(); ctx->hx.release(); ctx->hy.release();
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
  ctx->dp_best.release(); ctx->a1_acc.release(); ctx->a1_tab.release(); ctx->a1_best.release(); ctx->dp_ioff.release(); ctx->dp_aoff.release(); ctx->dp_tot.release();
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
  ctx->up.release(); ctx->down.release();
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evv0) cudaEventDestroy(ctx->evv0);
  if (ctx->evv1) cudaEventDestroy(ctx->evv1);
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
