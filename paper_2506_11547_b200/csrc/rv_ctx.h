// rv_ctx.h -- librotvote's internal context (rv_ctx) and the helpers its translation units
// share: growable device buffers, pinned staging, the run-time NCCL table, the host trace, and
// the declarations of the solve steps (rv_api.cpp: the C-ABI; rv_setup.cpp: setup and
// refinement; rv_host_plan.cpp: the host-planner paths, several rotations, rigid pose;
// rv_level_loop.cpp: the device level loop, culling and the one-pass single solve).
#pragma once
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
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
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges per phase (Nsight Systems timelines)
#include <nccl.h>  // types only; the library is dlopen'ed (libnccl.so.2) when world > 1

#include "../../include/rotvote.h"
#include "../../include/rotvote_plan.h"
#include "rv_geom.h"
#include "rv_alg1.h"
#include "rv_dplan.h"
#include "rv_rigid.h"
#include "rv_kernels.h"

namespace rvi {

inline constexpr int32_t kDefaultChain[6] = {5, 15, 45, 90, 180, 360};
// Extra guard for K3-TC bound counts: worst-case |S'_tc - (s - t)| of the fp16-split MMA
// (split remainders <= 3 * 2^-22 * sum|k phi| <= 2.9e-6, threshold split 2.4e-7, fp32
// accumulation of 32 exact products <= 32 * 2^-24 * 5 = 9.5e-6) < 1.3e-5; measured 3.7e-7.
inline constexpr float kTcExtraGuard = 1.5e-5f;

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

inline NcclApi& nccl() {
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
// Bumped by every workspace (re)allocation: a captured one-pass graph holds raw device pointers,
// so it is replayed only while this is unchanged since its capture.
inline std::atomic<uint64_t> g_realloc_epoch{0};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    g_realloc_epoch.fetch_add(1);
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


}  // namespace rvi

using rvi::DevBuf;
using rvi::Staging;
using rvi::Trace;


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
  DevBuf<unsigned long long> dp_best, dp_best_r;  // (_r: per-rank winners, sharded one pass)
  DevBuf<int32_t> dp_ties_r;
  DevBuf<double> excl_q;        // NEXT-2: the earlier peaks' rotations (device copy)
  bool reuse_l0 = false;        // NEXT-2: a later peak's one-pass solve keeps setup + level 0
  int64_t op_cap = (int64_t)1 << 18;  // one-pass level-list capacity (blocks; grows on overflow)
  int32_t op_lshift = 4;        // one-pass culling-list capacity: level-0 pairs >> this
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
  DevBuf<int32_t> dp_tdone;  // last-CTA counter of the tail scans (zeroed at create)
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
    cudaGetLastError();
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
  const int64_t* cull_pre_act = nullptr;  // see launch_cull_items (one-pass branch and bound)
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
    cudaGetLastError();
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
  Staging up2, down2;           // a second pair for work enqueued while the first is in flight
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evv0 = nullptr, evv1 = nullptr;
  cudaEvent_t ph[8] = {};       // phase boundaries of a one-pass solve (rv_result.t_*_ms)
  // one-pass solves as a CUDA graph: the enqueue sequence of a single solve depends only on
  // (x, y, n, eps, levels, mask) and the context, so the second consecutive solve with the same
  // key is captured (on gstream, forked from / joined to the caller's stream) and later ones
  // replay it; grb is the graph's pinned read-back block (never reallocated)
  cudaStream_t gstream = nullptr;
  cudaEvent_t gfork = nullptr, gjoin = nullptr;
  cudaGraphExec_t gexec = nullptr;
  bool graphs_on = true;        // cleared for good if a capture fails
  uint64_t gepoch = 0;          // g_realloc_epoch at the capture
  uint64_t gkey[8] = {}, lastkey[8] = {};
  bool gkey_ok = false, lastkey_ok = false;
  char* grb = nullptr;          // pinned, 4 KB
  bool capturing = false;
  // an event record that becomes an event node of a captured graph (timing inside the graph)
  cudaError_t record(cudaEvent_t e, cudaStream_t s) const {
    return capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                     : cudaEventRecord(e, s);
  }
  struct OnePassHost {          // host values of the captured enqueue (same on every replay)
    int64_t m0 = 0;
    int nph = 0;
    bool cull = false;
    int32_t launches = 0, vote_launches = 0, cull_launches = 0, cull_tc_launches = 0;
    size_t evn = 0, cevn = 0;
  } ghost;
  int32_t host_syncs = 0;       // host waits on the device in this call
  bool retried = false;         // a one-pass solve was redone by the per-level loop
  int32_t redo_reason = 0;      // its error word
  // per-call counters reported in rv_result
  float vote_ms = 0, cull_ms = 0;
  uint64_t vote_pairs = 0, cull_pairs = 0;
  int32_t launches = 0, vote_launches = 0, cull_launches = 0, cull_tc_launches = 0;
  void reset_counters() {
    host_syncs = 0; retried = false; redo_reason = 0;
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
    r.host_syncs = host_syncs;
    if (retried) r.flags |= RV_RETRIED;
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

// a host wait on the device inside a call (counted in rv_result.host_syncs)
#define RV_STR2(x) #x
#define RV_STR(x) RV_STR2(x)
#define RV_SYNC(call, what)                                                        \
  do {                                                                             \
    ctx->host_syncs += 1;                                                          \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return ctx->cuda_fail(e_, what " (" __FILE__ ":" RV_STR(__LINE__) ")"); \
  } while (0)
#define RV_CUDA(call, what)                                                        \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return ctx->cuda_fail(e_, what " (" __FILE__ ":" RV_STR(__LINE__) ")"); \
  } while (0)

namespace rvi {

// ---- the steps, one translation unit each (definitions carry no default arguments) ------------
// rv_host_plan.cpp: host-built K3-TC items and launch (also the count_cells test entries)
void build_tc_items(const std::vector<int64_t>& ncell, const std::vector<int64_t>& ncorr,
                    int slots, std::vector<rv::VoteItem>& items, std::vector<rv::ABlock>& ablocks,
                    int64_t cpb = rv::kTcM, const std::vector<const void*>* seg_key = nullptr);
int launch_tc(rv_ctx* ctx, const std::vector<rv::ABlock>& ab, int32_t n_items, bool fin,
              float* dump = nullptr, int64_t ld = 0);
int eval_request(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps, int32_t B,
                 int32_t mode, int64_t m, const uint32_t* lins, uint32_t* cnt_a, uint32_t* cnt_b,
                 bool auto_tc = true);
// rv_setup.cpp
// cull_rows = false: the culled levels' row tables (K3-CT / K3-C) are not written (a solve that
// cannot cull).  dev_offsets (P == 1 only): the offset tables are written by a kernel from its arguments instead
// of copied from pinned staging (a captured graph must not point at reusable host memory)
int run_setup(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
              std::vector<int64_t>& koff_out, bool dev_offsets = false, bool cull_rows = true);
int check_bad(rv_ctx* ctx);
struct RefineOut {            // enqueue_refine's read-back (pinned, valid after the next wait)
  double* q = nullptr;
  int32_t* flags = nullptr;
  uint32_t* ninl = nullptr;
};
int enqueue_refine(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
                   double eps, int32_t rounds, const int64_t* mask_words, uint32_t* masks,
                   RefineOut& out);
int run_refine(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets, int32_t P,
               const int32_t* prob_ids, double eps, const double* qs0, int32_t rounds,
               const int64_t* mask_words, uint32_t* masks, double* q_out, int32_t* flags_out,
               uint32_t* ninl_out);
// rv_api.cpp
void canonicalize(double q[4]);
void canonical_cell_quat(int32_t B, uint32_t lin, double q[4]);
int validate_common(rv_ctx* ctx, const void* x, const void* y, double eps, int32_t levels);
void fill_result(const rv_plan_result& pr, rv_result* out);
// rv_host_plan.cpp
int solve_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps, int32_t levels,
               rv_result* out, uint32_t* mask);
int solve_multi_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                     int32_t levels, int32_t K, double rho, rv_result* out, int32_t* n_found);
int translation_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, const double* q,
                     double t_lo, double t_hi, double t_step, int64_t* lin, uint32_t* votes,
                     double* t, double* t_mean);
int rigid_impl(rv_ctx* ctx, const float* x, const float* y, int64_t n, double mu_t, double eps,
               int32_t levels, double t_lo, double t_hi, double t_step, rv_rigid_result* out,
               int32_t* pair_ij, int64_t pair_cap);
struct BatchReq {
  int32_t prob;        // local problem index
  int32_t B, mode;
  int64_t m;
  const uint32_t* lins;
  bool full_grid;      // the complete candidate list of B: served from one device copy
};
int eval_batch(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode,
               const std::vector<BatchReq>& reqs, std::vector<std::vector<uint32_t>>& ca,
               std::vector<std::vector<uint32_t>>& cb, uint32_t* keep_dev = nullptr);
int vote_lists(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode, int32_t B,
               const uint32_t* dlins, const std::vector<int64_t>& hoff,
               const std::vector<int32_t>& hcnt, int64_t span, uint32_t* dca, uint32_t* dcb);
// rv_level_loop.cpp
int cull_prepare(rv_ctx* ctx, int32_t B0, int64_t m0, int32_t PL);
int cull_build_lists(rv_ctx* ctx, int32_t PL, int64_t m0, const uint32_t* l0cnt,
                     bool force = false);
int vote_level(rv_ctx* ctx, const float* x, const float* y, const std::vector<int64_t>& rows,
               const std::vector<int64_t>& koff, double eps, int32_t mode, int32_t B,
               const rv::DpList& Ld, int32_t PL, int64_t entries_bound, int64_t nmax,
               bool emit_bits = false, const rv::DiveStep* dive = nullptr);
bool dplan_applies(rv_ctx* ctx, int32_t levels_eff, int32_t B0, double eps);
int solve_batched_impl(rv_ctx* ctx, const float* x, const float* y, const int64_t* offsets,
                       int32_t P, double eps, int32_t levels, rv_result* out, uint32_t* masks);
// the one-pass single solve (rv_level_loop.cpp); excl: NEXT-2 exclusion balls (no graph);
// *redo: a capacity or the re-dive trigger -- redo the solve another way
bool one_pass_applies(rv_ctx* ctx, int32_t P);
int solve_one_pass(rv_ctx* ctx, const float* x, const float* y, int64_t n, double eps,
                   const std::vector<int32_t>& ch, rv_result* out, uint32_t* mask, bool* redo,
                   const rv::Excl* excl = nullptr);

}  // namespace rvi

