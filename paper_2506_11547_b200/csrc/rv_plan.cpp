// rv_plan.cpp -- host planner of the certified coarse-to-fine search (include/rotvote_plan.h).
//
// Reading R6: on a chain of nested grids B_0 | B_1 | ... | B_{L-1}
// (B_{L-1} = the paper's accumulator resolution),
//   UB(c) = #{i : s_i(q_c) >= cos(min(pi, eps + r(c))) - guard}
// bounds the count of every finest block whose centre lies in block c.  The search:
//   1. level 0: UB of every candidate block;
//   2. dive: from the level-0 block of largest excess UB - n(1 - t_c)/2 (t_c the unguarded
//      bound threshold, n(1-t_c)/2 the uniform-outlier background, Archimedes), vote the
//      children of its 3x3x3 neighbourhood level by level, re-ranking by excess, down to
//      the finest level, where LB* = max #{s32 >= tau + guard} is a certified lower bound
//      of the best exact count;
//   3. branch and bound: keep blocks with UB >= LB* (ties kept), vote their children, ...;
//   4. finest level: cnt_hi = #{s32 >= tau - guard} >= exact >= cnt_lo = #{s32 >= tau + guard};
//      blocks with hi >= max lo and hi != lo get the exact fp64 recheck (RV_MODE_EXACT);
//      winner = max exact count, ties -> lowest lin (R7).
// The result equals the exhaustive scan of the finest grid for every chain and `levels`.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/rotvote.h"
#include "../../include/rotvote_plan.h"
#include "rv_geom.h"

namespace {

enum Phase { PH_L0, PH_DIVE, PH_NEED_SURV, PH_BNB, PH_REDIVE, PH_RECHECK, PH_DONE };

std::vector<uint32_t> candidates_of(int32_t B) {
  std::vector<uint32_t> out;
  for (int32_t i = 0; i < B; ++i)
    for (int32_t j = 0; j < B; ++j)
      for (int32_t k = 0; k < B; ++k)
        if (rv::is_candidate(B, i, j, k)) out.push_back(rv::ijk_to_lin(i, j, k, B));
  return out;
}

// The dive starts and steps only through blocks whose centre lies inside the ball when there
// are any: blocks that merely touch the ball from outside represent rotations of the far side
// (a heuristic -- the certified pruning is unaffected).
using rv::centre_inside;

// Process-wide caches of a grid's candidate list and of the per-candidate uniform-outlier
// background (1 - cos(min(pi, eps + r(c))))/2 (batched solves create thousands of planners
// on the same grid and eps).  Entries are never erased, so references stay valid.
struct GridCache {
  std::vector<uint32_t> cand;
  std::map<uint64_t, std::vector<double>> bg;  // keyed by the bits of eps
};
std::mutex g_cache_mu;
std::map<int32_t, std::unique_ptr<GridCache>> g_cache;

GridCache& grid_cache(int32_t B) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  std::unique_ptr<GridCache>& e = g_cache[B];
  if (!e) {
    e.reset(new GridCache());
    e->cand = candidates_of(B);
  }
  return *e;
}

const std::vector<double>* grid_background(int32_t B, double eps) {
  GridCache& gc = grid_cache(B);
  uint64_t key;
  std::memcpy(&key, &eps, sizeof(key));
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = gc.bg.find(key);
  if (it != gc.bg.end()) return &it->second;
  if (gc.bg.size() >= 64) return nullptr;  // bounded: fall back to direct evaluation
  std::vector<double>& v = gc.bg[key];
  v.resize(gc.cand.size());
  for (size_t e = 0; e < gc.cand.size(); ++e) {
    int32_t i, j, k;
    rv::lin_to_ijk(gc.cand[e], B, i, j, k);
    v[e] = (1.0 - rv::bound_threshold(B, i, j, k, eps)) * 0.5;
  }
  return &v;
}

}  // namespace

struct rv_plan {
  std::vector<int32_t> chain;
  int64_t n = 0;
  double eps = 0, guard = 0;
  Phase phase = PH_L0;
  int level = 0;
  int32_t mode = RV_MODE_BOUND;
  std::vector<uint32_t> cells;  // pending request

  std::vector<uint32_t> l0_cells, l0_ub;
  // re-dive (reading R18): when a branch-and-bound level >= 2 would keep more than half of all
  // possible children, the dive's lb* is too weak; dive once more from the best-excess block
  // of the parent level, raise lb* to that dive's finest-level lower bound, and recompute
  // the survivors
  // (only for a level of at least kRediveMin blocks: a cheap level needs no stronger bound)
  static constexpr int64_t kRediveMin = 16384;
  bool redived = false;
  int redive_parent = 0;
  std::vector<uint32_t> redive_cells, redive_ub;
  // NEXT-2 exclusion balls (earlier peaks' block-centre rotations, suppression angle rho):
  // a finest block is excluded iff |q_c . q_e| >= cos(rho/2) (angle <= rho); a coarser block
  // is dropped only when all of it is: angle(q_c, q_e) + r(c) <= rho (r(c) bounds the
  // rotation angle from q_c to any rotation of the block, as in the certified bound)
  std::vector<std::array<double, 4>> excl;
  double rho = 0.0, cos_half_rho = 2.0;
  bool l0_ext = false;  // level 0 reduced by the caller (rv_plan_feed_l0_start / _survivors)
  int64_t lb_star = 0;
  // finest level
  std::vector<uint32_t> fin_cells, fin_lo, fin_hi, recheck_idx;
  rv_plan_result res{};

  int last() const { return (int)chain.size() - 1; }

  bool excluded(int l, uint32_t lin) const {
    if (excl.empty()) return false;
    const int32_t B = chain[l];
    int32_t i, j, k;
    rv::lin_to_ijk(lin, B, i, j, k);
    double q[4];
    rv::cell_quat(B, i, j, k, q);
    const double r = l == last() ? 0.0 : rv::bound_radius(B, i, j, k);
    for (const auto& e : excl) {
      const double d = std::fabs(q[0] * e[0] + q[1] * e[1] + q[2] * e[2] + q[3] * e[3]);
      if (l == last()) {
        if (d >= cos_half_rho) return true;
      } else {
        const double ang = 2.0 * std::acos(std::min(1.0, d));
        if (ang + r <= rho - 1e-9) return true;
      }
    }
    return false;
  }
  void drop_excluded(int l, std::vector<uint32_t>& v) const {
    if (excl.empty()) return;
    size_t w = 0;
    for (uint32_t c : v)
      if (!excluded(l, c)) v[w++] = c;
    v.resize(w);
  }
  int32_t mode_for(int l) const { return l == last() ? RV_MODE_FINAL : RV_MODE_BOUND; }

  void note_request() {
    res.pair_votes += (uint64_t)cells.size() * (uint64_t)n;
    res.cells_evaluated += cells.size();
    if (res.n_phases < 16) res.cells_per_phase[res.n_phases++] = (int64_t)cells.size();
  }

  double excess(int32_t B, uint32_t lin, uint32_t ub) const {
    int32_t i, j, k;
    rv::lin_to_ijk(lin, B, i, j, k);
    double t = rv::bound_threshold(B, i, j, k, eps);
    return (double)ub - (double)n * (1.0 - t) * 0.5;
  }

  // NEXT-2 dive preference of block lin at level l: 2 = entirely outside every exclusion
  // ball (angle(q_c, q_e) - r(c) > rho), 1 = centre outside, 0 = centre inside a ball
  int excl_rank(int l, uint32_t lin) const {
    if (excl.empty()) return 2;
    const int32_t B = chain[l];
    int32_t i, j, k;
    rv::lin_to_ijk(lin, B, i, j, k);
    double q[4];
    rv::cell_quat(B, i, j, k, q);
    const double r = rv::bound_radius(B, i, j, k);
    int rank = 2;
    for (const auto& e : excl) {
      const double d = std::fabs(q[0] * e[0] + q[1] * e[1] + q[2] * e[2] + q[3] * e[3]);
      if (d >= cos_half_rho) return 0;
      if (2.0 * std::acos(std::min(1.0, d)) - r <= rho) rank = 1;
    }
    return rank;
  }

  // index of the max-excess block, ties -> lowest lin; blocks whose centre lies inside the
  // ball come first, and (NEXT-2) blocks away from the exclusion balls before those (excl_rank)
  // -- a dive into or next to a suppressed region would end with a weak lb*
  size_t best_excess(int l, const std::vector<uint32_t>& c, const uint32_t* ub,
                     const double* bg = nullptr) const {
    const int32_t B = chain[l];
    size_t best = 0;
    double be = -1e300;
    int bk = -1;  // rank: 2 * excl_rank + (centre inside the ball)
    for (size_t e = 0; e < c.size(); ++e) {
      const int kk = 2 * excl_rank(l, c[e]) + (centre_inside(B, c[e]) ? 1 : 0);
      if (kk < bk) continue;
      const double x = bg ? (double)ub[e] - (double)n * bg[e] : excess(B, c[e], ub[e]);
      if (kk > bk || x > be || (x == be && c[e] < c[best])) { be = x; best = e; bk = kk; }
    }
    return best;
  }

  // candidate children at level l+1 of level-l blocks, in generation order (parents in the
  // given order, children in (a,b,c) order).  The order is deterministic, so every rank
  // builds the identical list; no decision depends on it (ties are broken by lin).
  std::vector<uint32_t> children(int l, const std::vector<uint32_t>& parents) const {
    const int32_t B = chain[l], Bc = chain[l + 1], f = Bc / B;
    std::vector<uint32_t> out;
    out.reserve(parents.size() * (size_t)(f * f * f));
    const int64_t BB = (int64_t)B * B;
    for (uint32_t p : parents) {
      int32_t i, j, k;
      rv::lin_to_ijk(p, B, i, j, k);
      // (B * farthest corner distance)^2 <= B^2  =>  every child meets the ball
      int64_t dmax2 = 0;
      for (int32_t v : {i, j, k}) {
        int64_t lo = 2 * (int64_t)v - B, hi = lo + 2;
        int64_t d = std::max(lo < 0 ? -lo : lo, hi < 0 ? -hi : hi);
        dmax2 += d * d;
      }
      const bool inside = dmax2 <= BB;
      for (int32_t a = 0; a < f; ++a)
        for (int32_t b = 0; b < f; ++b)
          for (int32_t c = 0; c < f; ++c) {
            int32_t ci = f * i + a, cj = f * j + b, ck = f * k + c;
            if (inside || rv::is_candidate(Bc, ci, cj, ck)) out.push_back(rv::ijk_to_lin(ci, cj, ck, Bc));
          }
    }
    drop_excluded(l + 1, out);
    return out;
  }

  std::vector<uint32_t> neighbourhood(int l, uint32_t lin) const {
    const int32_t B = chain[l];
    int32_t i, j, k;
    rv::lin_to_ijk(lin, B, i, j, k);
    std::vector<uint32_t> out;
    for (int32_t a = -1; a <= 1; ++a)
      for (int32_t b = -1; b <= 1; ++b)
        for (int32_t c = -1; c <= 1; ++c) {
          int32_t ni = i + a, nj = j + b, nk = k + c;
          if (ni < 0 || nj < 0 || nk < 0 || ni >= B || nj >= B || nk >= B) continue;
          if (rv::is_candidate(B, ni, nj, nk)) out.push_back(rv::ijk_to_lin(ni, nj, nk, B));
        }
    std::sort(out.begin(), out.end());
    return out;
  }

  void start_bnb() {
    std::vector<uint32_t> surv;
    for (size_t e = 0; e < l0_cells.size(); ++e)
      if ((int64_t)l0_ub[e] >= lb_star) surv.push_back(l0_cells[e]);
    start_bnb_from(surv);
  }
  void start_bnb_from(const std::vector<uint32_t>& surv) {
    phase = PH_BNB;
    level = 1;
    mode = mode_for(level);
    cells = children(0, surv);
    note_request();
  }
  // back to branch and bound at the level whose children triggered the re-dive
  void resume_bnb() {
    std::vector<uint32_t> surv;
    for (size_t e = 0; e < redive_cells.size(); ++e)
      if ((int64_t)redive_ub[e] >= lb_star) surv.push_back(redive_cells[e]);
    phase = PH_BNB;
    level = redive_parent;
    cells = children(level, surv);
    ++level;
    mode = mode_for(level);
    note_request();
  }
  void start_dive_or_bnb(size_t s) {
    if (l0_cells.empty()) {  // every level-0 block excluded: nothing left
      lb_star = 0;
      level = last();
      mode = RV_MODE_FINAL;
      cells.clear();
      fin_cells.clear();
      finalize();
      return;
    }
    start_dive(s);
  }
  void start_dive(size_t s) {
    phase = PH_DIVE;
    level = 1;
    mode = mode_for(level);
    cells = children(0, neighbourhood(0, l0_cells[s]));
    note_request();
  }

  void finalize() {
    // exact counts are known for blocks with lo == hi or rechecked; every other block
    // has hi < max lo <= the best exact count, so it cannot win or tie.
    std::vector<int64_t> exact(fin_cells.size(), -1);
    for (size_t e = 0; e < fin_cells.size(); ++e)
      if (fin_lo[e] == fin_hi[e]) exact[e] = fin_lo[e];
    for (size_t r = 0; r < recheck_idx.size(); ++r) exact[recheck_idx[r]] = (int64_t)cells_exact[r];
    int64_t best = -1;
    uint32_t best_lin = 0;
    int32_t tied = 0;  // stays 0 (votes 0) when every block was excluded
    for (size_t e = 0; e < fin_cells.size(); ++e) {
      if (exact[e] < 0) continue;
      if (exact[e] > best) { best = exact[e]; best_lin = fin_cells[e]; tied = 1; }
      else if (exact[e] == best) { ++tied; if (fin_cells[e] < best_lin) best_lin = fin_cells[e]; }
    }
    res.lin = best_lin;
    res.B = chain.back();
    res.votes = (uint32_t)(best < 0 ? 0 : best);
    res.n_tied = tied;
    res.lb_star = (uint32_t)lb_star;
    res.n_rechecked = (int32_t)recheck_idx.size();
    phase = PH_DONE;
    cells.clear();
  }

  void enter_final(const uint32_t* a, const uint32_t* b) {
    fin_cells = cells;
    fin_hi.assign(a, a + cells.size());
    fin_lo.assign(b, b + cells.size());
    uint32_t L = 0;
    for (uint32_t v : fin_lo) L = std::max(L, v);
    recheck_idx.clear();
    for (size_t e = 0; e < fin_cells.size(); ++e)
      if (fin_hi[e] >= L && fin_hi[e] != fin_lo[e]) recheck_idx.push_back(e);
    if (recheck_idx.empty()) { finalize(); return; }
    phase = PH_RECHECK;
    mode = RV_MODE_EXACT;
    cells.clear();
    for (size_t r : recheck_idx) cells.push_back(fin_cells[r]);
    note_request();
  }

  std::vector<uint32_t> cells_exact;

  int feed(const uint32_t* a, const uint32_t* b) {
    if (phase == PH_DONE) return -1;
    if (mode == RV_MODE_FINAL && (b == nullptr || a == nullptr) && !cells.empty()) return -1;
    if (a == nullptr && !cells.empty()) return -1;
    switch (phase) {
      case PH_L0: {
        if (mode == RV_MODE_FINAL) { enter_final(a, b); return 0; }  // levels == 1
        l0_cells = cells;
        l0_ub.assign(a, a + cells.size());
        // (1 - t_c)/2 of the full grid, cached (not aligned with a filtered list)
        const std::vector<double>* bg = excl.empty() ? grid_background(chain[0], eps) : nullptr;
        size_t s = l0_cells.empty() ? 0 : best_excess(0, l0_cells, l0_ub.data(),
                                                      bg ? bg->data() : nullptr);
        start_dive_or_bnb(s);
        return 0;
      }
      case PH_DIVE: {
        if (mode == RV_MODE_BOUND && cells.empty()) {
          // every block of the neighbourhood excluded: no dive bound (lb* = 0)
          lb_star = 0;
          if (l0_ext) { phase = PH_NEED_SURV; cells.clear(); } else { start_bnb(); }
          return 0;
        }
        if (mode == RV_MODE_BOUND) {
          size_t s = best_excess(level, cells, a);
          uint32_t pick = cells[s];
          cells = children(level, neighbourhood(level, pick));
          ++level;
          mode = mode_for(level);
          note_request();
        } else {
          lb_star = 0;
          for (size_t e = 0; e < cells.size(); ++e) lb_star = std::max<int64_t>(lb_star, b[e]);
          if (l0_ext) {  // the caller compacts the level-0 survivors (UB >= lb_star)
            phase = PH_NEED_SURV;
            cells.clear();
          } else {
            start_bnb();
          }
        }
        return 0;
      }
      case PH_BNB: {
        if (mode == RV_MODE_BOUND) {
          std::vector<uint32_t> surv;
          for (size_t e = 0; e < cells.size(); ++e)
            if ((int64_t)a[e] >= lb_star) surv.push_back(cells[e]);
          std::vector<uint32_t> ch = children(level, surv);
          const int64_t f = chain[level + 1] / chain[level];
          if (!redived && level >= 1 && !cells.empty() && (int64_t)ch.size() >= kRediveMin &&
              2 * (int64_t)ch.size() > (int64_t)cells.size() * f * f * f) {
            redived = true;
            redive_parent = level;
            redive_cells = cells;
            redive_ub.assign(a, a + cells.size());
            const uint32_t pick = cells[best_excess(level, cells, a)];
            phase = PH_REDIVE;
            cells = children(level, neighbourhood(level, pick));
            ++level;
            mode = mode_for(level);
            if (cells.empty()) { resume_bnb(); return 0; }
            note_request();
            return 0;
          }
          cells = std::move(ch);
          ++level;
          mode = mode_for(level);
          note_request();
        } else {
          enter_final(a, b);
        }
        return 0;
      }
      case PH_REDIVE: {
        if (mode == RV_MODE_BOUND) {
          const uint32_t pick = cells[best_excess(level, cells, a)];
          cells = children(level, neighbourhood(level, pick));
          ++level;
          mode = mode_for(level);
          if (cells.empty()) { resume_bnb(); return 0; }
          note_request();
        } else {
          for (size_t e = 0; e < cells.size(); ++e) lb_star = std::max<int64_t>(lb_star, b[e]);
          resume_bnb();
        }
        return 0;
      }
      case PH_RECHECK: {
        cells_exact.assign(a, a + cells.size());
        finalize();
        return 0;
      }
      default:
        return -1;
    }
  }
};

extern "C" {

int rv_plan_create(const int32_t* chain, int32_t chain_len, int32_t levels, int64_t n, double eps,
                   double guard, rv_plan** out) {
  return rv_plan_create_ex(chain, chain_len, levels, n, eps, guard, nullptr, 0, 0.0, out);
}

int rv_plan_create_ex(const int32_t* chain, int32_t chain_len, int32_t levels, int64_t n,
                      double eps, double guard, const double* excl_q, int32_t n_excl, double rho,
                      rv_plan** out) {
  if (!out) return -1;
  *out = nullptr;
  if (!chain || chain_len < 1 || chain_len > RV_MAX_CHAIN || n < 1) return -1;
  if (!(eps > 0.0) || !(eps < 3.141592653589793) || !(guard >= 0.0)) return -1;
  for (int l = 0; l < chain_len; ++l) {
    if (chain[l] < 1 || chain[l] > 1625) return -1;
    if (l > 0 && chain[l] % chain[l - 1] != 0) return -1;
  }
  if (levels == 0) levels = chain_len < 5 ? chain_len : 5;
  if (levels < 1 || levels > chain_len) return -1;
  rv_plan* p = new rv_plan();
  p->chain.assign(chain + (chain_len - levels), chain + chain_len);
  p->n = n;
  p->eps = eps;
  p->guard = guard;
  p->phase = PH_L0;
  p->level = 0;
  p->mode = p->mode_for(0);
  if (n_excl < 0 || (n_excl > 0 && (!excl_q || !(rho >= 0.0) || !(rho <= 3.141592653589793)))) {
    delete p;
    return -1;
  }
  for (int32_t e = 0; e < n_excl; ++e) {
    std::array<double, 4> q{excl_q[4 * e], excl_q[4 * e + 1], excl_q[4 * e + 2], excl_q[4 * e + 3]};
    const double nq = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(nq > 0.0)) { delete p; return -1; }
    for (double& v : q) v /= nq;
    p->excl.push_back(q);
  }
  p->rho = rho;
  p->cos_half_rho = std::cos(rho / 2.0);
  p->cells = grid_cache(p->chain[0]).cand;
  p->drop_excluded(0, p->cells);
  p->note_request();
  *out = p;
  return 0;
}

void rv_plan_destroy(rv_plan* p) { delete p; }

int rv_plan_request(const rv_plan* p, int32_t* B, int32_t* mode, int64_t* m, const uint32_t** lins) {
  if (!p || p->phase == PH_DONE || p->phase == PH_NEED_SURV) return 0;
  if (B) *B = p->chain[p->level];
  if (mode) *mode = p->mode;
  if (m) *m = (int64_t)p->cells.size();
  if (lins) *lins = p->cells.data();
  return 1;
}

int rv_plan_feed_l0_start(rv_plan* p, int64_t start) {
  if (!p || p->phase != PH_L0 || p->mode != RV_MODE_BOUND) return -1;
  if (start < 0 || start >= (int64_t)p->cells.size()) return -1;
  p->l0_cells = p->cells;
  p->l0_ub.clear();
  p->l0_ext = true;
  p->start_dive((size_t)start);
  return 0;
}

int rv_plan_needs_l0_survivors(const rv_plan* p, int64_t* lb_star) {
  if (!p || p->phase != PH_NEED_SURV) return 0;
  if (lb_star) *lb_star = p->lb_star;
  return 1;
}

int rv_plan_feed_l0_survivors(rv_plan* p, const int32_t* idx, int64_t k) {
  if (!p || p->phase != PH_NEED_SURV || k < 0 || (k > 0 && !idx)) return -1;
  std::vector<uint32_t> surv;
  surv.reserve(k);
  for (int64_t e = 0; e < k; ++e) {
    if (idx[e] < 0 || idx[e] >= (int64_t)p->l0_cells.size()) return -1;
    surv.push_back(p->l0_cells[idx[e]]);
  }
  p->start_bnb_from(surv);
  return 0;
}

int rv_plan_request_is_full_grid(const rv_plan* p) {
  return p && p->phase == PH_L0 && p->excl.empty() ? 1 : 0;
}

int rv_plan_feed(rv_plan* p, const uint32_t* cnt_a, const uint32_t* cnt_b) {
  if (!p) return -1;
  return p->feed(cnt_a, cnt_b);
}

const double* rv_plan_l0_background(int32_t B, double eps, int64_t* m) {
  const std::vector<double>* bg = grid_background(B, eps);
  if (m) *m = bg ? (int64_t)bg->size() : 0;
  return bg ? bg->data() : nullptr;
}

int rv_plan_get_result(const rv_plan* p, rv_plan_result* out) {
  if (!p || !out || p->phase != PH_DONE) return -1;
  *out = p->res;
  return 0;
}

void rv_shard_range(int64_t m, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
  if (world < 1) world = 1;
  *begin = m * rank / world;
  *end = m * (rank + 1) / world;
}

int64_t rv_grid_candidates(int32_t B, uint32_t* out, int64_t cap) {
  if (B < 1 || B > 1625) return -1;
  int64_t m = 0;
  for (int32_t i = 0; i < B; ++i)
    for (int32_t j = 0; j < B; ++j)
      for (int32_t k = 0; k < B; ++k)
        if (rv::is_candidate(B, i, j, k)) {
          if (out && m < cap) out[m] = rv::ijk_to_lin(i, j, k, B);
          ++m;
        }
  return m;
}

int64_t rv_cull_groups(int32_t B0, int32_t gi, int32_t gj, int32_t gk, int32_t* group_of,
                       int32_t* goff, int32_t* gmem) {
  if (B0 < 1 || B0 > 1625 || gi < 1 || gj < 1 || gk < 1) return -1;
  const int64_t m0 = rv_grid_candidates(B0, nullptr, 0);
  std::vector<uint32_t> rows((size_t)m0);
  rv_grid_candidates(B0, rows.data(), m0);
  // group key of a row -> group id, numbered by first appearance in row (lin) order
  std::unordered_map<int64_t, int32_t> id;
  std::vector<int32_t> g_of((size_t)m0), size;
  for (int64_t a = 0; a < m0; ++a) {
    int32_t i, j, k;
    rv::lin_to_ijk(rows[a], B0, i, j, k);
    const int64_t key = ((int64_t)(i / gi) * B0 + j / gj) * B0 + k / gk;
    auto it = id.find(key);
    if (it == id.end()) {
      it = id.emplace(key, (int32_t)size.size()).first;
      size.push_back(0);
    }
    g_of[a] = it->second;
    ++size[it->second];
  }
  const int64_t G = (int64_t)size.size();
  std::vector<int32_t> off((size_t)G + 1, 0);
  for (int64_t g = 0; g < G; ++g) off[g + 1] = off[g] + size[g];
  if (group_of) std::copy(g_of.begin(), g_of.end(), group_of);
  if (goff) std::copy(off.begin(), off.end(), goff);
  if (gmem) {
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int64_t a = 0; a < m0; ++a) gmem[fill[g_of[a]]++] = (int32_t)a;  // ascending rows
  }
  return G;
}

int rv_cull_partition(int32_t B0, int32_t gi, int32_t gj, int32_t gk, int32_t world,
                      int64_t* slice, int64_t* gslice) {
  if (world < 1 || !slice || !gslice) return -1;
  const int64_t G = rv_cull_groups(B0, gi, gj, gk, nullptr, nullptr, nullptr);
  if (G < 0) return -1;
  const int64_t m0 = rv_grid_candidates(B0, nullptr, 0);
  std::vector<uint32_t> rows((size_t)m0);
  rv_grid_candidates(B0, rows.data(), m0);
  std::vector<int32_t> g_of((size_t)m0), goff((size_t)G + 1), gmem((size_t)m0);
  rv_cull_groups(B0, gi, gj, gk, g_of.data(), goff.data(), gmem.data());
  // a run of consecutive rows that holds whole groups: the i-slab of gi rows when gi > 1 (the
  // rows of i .. i+gi-1 are contiguous in lin order), else the (i, j / gj) row slab, else the
  // (i, j, k / gk) run
  auto slab = [&](int64_t a) -> int64_t {
    int32_t i, j, k;
    rv::lin_to_ijk(rows[a], B0, i, j, k);
    if (gi > 1) return i / gi;
    if (gj > 1) return (int64_t)i * B0 + j / gj;
    return ((int64_t)i * B0 + j) * B0 + k / gk;
  };
  slice[0] = 0;
  for (int32_t r = 1; r < world; ++r) {
    int64_t a = std::max<int64_t>(slice[r - 1], (m0 * r + world - 1) / world);
    while (a < m0 && a > 0 && slab(a) == slab(a - 1)) ++a;
    slice[r] = std::min<int64_t>(a, m0);
  }
  slice[world] = m0;
  gslice[0] = 0;
  for (int32_t r = 1; r <= world; ++r) {
    int64_t g = gslice[r - 1];
    while (g < G && gmem[goff[g]] < slice[r]) ++g;
    gslice[r] = g;
  }
  return 0;
}

}  // extern "C"
