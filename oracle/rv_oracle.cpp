// ============================================================================
//  rv_oracle.cpp -- ORACLE.  TEST INFRASTRUCTURE ONLY.
//
//  A plain, slow, single-threaded, double-precision CPU implementation of what
//  the hot path computes, written from the paper (arXiv 2506.11547, PAPER.md)
//  and SURVEY.md §8(c)'s readings.  Only tests/, __graft_entry__.smoke() and
//  bench.py's cpu_baseline / --impl reference legs may load this library.  It
//  shares no code, header, table or constant generator with the CUDA path
//  (paper_2506_11547_b200/csrc) and neither side includes the other.
//
//  Citation keys:  P:n = PAPER.md line n;  S:n = SPEC.md line n.
//
//  Definition computed:
//    1. x̂ = x/‖x‖, ŷ = y/‖y‖ in double ("normalize all data again").
//    2. vote statistic s_i(q) = ŷ_iᵀ R(q) x̂_i with R(q) exactly the matrix of
//       P:955-961  (R a = b  <=>  bᵀ R a = 1).  The oracle deliberately
//       does NOT use the 10-entry quadratic form K_i that the GPU uses.
//    3. inlier test s_i(q) >= tau, tau = cos(eps)  (angle(R x̂, ŷ) <= eps).
//    4. cells: the paper's accumulator grid, the cube [-1,1]^3 divided into
//       B^3 blocks (Alg. 1 line 1; eps_grid = 1/180 -> B = 360);
//       a block is a candidate iff it meets the closed unit ball (hemisphere +
//       equator); its rotation is q_c = P'(p_c) at the block centre
//       ("the center of the block ... is returned").
//    5. count(c) = #{i : s_i(q_c) >= tau};  winner = argmax count, ties -> the
//       lowest linear index lin = (i*B + j)*B + k.
//    6. refinement (Horn P:125-150): I_r = {i : s_i(q_{r-1}) >= tau},
//       S_r = sum_{I_r} M_i with M_i the Appendix-A matrix,
//       q_r = eigenvector of the largest eigenvalue (cyclic Jacobi), then the
//       hemisphere representative (q3 <= 0).  Mask at the final q.
//
//  Two search modes return the identical (cell, count):
//    exhaustive : every candidate cell at the finest resolution.
//    certified  : depth-first branch and bound over the nested resolution
//                 chain; a coarse block's upper bound counts
//                 s_i(q_c) >= cos(min(pi, eps + r(c))) - guard with
//                 r(c) = 2 * (2/(1+dmin^2)) * sqrt(3)/B  (conformal factor of
//                 P' maximised over the block, times the half diagonal, times 2
//                 for the quaternion->rotation angle); a block is expanded
//                 unless its bound is strictly below the best exact count.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

const double kPi = 3.14159265358979323846;

struct Data {  // normalised correspondences, SoA so the count loop vectorises
  std::vector<double> x0, x1, x2, y0, y1, y2;
  int64_t n = 0;
};

// returns -1 when every row normalises, else the first bad row
int64_t load_normalized(const float* x, const float* y, int64_t n, Data& d) {
  d.n = n;
  d.x0.resize(n); d.x1.resize(n); d.x2.resize(n);
  d.y0.resize(n); d.y1.resize(n); d.y2.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    double a0 = x[3 * i], a1 = x[3 * i + 1], a2 = x[3 * i + 2];
    double b0 = y[3 * i], b1 = y[3 * i + 1], b2 = y[3 * i + 2];
    double na = std::sqrt(a0 * a0 + a1 * a1 + a2 * a2);
    double nb = std::sqrt(b0 * b0 + b1 * b1 + b2 * b2);
    if (!(na > 0.0) || !(nb > 0.0) || !std::isfinite(na) || !std::isfinite(nb)) return i;
    d.x0[i] = a0 / na; d.x1[i] = a1 / na; d.x2[i] = a2 / na;
    d.y0[i] = b0 / nb; d.y1[i] = b1 / nb; d.y2[i] = b2 / nb;
  }
  return -1;
}

}  // namespace

extern "C" {

// ---- rotation algebra -------------------------------------------------------

// R(q), scalar-first q = [q0,q1,q2,q3], row-major R[3][3].
void or_quat_to_R(const double* q, double* R) {
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

// s = bᵀ R(q) a.
double or_vote_stat(const double* q, const double* a, const double* b) {
  double R[9];
  or_quat_to_R(q, R);
  double ra0 = R[0] * a[0] + R[1] * a[1] + R[2] * a[2];
  double ra1 = R[3] * a[0] + R[4] * a[1] + R[5] * a[2];
  double ra2 = R[6] * a[0] + R[7] * a[1] + R[8] * a[2];
  return b[0] * ra0 + b[1] * ra1 + b[2] * ra2;
}

// Stereographic projection P(q) and its inverse P'(p).
void or_project(const double* q, double* p) {
  double d = 1.0 - q[3];
  p[0] = q[0] / d; p[1] = q[1] / d; p[2] = q[2] / d;
}
void or_unproject(const double* p, double* q) {
  double pp = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
  double d = 1.0 + pp;
  q[0] = 2.0 * p[0] / d; q[1] = 2.0 * p[1] / d; q[2] = 2.0 * p[2] / d;
  q[3] = (pp - 1.0) / d;
}

// Hemisphere representative (rule of S:361-369): q3 < 0 kept, q3 > 0
// negated; |q3| <= 1e-15: the first nonzero of (q0,q1,q2) made positive.
void or_canonicalize(double* q) {
  bool flip;
  if (q[3] < -1e-15) flip = false;
  else if (q[3] > 1e-15) flip = true;
  else {
    flip = false;
    for (int a = 0; a < 3; ++a)
      if (q[a] != 0.0) { flip = q[a] < 0.0; break; }
  }
  if (flip) for (int a = 0; a < 4; ++a) q[a] = -q[a];
}

// Appendix A matrix M = A(a)ᵀ B(b) with qᵀ M q = bᵀ R(q) a.
void or_constraint_M(const double* a, const double* b, double* M) {
  const double a1 = a[0], a2 = a[1], a3 = a[2];
  const double b1 = b[0], b2 = b[1], b3 = b[2];
  const double A[16] = {0, -a1, -a2, -a3,
                        a1, 0, a3, -a2,
                        a2, -a3, 0, a1,
                        a3, a2, -a1, 0};
  const double Bm[16] = {0, -b1, -b2, -b3,
                         b1, 0, -b3, b2,
                         b2, b3, 0, -b1,
                         b3, -b2, b1, 0};
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
      for (int k = 0; k < 4; ++k) s += A[k * 4 + r] * Bm[k * 4 + c];  // (Aᵀ)_{rk} B_{kc}
      M[r * 4 + c] = s;
    }
}

// Symmetric 4x4 eigen-decomposition by cyclic Jacobi rotations (textbook,
// S:216 design decision).  evals sorted descending; evecs column j (row-major
// evecs[r*4+j]) belongs to evals[j].  Returns the number of sweeps.
int or_sym_eig4(const double* S_in, double* evals, double* evecs) {
  double a[4][4], v[4][4];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      a[r][c] = 0.5 * (S_in[r * 4 + c] + S_in[c * 4 + r]);
      v[r][c] = (r == c) ? 1.0 : 0.0;
    }
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) {
        tot += a[r][c] * a[r][c];
        if (r != c) off += a[r][c] * a[r][c];
      }
    if (off <= 1e-36 * tot || off == 0.0) break;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 4; ++q) {
        if (a[p][q] == 0.0) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 4; ++k) {  // A <- A J  (columns p,q)
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 4; ++k) {  // A <- Jᵀ A  (rows p,q)
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 4; ++k) {  // V <- V J
          double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int idx[4] = {0, 1, 2, 3};
  std::sort(idx, idx + 4, [&](int i, int j) { return a[i][i] > a[j][j]; });
  for (int j = 0; j < 4; ++j) {
    evals[j] = a[idx[j]][idx[j]];
    for (int r = 0; r < 4; ++r) evecs[r * 4 + j] = v[r][idx[j]];
  }
  return sweep;
}

// ---- the accumulator grid --------------------------------------------

// centre of block (i,j,k) of the B^3 division of [-1,1]^3
void or_cell_center(int32_t B, int64_t i, int64_t j, int64_t k, double* p) {
  p[0] = -1.0 + (2.0 * i + 1.0) / B;
  p[1] = -1.0 + (2.0 * j + 1.0) / B;
  p[2] = -1.0 + (2.0 * k + 1.0) / B;
}

// (B * distance from the origin to the block)^2, exact in integers.
int64_t or_cell_dmin2_scaled(int32_t B, int64_t i, int64_t j, int64_t k) {
  int64_t idx[3] = {i, j, k}, s = 0;
  for (int a = 0; a < 3; ++a) {
    int64_t lo = 2 * idx[a] - B, hi = 2 * idx[a] + 2 - B;  // B * block bounds
    int64_t d = lo > 0 ? lo : (hi < 0 ? -hi : 0);
    s += d * d;
  }
  return s;  // = (B * dmin)^2, since lo/hi are the block bounds times B
}

// block meets the closed unit ball (hemisphere incl. equator)
int32_t or_cell_is_candidate(int32_t B, int64_t i, int64_t j, int64_t k) {
  return or_cell_dmin2_scaled(B, i, j, k) <= (int64_t)B * B ? 1 : 0;
}

// r(c): bound on the rotation angle between R(q_c) and R(q) for any q = P'(p),
// p in the block (reading R6).
double or_cell_radius(int32_t B, int64_t i, int64_t j, int64_t k) {
  double dmin2 = (double)or_cell_dmin2_scaled(B, i, j, k) / ((double)B * B);
  return 2.0 * (2.0 / (1.0 + dmin2)) * std::sqrt(3.0) / B;
}

// cos(min(pi, eps + r(c))): the bound-level threshold before the guard
double or_cell_bound_threshold(int32_t B, int64_t lin, double eps) {
  int64_t i = lin / ((int64_t)B * B), j = (lin / B) % B, k = lin % B;
  double a = eps + or_cell_radius(B, i, j, k);
  return std::cos(a < kPi ? a : kPi);
}

void or_cell_quat(int32_t B, int64_t lin, double* q) {
  int64_t i = lin / ((int64_t)B * B), j = (lin / B) % B, k = lin % B;
  double p[3];
  or_cell_center(B, i, j, k, p);
  or_unproject(p, q);
}

// all candidate blocks of the B^3 grid, ascending lin.  Returns the count;
// writes at most cap entries.
int64_t or_candidates(int32_t B, uint32_t* out, int64_t cap) {
  int64_t m = 0;
  for (int64_t i = 0; i < B; ++i)
    for (int64_t j = 0; j < B; ++j)
      for (int64_t k = 0; k < B; ++k)
        if (or_cell_is_candidate(B, i, j, k)) {
          if (m < cap) out[m] = (uint32_t)((i * B + j) * B + k);
          ++m;
        }
  return m;
}

// ---- counting -----------------------------------------------------------------

// counts of s_i(q) >= t and of |s_i(q) - t| < band, over normalised data.
static void count_one(const Data& d, const double* q, double t, double band,
                      uint32_t* cnt, uint32_t* nearc) {
  double R[9];
  or_quat_to_R(q, R);
  const double r0 = R[0], r1 = R[1], r2 = R[2], r3 = R[3], r4 = R[4], r5 = R[5],
               r6 = R[6], r7 = R[7], r8 = R[8];
  uint32_t c = 0, nr = 0;
  const double* x0 = d.x0.data(); const double* x1 = d.x1.data(); const double* x2 = d.x2.data();
  const double* y0 = d.y0.data(); const double* y1 = d.y1.data(); const double* y2 = d.y2.data();
  for (int64_t i = 0; i < d.n; ++i) {
    double s = y0[i] * (r0 * x0[i] + r1 * x1[i] + r2 * x2[i]) +
               y1[i] * (r3 * x0[i] + r4 * x1[i] + r5 * x2[i]) +
               y2[i] * (r6 * x0[i] + r7 * x1[i] + r8 * x2[i]);
    c += (s >= t) ? 1u : 0u;
  }
  if (nearc && band > 0.0)
    for (int64_t i = 0; i < d.n; ++i) {
      double s = y0[i] * (r0 * x0[i] + r1 * x1[i] + r2 * x2[i]) +
                 y1[i] * (r3 * x0[i] + r4 * x1[i] + r5 * x2[i]) +
                 y2[i] * (r6 * x0[i] + r7 * x1[i] + r8 * x2[i]);
      nr += (std::fabs(s - t) < band) ? 1u : 0u;
    }
  *cnt = c;
  if (nearc) *nearc = nr;
}

// Normalise fp32 [n][3] rows into double.  Returns -1 or the first bad row.
int64_t or_normalize(const float* v, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double a0 = v[3 * i], a1 = v[3 * i + 1], a2 = v[3 * i + 2];
    double na = std::sqrt(a0 * a0 + a1 * a1 + a2 * a2);
    if (!(na > 0.0) || !std::isfinite(na)) return i;
    out[3 * i] = a0 / na; out[3 * i + 1] = a1 / na; out[3 * i + 2] = a2 / na;
  }
  return -1;
}

// Per-cell counts with explicit thresholds thr[m] (double):
//   cnt[c]  = #{i : s_i(q_c) >= thr[c]},  nearc[c] = #{i : |s_i(q_c) - thr[c]| < band}.
// Returns -1 on success or the first row that cannot be normalised.
int64_t or_count_cells(const float* x, const float* y, int64_t n, int32_t B,
                       const uint32_t* lins, int64_t m, const double* thr, double band,
                       uint32_t* cnt, uint32_t* nearc) {
  Data d;
  int64_t bad = load_normalized(x, y, n, d);
  if (bad >= 0) return bad;
  for (int64_t c = 0; c < m; ++c) {
    double q[4];
    or_cell_quat(B, lins[c], q);
    count_one(d, q, thr[c], band, &cnt[c], nearc ? &nearc[c] : nullptr);
  }
  return -1;
}

// per-pair decisions s_i(q) >= t for an arbitrary q (bytes), plus s itself.
int64_t or_pair_stats(const float* x, const float* y, int64_t n, const double* q,
                      double* s_out) {
  Data d;
  int64_t bad = load_normalized(x, y, n, d);
  if (bad >= 0) return bad;
  for (int64_t i = 0; i < n; ++i) {
    double a[3] = {d.x0[i], d.x1[i], d.x2[i]}, b[3] = {d.y0[i], d.y1[i], d.y2[i]};
    s_out[i] = or_vote_stat(q, a, b);
  }
  return -1;
}

// ---- solve ------------------------------------------------------------------

struct or_result {
  double q[4];          // refined rotation, hemisphere representative
  double q_cell[4];     // rotation of the winning block centre
  uint32_t votes;       // count of the winning block
  uint32_t n_inliers;   // |{i : s_i(q) >= tau}| at the returned q
  int32_t cell[3];      // winning block (i,j,k) at the finest resolution
  int32_t flags;        // 1 refined, 2 degenerate
  int32_t B;            // finest resolution
  int32_t n_tied;       // number of finest blocks sharing the winning count
  uint64_t pair_evals;  // number of s_i(q_c) evaluations performed
  uint64_t cells_evaluated;
  uint32_t winner_near; // pairs at the winner with |s - tau| < 1e-12
  uint32_t pad;
};

namespace {

struct Search {
  const Data* d;
  std::vector<int32_t> chain;  // resolutions used (coarse -> fine)
  double eps, tau, guard;
  int64_t best = -1;
  uint32_t best_lin = 0;
  int32_t n_tied = 0;
  uint64_t pair_evals = 0, cells = 0;

  uint32_t eval(int32_t B, uint32_t lin, double t) {
    double q[4];
    or_cell_quat(B, lin, q);
    uint32_t c;
    count_one(*d, q, t, 0.0, &c, nullptr);
    pair_evals += (uint64_t)d->n;
    cells += 1;
    return c;
  }
  void offer(uint32_t lin, int64_t cnt) {  // exact count of a finest block
    if (cnt > best) { best = cnt; best_lin = lin; n_tied = 1; }
    else if (cnt == best) { ++n_tied; if (lin < best_lin) best_lin = lin; }
  }
  struct Node { uint32_t lin; int64_t ub; double excess; };

  // evaluate and order the candidate children of `parents` at level l
  std::vector<Node> expand(int l, const std::vector<uint32_t>& lins) {
    const int32_t B = chain[l];
    std::vector<Node> out;
    out.reserve(lins.size());
    for (uint32_t lin : lins) {
      double t = or_cell_bound_threshold(B, lin, eps);
      int64_t ub = eval(B, lin, t - guard);
      out.push_back({lin, ub, (double)ub - (double)d->n * (1.0 - t) / 2.0});
    }
    std::sort(out.begin(), out.end(), [](const Node& a, const Node& b) {
      return a.excess != b.excess ? a.excess > b.excess : a.lin < b.lin;
    });
    return out;
  }
  std::vector<uint32_t> children(int l, uint32_t lin) {  // level l -> l+1
    const int64_t B = chain[l], Bc = chain[l + 1], f = Bc / B;
    int64_t i = lin / (B * B), j = (lin / B) % B, k = lin % B;
    std::vector<uint32_t> out;
    for (int64_t a = 0; a < f; ++a)
      for (int64_t b = 0; b < f; ++b)
        for (int64_t c = 0; c < f; ++c) {
          int64_t ci = f * i + a, cj = f * j + b, ck = f * k + c;
          if (or_cell_is_candidate((int32_t)Bc, ci, cj, ck))
            out.push_back((uint32_t)((ci * Bc + cj) * Bc + ck));
        }
    return out;
  }
  void visit(int l, const std::vector<Node>& nodes) {
    const int last = (int)chain.size() - 1;
    for (const Node& nd : nodes) {
      if (nd.ub < best) continue;  // certified prune (ties kept)
      std::vector<uint32_t> ch = children(l, nd.lin);
      if (l + 1 == last) {
        for (uint32_t c : ch) offer(c, eval(chain[last], c, tau));
      } else {
        visit(l + 1, expand(l + 1, ch));
      }
    }
  }
};

}  // namespace

// Full solve.  chain[chain_len]: nested resolutions (each divides the next);
// levels in [1, chain_len] uses the last `levels` entries (0 -> min(5, len)).
// exhaustive != 0 ignores the chain and scans every finest candidate block.
// mask: n bytes (1 = inlier at the returned q) or NULL.
// Returns 0, -1 (bad arguments) or -2 (a row that cannot be normalised).
int32_t or_solve(const float* x, const float* y, int64_t n, double eps,
                 const int32_t* chain, int32_t chain_len, int32_t levels,
                 int32_t exhaustive, int32_t refine_rounds, double guard,
                 or_result* out, uint8_t* mask) {
  if (n < 2 || !(eps > 0.0) || !(eps < kPi) || chain_len < 1) return -1;
  if (levels == 0) levels = chain_len < 5 ? chain_len : 5;
  if (levels < 1 || levels > chain_len) return -1;
  for (int l = 1; l < chain_len; ++l)
    if (chain[l] % chain[l - 1] != 0) return -1;
  Data d;
  if (load_normalized(x, y, n, d) >= 0) return -2;
  std::memset(out, 0, sizeof(*out));

  Search S;
  S.d = &d;
  S.chain.assign(chain + (chain_len - levels), chain + chain_len);
  S.eps = eps;
  S.tau = std::cos(eps);
  S.guard = guard;
  const int32_t Bf = S.chain.back();

  if (exhaustive || levels == 1) {
    for (int64_t i = 0; i < Bf; ++i)
      for (int64_t j = 0; j < Bf; ++j)
        for (int64_t k = 0; k < Bf; ++k)
          if (or_cell_is_candidate(Bf, i, j, k)) {
            uint32_t lin = (uint32_t)((i * Bf + j) * Bf + k);
            S.offer(lin, S.eval(Bf, lin, S.tau));
          }
  } else {
    std::vector<uint32_t> top(0);
    int32_t B0 = S.chain[0];
    int64_t m0 = or_candidates(B0, nullptr, 0);
    top.resize(m0);
    or_candidates(B0, top.data(), m0);
    S.visit(0, S.expand(0, top));
  }

  out->votes = (uint32_t)S.best;
  out->B = Bf;
  out->cell[0] = (int32_t)(S.best_lin / ((uint32_t)Bf * Bf));
  out->cell[1] = (int32_t)((S.best_lin / Bf) % Bf);
  out->cell[2] = (int32_t)(S.best_lin % Bf);
  out->n_tied = S.n_tied;
  out->pair_evals = S.pair_evals;
  out->cells_evaluated = S.cells;

  double qc[4];
  or_cell_quat(Bf, S.best_lin, qc);
  {
    uint32_t c, nr;
    count_one(d, qc, S.tau, 1e-12, &c, &nr);
    out->winner_near = nr;
  }
  or_canonicalize(qc);
  std::memcpy(out->q_cell, qc, sizeof(qc));

  // ---- linear refinement on the inlier set (Horn P:125-150) ----
  double q[4];
  std::memcpy(q, qc, sizeof(q));
  for (int r = 0; r < refine_rounds; ++r) {
    double S4[16] = {0};
    int64_t ni = 0;
    for (int64_t i = 0; i < n; ++i) {
      double a[3] = {d.x0[i], d.x1[i], d.x2[i]}, b[3] = {d.y0[i], d.y1[i], d.y2[i]};
      if (or_vote_stat(q, a, b) >= S.tau) {
        double M[16];
        or_constraint_M(a, b, M);
        for (int e = 0; e < 16; ++e) S4[e] += M[e];
        ++ni;
      }
    }
    if (ni < 2) { out->flags |= 2; break; }
    double ev[4], V[16];
    or_sym_eig4(S4, ev, V);
    if (ev[0] - ev[1] <= 1e-12 * std::fabs(ev[0])) { out->flags |= 2; break; }
    double nq = 0.0;
    for (int a = 0; a < 4; ++a) nq += V[a * 4] * V[a * 4];
    nq = std::sqrt(nq);
    for (int a = 0; a < 4; ++a) q[a] = V[a * 4] / nq;
    or_canonicalize(q);
    out->flags |= 1;
  }
  std::memcpy(out->q, q, sizeof(q));
  uint32_t ninl = 0;
  for (int64_t i = 0; i < n; ++i) {
    double a[3] = {d.x0[i], d.x1[i], d.x2[i]}, b[3] = {d.y0[i], d.y1[i], d.y2[i]};
    uint8_t in = or_vote_stat(q, a, b) >= S.tau ? 1 : 0;
    ninl += in;
    if (mask) mask[i] = in;
  }
  out->n_inliers = ninl;
  return 0;
}

// Refinement alone from a given start rotation (same arithmetic as in or_solve).
int32_t or_refine(const float* x, const float* y, int64_t n, double eps, const double* q0,
                  int32_t rounds, double* q_out, int32_t* flags, uint8_t* mask) {
  Data d;
  if (load_normalized(x, y, n, d) >= 0) return -2;
  const double tau = std::cos(eps);
  double q[4];
  std::memcpy(q, q0, sizeof(q));
  const double nq0 = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (int a = 0; a < 4; ++a) q[a] /= nq0;  // a rotation is a unit quaternion
  or_canonicalize(q);
  int32_t fl = 0;
  for (int r = 0; r < rounds; ++r) {
    double S4[16] = {0};
    int64_t ni = 0;
    for (int64_t i = 0; i < n; ++i) {
      double a[3] = {d.x0[i], d.x1[i], d.x2[i]}, b[3] = {d.y0[i], d.y1[i], d.y2[i]};
      if (or_vote_stat(q, a, b) >= tau) {
        double M[16];
        or_constraint_M(a, b, M);
        for (int e = 0; e < 16; ++e) S4[e] += M[e];
        ++ni;
      }
    }
    if (ni < 2) { fl |= 2; break; }
    double ev[4], V[16];
    or_sym_eig4(S4, ev, V);
    if (ev[0] - ev[1] <= 1e-12 * std::fabs(ev[0])) { fl |= 2; break; }
    double nq = 0.0;
    for (int a = 0; a < 4; ++a) nq += V[a * 4] * V[a * 4];
    nq = std::sqrt(nq);
    for (int a = 0; a < 4; ++a) q[a] = V[a * 4] / nq;
    or_canonicalize(q);
    fl |= 1;
  }
  std::memcpy(q_out, q, sizeof(q));
  if (flags) *flags = fl;
  if (mask)
    for (int64_t i = 0; i < n; ++i) {
      double a[3] = {d.x0[i], d.x1[i], d.x2[i]}, b[3] = {d.y0[i], d.y1[i], d.y2[i]};
      mask[i] = or_vote_stat(q, a, b) >= tau ? 1 : 0;
    }
  return 0;
}


// ---- NEXT-4: the paper's Algorithm 1 (sampled voting), P:483-503 -------------------------
// The quaternion circle of (a, b): q(alpha) = q_b1 cos(alpha/2) + q_b2 sin(alpha/2) with
// q_b1 the quaternion of the minimal geodesic rotation a -> b, [cos(theta/2), sin(theta/2) c],
// c = a x b / |a x b|, and q_b2 = [-b.q123, q0 b + b x q123].
// Readings (R13-R15): cos/sin(theta/2) by the half-angle identities
// sqrt((1 +- a.b)/2) (theta = arccos(a.b) in [0, pi]); when a x b = 0 (a = +-b, where the
// paper leaves c open) c = normalize(a x e_k), e_k the axis of the smallest |a_k| (lowest k
// on ties); alpha_j = -pi + 2 pi j / J, j = 0..J-1 ("discretizing [-pi, pi] uniformly",
// Alg. 1 line 2; alpha = pi is the antipode of alpha = -pi, the same rotation, so it is not
// sampled twice); each sample is taken to the half sphere q3 <= 0 (negated if q3 > 0),
// projected by P and binned at step 2/B over [-1, 1]^3 (Alg. 1 line 1; B = 360,
// P:635), index clamped to [0, B-1]; every sample adds 1 (Alg. 1 line 8).
void or_alg1_basis(const double* a, const double* b, double* qb1, double* qb2) {
  double d = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
  if (d > 1.0) d = 1.0;
  if (d < -1.0) d = -1.0;
  const double ch = std::sqrt((1.0 + d) / 2.0), sh = std::sqrt((1.0 - d) / 2.0);
  double c[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
  double nc = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
  if (nc == 0.0) {
    int k = 0;
    for (int t = 1; t < 3; ++t)
      if (std::fabs(a[t]) < std::fabs(a[k])) k = t;
    double e[3] = {0.0, 0.0, 0.0};
    e[k] = 1.0;
    c[0] = a[1] * e[2] - a[2] * e[1];
    c[1] = a[2] * e[0] - a[0] * e[2];
    c[2] = a[0] * e[1] - a[1] * e[0];
    nc = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
  }
  qb1[0] = ch;
  for (int t = 0; t < 3; ++t) qb1[1 + t] = sh * (c[t] / nc);
  const double* v = qb1 + 1;  // q123
  qb2[0] = -(b[0] * v[0] + b[1] * v[1] + b[2] * v[2]);
  const double bxv[3] = {b[1] * v[2] - b[2] * v[1], b[2] * v[0] - b[0] * v[2],
                         b[0] * v[1] - b[1] * v[0]};
  for (int t = 0; t < 3; ++t) qb2[1 + t] = qb1[0] * b[t] + bxv[t];
}

// the bin of every sample: bins[i*J + j] = lin of sample j of correspondence i
int64_t or_alg1_bins(const float* x, const float* y, int64_t n, int32_t B, int32_t J,
                     int64_t* bins) {
  if (B < 1 || J < 1) return -1;
  const double pi = 3.14159265358979323846;
  std::vector<double> cs(J), sn(J);
  for (int32_t j = 0; j < J; ++j) {
    const double half = (-pi + 2.0 * pi * (double)j / (double)J) / 2.0;
    cs[j] = std::cos(half);
    sn[j] = std::sin(half);
  }
  const double hb = (double)B / 2.0;
  for (int64_t i = 0; i < n; ++i) {
    double a[3], b[3];
    if (or_normalize(x + 3 * i, 1, a) != -1 || or_normalize(y + 3 * i, 1, b) != -1) return -2;
    double qb1[4], qb2[4];
    or_alg1_basis(a, b, qb1, qb2);
    for (int32_t j = 0; j < J; ++j) {
      double q[4];
      for (int t = 0; t < 4; ++t) q[t] = qb1[t] * cs[j] + qb2[t] * sn[j];
      if (q[3] > 0.0)
        for (int t = 0; t < 4; ++t) q[t] = -q[t];
      const double den = 1.0 - q[3];
      int64_t idx[3];
      for (int t = 0; t < 3; ++t) {
        const double pt = q[t] / den;
        int64_t v = (int64_t)std::floor((pt + 1.0) * hb);
        if (v < 0) v = 0;
        if (v > B - 1) v = B - 1;
        idx[t] = v;
      }
      bins[i * J + j] = (idx[0] * B + idx[1]) * B + idx[2];
    }
  }
  return 0;
}

// Algorithm 1 end to end: the dense B^3 accumulator, its maximum (ties -> lowest lin) and the
// block centre's rotation (hemisphere representative).
int64_t or_alg1_solve(const float* x, const float* y, int64_t n, int32_t B, int32_t J,
                      int64_t* lin_out, uint32_t* votes_out, double* q_out) {
  std::vector<int64_t> bins((size_t)n * J);
  if (int64_t rc = or_alg1_bins(x, y, n, B, J, bins.data())) return rc;
  std::vector<uint32_t> acc((size_t)B * B * B, 0u);
  for (int64_t v : bins) ++acc[(size_t)v];
  int64_t best = 0;
  for (int64_t e = 1; e < (int64_t)acc.size(); ++e)
    if (acc[(size_t)e] > acc[(size_t)best]) best = e;
  *lin_out = best;
  *votes_out = acc[(size_t)best];
  const int64_t i = best / ((int64_t)B * B), j = (best / B) % B, k = best % B;
  double p[3];
  or_cell_center(B, i, j, k, p);
  or_unproject(p, q_out);
  or_canonicalize(q_out);
  return 0;
}


// ---- NEXT-3: rigid pose front end ------------------------------------------------
// Pairs: for every i < j (lexicographic order) m = x_i - x_j, n = y_i - y_j,
// computed in double (exact for fp32 inputs) and kept iff both are non-zero and the
// rotation-invariant length check |‖m‖ - ‖n‖| <= mu_t holds (mu_t is a parameter,
// the paper does not give it: reading R17).  Kept pairs are returned as fp32 (the rotation
// vote's input format) with their (i, j).  Returns the number kept (writes up to cap).
int64_t or_rigid_pairs(const float* x, const float* y, int64_t n, double mu_t, int64_t cap,
                       int64_t* ij, float* m_out, float* n_out) {
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      double m[3], d[3];
      for (int t = 0; t < 3; ++t) {
        m[t] = (double)x[3 * i + t] - (double)x[3 * j + t];
        d[t] = (double)y[3 * i + t] - (double)y[3 * j + t];
      }
      const double lm = std::sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
      const double ld = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
      if (!(lm > 0.0) || !(ld > 0.0) || !(std::fabs(lm - ld) <= mu_t)) continue;
      if (k < cap) {
        ij[2 * k] = i;
        ij[2 * k + 1] = j;
        for (int t = 0; t < 3; ++t) {
          m_out[3 * k + t] = (float)m[t];
          n_out[3 * k + t] = (float)d[t];
        }
      }
      ++k;
    }
  return k;
}

// Translation vote: t_i = y_i - R(q) x_i (double, R(q) of P:955-961) for every
// correspondence, binned on [lo, hi)^3 at `step` ([-5,5]^3, 0.025) with
// index floor((t - lo) * (1/step)); candidates outside the domain do not vote (R17).  Winner:
// the fullest bin, ties -> lowest lin; t_out = its centre, t_mean = the mean of its
// candidates.  Returns 0, or -1 when no candidate falls in the domain.
int64_t or_translation_vote(const float* x, const float* y, int64_t n, const double* q,
                            double lo, double hi, double step, int64_t* lin_out,
                            uint32_t* votes_out, double* t_out, double* t_mean) {
  double R[9];
  or_quat_to_R(q, R);
  const double inv = 1.0 / step;
  const int64_t Bt = (int64_t)std::llround((hi - lo) * inv);
  std::vector<int64_t> bins;
  std::vector<double> ts;
  for (int64_t i = 0; i < n; ++i) {
    const double a[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    double t[3];
    bool ok = true;
    int64_t idx[3];
    for (int r = 0; r < 3; ++r) {
      const double ra = R[3 * r] * a[0] + R[3 * r + 1] * a[1] + R[3 * r + 2] * a[2];
      t[r] = (double)y[3 * i + r] - ra;
      const double f = std::floor((t[r] - lo) * inv);
      if (!(f >= 0.0) || !(f < (double)Bt)) ok = false;
      idx[r] = ok ? (int64_t)f : 0;
    }
    if (!ok) continue;
    bins.push_back((idx[0] * Bt + idx[1]) * Bt + idx[2]);
    ts.insert(ts.end(), t, t + 3);
  }
  if (bins.empty()) return -1;
  std::vector<int64_t> sorted = bins;
  std::sort(sorted.begin(), sorted.end());
  int64_t best = sorted[0], bestc = 0;
  for (size_t a = 0; a < sorted.size();) {
    size_t b = a;
    while (b < sorted.size() && sorted[b] == sorted[a]) ++b;
    if ((int64_t)(b - a) > bestc) { bestc = (int64_t)(b - a); best = sorted[a]; }
    a = b;
  }
  *lin_out = best;
  *votes_out = (uint32_t)bestc;
  const int64_t id[3] = {best / (Bt * Bt), (best / Bt) % Bt, best % Bt};
  for (int r = 0; r < 3; ++r) t_out[r] = lo + ((double)id[r] + 0.5) * step;
  double sm[3] = {0, 0, 0};
  for (size_t e = 0; e < bins.size(); ++e)
    if (bins[e] == best)
      for (int r = 0; r < 3; ++r) sm[r] += ts[3 * e + r];
  for (int r = 0; r < 3; ++r) t_mean[r] = sm[r] / (double)bestc;
  return 0;
}

}  // extern "C"
