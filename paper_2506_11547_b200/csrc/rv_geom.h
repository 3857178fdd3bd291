// rv_geom.h -- grid geometry of the certified search, shared by the host planner
// and the CUDA kernels of librotvote (product code; independent of oracle/).
//
// Grid: the cube [-1,1]^3 cut into B^3 blocks (Alg. 1 line 1).
// Block (i,j,k) has lin = (i*B + j)*B + k, centre p = -1 + (2*(i,j,k)+1)/B, and is a
// candidate iff it meets the closed unit ball -- the stereographic image of the
// half quaternion sphere incl. the equator.  Its rotation is
// q_c = P'(p_c).
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define RV_HD __host__ __device__ __forceinline__
#else
#define RV_HD inline
#endif

namespace rv {

RV_HD void lin_to_ijk(uint32_t lin, int32_t B, int32_t& i, int32_t& j, int32_t& k) {
  const uint32_t b = (uint32_t)B;
  k = (int32_t)(lin % b);
  uint32_t r = lin / b;
  j = (int32_t)(r % b);
  i = (int32_t)(r / b);
}

RV_HD uint32_t ijk_to_lin(int32_t i, int32_t j, int32_t k, int32_t B) {
  return ((uint32_t)i * (uint32_t)B + (uint32_t)j) * (uint32_t)B + (uint32_t)k;
}

// (B * distance from the origin to the block)^2, exact integer arithmetic:
// per axis the block spans [(2i-B)/B, (2i+2-B)/B].
RV_HD int64_t dmin2_scaled(int32_t B, int32_t i, int32_t j, int32_t k) {
  int64_t s = 0;
  const int32_t v[3] = {i, j, k};
  for (int a = 0; a < 3; ++a) {
    int64_t lo = 2 * (int64_t)v[a] - B, hi = lo + 2;
    int64_t d = lo > 0 ? lo : (hi < 0 ? -hi : 0);
    s += d * d;
  }
  return s;
}

RV_HD bool is_candidate(int32_t B, int32_t i, int32_t j, int32_t k) {
  return dmin2_scaled(B, i, j, k) <= (int64_t)B * B;
}

// Centre of block (i,j,k) inside the closed unit ball (its rotation lies in the q3 <= 0
// hemisphere proper); used by the dive heuristic only.
RV_HD bool centre_inside(int32_t B, uint32_t lin) {
  int32_t i, j, k;
  lin_to_ijk(lin, B, i, j, k);
  const int64_t a = 2 * (int64_t)i + 1 - B, b = 2 * (int64_t)j + 1 - B, c = 2 * (int64_t)k + 1 - B;
  return a * a + b * b + c * c <= (int64_t)B * B;
}

// Reading R6: every rotation of the block lies within rotation angle
//   r(c) = 2 * (2 / (1 + dmin^2)) * sqrt(3) / B
// of R(q_c): the half diagonal sqrt(3)/B times the largest conformal factor of P'
// over the block (geodesic length on S^3), times 2 (quaternion angle -> rotation angle).
RV_HD double bound_radius(int32_t B, int32_t i, int32_t j, int32_t k) {
  const double d2 = (double)dmin2_scaled(B, i, j, k) / ((double)B * (double)B);
  return 4.0 * 1.7320508075688772 / ((double)B * (1.0 + d2));
}

// cos(min(pi, eps + r(c))): any inlier of any rotation in the block has at least
// this vote statistic at the block centre (triangle inequality on angles).
RV_HD double bound_threshold(int32_t B, int32_t i, int32_t j, int32_t k, double eps) {
  double a = eps + bound_radius(B, i, j, k);
  return cos(a < 3.141592653589793 ? a : 3.141592653589793);
}

// q_c = P'(p_c), P:417 (inverse stereographic projection from the pole [0,0,0,1]).
RV_HD void cell_quat(int32_t B, int32_t i, int32_t j, int32_t k, double q[4]) {
  const double inv = 1.0 / (double)B;
  const double px = -1.0 + (2.0 * i + 1.0) * inv;
  const double py = -1.0 + (2.0 * j + 1.0) * inv;
  const double pz = -1.0 + (2.0 * k + 1.0) * inv;
  const double pp = px * px + py * py + pz * pz;
  const double d = 1.0 / (1.0 + pp);
  q[0] = 2.0 * px * d;
  q[1] = 2.0 * py * d;
  q[2] = 2.0 * pz * d;
  q[3] = (pp - 1.0) * d;
}

// phi(q) for the 9-entry traceless form:  q^T K q = phi(q) . k  with
// k = [K00, K11, K22, K01, K02, K03, K12, K13, K23] and K33 = -(K00 + K11 + K22).
RV_HD void phi9(const double q[4], double f[9]) {
  const double q33 = q[3] * q[3];
  f[0] = q[0] * q[0] - q33;
  f[1] = q[1] * q[1] - q33;
  f[2] = q[2] * q[2] - q33;
  f[3] = 2.0 * q[0] * q[1];
  f[4] = 2.0 * q[0] * q[2];
  f[5] = 2.0 * q[0] * q[3];
  f[6] = 2.0 * q[1] * q[2];
  f[7] = 2.0 * q[1] * q[3];
  f[8] = 2.0 * q[2] * q[3];
}

// K_i of a correspondence: y^T R(q) x = q^T K q (equal to Appendix-A M):
//   K = [[x.y, (x cross y)^T], [x cross y, x y^T + y x^T - (x.y) I]].
RV_HD void k9_of(const double x[3], const double y[3], double k[9]) {
  const double d = x[0] * y[0] + x[1] * y[1] + x[2] * y[2];
  k[0] = d;
  k[1] = 2.0 * x[0] * y[0] - d;
  k[2] = 2.0 * x[1] * y[1] - d;
  k[3] = x[1] * y[2] - x[2] * y[1];
  k[4] = x[2] * y[0] - x[0] * y[2];
  k[5] = x[0] * y[1] - x[1] * y[0];
  k[6] = x[0] * y[1] + x[1] * y[0];
  k[7] = x[0] * y[2] + x[2] * y[0];
  k[8] = x[1] * y[2] + x[2] * y[1];
}

// NEXT-2 (several rotations, reading R16): the earlier peaks' block-centre rotations q[4e..4e+3],
// e < n, and the suppression angle rho.  A finest block is excluded iff |q_c . q_e| >= cos(rho/2)
// (its centre within rotation angle rho of a peak); a coarser block only when all of it is:
// angle(q_c, q_e) + r(c) <= rho - 1e-9 (r(c) as in the certified bound) -- the host planner's
// rule (rv_plan.cpp).  n = 0: nothing excluded.
struct Excl {
  const double* q = nullptr;
  int32_t n = 0;
  double rho = 0.0, cos_half_rho = 2.0;
};
RV_HD bool excl_dropped(const Excl& ex, int32_t B, uint32_t lin, bool finest) {
  if (ex.n == 0) return false;
  int32_t i, j, k;
  lin_to_ijk(lin, B, i, j, k);
  double q[4];
  cell_quat(B, i, j, k, q);
  const double r = finest ? 0.0 : bound_radius(B, i, j, k);
  for (int32_t e = 0; e < ex.n; ++e) {
    const double* qe = ex.q + 4 * e;
    const double d = fabs(q[0] * qe[0] + q[1] * qe[1] + q[2] * qe[2] + q[3] * qe[3]);
    if (finest) {
      if (d >= ex.cos_half_rho) return true;
    } else if (2.0 * acos(d < 1.0 ? d : 1.0) + r <= ex.rho - 1e-9) {
      return true;
    }
  }
  return false;
}
// the dive's preference: 2 = entirely outside every ball, 1 = centre outside, 0 = centre inside
RV_HD int excl_rank(const Excl& ex, int32_t B, uint32_t lin) {
  if (ex.n == 0) return 2;
  int32_t i, j, k;
  lin_to_ijk(lin, B, i, j, k);
  double q[4];
  cell_quat(B, i, j, k, q);
  const double r = bound_radius(B, i, j, k);
  int rank = 2;
  for (int32_t e = 0; e < ex.n; ++e) {
    const double* qe = ex.q + 4 * e;
    const double d = fabs(q[0] * qe[0] + q[1] * qe[1] + q[2] * qe[2] + q[3] * qe[3]);
    if (d >= ex.cos_half_rho) return 0;
    if (2.0 * acos(d < 1.0 ? d : 1.0) - r <= ex.rho) rank = 1;
  }
  return rank;
}

}  // namespace rv
