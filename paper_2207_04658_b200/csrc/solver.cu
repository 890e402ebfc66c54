// solver.cu -- the closed-form quantization-scheme solver, host
// code behind the C ABI (include/qmpm.h).  P:n = PAPER.md line n, S:n = SPEC.md line n.
//
//   qmpm_predict_error         Eq. 8: sigma_pred = sqrt(1/12 sum Delta_h^2 g_h)
//   qmpm_solve_error_bounded   Eq. 9 Lagrange solution + Algorithm 1 line 15
//                              (P:391): b_h = ceil(-log2(Delta_h / R_h))
//   qmpm_solve_memory_bounded  Eq. 7; closed form deferred to the paper's
//                              supplement, stationarity solution of S:342:
//                              Delta_h = c sqrt(P_h / g_h), b_h = floor(-log2(Delta_h / R_h))
// The gradient tally g_h (Eq. 8) comes from the caller (the adjoint simulation that
// produces it, Alg. 1 line 12, is SURVEY §8(f) row f3, not built).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "qmpm.h"

namespace qmpm {
void set_thread_error(const char* msg);  // api.cu: qmpm_last_error(NULL)
}

namespace {
qmpm_status bad(const char* msg) {
  qmpm::set_thread_error(msg);
  return QMPM_EINVAL;
}

qmpm_status check(uint32_t H, const double* P, const double* g, const double* R, int32_t b_min, int32_t b_max) {
  if (H == 0 || !P || !g || !R) return bad("solver: H == 0 or NULL array");
  if (b_min < 0 || b_max > 31 || b_min > b_max) return bad("solver: need 0 <= b_min <= b_max <= 31");
  for (uint32_t h = 0; h < H; ++h) {
    if (!(P[h] > 0.0) || !(g[h] >= 0.0) || !(R[h] > 0.0) || !std::isfinite(g[h]) || !std::isfinite(R[h]))
      return bad("solver: need P_h > 0, finite g_h >= 0, finite R_h > 0");
  }
  return QMPM_OK;
}

int32_t clampi(double v, int32_t lo, int32_t hi) {
  if (!(v > lo)) return lo;  // also NaN
  if (v > hi) return hi;
  return (int32_t)v;
}
}  // namespace

extern "C" {

qmpm_status qmpm_predict_error(uint32_t H, const double* delta, const double* g, double* sigma_out) {
  if (H == 0 || !delta || !g || !sigma_out) return bad("predict_error: NULL argument");
  double e = 0.0;
  for (uint32_t h = 0; h < H; ++h) e += delta[h] * delta[h] * g[h];
  *sigma_out = std::sqrt(e / 12.0);
  return QMPM_OK;
}

qmpm_status qmpm_solve_error_bounded(uint32_t H, const double* P, const double* g, const double* R, double z,
                                     double eps_err, int32_t b_min, int32_t b_max, double* delta_out,
                                     int32_t* bits_out) {
  qmpm_status rc = check(H, P, g, R, b_min, b_max);
  if (rc) return rc;
  if (!(eps_err > 0.0) || !(z != 0.0) || !std::isfinite(z)) return bad("solve_error_bounded: need eps > 0, z != 0");
  if (!delta_out || !bits_out) return bad("solve_error_bounded: NULL output");
  double sum_p = 0.0;
  for (uint32_t h = 0; h < H; ++h) sum_p += P[h];
  const double ez2 = (eps_err * z) * (eps_err * z);
  for (uint32_t h = 0; h < H; ++h) {
    if (g[h] == 0.0) {  // does not enter E[dz]: the smallest width
      delta_out[h] = INFINITY;
      bits_out[h] = b_min;
      continue;
    }
    const double d = std::sqrt(12.0 * P[h] * ez2 / (g[h] * sum_p));
    delta_out[h] = d;
    bits_out[h] = clampi(std::ceil(-std::log2(d / R[h])), b_min, b_max);
  }
  // the b_max clamp can leave sigma_pred above eps |z|: report it (outputs stay filled)
  double e = 0.0;
  for (uint32_t h = 0; h < H; ++h) {
    const double dq = std::ldexp(R[h], -bits_out[h]);
    e += dq * dq * g[h];
  }
  if (std::sqrt(e / 12.0) > std::fabs(eps_err * z) * (1.0 + 1e-12)) {
    qmpm::set_thread_error("solve_error_bounded: the error bound cannot be met with b <= b_max");
    return QMPM_EDOMAIN;
  }
  return QMPM_OK;
}

qmpm_status qmpm_solve_memory_bounded(uint32_t H, const double* P, const double* g, const double* R,
                                      double budget_bits, int32_t b_min, int32_t b_max, double* delta_out,
                                      int32_t* bits_out) {
  qmpm_status rc = check(H, P, g, R, b_min, b_max);
  if (rc) return rc;
  if (!delta_out || !bits_out) return bad("solve_memory_bounded: NULL output");
  double floor_bits = 0.0;
  for (uint32_t h = 0; h < H; ++h) floor_bits += P[h] * b_min;
  if (floor_bits > budget_bits) return bad("solve_memory_bounded: budget below b_min for every quantity");
  // Active set over the box [b_min, b_max]: quantities with g_h = 0 take b_min; the
  // stationarity solution is computed over the free quantities with the budget
  // the fixed ones leave; a free quantity whose floored width leaves the box is fixed at
  // the bound and the rest re-solved, until no width leaves the box.
  std::vector<int> state(H, 0);  // 0 free, 1 fixed at its bits_out
  for (uint32_t h = 0; h < H; ++h) {
    delta_out[h] = INFINITY;
    bits_out[h] = b_min;
    if (g[h] == 0.0) state[h] = 1;
  }
  for (uint32_t iter = 0; iter <= H; ++iter) {
    double B = budget_bits, sum_pa = 0.0, acc = 0.0;
    for (uint32_t h = 0; h < H; ++h) {
      if (state[h]) {
        B -= P[h] * bits_out[h];
      } else {
        sum_pa += P[h];
        acc += P[h] * (std::log2(R[h]) - 0.5 * std::log2(P[h] / g[h]));
      }
    }
    if (sum_pa == 0.0) break;
    const double log2c = (acc - B) / sum_pa;
    bool changed = false;
    for (uint32_t h = 0; h < H; ++h) {
      if (state[h]) continue;
      const double d = std::exp2(log2c) * std::sqrt(P[h] / g[h]);
      const double b = std::floor(-std::log2(d / R[h]));
      delta_out[h] = d;
      bits_out[h] = clampi(b, b_min, b_max);
      if (!(b >= b_min) || b > b_max) {
        state[h] = 1;
        changed = true;
      }
    }
    if (!changed) break;
  }
  double used = 0.0;
  for (uint32_t h = 0; h < H; ++h) used += P[h] * bits_out[h];
  if (used > budget_bits * (1.0 + 1e-12)) return bad("solve_memory_bounded: no scheme within [b_min, b_max] fits");
  return QMPM_OK;
}

}  // extern "C"
