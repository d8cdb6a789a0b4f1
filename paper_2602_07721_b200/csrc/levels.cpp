// Offline constants on the host: Prop. 1 magnitude levels and the (rho, beta) schedule.
//
// Prop. 1: (u_b)_j^2 ~ Beta(1/2, (m-1)/2). Reading AMB-5: 8 equal-probability bins of |u_j|, level =
// conditional mean of |u_j| in its bin. Computed here in the angle domain |u_j| = sin(theta), where theta has
// density cos^{m-2}(theta) / I_{m-2}(pi/2) on [0, pi/2] and I_n(x) = int_0^x cos^n is evaluated by the
// reduction formula I_n = cos^{n-1} sin / n + (n-1)/n I_{n-2}. Bin edges by bisection on the CDF; the
// conditional mean has the closed form  E[sin; theta_i..theta_{i+1}] = (cos^{m-1} theta_i - cos^{m-1}
// theta_{i+1}) / ((m-1) I_{m-2}(pi/2)). (The CPU oracle derives the same levels independently from the
// regularised incomplete beta function; a -m "not gpu" test checks the fp32 values agree bit for bit.)
#include <cmath>
#include <cstring>

#include "internal.h"

namespace pkv {
namespace {

double cos_power_integral(int n, double x) {  // int_0^x cos^n(t) dt, n >= 0
  if (n == 0) return x;
  if (n == 1) return std::sin(x);
  const double c = std::cos(x), s = std::sin(x);
  return std::pow(c, n - 1) * s / n + (double)(n - 1) / n * cos_power_integral(n - 2, x);
}

}  // namespace

void prop1_levels(int m, double out[8]) {
  const double half_pi = 1.5707963267948966;
  const int n = m - 2;
  const double total = cos_power_integral(n, half_pi);
  double edge[9];
  edge[0] = 0.0;
  edge[8] = half_pi;
  for (int i = 1; i < 8; ++i) {
    const double target = total * i / 8.0;
    double lo = 0.0, hi = half_pi;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (cos_power_integral(n, mid) < target) lo = mid;
      else hi = mid;
      if (hi - lo <= 0.0) break;
    }
    edge[i] = 0.5 * (lo + hi);
  }
  for (int i = 0; i < 8; ++i) {
    const double a = std::pow(std::cos(edge[i]), m - 1), b = std::pow(std::cos(edge[i + 1]), m - 1);
    out[i] = 8.0 * (a - b) / ((m - 1) * total);
  }
}

}  // namespace pkv

extern "C" pkv_status pkv_config_init(pkv_config* cfg, int32_t n_q_heads, int32_t n_kv_heads,
                                      const uint8_t* rot_sign) {
  if (!cfg || !rot_sign) return pkv::set_error(PKV_ERR_INVALID_ARG, "pkv_config_init: null pointer");
  if (n_q_heads <= 0 || n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0 || n_q_heads / n_kv_heads > pkv::GMAX)
    return pkv::set_error(PKV_ERR_INVALID_ARG, "pkv_config_init: need n_q % n_kv == 0 and n_q/n_kv <= 4");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->head_dim = PKV_HEAD_DIM;
  cfg->n_subspaces = PKV_SUBSPACES;
  cfg->subspace_dim = PKV_SUBSPACE_DIM;
  cfg->n_q_heads = n_q_heads;
  cfg->n_kv_heads = n_kv_heads;
  cfg->n_tiers = 6;
  for (int i = 0; i < 6; ++i) cfg->tier_bonus[i] = 6 - i;
  double L[8];
  pkv::prop1_levels(PKV_SUBSPACE_DIM, L);
  for (int i = 0; i < 8; ++i) cfg->mag_levels[i] = (float)L[i];
  for (int t = 0; t < 7; ++t) {
    const double mid = ((double)cfg->mag_levels[t] + (double)cfg->mag_levels[t + 1]) / 2.0;  // exact
    cfg->mag_mid_sq[t] = mid * mid;                                                           // exact
  }
  for (int d = 0; d < PKV_HEAD_DIM; ++d) cfg->rot_sign[d] = rot_sign[d] ? 1 : 0;
  cfg->rot_rounds = 1;
  return PKV_OK;
}

// (min_length, rho, beta) in basis points — reading AMB-11
static void schedule_bp(int64_t n, int64_t* rho, int64_t* beta) {
  static const int64_t table[4][3] = {{0, 1500, 1000}, {20000, 1200, 800}, {60000, 1000, 600}, {200000, 800, 500}};
  *rho = table[0][1];
  *beta = table[0][2];
  for (auto& r : table)
    if (n >= r[0]) {
      *rho = r[1];
      *beta = r[2];
    }
}

// Key-fraction reading of rho (AMB-8b): rho_keys = ceil(rho n) keys per subspace must be covered by
// the probed centroids.
extern "C" pkv_status pkv_schedule_key_fraction(int64_t n, int64_t* rho_keys) {
  if (n < 0 || !rho_keys) return pkv::set_error(PKV_ERR_INVALID_ARG, "pkv_schedule_key_fraction: bad argument");
  int64_t rho, beta;
  schedule_bp(n, &rho, &beta);
  *rho_keys = (rho * n + 9999) / 10000;
  return PKV_OK;
}

extern "C" pkv_status pkv_schedule(int64_t n, int32_t top_k, int32_t* probes_T, int64_t* n_cand) {
  if (n < 0 || top_k < 1 || !probes_T || !n_cand)
    return pkv::set_error(PKV_ERR_INVALID_ARG, "pkv_schedule: bad argument");
  int64_t rho, beta;
  schedule_bp(n, &rho, &beta);
  *probes_T = (int32_t)((rho * PKV_CENTROIDS + 9999) / 10000);
  int64_t c = (beta * n + 9999) / 10000;
  const int64_t lo = top_k < n ? top_k : n;
  if (c < lo) c = lo;
  if (c > n) c = n;
  *n_cand = c;
  return PKV_OK;
}
