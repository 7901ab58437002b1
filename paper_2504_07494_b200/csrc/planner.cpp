// Adaptive runtime scheduler of Apt-Serve (NEXT row f2): the request manager's per-iteration
// decision S = {(alpha_i, beta_i)} (§4.2, §5).  Host-only C++;
// it produces the cache-mode assignment beta that the GPU path consumes (hc_append modes),
// and is not on the GPU hot path.  Semantics are specified in include/hc.h; the fp64
// reference is oracle/planner_oracle.py.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hc.h"

namespace {

struct Stage {
  double theta;
  double dm;
  int32_t idx;   // candidate index (input order)
  int32_t kind;  // 0 hidden, 1 upgrade, 2 direct KV
};

double kv_units(int64_t tokens, int32_t B) {
  const int64_t b = B > 0 ? B : 1;
  return 2.0 * (double)((tokens + b - 1) / b);
}

}  // namespace

extern "C" {

double hc_calibrate_rho(int32_t n, const double* m, const double* t) {
  if (n < 1 || !m || !t) return -1.0;
  double mt = 0.0, mm = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    mt += m[i] * t[i];
    mm += m[i] * m[i];
  }
  return mm > 0.0 ? mt / mm : -1.0;
}

hc_status hc_schedule(const hc_sched_config* cfg, int32_t n, const hc_sched_request* reqs, double now,
                      int32_t* alpha, int32_t* beta, double* g, hc_sched_result* result) {
  if (!cfg || n < 0 || (n > 0 && (!reqs || !alpha || !beta)) || !result) return HC_E_INVALID;
  if (cfg->rho < 0 || cfg->total_units < 0 || (cfg->fallback == 1 && (cfg->decay <= 0 || cfg->decay > 1)))
    return HC_E_INVALID;
  *result = hc_sched_result{-1, 0, 0.0, 0.0, 0.0};
  for (int32_t i = 0; i < n; ++i) alpha[i] = beta[i] = 0;
  // ---- runtime tracking: pending time p_i, max memory m_i, SLO state
  std::vector<double> p(n), m(n);
  double sum_w = 0.0, sum_r = 0.0, m_running = 0.0;
  int32_t n_w = 0, n_r = 0;
  for (int32_t i = 0; i < n; ++i) {
    const hc_sched_request& r = reqs[i];
    if (r.seq_len < 0) return HC_E_INVALID;
    p[i] = std::max(0.0, r.has_token ? now - r.last_token_time : now - r.arrival_time);
    m[i] = kv_units(r.seq_len + 1, cfg->block_size);
    if (r.running) {
      sum_r += p[i];
      m_running += m[i];
      ++n_r;
    } else {
      sum_w += p[i];
      ++n_w;
    }
  }
  // ---- iteration type: the queue with the larger cumulative pending time
  int32_t type;
  if (n_w == 0 && n_r == 0) return HC_OK;   // idle
  if (n_r == 0) type = 1;
  else if (n_w == 0) type = 0;
  else type = sum_w > sum_r ? 1 : 0;        // tie -> decode
  const double M = type == 1 ? std::max(0.0, cfg->total_units - m_running) : cfg->total_units;
  const double N = (double)(n_w + n_r);
  // ---- candidates U^e with fallback-adjusted pending time
  std::vector<int32_t> cand;
  std::vector<double> pc;
  for (int32_t i = 0; i < n; ++i) {
    if ((reqs[i].running != 0) != (type == 0)) continue;
    double pi = p[i];
    const double slo = reqs[i].has_token ? cfg->tbt_slo : cfg->ttft_slo;
    if (slo > 0 && pi > slo) pi = cfg->fallback == 1 ? cfg->decay * pi : cfg->eps;
    cand.push_back(i);
    pc.push_back(pi);
  }
  const int32_t nc = (int32_t)cand.size();
  auto value = [&](int32_t c, int32_t b) { return pc[c] - b * N * cfg->rho * m[cand[c]]; };  // Eq. 5-6
  // ---- marginal gains theta -> candidate schedule set Upsilon (Eq. 10)
  std::vector<Stage> ups;
  ups.reserve(2 * (size_t)nc);
  for (int32_t c = 0; c < nc; ++c) {
    const double mi = m[cand[c]];
    if (mi <= 0) continue;
    if (cfg->hybrid && pc[c] / mi >= 2.0 * N * cfg->rho) {
      ups.push_back({2.0 * pc[c] / mi - 2.0 * N * cfg->rho, mi / 2.0, c, 0});
      ups.push_back({2.0 * N * cfg->rho, mi / 2.0, c, 1});
    } else {
      ups.push_back({pc[c] / mi, mi, c, 2});
    }
  }
  // ties: theta desc, delta-m asc, lower request id, then input order
  std::sort(ups.begin(), ups.end(), [&](const Stage& a, const Stage& b) {
    if (a.theta != b.theta) return a.theta > b.theta;
    if (a.dm != b.dm) return a.dm < b.dm;
    const int64_t ia = reqs[cand[a.idx]].id, ib = reqs[cand[b.idx]].id;
    if (ia != ib) return ia < ib;
    if (a.idx != b.idx) return a.idx < b.idx;
    return a.kind < b.kind;
  });
  // ---- greedy (Eq. 11)
  std::vector<int32_t> ca(nc, 0), cb(nc, 0);
  double used = 0.0;
  const double tol = 1e-9 * std::max(1.0, M);
  for (const Stage& s : ups) {
    if (used + s.dm > M + tol) continue;
    if (s.kind == 0) {
      ca[s.idx] = 1;
      cb[s.idx] = 1;
    } else if (s.kind == 1) {
      if (!(ca[s.idx] && cb[s.idx])) continue;   // upgrade only after its hidden stage
      cb[s.idx] = 0;
    } else {
      ca[s.idx] = 1;
      cb[s.idx] = 0;
    }
    used += s.dm;
  }
  double obj = 0.0;
  for (int32_t c = 0; c < nc; ++c)
    if (ca[c]) obj += value(c, cb[c]);
  // ---- best single feasible assignment (KV, or hidden when allowed; R14)
  double best = obj;
  int32_t best_c = -1, best_b = 0;
  for (int32_t c = 0; c < nc; ++c) {
    for (int32_t b = 0; b <= (cfg->hybrid ? 1 : 0); ++b) {
      const double need = m[cand[c]] * (1.0 - 0.5 * b);
      if (need > M + tol) continue;
      const double gv = value(c, b);
      if (gv > best) {
        best = gv;
        best_c = c;
        best_b = b;
      }
    }
  }
  if (best_c >= 0) {
    std::fill(ca.begin(), ca.end(), 0);
    std::fill(cb.begin(), cb.end(), 0);
    ca[best_c] = 1;
    cb[best_c] = best_b;
    obj = best;
  }
  double mem = 0.0;
  for (int32_t c = 0; c < nc; ++c) {
    alpha[cand[c]] = ca[c];
    beta[cand[c]] = cb[c];
    if (ca[c]) mem += (1.0 - 0.5 * cb[c]) * m[cand[c]];
    if (g) g[cand[c]] = value(c, cb[c]);
  }
  *result = hc_sched_result{type, nc, M, obj, mem};
  return HC_OK;
}

}  // extern "C"
