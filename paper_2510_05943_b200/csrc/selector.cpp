// selector.cpp -- host side of NEXT-4: the Parallelism Selector's policy (PAPER.md:184-189,
// Eq. (1) at PAPER.md:233-237; readings s1-s4 in DESIGN.md).  Pure host code: no CUDA calls.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "../../include/earl_dispatch.h"

namespace earl {
earl_status_t set_error(earl_status_t st, const char* msg);  // api.cu
}

struct earl_policy {
  std::vector<int32_t> table;   // configuration per context range
  std::vector<int64_t> bounds;  // n_buckets + 1
  std::vector<uint8_t> oom;     // [n_configs][n_buckets] (empty: no OOM probe)
  int32_t n_configs = 0;
  int64_t hysteresis = 0;
};

namespace {

earl_status_t fail(earl_status_t st, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return earl::set_error(st, buf);
}

}  // namespace

extern "C" earl_status_t earl_speedup_pct(double tgs_a, double tgs_b, double* out) {
  if (!out) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL out");
  if (!(tgs_a > 0)) return fail(EARL_ERR_INVALID_ARGUMENT, "TGS(a) must be positive, got %g", tgs_a);
  *out = (tgs_b - tgs_a) / tgs_a * 100.0;
  return EARL_OK;
}

extern "C" earl_status_t earl_policy_build(int32_t n_configs, const int32_t* config_tp,
                                           int32_t n_buckets, const int64_t* bounds,
                                           const double* tgs, const uint8_t* oom,
                                           int64_t hysteresis_tokens, earl_policy_t* out) {
  if (!out || !config_tp || !bounds || !tgs) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (n_configs <= 0 || n_buckets <= 0)
    return fail(EARL_ERR_INVALID_ARGUMENT, "need >= 1 configuration and >= 1 context range");
  if (hysteresis_tokens < 0) return fail(EARL_ERR_INVALID_ARGUMENT, "hysteresis must be >= 0");
  for (int32_t b = 0; b < n_buckets; ++b)
    if (bounds[b] >= bounds[b + 1])
      return fail(EARL_ERR_INVALID_ARGUMENT, "context range bounds must ascend (bounds[%d] >= bounds[%d])", b, b + 1);
  std::vector<int32_t> table(n_buckets);
  for (int32_t b = 0; b < n_buckets; ++b) {
    int32_t best = -1;
    for (int32_t c = 0; c < n_configs; ++c) {
      const size_t k = (size_t)c * n_buckets + b;
      if (oom && oom[k]) continue;
      if (!(tgs[k] > 0))
        return fail(EARL_ERR_INVALID_ARGUMENT, "TGS of configuration %d in range %d must be positive", c, b);
      if (best < 0) {
        best = c;
        continue;
      }
      const double tb = tgs[(size_t)best * n_buckets + b];
      // highest TGS; ties: smaller TP, then lower index (c > best, so only TP can win a tie)
      if (tgs[k] > tb || (tgs[k] == tb && config_tp[c] < config_tp[best])) best = c;
    }
    if (best < 0)
      return fail(EARL_ERR_POLICY, "every configuration runs out of memory in context range %d [%lld, %lld)",
                  b, (long long)bounds[b], (long long)bounds[b + 1]);
    table[b] = best;
  }
  earl_policy* p = new earl_policy;
  p->table = std::move(table);
  p->bounds.assign(bounds, bounds + n_buckets + 1);
  p->n_configs = n_configs;
  p->hysteresis = hysteresis_tokens;
  if (oom) p->oom.assign(oom, oom + (size_t)n_configs * n_buckets);
  *out = p;
  return EARL_OK;
}

extern "C" earl_status_t earl_policy_table(earl_policy_t p, int32_t* config_of_bucket) {
  if (!p || !config_of_bucket) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  for (size_t b = 0; b < p->table.size(); ++b) config_of_bucket[b] = p->table[b];
  return EARL_OK;
}

extern "C" earl_status_t earl_policy_select(earl_policy_t p, double avg_len, int32_t current,
                                            int32_t* next, int32_t* switched) {
  if (!p || !next || !switched) return fail(EARL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (current < 0 || current >= p->n_configs)
    return fail(EARL_ERR_INVALID_ARGUMENT, "current configuration %d outside [0, %d)", current, p->n_configs);
  const int nb = (int)p->table.size();
  int b = -1;
  for (int k = 0; k < nb; ++k)
    if ((double)p->bounds[k] <= avg_len && avg_len < (double)p->bounds[k + 1]) b = k;
  if (b < 0)
    return fail(EARL_ERR_POLICY, "average length %g outside [%lld, %lld)", avg_len,
                (long long)p->bounds[0], (long long)p->bounds[nb]);
  int32_t want = p->table[b];
  const double h = (double)p->hysteresis;
  const bool current_oom = !p->oom.empty() && p->oom[(size_t)current * nb + b];
  if (want != current && !current_oom) {
    // hysteresis: a range of the current configuration borders this one and avg_len sits
    // within h tokens of the shared boundary (never onto a configuration that OOMs here)
    if (b > 0 && p->table[b - 1] == current && avg_len - (double)p->bounds[b] < h) want = current;
    if (b + 1 < nb && p->table[b + 1] == current && (double)p->bounds[b + 1] - avg_len < h) want = current;
  }
  *next = want;
  *switched = want != current;
  return EARL_OK;
}

extern "C" earl_status_t earl_policy_destroy(earl_policy_t p) {
  delete p;
  return EARL_OK;
}
