// host_plan.cpp — restoration-scheduler arithmetic on the host.
//
// Split points must be bit-exact with the reference, so the double
// arithmetic below follows proj/src/scheduler.cpp operation for operation
// (same products, same llround, same nudge order); only the cost model gains
// optional GQA / bf16 / SwiGLU terms (zero = the reference formula).
#include <algorithm>
#include <set>
#include <string>
#include <cmath>
#include <limits>
#include <map>

#include "host.hpp"

namespace kb {

Cost cost_from(const krul_cost_model* m) {
  Cost c;
  if (!m) return c;
  c.f = m->f_peak;
  c.b = m->b_peak;
  c.ffn_mult = m->ffn_mult;
  c.kv_dim = m->kv_dim;
  c.q_dim = m->q_dim;
  c.ffn_hidden = m->ffn_hidden;
  c.bpe = m->bytes_per_elem > 0 ? m->bytes_per_elem : 4.0;
  c.ffn_kind = m->ffn_kind;
  return c;
}

// scheduler.hpp:22-28; extended: projections 2p d (q + 2 kv) + 2p q d, FFN
// 2p d F x (2 tanh | 3 SwiGLU), attention 4 q sum(r + 1).
double Cost::layer_flops(int64_t p, int64_t d) const {
  const double pd = double(p), dd = double(d);
  const double span = 0.5 * pd * (pd + 1.0);
  if (kv_dim <= 0) return pd * (8.0 * dd * dd + 4.0 * dd * ffn_mult * dd) + 4.0 * dd * span;
  const double q = double(q_dim > 0 ? q_dim : d), kv = double(kv_dim), F = double(ffn_hidden);
  const double ffn = (ffn_kind == KRUL_FFN_SWIGLU ? 6.0 : 4.0) * dd * F;
  return pd * (2.0 * dd * (q + 2.0 * kv) + 2.0 * q * dd + ffn) + 4.0 * q * span;
}
// scheduler.hpp:36-38; extended: 2 tensors x span x kv_dim x bytes/elem.
double Cost::blob_bytes(int64_t span, int64_t d) const {
  if (kv_dim <= 0) return 2.0 * double(span) * double(d) * 4.0;
  return 2.0 * double(span) * double(kv_dim) * bpe;
}

// strategy.cpp:16-25
int quota(int n_layers, double r_l) {
  if (r_l < 0.0 || r_l > 1.0) fail(KRUL_E_CONFIG, "r_l must lie in [0, 1]");
  if (n_layers < 0) fail(KRUL_E_CONFIG, "n_layers must be non-negative");
  const double q = std::ceil(double(n_layers) * r_l - 1e-9);
  return q < 0.0 ? 0 : int(q);
}

// kvstore.cpp:173-205 — one blob per pair over the deep member's load span,
// one per unpaired layer; service order = shallowest owner.
std::vector<krul_blob_spec> blob_specs(const std::vector<int64_t>& p, int64_t L,
                                       const krul_pair* pairs, int np) {
  const int n = int(p.size());
  std::vector<int> partner(size_t(n), -2);  // -2 unpaired, else other member
  std::vector<char> is_shallow(size_t(n), 0);
  for (int k = 0; k < np; ++k) {
    const int a = pairs[k].shallow, b = pairs[k].deep;
    if (a < 0 || b >= n || a >= b) fail(KRUL_E_SNAPSHOT, "strategy pair outside the plan's layers");
    if (partner[size_t(a)] != -2 || partner[size_t(b)] != -2)
      fail(KRUL_E_SNAPSHOT, "layer appears in two pairs");
    partner[size_t(a)] = b;
    partner[size_t(b)] = a;
    is_shallow[size_t(a)] = 1;
  }
  std::vector<krul_blob_spec> out;
  for (int l = 0; l < n; ++l) {
    if (partner[size_t(l)] != -2 && !is_shallow[size_t(l)]) continue;  // deep member
    krul_blob_spec s;
    s.owners[0] = l;
    s.owners[1] = partner[size_t(l)] == -2 ? -1 : partner[size_t(l)];
    const int span_layer = s.owners[1] >= 0 ? s.owners[1] : l;
    s.start = p[size_t(span_layer)];
    s.end = L;
    out.push_back(s);
  }
  return out;
}

static void check_ratio(double r) {
  if (!(r >= 0.0) || r > 1.0) fail(KRUL_E_CONFIG, "r_c must lie in [0, 1]");
}

// scheduler.cpp:53-128
std::vector<int64_t> build_plan(int64_t L, int N, double r_c, const krul_pair* pairs, int np) {
  check_ratio(r_c);
  if (N < 1) fail(KRUL_E_CONFIG, "n_layers must be >= 1");
  if (L < 0) fail(KRUL_E_CONFIG, "history_len must be >= 0");
  for (int k = 0; k < np; ++k)
    if (pairs[k].shallow < 0 || pairs[k].deep >= N)
      fail(KRUL_E_PLAN_INVALID, "strategy pair outside the layer range");
  std::vector<int64_t> p(size_t(N), 0);
  if (N == 1) {
    p[0] = std::llround(r_c * double(L));
    return p;
  }
  const double denom = double(N - 1);
  for (int l = 0; l < N; ++l) {
    const double frac = r_c <= 0.5 ? 2.0 * r_c * double(N - 1 - l) / denom
                                   : 1.0 - 2.0 * (1.0 - r_c) * double(l) / denom;
    p[size_t(l)] = std::llround(std::min(std::max(frac, 0.0), 1.0) * double(L));
  }
  for (int l = 1; l < N; ++l) p[size_t(l)] = std::min(p[size_t(l)], p[size_t(l - 1)]);
  const double target = r_c * double(L) * double(N);
  const double tol = double(N);
  int64_t sum = 0;
  for (int64_t x : p) sum += x;
  // grow from the deepest layer that still has headroom under its parent
  while (double(sum) < target - tol) {
    int l = N - 1;
    while (l >= 0 && p[size_t(l)] >= (l == 0 ? L : p[size_t(l - 1)])) --l;
    if (l < 0) break;
    ++p[size_t(l)];
    ++sum;
  }
  // shrink from the deepest layer still above its child
  while (double(sum) > target + tol) {
    int l = N - 1;
    while (l >= 0 && p[size_t(l)] <= (l == N - 1 ? 0 : p[size_t(l + 1)])) --l;
    if (l < 0) break;
    --p[size_t(l)];
    --sum;
  }
  return p;
}

// scheduler.cpp:130-140
std::vector<int64_t> uniform_plan(int64_t L, int N, double r_c) {
  check_ratio(r_c);
  if (N < 1) fail(KRUL_E_CONFIG, "n_layers must be >= 1");
  if (L < 0) fail(KRUL_E_CONFIG, "history_len must be >= 0");
  const int64_t v = std::min<int64_t>(std::max<int64_t>(std::llround(r_c * double(L)), 0), L);
  return std::vector<int64_t>(size_t(N), v);
}

// scheduler.cpp:142-163 — argmin |T_C - T_L| over the sorted grid, strict <.
double calibrate(const Cost& c, int N, int64_t L, int64_t d, const krul_pair* pairs, int np,
                 const double* grid, int ng) {
  if (ng <= 0) fail(KRUL_E_CONFIG, "calibration grid is empty");
  std::vector<double> g(grid, grid + ng);
  std::sort(g.begin(), g.end());
  double best = g.front(), best_gap = std::numeric_limits<double>::infinity();
  for (double r : g) {
    check_ratio(r);
    const std::vector<int64_t> p = build_plan(L, N, r, pairs, np);
    double flops = 0.0;
    for (int64_t x : p) flops += c.layer_flops(x, d);
    double bytes = 0.0;
    for (const auto& s : blob_specs(p, L, pairs, np)) bytes += c.blob_bytes(s.end - s.start, d);
    const double gap = std::abs(flops / c.f - bytes / c.b);
    if (gap < best_gap) {
      best_gap = gap;
      best = r;
    }
  }
  return best;
}

// scheduler.cpp:165-177
std::vector<double> default_grid(double step) {
  if (!(step > 0.0) || step > 1.0) fail(KRUL_E_CONFIG, "grid step must lie in (0, 1]");
  std::vector<double> g;
  for (int64_t k = 0;; ++k) {
    const double v = double(k) * step;
    if (v > 1.0 + 1e-12) break;
    g.push_back(v < 1.0 ? v : 1.0);
  }
  if (g.back() < 1.0 - 1e-12) g.push_back(1.0);
  return g;
}

// scheduler.cpp:179-221 (bitmask of violation kinds).
int validate_plan(int64_t L, const std::vector<int64_t>& p, const krul_pair* pairs, int np) {
  int m = 0;
  const int n = int(p.size());
  if (L < 0) m |= 1;
  for (int l = 0; l < n; ++l) {
    if (p[size_t(l)] < 0 || p[size_t(l)] > L) m |= 1;
    if (l > 0 && p[size_t(l)] > p[size_t(l - 1)]) m |= 2;
  }
  for (int k = 0; k < np; ++k) {
    const int a = pairs[k].shallow, b = pairs[k].deep;
    if (a < 0 || b >= n || a >= b || p[size_t(b)] > p[size_t(a)]) m |= 8;
  }
  return m;
}

// scheduler.cpp:223-264
int validate_plan_snapshot(const std::vector<int64_t>& p, int64_t L, const Snapshot& s) {
  int m = validate_plan(L, p, s.pairs.data(), int(s.pairs.size()));
  const int n = int(p.size());
  if (s.L != L || s.N != n) return m | 1;
  std::vector<int> owner_blob(size_t(n), -1);
  for (size_t b = 0; b < s.blobs.size(); ++b)
    for (int o : s.blobs[b].owners) {
      if (o == -1) continue;
      if (o < 0 || o >= n) {
        m |= 8;
        continue;
      }
      if (owner_blob[size_t(o)] >= 0) m |= 8;
      owner_blob[size_t(o)] = int(b);
    }
  for (int l = 0; l < n; ++l) {
    if (owner_blob[size_t(l)] < 0) {
      m |= 8;
      continue;
    }
    const auto& bl = s.blobs[size_t(owner_blob[size_t(l)])];
    if (bl.end != L || bl.start > p[size_t(l)]) m |= 8;
  }
  return m;
}

// strategy.cpp:76-131 — every violation in the reference's order, as a
// bitmask (1 pair orientation, 2 layer range, 4 non-I-R member, 8 layer
// reuse, 16 distance order, 32 shared size, 64 quota shortfall) plus the
// reference's "kind: detail" lines.
int validate_strategy(const krul_pair* pairs, int np, const std::set<int>& shared, bool exhausted,
                      const std::set<int>& ir, int n_layers, double r_l, std::string* lines) {
  int mask = 0;
  auto note = [&](int bit, const char* kind, const std::string& detail) {
    mask |= bit;
    if (lines) *lines += std::string(kind) + ": " + detail + "\n";
  };
  std::set<int> seen;
  double last = -1.0;
  for (int k = 0; k < np; ++k) {
    const krul_pair& pr = pairs[k];
    const std::string tag = "(" + std::to_string(pr.shallow) + "," + std::to_string(pr.deep) + ")";
    if (pr.shallow >= pr.deep) note(1, "pair orientation", "pair " + tag + " is not ordered shallow<deep");
    for (const int m : {pr.shallow, pr.deep}) {
      if (m < 0 || m >= n_layers)
        note(2, "layer range", "layer " + std::to_string(m) + " outside [0, " + std::to_string(n_layers) + ")");
      if (!ir.count(m)) note(4, "non-I-R member", "layer " + std::to_string(m) + " in pair " + tag);
      if (!seen.insert(m).second) note(8, "layer reuse", "layer " + std::to_string(m) + " appears in two pairs");
    }
    if (pr.distance < last) note(16, "distance order", "pair " + tag + " breaks the non-decreasing selection order");
    last = pr.distance;
  }
  if (shared != seen)
    note(32, "shared size", "shared set does not equal the union of pair members");
  else if (shared.size() != 2 * size_t(np))
    note(32, "shared size", "|shared| != 2 * |pairs|");
  const int q = quota(n_layers, r_l);
  if (int(shared.size()) < q && !exhausted)
    note(64, "quota shortfall", "|shared| = " + std::to_string(shared.size()) + " below quota " +
                                    std::to_string(q) + " without the exhaustion flag");
  return mask;
}

}  // namespace kb
