// krul_b200.hpp — the C++ drop-in over the C ABI (include/krul_b200.h), in
// the reference's own vocabulary.
//
// The reference (/root/reference/proj) is a C++ library consumed through
// proj/include/krul/*.hpp and has no FFI. This header is the shim a
// maintainer compiles into the reference's tree: it includes the reference's
// own headers for the types that cross the boundary -- the exception
// hierarchy (common.hpp:25-63, krul_status mapped 1:1) and RestorationPlan
// (plan.hpp:15-46) -- and forwards every call to libkrul_b200.so. Build with
// `-I <reference>/proj/include -I <this repo>/include` and link the library.
// tests/cpp/test_shim.cpp compiles it against the reference's headers.
#pragma once

#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "krul/common.hpp"
#include "krul/plan.hpp"
#include "krul_b200.h"

namespace krul::b200 {

// krul_status -> the reference exception of the same name (common.hpp:25-63).
[[noreturn]] inline void raise(int rc, const char* field = nullptr) {
  char msg[1024];
  krul_last_error(msg, sizeof msg);
  switch (rc) {
    case KRUL_E_CONFIG: throw ConfigError(msg);
    case KRUL_E_RESTORATION_GAP: throw RestorationGapError(msg);
    case KRUL_E_STATE_CORRUPTION: throw StateCorruptionError(msg);
    case KRUL_E_ACCOUNTING: throw AccountingError(msg);
    case KRUL_E_PLAN_INVALID: throw PlanInvalidError(msg);
    case KRUL_E_CLASSIFICATION: throw ClassificationError(msg);
    case KRUL_E_SNAPSHOT: throw SnapshotError(msg);
    case KRUL_E_SNAPSHOT_LOAD: throw SnapshotLoadError(field ? field : "", msg);
    default: throw std::runtime_error(std::string("krul_b200: ") + msg);
  }
}
inline void check(int rc) {
  if (rc != KRUL_OK) raise(rc);
}

// strategy::StrategyPair (strategy.hpp:18-24).
struct Pair {
  int shallow = 0, deep = 0;
  double distance = 0.0;
};
inline std::vector<krul_pair> to_c(const std::vector<Pair>& p) {
  std::vector<krul_pair> out;
  for (const Pair& x : p) out.push_back({x.shallow, x.deep, x.distance});
  return out;
}

// ---- strategy (strategy.cpp:16-74) -------------------------------------
inline int shared_layer_quota(int n_layers, double r_l) {
  int q = 0;
  check(krul_quota(n_layers, r_l, &q));
  return q;
}

// ---- scheduler (scheduler.cpp:53-177) ----------------------------------
inline RestorationPlan build_plan(int64_t L, int n_layers, double r_c, const std::vector<Pair>& pairs = {}) {
  const auto cp = to_c(pairs);
  RestorationPlan plan;
  plan.history_len = L;
  plan.recompute_len.resize(size_t(n_layers > 0 ? n_layers : 0));
  check(krul_build_plan(L, n_layers, r_c, cp.data(), int(cp.size()), plan.recompute_len.data()));
  return plan;
}
inline RestorationPlan uniform_plan(int64_t L, int n_layers, double r_c) {
  RestorationPlan plan;
  plan.history_len = L;
  plan.recompute_len.resize(size_t(n_layers > 0 ? n_layers : 0));
  check(krul_uniform_plan(L, n_layers, r_c, plan.recompute_len.data()));
  return plan;
}
inline std::vector<double> default_rc_grid(double step = 0.05) {
  int n = 0;
  check(krul_default_rc_grid(step, nullptr, &n));
  std::vector<double> g(static_cast<size_t>(n));
  check(krul_default_rc_grid(step, g.data(), &n));
  return g;
}
// scheduler::CostModel (scheduler.hpp:14-39); the extension fields at zero
// keep the reference's f32-MHA formulas.
struct CostModel {
  double f_peak = 312e12, b_peak = 139e9, ffn_mult = 4.0;
  krul_cost_model c() const { return {f_peak, b_peak, ffn_mult, 0, 0, 0, 0.0, 0}; }
};
inline double calibrate_rc(const CostModel& cost, int n_layers, int64_t L, int64_t d, const std::vector<Pair>& pairs,
                           const std::vector<double>& grid) {
  const auto cp = to_c(pairs);
  const krul_cost_model cm = cost.c();
  double r = 0.0;
  check(krul_calibrate_rc(&cm, n_layers, L, d, cp.data(), int(cp.size()), grid.data(), int(grid.size()), &r));
  return r;
}

// ---- device context / conversations -------------------------------------
class Context {
 public:
  Context(int device, const krul_model_desc& desc) { check(krul_ctx_create(device, &desc, &h_)); }
  ~Context() { krul_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  krul_ctx* get() const { return h_; }

 private:
  krul_ctx* h_ = nullptr;
};

class Conversation {
 public:
  Conversation(Context& ctx, int64_t capacity) { check(krul_conv_create(ctx.get(), capacity, &h_)); }
  ~Conversation() { krul_conv_destroy(h_); }
  Conversation(const Conversation&) = delete;
  Conversation& operator=(const Conversation&) = delete;
  krul_conv* get() const { return h_; }

 private:
  krul_conv* h_ = nullptr;
};

// ---- compressed KV store (kvstore.cpp:173-511) --------------------------
// KVCacheLayer's content as the expand view returns it (kvstore.cpp:316-343):
// per KV head [rows][head_dim], keys and values.
struct LayerKV {
  TokenSpan span;
  std::vector<float> k, v;
};

class Snapshot {
 public:
  explicit Snapshot(krul_snapshot* h) : h_(h) {}
  ~Snapshot() { krul_snapshot_destroy(h_); }
  Snapshot(Snapshot&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Snapshot(const Snapshot&) = delete;
  Snapshot& operator=(const Snapshot&) = delete;
  krul_snapshot* get() const { return h_; }

  // kvstore::load (kvstore.cpp:394-511); ctx null = host-only (inspect /
  // expand / save), otherwise a pinned store ready to restore. A failed check
  // throws SnapshotLoadError with the reference's field name.
  static Snapshot load(Context* ctx, const std::string& bytes, std::optional<uint64_t> expected_hash = {}) {
    krul_snapshot* h = nullptr;
    char field[32] = {0};
    const uint64_t eh = expected_hash.value_or(0);
    const int rc = krul_snapshot_load(ctx ? ctx->get() : nullptr, bytes.data(), bytes.size(),
                                      expected_hash ? &eh : nullptr, &h, field, int(sizeof field));
    if (rc != KRUL_OK) raise(rc, field);
    return Snapshot(h);
  }
  // kvstore::compress_and_snapshot (kvstore.cpp:243-314), on the device.
  static Snapshot compress(Context& ctx, Conversation& conv, const std::vector<Pair>& pairs,
                           const RestorationPlan& plan, krul_merge_mode mode) {
    const auto cp = to_c(pairs);
    krul_snapshot* h = nullptr;
    check(krul_snapshot_compress(ctx.get(), conv.get(), cp.data(), int(cp.size()), plan.recompute_len.data(),
                                 plan.history_len, mode, &h));
    return Snapshot(h);
  }

  RestorationPlan plan() const {
    int n = 0;
    check(krul_snapshot_header(h_, nullptr, &n, nullptr, nullptr, nullptr, nullptr, nullptr));
    RestorationPlan p;
    p.recompute_len.resize(size_t(n));
    check(krul_snapshot_plan(h_, p.recompute_len.data(), &p.history_len));
    return p;
  }
  void set_plan(const RestorationPlan& p) { check(krul_snapshot_set_plan(h_, p.recompute_len.data())); }

  // kvstore::expand (kvstore.cpp:316-343): the layer's load span.
  LayerKV expand(int layer) const {
    int heads = 0, hd = 0;
    int64_t L = 0;
    check(krul_snapshot_header(h_, nullptr, nullptr, &heads, &hd, &L, nullptr, nullptr));
    const size_t cap = size_t(heads) * size_t(L > 0 ? L : 1) * size_t(hd);
    LayerKV out;
    out.k.resize(cap);
    out.v.resize(cap);
    check(krul_expand(h_, layer, out.k.data(), out.v.data(), &out.span.start, &out.span.end));
    out.k.resize(size_t(heads) * size_t(out.span.length()) * size_t(hd));
    out.v.resize(out.k.size());
    return out;
  }

  // kvstore::storage_report (kvstore.cpp:345-358): (full, stored) bytes.
  std::pair<uint64_t, uint64_t> storage() const {
    uint64_t f = 0, s = 0;
    check(krul_snapshot_storage(h_, &f, &s));
    return {f, s};
  }

 private:
  krul_snapshot* h_ = nullptr;
};

// ---- restoration (scheduler.cpp:320-400) ---------------------------------
// execute_restore: the device conversation replaces vector<KVCacheLayer>.
inline krul_restore_stats execute_restore(Context& ctx, Conversation& conv, const Snapshot& snap,
                                          const std::vector<int32_t>& history) {
  krul_restore_stats st{};
  check(krul_restore(ctx.get(), conv.get(), snap.get(), history.data(), int64_t(history.size()), &st));
  return st;
}
// Restore + the new-input prefill (harness.cpp:125-131): logits of the last
// new row; returns the device TTFT in ms.
inline double restore_and_prefill(Context& ctx, Conversation& conv, const Snapshot& snap,
                                  const std::vector<int32_t>& history, const std::vector<int32_t>& new_tokens,
                                  std::vector<float>& logits, int vocab) {
  logits.resize(size_t(vocab));
  krul_restore_stats st{};
  double ttft = 0.0;
  check(krul_restore_and_prefill(ctx.get(), conv.get(), snap.get(), history.data(), int64_t(history.size()),
                                 new_tokens.data(), int64_t(new_tokens.size()), logits.data(), &st, &ttft));
  return ttft;
}

}  // namespace krul::b200
