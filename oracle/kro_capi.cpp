// kro_capi.cpp — C ABI over the CPU oracle, for the Python parity tests.
// TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
// bench.py's CPU-baseline leg; never by the product.
//
// Handles are opaque pointers. Every entry returns a kro::Status (0 = ok);
// kro_last_error copies the message of the last failure on this thread.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <omp.h>
#include <cstring>
#include <string>

#include "krul_oracle.hpp"

using namespace kro;

namespace {
thread_local std::string g_err;
thread_local int g_code = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_code = 0;
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    g_code = e.code;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_code = 99;
    return 99;
  }
}

struct KVSet {
  std::vector<KVLayer> kv;
};
struct PrefillH {
  PrefillOut out;
};

Strategy make_strategy(const int* sh, const int* dp, const double* dist, int n) {
  Strategy s;
  for (int i = 0; i < n; ++i) {
    s.pairs.push_back({sh[i], dp[i], dist ? dist[i] : 0.0});
    s.shared.insert(sh[i]);
    s.shared.insert(dp[i]);
  }
  return s;
}

void copy_kv_layer(const KVLayer& l, float* k, float* v, int hd) {
  for (size_t g = 0; g < l.k.size(); ++g) {
    const size_t n = size_t(l.k[g].r) * size_t(hd);
    if (k) std::memcpy(k + g * n, l.k[g].v.data(), n * sizeof(float));
    if (v) std::memcpy(v + g * n, l.v[g].v.data(), n * sizeof(float));
  }
}
}  // namespace

extern "C" {

int kro_last_error(char* buf, size_t n) {
  if (buf && n) {
    std::strncpy(buf, g_err.c_str(), n - 1);
    buf[n - 1] = 0;
  }
  return g_code;
}

uint64_t kro_fnv1a64(const void* p, size_t n, uint64_t basis) { return fnv1a64(p, n, basis); }
uint32_t kro_crc32(const void* p, size_t n, uint32_t crc) { return crc32(p, n, crc); }

// Uniform stream draws (common.hpp:68-86): fills `out[n]` with next(lo, hi).
void kro_uniform_fill(uint64_t seed, float lo, float hi, float* out, int64_t n) {
  Uniform u(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = u.next(lo, hi);
}
void kro_uniform_index(uint64_t seed, uint64_t mod, uint64_t* out, int64_t n) {
  Uniform u(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = u.index(mod);
}

// ---- model ----------------------------------------------------------------
struct kro_cfg {
  int n_layers, n_heads, n_kv_heads, head_dim, d_model, vocab;
  float ffn_mult;
  int ffn_kind;
  uint64_t seed;
  double rope_theta;
};
static ModelConfig to_cfg(const kro_cfg* c) {
  ModelConfig m;
  m.n_layers = c->n_layers;
  m.n_heads = c->n_heads;
  m.n_kv_heads = c->n_kv_heads;
  m.head_dim = c->head_dim;
  m.d_model = c->d_model;
  m.vocab = c->vocab;
  m.ffn_mult = c->ffn_mult;
  m.ffn_kind = c->ffn_kind;
  m.seed = c->seed;
  m.rope_theta = c->rope_theta;
  return m;
}

int kro_config_hash(const kro_cfg* c, uint64_t* out) {
  return guard([&] { *out = to_cfg(c).hash(); });
}
int kro_config_ffn_hidden(const kro_cfg* c, int* out) {
  return guard([&] { *out = to_cfg(c).ffn_hidden(); });
}
int kro_config_validate(const kro_cfg* c) {
  return guard([&] { to_cfg(c).validate(); });
}

int kro_model_build(const kro_cfg* c, void** out) {
  return guard([&] { *out = new Model(build_model(to_cfg(c))); });
}
void kro_model_free(void* m) { delete static_cast<Model*>(m); }

// Timing-only model (bench CPU legs at the Llama shapes): the reference's
// layout and U[-1/sqrt(d), 1/sqrt(d)) bound, but filled in parallel from a
// counter-based hash instead of the sequential mt19937_64 draw (which takes
// minutes for 8 B weights). Not a parity model.
int kro_model_build_fast(const kro_cfg* c, uint64_t seed, void** out) {
  return guard([&] {
    const ModelConfig cfg = to_cfg(c);
    cfg.validate();
    auto* m = new Model;
    m->cfg = cfg;
    const float bound = 1.0f / std::sqrt(float(cfg.d_model));
    const int64_t d = cfg.d_model, F = cfg.ffn_hidden();
    const int64_t qd = int64_t(cfg.n_heads) * cfg.head_dim, kvd = int64_t(cfg.kv_heads()) * cfg.head_dim;
    uint64_t stream = 0;
    auto fill = [&](std::vector<float>& v) {
      const uint64_t sid = ++stream;
      const int64_t n = int64_t(v.size());
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        uint64_t z = seed ^ (sid << 40) ^ uint64_t(i) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        v[size_t(i)] = -bound + 2.0f * bound * float(uint32_t(z >> 40)) * (1.0f / 16777216.0f);
      }
    };
    auto mat = [&](int64_t r, int64_t cc) {
      Mat x(r, cc);
      fill(x.v);
      return x;
    };
    m->embed = mat(cfg.vocab, d);
    m->layers.resize(size_t(cfg.n_layers));
    for (auto& w : m->layers) {
      w.wq = mat(d, qd); w.wk = mat(d, kvd); w.wv = mat(d, kvd); w.wo = mat(qd, d);
      w.w1 = mat(d, F); w.w2 = mat(F, d);
      if (cfg.ffn_kind == 0) {
        w.b1.assign(size_t(F), 0.f); fill(w.b1);
        w.b2.assign(size_t(d), 0.f); fill(w.b2);
      } else {
        w.wu = mat(d, F);
      }
    }
    m->unembed = mat(d, cfg.vocab);
    *out = m;
  });
}

void kro_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int kro_max_threads(void) { return omp_get_max_threads(); }

// KV set of n_layers x [0, L) filled with U(-1, 1) (timing-only snapshots).
void* kro_kv_synthetic(int n_layers, int kv_heads, int hd, int64_t L, uint64_t seed) {
  auto* s = new KVSet;
  s->kv.resize(size_t(n_layers));
  for (int l = 0; l < n_layers; ++l) {
    KVLayer& x = s->kv[size_t(l)];
    x.span = {0, L};
    for (int g = 0; g < kv_heads; ++g)
      for (int kvi = 0; kvi < 2; ++kvi) {
        Mat m(L, hd);
        const int64_t n = L * hd;
        const uint64_t sid = (uint64_t(l) * 64 + uint64_t(g)) * 2 + uint64_t(kvi);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
          uint64_t z = seed ^ (sid << 36) ^ uint64_t(i) * 0x9e3779b97f4a7c15ull;
          z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
          z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
          z ^= z >> 31;
          m.v[size_t(i)] = -1.0f + 2.0f * float(uint32_t(z >> 40)) * (1.0f / 16777216.0f);
        }
        (kvi ? x.v : x.k).push_back(std::move(m));
      }
  }
  return s;
}

// Flat weights in reference draw order (engine.cpp:368-393). Returns the
// float count when out == nullptr.
int64_t kro_model_weights(void* mh, float* out) {
  const Model& m = *static_cast<Model*>(mh);
  int64_t n = 0;
  auto put = [&](const std::vector<float>& v) {
    if (out) std::memcpy(out + n, v.data(), v.size() * sizeof(float));
    n += int64_t(v.size());
  };
  put(m.embed.v);
  for (const LayerW& w : m.layers) {
    put(w.wq.v); put(w.wk.v); put(w.wv.v); put(w.wo.v);
    if (m.cfg.ffn_kind == 0) {
      put(w.w1.v); put(w.b1); put(w.w2.v); put(w.b2);
    } else {
      put(w.w1.v); put(w.wu.v); put(w.w2.v);
    }
  }
  put(m.unembed.v);
  return n;
}

// ---- prefill / decode / partial -------------------------------------------
// preload: optional KV set (as produced by kro_restore / kro_partial / a
// prefill) restricted to suffixes via kro_kv_suffix.
int kro_prefill(void* mh, const int32_t* toks, int64_t n, void* preload, int capture, void** out) {
  return guard([&] {
    std::vector<int32_t> t(toks, toks + n);
    auto* h = new PrefillH;
    try {
      h->out = prefill(*static_cast<Model*>(mh), t,
                       preload ? &static_cast<KVSet*>(preload)->kv : nullptr, capture != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void kro_prefill_free(void* h) { delete static_cast<PrefillH*>(h); }
void kro_prefill_logits(void* h, float* out) {
  const auto& l = static_cast<PrefillH*>(h)->out.logits;
  std::memcpy(out, l.data(), l.size() * sizeof(float));
}
// Attention probabilities of layer l, head h: [rows x width].
int kro_prefill_attn(void* h, int layer, int head, float* out, int64_t* rows, int64_t* width) {
  return guard([&] {
    const auto& rec = static_cast<PrefillH*>(h)->out.attn;
    const Mat& m = rec.layers.at(size_t(layer)).prefill.at(size_t(head));
    if (rows) *rows = m.r;
    if (width) *width = m.c;
    if (out) std::memcpy(out, m.v.data(), m.v.size() * sizeof(float));
  });
}
// Moves the prefill's KV into a KV set handle (prefill handle keeps nothing).
void* kro_prefill_take_kv(void* h) {
  auto* s = new KVSet;
  s->kv = std::move(static_cast<PrefillH*>(h)->out.kv);
  return s;
}

void kro_kv_free(void* s) { delete static_cast<KVSet*>(s); }
void* kro_kv_clone(void* s) { return new KVSet(*static_cast<KVSet*>(s)); }
int kro_kv_span(void* s, int layer, int64_t* start, int64_t* end) {
  return guard([&] {
    const auto& l = static_cast<KVSet*>(s)->kv.at(size_t(layer));
    *start = l.span.start;
    *end = l.span.end;
  });
}
// K/V of one layer as [kv_heads][rows][hd].
int kro_kv_get(void* s, int layer, int hd, float* k, float* v) {
  return guard([&] { copy_kv_layer(static_cast<KVSet*>(s)->kv.at(size_t(layer)), k, v, hd); });
}
// Builds a KV set from host arrays: per layer [kv_heads][rows_l][hd] with
// span [start_l, end_l).
void* kro_kv_from_host(int n_layers, int kv_heads, int hd, const int64_t* starts,
                       const int64_t* ends, const float* const* ks, const float* const* vs) {
  auto* s = new KVSet;
  s->kv.resize(size_t(n_layers));
  for (int l = 0; l < n_layers; ++l) {
    KVLayer& x = s->kv[size_t(l)];
    x.span = {starts[l], ends[l]};
    const int64_t rows = std::max<int64_t>(0, ends[l] - starts[l]);
    for (int g = 0; g < kv_heads; ++g) {
      Mat k(rows, hd), v(rows, hd);
      if (rows) {
        std::memcpy(k.v.data(), ks[l] + size_t(g) * size_t(rows * hd), size_t(rows * hd) * 4);
        std::memcpy(v.v.data(), vs[l] + size_t(g) * size_t(rows * hd), size_t(rows * hd) * 4);
      }
      x.k.push_back(std::move(k));
      x.v.push_back(std::move(v));
    }
  }
  return s;
}

int kro_decode(void* mh, void* kvs, int32_t tok, float* logits, float* rows_out) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(mh);
    DecodeOut d = decode_step(m, static_cast<KVSet*>(kvs)->kv, tok);
    std::memcpy(logits, d.logits.data(), d.logits.size() * sizeof(float));
    if (rows_out) {
      size_t off = 0;
      for (const Mat& r : d.rows) {
        std::memcpy(rows_out + off, r.v.data(), r.v.size() * sizeof(float));
        off += r.v.size();
      }
    }
  });
}

int kro_partial(void* mh, const int32_t* toks, int64_t n, const int64_t* p, int np, void** out) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(mh);
    std::vector<int32_t> t(toks, toks + n);
    std::vector<int64_t> pv(p, p + np);
    PartialOut po = partial_prefix_recompute(m, t, pv);
    auto* s = new KVSet;
    s->kv = std::move(po.kv);
    *out = s;
  });
}

// ---- analysis -------------------------------------------------------------
// probs: [N][H][rows][W] f32 (zeros above the causal diagonal).
int kro_classify(const float* probs, int N, int H, int64_t rows, int64_t W, int64_t first_q,
                 double gamma, double ifrac, double rfrac, double* avg, int* is_ir) {
  return guard([&] {
    AttnRecord rec;
    rec.first_q = first_q;
    rec.layers.resize(size_t(N));
    for (int l = 0; l < N; ++l)
      for (int h = 0; h < H; ++h) {
        Mat m(rows, W);
        std::memcpy(m.v.data(), probs + (size_t(l) * H + h) * size_t(rows * W), size_t(rows * W) * 4);
        rec.layers[size_t(l)].prefill.push_back(std::move(m));
      }
    ClassReport r = classify_layers(rec, gamma, ifrac, rfrac);
    for (int l = 0; l < N; ++l) {
      avg[l] = r.avg[size_t(l)];
      is_ir[l] = std::find(r.ir.begin(), r.ir.end(), l) != r.ir.end();
    }
  });
}
int kro_classify_prefill(void* ph, double gamma, double ifrac, double rfrac, double* avg, int* is_ir) {
  return guard([&] {
    const auto& rec = static_cast<PrefillH*>(ph)->out.attn;
    ClassReport r = classify_layers(rec, gamma, ifrac, rfrac);
    for (size_t l = 0; l < r.avg.size(); ++l) {
      avg[l] = r.avg[l];
      is_ir[l] = std::find(r.ir.begin(), r.ir.end(), int(l)) != r.ir.end();
    }
  });
}

int kro_acc_create(const int* ir, int n, int H, void** out) {
  return guard([&] { *out = new Accumulator(std::vector<int>(ir, ir + n), H); });
}
void kro_acc_free(void* a) { delete static_cast<Accumulator*>(a); }
int kro_acc_fold_prefill(void* a, const float* probs, int N, int H, int64_t rows, int64_t W) {
  return guard([&] {
    AttnRecord rec;
    rec.layers.resize(size_t(N));
    for (int l = 0; l < N; ++l)
      for (int h = 0; h < H; ++h) {
        Mat m(rows, W);
        std::memcpy(m.v.data(), probs + (size_t(l) * H + h) * size_t(rows * W), size_t(rows * W) * 4);
        rec.layers[size_t(l)].prefill.push_back(std::move(m));
      }
    static_cast<Accumulator*>(a)->fold_prefill(rec);
  });
}
int kro_acc_fold_prefill_handle(void* a, void* ph) {
  return guard([&] { static_cast<Accumulator*>(a)->fold_prefill(static_cast<PrefillH*>(ph)->out.attn); });
}
// rows: [N][H][W]
int kro_acc_fold_decode(void* a, const float* rows, int N, int H, int64_t W) {
  return guard([&] {
    std::vector<Mat> v;
    for (int l = 0; l < N; ++l) {
      Mat m(H, W);
      std::memcpy(m.v.data(), rows + size_t(l) * H * size_t(W), size_t(H * W) * 4);
      v.push_back(std::move(m));
    }
    static_cast<Accumulator*>(a)->fold_decode(v);
  });
}
int kro_acc_sums(void* a, double* out) {
  return guard([&] {
    const auto& s = static_cast<Accumulator*>(a)->sums;
    std::memcpy(out, s.data(), s.size() * sizeof(double));
  });
}
int kro_acc_finalize(void* a, double* D) {
  return guard([&] {
    auto v = static_cast<Accumulator*>(a)->finalize();
    std::memcpy(D, v.data(), v.size() * sizeof(double));
  });
}
double kro_stable_sq(const float* a, const float* b, int64_t n) { return stable_sq(a, b, n); }

// ---- strategy -------------------------------------------------------------
int kro_quota(int n_layers, double r_l, int* out) {
  return guard([&] { *out = shared_layer_quota(n_layers, r_l); });
}
// D [n x n] over dm_layers; out arrays sized >= n/2.
int kro_select(const double* D, const int* dm_layers, int n, const int* ir, int n_ir, double r_l,
               int n_layers, int* shallow, int* deep, double* dist, int* n_pairs, int* exhausted) {
  return guard([&] {
    Strategy s = select_strategy(std::vector<double>(D, D + size_t(n) * size_t(n)),
                                 std::vector<int>(dm_layers, dm_layers + n),
                                 std::vector<int>(ir, ir + n_ir), r_l, n_layers);
    *n_pairs = int(s.pairs.size());
    for (size_t i = 0; i < s.pairs.size(); ++i) {
      shallow[i] = s.pairs[i].shallow;
      deep[i] = s.pairs[i].deep;
      dist[i] = s.pairs[i].distance;
    }
    *exhausted = s.exhausted;
  });
}

// strategy.cpp:76-131 (bitmask of violation kinds, krul_oracle.hpp)
int kro_validate_strategy(const int* sh, const int* dp, const double* dist, int np, const int* shared,
                          int n_shared, int exhausted, const int* ir, int n_ir, int n_layers, double r_l,
                          int* mask) {
  return guard([&] {
    Strategy s;
    for (int i = 0; i < np; ++i) s.pairs.push_back({sh[i], dp[i], dist[i]});
    s.shared = std::set<int>(shared, shared + n_shared);
    s.exhausted = exhausted != 0;
    *mask = validate_strategy(s, std::vector<int>(ir, ir + n_ir), n_layers, r_l);
  });
}

// ---- plans / scheduler ----------------------------------------------------
int kro_build_plan(int64_t L, int N, double r_c, const int* sh, const int* dp, int np, int64_t* out) {
  return guard([&] {
    Plan p = build_plan(L, N, r_c, make_strategy(sh, dp, nullptr, np));
    std::copy(p.p.begin(), p.p.end(), out);
  });
}
int kro_uniform_plan(int64_t L, int N, double r_c, int64_t* out) {
  return guard([&] {
    Plan p = uniform_plan(L, N, r_c);
    std::copy(p.p.begin(), p.p.end(), out);
  });
}
int kro_calibrate(double f_peak, double b_peak, double ffn_mult, int N, int64_t L, int64_t d,
                  const int* sh, const int* dp, int np, const double* grid, int ng, double* out) {
  return guard([&] {
    CostModel c{f_peak, b_peak, ffn_mult};
    *out = calibrate_rc(c, N, L, d, make_strategy(sh, dp, nullptr, np), std::vector<double>(grid, grid + ng));
  });
}
int kro_default_grid(double step, double* out, int* n) {
  return guard([&] {
    auto g = default_rc_grid(step);
    *n = int(g.size());
    if (out) std::copy(g.begin(), g.end(), out);
  });
}
int kro_validate_plan(int64_t L, const int64_t* p, int N, const int* sh, const int* dp, int np, int* mask) {
  return guard([&] {
    Plan plan{std::vector<int64_t>(p, p + N), L};
    *mask = validate_plan(plan, make_strategy(sh, dp, nullptr, np));
  });
}
// owners_out [N*2] (-1 padded), spans_out [N*2]; returns count via n_out.
int kro_blob_specs(int64_t L, const int64_t* p, int N, const int* sh, const int* dp, int np,
                   int* owners_out, int64_t* spans_out, int* n_out) {
  return guard([&] {
    Plan plan{std::vector<int64_t>(p, p + N), L};
    auto specs = plan_blob_specs(make_strategy(sh, dp, nullptr, np), plan);
    *n_out = int(specs.size());
    for (size_t i = 0; i < specs.size(); ++i) {
      owners_out[2 * i] = specs[i].owners[0];
      owners_out[2 * i + 1] = specs[i].owners.size() > 1 ? specs[i].owners[1] : -1;
      spans_out[2 * i] = specs[i].span.start;
      spans_out[2 * i + 1] = specs[i].span.end;
    }
  });
}
int kro_simulate(int64_t L, const int64_t* p, int N, const int* sh, const int* dp, int np,
                 double f_peak, double b_peak, double ffn_mult, int64_t d, double* out6) {
  return guard([&] {
    Plan plan{std::vector<int64_t>(p, p + N), L};
    Trace t = simulate_pipeline(plan, make_strategy(sh, dp, nullptr, np), CostModel{f_peak, b_peak, ffn_mult}, d);
    out6[0] = t.makespan; out6[1] = t.compute_finish; out6[2] = t.load_finish;
    out6[3] = t.bubble_compute; out6[4] = t.bubble_load;
    out6[5] = double(t.compute.size() * 1000 + t.load.size());
  });
}
double kro_layer_flops(double ffn_mult, int64_t p, int64_t d) { return CostModel{312e12, 139e9, ffn_mult}.layer_flops(p, d); }
double kro_prefill_flops(double ffn_mult, int64_t n, int64_t h, int64_t d, int N) {
  return CostModel{312e12, 139e9, ffn_mult}.prefill_flops(n, h, d, N);
}

// ---- kvstore / restore ----------------------------------------------------
int kro_snapshot(void* kvs, const kro_cfg* c, const int* sh, const int* dp, const double* dist, int np,
                 const int64_t* p, int64_t L, int mode, void** out) {
  return guard([&] {
    ModelConfig cfg = to_cfg(c);
    Plan plan{std::vector<int64_t>(p, p + cfg.n_layers), L};
    *out = new Snapshot(compress_and_snapshot(static_cast<KVSet*>(kvs)->kv,
                                              make_strategy(sh, dp, dist, np), plan, mode, "bench", cfg));
  });
}
void kro_snapshot_free(void* s) { delete static_cast<Snapshot*>(s); }
int kro_snapshot_n_blobs(void* s) { return int(static_cast<Snapshot*>(s)->blobs.size()); }
// owners[2] (-1 padded), span[2]; k/v [kv_heads][rows][hd] when non-null.
int kro_snapshot_blob(void* s, int b, int* owners, int64_t* span, float* k, float* v) {
  return guard([&] {
    const Snapshot& sn = *static_cast<Snapshot*>(s);
    const Blob& bl = sn.blobs.at(size_t(b));
    owners[0] = bl.owners[0];
    owners[1] = bl.owners.size() > 1 ? bl.owners[1] : -1;
    span[0] = bl.span.start;
    span[1] = bl.span.end;
    const size_t n = size_t(bl.span.len()) * size_t(sn.head_dim);
    for (size_t g = 0; g < bl.k.size(); ++g) {
      if (k) std::memcpy(k + g * n, bl.k[g].v.data(), n * 4);
      if (v) std::memcpy(v + g * n, bl.v[g].v.data(), n * 4);
    }
  });
}
int kro_snapshot_storage(void* s, uint64_t* full, uint64_t* stored) {
  return guard([&] { storage_report(*static_cast<Snapshot*>(s), full, stored); });
}
int kro_snapshot_set_plan(void* s, const int64_t* p) {
  return guard([&] {
    Snapshot& sn = *static_cast<Snapshot*>(s);
    std::copy(p, p + sn.n_layers, sn.plan.p.begin());
  });
}
int kro_expand(void* s, int layer, float* k, float* v, int64_t* span) {
  return guard([&] {
    const Snapshot& sn = *static_cast<Snapshot*>(s);
    KVLayer l = expand(sn, layer);
    span[0] = l.span.start;
    span[1] = l.span.end;
    copy_kv_layer(l, k, v, sn.head_dim);
  });
}
// One restoration turn's TTFT work on the CPU, timed (harness.cpp:125-131):
// execute_restore(model, history, snapshot) then prefill(history + new,
// restored) with the attention record (the reference always captures).
// out[0] = restore seconds, out[1] = new-input prefill seconds; logits
// (optional) receives the last-row logits.
int kro_time_turn(void* mh, const int32_t* hist, int64_t L, void* snap, const int32_t* newtok,
                  int64_t n_new, double* out, float* logits) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(mh);
    std::vector<int32_t> h(hist, hist + L);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<KVLayer> restored = execute_restore(m, h, *static_cast<Snapshot*>(snap));
    auto t1 = std::chrono::steady_clock::now();
    h.insert(h.end(), newtok, newtok + n_new);
    PrefillOut pf = prefill(m, h, &restored, true);
    auto t2 = std::chrono::steady_clock::now();
    out[0] = std::chrono::duration<double>(t1 - t0).count();
    out[1] = std::chrono::duration<double>(t2 - t1).count();
    if (logits) std::memcpy(logits, pf.logits.data(), pf.logits.size() * sizeof(float));
  });
}

int kro_restore(void* mh, const int32_t* hist, int64_t n, void* snap, void** out) {
  return guard([&] {
    std::vector<int32_t> t(hist, hist + n);
    auto v = execute_restore(*static_cast<Model*>(mh), t, *static_cast<Snapshot*>(snap));
    auto* s = new KVSet;
    s->kv = std::move(v);
    *out = s;
  });
}
// Restricts a full-span KV set to per-layer suffixes [start_l, end) (a
// `preloaded` argument for prefill over restored state).
void* kro_kv_suffix(void* kvs, const int64_t* starts) {
  const auto& src = static_cast<KVSet*>(kvs)->kv;
  auto* s = new KVSet;
  for (size_t l = 0; l < src.size(); ++l) {
    KVLayer x;
    x.span = {starts[l], src[l].span.end};
    const int64_t rows = x.span.len();
    for (size_t g = 0; g < src[l].k.size(); ++g) {
      const int hd = int(src[l].k[g].c);
      Mat k(rows, hd), v(rows, hd);
      if (rows > 0) {
        std::memcpy(k.v.data(), src[l].k[g].row(starts[l]), size_t(rows * hd) * 4);
        std::memcpy(v.v.data(), src[l].v[g].row(starts[l]), size_t(rows * hd) * 4);
      }
      x.k.push_back(std::move(k));
      x.v.push_back(std::move(v));
    }
    s->kv.push_back(std::move(x));
  }
  return s;
}

// ---- timing helper for the CPU baseline (bench.py) -------------------------
// Times one layer_forward-equivalent recompute: partial prefix recompute with
// recompute_len = {p, p, ..., 0...} on a model; returns seconds.
double kro_time_partial(void* mh, const int32_t* toks, int64_t n, const int64_t* p) {
  const Model& m = *static_cast<Model*>(mh);
  std::vector<int32_t> t(toks, toks + n);
  std::vector<int64_t> pv(p, p + m.cfg.n_layers);
  auto t0 = std::chrono::steady_clock::now();
  PartialOut po = partial_prefix_recompute(m, t, pv);
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
