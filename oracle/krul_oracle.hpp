// krul_oracle.hpp — CPU restatement of the Krul reference hot path.
//
// TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200
// product under paper_2507_08045_b200/. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it. The
// product never links, calls or falls back to it.
//
// It restates, function by function, the reference C++ under
// /root/reference/proj (cited as `proj/<file>:<line>`), which cannot be built
// in this image (Eigen3 and the vendored single headers are absent; see
// DESIGN.md "Oracle"). Eigen is replaced by a row-major float matrix. Where
// the reference arithmetic is defined by Eigen's reduction order (GEMMs,
// squaredNorm, exp) the restatement uses a plain left-to-right order, so
// floating-point parity at the Eigen boundary is "unpinned" and
// is checked by the reference's own self-consistency tolerances instead.
// Integer/plan/selection arithmetic is restated exactly.
#pragma once

#include <cstddef>
#include <cstdint>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace kro {

// ---- errors (proj/include/krul/common.hpp:25-63) -------------------------
// One status code per reference exception type; the C-ABI maps them 1:1.
enum Status : int {
  kOk = 0,
  kConfig = 1,
  kRestorationGap = 2,
  kStateCorruption = 3,
  kAccounting = 4,
  kPlanInvalid = 5,
  kClassification = 6,
  kSnapshot = 7,
  kSnapshotLoad = 8,
};

struct Error : std::runtime_error {
  Status code;
  std::string field;  // SnapshotLoadError field name (common.hpp:58-63)
  Error(Status c, const std::string& msg, std::string f = "")
      : std::runtime_error(msg), code(c), field(std::move(f)) {}
};

[[noreturn]] void fail(Status c, const std::string& msg);

struct Span {  // TokenSpan, common.hpp:13-23
  int64_t start = 0, end = 0;
  int64_t len() const { return end - start; }
  bool empty() const { return end <= start; }
  bool operator==(const Span&) const = default;
};

// mt19937_64 -> 24-bit mantissa mapping (common.hpp:68-86).
struct Uniform {
  std::mt19937_64 g;
  explicit Uniform(uint64_t seed) : g(seed) {}
  float next(float lo, float hi) {
    uint32_t top = static_cast<uint32_t>(g() >> 40);
    float u = static_cast<float>(top) * (1.0f / 16777216.0f);
    return lo + (hi - lo) * u;
  }
  uint64_t index(uint64_t n) { return g() % n; }
};

uint64_t fnv1a64(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ull);
uint32_t crc32(const void* p, size_t n, uint32_t crc = 0);

// ---- dense row-major matrix (replaces Eigen::MatrixXf) -------------------
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<float> v;
  Mat() = default;
  Mat(int64_t rows, int64_t cols) : r(rows), c(cols), v(size_t(rows * cols), 0.f) {}
  float& at(int64_t i, int64_t j) { return v[size_t(i * c + j)]; }
  float at(int64_t i, int64_t j) const { return v[size_t(i * c + j)]; }
  float* row(int64_t i) { return v.data() + i * c; }
  const float* row(int64_t i) const { return v.data() + i * c; }
};

// ---- engine (proj/include/krul/engine.hpp, proj/src/engine.cpp) ---------
// Extensions beyond the reference (documented in DESIGN.md): n_kv_heads
// (GQA), ffn_kind (0 = tanh+bias reference FFN, 1 = SwiGLU with a gain-less
// RMSNorm before it, as Llama), rope_theta.
// Defaults reproduce the reference architecture exactly.
struct ModelConfig {
  int n_layers = 4, n_heads = 2, head_dim = 8, d_model = 16, vocab = 64;
  float ffn_mult = 4.0f;
  uint64_t seed = 0;
  int n_kv_heads = 0;  // 0 -> n_heads
  int ffn_kind = 0;
  double rope_theta = 10000.0;

  int kv_heads() const { return n_kv_heads > 0 ? n_kv_heads : n_heads; }
  int ffn_hidden() const;
  void validate() const;
  uint64_t hash() const;
};

struct LayerW {
  Mat wq, wk, wv, wo;  // [d x H*hd], [d x Hkv*hd] x2, [H*hd x d]
  Mat w1;              // [d x F] (tanh: W1; swiglu: gate)
  Mat wu;              // swiglu only: up [d x F]
  std::vector<float> b1, b2;
  Mat w2;  // [F x d]
};

struct Model {
  ModelConfig cfg;
  Mat embed, unembed;  // [V x d], [d x V]
  std::vector<LayerW> layers;
};

Model build_model(const ModelConfig& cfg);  // engine.cpp:361-395

struct KVLayer {  // KVCacheLayer, engine.hpp:31-39 (per kv head [rows x hd])
  std::vector<Mat> k, v;
  Span span;
};

struct LayerAttn {
  std::vector<Mat> prefill;  // per head [rows x width]
};
struct AttnRecord {
  int64_t first_q = 0;
  std::vector<LayerAttn> layers;
  int64_t rows() const {
    return layers.empty() || layers[0].prefill.empty() ? 0 : layers[0].prefill[0].r;
  }
  int64_t width() const {
    return layers.empty() || layers[0].prefill.empty() ? 0 : layers[0].prefill[0].c;
  }
};

struct PrefillOut {
  std::vector<float> logits;
  std::vector<KVLayer> kv;
  AttnRecord attn;
};

PrefillOut prefill(const Model& m, const std::vector<int32_t>& toks,
                   const std::vector<KVLayer>* preloaded, bool capture);

struct DecodeOut {
  std::vector<float> logits;
  std::vector<Mat> rows;  // per layer [H x (s+1)]
};
DecodeOut decode_step(const Model& m, std::vector<KVLayer>& kv, int32_t tok);

struct PartialOut {
  std::vector<KVLayer> kv;
  bool has_final = false;
  Mat final_hidden;
};
PartialOut partial_prefix_recompute(const Model& m,
                                    const std::vector<int32_t>& toks,
                                    const std::vector<int64_t>& recompute_len);

// ---- analysis (proj/src/analysis.cpp) ------------------------------------
struct ClassReport {
  std::vector<int> ir, non_ir;
  std::vector<double> avg;
};
ClassReport classify_layers(const AttnRecord& rec, double gamma,
                            double initial_frac, double recent_frac);

double stable_sq(const float* a, const float* b, int64_t n);  // analysis.hpp:37-50

struct Accumulator {  // SimilarityAccumulator, analysis.hpp:66-94
  std::vector<int> layers;
  int H = 1;
  std::vector<std::pair<int, int>> pairs;
  std::vector<double> sums;  // [pair*H + h]
  bool prefill_done = false;
  int64_t prefill_rows = 0, decode_steps = 0;

  Accumulator(std::vector<int> ir, int n_heads);
  void fold_prefill(const AttnRecord& rec);
  // rows_per_layer[l] is [H x width] (absolute layer index).
  void fold_decode(const std::vector<Mat>& rows_per_layer);
  // values [n x n] row-major over sorted `layers`.
  std::vector<double> finalize() const;
};

// ---- strategy (proj/src/strategy.cpp) ------------------------------------
struct Pair {
  int shallow = 0, deep = 0;
  double distance = 0.0;
  bool operator==(const Pair&) const = default;
};
struct Strategy {
  std::vector<Pair> pairs;
  std::set<int> shared;
  bool exhausted = false;
  bool operator==(const Strategy&) const = default;
};
int shared_layer_quota(int n_layers, double r_l);
// D is [n x n] over sorted unique `dm_layers`.
Strategy select_strategy(const std::vector<double>& D,
                         const std::vector<int>& dm_layers,
                         const std::vector<int>& ir, double r_l, int n_layers);
// bitmask of violation kinds: 1 orientation, 2 range, 4 non-I-R, 8 reuse,
// 16 distance order, 32 shared size, 64 quota shortfall.
int validate_strategy(const Strategy& s, const std::vector<int>& ir,
                      int n_layers, double r_l);

// ---- plan + kvstore (proj/include/krul/plan.hpp, proj/src/kvstore.cpp) --
struct Plan {
  std::vector<int64_t> p;  // recompute_len
  int64_t L = 0;
  Span load_span(int l) const { return {p.at(size_t(l)), L}; }
};

struct BlobSpec {
  std::vector<int> owners;
  Span span;
  bool operator==(const BlobSpec&) const = default;
};
std::vector<BlobSpec> plan_blob_specs(const Strategy& s, const Plan& plan);

struct Blob {
  std::vector<int> owners;
  Span span;
  std::vector<Mat> k, v;  // per kv head [rows x hd]
};
struct Snapshot {
  uint32_t version = 1;
  std::string id;
  uint64_t config_hash = 0;
  int n_layers = 0, n_heads = 0, head_dim = 0;
  int64_t L = 0;
  int mode = 0;  // 0 mean, 1 keep-deeper
  Strategy strategy;
  Plan plan;
  ClassReport classifier;
  std::vector<Blob> blobs;
};
Snapshot compress_and_snapshot(const std::vector<KVLayer>& kv,
                               const Strategy& s, const Plan& plan, int mode,
                               const std::string& id, const ModelConfig& cfg);
KVLayer expand(const Snapshot& snap, int layer);
void storage_report(const Snapshot& snap, uint64_t* full, uint64_t* stored);

// ---- scheduler (proj/src/scheduler.cpp) -----------------------------------
struct CostModel {
  double f_peak = 312e12, b_peak = 139e9, ffn_mult = 4.0;
  double layer_flops(int64_t p, int64_t d) const;
  double prefill_flops(int64_t n, int64_t hist, int64_t d, int N) const;
  double blob_bytes(int64_t span, int64_t d) const;
};
Plan build_plan(int64_t L, int N, double r_c, const Strategy& s);
Plan uniform_plan(int64_t L, int N, double r_c);
double calibrate_rc(const CostModel& c, int N, int64_t L, int64_t d,
                    const Strategy& s, const std::vector<double>& grid);
std::vector<double> default_rc_grid(double step);
// bitmask: 1 bounds, 2 monotonicity, 4 totals, 8 coverage
int validate_plan(const Plan& plan, const Strategy& s);
int validate_plan_snapshot(const Plan& plan, const Snapshot& snap);

struct Task {
  int layer = 0;
  double start = 0, end = 0;
};
struct Trace {
  std::vector<Task> compute, load;
  double makespan = 0, compute_finish = 0, load_finish = 0;
  double bubble_compute = 0, bubble_load = 0;
};
Trace simulate_pipeline(const Plan& plan, const Strategy& s,
                        const CostModel& c, int64_t d);

std::vector<KVLayer> execute_restore(const Model& m,
                                     const std::vector<int32_t>& history,
                                     const Snapshot& snap);

}  // namespace kro
