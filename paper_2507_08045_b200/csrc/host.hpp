// host.hpp — host-side building blocks shared by the C ABI translation units.
#pragma once
#include <set>
#include <string>
#include <vector>

#include "kb.hpp"
#include "kvcode.hpp"

namespace kb {

struct WS {  // per-stream activation workspace
  float *h = nullptr, *h2 = nullptr, *qkv = nullptr, *hmid = nullptr;
  void *xn = nullptr, *q = nullptr, *attn = nullptr, *hmidc = nullptr, *act = nullptr;
  DevBuf* part = nullptr;
};

Ctx* ctx_create(int device, const krul_model_desc& desc);
void weights_upload_f32(Ctx& c, const float* w, int64_t n);
void weights_init_device(Ctx& c, uint64_t seed);
Conv* conv_create(Ctx& c, int64_t capacity);
WS ws_get(Ctx& c, int set, int64_t rows);
// Fused recompute + new-input step of one layer: rows [0, n_new) are the new
// input (at pos0 + r), rows [n_new, rows) the history prefix being recomputed
// (positions 0..); rec_out of them feed the next layer. The step waits for
// `waits` (the layer's loaded suffix) before it starts; `computed` is
// recorded once the layer's recomputed K/V are in the pages.
struct FusedSeg {
  int64_t n_new = 0, rec_out = 0;
  const cudaEvent_t* waits = nullptr;
  int n_waits = 0;
  const Mark* computed = nullptr;
};
void layer_forward(Ctx& c, cudaStream_t s, const WS& w, Conv& conv, int l, const float* h_in,
                   int64_t rows, int64_t pos0, int64_t out_rows, float* h_out,
                   const AttnArgs* cap, const FusedSeg* fs = nullptr);
void forward_fused(Ctx& c, cudaStream_t s, int set, Conv& conv, const int32_t* d_new, int64_t n,
                   int64_t L, const int32_t* d_hist, const std::vector<int64_t>& p, float* d_logits,
                   const Mark* loaded, const Mark* computed, const Mark* layer_done, const Mark* compute_end);
void check_tokens(const Ctx& c, const int32_t* t, int64_t n);
int32_t* upload_tokens(Ctx& c, cudaStream_t s, const int32_t* t, int64_t n, DevBuf& buf);
void forward_rows(Ctx& c, cudaStream_t s, int set, Conv& conv, const int32_t* d_tok, int64_t n,
                  int64_t pos0, float* d_logits, const std::vector<cudaEvent_t>* waits,
                  const Mark* layer_done = nullptr);
void prefill(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, float* logits);
void prefill_new(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, float* logits);
void decode_step(Ctx& c, Conv& conv, int32_t tok, float* logits);
void enqueue_partial(Ctx& c, cudaStream_t s, Conv& conv, const int32_t* d_tok,
                     const std::vector<int64_t>& p, bool full_last, const Mark* ev);
void check_plan_shape(const Ctx& c, int64_t n, const int64_t* p, int np);
void partial_recompute(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, const int64_t* p,
                       int np);

// ---- scheduler arithmetic (scheduler.cpp) ----------------------------------
struct Cost {
  double f = 312e12, b = 139e9, ffn_mult = 4.0;
  int64_t kv_dim = 0, q_dim = 0, ffn_hidden = 0;
  double bpe = 4.0;
  int ffn_kind = 0;
  double layer_flops(int64_t p, int64_t d) const;
  double blob_bytes(int64_t span, int64_t d) const;
};
Cost cost_from(const krul_cost_model* m);
int quota(int n_layers, double r_l);
std::vector<krul_blob_spec> blob_specs(const std::vector<int64_t>& p, int64_t L,
                                       const krul_pair* pairs, int np);
std::vector<int64_t> build_plan(int64_t L, int N, double r_c, const krul_pair* pairs, int np);
std::vector<int64_t> uniform_plan(int64_t L, int N, double r_c);
double calibrate(const Cost& c, int N, int64_t L, int64_t d, const krul_pair* pairs, int np,
                 const double* grid, int ng);
std::vector<double> default_grid(double step);
int validate_plan(int64_t L, const std::vector<int64_t>& p, const krul_pair* pairs, int np);
int validate_strategy(const krul_pair* pairs, int np, const std::set<int>& shared, bool exhausted,
                      const std::set<int>& ir, int n_layers, double r_l, std::string* lines);

// ---- compressed KV store ---------------------------------------------------
// Container metadata the hot path does not use but the KRUL v1 container
// carries (kvstore.hpp:46-59): conversation id, the selector's quota flag
// and the layer classifier report.
struct SnapMeta {
  std::string conversation_id;
  bool exhausted_before_quota = false;
  std::vector<int> ir_layers, non_ir_layers;
  std::vector<double> avg_weight_sum;
  std::vector<int> shared;  // strategy.shared as loaded; empty = derived from the pairs
};

struct Snapshot {
  Ctx* ctx = nullptr;  // null for a host-only snapshot (container load without a device)
  size_t esz = 4;      // element bytes of `host` (ctx compute dtype; 4 when host-only)
  SnapMeta meta;
  uint64_t config_hash = 0;
  int N = 0, Hkv = 0, hd = 0;
  int64_t L = 0;
  int mode = 0;
  std::vector<krul_pair> pairs;
  std::vector<int64_t> p;
  struct Blob {
    int owners[2];
    int64_t start, end;
    size_t off;    // byte offset of the raw blob (device staging; `host` when raw)
    size_t bytes;  // raw bytes
    size_t coff = 0, cbytes = 0;  // coded image in `host` (coded stores)
    uint32_t ec_chunks = 0;
  };
  std::vector<Blob> blobs;
  PinnedBuf host;  // raw: all blobs, compute dtype, [K: Hkv][rows][hd][V: ...];
                   // coded: the exponent-coded images (kvcode.hpp)
  size_t total = 0;   // raw bytes of all blobs (device staging size)
  bool coded = false;
  std::unique_ptr<EcCode> code;  // the snapshot's exponent code (coded stores)
  DevBuf lut_dev;                // its decode LUT on the device
  size_t ctotal = 0;             // coded image bytes
  uint64_t serial = 0;  // changes whenever blobs or plan change (graph cache key)
};
uint64_t next_serial();
int validate_plan_snapshot(const std::vector<int64_t>& p, int64_t L, const Snapshot& s);
// KRUL v1 container (host_container.cpp).
struct LoadError : Error {
  std::string field;
  LoadError(std::string f, const std::string& m) : Error(KRUL_E_SNAPSHOT_LOAD, f + ": " + m), field(std::move(f)) {}
};
uint32_t crc32(const void* p, size_t n, uint32_t crc = 0);
// exponent-coded store (host_kvcode.cpp)
void snapshot_encode(Ctx& c, Snapshot& s, const char* dev_raw, cudaStream_t st);
const char* snapshot_raw_blob(const Snapshot& s, int b, std::vector<uint16_t>& tmp);
uint64_t container_size(const Snapshot& s);
void container_write(const Snapshot& s, char* out);  // exactly container_size bytes
void container_write_file(const Snapshot& s, const char* path);
Snapshot* container_read(Ctx* c, const char* buf, size_t n, const uint64_t* expected_hash);
Snapshot* container_read_file(Ctx* c, const char* path, const uint64_t* expected_hash);
void restore_timeline(Ctx& c);  // reads the last restore's per-layer events
void restore(Ctx& c, Conv& conv, Snapshot& snap, const int32_t* hist, int64_t L,
             krul_restore_stats* st, const int32_t* new_tok, int64_t n_new, float* logits,
             double* ttft_ms);
void restore_batch(Ctx& c, int n, Conv* const* convs, Snapshot* const* snaps, const int32_t* const* hists,
                   const int64_t* Ls, const int32_t* const* news, const int64_t* n_news, float* logits,
                   double* ttft_ms, double* total_ms);

}  // namespace kb
