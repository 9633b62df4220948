// kb.hpp — internal types of the B200 Krul library (not part of the ABI).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/krul_b200.h"

namespace kb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);

#define KB_CUDA(x)                                                           \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess)                                                   \
      ::kb::fail(KRUL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
// Every kernel launch of the library is followed by KB_LAUNCH(), which also
// counts it (krul_launch_count: the bench's gpu_launches evidence).
extern std::atomic<uint64_t> g_launches;
// bumped whenever a DevBuf / PinnedBuf (re)allocates: a captured CUDA graph
// that baked in workspace addresses is stale once this moves
extern std::atomic<uint64_t> g_buf_gen;
#define KB_LAUNCH()                                   \
  do {                                                \
    ::kb::g_launches.fetch_add(1, std::memory_order_relaxed); \
    KB_CUDA(cudaGetLastError());                      \
  } while (0)

// Blocking copies/memsets that are ordered against the library's
// non-blocking streams: plain cudaMemcpy/cudaMemset run on the legacy stream,
// which does not synchronise with cudaStreamNonBlocking streams, and a
// pageable H2D cudaMemcpy may return before its DMA lands.
inline cudaError_t kb_memcpy_sync(void* d, const void* s, size_t n, cudaMemcpyKind k) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(d, s, n, k);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}
inline cudaError_t kb_memset_sync(void* d, int v, size_t n) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  e = cudaMemset(d, v, n);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

constexpr int kPageTokens = 64;  // tokens per KV page
constexpr int kFoldChunk = 256;  // estimator fold: columns per stage-1 CTA

// Model configuration (engine.hpp:17-29 + extensions).
struct Cfg {
  int N = 0, H = 0, Hkv = 0, hd = 0, d = 0, V = 0, F = 0;
  float ffn_mult = 4.f;
  int ffn_kind = 0;
  uint64_t seed = 0;
  double theta = 1e4;
  int dtype = KRUL_F32;
  int64_t max_tokens = 0;
  int qd() const { return H * hd; }
  int kvd() const { return Hkv * hd; }
  int nqkv() const { return (H + 2 * Hkv) * hd; }
};
Cfg cfg_from_desc(const krul_model_desc& d);
uint64_t config_hash(const Cfg& c);  // engine.cpp:27-36 (+ extension fold)

// Owning device allocation that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void* ensure(size_t n);  // grows (contents not preserved)
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool pageable = false;    // plain host memory (host-only snapshots, no device needed)
  bool registered = false;  // pageable memory page-locked with cudaHostRegister
  void pin();               // pageable -> registered (H2D-ready like cudaMallocHost)
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf();
  void* ensure(size_t n);
};

// Per-layer device weights, compute dtype (f32 or bf16). All projection
// matrices are stored transposed ([out][in], K-major) for the GEMM's B
// operand. SwiGLU gate/up rows are interleaved in 64-row blocks.
struct LayerW {
  void* wqkv = nullptr;  // [(H + 2 Hkv) hd][d]
  void* wo = nullptr;    // [d][H hd]
  void* w1 = nullptr;    // tanh: [F][d]; swiglu: [2F][d] interleaved
  void* w2 = nullptr;    // [d][F]
  float* b1 = nullptr;   // [F] (tanh only)
  float* b2 = nullptr;   // [d] (tanh only)
};

struct Ctx;

// A conversation: page table into the ctx KV pool plus its length.
struct Conv {
  Ctx* ctx = nullptr;
  int64_t len = 0;
  int64_t capacity = 0;
  int max_pages = 0;
  std::vector<int> pages;  // host copy [N][max_pages]
  int* d_pt = nullptr;     // device page table [N][max_pages]
  // unique per conversation object: the restore-graph cache key (a freed
  // Conv's heap address can be reused by the next one)
  uint64_t serial = 0;
  ~Conv();
};

struct Est;

// Per-launch kernel timing (krul_ktime_*): CUDA events bracket each
// instrumented launch on the stream it runs on; algorithmic flops / bytes
// are attached so the bench derives achieved TFLOP/s and GB/s per kernel
// class from the same timed step.
enum KTag { KT_GEMM = 0, KT_ATTN = 1, KT_EXPAND = 2, KT_FOLD_DECODE = 3, KT_FOLD_PREFILL = 4,
            KT_SELECT = 5, KT_COMPRESS = 6, KT_GEMM_STREAM = 7, KT_DECODE = 8, KT_LOGITS = 9,
            KT_DECODE_EXPAND = 10, KT_NTAGS = 11 };
struct KTime {
  bool on = false;
  struct Rec {
    int tag;
    double flops, bytes;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t ev();
  ~KTime();
};
// Timing events recorded while a stream is being captured must be external
// event-record nodes (a plain cudaEventRecord under capture only expresses a
// dependency and cannot be timed). A Mark is a dependency event (waited on
// by other streams) plus a timing event.
cudaError_t record_timing(cudaEvent_t e, cudaStream_t s);
struct Mark {
  cudaEvent_t dep = nullptr, tim = nullptr;
};
void record_mark(const Mark& m, cudaStream_t s);
// returns the start event (nullptr when timing is off)
cudaEvent_t kt_begin(const Ctx& c, cudaStream_t s);
void kt_end(const Ctx& c, cudaStream_t s, cudaEvent_t a, int tag, double flops, double bytes);

struct Ctx {
  int device = 0;
  Cfg cfg;
  size_t esz = 4;  // compute element size
  cudaStream_t s_comp = nullptr, s_load = nullptr, s_new = nullptr, s_est = nullptr;
  cudaStream_t s_exp = nullptr;  // expand (K5) behind the H2D copies
  int sm_count = 0;

  // weights
  DevBuf wbuf;  // one arena
  std::vector<LayerW> L;
  void* embed = nullptr;     // [V][d]
  void* unembedT = nullptr;  // [V][d]
  float* rope_cos = nullptr; // [max_tokens][hd/2] (host double -> float)
  float* rope_sin = nullptr;
  DevBuf rope;
  bool weights_ready = false;

  // KV page pool: page = [K: Hkv][P][hd] then [V^T: Hkv][hd][P]
  DevBuf pool;
  int pool_pages = 0;
  std::vector<int> free_pages;
  size_t page_elems() const { return size_t(2) * cfg.Hkv * kPageTokens * cfg.hd; }

  // workspaces (grown on demand)
  DevBuf ws_h, ws_h2, ws_xn, ws_qkv, ws_q, ws_attn, ws_hmid, ws_hmidc, ws_act, ws_y;
  DevBuf ws_tok, ws_tok2, ws_logits;
  DevBuf ws_new_h, ws_new_h2;  // new-input prefill stream
  DevBuf ws_part, ws2_part;    // split-KV attention partials per stream
  mutable DevBuf ws_gpart, ws2_gpart;  // split-K GEMM partials per stream
  // second workspace set for the concurrent new-input prefill stream
  DevBuf ws2_xn, ws2_qkv, ws2_q, ws2_attn, ws2_hmid, ws2_hmidc, ws2_act, ws2_y;

  // capture (0 off, 1 the reference's materialised attention record, 2 K2:
  // Q + softmax statistics, the estimator recomputes the probabilities)
  int capture_probs = 0;
  int cap_mode = 0;                // capture_probs when the last capture was taken
  const Conv* cap_conv = nullptr;  // the conversation the capture was taken on
  uint64_t cap_conv_serial = 0;
  std::vector<const Conv*> convs;  // live conversations (cap_conv validity)
  DevBuf cap_probs;       // [N][H][rows][W] f32 (when capture_probs)
  int64_t cap_rows = 0, cap_width = 0, cap_first_q = 0;
  bool cap_valid = false;
  DevBuf cap_mass;        // [N][H][rows] f64 region masses (classifier)
  DevBuf cap_q;           // capture mode 2: [N][rows][H*hd] rotated Q of the prefill rows (cdt)
  DevBuf cap_stats;       // capture mode 2: [N][H][rows][2] softmax (max, sum)
  bool cap_stats_log2 = false;  // the stats' domain (FA: log2)
  double cap_ifrac = 0.1, cap_rfrac = 0.1;
  int64_t cap_il = 0, cap_rs = 0;
  DevBuf dec_rows;        // [N][H][dec_pitch] f32 last decode step (pitch: 16-byte rows)
  int64_t dec_pitch = 0;
  DevBuf dec_part;        // split-key partials of the decode attention
  int64_t dec_width = 0;
  bool dec_valid = false;

  // restore staging + last measured timeline (ms from launch)
  bool tl_pending = false, tl_has_new = false;  // per-layer timeline not yet read back
  DevBuf staging;
  DevBuf cstaging;       // coded blob images (H2D target; decoded into `staging`)
  DevBuf staging2, cstaging2, batch_tok;  // restore_batch: the second staging slot, the batch's tokens
  // restore_batch graph mode: one captured DAG per (snapshot, conversation,
  // parity), launched on alternating streams with external-event hand-offs
  struct BatchGraph {
    uint64_t snap_serial = 0, conv_serial = 0, buf_gen = 0;
    int64_t L = 0, n_new = 0;
    int slot = 0;
    cudaGraphExec_t exec = nullptr;
    PinnedBuf tok, logits;
    DevBuf dtok;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    std::vector<Mark> ev;  // dependency marks only (no timing events)
    ~BatchGraph();
  };
  std::vector<BatchGraph*> bgraphs;
  cudaEvent_t b_dec[2] = {nullptr, nullptr}, b_comp[2] = {nullptr, nullptr}, b_new[2] = {nullptr, nullptr},
              b_h2d[2] = {nullptr, nullptr};
  cudaStream_t b_launch[2] = {nullptr, nullptr};
  bool kv_coding = true; // exponent-code bf16 snapshots at compress (KRUL_KV_CODING=0: off)
  PinnedBuf tok_pin;     // pinned token staging (history | new input) for async / graph H2D
  DevBuf sel_dev;        // selector (K3) candidates + results, grown once
  PinnedBuf sel_host;    // their pinned host image (one H2D, one D2H per call)
  PinnedBuf logits_pin;  // pinned logits landing buffer
  // CUDA graph of the last restore DAG (replayed when the key repeats)
  struct RestoreGraph {
    uint64_t snap_serial = 0;
    uint64_t conv_serial = 0;
    int64_t L = -1, n_new = -1;
    bool kt_on = false, logits = false;
    int capture_probs = -1;
    uint64_t buf_gen = 0;
    bool two_stream = true;
    bool fused = false;
    bool timeline = false;
    bool span = false;
    int seen = 0;  // eager runs with this key (capture on the second)
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
    std::vector<Mark> ev;  // ev0, c_end, l_end, end, h2d_end, computed[N], loaded[N], newp[N]
    double h2d = 0, expand_bytes = 0;
  } rg;
  bool use_graphs = true;
  bool two_stream = true;  // new-input prefill concurrent with the recompute (krul_set_concurrency)
  // restore + prefill DAG variant: the recompute rows ride in the new-input
  // prefill's GEMMs layer by layer (one weight pass per layer) instead of a
  // separate recompute stream (krul_set_fused_recompute). Measured slower on
  // the bench workload, so off by default.
  bool fused = false;
  // per-layer timing events in the restore graph (computed / loaded /
  // new-prefill timeline). On by default: measured, the graph without the
  // per-layer external event-record nodes runs the restore 4-7 ms slower
  // at r_c > 0 (the nodes keep the streams' kernels interleaved).
  bool timeline = true;
  // device-side spans of the weight-streaming GEMM launches (no events in
  // the stream: first-CTA entry to last-CTA exit per launch, krul_span_*)
  bool span_on = false;
  int span_next = 0;
  std::vector<double> span_bytes;
  DevBuf span_buf;
  static constexpr int kSpanSlots = 4096;
  std::vector<double> tl_compute, tl_load, tl_new;
  double tl_h2d_ms = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;

  mutable KTime kt;
  ~Ctx();
  cudaEvent_t event();  // recycled timing-capable events
  void drop_graph();
  void reset_events() { ev_next = 0; }
};

// ---- kernels (launch wrappers, .cu) ---------------------------------------
struct EpiKV {  // QKV epilogue: RoPE + paged K / V^T scatter + rotated Q
  const int* pt = nullptr;  // page table of the layer
  char* pool = nullptr;
  int64_t page_bytes = 0;
  int H = 0, Hkv = 0, hd = 0;
  int64_t pos0 = 0, q_rows = 0;
  // two row segments (fused recompute + new-input step): rows < seg_rows sit
  // at pos0 + r, rows >= seg_rows at pos1 + (r - seg_rows)
  int64_t seg_rows = INT64_MAX, pos1 = 0;
  __host__ __device__ int64_t pos(int64_t r) const { return r < seg_rows ? pos0 + r : pos1 + (r - seg_rows); }
  const float* cosT = nullptr;  // [pos][hd/2]
  const float* sinT = nullptr;
  void* q = nullptr;  // [q_rows][H*hd] cdt
};
struct Epi {  // GEMM epilogue
  enum Kind { F32 = 0, CDT = 1, RESID = 2, TANH = 3, SWIGLU = 4, NONE = 5,
              STAGE_ONLY = 6, F32_DIRECT = 7,  // 5..7: benchmark/debug only
              QKV = 10 };                      // tcgen05 path only
  int kind = F32;
  void* out = nullptr;        // F32/RESID: float*, CDT/TANH/SWIGLU: cdt*
  int64_t ldo = 0;
  const float* bias = nullptr;
  const float* resid = nullptr;  // RESID: out = acc + bias + resid
  int64_t ldr = 0;
  void* out2 = nullptr;          // RESID: optional cdt copy of out
  int64_t ldo2 = 0;
  EpiKV kv;                      // QKV
  // rows of A the caller has allocated (>= M; 0 = M): with M < 128 the
  // 1-SM kernel then loads real (ignored) rows instead of TMA out-of-bounds
  // fill, measured 77 -> 55 us on the M = 1 FFN1 (layer workspaces hold 128)
  int64_t a_rows = 0;
  // span slot of the weight-streaming GEMM launch (krul_span_enable): the
  // kernel stamps its first CTA entry / last CTA exit (%globaltimer) there
  int span = -1;
};

extern int g_gemm_force, g_gemm_splits;
void gemm_set_span(unsigned long long* d);  // [2][slots] entry (min) / exit (max) stamps  // debug knobs (krul_debug_gemm_bench)
void gemm_set_timeline(unsigned long long* d);  // debug phase stamps (krul_debug_gemm_timeline)
extern int g_attn_target, g_attn_dbg;    // debug knobs (krul_debug_attn_bench)
void attn_set_timeline(unsigned long long* d);  // debug phase stamps (krul_debug_attn_timeline)
// True when gemm() will take the tcgen05 path for these operands (fused
// epilogues such as Epi::QKV exist only there).
bool gemm_uses_tc(const Ctx& c, const void* A, int64_t lda, const void* B, int64_t ldb);
// C = A[M,K] * B[N,K]^T with epilogue; A,B in compute dtype.
void gemm(const Ctx& c, cudaStream_t s, int64_t M, int64_t N, int64_t K,
          const void* A, int64_t lda, const void* B, int64_t ldb, const Epi& e);

void launch_embed(const Ctx& c, cudaStream_t s, const int32_t* tok, int64_t n, float* h);
void launch_rmsnorm(const Ctx& c, cudaStream_t s, const float* h, int64_t rows, void* xn);
// qkv f32 [rows][(H+2Hkv)hd] -> rope, K/V^T into pages at [pos0, pos0+rows),
// Q (roped, cdt) for rows < q_rows.
void launch_rope_scatter(const Ctx& c, cudaStream_t s, const float* qkv, int64_t rows,
                         int64_t pos0, int64_t q_rows, void* q, const Conv& conv, int layer,
                         int64_t seg_rows = INT64_MAX, int64_t pos1 = 0);
struct DevBuf;
struct AttnArgs {
  const void* q = nullptr;  // [rows][H*hd] cdt
  int64_t rows = 0, pos0 = 0;
  void* out = nullptr;      // [rows][H*hd] cdt
  float* probs = nullptr;   // optional [H][rows][ld_probs]
  int64_t ld_probs = 0;
  int64_t probs_row0 = 0;   // row offset into the capture
  int64_t probs_rows = 0;   // rows per head in the capture
  double* mass = nullptr;   // optional [H][mass_rows] region mass
  int64_t mass_rows = 0;
  // K2 (estimator prefill fold without the probability record): per row the
  // softmax statistics (max, sum) [H][mass_rows][2] -- natural-log domain
  // (SIMT: P = exp(s - m) / l) or log2 domain (FA: P = exp2(s log2e - m) / l)
  // -- and a copy of the rotated Q rows [rows][H * hd]
  float* stats = nullptr;
  void* q_save = nullptr;
  int64_t il = 0, rs = 0;   // classifier regions [0,il) U [rs, W)
  DevBuf* part = nullptr;   // split-KV scratch owned by the calling stream
};
void launch_attention(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                      const AttnArgs& a);
bool attention_tc_supported(const Ctx& c, const AttnArgs& a);
void launch_attention_tc(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                         const AttnArgs& a, DevBuf& scratch);
void launch_bias_act(const Ctx& c, cudaStream_t s, const float* in, int64_t rows, int64_t F,
                     const float* b1, int kind, void* out);  // tanh(x+b) or swiglu pairs
void launch_resid_add(const Ctx& c, cudaStream_t s, const float* y, const float* bias,
                      const float* resid, int64_t rows, int64_t d, float* out, void* outc);
void launch_logits(const Ctx& c, cudaStream_t s, const float* h_last, float* logits);
void launch_convert_weights(const Ctx& c, cudaStream_t s, const float* src, void* dst,
                            int64_t rows, int64_t cols, int transpose, int interleave64);
void launch_init_uniform(const Ctx& c, cudaStream_t s, void* dst, int64_t n, uint64_t seed,
                         uint64_t stream_id, float bound);
void launch_init_uniform_f32(cudaStream_t s, float* dst, int64_t n, uint64_t seed,
                             uint64_t stream_id, float bound);

// KV page transfer helpers (f32 host views)
void launch_kv_gather(const Ctx& c, cudaStream_t s, const Conv& conv, int layer, int64_t start,
                      int64_t end, float* k, float* v);  // -> [Hkv][rows][hd] f32 device
void launch_kv_scatter_f32(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                           int64_t start, int64_t end, const float* k, const float* v);
// Blob (cdt [2][Hkv][rows][hd], rows = [blob_start, L)) -> pages of `layer`
// for positions [from, L).
// coded blob -> owners' pages in one pass (kvcode format, bf16, hd = 128)
void launch_ec_decode_expand(const Ctx& c, cudaStream_t s, const void* blob, int64_t n_chunks,
                             const uint16_t* lut, int64_t blob_start, int64_t L, const Conv& conv,
                             const int* owners, const int64_t* from, double coded_bytes, int ctas_per_sm = 4);
void launch_expand(const Ctx& c, cudaStream_t s, const void* blob, int64_t blob_start,
                   int64_t L, const Conv& conv, int layer, int64_t from);
// Pages -> blob (compress, K8); mean-merge rows [merge_from, L) with `other`.
void launch_compress(const Ctx& c, cudaStream_t s, const Conv& conv, int deep, int shallow,
                     int64_t blob_start, int64_t L, int64_t merge_from, void* blob);
void launch_cvt_to_f32(const Ctx& c, cudaStream_t s, const void* src, float* dst, int64_t n);
void launch_cvt_from_f32(const Ctx& c, cudaStream_t s, const float* src, void* dst, int64_t n);

// estimator kernels
void launch_fold_decode(cudaStream_t s, const float* rows, int64_t W, int H, const int* d_layers,
                        int n, double* sums, double* partial, int64_t partial_cap);
void launch_fold_prefill(cudaStream_t s, const float* probs, int64_t rows, int64_t W, int H,
                         const int* d_layers, int n, double* sums, double* partial,
                         int64_t partial_cap);
void launch_finalize(cudaStream_t s, const double* sums, int n, int H, double* D);
// K2 (fold.cu): the prefill probabilities of the tracked layers for key
// columns [c0, c0 + wc), recomputed from the saved Q, the paged K and the
// softmax statistics -> out [n][H][rows][wc] f32 (zero past a row's causal
// width or the key count)
void launch_prefill_probs(const Ctx& c, cudaStream_t s, const Conv& conv, const int* d_layers, int n,
                          int64_t rows, int64_t first_q, int64_t c0, int wc, float* out);
// K1 decode fold (fold.cu): rows [layer][head][.] f32 with 16-byte aligned
// strides (head stride >= the 16-byte-padded width); adds into seg, the
// resident per-(head, segment, pair) f64 slots ([H][seg_S][P], zero at
// creation, seg_S = fold_seg_slots(H, sms)); launch_fold_collect moves the
// slots into sums[p][h] and zeroes them.
int fold_seg_slots(int H, int sms);
void fold_set_timeline(unsigned long long* d);  // debug: per-CTA %globaltimer stamps [cta][8]
// stride > 1: the sampled token subset (opt-in, krul_est_set_sampling):
// 64-column blocks phase, phase + stride, ... folded, scaled by W / sampled
void launch_fold_direct(cudaStream_t s, const float* rows, int64_t layer_stride, int64_t head_stride, int64_t W,
                        int H, const int* d_layers, int n, double* seg, int seg_S, int sms, int stride = 1,
                        int phase = 0);
void launch_fold_collect(cudaStream_t s, double* seg, int seg_S, int n, int H, double* sums);
// selector: candidates sorted on device then greedily matched
void launch_select(cudaStream_t s, const double* cand_d, const int* cand_i, const int* cand_j,
                   int n_cand, int quota, int* out_i, int* out_j, double* out_d, int* out_n);

}  // namespace kb
