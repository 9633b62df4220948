/* krul_b200.h — C ABI of the B200-native Krul state-restoration hot path.
 *
 * This is the drop-in boundary. The reference
 * (/root/reference/proj) is a C++ static library consumed through
 * proj/include/krul/ headers; it has no FFI. Each entry point below replaces one
 * reference call on the hot path (cited as `proj/<file>:<line>`); the C++
 * drop-in include/krul_b200.hpp (compiled against the reference's own
 * krul/common.hpp + krul/plan.hpp, tests/cpp/test_shim.cpp) and the Python
 * mirror in paper_2507_08045_b200/ are thin layers over exactly these symbols.
 *
 * Conventions
 *  - Every function returns a krul_status (0 = KRUL_OK). Errors are raised
 *    before any device work is enqueued, mirroring the reference's
 *    "validate before compute" contract (engine.cpp:452-464,
 *    scheduler.cpp:331-336). krul_last_error() returns the message of the
 *    calling thread's last failure; codes map 1:1 to the reference's
 *    exception types (common.hpp:25-63).
 *  - Plain pointers and sizes only. Host arrays are row-major. Tensors
 *    crossing the ABI as float are f32; device storage may be bf16.
 *  - A krul_ctx owns one CUDA device, its weights and streams. Calls on one
 *    ctx must come from one host thread at a time.
 */
#ifndef KRUL_B200_H_
#define KRUL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRUL_ABI_VERSION 1

typedef enum {
  KRUL_OK = 0,
  KRUL_E_CONFIG = 1,            /* ConfigError */
  KRUL_E_RESTORATION_GAP = 2,   /* RestorationGapError */
  KRUL_E_STATE_CORRUPTION = 3,  /* StateCorruptionError */
  KRUL_E_ACCOUNTING = 4,        /* AccountingError */
  KRUL_E_PLAN_INVALID = 5,      /* PlanInvalidError */
  KRUL_E_CLASSIFICATION = 6,    /* ClassificationError */
  KRUL_E_SNAPSHOT = 7,          /* SnapshotError */
  KRUL_E_SNAPSHOT_LOAD = 8,     /* SnapshotLoadError */
  KRUL_E_CUDA = 9,              /* CUDA runtime / launch failure */
  KRUL_E_ARG = 10               /* bad pointer / size at the ABI */
} krul_status;

typedef enum { KRUL_F32 = 0, KRUL_BF16 = 1 } krul_dtype;
typedef enum { KRUL_FFN_TANH = 0, KRUL_FFN_SWIGLU = 1 } krul_ffn_kind;
typedef enum { KRUL_MERGE_MEAN = 0, KRUL_MERGE_KEEP_DEEPER = 1 } krul_merge_mode;

typedef struct krul_ctx krul_ctx;
typedef struct krul_conv krul_conv;
typedef struct krul_est krul_est;
typedef struct krul_snapshot krul_snapshot;

/* ModelConfig (engine.hpp:17-29). n_kv_heads / ffn_kind / rope_theta are
 * documented extensions; n_kv_heads == n_heads, FFN_TANH, 1e4 is the
 * reference architecture. */
typedef struct {
  int n_layers;
  int n_heads;
  int n_kv_heads;
  int head_dim;
  int d_model;
  int vocab_size;
  float ffn_mult;
  int ffn_kind;
  uint64_t seed;
  double rope_theta;
  int dtype;          /* krul_dtype: F32 = parity mode, BF16 = tcgen05 path */
  int64_t max_tokens; /* per-conversation capacity (RoPE table, workspaces) */
} krul_model_desc;

/* StrategyPair (strategy.hpp:18-24). */
typedef struct {
  int shallow;
  int deep;
  double distance;
} krul_pair;

/* CostModel (scheduler.hpp:14-39). The trailing fields extend the
 * reference formulas to GQA / SwiGLU / bf16 storage; all-zero keeps the
 * reference's f32-MHA arithmetic (parity mode). */
typedef struct {
  double f_peak;         /* recompute throughput, flop/s */
  double b_peak;         /* host-to-device load bandwidth, bytes/s */
  double ffn_mult;
  int64_t kv_dim;        /* n_kv_heads * head_dim (0 = reference formula) */
  int64_t q_dim;         /* n_heads * head_dim */
  int64_t ffn_hidden;    /* F */
  double bytes_per_elem; /* stored KV element size (4 = reference f32) */
  int ffn_kind;          /* krul_ffn_kind */
} krul_cost_model;

/* BlobSpec (kvstore.hpp:28-33); owners[1] = -1 for an unpaired layer. */
typedef struct {
  int owners[2];
  int64_t start;
  int64_t end;
} krul_blob_spec;

/* Measured restore timeline (device CUDA events, ms from restore launch). */
typedef struct {
  double restore_ms;      /* launch -> every layer restored */
  double compute_ms;      /* recompute stream finish */
  double load_ms;         /* load stream finish */
  double bubble_compute;  /* (makespan - compute_finish) / makespan */
  double bubble_load;
  double h2d_bytes;
  double expand_bytes;    /* algorithmic bytes moved by the expand kernels */
  double recompute_flops;
  double h2d_ms;          /* copy-engine finish of the last blob */
} krul_restore_stats;

int krul_abi_version(void);
int krul_last_error(char* buf, size_t n);

/* ---- context / weights ------------------------------------------------ */
int krul_ctx_create(int device, const krul_model_desc* desc, krul_ctx** out);
int krul_ctx_destroy(krul_ctx* ctx);
int krul_ctx_sync(krul_ctx* ctx);
int krul_config_hash(const krul_model_desc* desc, uint64_t* out); /* engine.cpp:27-36 */
/* Weights in the reference draw order (engine.cpp:368-393), f32. */
int krul_weights_upload_f32(krul_ctx* ctx, const float* w, int64_t n);
/* Counter-based uniform init on device (perf configs; same bound). */
int krul_weights_init_device(krul_ctx* ctx, uint64_t seed);

/* ---- conversations: paged KV cache ----------------------------------- */
int krul_conv_create(krul_ctx* ctx, int64_t capacity_tokens, krul_conv** out);
int krul_conv_destroy(krul_conv* conv);
int krul_conv_length(krul_conv* conv, int64_t* len);
/* K/V of one layer over [start, end) as f32 [kv_heads][rows][head_dim]. */
int krul_conv_kv_read(krul_conv* conv, int layer, int64_t start, int64_t end,
                      float* k, float* v);
int krul_conv_kv_write(krul_conv* conv, int layer, int64_t start, int64_t end,
                       const float* k, const float* v);

/* ---- engine (engine.hpp:106-139) -------------------------------------- */
/* capture_probs != 0 keeps the full prefill attention on device (f32
 * [N][H][rows][width]); decode rows are always kept for the estimator.
 * The classifier regions (ClassifierConfig initial/recent fractions,
 * analysis.hpp:15-21) are reduced inside the attention kernel and must be
 * set before the prefill they classify. */
int krul_set_capture(krul_ctx* ctx, int capture_probs);
int krul_set_classifier_regions(krul_ctx* ctx, double initial_frac,
                                double recent_frac);
/* Fresh causal prefill over tokens[0, n)  (engine.cpp:282-340). */
int krul_prefill(krul_ctx* ctx, krul_conv* conv, const int32_t* tokens,
                 int64_t n, float* logits);
/* New-input prefill over the conversation's restored KV [0, L): tokens are
 * the n_new new ids at positions [L, L + n_new)  (engine.cpp:401-404). */
int krul_prefill_new(krul_ctx* ctx, krul_conv* conv, const int32_t* tokens,
                     int64_t n_new, float* logits);
/* decode_step (engine.cpp:406-446). */
int krul_decode_step(krul_ctx* ctx, krul_conv* conv, int32_t token,
                     float* logits);
/* Pyramid recompute of per-layer prefixes (engine.cpp:448-489). */
int krul_partial_recompute(krul_ctx* ctx, krul_conv* conv,
                           const int32_t* tokens, int64_t n,
                           const int64_t* recompute_len, int n_plan);
/* Captured prefill attention of (layer, head) -> [rows x width] f32. */
int krul_capture_prefill(krul_ctx* ctx, int layer, int head, float* out,
                         int64_t* rows, int64_t* width);
/* Last decode step's rows -> [n_layers][n_heads][width] f32. */
int krul_capture_decode(krul_ctx* ctx, float* out, int64_t* width);

/* ---- analysis: classifier + streaming estimator (analysis.hpp) -------- */
/* classify_layers over the last prefill (analysis.cpp:20-63); region
 * masses are produced by the attention kernel itself. */
int krul_classify(krul_ctx* ctx, double gamma, double initial_frac,
                  double recent_frac, double* avg_weight_sum, int* is_ir);
int krul_est_create(krul_ctx* ctx, const int* ir_layers, int n,
                    krul_est** out);
int krul_est_destroy(krul_est* est);
/* Fold the last prefill / last decode step captured on device. */
int krul_est_fold_prefill(krul_est* est);
int krul_est_fold_decode(krul_est* est);
/* Host-fed variants (tests): probs [N][H][rows][width], rows [N][H][width]. */
int krul_est_fold_prefill_host(krul_est* est, const float* probs, int n_layers,
                               int64_t rows, int64_t width);
int krul_est_fold_decode_host(krul_est* est, const float* rows, int n_layers,
                              int64_t width);
/* Opt-in sampled token subset for the decode folds (north_star; not in the
 * reference, so never used by the parity runs): fold every stride-th
 * 64-column block of the attention row (phase = decode step mod stride, so
 * each block is folded once per stride steps), scaled by W / sampled
 * columns. stride 1 (default) folds every column exactly as the reference. */
int krul_est_set_sampling(krul_est* est, int stride);
int krul_est_sums(krul_est* est, double* sums); /* [pairs * n_heads] */
int krul_est_finalize(krul_est* est, double* D); /* [n x n] */
int krul_est_counts(krul_est* est, int64_t* prefill_rows, int64_t* decode_steps);

/* ---- strategy selector (strategy.cpp:16-74), K3 on device ------------- */
int krul_quota(int n_layers, double r_l, int* out);
int krul_select(krul_ctx* ctx, const double* D, const int* dm_layers, int n,
                const int* ir_layers, int n_ir, double r_l, int n_layers,
                krul_pair* out, int* n_out, int* exhausted);

/* validate_strategy (strategy.cpp:76-131): violation bitmask 1 pair
 * orientation, 2 layer range, 4 non-I-R member, 8 layer reuse, 16 distance
 * order, 32 shared size, 64 quota shortfall; `details` (optional) receives
 * the reference's "kind: detail" lines, newline-separated. */
int krul_validate_strategy(const krul_pair* pairs, int n_pairs, const int* shared, int n_shared,
                           int exhausted, const int* ir_layers, int n_ir, int n_layers, double r_l,
                           int* mask, char* details, size_t details_cap);

/* ---- scheduler (scheduler.cpp:15-318), host --------------------------- */
int krul_build_plan(int64_t L, int n_layers, double r_c, const krul_pair* pairs,
                    int n_pairs, int64_t* recompute_len);
int krul_uniform_plan(int64_t L, int n_layers, double r_c, int64_t* recompute_len);
int krul_default_rc_grid(double step, double* out, int* n);
int krul_calibrate_rc(const krul_cost_model* cost, int n_layers, int64_t L,
                      int64_t d, const krul_pair* pairs, int n_pairs,
                      const double* grid, int n_grid, double* r_c);
/* Violation bitmask: 1 bounds, 2 monotonicity, 4 totals, 8 coverage. */
int krul_validate_plan(int64_t L, const int64_t* recompute_len, int n_layers,
                       const krul_pair* pairs, int n_pairs, int* mask);
int krul_blob_specs(int64_t L, const int64_t* recompute_len, int n_layers,
                    const krul_pair* pairs, int n_pairs, krul_blob_spec* out,
                    int* n_out);
/* out[0..4] = makespan, compute_finish, load_finish, bubble_c, bubble_l. */
int krul_simulate(int64_t L, const int64_t* recompute_len, int n_layers,
                  const krul_pair* pairs, int n_pairs,
                  const krul_cost_model* cost, int64_t d, double* out);

/* ---- compressed KV store (kvstore.cpp:173-358) ------------------------ */
/* End-of-turn snapshot of conv's KV [0, L) into pinned host blobs (K8). */
int krul_snapshot_compress(krul_ctx* ctx, krul_conv* conv,
                           const krul_pair* pairs, int n_pairs,
                           const int64_t* recompute_len, int64_t L, int mode,
                           krul_snapshot** out);
/* Snapshot from host f32 blobs (parity): blob b covers [starts[b], L) with
 * k[b], v[b] laid out [kv_heads][rows][head_dim]. */
int krul_snapshot_from_host(krul_ctx* ctx, const krul_pair* pairs, int n_pairs,
                            const int64_t* recompute_len, int64_t L, int mode,
                            const float* const* k, const float* const* v,
                            krul_snapshot** out);
int krul_snapshot_destroy(krul_snapshot* snap);
int krul_snapshot_n_blobs(krul_snapshot* snap);
int krul_snapshot_blob(krul_snapshot* snap, int b, krul_blob_spec* spec,
                       float* k, float* v);
int krul_snapshot_storage(krul_snapshot* snap, uint64_t* full_bytes,
                          uint64_t* stored_bytes);
int krul_snapshot_plan(krul_snapshot* snap, int64_t* recompute_len,
                       int64_t* L);
int krul_snapshot_set_plan(krul_snapshot* snap, const int64_t* recompute_len);
/* expand (kvstore.cpp:316-343): layer's load span as f32. */
int krul_expand(krul_snapshot* snap, int layer, float* k, float* v,
                int64_t* start, int64_t* end);

/* ---- exponent-coded store (B200 extension of the kvstore snapshot) -------
 * The restore is PCIe-bound; a bf16 KV element's exponent carries ~2.6 bits
 * of entropy. A coded store keeps each element's sign+mantissa byte raw and
 * Huffman-codes its exponent (<= 12-bit canonical codes, 32 interleaved
 * streams per 8192-element chunk); the restore copies the coded image H2D
 * and decodes it on the expand stream. Lossless: the restored KV is
 * bit-identical to the raw store. On by default for bf16 contexts at
 * krul_snapshot_compress (KRUL_KV_CODING=0 or krul_set_kv_coding(ctx, 0)
 * disables it). */
int krul_set_kv_coding(krul_ctx* ctx, int on);
/* Re-encode a raw bf16 snapshot bound to a context (from host / container). */
int krul_snapshot_encode(krul_snapshot* snap);
/* coded: 1 when the store is coded; raw/coded bytes of all blobs (coded ==
 * raw for a raw store). */
int krul_snapshot_coding(krul_snapshot* snap, int* coded, uint64_t* raw_bytes,
                         uint64_t* coded_bytes);
/* Codec checks: the host codec round trip (no device) and the device
 * encoder/decoder on one array; img (NULL = size query) receives the coded
 * image, decoded the decoded elements. */
int krul_ec_host_roundtrip(const uint16_t* x, uint64_t n, void* img, uint64_t cap,
                           uint64_t* img_bytes, uint16_t* decoded);
int krul_debug_ec_device(krul_ctx* ctx, const uint16_t* x, uint64_t n, void* img,
                         uint64_t cap, uint64_t* img_bytes, uint16_t* decoded);

/* ---- KRUL v1 container (kvstore.hpp:88-98; kvstore.cpp:360-511) ---------
 * "KRUL" | u32 version | u64 config_hash | u64 metadata_len | metadata
 * (key-sorted compact JSON, byte-identical to the reference's nlohmann dump)
 * | u32 blob_count | blobs (owners, span, f32 payload keys then values,
 * [heads][rows][head_dim]) | u32 crc32 of all preceding bytes.
 * "n_heads" in the container is the number of KV heads (= heads in the
 * reference's MHA model). The bf16 store widens exactly to f32 on save and
 * rounds to nearest-even on load; an f32 store round-trips bit-exactly. */
/* The container metadata beside the store (kvstore.hpp:46-59). */
typedef struct {
  const char* conversation_id; /* UTF-8, NUL-terminated */
  int exhausted_before_quota;  /* CompressionStrategy::exhausted_before_quota */
  const int32_t* ir_layers;    /* LayerClassReport (analysis.hpp:23-27) */
  int n_ir_layers;
  const int32_t* non_ir_layers;
  int n_non_ir_layers;
  const double* avg_weight_sum;
  int n_avg_weight_sum;
} krul_snapshot_meta;
int krul_snapshot_set_meta(krul_snapshot* snap, const krul_snapshot_meta* meta);
/* Pointers stay valid until the snapshot is destroyed or its meta is reset. */
int krul_snapshot_get_meta(krul_snapshot* snap, krul_snapshot_meta* meta);
/* Header fields of a snapshot (n_heads = KV heads). Any pointer may be NULL. */
int krul_snapshot_header(krul_snapshot* snap, uint64_t* config_hash, int* n_layers,
                         int* n_heads, int* head_dim, int64_t* history_len,
                         int* mode, int* n_pairs);
/* strategy.pairs in selection order (n_pairs from krul_snapshot_header). */
int krul_snapshot_pairs(krul_snapshot* snap, krul_pair* out);
/* kvstore::save (kvstore.cpp:360-392) into buf. *len = container bytes; buf
 * NULL = size query; cap smaller than the container = KRUL_E_ARG. */
int krul_snapshot_save(krul_snapshot* snap, void* buf, uint64_t cap, uint64_t* len);
int krul_snapshot_save_file(krul_snapshot* snap, const char* path);
/* kvstore::load (kvstore.cpp:394-511): the same checks in the same order.
 * ctx non-NULL: the store is pinned host memory in the ctx dtype, ready for
 * krul_restore. ctx NULL: host-only f32 snapshot (inspect / expand / save;
 * krul_restore rejects it). expected_config_hash may be NULL. On
 * KRUL_E_SNAPSHOT_LOAD the failing field ("magic", "checksum", "version",
 * "config", "metadata", "plan", "blob", "coverage") is copied to field. */
int krul_snapshot_load(krul_ctx* ctx, const void* buf, uint64_t len,
                       const uint64_t* expected_config_hash, krul_snapshot** out,
                       char* field, int field_cap);
int krul_snapshot_load_file(krul_ctx* ctx, const char* path,
                            const uint64_t* expected_config_hash,
                            krul_snapshot** out, char* field, int field_cap);
/* crc32 (common.cpp:34-42), all host threads for large buffers. */
uint32_t krul_crc32(const void* data, uint64_t len, uint32_t crc);

/* ---- restoration (scheduler.cpp:320-400) ------------------------------ */
/* Restores conv to full-span KV [0, L): recompute stream rebuilds the
 * per-layer prefixes while the load stream streams blobs H2D and expands
 * them into the paged cache, joined per layer by CUDA events. */
int krul_restore(krul_ctx* ctx, krul_conv* conv, krul_snapshot* snap,
                 const int32_t* history, int64_t L, krul_restore_stats* stats);
/* Restore immediately followed by the new-input prefill; TTFT = restore
 * launch -> last-row logits (harness.cpp:125-131). Device-timed. */
int krul_restore_and_prefill(krul_ctx* ctx, krul_conv* conv,
                             krul_snapshot* snap, const int32_t* history,
                             int64_t L, const int32_t* new_tokens, int64_t n_new,
                             float* logits, krul_restore_stats* stats,
                             double* ttft_ms);
/* Restore + new-input prefill of n conversations pipelined back to back
 * (configs[3]): conversation i+1's blob copies start under conversation i's
 * new-input prefill tail. convs[i] != convs[i-1]. logits: n x V floats (may be
 * NULL); ttft_ms[i] = device time from item i's first copy to its logits;
 * total_ms = first copy to the last logits. No counterpart in the reference
 * (harness.cpp restores one conversation at a time). */
int krul_restore_batch(krul_ctx* ctx, int n, krul_conv* const* convs, krul_snapshot* const* snaps,
                       const int32_t* const* histories, const int64_t* L, const int32_t* const* new_tokens,
                       const int64_t* n_new, float* logits, double* ttft_ms, double* total_ms);

/* Record the per-layer timeline events in the restore DAG (default on). */
int krul_set_timeline(krul_ctx* ctx, int on);
/* Per-layer timeline of the last restore (ms from launch, CUDA events; zeros
 * when krul_set_timeline is off):
 * compute[l] = recompute of layer l done, load[l] = layer l expanded,
 * new_prefill[l] = new-input prefill of layer l done (0 without one). */
int krul_restore_timeline(krul_ctx* ctx, double* compute, double* load,
                          double* new_prefill);

/* calibrate_rc_measured (scheduler.cpp:402-443) with the real device
 * restore: per grid ratio, compress `prev` (full KV of the L-token history)
 * under build_plan(ratio) and time the two-stream restore into `scratch`;
 * returns argmin |T_C - T_L|. tc/tl ([n_grid], optional) get the measured
 * stream times in sorted-grid order. */
int krul_calibrate_rc_measured(krul_ctx* ctx, krul_conv* prev,
                               krul_conv* scratch, const int32_t* history,
                               int64_t L, const krul_pair* pairs, int n_pairs,
                               const double* grid, int n_grid, int mode,
                               double* r_c, double* tc, double* tl);

/* B200 extension of calibrate_rc_measured (scheduler.cpp:402-443): argmin of
 * the measured TTFT of the full restore + new-input prefill DAG over the
 * grid (median of `reps` runs per ratio); ttft ([n_grid], optional) gets
 * the medians in sorted-grid order. */
int krul_calibrate_rc_ttft(krul_ctx* ctx, krul_conv* prev, krul_conv* scratch,
                           const int32_t* history, int64_t L, const int32_t* new_tokens,
                           int64_t n_new, const krul_pair* pairs, int n_pairs,
                           const double* grid, int n_grid, int mode, int reps,
                           double* r_c, double* ttft);

/* ---- measured stream rates (calibrate_rc_measured, scheduler.cpp:402) - */
/* Times pinned H2D bandwidth (bytes/s) and recompute throughput (flop/s)
 * on this device; feeds krul_cost_model. */
int krul_measure_rates(krul_ctx* ctx, krul_conv* scratch, double* h2d_bps,
                       double* flops);

/* ---- diagnostics (tests) ------------------------------------------------ */
/* C[M,N] = A[M,K] B[N,K]^T through the engine GEMM (inputs rounded to the
 * ctx dtype; tcgen05 path for bf16). epi: 0 = f32 store, 2 = resid (C +=),
 * 3 = tanh(acc + bias), 4 = swiglu over column pairs (C is [M, N/2]). */
/* Restore scheduling: 1 (default) = new-input prefill concurrent with the
 * recompute on its own stream; 0 = serialised behind it. */
/* Restore + prefill DAG: 1 folds the pyramid recompute rows into the
 * new-input prefill's layer steps (one weight pass per layer, each step
 * behind its layer's loaded suffix); 0 (default) runs the recompute on its
 * own stream ahead of the loads. Restore without new input always uses the
 * separate recompute stream. */
int krul_set_fused_recompute(krul_ctx* ctx, int on);
int krul_set_concurrency(krul_ctx* ctx, int two_stream);
/* Capture repeated restore DAGs into CUDA graphs (default on); off = every
 * restore is enqueued eagerly, as the first restore of a conversation is. */
int krul_set_graphs(krul_ctx* ctx, int on);
/* Diagnostics: device-side spans (first CTA entry -> last CTA exit,
 * %globaltimer) of the weight-streaming GEMM launches of each restore, with
 * no timing events in the streams; read after a restore. */
int krul_span_enable(krul_ctx* ctx, int on);
int krul_span_read(krul_ctx* ctx, int64_t* launches, double* ms, double* bytes);

/* ---- measurement support (not on the reference's interface) ----------
 * krul_launch_count: number of kernels this library has launched (process
 * wide). krul_ktime_*: per-launch CUDA-event timing of instrumented kernel
 * classes (tag: 0 GEMM, 1 attention, 2 expand, 3 decode fold, 4 prefill
 * fold, 5 selector, 6 compress, 7 weight-streaming GEMM with M <= 128, 8 blob
 * decode, 9 LM-head GEMV, 10 fused decode + expand) with their algorithmic
 * flops / bytes. */
int krul_launch_count(uint64_t* n);
int krul_ktime_enable(krul_ctx* ctx, int on);
int krul_ktime_read(krul_ctx* ctx, int tag, int64_t* launches, double* ms, double* flops,
                    double* bytes);
/* sum over the timed launches of a class of max(flops / peak, bytes / peak) */
int krul_ktime_roofline(krul_ctx* ctx, int tag, double peak_tflops, double peak_gbs,
                        double* ideal_ms);

/* Device time of one decode fold (K1) on the last captured decode rows,
 * `iters` back to back in one captured graph, into scratch segment slots
 * (estimator state untouched). */
int krul_est_fold_bench(krul_est* est, int iters, float* ms_per_fold, double* bytes_per_fold);

/* Kernel-tuning aid: times `iters` tcgen05 attention launches over conv's pages. */
int krul_debug_attn_bench(krul_ctx* ctx, krul_conv* conv, int layer, int64_t rows, int64_t pos0,
                          int dbg, int target, int iters, float* ms_per_iter);
/* Kernel-tuning aid: %globaltimer phase stamps of one attention launch, ts[cta * 8 + slot]. */
// Debug: per-CTA %globaltimer stamps of the K1 decode fold ([cta][8]: entry,
// setup done, chunk loop done, chunks 0-3 in shared memory; [7] = the SM
// id). on = 1 arms, on = 0 copies n_ts stamps into ts and disarms.
int krul_debug_fold_timeline(int on, unsigned long long* ts, int64_t n_ts);
// Debug: refold the rows of the last krul_est_fold_decode_host iters times
// back to back on the device (one captured graph) -> ms per fold (the sums
// keep accumulating).
int krul_debug_fold_repeat(krul_est* est, int iters, float* ms_per_fold);
int krul_debug_attn_timeline(krul_ctx* ctx, krul_conv* conv, int layer, int64_t rows, int64_t pos0, int target,
                             unsigned long long* ts, int64_t n_ts);
/* Kernel-tuning aid: times `iters` device-resident bf16 GEMMs (not a product entry). */
/* Pin the GEMM plan of later calls (tests): force 0 auto, 1/2 1-SM 256/128
 * wide, 3 CTA pair, 5/6 stream-K 256/128 wide; splits 0 = auto. */
int krul_debug_set_gemm_plan(int force, int splits);
int krul_debug_gemm_timeline(krul_ctx* ctx, int64_t M, int64_t N, int64_t K, int epi, int force, int splits,
                             unsigned long long* ts_out);
int krul_debug_gemm_bench(krul_ctx* ctx, int64_t M, int64_t N, int64_t K, int epi, int force,
                          int splits, int iters, float* ms_per_iter);
int krul_debug_gemm(krul_ctx* ctx, int64_t M, int64_t N, int64_t K,
                    const float* A, const float* B, const float* bias, int epi,
                    float* C);

#ifdef __cplusplus
}
#endif
#endif /* KRUL_B200_H_ */
