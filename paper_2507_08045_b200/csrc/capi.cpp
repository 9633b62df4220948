// capi.cpp — the extern "C" boundary (include/krul_b200.h).
//
// Every entry validates on the host first (reference "validate before
// compute"), runs device work through kb::, and maps kb::Error codes to
// krul_status. The estimator and selector live here because they are thin:
// their arithmetic is the K1/K2/K3 kernels in kernels.cu.
#include <functional>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "host.hpp"

using namespace kb;

struct krul_ctx {
  Ctx* c;
};
struct krul_conv {
  Conv* v;
};
struct krul_snapshot {
  Snapshot* s;
};

namespace kb {
Snapshot* snapshot_compress(Ctx& c, Conv& conv, const krul_pair* pairs, int np, const int64_t* p,
                            int64_t L, int mode);
Snapshot* snapshot_from_host(Ctx& c, const krul_pair* pairs, int np, const int64_t* p, int64_t L,
                             int mode, const float* const* k, const float* const* v);
void snapshot_blob_f32(const Snapshot& s, int b, int64_t row0, int64_t rows, float* k, float* v);
void snapshot_expand(const Snapshot& s, int layer, float* k, float* v, int64_t* start,
                     int64_t* end);

// Streaming estimator state (analysis.hpp:66-126): tracked layers, fp64
// per-(pair, head) sums resident on the device.
struct Est {
  Ctx* ctx = nullptr;
  std::vector<int> layers;
  int H = 1;
  DevBuf d_layers, sums, partial, D, tmp, ident;
  DevBuf seg;  // K1 decode fold: resident per-(head, segment, pair) f64 slots [H][seg_S][P]
  int seg_S = 0;
  int64_t partial_cap = 0;
  bool prefill_done = false;
  int64_t prefill_rows = 0, decode_steps = 0;
  int sample_stride = 1;               // decode folds: every stride-th 64-column block (opt-in)
  int64_t host_W = 0, host_pitch = 0;  // rows of the last krul_est_fold_decode_host (in tmp)
  int host_N = 0;
  int P() const { return int(layers.size() * (layers.size() - 1) / 2); }
};
}  // namespace kb

struct krul_est {
  Est* e;
};

namespace {
thread_local std::string g_msg;
thread_local int g_code = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_code = 0;
    return KRUL_OK;
  } catch (const kb::Error& e) {
    g_msg = e.what();
    g_code = e.code;
  } catch (const std::bad_alloc&) {
    g_msg = "host allocation failed";
    g_code = KRUL_E_CUDA;
  } catch (const std::exception& e) {
    g_msg = e.what();
    g_code = KRUL_E_CUDA;
  }
  return g_code;
}
void need(const void* p, const char* what) {
  if (!p) fail(KRUL_E_ARG, std::string("null ") + what);
}
void ensure_partial(Est& e, int64_t chunks) {
  // per chunk and head: the packed upper-triangle Gram (n(n+1)/2 entries)
  const int64_t n = int64_t(e.layers.size());
  const int64_t need_n = (std::max<int64_t>(chunks, 1) + 1) * std::max<int64_t>(n * (n + 1) / 2, 1) * e.H;
  if (need_n > e.partial_cap) {
    e.partial.ensure(size_t(need_n) * 8);
    e.partial_cap = need_n;
  }
}
// the K1 decode fold's resident segment slots -> sums (stream-ordered on s_est)
void collect_segments(Est& e) {
  launch_fold_collect(e.ctx->s_est, e.seg.as<double>(), e.seg_S, int(e.layers.size()), e.H, e.sums.as<double>());
  KB_CUDA(cudaStreamSynchronize(e.ctx->s_est));
}
}  // namespace

extern "C" {

int krul_abi_version(void) { return KRUL_ABI_VERSION; }

int krul_last_error(char* buf, size_t n) {
  if (buf && n) {
    std::strncpy(buf, g_msg.c_str(), n - 1);
    buf[n - 1] = 0;
  }
  return g_code;
}

// ---------------------------------------------------------------- context
int krul_ctx_create(int device, const krul_model_desc* desc, krul_ctx** out) {
  return guard([&] {
    need(desc, "desc");
    need(out, "out");
    *out = new krul_ctx{ctx_create(device, *desc)};
  });
}
int krul_ctx_destroy(krul_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    delete ctx->c;
    delete ctx;
  });
}
int krul_ctx_sync(krul_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    KB_CUDA(cudaSetDevice(ctx->c->device));
    KB_CUDA(cudaDeviceSynchronize());
  });
}
int krul_config_hash(const krul_model_desc* desc, uint64_t* out) {
  return guard([&] {
    need(desc, "desc");
    krul_model_desc d = *desc;
    if (d.max_tokens < 1) d.max_tokens = 1;
    *out = config_hash(cfg_from_desc(d));
  });
}
int krul_weights_upload_f32(krul_ctx* ctx, const float* w, int64_t n) {
  return guard([&] {
    need(ctx, "ctx");
    need(w, "weights");
    weights_upload_f32(*ctx->c, w, n);
  });
}
int krul_weights_init_device(krul_ctx* ctx, uint64_t seed) {
  return guard([&] {
    need(ctx, "ctx");
    weights_init_device(*ctx->c, seed);
  });
}

// ---------------------------------------------------------------- conversations
int krul_conv_create(krul_ctx* ctx, int64_t cap, krul_conv** out) {
  return guard([&] {
    need(ctx, "ctx");
    *out = new krul_conv{conv_create(*ctx->c, cap)};
  });
}
int krul_conv_destroy(krul_conv* conv) {
  return guard([&] {
    if (!conv) return;
    delete conv->v;
    delete conv;
  });
}
int krul_conv_length(krul_conv* conv, int64_t* len) {
  return guard([&] {
    need(conv, "conv");
    *len = conv->v->len;
  });
}
int krul_conv_kv_read(krul_conv* conv, int layer, int64_t start, int64_t end, float* k, float* v) {
  return guard([&] {
    need(conv, "conv");
    Conv& cv = *conv->v;
    Ctx& c = *cv.ctx;
    if (layer < 0 || layer >= c.cfg.N) fail(KRUL_E_CONFIG, "layer out of range");
    if (start < 0 || end > cv.capacity || start > end) fail(KRUL_E_CONFIG, "span out of range");
    const size_t n = size_t(c.cfg.Hkv) * size_t(end - start) * c.cfg.hd;
    if (!n) return;
    KB_CUDA(cudaSetDevice(c.device));
    DevBuf tmp;
    float* d = static_cast<float*>(tmp.ensure(2 * n * 4));
    launch_kv_gather(c, c.s_comp, cv, layer, start, end, d, d + n);
    KB_CUDA(cudaStreamSynchronize(c.s_comp));
    if (k) KB_CUDA(kb_memcpy_sync(k, d, n * 4, cudaMemcpyDeviceToHost));
    if (v) KB_CUDA(kb_memcpy_sync(v, d + n, n * 4, cudaMemcpyDeviceToHost));
  });
}
int krul_conv_kv_write(krul_conv* conv, int layer, int64_t start, int64_t end, const float* k,
                       const float* v) {
  return guard([&] {
    need(conv, "conv");
    need(k, "k");
    need(v, "v");
    Conv& cv = *conv->v;
    Ctx& c = *cv.ctx;
    if (layer < 0 || layer >= c.cfg.N) fail(KRUL_E_CONFIG, "layer out of range");
    if (start < 0 || end > cv.capacity || start > end) fail(KRUL_E_CONFIG, "span out of range");
    const size_t n = size_t(c.cfg.Hkv) * size_t(end - start) * c.cfg.hd;
    if (!n) return;
    KB_CUDA(cudaSetDevice(c.device));
    DevBuf tmp;
    float* d = static_cast<float*>(tmp.ensure(2 * n * 4));
    KB_CUDA(kb_memcpy_sync(d, k, n * 4, cudaMemcpyHostToDevice));
    KB_CUDA(kb_memcpy_sync(d + n, v, n * 4, cudaMemcpyHostToDevice));
    launch_kv_scatter_f32(c, c.s_comp, cv, layer, start, end, d, d + n);
    KB_CUDA(cudaStreamSynchronize(c.s_comp));
    cv.len = std::max(cv.len, end);
  });
}

// ---------------------------------------------------------------- engine
int krul_set_capture(krul_ctx* ctx, int capture_probs) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->capture_probs = capture_probs;
  });
}
int krul_set_classifier_regions(krul_ctx* ctx, double ifrac, double rfrac) {
  return guard([&] {
    need(ctx, "ctx");
    if (!(ifrac > 0.0) || !(rfrac > 0.0) || ifrac + rfrac >= 1.0)
      fail(KRUL_E_CONFIG, "region fractions must be positive and sum below 1");
    ctx->c->cap_ifrac = ifrac;
    ctx->c->cap_rfrac = rfrac;
  });
}
int krul_prefill(krul_ctx* ctx, krul_conv* conv, const int32_t* t, int64_t n, float* logits) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    if (n > 0) need(t, "tokens");
    prefill(*ctx->c, *conv->v, t, n, logits);
  });
}
int krul_prefill_new(krul_ctx* ctx, krul_conv* conv, const int32_t* t, int64_t n, float* logits) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    if (n > 0) need(t, "tokens");
    prefill_new(*ctx->c, *conv->v, t, n, logits);
  });
}
int krul_decode_step(krul_ctx* ctx, krul_conv* conv, int32_t tok, float* logits) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    decode_step(*ctx->c, *conv->v, tok, logits);
  });
}
int krul_partial_recompute(krul_ctx* ctx, krul_conv* conv, const int32_t* t, int64_t n,
                           const int64_t* p, int np) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    need(p, "recompute_len");
    partial_recompute(*ctx->c, *conv->v, t, n, p, np);
  });
}
int krul_capture_prefill(krul_ctx* ctx, int layer, int head, float* out, int64_t* rows,
                         int64_t* width) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    if (!c.cap_valid || c.cap_mode != 1) fail(KRUL_E_STATE_CORRUPTION, "no captured prefill attention");
    if (layer < 0 || layer >= c.cfg.N || head < 0 || head >= c.cfg.H) fail(KRUL_E_CONFIG, "index out of range");
    if (rows) *rows = c.cap_rows;
    if (width) *width = c.cap_width;
    if (out) {
      const size_t n = size_t(c.cap_rows * c.cap_width);
      const float* src = c.cap_probs.as<float>() + (size_t(layer) * c.cfg.H + head) * n;
      KB_CUDA(kb_memcpy_sync(out, src, n * 4, cudaMemcpyDeviceToHost));
    }
  });
}
int krul_capture_decode(krul_ctx* ctx, float* out, int64_t* width) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    if (!c.dec_valid) fail(KRUL_E_STATE_CORRUPTION, "no captured decode step");
    if (width) *width = c.dec_width;
    if (out) {
      KB_CUDA(cudaDeviceSynchronize());
      KB_CUDA(cudaMemcpy2D(out, size_t(c.dec_width) * 4, c.dec_rows.p, size_t(c.dec_pitch) * 4,
                           size_t(c.dec_width) * 4, size_t(c.cfg.N) * c.cfg.H, cudaMemcpyDeviceToHost));
      KB_CUDA(cudaDeviceSynchronize());
    }
  });
}

// ---------------------------------------------------------------- analysis
// analysis.cpp:20-63 over the masses the attention kernel reduced.
int krul_classify(krul_ctx* ctx, double gamma, double ifrac, double rfrac, double* avg,
                  int* is_ir) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    if (!(gamma > 0.0) || gamma > 1.0) fail(KRUL_E_CONFIG, "gamma must lie in (0, 1]");
    if (!(ifrac > 0.0) || !(rfrac > 0.0) || ifrac + rfrac >= 1.0)
      fail(KRUL_E_CONFIG, "region fractions must be positive and sum below 1");
    if (!c.cap_valid || c.cap_rows == 0) fail(KRUL_E_CLASSIFICATION, "classification requires prefill attention");
    const int64_t W = c.cap_width;
    const int64_t il = int64_t(ifrac * double(W)), rl = int64_t(rfrac * double(W));
    if (il < 1 || rl < 1) fail(KRUL_E_CLASSIFICATION, "sequence too short to form both attention regions");
    if (ifrac != c.cap_ifrac || rfrac != c.cap_rfrac)
      fail(KRUL_E_CONFIG, "classifier regions differ from those set before the prefill");
    const int N = c.cfg.N, H = c.cfg.H;
    const int64_t R = c.cap_rows;
    std::vector<double> m(size_t(N) * H * R);
    KB_CUDA(kb_memcpy_sync(m.data(), c.cap_mass.p, m.size() * 8, cudaMemcpyDeviceToHost));
    for (int l = 0; l < N; ++l) {
      double mass = 0.0;
      for (int h = 0; h < H; ++h) {
        double hm = 0.0;
        for (int64_t r = 0; r < R; ++r) hm += m[(size_t(l) * H + h) * R + r];
        mass += hm;
      }
      const double a = mass / (double(H) * double(R));
      if (avg) avg[l] = a;
      if (is_ir) is_ir[l] = a >= gamma ? 1 : 0;
    }
  });
}

int krul_est_create(krul_ctx* ctx, const int* ir, int n, krul_est** out) {
  return guard([&] {
    need(ctx, "ctx");
    auto* e = new Est;
    e->ctx = ctx->c;
    e->H = ctx->c->cfg.H;
    e->layers.assign(ir, ir + n);
    std::sort(e->layers.begin(), e->layers.end());
    e->layers.erase(std::unique(e->layers.begin(), e->layers.end()), e->layers.end());
    if (!e->layers.empty() && e->layers.front() < 0) {
      delete e;
      fail(KRUL_E_CONFIG, "layer indices must be non-negative");
    }
    KB_CUDA(cudaSetDevice(ctx->c->device));
    const size_t nl = std::max<size_t>(e->layers.size(), 1);
    e->d_layers.ensure(nl * 4);
    if (!e->layers.empty())
      KB_CUDA(kb_memcpy_sync(e->d_layers.p, e->layers.data(), e->layers.size() * 4, cudaMemcpyHostToDevice));
    const size_t ns = size_t(std::max(e->P(), 1)) * e->H;
    e->sums.ensure(ns * 8);
    KB_CUDA(kb_memset_sync(e->sums.p, 0, ns * 8));
    e->seg_S = fold_seg_slots(e->H, ctx->c->sm_count > 0 ? ctx->c->sm_count : 148);
    const size_t nseg = size_t(e->seg_S) * ns;
    e->seg.ensure(nseg * 8);
    KB_CUDA(kb_memset_sync(e->seg.p, 0, nseg * 8));
    *out = new krul_est{e};
  });
}
int krul_est_destroy(krul_est* est) {
  return guard([&] {
    if (!est) return;
    delete est->e;
    delete est;
  });
}
static void fold_prefill_dev(Est& e, const float* probs, int64_t rows, int64_t W, int N) {
  if (e.prefill_done) fail(KRUL_E_ACCOUNTING, "prefill attention folded twice");
  if (!e.layers.empty() && e.layers.back() >= N) fail(KRUL_E_CONFIG, "record does not cover all tracked layers");
  Ctx& c = *e.ctx;
  ensure_partial(e, (rows * W + kFoldChunk - 1) / kFoldChunk);
  cudaEvent_t kt0 = kt_begin(c, c.s_est);
  launch_fold_prefill(c.s_est, probs, rows, W, e.H, e.d_layers.as<int>(), int(e.layers.size()),
                      e.sums.as<double>(), e.partial.as<double>(), e.partial_cap);
  kt_end(c, c.s_est, kt0, KT_FOLD_PREFILL, 0.0,
         double(e.layers.size()) * e.H * double(rows) * double(W) * 4.0 + double(e.P()) * e.H * 16.0);
  KB_CUDA(cudaStreamSynchronize(c.s_est));
  e.prefill_done = true;
  e.prefill_rows = rows;
}
// rows: [N][H][pitch] f32, pitch % 4 == 0 (the decode step's capture layout)
static void fold_decode_dev(Est& e, const float* rows, int64_t W, int64_t pitch, int N) {
  if (!e.layers.empty() && e.layers.back() >= N)
    fail(KRUL_E_STATE_CORRUPTION, "decode rows do not cover all tracked layers");
  Ctx& c = *e.ctx;
  const int n = int(e.layers.size());
  const int sms = c.sm_count > 0 ? c.sm_count : 148;
  cudaEvent_t kt0 = kt_begin(c, c.s_est);
  // the sampled token subset rotates its phase per step, so every block is
  // folded once per `stride` steps
  const int stride = e.sample_stride, phase = int(e.decode_steps % stride);
  launch_fold_direct(c.s_est, rows, int64_t(e.H) * pitch, pitch, W, e.H, e.d_layers.as<int>(), n,
                     e.seg.as<double>(), e.seg_S, sms, stride, phase);
  // algorithmic bytes: tracked rows read once + f64 accumulator RMW
  kt_end(c, c.s_est, kt0, KT_FOLD_DECODE, 0.0,
         double(e.layers.size()) * e.H * double(W) * 4.0 + double(e.P()) * e.H * 16.0);
  KB_CUDA(cudaStreamSynchronize(c.s_est));
  ++e.decode_steps;
}
// K2: the prefill fold without the probability record. The tracked layers'
// probabilities are recomputed one key-column chunk at a time (bounded
// scratch, independent of W) from the Q rows, the paged K and the softmax
// statistics the prefill saved, and each chunk [n][H][rows x wc] is folded
// by the decode-fold kernel (the sum over the full rows x width rectangle is
// a sum over its column chunks, analysis.cpp:97-122).
static void fold_prefill_recompute(Est& e, Ctx& c) {
  if (e.prefill_done) fail(KRUL_E_ACCOUNTING, "prefill attention folded twice");
  const int N = c.cfg.N, H = e.H, n = int(e.layers.size());
  if (!e.layers.empty() && e.layers.back() >= N) fail(KRUL_E_CONFIG, "record does not cover all tracked layers");
  const Conv* conv = c.cap_conv;
  if (!conv || std::find(c.convs.begin(), c.convs.end(), conv) == c.convs.end() ||
      conv->serial != c.cap_conv_serial)
    fail(KRUL_E_STATE_CORRUPTION, "the captured prefill's conversation is gone");
  const int64_t rows = c.cap_rows, W = c.cap_width, first_q = c.cap_first_q;
  if (n >= 2 && rows > 0) {
    const int sms = c.sm_count > 0 ? c.sm_count : 148;
    const double per_col = double(n) * H * double(rows) * 4.0;
    const int64_t wc = std::max<int64_t>(64, std::min<int64_t>((W + 63) / 64 * 64,
                                                              int64_t((256.0 * 1024 * 1024) / per_col) / 64 * 64));
    float* P = static_cast<float*>(e.tmp.ensure(size_t(n) * H * size_t(rows) * size_t(wc) * 4));
    std::vector<int> ident(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) ident[size_t(i)] = i;
    int* d_ident = static_cast<int*>(e.ident.ensure(size_t(n) * 4));
    KB_CUDA(kb_memcpy_sync(d_ident, ident.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
    cudaEvent_t kt0 = kt_begin(c, c.s_est);
    for (int64_t c0 = 0; c0 < W; c0 += wc) {
      launch_prefill_probs(c, c.s_est, *conv, e.d_layers.as<int>(), n, rows, first_q, c0, int(wc), P);
      launch_fold_direct(c.s_est, P, int64_t(H) * rows * wc, rows * wc, rows * wc, H, d_ident, n,
                         e.seg.as<double>(), e.seg_S, sms);
    }
    kt_end(c, c.s_est, kt0, KT_FOLD_PREFILL, 0.0, double(n) * H * double(rows) * double(W) * 4.0);
    KB_CUDA(cudaStreamSynchronize(c.s_est));
  }
  e.prefill_done = true;
  e.prefill_rows = rows;
}
int krul_est_fold_prefill(krul_est* est) {
  return guard([&] {
    need(est, "est");
    Est& e = *est->e;
    Ctx& c = *e.ctx;
    if (!c.cap_valid || !c.cap_mode) fail(KRUL_E_STATE_CORRUPTION, "no captured prefill attention (krul_set_capture)");
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaStreamSynchronize(c.s_comp));
    KB_CUDA(cudaStreamSynchronize(c.s_new));
    if (c.cap_mode == 2)
      fold_prefill_recompute(e, c);
    else
      fold_prefill_dev(e, c.cap_probs.as<float>(), c.cap_rows, c.cap_width, c.cfg.N);
  });
}
int krul_est_fold_decode(krul_est* est) {
  return guard([&] {
    need(est, "est");
    Est& e = *est->e;
    Ctx& c = *e.ctx;
    if (!c.dec_valid) fail(KRUL_E_STATE_CORRUPTION, "no captured decode step");
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaStreamSynchronize(c.s_comp));
    fold_decode_dev(e, c.dec_rows.as<float>(), c.dec_width, c.dec_pitch, c.cfg.N);
  });
}
int krul_est_fold_prefill_host(krul_est* est, const float* probs, int N, int64_t rows, int64_t W) {
  return guard([&] {
    need(est, "est");
    need(probs, "probs");
    Est& e = *est->e;
    if (e.prefill_done) fail(KRUL_E_ACCOUNTING, "prefill attention folded twice");
    KB_CUDA(cudaSetDevice(e.ctx->device));
    const size_t n = size_t(N) * e.H * size_t(rows) * size_t(W);
    float* d = static_cast<float*>(e.tmp.ensure(std::max<size_t>(n, 1) * 4));
    KB_CUDA(kb_memcpy_sync(d, probs, n * 4, cudaMemcpyHostToDevice));
    fold_prefill_dev(e, d, rows, W, N);
  });
}
int krul_est_fold_decode_host(krul_est* est, const float* rows, int N, int64_t W) {
  return guard([&] {
    need(est, "est");
    need(rows, "rows");
    Est& e = *est->e;
    KB_CUDA(cudaSetDevice(e.ctx->device));
    static const int64_t pad = [] {  // diagnostics: extra row pitch (floats, multiple of 4)
      const char* v = std::getenv("KRUL_FOLD_ROW_PAD");
      return v ? int64_t(std::atoi(v)) / 4 * 4 : int64_t(0);
    }();
    const int64_t pitch = (W + 3) / 4 * 4 + pad;
    const size_t n = size_t(N) * e.H * size_t(pitch);
    float* d = static_cast<float*>(e.tmp.ensure(std::max<size_t>(n, 1) * 4));
    KB_CUDA(cudaDeviceSynchronize());
    if (W > 0)
      KB_CUDA(cudaMemcpy2D(d, size_t(pitch) * 4, rows, size_t(W) * 4, size_t(W) * 4, size_t(N) * e.H,
                           cudaMemcpyHostToDevice));
    // a pageable H2D copy may return before its DMA lands; the fold runs on a
    // non-blocking stream that does not order against the legacy stream
    KB_CUDA(cudaDeviceSynchronize());
    fold_decode_dev(e, d, W, pitch, N);
    e.host_W = W;
    e.host_pitch = pitch;
    e.host_N = N;
  });
}
// Debug: refold the rows of the last krul_est_fold_decode_host iters times
// back to back (device-resident, CUDA events) -> ms per fold. The sums keep
// accumulating: diagnostics only.
int krul_debug_fold_repeat(krul_est* est, int iters, float* ms_per_fold) {
  return guard([&] {
    need(est, "est");
    need(ms_per_fold, "ms_per_fold");
    Est& e = *est->e;
    Ctx& c = *e.ctx;
    if (e.host_W <= 0) fail(KRUL_E_STATE_CORRUPTION, "no host rows folded yet");
    KB_CUDA(cudaSetDevice(c.device));
    const int n = int(e.layers.size());
    const int sms = c.sm_count > 0 ? c.sm_count : 148;
    const float* rows = e.tmp.as<float>();
    iters = std::max(iters, 1);
    // the folds captured as one graph: launch-gap free, like the restore DAG
    launch_fold_direct(c.s_est, rows, int64_t(e.H) * e.host_pitch, e.host_pitch, e.host_W, e.H,
                       e.d_layers.as<int>(), n, e.seg.as<double>(), e.seg_S, sms);  // warm (attributes)
    KB_CUDA(cudaStreamSynchronize(c.s_est));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    KB_CUDA(cudaStreamBeginCapture(c.s_est, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i)
      launch_fold_direct(c.s_est, rows, int64_t(e.H) * e.host_pitch, e.host_pitch, e.host_W, e.H,
                         e.d_layers.as<int>(), n, e.seg.as<double>(), e.seg_S, sms);
    KB_CUDA(cudaStreamEndCapture(c.s_est, &g));
    KB_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    KB_CUDA(cudaEventCreate(&a));
    KB_CUDA(cudaEventCreate(&b));
    KB_CUDA(cudaGraphLaunch(ge, c.s_est));
    KB_CUDA(cudaEventRecord(a, c.s_est));
    KB_CUDA(cudaGraphLaunch(ge, c.s_est));
    KB_CUDA(cudaEventRecord(b, c.s_est));
    KB_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    KB_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    *ms_per_fold = ms / float(std::max(iters, 1));
  });
}
int krul_est_set_sampling(krul_est* est, int stride) {
  return guard([&] {
    need(est, "est");
    if (stride < 1) fail(KRUL_E_CONFIG, "sampling stride must be >= 1");
    est->e->sample_stride = stride;
  });
}
int krul_est_sums(krul_est* est, double* sums) {
  return guard([&] {
    need(est, "est");
    Est& e = *est->e;
    KB_CUDA(cudaSetDevice(e.ctx->device));
    collect_segments(e);
    if (e.P() > 0) KB_CUDA(kb_memcpy_sync(sums, e.sums.p, size_t(e.P()) * e.H * 8, cudaMemcpyDeviceToHost));
  });
}
int krul_est_finalize(krul_est* est, double* D) {
  return guard([&] {
    need(est, "est");
    Est& e = *est->e;
    if (!e.prefill_done) fail(KRUL_E_ACCOUNTING, "finalize requires the prefill part to be folded");
    const int n = int(e.layers.size());
    if (n == 0) return;
    KB_CUDA(cudaSetDevice(e.ctx->device));
    double* dD = static_cast<double*>(e.D.ensure(size_t(n) * n * 8));
    collect_segments(e);
    launch_finalize(e.ctx->s_est, e.sums.as<double>(), n, e.H, dD);
    KB_CUDA(cudaStreamSynchronize(e.ctx->s_est));
    KB_CUDA(kb_memcpy_sync(D, dD, size_t(n) * n * 8, cudaMemcpyDeviceToHost));
  });
}
int krul_est_counts(krul_est* est, int64_t* pr, int64_t* ds) {
  return guard([&] {
    need(est, "est");
    if (pr) *pr = est->e->prefill_done ? est->e->prefill_rows : 0;
    if (ds) *ds = est->e->decode_steps;
  });
}

// ---------------------------------------------------------------- selector
int krul_quota(int n_layers, double r_l, int* out) {
  return guard([&] { *out = quota(n_layers, r_l); });
}
// strategy.cpp:27-74: host assembles the (d, i, j) candidates, K3 sorts and
// greedily matches them on the device.
int krul_select(krul_ctx* ctx, const double* D, const int* dm_layers, int n, const int* ir,
                int n_ir, double r_l, int n_layers, krul_pair* out, int* n_out, int* exhausted) {
  return guard([&] {
    need(ctx, "ctx");
    if (r_l < 0.0 || r_l > 1.0) fail(KRUL_E_CONFIG, "r_l must lie in [0, 1]");
    const int q = quota(n_layers, r_l);
    *n_out = 0;
    *exhausted = 0;
    if (q == 0) return;
    std::vector<int> layers(ir, ir + n_ir);
    std::sort(layers.begin(), layers.end());
    layers.erase(std::unique(layers.begin(), layers.end()), layers.end());
    if (layers.size() < 2) {
      *exhausted = 1;
      return;
    }
    if (layers.back() >= 256 || layers.front() < 0) fail(KRUL_E_CONFIG, "layer index outside [0, 256)");
    auto pos = [&](int layer) {
      const int* it = std::lower_bound(dm_layers, dm_layers + n, layer);
      if (it == dm_layers + n || *it != layer) fail(KRUL_E_CONFIG, "layer not tracked by the distance matrix");
      return int(it - dm_layers);
    };
    std::vector<double> cd;
    std::vector<int> ci, cj;
    for (size_t a = 0; a < layers.size(); ++a)
      for (size_t b = a + 1; b < layers.size(); ++b) {
        cd.push_back(D[size_t(pos(layers[a])) * n + pos(layers[b])]);
        ci.push_back(layers[a]);
        cj.push_back(layers[b]);
      }
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    const int nc = int(cd.size());
    // one block each way: [d nc f64][i nc][j nc] in, [d nc f64][i nc][j nc][n] out,
    // staged through ctx-owned pinned / device buffers (grown once)
    const size_t in_b = size_t(nc) * 16, out_b = size_t(nc) * 16 + 16;
    char* h = static_cast<char*>(c.sel_host.ensure(in_b + out_b));
    char* p = static_cast<char*>(c.sel_dev.ensure(in_b + out_b));
    std::memcpy(h, cd.data(), size_t(nc) * 8);
    std::memcpy(h + size_t(nc) * 8, ci.data(), size_t(nc) * 4);
    std::memcpy(h + size_t(nc) * 12, cj.data(), size_t(nc) * 4);
    double* d_cd = reinterpret_cast<double*>(p);
    int* d_ci = reinterpret_cast<int*>(d_cd + nc);
    int* d_cj = d_ci + nc;
    double* d_od = reinterpret_cast<double*>(p + in_b);
    int* d_oi = reinterpret_cast<int*>(d_od + nc);
    int* d_oj = d_oi + nc;
    int* d_on = d_oj + nc;
    KB_CUDA(cudaMemcpyAsync(p, h, in_b, cudaMemcpyHostToDevice, c.s_est));
    launch_select(c.s_est, d_cd, d_ci, d_cj, nc, q, d_oi, d_oj, d_od, d_on);
    KB_CUDA(cudaMemcpyAsync(h + in_b, p + in_b, out_b, cudaMemcpyDeviceToHost, c.s_est));
    KB_CUDA(cudaStreamSynchronize(c.s_est));
    const char* o = h + in_b;
    int np = 0;
    std::memcpy(&np, o + size_t(nc) * 16, 4);
    if (np < 0 || np > nc) fail(KRUL_E_CUDA, "selector returned a bad pair count");
    std::vector<double> od(size_t(std::max(np, 1)));
    std::vector<int> oi(od.size()), oj(od.size());
    if (np) {
      std::memcpy(od.data(), o, size_t(np) * 8);
      std::memcpy(oi.data(), o + size_t(nc) * 8, size_t(np) * 4);
      std::memcpy(oj.data(), o + size_t(nc) * 12, size_t(np) * 4);
    }
    for (int k = 0; k < np; ++k) out[k] = krul_pair{oi[size_t(k)], oj[size_t(k)], od[size_t(k)]};
    *n_out = np;
    *exhausted = 2 * np < q ? 1 : 0;
  });
}

// ---------------------------------------------------------------- scheduler
int krul_build_plan(int64_t L, int N, double r_c, const krul_pair* pairs, int np, int64_t* out) {
  return guard([&] {
    auto p = build_plan(L, N, r_c, pairs, np);
    std::copy(p.begin(), p.end(), out);
  });
}
int krul_uniform_plan(int64_t L, int N, double r_c, int64_t* out) {
  return guard([&] {
    auto p = uniform_plan(L, N, r_c);
    std::copy(p.begin(), p.end(), out);
  });
}
int krul_default_rc_grid(double step, double* out, int* n) {
  return guard([&] {
    auto g = default_grid(step);
    *n = int(g.size());
    if (out) std::copy(g.begin(), g.end(), out);
  });
}
int krul_calibrate_rc(const krul_cost_model* cost, int N, int64_t L, int64_t d,
                      const krul_pair* pairs, int np, const double* grid, int ng, double* out) {
  return guard([&] { *out = calibrate(cost_from(cost), N, L, d, pairs, np, grid, ng); });
}
int krul_validate_plan(int64_t L, const int64_t* p, int N, const krul_pair* pairs, int np, int* mask) {
  return guard([&] { *mask = validate_plan(L, std::vector<int64_t>(p, p + N), pairs, np); });
}
int krul_validate_strategy(const krul_pair* pairs, int n_pairs, const int* shared, int n_shared,
                           int exhausted, const int* ir_layers, int n_ir, int n_layers, double r_l,
                           int* mask, char* details, size_t details_cap) {
  return guard([&] {
    need(mask, "mask");
    if (n_pairs > 0) need(pairs, "pairs");
    if (n_shared > 0) need(shared, "shared");
    if (n_ir > 0) need(ir_layers, "ir_layers");
    std::string lines;
    *mask = validate_strategy(pairs, n_pairs, std::set<int>(shared, shared + std::max(n_shared, 0)),
                              exhausted != 0, std::set<int>(ir_layers, ir_layers + std::max(n_ir, 0)),
                              n_layers, r_l, &lines);
    if (details && details_cap) {
      std::strncpy(details, lines.c_str(), details_cap - 1);
      details[details_cap - 1] = 0;
    }
  });
}
int krul_blob_specs(int64_t L, const int64_t* p, int N, const krul_pair* pairs, int np,
                    krul_blob_spec* out, int* n_out) {
  return guard([&] {
    auto s = blob_specs(std::vector<int64_t>(p, p + N), L, pairs, np);
    *n_out = int(s.size());
    if (out) std::copy(s.begin(), s.end(), out);
  });
}
// scheduler.cpp:282-318
int krul_simulate(int64_t L, const int64_t* p, int N, const krul_pair* pairs, int np,
                  const krul_cost_model* cost, int64_t d, double* out) {
  return guard([&] {
    const Cost c = cost_from(cost);
    std::vector<int64_t> pv(p, p + N);
    double tc = 0.0, tl = 0.0;
    for (int l = 0; l < N; ++l) tc += c.layer_flops(pv[size_t(l)], d) / c.f;
    for (const auto& s : blob_specs(pv, L, pairs, np)) tl += c.blob_bytes(s.end - s.start, d) / c.b;
    const double mk = std::max(tc, tl);
    out[0] = mk;
    out[1] = tc;
    out[2] = tl;
    out[3] = mk > 0 && tc > 0 ? (mk - tc) / mk : 0.0;
    out[4] = mk > 0 && tl > 0 ? (mk - tl) / mk : 0.0;
  });
}

// ---------------------------------------------------------------- kvstore
int krul_snapshot_compress(krul_ctx* ctx, krul_conv* conv, const krul_pair* pairs, int np,
                           const int64_t* p, int64_t L, int mode, krul_snapshot** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    need(p, "recompute_len");
    Ctx& c = *ctx->c;
    std::vector<int64_t> pv(p, p + c.cfg.N);
    (void)blob_specs(pv, L, pairs, np);  // SnapshotError on malformed strategy
    *out = new krul_snapshot{snapshot_compress(c, *conv->v, pairs, np, p, L, mode)};
  });
}
int krul_snapshot_from_host(krul_ctx* ctx, const krul_pair* pairs, int np, const int64_t* p,
                            int64_t L, int mode, const float* const* k, const float* const* v,
                            krul_snapshot** out) {
  return guard([&] {
    need(ctx, "ctx");
    *out = new krul_snapshot{snapshot_from_host(*ctx->c, pairs, np, p, L, mode, k, v)};
  });
}
int krul_snapshot_destroy(krul_snapshot* s) {
  return guard([&] {
    if (!s) return;
    delete s->s;
    delete s;
  });
}
int krul_snapshot_n_blobs(krul_snapshot* s) { return s ? int(s->s->blobs.size()) : 0; }
int krul_snapshot_blob(krul_snapshot* s, int b, krul_blob_spec* spec, float* k, float* v) {
  return guard([&] {
    need(s, "snapshot");
    const Snapshot& sn = *s->s;
    if (b < 0 || b >= int(sn.blobs.size())) fail(KRUL_E_CONFIG, "blob index out of range");
    const auto& bl = sn.blobs[size_t(b)];
    if (spec) *spec = krul_blob_spec{{bl.owners[0], bl.owners[1]}, bl.start, bl.end};
    if (k || v) snapshot_blob_f32(sn, b, 0, bl.end - bl.start, k, v);
  });
}
// kvstore.cpp:345-358 (the reference accounts f32 rows; bf16 halves it).
int krul_snapshot_storage(krul_snapshot* s, uint64_t* full, uint64_t* stored) {
  return guard([&] {
    need(s, "snapshot");
    const Snapshot& sn = *s->s;
    const uint64_t row = 2ull * uint64_t(sn.Hkv) * uint64_t(sn.hd) * uint64_t(sn.esz);
    *full = uint64_t(sn.N) * uint64_t(sn.L) * row;
    *stored = 0;
    for (const auto& b : sn.blobs) *stored += uint64_t(b.end - b.start) * row;
  });
}
int krul_snapshot_plan(krul_snapshot* s, int64_t* p, int64_t* L) {
  return guard([&] {
    need(s, "snapshot");
    if (p) std::copy(s->s->p.begin(), s->s->p.end(), p);
    if (L) *L = s->s->L;
  });
}
int krul_snapshot_set_plan(krul_snapshot* s, const int64_t* p) {
  return guard([&] {
    need(s, "snapshot");
    std::copy(p, p + s->s->N, s->s->p.begin());
    s->s->serial = next_serial();
  });
}
// ------------------------------------------ exponent-coded store (kvcode)
int krul_set_kv_coding(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->kv_coding = on != 0;
  });
}
int krul_snapshot_encode(krul_snapshot* s) {
  return guard([&] {
    need(s, "snapshot");
    Snapshot& sn = *s->s;
    if (sn.coded) return;
    if (!sn.ctx || sn.host.pageable) fail(KRUL_E_SNAPSHOT, "encoding needs a snapshot bound to a context");
    if (sn.esz != 2) fail(KRUL_E_CONFIG, "exponent coding needs a bf16 store");
    Ctx& c = *sn.ctx;
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.s_load;
    char* stg = static_cast<char*>(c.staging.ensure(std::max<size_t>(sn.total, 256)));
    if (sn.total) KB_CUDA(cudaMemcpyAsync(stg, sn.host.p, sn.total, cudaMemcpyHostToDevice, st));
    snapshot_encode(c, sn, stg, st);
  });
}
int krul_snapshot_coding(krul_snapshot* s, int* coded, uint64_t* raw_bytes, uint64_t* coded_bytes) {
  return guard([&] {
    need(s, "snapshot");
    const Snapshot& sn = *s->s;
    uint64_t raw = 0, cod = 0;
    for (const auto& b : sn.blobs) {
      raw += b.bytes;
      cod += sn.coded ? b.cbytes : b.bytes;
    }
    if (coded) *coded = sn.coded ? 1 : 0;
    if (raw_bytes) *raw_bytes = raw;
    if (coded_bytes) *coded_bytes = cod;
  });
}
// Host codec round trip (no device): histogram -> code -> ec_encode_host ->
// ec_decode_host. img may be NULL (size query via *img_bytes).
int krul_ec_host_roundtrip(const uint16_t* x, uint64_t n, void* img, uint64_t cap, uint64_t* img_bytes,
                           uint16_t* decoded) {
  return guard([&] {
    need(img_bytes, "img_bytes");
    if (n && !x) fail(KRUL_E_ARG, "null input");
    uint64_t hist[256] = {0};
    for (uint64_t i = 0; i < n; ++i) ++hist[(x[i] >> 7) & 0xFF];
    const auto code = std::make_unique<EcCode>(ec_build_code(hist));
    const std::vector<uint8_t> enc = ec_encode_host(x, n, *code);
    *img_bytes = enc.size();
    if (img) {
      if (cap < enc.size()) fail(KRUL_E_ARG, "buffer smaller than the coded image");
      std::memcpy(img, enc.data(), enc.size());
    }
    if (decoded && n) ec_decode_host(enc.data(), code->lut, decoded);
  });
}
// The device encoder + decoder on one host array (GPU parity of the codec).
int krul_debug_ec_device(krul_ctx* ctx, const uint16_t* x, uint64_t n, void* img, uint64_t cap,
                         uint64_t* img_bytes, uint16_t* decoded) {
  return guard([&] {
    need(ctx, "ctx");
    need(img_bytes, "img_bytes");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.s_load;
    Snapshot sn;
    sn.ctx = &c;
    sn.esz = 2;
    sn.blobs.push_back(Snapshot::Blob{{0, -1}, 0, 0, 0, size_t(n) * 2});
    sn.total = size_t(n) * 2;
    DevBuf raw, out, cimg;
    char* d = static_cast<char*>(raw.ensure(std::max<size_t>(sn.total, 256)));
    if (n) KB_CUDA(cudaMemcpyAsync(d, x, sn.total, cudaMemcpyHostToDevice, st));
    snapshot_encode(c, sn, d, st);
    const auto& b = sn.blobs[0];
    *img_bytes = b.cbytes;
    if (img) {
      if (cap < b.cbytes) fail(KRUL_E_ARG, "buffer smaller than the coded image");
      std::memcpy(img, static_cast<char*>(sn.host.p) + b.coff, b.cbytes);
    }
    if (decoded && n) {
      char* ci = static_cast<char*>(cimg.ensure(std::max<size_t>(b.cbytes, 256)));
      KB_CUDA(cudaMemcpyAsync(ci, static_cast<char*>(sn.host.p) + b.coff, b.cbytes, cudaMemcpyHostToDevice, st));
      void* o = out.ensure(sn.total);
      launch_ec_decode(st, ci, int64_t(b.ec_chunks), sn.lut_dev.as<uint16_t>(), o);
      KB_CUDA(cudaMemcpyAsync(decoded, o, sn.total, cudaMemcpyDeviceToHost, st));
    }
    KB_CUDA(cudaStreamSynchronize(st));
  });
}
// ------------------------------------------------ KRUL v1 container (f3)
int krul_snapshot_set_meta(krul_snapshot* s, const krul_snapshot_meta* m) {
  return guard([&] {
    need(s, "snapshot");
    need(m, "meta");
    SnapMeta& t = s->s->meta;
    t.conversation_id = m->conversation_id ? m->conversation_id : "";
    t.exhausted_before_quota = m->exhausted_before_quota != 0;
    if ((m->n_ir_layers > 0 && !m->ir_layers) || (m->n_non_ir_layers > 0 && !m->non_ir_layers) ||
        (m->n_avg_weight_sum > 0 && !m->avg_weight_sum))
      fail(KRUL_E_ARG, "null meta array with a positive length");
    t.ir_layers.assign(m->ir_layers, m->ir_layers + std::max(m->n_ir_layers, 0));
    t.non_ir_layers.assign(m->non_ir_layers, m->non_ir_layers + std::max(m->n_non_ir_layers, 0));
    t.avg_weight_sum.assign(m->avg_weight_sum, m->avg_weight_sum + std::max(m->n_avg_weight_sum, 0));
  });
}
int krul_snapshot_get_meta(krul_snapshot* s, krul_snapshot_meta* m) {
  return guard([&] {
    need(s, "snapshot");
    need(m, "meta");
    const SnapMeta& t = s->s->meta;
    m->conversation_id = t.conversation_id.c_str();
    m->exhausted_before_quota = t.exhausted_before_quota ? 1 : 0;
    m->ir_layers = t.ir_layers.data();
    m->n_ir_layers = int(t.ir_layers.size());
    m->non_ir_layers = t.non_ir_layers.data();
    m->n_non_ir_layers = int(t.non_ir_layers.size());
    m->avg_weight_sum = t.avg_weight_sum.data();
    m->n_avg_weight_sum = int(t.avg_weight_sum.size());
  });
}
int krul_snapshot_header(krul_snapshot* s, uint64_t* config_hash, int* n_layers, int* n_heads,
                         int* head_dim, int64_t* history_len, int* mode, int* n_pairs) {
  return guard([&] {
    need(s, "snapshot");
    const Snapshot& sn = *s->s;
    if (config_hash) *config_hash = sn.config_hash;
    if (n_layers) *n_layers = sn.N;
    if (n_heads) *n_heads = sn.Hkv;
    if (head_dim) *head_dim = sn.hd;
    if (history_len) *history_len = sn.L;
    if (mode) *mode = sn.mode;
    if (n_pairs) *n_pairs = int(sn.pairs.size());
  });
}
int krul_snapshot_pairs(krul_snapshot* s, krul_pair* out) {
  return guard([&] {
    need(s, "snapshot");
    need(out, "out");
    std::copy(s->s->pairs.begin(), s->s->pairs.end(), out);
  });
}
int krul_snapshot_save(krul_snapshot* s, void* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    need(s, "snapshot");
    need(len, "len");
    const uint64_t n = container_size(*s->s);
    *len = n;
    if (!buf) return;
    if (cap < n) fail(KRUL_E_ARG, "buffer smaller than the container");
    container_write(*s->s, static_cast<char*>(buf));
  });
}
int krul_snapshot_save_file(krul_snapshot* s, const char* path) {
  return guard([&] {
    need(s, "snapshot");
    need(path, "path");
    container_write_file(*s->s, path);
  });
}
static int load_common(krul_ctx* ctx, char* field, int field_cap, const std::function<Snapshot*(Ctx*)>& f,
                       krul_snapshot** out) {
  std::string fld;
  if (field && field_cap > 0) field[0] = 0;
  const int rc = guard([&] {
    need(out, "out");
    *out = nullptr;
    Ctx* c = ctx ? ctx->c : nullptr;
    if (c) KB_CUDA(cudaSetDevice(c->device));
    try {
      *out = new krul_snapshot{f(c)};
    } catch (const LoadError& e) {
      fld = e.field;
      throw;
    }
  });
  if (field && field_cap > 0 && !fld.empty()) {
    std::strncpy(field, fld.c_str(), size_t(field_cap) - 1);
    field[field_cap - 1] = 0;
  }
  return rc;
}
int krul_snapshot_load(krul_ctx* ctx, const void* buf, uint64_t len, const uint64_t* expected_config_hash,
                       krul_snapshot** out, char* field, int field_cap) {
  if (!buf && len) return guard([] { fail(KRUL_E_ARG, "null buffer"); });
  return load_common(ctx, field, field_cap, [&](Ctx* c) {
    return container_read(c, buf ? static_cast<const char*>(buf) : "", size_t(len), expected_config_hash);
  }, out);
}
int krul_snapshot_load_file(krul_ctx* ctx, const char* path, const uint64_t* expected_config_hash,
                            krul_snapshot** out, char* field, int field_cap) {
  if (!path) return guard([] { fail(KRUL_E_ARG, "null path"); });
  return load_common(ctx, field, field_cap, [&](Ctx* c) {
    return container_read_file(c, path, expected_config_hash);
  }, out);
}
uint32_t krul_crc32(const void* data, uint64_t len, uint32_t crc) {
  return data || !len ? kb::crc32(data ? data : "", size_t(len), crc) : crc;
}
int krul_expand(krul_snapshot* s, int layer, float* k, float* v, int64_t* start, int64_t* end) {
  return guard([&] {
    need(s, "snapshot");
    snapshot_expand(*s->s, layer, k, v, start, end);
  });
}

// ---------------------------------------------------------------- restore
int krul_restore(krul_ctx* ctx, krul_conv* conv, krul_snapshot* snap, const int32_t* hist,
                 int64_t L, krul_restore_stats* st) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    need(snap, "snapshot");
    if (L > 0) need(hist, "history");
    restore(*ctx->c, *conv->v, *snap->s, hist, L, st, nullptr, 0, nullptr, nullptr);
  });
}
int krul_restore_and_prefill(krul_ctx* ctx, krul_conv* conv, krul_snapshot* snap,
                             const int32_t* hist, int64_t L, const int32_t* nt, int64_t n_new,
                             float* logits, krul_restore_stats* st, double* ttft_ms) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    need(snap, "snapshot");
    need(nt, "new tokens");
    if (L > 0) need(hist, "history");
    restore(*ctx->c, *conv->v, *snap->s, hist, L, st, nt, n_new, logits, ttft_ms);
  });
}

int krul_restore_batch(krul_ctx* ctx, int n, krul_conv* const* convs, krul_snapshot* const* snaps,
                       const int32_t* const* histories, const int64_t* L, const int32_t* const* new_tokens,
                       const int64_t* n_new, float* logits, double* ttft_ms, double* total_ms) {
  return guard([&] {
    need(ctx, "ctx");
    if (n <= 0) fail(KRUL_E_CONFIG, "empty restore batch");
    need(convs, "convs");
    need(snaps, "snapshots");
    need(histories, "histories");
    need(L, "L");
    need(new_tokens, "new tokens");
    need(n_new, "n_new");
    std::vector<Conv*> cv(static_cast<size_t>(n));
    std::vector<Snapshot*> sv(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      need(convs[i], "conv");
      need(snaps[i], "snapshot");
      need(new_tokens[i], "new tokens");
      if (L[i] > 0) need(histories[i], "history");
      cv[size_t(i)] = convs[i]->v;
      sv[size_t(i)] = snaps[i]->s;
    }
    restore_batch(*ctx->c, n, cv.data(), sv.data(), histories, L, new_tokens, n_new, logits, ttft_ms, total_ms);
  });
}

// Measured stream rates (calibrate_rc_measured, scheduler.cpp:402-443, as
// device rates rather than a wall-clock grid): pinned H2D bytes/s over a
// 256 MiB copy and recompute flop/s of one full layer at 2048 rows.
int krul_measure_rates(krul_ctx* ctx, krul_conv* scratch, double* h2d_bps, double* flops) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    if (h2d_bps) {
      const size_t n = size_t(256) << 20;
      PinnedBuf hb;
      DevBuf db;
      void* h = hb.ensure(n);
      void* d = db.ensure(n);
      std::memset(h, 1, n);
      cudaEvent_t a, b;
      KB_CUDA(cudaEventCreate(&a));
      KB_CUDA(cudaEventCreate(&b));
      float best = 1e30f;
      for (int i = 0; i < 4; ++i) {
        KB_CUDA(cudaEventRecord(a, c.s_load));
        KB_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c.s_load));
        KB_CUDA(cudaEventRecord(b, c.s_load));
        KB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KB_CUDA(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      *h2d_bps = double(n) / (double(best) * 1e-3);
    }
    if (flops) {
      need(scratch, "scratch conversation");
      Conv& cv = *scratch->v;
      const int64_t rows = std::min<int64_t>(2048, cv.capacity);
      WS w = ws_get(c, 0, rows);
      std::vector<int32_t> tok(static_cast<size_t>(rows));
      for (int64_t i = 0; i < rows; ++i) tok[size_t(i)] = int32_t((i * 7919) % c.cfg.V);
      int32_t* d_tok = upload_tokens(c, c.s_comp, tok.data(), rows, c.ws_tok);
      launch_embed(c, c.s_comp, d_tok, rows, w.h);
      cudaEvent_t a, b;
      KB_CUDA(cudaEventCreate(&a));
      KB_CUDA(cudaEventCreate(&b));
      float best = 1e30f;
      for (int i = 0; i < 3; ++i) {
        KB_CUDA(cudaEventRecord(a, c.s_comp));
        layer_forward(c, c.s_comp, w, cv, 0, w.h, rows, 0, rows, w.h2, nullptr);
        KB_CUDA(cudaEventRecord(b, c.s_comp));
        KB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KB_CUDA(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      Cost cm;
      cm.kv_dim = c.cfg.kvd();
      cm.q_dim = c.cfg.qd();
      cm.ffn_hidden = c.cfg.F;
      cm.ffn_kind = c.cfg.ffn_kind;
      *flops = cm.layer_flops(rows, c.cfg.d) / (double(best) * 1e-3);
    }
  });
}

// calibrate_rc_measured (scheduler.cpp:402-443) on the device: for each grid
// ratio, build the plan, compress the previous turn's KV (conv `prev`, full
// span [0, L)) into a snapshot and run the real two-stream restore into
// `scratch`; pick argmin |T_C - T_L| of the measured stream finish times
// (strict <, ties to the smaller ratio). tc/tl (optional, [ng]) receive the
// measured times in sorted-grid order.
int krul_calibrate_rc_measured(krul_ctx* ctx, krul_conv* prev, krul_conv* scratch,
                               const int32_t* hist, int64_t L, const krul_pair* pairs, int np,
                               const double* grid, int ng, int mode, double* r_out, double* tc,
                               double* tl) {
  return guard([&] {
    need(ctx, "ctx");
    need(prev, "prev");
    need(scratch, "scratch");
    if (ng <= 0) fail(KRUL_E_CONFIG, "calibration grid is empty");
    Ctx& c = *ctx->c;
    std::vector<double> g(grid, grid + ng);
    std::sort(g.begin(), g.end());
    double best = g.front(), gap = 1e300;
    for (int k = 0; k < ng; ++k) {
      const std::vector<int64_t> p = build_plan(L, c.cfg.N, g[size_t(k)], pairs, np);
      std::unique_ptr<Snapshot> s(snapshot_compress(c, *prev->v, pairs, np, p.data(), L, mode));
      krul_restore_stats st{};
      restore(c, *scratch->v, *s, hist, L, &st, nullptr, 0, nullptr, nullptr);  // warm
      restore(c, *scratch->v, *s, hist, L, &st, nullptr, 0, nullptr, nullptr);
      if (tc) tc[k] = st.compute_ms;
      if (tl) tl[k] = st.load_ms;
      const double d = std::abs(st.compute_ms - st.load_ms);
      if (d < gap) {
        gap = d;
        best = g[size_t(k)];
      }
    }
    *r_out = best;
  });
}

// B200 extension of calibrate_rc_measured: the objective is the measured
// time to first token of the real restore + new-input prefill DAG (the
// prefill stream competes with the recompute stream for SMs, so the split
// that balances the bare restore is not the one that minimises TTFT). For
// each grid ratio: build the plan, compress `prev` into a snapshot, run
// `reps` restores (after one warm-up) and keep the median TTFT; returns the
// argmin (strict <, ties to the smaller ratio). ttft ([n_grid], optional)
// receives the medians in sorted-grid order.
int krul_calibrate_rc_ttft(krul_ctx* ctx, krul_conv* prev, krul_conv* scratch,
                           const int32_t* hist, int64_t L, const int32_t* new_tok, int64_t n_new,
                           const krul_pair* pairs, int np, const double* grid, int ng, int mode,
                           int reps, double* r_out, double* ttft) {
  return guard([&] {
    need(ctx, "ctx");
    need(prev, "prev");
    need(scratch, "scratch");
    if (ng <= 0) fail(KRUL_E_CONFIG, "calibration grid is empty");
    if (!new_tok || n_new <= 0) fail(KRUL_E_CONFIG, "TTFT calibration needs new input tokens");
    Ctx& c = *ctx->c;
    std::vector<double> g(grid, grid + ng);
    std::sort(g.begin(), g.end());
    double best = g.front(), best_t = 1e300;
    std::vector<float> logits(size_t(c.cfg.V));
    for (int k = 0; k < ng; ++k) {
      const std::vector<int64_t> p = build_plan(L, c.cfg.N, g[size_t(k)], pairs, np);
      std::unique_ptr<Snapshot> s(snapshot_compress(c, *prev->v, pairs, np, p.data(), L, mode));
      std::vector<double> ts;
      for (int rep = 0; rep <= std::max(1, reps); ++rep) {
        double t = 0;
        restore(c, *scratch->v, *s, hist, L, nullptr, new_tok, n_new, logits.data(), &t);
        if (rep > 0) ts.push_back(t);
      }
      std::sort(ts.begin(), ts.end());
      const double med = ts[ts.size() / 2];
      if (ttft) ttft[k] = med;
      if (med < best_t) {
        best_t = med;
        best = g[size_t(k)];
      }
    }
    *r_out = best;
  });
}

int krul_restore_timeline(krul_ctx* ctx, double* comp, double* load, double* newp) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    if (c.tl_compute.empty()) fail(KRUL_E_STATE_CORRUPTION, "no restore has run on this context");
    restore_timeline(c);
    const size_t n = c.tl_compute.size();
    if (comp) std::copy(c.tl_compute.begin(), c.tl_compute.end(), comp);
    if (load) std::copy(c.tl_load.begin(), c.tl_load.end(), load);
    if (newp) std::copy(c.tl_new.begin(), c.tl_new.begin() + n, newp);
  });
}

int krul_debug_gemm(krul_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A,
                    const float* B, const float* bias, int epi, float* Cout) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t s = c.s_comp;
    DevBuf a32, b32, a, b, out, outc, bb;
    float* da = static_cast<float*>(a32.ensure(size_t(M * K) * 4));
    float* db = static_cast<float*>(b32.ensure(size_t(N * K) * 4));
    KB_CUDA(kb_memcpy_sync(da, A, size_t(M * K) * 4, cudaMemcpyHostToDevice));
    KB_CUDA(kb_memcpy_sync(db, B, size_t(N * K) * 4, cudaMemcpyHostToDevice));
    void* ca = a.ensure(size_t(M * K) * c.esz);
    void* cb = b.ensure(size_t(N * K) * c.esz);
    launch_cvt_from_f32(c, s, da, ca, M * K);
    launch_cvt_from_f32(c, s, db, cb, N * K);
    const int64_t ncols = epi == Epi::SWIGLU ? N / 2 : N;
    float* o = static_cast<float*>(out.ensure(size_t(M * ncols) * 4 + 16));
    Epi e;
    e.kind = epi;
    e.ldo = ncols;
    if (bias) {
      float* dbias = static_cast<float*>(bb.ensure(size_t(N) * 4));
      KB_CUDA(kb_memcpy_sync(dbias, bias, size_t(N) * 4, cudaMemcpyHostToDevice));
      e.bias = dbias;
    }
    if (epi == Epi::F32 || epi == Epi::RESID) {
      e.out = o;
      if (epi == Epi::RESID) {
        KB_CUDA(kb_memcpy_sync(o, Cout, size_t(M * N) * 4, cudaMemcpyHostToDevice));
        e.resid = o;
        e.ldr = N;
      }
    } else {
      e.out = outc.ensure(size_t(M * ncols) * c.esz + 16);
    }
    gemm(c, s, M, N, K, ca, K, cb, K, e);
    if (epi == Epi::TANH || epi == Epi::SWIGLU || epi == Epi::CDT) launch_cvt_to_f32(c, s, e.out, o, M * ncols);
    KB_CUDA(cudaStreamSynchronize(s));
    KB_CUDA(kb_memcpy_sync(Cout, o, size_t(M * ncols) * 4, cudaMemcpyDeviceToHost));
  });
}


// Device-resident GEMM timing for kernel tuning (not on the product path):
// random bf16 A[M,K], B[N,K], `iters` back-to-back launches timed with CUDA
// events on the compute stream. force: 0 planner, 1 1-SM BN256, 2 1-SM
// BN128, 3 pair, 4 pair BK128; splits: 0 planner.
// Pins the GEMM plan of later calls (tests): force 0 auto, 1 / 2 1-SM 256 /
// 128-wide, 3 pair, 5 / 6 stream-K 256 / 128-wide; splits 0 = auto.
int krul_debug_set_gemm_plan(int force, int splits) {
  return guard([&] {
    g_gemm_force = force;
    g_gemm_splits = splits;
  });
}
// Phase timeline of one weight-streaming GEMM launch (globaltimer ns, see
// g_gemm_ts in gemm.cu): ts[0..9] CTA 0 phases, ts[32 + b] / ts[288 + b]
// entry / exit of CTA b (b < 256). The weights are streamed from HBM.
int krul_debug_gemm_timeline(krul_ctx* ctx, int64_t M, int64_t N, int64_t K, int epi, int force, int splits,
                             unsigned long long* ts_out /* [544] */) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t s = c.s_comp;
    DevBuf a, b, out, res, out2, ts, flush;
    void* da = a.ensure(size_t(std::max<int64_t>(M, 128) * K) * 2);
    void* db = b.ensure(size_t(N * K) * 2);
    launch_init_uniform(c, s, da, std::max<int64_t>(M, 128) * K, 1, 1, 1.0f);
    launch_init_uniform(c, s, db, N * K, 1, 2, 0.02f);
    Epi e;
    e.kind = epi;
    e.a_rows = std::max<int64_t>(M, 128);
    e.out = out.ensure(size_t(M * N) * 4 + 16);
    e.ldo = epi == Epi::SWIGLU ? N / 2 : N;
    if (epi == Epi::RESID) {
      e.resid = static_cast<float*>(res.ensure(size_t(M * N) * 4));
      KB_CUDA(cudaMemsetAsync(const_cast<float*>(e.resid), 0, size_t(M * N) * 4, s));
      e.ldr = N;
      e.out2 = out2.ensure(size_t(M * N) * 2);
      e.ldo2 = N;
    }
    unsigned long long* dts = static_cast<unsigned long long*>(ts.ensure(544 * 8));
    KB_CUDA(cudaMemsetAsync(dts, 0, 544 * 8, s));
    g_gemm_force = force;
    g_gemm_splits = splits;
    try {
      gemm(c, s, M, N, K, da, K, db, K, e);  // warm (plan, maps)
      void* fl = flush.ensure(size_t(256) << 20);  // evict the weights from L2
      KB_CUDA(cudaMemsetAsync(fl, 1, size_t(256) << 20, s));
      // the activations / residual were just written by the producing kernel
      // in the layer chain: L2-resident, as there
      launch_init_uniform(c, s, da, std::max<int64_t>(M, 128) * K, 1, 1, 1.0f);
      if (epi == Epi::RESID) KB_CUDA(cudaMemsetAsync(const_cast<float*>(e.resid), 0, size_t(M * N) * 4, s));
      KB_CUDA(cudaStreamSynchronize(s));
      gemm_set_timeline(dts);
      gemm(c, s, M, N, K, da, K, db, K, e);
      KB_CUDA(cudaStreamSynchronize(s));
      gemm_set_timeline(nullptr);
    } catch (...) {
      g_gemm_force = 0;
      g_gemm_splits = 0;
      gemm_set_timeline(nullptr);
      throw;
    }
    g_gemm_force = 0;
    g_gemm_splits = 0;
    KB_CUDA(cudaMemcpy(ts_out, dts, 544 * 8, cudaMemcpyDeviceToHost));
  });
}

int krul_debug_gemm_bench(krul_ctx* ctx, int64_t M, int64_t N, int64_t K, int epi, int force,
                          int splits, int iters, float* ms_per_iter) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    if (c.cfg.dtype != KRUL_BF16) fail(KRUL_E_CONFIG, "gemm bench needs a bf16 context");
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t s = c.s_comp;
    DevBuf a, b, out, res, out2, bias;
    // A padded to a 128-row tile like the layer workspaces (Epi::a_rows)
    void* da = a.ensure(size_t(std::max<int64_t>(M, 128) * K) * 2);
    // weights rotate over >= 320 MB so every launch streams them from HBM as
    // in the restore DAG (one layer's weights fit the 126 MB L2)
    const size_t wbytes = size_t(N * K) * 2;
    const int nb = int(std::max<size_t>(1, ((size_t(320) << 20) + wbytes - 1) / wbytes));
    char* db0 = static_cast<char*>(b.ensure(wbytes * nb));
    launch_init_uniform(c, s, da, std::max<int64_t>(M, 128) * K, 1, 1, 1.0f);
    launch_init_uniform(c, s, db0, N * K * nb, 1, 2, 0.02f);
    Epi e;
    e.kind = epi;
    e.a_rows = std::max<int64_t>(M, 128);
    e.out = out.ensure(size_t(M * N) * 4 + 16);
    e.ldo = epi == Epi::SWIGLU ? N / 2 : N;
    if (epi == Epi::RESID) {
      e.resid = static_cast<float*>(res.ensure(size_t(M * N) * 4));
      KB_CUDA(cudaMemsetAsync(const_cast<float*>(e.resid), 0, size_t(M * N) * 4, s));
      e.ldr = N;
      e.out2 = out2.ensure(size_t(M * N) * 2);
      e.ldo2 = N;
    }
    if (epi == Epi::TANH) {
      e.bias = static_cast<float*>(bias.ensure(size_t(N) * 4));
      KB_CUDA(cudaMemsetAsync(const_cast<float*>(e.bias), 0, size_t(N) * 4, s));
    }
    g_gemm_force = force;
    g_gemm_splits = splits;
    try {
      for (int i = 0; i < 2; ++i) gemm(c, s, M, N, K, da, K, db0 + wbytes * (i % nb), K, e);
      KB_CUDA(cudaStreamSynchronize(s));
      // the launches are captured into a graph and replayed (as in the restore
      // DAG): device time, not the host's per-launch cost
      cudaGraph_t graph = nullptr;
      cudaGraphExec_t exec = nullptr;
      KB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
      for (int i = 0; i < iters; ++i) gemm(c, s, M, N, K, da, K, db0 + wbytes * (i % nb), K, e);
      KB_CUDA(cudaStreamEndCapture(s, &graph));
      KB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      KB_CUDA(cudaGraphLaunch(exec, s));  // warm
      cudaEvent_t e0 = c.event(), e1 = c.event();
      KB_CUDA(cudaEventRecord(e0, s));
      KB_CUDA(cudaGraphLaunch(exec, s));
      KB_CUDA(cudaEventRecord(e1, s));
      KB_CUDA(cudaEventSynchronize(e1));
      cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
      float ms = 0;
      KB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      *ms_per_iter = ms / float(iters);
    } catch (...) {
      g_gemm_force = 0;
      g_gemm_splits = 0;
      throw;
    }
    g_gemm_force = 0;
    g_gemm_splits = 0;
    c.reset_events();
  });
}


// ---- measurement support (bench evidence) -----------------------------------
int krul_launch_count(uint64_t* n) {
  return guard([&] {
    need(n, "n");
    *n = g_launches.load();
  });
}
int krul_ktime_enable(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaDeviceSynchronize());
    c.drop_graph();  // captured event nodes belong to the previous timing window
    c.kt.on = on != 0;
    c.kt.recs.clear();
    c.kt.next = 0;
  });
}
int krul_ktime_read(krul_ctx* ctx, int tag, int64_t* launches, double* ms, double* flops,
                    double* bytes) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaDeviceSynchronize());
    int64_t n = 0;
    double t = 0, f = 0, b = 0;
    for (const auto& r : c.kt.recs) {
      if (r.tag != tag) continue;
      float x = 0;
      KB_CUDA(cudaEventElapsedTime(&x, r.a, r.b));
      ++n;
      t += x;
      f += r.flops;
      b += r.bytes;
    }
    if (launches) *launches = n;
    if (ms) *ms = t;
    if (flops) *flops = f;
    if (bytes) *bytes = b;
  });
}


// Attention timing for kernel tuning (not on the product path): fills
// `conv`'s pages for [0, pos0 + rows) of `layer` with the history's real
// prefill first (caller's job), then times `iters` launches of the tcgen05
// attention for `rows` query rows at position pos0 with random Q.
int krul_debug_attn_bench(krul_ctx* ctx, krul_conv* conv, int layer, int64_t rows, int64_t pos0,
                          int dbg, int target, int iters, float* ms_per_iter) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    Ctx& c = *ctx->c;
    if (c.cfg.dtype != KRUL_BF16) fail(KRUL_E_CONFIG, "attention bench needs a bf16 context");
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t s = c.s_comp;
    DevBuf q, out, part;
    void* dq = q.ensure(size_t(rows) * c.cfg.qd() * 2);
    launch_init_uniform(c, s, dq, rows * c.cfg.qd(), 5, 5, 1.0f);
    AttnArgs a{};
    a.q = dq;
    a.rows = rows;
    a.pos0 = pos0;
    a.out = out.ensure(size_t(rows) * c.cfg.qd() * 2);
    a.part = &part;
    g_attn_target = target;
    g_attn_dbg = dbg;
    for (int i = 0; i < 2; ++i) launch_attention_tc(c, s, *conv->v, layer, a, part);
    // the launches are captured into a graph and replayed, so the timing
    // is device time (host tensor-map encoding would otherwise dominate)
    KB_CUDA(cudaStreamSynchronize(s));
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    KB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < iters; ++i) launch_attention_tc(c, s, *conv->v, layer, a, part);
    KB_CUDA(cudaStreamEndCapture(s, &graph));
    KB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    KB_CUDA(cudaGraphLaunch(exec, s));  // warm
    cudaEvent_t e0 = c.event(), e1 = c.event();
    KB_CUDA(cudaEventRecord(e0, s));
    KB_CUDA(cudaGraphLaunch(exec, s));
    KB_CUDA(cudaEventRecord(e1, s));
    KB_CUDA(cudaEventSynchronize(e1));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    g_attn_target = 0;
    g_attn_dbg = 0;
    float ms = 0;
    KB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_iter = ms / float(iters);
    c.reset_events();
  });
}

// Phase stamps of one tcgen05 attention launch (kernel tuning, not on the
// product path): ts[cta * 8 + slot] in ns (%globaltimer), see attn_ts.
int krul_debug_attn_timeline(krul_ctx* ctx, krul_conv* conv, int layer, int64_t rows, int64_t pos0, int target,
                             unsigned long long* ts, int64_t n_ts) {
  return guard([&] {
    need(ctx, "ctx");
    need(conv, "conv");
    need(ts, "ts");
    Ctx& c = *ctx->c;
    if (c.cfg.dtype != KRUL_BF16) fail(KRUL_E_CONFIG, "attention timeline needs a bf16 context");
    KB_CUDA(cudaSetDevice(c.device));
    cudaStream_t s = c.s_comp;
    DevBuf q, out, part, dts;
    void* dq = q.ensure(size_t(rows) * c.cfg.qd() * 2);
    launch_init_uniform(c, s, dq, rows * c.cfg.qd(), 5, 5, 1.0f);
    AttnArgs a{};
    a.q = dq;
    a.rows = rows;
    a.pos0 = pos0;
    a.out = out.ensure(size_t(rows) * c.cfg.qd() * 2);
    a.part = &part;
    g_attn_target = target;
    for (int i = 0; i < 2; ++i) launch_attention_tc(c, s, *conv->v, layer, a, part);
    unsigned long long* d = static_cast<unsigned long long*>(dts.ensure(size_t(n_ts) * 8));
    KB_CUDA(cudaMemsetAsync(d, 0, size_t(n_ts) * 8, s));
    KB_CUDA(cudaStreamSynchronize(s));
    attn_set_timeline(d);
    launch_attention_tc(c, s, *conv->v, layer, a, part);
    KB_CUDA(cudaStreamSynchronize(s));
    attn_set_timeline(nullptr);
    g_attn_target = 0;
    KB_CUDA(cudaMemcpy(ts, d, size_t(n_ts) * 8, cudaMemcpyDeviceToHost));
  });
}


// Device time of the decode fold (K1) on the last captured decode rows:
// `iters` folds enqueued back to back on the estimator stream between two
// events (no host gaps), into a scratch accumulator (the estimator's sums
// are untouched). bytes_per_fold = the algorithmic HBM bytes of one fold.
int krul_est_fold_bench(krul_est* est, int iters, float* ms_per_fold, double* bytes_per_fold) {
  return guard([&] {
    need(est, "est");
    Est& e = *est->e;
    Ctx& c = *e.ctx;
    if (!c.dec_valid) fail(KRUL_E_STATE_CORRUPTION, "no captured decode step");
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaDeviceSynchronize());
    const int64_t W = c.dec_width, pitch = c.dec_pitch;
    const int n = int(e.layers.size());
    const int sms = c.sm_count > 0 ? c.sm_count : 148;
    DevBuf scratch;  // the bench folds into scratch slots: the estimator's sums stay untouched
    const size_t nseg = size_t(e.seg_S) * std::max(e.P(), 1) * e.H;
    double* seg = static_cast<double*>(scratch.ensure(nseg * 8));
    KB_CUDA(kb_memset_sync(seg, 0, nseg * 8));
    const float* rows = c.dec_rows.as<float>();
    auto fold = [&] {
      launch_fold_direct(c.s_est, rows, int64_t(e.H) * pitch, pitch, W, e.H, e.d_layers.as<int>(), n, seg,
                         e.seg_S, sms);
    };
    fold();  // warm
    KB_CUDA(cudaStreamSynchronize(c.s_est));
    // the folds as one captured graph (as in a captured decode loop): device
    // time without host launch gaps
    iters = std::max(iters, 1);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    KB_CUDA(cudaStreamBeginCapture(c.s_est, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) fold();
    KB_CUDA(cudaStreamEndCapture(c.s_est, &g));
    KB_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    KB_CUDA(cudaEventCreate(&a));
    KB_CUDA(cudaEventCreate(&b));
    KB_CUDA(cudaGraphLaunch(ge, c.s_est));
    KB_CUDA(cudaEventRecord(a, c.s_est));
    KB_CUDA(cudaGraphLaunch(ge, c.s_est));
    KB_CUDA(cudaEventRecord(b, c.s_est));
    KB_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    KB_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    *ms_per_fold = ms / float(std::max(iters, 1));
    *bytes_per_fold = double(e.layers.size()) * e.H * double(W) * 4.0 + double(e.P()) * e.H * 16.0;
  });
}

// Debug: per-CTA %globaltimer stamps of the next decode folds ([cta][8] u64:
// entry, after setup, after the chunk loop, chunks 0-3 in shared memory;
// [7] = SM id; a CTA with an empty range stamps only entry). on = 1 arms a device
// buffer, on = 0 copies it into ts (n_ts entries) and disarms.
int krul_debug_fold_timeline(int on, unsigned long long* ts, int64_t n_ts) {
  return guard([&] {
    static DevBuf buf;
    if (on) {
      buf.ensure(size_t(std::max<int64_t>(n_ts, 8)) * 8);
      KB_CUDA(cudaMemset(buf.p, 0, size_t(std::max<int64_t>(n_ts, 8)) * 8));
      fold_set_timeline(static_cast<unsigned long long*>(buf.p));
    } else {
      need(ts, "ts");
      KB_CUDA(cudaDeviceSynchronize());
      KB_CUDA(cudaMemcpy(ts, buf.p, size_t(n_ts) * 8, cudaMemcpyDeviceToHost));
      fold_set_timeline(nullptr);
    }
  });
}

// Restore scheduling mode: 1 (default) runs the new-input prefill on its own
// stream, concurrent with the recompute; 0 serialises it behind the
// recompute (kernel-efficiency measurements without SM sharing).
int krul_set_timeline(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->timeline = on != 0;
  });
}
// Device-side spans of the weight-streaming GEMMs (M <= 128) of the next
// restores: every launch stamps its first CTA entry and last CTA exit
// (%globaltimer) into its slot; no events sit between the kernels.
int krul_span_enable(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaDeviceSynchronize());
    c.drop_graph();
    c.span_on = on != 0;
    unsigned long long* d = nullptr;
    if (c.span_on) d = static_cast<unsigned long long*>(c.span_buf.ensure(sizeof(unsigned long long) * 2 * Ctx::kSpanSlots));
    gemm_set_span(d);
  });
}
// Sum over the last restore's stamped launches: count, span ms, algorithmic bytes.
int krul_span_read(krul_ctx* ctx, int64_t* launches, double* ms, double* bytes) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    KB_CUDA(cudaSetDevice(c.device));
    KB_CUDA(cudaDeviceSynchronize());
    const int n = std::min<int>(c.span_next, Ctx::kSpanSlots);
    std::vector<unsigned long long> h(size_t(2) * Ctx::kSpanSlots);
    if (c.span_on && n > 0) KB_CUDA(cudaMemcpy(h.data(), c.span_buf.p, h.size() * 8, cudaMemcpyDeviceToHost));
    int64_t k = 0;
    double t = 0, b = 0;
    for (int i = 0; i < n; ++i) {
      const unsigned long long a = h[size_t(i)], e = h[size_t(Ctx::kSpanSlots + i)];
      if (a == ~0ull || e == 0 || e < a) continue;
      ++k;
      t += double(e - a) * 1e-6;
      b += c.span_bytes[size_t(i)];
    }
    if (launches) *launches = k;
    if (ms) *ms = t;
    if (bytes) *bytes = b;
  });
}
int krul_set_graphs(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->drop_graph();
    ctx->c->use_graphs = on != 0;
  });
}
int krul_set_fused_recompute(krul_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->fused = on != 0;
  });
}
int krul_set_concurrency(krul_ctx* ctx, int two_stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->two_stream = two_stream != 0;
  });
}


// Roofline-normalised time of the timed launches of a kernel class: the sum
// over launches of max(flops / peak_flops, bytes / peak_bytes) -- what the
// launches would take at the binding roof (tensor or HBM) of each shape.
int krul_ktime_roofline(krul_ctx* ctx, int tag, double peak_tflops, double peak_gbs, double* ideal_ms) {
  return guard([&] {
    need(ctx, "ctx");
    need(ideal_ms, "ideal_ms");
    Ctx& c = *ctx->c;
    double t = 0;
    for (const auto& r : c.kt.recs) {
      if (r.tag != tag) continue;
      const double tf = peak_tflops > 0 ? r.flops / (peak_tflops * 1e12) : 0.0;
      const double tb = peak_gbs > 0 ? r.bytes / (peak_gbs * 1e9) : 0.0;
      t += 1e3 * std::max(tf, tb);
    }
    *ideal_ms = t;
  });
}

}  // extern "C"
