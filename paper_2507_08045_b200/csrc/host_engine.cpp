// host_engine.cpp — the engine on the device: weights, paged conversations,
// one-layer forward (K6/K7 building block), prefill, decode, pyramid
// recompute, and the two-stream restore DAG (K4/K5 || K6).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kb.hpp"
#include "host.hpp"

namespace kb {

// ---------------------------------------------------------------- context
Ctx* ctx_create(int device, const krul_model_desc& desc) {
  Cfg cfg = cfg_from_desc(desc);
  int ndev = 0;
  KB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(KRUL_E_CONFIG, "device index out of range");
  KB_CUDA(cudaSetDevice(device));
  auto* c = new Ctx;
  c->device = device;
  c->cfg = cfg;
  c->esz = cfg.dtype == KRUL_BF16 ? 2 : 4;
  try {
    KB_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    KB_CUDA(cudaStreamCreateWithFlags(&c->s_load, cudaStreamNonBlocking));
    {
      // stream priorities (lower number = higher priority): the new-input
      // prefill and the recompute are both on the TTFT critical path
      int lo = 0, hi = 0;
      KB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const char* pv = std::getenv("KRUL_NEW_PRIO");
      const int prio = pv && pv[0] == 'h' ? hi : lo;
      KB_CUDA(cudaStreamCreateWithPriority(&c->s_new, cudaStreamNonBlocking, prio));
      const char* cv = std::getenv("KRUL_COMP_PRIO");
      if (cv && cv[0] == 'h') {
        KB_CUDA(cudaStreamDestroy(c->s_comp));
        KB_CUDA(cudaStreamCreateWithPriority(&c->s_comp, cudaStreamNonBlocking, hi));
      }
    }
    KB_CUDA(cudaStreamCreateWithFlags(&c->s_est, cudaStreamNonBlocking));
    {
      // decode + expand of the blob the load stream just landed gate the
      // new-input prefill of that layer: their CTAs go first when SMs free up
      int lo = 0, hi = 0;
      KB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const char* ev = std::getenv("KRUL_EXP_PRIO");
      KB_CUDA(cudaStreamCreateWithPriority(&c->s_exp, cudaStreamNonBlocking, ev && ev[0] == 'l' ? lo : hi));
    }
    KB_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    // RoPE table: angles in double, cast to float (engine.cpp:131-136).
    const int half = cfg.hd / 2;
    const int64_t T = cfg.max_tokens + 1;
    std::vector<float> cs(size_t(T) * std::max(half, 1)), sn(cs.size());
    for (int64_t pos = 0; pos < T; ++pos)
      for (int i = 0; i < half; ++i) {
        const double th = double(pos) * std::pow(cfg.theta, -2.0 * i / double(cfg.hd));
        cs[size_t(pos) * half + i] = float(std::cos(th));
        sn[size_t(pos) * half + i] = float(std::sin(th));
      }
    c->rope.ensure(2 * cs.size() * sizeof(float));
    c->rope_cos = c->rope.as<float>();
    c->rope_sin = c->rope_cos + cs.size();
    KB_CUDA(kb_memcpy_sync(c->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
    KB_CUDA(kb_memcpy_sync(c->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
    // KV page pool: room for KRUL_KV_POOL_CONVS conversations of max_tokens.
    int convs = 2;
    if (const char* v = std::getenv("KRUL_KV_POOL_CONVS")) convs = std::max(1, std::atoi(v));
    const int64_t pages_per_layer = (cfg.max_tokens + kPageTokens - 1) / kPageTokens;
    c->pool_pages = int(pages_per_layer * cfg.N * convs);
    c->pool.ensure(size_t(c->pool_pages) * c->page_elems() * c->esz);
    // zeroed once so never-written positions of a page are finite (masked
    // keys still multiply V inside the tensor-core P V product)
    KB_CUDA(kb_memset_sync(c->pool.p, 0, size_t(c->pool_pages) * c->page_elems() * c->esz));
    c->free_pages.resize(size_t(c->pool_pages));
    for (int i = 0; i < c->pool_pages; ++i) c->free_pages[size_t(i)] = c->pool_pages - 1 - i;
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

// Weight arena: per layer wqkv, wo, w1, w2 (compute dtype) + biases (f32),
// then embed and unembed^T.
static void carve_weights(Ctx& c) {
  const Cfg& g = c.cfg;
  const int64_t d = g.d, F = g.F;
  const int64_t w1rows = g.ffn_kind == KRUL_FFN_SWIGLU ? 2 * F : F;
  const int64_t per_layer = int64_t(g.nqkv()) * d + d * g.qd() + w1rows * d + d * F;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t total = 0;
  std::vector<size_t> off;
  for (int l = 0; l < g.N; ++l) {
    off.push_back(total);
    total = align(total + size_t(per_layer) * c.esz);
    off.push_back(total);
    total = align(total + size_t(F + d) * 4);
  }
  const size_t emb_off = total;
  total = align(total + size_t(g.V) * d * c.esz);
  const size_t un_off = total;
  total = align(total + size_t(g.V) * d * c.esz);
  char* base = static_cast<char*>(c.wbuf.ensure(total));
  KB_CUDA(kb_memset_sync(base, 0, total));
  c.L.assign(size_t(g.N), LayerW{});
  for (int l = 0; l < g.N; ++l) {
    char* p = base + off[size_t(2 * l)];
    LayerW& w = c.L[size_t(l)];
    w.wqkv = p;
    p += size_t(g.nqkv()) * d * c.esz;
    w.wo = p;
    p += size_t(d) * g.qd() * c.esz;
    w.w1 = p;
    p += size_t(w1rows) * d * c.esz;
    w.w2 = p;
    float* b = reinterpret_cast<float*>(base + off[size_t(2 * l + 1)]);
    w.b1 = b;
    w.b2 = b + F;
  }
  c.embed = base + emb_off;
  c.unembedT = base + un_off;
}

// engine.cpp:361-395 draw order: embed, per layer wq wk wv wo w1 b1 w2 b2
// (SwiGLU: wq wk wv wo gate up w2), unembed. Row-major [in][out] f32.
void weights_upload_f32(Ctx& c, const float* w, int64_t n) {
  const Cfg& g = c.cfg;
  const int64_t d = g.d, F = g.F, qd = g.qd(), kvd = g.kvd();
  int64_t need = 2 * int64_t(g.V) * d;
  for (int l = 0; l < g.N; ++l) {
    need += d * qd + 2 * d * kvd + qd * d + d * F + F * d;
    need += g.ffn_kind == KRUL_FFN_SWIGLU ? d * F : F + d;
  }
  if (n != need) fail(KRUL_E_CONFIG, "weight count " + std::to_string(n) + " != expected " + std::to_string(need));
  KB_CUDA(cudaSetDevice(c.device));
  carve_weights(c);
  cudaStream_t s = c.s_comp;
  DevBuf tmp;
  const float* src = w;
  auto upload = [&](int64_t rows, int64_t cols) -> float* {
    float* p = static_cast<float*>(tmp.ensure(size_t(rows * cols) * 4));
    KB_CUDA(cudaStreamSynchronize(s));
    KB_CUDA(kb_memcpy_sync(p, src, size_t(rows * cols) * 4, cudaMemcpyHostToDevice));
    src += rows * cols;
    return p;
  };
  auto at_row = [&](void* base, int64_t row, int64_t ld) {
    return static_cast<char*>(base) + size_t(row * ld) * c.esz;
  };
  // embed [V][d] as is
  launch_convert_weights(c, s, upload(g.V, d), c.embed, g.V, d, 0, 0);
  for (int l = 0; l < g.N; ++l) {
    LayerW& lw = c.L[size_t(l)];
    launch_convert_weights(c, s, upload(d, qd), lw.wqkv, d, qd, 1, 0);
    launch_convert_weights(c, s, upload(d, kvd), at_row(lw.wqkv, qd, d), d, kvd, 1, 0);
    launch_convert_weights(c, s, upload(d, kvd), at_row(lw.wqkv, qd + kvd, d), d, kvd, 1, 0);
    launch_convert_weights(c, s, upload(qd, d), lw.wo, qd, d, 1, 0);
    if (g.ffn_kind == KRUL_FFN_TANH) {
      launch_convert_weights(c, s, upload(d, F), lw.w1, d, F, 1, 0);
      KB_CUDA(kb_memcpy_sync(lw.b1, src, size_t(F) * 4, cudaMemcpyHostToDevice));
      src += F;
      launch_convert_weights(c, s, upload(F, d), lw.w2, F, d, 1, 0);
      KB_CUDA(kb_memcpy_sync(lw.b2, src, size_t(d) * 4, cudaMemcpyHostToDevice));
      src += d;
    } else {
      launch_convert_weights(c, s, upload(d, F), lw.w1, d, F, 1, 1);  // gate -> even rows
      launch_convert_weights(c, s, upload(d, F), lw.w1, d, F, 1, 2);  // up -> odd rows
      launch_convert_weights(c, s, upload(F, d), lw.w2, F, d, 1, 0);
    }
  }
  launch_convert_weights(c, s, upload(d, g.V), c.unembedT, d, g.V, 1, 0);
  KB_CUDA(cudaStreamSynchronize(s));
  c.weights_ready = true;
}

void weights_init_device(Ctx& c, uint64_t seed) {
  const Cfg& g = c.cfg;
  KB_CUDA(cudaSetDevice(c.device));
  carve_weights(c);
  cudaStream_t s = c.s_comp;
  const float bound = 1.0f / std::sqrt(float(g.d));
  const int64_t d = g.d, F = g.F;
  const int64_t w1rows = g.ffn_kind == KRUL_FFN_SWIGLU ? 2 * F : F;
  uint64_t sid = 1;
  launch_init_uniform(c, s, c.embed, int64_t(g.V) * d, seed, sid++, bound);
  for (int l = 0; l < g.N; ++l) {
    LayerW& w = c.L[size_t(l)];
    launch_init_uniform(c, s, w.wqkv, int64_t(g.nqkv()) * d, seed, sid++, bound);
    launch_init_uniform(c, s, w.wo, d * g.qd(), seed, sid++, bound);
    launch_init_uniform(c, s, w.w1, w1rows * d, seed, sid++, bound);
    launch_init_uniform(c, s, w.w2, d * F, seed, sid++, bound);
    if (g.ffn_kind == KRUL_FFN_TANH) {
      launch_init_uniform_f32(s, w.b1, F, seed, sid++, bound);
      launch_init_uniform_f32(s, w.b2, d, seed, sid++, bound);
    }
  }
  launch_init_uniform(c, s, c.unembedT, int64_t(g.V) * d, seed, sid++, bound);
  KB_CUDA(cudaStreamSynchronize(s));
  c.weights_ready = true;
}

// ---------------------------------------------------------------- conversations
Conv* conv_create(Ctx& c, int64_t capacity) {
  if (capacity < 1 || capacity > c.cfg.max_tokens)
    fail(KRUL_E_CONFIG, "conversation capacity must lie in [1, max_tokens]");
  const int maxp = int((capacity + kPageTokens - 1) / kPageTokens);
  const size_t need = size_t(maxp) * c.cfg.N;
  if (c.free_pages.size() < need) fail(KRUL_E_CONFIG, "KV page pool exhausted (raise KRUL_KV_POOL_CONVS)");
  auto* v = new Conv;
  v->ctx = &c;
  v->capacity = capacity;
  v->max_pages = maxp;
  v->serial = next_serial();
  c.convs.push_back(v);
  v->pages.resize(need);
  for (size_t i = 0; i < need; ++i) {
    v->pages[i] = c.free_pages.back();
    c.free_pages.pop_back();
  }
  KB_CUDA(cudaSetDevice(c.device));
  KB_CUDA(cudaMalloc(&v->d_pt, need * sizeof(int)));
  g_buf_gen.fetch_add(1);  // a captured graph never outlives the page tables it baked in
  KB_CUDA(kb_memcpy_sync(v->d_pt, v->pages.data(), need * sizeof(int), cudaMemcpyHostToDevice));
  return v;
}

// ---------------------------------------------------------------- workspaces
constexpr int64_t kWsMinRows = 128;
WS ws_get(Ctx& c, int set, int64_t rows) {
  const Cfg& g = c.cfg;
  const size_t r = size_t(std::max<int64_t>(rows, 1));
  const size_t ra = std::max<size_t>(r, kWsMinRows);  // GEMM A operands: >= one 128-row tile
  WS w;
  DevBuf* h = set == 0 ? &c.ws_h : &c.ws_new_h;
  DevBuf* h2 = set == 0 ? &c.ws_h2 : &c.ws_new_h2;
  DevBuf* xn = set == 0 ? &c.ws_xn : &c.ws2_xn;
  DevBuf* qkv = set == 0 ? &c.ws_qkv : &c.ws2_qkv;
  DevBuf* q = set == 0 ? &c.ws_q : &c.ws2_q;
  DevBuf* at = set == 0 ? &c.ws_attn : &c.ws2_attn;
  DevBuf* hm = set == 0 ? &c.ws_hmid : &c.ws2_hmid;
  DevBuf* hc = set == 0 ? &c.ws_hmidc : &c.ws2_hmidc;
  DevBuf* act = set == 0 ? &c.ws_act : &c.ws2_act;
  w.h = static_cast<float*>(h->ensure(r * g.d * 4));
  w.h2 = static_cast<float*>(h2->ensure(r * g.d * 4));
  w.xn = xn->ensure(ra * g.d * c.esz);
  w.qkv = static_cast<float*>(qkv->ensure(r * g.nqkv() * 4));
  w.q = q->ensure(r * g.qd() * c.esz);
  w.attn = at->ensure(ra * g.qd() * c.esz);
  w.hmid = static_cast<float*>(hm->ensure(r * g.d * 4));
  w.hmidc = hc->ensure(ra * g.d * c.esz);
  w.act = act->ensure(ra * g.F * c.esz);
  w.part = set == 0 ? &c.ws_part : &c.ws2_part;
  return w;
}

// ---------------------------------------------------------------- one layer
// engine.cpp:150-193: block rows [pos0, pos0 + rows) append K/V to `layer`'s
// pages; attention + FFN for the leading out_rows rows -> h_out.
void layer_forward(Ctx& c, cudaStream_t s, const WS& w, Conv& conv, int l, const float* h_in,
                   int64_t rows, int64_t pos0, int64_t out_rows, float* h_out,
                   const AttnArgs* cap, const FusedSeg* fs) {
  const Cfg& g = c.cfg;
  const LayerW& lw = c.L[size_t(l)];
  if (rows <= 0) return;
  // the fused step waits for the layer's loaded suffix before it starts: a
  // QKV GEMM launched early holds every SM's shared memory while the blob's
  // decode + expand (the critical path) need them
  if (fs)
    for (int k = 0; k < fs->n_waits; ++k) KB_CUDA(cudaStreamWaitEvent(s, fs->waits[k], 0));
  launch_rmsnorm(c, s, h_in, rows, w.xn);
  Epi e;
  e.a_rows = kWsMinRows;  // workspace A operands hold >= 128 rows
  if (gemm_uses_tc(c, w.xn, g.d, lw.wqkv, g.d) && g.hd % 32 == 0) {
    // tcgen05 path: RoPE + paged K/V^T scatter + Q fused into the epilogue
    e.kind = Epi::QKV;
    e.kv.pt = conv.d_pt + int64_t(l) * conv.max_pages;
    e.kv.pool = static_cast<char*>(c.pool.p);
    e.kv.page_bytes = int64_t(c.page_elems() * c.esz);
    e.kv.H = g.H;
    e.kv.Hkv = g.Hkv;
    e.kv.hd = g.hd;
    e.kv.pos0 = pos0;
    e.kv.q_rows = out_rows;
    if (fs) {
      e.kv.seg_rows = fs->n_new;
      e.kv.pos1 = 0;
    }
    e.kv.cosT = c.rope_cos;
    e.kv.sinT = c.rope_sin;
    e.kv.q = w.q;
    gemm(c, s, rows, g.nqkv(), g.d, w.xn, g.d, lw.wqkv, g.d, e);
  } else {
    e.kind = Epi::F32;
    e.out = w.qkv;
    e.ldo = g.nqkv();
    gemm(c, s, rows, g.nqkv(), g.d, w.xn, g.d, lw.wqkv, g.d, e);
    launch_rope_scatter(c, s, w.qkv, rows, pos0, out_rows, w.q, conv, l, fs ? fs->n_new : INT64_MAX, 0);
  }
  if (fs && fs->computed) record_mark(*fs->computed, s);
  if (out_rows <= 0) return;
  if (cap && cap->q_save)  // K2: the rotated Q of the captured rows
    KB_CUDA(cudaMemcpyAsync(cap->q_save, w.q, size_t(fs ? fs->n_new : out_rows) * g.qd() * c.esz,
                            cudaMemcpyDeviceToDevice, s));
  AttnArgs a = cap ? *cap : AttnArgs{};
  a.part = w.part;
  a.q = w.q;
  a.rows = fs ? fs->n_new : out_rows;
  a.pos0 = pos0;
  a.out = w.attn;
  if (fs) {
    // recomputed rows first (their keys are this step's own), then the new
    // rows once the layer's loaded suffix is in the pages
    if (fs->rec_out > 0) {
      AttnArgs ar{};
      ar.part = w.part;
      const size_t off = size_t(fs->n_new) * size_t(g.qd()) * c.esz;
      ar.q = static_cast<const char*>(w.q) + off;
      ar.rows = fs->rec_out;
      ar.pos0 = 0;
      ar.out = static_cast<char*>(w.attn) + off;
      launch_attention(c, s, conv, l, ar);
    }
  }
  launch_attention(c, s, conv, l, a);
  Epi eo;
  eo.a_rows = kWsMinRows;  // workspace A operands hold >= 128 rows
  eo.kind = Epi::RESID;
  eo.out = w.hmid;
  eo.ldo = g.d;
  eo.resid = h_in;
  eo.ldr = g.d;
  eo.out2 = w.hmidc;
  eo.ldo2 = g.d;
  gemm(c, s, out_rows, g.d, g.qd(), w.attn, g.qd(), lw.wo, g.qd(), eo);
  Epi e1;
  e1.a_rows = kWsMinRows;  // workspace A operands hold >= 128 rows
  e1.out = w.act;
  e1.ldo = g.F;
  if (g.ffn_kind == KRUL_FFN_TANH) {
    e1.kind = Epi::TANH;
    e1.bias = lw.b1;
    gemm(c, s, out_rows, g.F, g.d, w.hmidc, g.d, lw.w1, g.d, e1);
  } else {
    // Llama FFN block: RMSNorm (gain-less, as the attention pre-norm) before
    // the gated FFN; the residual keeps the un-normalised h_mid
    launch_rmsnorm(c, s, w.hmid, out_rows, w.hmidc);
    e1.kind = Epi::SWIGLU;
    gemm(c, s, out_rows, 2 * int64_t(g.F), g.d, w.hmidc, g.d, lw.w1, g.d, e1);
  }
  Epi e2;
  e2.a_rows = kWsMinRows;  // workspace A operands hold >= 128 rows
  e2.kind = Epi::RESID;
  e2.out = h_out;
  e2.ldo = g.d;
  e2.resid = w.hmid;
  e2.ldr = g.d;
  e2.bias = g.ffn_kind == KRUL_FFN_TANH ? lw.b2 : nullptr;
  gemm(c, s, out_rows, g.d, g.F, w.act, g.F, lw.w2, g.F, e2);
}

void check_tokens(const Ctx& c, const int32_t* t, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (t[i] < 0 || t[i] >= c.cfg.V) fail(KRUL_E_CONFIG, "token id out of vocabulary range");
}

int32_t* upload_tokens(Ctx& c, cudaStream_t s, const int32_t* t, int64_t n, DevBuf& buf) {
  int32_t* d = static_cast<int32_t*>(buf.ensure(size_t(std::max<int64_t>(n, 1)) * 4));
  if (n > 0) KB_CUDA(cudaMemcpyAsync(d, t, size_t(n) * 4, cudaMemcpyHostToDevice, s));
  return d;
}

static void prepare_capture(Ctx& c, cudaStream_t s, int64_t rows, int64_t W, int64_t first_q,
                            AttnArgs& a) {
  const Cfg& g = c.cfg;
  c.cap_rows = rows;
  c.cap_width = W;
  c.cap_mode = c.capture_probs;
  c.cap_first_q = first_q;
  c.cap_il = int64_t(c.cap_ifrac * double(W));
  const int64_t rl = int64_t(c.cap_rfrac * double(W));
  c.cap_rs = std::max(c.cap_il, W - rl);
  double* mass = static_cast<double*>(c.cap_mass.ensure(size_t(g.N) * g.H * rows * 8));
  a.mass = mass;
  a.mass_rows = rows;
  a.il = c.cap_il;
  a.rs = c.cap_rs;
  if (c.capture_probs == 1) {  // the reference's attention record, materialised
    const size_t n = size_t(g.N) * g.H * rows * W;
    float* p = static_cast<float*>(c.cap_probs.ensure(n * 4));
    KB_CUDA(cudaMemsetAsync(p, 0, n * 4, s));
    a.probs = p;
    a.ld_probs = W;
    a.probs_rows = rows;
  } else if (c.capture_probs == 2) {  // K2: Q rows + softmax statistics only
    a.q_save = c.cap_q.ensure(size_t(g.N) * rows * g.qd() * c.esz);
    a.stats = static_cast<float*>(c.cap_stats.ensure(size_t(g.N) * g.H * rows * 2 * 4));
    c.cap_stats_log2 = false;  // set per launch below (FA: log2 domain)
  }
  c.cap_valid = true;
}
static AttnArgs capture_for_layer(const Ctx& c, const AttnArgs& base, int l) {
  AttnArgs a = base;
  const int64_t per_layer = int64_t(c.cfg.H) * base.probs_rows * base.ld_probs;
  if (a.probs) a.probs += l * per_layer;
  if (a.mass) a.mass += int64_t(l) * c.cfg.H * base.mass_rows;
  if (a.stats) a.stats += int64_t(l) * c.cfg.H * base.mass_rows * 2;
  if (a.q_save) a.q_save = static_cast<char*>(a.q_save) + size_t(l) * base.mass_rows * c.cfg.qd() * c.esz;
  return a;
}

// New rows [pos0, pos0 + n) through every layer over the conversation's
// cache (fresh prefill when pos0 == 0; new-input prefill otherwise).
// Per-layer waits (restore events) are honoured when given.
void forward_rows(Ctx& c, cudaStream_t s, int set, Conv& conv, const int32_t* d_tok, int64_t n,
                  int64_t pos0, float* d_logits, const std::vector<cudaEvent_t>* waits,
                  const Mark* layer_done) {
  const Cfg& g = c.cfg;
  WS w = ws_get(c, set, n);
  AttnArgs cap{};
  prepare_capture(c, s, n, pos0 + n, pos0, cap);
  c.cap_conv = &conv;
  c.cap_conv_serial = conv.serial;
  launch_embed(c, s, d_tok, n, w.h);
  float* hin = w.h;
  float* hout = w.h2;
  for (int l = 0; l < g.N; ++l) {
    if (waits) {
      for (size_t k = 0; k < waits->size() / g.N; ++k)
        KB_CUDA(cudaStreamWaitEvent(s, (*waits)[k * g.N + size_t(l)], 0));
    }
    AttnArgs a = capture_for_layer(c, cap, l);
    layer_forward(c, s, w, conv, l, hin, n, pos0, n, hout, &a);
    if (layer_done) record_mark(layer_done[l], s);
    std::swap(hin, hout);
  }
  launch_logits(c, s, hin + (n - 1) * g.d, d_logits);
}

// Restore + new-input prefill with the pyramid recompute folded into the
// prefill's layer steps: layer l runs rows [new input | history prefix
// [0, p_l)] through one norm + QKV GEMM (two position segments in the fused
// RoPE/scatter epilogue), attends the recomputed rows over their own prefix,
// waits for layer l's loaded suffix, attends the new rows over the whole
// cache, and carries the new rows plus the p_{l+1} prefix rows the next layer
// needs through the O and FFN GEMMs. Each layer's weights stream from HBM
// once for both; the recompute rows fill the weight-bound small-M GEMMs.
void forward_fused(Ctx& c, cudaStream_t s, int set, Conv& conv, const int32_t* d_new, int64_t n,
                   int64_t L, const int32_t* d_hist, const std::vector<int64_t>& p, float* d_logits,
                   const Mark* loaded, const Mark* computed, const Mark* layer_done,
                   const Mark* compute_end) {
  const Cfg& g = c.cfg;
  const int64_t p0 = std::max<int64_t>(p[0], 0);
  WS w = ws_get(c, set, n + p0);
  AttnArgs cap{};
  prepare_capture(c, s, n, L + n, L, cap);
  c.cap_conv = &conv;
  c.cap_conv_serial = conv.serial;
  launch_embed(c, s, d_new, n, w.h);
  if (p0 > 0) launch_embed(c, s, d_hist, p0, w.h + n * g.d);
  float* hin = w.h;
  float* hout = w.h2;
  for (int l = 0; l < g.N; ++l) {
    const int64_t pl = p[size_t(l)], pn = l + 1 < g.N ? p[size_t(l + 1)] : 0;
    const cudaEvent_t wl = loaded[l].dep;
    FusedSeg fs;
    fs.n_new = n;
    fs.rec_out = pn;
    fs.waits = &wl;
    fs.n_waits = 1;
    fs.computed = &computed[l];
    AttnArgs a = capture_for_layer(c, cap, l);
    layer_forward(c, s, w, conv, l, hin, n + pl, L, n + pn, hout, &a, &fs);
    if (layer_done) record_mark(layer_done[l], s);
    std::swap(hin, hout);
  }
  if (compute_end) record_mark(*compute_end, s);
  launch_logits(c, s, hin + (n - 1) * g.d, d_logits);
}

void prefill(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, float* logits) {
  if (n <= 0) fail(KRUL_E_CONFIG, "prefill requires a non-empty input");
  if (n > conv.capacity) fail(KRUL_E_CONFIG, "prefill exceeds the conversation capacity");
  check_tokens(c, tok, n);
  if (!c.weights_ready) fail(KRUL_E_CONFIG, "weights not initialised");
  KB_CUDA(cudaSetDevice(c.device));
  cudaStream_t s = c.s_comp;
  int32_t* d_tok = upload_tokens(c, s, tok, n, c.ws_tok);
  float* d_logits = static_cast<float*>(c.ws_logits.ensure(size_t(c.cfg.V) * 4));
  forward_rows(c, s, 0, conv, d_tok, n, 0, d_logits, nullptr);
  conv.len = n;
  if (logits) KB_CUDA(cudaMemcpyAsync(logits, d_logits, size_t(c.cfg.V) * 4, cudaMemcpyDeviceToHost, s));
  KB_CUDA(cudaStreamSynchronize(s));
}

void prefill_new(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, float* logits) {
  if (n <= 0) fail(KRUL_E_RESTORATION_GAP, "prefill over preloaded history requires new input tokens");
  if (conv.len + n > conv.capacity) fail(KRUL_E_CONFIG, "prefill exceeds the conversation capacity");
  check_tokens(c, tok, n);
  KB_CUDA(cudaSetDevice(c.device));
  cudaStream_t s = c.s_comp;
  int32_t* d_tok = upload_tokens(c, s, tok, n, c.ws_tok);
  float* d_logits = static_cast<float*>(c.ws_logits.ensure(size_t(c.cfg.V) * 4));
  forward_rows(c, s, 0, conv, d_tok, n, conv.len, d_logits, nullptr);
  conv.len += n;
  if (logits) KB_CUDA(cudaMemcpyAsync(logits, d_logits, size_t(c.cfg.V) * 4, cudaMemcpyDeviceToHost, s));
  KB_CUDA(cudaStreamSynchronize(s));
}

// engine.cpp:406-446; attention rows of every layer are kept on device for
// the streaming estimator (K1 consumes them).
void decode_step(Ctx& c, Conv& conv, int32_t tok, float* logits) {
  const Cfg& g = c.cfg;
  if (tok < 0 || tok >= g.V) fail(KRUL_E_CONFIG, "token id out of vocabulary range");
  if (conv.len + 1 > conv.capacity) fail(KRUL_E_STATE_CORRUPTION, "conversation capacity exceeded");
  KB_CUDA(cudaSetDevice(c.device));
  cudaStream_t s = c.s_comp;
  const int64_t pos = conv.len, W = pos + 1;
  int32_t* d_tok = upload_tokens(c, s, &tok, 1, c.ws_tok);
  float* d_logits = static_cast<float*>(c.ws_logits.ensure(size_t(g.V) * 4));
  const int64_t pitch = (W + 3) / 4 * 4;  // 16-byte rows for the fold's vector loads
  float* rows = static_cast<float*>(c.dec_rows.ensure(size_t(g.N) * g.H * pitch * 4));
  WS w = ws_get(c, 0, 1);
  launch_embed(c, s, d_tok, 1, w.h);
  float* hin = w.h;
  float* hout = w.h2;
  for (int l = 0; l < g.N; ++l) {
    AttnArgs a{};
    a.probs = rows + int64_t(l) * g.H * pitch;
    a.ld_probs = pitch;
    a.probs_rows = 1;
    layer_forward(c, s, w, conv, l, hin, 1, pos, 1, hout, &a);
    std::swap(hin, hout);
  }
  launch_logits(c, s, hin, d_logits);
  conv.len = W;
  c.dec_width = W;
  c.dec_pitch = pitch;
  c.dec_valid = true;
  if (logits) KB_CUDA(cudaMemcpyAsync(logits, d_logits, size_t(g.V) * 4, cudaMemcpyDeviceToHost, s));
  KB_CUDA(cudaStreamSynchronize(s));
}

// engine.cpp:448-489, enqueued on `s`; records ev[l] after layer l's K/V.
void enqueue_partial(Ctx& c, cudaStream_t s, Conv& conv, const int32_t* d_tok,
                     const std::vector<int64_t>& p, bool full_last, const Mark* ev) {
  const Cfg& g = c.cfg;
  WS w = ws_get(c, 0, p[0]);
  launch_embed(c, s, d_tok, p[0], w.h);
  float* hin = w.h;
  float* hout = w.h2;
  for (int l = 0; l < g.N; ++l) {
    const int64_t pre = p[size_t(l)];
    const int64_t out = l + 1 < g.N ? p[size_t(l + 1)] : (full_last ? pre : 0);
    if (pre > 0) {
      layer_forward(c, s, w, conv, l, hin, pre, 0, out, hout, nullptr);
      std::swap(hin, hout);
    }
    if (ev) record_mark(ev[l], s);
  }
}

void check_plan_shape(const Ctx& c, int64_t n, const int64_t* p, int np) {
  if (np != c.cfg.N) fail(KRUL_E_PLAN_INVALID, "plan layer count mismatch");
  for (int l = 0; l < np; ++l) {
    if (p[l] < 0 || p[l] > n) fail(KRUL_E_PLAN_INVALID, "recompute prefix exceeds the token history");
    if (l > 0 && p[l] > p[l - 1]) fail(KRUL_E_PLAN_INVALID, "recompute_len must be non-increasing with depth");
  }
}

void partial_recompute(Ctx& c, Conv& conv, const int32_t* tok, int64_t n, const int64_t* p,
                       int np) {
  check_plan_shape(c, n, p, np);
  check_tokens(c, tok, n);
  if (n > conv.capacity) fail(KRUL_E_CONFIG, "history exceeds the conversation capacity");
  KB_CUDA(cudaSetDevice(c.device));
  cudaStream_t s = c.s_comp;
  int32_t* d_tok = upload_tokens(c, s, tok, std::max<int64_t>(p[0], 0), c.ws_tok);
  std::vector<int64_t> pv(p, p + np);
  if (pv[0] > 0) enqueue_partial(c, s, conv, d_tok, pv, true, nullptr);
  conv.len = pv[0];
  KB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace kb
