// host_ctx.cpp — device context, weights, paged KV pool, conversations.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "host.hpp"

namespace kb {

void fail(int code, const std::string& msg) { throw Error(code, msg); }

std::atomic<uint64_t> g_launches{0};
// Off by default: measured on the Llama-3-8B restore, the early-launched
// dependents' resident CTAs hold SMs the concurrent restore streams need
// (TTFT 11.23 -> 11.62 ms) although each chain alone runs ~6% faster
// (KRUL_PDL=1 to enable).
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("KRUL_PDL");
    return v && v[0] == '1';
  }();
  return on;
}
std::atomic<uint64_t> g_buf_gen{0};

cudaEvent_t KTime::ev() {
  if (next == pool.size()) {
    cudaEvent_t e;
    KB_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[next++];
}
KTime::~KTime() {
  for (auto e : pool) cudaEventDestroy(e);
}
cudaError_t record_timing(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t r = cudaStreamIsCapturing(s, &cs);
  if (r != cudaSuccess) return r;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}
void record_mark(const Mark& m, cudaStream_t s) {
  // timing node first: a join on `dep` then also covers it under capture
  if (m.tim) KB_CUDA(record_timing(m.tim, s));
  if (m.dep) KB_CUDA(cudaEventRecord(m.dep, s));
}
cudaEvent_t kt_begin(const Ctx& c, cudaStream_t s) {
  if (!c.kt.on) return nullptr;
  cudaEvent_t a = c.kt.ev();
  KB_CUDA(record_timing(a, s));
  return a;
}
void kt_end(const Ctx& c, cudaStream_t s, cudaEvent_t a, int tag, double flops, double bytes) {
  if (!a) return;
  cudaEvent_t b = c.kt.ev();
  KB_CUDA(record_timing(b, s));
  c.kt.recs.push_back({tag, flops, bytes, a, b});
}

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}
void* DevBuf::ensure(size_t n) {
  if (n > bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    KB_CUDA(cudaMalloc(&p, n));
    bytes = n;
    g_buf_gen.fetch_add(1);
  }
  return p;
}
void PinnedBuf::pin() {
  if (!p || !pageable || registered) return;
  KB_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  registered = true;
}
PinnedBuf::~PinnedBuf() {
  if (p) {
    if (registered) cudaHostUnregister(p);
    if (pageable)
      std::free(p);
    else
      cudaFreeHost(p);
  }
}
void* PinnedBuf::ensure(size_t n) {
  if (n > bytes) {
    if (p) {
      if (registered) cudaHostUnregister(p);
      registered = false;
      if (pageable)
        std::free(p);
      else
        cudaFreeHost(p);
    }
    p = nullptr;
    bytes = 0;
    if (pageable) {
      p = std::malloc(n);
      if (!p) throw std::bad_alloc();
    } else {
      KB_CUDA(cudaMallocHost(&p, n));
    }
    bytes = n;
    g_buf_gen.fetch_add(1);
  }
  return p;
}

// engine.cpp:10-25 (+ GQA / ffn_kind checks of the extensions).
Cfg cfg_from_desc(const krul_model_desc& d) {
  Cfg c;
  c.N = d.n_layers;
  c.H = d.n_heads;
  c.Hkv = d.n_kv_heads > 0 ? d.n_kv_heads : d.n_heads;
  c.hd = d.head_dim;
  c.d = d.d_model;
  c.V = d.vocab_size;
  c.ffn_mult = d.ffn_mult;
  c.ffn_kind = d.ffn_kind;
  c.seed = d.seed;
  c.theta = d.rope_theta > 0 ? d.rope_theta : 1e4;
  c.dtype = d.dtype;
  c.max_tokens = d.max_tokens;
  if (c.N < 2) fail(KRUL_E_CONFIG, "n_layers must be >= 2");
  if (c.H < 1) fail(KRUL_E_CONFIG, "n_heads must be >= 1");
  if (c.hd < 1) fail(KRUL_E_CONFIG, "head_dim must be >= 1");
  if (c.d != c.H * c.hd) fail(KRUL_E_CONFIG, "d_model must equal n_heads * head_dim");
  if (c.V < 2) fail(KRUL_E_CONFIG, "vocab_size must be >= 2");
  c.F = int(std::lround(c.ffn_mult * float(c.d)));
  if (!(c.ffn_mult > 0.f) || c.F < 1) fail(KRUL_E_CONFIG, "ffn_mult must yield a positive hidden width");
  if (c.H % c.Hkv != 0) fail(KRUL_E_CONFIG, "n_heads must be a multiple of n_kv_heads");
  if (c.ffn_kind != KRUL_FFN_TANH && c.ffn_kind != KRUL_FFN_SWIGLU) fail(KRUL_E_CONFIG, "unknown ffn_kind");
  if (c.dtype != KRUL_F32 && c.dtype != KRUL_BF16) fail(KRUL_E_CONFIG, "unknown dtype");
  if (c.max_tokens < 1) fail(KRUL_E_CONFIG, "max_tokens must be >= 1");
  return c;
}

static uint64_t fnv(const void* p, size_t n, uint64_t h) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// ModelConfig::hash (engine.cpp:27-36): FNV-1a over the fields in order;
// extension fields fold in only when they leave the reference architecture.
uint64_t config_hash(const Cfg& c) {
  uint64_t h = 0xcbf29ce484222325ull;
  h = fnv(&c.N, sizeof c.N, h);
  h = fnv(&c.H, sizeof c.H, h);
  h = fnv(&c.hd, sizeof c.hd, h);
  h = fnv(&c.d, sizeof c.d, h);
  h = fnv(&c.V, sizeof c.V, h);
  h = fnv(&c.ffn_mult, sizeof c.ffn_mult, h);
  h = fnv(&c.seed, sizeof c.seed, h);
  if (c.Hkv != c.H || c.ffn_kind != 0 || c.theta != 1e4) {
    h = fnv(&c.Hkv, sizeof c.Hkv, h);
    h = fnv(&c.ffn_kind, sizeof c.ffn_kind, h);
    h = fnv(&c.theta, sizeof c.theta, h);
  }
  return h;
}

void Ctx::drop_graph() {
  if (tl_pending) {  // the timeline's events die with the graph: read them now
    try {
      restore_timeline(*this);
    } catch (...) {
      tl_pending = false;
    }
  }
  if (rg.exec) cudaGraphExecDestroy(rg.exec);
  for (auto& m : rg.ev) {
    if (m.dep) cudaEventDestroy(m.dep);
    if (m.tim) cudaEventDestroy(m.tim);
  }
  rg = RestoreGraph{};
}

Ctx::BatchGraph::~BatchGraph() {
  if (exec) cudaGraphExecDestroy(exec);
  if (t0) cudaEventDestroy(t0);
  if (t1) cudaEventDestroy(t1);
  for (auto& m : ev)
    if (m.dep) cudaEventDestroy(m.dep);
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  drop_graph();
  for (auto* b : bgraphs) delete b;
  for (int i = 0; i < 2; ++i) {
    for (auto e : {b_dec[i], b_comp[i], b_new[i], b_h2d[i]})
      if (e) cudaEventDestroy(e);
    if (b_launch[i]) cudaStreamDestroy(b_launch[i]);
  }
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (auto s : {s_comp, s_load, s_new, s_est, s_exp})
    if (s) cudaStreamDestroy(s);
}

cudaEvent_t Ctx::event() {
  if (ev_next == ev_pool.size()) {
    cudaEvent_t e;
    KB_CUDA(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_next++];
}

Conv::~Conv() {
  if (ctx) {
    if (ctx->rg.conv_serial == serial) ctx->drop_graph();  // its kernels hold d_pt
    auto& cv = ctx->convs;
    cv.erase(std::remove(cv.begin(), cv.end(), this), cv.end());
    if (ctx->cap_conv == this) ctx->cap_conv = nullptr;
    for (int p : pages) ctx->free_pages.push_back(p);
  }
  if (d_pt) cudaFree(d_pt);
}

}  // namespace kb
