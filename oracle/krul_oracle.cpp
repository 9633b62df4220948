// krul_oracle.cpp — CPU restatement of the Krul reference hot path.
// TEST INFRASTRUCTURE ONLY (see krul_oracle.hpp header comment).
//
// Every function cites the reference file:line it restates, abbreviated
// `proj/...` = /root/reference/proj/... .
#include "krul_oracle.hpp"

#include <algorithm>
#include <array>
#include <immintrin.h>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <map>
#include <thread>
#include <tuple>

namespace kro {

void fail(Status c, const std::string& msg) { throw Error(c, msg); }

// proj/src/common.cpp:8-16 — FNV-1a 64.
uint64_t fnv1a64(const void* p, size_t n, uint64_t h) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

// proj/src/common.cpp:20-42 — reflected CRC-32 (poly 0xEDB88320).
uint32_t crc32(const void* p, size_t n, uint32_t crc) {
  static const std::array<uint32_t, 256> tab = [] {
    std::array<uint32_t, 256> t{};
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xedb88320u : 0u);
      t[i] = c;
    }
    return t;
  }();
  const unsigned char* b = static_cast<const unsigned char*>(p);
  uint32_t c = ~crc;
  for (size_t i = 0; i < n; ++i) c = tab[(c ^ b[i]) & 0xffu] ^ (c >> 8);
  return ~c;
}

// ===========================================================================
// engine
// ===========================================================================

// proj/src/engine.cpp:10-12
int ModelConfig::ffn_hidden() const {
  return static_cast<int>(std::lround(ffn_mult * static_cast<float>(d_model)));
}

// proj/src/engine.cpp:14-25 (+ GQA / ffn_kind extension checks)
void ModelConfig::validate() const {
  if (n_layers < 2) fail(kConfig, "n_layers must be >= 2");
  if (n_heads < 1) fail(kConfig, "n_heads must be >= 1");
  if (head_dim < 1) fail(kConfig, "head_dim must be >= 1");
  if (d_model != n_heads * head_dim)
    fail(kConfig, "d_model must equal n_heads * head_dim");
  if (vocab < 2) fail(kConfig, "vocab_size must be >= 2");
  if (!(ffn_mult > 0.0f) || ffn_hidden() < 1)
    fail(kConfig, "ffn_mult must yield a positive hidden width");
  if (kv_heads() < 1 || n_heads % kv_heads() != 0)
    fail(kConfig, "n_heads must be a multiple of n_kv_heads");
  if (ffn_kind != 0 && ffn_kind != 1) fail(kConfig, "unknown ffn_kind");
}

// proj/src/engine.cpp:27-36. Extension fields are folded in only when they
// differ from the reference architecture so reference hashes are unchanged.
uint64_t ModelConfig::hash() const {
  uint64_t h = fnv1a64(&n_layers, sizeof n_layers);
  h = fnv1a64(&n_heads, sizeof n_heads, h);
  h = fnv1a64(&head_dim, sizeof head_dim, h);
  h = fnv1a64(&d_model, sizeof d_model, h);
  h = fnv1a64(&vocab, sizeof vocab, h);
  h = fnv1a64(&ffn_mult, sizeof ffn_mult, h);
  h = fnv1a64(&seed, sizeof seed, h);
  if (kv_heads() != n_heads || ffn_kind != 0 || rope_theta != 10000.0) {
    int kvh = kv_heads();
    h = fnv1a64(&kvh, sizeof kvh, h);
    h = fnv1a64(&ffn_kind, sizeof ffn_kind, h);
    h = fnv1a64(&rope_theta, sizeof rope_theta, h);
  }
  return h;
}

namespace {

void fill(Mat& m, Uniform& u, float bound) {  // engine.cpp:99-105 (row-major draw)
  for (auto& x : m.v) x = u.next(-bound, bound);
}
void fill(std::vector<float>& v, Uniform& u, float bound) {
  for (auto& x : v) x = u.next(-bound, bound);
}

// C[M x N] = A[M x K] * B[K x N]. Every element is the left-to-right sum
// c = (((0 + a0 b0) + a1 b1) + ...) with separately rounded products (no FMA:
// -ffp-contract=off), exactly the order of the naive i-k-j loop; the blocking
// below only changes which elements are in flight (6 rows x 16 columns held
// in AVX2 registers across the whole k loop, a 16-column strip of B reused
// from cache by every row block), not any element's arithmetic.
Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  const int64_t M = A.r, K = A.c, N = B.c;
  constexpr int64_t MR = 6, NR = 16;
  const int64_t nstrips = (N + NR - 1) / NR;
#pragma omp parallel
  {
  std::vector<float> bp(size_t(K) * NR);  // the strip of B packed contiguously (TLB / prefetch)
#pragma omp for schedule(dynamic, 1)
  for (int64_t js = 0; js < nstrips; ++js) {
    const int64_t j0 = js * NR;
    const int64_t nj = std::min<int64_t>(NR, N - j0);
    if (nj == NR)
      for (int64_t k = 0; k < K; ++k) std::memcpy(bp.data() + k * NR, B.row(k) + j0, sizeof(float) * NR);
    for (int64_t i0 = 0; i0 < M; i0 += MR) {
      const int64_t mi = std::min<int64_t>(MR, M - i0);
      if (nj == NR && mi == MR) {
        __m256 c[MR][2];
        for (int r = 0; r < MR; ++r) c[r][0] = c[r][1] = _mm256_setzero_ps();
        const float* a = A.row(i0);
        for (int64_t k = 0; k < K; ++k) {
          const float* b = bp.data() + k * NR;
          const __m256 b0 = _mm256_loadu_ps(b), b1 = _mm256_loadu_ps(b + 8);
          for (int r = 0; r < MR; ++r) {
            const __m256 s = _mm256_set1_ps(a[r * K + k]);
            c[r][0] = _mm256_add_ps(c[r][0], _mm256_mul_ps(s, b0));
            c[r][1] = _mm256_add_ps(c[r][1], _mm256_mul_ps(s, b1));
          }
        }
        for (int r = 0; r < MR; ++r) {
          _mm256_storeu_ps(C.row(i0 + r) + j0, c[r][0]);
          _mm256_storeu_ps(C.row(i0 + r) + j0 + 8, c[r][1]);
        }
      } else {  // ragged edge: the plain loop, same order
        for (int64_t i = i0; i < i0 + mi; ++i) {
          float* c = C.row(i) + j0;
          const float* a = A.row(i);
          for (int64_t k = 0; k < K; ++k) {
            const float s = a[k];
            const float* b = B.row(k) + j0;
            for (int64_t j = 0; j < nj; ++j) c[j] += s * b[j];
          }
        }
      }
    }
  }
  }
  return C;
}

Mat top_rows(const Mat& m, int64_t n) {
  Mat o(n, m.c);
  std::memcpy(o.v.data(), m.v.data(), sizeof(float) * size_t(n * m.c));
  return o;
}

// engine.cpp:117-124 — weightless RMSNorm, eps 1e-6.
Mat rmsnorm(const Mat& x) {
  Mat o(x.r, x.c);
  for (int64_t i = 0; i < x.r; ++i) {
    float ss = 0.f;
    for (int64_t j = 0; j < x.c; ++j) ss += x.at(i, j) * x.at(i, j);
    const float inv = std::sqrt(ss / static_cast<float>(x.c) + 1e-6f);
    for (int64_t j = 0; j < x.c; ++j) o.at(i, j) = x.at(i, j) / inv;
  }
  return o;
}

// engine.cpp:128-143 — interleaved RoPE, angles in double, cast to float.
// `m` holds `heads` heads of width hd side by side.
void rope(Mat& m, int64_t pos0, int hd, int heads, double theta) {
  const int half = hd / 2;
  for (int64_t r = 0; r < m.r; ++r) {
    const double pos = static_cast<double>(pos0 + r);
    for (int i = 0; i < half; ++i) {
      const double ang = pos * std::pow(theta, -2.0 * i / static_cast<double>(hd));
      const float c = static_cast<float>(std::cos(ang));
      const float s = static_cast<float>(std::sin(ang));
      for (int h = 0; h < heads; ++h) {
        float* x = m.row(r) + h * hd;
        const float x0 = x[2 * i], x1 = x[2 * i + 1];
        x[2 * i] = x0 * c - x1 * s;
        x[2 * i + 1] = x0 * s + x1 * c;
      }
    }
  }
}

void grow(KVLayer& kv, int64_t total, int hd) {
  for (auto* vec : {&kv.k, &kv.v})
    for (auto& m : *vec) {
      Mat g(total, hd);
      const int64_t keep = std::min(m.r, total);
      std::memcpy(g.v.data(), m.v.data(), sizeof(float) * size_t(keep * hd));
      m = std::move(g);
    }
}

// engine.cpp:150-193 — one layer over block rows [pos0, pos0+rows); kv must
// cover [0, pos0) on entry and is grown with the block's K/V; attention and
// FFN outputs are produced for the leading out_rows rows only.
Mat layer_forward(const ModelConfig& cfg, const LayerW& w, const Mat& h_in,
                  int64_t pos0, KVLayer& kv, int64_t out_rows,
                  std::vector<Mat>* capture) {
  const int64_t rows = h_in.r;
  const int hd = cfg.head_dim, H = cfg.n_heads, Hkv = cfg.kv_heads();
  const int64_t total = pos0 + rows;
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  const Mat xn = rmsnorm(h_in);

  Mat kall = matmul(xn, w.wk), vall = matmul(xn, w.wv);
  rope(kall, pos0, hd, Hkv, cfg.rope_theta);
  grow(kv, total, hd);
  for (int g = 0; g < Hkv; ++g)
    for (int64_t r = 0; r < rows; ++r) {
      std::memcpy(kv.k[size_t(g)].row(pos0 + r), kall.row(r) + g * hd, sizeof(float) * hd);
      std::memcpy(kv.v[size_t(g)].row(pos0 + r), vall.row(r) + g * hd, sizeof(float) * hd);
    }
  if (out_rows == 0) return Mat(0, cfg.d_model);

  Mat q = matmul(top_rows(xn, out_rows), w.wq);
  rope(q, pos0, hd, H, cfg.rope_theta);
  Mat ctx(out_rows, int64_t(H) * hd);
  const int grp = H / Hkv;
  std::vector<Mat> kt(static_cast<size_t>(Hkv));  // K^T [hd][total] per kv head: 8 keys per vector below
  for (int g = 0; g < Hkv; ++g) {
    const Mat& K = kv.k[size_t(g)];
    kt[size_t(g)] = Mat(hd, total);
    for (int64_t c = 0; c < total; ++c)
      for (int t = 0; t < hd; ++t) kt[size_t(g)].at(t, c) = K.at(c, t);
  }
  for (int h = 0; h < H; ++h) {
    const Mat& KT = kt[size_t(h / grp)];
    const Mat& V = kv.v[size_t(h / grp)];
    Mat probs(out_rows, total);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < out_rows; ++r) {
      const int64_t width = pos0 + r + 1;
      const float* qr = q.row(r) + h * hd;
      float* pr = probs.row(r);
      float mx = -std::numeric_limits<float>::infinity();
      // dot(q, k_c) = (((0 + q0 k0) + q1 k1) + ...) per key, 8 keys per lane set
      int64_t c = 0;
      for (; c + 8 <= width; c += 8) {
        __m256 dot = _mm256_setzero_ps();
        for (int t = 0; t < hd; ++t)
          dot = _mm256_add_ps(dot, _mm256_mul_ps(_mm256_set1_ps(qr[t]), _mm256_loadu_ps(KT.row(t) + c)));
        _mm256_storeu_ps(pr + c, _mm256_mul_ps(dot, _mm256_set1_ps(scale)));
      }
      for (; c < width; ++c) {
        float dot = 0.f;
        for (int t = 0; t < hd; ++t) dot += qr[t] * KT.at(t, c);
        pr[c] = dot * scale;
      }
      for (c = 0; c < width; ++c) mx = std::max(mx, pr[c]);
      float sum = 0.f;
      for (int64_t c = 0; c < width; ++c) {
        pr[c] = std::exp(pr[c] - mx);
        sum += pr[c];
      }
      for (int64_t c = 0; c < width; ++c) pr[c] = pr[c] / sum;
      float* cr = ctx.row(r) + h * hd;
      for (int64_t c = 0; c < width; ++c) {
        const float p = pr[c];
        const float* vr = V.row(c);
        for (int t = 0; t < hd; ++t) cr[t] += p * vr[t];
      }
    }
    if (capture) (*capture)[size_t(h)] = std::move(probs);
  }

  Mat hmid = matmul(ctx, w.wo);
  for (int64_t r = 0; r < out_rows; ++r)
    for (int64_t j = 0; j < hmid.c; ++j) hmid.at(r, j) += h_in.at(r, j);
  Mat out = hmid;
  if (cfg.ffn_kind == 0) {  // engine.cpp:191-192
    Mat act = matmul(hmid, w.w1);
    for (int64_t r = 0; r < act.r; ++r)
      for (int64_t j = 0; j < act.c; ++j)
        act.at(r, j) = std::tanh(act.at(r, j) + w.b1[size_t(j)]);
    Mat y = matmul(act, w.w2);
    for (int64_t r = 0; r < out.r; ++r)
      for (int64_t j = 0; j < out.c; ++j)
        out.at(r, j) += y.at(r, j) + w.b2[size_t(j)];
  } else {  // SwiGLU extension, Llama's FFN block: h_mid + (silu(n Wg) * (n Wu)) W2,
            // n = rmsnorm(h_mid) (gain-less like engine.cpp:117-124); without the
            // norm the quadratic gate makes the residual grow doubly exponentially
    const Mat hn = rmsnorm(hmid);
    Mat g = matmul(hn, w.w1), u = matmul(hn, w.wu);
    for (size_t i = 0; i < g.v.size(); ++i) {
      const float x = g.v[i];
      g.v[i] = x / (1.0f + std::exp(-x)) * u.v[i];
    }
    Mat y = matmul(g, w.w2);
    for (size_t i = 0; i < out.v.size(); ++i) out.v[i] += y.v[i];
  }
  return out;
}

Mat embed_rows(const Model& m, const std::vector<int32_t>& t, int64_t b,
               int64_t e) {  // engine.cpp:195-207
  Mat h(e - b, m.cfg.d_model);
  for (int64_t i = b; i < e; ++i) {
    const int32_t id = t[size_t(i)];
    if (id < 0 || id >= m.cfg.vocab) fail(kConfig, "token id out of vocabulary range");
    std::memcpy(h.row(i - b), m.embed.row(id), sizeof(float) * size_t(m.cfg.d_model));
  }
  return h;
}

std::vector<KVLayer> empty_kv(const ModelConfig& cfg) {  // engine.cpp:209-219
  std::vector<KVLayer> kv(size_t(cfg.n_layers));
  for (auto& l : kv) {
    l.k.assign(size_t(cfg.kv_heads()), Mat(0, cfg.head_dim));
    l.v.assign(size_t(cfg.kv_heads()), Mat(0, cfg.head_dim));
  }
  return kv;
}

std::vector<float> logits_of(const Model& m, const float* h) {
  // out[j] = sum_k h[k] u[k][j], k ascending per element; column chunks in parallel
  const int64_t d = m.cfg.d_model, V = m.cfg.vocab;
  std::vector<float> out(size_t(V), 0.f);
  constexpr int64_t CH = 2048;
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < V; j0 += CH) {
    const int64_t j1 = std::min(V, j0 + CH);
    for (int64_t k = 0; k < d; ++k) {
      const float s = h[k];
      const float* u = m.unembed.row(k);
      for (int64_t j = j0; j < j1; ++j) out[size_t(j)] += s * u[j];
    }
  }
  return out;
}

// engine.cpp:228-280 — prefix lengths implied by preloaded suffixes.
std::vector<int64_t> preload_layout(const ModelConfig& cfg,
                                    const std::vector<KVLayer>& pre,
                                    int64_t n_tok, int64_t* hist) {
  if (int(pre.size()) != cfg.n_layers)
    fail(kRestorationGap, "preloaded KV must cover every layer");
  int64_t end = -1;
  for (const auto& l : pre) {
    if (l.span.empty()) continue;
    if (end == -1) end = l.span.end;
    else if (l.span.end != end)
      fail(kRestorationGap, "preloaded suffixes end at different positions");
  }
  *hist = end == -1 ? 0 : end;
  if (*hist > n_tok) fail(kRestorationGap, "preloaded span extends past the token history");
  std::vector<int64_t> pl(size_t(cfg.n_layers));
  for (int l = 0; l < cfg.n_layers; ++l) {
    const KVLayer& x = pre[size_t(l)];
    const int64_t start = x.span.empty() ? *hist : x.span.start;
    if (start < 0 || start > *hist) fail(kRestorationGap, "preloaded span start out of range");
    if (!x.span.empty()) {
      if (int(x.k.size()) != cfg.kv_heads() || int(x.v.size()) != cfg.kv_heads())
        fail(kStateCorruption, "preloaded head count mismatch");
      for (int g = 0; g < cfg.kv_heads(); ++g)
        if (x.k[size_t(g)].r != x.span.len() || x.v[size_t(g)].r != x.span.len() ||
            x.k[size_t(g)].c != cfg.head_dim)
          fail(kStateCorruption, "preloaded tensor shape mismatch");
    }
    pl[size_t(l)] = start;
    if (l > 0 && start > pl[size_t(l - 1)])
      fail(kRestorationGap, "preloaded span not contiguous with the computable prefix");
  }
  return pl;
}

}  // namespace

// engine.cpp:361-395 — one UniformStream in fixed draw order.
Model build_model(const ModelConfig& cfg) {
  cfg.validate();
  Model m;
  m.cfg = cfg;
  Uniform u(cfg.seed);
  const float bound = 1.0f / std::sqrt(static_cast<float>(cfg.d_model));
  const int64_t d = cfg.d_model, F = cfg.ffn_hidden();
  const int64_t qd = int64_t(cfg.n_heads) * cfg.head_dim;
  const int64_t kvd = int64_t(cfg.kv_heads()) * cfg.head_dim;
  m.embed = Mat(cfg.vocab, d);
  fill(m.embed, u, bound);
  m.layers.resize(size_t(cfg.n_layers));
  for (auto& w : m.layers) {
    w.wq = Mat(d, qd); w.wk = Mat(d, kvd); w.wv = Mat(d, kvd); w.wo = Mat(qd, d);
    w.w1 = Mat(d, F); w.w2 = Mat(F, d);
    fill(w.wq, u, bound); fill(w.wk, u, bound); fill(w.wv, u, bound); fill(w.wo, u, bound);
    if (cfg.ffn_kind == 0) {
      w.b1.assign(size_t(F), 0.f); w.b2.assign(size_t(d), 0.f);
      fill(w.w1, u, bound); fill(w.b1, u, bound); fill(w.w2, u, bound); fill(w.b2, u, bound);
    } else {
      w.wu = Mat(d, F);
      fill(w.w1, u, bound); fill(w.wu, u, bound); fill(w.w2, u, bound);
    }
  }
  m.unembed = Mat(d, cfg.vocab);
  fill(m.unembed, u, bound);
  return m;
}

// engine.cpp:282-340 (+ prefill() wrappers :397-404)
PrefillOut prefill(const Model& m, const std::vector<int32_t>& toks,
                   const std::vector<KVLayer>* pre, bool capture) {
  const ModelConfig& cfg = m.cfg;
  if (toks.empty()) fail(kConfig, "prefill requires a non-empty input");
  const int64_t n = int64_t(toks.size());
  std::vector<int64_t> pl(size_t(cfg.n_layers), 0);
  int64_t hist = 0;
  if (pre) {
    pl = preload_layout(cfg, *pre, n, &hist);
    if (hist == n && hist > 0)
      fail(kRestorationGap, "prefill over preloaded history requires new input tokens");
  }
  PrefillOut out;
  out.kv = empty_kv(cfg);
  out.attn.first_q = hist;
  out.attn.layers.resize(size_t(cfg.n_layers));
  Mat h_pre = embed_rows(m, toks, 0, pl[0]);
  Mat h_new = embed_rows(m, toks, hist, n);
  for (int l = 0; l < cfg.n_layers; ++l) {
    const LayerW& w = m.layers[size_t(l)];
    KVLayer& kv = out.kv[size_t(l)];
    const int64_t pre_len = pl[size_t(l)];
    const int64_t next = l + 1 < cfg.n_layers ? pl[size_t(l + 1)] : 0;
    if (pre_len > 0) h_pre = layer_forward(cfg, w, h_pre, 0, kv, next, nullptr);
    if (pre && hist > pre_len) {
      const KVLayer& suf = (*pre)[size_t(l)];
      grow(kv, hist, cfg.head_dim);
      for (int g = 0; g < cfg.kv_heads(); ++g) {
        std::memcpy(kv.k[size_t(g)].row(pre_len), suf.k[size_t(g)].v.data(),
                    sizeof(float) * size_t((hist - pre_len) * cfg.head_dim));
        std::memcpy(kv.v[size_t(g)].row(pre_len), suf.v[size_t(g)].v.data(),
                    sizeof(float) * size_t((hist - pre_len) * cfg.head_dim));
      }
    }
    std::vector<Mat> cap(size_t(cfg.n_heads));
    h_new = layer_forward(cfg, w, h_new, hist, kv, n - hist, &cap);
    if (capture) out.attn.layers[size_t(l)].prefill = std::move(cap);
    kv.span = {0, n};
  }
  out.logits = logits_of(m, h_new.row(h_new.r - 1));
  return out;
}

// engine.cpp:406-446
DecodeOut decode_step(const Model& m, std::vector<KVLayer>& kv, int32_t tok) {
  const ModelConfig& cfg = m.cfg;
  if (int(kv.size()) != cfg.n_layers) fail(kStateCorruption, "cache layer count mismatch");
  const Span sp = kv[0].span;
  if (sp.start != 0) fail(kStateCorruption, "decode requires caches anchored at position 0");
  for (const auto& l : kv) {
    if (!(l.span == sp)) fail(kStateCorruption, "ragged kv spans across layers");
    if (int(l.k.size()) != cfg.kv_heads()) fail(kStateCorruption, "cache head count mismatch");
  }
  if (tok < 0 || tok >= cfg.vocab) fail(kConfig, "token id out of vocabulary range");
  const int64_t pos = sp.end;
  Mat h(1, cfg.d_model);
  std::memcpy(h.row(0), m.embed.row(tok), sizeof(float) * size_t(cfg.d_model));
  DecodeOut out;
  out.rows.resize(kv.size());
  for (int l = 0; l < cfg.n_layers; ++l) {
    std::vector<Mat> cap(size_t(cfg.n_heads));
    h = layer_forward(cfg, m.layers[size_t(l)], h, pos, kv[size_t(l)], 1, &cap);
    Mat rows(cfg.n_heads, pos + 1);
    for (int hh = 0; hh < cfg.n_heads; ++hh)
      std::memcpy(rows.row(hh), cap[size_t(hh)].row(0), sizeof(float) * size_t(pos + 1));
    out.rows[size_t(l)] = std::move(rows);
    kv[size_t(l)].span = {0, pos + 1};
  }
  out.logits = logits_of(m, h.row(0));
  return out;
}

// engine.cpp:448-489 — pyramid prefix recompute.
PartialOut partial_prefix_recompute(const Model& m,
                                    const std::vector<int32_t>& toks,
                                    const std::vector<int64_t>& p) {
  const ModelConfig& cfg = m.cfg;
  if (int(p.size()) != cfg.n_layers) fail(kPlanInvalid, "plan layer count mismatch");
  const int64_t n = int64_t(toks.size());
  for (size_t l = 0; l < p.size(); ++l) {
    if (p[l] < 0 || p[l] > n) fail(kPlanInvalid, "recompute prefix exceeds the token history");
    if (l > 0 && p[l] > p[l - 1]) fail(kPlanInvalid, "recompute_len must be non-increasing with depth");
  }
  PartialOut out;
  out.kv = empty_kv(cfg);
  Mat h = embed_rows(m, toks, 0, p[0]);
  for (int l = 0; l < cfg.n_layers; ++l) {
    const int64_t pre = p[size_t(l)];
    const int64_t out_rows = l + 1 < cfg.n_layers ? p[size_t(l + 1)] : pre;
    if (pre > 0) h = layer_forward(cfg, m.layers[size_t(l)], h, 0, out.kv[size_t(l)], out_rows, nullptr);
    out.kv[size_t(l)].span = {0, pre};
  }
  if (p.back() > 0) {
    out.has_final = true;
    out.final_hidden = std::move(h);
  }
  return out;
}

// ===========================================================================
// analysis
// ===========================================================================

// proj/src/analysis.cpp:20-63
ClassReport classify_layers(const AttnRecord& rec, double gamma,
                            double ifrac, double rfrac) {
  if (!(gamma > 0.0) || gamma > 1.0) fail(kConfig, "gamma must lie in (0, 1]");
  if (!(ifrac > 0.0) || !(rfrac > 0.0) || ifrac + rfrac >= 1.0)
    fail(kConfig, "region fractions must be positive and sum below 1");
  const int64_t W = rec.width(), R = rec.rows();
  if (R == 0) fail(kClassification, "classification requires prefill attention");
  const int64_t il = static_cast<int64_t>(ifrac * static_cast<double>(W));
  const int64_t rl = static_cast<int64_t>(rfrac * static_cast<double>(W));
  if (il < 1 || rl < 1) fail(kClassification, "sequence too short to form both attention regions");
  const int64_t rs = std::max(il, W - rl);
  ClassReport rep;
  rep.avg.resize(rec.layers.size());
  for (size_t l = 0; l < rec.layers.size(); ++l) {
    const auto& heads = rec.layers[l].prefill;
    double mass = 0.0;
    for (const Mat& hm : heads) {
      if (hm.r != R || hm.c != W) fail(kStateCorruption, "ragged prefill attention across heads");
      double a = 0.0, b = 0.0;
      for (int64_t r = 0; r < R; ++r) {
        for (int64_t c = 0; c < il; ++c) a += double(hm.at(r, c));
        for (int64_t c = rs; c < W; ++c) b += double(hm.at(r, c));
      }
      mass += a;
      mass += b;
    }
    const double denom = double(heads.size()) * double(R);
    const double avg = denom > 0.0 ? mass / denom : 0.0;
    rep.avg[l] = avg;
    (avg < gamma ? rep.non_ir : rep.ir).push_back(int(l));
  }
  return rep;
}

// proj/include/krul/analysis.hpp:37-50 — expanded form in double, clamped.
double stable_sq(const float* a, const float* b, int64_t n) {
  double aa = 0.0, bb = 0.0, ab = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = a[i], y = b[i];
    aa += x * x;
    bb += y * y;
    ab += x * y;
  }
  const double d = aa + bb - 2.0 * ab;
  return d > 0.0 ? d : 0.0;
}

// proj/src/analysis.cpp:80-95
Accumulator::Accumulator(std::vector<int> ir, int n_heads) : layers(std::move(ir)), H(n_heads) {
  if (H < 1) fail(kConfig, "n_heads must be >= 1");
  std::sort(layers.begin(), layers.end());
  layers.erase(std::unique(layers.begin(), layers.end()), layers.end());
  if (!layers.empty() && layers.front() < 0) fail(kConfig, "layer indices must be non-negative");
  for (size_t a = 0; a < layers.size(); ++a)
    for (size_t b = a + 1; b < layers.size(); ++b) pairs.emplace_back(layers[a], layers[b]);
  sums.assign(pairs.size() * size_t(H), 0.0);
}

// proj/src/analysis.cpp:97-122
void Accumulator::fold_prefill(const AttnRecord& rec) {
  if (prefill_done) fail(kAccounting, "prefill attention folded twice");
  if (!layers.empty() && layers.back() >= int(rec.layers.size()))
    fail(kConfig, "record does not cover all tracked layers");
  for (size_t p = 0; p < pairs.size(); ++p) {
    const auto& A = rec.layers[size_t(pairs[p].first)].prefill;
    const auto& B = rec.layers[size_t(pairs[p].second)].prefill;
    if (int(A.size()) != H || int(B.size()) != H) fail(kStateCorruption, "prefill head count mismatch");
    for (int h = 0; h < H; ++h) {
      const Mat& a = A[size_t(h)];
      const Mat& b = B[size_t(h)];
      if (a.r != b.r || a.c != b.c) fail(kConfig, "stable_squared_distance: shape mismatch");
      sums[p * size_t(H) + size_t(h)] += stable_sq(a.v.data(), b.v.data(), a.r * a.c);
    }
  }
  prefill_done = true;
  prefill_rows = rec.rows();
}

// proj/src/analysis.cpp:124-151 — f32 difference, squared-summed in double.
void Accumulator::fold_decode(const std::vector<Mat>& rows) {
  if (!layers.empty() && layers.back() >= int(rows.size()))
    fail(kStateCorruption, "decode rows do not cover all tracked layers");
  int64_t width = -1;
  for (const Mat& m : rows) {
    if (m.r * m.c == 0) continue;
    if (width == -1) width = m.c;
    if (m.c != width) fail(kStateCorruption, "decode row width mismatch across layers");
  }
  for (size_t p = 0; p < pairs.size(); ++p) {
    const Mat& a = rows[size_t(pairs[p].first)];
    const Mat& b = rows[size_t(pairs[p].second)];
    if (a.r != H || b.r != H) fail(kStateCorruption, "decode head count mismatch");
    for (int h = 0; h < H; ++h) {
      double s = 0.0;
      for (int64_t c = 0; c < a.c; ++c) {
        const double d = double(a.at(h, c) - b.at(h, c));
        s += d * d;
      }
      sums[p * size_t(H) + size_t(h)] += s;
    }
  }
  ++decode_steps;
}

// proj/src/analysis.cpp:153-179
std::vector<double> Accumulator::finalize() const {
  if (!prefill_done) fail(kAccounting, "finalize requires the prefill part to be folded");
  const size_t n = layers.size();
  std::vector<double> D(n * n, 0.0);
  for (size_t p = 0; p < pairs.size(); ++p) {
    double mean = 0.0;
    for (int h = 0; h < H; ++h) mean += std::sqrt(sums[p * size_t(H) + size_t(h)]);
    mean /= double(H);
    const size_t i = size_t(std::lower_bound(layers.begin(), layers.end(), pairs[p].first) - layers.begin());
    const size_t j = size_t(std::lower_bound(layers.begin(), layers.end(), pairs[p].second) - layers.begin());
    D[i * n + j] = mean;
    D[j * n + i] = mean;
  }
  return D;
}

// ===========================================================================
// strategy
// ===========================================================================

// proj/src/strategy.cpp:16-25
int shared_layer_quota(int n_layers, double r_l) {
  if (r_l < 0.0 || r_l > 1.0) fail(kConfig, "r_l must lie in [0, 1]");
  if (n_layers < 0) fail(kConfig, "n_layers must be non-negative");
  const double q = std::ceil(double(n_layers) * r_l - 1e-9);
  return q < 0.0 ? 0 : int(q);
}

// proj/src/strategy.cpp:27-74
Strategy select_strategy(const std::vector<double>& D,
                         const std::vector<int>& dm_layers,
                         const std::vector<int>& ir_in, double r_l, int n_layers) {
  if (r_l < 0.0 || r_l > 1.0) fail(kConfig, "r_l must lie in [0, 1]");
  const int quota = shared_layer_quota(n_layers, r_l);
  Strategy s;
  if (quota == 0) return s;
  std::vector<int> ir = ir_in;
  std::sort(ir.begin(), ir.end());
  ir.erase(std::unique(ir.begin(), ir.end()), ir.end());
  if (ir.size() < 2) {
    s.exhausted = true;
    return s;
  }
  const size_t n = dm_layers.size();
  auto pos = [&](int layer) {  // DistanceMatrix::at (analysis.cpp:65-74)
    auto it = std::lower_bound(dm_layers.begin(), dm_layers.end(), layer);
    if (it == dm_layers.end() || *it != layer) fail(kConfig, "layer not tracked by the distance matrix");
    return size_t(it - dm_layers.begin());
  };
  std::vector<std::tuple<double, int, int>> cand;
  for (size_t a = 0; a < ir.size(); ++a)
    for (size_t b = a + 1; b < ir.size(); ++b)
      cand.emplace_back(D[pos(ir[a]) * n + pos(ir[b])], ir[a], ir[b]);
  std::sort(cand.begin(), cand.end());
  for (const auto& [d, i, j] : cand) {
    if (int(s.shared.size()) >= quota) break;
    if (s.shared.count(i) || s.shared.count(j)) continue;
    s.pairs.push_back({i, j, d});
    s.shared.insert(i);
    s.shared.insert(j);
  }
  if (int(s.shared.size()) < quota) s.exhausted = true;
  return s;
}

// proj/src/strategy.cpp:76-131
int validate_strategy(const Strategy& s, const std::vector<int>& ir_v,
                      int n_layers, double r_l) {
  int mask = 0;
  std::set<int> ir(ir_v.begin(), ir_v.end()), seen;
  double last = -1.0;
  for (const Pair& p : s.pairs) {
    if (p.shallow >= p.deep) mask |= 1;
    for (int m : {p.shallow, p.deep}) {
      if (m < 0 || m >= n_layers) mask |= 2;
      if (!ir.count(m)) mask |= 4;
      if (!seen.insert(m).second) mask |= 8;
    }
    if (p.distance < last) mask |= 16;
    last = p.distance;
  }
  if (s.shared != seen) mask |= 32;
  else if (s.shared.size() != 2 * s.pairs.size()) mask |= 32;
  if (int(s.shared.size()) < shared_layer_quota(n_layers, r_l) && !s.exhausted) mask |= 64;
  return mask;
}

// ===========================================================================
// kvstore
// ===========================================================================

// proj/src/kvstore.cpp:173-205 — ordered by shallowest owner.
std::vector<BlobSpec> plan_blob_specs(const Strategy& s, const Plan& plan) {
  const int n = int(plan.p.size());
  std::map<int, BlobSpec> by_first;
  std::vector<char> taken(size_t(n), 0);
  for (const Pair& p : s.pairs) {
    if (p.shallow < 0 || p.deep >= n || p.shallow >= p.deep)
      fail(kSnapshot, "strategy pair outside the plan's layers");
    if (taken[size_t(p.shallow)] || taken[size_t(p.deep)]) fail(kSnapshot, "layer appears in two pairs");
    taken[size_t(p.shallow)] = taken[size_t(p.deep)] = 1;
    by_first[p.shallow] = BlobSpec{{p.shallow, p.deep}, plan.load_span(p.deep)};
  }
  for (int l = 0; l < n; ++l)
    if (!taken[size_t(l)]) by_first[l] = BlobSpec{{l}, plan.load_span(l)};
  std::vector<BlobSpec> out;
  for (auto& kv : by_first) out.push_back(kv.second);
  return out;
}

// proj/src/kvstore.cpp:243-314
Snapshot compress_and_snapshot(const std::vector<KVLayer>& kv, const Strategy& s,
                               const Plan& plan, int mode, const std::string& id,
                               const ModelConfig& cfg) {
  const int n = int(plan.p.size());
  if (n != cfg.n_layers || int(kv.size()) != n)
    fail(kSnapshot, "plan, cache, and config disagree on the layer count");
  const int64_t L = plan.L;
  const int heads = cfg.kv_heads(), hd = cfg.head_dim;
  for (const KVLayer& l : kv) {
    if (l.span.start != 0 || l.span.end != L) fail(kSnapshot, "cache span does not cover the plan's history");
    if (int(l.k.size()) != heads || int(l.v.size()) != heads)
      fail(kSnapshot, "cache head count does not match the config");
  }
  Snapshot snap;
  snap.id = id;
  snap.config_hash = cfg.hash();
  snap.n_layers = n;
  snap.n_heads = heads;
  snap.head_dim = hd;
  snap.L = L;
  snap.mode = mode;
  snap.strategy = s;
  snap.plan = plan;
  auto slice = [&](const Mat& m, int64_t start, int64_t rows) {
    Mat o(rows, hd);
    if (rows > 0) std::memcpy(o.v.data(), m.row(start), sizeof(float) * size_t(rows * hd));
    return o;
  };
  for (const BlobSpec& spec : plan_blob_specs(s, plan)) {
    Blob b;
    b.owners = spec.owners;
    b.span = spec.span;
    const int64_t rows = spec.span.len(), start = spec.span.start;
    for (int g = 0; g < heads; ++g) {
      const KVLayer& deep = kv[size_t(spec.owners.back())];
      Mat k = slice(deep.k[size_t(g)], start, rows), v = slice(deep.v[size_t(g)], start, rows);
      if (spec.owners.size() == 2 && mode == 0) {
        const KVLayer& sh = kv[size_t(spec.owners[0])];
        const int64_t ms = plan.p[size_t(spec.owners[0])];
        const int64_t mr = L - ms;
        for (int64_t r = 0; r < mr; ++r)
          for (int t = 0; t < hd; ++t) {
            const int64_t br = rows - mr + r;
            k.at(br, t) = 0.5f * (sh.k[size_t(g)].at(ms + r, t) + deep.k[size_t(g)].at(ms + r, t));
            v.at(br, t) = 0.5f * (sh.v[size_t(g)].at(ms + r, t) + deep.v[size_t(g)].at(ms + r, t));
          }
      }
      b.k.push_back(std::move(k));
      b.v.push_back(std::move(v));
    }
    snap.blobs.push_back(std::move(b));
  }
  return snap;
}

// proj/src/kvstore.cpp:316-343
KVLayer expand(const Snapshot& snap, int layer) {
  const Blob* blob = nullptr;
  for (const Blob& b : snap.blobs)
    if (std::find(b.owners.begin(), b.owners.end(), layer) != b.owners.end()) {
      blob = &b;
      break;
    }
  if (!blob) fail(kRestorationGap, "layer " + std::to_string(layer) + " is not covered by any stored blob");
  const Span want = snap.plan.load_span(layer);
  if (want.start < blob->span.start || want.end != blob->span.end)
    fail(kRestorationGap, "stored span does not cover the load span");
  KVLayer out;
  out.span = want;
  const int64_t off = want.start - blob->span.start, rows = want.len();
  const int hd = snap.head_dim;
  for (size_t g = 0; g < blob->k.size(); ++g) {
    Mat k(rows, hd), v(rows, hd);
    if (rows > 0) {
      std::memcpy(k.v.data(), blob->k[g].row(off), sizeof(float) * size_t(rows * hd));
      std::memcpy(v.v.data(), blob->v[g].row(off), sizeof(float) * size_t(rows * hd));
    }
    out.k.push_back(std::move(k));
    out.v.push_back(std::move(v));
  }
  return out;
}

// proj/src/kvstore.cpp:345-358
void storage_report(const Snapshot& snap, uint64_t* full, uint64_t* stored) {
  const uint64_t row = 2ull * uint64_t(snap.n_heads) * uint64_t(snap.head_dim) * sizeof(float);
  *full = uint64_t(snap.n_layers) * uint64_t(snap.L) * row;
  *stored = 0;
  for (const Blob& b : snap.blobs) *stored += uint64_t(b.span.len()) * row;
}

// ===========================================================================
// scheduler
// ===========================================================================

// proj/include/krul/scheduler.hpp:22-28
double CostModel::layer_flops(int64_t p, int64_t d) const {
  const double pd = double(p), dd = double(d);
  return pd * (8.0 * dd * dd + 4.0 * dd * ffn_mult * dd) + 4.0 * dd * (0.5 * pd * (pd + 1.0));
}
// proj/src/scheduler.cpp:42-51
double CostModel::prefill_flops(int64_t n, int64_t hist, int64_t d, int N) const {
  const double nn = double(n), hh = double(hist), dd = double(d);
  const double span = nn * hh + 0.5 * nn * (nn + 1.0);
  return (nn * (8.0 * dd * dd + 4.0 * dd * ffn_mult * dd) + 4.0 * dd * span) * double(N);
}
// proj/include/krul/scheduler.hpp:36-38
double CostModel::blob_bytes(int64_t span, int64_t d) const {
  return 2.0 * double(span) * double(d) * 4.0;
}

namespace {
void check_ratio(double r) {
  if (!(r >= 0.0) || r > 1.0) fail(kConfig, "r_c must lie in [0, 1]");
}
double compute_s(const CostModel& c, const Plan& plan, int64_t d) {  // scheduler.cpp:15-22
  double f = 0.0;
  for (int64_t p : plan.p) f += c.layer_flops(p, d);
  return f / c.f_peak;
}
double load_s(const CostModel& c, const Plan& plan, const Strategy& s, int64_t d) {  // :24-32
  double b = 0.0;
  for (const BlobSpec& sp : plan_blob_specs(s, plan)) b += c.blob_bytes(sp.span.len(), d);
  return b / c.b_peak;
}
}  // namespace

// proj/src/scheduler.cpp:53-128
Plan build_plan(int64_t L, int N, double r_c, const Strategy& s) {
  check_ratio(r_c);
  if (N < 1) fail(kConfig, "n_layers must be >= 1");
  if (L < 0) fail(kConfig, "history_len must be >= 0");
  for (const Pair& p : s.pairs)
    if (p.shallow < 0 || p.deep >= N) fail(kPlanInvalid, "strategy pair outside the layer range");
  Plan plan;
  plan.L = L;
  plan.p.assign(size_t(N), 0);
  if (N == 1) {
    plan.p[0] = std::llround(r_c * double(L));
    return plan;
  }
  const double den = double(N - 1);
  for (int l = 0; l < N; ++l) {
    double f = r_c <= 0.5 ? 2.0 * r_c * double(N - 1 - l) / den
                          : 1.0 - 2.0 * (1.0 - r_c) * double(l) / den;
    f = std::clamp(f, 0.0, 1.0);
    plan.p[size_t(l)] = std::llround(f * double(L));
  }
  for (int l = 1; l < N; ++l) plan.p[size_t(l)] = std::min(plan.p[size_t(l)], plan.p[size_t(l - 1)]);
  const double target = r_c * double(L) * double(N), tol = double(N);
  auto total = [&] {
    int64_t t = 0;
    for (int64_t x : plan.p) t += x;
    return t;
  };
  while (double(total()) < target - tol) {
    bool moved = false;
    for (int l = N - 1; l >= 0; --l) {
      const int64_t cap = l == 0 ? L : plan.p[size_t(l - 1)];
      if (plan.p[size_t(l)] < cap) {
        ++plan.p[size_t(l)];
        moved = true;
        break;
      }
    }
    if (!moved) break;
  }
  while (double(total()) > target + tol) {
    bool moved = false;
    for (int l = N - 1; l >= 0; --l) {
      const int64_t floor_v = l == N - 1 ? 0 : plan.p[size_t(l + 1)];
      if (plan.p[size_t(l)] > floor_v) {
        --plan.p[size_t(l)];
        moved = true;
        break;
      }
    }
    if (!moved) break;
  }
  return plan;
}

// proj/src/scheduler.cpp:130-140
Plan uniform_plan(int64_t L, int N, double r_c) {
  check_ratio(r_c);
  if (N < 1) fail(kConfig, "n_layers must be >= 1");
  if (L < 0) fail(kConfig, "history_len must be >= 0");
  Plan plan;
  plan.L = L;
  plan.p.assign(size_t(N), std::clamp<int64_t>(std::llround(r_c * double(L)), 0, L));
  return plan;
}

// proj/src/scheduler.cpp:142-163 — strict `<`, ties keep the smaller ratio.
double calibrate_rc(const CostModel& c, int N, int64_t L, int64_t d,
                    const Strategy& s, const std::vector<double>& grid) {
  if (grid.empty()) fail(kConfig, "calibration grid is empty");
  std::vector<double> g = grid;
  std::sort(g.begin(), g.end());
  double best = g.front(), best_diff = std::numeric_limits<double>::infinity();
  for (double r : g) {
    check_ratio(r);
    const Plan plan = build_plan(L, N, r, s);
    const double diff = std::abs(compute_s(c, plan, d) - load_s(c, plan, s, d));
    if (diff < best_diff) {
      best_diff = diff;
      best = r;
    }
  }
  return best;
}

// proj/src/scheduler.cpp:165-177
std::vector<double> default_rc_grid(double step) {
  if (!(step > 0.0) || step > 1.0) fail(kConfig, "grid step must lie in (0, 1]");
  std::vector<double> g;
  for (int64_t k = 0;; ++k) {
    const double v = double(k) * step;
    if (v > 1.0 + 1e-12) break;
    g.push_back(std::min(v, 1.0));
  }
  if (g.back() < 1.0 - 1e-12) g.push_back(1.0);
  return g;
}

// proj/src/scheduler.cpp:179-221
int validate_plan(const Plan& plan, const Strategy& s) {
  int mask = 0;
  const int n = int(plan.p.size());
  if (plan.L < 0) mask |= 1;
  for (int l = 0; l < n; ++l) {
    const int64_t p = plan.p[size_t(l)];
    if (p < 0 || p > plan.L) mask |= 1;
    if (l > 0 && p > plan.p[size_t(l - 1)]) mask |= 2;
    if (p + (plan.L - p) != plan.L) mask |= 4;
  }
  for (const Pair& pr : s.pairs) {
    if (pr.shallow < 0 || pr.deep >= n || pr.shallow >= pr.deep) {
      mask |= 8;
      continue;
    }
    if (plan.p[size_t(pr.deep)] > plan.p[size_t(pr.shallow)]) mask |= 8;
  }
  return mask;
}

// proj/src/scheduler.cpp:223-264
int validate_plan_snapshot(const Plan& plan, const Snapshot& snap) {
  int mask = validate_plan(plan, snap.strategy);
  const int n = int(plan.p.size());
  if (snap.L != plan.L || snap.n_layers != n) return mask | 1;
  std::vector<const Blob*> of(size_t(n), nullptr);
  for (const Blob& b : snap.blobs)
    for (int o : b.owners) {
      if (o < 0 || o >= n) {
        mask |= 8;
        continue;
      }
      if (of[size_t(o)]) mask |= 8;
      of[size_t(o)] = &b;
    }
  for (int l = 0; l < n; ++l) {
    const Blob* b = of[size_t(l)];
    if (!b) {
      mask |= 8;
      continue;
    }
    if (b->span.end != plan.L || b->span.start > plan.p[size_t(l)]) mask |= 8;
  }
  return mask;
}

// proj/src/scheduler.cpp:282-318
Trace simulate_pipeline(const Plan& plan, const Strategy& s, const CostModel& c, int64_t d) {
  Trace t;
  double clock = 0.0;
  for (int l = 0; l < int(plan.p.size()); ++l) {
    const double secs = c.layer_flops(plan.p[size_t(l)], d) / c.f_peak;
    if (secs <= 0.0) continue;
    t.compute.push_back({l, clock, clock + secs});
    clock += secs;
  }
  t.compute_finish = clock;
  clock = 0.0;
  for (const BlobSpec& sp : plan_blob_specs(s, plan)) {
    const double secs = c.blob_bytes(sp.span.len(), d) / c.b_peak;
    if (secs <= 0.0) continue;
    t.load.push_back({sp.owners.front(), clock, clock + secs});
    clock += secs;
  }
  t.load_finish = clock;
  t.makespan = std::max(t.compute_finish, t.load_finish);
  if (t.makespan > 0.0) {
    if (!t.compute.empty()) t.bubble_compute = (t.makespan - t.compute_finish) / t.makespan;
    if (!t.load.empty()) t.bubble_load = (t.makespan - t.load_finish) / t.makespan;
  }
  return t;
}

// proj/src/scheduler.cpp:320-400 — loader thread expands blobs in service
// order while the caller recomputes prefixes; per-layer splice afterwards.
std::vector<KVLayer> execute_restore(const Model& m, const std::vector<int32_t>& hist,
                                     const Snapshot& snap) {
  const ModelConfig& cfg = m.cfg;
  if (snap.config_hash != cfg.hash()) fail(kSnapshot, "snapshot was taken under a different model config");
  if (int64_t(hist.size()) != snap.L) fail(kRestorationGap, "history length does not match the snapshot");
  const Plan& plan = snap.plan;
  // First violation decides the exception type (scheduler.cpp:331-336);
  // validate_plan emits bounds/monotonicity/totals before coverage.
  const int mask = validate_plan_snapshot(plan, snap);
  if (mask) {
    // re-derive the first violation's kind in emission order
    const int first_kind = validate_plan(plan, snap.strategy);
    if (first_kind & 7) fail(kPlanInvalid, "plan violation");
    if (first_kind & 8) fail(kRestorationGap, "coverage violation");
    if (snap.L != plan.L || snap.n_layers != int(plan.p.size())) fail(kPlanInvalid, "bounds: snapshot header disagrees with the plan");
    fail(kRestorationGap, "coverage: stored span does not cover its load span");
  }
  std::vector<KVLayer> loaded(size_t(cfg.n_layers));
  std::exception_ptr loader_err;
  std::thread loader([&] {
    try {
      for (const Blob& b : snap.blobs)
        for (int o : b.owners) loaded[size_t(o)] = expand(snap, o);
    } catch (...) {
      loader_err = std::current_exception();
    }
  });
  PartialOut part;
  try {
    part = partial_prefix_recompute(m, hist, plan.p);
  } catch (...) {
    loader.join();
    throw;
  }
  loader.join();
  if (loader_err) std::rethrow_exception(loader_err);
  const int hd = cfg.head_dim;
  std::vector<KVLayer> out(size_t(cfg.n_layers));
  for (int l = 0; l < cfg.n_layers; ++l) {
    const KVLayer& ld = loaded[size_t(l)];
    if (!(ld.span == plan.load_span(l))) fail(kRestorationGap, "loaded span does not abut the prefix");
    const KVLayer& cp = part.kv[size_t(l)];
    const int64_t pre = plan.p[size_t(l)];
    KVLayer& o = out[size_t(l)];
    for (int g = 0; g < cfg.kv_heads(); ++g) {
      Mat k(plan.L, hd), v(plan.L, hd);
      if (pre > 0) {
        std::memcpy(k.v.data(), cp.k[size_t(g)].v.data(), sizeof(float) * size_t(pre * hd));
        std::memcpy(v.v.data(), cp.v[size_t(g)].v.data(), sizeof(float) * size_t(pre * hd));
      }
      if (ld.span.len() > 0) {
        std::memcpy(k.row(pre), ld.k[size_t(g)].v.data(), sizeof(float) * size_t(ld.span.len() * hd));
        std::memcpy(v.row(pre), ld.v[size_t(g)].v.data(), sizeof(float) * size_t(ld.span.len() * hd));
      }
      o.k.push_back(std::move(k));
      o.v.push_back(std::move(v));
    }
    o.span = {0, plan.L};
  }
  return out;
}

}  // namespace kro
