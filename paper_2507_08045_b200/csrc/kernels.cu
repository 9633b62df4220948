// kernels.cu — elementwise, attention, KV paging, estimator and selector
// kernels of the B200 Krul hot path. Templated on the compute dtype T
// (float = parity mode, __nv_bfloat16 = perf mode). GEMMs live in
// gemm_simt.cu / gemm_sm100.cu.
#include <cstdlib>
#include <cstring>
#include <cfloat>
#include <cmath>

#include "kb.hpp"
#include "dev.cuh"
#include "kvcode.hpp"

namespace kb {

// ---------------------------------------------------------------- embed
// engine.cpp:195-207 (token range is validated on the host first).
template <class T>
__global__ void k_embed(const int32_t* tok, int64_t n, const T* emb, int d, float* h) {
  const int64_t r = blockIdx.x;
  const T* src = emb + int64_t(tok[r]) * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) h[r * d + j] = tof(src[j]);
}
void launch_embed(const Ctx& c, cudaStream_t s, const int32_t* tok, int64_t n, float* h) {
  if (n <= 0) return;
  if (c.cfg.dtype == KRUL_BF16)
    k_embed<<<unsigned(n), 256, 0, s>>>(tok, n, (const bf16*)c.embed, c.cfg.d, h);
  else
    k_embed<<<unsigned(n), 256, 0, s>>>(tok, n, (const float*)c.embed, c.cfg.d, h);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- rmsnorm
// engine.cpp:117-124: xn = x / sqrt(mean(x^2) + 1e-6), no gain.
template <class T>
__global__ void k_rmsnorm(const float* h, int d, T* out) {
  const int64_t r = blockIdx.x;
  const float* x = h + r * d;
  float ss = 0.f;
  for (int j = threadIdx.x; j < d; j += blockDim.x) ss += x[j] * x[j];
  ss = block_sum(ss);
  const float denom = sqrtf(ss / float(d) + 1e-6f);
  for (int j = threadIdx.x; j < d; j += blockDim.x) out[r * d + j] = fromf<T>(x[j] / denom);
}
// bf16 fast path (d in {256, 512, 4096}): one warp per row, the row held
// in registers (16-byte loads, one HBM pass), shuffle reduction, 8-byte
// packed bf16 stores; same arithmetic per element as k_rmsnorm.
template <int V>  // float4 vectors per lane: d = 128 * V
__global__ void __launch_bounds__(256) k_rmsnorm_warp(const float* __restrict__ h, int64_t rows,
                                                      int d, bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const float4* x = reinterpret_cast<const float4*>(h + r * d);
  float4 v[V];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    v[i] = __ldg(x + lane + 32 * i);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum(ss);
  const float denom = sqrtf(ss / float(d) + 1e-6f);
  uint2* o = reinterpret_cast<uint2*>(out + r * d);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[i].x / denom, v[i].y / denom);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[i].z / denom, v[i].w / denom);
    o[lane + 32 * i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}
// Few rows (the new-input prefill's 128): one 256-thread CTA per row so the
// norm spreads over the SMs instead of 16 CTAs (measured 9 us -> the launch
// floor); same arithmetic order per element, block reduction of the sum.
template <int V>  // float4 vectors per thread: d = 1024 * V
__global__ void __launch_bounds__(256) k_rmsnorm_cta(const float* __restrict__ h, int d,
                                                     bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t r = blockIdx.x;
  const float4* x = reinterpret_cast<const float4*>(h + r * d);
  float4 v[V];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    v[i] = __ldg(x + threadIdx.x + 256 * i);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = block_sum(ss);
  const float denom = sqrtf(ss / float(d) + 1e-6f);
  uint2* o = reinterpret_cast<uint2*>(out + r * d);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[i].x / denom, v[i].y / denom);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[i].z / denom, v[i].w / denom);
    o[threadIdx.x + 256 * i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}
void launch_rmsnorm(const Ctx& c, cudaStream_t s, const float* h, int64_t rows, void* xn) {
  if (rows <= 0) return;
  const int d = c.cfg.d;
  if (c.cfg.dtype == KRUL_BF16 && rows <= 2 * 148 && (d == 4096 || d == 8192)) {
    if (d == 4096)
      KB_CUDA(launch_pdl(k_rmsnorm_cta<4>, dim3(unsigned(rows)), dim3(256), 0, s, h, d, (bf16*)xn));
    else
      KB_CUDA(launch_pdl(k_rmsnorm_cta<8>, dim3(unsigned(rows)), dim3(256), 0, s, h, d, (bf16*)xn));
    KB_LAUNCH();
    return;
  }
  if (c.cfg.dtype == KRUL_BF16 && d % 128 == 0 && d <= 128 * 32) {
    const unsigned blocks = unsigned((rows + 7) / 8);
    switch (d / 128) {
      case 32: KB_CUDA(launch_pdl(k_rmsnorm_warp<32>, dim3(blocks), dim3(256), 0, s, h, rows, d, (bf16*)xn)); KB_LAUNCH(); return;
      case 2: KB_CUDA(launch_pdl(k_rmsnorm_warp<2>, dim3(blocks), dim3(256), 0, s, h, rows, d, (bf16*)xn)); KB_LAUNCH(); return;
      case 4: KB_CUDA(launch_pdl(k_rmsnorm_warp<4>, dim3(blocks), dim3(256), 0, s, h, rows, d, (bf16*)xn)); KB_LAUNCH(); return;
      default: break;
    }
  }
  if (c.cfg.dtype == KRUL_BF16)
    k_rmsnorm<<<unsigned(rows), 256, 0, s>>>(h, d, (bf16*)xn);
  else
    k_rmsnorm<<<unsigned(rows), 256, 0, s>>>(h, d, (float*)xn);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- paging
struct PageView {
  const int* pt;   // [max_pages] for one layer
  char* pool;
  int64_t page_bytes;
  int Hkv, hd, esz;
  __device__ __forceinline__ char* page(int64_t pos) const {
    return pool + int64_t(pt[pos / kPageTokens]) * page_bytes;
  }
  // element offsets inside a page
  __device__ __forceinline__ int64_t k_off(int g, int64_t pos, int t) const {
    return (int64_t(g) * kPageTokens + pos % kPageTokens) * hd + t;
  }
  __device__ __forceinline__ int64_t v_off(int g, int64_t pos, int t) const {  // V^T
    return int64_t(Hkv) * kPageTokens * hd + (int64_t(g) * hd + t) * kPageTokens + pos % kPageTokens;
  }
};
static PageView page_view(const Ctx& c, const Conv& conv, int layer) {
  PageView v;
  v.pt = conv.d_pt + int64_t(layer) * conv.max_pages;
  v.pool = static_cast<char*>(c.pool.p);
  v.page_bytes = int64_t(c.page_elems() * c.esz);
  v.Hkv = c.cfg.Hkv;
  v.hd = c.cfg.hd;
  v.esz = int(c.esz);
  return v;
}

// ---------------------------------------------------------------- rope + scatter
// engine.cpp:128-143 (interleaved pairs, odd trailing dim passes through) and
// :162-170 (K/V of every block row appended before attention).
template <class T>
__global__ void k_rope_scatter(const float* qkv, int64_t pos0, int64_t q_rows, T* q, PageView pv,
                               const float* cosT, const float* sinT, int H, int64_t seg_rows, int64_t pos1) {
  const int64_t r = blockIdx.x;
  const int hd = pv.hd, Hkv = pv.Hkv, half = hd / 2;
  const int64_t pos = r < seg_rows ? pos0 + r : pos1 + (r - seg_rows);
  const int nq = H * hd, nkv = Hkv * hd;
  const float* row = qkv + r * int64_t(nq + 2 * nkv);
  const float* cs = cosT + pos * half;
  const float* sn = sinT + pos * half;
  T* page = reinterpret_cast<T*>(pv.page(pos));
  // rotate Q (only the leading q_rows rows need Q)
  if (r < q_rows) {
    for (int e = threadIdx.x; e < nq; e += blockDim.x) {
      const int t = e % hd;
      float y;
      if (t < 2 * half) {
        const int i = t >> 1;
        const float x0 = row[e - (t & 1)], x1 = row[e - (t & 1) + 1];
        y = (t & 1) ? (x0 * sn[i] + x1 * cs[i]) : (x0 * cs[i] - x1 * sn[i]);
      } else {
        y = row[e];
      }
      q[r * nq + e] = fromf<T>(y);
    }
  }
  for (int e = threadIdx.x; e < nkv; e += blockDim.x) {
    const int g = e / hd, t = e % hd;
    const float* kr = row + nq;
    float y;
    if (t < 2 * half) {
      const int i = t >> 1;
      const float x0 = kr[e - (t & 1)], x1 = kr[e - (t & 1) + 1];
      y = (t & 1) ? (x0 * sn[i] + x1 * cs[i]) : (x0 * cs[i] - x1 * sn[i]);
    } else {
      y = kr[e];
    }
    page[pv.k_off(g, pos, t)] = fromf<T>(y);
    page[pv.v_off(g, pos, t)] = fromf<T>(row[nq + nkv + e]);
  }
}
void launch_rope_scatter(const Ctx& c, cudaStream_t s, const float* qkv, int64_t rows,
                         int64_t pos0, int64_t q_rows, void* q, const Conv& conv, int layer,
                         int64_t seg_rows, int64_t pos1) {
  if (rows <= 0) return;
  PageView pv = page_view(c, conv, layer);
  if (c.cfg.dtype == KRUL_BF16)
    k_rope_scatter<<<unsigned(rows), 128, 0, s>>>(qkv, pos0, q_rows, (bf16*)q, pv, c.rope_cos,
                                                  c.rope_sin, c.cfg.H, seg_rows, pos1);
  else
    k_rope_scatter<<<unsigned(rows), 128, 0, s>>>(qkv, pos0, q_rows, (float*)q, pv, c.rope_cos,
                                                  c.rope_sin, c.cfg.H, seg_rows, pos1);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- attention (SIMT)
// engine.cpp:174-188: per head, scores = q K^T * (1/sqrt(hd)), causal width
// pos0 + r + 1, softmax with max subtraction, ctx = P V. One CTA per
// (row, head); the score row lives in shared memory. Optionally emits the
// normalised probabilities (capture) and the classifier region mass
// (analysis.cpp:46-54) accumulated in double.
template <class T>
__global__ void k_attn_simt(const T* q, int64_t pos0, PageView pv, int H, float scale, T* out,
                            float* probs, int64_t ld_probs, int64_t probs_row0, int64_t probs_rows,
                            double* mass, int64_t mass_rows, int64_t il, int64_t rs, float* stats) {
  extern __shared__ float sm[];
  const int64_t r = blockIdx.x;
  const int h = blockIdx.y;
  const int hd = pv.hd;
  const int g = h / (H / pv.Hkv);
  const int64_t W = pos0 + r + 1;
  float* qs = sm;            // [hd]
  float* sc = sm + hd;       // [W]
  for (int t = threadIdx.x; t < hd; t += blockDim.x) qs[t] = tof(q[(r * H + h) * hd + t]);
  __syncthreads();
  float mx = -FLT_MAX;
  for (int64_t k = threadIdx.x; k < W; k += blockDim.x) {
    const T* kr = reinterpret_cast<const T*>(pv.page(k)) + pv.k_off(g, k, 0);
    float dot = 0.f;
    for (int t = 0; t < hd; ++t) dot += qs[t] * tof(kr[t]);
    const float sv = dot * scale;
    sc[k] = sv;
    mx = fmaxf(mx, sv);
  }
  mx = block_max(mx);
  float sum = 0.f;
  for (int64_t k = threadIdx.x; k < W; k += blockDim.x) {
    const float e = expf(sc[k] - mx);
    sc[k] = e;
    sum += e;
  }
  sum = block_sum(sum);
  if (stats && threadIdx.x == 0) {
    stats[(int64_t(h) * mass_rows + probs_row0 + r) * 2] = mx;
    stats[(int64_t(h) * mass_rows + probs_row0 + r) * 2 + 1] = sum;
  }
  double ms = 0.0;
  for (int64_t k = threadIdx.x; k < W; k += blockDim.x) {
    const float p = sc[k] / sum;
    sc[k] = p;
    if (probs) probs[(int64_t(h) * probs_rows + probs_row0 + r) * ld_probs + k] = p;
    if (mass && (k < il || k >= rs)) ms += double(p);
  }
  if (mass) {
    ms = block_sum_d(ms);
    if (threadIdx.x == 0) mass[int64_t(h) * mass_rows + probs_row0 + r] = ms;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < hd; t += blockDim.x) {
    float acc = 0.f;
    for (int64_t k = 0; k < W; ++k) {
      const T* vr = reinterpret_cast<const T*>(pv.page(k));
      acc += sc[k] * tof(vr[pv.v_off(g, k, t)]);
    }
    out[(r * H + h) * hd + t] = fromf<T>(acc);
  }
}

// ---------------------------------------------------------------- decode attention
// One query row per head (decode_step, engine.cpp:406-446) over W keys, bf16
// cache, hd = 128, GQA group G = H / Hkv <= 8: the keys are split over
// CTAs (chunks of 256 keys x KV head) so the whole GPU streams the cache
// (the per-(row, head) SIMT kernel ran 32 CTAs for 1.2 ms per layer at 8K).
// Pass 1: each lane scores one key for the group's G heads (K row read once),
// chunk max / sum / partial P.V per head; raw scores go to the capture row.
// Pass 2 (one CTA per head): merges the chunk partials, writes the context
// row and normalises the captured probabilities (+ region mass) in place.
constexpr int kDecChunk = 256, kDecMaxG = 8;
__global__ void __launch_bounds__(256) k_attn_decode1(const bf16* __restrict__ q, int64_t W, PageView pv,
                                                      int H, float scale, float* __restrict__ probs,
                                                      int64_t ld_probs, float* __restrict__ part) {
  constexpr int HD = 128;
  const int g = blockIdx.y, G = H / pv.Hkv, h0 = g * G;
  const int64_t k0 = int64_t(blockIdx.x) * kDecChunk;
  const int nk = int(W - k0 < kDecChunk ? W - k0 : kDecChunk);
  __shared__ float qs[kDecMaxG][HD];
  __shared__ __align__(16) float ps[kDecMaxG][kDecChunk];
  __shared__ float red[kDecMaxG][8];
  __shared__ float o2[kDecMaxG][HD];
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) qs[i / HD][i % HD] = __bfloat162float(q[(h0 + i / HD) * HD + i % HD]) * scale;
  __syncthreads();
  // scores: thread j -> key k0 + j
  float sc[kDecMaxG];
  const int j = threadIdx.x;
  if (j < nk) {
    const int64_t k = k0 + j;
    const uint4* kr = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(pv.page(k)) + pv.k_off(g, k, 0));
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh) sc[hh] = 0.f;
#pragma unroll 4
    for (int v = 0; v < HD / 8; ++v) {
      const uint4 x = __ldg(kr + v);
      const uint32_t u[4] = {x.x, x.y, x.z, x.w};
      float f[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[e]));
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
      }
#pragma unroll
      for (int hh = 0; hh < kDecMaxG; ++hh) {
        if (hh < G) {
          float a = sc[hh];
#pragma unroll
          for (int e = 0; e < 8; ++e) a += qs[hh][8 * v + e] * f[e];
          sc[hh] = a;
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh) {
      if (hh < G) {
        ps[hh][j] = sc[hh];
        if (probs) probs[int64_t(h0 + hh) * ld_probs + k] = sc[hh];  // raw score, normalised in pass 2
      }
    }
  }
  __syncthreads();
  // chunk max and sum per head (warp w reduces head w's row)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < G) {
    float m = -FLT_MAX;
    for (int i = lane; i < nk; i += 32) m = fmaxf(m, ps[warp][i]);
    m = warp_max(m);
    float l = 0.f;
    for (int i = lane; i < nk; i += 32) {
      const float e = expf(ps[warp][i] - m);
      ps[warp][i] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      red[warp][0] = m;
      red[warp][1] = l;
    }
  }
  __syncthreads();
  // partial P.V: thread -> dimension d, key half
  const int d = threadIdx.x & (HD - 1), half = threadIdx.x >> 7;
  float acc[kDecMaxG];
#pragma unroll
  for (int hh = 0; hh < kDecMaxG; ++hh) acc[hh] = 0.f;
  const int i0 = half * (kDecChunk / 2), i1 = min(nk, i0 + kDecChunk / 2);
  // V^T rows are token-contiguous inside a page: 8 tokens per 16-byte load
  int i = i0;
  for (; i + 8 <= i1; i += 8) {
    const int64_t k = k0 + i;
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(pv.page(k)) +
                                                         pv.v_off(g, k, d)));
    const uint32_t u[4] = {x.x, x.y, x.z, x.w};
    float t[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[e]));
      t[2 * e] = f.x;
      t[2 * e + 1] = f.y;
    }
    // the 8 probabilities of each head as two broadcast 16-byte shared loads
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh) {
      if (hh < G) {
        const float4 p0 = *reinterpret_cast<const float4*>(&ps[hh][i]);
        const float4 p1 = *reinterpret_cast<const float4*>(&ps[hh][i + 4]);
        acc[hh] += p0.x * t[0] + p0.y * t[1] + p0.z * t[2] + p0.w * t[3] + p1.x * t[4] + p1.y * t[5] +
                   p1.z * t[6] + p1.w * t[7];
      }
    }
  }
  for (; i < i1; ++i) {
    const int64_t k = k0 + i;
    const float v = __bfloat162float(reinterpret_cast<const bf16*>(pv.page(k))[pv.v_off(g, k, d)]);
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh)
      if (hh < G) acc[hh] += ps[hh][i] * v;
  }
  if (half == 1) {
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh)
      if (hh < G) o2[hh][d] = acc[hh];
  }
  __syncthreads();
  if (half == 0) {
    float* pp = part + (int64_t(blockIdx.x) * H + h0) * (HD + 2);
#pragma unroll
    for (int hh = 0; hh < kDecMaxG; ++hh) {
      if (hh < G) {
        pp[int64_t(hh) * (HD + 2) + d] = acc[hh] + o2[hh][d];
        if (d == 0) {
          pp[int64_t(hh) * (HD + 2) + HD] = red[hh][0];
          pp[int64_t(hh) * (HD + 2) + HD + 1] = red[hh][1];
        }
      }
    }
  }
}
// grid (H, nsub): every CTA merges the chunk statistics (cheap) and
// normalises its slice of the captured row; sub-block 0 writes the context.
__global__ void __launch_bounds__(256) k_attn_decode2(const float* __restrict__ part, int nchunks, int64_t W,
                                                      int H, bf16* __restrict__ out, float* __restrict__ probs,
                                                      int64_t ld_probs, double* mass, int64_t il, int64_t rs) {
  constexpr int HD = 128;
  const int h = blockIdx.x;
  __shared__ float sh_ml[2];
  float m = -FLT_MAX;
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) m = fmaxf(m, part[(int64_t(c) * H + h) * (HD + 2) + HD]);
  m = block_max(m);
  float l = 0.f;
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) {
    const float* pp = part + (int64_t(c) * H + h) * (HD + 2);
    l += pp[HD + 1] * expf(pp[HD] - m);
  }
  l = block_sum(l);
  if (threadIdx.x == 0) {
    sh_ml[0] = m;
    sh_ml[1] = l;
  }
  __syncthreads();
  m = sh_ml[0];
  l = sh_ml[1];
  if (blockIdx.y == 0) {  // context row: the two thread halves take alternate chunks, loads batched
    __shared__ float oh[HD];
    const int d = threadIdx.x & (HD - 1), hf = threadIdx.x >> 7;
    float o = 0.f;
    for (int c0 = hf; c0 < nchunks; c0 += 16) {
      float pv[8], ev[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + 2 * u;
        const float* pp = part + (int64_t(c) * H + h) * (HD + 2);
        pv[u] = c < nchunks ? pp[d] : 0.f;
        ev[u] = c < nchunks ? pp[HD] : -FLT_MAX;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) o += pv[u] * expf(ev[u] - m);
    }
    if (hf == 1) oh[d] = o;
    __syncthreads();
    if (hf == 0) out[int64_t(h) * HD + d] = __float2bfloat16_rn((o + oh[d]) / l);
  }
  if (probs) {
    const int64_t per = (W + gridDim.y - 1) / gridDim.y;
    const int64_t a = int64_t(blockIdx.y) * per, b = a + per < W ? a + per : W;
    double ms = 0.0;
    float* pr = probs + int64_t(h) * ld_probs;
    for (int64_t k0 = a + threadIdx.x; k0 < b; k0 += 8 * int64_t(blockDim.x)) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + int64_t(u) * blockDim.x;
        x[u] = k < b ? pr[k] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + int64_t(u) * blockDim.x;
        if (k < b) {
          const float p = expf(x[u] - m) / l;
          pr[k] = p;
          if (mass && (k < il || k >= rs)) ms += double(p);
        }
      }
    }
    if (mass) {  // mass requests run with one sub-block per head
      ms = block_sum_d(ms);
      if (threadIdx.x == 0) mass[h] = ms;
    }
  }
}
static bool attention_decode_supported(const Ctx& c, const AttnArgs& a) {
  static const bool simt = [] {  // KRUL_DECODE_ATTN=simt: the per-(row, head) kernel (tests)
    const char* v = std::getenv("KRUL_DECODE_ATTN");
    return v && std::strcmp(v, "simt") == 0;
  }();
  return !simt && a.rows == 1 && c.cfg.dtype == KRUL_BF16 && c.cfg.hd == 128 && c.cfg.H % c.cfg.Hkv == 0 &&
         c.cfg.H / c.cfg.Hkv <= kDecMaxG && (!a.probs || a.probs_rows == 1) && a.probs_row0 == 0 &&
         (!a.mass || a.mass_rows == 1) && !a.stats;
}
static void launch_attention_decode(const Ctx& c, cudaStream_t s, const Conv& conv, int layer, const AttnArgs& a) {
  PageView pv = page_view(c, conv, layer);
  const int64_t W = a.pos0 + 1;
  const int nch = int((W + kDecChunk - 1) / kDecChunk);
  float* part = static_cast<float*>(const_cast<Ctx&>(c).dec_part.ensure(size_t(nch) * c.cfg.H * (128 + 2) * 4));
  const float scale = 1.0f / sqrtf(float(c.cfg.hd));
  k_attn_decode1<<<dim3(unsigned(nch), unsigned(c.cfg.Hkv)), 256, 0, s>>>(
      (const bf16*)a.q, W, pv, c.cfg.H, scale, a.probs, a.ld_probs, part);
  KB_LAUNCH();
  const unsigned nsub = a.mass ? 1u : unsigned(std::min<int64_t>(16, (W + 2047) / 2048));
  k_attn_decode2<<<dim3(unsigned(c.cfg.H), nsub), 256, 0, s>>>(part, nch, W, c.cfg.H, (bf16*)a.out, a.probs,
                                                               a.ld_probs, a.mass, a.il, a.rs);
  KB_LAUNCH();
}

void launch_attention(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                      const AttnArgs& a) {
  if (a.rows <= 0) return;
  if (a.stats) const_cast<Ctx&>(c).cap_stats_log2 = a.part && attention_tc_supported(c, a);
  if (a.part && attention_tc_supported(c, a)) {
    // algorithmic flops: QK^T + PV over the causally visible keys of each row
    const double vis = double(a.rows) * double(a.pos0) + 0.5 * double(a.rows) * double(a.rows + 1);
    cudaEvent_t kt0 = kt_begin(c, s);
    launch_attention_tc(c, s, conv, layer, a, *a.part);
    kt_end(c, s, kt0, KT_ATTN, 4.0 * c.cfg.hd * double(c.cfg.H) * vis, 0.0);
    return;
  }
  if (attention_decode_supported(c, a)) {
    cudaEvent_t kt0 = kt_begin(c, s);
    launch_attention_decode(c, s, conv, layer, a);
    kt_end(c, s, kt0, KT_ATTN, 4.0 * c.cfg.hd * double(c.cfg.H) * double(a.pos0 + 1), 0.0);
    return;
  }
  PageView pv = page_view(c, conv, layer);
  const float scale = 1.0f / sqrtf(float(c.cfg.hd));
  const size_t smem = sizeof(float) * size_t(c.cfg.hd + a.pos0 + a.rows);
  dim3 grid(unsigned(a.rows), unsigned(c.cfg.H));
  if (c.cfg.dtype == KRUL_BF16) {
    auto k = k_attn_simt<bf16>;
    KB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k<<<grid, 128, smem, s>>>((const bf16*)a.q, a.pos0, pv, c.cfg.H, scale, (bf16*)a.out, a.probs,
                              a.ld_probs, a.probs_row0, a.probs_rows, a.mass, a.mass_rows, a.il,
                              a.rs, a.stats);
  } else {
    auto k = k_attn_simt<float>;
    KB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k<<<grid, 128, smem, s>>>((const float*)a.q, a.pos0, pv, c.cfg.H, scale, (float*)a.out,
                              a.probs, a.ld_probs, a.probs_row0, a.probs_rows, a.mass,
                              a.mass_rows, a.il, a.rs, a.stats);
  }
  KB_LAUNCH();
}

// ---------------------------------------------------------------- K2 probabilities
// The prefill attention probabilities of tracked layer layers[li] for key
// columns [c0, c0 + 64 * gridDim.x), recomputed (never the whole record):
// CTA = (li, kv head g, 64-key block) stages the block's K rows (one page)
// in shared memory as f32 and every thread scores one query row (head of
// the GQA group, prefill row) of the Q saved by the prefill against the 64
// keys. The arithmetic is the attention kernel's own: the dot product in
// the order t = 0..hd-1 and P = exp(s - m) / l (SIMT, f32: bit-identical
// to its capture) or P = exp2(s log2e - m) / l with the ex2 approximation
// (FA, bf16), m and l being the softmax statistics the kernel saved.
template <class T, int HD>
__global__ void __launch_bounds__(256) k_prefill_probs(const T* __restrict__ qsave, const float* __restrict__ stats,
                                                       PageView pv, const int* __restrict__ pt_base,
                                                       int64_t pt_stride, const int* __restrict__ layers, int H,
                                                       int64_t rows, int64_t first_q, int64_t c0, int wc,
                                                       float scale, int log2dom, float* __restrict__ out) {
  __shared__ float ks[64][HD + 1];
  const int li = blockIdx.z, g = blockIdx.y;
  const int64_t k0 = c0 + int64_t(blockIdx.x) * 64;
  const int layer = layers[li];
  pv.pt = pt_base + int64_t(layer) * pt_stride;
  const int64_t kv_total = first_q + rows;
  const int grp = H / pv.Hkv;
  for (int i = threadIdx.x; i < 64 * HD; i += blockDim.x) {
    const int kk = i / HD, t = i % HD;
    const int64_t key = k0 + kk;
    ks[kk][t] = key < kv_total ? tof(reinterpret_cast<const T*>(pv.page(key))[pv.k_off(g, key, t)]) : 0.f;
  }
  __syncthreads();
  const int64_t qd = int64_t(H) * HD;
  for (int64_t qi = threadIdx.x; qi < int64_t(grp) * rows; qi += blockDim.x) {
    const int h = g * grp + int(qi / rows);
    const int64_t r = qi % rows;
    float q[HD];
    const T* qr = qsave + (int64_t(li) * rows + r) * qd + int64_t(h) * HD;
#pragma unroll
    for (int t = 0; t < HD; ++t) q[t] = tof(qr[t]);
    const float m = stats[((int64_t(li) * H + h) * rows + r) * 2];
    const float l = stats[((int64_t(li) * H + h) * rows + r) * 2 + 1];
    const int64_t last = first_q + r;  // causal: keys <= the row's position
    float* o = out + ((int64_t(li) * H + h) * rows + r) * wc + (k0 - c0);
    for (int kk = 0; kk < 64; kk += 4) {
      float pr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float dot = 0.f;
#pragma unroll
        for (int t = 0; t < HD; ++t) dot += q[t] * ks[kk + u][t];
        float pv_ = 0.f;
        if (k0 + kk + u <= last && k0 + kk + u < kv_total) {
          const float sv = __fmul_rn(dot, scale);  // rounded like the kernels' stored scores
          if (log2dom) {
            float e;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(sv - m));
            pv_ = e / l;
          } else {
            pv_ = expf(sv - m) / l;
          }
        }
        pr[u] = pv_;
      }
      *reinterpret_cast<float4*>(o + kk) = make_float4(pr[0], pr[1], pr[2], pr[3]);
    }
  }
}
void launch_prefill_probs(const Ctx& c, cudaStream_t s, const Conv& conv, const int* d_layers, int n,
                          int64_t rows, int64_t first_q, int64_t c0, int wc, float* out) {
  if (n <= 0 || rows <= 0 || wc <= 0) return;
  if (wc % 64 || c0 % 64) fail(KRUL_E_CUDA, "prefill probability chunks must be whole 64-key blocks");
  PageView pv = page_view(c, conv, 0);
  const dim3 grid(unsigned(wc / 64), unsigned(c.cfg.Hkv), unsigned(n));
  const bool lg = c.cap_stats_log2;
  const float scale = lg ? (1.0f / sqrtf(float(c.cfg.hd))) * 1.4426950408889634f : 1.0f / sqrtf(float(c.cfg.hd));
  const float* st = c.cap_stats.as<float>();
#define KB_PP(T, HDV)                                                                                         \
  k_prefill_probs<T, HDV><<<grid, 256, 0, s>>>(static_cast<const T*>(c.cap_q.p), st, pv, conv.d_pt,          \
                                               int64_t(conv.max_pages), d_layers, c.cfg.H, rows, first_q, c0, \
                                               wc, scale, lg ? 1 : 0, out)
  if (c.cfg.dtype == KRUL_BF16 && c.cfg.hd == 128) KB_PP(bf16, 128);
  else if (c.cfg.dtype == KRUL_BF16 && c.cfg.hd == 64) KB_PP(bf16, 64);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 64) KB_PP(float, 64);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 128) KB_PP(float, 128);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 4) KB_PP(float, 4);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 8) KB_PP(float, 8);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 16) KB_PP(float, 16);
  else if (c.cfg.dtype == KRUL_F32 && c.cfg.hd == 32) KB_PP(float, 32);
  else fail(KRUL_E_CONFIG, "estimator prefill recompute: unsupported head_dim");
#undef KB_PP
  KB_LAUNCH();
}

// ---------------------------------------------------------------- FFN pieces (SIMT path)
template <class T>
__global__ void k_bias_act(const float* in, int64_t rows, int64_t F, const float* b1, int kind,
                           T* out) {
  const int64_t n = rows * F;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / F, j = i % F;
    float y;
    if (kind == 0) {
      y = tanhf(in[i] + b1[j]);  // engine.cpp:191
    } else {  // gate/up interleaved per column pair
      const float g = in[r * 2 * F + 2 * j], u = in[r * 2 * F + 2 * j + 1];
      y = g / (1.0f + expf(-g)) * u;
    }
    out[i] = fromf<T>(y);
  }
}
void launch_bias_act(const Ctx& c, cudaStream_t s, const float* in, int64_t rows, int64_t F,
                     const float* b1, int kind, void* out) {
  if (rows <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((rows * F + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16)
    k_bias_act<<<blocks, 256, 0, s>>>(in, rows, F, b1, kind, (bf16*)out);
  else
    k_bias_act<<<blocks, 256, 0, s>>>(in, rows, F, b1, kind, (float*)out);
  KB_LAUNCH();
}

template <class T>
__global__ void k_resid_add(const float* y, const float* bias, const float* resid, int64_t rows,
                            int64_t d, float* out, T* outc) {
  const int64_t n = rows * d;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float v = resid[i] + (bias ? y[i] + bias[i % d] : y[i]);
    out[i] = v;
    if (outc) outc[i] = fromf<T>(v);
  }
}
void launch_resid_add(const Ctx& c, cudaStream_t s, const float* y, const float* bias,
                      const float* resid, int64_t rows, int64_t d, float* out, void* outc) {
  if (rows <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((rows * d + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16)
    k_resid_add<<<blocks, 256, 0, s>>>(y, bias, resid, rows, d, out, (bf16*)outc);
  else
    k_resid_add<<<blocks, 256, 0, s>>>(y, bias, resid, rows, d, out, (float*)outc);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- logits
// engine.cpp:338 / :444 — last row times the unembedding (stored [V][d]).
template <class T>
__global__ void k_logits(const float* h, const T* wT, int d, int V, float* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = blockIdx.x * (blockDim.x >> 5) + warp;
  if (v >= V) return;
  const T* w = wT + int64_t(v) * d;
  float acc = 0.f;
  for (int k = lane; k < d; k += 32) acc += h[k] * tof(w[k]);
  acc = warp_sum(acc);
  if (lane == 0) out[v] = acc;
}
// bf16 fast path (d % 256 == 0, d <= 8192): the last hidden row is staged
// in shared memory once per block; each warp owns one vocabulary row and
// issues all its 16-byte weight loads before the FMAs, so the unembedding
// (V x d bf16 -- 1 GB for Llama-3) streams at HBM rate. This GEMV is the
// last kernel before the first token.
template <int NV>  // 16-byte vectors per lane: d = 256 * NV
__global__ void __launch_bounds__(256) k_logits_vec(const float* __restrict__ h,
                                                    const bf16* __restrict__ wT, int V,
                                                    float* __restrict__ out) {
  constexpr int D = 256 * NV;
  __shared__ __align__(16) float hs[D];
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i < D; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v = blockIdx.x * 8 + warp; v < V; v += gridDim.x * 8) {
    const uint4* w = reinterpret_cast<const uint4*>(wT + int64_t(v) * D);
    uint4 x[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) x[j] = __ldg(w + lane + 32 * j);
    // h as two float4 shared loads per weight vector (the scalar form was an
    // 8-way bank conflict: lanes 32 B apart)
    float acc0 = 0.f, acc1 = 0.f;
    const float4* h4 = reinterpret_cast<const float4*>(hs);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int k4 = (lane + 32 * j) * 2;
      const float4 ha = h4[k4], hb = h4[k4 + 1];
      const uint32_t u[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[0]));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[1]));
      const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[2]));
      const float2 f3 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[3]));
      acc0 += ha.x * f0.x + ha.y * f0.y + ha.z * f1.x + ha.w * f1.y;
      acc1 += hb.x * f2.x + hb.y * f2.y + hb.z * f3.x + hb.w * f3.y;
    }
    float acc = warp_sum(acc0 + acc1);
    if (lane == 0) out[v] = acc;
  }
}
void launch_logits(const Ctx& c, cudaStream_t s, const float* h_last, float* logits) {
  const int V = c.cfg.V;
  const unsigned blocks = unsigned((V + 7) / 8);
  if (c.cfg.dtype == KRUL_BF16 && c.cfg.d % 256 == 0 && (c.cfg.d == 4096 || c.cfg.d == 8192)) {
    // exactly one wave of resident CTAs (grid-stride over the rows): a
    // second partial wave left a third of the GEMV at a third of the SMs
    static int per_sm[2] = {0, 0};
    const int vi = c.cfg.d == 4096 ? 0 : 1;
    if (!per_sm[vi]) {
      if (vi == 0)
        KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], k_logits_vec<16>, 256, 0));
      else
        KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], k_logits_vec<32>, 256, 0));
      per_sm[vi] = std::max(per_sm[vi], 1);
    }
    const unsigned grid =
        unsigned(std::min<int64_t>(blocks, int64_t(c.sm_count > 0 ? c.sm_count : 148) * per_sm[vi]));
    cudaEvent_t kt0 = kt_begin(c, s);
    if (c.cfg.d == 4096)
      KB_CUDA(launch_pdl(k_logits_vec<16>, dim3(grid), dim3(256), 0, s, h_last, (const bf16*)c.unembedT, V, logits));
    else
      KB_CUDA(launch_pdl(k_logits_vec<32>, dim3(grid), dim3(256), 0, s, h_last, (const bf16*)c.unembedT, V, logits));
    KB_LAUNCH();
    kt_end(c, s, kt0, KT_LOGITS, 2.0 * double(V) * c.cfg.d, double(V) * c.cfg.d * 2.0 + double(V) * 4.0);
    return;
  }
  if (c.cfg.dtype == KRUL_BF16)
    k_logits<<<blocks, 256, 0, s>>>(h_last, (const bf16*)c.unembedT, c.cfg.d, V, logits);
  else
    k_logits<<<blocks, 256, 0, s>>>(h_last, (const float*)c.unembedT, c.cfg.d, V, logits);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- weights
// dst[(j * rstride + roff)][i] = src[i][j] (transpose) or dst[i][j] = src[i][j]
template <class T>
__global__ void k_convert(const float* src, T* dst, int64_t rows, int64_t cols, int transpose,
                          int64_t rstride, int64_t roff, int64_t dcols) {
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    if (transpose)
      dst[(j * rstride + roff) * dcols + i] = fromf<T>(src[e]);
    else
      dst[e] = fromf<T>(src[e]);
  }
}
void launch_convert_weights(const Ctx& c, cudaStream_t s, const float* src, void* dst,
                            int64_t rows, int64_t cols, int transpose, int interleave) {
  // interleave: 0 -> plain; 1 -> even rows (gate); 2 -> odd rows (up)
  const int64_t rstride = interleave ? 2 : 1, roff = interleave == 2 ? 1 : 0;
  const unsigned blocks = unsigned(std::min<int64_t>((rows * cols + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16)
    k_convert<<<blocks, 256, 0, s>>>(src, (bf16*)dst, rows, cols, transpose, rstride, roff, rows);
  else
    k_convert<<<blocks, 256, 0, s>>>(src, (float*)dst, rows, cols, transpose, rstride, roff, rows);
  KB_LAUNCH();
}

// Counter-based uniform in [-bound, bound) (splitmix64 of (seed, stream, i));
// perf configs only — parity configs upload the reference UniformStream.
__device__ __forceinline__ float hash_uniform(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return float(uint32_t(z >> 40)) * (1.0f / 16777216.0f);
}
template <class T>
__global__ void k_init(T* dst, int64_t n, uint64_t seed, uint64_t stream, float bound) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = fromf<T>(-bound + 2.f * bound * hash_uniform(seed, stream, uint64_t(i)));
}
void launch_init_uniform(const Ctx& c, cudaStream_t s, void* dst, int64_t n, uint64_t seed,
                         uint64_t stream, float bound) {
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 64));
  if (c.cfg.dtype == KRUL_BF16)
    k_init<<<blocks, 256, 0, s>>>((bf16*)dst, n, seed, stream, bound);
  else
    k_init<<<blocks, 256, 0, s>>>((float*)dst, n, seed, stream, bound);
  KB_LAUNCH();
}
void launch_init_uniform_f32(cudaStream_t s, float* dst, int64_t n, uint64_t seed,
                             uint64_t stream, float bound) {
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 64));
  k_init<<<blocks, 256, 0, s>>>(dst, n, seed, stream, bound);
  KB_LAUNCH();
}

template <class S, class D>
__global__ void k_cvt(const S* src, D* dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = fromf<D>(tof(src[i]));
}
void launch_cvt_to_f32(const Ctx& c, cudaStream_t s, const void* src, float* dst, int64_t n) {
  if (n <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16) k_cvt<<<blocks, 256, 0, s>>>((const bf16*)src, dst, n);
  else k_cvt<<<blocks, 256, 0, s>>>((const float*)src, dst, n);
  KB_LAUNCH();
}
void launch_cvt_from_f32(const Ctx& c, cudaStream_t s, const float* src, void* dst, int64_t n) {
  if (n <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16) k_cvt<<<blocks, 256, 0, s>>>(src, (bf16*)dst, n);
  else k_cvt<<<blocks, 256, 0, s>>>(src, (float*)dst, n);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- KV <-> f32 views
template <class T>
__global__ void k_kv_gather(PageView pv, int64_t start, int64_t rows, float* k, float* v) {
  const int64_t n = int64_t(pv.Hkv) * rows * pv.hd;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int t = int(e % pv.hd);
    const int64_t r = (e / pv.hd) % rows;
    const int g = int(e / (int64_t(pv.hd) * rows));
    const int64_t pos = start + r;
    const T* page = reinterpret_cast<const T*>(pv.page(pos));
    k[e] = tof(page[pv.k_off(g, pos, t)]);
    v[e] = tof(page[pv.v_off(g, pos, t)]);
  }
}
template <class T>
__global__ void k_kv_scatter(PageView pv, int64_t start, int64_t rows, const float* k,
                             const float* v) {
  const int64_t n = int64_t(pv.Hkv) * rows * pv.hd;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int t = int(e % pv.hd);
    const int64_t r = (e / pv.hd) % rows;
    const int g = int(e / (int64_t(pv.hd) * rows));
    const int64_t pos = start + r;
    T* page = reinterpret_cast<T*>(pv.page(pos));
    page[pv.k_off(g, pos, t)] = fromf<T>(k[e]);
    page[pv.v_off(g, pos, t)] = fromf<T>(v[e]);
  }
}
void launch_kv_gather(const Ctx& c, cudaStream_t s, const Conv& conv, int layer, int64_t start,
                      int64_t end, float* k, float* v) {
  const int64_t rows = end - start;
  if (rows <= 0) return;
  PageView pv = page_view(c, conv, layer);
  const unsigned blocks = unsigned(std::min<int64_t>((rows * pv.Hkv * pv.hd + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16) k_kv_gather<bf16><<<blocks, 256, 0, s>>>(pv, start, rows, k, v);
  else k_kv_gather<float><<<blocks, 256, 0, s>>>(pv, start, rows, k, v);
  KB_LAUNCH();
}
void launch_kv_scatter_f32(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                           int64_t start, int64_t end, const float* k, const float* v) {
  const int64_t rows = end - start;
  if (rows <= 0) return;
  PageView pv = page_view(c, conv, layer);
  const unsigned blocks = unsigned(std::min<int64_t>((rows * pv.Hkv * pv.hd + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16) k_kv_scatter<bf16><<<blocks, 256, 0, s>>>(pv, start, rows, k, v);
  else k_kv_scatter<float><<<blocks, 256, 0, s>>>(pv, start, rows, k, v);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- expand (K5)
// kvstore.cpp:316-343 + the splice of scheduler.cpp:368-393: a staged blob
// [K: Hkv][rows][hd] [V: Hkv][rows][hd] covering [blob_start, L) is written
// into `layer`'s pages for positions [from, L). One CTA per (page tile,
// kv head): K rows copy with 16-byte vectors; V is transposed through shared
// memory into the page's V^T block so PV reads stay K-major.
template <class T>
__device__ __forceinline__ void expand_tile(const T* blob, int64_t blob_start, int64_t L,
                                            const PageView& pv, int64_t from, int64_t ti, T* tile) {
  const int hd = pv.hd, Hkv = pv.Hkv;
  const int g = blockIdx.y;
  const int64_t p0 = (from / kPageTokens + ti) * kPageTokens;
  const int64_t lo = p0 > from ? p0 : from, hi = p0 + kPageTokens < L ? p0 + kPageTokens : L;
  if (lo >= hi) return;
  const int64_t rows_blob = L - blob_start;
  const T* kb = blob + (int64_t(g) * rows_blob) * hd;
  const T* vb = blob + (int64_t(Hkv + g) * rows_blob) * hd;
  T* page = reinterpret_cast<T*>(pv.page(lo));
  const int n = int(hi - lo);
  // K: straight row copy (contiguous [rows][hd] on both sides)
  const int64_t krow0 = lo - blob_start;
  T* kdst = page + pv.k_off(g, lo, 0);
  const int elems = n * hd;
  if ((hd * int(sizeof(T))) % 16 == 0) {
    const int vec = 16 / int(sizeof(T));
    const int4* src = reinterpret_cast<const int4*>(kb + krow0 * hd);
    int4* dst = reinterpret_cast<int4*>(kdst);
    for (int i = threadIdx.x; i < elems / vec; i += blockDim.x) dst[i] = src[i];
  } else {
    for (int i = threadIdx.x; i < elems; i += blockDim.x) kdst[i] = kb[krow0 * hd + i];
  }
  // V: stage [n][hd] (16-byte loads; row pitch hd + 2 elements keeps the
  // column reads below spread over the banks), then write V^T [hd][pos%P]
  // as 16-byte runs of 8 consecutive tokens when the span is page-aligned
  const int ldt = hd + 2;
  if (sizeof(T) == 2 && hd % 8 == 0) {
    const int vpr = hd / 8;
    for (int i = threadIdx.x; i < n * vpr; i += blockDim.x) {
      const int r = i / vpr, t8 = (i % vpr) * 8;
      const int4 x = *reinterpret_cast<const int4*>(vb + (krow0 + r) * hd + t8);
      const uint32_t w[4] = {uint32_t(x.x), uint32_t(x.y), uint32_t(x.z), uint32_t(x.w)};
      uint32_t* d = reinterpret_cast<uint32_t*>(tile + r * ldt + t8);
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = w[j];
    }
  } else {
    for (int i = threadIdx.x; i < elems; i += blockDim.x) {
      const int r = i / hd, t = i % hd;
      tile[r * ldt + t] = vb[(krow0 + r) * hd + t];
    }
  }
  __syncthreads();
  if (sizeof(T) == 2 && n == kPageTokens) {
    T* vt = page + pv.v_off(g, lo, 0);  // lo is page-aligned: [hd][64] contiguous
    for (int i = threadIdx.x; i < hd * 8; i += blockDim.x) {
      const int t = i >> 3, c = (i & 7) * 8;
      uint16_t u[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = reinterpret_cast<const uint16_t*>(tile)[(c + j) * ldt + t];
      *reinterpret_cast<uint4*>(vt + t * kPageTokens + c) =
          make_uint4(u[0] | (uint32_t(u[1]) << 16), u[2] | (uint32_t(u[3]) << 16),
                     u[4] | (uint32_t(u[5]) << 16), u[6] | (uint32_t(u[7]) << 16));
    }
  } else {
    for (int i = threadIdx.x; i < hd * n; i += blockDim.x) {
      const int t = i / n, r = i % n;
      page[pv.v_off(g, lo + r, t)] = tile[r * ldt + t];
    }
  }
}
// TMA-staged full page (bf16, every page but a ragged head / tail): the
// blob's K rows [64][hd] and V rows [64][hd] arrive in shared memory by two
// bulk copies (cp.async.bulk, one mbarrier); the K block leaves by one bulk
// store to the page's contiguous K block; V is transposed in shared memory
// (lane = one 32-bit column pair, conflict-free reads) into a [hd][64 + 8]
// tile whose rows leave as hd bulk stores of 128 B (the page's V^T block).
// Returns false when the tile does not qualify (the caller takes the
// vector path): partial page, or a blob source not 16-byte aligned.
constexpr int kExVtPitch = kPageTokens + 8;  // bf16 elements; 144 B rows (16-byte aligned, 2-way stores)
__device__ __forceinline__ uint32_t ex_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ bool expand_tile_tma(const bf16* blob, int64_t blob_start, int64_t L,
                                                const PageView& pv, int64_t from, int64_t ti,
                                                unsigned char* sm, uint32_t& phase) {
  const int hd = pv.hd, Hkv = pv.Hkv;
  const int g = blockIdx.y;
  const int64_t p0 = (from / kPageTokens + ti) * kPageTokens;
  if (p0 < from || p0 + kPageTokens > L || (hd % 8) != 0) return false;
  const int64_t rows_blob = L - blob_start;
  const int64_t krow0 = p0 - blob_start;
  const bf16* ksrc = blob + (int64_t(g) * rows_blob + krow0) * hd;
  const bf16* vsrc = blob + (int64_t(Hkv + g) * rows_blob + krow0) * hd;
  if (((reinterpret_cast<uintptr_t>(ksrc) | reinterpret_cast<uintptr_t>(vsrc)) & 15) != 0) return false;
  const uint32_t bytes = uint32_t(kPageTokens) * hd * 2;
  bf16* kbuf = reinterpret_cast<bf16*>(sm);
  bf16* vbuf = kbuf + kPageTokens * hd;
  bf16* vt = vbuf + kPageTokens * hd;  // [hd][kExVtPitch]
  uint64_t* bar = reinterpret_cast<uint64_t*>(vt + hd * kExVtPitch);
  bf16* page = reinterpret_cast<bf16*>(pv.page(p0));
  bf16* kdst = page + pv.k_off(g, p0, 0);
  bf16* vdst = page + pv.v_off(g, p0, 0);  // [hd][64] contiguous
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ex_smem_u32(bar)),
                 "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ex_smem_u32(kbuf)), "l"(ksrc), "r"(bytes), "r"(ex_smem_u32(bar)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ex_smem_u32(vbuf)), "l"(vsrc), "r"(bytes), "r"(ex_smem_u32(bar)) : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "EXW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra EXD_%=;\n\t"
      "bra EXW_%=;\n"
      "EXD_%=:\n\t}" ::"r"(ex_smem_u32(bar)), "r"(phase) : "memory");
  phase ^= 1u;
  if (threadIdx.x == 0)  // K: the staged block is the page's K block
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(kdst), "r"(ex_smem_u32(kbuf)), "r"(bytes) : "memory");
  // V^T: work item = (column pair, 8-row group); a warp's 32 lanes read 32
  // consecutive 32-bit words of one row -> 32 distinct banks
  const uint32_t* vw = reinterpret_cast<const uint32_t*>(vbuf);
  const int cp = hd / 2;
  for (int i = threadIdx.x; i < cp * (kPageTokens / 8); i += blockDim.x) {
    const int c2 = i % cp, r8 = (i / cp) * 8;
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = vw[(r8 + j) * cp + c2];
    uint4 lo, hi;
    lo.x = (w[0] & 0xffffu) | (w[1] << 16); lo.y = (w[2] & 0xffffu) | (w[3] << 16);
    lo.z = (w[4] & 0xffffu) | (w[5] << 16); lo.w = (w[6] & 0xffffu) | (w[7] << 16);
    hi.x = (w[0] >> 16) | (w[1] & 0xffff0000u); hi.y = (w[2] >> 16) | (w[3] & 0xffff0000u);
    hi.z = (w[4] >> 16) | (w[5] & 0xffff0000u); hi.w = (w[6] >> 16) | (w[7] & 0xffff0000u);
    *reinterpret_cast<uint4*>(vt + (2 * c2) * kExVtPitch + r8) = lo;
    *reinterpret_cast<uint4*>(vt + (2 * c2 + 1) * kExVtPitch + r8) = hi;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  for (int t = threadIdx.x; t < hd; t += blockDim.x)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(vdst + int64_t(t) * kPageTokens), "r"(ex_smem_u32(vt + t * kExVtPitch)),
                 "r"(uint32_t(kPageTokens * 2)) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before smem reuse / exit
  return true;
}
__host__ __device__ inline size_t expand_tma_smem(int hd) {
  return size_t(2) * kPageTokens * hd * 2 + size_t(hd) * kExVtPitch * 2 + 16;
}

// One CTA per (page tile, kv head), or a CTA-capped grid-stride loop over
// the tiles (KRUL_EXPAND_CTAS) so the scatter leaves SMs to the recompute.
template <class T>
__global__ void k_expand(const T* blob, int64_t blob_start, int64_t L, PageView pv, int64_t from,
                         int64_t tiles) {
  extern __shared__ __align__(128) unsigned char smraw[];
  T* tile = reinterpret_cast<T*>(smraw);  // [kPageTokens][hd + pad]
  uint32_t phase = 0;
  if constexpr (sizeof(T) == 2) {
    if (threadIdx.x == 0) {
      uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + expand_tma_smem(pv.hd) - 16);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ex_smem_u32(bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  for (int64_t ti = blockIdx.x; ti < tiles; ti += gridDim.x) {
    bool done = false;
    if constexpr (sizeof(T) == 2)
      done = expand_tile_tma(reinterpret_cast<const bf16*>(blob), blob_start, L, pv, from, ti, smraw, phase);
    if (!done) expand_tile(blob, blob_start, L, pv, from, ti, tile);
    __syncthreads();
  }
}

// K4b + K5 fused (coded store, hd = 128): with hd equal to a lane's
// 128-element stream, lane j of a 4096-element chunk holds exactly one blob
// row -- token blob_start + r of head g, K or V -- and writes it straight
// into the owners' pages: K rows as one 32-byte store per 16 elements (full
// L2 sectors), V^T columns as per-dimension stores contiguous across the
// warp's 32 consecutive tokens. No raw staging round trip, one launch per
// blob.
//
// Sized to share SMs with the restore's other kernels (the GEMM / attention
// CTAs hold ~225 KB of shared memory each): no shared memory at all -- the
// 8 KB decode LUT and the exponent words are read through L1 (__ldg) --
// and a small CTA (128 threads), so the decode CTAs co-reside with them
// instead of queueing behind them. A persistent grid walks the chunks; every warp
// decodes two chunks at once (two independent bit-stream chains per lane:
// the LUT lookup latency of one chain hides behind the other).
struct EcLane {  // one lane's position in its chunk's exponent stream + its row's destinations
  uint32_t wa, wb, wc, bo;
  const uint32_t* wp;  // the word after wc
  const uint4* smv;    // the row's sign+mantissa bytes
  uint16_t *d0, *d1;   // the row in each owner's page (K row / V^T column), null = not written
  bool isv;
};
__device__ __forceinline__ void ec_lane_init(EcLane& st, const uint8_t* blob, const EcHeader& h, int64_t ch,
                                             int lane, int64_t rows, const PageView& pv0, const PageView& pv1,
                                             int64_t blob_start, int64_t from0, int64_t from1, int n_owners) {
  const uint32_t* base_t = reinterpret_cast<const uint32_t*>(blob + h.base_off);
  const uint8_t* cnt_t = blob + h.cnt_off;
  const uint32_t* ex = reinterpret_cast<const uint32_t*>(blob + h.exp_off);
  const uint32_t base = __ldg(base_t + ch);
  const uint32_t c = __ldg(cnt_t + ch * 32 + lane);
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const uint32_t* w = ex + base + (inc - c);
  st.wa = __ldg(w);
  st.wb = __ldg(w + 1);
  st.wc = __ldg(w + 2);  // the image ends with a pad word past the last stream; a third read stays inside
  st.wp = w + 3;
  st.bo = 0;
  const int64_t nrows = int64_t(h.n_elems) / 128;
  const int64_t R = ch * 32 + lane;  // flattened (kv, g, r) row of this lane
  const bool live = R < nrows;
  const int64_t r = live ? R % rows : 0;
  const int64_t hg = live ? R / rows : 0;
  const int Hkv = pv0.Hkv;
  st.isv = hg >= Hkv;
  const int g = int(hg % Hkv);
  const int64_t pos = blob_start + r;
  st.smv = reinterpret_cast<const uint4*>(blob + h.sm_off + R * 128);
  auto dst = [&](const PageView& pv) {
    uint16_t* page = reinterpret_cast<uint16_t*>(pv.page(pos));
    return page + (st.isv ? pv.v_off(g, pos, 0) : pv.k_off(g, pos, 0));
  };
  st.d0 = live && pos >= from0 ? dst(pv0) : nullptr;
  st.d1 = live && n_owners > 1 && pos >= from1 ? dst(pv1) : nullptr;
  if (!live) st.smv = nullptr;
}
__device__ __forceinline__ uint32_t ec_next(EcLane& st, const uint16_t* __restrict__ lut) {
  const uint32_t win = __funnelshift_l(st.wb, st.wa, st.bo);
  const uint32_t e = __ldg(lut + (win >> (32 - kEcMaxLen)));
  st.bo += e >> 8;
  if (st.bo >= 32) {  // next word; the one after it is already in flight
    st.bo -= 32;
    st.wa = st.wb;
    st.wb = st.wc;
    st.wc = __ldg(st.wp++);
  }
  return e;
}
__device__ __forceinline__ void ec_store16(const EcLane& st, const uint32_t (&o)[8], int gq) {
#pragma unroll
  for (int ow = 0; ow < 2; ++ow) {
    uint16_t* d = ow == 0 ? st.d0 : st.d1;
    if (!d) continue;
    if (!st.isv) {  // one 32-byte store per lane (STG.256): whole L2 sectors
      asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d + 16 * gq), "r"(o[0]),
                   "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                   : "memory");
    } else {
      uint16_t* vt = d + int64_t(16 * gq) * kPageTokens;
#pragma unroll
      for (int k = 0; k < 16; ++k) vt[k * kPageTokens] = uint16_t(o[k >> 1] >> (16 * (k & 1)));
    }
  }
}
__global__ void __launch_bounds__(128, 4) k_ec_decode_expand(const uint8_t* __restrict__ blob,
                                                             const uint16_t* __restrict__ lut,
                                                             int64_t blob_start, int64_t rows, PageView pv0,
                                                             int64_t from0, PageView pv1, int64_t from1,
                                                             int n_owners) {
  const EcHeader h = *reinterpret_cast<const EcHeader*>(blob);
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t wid = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t ch = 2 * wid; ch < h.n_chunks; ch += 2 * warps) {
    EcLane a, b;
    ec_lane_init(a, blob, h, ch, lane, rows, pv0, pv1, blob_start, from0, from1, n_owners);
    if (ch + 1 < h.n_chunks) {
      ec_lane_init(b, blob, h, ch + 1, lane, rows, pv0, pv1, blob_start, from0, from1, n_owners);
    } else {
      b = a;
      b.smv = nullptr;
      b.d0 = b.d1 = nullptr;
    }
#pragma unroll 1
    for (int gq = 0; gq < 8; ++gq) {  // 16 elements per group and chain
      const uint4 sa = a.smv ? __ldg(a.smv + gq) : make_uint4(0, 0, 0, 0);
      const uint4 sb = b.smv ? __ldg(b.smv + gq) : make_uint4(0, 0, 0, 0);
      uint32_t oa[8], ob[8];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t ea = ec_next(a, lut);
        const uint32_t eb = ec_next(b, lut);
        // bf16 = sign | exponent | 7 mantissa bits; the byte plane holds sign + mantissa
        const uint32_t wa = k < 4 ? sa.x : k < 8 ? sa.y : k < 12 ? sa.z : sa.w;
        const uint32_t wb = k < 4 ? sb.x : k < 8 ? sb.y : k < 12 ? sb.z : sb.w;
        const uint32_t ya = (wa >> (8 * (k & 3))) & 0xFFu, yb = (wb >> (8 * (k & 3))) & 0xFFu;
        const uint32_t va = ((ya & 0x80u) << 8) | ((ea & 0xFFu) << 7) | (ya & 0x7Fu);
        const uint32_t vb = ((yb & 0x80u) << 8) | ((eb & 0xFFu) << 7) | (yb & 0x7Fu);
        if (k & 1) {
          oa[k >> 1] |= va << 16;
          ob[k >> 1] |= vb << 16;
        } else {
          oa[k >> 1] = va;
          ob[k >> 1] = vb;
        }
      }
      ec_store16(a, oa, gq);
      ec_store16(b, ob, gq);
    }
  }
}
void launch_ec_decode_expand(const Ctx& c, cudaStream_t s, const void* blob, int64_t n_chunks,
                             const uint16_t* lut, int64_t blob_start, int64_t L, const Conv& conv,
                             const int* owners, const int64_t* from, double coded_bytes, int ctas_per_sm) {
  if (n_chunks <= 0) return;
  const int no = owners[1] >= 0 ? 2 : 1;
  const PageView pv0 = page_view(c, conv, owners[0]);
  const PageView pv1 = no > 1 ? page_view(c, conv, owners[1]) : pv0;
  // persistent: 4 CTAs (128 registers x 128 threads) per SM, two chunks per warp and pass
  const int sms = c.sm_count > 0 ? c.sm_count : 148;
  const int cps = std::max(1, std::min(4, ctas_per_sm));
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((n_chunks + 7) / 8, int64_t(sms) * cps)));
  cudaEvent_t kt0 = kt_begin(c, s);
  k_ec_decode_expand<<<blocks, 128, 0, s>>>(static_cast<const uint8_t*>(blob), lut, blob_start, L - blob_start,
                                            pv0, from[0], pv1, no > 1 ? from[1] : L, no);
  KB_LAUNCH();
  // algorithmic bytes: the coded image read once + every owner's pages written
  double bytes = coded_bytes;
  for (int i = 0; i < no; ++i) bytes += 2.0 * double(L - from[i]) * c.cfg.Hkv * c.cfg.hd * 2.0;
  kt_end(c, s, kt0, KT_DECODE_EXPAND, 0.0, bytes);
}

void launch_expand_impl(const Ctx& c, cudaStream_t s, const void* blob, int64_t blob_start, int64_t L,
                        const Conv& conv, int layer, int64_t from);
void launch_expand(const Ctx& c, cudaStream_t s, const void* blob, int64_t blob_start, int64_t L,
                   const Conv& conv, int layer, int64_t from) {
  if (from >= L) return;
  cudaEvent_t kt0 = kt_begin(c, s);
  launch_expand_impl(c, s, blob, blob_start, L, conv, layer, from);
  // bytes: the K and V rows read from the staged blob and written to pages
  kt_end(c, s, kt0, KT_EXPAND, 0.0, 2.0 * 2.0 * double(L - from) * c.cfg.Hkv * c.cfg.hd * double(c.esz));
}
void launch_expand_impl(const Ctx& c, cudaStream_t s, const void* blob, int64_t blob_start, int64_t L,
                        const Conv& conv, int layer, int64_t from) {
  PageView pv = page_view(c, conv, layer);
  const int64_t tiles = (L - 1) / kPageTokens - from / kPageTokens + 1;
  dim3 grid(unsigned(tiles), unsigned(c.cfg.Hkv));
  static const int cap = [] {
    const char* v = std::getenv("KRUL_EXPAND_CTAS");
    return v ? std::atoi(v) : 0;
  }();
  if (cap > 0) grid.x = unsigned(std::min<int64_t>(tiles, std::max(1, cap / int(c.cfg.Hkv))));
  size_t smem = size_t(kPageTokens) * (c.cfg.hd + 2) * c.esz + 16;
  if (c.cfg.dtype == KRUL_BF16) {
    smem = std::max(smem, expand_tma_smem(c.cfg.hd));
    KB_CUDA(cudaFuncSetAttribute(k_expand<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    k_expand<bf16><<<grid, 256, smem, s>>>((const bf16*)blob, blob_start, L, pv, from, tiles);
  } else {
    KB_CUDA(cudaFuncSetAttribute(k_expand<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    k_expand<float><<<grid, 256, smem, s>>>((const float*)blob, blob_start, L, pv, from, tiles);
  }
  KB_LAUNCH();
}

// ---------------------------------------------------------------- compress (K8)
// kvstore.cpp:243-314: blob rows = deep member over [blob_start, L); with
// the mean merge, rows [merge_from, L) become 0.5f * (shallow + deep).
template <class T>
__global__ void k_compress(PageView deep, PageView shal, int use_shallow, int64_t blob_start,
                           int64_t L, int64_t merge_from, T* blob) {
  const int hd = deep.hd, Hkv = deep.Hkv;
  const int64_t rows = L - blob_start;
  const int64_t n = int64_t(Hkv) * rows * hd;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int t = int(e % hd);
    const int64_t r = (e / hd) % rows;
    const int g = int(e / (int64_t(hd) * rows));
    const int64_t pos = blob_start + r;
    const T* dp = reinterpret_cast<const T*>(deep.page(pos));
    float k = tof(dp[deep.k_off(g, pos, t)]);
    float v = tof(dp[deep.v_off(g, pos, t)]);
    if (use_shallow && pos >= merge_from) {
      const T* sp = reinterpret_cast<const T*>(shal.page(pos));
      k = 0.5f * (tof(sp[shal.k_off(g, pos, t)]) + k);
      v = 0.5f * (tof(sp[shal.v_off(g, pos, t)]) + v);
    }
    blob[e] = fromf<T>(k);
    blob[n + e] = fromf<T>(v);
  }
}
void launch_compress(const Ctx& c, cudaStream_t s, const Conv& conv, int deep, int shallow,
                     int64_t blob_start, int64_t L, int64_t merge_from, void* blob) {
  const int64_t rows = L - blob_start;
  if (rows <= 0) return;
  PageView dp = page_view(c, conv, deep);
  PageView sp = page_view(c, conv, shallow >= 0 ? shallow : deep);
  const unsigned blocks =
      unsigned(std::min<int64_t>((rows * c.cfg.Hkv * c.cfg.hd + 255) / 256, 65535));
  if (c.cfg.dtype == KRUL_BF16)
    k_compress<<<blocks, 256, 0, s>>>(dp, sp, shallow >= 0, blob_start, L, merge_from,
                                      (bf16*)blob);
  else
    k_compress<<<blocks, 256, 0, s>>>(dp, sp, shallow >= 0, blob_start, L, merge_from,
                                      (float*)blob);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- estimator (K1/K2)
// Pair p enumerates (a < b) over the sorted tracked layers, as
// analysis.cpp:84-93. Stage 1: one CTA per (head, column chunk) loads the
// chunk of every tracked layer's row into shared memory once (coalesced
// 128-bit loads) and one warp per pair reduces sum((f32 a - f32 b)^2) in
// double (analysis.cpp:146-147) with warp shuffles. Stage 2 adds the chunk
// partials in a fixed order (deterministic, no fp atomics).
// Estimator fold as a per-head Gram matrix on the FP64 tensor path.
// For every tracked pair (a, b) and head h the reference accumulates
// sum_w (A_a - A_b)^2 (decode: analysis.cpp:146-147; prefill: the expanded
// sum a^2 + sum b^2 - 2 sum ab of analysis.hpp:37-50). Both equal
// G_aa + G_bb - 2 G_ab with G = R R^T, R = the tracked layers' rows of head
// h. G is computed with mma.sync.m8n8k4 f64 over 8x8 layer tiles: the f32
// probabilities are widened once per element (not once per pair), products
// are exact in f64 and accumulation is f64, so the prefill fold is the
// reference's expanded form up to summation order and the decode fold
// differs from the reference's f32-rounded difference by <= 2^-23 relative
// per term. Stage 1: one CTA per (column chunk, head) stages the chunk of
// every tracked row in shared memory (the only HBM read), each warp owns a
// set of upper-triangle 8x8 tiles, and the CTA writes the chunk's packed
// upper-triangle Gram [n(n+1)/2]. Stage 2 sums the chunks in fixed order
// (deterministic, no fp atomics) and folds G into the [pair][head] sums.
constexpr int kGramPitch = kFoldChunk + 4;  // f64 row pitch: fragment loads spread over banks
constexpr int kGramThreads = 256;
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(kGramThreads) k_fold_gram(
    const float* __restrict__ rows, int64_t layer_stride, int64_t head_stride, int64_t total, int H,
    const int* layers, int n, int chunks_per_cta, double* __restrict__ partial) {
  extern __shared__ double R[];  // [n8][kGramPitch] then G [n8][n8]
  const int n8 = (n + 7) & ~7;
  double* G = R + n8 * kGramPitch;
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = n8 / 8, ntiles = T * (T + 1) / 2;
  constexpr int kMaxTilesPerWarp = 7;  // 55 tiles (80 layers) over 8 warps
  double acc[kMaxTilesPerWarp][2];
#pragma unroll
  for (int j = 0; j < kMaxTilesPerWarp; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int cc = 0; cc < chunks_per_cta; ++cc) {
  const int64_t c0 = (int64_t(blockIdx.x) * chunks_per_cta + cc) * kFoldChunk;
  if (c0 >= total) break;
  const int cw = int(total - c0 < kFoldChunk ? total - c0 : kFoldChunk);
  __syncthreads();  // the previous chunk's fragments have been consumed
  // thread -> 4 consecutive columns of rows q, q + 4, q + 8, ...; batches of
  // 8 independent 16-byte loads in flight (a store-after-load loop would
  // serialise one HBM round trip per row)
  {
    const int c4 = (threadIdx.x & 63) * 4, q = threadIdx.x >> 6;
    const bool vec = cw == kFoldChunk && ((reinterpret_cast<uintptr_t>(rows) | layer_stride | head_stride) & 3) == 0;
    for (int a0 = q; a0 < n8; a0 += 32) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int a = a0 + 4 * u;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a < n) {
          const float* src = rows + int64_t(layers[a]) * layer_stride + int64_t(h) * head_stride + c0 + c4;
          if (vec) {
            v[u] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            v[u].x = c4 < cw ? __ldg(src) : 0.f;
            v[u].y = c4 + 1 < cw ? __ldg(src + 1) : 0.f;
            v[u].z = c4 + 2 < cw ? __ldg(src + 2) : 0.f;
            v[u].w = c4 + 3 < cw ? __ldg(src + 3) : 0.f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int a = a0 + 4 * u;
        if (a < n8) {
          double* d = R + a * kGramPitch + c4;
          d[0] = v[u].x;
          d[1] = v[u].y;
          d[2] = v[u].z;
          d[3] = v[u].w;
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kMaxTilesPerWarp; ++j) {
    const int t = warp + j * (kGramThreads / 32);
    if (t >= ntiles) break;
    int I = 0, rem = t;  // t -> (I <= J)
    while (rem >= T - I) {
      rem -= T - I;
      ++I;
    }
    const int J = I + rem;
    const double* ra = R + (I * 8 + (lane >> 2)) * kGramPitch + (lane & 3);
    const double* rb = R + (J * 8 + (lane >> 2)) * kGramPitch + (lane & 3);
#pragma unroll 8
    for (int k = 0; k < kFoldChunk; k += 4) dmma_8x8x4(acc[j][0], acc[j][1], ra[k], rb[k]);
  }
  }  // chunk loop
#pragma unroll
  for (int j = 0; j < kMaxTilesPerWarp; ++j) {
    const int t = warp + j * (kGramThreads / 32);
    if (t >= ntiles) break;
    int I = 0, rem = t;
    while (rem >= T - I) {
      rem -= T - I;
      ++I;
    }
    const int J = I + rem;
    const int gr = I * 8 + (lane >> 2), gc = J * 8 + (lane & 3) * 2;
    G[gr * n8 + gc] = acc[j][0];
    G[gr * n8 + gc + 1] = acc[j][1];
  }
  __syncthreads();
  const int NE = n * (n + 1) / 2;
  double* out = partial + (int64_t(blockIdx.x) * H + h) * NE;
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    int a = 0, rem = e;  // packed upper triangle incl. diagonal, row-major
    while (rem >= n - a) {
      rem -= n - a;
      ++a;
    }
    out[e] = G[a * n8 + a + rem];
  }
}
__device__ __forceinline__ int gram_idx(int n, int a, int b) {  // a <= b
  return a * n - a * (a - 1) / 2 + (b - a);
}
// Stage 2a: fixed-order sums of the per-chunk Gram entries (one thread per
// (head, entry), all chunk loads in flight; deterministic, no fp atomics).
__global__ void k_fold_gsum(const double* __restrict__ partial, int groups, int NE, int H,
                            double* __restrict__ gsum) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // = h * NE + e
  if (i >= int64_t(H) * NE) return;
  const int h = int(i / NE), e = int(i % NE);
  double acc = 0.0;
  for (int g0 = 0; g0 < groups; g0 += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      v[u] = g0 + u < groups ? partial[(int64_t(g0 + u) * H + h) * NE + e] : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += v[u];
  }
  gsum[i] = acc;
}
// Stage 2b: sums[p][h] += max(0, G_aa + G_bb - 2 G_ab) (clamp: analysis.hpp:49).
__global__ void k_fold_pairs(const double* __restrict__ gsum, int n, int H, double* sums) {
  const int P = n * (n - 1) / 2, NE = n * (n + 1) / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // = p * H + h (sums layout)
  if (i >= P * H) return;
  const int p = i / H, h = i % H;
  int a = 0, rem = p;  // p -> (a, b), a < b, analysis.cpp:84-93 order
  while (rem >= n - 1 - a) {
    rem -= n - 1 - a;
    ++a;
  }
  const int b = a + 1 + rem;
  const double* g = gsum + int64_t(h) * NE;
  const double v = g[gram_idx(n, a, a)] + g[gram_idx(n, b, b)] - 2.0 * g[gram_idx(n, a, b)];
  sums[i] += v > 0.0 ? v : 0.0;
}
static void fold_common(cudaStream_t s, const float* rows, int64_t layer_stride,
                        int64_t head_stride, int64_t total, int H, const int* d_layers, int n,
                        double* sums, double* partial, int64_t partial_cap) {
  if (n < 2 || total <= 0) return;
  const int P = n * (n - 1) / 2, NE = n * (n + 1) / 2;
  const int chunks = int((total + kFoldChunk - 1) / kFoldChunk);
  const int n8 = (n + 7) & ~7;
  if ((n8 / 8) * (n8 / 8 + 1) / 2 > 8 * 7) fail(KRUL_E_CONFIG, "too many tracked layers for the estimator fold");
  // chunk groups: enough CTAs (groups x heads) for ~2 per SM, each CTA
  // accumulating its chunks' Gram tiles in registers
  // chunk groups: ~2 CTAs (groups x heads) per SM, each CTA accumulating its
  // chunks' Gram tiles in registers (measured: 1 chunk per CTA is 1.8x slower)
  const int groups = std::max(1, std::min(chunks, (2 * 148 + H - 1) / H));
  const int per = (chunks + groups - 1) / groups;
  const int g_used = (chunks + per - 1) / per;
  if (int64_t(g_used + 1) * NE * H > partial_cap) fail(KRUL_E_CUDA, "fold partial buffer too small");
  const size_t smem = (size_t(n8) * kGramPitch + size_t(n8) * n8) * sizeof(double);
  if (smem > 227 * 1024) fail(KRUL_E_CONFIG, "too many tracked layers for the estimator fold");
  static int smem_set = 0;  // raise the opt-in limit once (host call, not per fold)
  if (int(smem) > smem_set) {
    KB_CUDA(cudaFuncSetAttribute(k_fold_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    smem_set = int(smem);
  }
  k_fold_gram<<<dim3(unsigned(g_used), unsigned(H)), kGramThreads, smem, s>>>(
      rows, layer_stride, head_stride, total, H, d_layers, n, per, partial);
  KB_LAUNCH();
  // the chunk sums land after the chunk partials in the same scratch
  double* gsum = partial + int64_t(g_used) * NE * H;
  k_fold_gsum<<<unsigned((int64_t(H) * NE + 255) / 256), 256, 0, s>>>(partial, g_used, NE, H, gsum);
  KB_LAUNCH();
  k_fold_pairs<<<unsigned((P * H + 255) / 256), 256, 0, s>>>(gsum, n, H, sums);
  KB_LAUNCH();

}
void launch_fold_decode(cudaStream_t s, const float* rows, int64_t W, int H, const int* d_layers,
                        int n, double* sums, double* partial, int64_t partial_cap) {
  fold_common(s, rows, int64_t(H) * W, W, W, H, d_layers, n, sums, partial, partial_cap);
}
// Prefill fold over the full [rows x W] rectangle per (pair, head): the
// direct sum of squared differences in double; the reference's expanded
// a^2 + b^2 - 2ab form (analysis.hpp:37-50) agrees within 1e-12 relative.
void launch_fold_prefill(cudaStream_t s, const float* probs, int64_t rows, int64_t W, int H,
                         const int* d_layers, int n, double* sums, double* partial,
                         int64_t partial_cap) {
  fold_common(s, probs, int64_t(H) * rows * W, rows * W, rows * W, H, d_layers, n, sums,
                    partial, partial_cap);
}

// analysis.cpp:153-179 — D(i,j) = mean over heads of sqrt(sums).
__global__ void k_finalize(const double* sums, int n, int H, double* D) {
  const int P = n * (n - 1) / 2;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) D[i] = 0.0;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int a = 0, rem = p;
    while (rem >= n - 1 - a) {
      rem -= n - 1 - a;
      ++a;
    }
    const int b = a + 1 + rem;
    double m = 0.0;
    for (int h = 0; h < H; ++h) m += sqrt(sums[int64_t(p) * H + h]);
    m /= double(H);
    D[a * n + b] = m;
    D[b * n + a] = m;
  }
}
void launch_finalize(cudaStream_t s, const double* sums, int n, int H, double* D) {
  k_finalize<<<1, 256, 0, s>>>(sums, n, H, D);
  KB_LAUNCH();
}

// ---------------------------------------------------------------- selector (K3)
// strategy.cpp:44-69: candidates sorted lexicographically by (d, i, j) with a
// shared-memory bitonic sort, then one thread walks the ranking accepting
// disjoint pairs until |shared| >= quota. Bit-exact with std::sort + the
// greedy loop on identical D (a strict total order on distinct (i, j)).
__device__ __forceinline__ bool cand_less(double da, int ia, int ja, double db, int ib, int jb) {
  if (da != db) return da < db;
  if (ia != ib) return ia < ib;
  return ja < jb;
}
__global__ void k_select(const double* cd, const int* ci, const int* cj, int n_cand, int cap,
                         int quota, int* out_i, int* out_j, double* out_d, int* out_n) {
  extern __shared__ unsigned char sraw[];
  double* d = reinterpret_cast<double*>(sraw);
  int* I = reinterpret_cast<int*>(d + cap);
  int* J = I + cap;
  for (int t = threadIdx.x; t < cap; t += blockDim.x) {
    if (t < n_cand) {
      d[t] = cd[t];
      I[t] = ci[t];
      J[t] = cj[t];
    } else {
      d[t] = INFINITY;
      I[t] = 0x7fffffff;
      J[t] = 0x7fffffff;
    }
  }
  __syncthreads();
  for (int k = 2; k <= cap; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < cap; t += blockDim.x) {
        const int u = t ^ j;
        if (u > t) {
          const bool up = (t & k) == 0;
          const bool gt = cand_less(d[u], I[u], J[u], d[t], I[t], J[t]);
          if (gt == up) {
            const double td = d[t]; d[t] = d[u]; d[u] = td;
            const int ti = I[t]; I[t] = I[u]; I[u] = ti;
            const int tj = J[t]; J[t] = J[u]; J[u] = tj;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long taken[4] = {0, 0, 0, 0};  // layers < 256
    int shared = 0, np = 0;
    for (int t = 0; t < n_cand; ++t) {
      if (shared >= quota) break;
      const int i = I[t], j = J[t];
      const bool ti = (taken[i >> 6] >> (i & 63)) & 1ull;
      const bool tj = (taken[j >> 6] >> (j & 63)) & 1ull;
      if (ti || tj) continue;
      taken[i >> 6] |= 1ull << (i & 63);
      taken[j >> 6] |= 1ull << (j & 63);
      out_i[np] = i;
      out_j[np] = j;
      out_d[np] = d[t];
      ++np;
      shared += 2;
    }
    *out_n = np;
  }
}
void launch_select(cudaStream_t s, const double* cand_d, const int* cand_i, const int* cand_j,
                   int n_cand, int quota, int* out_i, int* out_j, double* out_d, int* out_n) {
  int cap = 1;
  while (cap < n_cand) cap <<= 1;
  const size_t smem = size_t(cap) * (sizeof(double) + 2 * sizeof(int));
  KB_CUDA(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  k_select<<<1, 1024, smem, s>>>(cand_d, cand_i, cand_j, n_cand, cap, quota, out_i, out_j, out_d,
                                 out_n);
  KB_LAUNCH();
}

}  // namespace kb
