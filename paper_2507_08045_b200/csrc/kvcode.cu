// kvcode.cu — lossless exponent coding of the bf16 KV store (the load
// stream's bytes). B200-native extension of kvstore.cpp's snapshot: the
// restore is PCIe-bound (H2D at 99% of a measured pinned copy), and the 8
// exponent bits of a bf16 KV element carry ~2.6 bits of entropy (Gaussian-
// like values span a few binades), so each element is stored as its raw
// sign+mantissa byte plus a Huffman-coded exponent (~10.6 of 16 bits). The
// restored KV is bit-identical to the uncoded store; the decode runs on the
// expand stream between the blob's H2D copy and its scatter into the pages.
//
// Coded blob image: see kvcode.hpp. Elements are cut into chunks of 4096
// (one warp); lane j codes the chunk's elements [128 j, 128 j + 128) MSB-first
// into its own run of 32-bit words (<= 48), so a warp decodes a chunk with 32
// independent bit streams. Codes are canonical Huffman, length <= 12: one
// 4096-entry LUT (symbol | length << 8) in shared memory decodes a symbol
// per lookup. The decoder stages the chunk's words in shared memory
// (coalesced), reads its 12-bit window with one funnel shift, and writes 16
// decoded elements (32 B) per vector store.
#include "kb.hpp"
#include "kvcode.hpp"

namespace kb {

__global__ void k_exp_hist(const uint16_t* __restrict__ x, int64_t n, unsigned long long* hist) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t n4 = n / 4;
  const uint2* x4 = reinterpret_cast<const uint2*>(x);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const uint2 v = __ldg(x4 + i);
    atomicAdd(&h[(v.x >> 7) & 0xFF], 1u);
    atomicAdd(&h[(v.x >> 23) & 0xFF], 1u);
    atomicAdd(&h[(v.y >> 7) & 0xFF], 1u);
    atomicAdd(&h[(v.y >> 23) & 0xFF], 1u);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(&h[(x[i] >> 7) & 0xFF], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, (unsigned long long)h[i]);
}

// words per (chunk, lane) stream
__global__ void k_ec_lane_words(const uint16_t* __restrict__ x, int64_t n, const uint8_t* __restrict__ len,
                                uint32_t* __restrict__ words) {
  __shared__ uint8_t sl[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sl[i] = len[i];
  __syncthreads();
  const int64_t streams = (n + kEcLaneSyms - 1) / kEcLaneSyms;
  const int64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < chunks * 32;
       t += int64_t(gridDim.x) * blockDim.x) {
    uint32_t bits = 0;
    if (t < streams) {
      const int64_t e0 = t * kEcLaneSyms;
      const int cnt = int(n - e0 < kEcLaneSyms ? n - e0 : kEcLaneSyms);
      for (int j = 0; j < cnt; ++j) bits += sl[(x[e0 + j] >> 7) & 0xFF];
    }
    words[t] = (bits + 31) / 32;
  }
}

__global__ void k_ec_encode(const uint16_t* __restrict__ x, int64_t n, const uint32_t* __restrict__ code,
                            const uint8_t* __restrict__ len, const uint32_t* __restrict__ lane_off,
                            uint8_t* __restrict__ sm, uint32_t* __restrict__ ex) {
  __shared__ uint32_t sc[256];
  __shared__ uint8_t sl[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    sc[i] = code[i];
    sl[i] = len[i];
  }
  __syncthreads();
  const int64_t streams = (n + kEcLaneSyms - 1) / kEcLaneSyms;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < streams;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e0 = t * kEcLaneSyms;
    const int cnt = int(n - e0 < kEcLaneSyms ? n - e0 : kEcLaneSyms);
    uint32_t* out = ex + lane_off[t];
    uint64_t acc = 0;
    int nb = 0;
    for (int j = 0; j < cnt; ++j) {
      const uint32_t v = x[e0 + j];
      sm[e0 + j] = uint8_t(((v >> 8) & 0x80u) | (v & 0x7Fu));
      const uint32_t e = (v >> 7) & 0xFF;
      const int l = sl[e];
      acc |= uint64_t(sc[e]) << (64 - nb - l);
      nb += l;
      if (nb >= 32) {
        *out++ = uint32_t(acc >> 32);
        acc <<= 32;
        nb -= 32;
      }
    }
    if (nb > 0) *out = uint32_t(acc >> 32);
  }
}

constexpr int kDecWarps = 4;

__device__ __forceinline__ uint32_t ec_bf16(uint32_t s, uint32_t e) {
  return ((s & 0x80u) << 8) | ((e & 0xFFu) << 7) | (s & 0x7Fu);
}

// One warp per chunk (grid-stride), kDecWarps warps per CTA; LUT and the
// chunk's words in shared memory.
__global__ void __launch_bounds__(32 * kDecWarps) k_ec_decode(const uint8_t* __restrict__ blob,
                                                              const uint16_t* __restrict__ lut,
                                                              uint16_t* __restrict__ out) {
  __shared__ uint16_t s_lut[1 << kEcMaxLen];
  __shared__ uint32_t s_w[kDecWarps][32 * kEcMaxLaneWords + 2];
  for (int i = threadIdx.x; i < (1 << kEcMaxLen); i += blockDim.x) s_lut[i] = lut[i];
  __syncthreads();
  const EcHeader h = *reinterpret_cast<const EcHeader*>(blob);
  const uint32_t* base_t = reinterpret_cast<const uint32_t*>(blob + h.base_off);
  const uint8_t* cnt_t = blob + h.cnt_off;
  const uint8_t* sm = blob + h.sm_off;
  const uint32_t* ex = reinterpret_cast<const uint32_t*>(blob + h.exp_off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* sw = s_w[warp];
  const int64_t n = int64_t(h.n_elems);
  for (int64_t ch = blockIdx.x * int64_t(kDecWarps) + warp; ch < h.n_chunks; ch += int64_t(gridDim.x) * kDecWarps) {
    const uint32_t base = __ldg(base_t + ch), total = __ldg(base_t + ch + 1) - base;
    // lane's first word: exclusive scan of the lane word counts
    const uint32_t c = __ldg(cnt_t + ch * 32 + lane);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t my = inc - c;
    __syncwarp();
    for (uint32_t i = lane; i < total + 1; i += 32) sw[i] = __ldg(ex + base + i);  // + the pad / next word
    __syncwarp();
    const int64_t e0 = ch * kEcChunk + int64_t(lane) * kEcLaneSyms;
    const int cnt = int(n - e0 >= kEcLaneSyms ? kEcLaneSyms : (n - e0 > 0 ? n - e0 : 0));
    uint32_t idx = my, w0 = sw[idx], w1 = sw[idx + 1], bo = 0;
    if (cnt == kEcLaneSyms) {
#pragma unroll 1
      for (int g = 0; g < kEcLaneSyms / 16; ++g) {
        const uint4 sv = __ldg(reinterpret_cast<const uint4*>(sm + e0) + g);
        const uint32_t sb[4] = {sv.x, sv.y, sv.z, sv.w};
        uint32_t o[8];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t win = __funnelshift_l(w1, w0, bo);
          const uint32_t e = s_lut[win >> (32 - kEcMaxLen)];
          bo += e >> 8;
          if (bo >= 32) {
            bo -= 32;
            w0 = w1;
            w1 = sw[++idx + 1];
          }
          const uint32_t v = ec_bf16((sb[k >> 2] >> (8 * (k & 3))) & 0xFFu, e);
          if (k & 1) o[k >> 1] |= v << 16;
          else o[k >> 1] = v;
        }
        uint4* dst = reinterpret_cast<uint4*>(out + e0 + 16 * g);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        const uint32_t win = __funnelshift_l(w1, w0, bo);
        const uint32_t e = s_lut[win >> (32 - kEcMaxLen)];
        bo += e >> 8;
        if (bo >= 32) {
          bo -= 32;
          w0 = w1;
          w1 = sw[++idx + 1];
        }
        out[e0 + j] = uint16_t(ec_bf16(__ldg(sm + e0 + j), e));
      }
    }
  }
}

void launch_exp_hist(cudaStream_t s, const void* x, int64_t n, unsigned long long* hist) {
  if (n <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 8));
  k_exp_hist<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, hist);
  KB_LAUNCH();
}
void launch_ec_lane_words(cudaStream_t s, const void* x, int64_t n, const uint8_t* len, uint32_t* words) {
  const int64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  if (chunks <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((chunks * 32 + 255) / 256, 148 * 16));
  k_ec_lane_words<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, len, words);
  KB_LAUNCH();
}
void launch_ec_encode(cudaStream_t s, const void* x, int64_t n, const uint32_t* code, const uint8_t* len,
                      const uint32_t* lane_off, uint8_t* sm, uint32_t* ex) {
  const int64_t streams = (n + kEcLaneSyms - 1) / kEcLaneSyms;
  if (streams <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((streams + 255) / 256, 148 * 16));
  k_ec_encode<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, code, len, lane_off, sm, ex);
  KB_LAUNCH();
}
void launch_ec_decode(cudaStream_t s, const void* blob, int64_t n_chunks, const uint16_t* lut, void* out) {
  if (n_chunks <= 0) return;
  // one warp per chunk; 6 CTAs (24 warps, 203 KB smem) per SM over the whole GPU
  const unsigned blocks = unsigned(std::min<int64_t>((n_chunks + kDecWarps - 1) / kDecWarps, 148 * 6));
  k_ec_decode<<<blocks, 32 * kDecWarps, 0, s>>>(static_cast<const uint8_t*>(blob), lut,
                                                static_cast<uint16_t*>(out));
  KB_LAUNCH();
}

}  // namespace kb
