// kvcode.cu — lossless exponent coding of the bf16 KV store (the load
// stream's bytes). B200-native extension of kvstore.cpp's snapshot: the
// restore is PCIe-bound (H2D at 99% of a measured pinned copy), and the 8
// exponent bits of a bf16 KV element carry ~2.6 bits of entropy (Gaussian-
// like values span a few binades), so each element is stored as its raw
// sign+mantissa byte plus a Huffman-coded exponent (~10.6 of 16 bits). The
// restored KV is bit-identical to the uncoded store; the decode runs on the
// expand stream between the blob's H2D copy and its scatter into the pages.
//
// Coded blob (host and device image, 16-B aligned sections):
//   EcHeader | lane offsets u32[n_chunks][32] | sign+mantissa bytes [n] |
//   exponent words u32[exp_words] + 1 pad word
// Elements are cut into chunks of 8192; lane j of a chunk codes elements
// j, j+32, ... MSB-first into its own run of 32-bit words, so a warp decodes
// a chunk with 32 independent bit streams and writes 64 contiguous bytes per
// step. Codes are canonical Huffman, length <= 12: one 4096-entry LUT
// (symbol | length << 8) in shared memory decodes a symbol per lookup.
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
  const int lane = threadIdx.x & 31;
  const int64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  for (int64_t ch = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; ch < chunks;
       ch += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t base = ch * kEcChunk;
    const int cnt = int(n - base < kEcChunk ? n - base : kEcChunk);
    uint32_t bits = 0;
    for (int j = lane; j < cnt; j += 32) bits += sl[(x[base + j] >> 7) & 0xFF];
    words[ch * 32 + lane] = (bits + 31) / 32;
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
  const int lane = threadIdx.x & 31;
  const int64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  for (int64_t ch = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; ch < chunks;
       ch += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t base = ch * kEcChunk;
    const int cnt = int(n - base < kEcChunk ? n - base : kEcChunk);
    uint32_t* out = ex + lane_off[ch * 32 + lane];
    uint64_t acc = 0;
    int nb = 0;
    for (int j = lane; j < cnt; j += 32) {
      const uint32_t v = x[base + j];
      sm[base + j] = uint8_t(((v >> 8) & 0x80u) | (v & 0x7Fu));
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

// One warp per chunk, 8 warps per CTA, grid-stride; LUT in shared memory.
__global__ void __launch_bounds__(256) k_ec_decode(const uint8_t* __restrict__ blob,
                                                   const uint16_t* __restrict__ lut,
                                                   uint16_t* __restrict__ out) {
  __shared__ uint16_t s_lut[1 << kEcMaxLen];
  for (int i = threadIdx.x; i < (1 << kEcMaxLen); i += blockDim.x) s_lut[i] = lut[i];
  __syncthreads();
  const EcHeader h = *reinterpret_cast<const EcHeader*>(blob);
  const uint32_t* lane_off = reinterpret_cast<const uint32_t*>(blob + sizeof(EcHeader));
  const uint8_t* sm = blob + h.sm_off;
  const uint32_t* ex = reinterpret_cast<const uint32_t*>(blob + h.exp_off);
  const int lane = threadIdx.x & 31;
  const int64_t n = int64_t(h.n_elems);
  for (int64_t ch = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); ch < h.n_chunks;
       ch += int64_t(gridDim.x) * (blockDim.x >> 5)) {
    const uint32_t* p = ex + __ldg(lane_off + ch * 32 + lane);
    const int64_t base = ch * kEcChunk;
    const int cnt = int(n - base < kEcChunk ? n - base : kEcChunk);
    uint64_t buf = 0;
    int have = 0;
#pragma unroll 4
    for (int j = lane; j < cnt; j += 32) {
      if (have < kEcMaxLen) {
        buf |= uint64_t(__ldg(p++)) << (32 - have);
        have += 32;
      }
      const uint32_t e = s_lut[buf >> (64 - kEcMaxLen)];
      const int l = int(e >> 8);
      buf <<= l;
      have -= l;
      const uint32_t s = __ldg(sm + base + j);
      out[base + j] = uint16_t(((s & 0x80u) << 8) | ((e & 0xFFu) << 7) | (s & 0x7Fu));
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
  const unsigned blocks = unsigned(std::min<int64_t>((chunks + 7) / 8, 148 * 16));
  k_ec_lane_words<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, len, words);
  KB_LAUNCH();
}
void launch_ec_encode(cudaStream_t s, const void* x, int64_t n, const uint32_t* code, const uint8_t* len,
                      const uint32_t* lane_off, uint8_t* sm, uint32_t* ex) {
  const int64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  if (chunks <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((chunks + 7) / 8, 148 * 16));
  k_ec_encode<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, code, len, lane_off, sm, ex);
  KB_LAUNCH();
}
void launch_ec_decode(cudaStream_t s, const void* blob, int64_t n_chunks, const uint16_t* lut, void* out) {
  if (n_chunks <= 0) return;
  // one warp per chunk; >= 2 resident CTAs per SM over the whole GPU
  const unsigned blocks = unsigned(std::min<int64_t>((n_chunks + 7) / 8, 148 * 4));
  k_ec_decode<<<blocks, 256, 0, s>>>(static_cast<const uint8_t*>(blob), lut, static_cast<uint16_t*>(out));
  KB_LAUNCH();
}

}  // namespace kb
