// kvcode.hpp — format of the exponent-coded bf16 KV store (kvcode.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace kb {

constexpr int kEcLaneSyms = 128;                // elements per lane stream
constexpr int kEcChunk = 32 * kEcLaneSyms;      // elements per chunk (one warp)
constexpr int kEcMaxLen = 12;                   // longest code; LUT = 2^12 entries
constexpr int kEcMaxLaneWords = (kEcLaneSyms * kEcMaxLen + 31) / 32;  // 48 (fits the u8 counts)

// Coded blob image (all offsets in bytes from the image start, 16-B aligned):
//   EcHeader | chunk base u32[n_chunks + 1] (word offset of each chunk's
//   first lane stream) | lane word counts u8[n_chunks][32] | sign+mantissa
//   bytes [n_elems] | exponent words u32[exp_words] + 1 pad word.
// Lane j of a chunk codes the chunk's elements [128 j, 128 j + 128) MSB-first;
// its stream starts at base[chunk] + sum of the counts of lanes < j.
struct EcHeader {
  uint32_t magic;      // 'E','C','1','7'
  uint32_t n_elems;
  uint32_t n_chunks;
  uint32_t base_off;   // chunk base table
  uint32_t cnt_off;    // lane word counts
  uint32_t sm_off;     // sign+mantissa plane
  uint32_t exp_off;    // exponent words
  uint32_t exp_words;  // words in the exponent streams (+1 pad word follows)
};
static_assert(sizeof(EcHeader) == 32, "EcHeader is 32 bytes");
constexpr uint32_t kEcMagic = 0x37314345u;  // "EC17"

// Canonical, length-limited (<= kEcMaxLen) Huffman code of an exponent
// histogram: code[s] (right-aligned, len[s] bits), len 0 = absent symbol,
// and the 4096-entry decode LUT (symbol | len << 8).
struct EcCode {
  uint32_t code[256];
  uint8_t len[256];
  uint16_t lut[1 << kEcMaxLen];
};
EcCode ec_build_code(const uint64_t* hist);

inline size_t ec_align16(size_t x) { return (x + 15) & ~size_t(15); }
// The image's section offsets, element count and lane offsets are u32: a
// blob fits the coded format when its worst-case image (every exponent at
// the longest code) stays below 4 GiB. Larger blobs stay in the raw store.
inline bool ec_fits(uint64_t n) {
  const uint64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  const uint64_t worst = 64 + 4 * (chunks + 1) + 32 * chunks + n +
                         4 * (chunks * 32 * uint64_t(kEcMaxLaneWords) + 1) + 64;
  return worst < (uint64_t(1) << 32);
}
// Section offsets of a coded blob of n elements whose streams hold exp_words.
inline void ec_layout(uint64_t n, uint64_t exp_words, EcHeader* h, size_t* total) {
  const uint64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  h->magic = kEcMagic;
  h->n_elems = uint32_t(n);
  h->n_chunks = uint32_t(chunks);
  h->base_off = uint32_t(sizeof(EcHeader));
  h->cnt_off = uint32_t(ec_align16(h->base_off + 4 * (chunks + 1)));
  h->sm_off = uint32_t(ec_align16(h->cnt_off + 32 * chunks));
  h->exp_off = uint32_t(ec_align16(h->sm_off + n));
  h->exp_words = uint32_t(exp_words);
  *total = ec_align16(size_t(h->exp_off) + 4 * (size_t(exp_words) + 1));
}
// Host codec (tests, inspection, container save): identical bytes / values
// to the device kernels.
std::vector<uint8_t> ec_encode_host(const uint16_t* x, uint64_t n, const EcCode& code);
void ec_decode_host(const uint8_t* blob, const uint16_t* lut, uint16_t* out);

void launch_exp_hist(cudaStream_t s, const void* x, int64_t n, unsigned long long* hist);
// words per (chunk, lane) stream -> words[chunk * 32 + lane]
void launch_ec_lane_words(cudaStream_t s, const void* x, int64_t n, const uint8_t* len, uint32_t* words);
// lane_off: absolute word offset of every (chunk, lane) stream
void launch_ec_encode(cudaStream_t s, const void* x, int64_t n, const uint32_t* code, const uint8_t* len,
                      const uint32_t* lane_off, uint8_t* sm, uint32_t* ex);
void launch_ec_decode(cudaStream_t s, const void* blob, int64_t n_chunks, const uint16_t* lut, void* out);

}  // namespace kb
