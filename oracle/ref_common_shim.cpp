// C entry points over the reference's own common.cpp / common.hpp (compiled
// from /root/reference by ref.mk). Test infrastructure: pins the oracle's
// restatement of UniformStream / fnv1a64 / crc32 (common.hpp:68-90,
// common.cpp:8-42) against the real reference.
#include <cstdint>

#include "krul/common.hpp"

extern "C" {
uint64_t ref_fnv1a64(const void* data, uint64_t len, uint64_t basis) {
  return krul::fnv1a64(data, static_cast<size_t>(len), basis);
}
uint32_t ref_crc32(const void* data, uint64_t len, uint32_t crc) {
  return krul::crc32(data, static_cast<size_t>(len), crc);
}
void ref_uniform_next(uint64_t seed, int64_t n, float lo, float hi, float* out) {
  krul::UniformStream s(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = s.next(lo, hi);
}
void ref_uniform_index(uint64_t seed, int64_t n, uint64_t mod, uint64_t* out) {
  krul::UniformStream s(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = s.next_index(mod);
}
}
