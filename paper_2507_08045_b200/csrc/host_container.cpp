// host_container.cpp — the KRUL v1 snapshot container (kvstore.hpp:88-98,
// kvstore.cpp:360-511): on-disk interchange between the
// pinned bf16/f32 store of this library and the reference's f32 snapshots.
//
// Layout (little-endian): "KRUL" | u32 version | u64 config_hash |
// u64 metadata_len | metadata (key-sorted compact JSON) | u32 blob_count |
// blobs (u32 owner_count, i32 owners, i64 start, i64 end, u64 payload_len,
// f32 payload: keys [heads][rows][hd] then values) | u32 crc32 of all
// preceding bytes.
//
// Host work, bounded by memory bandwidth: the payload is converted
// (bf16 <-> f32) and checksummed by all host threads — slicing-by-8 CRC per
// chunk, chunks joined with the GF(2) crc32_combine — so a 1.5 GB container
// of the Llama-3-8B 8K snapshot saves/loads at tens of GB/s instead of the
// ~0.5 GB/s of a byte-at-a-time CRC. The metadata writer reproduces
// nlohmann::json::dump() byte for byte (std::map key order, Grisu2 shortest
// doubles with nlohmann's fixed/exponent switch at 10^-5 / 10^15), so a
// container saved here is bit-identical to the reference's save of the same
// f32 snapshot (tests/test_container.py pins it against nlohmann 3.11.3).
#include <locale.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>

#include "host.hpp"

namespace kb {

// --------------------------------------------------------------- threads
template <class F>
static void parallel_chunks(size_t n, size_t min_chunk, F&& f) {
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t t = std::max<size_t>(1, std::min<size_t>({hw, 32, n / std::max<size_t>(min_chunk, 1)}));
  if (t <= 1) {
    f(size_t(0), size_t(0), n);
    return;
  }
  const size_t per = (n + t - 1) / t;
  std::vector<std::thread> th;
  for (size_t i = 1; i < t; ++i) {
    const size_t b = std::min(n, i * per), e = std::min(n, b + per);
    th.emplace_back([&f, i, b, e] { f(i, b, e); });
  }
  f(0, 0, std::min(n, per));
  for (auto& x : th) x.join();
}

// ----------------------------------------------------------------- crc32
// common.cpp:34-42: reflected 0xEDB88320, pre/post inversion.
namespace {
struct CrcTables {
  uint32_t t[8][256];
  CrcTables() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xedb88320u ^ (c >> 1) : c >> 1;
      t[0][i] = c;
    }
    for (int k = 1; k < 8; ++k)
      for (int i = 0; i < 256; ++i) t[k][i] = (t[k - 1][i] >> 8) ^ t[0][t[k - 1][i] & 0xffu];
  }
};
const CrcTables& crc_tables() {
  static const CrcTables tb;
  return tb;
}
uint32_t crc_update(uint32_t c, const unsigned char* p, size_t n) {  // c: inverted register
  const auto& T = crc_tables().t;
  while (n && (reinterpret_cast<uintptr_t>(p) & 7)) {
    c = T[0][(c ^ *p++) & 0xffu] ^ (c >> 8);
    --n;
  }
  while (n >= 8) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    w ^= c;
    c = T[7][w & 0xff] ^ T[6][(w >> 8) & 0xff] ^ T[5][(w >> 16) & 0xff] ^ T[4][(w >> 24) & 0xff] ^
        T[3][(w >> 32) & 0xff] ^ T[2][(w >> 40) & 0xff] ^ T[1][(w >> 48) & 0xff] ^ T[0][w >> 56];
    p += 8;
    n -= 8;
  }
  while (n--) c = T[0][(c ^ *p++) & 0xffu] ^ (c >> 8);
  return c;
}
uint32_t gf2_times(const uint32_t* mat, uint32_t vec) {
  uint32_t sum = 0;
  for (; vec; vec >>= 1, ++mat)
    if (vec & 1u) sum ^= *mat;
  return sum;
}
void gf2_square(uint32_t* sq, const uint32_t* mat) {
  for (int n = 0; n < 32; ++n) sq[n] = gf2_times(mat, mat[n]);
}
// crc(A || B) from crc(A), crc(B) and |B|: B's length of zero bits applied to
// crc(A) by repeated squaring of the one-zero-bit operator.
uint32_t crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  if (len2 == 0) return crc1;
  uint32_t even[32], odd[32];
  odd[0] = 0xedb88320u;
  uint32_t row = 1;
  for (int n = 1; n < 32; ++n, row <<= 1) odd[n] = row;
  gf2_square(even, odd);
  gf2_square(odd, even);
  do {
    gf2_square(even, odd);
    if (len2 & 1) crc1 = gf2_times(even, crc1);
    len2 >>= 1;
    if (!len2) break;
    gf2_square(odd, even);
    if (len2 & 1) crc1 = gf2_times(odd, crc1);
    len2 >>= 1;
  } while (len2);
  return crc1 ^ crc2;
}
}  // namespace

uint32_t crc32(const void* data, size_t n, uint32_t crc) {
  const auto* p = static_cast<const unsigned char*>(data);
  constexpr size_t kChunk = size_t(4) << 20;
  if (n < 2 * kChunk) return crc_update(crc ^ 0xffffffffu, p, n) ^ 0xffffffffu;
  std::vector<uint32_t> part(64, 0);
  std::vector<size_t> len(64, 0);
  parallel_chunks(n, kChunk, [&](size_t i, size_t b, size_t e) {
    part[i] = crc_update(0xffffffffu, p + b, e - b) ^ 0xffffffffu;
    len[i] = e - b;
  });
  uint32_t c = crc;
  for (size_t i = 0; i < 64; ++i)
    if (len[i]) c = crc32_combine(c, part[i], len[i]);
  return c;
}

// ------------------------------------------------------ payload conversion
static inline float bf16f(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f2bf(float f) {  // RNE, == __float2bfloat16_rn
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
// store (esz bytes/elem) -> little-endian f32 bytes
static void to_f32(const void* src, size_t esz, char* dst, size_t n) {
  parallel_chunks(n, size_t(1) << 20, [&](size_t, size_t b, size_t e) {
    if (esz == 4) {
      std::memcpy(dst + b * 4, static_cast<const char*>(src) + b * 4, (e - b) * 4);
    } else {
      const uint16_t* s = static_cast<const uint16_t*>(src);
      for (size_t i = b; i < e; ++i) {
        const float f = bf16f(s[i]);
        std::memcpy(dst + i * 4, &f, 4);
      }
    }
  });
}
static void from_f32(const char* src, size_t esz, void* dst, size_t n) {
  parallel_chunks(n, size_t(1) << 20, [&](size_t, size_t b, size_t e) {
    if (esz == 4) {
      std::memcpy(static_cast<char*>(dst) + b * 4, src + b * 4, (e - b) * 4);
    } else {
      uint16_t* d = static_cast<uint16_t*>(dst);
      for (size_t i = b; i < e; ++i) {
        float f;
        std::memcpy(&f, src + i * 4, 4);
        d[i] = f2bf(f);
      }
    }
  });
}

// ------------------------------------------------------------ JSON writer
// nlohmann::json::dump() (compact) of the values the metadata holds.
namespace {
struct CachedPow {
  uint64_t f;
  int e, k;
};
// round(10^k * 2^-e), k = -300..324 step 8 (tools/gen_pow10.py)
const CachedPow kPow10[] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300},
    {0xFF77B1FCBEBCDC4FULL, -1034, -292},
    {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276},
    {0xD3515C2831559A83ULL, -954, -268},
    {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252},
    {0xAECC49914078536DULL, -874, -244},
    {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228},
    {0x9096EA6F3848984FULL, -794, -220},
    {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204},
    {0xEF340A98172AACE5ULL, -715, -196},
    {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180},
    {0xC5DD44271AD3CDBAULL, -635, -172},
    {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156},
    {0xA3AB66580D5FDAF6ULL, -555, -148},
    {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132},
    {0x87625F056C7C4A8BULL, -475, -124},
    {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108},
    {0xDFF9772470297EBDULL, -396, -100},
    {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84},
    {0xB94470938FA89BCFULL, -316, -76},
    {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60},
    {0x993FE2C6D07B7FACULL, -236, -52},
    {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36},
    {0xFD87B5F28300CA0EULL, -157, -28},
    {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12},
    {0xD1B71758E219652CULL, -77, -4},
    {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12},
    {0xAD78EBC5AC620000ULL, 3, 20},
    {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36},
    {0x8F7E32CE7BEA5C70ULL, 83, 44},
    {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60},
    {0xED63A231D4C4FB27ULL, 162, 68},
    {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84},
    {0xC45D1DF942711D9AULL, 242, 92},
    {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108},
    {0xA26DA3999AEF774AULL, 322, 116},
    {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132},
    {0x865B86925B9BC5C2ULL, 402, 140},
    {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156},
    {0xDE469FBD99A05FE3ULL, 481, 164},
    {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180},
    {0xB7DCBF5354E9BECEULL, 561, 188},
    {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204},
    {0x98165AF37B2153DFULL, 641, 212},
    {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228},
    {0xFB9B7CD9A4A7443CULL, 720, 236},
    {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252},
    {0xD01FEF10A657842CULL, 800, 260},
    {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276},
    {0xAC2820D9623BF429ULL, 880, 284},
    {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300},
    {0x8E679C2F5E44FF8FULL, 960, 308},
    {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324},
};
struct Fp {
  uint64_t f;
  int e;
};
Fp fp_mul(Fp x, Fp y) {
  const unsigned __int128 p = (unsigned __int128)x.f * y.f + (uint64_t(1) << 63);
  return {uint64_t(p >> 64), x.e + y.e + 64};
}
Fp fp_norm(Fp x) {
  while (!(x.f >> 63)) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}
void grisu_round(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}
// Grisu2 (Loitsch 2010) with the boundaries of the double's rounding interval,
// target exponent window [-60, -32]: digits of a short representation that
// round-trips, and its decimal exponent. Positive finite v only.
int grisu2(char* buf, int* dec_exp, double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = bits >> 52, F = bits & ((uint64_t(1) << 52) - 1);
  const Fp w0 = E == 0 ? Fp{F, -1074} : Fp{F + (uint64_t(1) << 52), int(E) - 1075};
  const bool closer = F == 0 && E > 1;
  const Fp mp = fp_norm(Fp{2 * w0.f + 1, w0.e - 1});
  Fp mm = closer ? Fp{4 * w0.f - 1, w0.e - 2} : Fp{2 * w0.f - 1, w0.e - 1};
  mm = Fp{mm.f << (mm.e - mp.e), mp.e};
  const Fp w = fp_norm(w0);
  const int f = -60 - mp.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0);
  const CachedPow& c = kPow10[(300 + k + 7) / 8];
  const Fp ck{c.f, c.e};
  const Fp ww = fp_mul(w, ck), wm = fp_mul(mm, ck), wp = fp_mul(mp, ck);
  const Fp Mm{wm.f + 1, wm.e}, Mp{wp.f - 1, wp.e};
  *dec_exp = -c.k;
  uint64_t delta = Mp.f - Mm.f, dist = Mp.f - ww.f;
  const int sh = -Mp.e;
  const uint64_t one = uint64_t(1) << sh;
  uint32_t p1 = uint32_t(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  uint32_t pow10 = 1;
  int n = 1;
  for (uint32_t t = 10; n < 10 && p1 >= t; t *= 10) {
    pow10 = t;
    ++n;
    if (t > 429496729u) break;
  }
  int len = 0;
  while (n > 0) {
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = char('0' + d);
    p1 = r;
    --n;
    const uint64_t rest = (uint64_t(p1) << sh) + p2;
    if (rest <= delta) {
      *dec_exp += n;
      grisu_round(buf, len, dist, delta, rest, uint64_t(pow10) << sh);
      return len;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = char('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  *dec_exp -= m;
  grisu_round(buf, len, dist, delta, p2, one);
  return len;
}
}  // namespace

static void json_double(std::string& o, double v) {
  if (!std::isfinite(v)) {
    o += "null";
    return;
  }
  if (std::signbit(v)) o += '-';
  v = std::fabs(v);
  if (v == 0) {
    o += "0.0";
    return;
  }
  char d[32];
  int de = 0;
  const int k = grisu2(d, &de, v);
  const int n = k + de;  // decimal point position relative to the digits
  std::string dg(d, size_t(k));
  if (k <= n && n <= 15) {
    o += dg;
    o.append(size_t(n - k), '0');
    o += ".0";
  } else if (0 < n && n <= 15) {
    o += dg.substr(0, size_t(n));
    o += '.';
    o += dg.substr(size_t(n));
  } else if (-4 < n && n <= 0) {
    o += "0.";
    o.append(size_t(-n), '0');
    o += dg;
  } else {
    o += dg[0];
    if (k > 1) {
      o += '.';
      o += dg.substr(1);
    }
    int ex = n - 1;
    o += 'e';
    o += ex < 0 ? '-' : '+';
    ex = std::abs(ex);
    char eb[8];
    std::snprintf(eb, sizeof eb, ex < 100 ? "%02d" : "%03d", ex);
    o += eb;
  }
}
static void json_int(std::string& o, int64_t v) { o += std::to_string(v); }
// Length of the well-formed UTF-8 sequence at p (RFC 3629), 0 if malformed.
static int utf8_seq(const unsigned char* p, const unsigned char* e) {
  const unsigned char c = *p;
  int len;
  uint32_t cp, lo;
  if (c < 0x80) return 1;
  if (c >= 0xc2 && c <= 0xdf) len = 2, cp = c & 0x1f, lo = 0x80;
  else if (c >= 0xe0 && c <= 0xef) len = 3, cp = c & 0x0f, lo = 0x800;
  else if (c >= 0xf0 && c <= 0xf4) len = 4, cp = c & 0x07, lo = 0x10000;
  else return 0;
  if (e - p < len) return 0;
  for (int j = 1; j < len; ++j) {
    if ((p[j] & 0xc0) != 0x80) return 0;
    cp = (cp << 6) | (p[j] & 0x3f);
  }
  if (cp < lo || cp > 0x10ffff || (cp >= 0xd800 && cp <= 0xdfff)) return 0;
  return len;
}
// strict UTF-8 (nlohmann's default error handler throws on invalid bytes);
// control characters escaped, everything else verbatim (ensure_ascii=false)
static void json_string(std::string& o, const std::string& s) {
  o += '"';
  for (size_t i = 0; i < s.size();) {
    const unsigned char c = static_cast<unsigned char>(s[i]);
    if (c < 0x80) {
      switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        default:
          if (c < 0x20) {
            char e[8];
            std::snprintf(e, sizeof e, "\\u%04x", unsigned(c));
            o += e;
          } else {
            o += char(c);
          }
      }
      ++i;
      continue;
    }
    const auto* u = reinterpret_cast<const unsigned char*>(s.data());
    const int len = utf8_seq(u + i, u + s.size());
    if (!len) fail(KRUL_E_SNAPSHOT, "conversation id is not valid UTF-8");
    o.append(s, i, size_t(len));
    i += size_t(len);
  }
  o += '"';
}
template <class T, class F>
static void json_array(std::string& o, const std::vector<T>& v, F&& put) {
  o += '[';
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ',';
    put(v[i]);
  }
  o += ']';
}

static std::vector<int> shared_layers(const Snapshot& s) {
  if (!s.meta.shared.empty() || s.pairs.empty()) return s.meta.shared;
  std::vector<int> v;
  for (const auto& p : s.pairs) {
    v.push_back(p.shallow);
    v.push_back(p.deep);
  }
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

// kvstore.cpp:362-371 (+ the *_to_json helpers at :100-143): keys in
// std::map order.
static std::string meta_text(const Snapshot& s) {
  std::string o;
  o.reserve(256 + 24 * (s.p.size() + s.meta.avg_weight_sum.size() + s.pairs.size()));
  const auto ints = [&o](const std::vector<int>& v) { json_array(o, v, [&o](int x) { json_int(o, x); }); };
  o += "{\"classifier\":{\"avg_weight_sum\":";
  json_array(o, s.meta.avg_weight_sum, [&o](double x) { json_double(o, x); });
  o += ",\"ir_layers\":";
  ints(s.meta.ir_layers);
  o += ",\"non_ir_layers\":";
  ints(s.meta.non_ir_layers);
  o += "},\"conversation_id\":";
  json_string(o, s.meta.conversation_id);
  o += ",\"head_dim\":";
  json_int(o, s.hd);
  o += ",\"history_len\":";
  json_int(o, s.L);
  o += ",\"mode\":";
  o += s.mode == KRUL_MERGE_KEEP_DEEPER ? "\"keep-deeper\"" : "\"mean\"";
  o += ",\"n_heads\":";
  json_int(o, s.Hkv);
  o += ",\"n_layers\":";
  json_int(o, s.N);
  o += ",\"plan\":{\"history_len\":";
  json_int(o, s.L);
  o += ",\"recompute_len\":";
  json_array(o, s.p, [&o](int64_t x) { json_int(o, x); });
  o += "},\"strategy\":{\"exhausted_before_quota\":";
  o += s.meta.exhausted_before_quota ? "true" : "false";
  o += ",\"pairs\":";
  json_array(o, s.pairs, [&o](const krul_pair& p) {
    o += '[';
    json_int(o, p.shallow);
    o += ',';
    json_int(o, p.deep);
    o += ',';
    json_double(o, p.distance);
    o += ']';
  });
  o += ",\"shared\":";
  ints(shared_layers(s));
  o += "}}";
  return o;
}

// ------------------------------------------------------------ JSON reader
namespace {
struct JV {
  enum T { NUL, BOOL, INT, UINT, DBL, STR, ARR, OBJ } t = NUL;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0;
  std::string s;
  std::vector<JV> a;
  std::vector<std::pair<std::string, JV>> o;
};
struct JErr {
  std::string m;
};
struct JParser {
  const char* p;
  const char* e;
  int depth = 0;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  [[noreturn]] void bad(const char* m) { throw JErr{std::string("parse error: ") + m}; }
  void lit(const char* w) {
    const size_t n = std::strlen(w);
    if (size_t(e - p) < n || std::memcmp(p, w, n)) bad("invalid literal");
    p += n;
  }
  static void put_utf8(std::string& s, uint32_t cp) {
    if (cp < 0x80) {
      s += char(cp);
    } else if (cp < 0x800) {
      s += char(0xc0 | (cp >> 6));
      s += char(0x80 | (cp & 0x3f));
    } else if (cp < 0x10000) {
      s += char(0xe0 | (cp >> 12));
      s += char(0x80 | ((cp >> 6) & 0x3f));
      s += char(0x80 | (cp & 0x3f));
    } else {
      s += char(0xf0 | (cp >> 18));
      s += char(0x80 | ((cp >> 12) & 0x3f));
      s += char(0x80 | ((cp >> 6) & 0x3f));
      s += char(0x80 | (cp & 0x3f));
    }
  }
  uint32_t hex4() {
    if (e - p < 4) bad("truncated \\u escape");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= uint32_t(c - '0');
      else if (c >= 'a' && c <= 'f') v |= uint32_t(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= uint32_t(c - 'A' + 10);
      else bad("invalid \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p;  // opening quote
    std::string s;
    for (;;) {
      if (p >= e) bad("unterminated string");
      const unsigned char c = static_cast<unsigned char>(*p++);
      if (c == '"') return s;
      if (c < 0x20) bad("control character in string");
      if (c >= 0x80) {  // the lexer accepts only well-formed UTF-8
        const int n = utf8_seq(reinterpret_cast<const unsigned char*>(p - 1),
                               reinterpret_cast<const unsigned char*>(e));
        if (!n) bad("invalid UTF-8 in string");
        s.append(p - 1, size_t(n));
        p += n - 1;
        continue;
      }
      if (c != '\\') {
        s += char(c);
        continue;
      }
      if (p >= e) bad("unterminated escape");
      const char x = *p++;
      switch (x) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case '/': s += '/'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'n': s += '\n'; break;
        case 'r': s += '\r'; break;
        case 't': s += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xd800 && cp <= 0xdbff) {
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') bad("unpaired surrogate");
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xdc00 || lo > 0xdfff) bad("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xd800) << 10) + (lo - 0xdc00);
          } else if (cp >= 0xdc00 && cp <= 0xdfff) {
            bad("unpaired surrogate");
          }
          put_utf8(s, cp);
          break;
        }
        default: bad("invalid escape");
      }
    }
  }
  JV num() {
    const char* b = p;
    bool is_float = false;
    if (p < e && *p == '-') ++p;
    if (p >= e || !(*p >= '0' && *p <= '9')) bad("invalid number");
    if (*p == '0') ++p;
    else while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p < e && *p == '.') {
      is_float = true;
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) bad("invalid number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) bad("invalid number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    const std::string t(b, p);
    JV v;
    if (!is_float) {
      errno = 0;
      if (t[0] == '-') {
        const long long x = std::strtoll(t.c_str(), nullptr, 10);
        if (errno == 0) {
          v.t = JV::INT;
          v.i = x;
          return v;
        }
      } else {
        const unsigned long long x = std::strtoull(t.c_str(), nullptr, 10);
        if (errno == 0) {
          v.t = JV::UINT;
          v.u = x;
          return v;
        }
      }
    }
    v.t = JV::DBL;
    // "C" locale: the process locale must not change the decimal point
    static const locale_t c_loc = newlocale(LC_ALL_MASK, "C", locale_t(0));
    v.d = strtod_l(t.c_str(), nullptr, c_loc);
    if (!std::isfinite(v.d)) bad("number overflow");  // nlohmann rejects, no inf
    return v;
  }
  JV value() {
    ws();
    if (p >= e) bad("unexpected end of input");
    if (++depth > 512) bad("nesting too deep");
    JV v;
    switch (*p) {
      case '{': {
        ++p;
        v.t = JV::OBJ;
        ws();
        if (p < e && *p == '}') {
          ++p;
          break;
        }
        for (;;) {
          ws();
          if (p >= e || *p != '"') bad("expected object key");
          std::string k = str();
          ws();
          if (p >= e || *p != ':') bad("expected ':'");
          ++p;
          JV x = value();
          // duplicate keys: the last one wins (std::map assignment)
          bool found = false;
          for (auto& kv : v.o)
            if (kv.first == k) {
              kv.second = std::move(x);
              found = true;
              break;
            }
          if (!found) v.o.emplace_back(std::move(k), std::move(x));
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == '}') {
            ++p;
            break;
          }
          bad("expected ',' or '}'");
        }
        break;
      }
      case '[': {
        ++p;
        v.t = JV::ARR;
        ws();
        if (p < e && *p == ']') {
          ++p;
          break;
        }
        for (;;) {
          v.a.push_back(value());
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == ']') {
            ++p;
            break;
          }
          bad("expected ',' or ']'");
        }
        break;
      }
      case '"':
        v.t = JV::STR;
        v.s = str();
        break;
      case 't':
        lit("true");
        v.t = JV::BOOL;
        v.b = true;
        break;
      case 'f':
        lit("false");
        v.t = JV::BOOL;
        break;
      case 'n':
        lit("null");
        break;
      default:
        v = num();
    }
    --depth;
    return v;
  }
};
JV json_parse(const char* b, size_t n) {
  JParser P{b, b + n};
  JV v = P.value();
  P.ws();
  if (P.p != P.e) throw JErr{"parse error: trailing characters"};
  return v;
}
// nlohmann accessors: at() needs an object with the key, get<T> the type
const JV& at(const JV& v, const char* key) {
  if (v.t != JV::OBJ) throw JErr{std::string("cannot use at() with a non-object for key ") + key};
  for (const auto& kv : v.o)
    if (kv.first == key) return kv.second;
  throw JErr{std::string("key '") + key + "' not found"};
}
const JV& at(const JV& v, size_t i) {
  if (v.t != JV::ARR) throw JErr{"cannot use at() with a non-array"};
  if (i >= v.a.size()) throw JErr{"array index out of range"};
  return v.a[i];
}
// static_cast of a double on x86-64 (what the reference is built for):
// out-of-range values convert to the "integer indefinite" INT_MIN.
int64_t get_i64(const JV& v) {
  switch (v.t) {
    case JV::INT: return v.i;
    case JV::UINT: return int64_t(v.u);
    case JV::DBL:
      return v.d >= -9223372036854775808.0 && v.d < 9223372036854775808.0 ? int64_t(v.d) : INT64_MIN;
    case JV::BOOL: return v.b ? 1 : 0;
    default: throw JErr{"type must be number"};
  }
}
int get_int(const JV& v) {
  if (v.t == JV::DBL) return v.d > -2147483649.0 && v.d < 2147483648.0 ? int(v.d) : INT32_MIN;
  return int(uint32_t(uint64_t(get_i64(v))));
}
double get_double(const JV& v) {
  switch (v.t) {
    case JV::INT: return double(v.i);
    case JV::UINT: return double(v.u);
    case JV::DBL: return v.d;
    case JV::BOOL: return v.b ? 1.0 : 0.0;
    default: throw JErr{"type must be number"};
  }
}
bool get_bool(const JV& v) {
  if (v.t != JV::BOOL) throw JErr{"type must be boolean"};
  return v.b;
}
const std::string& get_str(const JV& v) {
  if (v.t != JV::STR) throw JErr{"type must be string"};
  return v.s;
}
const std::vector<JV>& get_arr(const JV& v) {
  if (v.t != JV::ARR) throw JErr{"type must be array"};
  return v.a;
}
}  // namespace

// ------------------------------------------------------------------- save
static size_t payload_elems(const Snapshot& s, const Snapshot::Blob& b) {
  return size_t(2) * size_t(s.Hkv) * size_t(b.end - b.start) * size_t(s.hd);
}
static void put32(char*& o, uint32_t v) {
  std::memcpy(o, &v, 4);
  o += 4;
}
static void put64(char*& o, uint64_t v) {
  std::memcpy(o, &v, 8);
  o += 8;
}
static size_t blob_header_bytes(const Snapshot::Blob& b) { return 4 + 4 * (b.owners[1] >= 0 ? 2 : 1) + 24; }

static size_t header_into(const Snapshot& s, const std::string& meta, char* o0) {
  char* o = o0;
  std::memcpy(o, "KRUL", 4);
  o += 4;
  put32(o, 1u);
  put64(o, s.config_hash);
  put64(o, meta.size());
  std::memcpy(o, meta.data(), meta.size());
  o += meta.size();
  put32(o, uint32_t(s.blobs.size()));
  return size_t(o - o0);
}
static size_t blob_header_into(const Snapshot& s, const Snapshot::Blob& b, char* o0) {
  char* o = o0;
  const bool pair = b.owners[1] >= 0;
  put32(o, pair ? 2u : 1u);
  put32(o, uint32_t(b.owners[0]));
  if (pair) put32(o, uint32_t(b.owners[1]));
  put64(o, uint64_t(b.start));
  put64(o, uint64_t(b.end));
  put64(o, uint64_t(payload_elems(s, b)) * 4);
  return size_t(o - o0);
}

uint64_t container_size(const Snapshot& s) {
  uint64_t n = 4 + 4 + 8 + 8 + meta_text(s).size() + 4 + 4;
  for (const auto& b : s.blobs) n += blob_header_bytes(b) + payload_elems(s, b) * 4;
  return n;
}

void container_write(const Snapshot& s, char* out) {
  const std::string meta = meta_text(s);
  char* o = out + header_into(s, meta, out);
  std::vector<uint16_t> tmp;
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    o += blob_header_into(s, b, o);
    const size_t n = payload_elems(s, b);
    to_f32(snapshot_raw_blob(s, int(bi), tmp), s.esz, o, n);
    o += n * 4;
  }
  const uint32_t c = crc32(out, size_t(o - out));
  put32(o, c);
}

void container_write_file(const Snapshot& s, const char* path) {
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
  if (!f) fail(KRUL_E_SNAPSHOT, std::string("cannot open ") + path + " for writing");
  const std::string meta = meta_text(s);
  std::vector<char> hb(meta.size() + 64);
  uint32_t crc = 0;
  auto emit = [&](const char* p, size_t n) {
    crc = crc32(p, n, crc);
    if (n && std::fwrite(p, 1, n, f.get()) != n) fail(KRUL_E_SNAPSHOT, "snapshot sink write failed");
  };
  emit(hb.data(), header_into(s, meta, hb.data()));
  constexpr size_t kBounce = size_t(64) << 20;  // f32 bytes per conversion chunk
  std::vector<char> bounce;
  std::vector<uint16_t> tmp;
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    const char* raw = snapshot_raw_blob(s, int(bi), tmp);
    char bh[64];
    emit(bh, blob_header_into(s, b, bh));
    const size_t n = payload_elems(s, b);
    if (bounce.size() < std::min(n * 4, kBounce)) bounce.resize(std::min(n * 4, kBounce));
    for (size_t i = 0; i < n; i += kBounce / 4) {
      const size_t m = std::min(kBounce / 4, n - i);
      to_f32(raw + i * s.esz, s.esz, bounce.data(), m);
      emit(bounce.data(), m * 4);
    }
  }
  char cb[4];
  std::memcpy(cb, &crc, 4);
  if (std::fwrite(cb, 1, 4, f.get()) != 4) fail(KRUL_E_SNAPSHOT, "snapshot sink write failed");
  if (std::fflush(f.get()) != 0) fail(KRUL_E_SNAPSHOT, "snapshot sink write failed");
}

// ------------------------------------------------------------------- load
namespace {
struct Reader {
  const char* b;
  size_t n, pos = 0;
  size_t remaining() const { return n - pos; }
  const char* take(size_t len, const char* field) {
    if (remaining() < len) throw LoadError(field, "container ends mid-field");
    const char* p = b + pos;
    pos += len;
    return p;
  }
  template <class T>
  T get(const char* field) {
    T v;
    std::memcpy(&v, take(sizeof(T), field), sizeof(T));
    return v;
  }
};
}  // namespace

// kvstore.cpp:394-511, same checks in the same order and the same failing
// field names; the f32 payload lands in the store in the ctx dtype (pinned),
// or as f32 in plain memory for a host-only snapshot (ctx null).
Snapshot* container_read(Ctx* c, const char* buf, size_t n, const uint64_t* expected_hash) {
  if (n >= 4 && std::memcmp(buf, "KRUL", 4) != 0) throw LoadError("magic", "not a snapshot container");
  if (n < 8) throw LoadError("checksum", "container shorter than its framing");
  uint32_t stored;
  std::memcpy(&stored, buf + n - 4, 4);
  const auto tc = std::chrono::steady_clock::now();
  if (stored != crc32(buf, n - 4)) throw LoadError("checksum", "container checksum mismatch");
  const double crc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc).count();
  Reader r{buf, n};
  r.take(4, "magic");
  const uint32_t version = r.get<uint32_t>("version");
  if (version != 1u) throw LoadError("version", "unsupported format version " + std::to_string(version));
  const uint64_t hash = r.get<uint64_t>("config");
  if (expected_hash && hash != *expected_hash)
    throw LoadError("config", "snapshot was taken under a different model configuration");
  const uint64_t meta_len = r.get<uint64_t>("metadata");
  const char* meta_ptr = r.take(size_t(meta_len), "metadata");

  std::unique_ptr<Snapshot> s(new Snapshot);
  s->ctx = c;
  s->esz = c ? c->esz : 4;
  // plain memory first-touched by the converting threads, then page-locked
  // in one cudaHostRegister: cudaMallocHost faults and pins serially
  s->host.pageable = true;
  s->config_hash = hash;
  int64_t plan_history = 0;
  try {
    const JV m = json_parse(meta_ptr, size_t(meta_len));
    s->meta.conversation_id = get_str(at(m, "conversation_id"));
    s->N = get_int(at(m, "n_layers"));
    s->Hkv = get_int(at(m, "n_heads"));
    s->hd = get_int(at(m, "head_dim"));
    s->L = get_i64(at(m, "history_len"));
    const std::string& mode = get_str(at(m, "mode"));
    if (mode == "mean") s->mode = KRUL_MERGE_MEAN;
    else if (mode == "keep-deeper") s->mode = KRUL_MERGE_KEEP_DEEPER;
    else throw LoadError("metadata", "unknown merge mode");
    const JV& st = at(m, "strategy");
    for (const JV& p : get_arr(at(st, "pairs")))
      s->pairs.push_back(krul_pair{get_int(at(p, size_t(0))), get_int(at(p, size_t(1))), get_double(at(p, size_t(2)))});
    for (const JV& l : get_arr(at(st, "shared"))) s->meta.shared.push_back(get_int(l));
    std::sort(s->meta.shared.begin(), s->meta.shared.end());
    s->meta.shared.erase(std::unique(s->meta.shared.begin(), s->meta.shared.end()), s->meta.shared.end());
    s->meta.exhausted_before_quota = get_bool(at(st, "exhausted_before_quota"));
    const JV& pl = at(m, "plan");
    plan_history = get_i64(at(pl, "history_len"));
    for (const JV& x : get_arr(at(pl, "recompute_len"))) s->p.push_back(get_i64(x));
    const JV& cl = at(m, "classifier");
    for (const JV& x : get_arr(at(cl, "ir_layers"))) s->meta.ir_layers.push_back(get_int(x));
    for (const JV& x : get_arr(at(cl, "non_ir_layers"))) s->meta.non_ir_layers.push_back(get_int(x));
    for (const JV& x : get_arr(at(cl, "avg_weight_sum"))) s->meta.avg_weight_sum.push_back(get_double(x));
  } catch (const JErr& e) {
    throw LoadError("metadata", e.m);
  }
  if (int64_t(s->p.size()) != int64_t(s->N) || plan_history != s->L)
    throw LoadError("plan", "plan does not match the snapshot header");
  if (s->N < 0 || s->Hkv < 0 || s->hd < 0) throw LoadError("metadata", "negative dimension");

  const uint32_t blob_count = r.get<uint32_t>("blob");
  std::vector<char> covered(size_t(s->N), 0);
  std::vector<const char*> payload;
  size_t off = 0;
  for (uint32_t bi = 0; bi < blob_count; ++bi) {
    Snapshot::Blob b{{-1, -1}, 0, 0, 0, 0};
    const uint32_t owners = r.get<uint32_t>("blob");
    if (owners < 1 || owners > 2) throw LoadError("blob", "blob must have one or two owners");
    for (uint32_t o = 0; o < owners; ++o) {
      const int32_t ow = r.get<int32_t>("blob");
      if (ow < 0 || ow >= s->N) throw LoadError("blob", "blob owner outside the layer range");
      if (covered[size_t(ow)]) throw LoadError("coverage", "layer covered by more than one blob");
      covered[size_t(ow)] = 1;
      b.owners[o] = ow;
    }
    b.start = r.get<int64_t>("blob");
    b.end = r.get<int64_t>("blob");
    if (b.start < 0 || b.start > b.end || b.end != s->L)
      throw LoadError("blob", "blob span must end at the history");
    const uint64_t plen = r.get<uint64_t>("blob");
    const uint64_t expect = 2ull * uint64_t(s->Hkv) * uint64_t(b.end - b.start) * uint64_t(s->hd) * 4ull;
    if (plen != expect) throw LoadError("blob", "payload length mismatch");
    payload.push_back(r.take(size_t(plen), "blob"));
    b.off = off;
    b.bytes = size_t(plen / 4) * s->esz;
    off += (b.bytes + 255) & ~size_t(255);
    s->blobs.push_back(b);
  }
  if (r.remaining() != 4) throw LoadError("blob", "trailing bytes after the blob table");
  for (int l = 0; l < s->N; ++l)
    if (!covered[size_t(l)])
      throw LoadError("coverage", "layer " + std::to_string(l) + " is not covered by any blob");
  s->total = off;
  const bool prof = std::getenv("KRUL_CONTAINER_PROFILE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  s->host.ensure(std::max<size_t>(off, 256));
  for (size_t bi = 0; bi < s->blobs.size(); ++bi)
    from_f32(payload[bi], s->esz, static_cast<char*>(s->host.p) + s->blobs[bi].off, s->blobs[bi].bytes / s->esz);
  const auto t1 = std::chrono::steady_clock::now();
  if (c) s->host.pin();
  const auto t2 = std::chrono::steady_clock::now();
  if (prof)
    std::fprintf(stderr, "[container] load %zu B: crc %.1f ms, convert %.1f ms, register %.1f ms\n", n, crc_ms,
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(t2 - t1).count());
  s->serial = next_serial();
  return s.release();
}

Snapshot* container_read_file(Ctx* c, const char* path, const uint64_t* expected_hash) {
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) fail(KRUL_E_SNAPSHOT, std::string("cannot open ") + path);
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    fail(KRUL_E_SNAPSHOT, std::string("cannot stat ") + path);
  }
  const size_t n = size_t(st.st_size);
  if (n == 0) {
    ::close(fd);
    return container_read(c, "", 0, expected_hash);
  }
  void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
  ::close(fd);
  if (m == MAP_FAILED) fail(KRUL_E_SNAPSHOT, std::string("cannot map ") + path);
  try {
    Snapshot* s = container_read(c, static_cast<const char*>(m), n, expected_hash);
    ::munmap(m, n);
    return s;
  } catch (...) {
    ::munmap(m, n);
    throw;
  }
}

}  // namespace kb
