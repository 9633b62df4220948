// host_kvcode.cpp — Huffman code construction, host codec and the snapshot
// encode step of the exponent-coded KV store (format: kvcode.hpp / kvcode.cu).
#include <algorithm>
#include <cstring>
#include <queue>
#include <thread>

#include "host.hpp"
#include "kvcode.hpp"

namespace kb {

// Huffman code lengths of the present symbols; frequencies are halved (kept
// >= 1) until the longest code fits kEcMaxLen, then codes are assigned
// canonically (by length, then symbol).
EcCode ec_build_code(const uint64_t* hist) {
  EcCode c;
  std::memset(&c, 0, sizeof c);
  std::vector<uint64_t> f(hist, hist + 256);
  int present = 0;
  for (int s = 0; s < 256; ++s) present += f[size_t(s)] > 0;
  if (present == 0) return c;
  if (present == 1) {
    for (int s = 0; s < 256; ++s)
      if (f[size_t(s)]) c.len[s] = 1;
  } else {
    for (;;) {
      // node weights, ties broken by node id for determinism
      using Node = std::pair<uint64_t, int>;
      std::priority_queue<Node, std::vector<Node>, std::greater<Node>> q;
      std::vector<int> parent(512, -1);
      int next = 256;
      for (int s = 0; s < 256; ++s)
        if (f[size_t(s)]) q.push({f[size_t(s)], s});
      while (q.size() > 1) {
        const Node a = q.top();
        q.pop();
        const Node b = q.top();
        q.pop();
        parent[size_t(a.second)] = next;
        parent[size_t(b.second)] = next;
        q.push({a.first + b.first, next++});
      }
      int maxlen = 0;
      for (int s = 0; s < 256; ++s) {
        if (!f[size_t(s)]) continue;
        int d = 0;
        for (int x = s; parent[size_t(x)] >= 0; x = parent[size_t(x)]) ++d;
        c.len[s] = uint8_t(d);
        maxlen = std::max(maxlen, d);
      }
      if (maxlen <= kEcMaxLen) break;
      for (auto& x : f)
        if (x) x = std::max<uint64_t>(1, x >> 1);
    }
  }
  // canonical assignment
  uint32_t code = 0;
  for (int l = 1; l <= kEcMaxLen; ++l) {
    for (int s = 0; s < 256; ++s)
      if (c.len[s] == l) {
        c.code[s] = code++;
        const int span = 1 << (kEcMaxLen - l);
        for (int i = 0; i < span; ++i) c.lut[(c.code[s] << (kEcMaxLen - l)) + uint32_t(i)] = uint16_t(s | (l << 8));
      }
    code <<= 1;
  }
  return c;
}

// Fills the chunk base table and lane counts of an image from per-stream
// word counts (stream t = chunk * 32 + lane); returns the absolute word
// offset of every stream and the total words.
static std::vector<uint32_t> ec_offsets(const std::vector<uint32_t>& words, uint64_t chunks, uint32_t* base,
                                        uint8_t* cnt, uint64_t* total) {
  std::vector<uint32_t> off(chunks * 32);
  uint64_t w = 0;
  for (uint64_t ch = 0; ch < chunks; ++ch) {
    base[ch] = uint32_t(w);
    for (int lane = 0; lane < 32; ++lane) {
      const uint32_t k = words[ch * 32 + uint64_t(lane)];
      off[ch * 32 + uint64_t(lane)] = uint32_t(w);
      cnt[ch * 32 + uint64_t(lane)] = uint8_t(k);
      w += k;
    }
  }
  base[chunks] = uint32_t(w);
  *total = w;
  return off;
}

std::vector<uint8_t> ec_encode_host(const uint16_t* x, uint64_t n, const EcCode& code) {
  const uint64_t chunks = (n + kEcChunk - 1) / kEcChunk;
  std::vector<uint32_t> words(chunks * 32, 0);
  for (uint64_t t = 0; t * kEcLaneSyms < n; ++t) {
    uint64_t bits = 0;
    for (uint64_t j = t * kEcLaneSyms; j < std::min<uint64_t>(n, (t + 1) * kEcLaneSyms); ++j)
      bits += code.len[(x[j] >> 7) & 0xFF];
    words[t] = uint32_t((bits + 31) / 32);
  }
  uint64_t total_words = 0;
  for (auto k : words) total_words += k;
  EcHeader h;
  size_t total = 0;
  ec_layout(n, total_words, &h, &total);
  std::vector<uint8_t> out(total, 0);
  std::memcpy(out.data(), &h, sizeof h);
  uint64_t tw = 0;
  const std::vector<uint32_t> off =
      ec_offsets(words, chunks, reinterpret_cast<uint32_t*>(out.data() + h.base_off), out.data() + h.cnt_off, &tw);
  uint8_t* sm = out.data() + h.sm_off;
  uint32_t* ex = reinterpret_cast<uint32_t*>(out.data() + h.exp_off);
  for (uint64_t t = 0; t * kEcLaneSyms < n; ++t) {
    uint32_t* o = ex + off[t];
    uint64_t acc = 0;
    int nb = 0;
    for (uint64_t j = t * kEcLaneSyms; j < std::min<uint64_t>(n, (t + 1) * kEcLaneSyms); ++j) {
      const uint32_t v = x[j];
      sm[j] = uint8_t(((v >> 8) & 0x80u) | (v & 0x7Fu));
      const uint32_t e = (v >> 7) & 0xFF;
      const int l = code.len[e];
      acc |= uint64_t(code.code[e]) << (64 - nb - l);
      nb += l;
      if (nb >= 32) {
        *o++ = uint32_t(acc >> 32);
        acc <<= 32;
        nb -= 32;
      }
    }
    if (nb > 0) *o = uint32_t(acc >> 32);
  }
  return out;
}

void ec_decode_host(const uint8_t* blob, const uint16_t* lut, uint16_t* out) {
  EcHeader h;
  std::memcpy(&h, blob, sizeof h);
  if (h.magic != kEcMagic) fail(KRUL_E_STATE_CORRUPTION, "coded KV blob has a bad header");
  const uint32_t* base = reinterpret_cast<const uint32_t*>(blob + h.base_off);
  const uint8_t* cnt = blob + h.cnt_off;
  const uint8_t* sm = blob + h.sm_off;
  const uint32_t* ex = reinterpret_cast<const uint32_t*>(blob + h.exp_off);
  const uint64_t n = h.n_elems;
  auto work = [&](uint64_t c0, uint64_t c1) {
    for (uint64_t ch = c0; ch < c1; ++ch) {
      uint32_t w = base[ch];
      for (int lane = 0; lane < 32; ++lane) {
        const uint64_t e0 = ch * kEcChunk + uint64_t(lane) * kEcLaneSyms;
        const uint32_t* p = ex + w;
        w += cnt[ch * 32 + uint64_t(lane)];
        uint64_t buf = 0;
        int have = 0;
        for (uint64_t j = e0; j < std::min<uint64_t>(n, e0 + kEcLaneSyms); ++j) {
          if (have < kEcMaxLen) {
            buf |= uint64_t(*p++) << (32 - have);
            have += 32;
          }
          const uint32_t e = lut[buf >> (64 - kEcMaxLen)];
          const int l = int(e >> 8);
          buf <<= l;
          have -= l;
          const uint32_t s = sm[j];
          out[j] = uint16_t(((s & 0x80u) << 8) | ((e & 0xFFu) << 7) | (s & 0x7Fu));
        }
      }
    }
  };
  const uint64_t chunks = h.n_chunks;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (chunks < 64 || hw == 1) {
    work(0, chunks);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t per = (chunks + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const uint64_t a = std::min<uint64_t>(chunks, t * per), b = std::min<uint64_t>(chunks, a + per);
    if (a < b) th.emplace_back(work, a, b);
  }
  for (auto& x : th) x.join();
}

// Raw (compute-dtype) bytes of blob b: the host store itself, or the blob
// decoded into `tmp` when the store is coded.
const char* snapshot_raw_blob(const Snapshot& s, int b, std::vector<uint16_t>& tmp) {
  const auto& bl = s.blobs[size_t(b)];
  const char* base = static_cast<const char*>(s.host.p);
  if (!s.coded) return base + bl.off;
  tmp.resize(bl.bytes / 2 + 1);
  if (bl.bytes) ec_decode_host(reinterpret_cast<const uint8_t*>(base + bl.coff), s.code->lut, tmp.data());
  return reinterpret_cast<const char*>(tmp.data());
}

// Encodes the raw bf16 blobs staged on the device (dev_raw + blob.off) into
// the coded host store: one exponent histogram over the snapshot, one code,
// per blob lane sizes -> host scan -> header + lane table uploaded into the
// device image -> encode kernel -> one D2H of the whole coded image.
void snapshot_encode(Ctx& c, Snapshot& s, const char* dev_raw, cudaStream_t st) {
  if (s.esz != 2) fail(KRUL_E_CONFIG, "exponent coding needs a bf16 store");
  for (const auto& b : s.blobs)
    if (!ec_fits(b.bytes / 2)) fail(KRUL_E_SNAPSHOT, "blob too large for the coded store (u32 image offsets)");
  DevBuf d_hist, d_code, d_words, d_img;
  auto* hist = static_cast<unsigned long long*>(d_hist.ensure(256 * 8));
  KB_CUDA(cudaMemsetAsync(hist, 0, 256 * 8, st));
  uint64_t chunks_total = 0;
  std::vector<uint64_t> chunk0(s.blobs.size());
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    const int64_t n = int64_t(b.bytes / 2);
    launch_exp_hist(st, dev_raw + b.off, n, hist);
    chunk0[bi] = chunks_total;
    chunks_total += uint64_t((n + kEcChunk - 1) / kEcChunk);
  }
  uint64_t h_hist[256];
  KB_CUDA(cudaMemcpyAsync(h_hist, hist, sizeof h_hist, cudaMemcpyDeviceToHost, st));
  KB_CUDA(cudaStreamSynchronize(st));
  auto code = std::make_unique<EcCode>(ec_build_code(h_hist));
  char* dc = static_cast<char*>(d_code.ensure(256 * 4 + 256));
  KB_CUDA(cudaMemcpyAsync(dc, code->code, 256 * 4, cudaMemcpyHostToDevice, st));
  KB_CUDA(cudaMemcpyAsync(dc + 1024, code->len, 256, cudaMemcpyHostToDevice, st));
  auto* words = static_cast<uint32_t*>(d_words.ensure(std::max<uint64_t>(chunks_total, 1) * 32 * 4));
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    launch_ec_lane_words(st, dev_raw + b.off, int64_t(b.bytes / 2), reinterpret_cast<const uint8_t*>(dc + 1024),
                         words + chunk0[bi] * 32);
  }
  std::vector<uint32_t> hw(chunks_total * 32);
  if (!hw.empty())
    KB_CUDA(cudaMemcpyAsync(hw.data(), words, hw.size() * 4, cudaMemcpyDeviceToHost, st));
  KB_CUDA(cudaStreamSynchronize(st));
  // layout of the coded image (blobs 256-B aligned, like the raw store):
  // per blob the chunk base table + lane counts (host, from the word
  // counts), and the absolute stream offsets the encode kernel writes at
  std::vector<EcHeader> hdr(s.blobs.size());
  std::vector<std::vector<uint8_t>> tables(s.blobs.size());
  std::vector<uint32_t> offs(chunks_total * 32);
  size_t off = 0;
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    auto& b = s.blobs[bi];
    const uint64_t n = b.bytes / 2;
    const uint64_t ch = (n + kEcChunk - 1) / kEcChunk;
    std::vector<uint32_t> wv(hw.begin() + int64_t(chunk0[bi] * 32), hw.begin() + int64_t((chunk0[bi] + ch) * 32));
    uint64_t w = 0;
    for (auto k : wv) w += k;
    size_t total = 0;
    ec_layout(n, w, &hdr[bi], &total);
    // header + base table + counts: bytes [0, sm_off) of the image
    tables[bi].assign(hdr[bi].sm_off, 0);
    std::memcpy(tables[bi].data(), &hdr[bi], sizeof(EcHeader));
    uint64_t tw = 0;
    const std::vector<uint32_t> o = ec_offsets(
        wv, ch, reinterpret_cast<uint32_t*>(tables[bi].data() + hdr[bi].base_off),
        tables[bi].data() + hdr[bi].cnt_off, &tw);
    std::copy(o.begin(), o.end(), offs.begin() + int64_t(chunk0[bi] * 32));
    b.coff = off;
    b.cbytes = n ? total : 0;
    b.ec_chunks = uint32_t(ch);
    off += (b.cbytes + 255) & ~size_t(255);
  }
  const size_t ctotal = std::max<size_t>(off, 256);
  char* img = static_cast<char*>(d_img.ensure(ctotal));
  KB_CUDA(cudaMemsetAsync(img, 0, ctotal, st));
  // tables + stream offsets, staged through pinned memory
  PinnedBuf meta;
  size_t meta_bytes = offs.size() * 4;
  for (const auto& t : tables) meta_bytes += t.size();
  char* mp = static_cast<char*>(meta.ensure(std::max<size_t>(meta_bytes, 64)));
  std::memcpy(mp, offs.data(), offs.size() * 4);
  uint32_t* d_offs = static_cast<uint32_t*>(d_words.p);  // reuse: same size as the word counts
  if (!offs.empty()) KB_CUDA(cudaMemcpyAsync(d_offs, mp, offs.size() * 4, cudaMemcpyHostToDevice, st));
  size_t mo = offs.size() * 4;
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    if (!b.cbytes) continue;
    std::memcpy(mp + mo, tables[bi].data(), tables[bi].size());
    KB_CUDA(cudaMemcpyAsync(img + b.coff, mp + mo, tables[bi].size(), cudaMemcpyHostToDevice, st));
    mo += tables[bi].size();
  }
  for (size_t bi = 0; bi < s.blobs.size(); ++bi) {
    const auto& b = s.blobs[bi];
    if (!b.cbytes) continue;
    char* base = img + b.coff;
    launch_ec_encode(st, dev_raw + b.off, int64_t(b.bytes / 2), reinterpret_cast<const uint32_t*>(dc),
                     reinterpret_cast<const uint8_t*>(dc + 1024), d_offs + chunk0[bi] * 32,
                     reinterpret_cast<uint8_t*>(base + hdr[bi].sm_off),
                     reinterpret_cast<uint32_t*>(base + hdr[bi].exp_off));
  }
  s.host.ensure(ctotal);
  KB_CUDA(cudaMemcpyAsync(s.host.p, img, ctotal, cudaMemcpyDeviceToHost, st));
  uint16_t* lut = static_cast<uint16_t*>(s.lut_dev.ensure(sizeof code->lut));
  KB_CUDA(cudaMemcpyAsync(lut, code->lut, sizeof code->lut, cudaMemcpyHostToDevice, st));
  KB_CUDA(cudaStreamSynchronize(st));
  s.code = std::move(code);
  s.coded = true;
  s.ctotal = ctotal;
  s.serial = next_serial();
}

}  // namespace kb
