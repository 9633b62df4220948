// host_restore.cpp — compressed KV store (pinned host blobs) and the
// two-stream restoration DAG.
//
// Restore (scheduler.cpp:320-400, re-designed for the GPU): the reference runs
// the whole prefix recompute on the caller thread while one loader thread
// expands blobs, then splices per layer. Here both streams write disjoint
// position ranges of the same paged cache, so there is no splice:
//   load stream    : per blob (service order = shallowest owner):
//                    cudaMemcpyAsync pinned -> staging (K4),
//                    expand kernel staging -> pages of each owner (K5),
//                    event loaded[owner]
//   compute stream : pyramid prefix recompute layer by layer (K6),
//                    event computed[l]
//   new stream     : (restore_and_prefill) new-input prefill of layer l waits
//                    on computed[l] and loaded[l] only (K7), so it overlaps the
//                    remaining restore instead of trailing it.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "host.hpp"

namespace kb {

static float bf16_to_f32(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
static uint16_t f32_to_bf16(float f) {  // round to nearest even (== __float2bfloat16_rn)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// Layout blobs of a snapshot from (strategy, plan).
static void layout_blobs(Ctx& c, Snapshot& s, bool alloc_host = true) {
  const auto specs = blob_specs(s.p, s.L, s.pairs.data(), int(s.pairs.size()));
  size_t off = 0;
  s.blobs.clear();
  for (const auto& sp : specs) {
    Snapshot::Blob b;
    b.owners[0] = sp.owners[0];
    b.owners[1] = sp.owners[1];
    b.start = sp.start;
    b.end = sp.end;
    b.off = off;
    b.bytes = size_t(2) * c.cfg.Hkv * size_t(sp.end - sp.start) * c.cfg.hd * c.esz;
    off += (b.bytes + 255) & ~size_t(255);
    s.blobs.push_back(b);
  }
  s.total = off;
  if (alloc_host) s.host.ensure(std::max<size_t>(off, 256));
}

static bool coding_on(const Ctx& c) {
  static const bool env = [] {
    const char* v = std::getenv("KRUL_KV_CODING");
    return !(v && v[0] == '0');
  }();
  return env && c.kv_coding && c.esz == 2;
}

static Snapshot* new_snapshot(Ctx& c, const krul_pair* pairs, int np, const int64_t* p, int64_t L,
                              int mode) {
  auto* s = new Snapshot;
  s->ctx = &c;
  s->esz = c.esz;
  s->config_hash = config_hash(c.cfg);
  s->N = c.cfg.N;
  s->Hkv = c.cfg.Hkv;
  s->hd = c.cfg.hd;
  s->L = L;
  s->mode = mode;
  s->pairs.assign(pairs, pairs + np);
  s->p.assign(p, p + c.cfg.N);
  s->serial = next_serial();
  return s;
}

// kvstore.cpp:243-314 on the device (K8): gather + mean-merge into a device
// staging image of all blobs, one D2H into pinned host memory.
Snapshot* snapshot_compress(Ctx& c, Conv& conv, const krul_pair* pairs, int np, const int64_t* p,
                            int64_t L, int mode) {
  if (mode != KRUL_MERGE_MEAN && mode != KRUL_MERGE_KEEP_DEEPER) fail(KRUL_E_CONFIG, "unknown merge mode");
  if (conv.len != L) fail(KRUL_E_SNAPSHOT, "cache span does not cover the plan's history");
  std::unique_ptr<Snapshot> s(new_snapshot(c, pairs, np, p, L, mode));
  layout_blobs(c, *s, false);
  bool code = coding_on(c);
  for (const auto& b : s->blobs) code = code && ec_fits(b.bytes / 2);  // u32 image offsets
  KB_CUDA(cudaSetDevice(c.device));
  cudaStream_t st = c.s_load;
  char* stg = static_cast<char*>(c.staging.ensure(std::max<size_t>(s->total, 256)));
  for (const auto& b : s->blobs) {
    const bool pair = b.owners[1] >= 0;
    const int deep = pair ? b.owners[1] : b.owners[0];
    const int shallow = pair && mode == KRUL_MERGE_MEAN ? b.owners[0] : -1;
    const int64_t merge_from = pair ? p[b.owners[0]] : L;
    launch_compress(c, st, conv, deep, shallow, b.start, L, merge_from, stg + b.off);
  }
  // a blob past the coded image's u32 offsets (> 4 GiB) keeps the snapshot raw
  const bool fits = std::all_of(s->blobs.begin(), s->blobs.end(), [](const auto& b) { return ec_fits(b.bytes / 2); });
  if (code && s->total && fits) {
    snapshot_encode(c, *s, stg, st);  // coded host store, one D2H of the coded image
  } else {
    s->host.ensure(std::max<size_t>(s->total, 256));
    if (s->total) KB_CUDA(cudaMemcpyAsync(s->host.p, stg, s->total, cudaMemcpyDeviceToHost, st));
  }
  KB_CUDA(cudaStreamSynchronize(st));
  return s.release();
}

Snapshot* snapshot_from_host(Ctx& c, const krul_pair* pairs, int np, const int64_t* p, int64_t L,
                             int mode, const float* const* k, const float* const* v) {
  std::unique_ptr<Snapshot> s(new_snapshot(c, pairs, np, p, L, mode));
  layout_blobs(c, *s);
  for (size_t bi = 0; bi < s->blobs.size(); ++bi) {
    const auto& b = s->blobs[bi];
    const size_t n = size_t(c.cfg.Hkv) * size_t(b.end - b.start) * c.cfg.hd;
    char* dst = static_cast<char*>(s->host.p) + b.off;
    for (int kv = 0; kv < 2; ++kv) {
      const float* src = kv == 0 ? k[bi] : v[bi];
      if (c.esz == 4) {
        std::memcpy(dst + kv * n * 4, src, n * 4);
      } else {
        uint16_t* o = reinterpret_cast<uint16_t*>(dst) + kv * n;
        for (size_t i = 0; i < n; ++i) o[i] = f32_to_bf16(src[i]);
      }
    }
  }
  return s.release();
}

void snapshot_blob_f32(const Snapshot& s, int b, int64_t row0, int64_t rows, float* k, float* v) {
  const auto& bl = s.blobs[size_t(b)];
  const int64_t brows = bl.end - bl.start;
  const size_t esz = s.esz;
  std::vector<uint16_t> tmp;
  const char* base = snapshot_raw_blob(s, b, tmp);
  for (int kv = 0; kv < 2; ++kv) {
    float* out = kv == 0 ? k : v;
    if (!out) continue;
    for (int g = 0; g < s.Hkv; ++g)
      for (int64_t r = 0; r < rows; ++r)
        for (int t = 0; t < s.hd; ++t) {
          const size_t src = ((size_t(kv) * s.Hkv + g) * size_t(brows) + size_t(row0 + r)) * s.hd + t;
          const size_t dst = (size_t(g) * size_t(rows) + size_t(r)) * s.hd + t;
          out[dst] = esz == 4 ? reinterpret_cast<const float*>(base)[src]
                              : bf16_to_f32(reinterpret_cast<const uint16_t*>(base)[src]);
        }
  }
}

// kvstore.cpp:316-343 (host view of the pinned store).
void snapshot_expand(const Snapshot& s, int layer, float* k, float* v, int64_t* start,
                     int64_t* end) {
  int found = -1;
  for (size_t b = 0; b < s.blobs.size() && found < 0; ++b)
    if (s.blobs[b].owners[0] == layer || (s.blobs[b].owners[1] == layer && layer >= 0))
      found = int(b);
  if (found < 0)
    fail(KRUL_E_RESTORATION_GAP, "layer " + std::to_string(layer) + " is not covered by any stored blob");
  const auto& bl = s.blobs[size_t(found)];
  const int64_t ws = s.p[size_t(layer)], we = s.L;
  if (ws < bl.start || we != bl.end) fail(KRUL_E_RESTORATION_GAP, "stored span does not cover the load span");
  *start = ws;
  *end = we;
  snapshot_blob_f32(s, found, ws - bl.start, we - ws, k, v);
}

uint64_t next_serial() {
  static std::atomic<uint64_t> s{1};
  return s.fetch_add(1);
}

// The restore DAG on the ctx streams (all asynchronous, joined back into
// s_comp). Events: ev[0] launch, ev[1] compute end, ev[2] load end, ev[3]
// end, ev[4] H2D end, ev[5..5+N) computed[l], then loaded[l], then newp[l].
// Pipelined batch mode (restore_batch): tokens already on the device
// (uploaded on the load stream, `tok_ready`), the coded / raw staging of this
// item's slot, no join into s_comp at the end (the next conversation's copies
// start under this one's new-input prefill tail), logits read back on the
// prefill stream.
struct PipeItem {
  const int32_t* d_tok = nullptr;
  const int32_t* d_new = nullptr;
  cudaEvent_t tok_ready = nullptr;
  char* stg = nullptr;
  char* cstg = nullptr;
  float* logits_host = nullptr;  // pinned, may be null
  // graph mode (the item's DAG captured once, launched on its own stream):
  // the item's own dependency marks (no timing events, so the graph never
  // refers to the ctx's restore-graph events) and the external hand-offs to
  // the neighbouring items -- the previous item's recompute end (workspace
  // set 0) and new-input prefill end (set 1)
  const Mark* ev = nullptr;
  cudaEvent_t wait_comp = nullptr, rec_comp = nullptr, wait_new = nullptr, rec_new = nullptr;
};
static void enqueue_restore(Ctx& c, Conv& conv, Snapshot& snap, int64_t L, const int32_t* tp_hist,
                            const int32_t* tp_new, int64_t n_new, float* lp, double* h2d_out,
                            double* expand_out, const PipeItem* pipe = nullptr) {
  const Cfg& g = c.cfg;
  const std::vector<int64_t>& p = snap.p;
  const Mark* E = pipe && pipe->ev ? pipe->ev : c.rg.ev.data();
  const Mark &ev0 = E[0], &ev_c_end = E[1], &ev_l_end = E[2], &ev_end = E[3], &ev_h2d_end = E[4];
  const Mark* computed = E + 5;
  const Mark* loaded = computed + g.N;
  const Mark* newp = loaded + g.N;
  cudaStream_t sc = c.s_comp, sl = c.s_load;
  char* stg = pipe ? pipe->stg : static_cast<char*>(c.staging.p);
  char* cstg = pipe ? pipe->cstg : static_cast<char*>(c.cstaging.p);
  float* d_logits = static_cast<float*>(c.ws_logits.p);

  const int32_t* d_tok;
  const int32_t* d_new;
  cudaEvent_t tok_ready;
  if (pipe) {
    record_mark(ev0, sl);
    d_tok = pipe->d_tok;
    d_new = pipe->d_new;
    tok_ready = pipe->tok_ready;
    KB_CUDA(cudaStreamWaitEvent(sc, tok_ready, 0));
    KB_CUDA(cudaStreamWaitEvent(c.s_exp, tok_ready, 0));
  } else {
    // token uploads first: a small H2D queued behind the blob copies on the
    // copy engine would hold the recompute back for the whole load (~14 ms)
    record_mark(ev0, sc);
    d_tok = upload_tokens(c, sc, tp_hist, std::max<int64_t>(p[0], 0), c.ws_tok);
    d_new = tp_new ? upload_tokens(c, sc, tp_new, n_new, c.ws_tok2) : nullptr;
    tok_ready = c.event();
    KB_CUDA(cudaEventRecord(tok_ready, sc));
    KB_CUDA(cudaStreamWaitEvent(sl, tok_ready, 0));
    KB_CUDA(cudaStreamWaitEvent(c.s_exp, ev0.dep, 0));
  }
  // ---- load stream: K4 H2D copies back to back on the copy engine; K5
  // expand kernels on their own stream behind each blob's copy, so the PCIe
  // link never idles while a scatter runs.
  double h2d = 0, expand_bytes = 0;
  std::vector<cudaEvent_t> copied(snap.blobs.size());
  for (size_t bi = 0; bi < snap.blobs.size(); ++bi) {
    const auto& b = snap.blobs[bi];
    copied[bi] = c.event();
    if (snap.coded && b.cbytes) {  // coded image -> cstaging, decoded on the expand stream
      KB_CUDA(cudaMemcpyAsync(cstg + b.coff, static_cast<char*>(snap.host.p) + b.coff, b.cbytes,
                              cudaMemcpyHostToDevice, sl));
      h2d += double(b.cbytes);
    } else if (!snap.coded && b.bytes) {
      KB_CUDA(cudaMemcpyAsync(stg + b.off, static_cast<char*>(snap.host.p) + b.off, b.bytes,
                              cudaMemcpyHostToDevice, sl));
      h2d += double(b.bytes);
    }
    KB_CUDA(cudaEventRecord(copied[bi], sl));
  }
  record_mark(ev_h2d_end, sl);
  for (size_t bi = 0; bi < snap.blobs.size(); ++bi) {
    const auto& b = snap.blobs[bi];
    KB_CUDA(cudaStreamWaitEvent(c.s_exp, copied[bi], 0));
    static const bool fuse_env = [] {
      const char* v = std::getenv("KRUL_DECODE_EXPAND");
      return !(v && v[0] == '0');
    }();
    if (snap.coded && b.cbytes && g.hd == kEcLaneSyms && c.esz == 2 && fuse_env) {
      // decode straight into the owners' pages (one pass, one launch)
      const int64_t from[2] = {p[size_t(b.owners[0])], b.owners[1] >= 0 ? p[size_t(b.owners[1])] : L};
      // blobs before the last one decode beside the new-input prefill: a
      // smaller grid (KRUL_DEXP_CPS CTAs per SM) leaves the prefill's GEMMs
      // their issue slots; the last blob is on the critical path and gets
      // the whole GPU
      static const int cps_env = [] {
        const char* v = std::getenv("KRUL_DEXP_CPS");
        return v ? std::atoi(v) : 4;
      }();
      const bool last = bi + 1 == snap.blobs.size();
      launch_ec_decode_expand(c, c.s_exp, cstg + b.coff, int64_t(b.ec_chunks), snap.lut_dev.as<uint16_t>(),
                              b.start, L, conv, b.owners, from, double(b.cbytes), last ? 4 : cps_env);
      for (int o : b.owners) {
        if (o < 0) continue;
        expand_bytes += 2.0 * double(L - p[size_t(o)]) * g.Hkv * g.hd * double(c.esz) * 2.0;
        record_mark(loaded[o], c.s_exp);
      }
      continue;
    }
    if (snap.coded && b.cbytes) {
      cudaEvent_t kt0 = kt_begin(c, c.s_exp);
      launch_ec_decode(c.s_exp, cstg + b.coff, int64_t(b.ec_chunks), snap.lut_dev.as<uint16_t>(), stg + b.off);
      kt_end(c, c.s_exp, kt0, KT_DECODE, 0.0, double(b.cbytes) + double(b.bytes));  // coded read + raw write
    }
    for (int o : b.owners) {
      if (o < 0) continue;
      launch_expand(c, c.s_exp, stg + b.off, b.start, L, conv, o, p[size_t(o)]);
      expand_bytes += 2.0 * double(L - p[size_t(o)]) * g.Hkv * g.hd * double(c.esz) * 2.0;
      record_mark(loaded[o], c.s_exp);
    }
  }
  record_mark(ev_l_end, c.s_exp);
  static const bool fused_env = [] {
    const char* v = std::getenv("KRUL_FUSED");
    return !(v && v[0] == '0');
  }();
  const bool has_new = d_new != nullptr;  // host tokens (single restore) or device tokens (pipelined)
  const bool fused = has_new && fused_env && c.fused;
  if (fused) {
    // ---- K6 + K7 fused: the recompute rows ride in the new-input prefill's
    // layer steps (forward_fused), one weight pass per layer
    cudaStream_t sn = c.s_new;
    KB_CUDA(cudaStreamWaitEvent(sn, tok_ready, 0));
    conv.len = L;
    forward_fused(c, sn, 1, conv, d_new, n_new, L, d_tok, p, d_logits, loaded, computed, newp, &ev_c_end);
    record_mark(ev_end, sn);
    KB_CUDA(cudaStreamWaitEvent(sc, ev_end.dep, 0));
    KB_CUDA(cudaStreamWaitEvent(sc, ev_l_end.dep, 0));
    KB_CUDA(cudaStreamWaitEvent(sc, ev_h2d_end.dep, 0));
    if (lp) KB_CUDA(cudaMemcpyAsync(lp, d_logits, size_t(g.V) * 4, cudaMemcpyDeviceToHost, sc));
    *h2d_out = h2d;
    *expand_out = expand_bytes;
    return;
  }
  // ---- compute stream: K6 pyramid recompute
  if (pipe && pipe->wait_comp) KB_CUDA(cudaStreamWaitEvent(sc, pipe->wait_comp, cudaEventWaitExternal));
  if (p[0] > 0) {
    enqueue_partial(c, sc, conv, d_tok, p, false, computed);
  } else {
    for (int l = 0; l < g.N; ++l) record_mark(computed[l], sc);
  }
  record_mark(ev_c_end, sc);
  if (pipe && pipe->rec_comp) KB_CUDA(cudaEventRecordWithFlags(pipe->rec_comp, sc, cudaEventRecordExternal));
  // ---- new-input prefill (K7) on its own stream, layer l behind
  // computed[l] and loaded[l], so it tracks the load events while the
  // recompute runs (KRUL_TWO_STREAM=0: same stream, after the recompute).
  static const bool two_stream_env = [] {
    const char* v = std::getenv("KRUL_TWO_STREAM");
    return !(v && v[0] == '0');
  }();
  const bool two_stream = two_stream_env && c.two_stream;
  if (has_new) {
    cudaStream_t sn = two_stream ? c.s_new : sc;
    if (two_stream) KB_CUDA(cudaStreamWaitEvent(sn, tok_ready, 0));
    if (pipe && pipe->wait_new) KB_CUDA(cudaStreamWaitEvent(sn, pipe->wait_new, cudaEventWaitExternal));
    std::vector<cudaEvent_t> waits;
    for (int l = 0; l < g.N; ++l) waits.push_back(computed[l].dep);
    for (int l = 0; l < g.N; ++l) waits.push_back(loaded[l].dep);
    conv.len = L;
    forward_rows(c, sn, 1, conv, d_new, n_new, L, d_logits, &waits, newp);
    if (pipe && pipe->logits_host)
      KB_CUDA(cudaMemcpyAsync(pipe->logits_host, d_logits, size_t(g.V) * 4, cudaMemcpyDeviceToHost, sn));
    record_mark(ev_end, sn);
    if (pipe && pipe->rec_new) KB_CUDA(cudaEventRecordWithFlags(pipe->rec_new, sn, cudaEventRecordExternal));
    if (pipe) {  // no join: the next conversation's restore starts under this tail
      *h2d_out = h2d;
      *expand_out = expand_bytes;
      return;
    }
    if (two_stream) KB_CUDA(cudaStreamWaitEvent(sc, ev_end.dep, 0));
  } else {
    record_mark(ev_end, sc);
  }
  // join every forked stream back into s_comp
  KB_CUDA(cudaStreamWaitEvent(sc, ev_l_end.dep, 0));
  KB_CUDA(cudaStreamWaitEvent(sc, ev_h2d_end.dep, 0));
  if (lp) KB_CUDA(cudaMemcpyAsync(lp, d_logits, size_t(g.V) * 4, cudaMemcpyDeviceToHost, sc));
  *h2d_out = h2d;
  *expand_out = expand_bytes;
}

// scheduler.cpp:320-336 checks, then the DAG. The DAG of a repeated
// (snapshot, conversation, shape) is captured once into a CUDA graph and
// replayed: one host launch instead of ~600, so the streams start
// back-to-back on the device.
static void check_restore(Ctx& c, Conv& conv, Snapshot& snap, const int32_t* hist, int64_t L,
                          const int32_t* new_tok, int64_t n_new) {
  const Cfg& g = c.cfg;
  if (snap.config_hash != config_hash(g)) fail(KRUL_E_SNAPSHOT, "snapshot was taken under a different model config");
  if (snap.esz != c.esz || (snap.host.pageable && !snap.host.registered))
    fail(KRUL_E_SNAPSHOT, "snapshot store is not pinned in this context's dtype (load it with the context)");
  if (L != snap.L) fail(KRUL_E_RESTORATION_GAP, "history length does not match the snapshot");
  const std::vector<int64_t>& p = snap.p;
  const int m = validate_plan_snapshot(p, L, snap);
  if (m) {
    const int base = validate_plan(L, p, snap.pairs.data(), int(snap.pairs.size()));
    if (base & 7) fail(KRUL_E_PLAN_INVALID, "plan violation (bounds/monotonicity)");
    if (base & 8) fail(KRUL_E_RESTORATION_GAP, "coverage: pair blob span misses the shallow member's load span");
    fail(KRUL_E_RESTORATION_GAP, "coverage: stored span does not cover its load span");
  }
  check_tokens(c, hist, L);
  if (new_tok) {
    if (n_new <= 0) fail(KRUL_E_RESTORATION_GAP, "prefill over preloaded history requires new input tokens");
    check_tokens(c, new_tok, n_new);
  }
  if (L + std::max<int64_t>(n_new, 0) > conv.capacity) fail(KRUL_E_CONFIG, "history exceeds the conversation capacity");
}

void restore(Ctx& c, Conv& conv, Snapshot& snap, const int32_t* hist, int64_t L,
             krul_restore_stats* st, const int32_t* new_tok, int64_t n_new, float* logits,
             double* ttft_ms) {
  const Cfg& g = c.cfg;
  check_restore(c, conv, snap, hist, L, new_tok, n_new);
  const std::vector<int64_t>& p = snap.p;
  KB_CUDA(cudaSetDevice(c.device));
  const int64_t nh = std::max<int64_t>(p[0], 0), nn = new_tok ? n_new : 0;

  // pinned token / logits staging (the previous restore has completed)
  int32_t* tp = static_cast<int32_t*>(c.tok_pin.ensure(size_t(nh + nn + 1) * 4));
  if (nh) std::memcpy(tp, hist, size_t(nh) * 4);
  if (nn) std::memcpy(tp + nh, new_tok, size_t(nn) * 4);
  float* lp = (logits && new_tok) ? static_cast<float*>(c.logits_pin.ensure(size_t(g.V) * 4)) : nullptr;
  c.staging.ensure(std::max<size_t>(snap.total, 256));
  if (snap.coded) c.cstaging.ensure(std::max<size_t>(snap.ctotal, 256));
  c.ws_logits.ensure(size_t(g.V) * 4);

  auto& G = c.rg;
  const bool same = G.snap_serial == snap.serial && G.conv_serial == conv.serial && G.L == L && G.n_new == nn &&
                    G.kt_on == c.kt.on && G.logits == (lp != nullptr) &&
                    G.capture_probs == c.capture_probs && G.buf_gen == g_buf_gen.load() &&
                    G.two_stream == c.two_stream && G.fused == c.fused && G.timeline == c.timeline &&
                    G.span == c.span_on;
  if (!same) {
    c.drop_graph();
    G.snap_serial = snap.serial;
    G.conv_serial = conv.serial;
    G.L = L;
    G.n_new = nn;
    G.kt_on = c.kt.on;
    G.logits = lp != nullptr;
    G.capture_probs = c.capture_probs;
    G.two_stream = c.two_stream;
    G.fused = c.fused;
    G.timeline = c.timeline;
    G.span = c.span_on;
    G.ev.resize(size_t(5 + 3 * g.N));
    for (size_t i = 0; i < G.ev.size(); ++i) {
      auto& m = G.ev[i];
      KB_CUDA(cudaEventCreateWithFlags(&m.dep, cudaEventDisableTiming));
      if (i < 5 || c.timeline) KB_CUDA(cudaEventCreate(&m.tim));  // per-layer timing on request
    }
    G.buf_gen = g_buf_gen.load();
  }
  static const bool graphs_env = [] {
    const char* v = std::getenv("KRUL_GRAPHS");
    return !(v && v[0] == '0');
  }();
  const bool graphs = c.use_graphs && graphs_env;
  const int32_t* tp_new = new_tok ? tp + nh : nullptr;
  if (c.span_on) {  // fresh stamps for this restore: entry = max, exit = 0
    unsigned long long* sp = static_cast<unsigned long long*>(c.span_buf.p);
    KB_CUDA(cudaMemsetAsync(sp, 0xFF, sizeof(unsigned long long) * Ctx::kSpanSlots, c.s_comp));
    KB_CUDA(cudaMemsetAsync(sp + Ctx::kSpanSlots, 0, sizeof(unsigned long long) * Ctx::kSpanSlots, c.s_comp));
  }
  if (graphs && G.exec) {
    KB_CUDA(cudaGraphLaunch(G.exec, c.s_comp));
    g_launches.fetch_add(G.launches);
    conv.len = L + nn;
  } else {
    if (!G.exec) {
      c.kt.recs.clear();
      c.kt.next = 0;
    }
    c.reset_events();
    c.span_next = 0;  // slots in enqueue order: identical on every replay
    c.span_bytes.clear();
    if (graphs && G.seen >= 1) {
      const uint64_t l0 = g_launches.load();
      KB_CUDA(cudaStreamBeginCapture(c.s_comp, cudaStreamCaptureModeRelaxed));
      try {
        enqueue_restore(c, conv, snap, L, tp, tp_new, nn, lp, &G.h2d, &G.expand_bytes);
      } catch (...) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(c.s_comp, &junk);
        if (junk) cudaGraphDestroy(junk);
        c.use_graphs = false;
        throw;
      }
      cudaGraph_t graph = nullptr;
      KB_CUDA(cudaStreamEndCapture(c.s_comp, &graph));
      const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        G.exec = nullptr;
        c.use_graphs = false;
        fail(KRUL_E_CUDA, std::string("restore graph instantiation failed: ") + cudaGetErrorString(ie));
      }
      G.launches = g_launches.load() - l0;
      G.buf_gen = g_buf_gen.load();
      KB_CUDA(cudaGraphLaunch(G.exec, c.s_comp));
    } else {
      enqueue_restore(c, conv, snap, L, tp, tp_new, nn, lp, &G.h2d, &G.expand_bytes);
      ++G.seen;
      G.buf_gen = g_buf_gen.load();  // workspaces sized by this run
    }
    conv.len = L + nn;
  }
  KB_CUDA(cudaStreamSynchronize(c.s_comp));
  if (lp) std::memcpy(logits, lp, size_t(g.V) * 4);

  std::vector<cudaEvent_t> E;
  for (const auto& mk : G.ev) E.push_back(mk.tim);
  float tc = 0, tl = 0, te = 0, th = 0;
  KB_CUDA(cudaEventElapsedTime(&tc, E[0], E[1]));
  KB_CUDA(cudaEventElapsedTime(&tl, E[0], E[2]));
  KB_CUDA(cudaEventElapsedTime(&te, E[0], E[3]));
  KB_CUDA(cudaEventElapsedTime(&th, E[0], E[4]));
  if (ttft_ms) *ttft_ms = te;
  // the per-layer timeline is read lazily (restore_timeline): ~100 event
  // queries would otherwise sit inside every call's host time
  c.tl_pending = true;
  c.tl_has_new = new_tok != nullptr;
  c.tl_compute.assign(size_t(g.N), 0.0);
  c.tl_h2d_ms = th;
  if (st) {
    Cost cm;
    cm.kv_dim = g.kvd();
    cm.q_dim = g.qd();
    cm.ffn_hidden = g.F;
    cm.ffn_kind = g.ffn_kind;
    cm.bpe = double(c.esz);
    double fl = 0;
    for (int64_t x : p) fl += cm.layer_flops(x, g.d);
    const double mk = std::max(tc, tl);
    st->compute_ms = tc;
    st->load_ms = tl;
    st->restore_ms = mk;
    st->bubble_compute = mk > 0 && p[0] > 0 ? (mk - tc) / mk : 0.0;
    st->bubble_load = mk > 0 && G.h2d > 0 ? (mk - tl) / mk : 0.0;
    st->h2d_bytes = G.h2d;
    st->expand_bytes = G.expand_bytes;
    st->recompute_flops = fl;
    st->h2d_ms = th;
  }
}

// measured per-layer timeline (ms from restore launch) of the last restore,
// the device counterpart of PipelineTrace (scheduler.hpp:71-97)
void restore_timeline(Ctx& c) {
  if (!c.tl_pending) return;
  const Cfg& g = c.cfg;
  const auto& E = c.rg.ev;
  c.tl_compute.assign(size_t(g.N), 0.0);
  c.tl_load.assign(size_t(g.N), 0.0);
  c.tl_new.assign(size_t(g.N), 0.0);
  for (int l = 0; l < g.N && c.rg.timeline; ++l) {
    float a = 0, b = 0, e = 0;
    KB_CUDA(cudaEventElapsedTime(&a, E[0].tim, E[size_t(5 + l)].tim));
    KB_CUDA(cudaEventElapsedTime(&b, E[0].tim, E[size_t(5 + g.N + l)].tim));
    c.tl_compute[size_t(l)] = a;
    c.tl_load[size_t(l)] = b;
    if (c.tl_has_new) {
      KB_CUDA(cudaEventElapsedTime(&e, E[0].tim, E[size_t(5 + 2 * g.N + l)].tim));
      c.tl_new[size_t(l)] = e;
    }
  }
  c.tl_pending = false;
}

// Pipelined restore of a batch of conversations (configs[3]: many
// conversations per GPU). The DAGs are enqueued back to back without a join:
// conversation i+1's token upload and blob copies start on the load stream as
// soon as conversation i's copies are done, under i's new-input prefill tail
// (the PCIe link is otherwise idle there). Coded / raw staging alternate
// between two slots (item i+2 reuses i's slot after i's decode + expand);
// consecutive items must restore into different conversations. Per item the
// device time from its first copy to its logits; total = first copy to the
// last logits.
void restore_batch(Ctx& c, int n, Conv* const* convs, Snapshot* const* snaps, const int32_t* const* hists,
                   const int64_t* Ls, const int32_t* const* news, const int64_t* n_news, float* logits,
                   double* ttft_ms, double* total_ms) {
  const Cfg& g = c.cfg;
  if (n <= 0) fail(KRUL_E_CONFIG, "empty restore batch");
  for (int i = 0; i < n; ++i) {
    check_restore(c, *convs[i], *snaps[i], hists[i], Ls[i], news[i], n_news[i]);
    if (n_news[i] <= 0) fail(KRUL_E_RESTORATION_GAP, "prefill over preloaded history requires new input tokens");
    if (i > 0 && convs[i] == convs[i - 1]) fail(KRUL_E_CONFIG, "consecutive batch items need different conversations");
  }
  if (c.fused) fail(KRUL_E_CONFIG, "the pipelined batch restore runs the two-stream DAG (fused recompute off)");
  KB_CUDA(cudaSetDevice(c.device));
  c.drop_graph();
  const bool kt_was = c.kt.on;
  c.kt.on = false;  // per-launch events would serialise the pipelined DAGs
  // tokens of every item in one pinned block and one device block
  std::vector<size_t> toff(size_t(n) + 1, 0);
  for (int i = 0; i < n; ++i) toff[size_t(i) + 1] = toff[size_t(i)] + size_t(std::max<int64_t>(snaps[i]->p[0], 0) + n_news[i]);
  int32_t* tp = static_cast<int32_t*>(c.tok_pin.ensure((toff[size_t(n)] + 1) * 4));
  int32_t* dt = static_cast<int32_t*>(c.batch_tok.ensure((toff[size_t(n)] + 1) * 4));
  size_t stg_max = 256, cstg_max = 256;
  for (int i = 0; i < n; ++i) {
    const int64_t nh = std::max<int64_t>(snaps[i]->p[0], 0);
    if (nh) std::memcpy(tp + toff[size_t(i)], hists[i], size_t(nh) * 4);
    std::memcpy(tp + toff[size_t(i)] + nh, news[i], size_t(n_news[i]) * 4);
    stg_max = std::max(stg_max, snaps[i]->total);
    if (snaps[i]->coded) cstg_max = std::max(cstg_max, snaps[i]->ctotal);
  }
  // ctx-owned, grow-only: a per-call cudaMalloc / cudaFree (which
  // synchronises the device) would cost more than the overlap gains
  char* stg_slot[2] = {static_cast<char*>(c.staging.ensure(stg_max)), static_cast<char*>(c.staging2.ensure(stg_max))};
  char* cstg_slot[2] = {static_cast<char*>(c.cstaging.ensure(cstg_max)),
                        static_cast<char*>(c.cstaging2.ensure(cstg_max))};
  c.ws_logits.ensure(size_t(g.V) * 4);
  float* lp = logits ? static_cast<float*>(c.logits_pin.ensure(size_t(n) * g.V * 4)) : nullptr;
  auto& G = c.rg;
  G.ev.resize(size_t(5 + 3 * g.N));
  for (size_t i = 0; i < G.ev.size(); ++i) {
    auto& m = G.ev[i];
    if (!m.dep) KB_CUDA(cudaEventCreateWithFlags(&m.dep, cudaEventDisableTiming));
  }
  G.snap_serial = 0;  // the graph key is void after a batch
  c.reset_events();
  const size_t nn = static_cast<size_t>(n);
  std::vector<cudaEvent_t> t0(nn), t1(nn), done(nn);
  for (int i = 0; i < n; ++i) {
    KB_CUDA(cudaEventCreate(&t0[size_t(i)]));
    KB_CUDA(cudaEventCreate(&t1[size_t(i)]));
    KB_CUDA(cudaEventCreateWithFlags(&done[size_t(i)], cudaEventDisableTiming));
  }
  cudaStream_t sl = c.s_load;
  // graph mode: every item's DAG captured once (after an eager pipelined
  // pass sized the workspaces) and replayed on alternating launch streams;
  // the hand-offs between neighbours are external events: staging slot (the
  // decode + expand of item i-2), recompute workspaces (item i-1's recompute
  // end) and prefill workspaces (item i-1's prefill end)
  static const bool graphs_env = [] {
    const char* v = std::getenv("KRUL_BATCH_GRAPHS");
    return !(v && v[0] == '0');
  }();
  const bool use_g = graphs_env && c.use_graphs;
  std::vector<Ctx::BatchGraph*> bg(nn, nullptr);
  bool all_cached = use_g;
  if (use_g) {
    for (int k = 0; k < 2; ++k) {
      if (!c.b_launch[k]) KB_CUDA(cudaStreamCreateWithFlags(&c.b_launch[k], cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&c.b_dec[k], &c.b_comp[k], &c.b_new[k], &c.b_h2d[k]})
        if (!*e) KB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    std::vector<Ctx::BatchGraph*> keep;
    for (int i = 0; i < n; ++i) {
      for (auto* x : c.bgraphs)
        if (x->snap_serial == snaps[i]->serial && x->conv_serial == convs[i]->serial && x->L == Ls[i] &&
            x->n_new == n_news[i] && x->slot == (i & 1) && x->buf_gen == g_buf_gen.load())
          bg[size_t(i)] = x;
      if (!bg[size_t(i)]) all_cached = false;
    }
    // drop cached graphs this batch does not use
    for (auto* x : c.bgraphs) {
      if (std::find(bg.begin(), bg.end(), x) != bg.end())
        keep.push_back(x);
      else
        delete x;
    }
    c.bgraphs = keep;
  }
  if (all_cached) {
    for (int i = 0; i < n; ++i) {
      Ctx::BatchGraph& x = *bg[size_t(i)];
      const int64_t nh = std::max<int64_t>(snaps[i]->p[0], 0);
      int32_t* tq = static_cast<int32_t*>(x.tok.p);
      if (nh) std::memcpy(tq, hists[i], size_t(nh) * 4);
      std::memcpy(tq + nh, news[i], size_t(n_news[i]) * 4);
      KB_CUDA(cudaGraphLaunch(x.exec, c.b_launch[i & 1]));
      convs[i]->len = Ls[i] + n_news[i];
    }
    KB_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < n; ++i) {
      float ms = 0;
      KB_CUDA(cudaEventElapsedTime(&ms, bg[size_t(i)]->t0, bg[size_t(i)]->t1));
      if (ttft_ms) ttft_ms[i] = ms;
      if (logits) std::memcpy(logits + size_t(i) * g.V, bg[size_t(i)]->logits.p, size_t(g.V) * 4);
    }
    float tot = 0;
    KB_CUDA(cudaEventElapsedTime(&tot, bg[0]->t0, bg[size_t(n - 1)]->t1));
    if (total_ms) *total_ms = tot;
    for (int i = 0; i < n; ++i) {
      cudaEventDestroy(t0[size_t(i)]);
      cudaEventDestroy(t1[size_t(i)]);
      cudaEventDestroy(done[size_t(i)]);
    }
    c.tl_pending = false;
    c.kt.on = kt_was;
    return;
  }
  for (int i = 0; i < n; ++i) {
    const int slot = i & 1;
    if (i >= 2) KB_CUDA(cudaStreamWaitEvent(sl, done[size_t(i - 2)], 0));  // the slot's previous item decoded
    const int64_t nh = std::max<int64_t>(snaps[i]->p[0], 0);
    int32_t* d = dt + toff[size_t(i)];
    KB_CUDA(cudaEventRecord(t0[size_t(i)], sl));
    KB_CUDA(cudaMemcpyAsync(d, tp + toff[size_t(i)], size_t(nh + n_news[i]) * 4, cudaMemcpyHostToDevice, sl));
    PipeItem it;
    it.d_tok = d;
    it.d_new = d + nh;
    it.tok_ready = c.event();
    KB_CUDA(cudaEventRecord(it.tok_ready, sl));
    it.stg = stg_slot[slot];
    it.cstg = cstg_slot[slot];
    it.logits_host = lp ? lp + size_t(i) * g.V : nullptr;
    double h2d = 0, eb = 0;
    enqueue_restore(c, *convs[i], *snaps[i], Ls[i], nullptr, nullptr, n_news[i], nullptr, &h2d, &eb, &it);
    KB_CUDA(cudaEventRecord(done[size_t(i)], c.s_exp));
    KB_CUDA(cudaEventRecord(t1[size_t(i)], c.s_new));
    convs[i]->len = Ls[i] + n_news[i];
  }
  // join everything back into s_comp
  KB_CUDA(cudaStreamWaitEvent(c.s_comp, t1[size_t(n - 1)], 0));
  KB_CUDA(cudaStreamWaitEvent(c.s_comp, done[size_t(n - 1)], 0));
  KB_CUDA(cudaStreamWaitEvent(c.s_comp, G.ev[4].dep, 0));
  KB_CUDA(cudaStreamSynchronize(c.s_comp));
  KB_CUDA(cudaDeviceSynchronize());
  for (int i = 0; i < n; ++i) {
    float ms = 0;
    KB_CUDA(cudaEventElapsedTime(&ms, t0[size_t(i)], t1[size_t(i)]));
    if (ttft_ms) ttft_ms[i] = ms;
  }
  float tot = 0;
  KB_CUDA(cudaEventElapsedTime(&tot, t0[0], t1[size_t(n - 1)]));
  if (total_ms) *total_ms = tot;
  if (logits) std::memcpy(logits, lp, size_t(n) * g.V * 4);
  for (int i = 0; i < n; ++i) {
    cudaEventDestroy(t0[size_t(i)]);
    cudaEventDestroy(t1[size_t(i)]);
    cudaEventDestroy(done[size_t(i)]);
  }
  // capture the items' graphs for the next call of this batch (the eager
  // pass above sized every workspace)
  if (use_g) {
    for (int i = 0; i < n; ++i) {
      if (bg[size_t(i)]) continue;
      auto* x = new Ctx::BatchGraph;
      c.bgraphs.push_back(x);
      x->snap_serial = snaps[i]->serial;
      x->conv_serial = convs[i]->serial;
      x->L = Ls[i];
      x->n_new = n_news[i];
      x->slot = i & 1;
      const int64_t nh = std::max<int64_t>(snaps[i]->p[0], 0);
      x->tok.ensure(size_t(nh + n_news[i] + 1) * 4);
      int32_t* dq = static_cast<int32_t*>(x->dtok.ensure(size_t(nh + n_news[i] + 1) * 4));
      x->logits.ensure(size_t(g.V) * 4);
      KB_CUDA(cudaEventCreate(&x->t0));
      KB_CUDA(cudaEventCreate(&x->t1));
      x->ev.resize(size_t(5 + 3 * g.N));
      for (auto& m : x->ev) KB_CUDA(cudaEventCreateWithFlags(&m.dep, cudaEventDisableTiming));
      const int slot = i & 1;
      c.reset_events();
      cudaStream_t sc = c.s_comp;
      KB_CUDA(cudaStreamBeginCapture(sc, cudaStreamCaptureModeRelaxed));
      try {
        cudaEvent_t fork = c.event();
        KB_CUDA(cudaEventRecord(fork, sc));
        KB_CUDA(cudaStreamWaitEvent(sl, fork, 0));
        KB_CUDA(cudaStreamWaitEvent(sl, c.b_dec[slot], cudaEventWaitExternal));
        // the link carries one conversation at a time: copies after the
        // previous item's (two copy streams would only share the link)
        KB_CUDA(cudaStreamWaitEvent(sl, c.b_h2d[slot ^ 1], cudaEventWaitExternal));
        KB_CUDA(record_timing(x->t0, sl));
        KB_CUDA(cudaMemcpyAsync(dq, x->tok.p, size_t(nh + n_news[i]) * 4, cudaMemcpyHostToDevice, sl));
        PipeItem it;
        it.d_tok = dq;
        it.d_new = dq + nh;
        it.tok_ready = c.event();
        KB_CUDA(cudaEventRecord(it.tok_ready, sl));
        it.stg = stg_slot[slot];
        it.cstg = cstg_slot[slot];
        it.logits_host = static_cast<float*>(x->logits.p);
        it.ev = x->ev.data();
        it.wait_comp = c.b_comp[slot ^ 1];
        it.rec_comp = c.b_comp[slot];
        it.wait_new = c.b_new[slot ^ 1];
        it.rec_new = c.b_new[slot];
        double h2d = 0, eb = 0;
        enqueue_restore(c, *convs[i], *snaps[i], Ls[i], nullptr, nullptr, n_news[i], nullptr, &h2d, &eb, &it);
        KB_CUDA(cudaEventRecordWithFlags(c.b_dec[slot], c.s_exp, cudaEventRecordExternal));
        KB_CUDA(cudaEventRecordWithFlags(c.b_h2d[slot], sl, cudaEventRecordExternal));
        KB_CUDA(record_timing(x->t1, c.s_new));
        for (cudaStream_t st : {sl, c.s_exp, c.s_new}) {  // join into the capture origin
          cudaEvent_t j = c.event();
          KB_CUDA(cudaEventRecord(j, st));
          KB_CUDA(cudaStreamWaitEvent(sc, j, 0));
        }
      } catch (...) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(sc, &junk);
        if (junk) cudaGraphDestroy(junk);
        throw;
      }
      cudaGraph_t graph = nullptr;
      KB_CUDA(cudaStreamEndCapture(sc, &graph));
      const cudaError_t ie = cudaGraphInstantiate(&x->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        x->exec = nullptr;
        fail(KRUL_E_CUDA, std::string("batch restore graph instantiation failed: ") + cudaGetErrorString(ie));
      }
    }
    // the key's buffer generation once every new graph's own buffers exist
    // (their allocations bump it too)
    for (auto* x : c.bgraphs) x->buf_gen = g_buf_gen.load();
  }
  c.tl_pending = false;
  c.kt.on = kt_was;
}

}  // namespace kb
