// fold.cu — K1: the streaming estimator's decode fold (analysis.cpp:124-151).
//
// For every tracked pair (a < b, analysis.cpp:84-93 order) and head h the
// reference adds sum_w double(float(A_a[h][w] - A_b[h][w]))^2 to sums[p][h]
// (the f32 difference of analysis.cpp:146-147, squared and summed in f64).
// One decode step reads every tracked layer's attention row once (N_I x H x
// W f32, HBM) and does P x H x W pair-element work, P = N_I (N_I - 1) / 2.
//
// One launch, 16 warps per CTA, one CTA per SM. The H x W column space is
// cut into equal contiguous ranges of 64-column blocks, one per CTA, and
// streamed HBM -> shared memory in 256-column chunks by 16-byte cp.async
// (3-stage ring, zero-filled past the row end and for padded layers). Each
// warp owns one 8-row layer-block unit (4x8 off-diagonal half-blocks and
// the 8x8 diagonal blocks: 16 units for 32 tracked layers) and keeps its 32
// pair accumulators in registers for the whole run of one head, walking two
// columns per lane with packed f32x2 arithmetic (FADD2: the reference's f32
// difference, FFMA2: its square accumulated). When the head's range ends
// the lanes are summed by a shuffle butterfly (lane l ends with pair l),
// widened to f64 and added to the CTA's own resident (head, segment, pair)
// slot: no atomics, no cross-CTA reduction per step; the slots are added to
// sums[p][h] in fixed order when the sums are read (k_fold_collect).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {

__device__ __forceinline__ uint32_t fold_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kFoldWarps = 16;
constexpr int kFoldStages = 3;
constexpr int kFoldMaxUnits = 112;  // 8-layer blocks squared: <= 80 tracked layers (100 units)
constexpr int kFoldMaxLayers = 80;

// Work unit of a warp (nb^2 per head, nb = ceil(n / 8) layer blocks; 16
// warps take units round by round, round r = units [16 r, 16 r + 16)):
//   OFF   rows I*8 + 4h .. +4  x  rows J*8 .. +8  (I < J, h = 0/1: 32 pairs)
//   DIAG  the 28 pairs a < b inside rows I*8 .. +8
// For 32 tracked layers that is 12 OFF + 4 DIAG: one unit per warp, 32 vs
// 28 pairs.
enum { kUnitOff = 0, kUnitDiag = 1 };
struct FoldDeal {
  uint32_t u[kFoldMaxUnits];  // type << 24 | I << 16 | J << 8 | h
  int units;
};

// Debug timeline (krul_debug_fold_timeline): per CTA, %globaltimer at
// entry (0), after setup (1), after the chunk loop (2), when thread 0 has
// chunk k (< 4) in shared memory (3 + k); slot 7 = %smid.
__device__ unsigned long long* g_fold_ts = nullptr;
__device__ __forceinline__ void fold_ts(int slot) {
  if (g_fold_ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fold_ts[blockIdx.x * 8 + slot] = t;
  }
}
void fold_set_timeline(unsigned long long* d) { KB_CUDA(cudaMemcpyToSymbol(g_fold_ts, &d, sizeof d)); }

__device__ __forceinline__ void fold_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(fold_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fold_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(fold_smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// acc += (a - b)^2 over two columns: FADD2 (the reference's f32 difference),
// FFMA2 (its square accumulated)
__device__ __forceinline__ void fold_pair(float2 x, float2 y, float2& acc) {
  const float2 d = __fadd2_rn(x, make_float2(-y.x, -y.y));
  acc = __ffma2_rn(d, d, acc);
}
// One 64-column step of a unit at column c; MASK zeroes the lane's columns
// at or past lim (the row end inside the last block: both rows of a pair
// read zero there, so the padding adds nothing)
template <int TYPE, int PITCH, bool MASK>
__device__ __forceinline__ void fold_step(const float* pa, const float* pb, int c, bool m0, bool m1,
                                          float2 (&acc)[32]) {
  auto ld = [&](const float* p) {
    float2 v = *reinterpret_cast<const float2*>(p);
    if constexpr (MASK) v = make_float2(m0 ? v.x : 0.f, m1 ? v.y : 0.f);
    return v;
  };
  if constexpr (TYPE == kUnitOff) {
    float2 x[4], y[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = ld(pa + i * PITCH + c);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = ld(pb + j * PITCH + c);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) fold_pair(x[i], y[j], acc[i * 8 + j]);
  } else {
    float2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = ld(pa + i * PITCH + c);
    int k = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = i + 1; j < 8; ++j) fold_pair(x[i], x[j], acc[k++]);
  }
}
// valid columns of the unit's rows in this stage; lane owns columns
// 2 lane, 2 lane + 1 of every 64
template <int TYPE, int PITCH>
__device__ __forceinline__ void fold_unit(const float* __restrict__ buf, int valid, int ra, int rb, int lane,
                                          float2 (&acc)[32]) {
  const float* pa = buf + ra * PITCH + 2 * lane;
  const float* pb = buf + rb * PITCH + 2 * lane;
  const int full = valid & ~63;
#pragma unroll 1
  for (int c = 0; c < full; c += 64) fold_step<TYPE, PITCH, false>(pa, pb, c, true, true, acc);
  if (full < valid) {
    const int lim = valid - full;
    fold_step<TYPE, PITCH, true>(pa, pb, full, 2 * lane < lim, 2 * lane + 1 < lim, acc);
  }
}
// The warp sum of each of the lane's 32 values: a butterfly that halves the
// value set each round (lane l ends with the total of value l).
__device__ __forceinline__ float warp_transpose_sum32(float (&v)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const float send = up ? v[k] : v[k + w];
      const float keep = up ? v[k + w] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0];
}

// Column space: head h's W columns are cw = ceil(W / 64) column blocks;
// the H x cw blocks (head-major) are split into equal contiguous ranges,
// one per CTA, so a CTA sees at most a few heads and most of a head's
// columns. A CTA keeps the pair accumulators in registers across its chunks
// of one head and, when the head (or its range) ends, adds one partial per
// pair to its own resident f64 slot: segment k (= CTA - first CTA of head
// h) -> seg_acc[h][k][p]. No two CTAs of a launch share a slot and launches
// are stream-ordered, so the slots need no atomics and no cross-CTA
// reduction; k_fold_collect adds them to sums[p][h] (fixed order) when the
// sums are read.
struct FoldGeom {
  int cw, Q, S, rounds;
};
// cw = column blocks per head in the fold's column space (all ceil(W / 64)
// blocks, or the sampled ones)
__host__ __device__ inline FoldGeom fold_geom(int n, int cw, int H, int grid) {
  FoldGeom g;
  g.cw = cw;
  const int64_t total = int64_t(H) * g.cw;
  g.Q = int((total + grid - 1) / grid);
  g.S = (g.cw + g.Q - 1) / g.Q + 1;
  const int nb = (n + 7) / 8;
  g.rounds = (nb * nb + kFoldWarps - 1) / kFoldWarps;
  return g;
}
// A CTA's chunk sequence (round-major over its range): head, column block,
// length in blocks. Advanced identically by every thread, no divisions.
struct FoldIt {
  int pos, h, b, round;
};

// Rows move HBM -> shared memory by 1D bulk copies (cp.async.bulk, one per
// layer row and chunk, one row per lane) into a kFoldStages ring with a
// full mbarrier per stage; the last warp to finish a stage (a shared
// counter) issues its refill, so no warp waits on another. Columns past W
// are masked in the fold. Padded layers (n..n8) are zero rows written once.
template <int PITCH>
__global__ void __launch_bounds__(kFoldWarps * 32, 1)
    k_fold_direct(const float* __restrict__ rows, int64_t layer_stride, int64_t head_stride, int64_t W, int H,
                  const int* __restrict__ layers, int n, const __grid_constant__ FoldDeal deal,
                  double* __restrict__ seg_acc, int seg_S, int cw, int stride, int phase, double scale,
                  int dbg) {
  extern __shared__ __align__(128) float fbuf[];  // [kFoldStages][n8][PITCH]
  __shared__ __align__(8) uint64_t full[kFoldStages];
  __shared__ unsigned s_done[kFoldStages];  // warps done with the stage's current chunk
  __shared__ const float* s_row[kFoldMaxLayers];
  constexpr int CB = PITCH / 64;
  const int n8 = (n + 7) & ~7;
  const int P = n * (n - 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  fold_ts(0);
  if (g_fold_ts && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_fold_ts[blockIdx.x * 8 + 7] = smid;
  }
  const FoldGeom g = fold_geom(n, cw, H, gridDim.x);
  const int total = H * g.cw;
  const int g0 = min(total, int(blockIdx.x) * g.Q), g1 = min(total, g0 + g.Q);
  if (g1 <= g0) return;
  const int h0 = g0 / g.cw, b0 = g0 - h0 * g.cw;
  const int stage_elems = n8 * PITCH;
  for (int li = threadIdx.x; li < n; li += blockDim.x) s_row[li] = rows + int64_t(layers[li]) * layer_stride;
  for (int i = n * PITCH + threadIdx.x; i < stage_elems; i += blockDim.x)  // padded layers: zero rows
    for (int st = 0; st < kFoldStages; ++st) fbuf[st * stage_elems + i] = 0.f;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kFoldStages; ++st) {
      fold_mbar_init(&full[st], 1);
      s_done[st] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto len_of = [&](const FoldIt& it) { return min(CB, min(g.cw - it.b, g1 - it.pos)); };
  auto advance = [&](FoldIt& it, int len) {
    it.pos += len;
    it.b += len;
    if (it.b == g.cw) {
      ++it.h;
      it.b = 0;
    }
    if (it.pos == g1) {
      ++it.round;
      it.pos = g0;
      it.h = h0;
      it.b = b0;
    }
  };
  // valid columns of the chunk `it` (only the row's last block is partial);
  // block b of the column space is row block phase + b * stride
  auto valid_of = [&](const FoldIt& it, int len) {
    const int64_t last = int64_t(phase) + int64_t(it.b + len - 1) * stride;
    return (len - 1) * 64 + int(min(int64_t(64), W - last * 64));
  };
  // one warp: chunk `it` -> stage st
  auto produce = [&](const FoldIt& it, int st) {
    const int len = len_of(it);
    float* dst = fbuf + st * stage_elems;
    __syncwarp();
    const uint32_t bar = fold_smem_u32(&full[st]);
    // whole 16-byte units: past W this reads the row pitch's padding (host
    // checks head_stride >= ceil4(W)), which the fold masks
    auto copy = [&](int li, int64_t c0, int cols, int soff) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              fold_smem_u32(dst + li * PITCH + soff)),
          "l"(s_row[li] + int64_t(it.h) * head_stride + c0), "r"(uint32_t(((cols + 3) & ~3) * 4)), "r"(bar)
          : "memory");
    };
    if (stride == 1) {  // contiguous: one copy per row
      const int64_t c0 = int64_t(it.b) * 64;
      const int bulk = (dbg & 2) ? 0 : (valid_of(it, len) + 3) & ~3;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(n * bulk * 4))
                     : "memory");
      __syncwarp();
      if (bulk > 0)  // one row per lane
        for (int li = lane; li < n; li += 32) copy(li, c0, bulk, 0);
    } else {  // sampled blocks: one copy per row and block
      const int tail = (valid_of(it, len) - (len - 1) * 64 + 3) & ~3;
      const uint32_t bytes = uint32_t(n) * uint32_t((len - 1) * 64 + tail) * 4u;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      __syncwarp();
      for (int t = lane; t < n * len; t += 32) {
        const int li = t / len, j = t - li * len;
        const int64_t c0 = (int64_t(phase) + int64_t(it.b + j) * stride) * 64;
        copy(li, c0, j == len - 1 ? tail : 64, j * 64);
      }
    }
  };
  const int nchunks = [&] {
    int c = 0;
    for (FoldIt t{g0, h0, b0, 0}; t.round == 0; advance(t, len_of(t))) ++c;
    return c * g.rounds;
  }();
  fold_ts(1);
  FoldIt ip{g0, h0, b0, 0};  // position of chunk k + kFoldStages (every warp tracks it)
  for (int k = 0; k < kFoldStages && k < nchunks; ++k) {
    if (warp == 0) produce(ip, k);
    advance(ip, len_of(ip));
  }
  float2 acc[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) acc[t] = make_float2(0.f, 0.f);
  FoldIt it{g0, h0, b0, 0};
  for (int k = 0; k < nchunks; ++k) {
    const int st = k % kFoldStages;
    const uint32_t ph = uint32_t(k / kFoldStages) & 1u;
    const int len = len_of(it);
    const int h = it.h, round = it.round;
    const int q = round * kFoldWarps + warp;
    const uint32_t u = q < deal.units ? deal.u[q] : 0xFFFFFFFFu;
    const int type = int(u >> 24), I = int((u >> 16) & 0xFF), J = int((u >> 8) & 0xFF), hh = int(u & 0xFF);
    const int ra = I * 8 + (type == kUnitOff ? 4 * hh : 0), rb = type == kUnitOff ? J * 8 : ra;
    const int valid = valid_of(it, len);
    fold_mbar_wait(&full[st], ph);
    if (k < 4) fold_ts(3 + k);
    const float* buf = fbuf + st * stage_elems;
    if (dbg & 1) {
    } else if (dbg & 32) {  // diagnostics: same FP work, broadcast shared loads (one wavefront each)
      fold_unit<kUnitOff, PITCH>(buf, valid, 0, 0, 0, acc);
    } else if (type == kUnitOff)
      fold_unit<kUnitOff, PITCH>(buf, valid, ra, rb, lane, acc);
    else if (type == kUnitDiag)
      fold_unit<kUnitDiag, PITCH>(buf, valid, ra, rb, lane, acc);
    // the last warp done with this stage refills it with chunk k + kFoldStages
    // (no warp waits for the others)
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&s_done[st], 1u) == kFoldWarps - 1;
      if (last) s_done[st] = 0;
      __threadfence_block();
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (k + kFoldStages < nchunks) {
      if (last) produce(ip, st);
      advance(ip, len_of(ip));
    }
    advance(it, len);
    if ((it.h != h || it.round != round) && !(dbg & 4)) {  // the head's segment ends here: flush the pairs
      const int seg = int(blockIdx.x) - (h * g.cw) / g.Q;
      if (type <= kUnitDiag) {
        float vv[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          vv[t] = acc[t].x + acc[t].y;
          acc[t] = make_float2(0.f, 0.f);
        }
        const float sum = warp_transpose_sum32(vv, lane);
        int a, bb;
        if (type == kUnitOff) {
          a = ra + (lane >> 3);
          bb = rb + (lane & 7);
        } else {  // lane -> the lane-th pair (i < j) of the 8-row block, row-major
          int i = 0, r = lane;
          while (i < 7 && r >= 7 - i) {
            r -= 7 - i;
            ++i;
          }
          a = ra + i;
          bb = i < 7 ? ra + i + 1 + r : -1;
        }
        if (a < bb && bb < n) {
          const int pp = a * n - a * (a + 1) / 2 + (bb - a - 1);
          seg_acc[(int64_t(h) * seg_S + seg) * P + pp] += double(sum) * scale;
        }
      }
    }
  }
  fold_ts(2);
}

// sums[p][h] += sum over k of seg[h][k][p] (fixed k order), seg := 0
__global__ void k_fold_collect(double* __restrict__ seg, int S, int P, int H, double* __restrict__ sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * H) return;
  const int h = i / P, p = i - h * P;
  double* ph = seg + int64_t(h) * S * P + p;
  double acc = 0.0;
  for (int k = 0; k < S; ++k) {
    acc += ph[int64_t(k) * P];
    ph[int64_t(k) * P] = 0.0;
  }
  sums[int64_t(p) * H + h] += acc;
}

static int fold_env(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : 0;
}
// Chunk width: 512 columns (2 KB per row and bulk copy; 256 measured 1.3x
// slower: half the bytes in flight per SM), halved until kFoldStages stages
// of n8 rows fit in ~200 KB of shared memory (KRUL_FOLD_PITCH=256/128 caps).
static int fold_pitch(int n8) {
  static const int env = fold_env("KRUL_FOLD_PITCH");
  int pitch = env == 256 || env == 128 ? env : 512;
  while (pitch > 128 && size_t(kFoldStages) * n8 * pitch * 4 > 200 * 1024) pitch /= 2;
  return pitch;
}

static FoldDeal fold_deal(int n) {
  const int nb = (n + 7) / 8;
  FoldDeal d{};
  auto unit = [](int type, int I, int J, int h) {
    return (uint32_t(type) << 24) | (uint32_t(I) << 16) | (uint32_t(J) << 8) | uint32_t(h);
  };
  if (nb * nb > kFoldMaxUnits) fail(KRUL_E_CONFIG, "too many tracked layers for the estimator fold (max 80)");
  for (int I = 0; I < nb; ++I)  // OFF units first (32 pairs), DIAG (28) last: rounds end with the light ones
    for (int J = I + 1; J < nb; ++J)
      for (int h = 0; h < 2; ++h) d.u[d.units++] = unit(kUnitOff, I, J, h);
  for (int I = 0; I < nb; ++I) d.u[d.units++] = unit(kUnitDiag, I, I, 0);
  return d;
}

static int fold_grid(int cw, int H, int sms) {
  return int(std::max<int64_t>(1, std::min<int64_t>(sms, int64_t(H) * cw)));
}

int fold_seg_slots(int H, int sms) { return sms / std::max(H, 1) + 2; }

void launch_fold_collect(cudaStream_t s, double* seg, int S, int n, int H, double* sums) {
  const int P = n * (n - 1) / 2;
  if (P <= 0) return;
  k_fold_collect<<<unsigned((P * H + 255) / 256), 256, 0, s>>>(seg, S, P, H, sums);
  KB_LAUNCH();
}

void launch_fold_direct(cudaStream_t s, const float* rows, int64_t layer_stride, int64_t head_stride, int64_t W,
                        int H, const int* d_layers, int n, double* seg, int seg_S, int sms, int stride, int phase) {
  if (n < 2 || W <= 0) return;
  if (stride < 1 || phase < 0 || phase >= stride) fail(KRUL_E_CONFIG, "fold sampling: need stride >= 1, 0 <= phase < stride");
  // sampled token subset (opt-in): row blocks phase, phase + stride, ...;
  // each sampled sum is scaled by W / sampled columns (an estimate of the
  // full-width sum; stride 1 folds every column with scale 1 exactly)
  const int64_t cw_all = (W + 63) / 64;
  if (phase >= cw_all) return;
  const int cw = int((cw_all - 1 - phase) / stride + 1);
  const int64_t last = phase + int64_t(cw - 1) * stride;
  const int64_t sampled_cols = int64_t(cw - 1) * 64 + std::min<int64_t>(64, W - last * 64);
  const double scale = stride == 1 ? 1.0 : double(W) / double(sampled_cols);
  if (n > kFoldMaxLayers) fail(KRUL_E_CONFIG, "too many tracked layers for the estimator fold (max 80)");
  const int n8 = (n + 7) & ~7;
  if (((reinterpret_cast<uintptr_t>(rows) | uintptr_t(layer_stride * 4) | uintptr_t(head_stride * 4)) & 15) != 0)
    fail(KRUL_E_CUDA, "decode fold rows must be 16-byte aligned with 16-byte row pitch");
  if (head_stride < (W + 3) / 4 * 4) fail(KRUL_E_CUDA, "decode fold rows: head stride below the 16-byte-padded width");
  const int pitch = fold_pitch(n8);
  const int grid = fold_grid(cw, H, sms);
  if (fold_geom(n, cw, H, grid).S > seg_S) fail(KRUL_E_CUDA, "fold segment slots too few");
  const FoldDeal deal = fold_deal(n);
  const size_t smem = size_t(kFoldStages) * n8 * pitch * 4;
  // diagnostics: 1 = skip the fold arithmetic, 2 = skip the row loads,
  // 4 = skip the flushes, 32 = broadcast shared loads (same FP work)
  static const int dbg = [] {
    const char* e = std::getenv("KRUL_FOLD_DBG");
    return e ? std::atoi(e) : 0;
  }();
  auto go = [&](auto pitch_c) {  // one static per pitch (the kernels share one signature)
    constexpr int PITCH = decltype(pitch_c)::value;
    static size_t smem_set = 0;
    if (smem > smem_set) {
      KB_CUDA(cudaFuncSetAttribute(k_fold_direct<PITCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      smem_set = smem;
    }
    k_fold_direct<PITCH><<<unsigned(grid), kFoldWarps * 32, smem, s>>>(rows, layer_stride, head_stride, W, H,
                                                                      d_layers, n, deal, seg, seg_S, cw, stride, phase,
                                                                      scale, dbg);
  };
  if (pitch == 512)
    go(std::integral_constant<int, 512>{});
  else if (pitch == 256)
    go(std::integral_constant<int, 256>{});
  else
    go(std::integral_constant<int, 128>{});
  KB_LAUNCH();
}

}  // namespace kb
