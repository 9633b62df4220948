// fold.cu — K1: the streaming estimator's decode fold (analysis.cpp:124-151).
//
// For every tracked pair (a < b, analysis.cpp:84-93 order) and head h the
// reference adds sum_w double(float(A_a[h][w] - A_b[h][w]))^2 to sums[p][h]
// (the f32 difference of analysis.cpp:146-147, squared and summed in f64).
// One decode step reads every tracked layer's attention row once (N_I x H x
// W f32, HBM) and does P x H x W pair-element work, P = N_I (N_I - 1) / 2.
//
// Work item = (head, column chunk). A persistent CTA (one per SM) streams
// its items' rows HBM -> shared memory with 16-byte cp.async (zero-filled
// past the row end and for padded layers), double-buffered so the next
// item's rows are in flight while this item is folded. Each warp owns a set
// of 8x8 layer-block pairs (an LPT deal computed on the host, so the
// diagonal blocks' 28 pairs are doubled up against the off-diagonal 64);
// a lane holds the 64 pair accumulators in registers and walks two columns
// at a time with packed f32x2 arithmetic (FADD2: the reference's f32
// difference, FFMA2: its square accumulated), 8 column pairs per lane and
// item. At the item's end the lane partials (two column halves added) are
// summed across the warp through a shared-memory transpose, widened to f64
// and written once per pair (f32 partials of <= 2 x 8 x 32 terms per item;
// the chunks then add up in f64). A second kernel adds the column
// chunks to sums[p][h] in fixed chunk order: deterministic, no fp atomics.
#include <algorithm>
#include <vector>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {

__device__ __forceinline__ uint32_t fold_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kFoldWarps = 8;
constexpr int kFoldMaxBP = 64;  // block pairs: 8-layer blocks, <= 80 tracked layers (55)
constexpr int kFoldMaxLayers = 80;

struct FoldDeal {
  uint16_t bp[kFoldMaxBP];      // (I << 8) | J, I <= J, grouped by warp
  uint8_t beg[kFoldWarps + 1];  // warp w owns bp[beg[w], beg[w + 1])
};

// acc[i][j] += (a_i - b_j)^2 for one step of two columns (DIAG: only j > i):
// FADD2 (the reference's f32 difference), FFMA2 (its square accumulated)
template <bool DIAG>
__device__ __forceinline__ void fold_step(const float2 (&a)[8], const float2 (&b)[8], float2 (&acc)[8][8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (DIAG && j <= i) continue;
      const float2 o = DIAG ? a[j] : b[j];
      const float2 d = __fadd2_rn(a[i], make_float2(-o.x, -o.y));
      acc[i][j] = __ffma2_rn(d, d, acc[i][j]);
    }
}
template <bool DIAG>
__device__ __forceinline__ void fold_load(const float* ra, const float* rb, int pitch, int c, float2 (&a)[8],
                                          float2 (&b)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float2*>(ra + i * pitch + c);
  if constexpr (!DIAG) {
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const float2*>(rb + j * pitch + c);
  }
}
// One 8x8 block pair over the chunk, two columns per lane and step; the next
// step's shared-memory loads are issued before this step's arithmetic.
template <bool DIAG>
__device__ __forceinline__ void fold_block(const float* __restrict__ buf, int pitch, int I, int J, int lane,
                                           float2 (&acc)[8][8]) {
  const float* ra = buf + I * 8 * pitch + 2 * lane;
  const float* rb = buf + J * 8 * pitch + 2 * lane;
  float2 a0[8], b0[8], a1[8], b1[8];
  fold_load<DIAG>(ra, rb, pitch, 0, a0, b0);
  int c = 0;
#pragma unroll 1
  for (; c + 128 <= pitch; c += 128) {
    fold_load<DIAG>(ra, rb, pitch, c + 64, a1, b1);
    fold_step<DIAG>(a0, b0, acc);
    if (c + 128 < pitch) fold_load<DIAG>(ra, rb, pitch, c + 128, a0, b0);
    fold_step<DIAG>(a1, b1, acc);
  }
  if (c < pitch) fold_step<DIAG>(a0, b0, acc);  // odd step count
}

// Warp reduction of 64 per-lane values through a padded shared-memory
// transpose: lane l ends with the warp sums of values l and l + 32.
constexpr int kRedPitch = 33;
__device__ __forceinline__ void warp_reduce64(const float (&v)[64], float* red, int lane, float& s0, float& s1) {
#pragma unroll
  for (int k = 0; k < 64; ++k) red[k * kRedPitch + lane] = v[k];
  __syncwarp();
  float t0[32], t1[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    t0[q] = red[lane * kRedPitch + q];
    t1[q] = red[(lane + 32) * kRedPitch + q];
  }
#pragma unroll
  for (int w = 16; w > 0; w >>= 1)  // pairwise tree (error ~ log2 32 roundings, not 32)
#pragma unroll
    for (int q = 0; q < w; ++q) {
      t0[q] += t0[q + w];
      t1[q] += t1[q + w];
    }
  s0 = t0[0];
  s1 = t1[0];
  __syncwarp();
}

__global__ void __launch_bounds__(kFoldWarps * 32, 1)
    k_fold_direct(const float* __restrict__ rows, int64_t layer_stride, int64_t head_stride, int64_t W, int H,
                  const int* __restrict__ layers, int n, int pitch, int chunks, const __grid_constant__ FoldDeal deal,
                  double* __restrict__ part) {
  extern __shared__ __align__(16) float fbuf[];  // [2][n8][pitch], then [warps][64][kRedPitch]
  const int n8 = (n + 7) & ~7;
  const int P = n * (n - 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = H * chunks;
  __shared__ const float* s_row[kFoldMaxLayers];  // tracked layer rows of head 0 (read once)
  for (int li = threadIdx.x; li < n; li += blockDim.x) s_row[li] = rows + int64_t(layers[li]) * layer_stride;
  __syncthreads();
  auto issue = [&](int item, int b) {  // rows of `item` -> buffer b (cp.async, zero-filled tail)
    const int h = item / chunks, ch = item % chunks;
    const int64_t c0 = int64_t(ch) * pitch;
    float* dst = fbuf + size_t(b) * n8 * pitch;
    const int left = int(W - c0);  // columns of this chunk that exist (may exceed pitch)
    for (int li = warp; li < n8; li += kFoldWarps) {  // one warp per layer row, 16 B per lane
      const float* row = (li < n ? s_row[li] + int64_t(h) * head_stride : rows) + c0;
      const uint32_t sdst = fold_smem_u32(dst + li * pitch);
      for (int cv = lane * 4; cv < pitch; cv += 128) {
        const int rem = li < n ? left - cv : 0;
        const int bytes = rem >= 4 ? 16 : rem > 0 ? 4 * rem : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst + 4u * uint32_t(cv)),
                     "l"(bytes ? row + cv : rows), "r"(bytes)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int it = blockIdx.x, b = 0;
  if (it < items) issue(it, 0);
  for (; it < items; it += gridDim.x, b ^= 1) {
    const int nx = it + gridDim.x;
    if (nx < items) {
      issue(nx, b ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* buf = fbuf + size_t(b) * n8 * pitch;
    const int h = it / chunks, ch = it % chunks;
    for (int q = deal.beg[warp]; q < deal.beg[warp + 1]; ++q) {
      const int I = deal.bp[q] >> 8, J = deal.bp[q] & 0xFF;
      float2 acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
      if (I == J)
        fold_block<true>(buf, pitch, I, J, lane, acc);
      else
        fold_block<false>(buf, pitch, I, J, lane, acc);
      // the two column halves, then the warp (f32: each lane partial holds
      // <= 8 squared differences; the f64 accumulation starts per item)
      float v[64];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i * 8 + j] = acc[i][j].x + acc[i][j].y;
      float s2[2];
      warp_reduce64(v, fbuf + size_t(2) * n8 * pitch + warp * 64 * kRedPitch, lane, s2[0], s2[1]);
      // lane l holds the sums of (i, j) = index l and l + 32 of i * 8 + j
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = (lane + 32 * e) >> 3, j = lane & 7;
        const int a = I * 8 + i, bb = J * 8 + j;
        if (a < bb && bb < n) {
          const int p = a * n - a * (a + 1) / 2 + (bb - a - 1);
          part[(int64_t(ch) * P + p) * H + h] = double(s2[e]);
        }
      }
    }
    __syncthreads();  // buffer b is free for the item after next
  }
}

// sums[p][h] += sum over chunks (fixed order) of the item partials. One
// thread per (pair, head); all of its chunk loads are issued before the first
// add (a chained 8-at-a-time loop was latency-bound: 14 us for 2.9 MB).
constexpr int kFoldChunkUnroll = 32;
__global__ void __launch_bounds__(128) k_fold_chunks(const double* __restrict__ part, int chunks, int PH,
                                                     double* __restrict__ sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= PH) return;
  double acc = 0.0;
  for (int c0 = 0; c0 < chunks; c0 += kFoldChunkUnroll) {
    double v[kFoldChunkUnroll];
#pragma unroll
    for (int u = 0; u < kFoldChunkUnroll; ++u)
      v[u] = c0 + u < chunks ? __ldcg(part + int64_t(c0 + u) * PH + i) : 0.0;
#pragma unroll
    for (int u = 0; u < kFoldChunkUnroll; ++u) acc += v[u];
  }
  sums[i] += acc;
}

// Column-chunk width: both buffers of n8 rows fit in ~200 KB of shared
// memory; the item count is rounded to whole waves of the SMs where possible.
constexpr int kFoldRedBytes = kFoldWarps * 64 * kRedPitch * 4;
static int fold_pitch(int n8, int64_t W, int H, int sms) {
  const int cap = std::max(64, ((200 * 1024 - kFoldRedBytes) / (2 * n8 * 4)) / 64 * 64);
  int best = 64;
  double best_t = 1e30;
  for (int pitch = 64; pitch <= std::min(cap, 1024); pitch += 64) {
    const int64_t items = int64_t(H) * ((W + pitch - 1) / pitch);
    const double waves = double((items + sms - 1) / sms);
    const double t = waves * (pitch + 96.0);  // per-item overhead ~ 96 columns of work
    if (t < best_t) {
      best_t = t;
      best = pitch;
    }
  }
  return best;
}

static FoldDeal fold_deal(int n) {
  const int nb = (n + 7) / 8;
  std::vector<std::pair<int, int>> bps;  // (work, bp)
  for (int I = 0; I < nb; ++I)
    for (int J = I; J < nb; ++J) bps.push_back({I == J ? 28 : 64, (I << 8) | J});
  if (int(bps.size()) > kFoldMaxBP) fail(KRUL_E_CONFIG, "too many tracked layers for the estimator fold (max 80)");
  std::stable_sort(bps.begin(), bps.end(), [](auto& x, auto& y) { return x.first > y.first; });
  std::vector<std::vector<int>> per(kFoldWarps);
  std::vector<int> load(kFoldWarps, 0);
  for (auto& x : bps) {  // LPT
    const int w = int(std::min_element(load.begin(), load.end()) - load.begin());
    per[size_t(w)].push_back(x.second);
    load[size_t(w)] += x.first;
  }
  FoldDeal d{};
  int q = 0;
  for (int w = 0; w < kFoldWarps; ++w) {
    d.beg[w] = uint8_t(q);
    for (int bp : per[size_t(w)]) d.bp[q++] = uint16_t(bp);
  }
  d.beg[kFoldWarps] = uint8_t(q);
  return d;
}

int64_t fold_direct_partial_elems(int n, int64_t W, int H, int sms) {
  const int n8 = (n + 7) & ~7;
  const int pitch = fold_pitch(n8, W, H, sms);
  return ((W + pitch - 1) / pitch) * int64_t(n) * (n - 1) / 2 * H;
}

void launch_fold_direct(cudaStream_t s, const float* rows, int64_t layer_stride, int64_t head_stride, int64_t W,
                        int H, const int* d_layers, int n, double* sums, double* part, int64_t part_cap, int sms) {
  if (n < 2 || W <= 0) return;
  const int n8 = (n + 7) & ~7;
  if (((reinterpret_cast<uintptr_t>(rows) | uintptr_t(layer_stride * 4) | uintptr_t(head_stride * 4)) & 15) != 0)
    fail(KRUL_E_CUDA, "decode fold rows must be 16-byte aligned with 16-byte row pitch");
  const int pitch = fold_pitch(n8, W, H, sms);
  const int chunks = int((W + pitch - 1) / pitch);
  const int P = n * (n - 1) / 2;
  if (int64_t(chunks) * P * H > part_cap) fail(KRUL_E_CUDA, "fold partial buffer too small");
  const FoldDeal deal = fold_deal(n);
  const size_t smem = size_t(2) * n8 * pitch * 4 + kFoldRedBytes;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    KB_CUDA(cudaFuncSetAttribute(k_fold_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    smem_set = smem;
  }
  const int items = H * chunks;
  k_fold_direct<<<unsigned(std::min(items, sms)), kFoldWarps * 32, smem, s>>>(
      rows, layer_stride, head_stride, W, H, d_layers, n, pitch, chunks, deal, part);
  KB_LAUNCH();
  k_fold_chunks<<<unsigned((P * H + 127) / 128), 128, 0, s>>>(part, chunks, P * H, sums);
  KB_LAUNCH();
}

}  // namespace kb
