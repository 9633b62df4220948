// attn_tc.cu — causal prefill attention on tcgen05 / TMEM over the paged KV
// cache (K6 recompute and K7 new-input prefill; engine.cpp:174-188).
//
// One CTA = one head x one 128-row query tile x one key split. Warp roles:
//   warps 0-3 : softmax + epilogue, thread r owns query row r (= TMEM lane r)
//   warp 4    : TMA producer (Q once; per 128-key block two K pages and two
//               V^T pages of the paged cache, 128B-swizzled)
//   warp 5    : MMA issuer: S(i) = Q K_i^T into a double-buffered TMEM S,
//               O += P_{i-1} V_{i-1} into TMEM O once softmax published P.
// P is written by the softmax warps straight into shared memory in the
// UMMA K-major SW128 layout. Online softmax runs in the log2 domain; the
// classifier region mass (analysis.cpp:46-54) is accumulated alongside the
// row sum and rescaled with it. Split-KV partials are merged by
// k_attn_combine.
#include <cuda.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {
namespace tca {

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D_%=;\n\t"
      "bra W_%=;\n"
      "D_%=:\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(su32(b))
      : "memory");
}
__device__ __forceinline__ uint64_t desc(const void* p) {  // K-major, SW128, SBO 1024
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(b))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define TCA_REGS32(r)                                                                          \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
      "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
      "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define TCA_IN32(r)                                                                           \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),     \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),       \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),     \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),     \
      "r"(r[29]), "r"(r[30]), "r"(r[31])

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TCA_REGS32(r)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TCA_IN32(r)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

}  // namespace tca

struct AttnTc {
  int H, Hkv, grp;
  int64_t rows, pos0, kv_total;  // keys [0, kv_total) exist; causal limit per row
  int n_qtiles, n_splits, split_blocks;
  float scale_log2;
  const int* pt;
  int max_pages;
  int k_rows_pp;   // K-view rows per page
  int v_rows_pp;   // V-view rows per page
  bf16* out;       // [rows][H*HD] (n_splits == 1)
  float* part;     // [split][rows][H][HD + 3] (o..., m, l, mass)
  double* mass;    // [H][rows] region mass, may be null
  int64_t il, rs;
  volatile int* dbg;  // KRUL_ATTN_DEBUG: per-CTA progress in host-mapped memory
};
#define DBG(slot, val)                                                                  \
  do {                                                                                  \
    if (p.dbg) {                                                                        \
      const int cta_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;   \
      p.dbg[cta_ * 8 + (slot)] = (val);                                                 \
      __threadfence_system();                                                           \
    }                                                                                   \
  } while (0)

template <int HD>
__global__ void __launch_bounds__(192, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnTc p) {
  constexpr int KB = 128;                 // keys per block
  constexpr int NSUB = HD / 64;           // 64-wide hd sub-tiles
  constexpr uint32_t Q_BYTES = 128 * HD * 2;
  constexpr uint32_t K_BYTES = KB * HD * 2;
  constexpr uint32_t V_BYTES = HD * KB * 2;
  constexpr uint32_t P_BYTES = 128 * KB * 2;
  constexpr int STAGES = 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;
  unsigned char* sK = sQ + Q_BYTES;
  unsigned char* sV = sK + STAGES * K_BYTES;
  unsigned char* sP = sV + STAGES * V_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 3;
  uint64_t* s_full = bars + 5;
  uint64_t* p_ready = bars + 7;
  uint64_t* o_done = bars + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heavy (late) query tiles first: causal work grows with the tile index
  const int qt = p.n_qtiles - 1 - int(blockIdx.x);
  const int h = blockIdx.y, split = blockIdx.z;
  const int g = h / p.grp;
  const int64_t q0 = int64_t(qt) * 128;
  const int64_t q_end = q0 + 128 < p.rows ? q0 + 128 : p.rows;
  const int64_t last_pos = p.pos0 + q_end - 1;
  const int64_t kv_hi_all = last_pos + 1 < p.kv_total ? last_pos + 1 : p.kv_total;
  const int nblk_all = int((kv_hi_all + KB - 1) / KB);
  const int b0 = split * p.split_blocks;
  const int b1 = min(nblk_all, b0 + p.split_blocks);
  const int nb = b1 - b0;  // may be <= 0 for trailing splits

  if (threadIdx.x == 0) DBG(7, 1);
  if (threadIdx.x == 0) {
    tca::bar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      tca::bar_init(&kv_full[s], 1);
      tca::bar_init(&kv_empty[s], 1);
      tca::bar_init(&s_full[s], 1);
    }
    tca::bar_init(p_ready, 128);
    tca::bar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        tca::su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tca::fence_before();
  __syncthreads();
  tca::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 256;
  if (threadIdx.x == 0) DBG(7, 2);

  if (warp == 4) {
    if (lane == 0 && nb > 0) {  // producer
      tca::bar_expect(q_full, Q_BYTES);
      for (int j = 0; j < NSUB; ++j)
        tca::tma2d(sQ + j * (128 * 128), &tmQ, q_full, h * HD + 64 * j, int(q0));
      for (int i = 0; i < nb; ++i) {
        const int s = i % STAGES;
        DBG(0, 1000 + i);
        tca::bar_wait(&kv_empty[s], ((i / STAGES) & 1) ^ 1);
        DBG(0, 2000 + i);
        tca::bar_expect(&kv_full[s], K_BYTES + V_BYTES);
        const int kb = b0 + i;
        const int pa = p.pt[min(2 * kb, p.max_pages - 1)];
        const int pb = p.pt[min(2 * kb + 1, p.max_pages - 1)];
        unsigned char* k_dst = sK + s * K_BYTES;
        for (int j = 0; j < NSUB; ++j) {
          tca::tma2d(k_dst + j * (KB * 128), &tmK, &kv_full[s], 64 * j, pa * p.k_rows_pp + g * 64);
          tca::tma2d(k_dst + j * (KB * 128) + 64 * 128, &tmK, &kv_full[s], 64 * j,
                     pb * p.k_rows_pp + g * 64);
        }
        unsigned char* v_dst = sV + s * V_BYTES;
        const int voff = p.Hkv * HD + g * HD;
        tca::tma2d(v_dst, &tmV, &kv_full[s], 0, pa * p.v_rows_pp + voff);
        tca::tma2d(v_dst + HD * 128, &tmV, &kv_full[s], 0, pb * p.v_rows_pp + voff);
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && nb > 0) {  // MMA issuer
      constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KB >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      constexpr uint32_t idO = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(HD >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      DBG(1, 1);
      tca::bar_wait(q_full, 0);
      DBG(1, 2);
      for (int i = 0; i <= nb; ++i) {
        if (i < nb) {
          const int s = i % STAGES;
          DBG(1, 1000 + i);
          tca::bar_wait(&kv_full[s], (i / STAGES) & 1);
          DBG(1, 2000 + i);
          tca::fence_after();
          const uint32_t dS = tS + uint32_t((i & 1) * 128);
#pragma unroll
          for (int j = 0; j < NSUB; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tca::mma(dS, tca::desc(sQ + j * (128 * 128) + k * 32),
                       tca::desc(sK + s * K_BYTES + j * (KB * 128) + k * 32), idS, (j | k) != 0);
          tca::commit(&s_full[i & 1]);
        }
        if (i > 0) {
          const int ip = i - 1, sp = ip % STAGES;
          DBG(2, 1000 + ip);
          tca::bar_wait(p_ready, ip & 1);
          DBG(2, 2000 + ip);
          tca::fence_after();
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tca::mma(tO, tca::desc(sP + j * (128 * 128) + k * 32),
                       tca::desc(sV + sp * V_BYTES + j * (HD * 128) + k * 32), idO,
                       (ip | j | k) != 0);
          tca::commit(o_done);
          tca::commit(&kv_empty[sp]);
        }
      }
    }
  } else {  // softmax warps 0..3: row r = TMEM lane r
    const int r = warp * 32 + lane;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const int64_t qpos = p.pos0 + q0 + r;
    float m = -INFINITY, l = 0.f, mn = 0.f;
    for (int i = 0; i < nb; ++i) {
      const int64_t k0 = int64_t(b0 + i) * KB;
      if (threadIdx.x == 0) DBG(3, 1000 + i);
      tca::bar_wait(&s_full[i & 1], (i >> 1) & 1);
      if (threadIdx.x == 0) DBG(3, 2000 + i);
      tca::fence_after();
      const uint32_t tsrc = tS + uint32_t((i & 1) * 128) + lane_off;
      uint32_t v[32];
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tca::ld32(tsrc + uint32_t(c * 32), v);
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int64_t kp = k0 + c * 32 + t;
          const float sv = __uint_as_float(v[t]) * p.scale_log2;
          if (kp <= qpos && kp < p.kv_total) mx = fmaxf(mx, sv);
        }
      }
      const float m_new = fmaxf(m, mx);
      const float alpha = (m == -INFINITY) ? (m_new == -INFINITY ? 1.f : 0.f) : exp2f(m - m_new);
      // the previous PV must finish before O is rescaled and P overwritten
      if (threadIdx.x == 0) DBG(3, 3000 + i);
      if (i > 0) {
        tca::bar_wait(o_done, (i - 1) & 1);
        tca::fence_after();
      }
      if (threadIdx.x == 0) DBG(3, 4000 + i);
      float sum = 0.f, msum = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        tca::ld32(tsrc + uint32_t(c * 32), v);
        uint32_t packed[16];
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          float pr[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int64_t kp = k0 + c * 32 + t + u;
            const bool ok = kp <= qpos && kp < p.kv_total && m_new != -INFINITY;
            const float e = ok ? exp2f(__uint_as_float(v[t + u]) * p.scale_log2 - m_new) : 0.f;
            pr[u] = e;
            sum += e;
            if (kp < p.il || kp >= p.rs) msum += e;
          }
          __nv_bfloat162 b2 = __floats2bfloat162_rn(pr[0], pr[1]);
          packed[t / 2] = *reinterpret_cast<uint32_t*>(&b2);
        }
        // columns [32c, 32c + 32) = four 16-byte chunks of sub-tile c / 2
        unsigned char* rowp = sP + (c >> 1) * (128 * 128) + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = (c & 1) * 4 + q;
          uint4 val = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
          *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) << 4)) = val;
        }
      }
      if (i > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          tca::ld32(tO + lane_off + uint32_t(c * 32), v);
#pragma unroll
          for (int t = 0; t < 32; ++t) v[t] = __float_as_uint(__uint_as_float(v[t]) * alpha);
          tca::st32(tO + lane_off + uint32_t(c * 32), v);
        }
      }
      l = l * alpha + sum;
      mn = mn * alpha + msum;
      m = m_new;
      tca::fence_before();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tca::bar_arrive(p_ready);
    }
    if (threadIdx.x == 0) DBG(3, 5000);
    if (nb > 0) {
      tca::bar_wait(o_done, (nb - 1) & 1);
      tca::fence_after();
    }
    if (threadIdx.x == 0) DBG(3, 6000);
    // tcgen05.ld is warp-collective: every lane loads, only valid rows store
    const int64_t row = q0 + r;
    const bool valid = row < p.rows;
    uint32_t v[32];
    if (p.n_splits == 1) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16* dst = p.out + (row * p.H + h) * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        tca::ld32(tO + lane_off + uint32_t(c * 32), v);
        if (!valid) continue;
#pragma unroll
        for (int t = 0; t < 32; t += 8) {
          uint4 o;
          __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(v[t]) * inv, __uint_as_float(v[t + 1]) * inv);
          __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(v[t + 2]) * inv, __uint_as_float(v[t + 3]) * inv);
          __nv_bfloat162 cc = __floats2bfloat162_rn(__uint_as_float(v[t + 4]) * inv, __uint_as_float(v[t + 5]) * inv);
          __nv_bfloat162 d = __floats2bfloat162_rn(__uint_as_float(v[t + 6]) * inv, __uint_as_float(v[t + 7]) * inv);
          o.x = *reinterpret_cast<uint32_t*>(&a);
          o.y = *reinterpret_cast<uint32_t*>(&b);
          o.z = *reinterpret_cast<uint32_t*>(&cc);
          o.w = *reinterpret_cast<uint32_t*>(&d);
          *reinterpret_cast<uint4*>(dst + c * 32 + t) = o;
        }
      }
      if (valid && p.mass) p.mass[int64_t(h) * p.rows + row] = l > 0.f ? double(mn) / double(l) : 0.0;
    } else {
      float* dst = p.part + ((int64_t(split) * p.rows + row) * p.H + h) * (HD + 3);
      if (nb > 0) {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          tca::ld32(tO + lane_off + uint32_t(c * 32), v);
          if (!valid) continue;
#pragma unroll
          for (int t = 0; t < 32; ++t) dst[c * 32 + t] = __uint_as_float(v[t]);
        }
      } else if (valid) {
        for (int t = 0; t < HD; ++t) dst[t] = 0.f;
      }
      if (valid) {
        dst[HD] = m;
        dst[HD + 1] = l;
        dst[HD + 2] = mn;
      }
    }
  }
  if (lane == 0) DBG(4 + (warp >= 4 ? warp - 3 : 0), 7000);
  __syncwarp();
  tca::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DBG(7, 9999);
  if (warp == 5) {
    tca::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Split-KV merge: weights 2^(m_s - M) (log2 domain).
template <int HD>
__global__ void k_attn_combine(const float* part, int n_splits, int64_t rows, int H, bf16* out,
                               double* mass) {
  const int64_t row = blockIdx.x;
  const int h = blockIdx.y;
  const int t = threadIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s)
    M = fmaxf(M, part[((int64_t(s) * rows + row) * H + h) * (HD + 3) + HD]);
  float L = 0.f, MN = 0.f, acc = 0.f;
  for (int s = 0; s < n_splits; ++s) {
    const float* q = part + ((int64_t(s) * rows + row) * H + h) * (HD + 3);
    const float w = (q[HD] == -INFINITY) ? 0.f : exp2f(q[HD] - M);
    L += w * q[HD + 1];
    MN += w * q[HD + 2];
    if (t < HD) acc += w * q[t];
  }
  if (t < HD) out[(row * H + h) * HD + t] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
  if (t == 0 && mass) mass[int64_t(h) * rows + row] = L > 0.f ? double(MN) / double(L) : 0.0;
}

// ---------------------------------------------------------------- host
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    KB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) fail(KRUL_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}
CUtensorMap map2d(const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                  uint32_t box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRUL_E_CUDA, "attention tensor map encode failed");
  return m;
}
}  // namespace

bool attention_tc_supported(const Ctx& c, const AttnArgs& a) {
  return c.cfg.dtype == KRUL_BF16 && !a.probs && (c.cfg.hd == 128 || c.cfg.hd == 64) &&
         a.rows >= 1;
}

// Returns the number of splits used (partials in `scratch`).
void launch_attention_tc(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                         const AttnArgs& a, DevBuf& scratch) {
  double* mass_f32 = a.mass;
  const Cfg& g = c.cfg;
  const int HD = g.hd;
  const int64_t kv_total = a.pos0 + a.rows;
  const int n_qtiles = int((a.rows + 127) / 128);
  const int nblk = int((kv_total + 127) / 128);
  int splits = 1;
  const int base = n_qtiles * g.H;
  if (base < 2 * c.sm_count) splits = std::max(1, std::min(nblk / 2, (2 * c.sm_count + base - 1) / base));
  const int split_blocks = (nblk + splits - 1) / splits;
  splits = (nblk + split_blocks - 1) / split_blocks;

  AttnTc p{};
  p.H = g.H;
  p.Hkv = g.Hkv;
  p.grp = g.H / g.Hkv;
  p.rows = a.rows;
  p.pos0 = a.pos0;
  p.kv_total = kv_total;
  p.n_qtiles = n_qtiles;
  p.n_splits = splits;
  p.split_blocks = split_blocks;
  p.scale_log2 = (1.0f / sqrtf(float(HD))) * 1.4426950408889634f;
  p.pt = conv.d_pt + int64_t(layer) * conv.max_pages;
  p.max_pages = conv.max_pages;
  const int64_t pe = int64_t(c.page_elems());
  p.k_rows_pp = int(pe / HD);
  p.v_rows_pp = int(pe / 64);
  p.out = static_cast<bf16*>(a.out);
  p.mass = mass_f32;
  p.il = a.il;
  p.rs = a.mass ? a.rs : INT64_MAX;
  if (!a.mass) p.il = 0;
  if (splits > 1) {
    p.part = static_cast<float*>(
        scratch.ensure(size_t(splits) * a.rows * g.H * (HD + 3) * sizeof(float)));
  }
  const uint64_t pool_elems = uint64_t(c.pool_pages) * pe;
  const CUtensorMap tq = map2d(a.q, uint64_t(a.rows), uint64_t(g.H) * HD, uint64_t(g.H) * HD, 128);
  const CUtensorMap tk = map2d(c.pool.p, pool_elems / HD, HD, HD, 64);
  const CUtensorMap tv = map2d(c.pool.p, pool_elems / 64, 64, 64, uint32_t(HD));
  // >= 116 KB so exactly one CTA is resident per SM: the CTA owns all 512
  // TMEM columns (S double buffer + O)
  const size_t smem = std::max<size_t>(
      1024 + size_t(128) * HD * 2 + 2 * size_t(128) * HD * 2 * 2 + 128 * 128 * 2 + 256, 116 * 1024 + 512);
  dim3 grid(unsigned(n_qtiles), unsigned(g.H), unsigned(splits));
  static const bool dbg_on = std::getenv("KRUL_ATTN_DEBUG") != nullptr;
  int* dbg_host = nullptr;
  const int n_cta = int(grid.x * grid.y * grid.z);
  if (dbg_on) {
    KB_CUDA(cudaHostAlloc(&dbg_host, size_t(n_cta) * 8 * 4, cudaHostAllocMapped));
    std::memset(dbg_host, 0, size_t(n_cta) * 8 * 4);
    int* dev = nullptr;
    KB_CUDA(cudaHostGetDevicePointer(&dev, dbg_host, 0));
    p.dbg = dev;
    std::fprintf(stderr, "[attn dbg] grid %u x %u x %u rows=%lld pos0=%lld splits=%d sb=%d smem=%zu\n",
                 grid.x, grid.y, grid.z, (long long)a.rows, (long long)a.pos0, splits, split_blocks, smem);
  }
  if (HD == 128) {
    static bool attr = false;
    if (!attr) {
      KB_CUDA(cudaFuncSetAttribute(k_attn_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = true;
    }
    k_attn_tc<128><<<grid, 192, smem, s>>>(tq, tk, tv, p);
  } else {
    static bool attr = false;
    if (!attr) {
      KB_CUDA(cudaFuncSetAttribute(k_attn_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = true;
    }
    k_attn_tc<64><<<grid, 192, smem, s>>>(tq, tk, tv, p);
  }
  KB_LAUNCH();
  if (dbg_on) {
    for (int t = 0; t < 300; ++t) {
      if (cudaStreamQuery(s) == cudaSuccess) break;
      usleep(10000);
    }
    if (cudaStreamQuery(s) != cudaSuccess) {
      std::fprintf(stderr, "[attn dbg] TIMEOUT; per-CTA progress (prod, mma, mma_p, soft, w0..3?, w4, w5, cta):\n");
      for (int c = 0; c < n_cta && c < 64; ++c) {
        std::fprintf(stderr, "cta %d:", c);
        for (int k = 0; k < 8; ++k) std::fprintf(stderr, " %d", dbg_host[c * 8 + k]);
        std::fprintf(stderr, "\n");
      }
      std::fflush(stderr);
      std::abort();
    }
    cudaFreeHost(dbg_host);
  }
  if (splits > 1) {
    dim3 g2(unsigned(a.rows), unsigned(g.H));
    if (HD == 128)
      k_attn_combine<128><<<g2, 128, 0, s>>>(p.part, splits, a.rows, g.H, p.out, mass_f32);
    else
      k_attn_combine<64><<<g2, 64, 0, s>>>(p.part, splits, a.rows, g.H, p.out, mass_f32);
    KB_LAUNCH();
  }
}

}  // namespace kb
