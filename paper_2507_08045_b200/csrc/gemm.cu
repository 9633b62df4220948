// gemm.cu — C[M,N] = A[M,K] * B[N,K]^T with fused epilogues.
//
//  * k_gemm_tc: bf16 tcgen05.mma (kind::f16, M=128, N=BN, fp32 accumulator
//    in TMEM), operands staged by TMA (128B swizzle) through an STAGES-deep
//    mbarrier ring; warp 0 = TMA producer, warp 1 = single-thread MMA
//    issuer + TMEM owner, warps 2-5 = epilogue (tcgen05.ld -> registers ->
//    fused epilogue -> global). This is the recompute-stream GEMM (K6/K7).
//  * k_gemm_simt: fp32 CUDA-core tiles for the f32 parity mode (and for
//    shapes TMA cannot describe, e.g. rows not 16-byte aligned).
#include <cuda.h>
#include <unordered_map>
#include <string>
#include <mutex>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {

int g_gemm_force = 0;   // debug: 0 auto, 1 1-SM BN256, 2 1-SM BN128, 3 pair, 4 pair BK128

// Debug timeline of the 1-SM GEMM (krul_debug_gemm_timeline): when set,
// %globaltimer stamps of CTA 0's phases plus every CTA's entry / exit.
__device__ unsigned long long* g_gemm_ts = nullptr;
__device__ __forceinline__ void gemm_ts(int slot) {
  if (g_gemm_ts) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_ts[slot] = t;
  }
}
int g_gemm_splits = 0;  // debug: force the split-K count (0 = planner)
__device__ unsigned long long* g_gemm_span = nullptr;  // [2][slots]: entry min, exit max
__device__ __forceinline__ void gemm_span_stamp(int slot, bool exit_stamp) {
  if (slot >= 0 && g_gemm_span) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (exit_stamp)
      atomicMax(g_gemm_span + 4096 + slot, t);
    else
      atomicMin(g_gemm_span + slot, t);
  }
}
void gemm_set_span(unsigned long long* d) { KB_CUDA(cudaMemcpyToSymbol(g_gemm_span, &d, sizeof d)); }

// ---------------------------------------------------------------- epilogue
template <class T>
__device__ __forceinline__ void epi_apply(const Epi& e, int64_t r, int64_t c0, const float* v,
                                          int n) {
  switch (e.kind) {
    case Epi::F32: {
      float* o = static_cast<float*>(e.out) + r * e.ldo + c0;
      for (int i = 0; i < n; ++i) o[i] = v[i];
      break;
    }
    case Epi::CDT: {
      T* o = static_cast<T*>(e.out) + r * e.ldo + c0;
      for (int i = 0; i < n; ++i) o[i] = fromf<T>(v[i]);
      break;
    }
    case Epi::RESID: {  // engine.cpp:190 / :192: resid + (acc [+ bias])
      float* o = static_cast<float*>(e.out) + r * e.ldo + c0;
      const float* rs = e.resid + r * e.ldr + c0;
      T* o2 = e.out2 ? static_cast<T*>(e.out2) + r * e.ldo2 + c0 : nullptr;
      for (int i = 0; i < n; ++i) {
        const float y = e.bias ? v[i] + e.bias[c0 + i] : v[i];
        const float h = rs[i] + y;
        o[i] = h;
        if (o2) o2[i] = fromf<T>(h);
      }
      break;
    }
    case Epi::TANH: {  // engine.cpp:191
      T* o = static_cast<T*>(e.out) + r * e.ldo + c0;
      for (int i = 0; i < n; ++i) o[i] = fromf<T>(tanhf(v[i] + e.bias[c0 + i]));
      break;
    }
    case Epi::SWIGLU: {  // gate/up interleaved column pairs
      T* o = static_cast<T*>(e.out) + r * e.ldo + c0 / 2;
      for (int i = 0; i + 1 < n; i += 2) {
        const float g = v[i], u = v[i + 1];
        o[i / 2] = fromf<T>(g / (1.0f + expf(-g)) * u);
      }
      break;
    }
  }
}

// ---------------------------------------------------------------- SIMT
template <class T>
__global__ void __launch_bounds__(256) k_gemm_simt(int64_t M, int64_t N, int64_t K, const T* A,
                                                   int64_t lda, const T* B, int64_t ldb, Epi e) {
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = int64_t(blockIdx.y) * 64, n0 = int64_t(blockIdx.x) * 64;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 1024; i += 256) {
      const int mm = i >> 4, kk = i & 15;
      const int64_t gm = m0 + mm, gk = k0 + kk, gn = n0 + mm;
      As[kk][mm] = (gm < M && gk < K) ? tof(A[gm * lda + gk]) : 0.f;
      Bs[kk][mm] = (gn < N && gk < K) ? tof(B[gn * ldb + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
  const int64_t c0 = n0 + tx * 4;
  if (c0 >= N) return;
  const int nv = int(N - c0 < 4 ? N - c0 : 4);
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty * 4 + i;
    if (r < M) epi_apply<T>(e, r, c0, acc[i], nv);
  }
}

// ---------------------------------------------------------------- tcgen05
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tc

// Element-wise epilogue on one accumulator value (row, col) — used by the
// coalesced (smem-transposed) tcgen05 epilogue and by the split-K reduce.
template <class T>
__device__ __forceinline__ void epi_elem(const Epi& e, int64_t r, int64_t c, float v) {
  switch (e.kind) {
    case Epi::F32:
      static_cast<float*>(e.out)[r * e.ldo + c] = v;
      break;
    case Epi::CDT:
      static_cast<T*>(e.out)[r * e.ldo + c] = fromf<T>(v);
      break;
    case Epi::RESID: {  // engine.cpp:190 / :192
      const float y = e.bias ? v + e.bias[c] : v;
      const float h = e.resid[r * e.ldr + c] + y;
      static_cast<float*>(e.out)[r * e.ldo + c] = h;
      if (e.out2) static_cast<T*>(e.out2)[r * e.ldo2 + c] = fromf<T>(h);
      break;
    }
    case Epi::TANH:  // engine.cpp:191
      static_cast<T*>(e.out)[r * e.ldo + c] = fromf<T>(tanhf(v + e.bias[c]));
      break;
  }
}
// silu(g) * u for the bf16 epilogues: MUFU exp2 + fast reciprocal (relative
// error ~1e-6, far below the bf16 output rounding). The accurate expf + IEEE
// division made the SwiGLU epilogue of a 128 x 256 tile ~8 us (measured with
// krul_debug_gemm_timeline): compute-bound on the 4 epilogue warps.
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

// Where the epilogue's accumulator values come from. Default: this CTA's TMEM.
// Cluster split-K (cs > 1): the cs CTAs of a thread-block cluster computed
// the same tile over disjoint k ranges. Each 32-column chunk has an owner
// rank ((chunk / unit) % cs); every CTA writes the chunks it does not own
// to a global (L2-resident) exchange buffer, one cluster barrier, then each
// owner adds the other ranks' partials to its own (still in TMEM) in rank
// order (deterministic) and runs the epilogue on its chunks: a reduce-scatter
// inside the GEMM, no reduce kernel. (The same exchange through DSMEM loads
// measured 2-3x slower: ~10-16 B/ns per SM of remote shared-memory reads.)
// Exchange layout: [tile][chunk][src rank][warp][column j][lane] floats, so
// every store / load is a coalesced 128-byte warp access.
struct AccSrc {
  int cs = 1, rank = 0, q = 0;
  const float* xw = nullptr;  // exchange buffer of this tile
  int nchunks = 0;            // 32-column chunks per tile
  __device__ __forceinline__ bool owns(int col, int unit) const { return cs <= 1 || (col / unit) % cs == rank; }
};
__device__ __forceinline__ int64_t xw_off(int chunk, int src, int cs, int q) {
  return ((int64_t(chunk) * cs + src) * 4 + q) * 1024;
}
__device__ __forceinline__ void acc_ld32(const AccSrc& src, uint32_t taddr, int crel, float* v) {
  tc::tmem_ld32(taddr, v);
  if (src.cs <= 1) return;
  const int lane = threadIdx.x & 31;
  float own[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    own[j] = v[j];
    v[j] = 0.f;
  }
  // rank order (deterministic); unrolled over the (<= 4) ranks so the
  // compiler can issue later ranks' loads ahead of earlier ranks' adds
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (r >= src.cs) break;
    const float* p = src.xw + xw_off(crel >> 5, r, src.cs, src.q) + lane;
    const bool mine = r == src.rank;
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += mine ? own[j] : __ldcg(p + 32 * j);
  }
}

// One 32x32 accumulator block of an epilogue warp: TMEM lanes row0..row0+31
// (this warp's quadrant), columns col0..col0+31. tcgen05.ld gives thread =
// row; the block is transposed through padded smem (`my`, 32x33 floats) so
// every global access below is a 128-byte row-coalesced warp access. The
// residual operand (RESID) is prefetched before the TMEM load so its latency
// overlaps it. P != nullptr stores an fp32 split-K partial instead.
__device__ __forceinline__ void epi_block(const Epi& e, float* my, uint32_t taddr, int64_t row0,
                                          int64_t col0, int64_t M, int64_t N, float* P,
                                          const AccSrc& src = AccSrc(), int crel = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t col = col0 + lane;
  const bool cok = col < N;
  float rv[32];
  const bool resid = !P && e.kind == Epi::RESID;
  if (resid) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t r = row0 + rr;
      rv[rr] = (r < M && cok) ? e.resid[r * e.ldr + col] : 0.f;
    }
  }
  float v[32];
  acc_ld32(src, taddr, crel, v);
  if (!P && e.kind == Epi::NONE) return;
  if (!P && e.kind == Epi::F32_DIRECT) {  // debug: row-per-thread 16-byte stores, no transpose
    const int64_t r = row0 + lane;
    if (r < M) {
      float4* o = reinterpret_cast<float4*>(static_cast<float*>(e.out) + r * e.ldo + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) my[lane * 33 + j] = v[j];
  __syncwarp();
  if (!P && e.kind == Epi::STAGE_ONLY) {  // debug: transpose through smem, no global access
    float acc = 0.f;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) acc += my[rr * 33 + lane];
    if (acc == 12345.678f) static_cast<float*>(e.out)[lane] = acc;
    __syncwarp();
    return;
  }
  if (P) {
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t r = row0 + rr;
      if (r < M && cok) P[r * N + col] = my[rr * 33 + lane];
    }
  } else if (e.kind == Epi::SWIGLU) {  // gate/up adjacent columns: even lane writes silu(g)*u
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t r = row0 + rr;
      const float g = my[rr * 33 + lane];
      const float up = __shfl_down_sync(0xffffffffu, g, 1);
      if (r < M && col + 1 < N && !(lane & 1))
        static_cast<bf16*>(e.out)[r * e.ldo + col / 2] = fromf<bf16>(silu_mul(g, up));
    }
  } else if (resid) {
    const float b = (e.bias && cok) ? e.bias[col] : 0.f;
    float* o = static_cast<float*>(e.out);
    bf16* o2 = static_cast<bf16*>(e.out2);
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t r = row0 + rr;
      if (r < M && cok) {
        const float h = rv[rr] + (my[rr * 33 + lane] + b);
        o[r * e.ldo + col] = h;
        if (o2) o2[r * e.ldo2 + col] = fromf<bf16>(h);
      }
    }
  } else {
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t r = row0 + rr;
      if (r < M && cok) epi_elem<bf16>(e, r, col, my[rr * 33 + lane]);
    }
  }
  __syncwarp();
}

// Epilogue kinds resolved at compile time (EK_GENERIC = runtime e.kind via
// epi_block, used when the output cannot be described by a TMA map).
enum : int { EK_F32 = 0, EK_CDT = 1, EK_RESID = 2, EK_TANH = 3, EK_SWIGLU = 4, EK_NONE = 5,
             EK_PARTIAL = 8, EK_GENERIC = 9, EK_QKV = 10 };

namespace tc {
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y,
                                             int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}
}  // namespace tc

// QKV epilogue (engine.cpp:128-143, :162-170 fused into the projection):
// thread = token row r (position pos0 + r), 32 consecutive output columns
// per TMEM chunk. Q columns are rotated and stored bf16 for rows < q_rows;
// K columns are rotated and stored as one contiguous 64-byte run of the
// token's K row in its page; V columns go to the transposed V^T page
// layout, where the warp's 32 consecutive tokens make each store a
// contiguous 64-byte run. hd % 32 == 0 so a chunk never straddles a head.
template <int BN>
__device__ __forceinline__ void epi_qkv(const Epi& e, uint32_t tbase, int64_t row0, int64_t col0,
                                        int64_t M, int64_t N, const AccSrc& src = AccSrc()) {
  const EpiKV& kv = e.kv;
  const int lane = threadIdx.x & 31;
  const int64_t r = row0 + lane;
  const bool rok = r < M;
  const int64_t pos = kv.pos(r);
  const int nq = kv.H * kv.hd, nkv = kv.Hkv * kv.hd, half = kv.hd / 2;
  bf16* page = rok ? reinterpret_cast<bf16*>(kv.pool + int64_t(kv.pt[pos / kPageTokens]) * kv.page_bytes)
                   : nullptr;
  const int64_t slot = pos % kPageTokens;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    const int64_t cc = col0 + c;
    if (cc >= N) break;
    if (!src.owns(c, 32)) continue;
    float v[32];
    acc_ld32(src, tbase + uint32_t(c), c, v);
    if (!rok) continue;
    const bool isq = cc < nq, isk = !isq && cc < nq + nkv;
    if (isq || isk) {
      if (isq && r >= kv.q_rows) continue;
      const int t0 = int((isq ? cc : cc - nq) % kv.hd);
      const float4* cs4 = reinterpret_cast<const float4*>(kv.cosT + pos * half + t0 / 2);
      const float4* sn4 = reinterpret_cast<const float4*>(kv.sinT + pos * half + t0 / 2);
      uint32_t w[16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 cq = __ldg(cs4 + j), sq = __ldg(sn4 + j);
        const float cv[4] = {cq.x, cq.y, cq.z, cq.w}, sv[4] = {sq.x, sq.y, sq.z, sq.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float x0 = v[8 * j + 2 * u], x1 = v[8 * j + 2 * u + 1];
          w[4 * j + u] = tc::pack_bf16(x0 * cv[u] - x1 * sv[u], x0 * sv[u] + x1 * cv[u]);
        }
      }
      uint4* dst;
      if (isq) {
        dst = reinterpret_cast<uint4*>(static_cast<bf16*>(kv.q) + r * nq + cc);
      } else {
        const int g = int((cc - nq) / kv.hd);
        dst = reinterpret_cast<uint4*>(page + (int64_t(g) * kPageTokens + slot) * kv.hd + t0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
    } else {
      const int64_t vc = cc - nq - nkv;
      const int g = int(vc / kv.hd), t0 = int(vc % kv.hd);
      bf16* vt = page + int64_t(kv.Hkv) * kPageTokens * kv.hd + (int64_t(g) * kv.hd + t0) * kPageTokens + slot;
#pragma unroll
      for (int j = 0; j < 32; ++j) vt[j * kPageTokens] = __float2bfloat16_rn(v[j]);
    }
  }
}

// One accumulator tile row-block of an epilogue warp through TMA stores.
// The warp owns TMEM lanes [32q, 32q+32) = output rows row0..row0+31; thread
// = row. Outputs are packed into a 32-row x 128-byte staging tile in the
// TMA SWIZZLE_128B layout (16-byte piece j of row r at piece j ^ (r & 7):
// conflict-free st.shared.v4), then one lane issues the bulk tensor store
// (rows >= M and columns >= N are clipped by the TMA unit). Two staging
// tiles per warp alternate; a tile is rewritten only after its previous
// store has finished reading shared memory.
//   F32 / RESID / PARTIAL : 32 accumulator columns per staging tile (f32)
//   CDT / TANH            : 64 columns (bf16)
//   SWIGLU                : 128 accumulator columns -> 64 bf16 outputs
// RESID reads its residual rows directly (16-byte loads issued before the
// TMEM load) and writes the optional bf16 copy with direct 16-byte stores.
template <int KIND, int BN>
__device__ __forceinline__ void epi_unit(const Epi& e, const CUtensorMap* tmC, unsigned char* stage,
                                         int& sbuf, uint32_t tbase, int64_t row0, int64_t col0,
                                         int64_t M, int64_t N, int ks, const AccSrc& src = AccSrc()) {
  constexpr int ACC = (KIND == EK_SWIGLU) ? 128 : (KIND == EK_CDT || KIND == EK_TANH) ? 64 : 32;
  constexpr int PIECES = 128 / (ACC / 32) / 16;  // 16-byte pieces per 32-column chunk
  const int lane = threadIdx.x & 31;
  const int64_t r = row0 + lane;
  const bool rok = r < M;
#pragma unroll 1
  for (int t = 0; t < BN; t += ACC) {
    if (col0 + t >= N) break;
    if (!src.owns(t, ACC)) continue;
    unsigned char* tile = stage + sbuf * 4096;
    if (lane == 0) tc::bulk_wait_read1();
    __syncwarp();
#pragma unroll
    for (int c = 0; c < ACC; c += 32) {
      const int64_t cc = col0 + t + c;  // first accumulator column of this chunk
      float rv[32];
      if constexpr (KIND == EK_RESID) {
        if (rok && cc + 32 <= N && ((e.ldr & 3) == 0)) {
          const float4* src = reinterpret_cast<const float4*>(e.resid + r * e.ldr + cc);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 x = __ldg(src + j);
            rv[4 * j] = x.x;
            rv[4 * j + 1] = x.y;
            rv[4 * j + 2] = x.z;
            rv[4 * j + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rv[j] = (rok && cc + j < N) ? e.resid[r * e.ldr + cc + j] : 0.f;
        }
      }
      float v[32];
      acc_ld32(src, tbase + uint32_t(t + c), t + c, v);
      uint32_t w[32];  // packed output words of this chunk for this row
      if constexpr (KIND == EK_F32 || KIND == EK_PARTIAL || KIND == EK_NONE) {
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(v[j]);
      } else if constexpr (KIND == EK_RESID) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float b = e.bias && cc + j < N ? __ldg(e.bias + cc + j) : 0.f;
          w[j] = __float_as_uint(rv[j] + (v[j] + b));
        }
        if (e.out2 && rok) {
          bf16* o2 = static_cast<bf16*>(e.out2) + r * e.ldo2 + cc;
          if (cc + 32 <= N && ((e.ldo2 & 7) == 0)) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 pk;
              pk.x = tc::pack_bf16(__uint_as_float(w[8 * j]), __uint_as_float(w[8 * j + 1]));
              pk.y = tc::pack_bf16(__uint_as_float(w[8 * j + 2]), __uint_as_float(w[8 * j + 3]));
              pk.z = tc::pack_bf16(__uint_as_float(w[8 * j + 4]), __uint_as_float(w[8 * j + 5]));
              pk.w = tc::pack_bf16(__uint_as_float(w[8 * j + 6]), __uint_as_float(w[8 * j + 7]));
              reinterpret_cast<uint4*>(o2)[j] = pk;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (cc + j < N) o2[j] = __float2bfloat16_rn(__uint_as_float(w[j]));
          }
        }
      } else if constexpr (KIND == EK_CDT) {
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
      } else if constexpr (KIND == EK_TANH) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float b0 = cc + 2 * j < N ? __ldg(e.bias + cc + 2 * j) : 0.f;
          const float b1 = cc + 2 * j + 1 < N ? __ldg(e.bias + cc + 2 * j + 1) : 0.f;
          w[j] = tc::pack_bf16(tanhf(v[2 * j] + b0), tanhf(v[2 * j + 1] + b1));
        }
      } else if constexpr (KIND == EK_SWIGLU) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          w[j] = tc::pack_bf16(silu_mul(v[4 * j], v[4 * j + 1]), silu_mul(v[4 * j + 2], v[4 * j + 3]));
      }
      if constexpr (KIND != EK_NONE) {
        const int p0 = (c / 32) * PIECES;
#pragma unroll
        for (int j = 0; j < PIECES; ++j) {
          const int piece = (p0 + j) ^ (lane & 7);
          *reinterpret_cast<uint4*>(tile + lane * 128 + piece * 16) =
              make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        }
      }
    }
    if constexpr (KIND != EK_NONE) {
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int x = int(KIND == EK_SWIGLU ? (col0 + t) / 2 : col0 + t);
        if constexpr (KIND == EK_PARTIAL)
          tc::tma_store_3d(tmC, tile, x, int(row0), ks);
        else
          tc::tma_store_2d(tmC, tile, x, int(row0));
        tc::bulk_commit();
      }
      sbuf ^= 1;
    }
  }
}

// CTA owning iteration i of a stream-K schedule over G CTAs.
__host__ __device__ inline long long sk_cta(long long i, int G, long long T) { return ((i + 1) * G - 1) / T; }
// Pieces (partial slots in use) of n-tile `n`.
__host__ __device__ inline int sk_pieces(int n, int num_k, int G, long long T) {
  const long long ts = (long long)n * num_k;
  return int(sk_cta(ts + num_k - 1, G, T) - sk_cta(ts, G, T) + 1);
}
// Partial-slot count of one output column for the split-K reduces: uniform
// `splits`, or the stream-K piece count of the column's tile.
struct SkInfo {
  int G = 0, num_k = 0, bn = 0;
  long long T = 0;
  __device__ __forceinline__ int slots(int splits, int64_t col) const {
    return T > 0 ? sk_pieces(int(col / bn), num_k, G, T) : splits;
  }
};

// Work unit of the 1-SM kernel: tile (m, n), k-blocks [k0, k1), partial slot.
struct Unit {
  int m, n, k0, k1, ks;
};
// Stream-K schedule (sk_T > 0, single m-tile): CTA c owns the k-block
// iterations [c*T/G, (c+1)*T/G) of the linearised (n_tile, k_block) space,
// so every CTA streams the same number of weight blocks whatever the tile
// count; each tile crossing starts a new piece whose slot is its index among
// the CTAs touching that tile (fixed order -> deterministic reduce).
// Otherwise units (m, n, split) are dealt round-robin, m fastest.
__device__ __forceinline__ bool unit_at(int i, int mt, int nt, int splits, int kb_per, int num_k, int sk_G,
                                        long long sk_T, Unit& u, int cs = 1) {
  if (cs > 1) {  // cluster split-K: one unit per CTA, cluster = tile, rank = k slice
    if (i > 0) return false;
    u.m = 0;
    u.n = int(blockIdx.x) / cs;
    u.ks = int(blockIdx.x) % cs;
    u.k0 = u.ks * kb_per;
    u.k1 = min(num_k, u.k0 + kb_per);
    return true;
  }
  if (sk_T > 0) {
    const long long c = blockIdx.x;
    const long long beg = c * sk_T / sk_G, end = (c + 1) * sk_T / sk_G;
    long long it = beg;
    for (int q = 0; q < i && it < end; ++q) it = (it / num_k + 1) * num_k;
    if (it >= end) return false;
    u.m = 0;
    u.n = int(it / num_k);
    const long long ts = (long long)u.n * num_k, te = ts + num_k;
    u.k0 = int(it - ts);
    u.k1 = int((end < te ? end : te) - ts);
    u.ks = int(c - ((ts + 1) * sk_G - 1) / sk_T);
    return true;
  }
  const int uu = blockIdx.x + i * gridDim.x;
  if (uu >= mt * nt * splits) return false;
  u.m = uu % mt;
  const int rest = uu / mt;
  u.n = rest % nt;
  u.ks = rest / nt;
  u.k0 = u.ks * kb_per;
  u.k1 = min(num_k, u.k0 + kb_per);
  return true;
}

// Persistent warp-specialised tcgen05 GEMM, C[M,N] = A[M,K] B[N,K]^T.
//   warp 0      : TMA producer (A 128x64 + B BNx64 bf16 tiles, SW128) into an
//                 STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      : TMEM owner + single-thread tcgen05.mma issuer; two TMEM
//                 accumulators (2 x BN fp32 columns) so the epilogue of unit
//                 i overlaps the mainloop of unit i+1 (tmem_full/tmem_empty)
//   warps 2..5  : epilogue; warp w reads TMEM lanes 32*(w%4).. via
//                 tcgen05.ld.32x32b, transposes each 32x32 block through
//                 padded smem so global stores/loads are row-coalesced, then
//                 applies the fused epilogue (or stores an fp32 split-K
//                 partial).
// Work units = (m_tile, n_tile, k_split), m fastest: co-resident CTAs share
// the weight (B) tile so each weight tile streams from HBM about once.
template <int BN, int STAGES, int KIND>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, int M, int N, int K, int mt, int nt, int splits, int kb_per, Epi e,
              float* __restrict__ partial, int sk_G, long long sk_T, int cs, float* __restrict__ xw) {
  constexpr int BM = 128, BK = 64;
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  extern __shared__ unsigned char smem_raw[];
  if (threadIdx.x == 0) {
    gemm_ts(32 + blockIdx.x);
    if (blockIdx.x == 0) gemm_ts(0);
    gemm_span_stamp(e.span, false);
  }
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  float* stg = reinterpret_cast<float*>(sB + STAGES * B_BYTES);  // 4 warps x 2 x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 4 * 2 * 1024);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_k = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_slot)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0 && blockIdx.x == 0) gemm_ts(1);
  pdl_trigger();  // the next kernel in the stream may start its prologue

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int s = 0;
      uint32_t ph = 0;
      Unit un;
      // weights do not depend on the preceding kernel: the first unit's first
      // stages of B are in flight before the dependency wait (PDL)
      int pre = 0;
      if (unit_at(0, mt, nt, splits, kb_per, num_k, sk_G, sk_T, un, cs)) {
        pre = min(STAGES, un.k1 - un.k0);
        for (int q = 0; q < pre; ++q) {
          tc::mbar_expect_tx(&full[q], A_BYTES + B_BYTES);
          tc::tma_load_2d(sB + q * B_BYTES, &tmB, &full[q], (un.k0 + q) * BK, un.n * BN);
        }
      }
      pdl_wait();
      for (int i = 0; unit_at(i, mt, nt, splits, kb_per, num_k, sk_G, sk_T, un, cs); ++i) {
        for (int kb = un.k0; kb < un.k1; ++kb) {
          if (i == 0 && kb - un.k0 < pre) {  // first pass over the ring: B already issued
            tc::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, un.m * BM);
          } else {
            tc::mbar_wait(&empty[s], ph ^ 1);
            tc::mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
            tc::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, un.m * BM);
            tc::tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, un.n * BN);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                                 (uint32_t(BM >> 4) << 24);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      Unit un;
      for (int i = 0; unit_at(i, mt, nt, splits, kb_per, num_k, sk_G, sk_T, un, cs); ++i) {
        const int k0 = un.k0, k1 = un.k1;
        tc::mbar_wait(&tempty[acc], aph ^ 1);  // epilogue drained this accumulator
        tc::fence_after();
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kb = k0; kb < k1; ++kb) {
          tc::mbar_wait(&full[s], ph);
          tc::fence_after();
          if (blockIdx.x == 0 && i == 0 && kb == k0) gemm_ts(2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = tc::sw128_desc(sA + s * A_BYTES + k * 32);
            const uint64_t db = tc::sw128_desc(sB + s * B_BYTES + k * 32);
            tc::mma_bf16(d, da, db, idesc, (kb > k0 || k > 0) ? 1u : 0u);
          }
          tc::mma_commit(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc::mma_commit(&tfull[acc]);
        if (blockIdx.x == 0 && i == 0) gemm_ts(3);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {  // epilogue warps 2..5
    pdl_wait();  // outputs / residual inputs belong to the dependency chain
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    float* my = stg + q * 32 * 33;
    unsigned char* stage = reinterpret_cast<unsigned char*>(stg) + q * 8192;
    int sbuf = 0;
    int acc = 0;
    uint32_t aph = 0;
    Unit un;
    for (int i = 0; unit_at(i, mt, nt, splits, kb_per, num_k, sk_G, sk_T, un, cs); ++i) {
      const int m = un.m, n = un.n, ks = un.ks;
      tc::mbar_wait(&tfull[acc], aph);
      tc::fence_after();
      if (blockIdx.x == 0 && warp == 2 && lane == 0 && i == 0) gemm_ts(4);
      const int64_t row0 = int64_t(m) * BM + 32 * q;
      float* P = partial ? partial + int64_t(ks) * M * N : nullptr;
      if (cs > 1) {  // hand the chunks other ranks own to the exchange buffer; reduced below
        const int unit = (KIND == EK_CDT || KIND == EK_TANH) ? 64 : 32;
        float* tile = xw + int64_t(n) * (BN / 32) * cs * 4096;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if ((c / unit) % cs == ks) continue;
          float v[32];
          tc::tmem_ld32(tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN + c), v);
          float* dst = tile + xw_off(c >> 5, ks, cs, q) + lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(dst + 32 * j, v[j]);
        }
      } else if constexpr (KIND == EK_GENERIC) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (int64_t(n) * BN + c >= N) break;
          epi_block(e, my, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN + c), row0,
                    int64_t(n) * BN + c, M, N, P);
        }
      } else if constexpr (KIND == EK_QKV) {
        epi_qkv<BN>(e, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN), row0, int64_t(n) * BN, M, N);
      } else {
        epi_unit<KIND, BN>(e, &tmC, stage, sbuf, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN),
                           row0, int64_t(n) * BN, M, N, ks);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&tempty[acc])) : "memory");
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  if (cs > 1) {
    if (blockIdx.x == 0 && warp == 2 && lane == 0) gemm_ts(5);
    // every rank's exchange writes are done (cluster-scope release/acquire)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (blockIdx.x == 0 && warp == 2 && lane == 0) gemm_ts(6);
    if (warp >= 2) {
      Unit un;
      unit_at(0, mt, nt, splits, kb_per, num_k, sk_G, sk_T, un, cs);
      AccSrc src;
      src.cs = cs;
      src.rank = un.ks;
      src.q = warp & 3;
      src.xw = xw + int64_t(un.n) * (BN / 32) * cs * 4096;
      const int q = warp & 3;
      float* my = stg + q * 32 * 33;
      unsigned char* stage = reinterpret_cast<unsigned char*>(stg) + q * 8192;
      int sbuf = 0;
      const int64_t row0 = 32 * q;
      const uint32_t tacc = tmem + (uint32_t(32 * q) << 16);  // single unit: accumulator 0
      if constexpr (KIND == EK_GENERIC) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (int64_t(un.n) * BN + c >= N) break;
          if (src.owns(c, 32)) epi_block(e, my, tacc + uint32_t(c), row0, int64_t(un.n) * BN + c, M, N, nullptr, src, c);
        }
      } else if constexpr (KIND == EK_QKV) {
        epi_qkv<BN>(e, tacc, row0, int64_t(un.n) * BN, M, N, src);
      } else {
        epi_unit<KIND, BN>(e, &tmC, stage, sbuf, tacc, row0, int64_t(un.n) * BN, M, N, 0, src);
      }
    }
    if (blockIdx.x == 0 && warp == 2 && lane == 0) gemm_ts(7);
  }
  if (blockIdx.x == 0 && warp == 2 && lane == 0) gemm_ts(8);
  if (warp >= 2 && lane == 0) tc::bulk_wait_all();
  if (blockIdx.x == 0 && warp == 2 && lane == 0) gemm_ts(9);
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(uint32_t(2 * BN)));
  }
  if (threadIdx.x == 0) {
    gemm_ts(32 + 256 + blockIdx.x);
    gemm_span_stamp(e.span, true);
  }
}

// ---------------------------------------------------------------- 2-SM pair
namespace tc {
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of CTA rank 0
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion bytes land on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}
}  // namespace tc

// CTA-pair (cta_group::2) variant for M > 128: the pair computes a 256x256
// tile; each CTA stages its own 128-row half of A and its own 128-row half
// of B (32 KB per k-block instead of 48 KB for a 1-SM 128x256 tile, so the
// L2->SM feed per MAC drops by a third), the leader's single thread issues
// M=256 x N=256 MMAs that read both CTAs' shared memory, and each CTA's
// TMEM receives its 128 accumulator rows. Same double-buffered TMEM and
// epilogue as k_gemm_tc; the leader's tmem_empty barrier collects the
// epilogue warps of both CTAs.
template <int STAGES, int KSUB, int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, int M, int N, int K, int mt, int nt, int splits, int kb_per, Epi e,
               float* __restrict__ partial) {
  constexpr int BK = 64 * KSUB, BN = 256;  // KSUB 64-wide SW128 sub-tiles per stage
  constexpr uint32_t SUB = 128 * 64 * 2;
  constexpr uint32_t A_BYTES = SUB * KSUB, B_BYTES = SUB * KSUB;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  float* stg = reinterpret_cast<float*>(sB + STAGES * B_BYTES);  // 4 warps x 2 x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 4 * 2 * 1024);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2] (leader: 8 arrivals = 4 warps x 2 CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cta_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int num_k = (K + BK - 1) / BK;
  const int units = mt * nt * splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own A half + own B half
      int s = 0;
      uint32_t ph = 0;
      for (int u = cid; u < units; u += ncl) {
        const int m = u % mt, rest = u / mt, n = rest % nt, ks = rest / nt;
        const int k0 = ks * kb_per, k1 = min(num_k, k0 + kb_per);
        for (int kb = k0; kb < k1; ++kb) {
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) tc::mbar_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
#pragma unroll
          for (int j = 0; j < KSUB; ++j) {
            tc::tma_load_2d_pair(sA + s * A_BYTES + j * SUB, &tmA, &full[s], kb * BK + 64 * j,
                                 m * 256 + int(rank) * 128);
            tc::tma_load_2d_pair(sB + s * B_BYTES + j * SUB, &tmB, &full[s], kb * BK + 64 * j,
                                 n * 256 + int(rank) * 128);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer (pair leader)
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) |
                                 (uint32_t(256 >> 4) << 24);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int u = cid; u < units; u += ncl) {
        const int ks = u / mt / nt;
        const int k0 = ks * kb_per, k1 = min(num_k, k0 + kb_per);
        tc::mbar_wait(&tempty[acc], aph ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kb = k0; kb < k1; ++kb) {
          tc::mbar_wait(&full[s], ph);
          tc::fence_after();
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t off = (k >> 2) * SUB + (k & 3) * 32;
            const uint64_t da = tc::sw128_desc(sA + s * A_BYTES + off);
            const uint64_t db = tc::sw128_desc(sB + s * B_BYTES + off);
            tc::mma_bf16_pair(d, da, db, idesc, (kb > k0 || k > 0) ? 1u : 0u);
          }
          tc::mma_commit_pair(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc::mma_commit_pair(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {  // epilogue warps 2..5 of both CTAs
    const int q = warp & 3;
    float* my = stg + q * 32 * 33;
    unsigned char* stage = reinterpret_cast<unsigned char*>(stg) + q * 8192;
    int sbuf = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int u = cid; u < units; u += ncl) {
      const int m = u % mt, rest = u / mt, n = rest % nt, ks = rest / nt;
      tc::mbar_wait(&tfull[acc], aph);
      tc::fence_after();
      const int64_t row0 = int64_t(m) * 256 + int64_t(rank) * 128 + 32 * q;
      float* P = partial ? partial + int64_t(ks) * M * N : nullptr;
      if constexpr (KIND == EK_GENERIC) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (int64_t(n) * BN + c >= N) break;
          epi_block(e, my, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN + c), row0,
                    int64_t(n) * BN + c, M, N, P);
        }
      } else if constexpr (KIND == EK_QKV) {
        epi_qkv<BN>(e, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN), row0, int64_t(n) * BN, M, N);
      } else {
        epi_unit<KIND, BN>(e, &tmC, stage, sbuf, tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN),
                           row0, int64_t(n) * BN, M, N, ks);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::arrive_leader(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  if (warp >= 2 && lane == 0) tc::bulk_wait_all();
  tc::fence_before();
  tc::cluster_sync();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
  }
}

// Deterministic split-K reduction (fixed split order) + fused epilogue; four
// consecutive columns per thread (128-bit partial loads) when N % 4 == 0.
template <class T>
__global__ void k_splitk_reduce(const float* __restrict__ P, int splits, int64_t M, int64_t N,
                                Epi e, SkInfo sk) {
  pdl_trigger();
  pdl_wait();
  const int64_t MN = M * N;
  if ((N & 3) == 0) {
    const int64_t q = N >> 2, total = M * q;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
      const int64_t r = i / q, c = (i % q) * 4;
      const int ns = sk.slots(splits, c);
      float4 a = *reinterpret_cast<const float4*>(P + r * N + c);
      for (int s0 = 1; s0 < ns; s0 += 4) {  // 4 partial loads in flight, fixed order
        float4 b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          b[u] = s0 + u < ns ? *reinterpret_cast<const float4*>(P + int64_t(s0 + u) * MN + r * N + c)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a.x += b[u].x;
          a.y += b[u].y;
          a.z += b[u].z;
          a.w += b[u].w;
        }
      }
      if (e.kind == Epi::SWIGLU) {
        T* o = static_cast<T*>(e.out) + r * e.ldo + c / 2;
        o[0] = fromf<T>(silu_mul(a.x, a.y));
        o[1] = fromf<T>(silu_mul(a.z, a.w));
      } else {
        epi_elem<T>(e, r, c, a.x);
        epi_elem<T>(e, r, c + 1, a.y);
        epi_elem<T>(e, r, c + 2, a.z);
        epi_elem<T>(e, r, c + 3, a.w);
      }
    }
    if (threadIdx.x == 0) gemm_span_stamp(e.span, true);  // the reduce ends the GEMM's span
    return;
  }
  const bool sw = e.kind == Epi::SWIGLU;
  const int64_t cols = sw ? N / 2 : N;
  const int64_t total = M * cols;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    if (sw) {
      float g = 0.f, u = 0.f;
      const int ns = sk.slots(splits, 2 * c);
      for (int s = 0; s < ns; ++s) {
        const float* p = P + int64_t(s) * MN + r * N + 2 * c;
        g += p[0];
        u += p[1];
      }
      static_cast<T*>(e.out)[r * e.ldo + c] = fromf<T>(silu_mul(g, u));
    } else {
      float a = 0.f;
      const int ns = sk.slots(splits, c);
      for (int s = 0; s < ns; ++s) a += P[int64_t(s) * MN + r * N + c];
      epi_elem<T>(e, r, c, a);
    }
  }
  if (threadIdx.x == 0) gemm_span_stamp(e.span, true);
}

// Split-K partner of the fused QKV epilogue (weight-streaming shapes, small
// M): sums the fp32 partials in fixed split order, then RoPE + Q store + paged
// K / V^T scatter exactly as epi_qkv. Block = 64 tokens x 32 columns staged
// in smem so both the token-major (Q, K) and the dimension-major (V^T)
// stores are contiguous runs.
__global__ void __launch_bounds__(256) k_qkv_reduce(const float* __restrict__ P, int splits,
                                                     int64_t M, int64_t N, EpiKV kv, SkInfo sk) {
  // block = 32 tokens x 32 columns (M = 128 -> 768 CTAs: enough warps per
  // SM to hide the partial loads); RoPE tables and page ids are fetched
  // before the partial sums, off the dependent chain
  constexpr int RB = 32, RJ = RB / 8;
  __shared__ float t[RB][33];
  pdl_trigger();
  pdl_wait();
  const int64_t r0 = int64_t(blockIdx.x) * RB;
  const int64_t cc = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // column, token group
  const int64_t MN = M * N;
  splits = sk.slots(splits, cc);  // a 32-column block never straddles a tile
  const int nq = kv.H * kv.hd, nkv = kv.Hkv * kv.hd, half = kv.hd / 2;
  const bool isq = cc < nq, isk = !isq && cc < nq + nkv;
  const int t0 = int((isq ? cc : cc - nq) % kv.hd);
  const int i = (t0 + tx) >> 1;
  float cs[RJ], sn[RJ];
#pragma unroll
  for (int j = 0; j < RJ; ++j) {
    const int64_t r = r0 + ty + 8 * j;
    cs[j] = sn[j] = 0.f;
    if ((isq || isk) && r < M) {
      const int64_t pos = kv.pos(r);
      cs[j] = __ldg(kv.cosT + pos * half + i);
      sn[j] = __ldg(kv.sinT + pos * half + i);
    }
  }
  // all partial loads of this thread in flight before the (fixed-order) sums
  float a[RJ];
#pragma unroll
  for (int j = 0; j < RJ; ++j) a[j] = 0.f;
  for (int s0 = 0; s0 < splits; s0 += 4) {
    float v[4][RJ];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int64_t r = r0 + ty + 8 * j;
        v[u][j] = (s0 + u < splits && r < M && cc + tx < N) ? P[int64_t(s0 + u) * MN + r * N + cc + tx] : 0.f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < RJ; ++j) a[j] += v[u][j];
  }
#pragma unroll
  for (int j = 0; j < RJ; ++j) t[ty + 8 * j][tx] = a[j];
  __syncthreads();
  if (isq || isk) {
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
      const int rr = ty + 8 * j;
      const int64_t r = r0 + rr;
      if (r >= M || (isq && r >= kv.q_rows)) continue;
      const int64_t pos = kv.pos(r);
      const float x0 = t[rr][tx & ~1], x1 = t[rr][tx | 1];
      const float y = (tx & 1) ? (x0 * sn[j] + x1 * cs[j]) : (x0 * cs[j] - x1 * sn[j]);
      if (isq) {
        static_cast<bf16*>(kv.q)[r * nq + cc + tx] = __float2bfloat16_rn(y);
      } else {
        const int g = int((cc - nq) / kv.hd);
        bf16* page = reinterpret_cast<bf16*>(kv.pool + int64_t(kv.pt[pos / kPageTokens]) * kv.page_bytes);
        page[(int64_t(g) * kPageTokens + pos % kPageTokens) * kv.hd + t0 + tx] = __float2bfloat16_rn(y);
      }
    }
  } else {
    const int64_t vc = cc - nq - nkv;
    const int g = int(vc / kv.hd), tv0 = int(vc % kv.hd);
    // thread -> (dimension d, 4 consecutive tokens)
    const int d = threadIdx.x >> 3, tg = (threadIdx.x & 7) * 4;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = r0 + tg + u;
      if (r >= M) break;
      const int64_t pos = kv.pos(r);
      bf16* page = reinterpret_cast<bf16*>(kv.pool + int64_t(kv.pt[pos / kPageTokens]) * kv.page_bytes);
      page[int64_t(kv.Hkv) * kPageTokens * kv.hd + (int64_t(g) * kv.hd + tv0 + d) * kPageTokens +
           pos % kPageTokens] = __float2bfloat16_rn(t[tg + u][d]);
    }
  }
}

// ---------------------------------------------------------------- host side
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    KB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(KRUL_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}
}  // namespace
// cuTensorMapEncodeTiled behind a cache keyed by every argument: a map only
// encodes an address, shape, strides and box (no data), so reuse is exact.
// Eager paths (decode steps: ~480 maps per token) otherwise spend
// milliseconds of host time re-encoding identical maps; graph replays
// carry their maps as kernel parameters and never come here.
CUresult tmap_encode_cached(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr,
                            const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                            const cuuint32_t* es, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                            CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  static std::mutex mu;
  static std::unordered_map<std::string, CUtensorMap> cache;
  std::string key;
  key.reserve(160);
  auto put = [&key](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
  put(&dt, sizeof dt);
  put(&rank, sizeof rank);
  put(&ptr, sizeof ptr);
  put(dims, sizeof(cuuint64_t) * rank);
  put(strides, sizeof(cuuint64_t) * (rank - 1));
  put(box, sizeof(cuuint32_t) * rank);
  put(es, sizeof(cuuint32_t) * rank);
  put(&il, sizeof il);
  put(&sw, sizeof sw);
  put(&l2, sizeof l2);
  put(&oob, sizeof oob);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return CUDA_SUCCESS;
  }
  const CUresult r = encode_fn()(m, dt, rank, ptr, dims, strides, box, es, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) {
    if (cache.size() > 8192) cache.clear();
    cache.emplace(std::move(key), *m);
  }
  return r;
}
namespace {
// Row-major bf16 [rows][cols] with leading dimension ld (elements); box
// [box_rows][64] with 128-byte swizzle.
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = tmap_encode_cached(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRUL_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

struct GemmPlan {
  int bn = 256, splits = 1, kb_per = 1, grid = 1;
  bool pair = false;  // cta_group::2, 256x256 tiles
  // stream-K (single m-tile, 1-SM kernel): grid CTAs share T = nt * num_k
  // k-block iterations evenly; `splits` = partial slots (max pieces per tile)
  long long sk_T = 0;
  int cs = 1;  // > 1: cluster split-K, cs CTAs per tile reduce over DSMEM (grid = nt * cs)
};

// Clusters of `cs` CTAs of the 1-SM kernel (BN-wide tiles, one CTA per SM)
// that can be resident at once -- the cluster split-K grid must fit in one
// wave (a cluster waiting for a second wave would serialise the tail).
int max_clusters(int bn, int cs);


// Pick the kernel (1-SM 128xBN or 2-SM 256x256), tile width and split-K
// count with a small cost model (ns). Per k-block time = max(MMA issue time,
// weight bytes streamed from HBM by this SM (shared by the co-resident
// m-tiles), operand bytes through L2 -> SM at the measured ~75 B/ns/SM);
// times the k-blocks on the busiest SM, plus the split-K partial round trip.
GemmPlan plan_gemm_f(int64_t M, int64_t N, int64_t K, int sms, bool allow_split, bool cs_ok, int force,
                     bool* found) {
  const int64_t num_k = (K + 63) / 64;
  GemmPlan best;
  double best_t = 1e30;
  GemmPlan cl;  // the cluster split-K candidate of the automatic plan
  cl.grid = 0;
  cl.cs = 99;
  // constants fitted to a measured sweep of every (variant, split) on the
  // pyramid / new-input shapes with weights streamed from HBM
  // (tools/gemm_sweep.py, 8B + 70B shapes; regret of the chosen plan 3.6% -> 2.1%)
  const double l2_bw = 140.0, hbm_bw = 7000.0, clk = 1.85, unit_ns = 2000.0, pair_eff = 0.8,
               split_ns = 1500.0, split_bw = 3000.0, cs_ns = 1500.0;
  for (int variant = 0; variant < 3; ++variant) {
    const bool pair = variant == 0;
    const int bn = variant == 2 ? 128 : 256;
    const int bm = pair ? 256 : 128;
    if (pair && M <= 128 && force != 3 && force != 4) continue;
    if ((force == 1 && variant != 1) || (force == 2 && variant != 2) ||
        ((force == 3 || force == 4) && variant != 0) || ((force == 5 || force == 6) && variant == 0))
      continue;
    const int64_t mt = (M + bm - 1) / bm, nt = (N + bn - 1) / bn;
    const int64_t slots = pair ? sms / 2 : sms;
    for (int s = 1; s <= 16 && force != 11 && force != 12; ++s) {
      const int64_t kb_per = (num_k + s - 1) / s;
      const int64_t splits = (num_k + kb_per - 1) / kb_per;
      if (splits != s) continue;
      if (g_gemm_splits > 0 && splits != g_gemm_splits) continue;
      if (!allow_split && splits > 1) break;
      if (splits > 1 && M * N * splits * 4 > (int64_t(256) << 20)) break;
      const int64_t units = mt * nt * splits;
      const int64_t active = std::min<int64_t>(units, slots);
      const int64_t per = (units + slots - 1) / slots;
      // per-SM quantities (a pair unit is two SMs' worth of work)
      const double mma_ns = (bn == 256 ? 512.0 : 256.0) / clk / (pair ? pair_eff : 1.0);
      const double b_bytes = (pair ? 128.0 : double(bn)) * 128.0, a_bytes = 128.0 * 128.0;
      const double share = double(std::min<int64_t>(mt, active));
      const double sm_active = double(active) * (pair ? 2.0 : 1.0);
      const double hbm_ns = (b_bytes / share) / (hbm_bw / sm_active);
      const double l2_ns = (a_bytes + b_bytes) / l2_bw;
      const double kb_ns = std::max(mma_ns, std::max(hbm_ns, l2_ns));
      double t = double(per) * double(kb_per) * kb_ns + double(per) * unit_ns;
      if (splits > 1) t += double(M) * double(N) * double(splits) * 8.0 / split_bw + split_ns;
      if (t < best_t * 0.97) {
        best_t = t;
        best.pair = pair;
        best.bn = bn;
        best.splits = int(splits);
        best.kb_per = int(kb_per);
        best.grid = int(active) * (pair ? 2 : 1);
        best.sk_T = 0;
        best.cs = 1;
      }
    }
    // cluster split-K (one m-tile, 1-SM kernel): cs CTAs per tile over
    // disjoint k ranges, reduced through DSMEM inside the GEMM (debug force
    // 11 / 12 = only these with 256- / 128-wide tiles, g_gemm_splits = cs;
    // force 9 = auto without them)
    const bool cs_forced = (force == 11 && bn == 256) || (force == 12 && bn == 128);
    if (!pair && mt == 1 && allow_split && cs_ok && (force == 0 || cs_forced)) {
      for (int cs = 2; cs <= 4; ++cs) {
        if (cs_forced && g_gemm_splits > 0 && cs != g_gemm_splits) continue;
        const int64_t kb_per = (num_k + cs - 1) / cs;
        if ((cs - 1) * kb_per >= num_k) continue;  // every rank gets k blocks
        const int64_t ctas = nt * cs;
        if (ctas > sms || nt > max_clusters(bn, cs)) continue;
        GemmPlan cp;
        cp.bn = bn;
        cp.splits = 1;
        cp.kb_per = int(kb_per);
        cp.grid = int(ctas);
        cp.cs = cs;
        if (cs_forced) {
          if (best_t > 0.0) {
            best_t = 0.0;
            best = cp;
          }
        } else if (ctas > cl.grid || (ctas == cl.grid && cs < cl.cs) ||
                   (ctas == cl.grid && cs == cl.cs && bn == 128)) {
          // measured (tools/gemm_cs_sweep.py, Llama-3-8B / 70B weight-streaming
          // shapes): the cluster plan with the most CTAs wins, then the smaller
          // cluster; the cost model's per-k-block terms do not rank these
          cl = cp;
        }
      }
    }
    // stream-K: one m-tile, every SM streams T / sms weight blocks
    // (debug force: 5 = stream-K with 256-wide tiles, 6 = with 128-wide).
    // Not a candidate of the automatic plan: measured slower than the best
    // split-K plan on every weight-streaming shape of the workloads.
    const bool sk_forced = (force == 5 && bn == 256) || (force == 6 && bn == 128);
    if (!pair && mt == 1 && allow_split && sk_forced) {
      const long long T = (long long)nt * num_k;
      if (T >= 2 * sms && (g_gemm_splits <= 0)) {
        int maxp = 1;
        for (int n = 0; n < nt; ++n) maxp = std::max(maxp, sk_pieces(n, int(num_k), sms, T));
        const double per = double(T) / double(sms);
        const double mma_ns = (bn == 256 ? 512.0 : 256.0) / clk;
        const double b_bytes = double(bn) * 128.0, a_bytes = 128.0 * 128.0;
        const double hbm_ns = b_bytes / (hbm_bw / double(sms));
        const double l2_ns = (a_bytes + b_bytes) / l2_bw;
        const double kb_ns = std::max(mma_ns, std::max(hbm_ns, l2_ns));
        const double pieces = double(nt + sms);  // partial tiles written + read (L2-resident)
        double t = per * kb_ns + 2.0 * 600.0 + pieces * 128.0 * bn * 4.0 * 2.0 / 12000.0 + 2500.0;
        if (sk_forced) t = 0.0;
        if (M * N * maxp * 4 <= (int64_t(256) << 20) && t < best_t * 0.97) {
          best_t = t;
          best.pair = false;
          best.bn = bn;
          best.splits = maxp;
          best.kb_per = 0;
          best.grid = sms;
          best.sk_T = T;
          best.cs = 1;
        }
      }
    }
  }
  if (force == 0 && g_gemm_splits <= 0 && cl.grid >= 64) {
    *found = true;
    return cl;
  }
  *found = best_t < 1e30;
  return best;
}
GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int sms, bool allow_split, bool cs_ok = false) {
  bool found = false;
  GemmPlan gp = plan_gemm_f(M, N, K, sms, allow_split, cs_ok, g_gemm_force, &found);
  if (!found) gp = plan_gemm_f(M, N, K, sms, allow_split, cs_ok, 0, &found);  // forced plan not applicable
  return gp;
}

// Output map for the TMA-store epilogue: 2-D [rows][cols] (or 3-D
// [splits][rows][cols] for split-K partials), 32-row x 128-byte boxes,
// SWIZZLE_128B. Returns false when the output cannot be described (address or
// row stride not 16-byte aligned) -> generic epilogue.
bool make_out_map(CUtensorMap* m, const Epi& e, int64_t M, int64_t N, int splits, float* partial,
                  int* kind) {
  std::memset(m, 0, sizeof *m);
  int k = partial ? EK_PARTIAL : e.kind;
  if (k == Epi::QKV) {
    *kind = EK_QKV;
    return true;
  }
  if (k == Epi::NONE) {
    *kind = EK_NONE;
    return true;
  }
  if (k == Epi::STAGE_ONLY || k == Epi::F32_DIRECT) return false;
  const bool f32 = k == EK_F32 || k == EK_RESID || k == EK_PARTIAL;
  void* ptr = partial ? static_cast<void*>(partial) : e.out;
  const int64_t cols = k == EK_SWIGLU ? N / 2 : N;
  const int64_t ld = partial ? N : e.ldo;
  const int64_t esz = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16 || cols <= 0) return false;
  if (k == EK_SWIGLU && (N & 1)) return false;
  cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(M), cuuint64_t(std::max(splits, 1))};
  cuuint64_t strides[2] = {cuuint64_t(ld * esz), cuuint64_t(ld * esz * M)};
  cuuint32_t box[3] = {cuuint32_t(128 / esz), 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const int rank = k == EK_PARTIAL ? 3 : 2;
  CUresult r = tmap_encode_cached(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           rank, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  *kind = k;
  return true;
}

constexpr size_t kEpiSmem = 4 * 2 * 4096;  // staging tiles of the 4 epilogue warps

template <int BN, int STAGES, int KIND>
void run_tc(const GemmPlan& gp, cudaStream_t s, const CUtensorMap& ta, const CUtensorMap& tb,
            const CUtensorMap& tcm, int64_t M, int64_t N, int64_t K, const Epi& e, float* partial, float* xw) {
  const size_t smem = 1024 + size_t(STAGES) * (128 * 64 * 2 + BN * 64 * 2) + kEpiSmem +
                      8 * (2 * STAGES + 4) + 16;
  auto kern = k_gemm_tc<BN, STAGES, KIND>;
  static bool attr = false;
  if (!attr) {
    KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int mt = int((M + 127) / 128), nt = int((N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gp.grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (gp.cs > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = unsigned(gp.cs);
    at[na].val.clusterDim.y = 1;
    at[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = unsigned(na);
  KB_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, int(M), int(N), int(K), mt, nt, gp.splits, gp.kb_per, e,
                             partial, gp.grid, gp.sk_T, gp.cs, xw));
  KB_LAUNCH();
}

template <int BN, int STAGES>
int max_clusters_of(int cs) {
  const size_t smem = 1024 + size_t(STAGES) * (128 * 64 * 2 + BN * 64 * 2) + kEpiSmem +
                      8 * (2 * STAGES + 4) + 16;
  auto kern = k_gemm_tc<BN, STAGES, EK_F32>;
  KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(cs));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}
int max_clusters(int bn, int cs) {
  static std::mutex mu;
  static std::unordered_map<int, int> memo;
  std::lock_guard<std::mutex> lk(mu);
  const int key = bn * 16 + cs;
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  const int n = bn == 256 ? max_clusters_of<256, 4>(cs) : max_clusters_of<128, 6>(cs);
  memo[key] = n;
  return n;
}

template <int STAGES, int KSUB, int KIND>
void run_tc2(const GemmPlan& gp, cudaStream_t s, const CUtensorMap& ta, const CUtensorMap& tb,
             const CUtensorMap& tcm, int64_t M, int64_t N, int64_t K, const Epi& e, float* partial, float*) {
  const size_t smem = 1024 + size_t(STAGES) * KSUB * (2 * 128 * 64 * 2) + kEpiSmem +
                      8 * (2 * STAGES + 4) + 16;
  auto kern = k_gemm_tc2<STAGES, KSUB, KIND>;
  static bool attr = false;
  if (!attr) {
    KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int mt = int((M + 255) / 256), nt = int((N + 255) / 256);
  const int kb_per = (gp.kb_per + KSUB - 1) / KSUB;
  kern<<<gp.grid, 192, smem, s>>>(ta, tb, tcm, int(M), int(N), int(K), mt, nt, gp.splits, kb_per, e,
                                  partial);
  KB_LAUNCH();
}

#define KB_EPI_DISPATCH(FN, ...)                                   \
  switch (kind) {                                                  \
    case EK_F32: FN<__VA_ARGS__, EK_F32>(ARGS); break;             \
    case EK_CDT: FN<__VA_ARGS__, EK_CDT>(ARGS); break;             \
    case EK_RESID: FN<__VA_ARGS__, EK_RESID>(ARGS); break;         \
    case EK_TANH: FN<__VA_ARGS__, EK_TANH>(ARGS); break;           \
    case EK_SWIGLU: FN<__VA_ARGS__, EK_SWIGLU>(ARGS); break;       \
    case EK_NONE: FN<__VA_ARGS__, EK_NONE>(ARGS); break;           \
    case EK_PARTIAL: FN<__VA_ARGS__, EK_PARTIAL>(ARGS); break;     \
    case EK_QKV: FN<__VA_ARGS__, EK_QKV>(ARGS); break;             \
    default: FN<__VA_ARGS__, EK_GENERIC>(ARGS); break;             \
  }

void launch_gemm_tc(const GemmPlan& gp, cudaStream_t s, int64_t M, int64_t N, int64_t K,
                    const void* A, int64_t lda, const void* B, int64_t ldb, const Epi& e,
                    float* partial, float* xw) {
  const int64_t a_rows = gp.pair ? M : std::max<int64_t>(M, std::min<int64_t>(e.a_rows, 128));
  const CUtensorMap ta = make_map(A, a_rows, K, lda, 128);
  const CUtensorMap tb = make_map(B, N, K, ldb, gp.pair ? 128 : gp.bn);
  CUtensorMap tcm;
  int kind = EK_GENERIC;
  if (!make_out_map(&tcm, e, M, N, gp.splits, partial, &kind)) kind = EK_GENERIC;
#define ARGS gp, s, ta, tb, tcm, M, N, K, e, partial, xw
  if (gp.pair && g_gemm_force == 4) {
    KB_EPI_DISPATCH(run_tc2, 3, 2)
  } else if (gp.pair) {
    KB_EPI_DISPATCH(run_tc2, 6, 1)
  } else if (gp.bn == 256) {
    KB_EPI_DISPATCH(run_tc, 256, 4)
  } else {
    KB_EPI_DISPATCH(run_tc, 128, 6)
  }
#undef ARGS
}

int gemm_mode() {  // 0 auto, 1 force SIMT
  static int m = [] {
    const char* v = std::getenv("KRUL_GEMM");
    return (v && std::strcmp(v, "simt") == 0) ? 1 : 0;
  }();
  return m;
}
}  // namespace

void gemm_set_timeline(unsigned long long* d) { KB_CUDA(cudaMemcpyToSymbol(g_gemm_ts, &d, sizeof d)); }

bool gemm_uses_tc(const Ctx& c, const void* A, int64_t lda, const void* B, int64_t ldb) {
  return c.cfg.dtype == KRUL_BF16 && gemm_mode() == 0 && lda % 8 == 0 && ldb % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

void gemm_impl(const Ctx& c, cudaStream_t s, int64_t M, int64_t N, int64_t K, const void* A,
               int64_t lda, const void* B, int64_t ldb, const Epi& e);

void gemm(const Ctx& c, cudaStream_t s, int64_t M, int64_t N, int64_t K, const void* A,
          int64_t lda, const void* B, int64_t ldb, const Epi& e) {
  if (M <= 0 || N <= 0) return;
  cudaEvent_t kt0 = kt_begin(c, s);
  // M <= 128: a weight-streaming GEMM (HBM-bound: algorithmic bytes = weights
  // + activations in + out); larger M: tensor-bound (2MNK flops)
  const double bytes = double(N) * K * c.esz + double(M) * K * c.esz + double(M) * N * 4.0;
  if (c.span_on && M <= 128 && c.span_next < Ctx::kSpanSlots) {
    Epi es = e;
    es.span = const_cast<Ctx&>(c).span_next++;
    const_cast<Ctx&>(c).span_bytes.push_back(bytes);
    gemm_impl(c, s, M, N, K, A, lda, B, ldb, es);
  } else {
    gemm_impl(c, s, M, N, K, A, lda, B, ldb, e);
  }
  kt_end(c, s, kt0, M <= 128 ? KT_GEMM_STREAM : KT_GEMM, 2.0 * double(M) * double(N) * double(K), bytes);
}

void gemm_impl(const Ctx& c, cudaStream_t s, int64_t M, int64_t N, int64_t K, const void* A,
               int64_t lda, const void* B, int64_t ldb, const Epi& e) {
  const bool tc_ok = gemm_uses_tc(c, A, lda, B, ldb) && K >= 1;
  if (e.kind == Epi::QKV && !tc_ok) fail(KRUL_E_CUDA, "fused QKV epilogue requires the tcgen05 path");
  if (tc_ok) {
    // SM budget per stream (experiment knob KRUL_NEW_SMS: the new-input
    // prefill stream's persistent GEMMs use that many SMs, the recompute
    // stream's the rest, so the two never wait for each other's CTAs)
    static const int new_sms = [] {
      const char* v = std::getenv("KRUL_NEW_SMS");
      return v ? std::atoi(v) : 0;
    }();
    int sms = c.sm_count > 0 ? c.sm_count : 148;
    if (new_sms > 0 && new_sms < sms) sms = (s == c.s_new) ? new_sms : sms - new_sms;
    // the SwiGLU epilogue packs 128 accumulator columns per store: not split
    // over a cluster's ranks
    const GemmPlan gp = plan_gemm(M, N, K, sms, true, e.kind != Epi::SWIGLU && new_sms == 0);
    float* part = nullptr;
    float* xw = nullptr;
    if (gp.splits > 1 || gp.sk_T > 0) {
      DevBuf& buf = s == c.s_new ? c.ws2_gpart : c.ws_gpart;
      part = static_cast<float*>(buf.ensure(size_t(M) * size_t(N) * gp.splits * 4));
    } else if (gp.cs > 1) {  // cluster split-K exchange: [tile][chunk][rank][128 rows][32 cols]
      DevBuf& buf = s == c.s_new ? c.ws2_gpart : c.ws_gpart;
      const int64_t nt = (N + gp.bn - 1) / gp.bn;
      xw = static_cast<float*>(buf.ensure(size_t(nt) * (gp.bn / 32) * gp.cs * 4096 * 4));
    }
    launch_gemm_tc(gp, s, M, N, K, A, lda, B, ldb, e, part, xw);
    SkInfo sk;
    if (gp.sk_T > 0) {
      sk.G = gp.grid;
      sk.T = gp.sk_T;
      sk.num_k = int((K + 63) / 64);
      sk.bn = gp.bn;
    }
    if (part && e.kind == Epi::QKV) {
      if (c.cfg.hd % 32) fail(KRUL_E_CUDA, "fused QKV epilogue needs head_dim % 32 == 0");
      const dim3 g2{unsigned((M + 31) / 32), unsigned((N + 31) / 32), 1u};
      KB_CUDA(launch_pdl(k_qkv_reduce, g2, dim3(256), 0, s, (const float*)part, gp.splits, M, N, e.kv, sk));
      KB_LAUNCH();
    } else if (part) {
      const int64_t work = (N % 4 == 0) ? M * N / 4 : (e.kind == Epi::SWIGLU ? M * N / 2 : M * N);
      const unsigned blocks = unsigned(std::min<int64_t>((work + 255) / 256, 8 * 148));
      KB_CUDA(launch_pdl(k_splitk_reduce<bf16>, dim3(blocks), dim3(256), 0, s, (const float*)part, gp.splits, M,
                         N, e, sk));
      KB_LAUNCH();
    }
    return;
  }
  dim3 grid(unsigned((N + 63) / 64), unsigned((M + 63) / 64));
  if (c.cfg.dtype == KRUL_BF16)
    k_gemm_simt<bf16><<<grid, 256, 0, s>>>(M, N, K, (const bf16*)A, lda, (const bf16*)B, ldb, e);
  else
    k_gemm_simt<float><<<grid, 256, 0, s>>>(M, N, K, (const float*)A, lda, (const float*)B, ldb,
                                            e);
  KB_LAUNCH();
}

}  // namespace kb
