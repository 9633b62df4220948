// attn_tc.cu — causal prefill attention on tcgen05 / TMEM over the paged KV
// cache (K6 recompute and K7 new-input prefill; engine.cpp:174-188).
//
// See k_attn_fa for the warp roles. Online softmax runs in the log2 domain;
// the classifier region mass (analysis.cpp:46-54) is accumulated alongside
// the row sum and rescaled with it. Split-KV partials are merged by
// k_attn_combine.
#include <cuda.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {
CUresult tmap_encode_cached(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr,
                            const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                            const cuuint32_t* es, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                            CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob);
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
  // non-blocking probe loop: the handoffs of this pipeline are short and a
  // suspended try_wait adds its wake-up latency to every one of them
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
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
// issue-only variants: several TMEM transfers in flight, one wait
__device__ __forceinline__ void ld32_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TCA_REGS32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st32_async(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TCA_IN32(r)
      : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TCA_IN32(r)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2, ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

}  // namespace tca
using tca::pack2;
using tca::ex2_approx;
using tca::imax64;
using tca::imin64;

struct AttnTc {
  int H, Hkv, grp, hpc;          // hpc: query heads per CTA (2 = a GQA pair sharing one KV head)
  int64_t rows, pos0, kv_total;  // keys [0, kv_total) exist; causal limit per row
  int n_qtiles, target;          // q tiles of 128 rows; key blocks (128) per work item
  float scale_log2;
  const int* pt;
  int max_pages;
  int k_rows_pp;   // K-view rows per page
  int v_rows_pp;   // V-view rows per page
  bf16* out;       // [rows][H*HD]
  float* part;     // [slot][h][HD + 3][rows] (o..., m, l, mass) for split q tiles
  double* mass;    // [H][rows] region mass, may be null
  float* stats;    // [H][rows][2] (m, l) in the log2 domain, may be null
  int64_t il, rs;
};

constexpr int kAttnKB = 128;  // keys per block = two 64-token pages
constexpr int kPgCache = 96;  // key blocks whose page ids are cached in smem

// number of key blocks q tile qt attends to, and its work-item count
__host__ __device__ __forceinline__ int attn_nblk(const AttnTc& p, int qt) {
  const int64_t q_end = min(int64_t(qt) * 128 + 128, p.rows);
  const int64_t hi = min(p.pos0 + q_end, p.kv_total);
  return int((hi + kAttnKB - 1) / kAttnKB);
}
__host__ __device__ __forceinline__ int attn_nsplit(const AttnTc& p, int qt) {
  return (attn_nblk(p, qt) + p.target - 1) / p.target;
}

namespace tca {
// A operand from TMEM (P), B from shared memory (V^T): the "TS" form
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// Warp-converged issue: all 32 lanes of the MMA warp run the issue loop (so
// descriptors and TMEM addresses stay in uniform registers) and elect.sync
// picks the one lane that issues -- the single-lane form compiled to an
// elect/broadcast loop per MMA whose issue cost (on a sub-partition shared
// with two busy softmax warps) exceeded the MMA's own execution time.
__device__ __forceinline__ void mma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_e(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(b))
      : "memory");
}
// suspending wait for the long waits of the producer / MMA warps (a probe
// loop there takes issue slots from the softmax warps of its sub-partition)
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
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
}  // namespace tca

// Debug timeline (krul_debug_attn_timeline): %globaltimer stamps per CTA,
// [cta][8] = entry, prologue done, Q in (MMA), MMA loop done, softmax done,
// epilogue done, exit; then a clock64 trace of CTA (0, 0) per key block:
// role (0/1 softmax A/B, 2 MMA) x block (< 64) x 4 events.
__device__ unsigned long long* g_attn_ts = nullptr;
__device__ __forceinline__ void attn_ts(int slot) {
  if (g_attn_ts) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_ts[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + slot] = t;
  }
}
__device__ __forceinline__ void attn_tr(int role, int i, int ev) {
  if (g_attn_ts && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_attn_ts[32768 + (role * 64 + i) * 4 + ev] = clock64();
}

// Causal flash attention over the paged KV cache, FA4-style on tcgen05.
// One CTA = one work item (q tile of 128 rows, key-block range) for up to
// two query heads; with GQA the two heads read the same KV head, so every
// K/V page is staged once for both. Key block = 128 keys = two 64-token
// pages (K [128][hd], V^T [hd][128], TMA SW128, 2-stage ring).
//   warps 0-3 / 4-7 : softmax of head A / B; thread = query row = TMEM lane.
//     S (128 fp32 columns) is read once into registers, the probabilities
//     are written back as bf16 into the first 64 columns of the same TMEM
//     region (P never touches shared memory), lazy O rescale (the running
//     max moves only when a row max exceeds it by > 8 in log2), MUFU ex2.
//   warp 8 : K TMA producer, warp 10 : V TMA producer.
//   warp 9 : MMA issuer, ping-pong over the heads: PV_A(i) (TS-MMA, A = P
//     from TMEM) then S_A(i+1) while head B is exponentiated, then PV_B(i),
//     S_B(i+1) while head A is -- the tensor pipe and the softmax warps
//     overlap across the two heads.
// TMEM (512 columns): S/P_A [0,128), S/P_B [128,256), O_A [256,..), O_B [384,..).
template <int HD>
__global__ void __launch_bounds__(352, 1)
    k_attn_fa(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnTc p) {
  constexpr int KB = kAttnKB;
  constexpr int NSUB = HD / 64;                 // 64-wide hd sub-tiles
  constexpr uint32_t Q_BYTES = 128 * HD * 2;    // per head
  constexpr uint32_t K_BYTES = KB * HD * 2;     // [NSUB][128 keys][128 B]
  constexpr uint32_t V_BYTES = HD * KB * 2;     // [2 key halves][HD rows][128 B]
  constexpr int KST = 3, VST = 2;  // separate K and V rings: K frees after S, V after PV
  extern __shared__ unsigned char smraw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;                        // [2][Q_BYTES]
  unsigned char* sK = sQ + 2 * Q_BYTES;            // [KST][K_BYTES]
  unsigned char* sV = sK + KST * K_BYTES;          // [VST][V_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * V_BYTES);
  uint64_t* q_full = bars;                  // 1
  uint64_t* k_full = bars + 1;              // KST
  uint64_t* k_empty = k_full + KST;         // KST
  uint64_t* v_full = k_empty + KST;         // VST
  uint64_t* v_empty = v_full + VST;         // VST
  uint64_t* s_full = v_empty + VST;         // [2 heads]
  uint64_t* p_ready = s_full + 2;           // [2 heads]
  uint64_t* pv_done = p_ready + 2;          // [2 heads]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(pv_done + 2);
  int* pg_s = reinterpret_cast<int*>(tslot + 4);  // [2 * kPgCache] page ids of this item

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) attn_ts(0);
  // work item -> (q tile, split); heavy (late) q tiles first
  int qt = p.n_qtiles - 1, split = int(blockIdx.x);
  for (; qt > 0; --qt) {
    const int ns = attn_nsplit(p, qt);
    if (split < ns) break;
    split -= ns;
  }
  const int nsplit = attn_nsplit(p, qt);
  const int nblk_all = attn_nblk(p, qt);
  const int b0 = split * p.target;
  const int b1 = min(nblk_all, b0 + p.target);
  const int nb = b1 - b0;
  const int hA = p.hpc * blockIdx.y, hB = hA + 1;
  const bool hasB = p.hpc == 2 && hB < p.H;
  const int g = hA / p.grp;
  const int64_t q0 = int64_t(qt) * 128;

  if (threadIdx.x == 0) {
    tca::bar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      tca::bar_init(&k_full[s], 1);
      tca::bar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      tca::bar_init(&v_full[s], 1);
      tca::bar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tca::bar_init(&s_full[i], 1);
      tca::bar_init(&p_ready[i], 128);
      tca::bar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        tca::su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // page ids of the item's key blocks, fetched once by all threads (a
  // dependent global load per block in the producer threads serialised the
  // K/V stream)
  for (int i = threadIdx.x; i < 2 * min(nb, kPgCache); i += blockDim.x)
    pg_s[i] = p.pt[min(2 * b0 + i, p.max_pages - 1)];
  tca::fence_before();
  __syncthreads();
  tca::fence_after();
  const uint32_t tmem = *tslot;
  pdl_trigger();
  pdl_wait();  // Q and this step's K / V rows come from the preceding kernels
  if (threadIdx.x == 0) attn_ts(1);
  auto page_of = [&](int i, int half) {
    return i < kPgCache ? pg_s[2 * i + half] : p.pt[min(2 * (b0 + i) + half, p.max_pages - 1)];
  };

  if (warp == 8) {
    if (lane == 0 && nb > 0) {  // TMA producer
      tca::bar_expect(q_full, (hasB ? 2 : 1) * Q_BYTES);
      for (int j = 0; j < NSUB; ++j) {
        tca::tma2d(sQ + j * (128 * 128), &tmQ, q_full, hA * HD + 64 * j, int(q0));
        if (hasB) tca::tma2d(sQ + Q_BYTES + j * (128 * 128), &tmQ, q_full, hB * HD + 64 * j, int(q0));
      }
      const int voff = p.Hkv * HD + g * HD;
      for (int i = 0; i < nb; ++i) {
        const int pa = page_of(i, 0), pb = page_of(i, 1);
        const int ks = i % KST;
        tca::bar_wait_sleep(&k_empty[ks], ((i / KST) & 1) ^ 1);
        unsigned char* kd = sK + ks * K_BYTES;
        tca::bar_expect(&k_full[ks], K_BYTES);
        for (int j = 0; j < NSUB; ++j) {
          tca::tma2d(kd + j * (KB * 128), &tmK, &k_full[ks], 64 * j, pa * p.k_rows_pp + g * 64);
          tca::tma2d(kd + j * (KB * 128) + 64 * 128, &tmK, &k_full[ks], 64 * j, pb * p.k_rows_pp + g * 64);
        }
      }
      (void)voff;
    }
  } else if (warp == 10) {
    // V producer: its own thread so a V slot still held by PV(i-2) never
    // holds back the K prefetch that the next QK^T waits for
    if (lane == 0 && nb > 0) {
      const int voff = p.Hkv * HD + g * HD;
      for (int i = 0; i < nb; ++i) {
        const int pa = page_of(i, 0), pb = page_of(i, 1);
        const int vs = i % VST;
        tca::bar_wait_sleep(&v_empty[vs], ((i / VST) & 1) ^ 1);
        unsigned char* vd = sV + vs * V_BYTES;
        tca::bar_expect(&v_full[vs], V_BYTES);
        tca::tma2d(vd, &tmV, &v_full[vs], 0, pa * p.v_rows_pp + voff);
        tca::tma2d(vd + HD * 128, &tmV, &v_full[vs], 0, pb * p.v_rows_pp + voff);
      }
    }
  } else if (warp == 9) {
    if (nb > 0) {  // MMA issuer: the whole warp, one elected lane issues
      constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KB >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      constexpr uint32_t idO = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(HD >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      const int nh = hasB ? 2 : 1;
      // descriptor of a tile + byte offset = descriptor + offset / 16 (the
      // 14-bit start-address field cannot carry inside shared memory)
      auto issue_s = [&](int h, int i) {  // S_h(i) = Q_h K_i^T -> TMEM [h*128, +128)
        const uint64_t dq = tca::desc(sQ + h * Q_BYTES), dk = tca::desc(sK + (i % KST) * K_BYTES);
        const uint32_t dS = tmem + uint32_t(h * 128);
#pragma unroll
        for (int j = 0; j < NSUB; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tca::mma_ss_e(dS, dq + uint64_t((j * (128 * 128) + k * 32) >> 4),
                          dk + uint64_t((j * (KB * 128) + k * 32) >> 4), idS, (j | k) != 0);
        tca::commit_e(&s_full[h]);
      };
      auto issue_pv = [&](int h, int i) {  // O_h += P_h(i) V_i, P from TMEM
        const uint64_t dv = tca::desc(sV + (i % VST) * V_BYTES);
        const uint32_t dO = tmem + 256 + uint32_t(h * 128);
        const uint32_t aP = tmem + uint32_t(h * 128);
#pragma unroll
        for (int k = 0; k < KB / 16; ++k)
          tca::mma_ts_e(dO, aP + uint32_t(k * 8), dv + uint64_t(((k >> 2) * (HD * 128) + (k & 3) * 32) >> 4),
                        idO, (i | k) != 0);
        tca::commit_e(&pv_done[h]);
      };
      tca::bar_wait_sleep(q_full, 0);
      attn_ts(2);
      tca::bar_wait_sleep(&k_full[0], 0);
      tca::fence_after();
      for (int h = 0; h < nh; ++h) issue_s(h, 0);
      tca::commit_e(&k_empty[0]);
      for (int i = 0; i < nb; ++i) {
        for (int h = 0; h < nh; ++h) {
          tca::bar_wait_sleep(&p_ready[h], i & 1);
          if (h == 0) tca::bar_wait_sleep(&v_full[i % VST], (i / VST) & 1);
          tca::fence_after();
          if (h == 0) attn_tr(2, i, 0);
          issue_pv(h, i);
          if (i + 1 < nb) {
            if (h == 0) tca::bar_wait_sleep(&k_full[(i + 1) % KST], ((i + 1) / KST) & 1);
            // P_h(i) lives in S_h's TMEM columns: S_h(i+1) is issued once
            // PV_h(i) has consumed them
            tca::bar_wait_sleep(&pv_done[h], i & 1);
            tca::fence_after();
            issue_s(h, i + 1);
          }
          if (h == 0) attn_tr(2, i, 1);
        }
        attn_tr(2, i, 2);
        tca::commit_e(&v_empty[i % VST]);                      // after PV_A(i), PV_B(i)
        if (i + 1 < nb) tca::commit_e(&k_empty[(i + 1) % KST]);  // after S_A(i+1), S_B(i+1)
      }
      attn_ts(3);
    }
  } else {  // softmax warp groups
    const int wg = warp >> 2;  // 0 = head A, 1 = head B
    const int h = wg == 0 ? hA : hB;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int64_t qpos = p.pos0 + q0 + r;
    const uint32_t tS = tmem + uint32_t(wg * 128) + lane_off;
    const uint32_t tO = tmem + 256 + uint32_t(wg * 128) + lane_off;
    float m = -INFINITY, l = 0.f, mn = 0.f;
    const bool active = wg == 0 || hasB;
    if (active) {
      for (int i = 0; i < nb; ++i) {
        const int64_t k0 = int64_t(b0 + i) * KB;
        const bool tr = (threadIdx.x & 127) == 0;
        if (tr) attn_tr(wg, i, 0);
        tca::bar_wait(&s_full[wg], i & 1);
        tca::fence_after();
        if (tr) attn_tr(wg, i, 1);
        uint32_t v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tca::ld32_async(tS + uint32_t(c * 32), v + 32 * c);
        tca::ld_wait();
        if (tr) attn_tr(wg, i, 2);
        // visible keys of this row in the block: [k0, k0 + nv); the raw
        // scores are masked only on edge blocks (causal diagonal, sequence end)
        const int nv = int(imax64(0, imin64(KB, min(qpos + 1, p.kv_total) - k0)));
        if (__any_sync(0xffffffffu, nv < KB)) {
#pragma unroll
          for (int t = 0; t < 128; ++t) v[t] = t < nv ? v[t] : __float_as_uint(-INFINITY);
        }
        float mx;
        {  // tree max
          float t64[64];
#pragma unroll
          for (int t = 0; t < 64; ++t) t64[t] = fmaxf(__uint_as_float(v[t]), __uint_as_float(v[t + 64]));
#pragma unroll
          for (int w = 32; w >= 1; w >>= 1)
#pragma unroll
            for (int t = 0; t < w; ++t) t64[t] = fmaxf(t64[t], t64[t + w]);
          mx = t64[0] * p.scale_log2;  // the log2-domain scale is positive: applied to the max
        }
        // lazy max: move only when the block max exceeds it by > 8 (log2)
        float m_new = m;
        if (mx > m + 8.f || m == -INFINITY) m_new = fmaxf(mx, m);
        const float alpha = (m == -INFINITY || m_new == m) ? 1.f : ex2_approx(m - m_new);
        // O rescale: PV(i-1) has completed (S(i) was issued after it)
        if (i > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          uint32_t o[32];
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            tca::ld32(tO + uint32_t(c * 32), o);
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
            tca::st32_async(tO + uint32_t(c * 32), o);
          }
          tca::st_wait();
        }
        const float mb = m_new == -INFINITY ? 0.f : m_new;  // all-masked rows: exp2(-inf) = 0
        const bool do_mass = p.mass != nullptr;
        const int ie = do_mass ? int(imax64(0, imin64(KB, p.il - k0))) : 0;
        const int rb = do_mass ? int(imax64(0, imin64(KB, p.rs - k0))) : KB;
        float sum = 0.f, msum = 0.f;
        // exponentiate and pack in place: v[j] <- bf16x2(p(2j), p(2j+1))
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          const float e0 = ex2_approx(fmaf(__uint_as_float(v[2 * j]), p.scale_log2, -mb));
          const float e1 = ex2_approx(fmaf(__uint_as_float(v[2 * j + 1]), p.scale_log2, -mb));
          sum += e0 + e1;
          if (do_mass) {
            if (2 * j < ie || 2 * j >= rb) msum += e0;
            if (2 * j + 1 < ie || 2 * j + 1 >= rb) msum += e1;
          }
          v[j] = pack2(e0, e1);
        }
        tca::st32_async(tS, v);
        tca::st32_async(tS + 32u, v + 32);
        tca::st_wait();
        if (tr) attn_tr(wg, i, 3);
        l = l * alpha + sum;
        mn = mn * alpha + msum;
        m = m_new;
        tca::fence_before();
        tca::bar_arrive(&p_ready[wg]);
      }
      if (nb > 0) {
        tca::bar_wait(&pv_done[wg], (nb - 1) & 1);
        tca::fence_after();
      }
      if (threadIdx.x == 0) attn_ts(4);
      const int64_t row = q0 + r;
      const bool valid = row < p.rows;
      uint32_t o[32];
      if (nsplit == 1) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* dst = p.out + (row * p.H + h) * HD;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          tca::ld32(tO + uint32_t(c * 32), o);
          if (!valid) continue;
#pragma unroll
          for (int t = 0; t < 32; t += 8) {
            uint4 w;
            w.x = pack2(__uint_as_float(o[t]) * inv, __uint_as_float(o[t + 1]) * inv);
            w.y = pack2(__uint_as_float(o[t + 2]) * inv, __uint_as_float(o[t + 3]) * inv);
            w.z = pack2(__uint_as_float(o[t + 4]) * inv, __uint_as_float(o[t + 5]) * inv);
            w.w = pack2(__uint_as_float(o[t + 6]) * inv, __uint_as_float(o[t + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + t) = w;
          }
        }
        if (valid && p.mass) p.mass[int64_t(h) * p.rows + row] = l > 0.f ? double(mn) / double(l) : 0.0;
        if (valid && p.stats) {
          p.stats[(int64_t(h) * p.rows + row) * 2] = m;
          p.stats[(int64_t(h) * p.rows + row) * 2 + 1] = l;
        }
      } else {
        // [slot][h][HD + 3][rows]: for each column the warp's 32 rows are
        // contiguous, so every store below is one coalesced 128-byte access
        float* dst = p.part + (int64_t(split) * p.H + h) * (HD + 3) * p.rows + row;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          if (nb > 0) tca::ld32(tO + uint32_t(c * 32), o);
          if (!valid) continue;
#pragma unroll
          for (int t = 0; t < 32; ++t) dst[int64_t(c * 32 + t) * p.rows] = nb > 0 ? __uint_as_float(o[t]) : 0.f;
        }
        if (valid) {
          dst[int64_t(HD) * p.rows] = m;
          dst[int64_t(HD + 1) * p.rows] = l;
          dst[int64_t(HD + 2) * p.rows] = mn;
        }
      }
    }
  }
  __syncwarp();
  if (threadIdx.x == 0) attn_ts(5);
  tca::fence_before();
  __syncthreads();
  if (warp == 9) {
    tca::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) attn_ts(6);
}

// One head per CTA (k_attn_fa1): S double-buffered in TMEM (S0, S1, O =
// 384 columns) so QK^T of block i+1 runs while block i is exponentiated and
// the per-head PV(i) -> S(i+1) chain no longer serialises the softmax; two
// softmax warps per TMEM lane quadrant split each 128-key block into column
// halves (row max / sums exchanged through shared memory), so one block's
// exponentials spread over 8 warps. Warp 8: TMA producers (lane 0 Q + K,
// lane 1 V), warp 9: MMA issuer (warp-converged). P goes back over S's own
// columns [0, 64) of its buffer; PV is a TS-MMA. Each K/V page is staged per
// head (twice the shared-memory fill of the head-pair kernel).
template <int HD>
__global__ void __launch_bounds__(320, 1)
    k_attn_fa1(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, AttnTc p) {
  constexpr int KB = kAttnKB;
  constexpr int NSUB = HD / 64;
  constexpr uint32_t Q_BYTES = 128 * HD * 2;
  constexpr uint32_t K_BYTES = KB * HD * 2;
  constexpr uint32_t V_BYTES = HD * KB * 2;
  constexpr int KST = 3, VST = 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = base;
  unsigned char* sK = sQ + Q_BYTES;
  unsigned char* sV = sK + KST * K_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * V_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;   // [buffer]
  uint64_t* p_ready = s_full + 2;     // [buffer]
  uint64_t* pv_done = p_ready + 2;    // [buffer]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(pv_done + 2);
  int* pg_s = reinterpret_cast<int*>(tslot + 4);              // [2 * kPgCache]
  float* xs = reinterpret_cast<float*>(pg_s + 2 * kPgCache);  // [block parity][half][128 rows][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) attn_ts(0);
  int qt = p.n_qtiles - 1, split = int(blockIdx.x);
  for (; qt > 0; --qt) {
    const int ns = attn_nsplit(p, qt);
    if (split < ns) break;
    split -= ns;
  }
  const int nsplit = attn_nsplit(p, qt);
  const int nblk_all = attn_nblk(p, qt);
  const int b0 = split * p.target;
  const int b1 = min(nblk_all, b0 + p.target);
  const int nb = b1 - b0;
  const int h = int(blockIdx.y);
  const int g = h / p.grp;
  const int64_t q0 = int64_t(qt) * 128;

  if (threadIdx.x == 0) {
    tca::bar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      tca::bar_init(&k_full[s], 1);
      tca::bar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      tca::bar_init(&v_full[s], 1);
      tca::bar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tca::bar_init(&s_full[i], 1);
      tca::bar_init(&p_ready[i], 256);
      tca::bar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        tca::su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 2 * min(nb, kPgCache); i += blockDim.x)
    pg_s[i] = p.pt[min(2 * b0 + i, p.max_pages - 1)];
  tca::fence_before();
  __syncthreads();
  tca::fence_after();
  const uint32_t tmem = *tslot;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) attn_ts(1);
  auto page_of = [&](int i, int half) {
    return i < kPgCache ? pg_s[2 * i + half] : p.pt[min(2 * (b0 + i) + half, p.max_pages - 1)];
  };

  if (warp == 8 && lane == 0) {
    if (nb > 0) {  // Q + K producer
      tca::bar_expect(q_full, Q_BYTES);
      for (int j = 0; j < NSUB; ++j) tca::tma2d(sQ + j * (128 * 128), &tmQ, q_full, h * HD + 64 * j, int(q0));
      for (int i = 0; i < nb; ++i) {
        const int pa = page_of(i, 0), pb = page_of(i, 1);
        const int ks = i % KST;
        tca::bar_wait_sleep(&k_empty[ks], ((i / KST) & 1) ^ 1);
        unsigned char* kd = sK + ks * K_BYTES;
        tca::bar_expect(&k_full[ks], K_BYTES);
        for (int j = 0; j < NSUB; ++j) {
          tca::tma2d(kd + j * (KB * 128), &tmK, &k_full[ks], 64 * j, pa * p.k_rows_pp + g * 64);
          tca::tma2d(kd + j * (KB * 128) + 64 * 128, &tmK, &k_full[ks], 64 * j, pb * p.k_rows_pp + g * 64);
        }
      }
    }
  } else if (warp == 8 && lane == 1) {
    if (nb > 0) {  // V producer
      const int voff = p.Hkv * HD + g * HD;
      for (int i = 0; i < nb; ++i) {
        const int pa = page_of(i, 0), pb = page_of(i, 1);
        const int vs = i % VST;
        tca::bar_wait_sleep(&v_empty[vs], ((i / VST) & 1) ^ 1);
        unsigned char* vd = sV + vs * V_BYTES;
        tca::bar_expect(&v_full[vs], V_BYTES);
        tca::tma2d(vd, &tmV, &v_full[vs], 0, pa * p.v_rows_pp + voff);
        tca::tma2d(vd + HD * 128, &tmV, &v_full[vs], 0, pb * p.v_rows_pp + voff);
      }
    }
  } else if (warp == 9) {
    if (nb > 0) {  // MMA issuer: the whole warp, one elected lane issues
      constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KB >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      constexpr uint32_t idO = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(HD >> 3) << 17) |
                               (uint32_t(128 >> 4) << 24);
      const uint64_t dq = tca::desc(sQ);
      auto issue_s = [&](int i) {  // S(i) -> TMEM buffer i % 2
        tca::bar_wait_sleep(&k_full[i % KST], (i / KST) & 1);
        tca::fence_after();
        const uint64_t dk = tca::desc(sK + (i % KST) * K_BYTES);
        const uint32_t dS = tmem + uint32_t((i & 1) * 128);
#pragma unroll
        for (int j = 0; j < NSUB; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tca::mma_ss_e(dS, dq + uint64_t((j * (128 * 128) + k * 32) >> 4),
                          dk + uint64_t((j * (KB * 128) + k * 32) >> 4), idS, (j | k) != 0);
        tca::commit_e(&s_full[i & 1]);
        tca::commit_e(&k_empty[i % KST]);
      };
      tca::bar_wait_sleep(q_full, 0);
      attn_ts(2);
      issue_s(0);
      if (nb > 1) issue_s(1);
      for (int i = 0; i < nb; ++i) {
        const int b = i & 1;
        tca::bar_wait_sleep(&p_ready[b], (i >> 1) & 1);
        tca::bar_wait_sleep(&v_full[i % VST], (i / VST) & 1);
        tca::fence_after();
        attn_tr(2, i, 0);
        const uint64_t dv = tca::desc(sV + (i % VST) * V_BYTES);
        const uint32_t dO = tmem + 256;
        const uint32_t aP = tmem + uint32_t(b * 128);
#pragma unroll
        for (int k = 0; k < KB / 16; ++k)
          tca::mma_ts_e(dO, aP + uint32_t(k * 8), dv + uint64_t(((k >> 2) * (HD * 128) + (k & 3) * 32) >> 4),
                        idO, (i | k) != 0);
        tca::commit_e(&pv_done[b]);
        tca::commit_e(&v_empty[i % VST]);
        if (i + 2 < nb) {  // buffer b holds P(i) until PV(i) has read it
          tca::bar_wait_sleep(&pv_done[b], (i >> 1) & 1);
          tca::fence_after();
          issue_s(i + 2);
        }
        attn_tr(2, i, 1);
      }
      attn_ts(3);
    }
  } else if (warp < 8) {  // softmax: two warps per TMEM lane quadrant, one per 64-column half
    const int hf = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int64_t qpos = p.pos0 + q0 + r;
    const uint32_t tO = tmem + 256 + uint32_t(hf * (HD / 2)) + lane_off;
    // row exchange slots, alternating with the block parity: with S double
    // buffered a half may reach block i+1 before its partner has read the
    // block-i slot, but not block i+2 (that needs the partner's arrival at
    // block i+1's barrier)
    auto xrow = [&](int i) { return xs + (((i & 1) * 2 + hf) * 128 + r) * 2; };
    auto xpart = [&](int i) { return xs + (((i & 1) * 2 + (hf ^ 1)) * 128 + r) * 2; };
    float m = -INFINITY, l = 0.f, mn = 0.f;
    for (int i = 0; i < nb; ++i) {
      const int b = i & 1;
      const uint32_t tS = tmem + uint32_t(b * 128) + lane_off;
      const int64_t k0 = int64_t(b0 + i) * KB + hf * 64;
      const bool tr = (warp & 3) == 0 && lane == 0;
      if (tr) attn_tr(hf, i, 0);
      tca::bar_wait(&s_full[b], (i >> 1) & 1);
      tca::fence_after();
      if (tr) attn_tr(hf, i, 1);
      uint32_t v[64];
      tca::ld32_async(tS + uint32_t(hf * 64), v);
      tca::ld32_async(tS + uint32_t(hf * 64 + 32), v + 32);
      tca::ld_wait();
      if (tr) attn_tr(hf, i, 2);
      const int nv = int(imax64(0, imin64(64, min(qpos + 1, p.kv_total) - k0)));
      if (__any_sync(0xffffffffu, nv < 64)) {
#pragma unroll
        for (int t = 0; t < 64; ++t) v[t] = t < nv ? v[t] : __float_as_uint(-INFINITY);
      }
      float mx;
      {
        float a8[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) a8[t] = __uint_as_float(v[t]);
#pragma unroll
        for (int t = 8; t < 64; ++t) a8[t & 7] = fmaxf(a8[t & 7], __uint_as_float(v[t]));
        mx = fmaxf(fmaxf(fmaxf(a8[0], a8[1]), fmaxf(a8[2], a8[3])), fmaxf(fmaxf(a8[4], a8[5]), fmaxf(a8[6], a8[7])));
      }
      // row max over both halves
      xrow(i)[0] = mx;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mx = fmaxf(mx, xpart(i)[0]) * p.scale_log2;
      float m_new = m;
      if (mx > m + 8.f || m == -INFINITY) m_new = fmaxf(mx, m);
      const float alpha = (m == -INFINITY || m_new == m) ? 1.f : ex2_approx(m - m_new);
      if (i > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // O (this half's columns) once PV(i-1) has landed
        tca::bar_wait(&pv_done[b ^ 1], ((i - 1) >> 1) & 1);
        tca::fence_after();
        uint32_t o[32];
#pragma unroll 1
        for (int c = 0; c < HD / 64; ++c) {
          tca::ld32(tO + uint32_t(c * 32), o);
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
          tca::st32_async(tO + uint32_t(c * 32), o);
        }
        tca::st_wait();
      }
      const float mb = m_new == -INFINITY ? 0.f : m_new;
      const bool do_mass = p.mass != nullptr;
      const int ie = do_mass ? int(imax64(0, imin64(64, p.il - k0))) : 0;
      const int rb = do_mass ? int(imax64(0, imin64(64, p.rs - k0))) : 64;
      float sum = 0.f, msum = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e0 = ex2_approx(fmaf(__uint_as_float(v[2 * j]), p.scale_log2, -mb));
        const float e1 = ex2_approx(fmaf(__uint_as_float(v[2 * j + 1]), p.scale_log2, -mb));
        sum += e0 + e1;
        if (do_mass) {
          if (2 * j < ie || 2 * j >= rb) msum += e0;
          if (2 * j + 1 < ie || 2 * j + 1 >= rb) msum += e1;
        }
        v[j] = pack2(e0, e1);
      }
      // P of this half's keys into columns [hf * 32, +32) of the buffer: both
      // halves have read their S columns (the barrier above)
      tca::st32_async(tS + uint32_t(hf * 32), v);
      tca::st_wait();
      if (tr) attn_tr(hf, i, 3);
      l = l * alpha + sum;
      mn = mn * alpha + msum;
      m = m_new;
      tca::fence_before();
      tca::bar_arrive(&p_ready[b]);
    }
    if (nb > 0) {
      tca::bar_wait(&pv_done[(nb - 1) & 1], ((nb - 1) >> 1) & 1);
      tca::fence_after();
    }
    xrow(nb)[0] = l;
    xrow(nb)[1] = mn;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    l += xpart(nb)[0];
    mn += xpart(nb)[1];
    if (threadIdx.x == 0) attn_ts(4);
    const int64_t row = q0 + r;
    const bool valid = row < p.rows;
    uint32_t o[32];
    if (nsplit == 1) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16* dst = p.out + (row * p.H + h) * HD + hf * (HD / 2);
#pragma unroll 1
      for (int c = 0; c < HD / 64; ++c) {
        tca::ld32(tO + uint32_t(c * 32), o);
        if (!valid) continue;
#pragma unroll
        for (int t = 0; t < 32; t += 8) {
          uint4 w;
          w.x = pack2(__uint_as_float(o[t]) * inv, __uint_as_float(o[t + 1]) * inv);
          w.y = pack2(__uint_as_float(o[t + 2]) * inv, __uint_as_float(o[t + 3]) * inv);
          w.z = pack2(__uint_as_float(o[t + 4]) * inv, __uint_as_float(o[t + 5]) * inv);
          w.w = pack2(__uint_as_float(o[t + 6]) * inv, __uint_as_float(o[t + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c * 32 + t) = w;
        }
      }
      if (valid && hf == 0 && p.mass) p.mass[int64_t(h) * p.rows + row] = l > 0.f ? double(mn) / double(l) : 0.0;
      if (valid && hf == 0 && p.stats) {
        p.stats[(int64_t(h) * p.rows + row) * 2] = m;
        p.stats[(int64_t(h) * p.rows + row) * 2 + 1] = l;
      }
    } else {
      float* dst = p.part + (int64_t(split) * p.H + h) * (HD + 3) * p.rows + row;
#pragma unroll 1
      for (int c = 0; c < HD / 64; ++c) {
        if (nb > 0) tca::ld32(tO + uint32_t(c * 32), o);
        if (!valid) continue;
        const int d0 = hf * (HD / 2) + c * 32;
#pragma unroll
        for (int t = 0; t < 32; ++t) dst[int64_t(d0 + t) * p.rows] = nb > 0 ? __uint_as_float(o[t]) : 0.f;
      }
      if (valid && hf == 0) {
        dst[int64_t(HD) * p.rows] = m;
        dst[int64_t(HD + 1) * p.rows] = l;
        dst[int64_t(HD + 2) * p.rows] = mn;
      }
    }
  }
  __syncwarp();
  if (threadIdx.x == 0) attn_ts(5);
  tca::fence_before();
  __syncthreads();
  if (warp == 9) {
    tca::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) attn_ts(6);
}

// Split-KV merge for rows of split q tiles: weights 2^(m_s - M) (log2
// domain); rows whose q tile ran as one item were written by the kernel.
// Block = (32 rows, head, 32-dim slice), 4 warps, lane = row, warp = 8 dims.
// Partials are [slot][h][HD + 3][rows], so every load is a coalesced
// 128-byte row segment; all split loads of a thread are issued up front
// (kMaxSplit unrolled, predicated) for memory-level parallelism. The merged
// 32x32 block leaves through smem as 64-byte bf16 row runs.
constexpr int kMaxSplit = 16;
template <int HD>
__global__ void __launch_bounds__(128) k_attn_combine(AttnTc p) {
  __shared__ float tile[32][33];
  pdl_trigger();
  pdl_wait();
  const int64_t r0 = int64_t(blockIdx.x) * 32;
  const int h = blockIdx.y, d0 = blockIdx.z * 32;
  const int n_splits = attn_nsplit(p, int(r0 / 128));
  if (n_splits <= 1) return;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t row = r0 + lane;
  const bool valid = row < p.rows;
  const int64_t sstride = int64_t(p.H) * (HD + 3) * p.rows;
  const float* base = p.part + (int64_t(h) * (HD + 3)) * p.rows + (valid ? row : 0);
  float ms[kMaxSplit], w[kMaxSplit];
  float M = -INFINITY;
#pragma unroll
  for (int s = 0; s < kMaxSplit; ++s) {
    ms[s] = (s < n_splits) ? base[s * sstride + int64_t(HD) * p.rows] : -INFINITY;
    M = fmaxf(M, ms[s]);
  }
  float L = 0.f, MN = 0.f;
  const bool do_mass = p.mass && blockIdx.z == 0 && wp == 0;
#pragma unroll
  for (int s = 0; s < kMaxSplit; ++s) {
    w[s] = (s < n_splits && ms[s] != -INFINITY) ? exp2f(ms[s] - M) : 0.f;
    if (s < n_splits) {
      L += w[s] * base[s * sstride + int64_t(HD + 1) * p.rows];
      if (do_mass) MN += w[s] * base[s * sstride + int64_t(HD + 2) * p.rows];
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  if (do_mass && valid) p.mass[int64_t(h) * p.rows + row] = L > 0.f ? double(MN) / double(L) : 0.0;
  if (p.stats && valid && blockIdx.z == 0 && wp == 0) {
    p.stats[(int64_t(h) * p.rows + row) * 2] = M;
    p.stats[(int64_t(h) * p.rows + row) * 2 + 1] = L;
  }
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
  for (int s = 0; s < kMaxSplit; ++s)
    if (s < n_splits) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += w[s] * base[s * sstride + int64_t(d0 + wp * 8 + j) * p.rows];
    }
#pragma unroll
  for (int j = 0; j < 8; ++j) tile[lane][wp * 8 + j] = acc[j] * inv;
  __syncthreads();
  // 32 rows x 16 bf16 pairs
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) {
    const int rr = i >> 4, d = 2 * (i & 15);
    if (r0 + rr < p.rows)
      *reinterpret_cast<uint32_t*>(p.out + ((r0 + rr) * p.H + h) * HD + d0 + d) = pack2(tile[rr][d], tile[rr][d + 1]);
  }
}

// ---------------------------------------------------------------- host
namespace {
CUtensorMap map2d(const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                  uint32_t box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = tmap_encode_cached(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
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

template <int HD>
void run_fa(cudaStream_t s, dim3 grid, const CUtensorMap& tq, const CUtensorMap& tk,
            const CUtensorMap& tv, const AttnTc& p) {
  const size_t smem = 1024 + 2 * size_t(128) * HD * 2 + (3 + 2) * (size_t(kAttnKB) * HD * 2) + 256 +
                      2 * kPgCache * sizeof(int);
  auto kern = k_attn_fa<HD>;
  static bool attr = false;
  if (!attr) {
    KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  KB_CUDA(launch_pdl(kern, grid, dim3(352), smem, s, tq, tk, tv, p));
  KB_LAUNCH();
}

template <int HD>
void run_fa1(cudaStream_t s, dim3 grid, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
             const AttnTc& p) {
  const size_t smem = 1024 + size_t(128) * HD * 2 + (3 + 2) * (size_t(kAttnKB) * HD * 2) + 256 +
                      2 * kPgCache * sizeof(int) + 2 * 2 * 128 * 2 * sizeof(float);
  auto kern = k_attn_fa1<HD>;
  static bool attr = false;
  if (!attr) {
    KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  KB_CUDA(launch_pdl(kern, grid, dim3(320), smem, s, tq, tk, tv, p));
  KB_LAUNCH();
}

void attn_set_timeline(unsigned long long* d) { KB_CUDA(cudaMemcpyToSymbol(g_attn_ts, &d, sizeof d)); }
int g_attn_target = 0;  // tuning knob (krul_debug_attn_bench): key blocks per work item
int g_attn_dbg = 0;     // tuning knob (krul_debug_attn_bench): unused by the pipelined kernel
void launch_attention_tc(const Ctx& c, cudaStream_t s, const Conv& conv, int layer,
                         const AttnArgs& a, DevBuf& scratch) {
  const Cfg& g = c.cfg;
  const int HD = g.hd;
  AttnTc p{};
  p.H = g.H;
  p.Hkv = g.Hkv;
  p.grp = g.H / g.Hkv;
  // kernel: one head per CTA with S double-buffered (default), or the
  // head-pair kernel (KRUL_ATTN_V=2; pairs only when they share a KV head)
  static const int variant = [] {
    const char* v = std::getenv("KRUL_ATTN_V");
    return v && v[0] == '2' ? 2 : 1;
  }();
  p.hpc = (variant == 2 && p.grp >= 2 && p.grp % 2 == 0) ? 2 : 1;
  p.rows = a.rows;
  p.pos0 = a.pos0;
  p.kv_total = a.pos0 + a.rows;
  p.n_qtiles = int((a.rows + 127) / 128);
  p.scale_log2 = (1.0f / sqrtf(float(HD))) * 1.4426950408889634f;
  p.pt = conv.d_pt + int64_t(layer) * conv.max_pages;
  p.max_pages = conv.max_pages;
  const int64_t pe = int64_t(c.page_elems());
  p.k_rows_pp = int(pe / HD);
  p.v_rows_pp = int(pe / 64);
  p.out = static_cast<bf16*>(a.out);
  p.mass = a.mass;
  p.stats = a.stats;
  p.il = a.mass ? a.il : 0;
  p.rs = a.mass ? a.rs : INT64_MAX;

  // key blocks per work item: about one SM's fair share of all block-units,
  // at least 4 (splitting costs a partial round trip + the merge)
  const int units_y = (g.H + p.hpc - 1) / p.hpc;
  int64_t total = 0;
  p.target = 1 << 30;
  for (int qt = 0; qt < p.n_qtiles; ++qt) total += attn_nblk(p, qt);
  const int64_t sms = c.sm_count > 0 ? c.sm_count : 148;
  p.target = int(std::max<int64_t>(4, (total * units_y + sms - 1) / sms));
  p.target = std::max(p.target, (attn_nblk(p, p.n_qtiles - 1) + kMaxSplit - 1) / kMaxSplit);
  {
    // wave quantisation: the fair share can leave a few items for a second
    // wave (70B / 32K new-input prefill: 160 items on 148 SMs = two waves of
    // 28 blocks); take the key-block count per item in [fair, 2 fair] that
    // minimises waves x blocks per item (ties: fewer splits to merge)
    const int t0 = p.target;
    int best_t = t0;
    int64_t best_cost = INT64_MAX;
    for (int t = t0; t <= 2 * t0; ++t) {
      p.target = t;
      int64_t items_t = 0;
      for (int qt = 0; qt < p.n_qtiles; ++qt) items_t += attn_nsplit(p, qt);
      const int64_t cost = (items_t * units_y + sms - 1) / sms * t;
      if (cost < best_cost) {
        best_cost = cost;
        best_t = t;
      }
    }
    p.target = best_t;
  }
  if (g_attn_target > 0) p.target = std::max(g_attn_target, (attn_nblk(p, p.n_qtiles - 1) + kMaxSplit - 1) / kMaxSplit);
  int items = 0, max_split = 1;
  for (int qt = 0; qt < p.n_qtiles; ++qt) {
    items += attn_nsplit(p, qt);
    max_split = std::max(max_split, attn_nsplit(p, qt));
  }
  if (max_split > 1)
    p.part = static_cast<float*>(
        scratch.ensure(size_t(max_split) * a.rows * g.H * (HD + 3) * sizeof(float)));
  const uint64_t pool_elems = uint64_t(c.pool_pages) * pe;
  const CUtensorMap tq = map2d(a.q, uint64_t(a.rows), uint64_t(g.H) * HD, uint64_t(g.H) * HD, 128);
  const CUtensorMap tk = map2d(c.pool.p, pool_elems / HD, HD, HD, 64);
  const CUtensorMap tv = map2d(c.pool.p, pool_elems / 64, 64, 64, uint32_t(HD));
  const dim3 grid{unsigned(items), unsigned(units_y), 1u};
  if (variant == 1) {
    if (HD == 128)
      run_fa1<128>(s, grid, tq, tk, tv, p);
    else
      run_fa1<64>(s, grid, tq, tk, tv, p);
  } else if (HD == 128) {
    run_fa<128>(s, grid, tq, tk, tv, p);
  } else {
    run_fa<64>(s, grid, tq, tk, tv, p);
  }
  if (max_split > 1) {
    const dim3 g2{unsigned((a.rows + 31) / 32), unsigned(g.H), unsigned(HD / 32)};
    if (HD == 128)
      KB_CUDA(launch_pdl(k_attn_combine<128>, g2, dim3(128), 0, s, p));
    else
      KB_CUDA(launch_pdl(k_attn_combine<64>, g2, dim3(128), 0, s, p));
    KB_LAUNCH();
  }
}

}  // namespace kb
