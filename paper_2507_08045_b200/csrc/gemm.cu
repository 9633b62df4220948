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

#include <cstdlib>
#include <cstring>

#include "dev.cuh"
#include "kb.hpp"

namespace kb {

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

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              int M, int N, int K, Epi e) {
  constexpr int BM = 128, BK = 64;
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // M-tile fastest: co-resident CTAs share one B (weight) tile, so each
  // weight tile streams from HBM once while the small A panel stays in L2
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int num_k = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_slot)),
                 "r"(uint32_t(BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < num_k; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        tc::mbar_wait(&empty[s], ph ^ 1);
        tc::mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
        tc::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
        tc::tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                                 (uint32_t(BM >> 4) << 24);
      for (int kb = 0; kb < num_k; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        tc::mbar_wait(&full[s], ph);
        tc::fence_after();
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t da = tc::sw128_desc(sA + s * A_BYTES + k * 32);
          const uint64_t db = tc::sw128_desc(sB + s * B_BYTES + k * 32);
          tc::mma_bf16(tmem, da, db, idesc, (kb | k) != 0);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(accum);
    }
  } else {  // epilogue warps 2..5 -> TMEM lanes 32*(warp%4)
    tc::mbar_wait(accum, 0);
    tc::fence_after();
    const int lane_base = 32 * (warp & 3);
    const int64_t r = int64_t(m0) + lane_base + lane;
    float v[32];
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      tc::tmem_ld32(tmem + (uint32_t(lane_base) << 16) + uint32_t(c), v);
      const int64_t col = int64_t(n0) + c;
      if (r < M && col < N) {
        const int nv = int(N - col < 32 ? N - col : 32);
        epi_apply<bf16>(e, r, col, v, nv);
      }
    }
  }
  __syncwarp();
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(uint32_t(BN)));
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
// Row-major bf16 [rows][cols] with leading dimension ld (elements); box
// [box_rows][64] with 128-byte swizzle.
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRUL_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

template <int BN, int STAGES>
void launch_tc(cudaStream_t s, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
               const void* B, int64_t ldb, const Epi& e) {
  const CUtensorMap ta = make_map(A, M, K, lda, 128);
  const CUtensorMap tb = make_map(B, N, K, ldb, BN);
  const size_t smem = 1024 + size_t(STAGES) * (128 * 64 * 2 + BN * 64 * 2) + 8 * (2 * STAGES + 1) + 16;
  auto kern = k_gemm_tc<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  dim3 grid(unsigned((M + 127) / 128), unsigned((N + BN - 1) / BN));
  kern<<<grid, 192, smem, s>>>(ta, tb, int(M), int(N), int(K), e);
  KB_LAUNCH();
}

int gemm_mode() {  // 0 auto, 1 force SIMT
  static int m = [] {
    const char* v = std::getenv("KRUL_GEMM");
    return (v && std::strcmp(v, "simt") == 0) ? 1 : 0;
  }();
  return m;
}
}  // namespace

void gemm(const Ctx& c, cudaStream_t s, int64_t M, int64_t N, int64_t K, const void* A,
          int64_t lda, const void* B, int64_t ldb, const Epi& e) {
  if (M <= 0 || N <= 0) return;
  const bool tc_ok = c.cfg.dtype == KRUL_BF16 && gemm_mode() == 0 && lda % 8 == 0 &&
                     ldb % 8 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(B) & 15) == 0 && K >= 1;
  if (tc_ok) {
    // wave efficiency of each tile width on this device; prefer the wider
    // (higher arithmetic intensity) tile unless it strands SMs
    const int64_t mt = (M + 127) / 128, sms = c.sm_count > 0 ? c.sm_count : 148;
    auto eff = [&](int64_t bn) {
      const int64_t t = mt * ((N + bn - 1) / bn);
      return double(t) / double(((t + sms - 1) / sms) * sms);
    };
    if (N >= 256 && eff(256) >= 0.8 * eff(128))
      launch_tc<256, 4>(s, M, N, K, A, lda, B, ldb, e);
    else
      launch_tc<128, 6>(s, M, N, K, A, lda, B, ldb, e);
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
