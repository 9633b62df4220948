// mma_rate.cu — tcgen05.mma issue/execute rate per instruction shape on one SM
// (kernel-tuning experiment, not product code). One CTA, one issuing thread:
// R back-to-back kind::f16 MMAs of M=128, N in {64,128,256}, K=16, A from
// shared memory (SS) or TMEM (TS), accumulate into TMEM; clock64 from the
// first issue to the commit's mbarrier completing.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* p) {  // K-major, SW128, SBO 1024
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool TS>
__global__ void k_rate(int reps, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = base;              // 128 x 64 bf16 (16 KB)
  unsigned char* sB = base + 16384;      // N x 64 bf16
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t d = tmem;            // accumulator columns [0, N)
    const uint32_t aT = tmem + 256;     // A (TS form): 128 x 64 bf16 = 32 columns
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t db = desc(sB + k * 32);
        if (TS) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(aT + uint32_t(k * 8)), "l"(db), "r"(id), "r"(1));
        } else {
          const uint64_t da = desc(sA + k * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(da), "l"(db), "r"(id), "r"(1));
        }
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS>
void run(long long* d) {
  const int reps = 256;
  const size_t smem = 1024 + 16384 + N * 128;
  cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int w = 0; w < 2; ++w) k_rate<N, TS><<<1, 128, smem>>>(reps, d);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double per = double(h[1]) / (reps * 4);
  printf("M=128 N=%3d K=16 %s: issue %.1f clk/MMA, complete %.1f clk/MMA, %.0f flop/clk (%s)\n", N, TS ? "TS" : "SS",
         double(h[0]) / (reps * 4), per, 128.0 * N * 16 * 2 / per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<64, false>(d);
  run<128, false>(d);
  run<256, false>(d);
  run<64, true>(d);
  run<128, true>(d);
  run<256, true>(d);
  return 0;
}
