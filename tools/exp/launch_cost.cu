// Device-side fixed cost of a kernel launch inside a CUDA graph (B200):
// graph of `iters` back-to-back launches of the same kernel, replayed, timed
// with events. Variants add the prologue pieces of the tcgen05 GEMM one by one.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o launch_cost launch_cost.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__global__ void k_empty() {}

template <int MODE>
__global__ void __launch_bounds__(192, 1) k_pro(float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(&bar[i]))), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE >= 1 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        uint32_t(__cvta_generic_to_shared(&slot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (MODE >= 2) {  // touch 16 KB of smem per thread-block (like a staging tile) and write one value out
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = float(i);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = reinterpret_cast<float*>(sm)[blockIdx.x & 4095];
  }
  __syncthreads();
  if (MODE >= 1 && warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
  }
}

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t r_ = (x);                                                            \
    if (r_ != cudaSuccess) {                                                         \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r_));       \
      fflush(stdout);                                                                \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)
template <class F>
float time_graph(F launch, int iters, cudaStream_t s) {
  cudaGraph_t g;
  cudaGraphExec_t e;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  for (int i = 0; i < iters; ++i) launch();
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&e, g, 0));
  CK(cudaGraphLaunch(e, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(e, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(e);
  cudaGraphDestroy(g);
  return ms * 1e3f / iters;
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  float* out;
  CK(cudaMalloc(&out, 1 << 20));
  printf("start\n");
  fflush(stdout);
  const int iters = 200;
  for (int grid : {1, 148, 296}) {
    printf("empty grid %3d: %.2f us/launch\n", grid, time_graph([&] { k_empty<<<grid, 192, 0, s>>>(); }, iters, s));
    fflush(stdout);
  }
  for (size_t smem : {size_t(0), size_t(100 << 10), size_t(220 << 10)}) {
    CK(cudaFuncSetAttribute(k_pro<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(k_pro<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(k_pro<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    printf("smem %3zu KB grid 148: barriers %.2f | +tmem %.2f | +smem fill+store %.2f us/launch\n", smem >> 10,
           time_graph([&] { k_pro<0><<<148, 192, smem, s>>>(out); }, iters, s),
           time_graph([&] { k_pro<1><<<148, 192, smem, s>>>(out); }, iters, s),
           time_graph([&] { k_pro<2><<<148, 192, smem, s>>>(out); }, iters, s));
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
