// graph_event.cu — ordering of external event record / wait nodes between two
// CUDA graphs launched on different streams (kernel-tuning experiment): graph
// A = spin ~1 ms, record E (external); graph B = wait E (external), stamp.
// If B's stamp follows A's spin, a wait node honours a record node of a graph
// launched before it (host order), as stream-ordered events do.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_event graph_event.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long now() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void spin(unsigned long long* out, long long ns) {
  unsigned long long t0 = now();
  while (now() - t0 < (unsigned long long)ns) {}
  out[0] = now();
}
__global__ void stamp(unsigned long long* out) { out[1] = now(); }
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaStream_t sa, sb, x, y;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&y, cudaStreamNonBlocking);
  cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaGraph_t ga, gb; cudaGraphExec_t ea, eb;
  cudaStreamBeginCapture(sa, cudaStreamCaptureModeRelaxed);
  spin<<<1, 1, 0, sa>>>(d, 1000000);
  cudaEventRecordWithFlags(e, sa, cudaEventRecordExternal);
  cudaStreamEndCapture(sa, &ga);
  cudaStreamBeginCapture(sb, cudaStreamCaptureModeRelaxed);
  cudaStreamWaitEvent(sb, e, cudaEventWaitExternal);
  stamp<<<1, 1, 0, sb>>>(d);
  cudaStreamEndCapture(sb, &gb);
  printf("capture: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaGraphInstantiate(&ea, ga, 0); cudaGraphInstantiate(&eb, gb, 0);
  for (int it = 0; it < 4; ++it) {
    cudaMemset(d, 0, 16); cudaDeviceSynchronize();
    cudaGraphLaunch(ea, x);
    cudaGraphLaunch(eb, y);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("iter %d: spin end %llu, B stamp %llu -> B %s A's record (%s)\n", it, h[0], h[1],
           h[1] >= h[0] ? "after" : "BEFORE", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
