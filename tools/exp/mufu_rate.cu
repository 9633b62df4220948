// mufu_rate.cu — MUFU.EX2 and FFMA issue rates per SM (kernel-tuning experiment).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(int reps, float* out, long long* clk) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) * -0.5f;         // MUFU + FMUL
      else v[i] = fmaf(v[i], 0.999f, 1e-3f);           // FFMA only
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  for (int warps : {4, 8, 16, 32}) {
    for (int mode = 0; mode < 2; ++mode) {
      const int reps = 1024;
      if (mode == 0) { k<0><<<148, warps * 32>>>(reps, o, c); k<0><<<148, warps * 32>>>(reps, o, c); }
      else { k<1><<<148, warps * 32>>>(reps, o, c); k<1><<<148, warps * 32>>>(reps, o, c); }
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double ops = double(reps) * 16 * warps * 32;  // per SM
      printf("%2d warps/SM %s: %.2f ops/clk/SM (%.1f clk per warp-instr per SMSP)\n", warps,
             mode == 0 ? "MUFU.EX2(+FMUL)" : "FFMA", ops / h, double(h) / (double(reps) * 16 * warps / 4));
    }
  }
  return 0;
}
