// fp2_rate.cu — FADD2/FFMA2 (packed f32x2) issue rates per SMSP, the K1 fold's
// inner op (kernel-tuning experiment).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp2_rate fp2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int reps, float* out, long long* clk) {
  float2 x[4], y[8], acc[32];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = make_float2(threadIdx.x * 2e-3f - i, i * 0.25f);
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 0) {  // FADD2 + FFMA2 (the fold)
          const float2 d = __fadd2_rn(x[i], make_float2(-y[j].x, -y[j].y));
          acc[i * 8 + j] = __ffma2_rn(d, d, acc[i * 8 + j]);
        } else if (MODE == 1) {  // FFMA2 only
          acc[i * 8 + j] = __ffma2_rn(x[i], y[j], acc[i * 8 + j]);
        } else if (MODE == 2) {  // scalar FADD + FFMA x2
          float d0 = x[i].x - y[j].x, d1 = x[i].y - y[j].y;
          acc[i * 8 + j].x = fmaf(d0, d0, acc[i * 8 + j].x);
          acc[i * 8 + j].y = fmaf(d1, d1, acc[i * 8 + j].y);
        } else {  // FFMA2 d*d with d from FFMA2 (x - y as fma(y, -1, x))
          const float2 d = __ffma2_rn(y[j], make_float2(-1.f, -1.f), x[i]);
          acc[i * 8 + j] = __ffma2_rn(d, d, acc[i * 8 + j]);
        }
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i].x += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  const int reps = 4096;
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {4, 8, 16}) {
      long long clk = 0;
      auto run = [&] {
        if (mode == 0) k<0><<<148, warps * 32>>>(reps, o, c);
        if (mode == 1) k<1><<<148, warps * 32>>>(reps, o, c);
        if (mode == 2) k<2><<<148, warps * 32>>>(reps, o, c);
        if (mode == 3) k<3><<<148, warps * 32>>>(reps, o, c);
      };
      run();
      run();
      cudaMemcpy(&clk, c, 8, cudaMemcpyDeviceToHost);
      const int ops_per_rep = mode == 1 ? 32 : mode == 2 ? 128 : 64;  // instructions per warp per rep
      double per_smsp = double(reps) * ops_per_rep * warps / 4.0;
      printf("mode %d warps %2d: %.2f cycles per FP instruction per SMSP\n", mode, warps, double(clk) / per_smsp);
    }
  return 0;
}
