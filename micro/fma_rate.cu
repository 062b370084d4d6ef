// fma_rate.cu -- FP32 FMA issue rate on sm_100a: 3-register FFMA vs packed FFMA2 (fp32x2),
// 8 / 16 / 32 warps per SM, 8 independent accumulator chains per thread, no memory traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rate fma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_k(float *out, float a, float b, int iters) {
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  float bb = b + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(r[i], a, bb);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_k(float *out, float a, float b, int iters) {
  unsigned long long r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x = threadIdx.x * 0.001f + i, y = x + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r[i]) : "f"(x), "f"(y));
  }
  unsigned long long av, bv;
  float bb = b + threadIdx.x * 1e-7f;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(bb));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(r[i]) : "l"(av), "l"(bv));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r[i]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_k(double *out, double a, double b, int iters) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001 + i;
  double bb = b + threadIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, bb);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float *out;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int k = 0; k < 2; ++k) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto run = [&]() {
        if (k == 0) ffma_k<<<148, warps * 32>>>(out, 0.999f, 0.001f, iters);
        else ffma2_k<<<148, warps * 32>>>(out, 0.999f, 0.001f, iters);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = 148.0 * warps * 32 * iters * 16;  // both kernels: 16 fp32 FMAs per thread-iteration
      int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
      printf("%s warps/SM=%2d: %.1f TFLOP/s  %.1f FMA/clk/SM (at %d MHz)\n", k ? "FFMA2" : "FFMA ", warps,
             2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / 148 / (khz * 1e3), khz / 1000);
    }
  }
  // FP64 (DFMA): the NF_MATH_FP64 path's ALU roofline
  double *dout;
  cudaMalloc(&dout, 148 * 1024 * sizeof(double));
  for (int warps : {4, 8, 16, 32}) {
    const int di = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    dfma_k<<<148, warps * 32>>>(dout, 0.999, 0.001, di);
    cudaEventRecord(e0);
    dfma_k<<<148, warps * 32>>>(dout, 0.999, 0.001, di);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = 148.0 * warps * 32 * di * 16;
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("DFMA  warps/SM=%2d: %.2f TFLOP/s  %.2f FMA/clk/SM (at %d MHz)\n", warps, 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / 148 / (khz * 1e3), khz / 1000);
  }
  return 0;
}
