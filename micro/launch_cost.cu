// launch_cost.cu -- host time of cudaLaunchKernelEx for a K6-shaped launch (120 CTAs in clusters
// of 8, 512 threads, ~200 KB dynamic smem) as a function of the parameter-buffer size and the
// cooperative attribute; and the device time of an empty such kernel (events around it).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 launch_cost.cu -o launch_cost
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int NB>
struct Pad {
  long long v[NB];
};

template <int NB>
__global__ void __launch_bounds__(512, 1) k_empty(const __grid_constant__ Pad<NB> p, long long *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.v[NB - 1] == 12345) out[0] = p.v[0];
}

template <int NB>
void run(bool coop, int smem) {
  static Pad<NB> p{};
  long long *out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_empty<NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_empty<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim = {8, 1, 1};
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop ? 2 : 1;
  cfg.gridDim = dim3(120);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cfg.stream = st;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double host = 0, dev = 0;
  const int n = 200;
  for (int it = 0; it < n + 10; ++it) {
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    auto t0 = std::chrono::high_resolution_clock::now();
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_empty<NB>, p, out);
    auto t1 = std::chrono::high_resolution_clock::now();
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e)); return; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 10) { host += std::chrono::duration<double, std::micro>(t1 - t0).count(); dev += ms * 1e3; }
  }
  printf("params %6zu B  coop %d  smem %6d: host launch %6.2f us  events around launch %6.2f us\n", sizeof(Pad<NB>), (int)coop,
         smem, host / n, dev / n);
  cudaFree(out);
  cudaStreamDestroy(st);
}

int main() {
  for (int smem : {0, 200 * 1024})
    for (bool coop : {false, true}) {
      run<4>(coop, smem);
      run<64>(coop, smem);
      run<512>(coop, smem);
      run<1040>(coop, smem);
    }
  return 0;
}
