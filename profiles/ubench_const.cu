// Microbenchmark (tooling, not product): DFMA throughput when one operand is a
// warp-uniform constant-bank value (LDCU), vs how many entries (independent
// FMAs) share each constant -- the factor-update kernel's inner-loop shape.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/ubench_const profiles/ubench_const.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double c_tab[1024];

template <int NE>
__global__ void __launch_bounds__(256, 2) k_const(double* out, int reps) {
  double acc[NE], x[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    acc[e] = 0.0;
    x[e] = 1.0 + 1e-3 * (threadIdx.x + e);
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 10
    for (int i = 0; i < 1000; ++i) {
      const double g = c_tab[i];
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] = fma(g, x[e], acc[e]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) s += acc[e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// same, but the constant is in shared memory (broadcast LDS)
template <int NE>
__global__ void __launch_bounds__(256, 2) k_smem(double* out, int reps) {
  __shared__ double s_tab[1000];
  for (int i = threadIdx.x; i < 1000; i += blockDim.x) s_tab[i] = 1e-3 * i;
  __syncthreads();
  double acc[NE], x[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    acc[e] = 0.0;
    x[e] = 1.0 + 1e-3 * (threadIdx.x + e);
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 10
    for (int i = 0; i < 1000; i += 2) {
      const double2 g = reinterpret_cast<const double2*>(s_tab)[i / 2];
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] = fma(g.y, x[e], fma(g.x, x[e], acc[e]));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) s += acc[e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
void run(const char* name, K kern, int ne, double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 2 * sms, reps = 200;
  kern<<<blocks, 256>>>(out, 2);
  cudaEventRecord(e0);
  kern<<<blocks, 256>>>(out, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = (double)blocks * 256 * reps * 1000.0 * ne;
  printf("%-6s NE=%d: %.2f TFLOP/s  (%s)\n", name, ne, 2 * fma / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 1e-3 * i;
  cudaMemcpyToSymbol(c_tab, h, sizeof(h));
  double* out;
  cudaMalloc(&out, 1 << 24);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run("const", k_const<1>, 1, out, sms);
  run("const", k_const<2>, 2, out, sms);
  run("const", k_const<4>, 4, out, sms);
  run("const", k_const<8>, 8, out, sms);
  run("smem", k_smem<1>, 1, out, sms);
  run("smem", k_smem<2>, 2, out, sms);
  run("smem", k_smem<4>, 4, out, sms);
  run("smem", k_smem<8>, 8, out, sms);
  return 0;
}
