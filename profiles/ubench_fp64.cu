// Microbenchmark (tooling, not product): FP64 dependent-chain latencies and
// pipe throughputs on the B200, used to size the sequential core-block solve
// and the all-prefix statistics kernel.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench profiles/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_dmul_dadd(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * a;
  long long t1 = clock64();
  double y = b;
  for (int i = 0; i < n; ++i) y = y + x;
  long long t2 = clock64();
  out[threadIdx.x] = x + y;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

__global__ void lat_shfl(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i & 31));
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ int idx[64];
  if (threadIdx.x < 64) idx[threadIdx.x] = (threadIdx.x + 1) & 63;
  __syncthreads();
  int j = threadIdx.x & 63;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// throughput: 8 independent chains per thread
__global__ void thr_dfma(double* out, double a, double b, int n) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = a + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void thr_dmma(double* out, double a, double b, int n) {
  double d[4][2] = {};
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) dmma884(d[k][0], d[k][1], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// both pipes at once: half the warps DFMA, half DMMA
__global__ void thr_mixed(double* out, double a, double b, int n) {
  double s = 0;
  if ((threadIdx.x >> 5) & 1) {
    double d[4][2] = {};
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma884(d[k][0], d[k][1], a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  } else {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = a + k;
    for (int i = 0; i < 4 * n; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 64);
  long long h[2];
  const int n = 4096;
  lat_dfma<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", (double)h[0] / n);
  lat_dmul_dadd<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cyc, DADD: %.2f cyc\n", (double)h[0] / n, (double)h[1] / n);
  lat_shfl<<<1, 32>>>(out, cyc, 1.0, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("SHFL.IDX (64-bit = 2 shfl) dependent latency: %.2f cyc\n", (double)h[0] / n);
  lat_lds<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cyc\n", (double)h[0] / n);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 20000;
  for (int warps : {4, 8, 16, 32}) {
    const int blocks = sms * 2;
    thr_dfma<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, 100);
    cudaEventRecord(e0);
    thr_dfma<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = (double)blocks * 32 * warps * it * 8;
    printf("DFMA thr (%2d warps/CTA, 2 CTA/SM): %.2f TFLOP/s\n", warps, 2 * fma / ms / 1e9);
    thr_dmma<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, 100);
    cudaEventRecord(e0);
    thr_dmma<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mm = (double)blocks * warps * it * 4 * 256;
    printf("DMMA thr (%2d warps/CTA, 2 CTA/SM): %.2f TFLOP/s\n", warps, 2 * mm / ms / 1e9);
    thr_mixed<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, 100);
    cudaEventRecord(e0);
    thr_mixed<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mix = (double)blocks * (warps / 2) * (it * 4 * 256.0 + 32.0 * 4 * it * 8);
    printf("mixed DFMA+DMMA (%2d warps/CTA): %.2f TFLOP/s (%.3f ms)\n", warps, 2 * mix / ms / 1e9, ms);
  }
  printf("SMs %d, clock %d kHz\n", sms, clk);
  return 0;
}
