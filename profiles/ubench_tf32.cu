// Throughput of warp-level mma.sync on sm_100a: TF32 m16n8k8 (fp32 accumulate)
// vs FP64 DMMA m8n8k4 -- decides whether a 3xTF32 Gram could replace DMMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tf32 ubench_tf32.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float* out, int iters) {
  float d[8][4] = {};
  unsigned a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x ^ 5u, 7u};
  unsigned b[2] = {threadIdx.x * 11u, 13u};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * 4, threads = 32 * warps / 4 * 4 / 4, iters = 4096;
    (void)threads;
    const int tpb = 32 * warps;
    k_tf32<<<sms, tpb>>>(o, 16);
    cudaEventRecord(e0);
    k_tf32<<<sms * 2, tpb>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (sms * 2.0) * warps;
    printf("TF32 mma.sync m16n8k8, %2d warps/CTA, 2 CTA/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    k_dmma<<<sms, tpb>>>((double*)o, 16);
    cudaEventRecord(e0);
    k_dmma<<<sms * 2, tpb>>>((double*)o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 2.0 * 8 * 8 * 4 * 8.0 * iters * (sms * 2.0) * warps;
    printf("DMMA m8n8k4,             %2d warps/CTA, 2 CTA/SM: %.1f TFLOP/s\n", warps, f2 / ms / 1e9);
    (void)blocks;
  }
  return 0;
}
