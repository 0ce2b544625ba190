// Microbenchmark (tooling): the core-block solve kernel alone, single block and pair group.
//   nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
//        -Ipaper_1904_02603_b200/csrc -o build/ubench_solve profiles/ubench_solve.cu
#include "vest_core_sall.cu"
#include <cstdio>
#include <vector>
namespace vest {
uint64_t& launch_counter() { static uint64_t c = 0; return c; }
void check(cudaError_t, const char*) {}
void ensure(Ctx&, double**, size_t*, size_t) {}
double reduce_chunk_sums(Ctx&, const double*, uint64_t) { return 0; }
void comm_allreduce(Ctx&, double*, uint64_t) {}
DevModel Ctx::model_view() const { return {}; }
DevCSF Ctx::csf_view(int) const { return {}; }
}  // namespace vest
using namespace vest;
int main() {
  const int nf = 10, Jm = 10, NS = 55, NAm = 55, nq = 100;
  std::vector<double> T(NS * NAm), C(2 * nq + 1), core(1000);
  for (int i = 0; i < NS * NAm; ++i) T[i] = 1e-3 * ((i * 7919) % 101);
  for (int f = 0; f < nf; ++f)  // dominant diagonal
    for (int c = 0; c < Jm; ++c) T[tri_idx(f, f, nf) * NAm + tri_idx(c, c, Jm)] += 10.0;
  for (int i = 0; i <= 2 * nq; ++i) C[i] = 0.1 * (i % 13);
  for (int i = 0; i < 1000; ++i) core[i] = 0.01 * (i % 17);
  std::vector<uint32_t> fib(nf);
  for (int f = 0; f < nf; ++f) fib[f] = 30 + f;
  double *dT, *dC, *dcore, *ddg, *ds;
  uint32_t* dfib;
  uint8_t* dmask;
  cudaMalloc(&dT, T.size() * 8); cudaMalloc(&dC, C.size() * 8); cudaMalloc(&dcore, 8000);
  cudaMalloc(&ddg, 8 * 256); cudaMalloc(&ds, 8); cudaMalloc(&dfib, 4 * nf); cudaMalloc(&dmask, 1000);
  cudaMemcpy(dT, T.data(), T.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dcore, core.data(), 8000, cudaMemcpyHostToDevice);
  cudaMemcpy(dfib, fib.data(), 4 * nf, cudaMemcpyHostToDevice);
  cudaMemset(dmask, 0, 1000);
  const size_t smem = (2 * (h_stride(nq) + kSolveSlack) + 2 * nq) * 8;
  double* dH;
  cudaMalloc(&dH, nq * nq * 8 + 16);
  k_expand_h<<<40, 256>>>(dT, 1, nf, Jm, dH);
  cudaFuncSetAttribute(k_core_solve_g<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_core_solve_g<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int reg = 0; reg < 2; ++reg) {
    auto kern = reg == 0 ? k_core_solve_g<0> : k_core_solve_g<1>;
    for (int two = 0; two < 2; ++two) {
    const double* Hb = two ? dH : nullptr;
    kern<<<1, 32, smem>>>(dH, Hb, Hb, dC, nf, Jm, dfib, dfib, dcore, dmask, 0.01, ddg, ds);
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) kern<<<1, 32, smem>>>(dH, Hb, Hb, dC, nf, Jm, dfib, dfib, dcore, dmask, 0.01, ddg, ds);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("reg %d, %s: %.2f us/launch  err=%s\n", reg, two ? "pair" : "single", ms * 10,
           cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
