// Cluster-shape study of the Rayleigh-Ritz Jacobi (jacobi_cluster_kernel<CL, GRP, NMAX>):
// microseconds per sweep for n = 160 / 128 / 96 on a random n x n matrix, 3 forced sweeps,
// for every (CTAs per cluster, lanes per pair) candidate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I paper_2306_08212_b200/csrc tools/bench_jacobi_cfg.cu -o gpurun_out/bench_jacobi_cfg
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "iso_kernels.cuh"

using namespace ctm::isok;
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      printf("{\"err\":\"%s\",\"line\":%d}\n", cudaGetErrorString(e_), __LINE__);          \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

static double urand(unsigned long long& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

static double *dX, *dU, *dSig;
static int* dst;
static cudaEvent_t e0, e1;

template <int CL, int GRP, int NMAX>
void run(int n, int sweeps) {
  using J = JacCfg<CL, GRP, NMAX>;
  if (n > NMAX) return;
  CK(cudaFuncSetAttribute(jacobi_cluster_kernel<CL, GRP, NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J::SMEM));
  auto launch = [&]() {
    jacobi_cluster_kernel<CL, GRP, NMAX><<<CL, J::THREADS, J::SMEM>>>(dX, n, 1, n, dU, dSig, dst + 1, sweeps, 1e-300, 0.0);
  };
  launch();
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  double sig0 = 0.0, sigl = 0.0;
  CK(cudaMemcpy(&sig0, dSig, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&sigl, dSig + n - 1, 8, cudaMemcpyDeviceToHost));
  const double us = 1e3 * ms / reps;
  printf("{\"n\":%d,\"cl\":%d,\"grp\":%d,\"nmax\":%d,\"threads\":%d,\"sweeps\":%d,\"us\":%.1f,\"us_per_sweep\":%.1f,"
         "\"s0\":%.12f,\"slast\":%.6e}\n",
         n, CL, GRP, NMAX, J::THREADS, sweeps, us, us / sweeps, sig0, sigl);
  fflush(stdout);
}

int main() {
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int nmax = 320;
  CK(cudaMalloc(&dX, 8ull * nmax * nmax));
  CK(cudaMalloc(&dU, 8ull * nmax * nmax));
  CK(cudaMalloc(&dSig, 8ull * nmax));
  CK(cudaMalloc(&dst, 64));
  CK(cudaMemset(dst, 0, 64));
  unsigned long long seed = 12345;
  std::vector<double> X((size_t)nmax * nmax);
  for (auto& v : X) v = urand(seed);
  CK(cudaMemcpy(dX, X.data(), 8ull * nmax * nmax, cudaMemcpyHostToDevice));
  for (int n : {160, 128, 64}) {
    const int sw = 3;
    run<4, 4, 128>(n, sw);
    run<4, 2, 128>(n, sw);
    run<8, 2, 128>(n, sw);
    run<8, 4, 128>(n, sw);
    run<4, 4, 160>(n, sw);
    run<4, 2, 160>(n, sw);
    run<8, 2, 160>(n, sw);
    run<8, 4, 160>(n, sw);
  }
  for (int n : {288, 232}) {   // C5 sizes (l = n_keep + 48)
    const int sw = 2;
    run<8, 2, 320>(n, sw);
    run<8, 4, 320>(n, sw);
  }
  return 0;
}
