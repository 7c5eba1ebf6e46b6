// Probe: concurrency of independent cuSOLVER SVDs (one handle + stream each) for the
// shapes of one column absorption: 1024x1024 and 1024x128.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <thread>
#include <chrono>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1);} } while (0)
struct Job { cusolverDnHandle_t h; cusolverDnParams_t p; gesvdjInfo_t gi; cudaStream_t s; double *A, *A0, *S, *U, *V, *work; void* hbuf; size_t dws, hws; int lw; int* info; };
int main() {
  const int NJ = 4;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int shape = 0; shape < 2; ++shape) {
    int m = 1024, n = shape == 0 ? 1024 : 128;
    std::vector<double> hA((size_t)m * n);
    for (auto& x : hA) x = (rand() / (double)RAND_MAX) - 0.5;
    for (int algo = 0; algo < 3; ++algo) {   // 0 gesvdp, 1 gesvdj, 2 Xgesvd
      Job J[NJ];
      for (int j = 0; j < NJ; ++j) {
        Job& b = J[j];
        CK(cusolverDnCreate(&b.h)); CK(cusolverDnCreateParams(&b.p)); CK(cudaStreamCreate(&b.s)); CK(cusolverDnSetStream(b.h, b.s));
        cusolverDnCreateGesvdjInfo(&b.gi); cusolverDnXgesvdjSetTolerance(b.gi, 2.2e-16); cusolverDnXgesvdjSetMaxSweeps(b.gi, 100);
        cudaMalloc(&b.A, 8ull * m * n); cudaMalloc(&b.A0, 8ull * m * n); cudaMalloc(&b.S, 8ull * n); cudaMalloc(&b.U, 8ull * m * n); cudaMalloc(&b.V, 8ull * n * n); cudaMalloc(&b.info, 4);
        cudaMemcpy(b.A0, hA.data(), 8ull * m * n, cudaMemcpyHostToDevice);
        if (algo == 0) { CK(cusolverDnXgesvdp_bufferSize(b.h, b.p, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_R_64F, b.A, m, CUDA_R_64F, b.S, CUDA_R_64F, b.U, m, CUDA_R_64F, b.V, n, CUDA_R_64F, &b.dws, &b.hws)); }
        else if (algo == 1) { CK(cusolverDnDgesvdj_bufferSize(b.h, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, b.A, m, b.S, b.U, m, b.V, n, &b.lw, b.gi)); b.dws = 8ull * b.lw; b.hws = 0; }
        else { CK(cusolverDnXgesvd_bufferSize(b.h, b.p, 'S', 'N', m, n, CUDA_R_64F, b.A, m, CUDA_R_64F, b.S, CUDA_R_64F, b.U, m, CUDA_R_64F, b.V, n, CUDA_R_64F, &b.dws, &b.hws)); }
        cudaMalloc(&b.work, b.dws + 8); b.hbuf = malloc(b.hws + 8);
      }
      auto run = [&](Job& b) {
        cudaMemcpyAsync(b.A, b.A0, 8ull * m * n, cudaMemcpyDeviceToDevice, b.s);
        double err;
        if (algo == 0) CK(cusolverDnXgesvdp(b.h, b.p, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_R_64F, b.A, m, CUDA_R_64F, b.S, CUDA_R_64F, b.U, m, CUDA_R_64F, b.V, n, CUDA_R_64F, b.work, b.dws, b.hbuf, b.hws, b.info, &err));
        else if (algo == 1) CK(cusolverDnDgesvdj(b.h, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, b.A, m, b.S, b.U, m, b.V, n, b.work, b.lw, b.info, b.gi));
        else CK(cusolverDnXgesvd(b.h, b.p, 'S', 'N', m, n, CUDA_R_64F, b.A, m, CUDA_R_64F, b.S, CUDA_R_64F, b.U, m, CUDA_R_64F, b.V, n, CUDA_R_64F, b.work, b.dws, b.hbuf, b.hws, b.info));
      };
      for (int j = 0; j < NJ; ++j) run(J[j]);   // warm
      cudaDeviceSynchronize();
      // sequential (host issues one after the other, waits each)
      cudaEventRecord(e0);
      for (int j = 0; j < NJ; ++j) { run(J[j]); cudaStreamSynchronize(J[j].s); }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float seq; cudaEventElapsedTime(&seq, e0, e1);
      // concurrent: one host thread per job would be needed for blocking APIs; try issue-all then sync
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int j = 0; j < NJ; ++j) run(J[j]);
      cudaDeviceSynchronize();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float conc; cudaEventElapsedTime(&conc, e0, e1);
      // threaded: one host thread per job
      cudaDeviceSynchronize();
      auto t0 = std::chrono::steady_clock::now();
      { std::vector<std::thread> th; for (int j = 0; j < NJ; ++j) th.emplace_back([&, j]() { run(J[j]); cudaStreamSynchronize(J[j].s); }); for (auto& x : th) x.join(); }
      auto t1 = std::chrono::steady_clock::now();
      double thr = std::chrono::duration<double, std::milli>(t1 - t0).count();
      printf("{\"threaded_ms\":%.2f}\n", thr);
      printf("{\"m\":%d,\"n\":%d,\"algo\":%d,\"jobs\":%d,\"ms_sequential\":%.2f,\"ms_issue_all\":%.2f}\n", m, n, algo, NJ, seq, conc);
      for (int j = 0; j < NJ; ++j) { Job& b = J[j]; cudaFree(b.A); cudaFree(b.A0); cudaFree(b.S); cudaFree(b.U); cudaFree(b.V); cudaFree(b.work); cudaFree(b.info); free(b.hbuf); cusolverDnDestroy(b.h); }
    }
  }
}
