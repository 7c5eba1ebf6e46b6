// Microbenchmark + self-check of the isometry-solver kernels (iso_kernels.cuh) at the C4
// sizes: Cholesky of an SPD l x l Gram, row-parallel triangular solve on 1024 x l, and the
// one-sided Jacobi SVD of an l x l matrix (full sweeps forced and to convergence).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o tools/bench_iso_kernels
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "iso_kernels.cuh"

using namespace ctm::isok;
#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("{\"err\":\"%s\",\"line\":%d}\n", cudaGetErrorString(e_), __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

static double urand(unsigned long long& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 160;
  const int m = 1024;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  unsigned long long seed = 12345;
  // Y (m x n) random, S = Y^T Y (host)
  std::vector<double> Y((size_t)m * n), S((size_t)n * n, 0.0);
  for (auto& v : Y) v = urand(seed);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double t = 0;
      for (int i = 0; i < m; ++i) t += Y[(size_t)i * n + a] * Y[(size_t)i * n + b];
      S[(size_t)a * n + b] = t;
    }
  double *dS, *dR, *drd, *dY, *dX, *dU, *dSig;
  int* dst;
  CK(cudaMalloc(&dS, 8ull * n * n));
  CK(cudaMalloc(&dR, 8ull * n * n));
  CK(cudaMalloc(&drd, 8ull * n));
  CK(cudaMalloc(&dY, 8ull * m * n));
  CK(cudaMalloc(&dX, 8ull * n * n));
  CK(cudaMalloc(&dU, 8ull * n * n));
  CK(cudaMalloc(&dSig, 8ull * n));
  CK(cudaMalloc(&dst, 64));
  double* dDinv;
  CK(cudaMalloc(&dDinv, 8ull * rpk_size(LMAX)));
  CK(cudaFuncSetAttribute(trsm_rows_kernel<(LMAX + 31) / 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * rpk_size(LMAX))));
  CK(cudaMemset(dst, 0, 64));
  CK(cudaMemcpy(dS, S.data(), 8ull * n * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dY, Y.data(), 8ull * m * n, cudaMemcpyHostToDevice));
  const size_t big = (size_t)LMAX * (LMAX + 1) * sizeof(double);
  CK(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_smem_bytes(LMAX)));
  CK(cudaFuncSetAttribute(jacobi_lsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * LMAX * (LMAX + 1))));
  auto timeit = [&](auto f, int reps) {
    f();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return 1e3 * ms / reps;
  };
  int st[4];
  if (n <= LMAX) {   // one-CTA Cholesky + trsm at n <= LMAX
  // ---- Cholesky
  const size_t smem_c = chol_smem_bytes(n);
  double us_chol = timeit([&]() { chol_kernel<<<1, CHOL_THREADS, smem_c>>>(dS, n, 0.0, dR, drd, dst, 0.0, nullptr, nullptr, dDinv); }, 20);
  std::vector<double> R((size_t)n * n);
  CK(cudaMemcpy(R.data(), dR, 8ull * n * n, cudaMemcpyDeviceToHost));
  double err = 0, nrm = 0;
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) {
      double t = 0;
      for (int i = 0; i <= a; ++i) t += R[(size_t)i * n + a] * R[(size_t)i * n + b];
      err = std::max(err, std::fabs(t - S[(size_t)a * n + b]));
      nrm = std::max(nrm, std::fabs(S[(size_t)a * n + b]));
    }
  CK(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
#ifdef CTM_CHOL_PROF
  {
    long long pr[64];
    CK(cudaMemcpyFromSymbol(pr, chol_prof, sizeof(pr)));
    printf("{\"chol_phase_cycles\": {");
    long long prev = pr[0];
    for (int b = 0; 32 * b < n; ++b) {   // stamps 1 + 2b: panel + look-ahead done; 2 + 2b: diag || trailing done
      printf("\"b%d_panel_la\": %lld, \"b%d_diag_trail\": %lld, ", b, pr[1 + 2 * b] - prev, b, pr[2 + 2 * b] - pr[1 + 2 * b]);
      prev = pr[2 + 2 * b];
    }
    printf("\"tail\": %lld, \"store\": %lld, \"pack\": %lld, \"dinv\": %lld}}\n", pr[40] - prev, pr[41] - pr[40], pr[43] - pr[41], pr[42] - pr[43]);
  }
#endif
  printf("{\"kernel\":\"chol\",\"n\":%d,\"us\":%.1f,\"rel_err\":%.3e,\"status\":%d}\n", n, us_chol, err / nrm, st[0]);
  // ---- triangular solve Y R^{-1}: then Q^T Q should be I
  double us_trsm = timeit([&]() {
    CK(cudaMemcpyAsync(dY, Y.data(), 0, cudaMemcpyHostToDevice));
    trsm_rows_kernel<(LMAX + 31) / 32><<<std::min(148, (m + 7) / 8), 256, 8 * rpk_size(n)>>>(dY, m, n, dDinv);
  }, 1);
  CK(cudaMemcpy(dY, Y.data(), 8ull * m * n, cudaMemcpyHostToDevice));
  trsm_rows_kernel<(LMAX + 31) / 32><<<std::min(148, (m + 7) / 8), 256, 8 * rpk_size(n)>>>(dY, m, n, dDinv);
  CK(cudaGetLastError());
  std::vector<double> Q((size_t)m * n);
  CK(cudaMemcpy(Q.data(), dY, 8ull * m * n, cudaMemcpyDeviceToHost));
  double orth = 0;
  for (int a = 0; a < n; a += 7)
    for (int b = 0; b < n; b += 5) {
      double t = 0;
      for (int i = 0; i < m; ++i) t += Q[(size_t)i * n + a] * Q[(size_t)i * n + b];
      orth = std::max(orth, std::fabs(t - (a == b ? 1.0 : 0.0)));
    }
  double us_trsm2 = timeit([&]() { trsm_rows_kernel<(LMAX + 31) / 32><<<std::min(148, (m + 7) / 8), 256, 8 * rpk_size(n)>>>(dY, m, n, dDinv); }, 20);
  printf("{\"kernel\":\"trsm_rows\",\"m\":%d,\"n\":%d,\"us\":%.1f,\"orth_err\":%.3e}\n", m, n, us_trsm2, orth);
  (void)us_trsm;
  }
  // ---- Jacobi on a random n x n matrix (X = R^T with trans = 1 means rows of R)
  std::vector<double> X((size_t)n * n);
  for (auto& v : X) v = urand(seed);
  CK(cudaMemcpy(dX, X.data(), 8ull * n * n, cudaMemcpyHostToDevice));
  const size_t smem_j = (size_t)n * (n + 1) * sizeof(double);
  using J2 = JacCfg<2, 8, LMAX>;
  using J4 = JacCfg<8, 4, LMAX_BIG>;
  CK(cudaFuncSetAttribute(jacobi_cluster_kernel<2, 8, LMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J2::SMEM));
  using J1 = JacCfg<1, 8, 128>;
  CK(cudaFuncSetAttribute(jacobi_cluster_kernel<1, 8, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J1::SMEM));
  CK(cudaFuncSetAttribute(jacobi_cluster_kernel<8, 4, LMAX_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J4::SMEM));
  for (int sweeps : {1, 60}) {
    CK(cudaMemset(dst, 0, 64));
    double us = timeit([&]() {
      if (n > LMAX) jacobi_cluster_kernel<8, 4, LMAX_BIG><<<8, J4::THREADS, J4::SMEM>>>(dX, n, 1, n, dU, dSig, dst + 1, sweeps, 1e-14);
      else if (n > 128) jacobi_cluster_kernel<2, 8, LMAX><<<2, J2::THREADS, J2::SMEM>>>(dX, n, 1, n, dU, dSig, dst + 1, sweeps, 1e-14);
      else jacobi_cluster_kernel<1, 8, 128><<<1, J1::THREADS, J1::SMEM>>>(dX, n, 1, n, dU, dSig, dst + 1, sweeps, 1e-14);
    }, 3);
    CK(cudaGetLastError());
    CK(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
    std::vector<double> U((size_t)n * n), sig(n);
    CK(cudaMemcpy(U.data(), dU, 8ull * n * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sig.data(), dSig, 8ull * n, cudaMemcpyDeviceToHost));
    double o = 0;
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        double t = 0;
        for (int i = 0; i < n; ++i) t += U[(size_t)i * n + a] * U[(size_t)i * n + b];
        o = std::max(o, std::fabs(t - (a == b ? 1.0 : 0.0)));
      }
    printf("{\"kernel\":\"jacobi_cluster\",\"n\":%d,\"max_sweeps\":%d,\"sweeps\":%d,\"us\":%.1f,\"us_per_sweep\":%.1f,\"orth_err\":%.3e,\"s0\":%.6f,\"slast\":%.3e}\n",
           n, sweeps, st[2], us, us / std::max(1, st[2]), o, sig[0], sig[n - 1]);
  }
  for (int sweeps : {1, 60}) {
    if (n > LMAX) break;   // one-CTA shared-memory Jacobi: n <= LMAX only
    for (double tol : {1e-14, 1e-8}) {
      if (sweeps == 1 && tol > 1e-10) continue;
      CK(cudaMemset(dst, 0, 64));
      double us = timeit([&]() { jacobi_lsv_kernel<<<1, jacobi_threads(n), smem_j>>>(dX, n, 1, n, dU, dSig, dst + 1, sweeps, tol); }, 3);
      CK(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
      std::vector<double> U((size_t)n * n), sig(n);
      CK(cudaMemcpy(U.data(), dU, 8ull * n * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(sig.data(), dSig, 8ull * n, cudaMemcpyDeviceToHost));
      // check: U^T U = I and X^T (rows of X) ... left singular vectors of X^T: X^T = U S V^T
      double o = 0;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
          double t = 0;
          for (int i = 0; i < n; ++i) t += U[(size_t)i * n + a] * U[(size_t)i * n + b];
          o = std::max(o, std::fabs(t - (a == b ? 1.0 : 0.0)));
        }
      printf("{\"kernel\":\"jacobi\",\"n\":%d,\"max_sweeps\":%d,\"tol\":%.0e,\"sweeps\":%d,\"us\":%.1f,\"us_per_sweep\":%.1f,"
             "\"orth_err\":%.3e,\"s0\":%.6f,\"slast\":%.3e}\n",
             n, sweeps, tol, st[2], us, us / std::max(1, st[2]), o, sig[0], sig[n - 1]);
    }
  }
  return 0;
}
