// One-off probe: cuSOLVER options for the top-k left singular vectors of an n x n FP64 matrix
// (the chi*D x D*chi isometry SVD of SURVEY 8(a) row a5). Reports time and subspace error
// against Xgesvd (QR-iteration) as reference.  Input to DESIGN.md "SVD choice".
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>
#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); exit(1);} } while (0)

static cusolverDnHandle_t sh; static cublasHandle_t bh; static cusolverDnParams_t prm;
static cudaEvent_t e0, e1;
static float tstart() { cudaEventRecord(e0); return 0; }
static float tstop() { cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms; }

// subspace mismatch: k - ||Ua^T Ub||_F^2  (0 = same span)
static double mismatch(const double* Ua, int lda, const double* Ub, int ldb, int n, int k) {
  double *G; cudaMalloc(&G, sizeof(double) * k * k);
  double one = 1, zero = 0;
  cublasDgemm(bh, CUBLAS_OP_T, CUBLAS_OP_N, k, k, n, &one, Ua, lda, Ub, ldb, &zero, G, k);
  std::vector<double> h(k * k); cudaMemcpy(h.data(), G, sizeof(double) * k * k, cudaMemcpyDeviceToHost);
  double s = 0; for (double x : h) s += x * x; cudaFree(G); return k - s;
}

int main(int argc, char** argv) {
  CK(cusolverDnCreate(&sh)); CK(cublasCreate(&bh)); CK(cusolverDnCreateParams(&prm));
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int n : {1024, 2560}) for (int kind = 0; kind < 2; ++kind) {
    int k = n / 8;
    std::vector<double> h((size_t)n * n);
    srand(1);
    for (size_t i = 0; i < h.size(); ++i) {
      double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
      h[i] = sqrt(-2 * log(u1)) * cos(6.283185307179586 * u2);
    }
    if (kind == 1) for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) h[(size_t)j * n + i] *= exp(-12.0 * j / n) * exp(-6.0 * i / n);
    double *A, *W, *S, *U, *V, *Uref; int* info;
    cudaMalloc(&A, sizeof(double) * n * n); cudaMalloc(&W, sizeof(double) * 4 * n * n);
    cudaMalloc(&S, sizeof(double) * 2 * n); cudaMalloc(&U, sizeof(double) * 4 * n * n); cudaMalloc(&V, sizeof(double) * n * n);
    cudaMalloc(&Uref, sizeof(double) * n * n); cudaMalloc(&info, sizeof(int));
    auto reset = [&]() { cudaMemcpy(A, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice); };
    size_t dws, hws; void* dbuf; std::vector<char> hbuf;
    // reference: Xgesvd jobu=S jobvt=N
    reset();
    CK(cusolverDnXgesvd_bufferSize(sh, prm, 'S', 'N', n, n, CUDA_R_64F, A, n, CUDA_R_64F, S, CUDA_R_64F, Uref, n, CUDA_R_64F, V, n, CUDA_R_64F, &dws, &hws));
    cudaMalloc(&dbuf, dws); hbuf.resize(hws + 1);
    for (int rep = 0; rep < 2; ++rep) { reset(); tstart();
      CK(cusolverDnXgesvd(sh, prm, 'S', 'N', n, n, CUDA_R_64F, A, n, CUDA_R_64F, S, CUDA_R_64F, Uref, n, CUDA_R_64F, V, n, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info));
      float ms = tstop(); if (rep) printf("{\"n\":%d,\"kind\":%d,\"method\":\"Xgesvd_S_N\",\"ms\":%.2f}\n", n, kind, ms); }
    std::vector<double> hs(n); cudaMemcpy(hs.data(), S, sizeof(double) * n, cudaMemcpyDeviceToHost);
    printf("{\"n\":%d,\"kind\":%d,\"s0\":%.3e,\"sk\":%.3e,\"sk1\":%.3e,\"smin\":%.3e}\n", n, kind, hs[0], hs[k - 1], hs[k], hs[n - 1]);
    cudaFree(dbuf);
    // gesvdp
    { reset(); double herr;
      CK(cusolverDnXgesvdp_bufferSize(sh, prm, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, A, n, CUDA_R_64F, S, CUDA_R_64F, U, n, CUDA_R_64F, V, n, CUDA_R_64F, &dws, &hws));
      cudaMalloc(&dbuf, dws); hbuf.resize(hws + 1);
      for (int rep = 0; rep < 2; ++rep) { reset(); tstart();
        CK(cusolverDnXgesvdp(sh, prm, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, A, n, CUDA_R_64F, S, CUDA_R_64F, U, n, CUDA_R_64F, V, n, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info, &herr));
        float ms = tstop(); if (rep) printf("{\"n\":%d,\"kind\":%d,\"method\":\"Xgesvdp\",\"ms\":%.2f,\"mismatch\":%.3e,\"err_sigma\":%.3e}\n", n, kind, ms, mismatch(U, n, Uref, n, n, k), herr); }
      cudaFree(dbuf); }
    // gesvdj tol=eps
    { gesvdjInfo_t gp; cusolverDnCreateGesvdjInfo(&gp); cusolverDnXgesvdjSetTolerance(gp, 2.2e-16); cusolverDnXgesvdjSetMaxSweeps(gp, 100);
      int lw; reset();
      CK(cusolverDnDgesvdj_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, A, n, S, U, n, V, n, &lw, gp));
      cudaMalloc(&dbuf, sizeof(double) * lw);
      for (int rep = 0; rep < 2; ++rep) { reset(); tstart();
        CK(cusolverDnDgesvdj(sh, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, A, n, S, U, n, V, n, (double*)dbuf, lw, info, gp));
        float ms = tstop(); if (rep) printf("{\"n\":%d,\"kind\":%d,\"method\":\"gesvdj\",\"ms\":%.2f,\"mismatch\":%.3e}\n", n, kind, ms, mismatch(U, n, Uref, n, n, k)); }
      cudaFree(dbuf); }
    // augmented symmetric [[0,A],[A^T,0]] syevd -> top-k eigvecs (u;v)/sqrt2
    { int N2 = 2 * n; std::vector<double> aug((size_t)N2 * N2, 0.0);
      for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) { double x = h[(size_t)j * n + i]; aug[(size_t)(n + j) * N2 + i] = x; aug[(size_t)i * N2 + n + j] = x; }
      double* Aug = U;  // 4n^2
      CK(cusolverDnXsyevd_bufferSize(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, N2, CUDA_R_64F, Aug, N2, CUDA_R_64F, S, CUDA_R_64F, &dws, &hws));
      cudaMalloc(&dbuf, dws); hbuf.resize(hws + 1);
      for (int rep = 0; rep < 2; ++rep) { cudaMemcpy(Aug, aug.data(), sizeof(double) * N2 * N2, cudaMemcpyHostToDevice); tstart();
        CK(cusolverDnXsyevd(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, N2, CUDA_R_64F, Aug, N2, CUDA_R_64F, S, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info));
        float ms = tstop();
        // top-k eigvecs are the last k columns; their first n rows are u/sqrt2
        if (rep) { double *Ut = W; cudaMemcpy2D(Ut, sizeof(double) * n, Aug + (size_t)(N2 - k) * N2, sizeof(double) * N2, sizeof(double) * n, k, cudaMemcpyDeviceToDevice);
          double two = 2.0; cublasDscal(bh, n * k, &two, Ut, 1); // |u/sqrt2|^2*2
          printf("{\"n\":%d,\"kind\":%d,\"method\":\"syevd_aug\",\"ms\":%.2f,\"mismatch_scaled\":%.3e}\n", n, kind, ms, mismatch(Ut, n, Uref, n, n, k) ); }
      }
      cudaFree(dbuf); }
    // Gram A A^T + syevd
    { double one = 1, zero = 0; reset();
      CK(cusolverDnXsyevd_bufferSize(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, W, n, CUDA_R_64F, S, CUDA_R_64F, &dws, &hws));
      cudaMalloc(&dbuf, dws); hbuf.resize(hws + 1);
      for (int rep = 0; rep < 2; ++rep) { tstart();
        cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, A, n, A, n, &zero, W, n);
        CK(cusolverDnXsyevd(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, W, n, CUDA_R_64F, S, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info));
        float ms = tstop();
        if (rep) printf("{\"n\":%d,\"kind\":%d,\"method\":\"gram_syevd\",\"ms\":%.2f,\"mismatch\":%.3e}\n", n, kind, ms, mismatch(W + (size_t)(n - k) * n, n, Uref, n, n, k)); }
      cudaFree(dbuf); }
    // Gram + syevdx top-k
    { double one = 1, zero = 0; int64_t meig; double vl = 0, vu = 0;
      CK(cusolverDnXsyevdx_bufferSize(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, W, n, &vl, &vu, n - k + 1, n, &meig, CUDA_R_64F, S, CUDA_R_64F, &dws, &hws));
      cudaMalloc(&dbuf, dws); hbuf.resize(hws + 1);
      for (int rep = 0; rep < 2; ++rep) { tstart();
        cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, A, n, A, n, &zero, W, n);
        CK(cusolverDnXsyevdx(sh, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, W, n, &vl, &vu, n - k + 1, n, &meig, CUDA_R_64F, S, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info));
        float ms = tstop();
        if (rep) printf("{\"n\":%d,\"kind\":%d,\"method\":\"gram_syevdx_topk\",\"ms\":%.2f,\"meig\":%ld,\"mismatch\":%.3e}\n", n, kind, ms, (long)meig, mismatch(W, n, Uref, n, n, k)); }
      cudaFree(dbuf); }
    cudaFree(A); cudaFree(W); cudaFree(S); cudaFree(U); cudaFree(V); cudaFree(Uref); cudaFree(info);
  }
  printf("{\"done\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
