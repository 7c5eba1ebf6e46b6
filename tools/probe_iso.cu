// Probe: latency of the dense building blocks an isometry solver could use at the
// C4 / C5 sizes: cuSOLVER potrf / geqrf+orgqr / syevd / syevj /
// XsyevBatched / gesvdaStridedBatched and cuBLAS trsm / dgemm.  One stream, CUDA events,
// median of 7 after 2 warm-ups.  Output: one JSON line per measurement.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/probe_iso.cu -lcusolver -lcublas -o tools/probe_iso
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>
#define CK(x)                                                                       \
  do {                                                                              \
    auto e_ = (x);                                                                  \
    if ((int)e_) {                                                                  \
      printf("{\"err\":%d,\"at\":\"%s:%d\"}\n", (int)e_, __FILE__, __LINE__);      \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

static cudaStream_t st;
static cudaEvent_t e0, e1;

double timeit(const std::function<void()>& f) {
  std::vector<float> v;
  for (int i = 0; i < 9; ++i) {
    CK(cudaEventRecord(e0, st));
    f();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (i >= 2) v.push_back(ms);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

__global__ void fill_spd(double* A, int n, int seed) {   // A = I*n + small symmetric noise
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * n) return;
  int r = i / n, c = i % n;
  unsigned h = (unsigned)(min(r, c) * 7919 + max(r, c) * 104729 + seed * 15485863);
  h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
  A[i] = (r == c ? (double)n : 0.0) + ((h & 0xffff) / 65536.0 - 0.5);
}
__global__ void fill_rand(double* A, long long n, int seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned h = (unsigned)(i * 2654435761u + seed * 97u);
  h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
  A[i] = (h & 0xffffff) / 16777216.0 - 0.5;
}

int main() {
  CK(cudaStreamCreate(&st));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  cusolverDnHandle_t sh;
  cusolverDnParams_t sp;
  cublasHandle_t bh;
  CK(cusolverDnCreate(&sh));
  CK(cusolverDnCreateParams(&sp));
  CK(cusolverDnSetStream(sh, st));
  CK(cublasCreate(&bh));
  CK(cublasSetStream(bh, st));
  double *A, *A0, *W, *work, *B, *Cm, *tau;
  int* info;
  const size_t big = 2560ull * 2560;
  CK(cudaMalloc(&A, 8 * big * 4));
  CK(cudaMalloc(&A0, 8 * big * 4));
  CK(cudaMalloc(&B, 8 * big));
  CK(cudaMalloc(&Cm, 8 * big));
  CK(cudaMalloc(&W, 8 * 4 * 2560));
  CK(cudaMalloc(&tau, 8 * 4 * 2560));
  CK(cudaMalloc(&work, 8ull << 28));
  CK(cudaMalloc(&info, 64));
  std::vector<char> hbuf(1 << 26);
  fill_rand<<<(unsigned)((big * 4 + 255) / 256), 256, 0, st>>>(B, big, 3);
  fill_rand<<<(unsigned)((big + 255) / 256), 256, 0, st>>>(Cm, big, 5);

  // potrf
  for (int n : {128, 160, 192, 256, 320, 512}) {
    fill_spd<<<(n * n + 255) / 256, 256, 0, st>>>(A0, n, 1);
    size_t dws, hws;
    CK(cusolverDnXpotrf_bufferSize(sh, sp, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n, CUDA_R_64F, &dws, &hws));
    double ms = timeit([&]() {
      cudaMemcpyAsync(A, A0, 8ull * n * n, cudaMemcpyDeviceToDevice, st);
      CK(cusolverDnXpotrf(sh, sp, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n, CUDA_R_64F, work, dws, hbuf.data(), hws, info));
    });
    printf("{\"op\":\"potrf\",\"n\":%d,\"ms\":%.4f}\n", n, ms);
    // trsm: Y (m x n, col-major) <- Y R^{-1}
    for (int m : {1024, 2560}) {
      double one = 1.0;
      double ms2 = timeit([&]() {
        CK(cublasDtrsm(bh, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, n, &one, A, n, B, m));
      });
      printf("{\"op\":\"trsm_right\",\"m\":%d,\"n\":%d,\"ms\":%.4f}\n", m, n, ms2);
    }
  }
  // syevd / syevj on small symmetric matrices
  for (int n : {128, 160, 192, 256, 320, 512, 1024}) {
    fill_spd<<<(n * n + 255) / 256, 256, 0, st>>>(A0, n, 2);
    size_t dws, hws;
    CK(cusolverDnXsyevd_bufferSize(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n,
                                   CUDA_R_64F, W, CUDA_R_64F, &dws, &hws));
    double ms = timeit([&]() {
      cudaMemcpyAsync(A, A0, 8ull * n * n, cudaMemcpyDeviceToDevice, st);
      CK(cusolverDnXsyevd(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n, CUDA_R_64F, W,
                          CUDA_R_64F, work, dws, hbuf.data(), hws, info));
    });
    printf("{\"op\":\"syevd\",\"n\":%d,\"ms\":%.4f}\n", n, ms);
    syevjInfo_t ji;
    CK(cusolverDnCreateSyevjInfo(&ji));
    int lw;
    CK(cusolverDnDsyevj_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, n, W, &lw, ji));
    double ms2 = timeit([&]() {
      cudaMemcpyAsync(A, A0, 8ull * n * n, cudaMemcpyDeviceToDevice, st);
      CK(cusolverDnDsyevj(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, n, W, work, lw, info, ji));
    });
    printf("{\"op\":\"syevj\",\"n\":%d,\"ms\":%.4f}\n", n, ms2);
    for (int batch : {1, 4}) {
      size_t d2, h2;
      if (cusolverDnXsyevBatched_bufferSize(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n,
                                            CUDA_R_64F, W, CUDA_R_64F, &d2, &h2, batch) != CUSOLVER_STATUS_SUCCESS) {
        printf("{\"op\":\"XsyevBatched\",\"n\":%d,\"batch\":%d,\"unsupported\":1}\n", n, batch);
        continue;
      }
      for (int b = 0; b < batch; ++b)
        cudaMemcpyAsync(A0 + (size_t)b * n * n, A0, 8ull * n * n, cudaMemcpyDeviceToDevice, st);
      double ms3 = timeit([&]() {
        cudaMemcpyAsync(A, A0, 8ull * n * n * batch, cudaMemcpyDeviceToDevice, st);
        CK(cusolverDnXsyevBatched(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, A, n,
                                  CUDA_R_64F, W, CUDA_R_64F, work, d2, hbuf.data(), h2, info, batch));
      });
      printf("{\"op\":\"XsyevBatched\",\"n\":%d,\"batch\":%d,\"ms\":%.4f}\n", n, batch, ms3);
    }
  }
  // syevdx top-k of 1024 / 2560
  for (int n : {1024, 2560}) {
    fill_spd<<<(n * n + 255) / 256, 256, 0, st>>>(A0, n, 4);
    for (int k : {128, 256}) {
      if (n == 2560) k *= 2;
      size_t dws, hws;
      int64_t h_meig;
      CK(cusolverDnXsyevdx_bufferSize(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_UPPER, n,
                                      CUDA_R_64F, A, n, nullptr, nullptr, n - k + 1, n, &h_meig, CUDA_R_64F, W,
                                      CUDA_R_64F, &dws, &hws));
      double ms = timeit([&]() {
        cudaMemcpyAsync(A, A0, 8ull * n * n, cudaMemcpyDeviceToDevice, st);
        CK(cusolverDnXsyevdx(sh, sp, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F,
                             A, n, nullptr, nullptr, n - k + 1, n, &h_meig, CUDA_R_64F, W, CUDA_R_64F, work, dws,
                             hbuf.data(), hws, info));
      });
      printf("{\"op\":\"syevdx_topk\",\"n\":%d,\"k\":%d,\"ms\":%.4f}\n", n, k, ms);
    }
  }
  // QR of tall-skinny: geqrf + orgqr
  for (int m : {1024, 2560})
    for (int n : {128, 160, 256, 320, 512}) {
      size_t dws, hws;
      CK(cusolverDnXgeqrf_bufferSize(sh, sp, m, n, CUDA_R_64F, A, m, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws));
      int lw;
      CK(cusolverDnDorgqr_bufferSize(sh, m, n, n, A, m, tau, &lw));
      double ms = timeit([&]() {
        cudaMemcpyAsync(A, B, 8ull * m * n, cudaMemcpyDeviceToDevice, st);
        CK(cusolverDnXgeqrf(sh, sp, m, n, CUDA_R_64F, A, m, CUDA_R_64F, tau, CUDA_R_64F, work, dws, hbuf.data(), hws, info));
      });
      double ms2 = timeit([&]() { CK(cusolverDnDorgqr(sh, m, n, n, A, m, tau, work, lw, info)); });
      printf("{\"op\":\"geqrf\",\"m\":%d,\"n\":%d,\"ms\":%.4f,\"orgqr_ms\":%.4f}\n", m, n, ms, ms2);
    }
  // gesvdaStridedBatched tall-skinny (stage 2 shape)
  for (int m : {1024, 2560})
    for (int batch : {1, 4}) {
      int n = m / 8, rank = n;
      long long sA = (long long)m * n, sU = (long long)m * rank, sV = (long long)n * rank;
      int lw;
      CK(cusolverDnDgesvdaStridedBatched_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, rank, m, n, A, m, sA, W, rank, Cm, m,
                                                    sU, A0, n, sV, &lw, batch));
      std::vector<double> res(batch);
      double ms = timeit([&]() {
        cudaMemcpyAsync(A, B, 8ull * m * n * batch, cudaMemcpyDeviceToDevice, st);
        CK(cusolverDnDgesvdaStridedBatched(sh, CUSOLVER_EIG_MODE_VECTOR, rank, m, n, A, m, sA, W, rank, Cm, m, sU, A0, n,
                                           sV, work, lw, info, res.data(), batch));
      });
      printf("{\"op\":\"gesvdaStridedBatched\",\"m\":%d,\"n\":%d,\"batch\":%d,\"ms\":%.4f}\n", m, n, batch, ms);
    }
  // cuBLAS dgemm reference shapes (col-major): (m,n,k)
  int shapes[][3] = {{1024, 256, 1024}, {256, 256, 1024}, {1024, 1024, 1024}, {2560, 512, 2560}, {512, 512, 2560}, {1024, 128, 128}};
  for (auto& s : shapes) {
    double one = 1.0, zero = 0.0;
    double ms = timeit([&]() {
      CK(cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_N, s[0], s[1], s[2], &one, B, s[0], Cm, s[2], &zero, A, s[0]));
    });
    printf("{\"op\":\"dgemm\",\"m\":%d,\"n\":%d,\"k\":%d,\"ms\":%.4f,\"tflops\":%.2f}\n", s[0], s[1], s[2], ms,
           2.0 * s[0] * s[1] * s[2] / (ms * 1e-3) / 1e12);
  }
  printf("{\"done\":1}\n");
  return 0;
}
