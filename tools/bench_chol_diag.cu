// Cycle count of the Cholesky kernel's 32 x 32 diagonal-block factorisation (chol_kernel's
// diag_block, one warp, lane = column) in isolation, with and without the other warps of the
// CTA busy on FP64 FMAs (the look-ahead overlaps it with the trailing update), and of a variant
// whose next pivot is formed on its own lane (one shuffle fewer on the dependent chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/bench_chol_diag.cu -o bcd
#include <cmath>
#include <cstdio>
#include <vector>

constexpr double DMIN = 2.2250738585072014e-308;
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y * y, 1.0);
  return fma(fma(e, 0.375, 0.5), y * e, y);
}

template <int VAR>
__global__ void diag_kernel(const double* S, double* R, long long* cyc, int busy, const int* repl, double repl_tol,
                            int LD) {
  extern __shared__ double A[];   // LD x LD, block at (0, 0)
  __shared__ double dorig[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * LD; i += blockDim.x) A[i] = 0.0;
  __syncthreads();
  for (int i = tid; i < 32 * 32; i += blockDim.x) A[(i / 32) * LD + i % 32] = S[i];
  if (tid < 32) dorig[tid] = S[tid * 33];
  __syncthreads();
  const int kb = 0;
  if (warp == 0) {
    long long t0 = clock64();
    double col[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) col[r] = r <= lane ? A[(kb + r) * LD + kb + lane] : 0.0;
    int badj = 0;
    double my_inv = 1.0;
    double d = __shfl_sync(0xffffffffu, col[0], 0);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool fin = isfinite(d);
      const bool dep = repl != nullptr && fin && !(d > repl_tol * dorig[kb + j]);
      if (!dep && !(d >= DMIN && fin) && badj == 0) badj = kb + j + 1;
      const bool ok = !dep && d >= DMIN && fin;
      const double inv = rsqrt_nr(ok ? d : 1.0);
      const double rj = lane == j ? (ok ? d * inv : 1.0) : (dep ? 0.0 : col[j] * inv);
      if (lane >= j) A[(kb + j) * LD + kb + lane] = rj;
      if (j + 1 < 32) {
        const double rn = __shfl_sync(0xffffffffu, rj, j + 1);
        if (VAR == 1) {
          const double dl = fma(-rj, rj, col[j + 1]);   // lane j+1: its own R[j][j+1], no shuffle
          col[j + 1] = fma(-rn, rj, col[j + 1]);
          d = __shfl_sync(0xffffffffu, dl, j + 1);
        } else {
          col[j + 1] = fma(-rn, rj, col[j + 1]);
          d = __shfl_sync(0xffffffffu, col[j + 1], j + 1);
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = j + 2; r < 32; ++r) col[r] = fma(-A[(kb + j) * LD + kb + r], rj, col[r]);
      if (lane == j) my_inv = inv;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    R[lane] = my_inv + badj;
  } else if (busy > 0 || (busy < 0 && warp != 4)) {
    const int nb = busy > 0 ? busy : -busy;
    // FMA-heavy filler like the trailing update (4 x 4 tiles from shared memory)
    double acc[4][4] = {};
    for (int it = 0; it < nb; ++it)
#pragma unroll 4
      for (int i = 0; i < 32; ++i) {
        const double* row = A + i * LD + 32;
        const double2 a = *reinterpret_cast<const double2*>(row + (tid & 15) * 4);
        const double2 b = *reinterpret_cast<const double2*>(row + (tid & 15) * 4 + 2);
        const double ar[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(ar[u], ar[v], acc[u][v]);
      }
    double s = 0;
    for (int u = 0; u < 4; ++u)
      for (int v = 0; v < 4; ++v) s += acc[u][v];
    if (s == 12345.0) R[64 + tid] = s;
  }
  __syncthreads();
  for (int i = tid; i < 32 * 32; i += blockDim.x) R[128 + i] = A[(i / 32) * LD + i % 32];
}

int main() {
  std::vector<double> S(32 * 32), X(32 * 64);
  unsigned long long s = 7;
  for (auto& v : X) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    v = ((s >> 11) * (1.0 / 9007199254740992.0)) * 2 - 1;
  }
  for (int a = 0; a < 32; ++a)
    for (int b = 0; b < 32; ++b) {
      double t = 0;
      for (int i = 0; i < 64; ++i) t += X[a * 64 + i] * X[b * 64 + i];
      S[a * 32 + b] = t;
    }
  double *dS, *dR;
  long long* dc;
  int* drepl;
  cudaMalloc(&dS, 8 * 1024);
  cudaMalloc(&dR, 8 * 4096);
  cudaMalloc(&dc, 64);
  cudaMalloc(&drepl, 4 * 64);
  cudaMemcpy(dS, S.data(), 8 * 1024, cudaMemcpyHostToDevice);
  const int LD = 160;
  const size_t smem = 8 * 32 * LD;
  cudaFuncSetAttribute(diag_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(diag_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int var = 0; var < 2; ++var)
    for (int threads : {32, 256})
      for (int busy : {0, 4, -4}) {
        if (threads == 32 && busy) continue;
        long long best = 1LL << 60;
        std::vector<double> Rh(128 + 1024);
        for (int rep = 0; rep < 5; ++rep) {
          if (var == 0) diag_kernel<0><<<1, threads, smem>>>(dS, dR, dc, busy, drepl, 1e-13, LD);
          else diag_kernel<1><<<1, threads, smem>>>(dS, dR, dc, busy, drepl, 1e-13, LD);
          long long c = 0;
          cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
          best = c < best ? c : best;
        }
        cudaMemcpy(Rh.data(), dR, 8 * (128 + 1024), cudaMemcpyDeviceToHost);
        // check R^T R = S
        double err = 0;
        for (int a = 0; a < 32; ++a)
          for (int b = a; b < 32; ++b) {
            double t = 0;
            for (int i = 0; i <= a; ++i) t += Rh[128 + i * 32 + a] * Rh[128 + i * 32 + b];
            err = fmax(err, fabs(t - S[a * 32 + b]) / fabs(S[a * 32 + a]));
          }
        printf("{\"variant\":%d,\"threads\":%d,\"busy\":%d,\"cycles\":%lld,\"cycles_per_col\":%.0f,\"rel_err\":%.2e,\"err\":\"%s\"}\n",
               var, threads, busy, best, best / 32.0, err, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
