// Dependent-chain latencies on this GPU (cycles per op, one warp): DFMA, DMUL, FFMA,
// double SHFL, rsqrt(double), 1/x (double), LDS (double, dependent address), __syncthreads
// (256 and 512 threads).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_latency.cu
#include <cstdio>
constexpr int N = 4096;
__global__ void chains(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  float xf = (float)x;
  long long t0, t1;
  const int lane = threadIdx.x & 31;
  // DFMA
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) xf = fmaf(xf, 1.0000001f, 1e-7f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) * 4;
  double z = x * 0.0 + 2.0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) z = rsqrt(z) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) * 4;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) z = 1.0 / z + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) * 4;
  int idx = (int)z & 1023;
  double acc = 0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) {
    const double v = sm[idx];
    idx = ((int)v + i) & 1023;
    acc += v;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 4;
  t0 = clock64();
  for (int i = 0; i < N / 4; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) * 4;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N / 4; ++i) z = sqrt(z) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) * 4;
  out[threadIdx.x] = x + xf + z + acc;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8 * 1024);
  cudaMallocManaged(&cyc, 8 * 16);
  const char* names[] = {"dfma", "dmul", "ffma", "shfl_f64", "rsqrt_f64", "rcp_f64_div", "lds_f64_dep", "syncthreads", "sqrt_f64"};
  for (int threads : {32, 256, 512}) {
    chains<<<1, threads>>>(out, cyc, 1.0);
    chains<<<1, threads>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    printf("{\"threads\":%d", threads);
    for (int i = 0; i < 9; ++i) printf(",\"%s\":%.1f", names[i], (double)cyc[i] / N);
    printf(",\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
