// Probe: DMMA.8x8x4 throughput vs resident warps per SM (one CTA per SM, 148 CTAs),
// with NACC independent accumulator chains per warp.  Sizing input for tc_gemm's tiles.
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void dmma_occ(double* out, int iters) {
  extern __shared__ double sm[];
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[NACC][2];
#pragma unroll
  for (int t = 0; t < NACC; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < NACC; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NACC; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
void run(int warps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000 / NACC * 8;
  size_t smem = 150 * 1024;  // force 1 CTA per SM
  cudaFuncSetAttribute(dmma_occ<NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dmma_occ<NACC><<<148, warps * 32, smem>>>(out, 10);
  cudaEventRecord(e0);
  dmma_occ<NACC><<<148, warps * 32, smem>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * NACC * (double)iters * 148 * warps;
  printf("{\"warps_per_sm\":%d,\"nacc\":%d,\"tflops\":%.2f}\n", warps, NACC, fl / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 148 * 1024 * 8);
  for (int w : {4, 8, 12, 16, 32}) { run<4>(w, out); run<8>(w, out); run<16>(w, out); run<32>(w, out); }
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
