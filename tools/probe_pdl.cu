// Programmatic dependent launch probe: a chain of N dependent small kernels (each reads
// the previous one's output) launched plainly vs with cudaLaunchAttributeProgrammaticStreamSerialization
// (the kernel waits with griddepcontrol.wait before touching memory and triggers its dependents
// at entry).  Reports us per kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_pdl.cu -o probe_pdl
#include <cstdio>
__global__ void step(const double* __restrict__ in, double* __restrict__ out, int n, int work) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = in[i];
    for (int k = 0; k < work; ++k) v = fma(v, 1.0000001, 1e-9);
    out[i] = v;
  }
}
int main() {
  const int n = 1 << 16, N = 400;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int work : {1, 64, 512}) {
    for (int grid : {1, 148}) {
      for (int pdl = 0; pdl < 2; ++pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = pdl ? at : nullptr;
        cfg.numAttrs = pdl ? 1 : 0;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0, s);
          for (int i = 0; i < N; ++i)
            cudaLaunchKernelEx(&cfg, step, (const double*)(i & 1 ? b : a), (i & 1 ? a : b), n, work);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"work\":%d,\"grid\":%d,\"pdl\":%d,\"us_per_kernel\":%.2f,\"err\":\"%s\"}\n", work, grid, pdl,
               1e3 * ms / N, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
