// Host launch throughput of cudaLaunchKernelEx from 1..4 threads, each on its own stream
// (the isometry stage's worker layout): are launches serialised across threads?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe_launch_mt.cu -o /tmp/plm
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

__global__ void tiny_kernel(double* p, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && n < 0) p[0] = 1.0;
}

int main() {
  const int N = 20000;
  double* d;
  cudaMalloc(&d, 8);
  for (int nt : {1, 2, 4}) {
    for (int pdl : {0, 1}) {
      std::vector<cudaStream_t> st(nt);
      for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      cudaDeviceSynchronize();
      auto t0 = std::chrono::high_resolution_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t]() {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(256);
          cfg.stream = st[t];
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = pdl ? at : nullptr;
          cfg.numAttrs = pdl ? 1 : 0;
          for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, tiny_kernel, d, i);
        });
      for (auto& x : th) x.join();
      auto t1 = std::chrono::high_resolution_clock::now();
      cudaDeviceSynchronize();
      auto t2 = std::chrono::high_resolution_clock::now();
      const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
      const double all_us = std::chrono::duration<double, std::micro>(t2 - t0).count();
      printf("{\"threads\": %d, \"pdl\": %d, \"launches\": %d, \"host_us_per_launch\": %.3f, \"wall_us_per_launch\": %.3f}\n",
             nt, pdl, nt * N, host_us / (nt * N), all_us / (nt * N));
      for (auto& s : st) cudaStreamDestroy(s);
    }
  }
}
