// kernels.cu -- HBM-bound helper kernels of libctm: site-leg permutation, Frobenius
// norms (sum of squares), normalise-and-commit, finiteness scan.  Grid sizes are
// multiples of the 148 SMs (grid-stride loops).
#include "ctm_internal.h"
#include "pdl.cuh"

namespace ctm {
namespace {

constexpr int kSMs = 148;

struct PermArgs {
  int rank;
  int dst_ext[8];
  long long src_str[8];   // source stride of each destination axis
};

__global__ void permute_kernel(const double* __restrict__ src, double* __restrict__ dst, long long n,
                               PermArgs a) {
  CTM_PDL_WAIT();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i, off = 0;
    for (int j = a.rank - 1; j >= 0; --j) {
      long long q = r / a.dst_ext[j];
      off += (r - q * a.dst_ext[j]) * a.src_str[j];
      r = q;
    }
    dst[i] = src[off];
  }
}

__global__ void zero_kernel(double* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

struct Parts {
  int n[8];
};

struct Multi {
  const double* src[8];
  double* dst[8];
  long long n[8];
};

// blockIdx.y = tensor; out[y] += sum of squares
__global__ void sumsq_kernel(Multi m, double* out) {
  CTM_PDL_WAIT();
  const int y = blockIdx.y;
  const double* __restrict__ s = m.src[y];
  const long long n = m.n[y];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = s[i];
    acc += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(out + y, v);
  }
}

// dst[y][i] = src[y][i] / ||src[y]||_F   (Frobenius normalisation, reading R13); the norm
// is the in-order sum of the per-tile partials written by the producing GEMM (deterministic).
__global__ void scale_commit_kernel(Multi m, const double* __restrict__ ss, Parts parts) {
  CTM_PDL_WAIT();
  const int y = blockIdx.y;
  __shared__ double inv_s;
  if (threadIdx.x < 32) {
    // warp 0 sums the partials in a fixed order (lane-strided, then a fixed xor tree): deterministic,
    // and 32x shorter than one thread's serial chain of global loads
    const double* p = ss + (size_t)y * CTM_SS_SLOTS;
    double acc = 0.0;
    for (int j = threadIdx.x; j < parts.n[y]; j += 32) acc += p[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) inv_s = 1.0 / sqrt(acc);
  }
  __syncthreads();
  const double inv = inv_s;
  const double* __restrict__ s = m.src[y];
  double* __restrict__ d = m.dst[y];
  const long long n = m.n[y];
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((((uintptr_t)s | (uintptr_t)d) & 15) == 0) {
    // 16-byte vector path for the even head, scalar tail
    const long long n2 = n >> 1;
    const double2* __restrict__ s2 = reinterpret_cast<const double2*>(s);
    double2* __restrict__ d2 = reinterpret_cast<double2*>(d);
    for (long long i = i0; i < n2; i += stride) {
      double2 v = s2[i];
      v.x *= inv;
      v.y *= inv;
      d2[i] = v;
    }
    i0 += 2 * n2;
    if (i0 < n && i0 == 2 * n2) d[i0] = s[i0] * inv;
    return;
  }
  for (long long i = i0; i < n; i += stride) d[i] = s[i] * inv;
}

__global__ void nonfinite_kernel(const double* __restrict__ p, long long n, int* cnt) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad += !isfinite(p[i]);
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(cnt, bad);
}

__global__ void abs_kernel(const double* __restrict__ s, double* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = fabs(s[i]);
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n, double* out) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(out, v);
  }
}

// One block: m = (rho + rho^T)/2 as (sA sB) x (tA tB); m /= Tr m; e = sum_ij m_ij h_ji.
__global__ void rho_finish_kernel(const double* __restrict__ rho, const double* __restrict__ hop, int n,
                                  double* __restrict__ rho_out, double* __restrict__ e_out) {
  __shared__ double tr;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += rho[i * n + i];
    tr = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double m = 0.5 * (rho[i * n + j] + rho[j * n + i]) / tr;
        e += m * hop[j * n + i];
        if (rho_out) rho_out[i * n + j] = m;
      }
    *e_out = e;
  }
}

// rho(sA, sB, tA, tB), d = 2: partial traces -> rho_A, rho_B (symmetrised, unit trace),
// out = (<Sx>_A, <Sz>_A, <Sx>_B, <Sz>_B) with S = sigma / 2.
__global__ void site_spins_kernel(const double* __restrict__ rho, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double rA[2][2] = {}, rB[2][2] = {};
  for (int s = 0; s < 2; ++s)
    for (int t = 0; t < 2; ++t)
      for (int u = 0; u < 2; ++u) {
        rA[s][t] += rho[((s * 2 + u) * 2 + t) * 2 + u];
        rB[s][t] += rho[((u * 2 + s) * 2 + u) * 2 + t];
      }
  const double (*rs[2])[2] = {rA, rB};
  for (int i = 0; i < 2; ++i) {
    const double (*r)[2] = rs[i];
    const double tr = r[0][0] + r[1][1];
    out[2 * i] = 0.5 * (r[0][1] + r[1][0]) / tr;        // Tr(rho_sym sigma_x) / 2
    out[2 * i + 1] = 0.5 * (r[0][0] - r[1][1]) / tr;    // Tr(rho sigma_z) / 2
  }
  // staggered magnetisation m_s = (|<S>_A| + |<S>_B|) / 2 (reading R23)
  out[4] = 0.5 * (sqrt(out[0] * out[0] + out[1] * out[1]) + sqrt(out[2] * out[2] + out[3] * out[3]));
}

int grid_for(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  long long cap = kSMs * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

void permute(Handle& h, const double* src, const std::vector<int>& ext, const std::vector<int>& perm,
             double* dst) {
  if (h.dry) return;
  int r = (int)ext.size();
  if (r > 8 || (int)perm.size() != r) throw Error(CTM_E_ARG, "permute: bad rank");
  std::vector<long long> st(r);
  long long acc = 1;
  for (int i = r - 1; i >= 0; --i) {
    st[i] = acc;
    acc *= ext[i];
  }
  PermArgs a{};
  a.rank = r;
  for (int j = 0; j < r; ++j) {
    a.dst_ext[j] = ext[perm[j]];
    a.src_str[j] = st[perm[j]];
  }
  launch_k(permute_kernel, dim3(grid_for(acc)), dim3(256), 0, h.stream, src, dst, acc, a);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void zero(Handle& h, double* p, size_t n) {
  if (h.dry || n == 0) return;
  zero_kernel<<<grid_for((long long)n), 256, 0, h.stream>>>(p, (long long)n);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void sumsq(Handle& h, const std::vector<const double*>& srcs, const std::vector<size_t>& ns,
           double* out) {
  if (h.dry) return;
  Multi m{};
  long long mx = 0;
  for (size_t i = 0; i < srcs.size(); ++i) {
    m.src[i] = srcs[i];
    m.n[i] = (long long)ns[i];
    mx = std::max(mx, m.n[i]);
  }
  dim3 grid(std::min(grid_for(mx), kSMs * 2), (unsigned)srcs.size());
  launch_k(sumsq_kernel, dim3(grid), dim3(256), 0, h.stream, m, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void scale_commit(Handle& h, const std::vector<const double*>& srcs, const std::vector<double*>& dsts,
                  const std::vector<size_t>& ns, const double* ss, const std::vector<int>& nparts) {
  if (h.dry) return;
  Parts parts{};
  for (size_t i = 0; i < nparts.size(); ++i) parts.n[i] = nparts[i];
  Multi m{};
  long long mx = 0;
  for (size_t i = 0; i < srcs.size(); ++i) {
    m.src[i] = srcs[i];
    m.dst[i] = dsts[i];
    m.n[i] = (long long)ns[i];
    mx = std::max(mx, m.n[i]);
  }
  dim3 grid(std::min(grid_for(mx), kSMs * 2), (unsigned)srcs.size());
  launch_k(scale_commit_kernel, dim3(grid), dim3(256), 0, h.stream, m, (const double*)ss, parts);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void nonfinite_count(Handle& h, const double* p, size_t n, int* dev_count) {
  if (h.dry) return;
  nonfinite_kernel<<<grid_for((long long)n), 256, 0, h.stream>>>(p, (long long)n, dev_count);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void rho_finish(Handle& h, const double* rho, const double* hop, int d, double* rho_out, double* e_dev) {
  if (h.dry) return;
  rho_finish_kernel<<<1, 32, 0, h.stream>>>(rho, hop, d * d, rho_out, e_dev);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void site_spins(Handle& h, const double* rho, double* out) {
  if (h.dry) return;
  site_spins_kernel<<<1, 32, 0, h.stream>>>(rho, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void dot(Handle& h, const double* a, const double* b, size_t n, double* out) {
  if (h.dry) return;
  CTM_CUDA(cudaMemsetAsync(out, 0, sizeof(double), h.stream));
  dot_kernel<<<std::min(grid_for((long long)n), kSMs * 2), 256, 0, h.stream>>>(a, b, (long long)n, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

void abs_copy(Handle& h, const double* src, double* dst, size_t n) {
  if (h.dry) return;
  abs_kernel<<<grid_for((long long)n), 256, 0, h.stream>>>(src, dst, (long long)n);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

}  // namespace ctm
