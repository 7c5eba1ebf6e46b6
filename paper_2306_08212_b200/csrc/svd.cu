// svd.cu -- truncated left singular vectors on the device (
// P:L46 "the unitary matrix U is reshaped ... truncation applied corresponding to the
// largest chi singular values", P:L60 two-stage recipe).  cuSOLVER does the
// factorisation (gesvdp / gesvdj / gesvd, chosen by ctm_params.svd_algo); a libctm
// kernel extracts the kept columns in row-major isometry layout with the sign rule
// (largest-|.| entry of each column positive, ties -> lowest row index).
// There is no CPU fallback: every path runs on the GPU.
#include <cmath>
#include <limits>

#include "ctm_internal.h"
#include "pdl.cuh"

namespace ctm {
namespace {

#define CTM_SOLVER(x)                                                                   \
  do {                                                                                  \
    cusolverStatus_t s_ = (x);                                                          \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                  \
      throw Error(CTM_E_SOLVER, std::string(#x) + " failed with status " + std::to_string((int)s_)); \
  } while (0)

// One block per kept column j: x_i = base[i*rs + j*cs], i < R.
__global__ void extract_signfix_kernel(const double* __restrict__ base, long long rs, long long cs, int R,
                                       int n_keep, double* __restrict__ out) {
  CTM_PDL_WAIT();
  const int j = blockIdx.x;
  const double* col = base + j * cs;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    double a = fabs(col[i * rs]);
    if (a > best || (a == best && i < bi)) {
      best = a;
      bi = i;
    }
  }
  // block arg-max with lowest-index tie break
  for (int o = 16; o > 0; o >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  __shared__ double sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sb[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    best = l < nw ? sb[l] : -1.0;
    bi = l < nw ? si[l] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (l == 0) si[0] = bi < R ? bi : 0;   // all-NaN column: no arg-max (non-finite, reported later)
  }
  __syncthreads();
  const double sgn = col[(long long)si[0] * rs] < 0.0 ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < R; i += blockDim.x) out[(long long)i * n_keep + j] = sgn * col[i * rs];
}

struct Plan {
  bool tall;     // R >= C: factor the column-major copy of mat itself and read U
  int m, n;      // cuSOLVER problem (m >= n)
  int econ;
  int ucols;     // columns of the U (or V) buffer we read from
};

Plan make_plan(int R, int C, int n_keep) {
  Plan p{};
  p.tall = R >= C;
  if (p.tall) {
    p.m = R;
    p.n = C;
    p.econ = n_keep <= C ? 1 : 0;
    p.ucols = p.econ ? C : R;
  } else {
    p.m = C;
    p.n = R;
    p.econ = 1;
    p.ucols = R;
  }
  return p;
}

size_t query_lwork_bytes(Handle& h, const Plan& p, double* A, double* S, double* U, double* V) {
  const int mn = std::min(p.m, p.n);
  const int ldu = p.m, ldv = p.n;
  size_t dws = 0, hws = 0;
  switch (h.prm.svd_algo) {
    case CTM_SVD_GESVDJ: {
      int lw = 0;
      CTM_SOLVER(cusolverDnDgesvdj_bufferSize(h.solver, CUSOLVER_EIG_MODE_VECTOR, p.econ, p.m, p.n, A, p.m, S, U,
                                              ldu, V, ldv, &lw, h.gesvdj_info));
      dws = (size_t)lw * sizeof(double);
      break;
    }
    case CTM_SVD_GESVD: {
      signed char jobu = p.tall ? (p.econ ? 'S' : 'A') : 'N';
      signed char jobvt = p.tall ? 'N' : 'S';
      CTM_SOLVER(cusolverDnXgesvd_bufferSize(h.solver, h.solver_params, jobu, jobvt, p.m, p.n, CUDA_R_64F, A, p.m,
                                             CUDA_R_64F, S, CUDA_R_64F, U, ldu, CUDA_R_64F, V, mn, CUDA_R_64F, &dws,
                                             &hws));
      break;
    }
    default: {
      CTM_SOLVER(cusolverDnXgesvdp_bufferSize(h.solver, h.solver_params, CUSOLVER_EIG_MODE_VECTOR, p.econ, p.m, p.n,
                                              CUDA_R_64F, A, p.m, CUDA_R_64F, S, CUDA_R_64F, U, ldu, CUDA_R_64F, V,
                                              ldv, CUDA_R_64F, &dws, &hws));
      break;
    }
  }
  if (h.host_buf.size() < hws + 16) h.host_buf.resize(hws + 16);
  return dws;
}

void signfix_launch(Handle& h, const double* base, long long rs, long long cs, int R, int n_keep, double* out) {
  launch_k(extract_signfix_kernel, dim3(n_keep), dim3(256), 0, h.stream, base, rs, cs, R, n_keep, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

bool use_gram(const Handle& h, int R, int C, int n_keep) {
  return h.prm.svd_algo == CTM_SVD_GRAM && n_keep < R && R <= C;
}

size_t gram_lwork_bytes(Handle& h, int R, double* G, double* W) {
  size_t dws = 0, hws = 0;
  CTM_SOLVER(cusolverDnXsyevd_bufferSize(h.solver, h.solver_params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R,
                                         CUDA_R_64F, G, R, CUDA_R_64F, W, CUDA_R_64F, &dws, &hws));
  if (h.host_buf.size() < hws + 16) h.host_buf.resize(hws + 16);
  return dws;
}

// Truncating cut through the Gram matrix: G = M M^T (R x R, DMMA GEMM), eigenvectors by
// cuSOLVER syevd (ascending), the last n_keep columns reversed are the first n_keep left
// singular vectors of M (sigma_i = sqrt(lambda_i)).
double svd_left_gram(Handle& h, const double* mat, int R, int C, int n_keep, double* out) {
  const size_t mark = h.ws.top;
  double* G = h.ws.take((size_t)R * R);
  double* W = h.ws.take((size_t)R);
  size_t lw_bytes = gram_lwork_bytes(h, R, G, W);
  double* work = h.ws.take(lw_bytes / sizeof(double) + 1);
  ++h.n_svd;
  Operand a{{mat}, "ic", {R, C}}, b{{mat}, "jc", {R, C}};
  OutOperand g{{G}, "ij", {R, R}, {}};
  if (h.dry) {
    const double flops_before = h.flops;
    contract(h, a, b, g);   // sizing pass: reserves the split-K slab
    h.flops = flops_before;
    h.ws.reset(mark);
    return std::numeric_limits<double>::infinity();
  }
  CTM_CUDA(cudaEventRecord(h.ev[2], h.stream));
  const double flops_before = h.flops;   // the Gram GEMM is solver work, not move flops (R21)
  contract(h, a, b, g);
  h.flops = flops_before;
  CTM_SOLVER(cusolverDnXsyevd(h.solver, h.solver_params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R,
                              CUDA_R_64F, G, R, CUDA_R_64F, W, CUDA_R_64F, work, lw_bytes, h.host_buf.data(),
                              h.host_buf.size(), h.dev_info));
  // column R-1-j of the (symmetric, so layout-free) eigenvector matrix is kept column j
  extract_signfix_kernel<<<n_keep, 256, 0, h.stream>>>(G + (size_t)(R - 1) * R, 1, -(long long)R, R, n_keep, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
  CTM_CUDA(cudaEventRecord(h.ev[3], h.stream));
  int info = 0;
  std::vector<double> lam(R);
  CTM_CUDA(cudaMemcpyAsync(&info, h.dev_info, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaMemcpyAsync(lam.data(), W, sizeof(double) * R, cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaStreamSynchronize(h.stream));
  float ms = 0.f;
  CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[2], h.ev[3]));
  h.ms_svd += ms;
  if (info != 0)
    throw Error(CTM_E_SOLVER, "Gram eigensolver did not converge (info=" + std::to_string(info) + ") for a " +
                                  std::to_string(R) + " x " + std::to_string(C) + " matrix");
  for (double x : lam)
    if (!std::isfinite(x))
      throw Error(CTM_E_NONFINITE, "non-finite Gram eigenvalue in a " + std::to_string(R) + " x " +
                                       std::to_string(C) + " truncation");
  h.ws.reset(mark);
  const double lk = lam[R - n_keep], lk1 = lam[R - n_keep - 1];
  double gap = lk1 > 0.0 ? std::sqrt(std::max(lk, 0.0) / lk1) : std::numeric_limits<double>::infinity();
  if (gap < h.min_gap) h.min_gap = gap;
  return gap;
}

}  // namespace

double svd_left(Handle& h, const double* mat, int R, int C, int n_keep, double* out, bool basis_only) {
  if (n_keep < 1 || n_keep > R) throw Error(CTM_E_ARG, "svd_left: n_keep out of range");
  if (basis_only && h.prm.svd_algo == CTM_SVD_ISO && n_keep == C && C <= R) {
    if (!h.dry) CTM_CUDA(cudaEventRecord(h.ev[2], h.stream));
    iso_basis(h, mat, R, C, out);   // synchronises the stream
    if (!h.dry) {
      CTM_CUDA(cudaEventRecord(h.ev[3], h.stream));
      CTM_CUDA(cudaEventSynchronize(h.ev[3]));
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[2], h.ev[3]));
      h.ms_svd += ms;
    }
    return std::numeric_limits<double>::infinity();
  }
  if (use_gram(h, R, C, n_keep)) return svd_left_gram(h, mat, R, C, n_keep, out);
  if (h.prm.svd_algo == CTM_SVD_ISO && iso_supported(R, C, n_keep)) {
    if (!h.dry) CTM_CUDA(cudaEventRecord(h.ev[2], h.stream));
    const double ms0 = h.ms_svd;
    bool ok = false;
    const double gap = iso_left_vectors(h, mat, R, C, n_keep, out, signfix_launch, &ok);
    if (!h.dry && ok) {   // iso_left_vectors synchronised the stream
      CTM_CUDA(cudaEventRecord(h.ev[3], h.stream));
      CTM_CUDA(cudaEventSynchronize(h.ev[3]));
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[2], h.ev[3]));
      h.ms_svd = ms0 + ms;
      if (gap < h.min_gap) h.min_gap = gap;
      return gap;
    }
    if (!h.dry) ++h.n_svd_fallback;   // not certified: the dense cuSOLVER factorisation below
    // (sizing pass: fall through so the workspace also covers the fallback)
  } else if (h.prm.svd_algo == CTM_SVD_ISO && !h.dry) {
    ++h.n_svd_fallback;   // shape outside the solver's range (l > 2 CTM_ISO_LMAX)
  }
  const Plan p = make_plan(R, C, n_keep);
  const int mn = std::min(p.m, p.n);
  const size_t mark = h.ws.top;
  double* W = h.ws.take((size_t)R * C);
  double* S = h.ws.take((size_t)mn);
  double* U = h.ws.take((size_t)p.m * (p.econ ? mn : p.m));
  double* V = h.ws.take((size_t)p.n * p.n);
  size_t lw_bytes = query_lwork_bytes(h, p, W, S, U, V);
  double* work = h.ws.take(lw_bytes / sizeof(double) + 1);
  ++h.n_svd;
  if (h.dry) {
    h.ws.reset(mark);
    return std::numeric_limits<double>::infinity();
  }
  CTM_CUDA(cudaEventRecord(h.ev[2], h.stream));
  if (p.tall) {
    permute(h, mat, {R, C}, {1, 0}, W);   // column-major R x C
  } else {
    CTM_CUDA(cudaMemcpyAsync(W, mat, sizeof(double) * (size_t)R * C, cudaMemcpyDeviceToDevice, h.stream));
  }
  const int ldu = p.m, ldv = p.n;
  const double* vecs = nullptr;
  long long rs = 1, cs = 0;
  switch (h.prm.svd_algo) {
    case CTM_SVD_GESVDJ: {
      CTM_SOLVER(cusolverDnDgesvdj(h.solver, CUSOLVER_EIG_MODE_VECTOR, p.econ, p.m, p.n, W, p.m, S, U, ldu, V, ldv,
                                   work, (int)(lw_bytes / sizeof(double)), h.dev_info, h.gesvdj_info));
      if (p.tall) { vecs = U; rs = 1; cs = ldu; }
      else { vecs = V; rs = 1; cs = ldv; }
      break;
    }
    case CTM_SVD_GESVD: {
      signed char jobu = p.tall ? (p.econ ? 'S' : 'A') : 'N';
      signed char jobvt = p.tall ? 'N' : 'S';
      CTM_SOLVER(cusolverDnXgesvd(h.solver, h.solver_params, jobu, jobvt, p.m, p.n, CUDA_R_64F, W, p.m, CUDA_R_64F,
                                  S, CUDA_R_64F, U, ldu, CUDA_R_64F, V, mn, CUDA_R_64F, work, lw_bytes,
                                  h.host_buf.data(), h.host_buf.size(), h.dev_info));
      if (p.tall) { vecs = U; rs = 1; cs = ldu; }
      else { vecs = V; rs = mn; cs = 1; }   // rows of VT (ld = mn)
      break;
    }
    default: {
      double err_sigma = 0.0;
      CTM_SOLVER(cusolverDnXgesvdp(h.solver, h.solver_params, CUSOLVER_EIG_MODE_VECTOR, p.econ, p.m, p.n, CUDA_R_64F,
                                   W, p.m, CUDA_R_64F, S, CUDA_R_64F, U, ldu, CUDA_R_64F, V, ldv, CUDA_R_64F, work,
                                   lw_bytes, h.host_buf.data(), h.host_buf.size(), h.dev_info, &err_sigma));
      if (p.tall) { vecs = U; rs = 1; cs = ldu; }
      else { vecs = V; rs = 1; cs = ldv; }
      break;
    }
  }
  launch_k(extract_signfix_kernel, dim3(n_keep), dim3(256), 0, h.stream, (const double*)vecs, rs, cs, R, n_keep, out);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
  CTM_CUDA(cudaEventRecord(h.ev[3], h.stream));
  // status + singular values (host sync: cuSOLVER already synchronised for gesvdp)
  int info = 0;
  std::vector<double> s(mn);
  CTM_CUDA(cudaMemcpyAsync(&info, h.dev_info, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaMemcpyAsync(s.data(), S, sizeof(double) * mn, cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaStreamSynchronize(h.stream));
  float ms = 0.f;
  CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[2], h.ev[3]));
  h.ms_svd += ms;
  if (info != 0)
    throw Error(CTM_E_SOLVER, "SVD did not converge (info=" + std::to_string(info) + ") for a " + std::to_string(R) +
                                  " x " + std::to_string(C) + " matrix");
  for (double x : s)
    if (!std::isfinite(x))
      throw Error(CTM_E_NONFINITE, "non-finite singular value in a " + std::to_string(R) + " x " +
                                       std::to_string(C) + " SVD");
  h.ws.reset(mark);
  double gap = std::numeric_limits<double>::infinity();
  if (n_keep < mn && s[n_keep] > 0.0) gap = s[n_keep - 1] / s[n_keep];
  if (gap < h.min_gap) h.min_gap = gap;
  return gap;
}

size_t svd_workspace_doubles(Handle& h, int R, int C) {
  const Plan p = make_plan(R, C, R);
  const int mn = std::min(p.m, p.n);
  size_t b = query_lwork_bytes(h, p, nullptr, nullptr, nullptr, nullptr);
  return (size_t)R * C + mn + (size_t)p.m * p.m + (size_t)p.n * p.n + b / sizeof(double) + 64;
}

}  // namespace ctm
