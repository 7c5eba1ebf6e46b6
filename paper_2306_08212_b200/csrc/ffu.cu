// ffu.cu -- imaginary-time evolution on the device: one fast-full-update (FFU) bond update
// and its Trotter gate ("imaginary-time evolution method with a
// second-order Suzuki-Trotter decomposition ... the fast full update scheme (FFU) ... to
// avoid recomputing the effective environments after each update step").  The readings
// R25-R30 that fix what the paper leaves to its reference are in DESIGN.md (and restated in
// oracle/ffu_oracle.py, the CPU oracle this path is compared with).
//
// Every contraction runs in tc_gemm; the truncated SVDs in libctm's svd_left (the ISO
// solver, sign rule); the positivisation of the bond environment (a symmetric eigenproblem
// of (dD)^2) and the ALS normal equations (Cholesky solves of (dD D)^2) in cuSOLVER -- the
// same library role as the SVD fallback (svd.cu); there is no CPU path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctm_internal.h"
#include "ctm_tensor.h"

namespace ctm {
namespace {

#define FFU_SOLVER(x)                                                                          \
  do {                                                                                         \
    cusolverStatus_t s_ = (x);                                                                 \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                         \
      throw Error(CTM_E_SOLVER, std::string(#x) + " failed with status " + std::to_string((int)s_)); \
  } while (0)

// g = exp(-delta H) for the n x n (n = d^2 <= 16) bond matrix H = hop (row-major), by scaling
// and squaring of a degree-18 Taylor series (reading R25: the exact exponential; the oracle
// takes the eigendecomposition -- both are exact to rounding).  One thread.
__global__ void expm_kernel(const double* __restrict__ hop, int n, double delta, double* __restrict__ g) {
  CTM_PDL_WAIT();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double X[256], T[256], S[256], W[256];
  double nrm = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = 0.0;
    for (int j = 0; j < n; ++j) {
      X[i * n + j] = -delta * 0.5 * (hop[i * n + j] + hop[j * n + i]);
      r += fabs(X[i * n + j]);
    }
    nrm = fmax(nrm, r);
  }
  int sq = 0;
  while (nrm > 0.125) {
    nrm *= 0.5;
    ++sq;
  }
  const double sc = ldexp(1.0, -sq);
  for (int i = 0; i < n * n; ++i) X[i] *= sc;
  for (int i = 0; i < n * n; ++i) {
    S[i] = (i % (n + 1) == 0) ? 1.0 : 0.0;
    T[i] = S[i];
  }
  for (int k = 1; k <= 18; ++k) {   // T <- T X / k, S += T
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double a = 0.0;
        for (int l = 0; l < n; ++l) a += T[i * n + l] * X[l * n + j];
        W[i * n + j] = a / k;
      }
    for (int i = 0; i < n * n; ++i) {
      T[i] = W[i];
      S[i] += W[i];
    }
  }
  for (int s = 0; s < sq; ++s) {   // S <- S S
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double a = 0.0;
        for (int l = 0; l < n; ++l) a += S[i * n + l] * S[l * n + j];
        W[i * n + j] = a;
      }
    for (int i = 0; i < n * n; ++i) S[i] = W[i];
  }
  for (int i = 0; i < n * n; ++i) g[i] = S[i];
}

// M (n x n) <- (M + M^T) / 2, one grid-stride pass over the upper triangle
__global__ void symmetrise_kernel(double* __restrict__ M, int n) {
  CTM_PDL_WAIT();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (long long)i * n);
    if (j > i) {
      const double v = 0.5 * (M[(size_t)i * n + j] + M[(size_t)j * n + i]);
      M[(size_t)i * n + j] = v;
      M[(size_t)j * n + i] = v;
    }
  }
}

// V (n x n row-major, row r = eigenvector r from syevd) <- diag(max(lam, 0) + 1e-12 max|lam|) V
// (reading R27's positivisation; lam ascending)
__global__ void clip_scale_rows_kernel(double* __restrict__ V, const double* __restrict__ lam, int n) {
  CTM_PDL_WAIT();
  const double big = fmax(fabs(lam[0]), fabs(lam[n - 1]));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / n);
    V[e] *= fmax(lam[r], 0.0) + 1e-12 * big;
  }
}

// Q (n x n) += (1e-12 tr Q / n) I   (one CTA; the ALS regularisation of reading R28)
__global__ void regularise_kernel(double* __restrict__ Q, int n) {
  CTM_PDL_WAIT();
  __shared__ double red[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += Q[(size_t)i * n + i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    red[0] = s;
  }
  __syncthreads();
  const double eps = 1e-12 * red[0] / n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) Q[(size_t)i * n + i] += eps;
}

// SVD split (reading R28): U (rows x n) <- U sqrt(s), SVt (n x cols) <- SVt / sqrt(s),
// s_a = ||row a of SVt|| (= sigma_a).  One CTA per kept index a.
__global__ void split_scale_kernel(double* __restrict__ U, double* __restrict__ SVt, int rows, int n, int cols) {
  CTM_PDL_WAIT();
  const int a = blockIdx.x;
  __shared__ double red[32];
  double t = 0.0;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) t += SVt[(size_t)a * cols + j] * SVt[(size_t)a * cols + j];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    red[0] = sqrt(fmax(sqrt(s), 1e-300));   // sqrt(sigma_a)
  }
  __syncthreads();
  const double q = red[0];
  for (int j = threadIdx.x; j < cols; j += blockDim.x) SVt[(size_t)a * cols + j] /= q;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) U[(size_t)i * n + a] *= q;
}

__global__ void scale_kernel(double* __restrict__ p, long long n, double f) {
  CTM_PDL_WAIT();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] *= f;
}

template <class K, class... Args>
void launch1(Handle& h, K k, dim3 g, dim3 b, Args... args) {
  if (h.dry) return;
  launch_k(k, g, b, 0, h.stream, args...);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

// device dot product into a host double (synchronises)
double dot_host(Handle& h, const double* a, const double* b, size_t n) {
  if (h.dry) {
    h.ws.take(1);
    return 0.0;
  }
  const size_t mark = h.ws.top;
  double* r = h.ws.take(1);
  dot(h, a, b, n, r);
  double v = 0.0;
  CTM_CUDA(cudaMemcpyAsync(&v, r, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaStreamSynchronize(h.stream));
  h.ws.reset(mark);
  return v;
}

// Q x = b for the symmetric positive n x n Q (row-major = column-major), nrhs right-hand
// sides stored as rows of B (row-major nrhs x n = column-major n x nrhs): Cholesky (cuSOLVER).
void spd_solve(Handle& h, double* Q, int n, double* B, int nrhs) {
  launch1(h, regularise_kernel, dim3(1), dim3(256), Q, n);
  int lwork = 0;
  FFU_SOLVER(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, n, Q, n, &lwork));
  const size_t mark = h.ws.top;
  double* work = h.ws.take((size_t)std::max(lwork, 1));
  if (!h.dry) {
    FFU_SOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, n, Q, n, work, lwork, h.dev_info));
    FFU_SOLVER(cusolverDnDpotrs(h.solver, CUBLAS_FILL_MODE_LOWER, n, nrhs, Q, n, B, n, h.dev_info));
  }
  h.ws.reset(mark);
}

// N (n x n) <- V diag(lam+) V^T with (lam, V) = eig((N + N^T)/2) (reading R27)
void positivise(Handle& h, double* N, int n) {
  const size_t mark = h.ws.top;
  launch1(h, symmetrise_kernel, dim3(std::min(148, (n * n + 255) / 256)), dim3(256), N, n);
  Ten V = alloc(h, {n, n});
  double* lam = h.ws.take((size_t)n);
  if (!h.dry) CTM_CUDA(cudaMemcpyAsync(V.p, N, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, h.stream));
  int lwork = 0;
  FFU_SOLVER(cusolverDnDsyevd_bufferSize(h.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, V.p, n, lam,
                                         &lwork));
  double* work = h.ws.take((size_t)std::max(lwork, 1));
  if (!h.dry)
    FFU_SOLVER(cusolverDnDsyevd(h.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, V.p, n, lam, work, lwork,
                                h.dev_info));
  // column-major eigenvectors read row-major: row r of V is eigenvector r
  Ten S = alloc(h, {n, n});
  if (!h.dry) CTM_CUDA(cudaMemcpyAsync(S.p, V.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, h.stream));
  launch1(h, clip_scale_rows_kernel, dim3(std::min(148, (n * n + 255) / 256)), dim3(256), S.p, (const double*)lam, n);
  Ten Nt{N, {n, n}};
  contract(h, op({&V}, "rj"), op({&S}, "rk"), out({&Nt}, "jk"));
  h.ws.reset(mark);
}

}  // namespace

// One FFU update of the horizontal bond A (left) - B (right), readings R26-R28; returns the
// final N-weighted error and <theta'|N|theta'> in cost[0..1] (cost may be null).
void ffu_bond_update_h(Handle& h, const double* Ap, const double* Bp, const ctm_env* env, const double* gate,
                       int sweeps, double* A2p, double* B2p, double* cost) {
  const int d = h.prm.d, D = h.prm.D;
  const int D3 = D * D * D, dD = d * D, m = std::min(D3, dD);
  const int n = std::min(D, m * d);   // the new bond (D: reading R28)
  const size_t mark = h.ws.top;
  // ---- R26 reductions: A as (u l c) x (s r), B as (u c r) x (s l) --------------------------
  Ten Am = alloc(h, {D, D, D, d, D});   // (u, l, c, s, r)
  Ten Bm = alloc(h, {D, D, D, d, D});   // (u, c, r, s, l)
  permute(h, Ap, {d, D, D, D, D}, {1, 2, 3, 0, 4}, Am.p);
  permute(h, Bp, {d, D, D, D, D}, {1, 3, 4, 0, 2}, Bm.p);
  Ten X = alloc(h, {D, D, D, m});       // (u, l, c, w)
  Ten Yt = alloc(h, {D, D, D, m});      // (u, c, r, v)
  svd_left(h, Am.p, D3, dD, m, X.p);
  svd_left(h, Bm.p, D3, dD, m, Yt.p);
  Ten aR = alloc(h, {m, d, D});         // (w, s, r)
  Ten bL = alloc(h, {m, d, D});         // (v, t, l)
  contract(h, op({&X}, "ulcw"), op({&Am}, "ulcsr"), out({&aR}, "wsr"));
  contract(h, op({&Yt}, "ucrv"), op({&Bm}, "ucrtl"), out({&bL}, "vtl"));
  // ---- R27 bond environment: the 2x1 window with X, Y (ctm_bond_energy's order) ----------
  Ten N = alloc(h, {m, m, m, m});        // (w, v, w', v')
  {
    const size_t mk = h.ws.top;
    const int a = 0, b = 1;
    Ten c1 = envC(env, a, 1), t2 = envT(env, a, 2, D), t1 = envT(env, a, 1, D), c4 = envC(env, a, 4),
        t4 = envT(env, a, 4, D);
    Ten E1 = alloc(h, {c1.ext[0], D, D, t2.ext[3]});
    contract(h, op({&c1}, "xy"), op({&t2}, "ymnY"), out({&E1}, "xmnY"));
    Ten E2 = alloc(h, {D, D, t2.ext[3], t1.ext[0], D, D});
    contract(h, op({&E1}, "xmnY"), op({&t1}, "Xkbx"), out({&E2}, "mnYXkb"));
    Ten E3 = alloc(h, {D, t2.ext[3], t1.ext[0], D, D, m});
    contract(h, op({&E2}, "mnYXkb"), op({&X}, "mkpw"), out({&E3}, "nYXbpw"));
    Ten E4 = alloc(h, {t2.ext[3], t1.ext[0], D, m, D, m});
    contract(h, op({&E3}, "nYXbpw"), op({&X}, "nbqe"), out({&E4}, "YXpwqe"));
    Ten F1 = alloc(h, {c4.ext[1], t4.ext[0], D, D});
    contract(h, op({&c4}, "ZX"), op({&t4}, "UpqZ"), out({&F1}, "XUpq"));
    Ten L = alloc(h, {t2.ext[3], t4.ext[0], m, m});
    contract(h, op({&E4}, "YXpwqe"), op({&F1}, "XUpq"), out({&L}, "YUwe"));
    Ten u2 = envT(env, b, 2, D), c2 = envC(env, b, 2), u3 = envT(env, b, 3, D), c3 = envC(env, b, 3),
        u4 = envT(env, b, 4, D);
    Ten G1 = alloc(h, {u2.ext[0], D, D, c2.ext[1]});
    contract(h, op({&u2}, "Ymnz"), op({&c2}, "zc"), out({&G1}, "Ymnc"));
    Ten G2 = alloc(h, {u2.ext[0], D, D, D, D, u3.ext[3]});
    contract(h, op({&G1}, "Ymnc"), op({&u3}, "cklW"), out({&G2}, "YmnklW"));
    Ten G3 = alloc(h, {u2.ext[0], D, D, u3.ext[3], D, m});
    contract(h, op({&G2}, "YmnklW"), op({&Yt}, "mpkf"), out({&G3}, "YnlWpf"));
    Ten G4 = alloc(h, {u2.ext[0], u3.ext[3], D, m, D, m});
    contract(h, op({&G3}, "YnlWpf"), op({&Yt}, "nqlg"), out({&G4}, "YWpfqg"));
    Ten H1 = alloc(h, {c3.ext[0], u4.ext[3], D, D});
    contract(h, op({&c3}, "WV"), op({&u4}, "VpqU"), out({&H1}, "WUpq"));
    Ten R = alloc(h, {u2.ext[0], u4.ext[3], m, m});
    contract(h, op({&G4}, "YWpfqg"), op({&H1}, "WUpq"), out({&R}, "YUfg"));
    contract(h, op({&L}, "YUwe"), op({&R}, "YUfg"), out({&N}, "wfeg"));
    h.ws.reset(mk);
  }
  positivise(h, N.p, m * m);
  // ---- R28 gate, truncated-SVD start, ALS ---------------------------------------------------
  Ten th0 = alloc(h, {m, d, d, m});
  contract(h, op({&aR}, "wsr"), op({&bL}, "vtr"), out({&th0}, "wstv"));
  Ten G{const_cast<double*>(gate), {d, d, d, d}};
  Ten th = alloc(h, {m, d, d, m});
  contract(h, op({&G}, "stpq"), op({&th0}, "wpqv"), out({&th}, "wstv"));
  Ten U = alloc(h, {m, d, n});          // aR1 (w, s, a)
  svd_left(h, th.p, m * d, d * m, n, U.p);
  Ten SV = alloc(h, {n, d, m});         // bL1 (a, t, v)
  contract(h, op({&U}, "wsa"), op({&th}, "wstv"), out({&SV}, "atv"));
  launch1(h, split_scale_kernel, dim3(n), dim3(256), U.p, SV.p, m * d, n, d * m);
  Ten Nt = alloc(h, {m, d, d, m});      // N theta' (ket side open)
  contract(h, op({&N}, "wvxy"), op({&th}, "xsty"), out({&Nt}, "wstv"));
  const double tNt = dot_host(h, th.p, Nt.p, th.size());
  const int na = m * n;
  Ten T1 = alloc(h, {n, d, m, m, m});
  Ten Q = alloc(h, {m, n, m, n});
  Ten rhs = alloc(h, {d, m, n});
  for (int sw = 0; sw < sweeps; ++sw) {
    // aR with bL fixed: Q_a[(w,a),(x,b)] = sum bL(a,t,v) N(w,v,x,y) bL(b,t,y)
    T1.ext = {n, d, m, m, m};
    contract(h, op({&SV}, "atv"), op({&N}, "wvxy"), out({&T1}, "atwxy"));
    Q.ext = {m, n, m, n};
    contract(h, op({&T1}, "atwxy"), op({&SV}, "bty"), out({&Q}, "waxb"));
    rhs.ext = {d, m, n};
    contract(h, op({&SV}, "atv"), op({&Nt}, "wstv"), out({&rhs}, "swa"));
    spd_solve(h, Q.p, na, rhs.p, d);
    permute(h, rhs.p, {d, m, n}, {1, 0, 2}, U.p);   // (s, w, a) -> (w, s, a)
    // bL with aR fixed: Q_b[(a,v),(b,y)] = sum aR(w,s,a) N(w,v,x,y) aR(x,s,b)
    T1.ext = {d, n, m, m, m};
    contract(h, op({&U}, "wsa"), op({&N}, "wvxy"), out({&T1}, "savxy"));
    Q.ext = {n, m, n, m};
    contract(h, op({&T1}, "savxy"), op({&U}, "xsb"), out({&Q}, "avby"));
    rhs.ext = {d, n, m};
    contract(h, op({&U}, "wsa"), op({&Nt}, "wstv"), out({&rhs}, "tav"));
    spd_solve(h, Q.p, na, rhs.p, d);
    permute(h, rhs.p, {d, n, m}, {1, 0, 2}, SV.p);  // (t, a, v) -> (a, t, v)
  }
  if (cost) {   // final N-weighted error ||phi - theta'||_N^2, phi = aR bL
    Ten phi = alloc(h, {m, d, d, m});
    Ten Nphi = alloc(h, {m, d, d, m});
    contract(h, op({&U}, "wsa"), op({&SV}, "atv"), out({&phi}, "wstv"));
    contract(h, op({&N}, "wvxy"), op({&phi}, "xsty"), out({&Nphi}, "wstv"));
    const double pNp = dot_host(h, phi.p, Nphi.p, phi.size());
    const double pNt = dot_host(h, phi.p, Nt.p, phi.size());
    cost[0] = pNp - 2.0 * pNt + tNt;
    cost[1] = tNt;
  }
  // ---- recombine and normalise ---------------------------------------------------------------
  Ten A2{A2p, {d, D, D, D, n}}, B2{B2p, {d, D, n, D, D}};
  contract(h, op({&X}, "ulcw"), op({&U}, "wsa"), out({&A2}, "sulca"));
  contract(h, op({&SV}, "atv"), op({&Yt}, "ucrv"), out({&B2}, "tuacr"));
  for (Ten* t : {&A2, &B2}) {   // Frobenius normalisation (deterministic dot, then one scale)
    const double nrm = std::sqrt(dot_host(h, t->p, t->p, t->size()));
    launch1(h, scale_kernel, dim3(std::min<size_t>(148, (t->size() + 255) / 256)), dim3(256), t->p,
            (long long)t->size(), nrm > 0.0 ? 1.0 / nrm : 1.0);
  }
  h.ws.reset(mark);
}

void ffu_gate(Handle& h, const double* hop, double delta, double* g) {
  const int n = h.prm.d * h.prm.d;
  if (n > 16) throw Error(CTM_E_UNSUPPORTED, "Trotter gate: d^2 > 16");
  launch1(h, expm_kernel, dim3(1), dim3(32), hop, n, delta, g);
}

}  // namespace ctm
