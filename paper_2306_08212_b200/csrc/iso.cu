// iso.cu -- libctm's own truncated-SVD solver for the isometries (
// P:L46 "the unitary matrix U is reshaped ... truncation applied corresponding to the
// largest chi singular values", P:L60 two-stage recipe; north star: "cuSOLVER gesvdj or a
// hand-written Jacobi kernel").
//
// What the paper needs from an SVD here is the first n left singular vectors of an R x C
// matrix M (R = chi D, n = chi' = R / D): a small slice of the spectrum.  Dense cuSOLVER
// factorisations of 1024^2 are latency bound (35-95 ms, profiles/r01_probe_svd.txt), so
// libctm computes only that slice:
//
//  * truncating cut (n < R):  subspace iteration on M M^T with a block of l = n + p columns
//      Y <- orth(M (M^T Y)),  orth = CholQR (Gram on the DMMA GEMM, one-CTA Cholesky,
//      row-parallel triangular solve), then a Rayleigh-Ritz step that never forms a Gram
//      of M: Z = M^T Y = Q_z R_z (shifted CholQR3, backward stable), the left singular
//      vectors W of R_z^T by one-sided Jacobi in shared memory, U = Y W.  Convergence is
//      certified by the residuals ||M M^T u_i - s_i^2 u_i|| of the kept Ritz vectors.
//  * non-truncating / tall cut (stage two of TS, n >= C):  M = Q_o R (shifted CholQR3),
//      U = Q_o * lsv(R) with lsv(R) by the same one-sided Jacobi kernel.
//
// Accuracy: the Rayleigh-Ritz and the tall path are backward stable in M (no squared
// condition number, unlike a Gram eigensolver, which failed c3_dl's conditioning test);
// subspace iteration adds a containment error that the residual test drives to the
// rounding floor.  The sign rule (largest-|.| entry of each column positive) is applied by
// the same extraction kernel the cuSOLVER path uses.
//
// Shapes this solver does not take (l > 2 CTM_ISO_LMAX, or a rank-deficient keep with
// n > C) go to cuSOLVER gesvdp (svd.cu); there is no CPU path.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <set>
#include <vector>

#include "ctm_internal.h"
#include "fgemm.cuh"
#include "iso_kernels.cuh"

namespace ctm {
namespace {

using namespace isok;
// Block oversampling p (l = n + p): 32, or 48 when l exceeds the one-CTA limit LMAX anyway
// (C5: 284 -> 269 ms per move; 16 / 24 were slower at C4, 48 / 64 at C4 cross the LMAX cliff).
// solver tuning knobs for A/B experiments (environment, read once; defaults are the tuned values)
static int knob_int(const char* name, int def) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : def;
}
static double knob_double(const char* name, double def) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : def;
}
static int iso_oversample(int n_keep) {
  static const int p = knob_int("CTM_ISO_P", 32);   // (A/B knob)
  return (n_keep + p > LMAX && n_keep + 48 <= LMAX_BIG) ? 48 : p;
}
constexpr double EPS = 2.220446049250313e-16;

// ---------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------
struct IsoFail : std::runtime_error {
  explicit IsoFail(const std::string& m) : std::runtime_error(m) {}
};

void set_smem(const void* f, size_t bytes) {
  CTM_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// CTM_ISO_JAC_OLD=1: the previous Jacobi cluster shapes (A/B)
static bool jac_old() {
  static const bool on = std::getenv("CTM_ISO_JAC_OLD") != nullptr;
  return on;
}

struct Solver {
  Handle& h;
  int* status;   // device: [0] CholQR pivot, [1] Jacobi failure, [2] Jacobi sweeps
  int last_sweeps = 0;
  int* repl;     // device: per-column "numerically dependent" flags (chol_kernel)
  unsigned seed = 0x9e3779b9u;
  // event timing of the Jacobi launch pending since the last check_status (which syncs)
  bool jac_pending = false;
  int jac_n = 0, jac_max = 0, jac_slot = 0, jac_ctas = 1;
  explicit Solver(Handle& hh) : h(hh) {
    status = reinterpret_cast<int*>(h.ws.take(8));
    repl = reinterpret_cast<int*>(h.ws.take(LMAX_BIG / 2 + 1));
    if (!h.dry) {
      CTM_CUDA(cudaMemsetAsync(status, 0, 8 * sizeof(double), h.stream));
      CTM_CUDA(cudaMemsetAsync(repl, 0, LMAX_BIG * sizeof(int), h.stream));
    }
  }
  // C (m x n) = A * B with row-major operands given by label strings.
  void gemm(const double* A, const char* la, std::vector<int> ea, const double* B, const char* lb,
            std::vector<int> eb, double* C, const char* lc, std::vector<int> ec, GemmPartials* defer = nullptr) {
    Operand a{{A}, la, ea}, b{{B}, lb, eb};
    OutOperand c{{C}, lc, ec, {}};
    const double f = h.flops;
    contract(h, a, b, c, 1.0, defer);
    h.flops = f;   // solver work is not part of the move's algorithmic flops (R21)
  }
  // C (M x N, ld N) = alpha op(A) X + beta Y + gamma W on fgemm_kernel (fgemm.cuh): one
  // launch, full K per CTA, no split-K slab.  A row-major with leading dimension lda,
  // op(A) = A^T when trans; X (K x N), Y and W (M x N, nullable; W may alias C).  Returns
  // false (nothing launched) when the operands miss its 16-byte A copies (the caller
  // then takes the tc_gemm path).  CTM_ISO_FGEMM=0 disables it (A/B).
  bool fgemm(const double* A, int lda, bool trans, int M, int K, const double* X, int N, double* C,
             double alpha = 1.0, const double* Y = nullptr, double beta = 0.0, const double* W = nullptr,
             double gamma = 0.0) {
    static const bool on = knob_int("CTM_ISO_FGEMM", 1) != 0;
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    if (!on || (lda & 1) || (trans ? (M & 1) : (K & 1)) || !al16(A)) return false;
    if (h.dry || M == 0 || N == 0) return true;
    fg::FgArgs a{A, X, C, Y, W, lda, N, N, N, M, N, K, alpha, beta, gamma};
    const bool xvec = (N & 1) == 0 && al16(X);
    const dim3 grid((N + fg::BN - 1) / fg::BN, (M + fg::BM - 1) / fg::BM);
    if (trans) {
      if (xvec) launch_k(fg::fgemm_kernel<true, true>, grid, dim3(fg::THREADS), fg::SMEM_BYTES, h.stream, a);
      else launch_k(fg::fgemm_kernel<true, false>, grid, dim3(fg::THREADS), fg::SMEM_BYTES, h.stream, a);
    } else {
      if (xvec) launch_k(fg::fgemm_kernel<false, true>, grid, dim3(fg::THREADS), fg::SMEM_BYTES, h.stream, a);
      else launch_k(fg::fgemm_kernel<false, false>, grid, dim3(fg::THREADS), fg::SMEM_BYTES, h.stream, a);
    }
    CTM_CUDA(cudaGetLastError());
    h.count_kernel();
    return true;
  }
  // One CholQR pass on Y (m x n): S = Y^T Y, S (+shift) = R^T R, Y <- Y R^{-1}.
  // replace: numerically dependent columns (pivot <= 1e-13 of the column's squared norm)
  // are overwritten with random directions instead of failing; a later pass re-orthonormalises.
  // also (optional, m x n): right-multiplied by the same R^{-1} (keeps a three-term
  // recurrence consistent across the orthonormalisation).
  void cholqr_pass(double* Y, int m, int n, double shift_factor, double* R, bool replace = false,
                   double* also = nullptr) {
    const size_t mark = h.ws.top;
    double* S = h.ws.take((size_t)n * n);
    double* rd = h.ws.take((size_t)n);
    double* Rpk = n <= LMAX ? h.ws.take(rpk_size(n)) : nullptr;
    // (tried: the Gram GEMM's split-K partials summed by chol_kernel's load instead of the reduction
    // launch -- no change at C3/C4/C5, profiles/r02s3_ab_chol_defer.jsonl; PDL already hides it)
    gemm(Y, "ia", {m, n}, Y, "ib", {m, n}, S, "ab", {n, n});
    if (h.dry) {
      if (n > LMAX) chol_two_block(S, n, shift_factor, R, rd, replace);   // reserves its scratch
      h.ws.reset(mark);
      return;
    }
    if (n <= LMAX) {
      launch_k(chol_kernel, dim3(1), dim3(CHOL_THREADS), chol_smem_bytes(n), h.stream, (const double*)S, n, shift_factor,
               R, rd, status, replace ? 1e-13 : 0.0, replace ? repl : nullptr, (const double*)nullptr, Rpk);
      CTM_CUDA(cudaGetLastError());
      h.count_kernel();
    } else {
      chol_two_block(S, n, shift_factor, R, rd, replace);
    }
    if (n <= LMAX) {
      trsm(Y, m, n, R, rd, Rpk, nullptr, also);   // (both matrices in one launch)
    } else {
      trsm(Y, m, n, R, rd, Rpk, nullptr);
      if (also) trsm(also, m, n, R, rd, Rpk, nullptr);
    }
    if (replace) {
      launch_k(replace_cols_kernel, dim3(std::min(n, 148)), dim3(256), 0, h.stream, Y, m, n, repl, seed += 0x6a09e667u);
      CTM_CUDA(cudaGetLastError());
      h.count_kernel();
    }
    h.ws.reset(mark);
  }
  void trsm(double* Y, int m, int n, const double* R, const double* rd, const double* Rpk, const int* dep,
            double* Y2 = nullptr) {
    const int rows_per_cta = 8;
    const int rows = Y2 ? 2 * m : m;
    const int grid = std::max(1, std::min(4 * 148, (rows + rows_per_cta - 1) / rows_per_cta));
    // one CTA per SM holds the 144 KB operand: 16 warps when the rows exceed 148 x 8
    const int threads = rows > 148 * 8 ? 512 : 256;
    const int grid_s = std::max(1, std::min(148, (rows + threads / 32 - 1) / (threads / 32)));
    if (n <= LMAX)
      launch_k(trsm_rows_kernel<(LMAX + 31) / 32>, dim3(grid_s), dim3(threads), rpk_size(n) * sizeof(double), h.stream,
               Y, m, n, Rpk, dep, Y2);
    else launch_k(trsm_rows_big_kernel, dim3(grid), dim3(256), 0, h.stream, Y, m, n, R, rd);   // dep: only at n1 = LMAX
    CTM_CUDA(cudaGetLastError());
    h.count_kernel();
  }
  // S (n x n, LMAX < n <= LMAX_BIG) + shift I = R^T R by two LMAX-sized blocks
  // (chol_diag_shift_kernel's comment); same status / replacement conventions as chol_kernel.
  void chol_two_block(double* S, int n, double shift_factor, double* R, double* rd, bool replace) {
    const size_t mark = h.ws.top;
    const int n1 = LMAX, n2 = n - n1;
    double* dref = h.ws.take((size_t)n);
    double* S11 = h.ws.take((size_t)n1 * n1);
    double* W = h.ws.take((size_t)n2 * n1);
    double* S22 = h.ws.take((size_t)n2 * n2);
    double* R11 = h.ws.take((size_t)n1 * n1);
    double* R22 = h.ws.take((size_t)n2 * n2);
    double* Rpk1 = h.ws.take(rpk_size(n1));
    if (h.dry) {
      h.ws.reset(mark);
      return;
    }
    const double tol = replace ? 1e-13 : 0.0;
    launch_k(chol_diag_shift_kernel, dim3(1), dim3(256), 0, h.stream, S, n, shift_factor, dref);
    CTM_CUDA(cudaGetLastError());
    const size_t sz = sizeof(double);
    CTM_CUDA(cudaMemcpy2DAsync(S11, n1 * sz, S, n * sz, n1 * sz, n1, cudaMemcpyDeviceToDevice, h.stream));
    CTM_CUDA(cudaMemcpy2DAsync(W, n1 * sz, S + (size_t)n1 * n, n * sz, n1 * sz, n2, cudaMemcpyDeviceToDevice, h.stream));
    CTM_CUDA(cudaMemcpy2DAsync(S22, n2 * sz, S + (size_t)n1 * n + n1, n * sz, n2 * sz, n2, cudaMemcpyDeviceToDevice,
                               h.stream));
    launch_k(chol_kernel, dim3(1), dim3(CHOL_THREADS), chol_smem_bytes(n1), h.stream, (const double*)S11, n1, 0.0, R11,
             rd, status, tol, replace ? repl : nullptr, (const double*)dref, Rpk1);
    CTM_CUDA(cudaGetLastError());
    trsm(W, n2, n1, R11, rd, Rpk1, replace ? repl : nullptr);   // W = S21 R11^{-1} = R12^T
    launch_k(chol_schur_kernel, dim3((n2 + 15) / 16, (n2 + 15) / 16), dim3(16, 16), 0, h.stream, S22, (const double*)W, n2, n1);
    CTM_CUDA(cudaGetLastError());
    launch_k(chol_kernel, dim3(1), dim3(CHOL_THREADS), chol_smem_bytes(n2), h.stream, (const double*)S22, n2, 0.0, R22,
             rd + n1, status, tol, replace ? repl + n1 : nullptr, (const double*)(dref + n1), (double*)nullptr);
    CTM_CUDA(cudaGetLastError());
    launch_k(chol_assemble_kernel, dim3(std::min(148, (n * n + 255) / 256)), dim3(256), 0, h.stream, R, n, n1,
             (const double*)R11, (const double*)W, (const double*)R22);
    CTM_CUDA(cudaGetLastError());
    h.count_kernel(5);
    h.ws.reset(mark);
  }
  // passes of CholQR (the first one shifted when `shifted`), R_total = R_p ... R_1.
  void cholqr(double* Y, int m, int n, int passes, bool shifted, double* Rtot, bool replace = false,
              double* also = nullptr) {
    const size_t mark = h.ws.top;
    double* R = h.ws.take((size_t)n * n);
    double* T = Rtot ? h.ws.take((size_t)n * n) : nullptr;
    for (int p = 0; p < passes; ++p) {
      const double sf = (shifted && p == 0) ? 11.0 * ((double)m * n + (double)n * (n + 1)) * EPS : 0.0;
      // the dense R is needed only to accumulate Rtot, or by the two-block path (l > LMAX)
      double* Rp = (Rtot && p == 0) ? Rtot : ((Rtot || n > LMAX) ? R : nullptr);
      // the first plain pass may replace numerically dependent columns
      cholqr_pass(Y, m, n, sf, Rp, replace && p == (shifted ? 1 : 0), passes == 1 ? also : nullptr);
      if (Rtot && p > 0) {   // Rtot <- R_p Rtot
        gemm(R, "ab", {n, n}, Rtot, "bc", {n, n}, T, "ac", {n, n});
        if (!h.dry) CTM_CUDA(cudaMemcpyAsync(Rtot, T, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, h.stream));
      }
    }
    h.ws.reset(mark);   // stream order makes the scratch reusable by the next call
  }
  // max_sweeps < 0: up to 60 sweeps, failure (status) if not converged; otherwise a capped
  // run whose result is used only as an estimate (no failure flag).
  void jacobi(const double* X, int n, int trans, int ncols, double* U, double* S, double tol = 1e-14,
              int max_sweeps = -1) {
    if (h.dry) return;
    const size_t smem = (size_t)n * (n + 1) * sizeof(double);
    int* st = max_sweeps < 0 ? status + 1 : status + 4;   // capped runs report into a scratch slot
    const int ms = max_sweeps < 0 ? 60 : max_sweeps;
    const double skip_tol = 1e-10;   // (1e-9 / 1e-8: no measurable change at C4 / C5)
    CTM_CUDA(cudaEventRecord(h.jev[0], h.stream));
    // cluster shapes from tools/bench_jacobi_cfg.cu (profiles/r02_jacobi_cluster_shapes.jsonl),
    // us per sweep: l = 160: 2 CTAs x 8-lane groups 322 -> 4 x 4-lane 242; n = 128: one CTA 214
    // -> 4 x 4-lane 150; l = 232: 8 x 4-lane 632 -> 8 x 2-lane 574
    if (n > LMAX && jac_old()) {   // A/B (CTM_ISO_JAC_OLD): the previous shapes
      using J = JacCfg<8, 4, LMAX_BIG>;
      launch_k(jacobi_cluster_kernel<8, 4, LMAX_BIG>, dim3(8), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S,
               st, ms, tol, skip_tol);
    } else if (n > LMAX) {   // C5: 8-CTA cluster, rows split eight ways, 2-lane groups
      using J = JacCfg<8, 2, LMAX_BIG>;
      launch_k(jacobi_cluster_kernel<8, 2, LMAX_BIG>, dim3(8), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S,
               st, ms, tol, skip_tol);
    } else if (n > 128 && jac_old()) {
      using J = JacCfg<2, 8, LMAX>;
      launch_k(jacobi_cluster_kernel<2, 8, LMAX>, dim3(2), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S, st,
               ms, tol, skip_tol);
    } else if (n > 128) {   // register-resident 4-CTA cluster, 4-lane groups
      using J = JacCfg<4, 4, LMAX>;
      launch_k(jacobi_cluster_kernel<4, 4, LMAX>, dim3(4), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S, st,
               ms, tol, skip_tol);
    } else if (n > 32 && !jac_old() && !std::getenv("CTM_ISO_JAC_SMEM")) {   // 4-CTA cluster, 4-lane groups
      using J = JacCfg<4, 4, 128>;
      launch_k(jacobi_cluster_kernel<4, 4, 128>, dim3(4), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S, st,
               ms, tol, skip_tol);
    } else if (n > 32 && !std::getenv("CTM_ISO_JAC_SMEM")) {   // register-resident, one CTA
      using J = JacCfg<1, 8, 128>;
      launch_k(jacobi_cluster_kernel<1, 8, 128>, dim3(1), dim3(J::THREADS), J::SMEM, h.stream, X, n, trans, ncols, U, S, st,
               ms, tol, skip_tol);
    } else {
      jacobi_lsv_kernel<<<1, jacobi_threads(n), smem, h.stream>>>(X, n, trans, ncols, U, S, st,
                                                                  max_sweeps < 0 ? 60 : max_sweeps, tol);
    }
    CTM_CUDA(cudaGetLastError());
    CTM_CUDA(cudaEventRecord(h.jev[1], h.stream));
    jac_pending = true;
    jac_n = n;
    jac_max = ms;
    jac_slot = max_sweeps < 0 ? 2 : 5;   // status int index holding the sweep count
    jac_ctas = n > LMAX ? 8 : (jac_old() ? (n > 128 ? 2 : 1) : (n > 32 ? 4 : 1));
    h.count_kernel();
  }
  // Preconditioned one-sided Jacobi (Drmac & Veselic): the left singular vectors of
  // Xc = (trans ? X^T : X) (n x n) equal those of R'^T where Xc^T = Q R' (sCholQR3; the
  // right factor Q^T drops out), and the columns of R'^T are far closer to orthogonal --
  // R' R'^T = Q^T (Xc^T Xc) Q is one step of the LR iteration on the Gram -- so the
  // Jacobi needs fewer sweeps.  Same outputs as jacobi(X, n, trans, ...).
  void jacobi_pc(const double* X, int n, int trans, int ncols, double* U, double* S, double tol = 1e-14,
                 int max_sweeps = -1) {
    const size_t mark = h.ws.top;
    double* T = h.ws.take((size_t)n * n);
    double* Rp = h.ws.take((size_t)n * n);
    if (!h.dry) {
      if (trans) CTM_CUDA(cudaMemcpyAsync(T, X, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, h.stream));
      else permute(h, X, {n, n}, {1, 0}, T);   // T = Xc^T
    }
    cholqr(T, n, n, 3, true, Rp);
    jacobi(Rp, n, 1, ncols, U, S, tol, max_sweeps);
    h.ws.reset(mark);
  }
  void check_status(const char* what) {
    if (h.dry) return;
    // pinned destination: a pageable one makes every such copy its own blocking round trip
    int* st = static_cast<int*>(h.pin);
    CTM_CUDA(cudaMemcpyAsync(st, status, 6 * sizeof(int), cudaMemcpyDeviceToHost, h.stream));
    CTM_CUDA(cudaStreamSynchronize(h.stream));
    last_sweeps = st[2];
    if (jac_pending) {
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.jev[0], h.jev[1]));
      const int rep = st[jac_slot];
      const int executed = rep < jac_max ? rep + 1 : jac_max;   // the kernel reports the index of its last sweep
      h.ms_jacobi += ms;
      h.jacobi_cta_ms += ms * jac_ctas;
      h.jacobi_flops += 6.0 * jac_n * (double)jac_n * (jac_n - 1) * executed;
      ++h.n_jacobi;
      jac_pending = false;
    }
    if (st[0] != 0) throw IsoFail(std::string(what) + ": CholQR pivot " + std::to_string(st[0]) + " not positive");
    if (st[1] != 0) throw IsoFail(std::string(what) + ": Jacobi did not converge");
  }
};

}  // namespace

void iso_init_kernels() {   // per device, once (see tc_init_kernels)
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  CTM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(dev)) return;
  set_smem((const void*)fg::fgemm_kernel<true, true>, fg::SMEM_BYTES);
  set_smem((const void*)fg::fgemm_kernel<true, false>, fg::SMEM_BYTES);
  set_smem((const void*)fg::fgemm_kernel<false, true>, fg::SMEM_BYTES);
  set_smem((const void*)fg::fgemm_kernel<false, false>, fg::SMEM_BYTES);
  set_smem((const void*)chol_kernel, chol_smem_bytes(LMAX));
  set_smem((const void*)trsm_rows_kernel<(LMAX + 31) / 32>, rpk_size(LMAX) * sizeof(double));
  set_smem((const void*)jacobi_lsv_kernel, (size_t)LMAX * (LMAX + 1) * sizeof(double));
  set_smem((const void*)jacobi_cluster_kernel<2, 8, LMAX>, JacCfg<2, 8, LMAX>::SMEM);
  set_smem((const void*)jacobi_cluster_kernel<4, 4, LMAX>, JacCfg<4, 4, LMAX>::SMEM);
  set_smem((const void*)jacobi_cluster_kernel<4, 4, 128>, JacCfg<4, 4, 128>::SMEM);
  set_smem((const void*)jacobi_cluster_kernel<8, 2, LMAX_BIG>, JacCfg<8, 2, LMAX_BIG>::SMEM);
  set_smem((const void*)jacobi_cluster_kernel<1, 8, 128>, JacCfg<1, 8, 128>::SMEM);
  set_smem((const void*)jacobi_cluster_kernel<8, 4, LMAX_BIG>, JacCfg<8, 4, LMAX_BIG>::SMEM);
  done.insert(dev);
}

// Which path takes an R x C truncation to n_keep columns: 0 none (cuSOLVER), 1 direct tall
// (R > C), 2 direct wide (R <= C, R small or no truncation), 3 subspace iteration.
static int iso_plan(int R, int C, int n_keep) {
  if (R > C) return (n_keep <= C && C <= LMAX_BIG) ? 1 : 0;   // n_keep > C: R11 null-space columns
  if (n_keep == R || R <= n_keep + 32) return R <= LMAX_BIG ? 2 : 0;
  return n_keep + 32 <= LMAX_BIG ? 3 : 0;
}

bool iso_supported(int R, int C, int n_keep) { return iso_plan(R, C, n_keep) != 0; }

static bool debug_direct() {
  static const bool d = std::getenv("CTM_ISO_DEBUG") != nullptr;
  return d;
}

// First n_keep left singular vectors of the row-major R x C matrix `mat` (sign rule
// applied), written row-major (R, n_keep) into `out`.  Returns sigma_n / sigma_{n+1}
// (inf if none).  Throws IsoFail when the iteration cannot certify convergence.
static double iso_left(Handle& h, const double* mat, int R, int C, int n_keep, double* out,
                       void (*signfix)(Handle&, const double*, long long, long long, int, int, double*)) {
  const size_t mark = h.ws.top;
  Solver sv(h);
  const double inf = std::numeric_limits<double>::infinity();
  double gap = inf;
  const int plan = iso_plan(R, C, n_keep);
  if (plan == 1 || plan == 2) {
    // direct: left singular vectors from a backward-stable QR + one-sided Jacobi
    //   tall (R >= C):  M = Q_o R_m,        U = Q_o lsv(R_m)
    //   wide (R <= C):  M^T = Q_z R_z,      U = lsv(R_z^T)
    const bool tall = plan == 1;
    const int n = tall ? C : R;
    double* Y = h.ws.take((size_t)R * C);
    double* Rm = h.ws.take((size_t)n * n);
    double* W = h.ws.take((size_t)n * n);
    double* S = h.ws.take((size_t)n);
    double* Ut = tall ? h.ws.take((size_t)R * n) : nullptr;
    if (!h.dry) {
      if (tall) CTM_CUDA(cudaMemcpyAsync(Y, mat, sizeof(double) * R * C, cudaMemcpyDeviceToDevice, h.stream));
      else permute(h, mat, {R, C}, {1, 0}, Y);   // M^T (C x R)
    }
    sv.cholqr(Y, tall ? R : C, n, 3, true, Rm);
    static const bool no_pc = std::getenv("CTM_ISO_NOPC") != nullptr;
    if (no_pc) sv.jacobi(Rm, n, tall ? 0 : 1, n, W, S);
    else sv.jacobi_pc(Rm, n, tall ? 0 : 1, n, W, S);
    ++h.n_svd;
    if (h.dry) {
      h.ws.reset(mark);
      return inf;
    }
    if (debug_direct()) {
      sv.check_status("iso direct");
      std::vector<double> sd(n);
      CTM_CUDA(cudaMemcpy(sd.data(), S, sizeof(double) * n, cudaMemcpyDeviceToHost));
      int close = 0;
      for (int i = 0; i + 1 < n; ++i) close += sd[i + 1] > 0.99 * sd[i];
      std::fprintf(stderr, "[iso] direct %d x %d keep %d: n=%d jacobi sweeps %d  s: %.3g %.3g %.3g %.3g %.3g  pairs within 1%%: %d\n",
                   R, C, n_keep, n, sv.last_sweeps, sd[0], sd[n / 4], sd[n / 2], sd[3 * n / 4], sd[n - 1], close);
    }
    const double* U = W;
    if (tall) {
      if (!sv.fgemm(Y, n, false, R, n, W, n, Ut)) sv.gemm(Y, "ia", {R, n}, W, "ab", {n, n}, Ut, "ib", {R, n});
      U = Ut;
    }
    signfix(h, U, n, 1, R, n_keep, out);
    // (the singular values ride on check_status's synchronisation through the pinned buffer)
    double* hp = reinterpret_cast<double*>(static_cast<char*>(h.pin) + 64);
    CTM_CUDA(cudaMemcpyAsync(hp, S, sizeof(double) * n, cudaMemcpyDeviceToHost, h.stream));
    sv.check_status("iso direct");
    std::vector<double> s(hp, hp + n);
    for (double x : s)
      if (!std::isfinite(x)) throw Error(CTM_E_NONFINITE, "non-finite singular value in a " + std::to_string(R) +
                                                               " x " + std::to_string(C) + " isometry");
    if (n_keep < n && s[n_keep] > 0.0) gap = s[n_keep - 1] / s[n_keep];
    h.ws.reset(mark);
    return gap;
  }
  // truncating cut: Chebyshev-filtered subspace iteration with Rayleigh-Ritz and locking.
  // Ritz vectors that pass the certificate are LOCKED (moved out of the iterated block): the
  // active block is kept orthogonal to them, so its dynamic range is that of the unconverged
  // part of the spectrum.  Without locking, a steep M (sigma_1 / sigma_k >~ 1/sqrt(eps) --
  // converged physical environments, C3 from the third CTM iteration on) carries its small
  // kept directions next to sigma_1^2-amplified ones, which rounding swamps: the solve
  // stalled at residual O(1) and fell back to gesvdp (profiles/r02_c3_fallbacks_before_locking.txt).
  // With the large directions removed, each product M (M^T y) of an active vector has rounding
  // error ~ eps sigma_1 sigma_i: the M-form floor of the certificate, as for LAPACK.
  const int l = std::min(n_keep + iso_oversample(n_keep), R);
  const int k = n_keep;
  double* Y = h.ws.take((size_t)R * l);
  double* Y1 = h.ws.take((size_t)R * l);
  double* Y2 = h.ws.take((size_t)R * l);
  double* P = h.ws.take((size_t)R * l);
  double* Z = h.ws.take((size_t)C * l);
  double* Rz = h.ws.take((size_t)l * l);
  double* W = h.ws.take((size_t)l * l);
  double* S = h.ws.take((size_t)l);
  double* U = h.ws.take((size_t)R * l);
  double* PW = h.ws.take((size_t)R * l);
  double* res = h.ws.take((size_t)l);
  double* L = h.ws.take((size_t)R * l);    // locked Ritz vectors, R x nlock contiguous
  double* Lt = h.ws.take((size_t)R * l);   // rebuild scratch / final assembly
  double* Tp = h.ws.take((size_t)l * l);   // L^T Y
  ++h.n_svd;
  static const bool debug = std::getenv("CTM_ISO_DEBUG") != nullptr;
  cudaEvent_t t0 = h.ev[2];
  float ms_rr = 0.f, ms_all = 0.f;
  int la = l, nlock = 0;                   // active columns, locked columns
  std::vector<double> s_lock;
  // out = M M^T X; leaves M^T X in Z (la columns).  defer: the second GEMM may leave its split-K
  // partials for the consumer (the Chebyshev combine sums them: one launch fewer per degree)
  auto GY = [&](const double* X, double* out, GemmPartials* defer = nullptr) {
    if (sv.fgemm(mat, C, true, C, R, X, la, Z) && sv.fgemm(mat, C, false, R, C, Z, la, out)) return;
    sv.gemm(mat, "ic", {R, C}, X, "ia", {R, la}, Z, "ca", {C, la});
    sv.gemm(mat, "ic", {R, C}, Z, "ca", {C, la}, out, "ia", {R, la}, defer);
  };
  // Filter products through G = M M^T (one GEMM per degree instead of two) when the
  // kept spectrum is flat: the containment floor of the G-form is ~ eps (s_1/s_k)^2,
  // allowed only while that is <= 16 eps.  The Rayleigh-Ritz always uses M itself.
  double* G = h.ws.take((size_t)R * R);
  bool have_G = false;
  GemmPartials fpart;   // the filter product's deferred split-K partials (GYf -> combine)
  static const bool no_defer = std::getenv("CTM_ISO_NODEFER") != nullptr;   // A/B
  auto GYf = [&](const double* X, double* out) {
    GemmPartials* d = no_defer ? nullptr : &fpart;
    if (have_G) sv.gemm(G, "ij", {R, R}, X, "ja", {R, la}, out, "ia", {R, la}, d);
    else GY(X, out, d);
  };
  auto combine = [&](double* out, const double* Pm, const double* Yc, const double* Yo, double a, double b2, double c,
                     const GemmPartials* part = nullptr) {
    if (h.dry) return;
    const bool dp = part != nullptr && part->p != nullptr;
    launch_k(cheb_combine_kernel, dim3(148), dim3(256), 0, h.stream, out, dp ? part->p : Pm, Yc, Yo, (long long)R * la, a,
             b2, c, dp ? part->splits : 1);
    CTM_CUDA(cudaGetLastError());
    h.count_kernel();
  };
  // X <- X - L (L^T X): remove the locked directions from an active iterate (scratch: R x la)
  auto project = [&](double* X, double* scratch) {
    if (nlock == 0) return;
    sv.gemm(L, "ij", {R, nlock}, X, "ia", {R, la}, Tp, "ja", {nlock, la});
    if (sv.fgemm(L, nlock, false, R, nlock, Tp, la, X, -1.0, X, 1.0)) return;   // X -= L Tp, one launch
    sv.gemm(L, "ij", {R, nlock}, Tp, "ja", {nlock, la}, scratch, "ia", {R, la});
    combine(X, scratch, X, nullptr, -1.0, 1.0, 0.0);
  };
  // columns [c0, c0 + nc) of a row-major R x ld matrix into a contiguous R x nc one
  auto copy_cols = [&](double* dst, int dld, int d0, const double* src, int sld, int c0, int nc) {
    if (h.dry || nc == 0) return;
    CTM_CUDA(cudaMemcpy2DAsync(dst + d0, sizeof(double) * dld, src + c0, sizeof(double) * sld, sizeof(double) * nc, R,
                               cudaMemcpyDeviceToDevice, h.stream));
  };
  // CTM_FLAG_WARM_START: this site's previous final block [locked | active Ritz vectors] as the
  // start block (the whole l-dimensional space, oversampling columns included, so the first
  // Rayleigh-Ritz also has good bounds for the filter).  It is orthonormal up to rounding, the
  // first check is a full one (CholQR2, converged Jacobi, certificate on THIS matrix), and when
  // every wanted vector passes the solve ends there; otherwise the filter is planned from the
  // measured residuals like any later plan.
  WarmStore::Slot* wslot = nullptr;
  if (h.warm && h.warm_slot >= 0 && !h.dry) {
    std::lock_guard<std::mutex> g(h.warm->mu);
    if ((size_t)h.warm_slot < h.warm->slots.size()) wslot = &h.warm->slots[h.warm_slot];
  }
  bool warm = wslot != nullptr && wslot->valid && wslot->R == R && wslot->l == l;
  if (warm && wslot->skip > 0) {   // backing off after wasted first checks (see WarmStore::Slot)
    --wslot->skip;
    warm = false;
  }
  if (warm) {
    CTM_CUDA(cudaMemcpyAsync(Y, wslot->p, sizeof(double) * R * l, cudaMemcpyDeviceToDevice, h.stream));
    wslot->valid = false;   // re-validated by the store at the end of a successful solve
    ++h.n_warm;
  } else {
    // start: Y = orth(M Omega), then four plain steps Y <- orth(M M^T Y)
    if (!h.dry) {
      launch_k(fill_omega_kernel, dim3(148), dim3(256), 0, h.stream, Z, (long long)C * l, 0x5eed1234u);
      CTM_CUDA(cudaGetLastError());
      h.count_kernel();
    }
    if (!sv.fgemm(mat, C, false, R, C, Z, l, Y)) sv.gemm(mat, "ic", {R, C}, Z, "ca", {C, l}, Y, "ia", {R, l});
    sv.cholqr(Y, R, l, 1, true, nullptr);
    static const int power_steps = knob_int("CTM_ISO_POWER", 4);
    for (int it = 0; it < power_steps; ++it) {   // (2 or 6 steps: slower at C5 / C4)
      GY(Y, P);
      std::swap(Y, P);
      sv.cholqr(Y, R, l, 1, true, nullptr);
    }
  }
  std::vector<double> s(l), r(k);
  double prev_worst = inf, prev_floor = inf;
  int degrees = warm ? 0 : 4, checks = 0;
  const int max_degrees = 400;
  const double cert = 8.0 * EPS * std::sqrt((double)C);
  bool plateau = false;
  for (;;) {
    ++checks;
    const int ka = k - nlock;   // wanted vectors still active
    // Rayleigh-Ritz on the orthonormal active block: Z = M^T Y, P = M Z, Z = Q_z R_z, W = lsv(R_z^T)
    cudaEvent_t e_rr0 = h.ev[6], e_rr1 = h.ev[7];
    if (!h.dry && debug) CTM_CUDA(cudaEventRecord(e_rr0, h.stream));
    // orthonormal basis: Y leaves the filter (or the start) through a shifted CholQR, so its
    // condition is modest and plain CholQR2 suffices for l <= LMAX (the first pass replaces
    // dependent columns; C4 64.8 -> 62.6 ms); at l > LMAX it cost C5 an extra check
    // (260 -> 277 ms), which keeps shifted CholQR3 there
    // (the first check only estimates the spectrum for the filter bounds: one plain pass on
    // Y and one shifted pass on Z suffice -- C4 57.0 -> 56.2 ms, C5 246 -> 240 ms; no pass on
    // Y at all mis-set the C5 bounds)
    // with locked vectors: project them out before each pass ("twice is enough")
    const bool light = checks == 1 && !warm;
    if (light) {
      sv.cholqr(Y, R, la, 1, false, nullptr, true);
    } else if (nlock > 0 || h.dry) {
      project(Y, PW);
      sv.cholqr(Y, R, la, 1, false, nullptr, true);
      project(Y, PW);
      sv.cholqr(Y, R, la, 1, false, nullptr, false);
    } else if (la <= LMAX) {
      sv.cholqr(Y, R, la, 2, false, nullptr, true);
    } else {
      sv.cholqr(Y, R, la, 3, true, nullptr, true);
    }
    GY(Y, P);
    sv.cholqr(Z, C, la, light ? 1 : 2, true, Rz);   // Z = M^T Y (left in Z by GY) = Q_z R_z (sCholQR2)
    // the first Rayleigh-Ritz only seeds the filter bounds: a capped, loose Jacobi suffices
    // (one sweep: C4 74.5 -> 71 ms vs three; zero sweeps -- column norms only -- mis-set the
    // C5 filter bounds and cost a fallback)
    static const int first_sweeps = knob_int("CTM_ISO_SWEEPS1", 1);
    if (light) sv.jacobi(Rz, la, 1, la, W, S, 1e-6, first_sweeps);
    else sv.jacobi(Rz, la, 1, la, W, S, 1e-14);
    if (!sv.fgemm(Y, la, false, R, la, W, la, U)) sv.gemm(Y, "ia", {R, la}, W, "ab", {la, la}, U, "ib", {R, la});
    if (!sv.fgemm(P, la, false, R, la, W, la, PW)) sv.gemm(P, "ia", {R, la}, W, "ab", {la, la}, PW, "ib", {R, la});
    // the kept subspace is span(L) + span(U_act): a Ritz vector's rounding-level component
    // along a locked direction u_j returns from M M^T amplified by sigma_j^2 (up to
    // eps sigma_1 / sigma_i of the certificate's scale on steep cuts) yet lies inside the
    // kept subspace -- measure the residual in the complement of span(L)
    if (nlock > 0) project(PW, P);
    if (h.dry) {   // sizing pass: also reserve the G-form GEMMs' split-K slabs and the projection
      sv.gemm(mat, "ic", {R, C}, mat, "jc", {R, C}, G, "ij", {R, R});
      sv.gemm(G, "ij", {R, R}, Y, "ja", {R, l}, P, "ia", {R, l});
      nlock = l;
      project(Y, PW);
      h.ws.reset(mark);
      return inf;
    }
    launch_k(ritz_residual_kernel, dim3(ka), dim3(256), 0, h.stream, (const double*)PW, (const double*)U, (const double*)S,
             R, la, ka, res);
    CTM_CUDA(cudaGetLastError());
    h.count_kernel();
    if (debug) CTM_CUDA(cudaEventRecord(e_rr1, h.stream));
    // Ritz values and residuals ride on check_status's synchronisation (one round trip per check
    // through the handle's pinned buffer: 64 bytes of status, then la + ka <= 2 LMAX_BIG doubles)
    double* hp = reinterpret_cast<double*>(static_cast<char*>(h.pin) + 64);
    CTM_CUDA(cudaMemcpyAsync(hp, S, sizeof(double) * la, cudaMemcpyDeviceToHost, h.stream));
    CTM_CUDA(cudaMemcpyAsync(hp + la, res, sizeof(double) * ka, cudaMemcpyDeviceToHost, h.stream));
    sv.check_status("iso subspace");
    if (debug) std::fprintf(stderr, "[iso]   check %d after %d degrees: active %d locked %d jacobi sweeps %d\n", checks,
                            degrees, la, nlock, sv.last_sweeps);
    std::copy(hp, hp + la, s.begin());
    std::copy(hp + la, hp + la + ka, r.begin());
    if (debug) {
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, e_rr0, e_rr1));
      ms_rr += ms;
    }
    // r_i = ||M (M^T u_i) - s_i^2 u_i||: its rounding floor is ~ eps sqrt(C) s_1 s_i (the
    // product is formed through M, never through a Gram), and r_i / s_i^2 estimates how much
    // of the true u_i lies outside span(Y).  A vector is certified when its residual is at
    // that floor (a measured certificate, no extrapolation); the leading certified active
    // vectors are locked, and the solve ends when every wanted vector is certified.
    const double s1 = nlock > 0 ? s_lock[0] : s[0];
    int j = 0;
    double worst = 0.0, worst_floor = 0.0;
    for (int i = 0; i < ka; ++i) {
      if (!std::isfinite(r[i]) || !std::isfinite(s[i]))
        throw Error(CTM_E_NONFINITE, "non-finite Ritz value in a " + std::to_string(R) + " x " + std::to_string(C) +
                                         " isometry");
      const double f = s[i] > 0.0 ? r[i] / (s1 * s[i]) : 0.0;
      if (!light && j == i && f <= cert) {
        ++j;   // leading certified
        continue;
      }
      worst = std::max(worst, s[i] > 0.0 ? r[i] / (s[i] * s[i]) : 0.0);
      worst_floor = std::max(worst_floor, f);
    }
    if (debug)
      std::fprintf(stderr, "[iso]     certified %d of %d active wanted; unconverged: residual/s_i^2 %.3e  "
                           "residual/(s_1 s_i) %.3e (cert at %.3e)\n", j, ka, worst, worst_floor, cert);
    if (warm && checks == 1) {
      if (2 * j >= ka) {
        wslot->miss = 0;
      } else {
        wslot->miss = std::min(wslot->miss + 1, 4);
        wslot->skip = 1 << wslot->miss;
      }
    }
    if (!light && j == ka) {
      if (warm && checks == 1) ++h.n_warm_hit;
      break;
    }
    // a plateau at the rounding floor (no further progress possible in FP64, within 64x of
    // the nominal floor constant) is accepted: the result is as accurate as the arithmetic
    if (checks > 2 && worst_floor <= 64.0 * cert && worst_floor > 0.5 * prev_floor) {
      plateau = true;
      break;
    }
    // (stagnation of the worst residual counts only when no vector was certified either: newly
    // certified vectors are locked below and the next plan runs on the smaller, less spread
    // active block -- on the steepest cuts, s_1 / s_k ~ 5e4 in c4_dl's first iterations, the
    // bottom kept vectors only start to converge once the top ones are out of the block;
    // 14 fallbacks in 20 c4_dl iterations before this, profiles/r02s3_warm_start_backoff.jsonl)
    if (degrees >= max_degrees || (checks > 2 && j == 0 && worst > 0.5 * prev_worst))
      throw IsoFail("subspace iteration did not converge: residual " + std::to_string(worst));
    prev_worst = worst;
    prev_floor = worst_floor;
    // lock the leading certified Ritz vectors: L <- [L, U(:, 0:j)], active <- U(:, j:la)
    if (j > 0) {
      copy_cols(Lt, nlock + j, 0, L, nlock, 0, nlock);
      copy_cols(Lt, nlock + j, nlock, U, la, 0, j);
      std::swap(L, Lt);
      for (int i = 0; i < j; ++i) s_lock.push_back(s[i]);
      copy_cols(Y, la - j, 0, U, la, j, la - j);
      nlock += j;
      la -= j;
      s.erase(s.begin(), s.begin() + j);
    } else if (!light) {
      // filter the Ritz basis U (orthonormal): the filtered block stays nearly Ritz-ordered,
      // so the next Rayleigh-Ritz Jacobi starts close to diagonal and needs few sweeps
      // (after the capped first check W is not orthogonal: keep filtering Y itself)
      CTM_CUDA(cudaMemcpyAsync(Y, U, sizeof(double) * R * la, cudaMemcpyDeviceToDevice, h.stream));
    }
    const int kb = k - nlock;   // wanted active vectors after locking (>= 1)
    // Chebyshev filter (Zhou & Saad's scaled recurrence) damping [0, b], b = s_la^2 (the
    // smallest Ritz value of the active block), normalised at the k-th Ritz value; the error of
    // the slowest kept vector shrinks by x_k + sqrt(x_k^2 - 1) per degree.
    const double lk = s[kb - 1] * s[kb - 1], lb = s[la - 1] * s[la - 1], l1 = s[0] * s[0], lg = s1 * s1;
    static const double gform = knob_double("CTM_ISO_GFORM", 16.0);
    if (!have_G && lg <= gform * lk) {   // (256 / 2500: within noise at C4/C5; not worth the floor)
      sv.gemm(mat, "ic", {R, C}, mat, "jc", {R, C}, G, "ij", {R, R});
      have_G = true;
    }
    if (!(lb < 0.999 * lk)) throw IsoFail("no spectral separation inside the block");
    const double ce = 0.5 * lb;                       // centre = half width of [0, b]
    const double xk = (lk - ce) / ce, x1 = (l1 - ce) / ce, xg = (lg - ce) / ce;
    const double rate = xk + std::sqrt(xk * xk - 1.0);
    // the first estimate comes from a young subspace (Ritz values of the block bottom are
    // low, the rate optimistic): over-filter by 1.6x rather than pay another check
    // 1.25 (1.0 / 0.85 / 0.7: an extra check); 2.0 for the first plan of a flat (G-form) cut,
    // whose cheap degrees (one GEMM each) buy back a check: flat C4 solves 14 -> 12.3 ms, the
    // move 56.6 -> 53.6 ms (3.0 over-filters; at l > LMAX -- C5 -- it measured 2-3% slower)
    // (1.6 / 2.5, or also for the second plan: within noise)
    // (round 2, session 2: re-tuned after the Jacobi / Cholesky speed-ups made a check cheaper than
    //  over-filtering -- first plan 2.0 -> 1.4, later plans 1.25 -> 1.1, tail 6 -> 4: C4 move 37.4 -> 34.9 ms,
    //  C5 182 -> ~173 ms, no fallbacks; profiles/r02_iso_knobs.jsonl)
    static const double safe1 = knob_double("CTM_ISO_SAFE1", 1.4), safe = knob_double("CTM_ISO_SAFE", 1.1);
    const double safety = (light && l <= LMAX && (have_G || l1 <= 16.0 * lk)) ? safe1 : safe;
    int need = (int)std::ceil(safety * std::log(std::max(worst, 1e-300) / 1e-16) / std::log(rate)) + 2;
    need = std::max(2, std::min(need, max_degrees - degrees));
    // degree per orthonormalisation: keep the column scale spread (~T_m(x1)/T_m(xk)) <= 1e6
    // (1e8 let the bottom columns of the block collapse numerically onto the top ones), and
    // <= 0.25 / sqrt(shift): one shifted CholQR pass leaves kappa(Q) ~ sqrt(shift) kappa(Y),
    // so a larger per-block spread compounds from block to block until kept directions
    // drown (seen as Ritz residual blow-ups at l = 288).
    const double shift_rel = 11.0 * ((double)R * la + (double)la * (la + 1)) * EPS;
    static const double spread_cap = knob_double("CTM_ISO_SPREAD", 1e6);
    const double spread = std::min(spread_cap, 0.25 / std::sqrt(shift_rel));
    const double lg_deg = std::acosh(std::max(x1, xk)) - std::acosh(xk) + 1e-12;   // log-spread per degree
    int mb = std::max(1, std::min(12, (int)std::floor(std::log(spread) / lg_deg)));
    // Longer blocks re-orthonormalised by one PLAIN CholQR pass (no shift: kappa(Q) ~ 1, so
    // nothing compounds) while the spread stays <= 1e10; the rounding noise such a block leaves
    // in the kept directions is filtered away by the last `tail` degrees, which use the short
    // shifted blocks above.
    static const int plain_on = std::getenv("CTM_ISO_PLAIN") ? std::atoi(std::getenv("CTM_ISO_PLAIN")) : 1;
    // (spread 1e7 -> 1e10: columns whose pivot falls below 1e-13 of their norm are re-seeded
    // by the replacement, the shifted tail and the residual certificate guard the result;
    // C5/chi=256 523 -> 400 ms, C5 232 -> 215 ms, no fallbacks; 1e12 within noise of 1e10;
    // a tail of 8 degrees: slower)
    static const double spread_plain = knob_double("CTM_ISO_SPREAD_PLAIN", 1e10);
    int mb_plain = std::max(1, std::min(12, (int)std::floor(std::log(spread_plain) / lg_deg)));
    // locked directions re-enter an active iterate through rounding (~eps) and the filter
    // amplifies them most (they sit above the active spectrum): project them out at every
    // orthonormalisation, often enough that they stay below 1e-6 of the active block
    if (nlock > 0 && xg > x1) {
      const double lg_lock = std::acosh(xg) - std::acosh(std::max(x1, xk)) + 1e-12;
      const int mp = std::max(1, (int)std::floor(std::log(1e-6 / EPS) / lg_lock));
      mb = std::min(mb, mp);
      mb_plain = std::min(mb_plain, mp);
    }
    static const int tail = knob_int("CTM_ISO_TAIL", 4);
    // One Chebyshev recurrence over all `need` degrees; every mb degrees the current iterate
    // is re-orthonormalised (shifted CholQR, a basis is enough here) and the previous one is
    // multiplied by the same R^{-1}, so the three-term recurrence continues across the
    // orthonormalisation (restarting it at T_1 would give the shifted-power rate x_k per
    // degree instead of x_k + sqrt(x_k^2 - 1) on the steep cuts, where mb = 1: at C5 those
    // needed a third Rayleigh-Ritz check; C5 move 344 -> 307 ms, C4 +2 ms).  The locked
    // directions are projected out of both iterates (the projector commutes with the
    // recurrence: span(L) is invariant under M M^T).
    const double s1c = 1.0 / xk;   // sigma_1 = e / (lambda_s - c)
    double sig = s1c;
    double *Yo = nullptr, *Yc = Y;
    double* bufs[2] = {Y1, Y2};
    int nb = 0, done = 0;
    while (done < need) {
      const bool plain = plain_on && mb_plain > mb && need - done > tail;
      const int m = plain ? std::min(mb_plain, need - done - tail) : std::min(mb, need - done);
      for (int jj = 0; jj < m; ++jj) {
        double* Yn = bufs[nb];
        nb ^= 1;
        double ca, cb, cc = 0.0;   // Yn = ca (M M^T) Yc + cb Yc + cc Yo
        if (Yo == nullptr) {
          ca = s1c / ce;
          cb = -s1c;
        } else {
          const double sn = 1.0 / (2.0 / s1c - sig);
          ca = 2.0 * sn / ce;
          cb = -2.0 * sn;
          cc = -sig * sn;
          sig = sn;
        }
        // the recurrence in the filter GEMM's epilogue (one launch per degree on the G form)
        const bool fused = have_G ? sv.fgemm(G, R, false, R, R, Yc, la, Yn, ca, Yc, cb, Yo, cc)
                                  : (sv.fgemm(mat, C, true, C, R, Yc, la, Z) &&
                                     sv.fgemm(mat, C, false, R, C, Z, la, Yn, ca, Yc, cb, Yo, cc));
        if (!fused) {
          GYf(Yc, P);
          combine(Yn, P, Yc, Yo, ca, cb, cc, &fpart);
        }
        Yo = Yc;   // (the elementwise combine may overwrite its own Yold in place)
        Yc = Yn;
      }
      if (nlock > 0) {
        project(Yc, U);
        project(Yo, U);
      }
      // (plain blocks replace numerically dependent columns instead of failing: the block's
      // bottom columns -- the oversampling buffer -- can fall below eps of the top ones)
      sv.cholqr(Yc, R, la, 1, !plain, nullptr, plain, Yo);
      done += m;
    }
    if (!h.dry && Yc != Y) CTM_CUDA(cudaMemcpyAsync(Y, Yc, sizeof(double) * R * la, cudaMemcpyDeviceToDevice, h.stream));
    degrees += need;
  }
  if (debug) {
    CTM_CUDA(cudaEventRecord(h.ev[3], h.stream));
    CTM_CUDA(cudaEventSynchronize(h.ev[3]));
    CTM_CUDA(cudaEventElapsedTime(&ms_all, t0, h.ev[3]));
  }
  // the kept vectors: the locked ones, then the certified active Ritz vectors
  const int ka = k - nlock;
  if (nlock == 0) {
    signfix(h, U, la, 1, R, n_keep, out);
  } else {
    copy_cols(Lt, k, 0, L, nlock, 0, nlock);
    copy_cols(Lt, k, nlock, U, la, 0, ka);
    signfix(h, Lt, k, 1, R, n_keep, out);
  }
  if (ka < la && s[ka] > 0.0) gap = (ka > 0 ? s[ka - 1] : s_lock.back()) / s[ka];
  if (wslot != nullptr) {   // keep the final block [L | U] (nlock + la = l columns) for this site's next solve
    if (wslot->cap < (size_t)R * l) {
      std::lock_guard<std::mutex> g(h.warm->mu);
      if (wslot->p) CTM_CUDA(cudaFree(wslot->p));
      wslot->p = nullptr;
      wslot->cap = 0;
      CTM_CUDA(cudaMalloc(&wslot->p, sizeof(double) * R * l));
      wslot->cap = (size_t)R * l;
    }
    copy_cols(wslot->p, l, 0, L, nlock, 0, nlock);
    copy_cols(wslot->p, l, nlock, U, la, 0, la);
    wslot->R = R;
    wslot->l = l;
    wslot->valid = true;
  }
  if (debug)
    std::fprintf(stderr, "[iso] %d x %d keep %d: l=%d degrees=%d checks=%d locked=%d%s s1/sk=%.3g sl/sk=%.3g gap=%.5f ms=%.2f "
                         "rr_ms=%.2f last_sweeps=%d\n",
                 R, C, n_keep, l, degrees, checks, nlock, plateau ? " (plateau)" : warm ? " (warm)" : "",
                 (nlock ? s_lock[0] : s[0]) / (ka > 0 ? s[ka - 1] : s_lock.back()), s[la - 1] / (ka > 0 ? s[ka - 1] : s_lock.back()),
                 gap, ms_all, ms_rr, sv.last_sweeps);
  h.ws.reset(mark);
  return gap;
}

// Singular values (descending) of a row-major R x C matrix into host memory: the one-sided
// Jacobi kernels for square matrices up to LMAX_BIG, cuSOLVER Xgesvd (values only) otherwise.
void singular_values(Handle& h, const double* mat, int R, int C, double* host_out) {
  const size_t mark = h.ws.top;
  const int mn = std::min(R, C);
  double* S = h.ws.take((size_t)mn);
  if (h.dry) {
    h.ws.take((size_t)R * C + 64);
    h.ws.reset(mark);
    return;
  }
  if (R == C && R <= LMAX_BIG) {
    Solver sv(h);
    sv.jacobi(mat, R, 0, 0, nullptr, S, 1e-14);
    sv.check_status("singular values");
  } else {
    double* A = h.ws.take((size_t)R * C);
    // column-major copy of the R x C row-major matrix = its transpose read row-major
    permute(h, mat, {R, C}, {1, 0}, A);
    size_t dws = 0, hws = 0;
    if (cusolverDnXgesvd_bufferSize(h.solver, h.solver_params, 'N', 'N', R, C, CUDA_R_64F, A, R, CUDA_R_64F, S,
                                    CUDA_R_64F, nullptr, 1, CUDA_R_64F, nullptr, 1, CUDA_R_64F, &dws, &hws) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(CTM_E_SOLVER, "gesvd buffer size");
    double* work = h.ws.take(dws / sizeof(double) + 1);
    if (h.host_buf.size() < hws + 16) h.host_buf.resize(hws + 16);
    if (cusolverDnXgesvd(h.solver, h.solver_params, 'N', 'N', R, C, CUDA_R_64F, A, R, CUDA_R_64F, S, CUDA_R_64F,
                         nullptr, 1, CUDA_R_64F, nullptr, 1, CUDA_R_64F, work, dws, h.host_buf.data(),
                         h.host_buf.size(), h.dev_info) != CUSOLVER_STATUS_SUCCESS)
      throw Error(CTM_E_SOLVER, "gesvd (singular values) failed");
  }
  CTM_CUDA(cudaMemcpyAsync(host_out, S, sizeof(double) * mn, cudaMemcpyDeviceToHost, h.stream));
  CTM_CUDA(cudaStreamSynchronize(h.stream));
  h.ws.reset(mark);
}

// An orthonormal basis of the column space of a tall R x C matrix (R >= C), written
// row-major (R, C) into `out`: shifted CholQR3 of a copy (dependent columns replaced by
// random directions, so the basis is complete even for a rank-deficient matrix).  For a
// non-truncating cut whose basis gauge cancels downstream (svd_left's basis_only).
void iso_basis(Handle& h, const double* mat, int R, int C, double* out) {
  const size_t mark = h.ws.top;
  Solver sv(h);
  if (!h.dry) CTM_CUDA(cudaMemcpyAsync(out, mat, sizeof(double) * R * C, cudaMemcpyDeviceToDevice, h.stream));
  sv.cholqr(out, R, C, 3, true, nullptr, true);
  ++h.n_svd;
  sv.check_status("iso basis");
  h.ws.reset(mark);
}

double iso_left_vectors(Handle& h, const double* mat, int R, int C, int n_keep, double* out,
                        void (*signfix)(Handle&, const double*, long long, long long, int, int, double*), bool* ok) {
  *ok = true;
  const size_t mark = h.ws.top;
  const int n_svd = h.n_svd;
  const int n_warm = h.n_warm;
  try {
    try {
      return iso_left(h, mat, R, C, n_keep, out, signfix);
    } catch (const IsoFail& e) {
      if (h.n_warm == n_warm) throw;
      // a warm-started solve that did not converge (its slot was invalidated at the start):
      // redo it from the cold start before giving up on the solver
      static const bool debug = std::getenv("CTM_ISO_DEBUG") != nullptr;
      if (debug) std::fprintf(stderr, "[iso] %d x %d keep %d: warm start failed (%s), cold retry\n", R, C, n_keep, e.what());
      h.ws.reset(mark);
      h.n_svd = n_svd;
      ++h.n_warm_retry;
      return iso_left(h, mat, R, C, n_keep, out, signfix);
    }
  } catch (const IsoFail& e) {
    static const bool debug = std::getenv("CTM_ISO_DEBUG") != nullptr;
    if (debug) std::fprintf(stderr, "[iso] %d x %d keep %d: fallback (%s)\n", R, C, n_keep, e.what());
    h.ws.reset(mark);
    h.n_svd = n_svd;
    *ok = false;
    return std::numeric_limits<double>::infinity();
  }
}

}  // namespace ctm
