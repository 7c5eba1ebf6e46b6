// ctm_internal.h -- host-side internals of libctm (not part of the ABI).
#pragma once
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ctm.h"
#include "tc_gemm.cuh"

namespace ctm {

// Error carrying an ABI status code; caught at the ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CTM_CUDA(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw ::ctm::Error(CTM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));  \
  } while (0)

// A (batch of) row-major tensor operand(s): labels name the legs, ext their extents.
struct Operand {
  std::vector<const double*> p;
  std::string lab;
  std::vector<int> ext;
};
struct OutOperand {
  std::vector<double*> p;
  std::string lab;
  std::vector<int> ext;
  std::vector<double*> sumsq;   // optional fused sum of squares (one per batch entry)
};

// Bump allocator over the caller-provided workspace.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, top = 0, peak = 0;
  bool dry = false;   // sizing pass: count bytes without a buffer
  double* take(size_t n_doubles) {
    size_t bytes = (n_doubles * sizeof(double) + 255) & ~size_t(255);
    if (!dry && top + bytes > cap)
      throw Error(CTM_E_NOMEM, "workspace too small: need > " + std::to_string(top + bytes) +
                                   " bytes, have " + std::to_string(cap));
    // sizing pass: a fake, never dereferenced, non-null address
    double* r = reinterpret_cast<double*>((dry ? reinterpret_cast<char*>(4096) : base) + top);
    top += bytes;
    if (top > peak) peak = top;
    return r;
  }
  void reset(size_t to = 0) { top = to; }
};

// CTM_FLAG_WARM_START: the final iterated block (locked + active Ritz vectors, R x l) of every
// truncating solve of a move, kept per solve site (direction, absorption, cut) and used as
// the start block of the same site's next solve.  In a CTM iteration the environment -- and
// with it every M -- converges, so the previous subspace is a near-solution; the solve still
// ends only on the residual certificate of the NEW matrix (iso.cu), so the result does not
// depend on the start beyond rounding.  Owned by the main handle, shared with its workers.
struct WarmStore {
  struct Slot {
    double* p = nullptr;   // device, R x l row-major
    size_t cap = 0;        // doubles allocated
    int R = 0, l = 0;
    bool valid = false;
    // back-off: a site whose warm first check certified less than half of the wanted vectors (an
    // environment that is not converging: the check was wasted) skips its next min(2^miss, 16)
    // warm attempts (the block is still refreshed by every solve); a good attempt resets it
    int miss = 0, skip = 0;
  };
  std::mutex mu;           // slot allocation (cudaMalloc from worker threads)
  std::vector<Slot> slots;
  ~WarmStore() {
    for (auto& s : slots)
      if (s.p) cudaFree(s.p);
  }
};
constexpr int CTM_WARM_SITES = 6;   // per absorption: x = a, b times {left side, right side, main}

struct Handle {
  ctm_params prm{};
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t solver_params = nullptr;
  gesvdjInfo_t gesvdj_info = nullptr;
  Arena ws;
  std::vector<char> host_buf;          // cuSOLVER host workspace
  int* dev_info = nullptr;              // cuSOLVER info (inside a small private alloc)
  double* dev_scalars = nullptr;        // small device scratch (norms etc.)
  void* pin = nullptr;                  // 8 KB of pinned host memory: the ISO solver's status / Ritz values /
                                        // residuals come back in one stream-ordered round trip per check
  cudaEvent_t ev[8]{};   // 2,3: svd timing; 4,5: isometry fork/join; 6,7: iso solver debug / K7 profile
  cudaEvent_t jev[2]{};  // ISO solver: the pending Jacobi launch (ms_jacobi)
  std::string last_error;
  int64_t kernel_count = 0;
  // per-call statistics
  double ms_svd = 0.0;
  double ms_iso = 0.0;                  // isometry-stage wall time (fork -> join)
  double flops = 0.0;
  double min_gap = 1e300;
  int n_svd = 0;
  int n_svd_fallback = 0;               // CTM_SVD_ISO truncations handed to cuSOLVER
  // CTM_FLAG_WARM_START (see WarmStore): the store (main handle owns, workers point to it), the
  // slot of the next truncating solve on this handle (-1: cold start), the move direction
  int n_warm = 0, n_warm_hit = 0;       // warm-started solves / of those certified at the first check
  int n_warm_retry = 0;                 // warm-started solves that failed and were redone cold
  std::shared_ptr<WarmStore> warm;
  int warm_slot = -1;
  int warm_dir = 0;
  double ms_jacobi = 0.0;               // ISO solver: Jacobi launches, event-timed
  double jacobi_flops = 0.0;
  double jacobi_cta_ms = 0.0;           // launch time x CTAs (1 CTA per SM): SM-weighted time
  int n_jacobi = 0;
  int n_kernels = 0;
  // per-cut truncation gaps of the call (min over its moves; +inf when nothing truncated):
  // main TS stage one, [absorption][cut ab, ba]; side TS stage one, [absorption][a-l, a-r, b-l, b-r]
  double cut_gap[2][2] = {{1e300, 1e300}, {1e300, 1e300}};
  double side_gap[2][4] = {{1e300, 1e300, 1e300, 1e300}, {1e300, 1e300, 1e300, 1e300}};
  int device = 0;                       // CUDA device the handle (and its workers) run on
  double ms_commit = 0.0, commit_bytes = 0.0;   // CTM_FLAG_PROFILE: K7 normalise + commit launches
  int n_commit = 0;
  bool dry = false;                     // sizing pass: no launches
  // CTM_FLAG_PROFILE: event pairs around each tc_gemm launch
  std::vector<cudaEvent_t> prof_ev;
  std::vector<double> prof_flops;
  int prof_used = 0;
  double prof_ms_subs = 0.0, prof_flops_subs = 0.0;   // worker sub-handles' launches, merged
  int prof_n_subs = 0;
  // worker sub-handles (own stream + cuSOLVER handle + workspace slice) for the
  // independent isometry tasks of a column absorption; cuSOLVER blocks the calling host
  // thread, so each worker is driven by its own host thread.
  std::vector<std::unique_ptr<Handle>> subs;
  size_t main_bytes = 0, sub_bytes = 0;
  bool owns_stream = false;
  void count_kernel(int n = 1) { kernel_count += n; n_kernels += n; }
};

// tc_gemm.cu: returns the number of sum-of-squares partials written per problem (slots
// 0..n-1 of C.sumsq[b]; at most CTM_SS_SLOTS).
constexpr int CTM_SS_SLOTS = 4096;
// Deferred split-K reduction: when a contraction with a plain row-major [M][N] output runs
// split-K, contract() may skip its reduction launch and hand the partial slab to the consumer
// (p = slab [splits][M][N], summed in split order like splitk_reduce_kernel); p == nullptr: the
// output was written to C as usual.  The slab stays valid in stream order until the next
// launch that takes workspace.
struct GemmPartials {
  const double* p = nullptr;
  int splits = 1;
  long long mn = 0;
};
int contract(Handle& h, const Operand& A, const Operand& B, const OutOperand& C,
             double alpha = 1.0, GemmPartials* defer = nullptr);
// Per-device one-time kernel attributes (dynamic shared memory > 48 KB): called by ctm_init
// on the handle's device before any worker thread exists (thread-safe, once per device).
void tc_init_kernels();

// kernels.cu
void permute(Handle& h, const double* src, const std::vector<int>& ext, const std::vector<int>& perm,
             double* dst);
void zero(Handle& h, double* p, size_t n);
void sumsq(Handle& h, const std::vector<const double*>& srcs, const std::vector<size_t>& ns,
           double* out);
// dst[i] = src[i] / sqrt(sum_{j < nparts[i]} ss[i*CTM_SS_SLOTS + j]) (partials summed in a fixed lane-strided
// order by one warp, so the result is deterministic)
void scale_commit(Handle& h, const std::vector<const double*>& srcs, const std::vector<double*>& dsts,
                  const std::vector<size_t>& ns, const double* ss, const std::vector<int>& nparts);
void nonfinite_count(Handle& h, const double* p, size_t n, int* dev_count);
void abs_copy(Handle& h, const double* src, double* dst, size_t n);
void dot(Handle& h, const double* a, const double* b, size_t n, double* out);
// rho (2,2,2,2) of the H bond -> (<Sx>_A, <Sz>_A, <Sx>_B, <Sz>_B, m_s) into out (device, 5 doubles)
void site_spins(Handle& h, const double* rho, double* out);   // out = a.b (device)
// rho (d,d,d,d) -> symmetrised, trace-normalised; e = Tr(rho h) into e_dev; rho_out nullable
void rho_finish(Handle& h, const double* rho, const double* hop, int d, double* rho_out, double* e_dev);

// svd.cu: first n_keep left singular vectors of the row-major R x C matrix `mat`
// (input preserved), written row-major (R, n_keep) with the sign rule.  Returns the
// truncation gap sigma_{n}/sigma_{n+1} (inf if none).
// basis_only: when nothing is truncated (n_keep == C <= R) and the caller's result does not
// depend on the basis gauge, any orthonormal basis of the column space is returned
// (CTM_SVD_ISO: shifted CholQR3, no SVD).
double svd_left(Handle& h, const double* mat, int R, int C, int n_keep, double* out, bool basis_only = false);

// ffu.cu: the imaginary-time / fast-full-update bond update (readings
// R25-R28): the horizontal bond A (left) - B (right) against the environment env; A2, B2
// (device, d D^4 each) receive the Frobenius-normalised updated sites; cost (host, nullable)
// = (final N-weighted error, <theta'|N|theta'>).  ffu_gate: g = exp(-delta h) (device d^4).
void ffu_bond_update_h(Handle& h, const double* A, const double* B, const ctm_env* env, const double* gate,
                       int sweeps, double* A2, double* B2, double* cost);
void ffu_gate(Handle& h, const double* hop, double delta, double* g);

// iso.cu: libctm's own truncated SVD (subspace iteration + CholQR + one-sided Jacobi).
#define CTM_ISO_LMAX 160
void iso_init_kernels();
void iso_basis(Handle& h, const double* mat, int R, int C, double* out);
void singular_values(Handle& h, const double* mat, int R, int C, double* host_out);
bool iso_supported(int R, int C, int n_keep);
// ok = false when convergence could not be certified (caller falls back to cuSOLVER).
double iso_left_vectors(Handle& h, const double* mat, int R, int C, int n_keep, double* out,
                        void (*signfix)(Handle&, const double*, long long, long long, int, int, double*), bool* ok);
size_t svd_workspace_doubles(Handle& h, int R, int C);


// Kernel launch with programmatic dependent launch (pdl.cuh) unless CTM_NO_PDL is set: the
// kernel must call CTM_PDL_WAIT() before touching global memory.
inline bool pdl_enabled() {
  static const bool on = std::getenv("CTM_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  const bool pdl = pdl_enabled();
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  CTM_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

}  // namespace ctm
