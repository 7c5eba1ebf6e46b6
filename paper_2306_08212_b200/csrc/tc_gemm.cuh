// tc_gemm.cuh -- FP64 tensor-contraction GEMM on the B200 DMMA pipe (sm_100a).
//
//   C[m, n] = alpha * sum_k A[m, k] * B[k, n]
//
// where m, n and k are multi-indices of up to CTM_MAXMODES modes each and every operand
// is addressed through per-mode element strides, so the index permutations of the
// CTMRG contractions are fused into the tile loads
// and the epilogue instead of being separate transpose passes.
//
// Design:
//  * math: mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4.  sm_100a has no
//    tcgen05 FP64 kind (ptxas rejects .kind::f64) and wgmma is sm_90a-only, so DMMA is
//    the FP64 tensor path; measured 37.1 TFLOP/s peak (= DFMA peak) on this B200.
//  * operand staging: cp.async (LDGSTS, 8 B) gathers from per-mode offset tables kept in
//    shared memory, multi-stage pipeline; the load thread mapping follows whichever index
//    is contiguous in global memory (m- or k-fast for A, k- or n-fast for B) so every
//    warp load is coalesced.
//  * epilogue: accumulators -> shared memory -> global in the order of C's contiguous
//    mode (coalesced stores for either layout), optional fused sum of squares for the
//    Frobenius normalisation (reading R13) accumulated per problem with atomics.
//  * batch: blockIdx.z selects one of up to CTM_MAXBATCH problems sharing shapes and
//    strides (the two chains / corners of an absorption run in one launch).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CTM_MAXMODES 4
#define CTM_MAXBATCH 4
#define CTM_KTAB_MAX 4096

struct TcArgs {
  const double* A[CTM_MAXBATCH];
  const double* B[CTM_MAXBATCH];
  double* C[CTM_MAXBATCH];
  double* sumsq[CTM_MAXBATCH];   // nullable: += sum of squares of the written tile
  int M, N, K;
  int nm, nn, nk;
  int m_ext[CTM_MAXMODES], n_ext[CTM_MAXMODES], k_ext[CTM_MAXMODES];
  int a_m[CTM_MAXMODES], a_k[CTM_MAXMODES];
  int b_k[CTM_MAXMODES], b_n[CTM_MAXMODES];
  int c_m[CTM_MAXMODES], c_n[CTM_MAXMODES];
  int a_kfast, b_kfast, c_nfast;
  double alpha;
  double beta;     // C = alpha*A*B + beta*C (beta != 0 only for K-chunked accumulation)
};

namespace tc {

__device__ __forceinline__ int mode_offset(int idx, int nmodes, const int* ext, const int* str) {
  int off = 0;
#pragma unroll
  for (int j = 0; j < CTM_MAXMODES; ++j) {
    if (j < nmodes) {
      int e = ext[j];
      int q = idx / e;
      off += (idx - q * e) * str[j];
      idx = q;
    }
  }
  return off;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct Cfg {
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int WTM = BM / WM;           // warp tile
  static constexpr int WTN = BN / WN;
  static constexpr int MT = WTM / 8;            // 8x8 mma tiles per warp
  static constexpr int NT = WTN / 8;
  static constexpr int PADA = 8, PADB = 8, PADC = 1;
  static constexpr int LDA = BM + PADA;         // smem row (k) stride, doubles
  static constexpr int LDB = BN + PADB;
  static constexpr int LDC = BN + PADC;
  static constexpr int STAGE_DOUBLES = BK * LDA + BK * LDB;
  static constexpr int PIPE_BYTES = STAGES * STAGE_DOUBLES * 8;
  static constexpr int EPI_BYTES = BM * LDC * 8;
  static constexpr int MAIN_BYTES = PIPE_BYTES > EPI_BYTES ? PIPE_BYTES : EPI_BYTES;
  // tables: A row offsets (BM), B col offsets (BN), C row/col offsets, K tables
  static constexpr int TAB_BYTES = (2 * BM + 2 * BN) * 4 + 2 * CTM_KTAB_MAX * 4;
  static constexpr int SMEM_BYTES = MAIN_BYTES + TAB_BYTES;
  static_assert(THREADS % BM == 0 || BM % (THREADS / BK) == 0, "A mapping");
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "tile/threads");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 4 == 0, "mma tiling");
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(32 * WM * WN, 1) tc_gemm_kernel(const TcArgs args) {
  using C_ = Cfg<BM, BN, BK, WM, WN, STAGES>;
  constexpr int THREADS = C_::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* pipe = reinterpret_cast<double*>(smem_raw);
  int* tab = reinterpret_cast<int*>(smem_raw + C_::MAIN_BYTES);
  int* a_moff = tab;                 // BM
  int* b_noff = a_moff + BM;         // BN
  int* c_moff = b_noff + BN;         // BM
  int* c_noff = c_moff + BM;         // BN
  int* a_koff = c_noff + BN;         // K (<= CTM_KTAB_MAX)
  int* b_koff = a_koff + CTM_KTAB_MAX;

  const int tid = threadIdx.x;
  const int bz = blockIdx.z;
  const int m0 = blockIdx.y * BM;
  const int n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;
  const double* __restrict__ Ag = args.A[bz];
  const double* __restrict__ Bg = args.B[bz];
  double* __restrict__ Cg = args.C[bz];

  // ---- offset tables -------------------------------------------------------------
  for (int i = tid; i < BM; i += THREADS) {
    int m = m0 + i;
    bool ok = m < M;
    a_moff[i] = ok ? mode_offset(m, args.nm, args.m_ext, args.a_m) : -1;
    c_moff[i] = ok ? mode_offset(m, args.nm, args.m_ext, args.c_m) : -1;
  }
  for (int i = tid; i < BN; i += THREADS) {
    int n = n0 + i;
    bool ok = n < N;
    b_noff[i] = ok ? mode_offset(n, args.nn, args.n_ext, args.b_n) : -1;
    c_noff[i] = ok ? mode_offset(n, args.nn, args.n_ext, args.c_n) : -1;
  }
  for (int k = tid; k < K; k += THREADS) {
    a_koff[k] = mode_offset(k, args.nk, args.k_ext, args.a_k);
    b_koff[k] = mode_offset(k, args.nk, args.k_ext, args.b_k);
  }
  __syncthreads();

  const int ktiles = (K + BK - 1) / BK;

  auto load_stage = [&](int stage, int kt) {
    double* As = pipe + stage * C_::STAGE_DOUBLES;
    double* Bs = As + BK * C_::LDA;
    const int k0 = kt * BK;
    // A tile: BM x BK -> As[k][m]
    if (args.a_kfast) {
      constexpr int ROWS_PER = THREADS / BK;
#pragma unroll
      for (int j = 0; j < (BM * BK) / THREADS; ++j) {
        int kl = tid % BK;
        int ml = tid / BK + j * ROWS_PER;
        int k = k0 + kl;
        int mo = a_moff[ml];
        bool ok = (k < K) && (mo >= 0);
        const double* src = ok ? Ag + (mo + a_koff[k]) : Ag;
        cp_async8(As + kl * C_::LDA + ml, src, ok);
      }
    } else {
#pragma unroll
      for (int j = 0; j < (BM * BK) / THREADS; ++j) {
        int e = tid + j * THREADS;
        int ml = e % BM;
        int kl = e / BM;
        int k = k0 + kl;
        int mo = a_moff[ml];
        bool ok = (k < K) && (mo >= 0);
        const double* src = ok ? Ag + (mo + a_koff[k]) : Ag;
        cp_async8(As + kl * C_::LDA + ml, src, ok);
      }
    }
    // B tile: BK x BN -> Bs[k][n]
    if (args.b_kfast) {
      constexpr int COLS_PER = THREADS / BK;
#pragma unroll
      for (int j = 0; j < (BN * BK) / THREADS; ++j) {
        int kl = tid % BK;
        int nl = tid / BK + j * COLS_PER;
        int k = k0 + kl;
        int no = b_noff[nl];
        bool ok = (k < K) && (no >= 0);
        const double* src = ok ? Bg + (no + b_koff[k]) : Bg;
        cp_async8(Bs + kl * C_::LDB + nl, src, ok);
      }
    } else {
#pragma unroll
      for (int j = 0; j < (BN * BK) / THREADS; ++j) {
        int e = tid + j * THREADS;
        int nl = e % BN;
        int kl = e / BN;
        int k = k0 + kl;
        int no = b_noff[nl];
        bool ok = (k < K) && (no >= 0);
        const double* src = ok ? Bg + (no + b_koff[k]) : Bg;
        cp_async8(Bs + kl * C_::LDB + nl, src, ok);
      }
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  double acc[C_::MT][C_::NT][2];
#pragma unroll
  for (int i = 0; i < C_::MT; ++i)
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // ---- prologue ---------------------------------------------------------------------
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  // ---- main loop --------------------------------------------------------------------
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* As = pipe + (kt % STAGES) * C_::STAGE_DOUBLES;
    const double* Bs = As + BK * C_::LDA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C_::MT], bf[C_::NT];
#pragma unroll
      for (int i = 0; i < C_::MT; ++i) af[i] = As[(kk + t) * C_::LDA + wm * C_::WTM + i * 8 + g];
#pragma unroll
      for (int j = 0; j < C_::NT; ++j) bf[j] = Bs[(kk + t) * C_::LDB + wn * C_::WTN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < C_::MT; ++i)
#pragma unroll
        for (int j = 0; j < C_::NT; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- epilogue: registers -> smem -> global (C's contiguous order) ------------------
  double* Cs = pipe;
  const double alpha = args.alpha, beta = args.beta;
#pragma unroll
  for (int i = 0; i < C_::MT; ++i)
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) {
      int r = wm * C_::WTM + i * 8 + g;
      int c = wn * C_::WTN + j * 8 + 2 * t;
      Cs[r * C_::LDC + c] = alpha * acc[i][j][0];
      Cs[r * C_::LDC + c + 1] = alpha * acc[i][j][1];
    }
  __syncthreads();
  double ss = 0.0;
  if (args.c_nfast) {
    for (int e = tid; e < BM * BN; e += THREADS) {
      int nl = e % BN, ml = e / BN;
      int mo = c_moff[ml], no = c_noff[nl];
      if (mo >= 0 && no >= 0) {
        double v = Cs[ml * C_::LDC + nl];
        if (beta != 0.0) v += beta * Cg[mo + no];
        Cg[mo + no] = v;
        ss += v * v;
      }
    }
  } else {
    for (int e = tid; e < BM * BN; e += THREADS) {
      int ml = e % BM, nl = e / BM;
      int mo = c_moff[ml], no = c_noff[nl];
      if (mo >= 0 && no >= 0) {
        double v = Cs[ml * C_::LDC + nl];
        if (beta != 0.0) v += beta * Cg[mo + no];
        Cg[mo + no] = v;
        ss += v * v;
      }
    }
  }
  if (args.sumsq[bz] != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) atomicAdd(args.sumsq[bz], ss);
  }
}

}  // namespace tc
