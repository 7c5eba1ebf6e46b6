// tc_gemm.cuh -- FP64 tensor-contraction GEMM on the B200 DMMA pipe (sm_100a).
//
//   C[m, n] = alpha * sum_k A[m, k] * B[k, n]  (+ beta * C)
//
// where m, n and k are multi-indices of up to CTM_MAXMODES modes each and every operand
// is addressed through per-mode element strides, so the index permutations of the
// CTMRG contractions are fused into the tile loads
// and the epilogue instead of being separate transpose passes.
//
// Design:
//  * math: mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4.  sm_100a has no
//    tcgen05 FP64 kind (ptxas rejects .kind::f64) and wgmma is sm_90a-only, so DMMA is
//    the FP64 tensor path; measured 37.1 TFLOP/s peak (= DFMA peak) on this B200, and
//    reached with as few as 4 warps/SM (profiles/r01_probe_dmma_occupancy.txt).
//  * two CTAs per SM (warp tile 32x32, <= 128 registers, ~100 KB shared memory each) so
//    one CTA's prologue / epilogue / load bursts overlap the other's DMMA stream (the
//    first version, one 128x128 CTA per SM, left the DMMA pipe idle ~47% of the time:
//    profiles/r01_ncu_c4_chain_v1.txt).
//  * operand staging: TMA boxes for the launches whose operands admit them (tc_gemm_tma.cuh);
//    otherwise cp.async (LDGSTS, 8 B) gathers, 3-stage pipeline; each thread's
//    fixed row/column offsets live in registers, the k offsets in a shared-memory table;
//    the thread mapping follows the operand's contiguous index (m/k-fast for A, k/n-fast
//    for B) so every warp load is coalesced.
//  * epilogue: direct stores from the DMMA accumulator layout through per-row/column
//    offset tables (any output permutation), fused sum of squares for the Frobenius
//    normalisation (reading R13).
//  * split-K (grid.z = batch x splits) for the small-M*N, large-K contractions (S3, S6,
//    corners): partial tiles go to a workspace slab and a deterministic reduction kernel
//    sums them in split order (no floating-point atomics on the data).
//  * batch: one launch serves up to CTM_MAXBATCH problems with identical shapes/strides.
#pragma once
#include "pdl.cuh"
#include <cstdint>
#include <cuda_runtime.h>

#define CTM_MAXMODES 4
#define CTM_MAXBATCH 4
#define CTM_KTAB_MAX 2048

struct TcArgs {
  const double* A[CTM_MAXBATCH];
  const double* B[CTM_MAXBATCH];
  double* C[CTM_MAXBATCH];
  double* sumsq[CTM_MAXBATCH];   // nullable: per-CTA partial sums of squares of the final C values,
                                 // slot blockIdx.y*gridDim.x+blockIdx.x (deterministic reduction later)
  double* part;                  // split-K partial slab [batch][split][M][N] (splits > 1)
  int M, N, K;
  int nm, nn, nk;
  int m_ext[CTM_MAXMODES], n_ext[CTM_MAXMODES], k_ext[CTM_MAXMODES];
  int a_m[CTM_MAXMODES], a_k[CTM_MAXMODES];
  int b_k[CTM_MAXMODES], b_n[CTM_MAXMODES];
  int c_m[CTM_MAXMODES], c_n[CTM_MAXMODES];
  // round-up reciprocal of every mode extent (q = (umulhi(i, mag) + i) >> sh for i < 2^31),
  // so the per-CTA offset tables need no integer divisions
  unsigned m_mag[CTM_MAXMODES], n_mag[CTM_MAXMODES], k_mag[CTM_MAXMODES];
  int m_sh[CTM_MAXMODES], n_sh[CTM_MAXMODES], k_sh[CTM_MAXMODES];
  int a_kfast, b_kfast;
  int ksep;        // k offsets separable by 16-wide tiles (tc_gemm_kernel<..., SEP>)
  int splits, ktiles_per_split;
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

// Offsets of one multi-index in two operands at once, divisions by magic multiply.
__device__ __forceinline__ void mode_offset2(int idx, int nmodes, const int* ext, const unsigned* mag, const int* sh,
                                             const int* s1, const int* s2, int& o1, int& o2) {
  int a = 0, b = 0;
  unsigned u = (unsigned)idx;
#pragma unroll
  for (int j = 0; j < CTM_MAXMODES; ++j) {
    if (j < nmodes) {
      const unsigned q = (__umulhi(u, mag[j]) + u) >> sh[j];
      const int r = (int)(u - q * (unsigned)ext[j]);
      a += r * s1[j];
      b += r * s2[j];
      u = q;
    }
  }
  o1 = a;
  o2 = b;
}

__device__ __forceinline__ void cp_async8(unsigned smem_addr, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Deterministic block sum (warp shuffles, then warps in order) stored by thread 0.
__device__ __forceinline__ void block_sum_store(double v, double* out) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *out = s;
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
struct Cfg {
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int WTM = BM / WM;           // warp tile
  static constexpr int WTN = BN / WN;
  static constexpr int MT = WTM / 8;            // 8x8 mma tiles per warp
  static constexpr int NT = WTN / 8;
  // row pad 4 doubles: a half-warp's DMMA fragment load (rows kk+t, t = 0..3, 4 consecutive
  // doubles each) then spans all 32 banks once (row stride 132 -> 8-bank offset per row);
  // pad 8 (16-bank offset) made every fragment load 2-way conflicted (ncu: 9-20 M
  // conflicts per chain launch) and the k-fast cp.async writes 8-way instead of 4-way
  static constexpr int PAD = 4;
  static constexpr int LDA = BM + PAD;          // smem row (k) stride, doubles
  static constexpr int LDB = BN + PAD;
  static constexpr int STAGE_DOUBLES = BK * LDA + BK * LDB;
  static constexpr int PIPE_BYTES = STAGES * STAGE_DOUBLES * 8;
  static constexpr int TAB_BYTES = (2 * BM + 2 * BN) * 4 + 2 * CTM_KTAB_MAX * 4;
  static constexpr int SMEM_BYTES = PIPE_BYTES + TAB_BYTES;
  static constexpr int A_PER = BM * BK / THREADS;   // A elements per thread per stage
  static constexpr int B_PER = BN * BK / THREADS;
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "tile/threads");
  static_assert(THREADS % BK == 0 && THREADS % BM == 0 && THREADS % BN == 0, "mapping");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 4 == 0, "mma tiling");
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool AKF, bool BKF, bool SEP, bool FB>
__global__ void __launch_bounds__(32 * WM * WN, MINB) tc_gemm_kernel(const TcArgs args) {
  using C_ = Cfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  constexpr int THREADS = C_::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* pipe = reinterpret_cast<double*>(smem_raw);
  int* tab = reinterpret_cast<int*>(smem_raw + C_::PIPE_BYTES);
  int* a_moff = tab;                 // BM
  int* b_noff = a_moff + BM;         // BN
  int* c_moff = b_noff + BN;         // BM
  int* c_noff = c_moff + BM;         // BN
  int* a_koff = c_noff + BN;         // K range of this split (<= CTM_KTAB_MAX)
  int* b_koff = a_koff + CTM_KTAB_MAX;

  const int tid = threadIdx.x;
  const int bz = blockIdx.z / args.splits;
  const int split = blockIdx.z - bz * args.splits;
  const int m0 = blockIdx.y * BM;
  const int n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;
  const int kt_begin = split * args.ktiles_per_split;
  const int kt_total = (K + BK - 1) / BK;
  const int kt_end = min(kt_total, kt_begin + args.ktiles_per_split);
  const int ktiles = max(0, kt_end - kt_begin);
  const int kbase = kt_begin * BK;
  const int kcount = min(K - kbase, ktiles * BK);
  const double* __restrict__ Ag = args.A[bz];
  const double* __restrict__ Bg = args.B[bz];

  // ---- offset tables -------------------------------------------------------------
  for (int i = tid; i < BM; i += THREADS) {
    const int m = m0 + i;
    int oa = -1, oc = -1;
    if (m < M) mode_offset2(m, args.nm, args.m_ext, args.m_mag, args.m_sh, args.a_m, args.c_m, oa, oc);
    a_moff[i] = oa;
    c_moff[i] = oc;
  }
  for (int i = tid; i < BN; i += THREADS) {
    const int n = n0 + i;
    int ob = -1, oc = -1;
    if (n < N) mode_offset2(n, args.nn, args.n_ext, args.n_mag, args.n_sh, args.b_n, args.c_n, ob, oc);
    b_noff[i] = ob;
    c_noff[i] = oc;
  }
  for (int k = tid; k < kcount; k += THREADS)
    mode_offset2(kbase + k, args.nk, args.k_ext, args.k_mag, args.k_sh, args.a_k, args.b_k, a_koff[k], b_koff[k]);
  __syncthreads();
  // programmatic dependent launch: the offset tables above use only the arguments, so they
  // overlap the previous kernel's tail; operands are read after the wait
  CTM_PDL_WAIT();

  // ---- per-thread load assignment (fixed across stages) -----------------------------
  // A: k-fast -> fixed kl, rows ml0 + j*(THREADS/BK);  m-fast -> fixed ml, kl0 + j*(THREADS/BM)
  // Rows / columns past the matrix edge read row / column 0 (their results are never
  // stored); only the K tail must be zero, and it is written with st.shared in the last
  // (partial) k-tile, so full k-tiles issue plain cp.async with no predicates.
  constexpr bool akf = AKF, bkf = BKF;
  const int a_fix = akf ? (tid % BK) : (tid % BM);
  const int a_var0 = akf ? (tid / BK) : (tid / BM);
  const int a_step = akf ? (THREADS / BK) : (THREADS / BM);
  const int b_fix = bkf ? (tid % BK) : (tid % BN);
  const int b_var0 = bkf ? (tid / BK) : (tid / BN);
  const int b_step = bkf ? (THREADS / BK) : (THREADS / BN);
  int a_row[C_::A_PER];   // k-fast: offsets of my rows; m-fast: only a_row[0] used
  int b_col[C_::B_PER];
#pragma unroll
  for (int j = 0; j < C_::A_PER; ++j) a_row[j] = max(0, akf ? a_moff[a_var0 + j * a_step] : a_moff[a_fix]);
#pragma unroll
  for (int j = 0; j < C_::B_PER; ++j) b_col[j] = max(0, bkf ? b_noff[b_var0 + j * b_step] : b_noff[b_fix]);
  if constexpr (SEP) {
    // separable k offsets (TcArgs::ksep): koff(k0 + kl) = koff(k0) + koff(kl) - koff(0) for every
    // tile start k0, so each load's in-tile part is folded into its row / column offset here and
    // a k-tile needs one table read per operand instead of one per load
    const int a0 = a_row[0], b0 = b_col[0];
#pragma unroll
    for (int j = 0; j < C_::A_PER; ++j) {
      const int kl = akf ? a_fix : (a_var0 + j * a_step);
      a_row[j] = (akf ? a_row[j] : a0) + (kl < kcount ? a_koff[kl] - a_koff[0] : 0);
    }
#pragma unroll
    for (int j = 0; j < C_::B_PER; ++j) {
      const int kl = bkf ? b_fix : (b_var0 + j * b_step);
      b_col[j] = (bkf ? b_col[j] : b0) + (kl < kcount ? b_koff[kl] - b_koff[0] : 0);
    }
  }
  const unsigned pipe_s = static_cast<unsigned>(__cvta_generic_to_shared(pipe));

  // one quarter of a stage's loads (part = 0..3), so they interleave with the DMMA steps
  constexpr int A_Q = (C_::A_PER + 3) / 4, B_Q = (C_::B_PER + 3) / 4;
  // ta / tb (SEP): the tile's k offset in A / B, read once per k-tile by the caller
  auto load_part = [&](int stage, int kt, int part, bool full, int ta, int tb) {
    const unsigned As = pipe_s + stage * C_::STAGE_DOUBLES * 8;
    const unsigned Bs = As + BK * C_::LDA * 8;
    const int k0 = kt * BK;   // relative to kbase
#pragma unroll
    for (int jj = 0; jj < A_Q; ++jj) {
      const int j = part * A_Q + jj;
      if (j < C_::A_PER) {
        const int kl = akf ? a_fix : (a_var0 + j * a_step);
        const int ml = akf ? (a_var0 + j * a_step) : a_fix;
        const int k = k0 + kl;
        const unsigned dst = As + (kl * C_::LDA + ml) * 8;
        if (full || k < kcount) {
          cp_async8(dst, Ag + (SEP ? a_row[j] + ta : a_row[akf ? j : 0] + a_koff[k]));
        } else {
          asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(dst), "d"(0.0));
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < B_Q; ++jj) {
      const int j = part * B_Q + jj;
      if (j < C_::B_PER) {
        const int kl = bkf ? b_fix : (b_var0 + j * b_step);
        const int nl = bkf ? (b_var0 + j * b_step) : b_fix;
        const int k = k0 + kl;
        const unsigned dst = Bs + (kl * C_::LDB + nl) * 8;
        if (full || k < kcount) {
          cp_async8(dst, Bg + (SEP ? b_col[j] + tb : b_col[bkf ? j : 0] + b_koff[k]));
        } else {
          asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(dst), "d"(0.0));
        }
      }
    }
  };
  const int ktiles_full = kcount / BK;   // k-tiles [0, ktiles_full) need no tail handling

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
    if (s < ktiles) {
#pragma unroll
      for (int part = 0; part < 4; ++part)
        load_part(s, s, part, s < ktiles_full, SEP ? a_koff[s * BK] : 0, SEP ? b_koff[s * BK] : 0);
    }
    cp_async_commit();
  }

  // ---- main loop --------------------------------------------------------------------
  static_assert(BK == 16, "the load interleave assumes 4 DMMA k-steps per k-tile");
  if constexpr (FB) {
    // fragment double buffering (CUTLASS sm80 style): the fragments of k-step kk + 1 are read
    // from shared memory while the DMMAs of kk issue; the stage barrier moves to the last k-step
    // of the previous tile, right after its fragments are in registers, so the next tile's first
    // fragments are prefetched under the last DMMAs of the current one
    double af[2][C_::MT], bf[2][C_::NT];
    auto frag = [&](int buf, int stage, int kk) {
      const double* As = pipe + stage * C_::STAGE_DOUBLES;
      const double* Bs = As + BK * C_::LDA;
#pragma unroll
      for (int i = 0; i < C_::MT; ++i) af[buf][i] = As[(kk + t) * C_::LDA + wm * C_::WTM + i * 8 + g];
#pragma unroll
      for (int j = 0; j < C_::NT; ++j) bf[buf][j] = Bs[(kk + t) * C_::LDB + wn * C_::WTN + j * 8 + g];
    };
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (ktiles > 0) frag(0, 0, 0);
    for (int kt = 0; kt < ktiles; ++kt) {
      const int nk = kt + STAGES - 1;
      const bool do_load = nk < ktiles;
      const bool nfull = nk < ktiles_full;
      const int cur = kt % STAGES;
      const int ta = (SEP && do_load) ? a_koff[nk * BK] : 0, tb = (SEP && do_load) ? b_koff[nk * BK] : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < 3) frag((q + 1) & 1, cur, 4 * (q + 1));
        if (do_load) load_part(nk % STAGES, nk, q, nfull, ta, tb);
        if (q == 3) {
          cp_async_commit();
          cp_async_wait<STAGES - 2>();
          __syncthreads();   // tile kt + 1 visible; every warp is done reading stage cur
          if (kt + 1 < ktiles) frag(0, (kt + 1) % STAGES, 0);
        }
#pragma unroll
        for (int i = 0; i < C_::MT; ++i)
#pragma unroll
          for (int j = 0; j < C_::NT; ++j) dmma(acc[i][j], af[q & 1][i], bf[q & 1][j]);
      }
    }
  } else {
    for (int kt = 0; kt < ktiles; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nk = kt + STAGES - 1;
      const bool do_load = nk < ktiles;
      const bool nfull = nk < ktiles_full;
      const double* As = pipe + (kt % STAGES) * C_::STAGE_DOUBLES;
      const double* Bs = As + BK * C_::LDA;
      const int ta = (SEP && do_load) ? a_koff[nk * BK] : 0, tb = (SEP && do_load) ? b_koff[nk * BK] : 0;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[C_::MT], bf[C_::NT];
#pragma unroll
        for (int i = 0; i < C_::MT; ++i) af[i] = As[(kk + t) * C_::LDA + wm * C_::WTM + i * 8 + g];
#pragma unroll
        for (int j = 0; j < C_::NT; ++j) bf[j] = Bs[(kk + t) * C_::LDB + wn * C_::WTN + j * 8 + g];
        if (do_load) load_part(nk % STAGES, nk, kk / 4, nfull, ta, tb);
#pragma unroll
        for (int i = 0; i < C_::MT; ++i)
#pragma unroll
          for (int j = 0; j < C_::NT; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
  CTM_PDL_TRIGGER();

  // ---- epilogue: direct stores from the accumulator layout ---------------------------
  const double alpha = args.alpha, beta = args.beta;
  double ss = 0.0;
  if (args.splits > 1) {
    double* __restrict__ P = args.part + ((size_t)blockIdx.z * M) * N;
    const bool even = (N & 1) == 0;   // (m N + n) even: 16-byte aligned pair
#pragma unroll
    for (int i = 0; i < C_::MT; ++i) {
      const int m = m0 + wm * C_::WTM + i * 8 + g;
#pragma unroll
      for (int j = 0; j < C_::NT; ++j) {
        const int n = n0 + wn * C_::WTN + j * 8 + 2 * t;
        if (m < M) {
          if (even && n + 1 < N) {
            *reinterpret_cast<double2*>(P + (size_t)m * N + n) = make_double2(acc[i][j][0], acc[i][j][1]);
          } else {
            if (n < N) P[(size_t)m * N + n] = acc[i][j][0];
            if (n + 1 < N) P[(size_t)m * N + n + 1] = acc[i][j][1];
          }
        }
      }
    }
    return;
  }
  double* __restrict__ Cg = args.C[bz];
#pragma unroll
  for (int i = 0; i < C_::MT; ++i) {
    const int r = wm * C_::WTM + i * 8 + g;
    const int mo = c_moff[r];
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) {
      const int c = wn * C_::WTN + j * 8 + 2 * t;
      const int no0 = c_noff[c], no1 = c_noff[c + 1];
      if (mo >= 0 && no0 >= 0 && no1 == no0 + 1 && ((mo + no0) & 1) == 0 && beta == 0.0) {
        // the pair of accumulator columns is contiguous and 16-byte aligned in C: one vector store
        const double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
        *reinterpret_cast<double2*>(Cg + mo + no0) = make_double2(v0, v1);
        ss += v0 * v0 + v1 * v1;
        continue;
      }
      if (mo >= 0) {
        if (no0 >= 0) {
          double v = alpha * acc[i][j][0];
          if (beta != 0.0) v += beta * Cg[mo + no0];
          Cg[mo + no0] = v;
          ss += v * v;
        }
        if (no1 >= 0) {
          double v = alpha * acc[i][j][1];
          if (beta != 0.0) v += beta * Cg[mo + no1];
          Cg[mo + no1] = v;
          ss += v * v;
        }
      }
    }
  }
  if (args.sumsq[bz] != nullptr) block_sum_store(ss, args.sumsq[bz] + blockIdx.y * gridDim.x + blockIdx.x);
}

}  // namespace tc
