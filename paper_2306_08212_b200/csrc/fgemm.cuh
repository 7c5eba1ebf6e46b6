// fgemm.cuh -- the ISO solver's filter GEMM on the DMMA pipe (sm_100a), with the Chebyshev
// three-term combine in its epilogue:
//
//   C (M x N) = alpha * op(A) X + beta * Y + gamma * W,    op(A) = A (M x K) or A^T (A: K x M)
//
// all operands dense row-major (leading dimensions lda, ldx, ldc, ldy; W shares ldc and may
// alias C: each element is read before the same thread overwrites it).  The solver's
// products are tall and skinny (M = K = chi D = 1024 at C4, N = the active block <= 160):
// one 1024 x 160 output has only 48 tiles of tc_gemm's 64 x 64, so tc_gemm splits K eight
// ways, writes 8 partial slabs and the combine kernel sums them -- two launches and ~10 MB
// of partial traffic per Chebyshev degree.  Here a 32 x 32 tile keeps the full K per CTA
// (160 CTAs at N = 160: one per SM), so the recurrence is one launch and no slab.
//
//  * 4 warps, 2 x 2 warp tiles of 16 x 16 (2 x 2 m8n8 DMMA tiles each), BK = 32, 3-stage
//    cp.async pipeline in dynamic shared memory (16-byte copies for A; 16-byte for X when
//    its rows are 16-byte aligned, 8-byte otherwise), zero-fill (src-size 0) outside the
//    matrix.  Build knobs FG_BK / FG_STAGES / FG_BM: BK = 16 with 4 stages (the first
//    version) had 24 KB in flight per SM and a block barrier every 16 k; A/B of the full
//    move: C4 33.12 -> 31.65 ms, C3 11.75 -> 11.44, C5 157.7 -> 156.4; deeper pipelines of
//    16, 2 stages of 32 and BK = 64 were slower (profiles/r02s3_ab_fgemm_bk.jsonl).
//  * shared pitches = 4 (mod 16) doubles: the m8n8k4 fragment reads of a warp hit 16
//    distinct 8-byte bank pairs per half-warp (conflict-free), for both A orientations.
//  * fragment double buffering: k-step kk + 1's fragments are read under kk's DMMAs.
#pragma once
#include "pdl.cuh"
#include <cuda_runtime.h>

namespace fg {

struct FgArgs {
  const double* A;
  const double* X;
  double* C;
  const double* Y;   // nullable (beta term)
  const double* W;   // nullable (gamma term), may alias C
  int lda, ldx, ldc, ldy;
  int M, N, K;
  double alpha, beta, gamma;
};

#ifndef FG_STAGES
#define FG_STAGES 3
#endif
#ifndef FG_BK
#define FG_BK 32
#endif
#ifndef FG_BM
#define FG_BM 32
#endif
// (tried: a second group of 4 warps per CTA on the upper half of every k-tile, accumulators added
// through shared memory at the end -- twice the warps behind the same loads: C4 31.9 -> 35.9 ms,
// C3 12.4 -> 13.8 ms, profiles/r02s3_ab_fgemm_ksplit.jsonl; removed)
// (tried: warp-level split-K -- every warp the whole 32 x 32 tile over a quarter of each k-tile's
// k-steps, 16 independent accumulators per warp and half the fragment loads, partial tiles summed
// through shared memory; ncu on the kernel alone shows `wait` as the top stall and the DMMA pipe at
// 49% (profiles/r02s3_ncu_solver_kernels.txt), but inside the move the concurrent solves already
// hide that latency: C4 31.65 -> 32.0 ms, C5 156.8 -> 157.3 ms, profiles/r02s3_ab_fgemm_wsplit.jsonl;
// removed)
constexpr int BM = FG_BM, BN = 32, BK = FG_BK, STAGES = FG_STAGES, THREADS = 128;
static_assert(BM == 32 || BM == 64, "fgemm: BM is 32 or 64");
constexpr int MI = BM / 16;                       // m8 DMMA tiles per warp (2 warp rows of BM / 2)
constexpr int MCH = BM / 2;                       // 16-byte chunks per k-row of a transposed A tile
static_assert(BK == 16 || BK == 32 || BK == 64, "fgemm: BK is 16, 32 or 64");
constexpr int KCH = BK / 2;                       // 16-byte chunks per k-row of a non-transposed A tile
constexpr int A_ITERS = BM * BK / 2 / THREADS;    // 16-byte A chunks per thread and k-tile
constexpr int X_ITERS = BK * BN / 2 / THREADS;    // 16-byte X chunks per thread and k-tile
constexpr int LDA_N = BK + 4;   // non-transposed A tile: As[m][k]
constexpr int LDA_T = BM + 4;   // transposed A tile:     As[k][m]
constexpr int LDB = BN + 4;     // X tile:                Bs[k][n]
constexpr int A_DOUBLES = BM * LDA_N > BK * LDA_T ? BM * LDA_N : BK * LDA_T;
constexpr int STAGE_DOUBLES = A_DOUBLES + BK * LDB;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_DOUBLES * sizeof(double);

__device__ __forceinline__ void cp16(unsigned dst, const void* src, bool in) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(in ? 16 : 0));
}
__device__ __forceinline__ void cp8(unsigned dst, const void* src, bool in) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(in ? 8 : 0));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// TRANS: op(A) = A^T.  XVEC: X rows 16-byte aligned and N even (16-byte X copies).
template <bool TRANS, bool XVEC>
__global__ void __launch_bounds__(THREADS) fgemm_kernel(const FgArgs p) {
  extern __shared__ __align__(16) double sm[];   // SMEM_BYTES (dynamic: deeper pipelines pass 48 KB)
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = p.M, N = p.N, K = p.K;
  const int ktiles = (K + BK - 1) / BK;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
  CTM_PDL_WAIT();

  auto load = [&](int stage, int kt) {
    const int k0 = kt * BK;
    const unsigned As = sbase + stage * STAGE_DOUBLES * 8;
    const unsigned Bs = As + A_DOUBLES * 8;
#pragma unroll
    for (int u = 0; u < A_ITERS; ++u) {   // A: BM BK / 2 16-byte chunks
      const int c = tid + THREADS * u;
      if (!TRANS) {
        const int r = c / KCH, kc = (c % KCH) * 2;
        const bool in = m0 + r < M && k0 + kc < K;
        cp16(As + (r * LDA_N + kc) * 8, in ? p.A + (size_t)(m0 + r) * p.lda + k0 + kc : p.A, in);
      } else {
        const int kr = c / MCH, mc = (c % MCH) * 2;
        const bool in = k0 + kr < K && m0 + mc < M;
        cp16(As + (kr * LDA_T + mc) * 8, in ? p.A + (size_t)(k0 + kr) * p.lda + m0 + mc : p.A, in);
      }
    }
    if (XVEC) {
#pragma unroll
      for (int u = 0; u < X_ITERS; ++u) {   // X: BK BN / 2 16-byte chunks
        const int c = tid + THREADS * u;
        const int kr = c >> 4, nc = (c & 15) * 2;
        const bool in = k0 + kr < K && n0 + nc < N;
        cp16(Bs + (kr * LDB + nc) * 8, in ? p.X + (size_t)(k0 + kr) * p.ldx + n0 + nc : p.X, in);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 2 * X_ITERS; ++u) {   // X: BK BN 8-byte elements
        const int c = tid + THREADS * u;
        const int kr = c >> 5, nc = c & 31;
        const bool in = k0 + kr < K && n0 + nc < N;
        cp8(Bs + (kr * LDB + nc) * 8, in ? p.X + (size_t)(k0 + kr) * p.ldx + n0 + nc : p.X, in);
      }
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  double acc[MI][2][2] = {};
  double af[2][MI], bf[2][2];
  auto frag = [&](int buf, int stage, int kk) {
    const double* As = sm + stage * STAGE_DOUBLES;
    const double* Bs = As + A_DOUBLES;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = wm * (BM / 2) + i * 8 + g;
      af[buf][i] = TRANS ? As[(kk + t) * LDA_T + m] : As[m * LDA_N + kk + t];
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[buf][j] = Bs[(kk + t) * LDB + wn * 16 + j * 8 + g];
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load(s, s);
    commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    wait_group<STAGES - 2>();
    __syncthreads();   // tile kt visible; every warp is done with the stage refilled below
    const int nk = kt + STAGES - 1;
    if (nk < ktiles) load(nk % STAGES, nk);
    commit();
    const int cur = kt % STAGES;
    frag(0, cur, 0);
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      if (q < BK / 4 - 1) frag((q + 1) & 1, cur, 4 * (q + 1));
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j], af[q & 1][i], bf[q & 1][j]);
    }
  }
  wait_group<0>();
  CTM_PDL_TRIGGER();

  // epilogue: C = alpha acc + beta Y + gamma W (accumulator pair = columns 2t, 2t + 1)
  const double alpha = p.alpha, beta = p.beta, gamma = p.gamma;
  const bool vec = ((p.ldc | p.ldy) & 1) == 0;   // (host: ldy = ldc when Y is null)
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int m = m0 + wm * (BM / 2) + i * 8 + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = n0 + wn * 16 + j * 8 + 2 * t;
      if (n >= N) continue;
      double* c = p.C + (size_t)m * p.ldc + n;
      const double* y = p.Y ? p.Y + (size_t)m * p.ldy + n : nullptr;
      const double* w = p.W ? p.W + (size_t)m * p.ldc + n : nullptr;
      if (vec && n + 1 < N) {
        double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        if (y) {
          const double2 yy = *reinterpret_cast<const double2*>(y);
          v.x = fma(beta, yy.x, v.x);
          v.y = fma(beta, yy.y, v.y);
        }
        if (w) {
          const double2 ww = *reinterpret_cast<const double2*>(w);
          v.x = fma(gamma, ww.x, v.x);
          v.y = fma(gamma, ww.y, v.y);
        }
        *reinterpret_cast<double2*>(c) = v;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (n + e >= N) break;
          double v = alpha * acc[i][j][e];
          if (y) v = fma(beta, y[e], v);
          if (w) v = fma(gamma, w[e], v);
          c[e] = v;
        }
      }
    }
  }
}

}  // namespace fg
