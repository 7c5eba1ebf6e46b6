// tc_gemm_tma.cuh -- the FP64 DMMA contraction kernel with its operand tiles staged by TMA
// (cp.async.bulk.tensor: UTMALDG in SASS) instead of per-thread cp.async gathers.
//
// Same tile shapes, fragment layout, DMMA main loop (fragment double buffering) and epilogue as
// tc_gemm_kernel<..., FB = true> (tc_gemm.cuh); what changes is how a k-tile reaches shared memory:
//
//  * one tensor map per operand and batch entry describes the operand through the planner's
//    modes: A = [m_0 (the contiguous m mode), k_0 .. k_{nk-1}, m_1 .. m_{nm-1}] (B likewise with n),
//    so a (BM x BK) tile is ONE box -- the permutation stays fused into the load;
//  * the box's inner extent is BM + 4 (BN + 4): the four extra elements over-fetch the next
//    tile's data (or zero-fill past the edge), which reproduces the padded row pitch that keeps
//    the DMMA fragment loads conflict-free (a box lands dense in shared memory);
//  * one elected thread issues both boxes of a stage against an mbarrier (expect-tx bytes); the
//    consumer warps wait on the stage's phase instead of cp.async groups; out-of-range rows and
//    the K tail arrive as zeros (no predicated stores).
//
// Eligible launches (tc_gemm.cu, tma_plan): m-fast A and n-fast B (the chain steps S1..S6),
// the contiguous mode a multiple of the tile width, at most five tensor dims per operand, k tiles
// that are whole boxes (every prefix product of the k extents divides 16 until one is a
// multiple of 16), 16-byte-multiple strides and 16-byte-aligned bases.
#pragma once
#include <cuda.h>

#include "tc_gemm.cuh"

struct TmaMaps {
  CUtensorMap a[CTM_MAXBATCH];
  CUtensorMap b[CTM_MAXBATCH];
  int a_rank, b_rank;
};

namespace tc {

__device__ __forceinline__ unsigned tma_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// coordinates of the box whose first element is (x0 of the contiguous-first mode group, k index
// kidx) in a map laid out as [x_0, k_0 .. k_{nk-1}, x_1 .. x_{nx-1}]
__device__ __forceinline__ void tma_coords(int x0, int kidx, int nx, const int* xext, int nk, const int* kext,
                                           int (&c)[5]) {
  c[0] = x0 % xext[0];
  int q = x0 / xext[0];
  int d = 1;
#pragma unroll
  for (int j = 0; j < CTM_MAXMODES; ++j)
    if (j < nk) {
      c[d++] = kidx % kext[j];
      kidx /= kext[j];
    }
#pragma unroll
  for (int j = 1; j < CTM_MAXMODES; ++j)
    if (j < nx) {
      c[d++] = q % xext[j];
      q /= xext[j];
    }
  for (; d < 5; ++d) c[d] = 0;
}

__device__ __forceinline__ void tma_load(unsigned dst, const CUtensorMap* map, int rank, const int (&c)[5],
                                         unsigned bar) {
  const unsigned long long m = reinterpret_cast<unsigned long long>(map);
  switch (rank) {
    case 1:
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(dst), "l"(m), "r"(c[0]), "r"(bar) : "memory");
      break;
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"(m), "r"(c[0]), "r"(c[1]), "r"(bar) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(bar) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(dst), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(bar) : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(dst), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar) : "memory");
      break;
  }
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(32 * WM * WN, MINB) tc_gemm_tma_kernel(const TcArgs args, const __grid_constant__ TmaMaps maps) {
  using C_ = Cfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  static_assert(BK == 16, "4 DMMA k-steps per k-tile");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* pipe = reinterpret_cast<double*>(smem_raw);
  int* tab = reinterpret_cast<int*>(smem_raw + C_::PIPE_BYTES);
  int* c_moff = tab;          // BM
  int* c_noff = c_moff + BM;  // BN
  __shared__ __align__(8) unsigned long long full[STAGES];

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

  for (int i = tid; i < BM; i += C_::THREADS) {
    int oc = -1, d;
    if (m0 + i < M) mode_offset2(m0 + i, args.nm, args.m_ext, args.m_mag, args.m_sh, args.c_m, args.c_m, oc, d);
    c_moff[i] = oc;
  }
  for (int i = tid; i < BN; i += C_::THREADS) {
    int oc = -1, d;
    if (n0 + i < N) mode_offset2(n0 + i, args.nn, args.n_ext, args.n_mag, args.n_sh, args.c_n, args.c_n, oc, d);
    c_noff[i] = oc;
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma_smem(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  CTM_PDL_WAIT();

  const unsigned pipe_s = tma_smem(pipe);
  constexpr unsigned STAGE_BYTES = C_::STAGE_DOUBLES * 8;
  constexpr unsigned TX = (BM + C_::PAD) * BK * 8 + (BN + C_::PAD) * BK * 8;
  const CUtensorMap* amap = &maps.a[bz];
  const CUtensorMap* bmap = &maps.b[bz];
  // one thread loads k-tile kt into stage s (the stage's previous contents are consumed: the
  // caller passed the barrier that follows their last fragment reads)
  // box coordinates: the m / n parts are fixed per CTA (computed once); the k digits of each
  // k-tile by the planner's magic-number divisions
  int ca[5], cb[5];
  if (tid == 0) {
    tma_coords(m0, kbase, args.nm, args.m_ext, args.nk, args.k_ext, ca);
    tma_coords(n0, kbase, args.nn, args.n_ext, args.nk, args.k_ext, cb);
  }
  auto issue = [&](int kt, int s) {
    const unsigned As = pipe_s + s * STAGE_BYTES;
    const unsigned Bs = As + BK * C_::LDA * 8;
    const unsigned bar = tma_smem(&full[s]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads before the async writes
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TX) : "memory");
    unsigned u = (unsigned)(kbase + kt * BK);
#pragma unroll
    for (int j = 0; j < CTM_MAXMODES; ++j)
      if (j < args.nk) {
        const unsigned q = (__umulhi(u, args.k_mag[j]) + u) >> args.k_sh[j];
        ca[1 + j] = cb[1 + j] = (int)(u - q * (unsigned)args.k_ext[j]);
        u = q;
      }
    tma_load(As, amap, maps.a_rank, ca, bar);
    tma_load(Bs, bmap, maps.b_rank, cb, bar);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s)
      if (s < ktiles) issue(s, s);
  }

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  double acc[C_::MT][C_::NT][2];
#pragma unroll
  for (int i = 0; i < C_::MT; ++i)
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double af[2][C_::MT], bf[2][C_::NT];
  auto frag = [&](int buf, int stage, int kk) {
    const double* As = pipe + stage * C_::STAGE_DOUBLES;
    const double* Bs = As + BK * C_::LDA;
#pragma unroll
    for (int i = 0; i < C_::MT; ++i) af[buf][i] = As[(kk + t) * C_::LDA + wm * C_::WTM + i * 8 + g];
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) bf[buf][j] = Bs[(kk + t) * C_::LDB + wn * C_::WTN + j * 8 + g];
  };
  if (ktiles > 0) {
    mbar_wait(tma_smem(&full[0]), 0);
    frag(0, 0, 0);
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int cur = kt % STAGES;
    // stage (kt - 1) % STAGES = (kt + STAGES - 1) % STAGES was released by the barrier that ended
    // iteration kt - 1
    if (tid == 0 && kt + STAGES - 1 < ktiles) issue(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < 3) frag((q + 1) & 1, cur, 4 * (q + 1));
      if (q == 3) {
        if (kt + 1 < ktiles) mbar_wait(tma_smem(&full[(kt + 1) % STAGES]), ((kt + 1) / STAGES) & 1);
        __syncthreads();   // every warp is done reading stage cur
        if (kt + 1 < ktiles) frag(0, (kt + 1) % STAGES, 0);
      }
#pragma unroll
      for (int i = 0; i < C_::MT; ++i)
#pragma unroll
        for (int j = 0; j < C_::NT; ++j) dmma(acc[i][j], af[q & 1][i], bf[q & 1][j]);
    }
  }
  CTM_PDL_TRIGGER();

  // ---- epilogue: tc_gemm_kernel's (split-K partial slab, or direct stores + sum of squares)
  const double alpha = args.alpha;
  if (args.splits > 1) {
    double* __restrict__ P = args.part + ((size_t)blockIdx.z * M) * N;
    const bool even = (N & 1) == 0;
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
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < C_::MT; ++i) {
    const int mo = c_moff[wm * C_::WTM + i * 8 + g];
#pragma unroll
    for (int j = 0; j < C_::NT; ++j) {
      const int c = wn * C_::WTN + j * 8 + 2 * t;
      const int no0 = c_noff[c], no1 = c_noff[c + 1];
      const double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
      if (mo < 0) continue;
      if (no0 >= 0 && no1 == no0 + 1 && ((mo + no0) & 1) == 0) {
        *reinterpret_cast<double2*>(Cg + mo + no0) = make_double2(v0, v1);
        ss += v0 * v0 + v1 * v1;
        continue;
      }
      if (no0 >= 0) {
        Cg[mo + no0] = v0;
        ss += v0 * v0;
      }
      if (no1 >= 0) {
        Cg[mo + no1] = v1;
        ss += v1 * v1;
      }
    }
  }
  if (args.sumsq[bz] != nullptr) block_sum_store(ss, args.sumsq[bz] + blockIdx.y * gridDim.x + blockIdx.x);
}

}  // namespace tc
