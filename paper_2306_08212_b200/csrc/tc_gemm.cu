// tc_gemm.cu -- contraction planner (labels -> strided GEMM modes) and launcher for the
// FP64 DMMA kernel of tc_gemm.cuh.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <set>

#include <cudaTypedefs.h>

#include "ctm_internal.h"
#include "tc_gemm_tma.cuh"

namespace ctm {
namespace {

// ---- TMA staging (tc_gemm_tma.cuh) -------------------------------------------------------
// CTM_TC_TMA=0 keeps every launch on the cp.async kernel (A/B).
bool tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CTM_TC_TMA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// One operand's tensor map [x_0, k_0 .. k_{nk-1}, x_1 .. x_{nx-1}] with box [tile + 4, k box, 1 ..]
// (the 4 extra inner elements give the padded row pitch of tc_gemm's shared tiles); false when
// the operand does not fit the TMA path.
bool tma_map(CUtensorMap* map, const double* base, int nx, const int* xext, const int* xstr, int nk,
             const int* kext, const int* kstr, int tile, int* rank_out) {
  if (xstr[0] != 1 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if (nx > 1 && xext[0] % tile != 0) return false;   // a tile never straddles the contiguous mode
  const int rank = 1 + nk + (nx - 1);
  if (rank > 5) return false;
  cuuint64_t dim[5], str[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  int d = 0;
  dim[d] = (cuuint64_t)xext[0];
  box[d++] = (cuuint32_t)(tile + 4);
  // k box: whole prefix of the k modes covering the 16-wide k-tile (one mode of any extent: the
  // tail arrives zero-filled)
  int need = 16;
  for (int j = 0; j < nk; ++j) {
    dim[d] = (cuuint64_t)kext[j];
    str[d - 1] = (cuuint64_t)kstr[j] * 8;
    if (need > 1) {
      if (nk > 1 && (kext[j] % need != 0 && need % kext[j] != 0)) return false;
      const int b = std::min(need, kext[j]);
      box[d] = (cuuint32_t)b;
      need /= b;
    } else {
      box[d] = 1;
    }
    ++d;
  }
  if (nk > 1 && need != 1) return false;
  for (int j = 1; j < nx; ++j) {
    dim[d] = (cuuint64_t)xext[j];
    str[d - 1] = (cuuint64_t)xstr[j] * 8;
    box[d++] = 1;
  }
  for (int j = 0; j < rank - 1; ++j)
    if (str[j] % 16 != 0 || str[j] >= (1ULL << 40)) return false;
  auto enc = tma_encode();
  if (enc == nullptr) return false;
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dim, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  *rank_out = rank;
  return true;
}

bool tma_plan(const TcArgs& a, int BM, int BN, int batch, TmaMaps& maps) {
  if (!tma_enabled() || a.beta != 0.0 || a.a_kfast || a.b_kfast) return false;
  for (int b = 0; b < batch; ++b) {
    int ra = 0, rb = 0;
    if (!tma_map(&maps.a[b], a.A[b], a.nm, a.m_ext, a.a_m, a.nk, a.k_ext, a.a_k, BM, &ra)) return false;
    if (!tma_map(&maps.b[b], a.B[b], a.nn, a.n_ext, a.b_n, a.nk, a.k_ext, a.b_k, BN, &rb)) return false;
    maps.a_rank = ra;
    maps.b_rank = rb;
  }
  return true;
}

// Split-K reduction: C[off(m,n)] = alpha * sum_s P[b][s][m][n] (+ beta C), in split order.
// Two consecutive n per thread (16-byte partial loads when N is even), the output offsets by
// the magic-number divisions of the GEMM's own offset tables (no integer divide per element;
// the plain-division version took 50 us for S6 at C4, four times its DRAM time).
__global__ void splitk_reduce_kernel(const TcArgs args) {
  CTM_PDL_WAIT();
  const int b = blockIdx.y;
  const long long MN = (long long)args.M * args.N;
  const int N = args.N;
  const bool even = (N & 1) == 0;
  const long long npair = even ? MN / 2 : MN;
  double ss = 0.0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < npair; q += (long long)gridDim.x * blockDim.x) {
    const long long e = even ? 2 * q : q;
    const int m = (int)(e / N), n = (int)(e - (long long)m * N);
    int om, dummy, on;
    tc::mode_offset2(m, args.nm, args.m_ext, args.m_mag, args.m_sh, args.c_m, args.c_m, om, dummy);
    tc::mode_offset2(n, args.nn, args.n_ext, args.n_mag, args.n_sh, args.c_n, args.c_n, on, dummy);
    const double* P = args.part + (size_t)b * args.splits * MN + e;
    if (even) {
      double v0 = 0.0, v1 = 0.0;
      for (int s = 0; s < args.splits; ++s) {
        const double2 w = *reinterpret_cast<const double2*>(P + (size_t)s * MN);
        v0 += w.x;
        v1 += w.y;
      }
      int on1;
      tc::mode_offset2(n + 1, args.nn, args.n_ext, args.n_mag, args.n_sh, args.c_n, args.c_n, on1, dummy);
      v0 *= args.alpha;
      v1 *= args.alpha;
      if (args.beta != 0.0) {
        v0 += args.beta * args.C[b][om + on];
        v1 += args.beta * args.C[b][om + on1];
      }
      args.C[b][om + on] = v0;
      args.C[b][om + on1] = v1;
      ss += v0 * v0 + v1 * v1;
    } else {
      double v = 0.0;
      for (int s = 0; s < args.splits; ++s) v += P[(size_t)s * MN];
      v *= args.alpha;
      if (args.beta != 0.0) v += args.beta * args.C[b][om + on];
      args.C[b][om + on] = v;
      ss += v * v;
    }
  }
  if (args.sumsq[b] != nullptr) tc::block_sum_store(ss, args.sumsq[b] + blockIdx.x);
}



struct Leg {
  char c;
  int ext;
  long long sa = -1, sb = -1, sc = -1;   // row-major element strides (-1: absent)
};

std::vector<long long> rowmajor_strides(const std::vector<int>& ext) {
  std::vector<long long> s(ext.size());
  long long acc = 1;
  for (int i = (int)ext.size() - 1; i >= 0; --i) {
    s[i] = acc;
    acc *= ext[i];
  }
  return s;
}

// Order the legs of one group by the strides of the operand `key` (ascending), then merge
// neighbours that are contiguous in both operands that carry the group.
struct ModeOut {
  std::vector<int> ext;
  std::vector<long long> s1, s2;
};

ModeOut build_modes(std::vector<Leg> legs, int key, int op1, int op2) {
  auto S = [](const Leg& l, int op) { return op == 0 ? l.sa : (op == 1 ? l.sb : l.sc); };
  std::sort(legs.begin(), legs.end(), [&](const Leg& x, const Leg& y) { return S(x, key) < S(y, key); });
  ModeOut mo;
  for (const Leg& l : legs) {
    if (l.ext == 1) continue;     // trivial legs contribute nothing
    if (!mo.ext.empty()) {
      size_t j = mo.ext.size() - 1;
      bool c1 = S(l, op1) == mo.s1[j] * mo.ext[j];
      bool c2 = S(l, op2) == mo.s2[j] * mo.ext[j];
      if (c1 && c2) {
        mo.ext[j] *= l.ext;
        continue;
      }
    }
    mo.ext.push_back(l.ext);
    mo.s1.push_back(S(l, op1));
    mo.s2.push_back(S(l, op2));
  }
  if (mo.ext.empty()) {   // all-trivial group: one mode of extent 1
    mo.ext.push_back(1);
    mo.s1.push_back(0);
    mo.s2.push_back(0);
  }
  return mo;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB, bool FB, bool AKF, bool BKF, bool SEP>
void launch_cfg3(Handle& h, const TcArgs& a, int gz) {
  using C_ = tc::Cfg<BM, BN, BK, WM, WN, ST, MINB>;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, gz);
  if constexpr (FB && !AKF && !BKF) {   // operand tiles by TMA where the operands allow it
    // (only launches with at least a wave of output tiles: the solver's small GEMMs would pay
    //  the host-side map encoding on their latency-bound critical path)
    TmaMaps maps;
    if ((long long)grid.x * grid.y * gz >= 256 && tma_plan(a, BM, BN, gz / a.splits, maps)) {
      launch_k(tc::tc_gemm_tma_kernel<BM, BN, BK, WM, WN, ST, MINB>, grid, dim3(C_::THREADS), C_::SMEM_BYTES, h.stream, a,
               maps);
      CTM_CUDA(cudaGetLastError());
      h.count_kernel();
      return;
    }
  }
  auto kern = tc::tc_gemm_kernel<BM, BN, BK, WM, WN, ST, MINB, AKF, BKF, SEP, FB>;   // attributes: tc_init_kernels
  launch_k(kern, grid, dim3(C_::THREADS), C_::SMEM_BYTES, h.stream, a);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB, bool FB, bool AKF, bool BKF>
void launch_cfg2(Handle& h, const TcArgs& a, int gz) {
  if (a.ksep) launch_cfg3<BM, BN, BK, WM, WN, ST, MINB, FB, AKF, BKF, true>(h, a, gz);
  else launch_cfg3<BM, BN, BK, WM, WN, ST, MINB, FB, AKF, BKF, false>(h, a, gz);
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB, bool FB>
void launch_cfg(Handle& h, const TcArgs& a, int gz) {
  if (a.a_kfast) {
    if (a.b_kfast) launch_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, true, true>(h, a, gz);
    else launch_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, true, false>(h, a, gz);
  } else {
    if (a.b_kfast) launch_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, false, true>(h, a, gz);
    else launch_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, false, false>(h, a, gz);
  }
}

// Dynamic shared memory above 48 KB is a per-device function attribute: set it for every
// instantiation once per device (ctm_init, before any worker thread launches).
template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB, bool FB, bool AKF, bool BKF>
void set_attr_cfg2() {
  using C_ = tc::Cfg<BM, BN, BK, WM, WN, ST, MINB>;
  CTM_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<BM, BN, BK, WM, WN, ST, MINB, AKF, BKF, false, FB>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_BYTES));
  CTM_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<BM, BN, BK, WM, WN, ST, MINB, AKF, BKF, true, FB>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_BYTES));
}
template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB, bool FB>
void set_attr_cfg() {
  if constexpr (FB) {
    using C_ = tc::Cfg<BM, BN, BK, WM, WN, ST, MINB>;
    CTM_CUDA(cudaFuncSetAttribute(tc::tc_gemm_tma_kernel<BM, BN, BK, WM, WN, ST, MINB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_BYTES));
  }
  set_attr_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, true, true>();
  set_attr_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, true, false>();
  set_attr_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, false, true>();
  set_attr_cfg2<BM, BN, BK, WM, WN, ST, MINB, FB, false, false>();
}

struct CfgInfo {
  int BM, BN;
  int per_sm;   // resident CTAs per SM
  double eff;   // relative per-tile efficiency (bigger tiles reuse operands more)
};
// 0: 128x64 (8 warps 4x2), 1: 64x128 (8 warps 2x4), 2: 64x64 (4 warps 2x2); warp tile 32x32
// (a 128x128 tile with 64x32 warp tiles -- 64 accumulator doubles, one CTA per SM -- measured
// slower than 128x64 on every chain step but S3: profiles/r02_launches_inject_cfg3.txt)
// The two 8-warp configs double-buffer their DMMA fragments (FB: tc_gemm.cuh), the 4-warp one
// does not (its 1024 x 160 solver GEMMs ran slower with it).  (round 2: 64x128 / 128x64 with
// four 32x64 / 64x32 warp tiles -- cuBLAS's sm80 DGEMM tiles for these shapes -- and 64x32 at
// three CTAs per SM were slower on every chain step: profiles/r02_launches_inject_tile_cfgs.txt)
const CfgInfo kCfgs[] = {{128, 64, 2, 1.00}, {64, 128, 2, 1.00}, {64, 64, 3, 0.85}};
constexpr int kNumCfgs = 3;
constexpr int kSMs = 148;

void launch_idx(Handle& h, int idx, const TcArgs& a, int gz) {
  switch (idx) {
    case 0: launch_cfg<128, 64, 16, 4, 2, 3, 2, true>(h, a, gz); break;
    case 1: launch_cfg<64, 128, 16, 2, 4, 3, 2, true>(h, a, gz); break;
    default: launch_cfg<64, 64, 16, 2, 2, 3, 3, false>(h, a, gz); break;
  }
}

}  // namespace

void tc_init_kernels() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  CTM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(dev)) return;
  set_attr_cfg<128, 64, 16, 4, 2, 3, 2, true>();
  set_attr_cfg<64, 128, 16, 2, 4, 3, 2, true>();
  set_attr_cfg<64, 64, 16, 2, 2, 3, 3, false>();
  done.insert(dev);
}

int contract(Handle& h, const Operand& A, const Operand& B, const OutOperand& C, double alpha, GemmPartials* defer) {
  if (defer) *defer = GemmPartials{};
  const int batch = (int)C.p.size();
  if (batch < 1 || batch > CTM_MAXBATCH || (int)A.p.size() != batch || (int)B.p.size() != batch)
    throw Error(CTM_E_ARG, "contract: bad batch");
  if (A.lab.size() != A.ext.size() || B.lab.size() != B.ext.size() || C.lab.size() != C.ext.size())
    throw Error(CTM_E_ARG, "contract: label/extent rank mismatch");
  std::map<char, Leg> legs;
  auto add = [&](const std::string& lab, const std::vector<int>& ext, int op) {
    auto st = rowmajor_strides(ext);
    for (size_t i = 0; i < lab.size(); ++i) {
      Leg& l = legs[lab[i]];
      if (l.c == 0) {
        l.c = lab[i];
        l.ext = ext[i];
      } else if (l.ext != ext[i]) {
        throw Error(CTM_E_ARG, std::string("contract: extent mismatch on leg ") + lab[i] + " (" +
                                   A.lab + "," + B.lab + "->" + C.lab + ")");
      }
      (op == 0 ? l.sa : op == 1 ? l.sb : l.sc) = st[i];
    }
  };
  add(A.lab, A.ext, 0);
  add(B.lab, B.ext, 1);
  add(C.lab, C.ext, 2);
  std::vector<Leg> gm, gn, gk;
  for (auto& kv : legs) {
    const Leg& l = kv.second;
    bool a = l.sa >= 0, b = l.sb >= 0, c = l.sc >= 0;
    if (a && c && !b) gm.push_back(l);
    else if (b && c && !a) gn.push_back(l);
    else if (a && b && !c) gk.push_back(l);
    else throw Error(CTM_E_ARG, std::string("contract: leg ") + l.c + " must be in exactly two operands");
  }
  auto fastest = [&](int op) {   // label with stride 1 in operand op
    for (auto& kv : legs) {
      const Leg& l = kv.second;
      long long s = op == 0 ? l.sa : op == 1 ? l.sb : l.sc;
      if (s == 1 && l.ext > 1) return l.c;
    }
    return (char)0;
  };
  auto in_group = [](const std::vector<Leg>& g, char c) {
    for (auto& l : g)
      if (l.c == c) return true;
    return false;
  };
  const char fa = fastest(0), fb = fastest(1), fc = fastest(2);
  const bool a_kfast = in_group(gk, fa);
  const bool b_kfast = in_group(gk, fb);
  const bool c_nfast = in_group(gn, fc);
  // m modes: A then C ; n modes: B then C ; k modes: A then B.
  int key_m = in_group(gm, fa) ? 0 : (in_group(gm, fc) ? 2 : 0);
  int key_n = in_group(gn, fb) ? 1 : (in_group(gn, fc) ? 2 : 1);
  int key_k = a_kfast ? 0 : (b_kfast ? 1 : 0);
  ModeOut mm = build_modes(gm, key_m, 0, 2);
  ModeOut mn = build_modes(gn, key_n, 1, 2);
  ModeOut mk = build_modes(gk, key_k, 0, 1);
  if (mm.ext.size() > CTM_MAXMODES || mn.ext.size() > CTM_MAXMODES || mk.ext.size() > CTM_MAXMODES)
    throw Error(CTM_E_ARG, "contract: more than 4 modes in a group (" + A.lab + "," + B.lab + "->" + C.lab + ")");
  TcArgs a{};
  long long M = 1, N = 1, K = 1;
  for (int e : mm.ext) M *= e;
  for (int e : mn.ext) N *= e;
  for (int e : mk.ext) K *= e;
  if (M >= (1LL << 31) || N >= (1LL << 31))
    throw Error(CTM_E_ARG, "contract: GEMM too large");
  // K beyond the shared-memory offset tables: split the slowest k mode into chunks and
  // accumulate (beta = 1) -- used only by the closures (K = chi D^2).
  const long long k_last = mk.ext.back();
  const long long k_inner = K / k_last;
  if (K > CTM_KTAB_MAX && k_inner > CTM_KTAB_MAX)
    throw Error(CTM_E_ARG, "contract: inner K too large, K=" + std::to_string(K));
  auto elems = [](const std::vector<int>& e) {
    long long n = 1;
    for (int x : e) n *= x;
    return n;
  };
  if (elems(A.ext) >= (1LL << 31) || elems(B.ext) >= (1LL << 31) || elems(C.ext) >= (1LL << 31))
    throw Error(CTM_E_ARG, "contract: operand exceeds 2^31 elements");
  a.M = (int)M;
  a.N = (int)N;
  a.K = (int)K;
  a.nm = (int)mm.ext.size();
  a.nn = (int)mn.ext.size();
  a.nk = (int)mk.ext.size();
  for (int i = 0; i < a.nm; ++i) {
    a.m_ext[i] = mm.ext[i];
    a.a_m[i] = (int)mm.s1[i];
    a.c_m[i] = (int)mm.s2[i];
  }
  for (int i = 0; i < a.nn; ++i) {
    a.n_ext[i] = mn.ext[i];
    a.b_n[i] = (int)mn.s1[i];
    a.c_n[i] = (int)mn.s2[i];
  }
  for (int i = 0; i < a.nk; ++i) {
    a.k_ext[i] = mk.ext[i];
    a.a_k[i] = (int)mk.s1[i];
    a.b_k[i] = (int)mk.s2[i];
  }
  // round-up reciprocals (Granlund-Montgomery, 31-bit dividends): sh = ceil(log2 e),
  // mag = floor(2^32 (2^sh - e) / e) + 1, q = (umulhi(i, mag) + i) >> sh
  auto magic = [](int e, unsigned& mag, int& sh) {
    int s2 = 0;
    while ((1LL << s2) < e) ++s2;
    sh = s2;
    mag = (unsigned)((((unsigned long long)1 << 32) * (((unsigned long long)1 << s2) - (unsigned long long)e)) /
                     (unsigned long long)e + 1ULL);
    if (e == 1) mag = 0;
  };
  for (int i = 0; i < a.nm; ++i) magic(a.m_ext[i], a.m_mag[i], a.m_sh[i]);
  for (int i = 0; i < a.nn; ++i) magic(a.n_ext[i], a.n_mag[i], a.n_sh[i]);
  for (int i = 0; i < a.nk; ++i) magic(a.k_ext[i], a.k_mag[i], a.k_sh[i]);
  a.a_kfast = a_kfast;
  a.b_kfast = b_kfast;
  // separable k offsets: the 16-wide k-tiles (starting at multiples of 16) never straddle a
  // k-mode boundary except by whole cycles of the inner modes -- some prefix product of the
  // k extents divides 16 while the next one is a multiple of 16 (or K ends first)
  a.ksep = [&] {
    long long P = 1;
    for (int e : mk.ext) {
      if (16 % P != 0) return 0;
      P *= e;
      if (P % 16 == 0) return 1;
    }
    return 1;
  }();
  if (std::getenv("CTM_TC_NOSEP")) a.ksep = 0;   // A/B
  (void)c_nfast;
  a.alpha = alpha;
  a.beta = 0.0;
  for (int b = 0; b < batch; ++b) {
    a.A[b] = A.p[b];
    a.B[b] = B.p[b];
    a.C[b] = C.p[b];
    a.sumsq[b] = C.sumsq.empty() ? nullptr : C.sumsq[b];
  }
  h.flops += 2.0 * (double)M * (double)N * (double)K * batch;
  a.splits = 1;
  a.ktiles_per_split = (int)((K + 15) / 16);
  a.part = nullptr;
  // tile-config choice: maximise (wave efficiency) x (tile fill) x (per-tile efficiency),
  // then split K when one wave is not filled (deterministic split-K reduction).
  int best = 0, best_splits = 1;
  double best_score = -1;
  const long long ktiles_all = (K + 15) / 16;
  static const int forced = [] {   // CTM_TC_CFG=0|1|2 pins the tile config (experiments)
    const char* e = std::getenv("CTM_TC_CFG");
    return e ? std::atoi(e) : -1;
  }();
  for (int i = 0; i < kNumCfgs; ++i) {
    if (forced >= 0 && i != forced) continue;
    const CfgInfo& c = kCfgs[i];
    long long tm = (M + c.BM - 1) / c.BM, tn = (N + c.BN - 1) / c.BN;
    long long tiles = tm * tn * batch;
    const long long slots = (long long)kSMs * c.per_sm;
    // candidates: no split, and (when one wave is not filled) the split that fills two
    // waves; a split pays its partial-tile traffic and the reduction (split_cost).  (S6 at
    // C4 -- 256 tiles on 296 slots -- runs one full-K wave instead of 3 splits + reduction.)
    int cand[2] = {1, 1};
    if (tiles < slots && K <= CTM_KTAB_MAX) {
      long long want = (2 * slots + tiles - 1) / tiles;
      cand[1] = (int)std::max(1LL, std::min({want, 8LL, ktiles_all / 4}));
    }
    const double fill = (double)M * N / ((double)tm * c.BM * tn * c.BN);
    for (int splits : cand) {
      const long long ctas = tiles * splits;
      const long long waves = (ctas + slots - 1) / slots;
      const double wave_eff = (double)ctas / (waves * (double)slots);
      const double split_cost = splits > 1 ? 0.97 : 1.0;
      const double score = fill * wave_eff * c.eff * split_cost;
      if (score > best_score + 1e-9) {
        best_score = score;
        best = i;
        best_splits = splits;
      }
    }
  }
  if (!C.sumsq.empty() && best_splits == 1) {
    // the fused sum of squares writes one partial per output tile into a CTM_SS_SLOTS slot
    // range (the split-K path writes one per reduction CTA, <= 2 x 148): refuse a launch
    // that would overflow into the neighbouring slots (fails in ctm_init's sizing pass)
    const long long tiles = ((M + kCfgs[best].BM - 1) / kCfgs[best].BM) * ((N + kCfgs[best].BN - 1) / kCfgs[best].BN);
    if (tiles > CTM_SS_SLOTS)
      throw Error(CTM_E_ARG, "contract: " + std::to_string(tiles) + " output tiles exceed the " +
                                 std::to_string(CTM_SS_SLOTS) + " sum-of-squares slots (chi D too large)");
  }
  if (h.dry) {
    // sizing pass: reserve exactly the split-K slab the real launch will take (the tile /
    // split choice above depends on shapes only); no slab when the launch is not split
    if (best_splits > 1) {
      const size_t mark = h.ws.top;
      h.ws.take((size_t)batch * best_splits * M * N);
      h.ws.reset(mark);
    }
    return 0;
  }
  const bool prof = (h.prm.flags & CTM_FLAG_PROFILE) != 0;
  auto prof_begin = [&]() {
    if (!prof) return;
    if ((int)h.prof_ev.size() < 2 * (h.prof_used + 1)) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        CTM_CUDA(cudaEventCreate(&e));
        h.prof_ev.push_back(e);
      }
    }
    CTM_CUDA(cudaEventRecord(h.prof_ev[2 * h.prof_used], h.stream));
  };
  auto prof_end = [&](double flops) {
    if (!prof) return;
    CTM_CUDA(cudaEventRecord(h.prof_ev[2 * h.prof_used + 1], h.stream));
    if ((int)h.prof_flops.size() <= h.prof_used) h.prof_flops.resize(h.prof_used + 1);
    h.prof_flops[h.prof_used] = flops;
    ++h.prof_used;
  };
  if (best_splits > 1) {
    const size_t mark = h.ws.top;
    a.splits = best_splits;
    a.ktiles_per_split = (int)((ktiles_all + best_splits - 1) / best_splits);
    a.part = h.ws.take((size_t)batch * best_splits * M * N);
    prof_begin();
    launch_idx(h, best, a, batch * best_splits);
    // deferred reduction: a single problem whose output is plain row-major [M][N] (the
    // slab's own layout), alpha = 1, no fused sum of squares -- the consumer sums the partials
    bool plain = defer != nullptr && batch == 1 && alpha == 1.0 && C.sumsq.empty();
    long long s = 1;
    for (int i = 0; plain && i < a.nn; ++i) {
      plain = a.c_n[i] == s;
      s *= a.n_ext[i];
    }
    for (int i = 0; plain && i < a.nm; ++i) {
      plain = a.c_m[i] == s;
      s *= a.m_ext[i];
    }
    if (plain) {
      prof_end(2.0 * (double)M * N * K * batch);
      defer->p = a.part;
      defer->splits = best_splits;
      defer->mn = (long long)M * N;
      h.ws.reset(mark);
      return 0;
    }
    int rb = (int)std::min<long long>(2 * kSMs, ((long long)M * N + 255) / 256);
    launch_k(splitk_reduce_kernel, dim3(rb, batch), dim3(256), 0, h.stream, a);
    CTM_CUDA(cudaGetLastError());
    h.count_kernel();
    prof_end(2.0 * (double)M * N * K * batch);
    h.ws.reset(mark);
    return rb;
  }
  // K beyond the shared-memory offset table: chunk the slowest k mode (beta = 1)
  const long long chunk = K > CTM_KTAB_MAX ? CTM_KTAB_MAX / k_inner : k_last;
  const int lk = a.nk - 1;
  const long long sa_last = mk.s1[lk], sb_last = mk.s2[lk];
  int nparts = 0;
  for (long long j0 = 0; j0 < k_last; j0 += chunk) {
    TcArgs c = a;
    const long long len = std::min(chunk, k_last - j0);
    c.k_ext[lk] = (int)len;
    magic(c.k_ext[lk], c.k_mag[lk], c.k_sh[lk]);
    c.K = (int)(k_inner * len);
    c.beta = j0 == 0 ? 0.0 : 1.0;
    c.splits = 1;
    c.ktiles_per_split = (c.K + 15) / 16;
    c.ksep = 0;   // (the chunk's last k extent differs from the planned one; closures only)
    for (int b = 0; b < batch; ++b) {
      c.A[b] = a.A[b] + j0 * sa_last;
      c.B[b] = a.B[b] + j0 * sb_last;
      c.sumsq[b] = (j0 + len >= k_last) ? a.sumsq[b] : nullptr;
    }
    prof_begin();
    launch_idx(h, best, c, batch);
    prof_end(2.0 * (double)c.M * c.N * c.K * batch);
    nparts = (int)(((M + kCfgs[best].BM - 1) / kCfgs[best].BM) * ((N + kCfgs[best].BN - 1) / kCfgs[best].BN));
  }
  return nparts;
}

}  // namespace ctm
