// tc_gemm.cu -- contraction planner (labels -> strided GEMM modes) and launcher for the
// FP64 DMMA kernel of tc_gemm.cuh.
#include <algorithm>
#include <cmath>
#include <map>

#include "ctm_internal.h"

namespace ctm {
namespace {

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

template <int BM, int BN, int BK, int WM, int WN, int ST>
void launch_cfg(Handle& h, const TcArgs& a, int batch) {
  using C_ = tc::Cfg<BM, BN, BK, WM, WN, ST>;
  auto kern = tc::tc_gemm_kernel<BM, BN, BK, WM, WN, ST>;
  static bool attr_set = false;
  if (!attr_set) {
    CTM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_BYTES));
    attr_set = true;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, batch);
  kern<<<grid, C_::THREADS, C_::SMEM_BYTES, h.stream>>>(a);
  CTM_CUDA(cudaGetLastError());
  h.count_kernel();
}

struct CfgInfo {
  int BM, BN;
  double eff;   // relative per-tile efficiency (bigger tiles reuse operands more)
};
const CfgInfo kCfgs[] = {{128, 128, 1.00}, {128, 64, 0.92}, {64, 128, 0.92}, {64, 64, 0.80}};

}  // namespace

void contract(Handle& h, const Operand& A, const Operand& B, const OutOperand& C, double alpha) {
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
  a.a_kfast = a_kfast;
  a.b_kfast = b_kfast;
  a.c_nfast = c_nfast;
  a.alpha = alpha;
  a.beta = 0.0;
  for (int b = 0; b < batch; ++b) {
    a.A[b] = A.p[b];
    a.B[b] = B.p[b];
    a.C[b] = C.p[b];
    a.sumsq[b] = C.sumsq.empty() ? nullptr : C.sumsq[b];
  }
  h.flops += 2.0 * (double)M * (double)N * (double)K * batch;
  if (h.dry) return;
  // tile-config choice: maximise (wave efficiency) x (tile fill) x (per-tile efficiency)
  int best = 0;
  double best_score = -1;
  for (int i = 0; i < 4; ++i) {
    const CfgInfo& c = kCfgs[i];
    long long tm = (M + c.BM - 1) / c.BM, tn = (N + c.BN - 1) / c.BN;
    long long tiles = tm * tn * batch;
    double fill = (double)M * N / ((double)tm * c.BM * tn * c.BN);
    long long waves = (tiles + 147) / 148;
    double wave_eff = (double)tiles / (waves * 148.0);
    double score = fill * wave_eff * c.eff;
    if (score > best_score + 1e-9) {
      best_score = score;
      best = i;
    }
  }
  const long long chunk = K > CTM_KTAB_MAX ? CTM_KTAB_MAX / k_inner : k_last;
  const int lk = a.nk - 1;
  const long long sa_last = mk.s1[lk], sb_last = mk.s2[lk];
  for (long long j0 = 0; j0 < k_last; j0 += chunk) {
    TcArgs c = a;
    const long long len = std::min(chunk, k_last - j0);
    c.k_ext[lk] = (int)len;
    c.K = (int)(k_inner * len);
    c.beta = j0 == 0 ? 0.0 : 1.0;
    for (int b = 0; b < batch; ++b) {
      c.A[b] = a.A[b] + j0 * sa_last;
      c.B[b] = a.B[b] + j0 * sb_last;
      c.sumsq[b] = (j0 + len >= k_last) ? a.sumsq[b] : nullptr;
    }
    switch (best) {
      case 0: launch_cfg<128, 128, 16, 2, 4, 3>(h, c, batch); break;
      case 1: launch_cfg<128, 64, 16, 2, 2, 4>(h, c, batch); break;
      case 2: launch_cfg<64, 128, 16, 2, 2, 4>(h, c, batch); break;
      default: launch_cfg<64, 64, 16, 2, 2, 4>(h, c, batch); break;
    }
  }
}

}  // namespace ctm
