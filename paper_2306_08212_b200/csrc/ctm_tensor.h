// ctm_tensor.h -- small host-side tensor views shared by the move driver (ctm_abi.cu) and
// the imaginary-time / FFU driver (ffu.cu): a row-major device tensor with its extents, the
// environment accessors, labelled operands for contract(), arena allocation, and the quarter
// turns of the picture (SURVEY 0 clockwise storage).
#pragma once
#include <vector>

#include "ctm_internal.h"

namespace ctm {

// ---------------------------------------------------------------------------------------
// small tensor views
// ---------------------------------------------------------------------------------------
struct Ten {
  double* p = nullptr;
  std::vector<int> ext;
  size_t size() const {
    size_t n = 1;
    for (int e : ext) n *= (size_t)e;
    return n;
  }
};

// ---------------------------------------------------------------------------------------
// Environment access
// ---------------------------------------------------------------------------------------
inline Ten envC(const ctm_env* e, int x, int k) {
  return Ten{e->C[x][k - 1], {e->ext[x][k - 1][0], e->ext[x][k - 1][1]}};
}
inline Ten envT(const ctm_env* e, int x, int k, int D) {
  return Ten{e->T[x][k - 1], {e->ext[x][4 + k - 1][0], D, D, e->ext[x][4 + k - 1][1]}};
}

inline Operand op(const std::vector<const Ten*>& ts, const char* lab) {
  Operand o;
  o.lab = lab;
  o.ext = ts[0]->ext;
  for (auto* t : ts) o.p.push_back(t->p);
  return o;
}
inline OutOperand out(const std::vector<Ten*>& ts, const char* lab, const std::vector<double*>& ss = {}) {
  OutOperand o;
  o.lab = lab;
  o.ext = ts[0]->ext;
  for (auto* t : ts) o.p.push_back(t->p);
  o.sumsq = ss;
  return o;
}
inline Ten alloc(Handle& h, std::vector<int> ext) {
  Ten t;
  t.ext = std::move(ext);
  t.p = h.ws.take(t.size());
  return t;
}

// Quarter turns (clockwise storage: relabel k -> k+1, no data movement).
inline void rotate_env_cw(ctm_env* e) {
  ctm_env o = *e;
  for (int x = 0; x < 2; ++x)
    for (int k = 0; k < 4; ++k) {
      int nk = (k + 1) % 4;
      e->C[x][nk] = o.C[x][k];
      e->T[x][nk] = o.T[x][k];
      e->ext[x][nk][0] = o.ext[x][k][0];
      e->ext[x][nk][1] = o.ext[x][k][1];
      e->ext[x][4 + nk][0] = o.ext[x][4 + k][0];
      e->ext[x][4 + nk][1] = o.ext[x][4 + k][1];
    }
}

// Site leg permutation for n clockwise quarter turns: (s,u,l,d,r) -> turned.
inline void rotate_site(Handle& h, const double* X, double* out, int turns) {
  static const int perms[4][5] = {{0, 1, 2, 3, 4}, {0, 2, 3, 4, 1}, {0, 3, 4, 1, 2}, {0, 4, 1, 2, 3}};
  const int* pm = perms[turns & 3];
  permute(h, X, {h.prm.d, h.prm.D, h.prm.D, h.prm.D, h.prm.D}, {pm[0], pm[1], pm[2], pm[3], pm[4]}, out);
}


}  // namespace ctm
