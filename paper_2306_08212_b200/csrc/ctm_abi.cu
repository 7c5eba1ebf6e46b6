// ctm_abi.cu -- libctm: the C ABI of include/ctm.h and the CTMRG move driver.
//
// Every contraction of the move runs in tc_gemm (FP64 DMMA, permutations fused into the
// loads), every SVD on the device (svd.cu), every elementwise step in kernels.cu.  The
// host code here only plans shapes, walks the paper's steps and checks statuses.
//
// Citations: P:Lnn = PAPER.md line; rows a1..a11 and S1..S6 = SURVEY.md 8(a).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <future>
#include <thread>
#include <exception>

#include "ctm_internal.h"
#include "ctm_tensor.h"

namespace ctm {
namespace {

// Site tensor in the two orientations the chain needs (S2 / S5 operands).
struct Site {
  Ten ket;   // (in, face, s, out, far)            "ifsoz"
  Ten bra;   // (s, face, in, out, far)            "sgjyw"
};

// X (s,u,l,d,r) -> chain orientation given by the source axes of (in, face, out, far).
Site make_site(Handle& h, const double* X, const double* Xb, int d, int D, int in, int face, int outl, int far) {
  Site s;
  s.ket = alloc(h, {D, D, d, D, D});
  s.bra = alloc(h, {d, D, D, D, D});
  if (!h.dry) {
    permute(h, X, {d, D, D, D, D}, {in, face, 0, outl, far}, s.ket.p);
    permute(h, Xb, {d, D, D, D, D}, {0, face, in, outl, far}, s.bra.p);
  }
  return s;
}
// (s,u,l,d,r) axes: s=0 u=1 l=2 d=3 r=4
Site site_left(Handle& h, const double* X, int d, int D) { return make_site(h, X, X, d, D, 3, 2, 1, 4); }
Site site_top(Handle& h, const double* X, int d, int D) { return make_site(h, X, X, d, D, 2, 1, 4, 3); }

struct Iso {
  Ten v1, v2;   // v1 (P, D, n1), v2 (n1, D, n2)
  double gap1 = std::numeric_limits<double>::infinity();   // stage one sigma_n1 / sigma_{n1+1}
  double gap2 = std::numeric_limits<double>::infinity();   // stage two (inf: nothing truncated)
};

// ---------------------------------------------------------------------------------------
// Rows a6-a8: sequential absorb/truncate chain S1..S6 (Fig 4(b)).
// Batched over jobs with identical shapes.
// ---------------------------------------------------------------------------------------
struct ChainJob {
  const Ten* T;          // (cin, D, D, cout) as (in, face_k, face_b, out)
  const Site* X;
  const Iso* in;         // v1 (cin, D, n1), v2 (n1, D, o1)
  const Iso* outv;       // v1 (cout, D, m1), v2 (m1, D, o2)
  Ten* res;              // (o1, D, D, o2), allocated by the caller
  double* ss;            // nullable: fused sum of squares of res
};

int chain_batch(Handle& h, const std::vector<ChainJob>& jobs) {
  const int B = (int)jobs.size();
  const ChainJob& j0 = jobs[0];
  const int D = j0.T->ext[1];
  const int d = j0.X->bra.ext[0];
  const int cout = j0.T->ext[3];
  const int n1 = j0.in->v1.ext[2], o1 = j0.in->v2.ext[2];
  const int m1 = j0.outv->v1.ext[2], o2 = j0.outv->v2.ext[2];
  const size_t mark = h.ws.top;
  std::vector<Ten> X1(B), X2(B), X3(B), X4(B), X5(B);
  for (int b = 0; b < B; ++b) {
    // buf1 holds X1 / X3 / X5, buf2 holds X2 / X4 (lifetimes do not overlap)
    size_t s1 = std::max({(size_t)D * n1 * D * D * cout, (size_t)n1 * D * d * D * m1, (size_t)m1 * D * D * D * o1});
    size_t s2 = std::max((size_t)n1 * D * d * D * D * cout, (size_t)d * D * D * D * m1 * o1);
    double* b1 = h.ws.take(s1);
    double* b2 = h.ws.take(s2);
    X1[b] = {b1, {D, n1, D, D, cout}};
    // X2 stored (o, q, a, g, s, z): S3 contracts (q, o), its slowest legs, so S3's A tile is
    // m-fast (a contiguous 128-element run) instead of k-fast
    X2[b] = {b2, {D, cout, n1, D, d, D}};
    X3[b] = {b1, {n1, D, d, D, m1}};
    X4[b] = {b2, {d, D, D, D, m1, o1}};
    X5[b] = {b1, {m1, D, D, D, o1}};
  }
  auto P = [&](auto f) {
    std::vector<const Ten*> v;
    for (int b = 0; b < B; ++b) v.push_back(f(b));
    return v;
  };
  auto Q = [&](std::vector<Ten>& t) {
    std::vector<Ten*> v;
    for (int b = 0; b < B; ++b) v.push_back(&t[b]);
    return v;
  };
  std::vector<Ten*> res;
  std::vector<double*> ss;
  for (auto& j : jobs) {
    res.push_back(j.res);
    if (j.ss) ss.push_back(j.ss);
  }
  if (!ss.empty() && (int)ss.size() != B) throw Error(CTM_E_ARG, "chain: partial sumsq");
  // S1: X1(i,a,f,g,q) = sum_p v1_in(p,i,a) T(p,f,g,q)                     K = chi
  contract(h, op(P([&](int b) { return &jobs[b].in->v1; }), "pia"), op(P([&](int b) { return jobs[b].T; }), "pfgq"),
           out(Q(X1), "iafgq"));
  // S2: X2(o,q,a,g,s,z) = sum_{i,f} X1(i,a,f,g,q) X(i,f,s,o,z)               K = D^2
  contract(h, op(P([&](int b) { return (const Ten*)&X1[b]; }), "iafgq"),
           op(P([&](int b) { return &jobs[b].X->ket; }), "ifsoz"), out(Q(X2), "oqagsz"));
  // S3: X3(a,g,s,z,b) = sum_{q,o} X2(o,q,a,g,s,z) v1_out(q,o,b)               K = chi D
  contract(h, op(P([&](int b) { return (const Ten*)&X2[b]; }), "oqagsz"),
           op(P([&](int b) { return &jobs[b].outv->v1; }), "qob"), out(Q(X3), "agszb"));
  // S4: X4(s,g,j,z,b,c) = sum_a X3(a,g,s,z,b) v2_in(a,j,c)                   K = chi'
  contract(h, op(P([&](int b) { return (const Ten*)&X3[b]; }), "agszb"),
           op(P([&](int b) { return &jobs[b].in->v2; }), "ajc"), out(Q(X4), "sgjzbc"));
  // S5: X5(b,y,z,w,c) = sum_{s,g,j} X4(s,g,j,z,b,c) X*(s,g,j,y,w)            K = d D^2
  contract(h, op(P([&](int b) { return (const Ten*)&X4[b]; }), "sgjzbc"),
           op(P([&](int b) { return &jobs[b].X->bra; }), "sgjyw"), out(Q(X5), "byzwc"));
  // S6: T'(c,z,w,d) = sum_{b,y} X5(b,y,z,w,c) v2_out(b,y,d)                  K = chi' D
  int np = contract(h, op(P([&](int b) { return (const Ten*)&X5[b]; }), "byzwc"),
                    op(P([&](int b) { return &jobs[b].outv->v2; }), "byd"), out(res, "czwd", ss));
  h.ws.reset(mark);
  return np;
}

bool same_shapes(const ChainJob& a, const ChainJob& b) {
  return a.T->ext == b.T->ext && a.in->v1.ext == b.in->v1.ext && a.in->v2.ext == b.in->v2.ext &&
         a.outv->v1.ext == b.outv->v1.ext && a.outv->v2.ext == b.outv->v2.ext;
}

// Returns the sum-of-squares partial count of each job's result.
std::vector<int> chains(Handle& h, const std::vector<ChainJob>& jobs) {
  if (jobs.size() == 2 && same_shapes(jobs[0], jobs[1])) {
    int np = chain_batch(h, jobs);
    return {np, np};
  }
  std::vector<int> r;
  for (auto& j : jobs) r.push_back(chain_batch(h, {j}));
  return r;
}

// ---------------------------------------------------------------------------------------
// Row a2 / a5: two-stage isometry TS(Q; c1, c2).
//   Q (P, D, D, F) as (boundary, ket, bra, far); returns v1 (P, D, n1), v2 (n1, D, n2) and
//   optionally Q2 = v1^T Q (n1, D, F), which the reduced env reuses for C' (row a4).
// ---------------------------------------------------------------------------------------
// basis2: a stage two that truncates nothing ((n1 D) x F keeping all F columns) returns an
// orthonormal basis of its column space instead of its left singular vectors (svd_left's
// basis_only; readings R24, R24b): the projector v v^T -- all the move uses -- is the same.
// The move takes it for every cut: side TS (R24: the output bond is contracted on both
// sides of M) and main TS (R24b: an orthogonal change of the new bond's basis is a gauge
// transformation of the new environment).
Iso ts_isometry(Handle& h, const Ten& Qt, int c1, int c2, Ten* Q2_keep, bool basis2 = false) {
  const int P = Qt.ext[0], K = Qt.ext[1], Bd = Qt.ext[2], F = Qt.ext[3];
  const int n1 = std::min(c1, P * K);
  Iso r;
  r.v1 = alloc(h, {P, K, n1});
  r.gap1 = svd_left(h, Qt.p, P * K, Bd * F, n1, r.v1.p);   // (warm-started from h.warm_slot, if set)
  h.warm_slot = -1;                                         // stage one only
  Ten Q2 = alloc(h, {n1, Bd, F});
  contract(h, op({&r.v1}, "pka"), op({&Qt}, "pkbq"), out({&Q2}, "abq"));   // v^1 contracted into Q
  const int n2 = std::min(c2, n1 * Bd);
  r.v2 = alloc(h, {n1, Bd, n2});
  r.gap2 = svd_left(h, Q2.p, n1 * Bd, F, n2, r.v2.p, basis2);
  if (Q2_keep) *Q2_keep = Q2;
  return r;
}

// ---------------------------------------------------------------------------------------
// Rows a1-a4: approximated reduced environment M = C'^1 T'^2 C'^2 (Fig 3(c),
// appendix).  Batched over the two cut types when shapes agree.
// ---------------------------------------------------------------------------------------
struct RenvIn {
  Ten C1, T2, C2, T1, T3;   // storage orders C1 (d,r), T2 (l,k,b,r), C2 (l,d), T1 (d,k,b,u), T3 (u,k,b,d)
  const Site* X;            // top orientation
};
struct RenvOut {
  Ten M;                    // (q, k, b, q')
  Iso vl, vr;
};

// a1 + a2 for one side: Q = C^1 T^1 (left) or C^2 T^3 (right), then TS(Q; chi'', chi'').
struct SideOut {
  Iso v;
  Ten Q2;   // v^1 contracted into Q: (n1, D, F), reused for C' / C'' (row a4)
};
SideOut side_ts(Handle& h, const RenvIn& in, bool left, int chi_pp) {
  const int D = in.T1.ext[1];
  SideOut o;
  if (left) {   // Q_l(p,k,b,q) = sum_x C1(x,p) T1(q,k,b,x)
    Ten Q = alloc(h, {in.C1.ext[1], D, D, in.T1.ext[0]});
    contract(h, op({&in.C1}, "xp"), op({&in.T1}, "qkbx"), out({&Q}, "pkbq"));
    o.v = ts_isometry(h, Q, chi_pp, chi_pp, &o.Q2, true);
  } else {      // Q_r(p,k,b,q) = sum_x C2(p,x) T3(x,k,b,q)
    Ten Q = alloc(h, {in.C2.ext[0], D, D, in.T3.ext[3]});
    contract(h, op({&in.C2}, "px"), op({&in.T3}, "xkbq"), out({&Q}, "pkbq"));
    o.v = ts_isometry(h, Q, chi_pp, chi_pp, &o.Q2, true);
  }
  return o;
}

// a1 + the v^1 contraction of a2 with INJECTED side isometries (no SVD): the reduced-env
// contractions timed alone (bench.py roofline_renv).  v (v1 (P, D, n1), v2 (n1, D, n2)).
SideOut side_inject(Handle& h, const RenvIn& in, bool left, const double* v1, const double* v2, int n1, int n2) {
  const int D = in.T1.ext[1];
  SideOut o;
  Ten Q = left ? alloc(h, {in.C1.ext[1], D, D, in.T1.ext[0]}) : alloc(h, {in.C2.ext[0], D, D, in.T3.ext[3]});
  if (left) contract(h, op({&in.C1}, "xp"), op({&in.T1}, "qkbx"), out({&Q}, "pkbq"));
  else contract(h, op({&in.C2}, "px"), op({&in.T3}, "xkbq"), out({&Q}, "pkbq"));
  const int P = Q.ext[0], F = Q.ext[3];
  o.v.v1 = Ten{const_cast<double*>(v1), {P, D, n1}};
  o.v.v2 = Ten{const_cast<double*>(v2), {n1, D, n2}};
  o.Q2 = alloc(h, {n1, D, F});
  contract(h, op({&o.v.v1}, "pka"), op({&Q}, "pkbq"), out({&o.Q2}, "abq"));
  return o;
}

// a3 + a4: M = C' T'^2 C'' from the two side isometries.
RenvOut renv_finish(Handle& h, const RenvIn& in, const SideOut& L, const SideOut& R) {
  RenvOut o;
  o.vl = L.v;
  o.vr = R.v;
  const int D = in.T1.ext[1];
  // a3: T'^2 = chain(T^2, X top orientation, in = v_l, out = v_r)
  Ten Tp = alloc(h, {o.vl.v2.ext[2], D, D, o.vr.v2.ext[2]});
  chains(h, {ChainJob{&in.T2, in.X, &o.vl, &o.vr, &Tp, nullptr}});
  // a4: C'(q,l) = sum_{a,b} Q2l(a,b,q) vl2(a,b,l); C''(r,q') = sum vr2(a,b,r) Q2r(a,b,q')
  Ten Cl = alloc(h, {L.Q2.ext[2], o.vl.v2.ext[2]});
  Ten Cr = alloc(h, {o.vr.v2.ext[2], R.Q2.ext[2]});
  contract(h, op({&L.Q2}, "abq"), op({&o.vl.v2}, "abl"), out({&Cl}, "ql"));
  contract(h, op({&o.vr.v2}, "abr"), op({&R.Q2}, "abq"), out({&Cr}, "rq"));
  //     M(q,k,b,q') = sum_{l,r} C'(q,l) T'(l,k,b,r) C''(r,q')
  Ten M1 = alloc(h, {Cl.ext[0], D, D, Tp.ext[3]});
  contract(h, op({&Cl}, "ql"), op({&Tp}, "lkbr"), out({&M1}, "qkbr"));
  o.M = alloc(h, {Cl.ext[0], D, D, Cr.ext[1]});
  contract(h, op({&M1}, "qkbr"), op({&Cr}, "rz"), out({&o.M}, "qkbz"));
  return o;
}

RenvOut reduced_env(Handle& h, const RenvIn& in, int chi_pp) {
  SideOut L = side_ts(h, in, true, chi_pp);
  SideOut R = side_ts(h, in, false, chi_pp);
  return renv_finish(h, in, L, R);
}

// Run tasks concurrently, one host thread each (sequentially in the sizing pass).
void run_parallel(Handle& h, std::vector<std::function<void()>>& tasks) {
  if (h.dry || tasks.size() == 1) {
    for (auto& t : tasks) t();
    return;
  }
  std::vector<std::exception_ptr> errs(tasks.size());
  std::vector<std::thread> th;
  for (size_t i = 0; i < tasks.size(); ++i)
    th.emplace_back([&, i]() {
      try {
        CTM_CUDA(cudaSetDevice(h.device));   // a new host thread starts on device 0
        tasks[i]();
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void sub_begin(Handle& s) {
  s.ms_svd = 0.0;
  s.flops = 0.0;
  s.min_gap = std::numeric_limits<double>::infinity();
  s.n_svd = 0;
  s.n_svd_fallback = 0;
  s.n_warm = s.n_warm_hit = s.n_warm_retry = 0;
  s.warm_slot = -1;
  s.ms_jacobi = 0.0;
  s.jacobi_flops = 0.0;
  s.jacobi_cta_ms = 0.0;
  s.n_jacobi = 0;
  s.n_kernels = 0;
  s.dry = false;
}
void sub_merge(Handle& h, Handle& s) {
  h.ms_svd += s.ms_svd;
  h.flops += s.flops;
  h.min_gap = std::min(h.min_gap, s.min_gap);
  h.n_svd += s.n_svd;
  h.n_svd_fallback += s.n_svd_fallback;
  h.n_warm += s.n_warm;
  h.n_warm_hit += s.n_warm_hit;
  h.n_warm_retry += s.n_warm_retry;
  h.ms_jacobi += s.ms_jacobi;
  h.jacobi_flops += s.jacobi_flops;
  h.jacobi_cta_ms += s.jacobi_cta_ms;
  h.n_jacobi += s.n_jacobi;
  h.n_kernels += s.n_kernels;
  if (s.prof_used && !h.dry) {   // CTM_FLAG_PROFILE: the workers' tc_gemm launches (blocks the host)
    CTM_CUDA(cudaEventSynchronize(s.prof_ev[2 * s.prof_used - 1]));
    for (int i = 0; i < s.prof_used; ++i) {
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, s.prof_ev[2 * i], s.prof_ev[2 * i + 1]));
      h.prof_ms_subs += ms;
      h.prof_flops_subs += s.prof_flops[i];
    }
    h.prof_n_subs += s.prof_used;
  }
  s.prof_used = 0;
  h.kernel_count += s.n_kernels;
}

// Isometry stage of one column absorption (rows a1-a5) on the worker sub-handles:
// phase A: the four side TS (x in {a,b}) x (left, right) concurrently;
// phase B: for each cut type the reduced env M_xy and the main TS(M; chi', chi).
// Right-side TS results of a left move.  A left move rewrites only C^1, T^1, C^4, so the
// right-side products Q_r = C_x^2 T_x^3 -- and their isometries -- are identical in its two
// column absorptions: the second absorption reuses the first one's (exact, not an
// approximation).  Buffers live in the main arena for the duration of the move.
struct SideCache {
  bool valid = false;
  SideOut side[2];   // x = a, b: right-side TS (v1, v2, Q2)
};

// Reserve the cache buffers in the caller's (left move's) part of the main arena.
void reserve_side_cache(Handle& h, const ctm_env* env, SideCache& c) {
  const ctm_params& p = h.prm;
  const int D = p.D;
  for (int x = 0; x < 2; ++x) {
    const int P = envC(env, x, 2).ext[0], F = envT(env, x, 3, D).ext[3];
    const int n1 = std::min(p.chi_pp, P * D), n2 = std::min(p.chi_pp, n1 * D);
    c.side[x].v.v1 = alloc(h, {P, D, n1});
    c.side[x].v.v2 = alloc(h, {n1, D, n2});
    c.side[x].Q2 = alloc(h, {n1, D, F});
  }
}

// On a worker error every sub-stream is drained before the exception leaves: the other
// chain may still have work in flight (the side-cache copy into the main arena included),
// and the caller's next call reuses the arena on h.stream with no ordering against them.
void drain_subs(Handle& h) {
  for (auto& s : h.subs) cudaStreamSynchronize(s->stream);
}

void isometry_stage(Handle& h, const ctm_env* env, const Site st[2], Iso V[2][2], int absorption,
                    SideCache* cache = nullptr) {
  const ctm_params& p = h.prm;
  const int D = p.D;
  for (auto& s : h.subs) {
    sub_begin(*s);
    s->dry = h.dry;
    s->ws.reset(0);
  }
  if (!h.dry) {
    CTM_CUDA(cudaEventRecord(h.ev[4], h.stream));   // fork point
    for (auto& s : h.subs) CTM_CUDA(cudaStreamWaitEvent(s->stream, h.ev[4], 0));
  }
  RenvIn ri[2];
  for (int x = 0; x < 2; ++x)
    ri[x] = RenvIn{envC(env, x, 1), envT(env, x, 2, D), envC(env, x, 2), envT(env, x, 1, D), envT(env, x, 3, D), &st[x]};
  SideOut side[4];
  const bool reuse = cache != nullptr && cache->valid;
  // CTM_FLAG_WARM_START: the solve sites of this (direction, absorption)
  const int warm_base = (h.warm_dir * 2 + absorption) * CTM_WARM_SITES;
  // Two independent chains, one per cut type x: [left side TS on sub 2x || right side TS on
  // sub 2x+1] -> reduced env M_x + main TS on sub 2x.  Each chain waits only for its own
  // right-side task (host future + stream event), not for the other chain's side tasks.
  std::promise<void> right_done[2];
  std::shared_future<void> right_fut[2] = {right_done[0].get_future().share(), right_done[1].get_future().share()};
  auto right_task = [&](int x) {   // sub 2x+1: right side TS (+ its copy into the move's cache)
    try {
      Handle& sub = *h.subs[2 * x + 1];
      if (h.warm) sub.warm_slot = warm_base + 3 * x + 1;
      side[2 * x + 1] = side_ts(sub, ri[x], false, p.chi_pp);
      if (cache != nullptr) {
        const SideOut& o = side[2 * x + 1];
        cache->side[x].v.gap1 = o.v.gap1;
        Ten* dst[3] = {&cache->side[x].v.v1, &cache->side[x].v.v2, &cache->side[x].Q2};
        const Ten* src[3] = {&o.v.v1, &o.v.v2, &o.Q2};
        for (int t = 0; t < 3; ++t) {
          if (dst[t]->size() != src[t]->size()) throw Error(CTM_E_ARG, "side cache: shape mismatch");
          dst[t]->ext = src[t]->ext;
          if (!h.dry)
            CTM_CUDA(cudaMemcpyAsync(dst[t]->p, src[t]->p, src[t]->size() * 8, cudaMemcpyDeviceToDevice, sub.stream));
        }
      }
      right_done[x].set_value();
    } catch (...) {
      right_done[x].set_exception(std::current_exception());
      throw;
    }
  };
  auto chain_task = [&](int x) {   // sub 2x: left side TS, then (after x's right side) a5
    Handle& s = *h.subs[2 * x];
    if (h.warm) s.warm_slot = warm_base + 3 * x;
    side[2 * x] = side_ts(s, ri[x], true, p.chi_pp);
    if (reuse) side[2 * x + 1] = cache->side[x];
    else right_fut[x].get();   // host: the right-side task has enqueued everything
    Handle& r = *h.subs[2 * x + 1];
    if (!h.dry) {   // device: sub 2x waits for sub 2x+1's stream (its outputs / the cached copy)
      CTM_CUDA(cudaEventRecord(r.ev[0], r.stream));
      CTM_CUDA(cudaStreamWaitEvent(s.stream, r.ev[0], 0));
    }
    RenvOut ro = renv_finish(s, ri[x], side[2 * x], side[2 * x + 1]);
    static const bool main_svd2 = std::getenv("CTM_TS_MAIN_SVD") != nullptr;   // A/B: SVD stage two
    if (h.warm) s.warm_slot = warm_base + 3 * x + 2;
    V[x][1 - x] = ts_isometry(s, ro.M, p.chi_p, p.chi, nullptr, !main_svd2);   // a5 (basis stage two: R24b)
  };
  std::vector<std::function<void()>> T;
  for (int x = 0; x < 2; ++x) {
    T.push_back([&, x]() { chain_task(x); });
    if (!reuse) T.push_back([&, x]() { right_task(x); });
  }
  if (h.dry) {   // sizing pass: sequential, right sides first (no waiting on futures)
    if (!reuse)
      for (int x = 0; x < 2; ++x) right_task(x);
    for (int x = 0; x < 2; ++x) chain_task(x);
  } else {
    try {
      run_parallel(h, T);
    } catch (...) {
      drain_subs(h);
      throw;
    }
  }
  if (cache != nullptr) cache->valid = true;
  if (!h.dry) {   // per-cut gaps: main TS [ab, ba], side TS [a-l, a-r, b-l, b-r]
    for (int c = 0; c < 2; ++c) {
      const Iso& v = c == 0 ? V[0][1] : V[1][0];
      h.cut_gap[absorption][c] = std::min(h.cut_gap[absorption][c], v.gap1);
    }
    for (int i = 0; i < 4; ++i)
      h.side_gap[absorption][i] = std::min(h.side_gap[absorption][i], side[i].v.gap1);
  }
  for (auto& s : h.subs) {
    if (!h.dry) {
      CTM_CUDA(cudaEventRecord(s->ev[1], s->stream));   // join
      CTM_CUDA(cudaStreamWaitEvent(h.stream, s->ev[1], 0));
    }
    sub_merge(h, *s);
  }
  if (!h.dry) {
    CTM_CUDA(cudaEventRecord(h.ev[5], h.stream));
    CTM_CUDA(cudaEventSynchronize(h.ev[5]));
    float ms = 0.f;
    CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[4], h.ev[5]));
    h.ms_iso += ms;
  }
}

// ---------------------------------------------------------------------------------------
// Row a9: corner growth (Fig 4(b)).
// ---------------------------------------------------------------------------------------
// Batched over jobs with identical shapes (the two windows of an absorption).
struct CornerJob {
  Ten C, T;            // top-left: C^1 (d,r), T^2 (l,k,b,r); bottom-left: C^4 (r,u), T^4 (r,k,b,l)
  const Iso* v;        // projector of the cut the corner row sits on
  Ten* res;
  double* ss;
};

int corner_batch(Handle& h, const std::vector<CornerJob>& jobs, bool top) {
  const int B = (int)jobs.size();
  const CornerJob& j0 = jobs[0];
  const int D = j0.T.ext[1];
  const size_t mark = h.ws.top;
  std::vector<Ten> Y1(B), Y2(B);
  for (int b = 0; b < B; ++b) {
    Y1[b] = alloc(h, {top ? j0.C.ext[1] : j0.C.ext[0], D, j0.v->v1.ext[2]});
    Y2[b] = alloc(h, {j0.v->v1.ext[2], D, top ? j0.T.ext[3] : j0.T.ext[0]});
  }
  std::vector<const Ten*> c, t, v1, v2, y1c, y2c;
  std::vector<Ten*> y1, y2, res;
  std::vector<double*> ss;
  for (int b = 0; b < B; ++b) {
    c.push_back(&jobs[b].C);
    t.push_back(&jobs[b].T);
    v1.push_back(&jobs[b].v->v1);
    v2.push_back(&jobs[b].v->v2);
    y1.push_back(&Y1[b]);
    y2.push_back(&Y2[b]);
    y1c.push_back(&Y1[b]);
    y2c.push_back(&Y2[b]);
    res.push_back(jobs[b].res);
    ss.push_back(jobs[b].ss);
  }
  // Y1(p,k,a) = sum_x C(x,p) v1(x,k,a)  [top: C^1 (d=x, r=p); bottom: C^4 (r=p, u=x)]
  contract(h, op(c, top ? "xp" : "px"), op(v1, "xka"), out(y1, "pka"));
  // Y2(a,b,r) = sum_{p,k} Y1(p,k,a) T(p,k,b,r)  [top: T^2 (l=p,k,b,r); bottom: T^4 (r,k,b,l=p)]
  contract(h, op(y1c, "pka"), op(t, top ? "pkbr" : "rkbp"), out(y2, "abr"));
  // C'(o,r) / C'(r,o) = sum_{a,b} Y2(a,b,r) v2(a,b,o)
  int np = contract(h, op(y2c, "abr"), op(v2, "abo"), out(res, top ? "or" : "ro", ss));
  h.ws.reset(mark);
  return np;
}

std::vector<int> corners(Handle& h, const std::vector<CornerJob>& jobs, bool top) {
  if (jobs.size() == 2 && jobs[0].C.ext == jobs[1].C.ext && jobs[0].T.ext == jobs[1].T.ext &&
      jobs[0].v->v1.ext == jobs[1].v->v1.ext && jobs[0].v->v2.ext == jobs[1].v->v2.ext) {
    int np = corner_batch(h, jobs, top);
    return {np, np};
  }
  std::vector<int> r;
  for (auto& j : jobs) r.push_back(corner_batch(h, {j}, top));
  return r;
}

// ---------------------------------------------------------------------------------------
// REDUCED strategy (Fig 3(a,b)): the exact reduced
// environment M, the one-shot 4-leg isometry V = first chi left singular vectors of M as
// (chi D^2) x chi ("chi D^2 x chi in FIG 3(b)"), and the absorption with V on both
// cuts -- O(chi^3 D^4) where the sequential order is O(chi^3 D^3).  Same contraction order
// as the oracle (oracle/ctm_oracle.py reduced_env_exact, absorb_one_shot, *_one_shot).
// ---------------------------------------------------------------------------------------
// M(q,kd,bd,q') = sum C1 T2 C2 T1 X X* T3 (the right half replaced by {C^2, T^3}); X is the
// site in the picture orientation (s,u,l,d,r).  M is allocated first (it outlives the
// intermediates, which reuse two buffers).
Ten reduced_env_exact(Handle& h, const RenvIn& in, const double* Xraw, const double* Xbraw) {
  const int d = h.prm.d, D = in.T1.ext[1];
  const int cx = in.C1.ext[0], cz = in.T2.ext[3], cy = in.C2.ext[1], cq = in.T1.ext[0], cw = in.T3.ext[3];
  Ten X{const_cast<double*>(Xraw), {d, D, D, D, D}};
  Ten Xb{const_cast<double*>(Xbraw), {d, D, D, D, D}};
  Ten M = alloc(h, {cq, D, D, cw});
  const size_t mark = h.ws.top;
  Ten R1 = alloc(h, {cx, D, D, cz});
  Ten R2 = alloc(h, {cx, D, D, cy});
  double* bufA = h.ws.take((size_t)D * D * cy * cq * D * D);       // R3 (kbyqlm), later R5 (yqdrew)
  double* bufB = h.ws.take((size_t)D * cy * D * cq * d * D * D);   // R4 (bymqsdr)
  Ten R3{bufA, {D, D, cy, cq, D, D}};
  Ten R4{bufB, {D, cy, D, cq, d, D, D}};
  Ten R5{bufA, {cy, cq, D, D, D, D}};
  contract(h, op({&in.C1}, "xp"), op({&in.T2}, "pkbz"), out({&R1}, "xkbz"));     // C1 (d=x, r=p), T2 (l=p,ku,bu,r=z)
  contract(h, op({&R1}, "xkbz"), op({&in.C2}, "zy"), out({&R2}, "xkby"));        // C2 (l=z, d=y)
  contract(h, op({&R2}, "xkby"), op({&in.T1}, "qlmx"), out({&R3}, "kbyqlm"));    // T1 (d=q, kl, bl, u=x)
  contract(h, op({&R3}, "kbyqlm"), op({&X}, "skldr"), out({&R4}, "bymqsdr"));    // X over ku, kl
  contract(h, op({&R4}, "bymqsdr"), op({&Xb}, "sbmew"), out({&R5}, "yqdrew"));   // X* over s, bu, bl
  contract(h, op({&R5}, "yqdrew"), op({&in.T3}, "yrwz"), out({&M}, "qdez"));     // T3 (u=y, kr, br, d=z)
  h.ws.reset(mark);
  return M;
}

// STANDARD ("8 individual tensors", Fig 2(c)): upper half of the 2x2 patch
//        C_x^1  T_x^2  T_y^2  C_y^2
//        T_x^1    X      Y    T_y^3
// open at the bottom: M_std(q, kX, bX, kY, bY, q').  Oracle order (half_network_standard).
Ten half_network_standard(Handle& h, const Ten& C1x, const Ten& T2x, const Ten& T2y, const Ten& C2y, const Ten& T1x,
                          const double* Xr, const double* Yr, const Ten& T3y) {
  const int d = h.prm.d, D = T1x.ext[1];
  Ten X{const_cast<double*>(Xr), {d, D, D, D, D}};
  Ten Y{const_cast<double*>(Yr), {d, D, D, D, D}};
  const int cP = T1x.ext[0], cf = C1x.ext[1], ci = T2x.ext[3], cl = T2y.ext[3], cm = C2y.ext[1], cQ = T3y.ext[3];
  Ten M = alloc(h, {cP, D, D, D, D, cQ});
  const size_t mark = h.ws.top;
  // left half: C1x(d=e, r=f) T1x(d=P, kl=p, bl=q, u=e) T2x(l=f, ku=g, bu=h, r=i) X(s,u=g,l=p,d=K,r=r) X*(s,u=h,l=q,d=B,r=w)
  Ten L1 = alloc(h, {cf, cP, D, D});
  Ten L2 = alloc(h, {cP, D, D, D, D, ci});
  Ten L3 = alloc(h, {cP, D, D, ci, d, D, D});
  Ten L4 = alloc(h, {cP, ci, D, D, D, D});
  contract(h, op({&C1x}, "ef"), op({&T1x}, "Ppqe"), out({&L1}, "fPpq"));
  contract(h, op({&L1}, "fPpq"), op({&T2x}, "fghi"), out({&L2}, "Ppqghi"));
  contract(h, op({&L2}, "Ppqghi"), op({&X}, "sgpKr"), out({&L3}, "PqhisKr"));
  contract(h, op({&L3}, "PqhisKr"), op({&X}, "shqBw"), out({&L4}, "PiKrBw"));
  // right half: T2y(l=i, ku=j, bu=k, r=l) C2y(l=l, d=m) T3y(u=m, kr=n, br=o, d=Q) Y(s,u=j,l=r,d=L,r=n) Y*(s,u=k,l=w,d=E,r=o)
  Ten R1 = alloc(h, {ci, D, D, cm});
  Ten R2 = alloc(h, {ci, D, D, D, D, cQ});
  Ten R3 = alloc(h, {ci, D, D, cQ, d, D, D});
  Ten R4 = alloc(h, {ci, cQ, D, D, D, D});
  contract(h, op({&T2y}, "ijkl"), op({&C2y}, "lm"), out({&R1}, "ijkm"));
  contract(h, op({&R1}, "ijkm"), op({&T3y}, "mnoQ"), out({&R2}, "ijknoQ"));
  contract(h, op({&R2}, "ijknoQ"), op({&Y}, "sjrLn"), out({&R3}, "ikoQsrL"));
  contract(h, op({&R3}, "ikoQsrL"), op({&Y}, "skwEo"), out({&R4}, "iQrLwE"));
  contract(h, op({&L4}, "PiKrBw"), op({&R4}, "iQrLwE"), out({&M}, "PKBLEQ"));
  (void)cl;
  h.ws.reset(mark);
  return M;
}

// V(p,k,b,n): first n = min(chi, rows) left singular vectors of M as (p k b) x (rest).
Ten one_shot_isometry(Handle& h, const Ten& M, int chi) {
  const int P = M.ext[0], K = M.ext[1], B = M.ext[2];
  int F = 1;
  for (size_t i = 3; i < M.ext.size(); ++i) F *= M.ext[i];
  const int n = std::min(chi, P * K * B);
  Ten V = alloc(h, {P, K, B, n});
  svd_left(h, M.p, P * K * B, F, n, V.p);
  return V;
}

// T'(o1,kz,bz,o2) = sum V_in(p,ki,bi,o1) T(p,kf,bf,q) X(s,ki,kf,ko,kz) X*(s,bi,bf,bo,bz) V_out(q,ko,bo,o2)
int absorb_one_shot(Handle& h, const Ten& T, const Site& X, const Ten& Vin, const Ten& Vout, Ten& res, double* ss) {
  const int D = T.ext[1], d = X.bra.ext[0];
  const int o1 = Vin.ext[3], q = T.ext[3];
  const size_t mark = h.ws.top;
  Ten Y1 = alloc(h, {D, D, o1, D, D, q});        // jkofgq
  Ten Y2 = alloc(h, {D, o1, D, q, d, D, D});     // kogqsaz
  Ten Y3{Y1.p, {o1, q, D, D, D, D}};             // oqazbw (reuses Y1: dead after Y2)
  contract(h, op({&Vin}, "pjko"), op({&T}, "pfgq"), out({&Y1}, "jkofgq"));
  contract(h, op({&Y1}, "jkofgq"), op({&X.ket}, "jfsaz"), out({&Y2}, "kogqsaz"));   // ket (in,face,s,out,far)
  contract(h, op({&Y2}, "kogqsaz"), op({&X.bra}, "sgkbw"), out({&Y3}, "oqazbw"));   // bra (s,face,in,out,far)
  std::vector<double*> sv;
  if (ss) sv.push_back(ss);
  int np = contract(h, op({&Y3}, "oqazbw"), op({&Vout}, "qabd"), out({&res}, "ozwd", sv));
  h.ws.reset(mark);
  return np;
}

// C^1'(o,r) = sum C1(x,p) T2(p,k,b,r) V(x,k,b,o);  C^4'(r,o) = sum C4(p,x) T4(r,k,b,p) V(x,k,b,o)
int corner_one_shot(Handle& h, const Ten& C, const Ten& T, const Ten& V, Ten& res, double* ss, bool top) {
  const int D = T.ext[1];
  const size_t mark = h.ws.top;
  Ten Y = alloc(h, {top ? C.ext[0] : C.ext[1], D, D, top ? T.ext[3] : T.ext[0]});   // xkbr
  contract(h, op({&C}, top ? "xp" : "px"), op({&T}, top ? "pkbr" : "rkbp"), out({&Y}, "xkbr"));
  std::vector<double*> sv;
  if (ss) sv.push_back(ss);
  int np = contract(h, op({&Y}, "xkbr"), op({&V}, "xkbo"), out({&res}, top ? "or" : "ro", sv));
  h.ws.reset(mark);
  return np;
}

void check_env(const ctm_env* e, const ctm_params& p) {
  for (int x = 0; x < 2; ++x)
    for (int j = 0; j < 8; ++j) {
      if ((j < 4 ? e->C[x][j] : e->T[x][j - 4]) == nullptr) throw Error(CTM_E_ARG, "env: null tensor pointer");
      for (int q = 0; q < 2; ++q)
        if (e->ext[x][j][q] < 1 || e->ext[x][j][q] > p.chi)
          throw Error(CTM_E_ARG, "env: boundary extent out of [1, chi]");
    }
}

// Normalise (Frobenius, reading R13) and commit the six new tensors of an absorption.
void commit_six(Handle& h, ctm_env* env, Ten nT[2], Ten nC1[2], Ten nC4[2], const double* ss,
                const std::vector<int>& nparts, int absorption) {
  const ctm_params& p = h.prm;
  if (!h.dry) {
    std::vector<const double*> src;
    std::vector<double*> dst;
    std::vector<size_t> n;
    for (int y = 0; y < 2; ++y) {
      src.push_back(nT[y].p);
      dst.push_back(env->T[y][0]);
      n.push_back(nT[y].size());
    }
    for (int y = 0; y < 2; ++y) {
      src.push_back(nC1[y].p);
      dst.push_back(env->C[y][0]);
      n.push_back(nC1[y].size());
    }
    for (int x = 0; x < 2; ++x) {
      src.push_back(nC4[x].p);
      dst.push_back(env->C[x][3]);
      n.push_back(nC4[x].size());
    }
    const bool prof = (p.flags & CTM_FLAG_PROFILE) != 0;
    if (prof) CTM_CUDA(cudaEventRecord(h.ev[6], h.stream));
    scale_commit(h, src, dst, n, ss, nparts);
    if (prof) {   // K7 (HBM-bound): one launch reads the six new tensors and writes them to the env
      CTM_CUDA(cudaEventRecord(h.ev[7], h.stream));
      CTM_CUDA(cudaEventSynchronize(h.ev[7]));
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[6], h.ev[7]));
      h.ms_commit += ms;
      size_t tot = 0;
      for (size_t v : n) tot += v;
      h.commit_bytes += 2.0 * 8.0 * (double)tot;
      ++h.n_commit;
    }
    if (p.flags & CTM_FLAG_CHECK_FINITE) {
      int* cnt = reinterpret_cast<int*>(h.dev_scalars);
      CTM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), h.stream));
      for (size_t i = 0; i < dst.size(); ++i) nonfinite_count(h, dst[i], n[i], cnt);
      int hc = 0;
      CTM_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(int), cudaMemcpyDeviceToHost, h.stream));
      CTM_CUDA(cudaStreamSynchronize(h.stream));
      if (hc) throw Error(CTM_E_NONFINITE, "non-finite entries after column absorption " + std::to_string(absorption));
    }
  }
  for (int y = 0; y < 2; ++y) {
    env->ext[y][4][0] = nT[y].ext[0];
    env->ext[y][4][1] = nT[y].ext[3];
    env->ext[y][0][0] = nC1[y].ext[0];
    env->ext[y][0][1] = nC1[y].ext[1];
  }
  for (int x = 0; x < 2; ++x) {
    env->ext[x][3][0] = nC4[x].ext[0];
    env->ext[x][3][1] = nC4[x].ext[1];
  }
}

// ---------------------------------------------------------------------------------------
// Row a10: one column absorption, both row-parity windows from one snapshot.
//   C_y^1 <- N[C_x^1 T_x^2 V_yx] ; T_y^1 <- N[V_xy T_x^1 X X* V_yx] ; C_x^4 <- N[V_yx C_y^4 T_y^4]
// ---------------------------------------------------------------------------------------
void column_absorption(Handle& h, const Site sl[2], const Site st[2], ctm_env* env, const double* iso_in,
                       double* iso_out, int absorption, SideCache* cache = nullptr) {
  const ctm_params& p = h.prm;
  const int D = p.D;
  const size_t mark = h.ws.top;
  Iso V[2][2];   // V[x][y] = projector of cut 'xy' (x above)
  if (iso_in) {
    const size_t n1 = (size_t)p.chi * D * p.chi_p, n2 = (size_t)p.chi_p * D * p.chi;
    for (int c = 0; c < 2; ++c) {   // c = 0: ab, 1: ba
      const double* base = iso_in + (size_t)(absorption * 2 + c) * (n1 + n2);
      Iso& v = c == 0 ? V[0][1] : V[1][0];
      v.v1 = Ten{const_cast<double*>(base), {p.chi, D, p.chi_p}};
      v.v2 = Ten{const_cast<double*>(base + n1), {p.chi_p, D, p.chi}};
    }
  } else {
    isometry_stage(h, env, st, V, absorption, cache);
  }
  if (iso_out) {
    const size_t n1 = (size_t)p.chi * D * p.chi_p, n2 = (size_t)p.chi_p * D * p.chi;
    for (int c = 0; c < 2; ++c) {
      Iso& v = c == 0 ? V[0][1] : V[1][0];
      if (v.v1.size() != n1 || v.v2.size() != n2) throw Error(CTM_E_ARG, "iso_out needs square extents chi");
      double* base = iso_out + (size_t)(absorption * 2 + c) * (n1 + n2);
      if (!h.dry) {
        CTM_CUDA(cudaMemcpyAsync(base, v.v1.p, n1 * 8, cudaMemcpyDeviceToDevice, h.stream));
        CTM_CUDA(cudaMemcpyAsync(base + n1, v.v2.p, n2 * 8, cudaMemcpyDeviceToDevice, h.stream));
      }
    }
  }
  // new tensors (snapshot semantics: written to workspace, committed at the end)
  double* ss = h.ws.take(6 * (size_t)CTM_SS_SLOTS);   // per-tile sum-of-squares partials
  Ten nT[2], nC1[2], nC4[2];
  std::vector<ChainJob> jobs;
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    Iso& vxy = V[x][y];
    Iso& vyx = V[y][x];
    nT[y] = alloc(h, {vxy.v2.ext[2], D, D, vyx.v2.ext[2]});
    nC1[y] = alloc(h, {vyx.v2.ext[2], envT(env, x, 2, D).ext[3]});
    nC4[x] = alloc(h, {envT(env, y, 4, D).ext[0], vyx.v2.ext[2]});
  }
  Ten T1[2] = {envT(env, 0, 1, D), envT(env, 1, 1, D)};
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    jobs.push_back(ChainJob{&T1[x], &sl[x], &V[x][y], &V[y][x], &nT[y], ss + (size_t)y * CTM_SS_SLOTS});
  }
  std::vector<int> np_t = chains(h, jobs);   // jobs[x] produces nT[y]
  std::vector<CornerJob> tl, bl;
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    tl.push_back(CornerJob{envC(env, x, 1), envT(env, x, 2, D), &V[y][x], &nC1[y], ss + (size_t)(2 + y) * CTM_SS_SLOTS});
    bl.push_back(CornerJob{envC(env, y, 4), envT(env, y, 4, D), &V[y][x], &nC4[x], ss + (size_t)(4 + x) * CTM_SS_SLOTS});
  }
  std::vector<int> np_tl = corners(h, tl, true);   // tl[x] -> nC1[y]
  std::vector<int> np_bl = corners(h, bl, false);  // bl[x] -> nC4[x]
  std::vector<int> nparts = {np_t[1], np_t[0], np_tl[1], np_tl[0], np_bl[0], np_bl[1]};
  commit_six(h, env, nT, nC1, nC4, ss, nparts, absorption);   // K7 (reading R13)
  h.ws.reset(mark);
}

// REDUCED column absorption (P:L43 with P:L53's projectors): the two cut types' exact
// reduced environments and one-shot isometries run concurrently on worker sub-handles 0/1.
void column_absorption_reduced(Handle& h, const Site sl[2], const double* raw[2], ctm_env* env, int absorption) {
  const ctm_params& p = h.prm;
  const int D = p.D;
  const size_t mark = h.ws.top;
  Ten V[2][2];   // V[x][y]: cut 'xy' (x above)
  for (auto& sub : h.subs) {
    sub_begin(*sub);
    sub->dry = h.dry;
    sub->ws.reset(0);
  }
  if (!h.dry) {
    CTM_CUDA(cudaEventRecord(h.ev[4], h.stream));
    for (int i = 0; i < 2; ++i) CTM_CUDA(cudaStreamWaitEvent(h.subs[i]->stream, h.ev[4], 0));
  }
  std::vector<std::function<void()>> tasks;
  for (int x = 0; x < 2; ++x)
    tasks.push_back([&, x]() {
      Handle& s = *h.subs[x];
      const int y = 1 - x;
      Ten M;
      if (p.strategy == CTM_STANDARD) {
        M = half_network_standard(s, envC(env, x, 1), envT(env, x, 2, D), envT(env, y, 2, D), envC(env, y, 2),
                                  envT(env, x, 1, D), raw[x], raw[y], envT(env, y, 3, D));
      } else {
        RenvIn ri{envC(env, x, 1), envT(env, x, 2, D), envC(env, x, 2), envT(env, x, 1, D), envT(env, x, 3, D), nullptr};
        M = reduced_env_exact(s, ri, raw[x], raw[x]);
      }
      V[x][y] = one_shot_isometry(s, M, p.chi);
    });
  try {
    run_parallel(h, tasks);
  } catch (...) {
    drain_subs(h);
    throw;
  }
  for (int i = 0; i < 2; ++i) {
    Handle& s = *h.subs[i];
    if (!h.dry) {
      CTM_CUDA(cudaEventRecord(s.ev[1], s.stream));
      CTM_CUDA(cudaStreamWaitEvent(h.stream, s.ev[1], 0));
    }
    sub_merge(h, s);
  }
  if (!h.dry) {
    CTM_CUDA(cudaEventRecord(h.ev[5], h.stream));
    CTM_CUDA(cudaEventSynchronize(h.ev[5]));
    float ms = 0.f;
    CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[4], h.ev[5]));
    h.ms_iso += ms;
  }
  double* ss = h.ws.take(6 * (size_t)CTM_SS_SLOTS);
  Ten nT[2], nC1[2], nC4[2];
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    nT[y] = alloc(h, {V[x][y].ext[3], D, D, V[y][x].ext[3]});
    nC1[y] = alloc(h, {V[y][x].ext[3], envT(env, x, 2, D).ext[3]});
    nC4[x] = alloc(h, {envT(env, y, 4, D).ext[0], V[y][x].ext[3]});
  }
  std::vector<int> np(6);
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    np[y] = absorb_one_shot(h, envT(env, x, 1, D), sl[x], V[x][y], V[y][x], nT[y], ss + (size_t)y * CTM_SS_SLOTS);
    np[2 + y] = corner_one_shot(h, envC(env, x, 1), envT(env, x, 2, D), V[y][x], nC1[y],
                                ss + (size_t)(2 + y) * CTM_SS_SLOTS, true);
    np[4 + x] = corner_one_shot(h, envC(env, y, 4), envT(env, y, 4, D), V[y][x], nC4[x],
                                ss + (size_t)(4 + x) * CTM_SS_SLOTS, false);
  }
  commit_six(h, env, nT, nC1, nC4, ss, np, absorption);
  h.ws.reset(mark);
}

void left_move(Handle& h, const double* A, const double* B, ctm_env* env, const double* iso_in, double* iso_out) {
  const ctm_params& p = h.prm;
  const size_t mark = h.ws.top;
  Site sl[2] = {site_left(h, A, p.d, p.D), site_left(h, B, p.d, p.D)};
  if (p.strategy == CTM_REDUCED_EXACT || p.strategy == CTM_STANDARD) {
    if (iso_in || iso_out) throw Error(CTM_E_UNSUPPORTED, "iso_in / iso_out are defined for CTM_SEQUENTIAL only");
    const double* raw[2] = {A, B};
    column_absorption_reduced(h, sl, raw, env, 0);
    column_absorption_reduced(h, sl, raw, env, 1);
    h.ws.reset(mark);
    return;
  }
  Site st[2];
  if (!iso_in) {
    st[0] = site_top(h, A, p.d, p.D);
    st[1] = site_top(h, B, p.d, p.D);
  }
  SideCache cache;   // right-side TS shared by the two absorptions (see SideCache)
  if (!iso_in) reserve_side_cache(h, env, cache);
  column_absorption(h, sl, st, env, iso_in, iso_out, 0, iso_in ? nullptr : &cache);
  column_absorption(h, sl, st, env, iso_in, iso_out, 1, iso_in ? nullptr : &cache);
  h.ws.reset(mark);
}

void move_dir(Handle& h, int dir, const double* A, const double* B, ctm_env* env, double* iso_out = nullptr) {
  static const int turns_for[4] = {0, 2, 3, 1};   // LEFT, RIGHT, UP, DOWN: cw turns bringing it left
  const int n = turns_for[dir];
  if (n == 0) {
    left_move(h, A, B, env, nullptr, iso_out);
    return;
  }
  const size_t mark = h.ws.top;
  const size_t ns = (size_t)h.prm.d * h.prm.D * h.prm.D * h.prm.D * h.prm.D;
  double* Ar = h.ws.take(ns);
  double* Br = h.ws.take(ns);
  if (!h.dry) {
    rotate_site(h, A, Ar, n);
    rotate_site(h, B, Br, n);
  }
  for (int i = 0; i < n; ++i) rotate_env_cw(env);
  h.warm_dir = dir;   // the warm-start sites of this direction
  try {
    left_move(h, Ar, Br, env, nullptr, iso_out);
  } catch (...) {
    h.warm_dir = 0;
    for (int i = 0; i < (4 - n) % 4; ++i) rotate_env_cw(env);
    throw;
  }
  h.warm_dir = 0;
  for (int i = 0; i < (4 - n) % 4; ++i) rotate_env_cw(env);
  h.ws.reset(mark);
}

// ---------------------------------------------------------------------------------------
// Imaginary-time evolution (readings R25-R30): one FFU bond
// update of any of the four bonds of the unit cell, by the same relabelling as the moves.
//   H1: A left of B;  H2: B left of A (sublattice labels exchanged, reading R2);
//   V1: A above B;    V2: B above A (picture turned counter-clockwise, sites turned back).
// ---------------------------------------------------------------------------------------
void swap_sublattices(ctm_env* e) {
  std::swap(e->C[0], e->C[1]);
  std::swap(e->T[0], e->T[1]);
  std::swap(e->ext[0], e->ext[1]);
}

void ffu_update(Handle& h, const double* A, const double* B, const ctm_env* env, const double* gate, int bond,
                int sweeps, double* A2, double* B2, double* cost) {
  const size_t mark = h.ws.top;
  ctm_env e = *env;
  if (bond == CTM_BOND_H1) {
    ffu_bond_update_h(h, A, B, &e, gate, sweeps, A2, B2, cost);
  } else if (bond == CTM_BOND_H2) {
    swap_sublattices(&e);
    ffu_bond_update_h(h, B, A, &e, gate, sweeps, B2, A2, cost);
  } else {
    const size_t ns = (size_t)h.prm.d * h.prm.D * h.prm.D * h.prm.D * h.prm.D;
    double* Ar = h.ws.take(ns);
    double* Br = h.ws.take(ns);
    double* a2 = h.ws.take(ns);
    double* b2 = h.ws.take(ns);
    rotate_site(h, A, Ar, 3);   // counter-clockwise quarter turn (= 3 clockwise)
    rotate_site(h, B, Br, 3);
    for (int i = 0; i < 3; ++i) rotate_env_cw(&e);
    if (bond == CTM_BOND_V1) {
      ffu_bond_update_h(h, Ar, Br, &e, gate, sweeps, a2, b2, cost);
    } else {
      swap_sublattices(&e);
      ffu_bond_update_h(h, Br, Ar, &e, gate, sweeps, b2, a2, cost);
    }
    rotate_site(h, a2, A2, 1);   // back: one clockwise quarter turn
    rotate_site(h, b2, B2, 1);
  }
  h.ws.reset(mark);
}

// ---------------------------------------------------------------------------------------
// Closures (Fig 1(c,d)).  Same pairwise structure as the paper's enlarged corners.
// ---------------------------------------------------------------------------------------
struct Closure {
  Ten Eul, Eur, Elr, Ell;
};

// Enlarged corner E = C . Ta . Tb . X . X*: generic helper on labels.
double norm_2x2_impl(Handle& h, const double* A, const double* B, const ctm_env* env, bool absval) {
  const int D = h.prm.D, d = h.prm.d;
  const size_t mark = h.ws.top;
  auto cp = [&](Ten t) {   // optional |.| copy
    if (!absval) return t;
    Ten r = alloc(h, t.ext);
    abs_copy(h, t.p, r.p, t.size());
    return r;
  };
  Ten sA = cp(Ten{const_cast<double*>(A), {d, D, D, D, D}});
  Ten sB = cp(Ten{const_cast<double*>(B), {d, D, D, D, D}});
  auto C = [&](int x, int k) { return cp(envC(env, x, k)); };
  auto T = [&](int x, int k) { return cp(envT(env, x, k, D)); };
  const int a = 0, b = 1;
  // E_ul: C_a^1(x,y) T_a^2(y,k,b,Y) T_a^1(X,l,m,x) A(s,k,l,d,r) A*(s,b,m,e,q) -> (Y,r,q,X,d,e)
  Ten c1 = C(a, 1), t2 = T(a, 2), t1 = T(a, 1);
  Ten E1 = alloc(h, {c1.ext[0], D, D, t2.ext[3]});
  contract(h, op({&c1}, "xy"), op({&t2}, "ykbY"), out({&E1}, "xkbY"));
  Ten E2 = alloc(h, {D, D, t2.ext[3], t1.ext[0], D, D});
  contract(h, op({&E1}, "xkbY"), op({&t1}, "Xlmx"), out({&E2}, "kbYXlm"));
  Ten E3 = alloc(h, {D, t2.ext[3], t1.ext[0], D, d, D, D});
  contract(h, op({&E2}, "kbYXlm"), op({&sA}, "skldr"), out({&E3}, "bYXmsdr"));
  Ten Eul = alloc(h, {t2.ext[3], D, D, t1.ext[0], D, D});
  contract(h, op({&E3}, "bYXmsdr"), op({&sA}, "sbmeq"), out({&Eul}, "YrqXde"));
  // E_ur: T_b^2(Y,k,b,z) C_b^2(z,w) T_b^3(w,l,m,W) B(s,k,t,d,l) B*(s,b,u,e,m) -> (Y,t,u,W,d,e)
  Ten u2 = T(b, 2), c2 = C(b, 2), u3 = T(b, 3);
  Ten F1 = alloc(h, {u2.ext[0], D, D, c2.ext[1]});
  contract(h, op({&u2}, "Ykbz"), op({&c2}, "zw"), out({&F1}, "Ykbw"));
  Ten F2 = alloc(h, {u2.ext[0], D, D, D, D, u3.ext[3]});
  contract(h, op({&F1}, "Ykbw"), op({&u3}, "wlmW"), out({&F2}, "YkblmW"));
  Ten F3 = alloc(h, {u2.ext[0], D, D, u3.ext[3], d, D, D});
  contract(h, op({&F2}, "YkblmW"), op({&sB}, "sktdl"), out({&F3}, "YbmWstd"));
  Ten Eur = alloc(h, {u2.ext[0], D, D, u3.ext[3], D, D});
  contract(h, op({&F3}, "YbmWstd"), op({&sB}, "sbuem"), out({&Eur}, "YtuWde"));
  // E_lr: T_a^3(W,k,b,v) C_a^3(v,V) T_a^4(V,m,n,U) A(s,u,t,m,k) A*(s,p,q,n,b) -> (W,U,u,t,p,q)
  Ten w3 = T(a, 3), c3 = C(a, 3), w4 = T(a, 4);
  Ten G1 = alloc(h, {w3.ext[0], D, D, c3.ext[1]});
  contract(h, op({&w3}, "Wkbv"), op({&c3}, "vV"), out({&G1}, "WkbV"));
  Ten G2 = alloc(h, {w3.ext[0], D, D, D, D, w4.ext[3]});
  contract(h, op({&G1}, "WkbV"), op({&w4}, "VmnU"), out({&G2}, "WkbmnU"));
  Ten G3 = alloc(h, {w3.ext[0], D, D, w4.ext[3], d, D, D});
  contract(h, op({&G2}, "WkbmnU"), op({&sA}, "sutmk"), out({&G3}, "WbnUsut"));
  Ten Elr = alloc(h, {w3.ext[0], w4.ext[3], D, D, D, D});
  contract(h, op({&G3}, "WbnUsut"), op({&sA}, "spqnb"), out({&Elr}, "WUutpq"));
  // E_ll: T_b^4(U,k,b,Z) C_b^4(Z,z) T_b^1(z,l,m,X) B(s,u,l,k,r) B*(s,p,m,b,q) -> (U,X,u,r,p,q)
  Ten z4 = T(b, 4), c4 = C(b, 4), z1 = T(b, 1);
  Ten H1 = alloc(h, {z4.ext[0], D, D, c4.ext[1]});
  contract(h, op({&z4}, "UkbZ"), op({&c4}, "Zz"), out({&H1}, "Ukbz"));
  Ten H2 = alloc(h, {z4.ext[0], D, D, D, D, z1.ext[3]});
  contract(h, op({&H1}, "Ukbz"), op({&z1}, "zlmX"), out({&H2}, "UkblmX"));
  Ten H3 = alloc(h, {z4.ext[0], D, D, z1.ext[3], d, D, D});
  contract(h, op({&H2}, "UkblmX"), op({&sB}, "sulkr"), out({&H3}, "UbmXsur"));
  Ten Ell = alloc(h, {z4.ext[0], z1.ext[3], D, D, D, D});
  contract(h, op({&H3}, "UbmXsur"), op({&sB}, "spmbq"), out({&Ell}, "UXurpq"));
  // ring
  Ten R1 = alloc(h, {Eul.ext[3], D, D, Eur.ext[3], D, D});
  contract(h, op({&Eul}, "YrqXde"), op({&Eur}, "YrqWfg"), out({&R1}, "XdeWfg"));
  Ten R2 = alloc(h, {Eul.ext[3], D, D, Elr.ext[1], D, D});
  contract(h, op({&R1}, "XdeWfg"), op({&Elr}, "WUfhgi"), out({&R2}, "XdeUhi"));
  // final full contraction: permute E_ll to R2's leg order (X,d,e,U,h,i), then a dot product
  Ten Ellp = alloc(h, {Ell.ext[1], D, D, Ell.ext[0], D, D});
  permute(h, Ell.p, Ell.ext, {1, 2, 4, 0, 3, 5}, Ellp.p);   // (U,X,d,h,e,i) -> (X,d,e,U,h,i)
  Ten res = alloc(h, {1});
  dot(h, R2.p, Ellp.p, R2.size(), res.p);
  double v = 0.0;
  if (!h.dry) {
    CTM_CUDA(cudaMemcpyAsync(&v, res.p, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
    CTM_CUDA(cudaStreamSynchronize(h.stream));
  }
  h.ws.reset(mark);
  return v;
}

// Bond energy on the 2x1 window (A left of B), reading R18:
//   C_a^1 T_a^2 T_b^2 C_b^2 / T_a^1 A B T_b^3 / C_a^4 T_a^4 T_b^4 C_b^3
// rho(sA,sB,tA,tB) = L(Y,U,sA,r,tA,w) R(Y,U,sB,r,tB,w); ket then bra absorbed per half
// (peak intermediate chi^2 d^2 D^4) so it also runs at C4 sizes.
// The 2x1 window's unnormalised rho(sA, sB, tA, tB) (H bond), allocated in the arena.
Ten bond_rho_raw(Handle& h, const double* A, const double* B, const ctm_env* env) {
  const int D = h.prm.D, d = h.prm.d;
  Ten rho = alloc(h, {d, d, d, d});
  const size_t mark = h.ws.top;
  Ten sA{const_cast<double*>(A), {d, D, D, D, D}}, sB{const_cast<double*>(B), {d, D, D, D, D}};
  const int a = 0, b = 1;
  Ten c1 = envC(env, a, 1), t2 = envT(env, a, 2, D), t1 = envT(env, a, 1, D), c4 = envC(env, a, 4),
      t4 = envT(env, a, 4, D);
  // left half
  Ten E1 = alloc(h, {c1.ext[0], D, D, t2.ext[3]});
  contract(h, op({&c1}, "xy"), op({&t2}, "ymnY"), out({&E1}, "xmnY"));
  Ten E2 = alloc(h, {D, D, t2.ext[3], t1.ext[0], D, D});
  contract(h, op({&E1}, "xmnY"), op({&t1}, "Xkbx"), out({&E2}, "mnYXkb"));
  Ten E3 = alloc(h, {D, t2.ext[3], t1.ext[0], D, d, D, D});
  contract(h, op({&E2}, "mnYXkb"), op({&sA}, "smkpr"), out({&E3}, "nYXbspr"));
  Ten E4 = alloc(h, {t2.ext[3], t1.ext[0], d, D, D, d, D, D});
  contract(h, op({&E3}, "nYXbspr"), op({&sA}, "tnbqw"), out({&E4}, "YXsprtqw"));
  Ten F1 = alloc(h, {c4.ext[1], t4.ext[0], D, D});
  contract(h, op({&c4}, "ZX"), op({&t4}, "UpqZ"), out({&F1}, "XUpq"));
  Ten L = alloc(h, {t2.ext[3], t4.ext[0], d, D, d, D});
  contract(h, op({&E4}, "YXsprtqw"), op({&F1}, "XUpq"), out({&L}, "YUsrtw"));
  // right half
  Ten u2 = envT(env, b, 2, D), c2 = envC(env, b, 2), u3 = envT(env, b, 3, D), c3 = envC(env, b, 3),
      u4 = envT(env, b, 4, D);
  Ten G1 = alloc(h, {u2.ext[0], D, D, c2.ext[1]});
  contract(h, op({&u2}, "Ymnz"), op({&c2}, "zc"), out({&G1}, "Ymnc"));
  Ten G2 = alloc(h, {u2.ext[0], D, D, D, D, u3.ext[3]});
  contract(h, op({&G1}, "Ymnc"), op({&u3}, "cklW"), out({&G2}, "YmnklW"));
  Ten G3 = alloc(h, {u2.ext[0], D, D, u3.ext[3], d, D, D});
  contract(h, op({&G2}, "YmnklW"), op({&sB}, "Smrpk"), out({&G3}, "YnlWSrp"));
  Ten G4 = alloc(h, {u2.ext[0], u3.ext[3], d, D, D, d, D, D});
  contract(h, op({&G3}, "YnlWSrp"), op({&sB}, "Tnwql"), out({&G4}, "YWSrpTwq"));
  Ten H1 = alloc(h, {c3.ext[0], u4.ext[3], D, D});
  contract(h, op({&c3}, "WV"), op({&u4}, "VpqU"), out({&H1}, "WUpq"));
  Ten R = alloc(h, {u2.ext[0], u4.ext[3], d, D, d, D});
  contract(h, op({&G4}, "YWSrpTwq"), op({&H1}, "WUpq"), out({&R}, "YUSrTw"));
  contract(h, op({&L}, "YUsrtw"), op({&R}, "YUSrTw"), out({&rho}, "sStT"));
  h.ws.reset(mark);
  return rho;
}

double bond_energy_impl(Handle& h, const double* A, const double* B, const ctm_env* env, const double* hop,
                        double* rho_out) {
  const int d = h.prm.d;
  const size_t mark = h.ws.top;
  Ten rho = bond_rho_raw(h, A, B, env);
  double* e_dev = h.ws.take(1);
  rho_finish(h, rho.p, hop, d, rho_out, e_dev);
  double e = 0.0;
  if (!h.dry) {
    CTM_CUDA(cudaMemcpyAsync(&e, e_dev, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
    CTM_CUDA(cudaStreamSynchronize(h.stream));
  }
  h.ws.reset(mark);
  return e;
}

// <S^x>, <S^z> of A and B from the H-bond rho by partial trace (reading R23), d = 2.
void site_spins_impl(Handle& h, const double* A, const double* B, const ctm_env* env, double* out_host) {
  if (h.prm.d != 2) throw Error(CTM_E_UNSUPPORTED, "site spins are defined for d = 2 (spin 1/2)");
  const size_t mark = h.ws.top;
  Ten rho = bond_rho_raw(h, A, B, env);
  double* o = h.ws.take(5);
  site_spins(h, rho.p, o);
  if (!h.dry) {
    CTM_CUDA(cudaMemcpyAsync(out_host, o, 5 * sizeof(double), cudaMemcpyDeviceToHost, h.stream));
    CTM_CUDA(cudaStreamSynchronize(h.stream));
  }
  h.ws.reset(mark);
}

}  // namespace
}  // namespace ctm

// =========================================================================================
// C ABI
// =========================================================================================
using ctm::Error;
using ctm::Handle;

struct ctm_handle_s {
  Handle h;
};

namespace {

template <class F>
int guarded(ctm_handle hh, F&& f) {
  if (!hh) return CTM_E_ARG;
  Handle& h = hh->h;
  h.last_error.clear();
  // run on the handle's device; the caller's current device is restored on return
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != h.device && cudaSetDevice(h.device) != cudaSuccess) {
    h.last_error = "cudaSetDevice failed";
    return CTM_E_CUDA;
  }
  struct Restore {
    int prev, cur;
    ~Restore() {
      if (prev >= 0 && prev != cur) cudaSetDevice(prev);
    }
  } restore{prev, h.device};
  try {
    f(h);
    return CTM_OK;
  } catch (const Error& e) {
    h.last_error = e.what();
    h.ws.reset(0);
    h.dry = false;
    return e.code;
  } catch (const std::exception& e) {
    h.last_error = e.what();
    h.ws.reset(0);
    h.dry = false;
    return CTM_E_CUDA;
  }
}

void begin_call(Handle& h) {
  h.ms_svd = 0.0;
  h.ms_iso = 0.0;
  h.flops = 0.0;
  h.min_gap = std::numeric_limits<double>::infinity();
  h.n_svd = 0;
  h.n_svd_fallback = 0;
  h.n_warm = h.n_warm_hit = h.n_warm_retry = 0;
  h.warm_slot = -1;
  h.ms_jacobi = 0.0;
  h.jacobi_flops = 0.0;
  h.jacobi_cta_ms = 0.0;
  h.n_jacobi = 0;
  h.n_kernels = 0;
  h.prof_used = 0;
  h.prof_ms_subs = 0.0;
  h.prof_flops_subs = 0.0;
  h.prof_n_subs = 0;
  h.ms_commit = 0.0;
  h.commit_bytes = 0.0;
  h.n_commit = 0;
  for (auto& r : h.cut_gap)
    for (double& g : r) g = std::numeric_limits<double>::infinity();
  for (auto& r : h.side_gap)
    for (double& g : r) g = std::numeric_limits<double>::infinity();
  if (!h.dry && h.ws.base == nullptr) throw Error(CTM_E_ARG, "workspace not set (ctm_set_workspace)");
  h.ws.reset(0);
}

void fill_stats(Handle& h, ctm_move_stats* st, float ms_total) {
  if (!st) return;
  st->ms_total = ms_total;
  st->ms_svd = h.ms_svd;
  st->ms_isometry = h.ms_iso;
  st->ms_contract = ms_total - h.ms_iso;
  st->flops = h.flops;
  st->min_gap = h.min_gap;
  st->n_svd = h.n_svd;
  st->n_svd_fallback = h.n_svd_fallback;
  st->n_warm = h.n_warm;
  st->n_warm_hit = h.n_warm_hit;
  st->n_warm_retry = h.n_warm_retry;
  st->ms_jacobi = h.ms_jacobi;
  st->jacobi_flops = h.jacobi_flops;
  st->n_jacobi = h.n_jacobi;
  st->jacobi_cta_ms = h.jacobi_cta_ms;
  st->n_kernels = h.n_kernels;
  st->ms_gemm = h.prof_ms_subs;
  st->gemm_flops = h.prof_flops_subs;
  st->gemm_launches = h.prof_used + h.prof_n_subs;
  st->ms_commit = h.ms_commit;
  st->commit_bytes = h.commit_bytes;
  st->n_commit = h.n_commit;
  for (int a = 0; a < 2; ++a) {
    for (int c = 0; c < 2; ++c) st->cut_gap[a][c] = h.cut_gap[a][c];
    for (int i = 0; i < 4; ++i) st->side_gap[a][i] = h.side_gap[a][i];
  }
  if (h.prof_used) {
    CTM_CUDA(cudaEventSynchronize(h.prof_ev[2 * h.prof_used - 1]));
    for (int i = 0; i < h.prof_used; ++i) {
      float ms = 0.f;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.prof_ev[2 * i], h.prof_ev[2 * i + 1]));
      st->ms_gemm += ms;
      st->gemm_flops += h.prof_flops[i];
    }
  }
}

// Dry run of a representative call sequence to size the workspace.
void set_dry(Handle& h, bool on) {
  h.dry = on;
  h.ws.dry = on;
  h.ws.reset(0);
  h.ws.peak = 0;
  if (on) {
    h.ws.base = nullptr;
    h.ws.cap = 0;
  }
  for (auto& s : h.subs) set_dry(*s, on);
}

// Dry run of representative call sequences to size the main and the worker arenas.
void size_workspace(Handle& h) {
  set_dry(h, true);
  const ctm_params& p = h.prm;
  ctm_env env{};
  static double dummy[1];
  for (int x = 0; x < 2; ++x) {
    for (int k = 0; k < 4; ++k) {
      env.C[x][k] = dummy;
      env.T[x][k] = dummy;
    }
    for (int j = 0; j < 8; ++j) env.ext[x][j][0] = env.ext[x][j][1] = p.chi;
  }
  ctm::move_dir(h, CTM_RIGHT, dummy, dummy, &env);
  size_t main_need = h.ws.peak;
  size_t sub_need = 0;
  for (auto& s : h.subs) sub_need = std::max(sub_need, s->ws.peak);
  // ctm_reduced_env runs the whole reduced env on the main handle
  h.ws.reset(0);
  h.ws.peak = 0;
  {
    ctm::Site st = ctm::make_site(h, dummy, dummy, p.d, p.D, 2, 1, 4, 3);
    const int c = p.chi, D = p.D;
    ctm::RenvIn ri{{dummy, {c, c}}, {dummy, {c, D, D, c}}, {dummy, {c, c}}, {dummy, {c, D, D, c}},
                   {dummy, {c, D, D, c}}, &st};
    ctm::reduced_env(h, ri, p.chi_pp);
    main_need = std::max(main_need, h.ws.peak);
    h.ws.reset(0);   // ctm_ts_isometry (main TS, chi' -> chi)
    h.ws.peak = 0;
    ctm::ts_isometry(h, ri.T1, std::max(p.chi_p, p.chi_pp), p.chi, nullptr, false);
    main_need = std::max(main_need, h.ws.peak);
    // optional entry points are sized when they fit the kernel's 2^31-element operand
    // limit; otherwise the handle still serves moves and those calls report CTM_E_ARG /
    // CTM_E_NOMEM when made (C5 at chi = 256: the closures' enlarged corners)
    auto optional = [&](auto&& f) {
      const size_t keep = main_need;
      try {
        h.ws.reset(0);
        h.ws.peak = 0;
        f();
        main_need = std::max(keep, h.ws.peak);
      } catch (const Error&) {
        main_need = keep;
      }
    };
    if (!(p.flags & CTM_FLAG_MOVE_ONLY) || p.strategy == CTM_REDUCED_EXACT)   // ctm_reduced_env(EXACT)
      optional([&]() { ctm::reduced_env_exact(h, ri, dummy, dummy); });
    if (!(p.flags & CTM_FLAG_MOVE_ONLY)) {
      optional([&]() { ctm::norm_2x2_impl(h, dummy, dummy, &env, true); });
      optional([&]() {
        const size_t ns = (size_t)p.d * p.D * p.D * p.D * p.D;
        h.ws.take(2 * ns);
        ctm::bond_energy_impl(h, dummy, dummy, &env, dummy, nullptr);
      });
      optional([&]() {   // ctm_bond_update / ctm_trotter_step (gates + two site buffers)
        const size_t ns = (size_t)p.d * p.D * p.D * p.D * p.D;
        h.ws.take(4 * ns + 2 * (size_t)p.d * p.d * p.d * p.d);
        double cost[2];
        ctm::ffu_update(h, dummy, dummy, &env, dummy, CTM_BOND_V2, 1, dummy, dummy, cost);
      });
    }
  }
  set_dry(h, false);
  const size_t margin = (size_t)32 * 1024 * 1024;   // cuSOLVER workspace size variations
  h.main_bytes = (main_need + margin + 4095) & ~size_t(4095);
  h.sub_bytes = (sub_need + margin + 4095) & ~size_t(4095);
  if (std::getenv("CTM_DEBUG_WS"))
    fprintf(stderr, "[ws] main %.3f GB, %zu subs x %.3f GB\n", h.main_bytes / 1e9, h.subs.size(), h.sub_bytes / 1e9);
}

void init_solver(Handle& h, const ctm_params* p) {
  if (cusolverDnCreate(&h.solver) != CUSOLVER_STATUS_SUCCESS) throw Error(CTM_E_SOLVER, "cusolverDnCreate failed");
  if (cusolverDnCreateParams(&h.solver_params) != CUSOLVER_STATUS_SUCCESS)
    throw Error(CTM_E_SOLVER, "cusolverDnCreateParams failed");
  if (cusolverDnCreateGesvdjInfo(&h.gesvdj_info) != CUSOLVER_STATUS_SUCCESS)
    throw Error(CTM_E_SOLVER, "cusolverDnCreateGesvdjInfo failed");
  double tol = p->svd_tol > 0 ? p->svd_tol : 2.220446049250313e-16;
  cusolverDnXgesvdjSetTolerance(h.gesvdj_info, tol);
  cusolverDnXgesvdjSetMaxSweeps(h.gesvdj_info, 100);
  cusolverDnSetStream(h.solver, h.stream);
  ctm::tc_init_kernels();   // per-device attributes, before any worker thread exists
  ctm::iso_init_kernels();
  CTM_CUDA(cudaMalloc(&h.dev_scalars, 4096));
  CTM_CUDA(cudaMallocHost(&h.pin, 8192));
  h.dev_info = reinterpret_cast<int*>(reinterpret_cast<char*>(h.dev_scalars) + 2048);
  for (auto& e : h.ev) CTM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDefault));
  for (auto& e : h.jev) CTM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDefault));
}

void destroy_handle(Handle& h) {
  for (auto& s : h.subs) destroy_handle(*s);
  h.subs.clear();
  h.warm.reset();   // frees the warm-start blocks (the workers' references went with subs)
  if (h.gesvdj_info) cusolverDnDestroyGesvdjInfo(h.gesvdj_info);
  if (h.solver_params) cusolverDnDestroyParams(h.solver_params);
  if (h.solver) cusolverDnDestroy(h.solver);
  for (auto& e : h.ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h.jev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h.prof_ev) cudaEventDestroy(e);
  if (h.dev_scalars) cudaFree(h.dev_scalars);
  if (h.pin) cudaFreeHost(h.pin);
  h.pin = nullptr;
  if (h.owns_stream && h.stream) cudaStreamDestroy(h.stream);
  h.gesvdj_info = nullptr;
  h.solver_params = nullptr;
  h.solver = nullptr;
  h.dev_scalars = nullptr;
}

}  // namespace

extern "C" {

int ctm_abi_version(void) { return CTM_ABI_VERSION; }

int ctm_init(ctm_handle* out, const ctm_params* p, uintptr_t stream, size_t* ws_bytes) {
  if (!out || !p) return CTM_E_ARG;
  *out = nullptr;
  if (p->d < 1 || p->D < 1 || p->chi < 1 || p->chi_p < 1 || p->chi_pp < 1) return CTM_E_ARG;
  if (p->strategy != CTM_SEQUENTIAL && p->strategy != CTM_REDUCED_EXACT && p->strategy != CTM_STANDARD)
    return CTM_E_UNSUPPORTED;
  std::unique_ptr<ctm_handle_s> hh(new ctm_handle_s());
  Handle& h = hh->h;
  h.prm = *p;
  int warn = 0;
  if (h.prm.chi_p > h.prm.chi * h.prm.D) {   // clamp chi' to chi D with a warning
    h.prm.chi_p = h.prm.chi * h.prm.D;
    warn = CTM_W_CLAMPED;
  }
  h.stream = reinterpret_cast<cudaStream_t>(stream);
  if (cudaGetDevice(&h.device) != cudaSuccess) return CTM_E_CUDA;   // the handle's device
  try {
    init_solver(h, &h.prm);
    for (int i = 0; i < 4; ++i) {   // workers of the isometry stage (4 side TS, 2 main TS)
      std::unique_ptr<Handle> s(new Handle());
      s->prm = h.prm;
      s->device = h.device;   // (CTM_FLAG_PROFILE kept: the solver's GEMMs are timed too)
      CTM_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
      s->owns_stream = true;
      init_solver(*s, &s->prm);
      h.subs.push_back(std::move(s));
    }
    if (h.prm.flags & CTM_FLAG_WARM_START) {
      h.warm = std::make_shared<ctm::WarmStore>();
      h.warm->slots.resize(4 * 2 * ctm::CTM_WARM_SITES);   // (direction, absorption, site); never resized
      for (auto& s : h.subs) s->warm = h.warm;
    }
    size_workspace(h);
    if (ws_bytes) *ws_bytes = h.main_bytes + h.subs.size() * h.sub_bytes;
  } catch (const Error& e) {
    fprintf(stderr, "ctm_init: %s\n", e.what());
    destroy_handle(h);
    return e.code;
  }
  *out = hh.release();
  return CTM_OK | warn;
}

int ctm_set_workspace(ctm_handle hh, void* dev, size_t bytes) {
  return guarded(hh, [&](Handle& h) {
    if (!dev) throw Error(CTM_E_ARG, "null workspace");
    const size_t need = h.main_bytes + h.subs.size() * h.sub_bytes;
    if (bytes < need) throw Error(CTM_E_NOMEM, "workspace smaller than ctm_init reported");
    char* base = static_cast<char*>(dev);
    h.ws.base = base;
    h.ws.cap = h.main_bytes;
    h.ws.reset(0);
    for (size_t i = 0; i < h.subs.size(); ++i) {
      Handle& s = *h.subs[i];
      s.ws.base = base + h.main_bytes + i * h.sub_bytes;
      s.ws.cap = h.sub_bytes;
      s.ws.reset(0);
    }
  });
}

int ctm_set_stream(ctm_handle hh, uintptr_t stream) {
  return guarded(hh, [&](Handle& h) {
    h.stream = reinterpret_cast<cudaStream_t>(stream);
    cusolverDnSetStream(h.solver, h.stream);
  });
}

int ctm_destroy(ctm_handle hh) {
  if (!hh) return CTM_E_ARG;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(hh->h.device);
  cudaStreamSynchronize(hh->h.stream);
  destroy_handle(hh->h);
  delete hh;
  if (prev >= 0) cudaSetDevice(prev);
  return CTM_OK;
}

const char* ctm_last_error(ctm_handle hh) { return hh ? hh->h.last_error.c_str() : "null handle"; }

int64_t ctm_kernel_count(ctm_handle hh) { return hh ? hh->h.kernel_count : 0; }

int ctm_warm_reset(ctm_handle hh) {
  if (!hh) return CTM_E_ARG;
  if (hh->h.warm)
    for (auto& s : hh->h.warm->slots) {
      s.valid = false;
      s.miss = s.skip = 0;
    }
  return CTM_OK;
}

double ctm_move_flops(int d, int D, int chi, int chi_p, int chi_pp) {
  // Sum of 2 M N K over the contractions of one left move for square extents, exactly as
  // issued by this library (SURVEY 8(a) closed form when chi = chi' = chi'').
  auto chain = [&](double cin, double n1, double o1, double cout, double m1, double o2) {
    double DD = D;
    return 2 * n1 * DD * DD * DD * cin * cout        // S1
           + 2 * n1 * DD * cout * d * DD * DD * DD * DD   // S2
           + 2 * n1 * DD * d * DD * m1 * cout * DD   // S3
           + 2 * DD * d * DD * m1 * DD * o1 * n1     // S4
           + 2 * DD * m1 * o1 * DD * DD * d * DD * DD     // S5
           + 2 * o1 * DD * DD * o2 * m1 * DD;        // S6
  };
  double c = chi, cp = std::min((double)chi_p, c * D);
  double n1 = std::min((double)chi_pp, c * D), n2 = std::min((double)chi_pp, n1 * D);
  double DD = D;
  double renv = 2 * (2 * c * c * c * DD * DD)            // a1: Q_l, Q_r
                + 2 * (2 * n1 * DD * c * c * DD)          // a2: v1^T Q (l and r)
                + chain(c, n1, n2, c, n1, n2)             // a3: T'^2
                + 2 * (2 * c * n2 * n1 * DD)              // a4: C', C''
                + 2 * c * DD * DD * n2 * n2               // a4: C' T'
                + 2 * c * DD * DD * n2 * c;               // a4: (C' T') C''
  double main_ts = 2 * cp * DD * c * c * DD;              // a5: v1^T M
  double ch = chain(c, cp, c, c, cp, c);
  double corner = 2 * c * c * DD * cp + 2 * cp * c * DD * DD * c + 2 * c * cp * DD * c;
  double col = 2 * (renv + main_ts) + 2 * ch + 4 * corner;
  return 2 * col;
}

int ctm_absorb_truncate(ctm_handle hh, const double* T, const double* X, const double* Xbra, const double* v1_in,
                        const double* v2_in, const double* v1_out, const double* v2_out, double* T_out) {
  return guarded(hh, [&](Handle& h) {
    if (!T || !X || !Xbra || !v1_in || !v2_in || !v1_out || !v2_out || !T_out) throw Error(CTM_E_ARG, "null pointer");
    begin_call(h);
    const ctm_params& p = h.prm;
    const int D = p.D, d = p.d, c = p.chi, cp = p.chi_p;
    // X given in chain orientation (s, in, face, out, far): axes s=0 in=1 face=2 out=3 far=4
    ctm::Site s;
    s.ket = ctm::alloc(h, {D, D, d, D, D});
    s.bra = ctm::alloc(h, {d, D, D, D, D});
    ctm::permute(h, X, {d, D, D, D, D}, {1, 2, 0, 3, 4}, s.ket.p);
    ctm::permute(h, Xbra, {d, D, D, D, D}, {0, 2, 1, 3, 4}, s.bra.p);
    ctm::Ten Tt{const_cast<double*>(T), {c, D, D, c}};
    ctm::Iso in{{const_cast<double*>(v1_in), {c, D, cp}}, {const_cast<double*>(v2_in), {cp, D, c}}};
    ctm::Iso ou{{const_cast<double*>(v1_out), {c, D, cp}}, {const_cast<double*>(v2_out), {cp, D, c}}};
    ctm::Ten res{T_out, {c, D, D, c}};
    ctm::chains(h, {ctm::ChainJob{&Tt, &s, &in, &ou, &res, nullptr}});
  });
}

int ctm_ts_isometry(ctm_handle hh, const double* Q, int P, int K, int Bd, int F, int c1, int c2, int mode,
                    double* v1_out, double* v2_out, double* gaps_host) {
  return guarded(hh, [&](Handle& h) {
    if (!Q || !v1_out || !v2_out) throw Error(CTM_E_ARG, "null pointer");
    if (mode != CTM_TS_SVD && mode != CTM_TS_BASIS) throw Error(CTM_E_ARG, "unknown TS mode");
    const ctm_params& p = h.prm;
    // the workspace is sized for the TS calls of a move: Q up to (chi, D, D, chi)
    if (P < 1 || F < 1 || c1 < 1 || c2 < 1 || P > p.chi || F > p.chi || K != p.D || Bd != p.D ||
        c1 > std::max(p.chi_p, p.chi_pp) || c2 > p.chi)
      throw Error(CTM_E_ARG, "TS shape outside the handle's (chi, D, D, chi) / chi', chi'' sizing");
    begin_call(h);
    ctm::Ten Qt{const_cast<double*>(Q), {P, K, Bd, F}};
    ctm::Iso v = ctm::ts_isometry(h, Qt, c1, c2, nullptr, mode == CTM_TS_BASIS);
    CTM_CUDA(cudaMemcpyAsync(v1_out, v.v1.p, v.v1.size() * 8, cudaMemcpyDeviceToDevice, h.stream));
    CTM_CUDA(cudaMemcpyAsync(v2_out, v.v2.p, v.v2.size() * 8, cudaMemcpyDeviceToDevice, h.stream));
    CTM_CUDA(cudaStreamSynchronize(h.stream));
    if (gaps_host) {
      gaps_host[0] = v.gap1;
      gaps_host[1] = v.gap2;
    }
  });
}

int ctm_reduced_env(ctm_handle hh, const double* C1, const double* T2, const double* C2, const double* T1,
                    const double* X, const double* Xbra, const double* T3, int mode, double* M_out,
                    const double* iso_in, double* iso_out) {
  return guarded(hh, [&](Handle& h) {
    if (!C1 || !T2 || !C2 || !T1 || !X || !Xbra || !T3 || !M_out) throw Error(CTM_E_ARG, "null pointer");
    if (mode != CTM_RENV_APPROX && mode != CTM_RENV_EXACT) throw Error(CTM_E_ARG, "unknown reduced-env mode");
    if (iso_in && mode != CTM_RENV_APPROX) throw Error(CTM_E_ARG, "iso_in needs CTM_RENV_APPROX");
    begin_call(h);
    const ctm_params& p = h.prm;
    const int D = p.D, c = p.chi;
    if (mode == CTM_RENV_EXACT) {
      ctm::RenvIn ri{{const_cast<double*>(C1), {c, c}},       {const_cast<double*>(T2), {c, D, D, c}},
                     {const_cast<double*>(C2), {c, c}},       {const_cast<double*>(T1), {c, D, D, c}},
                     {const_cast<double*>(T3), {c, D, D, c}}, nullptr};
      ctm::Ten M = ctm::reduced_env_exact(h, ri, X, Xbra);
      CTM_CUDA(cudaMemcpyAsync(M_out, M.p, M.size() * 8, cudaMemcpyDeviceToDevice, h.stream));
      CTM_CUDA(cudaStreamSynchronize(h.stream));
      return;
    }
    ctm::Site st = ctm::make_site(h, X, Xbra, p.d, D, 2, 1, 4, 3);
    ctm::RenvIn ri{{const_cast<double*>(C1), {c, c}},       {const_cast<double*>(T2), {c, D, D, c}},
                   {const_cast<double*>(C2), {c, c}},       {const_cast<double*>(T1), {c, D, D, c}},
                   {const_cast<double*>(T3), {c, D, D, c}}, &st};
    ctm::RenvOut ro;
    if (iso_in) {   // injected side isometries: the contractions of rows a1, a3, a4 only
      const int n1 = std::min(p.chi_pp, c * D), n2 = std::min(p.chi_pp, n1 * D);
      const size_t s1 = (size_t)c * D * n1, s2 = (size_t)n1 * D * n2;
      ctm::SideOut L = ctm::side_inject(h, ri, true, iso_in, iso_in + s1, n1, n2);
      ctm::SideOut R = ctm::side_inject(h, ri, false, iso_in + s1 + s2, iso_in + 2 * s1 + s2, n1, n2);
      ro = ctm::renv_finish(h, ri, L, R);
    } else {
      ro = ctm::reduced_env(h, ri, p.chi_pp);
    }
    CTM_CUDA(cudaMemcpyAsync(M_out, ro.M.p, ro.M.size() * 8, cudaMemcpyDeviceToDevice, h.stream));
    if (iso_out) {
      double* o = iso_out;
      for (const ctm::Ten* t : {&ro.vl.v1, &ro.vl.v2, &ro.vr.v1, &ro.vr.v2}) {
        CTM_CUDA(cudaMemcpyAsync(o, t->p, t->size() * 8, cudaMemcpyDeviceToDevice, h.stream));
        o += t->size();
      }
    }
    if (!iso_in) CTM_CUDA(cudaStreamSynchronize(h.stream));   // (injected: no SVD, asynchronous)
  });
}

int ctm_left_move(ctm_handle hh, const double* A, const double* B, ctm_env* env, const double* iso_in,
                  double* iso_out, ctm_move_stats* st) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env) throw Error(CTM_E_ARG, "null pointer");
    begin_call(h);
    ctm::check_env(env, h.prm);
    CTM_CUDA(cudaEventRecord(h.ev[0], h.stream));
    ctm::left_move(h, A, B, env, iso_in, iso_out);
    CTM_CUDA(cudaEventRecord(h.ev[1], h.stream));
    if (st) {
      CTM_CUDA(cudaEventSynchronize(h.ev[1]));
      float ms = 0;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]));
      fill_stats(h, st, ms);
    }
  });
}

int ctm_move(ctm_handle hh, int dir, const double* A, const double* B, ctm_env* env, double* iso_out,
             ctm_move_stats* st) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || dir < 0 || dir > 3) throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    CTM_CUDA(cudaEventRecord(h.ev[0], h.stream));
    ctm::move_dir(h, dir, A, B, env, iso_out);
    CTM_CUDA(cudaEventRecord(h.ev[1], h.stream));
    if (st) {
      CTM_CUDA(cudaEventSynchronize(h.ev[1]));
      float ms = 0;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]));
      fill_stats(h, st, ms);
    }
  });
}

int ctm_iterate(ctm_handle hh, const double* A, const double* B, ctm_env* env, int n_iter, ctm_move_stats* st) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || n_iter < 0) throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    CTM_CUDA(cudaEventRecord(h.ev[0], h.stream));
    for (int it = 0; it < n_iter; ++it)
      for (int dir : {CTM_LEFT, CTM_RIGHT, CTM_UP, CTM_DOWN}) ctm::move_dir(h, dir, A, B, env);
    CTM_CUDA(cudaEventRecord(h.ev[1], h.stream));
    if (st) {
      CTM_CUDA(cudaEventSynchronize(h.ev[1]));
      float ms = 0;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]));
      fill_stats(h, st, ms);
    }
  });
}

namespace {
// Corner spectra normalised to unit sum and their distance (reading R22).
std::vector<std::vector<double>> corner_spectra(Handle& h, const ctm_env* env) {
  std::vector<std::vector<double>> out;
  for (int x = 0; x < 2; ++x)
    for (int k = 0; k < 4; ++k) {
      const int r = env->ext[x][k][0], c = env->ext[x][k][1];
      std::vector<double> sv(std::min(r, c));
      ctm::singular_values(h, env->C[x][k], r, c, sv.data());
      double t = 0.0;
      for (double v : sv) t += v;
      for (double& v : sv) v = t > 0.0 ? v / t : 0.0;
      out.push_back(std::move(sv));
    }
  return out;
}
double spectra_distance(const std::vector<std::vector<double>>& a, const std::vector<std::vector<double>>& b) {
  double out = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const size_t n = std::max(a[i].size(), b[i].size());
    double d = 0.0;
    for (size_t j = 0; j < n; ++j) d += std::fabs((j < a[i].size() ? a[i][j] : 0.0) - (j < b[i].size() ? b[i][j] : 0.0));
    out = std::max(out, d);
  }
  return out;
}
}  // namespace

int ctm_converge(ctm_handle hh, const double* A, const double* B, ctm_env* env, int max_iter, double tol,
                 int* iters_out, double* delta_out, ctm_move_stats* st) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || max_iter < 1 || !(tol >= 0.0)) throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    CTM_CUDA(cudaEventRecord(h.ev[0], h.stream));
    auto prev = corner_spectra(h, env);
    double delta = std::numeric_limits<double>::infinity();
    int it = 0;
    while (it < max_iter) {
      ++it;
      for (int dir : {CTM_LEFT, CTM_RIGHT, CTM_UP, CTM_DOWN}) ctm::move_dir(h, dir, A, B, env);
      auto cur = corner_spectra(h, env);
      delta = spectra_distance(prev, cur);
      if (delta < tol) break;
      prev = std::move(cur);
    }
    if (iters_out) *iters_out = it;
    if (delta_out) *delta_out = delta;
    CTM_CUDA(cudaEventRecord(h.ev[1], h.stream));
    if (st) {
      CTM_CUDA(cudaEventSynchronize(h.ev[1]));
      float ms = 0;
      CTM_CUDA(cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]));
      fill_stats(h, st, ms);
    }
  });
}

int ctm_trotter_gate(ctm_handle hh, const double* hop, double delta, double* gate_out) {
  return guarded(hh, [&](Handle& h) {
    if (!hop || !gate_out) throw Error(CTM_E_ARG, "null pointer");
    begin_call(h);
    ctm::ffu_gate(h, hop, delta, gate_out);
  });
}

int ctm_bond_update(ctm_handle hh, const double* A, const double* B, const ctm_env* env, const double* gate,
                    int bond, int sweeps, double* A_out, double* B_out, double* cost_host) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || !gate || !A_out || !B_out || sweeps < 0 || bond < 0 || bond > 3)
      throw Error(CTM_E_ARG, "bad argument");
    if (A_out == A || A_out == B || B_out == A || B_out == B) throw Error(CTM_E_ARG, "outputs must not alias the sites");
    begin_call(h);
    ctm::check_env(env, h.prm);
    ctm::ffu_update(h, A, B, env, gate, bond, sweeps, A_out, B_out, cost_host);
  });
}

int ctm_trotter_step(ctm_handle hh, double* A, double* B, ctm_env* env, const double* hop, double delta, int sweeps,
                     int refresh, double* cost_host) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || !hop || sweeps < 0) throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    const ctm_params& p = h.prm;
    const size_t ns = (size_t)p.d * p.D * p.D * p.D * p.D, ng = (size_t)p.d * p.d * p.d * p.d;
    double* g_half = h.ws.take(ng);
    double* g_full = h.ws.take(ng);
    double* A2 = h.ws.take(ns);
    double* B2 = h.ws.take(ns);
    ctm::ffu_gate(h, hop, 0.5 * delta, g_half);
    ctm::ffu_gate(h, hop, delta, g_full);
    // reading R29: H1(d/2) H2(d/2) V1(d/2) V2(d) V1(d/2) H2(d/2) H1(d/2); R30: one CTM
    // iteration after every bond update (FFU)
    static const int order[7] = {CTM_BOND_H1, CTM_BOND_H2, CTM_BOND_V1, CTM_BOND_V2, CTM_BOND_V1, CTM_BOND_H2,
                                 CTM_BOND_H1};
    for (int i = 0; i < 7; ++i) {
      const double* g = i == 3 ? g_full : g_half;
      ctm::ffu_update(h, A, B, env, g, order[i], sweeps, A2, B2, cost_host ? cost_host + 2 * i : nullptr);
      CTM_CUDA(cudaMemcpyAsync(A, A2, ns * 8, cudaMemcpyDeviceToDevice, h.stream));
      CTM_CUDA(cudaMemcpyAsync(B, B2, ns * 8, cudaMemcpyDeviceToDevice, h.stream));
      if (refresh)
        for (int dir : {CTM_LEFT, CTM_RIGHT, CTM_UP, CTM_DOWN}) ctm::move_dir(h, dir, A, B, env);
    }
    CTM_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int ctm_norm_2x2(ctm_handle hh, const double* A, const double* B, const ctm_env* env, double* out_host,
                 double* cancel_ratio_host) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || !out_host) throw Error(CTM_E_ARG, "null pointer");
    begin_call(h);
    ctm::check_env(env, h.prm);
    double v = ctm::norm_2x2_impl(h, A, B, env, false);
    *out_host = v;
    if (cancel_ratio_host) {
      double va = ctm::norm_2x2_impl(h, A, B, env, true);
      *cancel_ratio_host = va != 0.0 ? v / va : 0.0;
    }
  });
}

int ctm_site_spins(ctm_handle hh, const double* A, const double* B, const ctm_env* env, double* out_host) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || !out_host) throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    ctm::site_spins_impl(h, A, B, env, out_host);
  });
}

int ctm_bond_energy(ctm_handle hh, const double* A, const double* B, const ctm_env* env, const double* hop,
                    int bond, double* rho_out, double* e_out_host) {
  return guarded(hh, [&](Handle& h) {
    if (!A || !B || !env || !hop || !e_out_host || (bond != CTM_BOND_H && bond != CTM_BOND_V))
      throw Error(CTM_E_ARG, "bad argument");
    begin_call(h);
    ctm::check_env(env, h.prm);
    if (bond == CTM_BOND_H) {
      *e_out_host = ctm::bond_energy_impl(h, A, B, env, hop, rho_out);
    } else {
      // A above B: one counter-clockwise quarter turn (= 3 clockwise) brings it to A left of B
      const size_t ns = (size_t)h.prm.d * h.prm.D * h.prm.D * h.prm.D * h.prm.D;
      double* Ar = h.ws.take(ns);
      double* Br = h.ws.take(ns);
      ctm::rotate_site(h, A, Ar, 3);
      ctm::rotate_site(h, B, Br, 3);
      ctm_env e = *env;
      for (int i = 0; i < 3; ++i) ctm::rotate_env_cw(&e);
      *e_out_host = ctm::bond_energy_impl(h, Ar, Br, &e, hop, rho_out);
    }
  });
}

}  // extern "C"
