/*
 * ctm.h -- C ABI of libctm: the CTMRG move of arXiv 2306.08212 (Lan & Evenbly,
 * "Reduced Contraction Costs of Corner-Transfer Methods for PEPS") on one B200, FP64.
 *
 * Citations: "P:Lnn" = PAPER.md line nn.  SURVEY.md sections 0 and 8 fix the readings
 * (listed in DESIGN.md "Readings").
 *
 * ---------------------------------------------------------------------------------
 * Conventions common to every call
 * ---------------------------------------------------------------------------------
 *  Tensors.  Every tensor argument is a DEVICE pointer to contiguous row-major float64
 *    memory, owned by the caller.  The library never frees or retains caller memory
 *    past the call.  Shapes follow the paper's definitions:
 *      site A, B           (d, D, D, D, D)  legs (s, u, l, d, r)            [P:L39]
 *      corner C_x^k        (chi, chi)                                      [P:L41]
 *      edge   T_x^k        (chi, D, D, chi)  (boundary, ket, bra, boundary) [P:L41]
 *    Environment tensors are stored walking the boundary clockwise:
 *      T^1 (d,k,b,u)  T^2 (l,k,b,r)  T^3 (u,k,b,d)  T^4 (r,k,b,l)
 *      C^1 (d,r)      C^2 (l,d)      C^3 (u,l)      C^4 (r,u)
 *    where k/b are the ket/bra legs facing the bulk (kept split).
 *    The bra layer is passed separately (Xbra) but all shipped configs are real.
 *  Isometries (Fig 4): v1 (chi_in, D, chi') and v2 (chi', D, chi_out),
 *    row-major, i.e. the first chi' (resp. chi_out) left singular vectors of the
 *    (chi D) x (D chi) and (chi' D) x chi matrices, columns sign-fixed so that the
 *    largest-|.| entry of each column is positive (ties: lowest row index).
 *  Stream.  All work is enqueued on the stream given to ctm_init (a cudaStream_t
 *    passed as uintptr_t; 0 = legacy default stream; ctm_set_stream changes it).
 *    Calls that run SVDs synchronise that stream (cuSOLVER status and host-side
 *    error checks); pure-contraction calls are asynchronous.
 *  Workspace.  ctm_init reports the bytes needed; the caller allocates device memory
 *    (e.g. a torch tensor) and hands it over with ctm_set_workspace before any compute
 *    call.  The handle owns only cuSOLVER/cuBLAS-free state (solver handle, events).
 *  Errors.  Every call returns an int status (below).  No C++ exception crosses the
 *    ABI.  ctm_last_error(h) returns a NUL-terminated message for the last failure of
 *    that handle (valid until the next call on it).  A failed call leaves output
 *    buffers unspecified; ctm_left_move commits the environment only after every
 *    check of the move passed (snapshot semantics).
 */
#ifndef CTM_H_
#define CTM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTM_ABI_VERSION 3

/* status codes */
#define CTM_OK 0
#define CTM_E_ARG 1          /* null pointer, bad extent, missing workspace          */
#define CTM_E_CUDA 2         /* CUDA runtime / launch failure                         */
#define CTM_E_SOLVER 3       /* SVD failed to converge (message carries m x n) */
#define CTM_E_NONFINITE 4    /* NaN/Inf produced (message names absorption, tensor)  */
#define CTM_E_NOMEM 5        /* workspace too small                                   */
#define CTM_E_UNSUPPORTED 6  /* strategy / mode not built in this library             */
#define CTM_W_CLAMPED 100    /* warning bit: chi' > chi D was clamped        */

/* strategies (ctm_params.strategy) */
#define CTM_SEQUENTIAL 0     /* reduced env + sequential ket/bra order: the hot path  */
#define CTM_REDUCED_EXACT 1  /* exact reduced env M (Fig 3(b)) + one-shot 4-leg
                                isometry from M as (chi D^2) x chi; O(chi^3 D^4)           */
#define CTM_STANDARD 2       /* 8-tensor upper half of Fig 1(d) (Fig 2(c)) + one-shot
                                isometry from (chi D^2) x (D^2 chi); O(chi^3 D^6)          */

/* SVD back-ends (ctm_params.svd_algo); all on the device, no CPU fallback */
#define CTM_SVD_GESVDP 0     /* cuSOLVER Xgesvdp (polar decomposition)                */
#define CTM_SVD_GESVDJ 1     /* cuSOLVER gesvdj (Jacobi), tolerance svd_tol            */
#define CTM_SVD_GESVD 2      /* cuSOLVER Xgesvd (QR iteration)                         */
#define CTM_SVD_GRAM 3       /* truncating cuts (n_keep < rows <= cols): top eigenvectors of
                                the Gram matrix M M^T (libctm DMMA GEMM + cuSOLVER syevd);
                                every other shape: Xgesvdp.  Subspace error
                                ~ eps (s_1/s_n)^2 / (1 - (s_{n+1}/s_n)^2) instead of
                                eps (s_1/s_n) / (1 - s_{n+1}/s_n).          */
#define CTM_SVD_ISO 4        /* libctm's own solver (default): subspace iteration on M M^T
                                with CholQR, Rayleigh-Ritz through a backward-stable QR and
                                one-sided Jacobi (all libctm kernels + DMMA GEMMs); tall /
                                small cuts: QR + one-sided Jacobi.  Shapes beyond its
                                range (block l = n_keep + 32 > 320, or a tall/small cut wider
                                than 320) or whose convergence it cannot certify fall back
                                to Xgesvdp (counted in n_svd_fallback). */

/* flags (ctm_params.flags) */
#define CTM_FLAG_CHECK_FINITE 1   /* scan every committed tensor for NaN/Inf         */
#define CTM_FLAG_MOVE_ONLY 2      /* size the workspace for moves only (no closures)  */
#define CTM_FLAG_PROFILE 4        /* time every contraction launch with CUDA events   */
#define CTM_FLAG_WARM_START 8     /* CTM_SVD_ISO, sequential strategy: every truncating solve of a move
                                     starts from the final block of the same solve site (direction,
                                     absorption, cut) of the handle's previous move instead of a random
                                     block.  A CTM iteration converges (N_CTM ~ 10-30 iterations),
                                     so the previous subspace is a near-solution; the solve still ends
                                     only on the residual certificate measured on the NEW matrix, so the
                                     result is start-independent up to rounding.  The blocks (R x l
                                     doubles per site, 48 sites) are device memory owned by the handle,
                                     allocated at a site's first solve, freed by ctm_destroy; a site
                                     whose shapes changed, and a warm solve that fails, start cold.
                                     ctm_warm_reset forgets them.  Off by default (a move is then a
                                     pure function of its inputs).                                  */

/* reduced-env modes (ctm_reduced_env) */
#define CTM_RENV_APPROX 0    /* {C'^1, T'^2, C'^2} with side isometries */
#define CTM_RENV_EXACT 1     /* exact Fig 3(b) network, P:L53 (NEXT on GPU)            */

/* two-stage isometry modes (ctm_ts_isometry) */
#define CTM_TS_SVD 0         /* both stages are SVDs (left singular vectors, sign rule)     */
#define CTM_TS_BASIS 1       /* what ctm_left_move runs for every cut: a stage two that
                                truncates nothing returns an orthonormal basis of its column
                                space (same projector v v^T; readings R24 side, R24b main)  */

/* bonds (ctm_bond_energy) */
#define CTM_BOND_H 0         /* A left of B: 2x1 window                               */
#define CTM_BOND_V 1         /* A above B: 1x2 window                                 */

/* the four bonds of the 2-site unit cell (ctm_bond_update, ctm_trotter_step) */
#define CTM_BOND_H1 0        /* A left of B (= CTM_BOND_H)                            */
#define CTM_BOND_V1 1        /* A above B   (= CTM_BOND_V)                            */
#define CTM_BOND_H2 2        /* B left of A                                           */
#define CTM_BOND_V2 3        /* B above A                                             */

/* directions (ctm_move) */
#define CTM_LEFT 0
#define CTM_RIGHT 1
#define CTM_UP 2
#define CTM_DOWN 3

typedef struct ctm_handle_s* ctm_handle;

typedef struct {
  int d;           /* physical dimension                                       */
  int D;           /* virtual bond dimension                                   */
  int chi;         /* boundary dimension chi                                   */
  int chi_p;       /* chi'  : first sequential isometry                        */
  int chi_pp;      /* chi'' : appendix side isometries v_l, v_r               */
  int strategy;    /* CTM_SEQUENTIAL                                                   */
  int svd_algo;    /* CTM_SVD_*                                                        */
  double svd_tol;  /* gesvdj tolerance (<= 0: machine epsilon)                         */
  int flags;       /* CTM_FLAG_*                                                       */
} ctm_params;

/* The 16 environment tensors (C_x^k, T_x^k, x in {a,b}, k = 1..4) and their
 * boundary extents.  C[x][k-1], T[x][k-1] with x = 0 for 'a', 1 for 'b'.
 * ext[x][j][0..1] = (first, last) boundary extent in STORAGE order, j = 0..3 for
 * C^1..C^4 and j = 4..7 for T^1..T^4.  Buffers must be allocated with capacity for the
 * target extents (chi x chi, chi x D x D x chi); moves update ext in place. */
typedef struct {
  double* C[2][4];
  double* T[2][4];
  int ext[2][8][2];
} ctm_env;

/* Per-call statistics (host struct, filled by ctm_left_move / ctm_move). */
typedef struct {
  double ms_total;      /* device time of the call (CUDA events)                       */
  double ms_svd;        /* summed device time of the SVD calls (cuSOLVER + sign fix); the
                           calls of one absorption overlap on worker streams, so this can
                           exceed ms_isometry                                           */
  double ms_contract;   /* ms_total - ms_isometry: absorb chains, corners, commit      */
  double flops;         /* algorithmic contraction flops (SURVEY 8(a) closed form)      */
  double min_gap;       /* min sigma_n / sigma_{n+1} over every truncation of the call  */
  int n_svd;            /* SVDs run                                                    */
  int n_kernels;        /* libctm kernels launched (excluding cuSOLVER internals)       */
  /* CTM_FLAG_PROFILE only: the contraction kernel (tc_gemm) timed launch by launch, on the
     caller's stream and on the isometry workers' streams (their solver GEMMs included) */
  double ms_gemm;       /* summed device time of the tc_gemm launches                  */
  double gemm_flops;    /* their algorithmic flops (sum of 2 M N K)                     */
  int gemm_launches;    /* number of tc_gemm launches                                  */
  double ms_isometry;   /* wall device time of the isometry stages (reduced envs + TS,  */
                        /* rows a1-a5) on the caller's stream, fork to join            */
  int n_svd_fallback;   /* CTM_SVD_ISO truncations that fell back to cuSOLVER Xgesvdp   */
  /* CTM_SVD_ISO: the one-sided Jacobi SVD launches of the solver, timed by CUDA events on
     their (worker) streams; flops = 6 n^2 (n - 1) per executed sweep (per rotation pair and
     round: three inner products, 6n, and the rotation, 6n)                                 */
  double ms_jacobi;     /* summed device time of the Jacobi launches                    */
  double jacobi_flops;  /* their algorithmic flops                                       */
  int n_jacobi;         /* number of Jacobi launches                                     */
  double jacobi_cta_ms; /* sum of launch time x CTAs (one CTA per SM): SM-weighted time  */
  /* Per-cut truncation gaps sigma_n / sigma_{n+1} of the stage-one SVD (SURVEY 8(b),
     8(d) "log min sigma_chi/sigma_{chi+1} per cut"), the minimum over the moves of the call;
     +inf where nothing was truncated or the isometries were injected.
       cut_gap[a][c]:  main TS(M; chi', chi) of absorption a = 0, 1, cut c = ab (0), ba (1);
       side_gap[a][i]: side TS(Q; chi'', chi'') of absorption a, i = a-left, a-right,
                       b-left, b-right (Q_l = C^1 T^1, Q_r = C^2 T^3).             */
  double cut_gap[2][2];
  double side_gap[2][4];
  /* CTM_FLAG_PROFILE only: the normalise + commit launches (K7, HBM-bound), timed by CUDA
     events; bytes = algorithmic traffic (read the six new tensors + write them to the env) */
  double ms_commit;
  double commit_bytes;
  int n_commit;
  /* CTM_FLAG_WARM_START: truncating solves that started from their site's previous block, how
     many of those were certified at their first Rayleigh-Ritz check (no filter degree at all),
     and how many failed to converge and were redone from the cold start                      */
  int n_warm;
  int n_warm_hit;
  int n_warm_retry;
} ctm_move_stats;

/* ctm_init: validate sizes, create the handle, report the workspace bytes needed by
 * every call for these params (the peak of SURVEY 8(a): intermediates of two
 * concurrent absorb chains + SVD buffers).  Env initialisation is NOT done here: the
 * seeded generator lives in the harness (ctm_inputs.py) so the oracle and the GPU see
 * bit-identical inputs.  Returns CTM_E_ARG for d, D, chi < 1. */
int ctm_init(ctm_handle* h, const ctm_params* p, uintptr_t stream, size_t* ws_bytes);
int ctm_set_workspace(ctm_handle h, void* dev, size_t bytes);
int ctm_set_stream(ctm_handle h, uintptr_t stream);
int ctm_destroy(ctm_handle h);
const char* ctm_last_error(ctm_handle h);
int ctm_abi_version(void);

/* ctm_reduced_env: SURVEY rows a1-a4 (Fig 3(c), appendix).
 * Inputs (all chi = params.chi):  C1 = C_x^1 (d,r); T2 = T_x^2 (l,k,b,r);
 * C2 = C_x^2 (l,d); T1 = T_x^1 (d,k,b,u); X, Xbra = site x (s,u,l,d,r);
 * T3 = T_x^3 (u,k,b,d).
 * Output M_out (chi, D, D, chi) = M(q, k_d, b_d, q') with q = T^1's d leg,
 * (k_d, b_d) = X's down legs, q' = T^3's d leg.  M is gauge-free (its legs are
 * existing bonds).  mode CTM_RENV_APPROX: M = C'^1 T'^2 C'^2 with side isometries
 * (v_l1, v_l2) = TS(C^1 T^1; chi'', chi''), (v_r1, v_r2) = TS(C^2 T^3; chi'', chi'').
 * iso_out (nullable) receives vl1, vl2, vr1, vr2 back to back (shapes
 * (chi,D,n1), (n1,D,n2) twice, n1 = min(chi'', chi D), n2 = min(chi'', n1 D)).
 * iso_in (nullable, APPROX only, same layout): inject the side isometries -- no SVD, only
 * the contractions of rows a1, a3, a4 (and v^1 Q of a2); asynchronous.
 * Otherwise synchronises the stream (SVDs). */
int ctm_reduced_env(ctm_handle h, const double* C1, const double* T2, const double* C2,
                    const double* T1, const double* X, const double* Xbra, const double* T3,
                    int mode, double* M_out, const double* iso_in, double* iso_out);

/* ctm_ts_isometry: the two-stage isometry TS(Q; c1, c2) of P:L60 ("we reshape it to matrix
 * of dimension chi D x chi D ... take the first chi' left singular vectors as U_d^1 ...
 * additional SVD on (chi' D, chi) matrix to obtain U_d^2"), rows a2 (side) and a5
 * (main) of SURVEY 8(a), on a caller tensor:
 *   Q (P, K, B, F) row-major device, P <= chi, K = B = D, F <= chi (the handle's sizing);
 *   stage one: v1 (P, K, n1) = first n1 = min(c1, P K) left singular vectors of Q as
 *              (P K) x (B F);   c1 <= max(chi', chi'');
 *   stage two: v2 (n1, B, n2) = first n2 = min(c2, n1 B) left singular vectors of
 *              Q2 = v1^T Q as (n1 B) x F;   c2 <= chi.
 *   v1_out, v2_out: device, caller-owned.  gaps_host (nullable, 2 doubles): the stage gaps
 *   sigma_n / sigma_{n+1} (+inf where nothing is truncated).
 *   mode CTM_TS_SVD / CTM_TS_BASIS (above).  Synchronises the stream.  The same routine the
 *   move runs for every cut (the a5 parity tests call it on a given M). */
int ctm_ts_isometry(ctm_handle h, const double* Q, int P, int K, int B, int F, int c1, int c2, int mode,
                    double* v1_out, double* v2_out, double* gaps_host);

/* ctm_absorb_truncate: SURVEY rows a6-a8 (Fig 4(b)): ket absorption,
 * v1 truncation, bra absorption, v2 truncation, in six contractions S1..S6.
 *   T      (chi, D, D, chi)      as (in, k_face, b_face, out)
 *   X, Xbra(d, D, D, D, D)       as (s, in, face, out, far)   (chain orientation)
 *   v1_in  (chi, D, chi'), v2_in (chi', D, chi)   isometry of the cut on the in side
 *   v1_out (chi, D, chi'), v2_out(chi', D, chi)   isometry of the cut on the out side
 *   T_out  (chi, D, D, chi)      as (o1, k_far, b_far, o2), NOT normalised.
 * Asynchronous. */
int ctm_absorb_truncate(ctm_handle h, const double* T, const double* X, const double* Xbra,
                        const double* v1_in, const double* v2_in, const double* v1_out,
                        const double* v2_out, double* T_out);

/* ctm_left_move: SURVEY rows a1-a11: two column absorptions, projectors
 * recomputed for each (reading R4); each absorption updates C_a^1, C_b^1, T_a^1,
 * T_b^1, C_a^4, C_b^4 from one snapshot (reading R3) and Frobenius-normalises them
 * (reading R13).  A, B (d,D,D,D,D) as (s,u,l,d,r).
 * iso_in (nullable): inject the main isometries instead of computing them (no reduced
 *   env, no SVD: the contraction-only path).  Layout: for absorption a = 0,1 and cut
 *   c = ab, ba: v1 (chi, D, chi') then v2 (chi', D, chi), back to back.
 * iso_out (nullable): receives the isometries used, same layout.
 * iso_in / iso_out require all env extents == chi.
 * st (nullable, host): timing and statistics. */
int ctm_left_move(ctm_handle h, const double* A, const double* B, ctm_env* env,
                  const double* iso_in, double* iso_out, ctm_move_stats* st);

/* ctm_move: the move in direction dir (CTM_LEFT/RIGHT/UP/DOWN) = relabel the
 * environment by quarter turns (clockwise storage: no data movement), permute the
 * site legs on the device, left move, turn back ("moves in other directions
 * can be adjusted accordingly").  iso_out (nullable): the move's isometries in the rotated
 * (left-move) picture, layout as ctm_left_move's.  ctm_iterate runs n_iter x (left, right,
 * up, down). */
int ctm_move(ctm_handle h, int dir, const double* A, const double* B, ctm_env* env,
             double* iso_out, ctm_move_stats* st);
/* ctm_converge: CTM iterations (left, right, up, down) until the corner spectra move by
 * less than tol between iterations, at most max_iter ("N_CTM ~ 10-30 times, the
 * environment tensors will become sufficiently converged").  Criterion (DESIGN.md reading
 * R22): the singular values of each of the 8 corners, sorted and normalised to unit sum;
 * distance = max over corners of the 1-norm of the difference (zero-padded).  Reports the
 * iterations run and the last distance (host pointers, nullable).  Synchronises the
 * stream. */
int ctm_converge(ctm_handle h, const double* A, const double* B, ctm_env* env, int max_iter, double tol,
                 int* iters_out, double* delta_out, ctm_move_stats* st);

int ctm_iterate(ctm_handle h, const double* A, const double* B, ctm_env* env, int n_iter,
                ctm_move_stats* st);

/* ctm_norm_2x2: <psi|psi> closed on the 2x2 patch of Fig 1(d):
 *     C_a^1 T_a^2 T_b^2 C_b^2 / T_a^1 A B T_b^3 / T_b^1 B A T_a^3 / C_b^4 T_b^4 T_a^4 C_a^3
 * = Tr(E_ul E_ur E_lr E_ll).  out_host: the value.  cancel_ratio_host (nullable): the
 * value divided by the same closure over entrywise |.| (conditioning report).
 * Synchronises the stream. */
int ctm_norm_2x2(ctm_handle h, const double* A, const double* B, const ctm_env* env,
                 double* out_host, double* cancel_ratio_host);

/* ctm_bond_energy: two-site reduced density matrix on the 2x1 (CTM_BOND_H) or 1x2
 * (CTM_BOND_V) window, symmetrised (rho + rho^T)/2 and trace-normalised;
 * e = Tr(rho h) with h (d,d,d,d) = <s_i s_j| h |s_i' s_j'> on the device.
 * rho_out (nullable, device): (d,d,d,d) as (s_A, s_B, t_A, t_B).
 * e_out_host: the energy.  Synchronises the stream. */
/* ctm_site_spins: single-site spin expectations for d = 2 (S = sigma/2), from the H-bond
 * 2x1-window rho by partial trace ("staggered magnetization"; DESIGN.md
 * reading R23).  out_host[5] = <S^x>_A, <S^z>_A, <S^x>_B, <S^z>_B (<S^y> = 0 for real
 * tensors) and the staggered magnetisation m_s = (|<S>_A| + |<S>_B|) / 2, all computed on
 * the device.  Synchronises the stream.  d != 2: CTM_E_UNSUPPORTED. */
int ctm_site_spins(ctm_handle h, const double* A, const double* B, const ctm_env* env, double* out_host);

int ctm_bond_energy(ctm_handle h, const double* A, const double* B, const ctm_env* env,
                    const double* hop, int bond, double* rho_out, double* e_out_host);

/* ---------------------------------------------------------------------------------
 * Imaginary-time evolution with the fast full update ("we used
 * imaginary-time evolution method with a second-order Suzuki-Trotter decomposition ... we
 * applied the fast full update scheme (FFU) ... to avoid recomputing the effective
 * environments after each update step").  Readings R25-R30 fix what the paper
 * leaves to its reference.
 * --------------------------------------------------------------------------------- */
/* ctm_trotter_gate: gate_out (d,d,d,d) device = exp(-delta h) of the bond operator hop
 * (d,d,d,d) device as (s_i, s_j, s_i', s_j') (R25).  Asynchronous.  d^2 <= 16. */
int ctm_trotter_gate(ctm_handle h, const double* hop, double delta, double* gate_out);

/* ctm_bond_update: one FFU update of `bond` (CTM_BOND_H1/H2/V1/V2) of the sites A, B
 * (d,D,D,D,D) device against the environment env (R26 reductions A = X aR, B = bL Y by SVD;
 * R27 bond environment N of the 2x1 window, positivised; R28 gate, truncated-SVD start and
 * `sweeps` ALS sweeps in the N metric, back to bond D).  A_out, B_out (device, same shapes,
 * must not alias A, B) receive the Frobenius-normalised sites.  cost_host (nullable, 2
 * doubles): the final N-weighted error ||aR bL - theta'||_N^2 and <theta'|N|theta'>.
 * Synchronises the stream.  Needs a handle without CTM_FLAG_MOVE_ONLY. */
int ctm_bond_update(ctm_handle h, const double* A, const double* B, const ctm_env* env, const double* gate,
                    int bond, int sweeps, double* A_out, double* B_out, double* cost_host);

/* ctm_trotter_step: one second-order Trotter step (R29) H1(delta/2) H2(delta/2) V1(delta/2)
 * V2(delta) V1(delta/2) H2(delta/2) H1(delta/2) of the bond operator hop, A and B updated in
 * place; refresh != 0: one CTM iteration (left, right, up, down) after every bond update
 * (R30, the fast full update).  cost_host (nullable, 14 doubles): ctm_bond_update's pair per
 * bond update.  Synchronises the stream. */
int ctm_trotter_step(ctm_handle h, double* A, double* B, ctm_env* env, const double* hop, double delta, int sweeps,
                     int refresh, double* cost_host);

/* Algorithmic FP64 flops of one left move for square extents (SURVEY 8(a) closed form):
 * F_move = 2 (2 F_renv + 2 F_chain + 4 F_corner). */
double ctm_move_flops(int d, int D, int chi, int chi_p, int chi_pp);

/* Number of libctm kernels launched since the handle was created (evidence counter). */
int64_t ctm_kernel_count(ctm_handle h);

/* CTM_FLAG_WARM_START (the truncated SVDs of P:L60 / P:L145 across the N_CTM iterations of P:L48): forget
 * every solve site's stored block (the next move starts cold; the
 * device buffers are kept for reuse).  Call it when A, B or the environment are replaced by
 * unrelated ones -- not required for correctness (every solve is certified on its own matrix),
 * only so that a stale block does not cost a failed warm solve.  CTM_OK also without the flag. */
int ctm_warm_reset(ctm_handle h);

#ifdef __cplusplus
}
#endif
#endif /* CTM_H_ */
