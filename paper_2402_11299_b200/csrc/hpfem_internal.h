/*
 * hpfem_internal.h -- interface between the host plan (plan.cpp, g++) and
 * the device kernels (kernels.cu, nvcc).  Plain structs, no torch types.
 */
#ifndef HPFEM_INTERNAL_H_
#define HPFEM_INTERNAL_H_

#include <cuda_runtime.h>

#include "ops1d.h"

namespace hpfem {

/* one 1D direction as seen by the device */
struct DirDev {
  int n;     // elements
  int p;     // degree (bubbles W_0..W_{p-2})
  int bc;    // 0 Dirichlet, 1 Neumann
  int nh;    // kept hats
  int N;     // dofs = nh + nb
  int nb;    // bubbles = (p-1) n
  const double* delta;  // device [n] element widths
  double rob0, rob1;    // Robin alpha at the left / right end (0 = none)
  const double* lw;     // device [N][4] load weights of each dof (k_load_tab), nullptr = computed inline
  const int* lr;        // device [N][4] their Legendre rows (-1 = none)
};

/* Factor tables of one shifted operator S = kap K + sig M of one direction
 * (Alg. 1 in chain + Schur form):
 *   il[b], g[b]  : chain reverse-Cholesky diag^{-1} and sub-diagonal, b = k n + e
 *   vL[b], vR[b] : D_e^{-1} B^T e_{hL(e)}, D_e^{-1} B^T e_{hR(e)} (static condensation)
 *   ilh[t], gh[t]: reverse Cholesky of the hat Schur complement A0 - B D^{-1} B^T
 *   cf           : chain-major copy for the TMA kernels, chain (e, pi) at
 *                  cf + (2e + pi) * cfs, position c at
 *                    [4c] = il_c, [4c+1] = hd_c = g_c il_c, [4c+2] = hu_c = g_{c-1} il_c,
 *                  so that each recurrence step is one dependent FMA,
 *                    y_c = il_c r_c - hd_c y_{c+1},   z_c = il_c y_c - hu_c z_{c-1},
 *                  and [4c+3] = il_c again, so that each sweep reads its two
 *                  factors with one 16-byte load: (il, hd) down, (hu, il) up;
 *                  cfs = 4 roundup8(chain_len(p, 0)) + 2 (spreads smem banks; see
 *                  fac_cfs for chains of more than 64 positions); the
 *                  positions past a chain up to the next multiple of 8 (the TMA
 *                  stage height) hold zero factors, so a stage-padded
 *                  recurrence step there yields exactly 0 with no select.
 * stored contiguously: [il | g | vL | vR | ilh | gh | cf], 256-byte aligned. */
struct FacView {
  const double* il;
  const double* g;
  const double* vL;
  const double* vR;
  const double* ilh;
  const double* gh;
  const double* cf;
  int cfs;
  double kap, sig;
};

/* Chains longer than 64 positions (p > 129) get tables over 128 positions and
 * the spike coefficients of the two-threads-per-chain x half-step (tma_step.cu,
 * k_xstep_tma2) behind them, at cf + fac_spk_off.  A half swept with entry 0
 * differs from the true sweep by the entry times a fixed vector: for c < 64,
 * zeta_c = (L^{-1} beta)_c with beta_63 = -hd_63, beta_c = -hd_c beta_{c+1} (the
 * influence of y_64 on z_c through y_c = a_c + beta_c y_64); for c >= 64,
 * gamma_c with gamma_64 = -hu_64, gamma_c = -hu_c gamma_{c-1} (the influence of
 * z_63 on z_c). */
HD int fac_cf_pos(const DirDev& d) { return d.p / 2 > 64 ? 128 : (d.p / 2 + 7) & ~7; }
HD int fac_spk_off(const DirDev& d) { return 4 * fac_cf_pos(d) + 2; }
HD int fac_cfs(const DirDev& d) { return fac_spk_off(d) + (d.p / 2 > 64 ? 128 : 0); }

HD size_t fac_cf_off(const DirDev& d) {
  size_t s = 4 * (size_t)d.nb + 2 * (size_t)d.nh;
  return (s + 31) & ~(size_t)31;
}

inline size_t fac_stride(const DirDev& d) {
  size_t s = fac_cf_off(d) + (size_t)d.n * 2 * fac_cfs(d);
  return (s + 31) & ~(size_t)31;  // 256-byte aligned sets
}

inline FacView fac_view(const DirDev& d, const double* base, double kap, double sig) {
  FacView f;
  f.il = base;
  f.g = base + d.nb;
  f.vL = base + 2 * (size_t)d.nb;
  f.vR = base + 3 * (size_t)d.nb;
  f.ilh = base + 4 * (size_t)d.nb;
  f.gh = base + 4 * (size_t)d.nb + d.nh;
  f.cf = base + fac_cf_off(d);
  f.cfs = fac_cfs(d);
  f.kap = kap;
  f.sig = sig;
  return f;
}

/* Internal (plan-owned) 2D array layout: row i = x-dof (unpadded), row
 * stride ld doubles, y-hats at columns 0..nh_y-1 and the y-bubbles from
 * column hb on, either
 *   degree-major  (emaj = 0): bubble (k, e) at hb + k np + e   (lanes over
 *                 elements coalesce: the LDG kernels), or
 *   element-major (emaj = 1): bubble (k, e) at hb + e Q + k    (a group of
 *                 whole elements is one contiguous run: the TMA kernels).
 * hb, np, Q and ld are even so every block starts on a 16-byte boundary
 * (DESIGN.md §5). */
struct Layout {
  int ld;
  int hb;
  int np;
  int Q;
  int emaj;
};

inline Layout make_layout(const DirDev& y, int emaj) {
  Layout L;
  // element-major: the bubble blocks and every row start on a 128-byte line
  // (16 doubles), so that the TMA boxes (128-byte rows) and the coalesced
  // stores cover whole 32-byte sectors -- a 16-byte offset made every
  // 128-byte row straddle 5 sectors and forced partial-sector writes
  L.hb = emaj ? (y.nh + 15) & ~15 : (y.nh + 1) & ~1;
  L.np = (y.n + 1) & ~1;
  L.Q = (y.p - 1 + 1) & ~1;
  L.emaj = emaj;
  L.ld = emaj ? (L.hb + y.n * L.Q + 15) & ~15 : L.hb + (y.p - 1) * L.np;
  if (L.ld < 2) L.ld = 2;
  return L;
}

/* Tuning switches, read from the environment ONCE per plan (read_tuning in
 * plan.cpp) and carried with every launch -- no process-wide statics, so
 * plans on several host threads / devices do not race (defaults in
 * parentheses; all are experiment knobs). */
struct Tuning {
  int hat_sms;        // HPFEM_HAT_SMS (-1): SMs the persistent TMA grid leaves to the side-stream hat lines
                      // (0: hat lines serial on the launch stream; < 0: side stream, no SMs reserved --
                      // they fill the bubble kernel's tail; 1, 2, 4, 8 measured the same total at config 5)
  int no_graph;       // HPFEM_NO_GRAPH (0)
  int no_small;       // HPFEM_NO_SMALL (0)
  int no_tma;         // HPFEM_NO_TMA (0)
  int no_wtab;        // HPFEM_NO_WTAB (0)
  int batch_streams;  // HPFEM_BATCH_STREAMS (8)
  int bub_reg;        // HPFEM_BUBBLE_KERNEL=reg (0): register variant of the LDG bubble kernel
  int hat_lb[2];      // HPFEM_HAT_LB_X / _Y (32): lines per hat Schur CTA
  int nst[2];         // HPFEM_NST_X / _Y (4): TMA ring depth
  int eg_y;           // HPFEM_EG_Y (0 = automatic): y-solve tile width
  int fake_stencil;   // HPFEM_FAKE_STENCIL (0): experiment only
  int hats_seq;       // HPFEM_HATS_SEQ (0): the sequential one-thread-per-line hat Schur kernel (experiment / A-B)
  int no_x2;          // HPFEM_NO_X2 (0): long x chains by the one-thread kernel (upper half parked in the output row)
  int no_hat_split;   // HPFEM_NO_HAT_SPLIT (0): hat Schur solves of the side-stream hat lines on the launch stream
  int transpose;      // HPFEM_TRANSPOSE (-1 auto, 0 never, 1 always): solve the transposed equation (R23)
};

/* Raise a kernel's dynamic shared-memory limit to `bytes` on the CURRENT
 * device, once per (kernel, device) (kernels.cu; mutex-protected, so host
 * threads may share the library).  cudaFuncSetAttribute can serialise with
 * in-flight launches of the same kernel, hence the cache. */
cudaError_t smem_optin(const void* func, size_t bytes);

/* cross-line stencil mode of a half-step kernel */
enum StencilMode { ST_NONE = 0, ST_APPLY = 1, ST_CORR = 2 };

/* One line-solve pass: out = S_s^{-1} r along direction `dir` for every line,
 *   r = alphaG * G  +  stencil_o(Xp)
 * ST_APPLY: stencil = -(kap_a K_o + tau M_o) Corr_o      (Alg. 2 apply)
 * ST_CORR : stencil = +Corr_o                            (final W_J C^{-1})
 * Corr_o maps the raw stored array (bubbles z, hats x_h) of the previous
 * solve along o to the true iterate: x_b = z_b - vL x_hL - vR x_hR. */
struct StepParams {
  int dir;  // 0: solve along x (lines = columns), 1: along y (lines = rows)
  int ld;   // internal row stride (Layout.ld)
  Layout lay;
  int lp_begin, lp_count;  // lines processed, in processing order (see row_of)
  DirDev s, o;
  const double* G;
  double alphaG;
  const double* Xp;
  int mode;
  double kap_a, tau;
  const double* cvL;  // correction vectors of the previous solve along o (may be null)
  const double* cvR;
  FacView f;  // factor of this solve
  double* out;
  const double* wtab;  // precomputed stencil weights of the bubble lines (TMA kernels; null = build in-kernel)
  /* element-major layout only (null otherwise): compact copy of the
   * chain-first bubbles (k = 0, 1) of every y-element, [row][n_y][2], i.e.
   * the only bubbles the y-hat rows of the stencil and the hat Schur
   * right-hand side touch -- contiguous instead of 16 bytes out of every Q. */
  double* z01;         // y-solves: written for every row of out
  const double* z01p;  // x-solves: the copy belonging to Xp
  /* hat Schur kernel K5 only: the lines it takes, as processing positions
   * [hl_begin, hl_end) -- y-solves: row positions (row_of: the x-bubble rows
   * first, [0, o.nb), then the x-hat rows); x-solves: internal columns (hats
   * and padding [0, lay.hb), then the y-bubbles).  hl_end <= 0 (e.g. zero-initialised): every line. */
  int hl_begin, hl_end;
  Tuning tun;          // host-side launch choices (not read by the kernels)
};

/* launchers (kernels.cu); return cudaError_t of the launch */
cudaError_t launch_factor(const DirDev& d, const double* kap, const double* sig, int nsets, double* fac,
                          size_t stride, int* err, cudaStream_t st);
cudaError_t launch_step_bubbles(const StepParams& P, cudaStream_t st);
cudaError_t launch_step_hats(const StepParams& P, cudaStream_t st);
/* can launch_step_hats take a sub-range of the lines (hl_begin / hl_end)? */
bool hats_split_ok(const StepParams& P);
cudaError_t launch_hat_lines(const StepParams& P, cudaStream_t st);  // element-major layout only
cudaError_t launch_copyin(const DirDev& x, const DirDev& y, const Layout& L, const double* G, double* Gp,
                          cudaStream_t st);
/* out (C x R) = in (R x C)^T, both row-major and contiguous */
cudaError_t launch_transpose(const double* in, int R, int C, double* out, cudaStream_t st);
cudaError_t launch_finalize(const DirDev& x, const DirDev& y, const Layout& L, const double* vL, const double* vR,
                            const double* X, double* U, cudaStream_t st);
/* 7-slot rows of A = K + (w^2/2) M and of M of one direction, slot-major
 * [7][N]: idx (-1 = absent), wA, wM = -(row entries) (0 where absent) */
struct ApplyTab {
  const int* idx;
  const double* wA;
  const double* wM;
};
cudaError_t launch_apply_tab(const DirDev& o, double omega, const ApplyTab& t, cudaStream_t st);
/* tx / ty: the plan's tables (null: stencils built per output, the round-1 kernel) */
cudaError_t launch_apply2d(const DirDev& x, const DirDev& y, double omega, const double* U, double* F,
                           cudaStream_t st, const ApplyTab* tx = nullptr, const ApplyTab* ty = nullptr);
/* accumulate = 1: G += load(Fleg) (the variable-coefficient operator adds
 * its Hadamard term onto hpfem_apply's output) */
cudaError_t launch_load_tab(const DirDev& d, int* r, double* w, cudaStream_t st);
cudaError_t launch_load2d(const DirDev& x, const DirDev& y, const double* Fleg, double* G, cudaStream_t st,
                          int accumulate = 0, double scale = 1.0);  // G (+)= scale * load(Fleg)
cudaError_t launch_solve1d(const DirDev& d, const FacView& f, int nrhs, const double* F, double* U,
                           cudaStream_t st);  // solve1d.cu
/* dx = 1: Legendre coefficients of du/dx instead of u (NEXT-4) */
cudaError_t launch_unload2d(const DirDev& x, const DirDev& y, const double* U, double* Cleg, cudaStream_t st,
                            int dx = 0);

/* K11 (kernels.cu): whole ADI solve of one small problem per CTA in shared memory */
struct SmallArgs {
  DirDev x, y;
  const double* fx;  // factor sets (plan layout), stride sx / sy doubles
  const double* fy;
  size_t sx, sy;
  const double* sh;   // [kap_x | sig_x | kap_y | sig_y] (J+1 each)
  const double* tau;  // [tau_A (J) | tau_B (J)]: apply shifts hw2 - p_j, hw2 + q_j
  int J, iters;
  const double* F;
  double* U;
};
size_t small_smem_bytes(const DirDev& x, const DirDev& y);
constexpr size_t SMALL_SMEM_MAX = 200 * 1024;
cudaError_t launch_adi_small(const SmallArgs& a, int batch, cudaStream_t st);

/* NEXT-3 (varcoef.cu): one 1D pass of a grid <-> Legendre transform,
 *   out[base(c) + k s] = [h[o] + alpha *] [g[o] *] sum_i A[k K + i] in[base(c) + i s],
 *   base(c) = (c / nb) bs + c % nb,  c < ncols,  k < M,  i < K. */
struct ElemApply {
  const double* A;
  int M, K;
  const double* in;
  double* out;
  const double* g;  // optional Hadamard factor at the output address (null = none)
  const double* h;  // optional: out = h[o] + alpha * acc * g[o] (NEXT-4 explicit Euler step; needs g)
  double alpha;
  long long ncols, nb, bs, s;
};
enum { CG_RZ = 0, CG_A = 1, CG_B = 2, CG_RRV = 3, CG_NSC = 4 };      // device scalar slots
enum { CG_RZ0 = 0, CG_ALPHA = 1, CG_RR = 2, CG_BETA = 3 };            // k_cg_scalar ops
constexpr int CG_BLOCKS = 296;                                       // 2 x 148 SMs
cudaError_t launch_elem_apply(const ElemApply& E, cudaStream_t st);
cudaError_t launch_dot(const double* a, const double* b, size_t n, double* partial, double* sc, int op,
                       cudaStream_t st);
cudaError_t launch_cg_xr(double* x, double* r, const double* p, const double* q, size_t n, double* partial,
                         double* sc, cudaStream_t st);
cudaError_t launch_cg_p(double* p, const double* z, size_t n, const double* sc, int first, cudaStream_t st);

}  // namespace hpfem

#endif
