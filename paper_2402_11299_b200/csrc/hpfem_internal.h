/*
 * hpfem_internal.h -- interface between the host plan (plan.cpp, g++) and
 * the device kernels (kernels.cu, nvcc).  Plain structs, no torch types.
 */
#ifndef HPFEM_INTERNAL_H_
#define HPFEM_INTERNAL_H_

#include <cuda_runtime.h>

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
};

/* Factor tables of one shifted operator S = kap K + sig M of one direction
 * (Alg. 1 in chain + Schur form):
 *   il[b], g[b]  : chain reverse-Cholesky diag^{-1} and sub-diagonal, b = k n + e
 *   vL[b], vR[b] : D_e^{-1} B^T e_{hL(e)}, D_e^{-1} B^T e_{hR(e)} (static condensation)
 *   ilh[t], gh[t]: reverse Cholesky of the hat Schur complement A0 - B D^{-1} B^T
 * stored contiguously: [il | g | vL | vR | ilh | gh], stride = 4 nb + 2 nh (+pad). */
struct FacView {
  const double* il;
  const double* g;
  const double* vL;
  const double* vR;
  const double* ilh;
  const double* gh;
  double kap, sig;
};

inline size_t fac_stride(const DirDev& d) {
  size_t s = 4 * (size_t)d.nb + 2 * (size_t)d.nh;
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
  f.kap = kap;
  f.sig = sig;
  return f;
}

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
  int ld;   // N_y
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
};

/* launchers (kernels.cu); return cudaError_t of the launch */
cudaError_t launch_factor(const DirDev& d, const double* kap, const double* sig, int nsets, double* fac,
                          size_t stride, int* err, cudaStream_t st);
cudaError_t launch_step_bubbles(const StepParams& P, cudaStream_t st);
cudaError_t launch_step_hats(const StepParams& P, cudaStream_t st);
cudaError_t launch_correct_rows(const DirDev& y, int Nx, const double* vL, const double* vR, double* U,
                                cudaStream_t st);
cudaError_t launch_apply2d(const DirDev& x, const DirDev& y, double omega, const double* U, double* F,
                           cudaStream_t st);
cudaError_t launch_load2d(const DirDev& x, const DirDev& y, const double* Fleg, double* G, cudaStream_t st);

}  // namespace hpfem

#endif
