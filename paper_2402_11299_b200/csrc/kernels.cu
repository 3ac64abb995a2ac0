/*
 * kernels.cu -- fp64 device kernels of the ADI hp-FEM solve for sm_100a.
 *
 * The path is banded / tridiagonal recurrence work with ~0.65 flop per byte
 * (DESIGN.md "Roofline"), so it is bound by HBM bandwidth and latency, not
 * by any tensor pipe: no tcgen05 / TMEM here by design.
 *
 *   K1  k_factor_chains / k_factor_hats  Alg. 1 for a batch of
 *       shifted operators S = kap K + sig M: per (shift, element, parity)
 *       bubble chain reverse Cholesky, the static-condensation vectors
 *       v = D_e^{-1} B^T e_h, and the hat Schur complement A0 - B D^{-1} B^T
 *       factored by reverse Cholesky.
 *   K2+K3+K4  k_bubbles<DIR,CL>: one pass over all lines of a half-step of
 *       Alg. 2: the cross-line sparse apply of the other
 *       direction is evaluated on the loads (K3 fused into K2/K4), then the
 *       element-local bubble solve z = D_e^{-1} r_b runs in registers
 *       (Cor. 4.3 P:L600-L614 in static-condensation form).
 *   K5  k_hats<DIR>: per line, hat RHS r_h - B z and the hat tridiagonal
 *       solve; the bubble correction x_b = z - v x_h is deferred into the
 *       consumer's loads (the next half-step's stencil, or K6).
 *   K6  k_correct_rows: materialises U = W_J C^{-1}.
 *   K7  k_apply2d: F = A_x U M_y + M_x U A_y.     K8 k_load2d: G = R^T M_P F M_P R.
 */
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "hpfem_internal.h"
#include "ops1d.h"
#include "ptx.cuh"

namespace hpfem {

cudaError_t smem_optin(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> opted-in bytes
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

/* ------------------------------------------------------------------ */
/* K1: factorisation of a batch of shifted 1D operators               */
/* ------------------------------------------------------------------ */
__device__ void report(int* err, int code, int set, int where, int k) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = set;
    err[2] = where;
    err[3] = k;
  }
}

__global__ void k_factor_chains(DirDev d, const double* __restrict__ kap, const double* __restrict__ sig, int nsets,
                                double* __restrict__ fac, size_t stride, int* err) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= nsets * d.n * 2) return;
  const int e = tid % d.n;
  const int pi = (tid / d.n) & 1;
  const int s = tid / (2 * d.n);
  const int m = chain_len(d.p, pi);
  if (m == 0) return;
  const double K = kap[s], S = sig[s], delta = d.delta[e];
  double* base = fac + (size_t)s * stride;
  double* il = base;
  double* g = base + d.nb;
  double* vL = base + 2 * (size_t)d.nb;
  double* vR = base + 3 * (size_t)d.nb;
  // chain T = L^T L, L lower bidiagonal (diag l_c, sub g_c = L[c+1,c]),
  // bottom-up (reverse Cholesky): l_{m-1} = sqrt(a_{m-1});
  // g_c = b_c / l_{c+1}; l_c = sqrt(a_c - g_c^2)
  double lnext = 0.0;
  for (int c = m - 1; c >= 0; --c) {
    const int k = pi + 2 * c;
    const int b = k * d.n + e;
    double a = s_bub_diag(K, S, delta, k);
    double gc = 0.0;
    if (c < m - 1) {
      gc = s_bub_off(S, delta, k) / lnext;
      a -= gc * gc;
    }
    if (!(a > 0.0) || !isfinite(a)) {
      report(err, 1, s, e, k);
      a = 1.0;
    }
    const double l = sqrt(a);
    il[b] = 1.0 / l;
    g[b] = gc;
    lnext = l;
  }
  {  // chain-major (il, g il, g_prev il, il) for the TMA kernels (hpfem_internal.h)
    double* cf = base + fac_cf_off(d) + (size_t)(2 * e + pi) * fac_cfs(d);
    double gprev = 0.0;
    for (int c = 0; c < m; ++c) {
      const int b = (pi + 2 * c) * d.n + e;
      cf[4 * c] = il[b];
      cf[4 * c + 1] = g[b] * il[b];
      cf[4 * c + 2] = gprev * il[b];
      cf[4 * c + 3] = il[b];
      gprev = g[b];
    }
    if (d.p / 2 > 64) {  // spike coefficients of the two-threads-per-chain x half-step (hpfem_internal.h)
      double* spk = cf + fac_spk_off(d);
      double bt = 1.0;
      for (int c = 63; c >= 0; --c) {
        bt = c < m ? -cf[4 * c + 1] * bt : 0.0;
        spk[c] = bt;
      }
      double zt = 0.0;  // zeta = L^{-1} beta (lower half): the entry's influence on z_c
      for (int c = 0; c < 64; ++c) {
        zt = fma(-cf[4 * c + 2], zt, cf[4 * c] * spk[c]);
        spk[c] = zt;
      }
      double gm = 1.0;
      for (int c = 64; c < 128; ++c) {
        gm = c < m ? -cf[4 * c + 2] * gm : 0.0;
        spk[c] = gm;
      }
    }
  }
  // v_side = T^{-1} (beta e_0): the chain-first bubble is the only one
  // coupled to the hats (W_0 / W_1, ops1d.h)
  for (int side = 0; side < 2; ++side) {
    const int h = hat_of_node(e + side, d.n, d.bc);
    const double beta = (h >= 0) ? s_hat_bub(S, delta, side, pi) : 0.0;
    double* v = side ? vR : vL;
    const int b0 = pi * d.n + e;
    double z = beta * il[b0] * il[b0];
    v[b0] = z;
    int bprev = b0;
    for (int c = 1; c < m; ++c) {
      const int b = (pi + 2 * c) * d.n + e;
      z = -g[bprev] * z * il[b];
      v[b] = z;
      bprev = b;
    }
  }
}

__device__ double schur_elem(const DirDev& d, double S, const double* vv, int e, int side_row) {
  // (B D^{-1} B^T)[h_row, h_col] restricted to element e: sum_k B[h_row, W_k] v_col[k]
  const double delta = d.delta[e];
  double acc = s_hat_bub(S, delta, side_row, 0) * vv[e];
  if (d.p - 2 >= 1) acc += s_hat_bub(S, delta, side_row, 1) * vv[d.n + e];
  return acc;
}

__global__ void k_factor_hats(DirDev d, const double* __restrict__ kap, const double* __restrict__ sig, int nsets,
                              double* __restrict__ fac, size_t stride, int* err) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsets || d.nh == 0) return;
  const double K = kap[s], S = sig[s];
  double* base = fac + (size_t)s * stride;
  const double* vL = base + 2 * (size_t)d.nb;
  const double* vR = base + 3 * (size_t)d.nb;
  double* ilh = base + 4 * (size_t)d.nb;
  double* gh = ilh + d.nh;
  double lnext = 0.0;
  for (int t = d.nh - 1; t >= 0; --t) {
    const int node = node_of_hat(t, d.bc);
    const int eL = node - 1, eR = node;
    double diag = 0.0;
    if (eL >= 0) diag += s_hat_diag_elem(K, S, d.delta[eL]) - schur_elem(d, S, vR, eL, 1);
    if (eR <= d.n - 1) diag += s_hat_diag_elem(K, S, d.delta[eR]) - schur_elem(d, S, vL, eR, 0);
    if (node == 0) diag += K * d.rob0;  // Robin boundary term alpha h(a)^2
    if (node == d.n) diag += K * d.rob1;
    double gc = 0.0;
    if (t < d.nh - 1) {
      // A~0(t, t+1): element eR lies between the two nodes; t is its left hat
      const double off = s_hat_off_elem(K, S, d.delta[eR]) - schur_elem(d, S, vR, eR, 0);
      gc = off / lnext;
      diag -= gc * gc;
    }
    if (!(diag > 0.0) || !isfinite(diag)) {
      report(err, 2, s, t, -1);
      diag = 1.0;
    }
    const double l = sqrt(diag);
    ilh[t] = 1.0 / l;
    gh[t] = gc;
    lnext = l;
  }
}

cudaError_t launch_factor(const DirDev& d, const double* kap, const double* sig, int nsets, double* fac,
                          size_t stride, int* err, cudaStream_t st) {
  const int nthr = nsets * d.n * 2;
  k_factor_chains<<<(nthr + 127) / 128, 128, 0, st>>>(d, kap, sig, nsets, fac, stride, err);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_factor_hats<<<(nsets + 31) / 32, 32, 0, st>>>(d, kap, sig, nsets, fac, stride, err);
  return cudaGetLastError();
}

/* ------------------------------------------------------------------ */
/* Cross-line stencil: row l (in direction o) of  -S_o Corr_o  (apply) */
/* or +Corr_o (final), as 7 fixed slots so it stays in registers.      */
/* Bubble row (k,e): [l, l-2n, l+2n, hL(e), hR(e), -, -]               */
/* Hat row t      : [t, t-1, t+1, (0,eL), (1,eL), (0,eR), (1,eR)]      */
/* ------------------------------------------------------------------ */
struct Stencil {
  int idx[7];
  double w[7];
};

__device__ __forceinline__ void stencil_build(const DirDev& o, int l, int mode, double kap, double tau,
                                              const double* __restrict__ cvL, const double* __restrict__ cvR,
                                              Stencil& st) {
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    st.idx[q] = -1;
    st.w[q] = 0.0;
  }
  if (mode == ST_NONE) return;
  const int n = o.n, nh = o.nh;
  if (l >= nh) {
    const int b = l - nh;
    const int k = b / n;
    const int e = b - k * n;
    const int hL = hat_of_node(e, n, o.bc), hR = hat_of_node(e + 1, n, o.bc);
    if (mode == ST_CORR) {
      st.idx[0] = l;
      st.w[0] = 1.0;
      if (hL >= 0 && cvL) { st.idx[3] = hL; st.w[3] = -cvL[b]; }
      if (hR >= 0 && cvR) { st.idx[4] = hR; st.w[4] = -cvR[b]; }
      return;
    }
    const double dl = o.delta[e];
    const bool hm = k >= 2, hp = k + 2 <= o.p - 2;
    const double sd = s_bub_diag(kap, tau, dl, k);
    const double sm = hm ? s_bub_off(tau, dl, k - 2) : 0.0;
    const double sp = hp ? s_bub_off(tau, dl, k) : 0.0;
    double cL = s_hat_bub(tau, dl, 0, k), cR = s_hat_bub(tau, dl, 1, k);
    if (cvL) {
      cL -= sd * cvL[b];
      if (hm) cL -= sm * cvL[b - 2 * n];
      if (hp) cL -= sp * cvL[b + 2 * n];
    }
    if (cvR) {
      cR -= sd * cvR[b];
      if (hm) cR -= sm * cvR[b - 2 * n];
      if (hp) cR -= sp * cvR[b + 2 * n];
    }
    st.idx[0] = l; st.w[0] = -sd;
    if (hm) { st.idx[1] = l - 2 * n; st.w[1] = -sm; }
    if (hp) { st.idx[2] = l + 2 * n; st.w[2] = -sp; }
    if (hL >= 0) { st.idx[3] = hL; st.w[3] = -cL; }
    if (hR >= 0) { st.idx[4] = hR; st.w[4] = -cR; }
  } else {
    const int t = l;
    if (mode == ST_CORR) {
      st.idx[0] = t;
      st.w[0] = 1.0;
      return;
    }
    const int node = node_of_hat(t, o.bc);
    const int eL = node - 1, eR = node;
    const bool k1 = o.p - 2 >= 1;
    double ctt = 0.0, ctm = 0.0, ctp = 0.0;
    bool has_m = false, has_p = false;
    if (eL >= 0) {
      const double dl = o.delta[eL];
      ctt += s_hat_diag_elem(kap, tau, dl);
      has_m = hat_of_node(node - 1, n, o.bc) >= 0;
      if (has_m) ctm += s_hat_off_elem(kap, tau, dl);
      const double s0 = s_hat_bub(tau, dl, 1, 0), s1 = k1 ? s_hat_bub(tau, dl, 1, 1) : 0.0;
      st.idx[3] = nh + eL; st.w[3] = -s0;
      if (k1) { st.idx[4] = nh + n + eL; st.w[4] = -s1; }
      if (cvR) ctt -= s0 * cvR[eL] + (k1 ? s1 * cvR[n + eL] : 0.0);
      if (cvL && has_m) ctm -= s0 * cvL[eL] + (k1 ? s1 * cvL[n + eL] : 0.0);
    }
    if (eR <= n - 1) {
      const double dr = o.delta[eR];
      ctt += s_hat_diag_elem(kap, tau, dr);
      has_p = hat_of_node(node + 1, n, o.bc) >= 0;
      if (has_p) ctp += s_hat_off_elem(kap, tau, dr);
      const double s0 = s_hat_bub(tau, dr, 0, 0), s1 = k1 ? s_hat_bub(tau, dr, 0, 1) : 0.0;
      st.idx[5] = nh + eR; st.w[5] = -s0;
      if (k1) { st.idx[6] = nh + n + eR; st.w[6] = -s1; }
      if (cvL) ctt -= s0 * cvL[eR] + (k1 ? s1 * cvL[n + eR] : 0.0);
      if (cvR && has_p) ctp -= s0 * cvR[eR] + (k1 ? s1 * cvR[n + eR] : 0.0);
    }
    if (node == 0) ctt += kap * o.rob0;  // Robin boundary term
    if (node == n) ctt += kap * o.rob1;
    st.idx[0] = t; st.w[0] = -ctt;
    if (has_m) { st.idx[1] = t - 1; st.w[1] = -ctm; }
    if (has_p) { st.idx[2] = t + 1; st.w[2] = -ctp; }
  }
}

/* the stencil rows of HAT row t alone (the idx[] stencil_build gives for
 * l = t < nh), without the weights' floating-point work */
__device__ __forceinline__ void hat_row_idx(const DirDev& o, int t, int mode, int* idx) {
#pragma unroll
  for (int q = 0; q < 7; ++q) idx[q] = -1;
  if (mode == ST_NONE) return;
  idx[0] = t;
  if (mode == ST_CORR) return;
  const int n = o.n, nh = o.nh;
  const int node = node_of_hat(t, o.bc);
  const int eL = node - 1, eR = node;
  const bool k1 = o.p - 2 >= 1;
  if (eL >= 0) {
    if (hat_of_node(node - 1, n, o.bc) >= 0) idx[1] = t - 1;
    idx[3] = nh + eL;
    if (k1) idx[4] = nh + n + eL;
  }
  if (eR <= n - 1) {
    if (hat_of_node(node + 1, n, o.bc) >= 0) idx[2] = t + 1;
    idx[5] = nh + eR;
    if (k1) idx[6] = nh + n + eR;
  }
}

/* internal column of y-dof d */
__host__ __device__ __forceinline__ int ycol_ke(const Layout& L, int k, int e) {
  return L.emaj ? L.hb + e * L.Q + k : L.hb + k * L.np + e;
}
__host__ __device__ __forceinline__ int ycol(const Layout& L, const DirDev& y, int d) {
  if (d < y.nh) return d;
  const int b = d - y.nh, k = b / y.n;
  return ycol_ke(L, k, b - k * y.n);
}

/* y-dof stored at internal column li, -1 for padding columns */
__device__ __forceinline__ int ydof_of_col(const Layout& L, const DirDev& y, int li) {
  if (li < y.nh) return li;
  if (li < L.hb) return -1;
  const int b = li - L.hb;
  int k, e;
  if (L.emaj) {
    e = b / L.Q;
    k = b - e * L.Q;
  } else {
    k = b / L.np;
    e = b - k * L.np;
  }
  if (e >= y.n || k >= y.p - 1) return -1;
  return y.nh + k * y.n + e;
}

/* Address of (line l, dof position d) for a solve along DIR, both already in
 * internal coordinates: DIR 0 -> l is a column, d a row; DIR 1 -> l is a
 * row, d a column. */
template <int DIR>
__device__ __forceinline__ size_t addr(int l, int d, int ld) {
  return DIR == 0 ? (size_t)d * ld + l : (size_t)l * ld + d;
}

/* internal position of the solve-direction dof (bubble (k, e) or hat t) */
template <int DIR>
__device__ __forceinline__ int spos_bub(const StepParams& P, int k, int e) {
  return DIR == 0 ? P.s.nh + k * P.s.n + e : ycol_ke(P.lay, k, e);
}

/* r(l, d) = alphaG G(l,d) + sum_q w_q Xp(idx_q, d)   (read-only inputs) */
template <int DIR>
__device__ __forceinline__ double rhs_at(const double* __restrict__ G, double alphaG, const double* __restrict__ Xp,
                                         const Stencil& st, int l, int d, int ld) {
  double acc = 0.0;
  if (alphaG != 0.0) acc = alphaG * __ldg(G + addr<DIR>(l, d, ld));
#pragma unroll
  for (int q = 0; q < 7; ++q)
    if (st.idx[q] >= 0) acc += st.w[q] * __ldg(Xp + addr<DIR>(st.idx[q], d, ld));
  return acc;
}

/* Line processing order of the y-solve (lines = rows): rows that are
 * x-neighbours in the apply stencil (same x-element, degrees k, k+-2) are
 * processed back to back so their W rows are reused from L2; hat rows last. */
__device__ __forceinline__ int row_of(const DirDev& o, int lp) {
  const int nb = o.nb, q = o.p - 1;
  if (lp >= nb) return lp - nb;
  const int e = lp / q, k = lp - e * q;
  return o.nh + k * o.n + e;
}

/* line dof index (in direction o) of processing position lp */
template <int DIR>
__device__ __forceinline__ int line_dof(const StepParams& P, int lp) {
  return DIR == 0 ? lp : row_of(P.o, lp);
}

/* Stencil for line l (a dof of direction o) with its indices mapped to
 * internal coordinates (columns for DIR 0, rows for DIR 1). */
template <int DIR>
__device__ __forceinline__ void line_stencil(const StepParams& P, int l, Stencil& st) {
  stencil_build(P.o, l, P.mode, P.kap_a, P.tau, P.cvL, P.cvR, st);
  if (DIR == 0) {
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (st.idx[q] >= 0) st.idx[q] = ycol(P.lay, P.o, st.idx[q]);
  }
}

/* thread -> (internal line coordinate li, line dof l, element e, parity pi) */
template <int DIR>
__device__ __forceinline__ bool thread_coords(const StepParams& P, int& li, int& l, int& e, int& pi) {
  const int n = P.s.n;
  int lp;
  if (DIR == 0) {
    lp = blockIdx.x * blockDim.x + threadIdx.x;
    e = blockIdx.y % n;
    pi = blockIdx.y / n;
  } else {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    e = (int)(idx % n);
    pi = (int)((idx / n) & 1);
    lp = (int)(idx / (2 * n));
  }
  if (lp >= P.lp_count) return false;
  lp += P.lp_begin;
  l = line_dof<DIR>(P, lp);
  li = DIR == 0 ? ycol(P.lay, P.o, l) : l;
  return true;
}

/* K2/K3/K4, register variant: chain kept in registers (CL <= 64). */
template <int DIR, int CL>
__global__ void __launch_bounds__(128) k_bubbles_reg(StepParams P) {
  int li, l, e, pi;
  if (!thread_coords<DIR>(P, li, l, e, pi)) return;
  const DirDev& s = P.s;
  const int m = chain_len(s.p, pi);
  if (m == 0) return;
  Stencil st;
  line_stencil<DIR>(P, l, st);
  double r[CL];
#pragma unroll
  for (int c = 0; c < CL; ++c)
    if (c < m) r[c] = rhs_at<DIR>(P.G, P.alphaG, P.Xp, st, li, spos_bub<DIR>(P, pi + 2 * c, e), P.ld);
  const double* __restrict__ il = P.f.il;
  const double* __restrict__ g = P.f.g;
  double y = 0.0;
#pragma unroll
  for (int c = CL - 1; c >= 0; --c)
    if (c < m) {
      const int b = (pi + 2 * c) * s.n + e;
      y = (r[c] - __ldg(g + b) * y) * __ldg(il + b);
      r[c] = y;
    }
  double z = 0.0, gp = 0.0;
#pragma unroll
  for (int c = 0; c < CL; ++c)
    if (c < m) {
      const int b = (pi + 2 * c) * s.n + e;
      z = (r[c] - gp * z) * __ldg(il + b);
      gp = __ldg(g + b);
      P.out[addr<DIR>(li, spos_bub<DIR>(P, pi + 2 * c, e), P.ld)] = z;
    }
}

/* K2/K3/K4, streaming variant (default): the apply is evaluated on the
 * loads while the chain is swept from its top degree down (L^T y = r), y is
 * parked in the output array -- at this occupancy the round trip stays in
 * L2 (~(resident chains) x 8m bytes << 126 MB), so DRAM sees one write --
 * and the ascending sweep (L z = y) overwrites it with z = D_e^{-1} r.
 * Loads are batched U chain positions at a time for memory-level
 * parallelism; ~70 registers instead of ~170. */
template <int DIR, int U>
__global__ void __launch_bounds__(256) k_bubbles(StepParams P) {
  int li, l, e, pi;
  if (!thread_coords<DIR>(P, li, l, e, pi)) return;
  const DirDev& s = P.s;
  const int m = chain_len(s.p, pi);
  if (m == 0) return;
  Stencil st;
  line_stencil<DIR>(P, l, st);
  const double* __restrict__ G = P.G;
  const double* __restrict__ Xp = P.Xp;
  const double* __restrict__ il = P.f.il;
  const double* __restrict__ g = P.f.g;
  double* __restrict__ out = P.out;
  const double aG = P.alphaG;
  const int n = s.n, ld = P.ld;
  double y = 0.0;
  for (int c0 = m - 1; c0 >= 0; c0 -= U) {
    double r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 - u;
      r[u] = c >= 0 ? rhs_at<DIR>(G, aG, Xp, st, li, spos_bub<DIR>(P, pi + 2 * c, e), ld) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 - u;
      if (c >= 0) {
        const int b = (pi + 2 * c) * n + e;
        y = (r[u] - __ldg(g + b) * y) * __ldg(il + b);
        out[addr<DIR>(li, spos_bub<DIR>(P, pi + 2 * c, e), ld)] = y;
      }
    }
  }
  double z = 0.0, gp = 0.0;
  for (int c0 = 0; c0 < m; c0 += U) {
    double yy[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      yy[u] = c < m ? out[addr<DIR>(li, spos_bub<DIR>(P, pi + 2 * c, e), ld)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      if (c < m) {
        const int b = (pi + 2 * c) * n + e;
        z = (yy[u] - gp * z) * __ldg(il + b);
        gp = __ldg(g + b);
        out[addr<DIR>(li, spos_bub<DIR>(P, pi + 2 * c, e), ld)] = z;
      }
    }
  }
}

/* K5: hat right-hand side r_h - B z for a tile of LB lines (parallel over
 * hats), then the hat tridiagonal reverse-Cholesky solve of each line from
 * shared memory, then the write-back.
 * smem: [nh][LB] values, hat factors il/g [nh] each, the per-hat coupling
 * coefficients B(h, W_0/W_1) of the left/right element [nh][4] (0 for an
 * absent element, whose index is clamped to the present one so that every
 * load is unconditional and issued ahead of the FMAs), (DIR 1) the LB row
 * stencils, then the int tables (elements [nh][2], stencil indices [LB][7]). */
__host__ __device__ constexpr size_t hats_smem_doubles(int nh, int LB) {
  return (size_t)nh * (LB + 6) + 7 * (size_t)LB + ((size_t)nh * 2 + 7 * (size_t)LB + 1) / 2;
}

template <int DIR, int LB>
__global__ void __launch_bounds__(256, 4) k_hats(StepParams P) {
  extern __shared__ double sh[];
  const DirDev& s = P.s;
  const int nh = s.nh, ld = P.ld, n = s.n;
  const int l0 = blockIdx.x * LB;  // first line (processing position) of the tile
  const double S = P.f.sig;
  const bool k1 = s.p - 2 >= 1;  // bubble W_1 exists (uniform)
  const double* __restrict__ G = P.G;
  const double* __restrict__ Xp = P.Xp;
  const double* __restrict__ out_r = P.out;  // chain-first bubbles of this half-step (read-only here)
  double* fil = sh + (size_t)nh * LB;
  double* fg = fil + nh;
  double* hz = fg + nh;
  double* stw = hz + 4 * (size_t)nh;
  int* hzi = reinterpret_cast<int*>(stw + 7 * LB);
  int* sti = hzi + 2 * nh;
  // phase 0: hat factors, coupling tables, (DIR 1) row stencils
  for (int t = threadIdx.x; t < nh; t += blockDim.x) {
    fil[t] = __ldg(P.f.ilh + t);
    fg[t] = __ldg(P.f.gh + t);
    const int node = node_of_hat(t, s.bc);
    const int eL = node - 1, eR = node;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if (eL >= 0) {
      const double dl = s.delta[eL];
      c0 = s_hat_bub(S, dl, 1, 0);
      if (k1) c1 = s_hat_bub(S, dl, 1, 1);
    }
    if (eR <= n - 1) {
      const double dr = s.delta[eR];
      c2 = s_hat_bub(S, dr, 0, 0);
      if (k1) c3 = s_hat_bub(S, dr, 0, 1);
    }
    hz[4 * t] = c0;
    hz[4 * t + 1] = c1;
    hz[4 * t + 2] = c2;
    hz[4 * t + 3] = c3;
    hzi[2 * t] = eL >= 0 ? eL : eR;
    hzi[2 * t + 1] = eR <= n - 1 ? eR : eL;
  }
  if (DIR == 1 && (int)threadIdx.x < LB) {
    const int lp = l0 + threadIdx.x;
    Stencil st;
    if (lp < P.o.N) {
      line_stencil<DIR>(P, row_of(P.o, lp), st);
    } else {
#pragma unroll
      for (int q = 0; q < 7; ++q) { st.idx[q] = -1; st.w[q] = 0.0; }
    }
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      sti[threadIdx.x * 7 + q] = st.idx[q];
      stw[threadIdx.x * 7 + q] = st.w[q];
    }
  }
  __syncthreads();
  // r_h - B z, B z = c0 z0(eL) + c1 z1(eL) + c2 z0(eR) + c3 z1(eR) (same order as before)
  auto coupling = [&](double rh, int t, double zl0, double zl1, double zr0, double zr1) {
    rh -= hz[4 * t] * zl0;
    if (k1) rh -= hz[4 * t + 1] * zl1;
    rh -= hz[4 * t + 2] * zr0;
    if (k1) rh -= hz[4 * t + 3] * zr1;
    return rh;
  };
  if (DIR == 0) {
    // lines = columns, taken in internal-column order: lane -> column (coalesced)
    const int j = threadIdx.x % LB, tg = threadIdx.x / LB, ng = blockDim.x / LB;
    const int li = l0 + j;
    const int l = li < ld ? ydof_of_col(P.lay, P.o, li) : -1;
    if (l >= 0) {
      Stencil st;
      line_stencil<DIR>(P, l, st);
#pragma unroll 2
      for (int t = tg; t < nh; t += ng) {
        const int eL = hzi[2 * t], eR = hzi[2 * t + 1];
        const double zl0 = __ldg(out_r + addr<DIR>(li, spos_bub<DIR>(P, 0, eL), ld));
        const double zr0 = __ldg(out_r + addr<DIR>(li, spos_bub<DIR>(P, 0, eR), ld));
        const double zl1 = k1 ? __ldg(out_r + addr<DIR>(li, spos_bub<DIR>(P, 1, eL), ld)) : 0.0;
        const double zr1 = k1 ? __ldg(out_r + addr<DIR>(li, spos_bub<DIR>(P, 1, eR), ld)) : 0.0;
        sh[t * LB + j] = coupling(rhs_at<DIR>(G, P.alphaG, Xp, st, li, t, ld), t, zl0, zl1, zr0, zr1);
      }
    }
  } else {
    // lines = rows; the LB x nh (row, hat) items are spread over all threads
    // (row-major: a warp reads contiguous hat columns of one or two rows)
    int j = threadIdx.x / nh, t = threadIdx.x - j * nh;
    for (; j < LB; t += blockDim.x) {
      while (t >= nh) { t -= nh; ++j; }
      if (j >= LB) break;
      const int lp = l0 + j;
      if (lp >= P.o.N) break;
      const int l = row_of(P.o, lp);
      const int eL = hzi[2 * t], eR = hzi[2 * t + 1];
      double zl0, zl1 = 0.0, zr0, zr1 = 0.0;
      if (P.z01) {  // chain-first bubbles from the compact copy
        const double* zr = P.z01 + (size_t)l * 2 * n;
        const double2 vl = __ldg(reinterpret_cast<const double2*>(zr + 2 * eL));
        const double2 vr = __ldg(reinterpret_cast<const double2*>(zr + 2 * eR));
        zl0 = vl.x; zl1 = vl.y; zr0 = vr.x; zr1 = vr.y;
      } else {
        zl0 = __ldg(out_r + addr<DIR>(l, spos_bub<DIR>(P, 0, eL), ld));
        zr0 = __ldg(out_r + addr<DIR>(l, spos_bub<DIR>(P, 0, eR), ld));
        if (k1) {
          zl1 = __ldg(out_r + addr<DIR>(l, spos_bub<DIR>(P, 1, eL), ld));
          zr1 = __ldg(out_r + addr<DIR>(l, spos_bub<DIR>(P, 1, eR), ld));
        }
      }
      double rh = P.alphaG != 0.0 ? P.alphaG * __ldg(G + addr<DIR>(l, t, ld)) : 0.0;
      const int* si = sti + 7 * j;
      const double* sw = stw + 7 * j;
#pragma unroll
      for (int q = 0; q < 7; ++q)
        if (si[q] >= 0) rh += sw[q] * __ldg(Xp + addr<DIR>(si[q], t, ld));
      sh[t * LB + j] = coupling(rh, t, zl0, zl1, zr0, zr1);
    }
  }
  __syncthreads();
  // sequential tridiagonal reverse-Cholesky solve per line, in shared memory;
  // loads batched HB positions ahead so that only the dependent FMA
  //   y_t = il_t r_t - (g_t il_t) y_{t+1},   x_t = il_t y_t - (g_{t-1} il_t) x_{t-1}
  // is on the critical path
  const int nlines = DIR == 0 ? ld : P.o.N;
  if (threadIdx.x < LB && l0 + (int)threadIdx.x < nlines &&
      (DIR == 1 || ydof_of_col(P.lay, P.o, l0 + (int)threadIdx.x) >= 0)) {
    constexpr int HB = 8;
    double* v = sh + threadIdx.x;  // v[t * LB]
    double y = 0.0;
    int t = nh - 1;
    for (; t >= HB - 1; t -= HB) {
      double a[HB], b[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        const double il = fil[t - u];
        a[u] = il * v[(t - u) * LB];
        b[u] = fg[t - u] * il;
      }
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        y = fma(-b[u], y, a[u]);
        v[(t - u) * LB] = y;
      }
    }
    for (; t >= 0; --t) {
      y = fma(-fg[t] * fil[t], y, fil[t] * v[t * LB]);
      v[t * LB] = y;
    }
    double x = 0.0;
    t = 0;
    for (; t + HB <= nh; t += HB) {
      double a[HB], b[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        const double il = fil[t + u];
        a[u] = il * v[(t + u) * LB];
        b[u] = (t + u > 0 ? fg[t + u - 1] : 0.0) * il;
      }
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        x = fma(-b[u], x, a[u]);
        v[(t + u) * LB] = x;
      }
    }
    for (; t < nh; ++t) {
      x = fma(-(t > 0 ? fg[t - 1] : 0.0) * fil[t], x, fil[t] * v[t * LB]);
      v[t * LB] = x;
    }
  }
  __syncthreads();
  if (DIR == 0) {
    const int j = threadIdx.x % LB, tg = threadIdx.x / LB, ng = blockDim.x / LB;
    const int li = l0 + j;
    if (li < ld && ydof_of_col(P.lay, P.o, li) >= 0)
      for (int t = tg; t < nh; t += ng) P.out[addr<DIR>(li, t, ld)] = sh[t * LB + j];
  } else {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = w; j < LB; j += nw) {
      const int lp = l0 + j;
      if (lp >= P.o.N) break;
      const int l = row_of(P.o, lp);
      for (int t = lane; t < nh; t += 32) P.out[addr<DIR>(l, t, ld)] = sh[t * LB + j];
    }
  }
}

template <int DIR, int CL>
static cudaError_t launch_bub_reg(const StepParams& P, cudaStream_t st) {
  if (DIR == 0) {
    dim3 grid((P.lp_count + 127) / 128, P.s.n * 2);
    k_bubbles_reg<DIR, CL><<<grid, 128, 0, st>>>(P);
  } else {
    const long long nthr = (long long)P.lp_count * 2 * P.s.n;
    k_bubbles_reg<DIR, CL><<<(unsigned)((nthr + 127) / 128), 128, 0, st>>>(P);
  }
  return cudaGetLastError();
}

template <int DIR>
static cudaError_t launch_bub_dir(const StepParams& P, cudaStream_t st) {
  const int m = chain_len(P.s.p, 0);
  if (P.tun.bub_reg && m <= 64) {  // HPFEM_BUBBLE_KERNEL=reg
    if (m <= 4) return launch_bub_reg<DIR, 4>(P, st);
    if (m <= 8) return launch_bub_reg<DIR, 8>(P, st);
    if (m <= 16) return launch_bub_reg<DIR, 16>(P, st);
    if (m <= 32) return launch_bub_reg<DIR, 32>(P, st);
    return launch_bub_reg<DIR, 64>(P, st);
  }
#ifndef HPFEM_LDG_UX
#define HPFEM_LDG_UX 4
#endif
#ifndef HPFEM_LDG_UY
#define HPFEM_LDG_UY 2
#endif
  // chain positions per load batch: smaller batches (fewer registers, more
  // resident threads) measured faster, most for the long y chains of
  // config 4 (p = 256: U 8 -> 2 cut the y kernel 1.48 -> 1.07 ms; x: U 4)
  constexpr int U = DIR == 0 ? HPFEM_LDG_UX : HPFEM_LDG_UY;
  if (DIR == 0) {
    dim3 grid((P.lp_count + 255) / 256, P.s.n * 2);
    k_bubbles<DIR, U><<<grid, 256, 0, st>>>(P);
  } else {
    const long long nthr = (long long)P.lp_count * 2 * P.s.n;
    k_bubbles<DIR, U><<<(unsigned)((nthr + 255) / 256), 256, 0, st>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_step_bubbles(const StepParams& P, cudaStream_t st) {
  if (P.lp_count <= 0) return cudaSuccess;
  return P.dir == 0 ? launch_bub_dir<0>(P, st) : launch_bub_dir<1>(P, st);
}

template <int DIR, int LB>
static cudaError_t launch_hats_lb(const StepParams& P, cudaStream_t st) {
  const size_t smem = sizeof(double) * hats_smem_doubles(P.s.nh, LB);
  cudaError_t e = smem_optin((const void*)k_hats<DIR, LB>, smem);
  if (e != cudaSuccess) return e;
  const int nlines = DIR == 0 ? P.ld : P.o.N;  // x-solve: internal columns (padding skipped)
  k_hats<DIR, LB><<<(nlines + LB - 1) / LB, 256, smem, st>>>(P);
  return cudaGetLastError();
}

/* lines per CTA of the hat kernel (tuning knob HPFEM_HAT_LB_X / _Y: 8 or 32);
 * fewer when the [nh][LB] tile would not fit in shared memory (many hats) */
template <int DIR>
static cudaError_t launch_hats_dir(const StepParams& P, cudaStream_t st) {
  const int lb = P.tun.hat_lb[DIR];
  const size_t cap = 227 * 1024;
  if (lb != 8 && sizeof(double) * hats_smem_doubles(P.s.nh, 32) <= cap) return launch_hats_lb<DIR, 32>(P, st);
  if (sizeof(double) * hats_smem_doubles(P.s.nh, 8) <= cap) return launch_hats_lb<DIR, 8>(P, st);
  return launch_hats_lb<DIR, 1>(P, st);
}

/* ------------------------------------------------------------------ */
/* Hat lines of the other direction (element-major layout): the few    */
/* lines whose cross-line stencil is the 7-point hat-row stencil.      */
/* Whole tiles are staged through shared memory with coalesced loads,  */
/* the chains are swept in shared memory, the tile is stored back.     */
/* ------------------------------------------------------------------ */

/* y-solve, lines = x-hat rows t: CTA = (t, group of EGH y-elements).
 * smem: 8 row segments [EGH*Q] (G + 7 stencil rows) and the chains'
 * factors [EGH][2][cfs]. */
#ifndef HPFEM_EGH
#define HPFEM_EGH 4
#endif
constexpr int EGH = HPFEM_EGH;  // y-elements per hat-row CTA

struct Aff {  // y = a + b * y_in
  double a, b;
};

__device__ __forceinline__ Aff aff_after(const Aff& f, const Aff& g) {  // f o g
  return Aff{fma(f.b, g.a, f.a), f.b * g.b};
}

/* In-place solve of one bubble chain held in shared memory, v[c * vs],
 * c < m, with the chain-major factors f ([4c] il, [4c+1] g il, [4c+2]
 * g_prev il): y_c = il_c v_c - hd_c y_{c+1} downwards, then z_c = il_c y_c -
 * hu_c z_{c-1} upwards.  Loads are batched CB positions ahead of the
 * dependent FMAs (the compiler cannot hoist them over the stores itself). */
__device__ __forceinline__ void chain_solve_smem(const double* f, double* v, int vs, int m) {
  constexpr int CB = 8;
  double y = 0.0;
  int c = m - 1;
  for (; c >= CB - 1; c -= CB) {
    double a[CB], b[CB];
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      a[u] = f[4 * (c - u)] * v[(c - u) * vs];
      b[u] = f[4 * (c - u) + 1];
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      y = fma(-b[u], y, a[u]);
      v[(c - u) * vs] = y;
    }
  }
  for (; c >= 0; --c) {
    y = fma(-f[4 * c + 1], y, f[4 * c] * v[c * vs]);
    v[c * vs] = y;
  }
  double z = 0.0;
  c = 0;
  for (; c + CB <= m; c += CB) {
    double a[CB], b[CB];
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      a[u] = f[4 * (c + u)] * v[(c + u) * vs];
      b[u] = f[4 * (c + u) + 2];
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      z = fma(-b[u], z, a[u]);
      v[(c + u) * vs] = z;
    }
  }
  for (; c < m; ++c) {
    z = fma(-f[4 * c + 2], z, f[4 * c] * v[c * vs]);
    v[c * vs] = z;
  }
}

__global__ void __launch_bounds__(128) k_hatrows_y(StepParams P) {
  extern __shared__ double sh[];
  const DirDev& y = P.s;  // solve direction (chains along the row)
  const DirDev& x = P.o;  // apply direction (stencil across rows)
  const Layout& L = P.lay;
  const int t = blockIdx.x;               // hat row
  const int e0 = blockIdx.y * EGH;
  const int ne = min(EGH, y.n - e0);
  const int W = EGH * L.Q;                // segment width (doubles)
  const size_t col0 = (size_t)L.hb + (size_t)e0 * L.Q;
  double* seg = sh;                       // [8][W]: 0 = G / r / y / z, 1..7 = stencil rows
  double* fac = sh + 8 * W;               // [EGH][2][cfs]
  __shared__ int s_idx[7];
  __shared__ double s_w[7];
  __shared__ __align__(8) uint64_t bar;
  const int nw = ne * L.Q;
  const int cfs = P.f.cfs;
  // Thread 0 needs only the stencil's ROWS (integer logic) to issue the bulk
  // copies; the weights (fp64 divides, ~1.5 us on one thread) are built by
  // warp 1 while the copies are in flight.
  if (threadIdx.x == 32) {
    Stencil st;
    stencil_build(x, t, P.mode, P.kap_a, P.tau, P.cvL, P.cvR, st);
    for (int q = 0; q < 7; ++q) s_w[q] = st.w[q];
  }
  if (threadIdx.x == 0) {
    hat_row_idx(x, t, P.mode, s_idx);
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // bulk copies of the G segment, the stencil rows and the chains' factors
    uint32_t bytes = 2 * ne * cfs * 8;
    for (int q = 0; q < 8; ++q)
      if (q == 0 ? P.alphaG != 0.0 : s_idx[q - 1] >= 0) bytes += nw * 8;
    mbar_expect_tx(&bar, bytes);
    for (int q = 0; q < 8; ++q) {
      const double* src = q == 0 ? (P.alphaG != 0.0 ? P.G + (size_t)t * P.ld : nullptr)
                                 : (s_idx[q - 1] >= 0 ? P.Xp + (size_t)s_idx[q - 1] * P.ld : nullptr);
      if (src) bulk_load(seg + q * W, src + col0, nw * 8, &bar);
    }
    bulk_load(fac, P.f.cf + (size_t)2 * e0 * cfs, 2 * ne * cfs * 8, &bar);
  }
  __syncthreads();  // s_idx, s_w and the barrier are visible
  // segments without a source read as zero
  for (int q = 0; q < 8; ++q) {
    const bool has = q == 0 ? P.alphaG != 0.0 : s_idx[q - 1] >= 0;
    if (!has)
      for (int j = threadIdx.x; j < W; j += blockDim.x) seg[q * W + j] = 0.0;
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  // r = alphaG G + sum_q w_q X_q (in place in segment 0)
  for (int j = threadIdx.x; j < nw; j += blockDim.x) {
    double r = P.alphaG != 0.0 ? P.alphaG * seg[j] : 0.0;
#pragma unroll
    for (int q = 0; q < 7; ++q) r += s_w[q] * seg[(q + 1) * W + j];
    seg[j] = r;
  }
  __syncthreads();
  // chains: thread (eo, pi); down sweep y, up sweep z, in place
  // (a warp-scan variant of the chain solve measured 54 -> 66 us per launch
  // at config 5: the chains are not this kernel's limiter)
  if (threadIdx.x < 2 * ne) {
    const int eo = threadIdx.x >> 1, pi = threadIdx.x & 1;
    const int m = chain_len(y.p, pi);
    const double* f = fac + (eo * 2 + pi) * cfs;
    double* v = seg + eo * L.Q + pi;
    chain_solve_smem(f, v, 2, m);
  }
  __syncthreads();
  double* out = P.out + (size_t)t * P.ld + col0;
  for (int j = threadIdx.x; j < nw; j += blockDim.x) {
    const int e = j / L.Q, k = j - e * L.Q;
    if (k < y.p - 1) out[j] = seg[j];
  }
  if (P.z01)  // chain-first bubbles: compact copy
    for (int j = threadIdx.x; j < 2 * ne; j += blockDim.x)
      P.z01[(size_t)t * 2 * y.n + 2 * e0 + j] = seg[(j >> 1) * L.Q + (j & 1)];
}

/* x-solve, lines = y-hat columns: CTA = (x-element e_x, parity pi, group
 * of TC hat columns l0..l0+TC-1).  For every row of the x-chain the CTA
 * stages G at its columns, the hat columns l0-1..l0+TC and the bubble 0/1
 * columns of the adjacent y-elements; the chains run in shared memory. */
constexpr int TC = 32;
constexpr int HREG = TC + 4;  // staged hat slots per row (TC + 2 used; rounding slack for 16-byte bulk copies)

__global__ void __launch_bounds__(256) k_hatcols_x(StepParams P) {
  extern __shared__ double sh[];
  const DirDev& x = P.s;  // solve direction (chains down the columns)
  const DirDev& y = P.o;  // apply direction (stencil across columns)
  const Layout& L = P.lay;
  const int e_x = blockIdx.x % x.n, pi = blockIdx.x / x.n;
  const int l0 = blockIdx.y * TC;
  const int nl = min(TC, y.nh - l0);
  const int m = chain_len(x.p, pi);
  // element range of the bubble columns the tile's stencils touch
  const int node0 = node_of_hat(l0, y.bc);
  const int elo = max(node0 - 1, 0);
  const int ehi = min(node_of_hat(l0 + nl - 1, y.bc), y.n - 1);
  const int nE = ehi - elo + 1;
  const int RW = TC + HREG + 2 * (TC + 2);  // per row: G | hats | bubbles 0/1 of elo..ehi, interleaved (16-byte aligned parts)
  double* rows = sh;                             // [m][RW]
  const int cfs = P.f.cfs;
  double* fac = sh + (size_t)m * RW;             // [cfs]
  const int hlo = (l0 - 1) & ~1;                 // first staged hat column (16-byte aligned)
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // per row: G[l0 .. l0+TC) and hats [hlo .. hlo+TC+2) as bulk copies (one thread);
  // bubble 0/1 columns of the adjacent elements as 16-byte gathers (all threads)
  const bool useG = P.alphaG != 0.0, useW = P.mode != ST_NONE;
  const int hs = hlo < 0 ? 0 : hlo;              // first hat column actually copied (hats < 0 do not exist)
  const int nh_c = min(l0 + nl + 1 - hs, y.nh - hs);  // hats hs .. l0+nl (the last line's right neighbour)
  const bool zc = useW && P.z01p;  // bubbles 0/1 from the compact copy (bulk) instead of 16-byte gathers
  if (threadIdx.x < 32) {  // warp 0 issues the copies, one row per lane
    uint32_t bytes = cfs * 8;
    const uint32_t gb = useG ? ((nl * 8 + 15) & ~15) : 0;
    const uint32_t hb = useW ? ((nh_c * 8 + 15) & ~15) : 0;
    const uint32_t zb = zc ? nE * 16 : 0;
    bytes += m * (gb + hb + zb);
    if (threadIdx.x == 0) mbar_expect_tx(&bar, bytes);
    __syncwarp();
    for (int c = threadIdx.x; c < m; c += 32) {
      const size_t rix = (size_t)(x.nh + (pi + 2 * c) * x.n + e_x);
      const size_t row = rix * P.ld;
      if (gb) bulk_load(rows + (size_t)c * RW, P.G + row + l0, gb, &bar);
      if (hb) bulk_load(rows + (size_t)c * RW + TC + (hs - hlo), P.Xp + row + hs, hb, &bar);
      if (zb) bulk_load(rows + (size_t)c * RW + TC + HREG, P.z01p + rix * 2 * y.n + 2 * elo, zb, &bar);
    }
    if (threadIdx.x == 0) bulk_load(fac, P.f.cf + (size_t)(2 * e_x + pi) * cfs, cfs * 8, &bar);
  }
  if (!useG)
    for (int idx = threadIdx.x; idx < m * TC; idx += blockDim.x) rows[(size_t)(idx / TC) * RW + idx % TC] = 0.0;
  if (!useW)
    for (int idx = threadIdx.x; idx < m * (TC + 2); idx += blockDim.x)
      rows[(size_t)(idx / (TC + 2)) * RW + TC + idx % (TC + 2)] = 0.0;
  else if (hs > hlo)  // the staged slots before hat 0 must read as zero
    for (int c = threadIdx.x; c < m; c += blockDim.x)
      for (int j = 0; j < hs - hlo; ++j) rows[(size_t)c * RW + TC + j] = 0.0;
  if (!zc) {
    const int nb = m * (TC + 2);  // (row, element) pairs, 2 doubles each
#pragma unroll 4
    for (int idx = threadIdx.x; idx < nb; idx += blockDim.x) {
      const int c = idx / (TC + 2), ei = idx - c * (TC + 2), e = elo + ei;
      double2 v = make_double2(0.0, 0.0);
      if (useW && e <= ehi) {
        const size_t row = (size_t)(x.nh + (pi + 2 * c) * x.n + e_x) * P.ld;
        v = __ldg(reinterpret_cast<const double2*>(P.Xp + row + L.hb + (size_t)e * L.Q));
        if (y.p - 2 < 1) v.y = 0.0;
      }
      double* R = rows + (size_t)c * RW + TC + HREG;
      R[2 * ei] = v.x;      // bubble 0
      R[2 * ei + 1] = v.y;  // bubble 1
    }
  }
  // right-hand sides and the chain solves split over the 8 warps: thread
  // (column j, warp w) owns chain positions [w BP, w BP + BP) of column j;
  // the block maps of the two recurrences are folded through shared memory
  // (the x chains run to 128 positions on the transposed path).  The column's
  // stencil (fp64 divides) is built while the copies are in flight.
  {
    const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool act = j < nl;
    double* fa = fac + cfs;  // [8][32] block maps (after the factors)
    double* fbm = fa + 8 * 32;
    const int BP = (m + 7) >> 3, ca = w * BP, cb = min(m, ca + BP);
    Stencil st;
    int off[7];
    if (act) {
      stencil_build(y, l0 + j, P.mode, P.kap_a, P.tau, P.cvL, P.cvR, st);
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const int d = st.idx[q];
        if (d < 0) {
          off[q] = 0;
          st.w[q] = 0.0;
        } else if (d < y.nh) {
          off[q] = TC + (d - hlo);
        } else {
          const int b = d - y.nh, k = b / y.n, e = b - k * y.n;
          off[q] = TC + HREG + 2 * (e - elo) + k;
        }
      }
    }
    mbar_wait(&bar, 0);
    __syncthreads();
    if (act) {
      const double aG = P.alphaG;
      // right-hand sides in place (each thread reads its stencil columns and
      // overwrites only its own G slot)
      for (int c = ca; c < cb; ++c) {
        const double* R = rows + (size_t)c * RW;
        double r = aG != 0.0 ? aG * R[j] : 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q) r += st.w[q] * R[off[q]];
        rows[(size_t)c * RW + j] = r;
      }
    }
    Aff f1{0.0, 1.0};
    for (int c = cb - 1; c >= ca; --c)
      f1 = Aff{fma(-fac[4 * c + 1], f1.a, fac[4 * c] * rows[(size_t)c * RW + j]), -fac[4 * c + 1] * f1.b};
    fa[w * 32 + j] = f1.a;
    fbm[w * 32 + j] = f1.b;
    __syncthreads();
    double yv = 0.0;
    for (int u = 7; u > w; --u) yv = fma(fbm[u * 32 + j], yv, fa[u * 32 + j]);
    for (int c = cb - 1; c >= ca; --c) {
      yv = fma(-fac[4 * c + 1], yv, fac[4 * c] * rows[(size_t)c * RW + j]);
      rows[(size_t)c * RW + j] = yv;
    }
    f1 = Aff{0.0, 1.0};
    for (int c = ca; c < cb; ++c)
      f1 = Aff{fma(-fac[4 * c + 2], f1.a, fac[4 * c] * rows[(size_t)c * RW + j]), -fac[4 * c + 2] * f1.b};
    __syncthreads();
    fa[w * 32 + j] = f1.a;
    fbm[w * 32 + j] = f1.b;
    __syncthreads();
    double zv = 0.0;
    for (int u = 0; u < w; ++u) zv = fma(fbm[u * 32 + j], zv, fa[u * 32 + j]);
    for (int c = ca; c < cb; ++c) {
      zv = fma(-fac[4 * c + 2], zv, fac[4 * c] * rows[(size_t)c * RW + j]);
      rows[(size_t)c * RW + j] = zv;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < m * TC; idx += blockDim.x) {
    const int c = idx / TC, j = idx - c * TC;
    if (j < nl) P.out[(size_t)(x.nh + (pi + 2 * c) * x.n + e_x) * P.ld + l0 + j] = rows[(size_t)c * RW + j];
  }
}

/* hat lines of the other direction (element-major layout only) */
cudaError_t launch_hat_lines(const StepParams& P, cudaStream_t st) {
  if (P.o.nh == 0 || P.s.nb == 0) return cudaSuccess;
  const Layout& L = P.lay;
  if (P.dir == 1) {
    const size_t smem = sizeof(double) * (8 * (size_t)EGH * L.Q + (size_t)EGH * 2 * P.f.cfs);
    cudaError_t e = smem_optin((const void*)k_hatrows_y, smem);
    if (e != cudaSuccess) return e;
    dim3 grid(P.o.nh, (P.s.n + EGH - 1) / EGH);
    k_hatrows_y<<<grid, 128, smem, st>>>(P);
  } else {
    const int m = chain_len(P.s.p, 0);
    const size_t smem = sizeof(double) * ((size_t)m * (TC + HREG + 2 * (TC + 2)) + P.f.cfs + 2 * 8 * 32);
    cudaError_t e = smem_optin((const void*)k_hatcols_x, smem);
    if (e != cudaSuccess) return e;
    dim3 grid(P.s.n * 2, (P.o.nh + TC - 1) / TC);
    k_hatcols_x<<<grid, 256, smem, st>>>(P);
  }
  return cudaGetLastError();
}

/* ------------------------------------------------------------------ */
/* K5, parallel form: the hat Schur solves with every thread busy.     */
/* The hat factor is the reverse Cholesky of the hat Schur complement   */
/* (Alg. 1 line 7 / R3): two first-order linear recurrences per line,  */
/*   y_t = il_t r_t - hd_t y_{t+1}   (t = nh-1 .. 0),                   */
/*   x_t = il_t y_t - hu_t x_{t-1}   (t = 0 .. nh-1),                   */
/* hd_t = g_t il_t, hu_t = g_{t-1} il_t.  A recurrence over a block of  */
/* hats is an affine map of the value entering the block; the maps of   */
/* the blocks are combined by a scan (warp shuffles / a shared-memory   */
/* fold) and every block then sweeps locally -- O(nh / P + log P) steps */
/* instead of nh (north_star K1: PCR / cyclic-reduction class).  Same   */
/* factors, same right-hand sides; only the association of the products */
/* differs from the sequential sweep (rounding-level, checked against   */
/* the oracle's rounding floor in tests/test_gpu_parity.py).            */
/* ------------------------------------------------------------------ */

/* per-hat tables of a hat Schur CTA: il, hd, hu, and the couplings
 * B(h, W_0 / W_1) of the left / right element (0 where absent) */
__device__ __forceinline__ void hat_tables(const StepParams& P, double* fil, double* fhd, double* fhu, double* cpl) {
  const DirDev& s = P.s;
  const double S = P.f.sig;
  const bool k1 = s.p - 2 >= 1;
  for (int t = threadIdx.x; t < s.nh; t += blockDim.x) {
    const double il = __ldg(P.f.ilh + t);
    fil[t] = il;
    fhd[t] = __ldg(P.f.gh + t) * il;
    fhu[t] = (t > 0 ? __ldg(P.f.gh + t - 1) : 0.0) * il;
    const int node = node_of_hat(t, s.bc);
    const int eL = node - 1, eR = node;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if (eL >= 0) {
      const double dl = s.delta[eL];
      c0 = s_hat_bub(S, dl, 1, 0);
      if (k1) c1 = s_hat_bub(S, dl, 1, 1);
    }
    if (eR <= s.n - 1) {
      const double dr = s.delta[eR];
      c2 = s_hat_bub(S, dr, 0, 0);
      if (k1) c3 = s_hat_bub(S, dr, 0, 1);
    }
    cpl[4 * t] = c0;
    cpl[4 * t + 1] = c1;
    cpl[4 * t + 2] = c2;
    cpl[4 * t + 3] = c3;
  }
}

/* y-solves (DIR 1): lines = rows, one warp per row.  Loads, right-hand
 * sides and stores touch hat t = lane + 32 i (coalesced: a warp request is
 * 256 contiguous bytes); the scan needs lane L to own the contiguous block
 * [L HB, L HB + HB), so the right-hand sides are handed over through a
 * per-warp shared-memory row (padded t + t/8: conflict-free in both
 * orders).  With the blocked mapping for the loads as well, each request
 * touched 31 sectors (ncu: L1-wavefront bound, 99 us at 255 hats). */
__device__ __forceinline__ int hpad(int t) { return t + (t >> 3); }

template <int HB>
__global__ void __launch_bounds__(256, 2) k_hats_rows(StepParams P) {
  constexpr int PADN = 32 * HB + 4 * HB;  // padded row length (hpad(32 HB - 1) < PADN)
  __shared__ double fil[PADN], fhd[PADN], fhu[PADN];  // padded, read in the blocked order
  __shared__ double cpl[4][32 * HB];                  // couplings [k][t], read in the strided order
  __shared__ double rs[8][PADN];                      // per-warp row handover
  const DirDev& s = P.s;
  const int nh = s.nh, n = s.n, ld = P.ld, dl = drop_left(s.bc);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t0 = lane * HB;
  const bool k1 = s.p - 2 >= 1;
  {
    const double S = P.f.sig;
    for (int t = threadIdx.x; t < nh; t += blockDim.x) {
      const double il = __ldg(P.f.ilh + t);
      fil[hpad(t)] = il;
      fhd[hpad(t)] = __ldg(P.f.gh + t) * il;
      fhu[hpad(t)] = (t > 0 ? __ldg(P.f.gh + t - 1) : 0.0) * il;
      const int node = node_of_hat(t, s.bc);
      const int eL = node - 1, eR = node;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      if (eL >= 0) {
        const double dlt = s.delta[eL];
        c0 = s_hat_bub(S, dlt, 1, 0);
        if (k1) c1 = s_hat_bub(S, dlt, 1, 1);
      }
      if (eR <= n - 1) {
        const double drt = s.delta[eR];
        c2 = s_hat_bub(S, drt, 0, 0);
        if (k1) c3 = s_hat_bub(S, drt, 0, 1);
      }
      cpl[0][t] = c0;
      cpl[1][t] = c1;
      cpl[2][t] = c2;
      cpl[3][t] = c3;
    }
  }
  __syncthreads();
  const double* __restrict__ G = P.G;
  const double* __restrict__ Xp = P.Xp;
  const double aG = P.alphaG;
  const bool anyW = P.mode != ST_NONE;
  double* row = rs[w];
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lp_hi = P.hl_end <= 0 ? P.o.N : P.hl_end;
  for (int lp = (P.hl_end <= 0 ? 0 : P.hl_begin) + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); lp < lp_hi; lp += nwarps) {
    const int l = row_of(P.o, lp);
    Stencil st;
    if (P.wtab && P.mode == ST_APPLY && l >= P.o.nh) {
      // bubble row (k, e): the five weights the bubble kernel uses (k_wtab_y:
      // [e][pi][kh][6], the same expressions as stencil_build) instead of
      // rebuilding them with fp64 divides on every lane; the rows from (k, e)
      const DirDev& o = P.o;
      const int b = l - o.nh, k = b / o.n, e = b - k * o.n;
      const double* wt = P.wtab + (((size_t)e * 2 + (k & 1)) * chain_len(o.p, 0) + (k >> 1)) * 6;
      const int hL = hat_of_node(e, o.n, o.bc), hR = hat_of_node(e + 1, o.n, o.bc);
      st.idx[0] = l;
      st.idx[1] = k >= 2 ? l - 2 * o.n : -1;
      st.idx[2] = k + 2 <= o.p - 2 ? l + 2 * o.n : -1;
      st.idx[3] = hL;
      st.idx[4] = hR;
      st.idx[5] = st.idx[6] = -1;
#pragma unroll
      for (int q = 0; q < 5; ++q) st.w[q] = __ldg(wt + q);
      st.w[5] = st.w[6] = 0.0;
    } else {
      line_stencil<1>(P, l, st);
    }
    // right-hand sides r_h - B z for t = lane + 32 i; all loads of a chunk of
    // HC hats issued before the FMAs (absent stencil rows clamped, skipped)
    constexpr int HC = HB < 4 ? HB : 2;  // no register spills at 128 registers
#pragma unroll
    for (int i0 = 0; i0 < HB; i0 += HC) {
      double gv[HC], xv[7][HC];
      double2 zl[HC], zr[HC];
#pragma unroll
      for (int u = 0; u < HC; ++u) {
        const int t = min(lane + 32 * (i0 + u), nh - 1);
        gv[u] = aG != 0.0 ? __ldg(G + (size_t)l * ld + t) : 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q)
          xv[q][u] = anyW ? __ldg(Xp + (size_t)(st.idx[q] >= 0 ? st.idx[q] : l) * ld + t) : 0.0;
        const int node = t + dl;
        const int eL = max(node - 1, 0), eR = min(node, n - 1);  // absent elements: zero couplings
        if (P.z01) {
          zl[u] = __ldg(reinterpret_cast<const double2*>(P.z01 + (size_t)l * 2 * n + 2 * eL));
          zr[u] = __ldg(reinterpret_cast<const double2*>(P.z01 + (size_t)l * 2 * n + 2 * eR));
        } else {
          zl[u].x = __ldg(P.out + (size_t)l * ld + ycol_ke(P.lay, 0, eL));
          zl[u].y = k1 ? __ldg(P.out + (size_t)l * ld + ycol_ke(P.lay, 1, eL)) : 0.0;
          zr[u].x = __ldg(P.out + (size_t)l * ld + ycol_ke(P.lay, 0, eR));
          zr[u].y = k1 ? __ldg(P.out + (size_t)l * ld + ycol_ke(P.lay, 1, eR)) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < HC; ++u) {
        const int i = i0 + u, t = lane + 32 * i;
        if (i >= HB) break;
        if (t < nh) {
          double rh = aG != 0.0 ? aG * gv[u] : 0.0;
#pragma unroll
          for (int q = 0; q < 7; ++q)
            if (st.idx[q] >= 0) rh += st.w[q] * xv[q][u];
          rh -= cpl[0][t] * zl[u].x;
          if (k1) rh -= cpl[1][t] * zl[u].y;
          rh -= cpl[2][t] * zr[u].x;
          if (k1) rh -= cpl[3][t] * zr[u].y;
          row[hpad(t)] = rh;
        }
      }
    }
    __syncwarp();
    double r[HB];
#pragma unroll
    for (int i = 0; i < HB; ++i) r[i] = t0 + i < nh ? row[hpad(t0 + i)] : 0.0;
    // down sweep: block map, suffix scan over the lanes, local sweep
    Aff f{0.0, 1.0};
#pragma unroll
    for (int i = HB - 1; i >= 0; --i) {
      const int t = t0 + i;
      if (t < nh) f = Aff{fma(-fhd[hpad(t)], f.a, fil[hpad(t)] * r[i]), -fhd[hpad(t)] * f.b};
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Aff g{__shfl_down_sync(0xffffffffu, f.a, d), __shfl_down_sync(0xffffffffu, f.b, d)};
      if (lane + d < 32) f = aff_after(f, g);
    }
    double v = __shfl_down_sync(0xffffffffu, f.a, 1);
    if (lane == 31) v = 0.0;
#pragma unroll
    for (int i = HB - 1; i >= 0; --i) {
      const int t = t0 + i;
      if (t < nh) {
        v = fma(-fhd[hpad(t)], v, fil[hpad(t)] * r[i]);
        r[i] = v;
      }
    }
    // up sweep: block map, prefix scan, local sweep
    f = Aff{0.0, 1.0};
#pragma unroll
    for (int i = 0; i < HB; ++i) {
      const int t = t0 + i;
      if (t < nh) f = Aff{fma(-fhu[hpad(t)], f.a, fil[hpad(t)] * r[i]), -fhu[hpad(t)] * f.b};
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Aff g{__shfl_up_sync(0xffffffffu, f.a, d), __shfl_up_sync(0xffffffffu, f.b, d)};
      if (lane >= d) f = aff_after(f, g);
    }
    v = __shfl_up_sync(0xffffffffu, f.a, 1);
    if (lane == 0) v = 0.0;
#pragma unroll
    for (int i = 0; i < HB; ++i) {
      const int t = t0 + i;
      if (t < nh) {
        v = fma(-fhu[hpad(t)], v, fil[hpad(t)] * r[i]);
        row[hpad(t)] = v;
      }
    }
    __syncwarp();
    double* __restrict__ out = P.out + (size_t)l * ld;
#pragma unroll
    for (int i = 0; i < HB; ++i) {
      const int t = lane + 32 * i;
      if (t < nh) out[t] = row[hpad(t)];
    }
    __syncwarp();  // the row buffer is rewritten by the next row
  }
}

/* x-solves (DIR 0): lines = internal columns, lane = column (coalesced),
 * the 8 warps of a CTA split each column's hats into 8 blocks; the block
 * maps are folded through shared memory */
constexpr int HC_COLS = 32;
__host__ __device__ constexpr size_t hats_cols_smem_doubles(int nh) {
  return (size_t)nh * HC_COLS + 7 * (size_t)nh + 2 * 8 * HC_COLS;
}

__global__ void __launch_bounds__(256, 2) k_hats_cols(StepParams P, int col_begin, int col_end) {
  extern __shared__ double sh[];
  const DirDev& s = P.s;
  const int nh = s.nh, n = s.n, ld = P.ld, dl = drop_left(s.bc);
  const bool k1 = s.p - 2 >= 1;
  double* v = sh;                          // [nh][32]: r, then y, per column
  double* fil = v + (size_t)nh * HC_COLS;
  double* fhd = fil + nh;
  double* fhu = fhd + nh;
  double* cpl = fhu + nh;                  // [nh][4]
  double* fa = cpl + 4 * nh;               // [8][32] block maps
  double* fb = fa + 8 * HC_COLS;
  hat_tables(P, fil, fhd, fhu, cpl);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int li = col_begin + blockIdx.x * HC_COLS + lane;  // columns [col_begin, col_end), col_end <= ld
  const int l = li < col_end ? ydof_of_col(P.lay, P.o, li) : -1;
  const int BH = (nh + 7) >> 3;
  const int ta = w * BH, tb = min(nh, ta + BH);
  __syncthreads();
  if (l >= 0) {
    Stencil st;
    if (P.wtab && P.mode == ST_APPLY && P.lay.emaj && l >= P.o.nh) {
      // bubble column (k, e): the bubble kernel's tabled weights (k_wtab_x:
      // [e][5][Q], the same expressions as stencil_build), internal columns
      const DirDev& o = P.o;
      const int b = l - o.nh, k = b / o.n, e = b - k * o.n;
      const double* wt = P.wtab + (size_t)e * 5 * P.lay.Q + k;
      st.idx[0] = li;
      st.idx[1] = k >= 2 ? li - 2 : -1;
      st.idx[2] = k + 2 <= o.p - 2 ? li + 2 : -1;
      st.idx[3] = hat_of_node(e, o.n, o.bc);      // (hat t sits at internal column t)
      st.idx[4] = hat_of_node(e + 1, o.n, o.bc);
      st.idx[5] = st.idx[6] = -1;
#pragma unroll
      for (int q = 0; q < 5; ++q) st.w[q] = __ldg(wt + (size_t)q * P.lay.Q);
      st.w[5] = st.w[6] = 0.0;
    } else {
      line_stencil<0>(P, l, st);
    }
    const double* __restrict__ G = P.G;
    const double* __restrict__ Xp = P.Xp;
    const double* __restrict__ Z = P.out;  // chain-first bubbles of this half-step
    const double aG = P.alphaG;
    // chunks of 2 hats, all loads of a chunk issued before the FMAs (as
    // k_hats_rows: absent stencil columns clamped, their terms skipped)
    const bool anyW = P.mode != ST_NONE;
    for (int t0 = ta; t0 < tb; t0 += 2) {
      double zv[2][4], gv[2], xv[7][2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = min(t0 + u, tb - 1);
        const int node = t + dl;
        const int eL = max(node - 1, 0), eR = min(node, n - 1);  // absent: zero coupling
        zv[u][0] = __ldg(Z + (size_t)(s.nh + eL) * ld + li);
        zv[u][1] = k1 ? __ldg(Z + (size_t)(s.nh + n + eL) * ld + li) : 0.0;
        zv[u][2] = __ldg(Z + (size_t)(s.nh + eR) * ld + li);
        zv[u][3] = k1 ? __ldg(Z + (size_t)(s.nh + n + eR) * ld + li) : 0.0;
        gv[u] = aG != 0.0 ? __ldg(G + (size_t)t * ld + li) : 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q)
          xv[q][u] = anyW ? __ldg(Xp + (size_t)t * ld + (st.idx[q] >= 0 ? st.idx[q] : li)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = t0 + u;
        if (t >= tb) break;
        double rh = aG != 0.0 ? aG * gv[u] : 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q)
          if (st.idx[q] >= 0) rh += st.w[q] * xv[q][u];
        const double* c = cpl + 4 * t;
        rh -= c[0] * zv[u][0];
        if (k1) rh -= c[1] * zv[u][1];
        rh -= c[2] * zv[u][2];
        if (k1) rh -= c[3] * zv[u][3];
        v[t * HC_COLS + lane] = rh;
      }
    }
  }
  // down sweep
  Aff f{0.0, 1.0};
  for (int t = tb - 1; t >= ta; --t) f = Aff{fma(-fhd[t], f.a, fil[t] * v[t * HC_COLS + lane]), -fhd[t] * f.b};
  fa[w * HC_COLS + lane] = f.a;
  fb[w * HC_COLS + lane] = f.b;
  __syncthreads();
  double y = 0.0;
  for (int u = 7; u > w; --u) y = fma(fb[u * HC_COLS + lane], y, fa[u * HC_COLS + lane]);
  for (int t = tb - 1; t >= ta; --t) {
    y = fma(-fhd[t], y, fil[t] * v[t * HC_COLS + lane]);
    v[t * HC_COLS + lane] = y;
  }
  f = Aff{0.0, 1.0};
  for (int t = ta; t < tb; ++t) f = Aff{fma(-fhu[t], f.a, fil[t] * v[t * HC_COLS + lane]), -fhu[t] * f.b};
  __syncthreads();  // every y of the block is written and the down-sweep maps are read
  fa[w * HC_COLS + lane] = f.a;
  fb[w * HC_COLS + lane] = f.b;
  __syncthreads();
  double x = 0.0;
  for (int u = 0; u < w; ++u) x = fma(fb[u * HC_COLS + lane], x, fa[u * HC_COLS + lane]);
  if (l >= 0)
    for (int t = ta; t < tb; ++t) {
      x = fma(-fhu[t], x, fil[t] * v[t * HC_COLS + lane]);
      P.out[(size_t)t * ld + li] = x;
    }
}

template <int HB>
static cudaError_t launch_hats_rows(const StepParams& P, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int warps = P.hl_end <= 0 ? P.o.N : P.hl_end - P.hl_begin, blocks = (warps + 7) / 8;
  if (blocks <= 0) return cudaSuccess;
  const int grid = blocks < 2 * sms ? blocks : 2 * sms;  // one wave of 2 CTAs per SM, grid-stride over rows
  k_hats_rows<HB><<<grid, 256, 0, st>>>(P);
  return cudaGetLastError();
}

bool hats_split_ok(const StepParams& P) {
  if (P.s.nh == 0 || P.tun.hats_seq) return false;
  if (P.dir == 1) return P.s.nh <= 256;
  return sizeof(double) * hats_cols_smem_doubles(P.s.nh) <= 200 * 1024;
}

cudaError_t launch_step_hats(const StepParams& P, cudaStream_t st) {
  if (P.s.nh == 0) return cudaSuccess;
  if (P.tun.hats_seq) return P.dir == 0 ? launch_hats_dir<0>(P, st) : launch_hats_dir<1>(P, st);  // experiment
  const int nh = P.s.nh;
  if (P.dir == 1 && nh <= 256) {
    switch ((nh + 31) / 32) {
      case 1: return launch_hats_rows<1>(P, st);
      case 2: return launch_hats_rows<2>(P, st);
      case 3: return launch_hats_rows<3>(P, st);
      case 4: return launch_hats_rows<4>(P, st);
      case 5: return launch_hats_rows<5>(P, st);
      case 6: return launch_hats_rows<6>(P, st);
      case 7: return launch_hats_rows<7>(P, st);
      default: return launch_hats_rows<8>(P, st);
    }
  }
  const size_t smem = sizeof(double) * hats_cols_smem_doubles(nh);
  if (P.dir == 0 && smem <= 200 * 1024) {
    cudaError_t e = smem_optin((const void*)k_hats_cols, smem);
    if (e != cudaSuccess) return e;
    const int cb = P.hl_end <= 0 ? 0 : P.hl_begin, ce = P.hl_end <= 0 ? P.ld : P.hl_end;
    if (ce > cb) k_hats_cols<<<(ce - cb + HC_COLS - 1) / HC_COLS, 256, smem, st>>>(P, cb, ce);
    return cudaGetLastError();
  }
  return P.dir == 0 ? launch_hats_dir<0>(P, st) : launch_hats_dir<1>(P, st);  // very many hats
}

/* K6: U = W_J C^{-1} materialised in the caller's layout:
 * U(i, j) = X(i, col j) for hats, z - vL x_hL - vR x_hR for bubbles (the
 * deferred correction of the final y-solve). */
__global__ void __launch_bounds__(256) k_finalize(DirDev y, int Nx, Layout L, const double* __restrict__ vL,
                                                   const double* __restrict__ vR, const double* __restrict__ X,
                                                   double* __restrict__ U) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= y.N || i >= Nx) return;
  const double* row = X + (size_t)i * L.ld;
  double v;
  if (j < y.nh) {
    v = row[j];
  } else {
    const int b = j - y.nh, k = b / y.n, e = b - k * y.n;
    const int hL = hat_of_node(e, y.n, y.bc), hR = hat_of_node(e + 1, y.n, y.bc);
    v = row[ycol_ke(L, k, e)];
    if (hL >= 0) v -= __ldg(vL + b) * row[hL];
    if (hR >= 0) v -= __ldg(vR + b) * row[hR];
  }
  U[(size_t)i * y.N + j] = v;
}

/* Element-major layout: per row, the bubbles are an (e, k) -> (k, e)
 * transpose; 32 x 32 tiles through shared memory keep both the internal
 * reads (along k) and the caller-layout writes (along e) coalesced.
 * grid (rows, e tiles, k tiles), block 32 x 8. */
__global__ void __launch_bounds__(256) k_finalize_t(DirDev y, Layout L, const double* __restrict__ vL,
                                                     const double* __restrict__ vR, const double* __restrict__ X,
                                                     double* __restrict__ U) {
  __shared__ double t[32][33];
  const int i = blockIdx.x, e0 = blockIdx.y * 32, k0 = blockIdx.z * 32;
  const int q = y.p - 1, n = y.n, tx = threadIdx.x, ty = threadIdx.y;
  const double* row = X + (size_t)i * L.ld;
  double* u = U + (size_t)i * y.N;
  if (blockIdx.y == 0 && blockIdx.z == 0)
    for (int j = ty * 32 + tx; j < y.nh; j += 256) u[j] = row[j];
#pragma unroll
  for (int ee = ty; ee < 32; ee += 8) {
    const int e = e0 + ee, k = k0 + tx;
    if (e < n && k < q) t[ee][tx] = row[L.hb + (size_t)e * L.Q + k];
  }
  __syncthreads();
  const int e = e0 + tx;
  if (e >= n) return;
  const int hL = hat_of_node(e, n, y.bc), hR = hat_of_node(e + 1, n, y.bc);
  const double xL = hL >= 0 ? row[hL] : 0.0, xR = hR >= 0 ? row[hR] : 0.0;
#pragma unroll
  for (int kk = ty; kk < 32; kk += 8) {
    const int k = k0 + kk;
    if (k >= q) break;
    const int b = k * n + e;
    double v = t[tx][kk];
    if (hL >= 0) v -= __ldg(vL + b) * xL;
    if (hR >= 0) v -= __ldg(vR + b) * xR;
    u[y.nh + b] = v;
  }
}

__global__ void __launch_bounds__(256) k_copyin_t(DirDev y, Layout L, const double* __restrict__ G,
                                                   double* __restrict__ Gp) {
  __shared__ double t[32][33];
  const int i = blockIdx.x, e0 = blockIdx.y * 32, k0 = blockIdx.z * 32;
  const int q = y.p - 1, n = y.n, tx = threadIdx.x, ty = threadIdx.y;
  const double* g = G + (size_t)i * y.N;
  double* o = Gp + (size_t)i * L.ld;
  if (blockIdx.y == 0 && blockIdx.z == 0)
    for (int j = ty * 32 + tx; j < y.nh; j += 256) o[j] = __ldg(g + j);
#pragma unroll
  for (int kk = ty; kk < 32; kk += 8) {
    const int k = k0 + kk, e = e0 + tx;
    if (k < q && e < n) t[kk][tx] = __ldg(g + y.nh + (size_t)k * n + e);
  }
  __syncthreads();
#pragma unroll
  for (int ee = ty; ee < 32; ee += 8) {
    const int e = e0 + ee, k = k0 + tx;
    if (k < q && e < n) o[L.hb + (size_t)e * L.Q + k] = t[tx][ee];
  }
}

cudaError_t launch_finalize(const DirDev& x, const DirDev& y, const Layout& L, const double* vL, const double* vR,
                            const double* X, double* U, cudaStream_t st) {
  if (L.emaj && y.nb > 0) {
    dim3 grid(x.N, (y.n + 31) / 32, (y.p - 1 + 31) / 32);
    k_finalize_t<<<grid, dim3(32, 8), 0, st>>>(y, L, vL, vR, X, U);
    return cudaGetLastError();
  }
  dim3 grid((y.N + 255) / 256, x.N);
  k_finalize<<<grid, 256, 0, st>>>(y, x.N, L, vL, vR, X, U);
  return cudaGetLastError();
}

/* plain transpose through 32 x 33 shared-memory tiles (coalesced both ways):
 * out[c][r] = in[r][c]; the transposed solve's copy-in / finalize (R23) */
__global__ void __launch_bounds__(256) k_transpose(const double* __restrict__ in, int R, int C,
                                                   double* __restrict__ out) {
  __shared__ double t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32, tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int rr = ty; rr < 32; rr += 8) {
    const int r = r0 + rr, c = c0 + tx;
    if (r < R && c < C) t[rr][tx] = __ldg(in + (size_t)r * C + c);
  }
  __syncthreads();
#pragma unroll
  for (int cc = ty; cc < 32; cc += 8) {
    const int c = c0 + cc, r = r0 + tx;
    if (r < R && c < C) out[(size_t)c * R + r] = t[tx][cc];
  }
}

cudaError_t launch_transpose(const double* in, int R, int C, double* out, cudaStream_t st) {
  if (R <= 0 || C <= 0) return cudaSuccess;
  dim3 grid((C + 31) / 32, (R + 31) / 32);
  k_transpose<<<grid, dim3(32, 8), 0, st>>>(in, R, C, out);
  return cudaGetLastError();
}

/* G (caller layout) -> Gp (internal layout) */
__global__ void __launch_bounds__(256) k_copyin(DirDev y, int Nx, Layout L, const double* __restrict__ G,
                                                 double* __restrict__ Gp) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= y.N || i >= Nx) return;
  Gp[(size_t)i * L.ld + ycol(L, y, j)] = __ldg(G + (size_t)i * y.N + j);
}

cudaError_t launch_copyin(const DirDev& x, const DirDev& y, const Layout& L, const double* G, double* Gp,
                          cudaStream_t st) {
  if (L.emaj && y.nb > 0) {
    dim3 grid(x.N, (y.n + 31) / 32, (y.p - 1 + 31) / 32);
    k_copyin_t<<<grid, dim3(32, 8), 0, st>>>(y, L, G, Gp);
    return cudaGetLastError();
  }
  dim3 grid((y.N + 255) / 256, x.N);
  k_copyin<<<grid, 256, 0, st>>>(y, x.N, L, G, Gp);
  return cudaGetLastError();
}

/* K7: F = A_x U M_y + M_x U A_y, A = K + (w^2/2) M */
__global__ void __launch_bounds__(128) k_apply2d(DirDev x, DirDev y, double half_w2, const double* __restrict__ U,
                                                  double* __restrict__ F) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= y.N) return;
  Stencil ax, mx, ay, my;  // weights are -(row entries)
  stencil_build(x, i, ST_APPLY, 1.0, half_w2, nullptr, nullptr, ax);
  stencil_build(x, i, ST_APPLY, 0.0, 1.0, nullptr, nullptr, mx);
  stencil_build(y, j, ST_APPLY, 1.0, half_w2, nullptr, nullptr, ay);
  stencil_build(y, j, ST_APPLY, 0.0, 1.0, nullptr, nullptr, my);
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 7; ++a) {
    if (ax.idx[a] < 0) continue;
    const double* row = U + (size_t)ax.idx[a] * y.N;
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      if (my.idx[b] < 0) continue;
      const double u = __ldg(row + my.idx[b]);
      t1 += my.w[b] * u;
      t2 += ay.w[b] * u;
    }
    acc += ax.w[a] * t1 + mx.w[a] * t2;
  }
  F[(size_t)i * y.N + j] = acc;
}

/* K7, tabled and streamed (round 2).  The kernel above rebuilds four stencils
 * per output (fp64 divides) and re-reads every U row from L2 once per stencil
 * row: 18.9 ms at config 5, 0.035 of the 16-byte-per-dof roofline.  Here the
 * 7-slot rows of A and M of both directions are tabled once per plan
 * (k_apply_tab: slot-major [7][N], weights = -(row entries) as stencil_build
 * gives them), and a block walks one x-chain (x-element, parity) for 256
 * columns: per U row it forms t1 = (U M_y)(row, j) and t2 = (U A_y)(row, j)
 * once (7 coalesced loads), keeps them for the rows c - 1, c, c + 1 in
 * registers and for the element's two hat rows, and emits
 * F(row_c, j) = sum_a wA_x[a] t1[a] + wM_x[a] t2[a].  The x-hat rows (7-point
 * rows) stay with the kernel above. */
__global__ void k_apply_tab(DirDev o, double half_w2, int* __restrict__ idx, double* __restrict__ wA,
                            double* __restrict__ wM) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= o.N) return;
  Stencil a, m;
  stencil_build(o, l, ST_APPLY, 1.0, half_w2, nullptr, nullptr, a);
  stencil_build(o, l, ST_APPLY, 0.0, 1.0, nullptr, nullptr, m);
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    idx[(size_t)q * o.N + l] = a.idx[q];  // (A and M have the same pattern)
    wA[(size_t)q * o.N + l] = a.idx[q] >= 0 ? a.w[q] : 0.0;
    wM[(size_t)q * o.N + l] = m.idx[q] >= 0 ? m.w[q] : 0.0;
  }
}

cudaError_t launch_apply_tab(const DirDev& o, double omega, const ApplyTab& t, cudaStream_t st) {
  k_apply_tab<<<(o.N + 127) / 128, 128, 0, st>>>(o, 0.5 * omega * omega, const_cast<int*>(t.idx),
                                                  const_cast<double*>(t.wA), const_cast<double*>(t.wM));
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256, 4) k_apply2d_chain(DirDev x, DirDev y, ApplyTab tx, ApplyTab ty,
                                                        const double* __restrict__ U, double* __restrict__ F) {
  extern __shared__ double xw[];  // [10][m]: wA slots 0-4, wM slots 0-4 of the chain's rows
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int e = blockIdx.y % x.n, pi = blockIdx.y / x.n;
  const int m = chain_len(x.p, pi);
  // the chain's x-rows of A and M into shared memory in one round of loads
  // (read per row from the tables they cost one L2 latency per chain
  // position: ncu long_scoreboard 36 stalls per issue, 65% of the samples)
  for (int idx = threadIdx.x; idx < 10 * m; idx += blockDim.x) {
    const int q = idx / m, c = idx - q * m;
    const int row = x.nh + (pi + 2 * c) * x.n + e;
    xw[idx] = q < 5 ? __ldg(tx.wA + (size_t)q * x.N + row) : __ldg(tx.wM + (size_t)(q - 5) * x.N + row);
  }
  __syncthreads();
  if (j >= y.N) return;
  // y-rows of A and M for column j (absent slots: weight 0, own column)
  int jy[7];
  double ya[7], ym[7];
#pragma unroll
  for (int b = 0; b < 7; ++b) {
    const int id = __ldg(ty.idx + (size_t)b * y.N + j);
    jy[b] = id >= 0 ? id : j;
    ya[b] = __ldg(ty.wA + (size_t)b * y.N + j);
    ym[b] = __ldg(ty.wM + (size_t)b * y.N + j);
  }
  auto row_t = [&](int row, double& t1, double& t2) {  // (U M_y)(row, j), (U A_y)(row, j), both negated
    const double* __restrict__ r = U + (size_t)row * y.N;
    double u[7];
#pragma unroll
    for (int b = 0; b < 7; ++b) u[b] = __ldg(r + jy[b]);
    t1 = 0.0;
    t2 = 0.0;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      t1 += ym[b] * u[b];
      t2 += ya[b] * u[b];
    }
  };
  const int hL = hat_of_node(e, x.n, x.bc), hR = hat_of_node(e + 1, x.n, x.bc);
  double h1[2] = {0.0, 0.0}, h2[2] = {0.0, 0.0};
  if (hL >= 0) row_t(hL, h1[0], h2[0]);
  if (hR >= 0) row_t(hR, h1[1], h2[1]);
  auto rowc = [&](int c) { return x.nh + (pi + 2 * c) * x.n + e; };
  double p1 = 0.0, p2 = 0.0, c1 = 0.0, c2 = 0.0, n1 = 0.0, n2 = 0.0;  // rows c - 1, c, c + 1
  if (m > 0) row_t(rowc(0), c1, c2);
  // groups of RG rows: the 7 RG loads of the next RG rows are issued together
  // (one row at a time left a single row of loads in flight per thread)
  constexpr int RG = 1;
  constexpr int PF = 8;  // L2 prefetch distance (rows) of the three bubble-column segments
#pragma unroll
  for (int c = 2; c < 2 + PF; ++c)
    if (c < m) {
      const double* r = U + (size_t)rowc(c) * y.N;
#pragma unroll
      for (int b = 0; b < 3; ++b) asm volatile("prefetch.global.L2 [%0];" ::"l"(r + jy[b]));
    }
  for (int c0 = 0; c0 < m; c0 += RG) {
    if (c0 + 2 + PF < m) {
      const double* r = U + (size_t)rowc(c0 + 2 + PF) * y.N;
#pragma unroll
      for (int b = 0; b < 3; ++b) asm volatile("prefetch.global.L2 [%0];" ::"l"(r + jy[b]));
    }
    double u[RG][7];
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const int cn = c0 + i + 1 < m ? c0 + i + 1 : m - 1;  // (clamped: unused past the chain)
      const double* __restrict__ r = U + (size_t)rowc(cn) * y.N;
#pragma unroll
      for (int b = 0; b < 7; ++b) u[i][b] = __ldg(r + jy[b]);
    }
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const int c = c0 + i;
      if (c < m) {
        n1 = 0.0;
        n2 = 0.0;
        if (c + 1 < m) {
#pragma unroll
          for (int b = 0; b < 7; ++b) {
            n1 += ym[b] * u[i][b];
            n2 += ya[b] * u[i][b];
          }
        }
        double acc = 0.0;  // slots: [0] own row, [1] k - 2, [2] k + 2, [3] hL, [4] hR
        acc += xw[c] * c1 + xw[5 * m + c] * c2;
        acc += xw[m + c] * p1 + xw[6 * m + c] * p2;
        acc += xw[2 * m + c] * n1 + xw[7 * m + c] * n2;
        acc += xw[3 * m + c] * h1[0] + xw[8 * m + c] * h2[0];
        acc += xw[4 * m + c] * h1[1] + xw[9 * m + c] * h2[1];
        F[(size_t)rowc(c) * y.N + j] = acc;
        p1 = c1;
        p2 = c2;
        c1 = n1;
        c2 = n2;
      }
    }
  }
}

cudaError_t launch_apply2d(const DirDev& x, const DirDev& y, double omega, const double* U, double* F,
                           cudaStream_t st, const ApplyTab* tx, const ApplyTab* ty) {
  if (tx && ty && tx->idx && ty->idx && x.nb > 0 && sizeof(double) * 10 * chain_len(x.p, 0) <= 48 * 1024) {
    if (x.nh > 0) {  // the x-hat rows: 7-point rows
      dim3 gh((y.N + 127) / 128, x.nh);
      k_apply2d<<<gh, 128, 0, st>>>(x, y, 0.5 * omega * omega, U, F);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    dim3 grid((y.N + 255) / 256, 2 * x.n);
    k_apply2d_chain<<<grid, 256, sizeof(double) * 10 * chain_len(x.p, 0), st>>>(x, y, *tx, *ty, U, F);
    return cudaGetLastError();
  }
  dim3 grid((y.N + 127) / 128, x.N);
  k_apply2d<<<grid, 128, 0, st>>>(x, y, 0.5 * omega * omega, U, F);
  return cudaGetLastError();
}

/* ------------------------------------------------------------------ */
/* K11 (small problems): the whole ADI solve of one problem in one CTA, all
 * three arrays (G, W_j, W_{j-1/2}) in shared memory -- for the
 * configurations whose half-steps are latency-bound (config 1: 31^2 dofs,
 * 23 KB), where the multi-kernel path spends ~9 us per kernel on almost no
 * data.  Same algebra as the oracle's Algorithm 2 (the "plus" form, R6),
 * with the iterate materialised after every solve (x_b = z - v_L x_hL -
 * v_R x_hR, no deferred correction) and the 1D solves of solve1d.cu
 * (static condensation with the factor tables of K1).  One CTA per
 * right-hand side: hpfem_solve_batched fills the GPU with problems. */
/* solve (kap K + sig M) along direction d for L lines of array A, entry
 * (line l, dof) at A[l ls + dof es], in place (solve1d.cu, all CTA threads) */
__device__ void small_line_solve(const DirDev& d, const double* __restrict__ base, double sig, int L, int ls,
                                 int es, double* A) {
  const int n = d.n, nh = d.nh, nb = d.nb;
  const double* __restrict__ il = base;
  const double* __restrict__ g = base + nb;
  const double* __restrict__ vL = base + 2 * (size_t)nb;
  const double* __restrict__ vR = base + 3 * (size_t)nb;
  const double* __restrict__ ilh = base + 4 * (size_t)nb;
  const double* __restrict__ gh = ilh + nh;
  for (int it = threadIdx.x; it < L * 2 * n; it += blockDim.x) {  // 1. chains z = D^{-1} r_b
    const int l = it / (2 * n), ch = it - l * 2 * n;
    const int pi = ch / n, e = ch - pi * n;
    const int m = chain_len(d.p, pi);
    double* a = A + (size_t)l * ls;
    double y = 0.0;
    for (int c = m - 1; c >= 0; --c) {
      const int b = (pi + 2 * c) * n + e;
      y = (a[(nh + b) * es] - __ldg(g + b) * y) * __ldg(il + b);
      a[(nh + b) * es] = y;
    }
    double z = 0.0, gp = 0.0;
    for (int c = 0; c < m; ++c) {
      const int b = (pi + 2 * c) * n + e;
      z = (a[(nh + b) * es] - gp * z) * __ldg(il + b);
      gp = __ldg(g + b);
      a[(nh + b) * es] = z;
    }
  }
  __syncthreads();
  const bool k1 = d.p - 2 >= 1;
  for (int it = threadIdx.x; it < L * nh; it += blockDim.x) {  // 2. hat rhs r_h - B z
    const int l = it / nh, t = it - l * nh;
    double* a = A + (size_t)l * ls;
    const int node = node_of_hat(t, d.bc), eL = node - 1, eR = node;
    double r = a[t * es];
    if (eL >= 0) {
      const double dl = d.delta[eL];
      r -= s_hat_bub(sig, dl, 1, 0) * a[(nh + eL) * es];
      if (k1) r -= s_hat_bub(sig, dl, 1, 1) * a[(nh + n + eL) * es];
    }
    if (eR <= n - 1) {
      const double dr = d.delta[eR];
      r -= s_hat_bub(sig, dr, 0, 0) * a[(nh + eR) * es];
      if (k1) r -= s_hat_bub(sig, dr, 0, 1) * a[(nh + n + eR) * es];
    }
    a[t * es] = r;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < L && nh > 0; l += blockDim.x) {  // 3. hat Schur solve per line
    double* a = A + (size_t)l * ls;
    double y = 0.0;
    for (int t = nh - 1; t >= 0; --t) {
      const double w = __ldg(ilh + t);
      y = fma(-__ldg(gh + t) * w, y, a[t * es] * w);
      a[t * es] = y;
    }
    double x = 0.0;
    for (int t = 0; t < nh; ++t) {
      const double w = __ldg(ilh + t);
      x = fma(-(t > 0 ? __ldg(gh + t - 1) : 0.0) * w, x, a[t * es] * w);
      a[t * es] = x;
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < L * nb; it += blockDim.x) {  // 4. x_b = z - v_L x_hL - v_R x_hR
    const int l = it / nb, b = it - l * nb;
    const int e = b % n;
    double* a = A + (size_t)l * ls;
    const int hl = hat_of_node(e, n, d.bc), hr = hat_of_node(e + 1, n, d.bc);
    double v = a[(nh + b) * es];
    if (hl >= 0) v -= __ldg(vL + b) * a[hl * es];
    if (hr >= 0) v -= __ldg(vR + b) * a[hr * es];
    a[(nh + b) * es] = v;
  }
  __syncthreads();
}

/* out[l ls + d es] = G[...] + sum_s w_s(d) in[l ls + idx_s(d) es] for every
 * line l < L and dof d < N of direction o (the -(kap K_o + tau M_o) apply) */
__device__ void small_apply(const DirDev& o, double tau, int L, int ls, int es, const double* G, const double* in,
                            double* out, Stencil* sst) {
  for (int d = threadIdx.x; d < o.N; d += blockDim.x) stencil_build(o, d, ST_APPLY, 1.0, tau, nullptr, nullptr, sst[d]);
  __syncthreads();
  for (int it = threadIdx.x; it < L * o.N; it += blockDim.x) {
    const int d = it % o.N, l = it / o.N;
    const Stencil& st = sst[d];
    double acc = G[(size_t)l * ls + (size_t)d * es];
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (st.idx[q] >= 0) acc += st.w[q] * in[(size_t)l * ls + (size_t)st.idx[q] * es];
    out[(size_t)l * ls + (size_t)d * es] = acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_adi_small(SmallArgs a) {
  extern __shared__ double sm[];
  const int Nx = a.x.N, Ny = a.y.N, nn = Nx * Ny;
  double* G = sm;
  double* W = G + nn;
  double* H = W + nn;
  Stencil* sst = reinterpret_cast<Stencil*>(H + nn);
  const double* F = a.F + (size_t)blockIdx.x * nn;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) {
    G[i] = F[i];
    W[i] = 0.0;
  }
  __syncthreads();
  const int J = a.J;
  for (int j = 0; j < a.iters; ++j) {
    // W_{j-1/2} = (G - (A_x - p_j M_x) W_{j-1}) (A_y + p_j M_y)^{-1}: x-apply (lines = columns), y-solves (rows)
    if (j == 0) {
      for (int i = threadIdx.x; i < nn; i += blockDim.x) H[i] = G[i];
      __syncthreads();
    } else {
      small_apply(a.x, a.tau[j], Ny, 1, Ny, G, W, H, sst);
    }
    small_line_solve(a.y, a.fy + a.sy * j, a.sh[3 * (J + 1) + j], Nx, Ny, 1, H);
    // W_j = (A_x - q_j M_x)^{-1} (G - W_{j-1/2} (A_y + q_j M_y)): y-apply (rows), x-solves (columns)
    small_apply(a.y, a.tau[J + j], Nx, Ny, 1, G, H, W, sst);
    small_line_solve(a.x, a.fx + a.sx * j, a.sh[(J + 1) + j], Ny, 1, Ny, W);
  }
  // U = W_J M_y^{-1}: row-wise mass solves
  small_line_solve(a.y, a.fy + a.sy * J, 1.0, Nx, Ny, 1, W);
  double* U = a.U + (size_t)blockIdx.x * nn;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) U[i] = W[i];
}

size_t small_smem_bytes(const DirDev& x, const DirDev& y) {
  const int Nmax = x.N > y.N ? x.N : y.N;
  return sizeof(double) * 3 * (size_t)x.N * y.N + sizeof(Stencil) * (size_t)Nmax;
}

cudaError_t launch_adi_small(const SmallArgs& a, int batch, cudaStream_t st) {
  const size_t smem = small_smem_bytes(a.x, a.y);
  cudaError_t e = smem_optin((const void*)k_adi_small, smem);
  if (e != cudaSuccess) return e;
  k_adi_small<<<batch, 256, smem, st>>>(a);
  return cudaGetLastError();
}

/* K8 helper: Legendre sources of dof l: (M_P R)[(m,e), l] (App. A) */
__device__ __forceinline__ int load_sources(const DirDev& o, int l, int* r, double* w) {
  const int n = o.n;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    r[q] = -1;
    w[q] = 0.0;
  }
  if (l >= o.nh) {
    const int b = l - o.nh, k = b / n, e = b - k * n;
    const double d = o.delta[e];
    r[0] = k * n + e;
    w[0] = (d / (2.0 * k + 1.0)) * (1.0 / (2.0 * k + 3.0));
    r[1] = (k + 2) * n + e;
    w[1] = (d / (2.0 * k + 5.0)) * (-1.0 / (2.0 * k + 3.0));
  } else {
    const int node = node_of_hat(l, o.bc), eL = node - 1, eR = node;
    if (eL >= 0) {  // right hat of eL: (1+t)/2 = P0/2 + P1/2
      const double d = o.delta[eL];
      r[0] = eL; w[0] = d * 0.5;
      r[1] = n + eL; w[1] = (d / 3.0) * 0.5;
    }
    if (eR <= n - 1) {  // left hat of eR: (1-t)/2 = P0/2 - P1/2
      const double d = o.delta[eR];
      r[2] = eR; w[2] = d * 0.5;
      r[3] = n + eR; w[3] = (d / 3.0) * -0.5;
    }
  }
  return 0;
}

/* the load sources of every dof of one direction, tabled once per plan (the
 * fp64 divides of load_sources would otherwise dominate k_load2d) */
__global__ void k_load_tab(DirDev o, int* __restrict__ r, double* __restrict__ w) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= o.N) return;
  int rr[4];
  double ww[4];
  load_sources(o, l, rr, ww);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    r[4 * l + q] = rr[q];
    w[4 * l + q] = ww[q];
  }
}

cudaError_t launch_load_tab(const DirDev& d, int* r, double* w, cudaStream_t st) {
  if (d.N <= 0) return cudaSuccess;
  k_load_tab<<<(d.N + 255) / 256, 256, 0, st>>>(d, r, w);
  return cudaGetLastError();
}

__device__ __forceinline__ void load_sources_tab(const DirDev& o, int l, int* r, double* w) {
  if (o.lw) {
    const int4 ri = *reinterpret_cast<const int4*>(o.lr + 4 * l);
    const double4 wi = *reinterpret_cast<const double4*>(o.lw + 4 * l);
    r[0] = ri.x; r[1] = ri.y; r[2] = ri.z; r[3] = ri.w;
    w[0] = wi.x; w[1] = wi.y; w[2] = wi.z; w[3] = wi.w;
  } else {
    load_sources(o, l, r, w);
  }
}

/* y-direction part of one source row: t = sum_b wy_b F(row, ry_b) */
__device__ __forceinline__ double load_trow(const double* __restrict__ Fl, size_t ldl, int row, const int* ry,
                                            const double* wy) {
  double t = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (ry[b] >= 0) t += wy[b] * __ldg(Fl + (size_t)row * ldl + ry[b]);
  return t;
}

/* generic rows (the x-hat rows here): G(i, j) = sum_a wx_a t(rx_a) */
__global__ void __launch_bounds__(128) k_load2d(DirDev x, DirDev y, const double* __restrict__ Fl,
                                                 double* __restrict__ G, int accumulate, double scale, int row0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = row_of(x, row0 + blockIdx.y);
  if (j >= y.N) return;
  int rx[4], ry[4];
  double wx[4], wy[4];
  load_sources_tab(x, i, rx, wx);
  load_sources_tab(y, j, ry, wy);
  const size_t ldl = (size_t)(y.p + 1) * y.n;
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    if (rx[a] < 0) continue;
    acc += wx[a] * load_trow(Fl, ldl, rx[a], ry, wy);
  }
  acc *= scale;
  if (accumulate) acc += G[(size_t)i * y.N + j];
  G[(size_t)i * y.N + j] = acc;
}

/* x-bubble rows (k, e_x), k in [k0, k0 + KB): their sources are the Legendre
 * rows (k, e_x) and (k + 2, e_x) (load_sources), so each y-contracted source
 * row t(m) is formed once and used by the outputs k = m and k = m - 2 (same
 * expressions as k_load2d, i.e. bitwise the same G).  grid (column blocks,
 * x-elements, degree chunks). */
constexpr int LOAD_KB = 16;
__global__ void __launch_bounds__(128) k_load2d_bub(DirDev x, DirDev y, const double* __restrict__ Fl,
                                                     double* __restrict__ G, int accumulate, double scale) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int ex = blockIdx.y, k0 = blockIdx.z * LOAD_KB, n = x.n, q = x.p - 1;
  if (j >= y.N) return;
  int ry[4];
  double wy[4];
  load_sources_tab(y, j, ry, wy);
  const size_t ldl = (size_t)(y.p + 1) * y.n;
  const int k1 = k0 + LOAD_KB < q ? k0 + LOAD_KB : q;
  double t0 = load_trow(Fl, ldl, k0 * n + ex, ry, wy);
  double t1 = k0 + 1 < k1 ? load_trow(Fl, ldl, (k0 + 1) * n + ex, ry, wy) : 0.0;
  for (int k = k0; k < k1; ++k) {
    const int i = x.nh + k * n + ex;
    int rx[4];
    double wx[4];
    load_sources_tab(x, i, rx, wx);  // rx = {(k, ex), (k + 2, ex), -1, -1}
    const double t2 = load_trow(Fl, ldl, rx[1], ry, wy);
    double acc = 0.0;
    acc += wx[0] * t0;
    acc += wx[1] * t2;
    acc *= scale;
    if (accumulate) acc += G[(size_t)i * y.N + j];
    G[(size_t)i * y.N + j] = acc;
    t0 = t1;
    t1 = t2;
  }
}

/* Unload (NEXT-1): Legendre coefficient (degree m, element e) of direction
 * o as a combination of <= 3 dofs (R of eq. app:1): bubbles
 * (m, e) [1/(2m+3)] and (m-2, e) [-1/(2m-1)], plus for m = 0, 1 the two hats
 * of e ((1 -+ t)/2 = P0/2 -+ P1/2). */
__device__ __forceinline__ void unload_sources(const DirDev& o, int r, int* d, double* w) {
  const int n = o.n, m = r / n, e = r - m * n;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    d[q] = -1;
    w[q] = 0.0;
  }
  if (m <= o.p - 2) {
    d[0] = o.nh + m * n + e;
    w[0] = 1.0 / (2.0 * m + 3.0);
  }
  if (m >= 2) {
    d[1] = o.nh + (m - 2) * n + e;
    w[1] = -1.0 / (2.0 * m - 1.0);
  } else {
    const int hl = hat_of_node(e, n, o.bc), hr = hat_of_node(e + 1, n, o.bc);
    d[1] = hl;
    w[1] = m == 0 ? 0.5 : -0.5;
    d[2] = hr;
    w[2] = 0.5;
  }
}

/* Derivative unload (NEXT-4): Legendre coefficient (degree m, element e) of
 * du/dx as a combination of <= 2 dofs: d/dx W_k = -(2/delta) P_{k+1}
 * (W_k' = -P_{k+1}, P:L84 with dx = delta/2 dt), d/dx (1 -+ t)/2 = -+ 1/delta. */
__device__ __forceinline__ void dunload_sources(const DirDev& o, int r, int* d, double* w) {
  const int n = o.n, m = r / n, e = r - m * n;
  const double dl = o.delta[e];
  d[0] = d[1] = d[2] = -1;
  w[0] = w[1] = w[2] = 0.0;
  if (m == 0) {
    d[0] = hat_of_node(e, n, o.bc);
    w[0] = -1.0 / dl;
    d[1] = hat_of_node(e + 1, n, o.bc);
    w[1] = 1.0 / dl;
  } else if (m - 1 <= o.p - 2) {
    d[0] = o.nh + (m - 1) * n + e;
    w[0] = -2.0 / dl;
  }
}

template <bool DX>
__global__ void __launch_bounds__(128) k_unload2d(DirDev x, DirDev y, const double* __restrict__ U,
                                                   double* __restrict__ C) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int Ly = (y.p + 1) * y.n;
  if (s >= Ly) return;
  int dx[3], dy[3];
  double wx[3], wy[3];
  if (DX)
    dunload_sources(x, r, dx, wx);
  else
    unload_sources(x, r, dx, wx);
  unload_sources(y, s, dy, wy);
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (dx[a] < 0) continue;
    double t = 0.0;
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (dy[b] >= 0) t += wy[b] * __ldg(U + (size_t)dx[a] * y.N + dy[b]);
    acc += wx[a] * t;
  }
  C[(size_t)r * Ly + s] = acc;
}

cudaError_t launch_unload2d(const DirDev& x, const DirDev& y, const double* U, double* Cleg, cudaStream_t st,
                            int dx) {
  dim3 grid(((y.p + 1) * y.n + 127) / 128, (x.p + 1) * x.n);
  if (dx)
    k_unload2d<true><<<grid, 128, 0, st>>>(x, y, U, Cleg);
  else
    k_unload2d<false><<<grid, 128, 0, st>>>(x, y, U, Cleg);
  return cudaGetLastError();
}

cudaError_t launch_load2d(const DirDev& x, const DirDev& y, const double* Fleg, double* G, cudaStream_t st,
                          int accumulate, double scale) {
  if (x.lw && x.nb > 0) {  // bubble rows by element and degree chunk, then the hat rows
    dim3 gb((y.N + 127) / 128, x.n, (x.p - 1 + LOAD_KB - 1) / LOAD_KB);
    k_load2d_bub<<<gb, 128, 0, st>>>(x, y, Fleg, G, accumulate, scale);
    if (x.nh > 0) {
      dim3 gh((y.N + 127) / 128, x.nh);
      k_load2d<<<gh, 128, 0, st>>>(x, y, Fleg, G, accumulate, scale, x.nb);
    }
    return cudaGetLastError();
  }
  dim3 grid((y.N + 127) / 128, x.N);
  k_load2d<<<grid, 128, 0, st>>>(x, y, Fleg, G, accumulate, scale, 0);
  return cudaGetLastError();
}

}  // namespace hpfem
