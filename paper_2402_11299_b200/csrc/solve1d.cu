/*
 * solve1d.cu -- batched 1D screened-Poisson solves (NEXT-2 of SURVEY 8(f),
 * the workload of the paper's Fig. 1):
 *
 *     (K + w^2 M) u = f     in the hat + integrated-Legendre basis,
 *
 * one CTA per right-hand side, with the reverse Cholesky factor of
 * Algorithm 1 in the static-condensation form of the 2D
 * kernels (the factor tables of k_factor_chains / k_factor_hats):
 *   1. bubble chains  z = D^{-1} f_b           (2n independent chains,
 *      bottom-up L^T y = f then top-down L z = y, Cor. 4.3 P:L600-L614)
 *   2. hat right-hand side  r_h = f_h - B z     (only the chain-first
 *      bubbles couple to the hats)
 *   3. hat Schur system (A0 - B D^{-1} B^T) x_h = r_h, tridiagonal, solved
 *      by its reverse Cholesky factor (one thread, loads batched ahead)
 *   4. bubbles  x_b = z - v_L x_hL - v_R x_hR.
 * The hat values live in the output row itself (no shared-memory limit on n).
 */
#include <cuda_runtime.h>

#include "hpfem_internal.h"
#include "ops1d.h"

namespace hpfem {

__global__ void __launch_bounds__(256) k_solve1d(DirDev d, FacView f, const double* __restrict__ F,
                                                 double* __restrict__ U) {
  const double* __restrict__ Fr = F + (size_t)blockIdx.x * d.N;
  double* __restrict__ Ur = U + (size_t)blockIdx.x * d.N;
  const int n = d.n, nh = d.nh;
  const double* __restrict__ il = f.il;
  const double* __restrict__ g = f.g;
  // 1. bubble chains (consecutive threads: consecutive elements, coalesced)
  for (int ch = threadIdx.x; ch < 2 * n; ch += blockDim.x) {
    const int pi = ch / n, e = ch - pi * n;
    const int m = chain_len(d.p, pi);
    double y = 0.0;
    for (int c = m - 1; c >= 0; --c) {
      const int b = (pi + 2 * c) * n + e;
      y = (Fr[nh + b] - g[b] * y) * il[b];
      Ur[nh + b] = y;
    }
    double z = 0.0, gp = 0.0;
    for (int c = 0; c < m; ++c) {
      const int b = (pi + 2 * c) * n + e;
      z = (Ur[nh + b] - gp * z) * il[b];
      gp = g[b];
      Ur[nh + b] = z;
    }
  }
  __syncthreads();
  // 2. hat right-hand sides r_h = f_h - B z (into the hat slots of the output)
  const double S = f.sig;
  const bool k1 = d.p - 2 >= 1;
  for (int t = threadIdx.x; t < nh; t += blockDim.x) {
    const int node = node_of_hat(t, d.bc), eL = node - 1, eR = node;
    double r = Fr[t];
    if (eL >= 0) {
      const double dl = d.delta[eL];
      r -= s_hat_bub(S, dl, 1, 0) * Ur[nh + eL];
      if (k1) r -= s_hat_bub(S, dl, 1, 1) * Ur[nh + n + eL];
    }
    if (eR <= n - 1) {
      const double dr = d.delta[eR];
      r -= s_hat_bub(S, dr, 0, 0) * Ur[nh + eR];
      if (k1) r -= s_hat_bub(S, dr, 0, 1) * Ur[nh + n + eR];
    }
    Ur[t] = r;
  }
  __syncthreads();
  // 3. hat Schur solve, one thread, loads HB positions ahead of the FMAs
  if (threadIdx.x == 0 && nh > 0) {
    constexpr int HB = 8;
    const double* __restrict__ ilh = f.ilh;
    const double* __restrict__ gh = f.gh;
    double y = 0.0;
    int t = nh - 1;
    for (; t >= HB - 1; t -= HB) {
      double a[HB], bb[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        a[u] = Ur[t - u] * ilh[t - u];
        bb[u] = gh[t - u] * ilh[t - u];
      }
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        y = fma(-bb[u], y, a[u]);
        Ur[t - u] = y;
      }
    }
    for (; t >= 0; --t) {
      y = fma(-gh[t] * ilh[t], y, Ur[t] * ilh[t]);
      Ur[t] = y;
    }
    double x = 0.0;
    t = 0;
    for (; t + HB <= nh; t += HB) {
      double a[HB], bb[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        a[u] = Ur[t + u] * ilh[t + u];
        bb[u] = (t + u > 0 ? gh[t + u - 1] : 0.0) * ilh[t + u];
      }
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        x = fma(-bb[u], x, a[u]);
        Ur[t + u] = x;
      }
    }
    for (; t < nh; ++t) {
      x = fma(-(t > 0 ? gh[t - 1] : 0.0) * ilh[t], x, Ur[t] * ilh[t]);
      Ur[t] = x;
    }
  }
  __syncthreads();
  // 4. bubble correction x_b = z - v_L x_hL - v_R x_hR
  for (int b = threadIdx.x; b < d.nb; b += blockDim.x) {
    const int k = b / n, e = b - k * n;
    (void)k;
    const int hl = hat_of_node(e, n, d.bc), hr = hat_of_node(e + 1, n, d.bc);
    double v = Ur[nh + b];
    if (hl >= 0) v -= f.vL[b] * Ur[hl];
    if (hr >= 0) v -= f.vR[b] * Ur[hr];
    Ur[nh + b] = v;
  }
}

cudaError_t launch_solve1d(const DirDev& d, const FacView& f, int nrhs, const double* F, double* U,
                           cudaStream_t st) {
  if (nrhs <= 0) return cudaSuccess;
  k_solve1d<<<nrhs, 256, 0, st>>>(d, f, F, U);
  return cudaGetLastError();
}

}  // namespace hpfem
