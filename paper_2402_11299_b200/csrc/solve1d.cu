/*
 * solve1d.cu -- batched 1D screened-Poisson solves (NEXT-2 of SURVEY 8(f),
 * the workload of the paper's Fig. 1):
 *
 *     (K + w^2 M) u = f     in the hat + integrated-Legendre basis,
 *
 * with the reverse Cholesky factor of Algorithm 1 in the
 * static-condensation form of the 2D kernels (the factor tables of
 * k_factor_chains / k_factor_hats):
 *   1. bubble chains  z = D^{-1} f_b           (2n independent chains,
 *      bottom-up L^T y = f then top-down L z = y, Cor. 4.3 P:L600-L614)
 *   2. hat right-hand side  r_h = f_h - B z     (only the chain-first
 *      bubbles couple to the hats)
 *   3. hat Schur system (A0 - B D^{-1} B^T) x_h = r_h, tridiagonal, solved
 *      by its reverse Cholesky factor: the two sweeps are first-order linear
 *      recurrences, split over the CTA's threads in contiguous blocks whose
 *      affine maps are combined by a scan (warp shuffles, then the 8 warp
 *      totals) -- O(nh / 256 + log) dependent steps instead of 2 nh, which
 *      makes the time independent of n at fixed N (Fig. 1)
 *   4. bubbles  x_b = z - v_L x_hL - v_R x_hR, fused into the up sweeps of
 *      step 1 (which therefore runs after the hat solve).
 * Grid: one wave of up to 8 CTAs per SM, each walking right-hand sides
 * b = blockIdx.x, +gridDim.x.  Algorithmic traffic 16 bytes per dof (F read,
 * U written); the down-sweep values make one extra round trip through the
 * output row (L2 when the rows in flight fit).
 */
#include <cuda_runtime.h>

#include "hpfem_internal.h"
#include "ops1d.h"

namespace hpfem {

namespace {

struct Aff {  // v = a + b * v_in
  double a, b;
};

__device__ __forceinline__ Aff after(const Aff& f, const Aff& g) { return Aff{fma(f.b, g.a, f.a), f.b * g.b}; }

constexpr int NT1 = 256, NW1 = NT1 / 32;

/* Value entering this thread's block for a recurrence that runs from the
 * LAST thread to the first (down sweep): thread i's block is entered by the
 * value leaving block i+1; the last block is entered by 0.  f: this
 * thread's block map.  sa/sb: NW1 doubles of shared scratch each. */
__device__ double enter_down(Aff f, double* sa, double* sb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Aff g{__shfl_down_sync(0xffffffffu, f.a, d), __shfl_down_sync(0xffffffffu, f.b, d)};
    if (lane + d < 32) f = after(f, g);
  }
  if (lane == 0) {
    sa[w] = f.a;
    sb[w] = f.b;
  }
  __syncthreads();
  double v = 0.0;  // value entering the last block of this warp
  for (int u = NW1 - 1; u > w; --u) v = fma(sb[u], v, sa[u]);
  const double na = __shfl_down_sync(0xffffffffu, f.a, 1), nb = __shfl_down_sync(0xffffffffu, f.b, 1);
  __syncthreads();  // sa / sb reused by the next scan
  return lane == 31 ? v : fma(nb, v, na);
}

/* the same for a recurrence from the first thread to the last (up sweep) */
__device__ double enter_up(Aff f, double* sa, double* sb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Aff g{__shfl_up_sync(0xffffffffu, f.a, d), __shfl_up_sync(0xffffffffu, f.b, d)};
    if (lane >= d) f = after(f, g);
  }
  if (lane == 31) {
    sa[w] = f.a;
    sb[w] = f.b;
  }
  __syncthreads();
  double v = 0.0;
  for (int u = 0; u < w; ++u) v = fma(sb[u], v, sa[u]);
  const double pa = __shfl_up_sync(0xffffffffu, f.a, 1), pb = __shfl_up_sync(0xffffffffu, f.b, 1);
  __syncthreads();
  return lane == 0 ? v : fma(pb, v, pa);
}

}  // namespace

/* One CTA per right-hand side at a time (grid-stride over them).  Passes
 * over the row: F read once; U written with the down-sweep values y, read
 * back and overwritten with the final x_b in the up sweep, into which the
 * bubble correction x_b = z_b - v_L x_hL - v_R x_hR is fused (the hat
 * solution is known by then: the hat right-hand side needs only the
 * chain-first z_0 = il_0 y_0, available right after the down sweep).
 * Chain loads are batched CB positions ahead of the dependent FMAs.
 * hats_in_smem: the hat values live in shared memory [nh] (else in the hat
 * slots of the output row, same code with global addresses). */
constexpr int CB = 4;   // chain positions per load batch (down sweeps)
constexpr int CBU = 4;  // the same for the up sweeps
constexpr int NCH = 1;  // chains per thread in flight (loads of all of them batched together)
constexpr int HU = 8;   // hats per load batch in the block sweeps

__global__ void __launch_bounds__(NT1) k_solve1d(DirDev d, FacView f, int nrhs, int hats_in_smem,
                                                    const double* __restrict__ F, double* __restrict__ U) {
  extern __shared__ double sh[];
  __shared__ double sa[NW1], sb[NW1];
  const int n = d.n, nh = d.nh;
  const double* __restrict__ il = f.il;
  const double* __restrict__ g = f.g;
  const double* __restrict__ ilh = f.ilh;
  const double* __restrict__ gh = f.gh;
  const double S = f.sig;
  const bool k1 = d.p - 2 >= 1;
  const int HB = (nh + NT1 - 1) / NT1;  // hats per thread (contiguous block)
  const int ta = threadIdx.x * HB, tb = min(nh, ta + HB);
  const int m0 = chain_len(d.p, 0);     // the longer (even) chain
  for (int rhs = blockIdx.x; rhs < nrhs; rhs += gridDim.x) {
    const double* __restrict__ Fr = F + (size_t)rhs * d.N;
    double* __restrict__ Ur = U + (size_t)rhs * d.N;
    double* H = hats_in_smem ? sh : Ur;  // hat values r -> y -> x
    // 1. down sweeps L^T y = f of every chain (consecutive threads:
    //    consecutive elements, coalesced); y parked in the output row, the
    //    chain-first slot gets z_0 = il_0 y_0 (the first up-sweep step)
    for (int ch0 = threadIdx.x; ch0 < 2 * n; ch0 += NT1 * NCH) {
      double y[NCH];
      int pe[NCH], mm[NCH];
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int ch = ch0 + j * NT1;
        const int pi = ch < n ? 0 : 1, e = ch - pi * n;
        mm[j] = ch < 2 * n ? chain_len(d.p, pi) : 0;
        pe[j] = pi * n + e;  // b of position c: pe + 2 c n
        y[j] = 0.0;
      }
      for (int c0 = m0 - 1; c0 >= 0; c0 -= CB) {
        double fv[NCH][CB], gv[NCH][CB], lv[NCH][CB];
#pragma unroll
        for (int j = 0; j < NCH; ++j)
#pragma unroll
          for (int u = 0; u < CB; ++u) {
            const int c = c0 - u;
            const bool ok = c >= 0 && c < mm[j];
            const int b = pe[j] + 2 * (ok ? c : 0) * n;
            fv[j][u] = ok ? Fr[nh + b] : 0.0;
            gv[j][u] = ok ? g[b] : 0.0;
            lv[j][u] = ok ? il[b] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < NCH; ++j)
#pragma unroll
          for (int u = 0; u < CB; ++u) {
            const int c = c0 - u;
            if (c >= 0 && c < mm[j]) {
              y[j] = (fv[j][u] - gv[j][u] * y[j]) * lv[j][u];
              Ur[nh + pe[j] + 2 * c * n] = c == 0 ? y[j] * lv[j][u] : y[j];
            }
          }
      }
    }
    __syncthreads();
    // 2. hat right-hand sides r_h = f_h - B z
#pragma unroll 4
    for (int t = threadIdx.x; t < nh; t += NT1) {
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
      H[t] = r;
    }
    __syncthreads();
    // 3. hat Schur solve: y_t = il_t r_t - (g_t il_t) y_{t+1} (t descending),
    //    then x_t = il_t y_t - (g_{t-1} il_t) x_{t-1} (t ascending), each as
    //    block maps + scan + local sweep; loads HU hats ahead
    if (nh > 0) {
      Aff fm{0.0, 1.0};
      for (int t0 = tb - 1; t0 >= ta; t0 -= HU) {
        double hv[HU], lv[HU], gv[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 - u >= ta ? t0 - u : ta;
          hv[u] = H[t];
          lv[u] = ilh[t];
          gv[u] = gh[t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 - u >= ta) {
            const double hd = gv[u] * lv[u];
            fm = Aff{fma(-hd, fm.a, lv[u] * hv[u]), -hd * fm.b};
          }
      }
      double v = enter_down(fm, sa, sb);
      for (int t0 = tb - 1; t0 >= ta; t0 -= HU) {
        double hv[HU], lv[HU], gv[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 - u >= ta ? t0 - u : ta;
          hv[u] = H[t];
          lv[u] = ilh[t];
          gv[u] = gh[t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 - u >= ta) {
            v = fma(-(gv[u] * lv[u]), v, lv[u] * hv[u]);
            H[t0 - u] = v;
          }
      }
      fm = Aff{0.0, 1.0};
      for (int t0 = ta; t0 < tb; t0 += HU) {
        double hv[HU], lv[HU], gv[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 + u < tb ? t0 + u : tb - 1;
          hv[u] = H[t];
          lv[u] = ilh[t];
          gv[u] = t > 0 ? gh[t - 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 + u < tb) {
            const double hu = gv[u] * lv[u];
            fm = Aff{fma(-hu, fm.a, lv[u] * hv[u]), -hu * fm.b};
          }
      }
      v = enter_up(fm, sa, sb);
      for (int t0 = ta; t0 < tb; t0 += HU) {
        double hv[HU], lv[HU], gv[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 + u < tb ? t0 + u : tb - 1;
          hv[u] = H[t];
          lv[u] = ilh[t];
          gv[u] = t > 0 ? gh[t - 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 + u < tb) {
            v = fma(-(gv[u] * lv[u]), v, lv[u] * hv[u]);
            H[t0 + u] = v;
          }
      }
      __syncthreads();
      if (hats_in_smem)
        for (int t = threadIdx.x; t < nh; t += NT1) Ur[t] = H[t];
    }
    // 4. up sweeps L z = y with the bubble correction fused:
    //    x_c = z_c - v_L x_hL - v_R x_hR, written once
    for (int ch0 = threadIdx.x; ch0 < 2 * n; ch0 += NT1 * NCH) {
      double z[NCH], gp[NCH], xl[NCH], xr[NCH];
      int pe[NCH], mm[NCH];
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int ch = ch0 + j * NT1;
        const int pi = ch < n ? 0 : 1, e = ch - pi * n;
        mm[j] = ch < 2 * n ? chain_len(d.p, pi) : 0;
        pe[j] = pi * n + e;
        const int hl = hat_of_node(e, n, d.bc), hr = hat_of_node(e + 1, n, d.bc);
        xl[j] = (mm[j] > 0 && hl >= 0) ? H[hl] : 0.0;  // 0: the term is skipped below
        xr[j] = (mm[j] > 0 && hr >= 0) ? H[hr] : 0.0;
        z[j] = 0.0;
        gp[j] = 0.0;
      }
      for (int c0 = 0; c0 < m0; c0 += CBU) {
        double yv[NCH][CBU], gv[NCH][CBU], lv[NCH][CBU], vl[NCH][CBU], vr[NCH][CBU];
#pragma unroll
        for (int j = 0; j < NCH; ++j)
#pragma unroll
          for (int u = 0; u < CBU; ++u) {
            const int c = c0 + u;
            const bool ok = c < mm[j];
            const int b = pe[j] + 2 * (ok ? c : 0) * n;
            yv[j][u] = ok ? Ur[nh + b] : 0.0;
            gv[j][u] = ok ? g[b] : 0.0;
            lv[j][u] = ok ? il[b] : 0.0;
            vl[j][u] = ok ? f.vL[b] : 0.0;
            vr[j][u] = ok ? f.vR[b] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int ch = ch0 + j * NT1;
          const int e = ch < n ? ch : ch - n;
          const bool hl = hat_of_node(e, n, d.bc) >= 0, hr = hat_of_node(e + 1, n, d.bc) >= 0;
#pragma unroll
          for (int u = 0; u < CBU; ++u) {
            const int c = c0 + u;
            if (c < mm[j]) {
              z[j] = c == 0 ? yv[j][u] : (yv[j][u] - gp[j] * z[j]) * lv[j][u];  // slot 0 holds z_0
              gp[j] = gv[j][u];
              double x = z[j];
              if (hl) x -= vl[j][u] * xl[j];
              if (hr) x -= vr[j][u] * xr[j];
              Ur[nh + pe[j] + 2 * c * n] = x;
            }
          }
        }
      }
    }
    __syncthreads();  // H (shared) is rewritten by the next right-hand side
  }
}

cudaError_t launch_solve1d(const DirDev& d, const FacView& f, int nrhs, const double* F, double* U,
                           cudaStream_t st) {
  if (nrhs <= 0) return cudaSuccess;
  // hats in shared memory when they are few enough not to limit occupancy
  const size_t hb = sizeof(double) * (size_t)d.nh;
  const int in_smem = hb <= 48 * 1024 ? 1 : 0;
  const size_t smem = in_smem ? hb : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one wave of up to 8 resident CTAs per SM, grid-stride over the rest
  long long g = 8LL * sms;
  if (g > nrhs) g = nrhs;
  k_solve1d<<<(unsigned)g, NT1, smem, st>>>(d, f, nrhs, in_smem, F, U);
  return cudaGetLastError();
}

}  // namespace hpfem
