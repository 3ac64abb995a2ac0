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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

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

/* One CTA takes RB right-hand sides at a time (grid-stride over groups of
 * RB).  Passes over a row: F read once; U written with the down-sweep values
 * y, read back and overwritten with the final x_b in the up sweep, into which
 * the bubble correction x_b = z_b - v_L x_hL - v_R x_hR is fused (the hat
 * solution is known by then: the hat right-hand side needs only the
 * chain-first z_0 = il_0 y_0, available right after the down sweep).
 * A thread sweeps the SAME chain of all RB right-hand sides together: the
 * chain factors (il, g, v_L, v_R -- 6 of the 8 loads per dof of a single
 * right-hand side) are loaded once per RB rows, and the RB recurrences are
 * independent (ILP).  Chain loads are batched CB positions ahead of the
 * dependent FMAs.  hats_in_smem: the hat values live in shared memory
 * [RB][nh] (else in the hat slots of the output rows, same code with global
 * addresses). */
constexpr int CB = 4;   // chain positions per load batch (down sweeps)
constexpr int CBU = 4;  // the same for the up sweeps
constexpr int HU = 8;   // hats per load batch in the block sweeps

template <int RB>
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
  for (int rhs0 = blockIdx.x * RB; rhs0 < nrhs; rhs0 += gridDim.x * RB) {
    const double* Fr[RB];
    double* Ur[RB];
    double* H[RB];  // hat values r -> y -> x
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int rhs = min(rhs0 + r, nrhs - 1);  // a ragged last group repeats its last row (same values rewritten)
      Fr[r] = F + (size_t)rhs * d.N;
      Ur[r] = U + (size_t)rhs * d.N;
      H[r] = hats_in_smem ? sh + (size_t)r * nh : Ur[r];
    }
    // 1. down sweeps L^T y = f of every chain (consecutive threads:
    //    consecutive elements, coalesced); y parked in the output row, the
    //    chain-first slot gets z_0 = il_0 y_0 (the first up-sweep step)
    for (int ch = threadIdx.x; ch < 2 * n; ch += NT1) {
      const int pi = ch < n ? 0 : 1, e = ch - pi * n;
      const int mm = chain_len(d.p, pi);
      const int pe = pi * n + e;  // b of position c: pe + 2 c n
      double y[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) y[r] = 0.0;
      for (int c0 = m0 - 1; c0 >= 0; c0 -= CB) {
        double fv[RB][CB], gv[CB], lv[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int c = c0 - u;
          const bool ok = c >= 0 && c < mm;
          const int b = pe + 2 * (ok ? c : 0) * n;
          gv[u] = ok ? g[b] : 0.0;
          lv[u] = ok ? il[b] : 0.0;
#pragma unroll
          for (int r = 0; r < RB; ++r) fv[r][u] = ok ? Fr[r][nh + b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int c = c0 - u;
          if (c >= 0 && c < mm) {
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              y[r] = (fv[r][u] - gv[u] * y[r]) * lv[u];
              Ur[r][nh + pe + 2 * c * n] = c == 0 ? y[r] * lv[u] : y[r];
            }
          }
        }
      }
    }
    __syncthreads();
    // 2. hat right-hand sides r_h = f_h - B z (coupling coefficients once per hat for the RB rows)
#pragma unroll 2
    for (int t = threadIdx.x; t < nh; t += NT1) {
      const int node = node_of_hat(t, d.bc), eL = node - 1, eR = node;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      if (eL >= 0) {
        const double dl = d.delta[eL];
        c0 = s_hat_bub(S, dl, 1, 0);
        if (k1) c1 = s_hat_bub(S, dl, 1, 1);
      }
      if (eR <= n - 1) {
        const double dr = d.delta[eR];
        c2 = s_hat_bub(S, dr, 0, 0);
        if (k1) c3 = s_hat_bub(S, dr, 0, 1);
      }
      const int iL = nh + max(eL, 0), iR = nh + min(eR, n - 1);  // absent elements: zero coefficients
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double rr = Fr[r][t];
        rr -= c0 * Ur[r][iL];
        if (k1) rr -= c1 * Ur[r][n + iL];
        rr -= c2 * Ur[r][iR];
        if (k1) rr -= c3 * Ur[r][n + iR];
        H[r][t] = rr;
      }
    }
    __syncthreads();
    // 3. hat Schur solve: y_t = il_t r_t - (g_t il_t) y_{t+1} (t descending),
    //    then x_t = il_t y_t - (g_{t-1} il_t) x_{t-1} (t ascending), each as
    //    block maps + scan + local sweep; loads HU hats ahead, the factors
    //    once for the RB rows
    if (nh > 0) {
      Aff fm[RB];
      double v[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) fm[r] = Aff{0.0, 1.0};
      for (int t0 = tb - 1; t0 >= ta; t0 -= HU) {
        double hv[RB][HU], lv[HU], hd[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 - u >= ta ? t0 - u : ta;
          lv[u] = ilh[t];
          hd[u] = gh[t] * lv[u];
#pragma unroll
          for (int r = 0; r < RB; ++r) hv[r][u] = H[r][t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 - u >= ta) {
#pragma unroll
            for (int r = 0; r < RB; ++r) fm[r] = Aff{fma(-hd[u], fm[r].a, lv[u] * hv[r][u]), -hd[u] * fm[r].b};
          }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) v[r] = enter_down(fm[r], sa, sb);
      for (int t0 = tb - 1; t0 >= ta; t0 -= HU) {
        double hv[RB][HU], lv[HU], hd[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 - u >= ta ? t0 - u : ta;
          lv[u] = ilh[t];
          hd[u] = gh[t] * lv[u];
#pragma unroll
          for (int r = 0; r < RB; ++r) hv[r][u] = H[r][t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 - u >= ta) {
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              v[r] = fma(-hd[u], v[r], lv[u] * hv[r][u]);
              H[r][t0 - u] = v[r];
            }
          }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) fm[r] = Aff{0.0, 1.0};
      for (int t0 = ta; t0 < tb; t0 += HU) {
        double hv[RB][HU], lv[HU], hu[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 + u < tb ? t0 + u : tb - 1;
          lv[u] = ilh[t];
          hu[u] = (t > 0 ? gh[t - 1] : 0.0) * lv[u];
#pragma unroll
          for (int r = 0; r < RB; ++r) hv[r][u] = H[r][t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 + u < tb) {
#pragma unroll
            for (int r = 0; r < RB; ++r) fm[r] = Aff{fma(-hu[u], fm[r].a, lv[u] * hv[r][u]), -hu[u] * fm[r].b};
          }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) v[r] = enter_up(fm[r], sa, sb);
      for (int t0 = ta; t0 < tb; t0 += HU) {
        double hv[RB][HU], lv[HU], hu[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          const int t = t0 + u < tb ? t0 + u : tb - 1;
          lv[u] = ilh[t];
          hu[u] = (t > 0 ? gh[t - 1] : 0.0) * lv[u];
#pragma unroll
          for (int r = 0; r < RB; ++r) hv[r][u] = H[r][t];
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
          if (t0 + u < tb) {
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              v[r] = fma(-hu[u], v[r], lv[u] * hv[r][u]);
              H[r][t0 + u] = v[r];
            }
          }
      }
      __syncthreads();
      if (hats_in_smem)
        for (int t = threadIdx.x; t < nh; t += NT1) {
#pragma unroll
          for (int r = 0; r < RB; ++r) Ur[r][t] = H[r][t];
        }
    }
    // 4. up sweeps L z = y with the bubble correction fused:
    //    x_c = z_c - v_L x_hL - v_R x_hR, written once
    for (int ch = threadIdx.x; ch < 2 * n; ch += NT1) {
      const int pi = ch < n ? 0 : 1, e = ch - pi * n;
      const int mm = chain_len(d.p, pi);
      const int pe = pi * n + e;
      const int hlt = hat_of_node(e, n, d.bc), hrt = hat_of_node(e + 1, n, d.bc);
      const bool hl = hlt >= 0, hr = hrt >= 0;
      double z[RB], xl[RB], xr[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        xl[r] = (mm > 0 && hl) ? H[r][hlt] : 0.0;  // 0: the term is skipped below
        xr[r] = (mm > 0 && hr) ? H[r][hrt] : 0.0;
        z[r] = 0.0;
      }
      double gp = 0.0;
      for (int c0 = 0; c0 < m0; c0 += CBU) {
        double yv[RB][CBU], gv[CBU], lv[CBU], vl[CBU], vr[CBU];
#pragma unroll
        for (int u = 0; u < CBU; ++u) {
          const int c = c0 + u;
          const bool ok = c < mm;
          const int b = pe + 2 * (ok ? c : 0) * n;
          gv[u] = ok ? g[b] : 0.0;
          lv[u] = ok ? il[b] : 0.0;
          vl[u] = ok ? f.vL[b] : 0.0;
          vr[u] = ok ? f.vR[b] : 0.0;
#pragma unroll
          for (int r = 0; r < RB; ++r) yv[r][u] = ok ? Ur[r][nh + b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CBU; ++u) {
          const int c = c0 + u;
          if (c < mm) {
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              z[r] = c == 0 ? yv[r][u] : (yv[r][u] - gp * z[r]) * lv[u];  // slot 0 holds z_0
              double x = z[r];
              if (hl) x -= vl[u] * xl[r];
              if (hr) x -= vr[u] * xr[r];
              Ur[r][nh + pe + 2 * c * n] = x;
            }
            gp = gv[u];
          }
        }
      }
    }
    __syncthreads();  // H (shared) is rewritten by the next group
  }
}

template <int RB>
static cudaError_t launch_solve1d_rb(const DirDev& d, const FacView& f, int nrhs, const double* F, double* U,
                                     cudaStream_t st) {
  // hats in shared memory when they are few enough not to limit occupancy
  const size_t hb = sizeof(double) * (size_t)d.nh * RB;
  const int in_smem = hb <= 48 * 1024 ? 1 : 0;
  const size_t smem = in_smem ? hb : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one wave of up to 8 resident CTAs per SM, grid-stride over the rest
  long long g = 8LL * sms;
  const long long groups = (nrhs + RB - 1) / RB;
  if (g > groups) g = groups;
  k_solve1d<RB><<<(unsigned)g, NT1, smem, st>>>(d, f, nrhs, in_smem, F, U);
  return cudaGetLastError();
}

/* ------------------------------------------------------------------ */
/* Cluster form (round 2): one thread-block CLUSTER per right-hand side, */
/* the row's down-sweep values held in the distributed shared memory of  */
/* its CTAs instead of making a round trip through the output row -- F   */
/* is read once and U written once (the 16 algorithmic bytes per dof;    */
/* the kernel above moves 32).  CTA r of the cluster owns the elements   */
/* [r EPC, (r+1) EPC) with their chains and left nodes (the last CTA     */
/* also node n).  The hat Schur recurrences cross the cluster as affine  */
/* maps: block maps per thread, a CTA scan that keeps the maps (not just */
/* their value at entry 0), the CTA totals exchanged through             */
/* distributed shared memory -- 4 cluster barriers per right-hand side.  */
/* Chain-first values and hat values of the neighbouring CTA (one        */
/* element / node each) are read remotely.                               */
/* ------------------------------------------------------------------ */
namespace {

/* exclusive suffix composition over the CTA's threads: the map from the value
 * entering the CTA's LAST thread to the value entering this thread (down
 * sweep, the recurrence runs from the last thread to the first); total = the
 * whole CTA's map.  f: this thread's block map. */
__device__ Aff suffix_maps(Aff f, double* sa, double* sb, Aff& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
  Aff C{0.0, 1.0};  // later warps: the value passes through warp nw-1 first
  for (int u = nw - 1; u > w; --u) C = after(Aff{sa[u], sb[u]}, C);
  Aff nx{__shfl_down_sync(0xffffffffu, f.a, 1), __shfl_down_sync(0xffffffffu, f.b, 1)};
  if (lane == 31) nx = Aff{0.0, 1.0};
  Aff T0{sa[0], sb[0]};
  Aff C0{0.0, 1.0};
  for (int u = nw - 1; u > 0; --u) C0 = after(Aff{sa[u], sb[u]}, C0);
  total = after(T0, C0);
  __syncthreads();  // sa / sb reused
  return after(nx, C);
}

/* the same for a recurrence from the first thread to the last (up sweep) */
__device__ Aff prefix_maps(Aff f, double* sa, double* sb, Aff& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
  Aff C{0.0, 1.0};  // earlier warps: the value passes through warp 0 first
  for (int u = 0; u < w; ++u) C = after(Aff{sa[u], sb[u]}, C);
  Aff pv{__shfl_up_sync(0xffffffffu, f.a, 1), __shfl_up_sync(0xffffffffu, f.b, 1)};
  if (lane == 0) pv = Aff{0.0, 1.0};
  Aff Ct{0.0, 1.0};
  for (int u = 0; u < nw; ++u) Ct = after(Aff{sa[u], sb[u]}, Ct);
  total = Ct;
  __syncthreads();
  return after(pv, C);
}

__device__ __forceinline__ int hpd(int i) { return i + (i >> 3); }  // padded hat slot (conflict-free blocks)

}  // namespace

struct Solve1dClSmem {
  int EPC, LC;  // elements per CTA, chains per CTA
  size_t y, zf, hs, tot, sc, total;  // byte offsets
};
__host__ __device__ inline Solve1dClSmem solve1d_cl_smem(int n, int p, int cs) {
  Solve1dClSmem m;
  m.EPC = (n + cs - 1) / cs;
  m.LC = 2 * m.EPC;
  const size_t m0 = (size_t)(p / 2);
  m.y = 0;
  m.zf = m.y + m0 * m.LC * 8;
  m.hs = m.zf + (size_t)2 * (m.EPC + 1) * 8;
  m.tot = m.hs + (size_t)(m.EPC + 2 + (m.EPC + 2) / 8 + 1) * 8;
  m.sc = m.tot + 4 * 8;
  m.total = m.sc + 2 * 32 * 8;
  return m;
}

__global__ void __launch_bounds__(NT1) k_solve1d_cl(DirDev d, FacView f, int nrhs, int cs, const double* __restrict__ F,
                                                       double* __restrict__ U) {
  extern __shared__ __align__(16) unsigned char sm1[];
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const Solve1dClSmem M = solve1d_cl_smem(d.n, d.p, cs);
  double* ysm = reinterpret_cast<double*>(sm1 + M.y);   // [c][LC]: down-sweep values (slot 0: z_0)
  double* zf = reinterpret_cast<double*>(sm1 + M.zf);   // [2][EPC + 1]: chain-first z of elements E0-1 .. E1-1
  double* Hs = reinterpret_cast<double*>(sm1 + M.hs);   // hat values of nodes E0 .. (padded slots)
  double* tot = reinterpret_cast<double*>(sm1 + M.tot); // CTA total maps: down (a, b), up (a, b)
  double* sa = reinterpret_cast<double*>(sm1 + M.sc);
  double* sb = sa + 32;
  const int n = d.n, nh = d.nh, dl = drop_left(d.bc);
  const int EPC = M.EPC, LC = M.LC;
  const int E0 = min(n, cr * EPC), E1 = min(n, E0 + EPC), ne = E1 - E0;
  const bool own_last = ne > 0 && E1 == n;      // this CTA also owns node n
  const int nown = ne + (own_last ? 1 : 0);     // owned nodes E0 .. E0 + nown - 1
  const double* __restrict__ il = f.il;
  const double* __restrict__ g = f.g;
  const double S = f.sig;
  const bool k1 = d.p - 2 >= 1;
  const int m0 = chain_len(d.p, 0);
  const int HB = (nown + NT1 - 1) / NT1;
  const int ia = min(nown, (int)threadIdx.x * HB), ib = min(nown, ia + HB);  // this thread's nodes (local)
  const int ncl = gridDim.x / cs;
  for (int rhs = blockIdx.x / cs; rhs < nrhs; rhs += ncl) {
    const double* __restrict__ Fr = F + (size_t)rhs * d.N;
    double* __restrict__ Ur = U + (size_t)rhs * d.N;
    // 1. down sweeps of the owned chains into shared memory (slot 0: z_0 = il_0 y_0).
    //    (Staging the slice of F through shared memory first and sweeping in
    //    place, so that every DRAM load is in flight at once, measured slower:
    //    single row 19 -> 31 us at N = 65535, p = 64.)
    for (int lc = threadIdx.x; lc < 2 * ne; lc += NT1) {
      const int pi = lc < ne ? 0 : 1, el = lc - pi * ne, e = E0 + el;
      const int mm = chain_len(d.p, pi);
      const int pe = pi * n + e;
      const int col = pi * EPC + el;
      double y = 0.0;
      for (int c0 = m0 - 1; c0 >= 0; c0 -= CB) {
        double fv[CB], gv[CB], lv[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int c = c0 - u;
          const bool ok = c >= 0 && c < mm;
          const int b = pe + 2 * (ok ? c : 0) * n;
          fv[u] = ok ? Fr[nh + b] : 0.0;
          gv[u] = ok ? g[b] : 0.0;
          lv[u] = ok ? il[b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int c = c0 - u;
          if (c >= 0 && c < mm) {
            y = (fv[u] - gv[u] * y) * lv[u];
            ysm[(size_t)c * LC + col] = c == 0 ? y * lv[u] : y;
            if (c == 0) zf[pi * (EPC + 1) + el + 1] = y * lv[u];
          }
        }
      }
      if (mm == 0) zf[pi * (EPC + 1) + el + 1] = 0.0;
    }
    cluster.sync();  // (1) chain-first values visible to the next CTA
    if (threadIdx.x < 2) {  // halo: element E0 - 1 of the previous CTA
      double v = 0.0;
      if (cr > 0 && ne > 0) {
        const double* rz = cluster.map_shared_rank(zf, cr - 1);
        v = rz[threadIdx.x * (EPC + 1) + EPC];  // its last element (the previous CTA is full)
      }
      zf[threadIdx.x * (EPC + 1)] = v;
    }
    __syncthreads();
    // 2. hat right-hand sides of the owned nodes
    for (int i = threadIdx.x; i < nown; i += NT1) {
      const int node = E0 + i, t = node - dl;
      double rr = 0.0;
      if (t >= 0 && t < nh) {
        rr = Fr[t];
        const int eL = node - 1, eR = node;
        if (eL >= 0) {
          const double dlt = d.delta[eL];
          rr -= s_hat_bub(S, dlt, 1, 0) * zf[i];
          if (k1) rr -= s_hat_bub(S, dlt, 1, 1) * zf[(EPC + 1) + i];
        }
        if (eR <= n - 1) {
          const double drt = d.delta[eR];
          rr -= s_hat_bub(S, drt, 0, 0) * zf[i + 1];
          if (k1) rr -= s_hat_bub(S, drt, 0, 1) * zf[(EPC + 1) + i + 1];
        }
      }
      Hs[hpd(i)] = rr;
    }
    __syncthreads();
    // 3. hat Schur solve across the cluster (dropped nodes: identity maps, value 0)
    {
      Aff fm{0.0, 1.0};
      for (int i = ib - 1; i >= ia; --i) {
        const int t = E0 + i - dl;
        if (t >= 0 && t < nh) {
          const double l = f.ilh[t], hd = f.gh[t] * l;
          fm = Aff{fma(-hd, fm.a, l * Hs[hpd(i)]), -hd * fm.b};
        }
      }
      Aff T;
      const Aff Sx = suffix_maps(fm, sa, sb, T);
      if (threadIdx.x == 0) {
        tot[0] = T.a;
        tot[1] = T.b;
      }
      cluster.sync();  // (2) CTA totals of the down sweep
      double E = 0.0;
      for (int r = cs - 1; r > cr; --r) {
        const double* rt = cluster.map_shared_rank(tot, r);
        E = fma(rt[1], E, rt[0]);
      }
      double v = fma(Sx.b, E, Sx.a);
      for (int i = ib - 1; i >= ia; --i) {
        const int t = E0 + i - dl;
        if (t >= 0 && t < nh) {
          const double l = f.ilh[t];
          v = fma(-(f.gh[t] * l), v, l * Hs[hpd(i)]);
          Hs[hpd(i)] = v;
        }
      }
      fm = Aff{0.0, 1.0};
      for (int i = ia; i < ib; ++i) {
        const int t = E0 + i - dl;
        if (t >= 0 && t < nh) {
          const double l = f.ilh[t], hu = (t > 0 ? f.gh[t - 1] : 0.0) * l;
          fm = Aff{fma(-hu, fm.a, l * Hs[hpd(i)]), -hu * fm.b};
        }
      }
      const Aff Px = prefix_maps(fm, sa, sb, T);
      if (threadIdx.x == 0) {
        tot[2] = T.a;
        tot[3] = T.b;
      }
      cluster.sync();  // (3) CTA totals of the up sweep
      E = 0.0;
      for (int r = 0; r < cr; ++r) {
        const double* rt = cluster.map_shared_rank(tot, r);
        E = fma(rt[3], E, rt[2]);
      }
      v = fma(Px.b, E, Px.a);
      for (int i = ia; i < ib; ++i) {
        const int t = E0 + i - dl;
        if (t >= 0 && t < nh) {
          const double l = f.ilh[t];
          v = fma(-((t > 0 ? f.gh[t - 1] : 0.0) * l), v, l * Hs[hpd(i)]);
          Hs[hpd(i)] = v;
          Ur[t] = v;
        }
      }
    }
    cluster.sync();  // (4) hat values visible to the previous CTA
    if (threadIdx.x == 0 && ne > 0 && !own_last) {  // node E1 belongs to the next CTA
      const double* rh = cluster.map_shared_rank(Hs, cr + 1);
      Hs[hpd(ne)] = rh[0];
    }
    __syncthreads();
    // 4. up sweeps with the bubble correction fused, written once
    for (int lc = threadIdx.x; lc < 2 * ne; lc += NT1) {
      const int pi = lc < ne ? 0 : 1, el = lc - pi * ne, e = E0 + el;
      const int mm = chain_len(d.p, pi);
      const int pe = pi * n + e;
      const int col = pi * EPC + el;
      const bool hl = hat_of_node(e, n, d.bc) >= 0, hr = hat_of_node(e + 1, n, d.bc) >= 0;
      const double xl = hl ? Hs[hpd(el)] : 0.0, xr = hr ? Hs[hpd(el + 1)] : 0.0;
      double z = 0.0, gp = 0.0;
      for (int c0 = 0; c0 < m0; c0 += CBU) {
        double gv[CBU], lv[CBU], vl[CBU], vr[CBU];
#pragma unroll
        for (int u = 0; u < CBU; ++u) {
          const int c = c0 + u;
          const bool ok = c < mm;
          const int b = pe + 2 * (ok ? c : 0) * n;
          gv[u] = ok ? g[b] : 0.0;
          lv[u] = ok ? il[b] : 0.0;
          vl[u] = ok ? f.vL[b] : 0.0;
          vr[u] = ok ? f.vR[b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CBU; ++u) {
          const int c = c0 + u;
          if (c < mm) {
            const double yv = ysm[(size_t)c * LC + col];
            z = c == 0 ? yv : (yv - gp * z) * lv[u];  // slot 0 holds z_0
            gp = gv[u];
            double x = z;
            if (hl) x -= vl[u] * xl;
            if (hr) x -= vr[u] * xr;
            Ur[nh + pe + 2 * c * n] = x;
          }
        }
      }
    }
    // (the next row's first cluster barrier orders its shared-memory writes
    // after every remote read of this row)
  }
  cluster.sync();  // no CTA exits while a neighbour may still read its shared memory
}

/* cluster size of the cluster form (0 = not applicable): the smallest that
 * lets three (else two, else one) CTAs share an SM */
static int solve1d_cluster_size(const DirDev& d) {
  for (size_t cap : {(size_t)72 * 1024, (size_t)110 * 1024, (size_t)220 * 1024})
    for (int cs : {1, 2, 4, 8})
      if (d.n >= cs && solve1d_cl_smem(d.n, d.p, cs).total <= cap) return cs;
  return 0;
}

static cudaError_t launch_solve1d_cl(const DirDev& d, const FacView& f, int nrhs, int cs, const double* F, double* U,
                                     cudaStream_t st) {
  const size_t smem = solve1d_cl_smem(d.n, d.p, cs).total;
  cudaError_t e = smem_optin((const void*)k_solve1d_cl, 227 * 1024);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = smem <= 72 * 1024 ? 3 : (smem <= 110 * 1024 ? 2 : 1);
  long long ncl = (long long)sms * per_sm / cs;
  if (ncl > nrhs) ncl = nrhs;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * cs));
  cfg.blockDim = dim3(NT1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_solve1d_cl, d, f, nrhs, cs, F, U);
}

cudaError_t launch_solve1d(const DirDev& d, const FacView& f, int nrhs, const double* F, double* U,
                           cudaStream_t st) {
  if (nrhs <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {  // Cluster form for batches that one round of resident clusters covers (a
     // latency kernel: single row at N = 65535 0.34 -> 0.038 ms at p = 4, 0.083
     // -> 0.019 ms at p = 64; its 4 cluster barriers per row make it 2-3x
     // slower than the row-per-CTA kernel at 1024 rows).  HPFEM_1D_CLUSTER=0
     // disables it, =1 forces it for any batch (tests).
    const char* v = std::getenv("HPFEM_1D_CLUSTER");
    const int mode = v ? std::atoi(v) : -1;
    const int cs = mode == 0 ? 0 : solve1d_cluster_size(d);
    if (cs > 0) {
      const size_t smem = solve1d_cl_smem(d.n, d.p, cs).total;
      const int per_sm = smem <= 72 * 1024 ? 3 : (smem <= 110 * 1024 ? 2 : 1);
      if (mode == 1 || (long long)nrhs * cs <= (long long)sms * per_sm)
        return launch_solve1d_cl(d, f, nrhs, cs, F, U, st);
    }
  }
  // two rows per CTA once there are enough rows to fill the SMs twice over
  // (measured at 1024 rows, N = 65535: 1 / 2 / 4 rows per CTA 0.578 / 0.498 /
  // 0.531 ms at p = 256, 1.97 / 1.63 / 1.80 ms at p = 4)
  if (nrhs >= 4 * sms) return launch_solve1d_rb<2>(d, f, nrhs, F, U, st);
  return launch_solve1d_rb<1>(d, f, nrhs, F, U, st);
}

}  // namespace hpfem
