/*
 * tma_step.cu -- TMA-fed, warp-specialised persistent half-step kernels
 * (K2-K4 for the bubble lines) for sm_100a.
 *
 * One ADI half-step (Alg. 2) = for every line: evaluate the
 * cross-line sparse apply of the other direction on the previous iterate,
 * then solve the element-local bubble chains (static condensation of the
 * reverse-Cholesky solve, Cor. 4.3 P:L600-L614 / P:L636-L638).
 *
 * Data movement: one elected producer thread streams the tiles a CTA needs
 * from HBM into a ring of shared-memory stages with cp.async.bulk.tensor
 * (TMA), completion tracked by mbarriers; eight consumer warps evaluate the
 * stencil from shared memory (each W value is fetched once per CTA and reused
 * by the 3-5 lines that need it) and run the chain recurrences with the
 * chain held in registers.  The producer runs ahead across tile boundaries
 * (persistent CTAs), so HBM stays busy while the consumers do the upward
 * sweep and the stores of a finished tile.
 *
 *  x-solve (DIR 0, lines = y-bubble columns):  tile = (x-element e_x,
 *    x-parity, a group of EG0 y-elements); stage c = one row d_c of the x-chain:
 *    G and W boxes [p_y-1][EG0] of the 3D view (e_y, k_y, row) plus the few
 *    y-hat columns the tile's stencils touch.  The y-stencil (k_y, k_y +- 2,
 *    hats) lies entirely inside the tile: no halo.
 *  y-solve (DIR 1, lines = x-bubble rows):  tile = (x-element e_x, x-parity,
 *    R consecutive rows of that x-chain, a group of EG1 y-elements); stage c =
 *    chain position c (y-degrees 2c, 2c+1): G box [R][2][EG1], W box
 *    [R+2][2][EG1] (the x-stencil rows k_x-2 .. k_x+2R of the same x-chain)
 *    and the two x-hat rows of e_x.  W rows are reused R/(R+2) from smem.
 *
 * Hat lines (n+-1 of them) are left to the LDG kernel of kernels.cu.
 */
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cstdio>

#include "hpfem_internal.h"
#include "ops1d.h"
#include "tma_step.h"
#include "ptx.cuh"

namespace hpfem {

/* the cross-line stencil (same construction as kernels.cu), device copy */
struct Sten5 {
  double w[5];  // weights of [l, l-2n, l+2n, hL, hR] (0 where absent)
};

__device__ __forceinline__ void sten5_build(const DirDev& o, int l, int mode, double kap, double tau,
                                            const double* __restrict__ cvL, const double* __restrict__ cvR,
                                            Sten5& st) {
  // l is a bubble dof (k, e) of direction o
  const int n = o.n, b = l - o.nh, k = b / n, e = b - k * n;
#pragma unroll
  for (int q = 0; q < 5; ++q) st.w[q] = 0.0;
  const bool hL = hat_of_node(e, n, o.bc) >= 0, hR = hat_of_node(e + 1, n, o.bc) >= 0;
  if (mode == ST_CORR) {
    st.w[0] = 1.0;
    if (hL && cvL) st.w[3] = -cvL[b];
    if (hR && cvR) st.w[4] = -cvR[b];
    return;
  }
  if (mode != ST_APPLY) return;
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
  st.w[0] = -sd;
  st.w[1] = -sm;
  st.w[2] = -sp;
  st.w[3] = hL ? -cL : 0.0;
  st.w[4] = hR ? -cR : 0.0;
}

/* n / d for 0 <= n < 2^31 by multiply-high (divisor fixed per launch) */
struct FDiv {
  uint32_t d, m, l;
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};

static inline FDiv make_fdiv(uint32_t d) {
  FDiv f;
  f.d = d < 1 ? 1 : d;
  f.l = 0;
  while ((1u << f.l) < f.d) ++f.l;
  f.m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << f.l) - f.d)) / f.d + 1);
  return f;
}

struct TmaStepArgs {
  StepParams P;
  int EG;           // y-elements per tile
  int R;            // rows per tile (y-solve)
  int ntiles;
  int nstages;      // ring depth NST (<= S, see below)
  int S;            // stages per tile (the same for every tile of a launch)
  int stage_bytes;  // bytes per ring stage (all boxes, 128-aligned)
  int off_w, off_h; // byte offsets of the W and hat boxes inside a stage
  int hi_g, hi_w, hi_h;  // two-threads-per-chain x kernel: byte offsets of the upper-half boxes from the lower ones
  int tx_bytes;     // bytes the TMA delivers per stage
  int hw;           // hat box width (x-solve)
  int out_off;      // y-solve: byte offset of the two output staging buffers
  int fac_off;      // byte offset of the two per-tile factor buffers
  int fac_doubles;  // doubles per factor buffer
  int fake_stencil; // experiment only (HPFEM_FAKE_STENCIL=1): skip the per-tile stencil build
  int wb_off;       // byte offset of the two per-tile stencil-weight buffers (when P.wtab)
  int wb_doubles;   // doubles per weight buffer
  int bar_off;      // byte offset of the full barriers [NST] and release counters [NST]
  int nwt;          // y-solve: row windows per x-element (both parities)
  FDiv fS, fN, fG, fT;  // divisions by S, NST, #element groups, and x.n (x-solve) / nwt (y-solve)
};

/* HPFEM_CHECKS (debug builds: HPFEM_NVCC_EXTRA=-DHPFEM_CHECKS): device-side
 * bounds checks of the ring / tile bookkeeping (trap on violation) and a NaN
 * poison of the whole ring before the first TMA issue, so that a stage read
 * before its bytes landed propagates NaN into the solution (the parity tests
 * then fail).  compute-sanitizer is closed on this pool; this is the
 * substitute (tests/test_gpu_parity.py, scripts/r2_checks.sh). */
#ifdef HPFEM_CHECKS
#define HPFEM_CHECK(cond) \
  do {                    \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define HPFEM_CHECK(cond) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ void poison_ring(unsigned char* ring, int bytes) {
#ifdef HPFEM_CHECKS
  double* r = reinterpret_cast<double*>(ring);
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) r[i] = __longlong_as_double(0x7ff8dead0000beefLL);
  fence_proxy_async();  // the generic-proxy poison before the async-proxy (TMA) fills
#else
  (void)ring;
  (void)bytes;
#endif
}

constexpr int NT = 256;    // threads per CTA
constexpr int NW = NT / 32;
constexpr int KR = 8;      // x-solve: chain positions (rows) per stage
constexpr int KCP = 8;     // y-solve: chain positions per stage (16 degrees)
#ifndef HPFEM_SPB
#define HPFEM_SPB 2
#endif
constexpr int SPB = HPFEM_SPB;  // y-solve: chain stages per output staging buffer (one proxy fence each)
#ifndef HPFEM_NOBUF
#define HPFEM_NOBUF 2
#endif
constexpr int NOBUF = HPFEM_NOBUF;  // y-solve: output staging buffers per warp
constexpr int KBOX = 16;   // y-solve: degrees per box row (one 128-byte line, 128B-swizzled in smem)

/* y-solve boxes are 128-byte rows stored with the TMA 128B swizzle: the
 * 16-byte chunk j of box row rho sits at chunk j ^ (rho & 7), so the lanes of
 * a warp (different rows rho = (row, element), same degree) hit different
 * banks.  Offset in doubles of degree (py + 2u) of box row rho: */
__device__ __forceinline__ int swz(int rho, int u, int py) { return rho * 16 + ((u ^ (rho & 7)) << 1) + py; }

/* Ring discipline.  Every tile of a launch has the same number S of stages
 * and this CTA's stages are numbered gs = 0, 1, ... in consumption order
 * (tile-local index gs / S, stage S-1 - gs % S of it); stage gs lives in slot
 * gs % NST and is complete when full[slot] flips.  There is no producer
 * thread: each warp, after reading a stage, bumps the slot's release counter,
 * and the warp that releases it LAST issues stage gs + NST into it (a handful
 * of instructions: the coordinates are a pure function of gs).  No warp ever
 * waits for another to release a slot.  A tile's chain factors (and stencil
 * weights) ride with its first stage into buffer (tile-local index & 1);
 * with NST <= S the first stage of tile t is issued only after every warp has
 * read a stage of tile t-1, i.e. after every warp has finished tile t-2,
 * the last user of that buffer. */
__device__ __forceinline__ bool release_is_last(uint32_t* cnt, int slot) {
  // acq_rel atomic: this warp's reads of the slot happen-before the last
  // releaser's refill; the reset of the counter is published by that warp's
  // mbarrier.arrive.expect_tx (release) before any consumer can bump it again
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(su32(&cnt[slot])) : "memory");
  if (old != NW - 1) return false;
  cnt[slot] = 0;
  fence_proxy_async();  // generic-proxy reads of the slot before the async-proxy (TMA) overwrite
  return true;
}

/* ------------------------------------------------------------------ */
/* x-solve (DIR 0), element-major layout                               */
/* tile = (x-element e_x, x-parity pi, group of EG y-elements); stage  */
/* s = chain positions [KR s, KR s + KR) of the x-chain (rows)         */
/* ------------------------------------------------------------------ */
template <int MODE, bool SPILL>
__device__ __forceinline__ void x_issue(const TmaStepArgs& A, uint32_t gs, unsigned char* ring, uint64_t* full,
                                        const CUtensorMap* mG0, const CUtensorMap* mG1, const CUtensorMap* mW0,
                                        const CUtensorMap* mW1, const CUtensorMap* mH0, const CUtensorMap* mH1,
                                        double* fbuf) {
  const StepParams& P = A.P;
  const DirDev& x = P.s;
  const DirDev& y = P.o;
  const uint32_t tl = A.fS.div(gs);
  const int s = A.S - 1 - (int)(gs - tl * A.S);
  const int tile = blockIdx.x + (int)tl * gridDim.x;
  if (tile >= A.ntiles) return;
  const int slot = (int)(gs - A.fN.div(gs) * A.nstages);
  const int rest = (int)A.fG.div(tile), g = tile - rest * (int)A.fG.d;
  const int pi = (int)A.fT.div(rest), e_x = rest - pi * x.n;
  HPFEM_CHECK(slot >= 0 && slot < A.nstages && s >= 0 && s < A.S && pi >= 0 && pi < 2 && e_x >= 0 && e_x < x.n &&
              g >= 0 && g * A.EG < y.n && A.tx_bytes <= A.stage_bytes);
  const int EG = A.EG;
  const int c0 = P.lay.hb + g * EG * P.lay.Q;
  const int hc = (g * EG - drop_left(y.bc)) & ~1;  // innermost TMA coordinate: 16-byte aligned
  const int row = KR * s < chain_len(x.p, pi) ? KR * s : 0;  // a stage past this parity's chain: any rows (unused)
  unsigned char* st = ring + (size_t)slot * A.stage_bytes;
  if (s == A.S - 1) {  // the tile's chain factors ride with its first stage
    const uint32_t fb = tl & 1;
    const uint32_t fbytes = P.f.cfs * 8;
    const int ne = (y.n - g * EG) < EG ? (y.n - g * EG) : EG;
    const uint32_t wbytes = P.wtab ? ne * 5 * P.lay.Q * 8 : 0;
    mbar_expect_tx(&full[slot], A.tx_bytes + fbytes + wbytes);
    bulk_load(fbuf + fb * A.fac_doubles, P.f.cf + (size_t)(2 * e_x + pi) * P.f.cfs, fbytes, &full[slot]);
    if (wbytes)
      bulk_load(reinterpret_cast<unsigned char*>(fbuf) + (A.wb_off - A.fac_off) + fb * A.wb_doubles * 8,
                P.wtab + (size_t)g * EG * 5 * P.lay.Q, wbytes, &full[slot]);
  } else {
    mbar_expect_tx(&full[slot], A.tx_bytes);
  }
  if (SPILL) {  // long chains: the streamed boxes leave L2 first (the parked values stay)
    const uint64_t pf = policy_evict_first();
    if (MODE != ST_CORR) tma_load_3d_hint(st, pi ? mG1 : mG0, &full[slot], c0, e_x, row, pf);
    if (MODE != ST_NONE) {
      tma_load_3d_hint(st + A.off_w, pi ? mW1 : mW0, &full[slot], c0, e_x, row, pf);
      tma_load_3d_hint(st + A.off_h, pi ? mH1 : mH0, &full[slot], hc, e_x, row, pf);
    }
    return;
  }
  if (MODE != ST_CORR) tma_load_3d(st, pi ? mG1 : mG0, &full[slot], c0, e_x, row);
  if (MODE != ST_NONE) {
    tma_load_3d(st + A.off_w, pi ? mW1 : mW0, &full[slot], c0, e_x, row);
    tma_load_3d(st + A.off_h, pi ? mH1 : mH0, &full[slot], hc, e_x, row);
  }
}

template <int CL, int MODE>
__global__ void __launch_bounds__(NT, 1) k_xstep_tma(const TmaStepArgs A, const __grid_constant__ CUtensorMap mG0,
                                                     const __grid_constant__ CUtensorMap mG1,
                                                     const __grid_constant__ CUtensorMap mW0,
                                                     const __grid_constant__ CUtensorMap mW1,
                                                     const __grid_constant__ CUtensorMap mH0,
                                                     const __grid_constant__ CUtensorMap mH1) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StepParams& P = A.P;
  const DirDev& x = P.s;  // solve direction
  const DirDev& y = P.o;  // apply direction
  const int NST = A.nstages;
  unsigned char* ring = smem_raw;
  double* fbuf = reinterpret_cast<double*>(smem_raw + A.fac_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + A.bar_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(full + NST);
  const int lane = threadIdx.x & 31;
  const int EG = A.EG, q = y.p - 1, Q = P.lay.Q, BW = EG * Q;
  const int ngroups = (y.n + EG - 1) / EG;
  if (threadIdx.x < NST) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) mbar_init(&full[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  poison_ring(ring, NST * A.stage_bytes);
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NST; ++k) x_issue<MODE, (CL > 64)>(A, k, ring, full, &mG0, &mG1, &mW0, &mW1, &mH0, &mH1, fbuf);
  const int tid = threadIdx.x;
  const int eo = tid / Q, ky = tid - eo * Q;
  const int mS = chain_len(x.p, 0);  // stages per tile cover the longer (even) chain
  int cslot = 0;
  uint32_t cround = 0, ctt = 0, gs = 0;
  for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++ctt) {
    const int g = tile % ngroups, rest = tile / ngroups;
    const int e_x = rest % x.n, pi = rest / x.n;
    const int e0 = g * EG, ey = e0 + eo;
    const int m = chain_len(x.p, pi);
    const double* fb = fbuf + (ctt & 1) * A.fac_doubles;  // [4c] il, [4c+1] g il, [4c+2] g_prev il
    const bool valid = eo < EG && ky < q && ey < y.n;
    const int h0 = (e0 - drop_left(y.bc)) & ~1;
    Sten5 st;
    int o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0;
    const bool wtab = P.wtab != nullptr && MODE == ST_APPLY;
    const double* wb = reinterpret_cast<const double*>(smem_raw + A.wb_off) + (ctt & 1) * A.wb_doubles;
    if (valid) {
      if (A.fake_stencil) { st.w[0] = -1.0; st.w[1] = st.w[2] = st.w[3] = st.w[4] = 0.0; }
      else if (!wtab) sten5_build(y, y.nh + ky * y.n + ey, MODE, P.kap_a, P.tau, P.cvL, P.cvR, st);
      o0 = eo * Q + ky;
      o1 = eo * Q + (ky >= 2 ? ky - 2 : ky);
      o2 = eo * Q + (ky + 2 < q ? ky + 2 : ky);
      const int hl = hat_of_node(ey, y.n, y.bc), hr = hat_of_node(ey + 1, y.n, y.bc);
      o3 = (hl >= 0 ? hl : h0 + 1) - h0;
      o4 = (hr >= 0 ? hr : h0 + 1) - h0;
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) st.w[k] = 0.0;
    }
    // chain positions [0, CR) stay in registers; longer chains (CL = 128:
    // the long direction of a transposed solve) park the down-
    // sweep values of positions >= CR at their final addresses in `out` (a
    // coalesced 256-byte row per warp, read back by the same thread in the up
    // sweep: an L2 round trip) and overwrite them with z.  The spilled stages
    // run as a rolled loop (the fully unrolled 128-position body overflowed
    // the instruction cache: ncu no_instruction stalls 12 per issue).
    constexpr int CR = CL > 64 ? 64 : CL;
    double ys[CR];
    double* __restrict__ outc = P.out + P.lay.hb + (size_t)(valid ? ey : 0) * Q + ky;
    auto orow = [&](int c) { return (size_t)(x.nh + (pi + 2 * c) * x.n + e_x) * P.ld; };
    double yv = 0.0;
    // one ring stage: wait, stencil of its KR rows, release, return r values
    auto stage_rhs = [&](int sg, double* rv) {
      const int slot = cslot;
      mbar_wait(&full[slot], cround & 1);
      if (wtab && KR * sg + KR >= mS) {  // first stage of the tile: the weights have landed
#pragma unroll
        for (int k = 0; k < 5; ++k) st.w[k] = valid ? wb[(eo * 5 + k) * Q + ky] : 0.0;
      }
      const unsigned char* stg = ring + (size_t)slot * A.stage_bytes;
#pragma unroll
      for (int kk = 0; kk < KR; ++kk) {
        const double* Gs = reinterpret_cast<const double*>(stg) + kk * BW;
        const double* Ws = reinterpret_cast<const double*>(stg + A.off_w) + kk * BW;
        const double* Hs = reinterpret_cast<const double*>(stg + A.off_h) + kk * A.hw;
        double r = 0.0;
        if (MODE != ST_CORR) r = Gs[o0];
        if (MODE != ST_NONE)
          r += st.w[0] * Ws[o0] + st.w[1] * Ws[o1] + st.w[2] * Ws[o2] + st.w[3] * Hs[o3] + st.w[4] * Hs[o4];
        rv[kk] = r;
      }
      __syncwarp();
      if (lane == 0 && release_is_last(cnt, slot))
        x_issue<MODE, (CL > 64)>(A, gs + NST, ring, full, &mG0, &mG1, &mW0, &mW1, &mH0, &mH1, fbuf);
      ++gs;
      if (++cslot == NST) {
        cslot = 0;
        ++cround;
      }
    };
    const uint64_t pkeep = CL > CR ? policy_evict_last() : 0;  // the parked values stay in L2
    if (CL > CR) {  // spilled stages (positions >= CR), rolled
#pragma unroll 1
      for (int sg = CL / KR - 1; sg >= CR / KR; --sg) {
        if (KR * sg < mS) {
          double rv[KR];
          stage_rhs(sg, rv);
#pragma unroll
          for (int kk = KR - 1; kk >= 0; --kk) {
            const int c = KR * sg + kk;
            if (c < m) {
              const double2 f = *reinterpret_cast<const double2*>(fb + 4 * c);  // (il, hd)
              yv = fma(-f.y, yv, f.x * rv[kk]);
              if (valid) st_hint(outc + orow(c), yv, pkeep);
            }
          }
        }
      }
    }
#pragma unroll
    for (int sg = CR / KR - 1; sg >= 0; --sg) {
      if (KR * sg < mS) {
        double rv[KR];
        stage_rhs(sg, rv);
#pragma unroll
        for (int kk = KR - 1; kk >= 0; --kk) {
          const int c = KR * sg + kk;
          if (c < m) {
            const double2 f = *reinterpret_cast<const double2*>(fb + 4 * c);  // (il, hd)
            yv = fma(-f.y, yv, f.x * rv[kk]);
            ys[c] = yv;
          }
        }
      }
    }
    if (valid) {
      double* __restrict__ out = outc;
      double z = 0.0;
      // factor pairs loaded KR at a time ahead of the stores (as in the y-solve)
#pragma unroll
      for (int c0 = 0; c0 < CR; c0 += KR) {
        if (c0 < m) {
          double2 fz[KR];
#pragma unroll
          for (int u = 0; u < KR; ++u) fz[u] = *reinterpret_cast<const double2*>(fb + 4 * (c0 + u) + 2);  // (hu, il)
#pragma unroll
          for (int u = 0; u < KR; ++u) {
            const int c = c0 + u;
            if (c < m) {
              z = fma(-fz[u].x, z, fz[u].y * ys[c]);
              out[orow(c)] = z;
            }
          }
        }
      }
      if (CL > CR) {  // spilled positions, rolled; y loaded one batch ahead
        double yn[KR];
#pragma unroll
        for (int u = 0; u < KR; ++u) yn[u] = CR + u < m ? ld_hint(out + orow(CR + u), pkeep) : 0.0;
#pragma unroll 1
        for (int c0 = CR; c0 < m; c0 += KR) {
          double yc[KR];
          double2 fz[KR];
#pragma unroll
          for (int u = 0; u < KR; ++u) {
            yc[u] = yn[u];
            fz[u] = *reinterpret_cast<const double2*>(fb + 4 * (c0 + u) + 2);  // (hu, il)
          }
#pragma unroll
          for (int u = 0; u < KR; ++u) {
            const int c = c0 + KR + u;
            yn[u] = c < m ? ld_hint(out + orow(c), pkeep) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < KR; ++u) {
            const int c = c0 + u;
            if (c < m) {
              z = fma(-fz[u].x, z, fz[u].y * yc[u]);
              out[orow(c)] = z;
            }
          }
        }
      }
    }
  }
}

/* ------------------------------------------------------------------ */
/* x-solve, chains of 65 .. 128 positions: two threads per chain       */
/* (round 2).  The lower half of a chain (positions 0-63) and its upper */
/* half (64-127) are held by the two half-warps of a warp, 64 positions */
/* in registers each, and swept concurrently: a first-order recurrence  */
/* over a half is affine in the value entering it, so each half sweeps  */
/* with entry 0 and the true entry (one shuffle at the end of the       */
/* sweep) is added through the tabled influence coefficients (spike     */
/* coefficients, hpfem_internal.h fac_spk_off):                         */
/*   z_c = u_c + zeta_c y_64  (c < 64),  z_c = u_c + gamma_c z_63 (c >= 64) */
/* Both half-warps run the same instructions (the entry is 0 where it   */
/* does not apply).  Same factors, same right-hand sides; the           */
/* association of the products differs from the sequential sweep        */
/* (rounding level, as the scan-form hat solves).  Against the          */
/* one-thread variant above (CL = 128: upper half parked in the output  */
/* row, rolled loops) nothing leaves the registers.                     */
/* tile = (e_x, parity, EG y-elements = <= 128 columns); stage s =      */
/* chain positions [8s, 8s+8) and [64+8s, 64+8s+8): two boxes per       */
/* array, the upper ones shifted by 128 bytes modulo 256 so the two     */
/* half-warps read different banks.                                     */
/* ------------------------------------------------------------------ */
constexpr int XH = 64;  // positions per half

template <int MODE>
__device__ __forceinline__ void x2_issue(const TmaStepArgs& A, uint32_t gs, unsigned char* ring, uint64_t* full,
                                         const CUtensorMap* mG0, const CUtensorMap* mG1, const CUtensorMap* mW0,
                                         const CUtensorMap* mW1, const CUtensorMap* mH0, const CUtensorMap* mH1,
                                         double* fbuf) {
  const StepParams& P = A.P;
  const DirDev& x = P.s;
  const DirDev& y = P.o;
  const uint32_t tl = A.fS.div(gs);
  const int s = A.S - 1 - (int)(gs - tl * A.S);
  const int tile = blockIdx.x + (int)tl * gridDim.x;
  if (tile >= A.ntiles) return;
  const int slot = (int)(gs - A.fN.div(gs) * A.nstages);
  const int rest = (int)A.fG.div(tile), g = tile - rest * (int)A.fG.d;
  const int pi = (int)A.fT.div(rest), e_x = rest - pi * x.n;
  HPFEM_CHECK(slot >= 0 && slot < A.nstages && s >= 0 && s < A.S && pi >= 0 && pi < 2 && e_x >= 0 && e_x < x.n &&
              g >= 0 && g * A.EG < y.n && A.tx_bytes <= A.stage_bytes);
  const int EG = A.EG;
  const int c0 = P.lay.hb + g * EG * P.lay.Q;
  const int hc = (g * EG - drop_left(y.bc)) & ~1;
  const int row = KR * s;  // rows past the chain: out of bounds, zero-filled (zero factors there)
  unsigned char* st = ring + (size_t)slot * A.stage_bytes;
  if (s == A.S - 1) {
    const uint32_t fb = tl & 1;
    const uint32_t fbytes = P.f.cfs * 8;
    const int ne = (y.n - g * EG) < EG ? (y.n - g * EG) : EG;
    const uint32_t wbytes = P.wtab ? ne * 5 * P.lay.Q * 8 : 0;
    mbar_expect_tx(&full[slot], A.tx_bytes + fbytes + wbytes);
    bulk_load(fbuf + fb * A.fac_doubles, P.f.cf + (size_t)(2 * e_x + pi) * P.f.cfs, fbytes, &full[slot]);
    if (wbytes)
      bulk_load(reinterpret_cast<unsigned char*>(fbuf) + (A.wb_off - A.fac_off) + fb * A.wb_doubles * 8,
                P.wtab + (size_t)g * EG * 5 * P.lay.Q, wbytes, &full[slot]);
  } else {
    mbar_expect_tx(&full[slot], A.tx_bytes);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (MODE != ST_CORR) tma_load_3d(st + h * A.hi_g, pi ? mG1 : mG0, &full[slot], c0, e_x, row + h * XH);
    if (MODE != ST_NONE) {
      tma_load_3d(st + A.off_w + h * A.hi_w, pi ? mW1 : mW0, &full[slot], c0, e_x, row + h * XH);
      tma_load_3d(st + A.off_h + h * A.hi_h, pi ? mH1 : mH0, &full[slot], hc, e_x, row + h * XH);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(NT, 1) k_xstep_tma2(const TmaStepArgs A, const __grid_constant__ CUtensorMap mG0,
                                                      const __grid_constant__ CUtensorMap mG1,
                                                      const __grid_constant__ CUtensorMap mW0,
                                                      const __grid_constant__ CUtensorMap mW1,
                                                      const __grid_constant__ CUtensorMap mH0,
                                                      const __grid_constant__ CUtensorMap mH1) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StepParams& P = A.P;
  const DirDev& x = P.s;
  const DirDev& y = P.o;
  const int NST = A.nstages;
  unsigned char* ring = smem_raw;
  double* fbuf = reinterpret_cast<double*>(smem_raw + A.fac_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + A.bar_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(full + NST);
  const int lane = threadIdx.x & 31;
  const int EG = A.EG, q = y.p - 1, Q = P.lay.Q, BW = EG * Q;
  const int ngroups = (y.n + EG - 1) / EG;
  if (threadIdx.x < NST) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) mbar_init(&full[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  poison_ring(ring, NST * A.stage_bytes);
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NST; ++k) x2_issue<MODE>(A, k, ring, full, &mG0, &mG1, &mW0, &mW1, &mH0, &mH1, fbuf);
  // thread -> (half h of the chain, column j of the tile)
  const int h = lane >> 4, j = (threadIdx.x >> 5) * 16 + (lane & 15);
  const int eo = j / Q, ky = j - eo * Q;
  const int cb = h * XH;  // first chain position of this thread's half
  const int spo = fac_spk_off(x);
  int cslot = 0;
  uint32_t cround = 0, ctt = 0, gs = 0;
  for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++ctt) {
    const int g = tile % ngroups, rest = tile / ngroups;
    const int e_x = rest % x.n, pi = rest / x.n;
    const int e0 = g * EG, ey = e0 + eo;
    const int m = chain_len(x.p, pi);
    const double* fb = fbuf + (ctt & 1) * A.fac_doubles;
    const double* fbh = fb + 4 * cb;        // this half's factors
    const double* sp = fb + spo + cb;       // this half's spike coefficients
    const bool valid = j < BW && ky < q && ey < y.n;
    const int h0 = (e0 - drop_left(y.bc)) & ~1;
    Sten5 st;
    int o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0;
    const bool wtab = P.wtab != nullptr && MODE == ST_APPLY;
    const double* wb = reinterpret_cast<const double*>(smem_raw + A.wb_off) + (ctt & 1) * A.wb_doubles;
    if (valid) {
      if (!wtab) sten5_build(y, y.nh + ky * y.n + ey, MODE, P.kap_a, P.tau, P.cvL, P.cvR, st);
      o0 = eo * Q + ky;
      o1 = eo * Q + (ky >= 2 ? ky - 2 : ky);
      o2 = eo * Q + (ky + 2 < q ? ky + 2 : ky);
      const int hl = hat_of_node(ey, y.n, y.bc), hr = hat_of_node(ey + 1, y.n, y.bc);
      o3 = (hl >= 0 ? hl : h0 + 1) - h0;
      o4 = (hr >= 0 ? hr : h0 + 1) - h0;
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) st.w[k] = 0.0;
    }
    double ys[XH];
    double yv = 0.0;
    // down sweep of both halves, entry 0
#pragma unroll
    for (int sg = XH / KR - 1; sg >= 0; --sg) {
      const int slot = cslot;
      mbar_wait(&full[slot], cround & 1);
      if (wtab && sg == XH / KR - 1) {  // first stage of the tile: the weights have landed
#pragma unroll
        for (int k = 0; k < 5; ++k) st.w[k] = valid ? wb[(eo * 5 + k) * Q + ky] : 0.0;
      }
      const unsigned char* stg = ring + (size_t)slot * A.stage_bytes;
      const double* Gb = reinterpret_cast<const double*>(stg + h * A.hi_g);
      const double* Wb = reinterpret_cast<const double*>(stg + A.off_w + h * A.hi_w);
      const double* Hb = reinterpret_cast<const double*>(stg + A.off_h + h * A.hi_h);
      double rv[KR];
#pragma unroll
      for (int kk = 0; kk < KR; ++kk) {
        const double* Gs = Gb + kk * BW;
        const double* Ws = Wb + kk * BW;
        const double* Hs = Hb + kk * A.hw;
        double r = 0.0;
        if (MODE != ST_CORR) r = Gs[o0];
        if (MODE != ST_NONE)
          r += st.w[0] * Ws[o0] + st.w[1] * Ws[o1] + st.w[2] * Ws[o2] + st.w[3] * Hs[o3] + st.w[4] * Hs[o4];
        rv[kk] = r;
      }
      __syncwarp();
      if (lane == 0 && release_is_last(cnt, slot))
        x2_issue<MODE>(A, gs + NST, ring, full, &mG0, &mG1, &mW0, &mW1, &mH0, &mH1, fbuf);
      ++gs;
      if (++cslot == NST) {
        cslot = 0;
        ++cround;
      }
#pragma unroll
      for (int kk = KR - 1; kk >= 0; --kk) {
        const int c = KR * sg + kk;
        const double2 f = *reinterpret_cast<const double2*>(fbh + 4 * c);  // (il, hd); zero past the chain
        yv = fma(-f.y, yv, f.x * rv[kk]);
        ys[c] = yv;
      }
    }
    // Each half has swept down with entry 0.  The true lower half is
    // y_c = a_c + beta_c y_64, so its up sweep is u_c + zeta_c y_64 with
    // zeta = L^{-1} beta tabled; the true upper half of the up sweep is
    // u_c + gamma_c z_63.  Both halves: one up sweep with entry 0, then one
    // tabled correction, z_c = u_c + t_c e (e = y_64 below, z_63 above).
    const double y64 = __shfl_sync(0xffffffffu, yv, (lane & 15) + 16);
    constexpr int UB = 8;
    double z = 0.0;
#pragma unroll
    for (int c0 = 0; c0 < XH; c0 += UB) {
      double2 fz[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) fz[u] = *reinterpret_cast<const double2*>(fbh + 4 * (c0 + u) + 2);  // (hu, il)
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int c = c0 + u;
        z = fma(-fz[u].x, z, fz[u].y * ys[c]);
        ys[c] = z;
      }
    }
    const double z63 = __shfl_sync(0xffffffffu, fma(sp[XH - 1], y64, z), lane & 15);  // (lower lanes: the true z_63)
    const double e2 = h ? z63 : y64;
    if (valid) {
      // row of chain position c: x.nh + (pi + 2 c) x.n + e_x, i.e. a fixed stride from the half's first row
      double* __restrict__ op =
          P.out + P.lay.hb + (size_t)ey * Q + ky + (size_t)(x.nh + (pi + 2 * cb) * x.n + e_x) * P.ld;
      const size_t rs = (size_t)2 * x.n * P.ld;
      const int mh = m - cb;  // positions of this half inside the chain
#pragma unroll
      for (int c0 = 0; c0 < XH; c0 += UB) {
        double sv[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) sv[u] = sp[c0 + u];
#pragma unroll
        for (int u = 0; u < UB; ++u)
          if (c0 + u < mh) op[(size_t)(c0 + u) * rs] = fma(sv[u], e2, ys[c0 + u]);
      }
    }
  }
}

/* ------------------------------------------------------------------ */
/* y-solve (DIR 1), element-major layout                               */
/* tile = (x-element e_x, x-parity, window of R rows of that x-chain,  */
/* group of EG y-elements); stage s = y-chain positions [8s, 8s+8)     */
/* ------------------------------------------------------------------ */
struct YTile {
  int e_x, pi, kw, g;
};

__device__ __forceinline__ YTile y_decode(const TmaStepArgs& A, int tile) {
  const DirDev& x = A.P.o;
  const int nw0 = (chain_len(x.p, 0) + A.R - 1) / A.R;
  YTile t;
  const int rest = (int)A.fG.div(tile);
  t.g = tile - rest * (int)A.fG.d;
  t.e_x = (int)A.fT.div(rest);
  const int w = rest - t.e_x * A.nwt;
  t.pi = w < nw0 ? 0 : 1;
  t.kw = t.pi == 0 ? w : w - nw0;
  return t;
}

template <int MODE>
__device__ __forceinline__ void y_issue(const TmaStepArgs& A, uint32_t gs, unsigned char* ring, uint64_t* full,
                                        const CUtensorMap* mG0, const CUtensorMap* mG1, const CUtensorMap* mW0,
                                        const CUtensorMap* mW1, const CUtensorMap* mH, double* fbuf) {
  const DirDev& y = A.P.s;
  const DirDev& x = A.P.o;
  const uint32_t tl = A.fS.div(gs);
  const int s = A.S - 1 - (int)(gs - tl * A.S);
  const int tile = blockIdx.x + (int)tl * gridDim.x;
  if (tile >= A.ntiles) return;
  const int slot = (int)(gs - A.fN.div(gs) * A.nstages);
  const YTile t = y_decode(A, tile);
  HPFEM_CHECK(slot >= 0 && slot < A.nstages && s >= 0 && s < A.S && t.pi >= 0 && t.pi < 2 && t.e_x >= 0 &&
              t.e_x < x.n && t.g >= 0 && t.g * A.EG < y.n && t.kw * A.R < chain_len(x.p, t.pi) &&
              A.tx_bytes <= A.stage_bytes);
  const int e0 = t.g * A.EG, kh0 = t.kw * A.R;
  const int hL = t.e_x - drop_left(x.bc);
  unsigned char* st = ring + (size_t)slot * A.stage_bytes;
  if (s == A.S - 1) {  // chain factors of the tile's EG elements x 2 parities (one contiguous block)
    const uint32_t fb = tl & 1;
    const int ne = (y.n - e0) < A.EG ? (y.n - e0) : A.EG;
    const uint32_t fbytes = 2 * ne * A.P.f.cfs * 8;
    const int mx = chain_len(x.p, 0), rows = (mx - kh0) < A.R ? (mx - kh0) : A.R;
    const uint32_t wbytes = A.P.wtab ? rows * 6 * 8 : 0;
    mbar_expect_tx(&full[slot], A.tx_bytes + fbytes + wbytes);
    bulk_load(fbuf + fb * A.fac_doubles, A.P.f.cf + (size_t)(2 * e0) * A.P.f.cfs, fbytes, &full[slot]);
    if (wbytes)
      bulk_load(reinterpret_cast<unsigned char*>(fbuf) + (A.wb_off - A.fac_off) + fb * A.wb_doubles * 8,
                A.P.wtab + ((size_t)(t.e_x * 2 + t.pi) * mx + kh0) * 6, wbytes, &full[slot]);
  } else {
    mbar_expect_tx(&full[slot], A.tx_bytes);
  }
  const int k0 = 2 * KCP * s;
  if (MODE != ST_CORR) tma_load_4d(st, t.pi ? mG1 : mG0, &full[slot], k0, e0, t.e_x, kh0);
  if (MODE != ST_NONE) {
    tma_load_4d(st + A.off_w, t.pi ? mW1 : mW0, &full[slot], k0, e0, t.e_x, kh0 - 1);
    tma_load_3d(st + A.off_h, mH, &full[slot], k0, e0, hL);
  }
}

template <int CL, int MODE, int EGT>
__global__ void __launch_bounds__(NT, 1)
    k_ystep_tma(const TmaStepArgs A, const __grid_constant__ CUtensorMap mG0, const __grid_constant__ CUtensorMap mG1,
                const __grid_constant__ CUtensorMap mW0, const __grid_constant__ CUtensorMap mW1,
                const __grid_constant__ CUtensorMap mH, const __grid_constant__ CUtensorMap mO0,
                const __grid_constant__ CUtensorMap mO1) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const StepParams& P = A.P;
  const DirDev& y = P.s;  // solve direction
  const DirDev& x = P.o;  // apply direction
  const int NST = A.nstages;
  unsigned char* ring = smem_raw;
  double* obuf = reinterpret_cast<double*>(smem_raw + A.out_off);  // 2 x NW x [RW][EG][16]
  double* fbuf = reinterpret_cast<double*>(smem_raw + A.fac_off);   // 2 x [EG][2][cfs]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + A.bar_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(full + NST);
  const int lane = threadIdx.x & 31;
  // EGT: the tile width as a compile-time constant, so that the swizzled box
  // addresses of the 6 stencil rows differ by immediates (one XOR per
  // position instead of one per row: the y kernel was address-ALU heavy)
  constexpr int EG = EGT;
  const int R = A.R;
  const int my = chain_len(y.p, 0);
  if (threadIdx.x < NST) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    if (su32(smem_raw) & 1023) __trap();  // the 128B swizzle needs 1024-byte aligned boxes
    for (int k = 0; k < NST; ++k) mbar_init(&full[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  poison_ring(ring, NST * A.stage_bytes);
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < NST; ++k) y_issue<MODE>(A, k, ring, full, &mG0, &mG1, &mW0, &mW1, &mH, fbuf);
  // thread -> (row r of the window, y-parity py, y-element eo)
  const int tid = threadIdx.x;
  const int eo = tid % EG, py = (tid / EG) & 1, r = tid / (2 * EG);
  const int cfs = P.f.cfs;
  int cslot = 0;
  uint32_t cround = 0, ctt = 0, gs = 0;
  int ob = 0;  // output staging buffer parity
#ifdef HPFEM_YPROF
  long long t_w0 = 0, t_w = 0, t_bwd = 0, t_br = 0, t_fe = 0, t_all = clock64(), t0, t1;
#endif
  for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++ctt) {
    const YTile t = y_decode(A, tile);
    const double* fb = fbuf + (ctt & 1) * A.fac_doubles + (eo * 2 + py) * cfs;  // this thread's chain
    const int e_x = t.e_x, pi = t.pi;
    const int e0 = t.g * EG, ey = e0 + eo;
    const int kx = pi + 2 * (t.kw * R + r);
    const int mthr = chain_len(y.p, py);
    const bool valid = r < R && kx <= x.p - 2 && ey < y.n;
    Sten5 st;
    const bool wtab = P.wtab != nullptr && MODE == ST_APPLY;
    const double* wb = reinterpret_cast<const double*>(smem_raw + A.wb_off) + (ctt & 1) * A.wb_doubles;
    if (valid) {
      if (A.fake_stencil) { st.w[0] = -1.0; st.w[1] = st.w[2] = st.w[3] = st.w[4] = 0.0; }
      else if (!wtab) sten5_build(x, x.nh + kx * x.n + e_x, MODE, P.kap_a, P.tau, P.cvL, P.cvR, st);
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) st.w[k] = 0.0;
    }
    const int rr = r < R ? r : 0;
    const int rg = rr * EG + eo;        // G box [R][EG][16]: box row of (r, eo)
    const int rw1 = rr * EG + eo;       // W box [R+2][EG][16]: row k_x - 2
    const int rw0 = (rr + 1) * EG + eo; //   k_x
    const int rw2 = (rr + 2) * EG + eo; //   k_x + 2
    const int rh0 = eo;                 // hat box [2][EG][16]: hL
    const int rh1 = EG + eo;            //   hR
    double ys[CL];
    double yv = 0.0;
    // Software-pipelined down sweep: the stencil of stage sg (independent
    // shared-memory loads and FMAs) is interleaved position by position with
    // the dependent recurrence of the previous stage sg + 1, so each warp has
    // independent work to issue under the FMA latency of its chain.  The
    // arithmetic per position is unchanged (bitwise the same result).
    // Positions past this parity's chain have zero factors (fac_cfs) and
    // finite (zero-padded) inputs: yv stays exactly 0 there, no select on the
    // dependent chain.
    double rv[KCP];
#pragma unroll
    for (int sg = CL / KCP - 1; sg >= 0; --sg) {
      if (KCP * sg < my) {
        const int slot = cslot;
#ifdef HPFEM_YPROF
        t0 = clock64();
#endif
        mbar_wait(&full[slot], cround & 1);
#ifdef HPFEM_YPROF
        t1 = clock64();
        if (KCP * sg + KCP >= my) t_w0 += t1 - t0; else t_w += t1 - t0;
#endif
        if (wtab && KCP * sg + KCP >= my) {  // first stage of the tile: the weights have landed
#pragma unroll
          for (int k = 0; k < 5; ++k) st.w[k] = valid ? wb[r * 6 + k] : 0.0;
        }
        const unsigned char* stg = ring + (size_t)slot * A.stage_bytes;
        const double* Gs = reinterpret_cast<const double*>(stg);
        const double* Ws = reinterpret_cast<const double*>(stg + A.off_w);
        const double* Hs = reinterpret_cast<const double*>(stg + A.off_h);
        const bool prev = sg + 1 < CL / KCP && KCP * (sg + 1) < my;  // stage sg + 1 awaits its recurrence
#pragma unroll
        for (int u = KCP - 1; u >= 0; --u) {
          double v = 0.0;
          if (MODE != ST_CORR) v = Gs[swz(rg, u, py)];
          if (MODE != ST_NONE)
            v += st.w[0] * Ws[swz(rw0, u, py)] + st.w[1] * Ws[swz(rw1, u, py)] + st.w[2] * Ws[swz(rw2, u, py)] +
                 st.w[3] * Hs[swz(rh0, u, py)] + st.w[4] * Hs[swz(rh1, u, py)];
          if (sg + 1 < CL / KCP && prev) {
            const int c = KCP * (sg + 1) + u;
            const double2 f = *reinterpret_cast<const double2*>(fb + 4 * c);  // (il, hd)
            yv = fma(-f.y, yv, f.x * rv[u]);
            ys[c] = yv;
          }
          rv[u] = v;
        }
        __syncwarp();
        if (lane == 0 && release_is_last(cnt, slot))
          y_issue<MODE>(A, gs + NST, ring, full, &mG0, &mG1, &mW0, &mW1, &mH, fbuf);
        ++gs;
        if (++cslot == NST) {
          cslot = 0;
          ++cround;
        }
      }
    }
#pragma unroll
    for (int u = KCP - 1; u >= 0; --u) {  // the recurrence of stage 0
      const double2 f = *reinterpret_cast<const double2*>(fb + 4 * u);
      yv = fma(-f.y, yv, f.x * rv[u]);
      ys[u] = yv;
    }
    // upward sweep, staged per warp through shared memory and stored with TMA
    // per 16 degrees (one box of this warp's RW rows; no CTA-wide barrier)
#ifdef HPFEM_YPROF
    const long long tb0 = clock64();
#endif
    double z = 0.0;
    const int RW = 16 / EG;            // rows per warp (EG is a power of two <= 8)
    const int wr0 = (tid >> 5) * RW;   // first row of this warp
#pragma unroll
    for (int sp = 0; sp < CL / KCP; sp += SPB) {  // SPB stages share one staging buffer / fence
      if (KCP * sp < my) {
        double* ob0 = obuf + ((size_t)ob * NW + (tid >> 5)) * (SPB * 32 * 8);  // SPB x [RW][EG][16]
#ifdef HPFEM_YPROF
        t0 = clock64();
#endif
        if (lane == 0) bulk_wait_read<NOBUF - 1>();  // the stores that last used this buffer have read it
        __syncwarp();
#ifdef HPFEM_YPROF
        t_br += clock64() - t0;
#endif
#pragma unroll
        // the group's factor pairs first: in program order after the staging
        // stores they could not be hoisted (the compiler cannot rule out
        // aliasing in shared memory) and each step waited a load latency
        double2 fz[SPB][KCP];
#pragma unroll
        for (int h = 0; h < SPB; ++h) {
          const int sg = sp + h;
          if (sg < CL / KCP && KCP * sg < my) {
#pragma unroll
            for (int u = 0; u < KCP; ++u) fz[h][u] = *reinterpret_cast<const double2*>(fb + 4 * (KCP * sg + u) + 2);
          }
        }
#pragma unroll
        for (int h = 0; h < SPB; ++h) {
          const int sg = sp + h;
          if (sg < CL / KCP && KCP * sg < my) {
            double* o = ob0 + h * 256;
#pragma unroll
            for (int u = 0; u < KCP; ++u) {
              const int c = KCP * sg + u;
              const double2 f = fz[h][u];  // (hu, il)
              z = fma(-f.x, z, f.y * ys[c]);  // 0 past the chain (see above)
              o[swz((r - wr0) * EG + eo, u, py)] = valid ? z : 0.0;
              if (sg == 0 && u == 0 && valid && c < mthr && P.z01)  // chain-first bubble (degree py): compact copy
                P.z01[(size_t)(x.nh + kx * x.n + e_x) * (2 * y.n) + 2 * ey + py] = z;
            }
          }
        }
#ifdef HPFEM_YPROF
        t0 = clock64();
#endif
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && wr0 < R) {
#pragma unroll
          for (int h = 0; h < SPB; ++h)
            if (sp + h < CL / KCP && KCP * (sp + h) < my)
              tma_store_4d(pi ? &mO1 : &mO0, ob0 + h * 256, 2 * KCP * (sp + h), e0, e_x, t.kw * R + wr0);
          bulk_commit();
        }
#ifdef HPFEM_YPROF
        t_fe += clock64() - t0;
#endif
        ob = ob + 1 == NOBUF ? 0 : ob + 1;
      }
    }
#ifdef HPFEM_YPROF
    t_bwd += clock64() - tb0;
#endif
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef HPFEM_YPROF
  t_all = clock64() - t_all;
  if (lane == 0 && blockIdx.x < 2)
    printf("yprof blk %d warp %d: all %lld  wait-first %lld  wait-other %lld  bwd %lld (wait_read %lld fence+store %lld) tiles %u\n",
           blockIdx.x, threadIdx.x >> 5, t_all, t_w0, t_w, t_bwd, t_br, t_fe, ctt);
#endif
}
/* ------------------------------------------------------------------ */
/* precomputed stencil weights of the bubble lines (one ST_APPLY step)  */
/* ------------------------------------------------------------------ */
__global__ void k_wtab_x(DirDev y, Layout L, double kap, double tau, const double* __restrict__ cvL,
                         const double* __restrict__ cvR, double* __restrict__ wt) {
  // lines = y-bubbles (k, e): table [e][5][Q]
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= y.nb) return;
  const int k = b / y.n, e = b - k * y.n;
  Sten5 st;
  sten5_build(y, y.nh + b, ST_APPLY, kap, tau, cvL, cvR, st);
#pragma unroll
  for (int q = 0; q < 5; ++q) wt[((size_t)e * 5 + q) * L.Q + k] = st.w[q];
}

__global__ void k_wtab_y(DirDev x, double kap, double tau, const double* __restrict__ cvL,
                         const double* __restrict__ cvR, double* __restrict__ wt) {
  // lines = x-bubble rows (k, e): table [e][pi][kh][6], k = pi + 2 kh
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= x.nb) return;
  const int k = b / x.n, e = b - k * x.n, pi = k & 1, kh = k >> 1;
  Sten5 st;
  sten5_build(x, x.nh + b, ST_APPLY, kap, tau, cvL, cvR, st);
  double* o = wt + (((size_t)e * 2 + pi) * chain_len(x.p, 0) + kh) * 6;
#pragma unroll
  for (int q = 0; q < 5; ++q) o[q] = st.w[q];
}

size_t tma_wtab_doubles(const DirDev& x, const DirDev& y, const Layout& L, int dir) {
  return dir == 0 ? (size_t)y.n * 5 * L.Q : (size_t)x.n * 2 * chain_len(x.p, 0) * 6;
}

cudaError_t tma_build_wtab(const DirDev& x, const DirDev& y, const Layout& L, int dir, double kap, double tau,
                           const double* cvL, const double* cvR, double* wtab, cudaStream_t st) {
  if (dir == 0)
    k_wtab_x<<<(y.nb + 255) / 256, 256, 0, st>>>(y, L, kap, tau, cvL, cvR, wtab);
  else
    k_wtab_y<<<(x.nb + 255) / 256, 256, 0, st>>>(x, kap, tau, cvL, cvR, wtab);
  return cudaGetLastError();
}

/* ------------------------------------------------------------------ */
/* host side: tensor maps and launch                                   */
/* ------------------------------------------------------------------ */
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = [] {  // thread-safe one-time initialisation
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (EncodeTiledFn)p;
    return (EncodeTiledFn) nullptr;
  }();
  return fn;
}

static bool encode(CUtensorMap* m, int rank, void* base, const uint64_t* dims, const uint64_t* strides_bytes,
                   const uint32_t* box, bool swizzle128 = false) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i < rank - 1) s[i] = strides_bytes[i];
  }
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TmaPlan {
  bool ok = false;
  int EG0 = 0, EG1 = 0, R = 0, hw = 0;
  int sms = 148;
  // per internal array a (0 = Gp, 1 = X1, 2 = X2)
  CUtensorMap xv[3][4];                 // x-solve views per array: [pi] bubble boxes, [2+pi] hat boxes
  CUtensorMap yG[3][2], yW[3][2], yH[3];
  CUtensorMap yO[2];                    // y-solve output stores (X1), per parity
  bool x2ok = false;                    // two-threads-per-chain x kernel (chains of 65 .. 128 positions)
  int EG2 = 0, hw2 = 0;
  CUtensorMap xv2[3][4];                // its views: <= 128 columns per box
};

static int even_up(int v) { return (v + 1) & ~1; }

/* y-solve tile shape: EG y-elements (a power of two <= 8, so that a warp
 * holds whole rows: RW = 16/EG rows per warp) x R rows of an x-chain (a
 * multiple of RW, with the R+2-row W box inside each parity's row count) */
static void y_tile_shape_eg(const DirDev& x, const DirDev& y, int eg, int& EG, int& R) {
  EG = eg;
  while (EG > y.n) EG >>= 1;
  const int RW = 16 / EG;
  R = NT / (2 * EG);
  if (R > chain_len(x.p, 1) - 2) R = chain_len(x.p, 1) - 2;
  R -= R % RW;
}

/* choose EG in {4, 8}: fewest idle rows in the x-chain windows, then the
 * larger window (W rows reused R/(R+2)); HPFEM_EG_Y overrides */
static void y_tile_shape(const DirDev& x, const DirDev& y, int forced, int& EG, int& R) {
  if (forced) {
    y_tile_shape_eg(x, y, forced, EG, R);
    return;
  }
  double best = -1.0;
  for (int eg : {4, 8}) {
    int e, r;
    y_tile_shape_eg(x, y, eg, e, r);
    if (r < 16 / e) continue;
    const int m0 = chain_len(x.p, 0), m1 = chain_len(x.p, 1);
    const double eff = double(m0 + m1) / double(((m0 + r - 1) / r + (m1 + r - 1) / r) * r);
    if (eff > best + 1e-9) {
      best = eff;
      EG = e;
      R = r;
    }
  }
  if (best < 0) y_tile_shape_eg(x, y, 8, EG, R);
}

/* shape conditions of the TMA path (both directions, element-major layout) */
bool tma_shape_ok(const DirDev& x, const DirDev& y, int eg_y) {
  const int Q = even_up(y.p - 1);
  int EG, R;
  y_tile_shape(x, y, eg_y, EG, R);
  return x.nb > 0 && y.nb > 0 && x.N >= 2 && Q <= 256 && Q >= KBOX && chain_len(x.p, 0) <= 128 &&
         chain_len(y.p, 0) <= 64 && R >= 16 / EG;
}

TmaPlan* tma_plan_create(const DirDev& x, const DirDev& y, const Layout& L, double* const arrays[3], int enable,
                         int eg_y) {
  TmaPlan* T = new TmaPlan();
  if (!enable || !L.emaj || !encode_fn() || !tma_shape_ok(x, y, eg_y)) return T;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&T->sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t ld8 = (uint64_t)L.ld * 8, Q8 = (uint64_t)L.Q * 8;
  bool ok = true;
  // ---- x-solve views: (column, e_x, kh) per x-parity; hat view = same with a narrow box
  T->EG0 = NT / L.Q < 1 ? 1 : NT / L.Q;
  if (T->EG0 > y.n) T->EG0 = y.n;
  T->hw = even_up(T->EG0 + 2);
  const int BW = T->EG0 * L.Q;
  for (int a = 0; ok && a < 3; ++a) {
    for (int pi = 0; ok && pi < 2; ++pi) {
      const int mpi = chain_len(x.p, pi) > 0 ? chain_len(x.p, pi) : 1;
      double* base = arrays[a] + (size_t)(x.nh + pi * x.n) * L.ld;
      const uint64_t d[3] = {(uint64_t)L.ld, (uint64_t)x.n, (uint64_t)mpi};
      const uint64_t s[2] = {ld8, 2 * (uint64_t)x.n * ld8};
      const uint32_t b[3] = {(uint32_t)BW, 1, (uint32_t)KR};
      ok = encode(&T->xv[a][pi], 3, base, d, s, b);
    }
    for (int pi = 0; ok && pi < 2; ++pi) {
      // same geometry, narrow box over the hat columns h0 .. h0+hw-1
      const int mpi = chain_len(x.p, pi) > 0 ? chain_len(x.p, pi) : 1;
      double* base = arrays[a] + (size_t)(x.nh + pi * x.n) * L.ld;
      const uint64_t d[3] = {(uint64_t)L.ld, (uint64_t)x.n, (uint64_t)mpi};
      const uint64_t s[2] = {ld8, 2 * (uint64_t)x.n * ld8};
      const uint32_t b[3] = {(uint32_t)T->hw, 1, (uint32_t)KR};
      ok = encode(&T->xv[a][2 + pi], 3, base, d, s, b);
    }
  }
  // ---- x-solve views of the two-threads-per-chain kernel (<= 128 columns per tile)
  if (chain_len(x.p, 0) > XH && L.Q <= 128) {
    T->EG2 = 128 / L.Q < 1 ? 1 : 128 / L.Q;
    if (T->EG2 > y.n) T->EG2 = y.n;
    T->hw2 = even_up(T->EG2 + 2);
    const int BW2 = T->EG2 * L.Q;
    bool ok2 = true;
    for (int a = 0; ok2 && a < 3; ++a)
      for (int k = 0; ok2 && k < 4; ++k) {
        const int pi = k & 1;
        const int mpi = chain_len(x.p, pi) > 0 ? chain_len(x.p, pi) : 1;
        double* base = arrays[a] + (size_t)(x.nh + pi * x.n) * L.ld;
        const uint64_t d[3] = {(uint64_t)L.ld, (uint64_t)x.n, (uint64_t)mpi};
        const uint64_t s[2] = {ld8, 2 * (uint64_t)x.n * ld8};
        const uint32_t b[3] = {(uint32_t)(k < 2 ? BW2 : T->hw2), 1, (uint32_t)KR};
        ok2 = encode(&T->xv2[a][k], 3, base, d, s, b);
      }
    T->x2ok = ok2;
  }
  // ---- y-solve views
  {
    int EG, R;
    y_tile_shape(x, y, eg_y, EG, R);
    const int RW = 16 / EG;
    T->EG1 = EG;
    T->R = R;
    ok = ok && R >= RW;
    for (int a = 0; ok && a < 3; ++a) {
      for (int pi = 0; ok && pi < 2; ++pi) {
        const int mpi = chain_len(x.p, pi);
        double* base = arrays[a] + L.hb + (size_t)(x.nh + pi * x.n) * L.ld;
        const uint64_t d4[4] = {(uint64_t)L.Q, (uint64_t)y.n, (uint64_t)x.n, (uint64_t)mpi};
        const uint64_t s4[3] = {Q8, ld8, 2 * (uint64_t)x.n * ld8};
        const uint32_t bG[4] = {KBOX, (uint32_t)EG, 1, (uint32_t)R};
        const uint32_t bW[4] = {KBOX, (uint32_t)EG, 1, (uint32_t)R + 2};
        ok = encode(&T->yG[a][pi], 4, base, d4, s4, bG, true) && encode(&T->yW[a][pi], 4, base, d4, s4, bW, true);
        if (ok && a == 1) {
          const uint32_t bO[4] = {16, (uint32_t)EG, 1, (uint32_t)RW};
          ok = encode(&T->yO[pi], 4, base, d4, s4, bO, true);
        }
      }
      if (ok) {
        const uint64_t d3[3] = {(uint64_t)L.Q, (uint64_t)y.n, (uint64_t)x.N};
        const uint64_t s3[2] = {Q8, ld8};
        const uint32_t b3[3] = {KBOX, (uint32_t)EG, 2};
        ok = encode(&T->yH[a], 3, arrays[a] + L.hb, d3, s3, b3, true);
      }
    }
  }
  T->ok = ok;
  return T;
}

void tma_plan_destroy(TmaPlan* T) { delete T; }

bool tma_supports(const TmaPlan* T, int dir) { return T && T->ok && (dir == 0 || dir == 1); }

constexpr int SMEM_OPTIN = 227 * 1024;  // the sm_100 per-CTA maximum

template <int CL, int MODE>
static cudaError_t launch_x(const TmaStepArgs& A, const CUtensorMap* g, const CUtensorMap* w, int grid, size_t smem,
                            cudaStream_t st) {
  auto k = k_xstep_tma<CL, MODE>;
  cudaError_t e = smem_optin((const void*)k, SMEM_OPTIN);  // once per (kernel, device)
  if (e != cudaSuccess) return e;
  k<<<grid, NT, smem, st>>>(A, g[0], g[1], w[0], w[1], w[2], w[3]);
  return cudaGetLastError();
}

template <int CL, int MODE, int EGT>
static cudaError_t launch_y(const TmaStepArgs& A, const TmaPlan* T, int gi, int wi, int grid, size_t smem,
                            cudaStream_t st) {
  auto k = k_ystep_tma<CL, MODE, EGT>;
  cudaError_t e = smem_optin((const void*)k, SMEM_OPTIN);
  if (e != cudaSuccess) return e;
  k<<<grid, NT, smem, st>>>(A, T->yG[gi][0], T->yG[gi][1], T->yW[wi][0], T->yW[wi][1], T->yH[wi], T->yO[0],
                            T->yO[1]);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t dispatch_x(int cl, const TmaStepArgs& A, const CUtensorMap* g, const CUtensorMap* w, int grid,
                              size_t smem, cudaStream_t st) {
  if (cl <= 8) return launch_x<8, MODE>(A, g, w, grid, smem, st);
  if (cl <= 16) return launch_x<16, MODE>(A, g, w, grid, smem, st);
  if (cl <= 32) return launch_x<32, MODE>(A, g, w, grid, smem, st);
  if (cl <= 64) return launch_x<64, MODE>(A, g, w, grid, smem, st);
  return launch_x<128, MODE>(A, g, w, grid, smem, st);
}

template <int MODE, int EGT>
static cudaError_t dispatch_y_eg(int cl, const TmaStepArgs& A, const TmaPlan* T, int gi, int wi, int grid,
                                 size_t smem, cudaStream_t st) {
  if (cl <= 8) return launch_y<8, MODE, EGT>(A, T, gi, wi, grid, smem, st);
  if (cl <= 16) return launch_y<16, MODE, EGT>(A, T, gi, wi, grid, smem, st);
  if (cl <= 32) return launch_y<32, MODE, EGT>(A, T, gi, wi, grid, smem, st);
  return launch_y<64, MODE, EGT>(A, T, gi, wi, grid, smem, st);
}

template <int MODE>
static cudaError_t dispatch_y(int cl, const TmaStepArgs& A, const TmaPlan* T, int gi, int wi, int grid, size_t smem,
                              cudaStream_t st) {
  switch (A.EG) {  // y_tile_shape: a power of two <= 8
    case 8: return dispatch_y_eg<MODE, 8>(cl, A, T, gi, wi, grid, smem, st);
    case 4: return dispatch_y_eg<MODE, 4>(cl, A, T, gi, wi, grid, smem, st);
    case 2: return dispatch_y_eg<MODE, 2>(cl, A, T, gi, wi, grid, smem, st);
    default: return dispatch_y_eg<MODE, 1>(cl, A, T, gi, wi, grid, smem, st);
  }
}

static int round128(int b) { return (b + 127) & ~127; }
static int round1024(int b) { return (b + 1023) & ~1023; }

template <int MODE>
static cudaError_t launch_x2_mode(const TmaStepArgs& A, const CUtensorMap* g, const CUtensorMap* w, int grid,
                                  size_t smem, cudaStream_t st) {
  auto k = k_xstep_tma2<MODE>;
  cudaError_t e = smem_optin((const void*)k, SMEM_OPTIN);
  if (e != cudaSuccess) return e;
  k<<<grid, NT, smem, st>>>(A, g[0], g[1], w[0], w[1], w[2], w[3]);
  return cudaGetLastError();
}

/* x-solve with two threads per chain (A.P set; shapes from the plan) */
static cudaError_t launch_x2(const TmaPlan* T, TmaStepArgs A, int gi, int wi, int sms, cudaStream_t st) {
  const StepParams& P = A.P;
  const DirDev& x = P.s;
  const DirDev& y = P.o;
  A.EG = T->EG2;
  A.hw = T->hw2;
  const int BW = A.EG * P.lay.Q;
  const int gb = (P.mode != ST_CORR) ? KR * BW * 8 : 0;
  const int wb = (P.mode != ST_NONE) ? KR * BW * 8 : 0;
  const int hb = (P.mode != ST_NONE) ? KR * A.hw * 8 : 0;
  // [G lo | G hi | W lo | W hi | H lo | H hi]; each upper box 128 bytes off the lower one modulo 256
  auto hi_off = [](int bytes) {
    int o = (bytes + 127) & ~127;
    if (o % 256 == 0) o += 128;
    return o;
  };
  A.hi_g = hi_off(gb);
  A.hi_w = hi_off(wb);
  A.hi_h = hi_off(hb);
  A.off_w = gb ? (A.hi_g + gb + 255) & ~255 : 0;
  A.off_h = A.off_w + (wb ? (A.hi_w + wb + 255) & ~255 : 0);
  A.stage_bytes = (A.off_h + (hb ? A.hi_h + hb : 0) + 255) & ~255;
  A.tx_bytes = 2 * (gb + wb + hb);
  A.fac_doubles = (P.f.cfs + 15) & ~15;
  A.wb_doubles = P.wtab ? A.EG * 5 * P.lay.Q : 0;
  A.S = XH / KR;
  const int budget = SMEM_OPTIN - 4096;
  A.nstages = (budget - 2 * A.fac_doubles * 8 - 2 * A.wb_doubles * 8) / A.stage_bytes;
  if (A.nstages > P.tun.nst[0]) A.nstages = P.tun.nst[0];
  if (A.nstages > A.S) A.nstages = A.S;
  if (A.nstages < 1) A.nstages = 1;
  A.fac_off = A.nstages * A.stage_bytes;
  A.wb_off = A.fac_off + 2 * A.fac_doubles * 8;
  A.bar_off = A.wb_off + 2 * A.wb_doubles * 8;
  const int ngroups = (y.n + A.EG - 1) / A.EG;
  A.ntiles = ngroups * x.n * 2;
  A.fS = make_fdiv(A.S);
  A.fN = make_fdiv(A.nstages);
  A.fG = make_fdiv(ngroups);
  A.fT = make_fdiv(x.n);
  const size_t smem = (size_t)A.bar_off + 2 * A.nstages * sizeof(uint64_t);
  const int grid = A.ntiles < sms ? A.ntiles : sms;
  const CUtensorMap* g = T->xv2[gi];
  const CUtensorMap* w = T->xv2[wi];
  switch (P.mode) {
    case ST_NONE: return launch_x2_mode<ST_NONE>(A, g, w, grid, smem, st);
    case ST_APPLY: return launch_x2_mode<ST_APPLY>(A, g, w, grid, smem, st);
    default: return launch_x2_mode<ST_CORR>(A, g, w, grid, smem, st);
  }
}

/* Launch the bubble-line part of one half-step.  ia_g / ia_w: indices of the
 * G and Xp arrays among (Gp, X1, X2) (-1 when unused). */
cudaError_t tma_launch_step(const TmaPlan* T, const StepParams& P, int ia_g, int ia_w, cudaStream_t st,
                            int spare_sms) {
  const int sms = T->sms - spare_sms > 1 ? T->sms - spare_sms : 1;
  TmaStepArgs A;
  std::memset(&A, 0, sizeof(A));
  A.P = P;
  A.fake_stencil = P.tun.fake_stencil;
  const int gi = ia_g >= 0 ? ia_g : ia_w, wi = ia_w >= 0 ? ia_w : ia_g;
  const int budget = SMEM_OPTIN - 4096;
  if (P.dir == 0) {
    const DirDev& x = P.s;
    const DirDev& y = P.o;
    A.EG = T->EG0;
    A.hw = T->hw;
    const int BW = A.EG * P.lay.Q;
    const int gb = (P.mode != ST_CORR) ? KR * BW * 8 : 0;
    const int wb = (P.mode != ST_NONE) ? KR * BW * 8 : 0;
    const int hb = (P.mode != ST_NONE) ? KR * A.hw * 8 : 0;
    A.off_w = round128(gb);
    A.off_h = A.off_w + round128(wb);
    A.stage_bytes = round128(A.off_h + hb);
    A.tx_bytes = gb + wb + hb;
    A.fac_doubles = (P.f.cfs + 15) & ~15;
    A.wb_doubles = P.wtab ? A.EG * 5 * P.lay.Q : 0;
    A.S = (chain_len(x.p, 0) - 1) / KR + 1;
    A.nstages = (budget - 2 * A.fac_doubles * 8 - 2 * A.wb_doubles * 8) / A.stage_bytes;
    if (A.nstages > P.tun.nst[0]) A.nstages = P.tun.nst[0];  // 4 measured best
    if (A.nstages > A.S) A.nstages = A.S;  // the factor double buffer relies on NST <= S
    if (A.nstages < 1) A.nstages = 1;
    A.fac_off = A.nstages * A.stage_bytes;
    A.wb_off = A.fac_off + 2 * A.fac_doubles * 8;
    A.bar_off = A.wb_off + 2 * A.wb_doubles * 8;
    const int ngroups = (y.n + A.EG - 1) / A.EG;
    A.ntiles = ngroups * x.n * 2;
    A.fS = make_fdiv(A.S);
    A.fN = make_fdiv(A.nstages);
    A.fG = make_fdiv(ngroups);
    A.fT = make_fdiv(x.n);
    const size_t smem = (size_t)A.bar_off + 2 * A.nstages * sizeof(uint64_t);
    const int grid = A.ntiles < sms ? A.ntiles : sms;
    const int cl = chain_len(x.p, 0);
    if (cl > XH && T->x2ok && !P.tun.no_x2) return launch_x2(T, A, gi, wi, sms, st);
    const CUtensorMap* g = T->xv[gi];
    const CUtensorMap* w = T->xv[wi];
    switch (P.mode) {
      case ST_NONE: return dispatch_x<ST_NONE>(cl, A, g, w, grid, smem, st);
      case ST_APPLY: return dispatch_x<ST_APPLY>(cl, A, g, w, grid, smem, st);
      default: return dispatch_x<ST_CORR>(cl, A, g, w, grid, smem, st);
    }
  }
  const DirDev& y = P.s;
  const DirDev& x = P.o;
  A.EG = T->EG1;
  A.R = T->R;
  const int gb = (P.mode != ST_CORR) ? A.R * A.EG * KBOX * 8 : 0;
  const int wb = (P.mode != ST_NONE) ? (A.R + 2) * A.EG * KBOX * 8 : 0;
  const int hb = (P.mode != ST_NONE) ? 2 * A.EG * KBOX * 8 : 0;
  A.off_w = round1024(gb);  // swizzled boxes: 1024-byte aligned
  A.off_h = A.off_w + round1024(wb);
  A.stage_bytes = round1024(A.off_h + hb);
  A.tx_bytes = gb + wb + hb;
  const int obytes = NOBUF * NW * SPB * 256 * 8;
  A.fac_doubles = (2 * A.EG * P.f.cfs + 15) & ~15;
  A.wb_doubles = P.wtab ? ((A.R * 6 + 15) & ~15) : 0;
  A.S = (chain_len(y.p, 0) - 1) / KCP + 1;
  A.nstages = (budget - obytes - 2 * A.fac_doubles * 8 - 2 * A.wb_doubles * 8) / A.stage_bytes;
  if (A.nstages > P.tun.nst[1]) A.nstages = P.tun.nst[1];
  if (A.nstages > A.S) A.nstages = A.S;  // see x-solve
  if (A.nstages < 1) A.nstages = 1;
  A.out_off = A.nstages * A.stage_bytes;
  A.fac_off = A.out_off + obytes;
  A.wb_off = A.fac_off + 2 * A.fac_doubles * 8;
  A.bar_off = A.wb_off + 2 * A.wb_doubles * 8;
  A.nwt = (chain_len(x.p, 0) + A.R - 1) / A.R + (chain_len(x.p, 1) + A.R - 1) / A.R;
  const int ngroups = (y.n + A.EG - 1) / A.EG;
  A.ntiles = ngroups * x.n * A.nwt;
  A.fS = make_fdiv(A.S);
  A.fN = make_fdiv(A.nstages);
  A.fG = make_fdiv(ngroups);
  A.fT = make_fdiv(A.nwt);
  const size_t smem = (size_t)A.bar_off + 2 * A.nstages * sizeof(uint64_t);
  const int grid = A.ntiles < sms ? A.ntiles : sms;
  const int cl = chain_len(y.p, 0);
  switch (P.mode) {
    case ST_NONE: return dispatch_y<ST_NONE>(cl, A, T, gi, wi, grid, smem, st);
    case ST_APPLY: return dispatch_y<ST_APPLY>(cl, A, T, gi, wi, grid, smem, st);
    default: return dispatch_y<ST_CORR>(cl, A, T, gi, wi, grid, smem, st);
  }
}

}  // namespace hpfem
