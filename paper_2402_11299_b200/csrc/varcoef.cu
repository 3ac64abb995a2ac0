/*
 * varcoef.cu -- NEXT-3 of SURVEY 8(f): grid <-> piecewise-Legendre
 * transforms (Section 6), the variable-coefficient operator of
 * eq. (evaluation) and the vector kernels of the
 * ADI-preconditioned conjugate gradient method (Section 7).
 *
 * Transforms.  Values at the p + 1 Chebyshev points of every element and
 * Legendre coefficients share one block layout (index i n + e, DESIGN.md
 * R18), and the reference-element matrix (F_p or F_p^{-1}, (p+1) x (p+1))
 * is the same for every element.  One 1D pass is therefore the dense
 * contraction
 *     out[base(c) + k s] = sum_i A[k, i] in[base(c) + i s],
 *     base(c) = (c / nb) bs + c % nb,
 * over "columns" c: along x (rows i n_x + e) every (e, column) pair is a
 * column, contiguous (nb = n_x L_y, s = n_x L_y); along y every (row, e)
 * pair is one (nb = n_y, bs = L_y, s = n_y).  k_elem_apply is a shared-memory
 * tiled fp64 GEMM (48 outputs x 64 columns per CTA, 3 x 4 per thread,
 * double-buffered chunks with register prefetch); the
 * Hadamard product with the coefficient grid is fused into the epilogue of
 * the inverse transform's second pass (P:L1005 'G o (...)').  fp64 has no
 * tcgen05 kind, so this runs on the FP64 pipes (K10).
 *
 * CG vectors.  Deterministic two-stage reductions (fixed block partition,
 * fixed tree order), scalars kept on the device.
 */
#include <cuda_runtime.h>

#include "hpfem_internal.h"

namespace hpfem {

namespace {

constexpr int TK = 48;   // outputs per CTA (p + 1 = 129: 3 tiles, 90% used)
constexpr int TC = 64;   // columns per CTA
constexpr int TI = 16;   // contraction chunk
constexpr int RK = 3;    // outputs per thread (16 thread rows x 3 = TK)
constexpr int RC = 4;    // columns per thread (16 thread columns x 4 = TC)

/* register-prefetched, double-buffered shared-memory tiles: the global loads
 * of chunk i0 + TI are issued before the FMAs of chunk i0 */
__global__ void __launch_bounds__(256) k_elem_apply(ElemApply E) {
  __shared__ double As[2][TI][TK + 1];
  __shared__ double Bs[2][TI][TC];
  const int t = threadIdx.x;
  const long long c0 = (long long)blockIdx.x * TC;
  const int k0 = blockIdx.y * TK;
  const int tx = t & 15, ty = t >> 4;
  const int lc = t & 63, li = t >> 6;  // B loads: 64 consecutive columns x 4 rows per pass
  const long long cl = c0 + lc;
  const bool lvalid = cl < E.ncols;
  const long long bl = lvalid ? (cl / E.nb) * E.bs + cl % E.nb : 0;
  double acc[RK][RC];
#pragma unroll
  for (int a = 0; a < RK; ++a)
#pragma unroll
    for (int b = 0; b < RC; ++b) acc[a][b] = 0.0;
  constexpr int NA = (TI * TK + 255) / 256;  // A elements per thread per chunk
  double ra[NA], rb[TI / 4];
  auto gload = [&](int i0) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int idx = t + 256 * q;
      const int k = idx / TI, i = idx % TI;
      const int kk = k0 + k, ii = i0 + i;
      ra[q] = (idx < TI * TK && kk < E.M && ii < E.K) ? __ldg(E.A + (size_t)kk * E.K + ii) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < TI / 4; ++r) {
      const int ii = i0 + li + 4 * r;
      rb[r] = (lvalid && ii < E.K) ? __ldg(E.in + bl + (long long)ii * E.s) : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int idx = t + 256 * q;
      if (idx < TI * TK) As[buf][idx % TI][idx / TI] = ra[q];
    }
#pragma unroll
    for (int r = 0; r < TI / 4; ++r) Bs[buf][li + 4 * r][lc] = rb[r];
  };
  gload(0);
  sstore(0);
  __syncthreads();
  int buf = 0;
  for (int i0 = 0; i0 < E.K; i0 += TI) {
    const bool more = i0 + TI < E.K;
    if (more) gload(i0 + TI);
#pragma unroll
    for (int i = 0; i < TI; ++i) {
      double a[RK], b[RC];
#pragma unroll
      for (int r = 0; r < RK; ++r) a[r] = As[buf][i][ty * RK + r];
#pragma unroll
      for (int r = 0; r < RC; ++r) b[r] = Bs[buf][i][tx + 16 * r];
#pragma unroll
      for (int x = 0; x < RK; ++x)
#pragma unroll
        for (int y = 0; y < RC; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int y = 0; y < RC; ++y) {
    const long long c = c0 + tx + 16 * y;
    if (c >= E.ncols) continue;
    const long long bo = (c / E.nb) * E.bs + c % E.nb;
#pragma unroll
    for (int x = 0; x < RK; ++x) {
      const int k = k0 + ty * RK + x;
      if (k >= E.M) continue;
      const long long o = bo + (long long)k * E.s;
      const double v = E.g ? acc[x][y] * __ldg(E.g + o) : acc[x][y];
      E.out[o] = E.h ? fma(E.alpha, v, __ldg(E.h + o)) : v;
    }
  }
}

constexpr int RB = 256;  // reduction block

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (threadIdx.x < 32) {
    v = threadIdx.x < (RB / 32) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

/* partial[b] = sum over block b's grid-stride share of a[i] * b[i] */
__global__ void __launch_bounds__(RB) k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                    size_t n, double* __restrict__ partial) {
  __shared__ double sh[RB / 32];
  double v = 0.0;
  for (size_t i = (size_t)blockIdx.x * RB + threadIdx.x; i < n; i += (size_t)gridDim.x * RB) v = fma(a[i], b[i], v);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

/* one block: s = sum(partial), then the CG scalar update `op`:
 *   CG_RZ0:   rz = s                                     (first iteration)
 *   CG_ALPHA: alpha = rz / s                             (s = p.q)
 *   CG_RR:    rr = s                                     (s = r.r)
 *   CG_BETA:  beta = s / rz, rz = s                      (s = r.z) */
__global__ void __launch_bounds__(RB) k_cg_scalar(const double* __restrict__ partial, int np, int op,
                                                  double* __restrict__ sc) {
  __shared__ double sh[RB / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += RB) v += partial[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    if (op == CG_RZ0) sc[CG_RZ] = v;
    else if (op == CG_ALPHA) sc[CG_A] = sc[CG_RZ] / v;
    else if (op == CG_RR) sc[CG_RRV] = v;
    else {
      sc[CG_B] = v / sc[CG_RZ];
      sc[CG_RZ] = v;
    }
  }
}

/* x += alpha p; r -= alpha q; partial of r.r */
__global__ void __launch_bounds__(RB) k_cg_xr(double* __restrict__ x, double* __restrict__ r,
                                              const double* __restrict__ p, const double* __restrict__ q, size_t n,
                                              const double* __restrict__ sc, double* __restrict__ partial) {
  __shared__ double sh[RB / 32];
  const double alpha = sc[CG_A];
  double v = 0.0;
  for (size_t i = (size_t)blockIdx.x * RB + threadIdx.x; i < n; i += (size_t)gridDim.x * RB) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v = fma(ri, ri, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

/* p = z + beta p  (beta = 0: p = z) */
__global__ void __launch_bounds__(RB) k_cg_p(double* __restrict__ p, const double* __restrict__ z, size_t n,
                                             const double* __restrict__ sc, int first) {
  const double beta = first ? 0.0 : sc[CG_B];
  for (size_t i = (size_t)blockIdx.x * RB + threadIdx.x; i < n; i += (size_t)gridDim.x * RB)
    p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

}  // namespace

cudaError_t launch_elem_apply(const ElemApply& E, cudaStream_t st) {
  if (E.ncols <= 0 || E.M <= 0) return cudaSuccess;
  dim3 grid((unsigned)((E.ncols + TC - 1) / TC), (E.M + TK - 1) / TK);
  k_elem_apply<<<grid, 256, 0, st>>>(E);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* a, const double* b, size_t n, double* partial, double* sc, int op,
                       cudaStream_t st) {
  k_dot_partial<<<CG_BLOCKS, RB, 0, st>>>(a, b, n, partial);
  k_cg_scalar<<<1, RB, 0, st>>>(partial, CG_BLOCKS, op, sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_xr(double* x, double* r, const double* p, const double* q, size_t n, double* partial,
                         double* sc, cudaStream_t st) {
  k_cg_xr<<<CG_BLOCKS, RB, 0, st>>>(x, r, p, q, n, sc, partial);
  k_cg_scalar<<<1, RB, 0, st>>>(partial, CG_BLOCKS, CG_RR, sc);
  return cudaGetLastError();
}

cudaError_t launch_cg_p(double* p, const double* z, size_t n, const double* sc, int first, cudaStream_t st) {
  k_cg_p<<<CG_BLOCKS, RB, 0, st>>>(p, z, n, sc, first);
  return cudaGetLastError();
}

}  // namespace hpfem
