/*
 * plan.cpp -- host plan and C ABI (include/hpfem.h) of the B200 ADI hp-FEM
 * solver.  Compiled with g++ (binary128 shift arithmetic needs libquadmath);
 * all array work is enqueued as the device kernels of kernels.cu.
 *
 * Plan (Alg. 2 "Precomputation"):
 *   1. element widths and closed-form 1D entries (ops1d.h, App. A);
 *   2. spectral interval of (A_d, M_d), A_d = K_d + w^2/2 M_d:
 *      lambda_min closed form, lambda_max by bisection on "sigma M - A is
 *      SPD" with the reverse Cholesky of Alg. 1 as the test (R4;
 *      replaces the Crawford eigensolver of P:L689);
 *   3. gamma, J and Zolotarev shifts in binary128 (R5);
 *   4. the 2J+1 shifted factorisations on the device (K1).
 */
#include <quadmath.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: no-ops unless a profiler injects itself

#include "../../include/hpfem.h"
#include "hpfem_internal.h"
#include "ops1d.h"
#include "tma_step.h"

using namespace hpfem;

namespace {

/* NVTX range for the host-side enqueue of one stage of the solve (visible in
 * nsys / ncu --nvtx timelines; one range per half-step of Alg. 2) */
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

thread_local std::string t_err;

int set_err(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

int cuda_err(cudaError_t e, const char* where) {
  return set_err(HPFEM_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

/* the tuning switches (hpfem_internal.h Tuning), read once per plan */
Tuning read_tuning() {
  Tuning t;
  t.hat_sms = env_int("HPFEM_HAT_SMS", -1);
  t.no_graph = env_int("HPFEM_NO_GRAPH", 0) == 1;
  t.no_small = env_int("HPFEM_NO_SMALL", 0) == 1;
  t.no_tma = env_int("HPFEM_NO_TMA", 0) == 1;
  t.no_wtab = env_int("HPFEM_NO_WTAB", 0) == 1;
  t.batch_streams = env_int("HPFEM_BATCH_STREAMS", 8);
  if (t.batch_streams < 1) t.batch_streams = 1;
  const char* bk = std::getenv("HPFEM_BUBBLE_KERNEL");
  t.bub_reg = bk && bk[0] == 'r';  // "reg" selects the register variant
  t.hat_lb[0] = env_int("HPFEM_HAT_LB_X", 32);
  t.hat_lb[1] = env_int("HPFEM_HAT_LB_Y", 32);
  t.nst[0] = env_int("HPFEM_NST_X", 4);
  t.nst[1] = env_int("HPFEM_NST_Y", 4);
  t.eg_y = env_int("HPFEM_EG_Y", 0);
  t.fake_stencil = env_int("HPFEM_FAKE_STENCIL", 0);
  t.hats_seq = env_int("HPFEM_HATS_SEQ", 0);
  t.no_hat_split = env_int("HPFEM_NO_HAT_SPLIT", 0) == 1;
  t.no_x2 = env_int("HPFEM_NO_X2", 0) == 1;
  t.transpose = env_int("HPFEM_TRANSPOSE", -1);
  return t;
}

/* 2D boundary code -> per-direction 1D codes (include/hpfem.h HPFEM_BC_2D) */
bool split_bc(int bc, int& bx, int& by) {
  if (bc >= HPFEM_BC_DIRICHLET && bc <= HPFEM_BC_NEUMANN_DIRICHLET) {
    bx = by = bc;
    return true;
  }
  if (bc < 16 || bc > 31) return false;
  bx = (bc - 16) & 3;
  by = ((bc - 16) >> 2) & 3;
  return true;
}

/* host view of one direction */
struct DirHost {
  int n = 0, p = 0, bc = 0, nh = 0, N = 0, nb = 0;
  double rob[2] = {0.0, 0.0};  // Robin alpha at the left / right end
  std::vector<double> xs, delta;
};

DirHost make_dir(const double* xs, int n, int p, int bc, const double* rob = nullptr) {
  DirHost d;
  if (rob) {
    d.rob[0] = rob[0];
    d.rob[1] = rob[1];
  }
  d.n = n;
  d.p = p;
  d.bc = bc;
  d.nh = n_hats(n, bc);
  d.nb = (p - 1) * n;
  d.N = d.nh + d.nb;
  d.xs.assign(xs, xs + n + 1);
  d.delta.resize(n);
  for (int e = 0; e < n; ++e) d.delta[e] = xs[e + 1] - xs[e];
  return d;
}

/* Host SPD test of S = kap K + sig M by the same chain / Schur-complement
 * reverse Cholesky the device factor kernel runs (Alg. 1). */
bool spd_host(const DirHost& d, double kap, double sig) {
  const int n = d.n;
  std::vector<double> il(d.nb), g(d.nb), vL(d.nb), vR(d.nb);
  for (int e = 0; e < n; ++e) {
    const double dl = d.delta[e];
    for (int pi = 0; pi < 2; ++pi) {
      const int m = chain_len(d.p, pi);
      double lnext = 0.0;
      for (int c = m - 1; c >= 0; --c) {
        const int k = pi + 2 * c, b = k * n + e;
        double a = s_bub_diag(kap, sig, dl, k), gc = 0.0;
        if (c < m - 1) {
          gc = s_bub_off(sig, dl, k) / lnext;
          a -= gc * gc;
        }
        if (!(a > 0.0) || !std::isfinite(a)) return false;
        const double l = std::sqrt(a);
        il[b] = 1.0 / l;
        g[b] = gc;
        lnext = l;
      }
      for (int side = 0; side < 2 && m > 0; ++side) {
        const int h = hat_of_node(e + side, n, d.bc);
        const double beta = h >= 0 ? s_hat_bub(sig, dl, side, pi) : 0.0;
        std::vector<double>& v = side ? vR : vL;
        const int b0 = pi * n + e;
        double z = beta * il[b0] * il[b0];
        v[b0] = z;
        int bp = b0;
        for (int c = 1; c < m; ++c) {
          const int b = (pi + 2 * c) * n + e;
          z = -g[bp] * z * il[b];
          v[b] = z;
          bp = b;
        }
      }
    }
  }
  auto schur = [&](const std::vector<double>& vv, int e, int side) {
    double acc = s_hat_bub(sig, d.delta[e], side, 0) * vv[e];
    if (d.p - 2 >= 1) acc += s_hat_bub(sig, d.delta[e], side, 1) * vv[n + e];
    return acc;
  };
  double lnext = 0.0;
  for (int t = d.nh - 1; t >= 0; --t) {
    const int node = node_of_hat(t, d.bc), eL = node - 1, eR = node;
    double diag = 0.0;
    if (eL >= 0) diag += s_hat_diag_elem(kap, sig, d.delta[eL]) - schur(vR, eL, 1);
    if (eR <= n - 1) diag += s_hat_diag_elem(kap, sig, d.delta[eR]) - schur(vL, eR, 0);
    if (node == 0) diag += kap * d.rob[0];  // Robin boundary term
    if (node == n) diag += kap * d.rob[1];
    if (t < d.nh - 1) {
      const double gc = (s_hat_off_elem(kap, sig, d.delta[eR]) - schur(vR, eR, 0)) / lnext;
      diag -= gc * gc;
    }
    if (!(diag > 0.0) || !std::isfinite(diag)) return false;
    lnext = std::sqrt(diag);
  }
  return true;
}

/* [lambda_min, lambda_max] of (A, M), A = K + w^2/2 M (reading R4). */
void spectral_interval(const DirHost& d, double omega, double lam[2]) {
  const double hw2 = 0.5 * omega * omega;
  if (d.N == 1) {  // single dof (n = 1, p = 2, Dirichlet): lambda = A/M exactly
    const double m = s_bub_diag(0.0, 1.0, d.delta[0], 0);
    const double a = s_bub_diag(1.0, hw2, d.delta[0], 0);
    lam[0] = lam[1] = a / m;
    return;
  }
  const double len = d.xs[d.n] - d.xs[0];
  const double pi = 3.141592653589793238462643383279502884;
  // closed-form lower bounds of the continuous spectrum: Dirichlet pi^2/L^2,
  // Neumann 0 (constants), mixed Dirichlet/Neumann pi^2/(4 L^2) (quarter wave)
  lam[0] = (d.bc == HPFEM_BC_DIRICHLET ? pi * pi / (len * len)
            : d.bc == HPFEM_BC_NEUMANN ? 0.0
                                       : pi * pi / (4.0 * len * len)) +
           hw2;
  if (d.rob[0] != 0.0 || d.rob[1] != 0.0) {
    // Robin ends (reading R22): bisection on "A - sigma M = K + (w^2/2 - sigma) M
    // is SPD" from the valid lower bound w^2/2, keeping the SPD-confirmed end
    double lo = hw2, hi = std::max(2.0 * lo, 1.0);
    for (int it = 0; it < 200 && spd_host(d, 1.0, hw2 - hi); ++it) {
      lo = hi;
      hi *= 2.0;
    }
    while (hi - lo > 1e-13 * hi) {
      const double mid = lo + 0.5 * (hi - lo);
      if (spd_host(d, 1.0, hw2 - mid))
        lo = mid;
      else
        hi = mid;
    }
    lam[0] = lo;
  }
  double h = d.delta[0];
  for (double x : d.delta) h = std::min(h, x);
  const double p2 = (double)d.p * d.p;
  // Lemma 5.2: lambda_max(A, M) <= (24 p^4 + w^2 h^2) / (2 h^2)
  double hi = std::max((24.0 * p2 * p2 + omega * omega * h * h) / (2.0 * h * h), 2.0 * lam[0]);
  for (int it = 0; it < 200 && !spd_host(d, -1.0, hi - hw2); ++it) hi *= 2.0;
  double lo = lam[0];
  while (hi - lo > 1e-13 * hi) {
    const double mid = lo + 0.5 * (hi - lo);
    if (spd_host(d, -1.0, mid - hw2))
      hi = mid;
    else
      lo = mid;
  }
  lam[1] = hi;
}

/* ---------------- Zolotarev shifts in binary128 (reading R5) ---------------- */
typedef __float128 f128;

f128 agm128(f128 a, f128 b) {
  while (fabsq(a - b) > 1e-33Q * fabsq(a)) {
    const f128 m = 0.5Q * (a + b);
    b = sqrtq(a * b);
    a = m;
  }
  return 0.5Q * (a + b);
}

/* Jacobi dn(u | k) for 0 <= u <= K/2 given k' (R5):
 * k' >= 1e-8: descending Landen (arithmetic-geometric mean) scheme;
 * k' <  1e-8: dn = sech u + (k'^2/4)(sinh u cosh u + u) tanh u sech u
 *             (first order in k'^2 near k = 1; remainder O(k'^2) relative). */
f128 dn_half(f128 u, f128 kp) {
  if (kp >= 1.0Q) return 1.0Q;
  if (kp < 1e-8Q) {
    const f128 c = coshq(u), s = sinhq(u);
    return 1.0Q / c + 0.25Q * kp * kp * (s * c + u) * (s / c) / c;
  }
  f128 A[80], Cc[80];
  f128 a = 1.0Q, b = kp, c = sqrtq((1.0Q - kp) * (1.0Q + kp));
  int N = 0;
  while (fabsq(c) > 1e-34Q && N < 78) {
    const f128 an = 0.5Q * (a + b);
    c = 0.5Q * (a - b);
    b = sqrtq(a * b);
    a = an;
    ++N;
    A[N] = a;
    Cc[N] = c;
  }
  f128 ph = ldexpq(a, N) * u, ph1 = ph;
  for (int i = N; i >= 1; --i) {
    ph1 = ph;
    ph = 0.5Q * (ph + asinq(Cc[i] / A[i] * sinq(ph)));
  }
  return N == 0 ? 1.0Q : cosq(ph) / cosq(ph1 - ph);
}

f128 dn128(f128 u, f128 K, f128 kp) {
  return (2 * u <= K) ? dn_half(u, kp) : kp / dn_half(K - u, kp);
}

int zolotarev(double a, double b, double c, double d, double tol, int& J, double& gamma, std::vector<double>& P,
              std::vector<double>& Q) {
  const f128 A = a, B = b, C = c, D = d;
  const f128 g = fabsq(C - A) * fabsq(D - B) / (fabsq(C - B) * fabsq(D - A));
  gamma = (double)g;
  const f128 pi = M_PIq;
  const f128 jr = logq(16.0Q * g) * logq(4.0Q / (f128)tol) / (pi * pi);
  if (!(jr == jr) || jr > 1e6Q) return set_err(HPFEM_ENUMERIC, "non-finite or huge J");
  J = (int)ceilq(jr);
  if (J < 1) J = 1;
  const f128 al = 2.0Q * g - 1.0Q + 2.0Q * sqrtq(g * g - g);  // cross-ratio image of gamma
  const f128 kp = 1.0Q / al;
  const f128 K = pi / (2.0Q * agm128(1.0Q, kp));
  P.resize(J);
  Q.resize(J);
  const bool sym = (c == -b) && (d == -a);
  // general Moebius T with T(-al)=a, T(-1)=b, T(1)=c as a 2x2 matrix:
  // S_z sends (-al,-1,1) -> (0,1,inf), S_w sends (a,b,c) -> (0,1,inf), T = S_w^{-1} S_z
  const f128 z1 = -al, z2 = -1.0Q, z3 = 1.0Q;
  const f128 sz[4] = {z2 - z3, -z1 * (z2 - z3), z2 - z1, -z3 * (z2 - z1)};
  const f128 sw[4] = {B - C, -A * (B - C), B - A, -C * (B - A)};
  const f128 iw[4] = {sw[3], -sw[1], -sw[2], sw[0]};  // adjugate = inverse up to scale
  const f128 T[4] = {iw[0] * sz[0] + iw[1] * sz[2], iw[0] * sz[1] + iw[1] * sz[3], iw[2] * sz[0] + iw[3] * sz[2],
                     iw[2] * sz[1] + iw[3] * sz[3]};
  auto mob = [&](f128 z) { return (T[0] * z + T[1]) / (T[2] * z + T[3]); };
  // one-point spectrum in exactly one direction (N = 1 there): the Moebius
  // map degenerates (al = 1); the shift at that point annihilates the error
  // of that direction in one step, the other is any point of its interval
  // (reading R15)
  const bool deg_x = a == b, deg_y = c == d;
  for (int j = 1; j <= J; ++j) {
    const f128 u = (f128)(2 * j - 1) * K / (2.0Q * J);
    const f128 dn = dn128(u, K, kp);
    if (deg_x != deg_y) {
      P[j - 1] = deg_x ? a : (double)sqrtq(A * B);
      Q[j - 1] = deg_y ? c : -(double)sqrtq(C * D);
    } else if (sym) {
      // T(z) = -b/z (al = b/a): p_j = a/dn_j, q_j = -p_j
      P[j - 1] = (double)(A / dn);
      Q[j - 1] = -P[j - 1];
    } else {
      P[j - 1] = (double)mob(-al * dn);
      Q[j - 1] = (double)mob(al * dn);
    }
    if (!std::isfinite(P[j - 1]) || !std::isfinite(Q[j - 1]) || !(P[j - 1] > 0) || !(Q[j - 1] < 0))
      return set_err(HPFEM_ENUMERIC, "non-finite or mis-signed shift");
  }
  return HPFEM_OK;
}

}  // namespace

/* ======================================================================= */
/* One set of solve buffers: the internal copy of G and the two iterates
 * (plus the side array and the TMA tensor maps bound to them).  The plan
 * owns one for hpfem_solve; hpfem_solve_batched adds one per stream slot. */
struct Workspace {
  double* Gp = nullptr;           // internal copy of G
  double* X1 = nullptr;           // W_{j-1/2} (deferred along y), final y-solve
  double* X2 = nullptr;           // W_j (deferred along x)
  double* Z01 = nullptr;          // chain-first y-bubbles of X1, [row][n_y][2] (element-major layout only)
  TmaPlan* tma = nullptr;         // TMA tensor maps over {Gp, X1, X2} (null = LDG kernels only)
  cudaStream_t st = nullptr;      // batched solves: the slot's stream
  cudaEvent_t done = nullptr;     // batched solves: join event
  cudaStream_t hs = nullptr;      // side stream: hat lines concurrent with the TMA bubble kernel
  cudaEvent_t hfork = nullptr, hjoin = nullptr;
};

struct hpfem_plan_s {
  DirHost hx, hy;
  DirDev dx{}, dy{};
  double omega = 0, tol = 0;
  int J = 0;
  double lam_x[2] = {0, 0}, lam_y[2] = {0, 0}, gamma = 0;
  std::vector<double> P, Q;
  size_t sx = 0, sy = 0;          // factor strides
  double* fx = nullptr;           // J sets (x-solves)
  double* fy = nullptr;           // J+1 sets (y-solves, last = mass)
  double* d_delta = nullptr;      // [n_x | n_y]
  double* d_ldtab = nullptr;      // load-source tables of both directions (DirDev::lw / lr)
  double* d_aptab = nullptr;      // hpfem_apply's tabled rows of A and M (ApplyTab), both directions
  ApplyTab apx{nullptr, nullptr, nullptr}, apy{nullptr, nullptr, nullptr};
  double* d_shift = nullptr;      // kap/sig arrays
  double* d_tau = nullptr;        // apply shifts [hw2 - p_j | hw2 + q_j] (K11)
  int* d_err = nullptr;
  Layout lay{};                   // internal padded layout (hpfem_internal.h)
  Workspace ws;                   // buffers of hpfem_solve
  std::vector<Workspace> bws;     // hpfem_solve_batched stream slots (allocated on first use)
  double* wx = nullptr;           // precomputed x-solve stencil weights, J tables
  double* wy = nullptr;           // precomputed y-solve stencil weights, J tables (table 0 unused)
  size_t wxs = 0, wys = 0;        // doubles per table
  bool use_tma = false;           // TMA half-step kernels + element-major layout
  /* Solve orientation.  Alg. 2 is symmetric in the two directions (eq.
   * adi:poisson transposed: A_y U^T M_x + M_y U^T A_x = G^T), so when the
   * long bubble chains lie along y (chains > 64 positions, beyond the TMA
   * y-solve kernel) but not along x, the plan runs Alg. 2 on the transposed
   * equation (swap = true): ox / oy are the directions of the SOLVE (ox = the
   * caller's y), oP / oQ its shifts (zolotarev with the intervals swapped),
   * the factor tables, layout, workspace and stencil tables are built in
   * that orientation, and copy-in / finalize transpose G and U (DESIGN.md
   * §6, reading R23).  Otherwise ox = dx, oy = dy, oP = P, oQ = Q. */
  bool swap = false;
  DirDev ox{}, oy{};
  std::vector<double> oP, oQ;
  Tuning tun{};                   // environment switches, read once at plan time
  long long launches = 0;
  // profiling (hpfem_plan_profile)
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;
  struct Rec { int kind, e0, e1; double bytes; };
  std::vector<Rec> recs;
  // NEXT-3 (transforms / variable coefficient / PCG), allocated on first use
  double* d_tr = nullptr;         // [T_x | V_x | T_y | V_y], (p+1)^2 each: F_p and F_p^{-1}
  double* gs0 = nullptr;          // two L_x x L_y grid / coefficient scratch arrays
  double* gs1 = nullptr;
  double* gs2 = nullptr;          // third grid array (NEXT-4 IMEX step), allocated on first use
  double* cg = nullptr;           // PCG vectors r | z | p | q (N_x N_y each)
  double* cg_part = nullptr;      // reduction partials [CG_BLOCKS]
  double* cg_sc = nullptr;        // device scalars [CG_NSC]
  double* h_sc = nullptr;         // pinned host copy of one scalar
  // CUDA graphs of whole ADI solves (launch-bound small problems), keyed by
  // (workspace, F, U, iters); captured on a plan-owned stream, launched on the caller's
  struct GraphEntry { const void* w; const double* F; double* U; int iters; cudaGraphExec_t exec; long long launches; };
  std::vector<GraphEntry> graphs;
  cudaStream_t cap = nullptr;
};

namespace {

int count_launch(hpfem_plan_t pl, cudaError_t e, const char* where, int kernels = 1) {
  if (e != cudaSuccess) return cuda_err(e, where);
  pl->launches += kernels;
  return HPFEM_OK;
}

void free_events(hpfem_plan_t pl) {
  for (cudaEvent_t e : pl->ev) cudaEventDestroy(e);
  pl->ev.clear();
  pl->ev_used = 0;
  pl->recs.clear();
}

/* record an event if profiling is on; returns its index or -1 */
int prof_mark(hpfem_plan_t pl, cudaStream_t st) {
  if (pl->ev_used >= (int)pl->ev.size()) return -1;
  if (cudaEventRecord(pl->ev[pl->ev_used], st) != cudaSuccess) return -1;
  return pl->ev_used++;
}

void prof_add(hpfem_plan_t pl, int kind, int e0, int e1, double bytes) {
  if (e0 >= 0 && e1 >= 0) pl->recs.push_back({kind, e0, e1, bytes});
}

void free_workspace(Workspace& w) {
  tma_plan_destroy(w.tma);
  cudaFree(w.Gp);
  cudaFree(w.X1);
  cudaFree(w.X2);
  cudaFree(w.Z01);
  if (w.done) cudaEventDestroy(w.done);
  if (w.st) cudaStreamDestroy(w.st);
  if (w.hfork) cudaEventDestroy(w.hfork);
  if (w.hjoin) cudaEventDestroy(w.hjoin);
  if (w.hs) cudaStreamDestroy(w.hs);
  w = Workspace();
}

void free_plan(hpfem_plan_t pl) {
  if (!pl) return;
  free_events(pl);
  free_workspace(pl->ws);
  for (Workspace& w : pl->bws) free_workspace(w);
  cudaFree(pl->fx);
  cudaFree(pl->fy);
  cudaFree(pl->d_delta);
  cudaFree(pl->d_ldtab);
  cudaFree(pl->d_aptab);
  cudaFree(pl->d_shift);
  cudaFree(pl->d_tau);
  cudaFree(pl->d_err);
  cudaFree(pl->wx);
  cudaFree(pl->wy);
  cudaFree(pl->d_tr);
  cudaFree(pl->gs0);
  cudaFree(pl->gs1);
  cudaFree(pl->gs2);
  cudaFree(pl->cg);
  cudaFree(pl->cg_part);
  cudaFree(pl->cg_sc);
  if (pl->h_sc) cudaFreeHost(pl->h_sc);
  for (auto& g : pl->graphs) cudaGraphExecDestroy(g.exec);
  if (pl->cap) cudaStreamDestroy(pl->cap);
  delete pl;
}

/* allocate (zeroed) solve buffers and bind the TMA tensor maps to them */
int alloc_workspace(hpfem_plan_t pl, Workspace& w, cudaStream_t st) {
  cudaError_t ce;
  auto fail = [&](cudaError_t e, const char* what) {
    free_workspace(w);
    return e == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, std::string(what) + ": out of device memory")
                                          : cuda_err(e, what);
  };
  const size_t bytes = sizeof(double) * ((size_t)pl->ox.N * pl->lay.ld + 64);  // +slack for bulk copies
  for (double** b : {&w.Gp, &w.X1, &w.X2}) {
    if ((ce = cudaMalloc(b, bytes)) != cudaSuccess) return fail(ce, "alloc workspace");
    if ((ce = cudaMemsetAsync(*b, 0, bytes, st)) != cudaSuccess) return fail(ce, "memset workspace");
  }
  if (pl->use_tma) {
    const size_t zb = sizeof(double) * ((size_t)pl->ox.N * 2 * pl->oy.n + 64);
    if ((ce = cudaMalloc(&w.Z01, zb)) != cudaSuccess) return fail(ce, "alloc workspace");
    if ((ce = cudaMemsetAsync(w.Z01, 0, zb, st)) != cudaSuccess) return fail(ce, "memset workspace");
  }
  double* const arrays[3] = {w.Gp, w.X1, w.X2};
  w.tma = tma_plan_create(pl->ox, pl->oy, pl->lay, arrays, pl->use_tma, pl->tun.eg_y);
  if (pl->use_tma && !tma_supports(w.tma, 0)) return fail(cudaErrorNotSupported, "TMA tensor maps");
  if (pl->use_tma) {
    if ((ce = cudaStreamCreateWithFlags(&w.hs, cudaStreamNonBlocking)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&w.hfork, cudaEventDisableTiming)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&w.hjoin, cudaEventDisableTiming)) != cudaSuccess)
      return fail(ce, "side stream");
  }
  return HPFEM_OK;
}

int validate_mesh(const double* xs, int n, int p) {
  if (!xs) return set_err(HPFEM_EINVAL, "null breakpoints");
  if (n < 1) return set_err(HPFEM_EINVAL, "n < 1");
  if (p < 2) return set_err(HPFEM_EINVAL, "p < 2");
  for (int e = 0; e < n; ++e)
    if (!(xs[e + 1] > xs[e]) || !std::isfinite(xs[e + 1]) || !std::isfinite(xs[e]))
      return set_err(HPFEM_EINVAL, "breakpoints must be finite and strictly increasing");
  return HPFEM_OK;
}

int build_plan(const double* xs, int nx, int px, const double* ys, int ny, int py, double omega, int bc, double tol,
               cudaStream_t st, hpfem_plan_t* out, const double* robin = nullptr) {
  if (!out) return set_err(HPFEM_EINVAL, "null out");
  *out = nullptr;
  int rc;
  if ((rc = validate_mesh(xs, nx, px)) != HPFEM_OK) return rc;
  if ((rc = validate_mesh(ys, ny, py)) != HPFEM_OK) return rc;
  int bx, by;
  if (!split_bc(bc, bx, by)) return set_err(HPFEM_EINVAL, "bad bc");
  if (!(tol > 0.0 && tol < 1.0)) return set_err(HPFEM_EINVAL, "tol must lie in (0,1)");
  if (!std::isfinite(omega)) return set_err(HPFEM_EINVAL, "omega not finite");
  double rob[4] = {0.0, 0.0, 0.0, 0.0};
  if (robin) {
    for (int k = 0; k < 4; ++k) {
      if (!(robin[k] >= 0.0) || !std::isfinite(robin[k])) return set_err(HPFEM_EINVAL, "Robin alpha < 0 or not finite");
      const int b1 = k < 2 ? bx : by;
      const bool dropped = (k % 2 == 0) ? drop_left(b1) : drop_right(b1);
      if (robin[k] != 0.0 && dropped) return set_err(HPFEM_EINVAL, "Robin alpha on a Dirichlet end");
      rob[k] = robin[k];
    }
  }
  const bool sing_x = bx == HPFEM_BC_NEUMANN && rob[0] == 0.0 && rob[1] == 0.0;
  const bool sing_y = by == HPFEM_BC_NEUMANN && rob[2] == 0.0 && rob[3] == 0.0;
  if ((sing_x || sing_y) && omega == 0.0) return set_err(HPFEM_EINVAL, "Neumann requires omega != 0 (P:L812)");
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) return set_err(HPFEM_ECUDA, "no CUDA device (no CPU fallback)");

  hpfem_plan_t pl = new hpfem_plan_s();
  pl->tun = read_tuning();
  pl->hx = make_dir(xs, nx, px, bx, rob);
  pl->hy = make_dir(ys, ny, py, by, rob + 2);
  pl->omega = omega;
  pl->tol = tol;
  spectral_interval(pl->hx, omega, pl->lam_x);
  spectral_interval(pl->hy, omega, pl->lam_y);
  for (double v : {pl->lam_x[0], pl->lam_x[1], pl->lam_y[0], pl->lam_y[1]})
    if (!std::isfinite(v) || !(v > 0)) {
      free_plan(pl);
      return set_err(HPFEM_ENUMERIC, "non-finite spectral bound");
    }
  // [a,b] = sigma(A_x, M_x); [c,d] = sigma(B, C) = -sigma(A_y, M_y)  (eq. adi:poisson)
  if ((rc = zolotarev(pl->lam_x[0], pl->lam_x[1], -pl->lam_y[1], -pl->lam_y[0], tol, pl->J, pl->gamma, pl->P,
                      pl->Q)) != HPFEM_OK) {
    free_plan(pl);
    return rc;
  }
  const int J = pl->J;
  const double hw2 = 0.5 * omega * omega;
  // device allocations
  auto fail_cuda = [&](cudaError_t e, const char* w) {
    free_plan(pl);
    return e == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, std::string(w) + ": out of device memory")
                                          : cuda_err(e, w);
  };
  DirHost& hx = pl->hx;
  DirHost& hy = pl->hy;
  if ((ce = cudaMalloc(&pl->d_delta, sizeof(double) * (nx + ny))) != cudaSuccess) return fail_cuda(ce, "alloc");
  if ((ce = cudaMemcpyAsync(pl->d_delta, hx.delta.data(), sizeof(double) * nx, cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return fail_cuda(ce, "copy");
  if ((ce = cudaMemcpyAsync(pl->d_delta + nx, hy.delta.data(), sizeof(double) * ny, cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return fail_cuda(ce, "copy");
  auto mkdev = [](const DirHost& h, const double* dd) {
    DirDev d;
    d.n = h.n; d.p = h.p; d.bc = h.bc; d.nh = h.nh; d.N = h.N; d.nb = h.nb; d.delta = dd;
    d.rob0 = h.rob[0]; d.rob1 = h.rob[1];
    d.lw = nullptr; d.lr = nullptr;
    return d;
  };
  pl->dx = mkdev(hx, pl->d_delta);
  pl->dy = mkdev(hy, pl->d_delta + nx);
  {  // load-source tables ([N][4] weights, then [N][4] rows) of both directions
    const size_t nxy = (size_t)pl->dx.N + pl->dy.N;
    if ((ce = cudaMalloc(&pl->d_ldtab, nxy * 4 * (sizeof(double) + sizeof(int)))) != cudaSuccess)
      return fail_cuda(ce, "alloc");
    double* w = pl->d_ldtab;
    int* r = reinterpret_cast<int*>(w + 4 * nxy);
    pl->dx.lw = w;
    pl->dx.lr = r;
    pl->dy.lw = w + 4 * (size_t)pl->dx.N;
    pl->dy.lr = r + 4 * (size_t)pl->dx.N;
    if ((ce = launch_load_tab(pl->dx, const_cast<int*>(pl->dx.lr), const_cast<double*>(pl->dx.lw), st)) != cudaSuccess ||
        (ce = launch_load_tab(pl->dy, const_cast<int*>(pl->dy.lr), const_cast<double*>(pl->dy.lw), st)) != cudaSuccess)
      return fail_cuda(ce, "load tables");
  }
  if (!env_int("HPFEM_NO_APPLY_TAB", 0)) {  // hpfem_apply's row tables ([7][N] idx, wA, wM per direction)
    const size_t nxy = (size_t)pl->dx.N + pl->dy.N;
    if ((ce = cudaMalloc(&pl->d_aptab, nxy * 7 * (2 * sizeof(double) + sizeof(int)))) != cudaSuccess)
      return fail_cuda(ce, "alloc");
    double* w = pl->d_aptab;
    int* r = reinterpret_cast<int*>(w + 14 * nxy);
    pl->apx = ApplyTab{r, w, w + 7 * (size_t)pl->dx.N};
    pl->apy = ApplyTab{r + 7 * (size_t)pl->dx.N, w + 14 * (size_t)pl->dx.N, w + 14 * (size_t)pl->dx.N + 7 * (size_t)pl->dy.N};
    if ((ce = launch_apply_tab(pl->dx, omega, pl->apx, st)) != cudaSuccess ||
        (ce = launch_apply_tab(pl->dy, omega, pl->apy, st)) != cudaSuccess)
      return fail_cuda(ce, "apply tables");
  }
  // solve orientation (see hpfem_plan_s::swap): transposed when only that
  // makes the half-steps expressible by the TMA kernels (or when forced by
  // HPFEM_TRANSPOSE=1 for testing), and only with the same J
  pl->ox = pl->dx;
  pl->oy = pl->dy;
  pl->oP = pl->P;
  pl->oQ = pl->Q;
  {
    const int tr = pl->tun.transpose;
    const bool want = tr == 1 || (tr < 0 && !pl->tun.no_tma && !tma_shape_ok(pl->dx, pl->dy, pl->tun.eg_y) &&
                                  tma_shape_ok(pl->dy, pl->dx, pl->tun.eg_y));
    if (want) {
      int Js = 0;
      double gs = 0.0;
      std::vector<double> sP, sQ;
      if (zolotarev(pl->lam_y[0], pl->lam_y[1], -pl->lam_x[1], -pl->lam_x[0], tol, Js, gs, sP, sQ) == HPFEM_OK &&
          Js == J) {
        pl->swap = true;
        pl->ox = pl->dy;
        pl->oy = pl->dx;
        pl->oP = sP;
        pl->oQ = sQ;
      }
    }
  }
  pl->sx = fac_stride(pl->ox);
  pl->sy = fac_stride(pl->oy);
  // shift parameter tables: x: J sets (kap=1, sig = w^2/2 - q_j); y: J sets (sig = w^2/2 + p_j) + mass
  std::vector<double> sh(4 * (size_t)(J + 1), 0.0);
  double* kx = sh.data();
  double* sgx = kx + (J + 1);
  double* ky = sgx + (J + 1);
  double* sgy = ky + (J + 1);
  for (int j = 0; j < J; ++j) {
    kx[j] = 1.0;
    sgx[j] = hw2 - pl->oQ[j];
    ky[j] = 1.0;
    sgy[j] = hw2 + pl->oP[j];
  }
  ky[J] = 0.0;
  sgy[J] = 1.0;  // C = M_y for the final W_J C^{-1}
  if ((ce = cudaMalloc(&pl->d_shift, sizeof(double) * sh.size())) != cudaSuccess) return fail_cuda(ce, "alloc");
  {  // apply shifts of the two half-steps, as solve_core forms them (A.tau, B.tau)
    std::vector<double> tau(2 * (size_t)J + 2, 0.0);
    for (int j = 0; j < J; ++j) {
      tau[j] = hw2 - pl->oP[j];
      tau[J + j] = hw2 + pl->oQ[j];
    }
    if ((ce = cudaMalloc(&pl->d_tau, sizeof(double) * tau.size())) != cudaSuccess) return fail_cuda(ce, "alloc");
    if ((ce = cudaMemcpyAsync(pl->d_tau, tau.data(), sizeof(double) * tau.size(), cudaMemcpyHostToDevice, st)) !=
        cudaSuccess)
      return fail_cuda(ce, "copy");
    if ((ce = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(ce, "copy");
  }
  if ((ce = cudaMemcpyAsync(pl->d_shift, sh.data(), sizeof(double) * sh.size(), cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return fail_cuda(ce, "copy");
  if ((ce = cudaMalloc(&pl->fx, sizeof(double) * pl->sx * J)) != cudaSuccess) return fail_cuda(ce, "alloc fx");
  if ((ce = cudaMalloc(&pl->fy, sizeof(double) * pl->sy * (J + 1))) != cudaSuccess) return fail_cuda(ce, "alloc fy");
  if ((ce = cudaMalloc(&pl->d_err, sizeof(int) * 8)) != cudaSuccess) return fail_cuda(ce, "alloc");
  if ((ce = cudaMemsetAsync(pl->d_err, 0, sizeof(int) * 8, st)) != cudaSuccess) return fail_cuda(ce, "memset");
  if ((ce = cudaMemsetAsync(pl->fx, 0, sizeof(double) * pl->sx * J, st)) != cudaSuccess) return fail_cuda(ce, "memset");
  if ((ce = cudaMemsetAsync(pl->fy, 0, sizeof(double) * pl->sy * (J + 1), st)) != cudaSuccess)
    return fail_cuda(ce, "memset");
  pl->use_tma = !pl->tun.no_tma && tma_shape_ok(pl->ox, pl->oy, pl->tun.eg_y);
  pl->lay = make_layout(pl->oy, pl->use_tma ? 1 : 0);
  if ((rc = alloc_workspace(pl, pl->ws, st)) != HPFEM_OK) {
    free_plan(pl);
    return rc;
  }
  if (pl->use_tma && !pl->tun.no_wtab) {  // stencil-weight tables of every ST_APPLY half-step
    pl->wxs = tma_wtab_doubles(pl->ox, pl->oy, pl->lay, 0);
    pl->wys = tma_wtab_doubles(pl->ox, pl->oy, pl->lay, 1);
    if ((ce = cudaMalloc(&pl->wx, sizeof(double) * pl->wxs * J)) != cudaSuccess) return fail_cuda(ce, "alloc wx");
    if ((ce = cudaMalloc(&pl->wy, sizeof(double) * pl->wys * J)) != cudaSuccess) return fail_cuda(ce, "alloc wy");
    if ((ce = cudaMemsetAsync(pl->wx, 0, sizeof(double) * pl->wxs * J, st)) != cudaSuccess) return fail_cuda(ce, "memset");
    if ((ce = cudaMemsetAsync(pl->wy, 0, sizeof(double) * pl->wys * J, st)) != cudaSuccess) return fail_cuda(ce, "memset");
  }
  const double* dsh = pl->d_shift;
  if ((ce = launch_factor(pl->ox, dsh, dsh + (J + 1), J, pl->fx, pl->sx, pl->d_err, st)) != cudaSuccess)
    return fail_cuda(ce, "factor x");
  if ((ce = launch_factor(pl->oy, dsh + 2 * (J + 1), dsh + 3 * (J + 1), J + 1, pl->fy, pl->sy, pl->d_err + 4, st)) !=
      cudaSuccess)
    return fail_cuda(ce, "factor y");
  if (pl->wx) {
    for (int j = 0; j < J; ++j) {
      // half-step B of iteration j: y-apply (A_y + q_j M_y) Corr_y(fy[j]) along the x-solve lines
      const FacView fyj = fac_view(pl->oy, pl->fy + pl->sy * j, 1.0, hw2 + pl->oP[j]);
      if ((ce = tma_build_wtab(pl->ox, pl->oy, pl->lay, 0, 1.0, hw2 + pl->oQ[j], fyj.vL, fyj.vR,
                               pl->wx + pl->wxs * j, st)) != cudaSuccess)
        return fail_cuda(ce, "stencil tables");
      if (j == 0) continue;  // half-step A of iteration 0 has no apply (W_0 = 0)
      const FacView fxp = fac_view(pl->ox, pl->fx + pl->sx * (j - 1), 1.0, hw2 - pl->oQ[j - 1]);
      if ((ce = tma_build_wtab(pl->ox, pl->oy, pl->lay, 1, 1.0, hw2 - pl->oP[j], fxp.vL, fxp.vR,
                               pl->wy + pl->wys * j, st)) != cudaSuccess)
        return fail_cuda(ce, "stencil tables");
    }
  }
  int herr[8];
  if ((ce = cudaMemcpyAsync(herr, pl->d_err, sizeof(herr), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return fail_cuda(ce, "copy err");
  if ((ce = cudaStreamSynchronize(st)) != cudaSuccess) return fail_cuda(ce, "plan sync");
  for (int dd = 0; dd < 2; ++dd)
    if (herr[4 * dd]) {
      char buf[256];
      std::snprintf(buf, sizeof buf, "non-positive pivot: direction %c, shift set %d, %s %d, degree %d",
                    dd ? 'y' : 'x', herr[4 * dd + 1], herr[4 * dd] == 1 ? "element" : "hat", herr[4 * dd + 2],
                    herr[4 * dd + 3]);
      free_plan(pl);
      return set_err(HPFEM_ENOTPD, buf);
    }
  pl->launches = 4;
  *out = pl;
  return HPFEM_OK;
}

FacView fview(hpfem_plan_t pl, int dir, int set) {
  const int J = pl->J;
  const double hw2 = 0.5 * pl->omega * pl->omega;
  if (dir == 0) return fac_view(pl->ox, pl->fx + pl->sx * set, 1.0, hw2 - pl->oQ[set]);
  if (set == J) return fac_view(pl->oy, pl->fy + pl->sy * set, 0.0, 1.0);
  return fac_view(pl->oy, pl->fy + pl->sy * set, 1.0, hw2 + pl->oP[set]);
}

bool overlap(const void* a, const void* b, size_t bytes) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bytes && y < x + bytes;
}

/* One line-solve pass.  Bubble lines: the TMA kernel when the shape allows
 * (else the LDG kernel); hat lines of the other direction: the LDG kernel;
 * then the hat solve.  Algorithmic bytes per dof: read G (if used), read the
 * previous iterate (if any), write the output.
 * ia_g / ia_w: which of {Gp, X1, X2} are G and Xp (-1 = unused). */
int run_step(hpfem_plan_t pl, const Workspace& w, StepParams P, cudaStream_t st, bool final_step, int ia_g,
             int ia_w) {
  const double per = 8.0 * ((P.alphaG != 0.0 ? 1 : 0) + (P.mode != ST_NONE ? 1 : 0) + 1);
  const int k0 = final_step ? 2 : (P.dir == 0 ? 5 : 0), k1 = final_step ? 2 : (P.dir == 0 ? 6 : 1);
  int rc;
  const int e0 = prof_mark(pl, st);
  // Concurrent hat lines: the persistent TMA grid leaves `spare` SMs to the
  // hat-line kernel on the side stream.  HPFEM_HAT_SMS sets `spare` (0 =
  // serial).  When profiling, the event after the bubble kernel is recorded
  // on the launch stream before the join, so it times the bubble kernel alone
  // in the same concurrent configuration (the hat lines are in no kind).
  P.tun = pl->tun;
  const int spare_env = pl->tun.hat_sms;
  if (tma_supports(w.tma, P.dir) && P.o.nh > 0 && spare_env != 0 && w.hs) {
    StepParams H = P;
    H.lp_begin = P.dir == 0 ? 0 : P.o.nb;
    H.lp_count = P.o.nh;
    cudaError_t ce;
    if ((ce = cudaEventRecord(w.hfork, st)) != cudaSuccess) return cuda_err(ce, "fork");
    rc = count_launch(pl, tma_launch_step(w.tma, P, ia_g, ia_w, st, spare_env > 0 ? spare_env : 0),
                      "TMA bubble kernel");
    if (rc) return rc;
    prof_add(pl, k0, e0, prof_mark(pl, st), per * (double)P.o.nb * P.s.nb);
    if ((ce = cudaStreamWaitEvent(w.hs, w.hfork, 0)) != cudaSuccess) return cuda_err(ce, "fork");
    rc = count_launch(pl, launch_hat_lines(H, w.hs), "hat-line kernel");
    if (rc) return rc;
    // The hat Schur solves of those hat lines follow them on the side stream;
    // the ones of the bubble lines need the bubble kernel only, so neither
    // waits for the other (joined before the next half-step).
    // (not for the stream slots of hpfem_solve_batched: their solves are
    // launch-bound and the extra launch costs more than the overlap gains --
    // config 2, B = 256: 220 -> 350 ms)
    const bool split = P.s.nh > 0 && hats_split_ok(P) && !pl->tun.no_hat_split && &w == &pl->ws;
    if (split) {
      StepParams K = P;
      K.hl_begin = P.dir == 1 ? P.o.nb : 0;
      K.hl_end = P.dir == 1 ? P.o.N : P.lay.hb;
      rc = count_launch(pl, launch_step_hats(K, w.hs), "hat kernel (hat lines)");
      if (rc) return rc;
      K.hl_begin = P.dir == 1 ? 0 : P.lay.hb;
      K.hl_end = P.dir == 1 ? P.o.nb : P.ld;
      const int e2 = prof_mark(pl, st);
      rc = count_launch(pl, launch_step_hats(K, st), "hat kernel");
      if (rc) return rc;
      prof_add(pl, k1, e2, prof_mark(pl, st), per * (double)P.o.nb * P.s.nh);
    }
    if ((ce = cudaEventRecord(w.hjoin, w.hs)) != cudaSuccess) return cuda_err(ce, "join");
    if ((ce = cudaStreamWaitEvent(st, w.hjoin, 0)) != cudaSuccess) return cuda_err(ce, "join");
    if (split) return HPFEM_OK;
  } else if (tma_supports(w.tma, P.dir)) {
    rc = count_launch(pl, tma_launch_step(w.tma, P, ia_g, ia_w, st), "TMA bubble kernel");
    if (rc) return rc;
    const int e1 = prof_mark(pl, st);
    prof_add(pl, k0, e0, e1, per * (double)P.o.nb * P.s.nb);
    // the other direction's hat lines
    StepParams H = P;
    H.lp_begin = P.dir == 0 ? 0 : P.o.nb;
    H.lp_count = P.o.nh;
    if (H.lp_count > 0) {
      rc = count_launch(pl, launch_hat_lines(H, st), "hat-line kernel");
      if (rc) return rc;
      prof_add(pl, k1, e1, prof_mark(pl, st), per * (double)P.o.nh * P.s.nb);
    }
  } else {
    rc = count_launch(pl, launch_step_bubbles(P, st), "bubble kernel");
    if (rc) return rc;
    prof_add(pl, k0, e0, prof_mark(pl, st), per * (double)P.o.N * P.s.nb);
  }
  if (P.s.nh > 0) {
    const int e2 = prof_mark(pl, st);
    rc = count_launch(pl, launch_step_hats(P, st), "hat kernel");
    if (rc) return rc;
    prof_add(pl, k1, e2, prof_mark(pl, st), per * (double)P.o.N * P.s.nh);
  }
  return HPFEM_OK;
}

}  // namespace

extern "C" {

const char* hpfem_last_error(void) { return t_err.c_str(); }

int hpfem_plan_mesh(const double* xs, int n_x, int p_x, const double* ys, int n_y, int p_y, double omega, int bc,
                    double tol, void* cuda_stream, hpfem_plan_t* out) {
  t_err.clear();
  return build_plan(xs, n_x, p_x, ys, n_y, p_y, omega, bc, tol, (cudaStream_t)cuda_stream, out);
}

int hpfem_plan_robin(const double* xs, int n_x, int p_x, const double* ys, int n_y, int p_y, double omega, int bc,
                     const double* alpha, double tol, void* cuda_stream, hpfem_plan_t* out) {
  t_err.clear();
  if (!alpha) return set_err(HPFEM_EINVAL, "null alpha");
  return build_plan(xs, n_x, p_x, ys, n_y, p_y, omega, bc, tol, (cudaStream_t)cuda_stream, out, alpha);
}

int hpfem_plan(int n_x, int p_x, int n_y, int p_y, double a, double b, double c, double d, double omega, int bc,
               double tol, void* cuda_stream, hpfem_plan_t* out) {
  t_err.clear();
  if (n_x < 1 || n_y < 1) return set_err(HPFEM_EINVAL, "n < 1");
  if (!(b > a) || !(d > c)) return set_err(HPFEM_EINVAL, "empty domain");
  std::vector<double> xs(n_x + 1), ys(n_y + 1);
  for (int e = 0; e <= n_x; ++e) xs[e] = a + (b - a) * ((double)e / n_x);
  for (int e = 0; e <= n_y; ++e) ys[e] = c + (d - c) * ((double)e / n_y);
  return build_plan(xs.data(), n_x, p_x, ys.data(), n_y, p_y, omega, bc, tol, (cudaStream_t)cuda_stream, out);
}

int hpfem_plan_info(hpfem_plan_t pl, int* N_x, int* N_y, int* J, double* lam_x, double* lam_y, double* gamma) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  if (N_x) *N_x = pl->hx.N;
  if (N_y) *N_y = pl->hy.N;
  if (J) *J = pl->J;
  if (lam_x) { lam_x[0] = pl->lam_x[0]; lam_x[1] = pl->lam_x[1]; }
  if (lam_y) { lam_y[0] = pl->lam_y[0]; lam_y[1] = pl->lam_y[1]; }
  if (gamma) *gamma = pl->gamma;
  return HPFEM_OK;
}

int hpfem_plan_dims(hpfem_plan_t pl, int* n_x, int* p_x, int* n_y, int* p_y) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  if (n_x) *n_x = pl->hx.n;
  if (p_x) *p_x = pl->hx.p;
  if (n_y) *n_y = pl->hy.n;
  if (p_y) *p_y = pl->hy.p;
  return HPFEM_OK;
}

static bool small_path(hpfem_plan_t pl);

int hpfem_plan_path(hpfem_plan_t pl, int* path, int* transposed) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  if (path) *path = small_path(pl) ? 0 : (pl->use_tma ? 1 : 2);
  if (transposed) *transposed = pl->swap ? 1 : 0;
  return HPFEM_OK;
}

int hpfem_plan_shifts(hpfem_plan_t pl, double* p, double* q) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  if (p) std::memcpy(p, pl->P.data(), sizeof(double) * pl->J);
  if (q) std::memcpy(q, pl->Q.data(), sizeof(double) * pl->J);
  return HPFEM_OK;
}

int hpfem_plan_launches(hpfem_plan_t pl, long long* launches) {
  if (!pl || !launches) return set_err(HPFEM_EINVAL, "null argument");
  *launches = pl->launches;
  return HPFEM_OK;
}

/* The 2 iters + 1 line-solve passes of Algorithm 2 on one workspace, in
 * order (run_step executes one). */
struct StepRec {
  StepParams P;
  bool fin;        // the final W_J C^{-1} pass (profile kind 2)
  int ia_g, ia_w;  // G / Xp among {Gp, X1, X2} (TMA tensor maps)
};

static void build_steps(hpfem_plan_t pl, const Workspace& w, int iters, std::vector<StepRec>& out) {
  const double hw2 = 0.5 * pl->omega * pl->omega;
  out.clear();
  auto base = [&](int dir) {
    StepParams P{};
    P.dir = dir;
    P.ld = pl->lay.ld;
    P.lay = pl->lay;
    P.s = dir == 0 ? pl->ox : pl->oy;
    P.o = dir == 0 ? pl->oy : pl->ox;
    P.lp_begin = 0;
    P.lp_count = P.o.N;
    P.tun = pl->tun;
    return P;
  };
  for (int j = 0; j < iters; ++j) {
    // half-step A: W_{j-1/2} = (G - (A_x - p_j M_x) W_{j-1}) (A_y + p_j M_y)^{-1}
    StepParams A = base(1);
    A.G = w.Gp;
    A.alphaG = 1.0;
    A.f = fview(pl, 1, j);
    A.out = w.X1;
    A.z01 = w.Z01;
    if (j == 0) {
      A.mode = ST_NONE;  // W_0 = 0
    } else {
      const FacView prev = fview(pl, 0, j - 1);
      A.mode = ST_APPLY;
      A.Xp = w.X2;
      A.kap_a = 1.0;
      A.tau = hw2 - pl->oP[j];
      A.cvL = prev.vL;
      A.cvR = prev.vR;
      if (pl->wy) A.wtab = pl->wy + pl->wys * j;
    }
    out.push_back({A, false, 0, j == 0 ? -1 : 2});
    // half-step B: W_j = (A_x - q_j M_x)^{-1} (G - W_{j-1/2} (A_y + q_j M_y))
    StepParams B = base(0);
    B.G = w.Gp;
    B.alphaG = 1.0;
    B.f = fview(pl, 0, j);
    B.out = w.X2;
    B.mode = ST_APPLY;
    B.Xp = w.X1;
    B.z01p = w.Z01;
    B.kap_a = 1.0;
    B.tau = hw2 + pl->oQ[j];
    B.cvL = A.f.vL;
    B.cvR = A.f.vR;
    if (pl->wx) B.wtab = pl->wx + pl->wxs * j;
    out.push_back({B, false, 0, 1});
  }
  // RETURN W_J C^{-1}: y-solves with the mass factor (then finalize materialises U)
  StepParams Fin = base(1);
  Fin.G = nullptr;
  Fin.alphaG = 0.0;
  Fin.f = fview(pl, 1, pl->J);
  Fin.out = w.X1;
  Fin.z01 = w.Z01;
  Fin.mode = ST_CORR;
  Fin.Xp = w.X2;
  const FacView last = fview(pl, 0, iters - 1);
  Fin.cvL = last.vL;
  Fin.cvR = last.vR;
  out.push_back({Fin, true, -1, 2});
}

/* Algorithm 2 on one workspace (validated arguments, iters >= 1), in three
 * parts: copy-in (the only kernels that read F), the 2 iters + 1 line-solve
 * passes (workspace buffers only), finalize (the only kernels that write U). */
static int solve_pre(hpfem_plan_t pl, const Workspace& w, const double* F, cudaStream_t st) {
  int rc;
  const int e0 = prof_mark(pl, st);
  if (pl->swap) {  // G^T into the scratch iterate X2 (dead until half-step B writes it)
    if ((rc = count_launch(pl, launch_transpose(F, pl->hx.N, pl->hy.N, w.X2, st), "transpose"))) return rc;
    F = w.X2;
  }
  if ((rc = count_launch(pl, launch_copyin(pl->ox, pl->oy, pl->lay, F, w.Gp, st), "copy-in"))) return rc;
  prof_add(pl, 2, e0, prof_mark(pl, st), 0.0);  // layout change, not algorithmic
  return HPFEM_OK;
}

static int solve_mid(hpfem_plan_t pl, const Workspace& w, int iters, cudaStream_t st) {
  int rc;
  std::vector<StepRec> steps;
  build_steps(pl, w, iters, steps);
  NvtxRange solve_range("hpfem_solve");
  for (const StepRec& r : steps) {
    NvtxRange nr(r.fin ? "final W_J C^-1" : (r.P.dir == 1 ? "ADI half-step A (y-solves)" : "ADI half-step B (x-solves)"));
    if ((rc = run_step(pl, w, r.P, st, r.fin, r.ia_g, r.ia_w))) return rc;
  }
  return HPFEM_OK;
}

static int solve_post(hpfem_plan_t pl, const Workspace& w, double* U, cudaStream_t st) {
  const FacView fin = fview(pl, 1, pl->J);  // the final mass solve's correction vectors
  const int e0 = prof_mark(pl, st);
  // (swap: U^T into the dead iterate X2, then transposed into U)
  int rc = count_launch(pl, launch_finalize(pl->ox, pl->oy, pl->lay, fin.vL, fin.vR, w.X1, pl->swap ? w.X2 : U, st),
                        "finalize");
  if (!rc && pl->swap) rc = count_launch(pl, launch_transpose(w.X2, pl->ox.N, pl->oy.N, U, st), "transpose");
  prof_add(pl, 2, e0, prof_mark(pl, st), 0.0);
  return rc;
}

static int solve_core(hpfem_plan_t pl, const Workspace& w, const double* F, double* U, int iters, cudaStream_t st) {
  int rc;
  if ((rc = solve_pre(pl, w, F, st))) return rc;
  if ((rc = solve_mid(pl, w, iters, st))) return rc;
  return solve_post(pl, w, U, st);
}

/* solve_core replayed from a CUDA graph: the whole solve (6J + 3 kernels and
 * the side-stream fork/joins) is captured once per (workspace, F, U, iters)
 * on a plan-owned stream and launched on `st` -- one launch instead of
 * hundreds, which is what bounds the small configurations.  Bitwise the same
 * kernels with the same arguments.  Not used while profiling (per-launch
 * events) or with HPFEM_NO_GRAPH=1; at most kMaxGraphs cached. */
static int solve_graph(hpfem_plan_t pl, const Workspace& w, const double* F, double* U, int iters,
                       cudaStream_t st, bool mid_only = false) {
  // mid_only (hpfem_solve_batched): the graph holds the line-solve passes only
  // -- they touch the workspace's buffers and nothing else, so one graph per
  // stream slot serves every right-hand side; copy-in and finalize are
  // launched around it.  Keyed by the workspace's Gp (the slots live in a
  // vector that may move them).
  if (pl->tun.no_graph || !pl->ev.empty())
    return mid_only ? solve_mid(pl, w, iters, st) : solve_core(pl, w, F, U, iters, st);
  cudaError_t ce;
  const void* key = mid_only ? (const void*)w.Gp : (const void*)&w;
  if (mid_only) {
    F = nullptr;
    U = nullptr;
  }
  for (auto& g : pl->graphs)
    if (g.w == key && g.F == F && g.U == U && g.iters == iters) {
      if ((ce = cudaGraphLaunch(g.exec, st)) != cudaSuccess) return cuda_err(ce, "graph launch");
      pl->launches += g.launches;
      return HPFEM_OK;
    }
  if (!pl->cap && (ce = cudaStreamCreateWithFlags(&pl->cap, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(ce, "capture stream");
  if ((ce = cudaStreamBeginCapture(pl->cap, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
    return cuda_err(ce, "begin capture");
  const long long l0 = pl->launches;
  int rc = mid_only ? solve_mid(pl, w, iters, pl->cap) : solve_core(pl, w, F, U, iters, pl->cap);
  cudaGraph_t graph = nullptr;
  ce = cudaStreamEndCapture(pl->cap, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return cuda_err(ce, "end capture");
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return cuda_err(ce, "graph instantiate");
  constexpr size_t kMaxGraphs = 16;  // (up to 8 stream slots of hpfem_solve_batched + single solves)
  if (pl->graphs.size() >= kMaxGraphs) {
    cudaGraphExecDestroy(pl->graphs.front().exec);
    pl->graphs.erase(pl->graphs.begin());
  }
  pl->graphs.push_back({key, F, U, iters, exec, pl->launches - l0});
  if ((ce = cudaGraphLaunch(exec, st)) != cudaSuccess) return cuda_err(ce, "graph launch");
  return HPFEM_OK;
}

/* K11: whole solve(s) in one kernel, one CTA per problem, when the three
 * arrays fit in shared memory (HPFEM_NO_SMALL=1 disables; not while
 * profiling, so that the per-kind profile stays the multi-kernel path's) */
static bool small_path(hpfem_plan_t pl) {
  if (pl->tun.no_small) return false;
  return !pl->swap && pl->ev.empty() && small_smem_bytes(pl->dx, pl->dy) <= SMALL_SMEM_MAX;
}

static int solve_small(hpfem_plan_t pl, int batch, const double* F, double* U, int iters, cudaStream_t st);

/* a full solve of one right-hand side by whichever path hpfem_solve takes */
static int solve_any(hpfem_plan_t pl, const double* F, double* U, cudaStream_t st) {
  return small_path(pl) ? solve_small(pl, 1, F, U, pl->J, st) : solve_graph(pl, pl->ws, F, U, pl->J, st);
}

static int solve_small(hpfem_plan_t pl, int batch, const double* F, double* U, int iters, cudaStream_t st) {
  SmallArgs a{};
  a.x = pl->dx;
  a.y = pl->dy;
  a.fx = pl->fx;
  a.fy = pl->fy;
  a.sx = pl->sx;
  a.sy = pl->sy;
  a.sh = pl->d_shift;
  a.tau = pl->d_tau;
  a.J = pl->J;
  a.iters = iters;
  a.F = F;
  a.U = U;
  return count_launch(pl, launch_adi_small(a, batch, st), "small ADI kernel");
}

int hpfem_solve_iters(hpfem_plan_t pl, const double* F, double* U, int iters, void* cuda_stream) {
  t_err.clear();
  if (!pl || !F || !U) return set_err(HPFEM_EINVAL, "null argument");
  if (iters < 0 || iters > pl->J) return set_err(HPFEM_EINVAL, "iters must lie in [0, J]");
  const size_t bytes = sizeof(double) * (size_t)pl->hx.N * pl->hy.N;
  if (overlap(F, U, bytes)) return set_err(HPFEM_EINVAL, "F and U overlap");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  pl->launches = 0;
  if (iters == 0) {  // W_0 = 0
    cudaError_t ce = cudaMemsetAsync(U, 0, bytes, st);
    return ce == cudaSuccess ? HPFEM_OK : cuda_err(ce, "memset");
  }
  if (small_path(pl)) return solve_small(pl, 1, F, U, iters, st);
  return solve_graph(pl, pl->ws, F, U, iters, st);
}

int hpfem_solve_batched(hpfem_plan_t pl, int batch, const double* F, double* U, void* cuda_stream) {
  t_err.clear();
  if (!pl || !F || !U) return set_err(HPFEM_EINVAL, "null argument");
  if (batch < 0) return set_err(HPFEM_EINVAL, "batch < 0");
  const size_t nn = (size_t)pl->hx.N * pl->hy.N;
  if (overlap(F, U, sizeof(double) * nn * (size_t)batch)) return set_err(HPFEM_EINVAL, "F and U overlap");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  pl->launches = 0;
  if (batch == 0) return HPFEM_OK;
  if (!pl->ev.empty()) return set_err(HPFEM_EINVAL, "profiling is on: batched solves run on several streams");
  if (small_path(pl)) return solve_small(pl, batch, F, U, pl->J, st);  // one CTA per problem
  int slots = batch < pl->tun.batch_streams ? batch : pl->tun.batch_streams;
  cudaError_t ce;
  while ((int)pl->bws.size() < slots) {  // stream slots, each with its own buffers
    Workspace w;
    int rc = alloc_workspace(pl, w, st);
    if (rc != HPFEM_OK) return rc;
    if ((ce = cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming)) != cudaSuccess) {
      free_workspace(w);
      return cuda_err(ce, "batch stream");
    }
    pl->bws.push_back(w);
  }
  // fork: every slot stream waits for the work already queued on st
  cudaEvent_t fork = pl->bws[0].done;
  if ((ce = cudaEventRecord(fork, st)) != cudaSuccess) return cuda_err(ce, "fork");
  for (int k = 0; k < slots; ++k)
    if ((ce = cudaStreamWaitEvent(pl->bws[k].st, fork, 0)) != cudaSuccess) return cuda_err(ce, "fork");
  long long total = 0;
  for (int b = 0; b < batch; ++b) {
    const Workspace& w = pl->bws[b % slots];
    pl->launches = 0;
    // copy-in, the slot's graph of the line-solve passes (one graph launch
    // instead of 6J + 1 kernel launches: the batch is launch-bound otherwise),
    // finalize
    int rc = solve_pre(pl, w, F + (size_t)b * nn, w.st);
    if (rc == HPFEM_OK) rc = solve_graph(pl, w, nullptr, nullptr, pl->J, w.st, true);
    if (rc == HPFEM_OK) rc = solve_post(pl, w, U + (size_t)b * nn, w.st);
    total += pl->launches;
    if (rc != HPFEM_OK) return rc;
  }
  pl->launches = total;
  // join
  for (int k = 0; k < slots; ++k) {
    if ((ce = cudaEventRecord(pl->bws[k].done, pl->bws[k].st)) != cudaSuccess) return cuda_err(ce, "join");
    if ((ce = cudaStreamWaitEvent(st, pl->bws[k].done, 0)) != cudaSuccess) return cuda_err(ce, "join");
  }
  return HPFEM_OK;
}

int hpfem_solve(hpfem_plan_t pl, const double* F, double* U, void* cuda_stream) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  return hpfem_solve_iters(pl, F, U, pl->J, cuda_stream);
}

int hpfem_apply(hpfem_plan_t pl, const double* U, double* F, void* cuda_stream) {
  t_err.clear();
  if (!pl || !U || !F) return set_err(HPFEM_EINVAL, "null argument");
  if (overlap(U, F, sizeof(double) * (size_t)pl->hx.N * pl->hy.N)) return set_err(HPFEM_EINVAL, "U and F overlap");
  pl->launches = 0;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int e0 = prof_mark(pl, st);
  const int rc = count_launch(pl, launch_apply2d(pl->dx, pl->dy, pl->omega, U, F, st, &pl->apx, &pl->apy), "apply");
  prof_add(pl, 4, e0, prof_mark(pl, st), 16.0 * pl->hx.N * pl->hy.N);
  return rc;
}

int hpfem_load(hpfem_plan_t pl, const double* F_leg, double* G, void* cuda_stream) {
  t_err.clear();
  if (!pl || !F_leg || !G) return set_err(HPFEM_EINVAL, "null argument");
  const size_t bl = sizeof(double) * (size_t)(pl->hx.p + 1) * pl->hx.n * (pl->hy.p + 1) * pl->hy.n;
  const size_t bg = sizeof(double) * (size_t)pl->hx.N * pl->hy.N;
  const char* a = (const char*)F_leg;
  const char* b = (const char*)G;
  if (a < b + bg && b < a + bl) return set_err(HPFEM_EINVAL, "F_leg and G overlap");
  pl->launches = 0;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int e0 = prof_mark(pl, st);
  const int rc = count_launch(pl, launch_load2d(pl->dx, pl->dy, F_leg, G, st), "load");
  prof_add(pl, 3, e0, prof_mark(pl, st), (double)bl + (double)bg);
  return rc;
}

int hpfem_unload(hpfem_plan_t pl, const double* U, double* C_leg, void* cuda_stream) {
  t_err.clear();
  if (!pl || !U || !C_leg) return set_err(HPFEM_EINVAL, "null argument");
  const size_t bu = sizeof(double) * (size_t)pl->hx.N * pl->hy.N;
  const size_t bl = sizeof(double) * (size_t)(pl->hx.p + 1) * pl->hx.n * (pl->hy.p + 1) * pl->hy.n;
  const char* a = (const char*)U;
  const char* b = (const char*)C_leg;
  if (a < b + bl && b < a + bu) return set_err(HPFEM_EINVAL, "U and C_leg overlap");
  pl->launches = 0;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int e0 = prof_mark(pl, st);
  const int rc = count_launch(pl, launch_unload2d(pl->dx, pl->dy, U, C_leg, st), "unload");
  prof_add(pl, 3, e0, prof_mark(pl, st), (double)bl + (double)bu);
  return rc;
}

/* ---------------- NEXT-3: transforms, variable coefficient, PCG ---------------- */
}  // extern "C"

namespace {

typedef long double ld_t;

/* reference points x_i = cos(pi (2i + 1) / (2m)), i = 0..m-1, m = p + 1: the
 * paper's first-kind Chebyshev points sin(pi (m - 2k + 1)/(2m)), k = i + 1
 * (reading R17), descending */
ld_t cheb_theta(int i, int m) { return 3.14159265358979323846264338327950288L * (2 * i + 1) / (2.0L * m); }

/* Legendre P_0..P_p at x (Bonnet recurrence) */
void legendre_all(ld_t x, int p, ld_t* P) {
  P[0] = 1.0L;
  if (p >= 1) P[1] = x;
  for (int k = 1; k < p; ++k) P[k + 1] = ((2 * k + 1) * x * P[k] - k * P[k - 1]) / (k + 1);
}

/* Gauss-Legendre nodes and weights (Newton on P_m) */
void gauss_legendre(int m, std::vector<ld_t>& x, std::vector<ld_t>& w) {
  x.resize(m);
  w.resize(m);
  std::vector<ld_t> P(m + 1);
  for (int i = 0; i < m; ++i) {
    ld_t z = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (m + 0.5L)), dp = 0;
    for (int it = 0; it < 100; ++it) {
      legendre_all(z, m, P.data());
      dp = m * (z * P[m] - P[m - 1]) / (z * z - 1.0L);
      const ld_t dz = P[m] / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    legendre_all(z, m, P.data());
    dp = m * (z * P[m] - P[m - 1]) / (z * z - 1.0L);
    x[i] = z;
    w[i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
}

/* T = F_p (values at the m = p + 1 points -> Legendre coefficients) as the
 * product of the DCT-II (values -> Chebyshev coefficients of the
 * interpolant, a_j = (2 - delta_j0)/m sum_i f_i cos(j theta_i)) with the
 * Chebyshev -> Legendre conversion L[k][j] = (k + 1/2) int P_k T_j (Gauss-
 * Legendre, m nodes: exact for k + j <= 2m - 1), the construction of
 * P:L904-L908; V = F_p^{-1}, V[i][k] = P_k(x_i).  Row-major (p+1)^2, extended
 * precision, rounded once. */
void transform_matrices(int p, double* T, double* V) {
  const int m = p + 1;
  std::vector<ld_t> gx, gw, P(m + 1), L((size_t)m * m, 0.0L), D((size_t)m * m);
  gauss_legendre(m, gx, gw);
  for (int q = 0; q < m; ++q) {
    legendre_all(gx[q], p, P.data());
    const ld_t th = acosl(gx[q]);
    for (int j = 0; j < m; ++j) {
      const ld_t Tj = cosl(j * th);
      for (int k = 0; k < m; ++k) L[(size_t)k * m + j] += (k + 0.5L) * gw[q] * P[k] * Tj;
    }
  }
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) D[(size_t)j * m + i] = (j == 0 ? 1.0L : 2.0L) / m * cosl(j * cheb_theta(i, m));
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < m; ++i) {
      ld_t acc = 0;
      for (int j = 0; j < m; ++j) acc += L[(size_t)k * m + j] * D[(size_t)j * m + i];
      T[(size_t)k * m + i] = (double)acc;
    }
  for (int i = 0; i < m; ++i) {
    legendre_all(cosl(cheb_theta(i, m)), p, P.data());
    for (int k = 0; k < m; ++k) V[(size_t)i * m + k] = (double)P[k];
  }
}

size_t leg_elems(const hpfem_plan_t pl) { return (size_t)(pl->hx.p + 1) * pl->hx.n * (pl->hy.p + 1) * pl->hy.n; }

int ensure_transforms(hpfem_plan_t pl, cudaStream_t st) {
  if (pl->d_tr) return HPFEM_OK;
  const int mx = pl->hx.p + 1, my = pl->hy.p + 1;
  std::vector<double> h((size_t)2 * mx * mx + (size_t)2 * my * my);
  transform_matrices(pl->hx.p, h.data(), h.data() + (size_t)mx * mx);
  transform_matrices(pl->hy.p, h.data() + (size_t)2 * mx * mx, h.data() + (size_t)2 * mx * mx + (size_t)my * my);
  cudaError_t ce;
  const size_t gb = sizeof(double) * leg_elems(pl);
  if ((ce = cudaMalloc(&pl->d_tr, sizeof(double) * h.size())) != cudaSuccess ||
      (ce = cudaMalloc(&pl->gs0, gb)) != cudaSuccess || (ce = cudaMalloc(&pl->gs1, gb)) != cudaSuccess) {
    cudaFree(pl->d_tr);
    cudaFree(pl->gs0);
    pl->d_tr = pl->gs0 = nullptr;
    return ce == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, "transform buffers: out of device memory")
                                           : cuda_err(ce, "transform buffers");
  }
  if ((ce = cudaMemcpyAsync(pl->d_tr, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return cuda_err(ce, "transform upload");
  return cudaStreamSynchronize(st) == cudaSuccess ? HPFEM_OK : cuda_err(cudaGetLastError(), "transform upload");
}

/* the two 1D passes of one 2D transform; inverse = 0: values -> coefficients
 * (F_x . F_y^T), 1: coefficients -> values, times g if given */
int transform2d(hpfem_plan_t pl, int inverse, const double* in, double* tmp, double* out, const double* g,
                cudaStream_t st) {
  const int mx = pl->hx.p + 1, my = pl->hy.p + 1, nx = pl->hx.n, ny = pl->hy.n;
  const long long Lx = (long long)mx * nx, Ly = (long long)my * ny;
  const double* Ax = pl->d_tr + (inverse ? (size_t)mx * mx : 0);
  const double* Ay = pl->d_tr + (size_t)2 * mx * mx + (inverse ? (size_t)my * my : 0);
  ElemApply E{};
  E.A = Ax; E.M = mx; E.K = mx; E.in = in; E.out = tmp; E.g = nullptr;
  E.ncols = (long long)nx * Ly; E.nb = E.ncols; E.bs = 0; E.s = (long long)nx * Ly;
  int rc = count_launch(pl, launch_elem_apply(E, st), "transform x");
  if (rc) return rc;
  E.A = Ay; E.M = my; E.K = my; E.in = tmp; E.out = out; E.g = g;
  E.ncols = Lx * ny; E.nb = ny; E.bs = Ly; E.s = ny;
  return count_launch(pl, launch_elem_apply(E, st), "transform y");
}

/* F = A_x U M_y + M_x U A_y + <v, c u>, the last by eq. (evaluation) */
int varcoef_core(hpfem_plan_t pl, const double* cgrid, const double* U, double* F, cudaStream_t st) {
  int rc;
  if ((rc = count_launch(pl, launch_apply2d(pl->dx, pl->dy, pl->omega, U, F, st, &pl->apx, &pl->apy), "apply"))) return rc;
  if ((rc = count_launch(pl, launch_unload2d(pl->dx, pl->dy, U, pl->gs0, st), "unload"))) return rc;
  if ((rc = transform2d(pl, 1, pl->gs0, pl->gs1, pl->gs0, cgrid, st))) return rc;  // c o values
  if ((rc = transform2d(pl, 0, pl->gs0, pl->gs1, pl->gs0, nullptr, st))) return rc;
  return count_launch(pl, launch_load2d(pl->dx, pl->dy, pl->gs0, F, st, 1), "load (accumulate)");
}

/* PCG / IMEX vectors: 4 N_x N_y arrays, reduction partials, device scalars */
int ensure_vectors(hpfem_plan_t pl) {
  if (pl->cg) return HPFEM_OK;
  const size_t bn = sizeof(double) * (size_t)pl->hx.N * pl->hy.N;
  cudaError_t ce;
  if ((ce = cudaMalloc(&pl->cg, 4 * bn)) != cudaSuccess ||
      (ce = cudaMalloc(&pl->cg_part, sizeof(double) * CG_BLOCKS)) != cudaSuccess ||
      (ce = cudaMalloc(&pl->cg_sc, sizeof(double) * CG_NSC)) != cudaSuccess ||
      (ce = cudaMallocHost(&pl->h_sc, sizeof(double))) != cudaSuccess) {
    cudaFree(pl->cg);
    cudaFree(pl->cg_part);
    cudaFree(pl->cg_sc);
    pl->cg = pl->cg_part = pl->cg_sc = nullptr;
    pl->h_sc = nullptr;
    return ce == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, "vector buffers: out of device memory")
                                           : cuda_err(ce, "vector buffers");
  }
  return HPFEM_OK;
}

bool overlap_n(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

}  // namespace

extern "C" {

int hpfem_grid(hpfem_plan_t pl, double* x, double* y) {
  t_err.clear();
  if (!pl || !x || !y) return set_err(HPFEM_EINVAL, "null argument");
  for (int d = 0; d < 2; ++d) {
    const DirHost& h = d == 0 ? pl->hx : pl->hy;
    double* out = d == 0 ? x : y;
    const int m = h.p + 1;
    for (int i = 0; i < m; ++i) {
      const ld_t t = cosl(cheb_theta(i, m));
      for (int e = 0; e < h.n; ++e)
        out[(size_t)i * h.n + e] = (double)((ld_t)h.xs[e] + (t + 1.0L) * ((ld_t)h.xs[e + 1] - (ld_t)h.xs[e]) / 2.0L);
    }
  }
  return HPFEM_OK;
}

int hpfem_transform(hpfem_plan_t pl, const double* V, double* C, void* cuda_stream) {
  t_err.clear();
  if (!pl || !V || !C) return set_err(HPFEM_EINVAL, "null argument");
  const size_t b = sizeof(double) * leg_elems(pl);
  if (overlap_n(V, b, C, b)) return set_err(HPFEM_EINVAL, "V and C overlap");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  pl->launches = 0;
  int rc = ensure_transforms(pl, st);
  if (rc) return rc;
  return transform2d(pl, 0, V, pl->gs0, C, nullptr, st);
}

int hpfem_itransform(hpfem_plan_t pl, const double* C, double* V, void* cuda_stream) {
  t_err.clear();
  if (!pl || !V || !C) return set_err(HPFEM_EINVAL, "null argument");
  const size_t b = sizeof(double) * leg_elems(pl);
  if (overlap_n(V, b, C, b)) return set_err(HPFEM_EINVAL, "C and V overlap");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  pl->launches = 0;
  int rc = ensure_transforms(pl, st);
  if (rc) return rc;
  return transform2d(pl, 1, C, pl->gs0, V, nullptr, st);
}

int hpfem_varcoef_apply(hpfem_plan_t pl, const double* cgrid, const double* U, double* F, void* cuda_stream) {
  t_err.clear();
  if (!pl || !cgrid || !U || !F) return set_err(HPFEM_EINVAL, "null argument");
  const size_t bn = sizeof(double) * (size_t)pl->hx.N * pl->hy.N, bl = sizeof(double) * leg_elems(pl);
  if (overlap_n(U, bn, F, bn) || overlap_n(cgrid, bl, F, bn)) return set_err(HPFEM_EINVAL, "F overlaps an input");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  pl->launches = 0;
  int rc = ensure_transforms(pl, st);
  if (rc) return rc;
  return varcoef_core(pl, cgrid, U, F, st);
}

int hpfem_pcg(hpfem_plan_t pl, const double* cgrid, const double* G, double* U, double rtol, int maxit, int* iters,
              double* relres, void* cuda_stream) {
  t_err.clear();
  if (!pl || !cgrid || !G || !U) return set_err(HPFEM_EINVAL, "null argument");
  if (!(rtol >= 0.0) || maxit < 0) return set_err(HPFEM_EINVAL, "rtol < 0 or maxit < 0");
  const size_t nn = (size_t)pl->hx.N * pl->hy.N, bn = sizeof(double) * nn, bl = sizeof(double) * leg_elems(pl);
  if (overlap_n(G, bn, U, bn) || overlap_n(cgrid, bl, U, bn)) return set_err(HPFEM_EINVAL, "U overlaps an input");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  long long launches = 0;
  pl->launches = 0;
  int rc = ensure_transforms(pl, st);
  if (rc) return rc;
  cudaError_t ce;
  if ((rc = ensure_vectors(pl))) return rc;
  double *r = pl->cg, *z = r + nn, *p = z + nn, *q = p + nn;
  auto read_rr = [&](double& v) {
    if ((ce = cudaMemcpyAsync(pl->h_sc, pl->cg_sc + CG_RRV, sizeof(double), cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess ||
        (ce = cudaStreamSynchronize(st)) != cudaSuccess)
      return cuda_err(ce, "pcg residual");
    v = *pl->h_sc;
    return (int)HPFEM_OK;
  };
  auto step = [&](int r_) {
    launches += pl->launches;
    pl->launches = 0;
    return r_;
  };
  if ((ce = cudaMemsetAsync(U, 0, bn, st)) != cudaSuccess) return cuda_err(ce, "pcg init");
  if ((ce = cudaMemcpyAsync(r, G, bn, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return cuda_err(ce, "pcg init");
  if ((rc = count_launch(pl, launch_dot(G, G, nn, pl->cg_part, pl->cg_sc, CG_RR, st), "pcg dot", 2))) return rc;
  double bb = 0.0;
  if ((rc = read_rr(bb))) return rc;
  const double nb = std::sqrt(bb);
  int it = 0;
  double rel = nb > 0.0 ? 1.0 : 0.0;
  if (nb > 0.0) {
    if ((rc = step(solve_any(pl, r, z, st)))) return rc;  // z = P r (ADI)
    if ((rc = count_launch(pl, launch_dot(r, z, nn, pl->cg_part, pl->cg_sc, CG_RZ0, st), "pcg dot", 2))) return rc;
    if ((rc = count_launch(pl, launch_cg_p(p, z, nn, pl->cg_sc, 1, st), "pcg p"))) return rc;
    while (it < maxit) {
      if ((rc = step(varcoef_core(pl, cgrid, p, q, st)))) return rc;  // q = A p
      if ((rc = count_launch(pl, launch_dot(p, q, nn, pl->cg_part, pl->cg_sc, CG_ALPHA, st), "pcg dot", 2)))
        return rc;
      if ((rc = count_launch(pl, launch_cg_xr(U, r, p, q, nn, pl->cg_part, pl->cg_sc, st), "pcg update", 2)))
        return rc;
      ++it;
      double rr = 0.0;
      if ((rc = read_rr(rr))) return rc;
      rel = std::sqrt(rr) / nb;
      if (!std::isfinite(rel)) return set_err(HPFEM_ENUMERIC, "pcg: non-finite residual");
      if (rel <= rtol) break;
      if ((rc = step(solve_any(pl, r, z, st)))) return rc;
      if ((rc = count_launch(pl, launch_dot(r, z, nn, pl->cg_part, pl->cg_sc, CG_BETA, st), "pcg dot", 2))) return rc;
      if ((rc = count_launch(pl, launch_cg_p(p, z, nn, pl->cg_sc, 0, st), "pcg p"))) return rc;
    }
  }
  pl->launches += launches;
  if (iters) *iters = it;
  if (relres) *relres = rel;
  return HPFEM_OK;
}

int hpfem_imex_step(hpfem_plan_t pl, double dt, const double* U_leg, double* U_next, void* cuda_stream) {
  t_err.clear();
  if (!pl || !U_leg || !U_next) return set_err(HPFEM_EINVAL, "null argument");
  if (!(dt > 0.0) || !std::isfinite(dt)) return set_err(HPFEM_EINVAL, "dt must be positive");
  if (pl->omega == 0.0) return set_err(HPFEM_EINVAL, "the plan's omega must be 1/sqrt(dt eps) > 0");
  const size_t bl = sizeof(double) * leg_elems(pl);
  if (overlap_n(U_leg, bl, U_next, bl)) return set_err(HPFEM_EINVAL, "U_leg and U_next overlap");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  long long launches = 0;
  pl->launches = 0;
  int rc = ensure_transforms(pl, st);
  if (rc) return rc;
  if ((rc = ensure_vectors(pl))) return rc;
  if (!pl->gs2) {
    cudaError_t ce = cudaMalloc(&pl->gs2, bl);
    if (ce != cudaSuccess) {
      pl->gs2 = nullptr;
      return ce == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, "imex buffer: out of device memory")
                                             : cuda_err(ce, "imex buffer");
    }
  }
  const size_t nn = (size_t)pl->hx.N * pl->hy.N;
  double *G = pl->cg, *W = G + nn;
  // linear half-step (implicit Euler): (I - dt eps Delta) w = u_k in the
  // Galerkin form (K(x)M + M(x)K + w^2 M(x)M) W = w^2 <v, u_k>, w^2 = 1/(dt eps)
  const double w2 = pl->omega * pl->omega;
  if ((rc = count_launch(pl, launch_load2d(pl->dx, pl->dy, U_leg, G, st, 0, w2), "imex load"))) return rc;
  launches += pl->launches;
  pl->launches = 0;
  if ((rc = solve_any(pl, G, W, st))) return rc;
  launches += pl->launches;
  pl->launches = 0;
  // nonlinear half-step (explicit Euler, reading R21):
  // U_{k+1} = F [V - dt V_x o V],  V = F^{-1} R W R^T F^{-T},  V_x = F^{-1} D W R^T F^{-T}
  if ((rc = count_launch(pl, launch_unload2d(pl->dx, pl->dy, W, pl->gs0, st, 0), "imex unload"))) return rc;
  if ((rc = transform2d(pl, 1, pl->gs0, pl->gs1, pl->gs2, nullptr, st))) return rc;  // V
  if ((rc = count_launch(pl, launch_unload2d(pl->dx, pl->dy, W, pl->gs0, st, 1), "imex dunload"))) return rc;
  {
    const int mx = pl->hx.p + 1, my = pl->hy.p + 1, nx = pl->hx.n, ny = pl->hy.n;
    const long long Lx = (long long)mx * nx, Ly = (long long)my * ny;
    ElemApply E{};
    E.A = pl->d_tr + (size_t)mx * mx;  // V_x (x pass of the inverse transform)
    E.M = mx; E.K = mx; E.in = pl->gs0; E.out = pl->gs1;
    E.ncols = (long long)nx * Ly; E.nb = E.ncols; E.bs = 0; E.s = (long long)nx * Ly;
    if ((rc = count_launch(pl, launch_elem_apply(E, st), "imex itransform x"))) return rc;
    E.A = pl->d_tr + (size_t)2 * mx * mx + (size_t)my * my;  // y pass, epilogue V - dt V_x o V
    E.M = my; E.K = my; E.in = pl->gs1; E.out = pl->gs0; E.g = pl->gs2; E.h = pl->gs2; E.alpha = -dt;
    E.ncols = Lx * ny; E.nb = ny; E.bs = Ly; E.s = ny;
    if ((rc = count_launch(pl, launch_elem_apply(E, st), "imex itransform y"))) return rc;
  }
  rc = transform2d(pl, 0, pl->gs0, pl->gs1, U_next, nullptr, st);
  pl->launches += launches;
  return rc;
}

/* ---------------- 1D solver workload (NEXT-2, the paper's Fig. 1) ---------------- */
}  // extern "C"

struct hpfem_plan1d_s {
  DirHost h;
  DirDev d{};
  double omega = 0;
  double* d_delta = nullptr;
  double* d_ks = nullptr;  // kap, sig
  double* fac = nullptr;
  int* d_err = nullptr;
};

static void free_plan1d(hpfem_plan1d_t pl) {
  if (!pl) return;
  cudaFree(pl->d_delta);
  cudaFree(pl->d_ks);
  cudaFree(pl->fac);
  cudaFree(pl->d_err);
  delete pl;
}

extern "C" {

int hpfem_plan1d(const double* xs, int n, int p, int bc, double omega, void* cuda_stream, hpfem_plan1d_t* out) {
  t_err.clear();
  if (!out) return set_err(HPFEM_EINVAL, "null out");
  *out = nullptr;
  int rc;
  if ((rc = validate_mesh(xs, n, p)) != HPFEM_OK) return rc;
  if (bc < HPFEM_BC_DIRICHLET || bc > HPFEM_BC_NEUMANN_DIRICHLET) return set_err(HPFEM_EINVAL, "bad bc");
  if (!std::isfinite(omega)) return set_err(HPFEM_EINVAL, "omega not finite");
  if (bc == HPFEM_BC_NEUMANN && omega == 0.0) return set_err(HPFEM_EINVAL, "Neumann requires omega != 0");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(HPFEM_ECUDA, "no CUDA device (no CPU fallback)");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  hpfem_plan1d_t pl = new hpfem_plan1d_s();
  pl->h = make_dir(xs, n, p, bc);
  pl->omega = omega;
  cudaError_t ce;
  auto fail = [&](cudaError_t e, const char* w) {
    free_plan1d(pl);
    return e == cudaErrorMemoryAllocation ? set_err(HPFEM_ENOMEM, std::string(w) + ": out of device memory")
                                          : cuda_err(e, w);
  };
  if ((ce = cudaMalloc(&pl->d_delta, sizeof(double) * n)) != cudaSuccess) return fail(ce, "alloc");
  if ((ce = cudaMemcpyAsync(pl->d_delta, pl->h.delta.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return fail(ce, "copy");
  DirDev& d = pl->d;
  d.n = n; d.p = p; d.bc = bc; d.nh = pl->h.nh; d.N = pl->h.N; d.nb = pl->h.nb; d.delta = pl->d_delta;
  const double ks[2] = {1.0, omega * omega};  // K + w^2 M
  if ((ce = cudaMalloc(&pl->d_ks, sizeof(ks))) != cudaSuccess) return fail(ce, "alloc");
  if ((ce = cudaMemcpyAsync(pl->d_ks, ks, sizeof(ks), cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return fail(ce, "copy");
  const size_t stride = fac_stride(d);
  if ((ce = cudaMalloc(&pl->fac, sizeof(double) * stride)) != cudaSuccess) return fail(ce, "alloc");
  if ((ce = cudaMemsetAsync(pl->fac, 0, sizeof(double) * stride, st)) != cudaSuccess) return fail(ce, "memset");
  if ((ce = cudaMalloc(&pl->d_err, sizeof(int) * 4)) != cudaSuccess) return fail(ce, "alloc");
  if ((ce = cudaMemsetAsync(pl->d_err, 0, sizeof(int) * 4, st)) != cudaSuccess) return fail(ce, "memset");
  if ((ce = launch_factor(d, pl->d_ks, pl->d_ks + 1, 1, pl->fac, stride, pl->d_err, st)) != cudaSuccess)
    return fail(ce, "factor");
  int herr[4];
  if ((ce = cudaMemcpyAsync(herr, pl->d_err, sizeof(herr), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return fail(ce, "copy err");
  if ((ce = cudaStreamSynchronize(st)) != cudaSuccess) return fail(ce, "sync");
  if (herr[0]) {
    free_plan1d(pl);
    return set_err(HPFEM_ENOTPD, "non-positive pivot in the 1D factorisation");
  }
  *out = pl;
  return HPFEM_OK;
}

int hpfem_plan1d_info(hpfem_plan1d_t pl, int* N) {
  if (!pl) return set_err(HPFEM_EINVAL, "null plan");
  if (N) *N = pl->h.N;
  return HPFEM_OK;
}

int hpfem_solve1d(hpfem_plan1d_t pl, int nrhs, const double* F, double* U, void* cuda_stream) {
  t_err.clear();
  if (!pl || !F || !U) return set_err(HPFEM_EINVAL, "null argument");
  if (nrhs < 0) return set_err(HPFEM_EINVAL, "nrhs < 0");
  if (overlap(F, U, sizeof(double) * (size_t)pl->h.N * nrhs)) return set_err(HPFEM_EINVAL, "F and U overlap");
  const FacView f = fac_view(pl->d, pl->fac, 1.0, pl->omega * pl->omega);
  const cudaError_t ce = launch_solve1d(pl->d, f, nrhs, F, U, (cudaStream_t)cuda_stream);
  return ce == cudaSuccess ? HPFEM_OK : cuda_err(ce, "solve1d");
}

void hpfem_plan1d_destroy(hpfem_plan1d_t pl) { free_plan1d(pl); }

int hpfem_plan_profile(hpfem_plan_t pl, int capacity) {
  if (!pl || capacity < 0) return set_err(HPFEM_EINVAL, "bad argument");
  free_events(pl);
  pl->ev.resize(capacity);
  for (int i = 0; i < capacity; ++i) {
    cudaError_t ce = cudaEventCreate(&pl->ev[i]);
    if (ce != cudaSuccess) {
      pl->ev.resize(i);
      free_events(pl);
      return cuda_err(ce, "event create");
    }
  }
  return HPFEM_OK;
}

int hpfem_plan_profile_read(hpfem_plan_t pl, double* ms, long long* n, double* bytes) {
  if (!pl || !ms || !n || !bytes) return set_err(HPFEM_EINVAL, "null argument");
  for (int k = 0; k < HPFEM_PROFILE_KINDS; ++k) {
    ms[k] = 0.0;
    n[k] = 0;
    bytes[k] = 0.0;
  }
  if (pl->ev_used > 0) {
    cudaError_t ce = cudaEventSynchronize(pl->ev[pl->ev_used - 1]);
    if (ce != cudaSuccess) return cuda_err(ce, "event sync");
  }
  for (const auto& r : pl->recs) {
    float t = 0.f;
    cudaError_t ce = cudaEventElapsedTime(&t, pl->ev[r.e0], pl->ev[r.e1]);
    if (ce != cudaSuccess) return cuda_err(ce, "event elapsed");
    ms[r.kind] += t;
    n[r.kind] += 1;
    bytes[r.kind] += r.bytes;
  }
  pl->recs.clear();
  pl->ev_used = 0;
  return HPFEM_OK;
}

void hpfem_plan_destroy(hpfem_plan_t pl) { free_plan(pl); }

}  // extern "C"
