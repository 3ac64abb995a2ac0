/*
 * hpfem_oracle.cpp -- plain, slow, obviously-correct CPU oracle for the ADI
 * hp-FEM screened-Poisson solve of arXiv 2402.11299 ("Optimal complexity
 * hp-FEM ... reverse Cholesky ... ADI").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2402_11299_b200/) shares no code with it and never
 * calls it.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (+ section /
 * equation / algorithm), "S:Lnnn" = SPEC.md line nnn.  Readings of silent or
 * garbled passages are listed in DESIGN.md "Readings"; they are marked
 * [READING Rn] below.
 *
 * Every step follows the paper's definitions in its order and notation:
 *   - element matrices  M_e = R_e^T M_P,e R_e   (App. A)
 *                       K_e = D_e^T M_P,e D_e   (App. A)
 *     assembled into the C basis and restricted to Q by dropping the
 *     boundary hats for Dirichlet;
 *   - reverse Cholesky A = L^T L by Algorithm 1 with the
 *     Schur complement of the Thm 4.2 proof [READING R3];
 *   - the O(N) solve of Corollary 4.3;
 *   - the spectral interval [READING R4], J and Zolotarev shifts
 *     [READING R5] in binary128;
 *   - Algorithm 2 literally, with A = A_x, D = M_x,
 *     B = -A_y, C = M_y (eq. adi:poisson P:L658-L666).
 * No blocking, fusion or reordering beyond those definitions.  Banded
 * factorisations use a generic banded reverse Cholesky (the definition
 * A = L^T L solved for L from the bottom-right), not the chain shortcut.
 *
 * Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC -lquadmath
 * OpenMP is used only across independent lines (rows / columns) of the
 * 2D arrays; it does not change any arithmetic.
 */
#include <omp.h>
#include <quadmath.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

/* ------------------------------------------------------------------ */
/* 1D space: mesh + degree + boundary condition */
/* ------------------------------------------------------------------ */
struct Space {
  int n = 0;               // elements
  int p = 0;               // max degree per element (bubbles W_0..W_{p-2})
  int bc = 0;              // 0 = zero Dirichlet (basis Q), 1 = zero Neumann (basis C),
                           // 2 = Dirichlet left / Neumann right, 3 = Neumann left / Dirichlet right
                           // (mixed: the hat keep/drop mask of P:L430-L435, NEXT-1 of SURVEY 8(f))
  std::vector<double> x;   // breakpoints x_0 < ... < x_n
  double rob[2] = {0.0, 0.0};  // Robin alpha at the left / right end (0 = none)

  // a Dirichlet end drops its boundary hat (Q drops h_0 and h_n; C keeps all)
  bool drop_left() const { return bc == 0 || bc == 2; }
  bool drop_right() const { return bc == 0 || bc == 3; }
  int nh() const { return n + 1 - (drop_left() ? 1 : 0) - (drop_right() ? 1 : 0); }
  // N = p n - 1 (Dirichlet) / p n + 1 (Neumann) / p n (mixed)
  int N() const { return nh() + (p - 1) * n; }
  // global index of the hat at node t (0..n), -1 if dropped; degree-major
  // ordering [H | W_0 | W_1 | ...] of P:L169-L171
  int hat(int node) const {
    if ((node == 0 && drop_left()) || (node == n && drop_right())) return -1;
    return node - (drop_left() ? 1 : 0);
  }
  int bub(int k, int e) const { return nh() + k * n + e; }
  double delta(int e) const { return x[e + 1] - x[e]; }
};

Space make_space(const double* xs, int n, int p, int bc, const double* rob = nullptr) {
  if (n < 1) throw std::invalid_argument("n < 1");
  if (p < 2) throw std::invalid_argument("p < 2");
  if (bc < 0 || bc > 3) throw std::invalid_argument("bc");
  Space s;
  s.n = n;
  s.p = p;
  s.bc = bc;
  s.x.assign(xs, xs + n + 1);
  for (int e = 0; e < n; ++e)
    if (!(s.x[e + 1] > s.x[e])) throw std::invalid_argument("breakpoints not increasing");
  if (rob) {
    for (int side = 0; side < 2; ++side) {
      if (!(rob[side] >= 0.0) || !std::isfinite(rob[side])) throw std::invalid_argument("Robin alpha < 0");
      if (rob[side] != 0.0 && (side == 0 ? s.drop_left() : s.drop_right()))
        throw std::invalid_argument("Robin alpha on a Dirichlet end");
      s.rob[side] = rob[side];
    }
  }
  return s;
}

/* Sparse symmetric matrix as rows of (col -> value). */
using SpRow = std::map<int, double>;
using SpMat = std::vector<SpRow>;

/* ------------------------------------------------------------------ */
/* Element matrices from the paper's definitions.                     */
/* Local basis order: [h_L, h_R, W_0, ..., W_{p-2}]  (size p+1)       */
/* Legendre modes P_0..P_p on the element.                            */
/* ------------------------------------------------------------------ */

/* Local connection R_e: column a = local basis fn, row m = Legendre mode.
 * App. A: h_0 = (1-x)/2 -> P_0/2 - P_1/2 ; h_1 = (1+x)/2 -> P_0/2 + P_1/2
 * (R_00, R_10 at P:L1084-L1096); W_k = (P_k - P_{k+2})/(2k+3) (eq. app:1,
 * P:L1074; the garbled "k = j +- 1" rule of P:L1100-L1106 is read through
 * app:1 [READING R1]). */
std::vector<double> local_R(int p) {
  const int nl = p + 1, nm = p + 1;
  std::vector<double> R(nm * nl, 0.0);
  auto at = [&](int m, int a) -> double& { return R[m * nl + a]; };
  at(0, 0) = 0.5;  at(1, 0) = -0.5;
  at(0, 1) = 0.5;  at(1, 1) = 0.5;
  for (int k = 0; k <= p - 2; ++k) {
    at(k, 2 + k) = 1.0 / (2 * k + 3);
    at(k + 2, 2 + k) = -1.0 / (2 * k + 3);
  }
  return R;
}

/* Local derivative D_e (maps local basis to Legendre coefficients of the
 * x-derivative), App. A: h_0' = -1/delta, h_1' = 1/delta
 * (on P_0), W_k' = -(2/delta) P_{k+1} (eq. deriv P:L84 + chain rule). */
std::vector<double> local_D(int p, double delta) {
  const int nl = p + 1, nm = p + 1;
  std::vector<double> D(nm * nl, 0.0);
  auto at = [&](int m, int a) -> double& { return D[m * nl + a]; };
  at(0, 0) = -1.0 / delta;
  at(0, 1) = 1.0 / delta;
  for (int k = 0; k <= p - 2; ++k) at(k + 1, 2 + k) = -2.0 / delta;
  return D;
}

/* Legendre mass on an element of width delta: (delta/2) * 2/(2m+1)
 * (P:L98 M_P, scaled per P:L201). */
std::vector<double> local_MP(int p, double delta) {
  std::vector<double> mp(p + 1);
  for (int m = 0; m <= p; ++m) mp[m] = (delta / 2.0) * (2.0 / (2 * m + 1));
  return mp;
}

/* E = X^T diag(mp) X for a (p+1)x(p+1) local map X (sum over Legendre
 * modes m in increasing order; zero entries of X are skipped). */
std::vector<double> gram(const std::vector<double>& X, const std::vector<double>& mp, int p) {
  const int nl = p + 1, nm = p + 1;
  std::vector<double> E(nl * nl, 0.0);
  std::vector<int> nz;
  for (int m = 0; m < nm; ++m) {
    nz.clear();
    for (int a = 0; a < nl; ++a)
      if (X[m * nl + a] != 0.0) nz.push_back(a);
    for (int a : nz)
      for (int b : nz) E[a * nl + b] += X[m * nl + a] * mp[m] * X[m * nl + b];
  }
  return E;
}

/* local index a -> global dof, -1 if dropped */
int local_to_global(const Space& s, int e, int a) {
  if (a == 0) return s.hat(e);
  if (a == 1) return s.hat(e + 1);
  return s.bub(a - 2, e);
}

/* Assemble the 1D mass M and stiffness -Delta. */
void assemble(const Space& s, SpMat& K, SpMat& M) {
  const int N = s.N(), nl = s.p + 1;
  K.assign(N, SpRow());
  M.assign(N, SpRow());
  const std::vector<double> R = local_R(s.p);
  for (int e = 0; e < s.n; ++e) {
    const double d = s.delta(e);
    const std::vector<double> mp = local_MP(s.p, d);
    const std::vector<double> Me = gram(R, mp, s.p);
    const std::vector<double> Ke = gram(local_D(s.p, d), mp, s.p);
    for (int a = 0; a < nl; ++a) {
      const int ga = local_to_global(s, e, a);
      if (ga < 0) continue;
      for (int b = 0; b < nl; ++b) {
        const int gb = local_to_global(s, e, b);
        if (gb < 0) continue;
        if (Me[a * nl + b] != 0.0) M[ga][gb] += Me[a * nl + b];
        if (Ke[a * nl + b] != 0.0) K[ga][gb] += Ke[a * nl + b];
      }
    }
  }
  // Robin ends: alpha <v, u>_{boundary} adds alpha h(x_end)^2 =
  // alpha to the diagonal of the end's (kept) hat; in 2D this is the
  // alpha <v,u>_{L2(side)} term of the tensor-product form
  if (s.rob[0] != 0.0) K[s.hat(0)][s.hat(0)] += s.rob[0];
  if (s.rob[1] != 0.0) K[s.hat(s.n)][s.hat(s.n)] += s.rob[1];
}

/* Entrywise combination X_ij = alpha * P_ij + beta * Q_ij over the union
 * pattern (the paper's "A - q_j D", "B - p_j C" written out). */
SpMat combine(double alpha, const SpMat& P, double beta, const SpMat& Q) {
  SpMat X(P.size());
  for (size_t i = 0; i < P.size(); ++i) {
    for (auto& kv : P[i]) X[i][kv.first] += alpha * kv.second;
    for (auto& kv : Q[i]) X[i][kv.first] += beta * kv.second;
  }
  return X;
}

double entry(const SpMat& A, int i, int j) {
  auto it = A[i].find(j);
  return it == A[i].end() ? 0.0 : it->second;
}

/* ------------------------------------------------------------------ */
/* Generic banded reverse Cholesky: A = L^T L, L lower, bandwidth w.   */
/* Solves the definition (L^T L)_{ij} = sum_{k >= max(i,j)} L_ki L_kj  */
/* for row j of L, from j = m-1 down to 0 (the "reverse" order)*/
/* Returns false on a non-positive / non-finite pivot.                 */
/* Storage: L[j*(w+1) + d] = L(j, j-d), d = 0..w.                      */
/* ------------------------------------------------------------------ */
template <class Get>
bool rev_chol_banded(int m, int w, Get A, std::vector<double>& L, int* bad) {
  L.assign((size_t)m * (w + 1), 0.0);
  auto Lat = [&](int r, int c) -> double {  // L(r, c), r >= c
    if (r < 0 || r >= m || c < 0 || r - c > w || r < c) return 0.0;
    return L[(size_t)r * (w + 1) + (r - c)];
  };
  for (int j = m - 1; j >= 0; --j) {
    double s = A(j, j);
    for (int k = j + 1; k <= std::min(m - 1, j + w); ++k) s -= Lat(k, j) * Lat(k, j);
    if (!(s > 0.0) || !std::isfinite(s)) {
      if (bad) *bad = j;
      return false;
    }
    const double ljj = std::sqrt(s);
    L[(size_t)j * (w + 1)] = ljj;
    for (int i = j - 1; i >= std::max(0, j - w); --i) {
      double t = A(j, i);
      for (int k = j + 1; k <= std::min(m - 1, i + w); ++k) t -= Lat(k, j) * Lat(k, i);
      L[(size_t)j * (w + 1) + (j - i)] = t / ljj;
    }
  }
  return true;
}

/* ------------------------------------------------------------------ */
/* Algorithm 1: reverse Cholesky of an SPD B^3-Arrowhead */
/* matrix A = [[A0, B],[B^T, D]], D = D_1 (+) ... (+) D_n.    */
/* Block bandwidth here: hats couple to bubble degree blocks 0 and 1  */
/* (ell = 2), bubble blocks couple k with k+-2 (sub-block bw 2).       */
/* ------------------------------------------------------------------ */
struct Factor {
  Space s;
  int ell = 2;                             // number of coupled degree blocks
  int wb = 2;                              // bandwidth of each D_e
  std::vector<std::vector<double>> Le;     // per element: banded L_e (p-1)x(p-1)
  std::vector<double> L0;                  // banded L0 (nh x nh), bandwidth 1
  // C block of L (rows: bubbles of degree k < ell, cols: hats):
  // C[(k,e), t] = (M_k)[t, e]; stored as Mk[k][t][e] sparse per element:
  // only hats adjacent to element e are nonzero (banded).
  std::vector<std::map<std::pair<int, int>, double>> Mk;  // Mk[k][(t,e)]
};

struct FactorError {
  int where;   // 0 = bubble block, 1 = hat Schur complement
  int elem;    // element (or hat row)
  int degree;  // bubble degree (or -1)
};

bool factor_b3(const Space& s, const SpMat& A, Factor& F, FactorError* err) {
  F.s = s;
  const int n = s.n, nb = s.p - 1, nh = s.nh();
  F.Le.assign(n, {});
  // Lines 1-3: banded reverse Cholesky of each D_k (here D_e per element)
  for (int e = 0; e < n; ++e) {
    auto get = [&](int k, int kk) { return entry(A, s.bub(k, e), s.bub(kk, e)); };
    int bad = -1;
    if (!rev_chol_banded(nb, F.wb, get, F.Le[e], &bad)) {
      if (err) *err = {0, e, bad};
      return false;
    }
  }
  // Lines 4-6: M_k = B_k Ltilde_{k,k} + ... + B_ell Ltilde_{ell,k}, with
  // Ltilde_{i,k} the (i,k) block of Ltilde^{-1} (diagonal over elements).
  // Ltilde^{-1} restricted to the first ell degree blocks is the inverse of
  // the leading ell x ell corner of each lower-triangular L_e.
  F.Mk.assign(F.ell, {});
  for (int e = 0; e < n; ++e) {
    const std::vector<double>& L = F.Le[e];
    const int w = F.wb;
    // inverse of the leading ell x ell lower-triangular corner of L_e
    const int c = std::min(F.ell, nb);
    std::vector<double> inv(F.ell * F.ell, 0.0);
    for (int col = 0; col < c; ++col) {
      // solve corner * z = e_col (forward substitution)
      for (int r = 0; r < c; ++r) {
        double t = (r == col) ? 1.0 : 0.0;
        for (int q = std::max(0, r - w); q < r; ++q) t -= L[(size_t)r * (w + 1) + (r - q)] * inv[q * F.ell + col];
        inv[r * F.ell + col] = t / L[(size_t)r * (w + 1)];
      }
    }
    for (int k = 0; k < c; ++k) {
      for (int node = e; node <= e + 1; ++node) {
        const int t = s.hat(node);
        if (t < 0) continue;
        double acc = 0.0;
        for (int i = k; i < c; ++i) acc += entry(A, t, s.bub(i, e)) * inv[i * F.ell + k];
        F.Mk[k][{t, e}] = acc;
      }
    }
  }
  // Line 7: Atilde_0 = A_0 - sum_k M_k M_k^T  (sign and A_0 term from the
  // Thm 4.2 proof; the listing at P:L576 omits them) [READING R3]
  std::vector<double> At(nh * 3, 0.0);  // tridiagonal: (t,t-1),(t,t),(t,t+1)
  auto Aget = [&](int t, int u) -> double& { return At[t * 3 + (u - t + 1)]; };
  for (int t = 0; t < nh; ++t)
    for (int u = std::max(0, t - 1); u <= std::min(nh - 1, t + 1); ++u) Aget(t, u) = entry(A, t, u);
  for (int k = 0; k < (int)F.Mk.size(); ++k) {
    for (int e = 0; e < n; ++e) {
      for (int n1 = e; n1 <= e + 1; ++n1) {
        const int t = s.hat(n1);
        if (t < 0) continue;
        for (int n2 = e; n2 <= e + 1; ++n2) {
          const int u = s.hat(n2);
          if (u < 0) continue;
          auto it1 = F.Mk[k].find({t, e});
          auto it2 = F.Mk[k].find({u, e});
          if (it1 == F.Mk[k].end() || it2 == F.Mk[k].end()) continue;
          Aget(t, u) -= it1->second * it2->second;
        }
      }
    }
  }
  // Line 8: banded reverse Cholesky of Atilde_0
  if (nh > 0) {
    auto get = [&](int t, int u) { return At[t * 3 + (u - t + 1)]; };
    int bad = -1;
    if (!rev_chol_banded(nh, 1, get, F.L0, &bad)) {
      if (err) *err = {1, bad, -1};
      return false;
    }
  } else {
    F.L0.clear();
  }
  return true;
}

/* Corollary 4.3: A x = f with A = L^T L,
 * L = [[L0, 0], [C, Ltilde]].  First L^T y = f, then L x = y. */
void solve_b3(const Factor& F, const double* f, double* xout) {
  const Space& s = F.s;
  const int n = s.n, nb = s.p - 1, nh = s.nh(), w = F.wb;
  std::vector<double> y(s.N());
  // L^T y = f, bottom block: Ltilde^T y_b = f_b (per element, upper
  // triangular, back substitution from the highest degree)
  for (int e = 0; e < n; ++e) {
    const std::vector<double>& L = F.Le[e];
    for (int k = nb - 1; k >= 0; --k) {
      double t = f[s.bub(k, e)];
      for (int r = k + 1; r <= std::min(nb - 1, k + w); ++r) t -= L[(size_t)r * (w + 1) + (r - k)] * y[s.bub(r, e)];
      y[s.bub(k, e)] = t / L[(size_t)k * (w + 1)];
    }
  }
  // top block: L0^T y_h = f_h - C^T y_b
  std::vector<double> rh(nh);
  for (int t = 0; t < nh; ++t) rh[t] = f[t];
  for (int k = 0; k < (int)F.Mk.size(); ++k)
    for (auto& kv : F.Mk[k]) rh[kv.first.first] -= kv.second * y[s.bub(k, kv.first.second)];
  for (int t = nh - 1; t >= 0; --t) {
    double v = rh[t];
    if (t + 1 < nh) v -= F.L0[(size_t)(t + 1) * 2 + 1] * y[t + 1];
    y[t] = v / F.L0[(size_t)t * 2];
  }
  // L x = y: top block L0 x_h = y_h (forward)
  std::vector<double> x(s.N());
  for (int t = 0; t < nh; ++t) {
    double v = y[t];
    if (t > 0) v -= F.L0[(size_t)t * 2 + 1] * x[t - 1];
    x[t] = v / F.L0[(size_t)t * 2];
  }
  // bottom block: Ltilde x_b = y_b - C x_h
  std::vector<double> rb(y.begin() + nh, y.end());
  for (int k = 0; k < (int)F.Mk.size(); ++k)
    for (auto& kv : F.Mk[k]) rb[k * n + kv.first.second] -= kv.second * x[kv.first.first];
  for (int e = 0; e < n; ++e) {
    const std::vector<double>& L = F.Le[e];
    for (int k = 0; k < nb; ++k) {
      double t = rb[k * n + e];
      for (int q = std::max(0, k - w); q < k; ++q) t -= L[(size_t)k * (w + 1) + (k - q)] * x[s.bub(q, e)];
      x[s.bub(k, e)] = t / L[(size_t)k * (w + 1)];
    }
  }
  std::memcpy(xout, x.data(), sizeof(double) * s.N());
}

/* ------------------------------------------------------------------ */
/* Spectral interval [READING R4]                                      */
/* lambda_min: Dirichlet pi^2/(b-a)^2 + w^2/2 (Poincare)  */
/*             Neumann  w^2/2 (constants in the space)         */
/* lambda_max: bisection on "sigma M - A is SPD", the SPD test being   */
/*             Algorithm 1 itself (P:L887-L889 inverse-iteration remark)*/
/* ------------------------------------------------------------------ */
struct Ops1D {
  Space s;
  SpMat K, M, A;  // stiffness, mass, A = K + (w^2/2) M
};

Ops1D make_ops(const Space& s, double omega) {
  Ops1D o;
  o.s = s;
  assemble(s, o.K, o.M);
  o.A = combine(1.0, o.K, omega * omega / 2.0, o.M);
  return o;
}

bool is_spd(const Ops1D& o, double sigma) {
  SpMat S = combine(sigma, o.M, -1.0, o.A);  // sigma M - A
  Factor F;
  return factor_b3(o.s, S, F, nullptr);
}

/* A - sigma M SPD  <=>  sigma < lambda_min (Robin ends, reading R22) */
bool is_spd_low(const Ops1D& o, double sigma) {
  SpMat S = combine(1.0, o.A, -sigma, o.M);
  Factor F;
  return factor_b3(o.s, S, F, nullptr);
}

void spectrum(const Ops1D& o, double omega, double lam[2]) {
  const Space& s = o.s;
  const double pi = 3.14159265358979323846;
  const double L = s.x[s.n] - s.x[0];
  // closed-form lower bounds of the continuous spectrum (reading R4): Dirichlet
  // pi^2/L^2, Neumann 0, mixed Dirichlet/Neumann pi^2/(4 L^2) (quarter wave)
  lam[0] = (s.bc == 0 ? pi * pi / (L * L) : s.bc == 1 ? 0.0 : pi * pi / (4.0 * L * L)) + omega * omega / 2.0;
  if (s.rob[0] != 0.0 || s.rob[1] != 0.0) {
    // Robin ends (reading R22): no closed form; bisection on "A - sigma M is
    // SPD" from the valid lower bound w^2/2 (K + alpha terms is PSD), keeping
    // the SPD-confirmed lower end
    double lo = omega * omega / 2.0, hi = std::max(2.0 * lo, 1.0);
    int g = 0;
    while (is_spd_low(o, hi) && g++ < 200) {
      lo = hi;
      hi *= 2.0;
    }
    while (hi - lo > 1e-13 * hi) {
      const double mid = 0.5 * (lo + hi);
      if (is_spd_low(o, mid)) lo = mid; else hi = mid;
    }
    lam[0] = lo;
  }
  // initial upper bracket: Lemma 5.2, lambda^{-1} <= (24p^4 + w^2 h^2)/(2h^2)
  double h = s.delta(0);
  for (int e = 1; e < s.n; ++e) h = std::min(h, s.delta(e));
  const double p4 = (double)s.p * s.p * s.p * s.p;
  if (s.N() == 1) {  // a single dof: the eigenvalue is A/M exactly
    lam[0] = lam[1] = entry(o.A, 0, 0) / entry(o.M, 0, 0);
    return;
  }
  double hi = (24.0 * p4 + omega * omega * h * h) / (2.0 * h * h);
  hi = std::max(hi, 2.0 * lam[0]);
  int guard = 0;
  while (!is_spd(o, hi) && guard++ < 200) hi *= 2.0;
  double lo = lam[0];
  while (hi - lo > 1e-13 * hi) {
    const double mid = 0.5 * (lo + hi);
    if (is_spd(o, mid)) hi = mid; else lo = mid;
  }
  lam[1] = hi;
}

/* ------------------------------------------------------------------ */
/* J and Zolotarev shifts in binary128 [READING R5]                    */
/* J = ceil(log(16 gamma) log(4/eps)/pi^2)                     */
/* ------------------------------------------------------------------ */
typedef __float128 q128;

q128 agm(q128 a, q128 b) {
  for (int i = 0; i < 200; ++i) {
    const q128 an = (a + b) / 2, bn = sqrtq(a * b);
    a = an;
    b = bn;
    if (fabsq(a - b) <= 1e-33Q * a) break;
  }
  return (a + b) / 2;
}

/* dn(u, k) by the descending Landen / AGM scheme (A&S 16.4), valid for
 * u <= K/2 (where cos(phi_0) has no cancellation); kp = k' = sqrt(1-k^2). */
q128 dn_landen(q128 u, q128 kp) {
  const q128 k = sqrtq((1 - kp) * (1 + kp));
  if (k == 0) return 1;
  q128 a[128], c[128];
  q128 aa = 1, bb = kp, cc = k;
  int Nn = 0;
  a[0] = aa;
  c[0] = cc;
  while (fabsq(cc) > 1e-34Q * aa && Nn < 120) {
    const q128 an = (aa + bb) / 2, bn = sqrtq(aa * bb), cn = (aa - bb) / 2;
    aa = an; bb = bn; cc = cn;
    ++Nn;
    a[Nn] = aa;
    c[Nn] = cc;
  }
  q128 phi = ldexpq(1, Nn) * a[Nn] * u;
  q128 phi_prev = phi;
  for (int i = Nn; i >= 1; --i) {
    phi_prev = phi;
    phi = (phi + asinq(c[i] * sinq(phi) / a[i])) / 2;
  }
  // phi = phi_0, phi_prev = phi_1
  if (Nn == 0) return 1;
  return cosq(phi) / cosq(phi_prev - phi);
}

/* dn(u, k) for k' < 1e-8 (k near 1): A&S 16.15.3,
 *   dn(u|m) = sech u + (m1/4)(sinh u cosh u + u) tanh u sech u + O(m1^2 e^{4u}),
 * m1 = k'^2.  For u <= K/2 (e^{2u} <= 4/k') the dropped term is O(k'^2)
 * relative, below binary128 rounding for k' < 1e-8, whereas the Landen
 * recurrence loses ~eps/k' there (measured 1e-7 at k' = 2e-28). */
q128 dn_near1(q128 u, q128 kp) {
  const q128 m1 = kp * kp;
  const q128 ch = coshq(u), sh = sinhq(u);
  const q128 sech = 1 / ch, th = sh / ch;
  return sech + m1 / 4 * (sh * ch + u) * th * sech;
}

q128 dn_q(q128 u, q128 K, q128 kp) {
  if (u > K / 2) return kp / dn_q(K - u, K, kp);  // dn(K-u) dn(u) = k'
  if (kp < 1e-8Q) return dn_near1(u, kp);
  return dn_landen(u, kp);
}

int shifts(double a, double b, double c, double d, double eps, int maxJ, int* Jout, double* gamma_out,
           double* P, double* Qs) {
  const q128 qa = a, qb = b, qc = c, qd = d;
  const q128 gam = fabsq(qc - qa) * fabsq(qd - qb) / (fabsq(qc - qb) * fabsq(qd - qa));
  const q128 pi = M_PIq;
  const q128 Jr = logq(16 * gam) * logq(4 / (q128)eps) / (pi * pi);
  int J = (int)ceilq(Jr);
  if (J < 1) J = 1;
  *Jout = J;
  *gamma_out = (double)gam;
  if (J > maxJ) return -1;
  const q128 alpha = -1 + 2 * gam + 2 * sqrtq(gam * gam - gam);
  const q128 kp = 1 / alpha;
  const q128 K = pi / (2 * agm(1, kp));
  const bool symmetric = (c == -b) && (d == -a);
  // [READING R15] exactly one interval is a single point (N = 1 in that
  // direction): alpha = 1 and the Moebius map through (-alpha, -1, 1)
  // degenerates.  r(z) = (z - p)/(z - q) with p (or q) at that point is
  // exactly 0 there, so the contraction factor max|r| max|1/r| of the ADI
  // error is 0; the other shift is taken inside its own interval
  // (geometric mean), keeping both shifted matrices definite.
  const bool pt_ab = (a == b), pt_cd = (c == d);
  for (int j = 1; j <= J; ++j) {
    const q128 u = (2 * j - 1) * K / (2 * (q128)J);
    const q128 dn = dn_q(u, K, kp);
    if (pt_ab && !pt_cd) {
      P[j - 1] = a;
      Qs[j - 1] = -(double)sqrtq(qc * qd);
    } else if (pt_cd && !pt_ab) {
      P[j - 1] = (double)sqrtq(qa * qb);
      Qs[j - 1] = c;
    } else if (symmetric) {
      // T(z) = -b/z maps (-alpha,-1,1,alpha) -> (a,b,-b,-a) since alpha = b/a
      P[j - 1] = (double)(qa / dn);
      Qs[j - 1] = (double)(-(qa / dn));
    } else {
      // Moebius T with T(-alpha)=a, T(-1)=b, T(1)=c via the cross ratio
      auto T = [&](q128 z) -> q128 {
        const q128 rho = (z + alpha) * (-2) / ((z - 1) * (alpha - 1));
        return (qa * (qb - qc) - rho * qc * (qb - qa)) / ((qb - qc) - rho * (qb - qa));
      };
      P[j - 1] = (double)T(-alpha * dn);
      Qs[j - 1] = (double)T(alpha * dn);
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* 2D helpers on row-major Nx x Ny arrays                              */
/* ------------------------------------------------------------------ */
/* Y = S X (left multiply, mixes rows) */
void left_mult(const SpMat& S, const double* X, double* Y, int Nx, int Ny) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < Nx; ++i) {
    double* yi = Y + (size_t)i * Ny;
    for (int j = 0; j < Ny; ++j) yi[j] = 0.0;
    for (auto& kv : S[i]) {
      const double* xr = X + (size_t)kv.first * Ny;
      for (int j = 0; j < Ny; ++j) yi[j] += kv.second * xr[j];
    }
  }
}
/* Y = X S (right multiply, mixes columns) */
void right_mult(const SpMat& S, const double* X, double* Y, int Nx, int Ny) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < Nx; ++i) {
    const double* xi = X + (size_t)i * Ny;
    double* yi = Y + (size_t)i * Ny;
    for (int j = 0; j < Ny; ++j) {
      double acc = 0.0;
      for (auto& kv : S[j]) acc += xi[kv.first] * kv.second;  // S symmetric: S[j'][j] = S[j][j']
      yi[j] = acc;
    }
  }
}
/* Y = S^{-1} X (column-wise 1D solves), sign = +1/-1 multiplies result */
void left_solve(const Factor& F, const double* X, double* Y, int Nx, int Ny, double sign) {
#pragma omp parallel
  {
    std::vector<double> col(Nx), out(Nx);
#pragma omp for schedule(static)
    for (int j = 0; j < Ny; ++j) {
      for (int i = 0; i < Nx; ++i) col[i] = X[(size_t)i * Ny + j];
      solve_b3(F, col.data(), out.data());
      for (int i = 0; i < Nx; ++i) Y[(size_t)i * Ny + j] = sign * out[i];
    }
  }
}
/* Y = X S^{-1} (row-wise solves; S symmetric, S^{-T} = S^{-1}) */
void right_solve(const Factor& F, const double* X, double* Y, int Nx, int Ny, double sign) {
#pragma omp parallel
  {
    std::vector<double> out(Ny);
#pragma omp for schedule(static)
    for (int i = 0; i < Nx; ++i) {
      solve_b3(F, X + (size_t)i * Ny, out.data());
      for (int j = 0; j < Ny; ++j) Y[(size_t)i * Ny + j] = sign * out[j];
    }
  }
}

thread_local std::string g_err;

int fail(const std::string& msg, int code) {
  g_err = msg;
  return code;
}

struct Problem {
  Ops1D ox, oy;
  double omega, tol;
};

/* 2D boundary code: 0..3 = the same 1D code in both directions; 16 + bx + 4 by
 * = per direction (bx, by in 0..3) */
void split_bc(int bc, int& bx, int& by) {
  if (bc >= 16) {
    bx = (bc - 16) & 3;
    by = ((bc - 16) >> 2) & 3;
  } else {
    bx = by = bc;
  }
}

/* Robin alphas (x-left, x-right, y-left, y-right) of the next calls
 * (oracle_set_robin; zeros = none) */
double g_robin[4] = {0.0, 0.0, 0.0, 0.0};

int make_problem(const double* xs, int nx, int px, const double* ys, int ny, int py, double omega, int bc,
                 double tol, Problem& P) {
  int bx, by;
  split_bc(bc, bx, by);
  const bool sx = bx == 1 && g_robin[0] == 0.0 && g_robin[1] == 0.0;  // pure Neumann: singular K
  const bool sy = by == 1 && g_robin[2] == 0.0 && g_robin[3] == 0.0;
  if ((sx || sy) && omega == 0.0) throw std::invalid_argument("Neumann requires omega != 0 (P:L812)");
  if (!(tol > 0.0 && tol < 1.0)) throw std::invalid_argument("tol not in (0,1)");
  P.ox = make_ops(make_space(xs, nx, px, bx, g_robin), omega);
  P.oy = make_ops(make_space(ys, ny, py, by, g_robin + 2), omega);
  P.omega = omega;
  P.tol = tol;
  return 0;
}

}  // namespace

/* ==================================================================== */
/* C ABI of the oracle (test infrastructure)                            */
/* ==================================================================== */
extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

/* Robin coefficients alpha >= 0 at (x = a, x = b, y = c, y = d) for the
 * following calls (alpha u + du/dn = 0); all zero = none.  The
 * 1D functions use the first two. */
void oracle_set_robin(const double* alpha4) {
  for (int k = 0; k < 4; ++k) g_robin[k] = alpha4 ? alpha4[k] : 0.0;
}

/* OpenMP threads the oracle's line loops use (bench.py cpu_baseline.cores) */
int oracle_threads(void) { return omp_get_max_threads(); }

/* Set the OpenMP thread count of the line loops (n <= 0: the default, all
 * host cores).  Test / baseline infrastructure only: bench.py times a
 * single-threaded sample next to the all-core run. */
void oracle_set_threads(int n) {
  static const int dflt = omp_get_max_threads();
  omp_set_num_threads(n > 0 ? n : dflt);
}

/* N of the 1D space */
int oracle_dim(int n, int p, int bc) {
  const int nh = n + 1 - ((bc == 0 || bc == 2) ? 1 : 0) - ((bc == 0 || bc == 3) ? 1 : 0);
  return nh + (p - 1) * n;
}

/* Dense alpha*K + beta*M (N x N, row-major) for tests on small N. */
int oracle_operator_dense(const double* xs, int n, int p, int bc, double alpha, double beta, double* out) {
  try {
    Space s = make_space(xs, n, p, bc, g_robin);
    SpMat K, M;
    assemble(s, K, M);
    SpMat S = combine(alpha, K, beta, M);
    const int N = s.N();
    std::memset(out, 0, sizeof(double) * N * N);
    for (int i = 0; i < N; ++i)
      for (auto& kv : S[i]) out[(size_t)i * N + kv.first] = kv.second;
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* Sparse (COO) K and M; returns nnz via *nnz when rows==NULL. */
int oracle_operator_coo(const double* xs, int n, int p, int bc, int which, int* rows, int* cols, double* vals,
                        int* nnz) {
  try {
    Space s = make_space(xs, n, p, bc, g_robin);
    SpMat K, M;
    assemble(s, K, M);
    const SpMat& S = which == 0 ? K : M;
    int c = 0;
    for (int i = 0; i < s.N(); ++i)
      for (auto& kv : S[i]) {
        if (rows) {
          rows[c] = i;
          cols[c] = kv.first;
          vals[c] = kv.second;
        }
        ++c;
      }
    *nnz = c;
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* Dense reverse-Cholesky factor L of S = alpha K + beta M (Alg. 1).
 * Returns -2 (ENOTPD) with info[0..2] = (where, elem, degree). */
int oracle_factor_dense(const double* xs, int n, int p, int bc, double alpha, double beta, double* Lout,
                        int* info) {
  try {
    Space s = make_space(xs, n, p, bc, g_robin);
    SpMat K, M;
    assemble(s, K, M);
    SpMat S = combine(alpha, K, beta, M);
    Factor F;
    FactorError err{-1, -1, -1};
    if (!factor_b3(s, S, F, &err)) {
      if (info) { info[0] = err.where; info[1] = err.elem; info[2] = err.degree; }
      return fail("not positive definite", -2);
    }
    const int N = s.N(), nh = s.nh(), nb = p - 1, w = F.wb;
    std::memset(Lout, 0, sizeof(double) * N * N);
    for (int t = 0; t < nh; ++t) {
      Lout[(size_t)t * N + t] = F.L0[(size_t)t * 2];
      if (t > 0) Lout[(size_t)t * N + t - 1] = F.L0[(size_t)t * 2 + 1];
    }
    for (int k = 0; k < (int)F.Mk.size(); ++k)
      for (auto& kv : F.Mk[k]) Lout[(size_t)s.bub(k, kv.first.second) * N + kv.first.first] = kv.second;
    for (int e = 0; e < n; ++e)
      for (int k = 0; k < nb; ++k)
        for (int d = 0; d <= std::min(w, k); ++d)
          Lout[(size_t)s.bub(k, e) * N + s.bub(k - d, e)] = F.Le[e][(size_t)k * (w + 1) + d];
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* x = (alpha K + beta M)^{-1} f via Alg. 1 + Cor. 4.3; nrhs vectors of length N. */
int oracle_solve1d(const double* xs, int n, int p, int bc, double alpha, double beta, const double* f, double* x,
                   int nrhs) {
  try {
    Space s = make_space(xs, n, p, bc, g_robin);
    SpMat K, M;
    assemble(s, K, M);
    SpMat S = combine(alpha, K, beta, M);
    Factor F;
    if (!factor_b3(s, S, F, nullptr)) return fail("not positive definite", -2);
    for (int r = 0; r < nrhs; ++r) solve_b3(F, f + (size_t)r * s.N(), x + (size_t)r * s.N());
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* [lambda_min, lambda_max] of the pencil (A, M), A = K + (w^2/2) M. */
int oracle_spectrum(const double* xs, int n, int p, int bc, double omega, double* lam) {
  try {
    Space s = make_space(xs, n, p, bc, g_robin);
    if (bc == 1 && omega == 0.0 && g_robin[0] == 0.0 && g_robin[1] == 0.0)
      return fail("Neumann requires omega != 0", -1);  // (mixed and Robin ends are definite)
    Ops1D o = make_ops(s, omega);
    spectrum(o, omega, lam);
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* J, gamma and Zolotarev shifts for [a,b], [c,d]. */
int oracle_shifts(double a, double b, double c, double d, double eps, int maxJ, int* J, double* gamma, double* P,
                  double* Q) {
  if (!(a <= b && c <= d && (b < c || d < a))) return fail("intervals must be ordered and disjoint", -1);
  return shifts(a, b, c, d, eps, maxJ, J, gamma, P, Q) == 0 ? 0 : fail("J > maxJ", -1);
}

/* Plan summary: N_x, N_y, J, lam_x[2], lam_y[2], gamma, shifts p,q (maxJ). */
int oracle_plan(const double* xs, int nx, int px, const double* ys, int ny, int py, double omega, int bc,
                double tol, int maxJ, int* dims /*Nx,Ny,J*/, double* lamx, double* lamy, double* gamma, double* P,
                double* Q) {
  try {
    Problem pr;
    make_problem(xs, nx, px, ys, ny, py, omega, bc, tol, pr);
    spectrum(pr.ox, omega, lamx);
    spectrum(pr.oy, omega, lamy);
    int J = 0;
    // [a,b] = sigma(A, D) = sigma(A_x, M_x);  [c,d] = sigma(B, C) = -sigma(A_y, M_y)
    if (shifts(lamx[0], lamx[1], -lamy[1], -lamy[0], tol, maxJ, &J, gamma, P, Q) != 0)
      return fail("J > maxJ", -1);
    dims[0] = pr.ox.s.N();
    dims[1] = pr.oy.s.N();
    dims[2] = J;
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* Algorithm 2 literally.  G: Nx x Ny row-major (the
 * right-hand side F of Alg. 2, i.e. G of eq. adi:poisson).  iters < 0
 * runs all J iterations; 0 <= iters < J runs the first `iters` (used by
 * the truncated full-size parity tests).  Output U = W_iters C^{-1}. */
int oracle_adi_solve(const double* xs, int nx, int px, const double* ys, int ny, int py, double omega, int bc,
                     double tol, const double* G, double* U, int iters, int* Jout) {
  try {
    Problem pr;
    make_problem(xs, nx, px, ys, ny, py, omega, bc, tol, pr);
    double lamx[2], lamy[2], gamma;
    spectrum(pr.ox, omega, lamx);
    spectrum(pr.oy, omega, lamy);
    const int maxJ = 4096;
    std::vector<double> P(maxJ), Q(maxJ);
    int J = 0;
    if (shifts(lamx[0], lamx[1], -lamy[1], -lamy[0], tol, maxJ, &J, &gamma, P.data(), Q.data()) != 0)
      return fail("J > maxJ", -1);
    if (Jout) *Jout = J;
    const int run = (iters < 0 || iters > J) ? J : iters;
    const int Nx = pr.ox.s.N(), Ny = pr.oy.s.N();
    // Alg. 2 inputs (eq. adi:poisson): A = A_x, D = M_x, B = -A_y, C = M_y
    const SpMat& A = pr.ox.A;
    const SpMat& D = pr.ox.M;
    const SpMat B = combine(-1.0, pr.oy.A, 0.0, pr.oy.M);
    const SpMat& C = pr.oy.M;
    // C = L^T L for the final W_J C^{-1}
    Factor FC;
    if (!factor_b3(pr.oy.s, C, FC, nullptr)) return fail("mass not positive definite", -2);
    const size_t NN = (size_t)Nx * Ny;
    std::vector<double> W(NN, 0.0), Wh(NN), T(NN);
    for (int j = 0; j < run; ++j) {
      const double pj = P[j], qj = Q[j];
      // precomputation lines 4-6: factorisations of A - q_j D and B - p_j C
      // (the latter is negative definite: factor -(B - p_j C)).
      const SpMat AmqD = combine(1.0, A, -qj, D);
      const SpMat BmpC = combine(1.0, B, -pj, C);
      const SpMat negBmpC = combine(-1.0, BmpC, 0.0, C);
      Factor Fx, Fy;
      if (!factor_b3(pr.ox.s, AmqD, Fx, nullptr)) return fail("A - q_j D not positive definite", -2);
      if (!factor_b3(pr.oy.s, negBmpC, Fy, nullptr)) return fail("-(B - p_j C) not positive definite", -2);
      // W_{j-1/2} = (F - (A - p_j D) W_{j-1}) (B - p_j C)^{-1}
      const SpMat AmpD = combine(1.0, A, -pj, D);
      left_mult(AmpD, W.data(), T.data(), Nx, Ny);
#pragma omp parallel for schedule(static)
      for (long long t = 0; t < (long long)NN; ++t) T[t] = G[t] - T[t];
      right_solve(Fy, T.data(), Wh.data(), Nx, Ny, -1.0);
      // W_j = (A - q_j D)^{-1} (F - W_{j-1/2} (B - q_j C))
      const SpMat BmqC = combine(1.0, B, -qj, C);
      right_mult(BmqC, Wh.data(), T.data(), Nx, Ny);
#pragma omp parallel for schedule(static)
      for (long long t = 0; t < (long long)NN; ++t) T[t] = G[t] - T[t];
      left_solve(Fx, T.data(), W.data(), Nx, Ny, 1.0);
    }
    // RETURN W_J C^{-1}
    right_solve(FC, W.data(), U, Nx, Ny, 1.0);
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* F = A U C - D U B = A_x U M_y + M_x U A_y (the Sylvester operator of
 * eq. adi:poisson). */
int oracle_apply(const double* xs, int nx, int px, const double* ys, int ny, int py, double omega, int bc,
                 const double* U, double* F) {
  try {
    Problem pr;
    make_problem(xs, nx, px, ys, ny, py, omega, bc, 0.5, pr);
    const int Nx = pr.ox.s.N(), Ny = pr.oy.s.N();
    const size_t NN = (size_t)Nx * Ny;
    std::vector<double> T1(NN), T2(NN);
    right_mult(pr.oy.M, U, T1.data(), Nx, Ny);      // U C
    left_mult(pr.ox.A, T1.data(), F, Nx, Ny);        // A U C
    right_mult(pr.oy.A, U, T1.data(), Nx, Ny);      // U A_y = -U B
    left_mult(pr.ox.M, T1.data(), T2.data(), Nx, Ny);  // D U A_y
#pragma omp parallel for schedule(static)
    for (long long t = 0; t < (long long)NN; ++t) F[t] += T2[t];
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* G = R_x^T M_{P,x} F_leg M_{P,y} R_y.  F_leg is
 * ((px+1) nx) x ((py+1) ny) row-major, degree-major / element-minor:
 * row index m*nx + e for Legendre degree m on x-element e. */
int oracle_load(const double* xs, int nx, int px, const double* ys, int ny, int py, int bc, const double* Fleg,
                double* G) {
  try {
    int bx, by;
    split_bc(bc, bx, by);
    Space sx = make_space(xs, nx, px, bx), sy = make_space(ys, ny, py, by);
    const std::vector<double> R_x = local_R(px), R_y = local_R(py);
    // global sparse Z = M_P R as rows (Legendre index) -> (dof, value)
    auto build = [](const Space& s, const std::vector<double>& Rl) {
      std::vector<std::vector<std::pair<int, double>>> Z((size_t)(s.p + 1) * s.n);
      const int nl = s.p + 1;
      for (int e = 0; e < s.n; ++e) {
        const std::vector<double> mp = local_MP(s.p, s.delta(e));
        for (int m = 0; m <= s.p; ++m)
          for (int a = 0; a < nl; ++a) {
            const double r = Rl[m * nl + a];
            if (r == 0.0) continue;
            const int g = local_to_global(s, e, a);
            if (g < 0) continue;
            Z[(size_t)m * s.n + e].push_back({g, mp[m] * r});
          }
      }
      return Z;
    };
    auto Zx = build(sx, R_x), Zy = build(sy, R_y);
    const int Lx = (px + 1) * nx, Ly = (py + 1) * ny, Nx = sx.N(), Ny = sy.N();
    std::vector<double> T((size_t)Lx * Ny, 0.0);  // F_leg M_P,y R_y
#pragma omp parallel for schedule(static)
    for (int r = 0; r < Lx; ++r)
      for (int c = 0; c < Ly; ++c) {
        const double f = Fleg[(size_t)r * Ly + c];
        for (auto& gv : Zy[c]) T[(size_t)r * Ny + gv.first] += f * gv.second;
      }
    std::memset(G, 0, sizeof(double) * (size_t)Nx * Ny);
    // G = (M_P,x R_x)^T T, parallel over columns to keep writes private
#pragma omp parallel for schedule(static)
    for (int j = 0; j < Ny; ++j)
      for (int r = 0; r < Lx; ++r) {
        const double t = T[(size_t)r * Ny + j];
        for (auto& gv : Zx[r]) G[(size_t)gv.first * Ny + j] += gv.second * t;
      }
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

/* Unload (NEXT-1; the coefficient map behind P:L392-L399):
 * the piecewise-Legendre coefficients of the FEM function u = sum U_ij
 * phi_i(x) psi_j(y),  C_leg = R_x U R_y^T, with R the same element-local
 * basis -> Legendre change of basis as in oracle_load (hats (1 -+ t)/2,
 * W_k = (P_k - P_{k+2})/(2k+3), eq. app:1 P:L1074) and no mass weight.
 * U: Nx x Ny; C_leg: ((px+1) nx) x ((py+1) ny), degree-major as F_leg. */
int oracle_unload(const double* xs, int nx, int px, const double* ys, int ny, int py, int bc, const double* U,
                  double* Cleg) {
  try {
    int bx, by;
    split_bc(bc, bx, by);
    Space sx = make_space(xs, nx, px, bx), sy = make_space(ys, ny, py, by);
    const std::vector<double> R_x = local_R(px), R_y = local_R(py);
    // global sparse R as rows (Legendre index) -> (dof, value)
    auto build = [](const Space& s, const std::vector<double>& Rl) {
      std::vector<std::vector<std::pair<int, double>>> Z((size_t)(s.p + 1) * s.n);
      const int nl = s.p + 1;
      for (int e = 0; e < s.n; ++e)
        for (int m = 0; m <= s.p; ++m)
          for (int a = 0; a < nl; ++a) {
            const double r = Rl[m * nl + a];
            if (r == 0.0) continue;
            const int g = local_to_global(s, e, a);
            if (g < 0) continue;
            Z[(size_t)m * s.n + e].push_back({g, r});
          }
      return Z;
    };
    auto Zx = build(sx, R_x), Zy = build(sy, R_y);
    const int Lx = (px + 1) * nx, Ly = (py + 1) * ny, Ny = sy.N();
    std::vector<double> T((size_t)Lx * Ny, 0.0);  // R_x U
#pragma omp parallel for schedule(static)
    for (int r = 0; r < Lx; ++r)
      for (auto& gv : Zx[r])
        for (int j = 0; j < Ny; ++j) T[(size_t)r * Ny + j] += gv.second * U[(size_t)gv.first * Ny + j];
    // C_leg = T R_y^T
#pragma omp parallel for schedule(static)
    for (int r = 0; r < Lx; ++r)
      for (int c = 0; c < Ly; ++c) {
        double acc = 0.0;
        for (auto& gv : Zy[c]) acc += T[(size_t)r * Ny + gv.first] * gv.second;
        Cleg[(size_t)r * Ly + c] = acc;
      }
    return 0;
  } catch (std::exception& ex) {
    return fail(ex.what(), -1);
  }
}

}  // extern "C"
