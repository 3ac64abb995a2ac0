/*
 * ops1d.h -- closed-form entries of the 1D hp-FEM operators, shared by the
 * host plan (plan.cpp) and the device kernels (kernels.cu).
 *
 * Per element of width delta, local functions h_L, h_R, W_0..W_{p-2}
 * (P:L138-L184).  Derived from App. A:
 *   W_k = (P_k - P_{k+2})/(2k+3)  (eq. app:1),  W_k' = -P_{k+1}  (eq. deriv),
 *   ||P_m||^2 = 2/(2m+1), hats (1 -+ t)/2, dx = delta/2 dt:
 *
 *   K = -Delta:  hat block (1/delta)[[1,-1],[-1,1]];  W_k,W_k: 4/(delta(2k+3));
 *                no hat-bubble and no bubble-bubble off-diagonal terms.
 *   M:           hat block (delta/6)[[2,1],[1,2]];
 *                <h_{L,R}, W_0> = delta/6; <h_L, W_1> = -delta/30, <h_R, W_1> = +delta/30;
 *                <W_k,W_k> = delta (1/(2k+1) + 1/(2k+5)) / (2k+3)^2;
 *                <W_k,W_{k+2}> = -delta / ((2k+3)(2k+5)(2k+7));  odd offsets 0.
 *
 * A shifted operator is S = kap K + sig M (kap in {1, 0, -1}).  These are
 * NOT the oracle's formulas (the oracle forms R^T M_P R and D^T M_P D); the
 * two agree to rounding (tests/test_gpu_parity.py).
 */
#ifndef HPFEM_OPS1D_H_
#define HPFEM_OPS1D_H_

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace hpfem {

/* bubble diagonal S(W_k, W_k) */
HD double s_bub_diag(double kap, double sig, double delta, int k) {
  const double t = 2.0 * k + 3.0;
  const double m = delta * (1.0 / (2.0 * k + 1.0) + 1.0 / (2.0 * k + 5.0)) / (t * t);
  return kap * (4.0 / (delta * t)) + sig * m;
}

/* bubble coupling S(W_k, W_{k+2}) */
HD double s_bub_off(double sig, double delta, int k) {
  return sig * (-delta / ((2.0 * k + 3.0) * (2.0 * k + 5.0) * (2.0 * k + 7.0)));
}

/* hat-bubble coupling S(h_side, W_k) for k in {0,1} (0 for k >= 2);
 * side 0 = left hat of the element, 1 = right hat */
HD double s_hat_bub(double sig, double delta, int side, int k) {
  if (k == 0) return sig * (delta / 6.0);
  if (k == 1) return side == 0 ? sig * (-delta / 30.0) : sig * (delta / 30.0);
  return 0.0;
}

/* element contribution to a hat diagonal S(h,h) and to S(h_L, h_R) */
HD double s_hat_diag_elem(double kap, double sig, double delta) { return kap / delta + sig * (delta / 3.0); }
HD double s_hat_off_elem(double kap, double sig, double delta) { return -kap / delta + sig * (delta / 6.0); }

/* index helpers (degree-major / element-minor ordering) */
/* 1D boundary codes: 0 Dirichlet both ends, 1 Neumann both ends, 2 Dirichlet
 * left / Neumann right, 3 Neumann left / Dirichlet right.  A Dirichlet end
 * drops its boundary hat, a Neumann end keeps it (basis C):
 * the per-side keep/drop mask of P:L430-L435. */
HD int drop_left(int bc) { return (bc == 0 || bc == 2) ? 1 : 0; }
HD int drop_right(int bc) { return (bc == 0 || bc == 3) ? 1 : 0; }
HD int n_hats(int n, int bc) { return n + 1 - drop_left(bc) - drop_right(bc); }
/* hat index of mesh node `node` (0..n), -1 if dropped (Dirichlet end) */
HD int hat_of_node(int node, int n, int bc) {
  if ((node == 0 && drop_left(bc)) || (node == n && drop_right(bc))) return -1;
  return node - drop_left(bc);
}
HD int node_of_hat(int t, int bc) { return t + drop_left(bc); }
/* chain lengths: parity 0 -> degrees 0,2,4..; parity 1 -> 1,3,5.. (k <= p-2) */
HD int chain_len(int p, int parity) { return parity == 0 ? p / 2 : (p - 1) / 2; }

}  // namespace hpfem

#endif
