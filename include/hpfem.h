/*
 * hpfem.h -- C ABI of the B200-native ADI hp-FEM screened-Poisson solver
 * (the hot path of arXiv 2402.11299).
 *
 * Problem (eq. poisson):  -Laplace(u) + w^2 u = f  on
 * [a,b] x [c,d] with zero Dirichlet (basis Q) or zero Neumann
 * (basis C) conditions, per side (HPFEM_BC_*), discretised in the
 * hat + integrated-Legendre (Babuska-Suri) basis of P:L138-L184 and solved
 * as the generalised Sylvester equation (eq. 2d:poisson P:L419-L424 /
 * eq. adi:poisson P:L658-L664)
 *
 *        A_x U M_y + M_x U A_y = G,     A_d = K_d + (w^2/2) M_d,
 *
 * by the generalised ADI method, Algorithm 2, whose 1D shifted
 * solves use the reverse Cholesky factorisation of Algorithm 1
 * (Cor. 4.3 P:L590-L615).
 *
 * Layout of every 2D array (U, F, G): fp64, N_x x N_y, row-major, contiguous
 * (leading dimension N_y); row i = x-dof, column j = y-dof.  Within each
 * dimension the dofs are ordered degree-major / element-minor as in
 * the kept hats first (n-1 for Dirichlet, n+1 for Neumann, n for
 * mixed ends), then for k = 0..p-2 the n bubbles W_{k,e}, e = 0..n-1.  N =
 * p n - 1 (Dirichlet), p n + 1 (Neumann) or p n (mixed).
 *
 * Ownership: the caller owns F, U, F_leg (DEVICE pointers, e.g. torch
 * tensors).  The plan owns its factor tables, shift tables, stencil-weight
 * tables and its workspace: three N_x x ld internal arrays (the plan's copy
 * of G and the two ADI iterates, ld ~ N_y, internal column order, see
 * DESIGN.md section 5) plus, on the TMA path, an N_x x 2 n_y side array.
 * All work is enqueued asynchronously on the stream passed in
 * (a cudaStream_t; NULL = legacy default stream).  A plan may be used by one
 * stream at a time (its workspace is shared by its solves).
 *
 * Errors: every call returns HPFEM_OK (0) or a negative code; a thread-local
 * message is available from hpfem_last_error().  Launch failures return
 * HPFEM_ECUDA immediately; asynchronous device faults surface at the
 * caller's next synchronisation.  There is no CPU fallback: on a machine
 * without a usable sm_100 device every call that touches the device returns
 * HPFEM_ECUDA.
 */
#ifndef HPFEM_H_
#define HPFEM_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpfem_plan_s* hpfem_plan_t; /* opaque; owned by the library */

/* Boundary conditions (zero data, eq. poisson).  A 1D
 * code fixes both ends of one direction: a Dirichlet end drops its boundary
 * hat (basis Q), a Neumann end keeps it (basis C), so N =
 * p n - 1, p n + 1 or p n (mixed).  A 2D `bc` argument is either a 1D code
 * (the same in both directions) or HPFEM_BC_2D(bc_x, bc_y), per direction. */
enum {
  HPFEM_BC_DIRICHLET = 0,          /* both ends Dirichlet */
  HPFEM_BC_NEUMANN = 1,            /* both ends Neumann (needs w != 0) */
  HPFEM_BC_DIRICHLET_NEUMANN = 2,  /* Dirichlet at a (resp. c), Neumann at b (resp. d) */
  HPFEM_BC_NEUMANN_DIRICHLET = 3   /* Neumann at a (resp. c), Dirichlet at b (resp. d) */
};
#define HPFEM_BC_2D(bc_x, bc_y) (16 + (bc_x) + 4 * (bc_y))

enum {
  HPFEM_OK = 0,
  HPFEM_EINVAL = -1,   /* bad argument: n < 1, p < 2, non-increasing breakpoints,
                          tol not in (0,1), Neumann with w = 0, aliasing,
                          bc not a 1D code or HPFEM_BC_2D(0..3, 0..3) */
  HPFEM_ENOTPD = -2,   /* a non-positive pivot in a reverse Cholesky factorisation */
  HPFEM_ECUDA = -3,    /* CUDA runtime / launch error, or no sm_100 device */
  HPFEM_ENOMEM = -4,   /* device allocation failed */
  HPFEM_ENUMERIC = -5  /* non-finite eigenvalue bound, gamma or shift */
};

/*
 * hpfem_plan -- Alg. 2 "Precomputation" on a uniform mesh.
 *   n_x elements on [a,b] of degree p_x; n_y elements on [c,d] of degree p_y
 *   (p >= 2: hats plus bubbles W_0..W_{p-2}); omega = w of eq. poisson;
 *   bc = HPFEM_BC_* or HPFEM_BC_2D(bc_x, bc_y); tol = epsilon of Lemma 5.1, 0 < tol < 1.
 * Builds the 1D operators (closed forms of App. A), the
 * spectral intervals [lambda_min, lambda_max] of (A_d, M_d) (DESIGN.md
 * reading R4), gamma, J = ceil(log(16 gamma) log(4/tol)/pi^2), the
 * Zolotarev shifts p_j > 0, q_j < 0 (reading R5), and factors the
 * 2J+1 shifted 1D matrices on the device (Alg. 1).  Synchronises
 * cuda_stream once (to read back the factorisation status).
 * On success *out receives a plan to be released with hpfem_plan_destroy.
 */
int hpfem_plan(int n_x, int p_x, int n_y, int p_y, double a, double b, double c, double d, double omega, int bc,
               double tol, void* cuda_stream, hpfem_plan_t* out);

/* As hpfem_plan with explicit strictly increasing breakpoints xs[0..n_x],
 * ys[0..n_y] (host arrays, copied; graded meshes). */
int hpfem_plan_mesh(const double* xs, int n_x, int p_x, const double* ys, int n_y, int p_y, double omega, int bc,
                    double tol, void* cuda_stream, hpfem_plan_t* out);

/* As hpfem_plan_mesh with Robin ends (alpha u + du/dn = 0,
 * the boundary term alpha <v, u>_{L2(side)} added to the stiffness of the
 * end's hat; NEXT-1 of SURVEY 8(f)).  alpha[4] >= 0 (host) at x = a, x = b,
 * y = c, y = d; a nonzero alpha needs a kept (Neumann-coded) end -- EINVAL
 * on a Dirichlet end.  w = 0 is allowed when no direction is Neumann at both
 * ends with zero alphas.  lambda_min of a Robin direction is found by
 * bisection (R22).  alpha = 0 everywhere is hpfem_plan_mesh. */
int hpfem_plan_robin(const double* xs, int n_x, int p_x, const double* ys, int n_y, int p_y, double omega, int bc,
                     const double* alpha, double tol, void* cuda_stream, hpfem_plan_t* out);

/* Plan summary (host outputs; any pointer may be NULL). */
int hpfem_plan_info(hpfem_plan_t plan, int* N_x, int* N_y, int* J, double* lam_x /*[2]*/, double* lam_y /*[2]*/,
                    double* gamma);

/* Mesh sizes of the plan (host outputs; any pointer may be NULL): elements
 * and degree per direction.  The Legendre-coefficient arrays of hpfem_load /
 * hpfem_unload / hpfem_transform are ((p_x+1) n_x) x ((p_y+1) n_y); the
 * bindings use this to check array sizes before a call (the C ABI takes raw
 * pointers and cannot). */
int hpfem_plan_dims(hpfem_plan_t plan, int* n_x, int* p_x, int* n_y, int* p_y);

/* Kernel path of hpfem_solve for this plan (host outputs; either may be
 * NULL): *path = 0 one-CTA-per-problem solve (K11, arrays in shared
 * memory), 1 TMA half-step kernels, 2 LDG half-step kernels;
 * *transposed = 1 when the plan runs Alg. 2 on the transposed equation
 * A_y U^T M_x + M_y U^T A_x = G^T (the long bubble chains then lie along the
 * rows of the internal arrays; reading R23) -- same J, the shifts
 * of the swapped intervals, U returned in the caller's layout. */
int hpfem_plan_path(hpfem_plan_t plan, int* path, int* transposed);

/* Host copies of the shifts: p[0..J-1] (used by the y-solves and the
 * x-applies), q[0..J-1] (x-solves and y-applies), ascending j. */
int hpfem_plan_shifts(hpfem_plan_t plan, double* p, double* q);

/*
 * hpfem_solve -- Alg. 2 "Solve": U = W_J C^{-1} with
 *   W_{j-1/2} = (G - (A_x - p_j M_x) W_{j-1}) (A_y + p_j M_y)^{-1}
 *   W_j       = (A_x - q_j M_x)^{-1} (G - W_{j-1/2} (A_y + q_j M_y))
 * (the "plus" form of the listing, reading R6), satisfying the
 * Lemma 5.1 bound ||V(U* - U)L^T|| <= tol ||V U* L^T||.
 *   F: device pointer, G of eq. adi:poisson (for a Legendre-coefficient f
 *      this is hpfem_load(f)), N_x x N_y.   U: device pointer, N_x x N_y.
 * F and U must not overlap (HPFEM_EINVAL).  F is not modified.
 */
int hpfem_solve(hpfem_plan_t plan, const double* F, double* U, void* cuda_stream);

/* As hpfem_solve but running only the first `iters` ADI iterations
 * (0 <= iters <= J) before the final W C^{-1}; iters = J is hpfem_solve.
 * Used for truncated-iteration parity at full size. */
int hpfem_solve_iters(hpfem_plan_t plan, const double* F, double* U, int iters, void* cuda_stream);

/* hpfem_solve_batched -- hpfem_solve for `batch` independent right-hand
 * sides with the same plan (NEXT-1 of SURVEY 8(f): many F per plan, for the
 * small configurations whose single solve cannot fill the GPU).
 *   F, U: device, batch x N_x x N_y contiguous (problem b at offset b N_x N_y,
 *   each in the layout above); U must not overlap F.
 * The problems are spread over min(batch, HPFEM_BATCH_STREAMS (default 8))
 * internal streams, each with its own workspace (allocated on first use and
 * kept by the plan: 3 N_x x ld arrays per stream), forked from and joined
 * back into cuda_stream, so the call is ordered like any other work on
 * cuda_stream.  Each stream replays one CUDA graph of the line-solve passes
 * per right-hand side.  Each U_b is bitwise what hpfem_solve(F_b) returns.
 * EINVAL also when profiling is on (hpfem_plan_profile records on one
 * stream).  batch = 0 is a no-op. */
int hpfem_solve_batched(hpfem_plan_t plan, int batch, const double* F, double* U, void* cuda_stream);

/* hpfem_apply -- F = A_x U M_y + M_x U A_y (the operator of eq. adi:poisson,
 * P:L658-L664).  U, F device pointers, N_x x N_y, must not overlap.  The
 * rows of A and M are tabled at plan time (HPFEM_NO_APPLY_TAB=1: built per
 * output, the round-1 kernel). */
int hpfem_apply(hpfem_plan_t plan, const double* U, double* F, void* cuda_stream);

/* hpfem_load -- G = R_x^T M_{P,x} F_leg M_{P,y} R_y.
 * F_leg: device, ((p_x+1) n_x) x ((p_y+1) n_y) row-major, degree-major /
 * element-minor (entry [m n_x + e, l n_y + f] multiplies P_m(x) P_l(y) on
 * element (e, f)).  G: device, N_x x N_y.  Must not overlap. */
int hpfem_load(hpfem_plan_t plan, const double* F_leg, double* G, void* cuda_stream);

/* hpfem_unload -- C_leg = R_x U R_y^T: the piecewise-Legendre coefficients
 * of the FEM function u = sum_ij U_ij phi_i(x) psi_j(y) (the inverse basis
 * change of the load, P:L392-L399 with the local R of eq. app:1, P:L1074;
 * NEXT-1 of SURVEY 8(f)).  U: device N_x x N_y (the layout above); C_leg:
 * device ((p_x+1) n_x) x ((p_y+1) n_y), degree-major / element-minor like
 * F_leg (row m n_x + e = Legendre degree m on x-element e).  One kernel, no
 * workspace.  EINVAL on null or overlapping buffers.  The profile kind of
 * this call is 3 (the load/unload kind). */
int hpfem_unload(hpfem_plan_t plan, const double* U, double* C_leg, void* cuda_stream);

/*
 * Transforms and the variable-coefficient solver (NEXT-3 of SURVEY 8(f);
 * Section 6 P:L897-L948 and Section 7).
 *
 * Grid: on every element the p + 1 Chebyshev points of the first kind
 * sin(pi (m - 2k + 1)/(2m)), k = 1..m, m = p + 1 (P:L908-L910 with m = p + 1
 * points for degree p: DESIGN.md R17), affinely mapped.  Grid arrays are
 * ((p_x+1) n_x) x ((p_y+1) n_y) like F_leg / C_leg: row i n_x + e = point i
 * (descending in x) of x-element e (R18).
 *
 * hpfem_grid       -- host arrays x[(p_x+1) n_x], y[(p_y+1) n_y] of the grid
 *                     coordinates (computed on the host, no device work).
 * hpfem_transform  -- C = F_x V F_y^T: values on the grid ->
 *                     Legendre coefficients of the piecewise tensor
 *                     interpolant.  V, C device, grid / F_leg layout.
 * hpfem_itransform -- V = F_x^{-1} C F_y^{-T}: Legendre
 *                     coefficients -> values on the grid.
 * hpfem_varcoef_apply -- F = A_x U M_y + M_x U A_y + <v, c u>, the last term
 *                     by eq. (evaluation) (R19):
 *                     R_x^T M_P F_x [c o (F_x^{-1} R_x U R_y^T F_y^{-T})]
 *                     F_y^T M_P R_y, with c given on the grid (device,
 *                     grid layout).  U, F: device N_x x N_y; F must not
 *                     overlap U or cgrid.
 * hpfem_pcg        -- solves varcoef_apply(U) = G by conjugate gradients
 *                     preconditioned with this plan's ADI solve (the plan's
 *                     tol is the preconditioner tolerance, 1e-4 in the paper,
 *                     P:L1008); U_0 = 0, stops when ||r||_2 <= rtol ||G||_2
 *                     (R20) or after maxit iterations.  *iters = iterations
 *                     (operator applications), *relres = final ||r||/||G||
 *                     (either pointer may be null).  Synchronises cuda_stream
 *                     once per iteration (the residual test); uses the plan's
 *                     solve workspace, so it must not run concurrently with
 *                     hpfem_solve on the same plan.  ENUMERIC on a non-finite
 *                     residual (e.g. an indefinite operator).
 * The transform matrices and scratch (2 grid arrays; 4 N_x N_y vectors for
 * PCG) are allocated on first use and owned by the plan.  EINVAL on null or
 * overlapping buffers, ENOMEM / ECUDA as above.
 */
int hpfem_grid(hpfem_plan_t plan, double* x, double* y);
int hpfem_transform(hpfem_plan_t plan, const double* V, double* C, void* cuda_stream);
int hpfem_itransform(hpfem_plan_t plan, const double* C, double* V, void* cuda_stream);
int hpfem_varcoef_apply(hpfem_plan_t plan, const double* cgrid, const double* U, double* F, void* cuda_stream);
int hpfem_pcg(hpfem_plan_t plan, const double* cgrid, const double* G, double* U, double rtol, int maxit, int* iters,
              double* relres, void* cuda_stream);

/*
 * hpfem_imex_step -- one implicit-explicit time step of the viscous Burgers
 * equation u_t + u u_x = eps Delta u, zero Dirichlet data (NEXT-4 of SURVEY
 * 8(f); Section 6):
 *   u_{k+1/2} = (I - dt eps Delta)^{-1} u_k        (implicit Euler, ADI solve)
 *   u_{k+1}   = u_{k+1/2} - dt u_{k+1/2} d/dx u_{k+1/2}   (explicit Euler on the
 *               grid; the sign of the PDE, R21)
 * The plan must be built with omega = 1/sqrt(dt eps) (the implicit step is
 * the screened problem -Delta w + omega^2 w = omega^2 u_k) and Dirichlet
 * ends in both directions; its tol is the ADI tolerance.  U_leg (in) and
 * U_next (out): device piecewise-Legendre coefficients ((p_x+1) n_x) x
 * ((p_y+1) n_y) (the F_leg layout); the product is formed on the grid (R17)
 * and transformed back: U_next = F [V - dt V_x o V], V = F^{-1} R W R^T
 * F^{-T}, V_x = F^{-1} D W R^T F^{-T}, D the derivative of the
 * hat/bubble expansion (W_k' = -P_{k+1}).  EINVAL on dt <= 0, a plan
 * with omega = 0, or overlapping buffers.  Uses the plan's solve workspace
 * and scratch (not concurrently with another call on the same plan).
 */
int hpfem_imex_step(hpfem_plan_t plan, double dt, const double* U_leg, double* U_next, void* cuda_stream);

/*
 * 1D solver workload (NEXT-2 of SURVEY 8(f); the paper's Fig. 1):
 * batched solves of the 1D screened Poisson discretisation
 *        (K + w^2 M) u = f      (Dirichlet basis Q, Neumann C or mixed)
 * with the reverse Cholesky factor of Algorithm 1 in static-
 * condensation form (one CTA per one or two right-hand sides; for small
 * batches one thread-block cluster per right-hand side, the row held in its
 * distributed shared memory -- same result to rounding).
 *   hpfem_plan1d: breakpoints xs[0..n] (host, strictly increasing), degree
 *     p >= 2, bc = a 1D code HPFEM_BC_DIRICHLET .. HPFEM_BC_NEUMANN_DIRICHLET,
 *     omega (Neumann at both ends needs omega != 0); factors on the device and
 *     synchronises cuda_stream once.  ENOTPD on a non-positive pivot.
 *   hpfem_solve1d: F, U device, nrhs x N row-major (N from hpfem_plan1d_info,
 *     dofs ordered as the 2D arrays' rows: hats, then degree-major bubbles);
 *     U must not overlap F.
 */
typedef struct hpfem_plan1d_s* hpfem_plan1d_t;
int hpfem_plan1d(const double* xs, int n, int p, int bc, double omega, void* cuda_stream, hpfem_plan1d_t* out);
int hpfem_plan1d_info(hpfem_plan1d_t plan, int* N);
int hpfem_solve1d(hpfem_plan1d_t plan, int nrhs, const double* F, double* U, void* cuda_stream);
void hpfem_plan1d_destroy(hpfem_plan1d_t plan);

/* Kernel launches enqueued by the last hpfem_* device call of this plan
 * (for the bench's launch accounting). */
int hpfem_plan_launches(hpfem_plan_t plan, long long* launches);

/*
 * Per-kernel timing with CUDA events recorded on the launch stream around
 * every kernel of subsequent hpfem_solve / hpfem_load / hpfem_apply calls
 * (bench.py's roofline).  hpfem_plan_profile(plan, capacity) creates
 * `capacity` events up front (0 disables and frees them).
 * hpfem_plan_profile_read synchronises on the last event and returns, per
 * kernel kind k (0 = bubble kernel K2-K4 of the half-steps A (y-solves),
 * 1 = their hat Schur kernel K5, 2 = final W C^{-1} kernels, 3 = load K8,
 * 4 = apply K7, 5 / 6 = as 0 / 1 for the half-steps B (x-solves)), the summed
 * duration ms[k], launch count n[k] and algorithmic HBM bytes bytes[k]
 * (DESIGN.md "Roofline"), then resets the counters.  Events beyond the
 * capacity are not recorded (n[] tells).  Profiling keeps the launch
 * configuration of an unprofiled solve (the TMA half-steps' hat lines still
 * run concurrently on the side stream and are then in no kind) but launches
 * the kernels directly instead of replaying the solve's CUDA graph, and
 * disables the one-CTA solve K11 (its passes are not separate kernels).
 */
int hpfem_plan_profile(hpfem_plan_t plan, int capacity);
#define HPFEM_PROFILE_KINDS 7
int hpfem_plan_profile_read(hpfem_plan_t plan, double* ms /*[7]*/, long long* n /*[7]*/, double* bytes /*[7]*/);

void hpfem_plan_destroy(hpfem_plan_t plan);

/* Thread-local message for the last error on this thread ("" if none). */
const char* hpfem_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HPFEM_H_ */
