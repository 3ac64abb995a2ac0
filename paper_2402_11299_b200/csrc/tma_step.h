/*
 * tma_step.h -- TMA-fed half-step kernels (tma_step.cu): tensor maps over
 * the plan's internal arrays and the launcher for the bubble lines.
 */
#ifndef HPFEM_TMA_STEP_H_
#define HPFEM_TMA_STEP_H_

#include <cuda_runtime.h>

#include "hpfem_internal.h"

namespace hpfem {

struct TmaPlan;

/* shape conditions of the TMA path (it then needs the element-major layout) */
bool tma_shape_ok(const DirDev& x, const DirDev& y, int eg_y = 0);  // eg_y: Tuning::eg_y

/* arrays = {Gp, X1, X2} (internal layout L); enable = 0 disables the path */
TmaPlan* tma_plan_create(const DirDev& x, const DirDev& y, const Layout& L, double* const arrays[3], int enable,
                         int eg_y = 0);
void tma_plan_destroy(TmaPlan* T);
/* can the TMA kernel handle the bubble lines of a solve along dir? */
bool tma_supports(const TmaPlan* T, int dir);
/* Precomputed stencil weights of the bubble lines for one ST_APPLY half-step
 * (the apply of direction o = other than the solve direction dir, with
 * S_o = kap K + tau M and the previous solve's correction vectors cvL/cvR):
 *   dir 0 (x-solve, lines = y-bubbles): [e_y][5][Q]
 *   dir 1 (y-solve, lines = x-bubble rows): [e_x][pi][kh][6] (5 used) */
size_t tma_wtab_doubles(const DirDev& x, const DirDev& y, const Layout& L, int dir);
cudaError_t tma_build_wtab(const DirDev& x, const DirDev& y, const Layout& L, int dir, double kap, double tau,
                           const double* cvL, const double* cvR, double* wtab, cudaStream_t st);

/* bubble lines of one half-step; ia_g / ia_w index {Gp, X1, X2} (-1 = unused);
 * the persistent grid leaves `spare_sms` SMs free for concurrent work */
cudaError_t tma_launch_step(const TmaPlan* T, const StepParams& P, int ia_g, int ia_w, cudaStream_t st,
                            int spare_sms = 0);

}  // namespace hpfem

#endif
