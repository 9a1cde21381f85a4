/*
 * pisob200.h -- C ABI of the B200-native differentiable PISO step.
 *
 * Drop-in boundary for the hot path of the reference `pisoflow`
 * (/root/reference/pkg/src/pisoflow, abbreviated S/ below): the forward
 * PISO step `piso.piso_step` (S/piso.py:561-654), its discrete adjoint
 * `adjoint.backward_step` (S/adjoint.py:412-506) and the Krylov solvers they
 * run (`linalg.cg_solve` S/linalg.py:258-273, `linalg.bicgstab_solve`
 * S/linalg.py:276-281, both through `_run_with_fallback` S/linalg.py:215-255).
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer (cudaMalloc / torch allocation) unless
 *    the parameter name ends in `_host`.  The library never allocates device
 *    memory: outputs and scratch are passed in by the caller (torch owns every
 *    buffer).  Scratch sizes come from pf_workspace_bytes().
 *  - `stream` is a cudaStream_t passed as void*; all work is stream ordered.
 *    Solver entry points synchronise `stream` to read convergence status.
 *  - Scalar fields are length n.  Vector fields are structure-of-arrays
 *    (d, n): component c of cell i lives at v[c * n + i].  The Python layer
 *    presents them as the reference's (n, d) arrays through transposed views.
 *  - Stencils (matrices on the cell-adjacency pattern, the reference's CSR
 *    `data` arrays, S/mesh.py:323-346) are stored as (2d + 1, n): row 0 is the
 *    diagonal, row 1 + f the coefficient coupling cell i to its neighbour
 *    across face f = 2 * axis + side (0 where the face is a boundary).
 *  - Boundary faces (S/mesh.py:348-380) are flattened in the reference's
 *    `domain.bfaces` order into m "boundary entries"; boundary velocities are
 *    (d, m) SoA.
 *  - Return value: 0 on success, a PF_ERR_* code otherwise; the message is
 *    available from pf_last_error().  A non-converged solve is NOT an error
 *    code: it is reported through pf_solver_report.converged == 0 (the Python
 *    layer maps it to linalg.SolverError with the reference's stage label).
 *  - Deterministic: no floating-point atomics; every reduction is a fixed
 *    order tree, so repeated calls are bitwise identical (the contract of
 *    T/test_adjoint.py:394-406).
 */
#ifndef PISOB200_H
#define PISOB200_H

#include <stdint.h>

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_ARG 1
#define PF_ERR_CUDA 2
#define PF_ERR_UNSUPPORTED 3

#define PF_TOPO_GATHER 0 /* multi-block: packed neighbour table          */
#define PF_TOPO_BOX 1    /* single block: neighbours by index arithmetic */

#define PF_PRECOND_NONE 0
#define PF_PRECOND_JACOBI 1
#define PF_PRECOND_MG 2
/* BiCGStab only: two Jacobi sweeps, M^-1 = D^-1 (2I - A D^-1), fused into
 * the tiled passes (single-device 3D boxes with whole 8 x 32 Y/Z tiles);
 * elsewhere it runs as PF_PRECOND_JACOBI */
#define PF_PRECOND_NEUMANN2 3

#define PF_GEOM_NONE (-1)
#define PF_GEOM_MULTIGRID 0
#define PF_GEOM_SPECTRAL 1

#define PF_BKIND_DIRICHLET 0
#define PF_BKIND_OUTFLOW 1

/* Static, immutable mesh description (replaces the arrays of
 * mesh.Domain, S/mesh.py:166-469).  All arrays are device pointers. */
typedef struct pf_plan_desc {
  int32_t dim;  /* 2 or 3 */
  int32_t topo; /* PF_TOPO_* */
  int64_t n;    /* number of cells */
  /* PF_TOPO_BOX: block shape (C order, last axis fastest), periodicity per
   * axis, and the first boundary-entry index of face (a, s) (-1 if periodic) */
  int64_t box_shape[3];
  int32_t box_periodic[3];
  int64_t box_face_offset[6];
  /* PF_TOPO_GATHER: (2d, n) packed neighbour table.  v >= 0: neighbour
   * cell (bits 0-25), its axis seen across the face (bits 26-27; the
   * reference's nbr_ax[a, s, i, a]) and orientation flip (bit 28;
   * nbr_sign[a, s, i, a] == -1).  v < 0: boundary entry ~v. */
  const int32_t *nbr;
  /* cell metrics (S/mesh.py:111-119, 247-268) */
  const double *jac;        /* (n)         J = det(dx/dxi)            */
  const double *tmat;       /* (d*d, n)    T[a][j] at row a*d + j      */
  const double *alpha_diag; /* (d, n)      alpha[a][a]                 */
  /* boundary entries (S/mesh.py:348-380) */
  int64_t m;
  const int32_t *bcell;  /* (m) adjacent cell                         */
  const int32_t *bface;  /* (m) face f = 2a + s | kind << 4           */
  const double *bjac;    /* (m) face J                                */
  const double *bt;      /* (d, m) face T[a][j], a = face axis        */
  const double *balpha;  /* (m) face alpha[a][a]                      */
  /* non-orthogonal grids only (NULL / 0 otherwise): the lagged cross
   * fluxes of S/piso.py:322-353, 375-392, 431-449 */
  const double *alpha_full;  /* (d*d, n) alpha[a][k] at row a*d + k       */
  const double *balpha_row;  /* (d, m)   face alpha[a][k], a = face axis  */
  const int32_t *bfid;       /* (m)      face id of each boundary entry   */
  const int32_t *finfo;      /* (nfaces, 8): offset, m, dim0, dim1,
                                tangential-terms active, axis, side, 0    */
  int32_t nfaces;
  int32_t has_cross;         /* cell cross terms active                   */
  /* PF_GEOM_MULTIGRID (0) or PF_GEOM_SPECTRAL: the pressure preconditioner
   * of a box plan.  SPECTRAL asserts that the periodic X / Z axes are
   * uniformly spaced; it falls back to multigrid where the topology does
   * not allow it. */
  int32_t geom_precond;
  /* Slab decomposition along axis 0 of a PF_TOPO_BOX plan (0 / 0: not
   * distributed).  The local box is box_shape[0] = nxl + 2 planes: the nxl
   * planes this rank owns (global planes slab_x0 .. slab_x0 + nxl - 1 of
   * slab_nx) between two ghost planes that mirror the neighbouring ranks'
   * edge planes (axis 0 must be periodic: the ranks form a ring).  Kernels
   * compute the owned cells only; reductions and solver scalars are global
   * over all ranks once a communicator is attached (pf_comm_create,
   * pf_plan_attach_comm). */
  int32_t slab_world;
  int32_t slab_rank;
  int64_t slab_nx;
  int64_t slab_x0;
  /* Separable (tensor-product, axis-aligned) box: the cell widths dx[a][k]
   * and their inverses along each axis (NULL otherwise).  Kernels then form
   * J = prod dx, T = diag(1/dx), alpha = J T^2 from these 1-D arrays (same
   * operation order as the full (n) arrays) instead of streaming 13 metric
   * values per cell from HBM. */
  const double *sep_dx[3];
  const double *sep_inv[3];
  /* optional (n) array 1 / jac (exactly 1.0 / jac[i]); kernels that divide
   * by J at several cells per cell load it instead */
  const double *ijac;
} pf_plan_desc;

typedef struct pf_plan pf_plan;

/* Outcome of one linear solve (replaces linalg.SolverReport,
 * S/linalg.py:29-35). */
typedef struct pf_solver_report {
  int32_t converged;
  int32_t iterations;
  double residual; /* true residual / |b| when converged */
  int32_t fallback_used;
  int32_t breakdown; /* 1 if the Krylov recurrence broke down */
} pf_solver_report;

PF_API const char *pf_last_error(void);
PF_API int pf_version(void);
/* number of kernels this library has launched in the process (for the
 * benchmark's gpu_launches accounting) */
PF_API unsigned long long pf_launch_count(void);

PF_API int pf_plan_create(const pf_plan_desc *desc, pf_plan **out);
PF_API int pf_plan_destroy(pf_plan *plan);
/* bytes of device scratch the solvers and reductions need for this plan */
PF_API int64_t pf_workspace_bytes(const pf_plan *plan);

/* ---- forward building blocks (S/piso.py) --------------------------------- */

/* U^a = J (T u)_a  -- piso.contravariant_flux, S/piso.py:123-125 */
PF_API int pf_contravariant_flux(const pf_plan *plan, const double *u, double *flux,
                          void *stream);

/* C = advection-diffusion stencil -- piso.assemble_momentum,
 * S/piso.py:293-319.  `flux_scratch` is (d, n). */
PF_API int pf_assemble_momentum(const pf_plan *plan, const double *u_n, double nu,
                         double dt, double *flux_scratch, double *c_out,
                         void *stream);

/* rhs = u_n/dt + S + boundary terms -- piso.momentum_rhs, S/piso.py:356-372
 * (orthogonal faces; the lagged non-orthogonal flux is zero there).
 * `source` is (d, n), or a (d) vector when source_is_uniform != 0. */
PF_API int pf_momentum_rhs(const pf_plan *plan, const double *u_n, const double *bc,
                    const double *source, int32_t source_is_uniform,
                    double nu, double dt, double *rhs_out, void *stream);

/* K = -P stencil -- piso.assemble_pressure, S/piso.py:395-412; K's diagonal
 * is the sum of the face coefficients, its off-diagonals the negated face
 * means.  `c` is the momentum stencil (its row 0, A, is read) or, when
 * c_is_a_inv != 0, the (n) vector A^-1 itself. */
PF_API int pf_assemble_pressure(const pf_plan *plan, const double *c,
                                int32_t c_is_a_inv, double *k_out,
                                void *stream);

/* h = A^-1 (rhs - H u) -- corrector h stage, S/piso.py:608-612 */
PF_API int pf_h_stage(const pf_plan *plan, const double *c, const double *u_cur,
               const double *rhs, double *h_out, void *stream);

/* b = divergence_rhs(h, bc), S/piso.py:415-428 (flux_scratch (d, n)) */
PF_API int pf_divergence_rhs(const pf_plan *plan, const double *h, const double *bc,
                      double *flux_scratch, double *b_out, void *stream);

/* u = h - A^-1 T^t wide_grad(p, mirror) -- piso.correct_velocity,
 * S/piso.py:452-455 with wide_grad S/piso.py:172-209 */
PF_API int pf_correct_velocity(const pf_plan *plan, const double *h, const double *p,
                        const double *c, double *u_out, void *stream);

/* max |divergence_rhs(u, bc) / J| -- StepDiagnostics.div_wide_max,
 * S/piso.py:458-460, 635-636.  Result written to *out_host. */
PF_API int pf_divergence_max(const pf_plan *plan, const double *u, const double *bc,
                      double *flux_scratch, void *workspace, double *out_host,
                      void *stream);
/* The same maximum written to the device scalar *out_dev without waiting
 * (the step's diagnostics read it lazily: no host round trip between the
 * forward step and the adjoint). */
PF_API int pf_divergence_max_dev(const pf_plan *plan, const double *u,
                                 const double *bc, double *flux_scratch,
                                 void *workspace, double *out_dev,
                                 void *stream);

/* y = A x (transpose != 0: y = A^t x) for a stencil A, ncomp right-hand
 * sides of length n each -- SystemPattern.matvec, S/linalg.py:80-83 and
 * _kernels_c.matvec S/_kernels_c.pyx:45-63 */
PF_API int pf_stencil_matvec(const pf_plan *plan, const double *a, int32_t transpose,
                      int32_t ncomp, const double *x, double *y, void *stream);

/* ---- solvers (S/linalg.py) ---------------------------------------------- */

/* Zero-mean (optional) Jacobi-preconditioned CG on stencil `a`, with the
 * reference's semantics: b projected to zero mean, relative tolerance,
 * true-residual verification <= 10 tol_abs, unpreconditioned retry from zero
 * with 2*maxiter on failure -- cg_solve / _cg_core / _run_with_fallback,
 * S/linalg.py:136-170, 215-273.  The right-hand side is b_scale * b.  x holds
 * the warm start on entry (has_x0 != 0; zero otherwise) and the solution on
 * exit. */
PF_API int pf_cg_solve(const pf_plan *plan, const double *a, const double *b,
                       double b_scale, double *x, int32_t has_x0, double tol,
                       int32_t maxiter, int32_t zero_mean, int32_t precond,
                       void *workspace, void *mg_workspace,
                       pf_solver_report *report_host, void *stream);

/* Geometric preconditioner for the pressure operator of a box plan (the GPU
 * replacement of the reference's ILU(0) preconditioner, S/linalg.py:88-108),
 * one of:
 *  - PF_GEOM_MULTIGRID: V(1,1) cycle, Y-line block-Jacobi smoothing, 2x
 *    coarsening with Galerkin aggregation, exact singular coarsest line
 *    solve;
 *  - PF_GEOM_SPECTRAL (desc.geom_precond == PF_GEOM_SPECTRAL and periodic
 *    power-of-two X / Z): exact inverse of the XZ-plane-averaged operator,
 *    Fourier in X and Z, tridiagonal in Y.
 * pf_cg_solve with precond == PF_PRECOND_MG uses the preconditioner last
 * built by pf_mg_setup on the same mg_workspace.  pf_mg_workspace_bytes
 * returns 0 (pf_mg_levels 0, pf_mg_kind PF_GEOM_NONE) when the plan supports
 * neither (gather topology, periodic line axis). */
PF_API int64_t pf_mg_workspace_bytes(const pf_plan *plan);
PF_API int pf_mg_levels(const pf_plan *plan);
PF_API int pf_mg_kind(const pf_plan *plan);
PF_API int pf_mg_setup(const pf_plan *plan, const double *k,
                       void *mg_workspace, void *stream);

/* ncomp independent preconditioned BiCGStab solves sharing matrix `a`
 * (transpose != 0 solves with A^t); precond PF_PRECOND_NONE, _JACOBI or
 * _NEUMANN2 (see above) -- bicgstab_solve / _bicgstab_core,
 * S/linalg.py:173-212, 276-281; the predictor loop S/piso.py:583-590 and the
 * adjoint momentum solve S/adjoint.py:369-380.  One report per component. */
PF_API int pf_bicgstab_solve(const pf_plan *plan, const double *a, int32_t transpose,
                      int32_t ncomp, const double *b, double *x,
                      int32_t has_x0, double tol, int32_t maxiter,
                      int32_t precond, void *workspace,
                      pf_solver_report *reports_host, void *stream);

/* Live timing of the CG iteration kernels on operator `a` (tol = 0, so the
 * recurrence never stops), over `iters` iterations, timed with CUDA events
 * on `stream`; average ms per iteration of:
 *   ms_host[0] SpMV + p.Ap   [1] x/r update + sums
 *   [2..6] multigrid level 0: line smooth | residual+restrict | all coarse
 *          levels | prolong+residual | line smooth with correction; or
 *          spectral: Z transform | X transform | Y solve | inverse X |
 *          inverse Z (precond == PF_PRECOND_MG; zero otherwise)
 *   [7] z sums   [8] direction update   [9] whole iteration
 *   [10] whole iteration replayed from the cached CUDA graph (MG only)
 *   [11] 1 when the direction update rides in a tiled SpMV (slot [0] then
 *        times k_cg_spmv_pt, slot [8] is empty).
 * Used by bench.py for the roofline figure. */
PF_API int pf_cg_profile(const pf_plan *plan, const double *a,
                         const double *b, int32_t iters, int32_t precond,
                         void *workspace, void *mg_workspace,
                         double *ms_host, void *stream);

/* Live per-pass timing of the batched BiCGStab iteration (bench.py roofline):
 * `iters` iterations with the production preconditioner (Neumann-2 where it
 * runs, else Jacobi) on `ncomp` right-hand sides of the operator a
 * (transposed if `transpose`), each pass bracketed by CUDA events on
 * `stream`.  ms_host[0..3] = mean ms of pass pv, pass st, pass xr and the
 * whole iteration; ms_host[4] = the preconditioner timed (1 Jacobi, 3
 * Neumann-2).  Not part of the reference interface. */
PF_API int pf_bicgstab_profile(const pf_plan *plan, const double *a,
                               int32_t transpose, int32_t ncomp,
                               const double *b, int32_t iters,
                               void *workspace, double *ms_host, void *stream);

/* ---- adjoint stage kernels (S/adjoint.py) --------------------------------- */

/* backward_correct_velocity, S/adjoint.py:78-91: dA += (cu . T^t g)/A^2,
 * cot_p = wide_grad_adjoint(-A^-1 T cu) (+ extra_cot_p if non-null). */
PF_API int pf_bwd_correct_velocity(const pf_plan *plan, const double *p,
                            const double *c, const double *cu, double *da,
                            double *cot_p, const double *extra_cot_p,
                            int32_t overwrite, void *workspace, void *stream);

/* dKf[f][i] += y_i (p_nb - p_i): face cotangents of the pressure stencil from
 * one adjoint pressure solve -- outer_on_pattern(y, p) S/adjoint.py:113
 * folded with the diagonal as backward_pressure_matrix consumes it.
 *
 * overwrite != 0 (here and in pf_bwd_correct_velocity, pf_bwd_h_stage,
 * pf_adj_momentum_rhs): the first writer of an accumulator stores instead
 * of adding (boundary faces get 0), so the caller need not zero-fill it;
 * owned cells only. */
PF_API int pf_bwd_pressure_outer(const pf_plan *plan, const double *y,
                          const double *p, double *dkf, int32_t overwrite,
                          void *stream);

/* dA += backward_pressure_matrix(a_inv, dP), S/adjoint.py:116-134 */
PF_API int pf_bwd_pressure_matrix(const pf_plan *plan, const double *c,
                           const double *dkf, double *da, void *stream);

/* _adj_divergence_rhs, S/adjoint.py:137-153, for the cotangent cot_scale*cot_b:
 * g_h += J T^t g_flux(cot_b),
 * dbc += N J_f cot_b T_f[a,:] */
PF_API int pf_adj_divergence_rhs(const pf_plan *plan, const double *cot_b,
                                 double cot_scale, double *g_h, double *dbc,
                                 void *stream);

/* h-stage adjoint, S/adjoint.py:477-487: dA -= A^-1 g_h.h; g_rhs += A^-1 g_h;
 * dC_off += outer(-A^-1 g_h, u_hin); cu = (C^t - A)(-A^-1 g_h). */
PF_API int pf_bwd_h_stage(const pf_plan *plan, const double *c, const double *g_h,
                   const double *h, const double *u_hin, double *da,
                   double *g_rhs, double *dc, double *cu_out,
                   int32_t overwrite, void *workspace, void *stream);

/* dC += outer(-y, u_star) on the pattern (diagonal included) -- the matrix
 * cotangent of the momentum solve, S/adjoint.py:380 */
PF_API int pf_bwd_momentum_outer(const pf_plan *plan, const double *y,
                          const double *u_star, double *dc, void *stream);

/* _adj_momentum_rhs, S/adjoint.py:236-268 (orthogonal faces):
 * du_n += cot/dt, dbc += ..., *dnu_dev += sum(...).  dnu_dev is a device
 * double accumulated in stream order. */
PF_API int pf_adj_momentum_rhs(const pf_plan *plan, const double *cot_rhs,
                        const double *bc, double nu, double dt, double *du_n,
                        double *dbc, double *dnu_dev, int32_t overwrite,
                        void *workspace, void *stream);

/* _adj_assemble_momentum, S/adjoint.py:307-340: du_n += J T^t g_flux(dC),
 * *dnu_dev += viscous part. */
PF_API int pf_adj_assemble_momentum(const pf_plan *plan, const double *dc,
                             double nu, double *du_n, double *dnu_dev,
                             void *workspace, void *stream);

/* ---- non-orthogonal grids (plans built with alpha_full) ------------------- */

/* rhs += momentum_cross_rhs(u_cross, nu), S/piso.py:322-342 (lagged viscous
 * cross fluxes divided by J; the tangential boundary flux of
 * S/piso.py:375-392 is part of pf_momentum_rhs on such plans) */
PF_API int pf_momentum_cross_rhs(const pf_plan *plan, const double *u,
                                 double nu, double *rhs_inout,
                                 void *workspace, void *stream);
/* b_out = b0 - pressure_cross_rhs(A^-1, p_prev), S/piso.py:431-449, 617 */
PF_API int pf_pressure_cross_rhs(const pf_plan *plan, const double *c,
                                 const double *p_prev, const double *b0,
                                 double *b_out, void *workspace, void *stream);
/* _adj_pressure_cross, S/adjoint.py:156-178, for the cotangent
 * cot_scale * cot_out: dA += ..., dp_prev = ... */
PF_API int pf_adj_pressure_cross(const pf_plan *plan, const double *c,
                                 const double *p_prev, const double *cot_out,
                                 double cot_scale, double *da,
                                 double *dp_prev, void *workspace,
                                 void *stream);
/* _adj_momentum_cross, S/adjoint.py:181-205: du_cross (+)= ..., *dnu_dev +=
 * ... */
PF_API int pf_adj_momentum_cross(const pf_plan *plan, const double *u,
                                 double nu, const double *cot_out,
                                 double *du_cross, int32_t accumulate,
                                 double *dnu_dev, void *workspace,
                                 void *stream);

/* ---- standalone building blocks (the public stage API) ------------------- */

/* wide_grad, S/piso.py:172-209: out (d, n) = wide central differences of
 * phi (n) along every grid axis; variant 0 "mirror", 1 "onesided", 2 "face"
 * (bc_cells (2d, n): row 2a+s holds the prescribed face values of the cells
 * missing neighbour (a, s); null for the other variants).  Not on slab
 * plans. */
PF_API int pf_wide_grad(const pf_plan *plan, const double *phi,
                        int32_t variant, const double *bc_cells, double *out,
                        void *stream);
/* wide_grad_adjoint, S/piso.py:218-264: out (n) = the adjoint w.r.t. phi of
 * cot (d, n); face variant: bc_cot (2d, n) receives the cotangent of the
 * prescribed face values (may be null). */
PF_API int pf_wide_grad_adjoint(const pf_plan *plan, const double *cot,
                                int32_t variant, double *out, double *bc_cot,
                                void *stream);

/* ---- channel drivers (S/piso.py:512-546) ---------------------------------- */

/* adaptive_dt's CFL peak, S/piso.py:512-520: *out_dev = max over the owned
 * cells of sum_a |U^a| / J (collective on slab plans: the global max). */
PF_API int pf_cfl_peak(const pf_plan *plan, const double *u, void *workspace,
                       double *out_dev, void *stream);
/* wall_shear_mean + wall_forcing_source, S/piso.py:523-542: for each of
 * nwall walls (entries seg[w] .. seg[w+1] of cells / dist: the first cell
 * row and its distance to the wall face) the mean of u[c, flow] / dist;
 * out_dev (d) = (0, .., nu mean_w |mean_w| / delta, .., 0) at flow_axis.
 * seg is a device array of nwall + 1 offsets (m = seg[nwall]), cnt (nwall,
 * device) the row sizes the sums are divided by (collective on slab plans:
 * the sums span the ranks, cnt holds the global sizes). */
PF_API int pf_wall_forcing(const pf_plan *plan, const double *u,
                           int32_t flow_axis, const int32_t *cells,
                           const double *dist, const int32_t *seg,
                           const double *cnt, int32_t nwall, int32_t m,
                           double nu, double delta, double *out_dev,
                           void *workspace, void *stream);

/* y += alpha x over len entries (device vectors) */
PF_API int pf_axpy(const pf_plan *plan, double alpha, const double *x,
                   double *y, int64_t len, void *stream);

/* ---- boundary preprocessing (S/piso.py:467-509) --------------------------- */

/* advective_outflow_update: relax outflow faces towards the adjacent cells
 * and rescale for zero net boundary flux.  bc_inout (d, m) is updated in
 * place; the scale factor is written to *scale_host. */
PF_API int pf_advective_outflow_update(const pf_plan *plan, const double *u,
                                double *bc_inout, double dt, void *workspace,
                                double *scale_host, void *stream);

/* generic deterministic reductions used by the host layer */
PF_API int pf_reduce_sum(const pf_plan *plan, const double *x, int64_t len,
                  void *workspace, double *out_host, void *stream);
PF_API int pf_reduce_dot(const pf_plan *plan, const double *x, const double *y,
                  int64_t len, void *workspace, double *out_host,
                  void *stream);
PF_API int pf_reduce_maxabs(const pf_plan *plan, const double *x, int64_t len,
                     void *workspace, double *out_host, void *stream);

/* ---- channel statistics (SURVEY.md §8 f; S/stats.py) ----------------------- */

/* frame_profile, S/stats.py:262-279 (slice_mean + slice_cov): for every
 * wall-normal slice j (index along `wall_axis` of a box plan) the mean
 * (Y, d) and the central covariance (Y, d, d) of the velocity (d, n) over
 * the slice's cells, population convention; m3 / m4 (optional, (Y, d)) are
 * the third and fourth central moments per component (ChannelAccumulator,
 * S/stats.py:325-376).  Two-pass (means, then central products), fixed-order
 * reductions; collective on slab plans (the slices span every rank). */
PF_API int pf_slice_moments(const pf_plan *plan, const double *u,
                            int32_t wall_axis, double *mean, double *cov,
                            double *m3, double *m4, void *workspace,
                            void *stream);
/* frame_profile_backward, S/stats.py:281-290: du (d, n) on the owned cells
 * from the cotangents of (mean, cov) of the same frame. */
PF_API int pf_slice_moments_backward(const pf_plan *plan, const double *u,
                                     int32_t wall_axis, const double *mean,
                                     const double *d_mean, const double *d_cov,
                                     double *du, void *stream);

/* ---- slab decomposition across GPUs (SURVEY.md §8 e) ----------------------
 * The reference is single-process; these entry points have no reference
 * counterpart.  A slab plan (pf_plan_desc.slab_world > 0) computes its owned
 * planes; a communicator links it to the other ranks' plans through peer
 * memory (NVLink P2P via CUDA IPC across processes, or direct pointers for
 * several slabs of one process on one device).  Once attached, every entry
 * point of the plan is COLLECTIVE: all ranks call the same entry points in
 * the same order, ghost planes of the arrays they read are exchanged inside
 * the call, and every reduction (solver dot products, means, maxima) is
 * global and bitwise identical on all ranks.  Ghost planes of every array
 * passed to a slab plan are owned by the library. */
typedef struct pf_comm pf_comm;

/* Allocate this rank's symmetric buffer (halo inboxes, reduction slots, the
 * spectral preconditioner's transposed spectrum) for a slab plan. */
PF_API int pf_comm_create(const pf_plan *plan, pf_comm **out);
/* 64-byte cudaIpcMemHandle of the symmetric buffer, for the other ranks. */
PF_API int pf_comm_ipc_handle(const pf_comm *comm, void *handle_host);
/* Map rank `peer`'s buffer from its IPC handle (cross-process, NVLink). */
PF_API int pf_comm_open_peer(pf_comm *comm, int32_t peer, const void *handle_host);
/* Same-process peer (several slab plans of one process on one device). */
PF_API int pf_comm_set_local_peer(pf_comm *comm, int32_t peer, const pf_comm *other);
PF_API int64_t pf_comm_bytes(const pf_comm *comm);
/* After every peer is mapped: make the plan (and its workspace) use it. */
PF_API int pf_plan_attach_comm(pf_plan *plan, pf_comm *comm, void *workspace,
                               void *stream);
/* PF_ERR_CUDA if a device-side wait for a peer timed out. */
PF_API int pf_comm_status(const pf_comm *comm, void *stream);
PF_API int pf_comm_destroy(pf_comm *comm);
/* Exchange the ghost planes of `count` (ncomp_host[j], n) arrays. */
PF_API int pf_halo_exchange(const pf_plan *plan, const uint64_t *arrays_host,
                            const int32_t *ncomp_host, int32_t count,
                            void *stream);
/* buf[0..k) <- sum (op 0) or max (op 1) over the ranks, in place. */
PF_API int pf_comm_allreduce(const pf_plan *plan, double *buf, int32_t k,
                             int32_t op, void *stream);
PF_API int pf_comm_barrier(const pf_plan *plan, void *stream);
/* Sequence numbers of the collectives this rank has completed: allreduce,
 * halo exchange, barrier, vector allreduce (tests and diagnostics). */
PF_API int pf_comm_counters(const pf_comm *comm, uint64_t *out4_host,
                            void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PISOB200_H */
