/*
 * linedg_b200.h -- C-ABI of the B200 (sm_100a) Line-DG hot path.
 *
 * This is the drop-in boundary for the part of the reference library
 * `linedg` whose sources are listed but absent from the reference tree
 * (reference proj/src/CMakeLists.txt:6-8: discretization.cpp, assembly.cpp,
 * sparse.cpp).  Their C++ surface is reconstructed from SPEC.md:
 *
 *   residual_first_order(ctx, U, t)            SPEC.md:218-226   -> ldg_residual (first-order physics)
 *   gradient_residual(ctx, U, Q, t)            SPEC.md:228-236   -> ldg_gradient
 *   residual_second_order(ctx, U, Q, t)        SPEC.md:238-246   -> ldg_residual_uq
 *   residual_primal(ctx, U, t)                 SPEC.md:248-256   -> ldg_residual (second-order physics)
 *   assemble_jacobians(ctx, U, t, Analytic)    SPEC.md:409-417   -> ldg_jacobian_assemble
 *   split_matvec(blocks, alpha_dt, v)          SPEC.md:419-427   -> ldg_split_matvec
 *   CscMatrix export                           SPEC.md:391-394      -> ldg_export_blocks
 *   triplet export / sparsity CSV              SPEC.md:465, 633     -> ldg_write_triplets, ldg_write_sparsity_csv
 *
 * Inputs are the reference's own setup objects, flattened (no Eigen, no C++
 * types): NodalBasis1D (reference basis.hpp:17-43), QuadMesh/Face/elem_face
 * (mesh.hpp:15-39), SwitchAssignment (mesh.hpp:74-89), ElementMapping
 * (mapping.hpp:19-33), GasModel (physics.hpp:10-14).  Grid functions use the
 * reference GridFunction layout value(e,node,c) = data[(e*npe+node)*m+c]
 * (field.hpp:8-9); the auxiliary gradient uses ((e*npe+node)*m+c)*D+d
 * (field.hpp:38-40 generalised to D).
 *
 * Device entry points take DEVICE pointers and are stream-ordered on the
 * stream given to ldg_create; every device vector must be 16-byte aligned
 * (it is read with 16-byte vector / bulk-async copies; a misaligned pointer is
 * rejected with LDG_ERR_INVALID_ARGUMENT).  The *_host variants take HOST
 * pointers and synchronise.  Every entry point returns an ldg_status; the message of the
 * last failure is available from ldg_last_error().  Status codes mirror the
 * reference exception taxonomy (errors.hpp:10-28):
 *   LDG_ERR_PHYSICAL_STATE  <-> physical_state_error (state via ldg_last_error_state)
 *   LDG_ERR_CONFIG          <-> config_error
 *   LDG_ERR_SOLVER          <-> solver_error
 */
#ifndef LINEDG_B200_H
#define LINEDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum ldg_status {
  LDG_OK = 0,
  LDG_ERR_PHYSICAL_STATE = 1,
  LDG_ERR_CONFIG = 2,
  LDG_ERR_SOLVER = 3,
  LDG_ERR_CUDA = 4,
  LDG_ERR_INVALID_ARGUMENT = 5
} ldg_status;

/* --------------------------------------------------------------- physics */
typedef enum ldg_physics_kind {
  LDG_POISSON = 0,         /* PoissonModel       physics.hpp:98-118  (m = 1)   */
  LDG_EULER = 1,           /* EulerModel         physics.hpp:138-162 (m = D+2) */
  LDG_NAVIER_STOKES = 2    /* NavierStokesModel  physics.hpp:164-187 (m = D+2) */
} ldg_physics_kind;

typedef enum ldg_riemann_kind {
  LDG_ROE = 0,  /* roe_flux, Harten entropy fix 0.05(|u.n|+a)  physics.hpp:196-198 */
  LDG_LLF = 1   /* local Lax-Friedrichs (extension; not in the reference)                      */
} ldg_riemann_kind;

/* Boundary conditions (BcKind, physics.hpp:16; SPEC.md:266,
 * 366-368).  value[] holds constant data per component (the reference's
 * std::function data cannot cross to the device).                          */
typedef enum ldg_bc_kind {
  LDG_BC_DIRICHLET = 0,        /* g_D = value: Riemann flux vs g_D (inviscid), F(u,q).n + C11_bd|n|(u - g_D)
                                  (viscous), u_hat = g_D                            */
  LDG_BC_NEUMANN = 1,          /* g_N = value: F_hat.n = g_N |n| (whole flux), u_hat = u (C22 = 0;
                                  PAPER.md:577-581)                                                   */
  LDG_BC_CHARACTERISTIC = 2,   /* far-field state = value: Riemann flux vs the free-stream ghost state
                                  (SPEC.md:266, 366); viscous terms as Dirichlet with the far state    */
  LDG_BC_SLIP_WALL = 3,        /* Riemann flux vs the interior state with mirrored normal momentum
                                  (SPEC.md:367); viscous F(u,q).n, u_hat = u; Euler / Navier-Stokes   */
  LDG_BC_NO_SLIP_ADIABATIC = 4 /* mixed wall: Riemann flux vs the interior state with its
                                  momentum reversed; viscous: momentum F(u,q).n + C11_bd|n| m (Dirichlet
                                  zero velocity), zero energy flux (adiabatic); u_hat = (rho, 0, E) of u;
                                  Euler / Navier-Stokes                                                */
} ldg_bc_kind;

typedef struct ldg_bc {
  int32_t tag;             /* mesh boundary tag (Face::tag, mesh.hpp:24) */
  int32_t kind;            /* ldg_bc_kind */
  double value[8];         /* g_D / g_N / far-field state per component (first m used) */
} ldg_bc;

typedef struct ldg_physics {
  int32_t kind;            /* ldg_physics_kind */
  int32_t riemann;         /* ldg_riemann_kind (Euler / Navier-Stokes) */
  double gamma;            /* GasModel::gamma   (physics.hpp:11) */
  double mu;               /* GasModel::mu      (physics.hpp:12) */
  double prandtl;          /* GasModel::prandtl (physics.hpp:13) */
  double c11;              /* LdgParams::C11 interior, >= 0 */
  double c22;              /* LdgParams::C22; must be 0 (residual_primal) */
  double c11_bd;           /* boundary C11 coefficient: C11_bd = c11_bd * p^2 / h_face */
  int32_t n_bc;            /* number of boundary conditions */
  const ldg_bc* bcs;       /* BoundaryTable (physics.hpp:35): one entry per boundary tag */
} ldg_physics;

/* ----------------------------------------------------------------- setup */
/* Flattened reference setup objects.  D = dim, np = p+1, npe = np^D,
 * NL = np^(D-1) lines per direction, nq = n_quad.                         */
typedef struct ldg_setup {
  int32_t dim;             /* 2 (reference) or 3 (hexahedral extension) */
  int32_t p;
  int32_t n_quad;          /* (3p+2)/2, basis.cpp:176 */
  int32_t n_elems;
  int32_t n_faces;
  /* NodalBasis1D (basis.hpp:17-33); matrices row-major [i][q] */
  const double* nodes;          /* [np]      */
  const double* quad_points;    /* [nq]      */
  const double* quad_weights;   /* [nq]      */
  const double* phi_at_quad;    /* [np][nq]  */
  const double* dphi_at_quad;   /* [np][nq]  */
  const double* mass;           /* [np][np]  SPD */
  /* QuadMesh faces (mesh.hpp:15-26) and elem_face (mesh.hpp:32).
   * face_orient: 2-D = Face::reversed (0/1); 3-D = dihedral code o in [0,8)
   * mapping elem_l's face parameter (a,b) to elem_r's:
   *   (x,y) = (o&1) ? (b,a) : (a,b);  a' = (o&2) ? p-x : x;  b' = (o&4) ? p-y : y.  */
  const int32_t* face_elem_l;
  const int32_t* face_face_l;
  const int32_t* face_elem_r;   /* -1 on boundary faces */
  const int32_t* face_face_r;
  const int32_t* face_orient;
  const int32_t* face_tag;      /* -1 on interior faces */
  const int32_t* elem_face;     /* [E][2D] */
  const int8_t* switch_plus;    /* [E][D] SwitchAssignment::plus_sign (mesh.hpp:76); NULL for first-order */
  /* ElementMapping (mapping.hpp:19-33) */
  const double* jac_at_nodes;   /* [E][npe]                */
  const double* nvec_quad;      /* [E][D][NL][nq][D]       */
  const double* normal_end;     /* [E][D][2][NL][D]        */
  const double* node_coords;    /* [E][npe][D] (nodes_xy); optional, may be NULL */
} ldg_setup;

/* ------------------------------------------------------------ Jacobians */
typedef enum ldg_matrix {
  LDG_K11 = 0,   /* dR/dU  block m x m              */
  LDG_K12 = 1,   /* dR/dQ  block m x mD (second-order physics) */
  LDG_K21 = 2    /* dD/dU  block mD x m, component-diagonal, U-independent */
} ldg_matrix;

/* Node-level pattern of one matrix in the REFERENCE numbering:
 * row/col are global node ids e*npe+node.  Sorted by (row, col). */
typedef struct ldg_pattern_info {
  int64_t n_rows;          /* global nodes                      */
  int64_t nnzb;            /* structural node blocks            */
  int32_t block_rows;      /* scalar rows per block (m, or mD for K21) */
  int32_t block_cols;      /* scalar cols per block             */
} ldg_pattern_info;

typedef struct ldg_ctx ldg_ctx;

/* Creation binds the context to one CUDA stream (cudaStream_t, may be NULL
 * for the legacy default stream).  All tables are copied; the setup memory
 * may be freed after return. */
int ldg_create(const ldg_setup* setup, const ldg_physics* physics, void* cuda_stream,
               ldg_ctx** out);
void ldg_destroy(ldg_ctx* ctx);
const char* ldg_last_error(const ldg_ctx* ctx);        /* ctx may be NULL (creation errors) */
/* After LDG_ERR_PHYSICAL_STATE: offending element, node and state (m doubles). */
int ldg_last_error_state(const ldg_ctx* ctx, int32_t* elem, int32_t* node, double* state);
int ldg_components(const ldg_ctx* ctx);               /* m */
int64_t ldg_num_dofs(const ldg_ctx* ctx);             /* E * npe * m */

/* Space- and time-dependent boundary data (the reference's std::function
 * g_D / g_N data, physics.hpp:20-31): fn(user, x[dim], t, out[m]) is evaluated
 * on the host at the end node of every boundary line end tagged `tag` (node
 * coordinates from ldg_setup.node_coords, required) and uploaded; it replaces
 * that condition's constant value[] (Dirichlet g_D, Neumann g_N, far-field
 * state).  Re-evaluated when a device call passes a different t.  fn = NULL
 * restores the constant data.  The callback runs on the calling host thread. */
typedef void (*ldg_bc_fn)(void* user, const double* x, double t, double* out);
int ldg_set_boundary_function(ldg_ctx* ctx, int32_t tag, ldg_bc_fn fn, void* user);

/* Optional nodal source S (E*npe*m doubles, host pointer), added to R
 * (PoissonModel::source_fn evaluated at the nodes, physics.hpp:102). */
int ldg_set_source(ldg_ctx* ctx, const double* source_host);

/* Residual.  First-order physics: R = S - (1/J) sum_dir r.
 * Second-order physics: residual_primal, Q = D(U) is computed first and
 * written to Q_or_null when non-NULL.  Device pointers.                 */
int ldg_residual(ldg_ctx* ctx, const double* U, double t, double* R, double* Q_or_null);
/* residual_second_order R(U,Q) for a given Q (device pointers). */
int ldg_residual_uq(ldg_ctx* ctx, const double* U, const double* Q, double t, double* R);
/* gradient_residual: Q = (1/J) sum_dir d (device pointers). */
int ldg_gradient(ldg_ctx* ctx, const double* U, double t, double* Q);

/* Jacobians (analytic), stored on the device in the line-structured block
 * store.  Second-order physics uses Q = D(U), computed internally. */
int ldg_jacobian_assemble(ldg_ctx* ctx, const double* U, double t);
/* Assembly at U with the gradient Q = D(U) the caller already holds on the
 * device (from ldg_residual(ctx, U, t, R, Q)): skips recomputing Q.  Q is
 * ignored (may be NULL) for first-order physics. */
int ldg_jacobian_assemble_q(ldg_ctx* ctx, const double* U, const double* Q, double t);
int ldg_pattern_info_get(const ldg_ctx* ctx, int which, ldg_pattern_info* info);
/* y = K x for K in {K11, K12, K21} (device pointers; x, y in reference numbering). */
int ldg_bsr_spmv(ldg_ctx* ctx, int which, const double* x, double* y);
/* y = v - alpha_dt (K11 v + K12 (K21 v)); first-order: y = v - alpha_dt K11 v */
int ldg_split_matvec(ldg_ctx* ctx, double alpha_dt, const double* v, double* y);

/* Block-Jacobi preconditioner: per element,
   the LU factors (partial pivoting) of I - alpha_dt A~, A~ = K11 + K12 K21 kept
   only on the block-diagonal Line-DG pattern (row and column node in the same
   element and on a common coordinate line; the product's entries landing there
   are exact, all other fill and inter-element couplings dropped).  Requires an
   assembled Jacobian.  Element blocks of up to 128 unknowns (2-D p <= 4,
   3-D p = 1) are factorised whole.  Above that (3-D p >= 2) the preconditioner
   keeps the line-based sparsity the paper calls for in 3-D (PAPER.md:741-746,
   "ADI iterations"): I - alpha_dt A~ ~ prod_d (I - alpha_dt A~_d), A~_d the
   couplings of A~ along direction-d lines (node-diagonal blocks split evenly
   over the D directions), one dense (p+1)m LU per line: D (p+1)^(D-1) blocks
   of ((p+1)m)^2 per element (C4: 40 GB).  LDG_ERR_CONFIG when the factors do
   not fit the free device memory, LDG_ERR_SOLVER for a singular block.
   Replaces build_preconditioner(blocks, alpha_dt). */
int ldg_precond_build(ldg_ctx* ctx, double alpha_dt);
/* Preconditioner mode: 0 (default) element-block LU (triangular solves per
   apply) where the element has <= 128 unknowns, line-ADI above; 1 element-
   block LU that also forms the explicit block inverses (build ~4x slower,
   apply ~2x faster: a dense block matvec at HBM rate) -- pays off when one
   build serves many applications; 2 line-ADI for any configuration.
   Invalidates a built preconditioner. */
int ldg_set_precond_mode(ldg_ctx* ctx, int mode);
/* z = (I - alpha_dt A~)^-1 r, device vectors (reference numbering). */
int ldg_precond_apply(ldg_ctx* ctx, const double* r, double* z);
int ldg_precond_apply_host(ldg_ctx* ctx, const double* r, double* z);
/* Right-preconditioned restarted GMRES with modified Gram-Schmidt
   (SPEC.md:429-437): solves (I - alpha_dt (K11 + K12 K21)) x = b with the split
   matvec as operator and, if use_precond, the block-Jacobi preconditioner;
   x0 = 0.  Returns when ||b - A x|| <= rtol ||b|| or after maxit iterations
   (never an error on stagnation); LDG_ERR_SOLVER on non-finite Krylov vectors.
   iters/converged/resnorm (true residual norm) are outputs.  Replaces
   gmres(operator, precond, b, rtol, maxit, restart). */
int ldg_gmres(ldg_ctx* ctx, double alpha_dt, const double* b, double* x, double rtol, int32_t maxit,
               int32_t restart, int32_t use_precond, int32_t* iters, int32_t* converged, double* resnorm);
int ldg_gmres_host(ldg_ctx* ctx, double alpha_dt, const double* b, double* x, double rtol, int32_t maxit,
                           int32_t restart, int32_t use_precond, int32_t* iters, int32_t* converged,
                           double* resnorm);
/* Time integration.
   rk4_step: classical explicit RK4 on dU/dt = R(U).  dirk3_step: the paper's
   L-stable three-stage third-order DIRK (alpha = 0.435866521508459), stage
   slopes K_i solved by Newton on K - R(U_n + dt (sum_{j<i} a_ij K_j + alpha K))
   with the shift form (I - alpha dt A) dK = -(K - R); each linear solve is
   gmres_iters iterations of (block-Jacobi preconditioned) GMRES.  Jacobian
   reuse: the context's assembled Jacobian is kept across
   stages and steps and reassembled (at the current stage state) only when a
   stage's Newton count reaches recompute_threshold, or when none exists; the
   preconditioner is rebuilt when the Jacobian or alpha dt changes.  U is a
   device vector updated in place.  Step failure (max_newton reached) ->
   LDG_ERR_SOLVER; non-finite stages -> LDG_ERR_PHYSICAL_STATE / LDG_ERR_SOLVER. */
typedef struct ldg_newton_cfg {
  int32_t gmres_iters;         /* GMRES iterations per Newton update (paper: 5) */
  int32_t recompute_threshold; /* Newton iterations of one stage solve before reassembly (paper: 15) */
  int32_t max_newton;          /* cap per stage solve */
  int32_t use_precond;         /* block-Jacobi (1) or none (0) */
  double newton_tol;           /* stage converged when ||K - R(U_stage)||_inf <= newton_tol */
} ldg_newton_cfg;
typedef struct ldg_solver_stats {
  int32_t newton_iters;        /* Newton updates over the step, all stages */
  int32_t gmres_iters;         /* GMRES iterations over the step */
  int32_t jacobian_assemblies; /* Jacobian (re)assemblies during the step */
  int32_t residual_evals;      /* residual evaluations during the step */
  double residual_norm;        /* final ||K - R||_inf of the last stage */
} ldg_solver_stats;
int ldg_rk4_step(ldg_ctx* ctx, double* U, double t, double dt);
/* Pseudo-transient continuation to a steady state (PAPER.md:
   641-652 "a sequence of increasing timesteps dt and a final step without the
   time derivatives", backward Euler): linearised backward-Euler updates
   (I - dt A) dU = dt R(U) with dt = dt0, dt0*growth, ... (n_steps of them),
   then Newton updates with dt = dt_final (default 1e12: the identity term is
   negligible, i.e. pure Newton on R(U) = 0), each linear solve gmres_iters
   iterations of (block-Jacobi) GMRES or fewer when ||b - A x|| <= gmres_rtol ||b||;
   Jacobian reused until recompute_threshold updates have been made with it.
   Converged when ||R(U)||_inf <= newton_tol (checked first: a steady U0 returns
   after one residual).  A continuation update that produces a non-physical
   state or grows the residual 1e4-fold is rejected: U restored, dt halved,
   Jacobian refreshed (at most 10 times).  A rejected final-phase
   update, or no convergence after n_steps + max_newton updates -> LDG_ERR_SOLVER.  U: device vector,
   updated in place.  log_csv (optional, host path): one row per update
   `step,stage,newton_iters,gmres_iters,jacobian_refreshed,residual_norm`
   (stage 0 = continuation, 1 = final Newton, 2 = rejected). */
typedef struct ldg_steady_cfg {
  double dt0;                  /* first pseudo-time step (> 0) */
  double growth;               /* dt_{k+1} = growth * dt_k (>= 1; SPEC default ramp: 2) */
  int32_t n_steps;             /* continuation updates (SPEC default 10) */
  double dt_final;             /* final-phase step (<= 0: 1e12) */
  int32_t gmres_iters;         /* GMRES iterations per update (cap) */
  double gmres_rtol;           /* GMRES early exit (0: run gmres_iters) */
  int32_t recompute_threshold; /* updates per Jacobian */
  int32_t max_newton;          /* final-phase update cap */
  int32_t use_precond;         /* block-Jacobi (1) or none (0) */
  double newton_tol;           /* ||R(U)||_inf target */
  const char* log_csv;         /* per-update CSV rows, or NULL */
} ldg_steady_cfg;
int ldg_steady_solve(ldg_ctx* ctx, double* U, double t, const ldg_steady_cfg* cfg, ldg_solver_stats* stats);
int ldg_dirk3_step(ldg_ctx* ctx, double* U, double t, double dt, const ldg_newton_cfg* cfg,
                   ldg_solver_stats* stats);

/* Export of the node pattern (host arrays of nnzb int64) and block values
 * (host array nnzb*block_rows*block_cols, row-major blocks), reference numbering.
 * Any pointer may be NULL. */
int ldg_export_blocks(ldg_ctx* ctx, int which, int64_t* rows, int64_t* cols, double* vals);

/* Same, restricted to the rows of the listed reference elements (all if
 * elems == NULL); *nnzb_out receives the number of blocks written.         */
int ldg_export_blocks_subset(ldg_ctx* ctx, int which, const int32_t* elems, int32_t n_elems,
                             int64_t* rows, int64_t* cols, double* vals, int64_t* nnzb_out);

/* Wire formats: matrix export as text triplets `i j value`, one
 * structural scalar entry per line (K11: every entry of every node block; K12:
 * all but the Navier-Stokes density row; K21: the component diagonal), 0-based
 * indices in the reference numbering (rows: DOF (e*npe+node)*m+c, or the Q
 * index for K21), ascending rows, %.17g values.  Replaces the reference's
 * triplet dump of a CscMatrix. */
int ldg_write_triplets(ldg_ctx* ctx, int which, const char* path);
/* Sparsity summary CSV `p,avg_cols_per_block_row,nnz`:
 * node-columns per node row (the Table-1 quantity) and the
 * structural scalar nonzeros of one matrix; append != 0 adds a row (header
 * only when the file is empty). */
int ldg_write_sparsity_csv(ldg_ctx* ctx, int which, const char* path, int append);

/* Error synchronisation.  By default every device entry point waits for its
 * kernels and reports a physical-state failure synchronously, like the
 * reference's exceptions.  ldg_set_sync_errors(ctx, 0) makes the device entry
 * points fully asynchronous (stream-ordered); ldg_synchronize() then waits and
 * reports any failure recorded since the last check.                       */
int ldg_set_sync_errors(ldg_ctx* ctx, int on);
int ldg_synchronize(ldg_ctx* ctx);

/* Host-buffer variants (end-to-end path: H2D, kernels, D2H).  With error
 * synchronisation on (default) each call synchronises before returning.  With
 * ldg_set_sync_errors(ctx, 0), ldg_residual_host / ldg_jacobian_assemble_host /
 * ldg_residual_assemble_host / ldg_bsr_spmv_host / ldg_split_matvec_host (two
 * staging slots) are asynchronous: uploads run on a copy stream, downloads
 * on another, ordered against the kernels by events (transfers of consecutive
 * calls overlap the kernels in both PCIe directions); the host buffers must
 * stay valid (pinned for overlap) and results are ready after ldg_synchronize.
 * ldg_bsr_spmv_host(K11) with y in mapped pinned memory (cudaHostAlloc /
 * cudaHostRegister under unified addressing) and m = 4 is zero-copy: the
 * product kernel writes y over PCIe while it runs (LDG_OPT_ZERO_COPY).        */
int ldg_residual_host(ldg_ctx* ctx, const double* U, double t, double* R, double* Q_or_null);
int ldg_jacobian_assemble_host(ldg_ctx* ctx, const double* U, double t);
/* gradient_residual / residual_second_order on host buffers (synchronous). */
int ldg_gradient_host(ldg_ctx* ctx, const double* U, double t, double* Q);
int ldg_residual_uq_host(ldg_ctx* ctx, const double* U, const double* Q, double t, double* R);
/* R(U) and the Jacobian at U from one upload of U (a Newton step): second-
 * order physics computes Q = D(U) once for both (Q_or_null receives it). */
int ldg_residual_assemble_host(ldg_ctx* ctx, const double* U, double t, double* R, double* Q_or_null);
int ldg_bsr_spmv_host(ldg_ctx* ctx, int which, const double* x, double* y);
int ldg_split_matvec_host(ldg_ctx* ctx, double alpha_dt, const double* v, double* y);

/* Execution options (defaults chosen by measurement).
 *   LDG_OPT_SPMV_ROW_ORDER  block-SpMV / split-matvec row walk: 0 auto (reverse
 *                           row order for K11 stores <= 1 GiB, whose tail is
 *                           still L2-resident after the assembly), 1 forward,
 *                           2 reverse.  Results are bitwise independent of it.
 *   LDG_OPT_ZERO_COPY       1 (default): ldg_bsr_spmv_host(K11) writes y
 *                           straight into mapped pinned memory; 0: staged copy.
 * Returns LDG_ERR_INVALID_ARGUMENT for an unknown option or value.          */
enum { LDG_OPT_SPMV_ROW_ORDER = 1, LDG_OPT_ZERO_COPY = 2 };
int ldg_set_option(ldg_ctx* ctx, int option, int64_t value);

/* Instrumentation: number of kernel launches issued by this context so far,
 * and the device-side byte footprint of the Jacobian store. */
int64_t ldg_kernel_launches(const ldg_ctx* ctx);
int64_t ldg_jacobian_bytes(const ldg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* LINEDG_B200_H */
