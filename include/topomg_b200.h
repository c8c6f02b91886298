/*
 * topomg_b200.h -- C ABI of the B200-native MG-PCG hot path.
 *
 * Drop-in boundary for the reference's solver/preconditioner interface
 * (reference package `topomg`, /root/reference/pkg/src/topomg).  The reference
 * is Python, so the binding a maintainer adds is a ctypes stub;
 * paper_2001_01655_b200/_lib.py is exactly that stub.  Each entry point names
 * the reference function it replaces.
 *
 * Conventions
 *   - All vector arguments named *_dev are DEVICE pointers (fp64, DOF-interleaved:
 *     dof = node*dofs_per_node + component, nodes lexicographic with x fastest,
 *     exactly the reference numbering, mesh.py:15-111).
 *   - Arguments named *_host are host pointers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Every function returns 0 on success and a negative code on failure;
 *     tmg_last_error() then holds a message (thread-local).  Invalid arguments
 *     that the reference rejects with ValueError return TMG_EINVAL; an index
 *     out of range (the reference's IndexError) returns TMG_ERANGE.
 *   - There is no CPU fallback: without a CUDA device every compute entry point
 *     returns TMG_ENODEV.
 */
#ifndef TOPOMG_B200_H
#define TOPOMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_OK 0
#define TMG_EINVAL (-1)  /* reference raises ValueError            */
#define TMG_ERANGE (-2)  /* reference raises IndexError            */
#define TMG_ECUDA (-3)   /* CUDA runtime failure                    */
#define TMG_ENODEV (-4)  /* no CUDA device: the product never falls back to the CPU */
#define TMG_ESTATE (-5)  /* solver failure (e.g. non-SPD coarse operator) */

typedef struct tmg_operator tmg_operator;   /* K(rho) on a structured grid   */
typedef struct tmg_hierarchy tmg_hierarchy; /* MgHierarchy                    */

/* StructuredMesh (mesh.py:15): element counts per axis + element edge lengths. */
typedef struct {
  int32_t ndim;      /* 2 (Q4, plane stress) or 3 (Hex8) */
  int32_t dims[3];   /* elements per axis (dims[2] ignored in 2D) */
  double h[3];       /* element edge lengths */
} tmg_mesh_desc;

/* SmootherConfig (multigrid.py:30).  kind: 0 weighted_jacobi, 1 block_jacobi,
 * 2 chebyshev (Jacobi-preconditioned Chebyshev of degree inner_iterations with a
 * lanczos_steps-step Lanczos bound; extension required by BASELINE.json),
 * 3 sor_chebyshev (multigrid.py:109), 4 sor_gmres (multigrid.py:153). */
typedef struct {
  int32_t kind;
  double weight;
  int32_t inner_iterations;
  int32_t lanczos_steps;
  uint64_t seed;
  double safeguard;  /* weighted_jacobi only: >0 caps the weight of every level at
                        safeguard/lambda_hat(D^-1 A) (Lanczos); 0 = reference behaviour */
  const double* power_start; /* sor_chebyshev only: the power-method start vector of
                        multigrid.py:119, numpy.random.default_rng(0).standard_normal(ndofs)
                        of the finest level (coarser levels use its prefix); host or
                        device pointer, copied during the build */
} tmg_smoother_desc;

/* SolveConfig (krylov.py:17).  tmg_pcg_solve reads rtol / max_iterations; the
 * host-buffer entry tmg_solve_compliance_host also dispatches on method like
 * SolverHarness.solve (optimization.py:90-95): 0 CG (extension, zero-initialised
 * default of this C struct; refused with TMG_EINVAL for the non-stationary
 * sor_chebyshev / sor_gmres smoothers), 1 gmres_solve (FGMRES when the smoother
 * is non-stationary, as the reference), 2 fgmres_solve, with restart (<= 0: the
 * reference's 200).  The Python SolveConfig keeps the reference's defaults
 * (gmres, rtol 1e-7). */
typedef struct {
  double rtol;            /* ||r|| <= rtol * ||b||, as krylov.py:63 */
  int32_t max_iterations;
  int32_t method;
  int32_t restart;
} tmg_solve_desc;

/* SolveRecord (krylov.py:31).  `converged` and `final_residual` follow the
 * reference's contract (krylov.py:124-129): the TRUE residual ||b - A x|| of the
 * returned iterate against rtol * ||b||; residual_history ends on it.  PCG
 * restarts from the true residual after a false convergence of its recursive
 * residual (`restarts`). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double initial_residual;
  double final_residual;      /* true residual at exit */
  double solve_ms;            /* device time of the solve (CUDA events) */
  double recursive_residual;  /* PCG: recursively updated residual at exit (GMRES: = final) */
  int32_t restarts;           /* PCG: cycles restarted after a false convergence (GMRES: 0) */
  int32_t reserved;
} tmg_solve_record;

/* hierarchy level description (MgHierarchy.summary, multigrid.py:247) */
typedef struct {
  int64_t size;        /* rows of the level operator */
  int64_t nonzeros;    /* stored scalar entries */
  int32_t provenance;  /* 0 geometric, 1 algebraic */
  int32_t storage;     /* 0 matrix-free element, 1 structured stencil, 2 BSR, 3 dense inverse */
} tmg_level_info;

const char* tmg_last_error(void);
int tmg_version(void);
int tmg_device_count(void);
/* Number of this library's kernel launches so far (CUDA-graph replays included). */
int64_t tmg_launch_count(void);

/* mesh.py:254 element_stiffness -> row-major (4|8)*ndim square matrix. Host only. */
int tmg_element_stiffness(const tmg_mesh_desc* mesh, double E, double nu, double* ke_host);

/* material.py:175 SimpLaw.modulus on the device: E = emin + (e0-emin)*rho^p. */
int tmg_simp_modulus(const double* rho_dev, int64_t n, double penalty, double e0, double emin,
                     double* E_dev, void* stream);

/* mesh.py:327 assemble_stiffness(mesh, bc, element_moduli): the operator is kept
 * matrix-free (element moduli + KE); fixed dofs are eliminated symmetrically with a
 * unit diagonal exactly as mesh.py:313.  fixed_dofs_host may contain duplicates.
 * The moduli are copied; the caller's buffer may be freed afterwards. */
int tmg_operator_create(const tmg_mesh_desc* mesh, const double* element_moduli_dev,
                        const int64_t* fixed_dofs_host, int64_t n_fixed, double nu,
                        void* stream, tmg_operator** out);
int tmg_operator_destroy(tmg_operator* op);
int64_t tmg_operator_size(const tmg_operator* op);
/* y = K x  (K @ x in the reference) */
int tmg_operator_apply(tmg_operator* op, const double* x_dev, double* y_dev, void* stream);
/* K.diagonal() */
int tmg_operator_diagonal(tmg_operator* op, double* d_dev, void* stream);

/* multigrid.py:318 build_gmg(mesh, K, coarse_max_dofs, smoother, n_pre, n_post).
 * max_levels <= 0 means no cap (reference behaviour). */
int tmg_gmg_build(tmg_operator* K, int64_t coarse_max_dofs, int32_t max_levels,
                  const tmg_smoother_desc* smoother, int32_t n_pre, int32_t n_post,
                  void* stream, tmg_hierarchy** out);
/* multigrid.py:555 build_sa_amg(K, near_nullspace, coarse_max_dofs, smoother, n_pre,
 * n_post, seed).  near_nullspace_host: row-major (ndofs x nvec), nvec 3 (2D) or 6
 * (3D).  beta: strength threshold (reference: 0.003, multigrid.py:22).
 * v0_host: the power-method start vector numpy.random.default_rng(seed)
 * .standard_normal(ndofs) of multigrid.py:509 (deeper levels use its prefix).
 * Both arrays may be host or device pointers (copied with cudaMemcpyDefault). */
int tmg_sa_amg_build(tmg_operator* K, const double* near_nullspace_host, int32_t nvec,
                     int64_t coarse_max_dofs, double beta, const double* v0_host,
                     const tmg_smoother_desc* smoother, int32_t n_pre, int32_t n_post,
                     int32_t isolated_mode, void* stream, tmg_hierarchy** out);
/* isolated_mode 0: reference behaviour (multigrid.py:418-423, 457-467: strength-
 * isolated nodes become singletons that the fallback folds into one aggregate);
 * 1 (extension): they stay unaggregated (zero rows of T), PyAMG-style. */
/* multigrid.py:573 build_hybrid(mesh, K, near_nullspace, n_geo, ...) for n_geo >= 1:
 * coarse_near_nullspace_host = rigid_body_modes(coarse_mesh) of the mesh reached
 * after the geometric levels (coarse_ndof rows), v0_host its start vector. */
int tmg_hybrid_build(tmg_operator* K, int32_t n_geo, const double* coarse_near_nullspace_host,
                     int64_t coarse_ndof, int32_t nvec, int64_t coarse_max_dofs, double beta,
                     const double* v0_host, const tmg_smoother_desc* smoother, int32_t n_pre,
                     int32_t n_post, int32_t isolated_mode, void* stream, tmg_hierarchy** out);
/* MgHierarchy.flags as a comma-separated list. */
int tmg_hierarchy_flags(const tmg_hierarchy* h, char* buf, int32_t cap);
/* Export level data for parity checks (two-call: NULL buffers return dims only).
 * what: 0 level operator (BSR; lattice levels converted), 1 smoothed P, 2 strength
 * graph (rowptr/col), 3 aggregate ids (col; val[0] = rho(D^-1 A)), 4 tentative T.
 * dims = {block rows, block cols (n_agg for 3), nnz blocks, R*1000+C}. */
int tmg_hierarchy_export(tmg_hierarchy* h, int32_t level, int32_t what, int64_t* dims,
                         int32_t* rowptr, int32_t* col, double* val, void* stream);
int tmg_hierarchy_destroy(tmg_hierarchy* h);
int tmg_hierarchy_num_levels(const tmg_hierarchy* h);
int tmg_hierarchy_level_info(const tmg_hierarchy* h, int32_t level, tmg_level_info* info);
/* multigrid.py:231 MgHierarchy.vcycle(b, k) (zero initial guess). */
int tmg_hierarchy_vcycle(tmg_hierarchy* h, int32_t level, const double* b_dev, double* x_dev,
                         void* stream);
/* multigrid.py:179 make_smoother(config, K): the finest level's smoother alone
 * (no coarse levels; tmg_hierarchy_vcycle / the solvers reject it). */
int tmg_smoother_create(tmg_operator* K, const tmg_smoother_desc* smoother, void* stream,
                        tmg_hierarchy** out);
/* The smoother's apply(x, b, passes) on a level (multigrid.py:57/90/131/161):
 * x_dev in/out; levels below the coarsest of a V-cycle hierarchy. */
int tmg_hierarchy_smooth(tmg_hierarchy* h, int32_t level, const double* b_dev, double* x_dev,
                         int32_t passes, void* stream);
/* y = A^level x (the Galerkin operator of a level), for parity checks. */
int tmg_hierarchy_level_apply(tmg_hierarchy* h, int32_t level, const double* x_dev,
                              double* y_dev, void* stream);
/* Chebyshev eigenvalue estimate of a level (NaN unless the smoother is chebyshev). */
int tmg_hierarchy_level_lmax(tmg_hierarchy* h, int32_t level, double* lmax_host, void* stream);

/* Average device time (ms) of one smoother sweep kernel of a level (weighted/block
 * Jacobi sweep or one Chebyshev step): `reps` launches captured into one CUDA graph
 * and timed with CUDA events as one replay (back to back, as inside the PCG graph).
 * Used by bench.py for the roofline of the dominant kernel. */
int tmg_hierarchy_time_smoother(tmg_hierarchy* h, int32_t level, int32_t reps, double* ms_host,
                                void* stream);
/* Same for one V-cycle started at `level` (diagnostics: per-level cost split). */
int tmg_hierarchy_time_vcycle(tmg_hierarchy* h, int32_t level, int32_t reps, double* ms_host, void* stream);
/* Same for one V-cycle phase of `level` (diagnostics): the residual, the
 * restriction to level+1, the prolongation-add from level+1, or (last level
 * only) the coarsest solve. */
enum { TMG_PHASE_RESIDUAL = 0, TMG_PHASE_RESTRICT = 1, TMG_PHASE_PROLONG = 2, TMG_PHASE_COARSE = 3 };
int tmg_hierarchy_time_phase(tmg_hierarchy* h, int32_t level, int32_t phase, int32_t reps, double* ms_host,
                             void* stream);

/* Preconditioned CG (extension; krylov.py:134 is the reference's GMRES entry).
 * h may be NULL (unpreconditioned).  x_dev holds x0 on entry when use_x0 != 0
 * and the solution on return.  residual_history_host (may be NULL) receives
 * iterations+1 norms. Synchronises the stream once at the end. */
int tmg_pcg_solve(tmg_operator* K, tmg_hierarchy* h, const double* b_dev, double* x_dev,
                  int32_t use_x0, const tmg_solve_desc* cfg, double* residual_history_host,
                  tmg_solve_record* rec, void* stream);

/* Right-preconditioned restarted GMRES / flexible GMRES (krylov.py:48-143, the
 * reference's default SolverHarness method).  Convergence, Givens rotations,
 * restarts, breakdown (1e-14) and the residual history follow krylov.py; the
 * Arnoldi step orthogonalises with CGS2 on the device.
 * residual_history_host (may be NULL) receives iterations+1 norms (capacity
 * max_iterations+1). */
typedef struct {
  double rtol;
  int32_t max_iterations;
  int32_t restart;
  int32_t flexible;  /* 1: fgmres_solve (stores the preconditioned basis) */
} tmg_gmres_desc;
int tmg_gmres_solve(tmg_operator* K, tmg_hierarchy* h, const double* b_dev, double* x_dev,
                    int32_t use_x0, const tmg_gmres_desc* cfg, double* residual_history_host,
                    tmg_solve_record* rec, void* stream);

/* optimization.py:106 element_strain_energies: ce_e = u_e^T KE u_e (unit modulus). */
int tmg_strain_energy(tmg_operator* K, const double* u_dev, double* ce_dev, void* stream);
/* optimization.py:128-129: dc_e = -p (e0-emin) rho_e^(p-1) ce_e, compliance = f.u */
int tmg_compliance_sensitivity(tmg_operator* K, const double* rho_dev, const double* f_dev,
                               const double* u_dev, double penalty, double e0, double emin,
                               double* dc_dev, double* compliance_host, void* stream);
/* Average device time (ms) of the fused compliance + sensitivity kernel: `reps`
 * launches in one CUDA graph, rotating over three copies of u and f so that they
 * stream from HBM (bench.py's `sensitivity` entry; a measurement helper like
 * tmg_hierarchy_time_smoother, it replaces no reference function). */
int tmg_operator_time_sensitivity(tmg_operator* K, const double* rho_dev, const double* f_dev,
                                  const double* u_dev, double penalty, double e0, double emin,
                                  double* dc_dev, int32_t reps, double* ms_host, void* stream);

/* End-to-end drop-in for compliance_and_sensitivity (optimization.py:114) given the
 * filtered densities: HOST buffers in and out; H2D copies, modulus, operator,
 * hierarchy (gmg / amg / hybrid), PCG solve, sensitivity and D2H copies all inside. */
typedef struct {
  int32_t strategy;          /* 0 gmg, 1 amg (smoothed aggregation), 2 hybrid */
  int64_t coarse_max_dofs;
  int32_t max_levels;        /* gmg only; <= 0: no cap */
  tmg_smoother_desc smoother;
  int32_t n_pre, n_post;
  int32_t n_geo;             /* hybrid */
  double beta;               /* amg/hybrid strength threshold */
  const double* near_nullspace_host;  /* amg: ndofs x nvec; hybrid: coarse_ndof x nvec */
  int32_t nvec;
  int64_t coarse_ndof;       /* hybrid: rows of near_nullspace_host */
  const double* v0_host;     /* amg/hybrid power-method start vector */
  int32_t isolated_mode;     /* amg/hybrid: 0 reference merge, 1 drop (see tmg_sa_amg_build) */
} tmg_mg_desc;
int tmg_solve_compliance_host(const tmg_mesh_desc* mesh, const double* rho_host,
                              const int64_t* fixed_dofs_host, int64_t n_fixed,
                              const double* f_host, double penalty, double e0, double emin,
                              double nu, const tmg_mg_desc* mg, const tmg_solve_desc* cfg,
                              double* u_host, double* dc_host, double* compliance_host,
                              tmg_solve_record* rec);

#ifdef __cplusplus
}
#endif
#endif /* TOPOMG_B200_H */
