/*
 * pba_gpu.h — C ABI of the B200 (sm_100a) photometric-bundle-adjustment hot path.
 *
 * This is the drop-in boundary for the per-iteration PBA step of arXiv 1704.06967
 * (inverse compositional with proxy templates = "IC", forwards compositional = "FC").
 * Every entry point replaces one responsibility of the reference C++ solver API in
 * /root/reference/proj/include/pba/solver.hpp; the replaced interface is cited on
 * each declaration (reference paths are relative to /root/reference/proj/).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Host arrays passed in are borrowed for the
 *    duration of the call; output arrays are caller-allocated.
 *  - A handle owns one CUDA stream and all device buffers of one problem
 *    (the reference's ProblemState, taken by value: solver.hpp:117,176).  A handle
 *    must be used by one host thread at a time (the reference IcSolver is not
 *    thread-safe either).  Every call is synchronous at return.
 *  - Status codes replace the reference's exception classes (errors.hpp:9-40);
 *    pba_gpu_last_error() returns the message the reference would have thrown.
 *  - Poses map reference-frame points into the target frame: X_t = R X_ref + t
 *    (geometry.hpp:22-28).  R is 3x3 row-major.
 *  - Residual / active arrays are indexed  o*P + k  where o is the observation
 *    index (point-major, frames ascending).  For the dense problem (obs_ptr==NULL)
 *    o = n*F + f, i.e. exactly the reference's (n*F + f)*P + k (solver.hpp:101).
 */
#ifndef PBA_GPU_H
#define PBA_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-40) --------------------------------------- */
enum {
  PBA_OK = 0,
  PBA_E_EMPTY_PROBLEM = 1,     /* pba::EmptyProblem    errors.hpp:32-35 */
  PBA_E_OUT_OF_BOUNDS = 2,     /* pba::OutOfBounds     errors.hpp:26-29 */
  PBA_E_INVALID_DEPTH = 3,     /* pba::InvalidDepth    errors.hpp:20-23 */
  PBA_E_DEGENERATE_DEPTH = 4,  /* pba::DegenerateDepth errors.hpp:14-17 */
  PBA_E_SINGULAR_HESSIAN = 5,  /* pba::Error("SingularHessian: ...") solver.cpp:192,401 */
  PBA_E_CUDA = 6,              /* CUDA runtime failure (no CPU fallback exists) */
  PBA_E_ARG = 7,               /* invalid argument */
  PBA_E_STATE = 8,             /* call-order error (e.g. IC step before build) */
  PBA_E_SPEC_INFEASIBLE = 9    /* pba::SpecInfeasible  errors.hpp:38-40 (scene generators) */
};

typedef struct pba_handle pba_handle;

/* ---- problem description (ProblemState, solver.hpp:33-43) ------------------ */
typedef struct pba_image {
  int32_t width, height;
  double fx, fy, cx, cy;       /* Intrinsics, image.hpp:14-23 */
  const float* data;           /* row-major width*height texels (fp32) */
} pba_image;

typedef struct pba_problem {
  pba_image ref;               /* ProblemState::ref */
  int32_t num_frames;          /* F */
  const pba_image* targets;    /* F target images */
  const double* pose_R;        /* F*9 */
  const double* pose_t;        /* F*3 */
  int32_t num_points;          /* N */
  const double* anchors_px;    /* N*2 (u, v) reference pixels */
  const double* inv_depths;    /* N, > 0 */
  int32_t pattern_size;        /* P in [1, 32] */
  const int32_t* pattern;      /* P*2 integer offsets; pattern[0] must be (0,0) (solver.cpp:116,311) */
  /* Observation-list extension (visibility masks / C4-C5
     storage).  NULL => dense: every point observed in every frame. */
  const int64_t* obs_ptr;      /* N+1 CSR offsets */
  const int32_t* obs_frame;    /* obs_ptr[N] frame ids, strictly increasing per point */
} pba_problem;

/* ---- SolverConfig (solver.hpp:45-54) --------------------------------------- */
typedef struct pba_config {
  double gamma;                /* Huber threshold (0.03 in [0,1] units) */
  double threshold_px;         /* convergence: max reprojected update */
  int32_t max_iters;
  double lambda0;              /* Levenberg damping floor */
  int32_t max_bad_steps;
  int32_t normalize_depth_gauge;
  int32_t refresh_ic_hessian;
  int32_t record_snapshots;
} pba_config;

/* IterationStats (solver.hpp:71-80) */
typedef struct pba_iter_stats {
  int32_t iter;
  double energy;
  double max_update_px;
  double wall_ms;              /* cumulative solver time */
  int32_t hessian_builds;      /* cumulative */
  int32_t hessian_factorizations;
  int64_t num_active;          /* extension: active residuals of the accepted pass */
  int32_t accepted;            /* extension: 1 if the iteration's step was accepted */
} pba_iter_stats;

/* SolveReport (solver.hpp:82-97).  Pointer members are caller-allocated and may
   be NULL; iters_capacity bounds both iters[] and the snapshot arrays. */
typedef struct pba_report {
  int32_t converged, diverged, iterations;
  int32_t hessian_builds, hessian_factorizations, rejected_steps;
  double final_energy, total_wall_ms;
  int64_t masked_residuals;
  double* final_R;             /* F*9 */
  double* final_t;             /* F*3 */
  double* final_inv_depths;    /* N */
  pba_iter_stats* iters;       /* iters_capacity entries */
  int32_t iters_capacity;
  int32_t num_iters;           /* filled by the call */
  double* snap_R;              /* iters_capacity*F*9, when record_snapshots */
  double* snap_t;              /* iters_capacity*F*3 */
  double* snap_d;              /* iters_capacity*N   */
  char message[256];           /* SolveReport::message */
} pba_report;

/* EnergyResult (solver.hpp:99-105) scalars */
typedef struct pba_energy_result {
  double energy;
  int64_t num_active;
  int64_t num_out_of_bounds;
} pba_energy_result;

/* ---- generic ---------------------------------------------------------------- */
const char* pba_status_string(int status);
void pba_config_default(pba_config* cfg);                 /* SolverConfig{} defaults */
/* perturb_parameters (synth.cpp:308-320), host only: R (9F), t (3F), d (N) in place; the
   std::mt19937_64 / std::normal_distribution stream of the reference CLI's `solve` (pba.cpp:62). */
int pba_perturb_parameters(int32_t F, double* R, double* t, int32_t N, double* d, double sigma, uint64_t seed);

/* ---- handle lifecycle: IcSolver(ProblemState, SolverConfig) solver.hpp:117,
   FcSolver(ProblemState, SolverConfig) solver.hpp:176.  Uploads the problem. */
int pba_gpu_create(const pba_problem* problem, pba_handle** out);
/* As pba_gpu_create, but it returns without waiting for the tail of the target-image upload: the
   caller keeps problem->targets[*].data valid until the first call on the handle that reads them
   (energy, ic_build, ic_run / fc_run, ic_begin / fc_begin, fc_build) returns.  ic_solve / fc_solve
   (solver.cpp:845-851) hold their ProblemState for the whole call, so they use this. */
int pba_gpu_create_deferred(const pba_problem* problem, pba_handle** out);
void pba_gpu_destroy(pba_handle* h);
const char* pba_gpu_last_error(const pba_handle* h);
int64_t pba_gpu_num_observations(const pba_handle* h);   /* N_obs */

/* ProblemState::poses / inv_depths (replace or read the problem's parameters) */
int pba_gpu_set_params(pba_handle* h, const double* R, const double* t, const double* inv_depths);
int pba_gpu_get_params(pba_handle* h, double* R, double* t, double* inv_depths);

/* energy_eval(state, huber, mask)  solver.hpp:110-111, solver.cpp:229-244.
   mask: NULL or N_obs*P bytes.  residuals/active: NULL or N_obs*P outputs. */
int pba_gpu_energy(pba_handle* h, double gamma, const uint8_t* mask,
                   pba_energy_result* out, double* residuals, uint8_t* active);

/* ---- IcSolver (solver.hpp:115-169) ------------------------------------------- */
int pba_gpu_ic_build(pba_handle* h, const pba_config* cfg);       /* IcSolver::build  solver.cpp:254-368 */
int pba_gpu_ic_gradient(pba_handle* h, double* g);                /* IcSolver::gradient solver.cpp:470-473, 6F+N */
int pba_gpu_ic_compute_step(pba_handle* h, double* dx);           /* IcSolver::compute_step solver.cpp:475-479 */
int pba_gpu_ic_solve_step(pba_handle* h, const double* g, double* dx); /* IcSolver::solve_step solver.cpp:404-434 */
int pba_gpu_ic_factorize(pba_handle* h, double lambda);           /* IcSolver::factorize solver.cpp:370-402 */
/* IcSolver::hessian() solver.hpp:129 — BlockHessian blocks (solver.hpp:59-69):
   pose_pose F*36 row-major, depth_depth N, pose_depth N_obs*6, lambda. */
int pba_gpu_ic_hessian(pba_handle* h, double* pose_pose, double* depth_depth,
                       double* pose_depth, double* lambda);
int pba_gpu_warning_count(const pba_handle* h);                   /* IcSolver::warnings() solver.hpp:130 */
int pba_gpu_warning(const pba_handle* h, int i, char* buf, int len);
/* All warnings at once, '\n'-separated and NUL-terminated (truncated to len - 1 bytes);
   returns the full length excluding the NUL.  Bulk form of warnings() for large problems. */
int64_t pba_gpu_warnings_text(const pba_handle* h, char* buf, int64_t len);
/* The zero-depth-Hessian warnings (solver.cpp:359-364, "point <i>: zero depth Hessian entry
   (unobservable depth)") are the last pba_gpu_warning_points() entries of warnings(), in
   ascending user point order: copies up to cap point indices into idx and returns how many
   there are.  Lets a binding format them on demand instead of parsing the bulk text. */
int64_t pba_gpu_warning_points(const pba_handle* h, int32_t* idx, int64_t cap);
int pba_gpu_ic_run(pba_handle* h, const pba_config* cfg, pba_report* rep); /* IcSolver::run / ic_solve solver.cpp:481-654,845-847 */

/* ---- FcSolver (solver.hpp:172-182) ------------------------------------------- */
/* One FC Hessian/gradient build at the problem's parameters (solver.cpp:688-724). */
int pba_gpu_fc_build(pba_handle* h, double gamma, double* pose_pose, double* depth_depth,
                     double* pose_depth, double* g);
int pba_gpu_fc_run(pba_handle* h, const pba_config* cfg, pba_report* rep); /* FcSolver::run / fc_solve solver.cpp:663-851 */

/* ---- stepping interface: the body of IcSolver::run / FcSolver::run split at the
   iteration boundary (for callers that interleave their own work, e.g. a DSO
   front end, and for benchmarking).  *_run == begin + iterate until done + end. */
int pba_gpu_ic_begin(pba_handle* h, const pba_config* cfg);
int pba_gpu_fc_begin(pba_handle* h, const pba_config* cfg);
int pba_gpu_iterate(pba_handle* h, pba_iter_stats* stats, int* done);
int pba_gpu_end(pba_handle* h, pba_report* rep);

/* ---- free function solve_normal_equations_schur (solver.hpp:190-192,
   solver.cpp:165-213) over a caller BlockHessian in observation layout. */
int pba_gpu_solve_normal_equations_schur(int32_t F, int32_t N, const int64_t* obs_ptr,
                                         const int32_t* obs_frame, const double* pose_pose,
                                         const double* depth_depth, const double* pose_depth,
                                         const double* g, double lambda, double* dx);

/* ---- sub-steps of the iteration (SURVEY.md §8b export set) -------------------- */
/* Candidate update of the problem parameters by dx (6F+N).  mode 0 = IC
   (apply_ic_update geometry.cpp:197-209 with the build's p0, solver.cpp:544-560),
   mode 1 = FC (pose_boxplus geometry.cpp:93-98 + additive depth, solver.cpp:744-750).
   Writes the candidate to R/t/d outputs (problem parameters unchanged);
   *invalid = 1 when a depth became non-positive. */
int pba_gpu_apply_update(pba_handle* h, int mode, const double* dx, double* R_out,
                         double* t_out, double* d_out, int* invalid);
/* max_reprojection_update_px (solver.cpp:105-131) between the problem parameters
   and (R, t, d).  +inf when a degenerate depth is met. */
int pba_gpu_max_reproj_update(pba_handle* h, const double* R, const double* t,
                              const double* d, double* px);
/* normalize_depth_gauge (solver.cpp:135-143) applied to the problem parameters. */
int pba_gpu_normalize_gauge(pba_handle* h);

/* ---- joint multi-host window with per-frame affine brightness ----
   NOT in the reference (single reference frame, no photometric parameters: solver.hpp:33-43,
   SPEC.md:318); this is the DSO-style joint form of BASELINE C2, forwards compositional, checked
   against the oracle's statement of the same model (oracle/multihost.cpp, which gives the
   equations).  Every point is hosted in one frame; it is observed in other frames through the
   relative pose T_t T_h^-1, with r = e^(a_t - a_h) (tpl - b_h) + b_t - I_t(warp).  Frame 0 is
   held.  With every point hosted in frame 0 and the affine parameters held, a run is the
   reference's FcSolver::run (solver.cpp:663-843) on frames 1..K-1. */
typedef struct pba_mh_problem {
  int32_t num_frames;            /* K >= 2 */
  const pba_image* images;       /* K images, each with its intrinsics */
  const double* pose_R;          /* 9K row-major, X_i = R_i X_w + t_i */
  const double* pose_t;          /* 3K */
  const double* affine_a;        /* K or NULL (= 0) */
  const double* affine_b;        /* K or NULL (= 0) */
  int32_t num_points;
  const int32_t* host;           /* N: host frame of each point */
  const double* anchors_px;      /* 2N: pixels of the host image */
  const double* inv_depths;      /* N: in the host camera */
  int32_t pattern_size;          /* P <= 32 */
  const int32_t* pattern;        /* 2P offsets, pattern[0] = (0, 0) */
  const int64_t* obs_ptr;        /* N+1 CSR of target frames (each != host), or NULL = every other frame */
  const int32_t* obs_frame;
  int32_t optimize_affine;       /* 1: (a, b) of frames 1..K-1 are parameters; 0: held */
} pba_mh_problem;
typedef struct pba_mh_handle pba_mh_handle;
int pba_gpu_mh_create(const pba_mh_problem* problem, pba_mh_handle** out);
void pba_gpu_mh_destroy(pba_mh_handle* h);
const char* pba_gpu_mh_last_error(const pba_mh_handle* h);
int pba_gpu_mh_energy(pba_mh_handle* h, double gamma, pba_energy_result* out);
/* FcSolver::run rules on the joint window; rep->final_R / final_t hold all K frames,
   a_out / b_out (K, or NULL) the final affine parameters. */
int pba_gpu_mh_fc_run(pba_mh_handle* h, const pba_config* cfg, pba_report* rep, double* a_out, double* b_out);

/* ---- point-sharded runs -------------------------------------
   Each rank's handle holds a disjoint subset of the points with all of their observations;
   frames, images and poses are replicated.  The reference has no multi-process path: the
   exchange replaces the sums over n of solver.cpp (assemble_gradient :450-468, the Schur
   update :381-389, the rhs term :407-416, the gauge mean :135-143, the energy :97) by sums
   over the ranks.  Per IC iteration one all-gather of {g_f, c_f, status} (12F + 8 doubles)
   and one of the depth sum; per (re)factorization one int64 sum of the fixed-point Schur
   accumulator (36F^2, exact); FC adds H (21F) to the first.  Every rank then runs the same
   replicated pose solve and LM decisions (bitwise identical inputs), and back-substitutes
   its own depths.
   op PBA_X_GATHER: send `count` doubles at `send` (device), receive world*count doubles
   rank-major at `recv` (device).  op PBA_X_SUM_I64: in-place sum of `count` int64 at `send`.
   The callee orders the exchange after the work queued on `stream` (a cudaStream_t) and
   before the work queued there after it returns (e.g. NCCL on that stream).  0 = success.
   fn == NULL restores the single-process path. */
enum { PBA_X_GATHER = 0, PBA_X_SUM_I64 = 1 };
typedef int (*pba_exchange_fn)(void* ctx, int op, void* send, void* recv, int64_t count, void* stream);
int pba_gpu_set_exchange(pba_handle* h, int32_t rank, int32_t world, int64_t num_points_total,
                         pba_exchange_fn fn, void* ctx);
/* The same exchange issued by the library itself over NCCL (no callback per candidate): rank 0 draws a
   128-byte ncclUniqueId with pba_gpu_nccl_unique_id, the caller distributes it (any channel), and
   every rank attaches its handle; the all-gathers and the int64 sum then run on the handle's stream.
   NCCL is loaded with dlopen on first use (PBA_E_CUDA when absent). */
int pba_gpu_nccl_unique_id(void* id128);
int pba_gpu_set_exchange_nccl(pba_handle* h, const void* id128, int32_t rank, int32_t world,
                              int64_t num_points_total);

/* ---- instrumentation ------------------------------------------------------- */
void* pba_gpu_stream(pba_handle* h);                 /* the handle's cudaStream_t */
/* When on, the hot kernels are bracketed by CUDA events on the handle's stream;
   pba_gpu_kernel_times returns {count, total ms} per kernel id (pba_kernel_id). */
int pba_gpu_set_profiling(pba_handle* h, int on);
enum {
  PBA_K_OBS_PASS = 0,      /* fused per-point residual/Huber/J^T W r (+FC J^T W J) pass */
  PBA_K_SCHUR = 1,         /* reduced camera system */
  PBA_K_CHOLESKY = 2,      /* dense Cholesky of the reduced system */
  PBA_K_TRISOLVE = 3,      /* two triangular solves */
  PBA_K_IC_BUILD = 4,      /* frozen J / H build */
  PBA_K_REDUCE = 5,        /* partial-sum finalize */
  PBA_K_COUNT = 6
};
int pba_gpu_kernel_times(pba_handle* h, int64_t* counts, double* total_ms);
/* Process-wide number of kernel launches issued by this library so far. */
int64_t pba_gpu_launch_count(void);
/* Bytes of device memory held by the handle. */
int64_t pba_gpu_device_bytes(const pba_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* PBA_GPU_H */
