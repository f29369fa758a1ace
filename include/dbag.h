/*
 * dbag.h — C-ABI of the B200-native D-ADMM bundle-adjustment core
 * (arXiv 1708.07954, data-parallel hot path). Plain C: fixed-width integers,
 * doubles, opaque handles; no CUDA or torch types cross this boundary.
 *
 * Each entry point replaces one call of the reference C++ API
 * (/root/reference/proj/include/dba/...), cited beside it. A C++ drop-in
 * wrapper with the reference's class and exception names is in dbag.hpp.
 *
 * Conventions (mirroring the reference):
 *  - Every call is synchronous: it returns after the device work finished,
 *    as the reference returns after the round (admm_solver.cpp:437-460).
 *  - Problem arrays are caller-owned only for the duration of dbag_create;
 *    the handle keeps device copies (the reference holds `const Problem&`,
 *    admm_solver.hpp:130 — here the caller may free them after create).
 *  - Errors are status codes (dbag_status) instead of the reference's
 *    exception hierarchy (errors.hpp:9-72); the message and, for
 *    DepthBelowGuard, the offending (point, camera) come from
 *    dbag_last_error / dbag_last_error_info (thread-local).
 *  - Observation-indexed per-copy state is in BLOCK ORDER: observations
 *    sorted by (cam_id, point_id) — the reference's partition() order for
 *    (1,1) blocks (admm_solver.cpp:19-27). dbag_get_block_order maps block
 *    index -> input observation index.
 *  - A handle is single-threaded (admm_solver.hpp:74 "not re-entrant").
 */
#ifndef DBAG_H_
#define DBAG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBAG_ABI_VERSION 1

/* errors.hpp:9-72 -> status codes */
typedef enum {
  DBAG_OK = 0,
  DBAG_ERR_VALIDATION = 1,      /* ValidationError                       */
  DBAG_ERR_SIZE_MISMATCH = 2,   /* SizeMismatch                          */
  DBAG_ERR_DEPTH_BELOW_GUARD = 3, /* DepthBelowGuard{depth,point,cam}    */
  DBAG_ERR_SINGULAR = 4,        /* SingularSystem                        */
  DBAG_ERR_CUDA = 5,            /* device failure (no reference analogue) */
  DBAG_ERR_NCCL = 6,            /* collective failure                    */
  DBAG_ERR_INDEX_OUT_OF_RANGE = 7, /* IndexOutOfRange                    */
  DBAG_ERR_DUPLICATE_OBSERVATION = 8, /* DuplicateObservation            */
  DBAG_ERR_UNSUPPORTED = 9,     /* valid for the reference, not built here */
  DBAG_ERR_GENERIC = 10,        /* Error (e.g. "local block N: ...")     */
  DBAG_ERR_PARSE = 11           /* ParseError (a ValidationError) with line */
} dbag_status;

typedef enum { DBAG_LOSS_SQUARED_L2 = 0, DBAG_LOSS_HUBER = 1 } dbag_loss; /* losses.hpp:13-29 */

/* A problem in SoA form (problem.hpp:11-56: Observation, CameraParams,
 * ScenePoint). Camera pose order is (alpha, beta, gamma, t1, t2, t3) with
 * R = Rz(gamma) Ry(beta) Rx(alpha) (geometry.hpp:20-47). */
typedef struct {
  int32_t num_cameras;   /* m */
  int32_t num_points;    /* n */
  int64_t num_obs;       /* l (< 2^31) */
  const int32_t* obs_cam;  /* [l] */
  const int32_t* obs_pt;   /* [l] */
  const double* obs_uv;    /* [l][2] pixels */
  const double* cam_pose;  /* [m][6] nominal record (validated only) */
  const double* cam_f;     /* [m]    nominal focal (validated only)  */
  const double* points;    /* [n][3] nominal record (validated), nullable */
} dbag_problem_view;

/* A ParamState (problem.hpp:36-41). f rides along, never optimised. */
typedef struct {
  int32_t num_cameras;
  int32_t num_points;
  const double* cam_pose;  /* [m][6] */
  const double* cam_f;     /* [m]; NULL -> the problem's cam_f */
  const double* points;    /* [n][3] */
} dbag_param_view;

/* AdmmOptions + InnerOptions + ProjectionGuard + BlockConfig
 * (admm_solver.hpp:15-33, local_opt.hpp:11-19, geometry.hpp:50-52). */
typedef struct {
  double rho_x, rho_y;
  int32_t max_iters;
  double primal_tol;
  int32_t stop_on_primal;
  int32_t loss;            /* dbag_loss */
  double huber_delta;
  int32_t inner_max_iters;
  double grad_tol, step_tol;
  int32_t lbfgs_memory;    /* 1..DBAG_MAX_LBFGS_MEMORY */
  double armijo_c, backtrack;
  int32_t max_line_search;
  double eps_depth;
  int32_t workers;         /* validated >= 1 (reference semantics); unused on GPU */
  int32_t points_per_block, cameras_per_block; /* BlockConfig (admm_solver.hpp:29-32);
                                                 * != (1,1): generalized blocks, EXACT numerics */
  int32_t device;          /* CUDA device ordinal */
  int32_t numerics;        /* dbag_numerics */
} dbag_options;

/* EXACT: every operation of the restated reference in the same order (no FMA
 * contraction, dense pivoted LDLT, sequential reductions, portable sin/cos):
 * the state trajectory is bit-identical to oracle/ (DESIGN.md §Parity).
 * FAST: FMA, Woodbury 2x2 solve, hardware sin/cos, tree reductions — the same
 * algorithm and control flow, different last-ulp rounding. */
typedef enum { DBAG_NUMERICS_FAST = 0, DBAG_NUMERICS_EXACT = 1 } dbag_numerics;

#define DBAG_MAX_LBFGS_MEMORY 8

/* IterationRecord (trace.hpp:12-21) + appended extension fields. */
typedef struct {
  int32_t iter;
  double mean_reproj_err;
  double max_primal_x, max_primal_y;
  double camera_mse, point_mse;   /* NaN without a reference */
  double wall_ms;                 /* device time of local+consensus+dual */
  int64_t comm_floats;
  /* extensions: dual residuals rho*max||xbar^{k+1}-xbar^k|| */
  double max_dual_x, max_dual_y;
  double sum_reproj_err;          /* sum ||z - pi(xbar, ybar)|| (mean * l) */
} dbag_iteration_record;

/* Device-event counters for the FLOP model. */
typedef struct {
  uint64_t n_jacobian;   /* Jacobian/gradient evaluations */
  uint64_t n_trial;      /* trial residual / value evaluations */
  uint64_t n_accept;     /* accepted steps */
  uint64_t n_direction;  /* L-BFGS two-loop directions */
  uint64_t n_pairs_used; /* L-BFGS: sum of history sizes over directions */
  double ms_local, ms_camera, ms_point, ms_final; /* last enqueued round */
  uint64_t n_model_flops; /* generalized blocks: model FLOPs counted per block
                           * from its dimension (DESIGN.md §Generalized blocks) */
} dbag_round_stats;

typedef struct dbag_solver dbag_solver;

int32_t dbag_abi_version(void);
const char* dbag_last_error(void);
/* DepthBelowGuard payload (errors.hpp:52-63); -1 when not applicable.
 * block: offending block index for "local block N" errors. */
void dbag_last_error_info(int32_t* point_id, int32_t* cam_id, double* depth, int64_t* block);

void dbag_options_default(dbag_options* o); /* AdmmOptions{} defaults */

/* Problem::create + AdmmSolver::AdmmSolver (problem.cpp:66-96,
 * admm_solver.cpp:103-142): validates, uploads, builds the block order and
 * copy maps on the device (partition, admm_solver.cpp:14-72; copy maps
 * :126-140; build_visibility, problem.cpp:12-64), copies = init, duals = 0. */
int dbag_create(const dbag_problem_view* problem, const dbag_param_view* init,
                const dbag_options* opts, dbag_solver** out);
void dbag_destroy(dbag_solver* h);

/* Phases (admm_solver.cpp:144-357). */
int dbag_local_update(dbag_solver* h, int64_t block); /* local_update(int) */
int dbag_local_update_all(dbag_solver* h);           /* local_update_all() */
int dbag_consensus_update(dbag_solver* h);           /* consensus_update() */
int dbag_dual_update(dbag_solver* h);                /* dual_update()      */

/* Reference state for the MSE columns of iterate()/run() (the reference
 * passes `const ParamState*` per call, admm_solver.hpp:97-100). NULL clears.
 * Always the GLOBAL state ([m][6], [n][3]); a sharded handle keeps its own
 * cameras and points of it. */
int dbag_set_reference(dbag_solver* h, const dbag_param_view* ref);
/* iterate(const ParamState*) (admm_solver.cpp:437-460); with_reference != 0
 * fills camera_mse/point_mse against the dbag_set_reference state. */
int dbag_iterate(dbag_solver* h, int32_t with_reference, dbag_iteration_record* out);
/* run(const ParamState*) (admm_solver.cpp:462-474): rounds until max_iters
 * (or stop_on_primal). Writes min(cap, rounds) records; *n_out = rounds. */
int dbag_run(dbag_solver* h, int32_t with_reference, dbag_iteration_record* trace, int64_t cap,
             int64_t* n_out);

/* state() queries (admm_solver.hpp:102-108). */
int dbag_get_consensus(dbag_solver* h, double* cam_pose /*[m][6]*/, double* cam_f /*[m], nullable*/,
                       double* points /*[n][3]*/);
int dbag_set_consensus(dbag_solver* h, const double* cam_pose, const double* points);
int dbag_get_copies(dbag_solver* h, double* local_points /*[l][3]*/, double* local_cams /*[l][6]*/,
                    double* dual_r /*[l][3]*/, double* dual_s /*[l][6]*/); /* block order */
int dbag_set_copies(dbag_solver* h, const double* local_points, const double* local_cams,
                    const double* dual_r, const double* dual_s);
int32_t dbag_iteration(dbag_solver* h);
int64_t dbag_num_blocks(dbag_solver* h);
/* observation ids of all blocks, concatenated in block order (== sorted by
 * (cam_id, point_id), admm_solver.cpp:19-27) */
int dbag_get_block_order(dbag_solver* h, int32_t* obs_ids /*[l]*/);
/* copy counts: sum of |point_ids| / |cam_ids| over blocks (== l for (1,1)).
 * dbag_get_copies / dbag_set_copies take [point_copies][3], [cam_copies][6],
 * [point_copies][3], [cam_copies][6], block by block in id order. */
int dbag_num_copies(dbag_solver* h, int64_t* point_copies, int64_t* cam_copies);
/* blocks() (admm_solver.hpp:102-108, LocalBlock admm_solver.hpp:35-45): CSR over
 * blocks; every pointer nullable. obs_off/pt_off/cam_off [B+1], pt_ids [PC],
 * cam_ids [CC], obs_*_local [l] (in block order). */
int dbag_get_blocks(dbag_solver* h, int64_t* obs_off, int64_t* pt_off, int32_t* pt_ids,
                    int64_t* cam_off, int32_t* cam_ids, int32_t* obs_pt_local,
                    int32_t* obs_cam_local);

/* Result/objective queries (admm_solver.hpp:110-127).
 * dbag_max_primal: max_primal_residual_points/cameras (admm_solver.cpp:359-383),
 *   one device pass. On a sharded handle: the maximum over this rank's copies
 *   (the reference's value is the maximum over the ranks).
 * dbag_dual_sums: dual_sum_point/camera (admm_solver.cpp:385-399) for every
 *   point and camera, in GLOBAL indexing. On a sharded handle: the sums over
 *   this rank's copies, zero where the rank holds no copy (the reference's
 *   sums are the element-wise sum over the ranks). */
int dbag_max_primal(dbag_solver* h, double* max_x, double* max_y);
int dbag_dual_sums(dbag_solver* h, double* point_sums /*[n][3]*/, double* cam_sums /*[m][6]*/);
int dbag_block_objective(dbag_solver* h, int64_t block, double* out);
int64_t dbag_ops_per_iteration(dbag_solver* h);  /* ops_per_iteration() */
int64_t dbag_comm_floats(dbag_solver* h);        /* comm_floats_per_iteration() */

/* problem.hpp:59-85 at the current consensus. */
int dbag_mean_reprojection_error(dbag_solver* h, double* out); /* throws-variant semantics */
int dbag_total_squared_error(dbag_solver* h, double* out);
int dbag_rms_reprojection_error(dbag_solver* h, double* out); /* problem.cpp:159-162 */
/* align_similarity (problem.cpp:204-237): Umeyama similarity of state's points
 * onto reference's, applied to points and cameras (f kept). Host views in,
 * host arrays out ([m][6], [n][3]); moments reduced on `device`. Tolerance
 * parity (Eigen's JacobiSVD is not bit-pinnable). SizeMismatch if the point
 * counts differ or n < 3. */
int dbag_align_similarity(const dbag_param_view* state, const dbag_param_view* reference,
                          int32_t device, double* out_pose, double* out_points);

/* Measurement hooks (no reference analogue): enqueue one full round
 * (local+consensus+dual+metrics) on the handle's stream without waiting;
 * dbag_stream returns the cudaStream_t as an opaque pointer. */
int dbag_enqueue_round(dbag_solver* h);
int dbag_reset(dbag_solver* h); /* restart from the init state: copies = init, duals = 0 */
void* dbag_stream(dbag_solver* h);
int dbag_synchronize(dbag_solver* h);
int dbag_set_profiling(dbag_solver* h, int32_t on); /* per-round kernel events, summed */
int dbag_get_round_stats(dbag_solver* h, dbag_round_stats* out); /* counters since reset */
int dbag_reset_stats(dbag_solver* h);
/* FP64 FMA throughput of the device (TFLOP/s, 2 flops per DFMA): the FP64
 * roofline denominator, which MEASURED_PEAKS.json does not carry. */
int dbag_measure_fp64_peak(int32_t device, double* tflops);
/* Test hook (no reference counterpart): runs n of the EXACT kernels'
 * branch-free reciprocals RN(1/d) over the exponent band they are used on and
 * counts the results that differ bitwise from IEEE 1.0/d. */
int dbag_selftest_division(int32_t device, int64_t n, uint64_t seed, int64_t* mismatches);

/* ---- multi-GPU ---------------------------------------------
 * Cameras are split into contiguous ranges balanced on observation counts;
 * rank r owns every observation of its cameras. Boundary points (cameras on
 * several ranks) exchange their copies' raw (x, r) once per round, each copy
 * only to the other ranks that hold its point (one grouped ncclSend/ncclRecv
 * pair per peer, no padding), so every holder recomputes the reference's
 * sequential consensus sum: the EXACT trajectory is bit-identical for any
 * number of ranks. Host-only plan functions below need no GPU (tested with
 * gloo on CPU). */
typedef struct {
  int32_t rank, world;
  int32_t cam_begin, cam_end;   /* this rank's camera range */
  int64_t local_obs;
  int32_t local_points;
  int32_t boundary_points;      /* global */
  int64_t boundary_copies;      /* global */
  int64_t send_count, recv_count; /* this rank's exchange slots per round (48 B each) */
  int64_t comm_floats;          /* reference communication_cost (global) */
} dbag_shard_info;
typedef struct dbag_shard_plan dbag_shard_plan;
int dbag_partition_cameras(int32_t m, const int64_t* obs_per_camera, int32_t world,
                           int32_t* cam_lo /*[world+1]*/);
int dbag_shard_plan_create(const dbag_problem_view* full, int32_t rank, int32_t world,
                           dbag_shard_plan** out, dbag_shard_info* info);
void dbag_shard_plan_get_info(const dbag_shard_plan* s, dbag_shard_info* info);
/* Any pointer may be NULL. Sizes: cam_lo [world+1]; local_obs [local_obs];
 * local_points, bp_of_local, owner_of_local [local_points]; gb_off
 * [boundary_points+1]; gmap [boundary_copies]: for a copy of a point this rank
 * holds, >= 0 its recv slot, -2 - q for this rank's own copy (local observation
 * q); -1 otherwise; send_obs_local [send_count] (local observation of each
 * send slot, grouped by destination peer, global copy order within a peer). */
int dbag_shard_plan_arrays(const dbag_shard_plan* s, int32_t* cam_lo, int64_t* local_obs,
                           int32_t* local_points, int32_t* bp_of_local, int8_t* owner_of_local,
                           int64_t* gb_off, int64_t* gmap, int64_t* send_obs_local);
/* send_off / recv_off [world+1]: slot ranges per destination / source peer. */
int dbag_shard_plan_exchange(const dbag_shard_plan* s, int64_t* send_off, int64_t* recv_off);
void dbag_shard_plan_destroy(dbag_shard_plan* s);

/* A solver for shard `rank` of `world` over the FULL problem/init (every rank
 * passes the same arrays). Queries return this rank's entries (global ids). */
int dbag_create_sharded(const dbag_problem_view* full, const dbag_param_view* init,
                        const dbag_options* opts, int32_t rank, int32_t world,
                        dbag_solver** out);
/* NCCL transport: rank 0 makes the id, the launcher broadcasts it, every rank
 * attaches; iterate/run/enqueue_round then exchange the boundary copies with
 * grouped ncclSend/ncclRecv and the partial records with ncclAllGather. */
int dbag_nccl_unique_id(uint8_t id[128]);
int dbag_attach_nccl(dbag_solver* h, const uint8_t id[128]);
/* External transport (tests, single-device emulation of several ranks): run a
 * round in phases and copy buffers between handles in between:
 *   phase 0: local solve + camera consensus/dual + pack boundary copies
 *   exchange_copy(dst, src, 0) for every (dst, src) pair
 *   phase 1: point consensus/dual/metric + partial metrics
 *   exchange_copy(dst, src, 1) for every pair
 *   phase 2: combine -> *out (only for phase 2; may be NULL otherwise).
 * The MSE columns are filled when a reference is set (dbag_set_reference). */
int dbag_round_phase(dbag_solver* h, int32_t phase, dbag_iteration_record* out);
int dbag_exchange_copy(dbag_solver* dst, dbag_solver* src, int32_t which);

/* ---- problem files and metrics CSV (bal_io.hpp:21-31, metrics_csv.hpp:11-19)
 * Host-only. parse: the reference's text format (optional `rotation euler|
 * angle-axis` header; m n l; l observation lines; 9 values per camera with zero
 * distortion; 3 per point) followed by Problem::create validation. serialize:
 * 17 significant digits (bit-exact round trip), observations from `problem`,
 * cameras/points from `state`. Two-phase outputs: buf NULL -> *len only. */
/* ---- centralized Levenberg-Marquardt baseline (lm_solver.hpp:13-54,
 * lm_solver.cpp): Schur complement on the device, the dense 6m x 6m camera
 * system by cuSOLVER. Tolerance parity (Eigen's blocked LDLT is not
 * bit-pinnable). DESIGN.md §12. */
typedef struct {
  int32_t max_iters;     /* LmOptions (lm_solver.hpp:14-23) */
  double error_stop, lambda_init, lambda_max, lambda_up, lambda_down;
  int32_t use_schur;     /* 0: the dense (6m+3n) step, <= 24000 unknowns */
  double eps_depth;      /* ProjectionGuard */
  int32_t device;
} dbag_lm_options;
typedef enum { DBAG_LM_ERROR_STOP = 0, DBAG_LM_LAMBDA_MAX = 1, DBAG_LM_MAX_ITERS = 2 } dbag_lm_stop;
typedef struct dbag_lm dbag_lm;
void dbag_lm_options_default(dbag_lm_options* o);
/* Problem::create validation + the initial state (copied to the device). */
int dbag_lm_create(const dbag_problem_view* problem, const dbag_param_view* init,
                   const dbag_lm_options* opts, dbag_lm** out);
/* solve_lm (lm_solver.cpp:153-218) from the handle's state; trace[0] is the
 * init row; loss must be DBAG_LOSS_SQUARED_L2; reference nullable (MSE). */
int dbag_lm_solve(dbag_lm* h, int32_t loss, const dbag_param_view* reference,
                  dbag_iteration_record* trace, int64_t cap, int64_t* n_trace, int32_t* stop,
                  int32_t* accepted_steps);
/* lm_compute_step (lm_solver.cpp:142-151) at the handle's state. */
int dbag_lm_compute_step(dbag_lm* h, double lambda, int32_t use_schur, double* d_cam /*[6m]*/,
                         double* d_pts /*[3n]*/);
int dbag_lm_get_state(dbag_lm* h, double* cam_pose /*[m][6]*/, double* points /*[n][3]*/);
void dbag_lm_destroy(dbag_lm* h);

/* ---- host-only: partition() and communication_cost() (admm_solver.hpp:47-54,
 * admm_solver.cpp:14-101) for any BlockConfig. No GPU needed. */
typedef struct dbag_partition_result dbag_partition_result;
int dbag_partition(const dbag_problem_view* problem, int32_t points_per_block,
                   int32_t cameras_per_block, dbag_partition_result** out, int64_t* n_blocks,
                   int64_t* n_point_copies, int64_t* n_cam_copies, int64_t* comm_floats);
int dbag_partition_fetch(const dbag_partition_result* r, int64_t* obs_off /*[B+1]*/,
                         int32_t* obs_ids /*[l]*/, int64_t* pt_off /*[B+1]*/,
                         int32_t* pt_ids /*[PC]*/, int64_t* cam_off /*[B+1]*/,
                         int32_t* cam_ids /*[CC]*/, int32_t* obs_pt_local /*[l]*/,
                         int32_t* obs_cam_local /*[l]*/);
void dbag_partition_destroy(dbag_partition_result* r);

typedef struct dbag_bal dbag_bal;
int dbag_parse_problem_text(const char* text, size_t len, dbag_bal** out, int32_t* m,
                            int32_t* n, int64_t* l);
int dbag_bal_fetch(const dbag_bal* b, int32_t* obs_cam, int32_t* obs_pt, double* obs_uv,
                   double* cam_pose, double* cam_f, double* points);
void dbag_bal_destroy(dbag_bal* b);
int dbag_serialize_problem_text(const dbag_problem_view* problem, const dbag_param_view* state,
                                char* buf, size_t cap, size_t* len);
int dbag_metrics_csv(const dbag_iteration_record* trace, int64_t n, char* buf, size_t cap,
                     size_t* len);
const char* dbag_io_last_error(int32_t* line); /* message and ParseError line (-1: none) */

/* Synthetic scenes of BASELINE.json configs 1-5 (host C++, deterministic in
 * seed). Two-phase: size query, then fill. scale in (0,1]
 * shrinks points/cameras proportionally for bounded samples. */
typedef struct {
  int32_t config;        /* 1..5 */
  uint64_t seed;
  double scale;          /* 1.0 = the BASELINE size */
  int32_t num_cameras, num_points;
  int64_t num_obs;
  double sigma_pixel, outlier_frac, sigma_init;
} dbag_scene_info;
typedef struct dbag_scene dbag_scene;
int dbag_scene_generate(int32_t config, uint64_t seed, double scale, dbag_scene** out,
                        dbag_scene_info* info);
/* gt_* = ground truth; init_* = perturb(gt, sigma_init); obs in emission order */
int dbag_scene_fetch(dbag_scene* s, int32_t* obs_cam, int32_t* obs_pt, double* obs_uv,
                     double* gt_pose, double* cam_f, double* gt_points, double* init_pose,
                     double* init_points);
void dbag_scene_destroy(dbag_scene* s);

#ifdef __cplusplus
}
#endif
#endif /* DBAG_H_ */
