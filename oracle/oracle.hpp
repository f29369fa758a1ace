// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// An Eigen-free CPU restatement of the reference D-ADMM bundle adjustment
// (arXiv 1708.07954, /root/reference/proj). It exists to check the B200 product
// path (libdbag) and to serve as the timed CPU baseline ("kind": "port") in
// bench.py. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it. The product never links or calls it.
//
// Every function cites the reference file:line it restates. Arithmetic follows
// the reference's operation order where that order is observable (projection,
// perspective Jacobian, consensus accumulation, dual update); dense reductions
// that Eigen vectorises internally (JᵀJ, dot products, LDLT inner products) are
// summed sequentially here — Eigen's SSE2 packet order is unpinned at bit level
// (SURVEY §8(c)).
#pragma once

#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using Vec2 = std::array<double, 2>;
using Vec3 = std::array<double, 3>;
using Vec6 = std::array<double, 6>;
using Mat3 = std::array<double, 9>;  // row-major

// ---- errors (proj/include/dba/errors.hpp:9-72) -----------------------------
enum ErrorKind {
  kOk = 0,
  kValidation = 1,
  kSizeMismatch = 2,
  kDepthBelowGuard = 3,
  kSingularSystem = 4,
  kIndexOutOfRange = 7,
  kDuplicateObservation = 8,
  kGenericError = 10,
  kProjectionFailed = 11,
};

struct Error : std::runtime_error {
  explicit Error(const std::string& w, int k = kGenericError) : std::runtime_error(w), kind(k) {}
  int kind;
};
struct ValidationError : Error {
  explicit ValidationError(const std::string& w, int k = kValidation) : Error(w, k) {}
};
struct SizeMismatch : ValidationError {
  explicit SizeMismatch(const std::string& w) : ValidationError(w, kSizeMismatch) {}
};
struct IndexOutOfRange : ValidationError {
  explicit IndexOutOfRange(const std::string& w) : ValidationError(w, kIndexOutOfRange) {}
};
struct DuplicateObservation : ValidationError {
  explicit DuplicateObservation(const std::string& w) : ValidationError(w, kDuplicateObservation) {}
};
struct DepthBelowGuard : Error {
  DepthBelowGuard(double depth, double eps, int point_id = -1, int cam_id = -1);
  double depth;
  int point_id, cam_id;
};

// ---- geometry (proj/src/geometry.cpp) -------------------------------------
struct Camera {
  double alpha = 0, beta = 0, gamma = 0;
  Vec3 t{0, 0, 0};
  double f = 1.0;
  Vec6 pose() const { return {alpha, beta, gamma, t[0], t[1], t[2]}; }
  void set_pose(const Vec6& p) {
    alpha = p[0];
    beta = p[1];
    gamma = p[2];
    t = {p[3], p[4], p[5]};
  }
};

struct Guard {
  double eps_depth = 1e-6;
};

void det_sincos(double x, double* sn, double* cs);
Mat3 mat_mul(const Mat3& a, const Mat3& b);
Vec3 mat_vec(const Mat3& a, const Vec3& x);
Mat3 rotation_from_euler(double alpha, double beta, double gamma);
Vec3 euler_from_rotation(const Mat3& R);
struct EulerRotation {
  Mat3 R, dA, dB, dG;
};
EulerRotation rotation_with_derivatives(double alpha, double beta, double gamma);
bool try_project(const Vec3& x, const Camera& y, const Guard& g, Vec2* out);
struct Expansion {
  Vec2 z;
  double Jp[2][3];
  double Jc[2][6];
};
bool try_project_with_jacobians(const Vec3& x, const Camera& y, const Guard& g, Expansion* out);

// ---- losses (proj/src/losses.cpp) -----------------------------------------
struct Loss {
  int type = 0;  // 0 squared L2, 1 Huber
  double delta = 1.0;
  bool is_huber() const { return type == 1; }
};
double loss_value(const Loss& k, const Vec2& r);
Vec2 loss_gradient(const Loss& k, const Vec2& r);

// ---- dense helpers + Eigen-style LDLT --------------------------------------
using VecX = std::vector<double>;
struct MatX {
  int rows = 0, cols = 0;
  std::vector<double> a;  // row-major
  MatX() = default;
  MatX(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * cols + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * cols + j]; }
};
// Restates Eigen's LDLT<MatrixXd,Lower> (symmetric diagonal pivoting,
// unblocked) followed by LDLT::solve, as called at proj/src/local_opt.cpp:56.
VecX ldlt_solve(const MatX& A, const VecX& b);

// ---- inner solvers (proj/src/local_opt.cpp) -------------------------------
struct InnerOptions {
  int max_iters = 10;
  double grad_tol = 1e-8;
  double step_tol = 1e-10;
  int lbfgs_memory = 8;
  double armijo_c = 1e-4;
  double backtrack = 0.5;
  int max_line_search = 40;
};
enum InnerStatus { kGradConverged = 0, kStepConverged, kMaxIters, kSingular, kLineSearchFailed };
struct InnerResult {
  VecX x;
  double objective = 0.0;
  int status = kMaxIters;
  int iters = 0;
};
using ResidualFn = std::function<bool(const VecX&, VecX*)>;
using JacobianFn = std::function<bool(const VecX&, MatX*)>;
using ValueFn = std::function<bool(const VecX&, double*)>;
using GradFn = std::function<bool(const VecX&, VecX*)>;
InnerResult gauss_newton(const ResidualFn& rf, const JacobianFn& jf, VecX x0, const InnerOptions& o);
InnerResult lbfgs(const ValueFn& vf, const GradFn& gf, VecX x0, const InnerOptions& o);

// ---- problem (proj/src/problem.cpp) ---------------------------------------
struct Observation {
  int cam_id = 0, point_id = 0;
  Vec2 z{0, 0};
};
struct Visibility {
  std::vector<std::vector<int>> points_in_camera, cameras_seeing_point;
};
Visibility build_visibility(const std::vector<Observation>& obs, int m, int n);
struct ParamState {
  std::vector<Camera> cameras;
  std::vector<Vec3> points;
};
struct Problem {
  std::vector<Camera> cameras;
  std::vector<Vec3> points;
  std::vector<Observation> observations;
  Visibility visibility;
  int num_cameras() const { return (int)cameras.size(); }
  int num_points() const { return (int)points.size(); }
  int num_observations() const { return (int)observations.size(); }
  static Problem create(std::vector<Camera> c, std::vector<Vec3> p, std::vector<Observation> o);
};
double mean_reprojection_error(const Problem& p, const ParamState& s, const Guard& g);
bool try_mean_reprojection_error(const Problem& p, const ParamState& s, const Guard& g, double* out);
bool try_total_squared_error(const Problem& p, const ParamState& s, const Guard& g, double* out);
struct MseResult {
  double camera_mse = 0, point_mse = 0;
};
MseResult parameter_mse(const ParamState& s, const ParamState& ref);

// ---- ADMM (proj/src/admm_solver.cpp, proj/include/dba/admm_solver.hpp) -----
struct AdmmOptions {
  double rho_x = 1.0, rho_y = 1.0;
  int max_iters = 1600;
  double primal_tol = 1e-6;
  bool stop_on_primal = false;
  Loss misfit_loss;
  InnerOptions inner;
  Guard guard;
  int workers = 1;
};
struct BlockConfig {
  int points_per_block = 1, cameras_per_block = 1;
};
struct LocalBlock {
  std::vector<int> point_ids, cam_ids, obs_ids, obs_point_local, obs_cam_local;
};
std::vector<LocalBlock> partition(const Problem& p, const BlockConfig& c);
int64_t communication_cost(const Problem& p, const BlockConfig& c);

struct IterationRecord {
  int iter = 0;
  double mean_reproj_err, max_primal_x = 0, max_primal_y = 0, camera_mse, point_mse, wall_ms = 0;
  int64_t comm_floats = 0;
  IterationRecord();
};

struct AdmmState {
  std::vector<std::vector<Vec3>> local_points;
  std::vector<std::vector<Vec6>> local_cameras;
  std::vector<std::vector<Vec3>> dual_r;
  std::vector<std::vector<Vec6>> dual_s;
  ParamState consensus;
  int iteration = 0;
};

// proj/src/parallel.cpp:5-91 — persistent fork-join pool; caller participates.
class WorkerPool {
 public:
  explicit WorkerPool(int workers);
  ~WorkerPool();
  void run(int n, const std::function<void(int)>& fn);

 private:
  void worker_loop();
  std::vector<std::thread> threads_;
  std::mutex mutex_;
  std::condition_variable start_cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int total_ = 0;
  std::atomic<int> next_{0}, remaining_{0};
  uint64_t generation_ = 0;
  int active_ = 0;
  bool stop_ = false;
};

class AdmmSolver {
 public:
  AdmmSolver(const Problem& p, ParamState init, AdmmOptions o, BlockConfig bc = {});
  void local_update(int b);
  void local_update_all();
  void consensus_update();
  void dual_update();
  IterationRecord iterate(const ParamState* ref = nullptr);
  std::vector<IterationRecord> run(const ParamState* ref = nullptr);
  AdmmState& state() { return state_; }
  const std::vector<LocalBlock>& blocks() const { return blocks_; }
  double max_primal_residual_points() const;
  double max_primal_residual_cameras() const;
  Vec3 dual_sum_point(int i) const;
  Vec6 dual_sum_camera(int j) const;
  double block_objective(int b) const;
  int64_t ops_per_iteration() const;
  int64_t comm_floats_per_iteration() const { return comm_floats_; }
  const AdmmOptions& options() const { return opts_; }

 private:
  const Problem& problem_;
  AdmmOptions opts_;
  std::vector<LocalBlock> blocks_;
  AdmmState state_;
  std::vector<std::vector<std::pair<int, int>>> point_copies_, camera_copies_;
  int64_t comm_floats_ = 0;
  std::unique_ptr<WorkerPool> pool_;
};

// ---- centralized LM baseline (proj/include/dba/lm_solver.hpp, proj/src/lm_solver.cpp)
struct LmOptions {
  int max_iters = 100;
  double error_stop = 1e-14;
  double lambda_init = 1e-3;
  double lambda_max = 1e16;
  double lambda_up = 10.0;
  double lambda_down = 10.0;
  bool use_schur = true;
  Guard guard;
};
enum LmStopReason { kLmErrorStop = 0, kLmLambdaMax = 1, kLmMaxIters = 2 };
struct LmStep {
  VecX delta_cameras;  // 6m
  VecX delta_points;   // 3n
};
struct LmResult {
  ParamState state;
  std::vector<IterationRecord> trace;
  int stop = kLmMaxIters;
  int accepted_steps = 0;
};
LmStep lm_compute_step(const Problem& p, const ParamState& s, double lambda, bool use_schur,
                       const Guard& g);
LmResult solve_lm(const Problem& p, const ParamState& init, const LmOptions& o, const Loss& loss,
                  const ParamState* reference);

// ---- rng + scene generation (proj/include/dba/rng.hpp, proj/src/scene_gen.cpp)
class Rng {
 public:
  explicit Rng(uint64_t seed) : engine_(seed) {}
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal();
  double normal(double mean, double sigma) { return mean + sigma * normal(); }
  uint64_t uniform_int(uint64_t n);

 private:
  std::mt19937_64 engine_;
};

struct SceneConfig {
  int n_cameras = 5, n_points = 10;
  double orbit_radius = 1000.0, altitude = 1500.0;
  Vec3 box_min{-250.0, -250.0, -50.0}, box_max{250.0, 250.0, 50.0};
  double jitter_trans = 10.0, jitter_rot = 0.01;
  int visibility_window = 5;
  double focal = 200.0;
  uint64_t rng_seed = 0;
};
struct GeneratedScene {
  Problem problem;
  ParamState ground_truth;
};
GeneratedScene generate_scene(const SceneConfig& c);
ParamState perturb(const ParamState& s, double sigma_cam, double sigma_point, uint64_t seed);

}  // namespace orc
