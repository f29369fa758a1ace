// dbag.hpp — header-only C++ drop-in for the reference's ADMM solver API,
// backed by the B200 C-ABI (dbag.h / libdbag.so).
//
// Mirrors /root/reference/proj/include/dba/{admm_solver,problem,trace,errors}.hpp:
// the same type, method and exception names in namespace dba::gpu, so a call
// site written against dba::AdmmSolver compiles against dba::gpu::AdmmSolver
// with a namespace change. Plain arrays (SoA) replace the
// Eigen types: a camera pose is (alpha, beta, gamma, t1, t2, t3).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "dbag.h"

namespace dba {
namespace gpu {

// ---- errors.hpp:9-72 -------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public Error {
 public:
  using Error::Error;
};
class DuplicateObservation : public ValidationError {
 public:
  using ValidationError::ValidationError;
};
class IndexOutOfRange : public ValidationError {
 public:
  using ValidationError::ValidationError;
};
class SizeMismatch : public ValidationError {
 public:
  using ValidationError::ValidationError;
};
class DepthBelowGuard : public Error {
 public:
  DepthBelowGuard(const std::string& w, double d, int p, int c)
      : Error(w), depth(d), point_id(p), cam_id(c) {}
  double depth;
  int point_id;
  int cam_id;
};
class SingularSystem : public Error {
 public:
  using Error::Error;
};
class DeviceError : public Error {  // no reference analogue: CUDA / NCCL failure
 public:
  using Error::Error;
};

inline void check(int rc) {
  if (rc == DBAG_OK) return;
  const std::string msg = dbag_last_error();
  int32_t pt = -1, cam = -1;
  double depth = 0.0;
  int64_t block = -1;
  dbag_last_error_info(&pt, &cam, &depth, &block);
  switch (rc) {
    case DBAG_ERR_VALIDATION: throw ValidationError(msg);
    case DBAG_ERR_SIZE_MISMATCH: throw SizeMismatch(msg);
    case DBAG_ERR_DEPTH_BELOW_GUARD: throw DepthBelowGuard(msg, depth, pt, cam);
    case DBAG_ERR_SINGULAR: throw SingularSystem(msg);
    case DBAG_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
    case DBAG_ERR_DUPLICATE_OBSERVATION: throw DuplicateObservation(msg);
    case DBAG_ERR_CUDA:
    case DBAG_ERR_NCCL: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

// ---- problem.hpp:11-56, trace.hpp:12-23 ----------------------------------------
struct Observation {
  int cam_id = 0;
  int point_id = 0;
  double z[2] = {0.0, 0.0};
};

struct ParamState {
  std::vector<double> cam_pose;  // [m][6]
  std::vector<double> cam_f;     // [m]
  std::vector<double> points;    // [n][3]
  int num_cameras() const { return static_cast<int>(cam_f.size()); }
  int num_points() const { return static_cast<int>(points.size() / 3); }
  dbag_param_view view() const {
    return {num_cameras(), num_points(), cam_pose.data(), cam_f.data(), points.data()};
  }
};

struct Problem {
  ParamState nominal;  // the file's / ground-truth camera and point record
  std::vector<int32_t> obs_cam, obs_pt;
  std::vector<double> obs_uv;  // [l][2]
  int num_cameras() const { return nominal.num_cameras(); }
  int num_points() const { return nominal.num_points(); }
  int64_t num_observations() const { return static_cast<int64_t>(obs_cam.size()); }
  ParamState nominal_state() const { return nominal; }
  static Problem create(ParamState cameras_points, const std::vector<Observation>& obs) {
    Problem p;
    p.nominal = std::move(cameras_points);
    p.obs_cam.reserve(obs.size());
    p.obs_pt.reserve(obs.size());
    p.obs_uv.reserve(2 * obs.size());
    for (const Observation& o : obs) {
      p.obs_cam.push_back(o.cam_id);
      p.obs_pt.push_back(o.point_id);
      p.obs_uv.push_back(o.z[0]);
      p.obs_uv.push_back(o.z[1]);
    }
    return p;  // validated on the device by AdmmSolver (Problem::create semantics)
  }
  dbag_problem_view view() const {
    return {num_cameras(),      num_points(),          num_observations(), obs_cam.data(),
            obs_pt.data(),      obs_uv.data(),         nominal.cam_pose.data(),
            nominal.cam_f.data(), nominal.points.data()};
  }
};

using IterationRecord = dbag_iteration_record;
using Trace = std::vector<IterationRecord>;

// ---- admm_solver.hpp:15-70 --------------------------------------------------
struct InnerOptions {
  int max_iters = 10;
  double grad_tol = 1e-8;
  double step_tol = 1e-10;
  int lbfgs_memory = 8;
  double armijo_c = 1e-4;
  double backtrack = 0.5;
  int max_line_search = 40;
};

struct LossKind {
  enum class Type { kSquaredL2 = DBAG_LOSS_SQUARED_L2, kHuber = DBAG_LOSS_HUBER };
  Type type = Type::kSquaredL2;
  double delta = 1.0;
  static LossKind squared_l2() { return {Type::kSquaredL2, 1.0}; }
  static LossKind huber(double d) {
    if (!(d > 0.0)) throw ValidationError("Huber delta must be > 0");
    return {Type::kHuber, d};
  }
  bool is_huber() const { return type == Type::kHuber; }
};

struct ProjectionGuard {
  double eps_depth = 1e-6;
};

struct AdmmOptions {
  double rho_x = 1.0;
  double rho_y = 1.0;
  int max_iters = 1600;
  double primal_tol = 1e-6;
  bool stop_on_primal = false;
  LossKind misfit_loss = LossKind::squared_l2();
  InnerOptions inner;
  ProjectionGuard guard;
  int workers = 1;  // validated (>= 1) like the reference; the device ignores it
  int device = 0;
  dbag_numerics numerics = DBAG_NUMERICS_EXACT;
};

struct BlockConfig {
  int points_per_block = 1;
  int cameras_per_block = 1;
};

struct AdmmResult {
  ParamState state;
  Trace trace;
};

// LocalBlock (admm_solver.hpp:35-45).
struct LocalBlock {
  std::vector<int32_t> point_ids, cam_ids, obs_ids, obs_point_local, obs_cam_local;
};

class AdmmSolver {
 public:
  AdmmSolver(const Problem& problem, const ParamState& init, const AdmmOptions& opts,
             BlockConfig block_config = {})
      : m_(problem.num_cameras()), n_(problem.num_points()), l_(problem.num_observations()),
        max_iters_(opts.max_iters), stop_on_primal_(opts.stop_on_primal),
        primal_tol_(opts.primal_tol) {
    dbag_options o;
    dbag_options_default(&o);
    o.rho_x = opts.rho_x;
    o.rho_y = opts.rho_y;
    o.max_iters = opts.max_iters;
    o.primal_tol = opts.primal_tol;
    o.stop_on_primal = opts.stop_on_primal ? 1 : 0;
    o.loss = static_cast<int32_t>(opts.misfit_loss.type);
    o.huber_delta = opts.misfit_loss.delta;
    o.inner_max_iters = opts.inner.max_iters;
    o.grad_tol = opts.inner.grad_tol;
    o.step_tol = opts.inner.step_tol;
    o.lbfgs_memory = opts.inner.lbfgs_memory;
    o.armijo_c = opts.inner.armijo_c;
    o.backtrack = opts.inner.backtrack;
    o.max_line_search = opts.inner.max_line_search;
    o.eps_depth = opts.guard.eps_depth;
    o.workers = opts.workers;
    o.points_per_block = block_config.points_per_block;
    o.cameras_per_block = block_config.cameras_per_block;
    o.device = opts.device;
    o.numerics = opts.numerics;
    const dbag_problem_view pv = problem.view();
    const dbag_param_view iv = init.view();
    check(dbag_create(&pv, &iv, &o, &h_));
  }
  ~AdmmSolver() {
    if (h_) dbag_destroy(h_);
  }
  AdmmSolver(const AdmmSolver&) = delete;
  AdmmSolver& operator=(const AdmmSolver&) = delete;

  void local_update(int64_t block_index) { check(dbag_local_update(h_, block_index)); }
  void local_update_all() { check(dbag_local_update_all(h_)); }
  void consensus_update() { check(dbag_consensus_update(h_)); }
  void dual_update() { check(dbag_dual_update(h_)); }

  IterationRecord iterate(const ParamState* reference = nullptr) {
    use_reference(reference);
    IterationRecord rec;
    check(dbag_iterate(h_, reference ? 1 : 0, &rec));
    return rec;
  }

  AdmmResult run(const ParamState* reference = nullptr) {
    use_reference(reference);
    AdmmResult out;
    const int64_t cap = std::max<int64_t>(1, max_iters_ - dbag_iteration(h_));
    out.trace.resize(cap);
    int64_t n = 0;
    check(dbag_run(h_, reference ? 1 : 0, out.trace.data(), cap, &n));
    out.trace.resize(std::min(n, cap));
    out.state = consensus();
    return out;
  }

  ParamState consensus() const {
    ParamState s;
    s.cam_pose.resize(6 * static_cast<size_t>(m_));
    s.cam_f.resize(m_);
    s.points.resize(3 * static_cast<size_t>(n_));
    check(dbag_get_consensus(h_, s.cam_pose.data(), s.cam_f.data(), s.points.data()));
    return s;
  }

  double max_primal_residual_points() const { return primal().first; }
  double max_primal_residual_cameras() const { return primal().second; }
  double block_objective(int64_t b) const {
    double v = 0.0;
    check(dbag_block_objective(h_, b, &v));
    return v;
  }
  int64_t ops_per_iteration() const { return dbag_ops_per_iteration(h_); }
  int64_t comm_floats_per_iteration() const { return dbag_comm_floats(h_); }
  int64_t num_blocks() const { return dbag_num_blocks(h_); }
  dbag_solver* handle() const { return h_; }

  // blocks() (admm_solver.hpp:108)
  std::vector<LocalBlock> blocks() const {
    const int64_t B = num_blocks();
    int64_t pc = 0, cc = 0;
    check(dbag_num_copies(h_, &pc, &cc));
    std::vector<int64_t> oo(B + 1), po(B + 1), co(B + 1);
    std::vector<int32_t> pid(pc), cid(cc), obs(l_), opl(l_), ocl(l_);
    check(dbag_get_blocks(h_, oo.data(), po.data(), pid.data(), co.data(), cid.data(), opl.data(),
                          ocl.data()));
    check(dbag_get_block_order(h_, obs.data()));
    std::vector<LocalBlock> out(B);
    for (int64_t b = 0; b < B; ++b) {
      out[b].point_ids.assign(pid.begin() + po[b], pid.begin() + po[b + 1]);
      out[b].cam_ids.assign(cid.begin() + co[b], cid.begin() + co[b + 1]);
      out[b].obs_ids.assign(obs.begin() + oo[b], obs.begin() + oo[b + 1]);
      out[b].obs_point_local.assign(opl.begin() + oo[b], opl.begin() + oo[b + 1]);
      out[b].obs_cam_local.assign(ocl.begin() + oo[b], ocl.begin() + oo[b + 1]);
    }
    return out;
  }

 private:
  std::pair<double, double> primal() const {
    double x = 0.0, y = 0.0;
    check(dbag_max_primal(h_, &x, &y));
    return {x, y};
  }
  void use_reference(const ParamState* ref) {
    if (ref && ref != ref_) {
      const dbag_param_view v = ref->view();
      check(dbag_set_reference(h_, &v));
      ref_ = ref;
    }
  }
  dbag_solver* h_ = nullptr;
  int m_, n_;
  int64_t l_;
  int max_iters_;
  bool stop_on_primal_;
  double primal_tol_;
  const ParamState* ref_ = nullptr;
};

// admm_solver.hpp:140-141
inline AdmmResult run_admm(const Problem& problem, const ParamState& init, const AdmmOptions& opts,
                           const BlockConfig& block_config = {},
                           const ParamState* reference = nullptr) {
  AdmmSolver solver(problem, init, opts, block_config);
  return solver.run(reference);
}

}  // namespace gpu
}  // namespace dba
