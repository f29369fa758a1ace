// ORACLE — TEST INFRASTRUCTURE ONLY. A flat C interface over oracle.cpp so the
// pytest suite (tests/) and bench.py's CPU-baseline leg can drive the CPU
// restatement through ctypes. Never linked into the product.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;
thread_local int g_err_kind = 0;
thread_local int g_err_pt = -1, g_err_cam = -1;
thread_local double g_err_depth = 0.0;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    g_err_kind = 0;
    return 0;
  } catch (const DepthBelowGuard& e) {
    g_err = e.what();
    g_err_kind = kDepthBelowGuard;
    g_err_pt = e.point_id;
    g_err_cam = e.cam_id;
    g_err_depth = e.depth;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_kind = e.kind;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_kind = kGenericError;
  }
  return g_err_kind;
}

std::vector<Camera> cams_from(int m, const double* pose, const double* f) {
  std::vector<Camera> c(m);
  for (int j = 0; j < m; ++j) {
    c[j].set_pose({pose[6 * j], pose[6 * j + 1], pose[6 * j + 2], pose[6 * j + 3], pose[6 * j + 4],
                   pose[6 * j + 5]});
    c[j].f = f[j];
  }
  return c;
}
std::vector<Vec3> pts_from(int n, const double* p) {
  std::vector<Vec3> v(n);
  for (int i = 0; i < n; ++i) v[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return v;
}
ParamState state_from(int m, int n, const double* pose, const double* f, const double* pts) {
  return {cams_from(m, pose, f), pts_from(n, pts)};
}
void state_to(const ParamState& s, double* pose, double* f, double* pts) {
  for (size_t j = 0; j < s.cameras.size(); ++j) {
    const Vec6 p = s.cameras[j].pose();
    for (int k = 0; k < 6; ++k) pose[6 * j + k] = p[k];
    if (f) f[j] = s.cameras[j].f;
  }
  for (size_t i = 0; i < s.points.size(); ++i)
    for (int k = 0; k < 3; ++k) pts[3 * i + k] = s.points[i][k];
}

struct SolverBox {
  Problem problem;
  std::unique_ptr<AdmmSolver> solver;
};
}  // namespace

extern "C" {

typedef struct {
  double rho_x, rho_y;
  int max_iters;
  double primal_tol;
  int stop_on_primal;
  int loss;
  double huber_delta;
  int inner_max_iters;
  double grad_tol, step_tol;
  int lbfgs_memory;
  double armijo_c, backtrack;
  int max_line_search;
  double eps_depth;
  int workers;
  int points_per_block, cameras_per_block;
} orc_options;

typedef struct {
  int iter;
  double mean_reproj_err, max_primal_x, max_primal_y, camera_mse, point_mse, wall_ms;
  long long comm_floats;
} orc_record;

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_error_kind(void) { return g_err_kind; }
void orc_last_error_info(int* pt, int* cam, double* depth) {
  *pt = g_err_pt;
  *cam = g_err_cam;
  *depth = g_err_depth;
}

// ---- geometry / losses --------------------------------------------------
void orc_sincos(int n, const double* x, double* s, double* c) {
  for (int i = 0; i < n; ++i) det_sincos(x[i], &s[i], &c[i]);
}
void orc_rotation_from_euler(double a, double b, double g, double* R) {
  const Mat3 m = rotation_from_euler(a, b, g);
  std::memcpy(R, m.data(), 9 * sizeof(double));
}
void orc_euler_from_rotation(const double* R, double* out) {
  Mat3 m;
  std::memcpy(m.data(), R, 9 * sizeof(double));
  const Vec3 e = euler_from_rotation(m);
  out[0] = e[0];
  out[1] = e[1];
  out[2] = e[2];
}
// cam: alpha,beta,gamma,t0,t1,t2,f. returns 1 if feasible.
int orc_project(const double* x, const double* cam, double eps, double* z) {
  Camera c;
  c.set_pose({cam[0], cam[1], cam[2], cam[3], cam[4], cam[5]});
  c.f = cam[6];
  Vec2 out;
  if (!try_project({x[0], x[1], x[2]}, c, Guard{eps}, &out)) return 0;
  z[0] = out[0];
  z[1] = out[1];
  return 1;
}
int orc_project_with_jacobians(const double* x, const double* cam, double eps, double* z,
                               double* Jp /*2x3*/, double* Jc /*2x6*/) {
  Camera c;
  c.set_pose({cam[0], cam[1], cam[2], cam[3], cam[4], cam[5]});
  c.f = cam[6];
  Expansion e;
  if (!try_project_with_jacobians({x[0], x[1], x[2]}, c, Guard{eps}, &e)) return 0;
  z[0] = e.z[0];
  z[1] = e.z[1];
  for (int r = 0; r < 2; ++r) {
    for (int k = 0; k < 3; ++k) Jp[3 * r + k] = e.Jp[r][k];
    for (int k = 0; k < 6; ++k) Jc[6 * r + k] = e.Jc[r][k];
  }
  return 1;
}
double orc_loss_value(int type, double delta, double r0, double r1) {
  return loss_value(Loss{type, delta}, {r0, r1});
}
void orc_loss_gradient(int type, double delta, double r0, double r1, double* g) {
  const Vec2 v = loss_gradient(Loss{type, delta}, {r0, r1});
  g[0] = v[0];
  g[1] = v[1];
}
void orc_ldlt_solve(int n, const double* A, const double* b, double* x) {
  MatX M(n, n);
  std::memcpy(M.a.data(), A, sizeof(double) * n * n);
  const VecX out = ldlt_solve(M, VecX(b, b + n));
  std::memcpy(x, out.data(), sizeof(double) * n);
}

// ---- generic inner solvers with C callbacks -------------------------------
typedef int (*orc_residual_cb)(int n, const double* x, int rows, double* r, void* ctx);
typedef int (*orc_jacobian_cb)(int n, const double* x, int rows, double* J, void* ctx);
typedef int (*orc_value_cb)(int n, const double* x, double* f, void* ctx);
typedef int (*orc_grad_cb)(int n, const double* x, double* g, void* ctx);

int orc_gauss_newton(int n, int rows, orc_residual_cb rcb, orc_jacobian_cb jcb, void* ctx,
                     const double* x0, const orc_options* o, double* x_out, double* obj,
                     int* status, int* iters) {
  return guarded([&] {
    InnerOptions io;
    io.max_iters = o->inner_max_iters;
    io.grad_tol = o->grad_tol;
    io.step_tol = o->step_tol;
    ResidualFn rf = [&](const VecX& x, VecX* r) {
      r->assign(rows, 0.0);
      return rcb(n, x.data(), rows, r->data(), ctx) != 0;
    };
    JacobianFn jf = [&](const VecX& x, MatX* J) {
      *J = MatX(rows, n);
      return jcb(n, x.data(), rows, J->a.data(), ctx) != 0;
    };
    const InnerResult res = gauss_newton(rf, jf, VecX(x0, x0 + n), io);
    std::memcpy(x_out, res.x.data(), sizeof(double) * n);
    *obj = res.objective;
    *status = res.status;
    *iters = res.iters;
  });
}

int orc_lbfgs(int n, orc_value_cb vcb, orc_grad_cb gcb, void* ctx, const double* x0,
              const orc_options* o, double* x_out, double* obj, int* status, int* iters) {
  return guarded([&] {
    InnerOptions io;
    io.max_iters = o->inner_max_iters;
    io.grad_tol = o->grad_tol;
    io.step_tol = o->step_tol;
    io.lbfgs_memory = o->lbfgs_memory;
    io.armijo_c = o->armijo_c;
    io.backtrack = o->backtrack;
    io.max_line_search = o->max_line_search;
    ValueFn vf = [&](const VecX& x, double* f) { return vcb(n, x.data(), f, ctx) != 0; };
    GradFn gf = [&](const VecX& x, VecX* g) {
      g->assign(n, 0.0);
      return gcb(n, x.data(), g->data(), ctx) != 0;
    };
    const InnerResult res = lbfgs(vf, gf, VecX(x0, x0 + n), io);
    std::memcpy(x_out, res.x.data(), sizeof(double) * n);
    *obj = res.objective;
    *status = res.status;
    *iters = res.iters;
  });
}

// ---- problem ----------------------------------------------------------------
int orc_problem_create(int m, int n, int l, const int* cam, const int* pt, const double* uv,
                       const double* pose, const double* f, const double* pts, void** out) {
  return guarded([&] {
    std::vector<Observation> obs(l);
    for (int k = 0; k < l; ++k) obs[k] = {cam[k], pt[k], {uv[2 * k], uv[2 * k + 1]}};
    auto* p = new Problem(Problem::create(cams_from(m, pose, f), pts_from(n, pts), std::move(obs)));
    *out = p;
  });
}
void orc_problem_destroy(void* p) { delete static_cast<Problem*>(p); }
int orc_problem_sizes(void* hp, int* m, int* n, int* l) {
  const Problem& p = *static_cast<Problem*>(hp);
  *m = p.num_cameras();
  *n = p.num_points();
  *l = p.num_observations();
  return 0;
}
void orc_problem_observations(void* hp, int* cam, int* pt, double* uv) {
  const Problem& p = *static_cast<Problem*>(hp);
  for (int k = 0; k < p.num_observations(); ++k) {
    cam[k] = p.observations[k].cam_id;
    pt[k] = p.observations[k].point_id;
    uv[2 * k] = p.observations[k].z[0];
    uv[2 * k + 1] = p.observations[k].z[1];
  }
}
void orc_problem_nominal(void* hp, double* pose, double* f, double* pts) {
  const Problem& p = *static_cast<Problem*>(hp);
  state_to({p.cameras, p.points}, pose, f, pts);
}
// CSR of the visibility lists: pic_off[m+1], pic[l]; csp_off[n+1], csp[l].
void orc_problem_visibility(void* hp, int* pic_off, int* pic, int* csp_off, int* csp) {
  const Problem& p = *static_cast<Problem*>(hp);
  int o = 0;
  for (int j = 0; j < p.num_cameras(); ++j) {
    pic_off[j] = o;
    for (int v : p.visibility.points_in_camera[j]) pic[o++] = v;
  }
  pic_off[p.num_cameras()] = o;
  o = 0;
  for (int i = 0; i < p.num_points(); ++i) {
    csp_off[i] = o;
    for (int v : p.visibility.cameras_seeing_point[i]) csp[o++] = v;
  }
  csp_off[p.num_points()] = o;
}
int orc_build_visibility(int m, int n, int l, const int* cam, const int* pt) {
  return guarded([&] {
    std::vector<Observation> obs(l);
    for (int k = 0; k < l; ++k) obs[k] = {cam[k], pt[k], {0.0, 0.0}};
    build_visibility(obs, m, n);
  });
}
int orc_mean_reprojection_error(void* hp, const double* pose, const double* f, const double* pts,
                                int m, int n, double eps, double* out) {
  return guarded([&] {
    *out = mean_reprojection_error(*static_cast<Problem*>(hp), state_from(m, n, pose, f, pts),
                                   Guard{eps});
  });
}
int orc_try_mean_reprojection_error(void* hp, const double* pose, const double* f,
                                    const double* pts, int m, int n, double eps, double* out) {
  return guarded([&] {
    if (!try_mean_reprojection_error(*static_cast<Problem*>(hp), state_from(m, n, pose, f, pts),
                                     Guard{eps}, out))
      *out = INFINITY;
  });
}
int orc_total_squared_error(void* hp, const double* pose, const double* f, const double* pts,
                            int m, int n, double eps, double* out) {
  return guarded([&] {
    if (!try_total_squared_error(*static_cast<Problem*>(hp), state_from(m, n, pose, f, pts),
                                 Guard{eps}, out))
      *out = INFINITY;
  });
}
int orc_parameter_mse(int m, int n, const double* pose_a, const double* pts_a, int m2, int n2,
                      const double* pose_b, const double* pts_b, double* out) {
  return guarded([&] {
    std::vector<double> fa(m, 1.0), fb(m2, 1.0);
    const MseResult r = parameter_mse(state_from(m, n, pose_a, fa.data(), pts_a),
                                      state_from(m2, n2, pose_b, fb.data(), pts_b));
    out[0] = r.camera_mse;
    out[1] = r.point_mse;
  });
}

// ---- scene generation ------------------------------------------------------
typedef struct {
  int n_cameras, n_points;
  double orbit_radius, altitude;
  double box_min[3], box_max[3];
  double jitter_trans, jitter_rot;
  int visibility_window;
  double focal;
  unsigned long long rng_seed;
} orc_scene_config;

void orc_scene_config_default(orc_scene_config* c) {
  SceneConfig d;
  c->n_cameras = d.n_cameras;
  c->n_points = d.n_points;
  c->orbit_radius = d.orbit_radius;
  c->altitude = d.altitude;
  for (int k = 0; k < 3; ++k) {
    c->box_min[k] = d.box_min[k];
    c->box_max[k] = d.box_max[k];
  }
  c->jitter_trans = d.jitter_trans;
  c->jitter_rot = d.jitter_rot;
  c->visibility_window = d.visibility_window;
  c->focal = d.focal;
  c->rng_seed = d.rng_seed;
}

// Returns a Problem handle whose nominal cameras/points are the ground truth.
int orc_generate_scene(const orc_scene_config* c, void** out) {
  return guarded([&] {
    SceneConfig s;
    s.n_cameras = c->n_cameras;
    s.n_points = c->n_points;
    s.orbit_radius = c->orbit_radius;
    s.altitude = c->altitude;
    for (int k = 0; k < 3; ++k) {
      s.box_min[k] = c->box_min[k];
      s.box_max[k] = c->box_max[k];
    }
    s.jitter_trans = c->jitter_trans;
    s.jitter_rot = c->jitter_rot;
    s.visibility_window = c->visibility_window;
    s.focal = c->focal;
    s.rng_seed = c->rng_seed;
    GeneratedScene g = generate_scene(s);
    *out = new Problem(std::move(g.problem));
  });
}
int orc_perturb(int m, int n, const double* pose, const double* f, const double* pts,
                double sigma_cam, double sigma_point, unsigned long long seed, double* pose_out,
                double* pts_out) {
  return guarded([&] {
    const ParamState s = perturb(state_from(m, n, pose, f, pts), sigma_cam, sigma_point, seed);
    state_to(s, pose_out, nullptr, pts_out);
  });
}
// Rng stream access for tests: kind 0 uniform, 1 normal, 2 uniform_int(arg).
void orc_rng_draw(unsigned long long seed, int kind, unsigned long long arg, int count,
                  double* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i)
    out[i] = kind == 0 ? r.uniform() : kind == 1 ? r.normal() : (double)r.uniform_int(arg);
}

// ---- ADMM solver -------------------------------------------------------------
static AdmmOptions to_opts(const orc_options* o) {
  AdmmOptions a;
  a.rho_x = o->rho_x;
  a.rho_y = o->rho_y;
  a.max_iters = o->max_iters;
  a.primal_tol = o->primal_tol;
  a.stop_on_primal = o->stop_on_primal != 0;
  a.misfit_loss = Loss{o->loss, o->huber_delta};
  a.inner.max_iters = o->inner_max_iters;
  a.inner.grad_tol = o->grad_tol;
  a.inner.step_tol = o->step_tol;
  a.inner.lbfgs_memory = o->lbfgs_memory;
  a.inner.armijo_c = o->armijo_c;
  a.inner.backtrack = o->backtrack;
  a.inner.max_line_search = o->max_line_search;
  a.guard.eps_depth = o->eps_depth;
  a.workers = o->workers;
  return a;
}

void orc_options_default(orc_options* o) {
  AdmmOptions a;
  o->rho_x = a.rho_x;
  o->rho_y = a.rho_y;
  o->max_iters = a.max_iters;
  o->primal_tol = a.primal_tol;
  o->stop_on_primal = 0;
  o->loss = 0;
  o->huber_delta = 1.0;
  o->inner_max_iters = a.inner.max_iters;
  o->grad_tol = a.inner.grad_tol;
  o->step_tol = a.inner.step_tol;
  o->lbfgs_memory = a.inner.lbfgs_memory;
  o->armijo_c = a.inner.armijo_c;
  o->backtrack = a.inner.backtrack;
  o->max_line_search = a.inner.max_line_search;
  o->eps_depth = a.guard.eps_depth;
  o->workers = 1;
  o->points_per_block = 1;
  o->cameras_per_block = 1;
}

// The solver copies the problem (the reference holds `const Problem&`; the box
// keeps it alive for the solver's lifetime).
int orc_admm_create(void* hp, int m, int n, const double* init_pose, const double* init_f,
                    const double* init_pts, const orc_options* o, void** out) {
  return guarded([&] {
    auto box = std::make_unique<SolverBox>();
    box->problem = *static_cast<Problem*>(hp);
    box->solver = std::make_unique<AdmmSolver>(
        box->problem, state_from(m, n, init_pose, init_f, init_pts), to_opts(o),
        BlockConfig{o->points_per_block, o->cameras_per_block});
    *out = box.release();
  });
}
void orc_admm_destroy(void* h) { delete static_cast<SolverBox*>(h); }
static AdmmSolver& S(void* h) { return *static_cast<SolverBox*>(h)->solver; }

int orc_admm_local_update(void* h, int b) { return guarded([&] { S(h).local_update(b); }); }
int orc_admm_local_update_all(void* h) { return guarded([&] { S(h).local_update_all(); }); }
int orc_admm_consensus_update(void* h) { return guarded([&] { S(h).consensus_update(); }); }
int orc_admm_dual_update(void* h) { return guarded([&] { S(h).dual_update(); }); }

static void rec_to(const IterationRecord& r, orc_record* o) {
  o->iter = r.iter;
  o->mean_reproj_err = r.mean_reproj_err;
  o->max_primal_x = r.max_primal_x;
  o->max_primal_y = r.max_primal_y;
  o->camera_mse = r.camera_mse;
  o->point_mse = r.point_mse;
  o->wall_ms = r.wall_ms;
  o->comm_floats = r.comm_floats;
}

int orc_admm_iterate(void* h, const double* ref_pose, const double* ref_pts, orc_record* out) {
  return guarded([&] {
    AdmmSolver& s = S(h);
    const int m = (int)s.state().consensus.cameras.size();
    const int n = (int)s.state().consensus.points.size();
    ParamState ref;
    const ParamState* rp = nullptr;
    if (ref_pose) {
      std::vector<double> ones(m, 1.0);
      ref = state_from(m, n, ref_pose, ones.data(), ref_pts);
      rp = &ref;
    }
    rec_to(s.iterate(rp), out);
  });
}
int orc_admm_run(void* h, const double* ref_pose, const double* ref_pts, orc_record* trace,
                 int cap, int* n_out) {
  return guarded([&] {
    AdmmSolver& s = S(h);
    const int m = (int)s.state().consensus.cameras.size();
    const int n = (int)s.state().consensus.points.size();
    ParamState ref;
    const ParamState* rp = nullptr;
    if (ref_pose) {
      std::vector<double> ones(m, 1.0);
      ref = state_from(m, n, ref_pose, ones.data(), ref_pts);
      rp = &ref;
    }
    const auto tr = s.run(rp);
    *n_out = (int)tr.size();
    for (int k = 0; k < (int)tr.size() && k < cap; ++k) rec_to(tr[k], &trace[k]);
  });
}
void orc_admm_get_consensus(void* h, double* pose, double* f, double* pts) {
  state_to(S(h).state().consensus, pose, f, pts);
}
void orc_admm_set_consensus(void* h, const double* pose, const double* pts) {
  AdmmState& st = S(h).state();
  for (size_t j = 0; j < st.consensus.cameras.size(); ++j)
    st.consensus.cameras[j].set_pose({pose[6 * j], pose[6 * j + 1], pose[6 * j + 2],
                                      pose[6 * j + 3], pose[6 * j + 4], pose[6 * j + 5]});
  for (size_t i = 0; i < st.consensus.points.size(); ++i)
    st.consensus.points[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
}
int orc_admm_num_blocks(void* h) { return (int)S(h).blocks().size(); }
int orc_admm_iteration(void* h) { return S(h).state().iteration; }
// Per-block copies for (1,1) blocks (one point and one camera per block).
void orc_admm_get_copies(void* h, double* lp, double* lc, double* r, double* s) {
  const AdmmState& st = S(h).state();
  for (size_t b = 0; b < st.local_points.size(); ++b) {
    for (int k = 0; k < 3; ++k) {
      lp[3 * b + k] = st.local_points[b][0][k];
      r[3 * b + k] = st.dual_r[b][0][k];
    }
    for (int k = 0; k < 6; ++k) {
      lc[6 * b + k] = st.local_cameras[b][0][k];
      s[6 * b + k] = st.dual_s[b][0][k];
    }
  }
}
void orc_admm_set_copies(void* h, const double* lp, const double* lc, const double* r,
                         const double* s) {
  AdmmState& st = S(h).state();
  for (size_t b = 0; b < st.local_points.size(); ++b) {
    for (int k = 0; k < 3; ++k) {
      st.local_points[b][0][k] = lp[3 * b + k];
      st.dual_r[b][0][k] = r[3 * b + k];
    }
    for (int k = 0; k < 6; ++k) {
      st.local_cameras[b][0][k] = lc[6 * b + k];
      st.dual_s[b][0][k] = s[6 * b + k];
    }
  }
}
// Copies of any BlockConfig, flattened block by block in id order ([PC][3],
// [CC][6], [PC][3], [CC][6]); dir 0 reads, 1 writes.
void orc_admm_num_copies(void* h, long long* pc, long long* cc) {
  long long a = 0, c = 0;
  for (const LocalBlock& b : S(h).blocks()) {
    a += (long long)b.point_ids.size();
    c += (long long)b.cam_ids.size();
  }
  *pc = a;
  *cc = c;
}
void orc_admm_copies_flat(void* h, double* lp, double* lc, double* r, double* s, int dir) {
  AdmmState& st = S(h).state();
  size_t a = 0, c = 0;
  for (size_t b = 0; b < st.local_points.size(); ++b) {
    for (size_t q = 0; q < st.local_points[b].size(); ++q, ++a)
      for (int k = 0; k < 3; ++k) {
        if (dir == 0) {
          lp[3 * a + k] = st.local_points[b][q][k];
          r[3 * a + k] = st.dual_r[b][q][k];
        } else {
          st.local_points[b][q][k] = lp[3 * a + k];
          st.dual_r[b][q][k] = r[3 * a + k];
        }
      }
    for (size_t q = 0; q < st.local_cameras[b].size(); ++q, ++c)
      for (int k = 0; k < 6; ++k) {
        if (dir == 0) {
          lc[6 * c + k] = st.local_cameras[b][q][k];
          s[6 * c + k] = st.dual_s[b][q][k];
        } else {
          st.local_cameras[b][q][k] = lc[6 * c + k];
          st.dual_s[b][q][k] = s[6 * c + k];
        }
      }
  }
}
// Block structure: counts per block then flattened ids.
void orc_admm_block_sizes(void* h, int* np, int* nc, int* no) {
  const auto& bl = S(h).blocks();
  for (size_t b = 0; b < bl.size(); ++b) {
    np[b] = (int)bl[b].point_ids.size();
    nc[b] = (int)bl[b].cam_ids.size();
    no[b] = (int)bl[b].obs_ids.size();
  }
}
void orc_admm_block_ids(void* h, int* pts, int* cams, int* obs, int* obs_pl, int* obs_cl) {
  int a = 0, c = 0, o = 0;
  for (const LocalBlock& b : S(h).blocks()) {
    for (int v : b.point_ids) pts[a++] = v;
    for (int v : b.cam_ids) cams[c++] = v;
    for (size_t k = 0; k < b.obs_ids.size(); ++k) {
      obs[o] = b.obs_ids[k];
      obs_pl[o] = b.obs_point_local[k];
      obs_cl[o] = b.obs_cam_local[k];
      ++o;
    }
  }
}
void orc_admm_max_primal(void* h, double* x, double* y) {
  *x = S(h).max_primal_residual_points();
  *y = S(h).max_primal_residual_cameras();
}
void orc_admm_dual_sum_point(void* h, int i, double* out) {
  const Vec3 v = S(h).dual_sum_point(i);
  for (int k = 0; k < 3; ++k) out[k] = v[k];
}
void orc_admm_dual_sum_camera(void* h, int j, double* out) {
  const Vec6 v = S(h).dual_sum_camera(j);
  for (int k = 0; k < 6; ++k) out[k] = v[k];
}
double orc_admm_block_objective(void* h, int b) { return S(h).block_objective(b); }
long long orc_admm_ops_per_iteration(void* h) { return S(h).ops_per_iteration(); }
long long orc_admm_comm_floats(void* h) { return S(h).comm_floats_per_iteration(); }

// ---- centralized LM (lm_solver.cpp)
typedef struct {
  int max_iters;
  double error_stop, lambda_init, lambda_max, lambda_up, lambda_down;
  int use_schur;
  double eps_depth;
} orc_lm_options;

void orc_lm_options_default(orc_lm_options* o) {
  const LmOptions d;
  o->max_iters = d.max_iters;
  o->error_stop = d.error_stop;
  o->lambda_init = d.lambda_init;
  o->lambda_max = d.lambda_max;
  o->lambda_up = d.lambda_up;
  o->lambda_down = d.lambda_down;
  o->use_schur = d.use_schur ? 1 : 0;
  o->eps_depth = d.guard.eps_depth;
}

static LmOptions lm_opts_from(const orc_lm_options* o) {
  LmOptions r;
  r.max_iters = o->max_iters;
  r.error_stop = o->error_stop;
  r.lambda_init = o->lambda_init;
  r.lambda_max = o->lambda_max;
  r.lambda_up = o->lambda_up;
  r.lambda_down = o->lambda_down;
  r.use_schur = o->use_schur != 0;
  r.guard.eps_depth = o->eps_depth;
  return r;
}

int orc_lm_solve(void* hp, const double* pose, const double* f, const double* pts,
                 const orc_lm_options* o, int loss_type, const double* ref_pose,
                 const double* ref_pts, double* out_pose, double* out_pts, orc_record* trace,
                 int cap, int* n_trace, int* stop, int* accepted) {
  return guarded([&] {
    const Problem& p = *static_cast<Problem*>(hp);
    const int m = p.num_cameras(), n = p.num_points();
    const ParamState init = state_from(m, n, pose, f, pts);
    ParamState ref;
    if (ref_pose) ref = state_from(m, n, ref_pose, f, ref_pts);
    Loss loss;
    loss.type = loss_type;
    const LmResult r = solve_lm(p, init, lm_opts_from(o), loss, ref_pose ? &ref : nullptr);
    state_to(r.state, out_pose, nullptr, out_pts);
    *n_trace = (int)r.trace.size();
    for (int k = 0; k < (int)r.trace.size() && k < cap; ++k) rec_to(r.trace[k], trace + k);
    *stop = r.stop;
    *accepted = r.accepted_steps;
  });
}

int orc_lm_compute_step(void* hp, const double* pose, const double* f, const double* pts,
                        double lambda, int use_schur, double eps_depth, double* dc, double* dp) {
  return guarded([&] {
    const Problem& p = *static_cast<Problem*>(hp);
    Guard g;
    g.eps_depth = eps_depth;
    const LmStep st = lm_compute_step(p, state_from(p.num_cameras(), p.num_points(), pose, f, pts),
                                      lambda, use_schur != 0, g);
    std::memcpy(dc, st.delta_cameras.data(), sizeof(double) * st.delta_cameras.size());
    std::memcpy(dp, st.delta_points.data(), sizeof(double) * st.delta_points.size());
  });
}

int orc_partition_count(void* hp, int ppb, int cpb, int* nblocks) {
  return guarded([&] { *nblocks = (int)partition(*static_cast<Problem*>(hp), {ppb, cpb}).size(); });
}
int orc_communication_cost(void* hp, int ppb, int cpb, long long* out) {
  return guarded([&] { *out = communication_cost(*static_cast<Problem*>(hp), {ppb, cpb}); });
}

}  // extern "C"
