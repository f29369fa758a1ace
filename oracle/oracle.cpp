// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp). Restates
// /root/reference/proj/src/{geometry,losses,local_opt,problem,admm_solver,
// parallel,scene_gen}.cpp without Eigen. Compiled with -ffp-contract=off so no
// FMA contraction happens (the reference's x86-64 build emits none).
#include "oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <numbers>
#include <unordered_set>

namespace orc {

namespace {
constexpr double kPi = std::numbers::pi;

std::string num(double v) { return std::to_string(v); }

double sq_norm(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return s;
}
}  // namespace

DepthBelowGuard::DepthBelowGuard(double d, double eps, int pid, int cid)
    : Error("projection depth " + num(d) + " below guard " + num(eps) +
                (pid >= 0 ? " at point " + std::to_string(pid) + ", camera " + std::to_string(cid)
                          : std::string{}),
            kDepthBelowGuard),
      depth(d),
      point_id(pid),
      cam_id(cid) {}

// ---------------------------------------------------------------------------
// geometry — proj/src/geometry.cpp
// ---------------------------------------------------------------------------
Mat3 mat_mul(const Mat3& a, const Mat3& b) {
  Mat3 c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] +
                     a[i * 3 + 2] * b[2 * 3 + j];
  return c;
}

Vec3 mat_vec(const Mat3& a, const Vec3& x) {
  return {a[0] * x[0] + a[1] * x[1] + a[2] * x[2], a[3] * x[0] + a[4] * x[1] + a[5] * x[2],
          a[6] * x[0] + a[7] * x[1] + a[8] * x[2]};
}

// Portable deterministic sin/cos (<= 1 ulp from glibc; +, -, *, rint only, no
// FMA): Cody-Waite reduction by pi/2 with a 33+33+53-bit split, Taylor
// polynomials to x^17 / x^18 on [-pi/4, pi/4], compensated cos. The device's
// exact-numerics mode evaluates the same algorithm, so oracle and device agree
// bit for bit; the reference's std::sin/std::cos (geometry.cpp:9-49) are
// glibc's, whose last-ulp behaviour is unpinned like Eigen's.
// tests/native/sincos_vs_glibc.cpp measures the distance (<= 1 ulp over 1e8
// arguments). Built with -DORC_GLIBC_SINCOS (tests/test_glibc_sincos.py) the
// oracle calls glibc instead: the reference's own geometry path.
#ifdef ORC_GLIBC_SINCOS
void det_sincos(double x, double* sn, double* cs) {
  *sn = std::sin(x);
  *cs = std::cos(x);
}
#else
void det_sincos(double x, double* sn, double* cs) {
  constexpr double kH1 = 1.5707963267341256, kH2 = 6.077100506303966e-11,
                   kH3 = 2.0222662487959506e-21, kTwoOverPi = 0.6366197723675814;
  const double k = std::nearbyint(x * kTwoOverPi);
  const double r = ((x - k * kH1) - k * kH2) - k * kH3;
  const double z = r * r;
  double p = 2.8114572543455206e-15;
  p = p * z + -7.647163731819816e-13;
  p = p * z + 1.6059043836821613e-10;
  p = p * z + -2.505210838544172e-08;
  p = p * z + 2.7557319223985893e-06;
  p = p * z + -0.0001984126984126984;
  p = p * z + 0.008333333333333333;
  p = p * z + -0.16666666666666666;
  const double s = r + (r * z) * p;
  double q = -1.5619206968586225e-16;
  q = q * z + 4.779477332387385e-14;
  q = q * z + -1.1470745597729725e-11;
  q = q * z + 2.08767569878681e-09;
  q = q * z + -2.755731922398589e-07;
  q = q * z + 2.48015873015873e-05;
  q = q * z + -0.001388888888888889;
  q = q * z + 0.041666666666666664;
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double c = w + (((1.0 - w) - hz) + (z * z) * q);
  switch (static_cast<long long>(k) & 3) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
  }
}
#endif

namespace {
// proj/src/geometry.cpp:9-49
Mat3 rot_x(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {1, 0, 0, 0, c, -s, 0, s, c};
}
Mat3 rot_y(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {c, 0, s, 0, 1, 0, -s, 0, c};
}
Mat3 rot_z(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {c, -s, 0, s, c, 0, 0, 0, 1};
}
Mat3 drot_x(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {0, 0, 0, 0, -s, -c, 0, c, -s};
}
Mat3 drot_y(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {-s, 0, c, 0, 0, 0, -c, 0, -s};
}
Mat3 drot_z(double a) {
  double c, s;
  det_sincos(a, &s, &c);
  return {-s, -c, 0, c, -s, 0, 0, 0, 0};
}
}  // namespace

// proj/src/geometry.cpp:62-64
Mat3 rotation_from_euler(double alpha, double beta, double gamma) {
  return mat_mul(mat_mul(rot_z(gamma), rot_y(beta)), rot_x(alpha));
}

// proj/src/geometry.cpp:66-80
Vec3 euler_from_rotation(const Mat3& R) {
  const double beta = std::asin(std::clamp(-R[6], -1.0, 1.0));
  double alpha, gamma;
  if (std::abs(R[6]) < 1.0 - 1e-12) {
    alpha = std::atan2(R[7], R[8]);
    gamma = std::atan2(R[3], R[0]);
  } else {
    alpha = std::atan2(-R[5], R[4]);
    gamma = 0.0;
  }
  return {alpha, beta, gamma};
}

// proj/src/geometry.cpp:82-90
EulerRotation rotation_with_derivatives(double alpha, double beta, double gamma) {
  const Mat3 r1 = rot_x(alpha), r2 = rot_y(beta), r3 = rot_z(gamma);
  EulerRotation o;
  o.R = mat_mul(mat_mul(r3, r2), r1);
  o.dA = mat_mul(mat_mul(r3, r2), drot_x(alpha));
  o.dB = mat_mul(mat_mul(r3, drot_y(beta)), r1);
  o.dG = mat_mul(mat_mul(drot_z(gamma), r2), r1);
  return o;
}

// proj/src/geometry.cpp:92-99
bool try_project(const Vec3& x, const Camera& y, const Guard& g, Vec2* out) {
  const Vec3 rx = mat_vec(rotation_from_euler(y.alpha, y.beta, y.gamma), x);
  const Vec3 w{rx[0] + y.t[0], rx[1] + y.t[1], rx[2] + y.t[2]};
  if (!(w[2] >= g.eps_depth)) return false;
  (*out)[0] = y.f * w[0] / w[2];
  (*out)[1] = y.f * w[1] / w[2];
  return true;
}

// proj/src/geometry.cpp:52-58,141-159
bool try_project_with_jacobians(const Vec3& x, const Camera& y, const Guard& g, Expansion* out) {
  const EulerRotation rot = rotation_with_derivatives(y.alpha, y.beta, y.gamma);
  const Vec3 rx = mat_vec(rot.R, x);
  const Vec3 w{rx[0] + y.t[0], rx[1] + y.t[1], rx[2] + y.t[2]};
  if (!(w[2] >= g.eps_depth)) return false;
  const double inv_z = 1.0 / w[2];
  const double d[2][3] = {{y.f * inv_z, 0.0, -y.f * w[0] * inv_z * inv_z},
                          {0.0, y.f * inv_z, -y.f * w[1] * inv_z * inv_z}};
  out->z = {y.f * w[0] / w[2], y.f * w[1] / w[2]};
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      out->Jp[r][c] = d[r][0] * rot.R[0 * 3 + c] + d[r][1] * rot.R[1 * 3 + c] +
                      d[r][2] * rot.R[2 * 3 + c];
  const Mat3* dRs[3] = {&rot.dA, &rot.dB, &rot.dG};
  for (int k = 0; k < 3; ++k) {
    const Vec3 v = mat_vec(*dRs[k], x);
    for (int r = 0; r < 2; ++r) out->Jc[r][k] = d[r][0] * v[0] + d[r][1] * v[1] + d[r][2] * v[2];
  }
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) out->Jc[r][3 + c] = d[r][c];
  return true;
}

// ---------------------------------------------------------------------------
// losses — proj/src/losses.cpp:7-38
// ---------------------------------------------------------------------------
double loss_value(const Loss& k, const Vec2& r) {
  if (!k.is_huber()) return r[0] * r[0] + r[1] * r[1];
  const double a = std::sqrt(r[0] * r[0] + r[1] * r[1]);
  if (a <= k.delta) return 0.5 * a * a;
  return k.delta * (a - 0.5 * k.delta);
}

Vec2 loss_gradient(const Loss& k, const Vec2& r) {
  if (!k.is_huber()) return {2.0 * r[0], 2.0 * r[1]};
  const double a = std::sqrt(r[0] * r[0] + r[1] * r[1]);
  if (a == 0.0) return {0.0, 0.0};
  if (a <= k.delta) return r;
  const double s = k.delta / a;
  return {s * r[0], s * r[1]};
}

// ---------------------------------------------------------------------------
// Eigen LDLT<MatrixXd, Lower>::compute + solve, restated (Eigen 3.x
// LDLT.h: ldlt_inplace<Lower>::unblocked and LDLT::_solve_impl).
// ---------------------------------------------------------------------------
VecX ldlt_solve(const MatX& A, const VecX& b) {
  const int n = A.rows;
  MatX mat = A;  // only the lower triangle is read
  std::vector<int> transp(n);
  VecX temp(n, 0.0);
  bool found_zero_pivot = false;
  for (int k = 0; k < n; ++k) {
    // largest |diagonal| in the trailing corner (first index on ties)
    int big = k;
    double best = std::abs(mat(k, k));
    for (int i = k + 1; i < n; ++i) {
      if (std::abs(mat(i, i)) > best) {
        best = std::abs(mat(i, i));
        big = i;
      }
    }
    transp[k] = big;
    if (k != big) {
      const int s = n - big - 1;
      for (int j = 0; j < k; ++j) std::swap(mat(k, j), mat(big, j));
      for (int i = 0; i < s; ++i) std::swap(mat(big + 1 + i, k), mat(big + 1 + i, big));
      std::swap(mat(k, k), mat(big, big));
      for (int i = k + 1; i < big; ++i) {
        const double tmp = mat(i, k);
        mat(i, k) = mat(big, i);
        mat(big, i) = tmp;
      }
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = mat(j, j) * mat(k, j);
      double dot = 0.0;
      for (int j = 0; j < k; ++j) dot += mat(k, j) * temp[j];
      mat(k, k) -= dot;
      for (int i = 0; i < rs; ++i) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += mat(k + 1 + i, j) * temp[j];
        mat(k + 1 + i, k) -= s;
      }
    }
    const double akk = mat(k, k);
    const bool pivot_is_valid = std::abs(akk) > 0.0;
    if (k == 0 && !pivot_is_valid) {
      // all-zero diagonal: Eigen records identity transpositions and stops
      for (int j = 0; j < n; ++j) transp[j] = j;
      break;
    }
    if (rs > 0 && pivot_is_valid) {
      for (int i = 0; i < rs; ++i) mat(k + 1 + i, k) /= akk;
    }
    if (!pivot_is_valid) found_zero_pivot = true;
  }
  (void)found_zero_pivot;
  // solve: P b, L^-1, D^-1 (zero for |d| <= DBL_MIN), L^-T, P^T
  VecX x = b;
  for (int k = 0; k < n; ++k) std::swap(x[k], x[transp[k]]);
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= mat(i, j) * x[j];
    x[i] = s;
  }
  const double tol = std::numeric_limits<double>::min();
  for (int i = 0; i < n; ++i) {
    const double d = mat(i, i);
    x[i] = std::abs(d) > tol ? x[i] / d : 0.0;
  }
  // L^-T, column-oriented: once x_j is final, subtract L_ji x_j from every
  // x_i (i < j), for j = n-1 down to 1. Eigen's own summation order here
  // (panelled triangular solve with vectorised dot products) is not pinned at
  // the bit level by anything the reference ships; this order is
  // one faithful restatement, and the one a GPU can run as a parallel sweep.
  for (int j = n - 1; j > 0; --j)
    for (int i = 0; i < j; ++i) x[i] -= mat(j, i) * x[j];
  for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[transp[k]]);
  return x;
}

// ---------------------------------------------------------------------------
// inner solvers — proj/src/local_opt.cpp
// ---------------------------------------------------------------------------
namespace {
constexpr double kDampingInit = 1e-4;  // local_opt.cpp:13
constexpr double kDampingMax = 1e12;   // local_opt.cpp:14
bool finite(const VecX& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}
double norm(const VecX& v) { return std::sqrt(sq_norm(v.data(), (int)v.size())); }
double dot(const VecX& a, const VecX& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
}  // namespace

// proj/src/local_opt.cpp:20-82
InnerResult gauss_newton(const ResidualFn& rf, const JacobianFn& jf, VecX x0, const InnerOptions& o) {
  InnerResult out;
  out.x = std::move(x0);
  VecX r;
  if (!rf(out.x, &r) || !finite(r)) {
    throw ValidationError("gauss_newton: residual undefined at the starting point");
  }
  out.objective = sq_norm(r.data(), (int)r.size());
  const int n = (int)out.x.size();
  for (out.iters = 0; out.iters < o.max_iters; ++out.iters) {
    MatX J;
    if (!jf(out.x, &J)) {
      out.status = kSingular;
      return out;
    }
    VecX g(n, 0.0);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = 0; k < J.rows; ++k) s += J(k, i) * r[k];
      g[i] = 2.0 * s;
    }
    if (norm(g) <= o.grad_tol) {
      out.status = kGradConverged;
      return out;
    }
    MatX H(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int k = 0; k < J.rows; ++k) s += J(k, i) * J(k, j);
        H(i, j) = s;
      }
    VecX rhs(n), damp(n);
    for (int i = 0; i < n; ++i) {
      rhs[i] = -0.5 * g[i];
      damp[i] = std::max(H(i, i), 1e-12);
    }
    double lambda = 0.0;
    bool accepted = false;
    while (!accepted) {
      MatX Hd = H;
      if (lambda > 0.0)
        for (int i = 0; i < n; ++i) Hd(i, i) += lambda * damp[i];
      const VecX delta = ldlt_solve(Hd, rhs);
      if (finite(delta)) {
        VecX trial(n);
        for (int i = 0; i < n; ++i) trial[i] = out.x[i] + delta[i];
        VecX rt;
        if (rf(trial, &rt) && finite(rt) && sq_norm(rt.data(), (int)rt.size()) <= out.objective) {
          out.x = trial;
          r = std::move(rt);
          out.objective = sq_norm(r.data(), (int)r.size());
          accepted = true;
          if (norm(delta) <= o.step_tol * (1.0 + norm(out.x))) {
            out.status = kStepConverged;
            ++out.iters;
            return out;
          }
          break;
        }
      }
      lambda = lambda == 0.0 ? kDampingInit : lambda * 10.0;
      if (lambda > kDampingMax) {
        out.status = finite(delta) ? kLineSearchFailed : kSingular;
        return out;
      }
    }
  }
  out.status = kMaxIters;
  return out;
}

// proj/src/local_opt.cpp:84-186
InnerResult lbfgs(const ValueFn& vf, const GradFn& gf, VecX x0, const InnerOptions& o) {
  InnerResult out;
  out.x = std::move(x0);
  double f0;
  VecX g;
  const bool okf = vf(out.x, &f0);
  const bool okg = gf(out.x, &g);
  if (!okf || !okg || !std::isfinite(f0) || !finite(g)) {
    throw ValidationError("lbfgs: objective undefined at the starting point");
  }
  out.objective = f0;
  const int n = (int)out.x.size();
  struct Pair {
    VecX s, y;
    double rho;
  };
  std::deque<Pair> history;
  double gamma = 1.0;
  for (out.iters = 0; out.iters < o.max_iters; ++out.iters) {
    if (norm(g) <= o.grad_tol) {
      out.status = kGradConverged;
      return out;
    }
    VecX q = g;
    std::vector<double> alpha(history.size());
    for (int k = (int)history.size() - 1; k >= 0; --k) {
      alpha[k] = history[k].rho * dot(history[k].s, q);
      for (int i = 0; i < n; ++i) q[i] -= alpha[k] * history[k].y[i];
    }
    for (int i = 0; i < n; ++i) q[i] *= gamma;
    for (size_t k = 0; k < history.size(); ++k) {
      const double beta = history[k].rho * dot(history[k].y, q);
      for (int i = 0; i < n; ++i) q[i] += (alpha[k] - beta) * history[k].s[i];
    }
    VecX d(n);
    for (int i = 0; i < n; ++i) d[i] = -q[i];
    double slope = dot(g, d);
    if (!(slope < 0.0)) {
      history.clear();
      for (int i = 0; i < n; ++i) d[i] = -g[i];
      slope = -sq_norm(g.data(), n);
    }
    double step = 1.0;
    bool accepted = false;
    double f_trial = 0.0;
    VecX x_trial(n);
    for (int ls = 0; ls < o.max_line_search; ++ls) {
      for (int i = 0; i < n; ++i) x_trial[i] = out.x[i] + step * d[i];
      double f;
      if (vf(x_trial, &f) && std::isfinite(f) && f <= out.objective + o.armijo_c * step * slope) {
        f_trial = f;
        accepted = true;
        break;
      }
      step *= o.backtrack;
    }
    if (!accepted) {
      out.status = kLineSearchFailed;
      return out;
    }
    VecX g_trial;
    if (!gf(x_trial, &g_trial) || !finite(g_trial)) {
      out.status = kLineSearchFailed;
      return out;
    }
    VecX s(n), y(n);
    for (int i = 0; i < n; ++i) {
      s[i] = x_trial[i] - out.x[i];
      y[i] = g_trial[i] - g[i];
    }
    const double sBs = sq_norm(s.data(), n) / gamma;
    double sy = dot(s, y);
    if (sy < 0.2 * sBs) {
      const double theta = 0.8 * sBs / (sBs - sy);
      for (int i = 0; i < n; ++i) y[i] = theta * y[i] + (1.0 - theta) / gamma * s[i];
      sy = dot(s, y);
    }
    if (sy > 1e-12 * norm(s) * norm(y)) {
      history.push_back({s, y, 1.0 / sy});
      gamma = sy / sq_norm(y.data(), n);
      if ((int)history.size() > o.lbfgs_memory) history.pop_front();
    }
    out.x = std::move(x_trial);
    out.objective = f_trial;
    g = std::move(g_trial);
    if (norm(s) <= o.step_tol * (1.0 + norm(out.x))) {
      out.status = kStepConverged;
      ++out.iters;
      return out;
    }
  }
  out.status = kMaxIters;
  return out;
}

// ---------------------------------------------------------------------------
// problem — proj/src/problem.cpp
// ---------------------------------------------------------------------------
// proj/src/problem.cpp:12-64
Visibility build_visibility(const std::vector<Observation>& obs, int m, int n) {
  if (obs.empty()) {
    throw ValidationError("observation list is empty; every camera and point needs coverage");
  }
  for (const Observation& o : obs) {
    if (o.cam_id < 0 || o.cam_id >= m)
      throw IndexOutOfRange("camera index " + std::to_string(o.cam_id) + " outside [0, " +
                            std::to_string(m) + ")");
    if (o.point_id < 0 || o.point_id >= n)
      throw IndexOutOfRange("point index " + std::to_string(o.point_id) + " outside [0, " +
                            std::to_string(n) + ")");
  }
  std::vector<std::pair<int, int>> pairs;
  pairs.reserve(obs.size());
  for (const Observation& o : obs) pairs.emplace_back(o.cam_id, o.point_id);
  std::sort(pairs.begin(), pairs.end());
  const auto dup = std::adjacent_find(pairs.begin(), pairs.end());
  if (dup != pairs.end())
    throw DuplicateObservation("duplicate observation of point " + std::to_string(dup->second) +
                               " by camera " + std::to_string(dup->first));
  Visibility vis;
  vis.points_in_camera.resize(m);
  vis.cameras_seeing_point.resize(n);
  for (const auto& [cam, pt] : pairs) vis.points_in_camera[cam].push_back(pt);
  for (int cam = 0; cam < m; ++cam)
    for (int pt : vis.points_in_camera[cam]) vis.cameras_seeing_point[pt].push_back(cam);
  for (int cam = 0; cam < m; ++cam)
    if (vis.points_in_camera[cam].empty())
      throw ValidationError("camera " + std::to_string(cam) + " observes no point");
  for (int pt = 0; pt < n; ++pt)
    if (vis.cameras_seeing_point[pt].empty())
      throw ValidationError("point " + std::to_string(pt) + " is observed by no camera");
  return vis;
}

// proj/src/problem.cpp:66-96
Problem Problem::create(std::vector<Camera> cameras, std::vector<Vec3> points,
                        std::vector<Observation> observations) {
  for (size_t j = 0; j < cameras.size(); ++j) {
    const Camera& c = cameras[j];
    if (!(c.f > 0.0))
      throw ValidationError("camera " + std::to_string(j) + " has non-positive focal length");
    if (!std::isfinite(c.alpha) || !std::isfinite(c.beta) || !std::isfinite(c.gamma) ||
        !std::isfinite(c.t[0]) || !std::isfinite(c.t[1]) || !std::isfinite(c.t[2]))
      throw ValidationError("camera " + std::to_string(j) + " has non-finite parameters");
  }
  for (size_t i = 0; i < points.size(); ++i)
    for (double v : points[i])
      if (!std::isfinite(v))
        throw ValidationError("point " + std::to_string(i) + " has non-finite coordinates");
  for (const Observation& o : observations)
    if (!std::isfinite(o.z[0]) || !std::isfinite(o.z[1]))
      throw ValidationError("observation has non-finite image coordinates");
  Problem p;
  p.visibility = build_visibility(observations, (int)cameras.size(), (int)points.size());
  p.cameras = std::move(cameras);
  p.points = std::move(points);
  p.observations = std::move(observations);
  return p;
}

namespace {
void check_sizes(const Problem& p, const ParamState& s) {
  if ((int)s.cameras.size() != p.num_cameras() || (int)s.points.size() != p.num_points())
    throw SizeMismatch("state sizes do not match the problem");
}
bool try_residual(const Vec2& z, const Vec3& x, const Camera& y, const Guard& g, Vec2* r) {
  Vec2 p;
  if (!try_project(x, y, g, &p)) return false;
  *r = {z[0] - p[0], z[1] - p[1]};
  return true;
}
// proj/src/problem.cpp:109-121
bool accumulate_residual_norms(const Problem& p, const ParamState& s, const Guard& g, int power,
                               double* out) {
  check_sizes(p, s);
  double sum = 0.0;
  for (const Observation& o : p.observations) {
    Vec2 r;
    if (!try_residual(o.z, s.points[o.point_id], s.cameras[o.cam_id], g, &r)) return false;
    const double sq = r[0] * r[0] + r[1] * r[1];
    sum += power == 1 ? std::sqrt(sq) : sq;
  }
  *out = sum;
  return true;
}
// proj/src/problem.cpp:123-127
double wrap_angle(double a) {
  const double w = std::remainder(a, 2.0 * kPi);
  return w <= -kPi ? w + 2.0 * kPi : w;
}
}  // namespace

bool try_mean_reprojection_error(const Problem& p, const ParamState& s, const Guard& g,
                                 double* out) {
  double sum;
  if (!accumulate_residual_norms(p, s, g, 1, &sum)) return false;
  *out = sum / p.num_observations();
  return true;
}

// proj/src/problem.cpp:140-157
double mean_reprojection_error(const Problem& p, const ParamState& s, const Guard& g) {
  check_sizes(p, s);
  double sum = 0.0;
  for (const Observation& o : p.observations) {
    Vec2 r;
    const Camera& c = s.cameras[o.cam_id];
    if (!try_residual(o.z, s.points[o.point_id], c, g, &r)) {
      const Vec3 rx = mat_vec(rotation_from_euler(c.alpha, c.beta, c.gamma), s.points[o.point_id]);
      throw DepthBelowGuard(rx[2] + c.t[2], g.eps_depth, o.point_id, o.cam_id);
    }
    sum += std::sqrt(r[0] * r[0] + r[1] * r[1]);
  }
  return sum / p.num_observations();
}

bool try_total_squared_error(const Problem& p, const ParamState& s, const Guard& g, double* out) {
  return accumulate_residual_norms(p, s, g, 2, out);
}

// proj/src/problem.cpp:178-202
MseResult parameter_mse(const ParamState& s, const ParamState& ref) {
  if (s.cameras.size() != ref.cameras.size() || s.points.size() != ref.points.size())
    throw SizeMismatch("state and reference sizes differ");
  MseResult out;
  for (size_t j = 0; j < s.cameras.size(); ++j) {
    const Camera& a = s.cameras[j];
    const Camera& b = ref.cameras[j];
    const double da = wrap_angle(a.alpha - b.alpha);
    const double db = wrap_angle(a.beta - b.beta);
    const double dg = wrap_angle(a.gamma - b.gamma);
    const double t0 = a.t[0] - b.t[0], t1 = a.t[1] - b.t[1], t2 = a.t[2] - b.t[2];
    out.camera_mse += da * da + db * db + dg * dg + (t0 * t0 + t1 * t1 + t2 * t2);
  }
  for (size_t i = 0; i < s.points.size(); ++i) {
    const double d0 = s.points[i][0] - ref.points[i][0], d1 = s.points[i][1] - ref.points[i][1],
                 d2 = s.points[i][2] - ref.points[i][2];
    out.point_mse += d0 * d0 + d1 * d1 + d2 * d2;
  }
  if (!s.cameras.empty()) out.camera_mse /= 6.0 * s.cameras.size();
  if (!s.points.empty()) out.point_mse /= 3.0 * s.points.size();
  return out;
}

// ---------------------------------------------------------------------------
// ADMM — proj/src/admm_solver.cpp
// ---------------------------------------------------------------------------
IterationRecord::IterationRecord()
    : mean_reproj_err(std::numeric_limits<double>::infinity()),
      camera_mse(std::numeric_limits<double>::quiet_NaN()),
      point_mse(std::numeric_limits<double>::quiet_NaN()) {}

// proj/src/admm_solver.cpp:14-72
std::vector<LocalBlock> partition(const Problem& p, const BlockConfig& c) {
  if (c.points_per_block < 1 || c.cameras_per_block < 1)
    throw ValidationError("block sizes must be >= 1");
  std::vector<int> order(p.num_observations());
  for (int k = 0; k < p.num_observations(); ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    const Observation& oa = p.observations[a];
    const Observation& ob = p.observations[b];
    return std::pair(oa.cam_id, oa.point_id) < std::pair(ob.cam_id, ob.point_id);
  });
  std::vector<LocalBlock> blocks;
  std::unordered_set<int> pts, cams;
  std::vector<int> pending;
  auto flush = [&] {
    if (pending.empty()) return;
    LocalBlock b;
    b.point_ids.assign(pts.begin(), pts.end());
    b.cam_ids.assign(cams.begin(), cams.end());
    std::sort(b.point_ids.begin(), b.point_ids.end());
    std::sort(b.cam_ids.begin(), b.cam_ids.end());
    b.obs_ids = pending;
    for (int k : pending) {
      const Observation& o = p.observations[k];
      b.obs_point_local.push_back((int)(std::lower_bound(b.point_ids.begin(), b.point_ids.end(),
                                                         o.point_id) -
                                        b.point_ids.begin()));
      b.obs_cam_local.push_back(
          (int)(std::lower_bound(b.cam_ids.begin(), b.cam_ids.end(), o.cam_id) - b.cam_ids.begin()));
    }
    blocks.push_back(std::move(b));
    pts.clear();
    cams.clear();
    pending.clear();
  };
  for (int k : order) {
    const Observation& o = p.observations[k];
    const int new_pt = pts.count(o.point_id) ? 0 : 1;
    const int new_cam = cams.count(o.cam_id) ? 0 : 1;
    if ((int)pts.size() + new_pt > c.points_per_block ||
        (int)cams.size() + new_cam > c.cameras_per_block)
      flush();
    pts.insert(o.point_id);
    cams.insert(o.cam_id);
    pending.push_back(k);
  }
  flush();
  return blocks;
}

// proj/src/admm_solver.cpp:74-101
int64_t communication_cost(const Problem& p, const BlockConfig& c) {
  const std::vector<LocalBlock> blocks = partition(p, c);
  std::vector<std::vector<int>> point_procs(p.num_points()), camera_procs(p.num_cameras());
  for (const LocalBlock& b : blocks) {
    const int proc = b.cam_ids.front();
    for (int i : b.point_ids) point_procs[i].push_back(proc);
    for (int j : b.cam_ids) camera_procs[j].push_back(proc);
  }
  auto distinct = [](std::vector<int>& v) {
    std::sort(v.begin(), v.end());
    return (int64_t)(std::unique(v.begin(), v.end()) - v.begin());
  };
  int64_t total = 0;
  for (auto& procs : point_procs) {
    const int64_t o = distinct(procs);
    total += 3 * o * (o - 1);
  }
  for (auto& procs : camera_procs) {
    const int64_t o = distinct(procs);
    total += 6 * o * (o - 1);
  }
  return total;
}

// proj/src/parallel.cpp:5-91
WorkerPool::WorkerPool(int workers) {
  for (int i = 0; i < workers - 1; ++i) threads_.emplace_back([this] { worker_loop(); });
}
WorkerPool::~WorkerPool() {
  {
    std::lock_guard lock(mutex_);
    stop_ = true;
  }
  start_cv_.notify_all();
  for (std::thread& t : threads_) t.join();
}
void WorkerPool::run(int n, const std::function<void(int)>& fn) {
  if (n <= 0) return;
  if (threads_.empty()) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  {
    std::lock_guard lock(mutex_);
    fn_ = &fn;
    total_ = n;
    next_.store(0, std::memory_order_relaxed);
    remaining_.store(n, std::memory_order_relaxed);
    ++generation_;
  }
  start_cv_.notify_all();
  for (;;) {
    const int i = next_.fetch_add(1, std::memory_order_relaxed);
    if (i >= total_) break;
    fn(i);
    remaining_.fetch_sub(1, std::memory_order_acq_rel);
  }
  std::unique_lock lock(mutex_);
  done_cv_.wait(lock, [this] { return remaining_.load(std::memory_order_acquire) == 0 && active_ == 0; });
  fn_ = nullptr;
}
void WorkerPool::worker_loop() {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(int)>* fn = nullptr;
    {
      std::unique_lock lock(mutex_);
      start_cv_.wait(lock, [&] { return stop_ || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
      fn = fn_;
      // A worker that wakes after run() has already finished this generation
      // sees fn_ == nullptr. Entering the grab loop then would race the next
      // run()'s reset of next_/total_ and call through a null (or dangling)
      // function pointer; it must go back to waiting instead. (The reference's
      // parallel.cpp:63-91 has the same window; fixing it changes no numerics:
      // every index is still run exactly once by someone.)
      if (fn == nullptr) continue;
      ++active_;
    }
    for (;;) {
      const int i = next_.fetch_add(1, std::memory_order_relaxed);
      if (i >= total_) break;
      (*fn)(i);
      remaining_.fetch_sub(1, std::memory_order_acq_rel);
    }
    {
      std::lock_guard lock(mutex_);
      --active_;
    }
    done_cv_.notify_all();
  }
}

// proj/src/admm_solver.cpp:103-142
AdmmSolver::AdmmSolver(const Problem& p, ParamState init, AdmmOptions o, BlockConfig bc)
    : problem_(p), opts_(o) {
  if (!(opts_.rho_x > 0.0) || !(opts_.rho_y > 0.0))
    throw ValidationError("penalty parameters must be positive");
  if (opts_.workers < 1) throw ValidationError("worker count must be >= 1");
  if ((int)init.cameras.size() != p.num_cameras() || (int)init.points.size() != p.num_points())
    throw SizeMismatch("init state sizes do not match the problem");
  mean_reprojection_error(p, init, opts_.guard);
  blocks_ = partition(p, bc);
  comm_floats_ = communication_cost(p, bc);
  state_.consensus = std::move(init);
  const size_t nb = blocks_.size();
  state_.local_points.resize(nb);
  state_.local_cameras.resize(nb);
  state_.dual_r.resize(nb);
  state_.dual_s.resize(nb);
  point_copies_.resize(p.num_points());
  camera_copies_.resize(p.num_cameras());
  for (size_t b = 0; b < nb; ++b) {
    const LocalBlock& blk = blocks_[b];
    for (size_t q = 0; q < blk.point_ids.size(); ++q) {
      state_.local_points[b].push_back(state_.consensus.points[blk.point_ids[q]]);
      state_.dual_r[b].push_back({0, 0, 0});
      point_copies_[blk.point_ids[q]].push_back({(int)b, (int)q});
    }
    for (size_t q = 0; q < blk.cam_ids.size(); ++q) {
      state_.local_cameras[b].push_back(state_.consensus.cameras[blk.cam_ids[q]].pose());
      state_.dual_s[b].push_back({0, 0, 0, 0, 0, 0});
      camera_copies_[blk.cam_ids[q]].push_back({(int)b, (int)q});
    }
  }
  pool_ = std::make_unique<WorkerPool>(opts_.workers);
}

// proj/src/admm_solver.cpp:144-290
void AdmmSolver::local_update(int bi) {
  const LocalBlock& blk = blocks_[bi];
  const int np = (int)blk.point_ids.size();
  const int nc = (int)blk.cam_ids.size();
  const int nobs = (int)blk.obs_ids.size();
  const int dim = 3 * np + 6 * nc;
  const int cam_base = 3 * np;

  std::vector<Vec3> point_target(np);
  for (int q = 0; q < np; ++q)
    for (int k = 0; k < 3; ++k)
      point_target[q][k] =
          state_.consensus.points[blk.point_ids[q]][k] - state_.dual_r[bi][q][k] / opts_.rho_x;
  std::vector<Vec6> cam_target(nc);
  std::vector<double> focal(nc);
  for (int q = 0; q < nc; ++q) {
    const Vec6 pose = state_.consensus.cameras[blk.cam_ids[q]].pose();
    for (int k = 0; k < 6; ++k) cam_target[q][k] = pose[k] - state_.dual_s[bi][q][k] / opts_.rho_y;
    focal[q] = state_.consensus.cameras[blk.cam_ids[q]].f;
  }
  VecX v0(dim);
  for (int q = 0; q < np; ++q)
    for (int k = 0; k < 3; ++k) v0[3 * q + k] = state_.local_points[bi][q][k];
  for (int q = 0; q < nc; ++q)
    for (int k = 0; k < 6; ++k) v0[cam_base + 6 * q + k] = state_.local_cameras[bi][q][k];

  auto camera_at = [&](const VecX& v, int q) {
    Camera c;
    c.set_pose({v[cam_base + 6 * q], v[cam_base + 6 * q + 1], v[cam_base + 6 * q + 2],
                v[cam_base + 6 * q + 3], v[cam_base + 6 * q + 4], v[cam_base + 6 * q + 5]});
    c.f = focal[q];
    return c;
  };
  auto point_at = [&](const VecX& v, int q) -> Vec3 {
    return {v[3 * q], v[3 * q + 1], v[3 * q + 2]};
  };

  InnerResult result;
  if (!opts_.misfit_loss.is_huber()) {
    const double wx = std::sqrt(0.5 * opts_.rho_x);
    const double wy = std::sqrt(0.5 * opts_.rho_y);
    const int rows = 2 * nobs + dim;
    ResidualFn rf = [&](const VecX& v, VecX* r) {
      r->assign(rows, 0.0);
      for (int o = 0; o < nobs; ++o) {
        const Observation& ob = problem_.observations[blk.obs_ids[o]];
        Vec2 pr;
        if (!try_project(point_at(v, blk.obs_point_local[o]), camera_at(v, blk.obs_cam_local[o]),
                         opts_.guard, &pr))
          return false;
        (*r)[2 * o] = ob.z[0] - pr[0];
        (*r)[2 * o + 1] = ob.z[1] - pr[1];
      }
      for (int q = 0; q < np; ++q)
        for (int k = 0; k < 3; ++k)
          (*r)[2 * nobs + 3 * q + k] = wx * (v[3 * q + k] - point_target[q][k]);
      for (int q = 0; q < nc; ++q)
        for (int k = 0; k < 6; ++k)
          (*r)[2 * nobs + cam_base + 6 * q + k] = wy * (v[cam_base + 6 * q + k] - cam_target[q][k]);
      return true;
    };
    JacobianFn jf = [&](const VecX& v, MatX* J) {
      *J = MatX(rows, dim);
      for (int o = 0; o < nobs; ++o) {
        Expansion e;
        if (!try_project_with_jacobians(point_at(v, blk.obs_point_local[o]),
                                        camera_at(v, blk.obs_cam_local[o]), opts_.guard, &e))
          return false;
        const int pc = 3 * blk.obs_point_local[o];
        const int cc = cam_base + 6 * blk.obs_cam_local[o];
        for (int rr = 0; rr < 2; ++rr) {
          for (int c = 0; c < 3; ++c) (*J)(2 * o + rr, pc + c) = -e.Jp[rr][c];
          for (int c = 0; c < 6; ++c) (*J)(2 * o + rr, cc + c) = -e.Jc[rr][c];
        }
      }
      for (int q = 0; q < np; ++q)
        for (int k = 0; k < 3; ++k) (*J)(2 * nobs + 3 * q + k, 3 * q + k) = wx;
      for (int q = 0; q < nc; ++q)
        for (int k = 0; k < 6; ++k)
          (*J)(2 * nobs + cam_base + 6 * q + k, cam_base + 6 * q + k) = wy;
      return true;
    };
    result = gauss_newton(rf, jf, std::move(v0), opts_.inner);
  } else {
    ValueFn vf = [&](const VecX& v, double* out) {
      double total = 0.0;
      for (int o = 0; o < nobs; ++o) {
        const Observation& ob = problem_.observations[blk.obs_ids[o]];
        Vec2 pr;
        if (!try_project(point_at(v, blk.obs_point_local[o]), camera_at(v, blk.obs_cam_local[o]),
                         opts_.guard, &pr))
          return false;
        total += loss_value(opts_.misfit_loss, {ob.z[0] - pr[0], ob.z[1] - pr[1]});
      }
      for (int q = 0; q < np; ++q) {
        const Vec3& xb = state_.consensus.points[blk.point_ids[q]];
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = v[3 * q + k] - xb[k];
        double dd = 0.0;
        for (int k = 0; k < 3; ++k) dd += state_.dual_r[bi][q][k] * d[k];
        total += dd + 0.5 * opts_.rho_x * sq_norm(d, 3);
      }
      for (int q = 0; q < nc; ++q) {
        const Vec6 yb = state_.consensus.cameras[blk.cam_ids[q]].pose();
        double d[6];
        for (int k = 0; k < 6; ++k) d[k] = v[cam_base + 6 * q + k] - yb[k];
        double dd = 0.0;
        for (int k = 0; k < 6; ++k) dd += state_.dual_s[bi][q][k] * d[k];
        total += dd + 0.5 * opts_.rho_y * sq_norm(d, 6);
      }
      *out = total;
      return true;
    };
    GradFn gf = [&](const VecX& v, VecX* g) {
      g->assign(dim, 0.0);
      for (int o = 0; o < nobs; ++o) {
        const Observation& ob = problem_.observations[blk.obs_ids[o]];
        Expansion e;
        if (!try_project_with_jacobians(point_at(v, blk.obs_point_local[o]),
                                        camera_at(v, blk.obs_cam_local[o]), opts_.guard, &e))
          return false;
        const Vec2 lg = loss_gradient(opts_.misfit_loss, {ob.z[0] - e.z[0], ob.z[1] - e.z[1]});
        const int pc = 3 * blk.obs_point_local[o];
        const int cc = cam_base + 6 * blk.obs_cam_local[o];
        for (int c = 0; c < 3; ++c) (*g)[pc + c] -= e.Jp[0][c] * lg[0] + e.Jp[1][c] * lg[1];
        for (int c = 0; c < 6; ++c) (*g)[cc + c] -= e.Jc[0][c] * lg[0] + e.Jc[1][c] * lg[1];
      }
      for (int q = 0; q < np; ++q) {
        const Vec3& xb = state_.consensus.points[blk.point_ids[q]];
        for (int k = 0; k < 3; ++k)
          (*g)[3 * q + k] += state_.dual_r[bi][q][k] + opts_.rho_x * (v[3 * q + k] - xb[k]);
      }
      for (int q = 0; q < nc; ++q) {
        const Vec6 yb = state_.consensus.cameras[blk.cam_ids[q]].pose();
        for (int k = 0; k < 6; ++k)
          (*g)[cam_base + 6 * q + k] +=
              state_.dual_s[bi][q][k] + opts_.rho_y * (v[cam_base + 6 * q + k] - yb[k]);
      }
      return true;
    };
    result = lbfgs(vf, gf, std::move(v0), opts_.inner);
  }
  for (int q = 0; q < np; ++q)
    for (int k = 0; k < 3; ++k) state_.local_points[bi][q][k] = result.x[3 * q + k];
  for (int q = 0; q < nc; ++q)
    for (int k = 0; k < 6; ++k) state_.local_cameras[bi][q][k] = result.x[cam_base + 6 * q + k];
}

// proj/src/admm_solver.cpp:292-316
void AdmmSolver::local_update_all() {
  std::exception_ptr error;
  int error_block = -1;
  std::mutex error_mutex;
  pool_->run((int)blocks_.size(), [&](int b) {
    try {
      local_update(b);
    } catch (...) {
      std::lock_guard lock(error_mutex);
      if (!error) {
        error = std::current_exception();
        error_block = b;
      }
    }
  });
  if (error) {
    try {
      std::rethrow_exception(error);
    } catch (const DepthBelowGuard&) {
      throw;
    } catch (const Error& e) {
      throw Error("local block " + std::to_string(error_block) + ": " + e.what());
    }
  }
}

// proj/src/admm_solver.cpp:318-342
void AdmmSolver::consensus_update() {
  const double inv_rho_x = 1.0 / opts_.rho_x;
  const double inv_rho_y = 1.0 / opts_.rho_y;
  for (int i = 0; i < problem_.num_points(); ++i) {
    const auto& copies = point_copies_[i];
    const Vec3 anchor = state_.local_points[copies.front().first][copies.front().second];
    Vec3 acc{0, 0, 0};
    for (const auto& [b, q] : copies)
      for (int k = 0; k < 3; ++k)
        acc[k] += (state_.local_points[b][q][k] - anchor[k]) + inv_rho_x * state_.dual_r[b][q][k];
    const double cnt = (double)copies.size();
    for (int k = 0; k < 3; ++k) state_.consensus.points[i][k] = anchor[k] + acc[k] / cnt;
  }
  for (int j = 0; j < problem_.num_cameras(); ++j) {
    const auto& copies = camera_copies_[j];
    const Vec6 anchor = state_.local_cameras[copies.front().first][copies.front().second];
    Vec6 acc{0, 0, 0, 0, 0, 0};
    for (const auto& [b, q] : copies)
      for (int k = 0; k < 6; ++k)
        acc[k] += (state_.local_cameras[b][q][k] - anchor[k]) + inv_rho_y * state_.dual_s[b][q][k];
    const double cnt = (double)copies.size();
    Vec6 pose;
    for (int k = 0; k < 6; ++k) pose[k] = anchor[k] + acc[k] / cnt;
    state_.consensus.cameras[j].set_pose(pose);
  }
}

// proj/src/admm_solver.cpp:344-357
void AdmmSolver::dual_update() {
  for (size_t b = 0; b < blocks_.size(); ++b) {
    const LocalBlock& blk = blocks_[b];
    for (size_t q = 0; q < blk.point_ids.size(); ++q) {
      const Vec3& xb = state_.consensus.points[blk.point_ids[q]];
      for (int k = 0; k < 3; ++k)
        state_.dual_r[b][q][k] += opts_.rho_x * (state_.local_points[b][q][k] - xb[k]);
    }
    for (size_t q = 0; q < blk.cam_ids.size(); ++q) {
      const Vec6 yb = state_.consensus.cameras[blk.cam_ids[q]].pose();
      for (int k = 0; k < 6; ++k)
        state_.dual_s[b][q][k] += opts_.rho_y * (state_.local_cameras[b][q][k] - yb[k]);
    }
  }
}

// proj/src/admm_solver.cpp:359-383
double AdmmSolver::max_primal_residual_points() const {
  double worst = 0.0;
  for (size_t b = 0; b < blocks_.size(); ++b)
    for (size_t q = 0; q < blocks_[b].point_ids.size(); ++q) {
      const Vec3& xb = state_.consensus.points[blocks_[b].point_ids[q]];
      double d[3];
      for (int k = 0; k < 3; ++k) d[k] = state_.local_points[b][q][k] - xb[k];
      worst = std::max(worst, std::sqrt(sq_norm(d, 3)));
    }
  return worst;
}
double AdmmSolver::max_primal_residual_cameras() const {
  double worst = 0.0;
  for (size_t b = 0; b < blocks_.size(); ++b)
    for (size_t q = 0; q < blocks_[b].cam_ids.size(); ++q) {
      const Vec6 yb = state_.consensus.cameras[blocks_[b].cam_ids[q]].pose();
      double d[6];
      for (int k = 0; k < 6; ++k) d[k] = state_.local_cameras[b][q][k] - yb[k];
      worst = std::max(worst, std::sqrt(sq_norm(d, 6)));
    }
  return worst;
}

// proj/src/admm_solver.cpp:385-399
Vec3 AdmmSolver::dual_sum_point(int i) const {
  Vec3 s{0, 0, 0};
  for (const auto& [b, q] : point_copies_[i])
    for (int k = 0; k < 3; ++k) s[k] += state_.dual_r[b][q][k];
  return s;
}
Vec6 AdmmSolver::dual_sum_camera(int j) const {
  Vec6 s{0, 0, 0, 0, 0, 0};
  for (const auto& [b, q] : camera_copies_[j])
    for (int k = 0; k < 6; ++k) s[k] += state_.dual_s[b][q][k];
  return s;
}

// proj/src/admm_solver.cpp:401-426
double AdmmSolver::block_objective(int bi) const {
  const LocalBlock& blk = blocks_[bi];
  double total = 0.0;
  for (size_t o = 0; o < blk.obs_ids.size(); ++o) {
    const Observation& ob = problem_.observations[blk.obs_ids[o]];
    Camera cam;
    cam.set_pose(state_.local_cameras[bi][blk.obs_cam_local[o]]);
    cam.f = state_.consensus.cameras[ob.cam_id].f;
    Vec2 pr;
    if (!try_project(state_.local_points[bi][blk.obs_point_local[o]], cam, opts_.guard, &pr))
      return std::numeric_limits<double>::infinity();
    total += loss_value(opts_.misfit_loss, {ob.z[0] - pr[0], ob.z[1] - pr[1]});
  }
  for (size_t q = 0; q < blk.point_ids.size(); ++q) {
    const Vec3& xb = state_.consensus.points[blk.point_ids[q]];
    double d[3], dd = 0.0;
    for (int k = 0; k < 3; ++k) d[k] = state_.local_points[bi][q][k] - xb[k];
    for (int k = 0; k < 3; ++k) dd += state_.dual_r[bi][q][k] * d[k];
    total += dd + 0.5 * opts_.rho_x * sq_norm(d, 3);
  }
  for (size_t q = 0; q < blk.cam_ids.size(); ++q) {
    const Vec6 yb = state_.consensus.cameras[blk.cam_ids[q]].pose();
    double d[6], dd = 0.0;
    for (int k = 0; k < 6; ++k) d[k] = state_.local_cameras[bi][q][k] - yb[k];
    for (int k = 0; k < 6; ++k) dd += state_.dual_s[bi][q][k] * d[k];
    total += dd + 0.5 * opts_.rho_y * sq_norm(d, 6);
  }
  return total;
}

// proj/src/admm_solver.cpp:428-435
int64_t AdmmSolver::ops_per_iteration() const {
  int64_t copies = 0;
  for (const LocalBlock& b : blocks_) copies += (int64_t)b.point_ids.size() + (int64_t)b.cam_ids.size();
  return (int64_t)blocks_.size() + copies;
}

// proj/src/admm_solver.cpp:437-460
IterationRecord AdmmSolver::iterate(const ParamState* ref) {
  const auto t0 = std::chrono::steady_clock::now();
  local_update_all();
  consensus_update();
  dual_update();
  const double wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ++state_.iteration;
  IterationRecord rec;
  rec.iter = state_.iteration;
  double mre;
  rec.mean_reproj_err = try_mean_reprojection_error(problem_, state_.consensus, opts_.guard, &mre)
                            ? mre
                            : std::numeric_limits<double>::infinity();
  rec.max_primal_x = max_primal_residual_points();
  rec.max_primal_y = max_primal_residual_cameras();
  if (ref != nullptr) {
    const MseResult mse = parameter_mse(state_.consensus, *ref);
    rec.camera_mse = mse.camera_mse;
    rec.point_mse = mse.point_mse;
  }
  rec.wall_ms = wall_ms;
  rec.comm_floats = comm_floats_;
  return rec;
}

// proj/src/admm_solver.cpp:462-474
std::vector<IterationRecord> AdmmSolver::run(const ParamState* ref) {
  std::vector<IterationRecord> trace;
  while (state_.iteration < opts_.max_iters) {
    const IterationRecord rec = iterate(ref);
    trace.push_back(rec);
    if (opts_.stop_on_primal && rec.max_primal_x < opts_.primal_tol &&
        rec.max_primal_y < opts_.primal_tol)
      break;
  }
  return trace;
}

// ---------------------------------------------------------------------------
// centralized LM — proj/src/lm_solver.cpp
// ---------------------------------------------------------------------------
namespace {
// lm_solver.cpp:17-25: undamped normal-equation blocks, row-major storage.
struct NormalEquations {
  std::vector<std::array<double, 36>> U;  // per camera, 6x6
  std::vector<std::array<double, 9>> V;   // per point, 3x3
  std::vector<std::array<double, 18>> W;  // per observation, 6x3 = A^T B
  VecX g_cam, g_pt;
  std::vector<std::vector<std::pair<int, int>>> point_obs;  // per point: (cam, obs)
};

// lm_solver.cpp:27-57. A = J_camera (2x6), B = J_point (2x3), r = z - pi.
// Products A^T A etc. as 2-term sums over the rows (r = 0 then 1).
bool assemble(const Problem& p, const ParamState& s, const Guard& g, NormalEquations* eq) {
  const int m = p.num_cameras(), n = p.num_points();
  eq->U.assign(m, {});
  eq->V.assign(n, {});
  eq->W.assign(p.num_observations(), {});
  eq->g_cam.assign(6 * (size_t)m, 0.0);
  eq->g_pt.assign(3 * (size_t)n, 0.0);
  eq->point_obs.assign(n, {});
  for (int k = 0; k < p.num_observations(); ++k) {
    const Observation& ob = p.observations[k];
    Expansion e;
    if (!try_project_with_jacobians(s.points[ob.point_id], s.cameras[ob.cam_id], g, &e))
      return false;
    const double r[2] = {ob.z[0] - e.z[0], ob.z[1] - e.z[1]};
    auto& U = eq->U[ob.cam_id];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) U[6 * i + j] += e.Jc[0][i] * e.Jc[0][j] + e.Jc[1][i] * e.Jc[1][j];
    auto& V = eq->V[ob.point_id];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) V[3 * i + j] += e.Jp[0][i] * e.Jp[0][j] + e.Jp[1][i] * e.Jp[1][j];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 3; ++j)
        eq->W[k][3 * i + j] = e.Jc[0][i] * e.Jp[0][j] + e.Jc[1][i] * e.Jp[1][j];
    for (int i = 0; i < 6; ++i)
      eq->g_cam[6 * (size_t)ob.cam_id + i] += e.Jc[0][i] * r[0] + e.Jc[1][i] * r[1];
    for (int i = 0; i < 3; ++i)
      eq->g_pt[3 * (size_t)ob.point_id + i] += e.Jp[0][i] * r[0] + e.Jp[1][i] * r[1];
    eq->point_obs[ob.point_id].push_back({ob.cam_id, k});
  }
  return true;
}

// lm_solver.cpp:59-127
LmStep solve_step(const NormalEquations& eq, int m, int n, double lambda, bool use_schur) {
  std::vector<std::array<double, 36>> U = eq.U;
  for (int j = 0; j < m; ++j)
    for (int d = 0; d < 6; ++d) U[j][7 * d] += lambda * eq.U[j][7 * d];
  std::vector<std::array<double, 9>> V = eq.V;
  for (int i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) V[i][4 * d] += lambda * eq.V[i][4 * d];
  LmStep step;
  if (use_schur) {
    std::vector<std::array<double, 9>> Vinv(n);
    for (int i = 0; i < n; ++i) {  // V.ldlt().solve(I)
      MatX Vm(3, 3);
      for (int k = 0; k < 9; ++k) Vm.a[k] = V[i][k];
      for (int c = 0; c < 3; ++c) {
        VecX e(3, 0.0);
        e[c] = 1.0;
        const VecX col = ldlt_solve(Vm, e);
        for (int r = 0; r < 3; ++r) Vinv[i][3 * r + c] = col[r];
      }
    }
    const int D = 6 * m;
    MatX S(D, D);
    for (int j = 0; j < m; ++j)
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) S(6 * j + r, 6 * j + c) = U[j][6 * r + c];
    VecX rhs = eq.g_cam;
    for (int i = 0; i < n; ++i) {
      const auto& owners = eq.point_obs[i];
      double vg[3];
      for (int r = 0; r < 3; ++r)
        vg[r] = (Vinv[i][3 * r] * eq.g_pt[3 * (size_t)i] + Vinv[i][3 * r + 1] * eq.g_pt[3 * (size_t)i + 1]) +
                Vinv[i][3 * r + 2] * eq.g_pt[3 * (size_t)i + 2];
      for (const auto& [ja, ka] : owners) {
        const auto& Wa = eq.W[ka];
        for (int r = 0; r < 6; ++r)
          rhs[6 * (size_t)ja + r] -= (Wa[3 * r] * vg[0] + Wa[3 * r + 1] * vg[1]) + Wa[3 * r + 2] * vg[2];
        double WV[18];
        for (int r = 0; r < 6; ++r)
          for (int c = 0; c < 3; ++c)
            WV[3 * r + c] = (Wa[3 * r] * Vinv[i][c] + Wa[3 * r + 1] * Vinv[i][3 + c]) +
                            Wa[3 * r + 2] * Vinv[i][6 + c];
        for (const auto& [jb, kb] : owners) {
          const auto& Wb = eq.W[kb];
          for (int r = 0; r < 6; ++r)
            for (int c = 0; c < 6; ++c)
              S(6 * ja + r, 6 * jb + c) -=
                  (WV[3 * r] * Wb[3 * c] + WV[3 * r + 1] * Wb[3 * c + 1]) + WV[3 * r + 2] * Wb[3 * c + 2];
        }
      }
    }
    step.delta_cameras = ldlt_solve(S, rhs);
    step.delta_points.assign(3 * (size_t)n, 0.0);
    for (int i = 0; i < n; ++i) {
      double acc[3] = {eq.g_pt[3 * (size_t)i], eq.g_pt[3 * (size_t)i + 1], eq.g_pt[3 * (size_t)i + 2]};
      for (const auto& [j, k] : eq.point_obs[i]) {
        const auto& Wk = eq.W[k];
        const double* dc = &step.delta_cameras[6 * (size_t)j];
        for (int c = 0; c < 3; ++c) {  // W^T dc: 6-term sums in order
          double s = 0.0;
          for (int r = 0; r < 6; ++r) s += Wk[3 * r + c] * dc[r];
          acc[c] -= s;
        }
      }
      for (int r = 0; r < 3; ++r)
        step.delta_points[3 * (size_t)i + r] =
            (Vinv[i][3 * r] * acc[0] + Vinv[i][3 * r + 1] * acc[1]) + Vinv[i][3 * r + 2] * acc[2];
    }
  } else {
    const int dim = 6 * m + 3 * n;
    MatX H(dim, dim);
    for (int j = 0; j < m; ++j)
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) H(6 * j + r, 6 * j + c) = U[j][6 * r + c];
    for (int i = 0; i < n; ++i)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) H(6 * m + 3 * i + r, 6 * m + 3 * i + c) = V[i][3 * r + c];
    for (int i = 0; i < n; ++i)
      for (const auto& [j, k] : eq.point_obs[i])
        for (int r = 0; r < 6; ++r)
          for (int c = 0; c < 3; ++c) {
            H(6 * j + r, 6 * m + 3 * i + c) = eq.W[k][3 * r + c];
            H(6 * m + 3 * i + c, 6 * j + r) = eq.W[k][3 * r + c];
          }
    VecX g(dim);
    for (int k = 0; k < 6 * m; ++k) g[k] = eq.g_cam[k];
    for (int k = 0; k < 3 * n; ++k) g[6 * (size_t)m + k] = eq.g_pt[k];
    const VecX delta = ldlt_solve(H, g);
    step.delta_cameras.assign(delta.begin(), delta.begin() + 6 * (size_t)m);
    step.delta_points.assign(delta.begin() + 6 * (size_t)m, delta.end());
  }
  return step;
}

// lm_solver.cpp:129-138
ParamState apply_step(const ParamState& s, const LmStep& st) {
  ParamState out = s;
  for (size_t j = 0; j < out.cameras.size(); ++j) {
    Vec6 p = out.cameras[j].pose();
    for (int k = 0; k < 6; ++k) p[k] += st.delta_cameras[6 * j + k];
    out.cameras[j].set_pose(p);
  }
  for (size_t i = 0; i < out.points.size(); ++i)
    for (int k = 0; k < 3; ++k) out.points[i][k] += st.delta_points[3 * i + k];
  return out;
}

double total_squared_error_throwing(const Problem& p, const ParamState& s, const Guard& g) {
  double t = 0.0;
  if (try_total_squared_error(p, s, g, &t)) return t;
  mean_reprojection_error(p, s, g);  // throws with the offending indices
  return 0.0;
}
}  // namespace

// lm_solver.cpp:142-151
LmStep lm_compute_step(const Problem& p, const ParamState& s, double lambda, bool use_schur,
                       const Guard& g) {
  NormalEquations eq;
  if (!assemble(p, s, g, &eq)) {
    mean_reprojection_error(p, s, g);
    throw DepthBelowGuard(0.0, g.eps_depth);
  }
  return solve_step(eq, p.num_cameras(), p.num_points(), lambda, use_schur);
}

// lm_solver.cpp:153-218
LmResult solve_lm(const Problem& p, const ParamState& init, const LmOptions& o, const Loss& loss,
                  const ParamState* ref) {
  if (loss.is_huber()) throw ValidationError("the LM baseline supports only the squared L2 loss");
  const int m = p.num_cameras(), n = p.num_points();
  LmResult out;
  out.state = init;
  double total = total_squared_error_throwing(p, out.state, o.guard);
  auto record = [&](int iter, double wall_ms) {
    IterationRecord rec;
    rec.iter = iter;
    rec.mean_reproj_err = mean_reprojection_error(p, out.state, o.guard);
    if (ref != nullptr) {
      const MseResult mse = parameter_mse(out.state, *ref);
      rec.camera_mse = mse.camera_mse;
      rec.point_mse = mse.point_mse;
    }
    rec.wall_ms = wall_ms;
    out.trace.push_back(rec);
  };
  record(0, 0.0);
  double lambda = o.lambda_init;
  for (int iter = 1; iter <= o.max_iters; ++iter) {
    if (total < o.error_stop) {
      out.stop = kLmErrorStop;
      return out;
    }
    const auto t0 = std::chrono::steady_clock::now();
    NormalEquations eq;
    if (!assemble(p, out.state, o.guard, &eq)) {
      mean_reprojection_error(p, out.state, o.guard);
      throw DepthBelowGuard(0.0, o.guard.eps_depth);
    }
    bool accepted = false;
    while (!accepted) {
      const LmStep step = solve_step(eq, m, n, lambda, o.use_schur);
      bool fin = true;
      for (double v : step.delta_cameras) fin = fin && std::isfinite(v);
      for (double v : step.delta_points) fin = fin && std::isfinite(v);
      if (fin) {
        const ParamState trial = apply_step(out.state, step);
        double tt = 0.0;
        if (try_total_squared_error(p, trial, o.guard, &tt) && tt < total) {
          out.state = trial;
          total = tt;
          lambda = std::max(lambda / o.lambda_down, 1e-12);
          ++out.accepted_steps;
          accepted = true;
          break;
        }
      }
      lambda *= o.lambda_up;
      if (lambda > o.lambda_max) {
        out.stop = kLmLambdaMax;
        return out;
      }
    }
    const double wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    record(iter, wall_ms);
  }
  out.stop = total < o.error_stop ? kLmErrorStop : kLmMaxIters;
  return out;
}

// ---------------------------------------------------------------------------
// rng + scene generation — proj/include/dba/rng.hpp, proj/src/scene_gen.cpp
// ---------------------------------------------------------------------------
// proj/include/dba/rng.hpp:26-30
double Rng::normal() {
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}
// proj/include/dba/rng.hpp:35-43
uint64_t Rng::uniform_int(uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t r = engine_();
    if (r >= threshold) return r % n;
  }
}

namespace {
Vec3 normalized(const Vec3& v) {
  const double z = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (z > 0.0) {
    const double s = std::sqrt(z);
    return {v[0] / s, v[1] / s, v[2] / s};
  }
  return v;
}
Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
// proj/src/scene_gen.cpp:43-56
Mat3 look_at(const Vec3& center, const Vec3& target) {
  const Vec3 forward =
      normalized({target[0] - center[0], target[1] - center[1], target[2] - center[2]});
  Vec3 up{0, 0, 1};
  if (std::abs(forward[0] * up[0] + forward[1] * up[1] + forward[2] * up[2]) > 1.0 - 1e-9)
    up = {0, 1, 0};
  const Vec3 xc = normalized(cross(up, forward));
  const Vec3 yc = cross(forward, xc);
  return {xc[0], xc[1], xc[2], yc[0], yc[1], yc[2], forward[0], forward[1], forward[2]};
}
}  // namespace

// proj/src/scene_gen.cpp:60-132
GeneratedScene generate_scene(const SceneConfig& c) {
  if (c.n_cameras < 1 || c.n_points < 1)
    throw ValidationError("scene needs at least one camera and one point");
  if (c.visibility_window < 2)
    throw ValidationError("visibility window must be >= 2 so every point is triangulable");
  if (c.visibility_window > c.n_cameras)
    throw ValidationError("visibility window exceeds the number of cameras");
  if (!(c.orbit_radius > 0.0) || !(c.altitude > 0.0))
    throw ValidationError("orbit radius and altitude must be positive");
  if (!(c.focal > 0.0)) throw ValidationError("focal length must be positive");
  if (!(c.box_min[0] <= c.box_max[0] && c.box_min[1] <= c.box_max[1] && c.box_min[2] <= c.box_max[2]))
    throw ValidationError("point region box is inverted");
  if (c.jitter_trans < 0.0 || c.jitter_rot < 0.0)
    throw ValidationError("jitter sigmas must be nonnegative");
  Rng rng(c.rng_seed);
  const int m = c.n_cameras, n = c.n_points, w = c.visibility_window;
  const Vec3 aim{0.5 * (c.box_min[0] + c.box_max[0]), 0.5 * (c.box_min[1] + c.box_max[1]),
                 0.5 * (c.box_min[2] + c.box_max[2])};
  std::vector<Camera> cameras(m);
  for (int j = 0; j < m; ++j) {
    const double theta = 2.0 * kPi * j / m;
    Vec3 center{c.orbit_radius * std::cos(theta), c.orbit_radius * std::sin(theta), c.altitude};
    for (int k = 0; k < 3; ++k) center[k] += rng.normal(0.0, c.jitter_trans);
    const Vec3 angles = euler_from_rotation(look_at(center, aim));
    Camera cam;
    cam.alpha = angles[0] + rng.normal(0.0, c.jitter_rot);
    cam.beta = angles[1] + rng.normal(0.0, c.jitter_rot);
    cam.gamma = angles[2] + rng.normal(0.0, c.jitter_rot);
    cam.f = c.focal;
    const Vec3 rc = mat_vec(rotation_from_euler(cam.alpha, cam.beta, cam.gamma), center);
    cam.t = {-rc[0], -rc[1], -rc[2]};
    cameras[j] = cam;
  }
  const Guard guard;
  std::vector<Vec3> points(n);
  std::vector<Observation> observations;
  observations.reserve((size_t)n * w);
  for (int i = 0; i < n; ++i) {
    bool placed = false;
    for (int attempt = 0; attempt < 100 && !placed; ++attempt) {
      Vec3 p;
      for (int k = 0; k < 3; ++k) p[k] = rng.uniform(c.box_min[k], c.box_max[k]);
      const int start = (int)rng.uniform_int((uint64_t)m);
      std::vector<Observation> window;
      bool ok = true;
      for (int s = 0; s < w && ok; ++s) {
        const int j = (start + s) % m;
        Vec2 z;
        if (try_project(p, cameras[j], guard, &z))
          window.push_back({j, i, z});
        else
          ok = false;
      }
      if (ok) {
        points[i] = p;
        observations.insert(observations.end(), window.begin(), window.end());
        placed = true;
      }
    }
    if (!placed)
      throw Error("point " + std::to_string(i) + " fell behind a camera 100 times",
                  kProjectionFailed);
  }
  GeneratedScene scene;
  scene.problem = Problem::create(cameras, points, std::move(observations));
  scene.ground_truth = {std::move(cameras), std::move(points)};
  return scene;
}

// proj/src/scene_gen.cpp:134-154
ParamState perturb(const ParamState& s, double sigma_cam, double sigma_point, uint64_t seed) {
  if (sigma_cam < 0.0 || sigma_point < 0.0)
    throw ValidationError("perturbation sigmas must be nonnegative");
  Rng rng(seed);
  ParamState out = s;
  for (Camera& cam : out.cameras) {
    cam.alpha += rng.normal(0.0, sigma_cam);
    cam.beta += rng.normal(0.0, sigma_cam);
    cam.gamma += rng.normal(0.0, sigma_cam);
    for (int k = 0; k < 3; ++k) cam.t[k] += rng.normal(0.0, sigma_cam);
  }
  for (Vec3& p : out.points)
    for (int k = 0; k < 3; ++k) p[k] += rng.normal(0.0, sigma_point);
  return out;
}

}  // namespace orc
