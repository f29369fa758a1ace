// dbag_io.cpp — the problem file format and metrics CSV behind `dba solve`
// (SURVEY §8(f) row 2), host C++: what makes the device path a drop-in for
// the reference's file-based workflow.
//
// Restates bal_io.cpp (parse_problem_text :100-185, serialize_problem_text
// :197-231, 17-significant-digit scientific format :17-21, angle-axis ->
// Euler conversion :87-96, zero-distortion rule :158-162), the Problem::create
// validation it runs (problem.cpp:12-96), and metrics_csv.cpp:10-38
// (shortest-round-trip std::to_chars, the reference header).
#include <algorithm>
#include <charconv>
#include <cctype>
#include <cmath>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/dbag.h"

namespace {

thread_local std::string g_io_err;
thread_local int32_t g_io_line = -1;

struct IoError {
  int code;
  std::string msg;
  int line;
};

[[noreturn]] void fail(int code, const std::string& msg, int line = -1) {
  throw IoError{code, line >= 0 ? msg + " (line " + std::to_string(line) + ")" : msg, line};
}

std::string format_double(double v) {  // bal_io.cpp:17-21
  char buf[48];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific, 16);
  return std::string(buf, res.ptr);
}

// What a field is, for error messages only: "<kind> <index> <field>[ <sub>]",
// e.g. "observation 5 camera index" or "camera 3 rotation parameter 0"; the
// text is built only when a field fails to parse.
struct Label {
  const char* kind;      // "camera count", "observation", "camera", "point", ...
  long long index = -1;  // -1: kind alone
  const char* field = nullptr;
  int sub = -1;          // -1: no trailing sub-index
  std::string str() const {
    std::string s = kind;
    if (index >= 0) s += " " + std::to_string(index);
    if (field) s += std::string(" ") + field;
    if (sub >= 0) s += " " + std::to_string(sub);
    return s;
  }
};

// Whitespace-separated fields of the problem text, scanned on demand (no
// token array: a multi-million-observation file is parsed in one pass), with
// the 1-based line of the last field returned for messages.
class FieldCursor {
 public:
  explicit FieldCursor(std::string_view text) : t_(text) {}

  // The next field; an empty view at the end of the input.
  std::string_view take() {
    skip_space();
    if (i_ >= t_.size()) return {};
    const size_t start = i_;
    while (i_ < t_.size() && !space(t_[i_])) ++i_;
    field_line_ = line_;
    return t_.substr(start, i_ - start);
  }
  // The next field without consuming it.
  std::string_view look() {
    const size_t i = i_;
    const int line = line_, fl = field_line_;
    const std::string_view f = take();
    i_ = i;
    line_ = line;
    field_line_ = fl;
    return f;
  }
  bool exhausted() {
    skip_space();
    return i_ >= t_.size();
  }
  int field_line() const { return field_line_; }  // of the last field taken (1 before any)
  int next_line() {                                // of the next field
    skip_space();
    return line_;
  }

  std::string_view require(const Label& what) {
    const std::string_view f = take();
    if (f.empty()) fail(DBAG_ERR_PARSE, "unexpected end of file, expected " + what.str(), field_line_);
    return f;
  }
  template <typename T>
  T number(const Label& what) {
    const std::string_view f = require(what);
    T v{};
    const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
    if (r.ec != std::errc{} || r.ptr != f.data() + f.size())
      fail(DBAG_ERR_PARSE, "expected " + what.str() + ", got '" + std::string(f) + "'", field_line_);
    return v;
  }

 private:
  static bool space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }
  void skip_space() {
    for (; i_ < t_.size() && space(t_[i_]); ++i_)
      if (t_[i_] == '\n') ++line_;
  }
  std::string_view t_;
  size_t i_ = 0;
  int line_ = 1, field_line_ = 1;
};

// Rodrigues rotation of an angle-axis vector, then the reference's Euler
// extraction (geometry.cpp:66-80).
void euler_from_angle_axis(const double aa[3], double out[3]) {
  const double theta = std::sqrt(aa[0] * aa[0] + aa[1] * aa[1] + aa[2] * aa[2]);
  if (theta == 0.0) {
    out[0] = out[1] = out[2] = 0.0;
    return;
  }
  const double ax[3] = {aa[0] / theta, aa[1] / theta, aa[2] / theta};
  const double s = std::sin(theta), c = std::cos(theta);
  const double sa[3] = {s * ax[0], s * ax[1], s * ax[2]};
  const double ca[3] = {(1.0 - c) * ax[0], (1.0 - c) * ax[1], (1.0 - c) * ax[2]};
  double R[9];
  double tmp = ca[0] * ax[1];
  R[1] = tmp - sa[2];
  R[3] = tmp + sa[2];
  tmp = ca[0] * ax[2];
  R[2] = tmp + sa[1];
  R[6] = tmp - sa[1];
  tmp = ca[1] * ax[2];
  R[5] = tmp - sa[0];
  R[7] = tmp + sa[0];
  R[0] = ca[0] * ax[0] + c;
  R[4] = ca[1] * ax[1] + c;
  R[8] = ca[2] * ax[2] + c;
  const double beta = std::asin(std::clamp(-R[6], -1.0, 1.0));
  double alpha, gamma;
  if (std::abs(R[6]) < 1.0 - 1e-12) {
    alpha = std::atan2(R[7], R[8]);
    gamma = std::atan2(R[3], R[0]);
  } else {
    alpha = std::atan2(-R[5], R[4]);
    gamma = 0.0;
  }
  out[0] = alpha;
  out[1] = beta;
  out[2] = gamma;
}

// Problem::create (problem.cpp:66-96) + build_visibility checks (:12-64).
void validate_problem(int m, int n, const std::vector<int32_t>& cam, const std::vector<int32_t>& pt,
                      const std::vector<double>& uv, const std::vector<double>& pose,
                      const std::vector<double>& f, const std::vector<double>& pts) {
  for (int j = 0; j < m; ++j) {
    if (!(f[j] > 0.0))
      fail(DBAG_ERR_VALIDATION, "camera " + std::to_string(j) + " has non-positive focal length");
    for (int k = 0; k < 6; ++k)
      if (!std::isfinite(pose[6 * (size_t)j + k]))
        fail(DBAG_ERR_VALIDATION, "camera " + std::to_string(j) + " has non-finite parameters");
  }
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k)
      if (!std::isfinite(pts[3 * (size_t)i + k]))
        fail(DBAG_ERR_VALIDATION, "point " + std::to_string(i) + " has non-finite coordinates");
  for (double v : uv)
    if (!std::isfinite(v)) fail(DBAG_ERR_VALIDATION, "observation has non-finite image coordinates");
  const size_t l = cam.size();
  if (l == 0)
    fail(DBAG_ERR_VALIDATION, "observation list is empty; every camera and point needs coverage");
  for (size_t k = 0; k < l; ++k) {
    if (cam[k] < 0 || cam[k] >= m)
      fail(DBAG_ERR_INDEX_OUT_OF_RANGE, "camera index " + std::to_string(cam[k]) + " outside [0, " +
                                            std::to_string(m) + ")");
    if (pt[k] < 0 || pt[k] >= n)
      fail(DBAG_ERR_INDEX_OUT_OF_RANGE, "point index " + std::to_string(pt[k]) + " outside [0, " +
                                            std::to_string(n) + ")");
  }
  std::vector<std::pair<int, int>> pairs(l);
  for (size_t k = 0; k < l; ++k) pairs[k] = {cam[k], pt[k]};
  std::sort(pairs.begin(), pairs.end());
  const auto dup = std::adjacent_find(pairs.begin(), pairs.end());
  if (dup != pairs.end())
    fail(DBAG_ERR_DUPLICATE_OBSERVATION, "duplicate observation of point " +
                                             std::to_string(dup->second) + " by camera " +
                                             std::to_string(dup->first));
  std::vector<char> cseen(m, 0), pseen(n, 0);
  for (const auto& pr : pairs) {
    cseen[pr.first] = 1;
    pseen[pr.second] = 1;
  }
  for (int j = 0; j < m; ++j)
    if (!cseen[j]) fail(DBAG_ERR_VALIDATION, "camera " + std::to_string(j) + " observes no point");
  for (int i = 0; i < n; ++i)
    if (!pseen[i])
      fail(DBAG_ERR_VALIDATION, "point " + std::to_string(i) + " is observed by no camera");
}

}  // namespace

namespace dbag {
int validate_problem_arrays(int m, int n, int64_t l, const int32_t* cam, const int32_t* pt,
                            const double* uv, const double* pose, const double* f,
                            const double* pts, std::string* msg) {
  try {
    validate_problem(m, n, std::vector<int32_t>(cam, cam + l), std::vector<int32_t>(pt, pt + l),
                     std::vector<double>(uv, uv + 2 * l), std::vector<double>(pose, pose + 6 * (size_t)m),
                     std::vector<double>(f, f + m), std::vector<double>(pts, pts + 3 * (size_t)n));
  } catch (const IoError& e) {
    *msg = e.msg;
    return e.code;
  }
  return DBAG_OK;
}
}  // namespace dbag

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_io_err.clear();
    g_io_line = -1;
    return DBAG_OK;
  } catch (const IoError& e) {
    g_io_err = e.msg;
    g_io_line = e.line;
    return e.code;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    g_io_line = -1;
    return DBAG_ERR_GENERIC;
  }
}

int copy_out(const std::string& s, char* buf, size_t cap, size_t* len) {
  *len = s.size();
  if (buf) {
    if (cap < s.size() + 1) return DBAG_ERR_SIZE_MISMATCH;
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
  }
  return DBAG_OK;
}

}  // namespace

struct dbag_bal {
  int32_t m = 0, n = 0;
  std::vector<int32_t> cam, pt;
  std::vector<double> uv, pose, f, pts;
};

extern "C" {

const char* dbag_io_last_error(int32_t* line) {
  if (line) *line = g_io_line;
  return g_io_err.c_str();
}

// bal_io.cpp:100-185
int dbag_parse_problem_text(const char* text, size_t len, dbag_bal** out, int32_t* m_out,
                            int32_t* n_out, int64_t* l_out) {
  *out = nullptr;
  auto* b = new dbag_bal();
  const int rc = guarded([&] {
    FieldCursor in(std::string_view(text, len));
    bool angle_axis = false;
    if (in.look() == "rotation") {
      in.take();
      const std::string_view v = in.require({"rotation encoding (euler | angle-axis)"});
      if (v == "euler")
        angle_axis = false;
      else if (v == "angle-axis")
        angle_axis = true;
      else
        fail(DBAG_ERR_PARSE, "unknown rotation encoding '" + std::string(v) + "'", in.field_line());
    }
    const long long m = in.number<long long>({"camera count"});
    const long long n = in.number<long long>({"point count"});
    const long long l = in.number<long long>({"observation count"});
    if (m < 1 || n < 1 || l < 1) fail(DBAG_ERR_VALIDATION, "header counts must all be >= 1");
    b->cam.resize(l);
    b->pt.resize(l);
    b->uv.resize(2 * l);
    for (long long k = 0; k < l; ++k) {
      b->cam[k] = (int32_t)in.number<long long>({"observation", k, "camera index"});
      b->pt[k] = (int32_t)in.number<long long>({"observation", k, "point index"});
      b->uv[2 * k] = in.number<double>({"observation", k, "u"});
      b->uv[2 * k + 1] = in.number<double>({"observation", k, "v"});
    }
    b->pose.resize(6 * m);
    b->f.resize(m);
    for (long long j = 0; j < m; ++j) {
      double rot[3];
      for (int k = 0; k < 3; ++k) rot[k] = in.number<double>({"camera", j, "rotation parameter", k});
      if (angle_axis) {
        double e[3];
        euler_from_angle_axis(rot, e);
        rot[0] = e[0];
        rot[1] = e[1];
        rot[2] = e[2];
      }
      for (int k = 0; k < 3; ++k) b->pose[6 * j + k] = rot[k];
      for (int k = 0; k < 3; ++k)
        b->pose[6 * j + 3 + k] = in.number<double>({"camera", j, "translation", k});
      b->f[j] = in.number<double>({"camera", j, "focal length"});
      const double k1 = in.number<double>({"camera", j, "distortion k1"});
      const double k2 = in.number<double>({"camera", j, "distortion k2"});
      if (k1 != 0.0 || k2 != 0.0)
        fail(DBAG_ERR_VALIDATION,
             "camera " + std::to_string(j) + " has nonzero distortion; this camera model has none");
    }
    b->pts.resize(3 * n);
    for (long long i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) b->pts[3 * i + k] = in.number<double>({"point", i, "coordinate", k});
    if (!in.exhausted()) fail(DBAG_ERR_PARSE, "unexpected trailing data", in.next_line());
    b->m = (int32_t)m;
    b->n = (int32_t)n;
    validate_problem(b->m, b->n, b->cam, b->pt, b->uv, b->pose, b->f, b->pts);
  });
  if (rc != DBAG_OK) {
    delete b;
    return rc;
  }
  *out = b;
  *m_out = b->m;
  *n_out = b->n;
  *l_out = (int64_t)b->cam.size();
  return DBAG_OK;
}

int dbag_bal_fetch(const dbag_bal* b, int32_t* cam, int32_t* pt, double* uv, double* pose,
                   double* f, double* pts) {
  auto cp = [](void* d, const void* s, size_t n) {
    if (d && n) std::memcpy(d, s, n);
  };
  cp(cam, b->cam.data(), 4 * b->cam.size());
  cp(pt, b->pt.data(), 4 * b->pt.size());
  cp(uv, b->uv.data(), 8 * b->uv.size());
  cp(pose, b->pose.data(), 8 * b->pose.size());
  cp(f, b->f.data(), 8 * b->f.size());
  cp(pts, b->pts.data(), 8 * b->pts.size());
  return DBAG_OK;
}

void dbag_bal_destroy(dbag_bal* b) { delete b; }

// bal_io.cpp:197-231. Observations from `problem`, cameras/points from `state`.
int dbag_serialize_problem_text(const dbag_problem_view* p, const dbag_param_view* state, char* buf,
                                size_t cap, size_t* len) {
  std::string out;
  const int rc = guarded([&] {
    if (p->num_obs == 0 || p->num_cameras == 0 || p->num_points == 0)
      fail(DBAG_ERR_VALIDATION, "refusing to serialize an empty problem");
    if (state->num_cameras != p->num_cameras || state->num_points != p->num_points)
      fail(DBAG_ERR_SIZE_MISMATCH, "state sizes do not match the problem");
    const double* f = state->cam_f ? state->cam_f : p->cam_f;
    out.reserve(64 * (size_t)(p->num_obs + 3 * p->num_cameras + p->num_points));
    out += "rotation euler\n";
    out += std::to_string(p->num_cameras) + " " + std::to_string(p->num_points) + " " +
           std::to_string(p->num_obs) + "\n";
    for (int64_t k = 0; k < p->num_obs; ++k)
      out += std::to_string(p->obs_cam[k]) + " " + std::to_string(p->obs_pt[k]) + " " +
             format_double(p->obs_uv[2 * k]) + " " + format_double(p->obs_uv[2 * k + 1]) + "\n";
    for (int32_t j = 0; j < state->num_cameras; ++j) {
      for (int k = 0; k < 6; ++k) out += format_double(state->cam_pose[6 * (size_t)j + k]) + "\n";
      out += format_double(f[j]) + "\n";
      out += format_double(0.0) + "\n" + format_double(0.0) + "\n";
    }
    for (int32_t i = 0; i < state->num_points; ++i)
      for (int k = 0; k < 3; ++k) out += format_double(state->points[3 * (size_t)i + k]) + "\n";
  });
  if (rc != DBAG_OK) return rc;
  return copy_out(out, buf, cap, len);
}

// metrics_csv.cpp:16-38
int dbag_metrics_csv(const dbag_iteration_record* trace, int64_t n, char* buf, size_t cap,
                     size_t* len) {
  auto fmt = [](double v) {
    char b[48];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    return std::string(b, r.ptr);
  };
  std::string out =
      "iter,mean_reproj_err,max_primal_x,max_primal_y,camera_mse,point_mse,wall_ms,comm_floats\n";
  for (int64_t k = 0; k < n; ++k) {
    const dbag_iteration_record& r = trace[k];
    out += std::to_string(r.iter) + "," + fmt(r.mean_reproj_err) + "," + fmt(r.max_primal_x) + "," +
           fmt(r.max_primal_y) + "," + fmt(r.camera_mse) + "," + fmt(r.point_mse) + "," +
           fmt(r.wall_ms) + "," + std::to_string(r.comm_floats) + "\n";
  }
  return copy_out(out, buf, cap, len);
}

}  // extern "C"
