// dbag_lm.cu — the centralized Levenberg–Marquardt comparator (SURVEY §8(f)
// row 3; proj/src/lm_solver.cpp, proj/include/dba/lm_solver.hpp) on the B200.
// Compiled with -fmad=false; projections and Jacobians are the EXACT camera
// model shared with the ADMM kernels (dbag_exact_geom.cuh).
//
// One LM iteration:
//  - assemble (lm_solver.cpp:27-57): one thread per observation forms A = J_c,
//    B = J_p, r and W = A^T B; U_j / g_cam_j are summed per camera (one CTA:
//    strided partial sums and a fixed-order tree) and V_i / g_pt_i per point
//    (one thread, the reference's order);
//  - Schur step (:59-127): V_i damped and inverted by the restated pivoted
//    LDLT (one thread per point); the 6m x 6m complement S = U - W V^-1 W^T and
//    its right-hand side are built by one CTA per camera block row, whose warps
//    own disjoint target blocks and each walk the camera's points in ascending
//    id — the order in which the reference's point loop reaches that row — so
//    every block sums in the reference's order, without CTA barriers;
//  - S is factored by cuSOLVER (Cholesky; Bunch–Kaufman if S is not positive
//    definite) — the one dense library solve, as SURVEY §8(f) plans. Eigen's
//    blocked LDLT is not bit-pinnable, so parity is tolerance-level;
//  - back substitution of the points, trial, total squared error (fixed-order
//    device reductions), accept / reject and the damping update on the host.
// The dense (non-Schur) step of the reference is kept for its test
// (use_schur = 0), limited to small systems.
#include <cusolverDn.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/dbag.h"
#include "dbag_errors.h"
#include "dbag_exact_geom.cuh"

using namespace dbag;

namespace {

struct LmErr {
  int code;
  std::string msg;
  int32_t pt = -1, cam = -1;
  double depth = 0.0;
};
#define LK(call)                                                                               \
  do {                                                                                         \
    const cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                                     \
      throw LmErr{DBAG_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " at " #call}; \
  } while (0)
#define LS(call)                                                                     \
  do {                                                                               \
    const cusolverStatus_t s_ = (call);                                              \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                               \
      throw LmErr{DBAG_ERR_CUDA, "cuSOLVER status " + std::to_string((int)s_) + " at " #call}; \
  } while (0)

constexpr int kRedBlocks = 592;
constexpr int kRedThreads = 256;

// Device view (by value).
struct LmDev {
  int32_t m, n;
  int64_t l;
  const int32_t* cam;       // [l] input order
  const int32_t* pt;        // [l]
  const double* uv;         // [l][2]
  const int64_t* cam_off;   // [m+1]
  const int32_t* cam_obs;   // camera's observations, ascending k
  const int32_t* cam_obs_p; // camera's observations, ascending point id
  const int64_t* pt_off;    // [n+1]
  const int32_t* pt_obs;    // point's observations, ascending k
  double* J;                // [l][18]: [J_p | J_c] row 0, row 1 (ejac layout)
  double* r;                // [l][2]
  double* W;                // [l][18]: A^T B (6 x 3, row-major)
  double* U;                // [m][36]
  double* V;                // [n][9]
  double* gc;               // [6m]
  double* gp;               // [3n]
  double* Vinv;             // [n][9]
  double* vg;               // [n][3]
  double* S;                // [D][D] column-major (D = 6m, or 6m+3n dense)
  double* rhs;              // [D]
  double* dp;               // [3n]
  // Schur pair lists (static): block (pair_ja[p], pair_jb[p]) gets one
  // contribution per point both cameras observe, triplets [pair_off[p],
  // pair_off[p+1]) of (obs in ja, obs in jb), points ascending
  int64_t npairs;
  const int32_t* pair_ja;
  const int32_t* pair_jb;
  const int64_t* pair_off;
  const int32_t* trip_a;
  const int32_t* trip_b;
  const int32_t* trip_i;    // the shared point (saves a dependent load)
  double eps;
};

// ---- assemble ----------------------------------------------------------------
__global__ void k_lm_jac(LmDev d, const double* pose, const double* f, const double* pts,
                         unsigned long long* bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.l) return;
  const int j = d.cam[k], i = d.pt[k];
  double v9[9];
  for (int c = 0; c < 3; ++c) v9[c] = pts[3 * (int64_t)i + c];
  for (int c = 0; c < 6; ++c) v9[3 + c] = pose[6 * (int64_t)j + c];
  exact::ETrig t;
  double R[9], w[3], z[2];
  if (!exact::eproject(v9, f[j], d.eps, t, R, w, z)) {
    atomicMin(bad, (unsigned long long)k);
    return;
  }
  double A0[9], A1[9];
  exact::erot(t, R);
  exact::ejac(v9, t, R, w, f[j], A0, A1);
  double* J = d.J + 18 * k;
  for (int c = 0; c < 9; ++c) {
    J[c] = A0[c];
    J[9 + c] = A1[c];
  }
  d.r[2 * k] = d.uv[2 * k] - z[0];
  d.r[2 * k + 1] = d.uv[2 * k + 1] - z[1];
  double* W = d.W + 18 * k;  // W(i,j) = Jc0_i Jp0_j + Jc1_i Jp1_j
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 3; ++b) W[3 * a + b] = A0[3 + a] * A0[b] + A1[3 + a] * A1[b];
}

// U_j and g_cam_j (42 sums per camera): each of the CTA's 256 threads sums a
// strided subset of the camera's observations (ascending k), then a fixed-order
// tree. Deterministic; the order differs from the reference's sequential sum,
// which the LM's tolerance parity (cuSOLVER) already allows.
constexpr int kCamThreadsLm = 256;
__global__ void __launch_bounds__(kCamThreadsLm) k_lm_cam(LmDev d) {
  __shared__ double red[kCamThreadsLm / 32][42];
  const int j = blockIdx.x, t = threadIdx.x;
  double acc[42];
#pragma unroll
  for (int e = 0; e < 42; ++e) acc[e] = 0.0;
  for (int64_t q = d.cam_off[j] + t; q < d.cam_off[j + 1]; q += kCamThreadsLm) {
    const int64_t k = d.cam_obs[q];
    const double* J = d.J + 18 * k;
    double c0[6], c1[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      c0[a] = J[3 + a];
      c1[a] = J[12 + a];
    }
    const double r0 = d.r[2 * k], r1 = d.r[2 * k + 1];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
#pragma unroll
      for (int b = 0; b < 6; ++b) acc[6 * a + b] += c0[a] * c0[b] + c1[a] * c1[b];
      acc[36 + a] += c0[a] * r0 + c1[a] * r1;
    }
  }
#pragma unroll
  for (int e = 0; e < 42; ++e)
    for (int off = 16; off > 0; off >>= 1) acc[e] += __shfl_down_sync(0xffffffffu, acc[e], off);
  if ((t & 31) == 0)
#pragma unroll
    for (int e = 0; e < 42; ++e) red[t >> 5][e] = acc[e];
  __syncthreads();
  if (t < 42) {
    double s = 0.0;
    for (int w = 0; w < kCamThreadsLm / 32; ++w) s += red[w][t];
    if (t < 36)
      d.U[36 * (int64_t)j + t] = s;
    else
      d.gc[6 * (int64_t)j + t - 36] = s;
  }
}

// V_i and g_pt_i, observations in input order.
__global__ void k_lm_pt(LmDev d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  double V[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, g[3] = {0, 0, 0};
  for (int64_t q = d.pt_off[i]; q < d.pt_off[i + 1]; ++q) {
    const int64_t k = d.pt_obs[q];
    const double* J = d.J + 18 * k;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) V[3 * a + b] += J[a] * J[b] + J[9 + a] * J[9 + b];
    for (int a = 0; a < 3; ++a) g[a] += J[a] * d.r[2 * k] + J[9 + a] * d.r[2 * k + 1];
  }
  for (int c = 0; c < 9; ++c) d.V[9 * i + c] = V[c];
  for (int c = 0; c < 3; ++c) d.gp[3 * i + c] = g[c];
}

// ---- the restated pivoted LDLT (oracle.cpp ldlt_solve), n = 3 ----------------
// Factor once, then solve for each right-hand side: the same operations the
// oracle performs per call.
struct Ldlt3 {
  double m[9];  // row-major; lower triangle used
  int transp[3];
};
__device__ void ldlt3_factor(const double A[9], Ldlt3& F) {
  for (int c = 0; c < 9; ++c) F.m[c] = A[c];
  double* mat = F.m;
  double temp[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k) {
    int big = k;
    double best = fabs(mat[4 * k]);
    for (int i = k + 1; i < 3; ++i)
      if (fabs(mat[4 * i]) > best) {
        best = fabs(mat[4 * i]);
        big = i;
      }
    F.transp[k] = big;
    if (k != big) {
      const int s = 3 - big - 1;
      for (int j = 0; j < k; ++j) {
        const double x = mat[3 * k + j];
        mat[3 * k + j] = mat[3 * big + j];
        mat[3 * big + j] = x;
      }
      for (int i = 0; i < s; ++i) {
        const double x = mat[3 * (big + 1 + i) + k];
        mat[3 * (big + 1 + i) + k] = mat[3 * (big + 1 + i) + big];
        mat[3 * (big + 1 + i) + big] = x;
      }
      const double x = mat[4 * k];
      mat[4 * k] = mat[4 * big];
      mat[4 * big] = x;
      for (int i = k + 1; i < big; ++i) {
        const double tmp = mat[3 * i + k];
        mat[3 * i + k] = mat[3 * big + i];
        mat[3 * big + i] = tmp;
      }
    }
    const int rs = 3 - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = mat[4 * j] * mat[3 * k + j];
      double dot = 0.0;
      for (int j = 0; j < k; ++j) dot += mat[3 * k + j] * temp[j];
      mat[4 * k] -= dot;
      for (int i = 0; i < rs; ++i) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += mat[3 * (k + 1 + i) + j] * temp[j];
        mat[3 * (k + 1 + i) + k] -= s;
      }
    }
    const double akk = mat[4 * k];
    const bool valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      for (int j = 0; j < 3; ++j) F.transp[j] = j;
      break;
    }
    if (rs > 0 && valid)
      for (int i = 0; i < rs; ++i) mat[3 * (k + 1 + i) + k] /= akk;
  }
}
__device__ void ldlt3_solve(const Ldlt3& F, const double b[3], double x[3]) {
  const double* mat = F.m;
  for (int c = 0; c < 3; ++c) x[c] = b[c];
  for (int k = 0; k < 3; ++k) {
    const double t = x[k];
    x[k] = x[F.transp[k]];
    x[F.transp[k]] = t;
  }
  for (int i = 0; i < 3; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= mat[3 * i + j] * x[j];
    x[i] = s;
  }
  const double tol = 2.2250738585072014e-308;
  for (int i = 0; i < 3; ++i) {
    const double dd = mat[4 * i];
    x[i] = fabs(dd) > tol ? x[i] / dd : 0.0;
  }
  for (int j = 2; j > 0; --j)
    for (int i = 0; i < j; ++i) x[i] -= mat[3 * j + i] * x[j];
  for (int k = 2; k >= 0; --k) {
    const double t = x[k];
    x[k] = x[F.transp[k]];
    x[F.transp[k]] = t;
  }
}

// V damped (lm_solver.cpp:67-71), Vinv = V.ldlt().solve(I) (:77-79), vg = Vinv g_pt.
__global__ void k_lm_vinv(LmDev d, double lambda) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  double V[9];
  for (int c = 0; c < 9; ++c) V[c] = d.V[9 * i + c];
  for (int a = 0; a < 3; ++a) V[4 * a] += lambda * d.V[9 * i + 4 * a];
  Ldlt3 F;
  ldlt3_factor(V, F);
  double Vi[9];
  for (int c = 0; c < 3; ++c) {
    const double e[3] = {c == 0 ? 1.0 : 0.0, c == 1 ? 1.0 : 0.0, c == 2 ? 1.0 : 0.0};
    double col[3];
    ldlt3_solve(F, e, col);
    for (int r = 0; r < 3; ++r) Vi[3 * r + c] = col[r];
  }
  for (int c = 0; c < 9; ++c) d.Vinv[9 * i + c] = Vi[c];
  const double* g = d.gp + 3 * i;
  for (int r = 0; r < 3; ++r)
    d.vg[3 * i + r] = (Vi[3 * r] * g[0] + Vi[3 * r + 1] * g[1]) + Vi[3 * r + 2] * g[2];
}

// S and rhs (lm_solver.cpp:73-97): one warp per camera-pair block (ja, jb).
// The block starts at U_ja damped (ja == jb) or 0 and subtracts
// (W_a Vinv_i) W_b^T for every point i the two cameras share, in ascending i —
// the order in which the reference's point loop reaches the block — held in
// registers (lane e: entry e, lanes 0..3 also entries 32..35) and stored once.
// On the diagonal block lanes 4..9 carry rhs_ja -= W_a (Vinv_i g_pt_i).
constexpr int kSchurWarps = 8;
constexpr int kSchurThreads = 32 * kSchurWarps;
__global__ void __launch_bounds__(kSchurThreads) k_lm_schur(LmDev d, double lambda) {
  const int lane = threadIdx.x & 31;
  const int64_t D = 6 * (int64_t)d.m;
  for (int64_t p = (int64_t)blockIdx.x * kSchurWarps + (threadIdx.x >> 5); p < d.npairs;
       p += (int64_t)gridDim.x * kSchurWarps) {
    const int ja = d.pair_ja[p], jb = d.pair_jb[p];
    const bool diag = ja == jb;
    const int r0 = lane / 6, c0 = lane % 6;      // entry lane
    const int r1 = (lane + 32) / 6, c1 = (lane + 32) % 6;  // entry lane + 32 (lanes 0..3)
    double a0 = 0.0, a1 = 0.0, rs = 0.0;
    if (diag) {
      const double* U = d.U + 36 * (int64_t)ja;
      a0 = U[lane] + (r0 == c0 ? lambda * U[lane] : 0.0);
      if (lane < 4) a1 = U[lane + 32] + (r1 == c1 ? lambda * U[lane + 32] : 0.0);
      if (lane >= 4 && lane < 10) rs = d.gc[6 * (int64_t)ja + lane - 4];
    }
#pragma unroll 4
    for (int64_t t = d.pair_off[p]; t < d.pair_off[p + 1]; ++t) {
      const int64_t ka = d.trip_a[t], kb = d.trip_b[t], i = d.trip_i[t];
      const double* Wa = d.W + 18 * ka;
      const double* Wb = d.W + 18 * kb;
      const double* Vi = d.Vinv + 9 * i;
      // row r of WV = Wa Vinv_i (the reference forms the 6x3 product first)
      auto wv = [&](int r, int k) {
        return (Wa[3 * r] * Vi[k] + Wa[3 * r + 1] * Vi[3 + k]) + Wa[3 * r + 2] * Vi[6 + k];
      };
      {
        const double w0 = wv(r0, 0), w1 = wv(r0, 1), w2 = wv(r0, 2);
        a0 -= (w0 * Wb[3 * c0] + w1 * Wb[3 * c0 + 1]) + w2 * Wb[3 * c0 + 2];
      }
      if (lane < 4) {
        const double w0 = wv(r1, 0), w1 = wv(r1, 1), w2 = wv(r1, 2);
        a1 -= (w0 * Wb[3 * c1] + w1 * Wb[3 * c1 + 1]) + w2 * Wb[3 * c1 + 2];
      }
      if (diag && lane >= 4 && lane < 10) {
        const int r = lane - 4;
        const double* g = d.gp + 3 * i;
        const double vg0 = (Vi[0] * g[0] + Vi[1] * g[1]) + Vi[2] * g[2];
        const double vg1 = (Vi[3] * g[0] + Vi[4] * g[1]) + Vi[5] * g[2];
        const double vg2 = (Vi[6] * g[0] + Vi[7] * g[1]) + Vi[8] * g[2];
        rs -= (Wa[3 * r] * vg0 + Wa[3 * r + 1] * vg1) + Wa[3 * r + 2] * vg2;
      }
    }
    d.S[(6 * (int64_t)jb + c0) * D + 6 * ja + r0] = a0;
    if (lane < 4) d.S[(6 * (int64_t)jb + c1) * D + 6 * ja + r1] = a1;
    if (diag && lane >= 4 && lane < 10) d.rhs[6 * (int64_t)ja + lane - 4] = rs;
  }
}

// delta_points (lm_solver.cpp:99-106) from dc.
__global__ void k_lm_dp(LmDev d, const double* dc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  double acc[3] = {d.gp[3 * i], d.gp[3 * i + 1], d.gp[3 * i + 2]};
  for (int64_t q = d.pt_off[i]; q < d.pt_off[i + 1]; ++q) {
    const int64_t k = d.pt_obs[q];
    const double* Wk = d.W + 18 * k;
    const double* x = dc + 6 * (int64_t)d.cam[k];
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int r = 0; r < 6; ++r) s += Wk[3 * r + c] * x[r];
      acc[c] -= s;
    }
  }
  const double* Vi = d.Vinv + 9 * i;
  for (int r = 0; r < 3; ++r)
    d.dp[3 * i + r] = (Vi[3 * r] * acc[0] + Vi[3 * r + 1] * acc[1]) + Vi[3 * r + 2] * acc[2];
}

// Dense H (lm_solver.cpp:107-126), column-major, dim 6m + 3n.
__global__ void k_lm_dense(LmDev d, double lambda, int64_t dim) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cb = 6 * (int64_t)d.m;
  if (t < 36 * (int64_t)d.m) {
    const int64_t j = t / 36;
    const int e = (int)(t % 36), r = e / 6, c = e % 6;
    double u = d.U[36 * j + e];
    if (r == c) u += lambda * d.U[36 * j + e];
    d.S[(6 * j + c) * dim + 6 * j + r] = u;
  }
  if (t < 9 * (int64_t)d.n) {
    const int64_t i = t / 9;
    const int e = (int)(t % 9), r = e / 3, c = e % 3;
    double v = d.V[9 * i + e];
    if (r == c) v += lambda * d.V[9 * i + e];
    d.S[(cb + 3 * i + c) * dim + cb + 3 * i + r] = v;
  }
  if (t < d.l) {
    const int j = d.cam[t], i = d.pt[t];
    const double* W = d.W + 18 * t;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 3; ++c) {
        d.S[(cb + 3 * (int64_t)i + c) * dim + 6 * (int64_t)j + r] = W[3 * r + c];
        d.S[(6 * (int64_t)j + r) * dim + cb + 3 * (int64_t)i + c] = W[3 * r + c];
      }
  }
  if (t < 6 * (int64_t)d.m) d.rhs[t] = d.gc[t];
  if (t < 3 * (int64_t)d.n) d.rhs[cb + t] = d.gp[t];
}

__global__ void k_lm_apply(int64_t n6, int64_t n3, const double* pose, const double* pts,
                           const double* dc, const double* dp, double* tpose, double* tpts,
                           int* nonfinite) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n6) {
    if (!isfinite(dc[t])) *nonfinite = 1;
    tpose[t] = pose[t] + dc[t];
  }
  if (t < n3) {
    if (!isfinite(dp[t])) *nonfinite = 1;
    tpts[t] = pts[t] + dp[t];
  }
}

// Sum over observations of ||z - pi||^power (power 1 or 2); first infeasible
// observation (input order) via atomicMin. One partial per CTA (fixed order).
__global__ void __launch_bounds__(kRedThreads) k_lm_err(LmDev d, const double* pose,
                                                        const double* f, const double* pts,
                                                        int power, double* part,
                                                        unsigned long long* bad) {
  __shared__ double red[kRedThreads / 32];
  double s = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; k < d.l;
       k += (int64_t)gridDim.x * kRedThreads) {
    const int j = d.cam[k], i = d.pt[k];
    double v9[9];
    for (int c = 0; c < 3; ++c) v9[c] = pts[3 * (int64_t)i + c];
    for (int c = 0; c < 6; ++c) v9[3 + c] = pose[6 * (int64_t)j + c];
    exact::ETrig tr;
    double R[9], w[3], z[2];
    if (!exact::eproject(v9, f[j], d.eps, tr, R, w, z)) {
      atomicMin(bad, (unsigned long long)k);
      continue;
    }
    const double e0 = d.uv[2 * k] - z[0], e1 = d.uv[2 * k + 1] - z[1];
    const double q = e0 * e0 + e1 * e1;
    s += power == 1 ? sqrt(q) : q;
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) a += red[w];
    part[blockIdx.x] = a;
  }
}

// parameter_mse partials (problem.cpp:178-202): [2 * CTA] camera, point.
__device__ __forceinline__ double wrap_angle(double a) {
  const double pi = 3.141592653589793;
  const double w = remainder(a, 2.0 * pi);
  return w <= -pi ? w + 2.0 * pi : w;
}
__global__ void __launch_bounds__(kRedThreads) k_lm_mse(int m, int n, const double* pose,
                                                        const double* pts, const double* rpose,
                                                        const double* rpts, double* part) {
  __shared__ double red[2][kRedThreads / 32];
  double c = 0.0, p = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kRedThreads;
  for (int64_t j = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; j < m; j += stride) {
    const double* a = pose + 6 * j;
    const double* b = rpose + 6 * j;
    const double da = wrap_angle(a[0] - b[0]), db = wrap_angle(a[1] - b[1]),
                 dg = wrap_angle(a[2] - b[2]);
    const double t0 = a[3] - b[3], t1 = a[4] - b[4], t2 = a[5] - b[5];
    c += da * da + db * db + dg * dg + (t0 * t0 + t1 * t1 + t2 * t2);
  }
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += stride) {
    const double d0 = pts[3 * i] - rpts[3 * i], d1 = pts[3 * i + 1] - rpts[3 * i + 1],
                 d2 = pts[3 * i + 2] - rpts[3 * i + 2];
    p += d0 * d0 + d1 * d1 + d2 * d2;
  }
  for (int off = 16; off > 0; off >>= 1) {
    c += __shfl_down_sync(0xffffffffu, c, off);
    p += __shfl_down_sync(0xffffffffu, p, off);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = c;
    red[1][threadIdx.x >> 5] = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
struct dbag_lm {
  dbag_lm_options opts{};
  int device = 0;
  cudaStream_t st = nullptr;
  cusolverDnHandle_t sol = nullptr;
  LmDev d{};
  std::vector<void*> pool;
  std::vector<double> h_f;        // focal lengths
  double* pose = nullptr;         // state
  double* f = nullptr;
  double* pts = nullptr;
  double* tpose = nullptr;        // trial
  double* tpts = nullptr;
  double* dc = nullptr;           // 6m (Schur) / dim (dense) solution
  double* part = nullptr;
  unsigned long long* bad = nullptr;
  int* flag = nullptr;            // [0] nonfinite, [1] solver info
  double* ref_pose = nullptr;
  double* ref_pts = nullptr;
  size_t s_cap = 0;               // doubles allocated for S
  double* work = nullptr;
  size_t work_cap = 0;
  int* ipiv = nullptr;
  int64_t* ipiv64 = nullptr;
  cudaEvent_t ev[2]{};

  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    LK(cudaMalloc(&p, sizeof(T) * (n ? n : 1)));
    pool.push_back(p);
    return static_cast<T*>(p);
  }
  ~dbag_lm() {
    cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    for (void* p : pool) cudaFree(p);
    if (sol) cusolverDnDestroy(sol);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
  }
  void sync() { LK(cudaStreamSynchronize(st)); }

  // sum of ||z - pi||^power at (P, X); false (and *bad_k) if infeasible.
  bool error_sum(const double* P, const double* X, int power, double* out, int64_t* bad_k) {
    LK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    k_lm_err<<<kRedBlocks, kRedThreads, 0, st>>>(d, P, f, X, power, part, bad);
    LK(cudaGetLastError());
    std::vector<double> h(kRedBlocks);
    unsigned long long hb = 0;
    LK(cudaMemcpyAsync(h.data(), part, sizeof(double) * kRedBlocks, cudaMemcpyDeviceToHost, st));
    LK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    sync();
    if (hb != ~0ull) {
      if (bad_k) *bad_k = (int64_t)hb;
      return false;
    }
    double s = 0.0;
    for (double v : h) s += v;
    *out = s;
    return true;
  }
  [[noreturn]] void depth_error(const double* P, const double* X, int64_t k) {
    // DepthBelowGuard with the offending indices (problem.cpp:140-157)
    int32_t j = 0, i = 0;
    LK(cudaMemcpy(&j, d.cam + k, 4, cudaMemcpyDeviceToHost));
    LK(cudaMemcpy(&i, d.pt + k, 4, cudaMemcpyDeviceToHost));
    double pose6[6], x3[3];
    LK(cudaMemcpy(pose6, P + 6 * (int64_t)j, sizeof(pose6), cudaMemcpyDeviceToHost));
    LK(cudaMemcpy(x3, X + 3 * (int64_t)i, sizeof(x3), cudaMemcpyDeviceToHost));
    const double ca = std::cos(pose6[0]), sa = std::sin(pose6[0]), cb = std::cos(pose6[1]),
                 sb = std::sin(pose6[1]);
    const double w2 = (-sb * x3[0] + (cb * sa) * x3[1]) + (cb * ca) * x3[2] + pose6[5];
    throw LmErr{DBAG_ERR_DEPTH_BELOW_GUARD,
                "point " + std::to_string(i) + " has depth " + std::to_string(w2) +
                    " below the guard in camera " + std::to_string(j),
                i, j, w2};
  }
  void ensure_s(size_t dim) {
    if (dim * dim > s_cap) {
      d.S = alloc<double>(dim * dim);
      d.rhs = alloc<double>(dim);
      dc = alloc<double>(dim);
      s_cap = dim * dim;
    }
  }
  // Solve S x = rhs (dim x dim, column-major, lower triangle) into dc.
  void dense_solve(int dim) {
    int lw = 0;
    LS(cusolverDnDpotrf_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, dim, d.S, dim, &lw));
    ensure_work((size_t)lw);
    // keep S for the indefinite fallback: factor a copy in dc's neighbour? S is
    // rebuilt on failure instead (cheap relative to the factorization).
    LK(cudaMemcpyAsync(dc, d.rhs, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
    LS(cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, dim, d.S, dim, work, lw, flag + 1));
    int info = 0;
    LK(cudaMemcpyAsync(&info, flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    sync();
    if (info == 0) {
      LS(cusolverDnDpotrs(sol, CUBLAS_FILL_MODE_LOWER, dim, 1, d.S, dim, dc, dim, flag + 1));
      return;
    }
    info_fallback = true;
  }
  void ensure_work(size_t n) {
    if (n > work_cap) {
      work = alloc<double>(n);
      work_cap = n;
    }
  }
  bool info_fallback = false;
  // Bunch-Kaufman for a symmetric indefinite S (rebuilt by the caller).
  void indefinite_solve(int dim) {
    int lw = 0;
    LS(cusolverDnDsytrf_bufferSize(sol, dim, d.S, dim, &lw));
    ensure_work((size_t)lw);
    if (!ipiv || (size_t)dim > ipiv_cap) {
      ipiv = alloc<int>(dim);
      ipiv64 = alloc<int64_t>(dim);
      ipiv_cap = dim;
    }
    LS(cusolverDnDsytrf(sol, CUBLAS_FILL_MODE_LOWER, dim, d.S, dim, ipiv, work, lw, flag + 1));
    std::vector<int> hp(dim);
    LK(cudaMemcpyAsync(hp.data(), ipiv, sizeof(int) * dim, cudaMemcpyDeviceToHost, st));
    sync();
    std::vector<int64_t> hp64(hp.begin(), hp.end());
    LK(cudaMemcpyAsync(ipiv64, hp64.data(), sizeof(int64_t) * dim, cudaMemcpyHostToDevice, st));
    LK(cudaMemcpyAsync(dc, d.rhs, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
    size_t wd = 0, wh = 0;
    LS(cusolverDnXsytrs_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, dim, 1, CUDA_R_64F, d.S, dim,
                                   ipiv64, CUDA_R_64F, dc, dim, &wd, &wh));
    ensure_work(wd / sizeof(double) + 1);
    std::vector<char> hw(wh + 1);
    LS(cusolverDnXsytrs(sol, CUBLAS_FILL_MODE_LOWER, dim, 1, CUDA_R_64F, d.S, dim, ipiv64,
                        CUDA_R_64F, dc, dim, work, wd, hw.data(), wh, flag + 1));
    sync();
  }
  size_t ipiv_cap = 0;

  // assemble at the current state (lm_solver.cpp:27-57)
  void assemble() {
    LK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    k_lm_jac<<<grid_for(d.l, 128), 128, 0, st>>>(d, pose, f, pts, bad);
    LK(cudaGetLastError());
    unsigned long long hb = 0;
    LK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    sync();
    if (hb != ~0ull) depth_error(pose, pts, (int64_t)hb);
    k_lm_cam<<<d.m, kCamThreadsLm, 0, st>>>(d);
    LK(cudaGetLastError());
    k_lm_pt<<<grid_for(d.n, 128), 128, 0, st>>>(d);
    LK(cudaGetLastError());
  }
  // one damped step (lm_solver.cpp:59-127) into dc[0..6m) and d.dp
  void solve_step(double lambda, bool schur) {
    const int m = d.m, n = d.n;
    if (schur) {
      const int dim = 6 * m;
      ensure_s((size_t)dim);
      k_lm_vinv<<<grid_for(n, 128), 128, 0, st>>>(d, lambda);
      LK(cudaGetLastError());
      for (int attempt = 0; attempt < 2; ++attempt) {
        LK(cudaMemsetAsync(d.S, 0, sizeof(double) * (size_t)dim * dim, st));
        const int64_t blocks = std::min<int64_t>((d.npairs + kSchurWarps - 1) / kSchurWarps,
                                                 148 * 64);
        k_lm_schur<<<(unsigned)std::max<int64_t>(blocks, 1), kSchurThreads, 0, st>>>(d, lambda);
        LK(cudaGetLastError());
        info_fallback = false;
        if (attempt == 0) {
          dense_solve(dim);
          if (!info_fallback) break;
        } else {
          indefinite_solve(dim);
        }
      }
      k_lm_dp<<<grid_for(n, 128), 128, 0, st>>>(d, dc);
      LK(cudaGetLastError());
    } else {
      const int64_t dim = 6 * (int64_t)m + 3 * (int64_t)n;
      if (dim > 24000)
        throw LmErr{DBAG_ERR_UNSUPPORTED, "dense (non-Schur) LM step limited to 24000 unknowns"};
      ensure_s((size_t)dim);
      for (int attempt = 0; attempt < 2; ++attempt) {
        LK(cudaMemsetAsync(d.S, 0, sizeof(double) * (size_t)dim * dim, st));
        const int64_t items = std::max<int64_t>({36 * (int64_t)m, 9 * (int64_t)n, d.l, dim});
        k_lm_dense<<<grid_for(items, 256), 256, 0, st>>>(d, lambda, dim);
        LK(cudaGetLastError());
        info_fallback = false;
        if (attempt == 0) {
          dense_solve((int)dim);
          if (!info_fallback) break;
        } else {
          indefinite_solve((int)dim);
        }
      }
      LK(cudaMemcpyAsync(d.dp, dc + 6 * (int64_t)m, sizeof(double) * 3 * (size_t)n,
                         cudaMemcpyDeviceToDevice, st));
    }
  }
  void record(dbag_iteration_record* r, int iter, double wall_ms, bool with_ref) {
    *r = dbag_iteration_record{};
    r->iter = iter;
    double s = 0.0;
    int64_t bk = -1;
    if (!error_sum(pose, pts, 1, &s, &bk)) depth_error(pose, pts, bk);
    r->sum_reproj_err = s;
    r->mean_reproj_err = s / (double)d.l;
    r->camera_mse = r->point_mse = std::numeric_limits<double>::quiet_NaN();
    if (with_ref) {
      k_lm_mse<<<kRedBlocks, kRedThreads, 0, st>>>(d.m, d.n, pose, pts, ref_pose, ref_pts, part);
      LK(cudaGetLastError());
      std::vector<double> h(2 * kRedBlocks);
      LK(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
      sync();
      double c = 0.0, p = 0.0;
      for (int b = 0; b < kRedBlocks; ++b) {
        c += h[2 * b];
        p += h[2 * b + 1];
      }
      r->camera_mse = d.m ? c / (6.0 * d.m) : 0.0;
      r->point_mse = d.n ? p / (3.0 * d.n) : 0.0;
    }
    r->wall_ms = wall_ms;
  }
};

extern "C" {

// ---- Schur pair lists on the device ------------------------------------------
// Every point contributes one triplet (obs a, obs b, point) per ordered pair of
// its observations to the list of block (cam a, cam b). Emitted point-major
// (points ascending, then a, then b: the host loop's order), then a stable
// radix sort by block key keeps that order inside each block's list.
__global__ void k_pair_count(int n, const int64_t* po, int64_t* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int64_t d = po[i + 1] - po[i];
    cnt[i] = d * d;
  }
}

__global__ void k_pair_emit(int n, int m, const int64_t* po, const int32_t* pobs,
                            const int32_t* cam, const int64_t* toff, uint32_t* key,
                            int32_t* ta, int32_t* tb, int32_t* ti, int32_t* idx) {
  // a warp per point: lanes stride over its d*d ordered pairs
  const int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t b0 = po[i], d = po[i + 1] - po[i], t0 = toff[i];
  for (int64_t e = lane; e < d * d; e += 32) {
    const int32_t ka = pobs[b0 + e / d], kb = pobs[b0 + e % d];
    const int64_t t = t0 + e;
    key[t] = (uint32_t)cam[ka] * (uint32_t)m + (uint32_t)cam[kb];
    ta[t] = ka;
    tb[t] = kb;
    ti[t] = i;
    idx[t] = (int32_t)t;
  }
}

__global__ void k_pair_gather(int64_t T, const int32_t* perm, const int32_t* ta,
                              const int32_t* tb, const int32_t* ti, int32_t* oa, int32_t* ob,
                              int32_t* oi) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = perm[t];
    oa[t] = ta[s];
    ob[t] = tb[s];
    oi[t] = ti[s];
  }
}

__global__ void k_pair_blocks(int64_t npairs, int m, const uint32_t* ukey, int32_t* ja,
                              int32_t* jb) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    ja[p] = (int32_t)(ukey[p] / (uint32_t)m);
    jb[p] = (int32_t)(ukey[p] % (uint32_t)m);
  }
}

void dbag_lm_options_default(dbag_lm_options* o) {  // lm_solver.hpp:14-23
  o->max_iters = 100;
  o->error_stop = 1e-14;
  o->lambda_init = 1e-3;
  o->lambda_max = 1e16;
  o->lambda_up = 10.0;
  o->lambda_down = 10.0;
  o->use_schur = 1;
  o->eps_depth = 1e-6;
  o->device = 0;
}

int dbag_lm_create(const dbag_problem_view* p, const dbag_param_view* init,
                   const dbag_lm_options* opts, dbag_lm** out) {
  *out = nullptr;
  auto* h = new dbag_lm();
  try {
    const int m = p->num_cameras, n = p->num_points;
    const int64_t l = p->num_obs;
    if (init->num_cameras != m || init->num_points != n)
      throw LmErr{DBAG_ERR_SIZE_MISMATCH, "init state sizes do not match the problem"};
    if (m > 16000)  // S alone would be (6m)^2 doubles = 74 GB; pair map m^2 on the host
      throw LmErr{DBAG_ERR_UNSUPPORTED, "the dense LM camera system is limited to 16000 cameras"};
    std::string msg;
    const int vrc = validate_problem_arrays(m, n, l, p->obs_cam, p->obs_pt, p->obs_uv, p->cam_pose,
                                            p->cam_f, p->points, &msg);
    if (vrc != DBAG_OK) throw LmErr{vrc, msg};
    h->opts = *opts;
    h->device = opts->device;
    LK(cudaSetDevice(h->device));
    LK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    LS(cusolverDnCreate(&h->sol));
    LS(cusolverDnSetStream(h->sol, h->st));
    for (auto& e : h->ev) LK(cudaEventCreate(&e));
    LmDev& d = h->d;
    d.m = m;
    d.n = n;
    d.l = l;
    d.eps = opts->eps_depth;
    // CSR maps (host, O(l)): camera -> obs ascending k / ascending point id,
    // point -> obs ascending k
    std::vector<int64_t> co(m + 1, 0), po(n + 1, 0);
    for (int64_t k = 0; k < l; ++k) {
      ++co[p->obs_cam[k] + 1];
      ++po[p->obs_pt[k] + 1];
    }
    for (int j = 0; j < m; ++j) co[j + 1] += co[j];
    for (int i = 0; i < n; ++i) po[i + 1] += po[i];
    std::vector<int32_t> cobs(l), pobs(l), cobs_p(l);
    {
      std::vector<int64_t> fc(co.begin(), co.end() - 1), fp(po.begin(), po.end() - 1);
      for (int64_t k = 0; k < l; ++k) {
        cobs[fc[p->obs_cam[k]]++] = (int32_t)k;
        pobs[fp[p->obs_pt[k]]++] = (int32_t)k;
      }
      // by point id: walking points ascending and their observations yields
      // each camera's observations in ascending point order
      std::vector<int64_t> fcp(co.begin(), co.end() - 1);
      for (int i = 0; i < n; ++i)
        for (int64_t q = po[i]; q < po[i + 1]; ++q) {
          const int32_t k = pobs[q];
          cobs_p[fcp[p->obs_cam[k]]++] = k;
        }
    }
    auto up = [&](auto* dst, const void* src, size_t bytes) {
      LK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->st));
    };
    int32_t* dcam = h->alloc<int32_t>(l);
    int32_t* dpt = h->alloc<int32_t>(l);
    double* duv = h->alloc<double>(2 * l);
    int64_t* dco = h->alloc<int64_t>(m + 1);
    int64_t* dpo = h->alloc<int64_t>(n + 1);
    int32_t* dcobs = h->alloc<int32_t>(l);
    int32_t* dcobs_p = h->alloc<int32_t>(l);
    int32_t* dpobs = h->alloc<int32_t>(l);
    up(dcam, p->obs_cam, 4 * l);
    up(dpt, p->obs_pt, 4 * l);
    up(duv, p->obs_uv, 16 * l);
    up(dco, co.data(), 8 * (m + 1));
    up(dpo, po.data(), 8 * (n + 1));
    up(dcobs, cobs.data(), 4 * l);
    up(dcobs_p, cobs_p.data(), 4 * l);
    up(dpobs, pobs.data(), 4 * l);
    d.cam = dcam;
    d.pt = dpt;
    d.uv = duv;
    d.cam_off = dco;
    d.pt_off = dpo;
    d.cam_obs = dcobs;
    d.cam_obs_p = dcobs_p;
    d.pt_obs = dpobs;
    {
      // Schur pair lists on the device (k_pair_*): count d_i^2 triplets per
      // point, emit them point-major, stable radix sort by block key, run
      // lengths -> (ja, jb, offsets). Same lists, same order as the host loop
      // over points / observation pairs it replaces.
      auto tmp = [&](size_t bytes) {
        void* q = nullptr;
        LK(cudaMalloc(&q, bytes ? bytes : 1));
        return q;
      };
      int64_t* cnt = static_cast<int64_t*>(tmp(8 * (size_t)(n + 1)));
      int64_t* toff = static_cast<int64_t*>(tmp(8 * (size_t)(n + 1)));
      k_pair_count<<<(n + 255) / 256, 256, 0, h->st>>>(n, dpo, cnt);
      LK(cudaMemsetAsync(cnt + n, 0, 8, h->st));
      size_t tb_bytes = 0;
      LK(cub::DeviceScan::ExclusiveSum(nullptr, tb_bytes, cnt, toff, n + 1, h->st));
      void* scan_tmp = tmp(tb_bytes);
      LK(cub::DeviceScan::ExclusiveSum(scan_tmp, tb_bytes, cnt, toff, n + 1, h->st));
      int64_t T = 0;
      LK(cudaMemcpyAsync(&T, toff + n, 8, cudaMemcpyDeviceToHost, h->st));
      h->sync();
      if (T >= (int64_t)std::numeric_limits<int32_t>::max())
        throw LmErr{DBAG_ERR_UNSUPPORTED, "more than 2^31 Schur triplets"};
      uint32_t* key = static_cast<uint32_t*>(tmp(4 * (size_t)T));
      uint32_t* key_s = static_cast<uint32_t*>(tmp(4 * (size_t)T));
      int32_t* ta = static_cast<int32_t*>(tmp(4 * (size_t)T));
      int32_t* tb = static_cast<int32_t*>(tmp(4 * (size_t)T));
      int32_t* ti = static_cast<int32_t*>(tmp(4 * (size_t)T));
      int32_t* idx = static_cast<int32_t*>(tmp(4 * (size_t)T));
      int32_t* perm = static_cast<int32_t*>(tmp(4 * (size_t)T));
      k_pair_emit<<<(unsigned)(((int64_t)n * 32 + 255) / 256), 256, 0, h->st>>>(
          n, m, dpo, dpobs, dcam, toff, key, ta, tb, ti, idx);
      LK(cudaGetLastError());
      int bits = 1;
      while (bits < 32 && ((uint64_t)m * (uint64_t)m >> bits) != 0) ++bits;
      size_t sb = 0;
      LK(cub::DeviceRadixSort::SortPairs(nullptr, sb, key, key_s, idx, perm, (int)T, 0, bits,
                                         h->st));
      void* sort_tmp = tmp(sb);
      LK(cub::DeviceRadixSort::SortPairs(sort_tmp, sb, key, key_s, idx, perm, (int)T, 0, bits,
                                         h->st));
      int32_t* dta = h->alloc<int32_t>(T);
      int32_t* dtb = h->alloc<int32_t>(T);
      int32_t* dti = h->alloc<int32_t>(T);
      k_pair_gather<<<592, 256, 0, h->st>>>(T, perm, ta, tb, ti, dta, dtb, dti);
      LK(cudaGetLastError());
      // run-length encode the sorted keys -> blocks and their triplet counts
      uint32_t* ukey = key;  // reuse: the unsorted keys are dead
      const int64_t max_runs = std::min<int64_t>(T, (int64_t)m * m);
      int64_t* rc = static_cast<int64_t*>(tmp(8 * (size_t)(max_runs + 1)));
      int64_t* nruns = static_cast<int64_t*>(tmp(8));
      size_t rb = 0;
      LK(cub::DeviceRunLengthEncode::Encode(nullptr, rb, key_s, ukey, rc, nruns, T, h->st));
      void* rle_tmp = tmp(rb);
      LK(cub::DeviceRunLengthEncode::Encode(rle_tmp, rb, key_s, ukey, rc, nruns, T, h->st));
      int64_t npairs = 0;
      LK(cudaMemcpyAsync(&npairs, nruns, 8, cudaMemcpyDeviceToHost, h->st));
      h->sync();
      int32_t* dja = h->alloc<int32_t>(npairs);
      int32_t* djb = h->alloc<int32_t>(npairs);
      int64_t* dpoff = h->alloc<int64_t>(npairs + 1);
      LK(cudaMemsetAsync(rc + npairs, 0, 8, h->st));
      size_t eb = 0;
      LK(cub::DeviceScan::ExclusiveSum(nullptr, eb, rc, dpoff, npairs + 1, h->st));
      void* ex_tmp = tmp(eb);
      LK(cub::DeviceScan::ExclusiveSum(ex_tmp, eb, rc, dpoff, npairs + 1, h->st));
      k_pair_blocks<<<592, 256, 0, h->st>>>(npairs, m, ukey, dja, djb);
      LK(cudaGetLastError());
      h->sync();
      for (void* q : {(void*)cnt, (void*)toff, scan_tmp, (void*)key, (void*)key_s, (void*)ta,
                      (void*)tb, (void*)ti, (void*)idx, (void*)perm, sort_tmp, (void*)rc,
                      (void*)nruns, rle_tmp, ex_tmp})
        cudaFree(q);
      d.npairs = npairs;
      d.pair_ja = dja;
      d.pair_jb = djb;
      d.pair_off = dpoff;
      d.trip_a = dta;
      d.trip_b = dtb;
      d.trip_i = dti;
    }
    d.J = h->alloc<double>(18 * l);
    d.r = h->alloc<double>(2 * l);
    d.W = h->alloc<double>(18 * l);
    d.U = h->alloc<double>(36 * (size_t)m);
    d.V = h->alloc<double>(9 * (size_t)n);
    d.gc = h->alloc<double>(6 * (size_t)m);
    d.gp = h->alloc<double>(3 * (size_t)n);
    d.Vinv = h->alloc<double>(9 * (size_t)n);
    d.vg = h->alloc<double>(3 * (size_t)n);
    d.dp = h->alloc<double>(3 * (size_t)n);
    h->pose = h->alloc<double>(6 * (size_t)m);
    h->f = h->alloc<double>(m);
    h->pts = h->alloc<double>(3 * (size_t)n);
    h->tpose = h->alloc<double>(6 * (size_t)m);
    h->tpts = h->alloc<double>(3 * (size_t)n);
    h->part = h->alloc<double>(2 * kRedBlocks);
    h->bad = h->alloc<unsigned long long>(1);
    h->flag = h->alloc<int>(2);
    h->ref_pose = h->alloc<double>(6 * (size_t)m);
    h->ref_pts = h->alloc<double>(3 * (size_t)n);
    const double* f0 = init->cam_f ? init->cam_f : p->cam_f;
    h->h_f.assign(f0, f0 + m);
    up(h->pose, init->cam_pose, 48 * (size_t)m);
    up(h->f, f0, 8 * (size_t)m);
    up(h->pts, init->points, 24 * (size_t)n);
    h->sync();
  } catch (const LmErr& e) {
    delete h;
    return set_error(e.code, e.msg, e.pt, e.cam, e.depth);
  }
  *out = h;
  return set_error(DBAG_OK, "");
}

void dbag_lm_destroy(dbag_lm* h) { delete h; }

int dbag_lm_get_state(dbag_lm* h, double* cam_pose, double* points) {
  try {
    LK(cudaSetDevice(h->device));
    LK(cudaMemcpy(cam_pose, h->pose, 48 * (size_t)h->d.m, cudaMemcpyDeviceToHost));
    LK(cudaMemcpy(points, h->pts, 24 * (size_t)h->d.n, cudaMemcpyDeviceToHost));
  } catch (const LmErr& e) {
    return set_error(e.code, e.msg);
  }
  return set_error(DBAG_OK, "");
}

int dbag_lm_compute_step(dbag_lm* h, double lambda, int32_t use_schur, double* d_cam,
                         double* d_pts) {
  try {
    LK(cudaSetDevice(h->device));
    h->assemble();
    h->solve_step(lambda, use_schur != 0);
    LK(cudaMemcpyAsync(d_cam, h->dc, 48 * (size_t)h->d.m, cudaMemcpyDeviceToHost, h->st));
    LK(cudaMemcpyAsync(d_pts, h->d.dp, 24 * (size_t)h->d.n, cudaMemcpyDeviceToHost, h->st));
    h->sync();
  } catch (const LmErr& e) {
    return set_error(e.code, e.msg, e.pt, e.cam, e.depth);
  }
  return set_error(DBAG_OK, "");
}

// solve_lm (lm_solver.cpp:153-218) from the handle's current state.
int dbag_lm_solve(dbag_lm* h, int32_t loss, const dbag_param_view* reference,
                  dbag_iteration_record* trace, int64_t cap, int64_t* n_trace, int32_t* stop,
                  int32_t* accepted_steps) {
  try {
    LK(cudaSetDevice(h->device));
    if (loss != DBAG_LOSS_SQUARED_L2)
      throw LmErr{DBAG_ERR_VALIDATION, "the LM baseline supports only the squared L2 loss"};
    const dbag_lm_options& o = h->opts;
    const int m = h->d.m, n = h->d.n;
    const bool with_ref = reference != nullptr;
    if (with_ref) {
      if (reference->num_cameras != m || reference->num_points != n)
        throw LmErr{DBAG_ERR_SIZE_MISMATCH, "state and reference sizes differ"};
      LK(cudaMemcpyAsync(h->ref_pose, reference->cam_pose, 48 * (size_t)m, cudaMemcpyHostToDevice,
                         h->st));
      LK(cudaMemcpyAsync(h->ref_pts, reference->points, 24 * (size_t)n, cudaMemcpyHostToDevice,
                         h->st));
    }
    int64_t nt = 0;
    auto push = [&](int iter, double ms) {
      dbag_iteration_record r;
      h->record(&r, iter, ms, with_ref);
      if (nt < cap) trace[nt] = r;
      ++nt;
    };
    double total = 0.0;
    int64_t bk = -1;
    if (!h->error_sum(h->pose, h->pts, 2, &total, &bk)) h->depth_error(h->pose, h->pts, bk);
    push(0, 0.0);
    int32_t st = 2, acc = 0;  // kMaxIters
    double lambda = o.lambda_init;
    bool done = false;
    for (int iter = 1; iter <= o.max_iters && !done; ++iter) {
      if (total < o.error_stop) {
        st = 0;  // kErrorStop
        done = true;
        break;
      }
      LK(cudaEventRecord(h->ev[0], h->st));
      h->assemble();
      bool accepted = false;
      while (!accepted) {
        h->solve_step(lambda, o.use_schur != 0);
        LK(cudaMemsetAsync(h->flag, 0, sizeof(int), h->st));
        const int64_t items = std::max<int64_t>(6 * (int64_t)m, 3 * (int64_t)n);
        k_lm_apply<<<grid_for(items, 256), 256, 0, h->st>>>(6 * (int64_t)m, 3 * (int64_t)n,
                                                            h->pose, h->pts, h->dc, h->d.dp,
                                                            h->tpose, h->tpts, h->flag);
        LK(cudaGetLastError());
        int nonfinite = 0;
        LK(cudaMemcpyAsync(&nonfinite, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->st));
        h->sync();
        if (!nonfinite) {
          double tt = 0.0;
          if (h->error_sum(h->tpose, h->tpts, 2, &tt, nullptr) && tt < total) {
            std::swap(h->pose, h->tpose);
            std::swap(h->pts, h->tpts);
            total = tt;
            lambda = std::max(lambda / o.lambda_down, 1e-12);
            ++acc;
            accepted = true;
            break;
          }
        }
        lambda *= o.lambda_up;
        if (lambda > o.lambda_max) {
          st = 1;  // kLambdaMax
          done = true;
          break;
        }
      }
      if (done) break;
      LK(cudaEventRecord(h->ev[1], h->st));
      h->sync();
      float ms = 0.f;
      LK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
      push(iter, ms);
    }
    if (!done) st = total < o.error_stop ? 0 : 2;
    *n_trace = nt;
    *stop = st;
    *accepted_steps = acc;
  } catch (const LmErr& e) {
    return set_error(e.code, e.msg, e.pt, e.cam, e.depth);
  }
  return set_error(DBAG_OK, "");
}

}  // extern "C"
