// dbag_metrics.cu — metric extras:
//  - align_similarity (problem.cpp:204-237): Umeyama's similarity (the
//    published algorithm, as Eigen::umeyama(src, dst, true) evaluates it:
//    means, sigma = dst_demean * src_demean^T / n, SVD, reflection fix on the
//    smallest singular value, c = tr(S D) / var(src)), then the gauge applied
//    to points (x' = sQ x + b) and cameras (R' = R Q^T, t' = s t - R' b);
//  - the point moments run on the device as fixed-order reductions; the 3x3
//    SVD and the m camera updates on the host.
// Tolerance parity only: Eigen's JacobiSVD is not bit-pinnable.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dbag.h"

namespace {

constexpr int kMomThreads = 256;
constexpr int kMomBlocks = 592;  // 148 SMs x 4; fixed, so the partial order is fixed

// stage 0: sums of src and dst (6); stage 1: sum of (dst-md)(src-ms)^T (9) and
// sum ||src-ms||^2 (1). One partial per CTA, tree order fixed by the launch.
__global__ void __launch_bounds__(kMomThreads) k_moments(int64_t n, const double* src,
                                                         const double* dst, const double* mean,
                                                         int stage, double* part) {
  __shared__ double red[kMomThreads / 32][10];
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * kMomThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kMomThreads) {
    const double* a = src + 3 * i;
    const double* b = dst + 3 * i;
    if (stage == 0) {
      for (int k = 0; k < 3; ++k) {
        acc[k] += a[k];
        acc[3 + k] += b[k];
      }
    } else {
      const double da[3] = {a[0] - mean[0], a[1] - mean[1], a[2] - mean[2]};
      const double db[3] = {b[0] - mean[3], b[1] - mean[4], b[2] - mean[5]};
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) acc[3 * r + c] += db[r] * da[c];
      acc[9] += (da[0] * da[0] + da[1] * da[1]) + da[2] * da[2];
    }
  }
  for (int k = 0; k < 10; ++k)
    for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], off);
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 10; ++k) red[threadIdx.x >> 5][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 10) {
    double s = 0.0;
    for (int w = 0; w < kMomThreads / 32; ++w) s += red[w][threadIdx.x];
    part[10 * blockIdx.x + threadIdx.x] = s;
  }
}

__global__ void k_transform_points(int64_t n, const double* x, const double* sQ, const double* b,
                                   double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = x + 3 * i;
  for (int r = 0; r < 3; ++r)
    out[3 * i + r] = ((sQ[3 * r] * p[0] + sQ[3 * r + 1] * p[1]) + sQ[3 * r + 2] * p[2]) + b[r];
}

// ---- host 3x3 linear algebra (row-major) ----------------------------------
double det3(const double* A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}

void matmul3(const double* A, const double* B, double* C) {  // C = A B
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = (A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c]) + A[3 * r + 2] * B[6 + c];
}

// One-sided Jacobi SVD, A = U diag(S) V^T, singular values descending.
void svd3(const double* A, double* U, double* S, double* V) {
  double B[9];
  std::memcpy(B, A, sizeof(B));
  for (int k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int k = 0; k < 3; ++k) {
          a += B[3 * k + p] * B[3 * k + p];
          b += B[3 * k + q] * B[3 * k + q];
          g += B[3 * k + p] * B[3 * k + q];
        }
        if (std::abs(g) <= 1e-300 || std::abs(g) <= 1e-17 * std::sqrt(a * b)) continue;
        rotated = true;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int k = 0; k < 3; ++k) {
          const double bp = B[3 * k + p], bq = B[3 * k + q];
          B[3 * k + p] = c * bp - s * bq;
          B[3 * k + q] = s * bp + c * bq;
          const double vp = V[3 * k + p], vq = V[3 * k + q];
          V[3 * k + p] = c * vp - s * vq;
          V[3 * k + q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  int ord[3] = {0, 1, 2};
  double sv[3];
  for (int c = 0; c < 3; ++c)
    sv[c] = std::sqrt(B[c] * B[c] + B[3 + c] * B[3 + c] + B[6 + c] * B[6 + c]);
  std::sort(ord, ord + 3, [&](int x, int y) { return sv[x] > sv[y]; });
  double Uo[9], Vo[9];
  for (int c = 0; c < 3; ++c) {
    const int o = ord[c];
    S[c] = sv[o];
    for (int k = 0; k < 3; ++k) {
      Vo[3 * k + c] = V[3 * k + o];
      Uo[3 * k + c] = sv[o] > 0.0 ? B[3 * k + o] / sv[o] : 0.0;
    }
  }
  // complete U where singular values vanish (rank < 3)
  for (int c = 0; c < 3; ++c) {
    if (S[c] > 0.0) continue;
    const int a = (c + 1) % 3, b = (c + 2) % 3;
    double u[3] = {Uo[3 + a] * Uo[6 + b] - Uo[6 + a] * Uo[3 + b],
                   Uo[6 + a] * Uo[b] - Uo[a] * Uo[6 + b], Uo[a] * Uo[3 + b] - Uo[3 + a] * Uo[b]};
    double nn = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    if (nn == 0.0) {
      u[0] = (c == 0);
      u[1] = (c == 1);
      u[2] = (c == 2);
      nn = 1.0;
    }
    for (int k = 0; k < 3; ++k) Uo[3 * k + c] = u[k] / nn;
  }
  std::memcpy(U, Uo, sizeof(Uo));
  std::memcpy(V, Vo, sizeof(Vo));
}

// geometry.cpp:62-80 (host, libm sin/cos: the metric is tolerance-checked).
void rotation_from_euler(double a, double b, double g, double* R) {
  const double ca = std::cos(a), sa = std::sin(a), cb = std::cos(b), sb = std::sin(b),
               cg = std::cos(g), sg = std::sin(g);
  const double Rz[9] = {cg, -sg, 0, sg, cg, 0, 0, 0, 1};
  const double Ry[9] = {cb, 0, sb, 0, 1, 0, -sb, 0, cb};
  const double Rx[9] = {1, 0, 0, 0, ca, -sa, 0, sa, ca};
  double T[9];
  matmul3(Rz, Ry, T);
  matmul3(T, Rx, R);
}
void euler_from_rotation(const double* R, double* out) {
  out[1] = std::asin(std::clamp(-R[6], -1.0, 1.0));
  if (std::abs(R[6]) < 1.0 - 1e-12) {
    out[0] = std::atan2(R[7], R[8]);
    out[2] = std::atan2(R[3], R[0]);
  } else {
    out[0] = std::atan2(-R[5], R[4]);
    out[2] = 0.0;
  }
}

struct MetErr {
  int code;
  std::string msg;
};
#define MK(call)                                                                   \
  do {                                                                             \
    const cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                         \
      throw MetErr{DBAG_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_)}; \
  } while (0)

}  // namespace

namespace dbag {
namespace metrics {

// Status code (dbag_status) and message; called by the C-ABI wrapper.
int align_similarity(const dbag_param_view* state, const dbag_param_view* reference,
                     int32_t device, double* out_pose, double* out_points, std::string* err) {
  std::vector<void*> pool;
  try {
    const int64_t n = state->num_points, m = state->num_cameras;
    if (reference->num_points != n || n < 3)
      throw MetErr{DBAG_ERR_SIZE_MISMATCH,
                   "similarity alignment needs matching point sets of size >= 3"};
    MK(cudaSetDevice(device));
    cudaStream_t st = nullptr;
    auto dal = [&](size_t bytes) {
      void* p = nullptr;
      MK(cudaMalloc(&p, bytes));
      pool.push_back(p);
      return static_cast<double*>(p);
    };
    double* d_src = dal(sizeof(double) * 3 * n);
    double* d_dst = dal(sizeof(double) * 3 * n);
    double* d_out = dal(sizeof(double) * 3 * n);
    double* d_part = dal(sizeof(double) * 10 * kMomBlocks);
    double* d_small = dal(sizeof(double) * 32);
    MK(cudaMemcpy(d_src, state->points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    MK(cudaMemcpy(d_dst, reference->points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    std::vector<double> part(10 * kMomBlocks);
    auto reduce = [&](int stage, double* out10) {
      k_moments<<<kMomBlocks, kMomThreads, 0, st>>>(n, d_src, d_dst, d_small, stage, d_part);
      MK(cudaGetLastError());
      MK(cudaMemcpy(part.data(), d_part, sizeof(double) * part.size(), cudaMemcpyDeviceToHost));
      for (int k = 0; k < 10; ++k) {
        double s = 0.0;
        for (int c = 0; c < kMomBlocks; ++c) s += part[10 * c + k];
        out10[k] = s;
      }
    };
    const double inv_n = 1.0 / (double)n;
    double mom[10], mean[6];
    reduce(0, mom);
    for (int k = 0; k < 6; ++k) mean[k] = mom[k] * inv_n;
    MK(cudaMemcpy(d_small, mean, sizeof(mean), cudaMemcpyHostToDevice));
    reduce(1, mom);
    double sigma[9];
    for (int k = 0; k < 9; ++k) sigma[k] = mom[k] * inv_n;
    const double src_var = mom[9] * inv_n;
    double U[9], Sv[3], V[9];
    svd3(sigma, U, Sv, V);
    double D[3] = {1.0, 1.0, 1.0};
    if (det3(U) * det3(V) < 0.0) D[2] = -1.0;  // reflection: flip the smallest
    double UD[9], Vt[9], R[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        UD[3 * r + c] = U[3 * r + c] * D[c];
        Vt[3 * r + c] = V[3 * c + r];
      }
    matmul3(UD, Vt, R);
    const double c = (1.0 / src_var) * ((Sv[0] * D[0] + Sv[1] * D[1]) + Sv[2] * D[2]);
    double sQ[9], b[3];
    for (int k = 0; k < 9; ++k) sQ[k] = c * R[k];
    for (int r = 0; r < 3; ++r)
      b[r] = mean[3 + r] - ((sQ[3 * r] * mean[0] + sQ[3 * r + 1] * mean[1]) + sQ[3 * r + 2] * mean[2]);
    // problem.cpp:215-236
    const double s = std::cbrt(det3(sQ));
    double Q[9];
    for (int k = 0; k < 9; ++k) Q[k] = sQ[k] / s;
    double hb[12];
    std::memcpy(hb, sQ, sizeof(sQ));
    std::memcpy(hb + 9, b, sizeof(b));
    MK(cudaMemcpy(d_small, hb, sizeof(hb), cudaMemcpyHostToDevice));
    k_transform_points<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d_src, d_small, d_small + 9,
                                                                     d_out);
    MK(cudaGetLastError());
    MK(cudaMemcpy(out_points, d_out, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < m; ++j) {
      const double* p = state->cam_pose + 6 * j;
      double Rc[9], Qt[9], Rn[9], ang[3];
      rotation_from_euler(p[0], p[1], p[2], Rc);
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) Qt[3 * r + cc] = Q[3 * cc + r];
      matmul3(Rc, Qt, Rn);
      euler_from_rotation(Rn, ang);
      double* o = out_pose + 6 * j;
      o[0] = ang[0];
      o[1] = ang[1];
      o[2] = ang[2];
      for (int r = 0; r < 3; ++r)
        o[3 + r] = s * p[3 + r] - ((Rn[3 * r] * b[0] + Rn[3 * r + 1] * b[1]) + Rn[3 * r + 2] * b[2]);
    }
    for (void* q : pool) cudaFree(q);
    return DBAG_OK;
  } catch (const MetErr& e) {
    for (void* q : pool) cudaFree(q);
    *err = e.msg;
    return e.code;
  }
}

}  // namespace metrics
}  // namespace dbag
