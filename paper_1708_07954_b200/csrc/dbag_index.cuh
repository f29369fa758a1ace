// dbag_index.cuh — K0: the once-per-solve integer index build, on the device.
//
// Restates build_visibility (problem.cpp:12-64: range/duplicate/coverage
// checks, sorted S(j) and its transpose), partition for (1,1) blocks
// (admm_solver.cpp:14-72: observations sorted by (cam_id, point_id)), the copy
// maps (:126-140: per point its blocks in ascending block order, per camera
// its contiguous block range) and communication_cost (:74-101). All integer,
// bit-exact: stable LSD radix sorts (CUB) on (cam<<32|pt) keys, integer
// atomicMin for "first offending index" reports.
#pragma once

#include "dbag_common.cuh"

namespace dbag {

struct IndexErrors {
  unsigned long long nonfinite_z;  // any observation with non-finite z
  unsigned long long bad_range;    // first input index out of range
  unsigned long long dup_pos;      // first sorted position equal to its predecessor
  unsigned long long empty_cam;    // first camera with no observation
  unsigned long long empty_pt;     // first point with no observation
  unsigned long long bad_point;    // first point with non-finite coordinates
};

__global__ void k_check_obs(int64_t L, int M, int N, const int32_t* cam, const int32_t* pt,
                            const double* uv, IndexErrors* e) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  if (!isfinite(uv[2 * k]) || !isfinite(uv[2 * k + 1])) atomicMin(&e->nonfinite_z, (unsigned long long)k);
  const int c = cam[k], p = pt[k];
  if (c < 0 || c >= M || p < 0 || p >= N) atomicMin(&e->bad_range, (unsigned long long)k);
}

__global__ void k_check_points(int N, const double* pts, IndexErrors* e) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (!isfinite(pts[3 * i]) || !isfinite(pts[3 * i + 1]) || !isfinite(pts[3 * i + 2]))
    atomicMin(&e->bad_point, (unsigned long long)i);
}

__global__ void k_make_keys(int64_t L, const int32_t* cam, const int32_t* pt, uint64_t* keys,
                            int32_t* vals) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  keys[k] = ((uint64_t)(uint32_t)cam[k] << 32) | (uint32_t)pt[k];
  vals[k] = (int32_t)k;
}

// After the (cam,pt) sort: block arrays, duplicate check, camera offsets.
__global__ void k_blocks_from_sorted(int64_t L, int M, const uint64_t* keys, DevState S,
                                     IndexErrors* e, uint32_t* pt_keys, int32_t* iota) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= L) return;
  const uint64_t key = keys[b];
  const int c = (int)(key >> 32);
  S.blk_cam[b] = c;
  S.blk_pt[b] = (int32_t)(key & 0xffffffffu);
  pt_keys[b] = (uint32_t)(key & 0xffffffffu);
  iota[b] = (int32_t)b;
  const int prev = b == 0 ? -1 : (int)(keys[b - 1] >> 32);
  if (b > 0 && keys[b - 1] == key) atomicMin(&e->dup_pos, (unsigned long long)b);
  for (int q = prev + 1; q <= c; ++q) S.cam_off[q] = (int32_t)b;
  if (b == L - 1)
    for (int q = c + 1; q <= M; ++q) S.cam_off[q] = (int32_t)L;
}

// After the stable point sort: point-major position of each block, pt_off,
// camera of each point-major position.
__global__ void k_points_from_sorted(int64_t L, int N, const uint32_t* pt_sorted,
                                     const int32_t* pm_blk, DevState S) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= L) return;
  const int b = pm_blk[p];
  S.blk_pos[b] = (int32_t)p;
  S.pm_cam[p] = S.blk_cam[b];
  const int i = (int)pt_sorted[p];
  const int prev = p == 0 ? -1 : (int)pt_sorted[p - 1];
  for (int q = prev + 1; q <= i; ++q) S.pt_off[q] = (int32_t)p;
  if (p == L - 1)
    for (int q = i + 1; q <= N; ++q) S.pt_off[q] = (int32_t)L;
}

// Coverage checks (problem.cpp:53-62) + track lengths + comm cost (Σ 3d(d-1)).
__global__ void k_coverage(DevState S, IndexErrors* e, uint32_t* len, int32_t* iota,
                           unsigned long long* comm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (t < S.M) {
    if (S.cam_off[t] == S.cam_off[t + 1]) atomicMin(&e->empty_cam, (unsigned long long)t);
  }
  if (t < S.N) {
    const int d = S.pt_off[t + 1] - S.pt_off[t];
    if (d == 0) atomicMin(&e->empty_pt, (unsigned long long)t);
    len[t] = (uint32_t)d;
    iota[t] = (int32_t)t;
    c = 3ull * (unsigned long long)d * (unsigned long long)(d > 0 ? d - 1 : 0);
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(comm, c);
}

// copies = init, duals = 0 (admm_solver.cpp:121-140); consensus = init.
__global__ void k_init_state(DevState S, const double* uv, const double* init_pose,
                             const double* init_pts) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= S.L) return;
  const int j = S.blk_cam[b], i = S.blk_pt[b];
  const int64_t k = S.blk_obs[b];
  PointRec r;
  r.x0 = init_pts[3 * (int64_t)i];
  r.x1 = init_pts[3 * (int64_t)i + 1];
  r.x2 = init_pts[3 * (int64_t)i + 2];
  r.r0 = r.r1 = r.r2 = 0.0;
  r.u = uv[2 * k];
  r.v = uv[2 * k + 1];
  S.prec[S.blk_pos[b]] = r;
  for (int q = 0; q < 6; ++q) {
    S.cam_soa[(int64_t)q * S.L + b] = init_pose[6 * (int64_t)j + q];
    S.cam_soa[(int64_t)(6 + q) * S.L + b] = 0.0;
  }
}

__global__ void k_init_consensus(DevState S, const double* init_pose, const double* init_f,
                                 const double* init_pts) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < S.N)
    S.xbar[t] = make_double4(init_pts[3 * t], init_pts[3 * t + 1], init_pts[3 * t + 2], 0.0);
  if (t < S.M) {
    double* y = S.ybar + 8 * t;
    for (int q = 0; q < 6; ++q) y[q] = init_pose[6 * t + q];
    y[6] = init_f[t];
    y[7] = 0.0;
  }
}

// dbag_reset: copies = initial consensus, duals = 0 (z untouched).
__global__ void k_reset_state(DevState S, const double* init_pose, const double* init_pts) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= S.L) return;
  const int j = S.blk_cam[b], i = S.blk_pt[b];
  double* r = reinterpret_cast<double*>(S.prec + S.blk_pos[b]);
  for (int q = 0; q < 3; ++q) {
    r[kRecX + q] = init_pts[3 * (int64_t)i + q];
    r[kRecR + q] = 0.0;
  }
  for (int q = 0; q < 6; ++q) {
    S.cam_soa[(int64_t)q * S.L + b] = init_pose[6 * (int64_t)j + q];
    S.cam_soa[(int64_t)(6 + q) * S.L + b] = 0.0;
  }
}

__global__ void k_reset_consensus(DevState S, const double* init_pose, const double* init_pts) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < S.N)
    S.xbar[t] = make_double4(init_pts[3 * t], init_pts[3 * t + 1], init_pts[3 * t + 2], 0.0);
  if (t < S.M)
    for (int q = 0; q < 6; ++q) S.ybar[8 * t + q] = init_pose[6 * t + q];
}

}  // namespace dbag
