// dbag_consensus.cuh — K3 (camera consensus + dual s + primal_y), K2 (point
// consensus + dual r + primal_x + the round's reprojection metric), the final
// deterministic reduction, and the query kernels.
//
// Restates consensus_update / dual_update / max_primal_residual_* /
// try_mean_reprojection_error (admm_solver.cpp:318-383, problem.cpp:109-138).
// Deterministic: fixed-shape trees, no floating-point atomics. Points sum
// their copies sequentially in the reference's copy order (ascending block),
// so the point consensus is bit-identical to the reference's for identical
// copies; cameras use a fixed 256-lane tree (long segments).
#pragma once

#include "dbag_common.cuh"

namespace dbag {

constexpr int kModeConsensus = 1, kModeDual = 2;
constexpr int kCamThreads = 256;
constexpr int kPtThreads = 256;

__device__ __forceinline__ void write_camR(const DevState& S, int j, const double* pose, double f) {
  Trig t;
  trig_of(pose[0], pose[1], pose[2], t);
  double R[9];
  rot_of(t, R);
  double* o = S.camR + 16 * (int64_t)j;
#pragma unroll
  for (int k = 0; k < 9; ++k) o[k] = R[k];
  o[9] = pose[3];
  o[10] = pose[4];
  o[11] = pose[5];
  o[12] = f;
}

// K3: one CTA per camera segment [cam_off[j], cam_off[j+1]) of block order.
template <int MODE>
__global__ void __launch_bounds__(kCamThreads) k_camera(DevState S) {
  if (__syncthreads_or(threadIdx.x == 0 && S.gate && *S.gate >= 0)) return;  // local solve raised
  __shared__ double smem[(kCamThreads / 32) * 6];
  __shared__ double ybar_s[6];
  const int j = blockIdx.x;
  const int64_t beg = S.cam_off[j], end = S.cam_off[j + 1];
  const double* Y = S.cam_soa;
  double* Sd = S.cam_soa + 6 * S.L;
  double dual_res = 0.0;
  if (MODE & kModeConsensus) {
    // anchor = first copy (lowest point), admm_solver.cpp:335
    double anchor[6], acc[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      anchor[k] = Y[k * S.L + beg];
      acc[k] = 0.0;
    }
    const double inv_rho = 1.0 / S.rho_y;  // :323
    for (int64_t b = beg + threadIdx.x; b < end; b += kCamThreads)
#pragma unroll
      for (int k = 0; k < 6; ++k) acc[k] += (Y[k * S.L + b] - anchor[k]) + inv_rho * Sd[k * S.L + b];
    block_sum<kCamThreads, 6>(acc, smem);
    if (threadIdx.x == 0) {
      const double cnt = (double)(end - beg);
      double* yb = S.ybar + 8 * (int64_t)j;
      double pose[6], d2 = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        pose[k] = anchor[k] + acc[k] / cnt;  // :340
        const double d = pose[k] - yb[k];
        d2 += d * d;
        yb[k] = pose[k];
        ybar_s[k] = pose[k];
      }
      dual_res = S.rho_y * sqrt(d2);
      write_camR(S, j, pose, yb[6]);
    }
    __syncthreads();
  } else {
    if (threadIdx.x < 6) ybar_s[threadIdx.x] = S.ybar[8 * (int64_t)j + threadIdx.x];
    __syncthreads();
  }
  if (MODE & kModeDual) {
    double yb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) yb[k] = ybar_s[k];
    double worst = 0.0;
    for (int64_t b = beg + threadIdx.x; b < end; b += kCamThreads) {
      double d2 = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double d = Y[k * S.L + b] - yb[k];
        Sd[k * S.L + b] += S.rho_y * d;  // admm_solver.cpp:351-355
        d2 += d * d;
      }
      worst = fmax(worst, sqrt(d2));  // :372-383
    }
    worst = block_max<kCamThreads>(worst, smem);
    if (threadIdx.x == 0) S.cam_stats[2 * j] = worst;
  }
  if (threadIdx.x == 0) S.cam_stats[2 * j + 1] = dual_res;
}

// K2: one thread per point, points visited in descending track length so a
// warp's segments are of similar length. Segment = pt_off[i]..pt_off[i+1] of
// the point-major record array.
template <int MODE, bool kMetric>
__global__ void __launch_bounds__(kPtThreads) k_point(DevState S) {
  if (__syncthreads_or(threadIdx.x == 0 && S.gate && *S.gate >= 0)) return;  // local solve raised
  __shared__ double smem[(kPtThreads / 32) * 2];
  const int64_t t = (int64_t)blockIdx.x * kPtThreads + threadIdx.x;
  double err_sum = 0.0, worst = 0.0, dual_res = 0.0, infeasible = 0.0;
  if (t < S.N) {
    const int i = S.pt_order[t];
    const int64_t beg = S.pt_off[i], end = S.pt_off[i + 1];
    double xb[3];
    if (MODE & kModeConsensus) {
      // admm_solver.cpp:324-332: anchor = first copy, sequential accumulation in
      // copy order. A boundary point of a sharded solve reads all its copies
      // (every rank's) from the all-gathered buffer, in the same global order.
      const double inv_rho = 1.0 / S.rho_x;
      double anc[3], acc[3] = {0.0, 0.0, 0.0}, cnt;
      const int bp = S.bp_of_local ? S.bp_of_local[i] : -1;
      if (bp >= 0) {
        const int64_t g0 = S.gb_off[bp], g1 = S.gb_off[bp + 1];
        double c[6];
        boundary_copy(S, S.gmap[g0], c);
        anc[0] = c[0];
        anc[1] = c[1];
        anc[2] = c[2];
        for (int64_t g = g0; g < g1; ++g) {
          boundary_copy(S, S.gmap[g], c);
          acc[0] += (c[0] - anc[0]) + inv_rho * c[3];
          acc[1] += (c[1] - anc[1]) + inv_rho * c[4];
          acc[2] += (c[2] - anc[2]) + inv_rho * c[5];
        }
        cnt = (double)(g1 - g0);
      } else {
        const PointRec& a = S.prec[beg];
        anc[0] = a.x0;
        anc[1] = a.x1;
        anc[2] = a.x2;
        for (int64_t p = beg; p < end; ++p) {
          const PointRec& r = S.prec[p];
          acc[0] += (r.x0 - anc[0]) + inv_rho * r.r0;
          acc[1] += (r.x1 - anc[1]) + inv_rho * r.r1;
          acc[2] += (r.x2 - anc[2]) + inv_rho * r.r2;
        }
        cnt = (double)(end - beg);
      }
      const double4 old = S.xbar[i];
#pragma unroll
      for (int k = 0; k < 3; ++k) xb[k] = anc[k] + acc[k] / cnt;
      const double d0 = xb[0] - old.x, d1 = xb[1] - old.y, d2 = xb[2] - old.z;
      dual_res = S.rho_x * sqrt(d0 * d0 + d1 * d1 + d2 * d2);
      S.xbar[i] = make_double4(xb[0], xb[1], xb[2], 0.0);
    } else {
      const double4 o = S.xbar[i];
      xb[0] = o.x;
      xb[1] = o.y;
      xb[2] = o.z;
    }
    if ((MODE & kModeDual) || kMetric) {
      for (int64_t p = beg; p < end; ++p) {
        PointRec& r = S.prec[p];
        const double d0 = r.x0 - xb[0], d1 = r.x1 - xb[1], d2 = r.x2 - xb[2];
        if (MODE & kModeDual) {
          r.r0 += S.rho_x * d0;  // admm_solver.cpp:345-350
          r.r1 += S.rho_x * d1;
          r.r2 += S.rho_x * d2;
          worst = fmax(worst, sqrt(d0 * d0 + d1 * d1 + d2 * d2));
        }
        if (kMetric) {
          // problem.cpp:109-121 at (xbar, ybar): camR from K3
          const double* c = S.camR + 16 * (int64_t)S.pm_cam[p];
          double w[3];
          cam_point(c, xb, c + 9, w);
          if (!feasible(w[2], S.eps_depth)) {
            infeasible = 1.0;
          } else {
            const double e0 = r.u - c[12] * w[0] / w[2];
            const double e1 = r.v - c[12] * w[1] / w[2];
            err_sum += sqrt(e0 * e0 + e1 * e1);
          }
        }
      }
    }
  }
  double sums[1] = {err_sum};
  block_sum<kPtThreads, 1>(sums, smem);
  const double mx = block_max<kPtThreads>(worst, smem);
  const double md = block_max<kPtThreads>(dual_res, smem);
  const double inf = block_max<kPtThreads>(infeasible, smem);
  if (threadIdx.x == 0) {
    double* o = S.part_pt + 4 * (int64_t)blockIdx.x;
    o[0] = sums[0];
    o[1] = mx;
    o[2] = md;
    o[3] = inf;
  }
}

// parameter_mse partials (problem.cpp:178-202) against the reference state.
__device__ __forceinline__ double wrap_angle(double a) {
  const double pi = 3.141592653589793;
  const double w = remainder(a, 2.0 * pi);
  return w <= -pi ? w + 2.0 * pi : w;
}

__global__ void __launch_bounds__(256) k_mse(DevState S) {
  __shared__ double smem[8 * 2];
  double c = 0.0, p = 0.0;
  const int64_t stride = (int64_t)gridDim.x * 256;
  for (int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x; j < S.M; j += stride) {
    const double* a = S.ybar + 8 * j;
    const double* b = S.ref_pose + 6 * j;
    const double da = wrap_angle(a[0] - b[0]), db = wrap_angle(a[1] - b[1]),
                 dg = wrap_angle(a[2] - b[2]);
    const double t0 = a[3] - b[3], t1 = a[4] - b[4], t2 = a[5] - b[5];
    c += da * da + db * db + dg * dg + (t0 * t0 + t1 * t1 + t2 * t2);
  }
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < S.N; i += stride) {
    if (S.owner_of_local && !S.owner_of_local[i]) continue;  // counted by its first copy's rank
    const double4 a = S.xbar[i];
    const double* b = S.ref_pts + 3 * i;
    const double d0 = a.x - b[0], d1 = a.y - b[1], d2 = a.z - b[2];
    p += d0 * d0 + d1 * d1 + d2 * d2;
  }
  double v[2] = {c, p};
  block_sum<256, 2>(v, smem);
  if (threadIdx.x == 0) {
    S.part_mse[2 * blockIdx.x] = v[0];
    S.part_mse[2 * blockIdx.x + 1] = v[1];
  }
}

// Final reduction (one CTA, fixed order): K2 partials, K3 per-camera stats,
// MSE partials -> this rank's partial record (raw sums) in S.metric_part.
__global__ void __launch_bounds__(1024) k_final(DevState S, int n_pt_parts, int n_mse_parts) {
  __shared__ double smem[32 * 4];
  double s = 0.0, px = 0.0, dx = 0.0, inf = 0.0, py = 0.0, dy = 0.0, cm = 0.0, pm = 0.0;
  for (int k = threadIdx.x; k < n_pt_parts; k += 1024) {
    const double* o = S.part_pt + 4 * (int64_t)k;
    s += o[0];
    px = fmax(px, o[1]);
    dx = fmax(dx, o[2]);
    inf = fmax(inf, o[3]);
  }
  for (int j = threadIdx.x; j < S.M; j += 1024) {
    py = fmax(py, S.cam_stats[2 * j]);
    dy = fmax(dy, S.cam_stats[2 * j + 1]);
  }
  for (int k = threadIdx.x; k < n_mse_parts; k += 1024) {
    cm += S.part_mse[2 * k];
    pm += S.part_mse[2 * k + 1];
  }
  double sums[3] = {s, cm, pm};
  block_sum<1024, 3>(sums, smem);
  const double a = block_max<1024>(px, smem);
  const double b = block_max<1024>(dx, smem);
  const double c = block_max<1024>(inf, smem);
  const double d = block_max<1024>(py, smem);
  const double e = block_max<1024>(dy, smem);
  if (threadIdx.x == 0) {
    double* o = S.metric_part;
    o[kRecSumErr] = sums[0];
    o[kRecMaxPx] = a;
    o[kRecMaxDx] = b;
    o[kRecInfeasible] = c;
    o[kRecMaxPy] = d;
    o[kRecMaxDy] = e;
    o[kRecCamMse] = sums[1];
    o[kRecPtMse] = sums[2];
  }
}

// Combine the ranks' partial records (rank order) into the round's record.
__global__ void k_combine(DevState S, const double* parts, int world, int32_t m_total,
                          int32_t n_total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double r[kRecFields];
  for (int f = 0; f < kRecFields; ++f) r[f] = parts[f];
  for (int w = 1; w < world; ++w) {
    const double* p = parts + (int64_t)w * kRecFields;
    r[kRecSumErr] += p[kRecSumErr];
    r[kRecCamMse] += p[kRecCamMse];
    r[kRecPtMse] += p[kRecPtMse];
    r[kRecMaxPx] = fmax(r[kRecMaxPx], p[kRecMaxPx]);
    r[kRecMaxPy] = fmax(r[kRecMaxPy], p[kRecMaxPy]);
    r[kRecMaxDx] = fmax(r[kRecMaxDx], p[kRecMaxDx]);
    r[kRecMaxDy] = fmax(r[kRecMaxDy], p[kRecMaxDy]);
    r[kRecInfeasible] = fmax(r[kRecInfeasible], p[kRecInfeasible]);
  }
  r[kRecCamMse] = m_total ? r[kRecCamMse] / (6.0 * m_total) : 0.0;
  r[kRecPtMse] = n_total ? r[kRecPtMse] / (3.0 * n_total) : 0.0;
  for (int f = 0; f < kRecFields; ++f) S.record[f] = r[f];
}

// Pack this rank's boundary copies (x, r) for the all-gather.
__global__ void k_pack_send(DevState S) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S.send_count) return;
  const PointRec& r = S.prec[S.send_pos[s]];
  double* o = S.send_buf + 6 * s;
  o[0] = r.x0;
  o[1] = r.x1;
  o[2] = r.x2;
  o[3] = r.r0;
  o[4] = r.r1;
  o[5] = r.r2;
}

// Shard setup: local observation -> point-major position for the send slots
// and for this rank's own entries of gmap (-2 - q -> -2 - position).
// obs2blk is the inverse of blk_obs.
__global__ void k_obs2blk(DevState S, int32_t* obs2blk) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < S.L) obs2blk[S.blk_obs[b]] = (int32_t)b;
}
__global__ void k_send_pos(DevState S, const int64_t* send_obs_local, const int32_t* obs2blk) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < S.send_count) S.send_pos[s] = S.blk_pos[obs2blk[send_obs_local[s]]];
}
__global__ void k_gmap_own(DevState S, int64_t n, const int32_t* obs2blk) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int64_t v = S.gmap[g];
  if (v <= -2) S.gmap[g] = -2 - (int64_t)S.blk_pos[obs2blk[-2 - v]];
}

// ---- queries ---------------------------------------------------------------
// camR for every camera from ybar (after set_consensus / at create).
__global__ void k_camR_all(DevState S) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < S.M) write_camR(S, j, S.ybar + 8 * (int64_t)j, S.ybar[8 * (int64_t)j + 6]);
}

// Reprojection at the consensus over blocks; first infeasible observation in
// INPUT order via integer atomicMin (mean_reprojection_error's DepthBelowGuard
// reports the first offending observation, problem.cpp:140-157). power 1: sum
// of norms, 2: sum of squares. Partial sums per CTA into part_pt[.][0].
template <int kPower>
__global__ void __launch_bounds__(256) k_reproj_blocks(DevState S) {
  __shared__ double smem[8];
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * 256;
  for (int64_t b = (int64_t)blockIdx.x * 256 + threadIdx.x; b < S.L; b += stride) {
    const double* c = S.camR + 16 * (int64_t)S.blk_cam[b];
    const double4 x = S.xbar[S.blk_pt[b]];
    const double xv[3] = {x.x, x.y, x.z};
    double w[3];
    cam_point(c, xv, c + 9, w);
    if (!feasible(w[2], S.eps_depth)) {
      atomicMin(reinterpret_cast<unsigned long long*>(S.err_obs), (unsigned long long)S.blk_obs[b]);
      continue;
    }
    const PointRec& r = S.prec[S.blk_pos[b]];
    const double e0 = r.u - c[12] * w[0] / w[2];
    const double e1 = r.v - c[12] * w[1] / w[2];
    const double q = e0 * e0 + e1 * e1;
    s += kPower == 1 ? sqrt(q) : q;
  }
  double v[1] = {s};
  block_sum<256, 1>(v, smem);
  if (threadIdx.x == 0) S.part_pt[4 * (int64_t)blockIdx.x] = v[0];
}

__global__ void k_sum_parts(DevState S, int n, double* out) {
  __shared__ double smem[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += 1024) s += S.part_pt[4 * (int64_t)k];
  double v[1] = {s};
  block_sum<1024, 1>(v, smem);
  if (threadIdx.x == 0) *out = v[0];
}

// Block objective (admm_solver.cpp:401-426) for one block, explicit form.
__global__ void k_block_objective(DevState S, int64_t b, double* out) {
  const int j = S.blk_cam[b];
  const PointRec r = S.prec[S.blk_pos[b]];
  double v[9];
  v[0] = r.x0;
  v[1] = r.x1;
  v[2] = r.x2;
  for (int k = 0; k < 6; ++k) v[3 + k] = S.cam_soa[(int64_t)k * S.L + b];
  const double* yb = S.ybar + 8 * (int64_t)j;
  const double4 xb = S.xbar[S.blk_pt[b]];
  Trig t;
  trig_of(v[3], v[4], v[5], t);
  double R[9], w[3];
  rot_of(t, R);
  cam_point(R, v, v + 6, w);
  if (!feasible(w[2], S.eps_depth)) {
    *out = __longlong_as_double(0x7ff0000000000000LL);
    return;
  }
  const double e0 = r.u - yb[6] * w[0] / w[2], e1 = r.v - yb[6] * w[1] / w[2];
  double total;
  if (S.loss == 0) {
    total = e0 * e0 + e1 * e1;
  } else {
    const double a = sqrt(e0 * e0 + e1 * e1);
    total = a <= S.huber_delta ? 0.5 * a * a : S.huber_delta * (a - 0.5 * S.huber_delta);
  }
  const double xv[3] = {xb.x, xb.y, xb.z};
  const double rv[3] = {r.r0, r.r1, r.r2};
  double dd = 0.0, q = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double d = v[k] - xv[k];
    dd += rv[k] * d;
    q += d * d;
  }
  total += dd + 0.5 * S.rho_x * q;
  dd = 0.0;
  q = 0.0;
  for (int k = 0; k < 6; ++k) {
    const double d = v[3 + k] - yb[k];
    dd += S.cam_soa[(int64_t)(6 + k) * S.L + b] * d;
    q += d * d;
  }
  total += dd + 0.5 * S.rho_y * q;
  *out = total;
}

// Dual sums (admm_solver.cpp:385-399): per point in copy order, per camera in
// block order (sequential per variable).
__global__ void k_dual_sums(DevState S, double* pts, double* cams) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < S.N) {
    double a[3] = {0, 0, 0};
    for (int64_t p = S.pt_off[t]; p < S.pt_off[t + 1]; ++p) {
      a[0] += S.prec[p].r0;
      a[1] += S.prec[p].r1;
      a[2] += S.prec[p].r2;
    }
    for (int k = 0; k < 3; ++k) pts[3 * t + k] = a[k];
  } else if (t < (int64_t)S.N + S.M) {
    const int j = (int)(t - S.N);
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t b = S.cam_off[j]; b < S.cam_off[j + 1]; ++b)
      for (int k = 0; k < 6; ++k) a[k] += S.cam_soa[(int64_t)(6 + k) * S.L + b];
    for (int k = 0; k < 6; ++k) cams[6 * (int64_t)j + k] = a[k];
  }
}

// max_primal_residual_points/cameras (admm_solver.cpp:359-383): max over this
// solver's copies of ||copy - consensus||_2, in LOCAL indexing (a shard's
// blk_pt/blk_cam index its own xbar/ybar). The squared norm is summed in the
// reference's component order with explicit _rn operations (this TU is built
// with FMA contraction on). std::max(worst, v) ignores a NaN v; inf counts.
// Non-negative doubles order like their bit patterns, so a 64-bit atomicMax
// per CTA gives the same value in any order. out[0..1] start at +0.
__global__ void k_max_primal(DevState S, unsigned long long* out) {
  unsigned long long wx = 0, wy = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < S.L;
       b += (int64_t)gridDim.x * blockDim.x) {
    const PointRec& rec = S.prec[S.blk_pos[b]];
    const double4 xb = S.xbar[S.blk_pt[b]];
    const double d0 = __dsub_rn(rec.x0, xb.x), d1 = __dsub_rn(rec.x1, xb.y),
                 d2 = __dsub_rn(rec.x2, xb.z);
    double a = 0.0;
    a = __dadd_rn(a, __dmul_rn(d0, d0));
    a = __dadd_rn(a, __dmul_rn(d1, d1));
    a = __dadd_rn(a, __dmul_rn(d2, d2));
    const double* yb = S.ybar + 8 * (int64_t)S.blk_cam[b];
    double c = 0.0;
    for (int k = 0; k < 6; ++k) {
      const double d = __dsub_rn(S.cam_soa[(int64_t)k * S.L + b], yb[k]);
      c = __dadd_rn(c, __dmul_rn(d, d));
    }
    const double va = __dsqrt_rn(a), vc = __dsqrt_rn(c);
    if (va == va) wx = max(wx, (unsigned long long)__double_as_longlong(va));
    if (vc == vc) wy = max(wy, (unsigned long long)__double_as_longlong(vc));
  }
  for (int o = 16; o; o >>= 1) {
    wx = max(wx, __shfl_xor_sync(0xffffffffu, wx, o));
    wy = max(wy, __shfl_xor_sync(0xffffffffu, wy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, wx);
    atomicMax(out + 1, wy);
  }
}

// Block-order AoS <-> device layout (get/set_copies). dir 0: device -> out.
__global__ void k_copies(DevState S, double* lp, double* lc, double* r, double* s, int dir) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= S.L) return;
  double* rec = reinterpret_cast<double*>(S.prec + S.blk_pos[b]);
  if (dir == 0) {
    for (int k = 0; k < 3; ++k) {
      lp[3 * b + k] = rec[kRecX + k];
      r[3 * b + k] = rec[kRecR + k];
    }
    for (int k = 0; k < 6; ++k) {
      lc[6 * b + k] = S.cam_soa[(int64_t)k * S.L + b];
      s[6 * b + k] = S.cam_soa[(int64_t)(6 + k) * S.L + b];
    }
  } else {
    for (int k = 0; k < 3; ++k) {
      rec[kRecX + k] = lp[3 * b + k];
      rec[kRecR + k] = r[3 * b + k];
    }
    for (int k = 0; k < 6; ++k) {
      S.cam_soa[(int64_t)k * S.L + b] = lc[6 * b + k];
      S.cam_soa[(int64_t)(6 + k) * S.L + b] = s[6 * b + k];
    }
  }
}

}  // namespace dbag
