// dbag_lbfgs.cuh — K1 for the Huber loss: the reference's L-BFGS local solve
// (admm_solver.cpp:231-282 -> local_opt.cpp:84-186) on one observation per
// thread. The value function keeps the reference's explicit dual-linear form
// (:232-253) and the gradient its -J^T grad(loss) + dual + rho*d form
// (:255-279). Control flow (two-loop recursion newest->oldest, descent reset,
// Armijo backtracking on the pre-step objective, Powell damping against
// B0 = I/gamma, pair acceptance test, eviction of the oldest pair beyond
// `lbfgs_memory`, step/grad exits) follows local_opt.cpp line by line.
#pragma once

#include "dbag_common.cuh"
#include "dbag_local.cuh"

namespace dbag {

constexpr int kHuberThreads = 128;

struct HuberProblem {
  double xb[9];    // consensus (xbar | ybar pose)
  double dual[9];  // r | s
  double z0, z1, f, delta, rho_x, rho_y, eps;
};

// Value at v; false if the projection is infeasible. Trig/R/w cached for the
// gradient at the same point.
__device__ __forceinline__ bool hub_value(const HuberProblem& P, const double v[9], Trig& tr,
                                          double R[9], double w[3], double& e0, double& e1,
                                          double& f) {
  trig_of(v[3], v[4], v[5], tr);
  rot_of(tr, R);
  cam_point(R, v, v + 6, w);
  if (!feasible(w[2], P.eps)) return false;
  e0 = P.z0 - P.f * w[0] / w[2];
  e1 = P.z1 - P.f * w[1] / w[2];
  const double a = sqrt(e0 * e0 + e1 * e1);  // losses.cpp:7-20
  double total = a <= P.delta ? 0.5 * a * a : P.delta * (a - 0.5 * P.delta);
  double dd = 0.0, q = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double d = v[k] - P.xb[k];
    dd += P.dual[k] * d;
    q += d * d;
  }
  total += dd + 0.5 * P.rho_x * q;
  dd = 0.0;
  q = 0.0;
#pragma unroll
  for (int k = 3; k < 9; ++k) {
    const double d = v[k] - P.xb[k];
    dd += P.dual[k] * d;
    q += d * d;
  }
  total += dd + 0.5 * P.rho_y * q;
  f = total;
  return true;
}

// Gradient at v from the cached projection state.
__device__ __forceinline__ void hub_grad(const HuberProblem& P, const double v[9], const Trig& tr,
                                         const double R[9], const double w[3], double e0,
                                         double e1, double g[9]) {
  double A0[9], A1[9];
  proj_jacobian(v, tr, R, w, P.f, A0, A1);
  const double a = sqrt(e0 * e0 + e1 * e1);  // losses.cpp:22-38
  double l0, l1;
  if (a == 0.0) {
    l0 = l1 = 0.0;
  } else if (a <= P.delta) {
    l0 = e0;
    l1 = e1;
  } else {
    const double s = P.delta / a;
    l0 = s * e0;
    l1 = s * e1;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double rho = k < 3 ? P.rho_x : P.rho_y;
    g[k] = -(A0[k] * l0 + A1[k] * l1) + (P.dual[k] + rho * (v[k] - P.xb[k]));
  }
}

__device__ __forceinline__ double dot9(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) s += a[k] * b[k];
  return s;
}

// local_opt.cpp:84-186. Returns false when the start is infeasible/non-finite.
__device__ __noinline__ bool local_lbfgs(const DevState& S, const HuberProblem& P, double v[9],
                                         LocalCounters& cnt) {
  Trig tr;
  double R[9], w[3], e0, e1, f;
  if (!hub_value(P, v, tr, R, w, e0, e1, f) || !isfinite(f)) return false;
  double g[9];
  hub_grad(P, v, tr, R, w, e0, e1, g);
  ++cnt.n_jac;
#pragma unroll
  {
    unsigned ex = 0;  // exponent-field max: 0x7ff iff some component is inf / NaN
#pragma unroll
    for (int k = 0; k < 9; ++k) ex = max(ex, (unsigned)__double2hiint(g[k]) & 0x7ff00000u);
    if (ex == 0x7ff00000u) return false;
  }
  double hs[DBAG_MAX_LBFGS_MEMORY][9], hy[DBAG_MAX_LBFGS_MEMORY][9], hrho[DBAG_MAX_LBFGS_MEMORY];
  int h_first = 0, h_size = 0;  // ring buffer: oldest at h_first
  double gamma = 1.0;
  const int mem = S.lbfgs_memory;
  for (int it = 0; it < S.inner_max_iters; ++it) {
    if (sqrt(dot9(g, g)) <= S.grad_tol) return true;  // kGradConverged
    // two-loop recursion (local_opt.cpp:111-122)
    double q[9], alpha[DBAG_MAX_LBFGS_MEMORY];
#pragma unroll
    for (int k = 0; k < 9; ++k) q[k] = g[k];
    for (int kk = h_size - 1; kk >= 0; --kk) {
      const int slot = (h_first + kk) % mem;
      alpha[kk] = hrho[slot] * dot9(hs[slot], q);
#pragma unroll
      for (int k = 0; k < 9; ++k) q[k] -= alpha[kk] * hy[slot][k];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) q[k] *= gamma;
    for (int kk = 0; kk < h_size; ++kk) {
      const int slot = (h_first + kk) % mem;
      const double beta = hrho[slot] * dot9(hy[slot], q);
#pragma unroll
      for (int k = 0; k < 9; ++k) q[k] += (alpha[kk] - beta) * hs[slot][k];
    }
    ++cnt.n_dir;
    cnt.n_pairs += h_size;
    double d[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) d[k] = -q[k];
    double slope = dot9(g, d);
    if (!(slope < 0.0)) {
      h_size = 0;
      h_first = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k) d[k] = -g[k];
      slope = -dot9(g, g);
    }
    // Armijo backtracking (local_opt.cpp:130-147)
    double step = 1.0, ft = 0.0, xt[9], et0 = 0.0, et1 = 0.0, Rt[9], wt[3];
    Trig trt;
    bool accepted = false;
    for (int ls = 0; ls < S.max_line_search; ++ls) {
#pragma unroll
      for (int k = 0; k < 9; ++k) xt[k] = v[k] + step * d[k];
      double fv;
      ++cnt.n_trial;
      if (hub_value(P, xt, trt, Rt, wt, et0, et1, fv) && isfinite(fv) &&
          fv <= f + S.armijo_c * step * slope) {
        ft = fv;
        accepted = true;
        break;
      }
      step *= S.backtrack;
    }
    if (!accepted) return true;  // kLineSearchFailed, best iterate kept
    double gt[9];
    hub_grad(P, xt, trt, Rt, wt, et0, et1, gt);
    ++cnt.n_jac;
    unsigned gex = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) gex = max(gex, (unsigned)__double2hiint(gt[k]) & 0x7ff00000u);
    if (gex == 0x7ff00000u) return true;  // kLineSearchFailed
    ++cnt.n_acc;
    double s[9], y[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      s[k] = xt[k] - v[k];
      y[k] = gt[k] - g[k];
    }
    // Powell damping (local_opt.cpp:155-165)
    const double sBs = dot9(s, s) / gamma;
    double sy = dot9(s, y);
    if (sy < 0.2 * sBs) {
      const double theta = 0.8 * sBs / (sBs - sy);
#pragma unroll
      for (int k = 0; k < 9; ++k) y[k] = theta * y[k] + (1.0 - theta) / gamma * s[k];
      sy = dot9(s, y);
    }
    const double sn = sqrt(dot9(s, s));
    if (sy > 1e-12 * sn * sqrt(dot9(y, y))) {
      // push_back, then pop_front beyond the memory (:166-172)
      int slot;
      if (h_size < mem) {
        slot = (h_first + h_size) % mem;
        ++h_size;
      } else {
        slot = h_first;  // overwrite the oldest == push + pop_front
        h_first = (h_first + 1) % mem;
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        hs[slot][k] = s[k];
        hy[slot][k] = y[k];
      }
      hrho[slot] = 1.0 / sy;
      gamma = sy / dot9(y, y);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      v[k] = xt[k];
      g[k] = gt[k];
    }
    f = ft;
    if (sn <= S.step_tol * (1.0 + sqrt(dot9(v, v)))) return true;  // kStepConverged
  }
  return true;  // kMaxIters
}

#ifndef DBAG_K1_HUB_MINB
#define DBAG_K1_HUB_MINB 3  // 168 regs: 149.8 ms; minBlocks 1 lets ptxas take ~255 regs (186 ms)
#endif
__global__ void __launch_bounds__(kHuberThreads, DBAG_K1_HUB_MINB) k_local_huber(DevState S, int64_t begin,
                                                               int64_t count) {
  const int64_t tix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  LocalCounters cnt;
  if (tix < count) {
    const int64_t b = S.order ? (int64_t)S.order[tix] : begin + tix;  // effort order (full launch)
    const int32_t j = S.blk_cam[b];
    const int32_t i = S.blk_pt[b];
    const int32_t p = S.blk_pos[b];
    const double* yb = S.ybar + 8 * (int64_t)j;
    const double4 xb = S.xbar[i];
    const PointRec rec = S.prec[p];
    HuberProblem P;
    double v[9];
    v[0] = rec.x0;
    v[1] = rec.x1;
    v[2] = rec.x2;
    P.xb[0] = xb.x;
    P.xb[1] = xb.y;
    P.xb[2] = xb.z;
    P.dual[0] = rec.r0;
    P.dual[1] = rec.r1;
    P.dual[2] = rec.r2;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      v[3 + k] = S.cam_soa[(int64_t)k * S.L + b];
      P.dual[3 + k] = S.cam_soa[(int64_t)(6 + k) * S.L + b];
      P.xb[3 + k] = yb[k];
    }
    P.z0 = rec.u;
    P.z1 = rec.v;
    P.f = yb[6];
    P.delta = S.huber_delta;
    P.rho_x = S.rho_x;
    P.rho_y = S.rho_y;
    P.eps = S.eps_depth;
    const unsigned nv0 = cnt.n_trial;
    const bool solved = local_lbfgs(S, P, v, cnt);
    if (S.effort) S.effort[b] = (uint16_t)min(cnt.n_trial - nv0, 65535u);
    if (!solved) {
      atomicMin(reinterpret_cast<unsigned long long*>(S.err_block), (unsigned long long)b);
    } else {
      double* xp = reinterpret_cast<double*>(S.prec + p);
      xp[0] = v[0];
      xp[1] = v[1];
      xp[2] = v[2];
#pragma unroll
      for (int k = 0; k < 6; ++k) S.cam_soa[(int64_t)k * S.L + b] = v[3 + k];
    }
  }
  flush_counters(S, cnt);
}

}  // namespace dbag
