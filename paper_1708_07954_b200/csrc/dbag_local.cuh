// dbag_local.cuh — K1: the per-observation local solve of one ADMM round.
//
// Restates AdmmSolver::local_update for (1,1) blocks (admm_solver.cpp:144-290)
// with the inner solvers of local_opt.cpp: Gauss-Newton (squared L2,
// :20-82) and L-BFGS (Huber, :84-186). One thread owns one observation's
// 9-dim problem (point copy x_i^j, pose copy y_j^i); every branch of the
// reference control flow (damping escalation, non-strict accept, step/grad
// exits, Armijo backtracking, Powell damping, history eviction) is kept.
//
// B200 choices: SoA camera-side state read with one coalesced 8 B load per
// component; the point-side 64 B record gathered from point-major order (the
// only irregular access of the round lives here, hidden behind FP64 work);
// the damped normal equations H + lambda*diag = A^T A + D (A = 2x9 projection
// Jacobian, D diagonal >= rho/2) solved exactly by Woodbury with a 2x2
// capacitance matrix instead of a dense 9x9 LDLT.
#pragma once

#include "dbag_common.cuh"

namespace dbag {

constexpr double kDampingInit = 1e-4;  // local_opt.cpp:13
constexpr double kDampingMax = 1e12;   // local_opt.cpp:14

struct LocalCounters {
  unsigned n_jac = 0, n_trial = 0, n_acc = 0, n_dir = 0, n_pairs = 0;
};

__device__ __forceinline__ void flush_counters(const DevState& S, const LocalCounters& c) {
  // warp-aggregate then one atomic per warp into a striped counter slot
  unsigned long long v[5] = {c.n_jac, c.n_trial, c.n_acc, c.n_dir, c.n_pairs};
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long* slot =
      S.counters + 8 * ((blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % kCounterStripes);
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    unsigned long long s = warp_sum(v[k]);
    if (lane == 0 && s) atomicAdd(slot + k, s);
  }
}

// Residual of the squared-L2 local problem at v (admm_solver.cpp:187-206):
// r = [z - pi(v) ; wx (v_x - tx) ; wy (v_y - ty)], objective ||r||^2 summed in
// row order. Returns false when the projection is infeasible.
struct GnProblem {
  double* tgt;     // x~ (3) and y~ (6), completed-square targets (:152-164), in
                   // shared memory with stride blockDim (keeps them out of spills)
  double z0, z1, f, wx, wy, eps;
  __device__ __forceinline__ double T(int k) const { return tgt[k * 128]; }
};

__device__ __forceinline__ bool gn_residual(const GnProblem& P, const double v[9], Trig& tr,
                                            double R[9], double w[3], double& e0, double& e1,
                                            double& obj) {
  fast_trig_of(v[3], v[4], v[5], tr);
  rot_of(tr, R);
  cam_point(R, v, v + 6, w);
  if (!feasible(w[2], P.eps)) return false;
  const double iw = fast_rcp(w[2]);
  e0 = P.z0 - P.f * w[0] * iw;
  e1 = P.z1 - P.f * w[1] * iw;
  double s = e0 * e0 + e1 * e1;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double wk = k < 3 ? P.wx : P.wy;
    const double rk = wk * (v[k] - P.T(k));
    s += rk * rk;
  }
  obj = s;
  return true;
}

// Projection Jacobian A = d pi / d v (2x9) at v, given R and w = Rx + t
// (geometry.cpp:52-58,141-159): A[:,0:3] = D R, A[:,3+k] = D (dR_k x),
// A[:,6:9] = D. dR_k x uses the staged products Rz Ry Rx.
__device__ __forceinline__ void proj_jacobian(const double v[9], const Trig& t, const double R[9],
                                              const double w[3], double f, double A0[9],
                                              double A1[9]) {
  const double inv_z = fast_rcp(w[2]);
  const double a = f * inv_z;
  const double b0 = -f * w[0] * inv_z * inv_z;
  const double b1 = -f * w[1] * inv_z * inv_z;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    A0[c] = a * R[c] + b0 * R[6 + c];
    A1[c] = a * R[3 + c] + b1 * R[6 + c];
  }
  // q = Rx x, s = Ry q, Rx' = R x (no t)
  const double q1 = t.ca * v[1] - t.sa * v[2];
  const double q2 = t.sa * v[1] + t.ca * v[2];
  const double q0 = v[0];
  const double s0 = t.cb * q0 + t.sb * q2;
  const double s2 = -t.sb * q0 + t.cb * q2;
  // d/dalpha: Rz Ry (0, -q2, q1)
  const double da0 = t.cg * (t.sb * q1) + t.sg * q2;
  const double da1 = t.sg * (t.sb * q1) - t.cg * q2;
  const double da2 = t.cb * q1;
  // d/dbeta: Rz (s2, 0, -s0)
  const double db0 = t.cg * s2, db1 = t.sg * s2, db2 = -s0;
  // d/dgamma: (-(Rx)_1, (Rx)_0, 0)
  const double rx0 = R[0] * v[0] + R[1] * v[1] + R[2] * v[2];
  const double rx1 = R[3] * v[0] + R[4] * v[1] + R[5] * v[2];
  const double dg0 = -rx1, dg1 = rx0;
  A0[3] = a * da0 + b0 * da2;
  A1[3] = a * da1 + b1 * da2;
  A0[4] = a * db0 + b0 * db2;
  A1[4] = a * db1 + b1 * db2;
  A0[5] = a * dg0;
  A1[5] = a * dg1;
  A0[6] = a;
  A1[6] = 0.0;
  A0[7] = 0.0;
  A1[7] = a;
  A0[8] = b0;
  A1[8] = b1;
}

#ifndef DBAG_K1_MINB
#define DBAG_K1_MINB 4  // 128 regs: 16 warps/SM beat spill-free 8 warps (84 -> 67 ms, config 5)
#endif

// FAST L2 K1: a persistent lane-refill state machine with the EXACT kernel's
// structure (one projection per loop iteration shared by a fresh start point
// and a trial point, a warp-local queue of claimed observations, warp-
// aggregated counters) and its later lessons: the Jacobian right
// after an accept / start point from the residual's trig values, R and w in
// registers (no accepted-state slots), the warp's index queue and counters in
// shared memory, and lambda, the objective, the observation and the camera
// pose copy in the shared slice instead of registers.
constexpr int kFast4Scr = 46;  // A0 | A1 | rhs | H_kk (0..35), pose 36..41, lambda, obj, z0, z1
constexpr size_t kFast4Smem = sizeof(double) * (9 + kFast4Scr) * 128;

__global__ void __launch_bounds__(128, DBAG_K1_MINB) k_local_persistent4(DevState S, int64_t begin,
                                                                         int64_t count) {
  extern __shared__ double fp_dyn[];
  __shared__ unsigned long long wcnt[4][3];
  __shared__ WarpQueueS wqs[4];
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wcnt[wid][0] = wcnt[wid][1] = wcnt[wid][2] = 0;
    wqs[wid].q0 = wqs[wid].q1 = 0;
    wqs[wid].end = 0;
  }
  __syncwarp();
  GnProblem P;
  P.tgt = fp_dyn + threadIdx.x;
  double* sc = fp_dyn + 9 * 128 + threadIdx.x;
#define VC(k) sc[(36 + (k)) * 128]
#define LAM sc[42 * 128]
#define OBJ sc[43 * 128]
#define Z0 sc[44 * 128]
#define Z1 sc[45 * 128]
#define CNT(slot, pred)                                                \
  {                                                                    \
    const unsigned c_ = __popc(__ballot_sync(0xffffffffu, pred));      \
    if ((threadIdx.x & 31) == 0 && c_) wcnt[wid][slot] += c_;         \
  }
  P.wx = S.w_x;  // admm_solver.cpp:183-184
  P.wy = S.w_y;
  P.eps = S.eps_depth;
  const double wx2 = P.wx * P.wx, wy2 = P.wy * P.wy;
  const double iwx2 = 1.0 / wx2, iwy2 = 1.0 / wy2;  // D^-1 of the undamped trial
  bool busy = false, exhausted = false;
  int64_t b = -1;
  int it = 0, pos = 0;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;  // the point copy; the pose copy is VC
  for (;;) {
    const int64_t idx = refill_batched_s<64>(S, !busy, count, exhausted, &wqs[wid]);
    const bool fresh = idx >= 0;
    if (fresh) {
      b = begin + idx;
      const int32_t j = S.blk_cam[b];
      const int32_t i = S.blk_pt[b];
      pos = S.blk_pos[b];
      const PointRec rec = S.prec[pos];
      const double* yb = S.ybar + 8 * (int64_t)j;
      const double4 xb = S.xbar[i];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        VC(k) = S.cam_soa[(int64_t)k * S.L + b];
        P.tgt[(3 + k) * 128] = yb[k] - S.cam_soa[(int64_t)(6 + k) * S.L + b] / S.rho_y;
      }
      v0 = rec.x0;
      v1 = rec.x1;
      v2 = rec.x2;
      P.tgt[0] = xb.x - rec.r0 / S.rho_x;
      P.tgt[128] = xb.y - rec.r1 / S.rho_x;
      P.tgt[256] = xb.z - rec.r2 / S.rho_x;
      Z0 = rec.u;
      Z1 = rec.v;
      P.f = yb[6];
      busy = true;
    }
    if (__ballot_sync(0xffffffffu, busy) == 0) {
      if (exhausted) break;
      continue;
    }
    bool done = false;
    // ---- damped solve by Woodbury (see k_local_persistent2)
    double vt[9], d2 = 0.0;
    bool proj = fresh;
    if (busy && !fresh) {
      const double lambda = LAM;
      double iD[9], u[9];
      double c00 = 1.0, c01 = 0.0, c11 = 1.0, a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const double A0k = sc[k * 128], A1k = sc[(9 + k) * 128];
        const double wk2 = k < 3 ? wx2 : wy2;
        iD[k] = lambda > 0.0 ? fast_rcp(wk2 + lambda * fmax(sc[(27 + k) * 128], 1e-12))
                             : (k < 3 ? iwx2 : iwy2);
        u[k] = sc[(18 + k) * 128] * iD[k];
        c00 += A0k * A0k * iD[k];
        c01 += A0k * A1k * iD[k];
        c11 += A1k * A1k * iD[k];
        a0 += A0k * u[k];
        a1 += A1k * u[k];
      }
      const double idet = fast_rcp(c00 * c11 - c01 * c01);  // C is SPD, det >= 1
      const double y0 = (c11 * a0 - c01 * a1) * idet;
      const double y1 = (c00 * a1 - c01 * a0) * idet;
      unsigned ex = 0;  // any non-finite step component: exponent field 0x7ff
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const double dk = u[k] - iD[k] * (sc[k * 128] * y0 + sc[(9 + k) * 128] * y1);
        ex = max(ex, (unsigned)__double2hiint(dk) & 0x7ff00000u);
        d2 += dk * dk;
        vt[k] = (k == 0 ? v0 : k == 1 ? v1 : k == 2 ? v2 : VC(k - 3)) + dk;
      }
      proj = ex != 0x7ff00000u;
    } else {
      vt[0] = v0;
      vt[1] = v1;
      vt[2] = v2;
#pragma unroll
      for (int k = 0; k < 6; ++k) vt[3 + k] = VC(k);
    }
    // ---- one projection + objective, then the Jacobian of a taken point
    bool accepted = false, did_jac = false;
    if (proj) {
      Trig trt;
      double Rt[9], wt[3], et0 = 0.0, et1 = 0.0, objt = 0.0;
      P.z0 = Z0;
      P.z1 = Z1;
      const bool feas = gn_residual(P, vt, trt, Rt, wt, et0, et1, objt);
      const unsigned ex = max(max((unsigned)__double2hiint(et0) & 0x7ff00000u,
                                  (unsigned)__double2hiint(et1) & 0x7ff00000u),
                              (unsigned)__double2hiint(objt) & 0x7ff00000u);
      const bool ok = feas && ex != 0x7ff00000u;
      bool take = false;
      if (fresh) {
        if (ok) {
          take = true;
          it = 0;
        } else {  // the reference throws (local_opt.cpp:25-28)
          atomicMin(reinterpret_cast<unsigned long long*>(S.err_block), (unsigned long long)b);
          busy = false;
        }
      } else if (ok && objt <= OBJ) {  // non-strict accept (:60)
        take = true;
        accepted = true;
        v0 = vt[0];
        v1 = vt[1];
        v2 = vt[2];
        double x2 = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          if (k >= 3) VC(k - 3) = vt[k];
          x2 += vt[k] * vt[k];
        }
        if (sqrt(d2) <= S.step_tol * (1.0 + sqrt(x2))) {
          done = true;  // kStepConverged
        } else {
          ++it;
        }
      }
      if (take) {
        OBJ = objt;
        if (!done) {
          if (it >= S.inner_max_iters) {
            done = true;  // kMaxIters
          } else {
            double A0[9], A1[9];
            proj_jacobian(vt, trt, Rt, wt, P.f, A0, A1);
            did_jac = true;
            double g2 = 0.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              const double wk = k < 3 ? P.wx : P.wy;
              const double jtr = -(A0[k] * et0 + A1[k] * et1) + wk * (wk * (vt[k] - P.T(k)));
              sc[k * 128] = A0[k];
              sc[(9 + k) * 128] = A1[k];
              sc[(18 + k) * 128] = -jtr;  // rhs = -0.5 g
              sc[(27 + k) * 128] = (A0[k] * A0[k] + A1[k] * A1[k]) + (k < 3 ? wx2 : wy2);
              const double gk = 2.0 * jtr;  // g = 2 J^T r
              g2 += gk * gk;
            }
            if (sqrt(g2) <= S.grad_tol) {
              done = true;  // kGradConverged
            } else {
              LAM = 0.0;
            }
          }
        }
      }
    }
    if (busy && !fresh && !accepted) {
      const double lam = LAM;
      const double ln = lam == 0.0 ? kDampingInit : lam * 10.0;
      LAM = ln;
      if (ln > kDampingMax) done = true;
    }
    CNT(1, proj && !fresh);
    CNT(2, accepted);
    CNT(0, did_jac);
    if (busy && done) {
      double* xp = reinterpret_cast<double*>(S.prec + pos);
      xp[0] = v0;
      xp[1] = v1;
      xp[2] = v2;
#pragma unroll
      for (int k = 0; k < 6; ++k) S.cam_soa[(int64_t)k * S.L + b] = VC(k);
      busy = false;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* slot =
        S.counters + 8 * ((blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % kCounterStripes);
    if (wcnt[wid][0]) atomicAdd(slot + 0, wcnt[wid][0]);
    if (wcnt[wid][1]) atomicAdd(slot + 1, wcnt[wid][1]);
    if (wcnt[wid][2]) atomicAdd(slot + 2, wcnt[wid][2]);
  }
#undef VC
#undef LAM
#undef OBJ
#undef Z0
#undef Z1
#undef CNT
}

}  // namespace dbag
