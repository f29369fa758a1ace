// dbag_common.cuh — device state layout and fp64 camera math shared by the
// B200 kernels. See DESIGN.md §HBM layout for the byte budget per observation.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

namespace dbag {

// Launch configuration of a persistent kernel on the CURRENT device: opts the
// kernel in to `smem` bytes of dynamic shared memory (the attribute applies to
// the current device only) and returns the resident CTA count (SMs x CTAs per
// SM). Cached per (kernel, device, threads, smem) under a mutex, so solvers on
// several devices or threads each get their own; every CUDA error is returned.
inline cudaError_t resident_ctas(const void* kern, int threads, size_t smem, int* out) {
  static std::mutex mu;
  static std::map<std::pair<std::pair<const void*, int>, std::pair<int, size_t>>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(std::make_pair(kern, dev), std::make_pair(threads, smem));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  int sms = 0, per_sm = 0;
  if (smem > 48 * 1024 &&
      (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
          cudaSuccess)
    return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem)) !=
      cudaSuccess)
    return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *out = cache[key] = sms * per_sm;
  return cudaSuccess;
}

// Point-side per-copy record, stored in POINT-MAJOR order (copies of one point
// contiguous, ascending camera = ascending block order, admm_solver.cpp:126-140).
// 64 B = two full 32 B sectors: the local solve gathers it once per round, the
// point consensus pass streams it.
// Sector A (bytes 0..31) = x | u: written by K1 (the copy). Sector B (32..63) =
// r | v: written by K2 (the dual). Each kernel dirties one 32 B sector of a
// record, so the write-back to HBM is 32 B per copy and kernel instead of 64.
struct __align__(32) PointRec {
  double x0, x1, x2;  // local point copy x_i^j
  double u;           // observation z (read-only)
  double r0, r1, r2;  // dual r_i^j
  double v;           // observation z (read-only)
};
constexpr int kRecX = 0, kRecU = 3, kRecR = 4, kRecV = 7;  // offsets in doubles
static_assert(sizeof(PointRec) == 64, "PointRec must be 64 B");

// 256-bit global loads / stores (sm_100: LDG.E.256 / STG.E.256), 32 B aligned
// addresses. A gather of 64 B records or 32 B consensus points by a warp costs
// one L1 wavefront per lane and per instruction, so halving the instruction
// count halves the L1 data-pipe work of the gather (K2 is bound by it).
__device__ __forceinline__ void ldg256(const void* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
// read-only data (not written by the running kernel)
__device__ __forceinline__ void ldg256_nc(const void* p, double& a, double& b, double& c,
                                          double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ PointRec load_rec256(const PointRec* p) {
  PointRec r;
  ldg256(p, r.x0, r.x1, r.x2, r.u);
  ldg256(reinterpret_cast<const double*>(p) + 4, r.r0, r.r1, r.r2, r.v);
  return r;
}

// Everything a kernel needs, passed by value (fits the 4 KB param space).
struct DevState {
  int64_t L;       // observations == blocks (1,1)
  int32_t M, N;    // cameras, points
  // block order (sorted by (cam, pt)): camera-side SoA [12][L] = y(6) | s(6)
  double* cam_soa;
  int32_t* blk_cam;   // [L]
  int32_t* blk_pt;    // [L]
  int32_t* blk_pos;   // [L] point-major position of block b
  int32_t* blk_obs;   // [L] input observation index of block b
  // point-major
  PointRec* prec;     // [L]
  int32_t* pm_cam;    // [L] camera of point-major position p
  int32_t* pt_off;    // [N+1]
  int32_t* pt_order;  // [N] processing order (by descending track length)
  int32_t* cam_off;   // [M+1]
  // consensus
  double4* xbar;      // [N] (x, y, z, 0)
  double* ybar;       // [M][8] (alpha, beta, gamma, t0, t1, t2, f, 0)
  double* camR;       // [M][16] R(9) t(3) f at ybar (for the fused metric)
  // reference state for the MSE columns
  double* ref_pose;   // [M][6] or null
  double* ref_pts;    // [N][3] or null
  // options
  double rho_x, rho_y, eps_depth, huber_delta;
  double w_x, w_y;  // sqrt(0.5 * rho): the residual row weights (admm_solver.cpp:183-184)
  double y_x, y_y;  // RN(1 / rho): the reciprocal the EXACT K1's target divisions correct (host '/')
  double grad_tol, step_tol, armijo_c, backtrack;
  int32_t inner_max_iters, lbfgs_memory, max_line_search, loss;
  // reductions
  double* part_pt;        // [gridK2][4] sum_err, max_px, max_dx, infeasible
  double* cam_stats;      // [M][2] primal_y, dual_y
  double* part_mse;       // [gridMSE][2]
  unsigned long long* counters;  // [kCounterStripes][8]
  int64_t* err_block;     // first block that raised (local_update_all)
  // Inside a fused round (iterate/run/enqueue_round) = err_block: the
  // consensus/dual kernels return at once when the round's local solve raised,
  // as the reference's local_update_all throws before consensus_update and
  // dual_update run (admm_solver.cpp:292-316, 437-443). Null otherwise.
  const int64_t* gate;
  int64_t* err_obs;       // first infeasible observation (input order)
  double* record;         // DevRecord
  double* metric_part;    // [kRecFields] this rank's partial record (raw sums)
  unsigned long long* work;  // K1 work counter (zeroed before each launch)
  int32_t k1_batch;          // K1 claim batch (0: the kernel's default), set per launch
  // effort-ordered Huber K1: value evaluations of each observation's last local
  // solve, and the processing order the next full launch uses (null: block order)
  uint16_t* effort;   // [L]
  const int32_t* order;  // [L] or null
  // pooled Huber K1 (EXACT): L-BFGS histories, one record per resident slot
  double* hub_hist;
  int64_t hub_hist_doubles;
  // ---- multi-GPU shard (null/0 on a single-GPU solver) ----
  int32_t world, rank;
  int32_t* bp_of_local;   // [N] global boundary index of a local point, or -1
  int8_t* owner_of_local; // [N] 1 if this rank counts the point in point-wise sums
  int64_t* gb_off;        // [B+1] global boundary copy ranges (reference copy order)
  int64_t* gmap;          // [G] per global boundary copy of a point held here: >= 0 its
                          // recv slot; -2 - p for an own copy at point-major position p
  int32_t* send_pos;      // [send_count] point-major position of each send slot
  int64_t send_count, recv_count;
  double* send_buf;       // [send_count][6] x(3) r(3), grouped by destination peer
  double* recv_buf;       // [recv_count][6], grouped by source peer
  double* metric_recv;    // [world][kRecFields]
};

constexpr int kCounterStripes = 64;

// Copy (x, r) of a boundary point from its gmap slot: a peer's copy in the
// receive buffer, or this rank's own copy in the point-major records.
__device__ __forceinline__ void boundary_copy(const DevState& S, int64_t slot, double c[6]) {
  if (slot >= 0) {
    const double* a = S.recv_buf + 6 * slot;
#pragma unroll
    for (int k = 0; k < 6; ++k) c[k] = a[k];
  } else {
    const double* a = reinterpret_cast<const double*>(S.prec + (-2 - slot));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c[k] = a[kRecX + k];
      c[3 + k] = a[kRecR + k];
    }
  }
}

// Lane-level work refill for persistent K1 kernels: every idle lane of the
// warp takes the next observation index (one atomic per warp). Returns the
// lane's new index or -1 when the work is exhausted.
__device__ __forceinline__ int64_t refill(const DevState& S, bool idle, int64_t count,
                                          bool& exhausted) {
  const unsigned full = 0xffffffffu;
  const unsigned m = __ballot_sync(full, idle && !exhausted);
  if (m == 0) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(S.work, (unsigned long long)__popc(m));
  base = __shfl_sync(full, base, leader);
  if (base + __popc(m) >= (unsigned long long)count) exhausted = true;
  if (!(m & (1u << lane))) return -1;
  const unsigned long long idx = base + __popc(m & ((1u << lane) - 1u));
  return idx < (unsigned long long)count ? (int64_t)idx : -1;
}

// refill() with a warp-local queue [q0, q1) of claimed indices, kept in shared
// memory (warp-uniform state off the register file; every lane reads it, the
// leader writes it back): one global atomic per batch of observations instead
// of one per refill. Every index is still taken exactly once; lanes take queue
// entries in lane order. The batch is kBatch, or S.k1_batch when smaller (a
// small problem takes smaller batches, so the warps' last claims even out).
struct WarpQueueS {
  unsigned long long q0, q1;
  unsigned end;
};
template <int kBatch>
__device__ __forceinline__ int64_t refill_batched_s(const DevState& S, bool idle, int64_t count,
                                                    bool& exhausted, WarpQueueS* q) {
  const unsigned full = 0xffffffffu;
  const unsigned m = __ballot_sync(full, idle && !exhausted);
  if (m == 0) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  const unsigned n = __popc(m);
  const unsigned rank = __popc(m & ((1u << lane) - 1u));
  unsigned long long q0 = q->q0, q1 = q->q1;
  bool end = q->end != 0;
  const unsigned long long r = q1 - q0;
  unsigned long long idx;
  if (r >= n) {
    idx = q0 + rank;
    q0 += n;
  } else {
    const unsigned need = n - (unsigned)r;
    const unsigned bsz =
        S.k1_batch > 0 && S.k1_batch < kBatch ? (unsigned)S.k1_batch : (unsigned)kBatch;
    const unsigned want = need > bsz ? need : bsz;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(S.work, (unsigned long long)want);
    base = __shfl_sync(full, base, leader);
    idx = rank < r ? q0 + rank : base + (rank - r);
    q0 = base + need;
    q1 = base + want;
    if (q1 >= (unsigned long long)count) {
      end = true;
      q1 = (unsigned long long)count;
      if (q0 > q1) q0 = q1;
    }
  }
  __syncwarp();
  if (lane == leader) {
    q->q0 = q0;
    q->q1 = q1;
    q->end = end;
  }
  __syncwarp();
  if (end && q0 >= q1) exhausted = true;
  if (!(m & (1u << lane))) return -1;
  return idx < (unsigned long long)count ? (int64_t)idx : -1;
}

// DevRecord layout (doubles)
enum RecField {
  kRecSumErr = 0, kRecMaxPx, kRecMaxPy, kRecMaxDx, kRecMaxDy, kRecInfeasible, kRecCamMse,
  kRecPtMse, kRecFields
};

// ---------------------------------------------------------------------------
// Camera model, geometry.cpp:9-99,141-159. R = Rz(g) Ry(b) Rx(a), formed as
// (Rz*Ry)*Rx like rotation_from_euler (geometry.cpp:62-64), with the
// structural zeros folded.
// ---------------------------------------------------------------------------
struct Trig {
  double sa, ca, sb, cb, sg, cg;
};

__device__ __forceinline__ void trig_of(double a, double b, double g, Trig& t) {
  sincos(a, &t.sa, &t.ca);
  sincos(b, &t.sb, &t.cb);
  sincos(g, &t.sg, &t.cg);
}

// FAST numerics helpers (never used by the EXACT kernels) ---------------------
// 1/x to ~1 ulp: MUFU.RCP64H seed + two Newton steps, branch-free.
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// sin and cos of |x| <= 1e5 (the Euler angles): Cody-Waite reduction by pi/2
// with FMA, Taylor polynomials to x^17 / x^18 on [-pi/4, pi/4], branch-free
// quadrant select; ~1 ulp. Straight-line code, so three calls interleave.
__device__ __forceinline__ void fast_sincos(double x, double* sn, double* cs) {
  const double k = rint(x * 0.6366197723675814);
  double r = fma(-k, 1.5707963267948966, x);
  r = fma(-k, 6.123233995736766e-17, r);
  const double z = r * r;
  double p = 2.8114572543455206e-15;
  p = fma(p, z, -7.647163731819816e-13);
  p = fma(p, z, 1.6059043836821613e-10);
  p = fma(p, z, -2.505210838544172e-08);
  p = fma(p, z, 2.7557319223985893e-06);
  p = fma(p, z, -0.0001984126984126984);
  p = fma(p, z, 0.008333333333333333);
  p = fma(p, z, -0.16666666666666666);
  const double s = fma(r * z, p, r);
  double q = -1.5619206968586225e-16;
  q = fma(q, z, 4.779477332387385e-14);
  q = fma(q, z, -1.1470745597729725e-11);
  q = fma(q, z, 2.08767569878681e-09);
  q = fma(q, z, -2.755731922398589e-07);
  q = fma(q, z, 2.48015873015873e-05);
  q = fma(q, z, -0.001388888888888889);
  q = fma(q, z, 0.041666666666666664);
  const double c = fma(z * z, q, fma(-0.5, z, 1.0));
  const int n = static_cast<int>(static_cast<long long>(k) & 3);
  const double s1 = (n & 1) ? c : s, c1 = (n & 1) ? s : c;
  *sn = (n & 2) ? -s1 : s1;
  *cs = ((n + 1) & 2) ? -c1 : c1;
}

__device__ __forceinline__ void fast_trig_of(double a, double b, double g, Trig& t) {
  if (fabs(a) < 1e5 && fabs(b) < 1e5 && fabs(g) < 1e5) {
    fast_sincos(a, &t.sa, &t.ca);
    fast_sincos(b, &t.sb, &t.cb);
    fast_sincos(g, &t.sg, &t.cg);
  } else {
    trig_of(a, b, g, t);
  }
}

__device__ __forceinline__ void rot_of(const Trig& t, double R[9]) {
  const double m01 = -t.sg, m02 = t.cg * t.sb;
  const double m11 = t.cg, m12 = t.sg * t.sb;
  const double m22 = t.cb;
  R[0] = t.cg * t.cb;
  R[1] = m01 * t.ca + m02 * t.sa;
  R[2] = m01 * (-t.sa) + m02 * t.ca;
  R[3] = t.sg * t.cb;
  R[4] = m11 * t.ca + m12 * t.sa;
  R[5] = m11 * (-t.sa) + m12 * t.ca;
  R[6] = -t.sb;
  R[7] = m22 * t.sa;
  R[8] = m22 * t.ca;
}

// w = R x + t (geometry.cpp:93)
__device__ __forceinline__ void cam_point(const double R[9], const double* x, const double* t,
                                          double w[3]) {
  w[0] = (R[0] * x[0] + R[1] * x[1] + R[2] * x[2]) + t[0];
  w[1] = (R[3] * x[0] + R[4] * x[1] + R[5] * x[2]) + t[1];
  w[2] = (R[6] * x[0] + R[7] * x[1] + R[8] * x[2]) + t[2];
}

// Feasibility test of geometry.cpp:95 (`!(w3 >= eps)` also rejects NaN).
__device__ __forceinline__ bool feasible(double w2, double eps) { return w2 >= eps; }

// Lower-pass block reduce helpers (deterministic fixed-shape trees).
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

template <int NT, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /*[NT/32][K]*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) smem[wid * K + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = smem[k];
      for (int w = 1; w < NT / 32; ++w) s += smem[w * K + k];
      v[k] = s;
    }
  }
  __syncthreads();
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = smem[0];
    for (int w = 1; w < NT / 32; ++w) s = fmax(s, smem[w]);
    v = s;
  }
  __syncthreads();
  return v;
}

}  // namespace dbag
