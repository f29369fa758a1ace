// dbag_blocks.cu — generalized local blocks (BlockConfig{π, κ}), EXACT numerics.
// Compiled with -fmad=false: every formula follows oracle/oracle.cpp (the
// restatement of admm_solver.cpp:14-290, local_opt.cpp:20-186) operation for
// operation, so the trajectory is bit-identical to the oracle's (tests/
// test_gpu_blocks.py). One CTA solves one block at a time (persistent grid):
//  - residuals / Jacobians / loss gradients: one thread per observation;
//  - g = 2 J^T r and H = J^T J: one thread per entry, each summing its rows in
//    the oracle's row order (observations ascending, then the weight row;
//    structurally-zero products are skipped, which is exact: +0 + ±0 = +0);
//  - the pivoted LDLT (oracle ldlt_solve, Eigen's left-looking algorithm):
//    its pivot sequence depends only on the ORIGINAL diagonal (a trailing
//    diagonal is never updated before its own step), so it is found up front by
//    one warp; the factorization of P Hd P^T then runs unpivoted with one
//    thread per row and two barriers per column, the solves as a column sweep
//    (forward) and a sequential chain (backward, its order is ascending j);
//  - sequential sums (objective, norms, dots) on one thread, in order.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "../../include/dbag.h"
#include "dbag_blocks.h"
#include "dbag_exact_geom.cuh"

namespace dbag {
namespace blocks {

// ---------------------------------------------------------------------------
// host: partition (admm_solver.cpp:14-72) and communication_cost (:74-101)
// ---------------------------------------------------------------------------
Partition partition_sorted(int64_t L, const int32_t* cam, const int32_t* pt, int32_t ppb,
                           int32_t cpb) {
  Partition P;
  P.obs_off.push_back(0);
  P.pt_off.push_back(0);
  P.cam_off.push_back(0);
  P.obs_pl.resize(L);
  P.obs_cl.resize(L);
  std::vector<int32_t> pts, cams;  // the block's sets (insertion order)
  int64_t begin = 0;
  auto flush = [&](int64_t end) {
    if (end == begin) return;
    std::sort(pts.begin(), pts.end());
    std::sort(cams.begin(), cams.end());
    for (int64_t k = begin; k < end; ++k) {
      P.obs_pl[k] = (int32_t)(std::lower_bound(pts.begin(), pts.end(), pt[k]) - pts.begin());
      P.obs_cl[k] = (int32_t)(std::lower_bound(cams.begin(), cams.end(), cam[k]) - cams.begin());
    }
    P.pt_ids.insert(P.pt_ids.end(), pts.begin(), pts.end());
    P.cam_ids.insert(P.cam_ids.end(), cams.begin(), cams.end());
    P.obs_off.push_back(end);
    P.pt_off.push_back((int64_t)P.pt_ids.size());
    P.cam_off.push_back((int64_t)P.cam_ids.size());
    P.max_np = std::max<int32_t>(P.max_np, (int32_t)pts.size());
    P.max_nc = std::max<int32_t>(P.max_nc, (int32_t)cams.size());
    P.max_nobs = std::max<int32_t>(P.max_nobs, (int32_t)(end - begin));
    pts.clear();
    cams.clear();
    begin = end;
  };
  for (int64_t k = 0; k < L; ++k) {
    // membership in the current block: linear scans are fine, |set| <= π, κ
    const bool new_pt = std::find(pts.begin(), pts.end(), pt[k]) == pts.end();
    const bool new_cam = std::find(cams.begin(), cams.end(), cam[k]) == cams.end();
    if ((int64_t)pts.size() + new_pt > ppb || (int64_t)cams.size() + new_cam > cpb) flush(k);
    if (std::find(pts.begin(), pts.end(), pt[k]) == pts.end()) pts.push_back(pt[k]);
    if (std::find(cams.begin(), cams.end(), cam[k]) == cams.end()) cams.push_back(cam[k]);
  }
  flush(L);
  return P;
}

int64_t communication_cost(const Partition& P, int32_t M, int32_t N) {
  std::vector<std::vector<int32_t>> pp(N), cp(M);
  for (int64_t b = 0; b < P.blocks(); ++b) {
    const int32_t owner = P.cam_ids[P.cam_off[b]];  // block.cam_ids.front()
    for (int64_t q = P.pt_off[b]; q < P.pt_off[b + 1]; ++q) pp[P.pt_ids[q]].push_back(owner);
    for (int64_t q = P.cam_off[b]; q < P.cam_off[b + 1]; ++q) cp[P.cam_ids[q]].push_back(owner);
  }
  auto distinct = [](std::vector<int32_t>& v) {
    std::sort(v.begin(), v.end());
    return (int64_t)(std::unique(v.begin(), v.end()) - v.begin());
  };
  int64_t total = 0;
  for (auto& v : pp) {
    const int64_t o = distinct(v);
    total += 3 * o * (o - 1);
  }
  for (auto& v : cp) {
    const int64_t o = distinct(v);
    total += 6 * o * (o - 1);
  }
  return total;
}

// ---------------------------------------------------------------------------
// device: shared-memory carve-out of one CTA
// ---------------------------------------------------------------------------
constexpr int kGenThreads = 128;
#ifndef DBAG_WARP_BLOCK_MAX_DIM
#define DBAG_WARP_BLOCK_MAX_DIM 64
#endif
constexpr int kWarpBlockMaxDim = DBAG_WARP_BLOCK_MAX_DIM;  // D at or below: a warp per block
constexpr double kDampingInit = 1e-4;  // local_opt.cpp:13
constexpr double kDampingMax = 1e12;   // local_opt.cpp:14

__host__ __device__ inline int64_t tri(int p, int q) { return (int64_t)p * (p + 1) / 2 + q; }

struct Carve {
  double *v, *tgt, *g, *hdg, *hd, *x, *vt, *dl, *piv, *fcam, *A, *r, *rt, *uv, *lg, *M, *red;
  double *hs, *hy, *hrho, *alpha;  // L-BFGS history (Huber)
  int *opl, *ocl, *pto_off, *pto, *cmo_off, *pco, *ord, *flag;
};

// Offsets for the maxima; returns the bytes (M included iff m_in_smem). mem > 0
// (Huber / L-BFGS) adds the consensus copy, loss gradients and the history;
// Gauss-Newton reuses x / dl / vt as pivot and temp scratch instead.
__host__ __device__ inline size_t carve(char* base, int D, int NP, int NC, int NO, int mem,
                                        bool m_in_smem, Carve* c) {
  size_t off = 0;
  auto take_d = [&](size_t n) {
    double* p = reinterpret_cast<double*>(base + off);
    off += sizeof(double) * n;
    return p;
  };
  Carve k{};
  k.v = take_d(D);
  k.tgt = take_d(D);
  k.g = take_d(D);
  k.hdg = take_d(D);
  k.hd = take_d(D);
  k.x = take_d(D);
  k.vt = take_d(D);
  k.dl = take_d(D);
  k.piv = mem > 0 ? take_d(D) : nullptr;
  k.fcam = take_d(NC);
  k.A = take_d((size_t)NO * 18);
  k.r = take_d((size_t)NO * 2);
  k.rt = take_d((size_t)NO * 2);
  k.uv = take_d((size_t)NO * 2);
  k.lg = mem > 0 ? take_d((size_t)NO * 2) : nullptr;
  k.red = take_d(8);
  k.hs = mem > 0 ? take_d((size_t)mem * D) : nullptr;
  k.hy = mem > 0 ? take_d((size_t)mem * D) : nullptr;
  k.hrho = mem > 0 ? take_d(mem) : nullptr;
  k.alpha = mem > 0 ? take_d(mem) : nullptr;
  k.M = m_in_smem ? take_d(tri(D, 0)) : nullptr;
  auto take_i = [&](size_t n) {
    int* p = reinterpret_cast<int*>(base + off);
    off += sizeof(int) * n;
    return p;
  };
  k.opl = take_i(NO);
  k.ocl = take_i(NO);
  k.pto_off = take_i(NP + 1);
  k.pto = take_i(NO);
  k.cmo_off = take_i(NC + 1);
  k.pco = take_i((size_t)NP * NC);
  k.ord = take_i(D);
  k.flag = take_i(8);
  off = (off + 15) & ~size_t(15);
  if (c) *c = k;
  return off;
}

// ---------------------------------------------------------------------------
// Thread groups: kT = 128 (a CTA per block) or 32 (a warp per block, for small
// blocks: four blocks per CTA, warp barriers).
template <int kT>
__device__ __forceinline__ int gtid() {
  return kT == kGenThreads ? (int)threadIdx.x : (int)(threadIdx.x & (kT - 1));
}
template <int kT>
__device__ __forceinline__ void gsync() {
  if (kT == 32)
    __syncwarp();
  else
    __syncthreads();
}

// ---------------------------------------------------------------------------
// device: one block's problem
// ---------------------------------------------------------------------------
struct Blk {
  int64_t b, o0, p0, c0;
  int nobs, np, nc, D, cb;
  double wx, wy;
};

// Project observation o at vector V (point block | camera block), eproject's
// order (geometry.cpp:92-99) on the 9 gathered parameters.
__device__ __forceinline__ bool gproject(const DevState& S, const Blk& k, const Carve& c,
                                         const double* V, int o, exact::ETrig& t, double R[9],
                                         double w[3], double z[2], double v9[9]) {
  const int q = c.opl[o], cc = c.ocl[o];
  v9[0] = V[3 * q];
  v9[1] = V[3 * q + 1];
  v9[2] = V[3 * q + 2];
#pragma unroll
  for (int m = 0; m < 6; ++m) v9[3 + m] = V[k.cb + 6 * cc + m];
  return exact::eproject(v9, c.fcam[cc], S.eps_depth, t, R, w, z);
}

// Variable i -> (is_point, local index, coordinate).
__device__ __forceinline__ void var_of(const Blk& k, int i, bool& pt, int& idx, int& co) {
  if (i < k.cb) {
    pt = true;
    idx = i / 3;
    co = i - 3 * idx;
  } else {
    pt = false;
    idx = (i - k.cb) / 6;
    co = i - k.cb - 6 * idx;
  }
}
// Column of variable i inside an observation's 2x9 Jacobian rows.
__device__ __forceinline__ int jcol(bool pt, int co) { return pt ? co : 3 + co; }

// Residuals at V for every observation (one thread each) into rr[2*nobs];
// flag[0] := 1 if any projection is infeasible or any row is non-finite.
template <int kT>
__device__ __forceinline__ void residuals(const DevState& S, const Blk& k, const Carve& c, const double* V,
                          double* rr) {
  for (int o = gtid<kT>(); o < k.nobs; o += kT) {
    exact::ETrig t;
    double R[9], w[3], z[2], v9[9];
    if (!gproject(S, k, c, V, o, t, R, w, z, v9)) {
      c.flag[0] = 1;
      continue;
    }
    const double e0 = c.uv[2 * o] - z[0], e1 = c.uv[2 * o + 1] - z[1];
    rr[2 * o] = e0;
    rr[2 * o + 1] = e1;
    if (!isfinite(e0) || !isfinite(e1)) c.flag[0] = 1;
  }
}

// Jacobian rows (positive e.Jp | e.Jc, geometry.cpp:141-159) at V.
template <int kT>
__device__ __forceinline__ void jacobians(const DevState& S, const Blk& k, const Carve& c, const double* V) {
  for (int o = gtid<kT>(); o < k.nobs; o += kT) {
    exact::ETrig t;
    double R[9], w[3], z[2], v9[9];
    if (!gproject(S, k, c, V, o, t, R, w, z, v9)) {
      c.flag[1] = 1;  // cannot happen at a feasible iterate; kSingular then
      continue;
    }
    exact::erot(t, R);
    double A0[9], A1[9];
    exact::ejac(v9, t, R, w, c.fcam[c.ocl[o]], A0, A1);
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      c.A[18 * o + m] = A0[m];
      c.A[18 * o + 9 + m] = A1[m];
    }
  }
}

// The observations touching variable i, ascending: [lo, hi) of `list` (or a
// contiguous range for a camera, whose observations are contiguous).
struct Span {
  const int* list;
  int lo, hi;
  __device__ int at(int n) const { return list ? list[n] : n; }
};
__device__ __forceinline__ Span obs_of(const Carve& c, bool pt, int idx) {
  if (pt) return Span{c.pto, c.pto_off[idx], c.pto_off[idx + 1]};
  return Span{nullptr, c.cmo_off[idx], c.cmo_off[idx + 1]};
}

// H(i,j) = sum_k J(k,i) J(k,j) over the rows in order (oracle gauss_newton);
// the weight row adds w*w on the diagonal only.
__device__ __forceinline__ double h_entry(const Blk& k, const Carve& c, int i, int j) {
  bool pi, pj;
  int ii, ij, ci, cj;
  var_of(k, i, pi, ii, ci);
  var_of(k, j, pj, ij, cj);
  const int ai = jcol(pi, ci), aj = jcol(pj, cj);
  double s = 0.0;
  if (pi == pj) {
    if (ii != ij) return 0.0;
    const Span sp = obs_of(c, pi, ii);
    for (int n = sp.lo; n < sp.hi; ++n) {
      const double* a = c.A + 18 * sp.at(n);
      s += a[ai] * a[aj];
      s += a[9 + ai] * a[9 + aj];
    }
    if (i == j) {
      const double w = pi ? k.wx : k.wy;
      s += w * w;
    }
    return s;
  }
  const int q = pi ? ii : ij, cm = pi ? ij : ii;
  const int o = c.pco[q * k.nc + cm];
  if (o < 0) return 0.0;
  const double* a = c.A + 18 * o;
  s += a[ai] * a[aj];
  s += a[9 + ai] * a[9 + aj];
  return s;
}

// Sequential sum of squares of the residual rows (sq_norm, oracle order).
__device__ __forceinline__ double objective_rows(const Blk& k, const Carve& c, const double* rr, const double* V) {
  double s = 0.0;
  for (int n = 0; n < 2 * k.nobs; ++n) s += rr[n] * rr[n];
  for (int i = 0; i < k.D; ++i) {
    const double w = i < k.cb ? k.wx : k.wy;
    const double rw = w * (V[i] - c.tgt[i]);
    s += rw * rw;
  }
  return s;
}

__device__ __forceinline__ bool weight_rows_finite(const Blk& k, const Carve& c, const double* V) {
  // all rows finite iff the largest exponent field stays below 0x7ff (inf and
  // NaN are exactly that field): independent rows, no short-circuit chain
  unsigned ex = 0;
  for (int i = 0; i < k.D; ++i) {
    const double w = i < k.cb ? k.wx : k.wy;
    ex = max(ex, (unsigned)__double2hiint(w * (V[i] - c.tgt[i])) & 0x7ff00000u);
  }
  return ex != 0x7ff00000u;
}

__device__ __forceinline__ double seq_dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// Pivot sequence of the oracle's ldlt_solve over |hd|: at step k the first
// position holding the largest value among k..D-1 (strict '>' from a[k]),
// then a transposition. One warp; ord[p] = variable at position p. Scratch:
// c.x (filled with the permuted right-hand side only afterwards).
template <int kT>
__device__ __forceinline__ void pivot_order(const Blk& k, const Carve& c) {
  if (gtid<kT>() >= 32) return;
  const int lane = gtid<kT>();
  double* a = c.x;
  for (int i = lane; i < k.D; i += 32) {
    a[i] = fabs(c.hd[i]);
    c.ord[i] = i;
  }
  __syncwarp();
  for (int s = 0; s < k.D; ++s) {
    double bv = -INFINITY;
    int bp = 0x7fffffff;
    for (int i = s + 1 + lane; i < k.D; i += 32) {
      const double ai = a[i];
      if (ai > bv) {  // positions ascend per lane: first max of the lane's subset
        bv = ai;
        bp = i;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
      const int op = __shfl_xor_sync(0xffffffffu, bp, d);
      if (ov > bv || (ov == bv && op < bp)) {
        bv = ov;
        bp = op;
      }
    }
    const double ak = a[s];
    const int big = bv > ak ? bp : s;  // NaN a[s]: nothing is larger, no swap
    __syncwarp();
    if (lane == 0 && big != s) {
      const double ta = a[s];
      a[s] = a[big];
      a[big] = ta;
      const int to = c.ord[s];
      c.ord[s] = c.ord[big];
      c.ord[big] = to;
    }
    __syncwarp();
  }
}

// The same pivot order in parallel, verified: every thread ranks its
// variables by |hd| (descending, ties by index) and scatters them. The
// selection loop yields exactly that order when the sorted values are
// strictly decreasing except for ties between consecutive variables (i, i+1)
// sorted to positions p, p+1 with p <= i: variables i and i+1 keep positions
// i and i+1 until step i (a variable moves only when displaced at its own
// position), so when their value becomes the largest at step p <= i, i comes
// first. This covers the structural ties, t_x and t_y of a camera (d00 ==
// d11 in every observation's Jacobian). Anything else (other ties, NaN)
// falls back to pivot_order. tests/test_pivot_network.py checks the rule.
template <int kT>
__device__ __forceinline__ void pivot_order_par(const Blk& k, const Carve& c) {
  const int D = k.D;
  if (gtid<kT>() == 0) c.flag[6] = 0;
  gsync<kT>();
  for (int i = gtid<kT>(); i < D; i += kT) {
    const double ai = fabs(c.hd[i]);
    int r = 0;
    for (int j = 0; j < D; ++j) {
      const double aj = fabs(c.hd[j]);
      r += (aj > ai || (aj == ai && j < i)) ? 1 : 0;
    }
    if (!(ai == ai) || r >= D) c.flag[6] = 1;  // NaN: ranks are not a permutation
    else c.ord[r] = i;
  }
  gsync<kT>();
  if (c.flag[6] == 0) {
    for (int p = gtid<kT>(); p + 1 < D; p += kT) {
      const int a = c.ord[p], b = c.ord[p + 1];
      const double x = fabs(c.hd[a]), y = fabs(c.hd[b]);
      if (!(x > y || (x == y && b == a + 1 && p <= a))) c.flag[6] = 1;
    }
  }
  gsync<kT>();
  if (c.flag[6] != 0) {
    gsync<kT>();
    pivot_order<kT>(k, c);
  }
}

// delta = (P^T LDL^T P)^{-1} rhs for Hd (oracle ldlt_solve on the permuted
// system). M: lower triangle of P Hd P^T (row p at p(p+1)/2), filled here.
// Result in c.dl. Scratch: c.dl / c.vt (temp[] double buffer), c.hdg is kept.
__device__ __forceinline__ int rowp(int i) { return i * (i + 1) / 2; }

__device__ __forceinline__ int mix(int i, int j, int D) { return rowp(i) + j; }

template <int kT, bool kSharedM>
__device__ __forceinline__ void ldlt_solve(const Blk& k, const Carve& c, double* M) {
  const int D = k.D;
  pivot_order_par<kT>(k, c);
  gsync<kT>();
  const int ne = rowp(D);
  for (int e = gtid<kT>(); e < ne; e += kT) {
    int p = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);  // approximate; fixed below
    while (rowp(p + 1) <= e) ++p;
    while (rowp(p) > e) --p;
    const int q = e - rowp(p);
    const int i = c.ord[p], j = c.ord[q];
    M[mix(p, q, D)] = p == q ? c.hd[i] : h_entry(k, c, i, j);
  }
  for (int p = gtid<kT>(); p < D; p += kT) c.x[p] = c.g[c.ord[p]];  // P rhs (g holds rhs)
  gsync<kT>();
  // Left-looking LDL^T, unpivoted (the permutation is already applied).
  // temp[j] = D_j L_kj for the next column is formed during this column's
  // division phase (double buffer), so each column costs two barriers.
  double* tbuf[2] = {c.dl, c.vt};
  bool stop = false;
  for (int kk = 0; kk < D && !stop; ++kk) {
    const double* tc = tbuf[kk & 1];
    double* tn = tbuf[(kk + 1) & 1];
    if (kk > 0) {
      for (int i = kk + gtid<kT>(); i < D; i += kT) {
        double s = 0.0;
        const double* Mi = M + rowp(i);
        for (int j = 0; j < kk; ++j) s += Mi[j] * tc[j];
        M[mix(i, kk, D)] = M[mix(i, kk, D)] - s;
      }
      gsync<kT>();
    }
    const double akk = M[mix(kk, kk, D)];
    const bool valid = fabs(akk) > 0.0;
    if (kk == 0 && !valid) {
      stop = true;  // Eigen: all-zero diagonal, nothing factorized
    } else {
      for (int i = kk + 1 + gtid<kT>(); i < D; i += kT) {
        const int e = mix(i, kk, D);
        if (valid) M[e] = M[e] / akk;
        if (i == kk + 1) tn[kk] = akk * M[e];  // D_kk L_{kk+1,kk}
      }
      if (kk + 1 < D)
        for (int j = gtid<kT>(); j < kk; j += kT) tn[j] = M[mix(j, j, D)] * M[mix(kk + 1, j, D)];
    }
    gsync<kT>();
  }
  // forward substitution, column sweep (same per-row order as the oracle)
  for (int j = 0; j < D - 1; ++j) {
    const double xj = c.x[j];
    for (int i = j + 1 + gtid<kT>(); i < D; i += kT) c.x[i] = c.x[i] - M[mix(i, j, D)] * xj;
    gsync<kT>();
  }
  const double tol = 2.2250738585072014e-308;  // DBL_MIN
  for (int i = gtid<kT>(); i < D; i += kT) {
    const double d = M[mix(i, i, D)];
    c.x[i] = fabs(d) > tol ? c.x[i] / d : 0.0;
  }
  gsync<kT>();
  // backward substitution, column sweep (oracle.cpp ldlt_solve: x_i -= L_ji x_j
  // for j = D-1 down to 1)
  for (int j = D - 1; j > 0; --j) {
    const double xj = c.x[j];
    for (int i = gtid<kT>(); i < j; i += kT) c.x[i] = c.x[i] - M[mix(j, i, D)] * xj;
    gsync<kT>();
  }
  for (int p = gtid<kT>(); p < D; p += kT) c.dl[c.ord[p]] = c.x[p];  // P^T y
  gsync<kT>();
}

// gauss_newton (local_opt.cpp:20-82) on one block. Returns false if the start
// is infeasible / non-finite (the reference throws).
// Model FLOPs per event (sincos, div, sqrt count 1), by block size:
// GN trial: LDLT D^3/3 + solves and M fill ~2.5 D^2 + residuals/objective
// ~260 per observation; GN Jacobian + g + H_ii ~400 per observation + 4 D;
// L-BFGS value ~100/obs + 10 D, gradient ~350/obs + 4 D, direction 4 h D + 8 D,
// accepted pair ~12 D.
__device__ __forceinline__ unsigned long long fl_trial(const Blk& k) {
  const unsigned long long D = (unsigned long long)k.D;
  return D * D * D / 3 + 5 * D * D / 2 + 260ull * k.nobs;
}

template <int kT, bool kSharedM>
__device__ __forceinline__ bool block_gn(const DevState& S, const Blk& k, const Carve& c, double* M,
                                         unsigned long long cnt[6]) {
  const int D = k.D;
  if (gtid<kT>() < 8) c.flag[gtid<kT>()] = 0;
  gsync<kT>();
  residuals<kT>(S, k, c, c.v, c.r);
  gsync<kT>();
  if (gtid<kT>() == 0) {
    const bool ok = c.flag[0] == 0 && weight_rows_finite(k, c, c.v);
    c.flag[2] = ok ? 0 : 1;
    if (ok) c.red[0] = objective_rows(k, c, c.r, c.v);
  }
  gsync<kT>();
  if (c.flag[2]) return false;
  for (int it = 0; it < S.inner_max_iters; ++it) {
    jacobians<kT>(S, k, c, c.v);
    gsync<kT>();
    if (c.flag[1]) return true;  // kSingular: x unchanged
    if (gtid<kT>() == 0) {
      ++cnt[0];
      cnt[5] += 400ull * k.nobs + 4ull * D;
    }
    // g = 2 J^T r, rows in order; H_ii
    for (int i = gtid<kT>(); i < D; i += kT) {
      bool pt;
      int idx, co;
      var_of(k, i, pt, idx, co);
      const int a = jcol(pt, co);
      const Span sp = obs_of(c, pt, idx);
      double s = 0.0, h = 0.0;
      for (int n = sp.lo; n < sp.hi; ++n) {
        const int o = sp.at(n);
        const double* A = c.A + 18 * o;
        s += (-A[a]) * c.r[2 * o];
        s += (-A[9 + a]) * c.r[2 * o + 1];
        h += A[a] * A[a];
        h += A[9 + a] * A[9 + a];
      }
      const double w = pt ? k.wx : k.wy;
      s += w * (w * (c.v[i] - c.tgt[i]));
      h += w * w;
      c.g[i] = 2.0 * s;
      c.hdg[i] = h;
    }
    gsync<kT>();
    if (gtid<kT>() == 0) c.flag[3] = sqrt(seq_dot(c.g, c.g, D)) <= S.grad_tol;
    gsync<kT>();
    if (c.flag[3]) return true;  // kGradConverged
    for (int i = gtid<kT>(); i < D; i += kT) c.g[i] = -0.5 * c.g[i];  // rhs
    double lambda = 0.0;
    bool next = false;
    while (!next) {
      for (int i = gtid<kT>(); i < D; i += kT) {
        const double h = c.hdg[i];
        const double damp = h < 1e-12 ? 1e-12 : h;  // std::max(H_ii, 1e-12)
        c.hd[i] = lambda > 0.0 ? h + lambda * damp : h;
      }
      gsync<kT>();
      ldlt_solve<kT, kSharedM>(k, c, kSharedM ? c.M : M);
      if (gtid<kT>() < 8) c.flag[gtid<kT>()] = 0;
      gsync<kT>();
      for (int i = gtid<kT>(); i < D; i += kT) {
        if (!isfinite(c.dl[i])) c.flag[4] = 1;
        c.vt[i] = c.v[i] + c.dl[i];
      }
      gsync<kT>();
      bool accepted = false;
      if (gtid<kT>() == 0) cnt[5] += fl_trial(k);
      if (!c.flag[4]) {
        if (gtid<kT>() == 0) ++cnt[1];
        residuals<kT>(S, k, c, c.vt, c.rt);
        gsync<kT>();
        if (gtid<kT>() == 0) {
          c.flag[5] = 0;
          if (c.flag[0] == 0 && weight_rows_finite(k, c, c.vt)) {
            const double objt = objective_rows(k, c, c.rt, c.vt);
            if (objt <= c.red[0]) {  // non-strict accept (local_opt.cpp:60)
              c.red[0] = objt;
              c.flag[5] = 1;
            }
          }
        }
        gsync<kT>();
        accepted = c.flag[5] != 0;
      }
      if (accepted) {
        for (int i = gtid<kT>(); i < D; i += kT) c.v[i] = c.vt[i];
        for (int n = gtid<kT>(); n < 2 * k.nobs; n += kT) c.r[n] = c.rt[n];
        gsync<kT>();
        if (gtid<kT>() == 0) {
          ++cnt[2];
          c.flag[6] = sqrt(seq_dot(c.dl, c.dl, D)) <= S.step_tol * (1.0 + sqrt(seq_dot(c.v, c.v, D)));
        }
        gsync<kT>();
        if (c.flag[6]) return true;  // kStepConverged
        next = true;
      } else {
        lambda = lambda == 0.0 ? kDampingInit : lambda * 10.0;
        if (lambda > kDampingMax) return true;
      }
    }
  }
  return true;
}

// ---- Huber: lbfgs (local_opt.cpp:84-186) with value_fn / grad_fn of
// admm_solver.cpp:231-282 (explicit dual-linear form).
__device__ __forceinline__ double huber_value(double e0, double e1, double delta) {
  const double a = sqrt(e0 * e0 + e1 * e1);  // losses.cpp:7-20
  return a <= delta ? 0.5 * a * a : delta * (a - 0.5 * delta);
}

// value at V into *out (thread 0); flag[0] set if infeasible. Residuals in rr.
template <int kT>
__device__ __forceinline__ void h_value(const DevState& S, const Blk& k, const Carve& c, const double* V,
                        double* rr, double* out) {
  residuals<kT>(S, k, c, V, rr);
  gsync<kT>();
  if (gtid<kT>() == 0 && c.flag[0] == 0) {
    double total = 0.0;
    for (int o = 0; o < k.nobs; ++o) total += huber_value(rr[2 * o], rr[2 * o + 1], S.huber_delta);
    for (int q = 0; q < k.np; ++q) {
      double d[3], dd = 0.0;
      for (int m = 0; m < 3; ++m) d[m] = V[3 * q + m] - c.piv[3 * q + m];  // piv: consensus
      for (int m = 0; m < 3; ++m) dd += c.hd[3 * q + m] * d[m];          // hd: duals
      total += dd + 0.5 * S.rho_x * exact::sqn(d, 3);
    }
    for (int q = 0; q < k.nc; ++q) {
      double d[6], dd = 0.0;
      const int o = k.cb + 6 * q;
      for (int m = 0; m < 6; ++m) d[m] = V[o + m] - c.piv[o + m];
      for (int m = 0; m < 6; ++m) dd += c.hd[o + m] * d[m];
      total += dd + 0.5 * S.rho_y * exact::sqn(d, 6);
    }
    *out = total;
  }
  gsync<kT>();
}

// gradient at V into G (flag[1] set if infeasible).
template <int kT>
__device__ __forceinline__ void h_grad(const DevState& S, const Blk& k, const Carve& c, const double* V, double* G) {
  for (int o = gtid<kT>(); o < k.nobs; o += kT) {
    exact::ETrig t;
    double R[9], w[3], z[2], v9[9];
    if (!gproject(S, k, c, V, o, t, R, w, z, v9)) {
      c.flag[1] = 1;
      continue;
    }
    exact::erot(t, R);
    double A0[9], A1[9];
    exact::ejac(v9, t, R, w, c.fcam[c.ocl[o]], A0, A1);
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      c.A[18 * o + m] = A0[m];
      c.A[18 * o + 9 + m] = A1[m];
    }
    const double e0 = c.uv[2 * o] - z[0], e1 = c.uv[2 * o + 1] - z[1];
    const double a = sqrt(e0 * e0 + e1 * e1);  // losses.cpp:22-38
    double l0, l1;
    if (a == 0.0) {
      l0 = l1 = 0.0;
    } else if (a <= S.huber_delta) {
      l0 = e0;
      l1 = e1;
    } else {
      const double s = S.huber_delta / a;
      l0 = s * e0;
      l1 = s * e1;
    }
    c.lg[2 * o] = l0;
    c.lg[2 * o + 1] = l1;
  }
  gsync<kT>();
  for (int i = gtid<kT>(); i < k.D; i += kT) {
    bool pt;
    int idx, co;
    var_of(k, i, pt, idx, co);
    const int a = jcol(pt, co);
    const Span sp = obs_of(c, pt, idx);
    double g = 0.0;
    for (int n = sp.lo; n < sp.hi; ++n) {
      const int o = sp.at(n);
      const double* A = c.A + 18 * o;
      g -= A[a] * c.lg[2 * o] + A[9 + a] * c.lg[2 * o + 1];
    }
    g += c.hd[i] + (pt ? S.rho_x : S.rho_y) * (V[i] - c.piv[i]);
    G[i] = g;
  }
  gsync<kT>();
}

template <int kT>
__device__ __forceinline__ bool block_lbfgs(const DevState& S, const Blk& k, const Carve& c,
                            unsigned long long cnt[6]) {
  const int D = k.D;
  const int mem = S.lbfgs_memory;
  if (gtid<kT>() < 8) c.flag[gtid<kT>()] = 0;
  gsync<kT>();
  h_value<kT>(S, k, c, c.v, c.r, &c.red[0]);
  h_grad<kT>(S, k, c, c.v, c.g);
  if (gtid<kT>() == 0) {
    unsigned ex = 0;  // exponent-field max: 0x7ff iff some component is inf / NaN
    for (int i = 0; i < D; ++i) ex = max(ex, (unsigned)__double2hiint(c.g[i]) & 0x7ff00000u);
    const bool ok = c.flag[0] == 0 && c.flag[1] == 0 && isfinite(c.red[0]) && ex != 0x7ff00000u;
    c.flag[2] = ok ? 0 : 1;
    ++cnt[0];
    cnt[5] += 450ull * k.nobs + 14ull * D;
  }
  gsync<kT>();
  if (c.flag[2]) return false;
  int h_first = 0, h_size = 0;  // ring buffer, oldest at h_first (uniform)
  double gamma = 1.0;
  for (int it = 0; it < S.inner_max_iters; ++it) {
    // q in c.x, direction d in c.dl; the two-loop recursion on thread 0
    if (gtid<kT>() == 0) {
      c.flag[3] = sqrt(seq_dot(c.g, c.g, D)) <= S.grad_tol;
      if (!c.flag[3]) {
        for (int i = 0; i < D; ++i) c.x[i] = c.g[i];
        for (int kk = h_size - 1; kk >= 0; --kk) {
          const int slot = (h_first + kk) % mem;
          const double* hs = c.hs + (size_t)slot * D;
          const double* hy = c.hy + (size_t)slot * D;
          c.alpha[kk] = c.hrho[slot] * seq_dot(hs, c.x, D);
          for (int i = 0; i < D; ++i) c.x[i] -= c.alpha[kk] * hy[i];
        }
        for (int i = 0; i < D; ++i) c.x[i] *= gamma;
        for (int kk = 0; kk < h_size; ++kk) {
          const int slot = (h_first + kk) % mem;
          const double* hs = c.hs + (size_t)slot * D;
          const double* hy = c.hy + (size_t)slot * D;
          const double beta = c.hrho[slot] * seq_dot(hy, c.x, D);
          for (int i = 0; i < D; ++i) c.x[i] += (c.alpha[kk] - beta) * hs[i];
        }
        ++cnt[3];
        cnt[4] += h_size;
        cnt[5] += (4ull * h_size + 8ull) * D;
        for (int i = 0; i < D; ++i) c.dl[i] = -c.x[i];
        double slope = seq_dot(c.g, c.dl, D);
        c.flag[4] = 0;
        if (!(slope < 0.0)) {
          c.flag[4] = 1;  // clear the history
          for (int i = 0; i < D; ++i) c.dl[i] = -c.g[i];
          slope = -seq_dot(c.g, c.g, D);
        }
        c.red[1] = slope;
      }
    }
    gsync<kT>();
    if (c.flag[3]) return true;  // kGradConverged
    if (c.flag[4]) {
      h_size = 0;
      h_first = 0;
    }
    // Armijo backtracking (local_opt.cpp:130-147)
    double step = 1.0;
    bool accepted = false;
    for (int ls = 0; ls < S.max_line_search; ++ls) {
      for (int i = gtid<kT>(); i < D; i += kT) c.vt[i] = c.v[i] + step * c.dl[i];
      if (gtid<kT>() == 0) {
        c.flag[0] = 0;
        ++cnt[1];
        cnt[5] += 100ull * k.nobs + 10ull * D;
      }
      gsync<kT>();
      h_value<kT>(S, k, c, c.vt, c.rt, &c.red[2]);
      const bool ok = c.flag[0] == 0 && isfinite(c.red[2]) &&
                      c.red[2] <= c.red[0] + S.armijo_c * step * c.red[1];
      gsync<kT>();
      if (ok) {
        accepted = true;
        break;
      }
      step *= S.backtrack;
    }
    if (!accepted) return true;  // kLineSearchFailed, best iterate kept
    if (gtid<kT>() == 0) c.flag[1] = 0;
    gsync<kT>();
    h_grad<kT>(S, k, c, c.vt, c.hdg);  // g_new in hdg
    if (gtid<kT>() == 0) {
      unsigned ex = 0;
      for (int i = 0; i < D; ++i) ex = max(ex, (unsigned)__double2hiint(c.hdg[i]) & 0x7ff00000u);
      const bool fin = c.flag[1] == 0 && ex != 0x7ff00000u;
      c.flag[5] = fin;
      if (fin) {
        ++cnt[0];
        ++cnt[2];
        cnt[5] += 350ull * k.nobs + 16ull * D;
        // s = trial - x (in c.x), y = g_new - g (in c.dl)
        for (int i = 0; i < D; ++i) {
          c.x[i] = c.vt[i] - c.v[i];
          c.dl[i] = c.hdg[i] - c.g[i];
        }
        const double sBs = seq_dot(c.x, c.x, D) / gamma;  // Powell damping (:155-165)
        double sy = seq_dot(c.x, c.dl, D);
        if (sy < 0.2 * sBs) {
          const double theta = 0.8 * sBs / (sBs - sy);
          for (int i = 0; i < D; ++i) c.dl[i] = theta * c.dl[i] + (1.0 - theta) / gamma * c.x[i];
          sy = seq_dot(c.x, c.dl, D);
        }
        const double sn = sqrt(seq_dot(c.x, c.x, D));
        c.flag[6] = 0;
        if (sy > 1e-12 * sn * sqrt(seq_dot(c.dl, c.dl, D))) {
          int slot;
          if (h_size < mem) {
            slot = (h_first + h_size) % mem;
          } else {
            slot = h_first;  // overwrite the oldest == push + pop_front
          }
          double* hs = c.hs + (size_t)slot * D;
          double* hy = c.hy + (size_t)slot * D;
          for (int i = 0; i < D; ++i) {
            hs[i] = c.x[i];
            hy[i] = c.dl[i];
          }
          c.hrho[slot] = 1.0 / sy;
          gamma = sy / seq_dot(c.dl, c.dl, D);
          c.flag[6] = 1;
        }
        c.red[3] = gamma;
        for (int i = 0; i < D; ++i) {
          c.v[i] = c.vt[i];
          c.g[i] = c.hdg[i];
        }
        c.red[0] = c.red[2];
        c.flag[7] = sn <= S.step_tol * (1.0 + sqrt(seq_dot(c.v, c.v, D)));
      }
    }
    gsync<kT>();
    if (!c.flag[5]) return true;  // kLineSearchFailed
    gamma = c.red[3];
    if (c.flag[6]) {
      if (h_size < mem) {
        ++h_size;
      } else {
        h_first = (h_first + 1) % mem;
      }
    }
    if (c.flag[7]) return true;  // kStepConverged
    gsync<kT>();
  }
  return true;  // kMaxIters
}

// ---- K1G: persistent CTAs, one block at a time ----------------------------
#ifndef DBAG_GEN_MINB
#define DBAG_GEN_MINB 4  // 128 registers: 4 CTAs per SM when shared memory allows
#endif
// kT threads per block: 128 (one block per CTA) or 32 (four per CTA, one per
// warp, each with its own shared slice of group_bytes).
template <int kT>
__global__ void __launch_bounds__(kGenThreads, DBAG_GEN_MINB) k_local_blocks(
    DevState S, GenState G, int64_t begin, int64_t count, size_t group_bytes) {
  constexpr int kGroups = kGenThreads / kT;
  extern __shared__ __align__(16) char smem_raw[];
  const int grp = (int)threadIdx.x / kT;
  Carve c;
  carve(smem_raw + (size_t)grp * group_bytes, G.max_dim, G.max_np, G.max_nc, G.max_nobs,
        S.loss == DBAG_LOSS_HUBER ? S.lbfgs_memory : 0, G.m_in_smem != 0, &c);
  double* M = G.m_in_smem ? nullptr
                          : G.mscratch + ((size_t)blockIdx.x * kGroups + grp) * tri(G.max_dim, 0);
  __shared__ int64_t next[kGroups];
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  for (;;) {
    if (gtid<kT>() == 0) next[grp] = (int64_t)atomicAdd(G.work, 1ull);
    gsync<kT>();
    const int64_t idx = next[grp];
    gsync<kT>();
    if (idx >= count) break;
    Blk k;
    k.b = begin + idx;
    k.o0 = G.obs_off[k.b];
    k.p0 = G.pc_off[k.b];
    k.c0 = G.cc_off[k.b];
    k.nobs = (int)(G.obs_off[k.b + 1] - k.o0);
    k.np = (int)(G.pc_off[k.b + 1] - k.p0);
    k.nc = (int)(G.cc_off[k.b + 1] - k.c0);
    k.cb = 3 * k.np;
    k.D = 3 * k.np + 6 * k.nc;
    k.wx = sqrt(0.5 * S.rho_x);  // admm_solver.cpp:183-184
    k.wy = sqrt(0.5 * S.rho_y);
    const bool huber = S.loss == DBAG_LOSS_HUBER;
    // load: copies, targets (x̄ - r/ρ: admm_solver.cpp:155-162) or, for Huber,
    // consensus (piv) and duals (hd); focal lengths; observations
    for (int i = gtid<kT>(); i < k.D; i += kT) {
      double xb, du, rho;
      if (i < k.cb) {
        const int q = i / 3, m = i - 3 * q;
        const int64_t slot = k.p0 + q;
        const double4 x4 = S.xbar[G.pt_ids[slot]];
        xb = m == 0 ? x4.x : (m == 1 ? x4.y : x4.z);
        du = G.gr[(int64_t)m * G.PC + slot];
        c.v[i] = G.gx[(int64_t)m * G.PC + slot];
        rho = S.rho_x;
      } else {
        const int q = (i - k.cb) / 6, m = i - k.cb - 6 * q;
        const int64_t slot = k.c0 + q;
        xb = S.ybar[8 * (int64_t)G.cam_ids[slot] + m];
        du = G.gs[(int64_t)m * G.CC + slot];
        c.v[i] = G.gy[(int64_t)m * G.CC + slot];
        rho = S.rho_y;
      }
      if (huber) {
        c.piv[i] = xb;
        c.hd[i] = du;
      } else {
        c.tgt[i] = xb - du / rho;
      }
    }
    for (int q = gtid<kT>(); q < k.nc; q += kT)
      c.fcam[q] = S.ybar[8 * (int64_t)G.cam_ids[k.c0 + q] + 6];
    for (int o = gtid<kT>(); o < k.nobs; o += kT) {
      const int64_t s = k.o0 + o;
      const PointRec& rec = S.prec[S.blk_pos[s]];
      c.uv[2 * o] = rec.u;
      c.uv[2 * o + 1] = rec.v;
      c.opl[o] = G.obs_pl[s];
      c.ocl[o] = G.obs_cl[s];
    }
    gsync<kT>();
    if (gtid<kT>() == 0) {  // observation lists per local point / camera
      for (int q = 0; q <= k.np; ++q) c.pto_off[q] = 0;
      for (int q = 0; q <= k.nc; ++q) c.cmo_off[q] = 0;
      for (int o = 0; o < k.nobs; ++o) {
        ++c.pto_off[c.opl[o] + 1];
        ++c.cmo_off[c.ocl[o] + 1];
      }
      for (int q = 0; q < k.np; ++q) c.pto_off[q + 1] += c.pto_off[q];
      for (int q = 0; q < k.nc; ++q) c.cmo_off[q + 1] += c.cmo_off[q];
      for (int e = 0; e < k.np * k.nc; ++e) c.pco[e] = -1;
      for (int o = 0; o < k.nobs; ++o) c.pco[c.opl[o] * k.nc + c.ocl[o]] = o;
    }
    gsync<kT>();
    if (gtid<kT>() == 0) {  // counting-sort fill of the point lists (ascending o)
      for (int q = 0; q < k.np; ++q) c.ord[q] = c.pto_off[q];
      for (int o = 0; o < k.nobs; ++o) c.pto[c.ord[c.opl[o]]++] = o;
    }
    gsync<kT>();
    // M in shared memory: the instantiation that reads c.M directly, so every
    // access compiles to LDS/STS (a shared-or-global pointer forces generic LD).
    const bool ok = huber ? block_lbfgs<kT>(S, k, c, cnt)
                          : (G.m_in_smem ? block_gn<kT, true>(S, k, c, nullptr, cnt)
                                         : block_gn<kT, false>(S, k, c, M, cnt));
    gsync<kT>();
    if (!ok) {
      if (gtid<kT>() == 0)
        atomicMin(reinterpret_cast<unsigned long long*>(S.err_block), (unsigned long long)k.b);
    } else {  // write back (admm_solver.cpp:284-289)
      for (int i = gtid<kT>(); i < k.D; i += kT) {
        if (i < k.cb) {
          const int q = i / 3, m = i - 3 * q;
          G.gx[(int64_t)m * G.PC + k.p0 + q] = c.v[i];
        } else {
          const int q = (i - k.cb) / 6, m = i - k.cb - 6 * q;
          G.gy[(int64_t)m * G.CC + k.c0 + q] = c.v[i];
        }
      }
    }
    gsync<kT>();
  }
  if (gtid<kT>() == 0) {
    unsigned long long* slot = S.counters + 8 * ((blockIdx.x * kGroups + grp) % kCounterStripes);
    for (int m = 0; m < 6; ++m)
      if (cnt[m]) atomicAdd(slot + m, cnt[m]);
  }
}

// ---- camera consensus / dual over copies (admm_solver.cpp:333-355) --------
constexpr int kGCamThreads = 128;
__global__ void __launch_bounds__(kGCamThreads) k_gen_cameras(DevState S, GenState G, int mode) {
  if (__syncthreads_or(threadIdx.x == 0 && S.gate && *S.gate >= 0)) return;  // local solve raised
  __shared__ double ybs[6];
  __shared__ double red[kGCamThreads / 32];
  const int j = blockIdx.x;
  const int64_t beg = G.camc_off[j], end = G.camc_off[j + 1];
  double dual_res = 0.0;
  if (mode & 1) {
    if (threadIdx.x < 6) {  // lane k: component k, sequential in block order
      const int m = threadIdx.x;
      const double inv_rho = 1.0 / S.rho_y;
      const double anchor = G.gy[(int64_t)m * G.CC + beg];
      double acc = 0.0;
      for (int64_t s = beg; s < end; ++s)
        acc += (G.gy[(int64_t)m * G.CC + s] - anchor) + inv_rho * G.gs[(int64_t)m * G.CC + s];
      ybs[m] = anchor + acc / (double)(end - beg);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double* yo = S.ybar + 8 * (int64_t)j;
      double d2 = 0.0;
      for (int m = 0; m < 6; ++m) {
        const double d = ybs[m] - yo[m];
        d2 += d * d;
      }
      dual_res = S.rho_y * sqrt(d2);
      for (int m = 0; m < 6; ++m) yo[m] = ybs[m];
      exact::ETrig t;
      exact::etrig(ybs[0], ybs[1], ybs[2], t);
      double R[9];
      exact::erot(t, R);
      double* o = S.camR + 16 * (int64_t)j;
      for (int m = 0; m < 9; ++m) o[m] = R[m];
      o[9] = ybs[3];
      o[10] = ybs[4];
      o[11] = ybs[5];
      o[12] = yo[6];
    }
  } else if (threadIdx.x < 6) {
    ybs[threadIdx.x] = S.ybar[8 * (int64_t)j + threadIdx.x];
  }
  __syncthreads();
  if (mode & 2) {
    double worst = 0.0;
    for (int64_t s = beg + threadIdx.x; s < end; s += kGCamThreads) {
      double d[6];
      for (int m = 0; m < 6; ++m) {
        d[m] = G.gy[(int64_t)m * G.CC + s] - ybs[m];
        G.gs[(int64_t)m * G.CC + s] += S.rho_y * d[m];  // admm_solver.cpp:351-355
      }
      worst = fmax(worst, sqrt(exact::sqn(d, 6)));
    }
    worst = warp_max(worst);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = red[0];
      for (int w = 1; w < kGCamThreads / 32; ++w) m = fmax(m, red[w]);
      S.cam_stats[2 * j] = m;
    }
  }
  if (threadIdx.x == 0) S.cam_stats[2 * j + 1] = dual_res;
}

// ---- point consensus / dual over copies + the metric over observations ----
constexpr int kGPtThreads = 256;
__global__ void __launch_bounds__(kGPtThreads) k_gen_points(DevState S, GenState G, int mode,
                                                            int metric) {
  if (__syncthreads_or(threadIdx.x == 0 && S.gate && *S.gate >= 0)) return;  // local solve raised
  __shared__ double smem[(kGPtThreads / 32) * 2];
  const int64_t tix = (int64_t)blockIdx.x * kGPtThreads + threadIdx.x;
  double err_sum = 0.0, worst = 0.0, dual_res = 0.0, infeasible = 0.0;
  if (tix < S.N) {
    const int i = S.pt_order[tix];
    const int64_t c0 = G.ptc_off[i], c1 = G.ptc_off[i + 1];
    double xb[3];
    if (mode & 1) {
      const double inv_rho = 1.0 / S.rho_x;
      double anc[3], acc[3] = {0.0, 0.0, 0.0};
      const int64_t a = G.ptc_slot[c0];
      for (int m = 0; m < 3; ++m) anc[m] = G.gx[(int64_t)m * G.PC + a];
      for (int64_t n = c0; n < c1; ++n) {
        const int64_t s = G.ptc_slot[n];
        for (int m = 0; m < 3; ++m)
          acc[m] += (G.gx[(int64_t)m * G.PC + s] - anc[m]) + inv_rho * G.gr[(int64_t)m * G.PC + s];
      }
      const double4 old = S.xbar[i];
      for (int m = 0; m < 3; ++m) xb[m] = anc[m] + acc[m] / (double)(c1 - c0);
      const double d0 = xb[0] - old.x, d1 = xb[1] - old.y, d2 = xb[2] - old.z;
      dual_res = S.rho_x * sqrt(d0 * d0 + d1 * d1 + d2 * d2);
      S.xbar[i] = make_double4(xb[0], xb[1], xb[2], 0.0);
    } else {
      const double4 o = S.xbar[i];
      xb[0] = o.x;
      xb[1] = o.y;
      xb[2] = o.z;
    }
    if (mode & 2) {
      for (int64_t n = c0; n < c1; ++n) {
        const int64_t s = G.ptc_slot[n];
        double d[3];
        for (int m = 0; m < 3; ++m) {
          d[m] = G.gx[(int64_t)m * G.PC + s] - xb[m];
          G.gr[(int64_t)m * G.PC + s] += S.rho_x * d[m];
        }
        worst = fmax(worst, sqrt(exact::sqn(d, 3)));
      }
    }
    if (metric) {  // every observation of the point at (x̄, ȳ) (problem.cpp:109-138)
      for (int64_t p = S.pt_off[i]; p < S.pt_off[i + 1]; ++p) {
        const PointRec& r = S.prec[p];
        const double* c = S.camR + 16 * (int64_t)S.pm_cam[p];
        const double w2 = exact::row3(c + 6, xb) + c[11];
        if (!(w2 >= S.eps_depth)) {
          infeasible = 1.0;
        } else {
          const double w0 = exact::row3(c, xb) + c[9], w1 = exact::row3(c + 3, xb) + c[10];
          const double e0 = r.u - c[12] * w0 / w2, e1 = r.v - c[12] * w1 / w2;
          err_sum += sqrt(e0 * e0 + e1 * e1);
        }
      }
    }
  }
  double sums[1] = {err_sum};
  block_sum<kGPtThreads, 1>(sums, smem);
  const double mx = block_max<kGPtThreads>(worst, smem);
  const double md = block_max<kGPtThreads>(dual_res, smem);
  const double inf = block_max<kGPtThreads>(infeasible, smem);
  if (threadIdx.x == 0) {
    double* o = S.part_pt + 4 * (int64_t)blockIdx.x;
    o[0] = sums[0];
    o[1] = mx;
    o[2] = md;
    o[3] = inf;
  }
}

__global__ void k_gen_init_copies(DevState S, GenState G) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < G.PC) {
    const double4 x = S.xbar[G.pt_ids[t]];
    G.gx[t] = x.x;
    G.gx[G.PC + t] = x.y;
    G.gx[2 * G.PC + t] = x.z;
    for (int m = 0; m < 3; ++m) G.gr[(int64_t)m * G.PC + t] = 0.0;
  }
  if (t < G.CC) {
    const double* y = S.ybar + 8 * (int64_t)G.cam_ids[t];
    for (int m = 0; m < 6; ++m) {
      G.gy[(int64_t)m * G.CC + t] = y[m];
      G.gs[(int64_t)m * G.CC + t] = 0.0;
    }
  }
}

// dual sums per point / camera in copy order (admm_solver.cpp:385-399)
__global__ void k_gen_dual_sums(DevState S, GenState G, double* pts, double* cams) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < S.N) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int64_t n = G.ptc_off[t]; n < G.ptc_off[t + 1]; ++n)
      for (int m = 0; m < 3; ++m) s[m] += G.gr[(int64_t)m * G.PC + G.ptc_slot[n]];
    for (int m = 0; m < 3; ++m) pts[3 * t + m] = s[m];
  }
  if (t < S.M) {
    double s[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t n = G.camc_off[t]; n < G.camc_off[t + 1]; ++n)
      for (int m = 0; m < 6; ++m) s[m] += G.gs[(int64_t)m * G.CC + n];
    for (int m = 0; m < 6; ++m) cams[6 * t + m] = s[m];
  }
}

// block_objective (admm_solver.cpp:401-426), one thread, explicit form.
__global__ void k_gen_block_objective(DevState S, GenState G, int64_t b, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t o0 = G.obs_off[b], o1 = G.obs_off[b + 1];
  const int64_t p0 = G.pc_off[b], c0 = G.cc_off[b];
  const int np = (int)(G.pc_off[b + 1] - p0), nc = (int)(G.cc_off[b + 1] - c0);
  double total = 0.0;
  for (int64_t s = o0; s < o1; ++s) {
    const int q = G.obs_pl[s], cq = G.obs_cl[s];
    double v9[9];
    for (int m = 0; m < 3; ++m) v9[m] = G.gx[(int64_t)m * G.PC + p0 + q];
    for (int m = 0; m < 6; ++m) v9[3 + m] = G.gy[(int64_t)m * G.CC + c0 + cq];
    const double f = S.ybar[8 * (int64_t)G.cam_ids[c0 + cq] + 6];
    exact::ETrig t;
    double R[9], w[3], z[2];
    if (!exact::eproject(v9, f, S.eps_depth, t, R, w, z)) {
      *out = INFINITY;
      return;
    }
    const PointRec& rec = S.prec[S.blk_pos[s]];
    const double e0 = rec.u - z[0], e1 = rec.v - z[1];
    total += S.loss == DBAG_LOSS_HUBER ? huber_value(e0, e1, S.huber_delta) : e0 * e0 + e1 * e1;
  }
  for (int q = 0; q < np; ++q) {
    const double4 x4 = S.xbar[G.pt_ids[p0 + q]];
    const double xb[3] = {x4.x, x4.y, x4.z};
    double d[3], dd = 0.0;
    for (int m = 0; m < 3; ++m) d[m] = G.gx[(int64_t)m * G.PC + p0 + q] - xb[m];
    for (int m = 0; m < 3; ++m) dd += G.gr[(int64_t)m * G.PC + p0 + q] * d[m];
    total += dd + 0.5 * S.rho_x * exact::sqn(d, 3);
  }
  for (int q = 0; q < nc; ++q) {
    const double* yb = S.ybar + 8 * (int64_t)G.cam_ids[c0 + q];
    double d[6], dd = 0.0;
    for (int m = 0; m < 6; ++m) d[m] = G.gy[(int64_t)m * G.CC + c0 + q] - yb[m];
    for (int m = 0; m < 6; ++m) dd += G.gs[(int64_t)m * G.CC + c0 + q] * d[m];
    total += dd + 0.5 * S.rho_y * exact::sqn(d, 6);
  }
  *out = total;
}

// max primal residuals over copies (admm_solver.cpp:359-383); out[0..1] must
// be zeroed; max of non-negative doubles via their ordered bit patterns.
__global__ void k_gen_max_primal(DevState S, GenState G, double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double px = 0.0, py = 0.0;
  if (t < G.PC) {
    const double4 x4 = S.xbar[G.pt_ids[t]];
    const double xb[3] = {x4.x, x4.y, x4.z};
    double d[3];
    for (int m = 0; m < 3; ++m) d[m] = G.gx[(int64_t)m * G.PC + t] - xb[m];
    px = sqrt(exact::sqn(d, 3));
  }
  if (t < G.CC) {
    const double* yb = S.ybar + 8 * (int64_t)G.cam_ids[t];
    double d[6];
    for (int m = 0; m < 6; ++m) d[m] = G.gy[(int64_t)m * G.CC + t] - yb[m];
    py = sqrt(exact::sqn(d, 6));
  }
  px = warp_max(px);
  py = warp_max(py);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(px));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1),
              (unsigned long long)__double_as_longlong(py));
  }
}

// ---------------------------------------------------------------------------
// host: GenSolver
// ---------------------------------------------------------------------------
namespace {
inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
template <typename T>
cudaError_t dalloc(std::vector<void*>& pool, T** p, size_t n) {
  void* q = nullptr;
  const cudaError_t e = cudaMalloc(&q, sizeof(T) * (n ? n : 1));
  if (e != cudaSuccess) return e;
  pool.push_back(q);
  *p = static_cast<T*>(q);
  return cudaSuccess;
}
template <typename T>
cudaError_t upload(std::vector<void*>& pool, T** p, const std::vector<T>& v, cudaStream_t st) {
  cudaError_t e = dalloc(pool, p, v.size());
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  e = cudaMemcpyAsync(*p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);  // v may be a temporary
}
#define GK(x)                              \
  do {                                     \
    const cudaError_t e_ = (x);            \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)
}  // namespace

GenSolver::~GenSolver() {
  cudaSetDevice(device);
  for (void* p : pool) cudaFree(p);
}

cudaError_t GenSolver::init(const DevState& S, int32_t ppb, int32_t cpb, int dev, cudaStream_t st) {
  device = dev;
  const int64_t L = S.L;
  std::vector<int32_t> cam(L), pt(L);
  GK(cudaMemcpyAsync(cam.data(), S.blk_cam, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, st));
  GK(cudaMemcpyAsync(pt.data(), S.blk_pt, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, st));
  GK(cudaStreamSynchronize(st));
  part = partition_sorted(L, cam.data(), pt.data(), ppb, cpb);
  comm_floats = communication_cost(part, S.M, S.N);
  const int64_t B = part.blocks(), PC = (int64_t)part.pt_ids.size(),
                CC = (int64_t)part.cam_ids.size();
  // point -> copy slots (block order), camera -> contiguous slots
  std::vector<int64_t> ptc_off(S.N + 1, 0), ptc_slot(PC), camc_off(S.M + 1, 0);
  for (int64_t s = 0; s < PC; ++s) ++ptc_off[part.pt_ids[s] + 1];
  for (int32_t i = 0; i < S.N; ++i) ptc_off[i + 1] += ptc_off[i];
  {
    std::vector<int64_t> fill(ptc_off.begin(), ptc_off.end() - 1);
    for (int64_t s = 0; s < PC; ++s) ptc_slot[fill[part.pt_ids[s]]++] = s;
  }
  for (int64_t s = 0; s < CC; ++s) ++camc_off[part.cam_ids[s] + 1];
  for (int32_t j = 0; j < S.M; ++j) camc_off[j + 1] += camc_off[j];
  for (int64_t s = 1; s < CC; ++s)  // a camera's copies are adjacent slots
    if (part.cam_ids[s] < part.cam_ids[s - 1] ||
        (part.cam_ids[s] != part.cam_ids[s - 1] && camc_off[part.cam_ids[s]] != s))
      return cudaErrorInvalidValue;
  G.B = B;
  G.PC = PC;
  G.CC = CC;
  G.L = L;
  int64_t *obs_off, *pc_off, *cc_off, *d_ptc_off, *d_ptc_slot, *d_camc_off;
  int32_t *pt_ids, *cam_ids, *obs_pl, *obs_cl;
  GK(upload(pool, &obs_off, part.obs_off, st));
  GK(upload(pool, &pc_off, part.pt_off, st));
  GK(upload(pool, &cc_off, part.cam_off, st));
  GK(upload(pool, &pt_ids, part.pt_ids, st));
  GK(upload(pool, &cam_ids, part.cam_ids, st));
  GK(upload(pool, &obs_pl, part.obs_pl, st));
  GK(upload(pool, &obs_cl, part.obs_cl, st));
  GK(upload(pool, &d_ptc_off, ptc_off, st));
  GK(upload(pool, &d_ptc_slot, ptc_slot, st));
  GK(upload(pool, &d_camc_off, camc_off, st));
  G.obs_off = obs_off;
  G.pc_off = pc_off;
  G.cc_off = cc_off;
  G.pt_ids = pt_ids;
  G.cam_ids = cam_ids;
  G.obs_pl = obs_pl;
  G.obs_cl = obs_cl;
  G.ptc_off = d_ptc_off;
  G.ptc_slot = d_ptc_slot;
  G.camc_off = d_camc_off;
  GK(dalloc(pool, &G.gx, 3 * (size_t)PC));
  GK(dalloc(pool, &G.gr, 3 * (size_t)PC));
  GK(dalloc(pool, &G.gy, 6 * (size_t)CC));
  GK(dalloc(pool, &G.gs, 6 * (size_t)CC));
  GK(dalloc(pool, &G.work, 1));
  G.max_np = part.max_np;
  G.max_nc = part.max_nc;
  G.max_nobs = part.max_nobs;
  G.max_dim = 3 * part.max_np + 6 * part.max_nc;
  // shared memory: everything, plus the LDLT matrix if it fits
  const int mem = S.loss == DBAG_LOSS_HUBER ? S.lbfgs_memory : 0;
  int max_optin = 0;
  GK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t with_m = carve(nullptr, G.max_dim, G.max_np, G.max_nc, G.max_nobs, mem, true, nullptr);
  const size_t without_m =
      carve(nullptr, G.max_dim, G.max_np, G.max_nc, G.max_nobs, mem, false, nullptr);
  G.m_in_smem = (mem == 0 && with_m <= (size_t)max_optin) ? 1 : 0;
  group_bytes = G.m_in_smem ? with_m : without_m;
  // small blocks: a warp per block (its parallel phases are no wider than ~D)
  warp_groups = G.max_dim <= kWarpBlockMaxDim && 4 * group_bytes <= (size_t)max_optin;
  const int groups = warp_groups ? kGenThreads / 32 : 1;
  smem_bytes = group_bytes * groups;
  if (smem_bytes > (size_t)max_optin) return cudaErrorInvalidConfiguration;
  int per_sm = 0, sms = 0;
  if (warp_groups) {
    GK(cudaFuncSetAttribute(k_local_blocks<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem_bytes));
    GK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_local_blocks<32>, kGenThreads,
                                                     smem_bytes));
  } else {
    GK(cudaFuncSetAttribute(k_local_blocks<kGenThreads>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
    GK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_local_blocks<kGenThreads>,
                                                     kGenThreads, smem_bytes));
  }
  GK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  resident = std::max(1, per_sm) * sms;
  if (!G.m_in_smem && mem == 0)
    GK(dalloc(pool, &G.mscratch, (size_t)resident * groups * (size_t)tri(G.max_dim, 0)));
  return reset_copies(S, st);
}

cudaError_t GenSolver::reset_copies(const DevState& S, cudaStream_t st) {
  const int64_t n = std::max(G.PC, G.CC);
  k_gen_init_copies<<<grid_for(n, 256), 256, 0, st>>>(S, G);
  return cudaGetLastError();
}

cudaError_t GenSolver::local(const DevState& S, int64_t begin, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  GK(cudaMemsetAsync(G.work, 0, sizeof(unsigned long long), st));
  const int groups = warp_groups ? kGenThreads / 32 : 1;
  const int64_t grid = std::min<int64_t>((count + groups - 1) / groups, resident);
  if (warp_groups)
    k_local_blocks<32><<<(unsigned)grid, kGenThreads, smem_bytes, st>>>(S, G, begin, count,
                                                                       group_bytes);
  else
    k_local_blocks<kGenThreads><<<(unsigned)grid, kGenThreads, smem_bytes, st>>>(S, G, begin,
                                                                                 count, group_bytes);
  return cudaGetLastError();
}

cudaError_t GenSolver::cameras(const DevState& S, int mode, cudaStream_t st) {
  k_gen_cameras<<<S.M, kGCamThreads, 0, st>>>(S, G, mode);
  return cudaGetLastError();
}

cudaError_t GenSolver::points(const DevState& S, int mode, bool metric, int n_parts,
                              cudaStream_t st) {
  if ((int64_t)n_parts * kGPtThreads < S.N) return cudaErrorInvalidValue;
  k_gen_points<<<n_parts, kGPtThreads, 0, st>>>(S, G, mode, metric ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t GenSolver::copies_io(double* lp, double* lc, double* r, double* s, int dir,
                                 cudaStream_t st) {
  // host layout [PC][3] / [CC][6] (AdmmState per block, q order) <-> device SoA
  const int64_t PC = G.PC, CC = G.CC;
  std::vector<double> tp(3 * (size_t)PC), tc(6 * (size_t)CC);
  auto one = [&](double* host, double* dev, int64_t n, int w, std::vector<double>& t) -> cudaError_t {
    if (!host) return cudaSuccess;
    if (dir == 0) {
      GK(cudaMemcpyAsync(t.data(), dev, sizeof(double) * w * n, cudaMemcpyDeviceToHost, st));
      GK(cudaStreamSynchronize(st));
      for (int64_t x = 0; x < n; ++x)
        for (int m = 0; m < w; ++m) host[w * x + m] = t[(size_t)m * n + x];
    } else {
      for (int64_t x = 0; x < n; ++x)
        for (int m = 0; m < w; ++m) t[(size_t)m * n + x] = host[w * x + m];
      GK(cudaMemcpyAsync(dev, t.data(), sizeof(double) * w * n, cudaMemcpyHostToDevice, st));
      GK(cudaStreamSynchronize(st));
    }
    return cudaSuccess;
  };
  GK(one(lp, G.gx, PC, 3, tp));
  GK(one(lc, G.gy, CC, 6, tc));
  GK(one(r, G.gr, PC, 3, tp));
  GK(one(s, G.gs, CC, 6, tc));
  return cudaSuccess;
}

cudaError_t GenSolver::dual_sums(const DevState& S, double* pts, double* cams, cudaStream_t st) {
  const int64_t n = std::max<int64_t>(S.N, S.M);
  k_gen_dual_sums<<<grid_for(n, 256), 256, 0, st>>>(S, G, pts, cams);
  return cudaGetLastError();
}

cudaError_t GenSolver::block_objective(const DevState& S, int64_t b, double* d_out,
                                       cudaStream_t st) {
  k_gen_block_objective<<<1, 32, 0, st>>>(S, G, b, d_out);
  return cudaGetLastError();
}

cudaError_t GenSolver::max_primal(const DevState& S, double* d_out2, cudaStream_t st) {
  GK(cudaMemsetAsync(d_out2, 0, 2 * sizeof(double), st));
  const int64_t n = std::max(G.PC, G.CC);
  k_gen_max_primal<<<grid_for(n, 256), 256, 0, st>>>(S, G, d_out2);
  return cudaGetLastError();
}

}  // namespace blocks
}  // namespace dbag
