// dbag_exact_geom.cuh — the EXACT-numerics camera model shared by the (1,1)
// kernels (dbag_exact.cu) and the generalized-block kernels (dbag_blocks.cu).
// Include ONLY from translation units compiled with -fmad=false: every formula
// follows the oracle's operation order (oracle/oracle.cpp, geometry.cpp:9-159)
// and must not be contracted into FMAs.
#pragma once

#include "dbag_common.cuh"

namespace dbag {
namespace exact {

constexpr double kDampingInit = 1e-4;  // local_opt.cpp:13
constexpr double kDampingMax = 1e12;   // local_opt.cpp:14

// Same algorithm and constants as oracle.cpp det_sincos. With DBAG_SINCOS_CONST
// the constants sit in constant memory, so each DMUL / DADD takes them as a
// c[] operand instead of materializing them with uniform moves (same values,
// same operations, same bits).
__constant__ double kSinCosC[20] = {
    1.5707963267341256,     6.077100506303966e-11,   2.0222662487959506e-21, 0.6366197723675814,
    2.8114572543455206e-15, -7.647163731819816e-13,  1.6059043836821613e-10, -2.505210838544172e-08,
    2.7557319223985893e-06, -0.0001984126984126984,  0.008333333333333333,   -0.16666666666666666,
    -1.5619206968586225e-16, 4.779477332387385e-14,  -1.1470745597729725e-11, 2.08767569878681e-09,
    -2.755731922398589e-07, 2.48015873015873e-05,    -0.001388888888888889,  0.041666666666666664};
#define DBAG_SC(i, v) kSinCosC[i]
__device__ __forceinline__ void det_sincos(double x, double* sn, double* cs) {
  const double kH1 = DBAG_SC(0, 1.5707963267341256), kH2 = DBAG_SC(1, 6.077100506303966e-11),
               kH3 = DBAG_SC(2, 2.0222662487959506e-21), kTwoOverPi = DBAG_SC(3, 0.6366197723675814);
  const double k = rint(x * kTwoOverPi);
  const double r = ((x - k * kH1) - k * kH2) - k * kH3;
  const double z = r * r;
  double p = DBAG_SC(4, 2.8114572543455206e-15);
  p = p * z + DBAG_SC(5, -7.647163731819816e-13);
  p = p * z + DBAG_SC(6, 1.6059043836821613e-10);
  p = p * z + DBAG_SC(7, -2.505210838544172e-08);
  p = p * z + DBAG_SC(8, 2.7557319223985893e-06);
  p = p * z + DBAG_SC(9, -0.0001984126984126984);
  p = p * z + DBAG_SC(10, 0.008333333333333333);
  p = p * z + DBAG_SC(11, -0.16666666666666666);
  const double s = r + (r * z) * p;
  double q = DBAG_SC(12, -1.5619206968586225e-16);
  q = q * z + DBAG_SC(13, 4.779477332387385e-14);
  q = q * z + DBAG_SC(14, -1.1470745597729725e-11);
  q = q * z + DBAG_SC(15, 2.08767569878681e-09);
  q = q * z + DBAG_SC(16, -2.755731922398589e-07);
  q = q * z + DBAG_SC(17, 2.48015873015873e-05);
  q = q * z + DBAG_SC(18, -0.001388888888888889);
  q = q * z + DBAG_SC(19, 0.041666666666666664);
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

struct ETrig {
  double sa, ca, sb, cb, sg, cg;
};

__device__ __forceinline__ void etrig(double a, double b, double g, ETrig& t) {
  det_sincos(a, &t.sa, &t.ca);
  det_sincos(b, &t.sb, &t.cb);
  det_sincos(g, &t.sg, &t.cg);
}

// R = (Rz*Ry)*Rx, geometry.cpp:62-64 / 82-90 (zeros folded).
__device__ __forceinline__ void erot(const ETrig& t, double R[9]) {
  const double M00 = t.cg * t.cb, M01 = -t.sg, M02 = t.cg * t.sb;
  const double M10 = t.sg * t.cb, M11 = t.cg, M12 = t.sg * t.sb;
  const double M20 = -t.sb, M22 = t.cb;
  R[0] = M00;
  R[1] = M01 * t.ca + M02 * t.sa;
  R[2] = M01 * (-t.sa) + M02 * t.ca;
  R[3] = M10;
  R[4] = M11 * t.ca + M12 * t.sa;
  R[5] = M11 * (-t.sa) + M12 * t.ca;
  R[6] = M20;
  R[7] = M22 * t.sa;
  R[8] = M22 * t.ca;
}

// mat_vec (oracle.cpp): (a0 x0 + a1 x1) + a2 x2
__device__ __forceinline__ double row3(const double* a, const double* x) {
  return (a[0] * x[0] + a[1] * x[1]) + a[2] * x[2];
}

// dR_k * x for k = alpha, beta, gamma (geometry.cpp:82-90), zeros folded.
__device__ __forceinline__ void edrot_x(const ETrig& t, const double* x, double vA[3],
                                        double vB[3], double vG[3]) {
  // dA = (Rz*Ry) * drot_x : columns 1,2 nonzero
  const double M01 = -t.sg, M02 = t.cg * t.sb, M11 = t.cg, M12 = t.sg * t.sb, M22 = t.cb;
  const double a01 = M01 * (-t.sa) + M02 * t.ca, a02 = M01 * (-t.ca) + M02 * (-t.sa);
  const double a11 = M11 * (-t.sa) + M12 * t.ca, a12 = M11 * (-t.ca) + M12 * (-t.sa);
  const double a21 = M22 * t.ca, a22 = M22 * (-t.sa);
  vA[0] = a01 * x[1] + a02 * x[2];
  vA[1] = a11 * x[1] + a12 * x[2];
  vA[2] = a21 * x[1] + a22 * x[2];
  // dB = (Rz*drot_y) * Rx
  const double N00 = t.cg * (-t.sb), N02 = t.cg * t.cb, N10 = t.sg * (-t.sb), N12 = t.sg * t.cb,
               N20 = -t.cb, N22 = -t.sb;
  vB[0] = (N00 * x[0] + (N02 * t.sa) * x[1]) + (N02 * t.ca) * x[2];
  vB[1] = (N10 * x[0] + (N12 * t.sa) * x[1]) + (N12 * t.ca) * x[2];
  vB[2] = (N20 * x[0] + (N22 * t.sa) * x[1]) + (N22 * t.ca) * x[2];
  // dG = (drot_z*Ry) * Rx : row 2 zero
  const double Q00 = (-t.sg) * t.cb, Q01 = -t.cg, Q02 = (-t.sg) * t.sb;
  const double Q10 = t.cg * t.cb, Q11 = -t.sg, Q12 = t.cg * t.sb;
  vG[0] = (Q00 * x[0] + (Q01 * t.ca + Q02 * t.sa) * x[1]) + (Q01 * (-t.sa) + Q02 * t.ca) * x[2];
  vG[1] = (Q10 * x[0] + (Q11 * t.ca + Q12 * t.sa) * x[1]) + (Q11 * (-t.sa) + Q12 * t.ca) * x[2];
  vG[2] = 0.0;
}

// try_project (geometry.cpp:92-99) given the trig values t of v's angles.
__device__ __forceinline__ bool eproject_t(const double v[9], double f, double eps,
                                           const ETrig& t, double R[9], double w[3],
                                           double z[2]) {
  erot(t, R);
  w[0] = row3(R, v) + v[6];
  w[1] = row3(R + 3, v) + v[7];
  w[2] = row3(R + 6, v) + v[8];
  if (!(w[2] >= eps)) return false;
  z[0] = f * w[0] / w[2];  // geometry.cpp:98
  z[1] = f * w[1] / w[2];
  return true;
}

// try_project (geometry.cpp:92-99): w = R x + t.
__device__ __forceinline__ bool eproject(const double v[9], double f, double eps, ETrig& t,
                                         double R[9], double w[3], double z[2]) {
  etrig(v[3], v[4], v[5], t);
  erot(t, R);
  w[0] = row3(R, v) + v[6];
  w[1] = row3(R + 3, v) + v[7];
  w[2] = row3(R + 6, v) + v[8];
  if (!(w[2] >= eps)) return false;
  z[0] = f * w[0] / w[2];  // geometry.cpp:98
  z[1] = f * w[1] / w[2];
  return true;
}

// try_project_with_jacobians (geometry.cpp:141-159) given cached t, R, w:
// A0/A1 = [Jp | Jc] rows 0/1.
__device__ __forceinline__ void ejac_inv(const double v[9], const ETrig& t, const double R[9],
                                         const double w[3], double inv_z, double f, double A0[9],
                                         double A1[9]) {
  const double d00 = f * inv_z, d02 = -f * w[0] * inv_z * inv_z;
  const double d11 = f * inv_z, d12 = -f * w[1] * inv_z * inv_z;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    A0[c] = d00 * R[c] + d02 * R[6 + c];
    A1[c] = d11 * R[3 + c] + d12 * R[6 + c];
  }
  double vA[3], vB[3], vG[3];
  edrot_x(t, v, vA, vB, vG);
  A0[3] = d00 * vA[0] + d02 * vA[2];
  A1[3] = d11 * vA[1] + d12 * vA[2];
  A0[4] = d00 * vB[0] + d02 * vB[2];
  A1[4] = d11 * vB[1] + d12 * vB[2];
  A0[5] = d00 * vG[0] + d02 * vG[2];
  A1[5] = d11 * vG[1] + d12 * vG[2];
  A0[6] = d00;
  A1[6] = 0.0;
  A0[7] = 0.0;
  A1[7] = d11;
  A0[8] = d02;
  A1[8] = d12;
}

// inv_z = __drcp_rn(w[2]) == 1.0 / w[2] (IEEE, round to nearest)
__device__ __forceinline__ void ejac(const double v[9], const ETrig& t, const double R[9],
                                     const double w[3], double f, double A0[9], double A1[9]) {
  ejac_inv(v, t, R, w, __drcp_rn(w[2]), f, A0, A1);
}

// sum of squares, sequential from 0.0 (oracle.cpp sqn). The first term is
// taken as the start value: a square is never -0, and 0.0 + p == p bitwise
// for every other p.
__device__ __forceinline__ double sqn(const double* a, int n) {
  double s = a[0] * a[0];
  for (int i = 1; i < n; ++i) s += a[i] * a[i];
  return s;
}

}  // namespace exact
}  // namespace dbag
