// Layered-medium building blocks shared by the device Green's build
// (greens.cu), the layered-model API entry points (spectral states, moment
// tables) and the receiver-side point evaluations (layered.cu): complex
// helpers, the interval geometry, the exponential pack and the per-interval
// factors of src/layered.cpp:222-317.
#pragma once

#include "common.cuh"

namespace emie_cu {
namespace {

// ------------------------------------------------------ complex helpers ----
// Smith's algorithm: the exact-path fallback of cdiv (zero or non-finite divisor)
__device__ __noinline__ cplx cdiv_smith(cplx a, cplx b) {
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, d = b.re + b.im * r;
    return {(a.re + a.im * r) / d, (a.im - a.re * r) / d};
  }
  const double r = b.re / b.im, d = b.re * r + b.im;
  return {(a.re * r + a.im) / d, (a.im * r - a.re) / d};
}

__device__ __forceinline__ cplx csqrt_pos(cplx z) {
  // principal square root, then the Re > 0 branch (layered.cpp:87-89)
  const double m = hypot(z.re, z.im);
  cplx r;
  if (m == 0.0) return {0.0, 0.0};
  const double t = sqrt(0.5 * (fabs(z.re) + m));
  if (z.re >= 0.0) r = {t, z.im / (2.0 * t)};
  else r = {fabs(z.im) / (2.0 * t), copysign(t, z.im)};
  if (r.re < 0.0) r = -r;
  return r;
}
// exp(x) - 1 without cancellation (layered.cpp:19-25)
__device__ __forceinline__ cplx cexpm1(cplx x) {
  const double em = expm1(x.re);
  double sh, ch;
  sincos(0.5 * x.im, &sh, &ch);
  // one sincos: cos x = 1 - 2 sin^2(x/2), sin x = 2 sin(x/2) cos(x/2)
  const double s = 2.0 * sh * ch, cm1 = -2.0 * sh * sh;
  return {em * (1.0 + cm1) + cm1, (em + 1.0) * s};
}
__device__ __forceinline__ cplx cexp(cplx x) {
  const double e = exp(x.re);
  double s, c;
  sincos(x.im, &s, &c);
  return {e * c, e * s};
}
// 2^e as a double for e in [-1022, 1023] (exponent bits built directly)
__device__ __forceinline__ double pow2i(int e) {
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}
// a * 2^e without the software scalbn: one multiply in the normal range, two
// half-steps outside it (exact unless the result itself under/overflows)
__device__ __forceinline__ cplx scal2(cplx a, int e) {
  if (e >= -1022 && e <= 1023) {
    const double f = pow2i(e);
    return {a.re * f, a.im * f};
  }
  e = max(-2200, min(2200, e));
  const int e1 = e / 2, e2 = e - e1;
  const double f1 = (e1 < -1022) ? 0.0 : pow2i(min(e1, 1023));
  const double f2 = (e2 < -1022) ? 0.0 : pow2i(min(e2, 1023));
  return {a.re * f1 * f2, a.im * f1 * f2};
}
// floor(log2 |x|) for finite x != 0 (ilogb without the library call)
__device__ __forceinline__ int ilog2(double x) {
  const long long b = __double_as_longlong(x);
  const int ex = static_cast<int>((b >> 52) & 0x7ff);
  if (ex != 0) return ex - 1023;
  return ilogb(x);  // subnormal: rare
}

// 1/d for d in [1, 8) to ~1 ulp: hardware reciprocal estimate + two Newton steps
__device__ __forceinline__ double rcp_unit(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
// a / b without FP64 divisions (nvcc emits each as an out-of-line call): b is
// scaled by the power of two of its larger component, so |b'|^2 is in [1, 2]
// and neither overflows nor underflows; a / b = a conj(b') / |b'|^2 * 2^-e.
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  const double m = fmax(fabs(b.re), fabs(b.im));
  if (!(m > 0.0) || !(m <= 1.0e300) || m < 1.0e-300) return cdiv_smith(a, b);
  const int e = ilog2(m);
  const double sc = pow2i(-e);
  const double br = b.re * sc, bi = b.im * sc;
  const double r = rcp_unit(br * br + bi * bi);
  const cplx q = {(a.re * br + a.im * bi) * r, (a.im * br - a.re * bi) * r};
  return scal2(q, -e);
}
__device__ __forceinline__ cplx crecip(cplx b) { return cdiv(cplx{1.0, 0.0}, b); }


// per-interval geometry (device arrays): a, b, h, d (top), dp (bottom), l
struct Interval {
  double a, b, h, d, dp, l;
  int layer;
  int has_p, has_q;
  cplx inv_sig;  // 1 / sigma_b of the interval
};

// Exponential pack of one interval (layered.cpp:222-273): everything from four
// exponentials through expm1 algebra, shared by both gammas
struct IvPack {
  cplx eta, ie, ie2, eta2, u, ehm1, eh, el2, elh;
  cplx epa, epa2m1, epabm1, epb2m1, eqb, eqabm1;
};
__device__ __forceinline__ IvPack iv_pack(const Interval& I, cplx eta, cplx ie, cplx el2) {
  IvPack k;
  k.eta = eta;
  k.ie = ie;  // 1/eta, 1/eta^2: the divisions of the factors become products
  k.ie2 = ie * ie;
  k.eta2 = eta * eta;
  k.ehm1 = cexpm1(-I.h * eta);
  k.eh = cplx{1.0, 0.0} + k.ehm1;
  k.u = -k.ehm1;
  k.el2 = el2;
  k.epa = {1.0, 0.0};
  k.epa2m1 = k.epabm1 = k.epb2m1 = {0.0, 0.0};
  k.eqb = {1.0, 0.0};
  k.eqabm1 = {0.0, 0.0};
  if (I.has_p) {
    const cplx epam1 = cexpm1(-(I.a - I.d) * eta);
    const cplx epbm1 = epam1 + k.ehm1 + epam1 * k.ehm1;
    k.epa = cplx{1.0, 0.0} + epam1;
    k.epa2m1 = 2.0 * epam1 + epam1 * epam1;
    k.epabm1 = epam1 + epbm1 + epam1 * epbm1;
    k.epb2m1 = 2.0 * epbm1 + epbm1 * epbm1;
  }
  if (I.has_q) {
    const cplx eqbm1 = cexpm1(-(I.dp - I.b) * eta);
    const cplx eqam1 = eqbm1 + k.ehm1 + eqbm1 * k.ehm1;
    k.eqb = cplx{1.0, 0.0} + eqbm1;
    k.eqabm1 = eqam1 + eqbm1 + eqam1 * eqbm1;
  }
  k.elh = (I.has_p && I.has_q) ? cexp((-(2.0 * I.l - I.h)) * eta) : cplx{0.0, 0.0};
  return k;
}

// Per-interval building blocks of one gamma's tables (layered.cpp:275-317):
// theta (chain step), H0/H1 (row factors), J0/J1 (column factors) and the
// diagonal moments W00d, W10d, W11d, W20d (the W11d/W20d jump-content choice
// of layered.cpp:305-315 kept)
struct IvFac {
  cplx theta, H0, H1, J0, J1, W00d, W10d, W11d, W20d;
};
__device__ __forceinline__ IvFac iv_factors(const Interval& I, const IvPack& k, cplx p, cplx q, cplx A, cplx one_p,
                                            cplx one_q) {
  const cplx Sa = one_p + p * k.epa2m1;
  const cplx Sab = one_p + p * k.epabm1;
  const cplx Mab = (cplx{2.0, 0.0} - one_p) - p * k.epabm1;
  const cplx Dp = one_p + p * k.epb2m1;
  const cplx Tq = one_q + q * k.eqabm1;
  const cplx TMq = (cplx{2.0, 0.0} - one_q) - q * k.eqabm1;
  const cplx iDp = crecip(Dp);
  IvFac f;
  f.theta = (k.eh * Sa) * iDp;
  f.H0 = ((k.u * Sab) * k.ie) * iDp;
  f.H1 = (k.u * Mab) * iDp;
  f.J0 = (A * k.u * Sa * Tq) * k.ie;
  f.J1 = -(A * k.u * Sa * TMq);
  const cplx Ip = (k.epa * k.u) * k.ie;
  const cplx Iq = (k.eqb * k.u) * k.ie;
  const cplx Sp = p * Ip * Ip, Sq = q * Iq * Iq;
  const cplx M0 = (2.0 * (I.h * k.eta + k.ehm1)) * k.ie2;
  const cplx P0 = 2.0 * ((k.elh * k.u) * k.ie2 - (I.h * k.el2) * k.ie);
  f.W00d = A * (Sp + Sq + M0 + p * q * P0);
  f.W10d = A * k.eta * (Sq - Sp);
  f.W11d = A * (k.eta2 * (Sp + Sq) + 2.0 * k.u - 2.0 * p * q * k.elh * k.u) - cplx{2.0 * I.h, 0.0};
  f.W20d = k.eta2 * f.W00d - cplx{2.0 * I.h, 0.0};
  return f;
}


}  // namespace
}  // namespace emie_cu
