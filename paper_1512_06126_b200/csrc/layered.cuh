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


// ------------------------------------------- point evaluations of U(z, z') ----
// fundamental_value (layered.hpp:60-66) and point_moments (layered.hpp:116-126)
// of one spectral state: see layered.cu for the closed forms
constexpr int kMaxL = 16;  // layers (greens.cu kMaxLayers)

struct StateDev {
  int L, gamma;
  double top[kMaxL], bot[kMaxL];  // top_of / bottom_of per layer (halfspaces: their single boundary)
  cplx sig[kMaxL], eta[kMaxL], p[kMaxL], q[kMaxL], one_p[kMaxL], one_q[kMaxL], e2l[kMaxL], em1[kMaxL],
      a[kMaxL];
};

__device__ __forceinline__ int layer_at(const StateDev& S, double z) {  // interface points belong below
  int m = 0;
  while (m < S.L && S.top[m + 1] <= z) ++m;
  return m;
}

__device__ __forceinline__ cplx ipow_c(cplx c, int n) {
  cplx r = {1.0, 0.0};
  for (int i = 0; i < n; ++i) r = r * c;
  return r;
}

__device__ cplx fundamental_dev(const StateDev& S, double z, double zs, int dz, int dzs, int lz, int lzs) {
  const bool swap = z > zs;
  const double za = swap ? zs : z, zb = swap ? z : zs;  // shallower, deeper
  const int da = swap ? dzs : dz, db = swap ? dz : dzs;
  const int rz = lz >= 0 ? lz : layer_at(S, z), rs = lzs >= 0 ? lzs : layer_at(S, zs);
  const int r = swap ? rs : rz, s = swap ? rz : rs;
  cplx amp, base;
  if (r == s) {
    amp = S.a[r];
    base = -(zb - za) * S.eta[r];
  } else {
    cplx chain = {1.0, 0.0};
    cplx path = {0.0, 0.0};
    for (int m = r; m < s; ++m) {
      chain = chain * cdiv(S.one_p[m + 1], S.em1[m] + S.e2l[m] * S.one_p[m]);
      if (m > r) path = path + (S.bot[m] - S.top[m]) * S.eta[m];
    }
    amp = S.a[s] * chain;
    base = -((zb - S.top[s]) * S.eta[s]) - (S.bot[r] - za) * S.eta[r] - path;
  }
  cplx Sp = {1.0, 0.0}, Mp = {1.0, 0.0};
  if (S.p[r].re != 0.0 || S.p[r].im != 0.0) {
    const cplx e = cexpm1((-2.0 * (za - S.top[r])) * S.eta[r]);
    Sp = S.one_p[r] + S.p[r] * e;
    Mp = (cplx{2.0, 0.0} - S.one_p[r]) - S.p[r] * e;
  }
  cplx Sq = {1.0, 0.0}, Mq = {1.0, 0.0};
  if (S.q[s].re != 0.0 || S.q[s].im != 0.0) {
    const cplx e = cexpm1((-2.0 * (S.bot[s] - zb)) * S.eta[s]);
    Sq = S.one_q[s] + S.q[s] * e;
    Mq = (cplx{2.0, 0.0} - S.one_q[s]) - S.q[s] * e;
  }
  cplx v = amp * cexp(base) * ipow_c(S.eta[r], da) * ipow_c(-S.eta[s], db) * (da & 1 ? Mp : Sp) *
           (db & 1 ? Mq : Sq);
  if (swap && S.gamma == 1) v = v * cdiv(S.sig[s], S.sig[r]);
  return v;
}

// P_m(za) / P_m(zb) inside layer m, za <= zb: the decaying-up solution's ratio
__device__ __forceinline__ cplx p_step(const StateDev& S, int m, double za, double zb) {
  const cplx e = cexp(-(zb - za) * S.eta[m]);
  if (m == 0 || (S.p[m].re == 0.0 && S.p[m].im == 0.0)) return e;
  const cplx sa = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (za - S.top[m])) * S.eta[m]);
  const cplx sb = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (zb - S.top[m])) * S.eta[m]);
  return e * cdiv(sa, sb);
}

// the piece of interval [a, b] in layer m below / above the observation depth:
// a_m / eta int_a^b of the source-side solution anchored at a (below) or b (above)
__device__ __forceinline__ cplx piece(const StateDev& S, int m, double a, double b, bool above) {
  const cplx eta = S.eta[m];
  const cplx u = -cexpm1(-(b - a) * eta);
  const bool hp = S.p[m].re != 0.0 || S.p[m].im != 0.0, hq = S.q[m].re != 0.0 || S.q[m].im != 0.0;
  cplx sp = {1.0, 0.0}, tq = {1.0, 0.0};
  if (above) {
    if (hp) sp = S.one_p[m] + S.p[m] * cexpm1(-(a + b - 2.0 * S.top[m]) * eta);
    if (hq) tq = S.one_q[m] + S.q[m] * cexpm1((-2.0 * (S.bot[m] - b)) * eta);
  } else {
    if (hp) sp = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (a - S.top[m])) * eta);
    if (hq) tq = S.one_q[m] + S.q[m] * cexpm1(-(2.0 * S.bot[m] - a - b) * eta);
  }
  return cdiv(S.a[m], eta) * u * sp * tq;
}

// single moments m0[j] = int_j U(z0, zs) dzs and m1[j] = d/dz of it at z0
// (layered.cpp:450-542 contract) for every interval of the partition
__device__ void point_moments_dev(const StateDev& S, const Interval* __restrict__ iv, const double* __restrict__ br,
                                  int nz, double z0, cplx* m0, cplx* m1) {
  const int r0 = layer_at(S, z0);
  const cplx e0 = S.eta[r0];
  // log-derivatives of the decaying-up (P) and decaying-down (Q) solutions at z0
  cplx dP = e0, dQ = -e0;
  if (r0 != 0 && (S.p[r0].re != 0.0 || S.p[r0].im != 0.0)) {
    const cplx e = cexpm1((-2.0 * (z0 - S.top[r0])) * e0);
    dP = e0 * cdiv((cplx{2.0, 0.0} - S.one_p[r0]) - S.p[r0] * e, S.one_p[r0] + S.p[r0] * e);
  }
  if (r0 != S.L && (S.q[r0].re != 0.0 || S.q[r0].im != 0.0)) {
    const cplx e = cexpm1((-2.0 * (S.bot[r0] - z0)) * e0);
    dQ = -e0 * cdiv((cplx{2.0, 0.0} - S.one_q[r0]) - S.q[r0] * e, S.one_q[r0] + S.q[r0] * e);
  }
  int k;  // interval holding z0; -1 above the partition, nz below it
  if (z0 <= br[0]) k = -1;
  else if (z0 >= br[nz]) k = nz;
  else {
    k = 0;
    while (br[k + 1] <= z0) ++k;
  }
  auto factors = [&](int j) {
    const Interval I = iv[j];
    const int m = I.layer;
    const IvPack pk = iv_pack(I, S.eta[m], crecip(S.eta[m]), S.e2l[m]);
    return iv_factors(I, pk, S.p[m], S.q[m], S.a[m], S.one_p[m], S.one_q[m]);
  };
  for (int j = 0; j < min(k, nz); ++j) {  // above: the source-side P branch to z0
    const IvFac f = factors(j);
    const cplx u1 = fundamental_dev(S, br[j + 1], z0, 0, 0, -1, -1);
    const cplx sf = S.gamma == 1 ? cdiv(S.sig[r0], S.sig[iv[j].layer]) : cplx{1.0, 0.0};
    m0[j] = sf * f.H0 * u1;
    m1[j] = m0[j] * dQ;
  }
  if (k >= 0 && k < nz) {  // the interval holding z0, split there
    const int m = iv[k].layer;
    const cplx up = z0 > br[k] ? piece(S, m, br[k], z0, true) : cplx{0.0, 0.0};
    const cplx lo = z0 < br[k + 1] ? piece(S, m, z0, br[k + 1], false) : cplx{0.0, 0.0};
    m0[k] = up + lo;
    m1[k] = dQ * up + dP * lo;
  }
  if (k < nz) {  // below: the observation-side P ratio chained down
    const int first = max(k + 1, 0);
    cplx T = {1.0, 0.0};
    double zc = z0;
    int m = r0;
    while (zc < br[first]) {
      const double seg = m < S.L ? fmin(S.bot[m], br[first]) : br[first];
      T = T * p_step(S, m, zc, seg);
      zc = seg;
      if (zc < br[first]) ++m;
    }
    for (int j = first; j < nz; ++j) {
      const IvFac f = factors(j);
      m0[j] = T * f.J0;
      m1[j] = dP * m0[j];
      T = T * f.theta;
    }
  }
}

}  // namespace
}  // namespace emie_cu
