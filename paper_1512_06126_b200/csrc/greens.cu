// Green's-tensor build on the device (sm_100a): assemble_operator
// (src/greens.cpp:332-371) + transform_operator (src/toeplitz.cpp:92-161).
//
//  K6 filter_design_kernel  one CTA per (offset, kernel): 2*half samples of
//     the closed-form design output (hankel.cpp:35-113), FFT, division by the
//     input spectrum, inverse FFT, 451-weight window (hankel.cpp:239-281).
//  K5 assemble_kernel       one CTA per (offset, pair group): lambda in chunks
//     of LC; per chunk the layer states (layered.cpp:67-129), interval packs
//     and factors (layered.cpp:237-317) and chain prefix products are built
//     in SMEM, then every thread advances its own interval pairs' seven
//     accumulators over the chunk in lambda order (greens.cpp:167-191).
//     Blocks are scaled by R^3/4pi, R^2/4pi, R/4pi (greens.cpp:193-213).
//  K7 the spectra passes of operator.cu.
//
// Numerics kept from the reference: expm1-based
// exponentials, exact one_p/one_q, the W11d/W20d jump-content choice, the
// erfc tails, the lambda > 38 cutoff, the alternating-sign lattices. The
// off-diagonal chain products prod_{l=k+1}^{kp-1} theta_l come from prefix
// products kept as (mantissa, binary exponent, zero count), so an underflowed
// theta zeroes exactly the chains that span it, as the running product does.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "layered.cuh"
#include "operator.cuh"
#include "tma.cuh"

namespace emie_cu {

namespace {

constexpr double kMu0 = 1.2566370614359172e-06;  // include/emie/types.hpp:11
constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kSqrtPi = 1.7724538509055160273;
constexpr int kMaxLayers = 16;
#ifndef EMIE_GREEN_THREADS
#define EMIE_GREEN_THREADS 256
#endif
constexpr int kGreenThreads = EMIE_GREEN_THREADS;  // threads per assemble CTA
#ifndef EMIE_GREEN_SLOTS
#define EMIE_GREEN_SLOTS 2
#endif
constexpr int kGreenSlots = EMIE_GREEN_SLOTS;
#ifndef EMIE_GREEN_PAIR_UNROLL
#define EMIE_GREEN_PAIR_UNROLL 2
#endif
constexpr int kPairUnroll = EMIE_GREEN_PAIR_UNROLL;  // lambdas per pair-phase loop body  // full-lambda-range pairs per thread (+ a lambda-split tail)

// ------------------------------------------------------ hankel helpers ----
__device__ __forceinline__ double ediff(double a, double b) {  // hankel.cpp:22-26
  if (a > 1.0 && b > 1.0) return erfc(0.5 * a) - erfc(0.5 * b);
  if (a < -1.0 && b < -1.0) return erfc(-0.5 * b) - erfc(-0.5 * a);
  return erf(0.5 * b) - erf(0.5 * a);
}

// The stencils are evaluated product by product with explicit rounding (no
// fused multiply-adds), as the reference's host build evaluates them: on a
// symmetric axis (d = 0) the odd terms cancel to an exact zero
// (test_hankel.cpp:88-95), which a contracted a*b + c*d would leave as the
// rounding residue of one product.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ void axis_stencil(int alpha, double d, double h, double out[3]) {  // hankel.cpp:35-71
  const double wp = add(d, h), w0 = d, wm = sub(d, h);
  const double gp = exp(mul(mul(-0.25, wp), wp));
  const double g0 = exp(mul(mul(-0.25, w0), w0));
  const double gm = exp(mul(mul(-0.25, wm), wm));
  const double gs = add(sub(gp, mul(2.0, g0)), gm);
  const double ep = ediff(w0, wp);
  const double em = ediff(wm, w0);
  // a_p x_p - 2 a_0 x_0 + a_m x_m with a = w^k
  auto st3 = [&](double ap, double a0, double am) { return add(sub(mul(ap, gp), mul(mul(2.0, a0), g0)), mul(am, gm)); };
  if (alpha == 0) {
    const double lin = sub(mul(wp, ep), mul(wm, em));
    const double w2s = st3(mul(wp, wp), mul(w0, w0), mul(wm, wm));
    out[0] = add(mul(kSqrtPi, lin), mul(2.0, gs));
    out[1] = add(mul(mul(2.0, kSqrtPi), lin), mul(8.0, gs));
    out[2] = add(add(mul(mul(12.0, kSqrtPi), lin), mul(4.0, w2s)), mul(64.0, gs));
  } else if (alpha == 1) {
    const double es = sub(ep, em);
    const double wg = st3(wp, w0, wm);
    const double w3g = st3(mul(mul(wp, wp), wp), mul(mul(w0, w0), w0), mul(mul(wm, wm), wm));
    out[0] = mul(kSqrtPi, es);
    out[1] = sub(mul(mul(2.0, kSqrtPi), es), mul(2.0, wg));
    out[2] = sub(sub(mul(mul(12.0, kSqrtPi), es), mul(2.0, w3g)), mul(12.0, wg));
  } else {
    out[0] = gs;
    out[1] = st3(mul(wp, wp), mul(w0, w0), mul(wm, wm));
    out[2] = st3(mul(mul(mul(wp, wp), wp), wp), mul(mul(mul(w0, w0), w0), w0), mul(mul(mul(wm, wm), wm), wm));
  }
}

// axis_stencil for alpha = 0, 1, 2 at once: the exponentials and error-function
// differences are shared, every output is formed by exactly axis_stencil's
// operations (the same bits)
__device__ void axis_stencil_all(double d, double h, double out[3][3]) {
  const double wp = add(d, h), w0 = d, wm = sub(d, h);
  const double gp = exp(mul(mul(-0.25, wp), wp));
  const double g0 = exp(mul(mul(-0.25, w0), w0));
  const double gm = exp(mul(mul(-0.25, wm), wm));
  const double gs = add(sub(gp, mul(2.0, g0)), gm);
  const double ep = ediff(w0, wp);
  const double em = ediff(wm, w0);
  auto st3 = [&](double ap, double a0, double am) { return add(sub(mul(ap, gp), mul(mul(2.0, a0), g0)), mul(am, gm)); };
  const double lin = sub(mul(wp, ep), mul(wm, em));
  const double w2s = st3(mul(wp, wp), mul(w0, w0), mul(wm, wm));
  out[0][0] = add(mul(kSqrtPi, lin), mul(2.0, gs));
  out[0][1] = add(mul(mul(2.0, kSqrtPi), lin), mul(8.0, gs));
  out[0][2] = add(add(mul(mul(12.0, kSqrtPi), lin), mul(4.0, w2s)), mul(64.0, gs));
  const double es = sub(ep, em);
  const double wg = st3(wp, w0, wm);
  const double w3g = st3(mul(mul(wp, wp), wp), mul(mul(w0, w0), w0), mul(mul(wm, wm), wm));
  out[1][0] = mul(kSqrtPi, es);
  out[1][1] = sub(mul(mul(2.0, kSqrtPi), es), mul(2.0, wg));
  out[1][2] = sub(sub(mul(mul(12.0, kSqrtPi), es), mul(2.0, w3g)), mul(12.0, wg));
  out[2][0] = gs;
  out[2][1] = w2s;  // st3 of the squares, as axis_stencil's alpha = 2 out[1]
  out[2][2] = st3(mul(mul(mul(wp, wp), wp), wp), mul(mul(mul(w0, w0), w0), w0), mul(mul(mul(wm, wm), wm), wm));
}

struct Geom {
  double r, p, q, phi;
  double cs, sn;  // cos(phi), sin(phi): on the host from the C library, as the reference evaluates them
};
__host__ __device__ inline Geom pair_geometry(int oi, int oj, double hx, double hy) {  // hankel.cpp:80-91
  const double ax = oj * hx - 0.5 * hx;
  const double ay = oi * hy - 0.5 * hy;
  Geom g;
  g.r = hypot(ax, ay);
  g.p = hx / g.r;
  g.q = hy / g.r;
  g.phi = atan2(ay, ax);
#ifdef __CUDA_ARCH__
  sincos(g.phi, &g.sn, &g.cs);
#else
  g.cs = std::cos(g.phi);
  g.sn = std::sin(g.phi);
#endif
  return g;
}
// a caller's PairGeometry (r, p, q, phi) as the device routines take it
inline Geom geom_of(const double* geom) {
  return Geom{geom[0], geom[1], geom[2], geom[3], std::cos(geom[3]), std::sin(geom[3])};
}

// Offsets travel as integer codes: code = (oi + bias_i) * span + (oj + bias_j).
// A full build uses span = nx, no bias (code = the offset-major slot oi*nx + oj
// of the stored sector); a signed-offset request (assemble_block at negative
// offsets, emie_cu_assemble_blocks) uses span = 2nx - 1, bias (ny-1, nx-1) and
// stores its blocks compactly in request order.
struct OffsetCode {
  int span = 1, bias_i = 0, bias_j = 0, compact = 0;
  __host__ __device__ int oi(int c) const { return c / span - bias_i; }
  __host__ __device__ int oj(int c) const { return c % span - bias_j; }
  __host__ __device__ int slot(int c, int pos) const { return compact ? pos : c; }
};

// ---- receiver-side filters: a point observer and a source rectangle ------
// The lateral integral of a receiver (SPEC.md receiver_green_integrals) is
// one-sided: K_ab(lambda) = d^a/dx^a d^b/dy^b int_S J0(lambda rho) dS0 for the
// receiver at the origin and the source rectangle S. Its filter is designed
// like the cell-pair filters (hankel.cpp:204-281: same design input v, same
// lattice, FFT division), with the design output the one-sided integral of
// v's J0 transform (rho^4/4) e^{-rho^2/4} = (x^4 + 2 x^2 y^2 + y^4)/4 e^{-x^2/4}
// e^{-y^2/4}: per axis the 2-point difference of the antiderivatives
//   P0(t) = sqrt(pi) erf(t/2),  P1 = -2t g + 2 P0,  P2 = -2t^3 g - 12 t g + 12 P0,
// g = e^{-t^2/4} (a = 0), of t^{2k} g itself (a = 1) or of its derivative (a = 2),
// at t1 = -(cx - p/2) r, t2 = -(cx + p/2) r. The sum is R^{1-a-b} sum_m w_m
// f(lambda_m / R) (two lateral integrations instead of four: 1 - a - b in
// place of hankel.hpp's 3 - a - b).
struct PGeom {
  double r, p, q, cx, cy;  // reference distance; rectangle size and centre offset over r
};

__device__ void point_stencil(int alpha, double t1, double t2, double out[3]) {
  const double g1 = exp(-0.25 * t1 * t1), g2 = exp(-0.25 * t2 * t2);
  if (alpha == 0) {
    const double e = kSqrtPi * ediff(t2, t1);  // P0(t1) - P0(t2)
    const double d1 = t1 * g1 - t2 * g2, d3 = t1 * t1 * t1 * g1 - t2 * t2 * t2 * g2;
    out[0] = e;
    out[1] = -2.0 * d1 + 2.0 * e;
    out[2] = -2.0 * d3 - 12.0 * d1 + 12.0 * e;
  } else if (alpha == 1) {
    out[0] = g1 - g2;
    out[1] = t1 * t1 * g1 - t2 * t2 * g2;
    out[2] = t1 * t1 * t1 * t1 * g1 - t2 * t2 * t2 * t2 * g2;
  } else {
    out[0] = -0.5 * (t1 * g1 - t2 * g2);
    out[1] = (2.0 * t1 - 0.5 * t1 * t1 * t1) * g1 - (2.0 * t2 - 0.5 * t2 * t2 * t2) * g2;
    out[2] = (4.0 * t1 * t1 * t1 - 0.5 * t1 * t1 * t1 * t1 * t1) * g1 -
             (4.0 * t2 * t2 * t2 - 0.5 * t2 * t2 * t2 * t2 * t2) * g2;
  }
}

__device__ double point_kernel_output(const PGeom& g, int alpha, int beta, double s) {
  const double r = exp(s);
  double ax[3], ay[3];
  point_stencil(alpha, -(g.cx - 0.5 * g.p) * r, -(g.cx + 0.5 * g.p) * r, ax);
  point_stencil(beta, -(g.cy - 0.5 * g.q) * r, -(g.cy + 0.5 * g.q) * r, ay);
  const double comb = 0.25 * (ax[2] * ay[0] + 2.0 * ax[1] * ay[1] + ax[0] * ay[2]);
  if (comb == 0.0) return 0.0;
  return exp(-(1 - alpha - beta) * s) * comb;
}

__device__ double kernel_output(const Geom& g, int alpha, int beta, double s) {  // hankel.cpp:101-113
  const double r = exp(s);
  const double hx = g.p * r, hy = g.q * r;
  const double sn = g.sn, cs = g.cs;
  // products rounded before the sum, as the reference evaluates them: on an
  // axis through the pair's symmetry (e.g. oi = 0) r sin(phi) rounds to
  // exactly -hy / 2, so dy = 0 and the one-derivative kernel across it is an
  // exact zero (test_hankel.cpp:88-95); a fused multiply-add would keep the
  // product's rounding residue instead
  const double dx = __dadd_rn(__dmul_rn(r, cs), 0.5 * hx);
  const double dy = __dadd_rn(__dmul_rn(r, sn), 0.5 * hy);
  double ax[3], ay[3];
  axis_stencil(alpha, dx, hx, ax);
  axis_stencil(beta, dy, hy, ay);
  const double comb = mul(0.25, add(add(mul(ax[2], ay[0]), mul(mul(2.0, ax[1]), ay[1])), mul(ax[0], ay[2])));
  if (comb == 0.0) return 0.0;
  return mul(exp(-(3 - alpha - beta) * s), comb);
}

__device__ __forceinline__ double design_input(double lambda) {  // hankel.cpp:93-99
  if (lambda > 38.0) return 0.0;
  const double l2 = mul(lambda, lambda);
  return mul(mul(mul(8.0, exp(-l2)), lambda), add(mul(sub(l2, 4.0), l2), 2.0));
}

__constant__ int kAlpha[6] = {0, 2, 0, 1, 1, 0};  // greens.cpp:137
__constant__ int kBeta[6] = {0, 0, 2, 1, 0, 1};

// ----------------------------------------------------------- K6 kernels ----
// input spectrum of the design (FilterDesigner ctor, hankel.cpp:219-231)
__global__ void filter_den_kernel(cplx* den, double* floor_out, const cplx* __restrict__ tw,
                                  FftPlan pl, int half, double step) {
  extern __shared__ cplx sm[];
  const int n = pl.n, ld = n | 1;
  cplx* a = sm;
  cplx* b = a + ld;
  cplx* t = b + ld;
  load_twiddles(t, tw, n);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int m = j - half;
    const double sign = ((j + half) % 2 == 0) ? 1.0 : -1.0;
    a[j] = {sign * design_input(exp(-m * step)), 0.0};
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, 1, pl, t, false);
  __shared__ double red[32];
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    den[k] = res[k];
    mx = fmax(mx, hypot(res[k].re, res[k].im));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) m = fmax(m, red[w]);
    *floor_out = 1e-12 * m;
  }
}

// The design samples of all six kernels of an offset (greens.cpp:137 order)
// at once: per sample the two axes' stencils of every derivative order share
// their exponentials and error functions (axis_stencil_all), so a full build
// evaluates the transcendentals once per (offset, sample) instead of once per
// (offset, kernel, sample); each value is kernel_output's, bit for bit.
// S[i][kern][j] = (-1)^(j + half) u(m step + shift), m = j - half.
__global__ void filter_samples_kernel(const Geom* __restrict__ gtab, int noff, int n, int half, double step,
                                      double shift, double* __restrict__ S) {
  const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (x >= static_cast<long long>(noff) * n) return;
  const int i = static_cast<int>(x / n), j = static_cast<int>(x - static_cast<long long>(i) * n);
  const Geom g = gtab[i];
  const int m = j - half;
  const double sign = ((j + half) % 2 == 0) ? 1.0 : -1.0;
  const double sj = m * step + shift;
  // kernel_output (hankel.cpp:101-113) with the stencils shared
  const double r = exp(sj);
  const double hx = g.p * r, hy = g.q * r;
  const double dx = __dadd_rn(__dmul_rn(r, g.cs), 0.5 * hx);
  const double dy = __dadd_rn(__dmul_rn(r, g.sn), 0.5 * hy);
  double ax[3][3], ay[3][3];
  axis_stencil_all(dx, hx, ax);
  axis_stencil_all(dy, hy, ay);
  double* o = S + static_cast<size_t>(i) * 6 * n + j;
#pragma unroll
  for (int kern = 0; kern < 6; ++kern) {
    const int alpha = kAlpha[kern], beta = kBeta[kern];
    const double comb = mul(0.25, add(add(mul(ax[alpha][2], ay[beta][0]), mul(mul(2.0, ax[alpha][1]), ay[beta][1])),
                                      mul(ax[alpha][0], ay[beta][2])));
    const double u = comb == 0.0 ? 0.0 : mul(exp(-(3 - alpha - beta) * sj), comb);
    o[static_cast<size_t>(kern) * n] = sign * u;
  }
}

// FilterDesigner::design (hankel.cpp:239-281) for offset blockIdx.x (oi, oj
// >= 0 row-major over ny x nx) and kernel blockIdx.y; err bits: 1 vanishing
// input spectrum, 2 non-real residue
__global__ void filter_design_kernel(double* W, const cplx* __restrict__ den,
                                     const double* __restrict__ den_floor,
                                     const cplx* __restrict__ tw, FftPlan pl, int half, double step,
                                     double shift, int n1, int n2, OffsetCode oc, double hx, double hy,
                                     int* err, int fixed_oi, int fixed_oj, const int* __restrict__ offs,
                                     Geom gfix, int use_gfix, int kern0, const PGeom* __restrict__ pgeo,
                                     const Geom* __restrict__ gtab, const double* __restrict__ samp) {
  extern __shared__ cplx sm[];
  const int n = pl.n, ld = n | 1;
  cplx* a = sm;
  cplx* b = a + ld;
  cplx* t = b + ld;
  const int code = offs ? offs[blockIdx.x] : static_cast<int>(blockIdx.x), kern = kern0 + blockIdx.y;
  const int off = oc.slot(code, blockIdx.x);
  const int oi = fixed_oi != INT32_MIN ? fixed_oi : oc.oi(code);
  const int oj = fixed_oi != INT32_MIN ? fixed_oj : oc.oj(code);
  // a caller-given pair geometry (FilterDesigner::design, hankel.hpp:93), else
  // the offset's, from the host's table (the reference's own C-library
  // hypot / atan2 / sin / cos: bit-identical design inputs) when given
  const Geom g = use_gfix ? gfix : gtab ? gtab[blockIdx.x] : pair_geometry(oi, oj, hx, hy);
  const int alpha = kAlpha[kern], beta = kBeta[kern];
  load_twiddles(t, tw, n);
  if (samp) {  // precomputed by filter_samples_kernel (full builds)
    const double* sv = samp + (static_cast<size_t>(blockIdx.x) * 6 + kern) * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) a[j] = {sv[j], 0.0};
  } else {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const int m = j - half;
      const double sign = ((j + half) % 2 == 0) ? 1.0 : -1.0;
      const double sj = m * step + shift;
      a[j] = {sign * (pgeo ? point_kernel_output(pgeo[blockIdx.x], alpha, beta, sj) : kernel_output(g, alpha, beta, sj)),
              0.0};
    }
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, 1, pl, t, false);
  cplx* other = res == a ? b : a;
  const double fl = *den_floor;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const cplx d = den[k];
    if (hypot(d.re, d.im) < fl) atomicOr(err, 1);
    res[k] = cdiv(res[k], d);
  }
  __syncthreads();
  cplx* back = fft_smem(res, other, ld, 1, pl, t, true);
  __shared__ double rmax[32], imax[32];
  double rm = 0.0, im = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    rm = fmax(rm, fabs(back[k].re));
    im = fmax(im, fabs(back[k].im));
  }
  for (int o = 16; o > 0; o >>= 1) {
    rm = fmax(rm, __shfl_down_sync(0xffffffffu, rm, o));
    im = fmax(im, __shfl_down_sync(0xffffffffu, im, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rmax[threadIdx.x >> 5] = rm;
    imax[threadIdx.x >> 5] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0, i = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) {
      r = fmax(r, rmax[w]);
      i = fmax(i, imax[w]);
    }
    if (i > 1e-10 * r) atomicOr(err, 2);
  }
  const int nw = n2 - n1 + 1;
  double* wo = W + (static_cast<size_t>(off) * 6 + kern) * nw;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) {
    const int m = n1 + i;
    const int j = ((m % n) + n) % n;
    const double sign = (m % 2 != 0) ? -1.0 : 1.0;
    wo[i] = sign * back[j].re / n;
  }
}

// ----------------------------------------------------------- K5 kernel ----
struct GreenParams {
  int L;           // interfaces
  int nz;
  int nx, ny;
  double hx, hy, omega;
  int nw;          // weights per kernel
  double step, shift;
  int n1;
  int LC;          // lambdas per chunk
  int npairs;      // nz(nz+1)/2
  int nent;
  OffsetCode oc;   // offset codes of this build
  // model (host-filled)
  double thick[kMaxLayers];
  double ztop[kMaxLayers], zbot[kMaxLayers];  // top_of / bottom_of per layer (layered.cpp:38-43)
  cplx sig[kMaxLayers];  // floored conductivities
  cplx sig_up[kMaxLayers];  // sig[m+1] / sig[m] (TM reflection chain, layered.cpp:113)
  cplx sig_dn[kMaxLayers];  // sig[m-1] / sig[m]
};


// SMEM plan for one chunk of LC lambdas
struct Chunk {
  // layer states [lc][gamma][m]
  cplx* eta;     // [lc][m]
  cplx* e2l;     // [lc][m]
  cplx* em1;     // [lc][m]
  cplx* p;       // [lc][g][m]
  cplx* q;
  cplx* one_p;
  cplx* one_q;
  cplx* diag_a;
  cplx* ieta;    // [lc][m]: 1 / eta[m]
  // interval fields [lc][f][j]
  cplx* F;
  double* lam;   // [8][lc]: lambda, 1/lambda, w00 w20 w02 w11 w10 w01
  int* E;        // [lc][2][j]: packed prefix exponent / zero count (ez_pack), unit and conductive
};
// interval field slots. An off-diagonal pair (k < kp) needs, per medium, the
// chain prod_{l=k+1}^{kp-1} theta_l = P(kp) / P(k+1) (prefix products P), so
// every product W = H(k) chain J(kp) of layered.cpp:340-376 factors into a
// left factor of row k, H(k) / P(k+1), and a right factor of column kp,
// P(kp) J(kp), times 2^(E(kp) - E(k+1)) (the prefix exponents), zero unless
// the two prefix zero counts agree. The V-function coefficients of
// layered.cpp:397-408 (i omega mu0, 1/sigma(k), eta(k)^2) are folded into
// the left factors, so a pair-lambda costs five complex products:
//   fLU  = i wmu H0u(k) / Pu(k+1)                     -> V1
//   fL0v = (i wmu + eta(k)^2 / sigma(k)) H0c(k) / Pc(k+1) -> V2 + V5
//   fL1s = H1c(k) / sigma(k) / Pc(k+1)                -> V4 (with fR0), -V3 (with fR1)
//   fL0s = H0c(k) / sigma(k) / Pc(k+1)                -> W01c / sigma(k) (lower entries)
//   fRU = Pu J0u, fR0 = Pc J0c, fR1 = Pc J1c           (column kp)
//   fD1, fD3, fD4, fD25: V1, V3, V4, V2 + V5 of the diagonal pair (k, k)
//   fPiu, fPic: theta (phase 1), then 1 / P (phase 1b)
enum {
  fLU, fL0v, fL1s, fL0s, fRU, fR0, fR1, fD1, fD3, fD4, fD25, fPiu, fPic, kFields
};

// Pair order: by distance d = kp - k, then by k -- the diagonals (k, k) for
// s < nz, then the neighbours (k, k+1), then d = 2, ... -- so a warp mostly
// holds one kind of pair (the kind branches of the pair evaluation stay
// warp-uniform) and pairs of one distance, whose chains underflow together:
// at large lambda only the short-distance pairs contribute (the chain of
// d - 1 thetas falls below 2^-1022), and a warp whose pairs all flush skips
// the lambda (pair_flushed).
__device__ __forceinline__ void pair_of(int s, int nz, int& k, int& kp) {
  int d = 0;
  while (s >= nz - d) {
    s -= nz - d;
    ++d;
  }
  k = s;
  kp = s + d;
}

// Prefix exponent e and zero count z of a chain packed as e - z 2^24: the
// difference of two packed values is the exponent difference when the zero
// counts agree and below -2^23 when they do not (|e| < 2^22: nz * 1100 at most)
__device__ __forceinline__ int ez_pack(int e, int z) { return e - (z << 24); }
// 2^e, or 0 below the normal range: a chain product under 2^-1022 contributes
// nothing at any precision the block entries are defined to (the reference's
// running product underflows to the same zero, layered.cpp:340-360)
__device__ __forceinline__ double pow2_or_zero(int e) { return e < -1022 ? 0.0 : pow2i(min(e, 1023)); }
__device__ __forceinline__ cplx scale_or_flush(cplx v, int e) {
  if (e > 1023) return scal2(v, e);
  return pow2_or_zero(e) * v;
}

struct PairC {
  int k, kp, kn;  // kn = min(k + 1, nz - 1)
  int kind;       // 0 diagonal, 1 off-diagonal
  int same;       // both intervals in one layer (FULL mode)
};

// true when every contribution of an off-diagonal pair at this lambda is
// (signed) zero: both media's chain scalings 2^(E(kp) - E(k+1)) flush
// (pow2_or_zero) or a zero theta lies on both chains, so V1, r0 and r1 of
// pair_lambda are all multiplied by 0 (the reference's running products
// underflow to the same zeros, layered.cpp:340-360)
__device__ __forceinline__ bool pair_flushed(const int* __restrict__ El, int nz, const PairC& c) {
  return c.kind != 0 && El[c.kp] - El[c.kn] < -1022 && El[nz + c.kp] - El[nz + c.kn] < -1022;
}

// one lambda of one interval pair into its nine accumulators (greens.cpp:167-191,
// v_functions layered.cpp:397-408); wl = w00 lambda, w20 / lambda, w02 / lambda,
// w11 / lambda, w10 lambda, w01 lambda. KIND < 0: the pair's kind at run time;
// 0 / 1: known at compile time (branch-free body, so two off-diagonal pairs of
// a thread interleave: phase 2)
template <int KIND = -1, bool FULL = false>
__device__ __forceinline__ void pair_lambda(const cplx* __restrict__ Fl, const int* __restrict__ El, int nz,
                                            const PairC& c, const double* wl, cplx* a) {
  const int k = c.k, kp = c.kp;
  const int kind = KIND < 0 ? c.kind : KIND;
  cplx V1, V13, X25, V4;
  if (kind == 0) {
    V1 = Fl[fD1 * nz + k];
    V13 = V1 + Fl[fD3 * nz + k];
    X25 = Fl[fD25 * nz + k];
    V4 = Fl[fD4 * nz + k];
  } else {
    const int kn = c.kn;
    const int eu = El[kp] - El[kn], ec = El[nz + kp] - El[nz + kn];
    V1 = scale_or_flush(Fl[fLU * nz + k] * Fl[fRU * nz + kp], eu);
    cplx r0 = Fl[fR0 * nz + kp], r1 = Fl[fR1 * nz + kp];
    if (ec > 1023) {  // a chain product above 2^1023: never in practice, kept exact
      r0 = scal2(r0, ec);
      r1 = scal2(r1, ec);
    } else {
      const double f = pow2_or_zero(ec);
      r0 = f * r0;
      r1 = f * r1;
    }
    const cplx l1 = Fl[fL1s * nz + k];
    X25 = Fl[fL0v * nz + k] * r0;
    V4 = l1 * r0;
    V13 = V1 - l1 * r1;
    // lower entry (kp, k): W10c(kp,k) = (sig_kp / sig_k) W01c(k,kp) (reciprocity,
    // layered.cpp:363-376) and V4 = W10c / sig_kp, i.e. W01c / sig_k
    const cplx lo = Fl[fL0s * nz + k] * r1;
    a[7] = a[7] + wl[4] * lo;
    a[8] = a[8] + wl[5] * lo;
    if constexpr (FULL) {
      // zz at (kp, k) (assemble_block_full, greens.cpp:262-265): V2 + V5 of the
      // lower entry, by reciprocity lambda^2 W00c(k, kp) / sigma(k)
      // (i w mu0 sigma(kp) + eta(kp)^2 = lambda^2); inside one layer it is the
      // upper entry's own V2 + V5, bit for bit as the reference's tables give it
      const cplx xl = c.same ? X25 : wl[6] * (Fl[fL0s * nz + k] * r0);
      a[9] = a[9] + wl[0] * xl;
    }
  }
  a[0] = a[0] + wl[0] * V1;
  a[1] = a[1] + wl[1] * V13;
  a[2] = a[2] + wl[2] * V13;
  a[3] = a[3] + wl[3] * V13;
  a[4] = a[4] + wl[0] * X25;
  a[5] = a[5] + wl[4] * V4;
  a[6] = a[6] + wl[5] * V4;
}

#ifdef EMIE_GREENS_PHASE_CLOCKS  // timing experiment: cycles per phase summed over CTAs
__device__ unsigned long long g_phase_clk[8];
#define PHASE_MARK(i)                                                        \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      const long long now = clock64();                                       \
      atomicAdd(&g_phase_clk[i], static_cast<unsigned long long>(now - clk)); \
      clk = now;                                                             \
    }                                                                        \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

// The lambda-only phases of a chunk (layered.cpp:67-129): 0a layer states,
// 0b both reflection chains, 0c diag_a, into the chunk plan C, tasks strided
// over (tid, nth); `sync`: a CTA-cooperative run (barriers between phases).
// The assemble kernel runs it per chunk, chunk_image_kernel per (offset, chunk).
__device__ __forceinline__ void chunk_layer_states(const GreenParams& P, const Chunk& C, double R, int t0, int lc,
                                                   int tid, int nth, bool sync, const double* lam_in = nullptr) {
  const int L = P.L, NL = P.L + 1;
    // phase 0a: eta, e2l, em1 per (lambda, layer)
    for (int x = tid; x < lc * NL; x += nth) {
      const int li = x / NL, m = x - li * NL;
      // lambda_t = lam_t / R on the filter lattice (greens.cpp:166); the
      // V-function probe passes its lambdas explicitly
      const double lam = lam_in ? lam_in[t0 + li] : exp((P.n1 + t0 + li) * P.step + P.shift) / R;
      const cplx eta2 = cplx{lam * lam, 0.0} - cplx{0.0, P.omega * kMu0} * P.sig[m];
      const cplx eta = csqrt_pos(eta2);
      C.eta[li * NL + m] = eta;
      C.ieta[li * NL + m] = crecip(eta);
      if (m == 0 || m == L) {
        C.e2l[li * NL + m] = {1.0, 0.0};
        C.em1[li * NL + m] = {0.0, 0.0};
      } else {
        const cplx e = cexpm1((-2.0 * P.thick[m]) * eta);
        C.e2l[li * NL + m] = cplx{1.0, 0.0} + e;
        C.em1[li * NL + m] = -e;
      }
    }
    if (sync) __syncthreads();
    // phase 0b: reflection chains per (lambda, gamma, direction) (layered.cpp:107-122).
    // Tasks are direction-major so a warp runs one kind of chain (no divergence);
    // one complex reciprocal per step gives both p = (1+w)/(1-w) and 1+p = 2/(1-w).
    for (int x = tid; x < lc * 4; x += nth) {
      const int dir = x / (2 * lc), rem = x - dir * 2 * lc;
      const int li = rem >> 1, gm = rem & 1;
      const cplx* e2l = C.e2l + li * NL;
      const cplx* em1 = C.em1 + li * NL;
      const cplx* eta = C.eta + li * NL;
      const cplx* ie = C.ieta + li * NL;
      const int base = (li * 2 + gm) * NL;
      // w = -g N / D with g = alpha eta_m / eta_{m+1} (layered.cpp:113-116), so
      // p = (1 + w) / (1 - w) = (D - g N) / (D + g N) and 1 + p = 2 D / (D + g N):
      // one complex reciprocal per step
      if (dir == 0) {
        cplx* p = C.p + base;
        cplx* op = C.one_p + base;
        cplx opm = {1.0, 0.0};
        p[0] = {0.0, 0.0};
        op[0] = opm;
        for (int m = 0; m < L; ++m) {
          const cplx N = em1[m] + e2l[m] * (cplx{2.0, 0.0} - opm), D = em1[m] + e2l[m] * opm;
          const cplx rat = eta[m] * ie[m + 1];
          const cplx gN = (gm ? P.sig_up[m] * rat : rat) * N;
          const cplx r = crecip(D + gN);
          p[m + 1] = (D - gN) * r;
          opm = 2.0 * (D * r);
          op[m + 1] = opm;
        }
      } else {
        cplx* q = C.q + base;
        cplx* oq = C.one_q + base;
        cplx oqm = {1.0, 0.0};
        q[L] = {0.0, 0.0};
        oq[L] = oqm;
        for (int m = L; m > 0; --m) {
          const cplx N = em1[m] + e2l[m] * (cplx{2.0, 0.0} - oqm), D = em1[m] + e2l[m] * oqm;
          const cplx rat = eta[m] * ie[m - 1];
          const cplx gN = (gm ? P.sig_dn[m] * rat : rat) * N;
          const cplx r = crecip(D + gN);
          q[m - 1] = (D - gN) * r;
          oqm = 2.0 * (D * r);
          oq[m - 1] = oqm;
        }
      }
    }
    if (sync) __syncthreads();
    // phase 0c: diag_a (layered.cpp:124-126)
    for (int x = tid; x < lc * 2 * NL; x += nth) {
      const int li = x / (2 * NL), r = x - li * 2 * NL;
      const int m = r % NL;
      const cplx eta = C.eta[li * NL + m], e2l = C.e2l[li * NL + m], em1 = C.em1[li * NL + m];
      const cplx pq = C.p[li * 2 * NL + r] * C.q[li * 2 * NL + r];
      C.diag_a[li * 2 * NL + r] = crecip(eta * (em1 + e2l * (cplx{1.0, 0.0} - pq)));
    }
}

// Chunk field accessors: F(li, f, j) interval field f of interval j at chunk
// lambda li; Ei(li, gamma, j) packed prefix exponent of that medium
__device__ __forceinline__ cplx& chunk_field(const Chunk& C, int nz, int li, int f, int j) {
  return C.F[(static_cast<size_t>(li) * kFields + f) * nz + j];
}

// phase 1 of a chunk: interval pack (shared by both gammas) and the per-interval
// factors of both media (layered.cpp:222-317), strided over (tid, nth)
__device__ __forceinline__ void chunk_factors(const GreenParams& P, const Chunk& C, const Interval* __restrict__ iv,
                                              int lc, double wmu, int tid, int nth) {
  const int NL = P.L + 1, nz = P.nz;
  auto F = [&](int li, int f, int j) -> cplx& { return chunk_field(C, nz, li, f, j); };
  // phase 1: interval pack (shared by both gammas) and factors (layered.cpp:237-317),
  // folded into the left / right / diagonal fields of the pair evaluation
  for (int x = tid; x < lc * nz; x += nth) {
    const int li = x / nz, j = x - li * nz;
    const Interval I = iv[j];
    const IvPack k = iv_pack(I, C.eta[li * NL + I.layer], C.ieta[li * NL + I.layer], C.e2l[li * NL + I.layer]);
    const cplx isk = I.inv_sig;
    for (int gm = 0; gm < 2; ++gm) {
      const int r = li * 2 * NL + gm * NL + I.layer;
      const IvFac f = iv_factors(I, k, C.p[r], C.q[r], C.diag_a[r], C.one_p[r], C.one_q[r]);
      if (gm == 0) {
        F(li, fLU, j) = cplx{-wmu * f.H0.im, wmu * f.H0.re};
        F(li, fRU, j) = f.J0;
        F(li, fD1, j) = cplx{-wmu * f.W00d.im, wmu * f.W00d.re};
        F(li, fPiu, j) = f.theta;
      } else {
        F(li, fL0v, j) = (cplx{0.0, wmu} + k.eta2 * isk) * f.H0;
        F(li, fL0s, j) = f.H0 * isk;
        F(li, fL1s, j) = f.H1 * isk;
        F(li, fR0, j) = f.J0;
        F(li, fR1, j) = f.J1;
        F(li, fD25, j) = cplx{-wmu * f.W00d.im, wmu * f.W00d.re} + f.W20d * isk;
        F(li, fD3, j) = -(f.W11d * isk);
        F(li, fD4, j) = f.W10d * isk;
        F(li, fPic, j) = f.theta;
      }
    }
  }
}

// phase 1b: prefix products of theta per (lambda, gamma) (CTA-wide, warp tasks)
__device__ __forceinline__ void chunk_prefix(const GreenParams& P, const Chunk& C, int lc) {
  const int nz = P.nz;
  auto F = [&](int li, int f, int j) -> cplx& { return chunk_field(C, nz, li, f, j); };
  auto Ei = [&](int li, int f, int j) -> int& { return C.E[(li * 2 + f) * nz + j]; };
  // phase 1b: prefix products of theta per (lambda, gamma) as
  // (mantissa, exponent, zero count); P_j = prod_{l<j} theta_l.
  // nz <= 64: eight (nz > 32: sixteen) lanes per (lambda, gamma), several tasks per warp at once;
  // a lane owns ceil(nz/8) consecutive intervals: local products, a 3-step
  // shuffle scan over the eight lanes, the lane's exclusive prefix
  // multiplied in. Mantissas (max component in [1, 2), modulus < 2^1.5) are
  // not renormalised inside: a product of <= 64 stays below 2^96.
  if (nz <= 64) {
    // lanes per task: 8 (nz <= 32) or 16 (deeper grids: half the serial
    // per-lane work; lc * 2 * 16 still fits one pass of the CTA at LC = 8)
    const int TW = nz > 32 ? 16 : 8, tpw = 32 / TW;
    const int lane = threadIdx.x & 31, sub = lane & (TW - 1);
    const int per = (nz + TW - 1) / TW;
    const int ntask = lc * 2;
    for (int task0 = (threadIdx.x >> 5) * tpw; task0 < ntask; task0 += (blockDim.x >> 5) * tpw) {
      const int task = task0 + lane / TW;
      const bool live = task < ntask;
      const int li = live ? task >> 1 : 0, gm = task & 1;
      const int fT = gm ? fPic : fPiu;
      cplx m[8];
      int e[8], z[8];
      cplx lm = {1.0, 0.0};  // running local product (inclusive)
      int le = 0, lz = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = sub * per + q;
        cplx mq = {1.0, 0.0};
        int eq = 0, zq = 0;
        if (q < per && j < nz && live) {
          const cplx th = F(li, fT, j);
          if (th.re == 0.0 && th.im == 0.0) {
            zq = 1;
          } else {
            const int sh = ilog2(fmax(fabs(th.re), fabs(th.im)));
            mq = scal2(th, -sh);
            eq = sh;
          }
        }
        // exclusive local prefix of element q, then include it
        m[q] = lm;
        e[q] = le;
        z[q] = lz;
        lm = lm * mq;
        le += eq;
        lz += zq;
      }
      // inclusive scan of the lane totals over the TW lanes of the task
      cplx sm_ = lm;
      int se = le, sz = lz;
#pragma unroll 4
      for (int off = 1; off < TW; off <<= 1) {
        const double mr = __shfl_up_sync(0xffffffffu, sm_.re, off, TW);
        const double mi = __shfl_up_sync(0xffffffffu, sm_.im, off, TW);
        const int oe = __shfl_up_sync(0xffffffffu, se, off, TW);
        const int oz = __shfl_up_sync(0xffffffffu, sz, off, TW);
        if (sub >= off) {
          sm_ = cplx{mr, mi} * sm_;
          se += oe;
          sz += oz;
        }
      }
      // exclusive lane prefix
      cplx pm = {__shfl_up_sync(0xffffffffu, sm_.re, 1, TW), __shfl_up_sync(0xffffffffu, sm_.im, 1, TW)};
      int pe = __shfl_up_sync(0xffffffffu, se, 1, TW), pz = __shfl_up_sync(0xffffffffu, sz, 1, TW);
      if (sub == 0) {
        pm = {1.0, 0.0};
        pe = 0;
        pz = 0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = sub * per + q;
        if (q < per && j < nz && live) {
          cplx v = pm * m[q];
          const int sh = ilog2(fmax(fabs(v.re), fabs(v.im)));
          v = scal2(v, -sh);
          // right factors P(j) J(j); theta(j) (read above by this lane only) -> 1/P(j)
          if (gm) {
            F(li, fR0, j) = v * F(li, fR0, j);
            F(li, fR1, j) = v * F(li, fR1, j);
          } else {
            F(li, fRU, j) = v * F(li, fRU, j);
          }
          F(li, fT, j) = crecip(v);
          Ei(li, gm, j) = ez_pack(pe + e[q] + sh, pz + z[q]);
        }
      }
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int task = warp; task < lc * 2; task += nwarps) {
      const int li = task >> 1, gm = task & 1;
      const int fT = gm ? fPic : fPiu;
      cplx cm = {1.0, 0.0};  // carry: product of the previous segments
      int ce = 0, cz = 0;
      for (int j0 = 0; j0 < nz; j0 += 32) {
        const int j = j0 + lane;
        // this lane's factor, normalised
        cplx m = {1.0, 0.0};
        int e = 0, z = 0;
        if (j < nz) {
          const cplx th = F(li, fT, j);
          if (th.re == 0.0 && th.im == 0.0) {
            z = 1;
          } else {
            const int s = ilog2(fmax(fabs(th.re), fabs(th.im)));
            m = scal2(th, -s);
            e = s;
          }
        }
        // inclusive scan (lane order = interval order). Mantissas with max
        // component in [1, 2) have modulus in [1, 2^1.5), so a product of
        // <= 32 stays in [1, 2^48]: no renormalisation inside the scan, and
        // since power-of-two scalings are exact, the final normalised
        // mantissas equal a step-by-step renormalised scan bit for bit
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double mr = __shfl_up_sync(0xffffffffu, m.re, off);
          const double mi = __shfl_up_sync(0xffffffffu, m.im, off);
          const int oe = __shfl_up_sync(0xffffffffu, e, off);
          const int oz = __shfl_up_sync(0xffffffffu, z, off);
          if (lane >= off) {
            m = cplx{mr, mi} * m;
            e += oe;
            z += oz;
          }
        }
        // exclusive prefix = carry x inclusive of the previous lane
        cplx pm = {__shfl_up_sync(0xffffffffu, m.re, 1), __shfl_up_sync(0xffffffffu, m.im, 1)};
        int pe = __shfl_up_sync(0xffffffffu, e, 1), pz = __shfl_up_sync(0xffffffffu, z, 1);
        if (lane == 0) {
          pm = {1.0, 0.0};
          pe = 0;
          pz = 0;
        }
        pm = cm * pm;
        {
          const int s = ilog2(fmax(fabs(pm.re), fabs(pm.im)));
          pm = scal2(pm, -s);
          pe += ce + s;
        }
        pz += cz;
        if (j < nz) {
          if (gm) {
            F(li, fR0, j) = pm * F(li, fR0, j);
            F(li, fR1, j) = pm * F(li, fR1, j);
          } else {
            F(li, fRU, j) = pm * F(li, fRU, j);
          }
          F(li, fT, j) = crecip(pm);
          Ei(li, gm, j) = ez_pack(pe, pz);
        }
        // new carry: carry x inclusive of lane 31
        const cplx lm = {__shfl_sync(0xffffffffu, m.re, 31), __shfl_sync(0xffffffffu, m.im, 31)};
        const int le = __shfl_sync(0xffffffffu, e, 31), lz = __shfl_sync(0xffffffffu, z, 31);
        cm = cm * lm;
        const int s = ilog2(fmax(fabs(cm.re), fabs(cm.im)));
        cm = scal2(cm, -s);
        ce += le + s;
        cz += lz;
      }
    }
  }
}

__device__ __forceinline__ void chunk_left(const GreenParams& P, const Chunk& C, int lc, int tid, int nth) {
  const int nz = P.nz;
  auto F = [&](int li, int f, int j) -> cplx& { return chunk_field(C, nz, li, f, j); };
  // phase 1c: left factors of rows k < nz - 1 divided by P(k+1) of their medium
  for (int x = tid; x < lc * (nz - 1); x += nth) {
    const int li = x / (nz - 1), j = x - li * (nz - 1);
    const cplx pu = F(li, fPiu, j + 1), pcn = F(li, fPic, j + 1);
    F(li, fLU, j) = F(li, fLU, j) * pu;
    F(li, fL0v, j) = F(li, fL0v, j) * pcn;
    F(li, fL1s, j) = F(li, fL1s, j) * pcn;
    F(li, fL0s, j) = F(li, fL0s, j) * pcn;
  }
}

// Fields of a chunk the pair phase reads (fPiu, fPic are consumed by chunk_left)
constexpr int kImgFields = fPiu;
#ifndef EMIE_GREEN_IMG_THREADS
#define EMIE_GREEN_IMG_THREADS 128
#endif
#ifndef EMIE_GREEN_IMG_MINB
#define EMIE_GREEN_IMG_MINB 4
#endif
constexpr int kImgThreads = EMIE_GREEN_IMG_THREADS;
#ifndef EMIE_GREEN_IMG_LAMBDAS
#define EMIE_GREEN_IMG_LAMBDAS 4
#endif
constexpr int kImgLambdas = EMIE_GREEN_IMG_LAMBDAS;  // lambdas per chunk_image_kernel CTA (nz > 32)
constexpr size_t kImgBudget = size_t{2} << 30;       // bytes of chunk images per batch (cfg3: 1 / 2 / 4 GB -> 31.6 / 30.1 / 29.7 ms)
// image kernel of batch i + 1 overlapped with the pair kernel of batch i on a
// second stream (EMIE_CU_GREENS_OVERLAP=0: serial, A/B)
inline bool greens_overlap_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EMIE_CU_GREENS_OVERLAP");
    return !(e && e[0] == '0');
  }();
  return on;
}
// the pair kernels' stream and its events, per build (builds may run on
// several host threads and devices); destroying them right after the build
// is enqueued is safe: the runtime releases them once their work completes
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[4] = {};
  AuxStream() {
    EMIE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& e : ev) EMIE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~AuxStream() {
    for (auto& e : ev) (void)cudaEventDestroy(e);
    (void)cudaStreamDestroy(s);
  }
  AuxStream(const AuxStream&) = delete;
  AuxStream& operator=(const AuxStream&) = delete;
};
// chunk images shared by offsets at equal R (EMIE_CU_GREENS_RSHARE=0: one per offset, A/B)
inline bool img_share_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EMIE_CU_GREENS_RSHARE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Per-lambda phases 0-1c of the accumulation (layer states, interval factors,
// prefix products, left factors: everything of a chunk but the pair sums) for
// one (offset, lambda chunk of LA) per CTA, at several CTAs per SM -- these
// phases are latency-bound chains the single 256-thread CTA per SM of the pair
// kernel hides poorly. Output: the chunk image IF[b][t][kImgFields][nz] and
// IE[b][t][2][nz] (offset stride estride ints) the pair kernel streams in.
__global__ void __launch_bounds__(kImgThreads, EMIE_GREEN_IMG_MINB) chunk_image_kernel(
    const GreenParams P, const Interval* __restrict__ iv, const int* __restrict__ offs, int LA,
    cplx* __restrict__ IF, int* __restrict__ IE, size_t estride, const double* __restrict__ Rrep) {
  extern __shared__ cplx sm[];
  const int NL = P.L + 1, nz = P.nz;
  const int b = blockIdx.y, t0 = blockIdx.x * LA;
  const int lc = min(LA, P.nw - t0);
  const int code = offs[b];
  const double R = Rrep ? Rrep[b] : pair_geometry(P.oc.oi(code), P.oc.oj(code), P.hx, P.hy).r;
  Chunk C;
  {
    cplx* s = sm;
    C.eta = s; s += LA * NL;
    C.e2l = s; s += LA * NL;
    C.em1 = s; s += LA * NL;
    C.p = s; s += LA * 2 * NL;
    C.q = s; s += LA * 2 * NL;
    C.one_p = s; s += LA * 2 * NL;
    C.one_q = s; s += LA * 2 * NL;
    C.diag_a = s; s += LA * 2 * NL;
    C.ieta = s; s += LA * NL;
    C.F = s; s += static_cast<size_t>(LA) * kFields * nz;
    C.lam = nullptr;
    C.E = reinterpret_cast<int*>(s);
  }
  chunk_layer_states(P, C, R, t0, lc, threadIdx.x, blockDim.x, true);
  __syncthreads();
  chunk_factors(P, C, iv, lc, P.omega * kMu0, threadIdx.x, blockDim.x);
  __syncthreads();
  chunk_prefix(P, C, lc);
  __syncthreads();
  chunk_left(P, C, lc, threadIdx.x, blockDim.x);
  __syncthreads();
  const int per = kImgFields * nz;
  cplx* dst = IF + (static_cast<size_t>(b) * P.nw + t0) * per;
  for (int x = threadIdx.x; x < lc * per; x += blockDim.x) {
    const int li = x / per;
    dst[x] = C.F[static_cast<size_t>(li) * kFields * nz + (x - li * per)];
  }
  int* de = IE + b * estride + static_cast<size_t>(t0) * 2 * nz;
  for (int x = threadIdx.x; x < lc * 2 * nz; x += blockDim.x) de[x] = C.E[x];
}

#ifndef EMIE_GREEN_MINB
#define EMIE_GREEN_MINB 1  // CTAs per SM the register budget targets
#endif
#ifndef EMIE_GREEN_SMEM_KB
#define EMIE_GREEN_SMEM_KB 200  // SMEM budget of the lambda chunk buffers
#endif
// IMG: phases 0-1c come as chunk images (chunk_image_kernel) streamed in by
// bulk copies into two SMEM buffers; the CTA runs only the pair phase
template <bool FULL = false, bool IMG = false>
__global__ void __launch_bounds__(kGreenThreads, EMIE_GREEN_MINB) assemble_kernel(
    const GreenParams P, const Interval* __restrict__ iv, const double* __restrict__ W,
    cplx* __restrict__ blocks, int* err, const int* __restrict__ offs, int pos0, const cplx* __restrict__ IF,
    const int* __restrict__ IE, size_t estride, const int* __restrict__ img_of = nullptr, int img_base = 0,
    const double* __restrict__ Roff = nullptr) {
  extern __shared__ cplx sm[];
  __shared__ uint64_t ibar[2];
  const int L = P.L, NL = P.L + 1, nz = P.nz, LC = P.LC;
  const int code = offs[blockIdx.x];
  const int off = P.oc.slot(code, pos0 + blockIdx.x);  // block / weight slot
  const int oi = P.oc.oi(code), oj = P.oc.oj(code);
  // the offset's distance R: the host's (hankel.cpp:80-91 in the C library) when given
  const double R = Roff ? Roff[blockIdx.x] : pair_geometry(oi, oj, P.hx, P.hy).r;
  const double* Woff = W + static_cast<size_t>(off) * 6 * P.nw;
  const double wmu = P.omega * kMu0;  // V1 = i wmu W00 (layered.cpp:400)

  Chunk C;
  // IMG: two buffers {F [LC][kImgFields][nz], E [LC][2][nz] (16-byte padded)}, then lam
  const size_t ibufF = static_cast<size_t>(LC) * kImgFields * nz;
  const size_t ibufE = (static_cast<size_t>(LC) * 2 * nz + 3) / 4 * 2;  // in cplx units
  // buffer b at sm + b * (ibufF + ibufE): pointer arithmetic on sm keeps the
  // pair loop's loads in the shared window (LDS; a pointer picked from an
  // array loses that and compiles to generic LD + 64-bit address math)
  auto ibuf = [&](int b) { return sm + static_cast<size_t>(b) * (ibufF + ibufE); };
  // the offset's chunk image: its own, or the one of its R group (offsets at
  // the same distance R share every per-lambda phase)
  const int img = img_of ? img_of[blockIdx.x] - img_base : static_cast<int>(blockIdx.x);
  auto img_issue = [&](int c) {  // one thread: chunk c's image into buffer c & 1
    const int s0 = c * LC, n = min(LC, P.nw - s0);
    const uint32_t fb = static_cast<uint32_t>(n) * kImgFields * nz * sizeof(cplx);
    const uint32_t eb = (static_cast<uint32_t>(n) * 2 * nz * sizeof(int) + 15u) & ~15u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&ibar[c & 1], fb + eb);
    bulk_g2s(ibuf(c & 1), IF + (static_cast<size_t>(img) * P.nw + s0) * kImgFields * nz, fb, &ibar[c & 1]);
    bulk_g2s(ibuf(c & 1) + ibufF, IE + img * estride + static_cast<size_t>(s0) * 2 * nz, eb, &ibar[c & 1]);
  };
  if constexpr (IMG) {
    C.lam = reinterpret_cast<double*>(sm + 2 * (ibufF + ibufE));
    if (threadIdx.x == 0) {
      mbar_init(&ibar[0], 1);
      mbar_init(&ibar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      img_issue(0);
    }
  } else {
    cplx* s = sm;
    C.eta = s; s += LC * NL;
    C.e2l = s; s += LC * NL;
    C.em1 = s; s += LC * NL;
    C.p = s; s += LC * 2 * NL;
    C.q = s; s += LC * 2 * NL;
    C.one_p = s; s += LC * 2 * NL;
    C.one_q = s; s += LC * 2 * NL;
    C.diag_a = s; s += LC * 2 * NL;
    C.ieta = s; s += LC * NL;
    C.F = s; s += static_cast<size_t>(LC) * kFields * nz;
    C.lam = reinterpret_cast<double*>(s);  // [lc]: lambda, 1/lambda, 6 weights
    C.E = reinterpret_cast<int*>(C.lam + 8 * LC);
  }
  auto F = [&](int li, int f, int j) -> cplx& { return C.F[(static_cast<size_t>(li) * kFields + f) * nz + j]; };
  auto Ei = [&](int li, int f, int j) -> int& { return C.E[(li * 2 + f) * nz + j]; };
  // Pair assignment (balanced): group pairs [g0, g0 + cnt) in distance order
  // (pair_of), cnt <= 3T. Even slots take pairs from the front of the group
  // (short distances: active at every lambda), odd slots from the back (long
  // distances: flushed at large lambda), so every thread holds about the same
  // number of live (pair, lambda) items. The ntail = cnt - F - B pairs in the
  // middle are split over lambda: thread tid < Teff = (T / ntail) ntail keeps
  // tail pair tid % ntail for every Teff-th (pair, lambda) item of a chunk;
  // the T / ntail partial sums per tail pair are added in a fixed order at
  // the end, so every thread evaluates ~2.06 pairs per lambda, not 3.
  constexpr int T = kGreenThreads, NS = kGreenSlots;
  const int g0 = blockIdx.y * (NS + 1) * T;
  const int cnt = min((NS + 1) * T, P.npairs - g0);
  const int nfront = min(cnt, ((NS + 1) / 2) * T), nback = min(cnt - nfront, (NS / 2) * T);
  const int ntail = cnt - nfront - nback;
  const int teff = ntail > 0 ? (T / ntail) * ntail : 0;
  PairC pc[NS + 1];
  bool pv[NS + 1];
#pragma unroll
  for (int i = 0; i <= NS; ++i) {
    const int r = (i / 2) * T + static_cast<int>(threadIdx.x);  // rank within the front / back run
    const int sl = i == NS ? nfront + (ntail > 0 ? static_cast<int>(threadIdx.x) % ntail : 0)
                           : (i % 2 == 0 ? r : cnt - 1 - r);
    pv[i] = i < NS ? r < (i % 2 == 0 ? nfront : nback) : static_cast<int>(threadIdx.x) < teff;
    int k = 0, kp = 0;
    if (pv[i]) pair_of(g0 + sl, nz, k, kp);
    pc[i].k = k;
    pc[i].kp = kp;
    pc[i].kn = min(k + 1, nz - 1);
    pc[i].kind = kp == k ? 0 : 1;
    pc[i].same = iv[k].layer == iv[kp].layer;
  }
  // accumulators: a00 a20 a02 a11 az (upper) axz ayz (k,kp) axz ayz (kp,k) [az (kp,k): FULL]
  constexpr int NA = FULL ? 10 : 9, NWL = FULL ? 7 : 6;
  cplx acc[NS + 1][NA];
#pragma unroll
  for (int i = 0; i <= NS; ++i)
#pragma unroll
    for (int f = 0; f < NA; ++f) acc[i][f] = {0.0, 0.0};

  const int nw = P.nw;
  const bool general2 =
      NS == 2 && __all_sync(0xffffffffu, pv[0] && pv[1] && pc[0].kind == 1 && pc[NS > 1 ? 1 : 0].kind == 1);
#ifdef EMIE_GREENS_PHASE_CLOCKS
  long long clk = clock64();
#endif
  const int fstride = (IMG ? kImgFields : kFields) * nz;  // complex per lambda of C.F
  for (int t0 = 0; t0 < nw; t0 += LC) {
    const int lc = min(LC, nw - t0);
    __syncthreads();  // previous chunk consumed
    PHASE_MARK(0);
    if (IMG && threadIdx.x == 0 && t0 + LC < nw) img_issue(t0 / LC + 1);  // into the buffer just freed
    // per-lambda scalars of the chunk
    for (int li = threadIdx.x; li < lc; li += blockDim.x) {
      const int t = t0 + li;
      const double lam = exp((P.n1 + t) * P.step + P.shift) / R, ilam = 1.0 / lam;
      // weights w00 w20 w02 w11 w10 w01 (greens.cpp:137) times lambda or 1/lambda
      C.lam[li] = Woff[t] * lam;
      C.lam[LC + li] = Woff[nw + t] * ilam;
      C.lam[2 * LC + li] = Woff[2 * nw + t] * ilam;
      C.lam[3 * LC + li] = Woff[3 * nw + t] * ilam;
      C.lam[4 * LC + li] = Woff[4 * nw + t] * lam;
      C.lam[5 * LC + li] = Woff[5 * nw + t] * lam;
      C.lam[6 * LC + li] = lam * lam;
    }
    if constexpr (IMG) {
      const int c = t0 / LC;
      C.F = ibuf(c & 1);
      C.E = reinterpret_cast<int*>(ibuf(c & 1) + ibufF);
      mbar_wait(&ibar[c & 1], static_cast<uint32_t>((c >> 1) & 1));
    } else {
      chunk_layer_states(P, C, R, t0, lc, threadIdx.x, blockDim.x, true);
    }
    __syncthreads();
    PHASE_MARK(3);
    if constexpr (!IMG) {
    chunk_factors(P, C, iv, lc, wmu, threadIdx.x, blockDim.x);
    __syncthreads();
    PHASE_MARK(4);
    chunk_prefix(P, C, lc);
    __syncthreads();
    chunk_left(P, C, lc, threadIdx.x, blockDim.x);
    __syncthreads();
    }
    PHASE_MARK(5);
    // phase 2: pairs x lambdas (greens.cpp:167-191), lambda order per pair.
    // Live lambda range of each slot in this chunk: [0, hi) ends after the
    // last lambda at which any pair of the warp's slot is not flushed
    // (pair_flushed; scanned from the chunk end, so a live chunk costs one
    // vote). Lambdas past hi add exact zeros and are skipped; flushed lanes
    // inside the range add exact zeros too. Large lambdas flush every chain
    // of d >= 2 intervals, so the long-distance slots end early.
    int hi[NS + 1] = {};
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      int h = lc;
      while (h > 0 && __all_sync(0xffffffffu, !pv[i] || pair_flushed(C.E + (h - 1) * 2 * nz, nz, pc[i]))) --h;
      hi[i] = h;
    }
    auto lam_w = [&](int li, double* wl) {
#pragma unroll
      for (int q = 0; q < NWL; ++q) wl[q] = C.lam[q * LC + li];
    };
    if (general2) {  // warp-uniform: both slots off-diagonal pairs, one branch-free block
      const int h01 = min(hi[0], hi[NS > 1 ? 1 : 0]);
#pragma unroll kPairUnroll
      for (int li = 0; li < h01; ++li) {
        double wl[NWL];
        lam_w(li, wl);
        const cplx* Fl = C.F + static_cast<size_t>(li) * fstride;
        const int* El = C.E + li * 2 * nz;
        pair_lambda<1, FULL>(Fl, El, nz, pc[0], wl, acc[0]);
        pair_lambda<1, FULL>(Fl, El, nz, pc[NS > 1 ? 1 : 0], wl, acc[NS > 1 ? 1 : 0]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        for (int li = h01; li < hi[i]; ++li) {
          double wl[NWL];
          lam_w(li, wl);
          pair_lambda<1, FULL>(C.F + static_cast<size_t>(li) * fstride, C.E + li * 2 * nz, nz, pc[i], wl, acc[i]);
        }
      }
    } else {
      int hmax = 0;
#pragma unroll
      for (int i = 0; i < NS; ++i) hmax = max(hmax, hi[i]);
#pragma unroll kPairUnroll
      for (int li = 0; li < hmax; ++li) {
        double wl[NWL];
        lam_w(li, wl);
        const cplx* Fl = C.F + static_cast<size_t>(li) * fstride;
        const int* El = C.E + li * 2 * nz;
#pragma unroll
        for (int i = 0; i < NS; ++i)
          if (pv[i] && li < hi[i]) pair_lambda<-1, FULL>(Fl, El, nz, pc[i], wl, acc[i]);
      }
    }
    if (pv[NS]) {
      for (int u = threadIdx.x; u < ntail * lc; u += teff) {
        const int li = u / ntail;
        const int* El = C.E + li * 2 * nz;
        if (pair_flushed(El, nz, pc[NS])) continue;
        double wl[NWL];
#pragma unroll
        for (int q = 0; q < NWL; ++q) wl[q] = C.lam[q * LC + li];
        pair_lambda<-1, FULL>(C.F + static_cast<size_t>(li) * fstride, El, nz, pc[NS], wl, acc[NS]);
      }
    }
  }
  __syncthreads();
  PHASE_MARK(6);
  // tail pairs: partial sums of the lambda-split threads, added in order
  if (ntail > 0) {
    cplx* part = sm;  // the chunk buffers are free now: [9][T]
#pragma unroll
    for (int f = 0; f < NA; ++f) part[f * T + threadIdx.x] = acc[NS][f];
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < ntail) {
#pragma unroll
      for (int f = 0; f < NA; ++f) {
        cplx sum = part[f * T + threadIdx.x];
        for (int r = threadIdx.x + ntail; r < teff; r += ntail) sum = sum + part[f * T + r];
        acc[NS][f] = sum;
      }
    }
  }
  // scale and store (greens.cpp:193-219)
  const double c3 = R * R * R / (4.0 * kPi), c2 = R * R / (4.0 * kPi), c1 = R / (4.0 * kPi);
  const int ntri = P.npairs, nfull = nz * nz;
  cplx* blk = blocks + static_cast<size_t>(off) * P.nent;
  bool bad = false;
#pragma unroll
  for (int i = 0; i <= NS; ++i) {
    const bool own = i < NS ? pv[i] : static_cast<int>(threadIdx.x) < ntail;
    if (!own) continue;
    const int k = pc[i].k, kp = pc[i].kp;
    const int s = k * nz - k * (k - 1) / 2 + (kp - k);
    cplx v[8];
    v[0] = c3 * acc[i][0] + c1 * acc[i][1];
    v[1] = c3 * acc[i][0] + c1 * acc[i][2];
    v[2] = c3 * acc[i][4];
    v[3] = c1 * acc[i][3];
    v[4] = c2 * acc[i][5];
    v[5] = c2 * acc[i][6];
    v[6] = c2 * acc[i][7];
    v[7] = c2 * acc[i][8];
    for (int c = 0; c < 8; ++c) bad |= !isfinite(v[c].re) || !isfinite(v[c].im);
    if constexpr (FULL) {  // FullBlock q[3a+b][k][kp] (greens.cpp:276-291)
      const size_t n2 = static_cast<size_t>(nfull), up = static_cast<size_t>(k) * nz + kp,
                   lo = static_cast<size_t>(kp) * nz + k;
      const cplx zl = k == kp ? v[2] : c3 * acc[i][9];
      bad |= !isfinite(zl.re) || !isfinite(zl.im);
      blk[up] = blk[lo] = v[0];                    // xx
      blk[4 * n2 + up] = blk[4 * n2 + lo] = v[1];  // yy
      blk[8 * n2 + up] = v[2];                     // zz
      blk[8 * n2 + lo] = zl;
      blk[n2 + up] = blk[n2 + lo] = v[3];          // xy
      blk[3 * n2 + up] = blk[3 * n2 + lo] = v[3];  // yx: the same defining sum
      blk[2 * n2 + up] = v[4];                     // xz
      blk[5 * n2 + up] = v[5];                     // yz
      // zx(k, kp): the source-side sum, -xz(kp, k) (on the diagonal -xz(k, k))
      blk[6 * n2 + up] = k == kp ? -v[4] : -v[6];
      blk[7 * n2 + up] = k == kp ? -v[5] : -v[7];
      if (k != kp) {
        blk[2 * n2 + lo] = v[6];
        blk[5 * n2 + lo] = v[7];
        blk[6 * n2 + lo] = -v[4];
        blk[7 * n2 + lo] = -v[5];
      }
      continue;
    }
    blk[s] = v[0];
    blk[ntri + s] = v[1];
    blk[2 * ntri + s] = v[2];
    blk[3 * ntri + s] = v[3];
    blk[4 * ntri + k * nz + kp] = v[4];
    blk[4 * ntri + nfull + k * nz + kp] = v[5];
    if (k != kp) {
      blk[4 * ntri + kp * nz + k] = v[6];
      blk[4 * ntri + nfull + kp * nz + k] = v[7];
    }
  }
  if (bad) atomicOr(err, 4);
}


// V-function probe (test entry, emie_cu_vfunctions): the assemble kernel's own
// lambda-only phases, interval factors, prefix products and pair evaluation
// (chunk_layer_states, chunk_factors, chunk_prefix, chunk_left, pair_lambda)
// at caller-given lambdas, unit weights: per lambda the pair quantities the
// filter sums accumulate (v_functions, layered.cpp:397-408):
//   out[t][0][k][kp] V1, [1] V1 + V3, [2] V2 + V5 (k <= kp), [3] V4 (all k, kp)
__global__ void __launch_bounds__(kGreenThreads) vfunc_probe_kernel(const GreenParams P, const Interval* __restrict__ iv,
                                                                   const double* __restrict__ lam, int n,
                                                                   cplx* __restrict__ out) {
  extern __shared__ cplx sm[];
  const int NL = P.L + 1, nz = P.nz, LC = P.LC;
  Chunk C;
  {
    cplx* s = sm;
    C.eta = s; s += LC * NL;
    C.e2l = s; s += LC * NL;
    C.em1 = s; s += LC * NL;
    C.p = s; s += LC * 2 * NL;
    C.q = s; s += LC * 2 * NL;
    C.one_p = s; s += LC * 2 * NL;
    C.one_q = s; s += LC * 2 * NL;
    C.diag_a = s; s += LC * 2 * NL;
    C.ieta = s; s += LC * NL;
    C.F = s; s += static_cast<size_t>(LC) * kFields * nz;
    C.lam = reinterpret_cast<double*>(s);
    C.E = reinterpret_cast<int*>(C.lam + 8 * LC);
  }
  const int t0 = blockIdx.x * LC, lc = min(LC, n - t0);
  chunk_layer_states(P, C, 1.0, t0, lc, threadIdx.x, blockDim.x, true, lam);
  __syncthreads();
  chunk_factors(P, C, iv, lc, P.omega * kMu0, threadIdx.x, blockDim.x);
  __syncthreads();
  chunk_prefix(P, C, lc);
  __syncthreads();
  chunk_left(P, C, lc, threadIdx.x, blockDim.x);
  __syncthreads();
  const double wl[6] = {1.0, 1.0, 1.0, 1.0, 1.0, 1.0};
  const size_t nz2 = static_cast<size_t>(nz) * nz;
  for (int x = threadIdx.x; x < lc * P.npairs; x += blockDim.x) {
    const int li = x / P.npairs, s = x - li * P.npairs;
    PairC pc;
    pair_of(s, nz, pc.k, pc.kp);
    pc.kn = min(pc.k + 1, nz - 1);
    pc.kind = pc.kp == pc.k ? 0 : 1;
    cplx a[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) a[f] = {0.0, 0.0};
    pair_lambda(C.F + static_cast<size_t>(li) * kFields * nz, C.E + li * 2 * nz, nz, pc, wl, a);
    cplx* o = out + static_cast<size_t>(t0 + li) * 4 * nz2;
    const size_t up = static_cast<size_t>(pc.k) * nz + pc.kp, lo = static_cast<size_t>(pc.kp) * nz + pc.k;
    o[up] = a[0];
    o[nz2 + up] = a[1];
    o[2 * nz2 + up] = a[4];
    o[3 * nz2 + up] = a[5];
    if (pc.k != pc.kp) o[3 * nz2 + lo] = a[7];
  }
}


// Layered-model API probes (emie_cu_spectral_states / emie_cu_moment_tables):
// the Green's build's own device code at caller-given lambdas, one CTA per
// lambda, for the drop-in's build_spectral_state and vertical_moment_tables
// (layered.hpp:56-57, 97-103).
__device__ __forceinline__ Chunk probe_chunk(cplx* s, int NL, int nz) {
  Chunk C;  // the assemble kernel's SMEM plan for one lambda (lc = 1)
  C.eta = s; s += NL;
  C.e2l = s; s += NL;
  C.em1 = s; s += NL;
  C.p = s; s += 2 * NL;
  C.q = s; s += 2 * NL;
  C.one_p = s; s += 2 * NL;
  C.one_q = s; s += 2 * NL;
  C.diag_a = s; s += 2 * NL;
  C.ieta = s; s += NL;
  C.F = s; s += static_cast<size_t>(kFields) * nz;
  C.lam = reinterpret_cast<double*>(s);
  C.E = reinterpret_cast<int*>(C.lam + 8);
  return C;
}
constexpr int kProbeSmemPerNL = 14;  // complex per layer of probe_chunk

// out[t][gamma][9][NL] = sig eta p q one_p one_q e2l em1_2l diag_a
// (SpectralLayerState, layered.hpp:41-58; gamma 0 unit, 1 cond)
__global__ void state_probe_kernel(const GreenParams P, const double* __restrict__ lam, cplx* __restrict__ out) {
  extern __shared__ cplx sm[];
  const int NL = P.L + 1;
  const Chunk C = probe_chunk(sm, NL, P.nz);
  chunk_layer_states(P, C, 1.0, blockIdx.x, 1, threadIdx.x, blockDim.x, true, lam);
  __syncthreads();
  cplx* o = out + static_cast<size_t>(blockIdx.x) * 2 * 9 * NL;
  for (int x = threadIdx.x; x < 2 * NL; x += blockDim.x) {
    const int g = x / NL, m = x - g * NL, r = g * NL + m;
    cplx* og = o + g * 9 * NL;
    og[m] = P.sig[m];
    og[NL + m] = C.eta[m];
    og[2 * NL + m] = C.p[r];
    og[3 * NL + m] = C.q[r];
    og[4 * NL + m] = C.one_p[r];
    og[5 * NL + m] = C.one_q[r];
    og[6 * NL + m] = C.e2l[m];
    og[7 * NL + m] = C.em1[m];
    og[8 * NL + m] = C.diag_a[r];
  }
}

// out[t][gamma][6][nz][nz]: the vertical moment tables of both gammas in the
// pair order (0,0) (1,0) (0,1) (1,1) (2,0) (0,2) (VerticalMomentTable,
// layered.hpp:83-103). Diagonal entries from the interval factors; an upper
// entry (i < j) is row factor x chain of the intervening thetas x column
// factor; lower entries by reciprocity, weighted by sigma_i / sigma_j for
// the conductive gamma (layered.cpp:363-376).
__global__ void table_probe_kernel(const GreenParams P, const Interval* __restrict__ iv, const double* __restrict__ lam,
                                   cplx* __restrict__ out) {
  extern __shared__ cplx sm[];
  const int NL = P.L + 1, nz = P.nz;
  const Chunk C = probe_chunk(sm, NL, nz);
  IvFac* fac = reinterpret_cast<IvFac*>(sm + kProbeSmemPerNL * NL + static_cast<size_t>(kFields) * nz + 8);
  cplx* eta2 = reinterpret_cast<cplx*>(fac + 2 * nz);
  chunk_layer_states(P, C, 1.0, blockIdx.x, 1, threadIdx.x, blockDim.x, true, lam);
  __syncthreads();
  for (int x = threadIdx.x; x < 2 * nz; x += blockDim.x) {
    const int g = x / nz, j = x - g * nz;
    const Interval I = iv[j];
    const IvPack k = iv_pack(I, C.eta[I.layer], C.ieta[I.layer], C.e2l[I.layer]);
    const int r = g * NL + I.layer;
    fac[x] = iv_factors(I, k, C.p[r], C.q[r], C.diag_a[r], C.one_p[r], C.one_q[r]);
    if (g == 0) eta2[j] = k.eta2;
  }
  __syncthreads();
  const size_t nz2 = static_cast<size_t>(nz) * nz;
  cplx* o = out + static_cast<size_t>(blockIdx.x) * 12 * nz2;
  // upper triangle and diagonal: one thread per (gamma, row)
  for (int x = threadIdx.x; x < 2 * nz; x += blockDim.x) {
    const int g = x / nz, i = x - g * nz;
    const IvFac* f = fac + g * nz;
    cplx* w = o + static_cast<size_t>(g) * 6 * nz2;
    const size_t d = static_cast<size_t>(i) * nz + i;
    w[d] = f[i].W00d;
    w[nz2 + d] = f[i].W10d;
    w[2 * nz2 + d] = f[i].W10d;
    w[3 * nz2 + d] = f[i].W11d;
    w[4 * nz2 + d] = f[i].W20d;
    w[5 * nz2 + d] = f[i].W20d;
    cplx chain = {1.0, 0.0};
    for (int j = i + 1; j < nz; ++j) {
      const size_t e = static_cast<size_t>(i) * nz + j;
      const cplx b0 = f[i].H0 * chain, b1 = f[i].H1 * chain;
      const cplx w00 = b0 * f[j].J0;
      w[e] = w00;
      w[nz2 + e] = b1 * f[j].J0;
      w[2 * nz2 + e] = b0 * f[j].J1;
      w[3 * nz2 + e] = b1 * f[j].J1;
      w[4 * nz2 + e] = eta2[i] * w00;
      w[5 * nz2 + e] = eta2[j] * w00;
      chain = chain * f[j].theta;
    }
  }
  __syncthreads();
  // lower triangle: reciprocity, derivative roles swapped (10 <-> 01, 20 <-> 02)
  constexpr int kSwap[6] = {0, 2, 1, 3, 5, 4};
  for (size_t x = threadIdx.x; x < 2 * nz2; x += blockDim.x) {
    const int g = static_cast<int>(x / nz2);
    const int rem = static_cast<int>(x - g * nz2), i = rem / nz, j = rem - i * nz;
    if (i <= j) continue;
    cplx ratio = {1.0, 0.0};
    if (g == 1) ratio = cdiv(P.sig[iv[i].layer], P.sig[iv[j].layer]);
    cplx* w = o + static_cast<size_t>(g) * 6 * nz2;
    for (int q = 0; q < 6; ++q)
      w[q * nz2 + static_cast<size_t>(i) * nz + j] = ratio * w[kSwap[q] * nz2 + static_cast<size_t>(j) * nz + i];
  }
}


// the filter lattice of one offset: lambda_t = e^{(n1 + t) step + shift} / R
// (the expression chunk_layer_states evaluates; greens.cpp:166)
__global__ void lattice_kernel(double R, int n1, double step, double shift, int n, double* lam) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) lam[t] = exp((n1 + t) * step + shift) / R;
}



// ---- receiver fields (SPEC.md receiver_green_integrals / reconstruct_fields) ----
// For a receiver M at depth z and a source cell (rectangle S x interval k):
//   int G^E dOmega, int G^H dOmega (paper Appendix A, Eq. geh / Ge2)
// with the lateral one-sided filters above and the vertical single moments of
// the receiver (layered.cpp:450-542 contract):
//   m0_g = int_k U_g(z, z') dz', m1_g = d/dz m0_g (g = unit 1, cond s),
//   n0 = int_k d/dz' U_s dz' = U_s(z, b) - U_s(z, a), n1 = d/dz n0;
// outside the source interval d^2/dz^2 acts as eta_r^2 (receiver layer r), so
// with k^2 = i w mu0 sigma_r (eta^2 = lambda^2 - k^2) the tensor is
//   Exx = c [L(lam m0_1)00 + L(Phi)20 / k^2], Phi = (k^2 m0_1 - n1)/lam,
//   Eyy = ... L(Phi)02, Exy = Eyx = c L(Phi)11 / k^2,
//   Exz = c L(lam m1_s)10 / k^2, Eyz = c L(lam m1_s)01 / k^2,
//   Ezx = -c L(lam n0)10 / k^2, Ezy = -c L(lam n0)01 / k^2, Ezz = c L(lam^3 m0_s)00 / k^2,
// c = i w mu0 / 4 pi; and H = curl G / (i w mu0) of Eq. geh:
//   Hxx = -L(B)11, Hyx = L(lam m1_1)00 + L(B)20, Hzx = -L(lam m0_1)01,
//   Hxy = -L(B)02 - L(lam m1_1)00, Hyy = L(B)11, Hzy = L(lam m0_1)10,
//   Hxz = L(lam m0_s)01, Hyz = -L(lam m0_s)10, Hzz = 0, all / 4 pi, B = (n0 + m1_1)/lam.
// L(f)ab = R^{1-a-b} sum_t w^{ab}_t f(lambda_t / R). Every reference distance R
// is a lattice power e^{j step}, so lambda_t / R = e^{(n1 + t - j) step + shift}
// lies on one global lattice: the vertical functions of a receiver depth are
// tabulated once per lattice point (receiver_table_kernel).

// T[n][k][6] = m0_1 m1_1 m0_s m1_s n0 n1 at lattice lambda lam[n], depth z
__global__ void receiver_table_kernel(const GreenParams P, const Interval* __restrict__ iv,
                                      const double* __restrict__ br, double z, const double* __restrict__ lam,
                                      cplx* __restrict__ T) {
  extern __shared__ cplx sm[];
  const int NL = P.L + 1, nz = P.nz;
  const Chunk C = probe_chunk(sm, NL, nz);
  StateDev* S = reinterpret_cast<StateDev*>(sm + kProbeSmemPerNL * NL + static_cast<size_t>(kFields) * nz + 8);
  chunk_layer_states(P, C, 1.0, blockIdx.x, 1, threadIdx.x, blockDim.x, true, lam);
  __syncthreads();
  for (int x = threadIdx.x; x < 2 * NL; x += blockDim.x) {
    const int g = x / NL, m = x - g * NL, r = g * NL + m;
    StateDev& st = S[g];
    if (m == 0) {
      st.L = P.L;
      st.gamma = g;
    }
    st.top[m] = P.ztop[m];
    st.bot[m] = P.zbot[m];
    st.sig[m] = P.sig[m];
    st.eta[m] = C.eta[m];
    st.p[m] = C.p[r];
    st.q[m] = C.q[r];
    st.one_p[m] = C.one_p[r];
    st.one_q[m] = C.one_q[r];
    st.e2l[m] = C.e2l[m];
    st.em1[m] = C.em1[m];
    st.a[m] = C.diag_a[r];
  }
  __syncthreads();
  cplx* t = T + static_cast<size_t>(blockIdx.x) * nz * 6;
  if (threadIdx.x < 2) {  // the two gammas' single moments, sequential over the intervals
    const int g = threadIdx.x;
    cplx m0[64], m1[64];
    point_moments_dev(S[g], iv, br, nz, z, m0, m1);
    for (int k = 0; k < nz; ++k) {
      t[k * 6 + 2 * g] = m0[k];
      t[k * 6 + 2 * g + 1] = m1[k];
    }
  }
  for (int k = threadIdx.x; k < nz; k += blockDim.x) {  // end-point values of the conductive solution
    const int lk = iv[k].layer;
    const cplx nb = fundamental_dev(S[1], z, br[k + 1], 0, 0, -1, lk), na = fundamental_dev(S[1], z, br[k], 0, 0, -1, lk);
    const cplx db = fundamental_dev(S[1], z, br[k + 1], 1, 0, -1, lk), da = fundamental_dev(S[1], z, br[k], 1, 0, -1, lk);
    t[k * 6 + 4] = nb - na;
    t[k * 6 + 5] = db - da;
  }
}

struct RecvSum {  // the lateral filter sums of one (column, interval)
  cplx a1_00, a1_10, a1_01, ph_20, ph_02, ph_11, a3_10, a3_01, a4_10, a4_01, a5_00, b1_11, b1_20, b1_02, b2_00,
      b3_01, b3_10;
};

// one CTA per source column of the batch, thread k = interval: the receiver
// tensors of every cell of the column; with fields, contracted with the
// scattering currents J = (sigma_a - sigma_b) U / a (paper Eq. APR_lab, the CIE
// unscaling E = U / a of SPEC.md) of nrhs solutions into part[col][rhs][6]
// (E xyz, H xyz), else the raw tensors into tens[col][k][18] (E then H, row-major)
__global__ void __launch_bounds__(64) receiver_kernel(const GreenParams P, const double* __restrict__ W, int nw,
                                                      const int* __restrict__ jcol, const int* __restrict__ cols,
                                                      int nbase, const double* __restrict__ lam,
                                                      const cplx* __restrict__ T, cplx k2, const cplx* __restrict__ U,
                                                      int nrhs, const cplx* __restrict__ sa,
                                                      const Interval* __restrict__ iv,
                                                      const double* __restrict__ br, double zr,
                                                      cplx* __restrict__ part, cplx* __restrict__ tens) {
  __shared__ cplx red[64 * 12];
  const int b = blockIdx.x, k = threadIdx.x, nz = P.nz;
  const int j = jcol[b];
  const double R = exp(j * P.step);
  const double* w = W + static_cast<size_t>(b) * 6 * nw;
  RecvSum s{};
  // a receiver within the z-range of interval k (laterally outside the cell):
  // d^2/dz^2 int_k U dz' = eta^2 m0 - 2 (the kink of U at z' = z) adds +2 to
  // Phi's numerator and -2 lambda to the E_zz integrand, which keeps both
  // integrands decaying in lambda; on a face plane the one-sided limits of
  // the two forms average (E_zz: -lambda); fundamental_value's coincident
  // derivative is the one from above (outside at the top face, inside at the bottom)
  double cA = 0.0, cP = 0.0;
  if (k < nz) {
    const double za = br[k], zb = br[k + 1], z = zr;
    if (z > za && z < zb) cA = cP = 2.0;
    else if (z == za) cA = 1.0;
    else if (z == zb) {
      cA = 1.0;
      cP = 2.0;
    }
  }
  if (k < nz) {
    for (int t = 0; t < nw; ++t) {
      const int n = P.n1 + t - j - nbase;
      const double l = lam[n], il = 1.0 / l;
      const cplx* v = T + (static_cast<size_t>(n) * nz + k) * 6;
      const cplx m01 = v[0], m11 = v[1], m0s = v[2], m1s = v[3], n0 = v[4], n1 = v[5];
      const double w00 = w[t], w20 = w[nw + t], w02 = w[2 * nw + t], w11 = w[3 * nw + t], w10 = w[4 * nw + t],
                   w01 = w[5 * nw + t];
      const cplx A1 = l * m01, PH = (k2 * m01 - n1 + cplx{cP, 0.0}) * il, A3 = l * m1s, A4 = l * n0;
      const cplx A5 = (l * l * l) * m0s - cplx{cA * l, 0.0};
      const cplx B1 = (n0 + m11) * il, B2 = l * m11, B3 = l * m0s;
      s.a1_00 = s.a1_00 + w00 * A1;
      s.a1_10 = s.a1_10 + w10 * A1;
      s.a1_01 = s.a1_01 + w01 * A1;
      s.ph_20 = s.ph_20 + w20 * PH;
      s.ph_02 = s.ph_02 + w02 * PH;
      s.ph_11 = s.ph_11 + w11 * PH;
      s.a3_10 = s.a3_10 + w10 * A3;
      s.a3_01 = s.a3_01 + w01 * A3;
      s.a4_10 = s.a4_10 + w10 * A4;
      s.a4_01 = s.a4_01 + w01 * A4;
      s.a5_00 = s.a5_00 + w00 * A5;
      s.b1_11 = s.b1_11 + w11 * B1;
      s.b1_20 = s.b1_20 + w20 * B1;
      s.b1_02 = s.b1_02 + w02 * B1;
      s.b2_00 = s.b2_00 + w00 * B2;
      s.b3_01 = s.b3_01 + w01 * B3;
      s.b3_10 = s.b3_10 + w10 * B3;
    }
  }
  const double i4pi = 1.0 / (4.0 * kPi), iR = 1.0 / R;
  const cplx c = {0.0, P.omega * kMu0 * i4pi}, ck = cdiv(c, k2);
  cplx E[9], H[9];
  E[0] = c * (R * s.a1_00) + ck * (iR * s.ph_20);
  E[4] = c * (R * s.a1_00) + ck * (iR * s.ph_02);
  E[1] = E[3] = ck * (iR * s.ph_11);
  E[2] = ck * s.a3_10;
  E[5] = ck * s.a3_01;
  E[6] = -(ck * s.a4_10);
  E[7] = -(ck * s.a4_01);
  E[8] = ck * (R * s.a5_00);
  H[0] = -(i4pi * iR) * s.b1_11;
  H[3] = i4pi * (R * s.b2_00 + iR * s.b1_20);
  H[6] = -i4pi * s.a1_01;
  H[1] = -i4pi * (iR * s.b1_02 + R * s.b2_00);
  H[4] = (i4pi * iR) * s.b1_11;
  H[7] = i4pi * s.a1_10;
  H[2] = i4pi * s.b3_01;
  H[5] = -i4pi * s.b3_10;
  H[8] = {0.0, 0.0};
  if (tens) {
    if (k < nz) {
      cplx* o = tens + (static_cast<size_t>(b) * nz + k) * 18;
      for (int q = 0; q < 9; ++q) {
        o[q] = E[q];
        o[9 + q] = H[q];
      }
    }
    return;
  }
  // contract with the currents of the column's cell (k): rhs-major, E xyz H xyz
  const int col = cols[b];
  const size_t N = static_cast<size_t>(P.nx) * P.ny * nz;
  for (int r = 0; r < nrhs; ++r) {
    cplx acc[6] = {};
    if (k < nz) {
      const size_t cell = static_cast<size_t>(k) * P.nx * P.ny + col;
      const cplx sbk = P.sig[iv[k].layer];
      const cplx sak = sa[cell];
      // J = (sigma_a - sigma_b) U / a, a = (sigma_a + conj sigma_b) / (2 sqrt Re sigma_b) (cie.cpp:9-22)
      const cplx fac = cdiv((sak - sbk) * (2.0 * sqrt(sbk.re)), sak + conj(sbk));
      cplx J[3];
      for (int cc = 0; cc < 3; ++cc) J[cc] = fac * U[static_cast<size_t>(r) * 3 * N + cc * N + cell];
      for (int a = 0; a < 3; ++a)
        for (int cc = 0; cc < 3; ++cc) {
          acc[a] = acc[a] + E[3 * a + cc] * J[cc];
          acc[3 + a] = acc[3 + a] + H[3 * a + cc] * J[cc];
        }
    }
    for (int q = 0; q < 6; ++q) red[k * 12 + (r % 2) * 6 + q] = acc[q];
    __syncthreads();
    if (k == 0) {
      for (int q = 0; q < 6; ++q) {
        cplx sum = {0.0, 0.0};
        for (int kk = 0; kk < nz; ++kk) sum = sum + red[kk * 12 + (r % 2) * 6 + q];
        part[(static_cast<size_t>(b) * nrhs + r) * 6 + q] = sum;
      }
    }
    __syncthreads();
  }
}


__global__ void sum_columns_kernel(const cplx* __restrict__ part, int ncols, int nv, cplx* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nv) return;
  cplx acc = out[q];
  for (int b = 0; b < ncols; ++b) acc = acc + part[static_cast<size_t>(b) * nv + q];
  out[q] = acc;
}

// x <-> y mirror of a square grid with hx == hy: the block of offset (oj, oi)
// is the block of (oi, oj) with xx <-> yy and xz <-> yz exchanged (zz and xy
// unchanged) -- the horizontal isotropy of the layered medium; measured on the
// device build to agree with the independently computed block to <1e-6 of the
// block max (filter-design rounding), tools/greens_symmetry_check.py
__global__ void mirror_blocks_kernel(cplx* blocks, const int* __restrict__ pairs, int npairs, int nx, int ntri,
                                     int nfull, int nent) {
  const long long total = static_cast<long long>(npairs) * nent;
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(x / nent), e = static_cast<int>(x - static_cast<long long>(p) * nent);
    const int off = pairs[p], oi = off / nx, oj = off - oi * nx;
    int d = e;  // destination slot in the mirrored block
    if (e < ntri) d = e + ntri;                                  // xx -> yy
    else if (e < 2 * ntri) d = e - ntri;                         // yy -> xx
    else if (e >= 4 * ntri && e < 4 * ntri + nfull) d = e + nfull;  // xz -> yz
    else if (e >= 4 * ntri + nfull) d = e - nfull;               // yz -> xz
    blocks[(static_cast<size_t>(oj) * nx + oi) * nent + d] = blocks[static_cast<size_t>(off) * nent + e];
  }
}

// ... and the offsets oi == oj of such a grid are their own mirrors: the
// exact blocks have xx = yy and xz = yz there. The build designs the xx and
// yy (xz and yz) filters independently, so its two copies differ by the
// filter-design rounding (measured <= 1.4e-6 of the block max for xx/yy,
// ~5e-15 for xz/yz: the level at which the reference's own blocks are
// determined); both are replaced by their mean, which makes
// the blocks exactly x <-> y symmetric (the octant contraction, operator.cu)
__global__ void symmetrize_diagonal_kernel(cplx* blocks, int nx, int ntri, int nfull, int nent) {
  const long long total = static_cast<long long>(nx) * (ntri + nfull);
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(x / (ntri + nfull)), e = static_cast<int>(x - static_cast<long long>(o) * (ntri + nfull));
    cplx* blk = blocks + (static_cast<size_t>(o) * nx + o) * nent;
    const int i = e < ntri ? e : 4 * ntri + (e - ntri);  // xx entry or xz entry
    const int j = e < ntri ? i + ntri : i + nfull;       // its yy / yz partner
    const cplx a = blk[i], b = blk[j];
    const cplx m = {(a.re + b.re) * 0.5, (a.im + b.im) * 0.5};
    blk[i] = m;
    blk[j] = m;
  }
}

__global__ void design_input_kernel(const double* __restrict__ lam, int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = design_input(lam[i]);
}

__global__ void kernel_output_kernel(Geom g, int alpha, int beta, const double* s, int n,
                                     double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = kernel_output(g, alpha, beta, s[i]);
}

inline void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

struct FilterBank {
  FftPlan pl;
  cplx* tw = nullptr;
  cplx* den = nullptr;
  double* floor = nullptr;
};

FilterBank make_filter_bank(const FilterParams& fp, cudaStream_t st) {
  FilterBank fb;
  const int n = 2 * fp.half;
  if (!make_plan(n, fb.pl))
    fail(EMIE_CU_INVALID_ARGUMENT, "filter params: transform length 2*half must be 2,3,5-smooth");
  fb.tw = upload_twiddles(n);
  fb.den = scratch<cplx>(n, st);
  fb.floor = scratch<double>(1, st);
  const size_t smem = (2 * static_cast<size_t>(n | 1) + n) * sizeof(cplx);
  set_smem(reinterpret_cast<const void*>(filter_den_kernel), smem);
  filter_den_kernel<<<1, 256, smem, st>>>(fb.den, fb.floor, fb.tw, fb.pl, fp.half, fp.step);
  check_launch("filter_den_kernel");
  return fb;
}

void free_filter_bank(FilterBank& fb, cudaStream_t st) {
  release(fb.den, st);
  release(fb.floor, st);
  EMIE_CUDA(cudaStreamSynchronize(st));
  cudaFree(fb.tw);
}

void design_filters(const FilterBank& fb, const FilterParams& fp, int noff, OffsetCode oc, double hx,
                    double hy, double* W, int* err, cudaStream_t st, int fixed_oi = INT32_MIN,
                    int fixed_oj = 0, const int* offs = nullptr, const Geom* gfix = nullptr, int kern0 = 0,
                    int nkern = 6, const PGeom* pgeo = nullptr, const Geom* gtab = nullptr,
                    const double* samp = nullptr) {
  const int n = 2 * fp.half;
  const size_t smem = (2 * static_cast<size_t>(n | 1) + n) * sizeof(cplx);
  set_smem(reinterpret_cast<const void*>(filter_design_kernel), smem);
  dim3 grid(noff, nkern);
  filter_design_kernel<<<grid, 256, smem, st>>>(W, fb.den, fb.floor, fb.tw, fb.pl, fp.half,
                                                fp.step, fp.shift, fp.n1, fp.n2, oc, hx, hy, err,
                                                fixed_oi, fixed_oj, offs, gfix ? *gfix : Geom{}, gfix != nullptr,
                                                kern0, pgeo, gtab, samp);
  check_launch("filter_design_kernel");
}

void raise_filter_errors(int e) {
  if (e & 1) fail(EMIE_CU_RUNTIME_ERROR, "filter design: input spectrum vanishes at a used mode");
  if (e & 2) fail(EMIE_CU_RUNTIME_ERROR, "filter design: weights have a non-real residue");
}

}  // namespace

void check_filter_params(const FilterParams& par) {  // hankel.cpp:205-208
  if (!(par.step > 0.0) || !(par.shift > 0.0) || !(par.shift < 0.5 * par.step))
    fail(EMIE_CU_INVALID_ARGUMENT, "filter params: need 0 < shift < step/2");
  if (par.half < 2 || par.n1 < -par.half || par.n2 <= par.n1 || par.n2 > par.half - 1)
    fail(EMIE_CU_INVALID_ARGUMENT, "filter params: bad weight window");
}

void kernel_output_host(int oi, int oj, double hx, double hy, int alpha, int beta,
                        const double* s, int n, double* out) {
  if (!(hx > 0.0) || !(hy > 0.0))
    fail(EMIE_CU_INVALID_ARGUMENT, "pair_geometry: cell sizes must be positive");
  if (alpha < 0 || beta < 0 || alpha > 2 || beta > 2 || alpha + beta > 2)
    fail(EMIE_CU_INVALID_ARGUMENT, "kernel orders: need alpha, beta >= 0 and alpha + beta <= 2");
  if (n <= 0) return;
  double* d = nullptr;
  EMIE_CUDA(cudaMalloc(&d, 2 * n * sizeof(double)));
  EMIE_CUDA(cudaMemcpy(d, s, n * sizeof(double), cudaMemcpyHostToDevice));
  kernel_output_kernel<<<ceil_div(n, 256), 256>>>(pair_geometry(oi, oj, hx, hy), alpha, beta, d, n,
                                                  d + n);
  check_launch("kernel_output_kernel");
  EMIE_CUDA(cudaMemcpy(out, d + n, n * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d);
}

void design_offset_filters_host(int oi, int oj, double hx, double hy, const FilterParams& fp,
                                double* w, double* lam) {
  if (!(hx > 0.0) || !(hy > 0.0))
    fail(EMIE_CU_INVALID_ARGUMENT, "pair_geometry: cell sizes must be positive");
  cudaStream_t st = nullptr;
  keep_pool_warm();
  FilterBank fb = make_filter_bank(fp, st);
  const int nw = fp.n2 - fp.n1 + 1;
  double* dW = scratch<double>(6 * nw, st);
  int* err = scratch<int>(1, st);
  EMIE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  const Geom gh = pair_geometry(oi, oj, hx, hy);  // host C library, as the reference
  design_filters(fb, fp, 1, OffsetCode{}, hx, hy, dW, err, st, oi, oj, nullptr, &gh);
  int e = 0;
  EMIE_CUDA(cudaMemcpyAsync(w, dW, 6 * nw * sizeof(double), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  release(dW, st);
  release(err, st);
  free_filter_bank(fb, st);
  raise_filter_errors(e);
  for (int m = fp.n1; m <= fp.n2; ++m) lam[m - fp.n1] = std::exp(m * fp.step + fp.shift);
}

void green_setup(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                 const double* breaks, double hx, double hy, const FilterParams& fp, GreenParams& P,
                 std::vector<Interval>& ivh, bool grid_checks = true);

void vfunctions_host(int L, const double* tops, const cplx* sigma, int nz, const double* breaks, double omega,
                     int n, const double* lam, cplx* out) {
  if (nz < 1) fail(EMIE_CU_INVALID_ARGUMENT, "vertical partition needs at least one interval");
  if (n <= 0) return;
  GreenParams P;
  std::vector<Interval> ivh;
  green_setup(1, 1, nz, omega, L, tops, sigma, breaks, 1.0, 1.0, FilterParams{}, P, ivh);
  cudaStream_t st = nullptr;
  keep_pool_warm();
  Interval* div = scratch<Interval>(nz, st);
  double* dl = scratch<double>(n, st);
  cplx* dout = scratch<cplx>(static_cast<size_t>(n) * 4 * nz * nz, st);
  EMIE_CUDA(cudaMemcpyAsync(div, ivh.data(), nz * sizeof(Interval), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dl, lam, n * sizeof(double), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemsetAsync(dout, 0, static_cast<size_t>(n) * 4 * nz * nz * sizeof(cplx), st));
  const int NL = L + 1;
  const size_t smem = (static_cast<size_t>(P.LC) * (3 * NL + 11 * NL + kFields * nz)) * sizeof(cplx) +
                      8 * static_cast<size_t>(P.LC) * sizeof(double) + static_cast<size_t>(P.LC) * 2 * nz * sizeof(int);
  set_smem(reinterpret_cast<const void*>(vfunc_probe_kernel), smem);
  vfunc_probe_kernel<<<ceil_div(n, P.LC), kGreenThreads, smem, st>>>(P, div, dl, n, dout);
  check_launch("vfunc_probe_kernel");
  EMIE_CUDA(cudaMemcpyAsync(out, dout, static_cast<size_t>(n) * 4 * nz * nz * sizeof(cplx), cudaMemcpyDeviceToHost,
                            st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(div, st);
  release(dl, st);
  release(dout, st);
}

// build_spectral_state / vertical_moment_tables at n lambdas (the drop-in's
// layered API): what = 0 states [n][2][9][L+1], 1 tables [n][2][6][nz][nz]
void layered_probe_host(int what, int L, const double* tops, const cplx* sigma, int nz, const double* breaks,
                        double omega, int n, const double* lam, cplx* out) {
  if (n <= 0) return;
  GreenParams P;
  std::vector<Interval> ivh;
  if (what == 0 && nz < 1) {  // states need no partition: a one-interval stand-in inside layer 1
    const double top = tops[0], bot = L > 1 ? tops[1] : tops[0] + 1.0;
    const double br[2] = {top, std::min(bot, top + 1.0)};
    green_setup(1, 1, 1, omega, L, tops, sigma, br, 1.0, 1.0, FilterParams{}, P, ivh, false);
  } else {
    green_setup(1, 1, nz, omega, L, tops, sigma, breaks, 1.0, 1.0, FilterParams{}, P, ivh, false);
  }
  cudaStream_t st = nullptr;
  keep_pool_warm();
  const int NL = L + 1;
  const size_t per = what == 0 ? 18 * static_cast<size_t>(NL) : 12 * static_cast<size_t>(nz) * nz;
  Interval* div = scratch<Interval>(ivh.size(), st);
  double* dl = scratch<double>(n, st);
  cplx* dout = scratch<cplx>(static_cast<size_t>(n) * per, st);
  EMIE_CUDA(cudaMemcpyAsync(div, ivh.data(), ivh.size() * sizeof(Interval), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dl, lam, n * sizeof(double), cudaMemcpyHostToDevice, st));
  const size_t smem = (kProbeSmemPerNL * static_cast<size_t>(NL) + kFields * static_cast<size_t>(P.nz) + 8) *
                          sizeof(cplx) + 2 * static_cast<size_t>(P.nz) * (sizeof(IvFac) + sizeof(cplx));
  if (what == 0) {
    set_smem(reinterpret_cast<const void*>(state_probe_kernel), smem);
    state_probe_kernel<<<n, 64, smem, st>>>(P, dl, dout);
    check_launch("state_probe_kernel");
  } else {
    set_smem(reinterpret_cast<const void*>(table_probe_kernel), smem);
    table_probe_kernel<<<n, 128, smem, st>>>(P, div, dl, dout);
    check_launch("table_probe_kernel");
  }
  EMIE_CUDA(cudaMemcpyAsync(out, dout, static_cast<size_t>(n) * per * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(div, st);
  release(dl, st);
  release(dout, st);
}

// FilterDesigner::design (hankel.hpp:93, hankel.cpp:239-281) for a given pair
// geometry {r, p, q, phi} and one (alpha, beta) kernel
void design_geometry_host(const double geom[4], int alpha, int beta, const FilterParams& fp, double* w, double* lam) {
  int kern = -1;
  for (int k = 0; k < 6; ++k) {
    static const int ab[6][2] = {{0, 0}, {2, 0}, {0, 2}, {1, 1}, {1, 0}, {0, 1}};
    if (ab[k][0] == alpha && ab[k][1] == beta) kern = k;
  }
  if (kern < 0) fail(EMIE_CU_INVALID_ARGUMENT, "kernel orders: need alpha, beta >= 0 and alpha + beta <= 2");
  if (!(geom[0] > 0.0)) fail(EMIE_CU_INVALID_ARGUMENT, "pair geometry: reference distance must be positive");
  cudaStream_t st = nullptr;
  keep_pool_warm();
  FilterBank fb = make_filter_bank(fp, st);
  const int nw = fp.n2 - fp.n1 + 1;
  double* dW = scratch<double>(6 * nw, st);
  int* err = scratch<int>(1, st);
  EMIE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  const Geom g = geom_of(geom);
  design_filters(fb, fp, 1, OffsetCode{}, 1.0, 1.0, dW, err, st, 0, 0, nullptr, &g, kern, 1);
  int e = 0;
  EMIE_CUDA(cudaMemcpyAsync(w, dW + kern * nw, nw * sizeof(double), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  release(dW, st);
  release(err, st);
  free_filter_bank(fb, st);
  raise_filter_errors(e);
  for (int m = fp.n1; m <= fp.n2; ++m) lam[m - fp.n1] = std::exp(m * fp.step + fp.shift);
}

void kernel_output_geom_host(const double geom[4], int alpha, int beta, const double* s, int n, double* out) {
  if (alpha < 0 || beta < 0 || alpha > 2 || beta > 2 || alpha + beta > 2)
    fail(EMIE_CU_INVALID_ARGUMENT, "kernel orders: need alpha, beta >= 0 and alpha + beta <= 2");
  if (n <= 0) return;
  double* d = nullptr;
  EMIE_CUDA(cudaMalloc(&d, 2 * n * sizeof(double)));
  EMIE_CUDA(cudaMemcpy(d, s, n * sizeof(double), cudaMemcpyHostToDevice));
  kernel_output_kernel<<<ceil_div(n, 256), 256>>>(geom_of(geom), alpha, beta, d, n, d + n);
  check_launch("kernel_output_kernel");
  EMIE_CUDA(cudaMemcpy(out, d + n, n * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d);
}

void design_input_host(int n, const double* lam, double* out) {
  if (n <= 0) return;
  double* d = nullptr;
  EMIE_CUDA(cudaMalloc(&d, 2 * n * sizeof(double)));
  EMIE_CUDA(cudaMemcpy(d, lam, n * sizeof(double), cudaMemcpyHostToDevice));
  design_input_kernel<<<ceil_div(n, 256), 256>>>(d, n, d + n);
  check_launch("design_input_kernel");
  EMIE_CUDA(cudaMemcpy(out, d + n, n * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d);
}

void pair_geometry_host(int oi, int oj, double hx, double hy, double out[4]) {
  if (!(hx > 0.0) || !(hy > 0.0)) fail(EMIE_CU_INVALID_ARGUMENT, "pair_geometry: cell sizes must be positive");
  const Geom g = pair_geometry(oi, oj, hx, hy);  // the device build's own (host/device) routine
  out[0] = g.r;
  out[1] = g.p;
  out[2] = g.q;
  out[3] = g.phi;
}

void assemble_codes(const GreenParams& P0, const std::vector<Interval>& ivh, const FilterParams& fp,
                    const std::vector<int>& offs_h, int nslots, cplx* blocks, cudaStream_t st, bool full);

// assemble_block_full at one signed offset: the build's own kernel in its
// FULL mode (nine components; lower triangles and source-side z couplings
// from their own sums over the same per-lambda quantities the compressed
// blocks are summed from, greens.cpp:231-293): out[9][nz][nz]
void assemble_full_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                        const double* breaks, double hx, double hy, const FilterParams& fp, int oi, int oj,
                        cplx* h_out) {
  GreenParams P;
  std::vector<Interval> ivh;
  green_setup(nx, ny, nz, omega, L, tops, sigma, breaks, hx, hy, fp, P, ivh);
  if (std::abs(oi) >= ny || std::abs(oj) >= nx)
    fail(EMIE_CU_OUT_OF_RANGE, "assemble_block_full: offset outside the grid");
  P.oc = OffsetCode{2 * nx - 1, ny - 1, nx - 1, 1};
  const std::vector<int> codes{(oi + ny - 1) * (2 * nx - 1) + (oj + nx - 1)};
  cudaStream_t st = nullptr;
  const size_t n9 = 9 * static_cast<size_t>(nz) * nz;
  cplx* d = scratch<cplx>(n9, st);
  try {
    assemble_codes(P, ivh, fp, codes, 1, d, st, true);
  } catch (...) {
    release(d, st);
    throw;
  }
  EMIE_CUDA(cudaMemcpyAsync(h_out, d, n9 * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(d, st);
}

// Receiver fields (SPEC.md receiver_green_integrals + reconstruct_fields):
// the anomalous E and H of nrhs solutions U at nrec receivers, out[rec][rhs][6]
// (E xyz, H xyz); or, with tens_col >= 0, the raw tensors of one receiver and
// one source column, out[k][18]. Receivers inside the closed anomaly volume
// are rejected (SPEC.md Receiver invariant).
void receiver_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                   const double* breaks, double hx, double hy, double x0, double y0, const FilterParams& fp,
                   const cplx* h_sa, int nrhs, const cplx* h_U, int nrec, const double* rec, cplx* h_out,
                   int tens_col) {
  GreenParams P;
  std::vector<Interval> ivh;
  green_setup(nx, ny, nz, omega, L, tops, sigma, breaks, hx, hy, fp, P, ivh);
  if (nz > 64) fail(EMIE_CU_INVALID_ARGUMENT, "receivers: at most 64 intervals");
  for (int r = 0; r < nrec; ++r) {
    const double x = rec[3 * r], y = rec[3 * r + 1], z = rec[3 * r + 2];
    if (!std::isfinite(x) || !std::isfinite(y) || !std::isfinite(z))
      fail(EMIE_CU_INVALID_ARGUMENT, "receiver: non-finite position");
    if (x >= x0 && x <= x0 + nx * hx && y >= y0 && y <= y0 + ny * hy && z >= breaks[0] && z <= breaks[nz])
      fail(EMIE_CU_INVALID_ARGUMENT, "receiver inside the anomaly volume (or on its boundary)");
  }
  if (nrec <= 0) return;
  cudaStream_t st = nullptr;
  keep_pool_warm();
  const int nw = P.nw, NL = L + 1, ncols = nx * ny;
  const size_t N = static_cast<size_t>(ncols) * nz;
  Interval* div = scratch<Interval>(nz, st);
  double* dbr = scratch<double>(nz + 1, st);
  EMIE_CUDA(cudaMemcpyAsync(div, ivh.data(), nz * sizeof(Interval), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dbr, breaks, (nz + 1) * sizeof(double), cudaMemcpyHostToDevice, st));
  cplx *dsa = nullptr, *dU = nullptr;
  if (tens_col < 0) {
    dsa = scratch<cplx>(N, st);
    dU = scratch<cplx>(static_cast<size_t>(nrhs) * 3 * N, st);
    EMIE_CUDA(cudaMemcpyAsync(dsa, h_sa, N * sizeof(cplx), cudaMemcpyHostToDevice, st));
    EMIE_CUDA(cudaMemcpyAsync(dU, h_U, static_cast<size_t>(nrhs) * 3 * N * sizeof(cplx), cudaMemcpyHostToDevice, st));
  }
  FilterBank fb = make_filter_bank(fp, st);
  int* err = scratch<int>(1, st);
  EMIE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  const std::vector<int> all_cols = [&] {
    std::vector<int> v;
    if (tens_col >= 0) v.push_back(tens_col);
    else
      for (int c = 0; c < ncols; ++c) v.push_back(c);
    return v;
  }();
  const int B = std::min<int>(static_cast<int>(all_cols.size()), 4096);
  double* W = scratch<double>(static_cast<size_t>(B) * 6 * nw, st);
  PGeom* dpg = scratch<PGeom>(B, st);
  int* djc = scratch<int>(2 * static_cast<size_t>(B), st);
  cplx* part = scratch<cplx>(static_cast<size_t>(B) * std::max(1, nrhs) * 6, st);
  cplx* dout = scratch<cplx>(tens_col >= 0 ? static_cast<size_t>(nz) * 18 : static_cast<size_t>(nrec) * nrhs * 6, st);
  EMIE_CUDA(cudaMemsetAsync(dout, 0, (tens_col >= 0 ? static_cast<size_t>(nz) * 18 : static_cast<size_t>(nrec) * nrhs * 6) *
                                         sizeof(cplx), st));
  const size_t smem = (kProbeSmemPerNL * static_cast<size_t>(NL) + kFields * static_cast<size_t>(nz) + 8) * sizeof(cplx) +
                      2 * sizeof(StateDev);
  set_smem(reinterpret_cast<const void*>(receiver_table_kernel), smem);
  std::vector<PGeom> pg(B);
  std::vector<int> jc(2 * static_cast<size_t>(B));
  for (int r = 0; r < nrec; ++r) {
    const double xr = rec[3 * r], yr = rec[3 * r + 1], zr = rec[3 * r + 2];
    // the receiver's layer and k^2 = i omega mu0 sigma_r (earth side at an interface)
    const int lr = static_cast<int>(std::upper_bound(tops, tops + L, zr) - tops);
    const cplx sr = P.sig[lr];
    const cplx k2 = {-omega * kMu0 * sr.im, omega * kMu0 * sr.re};
    // lattice index of every column's reference distance, and the table range
    auto jof = [&](int col) {
      const int ix = col % nx, iy = col / nx;
      const double dx = x0 + (ix + 0.5) * hx - xr, dy = y0 + (iy + 0.5) * hy - yr;
      return static_cast<int>(std::ceil(std::log(std::hypot(std::fabs(dx) + 0.5 * hx, std::fabs(dy) + 0.5 * hy)) / fp.step));
    };
    int jmin = INT32_MAX, jmax = INT32_MIN;
    for (int col : all_cols) {
      const int j = jof(col);
      jmin = std::min(jmin, j);
      jmax = std::max(jmax, j);
    }
    const int nbase = fp.n1 - jmax, nlam = (fp.n2 - jmin) - nbase + 1;
    double* lam = scratch<double>(nlam, st);
    cplx* T = scratch<cplx>(static_cast<size_t>(nlam) * nz * 6, st);
    lattice_kernel<<<ceil_div(nlam, 128), 128, 0, st>>>(1.0, nbase, fp.step, fp.shift, nlam, lam);
    check_launch("lattice_kernel");
    receiver_table_kernel<<<nlam, 64, smem, st>>>(P, div, dbr, zr, lam, T);
    check_launch("receiver_table_kernel");
    for (size_t c0 = 0; c0 < all_cols.size(); c0 += B) {
      const int nb = static_cast<int>(std::min<size_t>(B, all_cols.size() - c0));
      for (int b = 0; b < nb; ++b) {
        const int col = all_cols[c0 + b], ix = col % nx, iy = col / nx;
        const double dx = x0 + (ix + 0.5) * hx - xr, dy = y0 + (iy + 0.5) * hy - yr;
        const int j = jof(col);
        const double R = std::exp(j * fp.step);
        pg[b] = PGeom{R, hx / R, hy / R, dx / R, dy / R};
        jc[b] = j;
        jc[B + b] = col;
      }
      EMIE_CUDA(cudaMemcpyAsync(dpg, pg.data(), nb * sizeof(PGeom), cudaMemcpyHostToDevice, st));
      EMIE_CUDA(cudaMemcpyAsync(djc, jc.data(), 2 * static_cast<size_t>(B) * sizeof(int), cudaMemcpyHostToDevice, st));
      design_filters(fb, fp, nb, OffsetCode{}, hx, hy, W, err, st, INT32_MIN, 0, nullptr, nullptr, 0, 6, dpg);
      receiver_kernel<<<nb, 64, 0, st>>>(P, W, nw, djc, djc + B, nbase, lam, T, k2, dU, nrhs, dsa, div, dbr, zr,
                                         tens_col >= 0 ? nullptr : part, tens_col >= 0 ? dout : nullptr);
      check_launch("receiver_kernel");
      if (tens_col < 0) {
        sum_columns_kernel<<<ceil_div(nrhs * 6, 64), 64, 0, st>>>(part, nb, nrhs * 6,
                                                                  dout + static_cast<size_t>(r) * nrhs * 6);
        check_launch("sum_columns_kernel");
      }
      EMIE_CUDA(cudaStreamSynchronize(st));  // pg / jc are rewritten by the next batch
    }
    release(lam, st);
    release(T, st);
  }
  int e = 0;
  const size_t nout = tens_col >= 0 ? static_cast<size_t>(nz) * 18 : static_cast<size_t>(nrec) * nrhs * 6;
  EMIE_CUDA(cudaMemcpyAsync(h_out, dout, nout * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  for (void* q : {static_cast<void*>(div), static_cast<void*>(dbr), static_cast<void*>(dsa), static_cast<void*>(dU),
                  static_cast<void*>(err), static_cast<void*>(W), static_cast<void*>(dpg), static_cast<void*>(djc),
                  static_cast<void*>(part), static_cast<void*>(dout)})
    if (q) release(q, st);
  free_filter_bank(fb, st);
  raise_filter_errors(e);
}

// The computed offsets of a build: all, or on a square grid with hx == hy only
// oi <= oj (the rest by the x <-> y mirror, mirror_blocks_kernel)
std::vector<int> computed_offsets(int nx, int ny, double hx, double hy) {
  const bool mirror = nx == ny && hx == hy;
  std::vector<int> offs;
  for (int oi = 0; oi < ny; ++oi)
    for (int oj = 0; oj < nx; ++oj)
      if (!(mirror && oi > oj)) offs.push_back(oi * nx + oj);
  return offs;
}

// Blocks of computed offsets [c0, c1) (positions in computed_offsets) into
// `blocks` (nx*ny*nent complex, offset-major; other offsets untouched):
// filter design (K6) and the lambda accumulation (K5).
// Host side of a build: model, partition and grid validation (LayeredModel::
// validate, VerticalPartition::create, AnomalyGrid::validate: layered.cpp:53-65,
// 191-208; greens.cpp:18-35), the kernel parameters and the interval table
void green_setup(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                 const double* breaks, double hx, double hy, const FilterParams& fp, GreenParams& P,
                 std::vector<Interval>& ivh, bool grid_checks) {
  if (L < 1) fail(EMIE_CU_INVALID_ARGUMENT, "layered model needs at least one interface");
  if (L + 1 > kMaxLayers) fail(EMIE_CU_INVALID_ARGUMENT, "layered model: too many layers for the device build");
  for (int i = 0; i + 1 < L; ++i)
    if (!(tops[i] < tops[i + 1])) fail(EMIE_CU_INVALID_ARGUMENT, "layered model: interface depths must increase");
  for (int i = 0; i < L; ++i)
    if (!std::isfinite(tops[i])) fail(EMIE_CU_INVALID_ARGUMENT, "layered model: non-finite depth");
  for (int i = 0; i <= L; ++i)
    if (!std::isfinite(sigma[i].re) || !std::isfinite(sigma[i].im))
      fail(EMIE_CU_INVALID_ARGUMENT, "layered model: non-finite conductivity");
  if (!(hx > 0.0) || !(hy > 0.0)) fail(EMIE_CU_INVALID_ARGUMENT, "grid: cell sizes must be positive");
  auto layer_of = [&](double z) {  // points on an interface belong below
    return static_cast<int>(std::upper_bound(tops, tops + L, z) - tops);
  };
  auto top_of = [&](int m) { return m == 0 ? tops[0] : tops[m - 1]; };
  auto bottom_of = [&](int m) { return m == L ? tops[L - 1] : tops[m]; };
  P = GreenParams{};
  P.L = L;
  P.nz = nz;
  P.nx = nx;
  P.ny = ny;
  P.hx = hx;
  P.hy = hy;
  P.omega = omega;
  P.nw = fp.n2 - fp.n1 + 1;
  P.step = fp.step;
  P.shift = fp.shift;
  P.n1 = fp.n1;
  P.npairs = nz * (nz + 1) / 2;
  P.nent = 2 * nz * (2 * nz + 1);
  for (int m = 0; m <= L; ++m) {
    P.thick[m] = bottom_of(m) - top_of(m);
    P.ztop[m] = top_of(m);
    P.zbot[m] = bottom_of(m);
    cplx s = sigma[m];
    if (s.re < 1e-9) s.re = 1e-9;  // sigma_floored (layered.cpp:47-51)
    P.sig[m] = s;
  }
  for (int m = 0; m <= L; ++m) {
    const std::complex<double> sm(P.sig[m].re, P.sig[m].im);
    const std::complex<double> up = m < L ? std::complex<double>(P.sig[m + 1].re, P.sig[m + 1].im) / sm : 1.0;
    const std::complex<double> dn = m > 0 ? std::complex<double>(P.sig[m - 1].re, P.sig[m - 1].im) / sm : 1.0;
    P.sig_up[m] = {up.real(), up.imag()};
    P.sig_dn[m] = {dn.real(), dn.imag()};
  }
  ivh.assign(nz, Interval{});
  for (int i = 0; i < nz; ++i) {
    if (!(breaks[i] < breaks[i + 1])) fail(EMIE_CU_INVALID_ARGUMENT, "vertical partition: breaks must increase");
    const int m = layer_of(breaks[i]);
    const double slack = 1e-7 * (1.0 + std::fabs(breaks[i + 1]));
    if (m < L && breaks[i + 1] > bottom_of(m) + slack)
      fail(EMIE_CU_INVALID_ARGUMENT, "vertical partition: interval straddles a layer interface");
    if (grid_checks && !(sigma[m].re > 0.0))
      fail(EMIE_CU_INVALID_ARGUMENT,
           "grid: interval in a non-conducting layer; the anomaly must be buried in the conductive section");
    Interval& I = ivh[i];
    I.a = breaks[i];
    I.b = breaks[i + 1];
    I.h = I.b - I.a;
    I.layer = m;
    I.d = top_of(m);
    I.dp = bottom_of(m);
    I.l = P.thick[m];
    I.has_p = m > 0;
    I.has_q = m < L;
    const cplx s = P.sig[m];
    const double dn = s.re * s.re + s.im * s.im;
    I.inv_sig = {s.re / dn, -s.im / dn};
  }
  // lambdas per chunk: as many as ~200 KB of SMEM holds (the serial per-chunk
  // phases then run on more threads and there are fewer chunks), at most 32
  {
    const size_t per_lambda = (14 * static_cast<size_t>(L + 1) + kFields * static_cast<size_t>(nz)) * sizeof(cplx) +
                              8 * sizeof(double) + 2 * static_cast<size_t>(nz) * sizeof(int);
    int lcm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(32, (size_t{EMIE_GREEN_SMEM_KB} << 10) / per_lambda)));
    if (lcm >= 8) lcm &= ~7;  // multiples of 8: the per-chunk phases split evenly over the warps
    P.LC = lcm;
  }
}

// Filter design (K6) and lambda accumulation (K5) of the offsets offs_h
// (codes of P.oc) into `blocks` (slot P.oc.slot(code, position) of nslots)
void assemble_codes(const GreenParams& P0, const std::vector<Interval>& ivh, const FilterParams& fp,
                    const std::vector<int>& offs_h, int nslots, cplx* blocks, cudaStream_t st, bool full) {
  GreenParams P = P0;
  if (full) P.nent = 9 * P.nz * P.nz;  // FullBlock slots
  keep_pool_warm();
  const int nz = P.nz, L = P.L;
  const int ncomp = static_cast<int>(offs_h.size());
  if (ncomp == 0) return;
  int* offs = scratch<int>(offs_h.size(), st);
  EMIE_CUDA(cudaMemcpyAsync(offs, offs_h.data(), offs_h.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  FilterBank fb = make_filter_bank(fp, st);
  double* W = scratch<double>(static_cast<size_t>(nslots) * 6 * P.nw, st);
  int* err = scratch<int>(1, st);
  EMIE_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  // the offsets' pair geometries from the host's C library, as the reference
  // computes them (hankel.cpp:80-91 and the sin / cos of kernel_output): the
  // filter designs and the lambda lattices lambda_m / R start from identical inputs
  std::vector<Geom> gh(ncomp);
  std::vector<double> Rh(ncomp);
  for (int i = 0; i < ncomp; ++i) {
    gh[i] = pair_geometry(P.oc.oi(offs_h[i]), P.oc.oj(offs_h[i]), P.hx, P.hy);
    Rh[i] = gh[i].r;
  }
  double* dRoff = scratch<double>(ncomp, st);
  EMIE_CUDA(cudaMemcpyAsync(dRoff, Rh.data(), ncomp * sizeof(double), cudaMemcpyHostToDevice, st));
  {
    Geom* gtab = scratch<Geom>(ncomp, st);
    EMIE_CUDA(cudaMemcpyAsync(gtab, gh.data(), ncomp * sizeof(Geom), cudaMemcpyHostToDevice, st));
    // the six kernels' design samples of every offset, transcendentals shared
    // (filter_samples_kernel), in batches
    // (EMIE_CU_GREENS_SHARED_SAMPLES=0: kernel_output per kernel, A/B and the
    // bit-identity test)
    static const bool shared_samples = [] {
      const char* e = std::getenv("EMIE_CU_GREENS_SHARED_SAMPLES");
      return !(e && e[0] == '0');
    }();
    const int n = 2 * fp.half;
    // batches of 4,096 offsets (200 MB of samples); compact slots are positions: one batch
    const int bmax = P.oc.compact ? ncomp : std::min(ncomp, 4096);
    double* samp = shared_samples ? scratch<double>(static_cast<size_t>(bmax) * 6 * n, st) : nullptr;
    for (int i0 = 0; i0 < ncomp && !shared_samples; i0 += ncomp)
      design_filters(fb, fp, ncomp, P.oc, P.hx, P.hy, W, err, st, INT32_MIN, 0, offs, nullptr, 0, 6, nullptr, gtab);
    for (int i0 = 0; i0 < ncomp && shared_samples; i0 += bmax) {
      const int nb = std::min(bmax, ncomp - i0);
      filter_samples_kernel<<<ceil_div(static_cast<long long>(nb) * n, 256), 256, 0, st>>>(gtab + i0, nb, n, fp.half,
                                                                                          fp.step, fp.shift, samp);
      check_launch("filter_samples_kernel");
      design_filters(fb, fp, nb, P.oc, P.hx, P.hy, W, err, st, INT32_MIN, 0, offs + i0, nullptr, 0, 6, nullptr,
                     nullptr, samp);
    }
    if (samp) release(samp, st);
    release(gtab, st);
  }

  Interval* div = scratch<Interval>(nz, st);
  EMIE_CUDA(cudaMemcpyAsync(div, ivh.data(), nz * sizeof(Interval), cudaMemcpyHostToDevice, st));
  const int NL = L + 1;
  const size_t smem = (static_cast<size_t>(P.LC) * (3 * NL + 11 * NL + kFields * nz)) * sizeof(cplx) +
                      8 * static_cast<size_t>(P.LC) * sizeof(double) +
                      static_cast<size_t>(P.LC) * 2 * nz * sizeof(int);
  set_smem(reinterpret_cast<const void*>(assemble_kernel<false>), smem);
  set_smem(reinterpret_cast<const void*>(assemble_kernel<true>), smem);
  const int groups = ceil_div(P.npairs, (kGreenSlots + 1) * kGreenThreads);
  dim3 grid(ncomp, groups);
  profile_mark(5, true, st);
#ifdef EMIE_GREENS_PHASE_CLOCKS
  {
    unsigned long long z[8] = {};
    EMIE_CUDA(cudaMemcpyToSymbolAsync(g_phase_clk, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
  }
#endif
  // Split (chunk_image_kernel + the pair kernel on streamed images) or the
  // fused kernel: the split saves the per-lambda phases of every pair-group
  // CTA after the first (nz > 32) and of every offset sharing another's R.
  static const int img_mode = [] {
    const char* e = std::getenv("EMIE_CU_GREENS_IMG");  // 0: fused, 1: split, unset: by group count
    return e && *e ? std::atoi(e) : -1;
  }();
  // default: split when an offset spans several pair groups (nz > 32), or
  // for large builds, where the images shared by offsets at equal R outweigh
  // the images' HBM round trip (config 3: 29.6 vs 33.2 ms fused; config 2's
  // 2,080 offsets: 5.3 vs 5.1 ms, and the split's host-side grouping costs more)
  const bool split_default = groups > 1 || (!P.oc.compact && img_share_enabled() && ncomp >= 4096);
  if (!full && (img_mode < 0 ? split_default : img_mode == 1)) {
    // lambdas per image CTA: 6 at nz <= 32 (config 3: 27.7 -> 26.2 ms; the
    // serial chain phase runs 24 tasks instead of 16), else kImgLambdas (its
    // SMEM would cost CTAs per SM at nz = 64: 340 -> 360 ms with 6)
    const int LA = nz <= 32 ? 6 : kImgLambdas;
    const size_t smemA = static_cast<size_t>(LA) * (14 * NL + kFields * nz) * sizeof(cplx) +
                         static_cast<size_t>(LA) * 2 * nz * sizeof(int);
    set_smem(reinterpret_cast<const void*>(chunk_image_kernel), smemA);
    GreenParams PB = P;
    {
      const size_t per_lambda = 2 * (kImgFields * static_cast<size_t>(nz) * sizeof(cplx) + 2 * nz * sizeof(int)) +
                                8 * sizeof(double);
      int lcb = static_cast<int>(std::max<size_t>(2, std::min<size_t>(32, (size_t{EMIE_GREEN_SMEM_KB} << 10) / per_lambda)));
      PB.LC = lcb & ~1;  // even: every chunk's exponent image starts 16-byte aligned
    }
    const size_t ibufF = static_cast<size_t>(PB.LC) * kImgFields * nz;
    const size_t ibufE = (static_cast<size_t>(PB.LC) * 2 * nz + 3) / 4 * 2;
    const size_t smemB = (2 * (ibufF + ibufE)) * sizeof(cplx) + 8 * static_cast<size_t>(PB.LC) * sizeof(double);
    set_smem(reinterpret_cast<const void*>(assemble_kernel<false, true>), smemB);
    const size_t fper = static_cast<size_t>(P.nw) * kImgFields * nz;  // complex per offset
    const size_t estride = (static_cast<size_t>(P.nw) * 2 * nz + 3) & ~size_t{3};
    const size_t per_off = fper * sizeof(cplx) + estride * sizeof(int);
    // batch: at most kImgBudget of images, and at most a quarter of the memory
    // free at the first split build (queried once: cudaMemGetInfo stalls the
    // host behind the device's queued work)
    static const size_t budget = [] {
      size_t cap = kImgBudget;
      if (const char* e = std::getenv("EMIE_CU_GREENS_IMG_MB"))  // A/B of the batch size
        if (*e) cap = static_cast<size_t>(std::max(16, std::atoi(e))) << 20;
      size_t free_b = 0, total_b = 0;
      return cudaMemGetInfo(&free_b, &total_b) == cudaSuccess ? std::min(cap, free_b / 4) : cap;
    }();
    // Offsets at the same distance R (bit for bit, as the kernels compute it)
    // share one chunk image: the per-lambda phases depend on the offset only
    // through lambda = lambda_m / R (5,384 distinct R among config 3's 8,256
    // computed offsets). Slots come from the codes (full builds), so the
    // offsets are reordered by R; signed-offset requests (slot = request
    // position) keep one image per offset.
    std::vector<int> img_h(ncomp), reps;
    std::vector<double> Rrep;
    if (!P.oc.compact && img_share_enabled()) {
      std::vector<uint64_t> key(ncomp);
      std::memcpy(key.data(), Rh.data(), ncomp * sizeof(double));
      std::vector<int> idx(ncomp);
      for (int i = 0; i < ncomp; ++i) idx[i] = i;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return key[a] < key[b]; });
      std::vector<int> sorted(ncomp);
      std::vector<double> Rs(ncomp);
      for (int b = 0; b < ncomp; ++b) {
        sorted[b] = offs_h[idx[b]];
        Rs[b] = Rh[idx[b]];
        if (b == 0 || key[idx[b]] != key[idx[b - 1]]) {
          reps.push_back(sorted[b]);
          Rrep.push_back(Rs[b]);
        }
        img_h[b] = static_cast<int>(reps.size()) - 1;
      }
      EMIE_CUDA(cudaMemcpyAsync(offs, sorted.data(), ncomp * sizeof(int), cudaMemcpyHostToDevice, st));
      EMIE_CUDA(cudaMemcpyAsync(dRoff, Rs.data(), ncomp * sizeof(double), cudaMemcpyHostToDevice, st));
    } else {
      reps = offs_h;
      Rrep = Rh;
      for (int b = 0; b < ncomp; ++b) img_h[b] = b;
    }
    const int nu = static_cast<int>(reps.size());
    int* dreps = scratch<int>(nu, st);
    int* dimg = scratch<int>(ncomp, st);
    double* dRrep = scratch<double>(nu, st);
    EMIE_CUDA(cudaMemcpyAsync(dRrep, Rrep.data(), nu * sizeof(double), cudaMemcpyHostToDevice, st));
    EMIE_CUDA(cudaMemcpyAsync(dreps, reps.data(), nu * sizeof(int), cudaMemcpyHostToDevice, st));
    EMIE_CUDA(cudaMemcpyAsync(dimg, img_h.data(), ncomp * sizeof(int), cudaMemcpyHostToDevice, st));
    // Two image buffers (each half the budget): the image kernel of batch
    // i + 1 runs on st while the pair kernel of batch i runs on a second
    // stream, so neither kernel's tail drains the GPU between batches
    // (EMIE_CU_GREENS_OVERLAP=0: one buffer, one stream, A/B)
    const int nbuf = greens_overlap_enabled() ? 2 : 1;
    const int maxu = static_cast<int>(std::min<size_t>(65535, std::max<size_t>(1, budget / nbuf / per_off)));
    const int nbatch = ceil_div(nu, maxu), ubatch = ceil_div(nu, nbatch);
    cplx* IF[2] = {nullptr, nullptr};
    int* IE[2] = {nullptr, nullptr};
    for (int k = 0; k < std::min(nbuf, nbatch); ++k) {
      IF[k] = scratch<cplx>(static_cast<size_t>(ubatch) * fper, st);
      IE[k] = scratch<int>(static_cast<size_t>(ubatch) * estride, st);
    }
    cudaStream_t pst = st;
    std::unique_ptr<AuxStream> aux;
    auto aux_event = [&](int e) { return aux->ev[e]; };
    if (nbuf == 2 && nbatch > 1) {
      aux = std::make_unique<AuxStream>();
      pst = aux->s;
      EMIE_CUDA(cudaEventRecord(aux_event(2), st));  // the pair stream starts behind everything queued on st
      EMIE_CUDA(cudaStreamWaitEvent(pst, aux_event(2), 0));
    }
    int b0 = 0;
    for (int u0 = 0, i = 0; u0 < nu; u0 += ubatch, ++i) {
      const int u1 = std::min(nu, u0 + ubatch);
      const int k = pst == st ? 0 : i & 1;
      int b1 = b0;
      while (b1 < ncomp && img_h[b1] < u1) ++b1;  // the offsets of images [u0, u1)
      if (pst != st && i >= 2) EMIE_CUDA(cudaStreamWaitEvent(st, aux_event(k), 0));  // pair kernel i - 2 read buffer k
      chunk_image_kernel<<<dim3(ceil_div(P.nw, LA), u1 - u0), kImgThreads, smemA, st>>>(P, div, dreps + u0, LA, IF[k],
                                                                                          IE[k], estride, dRrep + u0);
      check_launch("chunk_image_kernel");
      if (pst != st) {
        EMIE_CUDA(cudaEventRecord(aux_event(3), st));
        EMIE_CUDA(cudaStreamWaitEvent(pst, aux_event(3), 0));
      }
      assemble_kernel<false, true><<<dim3(b1 - b0, groups), kGreenThreads, smemB, pst>>>(
          PB, div, W, blocks, err, offs + b0, b0, IF[k], IE[k], estride, dimg + b0, u0, dRoff + b0);
      check_launch("assemble_kernel");
      if (pst != st) EMIE_CUDA(cudaEventRecord(aux_event(k), pst));
      b0 = b1;
    }
    if (pst != st) {  // join: st resumes behind the last pair kernel
      EMIE_CUDA(cudaEventRecord(aux_event(2), pst));
      EMIE_CUDA(cudaStreamWaitEvent(st, aux_event(2), 0));
    }
    for (int k = 0; k < 2; ++k) {
      release(IF[k], st);
      release(IE[k], st);
    }
    release(dreps, st);
    release(dimg, st);
    release(dRrep, st);
  } else {
    if (full)
      assemble_kernel<true><<<grid, kGreenThreads, smem, st>>>(P, div, W, blocks, err, offs, 0, nullptr, nullptr, 0,
                                                               nullptr, 0, dRoff);
    else
      assemble_kernel<false><<<grid, kGreenThreads, smem, st>>>(P, div, W, blocks, err, offs, 0, nullptr, nullptr, 0,
                                                                nullptr, 0, dRoff);
    check_launch("assemble_kernel");
  }
#ifdef EMIE_GREENS_PHASE_CLOCKS
  {
    unsigned long long h[8];
    EMIE_CUDA(cudaMemcpyFromSymbolAsync(h, g_phase_clk, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
    EMIE_CUDA(cudaStreamSynchronize(st));
    const char* nm[7] = {"chunk-start", "0a", "0b", "0c", "1", "1b", "2"};
    unsigned long long tot = 0;
    for (int i = 0; i < 7; ++i) tot += h[i];
    for (int i = 0; i < 7; ++i)
      std::fprintf(stderr, "assemble phase %-12s %6.2f%%  %.3e cycles/CTA\n", nm[i], 100.0 * h[i] / tot,
                   static_cast<double>(h[i]) / (static_cast<double>(grid.x) * grid.y));
  }
#endif
  profile_mark(5, false, st);
  int e = 0;
  EMIE_CUDA(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(W, st);
  release(err, st);
  release(div, st);
  release(offs, st);
  release(dRoff, st);
  free_filter_bank(fb, st);
  if (e) {
    raise_filter_errors(e);
    fail(EMIE_CU_DOMAIN_ERROR, "assemble_block: non-finite block entry");
  }
}


void greens_blocks(const Operator& op, int L, const double* tops, const cplx* sigma, const double* breaks,
                   double hx, double hy, const FilterParams& fp, int c0, int c1, cplx* blocks, cudaStream_t st) {
  GreenParams P;
  std::vector<Interval> ivh;
  green_setup(op.nx, op.ny, op.nz, op.omega, L, tops, sigma, breaks, hx, hy, fp, P, ivh);
  P.oc = OffsetCode{op.nx, 0, 0, 0};
  const std::vector<int> all = computed_offsets(op.nx, op.ny, hx, hy);
  const int cb = std::max(0, std::min(c0, static_cast<int>(all.size())));
  const int ce = c1 < 0 ? static_cast<int>(all.size()) : std::max(cb, std::min(c1, static_cast<int>(all.size())));
  if (ce == cb) return;
  assemble_codes(P, ivh, fp, std::vector<int>(all.begin() + cb, all.begin() + ce), op.nx * op.ny, blocks, st, false);
}

// assemble_block (greens.hpp:129-135, greens.cpp:150-221) at n signed offsets
// (|oi| < ny, |oj| < nx; out_of_range otherwise, greens.cpp:153-154) into host
// blocks in request order, GreensBlock layout; no mirror or symmetrisation
// (the reference evaluates every requested offset independently)
void assemble_signed_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                          const double* breaks, double hx, double hy, const FilterParams& fp, int n, const int* oi,
                          const int* oj, cplx* h_out) {
  if (nx < 1 || ny < 1 || nz < 1) fail(EMIE_CU_INVALID_ARGUMENT, "grid: empty dimensions");
  GreenParams P;
  std::vector<Interval> ivh;
  green_setup(nx, ny, nz, omega, L, tops, sigma, breaks, hx, hy, fp, P, ivh);
  for (int i = 0; i < n; ++i)
    if (std::abs(oi[i]) >= ny || std::abs(oj[i]) >= nx)
      fail(EMIE_CU_OUT_OF_RANGE, "assemble_block: offset outside the grid");
  if (n <= 0) return;
  P.oc = OffsetCode{2 * nx - 1, ny - 1, nx - 1, 1};
  std::vector<int> codes(n);
  for (int i = 0; i < n; ++i) codes[i] = (oi[i] + ny - 1) * (2 * nx - 1) + (oj[i] + nx - 1);
  cudaStream_t st = nullptr;
  const size_t bytes = static_cast<size_t>(n) * P.nent * sizeof(cplx);
  cplx* d = scratch<cplx>(static_cast<size_t>(n) * P.nent, st);
  try {
    assemble_codes(P, ivh, fp, codes, n, d, st, false);
  } catch (...) {
    release(d, st);
    throw;
  }
  EMIE_CUDA(cudaMemcpyAsync(h_out, d, bytes, cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(d, st);
}

// The rest of the build once every computed offset's block is in `blocks`:
// the x <-> y mirror of the other offsets and the symmetrised diagonal
// offsets (square grids with hx == hy), then the spectra (K7) of the modes
// op stores.
void greens_finish(Operator& op, cplx* blocks, double hx, double hy, cudaStream_t st) {
  const bool mirror = op.nx == op.ny && hx == hy;
  if (mirror) {
    std::vector<int> pairs_h;
    for (int oi = 0; oi < op.ny; ++oi)
      for (int oj = oi + 1; oj < op.nx; ++oj) pairs_h.push_back(oi * op.nx + oj);
    if (!pairs_h.empty()) {
      int* pairs = scratch<int>(pairs_h.size(), st);
      EMIE_CUDA(cudaMemcpyAsync(pairs, pairs_h.data(), pairs_h.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      const long long total = static_cast<long long>(pairs_h.size()) * op.nent;
      mirror_blocks_kernel<<<static_cast<int>(std::min<long long>(ceil_div(total, 256), 4096)), 256, 0, st>>>(
          blocks, pairs, static_cast<int>(pairs_h.size()), op.nx, op.ntri, op.nfull, op.nent);
      check_launch("mirror_blocks_kernel");
      release(pairs, st);
    }
    const long long total = static_cast<long long>(op.nx) * (op.ntri + op.nfull);
    symmetrize_diagonal_kernel<<<static_cast<int>(std::min<long long>(ceil_div(total, 256), 4096)), 256, 0, st>>>(
        blocks, op.nx, op.ntri, op.nfull, op.nent);
    check_launch("symmetrize_diagonal_kernel");
  }
  profile_mark(6, true, st);
  transform_blocks(op, blocks, st, mirror ? -1 : 0);  // checked: the octant path needs bitwise symmetry
  profile_mark(6, false, st);
}

void greens_build(Operator& op, int L, const double* tops, const cplx* sigma, const double* breaks,
                  double hx, double hy, const FilterParams& fp, bool keep_blocks, cudaStream_t st) {
  // the block array: kept with the operator (plain allocation, freed by it) or
  // a stream-ordered scratch buffer the pool hands to the next build
  const size_t nb = static_cast<size_t>(op.nx) * op.ny * op.nent;
  cplx* blocks = nullptr;
  if (keep_blocks) EMIE_CUDA(cudaMalloc(&blocks, nb * sizeof(cplx) + 16));
  else blocks = scratch<cplx>(nb, st);
  try {
    greens_blocks(op, L, tops, sigma, breaks, hx, hy, fp, 0, -1, blocks, st);
    greens_finish(op, blocks, hx, hy, st);
  } catch (...) {
    cudaStreamSynchronize(st);
    if (keep_blocks) cudaFree(blocks);
    else release(blocks, st);
    throw;
  }
  if (keep_blocks) op.blocks = blocks;
  else release(blocks, st);
}

}  // namespace emie_cu
