// Batched complex128 Stockham FFT staged in shared memory (sm_100a).
//
// The reference runs its lateral transforms through FFTW
// (src/toeplitz.cpp:39-56, 152, 191, 274; src/hankel.cpp:213-256). Here a
// CTA loads a tile of transforms into shared memory (the kernel decides the
// coalesced global mapping, the zero padding and the parity embedding),
// runs the mixed-radix passes below, and stores straight into the layout
// the next stage wants, so no transform ever round-trips HBM between passes.
//
// Lengths: any product of 2, 3, 4 and 5 (the circulant embeddings are
// 5-smooth by construction, toeplitz.cpp:18-26; the filter design uses
// 2*half). Twiddles come from a host table computed in long double.
#pragma once

#include "common.cuh"

namespace emie_cu {

constexpr int kMaxPasses = 24;

struct FftPlan {
  int n = 1;
  int npass = 0;
  int radix[kMaxPasses] = {};
};

// factor n into radix-4/2/3/5 passes; returns false for other primes
inline bool make_plan(int n, FftPlan& p) {
  p = FftPlan{};
  p.n = n;
  int r = n;
  while (r % 4 == 0) { p.radix[p.npass++] = 4; r /= 4; }
  while (r % 2 == 0) { p.radix[p.npass++] = 2; r /= 2; }
  while (r % 3 == 0) { p.radix[p.npass++] = 3; r /= 3; }
  while (r % 5 == 0) { p.radix[p.npass++] = 5; r /= 5; }
  return r == 1 && p.npass <= kMaxPasses;
}

// small DFTs; s = -1 forward (e^{-2 pi i jk/n}), +1 backward
template <int R>
__device__ __forceinline__ void butterfly(cplx* v, double s);

template <>
__device__ __forceinline__ void butterfly<2>(cplx* v, double) {
  const cplx a = v[0], b = v[1];
  v[0] = a + b;
  v[1] = a - b;
}

template <>
__device__ __forceinline__ void butterfly<4>(cplx* v, double s) {
  const cplx t0 = v[0] + v[2], t1 = v[0] - v[2];
  const cplx t2 = v[1] + v[3], d = v[1] - v[3];
  const cplx t3 = {-s * d.im, s * d.re};  // d * (s i)
  v[0] = t0 + t2;
  v[2] = t0 - t2;
  v[1] = t1 + t3;
  v[3] = t1 - t3;
}

template <>
__device__ __forceinline__ void butterfly<3>(cplx* v, double s) {
  const double c = -0.5, sn = 0.86602540378443864676 * s;  // e^{s 2 pi i/3}
  const cplx t = v[1] + v[2], d = v[1] - v[2];
  const cplx a = {v[0].re + c * t.re, v[0].im + c * t.im};
  const cplx b = {-sn * d.im, sn * d.re};  // i sn d
  v[0] = v[0] + t;
  v[1] = a + b;
  v[2] = a - b;
}

template <>
__device__ __forceinline__ void butterfly<5>(cplx* v, double s) {
  // e^{s 2 pi i k/5}: cos and sin of 72 and 144 degrees
  const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
  const double s1 = 0.95105651629515357212 * s, s2 = 0.58778525229247312917 * s;
  const cplx t1 = v[1] + v[4], t2 = v[2] + v[3];
  const cplx d1 = v[1] - v[4], d2 = v[2] - v[3];
  const cplx a1 = {v[0].re + c1 * t1.re + c2 * t2.re, v[0].im + c1 * t1.im + c2 * t2.im};
  const cplx a2 = {v[0].re + c2 * t1.re + c1 * t2.re, v[0].im + c2 * t1.im + c1 * t2.im};
  // b1 = i (s1 d1 + s2 d2), b2 = i (s2 d1 - s1 d2)
  const cplx b1 = {-(s1 * d1.im + s2 * d2.im), s1 * d1.re + s2 * d2.re};
  const cplx b2 = {-(s2 * d1.im - s1 * d2.im), s2 * d1.re - s1 * d2.re};
  v[0] = v[0] + t1 + t2;
  v[1] = a1 + b1;
  v[4] = a1 - b1;
  v[2] = a2 + b2;
  v[3] = a2 - b2;
}

template <int R>
__device__ __forceinline__ void stockham_pass(const cplx* __restrict__ src, cplx* __restrict__ dst,
                                              int ld, int ntr, int n, int ns,
                                              const cplx* __restrict__ tw, double s) {
  const int m = n / R;
  const int tstep = n / (ns * R);
  const int work = ntr * m;
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int t = w / m;
    const int j = w - t * m;
    const int k = j % ns;
    const cplx* a = src + t * ld + j;
    cplx v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cplx x = a[r * m];
      if (r > 0 && k > 0) {
        cplx wv = tw[r * k * tstep];  // e^{-2 pi i (rk/(ns R))}
        if (s > 0) wv.im = -wv.im;    // backward transform: conjugate
        x = x * wv;
      }
      v[r] = x;
    }
    butterfly<R>(v, s);
    cplx* d = dst + t * ld + (j / ns) * ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * ns] = v[r];
  }
}

// Runs the transform on ntr sequences (element j of sequence t at
// a[t*ld + j]); b is scratch of the same shape. Returns the buffer that
// holds the result. Ends with a __syncthreads(). The caller must have
// synchronised after filling a and the twiddle table.
// tw[m] = e^{-2 pi i m / n}; inverse = false -> forward (sign -1).
__device__ inline cplx* fft_smem(cplx* a, cplx* b, int ld, int ntr, const FftPlan& pl,
                                 const cplx* tw, bool inverse) {
  const double s = inverse ? 1.0 : -1.0;
  int ns = 1;
  for (int p = 0; p < pl.npass; ++p) {
    const int R = pl.radix[p];
    switch (R) {
      case 4: stockham_pass<4>(a, b, ld, ntr, pl.n, ns, tw, s); break;
      case 2: stockham_pass<2>(a, b, ld, ntr, pl.n, ns, tw, s); break;
      case 3: stockham_pass<3>(a, b, ld, ntr, pl.n, ns, tw, s); break;
      default: stockham_pass<5>(a, b, ld, ntr, pl.n, ns, tw, s); break;
    }
    __syncthreads();
    cplx* t = a;
    a = b;
    b = t;
    ns *= R;
  }
  return a;
}

// copy the twiddle table into shared memory
__device__ __forceinline__ void load_twiddles(cplx* dst, const cplx* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = ldg(src + i);
}

}  // namespace emie_cu
