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

#include <type_traits>

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

namespace emie_cu {

// ===================================================================
// Power-of-two fast path: in-place Stockham with radix-16/8/4/2 passes,
// every thread holding EPT elements in registers across a pass (loads,
// barrier, butterflies, stores, barrier), so one SMEM tile suffices and a
// 256-point transform needs two passes. Tile element i of transform t
// lives at phys(t*n + i) = idx + idx/16: the stride-R stores of a pass
// then fall on distinct 16-byte banks.
// ===================================================================
constexpr int kFftEPT = 16;

__host__ __device__ __forceinline__ int fft_phys(int idx) { return idx + (idx >> 4); }
// 2-D form: transform t starts at t*ldp with ldp = n + n/16 + 1 (odd), so
// element j of consecutive transforms also falls on distinct banks
__host__ __device__ __forceinline__ int fft_ldp(int n) { return n + (n >> 4) + 1; }
__host__ __device__ __forceinline__ int fft_phys2(int t, int j, int ldp) { return t * ldp + j + (j >> 4); }

inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// e^{s 2 pi i m / 16}, m = 0..15 (s = -1 forward)
__host__ __device__ constexpr double cos16(int m) {
  return (m & 15) == 0 ? 1.0 : (m & 15) == 1 ? 0.92387953251128675613 : (m & 15) == 2 ? 0.70710678118654752440
       : (m & 15) == 3 ? 0.38268343236508977173 : (m & 15) == 4 ? 0.0 : (m & 15) == 5 ? -0.38268343236508977173
       : (m & 15) == 6 ? -0.70710678118654752440 : (m & 15) == 7 ? -0.92387953251128675613 : (m & 15) == 8 ? -1.0
       : (m & 15) == 9 ? -0.92387953251128675613 : (m & 15) == 10 ? -0.70710678118654752440
       : (m & 15) == 11 ? -0.38268343236508977173 : (m & 15) == 12 ? 0.0 : (m & 15) == 13 ? 0.38268343236508977173
       : (m & 15) == 14 ? 0.70710678118654752440 : 0.92387953251128675613;
}
__device__ __forceinline__ cplx w16(int m, double s) {
  return {cos16(m), s * cos16(m + 12)};  // sin(x) = cos(x - pi/2)
}

// x * e^{s 2 pi i m / 16} for a compile-time m, without the multiplications
// by 0 and 1 that IEEE semantics keep in a general product
template <int m>
__device__ __forceinline__ cplx mulw16(cplx x, double s) {
  constexpr int q = m & 15;
  constexpr double h = 0.70710678118654752440;
  if constexpr (q == 0) {
    return x;
  } else if constexpr (q == 4) {  // s i
    return {-s * x.im, s * x.re};
  } else if constexpr (q == 8) {
    return {-x.re, -x.im};
  } else if constexpr (q == 12) {  // -s i
    return {s * x.im, -s * x.re};
  } else if constexpr (q == 2 || q == 6 || q == 10 || q == 14) {
    // (c + i s sn) with |c| = |sn| = h
    constexpr double c = (q == 2 || q == 14) ? h : -h;
    constexpr double sn = (q == 2 || q == 6) ? h : -h;
    const double si = s * sn;
    return {c * x.re - si * x.im, c * x.im + si * x.re};
  } else {
    const cplx w = w16(q, s);
    return x * w;
  }
}

template <>
__device__ __forceinline__ void butterfly<8>(cplx* v, double s) {
  // 8 = 2 x 4: DFT4 over (a + 2c), twiddle W8^{ab}, DFT2 over a
  cplx e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  butterfly<4>(e, s);
  butterfly<4>(o, s);
  const cplx t[4] = {o[0], mulw16<2>(o[1], s), mulw16<4>(o[2], s), mulw16<6>(o[3], s)};
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    v[b] = e[b] + t[b];
    v[b + 4] = e[b] - t[b];
  }
}

template <>
__device__ __forceinline__ void butterfly<16>(cplx* v, double s) {
  // 16 = 4 x 4 (n = a + 4c, k = b + 4d), in place; the final 4x4 transpose
  // is a register renaming once unrolled
  auto col = [&](auto A) {
    constexpr int a = decltype(A)::value;
    cplx q[4] = {v[a], v[a + 4], v[a + 8], v[a + 12]};
    butterfly<4>(q, s);
    v[a] = q[0];
    v[a + 4] = mulw16<a * 1>(q[1], s);
    v[a + 8] = mulw16<a * 2>(q[2], s);
    v[a + 12] = mulw16<a * 3>(q[3], s);
  };
  col(std::integral_constant<int, 0>{});
  col(std::integral_constant<int, 1>{});
  col(std::integral_constant<int, 2>{});
  col(std::integral_constant<int, 3>{});
  // v[a + 4b] = y[a][b]
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    cplx q[4] = {v[4 * b], v[4 * b + 1], v[4 * b + 2], v[4 * b + 3]};
    butterfly<4>(q, s);
#pragma unroll
    for (int d = 0; d < 4; ++d) v[4 * b + d] = q[d];
  }
  // X[b + 4d] sits at v[4b + d]: transpose
  cplx t[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) t[r] = v[4 * (r & 3) + (r >> 2)];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = t[r];
}

inline bool make_pow2_plan(int n, FftPlan& p) {
  if (!is_pow2(n) || n > 4096) return false;
  p = FftPlan{};
  p.n = n;
  int r = n;
  while (r >= 16) { p.radix[p.npass++] = 16; r /= 16; }
  if (r > 1) p.radix[p.npass++] = r;  // 8, 4 or 2
  return true;
}

template <int R>
__device__ __forceinline__ void pow2_pass(cplx* buf, int n, int ldp, int ns, int work, const cplx* tw,
                                          double s) {
  constexpr int B = kFftEPT / R;  // butterflies per thread
  const int m = n / R;
  const int tstep = n / (ns * R);
  cplx v[B][R];
  int dt[B], dj[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int w = threadIdx.x + b * blockDim.x;
    dt[b] = -1;
    if (w < work) {
      const int t = w / m, j = w - t * m;
      const int k = j & (ns - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        cplx x = buf[fft_phys2(t, j + r * m, ldp)];
        if (r > 0 && k > 0) {
          cplx wv = tw[r * k * tstep];
          if (s > 0) wv.im = -wv.im;
          x = x * wv;
        }
        v[b][r] = x;
      }
      butterfly<R>(v[b], s);
      dt[b] = t;
      dj[b] = (j / ns) * ns * R + k;
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b)
    if (dt[b] >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) buf[fft_phys2(dt[b], dj[b] + r * ns, ldp)] = v[b][r];
    }
  __syncthreads();
}

// In-place transform of ntr sequences of length n (pow2) in a padded tile;
// ntr * n must be <= blockDim.x * kFftEPT. Caller synchronises after the
// fill; returns synchronised.
__device__ inline void fft_pow2(cplx* buf, int ntr, const FftPlan& pl, const cplx* tw,
                                bool inverse) {
  const double s = inverse ? 1.0 : -1.0;
  const int n = pl.n, ldp = fft_ldp(n);
  const int lg = 31 - __clz(n);  // n = 2^lg: lg/4 radix-16 passes, then 2^(lg%4)
  int ns = 1;
  for (int p = 0; p < (lg >> 2); ++p) {
    pow2_pass<16>(buf, n, ldp, ns, ntr * (n >> 4), tw, s);
    ns <<= 4;
  }
  switch (lg & 3) {
    case 3: pow2_pass<8>(buf, n, ldp, ns, ntr * (n >> 3), tw, s); break;
    case 2: pow2_pass<4>(buf, n, ldp, ns, ntr * (n >> 2), tw, s); break;
    case 1: pow2_pass<2>(buf, n, ldp, ns, ntr * (n >> 1), tw, s); break;
    default: break;
  }
}

}  // namespace emie_cu
