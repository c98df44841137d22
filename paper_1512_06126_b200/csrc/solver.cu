// Device FGMRES for A U = rhs with A = apply(SystemOperator) — the
// reference's fgmres (src/cie.cpp:117-238) restated for the GPU.
//
// What stays on the host: the (m+1) x m Hessenberg column, the complex
// Givens rotations with real cosine (cie.cpp:100-113), the breakdown test
// (cie.cpp:171-187), the back substitution (cie.cpp:205-212) — O(m^2)
// scalars per cycle, bit-for-bit the reference's arithmetic.
// What runs on the device: every vector operation (norms, the conjugated
// dots, axpys, scalings) and the operator applies. Basis vectors of all
// right-hand sides share one apply call per step (the two MT polarisations
// read the operator once).
//
// Orthogonalisation: classical Gram-Schmidt run twice (CGS2) instead of the
// reference's modified Gram-Schmidt run twice (cie.cpp:158-165). Both
// produce the same Krylov basis in exact arithmetic and are "twice is
// enough" stable; CGS2 turns the (j+1) sequential dot/axpy pairs into one
// batched dot sweep and one batched update sweep per pass. All reductions
// are fixed-order (per-block partials, then an ordered final sum), so
// solves are bit-reproducible.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "../../include/emie_cu.h"
#include "operator.cuh"
#include "tma.cuh"

namespace emie_cu {

namespace {

constexpr int kRedThreads = 256;
constexpr int kChunk = 8;

int red_blocks(std::size_t n) {
  return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(592, (n + kRedThreads - 1) / kRedThreads)));
}

// block-wide sum of NV doubles per thread into out[0..NV) (thread 0 writes)
template <int NV>
__device__ void block_sum(double (&v)[NV], double* out) {
  __shared__ double red[kRedThreads / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][i] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < kRedThreads / 32; ++w) s += red[w][i];
      out[i] = s;
    }
  }
  __syncthreads();
}

// partial[blk][2*(l0+l) .. +1] = sum_e conj(V_l[e]) w[e] for l in chunk;
// partial[blk][2*nv] = sum_e |w[e]|^2 when with_norm (chunk 0 only)
__global__ void __launch_bounds__(kRedThreads) dots_kernel(const cplx* __restrict__ V, std::size_t vstride,
                                                           int nv, const cplx* __restrict__ w,
                                                           std::size_t n, double* partial, int pstride,
                                                           int with_norm) {
  const int nchunks = max(1, (nv + kChunk - 1) / kChunk);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int l0 = ci * kChunk;
    double acc[2 * kChunk + 1];
#pragma unroll
    for (int i = 0; i < 2 * kChunk + 1; ++i) acc[i] = 0.0;
    const int nl = max(0, min(kChunk, nv - l0));
    for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
      const cplx wv = ldg(w + e);
      if (l0 == 0) acc[2 * kChunk] = fma(wv.re, wv.re, fma(wv.im, wv.im, acc[2 * kChunk]));
#pragma unroll
      for (int l = 0; l < kChunk; ++l) {
        if (l < nl) {
          const cplx v = ldg(V + (l0 + l) * vstride + e);
          acc[2 * l] = fma(v.re, wv.re, fma(v.im, wv.im, acc[2 * l]));
          acc[2 * l + 1] = fma(v.re, wv.im, fma(-v.im, wv.re, acc[2 * l + 1]));
        }
      }
    }
    __shared__ double tot[2 * kChunk + 1];
    block_sum<2 * kChunk + 1>(acc, tot);
    if (threadIdx.x < 2 * nl) partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * l0 + threadIdx.x] = tot[threadIdx.x];
    if (l0 == 0 && with_norm && threadIdx.x == 0)
      partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * nv] = tot[2 * kChunk];
  }
}

// out[i] = sum over blocks of partial[b][i]: block i, thread t sums blocks
// b = t, t + 256, ... in order, then a fixed shuffle / warp tree (deterministic)
constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const double* partial, int nblocks, int pstride,
                                                               int nvals, double* out) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  if (i >= nvals) return;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kFinThreads) s += partial[static_cast<std::size_t>(b) * pstride + i];
  double v[1] = {s};
  __shared__ double tot[1];
  block_sum<1>(v, tot);
  if (threadIdx.x == 0) out[i] = tot[0];
}

// w[e] -= sum_l h[l] V_l[e]; optional per-block |w|^2 partial at pstride slot 0
__global__ void __launch_bounds__(kRedThreads) update_kernel(cplx* w, const cplx* __restrict__ V,
                                                             std::size_t vstride, int nv,
                                                             const double* __restrict__ h,
                                                             std::size_t n, double* partial) {
  double acc[1] = {0.0};
  for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    cplx x = w[e];
    for (int l = 0; l < nv; ++l) {
      const cplx v = ldg(V + l * vstride + e);
      const double hr = h[2 * l], hi = h[2 * l + 1];
      // x -= h v
      x.re = fma(-hr, v.re, fma(hi, v.im, x.re));
      x.im = fma(-hr, v.im, fma(-hi, v.re, x.im));
    }
    w[e] = x;
    acc[0] = fma(x.re, x.re, fma(x.im, x.im, acc[0]));
  }
  if (partial) {
    __shared__ double tot[1];
    block_sum<1>(acc, tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot[0];
  }
}

// ---- tiled CGS2 sweeps (TMA-staged) ---------------------------------------
// The basis vectors and w are cut into tiles of kTE elements; a producer warp
// brings tile t of every V_l and of w into a SMEM stage with one bulk copy
// per vector (lane l issues V_l's), two stages deep behind full/empty
// mbarriers, so each sweep reads the basis from HBM once at full rate.
//   MODE 0: dots conj(V_l) . w (+ |w|^2)                      (CGS2 pass 1)
//   MODE 1: w' = w - V h, then conj(V_l) . w'                  (pass-1 update + pass-2 dots)
//   MODE 2: w'' = w' - V h and |w''|^2                          (pass-2 update + norm)
// MODE 1 walks the tiles in reverse: its first tiles are those the MODE 0
// sweep read last, still in L2 (and MODE 2's first those MODE 1 read last).
// The update keeps update_kernel's arithmetic (sequential in l, same FMAs),
// so w', w'' are bit-identical to it. Dots: compute warp k owns vectors
// l = k, k + 8, ..., lanes own elements; per-lane partials live in registers
// across tiles and are reduced in a fixed order at the end (one CTA per SM,
// fixed grid: the summation order does not depend on the GPU).
#ifndef EMIE_CGS_REVERSE
#define EMIE_CGS_REVERSE 1
#endif
constexpr bool kCgsReverse = EMIE_CGS_REVERSE;  // MODE 1 tiles in reverse (A/B switch)
constexpr int kTE = 128;        // elements per tile
constexpr int kTileMaxV = 41;   // basis vectors per staged tile (restart <= 40)
constexpr int kCgsWarps = 8;    // compute warps
constexpr int kCgsThreads = (kCgsWarps + 1) * 32;
constexpr int kCgsBlocks = 148;
constexpr int kLPerWarp = (kTileMaxV + kCgsWarps - 1) / kCgsWarps;

__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCgsWarps * 32) : "memory");
}

// DCGS2 (delayed classical Gram-Schmidt with reorthogonalisation, one
// projection sweep fewer per Arnoldi step than CGS2): the last basis vector
// v_j = V[nv-1] arrives projected once; MODE 3 reads the basis and w once for
// both dot sets, V[<nv-1]^H v_j (v_j's delayed second projection) and
// V^H w (+ |w|^2, |v_j|^2); dcgs_coef_kernel turns them into v_j's
// correction a, its norm alpha and w's coefficients against the corrected
// basis; MODE 4 corrects v_j in place, v_j <- (v_j - V a) / alpha, and
// projects w once, w <- w - V h, with |w|^2 (h: [h 2nv][a 2(nv-1)][1/alpha]).
template <int MODE>
__global__ void __launch_bounds__(kCgsThreads, 1)
    cgs_tile_kernel(cplx* w, const cplx* V, std::size_t vstride, int nv,  // V: TMA source only (MODE 4 writes V[nv-1])
                    const double* __restrict__ h, std::size_t n, double* partial, int pstride, int with_norm,
                    cplx* Vlast = nullptr) {
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 2;
  const std::size_t stage_elems = static_cast<std::size_t>(nv + 1) * kTE;
  cplx* stage0 = reinterpret_cast<cplx*>(sm + 128);
  cplx* xs = stage0 + 2 * stage_elems;
  double* hs = reinterpret_cast<double*>(xs + kTE);
  double* red = hs + 4 * kTileMaxV + 2;  // kCgsWarps
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kCgsWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // h and the vectors come from the previous kernels
  if (MODE == 1 || MODE == 2)
    for (int i = tid; i < 2 * nv; i += blockDim.x) hs[i] = h[i];
  if (MODE == 4)
    for (int i = tid; i < 4 * nv - 1; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  const std::size_t ntiles = (n + kTE - 1) / kTE;

  if (warp == kCgsWarps) {  // ---- producer
    int j = 0;
    for (std::size_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++j) {
      const std::size_t t = (kCgsReverse && MODE == 1) ? ntiles - 1 - tt : tt;
      const int s = j & 1;
      if (j >= 2) mbar_wait(empty + s, static_cast<uint32_t>(((j >> 1) - 1) & 1));
      const std::size_t e0 = t * kTE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<std::size_t>(kTE), n - e0) * sizeof(cplx));
      if (lane == 0) mbar_expect_tx(full + s, (nv + 1) * bytes);
      __syncwarp();
      cplx* st = stage0 + s * stage_elems;
      for (int l = lane; l <= nv; l += 32)
        bulk_g2s(st + static_cast<std::size_t>(l) * kTE, l < nv ? V + l * vstride + e0 : w + e0, bytes, full + s);
    }
    return;
  }

  // ---- compute warps
  double acc[kLPerWarp][2];
  double accv[MODE == 3 ? kLPerWarp : 1][2];  // MODE 3: dots with v_j = V[nv-1]
#pragma unroll
  for (int i = 0; i < kLPerWarp; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < (MODE == 3 ? kLPerWarp : 1); ++i) accv[i][0] = accv[i][1] = 0.0;
  double nacc = 0.0, vacc = 0.0;
  int j = 0;
  for (std::size_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++j) {
    const std::size_t t = (kCgsReverse && MODE == 1) ? ntiles - 1 - tt : tt;  // see the producer
    const int s = j & 1;
    mbar_wait(full + s, static_cast<uint32_t>((j >> 1) & 1));
    const cplx* Vt = stage0 + s * stage_elems;
    const cplx* wt = Vt + static_cast<std::size_t>(nv) * kTE;
    const std::size_t e0 = t * kTE;
    const int cnt = static_cast<int>(min(static_cast<std::size_t>(kTE), n - e0));
    const cplx* x_src = wt;
    if (MODE == 4) {
      // v_j <- (v_j - sum_l a_l V_l) / alpha; w <- w - sum_l h_l V_l - h_{nv-1} v_j (l < nv - 1)
      if (tid < cnt) {
        const int jv = nv - 1;
        const double* ha = hs + 2 * nv;
        cplx x = wt[tid], vf = Vt[jv * kTE + tid];
        for (int l = 0; l < jv; ++l) {
          const cplx v = Vt[l * kTE + tid];
          const double hr = hs[2 * l], hi = hs[2 * l + 1], ar = ha[2 * l], ai = ha[2 * l + 1];
          x.re = fma(-hr, v.re, fma(hi, v.im, x.re));
          x.im = fma(-hr, v.im, fma(-hi, v.re, x.im));
          vf.re = fma(-ar, v.re, fma(ai, v.im, vf.re));
          vf.im = fma(-ar, v.im, fma(-ai, v.re, vf.im));
        }
        const double ia = ha[2 * jv];
        vf.re *= ia;
        vf.im *= ia;
        const double hr = hs[2 * jv], hi = hs[2 * jv + 1];
        x.re = fma(-hr, vf.re, fma(hi, vf.im, x.re));
        x.im = fma(-hr, vf.im, fma(-hi, vf.re, x.im));
        w[e0 + tid] = x;
        Vlast[e0 + tid] = vf;
        nacc = fma(x.re, x.re, fma(x.im, x.im, nacc));
      }
    } else if (MODE != 0 && MODE != 3) {
      // update: thread e < kTE owns element e (update_kernel's arithmetic)
      if (tid < cnt) {
        cplx x = wt[tid];
        for (int l = 0; l < nv; ++l) {
          const cplx v = Vt[l * kTE + tid];
          const double hr = hs[2 * l], hi = hs[2 * l + 1];
          x.re = fma(-hr, v.re, fma(hi, v.im, x.re));
          x.im = fma(-hr, v.im, fma(-hi, v.re, x.im));
        }
        w[e0 + tid] = x;
        if (MODE == 1) xs[tid] = x;
        if (MODE == 2) nacc = fma(x.re, x.re, fma(x.im, x.im, nacc));
      }
      if (MODE == 1) compute_bar();
      x_src = xs;
    }
    if (MODE == 0 || MODE == 1 || MODE == 3) {
      cplx wv[kTE / 32];
#pragma unroll
      for (int k = 0; k < kTE / 32; ++k) {
        const int e = lane + 32 * k;
        wv[k] = e < cnt ? x_src[e] : cplx{0.0, 0.0};
      }
      if ((MODE == 3 || (MODE == 0 && with_norm)) && warp == 0) {
#pragma unroll
        for (int k = 0; k < kTE / 32; ++k) nacc = fma(wv[k].re, wv[k].re, fma(wv[k].im, wv[k].im, nacc));
      }
      cplx vj[MODE == 3 ? kTE / 32 : 1];
      if constexpr (MODE == 3) {
#pragma unroll
        for (int k = 0; k < kTE / 32; ++k) {
          const int e = lane + 32 * k;
          vj[k] = e < cnt ? Vt[(nv - 1) * kTE + e] : cplx{0.0, 0.0};
        }
        if (warp == 1) {
#pragma unroll
          for (int k = 0; k < kTE / 32; ++k) vacc = fma(vj[k].re, vj[k].re, fma(vj[k].im, vj[k].im, vacc));
        }
      }
#pragma unroll
      for (int i = 0; i < kLPerWarp; ++i) {
        const int l = warp + kCgsWarps * i;
        if (l < nv) {
#pragma unroll
          for (int k = 0; k < kTE / 32; ++k) {
            const int e = lane + 32 * k;
            if (e < cnt) {
              const cplx v = Vt[l * kTE + e];
              acc[i][0] = fma(v.re, wv[k].re, fma(v.im, wv[k].im, acc[i][0]));
              acc[i][1] = fma(v.re, wv[k].im, fma(-v.im, wv[k].re, acc[i][1]));
              if constexpr (MODE == 3) {
                if (l < nv - 1) {
                  accv[i][0] = fma(v.re, vj[k].re, fma(v.im, vj[k].im, accv[i][0]));
                  accv[i][1] = fma(v.re, vj[k].im, fma(-v.im, vj[k].re, accv[i][1]));
                }
              }
            }
          }
        }
      }
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);  // this warp is done with the stage
    if (MODE == 1) compute_bar();  // xs is rewritten by the next tile
  }
  // ---- fixed-order reductions (MODE 3 layout: [2nv w-dots][|w|^2][2(nv-1) v_j-dots][|v_j|^2])
  if (MODE == 3) {
#pragma unroll
    for (int i = 0; i < kLPerWarp; ++i) {
      const int l = warp + kCgsWarps * i;
      double r = accv[i][0], im = accv[i][1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_down_sync(0xffffffffu, r, o);
        im += __shfl_down_sync(0xffffffffu, im, o);
      }
      if (lane == 0 && l < nv - 1) {
        partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * nv + 1 + 2 * l] = r;
        partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * nv + 2 + 2 * l] = im;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vacc += __shfl_down_sync(0xffffffffu, vacc, o);
    if (warp == 1 && lane == 0) partial[static_cast<std::size_t>(blockIdx.x) * pstride + 4 * nv - 1] = vacc;
  }
  if (MODE == 0 || MODE == 1 || MODE == 3) {
#pragma unroll
    for (int i = 0; i < kLPerWarp; ++i) {
      const int l = warp + kCgsWarps * i;
      double r = acc[i][0], im = acc[i][1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r += __shfl_down_sync(0xffffffffu, r, o);
        im += __shfl_down_sync(0xffffffffu, im, o);
      }
      if (lane == 0 && l < nv) {
        partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * l] = r;
        partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * l + 1] = im;
      }
    }
  }
  if (MODE == 2 || MODE == 4 || MODE == 3 || (MODE == 0 && with_norm)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
    if (lane == 0) red[warp] = nacc;
    compute_bar();
    if (tid == 0) {
      double sum = 0.0;
      for (int k = 0; k < kCgsWarps; ++k) sum += red[k];
      if (MODE == 2 || MODE == 4) partial[blockIdx.x] = sum;
      else partial[static_cast<std::size_t>(blockIdx.x) * pstride + 2 * nv] = sum;
    }
  }
}

// DCGS2 coefficients from the finalized MODE 3 sums s (one warp, fixed-order
// butterfly sums): a = V[<nv-1]^H v_j, alpha = sqrt(|v_j|^2 - |a|^2) (the
// corrected v_j's norm, V orthonormal), h_l = V_l^H w (l < nv-1) and
// h_{nv-1} = (v_j^H w - a^H h_{<nv-1}) / alpha (w against the corrected v_j).
// coef = [h 2nv][a 2(nv-1)][1/alpha] for MODE 4; host slots: s0 = [h][|w|^2],
// s1 = [a][alpha]
__global__ void __launch_bounds__(32) dcgs_coef_kernel(const double* __restrict__ s, int nv, double* coef,
                                                       double* s0, double* s1) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x;
  const int jv = nv - 1;
  const double* a = s + 2 * nv + 1;
  double an = 0.0, cr = 0.0, ci = 0.0;
  for (int l = lane; l < jv; l += 32) {
    const double ar = a[2 * l], ai = a[2 * l + 1], br = s[2 * l], bi = s[2 * l + 1];
    an = fma(ar, ar, fma(ai, ai, an));
    cr = fma(ar, br, fma(ai, bi, cr));  // conj(a_l) b_l
    ci = fma(ar, bi, fma(-ai, br, ci));
    coef[2 * l] = s0[2 * l] = br;
    coef[2 * l + 1] = s0[2 * l + 1] = bi;
    coef[2 * nv + 2 * l] = s1[2 * l] = ar;
    coef[2 * nv + 2 * l + 1] = s1[2 * l + 1] = ai;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    an += __shfl_xor_sync(0xffffffffu, an, o);
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    ci += __shfl_xor_sync(0xffffffffu, ci, o);
  }
  if (lane == 0) {
    const double a2 = s[4 * nv - 1] - an;
    const double alpha = a2 > 0.0 ? sqrt(a2) : 0.0;
    const double ia = alpha > 0.0 ? 1.0 / alpha : 0.0;
    coef[2 * jv] = s0[2 * jv] = (s[2 * jv] - cr) * ia;
    coef[2 * jv + 1] = s0[2 * jv + 1] = (s[2 * jv + 1] - ci) * ia;
    coef[4 * nv - 2] = ia;
    s0[2 * nv] = s[2 * nv];
    s1[2 * jv] = alpha;
  }
}

std::size_t cgs_smem(int nv) {
  return 128 + 2 * static_cast<std::size_t>(nv + 1) * kTE * sizeof(cplx) + kTE * sizeof(cplx) +
         (4 * kTileMaxV + 2 + kCgsWarps) * sizeof(double);
}

// y[e] = a * x[e] (real a)
__global__ void scale_kernel(cplx* y, const cplx* __restrict__ x, double a, std::size_t n) {
  for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    y[e] = a * ldg(x + e);
}

// y[e] = x[e] / sqrt(*nrm2): the next basis vector normalised on the device
// (same IEEE sqrt and division as the host path, so bit-identical to it)
// y2 (optional): a second copy, the next round's apply batch slot
__global__ void scale_by_norm_kernel(cplx* y, const cplx* __restrict__ x, const double* nrm2, std::size_t n,
                                     cplx* y2 = nullptr) {
  pdl_trigger();
  pdl_wait();
  const double s = *nrm2;
  const double a = s > 0.0 ? 1.0 / std::sqrt(s) : 0.0;
  for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const cplx v = a * ldg(x + e);
    y[e] = v;
    if (y2) y2[e] = v;
  }
}

// x[e] += sum_k y[k] V_k[e] in k order (cie.cpp:213-214)
__global__ void combine_kernel(cplx* x, const cplx* __restrict__ V, std::size_t vstride, int nv,
                               const double* __restrict__ y, std::size_t n) {
  for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    cplx acc = x[e];
    for (int k = 0; k < nv; ++k) acc = acc + cplx{y[2 * k], y[2 * k + 1]} * ldg(V + k * vstride + e);
    x[e] = acc;
  }
}

// r[e] = b[e] - t[e], per-block |r|^2 partials
__global__ void __launch_bounds__(kRedThreads) residual_kernel(cplx* r, const cplx* __restrict__ b,
                                                               const cplx* __restrict__ t,
                                                               std::size_t n, double* partial) {
  double acc[1] = {0.0};
  for (std::size_t e = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const cplx v = ldg(b + e) - ldg(t + e);
    r[e] = v;
    acc[0] = fma(v.re, v.re, fma(v.im, v.im, acc[0]));
  }
  __shared__ double tot[1];
  block_sum<1>(acc, tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot[0];
}

using cd = std::complex<double>;

// reference make_rotation (cie.cpp:100-113)
void make_rotation(cd f, cd g, double& c, cd& s) {
  if (g == 0.0) {
    c = 1.0;
    s = 0.0;
  } else if (f == 0.0) {
    c = 0.0;
    s = std::conj(g) / std::abs(g);
  } else {
    const double t = std::sqrt(std::norm(f) + std::norm(g));
    c = std::abs(f) / t;
    s = f / std::abs(f) * std::conj(g) / t;
  }
}

// tiled sweep launch: grid = kCgsBlocks (or fewer tiles), one CTA per SM
template <int MODE>
int cgs_launch(cplx* w, const cplx* V, std::size_t vstride, int nv, const double* h, std::size_t n,
               double* partial, int pstride, int with_norm, cudaStream_t st, cplx* Vlast = nullptr) {
  const std::size_t smem = cgs_smem(kTileMaxV);
  (void)resident_ctas(reinterpret_cast<const void*>(cgs_tile_kernel<MODE>), kCgsThreads, smem);
  const int G = static_cast<int>(std::max<std::size_t>(
      1, std::min<std::size_t>(kCgsBlocks, (n + kTE - 1) / kTE)));
  launch_pdl(cgs_tile_kernel<MODE>, G, kCgsThreads, cgs_smem(nv), st, w, V, vstride, nv, h, n, partial, pstride,
             with_norm, Vlast);
  check_launch("cgs_tile_kernel");
  return G;
}

struct Workspace {
  cudaStream_t st;
  std::size_t n;  // complex entries per field
  int G;          // reduction blocks
  double* partial = nullptr;  // G x pstride
  double* dvals = nullptr;    // finalized values
  double* hpin = nullptr;     // pinned host mirror
  int pstride = 0;

  Workspace(cudaStream_t s, std::size_t n_, int maxv) : st(s), n(n_) {
    G = red_blocks(n);
    pstride = 4 * maxv + 4;  // DCGS2 dots: 4 nv values per block
    // rows for the reduction kernels' blocks and the tiled sweeps' (cgs_launch)
    partial = scratch<double>(static_cast<std::size_t>(std::max(G, kCgsBlocks)) * pstride, st);
    dvals = scratch<double>(pstride, st);
    EMIE_CUDA(cudaMallocHost(&hpin, pstride * sizeof(double)));
  }
  ~Workspace() {
    release(partial, st);
    release(dvals, st);
    cudaFreeHost(hpin);
  }

  // dots of w against nv vectors (+ |w|^2): values land in dvals and hpin
  void dots(const cplx* V, std::size_t vstride, int nv, const cplx* w, bool with_norm) {
    dots_kernel<<<G, kRedThreads, 0, st>>>(V, vstride, nv, w, n, partial, pstride, with_norm);
    check_launch("dots_kernel");
    finalize(2 * nv + (with_norm ? 1 : 0), with_norm ? 0 : -1);
  }
  // finalize partial sums; when norm_slot_src >= 0 the |w|^2 lives at 2*nv
  void finalize(int nvals, int) {
    launch_pdl(finalize_kernel, nvals, kFinThreads, 0, st, partial, G, pstride, nvals, dvals);
    check_launch("finalize_kernel");
  }
  double norm_of(const cplx* w) {
    dots_kernel<<<G, kRedThreads, 0, st>>>(w, 0, 0, w, n, partial, pstride, 1);
    check_launch("dots_kernel");
    launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, partial, G, pstride, 1, dvals);
    check_launch("finalize_kernel");
    fetch(1);
    return std::sqrt(hpin[0]);
  }
  void fetch(int nvals) {
    EMIE_CUDA(cudaMemcpyAsync(hpin, dvals, nvals * sizeof(double), cudaMemcpyDeviceToHost, st));
    EMIE_CUDA(cudaStreamSynchronize(st));
  }
};

// one right-hand side's FGMRES state, advanced between operator applies
struct Rhs {
  enum Phase { kInner, kResidual, kDone };
  int idx = 0;
  Phase phase = kDone;
  cplx* x = nullptr;    // solution (device)
  const cplx* b = nullptr;
  cplx* r = nullptr;    // residual (device)
  cplx* V = nullptr;    // basis (m+1) vectors (device)
  cplx* w = nullptr;    // apply output (device)
  cplx* Z = nullptr;    // preconditioned directions m vectors (device; flexible FGMRES only)
  double bnorm = 0, rnorm = 0;
  int iter = 0, j = 0, cols = 0;
  bool broke = false;
  std::vector<cd> h, g, rot_s;
  std::vector<double> rot_c, history;
  // DCGS2: unrotated Hessenberg columns, g before each rotation, the norms
  // rho_j of the once-projected w_j, v_j's correction a_j and alpha_j
  std::vector<cd> hraw, gpre, acoef;
  std::vector<double> rho, alpha;
  emie_cu_report rep{1, 0, 0.0, 0};
  // finalized reductions of the current step (device) and their pinned host
  // mirror: [0] pass-1 dots + |w|^2, [1] pass-2 dots, [2] the new norm
  double* dv = nullptr;
  double* hp = nullptr;
};

}  // namespace

void fgmres_device(const System& sys, const cplx* d_rhs, cplx* d_x, int nrhs, double tol,
                   int m, int max_iters, emie_cu_report* reports, double* h_history,
                   int hist_cap, cudaStream_t st) {
  KrylovMap A;
  A.n = 3 * sys.op->cells();
  A.apply = [&sys](const cplx* in, cplx* out, int nb, cudaStream_t s) { apply_b(*sys.op, in, out, nb, &sys, s); };
  fgmres_map(A, d_rhs, d_x, nrhs, tol, m, max_iters, reports, h_history, hist_cap, st);
}

void fgmres_map(const KrylovMap& A, const cplx* d_rhs, cplx* d_x, int nrhs, double tol, int m, int max_iters,
                emie_cu_report* reports, double* h_history, int hist_cap, cudaStream_t st) {
  if (!(tol > 0.0) || m < 1 || max_iters < 1)
    fail(EMIE_CU_INVALID_ARGUMENT, "fgmres: bad solver configuration");
  const std::size_t n = A.n;
  Workspace ws(st, n, m + 1);
  const int T = 256;
  const int GB = red_blocks(n);

  // device storage: basis V[r][m+1][n], residual, apply in/out batches
  cplx* Vall = scratch<cplx>(static_cast<std::size_t>(nrhs) * (m + 1) * n, st);
  cplx* Rall = scratch<cplx>(static_cast<std::size_t>(nrhs) * n, st);
  cplx* Wall = scratch<cplx>(static_cast<std::size_t>(nrhs) * n, st);
  cplx* Bin = scratch<cplx>(static_cast<std::size_t>(nrhs) * n, st);
  double* ycoef = scratch<double>(2 * (m + 1), st);
  // flexible right preconditioning: the directions z_j = M v_j (cie.cpp:151-153)
  cplx* Zall = A.precond ? scratch<cplx>(static_cast<std::size_t>(nrhs) * m * n, st) : nullptr;

  std::vector<Rhs> rs(nrhs);
  const int ps = ws.pstride;
  // orthogonalisation: DCGS2 (two sweeps per step) unless EMIE_CU_DCGS2=0 or
  // the restart exceeds the tiled sweeps' basis cap (CGS2, three sweeps)
  static const bool dcgs2_env = [] {
    const char* e = std::getenv("EMIE_CU_DCGS2");
    return !(e && e[0] == '0');
  }();
  const bool dcgs2 = dcgs2_env && m + 1 <= kTileMaxV;
  double* dsum = scratch<double>(4 * static_cast<std::size_t>(m + 1) + 4, st);
  double* dcoef = scratch<double>(4 * static_cast<std::size_t>(m + 1) + 4, st);
  // finalized reductions per rhs, two rounds deep (parity): [par][3][ps]
  double* dv_all = scratch<double>(static_cast<std::size_t>(nrhs) * 6 * ps, st);
  struct Pinned {  // freed on every exit path
    double* p = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Pinned() {
      cudaFreeHost(p);
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    }
  } pinned;
  EMIE_CUDA(cudaMallocHost(&pinned.p, static_cast<std::size_t>(nrhs) * 6 * ps * sizeof(double)));
  for (cudaEvent_t& e : pinned.ev) EMIE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  double* hp_all = pinned.p;
  for (int i = 0; i < nrhs; ++i) {
    Rhs& R = rs[i];
    R.idx = i;
    R.dv = dv_all + static_cast<std::size_t>(i) * 6 * ps;
    R.hp = hp_all + static_cast<std::size_t>(i) * 6 * ps;
    R.x = d_x + i * n;
    R.b = d_rhs + i * n;
    R.r = Rall + i * n;
    R.V = Vall + static_cast<std::size_t>(i) * (m + 1) * n;
    R.w = Wall + i * n;
    if (Zall) R.Z = Zall + static_cast<std::size_t>(i) * m * n;
    EMIE_CUDA(cudaMemsetAsync(R.x, 0, n * sizeof(cplx), st));
    R.bnorm = ws.norm_of(R.b);
    if (R.bnorm == 0.0) {  // cie.cpp:124-128
      R.rep.status = 0;
      R.phase = Rhs::kDone;
      continue;
    }
    EMIE_CUDA(cudaMemcpyAsync(R.r, R.b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    R.rnorm = R.bnorm;
    R.phase = Rhs::kResidual;  // marker: start a cycle below
  }

  // start a restart cycle (cie.cpp:136-147); returns false when the
  // iteration budget is exhausted
  auto start_cycle = [&](Rhs& R) -> bool {
    if (!(R.iter < max_iters)) return false;
    scale_kernel<<<GB, T, 0, st>>>(R.V, R.r, 1.0 / R.rnorm, n);
    check_launch("scale_kernel");
    R.h.assign(static_cast<std::size_t>(m + 1) * m, cd(0.0));
    R.rot_c.assign(m, 0.0);
    R.rot_s.assign(m, cd(0.0));
    R.g.assign(m + 1, cd(0.0));
    if (dcgs2) {
      R.hraw.assign(static_cast<std::size_t>(m + 1) * m, cd(0.0));
      R.gpre.assign(m + 1, cd(0.0));
      R.acoef.assign(static_cast<std::size_t>(m + 1) * (m + 1), cd(0.0));
      R.rho.assign(m + 1, 0.0);
      R.alpha.assign(m + 1, 1.0);
    }
    R.g[0] = R.rnorm;
    R.cols = 0;
    R.j = 0;
    R.phase = Rhs::kInner;
    return true;
  };
  auto finish = [&](Rhs& R) {
    if (R.broke && R.rnorm / R.bnorm <= tol) R.rep.status = 0;  // cie.cpp:232-233
    R.phase = Rhs::kDone;
  };
  for (Rhs& R : rs)
    if (R.phase == Rhs::kResidual && !start_cycle(R)) finish(R);

  // end of a cycle: update x, then request the explicit residual
  auto close_cycle = [&](Rhs& R) {
    if (R.cols > 0) {  // back substitution (cie.cpp:205-215)
      std::vector<cd> y(R.cols);
      for (int k = R.cols - 1; k >= 0; --k) {
        cd acc = R.g[k];
        for (int l = k + 1; l < R.cols; ++l)
          acc -= R.h[static_cast<std::size_t>(l) * (m + 1) + k] * y[l];
        y[k] = acc / R.h[static_cast<std::size_t>(k) * (m + 1) + k];
      }
      if (dcgs2 && !R.Z) {
        // the applies saw v_j before its delayed correction: v_j(applied) =
        // alpha_j v_j + sum_{i<j} a_{j,i} v_i in the corrected basis V
        std::vector<cd> yc(R.cols);
        for (int i = 0; i < R.cols; ++i) {
          cd acc = R.alpha[i] * y[i];
          for (int jj = i + 1; jj < R.cols; ++jj) acc += R.acoef[static_cast<std::size_t>(jj) * (m + 1) + i] * y[jj];
          yc[i] = acc;
        }
        y.swap(yc);
      }
      EMIE_CUDA(cudaMemcpyAsync(ycoef, y.data(), R.cols * sizeof(cd), cudaMemcpyHostToDevice, st));
      combine_kernel<<<GB, T, 0, st>>>(R.x, R.Z ? R.Z : R.V, n, R.cols, ycoef, n);
      check_launch("combine_kernel");
      EMIE_CUDA(cudaStreamSynchronize(st));  // ycoef is reused by the next rhs
    }
    R.phase = Rhs::kResidual;
  };

  // One round = one batched apply of every listed right-hand side plus each
  // one's reductions (CGS2 for a basis vector, the residual norm for x), all
  // stream ordered; the finalized values land in the pinned mirror of round
  // parity `par`, and ev[par] marks their arrival. The reductions' update
  // coefficients are read on the device, so a round never waits for the host.
  struct Entry {
    Rhs* R;
    bool inner;
    int j;
    int slot;             // position in its round's batch (Bin / Wall slot)
    bool staged = false;  // v_j already written into its Bin slot (speculative normalisation)
  };
  auto enqueue_round = [&](const std::vector<Entry>& es, int par) {
    for (std::size_t q = 0; q < es.size(); ++q) {
      const Rhs& R = *es[q].R;  // es[q].slot == q
      const cplx* src = es[q].inner ? R.V + static_cast<std::size_t>(es[q].j) * n : R.x;
      if (es[q].inner && R.Z) {  // z_j = M v_j, then A z_j (cie.cpp:151-153)
        cplx* z = R.Z + static_cast<std::size_t>(es[q].j) * n;
        A.precond(src, z, st);
        src = z;
      }
      if (!es[q].staged)
        EMIE_CUDA(cudaMemcpyAsync(Bin + q * n, src, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    }
    A.apply(Bin, Wall, static_cast<int>(es.size()), st);
    for (std::size_t q = 0; q < es.size(); ++q) {
      Rhs& R = *es[q].R;
      cplx* w = Wall + q * n;
      double* dv = R.dv + par * 3 * ps;
      double* hp = R.hp + par * 3 * ps;
      auto to_host = [&](int slot, int nvals) {
        EMIE_CUDA(cudaMemcpyAsync(hp + slot * ps, dv + slot * ps, nvals * sizeof(double), cudaMemcpyDeviceToHost,
                                  st));
      };
      if (!es[q].inner) {  // cie.cpp:217-229
        residual_kernel<<<ws.G, kRedThreads, 0, st>>>(R.r, R.b, w, n, ws.partial);
        check_launch("residual_kernel");
        launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, ws.partial, ws.G, 1, 1, dv + 2 * ps);
        check_launch("finalize_kernel");
        to_host(2, 1);
        continue;
      }
      const int j = es[q].j;
      if (dcgs2) {
        // one dots sweep (v_j's delayed reorthogonalisation and w's
        // projection), the coefficients, one update sweep (v_j corrected in
        // place, w projected) with the new |w|^2
        const int nv = j + 1;
        int g = cgs_launch<3>(w, R.V, n, nv, nullptr, n, ws.partial, ps, 0, st);
        launch_pdl(finalize_kernel, 4 * nv, kFinThreads, 0, st, ws.partial, g, ps, 4 * nv, dsum);
        check_launch("finalize_kernel");
        launch_pdl(dcgs_coef_kernel, 1, 32, 0, st, dsum, nv, dcoef, dv, dv + ps);
        check_launch("dcgs_coef_kernel");
        to_host(0, 2 * nv + 1);
        to_host(1, 2 * nv - 1);
        g = cgs_launch<4>(w, R.V, n, nv, dcoef, n, ws.partial, 1, 0, st, R.V + static_cast<std::size_t>(j) * n);
        launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, ws.partial, g, 1, 1, dv + 2 * ps);
        check_launch("finalize_kernel");
        to_host(2, 1);
        continue;
      }
      // CGS2 pass 1: dots against v_0..v_j plus |w|^2, then w -= V h
      if (j + 1 <= kTileMaxV) {
        int g = cgs_launch<0>(w, R.V, n, j + 1, nullptr, n, ws.partial, ps, 1, st);
        launch_pdl(finalize_kernel, 2 * (j + 1) + 1, kFinThreads, 0, st, ws.partial, g, ps, 2 * (j + 1) + 1, dv);
        check_launch("finalize_kernel");
        to_host(0, 2 * (j + 1) + 1);
        // w -= V h1 fused with the pass-2 dots, then w -= V h2 with the new norm
        g = cgs_launch<1>(w, R.V, n, j + 1, dv, n, ws.partial, ps, 0, st);
        launch_pdl(finalize_kernel, 2 * (j + 1), kFinThreads, 0, st, ws.partial, g, ps, 2 * (j + 1), dv + ps);
        check_launch("finalize_kernel");
        to_host(1, 2 * (j + 1));
        g = cgs_launch<2>(w, R.V, n, j + 1, dv + ps, n, ws.partial, 1, 0, st);
        launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, ws.partial, g, 1, 1, dv + 2 * ps);
        check_launch("finalize_kernel");
        to_host(2, 1);
        continue;
      }
      dots_kernel<<<ws.G, kRedThreads, 0, st>>>(R.V, n, j + 1, w, n, ws.partial, ps, 1);
      check_launch("dots_kernel");
      launch_pdl(finalize_kernel, 2 * (j + 1) + 1, kFinThreads, 0, st, ws.partial, ws.G, ps, 2 * (j + 1) + 1, dv);
      check_launch("finalize_kernel");
      to_host(0, 2 * (j + 1) + 1);
      update_kernel<<<ws.G, kRedThreads, 0, st>>>(w, R.V, n, j + 1, dv, n, nullptr);
      check_launch("update_kernel");
      // pass 2, with the new |w|^2
      dots_kernel<<<ws.G, kRedThreads, 0, st>>>(R.V, n, j + 1, w, n, ws.partial, ps, 0);
      check_launch("dots_kernel");
      launch_pdl(finalize_kernel, 2 * (j + 1), kFinThreads, 0, st, ws.partial, ws.G, ps, 2 * (j + 1), dv + ps);
      check_launch("finalize_kernel");
      to_host(1, 2 * (j + 1));
      update_kernel<<<ws.G, kRedThreads, 0, st>>>(w, R.V, n, j + 1, dv + ps, n, ws.partial);
      check_launch("update_kernel");
      launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, ws.partial, ws.G, 1, 1, dv + 2 * ps);
      check_launch("finalize_kernel");
      to_host(2, 1);
    }
    EMIE_CUDA(cudaEventRecord(pinned.ev[par], st));
  };

  // host side of a processed round entry (cie.cpp:148-203 / 217-229);
  // `scaled`: the next basis vector was already normalised on the device.
  // Returns true when the rhs goes on with inner step j + 1.
  auto process = [&](const Entry& e, int par, bool scaled) -> bool {
    Rhs& R = *e.R;
    const double* hp = R.hp + par * 3 * ps;
    cplx* w = Wall + static_cast<std::size_t>(e.slot) * n;
    if (!e.inner) {
      R.rnorm = std::sqrt(hp[2 * ps]);
      if (R.rnorm / R.bnorm <= tol) {
        R.rep.status = 0;
        finish(R);
      } else if (R.broke) {
        R.rep.status = 2;
        finish(R);
      } else if (!start_cycle(R)) {
        finish(R);
      }
      return false;
    }
    ++R.iter;
    const int j = R.j;
    cd* hj = R.h.data() + static_cast<std::size_t>(j) * (m + 1);
    const double wn0 = std::sqrt(hp[2 * (j + 1)]);
    const double hnext = std::sqrt(hp[2 * ps]);
    if (dcgs2) {
      // v_j was applied before its second projection: v_j(applied) =
      // alpha v_j + V a, so column j - 1 gains rho_{j-1} a and its subdiagonal
      // becomes rho_{j-1} alpha; it is re-rotated from its raw entries
      const double alpha = hp[ps + 2 * j];
      R.alpha[j] = alpha;
      for (int i = 0; i < j; ++i)
        R.acoef[static_cast<std::size_t>(j) * (m + 1) + i] = cd(hp[ps + 2 * i], hp[ps + 2 * i + 1]);
      if (j >= 1) {
        cd* hr = R.hraw.data() + static_cast<std::size_t>(j - 1) * (m + 1);
        for (int i = 0; i < j; ++i) hr[i] += R.rho[j - 1] * R.acoef[static_cast<std::size_t>(j) * (m + 1) + i];
        hr[j] = R.rho[j - 1] * alpha;
        cd* hc = R.h.data() + static_cast<std::size_t>(j - 1) * (m + 1);
        for (int i = 0; i <= j; ++i) hc[i] = hr[i];
        for (int i = 0; i < j - 1; ++i) {
          const cd t = R.rot_c[i] * hc[i] + R.rot_s[i] * hc[i + 1];
          hc[i + 1] = -std::conj(R.rot_s[i]) * hc[i] + R.rot_c[i] * hc[i + 1];
          hc[i] = t;
        }
        make_rotation(hc[j - 1], hc[j], R.rot_c[j - 1], R.rot_s[j - 1]);
        const cd t = R.rot_c[j - 1] * hc[j - 1] + R.rot_s[j - 1] * hc[j];
        hc[j] = 0.0;
        hc[j - 1] = t;
        R.g[j] = -std::conj(R.rot_s[j - 1]) * R.gpre[j - 1];
        R.g[j - 1] = R.rot_c[j - 1] * R.gpre[j - 1];
      }
      cd* hr = R.hraw.data() + static_cast<std::size_t>(j) * (m + 1);
      for (int i = 0; i <= j; ++i) hj[i] = hr[i] = cd(hp[2 * i], hp[2 * i + 1]);
      hr[j + 1] = hnext;
      R.rho[j] = hnext;
    } else {
      for (int i = 0; i <= j; ++i) hj[i] += cd(hp[2 * i], hp[2 * i + 1]);
      for (int i = 0; i <= j; ++i) hj[i] += cd(hp[ps + 2 * i], hp[ps + 2 * i + 1]);
    }
    for (int i = 0; i < j; ++i) {
      const cd t = R.rot_c[i] * hj[i] + R.rot_s[i] * hj[i + 1];
      hj[i + 1] = -std::conj(R.rot_s[i]) * hj[i] + R.rot_c[i] * hj[i + 1];
      hj[i] = t;
    }
    bool end_inner = false;
    if (hnext <= 1e-13 * std::max(wn0, 1e-300)) {
      double colmax = hnext;
      for (int i = 0; i <= j; ++i) colmax = std::max(colmax, std::abs(hj[i]));
      if (std::abs(hj[j]) > 1e-13 * std::max(colmax, 1e-300)) {
        R.cols = j + 1;
      } else {
        R.cols = j;
        R.broke = true;
        R.history.push_back(R.rnorm / R.bnorm);
        if (A.on_iteration) A.on_iteration(R.idx, R.iter, R.rnorm / R.bnorm);
      }
      end_inner = true;
    } else {
      hj[j + 1] = hnext;
      if (!scaled) {
        scale_kernel<<<GB, T, 0, st>>>(R.V + static_cast<std::size_t>(j + 1) * n, w, 1.0 / hnext, n);
        check_launch("scale_kernel");
      }
      make_rotation(hj[j], hnext, R.rot_c[j], R.rot_s[j]);
      const cd t = R.rot_c[j] * hj[j] + R.rot_s[j] * hj[j + 1];
      hj[j + 1] = 0.0;
      hj[j] = t;
      if (dcgs2) R.gpre[j] = R.g[j];
      R.g[j + 1] = -std::conj(R.rot_s[j]) * R.g[j];
      R.g[j] = R.rot_c[j] * R.g[j];
      R.cols = j + 1;
      const double est = std::abs(R.g[j + 1]) / R.bnorm;
      R.history.push_back(est);
      if (A.on_iteration) A.on_iteration(R.idx, R.iter, est);
      if (est <= tol) end_inner = true;
    }
    if (!end_inner) {
      ++R.j;
      if (!(R.j < m && R.iter < max_iters)) end_inner = true;
    }
    if (end_inner) {
      close_cycle(R);
      return false;
    }
    return true;
  };

  // Pipeline: while the host reads round k's reductions, the device already
  // runs round k + 1 for every rhs that can only go on with its next inner
  // step (speculation: the next basis vector is normalised on the device,
  // then applied and orthogonalised). A rhs that instead converges or breaks
  // down at round k discards its speculative work (never read: it only
  // touches the unused next basis slot and scratch) and the pipeline drains
  // once so its residual apply batches with the others again.
  std::vector<Entry> pending;
  int par = 0;
  bool drain = false;
  while (true) {
    if (pending.empty()) {
      for (Rhs& R : rs)
        if (R.phase == Rhs::kInner || R.phase == Rhs::kResidual)
          pending.push_back({&R, R.phase == Rhs::kInner, R.j, static_cast<int>(pending.size())});
      if (pending.empty()) break;
      enqueue_round(pending, par);
    }
    bool spec = !drain && A.speculate;
    for (const Entry& e : pending)
      if (!e.inner || !(e.j + 1 < m && e.R->iter + 1 < max_iters)) spec = false;
    std::vector<Entry> next;
    if (spec) {
      for (std::size_t q = 0; q < pending.size(); ++q) {
        const Entry& e = pending[q];
        const Rhs& R = *e.R;
        // the normalised v_{j+1} also lands in its slot of the next round's
        // apply batch (no preconditioner: the batch holds v itself)
        const bool stage = !R.Z;
        scale_by_norm_kernel<<<GB, T, 0, st>>>(R.V + static_cast<std::size_t>(e.j + 1) * n,
                                               Wall + static_cast<std::size_t>(e.slot) * n,
                                               R.dv + par * 3 * ps + 2 * ps, n,
                                               stage ? Bin + q * n : nullptr);
        check_launch("scale_by_norm_kernel");
        next.push_back({e.R, true, e.j + 1, static_cast<int>(q), stage});
      }
      enqueue_round(next, par ^ 1);
    }
    EMIE_CUDA(cudaEventSynchronize(pinned.ev[par]));
    std::vector<Entry> keep;
    bool all = true;
    for (std::size_t q = 0; q < pending.size(); ++q) {
      const bool goes_on = process(pending[q], par, spec);
      if (spec && goes_on) keep.push_back(next[q]);
      all = all && goes_on;
    }
    drain = spec && !all;
    if (spec) {
      pending = keep;  // their speculative round is exactly their next step
      par ^= 1;
    } else {
      pending.clear();
    }
  }
  // the speculative rounds of finished rhs may still run: wait before releasing
  EMIE_CUDA(cudaStreamSynchronize(st));

  for (int i = 0; i < nrhs; ++i) {
    Rhs& R = rs[i];
    R.rep.iterations = R.iter;
    R.rep.residual = R.bnorm == 0.0 ? 0.0 : R.rnorm / R.bnorm;
    R.rep.history_len = static_cast<int>(R.history.size());
    if (reports) reports[i] = R.rep;
    if (h_history)
      for (int k = 0; k < hist_cap && k < static_cast<int>(R.history.size()); ++k)
        h_history[static_cast<std::size_t>(i) * hist_cap + k] = R.history[k];
  }
  release(Vall, st);
  release(Rall, st);
  release(Wall, st);
  release(Bin, st);
  release(ycoef, st);
  release(dsum, st);
  release(dcoef, st);
  release(dv_all, st);
  if (Zall) release(Zall, st);
  EMIE_CUDA(cudaStreamSynchronize(st));
}

// ---- slab vector operations of the sharded FGMRES (distributed.py) --------
// Local sums over this rank's slab, finalized on the device into `out`; the
// caller all-reduces them across ranks. Same kernels as fgmres_device.
void vec_dots(const cplx* V, std::size_t vstride, int nv, const cplx* w, std::size_t n, bool with_norm,
              double* out, cudaStream_t st) {
  const int ps = 2 * nv + 2;
  const int nvals = 2 * nv + (with_norm ? 1 : 0);
  double* partial = scratch<double>(static_cast<std::size_t>(std::max(red_blocks(n), kCgsBlocks)) * ps, st);
  int g;
  if (nv >= 1 && nv <= kTileMaxV) {
    g = cgs_launch<0>(const_cast<cplx*>(w), V, vstride, nv, nullptr, n, partial, ps, with_norm ? 1 : 0, st);
  } else {
    g = red_blocks(n);
    dots_kernel<<<g, kRedThreads, 0, st>>>(V, vstride, nv, w, n, partial, ps, with_norm ? 1 : 0);
    check_launch("dots_kernel");
  }
  if (nvals > 0) {
    launch_pdl(finalize_kernel, nvals, kFinThreads, 0, st, partial, g, ps, nvals, out);
    check_launch("finalize_kernel");
  }
  release(partial, st);
}

void vec_dcgs_dots(const cplx* V, std::size_t vstride, int nv, const cplx* w, std::size_t n, double* out,
                   cudaStream_t st) {
  if (nv < 1 || nv > kTileMaxV) fail(EMIE_CU_INVALID_ARGUMENT, "vec_dcgs_dots: nv outside [1, 41]");
  const int ps = 4 * nv + 4;
  double* partial = scratch<double>(static_cast<std::size_t>(kCgsBlocks) * ps, st);
  const int g = cgs_launch<3>(const_cast<cplx*>(w), V, vstride, nv, nullptr, n, partial, ps, 0, st);
  launch_pdl(finalize_kernel, 4 * nv, kFinThreads, 0, st, partial, g, ps, 4 * nv, out);
  check_launch("finalize_kernel");
  release(partial, st);
}

void vec_dcgs_update(cplx* w, cplx* V, std::size_t vstride, int nv, const double* coef, std::size_t n,
                     double* norm_out, cudaStream_t st) {
  if (nv < 1 || nv > kTileMaxV) fail(EMIE_CU_INVALID_ARGUMENT, "vec_dcgs_update: nv outside [1, 41]");
  double* partial = scratch<double>(kCgsBlocks, st);
  const int g = cgs_launch<4>(w, V, vstride, nv, coef, n, partial, 1, 0, st, V + (nv - 1) * vstride);
  launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, partial, g, 1, 1, norm_out);
  check_launch("finalize_kernel");
  release(partial, st);
}

void vec_update(cplx* w, const cplx* V, std::size_t vstride, int nv, const double* h, std::size_t n,
                double* dots_out, double* norm_out, cudaStream_t st) {
  const int ps = 2 * nv + 2;
  double* partial = scratch<double>(static_cast<std::size_t>(std::max(red_blocks(n), kCgsBlocks)) * ps, st);
  const bool tiled = nv >= 1 && nv <= kTileMaxV;
  if (tiled && dots_out && !norm_out) {
    const int g = cgs_launch<1>(w, V, vstride, nv, h, n, partial, ps, 0, st);
    launch_pdl(finalize_kernel, 2 * nv, kFinThreads, 0, st, partial, g, ps, 2 * nv, dots_out);
    check_launch("finalize_kernel");
  } else if (tiled && !dots_out) {
    const int g = cgs_launch<2>(w, V, vstride, nv, h, n, partial, 1, 0, st);
    if (norm_out) {
      launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, partial, g, 1, 1, norm_out);
      check_launch("finalize_kernel");
    }
  } else {
    const int g = red_blocks(n);
    if (nv > 0) {
      update_kernel<<<g, kRedThreads, 0, st>>>(w, V, vstride, nv, h, n, norm_out ? partial : nullptr);
      check_launch("update_kernel");
    }
    if (norm_out) {
      if (nv == 0) {
        dots_kernel<<<g, kRedThreads, 0, st>>>(w, 0, 0, w, n, partial, 1, 1);
        check_launch("dots_kernel");
      }
      launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, partial, g, 1, 1, norm_out);
      check_launch("finalize_kernel");
    }
    if (dots_out && nv > 0) {
      dots_kernel<<<g, kRedThreads, 0, st>>>(V, vstride, nv, w, n, partial, ps, 0);
      check_launch("dots_kernel");
      launch_pdl(finalize_kernel, 2 * nv, kFinThreads, 0, st, partial, g, ps, 2 * nv, dots_out);
      check_launch("finalize_kernel");
    }
  }
  release(partial, st);
}

void vec_combine(cplx* x, const cplx* V, std::size_t vstride, int nv, const double* y, std::size_t n,
                 cudaStream_t st) {
  if (nv < 1) return;
  combine_kernel<<<red_blocks(n), 256, 0, st>>>(x, V, vstride, nv, y, n);
  check_launch("combine_kernel");
}

void vec_scale(cplx* y, const cplx* x, double a, std::size_t n, cudaStream_t st) {
  scale_kernel<<<red_blocks(n), 256, 0, st>>>(y, x, a, n);
  check_launch("scale_kernel");
}

void vec_residual(cplx* r, const cplx* b, const cplx* t, std::size_t n, double* norm_out, cudaStream_t st) {
  const int g = red_blocks(n);
  double* partial = scratch<double>(static_cast<std::size_t>(g), st);
  residual_kernel<<<g, kRedThreads, 0, st>>>(r, b, t, n, partial);
  check_launch("residual_kernel");
  launch_pdl(finalize_kernel, 1, kFinThreads, 0, st, partial, g, 1, 1, norm_out);
  check_launch("finalize_kernel");
  release(partial, st);
}

}  // namespace emie_cu
