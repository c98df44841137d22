// Lateral (x, y) transforms of the operator apply and of the spectra build,
// for sm_100a. Every kernel loads a tile of transforms from HBM with a
// coalesced mapping (doing the zero padding, the r2 scaling or the parity
// embedding on the way in), transforms it in shared memory and stores it in
// the layout the next stage reads, so there is one HBM round trip per pass.
//
// Two engines: power-of-two lengths (every benchmark grid) run the in-place
// radix-16 Stockham (fft.cuh, fft_pow2); other 5-smooth lengths (the
// reference's 3, 9, 12-point test grids) the ping-pong mixed-radix one.
//
// Reference: src/toeplitz.cpp:92-161 (spectra), 163-283 (apply), cie.cpp:56-73.
#include <cstdlib>
#include <algorithm>

#include <cudaTypedefs.h>

#include "operator.cuh"
#include "tma.cuh"

namespace emie_cu {

namespace {

__constant__ int kParX[6] = {1, 1, 1, -1, -1, 1};  // toeplitz.cpp:59
__constant__ int kParY[6] = {1, 1, 1, -1, 1, -1};  // toeplitz.cpp:60

__device__ __forceinline__ int comp_of(int e, int ntri, int nfull) {
  return e < 4 * ntri ? e / ntri : 4 + (e - 4 * ntri) / nfull;
}

// SMEM tile of ntr transforms of length n for either engine
template <bool P2>
struct Tile {
  cplx* a;
  cplx* b;
  cplx* tw;
  int n, ld;
  __device__ Tile(cplx* sm, int ntr, int n_) : n(n_) {
    if (P2) {
      ld = fft_ldp(n);
      a = sm;
      b = nullptr;
      tw = sm + ntr * ld;
    } else {
      ld = n | 1;  // odd: column walks hit distinct banks
      a = sm;
      b = sm + ntr * ld;
      tw = b + ntr * ld;
    }
  }
  __device__ __forceinline__ int at(int t, int j) const { return P2 ? fft_phys2(t, j, ld) : t * ld + j; }
  __device__ cplx* run(int ntr, const FftPlan& pl, bool inverse) {
    if (P2) {
      fft_pow2(a, ntr, pl, tw, inverse);
      return a;
    }
    return fft_smem(a, b, ld, ntr, pl, tw, inverse);
  }
};

// Fill a tile through fetch(idx, pos) -> value. On the power-of-two path
// every thread issues all of its kFftEPT global loads before the first SMEM
// store, so each thread keeps 16 independent loads in flight.
template <bool P2, class F>
__device__ __forceinline__ void fill_tile(Tile<P2>& T, int total, F&& fetch) {
  if constexpr (P2) {
    cplx v[kFftEPT];
    int pos[kFftEPT];
#pragma unroll
    for (int e = 0; e < kFftEPT; ++e) {
      const int idx = threadIdx.x + e * blockDim.x;
      v[e] = idx < total ? fetch(idx, pos[e]) : cplx{0.0, 0.0};
      if (idx >= total) pos[e] = -1;
    }
#pragma unroll
    for (int e = 0; e < kFftEPT; ++e)
      if (pos[e] >= 0) T.a[pos[e]] = v[e];
  } else {
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      int pos;
      const cplx v = fetch(idx, pos);
      T.a[pos] = v;
    }
  }
}

size_t tile_bytes(bool p2, int ntr, int n) {
  const size_t e = p2 ? static_cast<size_t>(ntr) * fft_ldp(n) + n
                      : 2 * static_cast<size_t>(ntr) * (n | 1) + n;
  return e * sizeof(cplx);
}

// ------------------------------------------------------------- spectra ----
// x pass over rows oi of the parity-extended offset sequence
// (toeplitz.cpp:140-151) for EC consecutive entries e; keep mx < qx:
// R[(oi*qx + mx)*nent + e]
template <bool P2>
__global__ void __launch_bounds__(256, 2) spectra_x_kernel(const cplx* __restrict__ blocks, cplx* __restrict__ R,
                                 const cplx* __restrict__ tw, FftPlan pl, int nx, int qx, int nent,
                                 int ntri, int nfull, int EC) {
  extern __shared__ cplx sm[];
  const int ex = pl.n;
  Tile<P2> T(sm, EC, ex);
  const int oi = blockIdx.x;
  const int e0 = blockIdx.y * EC;
  load_twiddles(T.tw, tw, ex);
  for (int idx = threadIdx.x; idx < EC * ex; idx += blockDim.x) {
    const int tt = idx % EC, j = idx / EC;
    const int e = e0 + tt;
    cplx v = {0.0, 0.0};
    if (e < nent) {
      const int c = comp_of(e, ntri, nfull);
      if (j < nx) {
        v = ldg(blocks + (static_cast<size_t>(oi) * nx + j) * nent + e);
      } else if (j > ex - nx) {
        v = static_cast<double>(kParX[c]) * ldg(blocks + (static_cast<size_t>(oi) * nx + (ex - j)) * nent + e);
      }
    }
    T.a[T.at(tt, j)] = v;
  }
  __syncthreads();
  const cplx* res = T.run(EC, pl, false);
  for (int idx = threadIdx.x; idx < EC * qx; idx += blockDim.x) {
    const int tt = idx % EC, mx = idx / EC;
    const int e = e0 + tt;
    if (e < nent) R[(static_cast<size_t>(oi) * qx + mx) * nent + e] = res[T.at(tt, mx)];
  }
}

// y pass, parity-extended in oi; keep my < qy; store through emap into the
// wrapped-diagonal mode blocks (operator.cuh)
template <bool P2>
__global__ void __launch_bounds__(256, 2) spectra_y_kernel(const cplx* __restrict__ R, cplx* __restrict__ spec,
                                 const cplx* __restrict__ tw, FftPlan pl, int ny, int qx, int qy,
                                 int nent, int ntri, int nfull, int EC, const int2* __restrict__ emap,
                                 int nentD, int qbase, int qcount) {
  extern __shared__ cplx sm[];
  const int ey = pl.n;
  Tile<P2> T(sm, EC, ey);
  const int mx = blockIdx.x;
  const int e0 = blockIdx.y * EC;
  load_twiddles(T.tw, tw, ey);
  for (int idx = threadIdx.x; idx < EC * ey; idx += blockDim.x) {
    const int tt = idx % EC, j = idx / EC;
    const int e = e0 + tt;
    cplx v = {0.0, 0.0};
    if (e < nent) {
      const int c = comp_of(e, ntri, nfull);
      if (j < ny) {
        v = ldg(R + (static_cast<size_t>(j) * qx + mx) * nent + e);
      } else if (j > ey - ny) {
        v = static_cast<double>(kParY[c]) * ldg(R + (static_cast<size_t>(ey - j) * qx + mx) * nent + e);
      }
    }
    T.a[T.at(tt, j)] = v;
  }
  __syncthreads();
  const cplx* res = T.run(EC, pl, false);
  for (int idx = threadIdx.x; idx < EC * qy; idx += blockDim.x) {
    const int tt = idx % EC, my = idx / EC;
    const int e = e0 + tt;
    const int qm = my * qx + mx;  // stored: quadrant modes [qbase, qbase + qcount)
    if (e < nent && qm >= qbase && qm < qbase + qcount) {
      const int2 m = emap[e];
      cplx* blk = spec + static_cast<size_t>(qm - qbase) * nentD;
      const cplx v = res[T.at(tt, my)];
      blk[m.x] = v;
      if (m.y >= 0) blk[m.y] = v;
    }
  }
}

// --------------------------------------------------------------- apply ----
// Layouts (complex128):
//   u   [r][plane][iy][ix]        GridVector, plane = c*nz + iz
//   T   [r][mx][plane][iy]        after the x pass (and before the inverse x)
//   S   [r][mx][my][plane]        spectrum, mode-major for the contraction
// Every load and store below walks a contiguous run of >= 128 B.
// The mirror-mode signs of the contraction (D = diag(fx, fy, 1), fx = -1 for
// mx > ex/2 on x planes, fy = -1 for my > ey/2 on y planes) are applied when
// the spectrum is stored and again when it is read back, so the per-mode
// contraction is sign-free: out = D M D u.
__device__ __forceinline__ double mirror_sign(int plane, int nz, int my, int mx, int ey, int ex) {
  // component c = plane / nz without the division: x planes [0, nz), y planes [nz, 2nz)
  return ((plane < nz && 2 * mx > ex) || (plane >= nz && plane < 2 * nz && 2 * my > ey)) ? -1.0 : 1.0;
}

// forward x of rows iy0.. of plane pr = r*np + plane; r2 (cie.cpp:63-65) on load
template <bool P2>
__global__ void __launch_bounds__(256, 2) apply_fx_kernel(const cplx* __restrict__ u, const cplx* __restrict__ r2,
                                                          cplx* __restrict__ Tout, const cplx* __restrict__ tw,
                                                          FftPlan pl, int nx, int ny, int nz, int RT) {
  extern __shared__ cplx sm[];
  const int ex = pl.n, np = 3 * nz;
  Tile<P2> T(sm, RT, ex);
  const int pr = blockIdx.x, iy0 = blockIdx.y * RT;
  const int r = pr / np, plane = pr - r * np, iz = plane % nz;
  load_twiddles(T.tw, tw, ex);
  auto fetch = [&](int idx, int& pos) {
    const int tt = idx / ex, j = idx - tt * ex;
    const int iy = iy0 + tt;
    pos = T.at(tt, j);
    cplx v = {0.0, 0.0};
    if (tt < RT && iy < ny && j < nx) {
      v = ldg(u + (static_cast<size_t>(pr) * ny + iy) * nx + j);
      if (r2) v = ldg(r2 + (static_cast<size_t>(iz) * ny + iy) * nx + j) * v;
    }
    return v;
  };
  fill_tile<P2>(T, RT * ex, fetch);
  __syncthreads();
  const cplx* res = T.run(RT, pl, false);
  for (int idx = threadIdx.x; idx < RT * ex; idx += blockDim.x) {
    const int tt = idx % RT, mx = idx / RT;
    const int iy = iy0 + tt;
    if (iy < ny) Tout[((static_cast<size_t>(r) * ex + mx) * np + plane) * ny + iy] = res[T.at(tt, mx)];
  }
}

// forward y of PC planes at column mx; stores mode-major S with mirror signs
template <bool P2>
__global__ void __launch_bounds__(256, 2) apply_fy_kernel(const cplx* __restrict__ Tin, cplx* __restrict__ S,
                                                          const cplx* __restrict__ tw, FftPlan pl, int ny,
                                                          int ex, int nz, int PC) {
  extern __shared__ cplx sm[];
  const int ey = pl.n, np = 3 * nz;
  Tile<P2> T(sm, PC, ey);
  const int mx = blockIdx.x, p0 = blockIdx.y * PC, r = blockIdx.z;
  const int pc = min(PC, np - p0);
  load_twiddles(T.tw, tw, ey);
  const cplx* src = Tin + ((static_cast<size_t>(r) * ex + mx) * np + p0) * ny;
  auto fetch = [&](int idx, int& pos) {
    const int p = idx / ey, j = idx - p * ey;
    pos = T.at(p, j);
    return (j < ny && p < pc) ? ldg(src + p * ny + j) : cplx{0.0, 0.0};
  };
  fill_tile<P2>(T, PC * ey, fetch);
  __syncthreads();
  const cplx* res = T.run(PC, pl, false);
  for (int idx = threadIdx.x; idx < PC * ey; idx += blockDim.x) {
    const int p = idx % PC, my = idx / PC;
    if (p < pc)
      S[((static_cast<size_t>(r) * ex + mx) * ey + my) * np + p0 + p] =
          mirror_sign(p0 + p, nz, my, mx, ey, ex) * res[T.at(p, my)];
  }
}

// inverse y of PC planes at column mx (undoing the mirror signs on load);
// keeps rows iy < ny
template <bool P2>
__global__ void __launch_bounds__(256, 2) apply_iy_kernel(const cplx* __restrict__ S, cplx* __restrict__ Tout,
                                                          const cplx* __restrict__ tw, FftPlan pl, int ny,
                                                          int ex, int nz, int PC) {
  extern __shared__ cplx sm[];
  const int ey = pl.n, np = 3 * nz;
  Tile<P2> T(sm, PC, ey);
  const int mx = blockIdx.x, p0 = blockIdx.y * PC, r = blockIdx.z;
  const int pc = min(PC, np - p0);
  load_twiddles(T.tw, tw, ey);
  auto fetch = [&](int idx, int& pos) {
    const int p = idx % PC, j = idx / PC;
    pos = T.at(p, j);
    cplx v = {0.0, 0.0};
    if (p < pc && j < ey)
      v = mirror_sign(p0 + p, nz, j, mx, ey, ex) *
          ldg(S + ((static_cast<size_t>(r) * ex + mx) * ey + j) * np + p0 + p);
    return v;
  };
  fill_tile<P2>(T, PC * ey, fetch);
  __syncthreads();
  const cplx* res = T.run(PC, pl, true);
  cplx* dst = Tout + ((static_cast<size_t>(r) * ex + mx) * np + p0) * ny;
  for (int idx = threadIdx.x; idx < PC * ny; idx += blockDim.x) {
    const int p = idx / ny, iy = idx - p * ny;
    if (p < pc) dst[p * ny + iy] = res[T.at(p, iy)];
  }
}

// inverse x of rows iy0.. of plane pr, truncate, 1/(ex ey), optional system
// epilogue s*u + r1*(.) (toeplitz.cpp:260-282, cie.cpp:67-72)
template <bool P2>
__global__ void __launch_bounds__(256, 2) apply_ix_kernel(const cplx* __restrict__ Tin, const cplx* __restrict__ u,
                                                          cplx* __restrict__ out, const cplx* __restrict__ s,
                                                          const double* __restrict__ r1,
                                                          const cplx* __restrict__ tw, FftPlan pl, int nx,
                                                          int ny, int nz, int RT, double inv) {
  extern __shared__ cplx sm[];
  const int ex = pl.n, np = 3 * nz;
  Tile<P2> T(sm, RT, ex);
  const int pr = blockIdx.x, iy0 = blockIdx.y * RT;
  const int r = pr / np, plane = pr - r * np, iz = plane % nz;
  load_twiddles(T.tw, tw, ex);
  auto fetch = [&](int idx, int& pos) {
    const int tt = idx % RT, mx = idx / RT;
    const int iy = iy0 + tt;
    pos = T.at(tt, mx);
    return (iy < ny && mx < ex) ? ldg(Tin + ((static_cast<size_t>(r) * ex + mx) * np + plane) * ny + iy)
                                : cplx{0.0, 0.0};
  };
  fill_tile<P2>(T, RT * ex, fetch);
  __syncthreads();
  const cplx* res = T.run(RT, pl, true);
  for (int idx = threadIdx.x; idx < RT * nx; idx += blockDim.x) {
    const int tt = idx / nx, ix = idx - tt * nx;
    const int iy = iy0 + tt;
    if (iy >= ny) continue;
    const size_t q = (static_cast<size_t>(pr) * ny + iy) * nx + ix;
    cplx v = inv * res[T.at(tt, ix)];
    if (s) {
      const size_t cell = (static_cast<size_t>(iz) * ny + iy) * nx + ix;
      v = ldg(s + cell) * ldg(u + q) + __ldg(r1 + cell) * v;
    }
    out[q] = v;
  }
}

// ------------------------------------------- streaming power-of-two path ----
// Persistent double-buffered variant of the four apply passes for
// power-of-two lengths 16 <= N <= 2048 (every benchmark grid), with N a
// template parameter so all FFT index math folds to shifts and constants.
// A CTA owns tiles of kStreamElems elements (2048/N transforms); while it
// transforms tile i in one padded SMEM buffer, tile i+1 streams into the
// other through cp.async (16 B per request, written straight into the padded
// FFT layout), so every SM keeps HBM reads in flight through the compute and
// store phases. The first radix-16 pass reads only the nin nonzero inputs of
// each transform (the zero half of the embedding is never loaded) and applies
// the per-element prescaling (r2, mirror signs); the operands of the prescale
// and of the system epilogue are fetched into registers when the tile starts.
#ifndef EMIE_STREAM_EXPERIMENT
// timing experiments only: 1 no FFT passes, 2 no loads, 3 no loads or stores, 4 loads only
#define EMIE_STREAM_EXPERIMENT 0
#endif
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
#if EMIE_STREAM_EXPERIMENT != 2 && EMIE_STREAM_EXPERIMENT != 3
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

constexpr int kStreamThreads = 128;                     // threads per CTA
constexpr int kStreamElems = kStreamThreads * kFftEPT;  // 2048-element tiles
constexpr int kStreamPre = 8;                           // register-prefetched operands per thread

template <int N>
struct Geo {
  static constexpr int ntr = kStreamElems / N;  // transforms per tile
  static constexpr int ldp = N + N / 16 + 1;    // = fft_ldp(N)
  static constexpr int tile = ntr * ldp;        // padded tile, elements
  __device__ static __forceinline__ int at(int t, int j) { return t * ldp + j + (j >> 4); }
};

// radix-R pass at stride NS (Stockham, in place): kFftEPT/R butterflies per thread
template <int N, int R, int NS, bool INV>
__device__ __forceinline__ void spass(cplx* buf, const cplx* tw) {
  using G = Geo<N>;
  constexpr int B = kFftEPT / R, M = N / R, TSTEP = N / (NS * R);
  constexpr double s = INV ? 1.0 : -1.0;
  cplx v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int w = threadIdx.x + b * kStreamThreads;
    const int t = w / M, j = w % M, k = j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cplx x = buf[G::at(t, j + r * M)];
      if (NS > 1 && r > 0) {
        cplx wv = tw[r * k * TSTEP];
        if (INV) wv.im = -wv.im;
        x = x * wv;
      }
      v[b][r] = x;
    }
    butterfly<R>(v[b], s);
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int w = threadIdx.x + b * kStreamThreads;
    const int t = w / M, j = w % M, k = j % NS;
    const int j0 = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[G::at(t, j0 + r * NS)] = v[b][r];
  }
  __syncthreads();
}

// radix of the last pass: 16 when N is a power of 16, else the remainder
template <int N>
constexpr int last_radix() {
  int n = N;
  while (n > 16) n /= 16;
  return n;
}

// passes at strides NS .. < N / last_radix (the middle passes)
template <int N, int NS, bool INV>
__device__ __forceinline__ void smid(cplx* buf, const cplx* tw) {
  constexpr int NSL = N / last_radix<N>();
  if constexpr (NS < NSL) {
    spass<N, 16, NS, INV>(buf, tw);
    smid<N, NS * 16, INV>(buf, tw);
  }
}

// Last pass (stride NS = N/R): thread b-th butterfly w -> (transform t, j);
// output r of it is element jo = j + r*NS of transform t, handed to
// p.emit(ops, t, jo, b, r, value) straight from registers. TF: transform
// index fastest across lanes (fx, fy: their global rows run along t), else
// element index fastest (iy, ix).
template <int N, bool TF>
__device__ __forceinline__ void last_coord(int b, int& t, int& j) {
  constexpr int R = last_radix<N>(), NS = N / R, NT = Geo<N>::ntr;
  const int w = threadIdx.x + b * kStreamThreads;
  if (TF) {
    t = w % NT;
    j = w / NT;
  } else {
    t = w / NS;
    j = w % NS;
  }
}
template <int N, bool INV, class P>
__device__ __forceinline__ void slast(const cplx* buf, const cplx* tw, const P& p, const typename P::Ops& ops) {
  using G = Geo<N>;
  constexpr int R = last_radix<N>(), NS = N / R, B = kFftEPT / R;
  constexpr double s = INV ? 1.0 : -1.0;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    int t, j;
    last_coord<N, P::kTFast>(b, t, j);
    cplx v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cplx x = buf[G::at(t, j + r * NS)];
      if (r > 0) {
        cplx wv = tw[r * j];  // e^{-2 pi i r j / N}: TSTEP = 1 in the last pass
        if (INV) wv.im = -wv.im;
        x = x * wv;
      }
      v[r] = x;
    }
    butterfly<R>(v, s);
#pragma unroll
    for (int r = 0; r < R; ++r) p.template emit<N>(ops, t, j + r * NS, b, r, v[r]);
  }
}

// first radix-16 pass (NS = 1, no twiddles): one butterfly per thread; inputs
// at jj >= p.nin are zero; p.pre(ops, t, r, jj, x) scales input r
template <int N, bool INV, class P>
__device__ __forceinline__ void spass_first(cplx* buf, const P& p, const typename P::Ops& ops) {
  using G = Geo<N>;
  constexpr int M = N / 16;
  constexpr double s = INV ? 1.0 : -1.0;
  const int t = threadIdx.x / M, j = threadIdx.x % M;
  cplx v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int jj = j + r * M;
    v[r] = jj < p.nin ? p.pre(ops, t, r, jj, buf[G::at(t, jj)]) : cplx{0.0, 0.0};
  }
  butterfly<16>(v, s);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[G::at(t, 16 * j + r)] = v[r];
  __syncthreads();
}

// The persistent driver. P supplies ntiles(), load<N>(tile, buf) (cp.async),
// prefetch<N>(tile, ops), pre(ops, t, r, jj, x), nin and store<N>(tile, buf, ops).
#ifndef EMIE_STREAM_NBUF
#define EMIE_STREAM_NBUF 2
#endif
constexpr int kStreamBufs = EMIE_STREAM_NBUF;  // tile buffers per CTA (prefetch depth + 1)

template <int N, class P>
__global__ void __launch_bounds__(kStreamThreads, kStreamBufs == 2 ? 3 : 2)
    stream_fft_kernel(P p, const cplx* __restrict__ tw) {
  using G = Geo<N>;
  constexpr int NB = kStreamBufs;
  extern __shared__ cplx sm[];
  cplx* tws = sm + NB * G::tile;
  load_twiddles(tws, tw, N);
  const int ntiles = p.ntiles();
  int tile = blockIdx.x;
#pragma unroll
  for (int b = 0; b < NB - 1; ++b) {
    const int t = tile + b * gridDim.x;
    if (t < ntiles) p.template load<N>(t, sm + b * G::tile);
    cp_async_commit();
  }
#pragma unroll 1
  for (int i = 0; tile < ntiles; ++i, tile += gridDim.x) {
    cplx* cur = sm + (i % NB) * G::tile;
    const int next = tile + (NB - 1) * gridDim.x;
    if (next < ntiles) p.template load<N>(next, sm + ((i + NB - 1) % NB) * G::tile);
    cp_async_commit();
    typename P::Ops ops;
    p.template prefetch<N>(tile, ops);
    cp_async_wait<NB - 1>();
    __syncthreads();
#if EMIE_STREAM_EXPERIMENT != 1 && EMIE_STREAM_EXPERIMENT != 4
    spass_first<N, P::kInverse>(cur, p, ops);
    smid<N, 16, P::kInverse>(cur, tws);
#endif
    slast<N, P::kInverse>(cur, tws, p, ops);
    __syncthreads();  // cur is refilled by the next iteration's load
  }
  cp_async_wait<0>();
}

// TMA-staged variant (N = 256, the benchmark grids): a tile arrives by one
// bulk copy (contiguous rows: fx, fy) or one tensor-map box with 128-byte
// swizzle (strided rows: iy, ix) into a dense staging buffer; the first radix
// pass reads it (p.staged) and writes the padded work buffer, after which the
// staging buffer takes the next tile. Bulk copies keep far more bytes in
// flight per SM than per-thread cp.async (no L1 miss-queue limit).
#ifndef EMIE_TMA_MINB_SMALL
#define EMIE_TMA_MINB_SMALL 3  // CTAs per SM the register budget targets for 16 KB stages
#endif
template <int N, class P, int NST>
__global__ void __launch_bounds__(kStreamThreads, P::kStageBytes <= 16384 ? (NST == 1 ? EMIE_TMA_MINB_SMALL : 3)
                                                                           : (NST == 1 ? 3 : 2))
    stream_tma_kernel(const __grid_constant__ P p, const cplx* __restrict__ tw) {
  using G = Geo<N>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  pdl_trigger();
  cplx* stage[NST];
#pragma unroll
  for (int b = 0; b < NST; ++b) stage[b] = reinterpret_cast<cplx*>(smraw + b * P::kStageBytes);
  cplx* work = reinterpret_cast<cplx*>(smraw + NST * P::kStageBytes);
  cplx* tws = work + G::tile;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tws + N);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NST; ++b) mbar_init(bar + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_twiddles(tws, tw, N);
  __syncthreads();
  pdl_wait();  // the previous kernel's outputs (this pass's input) are complete
  const int ntiles = p.ntiles();
  int tile = blockIdx.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NST; ++b)
      if (tile + b * static_cast<int>(gridDim.x) < ntiles)
        p.template issue<N>(tile + b * gridDim.x, stage[b], bar + b);
  }
#pragma unroll 1
  for (int i = 0; tile < ntiles; ++i, tile += gridDim.x) {
    const int st = i % NST;
    typename P::Ops ops;
    p.template prefetch<N>(tile, ops);
    mbar_wait(bar + st, static_cast<uint32_t>((i / NST) & 1));
    {  // first radix-16 pass: staging -> work (NS = 1, no twiddles)
      constexpr int M = N / 16;
      constexpr double s = P::kInverse ? 1.0 : -1.0;
      const int t = threadIdx.x / M, j = threadIdx.x % M;
      cplx v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int jj = j + r * M;
        v[r] = jj < p.nin ? p.pre(ops, t, r, jj, p.template staged<N>(stage[st], t, jj)) : cplx{0.0, 0.0};
      }
      butterfly<16>(v, s);
#pragma unroll
      for (int r = 0; r < 16; ++r) work[G::at(t, 16 * j + r)] = v[r];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging reads before its TMA refill
      __syncthreads();  // staging[st] consumed, work filled
    }
    const int next = tile + NST * gridDim.x;
    if (threadIdx.x == 0 && next < ntiles) p.template issue<N>(next, stage[st], bar + st);
    smid<N, 16, P::kInverse>(work, tws);
    slast<N, P::kInverse>(work, tws, p, ops);
    __syncthreads();  // work is rewritten by the next tile's first pass
  }
}

// global store of the streaming passes
__device__ __forceinline__ void gst(cplx* p, cplx v) {
#if EMIE_STREAM_EXPERIMENT != 3 && EMIE_STREAM_EXPERIMENT != 4
  *p = v;
#endif
}

// Loops over a tile run a compile-time count: a power-of-two embedding of
// 2n-1 points has n in (N/4, N/2], so rows are walked as N/2-wide with a
// predicate. Thread-constant parts of the mirror signs are hoisted per tile.
template <int N>
struct Half {
  static constexpr int H = N / 2;                                   // row width walked
  static constexpr int per = (Geo<N>::ntr * H) / kStreamThreads;    // elements per thread
  __device__ static __forceinline__ void rc(int e, int& t, int& j) {  // element e of the thread
    const int idx = threadIdx.x + e * kStreamThreads;
    t = idx / H;
    j = idx % H;
  }
};

// x forward: tile = RT rows iy0.. of plane pr (nrhs*np planes); r2 on load
struct FxStream {
  static constexpr bool kInverse = false, kTFast = true;
  static constexpr int kRowBytes = 8 * 128 * 16;     // 8 rows of <= 128 points (N = 256) or 4 of <= 256 (N = 512)
#ifndef EMIE_FX_STAGE_R2
#define EMIE_FX_STAGE_R2 1  // 0: r2 by per-thread loads, 16 KB stages (two per CTA at three CTAs per SM)
#endif
  static constexpr bool kStageR2 = EMIE_FX_STAGE_R2;
  static constexpr int kStageBytes = (kStageR2 ? 2 : 1) * kRowBytes;  // u rows, then the matching r2 rows
  const cplx* u;
  const cplx* r2;
  cplx* T;
  int nx, ny, nz, np, ex, tpp, nplanes, nin;
  bool r2_staged;  // TMA path: r2 arrives with the tile (no per-thread loads)
  struct Ops {
    cplx r2v[kStreamPre];
    cplx* dst;  // T at (r, mx = 0, plane, iy0)
    int rows;
  };
  __device__ int ntiles() const { return nplanes * tpp; }
  template <int N>
  __device__ void load(int tile, cplx* buf) const {
    constexpr int RT = Geo<N>::ntr;
    const int pr = tile / tpp, iy0 = (tile - pr * tpp) * RT;
    const cplx* src = u + (static_cast<size_t>(pr) * ny + iy0) * nx;
    const int rows = min(RT, ny - iy0);
#pragma unroll
    for (int e = 0; e < Half<N>::per; ++e) {
      int t, j;
      Half<N>::rc(e, t, j);
      if (t < rows && j < nx) cp_async16(buf + Geo<N>::at(t, j), src + t * nx + j);
    }
  }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    constexpr int RT = Geo<N>::ntr, M = N / 16;
    const int pr = tile / tpp, iy0 = (tile - pr * tpp) * RT;
    const int r = pr / np, plane = pr - r * np;
    o.rows = min(RT, ny - iy0);
    o.dst = T + ((static_cast<size_t>(r) * ex) * np + plane) * ny + iy0;
    if (!r2 || r2_staged) return;
    const int iz = plane % nz;
    const int t = threadIdx.x / M, j = threadIdx.x % M;
    const int iy = min(iy0 + t, ny - 1);
    const cplx* row = r2 + (static_cast<size_t>(iz) * ny + iy) * nx;
#pragma unroll
    for (int q = 0; q < kStreamPre; ++q) {
      const int jj = j + q * M;
      o.r2v[q] = jj < nx ? ldg(row + jj) : cplx{0.0, 0.0};
    }
  }
  __device__ cplx pre(const Ops& o, int, int r, int, cplx x) const {
    return (r2 && !r2_staged && r < kStreamPre) ? o.r2v[r] * x : x;
  }
  // TMA staging: the tile's rows are one contiguous run of u, the matching
  // rows of r2 (cells of plane iz) another
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    constexpr int RT = Geo<N>::ntr;
    const int pr = tile / tpp, iy0 = (tile - pr * tpp) * RT;
    const uint32_t bytes = static_cast<uint32_t>(min(RT, ny - iy0) * nx) * sizeof(cplx);
    mbar_expect_tx(bar, r2 && r2_staged ? 2 * bytes : bytes);
    bulk_g2s(stg, u + (static_cast<size_t>(pr) * ny + iy0) * nx, bytes, bar);
    if (r2 && r2_staged) {
      const int iz = (pr % np) % nz;
      bulk_g2s(stg + kRowBytes / sizeof(cplx), r2 + (static_cast<size_t>(iz) * ny + iy0) * nx, bytes, bar);
    }
  }
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const {
    const cplx x = stg[t * nx + jj];
    return r2 && r2_staged ? stg[kRowBytes / sizeof(cplx) + t * nx + jj] * x : x;
  }
  // T[r][mx][plane][iy]: lanes t (= iy) fastest, 128 B runs per mx
  template <int N>
  __device__ void emit(const Ops& o, int t, int mx, int, int, cplx v) const {
    if (t < o.rows) gst(o.dst + static_cast<size_t>(mx) * np * ny + t, v);
  }
};

// y forward: tile = PC planes p0.. at column mx of rhs r; mirror signs on store
struct FyStream {
  static constexpr bool kInverse = false, kTFast = true;
  static constexpr int kStageBytes = 8 * 128 * 16;  // 8 planes of <= 128 points (N = 256) or 4 of <= 256
  const cplx* T;
  cplx* S;
  int ny, ex, ey, nz, np, gpc, nrhs, nin;
  struct Ops {
    cplx* dst;  // S at (r, mx, my = 0, p0)
    int p0;
    bool mxflip;
  };
  __device__ int ntiles() const { return nrhs * ex * gpc; }
  template <int N>
  __device__ void coords(int tile, int& r, int& mx, int& p0) const {
    const int g = tile % gpc, rm = tile / gpc;
    mx = rm % ex;
    r = rm / ex;
    p0 = g * Geo<N>::ntr;
  }
  template <int N>
  __device__ void load(int tile, cplx* buf) const {
    int r, mx, p0;
    coords<N>(tile, r, mx, p0);
    const int pc = min(Geo<N>::ntr, np - p0);
    const cplx* src = T + ((static_cast<size_t>(r) * ex + mx) * np + p0) * ny;
#pragma unroll
    for (int e = 0; e < Half<N>::per; ++e) {
      int t, j;
      Half<N>::rc(e, t, j);
      if (t < pc && j < ny) cp_async16(buf + Geo<N>::at(t, j), src + t * ny + j);
    }
  }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    int r, mx;
    coords<N>(tile, r, mx, o.p0);
    o.dst = S + (static_cast<size_t>(r) * ex + mx) * N * np + o.p0;
    o.mxflip = 2 * mx > ex;
  }
  __device__ cplx pre(const Ops&, int, int, int, cplx x) const { return x; }
  // TMA staging: the tile's planes are one contiguous run of T
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    int r, mx, p0;
    coords<N>(tile, r, mx, p0);
    const uint32_t bytes = static_cast<uint32_t>(min(Geo<N>::ntr, np - p0) * ny) * sizeof(cplx);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(stg, T + ((static_cast<size_t>(r) * ex + mx) * np + p0) * ny, bytes, bar);
  }
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const { return stg[t * ny + jj]; }
  // S[r][mx][my][plane] with the mirror signs: lanes t (= plane) fastest
  template <int N>
  __device__ void emit(const Ops& o, int t, int my, int, int, cplx v) const {
    const int plane = o.p0 + t;
    if (plane >= np) return;
    const bool flip = (plane < nz && o.mxflip) || (plane >= nz && plane < 2 * nz && 2 * my > N);
    gst(o.dst + static_cast<size_t>(my) * np + t, flip ? -v : v);
  }
};

// y forward of a depth slab in the sharded apply, fused with the forward
// transpose: the spectrum column of mode m is stored straight into the
// full-depth spectrum of m's owner rank (peer memory over NVLink) at depth
// offset zoff, S_g[r][m][c*nzf + zoff + z], instead of the slab's own S
constexpr int kMaxFyPeers = 64;
// The owner of mode (mx, my) comes from the plan -- no global-memory load on
// the store path (a per-mode owner table in HBM cost the pass 2x: 113 vs 58 us
// for one rank at config 3) -- or, for any other plan, from that table:
//   octant plans: the rank whose rows [split_g, split_g+1) hold max(qmx, qmy),
//     one byte of a row -> rank table in the kernel parameters;
//   quadrant plans: the rank whose range holds qm = qmy qx + qmx (split scan),
// with (qmx, qmy) the quadrant mode of (mx, my) (folds mx -> ex - mx past ex/2).
constexpr int kMaxFyRows = 260;  // quadrant rows of a 512-point embedding (257), padded
struct FyPeerStream : FyStream {
  cplx* pdst[kMaxFyPeers];     // owner rank -> its full-depth spectrum
  const int* owner;            // mode (mx*ey + my) -> owner rank, or nullptr: the splits
  int split[kMaxFyPeers + 1];  // split[g] .. split[g+1]: rank g's rows (oct) or quadrant modes
  int G, oct, qx;
  unsigned char row_owner[kMaxFyRows];  // oct: quadrant row -> owner rank
  int nzf, zoff;               // full depth, this slab's first interval
  // the last pass gives each thread one plane of the tile (t = tid mod 8,
  // transform index fastest), so its depth offset and sign class are per tile
  struct Ops {
    long long rE;  // r * ex * ey
    int mx, poff;  // poff: c * nzf + zoff + z of the thread's plane, -1 past the slab
    int qmx;       // quadrant column of mx
    bool xflip, ycls;
  };
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    int r, p0;
    coords<N>(tile, r, o.mx, p0);
    o.qmx = 2 * o.mx > ex ? ex - o.mx : o.mx;
    o.rE = static_cast<long long>(r) * ex * N;
    const int plane = p0 + static_cast<int>(threadIdx.x) % Geo<N>::ntr;
    const int c = plane / nz, z = plane - c * nz;
    o.poff = plane < np ? c * nzf + zoff + z : -1;
    o.xflip = c == 0 && 2 * o.mx > ex;
    o.ycls = c == 1;
  }
  __device__ cplx pre(const Ops&, int, int, int, cplx x) const { return x; }
  template <int N>
  __device__ void emit(const Ops& o, int, int my, int, int, cplx v) const {
    if (o.poff < 0) return;
    const bool flip = o.xflip || (o.ycls && 2 * my > N);
    const int m = o.mx * N + my;
    int g = 0;
    if (owner) {
      g = __ldg(owner + m);
    } else if (oct) {  // one indexed constant-bank byte
      g = row_owner[max(o.qmx, 2 * my > N ? N - my : my)];
    } else {
      const int qmy = 2 * my > N ? N - my : my;
      const int key = qmy * qx + o.qmx;
      for (int i = 1; i < G; ++i) g += key >= split[i] ? 1 : 0;
    }
    // indexed constant-bank load (measured: a 7-deep register select chain
    // over the destinations is slower, 103 vs 58 us for one rank at config 3)
    gst(pdst[g] + (o.rE + m) * 3 * nzf + o.poff, flip ? -v : v);
  }
};

// byte offset of 16-byte chunk t of staged row jj: N = 256 rows of 128 B with
// the 128-byte swizzle (chunk ^ row mod 8), N = 512 rows of 64 B with the
// 64-byte swizzle (chunk ^ (row / 2) mod 4)
template <int N>
__device__ __forceinline__ int stage_off(int t, int jj) {
  if constexpr (N == 256) return jj * 128 + ((t ^ (jj & 7)) << 4);
  else return jj * 64 + ((t ^ ((jj >> 1) & 3)) << 4);
}

// y inverse: tile = PC planes p0.. at column mx; mirror signs undone on load
struct IyStream {
  static constexpr bool kInverse = true, kTFast = false;
  // N = 256: [my][8 planes] (128-byte rows, 128-byte swizzle); N = 512:
  // [my][4 planes] (64-byte rows, 64-byte swizzle), two boxes of 256 my
  static constexpr int kStageBytes = 256 * 128;
  CUtensorMap tm;  // S as {2 np doubles, ey, nrhs ex}, box {16, 256, 1} (N = 512: {8, 256, 1})
  const cplx* S;
  cplx* T;
  int ny, ex, ey, nz, np, gpc, nrhs, nin;
  struct Ops {
    cplx* dst;  // T at (r, mx, p0, iy = 0)
    int p0;
    bool fx, yp;  // sign flags of the thread's first-pass transform
  };
  __device__ int ntiles() const { return nrhs * ex * gpc; }
  template <int N>
  __device__ void coords(int tile, int& r, int& mx, int& p0) const {
    const int g = tile % gpc, rm = tile / gpc;
    mx = rm % ex;
    r = rm / ex;
    p0 = g * Geo<N>::ntr;
  }
  template <int N>
  __device__ void load(int tile, cplx* buf) const {
    constexpr int PC = Geo<N>::ntr;
    int r, mx, p0;
    coords<N>(tile, r, mx, p0);
    const int p = threadIdx.x % PC;  // same for every e (PC divides 128)
    if (p0 + p >= np) return;
    const cplx* src = S + (static_cast<size_t>(r) * ex + mx) * N * np + p0 + p;
#pragma unroll
    for (int e = 0; e < PC * N / kStreamThreads; ++e) {
      const int j = (threadIdx.x + e * kStreamThreads) / PC;
      cp_async16(buf + Geo<N>::at(p, j), src + j * np);
    }
  }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    int r, mx;
    coords<N>(tile, r, mx, o.p0);
    o.dst = T + ((static_cast<size_t>(r) * ex + mx) * np + o.p0) * ny;
    const int plane = o.p0 + threadIdx.x / (N / 16);  // first-pass transform of the thread
    o.fx = plane < nz && 2 * mx > ex;
    o.yp = plane >= nz && plane < 2 * nz;
  }
  __device__ cplx pre(const Ops& o, int, int, int jj, cplx x) const {
    return (o.fx || (o.yp && 2 * jj > ey)) ? -x : x;
  }
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    int r, mx, p0;
    coords<N>(tile, r, mx, p0);
    mbar_expect_tx(bar, kStageBytes);
#pragma unroll
    for (int h = 0; h < N / 256; ++h)
      tma_load_3d(reinterpret_cast<unsigned char*>(stg) + h * (kStageBytes * 256 / N), &tm, 2 * p0, 256 * h,
                  r * ex + mx, bar);
  }
  // element jj (my) of transform t (plane): 16-byte chunk t of row jj, swizzled
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const {
    return *reinterpret_cast<const cplx*>(reinterpret_cast<const unsigned char*>(stg) + stage_off<N>(t, jj));
  }
  // T[r][mx][plane][iy], iy < ny: lanes j (= iy) fastest
  template <int N>
  __device__ void emit(const Ops& o, int t, int iy, int, int, cplx v) const {
    if (iy < ny && o.p0 + t < np) gst(o.dst + t * ny + iy, v);
  }
};

// x inverse: tile = RT rows iy0.. of plane pr; truncation, 1/(ex ey) and the
// system epilogue s*u + r1*(.) (cie.cpp:67-72), its operands prefetched for
// the thread's kept outputs (slot b*R/2 + r, r < R/2: ix < N/2)
struct IxStream {
  static constexpr bool kInverse = true, kTFast = false;
  // N = 256: [mx][8 rows], 128-byte swizzle; N = 512: [mx][4 rows], 64-byte swizzle, two boxes
  static constexpr int kStageBytes = 256 * 128;
  CUtensorMap tm;  // T as {2 ny doubles, np, ex, nrhs}, box {16, 1, 256, 1} (N = 512: {8, 1, 256, 1})
  const cplx* T;
  const cplx* u;
  cplx* out;
  const cplx* s;
  const double* r1;
  int nx, ny, nz, np, ex, tpp, nplanes, nin;
  double inv;
  struct Ops {
    cplx uv[kStreamPre], sv[kStreamPre];
    double rv[kStreamPre];
    int pr, iy0;
  };
  __device__ int ntiles() const { return nplanes * tpp; }
  template <int N>
  __device__ void load(int tile, cplx* buf) const {
    constexpr int RT = Geo<N>::ntr;
    const int pr = tile / tpp, iy0 = (tile - pr * tpp) * RT;
    const int r = pr / np, plane = pr - r * np;
    const int rows = min(RT, ny - iy0);
    const cplx* src = T + ((static_cast<size_t>(r) * ex) * np + plane) * ny + iy0;
    const size_t mstride = static_cast<size_t>(np) * ny;
    const int tt = threadIdx.x % RT;  // same for every e (RT divides 128)
    if (tt >= rows) return;
#pragma unroll
    for (int e = 0; e < RT * N / kStreamThreads; ++e) {
      const int mx = (threadIdx.x + e * kStreamThreads) / RT;
      cp_async16(buf + Geo<N>::at(tt, mx), src + mx * mstride + tt);
    }
  }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    constexpr int RT = Geo<N>::ntr, R = last_radix<N>(), NS = N / R, B = kFftEPT / R;
    o.pr = tile / tpp;
    o.iy0 = (tile - o.pr * tpp) * RT;
    if (!s) return;
    const int iz = (o.pr % np) % nz;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      int t, j;
      last_coord<N, false>(b, t, j);
#pragma unroll
      for (int r = 0; r < R / 2; ++r) {
        const int q = b * (R / 2) + r, ix = j + r * NS, iy = o.iy0 + t;
        if (iy < ny && ix < nx) {
          const size_t cell = (static_cast<size_t>(iz) * ny + iy) * nx + ix;
          o.uv[q] = ldg(u + (static_cast<size_t>(o.pr) * ny + iy) * nx + ix);
          o.sv[q] = ldg(s + cell);
          o.rv[q] = __ldg(r1 + cell);
        }
      }
    }
  }
  __device__ cplx pre(const Ops&, int, int, int, cplx x) const { return x; }
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    constexpr int RT = Geo<N>::ntr;
    const int pr = tile / tpp, iy0 = (tile - pr * tpp) * RT;
    const int r = pr / np, plane = pr - r * np;
    mbar_expect_tx(bar, kStageBytes);
#pragma unroll
    for (int h = 0; h < N / 256; ++h)
      tma_load_4d(reinterpret_cast<unsigned char*>(stg) + h * (kStageBytes * 256 / N), &tm, 2 * iy0, plane, 256 * h,
                  r, bar);
  }
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const {
    return *reinterpret_cast<const cplx*>(reinterpret_cast<const unsigned char*>(stg) + stage_off<N>(t, jj));
  }
  // out[pr][iy][ix], ix < nx: lanes j (= ix) fastest
  template <int N>
  __device__ void emit(const Ops& o, int t, int ix, int b, int r, cplx v) const {
    constexpr int R = last_radix<N>();
    const int iy = o.iy0 + t;
    if (r >= R / 2 || ix >= nx || iy >= ny) return;
    const size_t q = (static_cast<size_t>(o.pr) * ny + iy) * nx + ix;
    v = inv * v;
    if (s) {
      const int k = b * (R / 2) + r;
      v = o.sv[k] * o.uv[k] + o.rv[k] * v;
    }
    gst(out + q, v);
  }
};

void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

// tile shape: elements per CTA and threads for the engine
constexpr int kTileElems = 2048;  // pow2 engine: kFftThreads * kFftEPT
constexpr int kFftThreads = kTileElems / kFftEPT;


// ---- spectra build on the TMA streaming engine (K7, toeplitz.cpp:92-161) ----
// The parity-extended offset sequences of the compressed blocks: a tile is TR
// consecutive entries e (the transforms) of one row of offsets; their nonzero
// inputs (offsets 0..n-1) arrive as one tensor-map box [offset][TR entries]
// (128-byte rows, N = 256; 64-byte rows, N = 512), the mirrored half
// (j > N - n: the entry at offset N - j, times the component's parity sign,
// toeplitz.cpp:140-151) is read from the same staged rows, the zero middle
// is never loaded. x pass: R[(oi qx + mx) nent + e] for mx < qx; y pass: the
// quadrant modes my < qy of the operator's shard, through emap into the
// device mode blocks (operator.cuh).
template <int N>
__device__ __forceinline__ cplx staged_parity(const cplx* stg, int t, int jj, int n) {
  const int row = jj < n ? jj : (jj > N - n ? N - jj : -1);
  if (row < 0) return cplx{0.0, 0.0};
  return *reinterpret_cast<const cplx*>(reinterpret_cast<const unsigned char*>(stg) + stage_off<N>(t, row));
}

struct SpxStream {
  static constexpr bool kInverse = false, kTFast = true;
  static constexpr int kStageBytes = 16384;  // <= N/2 offsets of 128-byte (64-byte) rows
  CUtensorMap tm;  // blocks as {2 nent doubles, nx, ny}, box {16 | 8, nx, 1}
  cplx* R;
  int nx, ny, qx, nent, ntri, nfull, nchunks, nin;
  uint32_t box_bytes;
  struct Ops {
    int oi, e0;
    double sgn;  // parity of the thread's first-pass transform (entry)
  };
  __device__ int ntiles() const { return ny * nchunks; }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    o.oi = tile / nchunks;
    o.e0 = (tile - o.oi * nchunks) * Geo<N>::ntr;
    const int e = o.e0 + static_cast<int>(threadIdx.x) / (N / 16);
    o.sgn = e < nent ? static_cast<double>(kParX[comp_of(e, ntri, nfull)]) : 1.0;
  }
  __device__ cplx pre(const Ops& o, int, int, int jj, cplx x) const { return jj >= nx ? o.sgn * x : x; }
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    const int oi = tile / nchunks, e0 = (tile - oi * nchunks) * Geo<N>::ntr;
    mbar_expect_tx(bar, box_bytes);
    tma_load_3d(stg, &tm, 2 * e0, 0, oi, bar);
  }
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const { return staged_parity<N>(stg, t, jj, nx); }
  template <int N>
  __device__ void emit(const Ops& o, int t, int mx, int, int, cplx v) const {
    const int e = o.e0 + t;
    if (mx < qx && e < nent) gst(R + (static_cast<size_t>(o.oi) * qx + mx) * nent + e, v);
  }
};

struct SpyStream {
  static constexpr bool kInverse = false, kTFast = true;
  static constexpr int kStageBytes = 16384;
  CUtensorMap tm;  // R as {2 nent doubles, qx, ny}, box {16 | 8, 1, ny}
  cplx* spec;
  const int2* emap;
  int ny, qx, qy, nent, ntri, nfull, nchunks, nentD, qbase, qcount, nin;
  int mirror;  // store the second slot of a symmetric entry here (else mirror_fill_kernel does, coalesced)
  uint32_t box_bytes;
  struct Ops {
    int mx, e0;
    double sgn;
  };
  __device__ int ntiles() const { return qx * nchunks; }
  template <int N>
  __device__ void prefetch(int tile, Ops& o) const {
    o.mx = tile / nchunks;
    o.e0 = (tile - o.mx * nchunks) * Geo<N>::ntr;
    const int e = o.e0 + static_cast<int>(threadIdx.x) / (N / 16);
    o.sgn = e < nent ? static_cast<double>(kParY[comp_of(e, ntri, nfull)]) : 1.0;
  }
  __device__ cplx pre(const Ops& o, int, int, int jj, cplx x) const { return jj >= ny ? o.sgn * x : x; }
  template <int N>
  __device__ void issue(int tile, cplx* stg, uint64_t* bar) const {
    const int mx = tile / nchunks, e0 = (tile - mx * nchunks) * Geo<N>::ntr;
    mbar_expect_tx(bar, box_bytes);
    tma_load_3d(stg, &tm, 2 * e0, mx, 0, bar);
  }
  template <int N>
  __device__ cplx staged(const cplx* stg, int t, int jj) const { return staged_parity<N>(stg, t, jj, ny); }
  template <int N>
  __device__ void emit(const Ops& o, int t, int my, int, int, cplx v) const {
    const int e = o.e0 + t;
    const int qm = my * qx + o.mx;
    if (my < qy && e < nent && qm >= qbase && qm < qbase + qcount) {
      const int2 m = __ldg(emap + e);
      cplx* blk = spec + static_cast<size_t>(qm - qbase) * nentD;
      gst(blk + m.x, v);
      if (mirror && m.y >= 0) gst(blk + m.y, v);
    }
  }
};

// Row-block layout (nz 48 / 64): the lower triangles of the symmetric dense
// blocks (xx yy zz xy) of every stored mode, from their upper triangles --
// one (mode, component) block per CTA through SMEM, so the y pass writes
// only the upper triangles row by row and the transposed copies leave here
// in whole rows instead of one 16-byte store per entry a row apart (the
// scattered stores cost config 4's y pass 38 ms for 26 GB)
__global__ void __launch_bounds__(256) mirror_fill_kernel(cplx* spec, int nz, int nentD) {
  extern __shared__ cplx tile[];  // nz x (nz + 1)
  cplx* blk = spec + static_cast<size_t>(blockIdx.x >> 2) * nentD + static_cast<size_t>(blockIdx.x & 3) * nz * nz;
  const int n2 = nz * nz, ld = nz + 1;
  // all of a thread's upper-triangle loads in flight at once (nz <= 64: 16 per thread)
  constexpr int kPer = 16;
  cplx v[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int i = threadIdx.x + q * 256;
    const int k = i / nz, kp = i - k * nz;
    if (i < n2 && kp > k) v[q] = blk[i];
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int i = threadIdx.x + q * 256;
    const int k = i / nz, kp = i - k * nz;
    if (i < n2 && kp > k) tile[k * ld + kp] = v[q];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    const int r = i / nz, c = i - r * nz;  // lower entry (r, c), c < r, = upper (c, r)
    if (c < r) blk[i] = tile[c * ld + r];
  }
}

int per_tile(int n) { return std::max(1, kTileElems / std::max(1, n)); }

// the streaming path takes power-of-two n in [16, 2048] whose nonzero input
// run is at most half the transform (always true of a circulant embedding)
bool stream_ok(bool p2, int n, int nin) { return p2 && n >= 32 && n <= kStreamElems && 2 * nin <= n; }

template <int N, class P>
void launch_stream_n(const P& p, int ntiles, const cplx* tw, cudaStream_t st) {
  const size_t smem = (kStreamBufs * static_cast<size_t>(Geo<N>::tile) + N) * sizeof(cplx);
  const int per_sm = resident_ctas(reinterpret_cast<const void*>(stream_fft_kernel<N, P>), kStreamThreads, smem);
  const int grid = std::max(1, std::min(ntiles, sm_count() * per_sm));
  stream_fft_kernel<N, P><<<grid, kStreamThreads, smem, st>>>(p, tw);
}

#ifndef EMIE_TMA_NST_INV
#define EMIE_TMA_NST_INV 1  // staging buffers of the inverse passes (1: three CTAs per SM)
#endif
#ifndef EMIE_TMA_NST_FWD
#define EMIE_TMA_NST_FWD 1
#endif
#ifndef EMIE_TMA_NST_FX
#define EMIE_TMA_NST_FX EMIE_TMA_NST_FWD
#endif
#ifndef EMIE_TMA_NST_FY
#define EMIE_TMA_NST_FY EMIE_TMA_NST_FWD
#endif
template <int N, class P, int NST>
void launch_tma(const P& p, int ntiles, const cplx* tw, cudaStream_t st, const char* what) {
  const size_t smem = NST * static_cast<size_t>(P::kStageBytes) +
                      (static_cast<size_t>(Geo<N>::tile) + N) * sizeof(cplx) + NST * sizeof(uint64_t);
  const int per_sm =
      resident_ctas(reinterpret_cast<const void*>(stream_tma_kernel<N, P, NST>), kStreamThreads, smem);
  const int grid = std::max(1, std::min(ntiles, sm_count() * per_sm));
  launch_pdl(stream_tma_kernel<N, P, NST>, grid, kStreamThreads, smem, st, p, tw);
  check_launch(what);
}

template <class P>
void launch_stream(const P& p, int ntiles, const cplx* tw, int n, cudaStream_t st, const char* what) {
  switch (n) {
    case 32: launch_stream_n<32>(p, ntiles, tw, st); break;
    case 64: launch_stream_n<64>(p, ntiles, tw, st); break;
    case 128: launch_stream_n<128>(p, ntiles, tw, st); break;
    case 256: launch_stream_n<256>(p, ntiles, tw, st); break;
    case 512: launch_stream_n<512>(p, ntiles, tw, st); break;
    case 1024: launch_stream_n<1024>(p, ntiles, tw, st); break;
    case 2048: launch_stream_n<2048>(p, ntiles, tw, st); break;
    default: fail(EMIE_CU_RUNTIME_ERROR, "stream FFT: unsupported length");
  }
  check_launch(what);
}

}  // namespace

// ------------------------------------------------------------------ host --
void encode_tensor_map_f64(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims,
                           const uint64_t* strides_bytes, const uint32_t* box, int swizzle) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    EMIE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) fail(EMIE_CU_RUNTIME_ERROR, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  cuuint64_t d[5], sb[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) sb[i] = strides_bytes[i];
  }
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), d, sb, b, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            swizzle == 0    ? CU_TENSOR_MAP_SWIZZLE_NONE
                            : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(EMIE_CU_RUNTIME_ERROR, "cuTensorMapEncodeTiled failed");
}

void lateral_spectra(const Operator& op, const cplx* d_blocks, cudaStream_t st) {
  const int nent = op.nent;
  cplx* R = scratch<cplx>(static_cast<size_t>(op.ny) * op.qx * nent, st);
  static const bool no_tma = [] {
    const char* e = std::getenv("EMIE_CU_SPECTRA_NO_TMA");  // A/B switch: the per-CTA load/FFT/store kernels
    return e && *e == '1';
  }();
  const bool tma_x = !no_tma && (op.ex == 256 || op.ex == 512), tma_y = !no_tma && (op.ey == 256 || op.ey == 512);
  if (tma_x) {
    SpxStream p{};
    const bool w = op.ex == 512;
    const int TR = w ? 4 : 8;
    p.R = R;
    p.nx = op.nx; p.ny = op.ny; p.qx = op.qx; p.nent = nent; p.ntri = op.ntri; p.nfull = op.nfull;
    p.nchunks = ceil_div(nent, TR); p.nin = op.ex;
    p.box_bytes = static_cast<uint32_t>(2 * TR * op.nx * sizeof(double));
    const uint64_t dims[3] = {2ull * nent, static_cast<uint64_t>(op.nx), static_cast<uint64_t>(op.ny)};
    const uint64_t strides[2] = {static_cast<uint64_t>(nent) * 16, static_cast<uint64_t>(op.nx) * nent * 16};
    const uint32_t box[3] = {static_cast<uint32_t>(2 * TR), static_cast<uint32_t>(op.nx), 1};
    encode_tensor_map_f64(&p.tm, d_blocks, 3, dims, strides, box, w ? 64 : 128);
    if (w) launch_tma<512, SpxStream, 1>(p, op.ny * p.nchunks, op.tw_x, st, "stream_tma_spectra_x");
    else launch_tma<256, SpxStream, 1>(p, op.ny * p.nchunks, op.tw_x, st, "stream_tma_spectra_x");
  } else {
    const bool p2 = op.p2x;
    const FftPlan& pl = p2 ? op.plan_x2 : op.plan_x;
    const int EC = std::min(16, per_tile(op.ex));
    const size_t smem = tile_bytes(p2, EC, op.ex);
    dim3 grid(op.ny, ceil_div(nent, EC));
    if (p2) {
      set_smem(reinterpret_cast<const void*>(spectra_x_kernel<true>), smem);
      spectra_x_kernel<true><<<grid, kFftThreads, smem, st>>>(d_blocks, R, op.tw_x, pl, op.nx, op.qx,
                                                              nent, op.ntri, op.nfull, EC);
    } else {
      set_smem(reinterpret_cast<const void*>(spectra_x_kernel<false>), smem);
      spectra_x_kernel<false><<<grid, 256, smem, st>>>(d_blocks, R, op.tw_x, pl, op.nx, op.qx, nent,
                                                       op.ntri, op.nfull, EC);
    }
    check_launch("spectra_x_kernel");
  }
  if (tma_y) {
    SpyStream p{};
    const bool w = op.ey == 512;
    const int TR = w ? 4 : 8;
    p.spec = op.spec; p.emap = op.emap;
    p.ny = op.ny; p.qx = op.qx; p.qy = op.qy; p.nent = nent; p.ntri = op.ntri; p.nfull = op.nfull;
    p.nchunks = ceil_div(nent, TR); p.nentD = op.nentD; p.qbase = op.qbase; p.qcount = op.qcount; p.nin = op.ey;
    p.mirror = op.rows ? 0 : 1;
    p.box_bytes = static_cast<uint32_t>(2 * TR * op.ny * sizeof(double));
    const uint64_t dims[3] = {2ull * nent, static_cast<uint64_t>(op.qx), static_cast<uint64_t>(op.ny)};
    const uint64_t strides[2] = {static_cast<uint64_t>(nent) * 16, static_cast<uint64_t>(op.qx) * nent * 16};
    const uint32_t box[3] = {static_cast<uint32_t>(2 * TR), 1, static_cast<uint32_t>(op.ny)};
    encode_tensor_map_f64(&p.tm, R, 3, dims, strides, box, w ? 64 : 128);
    if (w) launch_tma<512, SpyStream, 1>(p, op.qx * p.nchunks, op.tw_y, st, "stream_tma_spectra_y");
    else launch_tma<256, SpyStream, 1>(p, op.qx * p.nchunks, op.tw_y, st, "stream_tma_spectra_y");
    if (op.rows && op.qcount > 0) {
      const size_t smem = static_cast<size_t>(op.nz) * (op.nz + 1) * sizeof(cplx);
      set_smem(reinterpret_cast<const void*>(mirror_fill_kernel), smem);
      mirror_fill_kernel<<<op.qcount * 4, 256, smem, st>>>(op.spec, op.nz, op.nentD);
      check_launch("mirror_fill_kernel");
    }
  } else {
    const bool p2 = op.p2y;
    const FftPlan& pl = p2 ? op.plan_y2 : op.plan_y;
    const int EC = std::min(16, per_tile(op.ey));
    const size_t smem = tile_bytes(p2, EC, op.ey);
    dim3 grid(op.qx, ceil_div(nent, EC));
    if (p2) {
      set_smem(reinterpret_cast<const void*>(spectra_y_kernel<true>), smem);
      spectra_y_kernel<true><<<grid, kFftThreads, smem, st>>>(R, op.spec, op.tw_y, pl, op.ny, op.qx, op.qy,
                                                              nent, op.ntri, op.nfull, EC, op.emap,
                                                              op.nentD, op.qbase, op.qcount);
    } else {
      set_smem(reinterpret_cast<const void*>(spectra_y_kernel<false>), smem);
      spectra_y_kernel<false><<<grid, 256, smem, st>>>(R, op.spec, op.tw_y, pl, op.ny, op.qx, op.qy,
                                                       nent, op.ntri, op.nfull, EC, op.emap,
                                                       op.nentD, op.qbase, op.qcount);
    }
    check_launch("spectra_y_kernel");
  }
  release(R, st);
}

void lateral_forward(const Operator& op, const cplx* d_in, const cplx* r2, cplx* T, cplx* S,
                     int nrhs, cudaStream_t st) {
  const int np = 3 * op.nz;
  profile_mark(0, true, st);
  if (stream_ok(op.p2x, op.ex, op.nx)) {
    FxStream p{};
    p.u = d_in; p.r2 = r2; p.T = T;
    p.nx = op.nx; p.ny = op.ny; p.nz = op.nz; p.np = np; p.ex = op.ex;
    p.tpp = ceil_div(op.ny, kStreamElems / op.ex); p.nplanes = nrhs * np; p.nin = op.nx;
    p.r2_staged = FxStream::kStageR2 && (op.ex == 256 || op.ex == 512);
    if (op.ex == 256) launch_tma<256, FxStream, EMIE_TMA_NST_FX>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_fx");
    else if (op.ex == 512) launch_tma<512, FxStream, EMIE_TMA_NST_FX>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_fx");
    else launch_stream(p, p.nplanes * p.tpp, op.tw_x, op.ex, st, "stream_fx");
  } else {
    const bool p2 = op.p2x;
    const FftPlan& pl = p2 ? op.plan_x2 : op.plan_x;
    const int RT = std::min(per_tile(op.ex), op.ny);
    const size_t smem = tile_bytes(p2, RT, op.ex);
    dim3 grid(nrhs * np, ceil_div(op.ny, RT));
    if (p2) {
      set_smem(reinterpret_cast<const void*>(apply_fx_kernel<true>), smem);
      apply_fx_kernel<true><<<grid, kFftThreads, smem, st>>>(d_in, r2, T, op.tw_x, pl, op.nx, op.ny, op.nz, RT);
    } else {
      set_smem(reinterpret_cast<const void*>(apply_fx_kernel<false>), smem);
      apply_fx_kernel<false><<<grid, 256, smem, st>>>(d_in, r2, T, op.tw_x, pl, op.nx, op.ny, op.nz, RT);
    }
    check_launch("apply_fx_kernel");
  }
  profile_mark(0, false, st);
  profile_mark(1, true, st);
  if (stream_ok(op.p2y, op.ey, op.ny)) {
    FyStream p{};
    p.T = T; p.S = S;
    p.ny = op.ny; p.ex = op.ex; p.ey = op.ey; p.nz = op.nz; p.np = np;
    p.gpc = ceil_div(np, kStreamElems / op.ey); p.nrhs = nrhs; p.nin = op.ny;
    if (op.ey == 256) launch_tma<256, FyStream, EMIE_TMA_NST_FY>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_fy");
    else if (op.ey == 512) launch_tma<512, FyStream, EMIE_TMA_NST_FY>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_fy");
    else launch_stream(p, nrhs * op.ex * p.gpc, op.tw_y, op.ey, st, "stream_fy");
  } else {
    const bool p2 = op.p2y;
    const FftPlan& pl = p2 ? op.plan_y2 : op.plan_y;
    const int PC = std::min(np, per_tile(op.ey));
    const size_t smem = tile_bytes(p2, PC, op.ey);
    dim3 grid(op.ex, ceil_div(np, PC), nrhs);
    if (p2) {
      set_smem(reinterpret_cast<const void*>(apply_fy_kernel<true>), smem);
      apply_fy_kernel<true><<<grid, kFftThreads, smem, st>>>(T, S, op.tw_y, pl, op.ny, op.ex, op.nz, PC);
    } else {
      set_smem(reinterpret_cast<const void*>(apply_fy_kernel<false>), smem);
      apply_fy_kernel<false><<<grid, 256, smem, st>>>(T, S, op.tw_y, pl, op.ny, op.ex, op.nz, PC);
    }
    check_launch("apply_fy_kernel");
  }
  profile_mark(1, false, st);
}

bool lateral_forward_peer_ok(const Operator& op) {
  return stream_ok(op.p2x, op.ex, op.nx) && stream_ok(op.p2y, op.ey, op.ny) && (op.ey == 256 || op.ey == 512) &&
         (op.ex == 256 || op.ex == 512);
}

void lateral_forward_peer(const Operator& op, const cplx* d_in, const cplx* r2, cplx* T, const int* owner,
                          const int* split, int oct, cplx* const* dsts, int G, int nzf, int zoff, int nrhs,
                          cudaStream_t st) {
  if (!lateral_forward_peer_ok(op)) fail(EMIE_CU_INVALID_ARGUMENT, "lateral_forward_peer: needs 256/512-point TMA passes");
  if (G < 1 || G > kMaxFyPeers) fail(EMIE_CU_INVALID_ARGUMENT, "lateral_forward_peer: bad rank count");
  const int np = 3 * op.nz;
  {  // x pass into the local T (TMA path, as lateral_forward)
    FxStream p{};
    p.u = d_in; p.r2 = r2; p.T = T;
    p.nx = op.nx; p.ny = op.ny; p.nz = op.nz; p.np = np; p.ex = op.ex;
    p.tpp = ceil_div(op.ny, kStreamElems / op.ex); p.nplanes = nrhs * np; p.nin = op.nx;
    p.r2_staged = FxStream::kStageR2;
    if (op.ex == 256) launch_tma<256, FxStream, EMIE_TMA_NST_FX>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_fx");
    else launch_tma<512, FxStream, EMIE_TMA_NST_FX>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_fx");
  }
  FyPeerStream p{};
  p.T = T; p.S = nullptr;
  p.ny = op.ny; p.ex = op.ex; p.ey = op.ey; p.nz = op.nz; p.np = np;
  p.gpc = ceil_div(np, kStreamElems / op.ey); p.nrhs = nrhs; p.nin = op.ny;
  for (int g = 0; g < G; ++g) p.pdst[g] = dsts[g];
  p.owner = owner; p.nzf = nzf; p.zoff = zoff;
  p.G = G; p.oct = oct; p.qx = op.qx;
  if (!owner) {
    for (int g = 0; g <= G; ++g) p.split[g] = split[g];
    if (oct) {
      if (op.qy > kMaxFyRows || G > 255) fail(EMIE_CU_INVALID_ARGUMENT, "lateral_forward_peer: embedding too large");
      for (int g = 0; g < G; ++g)
        for (int r = split[g]; r < split[g + 1]; ++r) p.row_owner[r] = static_cast<unsigned char>(g);
    }
  }
  if (op.ey == 256) launch_tma<256, FyPeerStream, EMIE_TMA_NST_FWD>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_fy_peer");
  else launch_tma<512, FyPeerStream, EMIE_TMA_NST_FWD>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_fy_peer");
}

void lateral_inverse(const Operator& op, const cplx* S, cplx* T, const cplx* d_in, cplx* d_out,
                     const cplx* s, const double* r1, int nrhs, cudaStream_t st) {
  const int np = 3 * op.nz;
  profile_mark(3, true, st);
  if (stream_ok(op.p2y, op.ey, op.ny)) {
    IyStream p{};
    p.S = S; p.T = T;
    p.ny = op.ny; p.ex = op.ex; p.ey = op.ey; p.nz = op.nz; p.np = np;
    p.gpc = ceil_div(np, kStreamElems / op.ey); p.nrhs = nrhs; p.nin = op.ey;
    if (op.ey == 256 || op.ey == 512) {
      const bool w = op.ey == 512;
      const uint64_t dims[3] = {2ull * np, static_cast<uint64_t>(op.ey), static_cast<uint64_t>(nrhs) * op.ex};
      const uint64_t strides[2] = {static_cast<uint64_t>(np) * 16, static_cast<uint64_t>(op.ey) * np * 16};
      const uint32_t box[3] = {w ? 8u : 16u, 256, 1};
      encode_tensor_map_f64(&p.tm, S, 3, dims, strides, box, w ? 64 : 128);
      if (w) launch_tma<512, IyStream, EMIE_TMA_NST_INV>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_iy");
      else launch_tma<256, IyStream, EMIE_TMA_NST_INV>(p, nrhs * op.ex * p.gpc, op.tw_y, st, "stream_tma_iy");
    } else {
      launch_stream(p, nrhs * op.ex * p.gpc, op.tw_y, op.ey, st, "stream_iy");
    }
  } else {
    const bool p2 = op.p2y;
    const FftPlan& pl = p2 ? op.plan_y2 : op.plan_y;
    const int PC = std::min(np, per_tile(op.ey));
    const size_t smem = tile_bytes(p2, PC, op.ey);
    dim3 grid(op.ex, ceil_div(np, PC), nrhs);
    if (p2) {
      set_smem(reinterpret_cast<const void*>(apply_iy_kernel<true>), smem);
      apply_iy_kernel<true><<<grid, kFftThreads, smem, st>>>(S, T, op.tw_y, pl, op.ny, op.ex, op.nz, PC);
    } else {
      set_smem(reinterpret_cast<const void*>(apply_iy_kernel<false>), smem);
      apply_iy_kernel<false><<<grid, 256, smem, st>>>(S, T, op.tw_y, pl, op.ny, op.ex, op.nz, PC);
    }
    check_launch("apply_iy_kernel");
  }
  profile_mark(3, false, st);
  profile_mark(4, true, st);
  if (stream_ok(op.p2x, op.ex, op.nx)) {
    IxStream p{};
    p.T = T; p.u = d_in; p.out = d_out; p.s = s; p.r1 = r1;
    p.nx = op.nx; p.ny = op.ny; p.nz = op.nz; p.np = np; p.ex = op.ex;
    p.tpp = ceil_div(op.ny, kStreamElems / op.ex); p.nplanes = nrhs * np; p.nin = op.ex;
    p.inv = 1.0 / static_cast<double>(op.lateral());
    if (op.ex == 256 || op.ex == 512) {
      const bool w = op.ex == 512;
      const uint64_t dims[4] = {2ull * op.ny, static_cast<uint64_t>(np), static_cast<uint64_t>(op.ex),
                                static_cast<uint64_t>(nrhs)};
      const uint64_t strides[3] = {static_cast<uint64_t>(op.ny) * 16, static_cast<uint64_t>(np) * op.ny * 16,
                                   static_cast<uint64_t>(op.ex) * np * op.ny * 16};
      const uint32_t box[4] = {w ? 8u : 16u, 1, 256, 1};
      encode_tensor_map_f64(&p.tm, T, 4, dims, strides, box, w ? 64 : 128);
      if (w) launch_tma<512, IxStream, EMIE_TMA_NST_INV>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_ix");
      else launch_tma<256, IxStream, EMIE_TMA_NST_INV>(p, p.nplanes * p.tpp, op.tw_x, st, "stream_tma_ix");
    } else {
      launch_stream(p, p.nplanes * p.tpp, op.tw_x, op.ex, st, "stream_ix");
    }
  } else {
    const bool p2 = op.p2x;
    const FftPlan& pl = p2 ? op.plan_x2 : op.plan_x;
    const int RT = std::min(per_tile(op.ex), op.ny);
    const size_t smem = tile_bytes(p2, RT, op.ex);
    const double inv = 1.0 / static_cast<double>(op.lateral());
    dim3 grid(nrhs * np, ceil_div(op.ny, RT));
    if (p2) {
      set_smem(reinterpret_cast<const void*>(apply_ix_kernel<true>), smem);
      apply_ix_kernel<true><<<grid, kFftThreads, smem, st>>>(T, d_in, d_out, s, r1, op.tw_x, pl, op.nx,
                                                             op.ny, op.nz, RT, inv);
    } else {
      set_smem(reinterpret_cast<const void*>(apply_ix_kernel<false>), smem);
      apply_ix_kernel<false><<<grid, 256, smem, st>>>(T, d_in, d_out, s, r1, op.tw_x, pl, op.nx, op.ny,
                                                      op.nz, RT, inv);
    }
    check_launch("apply_ix_kernel");
  }
  profile_mark(4, false, st);
}

}  // namespace emie_cu
