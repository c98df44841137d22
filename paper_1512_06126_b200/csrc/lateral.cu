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
#include <algorithm>

#include "operator.cuh"

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
                                 int nentD) {
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
    if (e < nent) {
      const int2 m = emap[e];
      cplx* blk = spec + (static_cast<size_t>(my) * qx + mx) * nentD;
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
  const int c = plane / nz;
  return ((c == 0 && mx > ex / 2) || (c == 1 && my > ey / 2)) ? -1.0 : 1.0;
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

void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

// tile shape: elements per CTA and threads for the engine
constexpr int kTileElems = 2048;  // pow2 engine: kFftThreads * kFftEPT
constexpr int kFftThreads = kTileElems / kFftEPT;

int per_tile(int n) { return std::max(1, kTileElems / std::max(1, n)); }

}  // namespace

// ------------------------------------------------------------------ host --
void lateral_spectra(const Operator& op, const cplx* d_blocks, cudaStream_t st) {
  const int nent = op.nent;
  cplx* R = scratch<cplx>(static_cast<size_t>(op.ny) * op.qx * nent, st);
  {
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
  {
    const bool p2 = op.p2y;
    const FftPlan& pl = p2 ? op.plan_y2 : op.plan_y;
    const int EC = std::min(16, per_tile(op.ey));
    const size_t smem = tile_bytes(p2, EC, op.ey);
    dim3 grid(op.qx, ceil_div(nent, EC));
    if (p2) {
      set_smem(reinterpret_cast<const void*>(spectra_y_kernel<true>), smem);
      spectra_y_kernel<true><<<grid, kFftThreads, smem, st>>>(R, op.spec, op.tw_y, pl, op.ny, op.qx, op.qy,
                                                              nent, op.ntri, op.nfull, EC, op.emap,
                                                              op.nentD);
    } else {
      set_smem(reinterpret_cast<const void*>(spectra_y_kernel<false>), smem);
      spectra_y_kernel<false><<<grid, 256, smem, st>>>(R, op.spec, op.tw_y, pl, op.ny, op.qx, op.qy,
                                                       nent, op.ntri, op.nfull, EC, op.emap,
                                                       op.nentD);
    }
    check_launch("spectra_y_kernel");
  }
  release(R, st);
}

void lateral_forward(const Operator& op, const cplx* d_in, const cplx* r2, cplx* T, cplx* S,
                     int nrhs, cudaStream_t st) {
  const int np = 3 * op.nz;
  profile_mark(0, true, st);
  {
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
  {
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

void lateral_inverse(const Operator& op, const cplx* S, cplx* T, const cplx* d_in, cplx* d_out,
                     const cplx* s, const double* r1, int nrhs, cudaStream_t st) {
  const int np = 3 * op.nz;
  profile_mark(3, true, st);
  {
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
  {
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
