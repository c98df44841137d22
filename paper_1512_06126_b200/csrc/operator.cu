// Spectral operator build (transform_operator) and the CIE operator apply
// (apply(SpectralOperator), apply(SystemOperator)) for sm_100a.
//
// Reference: src/toeplitz.cpp:92-161 (spectra), 163-283 (apply),
//            src/cie.cpp:56-73 (system apply).
//
// Apply data flow for nrhs fields (all complex128):
//   u [r][plane][iy][ix]            plane = c*nz + iz (GridVector layout)
//   K_fx : r2-scale, zero-pad, x-FFT        -> T [r][plane][iy][mx]
//   K_fy : zero-pad, y-FFT, transpose       -> S [r][my][mx][plane]  (mode-major)
//   K_ct : per quadrant mode, 3nz x 3nz block times 4 mirror modes x nrhs
//                                            -> S (in place)
//   K_iy : inverse y-FFT, keep iy < ny       -> T
//   K_ix : inverse x-FFT, keep ix < nx, 1/(ex ey), s*u + r1*(.) epilogue -> out
// The mode-major spectrum makes every contraction read/write a contiguous
// 3nz run per (mode, rhs); the transposes ride inside the FFT kernels' SMEM.
#include <algorithm>
#include <cmath>

#include "operator.cuh"

namespace emie_cu {

namespace {

__constant__ int kParX[6] = {1, 1, 1, -1, -1, 1};  // toeplitz.cpp:59
__constant__ int kParY[6] = {1, 1, 1, -1, 1, -1};  // toeplitz.cpp:60

__device__ __forceinline__ int comp_of(int e, int ntri, int nfull) {
  return e < 4 * ntri ? e / ntri : 4 + (e - 4 * ntri) / nfull;
}

// ld of an SMEM transform buffer: odd, so column walks hit distinct banks
__host__ __device__ inline int smem_ld(int n) { return n | 1; }

// ------------------------------------------------------------- spectra ----
// x pass: rows oi of the parity-extended offset sequence (toeplitz.cpp:140-151)
// for EC consecutive entries e; keep mx < qx.  R[(oi*qx + mx)*nent + e]
__global__ void spectra_x_kernel(const cplx* __restrict__ blocks, cplx* __restrict__ R,
                                 const cplx* __restrict__ tw, FftPlan pl, int nx, int qx,
                                 int nent, int ntri, int nfull, int EC) {
  extern __shared__ cplx sm[];
  const int ex = pl.n, ld = smem_ld(ex);
  cplx* a = sm;
  cplx* b = a + EC * ld;
  cplx* t = b + EC * ld;
  const int oi = blockIdx.x;
  const int e0 = blockIdx.y * EC;
  load_twiddles(t, tw, ex);
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
    a[tt * ld + j] = v;
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, EC, pl, t, false);
  for (int idx = threadIdx.x; idx < EC * qx; idx += blockDim.x) {
    const int tt = idx % EC, mx = idx / EC;
    const int e = e0 + tt;
    if (e < nent) R[(static_cast<size_t>(oi) * qx + mx) * nent + e] = res[tt * ld + mx];
  }
}

// y pass over the x-transformed rows, parity-extended in oi; keep my < qy
__global__ void spectra_y_kernel(const cplx* __restrict__ R, cplx* __restrict__ spec,
                                 const cplx* __restrict__ tw, FftPlan pl, int ny, int qx,
                                 int qy, int nent, int ntri, int nfull, int EC,
                                 const int2* __restrict__ emap, int nentD) {
  extern __shared__ cplx sm[];
  const int ey = pl.n, ld = smem_ld(ey);
  cplx* a = sm;
  cplx* b = a + EC * ld;
  cplx* t = b + EC * ld;
  const int mx = blockIdx.x;
  const int e0 = blockIdx.y * EC;
  load_twiddles(t, tw, ey);
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
    a[tt * ld + j] = v;
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, EC, pl, t, false);
  for (int idx = threadIdx.x; idx < EC * qy; idx += blockDim.x) {
    const int tt = idx % EC, my = idx / EC;
    const int e = e0 + tt;
    if (e < nent) {
      const int2 m = emap[e];
      cplx* blk = spec + (static_cast<size_t>(my) * qx + mx) * nentD;
      const cplx v = res[tt * ld + my];
      blk[m.x] = v;
      if (m.y >= 0) blk[m.y] = v;
    }
  }
}

// --------------------------------------------------------------- apply ----
// forward x: rows q = (r, plane, iy) are contiguous in the GridVector layout
__global__ void apply_fx_kernel(const cplx* __restrict__ u, const cplx* __restrict__ r2,
                                cplx* __restrict__ T, const cplx* __restrict__ tw, FftPlan pl,
                                int nx, int ny, int nz, long long rows, int RT) {
  extern __shared__ cplx sm[];
  const int ex = pl.n, ld = smem_ld(ex);
  cplx* a = sm;
  cplx* b = a + RT * ld;
  cplx* t = b + RT * ld;
  const long long q0 = static_cast<long long>(blockIdx.x) * RT;
  load_twiddles(t, tw, ex);
  const int ny_nx = ny * nx;
  for (int idx = threadIdx.x; idx < RT * ex; idx += blockDim.x) {
    const int tt = idx / ex, j = idx - tt * ex;
    const long long q = q0 + tt;
    cplx v = {0.0, 0.0};
    if (q < rows && j < nx) {
      v = ldg(u + q * nx + j);
      if (r2) {
        // cell index: plane % nz, iy; r2 is shared by the three components
        const long long pr = q / ny;  // r*3nz + plane
        const int iz = static_cast<int>(pr % (3 * nz)) % nz;
        const int iy = static_cast<int>(q % ny);
        v = ldg(r2 + static_cast<long long>(iz) * ny_nx + iy * nx + j) * v;
      }
    }
    a[tt * ld + j] = v;
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, RT, pl, t, false);
  for (int idx = threadIdx.x; idx < RT * ex; idx += blockDim.x) {
    const int tt = idx / ex, j = idx - tt * ex;
    const long long q = q0 + tt;
    if (q < rows) T[q * ex + j] = res[tt * ld + j];
  }
}

// forward y with transpose to mode-major S[r][my][mx][plane].
// CTA tile: PC planes x XC columns of one rhs.
__global__ void apply_fy_kernel(const cplx* __restrict__ T, cplx* __restrict__ S,
                                const cplx* __restrict__ tw, FftPlan pl, int ny, int ex,
                                int np, int PC, int XC) {
  extern __shared__ cplx sm[];
  const int ey = pl.n, ld = smem_ld(ey);
  const int ntr = PC * XC;
  cplx* a = sm;
  cplx* b = a + ntr * ld;
  cplx* t = b + ntr * ld;
  const int x0 = blockIdx.x * XC;
  const int p0 = blockIdx.y * PC;
  const int r = blockIdx.z;
  load_twiddles(t, tw, ey);
  const int xc = min(XC, ex - x0), pc = min(PC, np - p0);
  for (int idx = threadIdx.x; idx < ntr * ey; idx += blockDim.x) {
    const int x = idx % XC;
    const int rest = idx / XC;
    const int p = rest % PC, j = rest / PC;
    cplx v = {0.0, 0.0};
    if (j < ny && x < xc && p < pc)
      v = ldg(T + ((static_cast<size_t>(r) * np + p0 + p) * ny + j) * ex + x0 + x);
    a[(p * XC + x) * ld + j] = v;
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, ntr, pl, t, false);
  for (int idx = threadIdx.x; idx < ntr * ey; idx += blockDim.x) {
    const int p = idx % PC;
    const int rest = idx / PC;
    const int x = rest % XC, my = rest / XC;
    if (x < xc && p < pc)
      S[((static_cast<size_t>(r) * ey + my) * ex + x0 + x) * np + p0 + p] = res[(p * XC + x) * ld + my];
  }
}

// inverse y from mode-major S back to T[r][plane][iy][mx], rows iy < ny
__global__ void apply_iy_kernel(const cplx* __restrict__ S, cplx* __restrict__ T,
                                const cplx* __restrict__ tw, FftPlan pl, int ny, int ex,
                                int np, int PC, int XC) {
  extern __shared__ cplx sm[];
  const int ey = pl.n, ld = smem_ld(ey);
  const int ntr = PC * XC;
  cplx* a = sm;
  cplx* b = a + ntr * ld;
  cplx* t = b + ntr * ld;
  const int x0 = blockIdx.x * XC;
  const int p0 = blockIdx.y * PC;
  const int r = blockIdx.z;
  load_twiddles(t, tw, ey);
  const int xc = min(XC, ex - x0), pc = min(PC, np - p0);
  for (int idx = threadIdx.x; idx < ntr * ey; idx += blockDim.x) {
    const int p = idx % PC;
    const int rest = idx / PC;
    const int x = rest % XC, j = rest / XC;
    cplx v = {0.0, 0.0};
    if (x < xc && p < pc) v = ldg(S + ((static_cast<size_t>(r) * ey + j) * ex + x0 + x) * np + p0 + p);
    a[(p * XC + x) * ld + j] = v;
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, ntr, pl, t, true);
  for (int idx = threadIdx.x; idx < ntr * ny; idx += blockDim.x) {
    const int x = idx % XC;
    const int rest = idx / XC;
    const int p = rest % PC, iy = rest / PC;
    if (x < xc && p < pc)
      T[((static_cast<size_t>(r) * np + p0 + p) * ny + iy) * ex + x0 + x] = res[(p * XC + x) * ld + iy];
  }
}

// inverse x, truncate, 1/(ex ey), optional system epilogue (cie.cpp:67-72)
__global__ void apply_ix_kernel(const cplx* __restrict__ T, const cplx* __restrict__ u,
                                cplx* __restrict__ out, const cplx* __restrict__ s,
                                const double* __restrict__ r1, const cplx* __restrict__ tw,
                                FftPlan pl, int nx, int ny, int nz, long long rows, int RT,
                                double inv) {
  extern __shared__ cplx sm[];
  const int ex = pl.n, ld = smem_ld(ex);
  cplx* a = sm;
  cplx* b = a + RT * ld;
  cplx* t = b + RT * ld;
  const long long q0 = static_cast<long long>(blockIdx.x) * RT;
  load_twiddles(t, tw, ex);
  for (int idx = threadIdx.x; idx < RT * ex; idx += blockDim.x) {
    const int tt = idx / ex, j = idx - tt * ex;
    const long long q = q0 + tt;
    a[tt * ld + j] = q < rows ? ldg(T + q * ex + j) : cplx{0.0, 0.0};
  }
  __syncthreads();
  cplx* res = fft_smem(a, b, ld, RT, pl, t, true);
  const int ny_nx = ny * nx;
  for (int idx = threadIdx.x; idx < RT * nx; idx += blockDim.x) {
    const int tt = idx / nx, ix = idx - tt * nx;
    const long long q = q0 + tt;
    if (q >= rows) continue;
    cplx v = inv * res[tt * ld + ix];
    if (s) {
      const long long pr = q / ny;
      const int iz = static_cast<int>(pr % (3 * nz)) % nz;
      const int iy = static_cast<int>(q % ny);
      const long long cell = static_cast<long long>(iz) * ny_nx + iy * nx + ix;
      v = ldg(s + cell) * ldg(u + q * nx + ix) + __ldg(r1 + cell) * v;
    }
    out[q * nx + ix] = v;
  }
}

// ------------------------------------------------------ contraction -------
// Per quadrant mode (qmy, qmx): out = M u for the 3nz x 3nz coupling M of the
// mode (toeplitz.cpp:197-258), applied to every mirror mode and rhs. Mirror
// modes reuse the quadrant block with the fold signs D = diag(fx, fy, 1):
// M(mirror) = D M D (toeplitz.cpp:213-250), folded into the staged inputs and
// the outputs. One warp owns one mode at a time (persistent grid-stride over
// modes); lane k computes output rows (x,k), (y,k), (z,k) for CB columns
// (column = (mirror, rhs)), stepping t over the wrapped diagonals so every
// coefficient load of the warp is one contiguous run (see operator.cuh).
// The inputs of the mode sit in the warp's SMEM slot: lane k reads entry
// (k + t) mod nz, 32 consecutive complex -> conflict-free.
constexpr int kCtWarps = 8;

template <int CB>
__global__ void __launch_bounds__(kCtWarps * 32, 1)
    contract_kernel(const cplx* __restrict__ op, cplx* S, int nz, int nsd, int nentD, int ex,
                    int ey, int qx, int nmodes, int nrhs) {
  extern __shared__ cplx sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = 3 * nz;
  cplx* U = sm + static_cast<size_t>(warp) * CB * np;  // [col][plane]
  const size_t E = static_cast<size_t>(ex) * ey;
  const int gw = blockIdx.x * kCtWarps + warp, nw = gridDim.x * kCtWarps;
  for (int qm = gw; qm < nmodes; qm += nw) {
    const int qmy = qm / qx, qmx = qm - qmy * qx;
    const bool mx_ok = qmx > 0 && (ex - qmx) > ex / 2;
    const bool my_ok = qmy > 0 && (ey - qmy) > ey / 2;
    int mode[4];
    int nmir = 0;
    mode[nmir++] = qmy * ex + qmx;
    if (mx_ok) mode[nmir++] = qmy * ex + (ex - qmx);
    if (my_ok) mode[nmir++] = (ey - qmy) * ex + qmx;
    if (mx_ok && my_ok) mode[nmir++] = (ey - qmy) * ex + (ex - qmx);
    // mirror mi's signs: x flipped for the 2nd (and 4th), y for the 3rd/4th
    auto fx_of = [&](int mi) { return (mx_ok && (mi & 1)) ? -1.0 : 1.0; };
    auto fy_of = [&](int mi) { return (my_ok && (mi >= (mx_ok ? 2 : 1))) ? -1.0 : 1.0; };
    const int ncol = nmir * nrhs;
    __syncwarp();
    for (int i = lane; i < CB * np; i += 32) {
      const int col = i / np, pl = i - col * np;
      cplx v = {0.0, 0.0};
      if (col < ncol) {
        const int mi = col / nrhs, r = col - mi * nrhs;
        v = S[(static_cast<size_t>(r) * E + mode[mi]) * np + pl];
        const int c = pl / nz;
        if (c == 0) v = fx_of(mi) * v;
        if (c == 1) v = fy_of(mi) * v;
      }
      U[i] = v;
    }
    __syncwarp();
    const cplx* blk = op + static_cast<size_t>(qm) * nentD;
    const cplx* Dxx = blk;
    const cplx* Dyy = blk + nsd * nz;
    const cplx* Dzz = blk + 2 * nsd * nz;
    const cplx* Dxy = blk + 3 * nsd * nz;
    const cplx* Dxz = blk + 4 * nsd * nz;
    const cplx* Dyz = Dxz + nz * nz;
    for (int kb = 0; kb < nz; kb += 32) {
      const int k = kb + lane;
      const int kc = k < nz ? k : 0;
      cplx ax[CB], ay[CB], az[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) ax[c] = ay[c] = az[c] = cplx{0.0, 0.0};
      // t visited in pairs (0, 1, nz-1, 2, nz-2, ...): the two uses of each
      // diagonal are adjacent, so the second hits L1
      for (int i = 0; i < nz; ++i) {
        const int t = (i == 0) ? 0 : ((i & 1) ? (i + 1) >> 1 : nz - (i >> 1));
        int kp = kc + t;
        if (kp >= nz) kp -= nz;
        const bool lo = t <= nz - t;
        const int so = (lo ? t : nz - t) * nz + (lo ? kc : kp);
        const cplx mxx = ldg(Dxx + so), myy = ldg(Dyy + so), mzz = ldg(Dzz + so), mxy = ldg(Dxy + so);
        const int tb = (t == 0) ? 0 : nz - t;
        const cplx xz_k = ldg(Dxz + t * nz + kc), yz_k = ldg(Dyz + t * nz + kc);
        const cplx xz_t = -ldg(Dxz + tb * nz + kp), yz_t = -ldg(Dyz + tb * nz + kp);
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const cplx* u = U + c * np;
          const cplx ux = u[kp], uy = u[nz + kp], uz = u[2 * nz + kp];
          cmac(ax[c], mxx, ux);
          cmac(ax[c], mxy, uy);
          cmac(ax[c], xz_k, uz);
          cmac(ay[c], mxy, ux);
          cmac(ay[c], myy, uy);
          cmac(ay[c], yz_k, uz);
          cmac(az[c], xz_t, ux);
          cmac(az[c], yz_t, uy);
          cmac(az[c], mzz, uz);
        }
      }
      if (k < nz) {
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          if (c < ncol) {
            const int mi = c / nrhs, r = c - mi * nrhs;
            cplx* o = S + (static_cast<size_t>(r) * E + mode[mi]) * np;
            o[k] = fx_of(mi) * ax[c];
            o[nz + k] = fy_of(mi) * ay[c];
            o[2 * nz + k] = az[c];
          }
        }
      }
    }
  }
}

int pick_rows(int n) { return std::max(1, std::min(64, 2048 / std::max(1, n))); }

void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

}  // namespace

// ------------------------------------------------------------------ host --
void transform_blocks(Operator& op, const cplx* d_blocks, cudaStream_t st) {
  const int nent = op.nent;
  cplx* R = scratch<cplx>(static_cast<size_t>(op.ny) * op.qx * nent, st);
  {
    const int EC = std::max(1, std::min(16, 4096 / op.ex));
    const size_t smem = (2 * static_cast<size_t>(EC) * smem_ld(op.ex) + op.ex) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(spectra_x_kernel), smem);
    dim3 grid(op.ny, ceil_div(nent, EC));
    spectra_x_kernel<<<grid, 256, smem, st>>>(d_blocks, R, op.tw_x, op.plan_x, op.nx, op.qx,
                                              nent, op.ntri, op.nfull, EC);
    check_launch("spectra_x_kernel");
  }
  {
    const int EC = std::max(1, std::min(16, 4096 / op.ey));
    const size_t smem = (2 * static_cast<size_t>(EC) * smem_ld(op.ey) + op.ey) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(spectra_y_kernel), smem);
    dim3 grid(op.qx, ceil_div(nent, EC));
    spectra_y_kernel<<<grid, 256, smem, st>>>(R, op.spec, op.tw_y, op.plan_y, op.ny, op.qx,
                                              op.qy, nent, op.ntri, op.nfull, EC, op.emap,
                                              op.nentD);
    check_launch("spectra_y_kernel");
  }
  release(R, st);
}

void apply_b(const Operator& op, const cplx* d_in, cplx* d_out, int nrhs, const System* sys,
             cudaStream_t st) {
  const int np = 3 * op.nz;
  const long long rows = static_cast<long long>(nrhs) * np * op.ny;
  cplx* T = scratch<cplx>(static_cast<size_t>(rows) * op.ex, st);
  cplx* S = scratch<cplx>(static_cast<size_t>(nrhs) * op.lateral() * np, st);
  // K_fx
  profile_mark(0, true, st);
  {
    const int RT = pick_rows(op.ex);
    const size_t smem = (2 * static_cast<size_t>(RT) * smem_ld(op.ex) + op.ex) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_fx_kernel), smem);
    apply_fx_kernel<<<ceil_div(rows, RT), 256, smem, st>>>(
        d_in, sys ? sys->r2 : nullptr, T, op.tw_x, op.plan_x, op.nx, op.ny, op.nz, rows, RT);
    check_launch("apply_fx_kernel");
  }
  profile_mark(0, false, st);
  // K_fy
  const int XC = std::min(2, op.ex);
  const int PC = std::max(1, std::min(np, 2048 / (op.ey * XC)));
  profile_mark(1, true, st);
  {
    const size_t smem =
        (2 * static_cast<size_t>(PC) * XC * smem_ld(op.ey) + op.ey) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_fy_kernel), smem);
    dim3 grid(ceil_div(op.ex, XC), ceil_div(np, PC), nrhs);
    apply_fy_kernel<<<grid, 256, smem, st>>>(T, S, op.tw_y, op.plan_y, op.ny, op.ex, np, PC, XC);
    check_launch("apply_fy_kernel");
  }
  profile_mark(1, false, st);
  // K_ct: up to two right-hand sides per launch (8 columns of a full mode)
  profile_mark(2, true, st);
  {
    int sms = 0, dev = 0;
    EMIE_CUDA(cudaGetDevice(&dev));
    EMIE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int nmodes = static_cast<int>(op.modes());
    const int grid = std::max(1, std::min(sms, ceil_div(nmodes, kCtWarps)));
    for (int r0 = 0; r0 < nrhs; r0 += 2) {
      const int g = std::min(2, nrhs - r0);
      cplx* Sg = S + static_cast<size_t>(r0) * op.lateral() * np;
      const int CB = g == 2 ? 8 : 4;
      const size_t smem = static_cast<size_t>(kCtWarps) * CB * np * sizeof(cplx);
      if (CB == 8) {
        set_smem(reinterpret_cast<const void*>(contract_kernel<8>), smem);
        contract_kernel<8><<<grid, kCtWarps * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD,
                                                               op.ex, op.ey, op.qx, nmodes, g);
      } else {
        set_smem(reinterpret_cast<const void*>(contract_kernel<4>), smem);
        contract_kernel<4><<<grid, kCtWarps * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD,
                                                               op.ex, op.ey, op.qx, nmodes, g);
      }
      check_launch("contract_kernel");
    }
  }
  profile_mark(2, false, st);
  // K_iy
  profile_mark(3, true, st);
  {
    const size_t smem =
        (2 * static_cast<size_t>(PC) * XC * smem_ld(op.ey) + op.ey) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_iy_kernel), smem);
    dim3 grid(ceil_div(op.ex, XC), ceil_div(np, PC), nrhs);
    apply_iy_kernel<<<grid, 256, smem, st>>>(S, T, op.tw_y, op.plan_y, op.ny, op.ex, np, PC, XC);
    check_launch("apply_iy_kernel");
  }
  profile_mark(3, false, st);
  // K_ix
  profile_mark(4, true, st);
  {
    const int RT = pick_rows(op.ex);
    const size_t smem = (2 * static_cast<size_t>(RT) * smem_ld(op.ex) + op.ex) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_ix_kernel), smem);
    const double inv = 1.0 / static_cast<double>(op.lateral());
    apply_ix_kernel<<<ceil_div(rows, RT), 256, smem, st>>>(
        T, d_in, d_out, sys ? sys->s : nullptr, sys ? sys->r1 : nullptr, op.tw_x, op.plan_x,
        op.nx, op.ny, op.nz, rows, RT, inv);
    check_launch("apply_ix_kernel");
  }
  profile_mark(4, false, st);
  release(S, st);
  release(T, st);
}

}  // namespace emie_cu
