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
                                 int qy, int nent, int ntri, int nfull, int EC) {
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
    if (e < nent) spec[(static_cast<size_t>(my) * qx + mx) * nent + e] = res[tt * ld + my];
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
// One CTA per quadrant mode (qmy, qmx). The block's six stored components
// are expanded in SMEM into symmetric / full 32x32 tiles (ld 33: row and
// column walks are both bank-conflict free), then warp a in {x, y, z}
// computes output rows (a, k) (lane = k) for CB columns at once; a column is
// one (mirror mode, rhs) pair. Mirror modes reuse the quadrant block with
// the fold signs D = diag(fx, fy, 1): M(mode) = D M(quadrant) D
// (toeplitz.cpp:213-250), applied to the staged inputs and to the outputs.
constexpr int kTile = 32;
constexpr int kTld = kTile + 1;
constexpr int kTsz = kTile * kTld;

template <int CB>
__global__ void __launch_bounds__(96) contract_kernel(const cplx* __restrict__ op, cplx* S,
                                                      const uint32_t* __restrict__ trilut, int nz,
                                                      int ex, int ey, int qx, int nrhs,
                                                      int ncolpad) {
  extern __shared__ cplx sm[];
  const int ntri = nz * (nz + 1) / 2, nfull = nz * nz, nent = 4 * ntri + 2 * nfull;
  const int np = 3 * nz;
  const size_t E = static_cast<size_t>(ex) * ey;
  const int qm = blockIdx.x;
  const int qmy = qm / qx, qmx = qm - qmy * qx;
  const bool mx_ok = qmx > 0 && (ex - qmx) > ex / 2;
  const bool my_ok = qmy > 0 && (ey - qmy) > ey / 2;
  int mode[4];
  double fxs[4], fys[4];
  int nmir = 0;
  mode[nmir] = qmy * ex + qmx; fxs[nmir] = 1.0; fys[nmir] = 1.0; ++nmir;
  if (mx_ok) { mode[nmir] = qmy * ex + (ex - qmx); fxs[nmir] = -1.0; fys[nmir] = 1.0; ++nmir; }
  if (my_ok) { mode[nmir] = (ey - qmy) * ex + qmx; fxs[nmir] = 1.0; fys[nmir] = -1.0; ++nmir; }
  if (mx_ok && my_ok) { mode[nmir] = (ey - qmy) * ex + (ex - qmx); fxs[nmir] = -1.0; fys[nmir] = -1.0; ++nmir; }
  const int ncol = nmir * nrhs;

  // tiles: 0 xx, 1 yy, 2 zz, 3 xy, 4 xz(kb,kpb), 5 yz(kb,kpb), 6 xz(kpb,kb), 7 yz(kpb,kb)
  cplx* tile = sm;
  cplx* U = sm + 8 * kTsz;  // [col][plane], ncolpad columns
  const cplx* blk = op + static_cast<size_t>(qm) * nent;

  // stage the inputs of every column (zero-padded to ncolpad)
  for (int i = threadIdx.x; i < ncolpad * np; i += blockDim.x) {
    const int col = i / np, pl = i - col * np;
    cplx v = {0.0, 0.0};
    if (col < ncol) {
      const int mi = col / nrhs, r = col - mi * nrhs;
      v = S[(static_cast<size_t>(r) * E + mode[mi]) * np + pl];
      const int c = pl / nz;
      if (c == 0) v = fxs[mi] * v;
      if (c == 1) v = fys[mi] * v;
    }
    U[i] = v;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = warp;  // output component
  for (int kb = 0; kb < nz; kb += kTile) {
    for (int cb = 0; cb < ncolpad; cb += CB) {
      cplx acc[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) acc[c] = {0.0, 0.0};
      for (int kpb = 0; kpb < nz; kpb += kTile) {
        __syncthreads();  // previous tile fully consumed (and U staged)
        // stage tiles for rows kb.., cols kpb..
        for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
          const int dk = i / kTile, dkp = i - dk * kTile;
          const int k = kb + dk, kp = kpb + dkp;
          const int o = dk * kTld + dkp;
          if (k < nz && kp < nz) {
            const int lo = min(k, kp), hi = max(k, kp);
            const int s = lo * nz - lo * (lo - 1) / 2 + (hi - lo);
            tile[0 * kTsz + o] = ldg(blk + s);
            tile[1 * kTsz + o] = ldg(blk + ntri + s);
            tile[2 * kTsz + o] = ldg(blk + 2 * ntri + s);
            tile[3 * kTsz + o] = ldg(blk + 3 * ntri + s);
            tile[4 * kTsz + o] = ldg(blk + 4 * ntri + k * nz + kp);
            tile[5 * kTsz + o] = ldg(blk + 4 * ntri + nfull + k * nz + kp);
            // transposed pair: element (kp, k) stored at [dkp][dk]
            tile[6 * kTsz + dkp * kTld + dk] = ldg(blk + 4 * ntri + kp * nz + k);
            tile[7 * kTsz + dkp * kTld + dk] = ldg(blk + 4 * ntri + nfull + kp * nz + k);
          } else {
            const cplx z = {0.0, 0.0};
            for (int m = 0; m < 6; ++m) tile[m * kTsz + o] = z;
            tile[6 * kTsz + dkp * kTld + dk] = z;
            tile[7 * kTsz + dkp * kTld + dk] = z;
          }
        }
        __syncthreads();
        // operand tiles of this warp's row component
        //  x: xx, xy, xz      y: xy, yy, yz      z: -xz^T, -yz^T, zz
        const cplx* A0 = tile + (a == 0 ? 0 : a == 1 ? 3 : 6) * kTsz;
        const cplx* A1 = tile + (a == 0 ? 3 : a == 1 ? 1 : 7) * kTsz;
        const cplx* A2 = tile + (a == 0 ? 4 : a == 1 ? 5 : 2) * kTsz;
        const double sg = a == 2 ? -1.0 : 1.0;
        const int kpn = min(kTile, nz - kpb);
        for (int dkp = 0; dkp < kpn; ++dkp) {
          // tiles 6/7 hold (kp, k) at [dkp][dk]: read with the row index swapped
          const int o = lane * kTld + dkp;
          const int ot = dkp * kTld + lane;
          const cplx m0 = sg * A0[a == 2 ? ot : o];
          const cplx m1 = sg * A1[a == 2 ? ot : o];
          const cplx m2 = A2[o];
          const int kp = kpb + dkp;
#pragma unroll
          for (int c = 0; c < CB; ++c) {
            const cplx* uc = U + (cb + c) * np;
            cmac(acc[c], m0, uc[kp]);
            cmac(acc[c], m1, uc[nz + kp]);
            cmac(acc[c], m2, uc[2 * nz + kp]);
          }
        }
      }
      const int k = kb + lane;
      if (k < nz) {
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const int col = cb + c;
          if (col < ncol) {
            const int mi = col / nrhs, r = col - mi * nrhs;
            cplx v = acc[c];
            if (a == 0) v = fxs[mi] * v;
            if (a == 1) v = fys[mi] * v;
            S[(static_cast<size_t>(r) * E + mode[mi]) * np + a * nz + k] = v;
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
                                              op.qy, nent, op.ntri, op.nfull, EC);
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
  {
    const int RT = pick_rows(op.ex);
    const size_t smem = (2 * static_cast<size_t>(RT) * smem_ld(op.ex) + op.ex) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_fx_kernel), smem);
    apply_fx_kernel<<<ceil_div(rows, RT), 256, smem, st>>>(
        d_in, sys ? sys->r2 : nullptr, T, op.tw_x, op.plan_x, op.nx, op.ny, op.nz, rows, RT);
    check_launch("apply_fx_kernel");
  }
  // K_fy
  const int XC = std::min(2, op.ex);
  const int PC = std::max(1, std::min(np, 2048 / (op.ey * XC)));
  {
    const size_t smem =
        (2 * static_cast<size_t>(PC) * XC * smem_ld(op.ey) + op.ey) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_fy_kernel), smem);
    dim3 grid(ceil_div(op.ex, XC), ceil_div(np, PC), nrhs);
    apply_fy_kernel<<<grid, 256, smem, st>>>(T, S, op.tw_y, op.plan_y, op.ny, op.ex, np, PC, XC);
    check_launch("apply_fy_kernel");
  }
  // K_ct
  {
    const int ncolmax = 4 * nrhs;
    int CB = 8;
    if (ncolmax <= 1) CB = 1;
    else if (ncolmax <= 2) CB = 2;
    else if (ncolmax <= 4) CB = 4;
    const int ncolpad = ceil_div(ncolmax, CB) * CB;
    const size_t smem = (8 * static_cast<size_t>(kTsz) + static_cast<size_t>(ncolpad) * np) * sizeof(cplx);
    const void* fn = CB == 8 ? reinterpret_cast<const void*>(contract_kernel<8>)
                   : CB == 4 ? reinterpret_cast<const void*>(contract_kernel<4>)
                   : CB == 2 ? reinterpret_cast<const void*>(contract_kernel<2>)
                             : reinterpret_cast<const void*>(contract_kernel<1>);
    set_smem(fn, smem);
    const int grid = static_cast<int>(op.modes());
    switch (CB) {
      case 8: contract_kernel<8><<<grid, 96, smem, st>>>(op.spec, S, op.trilut, op.nz, op.ex, op.ey, op.qx, nrhs, ncolpad); break;
      case 4: contract_kernel<4><<<grid, 96, smem, st>>>(op.spec, S, op.trilut, op.nz, op.ex, op.ey, op.qx, nrhs, ncolpad); break;
      case 2: contract_kernel<2><<<grid, 96, smem, st>>>(op.spec, S, op.trilut, op.nz, op.ex, op.ey, op.qx, nrhs, ncolpad); break;
      default: contract_kernel<1><<<grid, 96, smem, st>>>(op.spec, S, op.trilut, op.nz, op.ex, op.ey, op.qx, nrhs, ncolpad); break;
    }
    check_launch("contract_kernel");
  }
  // K_iy
  {
    const size_t smem =
        (2 * static_cast<size_t>(PC) * XC * smem_ld(op.ey) + op.ey) * sizeof(cplx);
    set_smem(reinterpret_cast<const void*>(apply_iy_kernel), smem);
    dim3 grid(ceil_div(op.ex, XC), ceil_div(np, PC), nrhs);
    apply_iy_kernel<<<grid, 256, smem, st>>>(S, T, op.tw_y, op.plan_y, op.ny, op.ex, np, PC, XC);
    check_launch("apply_iy_kernel");
  }
  // K_ix
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
  release(S, st);
  release(T, st);
}

}  // namespace emie_cu
