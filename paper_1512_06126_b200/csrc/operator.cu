// Spectral operator build (transform_operator) and the CIE operator apply
// (apply(SpectralOperator), apply(SystemOperator)) for sm_100a.
//
// Reference: src/toeplitz.cpp:92-161 (spectra), 163-283 (apply),
//            src/cie.cpp:56-73 (system apply).
//
// The lateral FFT stages live in lateral.cu. Apply data flow for nrhs fields (all complex128):
//   u [r][plane][iy][ix]            plane = c*nz + iz (GridVector layout)
//   K_fx : r2-scale, zero-pad, x-FFT        -> T [r][plane][iy][mx]
//   K_fy : zero-pad, y-FFT, transpose       -> S [r][mx][my][plane]  (mode-major)
//   K_ct : per quadrant mode, 3nz x 3nz block times 4 mirror modes x nrhs
//                                            -> S (in place)
//   K_iy : inverse y-FFT, keep iy < ny       -> T
//   K_ix : inverse x-FFT, keep ix < nx, 1/(ex ey), s*u + r1*(.) epilogue -> out
// The mode-major spectrum makes every contraction read/write a contiguous
// 3nz run per (mode, rhs); the transposes ride inside the FFT kernels' SMEM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "operator.cuh"

namespace emie_cu {

namespace {

// ------------------------------------------------------ contraction -------
// Per quadrant mode (qmy, qmx): out = M u for the 3nz x 3nz coupling M of the
// mode (toeplitz.cpp:197-258), applied to every mirror mode and rhs. Mirror
// modes reuse the quadrant block: M(mirror) = D M D with the fold signs
// D = diag(fx, fy, 1) (toeplitz.cpp:213-250); the spectrum passes apply D on
// store and on load (lateral.cu), so this kernel is sign-free.
// One warp owns one mode at a time (persistent, grid-stride over modes);
// lane k computes output rows (x,k), (y,k), (z,k) for CB columns (column =
// (mirror, rhs)), stepping t over the wrapped diagonals so every coefficient
// load of the warp is one contiguous run (see operator.cuh). The inputs of
// the next mode are brought into the warp's second SMEM buffer by TMA bulk
// copies (cp.async.bulk, one per column, mbarrier-tracked) while the current
// mode computes; lane k reads entry (k + t) mod nz -> conflict-free.
constexpr int kCtWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}

struct ModeCols {
  int mode[4];
  int nmir;
};
__device__ __forceinline__ ModeCols mode_cols(int qm, int qx, int ex, int ey) {
  ModeCols mc;
  const int qmy = qm / qx, qmx = qm - qmy * qx;
  const bool mx_ok = qmx > 0 && (ex - qmx) > ex / 2;
  const bool my_ok = qmy > 0 && (ey - qmy) > ey / 2;
  mc.nmir = 0;
  // spectrum mode index mx*ey + my (S layout [r][mx][my][plane], lateral.cu)
  mc.mode[mc.nmir++] = qmx * ey + qmy;
  if (mx_ok) mc.mode[mc.nmir++] = (ex - qmx) * ey + qmy;
  if (my_ok) mc.mode[mc.nmir++] = qmx * ey + (ey - qmy);
  if (mx_ok && my_ok) mc.mode[mc.nmir++] = (ex - qmx) * ey + (ey - qmy);
  return mc;
}

template <int CB>
__global__ void __launch_bounds__(kCtWarps * 32, 1)
    contract_kernel(const cplx* __restrict__ op, cplx* S, int nz, int nsd, int nentD, int ex,
                    int ey, int qx, int nmodes, int nrhs) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = 3 * nz;
  const size_t colbytes = static_cast<size_t>(np) * sizeof(cplx);
  // per warp: mbarriers[2] then two buffers of CB columns
  const int wpb = blockDim.x >> 5;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw) + 2 * warp;
  cplx* ubase = reinterpret_cast<cplx*>(smraw + 16 * wpb) + static_cast<size_t>(warp) * 2 * CB * np;
  const size_t E = static_cast<size_t>(ex) * ey;
  const int gw = blockIdx.x * wpb + warp, nw = gridDim.x * wpb;
  if (lane == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = lane; i < 2 * CB * np; i += 32) ubase[i] = cplx{0.0, 0.0};
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  auto issue = [&](int qm, int buf) {
    if (lane == 0) {
      const ModeCols mc = mode_cols(qm, qx, ex, ey);
      const int ncol = mc.nmir * nrhs;
      mbar_expect_tx(mbar + buf, static_cast<uint32_t>(ncol * colbytes));
      cplx* dst = ubase + static_cast<size_t>(buf) * CB * np;
      for (int col = 0; col < ncol; ++col) {
        const int mi = col / nrhs, r = col - mi * nrhs;
        bulk_g2s(dst + static_cast<size_t>(col) * np, S + (static_cast<size_t>(r) * E + mc.mode[mi]) * np,
                 static_cast<uint32_t>(colbytes), mbar + buf);
      }
    }
  };
  uint32_t phase[2] = {0u, 0u};
  if (gw < nmodes) issue(gw, 0);
  int it = 0;
  for (int qm = gw; qm < nmodes; qm += nw, ++it) {
    const int buf = it & 1;
    if (qm + nw < nmodes) issue(qm + nw, buf ^ 1);
    mbar_wait(mbar + buf, phase[buf]);
    phase[buf] ^= 1u;
    const cplx* U = ubase + static_cast<size_t>(buf) * CB * np;
    const ModeCols mc = mode_cols(qm, qx, ex, ey);
    const int ncol = mc.nmir * nrhs;
    const cplx* blk = op + static_cast<size_t>(qm) * nentD;
    const int ntri = nz * (nz + 1) / 2;
    const cplx* Dxx = blk;
    const cplx* Dyy = blk + ntri;
    const cplx* Dzz = blk + 2 * ntri;
    const cplx* Dxy = blk + 3 * ntri;
    const cplx* Dxz = blk + 4 * ntri;
    const cplx* Dyz = Dxz + nz * nz;
    for (int kb = 0; kb < nz; kb += 32) {
      const int k = kb + lane;
      const int kc = k < nz ? k : 0;
      cplx ax[CB], ay[CB], az[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) ax[c] = ay[c] = az[c] = cplx{0.0, 0.0};
      // t visited in pairs (0, 1, nz-1, 2, nz-2, ...): the two uses of each
      // diagonal are adjacent, so the second hits L1. The coefficients of
      // step i+1 are loaded while step i computes (L2 latency hidden).
      struct MSet {
        cplx xx, yy, zz, xy, xzk, yzk, xzt, yzt;
        int kp;
      };
      auto fetch = [&](int i) {
        MSet m;
        const int t = (i == 0) ? 0 : ((i & 1) ? (i + 1) >> 1 : nz - (i >> 1));
        int kp = kc + t;
        if (kp >= nz) kp -= nz;
        // symmetric slot (compact wrapped diagonals, operator.cuh)
        const int so = (2 * t < nz)   ? t * nz + kc
                       : (2 * t > nz) ? (nz - t) * nz + kp
                                      : t * nz + min(kc, kp);
        const int tb = (t == 0) ? 0 : nz - t;
        m.xx = ldg(Dxx + so);
        m.yy = ldg(Dyy + so);
        m.zz = ldg(Dzz + so);
        m.xy = ldg(Dxy + so);
        m.xzk = ldg(Dxz + t * nz + kc);
        m.yzk = ldg(Dyz + t * nz + kc);
        m.xzt = ldg(Dxz + tb * nz + kp);
        m.yzt = ldg(Dyz + tb * nz + kp);
        m.kp = kp;
        return m;
      };
      MSet cur = fetch(0);
      for (int i = 0; i < nz; ++i) {
        MSet nxt = cur;
        if (i + 1 < nz) nxt = fetch(i + 1);
        const int kp = cur.kp;
        const cplx mxzt = -cur.xzt, myzt = -cur.yzt;
        // term-major: consecutive MACs hit different columns (independent)
        cplx u[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = U[c * np + kp];
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ax[c], cur.xx, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ay[c], cur.xy, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(az[c], mxzt, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = U[c * np + nz + kp];
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ax[c], cur.xy, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ay[c], cur.yy, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(az[c], myzt, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = U[c * np + 2 * nz + kp];
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ax[c], cur.xzk, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ay[c], cur.yzk, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(az[c], cur.zz, u[c]);
        cur = nxt;
      }
      if (k < nz) {
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          if (c < ncol) {
            const int mi = c / nrhs, r = c - mi * nrhs;
            cplx* o = S + (static_cast<size_t>(r) * E + mc.mode[mi]) * np;
            o[k] = ax[c];
            o[nz + k] = ay[c];
            o[2 * nz + k] = az[c];
          }
        }
      }
    }
    // this buffer is refilled (async proxy) after the next iteration's wait
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
}

// ------------------------------------------- contraction on FP64 MMA -----
// Same product as contract_kernel, on the FP64 tensor cores (DMMA.8x8x4 via
// mma.sync.m8n8k4.f64): measured 37 TF/s at 4 warps/SM on B200, where DFMA
// needs ~32 warps to approach it. Used when nz is a multiple of 8 and
// nz <= 32 (the whole mode block fits in SMEM twice).
// One CTA (4 warps) owns one quadrant mode at a time, persistent over modes.
// An elected thread brings the next mode's coefficient block (nentD complex,
// one TMA bulk copy) and its input columns (one bulk copy per (mirror, rhs),
// column stride np + 4 for conflict-free fragment loads) into the second
// buffer while the CTA computes the current one.
// Output rows are 8-row tiles (component a, rows k0..k0+7): 3nz/8 tiles,
// round-robin over 8 warps (two per SMSP, so one warp's operand loads and
// adds overlap the other's MMAs; for nz = 32 every SMSP gets 3 tiles); the 8 columns are the MMA's N; K runs over
// (component b, kp) in steps of 4. Complex products use three real MMAs
// (P1 = Ar Br, P2 = Ai Bi, P3 = (Ar+Ai)(Br+Bi); re = P1 - P2, im = P3 - P1 - P2).
constexpr int kMmaWarps = 8;
constexpr int kMmaTilesPerWarp = 3;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NZ>
__global__ void __launch_bounds__(kMmaWarps * 32, 1)
    contract_mma_kernel(const cplx* __restrict__ op, const uint32_t* __restrict__ ctab, cplx* S,
                        int ex, int ey, int qx, int nmodes, int nrhs, int nentD) {
  constexpr int np = 3 * NZ, ldu = np + 4;
  constexpr int ntiles = np / 8, nk = np / 4;
  constexpr int TPW = (ntiles + kMmaWarps - 1) / kMmaWarps;  // tiles per warp
  constexpr int kBlkStages = 3, kUStages = 2;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bbar = reinterpret_cast<uint64_t*>(smraw);   // block stages
  uint64_t* ubar = bbar + kBlkStages;                     // input stages
  cplx* blkbuf = reinterpret_cast<cplx*>(smraw + 128);
  cplx* ubuf = blkbuf + kBlkStages * nentD;
  const size_t E = static_cast<size_t>(ex) * ey;
  constexpr uint32_t colbytes = np * sizeof(cplx);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBlkStages; ++i) mbar_init(bbar + i, 1);
    for (int i = 0; i < kUStages; ++i) mbar_init(ubar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kUStages * 8 * ldu; i += blockDim.x) ubuf[i] = cplx{0.0, 0.0};
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int G = gridDim.x;
  // j-th mode of this CTA: blockIdx.x + j*G
  auto issue_block = [&](int j) {
    const int qm = blockIdx.x + j * G;
    if (threadIdx.x == 0 && qm < nmodes) {
      const uint32_t blkbytes = nentD * sizeof(cplx);
      const int st = j % kBlkStages;
      mbar_expect_tx(bbar + st, blkbytes);
      bulk_g2s(blkbuf + st * nentD, op + static_cast<size_t>(qm) * nentD, blkbytes, bbar + st);
    }
  };
  auto issue_cols = [&](int j) {
    const int qm = blockIdx.x + j * G;
    if (threadIdx.x == 0 && qm < nmodes) {
      const ModeCols mc = mode_cols(qm, qx, ex, ey);
      const int ncol = mc.nmir * nrhs;
      const int st = j % kUStages;
      mbar_expect_tx(ubar + st, ncol * colbytes);
      cplx* dst = ubuf + st * 8 * ldu;
      for (int col = 0; col < ncol; ++col) {
        const int mi = col / nrhs, r = col - mi * nrhs;
        bulk_g2s(dst + col * ldu, S + (static_cast<size_t>(r) * E + mc.mode[mi]) * np, colbytes, ubar + st);
      }
    }
  };
  // fragment coordinates: A row fr / k fc; B k fc / col fr; C row fr, cols 2fc..2fc+1.
  // Tile m of component a holds rows {4m..4m+3} u {4m+nz/2..4m+nz/2+3}
  // (row fr -> 4m + fr/2 + (fr&1) nz/2): each quarter-warp reads rows r and
  // r + nz/2, which the MMA layout puts in disjoint banks (operator.cuh).
  const int fr = lane >> 2, fc = lane & 3;
  auto tile_row = [&](int rt) {
    const int a = (8 * rt) / NZ, m = rt - a * (NZ / 8);
    return a * NZ + 4 * m + (fr >> 1) + (fr & 1) * (NZ / 2);
  };
  // per-lane coefficient offsets of every (own tile, k step): mode independent
  uint32_t off[TPW][nk];
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    const int rt = warp + i * kMmaWarps;
    const int row = tile_row(rt), a = row / NZ, k = row - a * NZ;
#pragma unroll
    for (int ks = 0; ks < nk; ++ks) {
      const int b = (4 * ks) / NZ, kp = 4 * ks - b * NZ + fc;
      off[i][ks] = rt < ntiles ? __ldg(ctab + ((a * 3 + b) * NZ + k) * NZ + kp) : 0u;
    }
  }
  // prologue: blocks of modes 0, 1; inputs of mode 0
  issue_block(0);
  issue_block(1);
  issue_cols(0);
  int j = 0;
  for (int qm = blockIdx.x; qm < nmodes; qm += G, ++j) {
    // stages freed by mode j-1 (all warps passed the barrier at its end)
    issue_cols(j + 1);
    issue_block(j + 2);
    const int bs_ = j % kBlkStages, us_ = j % kUStages;
    mbar_wait(bbar + bs_, static_cast<uint32_t>((j / kBlkStages) & 1));
    mbar_wait(ubar + us_, static_cast<uint32_t>((j / kUStages) & 1));
    const cplx* blk = blkbuf + bs_ * nentD;
    const cplx* U = ubuf + us_ * 8 * ldu + fr * ldu + fc;
    double p1[TPW][2], p2[TPW][2], p3[TPW][2];
#pragma unroll
    for (int i = 0; i < TPW; ++i) p1[i][0] = p1[i][1] = p2[i][0] = p2[i][1] = p3[i][0] = p3[i][1] = 0.0;
    {
#pragma unroll
      for (int ks = 0; ks < nk; ++ks) {
        const cplx bu = U[4 * ks];  // B[k = fc][col = fr]
        const double bs = bu.re + bu.im;
        // Branch-free: tiles past ntiles compute on offset 0 and are never
        // stored; the zx / zy negation flips the sign bit of the (shared) B
        // fragment (with NZ == 32 and 8 warps, tile i = 1 is the z component,
        // so the flag folds at compile time).
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const uint32_t o = off[i][ks];
          const cplx m = blk[o & 0x7fffffffu];
          unsigned long long sg;
          if (NZ == 32 && kMmaWarps == 8)  // tiles w, w+8: only i == 1 is a z tile
            sg = (i == 1 && (4 * ks) / NZ < 2) ? 0x8000000000000000ull : 0ull;
          else
            sg = static_cast<unsigned long long>(o >> 31) << 63;
          const double br = __longlong_as_double(__double_as_longlong(bu.re) ^ sg);
          const double bi = __longlong_as_double(__double_as_longlong(bu.im) ^ sg);
          const double bss = __longlong_as_double(__double_as_longlong(bs) ^ sg);
          dmma(p1[i][0], p1[i][1], m.re, br);
          dmma(p2[i][0], p2[i][1], m.im, bi);
          dmma(p3[i][0], p3[i][1], m.re + m.im, bss);
        }
      }
    }
    const ModeCols mc = mode_cols(qm, qx, ex, ey);
    const int ncol = mc.nmir * nrhs;
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int rt = warp + i * kMmaWarps;
      if (rt >= ntiles) continue;
      const int plane = tile_row(rt);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 2 * fc + h;
        if (col < ncol) {
          const int mi = nrhs == 2 ? col >> 1 : col, r = nrhs == 2 ? col & 1 : 0;
          const cplx v = {p1[i][h] - p2[i][h], p3[i][h] - p1[i][h] - p2[i][h]};
          S[(static_cast<size_t>(r) * E + mc.mode[mi]) * np + plane] = v;
        }
      }
    }
    // stages of mode j fully consumed (their reads are done: values are in
    // registers) before the next iterations refill them. The buffers are only
    // ever read through the generic proxy, so no proxy fence is needed here
    // (one after the initial zero fill suffices).
    __syncthreads();
  }
}

void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

}  // namespace

// ------------------------------------------------------------------ host --
void transform_blocks(Operator& op, const cplx* d_blocks, cudaStream_t st) {
  lateral_spectra(op, d_blocks, st);
}

void apply_b(const Operator& op, const cplx* d_in, cplx* d_out, int nrhs, const System* sys,
             cudaStream_t st) {
  const int np = 3 * op.nz;
  const long long rows = static_cast<long long>(nrhs) * np * op.ny;
  cplx* T = scratch<cplx>(static_cast<size_t>(rows) * op.ex, st);
  cplx* S = scratch<cplx>(static_cast<size_t>(nrhs) * op.lateral() * np, st);
  lateral_forward(op, d_in, sys ? sys->r2 : nullptr, T, S, nrhs, st);
  // K_ct: up to two right-hand sides per launch (8 columns of a full mode)
  profile_mark(2, true, st);
  {
    int sms = 0, dev = 0;
    EMIE_CUDA(cudaGetDevice(&dev));
    EMIE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int nmodes = static_cast<int>(op.modes());
    for (int r0 = 0; r0 < nrhs; r0 += 2) {
      const int g = std::min(2, nrhs - r0);
      cplx* Sg = S + static_cast<size_t>(r0) * op.lateral() * np;
      const bool mma = op.mma;
      if (mma) {
        const size_t smem = 128 + 3 * static_cast<size_t>(op.nentD) * sizeof(cplx) +
                            2 * 8 * static_cast<size_t>(np + 4) * sizeof(cplx);
        const int grid = std::max(1, std::min(sms, nmodes));
        const void* fn = op.nz == 8 ? reinterpret_cast<const void*>(contract_mma_kernel<8>)
                       : op.nz == 16 ? reinterpret_cast<const void*>(contract_mma_kernel<16>)
                                     : reinterpret_cast<const void*>(contract_mma_kernel<32>);
        set_smem(fn, smem);
        if (op.nz == 8)
          contract_mma_kernel<8><<<grid, kMmaWarps * 32, smem, st>>>(op.spec, op.ctab, Sg, op.ex, op.ey, op.qx, nmodes, g, op.nentD);
        else if (op.nz == 16)
          contract_mma_kernel<16><<<grid, kMmaWarps * 32, smem, st>>>(op.spec, op.ctab, Sg, op.ex, op.ey, op.qx, nmodes, g, op.nentD);
        else
          contract_mma_kernel<32><<<grid, kMmaWarps * 32, smem, st>>>(op.spec, op.ctab, Sg, op.ex, op.ey, op.qx, nmodes, g, op.nentD);
        check_launch("contract_mma_kernel");
        continue;
      }
      const int CB = g == 2 ? 8 : 4;
      // two input buffers per warp; as many warps as 220 KB of SMEM holds
      const size_t per_warp = 16 + 2 * static_cast<size_t>(CB) * np * sizeof(cplx);
      const int wpb = static_cast<int>(std::max<size_t>(1, std::min<size_t>(kCtWarps, (220u << 10) / per_warp)));
      const size_t smem = per_warp * wpb;
      const int grid = std::max(1, std::min(sms, ceil_div(nmodes, wpb)));
      if (CB == 8) {
        set_smem(reinterpret_cast<const void*>(contract_kernel<8>), smem);
        contract_kernel<8><<<grid, wpb * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD, op.ex,
                                                         op.ey, op.qx, nmodes, g);
      } else {
        set_smem(reinterpret_cast<const void*>(contract_kernel<4>), smem);
        contract_kernel<4><<<grid, wpb * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD, op.ex,
                                                         op.ey, op.qx, nmodes, g);
      }
      check_launch("contract_kernel");
    }
  }
  profile_mark(2, false, st);
  lateral_inverse(op, S, T, d_in, d_out, sys ? sys->s : nullptr, sys ? sys->r1 : nullptr, nrhs,
                  st);
  release(S, st);
  release(T, st);
}

}  // namespace emie_cu
