// Spectral operator build (transform_operator) and the CIE operator apply
// (apply(SpectralOperator), apply(SystemOperator)) for sm_100a.
//
// Reference: src/toeplitz.cpp:92-161 (spectra), 163-283 (apply),
//            src/cie.cpp:56-73 (system apply).
//
// The lateral FFT stages live in lateral.cu. Apply data flow for nrhs fields (all complex128):
//   u [r][plane][iy][ix]            plane = c*nz + iz (GridVector layout)
//   K_fx : r2-scale, zero-pad, x-FFT        -> T [r][mx][plane][iy]
//   K_fy : zero-pad, y-FFT, transpose       -> S [r][mx][my][plane]  (mode-major)
//   K_ct : per quadrant (or octant) mode, 3nz x 3nz block times its mirror
//          modes x nrhs (and the transposed mode's) -> S (in place):
//          contract_mma_kernel (nz 8/16/32: whole block by TMA, DMMA),
//          contract_rows_kernel (nz 48/64: row blocks streamed as K-chunks, DMMA),
//          contract_kernel (other nz: wrapped diagonals, DFMA)
//   K_iy : inverse y-FFT, keep iy < ny       -> T
//   K_ix : inverse x-FFT, keep ix < nx, 1/(ex ey), s*u + r1*(.) epilogue -> out
// The mode-major spectrum makes every contraction read/write a contiguous
// 3nz run per (mode, rhs); the transposes ride inside the FFT kernels' SMEM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <type_traits>

#include "operator.cuh"
#include "tma.cuh"

#ifndef EMIE_CT_EXPERIMENT
#define EMIE_CT_EXPERIMENT 0  // 1: no MMAs, 2: no copies (timing experiments only)
#endif

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

// octv != nullptr (operator.xysym): work items are the codes 2 qm + sw of the
// octant modes qm; sw = 1 applies qm's block to the transposed mode's columns
// with their x and y thirds exchanged (the two halves of an item are adjacent
// in the list, so they run on neighbouring warp groups of one CTA and share
// the block through L1/L2: HBM reads the octant blocks once)
template <int CB>
__global__ void __launch_bounds__(kCtWarps * 32, 1)
    contract_kernel(const cplx* __restrict__ op, cplx* S, int nz, int nsd, int nentD, int ex,
                    int ey, int qx, int q0, int q1, int qbase, int nrhs, int pair,
                    const int* __restrict__ octv, int noctv) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = 3 * nz;
  const size_t colbytes = static_cast<size_t>(np) * sizeof(cplx);
  // pair = 1 (nz > 32): a warp pair shares a mode and its input buffers, each
  // warp one 32-row half; the pair walks the diagonals in the same order, so
  // the transposed reads of a diagonal (t and nz - t, adjacent in the walk)
  // hit L1 instead of coming back from L2/HBM a whole pass later.
  const int group = pair ? warp >> 1 : warp, role = pair ? warp & 1 : 0;
  const int ngroups = (blockDim.x >> 5) >> pair;
  // per group: mbarriers[2] then two buffers of CB columns
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw) + 2 * group;
  cplx* ubase = reinterpret_cast<cplx*>(smraw + 16 * ngroups) + static_cast<size_t>(group) * 2 * CB * np;
  const size_t E = static_cast<size_t>(ex) * ey;
  const int gw = blockIdx.x * ngroups + group, nw = gridDim.x * ngroups;
  if (lane == 0 && role == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (role == 0)
    for (int i = lane; i < 2 * CB * np; i += 32) ubase[i] = cplx{0.0, 0.0};
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  auto group_sync = [&]() {
    if (pair) asm volatile("bar.sync %0, 64;" ::"r"(1 + group) : "memory");
    else __syncwarp();
  };
  // work item v -> (block mode, column mode, swap)
  auto item = [&](int v, int& qb, int& qc, bool& sw) {
    if (octv) {
      const int code = __ldg(octv + v);
      qb = code >> 1;
      sw = code & 1;
      const int qy_ = qb / qx, qx_ = qb - qy_ * qx;
      qc = sw ? qx_ * qx + qy_ : qb;
    } else {
      qb = qc = q0 + v;
      sw = false;
    }
  };
  const int nwork = octv ? noctv : q1 - q0;
  auto issue = [&](int v, int buf) {
    if (lane == 0 && role == 0) {
      int qb, qm;
      bool sw;
      item(v, qb, qm, sw);
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
  if (gw < nwork) issue(gw, 0);
  int it = 0;
  for (int v = gw; v < nwork; v += nw, ++it) {
    const int buf = it & 1;
    if (v + nw < nwork) issue(v + nw, buf ^ 1);
    mbar_wait(mbar + buf, phase[buf]);
    phase[buf] ^= 1u;
    const cplx* U = ubase + static_cast<size_t>(buf) * CB * np;
    int qb, qm;
    bool sw;
    item(v, qb, qm, sw);
    // transposed-mode columns: x and y thirds exchanged on load and store
    const int ox = sw ? nz : 0, oy = sw ? 0 : nz;
    const ModeCols mc = mode_cols(qm, qx, ex, ey);
    const int ncol = mc.nmir * nrhs;
    const cplx* blk = op + static_cast<size_t>(qb - qbase) * nentD;
    const int ntri = nz * (nz + 1) / 2;
    const cplx* Dxx = blk;
    const cplx* Dyy = blk + ntri;
    const cplx* Dzz = blk + 2 * ntri;
    const cplx* Dxy = blk + 3 * ntri;
    const cplx* Dxz = blk + 4 * ntri;
    const cplx* Dyz = Dxz + nz * nz;
    for (int kb = pair ? 32 * role : 0; kb < nz; kb += pair ? nz : 32) {
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
        for (int c = 0; c < CB; ++c) u[c] = U[c * np + ox + kp];
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ax[c], cur.xx, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(ay[c], cur.xy, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) cmac(az[c], mxzt, u[c]);
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = U[c * np + oy + kp];
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
            o[ox + k] = ax[c];
            o[oy + k] = ay[c];
            o[2 * nz + k] = az[c];
          }
        }
      }
    }
    // this buffer is refilled (async proxy) after the next iteration's wait
    group_sync();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
}

// ------------------------------------------- contraction on FP64 MMA -----
// Same product as contract_kernel, on the FP64 tensor cores (DMMA.8x8x4 via
// mma.sync.m8n8k4.f64): measured 37 TF/s at 4 warps/SM on B200, where DFMA
// needs ~32 warps to approach it. Used for nz in {8, 16, 32} with the MMA
// operator layout (operator.cuh).
// One CTA per SM, persistent over quadrant modes, warp-specialised:
//  - 3nz/8 consumer warps, one 8-row output tile each (component a, rows
//    {4m..4m+3} u {4m+nz/2..4m+nz/2+3}); for nz = 32 that is 12 warps, three
//    per SMSP, so every SMSP's DMMA pipe has three independent tiles;
//  - one producer warp whose elected lane brings each mode's coefficient
//    block (one TMA bulk copy of nentD complex) and its input columns (one
//    bulk copy per (mirror, rhs), column stride np + 4) into stage buffers
//    guarded by full (tx-count) and empty (one arrive per consumer warp)
//    mbarriers, so no CTA-wide barrier sits between modes.
// The 8 columns (<= 4 mirrors x 2 rhs) are the MMA's N; K runs over
// (component b, kp) in steps of 4. Complex products use three real MMAs
// (P1 = Ar Br, P2 = Ai Bi, P3 = (Ar+Ai)(Br+Bi); re = P1 - P2, im = P3 - P1 - P2).
// The zx / zy blocks (-xz^T, -yz^T) flip the sign bit of the B fragment.
constexpr long long kSwapColPeer = 1LL << 60;  // = kSwapCol (below)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- staged peer epilogue (sharded apply): a mode's output columns are
// assembled in its input-column stage -- free once every consumer warp has
// finished the mode's MMAs -- in owner-major order (owner h's rows of the
// three components, 3 (z[h+1] - z[h]) values, contiguous), then each
// (column, owner) segment goes to the owner's spectrum in one bulk copy
// shared -> global over NVLink instead of a 16-byte store per lane.
__device__ __forceinline__ void consumers_sync(int nthreads) {  // named barrier 1: the consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// the owner of output row k: index h, first row z[h], rows pnz
__device__ __forceinline__ void peer_owner(const PeerOut& po, int k, int& h, int& zh, int& pnz) {
  h = 0;
  while (h + 1 < po.G && k >= po.z[h + 1]) ++h;
  zh = po.z[h];
  pnz = po.z[h + 1] - zh;
}
// issue the staged columns of one mode (lane c < NC of one consumer warp: its
// column's owner segments); with a stage shared with the input columns, wait
// until the copies have read it (the producer refills it next), else the wait
// comes before the stage's next use
template <int NC, int np, int ldu>
__device__ __forceinline__ void peer_push(const PeerOut& po, const long long* colbase, const cplx* stage, int lane,
                                          bool wait_read) {
  if (lane < NC) {
    const long long cb = colbase[lane];
    if (cb >= 0) {
      const long long col = (cb & ~kSwapColPeer) / np;  // r E + mode
      const cplx* src = stage + static_cast<size_t>(lane) * ldu;
      for (int h = 0; h < po.G; ++h) {
        const int zh = po.z[h], pnz = po.z[h + 1] - zh;
        if (pnz > 0)
          bulk_s2g(po.dst[h] + col * 3 * pnz, src + 3 * zh, static_cast<uint32_t>(3 * pnz * sizeof(cplx)));
      }
      bulk_commit();
      if (wait_read) bulk_wait_read_all();
    }
  }
}

// mirror mi (0 .. nmir-1) of quadrant mode qm, in mode_cols order
__device__ __forceinline__ int mirror_mode(int qm, int mi, int qx, int ex, int ey) {
  const int qmy = qm / qx, qmx = qm - qmy * qx;
  const bool mx_ok = qmx > 0 && (ex - qmx) > ex / 2;
  const int mx = (mi == 3 || (mi == 1 && mx_ok)) ? ex - qmx : qmx;
  const int my = (mi >= 2 || (mi == 1 && !mx_ok)) ? ey - qmy : qmy;
  return mx * ey + my;
}
__device__ __forceinline__ int mirror_count(int qm, int qx, int ex, int ey) {
  const int qmy = qm / qx, qmx = qm - qmy * qx;
  const int a = (qmx > 0 && (ex - qmx) > ex / 2) ? 1 : 0;
  const int b = (qmy > 0 && (ey - qmy) > ey / 2) ? 1 : 0;
  return (1 + a) * (1 + b);
}

template <int NZ>
constexpr int mma_warps() { return 3 * NZ / 8; }
constexpr int kBlkStages = 3, kUStages = 2;
#ifndef EMIE_CT_OCT_BST
#define EMIE_CT_OCT_BST 2
#endif
constexpr int kBlkStagesOct = EMIE_CT_OCT_BST;  // 16-column stages leave SMEM for two blocks
#ifndef EMIE_CT_L2AHEAD
#define EMIE_CT_L2AHEAD 0
#endif
constexpr int kL2Ahead = EMIE_CT_L2AHEAD;  // modes past the SMEM stages prefetched to L2
// column-table flag: the column belongs to the transposed mode (x <-> y exchanged)
constexpr long long kSwapCol = kSwapColPeer;

template <bool OCT>
constexpr int ct_cols() { return OCT ? 16 : 8; }
template <bool OCT>
constexpr int ct_blk_stages() { return OCT ? kBlkStagesOct : kBlkStages; }

// OCT (operator.xysym): work item t is octant mode octl[t] = (qmy, qmx) with
// qmx <= qmy. Columns 0-7 are its own (mirror, rhs) columns; columns 8-15 are
// those of the transposed mode (qmx, qmy), read with their x and y thirds
// exchanged and stored back exchanged: M(qmx, qmy) = P M(qmy, qmx) P with P
// the x <-> y permutation, so one block read serves both modes and the MMA's
// A fragment feeds two n8 products.
// PEER (sharded apply): the results go to the slab owners' spectra through po
// (peer memory over NVLink) instead of back into S; with OCT the rank's octant
// items are its rows of the octant (Operator::shard_octant)
template <int NZ, bool OCT, bool PEER = false>
__global__ void __launch_bounds__((mma_warps<NZ>() + 1) * 32, 1)
    contract_mma_kernel(const cplx* __restrict__ op, const uint32_t* __restrict__ ctab, cplx* S,
                        int ex, int ey, int qx, int q0, int q1, int qbase, int nrhs, int nentD,
                        const int* __restrict__ octl, int noct, const __grid_constant__ PeerOut po) {
  pdl_trigger();
  constexpr int np = 3 * NZ, ldu = np + 4;
  constexpr int nk = np / 4;
  constexpr int W = mma_warps<NZ>();
  constexpr int NC = ct_cols<OCT>(), BST = ct_blk_stages<OCT>();
  extern __shared__ __align__(128) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* bempty = bfull + BST;
  uint64_t* ufull = bempty + BST;
  uint64_t* uempty = ufull + kUStages;
  // per input stage: output offsets (r*E + mode)*np of its NC columns (-1: none)
  long long* colbase = reinterpret_cast<long long*>(smraw + 128);
  cplx* blkbuf = reinterpret_cast<cplx*>(smraw + 128 + kUStages * NC * sizeof(long long));
  cplx* ubuf = blkbuf + BST * nentD;
  const size_t E = static_cast<size_t>(ex) * ey;
  constexpr uint32_t colbytes = np * sizeof(cplx);
  if (threadIdx.x == 0) {
    for (int i = 0; i < BST; ++i) {
      mbar_init(bfull + i, 1);
      mbar_init(bempty + i, W);
    }
    for (int i = 0; i < kUStages; ++i) {
      mbar_init(ufull + i, 1);
      mbar_init(uempty + i, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // columns past a mode's ncol are multiplied but never stored: keep them finite
  for (int i = threadIdx.x; i < kUStages * NC * ldu; i += blockDim.x) ubuf[i] = cplx{0.0, 0.0};
  // every writing thread orders its generic zero stores before the producer's
  // later TMA writes into ubuf (write, fence, barrier, then bulk copy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  pdl_wait();  // the spectra S of the y pass are complete
  const int G = gridDim.x;
  const int nwork = OCT ? noct : q1 - q0;

  if (warp == W) {  // ---- producer warp: lane c issues column c's copy
    int j = 0;
    for (int t = blockIdx.x; t < nwork; t += G, ++j) {
      const int qm = OCT ? __ldg(octl + t) : q0 + t;
      const int bs = j % BST, us = j % kUStages;
      if (j >= BST) mbar_wait(bempty + bs, static_cast<uint32_t>((j / BST - 1) & 1));
      const uint32_t blkbytes = nentD * sizeof(cplx);
      if (lane == 0) {
        // blocks of the modes after the SMEM stages go to L2 ahead of their copy
        for (int d = (j == 0 ? BST : kL2Ahead); !OCT && kL2Ahead > 0 && d <= kL2Ahead; ++d) {
          const int qp = qm + d * G;
          if (qp < q1) bulk_prefetch_l2(op + static_cast<size_t>(qp - qbase) * nentD, blkbytes);
        }
#if EMIE_CT_EXPERIMENT == 2
        mbar_expect_tx(bfull + bs, 0);
#else
        mbar_expect_tx(bfull + bs, blkbytes);
        bulk_g2s(blkbuf + bs * nentD, op + static_cast<size_t>(qm - qbase) * nentD, blkbytes, bfull + bs);
#endif
      }
      if (j >= kUStages) mbar_wait(uempty + us, static_cast<uint32_t>((j / kUStages - 1) & 1));
      const int ncol = mirror_count(qm, qx, ex, ey) * nrhs;
      const int qmy = qm / qx, qmx = qm - qmy * qx;
      const int ncol2 = OCT && qmx != qmy ? ncol : 0;
      // slot `lane`: column (mirror, rhs) of the mode, then those of the
      // transposed mode (qmx, qmy) (same mirror count: ex == ey) -- packed
      // behind them when both fit one n8 group (nrhs = 1), else in slots 8-15
      const int t0 = ncol + ncol2 <= 8 ? ncol : 8;
      const bool tr = OCT && lane >= t0 && lane < t0 + ncol2;
      const int c = tr ? lane - t0 : lane;
      const int mi = c / nrhs, r = c - mi * nrhs;
      long long base = -1LL;
      if (lane < ncol)
        base = (static_cast<long long>(r) * E + mirror_mode(qm, mi, qx, ex, ey)) * np;
      else if (tr)
        base = (static_cast<long long>(r) * E + mirror_mode(qmx * qx + qmy, mi, qx, ex, ey)) * np;
      if (lane < NC) colbase[us * NC + lane] = base < 0 ? -1LL : (tr ? base | kSwapCol : base);
      __syncwarp();
      // the column table is published by this arrive (release); the copies
      // complete on it only after it set the expected bytes
      if (lane == 0) mbar_expect_tx(ufull + us, EMIE_CT_EXPERIMENT == 2 ? 0u : (ncol + ncol2) * colbytes);
      __syncwarp();
#if EMIE_CT_EXPERIMENT != 2
      if (base >= 0) bulk_g2s(ubuf + (us * NC + lane) * ldu, S + base, colbytes, ufull + us);
#endif
    }
    return;
  }

  // ---- consumers. Fragment coordinates: A row fr / k fc; B k fc / col fr;
  // C row fr, cols 2fc..2fc+1. Row fr of the tile -> 4m + fr/2 + (fr&1) nz/2:
  // each quarter-warp reads rows r and r + nz/2, which the MMA layout puts in
  // disjoint banks (operator.cuh).
  const int fr = lane >> 2, fc = lane & 3;
  const int a_rt = warp / (NZ / 8), m = warp - a_rt * (NZ / 8);
  const int k = 4 * m + (fr >> 1) + (fr & 1) * (NZ / 2);
  // PEER: the slab owner of this lane's output row k
  int pzh = 0, pnz = 0;
  if constexpr (PEER) {
    int h;
    peer_owner(po, k, h, pzh, pnz);
  }
  // The warp's component a is a template constant inside consume(): the
  // zx / zy negation (-xz^T, -yz^T: the z tile, b < 2) is then a compile-time
  // operand sign that the DMMA applies for free.
  auto consume = [&](auto AC) {
    constexpr int a = decltype(AC)::value;
    const int plane = a * NZ + k;
    const int plane_sw = (a == 2 ? 2 : 1 - a) * NZ + k;  // row of a transposed-mode column
    // per-lane coefficient offsets of every k step: mode independent
    uint32_t off[nk];
#pragma unroll
    for (int ks = 0; ks < nk; ++ks) {
      const int b = (4 * ks) / NZ, kp = 4 * ks - b * NZ + fc;
      off[ks] = __ldg(ctab + ((a * 3 + b) * NZ + k) * NZ + kp) & 0x7fffffffu;
    }
    // NG n8 column groups share every A fragment; group 1 (transposed-mode
    // columns) reads k step ks of third b from third (x <-> y)(b)
    auto run = [&](auto NGC, const cplx* blk, const cplx* U, int bs, int us) {
      constexpr int NG = decltype(NGC)::value;
      auto kswap = [](int ks) {
        constexpr int q = NZ / 4;  // k steps per third
        return ks < q ? ks + q : ks < 2 * q ? ks - q : ks;
      };
      // one group: this lane's B column may be a packed transposed-mode column
      long long cbl = 0;
      if (OCT && NG == 1) cbl = colbase[us * NC + fr];
      const bool swp = OCT && NG == 1 && cbl >= 0 && (cbl & kSwapCol);
      auto kof = [&](int g, int ks) { return (g == 1 || swp) ? kswap(ks) : ks; };
      double p1[NG][2], p2[NG][2], p3[NG][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) p1[g][0] = p1[g][1] = p2[g][0] = p2[g][1] = p3[g][0] = p3[g][1] = 0.0;
      // operands PD k-steps ahead of their MMAs (SMEM latency off the DMMA chain)
#ifndef EMIE_CT_PD
#define EMIE_CT_PD 6
#endif
      constexpr int PD = EMIE_CT_PD;
      cplx av[PD], bv[PD][NG];
#pragma unroll
      for (int ks = 0; ks < PD; ++ks) {
        av[ks] = blk[off[ks]];
#pragma unroll
        for (int g = 0; g < NG; ++g) bv[ks][g] = U[g * 8 * ldu + 4 * kof(g, ks)];
      }
#pragma unroll
      for (int ks = 0; ks < (EMIE_CT_EXPERIMENT == 1 ? 0 : nk); ++ks) {
        const cplx mv = av[ks % PD];
        cplx bu[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) bu[g] = bv[ks % PD][g];  // B[k = fc][col = fr]
        if (ks + PD < nk) {
          av[ks % PD] = blk[off[ks + PD]];
#pragma unroll
          for (int g = 0; g < NG; ++g) bv[ks % PD][g] = U[g * 8 * ldu + 4 * kof(g, ks + PD)];
        }
        constexpr bool kz = a == 2;
        const bool neg = kz && (4 * ks) / NZ < 2;  // compile time after unrolling
        const double ms = mv.re + mv.im;
        double bs[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) bs[g] = bu[g].re + bu[g].im;
        // products sharing an A operand back to back
#pragma unroll
        for (int g = 0; g < NG; ++g) dmma(p1[g][0], p1[g][1], mv.re, neg ? -bu[g].re : bu[g].re);
#pragma unroll
        for (int g = 0; g < NG; ++g) dmma(p2[g][0], p2[g][1], mv.im, neg ? -bu[g].im : bu[g].im);
#pragma unroll
        for (int g = 0; g < NG; ++g) dmma(p3[g][0], p3[g][1], ms, neg ? -bs[g] : bs[g]);
      }
      // block stage reads are complete (the DMMAs consumed them): release it
      // (the proxy fence orders these generic reads before the TMA refill)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(bempty + bs);
      if (PEER && po.G == 1) {
        // one rank: the owner is this rank's own spectrum; 16-byte stores
        // (staging only costs barriers here: 4,038 vs 3,694 applies/s)
        constexpr int asw = a == 2 ? 2 : 1 - a;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long cb = colbase[us * NC + 8 * g + 2 * fc + h];
            if (cb >= 0) {
              const int ap = (OCT && (cb & kSwapCol)) ? asw : a;
              po.dst[0][((cb & ~kSwapCol) / np) * np + ap * NZ + k] =
                  cplx{p1[g][h] - p2[g][h], p3[g][h] - p1[g][h] - p2[g][h]};
            }
          }
      } else if constexpr (PEER) {
        // several owners: the mode's outputs staged in SMEM (barrier: every
        // consumer warp has finished the mode), then one bulk copy per
        // (column, owner) over NVLink instead of a 16-byte store per lane; a
        // transposed-mode column's row goes to the exchanged third.
        // own stage (po.sep): the previous mode's copies must have read it
        cplx* stage = ubuf + static_cast<size_t>(po.sep ? kUStages : us) * NC * ldu;
        if (po.sep && warp == 0) bulk_wait_read_all();
        consumers_sync(W * 32);
        constexpr int asw = a == 2 ? 2 : 1 - a;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = 8 * g + 2 * fc + h;
            const long long cb = colbase[us * NC + c];
            if (cb >= 0) {
              const int ap = (OCT && (cb & kSwapCol)) ? asw : a;
              stage[c * ldu + 3 * pzh + ap * pnz + (k - pzh)] =
                  cplx{p1[g][h] - p2[g][h], p3[g][h] - p1[g][h] - p2[g][h]};
            }
          }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before the bulk reads
        consumers_sync(W * 32);
        if (warp == 0) peer_push<NC, np, ldu>(po, colbase + us * NC, stage, lane, !po.sep);
      } else {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long cb = colbase[us * NC + 8 * g + 2 * fc + h];
            if (cb >= 0) {
              const cplx v = cplx{p1[g][h] - p2[g][h], p3[g][h] - p1[g][h] - p2[g][h]};
              const long long o = (cb & ~kSwapCol) + ((cb & kSwapCol) ? plane_sw : plane);
              S[o] = v;
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(uempty + us);  // input columns and their table
    };
    int j = 0;
    for (int t = blockIdx.x; t < nwork; t += G, ++j) {
      const int bs = j % BST, us = j % kUStages;
      mbar_wait(bfull + bs, static_cast<uint32_t>((j / BST) & 1));
      mbar_wait(ufull + us, static_cast<uint32_t>((j / kUStages) & 1));
      const cplx* blk = blkbuf + bs * nentD;
      const cplx* U = ubuf + us * NC * ldu + fr * ldu + fc;
      if (OCT && colbase[us * NC + 8] >= 0) run(std::integral_constant<int, 2>{}, blk, U, bs, us);
      else run(std::integral_constant<int, 1>{}, blk, U, bs, us);  // (packed transposed columns: swp)
    }
  };
  if (a_rt == 0) consume(std::integral_constant<int, 0>{});
  else if (a_rt == 1) consume(std::integral_constant<int, 1>{});
  else consume(std::integral_constant<int, 2>{});
  if constexpr (PEER) {
    if (warp == 0) bulk_wait_all();  // the staged columns have landed in the owners' spectra
  }
}

// ------------------------------ contraction, streamed row blocks (nz 48/64) -----
// For nz in {48, 64} (config 4: nz = 64) a mode block no longer fits SMEM
// (265 KB even in triangle form at nz = 64), so the operator is stored as
// six dense row-major nz x nz blocks per mode, [xx yy zz xy xz yz] (the
// symmetric components hold both triangles), and the block streams through a
// ring of K-chunks like a GEMM main loop. Chunk (b, kc) = columns kp in
// [8kc, 8kc+8) of third b of M = [[xx xy xz] [xy yy yz] [-xz^T -yz^T zz]] for
// all 3nz rows: one tensor-map box per row third a -- a column slice of the
// stored block (8 columns x nz rows, 128-byte swizzle; M_ab = M_ba^T for the
// symmetric parts), or for -xz^T, -yz^T a row slice of xz / yz (8 rows x nz
// columns, unswizzled, read transposed by the consumers: 16-byte lanes along
// a row, so a warp's load still spans four 128-byte runs). The transposed
// copies xz^T, yz^T the layout once stored were 2 of 8 blocks of HBM traffic. 3nz/16 consumer warps own two
// 8-row output tiles each; the products, the 3-multiply complex form, the
// octant column groups and the output stores are those of contract_mma_kernel.
constexpr int kRowsRing = 4;  // K-chunk stages
template <int NZ>
constexpr int rows_warps() { return 3 * NZ / 16; }
__host__ __device__ constexpr int rows_block_id(int a, int b) {
  // M_ab -> stored block: xx yy zz xy xz yz = 0..5 (a = 2, b < 2: block 4 + b, transposed)
  return a == b ? a : (a < 2 && b < 2) ? 3 : b == 2 ? 4 + a : 4 + b;
}
__host__ __device__ constexpr bool rows_transposed(int a, int b) { return a == 2 && b < 2; }

template <int NZ, bool OCT, bool PEER = false>
__global__ void __launch_bounds__((rows_warps<NZ>() + 1) * 32, 1)
    contract_rows_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmT, cplx* S,
                         int ex, int ey, int qx, int q0, int q1,
                         int qbase, int nrhs, const int* __restrict__ octl, int noct,
                         const __grid_constant__ PeerOut po) {
  pdl_trigger();
  constexpr int np = 3 * NZ, ldu = np + 4;
  constexpr int W = rows_warps<NZ>();
  constexpr int NC = ct_cols<OCT>();
  constexpr int NT = NZ / 8;           // row tiles (and K-chunks) per third
  constexpr int NCH = 3 * NT;          // K-chunks per mode
  constexpr uint32_t kBox = NZ * 128;  // one box: nz rows x 8 complex
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* rempty = rfull + kRowsRing;
  uint64_t* ufull = rempty + kRowsRing;
  uint64_t* uempty = ufull + kUStages;
  long long* colbase = reinterpret_cast<long long*>(smraw + 128);
  unsigned char* ring = smraw + 1024;  // 1024-aligned boxes (swizzle atoms)
  cplx* ubuf = reinterpret_cast<cplx*>(ring + kRowsRing * 3 * kBox);
  const size_t E = static_cast<size_t>(ex) * ey;
  constexpr uint32_t colbytes = np * sizeof(cplx);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRowsRing; ++i) {
      mbar_init(rfull + i, 1);
      mbar_init(rempty + i, W);
    }
    for (int i = 0; i < kUStages; ++i) {
      mbar_init(ufull + i, 1);
      mbar_init(uempty + i, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kUStages * NC * ldu; i += blockDim.x) ubuf[i] = cplx{0.0, 0.0};
  // every writing thread orders its generic zero stores before the producer's
  // later TMA writes into ubuf (write, fence, barrier, then bulk copy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  pdl_wait();  // the spectra S of the y pass are complete
  const int G = gridDim.x;
  const int nwork = OCT ? noct : q1 - q0;

  if (warp == W) {  // ---- producer warp
    int j = 0;
    for (int t = blockIdx.x; t < nwork; t += G, ++j) {
      const int qm = OCT ? __ldg(octl + t) : q0 + t;
      const int us = j % kUStages;
      if (j >= kUStages) mbar_wait(uempty + us, static_cast<uint32_t>((j / kUStages - 1) & 1));
      const int ncol = mirror_count(qm, qx, ex, ey) * nrhs;
      const int qmy = qm / qx, qmx = qm - qmy * qx;
      const int ncol2 = OCT && qmx != qmy ? ncol : 0;
      const int t0 = ncol + ncol2 <= 8 ? ncol : 8;
      const bool tr = OCT && lane >= t0 && lane < t0 + ncol2;
      const int c = tr ? lane - t0 : lane;
      const int mi = c / nrhs, r = c - mi * nrhs;
      long long base = -1LL;
      if (lane < ncol)
        base = (static_cast<long long>(r) * E + mirror_mode(qm, mi, qx, ex, ey)) * np;
      else if (tr)
        base = (static_cast<long long>(r) * E + mirror_mode(qmx * qx + qmy, mi, qx, ex, ey)) * np;
      if (lane < NC) colbase[us * NC + lane] = base < 0 ? -1LL : (tr ? base | kSwapCol : base);
      __syncwarp();
      if (lane == 0) mbar_expect_tx(ufull + us, (ncol + ncol2) * colbytes);
      __syncwarp();
      if (base >= 0) bulk_g2s(ubuf + (us * NC + lane) * ldu, S + base, colbytes, ufull + us);
      // the block's K-chunks through the ring
      if (lane == 0) {
        const int mode = qm - qbase;
        for (int ch = 0; ch < NCH; ++ch) {
          const long long gc = static_cast<long long>(j) * NCH + ch;
          const int st = static_cast<int>(gc % kRowsRing);
          if (gc >= kRowsRing) mbar_wait(rempty + st, static_cast<uint32_t>((gc / kRowsRing - 1) & 1));
          const int b = ch / NT, kc = ch - b * NT;
          mbar_expect_tx(rfull + st, 3 * kBox);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (rows_transposed(a, b))  // rows 8kc.. of xz / yz, all columns
              tma_load_4d(ring + (st * 3 + a) * kBox, &tmT, 0, 8 * kc, rows_block_id(a, b), mode, rfull + st);
            else
              tma_load_4d(ring + (st * 3 + a) * kBox, &tm, 16 * kc, 0, rows_block_id(a, b), mode, rfull + st);
          }
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---- consumers: tiles warp and warp + W (row tile ti: third a = ti / NT, rows 8 (ti % NT) ..)
  const int fr = lane >> 2, fc = lane & 3;
  int ta[2], trow[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int ti = warp + i * W;
    ta[i] = ti / NT;
    trow[i] = (ti - ta[i] * NT) * 8 + fr;  // this lane's A row inside third ta[i]
  }
  auto run = [&](auto NGC, int us, long long gc0) {
    constexpr int NG = decltype(NGC)::value;
    const cplx* U = ubuf + us * NC * ldu + fr * ldu + fc;
    long long cbl = 0;
    if (OCT && NG == 1) cbl = colbase[us * NC + fr];
    const bool swp = OCT && NG == 1 && cbl >= 0 && (cbl & kSwapCol);
    double p1[2][NG][2], p2[2][NG][2], p3[2][NG][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int g = 0; g < NG; ++g) p1[i][g][0] = p1[i][g][1] = p2[i][g][0] = p2[i][g][1] = p3[i][g][0] = p3[i][g][1] = 0.0;
#pragma unroll 1
    for (int b = 0; b < 3; ++b) {
      const int bsw = b == 2 ? 2 : 1 - b;  // third of a transposed-mode column
#pragma unroll 1
      for (int kc = 0; kc < NT; ++kc) {
        const long long gc = gc0 + b * NT + kc;
        const int st = static_cast<int>(gc % kRowsRing);
        mbar_wait(rfull + st, static_cast<uint32_t>((gc / kRowsRing) & 1));
        const unsigned char* box = ring + st * 3 * kBox;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int col = 4 * ks + fc;  // complex column inside the chunk
          cplx bu[NG];
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            const int third = (g == 1 || swp) ? bsw : b;
            bu[g] = U[g * 8 * ldu + third * NZ + 8 * kc + 4 * ks];
          }
          double bsum[NG];
#pragma unroll
          for (int g = 0; g < NG; ++g) bsum[g] = bu[g].re + bu[g].im;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int row = trow[i];
            const bool neg = rows_transposed(ta[i], b);  // -xz^T, -yz^T: a transposed row-slice box
            const cplx mv = *reinterpret_cast<const cplx*>(
                box + ta[i] * kBox + (neg ? col * (NZ * 16) + row * 16 : row * 128 + ((col ^ (row & 7)) << 4)));
            const double sg = neg ? -1.0 : 1.0;
            const double ar = sg * mv.re, ai = sg * mv.im;
            const double as = ar + ai;
#pragma unroll
            for (int g = 0; g < NG; ++g) dmma(p1[i][g][0], p1[i][g][1], ar, bu[g].re);
#pragma unroll
            for (int g = 0; g < NG; ++g) dmma(p2[i][g][0], p2[i][g][1], ai, bu[g].im);
#pragma unroll
            for (int g = 0; g < NG; ++g) dmma(p3[i][g][0], p3[i][g][1], as, bsum[g]);
          }
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA refill
        __syncwarp();
        if (lane == 0) mbar_arrive(rempty + st);
      }
    }
    // PEER: the input-column stage us becomes the output stage once every
    // consumer warp has finished its K-chunks (barrier); rows in owner-major
    // order, one bulk copy per (column, owner) (peer_push)
    cplx* stage = ubuf + static_cast<size_t>(us) * NC * ldu;
    const bool staged = PEER && po.G > 1;  // one rank: direct 16-byte stores into its own spectrum
    if (staged) consumers_sync(W * 32);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int a = ta[i];
      const int rowc = trow[i];  // C row fr of the tile = the lane's A row
      const int plane = a * NZ + rowc;
      const int asw = a == 2 ? 2 : 1 - a;
      int pzh = 0, pnz = 0;  // PEER: the slab owner of output row rowc
      if constexpr (PEER) {
        int hh;
        peer_owner(po, rowc, hh, pzh, pnz);
      }
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 8 * g + 2 * fc + h;
          const long long cb = colbase[us * NC + c];
          if (cb >= 0) {
            const cplx v = cplx{p1[i][g][h] - p2[i][g][h], p3[i][g][h] - p1[i][g][h] - p2[i][g][h]};
            if constexpr (PEER) {
              // a transposed-mode column's row goes to the exchanged third
              const int ap = (OCT && (cb & kSwapCol)) ? asw : a;
              if (staged) stage[c * ldu + 3 * pzh + ap * pnz + (rowc - pzh)] = v;
              else po.dst[0][((cb & ~kSwapCol) / np) * np + ap * NZ + rowc] = v;
            } else {
              const long long o = (cb & ~kSwapCol) + ((cb & kSwapCol) ? asw * NZ + rowc : plane);
              S[o] = v;
            }
          }
        }
    }
    if (staged) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before the bulk reads
      consumers_sync(W * 32);
      if (warp == 0) peer_push<NC, np, ldu>(po, colbase + us * NC, stage, lane, true);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(uempty + us);
  };
  int j = 0;
  for (int t = blockIdx.x; t < nwork; t += G, ++j) {
    const int us = j % kUStages;
    mbar_wait(ufull + us, static_cast<uint32_t>((j / kUStages) & 1));
    const long long gc0 = static_cast<long long>(j) * NCH;
    if (OCT && colbase[us * NC + 8] >= 0) run(std::integral_constant<int, 2>{}, us, gc0);
    else run(std::integral_constant<int, 1>{}, us, gc0);
  }
  if constexpr (PEER) {
    if (warp == 0) bulk_wait_all();  // the staged columns have landed in the owners' spectra
  }
}

// exact x <-> y symmetry of the compressed blocks (the property the octant
// contraction relies on): block(oj, oi) == block(oi, oj) with xx <-> yy and
// xz <-> yz, bit for bit, for every offset pair including oi == oj
__global__ void xy_symmetry_kernel(const cplx* __restrict__ blocks, int nx, int ntri, int nfull, int nent,
                                   int* bad) {
  const long long total = static_cast<long long>(nx) * nx * nent;
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int off = static_cast<int>(x / nent), e = static_cast<int>(x - static_cast<long long>(off) * nent);
    const int oi = off / nx, oj = off - oi * nx;
    int d = e;
    if (e < ntri) d = e + ntri;
    else if (e < 2 * ntri) d = e - ntri;
    else if (e >= 4 * ntri && e < 4 * ntri + nfull) d = e + nfull;
    else if (e >= 4 * ntri + nfull) d = e - nfull;
    const cplx u = blocks[x], v = blocks[(static_cast<size_t>(oj) * nx + oi) * nent + d];
    if (__double_as_longlong(u.re) != __double_as_longlong(v.re) ||
        __double_as_longlong(u.im) != __double_as_longlong(v.im))
      *bad = 1;
  }
}

void set_smem(const void* fn, size_t bytes) {
  EMIE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
}

}  // namespace

// ------------------------------------------------------------------ host --
void transform_blocks(Operator& op, const cplx* d_blocks, cudaStream_t st, int sym_known) {
  lateral_spectra(op, d_blocks, st);
  bool sym = false;
  // whole rows of quadrant modes (a full operator or a row-aligned mode shard):
  // the octant lists cover them (set_octant_lists)
  const bool rows = op.qx > 0 && op.qcount > 0 && op.qbase % op.qx == 0 && op.qcount % op.qx == 0;
  if (rows && op.nx == op.ny && op.ex == op.ey && sym_known != 0) {
    sym = true;
    if (sym_known < 0) {
      int* bad = scratch<int>(1, st);
      EMIE_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
      const long long total = static_cast<long long>(op.nx) * op.nx * op.nent;
      xy_symmetry_kernel<<<static_cast<int>(std::min<long long>(ceil_div(total, 256), 8 * sm_count())), 256, 0,
                           st>>>(d_blocks, op.nx, op.ntri, op.nfull, op.nent, bad);
      check_launch("xy_symmetry_kernel");
      int h = 1;
      EMIE_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
      EMIE_CUDA(cudaStreamSynchronize(st));
      release(bad, st);
      sym = h == 0;
    }
  }
  op.xysym = sym;
  set_octant_lists(op, st);
}

// The octant work lists of op's stored rows (qbase and qcount whole rows of
// qx quadrant modes; every row of a full operator): octant modes qmx <= qmy
// with qmy in those rows -- off-diagonal (two modes per block) first, the
// diagonal (one mode) last, so the lighter items fill the tail -- then the
// DFMA contraction's item codes. None unless op.xysym.
void set_octant_lists(Operator& op, cudaStream_t st) {
  cudaFree(op.octl);
  op.octl = nullptr;
  op.noct = op.noctv = 0;
  if (!op.xysym || op.qx == 0 || op.qbase % op.qx != 0 || op.qcount % op.qx != 0 || op.qcount == 0) {
    op.xysym = false;
    return;
  }
  const int y0 = op.qbase / op.qx, y1 = (op.qbase + op.qcount) / op.qx;
  std::vector<int> l;
  for (int qmy = y0; qmy < y1; ++qmy)
    for (int qmx = 0; qmx < qmy; ++qmx) l.push_back(qmy * op.qx + qmx);
  for (int q = y0; q < y1; ++q) l.push_back(q * op.qx + q);
  // the DFMA contraction's items: 2 qm (+ 2 qm + 1 for the transposed mode)
  std::vector<int> v;
  for (int qm : l) {
    v.push_back(2 * qm);
    if (qm / op.qx != qm % op.qx) v.push_back(2 * qm + 1);
  }
  EMIE_CUDA(cudaMalloc(&op.octl, (l.size() + v.size()) * sizeof(int)));
  EMIE_CUDA(cudaMemcpyAsync(op.octl, l.data(), l.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(op.octl + l.size(), v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  op.noct = static_cast<int>(l.size());
  op.noctv = static_cast<int>(v.size());
}

// the ROWS layout's stored modes as {2nz doubles, nz rows, 6 blocks, modes}:
// column-slice boxes (8 complex x nz rows, 128-byte swizzle) and row-slice
// boxes (nz complex x 8 rows, unswizzled) for the transposed thirds
static void rows_tensor_maps(const Operator& op, CUtensorMap* tm, CUtensorMap* tmT) {
  const uint64_t dims[4] = {2ull * op.nz, static_cast<uint64_t>(op.nz), static_cast<uint64_t>(kRowsBlocks),
                            static_cast<uint64_t>(op.qcount)};
  const uint64_t strides[3] = {static_cast<uint64_t>(op.nz) * 16, static_cast<uint64_t>(op.nz) * op.nz * 16,
                               static_cast<uint64_t>(kRowsBlocks) * op.nz * op.nz * 16};
  const uint32_t box[4] = {16, static_cast<uint32_t>(op.nz), 1, 1};
  encode_tensor_map_f64(tm, op.spec, 4, dims, strides, box);
  const uint32_t boxT[4] = {2u * static_cast<uint32_t>(op.nz), 8, 1, 1};
  encode_tensor_map_f64(tmT, op.spec, 4, dims, strides, boxT, 0);
}

// octant contraction in use (EMIE_CU_NO_OCTANT=1 turns it off, for A/B runs)
static bool use_octant(const Operator& op, int q0, int q1) {
  static const bool off = [] {
    const char* e = std::getenv("EMIE_CU_NO_OCTANT");
    return e && e[0] == '1';
  }();
  // a mode shard contracts its octant rows only when the sharded apply's plan
  // delivers the transposed modes' columns too (Operator::shard_octant)
  const bool full = op.qbase == 0 && op.qcount == static_cast<int>(op.modes());
  return !off && op.xysym && op.noct > 0 && q0 == op.qbase && q1 == op.qbase + op.qcount &&
         (full || op.shard_octant);
}

// K_ct over quadrant modes [q0, q1) (all stored in op: qbase <= q0, q1 <= qbase + qcount):
// up to two right-hand sides per launch (8 columns of a full mode)
void contract_modes(const Operator& op, cplx* S, int nrhs, int q0, int q1, cudaStream_t st) {
  if (q0 < op.qbase || q1 > op.qbase + op.qcount || q0 > q1)
    fail(EMIE_CU_OUT_OF_RANGE, "contraction: quadrant modes outside the stored range");
  if (q0 == q1) return;
  const int np = 3 * op.nz;
  const int sms = sm_count();
  const int nmodes = q1 - q0;
  for (int r0 = 0; r0 < nrhs; r0 += 2) {
    const int g = std::min(2, nrhs - r0);
    cplx* Sg = S + static_cast<size_t>(r0) * op.lateral() * np;
    if (op.rows) {
      const bool oct = use_octant(op, q0, q1);
      const int nc = oct ? ct_cols<true>() : ct_cols<false>();
      const size_t smem = 1024 + static_cast<size_t>(kRowsRing) * 3 * op.nz * 128 +
                          kUStages * nc * static_cast<size_t>(np + 4) * sizeof(cplx);
      // the stored modes as {2nz doubles, nz rows, 8 blocks, modes}; box = 8 complex x nz rows
      CUtensorMap tm, tmT;
      rows_tensor_maps(op, &tm, &tmT);
      const int nwork = oct ? op.noct : nmodes;
      auto launch = [&](auto kern, int warps) {
        const int per_sm = resident_ctas(reinterpret_cast<const void*>(kern), (warps + 1) * 32, smem);
        const int grid = std::max(1, std::min(sms * per_sm, nwork));
        launch_pdl(kern, grid, (warps + 1) * 32, smem, st, tm, tmT, Sg, op.ex, op.ey, op.qx, q0, q1, op.qbase, g, op.octl,
                                                   op.noct, PeerOut{});
      };
      if (op.nz == 48) {
        if (oct) launch(contract_rows_kernel<48, true>, rows_warps<48>());
        else launch(contract_rows_kernel<48, false>, rows_warps<48>());
      } else {
        if (oct) launch(contract_rows_kernel<64, true>, rows_warps<64>());
        else launch(contract_rows_kernel<64, false>, rows_warps<64>());
      }
      check_launch("contract_rows_kernel");
      continue;
    }
    if (op.mma) {
      const bool oct = use_octant(op, q0, q1);
      const int nc = oct ? ct_cols<true>() : ct_cols<false>();
      const int bst = oct ? ct_blk_stages<true>() : ct_blk_stages<false>();
      const size_t smem = 128 + kUStages * nc * sizeof(long long) +
                          bst * static_cast<size_t>(op.nentD) * sizeof(cplx) +
                          kUStages * nc * static_cast<size_t>(np + 4) * sizeof(cplx);
      const int nwork = oct ? op.noct : nmodes;
      auto launch = [&](auto kern, int warps) {
        const int per_sm = resident_ctas(reinterpret_cast<const void*>(kern), (warps + 1) * 32, smem);
        const int grid = std::max(1, std::min(sms * per_sm, nwork));
        launch_pdl(kern, grid, (warps + 1) * 32, smem, st, op.spec, op.ctab, Sg, op.ex, op.ey, op.qx, q0, q1, op.qbase,
                                                   g, op.nentD, op.octl, op.noct, PeerOut{});
      };
      if (oct) {
        if (op.nz == 8) launch(contract_mma_kernel<8, true>, mma_warps<8>());
        else if (op.nz == 16) launch(contract_mma_kernel<16, true>, mma_warps<16>());
        else launch(contract_mma_kernel<32, true>, mma_warps<32>());
      } else {
        if (op.nz == 8) launch(contract_mma_kernel<8, false>, mma_warps<8>());
        else if (op.nz == 16) launch(contract_mma_kernel<16, false>, mma_warps<16>());
        else launch(contract_mma_kernel<32, false>, mma_warps<32>());
      }
      check_launch("contract_mma_kernel");
      continue;
    }
    const int CB = g == 2 ? 8 : 4;
    // nz in (32, 64]: warp pairs, one 32-row half each
    const int pair = (op.nz > 32 && op.nz <= 64) ? 1 : 0;
    // two input buffers per warp group; as many groups as 220 KB of SMEM holds
    const size_t per_group = 16 + 2 * static_cast<size_t>(CB) * np * sizeof(cplx);
    const int groups = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(kCtWarps >> pair, (220u << 10) / per_group)));
    const int wpb = groups << pair;
    const size_t smem = per_group * groups;
    const int nitems = use_octant(op, q0, q1) ? op.noctv : nmodes;
    const int grid = std::max(1, std::min(sms, ceil_div(nitems, groups)));
    const bool oct = use_octant(op, q0, q1);
    const int* octv = oct ? op.octl + op.noct : nullptr;
    const int noctv = oct ? op.noctv : 0;
    if (CB == 8) {
      set_smem(reinterpret_cast<const void*>(contract_kernel<8>), smem);
      contract_kernel<8><<<grid, wpb * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD, op.ex, op.ey, op.qx,
                                                       q0, q1, op.qbase, g, pair, octv, noctv);
    } else {
      set_smem(reinterpret_cast<const void*>(contract_kernel<4>), smem);
      contract_kernel<4><<<grid, wpb * 32, smem, st>>>(op.spec, Sg, op.nz, op.nsd, op.nentD, op.ex, op.ey, op.qx,
                                                       q0, q1, op.qbase, g, pair, octv, noctv);
    }
    check_launch("contract_kernel");
  }
}

void contract_modes_peer(const Operator& op, const cplx* S, int nrhs, int q0, int q1, const PeerOut& po,
                         cudaStream_t st) {
  if (!op.mma && !op.rows)
    fail(EMIE_CU_INVALID_ARGUMENT, "contract_modes_peer: needs the MMA or row-block layout (nz in {8, 16, 32, 48, 64})");
  if (q0 < op.qbase || q1 > op.qbase + op.qcount || q0 > q1)
    fail(EMIE_CU_OUT_OF_RANGE, "contraction: quadrant modes outside the stored range");
  if (po.G < 1 || po.G > kMaxPeerRanks || po.z[0] != 0 || po.z[po.G] != op.nz)
    fail(EMIE_CU_INVALID_ARGUMENT, "contract_modes_peer: bad depth slabs");
  if (q0 == q1) return;
  const int np = 3 * op.nz;
  const int sms = sm_count();
  for (int r0 = 0; r0 < nrhs; r0 += 2) {
    const int g = std::min(2, nrhs - r0);
    const cplx* Sg = S + static_cast<size_t>(r0) * op.lateral() * np;
    PeerOut pg = po;  // the group's rhs offset: mode index r*E + m counts from r0
    for (int h = 0; h < po.G; ++h)
      pg.dst[h] = po.dst[h] + static_cast<size_t>(r0) * op.lateral() * 3 * (po.z[h + 1] - po.z[h]);
    const bool oct = use_octant(op, q0, q1);
    const int nc = oct ? ct_cols<true>() : ct_cols<false>();
    const int nwork = oct ? op.noct : q1 - q0;
    if (op.rows) {
      const size_t smem = 1024 + static_cast<size_t>(kRowsRing) * 3 * op.nz * 128 +
                          kUStages * nc * static_cast<size_t>(np + 4) * sizeof(cplx);
      CUtensorMap tm, tmT;
      rows_tensor_maps(op, &tm, &tmT);
      auto launch_rows = [&](auto kern, int warps) {
        const int per_sm = resident_ctas(reinterpret_cast<const void*>(kern), (warps + 1) * 32, smem);
        const int grid = std::max(1, std::min(sms * per_sm, nwork));
        launch_pdl(kern, grid, (warps + 1) * 32, smem, st, tm, tmT, const_cast<cplx*>(Sg), op.ex, op.ey, op.qx, q0, q1,
                                                   op.qbase, g, op.octl, op.noct, pg);
      };
      if (op.nz == 48) {
        if (oct) launch_rows(contract_rows_kernel<48, true, true>, rows_warps<48>());
        else launch_rows(contract_rows_kernel<48, false, true>, rows_warps<48>());
      } else {
        if (oct) launch_rows(contract_rows_kernel<64, true, true>, rows_warps<64>());
        else launch_rows(contract_rows_kernel<64, false, true>, rows_warps<64>());
      }
      check_launch("contract_rows_kernel (peer epilogue)");
      continue;
    }
    const int bst = oct ? ct_blk_stages<true>() : ct_blk_stages<false>();
    size_t smem = 128 + kUStages * nc * sizeof(long long) + bst * static_cast<size_t>(op.nentD) * sizeof(cplx) +
                  kUStages * nc * static_cast<size_t>(np + 4) * sizeof(cplx);
    // the staged epilogue's own output stage where SMEM allows (octant, nz <=
    // 32: 209 KB), else it reuses the input-column stage
    {
      static const int optin = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        return v;
      }();
      const size_t extra = nc * static_cast<size_t>(np + 4) * sizeof(cplx);
      pg.sep = smem + extra <= static_cast<size_t>(optin) ? 1 : 0;
      if (pg.sep) smem += extra;
    }
    auto launch = [&](auto kern, int warps) {
      const int per_sm = resident_ctas(reinterpret_cast<const void*>(kern), (warps + 1) * 32, smem);
      const int grid = std::max(1, std::min(sms * per_sm, nwork));
      launch_pdl(kern, grid, (warps + 1) * 32, smem, st, op.spec, op.ctab, const_cast<cplx*>(Sg), op.ex, op.ey, op.qx, q0,
                                                 q1, op.qbase, g, op.nentD, op.octl, op.noct, pg);
    };
    if (oct) {
      if (op.nz == 8) launch(contract_mma_kernel<8, true, true>, mma_warps<8>());
      else if (op.nz == 16) launch(contract_mma_kernel<16, true, true>, mma_warps<16>());
      else launch(contract_mma_kernel<32, true, true>, mma_warps<32>());
    } else {
      if (op.nz == 8) launch(contract_mma_kernel<8, false, true>, mma_warps<8>());
      else if (op.nz == 16) launch(contract_mma_kernel<16, false, true>, mma_warps<16>());
      else launch(contract_mma_kernel<32, false, true>, mma_warps<32>());
    }
    check_launch("contract_mma_kernel (peer epilogue)");
  }
}

void apply_b(const Operator& op, const cplx* d_in, cplx* d_out, int nrhs, const System* sys,
             cudaStream_t st) {
  if (op.qbase != 0 || op.qcount != static_cast<int>(op.modes()))
    fail(EMIE_CU_INVALID_ARGUMENT, "apply: operator holds a mode shard (use the sharded apply)");
  const int np = 3 * op.nz;
  const long long rows = static_cast<long long>(nrhs) * np * op.ny;
  cplx* T = scratch<cplx>(static_cast<size_t>(rows) * op.ex, st);
  cplx* S = scratch<cplx>(static_cast<size_t>(nrhs) * op.lateral() * np, st);
  lateral_forward(op, d_in, sys ? sys->r2 : nullptr, T, S, nrhs, st);
  profile_mark(2, true, st);
  contract_modes(op, S, nrhs, op.qbase, op.qbase + op.qcount, st);
  profile_mark(2, false, st);
  lateral_inverse(op, S, T, d_in, d_out, sys ? sys->s : nullptr, sys ? sys->r1 : nullptr, nrhs,
                  st);
  release(S, st);
  release(T, st);
}

}  // namespace emie_cu
