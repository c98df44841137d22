// O(N^2) direct apply of a compressed operator on the device: the
// reference's dense_reference_apply (src/toeplitz.cpp:285-312), the oracle its
// own tests compare the FFT apply against (test_toeplitz.cpp:314-325). Not
// a hot path: the drop-in keeps the reference's 4096-cell guard.
//
// One thread per output entry (a, k, iy, ix); it walks every source cell and
// the 3 x nz source entries of the block at the signed offset between them,
// read straight from the compressed storage with the sign and transposition
// rules of fetch_block (greens.cpp:295-330):
//   xx yy zz   symmetric triangles, even in both offsets
//   xy = yx    triangle, sign sx sy
//   xz         full, sign sx;  zx(k, kp) = -xz(kp, k)
//   yz         full, sign sy;  zy(k, kp) = -yz(kp, k)
// with sx = -1 for a negative x offset, sy likewise. Fixed summation order.
#include <algorithm>

#include "operator.cuh"

namespace emie_cu {

namespace {

__device__ __forceinline__ int tri_index(int k, int kp, int nz) {  // greens.hpp:61-65, k <= kp
  return k * nz - k * (k - 1) / 2 + (kp - k);
}

// entry (a, b, k, kp) of the full tensor at offset (oi, oj)
__device__ __forceinline__ cplx tensor_entry(const cplx* __restrict__ blk, int nz, int a, int b, int k, int kp,
                                             double sx, double sy) {
  const int nt = nz * (nz + 1) / 2, nf = nz * nz;
  const int lo = min(k, kp), hi = max(k, kp);
  if (a == b) return blk[a * nt + tri_index(lo, hi, nz)];            // xx yy zz
  if (a + b == 1) return (sx * sy) * blk[3 * nt + tri_index(lo, hi, nz)];  // xy, yx
  // a z-coupling: (x|y, z) stored, (z, x|y) the negative transpose
  const bool zrow = a == 2;
  const int lat = zrow ? b : a;                 // 0: x, 1: y
  const double s = lat == 0 ? sx : sy;
  const cplx* full = blk + 4 * nt + lat * nf;
  const cplx v = zrow ? full[kp * nz + k] : full[k * nz + kp];
  return (zrow ? -s : s) * v;
}

__global__ void dense_apply_kernel(const cplx* __restrict__ blocks, const cplx* __restrict__ v,
                                   cplx* __restrict__ out, int nx, int ny, int nz) {
  const long long N = 3LL * nx * ny * nz;
  const int nent = 2 * nz * (2 * nz + 1);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < N;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ix = static_cast<int>(e % nx);
    const int iy = static_cast<int>((e / nx) % ny);
    const int k = static_cast<int>((e / (static_cast<long long>(nx) * ny)) % nz);
    const int a = static_cast<int>(e / (static_cast<long long>(nx) * ny * nz));
    cplx acc = {0.0, 0.0};
    for (int jy = 0; jy < ny; ++jy)
      for (int jx = 0; jx < nx; ++jx) {
        const int oi = iy - jy, oj = ix - jx;
        const cplx* blk = blocks + (static_cast<size_t>(abs(oi)) * nx + abs(oj)) * nent;
        const double sx = oj < 0 ? -1.0 : 1.0, sy = oi < 0 ? -1.0 : 1.0;
        for (int b = 0; b < 3; ++b)
          for (int kp = 0; kp < nz; ++kp) {
            const cplx g = tensor_entry(blk, nz, a, b, k, kp, sx, sy);
            const cplx x = v[((static_cast<size_t>(b) * nz + kp) * ny + jy) * nx + jx];
            acc = acc + g * x;
          }
      }
    out[e] = acc;
  }
}

}  // namespace

void dense_apply_host(int nx, int ny, int nz, const cplx* h_blocks, const cplx* h_in, cplx* h_out) {
  if (nx < 1 || ny < 1 || nz < 1) fail(EMIE_CU_INVALID_ARGUMENT, "dense_reference_apply: empty operator");
  const size_t nb = static_cast<size_t>(nx) * ny * 2 * nz * (2 * nz + 1), nv = 3ull * nx * ny * nz;
  cudaStream_t st = nullptr;
  cplx* d = scratch<cplx>(nb + 2 * nv, st);
  EMIE_CUDA(cudaMemcpyAsync(d, h_blocks, nb * sizeof(cplx), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(d + nb, h_in, nv * sizeof(cplx), cudaMemcpyHostToDevice, st));
  dense_apply_kernel<<<std::min(ceil_div(static_cast<long long>(nv), 128), 4096), 128, 0, st>>>(
      d, d + nb, d + nb + nv, nx, ny, nz);
  check_launch("dense_apply_kernel");
  EMIE_CUDA(cudaMemcpyAsync(h_out, d + nb + nv, nv * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(d, st);
}

}  // namespace emie_cu
