// Column moves of the sharded apply: the spectrum of a
// depth slab, S_loc[r][m][c*nzh + z] (mode-major, mode m = mx*ey + my), and
// the full-depth spectrum of a rank's quadrant-mode shard, S[r][m][c*nz + z],
// exchange columns through packed all-to-all buffers [r][i][c*nzh + z]
// (i over the destination's mirror-mode list). One gather/scatter kernel
// covers the four directions: each side is either "mapped" (mode = idx[i] of
// modes_total) or "packed" (mode = i of nidx), with its own plane stride and
// depth offset. Reference: the stages of apply(SystemOperator)
// (src/cie.cpp:56-73, src/toeplitz.cpp:163-283) split at the contraction.
#include "operator.cuh"

namespace emie_cu {

namespace {

__global__ void move_planes_kernel(const cplx* __restrict__ src, cplx* __restrict__ dst, int nrhs, int nidx,
                                   const int* __restrict__ idx, long long E, int4 sd, int4 dd, int nzh) {
  const long long per = 3LL * nzh;  // planes moved per (r, i)
  const long long total = static_cast<long long>(nrhs) * nidx * per;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long ri = e / per;
    const int w = static_cast<int>(e - ri * per);
    const int c = w / nzh, z = w - c * nzh;
    const int r = static_cast<int>(ri / nidx), i = static_cast<int>(ri - static_cast<long long>(r) * nidx);
    const long long ms = sd.x ? static_cast<long long>(r) * E + __ldg(idx + i) : ri;
    const long long md = dd.x ? static_cast<long long>(r) * E + __ldg(idx + i) : ri;
    dst[md * dd.y + c * dd.z + dd.w + z] = ldg(src + ms * sd.y + c * sd.z + sd.w + z);
  }
}

}  // namespace

void move_planes(const cplx* src, cplx* dst, int nrhs, int nidx, const int* idx, long long modes_total,
                 const int src_desc[4], const int dst_desc[4], int nzh, cudaStream_t st) {
  const long long total = static_cast<long long>(nrhs) * nidx * 3 * nzh;
  if (total == 0) return;
  int sms = 0, dev = 0;
  EMIE_CUDA(cudaGetDevice(&dev));
  EMIE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = static_cast<int>(std::min<long long>(ceil_div(total, 256), 8LL * sms));
  move_planes_kernel<<<grid, 256, 0, st>>>(src, dst, nrhs, nidx, idx, modes_total,
                                           make_int4(src_desc[0], src_desc[1], src_desc[2], src_desc[3]),
                                           make_int4(dst_desc[0], dst_desc[1], dst_desc[2], dst_desc[3]), nzh);
  check_launch("move_planes_kernel");
}

}  // namespace emie_cu
