// Point evaluations of the layered-medium fundamental solution on the device:
// fundamental_value (layered.hpp:60-66) and point_moments (layered.hpp:116-126),
// the receiver-side single moments. A spectral state (SpectralLayerState,
// layered.hpp:41-58) arrives by value; every thread evaluates one point (or
// one observation depth) in the closed forms below. Used by the drop-in's
// layered API and by the receiver-field evaluation.
//
// Fundamental solution of the 1-D two-point problem for depths z <= z'
// (lower = shallower point, layers r <= s):
//   U = amp e^{base} S_p(z) S_q(z'),
//   same layer: amp = a_r (diag_a), base = -eta_r (z' - z);
//   else        amp = a_s prod_{m=r}^{s-1} (1 + p_{m+1}) / (em1_m + e2l_m (1 + p_m)),
//               base = -eta_s (z' - top_s) - eta_r (bot_r - z) - sum_{r<m<s} eta_m l_m,
//   S_p(z) = 1 + p_r e^{-2 eta_r (z - top_r)}, S_q(z') = 1 + q_s e^{-2 eta_s (bot_s - z')},
// each evaluated as (1 + p) + p expm1(.) so near-total reflection keeps its
// digits. A derivative in the shallower point multiplies by eta_r and turns
// S_p into M_p = 1 - p e^{...}; one in the deeper point multiplies by -eta_s
// and turns S_q into M_q. For the conductive gamma the value with z > z'
// carries sigma_s / sigma_r (the sigma-weighted derivative continuity).
#include <algorithm>
#include <vector>

#include "layered.cuh"
#include "operator.cuh"

namespace emie_cu {

namespace {

__global__ void fundamental_kernel(const StateDev S, int n, const double* __restrict__ z,
                                   const double* __restrict__ zs, const int* __restrict__ ord,
                                   cplx* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fundamental_dev(S, z[i], zs[i], ord[4 * i], ord[4 * i + 1], ord[4 * i + 2], ord[4 * i + 3]);
}

// one observation depth per thread
__global__ void point_moments_kernel(const StateDev S, const Interval* __restrict__ iv, const double* __restrict__ br,
                                     int nz, int n, const double* __restrict__ zobs, cplx* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  cplx* m0 = out + static_cast<size_t>(t) * 2 * nz;
  point_moments_dev(S, iv, br, nz, zobs[t], m0, m0 + nz);
}

StateDev state_of(int L, const double* tops, const cplx* st9, int gamma) {
  if (L < 1 || L + 1 > kMaxL) fail(EMIE_CU_INVALID_ARGUMENT, "spectral state: unsupported layer count");
  StateDev S{};
  S.L = L;
  S.gamma = gamma;
  const int NL = L + 1;
  for (int m = 0; m <= L; ++m) {
    S.top[m] = m == 0 ? tops[0] : tops[m - 1];
    S.bot[m] = m == L ? tops[L - 1] : tops[m];
    S.sig[m] = st9[m];
    S.eta[m] = st9[NL + m];
    S.p[m] = st9[2 * NL + m];
    S.q[m] = st9[3 * NL + m];
    S.one_p[m] = st9[4 * NL + m];
    S.one_q[m] = st9[5 * NL + m];
    S.e2l[m] = st9[6 * NL + m];
    S.em1[m] = st9[7 * NL + m];
    S.a[m] = st9[8 * NL + m];
  }
  return S;
}

}  // namespace

void fundamental_values_host(int L, const double* tops, const cplx* st9, int gamma, int n, const double* z,
                             const double* zs, const int* ord, cplx* out) {
  if (n <= 0) return;
  const StateDev S = state_of(L, tops, st9, gamma);
  cudaStream_t st = nullptr;
  double* dz = scratch<double>(2 * static_cast<size_t>(n), st);
  int* dord = scratch<int>(4 * static_cast<size_t>(n), st);
  cplx* dout = scratch<cplx>(n, st);
  EMIE_CUDA(cudaMemcpyAsync(dz, z, n * sizeof(double), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dz + n, zs, n * sizeof(double), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dord, ord, 4 * n * sizeof(int), cudaMemcpyHostToDevice, st));
  fundamental_kernel<<<ceil_div(n, 128), 128, 0, st>>>(S, n, dz, dz + n, dord, dout);
  check_launch("fundamental_kernel");
  EMIE_CUDA(cudaMemcpyAsync(out, dout, n * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(dz, st);
  release(dord, st);
  release(dout, st);
}

void point_moments_host(int L, const double* tops, const cplx* st9, int gamma, int nz, const double* breaks,
                        const int* layer, int n, const double* zobs, cplx* out) {
  if (n <= 0 || nz <= 0) return;
  const StateDev S = state_of(L, tops, st9, gamma);
  std::vector<Interval> ivh(nz);
  for (int i = 0; i < nz; ++i) {
    Interval& I = ivh[i];
    const int m = layer[i];
    if (m < 0 || m > L) fail(EMIE_CU_INVALID_ARGUMENT, "point_moments: interval layer out of range");
    I.a = breaks[i];
    I.b = breaks[i + 1];
    I.h = I.b - I.a;
    I.layer = m;
    I.d = S.top[m];
    I.dp = S.bot[m];
    I.l = S.bot[m] - S.top[m];
    I.has_p = m > 0;
    I.has_q = m < L;
    I.inv_sig = {0.0, 0.0};
  }
  cudaStream_t st = nullptr;
  Interval* div = scratch<Interval>(nz, st);
  double* dbr = scratch<double>(nz + 1 + static_cast<size_t>(n), st);
  cplx* dout = scratch<cplx>(static_cast<size_t>(n) * 2 * nz, st);
  EMIE_CUDA(cudaMemcpyAsync(div, ivh.data(), nz * sizeof(Interval), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dbr, breaks, (nz + 1) * sizeof(double), cudaMemcpyHostToDevice, st));
  EMIE_CUDA(cudaMemcpyAsync(dbr + nz + 1, zobs, n * sizeof(double), cudaMemcpyHostToDevice, st));
  point_moments_kernel<<<ceil_div(n, 64), 64, 0, st>>>(S, div, dbr, nz, n, dbr + nz + 1, dout);
  check_launch("point_moments_kernel");
  EMIE_CUDA(cudaMemcpyAsync(out, dout, static_cast<size_t>(n) * 2 * nz * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  EMIE_CUDA(cudaStreamSynchronize(st));
  release(div, st);
  release(dbr, st);
  release(dout, st);
}

}  // namespace emie_cu
