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

constexpr int kMaxL = 16;  // layers (greens.cu kMaxLayers)

struct StateDev {
  int L, gamma;
  double top[kMaxL], bot[kMaxL];  // top_of / bottom_of per layer (halfspaces: their single boundary)
  cplx sig[kMaxL], eta[kMaxL], p[kMaxL], q[kMaxL], one_p[kMaxL], one_q[kMaxL], e2l[kMaxL], em1[kMaxL],
      a[kMaxL];
};

__device__ __forceinline__ int layer_at(const StateDev& S, double z) {  // interface points belong below
  int m = 0;
  while (m < S.L && S.top[m + 1] <= z) ++m;
  return m;
}

__device__ __forceinline__ cplx ipow_c(cplx c, int n) {
  cplx r = {1.0, 0.0};
  for (int i = 0; i < n; ++i) r = r * c;
  return r;
}

__device__ cplx fundamental_dev(const StateDev& S, double z, double zs, int dz, int dzs, int lz, int lzs) {
  const bool swap = z > zs;
  const double za = swap ? zs : z, zb = swap ? z : zs;  // shallower, deeper
  const int da = swap ? dzs : dz, db = swap ? dz : dzs;
  const int rz = lz >= 0 ? lz : layer_at(S, z), rs = lzs >= 0 ? lzs : layer_at(S, zs);
  const int r = swap ? rs : rz, s = swap ? rz : rs;
  cplx amp, base;
  if (r == s) {
    amp = S.a[r];
    base = -(zb - za) * S.eta[r];
  } else {
    cplx chain = {1.0, 0.0};
    cplx path = {0.0, 0.0};
    for (int m = r; m < s; ++m) {
      chain = chain * cdiv(S.one_p[m + 1], S.em1[m] + S.e2l[m] * S.one_p[m]);
      if (m > r) path = path + (S.bot[m] - S.top[m]) * S.eta[m];
    }
    amp = S.a[s] * chain;
    base = -((zb - S.top[s]) * S.eta[s]) - (S.bot[r] - za) * S.eta[r] - path;
  }
  cplx Sp = {1.0, 0.0}, Mp = {1.0, 0.0};
  if (S.p[r].re != 0.0 || S.p[r].im != 0.0) {
    const cplx e = cexpm1((-2.0 * (za - S.top[r])) * S.eta[r]);
    Sp = S.one_p[r] + S.p[r] * e;
    Mp = (cplx{2.0, 0.0} - S.one_p[r]) - S.p[r] * e;
  }
  cplx Sq = {1.0, 0.0}, Mq = {1.0, 0.0};
  if (S.q[s].re != 0.0 || S.q[s].im != 0.0) {
    const cplx e = cexpm1((-2.0 * (S.bot[s] - zb)) * S.eta[s]);
    Sq = S.one_q[s] + S.q[s] * e;
    Mq = (cplx{2.0, 0.0} - S.one_q[s]) - S.q[s] * e;
  }
  cplx v = amp * cexp(base) * ipow_c(S.eta[r], da) * ipow_c(-S.eta[s], db) * (da & 1 ? Mp : Sp) *
           (db & 1 ? Mq : Sq);
  if (swap && S.gamma == 1) v = v * cdiv(S.sig[s], S.sig[r]);
  return v;
}

__global__ void fundamental_kernel(const StateDev S, int n, const double* __restrict__ z,
                                   const double* __restrict__ zs, const int* __restrict__ ord,
                                   cplx* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fundamental_dev(S, z[i], zs[i], ord[4 * i], ord[4 * i + 1], ord[4 * i + 2], ord[4 * i + 3]);
}

// P_m(za) / P_m(zb) inside layer m, za <= zb: the decaying-up solution's ratio
__device__ __forceinline__ cplx p_step(const StateDev& S, int m, double za, double zb) {
  const cplx e = cexp(-(zb - za) * S.eta[m]);
  if (m == 0 || (S.p[m].re == 0.0 && S.p[m].im == 0.0)) return e;
  const cplx sa = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (za - S.top[m])) * S.eta[m]);
  const cplx sb = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (zb - S.top[m])) * S.eta[m]);
  return e * cdiv(sa, sb);
}

// the piece of interval [a, b] in layer m below / above the observation depth:
// a_m / eta int_a^b of the source-side solution anchored at a (below) or b (above)
__device__ __forceinline__ cplx piece(const StateDev& S, int m, double a, double b, bool above) {
  const cplx eta = S.eta[m];
  const cplx u = -cexpm1(-(b - a) * eta);
  const bool hp = S.p[m].re != 0.0 || S.p[m].im != 0.0, hq = S.q[m].re != 0.0 || S.q[m].im != 0.0;
  cplx sp = {1.0, 0.0}, tq = {1.0, 0.0};
  if (above) {
    if (hp) sp = S.one_p[m] + S.p[m] * cexpm1(-(a + b - 2.0 * S.top[m]) * eta);
    if (hq) tq = S.one_q[m] + S.q[m] * cexpm1((-2.0 * (S.bot[m] - b)) * eta);
  } else {
    if (hp) sp = S.one_p[m] + S.p[m] * cexpm1((-2.0 * (a - S.top[m])) * eta);
    if (hq) tq = S.one_q[m] + S.q[m] * cexpm1(-(2.0 * S.bot[m] - a - b) * eta);
  }
  return cdiv(S.a[m], eta) * u * sp * tq;
}

// single moments m[az][j] = d^az/dz^az int_j U(z_obs, zs) dzs, az in {0, 1}
// (layered.cpp:450-542 contract), one observation depth per thread
__global__ void point_moments_kernel(const StateDev S, const Interval* __restrict__ iv, const double* __restrict__ br,
                                     int nz, int n, const double* __restrict__ zobs, cplx* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double z0 = zobs[t];
  cplx* m0 = out + static_cast<size_t>(t) * 2 * nz;
  cplx* m1 = m0 + nz;
  const int r0 = layer_at(S, z0);
  const cplx e0 = S.eta[r0];
  // log-derivatives of the decaying-up (P) and decaying-down (Q) solutions at z0
  cplx dP = e0, dQ = -e0;
  if (r0 != 0 && (S.p[r0].re != 0.0 || S.p[r0].im != 0.0)) {
    const cplx e = cexpm1((-2.0 * (z0 - S.top[r0])) * e0);
    dP = e0 * cdiv((cplx{2.0, 0.0} - S.one_p[r0]) - S.p[r0] * e, S.one_p[r0] + S.p[r0] * e);
  }
  if (r0 != S.L && (S.q[r0].re != 0.0 || S.q[r0].im != 0.0)) {
    const cplx e = cexpm1((-2.0 * (S.bot[r0] - z0)) * e0);
    dQ = -e0 * cdiv((cplx{2.0, 0.0} - S.one_q[r0]) - S.q[r0] * e, S.one_q[r0] + S.q[r0] * e);
  }
  int k;  // interval holding z0; -1 above the partition, nz below it
  if (z0 <= br[0]) k = -1;
  else if (z0 >= br[nz]) k = nz;
  else {
    k = 0;
    while (br[k + 1] <= z0) ++k;
  }
  auto factors = [&](int j) {
    const Interval I = iv[j];
    const int m = I.layer;
    const IvPack pk = iv_pack(I, S.eta[m], crecip(S.eta[m]), S.e2l[m]);
    return iv_factors(I, pk, S.p[m], S.q[m], S.a[m], S.one_p[m], S.one_q[m]);
  };
  for (int j = 0; j < min(k, nz); ++j) {  // above: the source-side P branch to z0
    const IvFac f = factors(j);
    const cplx u1 = fundamental_dev(S, br[j + 1], z0, 0, 0, -1, -1);
    const cplx sf = S.gamma == 1 ? cdiv(S.sig[r0], S.sig[iv[j].layer]) : cplx{1.0, 0.0};
    m0[j] = sf * f.H0 * u1;
    m1[j] = m0[j] * dQ;
  }
  if (k >= 0 && k < nz) {  // the interval holding z0, split there
    const int m = iv[k].layer;
    const cplx up = z0 > br[k] ? piece(S, m, br[k], z0, true) : cplx{0.0, 0.0};
    const cplx lo = z0 < br[k + 1] ? piece(S, m, z0, br[k + 1], false) : cplx{0.0, 0.0};
    m0[k] = up + lo;
    m1[k] = dQ * up + dP * lo;
  }
  if (k < nz) {  // below: the observation-side P ratio chained down
    const int first = max(k + 1, 0);
    cplx T = {1.0, 0.0};
    double zc = z0;
    int m = r0;
    while (zc < br[first]) {
      const double seg = m < S.L ? fmin(S.bot[m], br[first]) : br[first];
      T = T * p_step(S, m, zc, seg);
      zc = seg;
      if (zc < br[first]) ++m;
    }
    for (int j = first; j < nz; ++j) {
      const IvFac f = factors(j);
      m0[j] = T * f.J0;
      m1[j] = dP * m0[j];
      T = T * f.theta;
    }
  }
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
