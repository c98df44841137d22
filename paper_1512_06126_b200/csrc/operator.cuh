// Device-resident operator objects behind the C ABI (include/emie_cu.h).
#pragma once

#include <cstdlib>
#include <utility>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

#include "../../include/emie_cu.h"
#include "common.cuh"
#include "fft.cuh"

namespace emie_cu {

// SpectralOperator (reference include/emie/toeplitz.hpp:21-35), device side.
// Spectra layout (HBM): mode-major, one contiguous block of nentD = nent =
// 2nz(2nz+1) complex per quadrant mode (a permutation of the reference's
// entries), each nz x nz component stored by WRAPPED DIAGONALS:
//   full F (xz, yz):       D_t[k] = F(k, (k+t) mod nz),  t = 0..nz-1
//   symmetric S (xx yy zz xy): D_t[k] = S(k, (k+t) mod nz) for 2t < nz;
//     S(k,kp) with t = (kp-k) mod nz, 2t > nz, is D_{nz-t}[kp]; for even nz
//     the half diagonal t = nz/2 keeps only k < nz/2 (S(k,kp) at
//     D_{nz/2}[min(k,kp)]), so each component is exactly nz(nz+1)/2 long
//   block = [xx | yy | zz | xy] (4 * ntri) then [xz | yz] (2 * nz^2)
// With lane k of a warp handling output row k, step t reads one contiguous
// (rotated) 32-entry run of every diagonal: the contraction streams each
// mode's coefficients straight from L2 with coalesced loads, no SMEM copy.
// emap[e] maps reference entry e (GreensBlock order: triangles tri(k,kp)
// then full k*nz+kp) to its diagonal slot(s).
struct Operator {
  int nx = 0, ny = 0, nz = 0;
  int ex = 0, ey = 0, qx = 0, qy = 0;
  double omega = 0.0;
  int ntri = 0, nfull = 0, nent = 0;
  int nsd = 0, nentD = 0;    // symmetric diagonals per component, diag block size
  cplx* spec = nullptr;      // qx*qy*nentD (diagonal or MMA layout)
  std::size_t spec_bytes = 0;  // its allocation (recycled by the next operator, capi.cu spec_alloc)
  int2* emap = nullptr;      // reference entry -> (slot, second slot or -1)
  std::vector<int2> emap_host;
  // MMA layout (nz in {8, 16, 32}, contraction on the FP64 tensor cores):
  // every nz x nz component is stored so that the element read by fragment
  // lane (row k, col kp) lies in 16-byte bank f(k,kp) = k + kp + 4[(k^kp)&nz/2]
  // (mod 8; the 4-term only for nz >= 16). Symmetric components (xx yy zz xy)
  // hold their upper triangle bank-sorted, padded to ntriP = 8 * (largest bank
  // count); full components (xz yz) are row-major with each aligned 8-run of
  // kp rotated to bank f. With the tile rows {4m..4m+3} u {4m+nz/2..} every
  // quarter-warp of a fragment load touches 8 distinct banks.
  bool mma = false;
  // ROWS layout (nz in {48, 64}, streamed contraction, operator.cu): per mode
  // six dense row-major nz x nz blocks [xx yy zz xy xz yz] (the symmetric
  // ones with both triangles; -xz^T / -yz^T are read as row slices of xz / yz)
  bool rows = false;
  int ntriP = 0;
  uint32_t* ctab = nullptr;  // [a][b][k][kp] -> slot of M_ab(k,kp), bit 31: negated
  cplx* blocks = nullptr;    // optional compressed blocks, (ny*nx)*nent
  cplx* tw_x = nullptr;      // e^{-2 pi i m/ex}
  cplx* tw_y = nullptr;      // e^{-2 pi i m/ey}

  FftPlan plan_x, plan_y;    // mixed-radix plans (any 5-smooth length)
  FftPlan plan_x2, plan_y2;  // radix-16 plans when the length is a power of two
  bool p2x = false, p2y = false;

  // stored quadrant modes [qbase, qbase + qcount): all of them unless the
  // operator is a mode shard of a sharded apply (or a lateral-only geometry, qcount = 0)
  int qbase = 0, qcount = 0;

  // x <-> y transposition symmetry (square grid, ex == ey, compressed blocks
  // with block(oj, oi) == block(oi, oj) under xx <-> yy, xz <-> yz exactly):
  // the block of quadrant mode (qmy, qmx) is then the block of (qmx, qmy)
  // with the x and y rows and columns exchanged, so the contraction reads
  // only the octant qmx <= qmy (octl: those modes, off-diagonal ones first)
  bool xysym = false;
  int* octl = nullptr;  // noct octant modes, then the DFMA kernel's noctv item codes
  int noct = 0, noctv = 0;
  // a row-aligned mode shard (qbase, qcount whole rows) of an xysym operator
  // contracts its octant rows -- the modes (qmy, qmx <= qmy) of its rows and
  // their transposes, i.e. every quadrant mode whose larger index is one of
  // its rows -- instead of its quadrant modes; set by the sharded apply whose
  // plan gives the rank those modes (emie_cu_operator_shard_octant)
  bool shard_octant = false;

  std::size_t modes() const { return static_cast<std::size_t>(qx) * qy; }
  std::size_t lateral() const { return static_cast<std::size_t>(ex) * ey; }
  std::size_t cells() const { return static_cast<std::size_t>(nx) * ny * nz; }
  ~Operator();
};

// SystemOperator (reference include/emie/cie.hpp:26-34), device side.
struct System {
  const Operator* op = nullptr;  // non-owning, like the reference
  cplx* s = nullptr;             // 1 - gamma, per cell
  double* r1 = nullptr;          // 2 sqrt(Re sigma_b) / V, per cell
  cplx* r2 = nullptr;            // -sqrt(Re sigma_b) gamma, per cell
  ~System();
};

// host helpers
// allocates spectra for quadrant modes [q0, q1) (q1 < 0: all; q0 == q1: lateral geometry only)
void init_operator_geometry(Operator& op, int nx, int ny, int nz, double omega, int q0 = 0, int q1 = -1);
void keep_pool_warm();
cplx* upload_twiddles(int n);

// lateral FFT stages (lateral.cu)
void lateral_spectra(const Operator& op, const cplx* d_blocks, cudaStream_t st);
void lateral_forward(const Operator& op, const cplx* d_in, const cplx* r2, cplx* T, cplx* S,
                     int nrhs, cudaStream_t st);
void lateral_inverse(const Operator& op, const cplx* S, cplx* T, const cplx* d_in, cplx* d_out,
                     const cplx* s, const double* r1, int nrhs, cudaStream_t st);
// the sharded apply's slab forward with the forward transpose fused into the
// y pass (stores into the owners' full-depth spectra, owner[mode] -> rank)
bool lateral_forward_peer_ok(const Operator& op);
// owner: mode -> rank table, or nullptr and the plan's splits (rows when oct, else quadrant modes)
void lateral_forward_peer(const Operator& op, const cplx* d_in, const cplx* r2, cplx* T, const int* owner,
                          const int* split, int oct, cplx* const* dsts, int G, int nzf, int zoff, int nrhs,
                          cudaStream_t st);

// stages (operator.cu)
// sym_known: 1 the blocks are x <-> y symmetric by construction, 0 they are
// not, -1 check on the device (bitwise)
void transform_blocks(Operator& op, const cplx* d_blocks, cudaStream_t st, int sym_known = -1);
void set_octant_lists(Operator& op, cudaStream_t st);
void apply_b(const Operator& op, const cplx* d_in, cplx* d_out, int nrhs,
             const System* sys, cudaStream_t st);
void contract_modes(const Operator& op, cplx* S, int nrhs, int q0, int q1, cudaStream_t st);
// the sharded apply's contraction with its results stored straight into the
// slab owners' spectra (peer memory): plane a*nz + k goes to rank h with
// z[h] <= k < z[h+1], at dst[h][(r*E + m)*3nzh + a*nzh + k - z[h]]
constexpr int kMaxPeerRanks = 64;
constexpr int kRowsBlocks = 6;  // dense blocks per mode of the ROWS layout
// launch with programmatic stream serialisation (the kernel calls
// pdl_trigger / pdl_wait): it may start while the previous kernel of the
// stream drains. EMIE_CU_PDL=0 launches plainly (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EMIE_CU_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct PeerOut {
  int G = 0;
  cplx* dst[kMaxPeerRanks];
  int z[kMaxPeerRanks + 1];
  int sep = 0;  // launcher-set: the staged epilogue has its own SMEM stage (else it reuses the input-column stage)
};
void contract_modes_peer(const Operator& op, const cplx* S, int nrhs, int q0, int q1, const PeerOut& po,
                         cudaStream_t st);

// sharded apply column moves (shard.cu); desc = {mapped, planes per column, component stride, depth offset}
void move_planes(const cplx* src, cplx* dst, int nrhs, int nidx, const int* idx, long long modes_total,
                 const int src_desc[4], const int dst_desc[4], int nzh, cudaStream_t st);

// peer-memory exchange flags (peer.cu): release-store `epoch` into slot `me`
// of every rank's flag array / wait until all G slots of `flags` reach it
void peer_signal(int* const* flag_ptrs, int G, int me, int epoch, cudaStream_t st);
int peer_status();
void peer_wait(const int* flags, int G, int epoch, cudaStream_t st);

// Green's build (greens.cu)
struct FilterParams {
  double step = 0.2, shift = 0.0964;
  int half = 512, n1 = -250, n2 = 200;
};
void check_filter_params(const FilterParams& fp);
void greens_build(Operator& op, int L, const double* tops, const cplx* sigma,
                  const double* breaks, double hx, double hy, const FilterParams& fp,
                  bool keep_blocks, cudaStream_t st);
// the build in two parts (sharded build): the blocks of computed offsets
// [c0, c1) of computed_offsets(), then mirror + spectra of op's stored modes
std::vector<int> computed_offsets(int nx, int ny, double hx, double hy);
void greens_blocks(const Operator& op, int L, const double* tops, const cplx* sigma, const double* breaks,
                   double hx, double hy, const FilterParams& fp, int c0, int c1, cplx* blocks, cudaStream_t st);
void greens_finish(Operator& op, cplx* blocks, double hx, double hy, cudaStream_t st);
void kernel_output_host(int oi, int oj, double hx, double hy, int alpha, int beta,
                        const double* s, int n, double* out);
void design_offset_filters_host(int oi, int oj, double hx, double hy, const FilterParams& fp,
                                double* w, double* lam);
void assemble_signed_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                          const double* breaks, double hx, double hy, const FilterParams& fp, int n, const int* oi,
                          const int* oj, cplx* h_out);
void dense_apply_host(int nx, int ny, int nz, const cplx* h_blocks, const cplx* h_in, cplx* h_out);
void layered_probe_host(int what, int L, const double* tops, const cplx* sigma, int nz, const double* breaks,
                        double omega, int n, const double* lam, cplx* out);
void fundamental_values_host(int L, const double* tops, const cplx* st9, int gamma, int n, const double* z,
                             const double* zs, const int* ord, cplx* out);
void point_moments_host(int L, const double* tops, const cplx* st9, int gamma, int nz, const double* breaks,
                        const int* layer, int n, const double* zobs, cplx* out);
void design_geometry_host(const double geom[4], int alpha, int beta, const FilterParams& fp, double* w, double* lam);
void kernel_output_geom_host(const double geom[4], int alpha, int beta, const double* s, int n, double* out);
void design_input_host(int n, const double* lam, double* out);
void pair_geometry_host(int oi, int oj, double hx, double hy, double out[4]);
void assemble_full_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                        const double* breaks, double hx, double hy, const FilterParams& fp, int oi, int oj,
                        cplx* h_out);
void receiver_host(int nx, int ny, int nz, double omega, int L, const double* tops, const cplx* sigma,
                   const double* breaks, double hx, double hy, double x0, double y0, const FilterParams& fp,
                   const cplx* h_sa, int nrhs, const cplx* h_U, int nrec, const double* rec, cplx* h_out,
                   int tens_col);
void vfunctions_host(int L, const double* tops, const cplx* sigma, int nz, const double* breaks, double omega,
                     int n, const double* lam, cplx* out);

// launch configuration cached per (device, kernel, threads, dynamic SMEM)
// (capi.cu): sets the SMEM opt-in once and returns the resident CTAs per SM;
// the hot paths launch the same kernels every apply, so these host queries
// stay out of the per-apply cost
int resident_ctas(const void* fn, int threads, std::size_t smem);
int sm_count();

// stage profiling (capi.cu): no-ops unless emie_cu_profile_enable(1)
void profile_mark(int stage, bool begin, cudaStream_t st);

// scratch from the stream-ordered pool (reentrant per call)
template <class T>
T* scratch(std::size_t n, cudaStream_t st) {
  void* p = nullptr;
  EMIE_CUDA(cudaMallocAsync(&p, n * sizeof(T) + 16, st));
  return static_cast<T*>(p);
}
// never throws: also used from destructors and unwinding paths
inline void release(void* p, cudaStream_t st) noexcept {
  if (p) (void)cudaFreeAsync(p, st);
}

// slab vector operations of the sharded FGMRES (solver.cu): local sums,
// finalized on the device; the caller all-reduces them
void vec_dots(const cplx* V, std::size_t vstride, int nv, const cplx* w, std::size_t n, bool with_norm,
              double* out, cudaStream_t st);
void vec_update(cplx* w, const cplx* V, std::size_t vstride, int nv, const double* h, std::size_t n,
                double* dots_out, double* norm_out, cudaStream_t st);
void vec_dcgs_dots(const cplx* V, std::size_t vstride, int nv, const cplx* w, std::size_t n, double* out,
                   cudaStream_t st);
void vec_dcgs_update(cplx* w, cplx* V, std::size_t vstride, int nv, const double* coef, std::size_t n,
                     double* norm_out, cudaStream_t st);
void vec_combine(cplx* x, const cplx* V, std::size_t vstride, int nv, const double* y, std::size_t n,
                 cudaStream_t st);
void vec_scale(cplx* y, const cplx* x, double a, std::size_t n, cudaStream_t st);
void vec_residual(cplx* r, const cplx* b, const cplx* t, std::size_t n, double* norm_out, cudaStream_t st);

void fgmres_device(const System& sys, const cplx* d_rhs, cplx* d_x, int nrhs, double tol,
                   int m, int max_iters, emie_cu_report* reports, double* h_history,
                   int hist_cap, cudaStream_t st);
// The same device FGMRES over any linear map: A applies nrhs device vectors
// of n complex entries (in -> out, stream ordered); precond, when set, is the
// flexible right preconditioner (cie.hpp:57, cie.cpp:151-156: z_j = M v_j,
// x += sum y_j z_j); on_iteration(rhs, iteration, residual estimate) is
// called live, where the reference calls SolverConfig::on_iteration
// (cie.cpp:178-185, 199-201). speculate = false when A or M has side effects
// the caller can observe (host callbacks): no speculative next-step apply.
struct KrylovMap {
  std::size_t n = 0;
  std::function<void(const cplx* in, cplx* out, int nrhs, cudaStream_t st)> apply;
  std::function<void(const cplx* in, cplx* out, cudaStream_t st)> precond;
  std::function<void(int rhs, int iteration, double residual)> on_iteration;
  bool speculate = true;
};
void fgmres_map(const KrylovMap& A, const cplx* d_rhs, cplx* d_x, int nrhs, double tol, int m, int max_iters,
                emie_cu_report* reports, double* h_history, int hist_cap, cudaStream_t st);

}  // namespace emie_cu
