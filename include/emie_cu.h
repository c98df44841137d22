/* emie_cu.h — C ABI of the B200 (sm_100a) CIE hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * torch or C++ types. Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj). The C++ mirror of the
 * reference API (include/emie/*.hpp, namespace emie) and the Python mirror
 * (paper_1512_06126_b200) are thin layers over these functions.
 *
 * Conventions
 *  - Complex numbers are interleaved double pairs, layout-compatible with
 *    std::complex<double> (the reference's cdouble, include/emie/types.hpp:9).
 *  - Field vectors use the reference GridVector layout
 *    ((c*nz + iz)*ny + iy)*nx + ix (include/emie/types.hpp:14-30); a batch of
 *    nrhs fields is nrhs such vectors back to back.
 *  - "d_" pointers are device pointers (cuda:0 context of the caller),
 *    "h_" pointers are host pointers.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Status codes map one-to-one onto the reference's exception types
 *    (SURVEY.md §8(b)): no exception crosses the ABI; the message of the last
 *    failure on the calling thread is emie_cu_last_error().
 *  - Every kernel is deterministic (no order-dependent atomics): repeated and
 *    concurrent calls return bit-identical results (test_toeplitz.cpp:416-434).
 */
#ifndef EMIE_CU_H
#define EMIE_CU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum emie_cu_status {
  EMIE_CU_OK = 0,
  EMIE_CU_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  EMIE_CU_DOMAIN_ERROR = 2,     /* std::domain_error */
  EMIE_CU_OUT_OF_RANGE = 3,     /* std::out_of_range */
  EMIE_CU_RUNTIME_ERROR = 4,    /* std::runtime_error */
  EMIE_CU_CUDA_ERROR = 5        /* device failure (no reference equivalent) */
};

typedef struct emie_cu_operator_s* emie_cu_operator; /* device SpectralOperator */
typedef struct emie_cu_system_s* emie_cu_system;     /* device SystemOperator */

const char* emie_cu_last_error(void);
const char* emie_cu_version(void);
int emie_cu_device_count(int* count);
/* grow the library's stream-ordered memory pool by `bytes` once (allocated
 * and freed; the pool keeps it reserved), so the first large build or solve
 * does not pay the device's first-touch allocation cost */
int emie_cu_pool_reserve(unsigned long long bytes);

/* smooth_embedding_size (include/emie/toeplitz.hpp:13, src/toeplitz.cpp:18-26) */
int emie_cu_smooth_embedding_size(int n, int* out);

/* ---------------------------------------------------------------------
 * Spectral operator (SpectralOperator, include/emie/toeplitz.hpp:21-35)
 * ------------------------------------------------------------------- */

/* transform_operator (include/emie/toeplitz.hpp:37, src/toeplitz.cpp:92-161)
 * from a host compressed operator (CompressedGreensOperator,
 * include/emie/greens.hpp:74-81): blocks[oi*nx + oj], each block the six
 * GreensBlock components xx yy zz xy (upper triangles, nz(nz+1)/2 entries,
 * index tri(k,kp) of greens.hpp:61-65) then xz yz (full nz*nz), i.e.
 * 2 nz (2 nz + 1) complex per block. The parity-extended 2-D lateral
 * transforms run on the device; the result stays device-resident. */
int emie_cu_operator_from_blocks(int nx, int ny, int nz, double omega,
                                 const double* h_blocks, emie_cu_operator* out,
                                 void* stream);

/* assemble_operator + transform_operator (include/emie/greens.hpp:144-147,
 * src/greens.cpp:332-371; toeplitz.cpp:92-161) entirely on the device:
 * filter design (hankel.cpp:204-281), lambda accumulation of the vertical
 * moment tables (greens.cpp:150-221, layered.cpp:67-408), spectra.
 * Model: L interfaces tops[L] (m), L+1 complex conductivities sigma.
 * Grid: nz intervals breaks[nz+1] (m), nx x ny cells of hx x hy (m).
 * filter: {step, shift, half, n1, n2} (FilterParams, hankel.hpp:20-26) or
 * NULL for the defaults. keep_blocks != 0 keeps the compressed blocks on
 * the device for emie_cu_operator_download_blocks. */
int emie_cu_greens_build(int L, const double* tops, const double* sigma, int nz,
                         const double* breaks, int nx, int ny, double hx, double hy,
                         double omega, const double* filter, int keep_blocks,
                         emie_cu_operator* out, void* stream);

/* assemble_block (include/emie/greens.hpp:129-135, src/greens.cpp:150-221) at
 * n signed lateral offsets (oi[i], oj[i]), |oi| < ny, |oj| < nx (else
 * EMIE_CU_OUT_OF_RANGE, greens.cpp:153-154): filter design and lambda
 * accumulation on the device for exactly these offsets, each evaluated
 * independently (no mirror). h_blocks: n blocks of 2 nz (2 nz + 1) complex in
 * GreensBlock order (xx yy zz xy upper triangles, xz yz full). */
int emie_cu_assemble_blocks(int L, const double* tops, const double* sigma, int nz, const double* breaks,
                            int nx, int ny, double hx, double hy, double omega, const double* filter,
                            int n, const int* h_oi, const int* h_oj, double* h_blocks);

/* a SpectralOperator given by its six host component arrays (the
 * emie_cu_operator_download_spectra layout): uploaded into the device
 * wrapped-diagonal layout, no transform */
int emie_cu_operator_from_spectra(int nx, int ny, int nz, double omega, const double* h_comp,
                                  emie_cu_operator* out);

/* dims = {nx, ny, nz, ex, ey, qx, qy}; omega */
int emie_cu_operator_dims(emie_cu_operator op, int dims[7], double* omega);

/* x <-> y transposition symmetry of the operator (no reference counterpart:
 * a property of src/toeplitz.cpp:92-161's spectra on a square grid whose
 * compressed blocks satisfy block(oj, oi) = block(oi, oj) with xx <-> yy and
 * xz <-> yz, checked bit for bit when the operator is built). *out = 1 when
 * the contraction reads only the octant modes qmx <= qmy. disable != 0 turns
 * the octant contraction off for this operator (A/B comparisons); it cannot
 * be turned back on. */
int emie_cu_operator_xy_symmetry(emie_cu_operator op, int disable, int* out);

/* SpectralOperator::comp (toeplitz.hpp:58-61): six host arrays written back
 * to back: comp[c][(my*qx + mx)*nent + s], nent = nz(nz+1)/2 for c < 4 and
 * nz^2 for c >= 4 (total qx*qy*2nz(2nz+1) complex). */
int emie_cu_operator_download_spectra(emie_cu_operator op, double* h_comp);

/* compressed blocks in the emie_cu_operator_from_blocks layout; only for
 * operators built with keep_blocks or from blocks. */
int emie_cu_operator_download_blocks(emie_cu_operator op, double* h_blocks);

/* filter weights of one offset: w[6][n2-n1+1], lam[n2-n1+1], in the
 * greens.cpp:137 order (0,0) (2,0) (0,2) (1,1) (1,0) (0,1); hankel.cpp:239-281 */
int emie_cu_design_offset_filters(int oi, int oj, double hx, double hy,
                                  const double* filter, double* h_w, double* h_lam);

/* kernel_output (hankel.hpp:32, hankel.cpp:101-113): the closed-form design
 * output of the (alpha, beta) kernel at log radii s[n], as the device filter
 * design samples it */
int emie_cu_kernel_output(int oi, int oj, double hx, double hy, int alpha, int beta,
                          const double* h_s, int n, double* h_out);

/* pair_geometry (hankel.hpp:35, hankel.cpp:80-91) -> out {r, p, q, phi}: the
 * device build's own geometry routine, evaluated on the host */
int emie_cu_pair_geometry(int oi, int oj, double hx, double hy, double* out);

/* FilterDesigner::design / design_weights (hankel.hpp:62-63, 93; hankel.cpp:
 * 239-281) of one (alpha, beta) kernel for a pair geometry {r, p, q, phi} on
 * the device: weights h_w[n2-n1+1], abscissae h_lam[n2-n1+1] */
int emie_cu_design_filter(const double* geom, int alpha, int beta, const double* filter, double* h_w,
                          double* h_lam);

/* design_input (hankel.hpp:44, hankel.cpp:93-99) at n lambdas, on the device */
int emie_cu_design_input(int n, const double* h_lam, double* h_out);

/* kernel_output (hankel.hpp:48) for a pair geometry {r, p, q, phi} */
int emie_cu_kernel_output_geom(const double* geom, int alpha, int beta, const double* h_s, int n, double* h_out);

/* assemble_block_full (greens.hpp:139-141, greens.cpp:231-293) at one signed
 * offset: device filter design, the moment tables of both gammas at the
 * offset's lattice, nine independent filter sums (lower triangles and the
 * source-side z couplings evaluated, not mirrored): h_out[9][nz][nz] complex,
 * q = 3a + b row-major (FullBlock). out_of_range outside the grid. */
int emie_cu_assemble_block_full(int L, const double* tops, const double* sigma, int nz, const double* breaks,
                                int nx, int ny, double hx, double hy, double omega, const double* filter,
                                int oi, int oj, double* h_out);

/* v_functions (include/emie/layered.hpp:108-114, src/layered.cpp:397-408)
 * of every interval pair at n given lambdas, as the device Green's build
 * evaluates them inside its filter sums (the same layer-state, interval-factor,
 * prefix-product and pair code as the build; greens.cpp:167-191 combinations):
 * h_out[t][4][nz][nz] complex = V1, V1 + V3, V2 + V5 (upper triangle k <= kp,
 * lower entries 0) and V4 (every k, kp). Pins the lambda accumulation's inputs
 * against the reference's moment tables (test_layered.cpp:362-401). */
int emie_cu_vfunctions(int L, const double* tops, const double* sigma, int nz, const double* breaks,
                       double omega, int n, const double* h_lam, double* h_out);

/* dense_reference_apply (include/emie/toeplitz.hpp:47, src/toeplitz.cpp:285-312):
 * the O(N^2) direct block-Toeplitz apply of host compressed blocks (the
 * emie_cu_operator_from_blocks layout) to one host field, on the device, in a
 * fixed summation order; the oracle the reference tests the FFT apply against */
int emie_cu_dense_apply(int nx, int ny, int nz, const double* h_blocks, const double* h_in, double* h_out);

/* ---- receivers (SPEC.md receiver_green_integrals, reconstruct_fields; the
 * reference leaves them as placeholders, src/receiver.cpp:1). For a receiver
 * M outside the anomaly and a cell: int_cell G^E(M, M0) dM0 and int_cell
 * G^H(M, M0) dM0 of paper Appendix A (Eq. geh, Ge2), with one-sided lateral
 * digital filters (point observer, source rectangle: designed on the device
 * like the cell-pair filters) and the receiver's vertical single moments
 * (point_moments). Receivers inside or on the closed anomaly volume are
 * rejected (EMIE_CU_INVALID_ARGUMENT). */

/* anomalous fields sum_n (sigma_a - sigma_b) E_n int_n G dOmega of nrhs CIE
 * solutions h_U (E_n = U_n / a_n, SPEC.md): h_rec[nrec][3] = (x, y, z) [m],
 * grid origin (x0, y0); h_out[rec][rhs][6] complex = E xyz, H xyz (add the
 * normal field for the total field) */
int emie_cu_receiver_fields(int L, const double* tops, const double* sigma, int nz, const double* breaks, int nx,
                            int ny, double hx, double hy, double x0, double y0, double omega, const double* filter,
                            const double* h_sigma_a, int nrhs, const double* h_U, int nrec, const double* h_rec,
                            double* h_out);

/* the tensors themselves for one receiver h_rec[3] and the cells of column
 * (ix, iy): h_out[k][18] complex = G^E (row-major 3x3, row = field component)
 * then G^H */
int emie_cu_receiver_tensors(int L, const double* tops, const double* sigma, int nz, const double* breaks, int nx,
                             int ny, double hx, double hy, double x0, double y0, double omega, const double* filter,
                             const double* h_rec, int ix, int iy, double* h_out);

/* ---- layered-medium API on the device (include/emie/layered.hpp), the
 * building blocks of the Green's build evaluated at caller-given lambdas
 * and depths. A spectral state is 9 arrays of L+1 complex, in the order
 * sig eta p q one_p one_q e2l em1_2l diag_a (SpectralLayerState,
 * layered.hpp:41-58); gamma 0 = Gamma::unit, 1 = Gamma::cond. */

/* build_spectral_state (layered.hpp:56-57, layered.cpp:67-129) at n lambdas,
 * both gammas: h_out[t][gamma][9][L+1] complex */
int emie_cu_spectral_states(int L, const double* tops, const double* sigma, double omega, int n,
                            const double* h_lam, double* h_out);

/* vertical_moment_tables (layered.hpp:97-103, layered.cpp:222-395) for the
 * partition breaks[nz+1] at n lambdas: h_out[t][gamma][6][nz][nz] complex, pair
 * order (0,0) (1,0) (0,1) (1,1) (2,0) (0,2), row-major (VerticalMomentTable::w) */
int emie_cu_moment_tables(int L, const double* tops, const double* sigma, int nz, const double* breaks,
                          double omega, int n, const double* h_lam, double* h_out);

/* fundamental_value (layered.hpp:60-66, layered.cpp:140-189) of one spectral
 * state at n point pairs: h_ord[4i..4i+3] = dz, dzs, layer_z, layer_zs
 * (-1: layer of the point) */
int emie_cu_fundamental_values(int L, const double* tops, const double* h_state, int gamma, int n,
                               const double* h_z, const double* h_zs, const int* h_ord, double* h_out);

/* point_moments (layered.hpp:116-126, layered.cpp:450-542) at n observation
 * depths for the partition breaks[nz+1] with interval layers layer[nz]:
 * h_out[t][2][nz] complex (m[0], m[1]) */
int emie_cu_point_moments(int L, const double* tops, const double* h_state, int gamma, int nz,
                          const double* breaks, const int* layer, int n, const double* h_zobs, double* h_out);

void emie_cu_operator_destroy(emie_cu_operator op);

/* apply(const SpectralOperator&, const GridVector&) (toeplitz.hpp:43,
 * src/toeplitz.cpp:163-283) on nrhs device fields; d_out may not alias d_in */
int emie_cu_apply_spectral(emie_cu_operator op, const double* d_in, double* d_out,
                           int nrhs, void* stream);

/* same, host fields in and out (H2D, apply, D2H inside the call) */
int emie_cu_apply_spectral_host(emie_cu_operator op, const double* h_in, double* h_out,
                                int nrhs, void* stream);

/* ---------------------------------------------------------------------
 * System operator A = S + R1 B R2 (include/emie/cie.hpp:26-39)
 * ------------------------------------------------------------------- */

/* build_system (cie.hpp:36-37, src/cie.cpp:24-54): per-cell contrast
 * coefficients (cie.cpp:9-22) from the host conductivities sigma_a
 * [(iz*ny + iy)*nx + ix] and sigma_b[iz] (complex) and the cell volumes
 * volume[iz] = hx*hy*dz (greens.hpp:35). The system references (does not
 * own) op; op must outlive it (cie.hpp:26-34). */
int emie_cu_system_create(emie_cu_operator op, const double* h_sigma_a,
                          const double* h_sigma_b, const double* h_volume,
                          emie_cu_system* out);
/* s (complex), r1 (real), r2 (complex) per cell, as SystemOperator holds them */
int emie_cu_system_download(emie_cu_system sys, double* h_s, double* h_r1, double* h_r2);
void emie_cu_system_destroy(emie_cu_system sys);

/* apply(const SystemOperator&, const GridVector&) (cie.hpp:39, cie.cpp:56-73) */
int emie_cu_apply_system(emie_cu_system sys, const double* d_in, double* d_out,
                         int nrhs, void* stream);

/* same, host buffers in and out: H2D, apply, D2H inside the call (the
 * reference-facing plugin call; used for the end-to-end measurement) */
int emie_cu_apply_system_host(emie_cu_system sys, const double* h_in, double* h_out,
                              int nrhs, void* stream);

/* ---------------------------------------------------------------------
 * Solve (include/emie/cie.hpp:41-80, src/cie.cpp:117-249)
 * ------------------------------------------------------------------- */

/* SolveReport (cie.hpp:43-48): status 0 converged, 1 max_iterations,
 * 2 breakdown (SolveStatus order) */
typedef struct {
  int status;
  int iterations;
  double residual;
  int history_len; /* entries written to the history buffer */
} emie_cu_report;

/* fgmres (cie.hpp:71-72, cie.cpp:117-238) with A = apply(sys, .), no
 * preconditioner, nrhs independent right-hand sides solved in lockstep
 * (they share every operator read). d_rhs, d_x: nrhs device fields; reports
 * nrhs entries; history: nrhs x hist_cap relative residuals (may be NULL). */
int emie_cu_fgmres(emie_cu_system sys, const double* d_rhs, double* d_x, int nrhs,
                   double tol, int restart, int max_iters, emie_cu_report* reports,
                   double* h_history, int hist_cap, void* stream);

/* Stage profiling: when enabled, every apply brackets its kernels with CUDA
 * events on the launching stream (stages: 0 fwd-x FFT, 1 fwd-y FFT,
 * 2 contraction, 3 inv-y FFT, 4 inv-x FFT + epilogue). collect synchronises
 * the recorded events and returns per-stage total milliseconds and launch
 * counts (arrays of n entries) since the last collect. */
int emie_cu_profile_enable(int on);
int emie_cu_profile_collect(double* ms, long long* count, int n);

/* FP64 throughput probe: the larger of a DFMA-bound and a DMMA-bound
 * (mma.sync m8n8k4 f64) kernel on the device, TFLOP/s (denominator of the
 * FP64 roofline, which MEASURED_PEAKS.json does not carry) */
int emie_cu_probe_fp64(double* tflops, void* stream);

/* live iteration hook (SolverConfig::on_iteration, cie.hpp:52, 58): called
 * with the right-hand side index, the iteration count and the residual
 * estimate exactly where the reference calls it (cie.cpp:178-185, 199-201) */
typedef void (*emie_cu_iter_fn)(void* ctx, int rhs, int iteration, double residual);

/* a linear map or preconditioner for emie_cu_fgmres_map: out = A(in), n complex
 * entries; returns 0 or a nonzero status code (the solve stops with that status) */
typedef int (*emie_cu_map_fn)(void* ctx, const double* in, double* out, long long n, void* stream);

/* emie_cu_fgmres / emie_cu_fgmres_host with the live iteration hook (hook may be NULL) */
int emie_cu_fgmres_ex(emie_cu_system sys, const double* d_rhs, double* d_x, int nrhs, double tol,
                      int restart, int max_iters, emie_cu_report* reports, double* h_history,
                      int hist_cap, emie_cu_iter_fn hook, void* hook_ctx, void* stream);
int emie_cu_fgmres_host_ex(emie_cu_system sys, const double* h_rhs, double* h_x, int nrhs, double tol,
                           int restart, int max_iters, emie_cu_report* reports, double* h_history,
                           int hist_cap, emie_cu_iter_fn hook, void* hook_ctx, void* stream);

/* fgmres(const LinearMap&, rhs, SolverConfig) (cie.hpp:71-72, cie.cpp:117-238)
 * over a caller-supplied map: the Krylov basis, the CGS2 orthogonalisation and
 * every vector operation stay on the device, the map (and the optional
 * flexible right preconditioner, SolverConfig::right_precond) is called once
 * per step. host_vectors != 0: rhs, x and the callbacks' vectors are host
 * memory (the library stages them); else device memory, the callbacks run
 * stream-ordered on `stream`. One right-hand side; report/history as
 * emie_cu_fgmres. */
int emie_cu_fgmres_map(long long n, int host_vectors, emie_cu_map_fn apply, void* apply_ctx,
                       emie_cu_map_fn precond, void* precond_ctx, emie_cu_iter_fn hook, void* hook_ctx,
                       const double* rhs, double* x, double tol, int restart, int max_iters,
                       emie_cu_report* report, double* h_history, int hist_cap, void* stream);

/* same with host right-hand sides and solutions */
int emie_cu_fgmres_host(emie_cu_system sys, const double* h_rhs, double* h_x, int nrhs,
                        double tol, int restart, int max_iters, emie_cu_report* reports,
                        double* h_history, int hist_cap, void* stream);

/* ---- sharded apply (one grid over G GPUs) -------------
 * apply(SystemOperator) (src/cie.cpp:56-73 over src/toeplitz.cpp:163-283)
 * split at its contraction: each rank transforms its depth slab (all three
 * components of intervals [z0, z1)), two all-to-alls (the caller's NCCL
 * plumbing, paper_1512_06126_b200/distributed.py) move spectrum columns
 * between the slab layout and the rank's quadrant-mode shard, and the rank
 * contracts only its modes. Spectrum layout S[r][m][plane], mode m =
 * mx*ey + my, plane = c*nz + iz (nz of the slab for slab spectra). */

/* lateral geometry (plans, twiddles) of an nx x ny x nz field, no spectra */
int emie_cu_geometry_create(int nx, int ny, int nz, emie_cu_operator* out);

/* a copy of op holding only quadrant modes [q0, q1) (a mode shard) */
int emie_cu_operator_restrict_modes(emie_cu_operator op, int q0, int q1, emie_cu_operator* out);

/* octant work for a mode shard (no reference counterpart: the reference has
 * one process, toeplitz.cpp:197-258 reads every quadrant mode). For an
 * x <-> y symmetric operator (emie_cu_operator_xy_symmetry) whose shard is
 * whole rows of quadrant modes (q0, q1 multiples of qx), enable = 1 makes
 * emie_cu_contract_modes / emie_cu_contract_modes_peer over the shard's range
 * contract its octant rows: each block (qmy, qmx <= qmy) is read once and
 * applied to that mode's columns and to the transposed mode's (qmx, qmy),
 * so the caller's spectrum must hold the columns of every quadrant mode
 * whose larger index is one of the shard's rows (distributed.ShardPlan with
 * octant=True). Errors: INVALID_ARGUMENT when the operator is not symmetric
 * or the shard not row-aligned. *out (optional) = the resulting state. */
int emie_cu_operator_shard_octant(emie_cu_operator op, int enable, int* out);

/* the full modes m = mx*ey + my of quadrant modes [q0, q1) in contraction
 * order (each quadrant mode's 1-4 mirrors); *count = total, at most cap written */
int emie_cu_mode_list(emie_cu_operator op, int q0, int q1, int* h_modes, int cap, int* count);

/* stage 1 (toeplitz.cpp:169-195, r2 scaling cie.cpp:63-65 if d_r2 != NULL):
 * zero-padded forward 2-D DFT of every plane into mode-major d_S */
int emie_cu_lateral_forward(emie_cu_operator geom, const double* d_in, const double* d_r2, double* d_S,
                            int nrhs, void* stream);

/* stage 3 (toeplitz.cpp:260-282; with d_s, d_r1: the system epilogue
 * s*u + r1*(.) of cie.cpp:67-72 on d_u): inverse 2-D DFT, truncation, 1/(ex ey) */
int emie_cu_lateral_inverse(emie_cu_operator geom, const double* d_S, const double* d_u, double* d_out,
                            const double* d_s, const double* d_r1, int nrhs, void* stream);

/* stage 2 (toeplitz.cpp:197-258) for quadrant modes [q0, q1), in place on the
 * full-depth spectrum d_S (all modes' storage, only these modes touched) */
int emie_cu_contract_modes(emie_cu_operator op, double* d_S, int nrhs, int q0, int q1, void* stream);

/* ---- sharded Green's build (SURVEY.md §8(e).3 "Green's build sharding:
 * offsets are independent"): assemble_operator (greens.cpp:332-371) split
 * over ranks by offset, the per-offset work (filter design, lambda
 * accumulation: greens.cpp:133-221) being the dominant cost. Each rank
 * computes its range of the build's computed offsets into a zeroed
 * full-size block array; the caller sums the arrays across ranks (every
 * offset is written by exactly one rank, so the sum is exact); every rank
 * then runs the mirror and transform_operator (toeplitz.cpp:92-161) for its
 * own quadrant-mode shard only. */

/* the offsets oi*nx + oj a build computes (all, or oi <= oj on a square
 * grid with hx == hy, the rest being mirrors); *count = their number */
int emie_cu_greens_offsets(int nx, int ny, double hx, double hy, int* h_offs, int cap, int* count);

/* blocks of computed offsets [c0, c1) into d_blocks (nx*ny*2nz(2nz+1)
 * complex, offset-major GreensBlock order; other offsets untouched) */
int emie_cu_greens_blocks(int L, const double* tops, const double* sigma, int nz, const double* breaks, int nx,
                          int ny, double hx, double hy, double omega, const double* filter, int c0, int c1,
                          double* d_blocks, void* stream);

/* the operator of quadrant modes [q0, q1) (q1 < 0: all) from the summed
 * blocks of every computed offset (d_blocks is completed in place by the
 * mirror) */
int emie_cu_operator_from_greens_blocks(int nx, int ny, int nz, double omega, double hx, double hy,
                                        double* d_blocks, int q0, int q1, emie_cu_operator* out, void* stream);

/* ---- sharded FGMRES vector operations ("FGMRES on
 * depth-sharded vectors: local partial dots, then an all-reduce"). The
 * vector kernels of src/cie.cpp:77-98 (dot, norm, axpy, scaled) as batched
 * CGS2 sweeps over this rank's slab; every reduction is the rank's local sum,
 * finalized on the device (fixed order) for the caller to all-reduce. Vectors
 * are complex128 of n entries, basis vector l at d_V + 2*l*vstride doubles. */

/* d_out[2l], d_out[2l+1] = sum conj(V_l) . w (l < nv); d_out[2nv] = |w|^2 if with_norm */
int emie_cu_vec_dots(const double* d_V, long long vstride, int nv, const double* d_w, long long n,
                     int with_norm, double* d_out, void* stream);

/* w -= sum_l h_l V_l (d_h: nv complex); then optionally (at most one of)
 * d_dots_out = conj(V_l) . w_new (2nv doubles) or d_norm_out = |w_new|^2 */
int emie_cu_vec_update(double* d_w, const double* d_V, long long vstride, int nv, const double* d_h,
                       long long n, double* d_dots_out, double* d_norm_out, void* stream);

/* DCGS2 step on the slab (the single-GPU solver's sweeps): dots sweep,
 * d_out (4nv doubles) = [conj(V_l) . w, l < nv][|w|^2][conj(V_l) . V_{nv-1},
 * l < nv-1][|V_{nv-1}|^2]; 1 <= nv <= 41 */
int emie_cu_vec_dcgs_dots(const double* d_V, long long vstride, int nv, const double* d_w, long long n,
                          double* d_out, void* stream);
/* DCGS2 update sweep from the caller's global coefficients d_coef =
 * [h (nv complex)][a (nv-1 complex)][1/alpha]: V_{nv-1} <- (V_{nv-1} -
 * sum a_l V_l) / alpha in place, w <- w - sum_{l<nv-1} h_l V_l - h_{nv-1}
 * V_{nv-1}(new); d_norm_out[0] = |w_new|^2 (local) */
int emie_cu_vec_dcgs_update(double* d_w, double* d_V, long long vstride, int nv, const double* d_coef, long long n,
                            double* d_norm_out, void* stream);

/* x += sum_l y_l V_l in l order (cie.cpp:213-214), d_y: nv complex */
int emie_cu_vec_combine(double* d_x, const double* d_V, long long vstride, int nv, const double* d_y,
                        long long n, void* stream);

/* y = a x (real a) */
int emie_cu_vec_scale(double* d_y, const double* d_x, double a, long long n, void* stream);

/* r = b - t; d_norm_out[0] = |r|^2 (cie.cpp:217-229) */
int emie_cu_vec_residual(double* d_r, const double* d_b, const double* d_t, long long n,
                         double* d_norm_out, void* stream);

/* column moves between slab spectra, full-depth spectra and packed exchange
 * buffers: element (r, i, c, z), i < nidx, c < 3, z < nzh, goes from
 * src[(mode_s)*desc[1] + c*desc[2] + desc[3] + z] to the same form in dst,
 * with mode = r*modes_total + d_idx[i] when desc[0] != 0 ("mapped") and
 * r*nidx + i otherwise ("packed") */
int emie_cu_move_planes(const double* d_src, double* d_dst, int nrhs, int nidx, const int* d_idx,
                        long long modes_total, const int src_desc[4], const int dst_desc[4], int nzh,
                        void* stream);

/* ---------------------------------------------------------------------
 * Peer-memory exchange of the sharded apply (replaces the
 * pack / all-to-all / unpack of the column transposes: a rank's
 * emie_cu_move_planes writes straight into the destination rank's buffer
 * over NVLink). No reference equivalent (the reference is single-node CPU).
 * ------------------------------------------------------------------- */

/* exchange buffer shareable through CUDA IPC (plain cudaMalloc, zeroed) */
int emie_cu_peer_alloc(size_t bytes, void** d_ptr);
int emie_cu_peer_free(void* d_ptr);
/* 64-byte IPC handle of a peer buffer / map a peer's buffer into this
 * process (peer access enabled lazily) / unmap it */
int emie_cu_ipc_handle(const void* d_ptr, void* h_handle);
int emie_cu_ipc_open(const void* h_handle, void** d_ptr);
int emie_cu_ipc_close(void* d_ptr);
/* emie_cu_lateral_forward of a depth slab (geometry nz = the slab's) fused
 * with the forward transpose: mode m's spectrum column goes straight into
 * the full-depth spectrum of rank d_owner[m] (device table over the ex*ey
 * modes), at h_dst[owner][(r*E + m)*3nz_full + c*nz_full + z_offset + z];
 * 256/512-point embeddings (emie_cu_lateral_forward_peer_supported) */
int emie_cu_lateral_forward_peer(emie_cu_operator geom, const double* d_in, const double* d_r2,
                                 const int* d_owner, double* const* h_dst, int G, int nz_full, int z_offset,
                                 int nrhs, void* stream);
int emie_cu_lateral_forward_peer_supported(emie_cu_operator geom, int* out);
/* emie_cu_lateral_forward_peer with the owners given by the shard plan's
 * G + 1 splits (host ints) instead of a per-mode table: octant = 1, rank g
 * owns the quadrant modes whose larger index lies in rows [split[g],
 * split[g+1]) (split[G] = qy); octant = 0, quadrant modes [split[g],
 * split[g+1]) (split[G] = qx qy). The owner is then computed on the store
 * path, no table load per element. */
int emie_cu_lateral_forward_peer_split(emie_cu_operator geom, const double* d_in, const double* d_r2,
                                       const int* h_split, int octant, double* const* h_dst, int G, int nz_full,
                                       int z_offset, int nrhs, void* stream);
/* emie_cu_contract_modes with the results stored straight into the slab
 * owners' spectra (fused contraction + return transpose; DMMA layouts, nz in
 * {8, 16, 32, 48, 64}): the contracted plane a*nz + k of mode m goes to rank h with
 * h_z[h] <= k < h_z[h+1], at h_dst[h][(r*E + m)*3nzh + a*nzh + k - h_z[h]]
 * (nzh = h_z[h+1] - h_z[h]); d_S is read only */
int emie_cu_contract_modes_peer(emie_cu_operator op, const double* d_S, int nrhs, int q0, int q1,
                                double* const* h_dst, const int* h_z, int G, void* stream);
/* after this stream's moves into the G ranks' buffers: release-store epoch
 * into slot `me` of each rank's flag array (h_flag_ptrs: G device pointers,
 * peers' flag arrays mapped into this process) */
int emie_cu_peer_signal(int* const* h_flag_ptrs, int G, int me, int epoch, void* stream);
/* before this stream reads its buffer: wait until all G slots of d_flags
 * reach epoch (bounded: after ~30 s without a peer's signal the wait gives
 * up and sets a sticky timeout flag; later waits return at once) */
int emie_cu_peer_wait(const int* d_flags, int G, int epoch, void* stream);
/* synchronise the device, then report (*timed_out = 1) and clear the sticky
 * timeout flag of the peer waits: a sharded apply whose exchange timed out
 * produced no valid result */
int emie_cu_peer_status(int* timed_out);

/* kernel launches issued by this library on the calling thread since the
 * last reset (evidence for bench.py's gpu_launches) */
long long emie_cu_launch_count(void);
void emie_cu_reset_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* EMIE_CU_H */
