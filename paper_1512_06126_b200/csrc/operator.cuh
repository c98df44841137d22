// Device-resident operator objects behind the C ABI (include/emie_cu.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../include/emie_cu.h"
#include "common.cuh"
#include "fft.cuh"

namespace emie_cu {

// SpectralOperator (reference include/emie/toeplitz.hpp:21-35), device side.
// Spectra layout (HBM): mode-major, one contiguous block per quadrant mode
//   spec[(my*qx + mx)*nent + e],  e over xx yy zz xy (triangles) | xz yz (full)
// i.e. the six reference components of one mode packed back to back, so the
// contraction reads each mode's 2nz(2nz+1) complex as one contiguous run.
struct Operator {
  int nx = 0, ny = 0, nz = 0;
  int ex = 0, ey = 0, qx = 0, qy = 0;
  double omega = 0.0;
  int ntri = 0, nfull = 0, nent = 0;
  cplx* spec = nullptr;      // qx*qy*nent
  cplx* blocks = nullptr;    // optional compressed blocks, (ny*nx)*nent
  cplx* tw_x = nullptr;      // e^{-2 pi i m/ex}
  cplx* tw_y = nullptr;      // e^{-2 pi i m/ey}
  uint32_t* trilut = nullptr;  // triangle slot -> (k << 16) | kp
  FftPlan plan_x, plan_y;

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
void init_operator_geometry(Operator& op, int nx, int ny, int nz, double omega);
cplx* upload_twiddles(int n);

// stages (operator.cu)
void transform_blocks(Operator& op, const cplx* d_blocks, cudaStream_t st);
void apply_b(const Operator& op, const cplx* d_in, cplx* d_out, int nrhs,
             const System* sys, cudaStream_t st);

// Green's build (greens.cu)
struct FilterParams {
  double step = 0.2, shift = 0.0964;
  int half = 512, n1 = -250, n2 = 200;
};
void check_filter_params(const FilterParams& fp);
void greens_build(Operator& op, int L, const double* tops, const cplx* sigma,
                  const double* breaks, double hx, double hy, const FilterParams& fp,
                  bool keep_blocks, cudaStream_t st);
void design_offset_filters_host(int oi, int oj, double hx, double hy, const FilterParams& fp,
                                double* w, double* lam);

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

void fgmres_device(const System& sys, const cplx* d_rhs, cplx* d_x, int nrhs, double tol,
                   int m, int max_iters, emie_cu_report* reports, double* h_history,
                   int hist_cap, cudaStream_t st);

}  // namespace emie_cu
