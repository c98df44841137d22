// emie-b200 drop-in: lateral spectra and the block-Toeplitz apply
// (reference: include/emie/toeplitz.hpp:13-48). SpectralOperator keeps the
// reference's public fields (comp is materialised on the host) and adds a
// handle to the device-resident copy that apply() uses.
#pragma once

#include <array>
#include <cstddef>
#include <memory>
#include <vector>

#include "emie/greens.hpp"
#include "emie/types.hpp"

namespace emie {

int smooth_embedding_size(int n);

struct DeviceOperator;  // opaque: owns an emie_cu_operator

struct SpectralOperator {
  int nx = 0, ny = 0, nz = 0;
  int ex = 0, ey = 0;
  int qx = 0, qy = 0;
  double omega = 0.0;
  std::array<std::vector<cdouble>, 6> comp;  // xx yy zz xy | xz yz, mode-major
  std::shared_ptr<DeviceOperator> device;    // created on first use if absent

  std::size_t mode_count() const { return std::size_t(qx) * qy; }
  std::size_t stored_complex_count() const;
};

SpectralOperator transform_operator(const CompressedGreensOperator& op);
GridVector apply(const SpectralOperator& sop, const GridVector& v);
GridVector dense_reference_apply(const CompressedGreensOperator& op, const GridVector& v);

}  // namespace emie
