// Green's-tensor build on the device (placeholder until the kernels land).
#include "operator.cuh"

namespace emie_cu {

void check_filter_params(const FilterParams& par) {  // hankel.cpp:205-208
  if (!(par.step > 0.0) || !(par.shift > 0.0) || !(par.shift < 0.5 * par.step))
    fail(EMIE_CU_INVALID_ARGUMENT, "filter params: need 0 < shift < step/2");
  if (par.half < 2 || par.n1 < -par.half || par.n2 <= par.n1 || par.n2 > par.half - 1)
    fail(EMIE_CU_INVALID_ARGUMENT, "filter params: bad weight window");
}

void greens_build(Operator&, int, const double*, const cplx*, const double*, double, double,
                  const FilterParams&, bool, cudaStream_t) {
  fail(EMIE_CU_RUNTIME_ERROR, "greens_build: not built yet");
}

void design_offset_filters_host(int, int, double, double, const FilterParams&, double*, double*) {
  fail(EMIE_CU_RUNTIME_ERROR, "design_offset_filters: not built yet");
}

}  // namespace emie_cu
