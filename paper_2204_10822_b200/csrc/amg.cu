// amg.cu — placeholder (replaced by the GPU aggregation AMG).
#include "ctx.cuh"

namespace seaice {
void amg_setup_impl(Ctx& c) { throw Error(SEAICE_EINVAL, "AMG not built yet"); }
void amg_vcycle(Ctx& c, const double* r, double* z) { throw Error(SEAICE_EINVAL, "AMG not built yet"); }
void amg_free(Ctx& c) { c.lv.clear(); }
}  // namespace seaice
