// forest.cu — K2 (tree-ensemble predictor, forest.hpp:80-85, 176-180, 227-235).
// Round-1 placeholder: the entry point exists so the ABI is complete; the
// cell-table kernel lands next.
#include "pals_internal.cuh"

namespace pals {

void forest_free(void*) {}

int forest_eval_plan(pals_plan*, const pals_model*, pals_ctx*) {
    return set_error(PALS_ECONFIG, "pals: forest models are not built yet");
}

}  // namespace pals

using namespace pals;

extern "C" int pals_model_forest(pals_ctx*, int32_t, int32_t, const pals_coeffs*, int32_t,
                                 const int64_t*, const int32_t*, const double*, const int32_t*,
                                 const int32_t*, const double*, int32_t, const int64_t*,
                                 const int32_t*, const double*, const int32_t*, const int32_t*,
                                 const double*, pals_model**) {
    return set_error(PALS_ECONFIG, "pals: forest models are not built yet");
}
