// Refinement (refine.hpp:53-332) — placeholder until the kernels land.
#include "context.h"

namespace lfdg {
void make_refine_tables(Ctx& c, const lfdg_energy_params& p, int sweep_levels) {
    (void)c; (void)p; (void)sweep_levels;
    throw Error(LFDG_STATE, "refinement not built yet");
}
void refine_iteration(Ctx& c, int l) {
    (void)c; (void)l;
    throw Error(LFDG_STATE, "refinement not built yet");
}
}  // namespace lfdg
