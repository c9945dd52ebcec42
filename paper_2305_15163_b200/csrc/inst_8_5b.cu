// More kernel specialisations for latent dims (n_int, n_gam) = (8, 5): the
// BASELINE configs 3 (480^2, 4 blocks as ~115 evaluation units, n_C = 10)
// and 4 (960^2, 16 blocks as ~600 units, n_C = 40: KKT workspace and, by the
// planner's choice, the evaluation buffers in L2) with 3-4 slots per CTA.
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_5_more(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 5, 4, false, (const void*)&k_solve<4, 8, 5, false>,
                          (const void*)&k_eval<4, 8, 5, false>,
                          (const void*)&k_dd_eval<4, 8, 5>,
                          (const void*)&k_dd_step<4, 8, 5, false>});
  t.push_back(KernelEntry{8, 5, 2, true, (const void*)&k_solve<2, 8, 5, true>,
                          (const void*)&k_eval<2, 8, 5, true>,
                          (const void*)&k_dd_eval<2, 8, 5>,
                          (const void*)&k_dd_step<2, 8, 5, true>});
  t.push_back(KernelEntry{8, 5, 4, true, (const void*)&k_solve<4, 8, 5, true>,
                          (const void*)&k_eval<4, 8, 5, true>,
                          (const void*)&k_dd_eval<4, 8, 5>,
                          (const void*)&k_dd_step<4, 8, 5, true>});
}
}  // namespace ddnm
