// Kernel specialisations for latent dims (n_int, n_gam) = (8, 4).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_4(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 4, 1, false, (const void*)&k_solve<1, 8, 4, false>,
                          (const void*)&k_eval<1, 8, 4, false>,
                          (const void*)&k_dd_eval<1, 8, 4>,
                          (const void*)&k_dd_step<1, 8, 4, false>});
  t.push_back(KernelEntry{8, 4, 2, false, (const void*)&k_solve<2, 8, 4, false>,
                          (const void*)&k_eval<2, 8, 4, false>,
                          (const void*)&k_dd_eval<2, 8, 4>,
                          (const void*)&k_dd_step<2, 8, 4, false>});
}
}  // namespace ddnm
