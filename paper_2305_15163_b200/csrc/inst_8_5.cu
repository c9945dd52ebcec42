// Kernel specialisations for latent dims (n_int, n_gam) = (8, 5).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_5(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 5, 1, (const void*)&k_solve<1, 8, 5>,
                          (const void*)&k_eval<1, 8, 5>});
  t.push_back(KernelEntry{8, 5, 2, (const void*)&k_solve<2, 8, 5>,
                          (const void*)&k_eval<2, 8, 5>});
}
}  // namespace ddnm
