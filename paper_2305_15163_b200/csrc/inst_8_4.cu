// Kernel specialisations for latent dims (n_int, n_gam) = (8, 4).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_4(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 4, 1, (const void*)&k_solve<1, 8, 4>,
                          (const void*)&k_eval<1, 8, 4>});
  t.push_back(KernelEntry{8, 4, 2, (const void*)&k_solve<2, 8, 4>,
                          (const void*)&k_eval<2, 8, 4>});
}
}  // namespace ddnm
