// Kernel specialisations for latent dims (n_int, n_gam) = (4, 3).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_4_3(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{4, 3, 1, (const void*)&k_solve<1, 4, 3>,
                          (const void*)&k_eval<1, 4, 3>});
  t.push_back(KernelEntry{4, 3, 2, (const void*)&k_solve<2, 4, 3>,
                          (const void*)&k_eval<2, 4, 3>});
}
}  // namespace ddnm
