// Kernel specialisations for latent dims (n_int, n_gam) = (6, 4).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_6_4(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{6, 4, 1, (const void*)&k_solve<1, 6, 4>,
                          (const void*)&k_eval<1, 6, 4>});
  t.push_back(KernelEntry{6, 4, 2, (const void*)&k_solve<2, 6, 4>,
                          (const void*)&k_eval<2, 6, 4>});
  t.push_back(KernelEntry{6, 4, 3, (const void*)&k_solve<3, 6, 4>,
                          (const void*)&k_eval<3, 6, 4>});
  t.push_back(KernelEntry{6, 4, 4, (const void*)&k_solve<4, 6, 4>,
                          (const void*)&k_eval<4, 6, 4>});
}
}  // namespace ddnm
