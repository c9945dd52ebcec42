// Kernel specialisations for latent dims (n_int, n_gam) = (20, 8).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_20_8(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{20, 8, 1, false, (const void*)&k_solve<1, 20, 8, false>,
                          (const void*)&k_eval<1, 20, 8, false>,
                          (const void*)&k_dd_eval<1, 20, 8>,
                          (const void*)&k_dd_step<1, 20, 8, false>});
}
}  // namespace ddnm
