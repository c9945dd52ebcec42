// Kernel specialisations for latent dims (n_int, n_gam) = (8, 11): SRPC LS tiny variant (8, 11).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_11(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 11, 1, false, (const void*)&k_solve<1, 8, 11, false>,
                          (const void*)&k_eval<1, 8, 11, false>,
                          (const void*)&k_dd_eval<1, 8, 11>,
                          (const void*)&k_dd_step<1, 8, 11, false>});
}
}  // namespace ddnm
