// Kernel specialisations for latent dims (n_int, n_gam) = (6, 11): SRPC NM config-0 variant (6, 11).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_6_11(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{6, 11, 1, false, (const void*)&k_solve<1, 6, 11, false>,
                          (const void*)&k_eval<1, 6, 11, false>,
                          (const void*)&k_dd_eval<1, 6, 11>,
                          (const void*)&k_dd_step<1, 6, 11, false>});
  t.push_back(KernelEntry{6, 11, 2, false, (const void*)&k_solve<2, 6, 11, false>,
                          (const void*)&k_eval<2, 6, 11, false>,
                          (const void*)&k_dd_eval<2, 6, 11>,
                          (const void*)&k_dd_step<2, 6, 11, false>});
}
}  // namespace ddnm
