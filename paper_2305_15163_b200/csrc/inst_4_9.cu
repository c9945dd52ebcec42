// Kernel specialisations for latent dims (n_int, n_gam) = (4, 9): SRPC NM tiny variant (4, 9).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_4_9(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{4, 9, 1, false, (const void*)&k_solve<1, 4, 9, false>,
                          (const void*)&k_eval<1, 4, 9, false>,
                          (const void*)&k_dd_eval<1, 4, 9>,
                          (const void*)&k_dd_step<1, 4, 9, false>});
  t.push_back(KernelEntry{4, 9, 2, false, (const void*)&k_solve<2, 4, 9, false>,
                          (const void*)&k_eval<2, 4, 9, false>,
                          (const void*)&k_dd_eval<2, 4, 9>,
                          (const void*)&k_dd_step<2, 4, 9, false>});
}
}  // namespace ddnm
