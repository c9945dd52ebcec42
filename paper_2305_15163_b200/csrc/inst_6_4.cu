// Kernel specialisations for latent dims (n_int, n_gam) = (6, 4).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_6_4(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{6, 4, 1, false, (const void*)&k_solve<1, 6, 4, false>,
                          (const void*)&k_eval<1, 6, 4, false>,
                          (const void*)&k_dd_eval<1, 6, 4>,
                          (const void*)&k_dd_step<1, 6, 4, false>});
  t.push_back(KernelEntry{6, 4, 2, false, (const void*)&k_solve<2, 6, 4, false>,
                          (const void*)&k_eval<2, 6, 4, false>,
                          (const void*)&k_dd_eval<2, 6, 4>,
                          (const void*)&k_dd_step<2, 6, 4, false>});
  t.push_back(KernelEntry{6, 4, 3, false, (const void*)&k_solve<3, 6, 4, false>,
                          (const void*)&k_eval<3, 6, 4, false>,
                          (const void*)&k_dd_eval<3, 6, 4>,
                          (const void*)&k_dd_step<3, 6, 4, false>});
  t.push_back(KernelEntry{6, 4, 4, false, (const void*)&k_solve<4, 6, 4, false>,
                          (const void*)&k_eval<4, 6, 4, false>,
                          (const void*)&k_dd_eval<4, 6, 4>,
                          (const void*)&k_dd_step<4, 6, 4, false>,
                          (const void*)&k_dd_step2<4, 6, 4, false>});
}
}  // namespace ddnm
