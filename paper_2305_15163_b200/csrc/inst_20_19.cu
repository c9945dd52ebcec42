// Kernel specialisations for latent dims (n_int, n_gam) = (20, 19): SRPC LS config-1 variant (20, 19).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_20_19(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{20, 19, 1, false, (const void*)&k_solve<1, 20, 19, false>,
                          (const void*)&k_eval<1, 20, 19, false>,
                          (const void*)&k_dd_eval<1, 20, 19>,
                          (const void*)&k_dd_step<1, 20, 19, false>});
  // 60x60 SRPC LS-ROM (n_C = 40, 196 x 196 KKT): KKT workspace in L2
  t.push_back(KernelEntry{20, 19, 1, true, (const void*)&k_solve<1, 20, 19, true>,
                          (const void*)&k_eval<1, 20, 19, true>,
                          (const void*)&k_dd_eval<1, 20, 19>,
                          (const void*)&k_dd_step<1, 20, 19, true>});
}
}  // namespace ddnm
