// Kernel specialisations for latent dims (n_int, n_gam) = (8, 5).
#include <vector>

#include "ddnm_registry.h"
#include "ddnm_solve.cuh"

namespace ddnm {
void register_8_5_more(std::vector<KernelEntry>& t);   // inst_8_5b.cu
void register_8_5(std::vector<KernelEntry>& t) {
  t.push_back(KernelEntry{8, 5, 1, false, (const void*)&k_solve<1, 8, 5, false>,
                          (const void*)&k_eval<1, 8, 5, false>,
                          (const void*)&k_dd_eval<1, 8, 5>,
                          (const void*)&k_dd_step<1, 8, 5, false>});
  t.push_back(KernelEntry{8, 5, 2, false, (const void*)&k_solve<2, 8, 5, false>,
                          (const void*)&k_eval<2, 8, 5, false>,
                          (const void*)&k_dd_eval<2, 8, 5>,
                          (const void*)&k_dd_step<2, 8, 5, false>});
  // many subdomains (16 blocks, n_C = 40: 248 x 248 KKT): KKT workspace in L2
  t.push_back(KernelEntry{8, 5, 1, true, (const void*)&k_solve<1, 8, 5, true>,
                          (const void*)&k_eval<1, 8, 5, true>,
                          (const void*)&k_dd_eval<1, 8, 5>,
                          (const void*)&k_dd_step<1, 8, 5, true>});
  register_8_5_more(t);
}
}  // namespace ddnm
