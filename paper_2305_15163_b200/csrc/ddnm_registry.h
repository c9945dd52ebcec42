// Registry of compiled kernel specialisations (one inst_<ni>_<ng>.cu each).
#pragma once
#include <vector>

namespace ddnm {
struct KernelEntry {
  int ni, ng, g;
  bool kkt_global;       // KKT workspace in global memory (kernels with KG = true)
  const void* solve;
  const void* eval;
  const void* dd_eval;   // subdomain-sharded round kernels
  const void* dd_step;
  const void* dd_step2 = nullptr;   // two CTAs per SM (batch-wide solve), or null
};
}  // namespace ddnm
