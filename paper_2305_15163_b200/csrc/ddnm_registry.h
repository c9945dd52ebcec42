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
};
}  // namespace ddnm
