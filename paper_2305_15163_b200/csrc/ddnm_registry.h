// Registry of compiled kernel specialisations (one inst_<ni>_<ng>.cu each).
#pragma once
#include <vector>

namespace ddnm {
struct KernelEntry {
  int ni, ng, g;
  const void* solve;
  const void* eval;
};
}  // namespace ddnm
