// k_wide.cu -- instantiations of K2w (apply_wide_kernel): depths 1..8 x {7-, 8-bit
// compare} x {binary64, binary32, binary16} leaf storage, kWideIndexWarps index warps.
#include "dispatch.h"
#include "wide_apply.cuh"

namespace obt {

template <int DI, int CMP>
static const void* wide_leaf(int leaf) {
  if (leaf == 0) return (const void*)apply_wide_kernel<DI, CMP, 0, kWideIndexWarps>;
  if (leaf == 1) return (const void*)apply_wide_kernel<DI, CMP, 1, kWideIndexWarps>;
  return (const void*)apply_wide_kernel<DI, CMP, 2, kWideIndexWarps>;
}

template <int DI>
static const void* wide_di(int cmp, int leaf) {
  return cmp == 7 ? wide_leaf<DI, 7>(leaf) : wide_leaf<DI, 8>(leaf);
}

const void* pick_wide(int di, int cmp, int leaf) {
  switch (di) {
    case 1: return wide_di<1>(cmp, leaf);
    case 2: return wide_di<2>(cmp, leaf);
    case 3: return wide_di<3>(cmp, leaf);
    case 4: return wide_di<4>(cmp, leaf);
    case 5: return wide_di<5>(cmp, leaf);
    case 6: return wide_di<6>(cmp, leaf);
    case 7: return wide_di<7>(cmp, leaf);
    case 8: return wide_di<8>(cmp, leaf);
    default: return nullptr;
  }
}

}  // namespace obt
