// k_wide.cu -- instantiations of K2w (apply_wide_kernel): depths 1..8 x {7-, 8-bit
// compare} x {binary64, binary32, binary16} leaf storage x {shared-memory ring, parameter-bank}
// descriptors, kWideIndexWarps index warps.
#include "dispatch.h"
#include "wide_apply.cuh"

namespace obt {

template <int DI, int CMP, int DSRC>
static const void* wide_leaf(int leaf) {
  if (leaf == 0) return (const void*)apply_wide_kernel<DI, CMP, 0, kWideIndexWarps, DSRC>;
  if (leaf == 1) return (const void*)apply_wide_kernel<DI, CMP, 1, kWideIndexWarps, DSRC>;
  return (const void*)apply_wide_kernel<DI, CMP, 2, kWideIndexWarps, DSRC>;
}

template <int DI>
static const void* wide_di(int cmp, int leaf, int dsrc) {
  if (dsrc) return cmp == 7 ? wide_leaf<DI, 7, 1>(leaf) : wide_leaf<DI, 8, 1>(leaf);
  return cmp == 7 ? wide_leaf<DI, 7, 0>(leaf) : wide_leaf<DI, 8, 0>(leaf);
}

const void* pick_wide(int di, int cmp, int leaf, int dsrc) {
  switch (di) {
    case 1: return wide_di<1>(cmp, leaf, dsrc);
    case 2: return wide_di<2>(cmp, leaf, dsrc);
    case 3: return wide_di<3>(cmp, leaf, dsrc);
    case 4: return wide_di<4>(cmp, leaf, dsrc);
    case 5: return wide_di<5>(cmp, leaf, dsrc);
    case 6: return wide_di<6>(cmp, leaf, dsrc);
    case 7: return wide_di<7>(cmp, leaf, dsrc);
    case 8: return wide_di<8>(cmp, leaf, dsrc);
    default: return nullptr;
  }
}

}  // namespace obt
