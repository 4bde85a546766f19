// k_apply_lo.cu -- instantiations of K2 (apply_kernel) for depths {1, 2, 3, 4, 5}.
#include "dispatch.h"

namespace obt {

template <int DI, int CMP, int DSRC>
static ApplyKernel apply_leaf(int leaf, bool write_idx) {
  ApplyKernel k;
  k.dsrc = DSRC;
  k.words = 1;
  if (write_idx) k.fn = (const void*)apply_kernel<DI, CMP, 1, true, 1, DSRC>;
  else if (leaf == 0) k.fn = (const void*)apply_kernel<DI, CMP, 0, false, 1, DSRC>;
  else if (leaf == 1) k.fn = (const void*)apply_kernel<DI, CMP, 1, false, 1, DSRC>;
  else if (leaf == 2) k.fn = (const void*)apply_kernel<DI, CMP, 2, false, 1, DSRC>;
  // 3 / 4: shuffle "permute" leaf selection of binary16 (depth <= 6) / binary32 (depth <= 5)
  else if constexpr (DI <= 6) {
    if (leaf == 3) k.fn = (const void*)apply_kernel<DI, CMP, 3, false, 1, DSRC>;
    else if constexpr (DI <= 5) k.fn = (const void*)apply_kernel<DI, CMP, 4, false, 1, DSRC>;
  }
  return k;
}

template <int DI>
static ApplyKernel apply_di(int cmp, int leaf, bool write_idx, int dsrc) {
  // parameter-bank descriptors exist for the 7-bit compare only
  if (cmp == 7) return dsrc ? apply_leaf<DI, 7, 1>(leaf, write_idx) : apply_leaf<DI, 7, 0>(leaf, write_idx);
  return apply_leaf<DI, 8, 0>(leaf, write_idx);
}

ApplyKernel pick_apply_lo(int di, int cmp, int leaf, bool write_idx, int dsrc) {
  switch (di) {
    case 1: return apply_di<1>(cmp, leaf, write_idx, dsrc);
    case 2: return apply_di<2>(cmp, leaf, write_idx, dsrc);
    case 3: return apply_di<3>(cmp, leaf, write_idx, dsrc);
    case 4: return apply_di<4>(cmp, leaf, write_idx, dsrc);
    case 5: return apply_di<5>(cmp, leaf, write_idx, dsrc);
    default: return ApplyKernel{};
  }
}

}  // namespace obt
