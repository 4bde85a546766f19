// k_split.cu -- instantiations of K2s (apply_split_kernel) and the K2 depth router.
#include "dispatch.h"

namespace obt {

ApplyKernel pick_apply_lo(int di, int cmp, int leaf, bool write_idx, int dsrc);
ApplyKernel pick_apply_hi(int di, int cmp, int leaf, bool write_idx, int dsrc);

ApplyKernel pick_apply(int di, int cmp, int leaf, bool write_idx, int dsrc) {
  return di <= 5 ? pick_apply_lo(di, cmp, leaf, write_idx, dsrc) : pick_apply_hi(di, cmp, leaf, write_idx, dsrc);
}

template <int DI, int CMP, int TPW>
static ApplyKernel split_leaf(int leaf) {
  ApplyKernel k;
  k.tpw = TPW;
  if (leaf == 0) k.fn = (const void*)apply_split_kernel<DI, CMP, 0, TPW>;
  else if (leaf == 1) k.fn = (const void*)apply_split_kernel<DI, CMP, 1, TPW>;
  else k.fn = (const void*)apply_split_kernel<DI, CMP, 2, TPW>;
  return k;
}

template <int DI, int TPW>
static ApplyKernel split_cmp(int cmp, int leaf) {
  return cmp == 7 ? split_leaf<DI, 7, TPW>(leaf) : split_leaf<DI, 8, TPW>(leaf);
}

ApplyKernel pick_split(int di, int cmp, int leaf, int tpw) {
  if (tpw == 2) {
    switch (di) {
      case 2: return split_cmp<2, 2>(cmp, leaf);
      case 4: return split_cmp<4, 2>(cmp, leaf);
      case 6: return split_cmp<6, 2>(cmp, leaf);
      case 8: return split_cmp<8, 2>(cmp, leaf);
    }
  } else if (tpw == 4) {
    switch (di) {
      case 4: return split_cmp<4, 4>(cmp, leaf);
      case 8: return split_cmp<8, 4>(cmp, leaf);
    }
  }
  return ApplyKernel{};
}

}  // namespace obt
