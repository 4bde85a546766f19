// k_apply_hi.cu -- instantiations of K2 (apply_kernel) for depths {6, 7, 8, 10, 12}.
#include <cstdlib>

#include "dispatch.h"

namespace obt {

// bucket words (4 objects each) per apply thread: 1, or 2 (8 objects per thread: half
// the threads, each with twice the independent work); OBT_WORDS_PER_THREAD overrides
static int words_per_thread() {
  static const int w = [] {
    const char* e = getenv("OBT_WORDS_PER_THREAD");
    return (e && atoi(e) == 2) ? 2 : 1;
  }();
  return w;
}

template <int DI, int CMP, int DSRC, int W>
static ApplyKernel apply_leaf_w(int leaf, bool write_idx) {
  ApplyKernel k;
  k.dsrc = DSRC;
  k.words = W;
  if (write_idx) k.fn = (const void*)apply_kernel<DI, CMP, 1, true, W, DSRC>;
  else if (leaf == 0) k.fn = (const void*)apply_kernel<DI, CMP, 0, false, W, DSRC>;
  else if (leaf == 1) k.fn = (const void*)apply_kernel<DI, CMP, 1, false, W, DSRC>;
  else k.fn = (const void*)apply_kernel<DI, CMP, 2, false, W, DSRC>;
  return k;
}

template <int DI, int CMP, int DSRC>
static ApplyKernel apply_leaf(int leaf, bool write_idx) {
  if constexpr (DSRC == 1) {
    return apply_leaf_w<DI, CMP, 1, 1>(leaf, write_idx);
  } else {
    return words_per_thread() == 2 && !write_idx ? apply_leaf_w<DI, CMP, DSRC, 2>(leaf, write_idx)
                                                 : apply_leaf_w<DI, CMP, DSRC, 1>(leaf, write_idx);
  }
}

template <int DI>
static ApplyKernel apply_di(int cmp, int leaf, bool write_idx, int dsrc) {
  // parameter-bank descriptors exist for the 7-bit compare only
  if (cmp == 7) return dsrc ? apply_leaf<DI, 7, 1>(leaf, write_idx) : apply_leaf<DI, 7, 0>(leaf, write_idx);
  return apply_leaf<DI, 8, 0>(leaf, write_idx);
}

ApplyKernel pick_apply_hi(int di, int cmp, int leaf, bool write_idx, int dsrc) {
  switch (di) {
    case 6: return apply_di<6>(cmp, leaf, write_idx, dsrc);
    case 7: return apply_di<7>(cmp, leaf, write_idx, dsrc);
    case 8: return apply_di<8>(cmp, leaf, write_idx, dsrc);
    case 10: return apply_di<10>(cmp, leaf, write_idx, dsrc);
    case 12: return apply_di<12>(cmp, leaf, write_idx, dsrc);
    default: return ApplyKernel{};
  }
}

}  // namespace obt
