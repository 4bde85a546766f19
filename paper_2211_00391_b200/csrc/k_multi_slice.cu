// k_multi_slice.cu -- instantiations of K4s (apply_multi_slice_kernel): depths
// {4, 6, 8, 10, 12} x output counts {2..16} x {7-, 8-bit compare} x {fp64, fp32 leaves}.
#include "dispatch.h"

namespace obt {

template <int DI, int CMP, int LEAF>
static const void* slice_c(int c) {
  switch (c) {
#define OBT_C(n) case n: return (const void*)apply_multi_slice_kernel<DI, CMP, LEAF, n>;
    OBT_C(2) OBT_C(3) OBT_C(4) OBT_C(5) OBT_C(6) OBT_C(7) OBT_C(8) OBT_C(9) OBT_C(10)
    OBT_C(11) OBT_C(12) OBT_C(13) OBT_C(14) OBT_C(15) OBT_C(16)
#undef OBT_C
    default: return nullptr;
  }
}

template <int DI>
static const void* slice_di(int cmp, int leaf, int c) {
  if (cmp == 7) return leaf == 0 ? slice_c<DI, 7, 0>(c) : slice_c<DI, 7, 1>(c);
  return leaf == 0 ? slice_c<DI, 8, 0>(c) : slice_c<DI, 8, 1>(c);
}

const void* pick_multi_slice(int di, int cmp, int leaf, int c, int* di_out) {
  const int d = multi_depth(di);
  if (di_out) *di_out = d;
  switch (d) {
    case 4: return slice_di<4>(cmp, leaf, c);
    case 6: return slice_di<6>(cmp, leaf, c);
    case 8: return slice_di<8>(cmp, leaf, c);
    case 10: return slice_di<10>(cmp, leaf, c);
    case 12: return slice_di<12>(cmp, leaf, c);
    default: return nullptr;
  }
}

// Slot bytes of one leaf record for the sliced kernel.
int multi_slice_slot(int leaf, int c) {
  if (leaf == 0) {
    const int rec = c * 8;
    return rec <= 16 ? 16 : rec <= 32 ? 32 : rec <= 64 ? 64 : 128;
  }
  const int rec = (c + 1) / 2 * 8;
  return rec <= 16 ? 16 : rec <= 32 ? 32 : rec <= 64 ? 64 : 128;
}

}  // namespace obt
