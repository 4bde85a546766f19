// k_multi.cu -- instantiations of K4 (apply_multi_kernel): depths {4, 6, 8, 10, 12}
// (shallower models run padded with sentinel splits) x output counts {2..16}.
#include "dispatch.h"

namespace obt {

int multi_depth(int d) {
  if (d <= 4) return 4;
  if (d <= 6) return 6;
  if (d <= 8) return 8;
  if (d <= 10) return 10;
  if (d <= 12) return 12;
  return -1;
}

template <int DI, int CMP, int LEAF>
static const void* multi_c(int c) {
  switch (c) {
#define OBT_C(n) case n: return (const void*)apply_multi_kernel<DI, CMP, LEAF, n>;
    OBT_C(2) OBT_C(3) OBT_C(4) OBT_C(5) OBT_C(6) OBT_C(7) OBT_C(8) OBT_C(9) OBT_C(10)
    OBT_C(11) OBT_C(12) OBT_C(13) OBT_C(14) OBT_C(15) OBT_C(16)
#undef OBT_C
    default: return nullptr;
  }
}

template <int DI>
static const void* multi_di(int cmp, int leaf, int c) {
  if (cmp == 7) return leaf == 0 ? multi_c<DI, 7, 0>(c) : multi_c<DI, 7, 1>(c);
  return leaf == 0 ? multi_c<DI, 8, 0>(c) : multi_c<DI, 8, 1>(c);
}

const void* pick_multi(int di, int cmp, int leaf, int c, int* di_out) {
  const int d = multi_depth(di);
  if (di_out) *di_out = d;
  switch (d) {
    case 4: return multi_di<4>(cmp, leaf, c);
    case 6: return multi_di<6>(cmp, leaf, c);
    case 8: return multi_di<8>(cmp, leaf, c);
    case 10: return multi_di<10>(cmp, leaf, c);
    case 12: return multi_di<12>(cmp, leaf, c);
    default: return nullptr;
  }
}

}  // namespace obt
