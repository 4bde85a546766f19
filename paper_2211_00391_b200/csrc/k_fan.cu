// k_fan.cu -- instantiations of K2f (apply_fan_kernel): depths 1..8 x {7-, 8-bit compare}
// x {binary64, binary32, binary16} leaf storage.
#include "dispatch.h"

namespace obt {

template <int DI, int CMP>
static const void* fan_leaf(int leaf) {
  if (leaf == 0) return (const void*)apply_fan_kernel<DI, CMP, 0>;
  if (leaf == 1) return (const void*)apply_fan_kernel<DI, CMP, 1>;
  return (const void*)apply_fan_kernel<DI, CMP, 2>;
}

template <int DI>
static const void* fan_di(int cmp, int leaf) {
  return cmp == 7 ? fan_leaf<DI, 7>(leaf) : fan_leaf<DI, 8>(leaf);
}

const void* pick_fan(int di, int cmp, int leaf) {
  switch (di) {
    case 1: return fan_di<1>(cmp, leaf);
    case 2: return fan_di<2>(cmp, leaf);
    case 3: return fan_di<3>(cmp, leaf);
    case 4: return fan_di<4>(cmp, leaf);
    case 5: return fan_di<5>(cmp, leaf);
    case 6: return fan_di<6>(cmp, leaf);
    case 7: return fan_di<7>(cmp, leaf);
    case 8: return fan_di<8>(cmp, leaf);
    default: return nullptr;
  }
}

}  // namespace obt
