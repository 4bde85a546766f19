// k_multi_staged.cu -- instantiations of K5 (apply_multi_staged_kernel): depths
// {4, 6, 8, 10} x output counts {2..10} x {7-, 8-bit compare}, fp32 records.
#include "dispatch.h"

namespace obt {

template <int DI, int CMP>
static const void* staged_c(int c) {
  switch (c) {
#define OBT_C(n) case n: return (const void*)apply_multi_staged_kernel<DI, CMP, n>;
    OBT_C(2) OBT_C(3) OBT_C(4) OBT_C(5) OBT_C(6) OBT_C(7) OBT_C(8) OBT_C(9) OBT_C(10)
#undef OBT_C
    default: return nullptr;
  }
}

const void* pick_multi_staged(int di, int cmp, int c, int* di_out) {
  const int d = multi_depth(di);
  if (di_out) *di_out = d;
  switch (d) {
    case 4: return cmp == 7 ? staged_c<4, 7>(c) : staged_c<4, 8>(c);
    case 6: return cmp == 7 ? staged_c<6, 7>(c) : staged_c<6, 8>(c);
    case 8: return cmp == 7 ? staged_c<8, 7>(c) : staged_c<8, 8>(c);
    case 10: return cmp == 7 ? staged_c<10, 7>(c) : staged_c<10, 8>(c);
    default: return nullptr;
  }
}

}  // namespace obt
