// k_multi_staged.cu -- instantiations of K5 (apply_multi_staged_kernel): depths
// {4, 6, 8, 10} x output counts {1..10} x {7-, 8-bit compare} x {binary32 records
// (binary64 family), binary16 records (binary16 family)}, plus binary64 records for one
// output.  One output: single-output models whose F bytes per object do not fit K2.
#include "dispatch.h"

namespace obt {

template <int DI, int CMP, int LEAF>
static const void* staged_c(int c) {
  switch (c) {
#define OBT_C(n) case n: return (const void*)apply_multi_staged_kernel<DI, CMP, n, LEAF>;
    OBT_C(1) OBT_C(2) OBT_C(3) OBT_C(4) OBT_C(5) OBT_C(6) OBT_C(7) OBT_C(8) OBT_C(9) OBT_C(10)
#undef OBT_C
    default: return nullptr;
  }
}

template <int DI>
static const void* staged_di(int cmp, int c, int leaf) {
  if (leaf == 2) return cmp == 7 ? staged_c<DI, 7, 2>(c) : staged_c<DI, 8, 2>(c);
  if (leaf == 1) return cmp == 7 ? staged_c<DI, 7, 1>(c) : staged_c<DI, 8, 1>(c);
  // binary64 records: one output only (large-F single-output models with leaves that are
  // not binary32-exact)
  if (leaf == 0 && c == 1)
    return cmp == 7 ? (const void*)apply_multi_staged_kernel<DI, 7, 1, 0> : (const void*)apply_multi_staged_kernel<DI, 8, 1, 0>;
  return nullptr;
}

const void* pick_multi_staged(int di, int cmp, int c, int leaf, int* di_out) {
  const int d = multi_depth(di);
  if (di_out) *di_out = d;
  switch (d) {
    case 4: return staged_di<4>(cmp, c, leaf);
    case 6: return staged_di<6>(cmp, c, leaf);
    case 8: return staged_di<8>(cmp, c, leaf);
    case 10: return staged_di<10>(cmp, c, leaf);
    default: return nullptr;
  }
}

}  // namespace obt
