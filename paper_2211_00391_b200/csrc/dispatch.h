// dispatch.h -- kernel selection across the per-family translation units (k_*.cu).
#pragma once

#include "obtree_kernels.cuh"

namespace obt {

using QuantFn = void (*)(QuantizeParams);
using QuantTmaFn = void (*)(const CUtensorMap, const QuantizeParams);

struct ApplyKernel {
  const void* fn = nullptr;
  int dsrc = 0;   // 0: descriptors in the shared-memory ring, 1: parameter bank
  int words = 1;  // bucket words per thread
  int tpw = 1;    // lanes per bucket word (depth-split kernel when > 1)
};

// K1, levels 0..8
QuantFn pick_quant(int levels, int layout, bool tiled);
QuantTmaFn pick_quant_tma(int levels);
// K1L, cell-table quantize with kmax (1..4) compares per value, 256 or 1024 cells
QuantTmaFn pick_quant_lut(int kmax, int cells);
// K1 (LDG-loaded rows) with the cell-table search, tiled output
QuantFn pick_quant_ldg_lut(int kmax, int cells, int layout);
// K2, depths {1..8, 10, 12}
ApplyKernel pick_apply(int di, int cmp, int leaf, bool write_idx, int dsrc);
// K2s, depth-split (tpw 2: depths 2/4/6/8, tpw 4: depths 4/8)
ApplyKernel pick_split(int di, int cmp, int leaf, int tpw);
// K4 multi-output: depths {4, 6, 8, 10, 12}, outputs <= 16; returns the depth / output
// capacity it was instantiated for through *di_out / *c_out
const void* pick_multi(int di, int cmp, int leaf, int c, int* di_out);
int multi_depth(int d);
// K2f fanned-out small-batch apply (depths 1..8)
const void* pick_fan(int di, int cmp, int leaf);
// K2w warp-specialised apply for wide feature sets (depths 1..8)
#ifndef OBT_WIDE_NIDX
#define OBT_WIDE_NIDX 8
#endif
constexpr int kWideIndexWarps = OBT_WIDE_NIDX;
const void* pick_wide(int di, int cmp, int leaf, int dsrc);
// K5 staged multi-output (depths 4/6/8/10, outputs 2..10; leaf 1 = binary32 records,
// 2 = binary16 records with binary32 accumulators)
const void* pick_multi_staged(int di, int cmp, int c, int leaf, int* di_out);

}  // namespace obt
