// k_quantize.cu -- instantiations of K1 / K1t (0..8 search levels) and K1L (1..4 cell compares).
#include "dispatch.h"

namespace obt {

template <int L>
static QuantFn quant_fn(int layout, bool tiled) {
  if (layout == 0) return tiled ? quantize_kernel<L, 0, true> : quantize_kernel<L, 0, false>;
  return tiled ? quantize_kernel<L, 1, true> : quantize_kernel<L, 1, false>;
}

QuantFn pick_quant(int levels, int layout, bool tiled) {
  switch (levels) {
    case 0: return quant_fn<0>(layout, tiled);
    case 1: return quant_fn<1>(layout, tiled);
    case 2: return quant_fn<2>(layout, tiled);
    case 3: return quant_fn<3>(layout, tiled);
    case 4: return quant_fn<4>(layout, tiled);
    case 5: return quant_fn<5>(layout, tiled);
    case 6: return quant_fn<6>(layout, tiled);
    case 7: return quant_fn<7>(layout, tiled);
    case 8: return quant_fn<8>(layout, tiled);
    default: return nullptr;
  }
}

QuantTmaFn pick_quant_tma(int levels) {
  switch (levels) {
    case 0: return quantize_tma_kernel<0>;
    case 1: return quantize_tma_kernel<1>;
    case 2: return quantize_tma_kernel<2>;
    case 3: return quantize_tma_kernel<3>;
    case 4: return quantize_tma_kernel<4>;
    case 5: return quantize_tma_kernel<5>;
    case 6: return quantize_tma_kernel<6>;
    case 7: return quantize_tma_kernel<7>;
    case 8: return quantize_tma_kernel<8>;
    default: return nullptr;
  }
}

template <int LAYOUT, int CELLS>
static QuantFn ldg_lut(int kmax) {
  switch (kmax) {
    case 1: return quantize_kernel<1, LAYOUT, true, CELLS>;
    case 2: return quantize_kernel<2, LAYOUT, true, CELLS>;
    case 3: return quantize_kernel<3, LAYOUT, true, CELLS>;
    case 4: return quantize_kernel<4, LAYOUT, true, CELLS>;
    default: return nullptr;
  }
}

QuantFn pick_quant_ldg_lut(int kmax, int cells, int layout) {
  if (cells == 1024) return layout == 0 ? ldg_lut<0, 1024>(kmax) : ldg_lut<1, 1024>(kmax);
  if (cells == 512) return layout == 0 ? ldg_lut<0, 512>(kmax) : ldg_lut<1, 512>(kmax);
  return layout == 0 ? ldg_lut<0, 256>(kmax) : ldg_lut<1, 256>(kmax);
}

QuantTmaFn pick_quant_lut(int kmax, int cells) {
  if (cells == 512) {
    switch (kmax) {
      case 1: return quantize_lut_kernel<1, 512>;
      case 2: return quantize_lut_kernel<2, 512>;
      case 3: return quantize_lut_kernel<3, 512>;
      case 4: return quantize_lut_kernel<4, 512>;
      default: return nullptr;
    }
  }
  if (cells == 1024) {
    switch (kmax) {
      case 1: return quantize_lut_kernel<1, 1024>;
      case 2: return quantize_lut_kernel<2, 1024>;
      case 3: return quantize_lut_kernel<3, 1024>;
      case 4: return quantize_lut_kernel<4, 1024>;
      default: return nullptr;
    }
  }
  switch (kmax) {
    case 1: return quantize_lut_kernel<1, 256>;
    case 2: return quantize_lut_kernel<2, 256>;
    case 3: return quantize_lut_kernel<3, 256>;
    case 4: return quantize_lut_kernel<4, 256>;
    default: return nullptr;
  }
}

}  // namespace obt
