// obtree_capi.cu -- host side of the C ABI declared in include/obtree_b200.h.
//
// Owns model validation and packing (the ModelTables / build_leaf_bank step of the
// reference, evaluate.py:138-166 and model.py:231-277), device residency, the
// per-call launch plan (tile size, workspace) and kernel dispatch.  No CPU compute
// path exists: if a kernel cannot run the call fails with an error code.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/obtree_b200.h"
#include "obtree_kernels.cuh"
#include "dispatch.h"
#include "wide_apply.cuh"

using obt::ApplyKernel;
using obt::QuantFn;
using obt::pick_apply;
using obt::pick_quant;
using obt::pick_quant_tma;
using obt::pick_quant_lut;
using obt::pick_split;

namespace {

thread_local std::string g_error;
thread_local int g_launches = 0;

// Path options (obt_set_path_option): each forces one automatic choice of the dispatch,
// for parity tests that cover every kernel path and for A/B measurements.  -1 (the
// default) leaves the choice to the planner; production callers never set them.
enum PathOption {
  OPT_DESC_SOURCE,   // 0: descriptors from the shared-memory ring, 1: kernel-parameter bank
  OPT_TPW,           // lanes per bucket word in K2 / K2s: 1, 2 or 4
  OPT_WIDE,          // 0 / 1: forbid / force K2w (where it fits)
  OPT_FAN,           // 0 / 1: forbid / force K2f (small batches)
  OPT_PDL,           // 0: no chained (programmatic dependent) parameter-bank launches
  OPT_TAIL_SPLIT,    // 0 / 1: forbid / force the tail-wave region
  OPT_QUANT_LUT,     // 0 / 1: Eytzinger (K1t) / cell-table (K1L) quantize
  OPT_LUT_CELLS,     // 256, 512 or 1024 cells per feature table (read at model creation)
  OPT_LEAF_STORAGE,  // 0: binary64 leaf tables even when binary32 is exact (model creation)
  OPT_MULTI_STAGED,  // 0 / 1: K4 / K5 for multi-output models (model creation)
  OPT_LEAF_SELECT,   // 1: K2 selects leaves by warp shuffle from register-resident tables
  OPT_COUNT
};
const char* const kPathOptionNames[OPT_COUNT] = {"desc_source", "tpw", "wide", "fan", "pdl",
                                                 "tail_split", "quant_lut", "lut_cells", "leaf_storage",
                                                 "multi_staged", "leaf_select"};
std::atomic<int> g_opt[OPT_COUNT] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
int opt(PathOption o) { return g_opt[o].load(std::memory_order_relaxed); }


int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t err__ = (expr);                                                        \
    if (err__ != cudaSuccess)                                                          \
      return fail(OBT_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(err__));      \
  } while (0)

constexpr int kMaxBorders = 254;  // model.py:21
constexpr int kMaxDepth = 12;     // smem-staged leaf tables (2^12 fp32 = 16 KiB per tree)
constexpr int kSentinel = 255;    // evaluate.py:32
#ifndef OBT_STAGES
#define OBT_STAGES 2
#endif
constexpr int kStages = OBT_STAGES;  // records in flight in the apply kernel's ring
constexpr int kMaxOutputs = 16;   // multi-output kernel instantiations
constexpr int kMultiTile = obt::kMultiTileObjects;  // objects per multi-output CTA

// Instantiated depths of the apply kernel; a model of depth D runs on the
// smallest instantiation >= D with sentinel (never-true) padding splits.
int instantiated_depth(int d) {
  if (d <= 8) return d < 1 ? 1 : d;
  if (d <= 10) return 10;
  if (d <= 12) return 12;
  return -1;
}

struct BorderTable {
  float* d = nullptr;  // [F][pitch] Eytzinger order, +inf padded
  int levels = 0;
  int pitch = 1;
};

// K1L cell tables of a border set (see quantize_lut_kernel): kmax = 0 when the set
// needs more than kLutMaxCompares compares in some cell (the Eytzinger K1t runs then).
struct LutTable {
  uint8_t* d_lut = nullptr;        // [F][cells]
  unsigned char* d_rec = nullptr;  // [F][rec_stride]
  int rec_stride = 0;
  int kmax = 0;
  int cells = 256;
};
constexpr int kLutMaxCompares = 4;

struct TilePlan {
  uint8_t* d_chunks = nullptr;          // [n_chunks][chunk_bytes] descriptor + leaf records
  std::vector<uint32_t> param_desc;     // [padded_trees][DI][2] {off, k replicated} for the parameter bank
  uint8_t* d_tables = nullptr;          // [n_chunks][tables_chunk_bytes] leaf tables only (parameter-bank launches)
  uint32_t tables_chunk_bytes = 0;
};

// K2w records: per chunk of kWideChunkTrees trees, the descriptors (kWideDescBytes(DI)
// per tree) and, in a second array, the leaf tables (`stride` bytes each), trees in the
// predict path's level order.
struct WidePlan {
  uint8_t* d_desc = nullptr;
  uint8_t* d_tables = nullptr;
  std::vector<uint32_t> bank;  // [n_chunks][kWideChunkTrees][2 DI] descriptors for the parameter bank
  int n_chunks = 0;
  int tstages[2] = {0, 0}, slots[2] = {0, 0};  // per descriptor source (0 ring, 1 bank)
  size_t smem[2] = {0, 0};
};

}  // namespace

struct obt_model {
  int device = 0;
  int n_features = 0, n_trees = 0, max_depth = 0, n_outputs = 1;
  int depth_inst = 1;        // DI
  int precision = OBT_PRECISION_BINARY64;
  int leaf_storage = 1;      // 0 fp64, 1 fp32, 2 fp16
  int compare_mode = 7;      // 7: all buckets < 128; 8: full byte compare
  BorderTable full;          // every border: obt_quantize_dev (reference buckets)
  BorderTable used;          // borders referenced by splits: the predict path
  LutTable used_lut;         // cell tables of `used` (K1L), kmax 0 if not applicable
  void* d_multi_leaves = nullptr;   // multi-output records [T][2^DI][CP] (K4) or [T][2^DI] slots (K4s)
  int multi_staged = 0;             // 1: K5 (tree tables + bucket rows staged in shared memory)
  // the K4 / K5 record path: multi-output models, and single-output models whose F bytes
  // per object leave no room for K2's 128-object bucket tile (K5 stages only the rows a
  // tree reads: the paper's epsilon model has F = 2,000)
  int multi_style = 0;
  int staged_stages = 0;
  uint32_t staged_table_bytes = 0, staged_stage_bytes = 0;
  int multi_slot = 0;
  uint32_t* d_multi_desc = nullptr; // multi-output descriptors [T][DI][2] for kMultiTile
  double scale = 1.0, bias = 0.0;
  // host copies used to (re)build descriptor records for a tile size
  std::vector<int32_t> split_feature;   // [T][DI]
  std::vector<uint8_t> split_ordinal;   // [T][DI]
  std::vector<uint8_t> leaf_bytes;      // [T][2^DI] in leaf_storage
  // predict-path level order: level_perm[t][j] = the reference level evaluated as depth j
  // (index bit j); index dumps keep the reference order (see level_order)
  std::vector<uint8_t> level_perm;      // [T][DI]
  // chunk geometry (independent of the tile size)
  int padded_trees = 0;
  int chunk_trees = 1, n_chunks = 0;
  uint32_t chunk_bytes = 128, desc_bytes = 0;
  int sm_count = 148;
  int smem_optin = 232448;
  std::mutex mu;
  std::map<int, TilePlan> plans;
  std::unique_ptr<WidePlan> wide;        // K2w records (built on first use, under mu)
  obt::ApplyArgs<1> param_args;  // launch-parameter staging (32 KB), guarded by mu
  ~obt_model() {
    if (wide && wide->d_desc) cudaFree(wide->d_desc);
    if (wide && wide->d_tables) cudaFree(wide->d_tables);
    for (auto& kv : plans) {
      cudaFree(kv.second.d_chunks);
      if (kv.second.d_tables) cudaFree(kv.second.d_tables);
    }
    if (full.d) cudaFree(full.d);
    if (d_multi_leaves) cudaFree(d_multi_leaves);
    if (d_multi_desc) cudaFree(d_multi_desc);
    if (used.d) cudaFree(used.d);
    if (used_lut.d_lut) cudaFree(used_lut.d_lut);
    if (used_lut.d_rec) cudaFree(used_lut.d_rec);
  }
};

namespace {

size_t leaf_size(int storage) { return storage == 0 ? 8 : storage == 1 ? 4 : 2; }

// binary64 -> binary16, round to nearest even (the numpy astype of model.py:263).
uint16_t half_rne(double x) {
  uint64_t bits;
  std::memcpy(&bits, &x, 8);
  const uint16_t sign = (uint16_t)((bits >> 48) & 0x8000u);
  const int exp = (int)((bits >> 52) & 0x7FF);
  const uint64_t man = bits & 0xFFFFFFFFFFFFFull;
  if (exp == 0x7FF) return (uint16_t)(sign | (man ? 0x7E00u : 0x7C00u));
  if (exp == 0) return sign;
  const int e = exp - 1023;
  if (e > 15) return (uint16_t)(sign | 0x7C00u);
  const uint64_t sig = man | (1ull << 52);
  const int shift = ((e < -14 ? -14 : e) - 10) - (e - 52);
  uint64_t q = 0;
  if (shift < 64) {
    q = sig >> shift;
    const uint64_t rem = sig & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (q & 1))) ++q;
  }
  if (e < -14) return (uint16_t)(sign | q);
  int he = e;
  if (q >= 2048) { q >>= 1; ++he; }
  if (he > 15) return (uint16_t)(sign | 0x7C00u);
  return (uint16_t)(sign | ((uint32_t)(he + 15) << 10) | (uint32_t)(q - 1024));
}

// saturation of every infinite result (finite overflow and infinite leaves) to
// +/-65504 (model.py:262-268: the reference tests isinf on the cast values only)
uint16_t half_bank_entry(double x) {
  uint16_t h = half_rne(x);
  if ((h & 0x7FFFu) == 0x7C00u) h = (uint16_t)((h & 0x8000u) | 0x7BFFu);
  return h;
}

void eytzinger_fill(const float* sorted, int n, float* out, int pitch, int& pos, int node) {
  // in-order walk of the implicit complete tree (children 2i+1, 2i+2)
  if (node >= pitch) return;
  eytzinger_fill(sorted, n, out, pitch, pos, 2 * node + 1);
  out[node] = pos < n ? sorted[pos] : INFINITY;
  ++pos;
  eytzinger_fill(sorted, n, out, pitch, pos, 2 * node + 2);
}

int build_border_table(const float* borders, const int32_t* counts, int F, int stride, BorderTable& out) {
  int bmax = 0;
  for (int f = 0; f < F; ++f) bmax = std::max(bmax, (int)counts[f]);
  int levels = 0;
  while (((1 << levels) - 1) < bmax) ++levels;
  out.levels = levels;
  out.pitch = std::max(1, (1 << levels) - 1);
  std::vector<float> eytz((size_t)F * out.pitch, INFINITY);
  for (int f = 0; f < F; ++f) {
    int pos = 0;
    if (levels > 0)
      eytzinger_fill(borders + (size_t)f * stride, counts[f], eytz.data() + (size_t)f * out.pitch,
                     (1 << levels) - 1, pos, 0);
  }
  CUDA_TRY(cudaMalloc(&out.d, eytz.size() * sizeof(float)));
  CUDA_TRY(cudaMemcpy(out.d, eytz.data(), eytz.size() * sizeof(float), cudaMemcpyHostToDevice));
  return OBT_OK;
}

// Cell tables for K1L.  Per feature (borders b_0 < ... < b_{U-1}): lo = b_0, hi = b_{U-1},
// s ~ 254 / (hi - lo), o = 1.5 * 2^23 - lo * s (+ nudges), checked with the device's own
// fp32 operations (fmaxf / fminf / fmaf, correctly rounded on both sides) so that every
// clamped x maps into [1.5 * 2^23, 1.5 * 2^23 + 255]; then cell c_k of each border,
// lut[c] = #{k : c_k < c}, and K = the most borders sharing a cell.  Returns kmax = 0
// (not applicable) if a feature needs more than kLutMaxCompares compares or its range
// does not fit the map.
// Host tables for `cells` cells per feature; returns kmax (0: not applicable).
int plan_lut_table(const float* borders, const int32_t* counts, int F, int stride, int cells,
                   std::vector<uint8_t>& lut, std::vector<unsigned char>& rec, int& rec_stride) {
  const float M = 12582912.0f;  // 1.5 * 2^23: floats in [2^23, 2^24) step by 1
  uint32_t mbits;
  std::memcpy(&mbits, &M, 4);
  int umax = 0;
  for (int f = 0; f < F; ++f) umax = std::max(umax, (int)counts[f]);
  const int P = (umax + 1 + 3) / 4 * 4;  // borders + one +inf pad (index U is read)
  rec_stride = obt::kLutRecHeader + 4 * P;
  lut.assign((size_t)F * cells, 0);
  rec.assign((size_t)F * rec_stride, 0);
  auto cell_of = [&](float x, float lo, float hi, float sc, float of) -> long {
    const float y = fmaf(fminf(fmaxf(x, lo), hi), sc, of);
    uint32_t yb;
    std::memcpy(&yb, &y, 4);
    if (!(y >= 8388608.0f && y < 16777216.0f)) return -1;
    return (long)yb - (long)mbits;
  };
  int kmax = 1;
  for (int f = 0; f < F; ++f) {
    const int U = counts[f];
    const float* b = borders + (size_t)f * stride;
    float lo = 0.0f, hi = 0.0f, sc = 0.0f, of = M;
    if (U >= 2) {
      lo = b[0];
      hi = b[U - 1];
      const double span = (double)hi - (double)lo;
      sc = (float)((double)(cells - 2) / span);
      if (!(span > 0) || !std::isfinite(sc) || !(sc > 0)) return 0;
      const double o0 = (double)M - (double)lo * (double)sc;
      if (!(o0 > 8388608.0 + 2 * cells && o0 < 16777216.0 - 2 * cells)) return 0;
      of = (float)std::floor(o0);
      bool ok = false;
      for (int it = 0; it < 8; ++it) {
        const long clo = cell_of(lo, lo, hi, sc, of), chi = cell_of(hi, lo, hi, sc, of);
        if (clo < 0) { of += 1.0f; continue; }
        if (chi > cells - 1) { of -= 1.0f; continue; }
        ok = clo >= 0 && chi <= cells - 1;
        break;
      }
      if (!ok) return 0;
    } else if (U == 1) {
      lo = hi = b[0];
    }
    // cells of the borders, lower-bound table, compares needed
    std::vector<int> per_cell(cells, 0);
    std::vector<long> cl(U);
    for (int k = 0; k < U; ++k) {
      const long c = cell_of(b[k], lo, hi, sc, of);
      if (c < 0 || c > cells - 1 || (k > 0 && c < cl[k - 1])) return 0;  // must be monotone
      cl[k] = c;
      ++per_cell[c];
    }
    int kf = 0;
    for (int c = 0, below = 0; c < cells; ++c) {
      lut[(size_t)f * cells + c] = (uint8_t)below;
      below += per_cell[c];
      kf = std::max(kf, per_cell[c]);
    }
    if (kf > kLutMaxCompares) return 0;
    kmax = std::max(kmax, kf);
    float* r = reinterpret_cast<float*>(rec.data() + (size_t)f * rec_stride);
    r[0] = lo; r[1] = hi; r[2] = sc; r[3] = of;
    float* bd = r + obt::kLutRecHeader / 4;
    for (int k = 0; k < P; ++k) bd[k] = k < U ? b[k] : INFINITY;
  }
  return kmax;
}

// Cell tables for K1L.  Per feature (borders b_0 < ... < b_{U-1}): lo = b_0, hi = b_{U-1},
// s ~ (cells - 2) / (hi - lo), o = 1.5 * 2^23 - lo * s (+ nudges), checked with the
// device's own fp32 operations (fmaxf / fminf / fmaf, correctly rounded on both sides) so
// that every clamped x maps into [1.5 * 2^23, 1.5 * 2^23 + cells - 1]; then cell c_k of
// each border, lut[c] = #{k : c_k < c}, and K = the most borders sharing a cell.  256
// cells unless some cell holds several borders and 1024 cells bring it to one compare.
// kmax = 0 (not applicable) if a feature needs more than kLutMaxCompares compares or its
// range does not fit the map.
int build_lut_table(const float* borders, const int32_t* counts, int F, int stride, LutTable& out) {
  std::vector<uint8_t> lut;
  std::vector<unsigned char> rec;
  int rs = 0;
  out.kmax = 0;
  out.cells = 256;
  int k = plan_lut_table(borders, counts, F, stride, 256, lut, rec, rs);
  const int forced = std::max(0, opt(OPT_LUT_CELLS));
  const int big = (forced == 512 || forced == 1024) ? forced : 1024;
  if ((k != 1 && forced != 256) || forced == 512 || forced == 1024) {
    std::vector<uint8_t> lut2;
    std::vector<unsigned char> rec2;
    int rs2 = 0;
    const int k2 = plan_lut_table(borders, counts, F, stride, big, lut2, rec2, rs2);
    if (k2 > 0 && (forced == big || (k2 <= 2 && (k == 0 || k2 < k)))) {
      lut.swap(lut2);
      rec.swap(rec2);
      rs = rs2;
      k = k2;
      out.cells = big;
    }
  }
  if (k <= 0) return OBT_OK;
  out.rec_stride = rs;
  CUDA_TRY(cudaMalloc(&out.d_lut, lut.size()));
  CUDA_TRY(cudaMemcpy(out.d_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&out.d_rec, rec.size()));
  CUDA_TRY(cudaMemcpy(out.d_rec, rec.data(), rec.size(), cudaMemcpyHostToDevice));
  out.kmax = k;
  return OBT_OK;
}

int validate(const obt_model_desc* d) {
  if (!d) return fail(OBT_E_INVALID, "invalid model: null description");
  if (d->n_features < 1) return fail(OBT_E_INVALID, "invalid model: model: at least one float feature is required");
  if (d->n_trees < 0) return fail(OBT_E_INVALID, "invalid model: negative tree count");
  if (d->n_outputs < 1 || d->n_outputs > kMaxOutputs)
    return fail(OBT_E_UNSUPPORTED, "n_outputs=%d outside 1..%d", d->n_outputs, kMaxOutputs);
  if (d->n_outputs > 1 && d->precision == OBT_PRECISION_BINARY16 && (d->n_outputs > 10 || d->max_depth > 10))
    return fail(OBT_E_UNSUPPORTED,
                "binary16 multi-output models run on the staged kernel: at most 10 outputs and depth 10");
  if (d->n_trees > 0 && (d->max_depth < 1 || d->max_depth > 16))
    return fail(OBT_E_INVALID, "invalid model: max_depth %d outside 1..16", d->max_depth);
  if (d->n_trees > 0 && instantiated_depth(d->max_depth) < 0)
    return fail(OBT_E_UNSUPPORTED, "depth %d exceeds the %d supported by the apply kernel", d->max_depth, kMaxDepth);
  if (!d->border_counts || !d->borders) return fail(OBT_E_INVALID, "invalid model: missing borders");
  if (d->precision != OBT_PRECISION_BINARY64 && d->precision != OBT_PRECISION_BINARY16)
    return fail(OBT_E_INVALID, "unknown precision %d", d->precision);
  for (int f = 0; f < d->n_features; ++f) {
    const int nb = d->border_counts[f];
    if (nb < 0 || nb > kMaxBorders || nb > d->border_stride)
      return fail(OBT_E_INVALID, "invalid model: float_features[%d]: %d borders exceed the limit of %d", f, nb, kMaxBorders);
    const float* b = d->borders + (size_t)f * d->border_stride;
    for (int k = 0; k < nb; ++k) {
      if (std::isnan(b[k])) return fail(OBT_E_INVALID, "invalid model: float_features[%d]: NaN border", f);
      if (k > 0 && !(b[k] > b[k - 1])) return fail(OBT_E_INVALID, "invalid model: float_features[%d]: non-ascending borders", f);
    }
  }
  if (d->n_trees > 0) {
    if (!d->split_feature || !d->split_ordinal || !d->leaves)
      return fail(OBT_E_INVALID, "invalid model: missing tree arrays");
    const int D = d->max_depth;
    for (int t = 0; t < d->n_trees; ++t) {
      for (int s = 0; s < D; ++s) {
        const int f = d->split_feature[(size_t)t * D + s];
        const int ord = d->split_ordinal[(size_t)t * D + s];
        if (ord == kSentinel) continue;
        if (f < 0 || f >= d->n_features)
          return fail(OBT_E_INVALID, "invalid model: trees[%d].splits[%d]: feature index %d out of range", t, s, f);
        if (ord >= d->border_counts[f])
          return fail(OBT_E_INVALID,
                      "invalid model: trees[%d].splits[%d]: border ordinal out of range (%d vs %d borders on feature %d)",
                      t, s, ord, d->border_counts[f], f);
      }
      const double* lv = d->leaves + (((size_t)t * d->n_outputs) << D);
      for (size_t j = 0; j < ((size_t)d->n_outputs << D); ++j)
        if (std::isnan(lv[j])) return fail(OBT_E_INVALID, "invalid model: trees[%d]: NaN leaf value", t);
    }
  }
  return OBT_OK;
}

size_t table_stride(const obt_model* m) {
  return (size_t)obt::leaf_table_stride(m->depth_inst, (int)leaf_size(m->leaf_storage));
}

// Chunk geometry: the ring of kStages records gets what the bucket tile leaves of the
// shared memory; records hold whole groups of obt::tree_group(depth) trees, and the
// model is padded with null trees to a multiple of the chunk.
void plan_chunks(obt_model* m) {
  const int DI = m->depth_inst;
  // descriptor region sized for the larger of the K2 ({off, k}) and K2s (16-byte) formats
  const size_t per_tree_desc = std::max<size_t>((size_t)obt::desc_words_per_tree(DI, m->compare_mode) * 4,
                                                (size_t)DI * obt::kSplitDescBytes);
  const size_t per_tree = per_tree_desc + table_stride(m);
  const int group = obt::tree_group(DI);
  // ring budget: what the bucket tile of the largest 256-quantum tile leaves over
  const int64_t avail = (int64_t)m->smem_optin - 512;
  const int64_t tile_cap = 4 * (obt::kApplyMaxThreads - obt::kApplyProducerThreads) / 128 * 128;
  const int64_t tile_objs = std::min<int64_t>(
      tile_cap, std::max<int64_t>(128, (avail - (int64_t)kStages * 4096) / m->n_features / 128 * 128));
  const int64_t ring = std::max<int64_t>((int64_t)kStages * per_tree * group, avail - tile_objs * m->n_features);
  int ct = (int)std::max<int64_t>(group, (ring / kStages - 512) / (int64_t)per_tree / group * group);
  ct = std::min(ct, 64);
  const int groups = (m->n_trees + group - 1) / group;
  if (groups > 0) ct = std::min(ct, groups * group);
  m->chunk_trees = ct;
  m->n_chunks = (m->n_trees + ct - 1) / ct;
  m->padded_trees = m->n_chunks * ct;
  m->desc_bytes = (uint32_t)((per_tree_desc * ct + 255) & ~(size_t)255);
  m->chunk_bytes = (uint32_t)((m->desc_bytes + table_stride(m) * ct + 255) & ~(size_t)255);
}

// Descriptor words of tree t (padded trees are all-sentinel) for a given tile size:
// 7-bit compare {off, k replicated}; 8-bit compare {(off << 8) | k, s}.  `ordered`: the
// predict path's level order (level_perm), else the reference's (index dumps).
void tree_descriptors(const obt_model* m, int t, int tile, uint32_t* out, bool ordered = true) {
  const int DI = m->depth_inst;
  for (int j = 0; j < DI; ++j) {
    const int d = (ordered && t < m->n_trees && !m->level_perm.empty()) ? m->level_perm[(size_t)t * DI + j] : j;
    const int ord = t < m->n_trees ? m->split_ordinal[(size_t)t * DI + d] : kSentinel;
    uint32_t w0 = 0, w1 = 0;  // sentinel: offset 0, k 0 never carries into bit 7
    if (ord != kSentinel) {
      const uint32_t off = (uint32_t)m->split_feature[(size_t)t * DI + d] * (uint32_t)tile;
      if (m->compare_mode == 7) {
        w0 = off;
        w1 = (uint32_t)(127 - ord) * 0x01010101u;              // q + 127 - ord >= 128 <=> q > ord
      } else {
        w0 = (off << 8) | (uint32_t)(127 - (ord & 127));
        w1 = ord < 128 ? 0xFFFFFFFFu : 0u;                    // or-with-q vs and-with-q
      }
    }
    out[2 * j] = w0;
    out[2 * j + 1] = w1;
  }
}

// Leaf i' of a tree evaluated in level order perm is leaf i = sum_j bit_j(i') << perm[j]
// of the reference order.
size_t reference_leaf(const uint8_t* perm, int DI, size_t ip) {
  size_t i = 0;
  for (int j = 0; j < DI; ++j) i |= ((ip >> j) & 1u) << perm[j];
  return i;
}

// Tree t's leaf table (2^DI entries of `ls` bytes) in the predict path's level order.
void ordered_leaves(const obt_model* m, int t, uint8_t* dst) {
  const int DI = m->depth_inst;
  const size_t ls = leaf_size(m->leaf_storage), n = (size_t)1 << DI;
  const uint8_t* src = m->leaf_bytes.data() + (size_t)t * n * ls;
  const uint8_t* perm = m->level_perm.data() + (size_t)t * DI;
  for (size_t ip = 0; ip < n; ++ip) std::memcpy(dst + ip * ls, src + reference_leaf(perm, DI, ip) * ls, ls);
}

// Predict-path level order of every tree (exact: a permutation of the index bits and of
// the leaf table).  A warp-wide gather from a 2^D-entry table costs as many shared-memory
// wavefronts as the most distinct entries any one bank is asked for; the bank is set by
// the low index bits.  Levels whose condition is nearly always true or false (ordinals
// near either end of the feature's borders: P(x > b_k) ~ 1 - (k+1)/(B+1) for quantile
// borders) take the high bits, where lanes then mostly agree, and the most uncertain
// levels the low (bank) bits.  Measured by Monte Carlo at depth 8 / fp32 leaves: ~4.0 ->
// ~2.6 wavefronts per warp gather (depth 6: 1.9 -> 1.7).  Sentinel levels go last.
void plan_level_order(obt_model* m, const obt_model_desc* d) {
  const int DI = m->depth_inst, D = m->max_depth;
  m->level_perm.assign((size_t)m->n_trees * DI, 0);
  std::vector<std::pair<double, int>> key(DI);
  for (int t = 0; t < m->n_trees; ++t) {
    for (int j = 0; j < DI; ++j) {
      double h = -1.0;  // sentinel / padding levels: never true, zero entropy
      if (j < D) {
        const int ord = d->split_ordinal[(size_t)t * D + j];
        if (ord != kSentinel) {
          const int nb = d->border_counts[d->split_feature[(size_t)t * D + j]];
          const double p = 1.0 - (ord + 1.0) / (nb + 1.0);
          h = (p <= 0.0 || p >= 1.0) ? 0.0 : -(p * std::log(p) + (1.0 - p) * std::log(1.0 - p));
        }
      }
      key[j] = {-h, j};
    }
    std::stable_sort(key.begin(), key.end());
    for (int j = 0; j < DI; ++j) m->level_perm[(size_t)t * DI + j] = (uint8_t)key[j].second;
  }
}

// Null tree: every leaf is -0.0, the exact identity of IEEE addition.
void write_null_leaves(const obt_model* m, uint8_t* dst) {
  for (size_t j = 0; j < ((size_t)1 << m->depth_inst); ++j) {
    if (m->leaf_storage == 0) { const double z = -0.0; std::memcpy(dst + j * 8, &z, 8); }
    else if (m->leaf_storage == 1) { const float z = -0.0f; std::memcpy(dst + j * 4, &z, 4); }
    else { const uint16_t z = 0x8000u; std::memcpy(dst + j * 2, &z, 2); }
  }
}

// K2s level order for tree t: perm[j] = the original level evaluated as depth j.  Lane
// part 0 evaluates depths [0, DI/2), part 1 [DI/2, DI); at step i they read the rows of
// depths i and DI/2 + i, which are conflict-free when the rows differ in parity (the
// swizzled bucket layout).  Levels are paired even-odd first; sentinel levels read no
// meaningful bucket, so they take whichever row parity their partner needs
// (wild_color[j] = the row parity for a sentinel at depth j).
void split_level_order(const obt_model* m, int t, int* perm, int* wild_color) {
  const int DI = m->depth_inst, half = DI / 2;
  for (int j = 0; j < DI; ++j) { perm[j] = j; wild_color[j] = 0; }
  if (DI < 2 || DI % 2 || t >= m->n_trees) return;
  std::vector<int> even, odd, wild;
  for (int d = 0; d < DI; ++d) {
    const size_t i = (size_t)t * DI + d;
    if (m->split_ordinal[i] == kSentinel) wild.push_back(d);
    else if (m->split_feature[i] & 1) odd.push_back(d);
    else even.push_back(d);
  }
  const int c_wild_odd = m->n_features > 1 ? 1 : 0;  // row 1 exists only with >= 2 features
  std::vector<std::pair<int, int>> p0, p1;  // (level, sentinel row parity) per part
  auto take = [](std::vector<int>& v) { const int x = v.back(); v.pop_back(); return x; };
  while (!even.empty() && !odd.empty()) { p0.push_back({take(even), 0}); p1.push_back({take(odd), 0}); }
  while (!even.empty() && !wild.empty()) { p0.push_back({take(even), 0}); p1.push_back({take(wild), c_wild_odd}); }
  while (!odd.empty() && !wild.empty()) { p0.push_back({take(odd), 0}); p1.push_back({take(wild), 0}); }
  while (wild.size() >= 2) { p0.push_back({take(wild), 0}); p1.push_back({take(wild), c_wild_odd}); }
  std::vector<int> rest;  // same-parity leftovers: pair among themselves (conflicting)
  for (int d : even) rest.push_back(d);
  for (int d : odd) rest.push_back(d);
  for (int d : wild) rest.push_back(d);
  for (size_t i = 0; i + 1 < rest.size(); i += 2) { p0.push_back({rest[i], 0}); p1.push_back({rest[i + 1], 0}); }
  for (int j = 0; j < half; ++j) {
    perm[j] = p0[j].first;
    wild_color[j] = p0[j].second;
    perm[half + j] = p1[j].first;
    wild_color[half + j] = p1[j].second;
  }
}

// Per-(tile size, variant) state: device records (descriptors + leaves) for the
// shared-memory descriptor path (variant 0: K2, variant 1: K2s with swizzled rows and
// paired level order), and the flat descriptor stream for the parameter-bank path.
int build_tile_plan(obt_model* m, int tile, int variant, TilePlan& out) {
  const int DI = m->depth_inst;
  const int dwt = obt::desc_words_per_tree(DI, m->compare_mode);  // words in the smem records
  const size_t per_tree_leaf = leaf_size(m->leaf_storage) << DI;  // bytes of real leaves
  const size_t stride = table_stride(m);                           // their slot in the record
  const int ct = m->chunk_trees;
  const size_t desc_bytes = m->desc_bytes, chunk_bytes = m->chunk_bytes;
  std::vector<uint8_t> host((size_t)std::max(m->n_chunks, 1) * chunk_bytes, 0);
  // parameter-bank launches read descriptors from the launch parameters: their ring
  // carries the leaf tables alone (27% fewer bytes per chunk at cfg2)
  const uint32_t tcb = (uint32_t)((stride * ct + 255) & ~(size_t)255);
  std::vector<uint8_t> host_tables(variant == 0 ? (size_t)std::max(m->n_chunks, 1) * tcb : 0, 0);
  // variant 0: predicts (level order of level_perm); 1: K2s; 2: index dumps (reference order)
  out.param_desc.assign((size_t)m->padded_trees * DI * 2, 0u);
  std::vector<uint32_t> words((size_t)DI * 2);
  std::vector<int> perm(DI), wild(DI);
  std::vector<uint8_t> permuted(per_tree_leaf);
  for (int t = 0; t < m->padded_trees; ++t) {
    const int c = t / ct, tl = t % ct;
    uint8_t* rec = host.data() + (size_t)c * chunk_bytes;
    tree_descriptors(m, t, tile, words.data(), variant == 0);
    if (m->compare_mode == 7) std::memcpy(out.param_desc.data() + (size_t)t * DI * 2, words.data(), (size_t)DI * 8);
    if (variant == 1) {
      // K2s: 16 bytes per split in paired level order, row offsets +- 64 for odd rows;
      // half-major: DI entries {off + sw, k} then DI entries {off - sw, k}
      split_level_order(m, t, perm.data(), wild.data());
      uint32_t* dst = reinterpret_cast<uint32_t*>(rec + (size_t)tl * DI * obt::kSplitDescBytes);
      uint32_t* dst_hi = dst + 2 * DI;
      for (int j = 0; j < DI; ++j) {
        const int d = perm[j];
        const bool sentinel = t >= m->n_trees || m->split_ordinal[(size_t)t * DI + d] == kSentinel;
        const int row = sentinel ? wild[j] : m->split_feature[(size_t)t * DI + d];
        const uint32_t off = (uint32_t)row * (uint32_t)tile, sw = (row & 1) ? 64u : 0u;
        const uint32_t kpart = m->compare_mode == 7 ? 0u : (words[2 * d] & 0xFFu);  // 8-bit: k in byte 0
        const uint32_t w1 = sentinel ? 0u : words[2 * d + 1];
        const uint32_t k7 = sentinel ? 0u : kpart;
        if (m->compare_mode == 7) {
          dst[2 * j + 0] = off + sw; dst[2 * j + 1] = w1; dst_hi[2 * j + 0] = off - sw; dst_hi[2 * j + 1] = w1;
        } else {
          dst[2 * j + 0] = ((off + sw) << 8) | k7; dst[2 * j + 1] = w1;
          dst_hi[2 * j + 0] = ((off - sw) << 8) | k7; dst_hi[2 * j + 1] = w1;
        }
      }
      uint8_t* leaf_dst = rec + desc_bytes + (size_t)tl * stride;
      if (t < m->n_trees) {
        // leaf i' of the permuted tree is leaf i of the original, i = sum_j bit_j(i') << perm[j]
        const size_t ls = leaf_size(m->leaf_storage);
        const uint8_t* src = m->leaf_bytes.data() + (size_t)t * per_tree_leaf;
        for (size_t ip = 0; ip < ((size_t)1 << DI); ++ip) {
          size_t i = 0;
          for (int j = 0; j < DI; ++j) i |= ((ip >> j) & 1u) << perm[j];
          std::memcpy(permuted.data() + ip * ls, src + i * ls, ls);
        }
        std::memcpy(leaf_dst, permuted.data(), per_tree_leaf);
      } else {
        write_null_leaves(m, leaf_dst);
      }
      continue;
    }
    if (dwt == DI) {  // packed 7-bit records: (off << 8) | k
      for (int d = 0; d < DI; ++d) words[d] = (words[2 * d] << 8) | (words[2 * d + 1] & 0xFFu);
    }
    // shared-memory copy: trees in groups of 4, each group's words contiguous
    std::memcpy(rec + (size_t)tl * dwt * 4, words.data(), (size_t)dwt * 4);
    uint8_t* leaf_dst = rec + desc_bytes + (size_t)tl * stride;
    if (t < m->n_trees) {
      if (variant == 0) ordered_leaves(m, t, leaf_dst);
      else std::memcpy(leaf_dst, m->leaf_bytes.data() + (size_t)t * per_tree_leaf, per_tree_leaf);
    } else {
      write_null_leaves(m, leaf_dst);
    }
    if (!host_tables.empty()) std::memcpy(host_tables.data() + (size_t)c * tcb + (size_t)tl * stride, leaf_dst, stride);
  }
  CUDA_TRY(cudaMalloc(&out.d_chunks, host.size()));
  CUDA_TRY(cudaMemcpy(out.d_chunks, host.data(), host.size(), cudaMemcpyHostToDevice));
  if (!host_tables.empty()) {
    CUDA_TRY(cudaMalloc(&out.d_tables, host_tables.size()));
    CUDA_TRY(cudaMemcpy(out.d_tables, host_tables.data(), host_tables.size(), cudaMemcpyHostToDevice));
    out.tables_chunk_bytes = tcb;
  }
  return OBT_OK;
}

int get_tile_plan(obt_model* m, int tile, int variant, const TilePlan** out) {
  std::lock_guard<std::mutex> lock(m->mu);
  const int key = tile * 4 + variant;
  auto it = m->plans.find(key);
  if (it == m->plans.end()) {
    TilePlan tp;
    const int rc = build_tile_plan(m, tile, variant, tp);
    if (rc != OBT_OK) return rc;
    it = m->plans.emplace(key, std::move(tp)).first;
  }
  *out = &it->second;
  return OBT_OK;
}

// Tiles are whole multiples of the quantize kernel's 256-object CTA, so a CTA never
// straddles two tiles; the apply kernel runs tile / 4 consumer threads + 1 producer warp.
constexpr int kTileQuantum = obt::kQuantObjects;
// The parameter-bank descriptor path re-reads the bucket tile once per extra launch.
constexpr int kMaxParamLaunches = 4;

// Largest tile (multiple of 256 objects) whose bucket tile fits next to the stage ring;
// then shrink for small batches so the grid still covers the SMs.
int plan_tile(const obt_model* m, int64_t n) {
  if (m->multi_style) return m->multi_staged ? obt::kStagedTile : kMultiTile;
  const int64_t fixed = 512 + (int64_t)kStages * m->chunk_bytes;
  int64_t tmax = (m->smem_optin - fixed) / m->n_features;
  tmax = std::min<int64_t>(tmax / kTileQuantum * kTileQuantum, 4 * (obt::kApplyMaxThreads - obt::kApplyProducerThreads) / kTileQuantum * kTileQuantum);
  if (tmax < kTileQuantum) return -1;
  int64_t want = (n + m->sm_count - 1) / m->sm_count;
  want = std::max<int64_t>(kTileQuantum, (want + kTileQuantum - 1) / kTileQuantum * kTileQuantum);
  return (int)std::min(tmax, want);
}

// Chunks one parameter-bank launch can cover (two words per split).
int param_chunks_per_launch(const obt_model* m) {
  const int words_per_chunk = 2 * m->depth_inst * m->chunk_trees;
  return obt::kParamDescWords / words_per_chunk;
}

// Parameter-bank descriptors (no descriptor wavefronts: uniform constant loads) for a
// region whose words have one lane each; the 7-bit compare only.  Measured on B200
// (cfg2): 13% faster per tree in one launch, still 4% faster split over 4 launches, so
// they are the default up to kMaxParamLaunches launches.
int use_param_descriptors(const obt_model* m, int tpw) {
  const int forced = opt(OPT_DESC_SOURCE);
  if (forced == 0) return 0;
  if (m->compare_mode != 7 || tpw != 1) return 0;
  const int per = param_chunks_per_launch(m);
  if (per < 1) return 0;
  if (forced == 1) return 1;
  return (m->n_chunks + per - 1) / per <= kMaxParamLaunches ? 1 : 0;
}

// ---------------------------------------------------------------------------
// kernel dispatch: the instantiations live in k_*.cu (compiled in parallel)
// Lanes per bucket word (measured on B200): depth-split lanes add descriptor and shuffle
// traffic to the shared-memory pipe, so they pay only when the tile -- F bytes per
// object -- leaves few warps (F = 500: 2 lanes); subject to TPW | depth.  OBT_TPW overrides.
int choose_tpw(const obt_model* m, int tile, bool write_idx) {
  if (write_idx || m->depth_inst > 8) return 1;
  const int words = tile / 4;
  const int cap = obt::kApplyMaxThreads - obt::kApplyProducerThreads;
  if (const int t = opt(OPT_TPW); t > 0) {
    if ((t == 2 || t == 4) && m->depth_inst % t == 0 && words * t <= cap) return t;
    return 1;
  }
  // measured at config 4 (F = 500, 4-8 warps): TPW 2 beats 1 by 1.6x and 4 by 1.3x
  if (words >= 192) return 1;
  return (m->depth_inst % 2 == 0 && words * 2 <= cap) ? 2 : 1;
}

// Lanes per bucket word for one predict, decided once (the quantize launch lays the
// buckets out for it).
int apply_lanes(const obt_model* m, int tile, bool write_idx) {
  if (m->multi_style) return 1;
  if (opt(OPT_DESC_SOURCE) == 1) return 1;  // the parameter-bank kernels have one lane per word
  return choose_tpw(m, tile, write_idx);
}

// Features per CTA (grid.y chunk): the fewest chunks whose Eytzinger arrays fit
// `budget` bytes, split evenly (multiples of the 8-feature step); small batches split
// finer until the grid has ~2 CTAs per SM, so a 10k-object batch is not quantized by 10
// CTAs.
int quantize_chunk_bytes(const obt_model* m, size_t per_feature, int64_t n_slots, size_t budget) {
  const int F = m->n_features;
  int chunks = per_feature ? (int)std::max<size_t>(1, (F * per_feature + budget - 1) / budget) : 1;
  int fc = 0;
  for (;; ++chunks) {
    fc = ((F + chunks - 1) / chunks + 7) / 8 * 8;
    if ((size_t)fc * per_feature <= budget || fc == 8) break;
  }
  // Chunks that start on 32-feature (128-byte) boundaries of the object-major rows: the
  // TMA reads of neighbouring chunks then never share an L2 line (balanced chunks of
  // 100 features read 0.99 GB for cfg2's 0.8 GB of features)
  if (chunks > 1 && per_feature) {
    const int fit = (int)(budget / per_feature) / 32 * 32;
    if (fit >= 32) fc = std::min(fit, (F + 7) / 8 * 8);
  }
  const int64_t blocks = (n_slots + obt::kQuantBlock - 1) / obt::kQuantBlock;
  while (fc > 8 && blocks * ((F + fc - 1) / fc) < 2 * m->sm_count) fc = std::max(8, (fc / 2 + 7) / 8 * 8);
  return fc;
}

int quantize_chunk(const obt_model* m, const BorderTable& bt, int64_t n_slots, size_t budget) {
  return quantize_chunk_bytes(m, bt.levels > 0 ? (size_t)bt.pitch * 4 : 0, n_slots, budget);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

#ifndef OBT_QUANT_RB
#define OBT_QUANT_RB 8
#endif
#ifndef OBT_TMA_L2
#define OBT_TMA_L2 128  // measured: 256 B reads 1.2 GB for 0.8 GB of features, 128 B 0.99 GB, same time
#endif
CUtensorMapL2promotion tma_l2_promotion() {
  return OBT_TMA_L2 == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : OBT_TMA_L2 == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : OBT_TMA_L2 == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                             : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// K1L over K1t when its dependent shared loads per value (one cell byte + kmax border
// compares) are fewer than the Eytzinger search's (levels - 2, the top two from
// registers).  Measured on B200: cfg2 (kmax 1 vs 6 levels) 0.219 vs 0.247 ms; cfg4
// (kmax 4 vs 7 levels) 6.12 vs 4.92 ms; cfg5 (kmax 3 vs 6 levels) 17.3 vs 16.6 ms.
// OBT_QUANT_LUT=1 forces K1L wherever its tables exist, 0 disables it.
bool lut_preferred(const obt_model* m) {
  if (m->used_lut.kmax <= 0) return false;
  if (opt(OPT_QUANT_LUT) == 0) return false;
  if (opt(OPT_QUANT_LUT) == 1) return true;
  // 1024-cell tables (1 KB per feature) pay off only against deep searches: cfg4 (7
  // levels) 4.49 vs 4.95 ms, cfg5 (6 levels) 17.1 vs 16.5 ms
  if (m->used_lut.cells > 256 && m->used.levels < 7) return false;
  return 1 + m->used_lut.kmax < m->used.levels - 2;
}

// Tiled output may have a second region (objects >= split, tiles of tile2 into out2):
// the tail-wave region of predict_impl, quantized by the same launch.
struct SecondRegion {
  int64_t split = -1;  // < 0: none
  uint8_t* out = nullptr;
  int tile = 0;
  bool swizzle = false;
};

int launch_quantize(const obt_model* m, const float* x, int64_t n, int layout, uint8_t* out, bool tiled,
                    int tile, int64_t n_slots, bool swizzle, cudaStream_t stream, SecondRegion r2 = SecondRegion()) {
  const BorderTable& bt = tiled ? m->used : m->full;
  const int F = m->n_features;
  obt::QuantizeParams p{};
  p.x = x;
  p.n = n;
  p.n_slots = n_slots;
  p.n_features = F;
  p.eytz = bt.d;
  p.eytz_pitch = bt.pitch;
  p.out = out;
  p.tile = tile;
  p.two = 2;
  p.swizzle = swizzle ? 1 : 0;
  p.ld = n;
  p.split = r2.split < 0 ? n_slots : r2.split;
  p.out2 = r2.out;
  p.tile2 = r2.tile > 0 ? r2.tile : tile;
  p.swizzle2 = r2.swizzle ? 1 : 0;
  const unsigned blocks = (unsigned)((n_slots + obt::kQuantBlock - 1) / obt::kQuantBlock);

  // K1t / K1L: TMA-staged rows (object-major, tiled, 16-byte row pitch and alignment);
  // K1L (cell tables) wherever the used-border set admits them
  const LutTable& lt = m->used_lut;
  const bool use_lut = tiled && lut_preferred(m);
  obt::QuantTmaFn tfn = use_lut ? pick_quant_lut(lt.kmax, lt.cells) : pick_quant_tma(bt.levels);
  if (tiled && layout == OBT_LAYOUT_OBJECT_MAJOR && F % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      tfn && encode_tiled()) {
    // two CTAs per SM: each gets half the SM's shared memory less the per-CTA reserve
    // (one CTA per SM with every feature of its rows measured slower: cfg2 0.239 vs 0.198 ms)
    const size_t half = (size_t)(m->smem_optin + 1024) / 2 - 1024;
    const size_t lut_fixed = use_lut ? 256 + 32 : 0;  // 256-byte alignment of the tables
    const int fc = use_lut ? quantize_chunk_bytes(m, (size_t)lt.cells + lt.rec_stride, n_slots,
                                                  half - obt::kQTSmemFixed - lut_fixed)
                           : quantize_chunk(m, bt, n_slots, half - obt::kQTSmemFixed);
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)F * 4};
    const cuuint32_t box[2] = {(cuuint32_t)obt::kQuantStep, (cuuint32_t)obt::kQTBoxRows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                      tma_l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
      p.chunk_features = fc;
      p.lut = lt.d_lut;
      p.lrec = lt.d_rec;
      p.lrec_stride = lt.rec_stride;
      p.chunk_inner = use_lut ? 1 : 0;
      const size_t smem = use_lut ? obt::kQTSmemFixed + lut_fixed + (size_t)std::min(fc, F) * (lt.cells + lt.rec_stride)
                                  : obt::kQTSmemFixed + (bt.levels > 0 ? (size_t)std::min(fc, F) * bt.pitch * 4 : 16);
      CUDA_TRY(cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));
      // K1L: up to OBT_QUANT_RB row blocks per CTA (the chunk's tables staged once for
      // all of them) while the grid keeps >= 8 waves of 2 CTAs per SM.  Config 4 (1.5 KB
      // of tables per feature): 1 / 4 / 8 blocks 4.57 / 3.85 / 3.81 ms; config 2 keeps 1
      // (fewer, longer CTAs measured 0.243 vs 0.204 ms there)
      const unsigned n_fch = (unsigned)((F + fc - 1) / fc);
      int rb = use_lut ? OBT_QUANT_RB : 1;
      while (rb > 1 && (blocks + rb - 1) / rb * n_fch < 16u * (unsigned)m->sm_count) --rb;
      p.row_blocks = rb;
      const dim3 grid((blocks + rb - 1) / rb * n_fch);
      tfn<<<grid, obt::kQTThreads, smem, stream>>>(map, p);
      ++g_launches;
      CUDA_TRY(cudaGetLastError());
      return OBT_OK;
    }
  }

  // K1 (rows loaded by each lane): the cell-table search where K1L would run, else Eytzinger
  const bool ldg_lut = use_lut;
  QuantFn fn = ldg_lut ? obt::pick_quant_ldg_lut(lt.kmax, lt.cells, layout) : pick_quant(bt.levels, layout, tiled);
  if (!fn) return fail(OBT_E_UNSUPPORTED, "no quantize kernel for %d levels", bt.levels);
  const int fc = ldg_lut ? quantize_chunk_bytes(m, (size_t)lt.cells + lt.rec_stride, n_slots, obt::kQuantSmem - 256)
                         : quantize_chunk(m, bt, n_slots, obt::kQuantSmem);
  const size_t smem = ldg_lut ? 256 + (size_t)std::min(fc, F) * (lt.cells + lt.rec_stride)
                              : (bt.levels > 0 ? (size_t)std::min(fc, F) * bt.pitch * 4 : 16);
  p.chunk_features = fc;
  p.lut = lt.d_lut;
  p.lrec = lt.d_rec;
  p.lrec_stride = lt.rec_stride;
  // the opt-in maximum, not this launch's size: the attribute is per function and
  // process-wide, so every caller must set the same value (concurrent launches race otherwise)
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));
  const dim3 grid(blocks * (unsigned)((F + fc - 1) / fc));
  fn<<<grid, obt::kQuantThreads, smem, stream>>>(p);
  ++g_launches;
  CUDA_TRY(cudaGetLastError());
  return OBT_OK;
}

// One or more launches of the apply kernel folding all trees in order; with the
// parameter-bank path each launch carries its trees' descriptors, and launches after
// the first continue the fold from the accumulators the previous one left in `out`.
// `tpw` (lanes per bucket word, from apply_lanes) must match the layout the quantize
// launch wrote: tpw > 1 reads the swizzled K2s layout.
int launch_apply(obt_model* m, const uint8_t* q, int64_t n, int tile, int tpw, double* out, uint16_t* idx_out,
                 int tree_begin, int tree_end, cudaStream_t stream, uint32_t* flags = nullptr) {
  const bool write_idx = idx_out != nullptr;
  const int dsrc = use_param_descriptors(m, tpw);
  const TilePlan* tp = nullptr;
  int rc = get_tile_plan(m, tile, tpw > 1 ? 1 : write_idx ? 2 : 0, &tp);
  if (rc != OBT_OK) return rc;
  // leaf selection: shared-memory gathers, or (path option leaf_select = 1) warp shuffles
  // from a register-resident table where the table is one word per lane
  int leaf_code = m->leaf_storage;
  if (opt(OPT_LEAF_SELECT) == 1 && !write_idx && tpw == 1 &&
      ((m->leaf_storage == 2 && m->depth_inst <= 6) || (m->leaf_storage == 1 && m->depth_inst <= 5)))
    leaf_code = m->leaf_storage == 2 ? 3 : 4;
  ApplyKernel k = tpw > 1 ? pick_split(m->depth_inst, m->compare_mode, m->leaf_storage, tpw)
                          : pick_apply(m->depth_inst, m->compare_mode, leaf_code, write_idx, dsrc);
  if (!k.fn) return fail(OBT_E_UNSUPPORTED, "no apply kernel for depth %d", m->depth_inst);
  const int64_t n_tiles = (n + tile - 1) / tile;
  // parameter-bank launches stream tables-only ring chunks (their descriptors travel in
  // the kernel parameters)
  const bool tables_only = dsrc && tp->d_tables;
  const uint32_t ring_chunk = tables_only ? tp->tables_chunk_bytes : m->chunk_bytes;
  const int stages = kStages;
  const size_t smem = 512 + (size_t)stages * ring_chunk + (size_t)m->n_features * tile;
  if (smem > (size_t)m->smem_optin)
    return fail(OBT_E_UNSUPPORTED, "tile of %d objects needs %zu bytes of shared memory", tile, smem);
  CUDA_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));

  obt::ApplyParams p{};
  p.q = q;
  p.chunks = tables_only ? tp->d_tables : tp->d_chunks;
  p.out = out;
  p.idx_out = idx_out;
  p.n = n;
  p.tile = tile;
  p.chunk_trees = m->chunk_trees;
  p.chunk_bytes = ring_chunk;
  p.desc_bytes = tables_only ? 0u : m->desc_bytes;
  p.q_tile_bytes = (uint32_t)((size_t)m->n_features * tile);
  p.n_stages = stages;
  p.tree_begin = tree_begin;
  p.tree_end = tree_end;
  p.scale = m->scale;
  p.bias = m->bias;
  const dim3 grid((unsigned)n_tiles),
      block((unsigned)(obt::kApplyProducerThreads + tile / (4 * k.words) * k.tpw));
  const int per = dsrc ? param_chunks_per_launch(m) : std::max(m->n_chunks, 1);
  const int n_launch = m->n_chunks == 0 ? 1 : (m->n_chunks + per - 1) / per;
  // Bucket tiles of one region are re-read by every launch.  Launches alternate the tile
  // order (the first runs last-to-first: the quantize launch wrote the high tiles last),
  // so each launch's first wave finds the previous pass's last tiles still in L2
  // (cfg2 apply 1.035 -> 1.024 ms; an L2 prefetch of the next wave's tile measured no gain).
  // Launch chaining (parameter-bank folds of several launches): launch k > 0 goes out
  // as a programmatic dependent launch, so its CTAs start on the SMs launch k - 1's
  // partial last wave leaves idle; a CTA waits only for its own tile's carry (per-tile
  // flags).  Not under stream capture.  Path option "pdl" = 0 disables it.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
  const bool chain = flags && dsrc && !write_idx && n_launch > 1 && k.words == 1 && cap == cudaStreamCaptureStatusNone &&
                     opt(OPT_PDL) != 0;
  if (chain) CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)n_tiles * 4, stream));
  p.tile_flags = flags;
  const bool alternate = !chain;  // chained launches keep one order
  p.l2_wave = 0;
  for (int l = 0; l < n_launch; ++l) {
    p.chunk_begin = l * per;
    p.chunk_end = std::min(m->n_chunks, (l + 1) * per);
    p.first = l == 0;
    p.last = l == n_launch - 1;
    // chained launches share one order; last-to-first by default, so the first launch's
    // first waves read the tiles the quantize wrote last (still in L2)
    p.reverse = chain ? 1 : (alternate && (l % 2 == 0) ? 1 : 0);
    p.flag_wait = chain ? l : 0;
    p.flag_set = chain && l < n_launch - 1 ? l + 1 : 0;
    if (dsrc) {
      auto* args = &m->param_args;  // scratch; the driver copies parameters at launch
      std::lock_guard<std::mutex> lock(m->mu);
      args->p = p;
      const size_t per_tree = 2 * (size_t)m->depth_inst;
      const size_t words = (size_t)(p.chunk_end - p.chunk_begin) * m->chunk_trees * per_tree;
      std::memcpy(args->desc, tp->param_desc.data() + (size_t)p.chunk_begin * m->chunk_trees * per_tree, words * 4);
      void* kargs[] = {args};
      if (chain && l > 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_TRY(cudaLaunchKernelExC(&cfg, k.fn, kargs));
      } else {
        CUDA_TRY(cudaLaunchKernel(k.fn, grid, block, kargs, smem, stream));
      }
    } else {
      obt::ApplyArgs<0> small{p};
      void* kargs[] = {&small};
      CUDA_TRY(cudaLaunchKernel(k.fn, grid, block, kargs, smem, stream));
    }
    ++g_launches;
  }
  return OBT_OK;
}

size_t fan_smem(const obt_model* m);
int fan_stages(const obt_model* m);

int launch_fan(obt_model* m, const uint8_t* q, int64_t n, double* out, cudaStream_t stream) {
  const void* fn = obt::pick_fan(m->depth_inst, m->compare_mode, m->leaf_storage);
  if (!fn) return fail(OBT_E_UNSUPPORTED, "no fanned-out apply kernel for depth %d", m->depth_inst);
  const TilePlan* tp = nullptr;
  int rc = get_tile_plan(m, 128, 0, &tp);
  if (rc != OBT_OK) return rc;
  obt::ApplyParams p{};
  p.q = q;
  p.chunks = tp->d_chunks;
  p.out = out;
  p.n = n;
  p.tile = 128;
  p.chunk_trees = m->chunk_trees;
  p.chunk_begin = 0;
  p.chunk_end = m->n_chunks;
  p.chunk_bytes = m->chunk_bytes;
  p.desc_bytes = m->desc_bytes;
  p.q_tile_bytes = (uint32_t)((size_t)m->n_features * 128);
  p.n_stages = fan_stages(m);
  p.tree_begin = 0;
  p.tree_end = m->n_trees;
  p.first = 1;
  p.last = 1;
  p.scale = m->scale;
  p.bias = m->bias;
  const size_t smem = fan_smem(m);
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));
  void* kargs[] = {&p};
  const dim3 grid((unsigned)((n + 127) / 128)), block(obt::kFanThreads);
  CUDA_TRY(cudaLaunchKernel(fn, grid, block, kargs, smem, stream));
  ++g_launches;
  return OBT_OK;
}

// K2w records for the 256-object tile, in the predict path's level order; null trees
// (sentinel descriptors, -0.0 leaves) pad the last chunk.
using obt::kWideChunkTrees;
// Shared memory of K2w with ts table stages and ns descriptor/panel slots (dsrc 1: the
// descriptors travel in the kernel parameters, no descriptor ring).
size_t wide_smem(const obt_model* m, int ts, int ns, int dsrc) {
  const int DI = m->depth_inst;
  return obt::kWideSmemSlack + (size_t)ts * obt::wide_tables_bytes(DI, m->leaf_storage) +
         (size_t)ns * ((dsrc ? 0 : obt::wide_desc_bytes(DI)) + obt::wide_panel_bytes(kWideChunkTrees)) +
         (((size_t)m->n_features * obt::kWideTile + 15) & ~(size_t)15);
}
// Ring depths: 3 table stages (2 if that is all that fits) and as many descriptor /
// panel slots as fit, up to 12 (the index warps' lead over the fold); then more table
// stages while they fit, up to 8: small chunks (config 2: 4 KB of tables folded in
// ~0.3 us) need more than two chunks of lead to cover a bulk copy's L2 latency.
bool wide_rings(const obt_model* m, int dsrc, int* ts, int* ns) {
  for (int t = 3; t >= 2; --t) {
    int n = 12;
    while (n >= 4 && wide_smem(m, t, n, dsrc) > (size_t)m->smem_optin) --n;
    if (n >= 4) {
      while (t < obt::kWideMaxTStages && wide_smem(m, t + 1, n, dsrc) <= (size_t)m->smem_optin) ++t;
      *ts = t; *ns = n;
      return true;
    }
  }
  return false;
}
// Descriptor source of K2w: the shared-memory ring (one launch) unless the path option
// asks for the parameter bank.  The bank (16 launches at config 4, each re-reading the
// 4 GB bucket matrix: 64 GB of DRAM reads per predict instead of 4) measured only 1.4%
// faster (47.29 vs 47.95 ms), not worth 16x the HBM traffic.
int wide_dsrc() { return opt(OPT_DESC_SOURCE) == 1 ? 1 : 0; }
int build_wide_plan(obt_model* m, WidePlan& w) {
  const int DI = m->depth_inst;
  const uint32_t stride = obt::wide_table_stride(DI, m->leaf_storage);
  for (int ds = 0; ds < 2; ++ds) {
    if (!wide_rings(m, ds, &w.tstages[ds], &w.slots[ds])) return OBT_E_UNSUPPORTED;
    w.smem[ds] = wide_smem(m, w.tstages[ds], w.slots[ds], ds);
  }
  w.n_chunks = (m->n_trees + kWideChunkTrees - 1) / kWideChunkTrees;
  const uint32_t dpt = obt::kWideDescBytes(DI), db = obt::wide_desc_bytes(DI);
  const uint32_t tb = obt::wide_tables_bytes(DI, m->leaf_storage);
  const size_t nch = (size_t)std::max(w.n_chunks, 1);
  std::vector<uint8_t> hd(nch * db, 0), ht(nch * tb, 0);
  std::vector<uint32_t> words((size_t)DI * 2);
  w.bank.assign(nch * kWideChunkTrees * 2 * DI, 0);
  for (int t = 0; t < w.n_chunks * kWideChunkTrees; ++t) {
    const int c = t / kWideChunkTrees, tl = t % kWideChunkTrees;
    tree_descriptors(m, t, obt::kWideTile, words.data(), true);
    std::memcpy(hd.data() + (size_t)c * db + (size_t)tl * dpt, words.data(), (size_t)DI * 8);
    std::memcpy(w.bank.data() + (size_t)t * 2 * DI, words.data(), (size_t)DI * 8);
    uint8_t* leaf_dst = ht.data() + (size_t)c * tb + (size_t)tl * stride;
    if (t < m->n_trees) ordered_leaves(m, t, leaf_dst);
    else write_null_leaves(m, leaf_dst);
  }
  CUDA_TRY(cudaMalloc(&w.d_desc, hd.size()));
  CUDA_TRY(cudaMemcpy(w.d_desc, hd.data(), hd.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&w.d_tables, ht.size()));
  CUDA_TRY(cudaMemcpy(w.d_tables, ht.data(), ht.size(), cudaMemcpyHostToDevice));
  return OBT_OK;
}

int get_wide_plan(obt_model* m, const WidePlan** out) {
  std::lock_guard<std::mutex> lock(m->mu);
  if (!m->wide) {
    std::unique_ptr<WidePlan> w(new WidePlan());
    const int rc = build_wide_plan(m, *w);
    if (rc != OBT_OK) return rc == OBT_E_UNSUPPORTED ? fail(rc, "K2w does not fit shared memory") : rc;
    m->wide = std::move(w);
  }
  *out = m->wide.get();
  return OBT_OK;
}

// K2w where the K2 tile would hold few objects: the bucket tile (F bytes per object)
// leaves K2 too few warps per SM (config 4, F = 500: 256 objects, 2 warps).
bool wide_eligible(const obt_model* m) {
  if (m->multi_style || m->depth_inst > 8 || m->n_trees == 0) return false;
  int ts = 0, ns = 0;
  if (!wide_rings(m, wide_dsrc(), &ts, &ns)) return false;
  if (!obt::pick_wide(m->depth_inst, m->compare_mode, m->leaf_storage, wide_dsrc())) return false;
  if (opt(OPT_WIDE) == 0) return false;
  if (opt(OPT_WIDE) == 1) return true;
  return plan_tile(m, (int64_t)1 << 40) <= 512;
}

int launch_wide(obt_model* m, const uint8_t* q, int64_t n, double* out, cudaStream_t stream) {
  const int ds = wide_dsrc();
  const void* fn = obt::pick_wide(m->depth_inst, m->compare_mode, m->leaf_storage, ds);
  if (!fn) return fail(OBT_E_UNSUPPORTED, "no K2w kernel for depth %d", m->depth_inst);
  const WidePlan* w = nullptr;
  int rc = get_wide_plan(m, &w);
  if (rc != OBT_OK) return rc;
  static thread_local obt::WideArgs<1> args;  // the driver copies the parameters at launch
  obt::WideParams& p = args.p;
  p = obt::WideParams{};
  p.q = q;
  p.desc = w->d_desc;
  p.tables = w->d_tables;
  p.out = out;
  p.n = n;
  p.n_tiles = (n + obt::kWideTile - 1) / obt::kWideTile;
  p.q_tile_bytes = (uint32_t)((size_t)m->n_features * obt::kWideTile);
  p.n_tstages = w->tstages[ds];
  p.n_slots = w->slots[ds];
  p.scale = m->scale;
  p.bias = m->bias;
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));
  const dim3 grid((unsigned)std::min<int64_t>(p.n_tiles, m->sm_count)),
      block(32 * (3 + obt::kWideIndexWarps + obt::kWideFoldWarps));
  // one launch (descriptor ring), or one per parameter bank of descriptors, the fold
  // carried through `out` between launches
  const int per = ds ? obt::wide_bank_chunks(m->depth_inst) : std::max(w->n_chunks, 1);
  const int n_launch = std::max(1, (w->n_chunks + per - 1) / per);
  const size_t per_chunk = (size_t)kWideChunkTrees * 2 * m->depth_inst;
  for (int l = 0; l < n_launch; ++l) {
    p.chunk_begin = l * per;
    p.n_chunks = std::min(w->n_chunks, (l + 1) * per) - p.chunk_begin;
    p.first = l == 0;
    p.last = l == n_launch - 1;
    if (ds) std::memcpy(args.desc, w->bank.data() + (size_t)p.chunk_begin * per_chunk, (size_t)p.n_chunks * per_chunk * 4);
    void* kargs[] = {&args};
    CUDA_TRY(cudaLaunchKernel(fn, grid, block, kargs, w->smem[ds], stream));
    ++g_launches;
  }
  return OBT_OK;
}

int launch_multi_staged(obt_model* m, const uint8_t* q, int64_t n, double* out, cudaStream_t stream) {
  int di = 0;
  const void* fn = obt::pick_multi_staged(m->depth_inst, m->compare_mode, m->n_outputs, m->leaf_storage, &di);
  if (!fn || di != m->depth_inst) return fail(OBT_E_UNSUPPORTED, "no staged multi-output kernel for depth %d", di);
  obt::StagedParams p{};
  p.q = q;
  p.desc = m->d_multi_desc;
  p.leaves = static_cast<const float*>(m->d_multi_leaves);
  p.out = out;
  p.n = n;
  p.n_features = m->n_features;
  p.tree_begin = 0;
  p.tree_end = m->n_trees;
  p.first = 1;
  p.last = 1;
  p.n_stages = m->staged_stages;
  p.table_bytes = m->staged_table_bytes;
  p.stage_bytes = m->staged_stage_bytes;
  p.scale = m->scale;
  p.bias = m->bias;
  const size_t smem = 128 + 128 + (size_t)p.n_stages * p.stage_bytes;
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem_optin));
  void* kargs[] = {&p};
  const dim3 grid((unsigned)((n + obt::kStagedTile - 1) / obt::kStagedTile)), block(obt::kStagedThreads);
  CUDA_TRY(cudaLaunchKernel(fn, grid, block, kargs, smem, stream));
  ++g_launches;
  return OBT_OK;
}

int launch_multi(obt_model* m, const uint8_t* q, int64_t n, double* out, cudaStream_t stream) {
  if (m->multi_staged) return launch_multi_staged(m, q, n, out, stream);
  int di = 0;
  const void* fn = obt::pick_multi(m->depth_inst, m->compare_mode, m->leaf_storage, m->n_outputs, &di);
  if (!fn || di != m->depth_inst) return fail(OBT_E_UNSUPPORTED, "no multi-output kernel for depth %d, %d outputs",
                                             m->depth_inst, m->n_outputs);
  obt::MultiParams p{};
  p.q = q;
  p.desc = m->d_multi_desc;
  p.leaves = m->d_multi_leaves;
  p.out = out;
  p.n = n;
  p.n_features = m->n_features;
  p.tile = kMultiTile;
  p.n_outputs = m->n_outputs;
  p.tree_begin = 0;
  p.tree_end = m->n_trees;
  p.first = 1;
  p.last = 1;
  p.scale = m->scale;
  p.bias = m->bias;
  void* kargs[] = {&p};
  const int threads = obt::kMultiThreads;
  const int64_t n_tiles = (n + kMultiTile - 1) / kMultiTile;
  // persistent grid: the resident CTAs loop over the tiles
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));
  const int64_t resident = (int64_t)std::max(per_sm, 1) * m->sm_count;
  const dim3 grid((unsigned)std::min<int64_t>(n_tiles, resident)), block(threads);
  CUDA_TRY(cudaLaunchKernel(fn, grid, block, kargs, 0, stream));
  ++g_launches;
  return OBT_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

size_t workspace_bytes(const obt_model* m, int64_t n, int tile) {
  const int64_t n_tiles = (n + tile - 1) / tile;
  return (size_t)n_tiles * tile * m->n_features;
}

// One predict over up to two object ranges: whole waves of the main tile (one tile per
// SM per wave), then the remainder -- what would be a partial last wave -- re-tiled so
// every SM gets a share.  The smaller tail tiles run with depth-split lanes when they
// leave few warps, so the tail finishes sooner than one more wave of main tiles
// (cfg2: 977 tiles = 6.6 waves of 1024 objects).  OBT_TAIL_SPLIT=0 disables it.
struct Regions {
  int n_reg = 1;
  int64_t begin[2] = {0, 0}, count[2] = {0, 0};
  int tile[2] = {-1, -1};
  bool fan = false;   // K2f: 128-object blocks, trees fanned out over the CTA's warps
  bool wide = false;  // K2w: 256-object tiles, persistent warp-specialised CTAs
};

// K2f for small batches: the 128-object blocks fill no more than two waves, the model
// has trees for every compute warp, and the CTA's ring, value panel and bucket tile fit.
// OBT_FAN=0 / 1 forbids / forces it (where it can run).
size_t fan_fixed_smem(const obt_model* m) {
  return 512 + 2 * (size_t)m->chunk_trees * 128 * leaf_size(m->leaf_storage) + (size_t)m->n_features * 128;
}
int fan_stages(const obt_model* m) {
  const int64_t room = ((int64_t)m->smem_optin - (int64_t)fan_fixed_smem(m)) / (int64_t)m->chunk_bytes;
  return (int)std::max<int64_t>(0, std::min<int64_t>({room, 8, std::max(m->n_chunks, 2)}));
}
size_t fan_smem(const obt_model* m) { return fan_fixed_smem(m) + (size_t)fan_stages(m) * m->chunk_bytes; }
bool fan_eligible(const obt_model* m, int64_t n) {
  if (m->multi_style || m->depth_inst > 8 || m->n_trees == 0 || n <= 0) return false;
  if (fan_stages(m) < 2 || fan_smem(m) > (size_t)m->smem_optin) return false;
  if (!obt::pick_fan(m->depth_inst, m->compare_mode, m->leaf_storage)) return false;
  if (opt(OPT_FAN) == 0) return false;
  if (opt(OPT_FAN) == 1) return true;
  const int64_t blocks = (n + 127) / 128;
  return blocks <= 2 * (int64_t)m->sm_count && m->n_trees >= 4 * obt::kFanComputeWarps;
}

Regions plan_regions(const obt_model* m, int64_t n, bool split_ok) {
  Regions r;
  r.count[0] = n;
  if (split_ok && fan_eligible(m, n)) {
    r.tile[0] = 128;
    r.fan = true;
    return r;
  }
  if (split_ok && wide_eligible(m)) {
    r.tile[0] = obt::kWideTile;
    r.wide = true;
    return r;
  }
  r.tile[0] = plan_tile(m, n);
  const int split = opt(OPT_TAIL_SPLIT);  // 0 never, 1 whenever a tail exists
  if (!split_ok || r.tile[0] < 0 || m->multi_style || split == 0) return r;
  // Not behind a parameter-bank main region: the tail then runs with shared-memory
  // descriptors at ~60% of the main region's rate, and one more launch; measured at
  // cfg2 (3 parameter-bank launches): apply 1.045 ms without the split, 1.081 with it.
  if (split != 1 && use_param_descriptors(m, apply_lanes(m, r.tile[0], false))) return r;
  const int64_t wave = (int64_t)m->sm_count * r.tile[0];
  const int64_t full = n / wave * wave, rest = n - full;
  if (full == 0 || rest == 0) return r;
  int64_t tb = (rest + m->sm_count - 1) / m->sm_count;
  tb = (tb + kTileQuantum - 1) / kTileQuantum * kTileQuantum;
  if (tb >= r.tile[0]) return r;
  r.n_reg = 2;
  r.count[0] = full;
  r.begin[1] = full;
  r.count[1] = rest;
  r.tile[1] = (int)tb;
  return r;
}

size_t regions_bucket_bytes(const obt_model* m, const Regions& r) {
  size_t b = 0;
  for (int i = 0; i < r.n_reg; ++i) b += workspace_bytes(m, r.count[i], r.tile[i]);
  return b;
}

// Bucket tiles of every region, then one 32-bit launch-chaining flag per tile of region 0.
size_t regions_workspace(const obt_model* m, const Regions& r) {
  const int64_t tiles0 = r.tile[0] > 0 ? (r.count[0] + r.tile[0] - 1) / r.tile[0] : 0;
  return regions_bucket_bytes(m, r) + (size_t)((tiles0 * 4 + 255) / 256 * 256);
}

int check_layout(int layout) {
  if (layout != OBT_LAYOUT_OBJECT_MAJOR && layout != OBT_LAYOUT_FEATURE_MAJOR)
    return fail(OBT_E_INVALID, "unknown layout %d", layout);
  return OBT_OK;
}

}  // namespace

extern "C" {

int obt_abi_version(void) { return OBT_ABI_VERSION; }

int obt_set_path_option(const char* name, int value) {
  if (!name) return fail(OBT_E_INVALID, "null option name");
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!strcmp(name, kPathOptionNames[i])) {
      g_opt[i].store(value < 0 ? -1 : value, std::memory_order_relaxed);
      return OBT_OK;
    }
  return fail(OBT_E_INVALID, "unknown path option '%s'", name);
}

int obt_get_path_option(const char* name, int* value) {
  if (!name || !value) return fail(OBT_E_INVALID, "null argument");
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!strcmp(name, kPathOptionNames[i])) {
      *value = opt((PathOption)i);
      return OBT_OK;
    }
  return fail(OBT_E_INVALID, "unknown path option '%s'", name);
}

const char* obt_last_error(void) { return g_error.c_str(); }

int obt_last_launch_count(void) { return g_launches; }

int obt_model_create(const obt_model_desc* d, int device, obt_model** out) {
  if (!out) return fail(OBT_E_INVALID, "null output handle");
  *out = nullptr;
  int rc = validate(d);
  if (rc != OBT_OK) return rc;
  int n_dev = 0;
  CUDA_TRY(cudaGetDeviceCount(&n_dev));
  if (device < 0 || device >= n_dev) return fail(OBT_E_INVALID, "device %d not present (%d visible)", device, n_dev);
  DeviceGuard guard(device);

  std::unique_ptr<obt_model> m(new obt_model());
  m->device = device;
  m->n_features = d->n_features;
  m->n_trees = d->n_trees;
  m->max_depth = d->n_trees > 0 ? d->max_depth : 0;
  m->n_outputs = d->n_outputs;
  m->precision = d->precision;
  m->scale = d->scale;
  m->bias = d->bias;
  m->multi_style = d->n_outputs > 1;  // (single-output models join below when K2 cannot hold them)
  m->depth_inst = d->n_trees > 0 ? (m->multi_style ? obt::multi_depth(d->max_depth) : instantiated_depth(d->max_depth))
                                  : (m->multi_style ? 4 : 1);
  CUDA_TRY(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaDeviceGetAttribute(&m->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));

  // Two border tables.  `full` holds every border (obt_quantize_dev returns the
  // reference's buckets).  `used` holds, per feature, only the borders some split
  // references: with R_f the sorted used borders, x > b[u_j] <=> #{i : x > R_f[i]} > j,
  // so the predict path quantizes against R_f and compares with the split's rank j.
  // Fewer borders mean fewer search levels, and <= 127 used borders per feature keep
  // the 7-bit SWAR compare even when a feature has up to 254 borders.
  const int D = m->max_depth;
  std::vector<std::vector<int>> used(d->n_features);
  for (int t = 0; t < m->n_trees; ++t)
    for (int s = 0; s < D; ++s) {
      const int ord = d->split_ordinal[(size_t)t * D + s];
      if (ord != kSentinel) used[d->split_feature[(size_t)t * D + s]].push_back(ord);
    }
  std::vector<std::vector<int>> rank(d->n_features);  // ordinal -> rank in R_f
  std::vector<float> used_borders((size_t)d->n_features * std::max(1, d->border_stride), INFINITY);
  std::vector<int32_t> used_counts(d->n_features, 0);
  for (int f = 0; f < d->n_features; ++f) {
    auto& u = used[f];
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    rank[f].assign(256, -1);
    for (size_t j = 0; j < u.size(); ++j) {
      rank[f][u[j]] = (int)j;
      used_borders[(size_t)f * d->border_stride + j] = d->borders[(size_t)f * d->border_stride + u[j]];
    }
    used_counts[f] = (int32_t)u.size();
  }
  int rc2 = build_border_table(d->borders, d->border_counts, d->n_features, d->border_stride, m->full);
  if (rc2 != OBT_OK) return rc2;
  rc2 = build_border_table(used_borders.data(), used_counts.data(), d->n_features, d->border_stride, m->used);
  if (rc2 != OBT_OK) return rc2;
  rc2 = build_lut_table(used_borders.data(), used_counts.data(), d->n_features, d->border_stride, m->used_lut);
  if (rc2 != OBT_OK) return rc2;
  int umax = 0;
  for (int f = 0; f < d->n_features; ++f) umax = std::max(umax, (int)used_counts[f]);
  m->compare_mode = umax <= 127 ? 7 : 8;

  // leaf bank: binary16 bits, or binary64 stored as fp32 when that is exact
  const size_t per_tree_in = (size_t)1 << D;
  const int C = d->n_outputs;
  if (d->precision == OBT_PRECISION_BINARY16) {
    m->leaf_storage = 2;
  } else {
    bool exact32 = true;
    for (size_t i = 0; i < (size_t)m->n_trees * C * per_tree_in && exact32; ++i) {
      const double v = d->leaves[i];
      const float f = (float)v;
      exact32 = std::isfinite(f) && (double)f == v && !(v == 0.0 && std::signbit(v) != std::signbit(f));
    }
    m->leaf_storage = (exact32 && opt(OPT_LEAF_STORAGE) != 0) ? 1 : 0;
  }

  // K2 holds a 128-object bucket tile (F bytes per object) next to a ring of at least one
  // tree group per stage; a single-output model that leaves no room for that runs on the
  // record path (K5 stages only the bucket rows each tree reads)
  if (!m->multi_style) {
    const int di = m->depth_inst;
    const size_t per_tree_rec = std::max<size_t>((size_t)obt::desc_words_per_tree(di, m->compare_mode) * 4,
                                                 (size_t)di * obt::kSplitDescBytes) +
                                (size_t)obt::leaf_table_stride(di, (int)leaf_size(m->leaf_storage));
    const size_t min_chunk = ((per_tree_rec * obt::tree_group(di) + 255) & ~(size_t)255) + 256;
    if (512 + (size_t)kStages * min_chunk + (size_t)m->n_features * kTileQuantum > (size_t)m->smem_optin) {
      m->multi_style = 1;
      m->depth_inst = obt::multi_depth(std::max(D, 1));
    }
  }
  const int DI = m->depth_inst;

  // splits (ordinals as ranks among the used borders), padded to the instantiated
  // depth with sentinels
  m->split_feature.assign((size_t)m->n_trees * DI, 0);
  m->split_ordinal.assign((size_t)m->n_trees * DI, (uint8_t)kSentinel);
  for (int t = 0; t < m->n_trees; ++t)
    for (int s = 0; s < D; ++s) {
      const int f = d->split_feature[(size_t)t * D + s];
      const int ord = d->split_ordinal[(size_t)t * D + s];
      m->split_feature[(size_t)t * DI + s] = f;
      m->split_ordinal[(size_t)t * DI + s] = ord == kSentinel ? (uint8_t)kSentinel : (uint8_t)rank[f][ord];
    }

  plan_level_order(m.get(), d);

  const size_t per_tree = (size_t)1 << DI;
  const size_t ls = leaf_size(m->leaf_storage);
  if (m->multi_style) {
    if (m->depth_inst < 0 || m->depth_inst > 10 + 2 * (C > 1))
      return fail(OBT_E_UNSUPPORTED, "%d features per object need the staged kernel, which takes depth <= 10",
                  m->n_features);
    // multi-output records, one leaf's C values contiguous in 16-byte rows (K4, K5)
    // K5 (staged tables and rows) for binary32 or binary16 records, C <= 10, depth <= 10,
    // when at least two stages (one tree's table + its bucket rows each) fit shared memory;
    // the binary16 family runs nowhere else
    {
      const int CPs = obt::staged_record_values(C, m->leaf_storage);
      const uint32_t table = (uint32_t)((per_tree * CPs * ls + 15) / 16 * 16);
      const uint32_t stage = (table + (uint32_t)DI * obt::kStagedTile + 127u) & ~127u;
      const int stages = std::min(8, (int)(((size_t)m->smem_optin - 512) / stage));
      int sdi = 0;
      const bool ok = (m->leaf_storage != 0 || C == 1) && C <= 10 && stages >= 2 &&
                      obt::pick_multi_staged(DI, m->compare_mode, C, m->leaf_storage, &sdi) != nullptr && sdi == DI;
      if (ok && (opt(OPT_MULTI_STAGED) != 0 || m->leaf_storage == 2)) {
        m->multi_staged = 1;
        m->staged_stages = stages;
        m->staged_table_bytes = table;
        m->staged_stage_bytes = stage;
      }
    }
    if (m->leaf_storage == 2 && !m->multi_staged)
      return fail(OBT_E_UNSUPPORTED, "binary16 multi-output model does not fit the staged kernel");
    m->multi_slot = m->multi_staged ? obt::staged_record_values(C, m->leaf_storage) * (int)ls
                                    : obt::multi_record_values(m->leaf_storage, C) * (int)ls;
    // records in the predict path's level order (record j' holds reference leaf
    // reference_leaf(perm, DI, j'); entries past 2^D belong to sentinel levels, never read)
    std::vector<uint8_t> rec((size_t)std::max(m->n_trees, 1) * per_tree * m->multi_slot, 0);
    for (int t = 0; t < m->n_trees; ++t)
      for (int c = 0; c < C; ++c)
        for (size_t j = 0; j < per_tree; ++j) {
          const size_t i = reference_leaf(m->level_perm.data() + (size_t)t * DI, DI, j);
          if (i >= per_tree_in) continue;
          const double v = d->leaves[(((size_t)t * C + c) << D) + i];
          uint8_t* dst = rec.data() + ((size_t)t * per_tree + j) * m->multi_slot + (size_t)c * ls;
          if (m->leaf_storage == 0) {
            std::memcpy(dst, &v, 8);
          } else if (m->leaf_storage == 1) {
            const float f = (float)v;
            std::memcpy(dst, &f, 4);
          } else {
            // the binary16 bank (model.py:262-268): the caller's bits, or RNE + saturation
            const uint16_t h = d->leaves_f16 ? d->leaves_f16[(((size_t)t * C + c) << D) + i] : half_bank_entry(v);
            std::memcpy(dst, &h, 2);
          }
        }
    CUDA_TRY(cudaMalloc(&m->d_multi_leaves, rec.size()));
    CUDA_TRY(cudaMemcpy(m->d_multi_leaves, rec.data(), rec.size(), cudaMemcpyHostToDevice));
    // descriptors for the fixed multi-output tile
    std::vector<uint32_t> desc((size_t)std::max(m->n_trees, 1) * DI * 2, 0);
    for (int t = 0; t < m->n_trees; ++t) tree_descriptors(m.get(), t, kMultiTile, desc.data() + (size_t)t * DI * 2);
    CUDA_TRY(cudaMalloc(&m->d_multi_desc, desc.size() * 4));
    CUDA_TRY(cudaMemcpy(m->d_multi_desc, desc.data(), desc.size() * 4, cudaMemcpyHostToDevice));
    *out = m.release();
    return OBT_OK;
  }
  m->leaf_bytes.assign((size_t)m->n_trees * per_tree * ls, 0);
  for (int t = 0; t < m->n_trees; ++t) {
    for (size_t j = 0; j < per_tree_in; ++j) {
      const double v = d->leaves[(size_t)t * per_tree_in + j];
      uint8_t* dst = m->leaf_bytes.data() + ((size_t)t * per_tree + j) * ls;
      if (m->leaf_storage == 0) {
        std::memcpy(dst, &v, 8);
      } else if (m->leaf_storage == 1) {
        const float f = (float)v;
        std::memcpy(dst, &f, 4);
      } else {
        const uint16_t h = d->leaves_f16 ? d->leaves_f16[(size_t)t * per_tree_in + j] : half_bank_entry(v);
        std::memcpy(dst, &h, 2);
      }
    }
  }
  plan_chunks(m.get());
  *out = m.release();
  return OBT_OK;
}

int obt_model_destroy(obt_model* m) {
  if (!m) return OBT_OK;
  DeviceGuard guard(m->device);
  delete m;
  return OBT_OK;
}

int obt_model_info(const obt_model* m, int32_t* n_features, int32_t* n_trees, int32_t* max_depth,
                   int32_t* n_outputs, int32_t* precision, int32_t* leaf_storage, int32_t* compare_mode) {
  if (!m) return fail(OBT_E_INVALID, "null model");
  if (n_features) *n_features = m->n_features;
  if (n_trees) *n_trees = m->n_trees;
  if (max_depth) *max_depth = m->max_depth;
  if (n_outputs) *n_outputs = m->n_outputs;
  if (precision) *precision = m->precision;
  if (leaf_storage) *leaf_storage = m->leaf_storage;
  if (compare_mode) *compare_mode = m->compare_mode;
  return OBT_OK;
}

int obt_model_quantize_kernel(const obt_model* m, int32_t* kind, int32_t* param) {
  if (!m) return fail(OBT_E_INVALID, "null model");
  const bool lut = lut_preferred(m);
  if (kind) *kind = lut ? (m->used_lut.cells == 1024 ? 2 : m->used_lut.cells == 512 ? 3 : 1) : 0;
  if (param) *param = lut ? m->used_lut.kmax : m->used.levels;
  return OBT_OK;
}

int obt_model_multi_kernel(const obt_model* m, int32_t* kind) {
  if (!m || !kind) return fail(OBT_E_INVALID, "null argument");
  *kind = !m->multi_style ? -1 : m->multi_staged ? 2 : 0;
  return OBT_OK;
}

int obt_workspace_size(const obt_model* m, int64_t n, size_t* bytes) {
  if (!m || !bytes) return fail(OBT_E_INVALID, "null argument");
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  const Regions one = plan_regions(m, std::max<int64_t>(n, 1), false), two = plan_regions(m, std::max<int64_t>(n, 1), true);
  if (one.tile[0] < 0) return fail(OBT_E_UNSUPPORTED, "%d features do not fit a 128-object tile", m->n_features);
  *bytes = n == 0 ? 0 : std::max(regions_workspace(m, one), regions_workspace(m, two));
  return OBT_OK;
}

// The library's own stream-ordered pool per device: workspace and staging buffers stay
// cached between calls (no driver round trip at every synchronisation) without touching
// the device's default pool, which belongs to the application.
static cudaMemPool_t workspace_pool(int device) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(device);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;  // fall back to the default pool
  } else {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  pools[device] = pool;
  return pool;
}

static cudaError_t pool_alloc(void** ptr, size_t bytes, int device, cudaStream_t stream) {
  cudaMemPool_t pool = workspace_pool(device);
  return pool ? cudaMallocFromPoolAsync(ptr, bytes, pool, stream) : cudaMallocAsync(ptr, bytes, stream);
}

static int predict_impl(obt_model* m, const float* x, int64_t n, int32_t layout, double* out, uint16_t* idx_out,
                        int tree_begin, int tree_end, void* ws, size_t ws_bytes, cudaStream_t stream,
                        cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_mid = nullptr, cudaEvent_t ev_end = nullptr) {
  const Regions reg = plan_regions(m, n, idx_out == nullptr);
  if (reg.tile[0] < 0) return fail(OBT_E_UNSUPPORTED, "%d features do not fit a 128-object tile", m->n_features);
  const size_t need = regions_workspace(m, reg);
  uint8_t* q = static_cast<uint8_t*>(ws);
  bool owned = false;
  // bucket tiles move by TMA bulk copies (16-byte aligned); predictions are doubles
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(OBT_E_INVALID, "workspace must be 256-byte aligned");
  if (out && (reinterpret_cast<uintptr_t>(out) & 7)) return fail(OBT_E_INVALID, "output must be 8-byte aligned");
  if (idx_out && (reinterpret_cast<uintptr_t>(idx_out) & 1)) return fail(OBT_E_INVALID, "index output must be 2-byte aligned");
  if (x && (reinterpret_cast<uintptr_t>(x) & 3)) return fail(OBT_E_INVALID, "features must be 4-byte aligned");
  if (!q || ws_bytes < need) {
    if (ws && ws_bytes < need) return fail(OBT_E_INVALID, "workspace of %zu bytes, need %zu", ws_bytes, need);
    CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&q), need, m->device, stream));
    owned = true;
  }
  // one quantize launch writes both regions' bucket tiles (each laid out for its tile
  // size and lanes per word), then one apply launch per region
  uint8_t* qr[2] = {q, q + workspace_bytes(m, reg.count[0], reg.tile[0])};
  uint32_t* flags = reinterpret_cast<uint32_t*>(q + regions_bucket_bytes(m, reg));
  int tpw[2] = {1, 1};
  for (int i = 0; i < reg.n_reg; ++i) tpw[i] = (reg.fan || reg.wide) ? 1 : apply_lanes(m, reg.tile[i], idx_out != nullptr);
  if (ev_begin) CUDA_TRY(cudaEventRecord(ev_begin, stream));
  SecondRegion r2;
  int64_t n_slots = ((reg.count[0] + reg.tile[0] - 1) / reg.tile[0]) * (int64_t)reg.tile[0];
  if (reg.n_reg == 2) {
    r2.split = reg.count[0];  // whole waves of whole tiles: a multiple of 128
    r2.out = qr[1];
    r2.tile = reg.tile[1];
    r2.swizzle = tpw[1] > 1;
    n_slots += ((reg.count[1] + reg.tile[1] - 1) / reg.tile[1]) * (int64_t)reg.tile[1];
  }
  int rc = launch_quantize(m, x, n, layout, q, true, reg.tile[0], n_slots, tpw[0] > 1, stream, r2);
  if (rc == OBT_OK && ev_mid) CUDA_TRY(cudaEventRecord(ev_mid, stream));
  for (int i = 0; i < reg.n_reg && rc == OBT_OK; ++i) {
    const int64_t b = reg.begin[i], c = reg.count[i];
    if (m->multi_style) {
      rc = idx_out ? fail(OBT_E_UNSUPPORTED, "leaf-index dumps are implemented for the K2 path (single output, "
                                             "F x 128 bytes of buckets in shared memory)")
                   : launch_multi(m, qr[i], c, out + b * m->n_outputs, stream);
    } else if (reg.fan) {
      rc = launch_fan(m, qr[i], c, out + b, stream);
    } else if (reg.wide) {
      rc = launch_wide(m, qr[i], c, out + b, stream);
    } else {
      rc = launch_apply(m, qr[i], c, reg.tile[i], tpw[i], out ? out + b : nullptr, idx_out, tree_begin, tree_end, stream,
                        i == 0 && reg.n_reg == 1 ? flags : nullptr);
    }
  }
  if (rc == OBT_OK && ev_end) CUDA_TRY(cudaEventRecord(ev_end, stream));
  if (owned) cudaFreeAsync(q, stream);
  return rc;
}

int obt_predict_dev(const obt_model* mc, const float* x, int64_t n, int32_t layout, double* out, void* ws,
                    size_t ws_bytes, void* stream) {
  g_launches = 0;
  obt_model* m = const_cast<obt_model*>(mc);  // only the per-tile chunk cache mutates (locked)
  if (!m) return fail(OBT_E_INVALID, "null model");
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  if (n == 0) return OBT_OK;
  if (!x || !out) return fail(OBT_E_INVALID, "null feature or output pointer");
  DeviceGuard guard(m->device);
  return predict_impl(m, x, n, layout, out, nullptr, 0, 0, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int obt_predict_dev_marked(const obt_model* mc, const float* x, int64_t n, int32_t layout, double* out, void* ws,
                           size_t ws_bytes, void* stream, void* ev_begin, void* ev_mid, void* ev_end) {
  g_launches = 0;
  obt_model* m = const_cast<obt_model*>(mc);
  if (!m) return fail(OBT_E_INVALID, "null model");
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (n <= 0) return n < 0 ? fail(OBT_E_INVALID, "negative object count") : OBT_OK;
  if (!x || !out) return fail(OBT_E_INVALID, "null feature or output pointer");
  DeviceGuard guard(m->device);
  return predict_impl(m, x, n, layout, out, nullptr, 0, 0, ws, ws_bytes, static_cast<cudaStream_t>(stream),
                      static_cast<cudaEvent_t>(ev_begin), static_cast<cudaEvent_t>(ev_mid),
                      static_cast<cudaEvent_t>(ev_end));
}

int obt_event_create(void** event) {
  if (!event) return fail(OBT_E_INVALID, "null event pointer");
  cudaEvent_t e;
  CUDA_TRY(cudaEventCreate(&e));
  *event = e;
  return OBT_OK;
}

int obt_event_record(void* event, void* stream) {
  CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)));
  return OBT_OK;
}

int obt_event_elapsed_ms(void* start, void* end, float* ms) {
  if (!ms) return fail(OBT_E_INVALID, "null output");
  CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(end)));
  CUDA_TRY(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)));
  return OBT_OK;
}

int obt_event_destroy(void* event) {
  if (event) CUDA_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return OBT_OK;
}

int obt_leaf_indices_dev(const obt_model* mc, const float* x, int64_t n, int32_t layout, int32_t tree_begin,
                         int32_t tree_end, uint16_t* idx, void* stream) {
  g_launches = 0;
  obt_model* m = const_cast<obt_model*>(mc);
  if (!m) return fail(OBT_E_INVALID, "null model");
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (tree_begin < 0 || tree_end < tree_begin || tree_end > m->n_trees)
    return fail(OBT_E_INVALID, "tree range [%d, %d) outside 0..%d", tree_begin, tree_end, m->n_trees);
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  if (n == 0 || tree_end == tree_begin) return OBT_OK;
  if (!x || !idx) return fail(OBT_E_INVALID, "null feature or index pointer");
  DeviceGuard guard(m->device);
  return predict_impl(m, x, n, layout, nullptr, idx, tree_begin, tree_end, nullptr, 0,
                      static_cast<cudaStream_t>(stream));
}

int obt_quantize_dev(const obt_model* m, const float* x, int64_t n, int32_t layout, uint8_t* buckets,
                     void* stream) {
  g_launches = 0;
  if (!m) return fail(OBT_E_INVALID, "null model");
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  if (n == 0) return OBT_OK;
  if (!x || !buckets) return fail(OBT_E_INVALID, "null feature or bucket pointer");
  DeviceGuard guard(m->device);
  return launch_quantize(m, x, n, layout, buckets, false, 0, n, false, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

// Pinned staging for pageable feature arrays (the literal drop-in call passes a plain
// numpy array): the driver stages a pageable H2D through its own small pinned buffer at
// ~10 GB/s and blocks the caller.  Here host threads copy each chunk into one of two
// pinned buffers (kept per device, allocated on first use) while the previous chunk's
// DMA and the one before's kernels run.
struct HostStaging {
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  size_t bytes = 0;
  cudaEvent_t h2d_done[2] = {nullptr, nullptr};
};
HostStaging* host_staging(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<HostStaging>> all;
  std::lock_guard<std::mutex> lock(mu);
  auto& s = all[device];
  if (!s) s.reset(new HostStaging());
  return s.get();
}

// memcpy with up to 16 host threads (one per 8 MB piece at least); measured on the GPU
// box's 16 cores from pageable into pinned memory: 14 GB/s on one thread, 51 on 16
// (tools/memcpy_probe.cu)
void parallel_copy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t piece = (size_t)8 << 20;
  const int nt = (int)std::min<size_t>(std::min(16u, hw), (bytes + piece - 1) / piece);
  if (nt <= 1) { std::memcpy(dst, src, bytes); return; }
  const size_t per = (bytes + nt - 1) / nt / 64 * 64 + 64;
  std::vector<std::thread> th;
  size_t next = per;  // piece 0 is this thread's; `next` = first byte not handed out
  try {
    for (int t = 1; t < nt && next < bytes; ++t) {
      const size_t b = next, len = std::min(per, bytes - next);
      th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, len); });
      next += len;
    }
  } catch (...) {
    // no thread to spare (std::system_error): the rest is copied here
  }
  std::memcpy(dst, src, std::min(per, bytes));
  if (next < bytes) std::memcpy(static_cast<char*>(dst) + next, static_cast<const char*>(src) + next, bytes - next);
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

// obt_predict_host over objects [0, n) of a host matrix whose feature-major rows are `ld`
// objects long (ld == n for a whole matrix; an object shard of a feature-major matrix
// keeps the parent's row length).  Object-major input ignores ld.
static int predict_host_impl(obt_model* m, const float* x_host, int64_t n, int64_t ld, int32_t layout,
                             double* out_host, cudaStream_t stream) {
  g_launches = 0;
  int rc = OBT_OK;
  DeviceGuard guard(m->device);
  const int F = m->n_features, C = m->n_outputs;
  // Chunked pipeline: the features of chunk i+1 cross PCIe on a copy stream while chunk
  // i is quantized and applied on `stream`; each chunk's scores go back right behind its
  // compute.  Two device buffers per side; chunks are whole 1024-object blocks of about
  // 128 MB of features (a single chunk when the batch is small).
  int64_t rows = std::max<int64_t>(1024, ((int64_t)128 << 20) / ((int64_t)F * 4) / 1024 * 1024);
  rows = std::min(rows, n);
  // Chunk boundaries: full chunks, then a tapered tail (rows/2, /4, /8, /8) so the work
  // left after the last copy -- that chunk's kernels and score copy -- is small.
  std::vector<int64_t> bounds{0};
  if (n <= rows) {
    bounds.push_back(n);  // one chunk: nothing to overlap
  } else {
    const int64_t r = rows;
    const int64_t tail[4] = {std::max<int64_t>(1024, r / 2), std::max<int64_t>(1024, r / 4),
                             std::max<int64_t>(1024, r / 8), std::max<int64_t>(1024, r / 8)};
    const int64_t tail_sum = tail[0] + tail[1] + tail[2] + tail[3];
    int64_t pos = 0;
    while (n - pos > tail_sum + r) { pos += r; bounds.push_back(pos); }
    if (n - pos > tail_sum) { pos = n - tail_sum; bounds.push_back(pos); }
    for (int i = 0; i < 4 && pos < n; ++i) {
      pos = std::min(n, pos + tail[i]);
      if (pos > bounds.back()) bounds.push_back(pos);
    }
    if (bounds.back() != n) bounds.push_back(n);
  }
  const int64_t n_chunks = (int64_t)bounds.size() - 1;
  if (n_chunks == 1) {
    // one chunk: nothing to overlap -- copy in, predict and copy out on `stream`
    float* xd = nullptr;
    double* od = nullptr;
    rc = OBT_OK;
    auto ok = [&](cudaError_t e, const char* what) {
      if (e != cudaSuccess && rc == OBT_OK) rc = fail(OBT_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
      return rc == OBT_OK;
    };
    if (ok(pool_alloc(reinterpret_cast<void**>(&xd), (size_t)n * F * 4, m->device, stream), "feature buffer") &&
        ok(pool_alloc(reinterpret_cast<void**>(&od), (size_t)n * C * 8, m->device, stream), "score buffer") &&
        ok(layout == OBT_LAYOUT_FEATURE_MAJOR && ld != n
               ? cudaMemcpy2DAsync(xd, (size_t)n * 4, x_host, (size_t)ld * 4, (size_t)n * 4, F, cudaMemcpyHostToDevice, stream)
               : cudaMemcpyAsync(xd, x_host, (size_t)n * F * 4, cudaMemcpyHostToDevice, stream),
           "H2D")) {
      rc = predict_impl(m, xd, n, layout, od, nullptr, 0, 0, nullptr, 0, stream);
      if (rc == OBT_OK) ok(cudaMemcpyAsync(out_host, od, (size_t)n * C * 8, cudaMemcpyDeviceToHost, stream), "D2H");
    }
    const int launches = g_launches;
    if (xd) cudaFreeAsync(xd, stream);
    if (od) cudaFreeAsync(od, stream);
    const cudaError_t e = cudaStreamSynchronize(stream);
    if (rc == OBT_OK && e != cudaSuccess) rc = fail(OBT_E_CUDA, "stream synchronize failed: %s", cudaGetErrorString(e));
    g_launches = launches;
    return rc;
  }
  const int nbuf = n_chunks > 1 ? 2 : 1;
  // pageable object-major features go through the pinned staging buffers; scores for a
  // pageable output gather on the device and cross once at the end (a D2H into pageable
  // memory blocks the host until the stream drains, which would serialise the pipeline)
  cudaPointerAttributes pattr{};
  const bool pageable = cudaPointerGetAttributes(&pattr, x_host) != cudaSuccess || pattr.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();  // an unregistered pointer is not an error here
  const bool out_pageable = cudaPointerGetAttributes(&pattr, out_host) != cudaSuccess ||
                            pattr.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  HostStaging* stg = nullptr;
  std::unique_lock<std::mutex> stg_lock;
  if (pageable && layout == OBT_LAYOUT_OBJECT_MAJOR) {
    stg = host_staging(m->device);
    stg_lock = std::unique_lock<std::mutex>(stg->mu);
    const size_t need = (size_t)rows * F * 4;
    if (stg->bytes < need) {
      for (int b = 0; b < 2; ++b) {
        if (stg->buf[b]) cudaFreeHost(stg->buf[b]);
        stg->buf[b] = nullptr;
      }
      stg->bytes = 0;
      bool ok = true;
      for (int b = 0; b < 2 && ok; ++b) ok = cudaHostAlloc(&stg->buf[b], need, cudaHostAllocPortable) == cudaSuccess;
      for (int b = 0; b < 2 && ok; ++b)
        if (!stg->h2d_done[b]) ok = cudaEventCreateWithFlags(&stg->h2d_done[b], cudaEventDisableTiming) == cudaSuccess;
      if (ok) {
        stg->bytes = need;
      } else {
        cudaGetLastError();
        stg_lock.unlock();
        stg = nullptr;  // no pinned memory to spare: the driver's own staging
      }
    }
  }
  float* x_dev[2] = {nullptr, nullptr};
  double* out_dev[2] = {nullptr, nullptr};
  double* out_all = nullptr;  // pageable output: every chunk's scores, one D2H at the end
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  rc = OBT_OK;
  auto cuda_ok = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == OBT_OK) rc = fail(OBT_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
    return rc == OBT_OK;
  };
  cuda_ok(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "copy stream");
  if (out_pageable)
    cuda_ok(pool_alloc(reinterpret_cast<void**>(&out_all), (size_t)n * C * 8, m->device, stream), "score buffer");
  for (int b = 0; b < nbuf && rc == OBT_OK; ++b) {
    cuda_ok(pool_alloc(reinterpret_cast<void**>(&x_dev[b]), (size_t)rows * F * 4, m->device, stream), "feature buffer");
    if (!out_pageable)
      cuda_ok(pool_alloc(reinterpret_cast<void**>(&out_dev[b]), (size_t)rows * C * 8, m->device, stream), "score buffer");
    cuda_ok(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming), "event");
  }
  // the copy stream must not start before the buffers exist on `stream`
  cudaEvent_t ready = nullptr;
  if (cuda_ok(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event")) {
    cuda_ok(cudaEventRecord(ready, stream), "event record");
    cuda_ok(cudaStreamWaitEvent(copy, ready, 0), "stream wait");
  }
  int launches = 0;
  for (int64_t i = 0; i < n_chunks && rc == OBT_OK; ++i) {
    const int b = (int)(i % nbuf);
    const int64_t o0 = bounds[i], ni = bounds[i + 1] - bounds[i];
    if (i >= nbuf) cuda_ok(cudaStreamWaitEvent(copy, done[b], 0), "stream wait");  // buffer b free again
    if (stg) {
      // staging buffer b is free once its previous DMA is done; fill it on the host
      // while the DMA of chunk i - 1 and the kernels of chunk i - 2 run
      if (i >= 2) cuda_ok(cudaEventSynchronize(stg->h2d_done[b]), "staging wait");
      if (rc != OBT_OK) break;
      parallel_copy(stg->buf[b], x_host + o0 * F, (size_t)ni * F * 4);
      cuda_ok(cudaMemcpyAsync(x_dev[b], stg->buf[b], (size_t)ni * F * 4, cudaMemcpyHostToDevice, copy), "H2D");
      cuda_ok(cudaEventRecord(stg->h2d_done[b], copy), "event record");
    } else if (layout == OBT_LAYOUT_OBJECT_MAJOR) {
      cuda_ok(cudaMemcpyAsync(x_dev[b], x_host + o0 * F, (size_t)ni * F * 4, cudaMemcpyHostToDevice, copy), "H2D");
    } else {  // feature-major: ni columns of every feature row
      cuda_ok(cudaMemcpy2DAsync(x_dev[b], (size_t)ni * 4, x_host + o0, (size_t)ld * 4, (size_t)ni * 4, F,
                                cudaMemcpyHostToDevice, copy), "H2D");
    }
    cuda_ok(cudaEventRecord(copied[b], copy), "event record");
    cuda_ok(cudaStreamWaitEvent(stream, copied[b], 0), "stream wait");
    if (rc != OBT_OK) break;
    double* od = out_pageable ? out_all + o0 * C : out_dev[b];
    rc = predict_impl(m, x_dev[b], ni, layout, od, nullptr, 0, 0, nullptr, 0, stream);
    launches += g_launches;
    if (!out_pageable)
      cuda_ok(cudaMemcpyAsync(out_host + o0 * C, od, (size_t)ni * C * 8, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_ok(cudaEventRecord(done[b], stream), "event record");
  }
  if (out_pageable && rc == OBT_OK)
    cuda_ok(cudaMemcpyAsync(out_host, out_all, (size_t)n * C * 8, cudaMemcpyDeviceToHost, stream), "D2H");
  g_launches = launches;
  // the stream-ordered frees below must also follow every copy issued on `copy` (an
  // error may have left a copy that `stream` never waited for)
  if (ready && copy && cudaEventRecord(ready, copy) == cudaSuccess) cudaStreamWaitEvent(stream, ready, 0);
  for (int b = 0; b < nbuf; ++b) {
    if (x_dev[b]) cudaFreeAsync(x_dev[b], stream);
    if (out_dev[b]) cudaFreeAsync(out_dev[b], stream);
  }
  if (out_all) cudaFreeAsync(out_all, stream);
  const cudaError_t e = cudaStreamSynchronize(stream);
  if (rc == OBT_OK && e != cudaSuccess) rc = fail(OBT_E_CUDA, "stream synchronize failed: %s", cudaGetErrorString(e));
  cudaStreamSynchronize(copy);
  for (int b = 0; b < nbuf; ++b) {
    if (copied[b]) cudaEventDestroy(copied[b]);
    if (done[b]) cudaEventDestroy(done[b]);
  }
  if (ready) cudaEventDestroy(ready);
  if (copy) cudaStreamDestroy(copy);
  return rc;
}

int obt_predict_host(const obt_model* mc, const float* x_host, int64_t n, int32_t layout, double* out_host,
                     void* stream_v) {
  g_launches = 0;
  obt_model* m = const_cast<obt_model*>(mc);
  if (!m) return fail(OBT_E_INVALID, "null model");
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  if (n == 0) return OBT_OK;
  if (!x_host || !out_host) return fail(OBT_E_INVALID, "null feature or output pointer");
  return predict_host_impl(m, x_host, n, n, layout, out_host, static_cast<cudaStream_t>(stream_v));
}

}  // extern "C"

namespace {

constexpr int kMaxShards = 16;

// Tree-sharded combine: the shards' raw partial sums added in shard order (binary64),
// then the affine finalize with two roundings (evaluate.py:298-299).
struct PartialSet {
  const double* part[kMaxShards];
};
__global__ void fold_partials_kernel(PartialSet ps, int n_parts, int64_t count, double scale, double bias,
                                     double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    double acc = ps.part[0][i];
    for (int s = 1; s < n_parts; ++s) acc = __dadd_rn(acc, ps.part[s][i]);
    out[i] = __dadd_rn(__dmul_rn(acc, scale), bias);
  }
}

// Object shards: shard s evaluates a contiguous object range (256-object quanta, as the
// Python ObjectShardedEvaluator) on its own device from its own host thread; every shard
// runs the chunked host pipeline of obt_predict_host.  No data crosses between devices.
int predict_sharded_objects(obt_model* const* shards, int n_shards, const float* x_host, int64_t n, int32_t layout,
                            double* out_host) {
  const int64_t units = (n + 255) / 256, base = units / n_shards, extra = units % n_shards;
  std::vector<int64_t> begin(n_shards + 1, 0);
  for (int s = 0; s < n_shards; ++s) begin[s + 1] = std::min(n, begin[s] + (base + (s < extra ? 1 : 0)) * 256);
  std::vector<int> rcs(n_shards, OBT_OK), launches(n_shards, 0);
  std::vector<std::string> errors(n_shards);
  auto run = [&](int s) {
    obt_model* m = shards[s];
    const int64_t b = begin[s], cnt = begin[s + 1] - begin[s];
    if (cnt == 0) return;
    DeviceGuard guard(m->device);
    cudaStream_t stream = nullptr;
    if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess) {
      rcs[s] = OBT_E_CUDA;
      errors[s] = "shard stream creation failed";
      cudaGetLastError();
      return;
    }
    const float* xs = layout == OBT_LAYOUT_OBJECT_MAJOR ? x_host + b * m->n_features : x_host + b;
    rcs[s] = predict_host_impl(m, xs, cnt, n, layout, out_host + b * m->n_outputs, stream);
    if (rcs[s] != OBT_OK) errors[s] = g_error;
    launches[s] = g_launches;
    cudaStreamDestroy(stream);
  };
  // this thread runs shard 0 and any shard no thread could be made for
  std::vector<std::thread> th;
  try {
    for (int s = 1; s < n_shards; ++s) th.emplace_back(run, s);
  } catch (...) {
  }
  run(0);
  for (int s = (int)th.size() + 1; s < n_shards; ++s) run(s);
  for (auto& t : th) t.join();
  int total = 0;
  for (int s = 0; s < n_shards; ++s) {
    total += launches[s];
    if (rcs[s] != OBT_OK) return fail(rcs[s], "shard %d: %s", s, errors[s].c_str());
  }
  g_launches = total;
  return OBT_OK;
}

// Tree shards: shard s holds trees [t_s, t_{s+1}) as a raw partial-sum model (scale 1,
// bias 0) on its own device.  Per chunk of objects every shard receives the chunk's
// features and evaluates its trees; the partial sums travel to shard 0's device with peer
// copies (NVLink between the GPUs of one box), are added there in shard order and
// finalized with the caller's scale and bias, and the scores go back to the host.  All
// asynchronous: the shards' streams wait on each other through events only.
int predict_sharded_trees(obt_model* const* shards, int n_shards, const float* x_host, int64_t n, int32_t layout,
                          double scale, double bias, double* out_host) {
  const int F = shards[0]->n_features, C = shards[0]->n_outputs;
  int64_t rows = std::max<int64_t>(1024, ((int64_t)128 << 20) / ((int64_t)F * 4) / 1024 * 1024);
  rows = std::min(rows, n);
  const size_t x_bytes = (size_t)rows * F * 4, p_bytes = (size_t)rows * C * 8;
  struct Shard {
    cudaStream_t stream = nullptr;
    float* x = nullptr;
    double* part = nullptr;      // on the shard's device
    double* gathered = nullptr;  // on shard 0's device (shards >= 1)
    cudaEvent_t part_ready = nullptr, part_taken = nullptr;
  };
  std::vector<Shard> sh(n_shards);
  double* out_dev = nullptr;
  int rc = OBT_OK, launches = 0;
  auto ok = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == OBT_OK) rc = fail(OBT_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
    return rc == OBT_OK;
  };
  const int root = shards[0]->device;
  for (int s = 0; s < n_shards && rc == OBT_OK; ++s) {
    DeviceGuard guard(shards[s]->device);
    ok(cudaStreamCreateWithFlags(&sh[s].stream, cudaStreamNonBlocking), "shard stream");
    if (rc != OBT_OK) break;
    ok(pool_alloc(reinterpret_cast<void**>(&sh[s].x), x_bytes, shards[s]->device, sh[s].stream), "feature buffer");
    ok(pool_alloc(reinterpret_cast<void**>(&sh[s].part), p_bytes, shards[s]->device, sh[s].stream), "partial-sum buffer");
    ok(cudaEventCreateWithFlags(&sh[s].part_ready, cudaEventDisableTiming), "event");
  }
  if (rc == OBT_OK) {
    DeviceGuard guard(root);
    ok(pool_alloc(reinterpret_cast<void**>(&out_dev), p_bytes, root, sh[0].stream), "score buffer");
    for (int s = 1; s < n_shards && rc == OBT_OK; ++s) {
      ok(pool_alloc(reinterpret_cast<void**>(&sh[s].gathered), p_bytes, root, sh[0].stream), "gather buffer");
      ok(cudaEventCreateWithFlags(&sh[s].part_taken, cudaEventDisableTiming), "event");
    }
  }
  for (int64_t o0 = 0; o0 < n && rc == OBT_OK; o0 += rows) {
    const int64_t ni = std::min(rows, n - o0);
    for (int s = 0; s < n_shards && rc == OBT_OK; ++s) {
      DeviceGuard guard(shards[s]->device);
      // the partial-sum buffer is free once shard 0 has taken the previous chunk's sums
      // (shard 0's own buffer is read by the fold on the same stream)
      if (s > 0 && o0 > 0) ok(cudaStreamWaitEvent(sh[s].stream, sh[s].part_taken, 0), "stream wait");
      if (layout == OBT_LAYOUT_OBJECT_MAJOR) {
        ok(cudaMemcpyAsync(sh[s].x, x_host + o0 * F, (size_t)ni * F * 4, cudaMemcpyHostToDevice, sh[s].stream), "H2D");
      } else {
        ok(cudaMemcpy2DAsync(sh[s].x, (size_t)ni * 4, x_host + o0, (size_t)n * 4, (size_t)ni * 4, F,
                             cudaMemcpyHostToDevice, sh[s].stream), "H2D");
      }
      if (rc != OBT_OK) break;
      rc = predict_impl(shards[s], sh[s].x, ni, layout, sh[s].part, nullptr, 0, 0, nullptr, 0, sh[s].stream);
      launches += g_launches;
      if (rc == OBT_OK) ok(cudaEventRecord(sh[s].part_ready, sh[s].stream), "event record");
    }
    if (rc != OBT_OK) break;
    DeviceGuard guard(root);
    PartialSet ps{};
    ps.part[0] = sh[0].part;
    for (int s = 1; s < n_shards && rc == OBT_OK; ++s) {
      ok(cudaStreamWaitEvent(sh[0].stream, sh[s].part_ready, 0), "stream wait");
      ok(cudaMemcpyPeerAsync(sh[s].gathered, root, sh[s].part, shards[s]->device, (size_t)ni * C * 8, sh[0].stream),
         "peer copy");
      ok(cudaEventRecord(sh[s].part_taken, sh[0].stream), "event record");
      ps.part[s] = sh[s].gathered;
    }
    if (rc != OBT_OK) break;
    const int64_t count = ni * C;
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, (int64_t)shards[0]->sm_count * 8);
    fold_partials_kernel<<<blocks, 256, 0, sh[0].stream>>>(ps, n_shards, count, scale, bias, out_dev);
    ok(cudaGetLastError(), "fold launch");
    ++launches;
    ok(cudaMemcpyAsync(out_host + o0 * C, out_dev, (size_t)count * 8, cudaMemcpyDeviceToHost, sh[0].stream), "D2H");
  }
  // drain every stream before the buffers go (shard 0 last: it consumes the others' sums)
  for (int s = n_shards - 1; s >= 0; --s) {
    if (!sh[s].stream) continue;
    DeviceGuard guard(shards[s]->device);
    const cudaError_t e = cudaStreamSynchronize(sh[s].stream);
    if (e != cudaSuccess && rc == OBT_OK) rc = fail(OBT_E_CUDA, "stream synchronize failed: %s", cudaGetErrorString(e));
  }
  {
    DeviceGuard guard(root);
    if (out_dev) cudaFreeAsync(out_dev, sh[0].stream);
    for (int s = 1; s < n_shards; ++s) {
      if (sh[s].gathered) cudaFreeAsync(sh[s].gathered, sh[0].stream);
      if (sh[s].part_taken) cudaEventDestroy(sh[s].part_taken);
    }
  }
  for (int s = 0; s < n_shards; ++s) {
    if (!sh[s].stream) continue;
    DeviceGuard guard(shards[s]->device);
    if (sh[s].x) cudaFreeAsync(sh[s].x, sh[s].stream);
    if (sh[s].part) cudaFreeAsync(sh[s].part, sh[s].stream);
    if (sh[s].part_ready) cudaEventDestroy(sh[s].part_ready);
    cudaStreamSynchronize(sh[s].stream);
    cudaStreamDestroy(sh[s].stream);
  }
  g_launches = launches;
  return rc;
}

}  // namespace

extern "C" {

int obt_predict_sharded(const obt_model* const* shards_c, int32_t n_shards, int32_t mode, const float* x_host,
                        int64_t n, int32_t layout, double scale, double bias, double* out_host) {
  g_launches = 0;
  if (!shards_c || n_shards < 1 || n_shards > kMaxShards)
    return fail(OBT_E_INVALID, "shard count must be 1..%d", kMaxShards);
  if (mode != OBT_SHARD_OBJECTS && mode != OBT_SHARD_TREES) return fail(OBT_E_INVALID, "unknown shard mode %d", mode);
  obt_model* const* shards = const_cast<obt_model* const*>(reinterpret_cast<const obt_model* const*>(shards_c));
  for (int s = 0; s < n_shards; ++s) {
    if (!shards[s]) return fail(OBT_E_INVALID, "null model (shard %d)", s);
    if (shards[s]->n_features != shards[0]->n_features || shards[s]->n_outputs != shards[0]->n_outputs ||
        shards[s]->precision != shards[0]->precision)
      return fail(OBT_E_INVALID, "shard %d differs from shard 0 in features, outputs or leaf precision", s);
    if (mode == OBT_SHARD_TREES && (shards[s]->scale != 1.0 || shards[s]->bias != 0.0))
      return fail(OBT_E_INVALID, "tree shard %d must be a raw partial-sum model (scale 1, bias 0)", s);
  }
  int rc = check_layout(layout);
  if (rc != OBT_OK) return rc;
  if (n < 0) return fail(OBT_E_INVALID, "negative object count");
  if (n == 0) return OBT_OK;
  if (!x_host || !out_host) return fail(OBT_E_INVALID, "null feature or output pointer");
  return mode == OBT_SHARD_OBJECTS ? predict_sharded_objects(shards, n_shards, x_host, n, layout, out_host)
                                   : predict_sharded_trees(shards, n_shards, x_host, n, layout, scale, bias, out_host);
}

}  // extern "C"
