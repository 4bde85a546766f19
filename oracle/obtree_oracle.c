/*
 * obtree_oracle.c -- CPU restatement of the reference obtree apply path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the results oracle for the GPU
 * kernels and the CPU baseline that bench.py reports beside them.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it; the product path (paper_2211_00391_b200/) never
 * does and fails loudly when its own CUDA library is missing.
 *
 * Every function restates one piece of the reference package
 * (/root/reference/pkg/src/obtree, pure Python + numpy) in plain C with IEEE
 * semantics: compiled with -O3 -ffp-contract=off and no fast-math, so float
 * compares, the binary64 left fold and the two-rounding finalize match numpy
 * bit for bit (vectorisation runs across independent objects, never across
 * one object's tree-order sum).  Parity of this restatement is pinned by tests/golden (fixtures
 * produced by the reference itself, see tests/golden/make_golden.py).
 *
 * Model layout shared by every entry point (flat, C order):
 *   borders       float  [F][border_stride]   ascending, first border_counts[f] used
 *   border_counts int32  [F]
 *   depths        int32  [T]                  per-tree depth (1..16)
 *   split_feature int32  [T][max_depth]       first depths[t] used
 *   split_ordinal int32  [T][max_depth]
 *   leaves        double [T][n_outputs][1 << max_depth]  first 1 << depths[t] used
 * Feature matrices are float32, object-major (o*F + f) or feature-major (f*N + o).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OBJECT_MAJOR 0
#define ORC_FEATURE_MAJOR 1

static inline float feature_at(const float* x, int64_t n, int32_t n_features, int layout,
                               int64_t o, int32_t f) {
  return layout == ORC_OBJECT_MAJOR ? x[o * (int64_t)n_features + f] : x[(int64_t)f * n + o];
}

int orc_version(void) { return 1; }

/* Thread count for the parallel loops (launchers such as torchrun export
   OMP_NUM_THREADS=1; the CPU baseline sets the host's core count explicitly). */
void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Stage 1 -- quantize.  quantize.py:121-133 (scalar, early exit) and
 * quantize.py:164-172 (block form: exhaustive count of borders with x > b,
 * NaN compares false everywhere and yields 0).
 */
int32_t orc_quantize_value(float value, const float* borders, int32_t n_borders) {
  int32_t count = 0;
  for (int32_t k = 0; k < n_borders; ++k) {
    if (value > borders[k]) ++count;
    else break;
  }
  return count;
}

/* Buckets of the whole matrix, written feature-major: out[f * n + o]
 * (the QuantizedBlock row layout of quantize.py:93-108 with block = n). */
void orc_quantize_matrix(const float* x, int64_t n, int32_t n_features, int layout,
                         const float* borders, const int32_t* border_counts,
                         int32_t border_stride, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < n; ++o) {
    for (int32_t f = 0; f < n_features; ++f) {
      const float v = feature_at(x, n, n_features, layout, o, f);
      const float* fb = borders + (int64_t)f * border_stride;
      uint32_t count = 0;
      for (int32_t k = 0; k < border_counts[f]; ++k) count += (v > fb[k]) ? 1u : 0u;
      out[(int64_t)f * n + o] = (uint8_t)count;
    }
  }
}

/* ---------------------------------------------------------------------------
 * Stage 2 -- leaf indices from buckets.  indexer.py:39-57 (idx |= bit_d << d,
 * root condition in bit 0) and the padded panel form evaluate.py:199-207
 * (ordinal 255 = sentinel, never true because buckets are <= 254).
 * q is feature-major [F][n]; split arrays are [T][max_depth]; out is [T][n].
 */
void orc_leaf_indices(const uint8_t* q, int64_t n, int32_t n_trees, int32_t max_depth,
                      const int32_t* split_feature, const int32_t* split_ordinal,
                      uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n_trees; ++t) {
    for (int64_t o = 0; o < n; ++o) {
      uint32_t idx = 0;
      for (int32_t d = 0; d < max_depth; ++d) {
        const int32_t f = split_feature[t * max_depth + d];
        const int32_t ord = split_ordinal[t * max_depth + d];
        idx |= ((uint32_t)q[(int64_t)f * n + o] > (uint32_t)ord ? 1u : 0u) << d;
      }
      out[t * n + o] = (uint16_t)idx;
    }
  }
}

/* ---------------------------------------------------------------------------
 * binary16 helpers -- model.py:231-277 (build_leaf_bank): leaves.astype(float16)
 * is a direct binary64 -> binary16 round-to-nearest-even conversion; every
 * +/-inf result (finite overflow or an infinite leaf) is saturated to +/-65504
 * (model.py:262-268).
 */
uint16_t orc_half_from_double(double x) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  const uint16_t sign = (uint16_t)((bits >> 48) & 0x8000u);
  const int32_t exp = (int32_t)((bits >> 52) & 0x7FF);
  const uint64_t man = bits & 0xFFFFFFFFFFFFFull;
  if (exp == 0x7FF) return (uint16_t)(sign | (man ? 0x7E00u : 0x7C00u));
  if (exp == 0) return sign; /* binary64 subnormals are far below 2^-25 */
  const int32_t e = exp - 1023;
  const uint64_t sig = man | (1ull << 52); /* 53-bit significand, value = sig * 2^(e-52) */
  if (e > 15) return (uint16_t)(sign | 0x7C00u);
  /* quantum of the result: 2^(max(e,-14) - 10); shift = (max(e,-14) - 10) - (e - 52) */
  const int32_t qexp = (e < -14 ? -14 : e) - 10;
  const int32_t shift = qexp - (e - 52);
  uint64_t q;
  if (shift >= 64) {
    q = 0; /* value < 2^-64 * quantum: rounds to zero */
  } else {
    q = sig >> shift;
    const uint64_t rem = sig & ((1ull << shift) - 1);
    const uint64_t half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (q & 1))) ++q;
  }
  /* q counts quanta; normal results have q in [1024, 2048] */
  if (e < -14) {
    /* subnormal range: q <= 1024; q == 1024 is the smallest normal (exp field 1) */
    return (uint16_t)(sign | q);
  }
  int32_t he = e;
  if (q >= 2048) { q >>= 1; ++he; }
  if (he > 15) return (uint16_t)(sign | 0x7C00u);
  return (uint16_t)(sign | ((uint32_t)(he + 15) << 10) | (uint32_t)(q - 1024));
}

uint16_t orc_half_saturated(double x) {
  uint16_t h = orc_half_from_double(x);
  if ((h & 0x7FFFu) == 0x7C00u) h = (uint16_t)((h & 0x8000u) | 0x7BFFu);
  return h;
}

float orc_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1F;
  const uint32_t man = h & 0x3FF;
  uint32_t bits;
  if (exp == 0x1F) {
    bits = sign | 0x7F800000u | (man << 13);
  } else if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else { /* subnormal half = man * 2^-24, exactly representable */
      float v = (float)man * 0x1p-24f;
      memcpy(&bits, &v, 4);
      bits |= sign;
    }
  } else {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float out;
  memcpy(&out, &bits, 4);
  return out;
}

/* Bank conversion of a whole leaf array; returns the saturation count. */
int64_t orc_half_bank(const double* leaves, int64_t count, uint16_t* out) {
  int64_t saturated = 0;
  for (int64_t i = 0; i < count; ++i) {
    const uint16_t raw = orc_half_from_double(leaves[i]);
    if ((raw & 0x7FFFu) == 0x7C00u) ++saturated; /* inf leaves too (model.py:264) */
    out[i] = orc_half_saturated(leaves[i]);
  }
  return saturated;
}

/* ---------------------------------------------------------------------------
 * The ground truth -- oracle.py:21-54 (evaluate_scalar), generalised to
 * n_outputs tables per tree and depth up to 16 for the multiclass config the
 * reference cannot express (SURVEY.md 8c "cfg5 restatement").  Each split is
 * evaluated on the RAW float32 value against the border it names (never on a
 * bucket), the index is assembled root-first into bit 0 (oracle.py:45-48), and
 * leaves are added in tree order:
 *   precision 0 (BINARY64): acc (binary64) += leaf            (oracle.py:49-50)
 *   precision 1 (BINARY16): acc (binary32) += f32(half(leaf)) (oracle.py:51-52)
 * then out = f64(acc) * scale + bias with two roundings (oracle.py:53-54).
 * out is [n][n_outputs].  Objects are independent, so threading over objects
 * does not change a single bit.
 */
#define ORC_BLOCK 256

int orc_evaluate_scalar(const float* x, int64_t n, int32_t n_features, int layout,
                        const float* borders, int32_t border_stride,
                        int32_t n_trees, int32_t max_depth, const int32_t* depths,
                        const int32_t* split_feature, const int32_t* split_ordinal,
                        const double* leaves, int32_t n_outputs, double scale, double bias,
                        int precision, double* out) {
  if (max_depth > 16 || n_outputs < 1) return -1;
  const int64_t table = (int64_t)1 << max_depth;
  uint16_t* bank16 = NULL;
  if (precision == 1) {
    const int64_t total = (int64_t)n_trees * n_outputs * table;
    bank16 = (uint16_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint16_t));
    if (!bank16) return -2;
    orc_half_bank(leaves, total, bank16);
  }
  const int64_t n_blocks = (n + ORC_BLOCK - 1) / ORC_BLOCK;
#pragma omp parallel
  {
    double* acc64 = (double*)malloc(sizeof(double) * ORC_BLOCK * (size_t)n_outputs);
    float* acc32 = (float*)malloc(sizeof(float) * ORC_BLOCK * (size_t)n_outputs);
    float* xb = (float*)malloc(sizeof(float) * ORC_BLOCK * (size_t)n_features);
    uint32_t idx[ORC_BLOCK];
#pragma omp for schedule(dynamic, 4)
    for (int64_t b = 0; b < n_blocks; ++b) {
      const int64_t o0 = b * ORC_BLOCK;
      const int64_t live = (n - o0) < ORC_BLOCK ? (n - o0) : ORC_BLOCK;
      /* the block's raw values, feature-major, so each split reads one contiguous row */
      for (int64_t i = 0; i < live; ++i)
        for (int32_t f = 0; f < n_features; ++f)
          xb[(int64_t)f * ORC_BLOCK + i] = feature_at(x, n, n_features, layout, o0 + i, f);
      for (int64_t i = 0; i < live * n_outputs; ++i) { acc64[i] = 0.0; acc32[i] = 0.0f; }
      for (int32_t t = 0; t < n_trees; ++t) {
        for (int64_t i = 0; i < live; ++i) idx[i] = 0;
        for (int32_t d = 0; d < depths[t]; ++d) {
          const int32_t f = split_feature[(int64_t)t * max_depth + d];
          const float border = borders[(int64_t)f * border_stride + split_ordinal[(int64_t)t * max_depth + d]];
          const float* row = xb + (int64_t)f * ORC_BLOCK;
          for (int64_t i = 0; i < live; ++i) idx[i] |= (row[i] > border ? 1u : 0u) << d;
        }
        for (int32_t c = 0; c < n_outputs; ++c) {
          const int64_t base = ((int64_t)t * n_outputs + c) * table;
          if (precision == 0) {
            const double* lv = leaves + base;
            for (int64_t i = 0; i < live; ++i) acc64[i * n_outputs + c] += lv[idx[i]];
          } else {
            const uint16_t* lv = bank16 + base;
            for (int64_t i = 0; i < live; ++i) acc32[i * n_outputs + c] += orc_half_to_float(lv[idx[i]]);
          }
        }
      }
      for (int64_t i = 0; i < live * n_outputs; ++i) {
        const double s = precision == 0 ? acc64[i] : (double)acc32[i];
        const double m = s * scale;
        out[o0 * n_outputs + i] = m + bias;
      }
    }
    free(acc64);
    free(acc32);
    free(xb);
  }
  free(bank16);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Seeded generators -- synthetic.py:28-167 (SplitMix64 state expansion,
 * xoshiro256**, multiply-shift bounded integers).  Restated so the GPU box can
 * regenerate the reference's own acceptance corpus (tests/test_acceptance.py
 * corpus_spec) without the reference package; pinned by hashes the reference
 * produced (tests/golden).
 */
typedef struct { uint64_t s[4]; } orc_xoshiro;

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_xoshiro_seed(orc_xoshiro* r, uint64_t seed) {
  uint64_t state = seed;
  for (int i = 0; i < 4; ++i) { /* synthetic.py:28-35 */
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    r->s[i] = z ^ (z >> 31);
  }
  if (!(r->s[0] | r->s[1] | r->s[2] | r->s[3])) r->s[0] = 1; /* synthetic.py:48-49 */
}

uint64_t orc_xoshiro_next(orc_xoshiro* r) { /* synthetic.py:51-62 */
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

double orc_xoshiro_unit(orc_xoshiro* r) { return (double)(orc_xoshiro_next(r) >> 11) * 0x1p-53; }

double orc_xoshiro_uniform(orc_xoshiro* r, double lo, double hi) {
  return lo + orc_xoshiro_unit(r) * (hi - lo);
}

uint64_t orc_xoshiro_below(orc_xoshiro* r, uint64_t n) {
  return (uint64_t)(((unsigned __int128)orc_xoshiro_next(r) * n) >> 64);
}

static int cmp_float(const void* a, const void* b) {
  const float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

/* generate_synthetic_model, synthetic.py:87-133.  Outputs use the flat model
 * layout above with border_stride = borders_per_feature and max_depth = depth.
 * Returns scale and bias through the pointers. */
int orc_synthetic_model(int32_t n_features, int32_t borders_per_feature, int32_t n_trees,
                        int32_t depth, uint64_t seed, float* borders, int32_t* split_feature,
                        int32_t* split_ordinal, double* leaves, double* scale, double* bias) {
  if (n_features < 1 || borders_per_feature < 1 || borders_per_feature > 254 || n_trees < 0 ||
      depth < 1 || depth > 8)
    return -1;
  orc_xoshiro r;
  orc_xoshiro_seed(&r, seed);
  for (int32_t f = 0; f < n_features; ++f) {
    float* fb = borders + (int64_t)f * borders_per_feature;
    int32_t have = 0;
    while (have < borders_per_feature) { /* distinct float32(unit()) draws */
      const float v = (float)orc_xoshiro_unit(&r);
      int dup = 0;
      for (int32_t k = 0; k < have; ++k) if (fb[k] == v) { dup = 1; break; }
      if (!dup) fb[have++] = v;
    }
    qsort(fb, (size_t)borders_per_feature, sizeof(float), cmp_float);
  }
  const int64_t leaves_per_tree = (int64_t)1 << depth;
  for (int32_t t = 0; t < n_trees; ++t) {
    for (int32_t d = 0; d < depth; ++d) {
      const int32_t f = (int32_t)orc_xoshiro_below(&r, (uint64_t)n_features);
      split_feature[(int64_t)t * depth + d] = f;
      split_ordinal[(int64_t)t * depth + d] = (int32_t)orc_xoshiro_below(&r, (uint64_t)borders_per_feature);
    }
    for (int64_t j = 0; j < leaves_per_tree; ++j)
      leaves[(int64_t)t * leaves_per_tree + j] = orc_xoshiro_uniform(&r, -1.0, 1.0);
  }
  *scale = orc_xoshiro_uniform(&r, 0.5, 1.5);
  *bias = orc_xoshiro_uniform(&r, -0.5, 0.5);
  return 0;
}

/* generate_feature_matrix, synthetic.py:136-167; out is object-major [n][F]. */
void orc_feature_matrix(int64_t n_objects, int32_t n_features, uint64_t seed, double lo, double hi,
                        double nan_fraction, double inf_fraction, float* out) {
  orc_xoshiro r;
  orc_xoshiro_seed(&r, seed);
  const double special = nan_fraction + inf_fraction;
  const int64_t total = n_objects * (int64_t)n_features;
  for (int64_t i = 0; i < total; ++i) {
    if (special > 0.0) {
      const double roll = orc_xoshiro_unit(&r);
      if (roll < nan_fraction) { out[i] = NAN; continue; }
      if (roll < special) { out[i] = orc_xoshiro_unit(&r) < 0.5 ? INFINITY : -INFINITY; continue; }
    }
    out[i] = (float)orc_xoshiro_uniform(&r, lo, hi);
  }
}
