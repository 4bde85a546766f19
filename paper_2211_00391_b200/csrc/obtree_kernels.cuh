// obtree_kernels.cuh -- sm_100a kernels of the oblivious-ensemble apply path.
//
//   K1 quantize  (reference stage 1, quantize.py:136-172)
//      float32 features -> uint8 bucket = #{k : x > border_k}; NaN -> 0.
//      Branchless Eytzinger search over +inf-padded borders; output either the
//      tile-blocked matrix Q[tile][F][TILE] the apply kernel streams, or the plain
//      feature-major [F][n] matrix (obt_quantize_dev, parity).
//   K2 apply     (reference stages 2+3 + finalize, indexer.py:39-57,
//                 accumulate.py:88-97, evaluate.py:189-248, 298-299)
//      One CTA owns TILE objects.  Its bucket tile (F x TILE bytes) arrives by one
//      bulk TMA copy; split descriptors + leaf tables stream through an S-stage
//      ring of bulk copies (mbarrier complete_tx).  Each thread owns 4 objects as
//      one 32-bit word per feature row (SWAR): per depth one LDS.32, one add that
//      lands the condition in bit 7 of every byte, one shift+mask-or into the four
//      packed leaf indices.  Leaves are gathered from shared memory and added in
//      tree order in binary64 (binary32 for the binary16 family), exactly the
//      reference fold, then out = acc * scale + bias with two roundings.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

namespace obt {

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D bulk async copy (TMA engine, no tensor map).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Copy `bytes` in pieces of at most 64 KiB (each piece completes on the same barrier).
__device__ __forceinline__ void bulk_g2s_split(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  constexpr uint32_t kPiece = 65536;
  uint32_t done = 0;
  while (done < bytes) {
    const uint32_t len = (bytes - done) < kPiece ? (bytes - done) : kPiece;
    bulk_g2s(static_cast<char*>(dst) + done, static_cast<const char*>(src) + done, len, bar);
    done += len;
  }
}

// ---------------------------------------------------------------------------
// K1: quantize.
struct QuantizeParams {
  const float* x;        // features, layout per template
  int64_t n;             // live objects
  int64_t n_slots;       // objects covered by the grid (n rounded up to the tile)
  int32_t n_features;
  const float* eytz;     // [F][eytz_pitch] Eytzinger-ordered borders, +inf padded
  int32_t eytz_pitch;    // 2^levels - 1
  uint8_t* out;          // tiled [tile][F][TILE] or plain [F][n]
  int32_t tile;          // TILE (tiled output only)
};

constexpr int kQuantObjects = 32;     // objects per CTA (one per lane)
constexpr int kQuantFeatures = 256;   // feature chunk per CTA (grid.y covers F)
constexpr int kQuantThreads = 256;

// bucket of x against one feature's Eytzinger array: i <- 2i + 1 + [x > e_i], L times.
template <int L>
__device__ __forceinline__ uint32_t eytz_bucket(float x, const float* __restrict__ e) {
  uint32_t i = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const float b = __ldg(e + i);
    i = 2 * i + 1 + (x > b ? 1u : 0u);
  }
  return i - ((1u << L) - 1u);
}

template <int L, int LAYOUT, bool TILED>
__global__ void __launch_bounds__(kQuantThreads) quantize_kernel(QuantizeParams p) {
  __shared__ float xs[kQuantObjects * (kQuantFeatures + 1)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o0 = (int64_t)blockIdx.x * kQuantObjects;
  const int f0 = blockIdx.y * kQuantFeatures;
  const int nf = min(kQuantFeatures, p.n_features - f0);
  constexpr int kPitch = kQuantFeatures + 1;  // odd pitch: column reads are conflict-free
  if (LAYOUT == 0) {
    // object-major: each warp copies whole row segments (coalesced) into smem.
    for (int r = warp; r < kQuantObjects; r += kQuantThreads / 32) {
      const int64_t o = o0 + r;
      const float* row = p.x + o * p.n_features + f0;
      for (int f = lane; f < nf; f += 32) xs[r * kPitch + f] = (o < p.n) ? __ldg(row + f) : 0.0f;
    }
    __syncthreads();
  }
  const int64_t o = o0 + lane;
  for (int fl = warp; fl < nf; fl += kQuantThreads / 32) {
    const int f = f0 + fl;
    float x;
    if (LAYOUT == 0) x = xs[lane * kPitch + fl];
    else x = (o < p.n) ? __ldg(p.x + (int64_t)f * p.n + o) : 0.0f;
    uint32_t q = eytz_bucket<L>(x, p.eytz + (int64_t)f * p.eytz_pitch);
    if (TILED) {
      if (o >= p.n) q = 0;  // padding slots are zero (quantize.py:172)
      const int64_t t = o / p.tile, w = o - t * p.tile;
      p.out[(t * p.n_features + f) * p.tile + w] = (uint8_t)q;
    } else if (o < p.n) {
      p.out[(int64_t)f * p.n + o] = (uint8_t)q;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: tree apply.
struct ApplyParams {
  const uint8_t* q;          // tiled buckets [n_tiles][F][tile]
  const uint8_t* chunks;     // [n_chunks][chunk_bytes] descriptor+leaf records
  double* out;               // [n] predictions (accumulate mode)
  uint16_t* idx_out;         // [tree_end - tree_begin][n] (index mode)
  int64_t n;
  int32_t tile;
  int32_t n_trees;
  int32_t chunk_trees;
  int32_t n_chunks;
  uint32_t chunk_bytes;      // multiple of 128
  uint32_t desc_bytes;       // descriptor part of a record (multiple of 16)
  uint32_t q_tile_bytes;     // F * tile
  int32_t n_stages;
  int32_t tree_begin, tree_end;
  double scale, bias;
};

// Descriptor of one (tree, depth) split.  off = byte offset of the feature's row in
// the bucket tile; k = per-byte addend that carries [q > ordinal] into bit 7;
// s = all-ones when ordinal < 128 (8-bit compare mode only).  A tree's descriptors
// are padded to a multiple of 16 bytes so they load as LDS.128 broadcasts.
struct alignas(8) Desc7 { uint32_t off, k; };
struct alignas(16) Desc8 { uint32_t off, k, s, pad; };

template <int CMP> struct DescT;
template <> struct DescT<7> { using D = Desc7; };
template <> struct DescT<8> { using D = Desc8; };

__host__ __device__ constexpr int desc_bytes_per_tree(int di, int cmp) {
  return cmp == 7 ? ((di * 8 + 15) / 16) * 16 : di * 16;
}

template <int LEAF> struct LeafT;
template <> struct LeafT<0> { using T = double; using Acc = double; static constexpr int kShift = 3;
  static __device__ __forceinline__ double widen(double v) { return v; } };
template <> struct LeafT<1> { using T = float; using Acc = double; static constexpr int kShift = 2;
  static __device__ __forceinline__ double widen(float v) { return (double)v; } };
template <> struct LeafT<2> { using T = __half; using Acc = float; static constexpr int kShift = 1;
  static __device__ __forceinline__ float widen(__half v) { return __half2float(v); } };

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (a & c) | (b & c);
}

// Byte k of a packed index word, zero-extended (one PRMT).
template <int K>
__device__ __forceinline__ uint32_t byte_of(uint32_t w) {
  return __byte_perm(w, 0u, 0x4440u | K);
}

template <int DI, int CMP, int LEAF, bool WRITE_IDX>
__global__ void __launch_bounds__(1024, 1) apply_kernel(ApplyParams p) {
  using LT = LeafT<LEAF>;
  using leaf_t = typename LT::T;
  using acc_t = typename LT::Acc;
  using Desc = typename DescT<CMP>::D;
  constexpr int kLeaves = 1 << DI;
  constexpr int kTreeDescBytes = desc_bytes_per_tree(DI, CMP);
  // When the scaled index still fits a byte, the SWAR words carry byte offsets
  // (index << kShift) directly and a gather is PRMT + LDS.
  constexpr bool kPrescaled = !WRITE_IDX && (DI + LT::kShift) <= 8;
  constexpr int kBitBase = kPrescaled ? LT::kShift : 0;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [0] tile, [1 + s] stage s
  unsigned char* stages = smem + 128;
  unsigned char* qtile = stages + (size_t)p.n_stages * p.chunk_bytes;

  const int tid = threadIdx.x;
  const int64_t tile_idx = blockIdx.x;
  if (tid == 0) {
    for (int i = 0; i <= p.n_stages; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bars[0], p.q_tile_bytes);
    bulk_g2s_split(qtile, p.q + tile_idx * (int64_t)p.q_tile_bytes, p.q_tile_bytes, &bars[0]);
    const int pre = p.n_chunks < p.n_stages ? p.n_chunks : p.n_stages;
    for (int s = 0; s < pre; ++s) {
      mbar_expect_tx(&bars[1 + s], p.chunk_bytes);
      bulk_g2s_split(stages + (size_t)s * p.chunk_bytes, p.chunks + (size_t)s * p.chunk_bytes,
                     p.chunk_bytes, &bars[1 + s]);
    }
  }
  mbar_wait(&bars[0], 0);

  const unsigned char* my_q = qtile + 4 * tid;  // this thread's 4 objects in every row
  const int64_t obj0 = tile_idx * p.tile + 4 * tid;
  acc_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;

  for (int c = 0; c < p.n_chunks; ++c) {
    const int s = c % p.n_stages;
    mbar_wait(&bars[1 + s], (uint32_t)(c / p.n_stages) & 1u);
    const unsigned char* st = stages + (size_t)s * p.chunk_bytes;
    const unsigned char* leaf_base = st + p.desc_bytes;
    const int t_base = c * p.chunk_trees;
    const int nt = min(p.chunk_trees, p.n_trees - t_base);
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      const Desc* desc = reinterpret_cast<const Desc*>(st + t * kTreeDescBytes);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int d = 0; d < DI; ++d) {
        const Desc ds = desc[d];
        const uint32_t w = *reinterpret_cast<const uint32_t*>(my_q + ds.off);
        uint32_t b7;  // [q > ordinal] in bit 7 of each byte, garbage below
        if constexpr (CMP == 7) {
          b7 = w + ds.k;
        } else {
          b7 = maj3((w & 0x7f7f7f7fu) + ds.k, w, ds.s);
        }
        const int pos = d + kBitBase;  // target bit of condition d inside each byte
        if (pos < 8) lo |= (pos == 7 ? b7 : (b7 >> (7 - pos))) & (0x01010101u << pos);
        else hi |= (pos == 15 ? b7 : (b7 >> (15 - pos))) & (0x01010101u << (pos - 8));
      }
      uint32_t i0, i1, i2, i3;
      if constexpr (DI > 8) {
        i0 = byte_of<0>(lo) | (byte_of<0>(hi) << 8);
        i1 = byte_of<1>(lo) | (byte_of<1>(hi) << 8);
        i2 = byte_of<2>(lo) | (byte_of<2>(hi) << 8);
        i3 = byte_of<3>(lo) | (byte_of<3>(hi) << 8);
      } else {
        i0 = byte_of<0>(lo);
        i1 = byte_of<1>(lo);
        i2 = byte_of<2>(lo);
        i3 = byte_of<3>(lo);
      }
      if constexpr (WRITE_IDX) {
        const int tg = t_base + t;
        if (tg >= p.tree_begin && tg < p.tree_end) {
          uint16_t* row = p.idx_out + (int64_t)(tg - p.tree_begin) * p.n;
          if (obj0 + 0 < p.n) row[obj0 + 0] = (uint16_t)i0;
          if (obj0 + 1 < p.n) row[obj0 + 1] = (uint16_t)i1;
          if (obj0 + 2 < p.n) row[obj0 + 2] = (uint16_t)i2;
          if (obj0 + 3 < p.n) row[obj0 + 3] = (uint16_t)i3;
        }
      } else {
        const unsigned char* tab = leaf_base + (size_t)t * (kLeaves * sizeof(leaf_t));
        constexpr int kSh = kPrescaled ? 0 : LT::kShift;
        acc0 += LT::widen(*reinterpret_cast<const leaf_t*>(tab + (i0 << kSh)));
        acc1 += LT::widen(*reinterpret_cast<const leaf_t*>(tab + (i1 << kSh)));
        acc2 += LT::widen(*reinterpret_cast<const leaf_t*>(tab + (i2 << kSh)));
        acc3 += LT::widen(*reinterpret_cast<const leaf_t*>(tab + (i3 << kSh)));
      }
    }
    __syncthreads();  // every thread is done reading stage s
    if (tid == 0 && c + p.n_stages < p.n_chunks) {
      mbar_expect_tx(&bars[1 + s], p.chunk_bytes);
      bulk_g2s_split(stages + (size_t)s * p.chunk_bytes,
                     p.chunks + (size_t)(c + p.n_stages) * p.chunk_bytes, p.chunk_bytes, &bars[1 + s]);
    }
  }

  if constexpr (!WRITE_IDX) {
    // finalize: f64(acc) * scale + bias, two roundings (evaluate.py:298-299, oracle.py:53-54)
    const double a[4] = {(double)acc0, (double)acc1, (double)acc2, (double)acc3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (obj0 + k < p.n) p.out[obj0 + k] = __dadd_rn(__dmul_rn(a[k], p.scale), p.bias);
    }
  }
}

}  // namespace obt
