// wide_apply.cuh -- K2w: warp-specialised tree apply for wide feature sets.
//
// The reference's stages 2+3 and finalize (indexer.py:39-57, accumulate.py:88-97,
// evaluate.py:189-248, 298-299) for models whose bucket tile -- F bytes per object --
// leaves room for only a few hundred objects per SM (BASELINE config 4: F = 500, a
// 256-object tile is 125 KB).  With one lane per bucket word such a tile has two warps
// of work, too few to cover shared-memory latency; K2w splits the work by role instead
// of by object:
//
//   producer warp   lane 0 streams tree chunks (descriptors + leaf tables) into an
//                   S-stage ring, lane 1 streams the CTA's bucket tiles (persistent
//                   CTA: one per SM, looping over tiles)
//   index warps     NIDX warps share each chunk's trees (tree j -> warp j mod NIDX);
//                   a lane builds the packed leaf indices of bucket words l and l + 32
//                   (8 objects, SWAR: per depth one LDS per word, one add carrying
//                   [q > ordinal] into bit 7 of each byte, one shift-and-or) and
//                   stores them to the chunk's index panel [tree][64 words]
//   fold warps      2 warps, lane = bucket word (4 objects): per tree one panel load,
//                   four leaf gathers and four adds in tree order -- the reference's
//                   left fold, binary64 (binary32 for the binary16 family) -- then the
//                   two-rounding finalize
//
// Shared-memory wavefronts per 128 object-trees at depth 8 (the resource that binds
// this path on B200): 8 bucket words, ~10.5 leaf gathers (4 x ~2.6 with entropy-ordered
// levels, see obtree_capi.cu level_order), 2 panel stores + loads, 2 descriptor
// broadcasts, ~4 of TMA ring fill (1 KB tables over 256 objects).
#pragma once

#include "obtree_kernels.cuh"

namespace obt {

constexpr int kWideTile = 256;                 // objects per tile (64 bucket words)
constexpr int kWideWords = kWideTile / 4;
constexpr int kWideFoldWarps = kWideWords / 32;  // one lane per word
constexpr int kWideMaxStages = 8;

struct WideParams {
  const uint8_t* q;          // tiled buckets [n_tiles][F][kWideTile]
  const uint8_t* chunks;     // [n_chunks][chunk_bytes]: descriptors (desc_bytes) + leaf tables
  double* out;               // [n]
  int64_t n;
  int64_t n_tiles;
  int32_t n_chunks;
  int32_t chunk_trees;       // trees per chunk (the last chunk is padded with null trees)
  uint32_t chunk_bytes;      // multiple of 256
  uint32_t desc_bytes;       // descriptor part of a chunk (multiple of 256)
  uint32_t table_stride;     // bytes between consecutive leaf tables
  uint32_t q_tile_bytes;     // F * kWideTile
  int32_t n_stages;          // <= kWideMaxStages
  double scale, bias;
};

// Warp-wide wait with a suspend hint: waiting warps leave the issue slots to the others.
__device__ __forceinline__ void wide_wait(uint64_t* bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try_suspend(bar, parity, 20000u))) {
  }
}

// Shared-memory layout (after the 256-byte aligned base):
//   [0, 256)             barriers: full[S], idx_done[S], empty[S], tile_full, tile_free
//   stages               S x chunk_bytes
//   panels               S x chunk_trees x kWideWords x 4 bytes
//   tile                 q_tile_bytes
__host__ __device__ constexpr size_t wide_panel_bytes(int chunk_trees) { return (size_t)chunk_trees * kWideWords * 4; }
// descriptor bytes per tree: DI pairs of words, rounded to whole 16-byte loads
__host__ __device__ constexpr uint32_t kWideDescBytes(int di) { return (uint32_t)((di + 1) / 2) * 16u; }

template <int DI, int CMP, int LEAF, int NIDX>
__global__ void __launch_bounds__(32 * (1 + NIDX + kWideFoldWarps), 1) apply_wide_kernel(const __grid_constant__ WideParams p) {
  static_assert(DI >= 1 && DI <= 8, "K2w: one index byte per object");
  using LT = LeafT<LEAF>;
  using acc_t = typename LT::Acc;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((256u - (smem_u32(smem_raw) & 255u)) & 255u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* idx_done = full + kWideMaxStages;
  uint64_t* empty = idx_done + kWideMaxStages;
  uint64_t* tile_full = empty + kWideMaxStages;
  uint64_t* tile_free = tile_full + 1;
  const int S = p.n_stages;
  unsigned char* stages = smem + 256;
  unsigned char* panels = stages + (size_t)S * p.chunk_bytes;
  const size_t panel_bytes = wide_panel_bytes(p.chunk_trees);
  unsigned char* qtile = panels + (size_t)S * panel_bytes;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&idx_done[i], NIDX * 32);
      mbar_init(&empty[i], kWideFoldWarps * 32);
    }
    mbar_init(tile_full, 1);
    mbar_init(tile_free, NIDX * 32);
    fence_mbar_init();
  }
  __syncthreads();

  const int warp = __shfl_sync(0xffffffffu, tid / 32, 0);
  const int lane = tid & 31;
  const int64_t n_my_tiles = p.n_tiles > blockIdx.x ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nc = p.n_chunks;

  if (warp == 0) {
    if (lane == 0) {
      // tree chunks, continuously across this CTA's tiles
      for (int64_t i = 0; i < n_my_tiles; ++i) {
        for (int c = 0; c < nc; ++c) {
          const int64_t seq = i * nc + c;
          const int s = (int)(seq % S);
          if (seq >= S) mbar_wait(&empty[s], (uint32_t)((seq / S - 1) & 1));
          mbar_expect_tx(&full[s], p.chunk_bytes);
          bulk_g2s_split(stages + (size_t)s * p.chunk_bytes, p.chunks + (size_t)c * p.chunk_bytes, p.chunk_bytes,
                         &full[s]);
        }
      }
    } else if (lane == 1) {
      // bucket tiles: the next one as soon as the index warps release the current one
      for (int64_t i = 0; i < n_my_tiles; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (i > 0) mbar_wait(tile_free, (uint32_t)((i - 1) & 1));
        mbar_expect_tx(tile_full, p.q_tile_bytes);
        bulk_g2s_split(qtile, p.q + tile * (int64_t)p.q_tile_bytes, p.q_tile_bytes, tile_full);
        if (i + 1 < n_my_tiles) bulk_prefetch_l2(p.q + (tile + gridDim.x) * (int64_t)p.q_tile_bytes, p.q_tile_bytes);
      }
    }
    return;
  }

  if (warp <= NIDX) {
    // ---------------- index warps
    const int iw = warp - 1;
    const uint32_t q0 = smem_u32(qtile) + 4u * lane;  // bucket word `lane` of every row; + 128: word lane + 32
    for (int64_t i = 0; i < n_my_tiles; ++i) {
      wide_wait(tile_full, (uint32_t)(i & 1));
      for (int c = 0; c < nc; ++c) {
        const int64_t seq = i * nc + c;
        const int s = (int)(seq % S);
        wide_wait(&full[s], (uint32_t)((seq / S) & 1));
        const unsigned char* st = stages + (size_t)s * p.chunk_bytes;
        uint32_t* panel = reinterpret_cast<uint32_t*>(panels + (size_t)s * panel_bytes);
        for (int t = iw; t < p.chunk_trees; t += NIDX) {
          // descriptors: DI pairs {off, k replicated} (7-bit) or {(off << 8) | k, s} (8-bit),
          // two pairs per broadcast LDS.128
          uint32_t dw[2 * DI + 2];
          const uint4* dsrc = reinterpret_cast<const uint4*>(st + (size_t)t * kWideDescBytes(DI));
#pragma unroll
          for (int v = 0; v < (DI + 1) / 2; ++v) {
            const uint4 q4 = dsrc[v];
            dw[4 * v + 0] = q4.x; dw[4 * v + 1] = q4.y; dw[4 * v + 2] = q4.z; dw[4 * v + 3] = q4.w;
          }
          uint32_t w0[DI], w1[DI];
#pragma unroll
          for (int d = 0; d < DI; ++d) {
            const uint32_t off = CMP == 7 ? dw[2 * d] : (dw[2 * d] >> 8);
            w0[d] = lds_u32<false>(q0 + off);
            w1[d] = lds_u32<false>(q0 + off + 128u);
          }
          uint32_t i0 = 0, i1 = 0;
#pragma unroll
          for (int d = 0; d < DI; ++d) {
            uint32_t b0, b1;
            if constexpr (CMP == 7) {
              b0 = w0[d] + dw[2 * d + 1];
              b1 = w1[d] + dw[2 * d + 1];
            } else {
              const uint32_t k = __byte_perm(dw[2 * d], 0u, 0x0000u) & 0x7f7f7f7fu;
              b0 = maj3((w0[d] & 0x7f7f7f7fu) + k, w0[d], dw[2 * d + 1]);
              b1 = maj3((w1[d] & 0x7f7f7f7fu) + k, w1[d], dw[2 * d + 1]);
            }
            const uint32_t mask = 0x01010101u << d;
            i0 |= (d == 7 ? b0 : (b0 >> (7 - d))) & mask;
            i1 |= (d == 7 ? b1 : (b1 >> (7 - d))) & mask;
          }
          panel[t * kWideWords + lane] = i0;
          panel[t * kWideWords + 32 + lane] = i1;
        }
        mbar_arrive(&idx_done[s]);
      }
      mbar_arrive(tile_free);
    }
    return;
  }

  // ---------------- fold warps: lane = bucket word fw * 32 + lane
  const int fw = warp - 1 - NIDX;
  const int wi = fw * 32 + lane;
  for (int64_t i = 0; i < n_my_tiles; ++i) {
    const int64_t tile = blockIdx.x + i * gridDim.x;
    const int64_t tile_base = tile * kWideTile;
    acc_t acc[4] = {(acc_t)0, (acc_t)0, (acc_t)0, (acc_t)0};
    for (int c = 0; c < nc; ++c) {
      const int64_t seq = i * nc + c;
      const int s = (int)(seq % S);
      wide_wait(&idx_done[s], (uint32_t)((seq / S) & 1));
      wide_wait(&full[s], (uint32_t)((seq / S) & 1));  // (already complete: makes the TMA writes visible here)
      const uint32_t panel = smem_u32(panels + (size_t)s * panel_bytes) + 4u * wi;
      const uint32_t tables = smem_u32(stages + (size_t)s * p.chunk_bytes + p.desc_bytes);
      // groups of 4 trees, software-pipelined: the panel words of group g + 1 are
      // requested before group g's 16 gathers, whose adds then run in tree order
      uint32_t nxt[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) nxt[j] = lds_u32<true>(panel + (uint32_t)j * (kWideWords * 4));
      for (int t0 = 0; t0 < p.chunk_trees; t0 += 4) {
        uint32_t iw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) iw[j] = nxt[j];
        if (t0 + 4 < p.chunk_trees) {
#pragma unroll
          for (int j = 0; j < 4; ++j) nxt[j] = lds_u32<true>(panel + (uint32_t)(t0 + 4 + j) * (kWideWords * 4));
        }
        typename LT::T v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t tab = tables + (uint32_t)(t0 + j) * p.table_stride;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            v[j][k] = lds_leaf<LEAF, true>(tab + (((iw[j] >> (8 * k)) & 0xffu) << LT::kShift));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (LEAF == 2 && OBT_FADD2) {
            fadd2(acc[0], acc[1], LT::widen(v[j][0]), LT::widen(v[j][1]));
            fadd2(acc[2], acc[3], LT::widen(v[j][2]), LT::widen(v[j][3]));
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] += LT::widen(v[j][k]);
          }
        }
      }
      mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t o = word_object(tile_base, wi, k);
      // finalize: f64(acc) * scale + bias, two roundings (evaluate.py:298-299)
      if (o < p.n) p.out[o] = __dadd_rn(__dmul_rn((double)acc[k], p.scale), p.bias);
    }
  }
}

}  // namespace obt
