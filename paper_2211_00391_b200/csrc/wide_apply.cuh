// wide_apply.cuh -- K2w: warp-specialised tree apply for wide feature sets.
//
// The reference's stages 2+3 and finalize (indexer.py:39-57, accumulate.py:88-97,
// evaluate.py:189-248, 298-299) for models whose bucket tile -- F bytes per object --
// leaves room for only a few hundred objects per SM (BASELINE config 4: F = 500, a
// 256-object tile is 125 KB).  With one lane per bucket word such a tile has two warps
// of work, too few to cover shared-memory latency; K2w splits the work by role instead
// of by object:
//
//   producer warps  three one-lane roles in three warps (three lanes of one warp, each in
//                   its own barrier wait, delayed each other's copies: config 4 apply 47.9
//                   -> 45.3 ms when split): chunk descriptors into an NS-slot ring, leaf
//                   tables into a TS-stage ring, the CTA's bucket tiles (persistent CTA:
//                   one per SM, looping over tiles)
//   index warps     NIDX warps share each chunk's 4-tree groups; the two halves of a warp
//                   take two trees of the group each, over all 256 objects: a lane builds
//                   the packed leaf indices of bucket words 4hl..4hl+3 (16 objects, SWAR:
//                   per depth one LDS.128, per word one add carrying [q > ordinal] into bit
//                   7 of each byte and one shift-and-or), so one descriptor load carries
//                   two trees' splits (one address per half-warp); the halves swap two
//                   words per tree (4 SHFL), each lane transposes the 4 x 4 index bytes of
//                   its two words (12 PRMT) so that one word holds one object's indices of
//                   the 4 trees, and stores them to the chunk's index panel [group][object]
//   fold warps      kWideTile / 32 warps, lane = object: per 4-tree group one panel load,
//                   four leaf gathers and four adds in tree order -- the reference's left
//                   fold, binary64 (binary32 for the binary16 family) -- then the
//                   two-rounding finalize and a coalesced store
//
// Shared-memory wavefronts per 128 object-trees at depth 8 (the resource that binds
// this path on B200): 8 bucket words, ~11 leaf gathers (4 x ~2.8 with entropy-ordered
// levels, see obtree_capi.cu level_order), 1 panel store + 1 panel load, 2 descriptor
// broadcasts (4 before the tree split), 0.5 index swaps.
#pragma once

#include "obtree_kernels.cuh"

namespace obt {

constexpr int kWideTile = 256;                   // objects per tile (64 bucket words)
constexpr int kWideWords = kWideTile / 4;
constexpr int kWideFoldWarps = kWideTile / 32;   // one lane per object
constexpr int kWideMaxTStages = 8;
constexpr int kWideMaxSlots = 16;
constexpr int kWideChunkTrees = 16;              // trees per ring chunk (null trees pad the last)
constexpr int kWideGroups = kWideChunkTrees / 4;  // 4-tree groups per chunk

// bytes between consecutive leaf tables of a chunk
__host__ __device__ constexpr uint32_t wide_table_stride(int di, int leaf) {
  return (((leaf == 0 ? 8u : leaf == 1 ? 4u : 2u) << di) + 15u) & ~15u;
}

struct WideParams {
  const uint8_t* q;          // tiled buckets [n_tiles][F][kWideTile]
  const uint8_t* desc;       // [n_chunks][wide_desc_bytes]: per tree DI {off, k} pairs
  const uint8_t* tables;     // [n_chunks][wide_tables_bytes]: leaf tables, kStride apart
  double* out;               // [n]
  int64_t n;
  int64_t n_tiles;
  int32_t n_chunks;
  uint32_t q_tile_bytes;     // F * kWideTile
  int32_t n_tstages;         // table ring stages (<= kWideMaxTStages)
  int32_t n_slots;           // descriptor + index-panel ring slots (<= kWideMaxSlots)
  int32_t chunk_begin;       // this launch folds chunks [chunk_begin, chunk_begin + n_chunks)
  int32_t first, last;       // start the fold at 0 / finalize into predictions (else carry in out)
  uint32_t zero;             // 0 (opaque to the compiler: see mbar_arrive_after)
  double scale, bias;
};

// Kernel arguments: DSRC 0 streams the descriptors through a shared-memory ring; DSRC 1
// carries this launch's descriptors in the kernel-parameter bank (uniform LDCU loads:
// no shared-memory wavefronts, and the bucket-word address takes the offset from a
// uniform register), one launch per kWideBankChunks chunks, the fold carried in `out`.
constexpr int kWideBankWords = (32760 - (int)sizeof(WideParams)) / 8 * 2;  // keeps the struct a multiple of 8 bytes
__host__ __device__ constexpr int wide_bank_chunks(int di) { return kWideBankWords / (kWideChunkTrees * 2 * di); }
template <int DSRC> struct WideArgs;
template <> struct WideArgs<0> { WideParams p; };
template <> struct WideArgs<1> { WideParams p; uint32_t desc[kWideBankWords]; };
static_assert(sizeof(WideArgs<1>) <= 32764, "kernel parameter space");

// Wait on the plain (potentially blocking) try_wait.  A suspend-time hint (a
// TRYWAIT / NANOSLEEP.SYNCS / PHASECHK loop) measured slower at config 4 (48.9 vs 48.2
// ms), and so did a nanosleep back-off in the fold warps' waits (200 ns: 47.74 vs 47.28).
__device__ __forceinline__ void wide_wait(uint64_t* bar, uint32_t parity) {
  // every lane retries on its own: two instructions per poll (try_wait, branch); the
  // voted warp-uniform loop (three) measured 45.05 vs 44.72 ms at config 4, one polling
  // lane joined by __syncwarp 89.6 ms
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WIDE_WAIT_RETRY:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra WIDE_WAIT_DONE;\n"
      "bra WIDE_WAIT_RETRY;\n"
      "WIDE_WAIT_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Shared-memory layout (2048-byte aligned base):
//   table ring           TS x kWideChunkTrees tables (each stride-aligned, so a gather
//                        address is one LOP3: (shifted index & mask) | table base, plus
//                        the tree's compile-time offset)
//   descriptor ring      NS x wide_desc_bytes
//   index-panel ring     NS x kWideGroups x kWideTile x 4 bytes
//   bucket tile          q_tile_bytes
//   barriers
// The descriptor / panel ring is deeper than the table ring: the index warps run up to
// NS chunks ahead of the fold, so neither side waits on the other's latency.
__host__ __device__ constexpr size_t wide_panel_bytes(int chunk_trees) { return (size_t)chunk_trees * kWideTile; }
// descriptor bytes per tree: DI pairs of words, rounded to whole 16-byte loads
__host__ __device__ constexpr uint32_t kWideDescBytes(int di) { return (uint32_t)((di + 1) / 2) * 16u; }
__host__ __device__ constexpr uint32_t wide_desc_bytes(int di) { return (kWideChunkTrees * kWideDescBytes(di) + 127u) & ~127u; }
__host__ __device__ constexpr uint32_t wide_tables_bytes(int di, int leaf) { return kWideChunkTrees * wide_table_stride(di, leaf); }
constexpr uint32_t kWideSmemAlign = 2048;  // the largest table stride (binary64, depth 8)
constexpr uint32_t kWideSmemSlack = kWideSmemAlign + 16 + 8 * (2 * kWideMaxTStages + 3 * kWideMaxSlots + 2);

// 4 x 4 byte transpose: out[k] byte j = in[j] byte k.
__device__ __forceinline__ void transpose4x4(const uint32_t (&in)[4], uint32_t (&out)[4]) {
  const uint32_t ab_lo = __byte_perm(in[0], in[1], 0x5140u);  // a0 b0 a1 b1
  const uint32_t ab_hi = __byte_perm(in[0], in[1], 0x7362u);  // a2 b2 a3 b3
  const uint32_t cd_lo = __byte_perm(in[2], in[3], 0x5140u);  // c0 d0 c1 d1
  const uint32_t cd_hi = __byte_perm(in[2], in[3], 0x7362u);  // c2 d2 c3 d3
  out[0] = __byte_perm(ab_lo, cd_lo, 0x5410u);                // a0 b0 c0 d0
  out[1] = __byte_perm(ab_lo, cd_lo, 0x7632u);                // a1 b1 c1 d1
  out[2] = __byte_perm(ab_hi, cd_hi, 0x5410u);
  out[3] = __byte_perm(ab_hi, cd_hi, 0x7632u);
}

// Ring position: slot and phase parity, advanced without divisions.
struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) { slot = 0; phase ^= 1u; }
  }
};

template <int DI, int CMP, int LEAF, int NIDX, int DSRC>
__global__ void __launch_bounds__(32 * (3 + NIDX + kWideFoldWarps), 1) apply_wide_kernel(const __grid_constant__ WideArgs<DSRC> args) {
  const WideParams& p = args.p;
  static_assert(DI >= 1 && DI <= 8, "K2w: one index byte per object");
  using LT = LeafT<LEAF>;
  using acc_t = typename LT::Acc;
  constexpr uint32_t kTablesBytes = wide_tables_bytes(DI, LEAF), kDescBytes = wide_desc_bytes(DI);
  constexpr uint32_t kPanelBytes = (uint32_t)wide_panel_bytes(kWideChunkTrees);
  constexpr uint32_t kStride = wide_table_stride(DI, LEAF);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((kWideSmemAlign - (smem_u32(smem_raw) & (kWideSmemAlign - 1u))) & (kWideSmemAlign - 1u));
  const int TS = p.n_tstages, NS = p.n_slots;
  unsigned char* tstages = smem;                                      // TS x kTablesBytes (stride-aligned)
  unsigned char* descs = tstages + (size_t)TS * kTablesBytes;         // NS x kDescBytes (DSRC 0)
  unsigned char* panels = descs + (DSRC == 0 ? (size_t)NS * kDescBytes : 0);  // NS x kPanelBytes
  unsigned char* qtile = panels + (size_t)NS * kPanelBytes;           // q_tile_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(qtile + ((p.q_tile_bytes + 15u) & ~15u));
  uint64_t* tfull = bars;                          // [TS] tables landed
  uint64_t* tfree = tfull + kWideMaxTStages;       // [TS] fold done with the tables
  uint64_t* dfull = tfree + kWideMaxTStages;       // [NS] descriptors landed (slot free)
  uint64_t* pfull = dfull + kWideMaxSlots;         // [NS] index panel written
  uint64_t* sfree = pfull + kWideMaxSlots;         // [NS] fold done with the panel
  uint64_t* tile_full = sfree + kWideMaxSlots;
  uint64_t* tile_free = tile_full + 1;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < TS; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tfree[i], kWideFoldWarps * 32);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&pfull[i], NIDX * 32);
      mbar_init(&sfree[i], kWideFoldWarps * 32);
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

  // producer roles, one per warp (lanes of one warp in three different waits serialise
  // each other's issue): warp 0 descriptors, the last two warps bucket tiles and tables
  const int role = warp == 0 ? 0 : warp == 1 + NIDX + kWideFoldWarps ? 1 : warp == 2 + NIDX + kWideFoldWarps ? 2 : -1;
  if (role >= 0) {
    if (lane != 0) return;
    if (role == 0 && DSRC == 0) {
      // descriptors, NS chunks ahead of the fold: index warps run ahead of the fold by
      // up to NS chunks, decoupled from the (larger) table ring
      RingPos r;
      for (int64_t i = 0; i < n_my_tiles; ++i) {
        for (int c = 0; c < nc; ++c) {
          if (i > 0 || c >= NS) mbar_wait(&sfree[r.slot], r.phase ^ 1u);
          mbar_expect_tx(&dfull[r.slot], kDescBytes);
          bulk_g2s(descs + (size_t)r.slot * kDescBytes, p.desc + (size_t)(p.chunk_begin + c) * kDescBytes, kDescBytes,
                   &dfull[r.slot]);
          r.next(NS);
        }
      }
    } else if (role == 1) {
      // bucket tiles: the next one as soon as the index warps release the current one
      for (int64_t i = 0; i < n_my_tiles; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (i > 0) mbar_wait(tile_free, (uint32_t)((i - 1) & 1));
        mbar_expect_tx(tile_full, p.q_tile_bytes);
        bulk_g2s_split(qtile, p.q + tile * (int64_t)p.q_tile_bytes, p.q_tile_bytes, tile_full);
        if (i + 1 < n_my_tiles) bulk_prefetch_l2(p.q + (tile + gridDim.x) * (int64_t)p.q_tile_bytes, p.q_tile_bytes);
      }
    } else if (role == 2) {
      // leaf tables, TS chunks ahead of the fold
      RingPos r;
      for (int64_t i = 0; i < n_my_tiles; ++i) {
        for (int c = 0; c < nc; ++c) {
          if (i > 0 || c >= TS) mbar_wait(&tfree[r.slot], r.phase ^ 1u);
          mbar_expect_tx(&tfull[r.slot], kTablesBytes);
          bulk_g2s_split(tstages + (size_t)r.slot * kTablesBytes, p.tables + (size_t)(p.chunk_begin + c) * kTablesBytes,
                         kTablesBytes, &tfull[r.slot]);
          r.next(TS);
        }
      }
    }
    return;
  }

  if (warp <= NIDX) {
    // ---------------- index warps
    const int iw = warp - 1;
    // lane l owns bucket words 2l and 2l + 1 (one LDS.64 per depth): objects
    // blk * 128 + p + 32k and blk * 128 + p + 1 + 32k, blk = l / 16, p = 2l mod 32
    const uint32_t q0 = smem_u32(qtile) + 8u * lane;
    const int obj0 = (lane >> 4) * 128 + ((2 * lane) & 31);
    int rr = iw;  // round-robin position of this warp's next group across chunks
    RingPos r;
    for (int64_t i = 0; i < n_my_tiles; ++i) {
      wide_wait(tile_full, (uint32_t)(i & 1));
      for (int c = 0; c < nc; ++c) {
        if constexpr (DSRC == 0) {
          wide_wait(&dfull[r.slot], r.phase);
        } else if (i > 0 || c >= NS) {
          wide_wait(&sfree[r.slot], r.phase ^ 1u);  // the fold is done with this panel slot
        }
        const unsigned char* st = descs + (size_t)r.slot * kDescBytes;
        const uint32_t panel = smem_u32(panels + (size_t)r.slot * kPanelBytes) + 4u * obj0;
        if constexpr (DSRC == 0) {
          // Tree-split halves (config 4 apply 45.1 -> 43.9 ms against every lane taking all
          // four trees of a group over 8 objects, the form the parameter-bank source keeps): lanes 0-15 take trees 4g, 4g+1 and lanes 16-31 trees 4g+2,
          // 4g+3, each half over all 256 objects (lane hl: bucket words 4hl..4hl+3, one
          // LDS.128 per depth).  One descriptor load now carries two trees' splits (one
          // address per half-warp), so a group costs half the descriptor broadcasts, half the
          // bucket loads and address adds; the halves then swap two words per tree (4 SHFL)
          // so that every lane holds the four trees' indices of 8 objects, as before.
          const int half = lane >> 4, hl = lane & 15;
          const uint32_t qh = smem_u32(qtile) + 16u * hl;
          const int w0i = 4 * hl + 2 * half;                       // first kept bucket word
          const int objk = (w0i >> 5) * 128 + (w0i & 31);
          const uint32_t panel_t = smem_u32(panels + (size_t)r.slot * kPanelBytes) + 4u * objk;
          const uint32_t sel_lo = half ? 0x1054u : 0x5410u, sel_hi = half ? 0x3276u : 0x7632u;
          for (; rr < kWideGroups; rr += NIDX) {
            const int g = rr;
            uint32_t ix[2][4];  // [local tree][word]
#pragma unroll
            for (int tl = 0; tl < 2; ++tl) {
              const int t = 4 * g + 2 * half + tl;
              uint32_t dw[2 * DI + 2];
              const uint4* dsrc = reinterpret_cast<const uint4*>(st + (size_t)t * kWideDescBytes(DI));
#pragma unroll
              for (int v = 0; v < (DI + 1) / 2; ++v) {
                const uint4 q4 = dsrc[v];
                dw[4 * v + 0] = q4.x; dw[4 * v + 1] = q4.y; dw[4 * v + 2] = q4.z; dw[4 * v + 3] = q4.w;
              }
              uint32_t w[DI][4];
#pragma unroll
              for (int d = 0; d < DI; ++d) {
                const uint32_t off = CMP == 7 ? dw[2 * d] : (dw[2 * d] >> 8);
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w[d][0]), "=r"(w[d][1]), "=r"(w[d][2]), "=r"(w[d][3]) : "r"(qh + off));
              }
              uint32_t a[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int d = 0; d < DI; ++d) {
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                  uint32_t b;
                  if constexpr (CMP == 7) {
                    b = w[d][x] + dw[2 * d + 1];
                  } else {
                    const uint32_t k = __byte_perm(dw[2 * d], 0u, 0x0000u) & 0x7f7f7f7fu;
                    b = maj3((w[d][x] & 0x7f7f7f7fu) + k, w[d][x], dw[2 * d + 1]);
                  }
                  a[x] = (a[x] >> 1) | (b & 0x80808080u);
                }
              }
#pragma unroll
              for (int x = 0; x < 4; ++x) ix[tl][x] = DI < 8 ? a[x] >> (8 - DI) : a[x];
            }
            // swap: a lane keeps words 2 half, 2 half + 1 and receives its partner's trees for them
            uint32_t own[2][2], got[2][2];
#pragma unroll
            for (int tl = 0; tl < 2; ++tl)
#pragma unroll
              for (int x = 0; x < 2; ++x) {
                own[tl][x] = half ? ix[tl][x + 2] : ix[tl][x];
                got[tl][x] = __shfl_xor_sync(0xffffffffu, half ? ix[tl][x] : ix[tl][x + 2], 16);
              }
            // 4 x 4 byte transpose per kept word; the selectors put the received pair first
            // (lanes 16-31: trees 4g, 4g+1 come from the partner) or second
            uint32_t o[2][4];
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              const uint32_t own_lo = __byte_perm(own[0][x], own[1][x], 0x5140u), own_hi = __byte_perm(own[0][x], own[1][x], 0x7362u);
              const uint32_t got_lo = __byte_perm(got[0][x], got[1][x], 0x5140u), got_hi = __byte_perm(got[0][x], got[1][x], 0x7362u);
              o[x][0] = __byte_perm(own_lo, got_lo, sel_lo);
              o[x][1] = __byte_perm(own_lo, got_lo, sel_hi);
              o[x][2] = __byte_perm(own_hi, got_hi, sel_lo);
              o[x][3] = __byte_perm(own_hi, got_hi, sel_hi);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(panel_t + (uint32_t)g * (kWideTile * 4) + 128u * k),
                           "r"(o[0][k]), "r"(o[1][k]) : "memory");
          }
        } else
        for (; rr < kWideGroups; rr += NIDX) {
          const int g = rr;
          uint32_t i0[4], i1[4];  // packed indices of trees 4g..4g+3, words 2l and 2l + 1
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = 4 * g + j;
            // descriptors: DI pairs {off, k replicated} (7-bit) or {(off << 8) | k, s}
            // (8-bit), two pairs per broadcast LDS.128
            uint32_t dw[2 * DI + 2];
            if constexpr (DSRC == 0) {
              const uint4* dsrc = reinterpret_cast<const uint4*>(st + (size_t)t * kWideDescBytes(DI));
#pragma unroll
              for (int v = 0; v < (DI + 1) / 2; ++v) {
                const uint4 q4 = dsrc[v];
                dw[4 * v + 0] = q4.x; dw[4 * v + 1] = q4.y; dw[4 * v + 2] = q4.z; dw[4 * v + 3] = q4.w;
              }
            } else {
              const uint32_t* bank = args.desc + ((size_t)c * kWideChunkTrees + t) * (2 * DI);
#pragma unroll
              for (int v = 0; v < 2 * DI; ++v) dw[v] = bank[v];
            }
            uint32_t w0[DI], w1[DI];
#pragma unroll
            for (int d = 0; d < DI; ++d) {
              const uint32_t off = CMP == 7 ? dw[2 * d] : (dw[2 * d] >> 8);
              asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0[d]), "=r"(w1[d]) : "r"(q0 + off));
            }
            // LSB-first: acc = (acc >> 1) | (bit 7 of each byte of b); after DI steps depth
            // d sits at bit 8 - DI + d of each byte (no bit crosses a byte: a bit reaches
            // position 0 only at the last step of a depth-8 tree)
            uint32_t a0 = 0, a1 = 0;
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
              a0 = (a0 >> 1) | (b0 & 0x80808080u);
              a1 = (a1 >> 1) | (b1 & 0x80808080u);
            }
            if constexpr (DI < 8) {
              a0 >>= 8 - DI;
              a1 >>= 8 - DI;
            }
            i0[j] = a0;
            i1[j] = a1;
          }
          uint32_t o0[4], o1[4];
          transpose4x4(i0, o0);
          transpose4x4(i1, o1);
          // objects obj0 + 32k and obj0 + 1 + 32k are adjacent panel words: one STS.64
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(panel + (uint32_t)g * (kWideTile * 4) + 128u * k),
                         "r"(o0[k]), "r"(o1[k]) : "memory");
        }
        rr -= kWideGroups;
        // (the descriptor slot is refilled only after the fold's sfree arrive, and every
        // descriptor and bucket word read here fed the panel stores above: none is in flight)
        mbar_arrive(&pfull[r.slot]);
        r.next(NS);
      }
      mbar_release(tile_free);  // the bucket tile is refilled by a bulk copy
    }
    return;
  }

  // ---------------- fold warps: lane = object fw * 32 + lane of the tile
  const int fw = warp - 1 - NIDX;
  const int ol = fw * 32 + lane;
  RingPos r, rt;
  // Table release.  The copy engine refills a table stage once every fold thread has
  // arrived on its tfree barrier, so a thread may arrive only after all its gathers from
  // that stage returned (mbar_release explains what happens otherwise).  The arrive's
  // address is made to depend on the chunk's final sum -- every gathered leaf went into
  // it -- and is issued one chunk later, behind the next chunk's gathers, so the wait for
  // the tail of the add chain overlaps their latency (arriving right behind the adds:
  // 46.9 ms at config 4; a proxy fence per chunk: 50.5).
  int pend = -1;  // table slot whose release awaits the sum of the chunk folded from it
  for (int64_t i = 0; i < n_my_tiles; ++i) {
    const int64_t tile = blockIdx.x + i * gridDim.x;
    const int64_t o = tile * kWideTile + ol;
    // continue the fold of the previous launch (exact: the carry holds acc_t values)
    acc_t acc = (p.first || o >= p.n) ? (acc_t)0 : (acc_t)p.out[o];
    for (int c = 0; c < nc; ++c) {
      wide_wait(&pfull[r.slot], r.phase);
      wide_wait(&tfull[rt.slot], rt.phase);
      const uint32_t panel = smem_u32(panels + (size_t)r.slot * kPanelBytes) + 4u * ol;
      const uint32_t tables = smem_u32(tstages + (size_t)rt.slot * kTablesBytes);  // kStride-aligned
      // the chunk's panel words, then its 4 x kWideGroups gathers (gather address: one
      // LOP3 of the shifted index byte into the aligned table base, plus the tree's
      // compile-time offset), then the adds in tree order
      uint32_t iwd[kWideGroups];
#pragma unroll
      for (int g = 0; g < kWideGroups; ++g) iwd[g] = lds_u32<false>(panel + (uint32_t)g * (kWideTile * 4));
      typename LT::T v[kWideGroups][4];
#pragma unroll
      for (int g = 0; g < kWideGroups; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[g][j] = lds_leaf<LEAF, false>((((iwd[g] >> (8 * j)) << LT::kShift) & (0xffu << LT::kShift) | tables) +
                                          (uint32_t)(4 * g + j) * kStride);
      mbar_arrive(&sfree[r.slot]);
      if (pend >= 0) mbar_arrive_after(&tfree[pend], dep_bits(acc), p.zero);  // acc: through the previous chunk
#pragma unroll
      for (int g = 0; g < kWideGroups; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc += LT::widen(v[g][j]);
      pend = rt.slot;
      r.next(NS);
      rt.next(TS);
    }
    if (pend >= 0) mbar_arrive_after(&tfree[pend], dep_bits(acc), p.zero);  // the tile's last chunk
    pend = -1;
    // finalize: f64(acc) * scale + bias, two roundings (evaluate.py:298-299)
    if (o < p.n) p.out[o] = p.last ? __dadd_rn(__dmul_rn((double)acc, p.scale), p.bias) : (double)acc;
  }
}

}  // namespace obt
