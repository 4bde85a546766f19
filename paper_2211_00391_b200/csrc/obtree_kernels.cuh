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
//
// Kernel index (DESIGN.md section 4 has each one's bound and measurements):
//   K1   quantize_kernel          LDG-loaded rows; Eytzinger search or cell tables
//   K1t  quantize_tma_kernel      TMA-staged rows, Eytzinger search
//   K1L  quantize_lut_kernel      TMA-staged rows, cell-table search (256 / 1024 cells)
//   K2   apply_kernel             one lane per bucket word; software-pipelined; descriptors
//                                 from the parameter bank (chained launches) or the ring
//   K2f  apply_fan_kernel         small batches: trees fanned out over 12 warps, in-order
//                                 fold by 4 fold warps
//   K2s  apply_split_kernel       depth-split lanes (wide feature sets)
//   K4   apply_multi_kernel       multi-output, records gathered from L2
//   K5   apply_multi_staged_kernel multi-output, per-tree tables + bucket rows staged by TMA
#pragma once

#include <cuda.h>
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

__device__ __forceinline__ uint32_t mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok;
}

// try_wait with a suspend-time hint: the thread sleeps in hardware until the phase
// completes (or the hint, in ns, elapses), instead of re-issuing the probe.
__device__ __forceinline__ uint32_t mbar_try_suspend(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok;
}

#ifndef OBT_PRODUCER_SUSPEND_NS
#define OBT_PRODUCER_SUSPEND_NS 1000000
#endif
// Single-thread wait (the producer).  A probe + nanosleep(64) loop measured 13 M
// re-issued probes per cfg2 apply launch (17% of the launch's warp instructions, issue
// slots taken from the consumer warps of the producer's SM sub-partition); with a
// suspend hint the producer sleeps until the consumers release the stage.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_suspend(bar, parity, OBT_PRODUCER_SUSPEND_NS)) {
  }
}

// Whole-warp wait whose retry branch is warp-uniform (vote), so code after it stays in
// uniform control flow and loop counters can live in uniform registers.
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try(bar, parity))) {
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer release of a buffer the producer refills with a bulk / tensor copy (async
// proxy) after this thread read it with ordinary shared loads (generic proxy): the proxy
// fence orders those reads before the refill.  Without it the arrive can overtake loads
// still queued in the shared-memory pipe, and the copy engine then overwrites the stage
// under them: K1L at F = 2,000 (a busy pipe: conflicted table lookups of the other warps)
// quantized one warp's 128 objects of one 8-feature step from the NEXT step's rows in
// ~20% of predicts (tests/stress/repro_buckets.py; 0 of 100 with the fence).
__device__ __forceinline__ void mbar_release(uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_arrive(bar);
}

// The same release without the fence, for K2w's fold warps, where a fence per chunk costs
// too much (config 4 apply 44.7 -> 50.5 ms): the arrive's barrier address is made to depend
// on `dep` (bar | (dep & zero), `zero` a kernel parameter that is 0), a value computed from
// every load of the buffer -- the chunk's final sum -- so the arrive cannot issue before
// all of them returned.
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, uint32_t dep, uint32_t zero) {
  uint32_t a;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xF8;" : "=r"(a) : "r"(smem_u32(bar)), "r"(dep), "r"(zero));
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ uint32_t dep_bits(double v) { return (uint32_t)__double2hiint(v); }
__device__ __forceinline__ uint32_t dep_bits(float v) { return __float_as_uint(v); }


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

// Launch chaining: let the dependent launch start (its CTAs take SMs as ours finish).
__device__ __forceinline__ void launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* a, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// Spin until *a >= want (bounded: a lost dependency traps instead of hanging the GPU).
__device__ __forceinline__ void wait_flag(const uint32_t* a, uint32_t want) {
  uint32_t spins = 0;
  while (ld_acquire_gpu(a) < want) {
    __nanosleep(256);
    if (++spins > (1u << 26)) asm volatile("trap;");
  }
}

// Named barrier among the CTA's consumer warps (id 1; the producer warp has left).
__device__ __forceinline__ void consumer_sync(int n_threads) {
  asm volatile("bar.sync 1, %0;" ::"r"(n_threads) : "memory");
}

// L2 prefetch of a global range by the TMA engine (no shared-memory destination), in
// pieces of at most 64 KiB.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  constexpr uint32_t kPiece = 65536;
  for (uint32_t done = 0; done < bytes; done += kPiece) {
    const uint32_t len = (bytes - done) < kPiece ? (bytes - done) : kPiece;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(src) + done), "r"(len)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// Tile layout of the bucket matrix Q[tile][F][TILE]: within each 128-object block of a
// tile, bucket word p (bytes 4p..4p+3 of every feature row) holds objects p, p+32, p+64,
// p+96 (byte k -> object p + 32k).  A quantize lane then owns objects one apart from its
// neighbours' (coalesced feature-major loads, conflict-free staged rows) and apply
// threads write consecutive outputs.  wi = word index within the tile.
__device__ __forceinline__ int64_t word_object(int64_t tile_base, int wi, int k) {
  return tile_base + (int64_t)((wi >> 5) * 128 + (wi & 31) + 32 * k);
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
  int32_t chunk_features;  // features per CTA (grid.y chunks), a multiple of 8
  int32_t two;             // the constant 2, passed at run time (see eytz_level)
  int32_t swizzle;         // tiled: odd feature rows XOR object byte offsets with 64 (K2s layout)
  int64_t ld;              // feature-major: row pitch in objects (>= n; a batch may be a column range)
  // tiled output in two regions: objects >= split (a multiple of 128) go to out2 in tiles
  // of tile2 with swizzle2 (the tail-wave region of predict_impl); split = n_slots if none
  int64_t split;
  uint8_t* out2;
  int32_t tile2, swizzle2;
  // K1L cell tables (used borders): luts [F][256] cell -> lower-bound bucket, recs [F]
  // of {lo, hi, s, o, borders[P] (+inf padded)} with stride lrec_stride bytes
  const uint8_t* lut;
  const unsigned char* lrec;
  int32_t lrec_stride;
  int32_t chunk_inner;  // grid order: feature chunk fastest (1) or row block fastest (0)
  int32_t row_blocks;   // K1L: consecutive 1024-row blocks per CTA (the chunk's tables staged once)
};

constexpr int kQuantObjects = 128;    // tile quantum: a quantize warp's 128 objects never straddle tiles
constexpr int kQuantThreads = 256;    // 8 warps x 128 objects = 1024 objects per CTA
constexpr int kQuantBlock = 1024;
constexpr int kQuantSmem = 48 * 1024; // Eytzinger arrays of one feature chunk

// Features per CTA chunk (grid.y): as many whole quads as fit kQuantSmem.
__host__ __device__ constexpr int quantize_chunk_features(int eytz_pitch, int n_features) {
  return eytz_pitch <= 0 ? ((n_features + 7) / 8 * 8)
         : (kQuantSmem / (eytz_pitch * 4) / 8 * 8 > 0 ? kQuantSmem / (eytz_pitch * 4) / 8 * 8 : 8);
}

// One level of the branchless Eytzinger walk, on byte offsets o = 4i into the shared
// array: i' = 2i + 1 + [x > e_i]  <=>  o' = two * o + (x > e_i ? 8 : 4).  `two` is the
// runtime value 2 (a kernel parameter) so the update is an IMAD on the FMA pipe; plain
// C++ (no asm) lets the compiler interleave the independent searches of a lane.
// NaN compares false and walks left, giving bucket 0 (quantize.py:171).
// The condition is applied as a predicated add written in PTX: ptxas then emits FSETP +
// a predicated IADD that it can place on the FMA pipe (IMAD.IADD), instead of FSETP +
// SEL, both on the ALU pipe that bounds this kernel (measured on B200).
__device__ __forceinline__ uint32_t add_if_greater(uint32_t r, float x, float b, uint32_t inc) {
  asm("{\n .reg .pred p;\n setp.gt.f32 p, %1, %2;\n @p add.u32 %0, %0, %3;\n}" : "+r"(r) : "f"(x), "f"(b), "r"(inc));
  return r;
}

__device__ __forceinline__ uint32_t eytz_level(uint32_t o, float x, const float* e, uint32_t two) {
  const float b = *reinterpret_cast<const float*>(reinterpret_cast<const unsigned char*>(e) + o);
  const uint32_t four = two + two;  // runtime 4: the adds stay IMAD-able
  return add_if_greater(o * two + four, x, b, four);
}

// Store the packed buckets of one feature for a lane's 4 objects (base + lane + 32k):
// tiled -> word `lane` of the 128-object block's row, plain -> 4 bytes of row f.
template <bool TILED>
__device__ __forceinline__ void store_bucket_word(const QuantizeParams& p, uint32_t word, int f, int64_t base, int lane,
                                                  bool full_objs) {
  const int64_t ob = base + lane;
  if (!full_objs) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (ob + 32 * k >= p.n) word &= ~(0xFFu << (8 * k));  // padding objects are zero (quantize.py:172)
  }
  if (TILED) {
    const bool second = base >= p.split;  // warp-uniform: blocks never straddle the split
    const int64_t rb = second ? base - p.split : base;
    const int64_t tl = second ? p.tile2 : p.tile;
    const bool sw = (second ? p.swizzle2 : p.swizzle) && (f & 1);
    const int64_t t = rb / tl, w = (rb - t * tl + 4 * lane) ^ (sw ? 64 : 0);
    uint32_t* dst = reinterpret_cast<uint32_t*>((second ? p.out2 : p.out) + (t * p.n_features + f) * tl + w);
    *dst = word;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (ob + 32 * k < p.n) p.out[(int64_t)f * p.n + ob + 32 * k] = (uint8_t)(word >> (8 * k));
  }
}

constexpr int kQuantStep = 8;  // features per step: one 32-byte sector per row

// The searches of one step (8 features x the lane's 4 objects) and its 8 packed
// bucket-word stores.  Lane objects are base + lane + 32k (the tile layout's word `lane`
// of the 128-object block at `base`); ey holds the feature chunk's Eytzinger arrays.
template <int L, bool TILED>
__device__ __forceinline__ void quantize_step(const QuantizeParams& p, const float* ey, const float (&v)[kQuantStep][4],
                                              int f0, int fq, int nf, int64_t base, int lane, bool full_objs) {
  constexpr int kE = (1 << L) - 1;
  constexpr int S = kQuantStep;
  const uint32_t two = (uint32_t)p.two;
  // 2^30, 2^6, 2^14, 2^22 from the run-time 2 (kept as IMAD multipliers, not shifts)
  const uint32_t m6 = two << 5, m14 = two << 13, m22 = two << 21, m30 = two << 29;
  const int F = p.n_features;
  const int64_t ob = base + lane;
  uint32_t o[S][4];
#pragma unroll
  for (int j = 0; j < S; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) o[j][k] = 0;
  // the top levels from registers: the feature's top nodes are loaded once (broadcast
  // loads) and serve the lane's 4 objects, so each value makes L - kTop dependent
  // shared-memory lookups instead of L.  Measured on B200 (cfg2, cfg4): kTop = 2 beats
  // 3 (more selects on the ALU pipe), 1 and 0 (more lookups)
#ifndef OBT_QUANT_TOP
#define OBT_QUANT_TOP 2
#endif
  constexpr int kTop = (OBT_QUANT_TOP == 3 && L >= 4) ? 3 : (OBT_QUANT_TOP == 2 && L >= 3) ? 2
                       : (OBT_QUANT_TOP == 1 && L >= 2) ? 1 : 0;
  if constexpr (kTop == 1) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const float n0 = ey[min(fq + j, nf - 1) * kE];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[j][k] = v[j][k] > n0 ? 8u : 4u;  // position 1 + c0 (x4)
    }
  }
  if constexpr (kTop == 2) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const float* e = ey + min(fq + j, nf - 1) * kE;
      const float n0 = e[0], n1 = e[1], n2 = e[2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = v[j][k];
        const bool c0 = x > n0;
        // Eytzinger position after two levels: 3 + 2 c0 + c1 (byte offset x4)
        const uint32_t o1 = add_if_greater(12u, x, n0, 8u);
        o[j][k] = add_if_greater(o1, x, c0 ? n2 : n1, 4u);
      }
    }
  }
  if constexpr (kTop == 3) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const float* e = ey + min(fq + j, nf - 1) * kE;
      float n[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) n[i] = e[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = v[j][k];
        const bool c0 = x > n[0];
        const bool c1 = x > (c0 ? n[2] : n[1]);
        const float b2 = c0 ? (c1 ? n[6] : n[5]) : (c1 ? n[4] : n[3]);
        const bool c2 = x > b2;
        // Eytzinger position after three levels: 7 + 4 c0 + 2 c1 + c2 (byte offset x4)
        o[j][k] = 28u + (c0 ? 16u : 0u) + (c1 ? 8u : 0u) + (c2 ? 4u : 0u);
      }
    }
  }
#pragma unroll
  for (int l = kTop; l < L; ++l)
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const float* e = ey + min(fq + j, nf - 1) * kE;
#pragma unroll
      for (int k = 0; k < 4; ++k) o[j][k] = eytz_level(o[j][k], v[j][k], e, two);
    }
#pragma unroll
  for (int j = 0; j < S; ++j) {
    if (fq + j >= nf) break;
    // bucket k = o_k / 4 - E in byte k (padding objects are zero, quantize.py:172):
    // word = (o0 >> 2) + 64 o1 + 2^14 o2 + 2^22 o3 - E * 0x01010101, as IMAD.HI + IMADs with
    // run-time multipliers, so the packing runs on the FMA pipe rather than the ALU pipe
    uint32_t word = __umulhi(o[j][0], m30) - (uint32_t)kE * 0x01010101u;
    word = o[j][1] * m6 + word;
    word = o[j][2] * m14 + word;
    word = o[j][3] * m22 + word;
    store_bucket_word<TILED>(p, word, f0 + fq + j, base, lane, full_objs);
  }
}

// One CTA: 1024 objects (8 warps x 32 lanes x 4 objects) x one chunk of features
// (grid.y).  The chunk's Eytzinger arrays are staged in shared memory once; each lane
// then walks its 4 objects (rows one apart from its neighbours') x 8 features per step:
// a 32-byte sector per row straight from HBM, 32 independent searches, 8 packed 32-bit
// bucket stores (each warp writes 128 contiguous bytes of a feature row of the tile).
// The fallback for inputs the TMA-staged kernel (K1t) does not take, and the plain
// [F][n] output of obt_quantize_dev.
template <int KMAX, int CELLS>
__device__ __forceinline__ void lut_step(const QuantizeParams& p, uint32_t luts_s, const unsigned char* recs,
                                         uint32_t recs_s, const float (&v)[kQuantStep][4], int f0, int fq, int nf,
                                         int64_t base, int lane, bool full_objs);
// LUT_CELLS > 0: the cell-table search (K1L's, tiled output only) with L = KMAX compares;
// the shared memory then holds the chunk's cell tables instead of Eytzinger arrays.
template <int L, int LAYOUT, bool TILED, int LUT_CELLS = 0>
__global__ void __launch_bounds__(kQuantThreads, 2) quantize_kernel(QuantizeParams p) {
  extern __shared__ __align__(16) unsigned char qsm[];
  constexpr int kE = LUT_CELLS ? 0 : (1 << L) - 1;
  constexpr int S = kQuantStep;
  float* ey = reinterpret_cast<float*>(qsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.n_features;
  const int fc = p.chunk_features;
  // grid.x = row blocks x feature chunks.  chunk_inner: the chunk varies fastest, so the
  // chunks of one row block run side by side and the L2 lines their row segments share
  // are read from HBM once (K1L at cfg2: 1.08 -> 0.96 GB, 0.217 -> 0.198 ms); otherwise
  // the row block varies fastest (the Eytzinger kernels measured 1-4% faster that way)
  const int n_fch = (p.n_features + fc - 1) / fc;
  const unsigned n_rb = gridDim.x / (unsigned)n_fch;
  const int f0 = (int)(p.chunk_inner ? blockIdx.x % (unsigned)n_fch : blockIdx.x / n_rb) * fc;
  const int64_t rblock = (int64_t)(p.chunk_inner ? blockIdx.x / (unsigned)n_fch : blockIdx.x % n_rb);
  const int nf = min(fc, F - f0);
  if (kE > 0) {
    const float* src = p.eytz + (int64_t)f0 * kE;
    for (int i = threadIdx.x; i < nf * kE; i += kQuantThreads) ey[i] = __ldg(src + i);
  }
  // cell tables: luts 256-aligned (the PRMT address trick), recs right behind them
  unsigned char* luts = qsm + ((256u - (smem_u32(qsm) & 255u)) & 255u);
  unsigned char* recs = luts + (size_t)nf * (LUT_CELLS ? LUT_CELLS : 1);
  if constexpr (LUT_CELLS > 0) {
    const uint4* src = reinterpret_cast<const uint4*>(p.lut + (size_t)f0 * LUT_CELLS);
    uint4* dst = reinterpret_cast<uint4*>(luts);
    for (int i = threadIdx.x; i < nf * LUT_CELLS / 16; i += kQuantThreads) dst[i] = __ldg(src + i);
    const uint4* rsrc = reinterpret_cast<const uint4*>(p.lrec + (size_t)f0 * p.lrec_stride);
    uint4* rdst = reinterpret_cast<uint4*>(recs);
    for (int i = threadIdx.x; i < nf * p.lrec_stride / 16; i += kQuantThreads) rdst[i] = __ldg(rsrc + i);
  }
  __syncthreads();

  // this lane's objects: base + lane + 32k (the tile layout's word `lane` of this block)
  const int64_t base = rblock * kQuantBlock + warp * 128;
  if (base >= p.n_slots) return;  // past the last tile (no barrier follows)
  const int64_t ob = base + lane;
  const bool full_objs = ob + 96 < p.n;
  const bool vec_rows =
      LAYOUT == 0 ? ((F & 3) == 0 && (f0 & 3) == 0 && (reinterpret_cast<uintptr_t>(p.x) & 15) == 0) : true;
  static_assert(kQuantStep == 8, "a 256-bit row load covers exactly one step");
  const bool sector_rows = LAYOUT == 0 && (F & 7) == 0 && (reinterpret_cast<uintptr_t>(p.x) & 31) == 0;
  const uint32_t two = (uint32_t)p.two;
  // raw values v[j][k] of one step: object ob + 32k, feature f0 + fq + j
  auto load_step = [&](float (&v)[S][4], int fq) {
    if (full_objs && vec_rows && fq + S <= nf) {
      if (LAYOUT == 0 && sector_rows) {
        // one 256-bit load per row: the lane takes a whole 32-byte sector at once (two
        // 128-bit loads per sector measured 43% excess L2 sectors: the second half
        // often missed L1 again)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float* row = p.x + (ob + 32 * k) * F + f0 + fq;
          asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=f"(v[0][k]), "=f"(v[1][k]), "=f"(v[2][k]), "=f"(v[3][k]),
                         "=f"(v[4][k]), "=f"(v[5][k]), "=f"(v[6][k]), "=f"(v[7][k])
                       : "l"(row));
        }
      } else if (LAYOUT == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4* row = reinterpret_cast<const float4*>(p.x + (ob + 32 * k) * F + f0 + fq);
#pragma unroll
          for (int h = 0; h < S / 4; ++h) {
            const float4 q = __ldg(row + h);
            v[4 * h + 0][k] = q.x; v[4 * h + 1][k] = q.y; v[4 * h + 2][k] = q.z; v[4 * h + 3][k] = q.w;
          }
        }
      } else {
        // feature-major: each load is one row segment shared by the warp's 32 lanes
#pragma unroll
        for (int j = 0; j < S; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) v[j][k] = __ldg(p.x + (int64_t)(f0 + fq + j) * p.ld + ob + 32 * k);
      }
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = ob + 32 * k < p.n && fq + j < nf;
          const int64_t idx = LAYOUT == 0 ? (ob + 32 * k) * F + f0 + fq + j : (int64_t)(f0 + fq + j) * p.ld + ob + 32 * k;
          v[j][k] = in ? __ldg(p.x + idx) : 0.0f;
        }
    }
  };

  // the 32 searches of one step and its 8 packed bucket-word stores

  for (int fq = 0; fq < nf; fq += S) {
    float v[S][4];
    load_step(v, fq);
    if constexpr (LUT_CELLS > 0) {
      static_assert(TILED, "cell tables cover the used borders: tiled output only");
      lut_step<L, LUT_CELLS>(p, smem_u32(luts), recs, smem_u32(recs), v, f0, fq, nf, base, lane, full_objs);
    } else {
      quantize_step<L, TILED>(p, ey, v, f0, fq, nf, base, lane, full_objs);
    }
  }
}

// ---------------------------------------------------------------------------
// K1t: TMA-staged quantize (object-major input, tiled output; F % 4 == 0, 16-byte
// aligned features).  A producer warp streams the CTA's 1024 feature rows, 8 features
// (one 32-byte sector) per row per step, with four 2-D tensor copies per stage
// (box 8 features x 256 rows, 32-byte swizzle) into a 2-stage ring; the 8 consumer
// warps read their rows back with two conflict-free LDS.128 each (rows l + 32k of a
// quarter-warp are 8 consecutive rows, and the swizzle spreads their 16-byte halves
// over all 8 bank quads), release the stage, and run the same searches and stores as
// K1.  The rows never occupy registers while in flight, and the TMA requests are whole
// sectors, so the consumer warps wait on shared memory instead of HBM.
constexpr int kQTConsumerWarps = kQuantBlock / 128;                  // 8
constexpr int kQTThreads = 32 * (1 + kQTConsumerWarps);              // producer + consumers
constexpr int kQTStages = 2;
constexpr int kQTBoxRows = 256;
constexpr int kQTStageBytes = kQuantBlock * kQuantStep * 4;          // 32 KB
constexpr int kQTSmemFixed = 1024 + kQTStages * kQTStageBytes + 64;  // alignment + ring + barriers

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}


template <int L>
__global__ void __launch_bounds__(kQTThreads, 2) quantize_tma_kernel(const __grid_constant__ CUtensorMap rows,
                                                                     const QuantizeParams p) {
  extern __shared__ __align__(16) unsigned char qt_raw[];
  unsigned char* ring = qt_raw + ((1024u - (smem_u32(qt_raw) & 1023u)) & 1023u);  // swizzle atoms need alignment
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kQTStages * kQTStageBytes);
  uint64_t* empty = full + kQTStages;
  float* ey = reinterpret_cast<float*>(empty + kQTStages);
  constexpr int kE = (1 << L) - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fc = p.chunk_features;
  // grid.x = row blocks x feature chunks.  chunk_inner: the chunk varies fastest, so the
  // chunks of one row block run side by side and the L2 lines their row segments share
  // are read from HBM once (K1L at cfg2: 1.08 -> 0.96 GB, 0.217 -> 0.198 ms); otherwise
  // the row block varies fastest (the Eytzinger kernels measured 1-4% faster that way)
  const int n_fch = (p.n_features + fc - 1) / fc;
  const unsigned n_rb = gridDim.x / (unsigned)n_fch;
  const int f0 = (int)(p.chunk_inner ? blockIdx.x % (unsigned)n_fch : blockIdx.x / n_rb) * fc;
  const int64_t rblock = (int64_t)(p.chunk_inner ? blockIdx.x / (unsigned)n_fch : blockIdx.x % n_rb);
  const int nf = min(fc, p.n_features - f0);
  const int n_steps = (nf + kQuantStep - 1) / kQuantStep;
  const int64_t row0 = rblock * kQuantBlock;
  // consumer warps whose 128-object block lies inside the grid's slots
  const int64_t blocks_left = (p.n_slots - row0 + 127) / 128;
  const int active = blocks_left < kQTConsumerWarps ? (int)blocks_left : kQTConsumerWarps;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQTStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32 * active);  // every active consumer thread releases its reads
    }
    fence_mbar_init();
  }
  if (kE > 0) {
    const float* src = p.eytz + (int64_t)f0 * kE;
    for (int i = threadIdx.x; i < nf * kE; i += kQTThreads) ey[i] = __ldg(src + i);
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      for (int st = 0; st < n_steps; ++st) {
        const int s = st % kQTStages;
        if (st >= kQTStages) mbar_wait(&empty[s], (uint32_t)(st / kQTStages - 1) & 1u);
        mbar_expect_tx(&full[s], kQTStageBytes);  // out-of-range rows/features arrive zero-filled
        unsigned char* dst = ring + (size_t)s * kQTStageBytes;
#pragma unroll
        for (int b = 0; b < kQuantBlock / kQTBoxRows; ++b)
          tma_load_2d(dst + b * kQTBoxRows * kQuantStep * 4, &rows, f0 + st * kQuantStep,
                      (int)(row0 + b * kQTBoxRows), &full[s]);
      }
    }
    return;
  }
  const int cw = warp - 1;
  if (cw >= active) return;
  const int64_t base = row0 + cw * 128;
  const bool full_objs = base + lane + 96 < p.n;
  for (int st = 0; st < n_steps; ++st) {
    const int s = st % kQTStages;
    mbar_wait_warp(&full[s], (uint32_t)(st / kQTStages) & 1u);
    const unsigned char* stage = ring + (size_t)s * kQTStageBytes;
    float v[kQuantStep][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // row r = 128 cw + lane + 32k: 32 bytes at 32 r, 16-byte halves swapped when bit 2 of r is set
      const int r = cw * 128 + lane + 32 * k;
      const unsigned char* rp = stage + 32 * r;
      const uint32_t sw = (uint32_t)((r >> 2) & 1) * 16u;
      const float4 a = *reinterpret_cast<const float4*>(rp + sw);
      const float4 b = *reinterpret_cast<const float4*>(rp + (16u ^ sw));
      v[0][k] = a.x; v[1][k] = a.y; v[2][k] = a.z; v[3][k] = a.w;
      v[4][k] = b.x; v[5][k] = b.y; v[6][k] = b.z; v[7][k] = b.w;
    }
    mbar_release(&empty[s]);  // the rows were requested: the producer may refill the stage once they are read
    quantize_step<L, true>(p, ey, v, f0, st * kQuantStep, nf, base, lane, full_objs);
  }
}

// ---------------------------------------------------------------------------
// K1L: cell-table quantize (TMA-staged rows as K1t, used borders only).  Per feature f
// the host chooses an affine map y = fma(clamp(x, lo_f, hi_f), s_f, o_f) whose results
// lie in [1.5 * 2^23, 1.5 * 2^23 + 255]: the low byte of y's bits is a cell c, monotone in
// x (clamp and a correctly rounded fma with s_f >= 0 are monotone; NaN clamps to lo_f).
// With c_k the cell of border k, lut_f[c] = #{k : c_k < c} and every border k with
// c_k < c is below any x of cell c, every border with c_k > c is >= it; so the bucket
// #{k : x > b_k} is lut_f[c] plus the count over the at most KMAX borders of cell c,
// which KMAX compares against the sorted, +inf-padded borders finish (a compare past
// the cell's borders is false).  The host evaluates the same fp32 ops (fmaf is correctly
// rounded in both places), so buckets are bit-exact.  Per value: 2 FMNMX, FFMA, PRMT,
// one byte load, KMAX x (address, load, compare-add) -- about a third of the Eytzinger
// search's instructions, with fewer dependent shared loads.
constexpr int kLutCells = 256;       // cells per feature table (1024 where 256 leave crowded cells)
constexpr int kLutRecHeader = 16;  // lo, hi, s, o

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// The cell-table searches of one step (8 features x a lane's 4 objects) and its 8 packed
// bucket-word stores (tiled output); luts / recs hold the chunk's tables in shared memory.
template <int KMAX, int CELLS>
__device__ __forceinline__ void lut_step(const QuantizeParams& p, uint32_t luts_s, const unsigned char* recs,
                                         uint32_t recs_s, const float (&v)[kQuantStep][4], int f0, int fq, int nf,
                                         int64_t base, int lane, bool full_objs) {
  const int rs = p.lrec_stride;
  uint32_t bk[kQuantStep][4];
#pragma unroll
  for (int j = 0; j < kQuantStep; ++j) {
    const int fl = min(fq + j, nf - 1);
    const float4 h = *reinterpret_cast<const float4*>(recs + (size_t)fl * rs);  // lo, hi, s, o (broadcast)
    const uint32_t lut_base = luts_s + (uint32_t)fl * CELLS;
    const uint32_t bord = recs_s + (uint32_t)fl * rs + kLutRecHeader;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x = v[j][k];
      const float y = __fmaf_rn(fminf(fmaxf(x, h.x), h.y), h.z, h.w);
      // 256 cells: the cell byte drops into byte 0 of the 256-aligned table address (PRMT);
      // 1024 cells: the low 10 bits of y's bits index the table
      const uint32_t cell_addr = CELLS == 256 ? __byte_perm(__float_as_uint(y), lut_base, 0x7650u)
                                              : lut_base + (__float_as_uint(y) & (uint32_t)(CELLS - 1));
      uint32_t b = lds_u8(cell_addr);
#pragma unroll
      for (int i = 0; i < KMAX; ++i) b = add_if_greater(b, x, lds_f32(bord + 4u * b), 1u);
      bk[j][k] = b;
    }
  }
#pragma unroll
  for (int j = 0; j < kQuantStep; ++j) {
    if (fq + j >= nf) break;
    uint32_t word = bk[j][3] * 256u + bk[j][2];
    word = word * 256u + bk[j][1];
    word = word * 256u + bk[j][0];
    store_bucket_word<true>(p, word, f0 + fq + j, base, lane, full_objs);
  }
}
template <int KMAX, int CELLS>
__global__ void __launch_bounds__(kQTThreads, 2) quantize_lut_kernel(const __grid_constant__ CUtensorMap rows,
                                                                     const QuantizeParams p) {
  extern __shared__ __align__(16) unsigned char qt_raw[];
  unsigned char* ring = qt_raw + ((1024u - (smem_u32(qt_raw) & 1023u)) & 1023u);  // swizzle atoms need alignment
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kQTStages * kQTStageBytes);
  uint64_t* empty = full + kQTStages;
  unsigned char* luts = reinterpret_cast<unsigned char*>(empty + kQTStages) + 32;  // 256-aligned below
  luts += (256u - (smem_u32(luts) & 255u)) & 255u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fc = p.chunk_features;
  // grid.x = row-block groups x feature chunks.  chunk_inner: the chunk varies fastest, so
  // the chunks of one row block run side by side and the L2 lines their row segments
  // share are read from HBM once (K1L at cfg2: 1.08 -> 0.96 GB, 0.217 -> 0.198 ms);
  // otherwise the row block varies fastest (the Eytzinger kernels measured 1-4% faster
  // that way).  A CTA quantizes row_blocks consecutive 1024-row blocks of its chunk, so
  // the chunk's tables (config 4: 32 features x 1.5 KB, as many bytes as 1.5 row blocks
  // of the chunk's features) are staged once per row_blocks blocks.
  const int n_fch = (p.n_features + fc - 1) / fc;
  const unsigned n_rg = gridDim.x / (unsigned)n_fch;
  const int f0 = (int)(p.chunk_inner ? blockIdx.x % (unsigned)n_fch : blockIdx.x / n_rg) * fc;
  const int64_t rgroup = (int64_t)(p.chunk_inner ? blockIdx.x / (unsigned)n_fch : blockIdx.x % n_rg);
  const int nf = min(fc, p.n_features - f0);
  unsigned char* recs = luts + (size_t)nf * CELLS;  // this chunk's nf features (the host sizes min(fc, F))
  const int rs = p.lrec_stride;
  const int n_steps = (nf + kQuantStep - 1) / kQuantStep;
  const int64_t row_first = rgroup * p.row_blocks * kQuantBlock;
  const int64_t rows_left = p.n_slots - row_first;
  const int64_t rb_left = (rows_left + kQuantBlock - 1) / kQuantBlock;
  const int n_rb = rb_left < p.row_blocks ? (int)rb_left : p.row_blocks;
  const int total = n_rb * n_steps;  // pipeline steps: row block r, feature step st
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQTStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32 * kQTConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int it) {  // producer: row stage `it` (row block it / n_steps, step it % n_steps)
    const int s = it % kQTStages;
    const int rb = it / n_steps, st = it - rb * n_steps;
    const int64_t row0 = row_first + (int64_t)rb * kQuantBlock;
    if (it >= kQTStages) mbar_wait(&empty[s], (uint32_t)(it / kQTStages - 1) & 1u);
    mbar_expect_tx(&full[s], kQTStageBytes);
    unsigned char* dst = ring + (size_t)s * kQTStageBytes;
#pragma unroll
    for (int b = 0; b < kQuantBlock / kQTBoxRows; ++b)
      tma_load_2d(dst + b * kQTBoxRows * kQuantStep * 4, &rows, f0 + st * kQuantStep, (int)(row0 + b * kQTBoxRows),
                  &full[s]);
  };
  // the first row stages land while every thread copies the chunk's tables (cfg4 K1L
  // 4.81 -> 4.57 ms; plain coalesced loads: two bulk copies measured slower, cfg2 0.215
  // vs 0.200 ms)
  const int head = total < kQTStages ? total : kQTStages;
  if (threadIdx.x == 0)
    for (int it = 0; it < head; ++it) issue(it);
  {
    const uint4* src = reinterpret_cast<const uint4*>(p.lut + (size_t)f0 * CELLS);
    uint4* dst = reinterpret_cast<uint4*>(luts);
    for (int i = threadIdx.x; i < nf * CELLS / 16; i += kQTThreads) dst[i] = __ldg(src + i);
    const uint4* rsrc = reinterpret_cast<const uint4*>(p.lrec + (size_t)f0 * rs);
    uint4* rdst = reinterpret_cast<uint4*>(recs);
    for (int i = threadIdx.x; i < nf * rs / 16; i += kQTThreads) rdst[i] = __ldg(rsrc + i);
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0)
      for (int it = head; it < total; ++it) issue(it);
    return;
  }
  const int cw = warp - 1;
  const uint32_t luts_s = smem_u32(luts), recs_s = smem_u32(recs);
  int s = 0;
  uint32_t phase = 0;
  for (int rb = 0; rb < n_rb; ++rb) {
    const int64_t base = row_first + (int64_t)rb * kQuantBlock + cw * 128;
    const bool live = base < p.n_slots;  // warp-uniform: rows past the grid's slots are skipped
    const bool full_objs = base + lane + 96 < p.n;
    for (int st = 0; st < n_steps; ++st) {
      mbar_wait_warp(&full[s], phase);
      const unsigned char* stage = ring + (size_t)s * kQTStageBytes;
      float v[kQuantStep][4];
      if (live) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = cw * 128 + lane + 32 * k;
          const unsigned char* rp = stage + 32 * r;
          const uint32_t sw = (uint32_t)((r >> 2) & 1) * 16u;
          const float4 a = *reinterpret_cast<const float4*>(rp + sw);
          const float4 b = *reinterpret_cast<const float4*>(rp + (16u ^ sw));
          v[0][k] = a.x; v[1][k] = a.y; v[2][k] = a.z; v[3][k] = a.w;
          v[4][k] = b.x; v[5][k] = b.y; v[6][k] = b.z; v[7][k] = b.w;
        }
      }
      mbar_release(&empty[s]);
      if (++s == kQTStages) { s = 0; phase ^= 1u; }
      if (live) lut_step<KMAX, CELLS>(p, luts_s, recs, recs_s, v, f0, st * kQuantStep, nf, base, lane, full_objs);
    }
  }
}

// ---------------------------------------------------------------------------
// K2: tree apply.
//
// A split descriptor is one 32-bit word (off << 8) | k (plus, in 8-bit mode, a second
// word s): off = byte offset of the feature's row in the bucket tile, and adding k
// replicated to the 4 bytes of a bucket word carries [q > ordinal] into bit 7 of each:
//   7-bit mode (all buckets <= 127): k = 127 - ordinal;                  sentinel k = 0
//   8-bit mode: k = 127 - (ordinal & 127), s = all-ones iff ordinal < 128;
//               condition = bit7(((q & 127) + k) | q) if ordinal < 128
//                         = bit7(((q & 127) + k) & q) otherwise;          sentinel k = s = 0
// Descriptors come either from the kernel-parameter bank (DSRC 1: uniform loads, no
// shared-memory traffic; a launch covers as many trees as the 32 KB parameter space
// holds and the next launch continues the same fold from the carried accumulators),
// or from the shared-memory ring next to the leaves (DSRC 0, any model size).
// Trees are processed in groups of 4 whose descriptors are contiguous (LDS.128 in
// DSRC 0); the tree count is padded to a multiple of 4 with null trees whose splits
// are sentinels and whose leaves are -0.0, and x + (-0.0) == x exactly for every x,
// so padding never changes a bit of the fold.
// 16 trees per group keep ~100 independent shared loads in flight per thread; deeper
// trees (larger leaf tables) use groups of 8 / 4 so a chunk still fits the ring without
// shrinking the bucket tile.
#ifndef OBT_GROUP_SHALLOW
#define OBT_GROUP_SHALLOW 32
#endif
#ifndef OBT_GROUP_D8
#define OBT_GROUP_D8 32
#endif
__host__ __device__ constexpr int tree_group(int di) { return di <= 6 ? OBT_GROUP_SHALLOW : di <= 8 ? OBT_GROUP_D8 : 4; }
#ifndef OBT_DESC_PAIR_LOADS
#define OBT_DESC_PAIR_LOADS 1  // parameter-bank descriptors: two splits per 128-bit uniform load
#endif
#ifndef OBT_PF_TREES
#define OBT_PF_TREES 2         // apply pipeline: bucket words requested this many trees ahead
#endif
#ifndef OBT_FOLD_LAG
#define OBT_FOLD_LAG 1         // apply pipeline: leaves folded this many trees after their request
#endif
// Shared-memory descriptor words per split: 7-bit compare {off, k replicated}, 8-bit
// {(off << 8) | k, s}.
__host__ __device__ constexpr int desc_words(int) { return 2; }
__host__ __device__ constexpr int desc_words_per_tree(int di, int cmp) { return di * desc_words(cmp); }

struct ApplyParams {
  const uint8_t* q;          // tiled buckets [n_tiles][F][tile]
  const uint8_t* chunks;     // [n_chunks][chunk_bytes] descriptor+leaf records
  double* out;               // [n] predictions; also the fold carry between launches
  uint16_t* idx_out;         // [tree_end - tree_begin][n] (index mode)
  int64_t n;
  int32_t tile;
  int32_t chunk_trees;
  int32_t chunk_begin, chunk_end;  // chunks (of chunk_trees trees) this launch folds
  uint32_t chunk_bytes;      // multiple of 256
  uint32_t desc_bytes;       // descriptor part of a record (multiple of 256)
  uint32_t q_tile_bytes;     // F * tile
  int32_t n_stages;
  int32_t tree_begin, tree_end;  // index mode: trees written
  int32_t first, last;       // start the fold at 0 / finalize into predictions
  // tile order and next-wave L2 prefetch: CTA b takes tile (reverse ? grid - 1 - b : b)
  // and, when l2_wave > 0, prefetches into L2 the bucket tile of CTA b + l2_wave (the
  // next wave's), so that wave's tile loads hit L2 instead of waiting on HBM
  int32_t reverse, l2_wave;
  // launch chaining (programmatic dependent launch): a CTA waits until tile_flags[tile]
  // >= flag_wait before reading the fold carry, and after its outputs stores flag_set
  // (0: neither); launches chained this way let the next launch fill the SMs the
  // previous one's partial last wave leaves idle
  uint32_t* tile_flags;
  int32_t flag_wait, flag_set;
  double scale, bias;
};

constexpr int kParamDescWords = 8144;  // 32576 bytes of descriptors + ApplyParams (128) <= 32764

template <int DSRC> struct ApplyArgs;
template <> struct ApplyArgs<0> { ApplyParams p; };
template <> struct ApplyArgs<1> { ApplyParams p; uint32_t desc[kParamDescWords]; };
static_assert(sizeof(ApplyArgs<1>) <= 32764, "kernel parameter space");

template <int LEAF> struct LeafT;
template <> struct LeafT<0> { using T = double; using Acc = double; static constexpr int kShift = 3;
  static __device__ __forceinline__ double widen(double v) { return v; } };
template <> struct LeafT<1> { using T = float; using Acc = double; static constexpr int kShift = 2;
  static __device__ __forceinline__ double widen(float v) { return (double)v; } };
template <> struct LeafT<2> { using T = __half; using Acc = float; static constexpr int kShift = 1;
  static __device__ __forceinline__ float widen(__half v) { return __half2float(v); } };
// Register/shuffle "permute" leaf selection (K2 only; PERMUTE16 / PERMUTE64 of the
// reference, accumulate.py:116-159, section 8.2-8.3): a tree's whole table, 128
// bytes, sits one word per lane, and a lane takes its objects' leaves with SHFL.
//   3: binary16 leaves, depth <= 6 (two leaves per word)   4: binary32 leaves, depth <= 5
template <> struct LeafT<3> : LeafT<2> {};
template <> struct LeafT<4> : LeafT<1> {};

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (a & c) | (b & c);
}

#ifndef OBT_FADD2
#define OBT_FADD2 1  // binary16 family: fold two objects per packed FADD2
#endif
// a += x, b += y as one packed f32x2 add (sm_100)
__device__ __forceinline__ void fadd2(float& a, float& b, float x, float y) {
  unsigned long long r, p, q;
  asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(x), "f"(y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(q));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
template <typename T>
__device__ __forceinline__ void fadd2(T&, T&, T, T) {}  // other accumulator types never reach it

// Byte k (runtime-unrolled constant) of a packed index word, zero-extended.
__device__ __forceinline__ uint32_t byte_of_rt(uint32_t w, int k) { return (w >> (8 * k)) & 0xffu; }

// Byte k of a packed index word, zero-extended (one PRMT).
template <int K>
__device__ __forceinline__ uint32_t byte_of(uint32_t w) {
  return __byte_perm(w, 0u, 0x4440u | K);
}


// Shared loads by 32-bit address.  VOL selects PTX-volatile loads, which ptxas keeps in
// program order: K2's software pipeline then decides how far ahead each load is issued
// (left to itself ptxas hoisted K2's bucket loads ~6 trees ahead and spilled).  The
// other kernels keep plain loads (volatile ones made K2s spill).
#ifndef OBT_LDS_VOLATILE
#define OBT_LDS_VOLATILE 1
#endif
#define OBT_LDS_SEL(VOL) ((VOL) && OBT_LDS_VOLATILE)

template <bool VOL = false>
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  if constexpr (OBT_LDS_SEL(VOL)) asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  else asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// W consecutive bucket words (4W objects) of one feature row.
template <int W, bool VOL = false>
__device__ __forceinline__ void lds_words(uint32_t addr, uint32_t (&w)[W]) {
  if constexpr (W == 1) {
    w[0] = lds_u32<VOL>(addr);
  } else if constexpr (W == 2) {
    if constexpr (OBT_LDS_SEL(VOL)) asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
    else asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
  } else {
    static_assert(W == 4, "1, 2 or 4 bucket words per thread");
    if constexpr (OBT_LDS_SEL(VOL))
      asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr));
    else
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr));
  }
}

// Leaf loads.
template <int LEAF, bool VOL = false>
__device__ __forceinline__ typename LeafT<LEAF>::T lds_leaf(uint32_t addr) {
  if constexpr (LEAF == 0) {
    double v;
    if constexpr (OBT_LDS_SEL(VOL)) asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    else asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
  } else if constexpr (LEAF == 1) {
    float v;
    if constexpr (OBT_LDS_SEL(VOL)) asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    else asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
  } else {
    unsigned short v;
    if constexpr (OBT_LDS_SEL(VOL)) asm volatile("ld.volatile.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    else asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return __ushort_as_half(v);
  }
}

// Leaf-table stride in a stage: prescaled tables sit on 256-byte boundaries so the
// gather address is one PRMT: (index byte) into byte 0 of the table's base address.
__host__ __device__ constexpr int leaf_table_stride(int di, int leaf_bytes) {
  return (1 << di) * leaf_bytes <= 256 ? 256 : (1 << di) * leaf_bytes;
}

constexpr int kApplyProducerThreads = 32;
// Block size cap: 128 registers per thread keep several tree groups of loads in flight.
#ifndef OBT_APPLY_MAXT
#define OBT_APPLY_MAXT 544
#endif
constexpr int kApplyMaxThreads = OBT_APPLY_MAXT;  // 16 consumer warps + the producer

template <int DI, int CMP, int LEAF, bool WRITE_IDX, int W, int DSRC>
__global__ void __launch_bounds__(kApplyMaxThreads, 1) apply_kernel(const __grid_constant__ ApplyArgs<DSRC> args) {
  const ApplyParams& p = args.p;
  // index dumps and 8-object threads keep more live values per tree: smaller unrolled
  // groups (chunks hold multiples of tree_group(DI), so any divisor tiles them)
  constexpr int kTreeGroup = (WRITE_IDX || W == 2) ? (tree_group(DI) < 8 ? tree_group(DI) : 8) : tree_group(DI);
  using LT = LeafT<LEAF>;
  using acc_t = typename LT::Acc;
  constexpr int kDW = desc_words(CMP);
  constexpr int kTabStride = leaf_table_stride(DI, (int)sizeof(typename LT::T));
  // When the scaled index still fits a byte, the SWAR words carry byte offsets
  // (index << kShift) directly and a gather is PRMT + LDS.
  constexpr bool kPrescaled = !WRITE_IDX && (DI + LT::kShift) <= 8;
  constexpr int kBitBase = kPrescaled ? LT::kShift : 0;
  constexpr bool kPermute = LEAF >= 3;
  constexpr bool kHalfFold = LEAF == 2 || LEAF == 3;
  static_assert(!kPermute || (kPrescaled && W == 1 && (1 << DI) * (int)sizeof(typename LT::T) <= 128),
                "permute selection: one 128-byte table per warp");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 256-byte aligned working base (the host reserves 256 bytes of slack)
  unsigned char* smem = smem_raw + ((256u - (smem_u32(smem_raw) & 255u)) & 255u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);    // [S]   stage landed
  uint64_t* empty = full + 8;                            // [S]   stage consumed
  uint64_t* tile_bar = full + 16;
  unsigned char* stages = smem + 256;
  unsigned char* qtile = stages + (size_t)p.n_stages * p.chunk_bytes;

  const int tid = threadIdx.x;
  const int n_consumer_warps = (blockDim.x - kApplyProducerThreads) / 32;
  const int64_t tile_idx = p.reverse ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int n_chunks = p.chunk_end - p.chunk_begin;
  if (p.flag_set > 0) launch_dependents();
  if (tid == 0) {
    for (int i = 0; i < p.n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], n_consumer_warps * 32);  // every consumer thread arrives
    }
    mbar_init(tile_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  // warp index broadcast from lane 0: provably warp-uniform, so the role split below is
  // a uniform branch and the consumer loop counters can live in uniform registers
  const int warp_id = __shfl_sync(0xffffffffu, tid / 32, 0);
  if (warp_id == 0) {
    // producer warp: the bucket tile once, then the leaf (+descriptor) ring
    if (tid == 0) {
      mbar_expect_tx(tile_bar, p.q_tile_bytes);
      bulk_g2s_split(qtile, p.q + tile_idx * (int64_t)p.q_tile_bytes, p.q_tile_bytes, tile_bar);
      if (p.l2_wave > 0 && (blockIdx.x + (unsigned)p.l2_wave < gridDim.x || p.flag_set > 0)) {
        // the next wave's tile; in the last wave of a chained launch, wrap to the first
        // wave's tiles (the next launch starts there, same order)
        const unsigned nb = (blockIdx.x + (unsigned)p.l2_wave) % gridDim.x;
        const int64_t nt = p.reverse ? (int64_t)(gridDim.x - 1 - nb) : (int64_t)nb;
        bulk_prefetch_l2(p.q + nt * (int64_t)p.q_tile_bytes, p.q_tile_bytes);
      }
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % p.n_stages;
        if (c >= p.n_stages) mbar_wait(&empty[s], (uint32_t)(c / p.n_stages - 1) & 1u);
        mbar_expect_tx(&full[s], p.chunk_bytes);
        bulk_g2s_split(stages + (size_t)s * p.chunk_bytes,
                       p.chunks + (size_t)(p.chunk_begin + c) * p.chunk_bytes, p.chunk_bytes, &full[s]);
      }
    }
    return;
  }

  const int ctid = tid - kApplyProducerThreads;
  constexpr int kObj = 4 * W;                            // objects per thread
  const uint32_t my_q = smem_u32(qtile) + kObj * ctid;   // this thread's words in every row
  const int64_t tile_base = tile_idx * p.tile;
  // accumulator 4x + k: byte k of this thread's word x
  auto obj_of = [&](int x, int k) { return word_object(tile_base, W * ctid + x, k); };
  acc_t acc[kObj];
  if (p.flag_wait > 0) {
    // the previous launch of this fold may still run (chained launch): its CTA for this
    // tile publishes the carry with a release store
    if (ctid == 0) wait_flag(p.tile_flags + tile_idx, (uint32_t)p.flag_wait);
    consumer_sync(n_consumer_warps * 32);
  }
#pragma unroll
  for (int k = 0; k < kObj; ++k) {
    // continue the fold of the previous launch (exact: the carry holds acc_t values)
    const int64_t o = obj_of(k / 4, k % 4);
    acc[k] = (p.first || WRITE_IDX || o >= p.n) ? (acc_t)0 : (acc_t)p.out[o];
  }
  mbar_wait_warp(tile_bar, 0);

  for (int c = 0; c < n_chunks; ++c) {
    const int s = c % p.n_stages;
    mbar_wait_warp(&full[s], (uint32_t)(c / p.n_stages) & 1u);
    const unsigned char* st = stages + (size_t)s * p.chunk_bytes;
    const uint32_t leaf_base = smem_u32(st + p.desc_bytes);
    const int t_base = (p.chunk_begin + c) * p.chunk_trees;
    for (int g = 0; g < p.chunk_trees / kTreeGroup; ++g) {
      uint32_t dw[DSRC == 0 ? kTreeGroup * DI * kDW : 1];
      if constexpr (DSRC == 0) {
        const uint4* dsrc = reinterpret_cast<const uint4*>(st + (size_t)g * kTreeGroup * DI * kDW * 4);
#pragma unroll
        for (int v = 0; v < kTreeGroup * DI * kDW / 4; ++v) {
          const uint4 q4 = dsrc[v];
          dw[4 * v + 0] = q4.x; dw[4 * v + 1] = q4.y; dw[4 * v + 2] = q4.z; dw[4 * v + 3] = q4.w;
        }
      }
      // parameter-bank descriptors of this group: {off, k replicated} word pairs (LDC.64
      // broadcasts from the constant bank, no shared-memory wavefronts; a packed 4-byte
      // form measured slower: its unpack runs on the vector ALU)
      const int gbase = (c * (p.chunk_trees / kTreeGroup) + g) * (kTreeGroup * DI * 2);
      // Software pipeline over the group's trees (all indices compile-time after
      // unrolling): iteration i requests the bucket words of tree i (stage A), builds the
      // index of tree i - kPF and requests its leaves (stage B), and folds the leaves of
      // tree i - kPF - 1 (stage C).  Each load's consumer thus sits about one tree of
      // instructions after it in issue order, and folds stay in tree order.
      constexpr int kPF = OBT_PF_TREES;
      uint32_t wbuf[kPF + 1][DI][W];  // bucket words of the trees in flight
      uint32_t kbuf[kPF + 1][DI];     // DSRC 1: k replicated per depth
      uint32_t twbuf[kPF + 1];         // permute: this lane's word of the tree's table
      (void)twbuf;
      constexpr int kLag = OBT_FOLD_LAG;
      typename LT::T gbuf[kLag + 1][4 * W];  // gathered leaves awaiting their fold
      (void)kbuf; (void)gbuf;
#pragma unroll
      for (int it = 0; it < kTreeGroup + kPF + kLag; ++it) {
        if (it < kTreeGroup) {  // stage A: bucket words of tree `it`
          const int tt = it, sl = it % (kPF + 1);
          uint32_t pend_off = 0, pend_k = 0;  // second split of a 128-bit descriptor pair
          (void)pend_off; (void)pend_k;
#pragma unroll
          for (int d = 0; d < DI; ++d) {
            if constexpr (DSRC == 1) {
              static_assert(CMP == 7 && W == 1, "parameter-bank descriptors: 7-bit compare, 4 objects per thread");
              // two splits per 128-bit load where the pair is 16-byte aligned (gbase is a
              // multiple of 4 words, so the parity of tt * DI + d decides at compile time);
              // ptxas splits it into two uniform LDCU.64 either way
              const int sidx = tt * DI + d;
              uint32_t off, krep;
              if (OBT_DESC_PAIR_LOADS && (sidx & 1) == 0 && d + 1 < DI) {
                const uint4 pr = *reinterpret_cast<const uint4*>(&args.desc[gbase + 2 * sidx]);
                off = pr.x; krep = pr.y; pend_off = pr.z; pend_k = pr.w;
              } else if (OBT_DESC_PAIR_LOADS && d > 0 && ((sidx - 1) & 1) == 0) {
                off = pend_off; krep = pend_k;
              } else {
                off = args.desc[gbase + 2 * sidx];
                krep = args.desc[gbase + 2 * sidx + 1];
              }
              wbuf[sl][d][0] = lds_u32<true>(my_q + off);
              kbuf[sl][d] = krep;
            } else {
              const uint32_t d0 = dw[(tt * DI + d) * kDW];
              lds_words<W, true>(my_q + (CMP == 7 ? d0 : (d0 >> 8)), wbuf[sl][d]);
            }
          }
          if constexpr (kPermute)  // one conflict-free word per lane: the table in registers
            twbuf[sl] = lds_u32<true>(leaf_base + (uint32_t)(g * kTreeGroup + tt) * 256u + 4u * (ctid & 31));
        }
        if (it >= kPF && it - kPF < kTreeGroup) {  // stage B: index + leaf requests of tree ti
          const int ti = it - kPF, sl = ti % (kPF + 1);
          const int t = g * kTreeGroup + ti;
          uint32_t lo_acc[W], hi[W];
#pragma unroll
          for (int x = 0; x < W; ++x) { lo_acc[x] = 0; hi[x] = 0; }
#pragma unroll
          for (int d = 0; d < DI; ++d) {
            uint32_t b7s[W];  // [q > ordinal] in bit 7 of each byte, garbage below
            if constexpr (DSRC == 1) {
              b7s[0] = wbuf[sl][d][0] + kbuf[sl][d];
            } else {
              // shared-memory descriptors: 7-bit {off, k replicated}; 8-bit {(off << 8) | k, s}
              const uint32_t d0 = dw[(ti * DI + d) * kDW], d1 = dw[(ti * DI + d) * kDW + 1];
              if constexpr (CMP == 7) {
#pragma unroll
                for (int x = 0; x < W; ++x) b7s[x] = wbuf[sl][d][x] + d1;
              } else {
                const uint32_t k = __byte_perm(d0, 0u, 0x0000u) & 0x7f7f7f7fu;
#pragma unroll
                for (int x = 0; x < W; ++x) {
                  const uint32_t wv = wbuf[sl][d][x];
                  b7s[x] = maj3((wv & 0x7f7f7f7fu) + k, wv, d1);
                }
              }
            }
#pragma unroll
            for (int x = 0; x < W; ++x) {
              const uint32_t b7 = b7s[x];
              const int pos = d + kBitBase;  // target bit of condition d inside each byte
              if (pos < 8) {
                const uint32_t term = (pos == 7 ? b7 : (b7 >> (7 - pos))) & (0x01010101u << pos);
                // one OR chain: each depth is one LOP3 (mask | acc) after its shift
                lo_acc[x] |= term;
              } else {
                hi[x] |= (pos == 15 ? b7 : (b7 >> (15 - pos))) & (0x01010101u << (pos - 8));
              }
            }
          }
#pragma unroll
          for (int x = 0; x < W; ++x) {
            const uint32_t lo = lo_acc[x];
            if constexpr (WRITE_IDX) {
              const int tg = t_base + t;
              if (tg >= p.tree_begin && tg < p.tree_end) {
                uint16_t* row = p.idx_out + (int64_t)(tg - p.tree_begin) * p.n;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint32_t idx = ((lo >> (8 * k)) & 0xffu) | (DI > 8 ? ((hi[x] >> (8 * k)) & 0xffu) << 8 : 0u);
                  const int64_t o = obj_of(x, k);
                  if (o < p.n) row[o] = (uint16_t)idx;
                }
              }
            } else if constexpr (kPermute) {
              // leaf of byte offset `off`: word off / 4 of the table, from lane off / 4;
              // binary16: the half (off / 2) & 1 of that word
              typename LT::T* gv = gbuf[ti % (kLag + 1)] + 4 * x;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t off = (lo >> (8 * k)) & 0xffu;
                const uint32_t v = __shfl_sync(0xffffffffu, twbuf[sl], (int)(off >> 2));
                if constexpr (LEAF == 3) {
                  gv[k] = __ushort_as_half((unsigned short)__byte_perm(v, 0u, (off & 2u) ? 0x3232u : 0x1010u));
                } else {
                  gv[k] = __uint_as_float(v);
                }
              }
            } else if constexpr (kPrescaled) {
              const uint32_t tab = leaf_base + (uint32_t)t * 256u;
              typename LT::T* gv = gbuf[ti % (kLag + 1)] + 4 * x;
              gv[0] = lds_leaf<LEAF, true>(__byte_perm(lo, tab, 0x7650u));
              gv[1] = lds_leaf<LEAF, true>(__byte_perm(lo, tab, 0x7651u));
              gv[2] = lds_leaf<LEAF, true>(__byte_perm(lo, tab, 0x7652u));
              gv[3] = lds_leaf<LEAF, true>(__byte_perm(lo, tab, 0x7653u));
            } else {
              const uint32_t tab = leaf_base + (uint32_t)t * kTabStride;
              uint32_t ix[4];
              ix[0] = byte_of<0>(lo); ix[1] = byte_of<1>(lo); ix[2] = byte_of<2>(lo); ix[3] = byte_of<3>(lo);
              if constexpr (DI > 8) {
                ix[0] |= byte_of<0>(hi[x]) << 8; ix[1] |= byte_of<1>(hi[x]) << 8;
                ix[2] |= byte_of<2>(hi[x]) << 8; ix[3] |= byte_of<3>(hi[x]) << 8;
              }
              typename LT::T* gv = gbuf[ti % (kLag + 1)] + 4 * x;
#pragma unroll
              for (int k = 0; k < 4; ++k) gv[k] = lds_leaf<LEAF, true>(tab + (ix[k] << LT::kShift));
            }
          }
        }
        if constexpr (!WRITE_IDX) {
          if (it >= kPF + kLag && it - kPF - kLag < kTreeGroup) {  // stage C: fold tree tf (tree order per object)
            const int tf = it - kPF - kLag;
#pragma unroll
            for (int k = 0; k < 4 * W; k += 2) {
              if constexpr (kHalfFold && OBT_FADD2) {
                // binary32 fold of two objects in one packed FADD2 (two independent
                // round-to-nearest adds: the same bits as two FADDs)
                fadd2(acc[k], acc[k + 1], LT::widen(gbuf[tf % (kLag + 1)][k]), LT::widen(gbuf[tf % (kLag + 1)][k + 1]));
              } else {
                acc[k] += LT::widen(gbuf[tf % (kLag + 1)][k]);
                acc[k + 1] += LT::widen(gbuf[tf % (kLag + 1)][k + 1]);
              }
            }
          }
        }
      }
    }
    mbar_release(&empty[s]);  // this thread is done reading stage s (no divergent branch)
  }

  if constexpr (!WRITE_IDX) {
#pragma unroll
    for (int k = 0; k < kObj; ++k) {
      const int64_t o = obj_of(k / 4, k % 4);
      if (o < p.n) {
        // finalize: f64(acc) * scale + bias, two roundings (evaluate.py:298-299, oracle.py:53-54)
        p.out[o] = p.last ? __dadd_rn(__dmul_rn((double)acc[k], p.scale), p.bias) : (double)acc[k];
      }
    }
    if (p.flag_set > 0) {
      consumer_sync(n_consumer_warps * 32);
      if (ctid == 0) {
        __threadfence();
        st_release_gpu(p.tile_flags + tile_idx, (uint32_t)p.flag_set);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2f: fanned-out apply for small batches.  K2 walks every tree of the model in order
// inside one CTA per tile, so a batch of a few thousand objects runs on a few SMs with
// one to three warps each (config 1: 79 CTAs of 128 objects, 18.5 us for 500 trees).
// Here a CTA owns one 128-object block and 16 warps: 12 compute warps split each chunk's
// trees among themselves (tree t of the chunk -> warp t mod 12; lane = 4 objects as in
// K2) and write the gathered leaves to a shared value panel [tree][object]; 4 fold warps
// (one object per thread) then add the panel's rows in tree order -- the binary64 (or
// binary32) fold is still the reference's left fold, only the index and gather work is
// spread.  Chunk records (descriptors + tables, the K2 shared-memory format for a
// 128-object tile) stream through an S-stage TMA ring (as many stages as fit, up to 8:
// a chunk's compute is short next to its load latency); the value panel is double buffered.
constexpr int kFanComputeWarps = 12;
constexpr int kFanFoldWarps = 4;
constexpr int kFanThreads = 32 * (kFanComputeWarps + kFanFoldWarps);

template <int DI, int CMP, int LEAF>
__global__ void __launch_bounds__(kFanThreads, 1) apply_fan_kernel(const __grid_constant__ ApplyParams p) {
  using LT = LeafT<LEAF>;
  using leaf_t = typename LT::T;
  using acc_t = typename LT::Acc;
  constexpr int kDW = desc_words(CMP);
  constexpr int kTabStride = leaf_table_stride(DI, (int)sizeof(leaf_t));
  extern __shared__ __align__(128) unsigned char fan_raw[];
  unsigned char* smem = fan_raw + ((256u - (smem_u32(fan_raw) & 255u)) & 255u);
  const int S = p.n_stages;                            // chunk-record ring depth (<= 8)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [S] chunk record landed
  uint64_t* sfree = full + 8;                          // [S] chunk record consumed (compute warps)
  uint64_t* vfull = full + 16;                         // [2] value panel written (compute warps)
  uint64_t* vfree = full + 18;                         // [2] value panel folded (fold warps)
  uint64_t* tile_bar = full + 20;
  unsigned char* stages = smem + 256;
  const int ct = p.chunk_trees;
  leaf_t* panel = reinterpret_cast<leaf_t*>(stages + (size_t)S * p.chunk_bytes);  // [2][ct][128]
  unsigned char* qtile = reinterpret_cast<unsigned char*>(panel + 2 * (size_t)ct * 128);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_chunks = p.chunk_end - p.chunk_begin;
  const int64_t blk = (int64_t)blockIdx.x * 128;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], 32 * kFanComputeWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&vfull[i], 32 * kFanComputeWarps);
      mbar_init(&vfree[i], 32 * kFanFoldWarps);
    }
    mbar_init(tile_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < kFanFoldWarps) {
    // fold warps: thread j folds object blk + j (word j & 31, byte j >> 5) in tree order
    const int j = tid;
    const int64_t o = blk + j;
    acc_t acc = (p.first || o >= p.n) ? (acc_t)0 : (acc_t)p.out[o];
    for (int c = 0; c < n_chunks; ++c) {
      const int v = c & 1;
      mbar_wait_warp(&vfull[v], (uint32_t)(c >> 1) & 1u);
      const leaf_t* row = panel + (size_t)v * ct * 128 + j;
      // eight loads (and widenings) ahead of their adds: only the add chain is serial
      int t = 0;
      for (; t + 8 <= ct; t += 8) {
        acc_t w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = LT::widen(row[(size_t)(t + u) * 128]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += w[u];
      }
      for (; t < ct; ++t) acc += LT::widen(row[(size_t)t * 128]);
      mbar_arrive(&vfree[v]);
    }
    if (o < p.n) p.out[o] = p.last ? __dadd_rn(__dmul_rn((double)acc, p.scale), p.bias) : (double)acc;
    return;
  }
  // compute warps
  const int cw = warp - kFanFoldWarps;
  if (cw == 0 && lane == 0) {
    mbar_expect_tx(tile_bar, p.q_tile_bytes);
    bulk_g2s_split(qtile, p.q + (int64_t)blockIdx.x * p.q_tile_bytes, p.q_tile_bytes, tile_bar);
    for (int c = 0; c < S && c < n_chunks; ++c) {
      mbar_expect_tx(&full[c], p.chunk_bytes);
      bulk_g2s_split(stages + (size_t)c * p.chunk_bytes, p.chunks + (size_t)(p.chunk_begin + c) * p.chunk_bytes,
                     p.chunk_bytes, &full[c]);
    }
  }
  const uint32_t my_q = smem_u32(qtile) + 4 * lane;
  mbar_wait_warp(tile_bar, 0);
  for (int c = 0; c < n_chunks; ++c) {
    const int s = c % S, v = c & 1;
    mbar_wait_warp(&full[s], (uint32_t)(c / S) & 1u);
    if (c >= 2) mbar_wait_warp(&vfree[v], (uint32_t)((c >> 1) - 1) & 1u);
    const unsigned char* st = stages + (size_t)s * p.chunk_bytes;
    const uint32_t* dw = reinterpret_cast<const uint32_t*>(st);
    const uint32_t leaf_base = smem_u32(st + p.desc_bytes);
    leaf_t* prow = panel + (size_t)v * ct * 128;
#pragma unroll 4
    for (int t = cw; t < ct; t += kFanComputeWarps) {
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int d = 0; d < DI; ++d) {
        const uint32_t d0 = dw[(t * DI + d) * kDW], d1 = dw[(t * DI + d) * kDW + 1];
        uint32_t b7;
        if constexpr (CMP == 7) {
          b7 = lds_u32(my_q + d0) + d1;
        } else {
          const uint32_t w = lds_u32(my_q + (d0 >> 8));
          b7 = maj3((w & 0x7f7f7f7fu) + (__byte_perm(d0, 0u, 0x0000u) & 0x7f7f7f7fu), w, d1);
        }
        if (d < 8) lo |= (b7 >> (7 - d)) & (0x01010101u << d);
        else hi |= (b7 >> (15 - d)) & (0x01010101u << (d - 8));
      }
      const uint32_t tab = leaf_base + (uint32_t)t * kTabStride;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t idx = byte_of_rt(lo, k) | (DI > 8 ? byte_of_rt(hi, k) << 8 : 0u);
        prow[(size_t)t * 128 + lane + 32 * k] = lds_leaf<LEAF>(tab + (idx << LT::kShift));
      }
    }
    mbar_release(&sfree[s]);
    mbar_arrive(&vfull[v]);
    // refill stage s with chunk c + S once every compute thread has read it
    if (cw == 0 && lane == 0 && c + S < n_chunks) {
      mbar_wait(&sfree[s], (uint32_t)(c / S) & 1u);
      mbar_expect_tx(&full[s], p.chunk_bytes);
      bulk_g2s_split(stages + (size_t)s * p.chunk_bytes, p.chunks + (size_t)(p.chunk_begin + c + S) * p.chunk_bytes,
                     p.chunk_bytes, &full[s]);
    }
  }
}

// ---------------------------------------------------------------------------
// K2s: depth-split tree apply.  TPW adjacent lanes share one 4-object bucket word:
// lane part p evaluates depths [p*DI/TPW, (p+1)*DI/TPW) of every tree, the partial
// index words are OR-combined with butterfly shuffles, and lane p then gathers and
// folds objects [p*4/TPW, (p+1)*4/TPW) of the word.  Every accumulator still sees
// the trees in order (the fold stays bit-exact) while the CTA runs TPW times more
// warps over the same bucket tile -- the lever against the latency bound when the
// tile (F bytes per object) limits the objects an SM can hold.
//
// Bank conflicts: the TPW lanes of a word read different feature rows at the same word
// offset, and rows start on 128-byte boundaries, so without care they hit the same bank.
// The K2s bucket layout therefore XORs the object byte offset of odd feature rows with
// 64 (the quantize kernel writes it so): a warp's 16 words (TPW 2) then sit in one bank
// half for even rows and in the other for odd rows, and the host orders each tree's
// levels so the two lanes of a pair read rows of opposite parity wherever the tree
// allows (the leaf table is permuted to match; the selected leaf is unchanged).
// Descriptors come from the shared-memory ring as 16 bytes per split, stored half-major:
// per tree DI entries {off+, k} then DI entries {off-, k} (7-bit; 8-bit: {(off << 8) | k, s}),
// off+- = row offset +- 64 for odd rows; a lane takes the half that matches bit 6 of its
// own word offset (warp-uniform), so the swizzle costs no instruction.
constexpr int kSplitDescBytes = 16;
template <int DI, int CMP, int LEAF, int TPW>
__global__ void __launch_bounds__(kApplyMaxThreads, 1) apply_split_kernel(const __grid_constant__ ApplyArgs<0> args) {
  static_assert(DI <= 8 && DI % TPW == 0, "depth-split needs TPW | DI and one index byte");
  const ApplyParams& p = args.p;
  using LT = LeafT<LEAF>;
  using acc_t = typename LT::Acc;
  constexpr int kTreeGroup = tree_group(DI);
  constexpr int kDPT = DI / TPW;        // depths per lane
  constexpr int kOPT = 4 / TPW;         // objects folded per lane
  constexpr bool kPrescaled = (DI + LT::kShift) <= 8;
  constexpr int kBitBase = kPrescaled ? LT::kShift : 0;
  constexpr int kTabStride = leaf_table_stride(DI, (int)sizeof(typename LT::T));

  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((256u - (smem_u32(smem_raw) & 255u)) & 255u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  uint64_t* tile_bar = full + 16;
  unsigned char* stages = smem + 256;
  unsigned char* qtile = stages + (size_t)p.n_stages * p.chunk_bytes;

  const int tid = threadIdx.x;
  const int n_consumers = blockDim.x - kApplyProducerThreads;
  const int64_t tile_idx = p.reverse ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int n_chunks = p.chunk_end - p.chunk_begin;
  if (tid == 0) {
    for (int i = 0; i < p.n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], n_consumers);
    }
    mbar_init(tile_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int warp_id = __shfl_sync(0xffffffffu, tid / 32, 0);
  if (warp_id == 0) {
    if (tid == 0) {
      mbar_expect_tx(tile_bar, p.q_tile_bytes);
      bulk_g2s_split(qtile, p.q + tile_idx * (int64_t)p.q_tile_bytes, p.q_tile_bytes, tile_bar);
      if (p.l2_wave > 0 && blockIdx.x + (unsigned)p.l2_wave < gridDim.x) {
        const unsigned nb = blockIdx.x + (unsigned)p.l2_wave;
        const int64_t nt = p.reverse ? (int64_t)(gridDim.x - 1 - nb) : (int64_t)nb;
        bulk_prefetch_l2(p.q + nt * (int64_t)p.q_tile_bytes, p.q_tile_bytes);
      }
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % p.n_stages;
        if (c >= p.n_stages) mbar_wait(&empty[s], (uint32_t)(c / p.n_stages - 1) & 1u);
        mbar_expect_tx(&full[s], p.chunk_bytes);
        bulk_g2s_split(stages + (size_t)s * p.chunk_bytes,
                       p.chunks + (size_t)(p.chunk_begin + c) * p.chunk_bytes, p.chunk_bytes, &full[s]);
      }
    }
    return;
  }

  const int ctid = tid - kApplyProducerThreads;
  const int word = ctid / TPW, part = ctid % TPW;
  const uint32_t my_q = smem_u32(qtile) + 4 * word;
  const int64_t tile_base = tile_idx * p.tile;
  auto obj_of = [&](int k) { return word_object(tile_base, word, part * kOPT + k); };  // k < kOPT
  // per-lane constants: the index bits this lane owns and the bytes it gathers
  uint32_t shift[kDPT], mask[kDPT];
#pragma unroll
  for (int i = 0; i < kDPT; ++i) {
    const int pos = part * kDPT + i + kBitBase;
    shift[i] = 7u - (uint32_t)pos;
    mask[i] = 0x01010101u << pos;
  }
  uint32_t sel[kOPT];
#pragma unroll
  for (int k = 0; k < kOPT; ++k) sel[k] = kPrescaled ? (0x7650u | (uint32_t)(part * kOPT + k)) : (0x4440u | (uint32_t)(part * kOPT + k));
  acc_t acc[kOPT];
#pragma unroll
  for (int k = 0; k < kOPT; ++k) acc[k] = (p.first || obj_of(k) >= p.n) ? (acc_t)0 : (acc_t)p.out[obj_of(k)];
  mbar_wait_warp(tile_bar, 0);

  // this lane's first descriptor in a tree: records are half-major, 8-byte {off, k}
  // entries [half][level], so a lane's kDPT levels are contiguous (two per 128-bit load
  // when kDPT is even: half the descriptor loads, and their wavefronts)
  const uint32_t my_desc = ((((4u * word) >> 6) & 1u) * (uint32_t)DI + (uint32_t)(part * kDPT)) * 8u;
  constexpr bool kPairDesc = (kDPT % 2) == 0;
  for (int c = 0; c < n_chunks; ++c) {
    const int s = c % p.n_stages;
    mbar_wait_warp(&full[s], (uint32_t)(c / p.n_stages) & 1u);
    const unsigned char* st = stages + (size_t)s * p.chunk_bytes;
    const uint32_t leaf_base = smem_u32(st + p.desc_bytes);
    const uint32_t desc_base = smem_u32(st) + my_desc;
    for (int g = 0; g < p.chunk_trees / kTreeGroup; ++g) {
#pragma unroll
      for (int tt = 0; tt < kTreeGroup; ++tt) {
        const int t = g * kTreeGroup + tt;
        const uint32_t tree_desc = desc_base + (uint32_t)t * (uint32_t)(DI * kSplitDescBytes);
        uint32_t part_a = 0, part_b = 0;
        uint32_t dsc[kDPT][2];
#pragma unroll
        for (int i = 0; i < kDPT; i += (kPairDesc ? 2 : 1)) {
          if constexpr (kPairDesc) {
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(dsc[i][0]), "=r"(dsc[i][1]), "=r"(dsc[i + 1][0]), "=r"(dsc[i + 1][1])
                         : "r"(tree_desc + 8u * i));
          } else {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(dsc[i][0]), "=r"(dsc[i][1]) : "r"(tree_desc + 8u * i));
          }
        }
#pragma unroll
        for (int i = 0; i < kDPT; ++i) {
          const uint32_t d0 = dsc[i][0], d1 = dsc[i][1];
          uint32_t b7;
          if constexpr (CMP == 7) {
            b7 = lds_u32(my_q + d0) + d1;
          } else {
            const uint32_t w = lds_u32(my_q + (d0 >> 8));
            b7 = maj3((w & 0x7f7f7f7fu) + (__byte_perm(d0, 0u, 0x0000u) & 0x7f7f7f7fu), w, d1);
          }
          const uint32_t term = (b7 >> shift[i]) & mask[i];
          if (i & 1) part_b |= term; else part_a |= term;
        }
        uint32_t lo = part_a | part_b;
        if constexpr (TPW >= 2) lo |= __shfl_xor_sync(0xffffffffu, lo, 1);
        if constexpr (TPW >= 4) lo |= __shfl_xor_sync(0xffffffffu, lo, 2);
        const uint32_t tab = leaf_base + (uint32_t)t * kTabStride;
#pragma unroll
        for (int k = 0; k < kOPT; ++k) {
          uint32_t addr;
          if constexpr (kPrescaled) addr = __byte_perm(lo, tab, sel[k]);
          else addr = tab + (__byte_perm(lo, 0u, sel[k]) << LT::kShift);
          acc[k] += LT::widen(lds_leaf<LEAF>(addr));
        }
      }
    }
    mbar_release(&empty[s]);
  }
#pragma unroll
  for (int k = 0; k < kOPT; ++k) {
    if (obj_of(k) < p.n) p.out[obj_of(k)] = p.last ? __dadd_rn(__dmul_rn((double)acc[k], p.scale), p.bias) : (double)acc[k];
  }
}

// ---------------------------------------------------------------------------
// K4: multi-output apply (C > 1 outputs per leaf; BASELINE config 5: C = 10, depth 10).
// A leaf record is C values (40 bytes at C = 10, fp32), so per-tile staging of leaf
// tables (40 KB per tree) cannot amortise; instead the tables stay in global memory and
// every CTA walks the trees in the same order, so the active window of tables stays
// L2-resident (with tree sharding across GPUs each GPU's tables fit L2 outright).
// No shared memory: many CTAs per SM hide the L2 latency.  Each thread owns 4 objects
// (one SWAR bucket word read from the tile-blocked matrix through L1), builds their
// leaf indices exactly as K2, then gathers each object's C-value record and folds every
// output in tree order in binary64.
struct MultiParams {
  const uint8_t* q;        // tiled buckets [n_tiles][F][tile]
  const uint32_t* desc;    // [T_pad][DI][2] {off = f * tile, k replicated} (7-bit) or {(off<<8)|k, s}
  const void* leaves;      // [T_pad][2^DI][CP] fp32 or fp64
  double* out;             // [n][C] predictions / fold carry
  int64_t n;
  int32_t n_features, tile, n_outputs;
  int32_t tree_begin, tree_end;  // trees folded by this launch
  int32_t first, last;
  double scale, bias;
};

#ifndef OBT_MULTI_OPL
#define OBT_MULTI_OPL 4
#endif
// Objects folded per lane: a bucket word's 4 objects are shared by 4 / kMultiOPL lanes
// (each evaluates the word's indices and folds its share), trading duplicate index
// work for fewer fp64 accumulators per thread and more resident warps.
constexpr int kMultiOPL = OBT_MULTI_OPL;
constexpr int kMultiLanesPerWord = 4 / kMultiOPL;
constexpr int kMultiTileObjects = 512;                    // one tile per CTA: 128 bucket words
constexpr int kMultiThreads = kMultiTileObjects / 4 * kMultiLanesPerWord;

// Values per multi-output leaf record: fp32 records in 16-byte rows (48 bytes at C = 10;
// 32-byte rows with 256-bit loads measured slower), fp64 records in 16-byte rows.
// Measured and dropped for K4: bucket words requested one tree ahead (590 against 565 ms
// at config 5 -- the held words cost more than the overlap), L2 prefetch of the bucket
// rows 4-16 trees ahead (no gain).
__host__ __device__ constexpr int multi_record_values(int leaf, int c) {
  return leaf == 1 ? (c + 3) / 4 * 4 : (c + 1) / 2 * 2;
}

#ifndef OBT_MULTI_MINB
// 4 resident CTAs per SM (a 128-register cap) up to C = 10: uncapped, ptxas took 196
// registers and config 5 ran at 767 ms instead of 565 ms (2 CTAs, half the record
// loads in flight).  More outputs need the accumulator registers (fewer CTAs).
#define OBT_MULTI_MINB 4
#endif
__host__ __device__ constexpr int multi_min_blocks(int leaf, int c) {
  return leaf == 0 ? (c <= 5 ? OBT_MULTI_MINB : 2) : (c <= 10 ? OBT_MULTI_MINB : c <= 12 ? 3 : 2);
}
template <int DI, int CMP, int LEAF, int C>
__global__ void __launch_bounds__(kMultiThreads, multi_min_blocks(LEAF, C)) apply_multi_kernel(const __grid_constant__ MultiParams p) {
  using leaf_t = typename LeafT<LEAF>::T;
  constexpr int CP = multi_record_values(LEAF, C);  // record stride: 32-byte rows (fp32), 16-byte (fp64)
  constexpr int OPL = kMultiOPL;
  const int word = threadIdx.x / kMultiLanesPerWord, sub = threadIdx.x % kMultiLanesPerWord;
  // persistent CTAs (grid = resident CTAs): every CTA starts its next tile when the
  // previous one ends, so all CTAs walk the trees nearly in step and the active window of
  // leaf records stays L2-resident (one launch of 31250 CTAs kept CTAs at every tree
  // position at once: all 4000 trees' records, 197 MB, competed for L2 at config 5)
  const int64_t n_tiles = (p.n + p.tile - 1) / p.tile;
  for (int64_t tile_idx = blockIdx.x; tile_idx < n_tiles; tile_idx += gridDim.x) {
    const uint8_t* qrow0 = p.q + tile_idx * (int64_t)p.n_features * p.tile + 4 * word;
    const int64_t tile_base = tile_idx * p.tile;
    auto obj_of = [&](int k) { return word_object(tile_base, word, sub * OPL + k); };  // k < OPL
    double acc[OPL][C];
#pragma unroll
    for (int k = 0; k < OPL; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c)
        acc[k][c] = (p.first || obj_of(k) >= p.n) ? 0.0 : p.out[obj_of(k) * C + c];
    for (int t = p.tree_begin; t < p.tree_end; ++t) {
      uint32_t wcur[DI];
      uint2 dcur[DI];
      const uint2* ds = reinterpret_cast<const uint2*>(p.desc) + (size_t)t * DI;
#pragma unroll
      for (int d = 0; d < DI; ++d) {
        dcur[d] = __ldg(ds + d);  // warp-uniform address: one broadcast
        wcur[d] = __ldg(reinterpret_cast<const uint32_t*>(qrow0 + (CMP == 7 ? dcur[d].x : (dcur[d].x >> 8))));
      }
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int d = 0; d < DI; ++d) {
        const uint2 dd = dcur[d];
        const uint32_t w = wcur[d];
        uint32_t b7;
        if constexpr (CMP == 7) {
          b7 = w + dd.y;
        } else {
          b7 = maj3((w & 0x7f7f7f7fu) + (__byte_perm(dd.x, 0u, 0x0000u) & 0x7f7f7f7fu), w, dd.y);
        }
        if (d < 8) lo |= (b7 >> (7 - d)) & (0x01010101u << d);
        else hi |= (b7 >> (15 - d)) & (0x01010101u << (d - 8));
      }
      const leaf_t* tab = reinterpret_cast<const leaf_t*>(p.leaves) + ((size_t)t << DI) * CP;
      // all 4 objects' records are requested before any is consumed: the L2 round trips
      // overlap (each record is CP values in 16-byte rows)
      {
        constexpr int kRows = CP * (int)sizeof(leaf_t) / 16;
        uint4 rec[OPL][kRows];
#pragma unroll
        for (int k = 0; k < OPL; ++k) {
          const int kb = sub * OPL + k;  // byte of the word
          const uint32_t idx = ((lo >> (8 * kb)) & 0xffu) | (DI > 8 ? ((hi >> (8 * kb)) & 0xffu) << 8 : 0u);
          const uint4* r = reinterpret_cast<const uint4*>(tab + (size_t)idx * CP);
#pragma unroll
          for (int i = 0; i < kRows; ++i) rec[k][i] = __ldg(r + i);
        }
#pragma unroll
        for (int k = 0; k < OPL; ++k) {
          const leaf_t* v = reinterpret_cast<const leaf_t*>(rec[k]);
#pragma unroll
          for (int c = 0; c < C; ++c) acc[k][c] += (double)v[c];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < OPL; ++k) {
      if (obj_of(k) >= p.n) continue;
#pragma unroll
      for (int c = 0; c < C; ++c)
        p.out[obj_of(k) * C + c] = p.last ? __dadd_rn(__dmul_rn((double)acc[k][c], p.scale), p.bias) : (double)acc[k][c];
    }
  }
}

// ---------------------------------------------------------------------------
// K5: staged multi-output apply (fp32 records).  K4 gathers records from L2 and is bound
// by the round trips each SM keeps in flight.  Here one CTA owns a 2048-object tile (16
// consumer warps, 4 objects per lane, C binary64 accumulators per object in registers)
// and a producer warp streams, per tree, the tree's whole record table (2^D x CP fp32,
// 48 KB at config 5) plus the tile's D bucket rows that tree reads (D x 2048 bytes) into
// an S-stage ring with bulk TMA copies.  Consumers read bucket words and records from
// shared memory only: one table load serves 2048 objects (24 B of L2 traffic per
// object-tree instead of a 48-byte record fetch), and every load the fold waits on is a
// shared-memory load.  Descriptors come from the K4 array ({f * 512, k} / {(f*512) << 8 | k, s}).
// K5 record: one leaf's C values.  Binary64 family: binary32 values in 16-byte rows (C
// rounded up to 4; a 48-byte record at C = 10 puts row r of record i in 16-byte bank
// group (3i + r) mod 8, all eight reachable).  Binary16 family: two values per 32-bit word
// (the half2 packing of PAPER.md:414, "combine 16-bit numbers into 32- or 64-bit words")
// in an ODD number of 8-byte units read with 8-byte loads, so a random record's unit u
// lands in 8-byte group (units * i + u) mod 16, every group reachable -- 32-byte records
// (even stride) reach only even groups and measured 371 vs 273 ms at config 5.  Measured
// and dropped for binary32 (round 1): odd-stride records read with 4-byte loads (441 vs
// 334 ms) and 8-byte loads of the C values (472 vs 334 ms).
__host__ __device__ constexpr int staged_half_units(int c) {
  return ((2 * c + 7) / 8) % 2 ? (2 * c + 7) / 8 : (2 * c + 7) / 8 + 1;
}
// One output (single-output models whose F bytes per object do not fit K2's bucket
// tile): a record is the leaf itself, binary64 / binary32 / binary16.
__host__ __device__ constexpr int staged_record_values(int c, int leaf) {
  return c == 1 ? 1 : leaf == 2 ? 4 * staged_half_units(c) : (c + 3) / 4 * 4;
}
constexpr int kStagedThreadsConsumers = 512;
constexpr int kStagedTile = 4 * kStagedThreadsConsumers;  // 2048 objects
constexpr int kStagedThreads = kStagedThreadsConsumers + 32;

struct StagedParams {
  const uint8_t* q;          // tiled buckets [n_tiles][F][2048]
  const uint32_t* desc;      // K4 descriptors [T][DI][2] (tile 512 offsets)
  const float* leaves;       // [T][2^DI] records of CP binary32 (or binary16) values
  double* out;               // [n][C]
  int64_t n;
  int32_t n_features;
  int32_t tree_begin, tree_end;
  int32_t first, last;
  int32_t n_stages;
  uint32_t table_bytes;      // 2^DI * CP * 4
  uint32_t stage_bytes;      // table_bytes + DI * 2048, 128-byte multiple
  double scale, bias;
};

template <int DI, int CMP, int C, int LEAF>
__global__ void __launch_bounds__(kStagedThreads, 1) apply_multi_staged_kernel(const __grid_constant__ StagedParams p) {
  static_assert(LEAF == 1 || LEAF == 2 || (LEAF == 0 && C == 1), "K5: binary32 or binary16 records (binary64: one output)");
  constexpr int CP = staged_record_values(C, LEAF);
  constexpr int kRecBytes = CP * (LEAF == 0 ? 8 : LEAF == 2 ? 2 : 4);
  constexpr int kRows = LEAF == 2 ? 0 : kRecBytes / 16;
  using acc_t = typename LeafT<LEAF>::Acc;  // binary64 / binary32 fold
  extern __shared__ __align__(128) unsigned char st_raw[];
  unsigned char* smem = st_raw + ((128u - (smem_u32(st_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [S]
  uint64_t* empty = full + 8;                          // [S]
  unsigned char* stages = smem + 128;
  const int tid = threadIdx.x;
  const int n_trees = p.tree_end - p.tree_begin;
  if (tid == 0) {
    for (int i = 0; i < p.n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kStagedThreadsConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t tile_idx = blockIdx.x;
  const uint8_t* qtile = p.q + tile_idx * (int64_t)p.n_features * kStagedTile;
  const int warp_id = __shfl_sync(0xffffffffu, tid / 32, 0);
  if (warp_id == 0) {
    // producer warp: lane d < DI copies the bucket row of depth d (its descriptor loaded
    // one tree ahead, so no global-load latency sits between a stage's release and its
    // refill), lane 0 the tree's record table and the stage's expect_tx.  Row copies may
    // complete before lane 0's arrive.expect_tx: the phase needs that arrival anyway.
    // Measured at config 5: binary16 records 196 ms with per-lane row copies vs 251 ms
    // with one thread issuing every copy; binary32 records the other way round (289 vs
    // 266 ms), so the binary32 family keeps the single issuing thread.
    constexpr bool kSerial = LEAF == 1 && C > 1;
    const int lane = tid;
    if (kSerial && lane > 0) return;
    const uint2* desc = reinterpret_cast<const uint2*>(p.desc);
    uint2 dd = lane < DI && n_trees > 0 ? __ldg(desc + (size_t)p.tree_begin * DI + lane) : make_uint2(0u, 0u);
    for (int i = 0; i < n_trees; ++i) {
      const int t = p.tree_begin + i;
      const int s = i % p.n_stages;
      const uint2 next = lane < DI && i + 1 < n_trees ? __ldg(desc + (size_t)(t + 1) * DI + lane) : make_uint2(0u, 0u);
      if (i >= p.n_stages) {
        if (lane == 0) mbar_wait(&empty[s], (uint32_t)(i / p.n_stages - 1) & 1u);
        if (!kSerial) __syncwarp();
      }
      unsigned char* dst = stages + (size_t)s * p.stage_bytes;
      if (kSerial) {
        const uint2* ds = desc + (size_t)t * DI;
        for (int d = 0; d < DI; ++d) {
          const uint2 e = __ldg(ds + d);
          const uint32_t off512 = CMP == 7 ? e.x : (e.x >> 8);
          bulk_g2s(dst + p.table_bytes + (size_t)d * kStagedTile, qtile + (size_t)(off512 / 512u) * kStagedTile,
                   kStagedTile, &full[s]);
        }
      } else if (lane < DI) {
        const uint32_t off512 = CMP == 7 ? dd.x : (dd.x >> 8);  // f * 512 (sentinel splits: 0)
        bulk_g2s(dst + p.table_bytes + (size_t)lane * kStagedTile, qtile + (size_t)(off512 / 512u) * kStagedTile,
                 kStagedTile, &full[s]);
      }
      if (lane == 0) {
        mbar_expect_tx(&full[s], p.table_bytes + (uint32_t)DI * kStagedTile);
        // tree t's records: 2^DI x kRecBytes = table_bytes (no padding between trees)
        bulk_g2s_split(dst, reinterpret_cast<const unsigned char*>(p.leaves) + (size_t)t * p.table_bytes, p.table_bytes,
                       &full[s]);
      }
      dd = next;
    }
    return;
  }
  const int word = tid - 32;  // bucket word of this thread: objects word_object(.., word, k)
  const int64_t tile_base = tile_idx * kStagedTile;
  auto obj_of = [&](int k) { return word_object(tile_base, word, k); };
  acc_t acc[4][C];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[k][c] = (p.first || obj_of(k) >= p.n) ? (acc_t)0 : (acc_t)p.out[obj_of(k) * C + c];
  const uint32_t stages_s = smem_u32(stages);
  // the binary16 family (40 binary32 accumulators) has the registers to load the next
  // tree's descriptors while this tree folds; the binary64 family (80) loads them per tree
  constexpr bool kPrefetch = LEAF == 2 || C == 1;
  const uint2* desc = reinterpret_cast<const uint2*>(p.desc);
  uint2 dnext[kPrefetch ? DI : 1];
  if constexpr (kPrefetch) {
#pragma unroll
    for (int d = 0; d < DI; ++d) dnext[d] = n_trees > 0 ? __ldg(desc + (size_t)p.tree_begin * DI + d) : make_uint2(0u, 0u);
  }
  for (int i = 0; i < n_trees; ++i) {
    const int t = p.tree_begin + i;
    const int s = i % p.n_stages;
    uint2 dcur[kPrefetch ? DI : 1];
    if constexpr (kPrefetch) {
#pragma unroll
      for (int d = 0; d < DI; ++d) {
        dcur[d] = dnext[d];
        dnext[d] = i + 1 < n_trees ? __ldg(desc + (size_t)(t + 1) * DI + d) : make_uint2(0u, 0u);
      }
    }
    mbar_wait_warp(&full[s], (uint32_t)(i / p.n_stages) & 1u);
    const uint32_t tab = stages_s + (uint32_t)s * p.stage_bytes;
    const uint32_t rows = tab + p.table_bytes + 4u * (uint32_t)word;
    const uint2* ds = desc + (size_t)t * DI;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int d = 0; d < DI; ++d) {
      const uint2 dd = kPrefetch ? dcur[kPrefetch ? d : 0] : __ldg(ds + d);  // warp-uniform: one broadcast
      const uint32_t w = lds_u32(rows + (uint32_t)d * kStagedTile);
      uint32_t b7;
      if constexpr (CMP == 7) {
        b7 = w + dd.y;
      } else {
        b7 = maj3((w & 0x7f7f7f7fu) + (__byte_perm(dd.x, 0u, 0x0000u) & 0x7f7f7f7fu), w, dd.y);
      }
      if (d < 8) lo |= (b7 >> (7 - d)) & (0x01010101u << d);
      else hi |= (b7 >> (15 - d)) & (0x01010101u << (d - 8));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t idx = ((lo >> (8 * k)) & 0xffu) | (DI > 8 ? ((hi >> (8 * k)) & 0xffu) << 8 : 0u);
      const uint32_t rec = tab + idx * (uint32_t)kRecBytes;
      if constexpr (C == 1) {
        acc[k][0] += LeafT<LEAF>::widen(lds_leaf<LEAF>(rec));
      } else if constexpr (LEAF == 1) {
        float v[CP];
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v[4 * r]), "=f"(v[4 * r + 1]), "=f"(v[4 * r + 2]), "=f"(v[4 * r + 3])
                       : "r"(rec + 16u * r));
        }
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] += (double)v[c];
      } else {
        // binary16 pairs, 8-byte units; the last unit loads only the word that holds values
        constexpr int kWords = (C + 1) / 2;
        uint32_t w[CP / 2];
#pragma unroll
        for (int u = 0; u < (kWords + 1) / 2; ++u) {
          if (2 * u + 1 < kWords) {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[2 * u]), "=r"(w[2 * u + 1]) : "r"(rec + 8u * u));
          } else {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[2 * u]) : "r"(rec + 8u * u));
          }
        }
        // widen each pair to binary32 and fold two outputs per packed FADD2 (two
        // independent round-to-nearest adds: the bits of two FADDs)
#pragma unroll
        for (int c = 0; c + 1 < C; c += 2) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[c / 2]));
          fadd2(acc[k][c], acc[k][c + 1], f.x, f.y);
        }
        if constexpr (C % 2) acc[k][C - 1] += __half2float(__ushort_as_half((unsigned short)(w[C / 2] & 0xffffu)));
      }
    }
    // (releasing one tree later instead, behind the loop's back edge and without the fence,
    // measured 270 vs 275 ms at config 5 but 14.2 vs 13.4 ms at the epsilon shape)
    mbar_release(&empty[s]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (obj_of(k) >= p.n) continue;
#pragma unroll
    for (int c = 0; c < C; ++c)
      p.out[obj_of(k) * C + c] = p.last ? __dadd_rn(__dmul_rn((double)acc[k][c], p.scale), p.bias) : (double)acc[k][c];
  }
}

}  // namespace obt
