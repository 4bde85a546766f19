/*
 * obtree_b200.h -- C ABI of the B200 (sm_100a) oblivious-ensemble apply path.
 *
 * The reference package (arxiv 2211.00391 re-implementation, "obtree") is pure
 * Python + numpy and has no FFI of its own; its drop-in boundary is the Python
 * API.  This header is the thin native layer under the Python shim in
 * paper_2211_00391_b200/ that keeps those names.  Each entry point below cites
 * the reference interface it replaces (paths under pkg/src/obtree/).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch/CUDA types in the signatures
 *     (streams travel as void* holding a cudaStream_t, 0 = legacy default);
 *   - every call returns OBT_OK (0) or a negative OBT_E* code and sets a
 *     thread-local message readable with obt_last_error();
 *   - device pointers ("_dev") must live on the model's device; host pointers
 *     ("_host") may be pageable or pinned (pinned is what makes copies async);
 *   - a model handle is immutable after creation and may be used from several
 *     host threads and streams at once (reference: SPEC.md "single-threaded by
 *     contract", model.py:10-11 read-only sharing, tests/test_evaluate.py:216-237).
 */
#ifndef OBTREE_B200_H
#define OBTREE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OBT_ABI_VERSION 1

/* status codes */
#define OBT_OK 0
#define OBT_E_INVALID (-1)     /* bad argument or model (message says which) */
#define OBT_E_CUDA (-2)        /* a CUDA runtime call failed */
#define OBT_E_UNSUPPORTED (-3) /* shape outside what the kernels implement */
#define OBT_E_NOMEM (-4)

/* feature matrix layouts -- quantize.py:25-29 (Layout), :59-90 (FeatureMatrix):
 * OBJECT_MAJOR element (o, f) at o*F + f; FEATURE_MAJOR at f*N + o. */
#define OBT_LAYOUT_OBJECT_MAJOR 0
#define OBT_LAYOUT_FEATURE_MAJOR 1

/* leaf precision families -- model.py:29-31 (LeafPrecision), accumulate.py:34-45:
 * BINARY64: binary64 leaves, binary64 tree-order accumulation (NAIVE/GATHER/PERMUTE64);
 * BINARY16: leaves rounded to binary16 (RNE, saturated to +/-65504, model.py:262-268),
 *           binary32 tree-order accumulation (NAIVE16/PERMUTE16). */
#define OBT_PRECISION_BINARY64 0
#define OBT_PRECISION_BINARY16 1

/* Host-side model description (everything is copied; the caller keeps ownership).
 * Replaces ModelTables.__init__ (evaluate.py:147-161) + build_leaf_bank
 * (model.py:231-277) as the "prepare once, evaluate many" step. */
typedef struct obt_model_desc {
  int32_t n_features;            /* F >= 1 (model.py:139-140) */
  int32_t n_trees;               /* T >= 0 */
  int32_t max_depth;             /* Dmax: 0 when T == 0, else 1..16 */
  int32_t n_outputs;             /* C >= 1 (the reference has C == 1) */
  const int32_t* border_counts;  /* [F], each 0..254 (model.py:21, 146-147) */
  const float* borders;          /* [F][border_stride], strictly ascending per feature */
  int32_t border_stride;         /* >= max(border_counts) */
  const int32_t* split_feature;  /* [T][Dmax]; padding slots may hold any valid feature */
  const uint8_t* split_ordinal;  /* [T][Dmax]; 255 = sentinel "never true" for trees
                                    shallower than Dmax (evaluate.py:32, 155-161) */
  const double* leaves;          /* [T][C][1 << Dmax] binary64 leaf values; slots past a
                                    shallow tree's 2^depth are never read */
  const uint16_t* leaves_f16;    /* optional [T][C][1 << Dmax] binary16 bank bits; NULL =
                                    convert from `leaves` with RNE + saturation */
  double scale;                  /* prediction = scale * sum + bias (model.py:93-95) */
  double bias;
  int32_t precision;             /* OBT_PRECISION_* */
} obt_model_desc;

typedef struct obt_model obt_model; /* opaque, device-resident */

/* Validate + upload.  Errors carry the reference's validate_model texts
 * (model.py:131-178) where they apply. */
int obt_model_create(const obt_model_desc* desc, int device, obt_model** out);
int obt_model_destroy(obt_model* model);

/* Introspection for the host shim and the bench (all written through pointers):
 * leaf storage actually used on the device: 0 = fp64, 1 = fp32 (chosen when every
 * binary64 leaf is exactly a binary32 value, so widening is exact), 2 = fp16. */
int obt_model_info(const obt_model* model, int32_t* n_features, int32_t* n_trees,
                   int32_t* max_depth, int32_t* n_outputs, int32_t* precision,
                   int32_t* leaf_storage, int32_t* compare_mode);

/* Which quantize search the predict path runs for TMA-eligible inputs (object-major,
 * F % 4 == 0, 16-byte aligned): kind 1 / 2 / 3 = cell tables (K1L, 256 / 1024 / 512 cells per
 * feature) with `param` compares per value, kind 0 = Eytzinger search (K1t) with `param`
 * levels.  Diagnostics for tests
 * and tuning; no reference counterpart (the reference always counts every border,
 * quantize.py:171). */
int obt_model_quantize_kernel(const obt_model* model, int32_t* kind, int32_t* param);

/* Which multi-output apply kernel a model with n_outputs > 1 runs: 0 = K4 (records
 * gathered from L2), 2 = K5 (tables and bucket rows staged in shared memory); -1 for
 * single-output models.  Diagnostics, like the above. */
int obt_model_multi_kernel(const obt_model* model, int32_t* kind);

/* Path options: force one of the planner's automatic choices, process-wide, so parity
 * tests can cover every kernel path and A/B runs can compare them.  value -1 restores the
 * automatic choice (the default; production callers never set these).  Names:
 *   "desc_source"  0 shared-memory ring, 1 kernel-parameter bank (K2 descriptors)
 *   "tpw"          lanes per bucket word in K2 / K2s (1, 2, 4)
 *   "wide"         0 / 1 forbid / force K2w (where it fits)
 *   "fan"          0 / 1 forbid / force K2f (small batches)
 *   "pdl"          0: no chained (programmatic dependent) parameter-bank launches
 *   "tail_split"   0 / 1 forbid / force the tail-wave region
 *   "quant_lut"    0 / 1 Eytzinger (K1t) / cell-table (K1L) quantize
 *   "lut_cells"    256, 512, 1024 cells per feature table (read by obt_model_create)
 *   "leaf_storage" 0: binary64 tables even when binary32 is exact (obt_model_create)
 *   "multi_staged" 0 / 1 K4 / K5 for multi-output models (obt_model_create)
 *   "leaf_select"  1: K2 takes leaves by warp shuffle from a register-resident table
 *                  (binary16 depth <= 6, binary32 depth <= 5; the PERMUTE16 / PERMUTE64
 *                  strategies of accumulate.py:116-159); default shared-memory gathers
 * Not synchronised with concurrent predict calls: set them between calls.  No
 * reference counterpart (the reference has one CPU path). */
int obt_set_path_option(const char* name, int value);
int obt_get_path_option(const char* name, int* value);

/* Bytes of scratch obt_predict_dev needs for n objects (the blocked bucket matrix). */
int obt_workspace_size(const obt_model* model, int64_t n_objects, size_t* bytes);

/* Evaluator.predict (evaluate.py:268-300) on device-resident features:
 * x_dev float32 [n][F] or [F][n] (4-byte aligned; 16-byte aligned object-major rows
 * with F % 4 == 0 take the TMA-staged quantize); out_dev float64 [n][C].  workspace
 * (256-byte aligned, obt_workspace_size bytes) may be NULL: then it comes from the
 * library's stream-ordered pool.  n == 0 is a no-op (evaluate.py:277-279).
 * Asynchronous on `stream`. */
int obt_predict_dev(const obt_model* model, const float* x_dev, int64_t n_objects,
                    int32_t layout, double* out_dev, void* workspace, size_t workspace_bytes,
                    void* stream);

/* evaluate() (evaluate.py:303-307) from host memory: copies x_host in chunks
 * (pinned buffers overlap the copy with compute), predicts, copies the
 * predictions back into out_host, and returns when out_host is valid. */
int obt_predict_host(const obt_model* model, const float* x_host, int64_t n_objects,
                     int32_t layout, double* out_host, void* stream);

/* One call over several devices of this process (the reference's
 * Evaluator.predict, evaluate.py:268-300, has one CPU path and no counterpart).  `shards`
 * holds n_shards (1..16) model handles, normally one per GPU (handles may share a device).
 *   OBT_SHARD_OBJECTS  every handle is the whole model; shard s evaluates a contiguous
 *                      range of objects (256-object quanta) on its device from its own host
 *                      thread through the obt_predict_host pipeline.  No data crosses
 *                      between devices; results are bit-identical to one device
 *                      (predictions depend only on their own row, oracle.py:42-51).
 *                      scale / bias are ignored (each handle carries the model's own).
 *   OBT_SHARD_TREES    handle s holds trees [t_s, t_{s+1}) as a raw partial-sum model
 *                      (scale 1, bias 0); every device evaluates every object against its
 *                      trees, the binary64 partial sums are copied to shard 0's device
 *                      (peer copies: NVLink between the GPUs of one box), added in shard
 *                      order and finalized as sum * scale + bias with two roundings.  This
 *                      reassociates the reference's tree-order fold (~1e-16 relative of the
 *                      partial magnitudes for binary64 leaves, ~1e-7 for the binary16 family).
 * x_host float32 [n][F] or [F][n]; out_host float64 [n][C]; returns when out_host is valid.
 * (The one-process-per-GPU form of both modes, with an NCCL all_reduce for the tree
 * shards, lives in the Python sharding module over torch.distributed.) */
#define OBT_SHARD_OBJECTS 0
#define OBT_SHARD_TREES 1
int obt_predict_sharded(const obt_model* const* shards, int32_t n_shards, int32_t mode,
                        const float* x_host, int64_t n_objects, int32_t layout, double scale,
                        double bias, double* out_host);

/* Stage 1 alone -- quantize_block (quantize.py:136-172) over the whole batch:
 * buckets_dev uint8 [F][n], bucket = #{k : x > border_k}, NaN -> 0. */
int obt_quantize_dev(const obt_model* model, const float* x_dev, int64_t n_objects,
                     int32_t layout, uint8_t* buckets_dev, void* stream);

/* Stage 2 alone -- compute_leaf_indices (indexer.py:39-57) / _leaf_index_panel
 * (evaluate.py:199-207) for trees [tree_begin, tree_end): idx_dev uint16
 * [tree_end - tree_begin][n], root condition in bit 0.  Runs the same quantize
 * and index code as obt_predict_dev. */
int obt_leaf_indices_dev(const obt_model* model, const float* x_dev, int64_t n_objects,
                         int32_t layout, int32_t tree_begin, int32_t tree_end,
                         uint16_t* idx_dev, void* stream);

/* obt_predict_dev with CUDA events recorded on `stream` before the quantize kernel,
 * between quantize and apply, and after apply (events from obt_event_create; any may
 * be NULL).  Used by bench.py to time each kernel on the stream it runs on. */
int obt_predict_dev_marked(const obt_model* model, const float* x_dev, int64_t n_objects,
                           int32_t layout, double* out_dev, void* workspace, size_t workspace_bytes,
                           void* stream, void* ev_begin, void* ev_mid, void* ev_end);

/* Minimal CUDA event helpers (timing-enabled events) for callers without a CUDA binding. */
int obt_event_create(void** event);
int obt_event_record(void* event, void* stream);
int obt_event_elapsed_ms(void* start, void* end, float* ms);
int obt_event_destroy(void* event);

/* Number of kernel launches the last predict on this thread issued (bench evidence). */
int obt_last_launch_count(void);

const char* obt_last_error(void);
int obt_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* OBTREE_B200_H */
