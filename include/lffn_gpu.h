/*
 * lffn_gpu.h -- C-ABI of the B200-native LookupFFN forward (sm_100a).
 *
 * This is the drop-in boundary for the reference library `lookupffn`
 * (namespace lffn, /root/reference/proj).  The reference exposes the hot path
 * as a C++ API (no FFI); every entry point below names the reference
 * interface it replaces.  INTEGRATION.md shows the C++ shim a maintainer adds
 * on the reference side (lffn::gpu::lookup_forward & co.) and the ctypes
 * binding used by the Python host package.
 *
 * Conventions (all kept from the reference):
 *   x      [n x d_in]  float32 row-major                (bench.cpp:102-112)
 *   z      [n x h*tau] float64, viewed as [n][h][tau]   (lookup.hpp:70-79)
 *   codes  [n x h]     uint32, bit j <- [z_{k*tau+j} >= 0], LSB first
 *                                                       (lookup.cpp:74-100)
 *   coeff  [n x h]     float32: the top-1 weight prod_j 1/(1+e^{-2|z_j|}),
 *                      times sum_j |z_j| for the scaled variants
 *                                                       (bench.cpp:162-180)
 *   T      [h][2^tau][d_out], row(k,c) = T + (k*2^tau + c)*d_out
 *                                                       (lookup.hpp:43-57)
 *   y      [n x d_out] float32                          (bench.cpp:182-194)
 *
 * Status codes map the reference error taxonomy (common.hpp:13-37):
 *   0 ok, 1 SizeError/UsageError, 2 NumericError (message names the stage:
 *   "projection forward input", "hash stage", "gather stage"), 3 CUDA runtime.
 * Device pointers are caller-owned; the context owns its workspace and never
 * allocates inside hash / lookup_accumulate / forward.  Calls are ordered on
 * the caller's stream (a cudaStream_t passed as void*; NULL = legacy default
 * stream).  Non-finite checks run on the device; kernels raise a flag that
 * lffn_sync() (and every blocking call) turns into status 2.  One context per
 * host thread.
 */
#ifndef LFFN_GPU_H
#define LFFN_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFFN_OK 0
#define LFFN_ERR_USAGE 1
#define LFFN_ERR_NUMERIC 2
#define LFFN_ERR_RUNTIME 3

/* ProjKind (projection.hpp:13) */
#define LFFN_PROJ_DENSE 0
#define LFFN_PROJ_BH 1
#define LFFN_PROJ_ACDC 2
#define LFFN_PROJ_SIGNFLIP 3

/* LookupVariant (lookup.hpp:20) */
#define LFFN_SOFTMAX 0
#define LFFN_SCALED 1
#define LFFN_SIGMOID_TAU1 2
#define LFFN_GELU_TAU1 3

/* element types of table storage / host buffers */
#define LFFN_F32 0
#define LFFN_BF16 1
#define LFFN_F64 2

/* LookupConfig (lookup.hpp:25-39) */
typedef struct lffn_cfg {
  int64_t d_in;
  int64_t d_out;
  int64_t tables;         /* h */
  int64_t code_bits;      /* tau */
  int32_t variant;        /* LFFN_SOFTMAX .. LFFN_GELU_TAU1 */
  int32_t neighbor_count; /* nc; the device path implements 1 <= nc <= 256 */
} lffn_cfg;

/* ProjectionSpec + Projection::blob() (projection.hpp:21-95).  blob is a
 * HOST pointer in the reference blob layout (projection.hpp:47-54); the
 * context copies what it needs at creation. */
typedef struct lffn_proj {
  int32_t kind;
  int32_t reserved;
  int64_t d_in;
  int64_t d_out; /* must equal tables * code_bits */
  int64_t stages;
  int64_t block;
  int64_t depth;
  const double* blob;
  int64_t blob_len;
} lffn_proj;

typedef struct lffn_ctx lffn_ctx;

/* ---- host-side configuration and parameter helpers -------------------- */

/* LookupConfig::validate (lookup.cpp:27-37) */
int lffn_cfg_validate(const lffn_cfg* cfg);
/* ProjectionSpec::validate (projection.cpp:29-40) + blob length check of
 * Projection::from_blob (projection.cpp:137-145) when blob != NULL */
int lffn_proj_validate(const lffn_proj* proj);
/* ProjectionSpec::transform_width (projection.hpp:30) */
int64_t lffn_transform_width(const lffn_proj* proj);
/* blob_size_for (projection.cpp:81-93) */
int64_t lffn_proj_blob_size(const lffn_proj* proj);
/* Projection::init (projection.cpp:97-135): fills blob_out[blob_size] */
int lffn_proj_init(const lffn_proj* spec, uint64_t seed, double* blob_out);
/* make_rng(seed) + fill_gaussian / fill_signs (common.hpp:44-55) */
int lffn_fill_gaussian(uint64_t seed, double* out, int64_t n, double stddev);
/* Elements [skip, skip + n) of the same make_rng(seed) + fill_gaussian stream
 * (one distribution object over the whole stream, the first `skip` draws
 * discarded): a table shard's slice of HashTables data without the rest. */
int lffn_fill_gaussian_slice(uint64_t seed, int64_t skip, double* out, int64_t n, double stddev);
int lffn_fill_signs(uint64_t seed, double* out, int64_t n);
/* HashTables::init (lookup.cpp:39-49): std 1/sqrt(h) */
int lffn_tables_init(const lffn_cfg* cfg, uint64_t seed, double* out);

/* Element conversion used by lffn_tables_upload: f64/f32/bf16 -> f64/f32/bf16,
 * each rounding a single round-to-nearest-even (the stored table values a
 * parity check must feed to the float64 oracle). */
int lffn_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n);

/* ---- device context ------------------------------------------------------ */

/* Validates like check_shapes (lookup.cpp:173-182) and allocates the
 * workspace for up to max_tokens rows (LookupWorkspaceF32, bench.cpp:102-112). */
int lffn_ctx_create(lffn_ctx** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                    const lffn_proj* proj);
/* Same for a table shard: this context owns tables [table_begin, table_end)
 * of the h-table stack; hash emits codes/coeffs only for those tables and
 * lookup_accumulate produces the partial sum over them (multi-GPU table
 * sharding; no reference counterpart). */
int lffn_ctx_create_shard(lffn_ctx** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                          const lffn_proj* proj, int64_t table_begin, int64_t table_end);
int lffn_ctx_destroy(lffn_ctx* ctx);
/* tables owned by this context: [*begin, *end) */
int lffn_ctx_table_range(const lffn_ctx* ctx, int64_t* begin, int64_t* end);

/* One-time upload of HashTables::data (lookup.hpp:43-66).  host_T is the FULL
 * [h][2^tau][d_out] stack in host_dtype (LFFN_F64 for the reference's double
 * tables, LFFN_F32, LFFN_BF16); it is converted (round-to-nearest-even) to
 * store_dtype (LFFN_F32 or LFFN_BF16) and a shard keeps only its slice.
 * Tables are read-only afterwards (lookup.hpp:41-42). */
int lffn_tables_upload(lffn_ctx* ctx, const void* host_T, int host_dtype, int store_dtype);
/* The same upload from a host buffer holding only this context's slice
 * [table_end-table_begin][2^tau][d_out] (a table shard built without the
 * rest of the stack, e.g. by lffn_fill_gaussian_slice). */
int lffn_tables_upload_slice(lffn_ctx* ctx, const void* host_slice, int host_dtype, int store_dtype);
/* Use a caller-owned device buffer holding this context's slice
 * [table_end-table_begin][2^tau][d_out] in dtype (no copy). */
int lffn_tables_attach(lffn_ctx* ctx, const void* d_T, int dtype);

/* ---- checkpoints: the reference's "LFFN" v1 file (checkpoint.hpp:17-26) --
 * header -> cfg (neighbor_count 1) + projection spec (proj->blob NULL,
 * proj->blob_len set) + total table length; load -> float64 blob and tables;
 * save writes the same format (save_checkpoint, checkpoint.cpp:52-84).
 * Errors: status 1 with the reference's messages (bad magic, unsupported
 * version, bad variant/kind byte, truncated file, trailing bytes). */
int lffn_checkpoint_header(const char* path, lffn_cfg* cfg, lffn_proj* proj, int64_t* tables_len);
int lffn_checkpoint_load(const char* path, double* blob, double* tables);
int lffn_checkpoint_save(const char* path, const lffn_cfg* cfg, const lffn_proj* proj,
                         const double* tables);
/* Context straight from a checkpoint (load_checkpoint, checkpoint.cpp:86-138):
 * tables [table_begin, table_end) (0, 0 = all) are streamed from the file
 * into the device copy in store_dtype without materialising the whole stack
 * on the host. */
int lffn_ctx_create_from_checkpoint(lffn_ctx** out, int device, int64_t max_tokens,
                                    const char* path, int store_dtype, int64_t table_begin,
                                    int64_t table_end);

/* Hash stage = Projection::forward (projection.cpp:167-266) + compute_codes
 * (lookup.cpp:81-100) + top-1 weight (lookup.cpp:185-189), i.e. the
 * lookup_hash_f32 + lookup_weights_f32 pair (bench.cpp:115-180), in one
 * kernel.  d_codes/d_coeff: [n x h_local x nc]; for nc > 1 the records of a
 * (token, table) are neighbor_codes (lookup.cpp:118-165) in the reference's
 * order with coefficient exp(<z,S_c> - logden) (x <z,S_c> when scaled,
 * lookup.cpp:241-252), the LookupCache slot layout (i*h + k)*nc + c.
 * d_z (optional, may be NULL): [n x h*tau] float64 projection output
 * (bit-identical to the reference's double Projection::forward for the
 * signflip, acdc, bh and exact-dense kinds). */
int lffn_hash(lffn_ctx* ctx, const float* d_x, int64_t n, uint32_t* d_codes, float* d_coeff,
              double* d_z, void* stream);

/* Gather stage = lookup_gather_f32 (bench.cpp:182-194): y_i (+)= sum_k
 * coeff[i,k] * T[k][codes[i,k]], tables in ascending order (nc > 1: records
 * (k, c) in slot order, forward_impl lookup.cpp:238-262).  accumulate = 0
 * overwrites y (the reference zero-fills first), 1 adds into y. */
int lffn_lookup_accumulate(lffn_ctx* ctx, const uint32_t* d_codes, const float* d_coeff,
                           int64_t n, float* d_y, int accumulate, void* stream);

/* Full forward = lookup_forward (lookup.cpp:191-282):
 * hash -> gather on the device, no host round trip. */
int lffn_forward(lffn_ctx* ctx, const float* d_x, int64_t n, float* d_y, void* stream);

/* Same with HOST x / y (pinned or pageable): the host<->device copies are
 * chunked and overlapped with the kernels on internal streams.  Blocking;
 * returns the deferred numeric status. */
int lffn_forward_host(lffn_ctx* ctx, const float* h_x, int64_t n, float* h_y);

/* ---- backward (training) --------------------------------
 * lookup_backward (lookup.cpp:292-347) at the forward's neighbour selection,
 * recomputed from x on the device: d_grad_y [n x d_out] float32 in;
 * d_grad_x [n x d_in] float64, d_grad_tables [h_local][2^tau][d_out] float32
 * (overwritten), d_grad_proj float64 in the blob layout (param_count entries:
 * dense W [d_in x h*tau], acdc diagonals, bh blocks; signflip: none --
 * Projection::param_count is 0; overwritten) out; any output may be NULL.  A
 * table shard produces its tables' gradient and the partial grad_x /
 * grad_proj over its tables (sum over shards = full).
 * Non-finite grad_y / outputs raise status 2 at lffn_sync ("lookup backward
 * input", "projection backward output", "lookup backward tables"). */
int lffn_backward(lffn_ctx* ctx, const float* d_x, const float* d_grad_y, int64_t n,
                  double* d_grad_x, float* d_grad_tables, double* d_grad_proj, void* stream);
/* Projection::backward (projection.cpp:279-386) for a given float64 grad_z
 * [n x h*tau]: grad_x and the parameter gradient bit-identical to the
 * reference for the same grad_z (every kind). */
int lffn_proj_backward(lffn_ctx* ctx, const float* d_x, const double* d_grad_z, int64_t n,
                       double* d_grad_x, double* d_grad_proj, void* stream);

/* Waits for `stream` and reports any non-finite flag raised since the last
 * check (status 2 with the stage named in lffn_last_error()). */
int lffn_sync(lffn_ctx* ctx, void* stream);

/* Context options:
 *   LFFN_OPT_DENSE_EXACT       1 = dense projection in exact float64 (z
 *                              bit-identical to projection.cpp:178-198);
 *                              0 (default) = tcgen05 split-precision GEMM (bf16
 *                              x3 terms, tf32 hi/lo when d_in % 8 != 0) with
 *                              exact float64 recomputation of |z| < 1e-4, so
 *                              codes stay bit-exact
 *   LFFN_OPT_TABLE_GROUP_BYTES walk the tables in L2-sized groups of this many
 *                              bytes (0 = one pass, the default)
 *   LFFN_OPT_GATHER_VARIANT    gather kernel: 0 = default (batches smaller
 *                              than the resident warp slots split each
 *                              token's table walk over 2-8 warps), -1 = one
 *                              warp per token (part) always
 *   LFFN_OPT_BF16_COEFF_FMA    1 (default) = bf16 tables: groups of tables
 *                              whose coefficients are bf16 values (e.g. the
 *                              top-1 weight 1.0) accumulate with the exact
 *                              mixed-precision FMA on the packed halves (bit-
 *                              identical to the fp32 FMA); 0 = always unpack
 *   LFFN_OPT_BWD_ONE_PASS      1 = the backward's single-pass table-row dot
 *                              (the A/B reference of the default two passes)
 *   LFFN_OPT_HASH_EXACT        1 = the signflip hash always runs the stage
 *                              order of fwht_kernel (z bit-identical); 0
 *                              (default) = the production kernel at D = 2048 /
 *                              4096 (reordered stages, codes bit-exact
 *                              wherever |z| > 1e-5) unless z is requested
 *   LFFN_OPT_HOST_CHUNKS       lffn_forward_host pipeline chunks (1 .. 16,
 *                              default 8)
 *   LFFN_OPT_SMALL_MAX_TOKENS  batches of at most this many tokens (<= 64,
 *                              default 64; 0 = never) run the whole forward
 *                              in one launch spread over (token, table
 *                              group) CTAs (signflip, D = 2048, top-1)
 *   LFFN_OPT_GATHER_SMS        persistent gather grid over this many SMs
 *                              (0 = all, the default)
 *   LFFN_OPT_HOST_DIRECT       1 (default) = lffn_forward_host on a small
 *                              batch with pinned buffers writes y and the
 *                              non-finite flag straight into host memory and
 *                              polls the flag; 0 = the CUDA-graph path with
 *                              copy nodes */
#define LFFN_OPT_DENSE_EXACT 1
#define LFFN_OPT_TABLE_GROUP_BYTES 2
#define LFFN_OPT_GATHER_VARIANT 3
#define LFFN_OPT_BF16_COEFF_FMA 5
#define LFFN_OPT_BWD_ONE_PASS 6
#define LFFN_OPT_HASH_EXACT 7
#define LFFN_OPT_HOST_CHUNKS 8
#define LFFN_OPT_SMALL_MAX_TOKENS 10
#define LFFN_OPT_GATHER_SMS 11
#define LFFN_OPT_HOST_DIRECT 12
int lffn_ctx_set_option(lffn_ctx* ctx, int option, int64_t value);

/* ---- multi-GPU table sharding (north star: tables split
 * over GPUs, partial sums combined by NCCL reduce-scatter or all-reduce) ----
 * One lffn_group per rank (one process per GPU).  The group owns an NCCL
 * communicator (libnccl.so.2, loaded at run time), the rank's table shard
 * (tables split_range(h, world, rank): the first h % world ranks own one
 * more) and a table-less hash context for the rank's token block.
 * lffn_forward_sharded(x = all n tokens, identical on every rank):
 *   hash of the rank's token block for all tables, one grouped NCCL
 *   send/recv exchange of the (code, coefficient) records (each rank
 *   receives its tables' records for all n tokens), then per token chunk the
 *   gather of the fp32 partial over the rank's tables and the combine on the
 *   group's stream, overlapped with the next chunk's gather:
 *     LFFN_COMBINE_REDUCE_SCATTER  y = rows [r n/P, (r+1) n/P) of the sum
 *                                  (n a multiple of world * chunks)
 *     LFFN_COMBINE_ALL_REDUCE      y = all n rows of the sum
 *     LFFN_COMBINE_NONE            y = the rank's partial over its tables
 * Stream-ordered on `stream`; returns after the non-finite check (like
 * lffn_forward + lffn_sync). */
typedef struct lffn_group lffn_group;
#define LFFN_COMBINE_REDUCE_SCATTER 0
#define LFFN_COMBINE_ALL_REDUCE 1
#define LFFN_COMBINE_NONE 2
/* ncclGetUniqueId into out[len >= 128]; rank 0 creates it and the ranks
 * share it out of band (e.g. torch.distributed broadcast, MPI_Bcast). */
int lffn_nccl_unique_id(void* out, int64_t len);
int lffn_group_create(lffn_group** out, int device, int64_t max_tokens, const lffn_cfg* cfg,
                      const lffn_proj* proj, const void* nccl_id, int rank, int world);
int lffn_group_destroy(lffn_group* group);
/* The rank's table shard: upload its tables with lffn_tables_upload(_slice)
 * or lffn_tables_attach; set options on it. */
lffn_ctx* lffn_group_shard(lffn_group* group);
/* Token chunks of the gather / combine pipeline (1 .. 8, default 4). */
int lffn_group_set_chunks(lffn_group* group, int chunks);
int lffn_forward_sharded(lffn_group* group, const float* d_x, int64_t n, float* d_y, int combine,
                         void* stream);

/* Number of kernels launched through this context since creation. */
int64_t lffn_ctx_launch_count(const lffn_ctx* ctx);

/* Per-launch device timing of the last forward's stages (ms; CUDA events on
 * the launching stream; 0 when timing is off).  enable = 1 turns stage
 * events on for subsequent forwards. */
int lffn_ctx_set_timing(lffn_ctx* ctx, int enable);
int lffn_ctx_stage_ms(lffn_ctx* ctx, float* hash_ms, float* gather_ms);

/* Bandwidth probe for the roofline denominators (no reference counterpart):
 * which = 0 L2 read GB/s (32 MiB re-read from every SM), 1 HBM read GB/s
 * (4 GiB stream), 2 L2 read GB/s of random 512-byte segments of a 32 MiB
 * buffer (the gather's pattern); best of reps CUDA-event-timed launches. */
int lffn_probe_bandwidth(int device, int which, int reps, double* gbs);

/* Thread-local message for the last non-zero status. */
const char* lffn_last_error(void);
/* The reference exception class of the last failure on this thread:
 * status 1 splits into SizeError (shape / size checks, e.g. lookup.cpp:28-36,
 * 176-181) and UsageError (unknown names, checkpoint I/O, wrong call order)
 * as the reference throws them (common.hpp:17-23). */
#define LFFN_CLASS_SIZE 1
#define LFFN_CLASS_USAGE 2
#define LFFN_CLASS_NUMERIC 3
#define LFFN_CLASS_RUNTIME 4
int lffn_last_error_class(void);

/* Library identification: "lffn_gpu <version> sm_100a". */
const char* lffn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LFFN_GPU_H */
