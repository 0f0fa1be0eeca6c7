/*
 * permez_b200.h -- C ABI of the B200-native PW_REL block compression path.
 *
 * Drop-in boundary for the reference package's compress/decompress path
 * (arXiv 2309.09778, "permez").  The reference's interface for this path is
 * Python (SPEC.md op signatures + transform.py); every entry point below names
 * the reference interface it replaces.  Python binds these through ctypes in
 * paper_2309_09778_b200/_native.py.
 *
 * Conventions:
 *  - plain pointers and sizes, no torch types; device pointers are CUDA
 *    global-memory pointers owned by the caller, `stream` is a cudaStream_t;
 *  - the library never allocates device memory: the caller passes a workspace
 *    of pmz_workspace_size() bytes;
 *  - no global mutable state; weights travel by value in pmz_params;
 *  - return value 0 or a negative PMZ_ERR_* status mapped 1:1 onto the
 *    reference exception classes (errors.py:4-128);
 *  - output is deterministic for any launch configuration.
 */
#ifndef PERMEZ_B200_H
#define PERMEZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMZ_ABI_VERSION 2

#if defined(__GNUC__)
#define PMZ_API __attribute__((visibility("default")))
#else
#define PMZ_API
#endif

/* status codes <-> errors.py exception classes */
enum pmz_status {
  PMZ_OK = 0,
  PMZ_ERR_CONFIG = -1,                /* ConfigError            errors.py:8   */
  PMZ_ERR_NONFINITE = -2,             /* NonFiniteInput         errors.py:18  */
  PMZ_ERR_DEGENERATE = -3,            /* DegenerateBlock        errors.py:22  */
  PMZ_ERR_SUBNORMAL = -4,             /* SubnormalMinimum       errors.py:26  */
  PMZ_ERR_NONREPRESENTABLE = -5,      /* NonRepresentableFactor errors.py:32  */
  PMZ_ERR_TOO_FEW_BLOCKS = -6,        /* TooFewBlocks           errors.py:50  */
  PMZ_ERR_BALANCE_FLAG = -7,          /* BalanceFlagNotDequantizable :64     */
  PMZ_ERR_DEGENERATE_ALPHABET = -8,   /* DegenerateAlphabet     errors.py:68  */
  PMZ_ERR_UNASSIGNED = -9,            /* UnassignedCode         errors.py:72  */
  PMZ_ERR_TRUNCATED = -10,            /* TruncatedStream        errors.py:76  */
  PMZ_ERR_INVALID_PREFIX = -11,       /* InvalidPrefix          errors.py:80  */
  PMZ_ERR_BAD_MAGIC = -12,            /* BadMagic               errors.py:90  */
  PMZ_ERR_UNSUPPORTED_VERSION = -13,  /* UnsupportedVersion     errors.py:94  */
  PMZ_ERR_CORRUPT = -14,              /* Corrupt                errors.py:98  */
  PMZ_ERR_BALANCE_UNDERFLOW = -15,    /* BalanceUnderflow       errors.py:102 */
  PMZ_ERR_CAPACITY = -16,             /* output buffer too small (no ref. class) */
  PMZ_ERR_CUDA = -17,                 /* CUDA runtime failure                  */
  PMZ_ERR_WORKSPACE = -18,            /* workspace too small                   */
  PMZ_ERR_UNRESOLVED_ROUNDING = -19   /* CR log2/exp2 undecided (never seen)   */
};

/* Compression parameters.  Mirrors the reference parameters: b_r (--rel-error),
 * block size (--block-size RxC), partition_rows (--partition-rows),
 * perceptron weights (PerceptronModel), coverage target
 * (--coverage-target).  b_a and onepbr2 are the host-evaluated scalars of
 * transform.py:118 and :160-162 (`float(np.log2(1.0 + b_r))`,
 * `(1.0 + b_r) ** 2`). */
typedef struct pmz_params {
  double b_r;
  double b_a;
  double onepbr2;
  double eps0;            /* float_floor(float32) = 2^-126, transform.py:37  */
  double repair_t;        /* repair_factor * b_r; SPEC default factor 1.5    */
  double coverage_target; /* 0.99 default                      */
  double slope;           /* leaky ReLU slope                  */
  double w1[8];           /* (S+1) x H, row-major              */
  double w2[2];           /* H                                               */
  int32_t block_rows, block_cols, partition_rows;
  int32_t S;              /* surface size: 3 (2-D) or 1 (1-D)   */
  int32_t H;              /* hidden width, 2                                 */
  int32_t m;              /* code width; 0 = select_m on validation blocks   */
  int32_t precision;      /* 0: FP64 parity -- the reference's arithmetic,
                           *    container version 1 (the default);
                           * 1: FP32 perceptron perf mode (north star):
                           *    float32 surfaces, predictor, quantizer and
                           *    recurrence, container version 2; 2-D fields
                           *    only (throughput path), codes may differ from
                           *    version 1 where float32 rounding moves them   */
  int32_t reserved;       /* 0                                               */
  uint64_t d_code_dump;   /* 0, or a device address of
                           * pmz_code_dump_elems() uint16: every final code
                           * (raster per 32-row partition, 0xFFFF at the
                           * anchor) -- for counting code mismatches between
                           * the two precisions                              */
} pmz_params;

/* Shard geometry: this process holds rows [0, rows) of its shard, which are
 * global block-rows starting at `block_row0`.  Single GPU: block_row0 = 0. */
typedef struct pmz_geom {
  uint64_t rows, cols;
  uint64_t block_row0;
  uint64_t global_rows;   /* rows of the full field (header)                 */
} pmz_geom;

typedef struct pmz_result {
  uint64_t header_bytes;  /* container header (0 when not written)           */
  uint64_t record_bytes;  /* this shard's block records                      */
  uint64_t nblocks, ntrivial, nbal, nrepair, ncodes;
  uint64_t coverage[18];  /* select_m histogram (index = required m; 17 none) */
  int32_t m;
  int32_t max_code_len;
  uint32_t unresolved;    /* undecided CR roundings (expected 0)             */
  uint32_t launches;      /* kernels this library launched for the call      */
} pmz_result;

/* Parsed container header (read_container, layout :496). */
typedef struct pmz_header {
  uint64_t rows, cols;
  uint32_t block_rows, block_cols, partition_rows;
  uint32_t version, elem, m, S, H;
  double b_r, coverage_target, slope, w1[8], w2[2];
  uint64_t nblocks;
  uint64_t header_bytes;
  uint64_t lens_offset;   /* byte offset of the 2^m code lengths             */
} pmz_header;

/* A block whose per-block logarithm of a general double (lg_neg =
 * np.log2(factor_neg), transform.py:120; np.log2(factor_pos - eps0), :123)
 * lies so close to a rounding midpoint that numpy may round it differently
 * from the correctly rounded value.  The library lists such blocks; the host
 * fills lg[i] = np.log2(arg[i]) for every bit i of mask and hands the entries
 * back, so per-block parameters equal the reference's bit for bit (DESIGN
 * D22).  Callers that skip this step get the CR values. */
typedef struct pmz_np_fix {
  int64_t block;
  double arg[2];   /* factor_neg, factor_pos - eps0 */
  double lg[2];    /* filled by the host: np.log2(arg[i]) */
  int32_t mask;    /* bit i: arg[i] needs the host */
  int32_t pad;
} pmz_np_fix;

/* library / ABI identification */
PMZ_API int pmz_abi_version(void);
/* elements of the pmz_params::d_code_dump buffer for a shard geometry:
 * partitions x partition_rows x block_cols */
PMZ_API int pmz_code_dump_elems(const pmz_params *p, const pmz_geom *g, uint64_t *elems);
PMZ_API const char *pmz_status_string(int status);

/* Workspace bytes for a shard.  Replaces nothing in the reference (the
 * reference allocates implicitly through numpy). */
PMZ_API int pmz_workspace_size(const pmz_params *p, const pmz_geom *g, uint64_t *bytes);

/* Upper bound of the container bytes for a shard (header + records). */
PMZ_API int pmz_max_container_size(const pmz_params *p, const pmz_geom *g, uint64_t *bytes);

/* --- compression --------------------------------------------------------- */

/* Stage 1a: compute_block_stats + make_transform_params (transform.py:84-167)
 * for every block of the shard (device, CR logarithms); zeroes the status,
 * coverage and histogram.  Stage 1b (pmz_compress_transform): forward map and
 * the select_m coverage of the validation blocks.  pmz_compress_analyze =
 * 1a + 1b.  Between the two the host may resolve the listed general-double
 * logarithms with numpy: pmz_compress_np_fixups synchronises `stream` and
 * copies up to `cap` entries (returns the count, or a negative status);
 * pmz_compress_np_apply uploads the host's values and re-derives the listed
 * blocks' parameters (stream-ordered). */
PMZ_API int pmz_compress_stats(const float *d_in, const pmz_geom *g, const pmz_params *p, void *d_ws,
                               uint64_t ws_bytes, void *stream);
PMZ_API int pmz_compress_transform(const float *d_in, const pmz_geom *g, const pmz_params *p,
                                   const int64_t *d_val_blocks, int64_t n_val, void *d_ws, uint64_t ws_bytes,
                                   void *stream);
PMZ_API int64_t pmz_compress_np_fixups(const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes,
                                       void *stream, pmz_np_fix *h_fix, int64_t cap);
PMZ_API int pmz_compress_np_apply(const pmz_geom *g, const pmz_params *p, void *d_ws, uint64_t ws_bytes,
                                  void *stream, const pmz_np_fix *h_fix, int64_t n);

/* Stage 1: per-block stats + transform parameters for every block of the
 * shard, and the select_m coverage histogram over the validation blocks the
 * shard owns.  Replaces compute_block_stats + make_transform_params
 * (transform.py:84-107, 138-167) and the residual part of trainer.select_m
 * (SPEC.md:362-370).  d_val_blocks: shard-local validation block ids. */
PMZ_API int pmz_compress_analyze(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val_blocks,
                         int64_t n_val, void *d_ws, uint64_t ws_bytes, void *stream);

/* Device pointer of the 18 x u64 coverage histogram inside the workspace
 * (sum it across shards before stage 2 when sharded). */
PMZ_API uint64_t *pmz_ws_coverage(void *d_ws, const pmz_params *p, const pmz_geom *g);

/* Stage 2: select_m, then compress_block + verify_and_repair for every block
 * and the validation-code histogram of
 * estimate_codebook. */
PMZ_API int pmz_compress_codes(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val_blocks,
                       int64_t n_val, void *d_ws, uint64_t ws_bytes, void *stream);

/* Device pointer of the 65536 x u64 validation histogram (sum across shards
 * before stage 3) and of the i32 count of non-trivial validation blocks. */
PMZ_API uint64_t *pmz_ws_histogram(void *d_ws, const pmz_params *p, const pmz_geom *g);

/* Stage 3: build_codebook, encode and
 * write_container (byte layout :496).  Writes the header at
 * d_out[0] when write_header != 0 and this shard's block records right after
 * it (or at d_out[0] when write_header == 0).  Synchronises `stream` and fills
 * *res.  Returns PMZ_ERR_CAPACITY (res filled with the required sizes) when
 * out_cap is too small (call pmz_compress_write_async again with a larger
 * buffer: the encoded state stays in the workspace).  d_in: the shard's input
 * (the throughput path codes every block after the codebook). */
PMZ_API int pmz_compress_finish(const float *d_in, const pmz_geom *g, const pmz_params *p, int write_header,
                                uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws,
                                uint64_t ws_bytes, void *stream, pmz_result *res);

/* Stage 3 in two parts: pmz_compress_encode = build_codebook + (throughput
 * path) compress_block / verify_and_repair of every block with the final
 * codebook, or (latency path) the per-partition payload bits;
 * pmz_compress_write_async = record sizes and offsets, header, block records,
 * block index.  pmz_compress_finish_async = both, enqueue only (stream
 * capture: the writers read m, sizes and the capacity verdict from the device
 * status; nothing is written on error); pmz_compress_result synchronises
 * `stream`, fills *res and returns the status (wrote_output = d_out was
 * non-null). */
PMZ_API int pmz_compress_encode(const float *d_in, const pmz_geom *g, const pmz_params *p, void *d_ws,
                                uint64_t ws_bytes, void *stream);
PMZ_API int pmz_compress_write_async(const pmz_geom *g, const pmz_params *p, int write_header, uint8_t *d_out,
                                     uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes,
                                     void *stream);
PMZ_API int pmz_compress_finish_async(const float *d_in, const pmz_geom *g, const pmz_params *p, int write_header,
                                      uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws,
                                      uint64_t ws_bytes, void *stream);
PMZ_API int pmz_compress_result(const pmz_geom *g, const pmz_params *p, int wrote_output, void *d_ws,
                                uint64_t ws_bytes, void *stream, pmz_result *res);

/* All three stages enqueued on `stream` with no host synchronisation (single
 * GPU): capturable into a CUDA graph; read the outcome with
 * pmz_compress_result. */
PMZ_API int pmz_compress_enqueue(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val_blocks,
                                 int64_t n_val, int write_header, uint8_t *d_out, uint64_t out_cap,
                                 uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes, void *stream);

/* One-call single-GPU compress (cmd_compress minus ingest/training). */
PMZ_API int pmz_compress(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_val_blocks,
                 int64_t n_val, uint8_t *d_out, uint64_t out_cap, uint64_t *d_block_offsets, void *d_ws,
                 uint64_t ws_bytes, void *stream, pmz_result *res);

/* --- container ------------------------------------------------------------ */

/* read_container header part: BadMagic / UnsupportedVersion /
 * Corrupt.  Host memory. */
PMZ_API int pmz_parse_header(const uint8_t *h_buf, uint64_t n, pmz_header *hdr);

/* Walk the block records (host memory) and emit the byte offset of each
 * block record (nblocks entries).  Corrupt / TruncatedStream on bad framing. */
PMZ_API int pmz_index_blocks(const uint8_t *h_buf, uint64_t n, const pmz_header *hdr, uint64_t *h_block_offsets);
/* The same walk over the blocks [b0, b1) only, starting at byte pos0 (the
 * end offset of block b0 - 1, or hdr->header_bytes for b0 = 0): fills
 * h_block_offsets[0 .. b1 - b0] (the last entry is the end of block b1 - 1).
 * The host pipeline walks one slab of block-rows at a time while the earlier
 * slabs are already uploading. */
PMZ_API int pmz_index_blocks_range(const uint8_t *h_buf, uint64_t n, const pmz_header *hdr, uint64_t b0, uint64_t b1,
                                   uint64_t pos0, uint64_t *h_block_offsets);

/* --- decompression --------------------------------------------------------- */

PMZ_API int pmz_decompress_workspace_size(const pmz_header *hdr, uint64_t *bytes);

/* decompress_block for every block + inverse_map
 * (transform.py:188-202) -> f32 grid (rows x cols).  d_buf: the container in
 * device memory; d_block_offsets: byte offset of each block record. */
/* b_a = float(np.log2(1.0 + hdr->b_r)), evaluated by the host as in
 * derive_transform_params (transform.py:118). */
PMZ_API int pmz_decompress(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                   const uint64_t *d_block_offsets, float *d_out, void *d_ws, uint64_t ws_bytes, void *stream);
/* pmz_decompress split for streaming: enqueue every kernel on `stream` (no
 * host synchronisation, the status stays in the workspace), then
 * pmz_decompress_result synchronises the stream and maps the device status
 * (same return codes as pmz_decompress). */
PMZ_API int pmz_decompress_enqueue(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                                   const uint64_t *d_block_offsets, float *d_out, void *d_ws, uint64_t ws_bytes,
                                   void *stream);
PMZ_API int pmz_decompress_result(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream);
/* pmz_decompress_result that also reports the kernels this library ran for
 * the call (res->launches, counted on the device) and nblocks / m. */
PMZ_API int pmz_decompress_status(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream, pmz_result *res);
/* pmz_decompress_enqueue split at the numpy fixup point: _prepare parses the
 * block records and derives the per-block parameters (+ decode tables);
 * pmz_decompress_np_fixups / _np_apply as for compression; _run decodes and
 * reconstructs.  pmz_decompress_enqueue = _prepare + _run. */
PMZ_API int pmz_decompress_prepare(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                                   const uint64_t *d_block_offsets, void *d_ws, uint64_t ws_bytes, void *stream);
PMZ_API int pmz_decompress_run(const uint8_t *d_buf, uint64_t n, const pmz_header *hdr, double b_a,
                               const uint64_t *d_block_offsets, float *d_out, void *d_ws, uint64_t ws_bytes,
                               void *stream);
PMZ_API int64_t pmz_decompress_np_fixups(const pmz_header *hdr, void *d_ws, uint64_t ws_bytes, void *stream,
                                         pmz_np_fix *h_fix, int64_t cap);
PMZ_API int pmz_decompress_np_apply(const pmz_header *hdr, double b_a, void *d_ws, uint64_t ws_bytes, void *stream,
                                    const pmz_np_fix *h_fix, int64_t n);

/* --- trainer objective ------------ */

/* Sums over the samples of train_step's objective with the perceptron of `p`
 * (p->w1, w2, slope, S): d_out12[0..7] = d(sum r^2)/d w1 (row-major (S+1) x H,
 * bias row last), [8..9] d/d w2, [10] sum r^2, [11] sample count, where
 * r = predict(surface) - target.  Deterministic (fixed summation order).
 * pmz_train_gradient: samples = every element but the partition anchors of
 * the blocks listed in d_blocks, surfaces from the TRUE forward-mapped values
 * (the compress workspace of pmz_workspace_size; synchronises `stream`).
 * pmz_train_gradient_batch: samples given as surfaces (n x S, row-major) and
 * targets; d_ws of PMZ_TRAIN_BATCH_WS bytes; stream-ordered. */
#define PMZ_TRAIN_BATCH_WS (296 * 12 * 8)
PMZ_API int pmz_train_gradient(const float *d_in, const pmz_geom *g, const pmz_params *p, const int64_t *d_blocks,
                               int64_t n_blocks, double *d_out12, void *d_ws, uint64_t ws_bytes, void *stream);
PMZ_API int pmz_train_gradient_batch(const double *d_surf, const double *d_tgt, uint64_t n, const pmz_params *p,
                                     double *d_out12, void *d_ws, uint64_t ws_bytes, void *stream);

/* --- SEG-Y ingest ----------------- */

/* read_segy's sample conversion: d_traces = the trace records of a rev-0
 * file (n_traces x (240-byte header + ns big-endian 32-bit samples)) in
 * device memory -> d_out[n_traces][ns] IEEE float32, traces as rows.
 * format_code 1 (IBM hex float, exact in double, one rounding to float32) or
 * 5 (IEEE); anything else -> PMZ_ERR_CONFIG (UnsupportedFormatCode is
 * raised by the host reader before).  Stream-ordered. */
PMZ_API int pmz_segy_samples(const uint8_t *d_traces, uint64_t n_traces, uint32_t ns, int format_code, float *d_out,
                             void *stream);

/* --- transform module (transform.py) on device ------------------------------ */

/* Per-block transform parameters: 10 doubles per block in TransformParams
 * field order (transform.py:61-81) + trivial flag. */
PMZ_API int pmz_transform_params(const float *d_in, const pmz_geom *g, const pmz_params *p, double *d_params10,
                         uint8_t *d_trivial, void *d_ws, uint64_t ws_bytes, void *stream);

/* compute_block_stats (transform.py:84-107) over n doubles (the reference
 * upcasts every element type to float64, :95): d_out6 = abs_min over nonzero
 * magnitudes, abs_max, has_zero, has_negative, nonfinite, count (abs_min =
 * abs_max = 0 when there is no nonzero element).  d_scratch: 64 device bytes.
 * Stream-ordered. */
PMZ_API int pmz_block_stats(const double *d_x, uint64_t n, double *d_out6, void *d_scratch, void *stream);

/* derive_transform_params (transform.py:110-135): d_in4 = factor_pos,
 * factor_neg, b_r, epsilon0; b_a = float(np.log2(1.0 + b_r)) from the host
 * (:118); d_out10 in TransformParams field order.  *d_mask bit i: np.log2 of
 * (factor_neg, factor_pos - epsilon0, factor_pos, epsilon0)[i] is too close
 * to a rounding midpoint to be decided without numpy (see pmz_np_fix). */
PMZ_API int pmz_derive_params(const double *d_in4, double b_a, double *d_out10, int32_t *d_mask, void *stream);

/* zero_sub_floor_magnitudes (transform.py:205-210): out = x with |x| <= eps0 -> 0. */
PMZ_API int pmz_zero_sub_floor(const double *d_x, uint64_t n, double eps0, double *d_out, void *stream);

/* forward_map / inverse_map (transform.py:170-202) elementwise with one
 * parameter set (TransformParams fields, transform.py:61-81). */
PMZ_API int pmz_forward_map(const double *d_x, uint64_t n, const double *params10, double *d_v, void *stream);
PMZ_API int pmz_inverse_map(const double *d_v, uint64_t n, const double *params10, double *d_x64, float *d_x32,
                    void *stream);

/* CR log2 of float32 values (exhaustive-check helper, see tests). Writes the
 * double result; counts undecided roundings into *d_amb. */
PMZ_API int pmz_log2_f32_batch(const float *d_x, uint64_t n, double *d_out, uint32_t *d_amb, int variant,
                               void *stream);

/* --- host pipeline helper ---------------------------------------------------- */

/* Pack n blocks of br x bc floats out of a row-major host field (row length
 * `cols`; block i starts at row h_r0[i], column h_c0[i]) into a dense host
 * array, block i at h_dst + i * br * bc, on `nthreads` host threads.  The
 * host-to-host pipeline (hostpipe.py) packs the validation blocks of
 * sample_blocks / split_validation this way into pinned
 * memory and uploads them as one copy, so m and the codebook exist before the
 * field's slabs are encoded.  Replaces nothing in the reference (numpy fancy
 * indexing on the host). */
PMZ_API int pmz_pack_blocks_host(const float *h_field, int64_t cols, int32_t br, int32_t bc, const int64_t *h_r0,
                                 const int64_t *h_c0, int64_t n, float *h_dst, int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif /* PERMEZ_B200_H */
