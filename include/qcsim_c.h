/*
 * qcsim_c.h -- C-ABI of the B200 compressed state-vector update path.
 *
 * This is the drop-in boundary for the hot loop of arXiv:1811.05630
 * (Algorithm 1): per gate, per slice -- decompress,
 * normalize, apply gate, recompress with the error-bounded "QCB1" codec.
 * Every entry point below replaces one declaration of the reference C++ API
 * under /root/reference/proj/include/qcsim/ (cited per function); the C++
 * shim in include/qcsim/ (*.hpp) rethrows the status codes as the reference's
 * exception types, so C++ callers see the reference behaviour unchanged.
 *
 * Conventions
 *   - plain pointers + sizes, no C++ or torch types;
 *   - every call returns a qcsim_status; on failure the message is available
 *     from qcsim_last_error() (thread-local, valid until the next failing
 *     call on the same thread);
 *   - "host" entry points take host buffers; "_device" entry points take
 *     device pointers and a cudaStream_t passed as void*.
 */
#ifndef QCSIM_C_H
#define QCSIM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exception taxonomy (errors.hpp:24-51). */
typedef enum qcsim_status {
    QCSIM_OK = 0,
    QCSIM_INVALID_ARGUMENT = 1, /* std::invalid_argument                  */
    QCSIM_CODEC = 2,            /* qcsim::CodecError (errors.hpp:24-27)    */
    QCSIM_CAPACITY = 3,         /* qcsim::CapacityError (errors.hpp:42-45) */
    QCSIM_PARSE = 4,            /* qcsim::ParseError (errors.hpp:30-39)    */
    QCSIM_NUMERIC = 5,          /* qcsim::NumericError (errors.hpp:48-51)  */
    QCSIM_CUDA = 6,             /* CUDA runtime failure (no ref analogue)  */
    QCSIM_NOMEM = 7,            /* allocation failure (std::bad_alloc)     */
    QCSIM_RUNTIME = 8           /* std::runtime_error (dump I/O)           */
} qcsim_status;

/* Message of the last failing call on this thread ("" if none). */
const char *qcsim_last_error(void);

/* Library identification: "qcsim-b200 <version> sm_100a". */
const char *qcsim_version(void);

/* ------------------------------------------------------------------------
 * Codec (codec.hpp:41-108)
 * ---------------------------------------------------------------------- */

/* CodecMode values (codec.hpp:41-45) and Predictor values (codec.hpp:47-50). */
enum { QCSIM_MODE_RANGE_RELATIVE = 0, QCSIM_MODE_ABSOLUTE = 1, QCSIM_MODE_LOSSLESS = 2 };
enum { QCSIM_PRED_PREVIOUS = 0, QCSIM_PRED_LINEAR = 1 };

/* CodecConfig (codec.hpp:52-60); defaults RangeRelative / 0.01 / 16 / Previous. */
typedef struct qcsim_codec_config {
    uint8_t mode;
    uint8_t predictor;
    uint16_t reserved;
    int32_t quant_code_bits; /* [4, 24] */
    double bound;
} qcsim_codec_config;

/* CodecStats (codec.hpp:89-94). */
typedef struct qcsim_codec_stats {
    uint64_t input_bytes;
    uint64_t output_bytes;
    double ratio;
    double outlier_fraction;
} qcsim_codec_stats;

/* CodecConfig::validate (codec.hpp:59, codec.cpp:331-341). */
qcsim_status qcsim_codec_validate(const qcsim_codec_config *cfg);

/* Upper bound of the serialized block size for an n-element plane. */
uint64_t qcsim_block_bound(uint64_t n, int32_t quant_code_bits);

/* compress_plane + CompressedBlock::to_bytes (codec.hpp:81,98-99;
 * codec.cpp:359-364,410-533).  Runs on the GPU: uploads `values`, encodes,
 * downloads the QCB1 bytes, byte-identical to the reference. */
qcsim_status qcsim_compress_plane(const double *values, uint64_t n,
                                  const qcsim_codec_config *cfg, uint8_t *out,
                                  uint64_t capacity, uint64_t *out_len,
                                  qcsim_codec_stats *stats);

/* CompressedBlock::from_bytes + decompress_plane (codec.hpp:85-86,103;
 * codec.cpp:366-408,535-633).  Runs on the GPU.  `*consumed` (optional)
 * receives the bytes of the block that was parsed. */
qcsim_status qcsim_decompress_plane(const uint8_t *block, uint64_t len,
                                    double *out, uint64_t capacity,
                                    uint64_t *n_out, uint64_t *consumed);

/* Batched, device-resident codec.  Plane p has n[p] doubles at values[p]
 * (device pointers).  Encode writes each block at out + offsets[p] where
 * offsets are chosen by the library (exclusive scan of exact sizes) and
 * returned in `offsets_host` (planes+1 entries; offsets_host[planes] is the
 * total).  `out` must hold `capacity` bytes. */
qcsim_status qcsim_compress_planes_device(const double *const *values,
                                          const uint64_t *n, uint32_t planes,
                                          const qcsim_codec_config *cfg,
                                          uint8_t *out, uint64_t capacity,
                                          uint64_t *offsets_host,
                                          qcsim_codec_stats *stats_host,
                                          void *stream);
qcsim_status qcsim_decompress_planes_device(const uint8_t *blocks,
                                            const uint64_t *offsets_host,
                                            uint32_t planes,
                                            double *const *out,
                                            const uint64_t *capacity,
                                            void *stream);

/* ------------------------------------------------------------------------
 * Gate actions (circuit.hpp:122-153): the flattened GateAction variant.
 * ---------------------------------------------------------------------- */
enum { QCSIM_ACTION_DIAGONAL = 0, QCSIM_ACTION_BUTTERFLY = 1, QCSIM_ACTION_SWAP = 2 };

typedef struct qcsim_action {
    uint32_t kind;     /* QCSIM_ACTION_*                                  */
    int32_t target;    /* ButterflyOp::target                             */
    int32_t a, b;      /* SwapOp::a, SwapOp::b                            */
    uint32_t reserved;
    uint64_t mask;     /* DiagonalOp::mask or ButterflyOp::control_mask   */
    double factor[2];  /* DiagonalOp::factor (re, im)                     */
    double u[8];       /* ButterflyOp::u: u00 re,im, u01, u10, u11        */
} qcsim_action;

/* ------------------------------------------------------------------------
 * Engine (the reference ships no engine source).
 * ---------------------------------------------------------------------- */
typedef struct qcsim_engine qcsim_engine;

/* EngineConfig. norm_every: 0 = off, 1 = every gate,
 * k = every k-th gate.  slice_bits < 0 selects default_slice_bits(n)
 * (statevec.hpp:50-53). */
typedef struct qcsim_engine_config {
    int32_t num_qubits;
    int32_t slice_bits;
    qcsim_codec_config codec;
    int32_t compression_enabled;
    int32_t norm_every;
    double norm_drift_tolerance; /* default 0.02 */
    int32_t device;              /* CUDA ordinal                         */
    int32_t rank;                /* slice shard: this rank owns slices   */
    int32_t world;               /*   [rank*S/world, (rank+1)*S/world)   */
    int32_t checkpoint_bits;     /* decode index granularity, 0 = auto   */
    uint64_t wave_bytes;         /* dense working-set budget of a gate   */
                                 /* pass (slices are processed in waves  */
                                 /* that fit it); 0 = 45% of the device  */
} qcsim_engine_config;

/* RunMetrics, accumulated over every compress call. */
typedef struct qcsim_run_metrics {
    double min_compression_ratio;
    double mean_compression_ratio;
    double wall_seconds;           /* device time of the gate passes      */
    double final_norm;             /* sum of per-slice sq_norm at the end */
    uint64_t compress_calls;
    uint64_t gates;
    uint64_t peak_compressed_bytes;
    uint64_t dense_bytes;          /* 2^(n+4)                             */
    uint64_t current_compressed_bytes;
    uint64_t index_bytes;          /* side index (not part of the ratio)  */
    uint64_t fallback_planes;      /* planes re-encoded on the serial path */
    uint64_t kernel_launches;      /* kernels launched by run()           */
} qcsim_run_metrics;

/* Per-gate row of RunMetrics (SPEC.md:310 per_gate_min_ratio; the CSV
 * report's gate_index, min_ratio, mean_ratio, seconds): one row
 * per compression pass since the last load -- row 0 is the load's initial
 * compression, row k the state after gate k-1 of the loaded state.
 * compressed_bytes / index_bytes: the state's QCB1 bytes and decode-index
 * bytes after that pass.  Compression-off engines report ratio 0. */
typedef struct qcsim_gate_metrics {
    double min_ratio;
    double mean_ratio;
    double seconds;             /* device time of the pass                 */
    uint64_t compressed_bytes;
    uint64_t index_bytes;
    uint64_t compress_calls;
} qcsim_gate_metrics;

/* Layout of an engine's gate pass: its local slices are processed in
 * `waves` batches of `wave_slices` slices (the dense working set is
 * O(wave), sized by qcsim_engine_config.wave_bytes). */
typedef struct qcsim_engine_info_t {
    uint64_t local_slices;
    uint64_t wave_slices;
    uint64_t waves;
    int32_t checkpoint_bits;
    int32_t reserved;
} qcsim_engine_info_t;

qcsim_status qcsim_engine_create(const qcsim_engine_config *cfg,
                                 qcsim_engine **out);
qcsim_status qcsim_engine_destroy(qcsim_engine *eng);

/* init_basis_state (statevec.hpp:118-119) followed by the initial
 * compression of every slice. */
qcsim_status qcsim_engine_load_basis(qcsim_engine *eng, uint64_t basis_index);

/* state_from_amplitudes (statevec.hpp:122-124): `amps` holds 2^n
 * interleaved (re, im) pairs in global index order (host memory). Sharded
 * engines read only their own slices. */
qcsim_status qcsim_engine_load_amplitudes(qcsim_engine *eng,
                                          const double *amps, uint64_t count);

/* Gate passes: applies `count` actions in order.
 * Metrics accumulate across calls; `metrics` (optional) receives the totals. */
qcsim_status qcsim_engine_run(qcsim_engine *eng, const qcsim_action *actions,
                              uint64_t count, qcsim_run_metrics *metrics);

/* Per-gate rows since the last load (pass rows = NULL to query `*count`). */
qcsim_status qcsim_engine_gate_metrics(qcsim_engine *eng, qcsim_gate_metrics *rows,
                                       uint64_t capacity, uint64_t *count);

/* Wave layout of the engine (see qcsim_engine_info_t). */
qcsim_status qcsim_engine_info(qcsim_engine *eng, qcsim_engine_info_t *info);

/* Releases the engine's gate-pass scratch (encoder buffers, decoded planes,
 * the idle arena); the compressed state stays.  The next pass re-allocates. */
qcsim_status qcsim_engine_trim(qcsim_engine *eng);

/* Device bytes held by the library's buffers: current and the high-water
 * mark (reset to the current value when reset_peak != 0). */
qcsim_status qcsim_device_memory(uint64_t *current, uint64_t *peak,
                                 int32_t reset_peak);

/* to_amplitudes / gather_state (statevec.hpp:128-129):
 * interleaved (re, im) of this rank's slices into host memory. Guarded by
 * `guard_qubits` (CapacityError). */
qcsim_status qcsim_engine_gather(qcsim_engine *eng, double *amps,
                                 uint64_t capacity, int32_t guard_qubits);

/* On-device comparison of two engines' current states (same qubits, slice
 * size and rank layout), e.g. a compressed run against a compression-off
 * FP64 run of the same circuit: max |a_k - b_k| over every amplitude, the
 * inner product <a|b> (statevec.hpp:83, conj(a).b), both squared norms and
 * fidelity = |<a|b>|^2 (statevec.hpp:84).  Sums are fixed pairwise trees. */
typedef struct qcsim_compare_result {
    double max_abs_diff;
    double inner_re, inner_im;
    double norm_a, norm_b;
    double fidelity;
} qcsim_compare_result;
qcsim_status qcsim_engine_compare(qcsim_engine *a, qcsim_engine *b,
                                  qcsim_compare_result *out);

/* Per-slice sq_norm cache (statevec.hpp:72) of this rank's slices. */
qcsim_status qcsim_engine_slice_norms(qcsim_engine *eng, double *out,
                                      uint64_t capacity);

/* Compressed state as QCB1 blocks (checkpoint): plane order is
 * slice-major (re, im).  Pass out = NULL to query `*len`. */
qcsim_status qcsim_engine_export_blocks(qcsim_engine *eng, uint8_t *out,
                                        uint64_t capacity, uint64_t *len,
                                        uint64_t *offsets, uint64_t offsets_cap);

/* Resume from a checkpoint (CompressedBlock::from_bytes,
 * codec.cpp:366-408): `blocks` holds this rank's 2 * local_slices QCB1 blocks
 * in export_blocks order (host bytes), offsets[planes + 1] their starts;
 * `sq_norms` is the table of EVERY slice's cached sq_norm (2^(n-s) doubles,
 * statevec.hpp:72) and `gates_done` the number of gates already applied (it
 * continues the gate numbering of norm_every and the drift message).  Every
 * block goes through the from_bytes / decompress_plane checks (CodecError
 * with the reference's message) and must match the engine's codec (mode,
 * predictor, quant_code_bits, element count).  The state is rebuilt wave by
 * wave on the device (decode -> the engine's own encoder, which reproduces
 * the block bytes and adds the decode index); a block that does not
 * re-encode to its own size is rejected (QCSIM_CODEC).  Absolute and
 * Lossless bounds only (a RangeRelative bound depends on the pre-compression
 * range, which a block does not carry). */
qcsim_status qcsim_engine_load_blocks(qcsim_engine *eng, const uint8_t *blocks,
                                      uint64_t len, const uint64_t *offsets,
                                      uint64_t planes, const double *sq_norms,
                                      uint64_t norm_count, uint64_t gates_done);

/* Multi-rank hooks (slice sharding).  A gate whose
 * butterfly/swap partner slice lives on another rank needs that slice's
 * compressed planes: `exchange_plan` lists (local slice, remote slice)
 * pairs for an action; the caller ships the blocks (export/import) over
 * its transport (NCCL / gloo) and passes them in before `run`. */
qcsim_status qcsim_engine_partner_blocks_needed(qcsim_engine *eng,
                                                const qcsim_action *action,
                                                uint64_t *remote_slices,
                                                uint64_t capacity,
                                                uint64_t *count);
qcsim_status qcsim_engine_export_slice(qcsim_engine *eng, uint64_t slice,
                                       uint8_t *out, uint64_t capacity,
                                       uint64_t *len);
/* Batched export_slice: the (re, im) blocks of `count` owned slices,
 * concatenated in the given order (one device gather, one copy to host);
 * offsets[k] = start of slice k, offsets[count] = total. */
qcsim_status qcsim_engine_export_slices(qcsim_engine *eng, const uint64_t *slices,
                                        uint64_t count, uint8_t *out,
                                        uint64_t capacity, uint64_t *len,
                                        uint64_t *offsets);
/* Device-direct exchange (NCCL/P2P on device buffers, no host staging):
 * export_slices_device gathers the (re, im) blocks of owned slices into a
 * caller-owned DEVICE buffer (out = NULL: query `*len`); plane_offsets (host,
 * 2*count+1 entries) receives each plane's start.  import_partners_device
 * registers partner slices held in a device buffer (same layout) for the
 * next run(); the buffer must stay valid until run() returns.  Imported
 * blocks are validated on the device (from_bytes + decoder checks). */
qcsim_status qcsim_engine_export_slices_device(qcsim_engine *eng,
                                               const uint64_t *slices,
                                               uint64_t count, void *out,
                                               uint64_t capacity, uint64_t *len,
                                               uint64_t *plane_offsets);
qcsim_status qcsim_engine_import_partners_device(qcsim_engine *eng,
                                                 const uint64_t *slices,
                                                 uint64_t count,
                                                 const void *blocks,
                                                 const uint64_t *plane_offsets);
qcsim_status qcsim_engine_import_partner(qcsim_engine *eng, uint64_t slice,
                                         const uint8_t *blocks, uint64_t len);
/* Replace the norm source with an all-gathered table of every slice's
 * sq_norm (2^(n-s) doubles, slice order) for the next gate. */
qcsim_status qcsim_engine_set_global_norms(qcsim_engine *eng,
                                           const double *norms,
                                           uint64_t count);

#ifdef __cplusplus
}
#endif

#endif /* QCSIM_C_H */
