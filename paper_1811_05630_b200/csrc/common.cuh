// common.cuh -- shared device definitions of the B200 QCB1 codec / engine.
//
// Numeric discipline: every floating-point operation that
// must match the reference bit-for-bit is spelled with the _rn intrinsics so
// no FMA contraction can occur; the library is additionally compiled with
// --fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qcb {

// Programmatic Dependent Launch (host: launch_k): wait until the previous
// kernel of the stream has completed and its writes are visible, then let
// the next kernel be scheduled as this one drains.  No-ops without PDL.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// codec.cpp:32-40
constexpr uint32_t kOutlierSym = 0;
constexpr uint32_t kMinRunLen = 5; // kMinRunRepeats + 1
constexpr int kMaxCodeLen = 57;
constexpr uint32_t kHeaderBytes = 40;

// Encoder tiling.
constexpr int kTile = 1024;          // elements per encoder tile
constexpr int kTileLog2 = 10;
static_assert((1 << kTileLog2) == kTile, "tile size");
constexpr int kEncThreads = 256;     // threads per encoder block
constexpr int kPerThread = kTile / kEncThreads;
// Symbol window histogrammed in shared memory: m in [-kWin/2, kWin/2).
constexpr int kWin = 8192;
// Decoder LUT width (codes up to kLutBits long are resolved in one probe).
constexpr int kLutBits = 11;

// Checkpoint of the decoder state at element e.  Written
// by the encoder next to every block it produces; lets the next decode run
// chunk-parallel while staying bit-exact.
struct IndexRec {
    double dprev;       // exact d[e-1] (prediction input), 0.0 at e = 0
    double dprev2;      // exact d[e-2] (linear predictor)
    uint64_t bitpos;    // stream bit position of the next token to read
    uint32_t run_left;  // elements of the current RUN still to emit
    uint32_t ocur;      // outlier records consumed before e
    uint32_t last_lit;  // last literal symbol (RUN symbol = none yet)
    uint32_t tok;       // token index of `bitpos` (encoder bookkeeping)
};
static_assert(sizeof(IndexRec) == 40, "IndexRec layout");

// Decode index stored next to its block: the block's arena
// slot is [QCB1 block | pad to 16 | IndexRec x nrec].  Record k (k >= 1,
// stored at k - 1) is the encoder's decoder state at the first fine
// checkpoint (a multiple of 2^log2Cmin elements) whose stream position is at
// least k * B bits, with its element index in `tok`; chunk k of the decoder
// runs from record k to record k + 1 (chunk 0 from the initial state).  So
// every chunk carries about B bits of tokens -- decode work is balanced by
// tokens, not by elements, and long constant runs cost nothing.  B = 4096
// bits, doubled until nrec fits the fine checkpoints; nrec follows from the
// block size alone, so the encoder (which knows the exact block size before
// packing) and any decoder agree without extra metadata, and the index is
// <= 40 B per 512 block bytes = 7.8% of the block.  Records past the end of
// the stream are end markers (empty chunks).  The QCB1 bytes are untouched.
constexpr uint64_t kIdxBlockBytesPerChunk = 512;
// (QCSIM_IDX_BPC overrides it for experiments; set once per device before
// any kernel runs -- encoder and decoder must agree)
__device__ uint64_t d_idx_bpc = kIdxBlockBytesPerChunk;
inline uint64_t h_idx_bpc = kIdxBlockBytesPerChunk;
// log2 of the record spacing in bytes of block (record k sits at k * 8 *
// 2^shift bits of stream)
__host__ __device__ __forceinline__ int index_shift(uint64_t n, uint64_t block_bytes, int log2Cmin) {
#ifdef __CUDA_ARCH__
    const uint64_t bpc = d_idx_bpc;
#else
    const uint64_t bpc = h_idx_bpc;
#endif
    const uint64_t fine = (n + (1ull << log2Cmin) - 1) >> log2Cmin; // fine checkpoints (incl. element 0)
    int sh = 0;
    while ((1ull << sh) < bpc) ++sh;
    while (sh < 62 && (block_bytes >> sh) > fine - 1) ++sh;
    return sh;
}
__host__ __device__ __forceinline__ uint64_t index_records(uint64_t n, uint64_t block_bytes, int log2Cmin) {
    return block_bytes >> index_shift(n, block_bytes, log2Cmin);
}
// byte offset of the index records of the block at `blk_off` (slot-relative
// arithmetic: slots start 16-byte aligned)
__host__ __device__ __forceinline__ uint64_t index_offset(uint64_t blk_off, uint64_t block_bytes) {
    return (blk_off + block_bytes + 15) & ~15ull;
}

// Per-plane codec parameters resolved on the device.
struct PlaneParams {
    double eb;       // effective absolute bound
    double q;        // 2.0 * eb
    double inv_q;    // RN(1/q) -- speculation only, never trusted
    uint32_t flags;  // kFlag*
    uint32_t pad;
};
enum : uint32_t {
    kFlagFallback = 1u,  // fast path refuted -> serial re-encode
    kFlagDone = 2u,
    kFlagError = 4u,
};

template <class T> __host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <class T> __host__ __device__ __forceinline__ T tmax(T a, T b) { return a < b ? b : a; }

// ---------------------------------------------------------- fp helpers
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ uint64_t bits_of(double d) { return (uint64_t)__double_as_longlong(d); }

// std::llround for |r| < 2^52 (round half away from zero), exact.
__device__ __forceinline__ long long llround_exact(double r) {
    double t = trunc(r);
    double f = dsub(r, t); // exact for |r| < 2^52
    long long m = (long long)t;
    if (f >= 0.5) m += 1;
    else if (f <= -0.5) m -= 1;
    return m;
}

// Closed-loop quantizer decision, codec.cpp:440-451 verbatim in order of
// operations.  eb > 0.  Returns the symbol (0 = outlier) and the
// reconstruction (undefined for outliers).  Uses a reciprocal estimate and
// falls back to IEEE division only when the estimate could round
// differently (near a half-integer or near the +-H window edge).
__device__ __forceinline__ uint32_t quantize(double x, double pred, double q, double inv_q,
                                             double eb, long long half, double *rec_out) {
    double diff = dsub(x, pred);
    double r = dmul(diff, inv_q);
    double ar = fabs(r);
    double fr = fabs(dsub(ar, trunc(ar)));
    double hh = (double)half;
    bool risky = !(fabs(dsub(fr, 0.5)) > 1e-9 * (ar + 1.0)) || !(fabs(dsub(ar, hh)) > 1e-9 * hh) ||
                 !isfinite(r) || !isfinite(inv_q);
    if (risky) r = ddiv(diff, q);
    uint32_t sym = kOutlierSym;
    if (isfinite(r) && fabs(r) < hh) {
        long long m = llround_exact(r);
        if (m > -half && m < half) {
            double rec = dadd(pred, dmul(q, (double)m));
            if (isfinite(rec) && fabs(dsub(x, rec)) <= eb) {
                sym = (uint32_t)(m + half);
                *rec_out = rec;
            }
        }
    }
    return sym;
}

// Linear extrapolation prediction (codec.cpp:306): 2.0*d[i-1] - d[i-2].
__device__ __forceinline__ double predict_linear(double d1, double d2) { return dsub(dmul(2.0, d1), d2); }

// ---------------------------------------------------- gate arithmetic
// DESIGN.md §3 (identical in oracle/qcsim_oracle.c): complex products
// (a+bi)(c+di) = (ac - bd) + (ad + bc)i, factor/matrix entry on the left.
__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double &cr, double &ci) {
    double t1 = dmul(ar, br), t2 = dmul(ai, bi), t3 = dmul(ar, bi), t4 = dmul(ai, br);
    cr = dsub(t1, t2);
    ci = dadd(t3, t4);
}

// Gate action in device-friendly form (mirrors qcsim_action).
struct DevAction {
    uint32_t kind; // 0 diag, 1 butterfly, 2 swap
    int32_t target, a, b;
    uint64_t mask;
    double f[2];
    double u[8];
};

// ------------------------------------------------------ bit utilities
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }
__host__ __device__ __forceinline__ int bit_width64(uint64_t v) {
#ifdef __CUDA_ARCH__
    return v ? 64 - __clzll((long long)v) : 0;
#else
    return v ? 64 - __builtin_clzll(v) : 0;
#endif
}

} // namespace qcb
