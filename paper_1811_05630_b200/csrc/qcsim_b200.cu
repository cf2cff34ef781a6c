// qcsim_b200.cu -- host side of the B200 compressed state-vector update
// path: codec batch drivers, the engine (Algorithm 1) and
// the C-ABI declared in include/qcsim_c.h.
//
// Built for sm_100a only, with --fmad=false.  There is no CPU
// fallback: every compute path below launches the kernels in *_kernels.cuh;
// without a CUDA device every entry point fails with QCSIM_CUDA.
#include <algorithm>
#include <array>
#include <cfloat>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "../../include/qcsim_c.h"
#include "common.cuh"
#include "decode_kernels.cuh"
#include "foreign_kernels.cuh"
#include "enc_tiles.cuh"
#include "sources.cuh"
#include "misc_kernels.cuh"
#include "pack_kernels.cuh"

#define QCSIM_VERSION "qcsim-b200 0.1.0 sm_100a"

using namespace qcb;

namespace {

thread_local std::string g_err;

struct Fail {
    qcsim_status st;
    std::string msg;
};

[[noreturn]] void raise(qcsim_status st, std::string msg) { throw Fail{st, std::move(msg)}; }

void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess) raise(QCSIM_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

template <class F> qcsim_status guarded(F &&f) {
    try {
        f();
        return QCSIM_OK;
    } catch (const Fail &e) {
        g_err = e.msg;
        return e.st;
    } catch (const std::bad_alloc &) {
        g_err = "out of memory";
        return QCSIM_NOMEM;
    } catch (const std::exception &e) {
        g_err = e.what();
        return QCSIM_RUNTIME;
    }
}

// Device bytes held by this library's buffers (peak: high-water mark since
// the last qcsim_device_memory reset).
uint64_t g_dev_cur = 0, g_dev_peak = 0;

// Grow-only device buffer (contents are not preserved on growth).
template <class T> struct DBuf {
    T *p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) {
            cudaFree(p);
            g_dev_cur -= cap * sizeof(T);
        }
        p = nullptr;
        cap = 0;
    }
    // returns true when (re)allocated
    bool ensure(size_t n, bool zero = false) {
        if (n <= cap && p) return false;
        release();
        size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&p, want * sizeof(T));
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            raise(QCSIM_NOMEM, "device allocation of " + std::to_string(want * sizeof(T)) + " bytes failed");
        }
        cap = want;
        g_dev_cur += cap * sizeof(T);
        g_dev_peak = std::max(g_dev_peak, g_dev_cur);
        if (zero) CK(cudaMemset(p, 0, want * sizeof(T)));
        return true;
    }
    void swap(DBuf &o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
};

int g_device_checked = -1;
void ensure_device(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        raise(QCSIM_CUDA, "no CUDA device available (qcsim-b200 has no CPU fallback)");
    }
    if (dev < 0 || dev >= n) raise(QCSIM_INVALID_ARGUMENT, "CUDA device ordinal out of range");
    CK(cudaSetDevice(dev));
    if (g_device_checked != dev) {
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dev));
        if (prop.major != 10) raise(QCSIM_CUDA, std::string("device is not sm_100 (Blackwell): ") + prop.name);
        g_device_checked = dev;
        static uint64_t bpc_set = 0; // per-device bitmask
        if (const char *v = std::getenv("QCSIM_IDX_BPC"); v && !(bpc_set & (1ull << dev))) {
            h_idx_bpc = std::max<uint64_t>(1, std::strtoull(v, nullptr, 10));
            CK(cudaMemcpyToSymbol(d_idx_bpc, &h_idx_bpc, sizeof h_idx_bpc));
            bpc_set |= 1ull << dev;
        }

    }
}

uint64_t g_launches = 0; // kernels launched by this library (per process)

// Optional per-kernel timing with CUDA events on the launching stream
// (bench.py reads it through qcsim_profile_read).  Pending event pairs are
// resolved at the synchronisation points the pipeline already has.
struct Profiler {
    bool on = false;
    struct Pend {
        const char *name;
        cudaEvent_t a, b;
    };
    std::vector<Pend> pend;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, std::pair<double, uint64_t>>> acc;
    cudaEvent_t get() {
        if (pool.empty()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    void add(const char *name, double ms) {
        for (auto &kv : acc)
            if (kv.first == name) {
                kv.second.first += ms;
                kv.second.second += 1;
                return;
            }
        acc.push_back({name, {ms, 1}});
    }
    void flush() {
        for (auto &p : pend) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) add(p.name, ms);
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pend.clear();
    }
};
Profiler g_prof;

struct ProfScope {
    const char *name;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(const char *n, cudaStream_t s) : name(n), st(s) {
        ++g_launches;
        if (g_prof.on) {
            a = g_prof.get();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() noexcept(false) {
        if (a) {
            cudaEvent_t b = g_prof.get();
            cudaEventRecord(b, st);
            g_prof.pend.push_back({name, a, b});
        }
        // QCSIM_DEBUG_SYNC=1: synchronise after every kernel and name the
        // one that failed (fault localisation without compute-sanitizer)
        static const bool dbg = [] {
            const char *v = std::getenv("QCSIM_DEBUG_SYNC");
            return v && v[0] == '1';
        }();
        if (dbg) {
            cudaError_t e = cudaStreamSynchronize(st);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) raise(QCSIM_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
        }
    }
};
#define PROF(name, st) ProfScope _prof_scope(name, st)

void validate_codec(const qcsim_codec_config &c) { // codec.cpp:331-341
    if (c.quant_code_bits < 4 || c.quant_code_bits > 24)
        raise(QCSIM_INVALID_ARGUMENT, "quant_code_bits must be in [4, 24]");
    if (c.mode > 2) raise(QCSIM_INVALID_ARGUMENT, "unknown codec mode");
    if (c.predictor > 1) raise(QCSIM_INVALID_ARGUMENT, "unknown predictor");
    if (c.mode != QCSIM_MODE_LOSSLESS) {
        if (!(c.bound > 0.0) || !std::isfinite(c.bound)) raise(QCSIM_INVALID_ARGUMENT, "error bound must be positive");
        if (c.mode == QCSIM_MODE_RANGE_RELATIVE && c.bound > 1.0)
            raise(QCSIM_INVALID_ARGUMENT, "range-relative bound must not exceed 1");
    }
}

int auto_log2C(uint64_t L) {
    int s = 0;
    while ((1ull << s) < L) ++s;
    static const int delta = std::getenv("QCSIM_CKPT_SHIFT") ? std::atoi(std::getenv("QCSIM_CKPT_SHIFT")) : 9; // (tuning)
    return std::max(5, std::min(10, s - delta)); // 2^14 planes: 512 chunks of 32 (s - 8 / s - 10 measured slower)
}

// Grow-only pinned host buffer.
template <class T> struct HBuf {
    T *p = nullptr;
    size_t cap = 0;
    HBuf() = default;
    HBuf(const HBuf &) = delete;
    HBuf &operator=(const HBuf &) = delete;
    ~HBuf() {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t n) {
        if (n <= cap && p) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        if (cudaHostAlloc((void **)&p, std::max<size_t>(n, 1) * sizeof(T), cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            raise(QCSIM_NOMEM, "pinned host allocation failed");
        }
        cap = std::max<size_t>(n, 1);
    }
};

// ------------------------------------------------------------ encoder
struct EncScratch {
    DBuf<PlaneParams> params;
    DBuf<double> x, dval, evc, oval, tilesum;
    DBuf<uint32_t> sym, evlist, opos, ocount, ntok, tsym, trep, hist, hspecial, symrange, nsym, err, nonfinite;
    DBuf<uint8_t> fl, cb_len, cub_tmp;
    DBuf<uint8_t> zx, ztriv; // run-aware tile flags (TileArgs), planes of many tiles
    DBuf<uint32_t> chain_prog; // enc_chain's per-plane front (enc_verify follows it)
    DBuf<uint32_t> lat_bad, lat_redo; // enc_gate_lattice: per-plane range flag, planes for enc_lattice to redo
    DBuf<int32_t> t_lastout, t_base, t_nev, t_evoff, t_firstb, t_lastb, t_nout, t_ooff, t_prevb, t_nextb, t_ntok,
        t_tokoff, t_cbits, t_coff;
    DBuf<unsigned long long> gamma;
    DBuf<uint64_t> cb_cnt, cb_code, cb_key, cb_ncnt, stream_bits, block_bytes, slot_bytes, slot_off, blk_off;
    DBuf<uint32_t> cb_sym;
    DBuf<int32_t> cb_parent;
    DBuf<uint32_t> overflow;
    DBuf<double> evD;
    DBuf<unsigned long long> lb; // enc_lattice event-offset look-back
    uint32_t lb_epoch = 0;
    DBuf<double> chain_carry; // enc_chain_scan chunk hand-off
    DBuf<double> chain_tcarry;   // tentative chunk values (from the maps)
    DBuf<uint32_t> chain_tflag;
    DBuf<uint32_t> chain_cnt, chain_done; // per-plane chain completion (enc_verify overlap)
    DBuf<uint32_t> ver_cnt, ver_done, ser_done; // per-plane verify / serial completion (tok_count overlap)
    uint32_t flow_epoch = 0;
    DBuf<uint32_t> chain_flag;
    uint32_t chain_epoch = 0;
    HBuf<uint64_t> h_bytes, h_off, h_misc;
    HBuf<PlaneParams> h_params;
    HBuf<uint32_t> h_err;
    PackArgs pack{};
    uint64_t planes = 0;
    uint64_t hist_stride = 0;
    uint64_t param_planes = 0;       // params valid for this many planes ...
    qcsim_codec_config param_cfg{};  // ... under this config
    DecTables dec_out{};             // where enc_codebook writes decode tables (optional)
    EngineDevStats *stats_out = nullptr; // deferred engine: run metrics fused into the slot scan
    uint64_t *blk_off_out = nullptr;     // deferred engine: the packer writes block offsets here directly
    uint64_t fixed_W = 0;                // deferred engine: plane p's slot at p * fixed_W (no slot scan)
    uint64_t fixed_planes = 0, fixed_at = 0;
    DBuf<uint64_t> fixed_off;
    bool pack_dense_hint = false;        // the state being re-encoded averages > 160 KB per plane
    DBuf<unsigned long long> pack_lb;    // pack_write look-back slots [plane][chunk]
    uint32_t pack_lb_epoch = 0;
    unsigned long long stats_gate = 0;
    uint64_t arena_base = 0;             // this batch's slots start here in the arena (earlier waves before it)
    GateRowDev *rows_out = nullptr;      // deferred engine: per-gate rows (slot_scan_stats)
    unsigned long long row0 = 0, nrows = 0;

    void ensure(uint64_t planes, uint64_t units, uint64_t L, int qb) {
        const uint64_t ntiles = (L + kTile - 1) / kTile;
        const uint64_t rsym1 = (1ull << qb) + 1;
        const uint64_t cap = std::min<uint64_t>(L + 1, rsym1);
        params.ensure(planes);
        x.ensure(planes * L);
        dval.ensure(planes * L);
        evc.ensure(planes * L + 8);       // TMA chunks round up to 16 bytes
        evlist.ensure(planes * L + 8);
        sym.ensure(planes * L);
        fl.ensure(planes * L);
        opos.ensure(planes * L);
        oval.ensure(planes * L);
        ocount.ensure(planes);
        tilesum.ensure(units * ntiles);
        tsym.ensure(planes * (L + 1));
        trep.ensure(planes * (L + 1));
        ntok.ensure(planes);
        for (DBuf<int32_t> *b : {&t_lastout, &t_base, &t_nev, &t_evoff, &t_firstb, &t_lastb, &t_nout, &t_ooff,
                                 &t_prevb, &t_nextb, &t_ntok, &t_tokoff, &t_cbits, &t_coff})
            b->ensure(planes * (ntiles + 2));
        // the dense histogram must be all-zero between uses (E3 re-zeroes)
        if (hist_stride != rsym1 || hist.cap < planes * rsym1) {
            hist.ensure(planes * rsym1);
            CK(cudaMemset(hist.p, 0, hist.cap * sizeof(uint32_t)));
            hist_stride = rsym1;
        }
        hspecial.ensure(2 * planes);
        symrange.ensure(2 * planes);
        gamma.ensure(planes);
        cb_sym.ensure(planes * cap);
        cb_cnt.ensure(planes * cap);
        cb_len.ensure(planes * cap);
        cb_code.ensure(planes * cap);
        cb_key.ensure(planes * cap * 2);
        cb_ncnt.ensure(planes * cap * 2);
        cb_parent.ensure(planes * cap * 2);
        nsym.ensure(planes);
        stream_bits.ensure(planes);
        block_bytes.ensure(planes);
        slot_bytes.ensure(planes);
        slot_off.ensure(planes + 1);
        blk_off.ensure(planes);
        err.ensure(planes);
        nonfinite.ensure(1);
        overflow.ensure(1);
    }
};

// enc_chain_scan counters: [0] resolve points, [1] refuted chunks redone
// serially, [4] chunks run serially because the maps did not fit
constexpr uint64_t kScanChainMaxPlanes = 256; // more planes fill the GPU with serial warps
constexpr int kMaxDevices = 64;
int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    if (dev < 0 || dev >= kMaxDevices) raise(QCSIM_CUDA, "device ordinal beyond the library's table");
    return dev;
}
// per-device counters (the buffer lives on the device that uses it)
uint32_t *chain_stats() {
    static DBuf<uint32_t> buf[kMaxDevices];
    DBuf<uint32_t> &b = buf[current_device()];
    if (!b.p) {
        b.ensure(16);
        CK(cudaMemset(b.p, 0, 16 * sizeof(uint32_t)));
    }
    return b.p;
}
// kernels needing more than 48 KB of dynamic shared memory: the attribute
// is per device, set once on each
template <class K> void set_smem_once(K kernel, size_t bytes, uint64_t *done_mask, int bit) {
    const int dev = current_device();
    if (done_mask[dev] & (1ull << bit)) return;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done_mask[dev] |= 1ull << bit;
}
uint64_t g_smem_set[kMaxDevices] = {};


// Every kernel launch goes through here: Programmatic Dependent Launch lets
// the next kernel of the stream be scheduled while this one drains (each
// kernel starts with pdl_wait(), so it still sees all of its predecessor's
// writes).  QCSIM_PDL=0 turns it off.
template <class... KArgs, class... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    static const bool pdl = [] {
        const char *v = std::getenv("QCSIM_PDL");
        return !(v && v[0] == '0');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// enc_verify launched alongside the block-parallel chain, waiting per plane
// (QCSIM_CHAIN_OVERLAP=0/1 forces it off/on)
bool chain_overlap(uint64_t planes) {
    static const int env = std::getenv("QCSIM_CHAIN_OVERLAP") ? std::atoi(std::getenv("QCSIM_CHAIN_OVERLAP")) : -1;
    // auto: batches of >= 64 planes (small batches finish faster with
    // grid-wide waits than with polled per-plane flags)
    return env >= 0 ? env != 0 : planes >= 64;
}
// 0 auto, 1 skip (debug), 2 serial warp chain, 3 block-parallel chain
int chain_choice() {
    static const int mode = [] {
        const char *v = std::getenv("QCSIM_CHAIN");
        return v ? std::atoi(v) : 0;
    }();
    return mode;
}
bool chain_scan_selected(uint64_t planes) {
    const int m = chain_choice();
    return m == 3 || (m == 0 && planes <= kScanChainMaxPlanes);
}

template <class K> void set_smem(K kernel, size_t bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

struct EncodeResult {
    std::vector<uint64_t> block_bytes; // per plane
    std::vector<uint64_t> blk_off;     // per plane, offset in the arena
    uint64_t total = 0;                // arena bytes used (incl. padding)
    uint64_t fallback = 0;
};

void launch_plane_scan(cudaStream_t st, const int32_t *in, int32_t *out, int ntiles, int planes, ScanKind kind);

// Block assembly: chunk bit counts + plane scan (once per batch), then the
// arena range is zeroed and every (plane, token chunk) writes its bits.
// Re-entrant after an arena overflow (count = false reuses the offsets).
void launch_pack(cudaStream_t st, EncScratch &S, DBuf<uint8_t> &arena, bool count = true) {
    if (!arena.p) arena.ensure(1 << 20);
    PackArgs P = S.pack;
    P.arena = arena.p + S.arena_base;
    P.arena_cap = arena.cap > S.arena_base ? arena.cap - S.arena_base : 0;
    const int nck = (int)((P.L + 1 + kPackTok - 1) / kPackTok);
    // (plane, K) blocks looping over the plane's chunks (pack_count / pack_write)
    const int K = std::min(nck, 32);
    const unsigned grid = (unsigned)(S.planes * K);
    // Chunk bit offsets by decoupled look-back inside pack_write (no counting
    // pass); the slots must be zero (stream words are OR-combined at chunk
    // seams): fixed slots are zeroed by the codebook grid, packed slots by
    // arena_zero over the batch's range.  QCSIM_PACK_COUNT=1: the counting
    // pass + plane scan instead.
    static const int count_env = std::getenv("QCSIM_PACK_COUNT") ? std::atoi(std::getenv("QCSIM_PACK_COUNT")) : -1;
    // (dense states -- hundreds of KB per plane -- pack a little faster with
    // the counting pass: 23.0 vs 25.0 ms per Random-30 pass at 680 MB; sparse
    // ones with the look-back: 5.4 vs 6.1 ms at 130 MB)
    const bool count_pass = count_env >= 0 ? count_env != 0 : S.pack_dense_hint;
    if (S.fixed_W || !count_pass) {
        if (S.pack_lb.ensure(S.planes * nck, /*zero=*/true)) S.pack_lb_epoch = 0;
        if (++S.pack_lb_epoch >= (1u << 29)) {
            CK(cudaMemsetAsync(S.pack_lb.p, 0, S.pack_lb.cap * sizeof(unsigned long long), st));
            S.pack_lb_epoch = 1;
        }
        P.lb = S.pack_lb.p;
        P.lb_epoch = S.pack_lb_epoch;
        if (!S.fixed_W || !count) {
            PROF("arena_zero", st);
            launch_k(arena_zero, 296, 256, 0, st, P.arena, P.arena_cap, S.slot_off.p + S.planes);
        }
    } else if (count) {
        {
            PROF("pack_count", st); // also zeroes the plane slots
            launch_k(pack_count, grid, 256, 0, st, P, (int)S.planes, nck, K, S.t_cbits.p);
        }
        launch_plane_scan(st, S.t_cbits.p, S.t_coff.p, nck, (int)S.planes, kScanSumExcl);
    } else {
        PROF("arena_zero", st); // re-pack after an arena overflow
        launch_k(arena_zero, 296, 256, 0, st, P.arena, P.arena_cap, S.slot_off.p + S.planes);
    }
    {
        PROF("pack_write", st);
        launch_k(pack_write, grid, 256, 0, st, P, (int)S.planes, nck, K, S.t_coff.p, S.t_cbits.p);
    }
    if (P.index) {
        const uint64_t nfine = (P.L + (1ull << P.log2C) - 1) >> P.log2C;
        PROF("index_select", st);
        launch_k(index_select, (unsigned)(S.planes * ((nfine + 255) / 256)), 256, 0, st, P, (int)S.planes);
    }
}

// Synchronous convenience wrapper (codec API).
template <int NP, class Src>
void encode_launch(cudaStream_t st, EncScratch &S, const Src &src, int units, uint64_t L,
                   const qcsim_codec_config &cfg, int log2C, IndexRec *index, DBuf<uint8_t> &arena,
                   bool check_finite, bool sync_now, bool host_results = true);
EncodeResult encode_finish(cudaStream_t st, EncScratch &S, DBuf<uint8_t> &arena);
template <int NP, class Src>
EncodeResult encode_batch(cudaStream_t st, EncScratch &S, const Src &src, int units, uint64_t L,
                          const qcsim_codec_config &cfg, int log2C, IndexRec *index, DBuf<uint8_t> &arena,
                          bool check_finite, bool /*want_offsets*/) {
    encode_launch<NP, Src>(st, S, src, units, L, cfg, log2C, index, arena, check_finite, true);
    return encode_finish(st, S, arena);
}

void launch_plane_scan(cudaStream_t st, const int32_t *in, int32_t *out, int ntiles, int planes, ScanKind kind) {
    if (ntiles <= kInlineTiles) return; // consumers compute the carry inline (carry_of)
    const int out_stride = kind == kScanSumExcl ? ntiles + 1 : ntiles;
    PROF("plane_scan", st);
    if (ntiles <= 256) launch_k(plane_scan<1>, planes, 256, 0, st, in, out, ntiles, planes, kind, ntiles, out_stride);
    else if (ntiles <= 1024) launch_k(plane_scan<4>, planes, 256, 0, st, in, out, ntiles, planes, kind, ntiles, out_stride);
    else if (ntiles <= 4096) launch_k(plane_scan<16>, planes, 256, 0, st, in, out, ntiles, planes, kind, ntiles, out_stride);
    else if (ntiles <= 8192) launch_k(plane_scan<32>, planes, 256, 0, st, in, out, ntiles, planes, kind, ntiles, out_stride);
    else raise(QCSIM_CAPACITY, "planes longer than 2^22 elements are not supported on the device path");
}

// Encodes units*NP planes produced by `src` into `arena` (grown as needed).
// `index` receives the decode checkpoints ([plane][nidx]).
template <int NP, class Src>
void encode_launch(cudaStream_t st, EncScratch &S, const Src &src, int units, uint64_t L,
                   const qcsim_codec_config &cfg, int log2C, IndexRec *index, DBuf<uint8_t> &arena,
                   bool check_finite, bool sync_now, bool host_results) {
    const uint64_t planes = (uint64_t)units * NP;
    const int qb = cfg.quant_code_bits;
    S.ensure(planes, units, L, qb);
    const int ntiles = (int)((L + kTile - 1) / kTile);
    const uint64_t cap = std::min<uint64_t>(L + 1, (1ull << qb) + 1);
    const unsigned tgrid_u = (unsigned)(units * ntiles), tgrid_p = (unsigned)(planes * ntiles);

    if (check_finite) CK(cudaMemsetAsync(S.nonfinite.p, 0, sizeof(uint32_t), st));
    // Per-plane bounds only change with the data in RangeRelative mode; for
    // fixed bounds they are computed once per batch shape (enc_x resets the
    // per-pass flags and histogram bookkeeping itself).
    const bool params_fresh = S.param_planes == planes && S.param_cfg.mode == cfg.mode &&
                              S.param_cfg.bound == cfg.bound && S.param_cfg.predictor == cfg.predictor &&
                              cfg.mode != QCSIM_MODE_RANGE_RELATIVE;
    if (check_finite || !params_fresh) {
        PROF("init_params", st);
        launch_k(init_params<NP, Src>, units, 256, 0, st, S.params.p, src, units, L, cfg.mode, cfg.bound, cfg.predictor,
                                                    check_finite ? S.nonfinite.p : nullptr, S.symrange.p,
                                                    S.hspecial.p, S.gamma.p);
        S.param_planes = cfg.mode == QCSIM_MODE_RANGE_RELATIVE ? 0 : planes;
        S.param_cfg = cfg;
    }
    if (check_finite) {
        uint32_t bad = 0;
        CK(cudaMemcpyAsync(&bad, S.nonfinite.p, sizeof bad, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        g_prof.flush();
        if (bad) raise(QCSIM_INVALID_ARGUMENT, "plane contains a non-finite value");
    }

    TileArgs A;
    A.params = S.params.p;
    A.x = S.x.p;
    A.sym = S.sym.p;
    A.fl = S.fl.p;
    A.evlist = S.evlist.p;
    A.evc = S.evc.p;
    A.dval = S.dval.p;
    A.t_firstb = S.t_firstb.p;
    A.t_lastb = S.t_lastb.p;
    A.t_nout = S.t_nout.p;
    A.index = index;
    A.t_lastout = S.t_lastout.p;
    A.t_base = S.t_base.p;
    A.t_evoff = reinterpret_cast<uint32_t *>(S.t_evoff.p);
    A.tilesum = S.tilesum.p;
    A.L = L;
    A.ntiles = ntiles;
    A.tile_sh = -1;
    if ((ntiles & (ntiles - 1)) == 0)
        for (int sh = 0; sh < 31; ++sh)
            if ((1 << sh) == ntiles) A.tile_sh = sh;
    A.log2C = log2C;
    A.qb = qb;
    A.predictor = cfg.predictor;
    A.symrange = S.symrange.p;
    A.hspecial = S.hspecial.p;
    A.gamma = S.gamma.p;
    A.t_nev = reinterpret_cast<uint32_t *>(S.t_nev.p);
    if (S.lb.ensure(planes * ntiles, /*zero=*/true)) S.lb_epoch = 0;
    if (++S.lb_epoch >= (1u << 30) - 4) { // epoch wrapped: clean slots
        CK(cudaMemsetAsync(S.lb.p, 0, S.lb.cap * sizeof(unsigned long long), st));
        S.lb_epoch = 1;
    }
    A.lb = S.lb.p;
    A.lb_epoch = S.lb_epoch;
    {
        // run-aware tile flags (QCSIM_ZERO_TILES=0: off)
        static const bool zoff = std::getenv("QCSIM_ZERO_TILES") && std::getenv("QCSIM_ZERO_TILES")[0] == '0';
        A.zx = A.ztriv = nullptr;
        if (!zoff && ntiles > kInlineTiles && cfg.predictor == 0) {
            S.zx.ensure(planes * ntiles);
            S.ztriv.ensure(planes * ntiles);
            A.zx = S.zx.p;
            A.ztriv = S.ztriv.p;
            CK(cudaMemsetAsync(S.ztriv.p, 0, planes * ntiles, st)); // (enc_verify's general path leaves 0)
        }
    }
    A.want_evD = chain_scan_selected(planes) ? 1 : 0;
    if (A.want_evD) S.evD.ensure(planes * L + 8); // (the serial warp chain needs no estimates)
    A.evD = S.evD.p;
    // Planes of many whole tiles, lossy absolute bound, previous-value
    // predictor: gate + lattice in ONE grid (enc_gate_lattice, base 0.0), then
    // enc_lattice again only for the planes that hold a speculative outlier
    // (QCSIM_FUSE_GL=0: the two separate grids).
    static const bool fuse_gl_off = std::getenv("QCSIM_FUSE_GL") && std::getenv("QCSIM_FUSE_GL")[0] == '0';
    const bool fused_gl = !fuse_gl_off && ntiles > kInlineTiles && L % kTile == 0 && cfg.mode == QCSIM_MODE_ABSOLUTE &&
                          cfg.predictor == 0;
    // event records at tile-local slots when the block-parallel chain reads
    // them (no look-back between the tiles of a plane)
    static const bool tile_local_off = std::getenv("QCSIM_EV_TILE_LOCAL") && std::getenv("QCSIM_EV_TILE_LOCAL")[0] == '0';
    A.ev_tile_local = (ntiles <= kInlineTiles && chain_scan_selected(planes) && !tile_local_off) ? 1 : 0;
    A.trace = nullptr;
    A.lat_bad = nullptr;
    A.chain_prog = nullptr;
    if (fused_gl) {
        S.lat_bad.ensure(planes);
        S.lat_redo.ensure(planes + 1);
        A.lat_bad = S.lat_bad.p;
        CK(cudaMemsetAsync(S.lat_bad.p, 0, planes * sizeof(uint32_t), st));
        {
            PROF("enc_gate_lattice", st);
            launch_k(enc_gate_lattice<NP, Src>, tgrid_u, kEncThreads, 0, st, A, src, units);
        }
        launch_plane_scan(st, S.t_lastout.p, S.t_base.p, ntiles, (int)planes, kScanMaxExcl);
        {
            PROF("lattice_redo", st);
            launch_k(lattice_redo_list, 1, 256, 0, st, A, (int)planes, S.lat_redo.p);
            const int rmax = (int)std::min<uint64_t>(planes, 16);
            launch_k(enc_lattice, (unsigned)(rmax * ntiles), kEncThreads, 0, st, A, (int)planes,
                     (const uint32_t *)S.lat_redo.p, rmax);
        }
    } else {
        {
            PROF("enc_x", st);
            static const bool vec_off = std::getenv("QCSIM_ENCX_VEC") && std::getenv("QCSIM_ENCX_VEC")[0] == '0';
            if (vec_off) launch_k(enc_x<NP, Src, false>, tgrid_u, kEncThreads, 0, st, A, src, units);
            else launch_k(enc_x<NP, Src, true>, tgrid_u, kEncThreads, 0, st, A, src, units);
        }
        launch_plane_scan(st, S.t_lastout.p, S.t_base.p, ntiles, (int)planes, kScanMaxExcl);
        // debug: QCSIM_LAT_TRACE_AT = encode call -> phase stamps to QCSIM_LAT_TRACE_FILE
        static const long lat_at = std::getenv("QCSIM_LAT_TRACE_AT") ? std::atol(std::getenv("QCSIM_LAT_TRACE_AT")) : -1;
        static long lat_calls = 0;
        static DBuf<unsigned long long> lat_trace;
        if (lat_at >= 0 && lat_calls++ == lat_at) {
            lat_trace.ensure(8 * (uint64_t)tgrid_p);
            CK(cudaMemsetAsync(lat_trace.p, 0, 8 * (uint64_t)tgrid_p * 8, st));
            A.trace = lat_trace.p;
        }
        PROF("enc_lattice", st);
        launch_k(enc_lattice, tgrid_p, kEncThreads, 0, st, A, (int)planes, (const uint32_t *)nullptr, 0);
        if (A.trace) {
            std::vector<unsigned long long> h(8 * (uint64_t)tgrid_p);
            CK(cudaMemcpyAsync(h.data(), A.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (FILE *f = std::fopen(std::getenv("QCSIM_LAT_TRACE_FILE"), "wb")) {
                std::fwrite(h.data(), 8, h.size(), f);
                std::fclose(f);
            }
            A.trace = nullptr;
        }
    }
    launch_plane_scan(st, S.t_nev.p, S.t_evoff.p, ntiles, (int)planes, kScanSumExcl);
    if (ntiles > kInlineTiles) {
        PROF("enc_compact", st);
        const int K = std::min(ntiles, 256);
        launch_k(enc_compact, (unsigned)(planes * K), kEncThreads, 0, st, A, (int)planes, K,
                 reinterpret_cast<unsigned long long *>(chain_stats() + 6));
    }
    {
        // debug: dump one encode call's event lists (QCSIM_CHAIN_DUMP_AT = call
        // number, QCSIM_CHAIN_DUMP_FILE = path)
        static const long dump_at = std::getenv("QCSIM_CHAIN_DUMP_AT") ? std::atol(std::getenv("QCSIM_CHAIN_DUMP_AT")) : -1;
        static long calls = 0;
        if (dump_at >= 0 && calls++ == dump_at) {
            CK(cudaStreamSynchronize(st));
            const uint64_t nel = planes * L;
            std::vector<uint32_t> h_ev(nel), h_nev(planes * ntiles);
            std::vector<double> h_c(nel), h_d(nel);
            std::vector<PlaneParams> h_pp(planes);
            CK(cudaMemcpy(h_ev.data(), S.evlist.p, nel * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h_c.data(), S.evc.p, nel * 8, cudaMemcpyDeviceToHost));
            if (A.want_evD) CK(cudaMemcpy(h_d.data(), S.evD.p, nel * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h_nev.data(), S.t_nev.p, planes * ntiles * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h_pp.data(), S.params.p, planes * sizeof(PlaneParams), cudaMemcpyDeviceToHost));
            if (FILE *f = std::fopen(std::getenv("QCSIM_CHAIN_DUMP_FILE"), "wb")) {
                const uint64_t hdr[3] = {planes, L, (uint64_t)ntiles};
                std::fwrite(hdr, 8, 3, f);
                std::fwrite(h_pp.data(), sizeof(PlaneParams), planes, f);
                std::fwrite(h_nev.data(), 4, planes * ntiles, f);
                std::fwrite(h_ev.data(), 4, nel, f);
                std::fwrite(h_c.data(), 8, nel, f);
                std::fwrite(h_d.data(), 8, nel, f);
                std::fclose(f);
            }
        }
    }
    uint32_t *verify_done = nullptr; // per-plane chain completion (enc_verify overlaps the chain grid)
    uint32_t verify_epoch = 0;
    {
        // (chain_mode / scan: chosen before enc_lattice, see chain_choice)
        static const int chain_debug = std::getenv("QCSIM_CHAIN_DEBUG") ? 1 : 0;
        set_smem_once(enc_chain, kChainSmem, g_smem_set, 0);
        set_smem_once(enc_chain_scan, kChainScanSmem, g_smem_set, 1);
        const bool scan = chain_scan_selected(planes);
        const int chain_mode = chain_choice();
        if (chain_mode != 1 && scan) {
            PROF("enc_chain_scan", st);
            const int cmax = (int)((L + kCsChunk - 1) / kCsChunk);
            S.chain_carry.ensure(planes * cmax);
            S.chain_tcarry.ensure(planes * cmax);
            bool fresh = S.chain_flag.ensure(planes * cmax, /*zero=*/true);
            fresh |= S.chain_tflag.ensure(planes * cmax, /*zero=*/true);
            fresh |= S.chain_cnt.ensure(planes, /*zero=*/true);
            fresh |= S.chain_done.ensure(planes, /*zero=*/true);
            if (fresh) {
                CK(cudaMemsetAsync(S.chain_flag.p, 0, S.chain_flag.cap * sizeof(uint32_t), st));
                CK(cudaMemsetAsync(S.chain_tflag.p, 0, S.chain_tflag.cap * sizeof(uint32_t), st));
                CK(cudaMemsetAsync(S.chain_cnt.p, 0, S.chain_cnt.cap * sizeof(uint32_t), st));
                CK(cudaMemsetAsync(S.chain_done.p, 0, S.chain_done.cap * sizeof(uint32_t), st));
                S.chain_epoch = 0;
            }
            // debug: QCSIM_CHAIN_TRACE_AT = launch number -> per-block phase times to
            // QCSIM_CHAIN_TRACE_FILE
            static const long trace_at = std::getenv("QCSIM_CHAIN_TRACE_AT") ? std::atol(std::getenv("QCSIM_CHAIN_TRACE_AT")) : -1;
            static long scan_calls = 0;
            static DBuf<unsigned long long> trace_buf;
            const bool tracing = trace_at >= 0 && scan_calls++ == trace_at;
            if (tracing) {
                trace_buf.ensure(8 * planes * cmax);
                CK(cudaMemsetAsync(trace_buf.p, 0, 8 * planes * cmax * 8, st));
            }
            ChainLink link{S.chain_carry.p, S.chain_flag.p, S.chain_tcarry.p, S.chain_tflag.p, cmax, ++S.chain_epoch,
                           tracing ? trace_buf.p : nullptr, S.chain_cnt.p, S.chain_done.p};
            if (link.epoch == 0) { // wrapped: start over from clean flags
                CK(cudaMemsetAsync(S.chain_flag.p, 0, S.chain_flag.cap * sizeof(uint32_t), st));
                CK(cudaMemsetAsync(S.chain_tflag.p, 0, S.chain_tflag.cap * sizeof(uint32_t), st));
                CK(cudaMemsetAsync(S.chain_done.p, 0, S.chain_done.cap * sizeof(uint32_t), st));
                link.epoch = S.chain_epoch = 1;
            }
            if (!chain_overlap(planes)) link.cnt = link.done = nullptr;
            verify_done = link.done;
            verify_epoch = link.epoch;
            launch_k(enc_chain_scan, (unsigned)(planes * cmax), kCsThreads, kChainScanSmem, st, A, (int)planes, link,
                                                                                        chain_stats(), chain_debug);
            if (tracing) {
                std::vector<unsigned long long> h(8 * planes * cmax);
                std::vector<uint32_t> hn(planes * ntiles);
                CK(cudaMemcpyAsync(h.data(), trace_buf.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(hn.data(), S.t_nev.p, hn.size() * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (FILE *f = std::fopen(std::getenv("QCSIM_CHAIN_TRACE_FILE"), "wb")) {
                    const uint64_t hdr[3] = {planes, (uint64_t)cmax, (uint64_t)ntiles};
                    std::fwrite(hdr, 8, 3, f);
                    std::fwrite(hn.data(), 4, hn.size(), f);
                    std::fwrite(h.data(), 8, h.size(), f);
                    std::fclose(f);
                }
            }
        } else if (chain_mode != 1) {
            // planes of many tiles: enc_verify is launched alongside the serial
            // chain and follows each plane's chain front (QCSIM_CHAIN_PIPE=0: off)
            static const bool pipe_off = std::getenv("QCSIM_CHAIN_PIPE") && std::getenv("QCSIM_CHAIN_PIPE")[0] == '0';
            if (!pipe_off && ntiles > kInlineTiles) {
                S.chain_prog.ensure(planes);
                CK(cudaMemsetAsync(S.chain_prog.p, 0, planes * sizeof(uint32_t), st));
                A.chain_prog = S.chain_prog.p;
            }
            PROF("enc_chain", st);
            const int nbufs = planes > 2 * 148 ? 2 : kChainBufs; // latency hidden by other warps
            launch_k(enc_chain, (unsigned)planes, 32, chain_smem_bytes(nbufs), st, A, (int)planes, nbufs);
        }
    }
    // verify -> serial -> tok_count hand-offs per plane (the scans between
    // them are inline for planes of <= kInlineTiles tiles)
    const bool flow = chain_overlap(planes) && ntiles <= kInlineTiles;
    PlaneFlow vflow{nullptr, nullptr, 0};
    uint32_t flow_epoch = 0;
    if (flow) {
        bool fresh = S.ver_cnt.ensure(planes, /*zero=*/true);
        fresh |= S.ver_done.ensure(planes, /*zero=*/true);
        fresh |= S.ser_done.ensure(planes, /*zero=*/true);
        if (fresh || ++S.flow_epoch == 0) {
            CK(cudaMemsetAsync(S.ver_cnt.p, 0, S.ver_cnt.cap * sizeof(uint32_t), st));
            CK(cudaMemsetAsync(S.ver_done.p, 0, S.ver_done.cap * sizeof(uint32_t), st));
            CK(cudaMemsetAsync(S.ser_done.p, 0, S.ser_done.cap * sizeof(uint32_t), st));
            S.flow_epoch = 1;
        }
        flow_epoch = S.flow_epoch;
        vflow = PlaneFlow{S.ver_cnt.p, S.ver_done.p, flow_epoch};
    }
    {
        PROF("enc_verify", st);
        launch_k(enc_verify, tgrid_p, kEncThreads, 0, st, A, (int)planes, (const uint32_t *)verify_done,
                 verify_epoch, vflow, flow ? S.ser_done.p : nullptr);
    }
    {
        PROF("enc_serial", st);
        launch_k(enc_serial_x, (unsigned)((planes + 31) / 32), 32, 0, st, A, (int)planes,
                 (const uint32_t *)(flow ? S.ver_done.p : nullptr), flow ? S.ser_done.p : nullptr, flow_epoch);
    }

    TokArgs T;
    T.sym = S.sym.p;
    T.x = S.x.p;
    T.tsym = S.tsym.p;
    T.trep = S.trep.p;
    T.opos = S.opos.p;
    T.oval = S.oval.p;
    T.ocount = S.ocount.p;
    T.ntok = S.ntok.p;
    T.hist = S.hist.p;
    T.hspecial = S.hspecial.p;
    T.symrange = S.symrange.p;
    T.gamma_bits = S.gamma.p;
    T.index = index;
    T.t_firstb = S.t_firstb.p;
    T.t_lastb = S.t_lastb.p;
    T.t_nout = S.t_nout.p;
    T.t_ooff = S.t_ooff.p;
    T.t_prevb = S.t_prevb.p;
    T.t_nextb = S.t_nextb.p;
    T.t_ntok = S.t_ntok.p;
    T.t_tokoff = S.t_tokoff.p;
    T.ztriv = A.ztriv;
    T.L = L;
    T.ntiles = ntiles;
    T.tile_sh = A.tile_sh;
    T.log2C = log2C;
    T.qb = qb;
    // (tile run statistics: written by enc_verify / enc_serial_x)
    launch_plane_scan(st, S.t_lastb.p, S.t_prevb.p, ntiles, (int)planes, kScanMaxExcl);
    launch_plane_scan(st, S.t_firstb.p, S.t_nextb.p, ntiles, (int)planes, kScanMinExclRev);
    launch_plane_scan(st, S.t_nout.p, S.t_ooff.p, ntiles, (int)planes, kScanSumExcl);
    {
        PROF("tok_count", st);
        launch_k(tok_count, tgrid_p, kEncThreads, 0, st, T, (int)planes,
                 (const uint32_t *)(flow ? S.ser_done.p : nullptr), flow_epoch);
    }
    launch_plane_scan(st, S.t_ntok.p, S.t_tokoff.p, ntiles, (int)planes, kScanSumExcl);
    {
        // debug: QCSIM_ZT_STATS=1 prints how many tiles took the run-aware paths
        static const bool zt_stats = std::getenv("QCSIM_ZT_STATS") != nullptr;
        if (zt_stats && A.zx) {
            std::vector<uint8_t> hx(planes * ntiles), ht(planes * ntiles);
            CK(cudaMemcpyAsync(hx.data(), S.zx.p, hx.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(ht.data(), S.ztriv.p, ht.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            uint64_t nx = 0, nt = 0;
            for (uint8_t v : hx) nx += v != 0;
            for (uint8_t v : ht) nt += v != 0;
            std::fprintf(stderr, "zero tiles: %llu of %llu zero-valued, %llu flat zero-code\n", (unsigned long long)nx,
                         (unsigned long long)hx.size(), (unsigned long long)nt);
        }
    }

    CodeBook B;
    B.hist = S.hist.p;
    B.hspecial = S.hspecial.p;
    B.symrange = S.symrange.p;
    B.gamma_bits = reinterpret_cast<const uint64_t *>(S.gamma.p);
    B.ocount = S.ocount.p;
    B.sym = S.cb_sym.p;
    B.cnt = S.cb_cnt.p;
    B.len = S.cb_len.p;
    B.code = S.cb_code.p;
    B.key = S.cb_key.p;
    B.ncnt = S.cb_ncnt.p;
    B.parent = S.cb_parent.p;
    B.nsym = S.nsym.p;
    B.stream_bits = S.stream_bits.p;
    B.block_bytes = S.block_bytes.p;
    B.slot_bytes = S.slot_bytes.p;
    B.err = S.err.p;
    B.cap = cap;
    B.qb = qb;
    B.L = L;
    B.log2C = log2C;
    B.dec = S.dec_out;
    if (S.fixed_W) {
        if (S.fixed_planes != planes || S.fixed_at != S.fixed_W) {
            std::vector<uint64_t> off(planes + 1);
            for (uint64_t k = 0; k <= planes; ++k) off[k] = k * S.fixed_W;
            S.fixed_off.ensure(planes + 1);
            CK(cudaMemcpyAsync(S.fixed_off.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
            S.fixed_planes = planes;
            S.fixed_at = S.fixed_W;
        }
        if (!arena.p || arena.cap < planes * S.fixed_W + 64) raise(QCSIM_NOMEM, "fixed-slot arena too small");
        B.zero_arena = arena.p;
        B.zero_W = S.fixed_W;
    }
    // debug: QCSIM_CB_TRACE_AT = encode call -> codebook phase stamps to QCSIM_CB_TRACE_FILE
    static const long cb_at = std::getenv("QCSIM_CB_TRACE_AT") ? std::atol(std::getenv("QCSIM_CB_TRACE_AT")) : -1;
    static long cb_calls = 0;
    static DBuf<unsigned long long> cb_trace;
    const bool cb_tracing = cb_at >= 0 && cb_calls++ == cb_at;
    if (cb_tracing) {
        cb_trace.ensure(16 * planes);
        CK(cudaMemsetAsync(cb_trace.p, 0, 16 * planes * 8, st));
        B.trace = cb_trace.p;
    }
    {
        // tokens and codebooks in one grid (both only consume tok_count)
        PROF("tok_emit_codebook", st);
        launch_k(tok_emit_codebook, (unsigned)planes + tgrid_p, 256, 0, st, T, B, (int)planes);
    }
    if (cb_tracing) {
        std::vector<unsigned long long> h(16 * planes);
        CK(cudaMemcpyAsync(h.data(), cb_trace.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (FILE *f = std::fopen(std::getenv("QCSIM_CB_TRACE_FILE"), "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }

    // slot offsets: exclusive scan of slot sizes (16-byte aligned slots);
    // fixed slots: none (run metrics: the next pass's decoder grid)
    if (S.fixed_W) {
    } else if (S.stats_out) {
        PROF("slot_scan_stats", st);
        launch_k(slot_scan_stats, 1, 256, 0, st, S.slot_bytes.p, S.slot_off.p, S.block_bytes.p, S.err.p, S.params.p,
                 (int)planes, L, S.stats_gate, S.stats_out, S.overflow.p, S.rows_out, S.row0, S.nrows, log2C);
    } else {
        PROF("slot_scan", st);
        launch_k(slot_scan, 1, 256, 0, st, S.slot_bytes.p, S.slot_off.p, (int)planes, S.overflow.p);
    }

    PackArgs P;
    P.tsym = S.tsym.p;
    P.trep = S.trep.p;
    P.ntok = S.ntok.p;
    P.cb_sym = S.cb_sym.p;
    P.cb_len = S.cb_len.p;
    P.cb_code = S.cb_code.p;
    P.nsym = S.nsym.p;
    P.stream_bits = S.stream_bits.p;
    P.block_bytes = S.block_bytes.p;
    P.slot_off = S.fixed_W ? S.fixed_off.p : S.slot_off.p;
    P.lb = nullptr;
    P.lb_epoch = 0;
    P.opos = S.opos.p;
    P.oval = S.oval.p;
    P.ocount = S.ocount.p;
    P.params = S.params.p;
    P.index = index;
    P.overflow = S.overflow.p;
    P.blk_off = S.blk_off_out ? S.blk_off_out : S.blk_off.p;
    P.L = L;
    P.cap = cap;
    P.log2C = log2C;
    P.qb = qb;
    P.mode = cfg.mode;
    P.predictor = cfg.predictor;
    P.planes_total = (int)planes;
    S.pack = P;
    S.planes = planes;
    launch_pack(st, S, arena); // (slot_scan cleared the overflow flag)
    if (!host_results) return; // deferred engine: slot_scan_stats consumes them on the device
    // results for the host, one batch of async copies into pinned memory
    S.h_bytes.ensure(planes);
    S.h_off.ensure(planes);
    S.h_params.ensure(planes);
    S.h_err.ensure(planes);
    S.h_misc.ensure(2);
    CK(cudaMemcpyAsync(S.h_bytes.p, S.block_bytes.p, planes * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.h_off.p, S.blk_off.p, planes * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.h_params.p, S.params.p, planes * sizeof(PlaneParams), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.h_err.p, S.err.p, planes * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.h_misc.p, S.slot_off.p + planes, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(S.h_misc.p + 1, S.overflow.p, 4, cudaMemcpyDeviceToHost, st));
    if (sync_now) {
        CK(cudaStreamSynchronize(st));
        g_prof.flush();
    }
}

// Grows a buffer keeping its first `keep` bytes.
void grow_keep(DBuf<uint8_t> &b, uint64_t want, uint64_t keep, cudaStream_t st) {
    if (b.cap >= want) return;
    DBuf<uint8_t> nb;
    nb.ensure(want);
    if (b.p && keep) CK(cudaMemcpyAsync(nb.p, b.p, keep, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    b.swap(nb);
}

// After the stream has been synchronised: errors, arena overflow (grow,
// keeping the earlier waves' slots, and re-pack; nothing was written),
// per-plane results.
EncodeResult encode_finish(cudaStream_t st, EncScratch &S, DBuf<uint8_t> &arena) {
    CK(cudaGetLastError());
    const uint64_t planes = S.planes;
    for (uint64_t p = 0; p < planes; ++p)
        if (S.h_err.p[p] == kErrDepth) raise(QCSIM_CODEC, "prefix code depth out of range");
    EncodeResult R;
    R.total = S.h_misc.p[0];
    if ((uint32_t)S.h_misc.p[1]) {
        grow_keep(arena, S.arena_base + R.total + R.total / 2 + (1 << 20), S.arena_base, st);
        CK(cudaMemsetAsync(S.overflow.p, 0, sizeof(uint32_t), st));
        launch_pack(st, S, arena, false);
        CK(cudaMemcpyAsync(S.h_off.p, S.blk_off.p, planes * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(S.h_misc.p + 1, S.overflow.p, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        g_prof.flush();
        if ((uint32_t)S.h_misc.p[1]) raise(QCSIM_NOMEM, "compressed arena overflow after growth");
    }
    R.block_bytes.assign(S.h_bytes.p, S.h_bytes.p + planes);
    R.blk_off.assign(S.h_off.p, S.h_off.p + planes);
    for (uint64_t p = 0; p < planes; ++p) R.fallback += (S.h_params.p[p].flags & kFlagFallback) ? 1 : 0;
    return R;
}

// ------------------------------------------------------------ decoder
struct DecScratch {
    DBuf<uint32_t> lut, count, basei, sorted, meta;
    DBuf<uint64_t> first;
    uint64_t cap = 0;
    void ensure(uint64_t planes, uint64_t L, int qb) { ensure_cap(planes, std::min<uint64_t>(L + 1, (1ull << qb) + 1)); }
    void ensure_cap(uint64_t planes, uint64_t c) {
        cap = c;
        lut.ensure(planes << kLutBits);
        first.ensure(planes * (kMaxCodeLen + 1));
        count.ensure(planes * (kMaxCodeLen + 1));
        basei.ensure(planes * (kMaxCodeLen + 1));
        sorted.ensure(planes * cap);
        meta.ensure(planes * 4);
    }
    DecTables tables() const {
        DecTables T;
        T.lut = lut.p;
        T.first = first.p;
        T.count = count.p;
        T.basei = basei.p;
        T.sorted = sorted.p;
        T.meta = meta.p;
        T.cap = cap;
        return T;
    }
};

// prepare = false: the tables were written by the encoder that produced the
// blocks (enc_codebook -> emit_dec_tables), no table-parsing pass needed.
void decode_batch(cudaStream_t st, DecScratch &S, const uint8_t *arena, const uint64_t *blk_off,
                  double *const *out, int planes, uint64_t L, int log2C, int qb,
                  bool prepare = true, const NormArgs *norm = nullptr, uint8_t *zflag = nullptr,
                  uint64_t zflag_planes = 0, const IndexRec *fine_index = nullptr) {
    if (prepare) S.ensure(planes, L, qb);
    const DecTables T = S.tables();
    DecPlanes D;
    D.arena = arena;
    D.blk_off = blk_off;
    D.out = out;
    D.L = L;
    D.log2C = log2C;
    if (zflag) { // zero-tile flags of the batch's slots (imported partner slots stay 0)
        D.zflag = zflag;
        D.ztiles = (uint32_t)((L + kTile - 1) / kTile);
        CK(cudaMemsetAsync(zflag, 0, zflag_planes * D.ztiles, st));
    }
    if (prepare) {
        PROF("dec_prepare", st);
        launch_k(dec_prepare, planes, 256, 0, st, D, T, planes);
    }
    const uint64_t nchunks = (L + (1ull << log2C) - 1) >> log2C;
    if (fine_index) { // the previous pass's encoder checkpoints (scratch), [plane][nidx]
        D.ext_index = fine_index + 1; // record k at fine[k]
        D.ext_stride = (L >> log2C) + 1;
        D.fine = log2C;
        D.ext_fixed_nrec = (uint32_t)(nchunks - 1);
    }
    const uint64_t groups = ((fine_index ? D.ext_stride + 1 : nchunks) + kDecThreads - 1) / kDecThreads;
    {
        set_smem_once(dec_chunks, kDecSmem, g_smem_set, 2);
        PROF("dec_chunks", st);
        NormArgs N{};
        if (norm) N = *norm;
        launch_k(dec_chunks, (unsigned)(groups * planes) + (N.enabled ? 1u : 0u), kDecThreads, kDecSmem, st, D, T,
                 planes, N);
    }
}

// Host-side from_bytes checks (codec.cpp:366-408), exact messages.
struct Header {
    uint8_t mode, pred, qb;
    uint64_t n, outliers, payload;
    double eb;
};
Header parse_header(const uint8_t *b, uint64_t len, uint64_t *consumed) {
    auto rd = [&](int off, int bytes) {
        uint64_t v = 0;
        for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[off + i];
        return v;
    };
    if (len < kHeaderBytes) raise(QCSIM_CODEC, "block header truncated");
    if (b[0] != 'Q' || b[1] != 'C' || b[2] != 'B' || b[3] != '1') raise(QCSIM_CODEC, "bad block magic");
    if (b[4] != 1) raise(QCSIM_CODEC, "unsupported block version " + std::to_string(b[4]));
    if (b[5] > 2) raise(QCSIM_CODEC, "bad codec mode byte");
    if (b[6] > 1) raise(QCSIM_CODEC, "bad predictor byte");
    Header h;
    h.mode = b[5];
    h.pred = b[6];
    h.qb = b[7];
    if (h.qb < 4 || h.qb > 24) raise(QCSIM_CODEC, "quant_code_bits out of range");
    h.n = rd(8, 8);
    uint64_t ebits = rd(16, 8);
    std::memcpy(&h.eb, &ebits, 8);
    h.outliers = rd(24, 8);
    h.payload = rd(32, 8);
    if (h.n == 0) raise(QCSIM_CODEC, "element_count must be at least 1");
    if (h.outliers > h.n) raise(QCSIM_CODEC, "outlier_count exceeds element_count");
    if (!(h.eb >= 0.0) || !std::isfinite(h.eb)) raise(QCSIM_CODEC, "bad effective_abs_bound");
    if (h.payload > len - kHeaderBytes) raise(QCSIM_CODEC, "block payload truncated");
    if (consumed) *consumed = kHeaderBytes + h.payload;
    return h;
}

const char *dec_message(uint32_t e) {
    switch (e) {
    case kDecPayloadSmall: return "payload smaller than code table header";
    case kDecTableEmpty: return "empty prefix-code table";
    case kDecTableTrunc: return "code table truncated";
    case kDecSymOrder: return "code table symbols not strictly increasing";
    case kDecSymRange: return "code table symbol out of range";
    case kDecLenRange: return "code length out of range";
    case kDecOverfull: return "prefix code table overfull";
    case kDecLenMismatch: return "payload/header length mismatch";
    case kDecStreamTrunc: return "code stream truncated";
    case kDecInvalidCode: return "invalid prefix code in stream";
    case kDecRunNoCode: return "run escape without preceding code";
    case kDecRunRange: return "run length out of range";
    case kDecRunOverflow: return "run overflows element count";
    case kDecOutExhausted: return "outlier list exhausted early";
    case kDecOutPos: return "outlier position mismatch";
    case kDecOutUnused: return "unused trailing outliers";
    case kDecStreamLen: return "code stream length mismatch";
    case kDecHdrTrunc: return "block header truncated";
    case kDecMagic: return "bad block magic";
    case kDecVersion: return "unsupported block version";
    case kDecModeByte: return "bad codec mode byte";
    case kDecPredByte: return "bad predictor byte";
    case kDecQbRange: return "quant_code_bits out of range";
    case kDecCount0: return "element_count must be at least 1";
    case kDecOutCount: return "outlier_count exceeds element_count";
    case kDecEbBad: return "bad effective_abs_bound";
    case kDecPayTrunc: return "block payload truncated";
    case kDecWrongLen: return "partner block length does not match the slice";
    default: return "decoder scratch exhausted";
    }
}

// Foreign-block decoding (no index next to the blocks): stage the blocks
// with 16-byte aligned code streams, validate header + table (fd_head),
// parse the tables, one validating token walk per plane leaving a record
// every kFdBits stream bits (fd_scan), then the chunk-parallel decoder.
struct ForeignScratch {
    DBuf<uint8_t> arena;
    HBuf<uint8_t> h_arena;
    DBuf<uint64_t> meta; // [offsets | lengths]
    DBuf<uint32_t> err, nrec, slow, nseg;
    DBuf<IndexRec> rec;
    DBuf<double *> outs;
    DBuf<FpBound> bnd;
    DBuf<FpSeg> seg;
    DBuf<FpEntry> ent;
    DBuf<double> ev;
    DBuf<uint8_t> evk;
    DecScratch tables;
    std::vector<uint32_t> h_err;
};
struct ForeignBlock {
    const uint8_t *src; // host or device bytes
    uint64_t len;       // bytes available at src
    uint32_t table_count;
    uint64_t payload;
    double *out;        // device plane
};

// Decodes blocks of one element count `n` into their device planes; returns
// the first failing block's error code (plane order) or 0.
uint32_t foreign_decode_batch(cudaStream_t st, ForeignScratch &F, const std::vector<ForeignBlock> &B,
                              bool src_device, uint64_t n, int qb);
uint32_t foreign_decode(cudaStream_t st, ForeignScratch &F, const std::vector<ForeignBlock> &B, bool src_device,
                        uint64_t n, int qb) {
    // sub-batches bound the event lists (8 B + 1 B per element)
    const uint64_t per = std::max<uint64_t>(1, (1ull << 27) / std::max<uint64_t>(n, 1));
    for (uint64_t k0 = 0; k0 < B.size(); k0 += per) {
        std::vector<ForeignBlock> part(B.begin() + k0, B.begin() + std::min<uint64_t>(B.size(), k0 + per));
        const uint32_t e = foreign_decode_batch(st, F, part, src_device, n, qb);
        if (e) return e;
    }
    return 0;
}
uint32_t foreign_decode_batch(cudaStream_t st, ForeignScratch &F, const std::vector<ForeignBlock> &B,
                              bool src_device, uint64_t n, int qb) {
    const uint64_t P = B.size();
    if (!P) return 0;
    std::vector<uint64_t> meta(2 * P);
    uint64_t end = 0, maxtc = 1, stride = 1;
    for (uint64_t k = 0; k < P; ++k) {
        const uint64_t pre = kHeaderBytes + 4 + 5ull * B[k].table_count;
        const uint64_t off = ((end + 15) & ~15ull) + ((16 - (pre & 15)) & 15); // stream 16-byte aligned
        meta[k] = off;
        meta[P + k] = B[k].len;
        end = off + B[k].len + 64; // padding: the bit window reads ahead
        maxtc = std::max<uint64_t>(maxtc, B[k].table_count);
        stride = std::max<uint64_t>(stride, (B[k].payload * 8) / kFdBits + 2);
    }
    F.arena.ensure(end + 64);
    if (src_device) {
        for (uint64_t k = 0; k < P; ++k)
            CK(cudaMemcpyAsync(F.arena.p + meta[k], B[k].src, B[k].len, cudaMemcpyDeviceToDevice, st));
    } else {
        F.h_arena.ensure(end + 64);
        for (uint64_t k = 0; k < P; ++k) std::memcpy(F.h_arena.p + meta[k], B[k].src, B[k].len);
        CK(cudaMemcpyAsync(F.arena.p, F.h_arena.p, end, cudaMemcpyHostToDevice, st));
    }
    F.meta.ensure(2 * P);
    CK(cudaMemcpyAsync(F.meta.p, meta.data(), 2 * P * 8, cudaMemcpyHostToDevice, st));
    std::vector<double *> outs(P);
    for (uint64_t k = 0; k < P; ++k) outs[k] = B[k].out;
    F.outs.ensure(P);
    CK(cudaMemcpyAsync(F.outs.p, outs.data(), P * sizeof(double *), cudaMemcpyHostToDevice, st));
    F.err.ensure(P);
    F.nrec.ensure(P);
    F.rec.ensure(P * stride);
    const uint64_t cap = std::min<uint64_t>(std::max<uint64_t>(maxtc, 1), 1ull << 25);
    (void)qb;
    F.tables.ensure_cap(P, cap);
    FdArgs A;
    A.arena = F.arena.p;
    A.blk_off = F.meta.p;
    A.avail = F.meta.p + P;
    A.err = F.err.p;
    A.n_expected = n;
    A.cap = F.tables.cap;
    A.rec = F.rec.p;
    A.nrec = F.nrec.p;
    A.stride = stride;
    {
        PROF("fd_head", st);
        launch_k(fd_head, (unsigned)((P + 31) / 32), 32, 0, st, A, (int)P);
    }
    DecPlanes D;
    D.arena = F.arena.p;
    D.blk_off = F.meta.p;
    D.out = F.outs.p;
    D.L = n;
    D.log2C = 10;
    D.skip = F.err.p;
    const DecTables T = F.tables.tables();
    {
        PROF("dec_prepare", st);
        launch_k(dec_prepare, (unsigned)P, 256, 0, st, D, T, (int)P);
    }
    // the parallel path (foreign_kernels.cuh); planes it declines: fd_scan
    static const bool serial_only = std::getenv("QCSIM_FOREIGN_SERIAL") != nullptr; // (debug)
    F.slow.ensure(P);
    if (serial_only) {
        CK(cudaMemsetAsync(F.slow.p, 0xFF, P * 4, st));
    } else {
        FpArgs G;
        G.arena = F.arena.p;
        G.blk_off = F.meta.p;
        G.err = F.err.p;
        G.slow = F.slow.p;
        G.stride = stride;
        F.bnd.ensure(P * stride * kFpM);
        F.seg.ensure(P * stride);
        F.ent.ensure(P * stride);
        F.nseg.ensure(P);
        F.ev.ensure(P * n);
        F.evk.ensure(P * n);
        G.bnd = F.bnd.p;
        G.seg = F.seg.p;
        G.ent = F.ent.p;
        G.nseg = F.nseg.p;
        G.ev = F.ev.p;
        G.evk = F.evk.p;
        G.rec = F.rec.p;
        G.nrec = F.nrec.p;
        G.rec_stride = stride;
        G.n = n;
        const unsigned segs = (unsigned)((P * stride + 127) / 128);
        {
            PROF("fp_spec", st);
            launch_k(fp_spec, segs, 128, 0, st, G, T, (int)P);
        }
        {
            PROF("fp_resolve", st);
            launch_k(fp_resolve, (unsigned)((P + 31) / 32), 32, 0, st, G, T, (int)P);
        }
        {
            PROF("fp_count", st);
            launch_k(fp_count, segs, 128, 0, st, G, T, (int)P);
        }
        {
            PROF("fp_evscan", st);
            launch_k(fp_evscan, (unsigned)((P + 31) / 32), 32, 0, st, G, (int)P);
        }
        {
            PROF("fp_events", st);
            launch_k(fp_events, segs, 128, 0, st, G, T, (int)P);
        }
        {
            PROF("fp_chain", st);
            launch_k(fp_chain, (unsigned)P, 32, 0, st, G, (int)P);
        }
    }
    A.only = F.slow.p;
    {
        PROF("fd_scan", st);
        launch_k(fd_scan, (unsigned)((P + 31) / 32), 32, 0, st, A, T, (int)P);
    }
    D.ext_index = F.rec.p;
    D.ext_nrec = F.nrec.p;
    D.ext_stride = stride;
    {
        set_smem_once(dec_chunks, kDecSmem, g_smem_set, 2);
        PROF("dec_chunks", st);
        const uint64_t groups = (stride + 1 + kDecThreads - 1) / kDecThreads;
        launch_k(dec_chunks, (unsigned)(groups * P), kDecThreads, kDecSmem, st, D, T, (int)P, NormArgs{});
    }
    F.h_err.resize(P);
    CK(cudaMemcpyAsync(F.h_err.data(), F.err.p, P * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    for (uint64_t k = 0; k < P; ++k)
        if (F.h_err[k]) return F.h_err[k];
    return 0;
}

// ------------------------------------------------------------- context
// Per-thread codec context for the single-plane / batched codec API.
struct CodecCtx {
    int dev = -1;
    cudaStream_t st = nullptr;
    EncScratch enc;
    ForeignScratch fore;
    DBuf<uint8_t> arena, bytes;
    DBuf<double> vals;
    DBuf<IndexRec> index;
    DBuf<const double *> ptrs;
    DBuf<double *> optrs;
    DBuf<uint64_t> offs;
};
// one context per (thread, device): streams and buffers belong to a device
thread_local CodecCtx *t_codec[kMaxDevices] = {};
CodecCtx &codec_ctx() {
    const int dev = current_device();
    ensure_device(dev);
    CodecCtx *&c = t_codec[dev];
    if (!c) {
        c = new CodecCtx();
        c->dev = dev;
        CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    }
    return *c;
}

} // namespace

// =================================================================== engine
// Per-gate run metrics (SPEC.md:309-314 per_gate_min_ratio; the CSV report's
// gate_index, min_ratio, mean_ratio, seconds), plus the state's bytes after
// the gate.
struct GateRow {
    double min_ratio, ratio_sum;
    uint64_t calls, bytes, index_bytes;
    double seconds;
};

struct qcsim_engine {
    qcsim_engine_config cfg{};
    int n = 0, s = 0;
    uint64_t S = 0, L = 0;       // slices (global), slice length
    uint64_t s0 = 0, ns = 0;     // this rank's slice range
    uint64_t wave = 0;           // slices per batch (wave) of a gate pass; ns = one batch
    int log2C = 0;
    uint64_t nidx = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evg = nullptr;
    bool compressed = true;
    bool loaded = false;
    // compressed state (ping-pong); every block's slot also holds its
    // decode index (common.cuh)
    DBuf<uint8_t> arena[2];
    DBuf<uint64_t> blk_off[2];         // device copy of the block offsets, plane order
    std::vector<uint64_t> blk_bytes_h; // current block sizes, plane order
    std::vector<uint64_t> blk_off_h;   // current block offsets, plane order
    DBuf<IndexRec> index;              // encoder scratch: fine decode-index records
    int cur = 0;
    // dense state (compression off); decoded old values of one batch,
    // [slot][re|im][L] (slots: the batch's units, then imported partners)
    DBuf<double> dense[2];
    DBuf<double> old;
    DBuf<uint8_t> zold;                // zero-tile flags of `old`, [plane][ntiles] (big planes only)
    DBuf<double *> outptrs;            // plane k of the batch -> old + k L
    uint64_t outptr_planes = 0;
    const double *outptr_base = nullptr;
    DBuf<uint64_t> wave_off;           // block offsets of one wave's planes
    HBuf<uint64_t> h_wave_off;
    DBuf<double> slice_sq;
    HBuf<double> h_sq;
    DBuf<double *> imp_ptrs;
    // partner slices imported from other ranks: slice -> QCB1 bytes
    std::vector<std::pair<uint64_t, std::vector<uint8_t>>> imported;
    // ... or resident in a caller-owned device buffer (import_partners_device):
    // slice -> (re offset, im offset, re length, im length)
    const uint8_t *dev_imp = nullptr;
    std::unordered_map<uint64_t, std::array<uint64_t, 4>> dev_imp_at;
    DBuf<uint64_t> dev_imp_meta; // [plane offsets | available lengths] of a batch
    std::vector<double> sq_norm; // all S slices (global view)
    EncScratch enc;
    DecScratch dec[2]; // decode tables of arena[0/1], written by the encoder (single-batch passes)
    DecScratch decw;   // decode tables parsed from the blocks (waves, compare, gather)
    ForeignScratch fore; // partner blocks imported from host bytes
    DBuf<uint8_t> imp_bytes;
    DBuf<uint64_t> imp_off;
    // deferred gate loop (no host round trip per gate): device scale,
    // device metrics, latched errors
    bool deferred = false;
    NormArgs norm{};          // this gate pass's deferred normalization (run by the decoder grid)
    DBuf<uint64_t> exp_meta;  // export_blocks gather: source / destination offsets, lengths
    DBuf<uint8_t> exp_buf;
    bool defer_fresh = false; // no pass has run yet in this deferred run
    DBuf<double> norm_buf[2], dev_scale;
    DBuf<EngineDevStats> dev_stats;
    HBuf<EngineDevStats> h_stats;
    DBuf<GateRowDev> dev_rows; // deferred run: one row per gate pass
    HBuf<GateRowDev> h_rows;
    uint64_t row0 = 0, nrows = 0;
    // metrics
    double ratio_min = INFINITY, ratio_sum = 0.0;
    uint64_t calls = 0, gates = 0, peak = 0, current = 0, fallback = 0;
    double wall = 0.0;
    uint64_t launches0 = 0;
    std::vector<GateRow> rows; // since the last load
};

namespace {

uint64_t partner_mask(const qcsim_action &a, int s) {
    if (a.kind == QCSIM_ACTION_BUTTERFLY && a.target >= s) return 1ull << (a.target - s);
    if (a.kind == QCSIM_ACTION_SWAP) {
        uint64_t hm = 0;
        if (a.a >= s) hm |= 1ull << (a.a - s);
        if (a.b >= s) hm |= 1ull << (a.b - s);
        return hm;
    }
    return 0;
}
uint64_t partner_slice(const qcsim_action &a, int s, uint64_t j) { return j ^ partner_mask(a, s); }

DevAction to_dev(const qcsim_action &a) {
    DevAction d{};
    d.kind = a.kind;
    d.target = a.target;
    d.a = a.a;
    d.b = a.b;
    d.mask = a.mask;
    d.f[0] = a.factor[0];
    d.f[1] = a.factor[1];
    for (int k = 0; k < 8; ++k) d.u[k] = a.u[k];
    return d;
}

double tree_sum_host(const double *v, uint64_t len) {
    if (len == 1) return v[0];
    const uint64_t h = len / 2;
    const double a = tree_sum_host(v, h), b = tree_sum_host(v + h, h);
    return a + b;
}

uint64_t index_bytes_of(const qcsim_engine *e, const std::vector<uint64_t> &bytes) {
    uint64_t t = 0;
    for (uint64_t b : bytes) t += index_records(e->L, b, e->log2C) * sizeof(IndexRec);
    return t;
}

// Run metrics of one encode pass over all local planes (plane order, as the
// oracle): min / mean ratio, bytes, and the per-gate row.
void record_sizes(qcsim_engine *e, const std::vector<uint64_t> &bytes, double seconds) {
    uint64_t tot = 0;
    GateRow row{INFINITY, 0.0, 0, 0, 0, seconds};
    for (uint64_t b : bytes) {
        const double ratio = (double)(8 * e->L) / (double)b;
        if (ratio < e->ratio_min) e->ratio_min = ratio;
        e->ratio_sum += ratio;
        e->calls++;
        if (ratio < row.min_ratio) row.min_ratio = ratio;
        row.ratio_sum += ratio;
        row.calls++;
        tot += b;
    }
    e->current = tot;
    e->peak = std::max(e->peak, tot);
    row.bytes = tot;
    row.index_bytes = index_bytes_of(e, bytes);
    e->rows.push_back(row);
}

// Identity source over [slot][2][L] planes (initial loads).
struct PlanarSrc {
    const double *v;
    uint64_t L;
    static constexpr bool kNorms = true;
    __device__ __forceinline__ void load(int unit, uint64_t i, double *o) const {
        o[0] = v[(uint64_t)unit * 2 * L + i];
        o[1] = v[(uint64_t)unit * 2 * L + L + i];
    }
    __device__ __forceinline__ void load2(int unit, uint64_t i, double *a, double *b) const { // i even, L even
        const double2 r = *reinterpret_cast<const double2 *>(v + (uint64_t)unit * 2 * L + i);
        const double2 m = *reinterpret_cast<const double2 *>(v + (uint64_t)unit * 2 * L + L + i);
        a[0] = r.x; a[1] = m.x; b[0] = r.y; b[1] = m.y;
    }
    template <bool> __device__ __forceinline__ void loadf(int unit, uint64_t i, double *o) const { load(unit, i, o); }
    template <bool> __device__ __forceinline__ void load2f(int unit, uint64_t i, double *a, double *b) const {
        load2(unit, i, a, b);
    }
    __device__ __forceinline__ bool flagged_sources(int, uint32_t) const { return false; }
};
// Basis state |x> on the batch's slices.
struct BasisSrc {
    uint64_t x;
    SliceMap map;
    int s;
    static constexpr bool kNorms = true;
    __device__ __forceinline__ void load(int unit, uint64_t i, double *o) const {
        const uint64_t g = ((map.s0 + map.slice_rel((uint32_t)unit)) << s) | i;
        o[0] = g == x ? 1.0 : 0.0;
        o[1] = 0.0;
    }
    __device__ __forceinline__ void load2(int unit, uint64_t i, double *a, double *b) const {
        load(unit, i, a);
        load(unit, i + 1, b);
    }
    template <bool> __device__ __forceinline__ void loadf(int unit, uint64_t i, double *o) const { load(unit, i, o); }
    template <bool> __device__ __forceinline__ void load2f(int unit, uint64_t i, double *a, double *b) const {
        load2(unit, i, a, b);
    }
    __device__ __forceinline__ bool flagged_sources(int, uint32_t) const { return false; }
};

// Slices per wave: the largest power of two whose dense working set (old
// planes, encoder scratch, decode tables, fine index) fits the budget
// (cfg.wave_bytes, else 85% of the device memory free at creation;
// QCSIM_WAVE_SLICES overrides for tests).  Grouped waves need a whole
// partner group (<= 4).
uint64_t choose_wave(const qcsim_engine *e) {
    if (!e->compressed) return e->ns;
    if (const char *v = std::getenv("QCSIM_WAVE_SLICES")) {
        uint64_t w = std::strtoull(v, nullptr, 10);
        uint64_t p = 1;
        while (p * 2 <= w && p * 2 <= e->ns) p *= 2;
        return std::max<uint64_t>(std::min<uint64_t>(4, e->ns), p);
    }
    uint64_t budget = e->cfg.wave_bytes;
    if (!budget) { // 85% of the device memory free when the engine is created
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            cudaGetLastError();
            fr = 160ull << 30;
        }
        budget = (uint64_t)(0.85 * (double)fr);
    }
    const uint64_t L = e->L;
    const uint64_t cap = std::min<uint64_t>(L + 1, (1ull << e->cfg.codec.quant_code_bits) + 1);
    const uint64_t per_plane = L * 70 + cap * 70 + (L >> e->log2C) * sizeof(IndexRec) + (8u << 10);
    const uint64_t per_slice = 2 * per_plane;
    uint64_t w = 1;
    while (w * 2 <= e->ns && (w * 2) * per_slice <= budget) w *= 2;
    return std::max<uint64_t>(std::min<uint64_t>(4, e->ns), w);
}

// Decode-output pointer table for batches of up to `planes` planes of `old`.
void ensure_outptrs(qcsim_engine *e, uint64_t planes) {
    e->old.ensure(planes * e->L);
    if (e->outptr_planes >= planes && e->outptr_base == e->old.p) return;
    std::vector<double *> ptrs(planes);
    for (uint64_t k = 0; k < planes; ++k) ptrs[k] = e->old.p + k * e->L;
    e->outptrs.ensure(planes);
    CK(cudaMemcpy(e->outptrs.p, ptrs.data(), planes * sizeof(double *), cudaMemcpyHostToDevice));
    e->outptr_planes = planes;
    e->outptr_base = e->old.p;
}

// Imported partner blocks (other ranks) of units [u0, u0 + cnt), decoded by
// the validating decoder into planes old[first_plane + 2u + p].
void decode_imports(qcsim_engine *e, const SliceMap &map, uint64_t u0, uint64_t cnt, uint64_t first_plane) {
    if (!cnt) return;
    if (e->dev_imp) {
        // device-resident partner blocks: no host staging; from_bytes checks
        // run on the device with the validating decoder
        // (headers gathered by one kernel + one copy; from_bytes checks on
        // the host copy, then the parallel foreign decoder reads the blocks
        // where they lie)
        const uint64_t P = 2 * cnt;
        std::vector<uint64_t> src_off(P), avail(P), meta(3 * P);
        for (uint64_t u = u0; u < u0 + cnt; ++u) {
            const uint64_t pj = (e->s0 + map.slice_rel((uint32_t)u)) ^ map.hm;
            auto it = e->dev_imp_at.find(pj);
            if (it == e->dev_imp_at.end())
                raise(QCSIM_INVALID_ARGUMENT,
                      "partner slice " + std::to_string(pj) + " not imported (multi-rank exchange missing)");
            const uint64_t k = u - u0;
            for (int p = 0; p < 2; ++p) {
                src_off[2 * k + p] = it->second[p];
                avail[2 * k + p] = it->second[2 + p];
            }
        }
        constexpr uint64_t kHead = 48; // header + table count, padded
        for (uint64_t k = 0; k < P; ++k) {
            meta[k] = src_off[k];
            meta[P + k] = k * kHead;
            meta[2 * P + k] = std::min<uint64_t>(44, avail[k]);
        }
        e->dev_imp_meta.ensure(3 * P);
        e->exp_buf.ensure(P * kHead + 16);
        CK(cudaMemcpyAsync(e->dev_imp_meta.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, e->st));
        {
            PROF("gather_heads", e->st);
            launch_k(gather_blocks, (unsigned)P, 64, 0, e->st, e->dev_imp, (const uint64_t *)e->dev_imp_meta.p, (int)P,
                     e->exp_buf.p);
        }
        std::vector<uint8_t> heads(P * kHead, 0);
        CK(cudaMemcpyAsync(heads.data(), e->exp_buf.p, P * kHead, cudaMemcpyDeviceToHost, e->st));
        CK(cudaStreamSynchronize(e->st));
        std::vector<ForeignBlock> fb(P);
        for (uint64_t k = 0; k < P; ++k) {
            uint8_t *h = heads.data() + k * kHead;
            if (avail[k] < 44) std::memset(h + avail[k], 0, 44 - avail[k]);
            uint64_t used = 0;
            const Header hd = parse_header(h, avail[k], &used);
            if (hd.n != e->L) raise(QCSIM_CODEC, "partner block length does not match the slice");
            const uint32_t tc = hd.payload >= 4 ? (uint32_t)(h[40] | (h[41] << 8) | (h[42] << 16) | ((uint32_t)h[43] << 24)) : 0;
            fb[k] = ForeignBlock{e->dev_imp + src_off[k], used, tc, hd.payload, e->old.p + (first_plane + k) * e->L};
        }
        const uint32_t err = foreign_decode(e->st, e->fore, fb, true, e->L, e->cfg.codec.quant_code_bits);
        if (err) raise(QCSIM_CODEC, dec_message(err));
        return;
    }
    std::unordered_map<uint64_t, size_t> where;
    for (size_t m = 0; m < e->imported.size(); ++m) where[e->imported[m].first] = m;
    std::vector<ForeignBlock> fb;
    for (uint64_t u = u0; u < u0 + cnt; ++u) {
        const uint64_t pj = (e->s0 + map.slice_rel((uint32_t)u)) ^ map.hm;
        auto it = where.find(pj);
        if (it == where.end())
            raise(QCSIM_INVALID_ARGUMENT,
                  "partner slice " + std::to_string(pj) + " not imported (multi-rank exchange missing)");
        const std::vector<uint8_t> &b = e->imported[it->second].second;
        uint64_t pos = 0;
        for (int p = 0; p < 2; ++p) {
            uint64_t used = 0;
            const Header h = parse_header(b.data() + pos, b.size() - pos, &used);
            if (h.n != e->L) raise(QCSIM_CODEC, "partner block length does not match the slice");
            const uint32_t tc = h.payload >= 4 ? (uint32_t)(b[pos + 40] | (b[pos + 41] << 8) | (b[pos + 42] << 16) |
                                                            ((uint32_t)b[pos + 43] << 24))
                                               : 0;
            fb.push_back(ForeignBlock{b.data() + pos, used, tc, h.payload,
                                      e->old.p + (first_plane + 2 * (u - u0) + p) * e->L});
            pos += used;
        }
    }
    const uint32_t err = foreign_decode(e->st, e->fore, fb, false, e->L, e->cfg.codec.quant_code_bits);
    if (err) raise(QCSIM_CODEC, dec_message(err));
}

// Decodes local slices [k0, k0 + cnt) (contiguous planes) into old slots
// [0, cnt): block offsets from the device table, tables parsed from the
// blocks.  Compare / gather.
void decode_range(qcsim_engine *e, uint64_t k0, uint64_t cnt) {
    ensure_outptrs(e, 2 * cnt);
    decode_batch(e->st, e->decw, e->arena[e->cur].p, e->blk_off[e->cur].p + 2 * k0, e->outptrs.p, (int)(2 * cnt),
                 e->L, e->log2C, e->cfg.codec.quant_code_bits, /*prepare=*/true);
}

// Plane values of local slices [k0, k0 + cnt) in [slot][re|im][L] layout on
// the device (decoded into `old`, or the dense state itself).
const double *state_range(qcsim_engine *e, uint64_t k0, uint64_t cnt) {
    if (!e->compressed) return e->dense[e->cur].p + k0 * 2 * e->L;
    decode_range(e, k0, cnt);
    return e->old.p;
}

// Run-aware gate pass for planes of many tiles (QCSIM_ZERO_TILES=0 turns it
// off): the decoder flags tiles of +0.0, the gate / lattice / verify /
// tokenizer grids take an O(1) path through tiles they know to be trivial.
bool zero_tiles_enabled(const qcsim_engine *e) {
    static const bool off = std::getenv("QCSIM_ZERO_TILES") && std::getenv("QCSIM_ZERO_TILES")[0] == '0';
    return !off && e->compressed && (e->L + kTile - 1) / kTile > (uint64_t)kInlineTiles &&
           e->cfg.codec.mode != QCSIM_MODE_LOSSLESS && e->cfg.codec.predictor == 0;
}

// One encode batch: `units` slices produced by `src` into arena[nxt] at
// enc.arena_base; the slice norms of the batch into h_sq[0, units).
template <class Src>
EncodeResult encode_units(qcsim_engine *e, const Src &src, uint64_t units, int nxt, bool tables) {
    e->index.ensure(2 * units * e->nidx);
    if (tables) {
        // the encoder also writes the decode tables of the blocks it packs
        e->dec[nxt].ensure(2 * units, e->L, e->cfg.codec.quant_code_bits);
        e->enc.dec_out = e->dec[nxt].tables();
    }
    encode_launch<2, Src>(e->st, e->enc, src, (int)units, e->L, e->cfg.codec, e->log2C, e->index.p, e->arena[nxt],
                          false, false);
    e->enc.dec_out = DecTables{};
    const uint64_t ntiles = (e->L + kTile - 1) / kTile;
    e->slice_sq.ensure(units);
    {
        PROF("slice_norms", e->st);
        if (ntiles > 64 && ntiles <= 4096)
            launch_k(slice_norms_block, (unsigned)units, 256, 0, e->st, e->enc.tilesum.p, (int)ntiles, (int)units,
                     e->slice_sq.p);
        else
            launch_k(slice_norms, (unsigned)((units + 127) / 128), 128, 0, e->st, e->enc.tilesum.p, (int)ntiles,
                     (int)units, e->slice_sq.p);
    }
    e->h_sq.ensure(units);
    CK(cudaMemcpyAsync(e->h_sq.p, e->slice_sq.p, units * sizeof(double), cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st)); // the host synchronisation of a batch
    g_prof.flush();
    return encode_finish(e->st, e->enc, e->arena[nxt]);
}

// A host-synchronous gate pass (or load) over the local slices in waves of
// e->wave slices.  `hm`: partner mask of the gate (0 for loads and local
// gates); `remote`: partners live on other ranks (imported); `decode`: the
// pass reads the old state.  make_src(map, old) returns the encoder source
// of a batch.  One wave (wave == ns) keeps the identity layout and the
// encoder-written decode tables; more waves decode with tables parsed from
// the blocks and group each wave under the partner mask.
template <class MakeSrc>
void engine_waves(qcsim_engine *e, uint64_t hm, bool remote, bool decode, MakeSrc make_src) {
    const int nxt = e->cur ^ 1;
    const uint64_t W = e->wave, nw = e->ns / W;
    const bool single = nw == 1;
    int gsh = 0;
    for (uint64_t h = hm; h; h &= h - 1) ++gsh;
    CK(cudaEventRecord(e->evg, e->st));
    std::vector<uint64_t> nbytes(2 * e->ns), noff(2 * e->ns);
    {
        // pre-size the new arena from the current state: a gate can grow the
        // state (an overflow costs a grow-and-copy plus a re-pack)
        uint64_t used = 0;
        for (uint64_t b : e->blk_bytes_h) used += b + 32;
        used += index_bytes_of(e, e->blk_bytes_h);
        // (a butterfly on a fresh qubit can double a sparse state: room for
        // 2x up to 4 GB of growth; a larger jump re-packs after growing)
        const uint64_t want = used + std::min<uint64_t>(used, 4ull << 30) + (256ull << 20);
        if (e->arena[nxt].cap < want) {
            e->arena[nxt].release();
            e->arena[nxt].ensure(want + std::min<uint64_t>(want / 2, 1ull << 30)); // (fewer reallocations as it grows)
        }
    }
    e->enc.arena_base = 0;
    {
        uint64_t cur = 0;
        for (uint64_t b : e->blk_bytes_h) cur += b;
        e->enc.pack_dense_hint = !e->blk_bytes_h.empty() && cur / e->blk_bytes_h.size() > (160u << 10);
    }
    uint64_t fb = 0;
    for (uint64_t w = 0; w < nw; ++w) {
        SliceMap map;
        map.s0 = e->s0;
        map.nunits = (uint32_t)W;
        if (remote) {
            map.mode = 2;
            map.hm = hm; // (global XOR: every partner is remote)
            map.gbase = w * W;
        } else if (single) {
            map.mode = 0;
            map.hm = hm;
        } else {
            map.mode = 1;
            map.hm = hm;
            map.gsh = (uint32_t)gsh;
            map.gbase = w * (W >> gsh);
        }
        const uint64_t slots = W + (remote ? W : 0);
        if (decode) {
            ensure_outptrs(e, 2 * slots);
            // zero-tile flags (planes of many tiles): long runs of +0.0 are
            // flagged instead of written, the gate kernel skips them
            uint8_t *zf = nullptr;
            if (zero_tiles_enabled(e)) {
                e->zold.ensure(2 * slots * ((e->L + kTile - 1) / kTile));
                zf = e->zold.p;
            }
            if (single) {
                decode_batch(e->st, e->dec[e->cur], e->arena[e->cur].p, e->blk_off[e->cur].p, e->outptrs.p,
                             (int)(2 * W), e->L, e->log2C, e->cfg.codec.quant_code_bits, /*prepare=*/false, nullptr, zf,
                             2 * slots);
            } else {
                e->h_wave_off.ensure(2 * W);
                for (uint64_t u = 0; u < W; ++u) {
                    const uint64_t k = map.slice_rel((uint32_t)u);
                    e->h_wave_off.p[2 * u] = e->blk_off_h[2 * k];
                    e->h_wave_off.p[2 * u + 1] = e->blk_off_h[2 * k + 1];
                }
                e->wave_off.ensure(2 * W);
                CK(cudaMemcpyAsync(e->wave_off.p, e->h_wave_off.p, 2 * W * 8, cudaMemcpyHostToDevice, e->st));
                decode_batch(e->st, e->decw, e->arena[e->cur].p, e->wave_off.p, e->outptrs.p, (int)(2 * W), e->L,
                             e->log2C, e->cfg.codec.quant_code_bits, /*prepare=*/true, nullptr, zf, 2 * slots);
            }
            if (remote) decode_imports(e, map, 0, W, 2 * W);
        }
        const auto src = make_src(map);
        EncodeResult R = encode_units(e, src, W, nxt, single);
        fb += R.fallback;
        for (uint64_t u = 0; u < W; ++u) {
            const uint64_t k = map.slice_rel((uint32_t)u);
            for (int p = 0; p < 2; ++p) {
                nbytes[2 * k + p] = R.block_bytes[2 * u + p];
                noff[2 * k + p] = e->enc.arena_base + R.blk_off[2 * u + p];
            }
            e->sq_norm[e->s0 + k] = e->h_sq.p[u];
        }
        e->enc.arena_base += R.total;
    }
    e->enc.arena_base = 0;
    e->blk_off[nxt].ensure(2 * e->ns);
    CK(cudaMemcpyAsync(e->blk_off[nxt].p, noff.data(), 2 * e->ns * 8, cudaMemcpyHostToDevice, e->st));
    CK(cudaEventRecord(e->ev1, e->st));
    CK(cudaEventSynchronize(e->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e->evg, e->ev1));
    e->blk_bytes_h = std::move(nbytes);
    e->blk_off_h = std::move(noff);
    e->fallback += fb;
    record_sizes(e, e->blk_bytes_h, ms * 1e-3);
    e->cur = nxt;
    e->loaded = true;
}

// Compression-off engine: one dense pass over all local slices.
template <class Src> void engine_dense(qcsim_engine *e, const Src &src) {
    const int nxt = e->cur ^ 1;
    const uint64_t ntiles = (e->L + kTile - 1) / kTile;
    CK(cudaEventRecord(e->evg, e->st));
    e->dense[nxt].ensure(e->ns * 2 * e->L);
    e->enc.tilesum.ensure(e->ns * ntiles);
    {
        PROF("dense_gate", e->st);
        launch_k(dense_gate<Src>, (unsigned)(e->ns * ntiles), 256, 0, e->st, src, (int)e->ns, e->L, e->dense[nxt].p,
                 e->enc.tilesum.p);
    }
    e->slice_sq.ensure(e->ns);
    {
        PROF("slice_norms", e->st);
        if (ntiles > 64 && ntiles <= 4096)
            launch_k(slice_norms_block, (unsigned)e->ns, 256, 0, e->st, e->enc.tilesum.p, (int)ntiles, (int)e->ns,
                     e->slice_sq.p);
        else
            launch_k(slice_norms, (unsigned)((e->ns + 127) / 128), 128, 0, e->st, e->enc.tilesum.p, (int)ntiles,
                     (int)e->ns, e->slice_sq.p);
    }
    e->h_sq.ensure(e->ns);
    CK(cudaMemcpyAsync(e->h_sq.p, e->slice_sq.p, e->ns * sizeof(double), cudaMemcpyDeviceToHost, e->st));
    CK(cudaEventRecord(e->ev1, e->st));
    CK(cudaEventSynchronize(e->ev1));
    g_prof.flush();
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e->evg, e->ev1));
    for (uint64_t k = 0; k < e->ns; ++k) e->sq_norm[e->s0 + k] = e->h_sq.p[k];
    e->rows.push_back(GateRow{0.0, 0.0, 0, 16ull * e->ns * e->L, 0, ms * 1e-3});
    e->cur = nxt;
    e->loaded = true;
}

// Deferred pass (single batch, identity layout, no host round trip): decode
// (its extra block runs the normalization and the previous pass's metrics),
// gate, encode with device-side run metrics.
void engine_deferred_pass(qcsim_engine *e, const GateSrc &g0) {
    const int nxt = e->cur ^ 1;
    ensure_outptrs(e, 2 * e->ns);
    // from the second pass of a run on, the blocks being decoded were written
    // by the previous pass, whose fine checkpoints are still in e->index:
    // one decode chunk per checkpoint instead of per stored record
    // (QCSIM_FINE_DECODE=0: the stored records only)
    static const bool fine_off = std::getenv("QCSIM_FINE_DECODE") && std::getenv("QCSIM_FINE_DECODE")[0] == '0';
    const IndexRec *fine = (!fine_off && !e->defer_fresh && e->index.p) ? e->index.p : nullptr;
    decode_batch(e->st, e->dec[e->cur], e->arena[e->cur].p, e->blk_off[e->cur].p, e->outptrs.p, (int)(2 * e->ns),
                 e->L, e->log2C, e->cfg.codec.quant_code_bits, /*prepare=*/false, &e->norm, nullptr, 0, fine);
    e->norm.enabled = 0;
    GateSrc g = g0;
    g.old = e->old.p;
    e->index.ensure(2 * e->ns * e->nidx);
    e->dec[nxt].ensure(2 * e->ns, e->L, e->cfg.codec.quant_code_bits);
    e->enc.dec_out = e->dec[nxt].tables();
    e->enc.stats_out = e->dev_stats.p;
    e->enc.stats_gate = e->gates;
    e->enc.rows_out = e->dev_rows.p;
    e->enc.row0 = e->row0;
    e->enc.nrows = e->nrows;
    e->blk_off[nxt].ensure(2 * e->ns);
    e->enc.blk_off_out = e->blk_off[nxt].p;
    encode_launch<2, GateSrc>(e->st, e->enc, g, (int)e->ns, e->L, e->cfg.codec, e->log2C, e->index.p,
                              e->arena[nxt], false, false, /*host_results=*/false);
    e->enc.dec_out = DecTables{};
    e->enc.stats_out = nullptr;
    e->enc.blk_off_out = nullptr;
    e->defer_fresh = false; // slice norms: next pass's engine_norm, or engine_defer_end
    e->cur = nxt;
}

// Frees the gate-pass scratch (encoder buffers, parsed decode tables,
// decoded planes, fine index, idle arena); the compressed state stays.
void engine_release_scratch(qcsim_engine *e) {
    e->enc.~EncScratch();
    new (&e->enc) EncScratch();
    e->decw.~DecScratch();
    new (&e->decw) DecScratch();
    e->old.release();
    e->outptr_planes = 0;
    e->index.release();
    e->arena[e->cur ^ 1].release();
    e->dec[e->cur ^ 1].~DecScratch();
    new (&e->dec[e->cur ^ 1]) DecScratch();
}

double g_host_t[4] = {0, 0, 0, 0}; // debug (QCSIM_ENQ_TIMING): gate prologue, decode, encode, total
void engine_gate(qcsim_engine *e, const qcsim_action &a) {
    const auto ht0 = std::chrono::steady_clock::now();
    if (a.kind > 2) raise(QCSIM_INVALID_ARGUMENT, "unknown action kind");
    if (a.kind == QCSIM_ACTION_BUTTERFLY && (a.target < 0 || a.target >= e->n))
        raise(QCSIM_INVALID_ARGUMENT, "action qubit out of range");
    if (a.kind == QCSIM_ACTION_SWAP && (a.a < 0 || a.a >= e->n || a.b < 0 || a.b >= e->n || a.a == a.b))
        raise(QCSIM_INVALID_ARGUMENT, "action qubit out of range");
    // normalization, computed on the host from the
    // deterministic tree over every slice's sq_norm
    const bool apply = e->cfg.norm_every > 0 && (e->gates % (uint64_t)e->cfg.norm_every) == 0;
    double scale = 1.0;
    e->norm = NormArgs{};
    if (e->deferred) {
        // run by the decoder grid's extra block: the previous pass's run
        // metrics (none before the first pass), then the slice norms of the
        // previous pass from its tile partials (or, for the first gate of a
        // run, the norms uploaded by engine_defer_begin) and the scale
        NormArgs &N = e->norm;
        N.norm = apply ? 1 : 0;
        N.tilesum = e->defer_fresh ? nullptr : e->enc.tilesum.p;
        N.ntiles = (int)((e->L + kTile - 1) / kTile);
        N.sq = e->slice_sq.p;
        N.b0 = e->norm_buf[0].p;
        N.b1 = e->norm_buf[1].p;
        N.S = e->S;
        N.tol10 = 10.0 * e->cfg.norm_drift_tolerance;
        N.gate = (unsigned long long)e->gates;
        N.scale = e->dev_scale.p;
        N.overflow = e->defer_fresh ? nullptr : e->enc.overflow.p;
        N.st = e->dev_stats.p;
        N.stats = (e->defer_fresh || !e->enc.fixed_W) ? 0 : 1; // (packed slots: slot_scan_stats counts)
        N.bytes = e->enc.block_bytes.p;
        N.err = e->enc.err.p;
        N.params = e->enc.params.p;
        N.planes = (int)(2 * e->ns);
        N.L = e->L;
        N.log2C = e->log2C;
        N.stats_gate = (unsigned long long)e->gates - 1;
        N.rows = e->dev_rows.p;
        N.row0 = e->row0;
        N.nrows = e->nrows;
        N.stamp = e->defer_fresh ? 1 : 0;
        N.enabled = N.norm || N.stats || N.stamp;
    } else if (apply) {
        const double G = tree_sum_host(e->sq_norm.data(), e->S);
        if (!std::isfinite(G) || std::fabs(G - 1.0) > 10.0 * e->cfg.norm_drift_tolerance) {
            char buf[160];
            std::snprintf(buf, sizeof buf, "norm drift before gate %llu: global sq_norm %.17g",
                          (unsigned long long)e->gates, G);
            raise(QCSIM_NUMERIC, buf);
        }
        scale = 1.0 / std::sqrt(G);
    }
    const uint64_t hm = partner_mask(a, e->s);
    const bool remote = (hm & ~(e->ns - 1)) != 0; // partner slices on other ranks
    GateSrc g;
    g.old = e->old.p;
    g.scale = scale;
    g.scale_dev = e->deferred ? e->dev_scale.p : nullptr;
    g.apply_scale = apply ? 1 : 0;
    g.act = to_dev(a);
    g.s = e->s;
    g.L = e->L;
    g.map.s0 = e->s0;
    g.map.hm = hm;
    g.map.nunits = (uint32_t)e->ns;
    const auto ht1 = std::chrono::steady_clock::now();
    if (e->deferred) {
        engine_deferred_pass(e, g);
    } else if (!e->compressed) {
        if (remote) raise(QCSIM_INVALID_ARGUMENT, "compression-off engines do not exchange partner slices");
        g.old = e->dense[e->cur].p;
        engine_dense(e, g);
    } else {
        for (;;) {
            try {
                engine_waves(e, hm, remote, /*decode=*/true, [&](const SliceMap &map) {
                    GateSrc b = g;
                    b.old = e->old.p;
                    b.map = map;
                    b.zold = zero_tiles_enabled(e) ? e->zold.p : nullptr;
                    b.ztiles = (uint32_t)((e->L + kTile - 1) / kTile);
                    return b;
                });
                break;
            } catch (const Fail &f) {
                // the compressed state grew into the scratch's room: smaller
                // waves, then the pass again (it only read arena[cur])
                if (f.st != QCSIM_NOMEM || e->wave <= std::min<uint64_t>(4, e->ns)) throw;
                CK(cudaStreamSynchronize(e->st));
                cudaGetLastError();
                engine_release_scratch(e);
                e->wave /= 2;
            }
        }
    }
    const auto ht2 = std::chrono::steady_clock::now();
    g_host_t[0] += std::chrono::duration<double, std::micro>(ht1 - ht0).count();
    g_host_t[2] += std::chrono::duration<double, std::micro>(ht2 - ht1).count();
    g_host_t[3] += std::chrono::duration<double, std::micro>(ht2 - ht0).count();
    e->gates++;
    e->imported.clear();
    e->dev_imp = nullptr;
    e->dev_imp_at.clear();
}

// Worst-case arena bytes for one gate pass (every plane at qcsim_block_bound,
// 16-byte slots, the largest decode index): with arenas that large a pass
// cannot overflow, so the gate loop needs no host round trip.
uint64_t fixed_slot_bytes(const qcsim_engine *e) {
    const uint64_t L = e->L;
    uint64_t nsym = (1ull << e->cfg.codec.quant_code_bits) + 1;
    if (nsym > L + 1) nsym = L + 1;
    const uint64_t bound = kHeaderBytes + 4 + 5 * nsym + (L * kMaxCodeLen + 7) / 8 + 16 + L * 16;
    // >= 16 + round_up(block bytes, 16) + its decode index: every slot_bytes fits
    return ((bound + 31) & ~15ull) + ((((L >> e->log2C) + 1) * sizeof(IndexRec) + 15) & ~15ull);
}
uint64_t arena_worst(const qcsim_engine *e) { return 2 * e->ns * fixed_slot_bytes(e) + (1 << 20); }

// Deferred gate loop: single rank, compressed, one batch, worst-case arenas
// within the budget (QCSIM_SYNC_GATES=1 forces the per-gate host round trip).
bool engine_defer_begin(qcsim_engine *e, uint64_t count) {
    static const bool forced_sync = std::getenv("QCSIM_SYNC_GATES") != nullptr;
    constexpr uint64_t kBudget = 8ull << 30;
    const uint64_t worst = arena_worst(e);
    if (forced_sync || e->cfg.world > 1 || !e->compressed || e->wave != e->ns || 2 * worst > kBudget ||
        !e->imported.empty() || e->dev_imp)
        return false;
    CK(cudaStreamSynchronize(e->st));
    {
        // current arena: keep its contents (up to the highest slot end)
        uint64_t hi = 0;
        for (uint64_t k = 0; k < e->blk_off_h.size(); ++k)
            hi = std::max(hi, index_offset(e->blk_off_h[k], e->blk_bytes_h[k]) +
                                  index_records(e->L, e->blk_bytes_h[k], e->log2C) * sizeof(IndexRec));
        grow_keep(e->arena[e->cur], worst, hi, e->st);
        grow_keep(e->arena[e->cur ^ 1], worst, 0, e->st);
    }
    e->enc.ensure(2 * e->ns, e->ns, e->L, e->cfg.codec.quant_code_bits);
    e->slice_sq.ensure(e->ns);
    e->norm_buf[0].ensure(e->S);
    e->norm_buf[1].ensure(e->S);
    e->dev_scale.ensure(1);
    e->dev_stats.ensure(1);
    e->h_stats.ensure(1);
    e->h_sq.ensure(e->ns);
    e->row0 = e->gates;
    e->nrows = count;
    e->dev_rows.ensure(count + 1);
    e->h_rows.ensure(count + 1);
    CK(cudaMemsetAsync(e->dev_rows.p, 0, (count + 1) * sizeof(GateRowDev), e->st));
    // the host view is authoritative between runs
    for (uint64_t k = 0; k < e->ns; ++k) e->h_sq.p[k] = e->sq_norm[e->s0 + k];
    CK(cudaMemcpyAsync(e->slice_sq.p, e->h_sq.p, e->ns * sizeof(double), cudaMemcpyHostToDevice, e->st));
    EngineDevStats &h = *e->h_stats.p;
    std::memset(&h, 0, sizeof h);
    h.ratio_min = e->ratio_min;
    h.ratio_sum = e->ratio_sum;
    h.calls = e->calls;
    h.current = e->current;
    h.peak = e->peak;
    h.fallback = e->fallback;
    CK(cudaMemcpyAsync(e->dev_stats.p, e->h_stats.p, sizeof h, cudaMemcpyHostToDevice, e->st));
    CK(cudaStreamSynchronize(e->st));
    e->deferred = true;
    e->defer_fresh = true;
    // one worst-case slot per plane: no slot scan per pass (QCSIM_FIXED_SLOTS=0
    // keeps the packed layout)
    static const int fixed_env = std::getenv("QCSIM_FIXED_SLOTS") ? std::atoi(std::getenv("QCSIM_FIXED_SLOTS")) : 1;
    const bool fixed = fixed_env != 0;
    e->enc.fixed_W = fixed ? fixed_slot_bytes(e) : 0;
    return true;
}

// The deferred run's last kernels (inside the timed region): the last
// pass's run metrics and slice norms.
void engine_defer_finish(qcsim_engine *e) {
    const bool fixed = e->enc.fixed_W != 0;
    if (!e->defer_fresh && fixed) { // run metrics of the last pass (the others: the next pass's decoder grid)
        NormArgs N{};
        N.st = e->dev_stats.p;
        N.stats = 1;
        N.bytes = e->enc.block_bytes.p;
        N.err = e->enc.err.p;
        N.params = e->enc.params.p;
        N.planes = (int)(2 * e->ns);
        N.L = e->L;
        N.log2C = e->log2C;
        N.stats_gate = (unsigned long long)e->gates - 1;
        N.rows = e->dev_rows.p;
        N.row0 = e->row0;
        N.nrows = e->nrows;
        PROF("pass_stats", e->st);
        launch_k(pass_stats_kernel, 1, 256, 0, e->st, N);
    }
    if (!e->defer_fresh) { // slice norms of the last pass, from its tile partials
        const uint64_t ntiles = (e->L + kTile - 1) / kTile;
        PROF("slice_norms", e->st);
        launch_k(slice_norms, (unsigned)((e->ns + 127) / 128), 128, 0, e->st, e->enc.tilesum.p, (int)ntiles, (int)e->ns,
                 e->slice_sq.p);
    }
}

// Settles a deferred run: metrics, norms, block sizes and offsets back to
// the host, latched errors raised.
void engine_defer_end(qcsim_engine *e, bool raise_errors, uint64_t done) {
    e->deferred = false;
    e->enc.fixed_W = 0;
    uint32_t ovf = 0;
    if (!e->defer_fresh) CK(cudaMemcpyAsync(&ovf, e->enc.overflow.p, 4, cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    g_prof.flush();
    CK(cudaGetLastError());
    CK(cudaMemcpy(e->h_stats.p, e->dev_stats.p, sizeof(EngineDevStats), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(e->h_sq.p, e->slice_sq.p, e->ns * sizeof(double), cudaMemcpyDeviceToHost));
    const EngineDevStats h = *e->h_stats.p;
    e->ratio_min = h.ratio_min;
    e->ratio_sum = h.ratio_sum;
    e->calls = h.calls;
    e->current = h.current;
    e->peak = h.peak;
    e->fallback = h.fallback;
    for (uint64_t k = 0; k < e->ns; ++k) e->sq_norm[e->s0 + k] = e->h_sq.p[k];
    e->blk_bytes_h.resize(2 * e->ns);
    e->blk_off_h.resize(2 * e->ns);
    CK(cudaMemcpy(e->blk_bytes_h.data(), e->enc.block_bytes.p, 2 * e->ns * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(e->blk_off_h.data(), e->blk_off[e->cur].p, 2 * e->ns * 8, cudaMemcpyDeviceToHost));
    // per-gate rows (seconds from the passes' global-timer stamps)
    if (done) {
        CK(cudaMemcpy(e->h_rows.p, e->dev_rows.p, (done + 1) * sizeof(GateRowDev), cudaMemcpyDeviceToHost));
        for (uint64_t k = 0; k < done; ++k) {
            const GateRowDev &r = e->h_rows.p[k + 1];
            const uint64_t t_prev = e->h_rows.p[k].t_ns;
            e->rows.push_back(GateRow{r.min_ratio, r.ratio_sum, r.calls, r.bytes, r.index_bytes,
                                      (t_prev && r.t_ns > t_prev) ? (double)(r.t_ns - t_prev) * 1e-9 : 0.0});
        }
    }
    if (!raise_errors) return;
    if (h.status == kEngNumeric) {
        // the gates queued after the failing one ran on an unnormalized
        // state: the engine must be reloaded (the host-synchronous path keeps
        // the failing gate's input instead)
        e->gates = h.status_gate;
        e->loaded = false;
        char buf[160];
        std::snprintf(buf, sizeof buf, "norm drift before gate %llu: global sq_norm %.17g",
                      (unsigned long long)h.status_gate, h.norm_G);
        raise(QCSIM_NUMERIC, buf);
    }
    if (h.status == kEngDepth) raise(QCSIM_CODEC, "prefix code depth out of range");
    if (h.status == kEngOverflow || ovf) raise(QCSIM_NOMEM, "compressed arena overflow");
}

// Decode-index bytes stored next to the current blocks (common.cuh).
uint64_t engine_index_bytes(const qcsim_engine *e) {
    if (!e->compressed) return 0;
    uint64_t t = 0;
    for (uint64_t b : e->blk_bytes_h) t += index_records(e->L, b, e->log2C) * sizeof(IndexRec);
    return t;
}

} // namespace

// ================================================================== C-ABI
extern "C" {

const char *qcsim_last_error(void) { return g_err.c_str(); }
const char *qcsim_version(void) { return QCSIM_VERSION; }

uint64_t qcsim_kernel_launches(void) { return g_launches; }

// Per-kernel device time (CUDA events) -- bench.py instrumentation.
int qcsim_profile_enable(int on) {
    g_prof.flush();
    g_prof.on = on != 0;
    if (on) g_prof.acc.clear();
    return 0;
}
int qcsim_profile_read(char (*names)[64], double *ms, uint64_t *count, double *bytes, int cap) {
    g_prof.flush();
    int k = 0;
    for (auto &kv : g_prof.acc) {
        if (k >= cap) break;
        std::snprintf(names[k], 64, "%s", kv.first.c_str());
        ms[k] = kv.second.first;
        count[k] = kv.second.second;
        bytes[k] = 0.0;
        ++k;
    }
    return k;
}

// Debug (not part of the public header): enc_chain_scan counters since the
// last call ([0] resolve points, [1] refuted chunks, [2] serial chunks,
// [3..4] events chained, u64 little-endian).
qcsim_status qcsim_debug_chain_stats(uint32_t *out3) { // out3[5]
    return guarded([&] {
        CK(cudaDeviceSynchronize());
        uint32_t v[16];
        CK(cudaMemcpy(v, chain_stats(), sizeof v, cudaMemcpyDeviceToHost));
        if (std::getenv("QCSIM_CHAIN_DEBUG"))
            std::fprintf(stderr, "chain maps: W0 %u W1 %u W2 %u W3 %u const %u poison %u\n", v[8], v[9], v[10], v[11],
                         v[13], v[14]);
        out3[0] = v[0];
        out3[1] = v[1];
        out3[2] = v[4];
        out3[3] = v[6]; // events (low, high words of a u64)
        out3[4] = v[7];
        CK(cudaMemset(chain_stats(), 0, sizeof v));
    });
}

// Debug (not part of the public header): encoder intermediates for one plane.
// sym[n], tsym/trep[n+1], flags = plane flags, idx = [n/C + 1] records.
qcsim_status qcsim_debug_encode(const double *values, uint64_t n, const qcsim_codec_config *cfg, uint32_t *sym,
                                uint32_t *tsym, uint32_t *trep, uint64_t *ntok, uint32_t *flags, void *idx,
                                int32_t *log2C_out) {
    return guarded([&] {
        validate_codec(*cfg);
        CodecCtx &C = codec_ctx();
        C.vals.ensure(n);
        CK(cudaMemcpy(C.vals.p, values, n * sizeof(double), cudaMemcpyHostToDevice));
        C.ptrs.ensure(1);
        const double *vp = C.vals.p;
        CK(cudaMemcpy(C.ptrs.p, &vp, sizeof vp, cudaMemcpyHostToDevice));
        RawSrc src{C.ptrs.p};
        const int log2C = auto_log2C(n);
        C.index.ensure(((n >> log2C) + 1));
        encode_batch<1, RawSrc>(C.st, C.enc, src, 1, n, *cfg, log2C, C.index.p, C.arena, true, true);
        uint32_t nt = 0;
        CK(cudaMemcpy(&nt, C.enc.ntok.p, 4, cudaMemcpyDeviceToHost));
        *ntok = nt;
        CK(cudaMemcpy(sym, C.enc.sym.p, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tsym, C.enc.tsym.p, (n + 1) * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(trep, C.enc.trep.p, (n + 1) * 4, cudaMemcpyDeviceToHost));
        PlaneParams pp;
        CK(cudaMemcpy(&pp, C.enc.params.p, sizeof pp, cudaMemcpyDeviceToHost));
        *flags = pp.flags;
        CK(cudaMemcpy(idx, C.index.p, ((n >> log2C) + 1) * sizeof(IndexRec), cudaMemcpyDeviceToHost));
        *log2C_out = log2C;
    });
}

qcsim_status qcsim_codec_validate(const qcsim_codec_config *cfg) {
    return guarded([&] {
        if (!cfg) raise(QCSIM_INVALID_ARGUMENT, "null config");
        validate_codec(*cfg);
    });
}

uint64_t qcsim_block_bound(uint64_t n, int32_t qb) {
    uint64_t nsym = (1ull << qb) + 1;
    if (nsym > n + 1) nsym = n + 1;
    return kHeaderBytes + 4 + 5 * nsym + (n * kMaxCodeLen + 7) / 8 + 16 + n * 16;
}

qcsim_status qcsim_compress_plane(const double *values, uint64_t n, const qcsim_codec_config *cfg, uint8_t *out,
                                  uint64_t capacity, uint64_t *out_len, qcsim_codec_stats *stats) {
    return guarded([&] {
        if (!cfg) raise(QCSIM_INVALID_ARGUMENT, "null config");
        validate_codec(*cfg);
        if (n == 0) raise(QCSIM_INVALID_ARGUMENT, "cannot compress an empty plane");
        if (n >= (1ull << 32)) raise(QCSIM_CAPACITY, "plane longer than 2^32 elements");
        CodecCtx &C = codec_ctx();
        C.vals.ensure(n);
        CK(cudaMemcpyAsync(C.vals.p, values, n * sizeof(double), cudaMemcpyHostToDevice, C.st));
        C.ptrs.ensure(1);
        const double *vp = C.vals.p;
        CK(cudaMemcpyAsync(C.ptrs.p, &vp, sizeof vp, cudaMemcpyHostToDevice, C.st));
        RawSrc src{C.ptrs.p};
        const int log2C = auto_log2C(n);
        C.index.ensure(((n >> log2C) + 1));
        EncodeResult R = encode_batch<1, RawSrc>(C.st, C.enc, src, 1, n, *cfg, log2C, C.index.p, C.arena, true, true);
        const uint64_t len = R.block_bytes[0];
        if (out_len) *out_len = len;
        if (stats) {
            stats->input_bytes = 8 * n;
            stats->output_bytes = len;
            stats->ratio = (double)stats->input_bytes / (double)len;
            uint32_t no = 0;
            CK(cudaMemcpy(&no, C.enc.ocount.p, 4, cudaMemcpyDeviceToHost));
            stats->outlier_fraction = (double)no / (double)n;
        }
        if (out) {
            if (len > capacity) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
            CK(cudaMemcpyAsync(out, C.arena.p + R.blk_off[0], len, cudaMemcpyDeviceToHost, C.st));
            CK(cudaStreamSynchronize(C.st));
        }
    });
}

qcsim_status qcsim_decompress_plane(const uint8_t *block, uint64_t len, double *out, uint64_t capacity,
                                    uint64_t *n_out, uint64_t *consumed) {
    return guarded([&] {
        uint64_t used = 0;
        Header h = parse_header(block, len, &used);
        if (consumed) *consumed = used;
        if (n_out) *n_out = h.n;
        if (!out) return;
        if (h.n > capacity) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        CodecCtx &C = codec_ctx();
        C.vals.ensure(h.n);
        uint32_t tc = 0;
        if (h.payload >= 4) tc = (uint32_t)(block[40] | (block[41] << 8) | (block[42] << 16) | ((uint32_t)block[43] << 24));
        // validating token walk + chunk-parallel decode (foreign_decode)
        const uint32_t e = foreign_decode(C.st, C.fore, {ForeignBlock{block, used, tc, h.payload, C.vals.p}}, false, h.n,
                                          h.qb);
        if (e) raise(QCSIM_CODEC, dec_message(e));
        CK(cudaMemcpyAsync(out, C.vals.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, C.st));
        CK(cudaStreamSynchronize(C.st));
    });
}

qcsim_status qcsim_compress_planes_device(const double *const *values, const uint64_t *n, uint32_t planes,
                                          const qcsim_codec_config *cfg, uint8_t *out, uint64_t capacity,
                                          uint64_t *offsets_host, qcsim_codec_stats *stats_host, void *stream) {
    return guarded([&] {
        if (!cfg) raise(QCSIM_INVALID_ARGUMENT, "null config");
        validate_codec(*cfg);
        if (planes == 0) return;
        for (uint32_t p = 1; p < planes; ++p)
            if (n[p] != n[0]) raise(QCSIM_INVALID_ARGUMENT, "batched planes must have equal length");
        if (n[0] == 0) raise(QCSIM_INVALID_ARGUMENT, "cannot compress an empty plane");
        CodecCtx &C = codec_ctx();
        cudaStream_t st = stream ? (cudaStream_t)stream : C.st;
        C.ptrs.ensure(planes);
        CK(cudaMemcpyAsync(C.ptrs.p, values, planes * sizeof(double *), cudaMemcpyHostToDevice, st));
        const uint64_t L = n[0];
        const int log2C = auto_log2C(L);
        C.index.ensure(planes * ((L >> log2C) + 1));
        RawSrc src{C.ptrs.p};
        EncodeResult R =
            encode_batch<1, RawSrc>(st, C.enc, src, (int)planes, L, *cfg, log2C, C.index.p, C.arena, true, true);
        uint64_t o = 0;
        for (uint32_t p = 0; p < planes; ++p) {
            offsets_host[p] = o;
            o += R.block_bytes[p];
        }
        offsets_host[planes] = o;
        if (o > capacity) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        for (uint32_t p = 0; p < planes; ++p) {
            CK(cudaMemcpyAsync(out + offsets_host[p], C.arena.p + R.blk_off[p], R.block_bytes[p],
                               cudaMemcpyDeviceToDevice, st));
            if (stats_host) {
                stats_host[p].input_bytes = 8 * L;
                stats_host[p].output_bytes = R.block_bytes[p];
                stats_host[p].ratio = (double)(8 * L) / (double)R.block_bytes[p];
            }
        }
        if (stats_host) {
            std::vector<uint32_t> oc(planes);
            CK(cudaMemcpyAsync(oc.data(), C.enc.ocount.p, planes * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
    g_prof.flush();
            for (uint32_t p = 0; p < planes; ++p) stats_host[p].outlier_fraction = (double)oc[p] / (double)L;
        }
        CK(cudaStreamSynchronize(st));
    g_prof.flush();
    });
}

qcsim_status qcsim_decompress_planes_device(const uint8_t *blocks, const uint64_t *offsets_host, uint32_t planes,
                                            double *const *out, const uint64_t *capacity, void *stream) {
    return guarded([&] {
        if (planes == 0) return;
        CodecCtx &C = codec_ctx();
        cudaStream_t st = stream ? (cudaStream_t)stream : C.st;
        // header checks on the host copy of each header (from_bytes order)
        std::vector<ForeignBlock> fb(planes);
        std::vector<uint64_t> ns(planes);
        std::vector<int> qbs(planes);
        for (uint32_t p = 0; p < planes; ++p) {
            uint8_t hdr[44] = {};
            const uint64_t avail = offsets_host[p + 1] - offsets_host[p];
            CK(cudaMemcpy(hdr, blocks + offsets_host[p], std::min<uint64_t>(44, avail), cudaMemcpyDeviceToHost));
            uint64_t used = 0;
            Header h = parse_header(hdr, avail, &used);
            if (h.n > capacity[p]) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
            const uint32_t tc = h.payload >= 4 ? (uint32_t)(hdr[40] | (hdr[41] << 8) | (hdr[42] << 16) | ((uint32_t)hdr[43] << 24)) : 0;
            fb[p] = ForeignBlock{blocks + offsets_host[p], used, tc, h.payload, out[p]};
            ns[p] = h.n;
            qbs[p] = h.qb;
        }
        // one foreign_decode per run of planes with the same element count
        for (uint32_t p0 = 0; p0 < planes;) {
            uint32_t p1 = p0 + 1;
            while (p1 < planes && ns[p1] == ns[p0]) ++p1;
            std::vector<ForeignBlock> part(fb.begin() + p0, fb.begin() + p1);
            const uint32_t e = foreign_decode(st, C.fore, part, true, ns[p0], qbs[p0]);
            if (e) raise(QCSIM_CODEC, dec_message(e));
            p0 = p1;
        }
        g_prof.flush();
    });
}

// ------------------------------------------------------------- engine API
qcsim_status qcsim_engine_create(const qcsim_engine_config *cfg, qcsim_engine **out) {
    return guarded([&] {
        if (!cfg || !out) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        *out = nullptr;
        const qcsim_engine_config &c = *cfg;
        if (c.num_qubits < 1 || c.num_qubits > 62) raise(QCSIM_INVALID_ARGUMENT, "qubit count must be in [1, 62]");
        int s = c.slice_bits < 0 ? std::min(c.num_qubits, 20) : c.slice_bits;
        if (s < 0 || s > c.num_qubits) raise(QCSIM_INVALID_ARGUMENT, "slice_bits must be in [0, num_qubits]");
        if (s > 22) raise(QCSIM_CAPACITY, "slice_bits above 22 not supported on the device path");
        if (c.compression_enabled) validate_codec(c.codec);
        if (!(c.norm_drift_tolerance >= 0.0)) raise(QCSIM_INVALID_ARGUMENT, "norm drift tolerance must be >= 0");
        if (c.norm_every < 0) raise(QCSIM_INVALID_ARGUMENT, "norm_every must be >= 0");
        const int world = c.world > 0 ? c.world : 1;
        const uint64_t S = 1ull << (c.num_qubits - s);
        if (c.rank < 0 || c.rank >= world || S % (uint64_t)world) raise(QCSIM_INVALID_ARGUMENT, "bad rank/world for slice count");
        if (((S / (uint64_t)world) & (S / (uint64_t)world - 1)) != 0)
            raise(QCSIM_INVALID_ARGUMENT, "world size must be a power of two");
        ensure_device(c.device);
        auto *e = new qcsim_engine();
        e->cfg = c;
        e->cfg.slice_bits = s;
        e->cfg.world = world;
        e->n = c.num_qubits;
        e->s = s;
        e->S = S;
        e->L = 1ull << s;
        e->ns = S / (uint64_t)world;
        e->s0 = (uint64_t)c.rank * e->ns;
        e->log2C = c.checkpoint_bits > 0 ? c.checkpoint_bits : auto_log2C(e->L);
        e->nidx = (e->L >> e->log2C) + 1;
        e->compressed = c.compression_enabled != 0;
        e->wave = choose_wave(e);
        e->sq_norm.assign(S, 0.0);
        e->launches0 = g_launches;
        cudaError_t err = cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking);
        if (err != cudaSuccess) {
            delete e;
            ck(err, "cudaStreamCreate");
        }
        CK(cudaEventCreate(&e->ev0));
        CK(cudaEventCreate(&e->ev1));
        CK(cudaEventCreate(&e->evg));
        *out = e;
    });
}

qcsim_status qcsim_engine_destroy(qcsim_engine *e) {
    return guarded([&] {
        if (!e) return;
        if (e->st) cudaStreamSynchronize(e->st);
        if (e->ev0) cudaEventDestroy(e->ev0);
        if (e->ev1) cudaEventDestroy(e->ev1);
        if (e->evg) cudaEventDestroy(e->evg);
        if (e->st) cudaStreamDestroy(e->st);
        delete e;
    });
}

qcsim_status qcsim_engine_load_basis(qcsim_engine *e, uint64_t x) {
    return guarded([&] {
        if (!e) raise(QCSIM_INVALID_ARGUMENT, "null engine");
        if (x >= (1ull << e->n)) raise(QCSIM_INVALID_ARGUMENT, "basis index out of range");
        CK(cudaSetDevice(e->cfg.device));
        std::fill(e->sq_norm.begin(), e->sq_norm.end(), 0.0);
        e->rows.clear();
        const uint64_t xs = x >> e->s;
        if (e->compressed) {
            engine_waves(e, 0, false, /*decode=*/false, [&](const SliceMap &map) { return BasisSrc{x, map, e->s}; });
        } else {
            SliceMap id;
            id.s0 = e->s0;
            id.nunits = (uint32_t)e->ns;
            engine_dense(e, BasisSrc{x, id, e->s});
        }
        // the owner knows the only nonzero norm; keep the global view exact
        e->sq_norm[xs] = 1.0;
    });
}

qcsim_status qcsim_engine_load_amplitudes(qcsim_engine *e, const double *amps, uint64_t count) {
    return guarded([&] {
        if (!e || !amps) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (count != (1ull << e->n)) raise(QCSIM_INVALID_ARGUMENT, "amplitude count must be 2^n");
        CK(cudaSetDevice(e->cfg.device));
        e->rows.clear();
        // the planar [slot][re|im][L] layout of local slices [k0, k0 + cnt)
        auto upload = [&](uint64_t k0, uint64_t cnt) {
            std::vector<double> planar(cnt * 2 * e->L);
            for (uint64_t k = 0; k < cnt; ++k)
                for (uint64_t i = 0; i < e->L; ++i) {
                    const uint64_t g = ((e->s0 + k0 + k) << e->s) | i;
                    planar[k * 2 * e->L + i] = amps[2 * g];
                    planar[k * 2 * e->L + e->L + i] = amps[2 * g + 1];
                }
            e->old.ensure(cnt * 2 * e->L);
            CK(cudaMemcpyAsync(e->old.p, planar.data(), planar.size() * sizeof(double), cudaMemcpyHostToDevice, e->st));
            CK(cudaStreamSynchronize(e->st));
        };
        if (e->compressed) {
            engine_waves(e, 0, false, /*decode=*/false, [&](const SliceMap &map) {
                upload(map.slice_rel(0), map.nunits);
                return PlanarSrc{e->old.p, e->L};
            });
        } else {
            upload(0, e->ns);
            engine_dense(e, PlanarSrc{e->old.p, e->L});
        }
    });
}

qcsim_status qcsim_engine_load_blocks(qcsim_engine *e, const uint8_t *blocks, uint64_t len, const uint64_t *offsets,
                                      uint64_t planes, const double *sq_norms, uint64_t norm_count,
                                      uint64_t gates_done) {
    return guarded([&] {
        if (!e || !blocks || !offsets || !sq_norms) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (!e->compressed) raise(QCSIM_INVALID_ARGUMENT, "engine is not compressed");
        if (e->cfg.codec.mode == QCSIM_MODE_RANGE_RELATIVE)
            raise(QCSIM_INVALID_ARGUMENT, "resume needs an absolute or lossless bound");
        if (planes != 2 * e->ns) raise(QCSIM_INVALID_ARGUMENT, "block count must be 2 * local slices");
        if (norm_count != e->S) raise(QCSIM_INVALID_ARGUMENT, "norm table must hold every slice");
        for (uint64_t k = 0; k < planes; ++k)
            if (offsets[k + 1] < offsets[k] || offsets[k + 1] > len)
                raise(QCSIM_INVALID_ARGUMENT, "block offsets must be non-decreasing and inside the buffer");
        CK(cudaSetDevice(e->cfg.device));
        // from_bytes checks of every block first (nothing is replaced on failure)
        std::vector<Header> hd(planes);
        std::vector<uint64_t> used(planes);
        for (uint64_t k = 0; k < planes; ++k) {
            hd[k] = parse_header(blocks + offsets[k], offsets[k + 1] - offsets[k], &used[k]);
            const Header &h = hd[k];
            if (h.n != e->L) raise(QCSIM_INVALID_ARGUMENT, "block element count does not match the slice");
            if (h.mode != e->cfg.codec.mode || h.pred != e->cfg.codec.predictor || h.qb != e->cfg.codec.quant_code_bits)
                raise(QCSIM_INVALID_ARGUMENT, "block codec (mode, predictor, quant_code_bits) differs from the engine's");
        }
        e->rows.clear();
        e->loaded = false;
        engine_waves(e, 0, false, /*decode=*/false, [&](const SliceMap &map) {
            // this wave's slices, decoded by the validating foreign decoder
            const uint64_t W = map.nunits;
            e->old.ensure(2 * W * e->L);
            std::vector<ForeignBlock> fb(2 * W);
            for (uint64_t u = 0; u < W; ++u) {
                const uint64_t k = map.slice_rel((uint32_t)u);
                for (int p = 0; p < 2; ++p) {
                    const uint64_t b = 2 * k + p;
                    const uint8_t *src = blocks + offsets[b];
                    const uint32_t tc = hd[b].payload >= 4 ? (uint32_t)(src[40] | (src[41] << 8) | (src[42] << 16) |
                                                                        ((uint32_t)src[43] << 24))
                                                           : 0;
                    fb[2 * u + p] = ForeignBlock{src, used[b], tc, hd[b].payload, e->old.p + (2 * u + p) * e->L};
                }
            }
            const uint32_t err = foreign_decode(e->st, e->fore, fb, false, e->L, e->cfg.codec.quant_code_bits);
            if (err) raise(QCSIM_CODEC, dec_message(err));
            return PlanarSrc{e->old.p, e->L};
        });
        for (uint64_t k = 0; k < planes; ++k)
            if (e->blk_bytes_h[k] != used[k]) {
                e->loaded = false;
                raise(QCSIM_CODEC, "block " + std::to_string(k) + " does not re-encode to itself (" +
                                       std::to_string(used[k]) + " -> " + std::to_string(e->blk_bytes_h[k]) + " bytes)");
            }
        // the cached norms are those of the pre-compression values
        std::memcpy(e->sq_norm.data(), sq_norms, e->S * sizeof(double));
        e->gates = gates_done;
    });
}

qcsim_status qcsim_engine_run(qcsim_engine *e, const qcsim_action *actions, uint64_t count,
                              qcsim_run_metrics *m) {
    return guarded([&] {
        if (!e) raise(QCSIM_INVALID_ARGUMENT, "null engine");
        if (!e->loaded) raise(QCSIM_INVALID_ARGUMENT, "engine has no state (load_basis / load_amplitudes first)");
        CK(cudaSetDevice(e->cfg.device));
        if (count) {
            const bool deferred = engine_defer_begin(e, count);
            CK(cudaEventRecord(e->ev0, e->st));
            const auto h0 = std::chrono::steady_clock::now();
            try {
                for (uint64_t k = 0; k < count; ++k) engine_gate(e, actions[k]);
                if (deferred) engine_defer_finish(e);
            } catch (...) {
                if (deferred) engine_defer_end(e, false, 0);
                throw;
            }
            const auto h1 = std::chrono::steady_clock::now();
            CK(cudaEventRecord(e->ev1, e->st));
            CK(cudaEventSynchronize(e->ev1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
            static const bool enq_timing = std::getenv("QCSIM_ENQ_TIMING") != nullptr; // debug
            if (enq_timing) {
                std::fprintf(stderr, "engine_run: %llu gates, host enqueue %.3f ms, device %.3f ms | per gate us: "
                             "prologue %.1f pass %.1f total %.1f\n",
                             (unsigned long long)count, std::chrono::duration<double, std::milli>(h1 - h0).count(), ms,
                             g_host_t[0] / count, g_host_t[2] / count, g_host_t[3] / count);
                for (double &v : g_host_t) v = 0;
            }
            e->wall += ms * 1e-3;
            if (deferred) engine_defer_end(e, true, count);
        }
        if (m) {
            std::memset(m, 0, sizeof *m);
            m->min_compression_ratio = e->calls ? e->ratio_min : 0.0;
            m->mean_compression_ratio = e->calls ? e->ratio_sum / (double)e->calls : 0.0;
            m->wall_seconds = e->wall;
            m->final_norm = tree_sum_host(e->sq_norm.data(), e->S);
            m->compress_calls = e->calls;
            m->gates = e->gates;
            m->peak_compressed_bytes = e->peak;
            m->dense_bytes = 16ull << e->n;
            m->current_compressed_bytes = e->current;
            m->index_bytes = engine_index_bytes(e);
            m->fallback_planes = e->fallback;
            m->kernel_launches = g_launches - e->launches0;
        }
    });
}

qcsim_status qcsim_engine_gate_metrics(qcsim_engine *e, qcsim_gate_metrics *rows, uint64_t capacity,
                                       uint64_t *count) {
    return guarded([&] {
        if (!e || !count) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        *count = e->rows.size();
        if (!rows) return;
        if (capacity < e->rows.size()) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        for (size_t k = 0; k < e->rows.size(); ++k) {
            const GateRow &r = e->rows[k];
            qcsim_gate_metrics &o = rows[k];
            o.min_ratio = r.calls ? r.min_ratio : 0.0;
            o.mean_ratio = r.calls ? r.ratio_sum / (double)r.calls : 0.0;
            o.seconds = r.seconds;
            o.compressed_bytes = r.bytes;
            o.index_bytes = r.index_bytes;
            o.compress_calls = r.calls;
        }
    });
}

qcsim_status qcsim_engine_info(qcsim_engine *e, qcsim_engine_info_t *info) {
    return guarded([&] {
        if (!e || !info) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        info->local_slices = e->ns;
        info->wave_slices = e->wave;
        info->waves = e->ns / e->wave;
        info->checkpoint_bits = e->log2C;
    });
}

qcsim_status qcsim_engine_trim(qcsim_engine *e) {
    return guarded([&] {
        if (!e) raise(QCSIM_INVALID_ARGUMENT, "null engine");
        CK(cudaSetDevice(e->cfg.device));
        CK(cudaStreamSynchronize(e->st));
        engine_release_scratch(e);
    });
}

qcsim_status qcsim_device_memory(uint64_t *current, uint64_t *peak, int32_t reset_peak) {
    return guarded([&] {
        if (current) *current = g_dev_cur;
        if (peak) *peak = g_dev_peak;
        if (reset_peak) g_dev_peak = g_dev_cur;
    });
}

qcsim_status qcsim_engine_gather(qcsim_engine *e, double *amps, uint64_t capacity, int32_t guard) {
    return guarded([&] {
        if (!e || !amps) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (e->n > guard)
            raise(QCSIM_CAPACITY, "dense materialization of " + std::to_string(e->n) + " qubits exceeds the " +
                                      std::to_string(guard) + "-qubit guard");
        if (capacity < 2 * e->ns * e->L) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        if (!e->loaded) raise(QCSIM_INVALID_ARGUMENT, "engine has no state");
        CK(cudaSetDevice(e->cfg.device));
        const uint64_t W = std::min<uint64_t>(e->wave, std::max<uint64_t>(1, (1ull << 30) / (16 * e->L)));
        std::vector<double> planar(W * 2 * e->L);
        for (uint64_t k0 = 0; k0 < e->ns; k0 += W) {
            const double *src = state_range(e, k0, W);
            CK(cudaMemcpyAsync(planar.data(), src, planar.size() * sizeof(double), cudaMemcpyDeviceToHost, e->st));
            CK(cudaStreamSynchronize(e->st));
            CK(cudaGetLastError());
            for (uint64_t k = 0; k < W; ++k)
                for (uint64_t i = 0; i < e->L; ++i) {
                    amps[2 * ((k0 + k) * e->L + i)] = planar[k * 2 * e->L + i];
                    amps[2 * ((k0 + k) * e->L + i) + 1] = planar[k * 2 * e->L + e->L + i];
                }
        }
    });
}

qcsim_status qcsim_engine_compare(qcsim_engine *a, qcsim_engine *b, qcsim_compare_result *out) {
    return guarded([&] {
        if (!a || !b || !out) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (a->n != b->n || a->s != b->s || a->s0 != b->s0 || a->ns != b->ns || a->cfg.device != b->cfg.device)
            raise(QCSIM_INVALID_ARGUMENT, "engines differ in qubits, slice size, slice range or device");
        if (!a->loaded || !b->loaded) raise(QCSIM_INVALID_ARGUMENT, "engine has no state");
        CK(cudaSetDevice(a->cfg.device));
        const uint64_t ntiles = (a->L + kTile - 1) / kTile;
        // bounded steps: the decoded planes of a step live in `old`
        const uint64_t W = std::min<uint64_t>(std::min(a->wave, b->wave), std::max<uint64_t>(1, (1ull << 30) / (16 * a->L)));
        DBuf<double> part;
        part.ensure(5 * W * ntiles);
        std::vector<double> h(5 * a->ns * ntiles);
        for (uint64_t k0 = 0; k0 < a->ns; k0 += W) {
            const double *pa = state_range(a, k0, W);
            CK(cudaStreamSynchronize(a->st));
            const double *pb = state_range(b, k0, W);
            CK(cudaStreamSynchronize(b->st));
            {
                PROF("state_compare", a->st);
                launch_k(state_compare, (unsigned)(W * ntiles), 256, 0, a->st, pa, pb, a->L, (int)W, part.p);
            }
            CK(cudaMemcpyAsync(h.data() + 5 * k0 * ntiles, part.p, 5 * W * ntiles * sizeof(double),
                               cudaMemcpyDeviceToHost, a->st));
            CK(cudaStreamSynchronize(a->st));
            CK(cudaGetLastError());
        }
        const uint64_t tiles = a->ns * ntiles;
        std::vector<double> col(tiles);
        double r[4];
        for (int q = 0; q < 4; ++q) {
            for (uint64_t k = 0; k < tiles; ++k) col[k] = h[5 * k + q];
            r[q] = tree_sum_host(col.data(), tiles);
        }
        double mx = 0.0;
        for (uint64_t k = 0; k < tiles; ++k) mx = std::max(mx, h[5 * k + 4]);
        out->max_abs_diff = mx;
        out->inner_re = r[0];
        out->inner_im = r[1];
        out->norm_a = r[2];
        out->norm_b = r[3];
        out->fidelity = r[0] * r[0] + r[1] * r[1];
    });
}

qcsim_status qcsim_engine_slice_norms(qcsim_engine *e, double *out, uint64_t capacity) {
    return guarded([&] {
        if (!e || !out) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (capacity < e->ns) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        std::memcpy(out, e->sq_norm.data() + e->s0, e->ns * sizeof(double));
    });
}

qcsim_status qcsim_engine_export_blocks(qcsim_engine *e, uint8_t *out, uint64_t capacity, uint64_t *len,
                                        uint64_t *offsets, uint64_t offsets_cap) {
    return guarded([&] {
        if (!e || !len) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (!e->compressed) raise(QCSIM_INVALID_ARGUMENT, "engine is not compressed");
        const uint64_t P = 2 * e->ns;
        uint64_t tot = 0;
        for (uint64_t k = 0; k < P; ++k) {
            if (offsets && k < offsets_cap) offsets[k] = tot;
            tot += e->blk_bytes_h[k];
        }
        if (offsets && P < offsets_cap) offsets[P] = tot;
        *len = tot;
        if (!out) return;
        if (capacity < tot) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        std::vector<uint64_t> off(P);
        CK(cudaMemcpyAsync(off.data(), e->blk_off[e->cur].p, P * 8, cudaMemcpyDeviceToHost, e->st));
        CK(cudaStreamSynchronize(e->st));
        // gather on the device (slots carry padding and the decode index
        // between the blocks), then one copy of exactly the blocks' bytes;
        // in steps of <= 256 MB so a large state needs no large staging buffer
        constexpr uint64_t kStep = 256ull << 20;
        uint64_t done = 0;
        for (uint64_t k0 = 0; k0 < P;) {
            uint64_t k1 = k0, bytes = 0;
            while (k1 < P && (k1 == k0 || bytes + e->blk_bytes_h[k1] <= kStep)) bytes += e->blk_bytes_h[k1++];
            const uint64_t n = k1 - k0;
            std::vector<uint64_t> meta(3 * n);
            for (uint64_t k = 0; k < n; ++k) {
                meta[k] = off[k0 + k];
                meta[n + k] = (k ? meta[n + k - 1] + e->blk_bytes_h[k0 + k - 1] : 0);
                meta[2 * n + k] = e->blk_bytes_h[k0 + k];
            }
            e->exp_meta.ensure(3 * n);
            e->exp_buf.ensure(bytes + 16);
            CK(cudaMemcpyAsync(e->exp_meta.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, e->st));
            launch_k(gather_blocks, (unsigned)n, 256, 0, e->st, (const uint8_t *)e->arena[e->cur].p,
                     (const uint64_t *)e->exp_meta.p, (int)n, e->exp_buf.p);
            CK(cudaMemcpyAsync(out + done, e->exp_buf.p, bytes, cudaMemcpyDeviceToHost, e->st));
            CK(cudaStreamSynchronize(e->st));
            done += bytes;
            k0 = k1;
        }
    });
}

qcsim_status qcsim_engine_partner_blocks_needed(qcsim_engine *e, const qcsim_action *a, uint64_t *remote,
                                                uint64_t capacity, uint64_t *count) {
    return guarded([&] {
        if (!e || !a || !count) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        std::vector<uint64_t> need;
        for (uint64_t k = 0; k < e->ns; ++k) {
            const uint64_t pj = partner_slice(*a, e->s, e->s0 + k);
            if (pj < e->s0 || pj >= e->s0 + e->ns) need.push_back(pj);
        }
        *count = need.size();
        if (remote) {
            if (capacity < need.size()) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
            std::copy(need.begin(), need.end(), remote);
        }
    });
}

qcsim_status qcsim_engine_export_slice(qcsim_engine *e, uint64_t slice, uint8_t *out, uint64_t capacity,
                                       uint64_t *len) {
    return guarded([&] {
        if (!e || !len) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (slice < e->s0 || slice >= e->s0 + e->ns) raise(QCSIM_INVALID_ARGUMENT, "slice not owned by this rank");
        if (!e->compressed) raise(QCSIM_INVALID_ARGUMENT, "engine is not compressed");
        const uint64_t k = slice - e->s0;
        const uint64_t b0 = e->blk_bytes_h[2 * k], b1 = e->blk_bytes_h[2 * k + 1];
        *len = b0 + b1;
        if (!out) return;
        if (capacity < b0 + b1) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        uint64_t off[2];
        CK(cudaMemcpyAsync(off, e->blk_off[e->cur].p + 2 * k, 16, cudaMemcpyDeviceToHost, e->st));
        CK(cudaStreamSynchronize(e->st));
        CK(cudaMemcpyAsync(out, e->arena[e->cur].p + off[0], b0, cudaMemcpyDeviceToHost, e->st));
        CK(cudaMemcpyAsync(out + b0, e->arena[e->cur].p + off[1], b1, cudaMemcpyDeviceToHost, e->st));
        CK(cudaStreamSynchronize(e->st));
    });
}

qcsim_status qcsim_engine_export_slices(qcsim_engine *e, const uint64_t *slices, uint64_t count, uint8_t *out,
                                        uint64_t capacity, uint64_t *len, uint64_t *offsets) {
    return guarded([&] {
        if (!e || !len || (count && !slices)) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (!e->compressed) raise(QCSIM_INVALID_ARGUMENT, "engine is not compressed");
        uint64_t tot = 0;
        std::vector<uint64_t> meta(3 * 2 * count);
        const uint64_t P = 2 * count;
        for (uint64_t k = 0; k < count; ++k) {
            if (slices[k] < e->s0 || slices[k] >= e->s0 + e->ns) raise(QCSIM_INVALID_ARGUMENT, "slice not owned by this rank");
            if (offsets) offsets[k] = tot;
            const uint64_t j = slices[k] - e->s0;
            for (int p = 0; p < 2; ++p) {
                meta[2 * k + p] = e->blk_off_h[2 * j + p];
                meta[P + 2 * k + p] = tot;
                meta[2 * P + 2 * k + p] = e->blk_bytes_h[2 * j + p];
                tot += e->blk_bytes_h[2 * j + p];
            }
        }
        if (offsets) offsets[count] = tot;
        *len = tot;
        if (!out || !count) return;
        if (capacity < tot) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        CK(cudaSetDevice(e->cfg.device));
        // one gather on the device, one device->host copy
        e->exp_meta.ensure(3 * P);
        e->exp_buf.ensure(tot + 16);
        CK(cudaMemcpyAsync(e->exp_meta.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, e->st));
        launch_k(gather_blocks, (unsigned)P, 256, 0, e->st, (const uint8_t *)e->arena[e->cur].p,
                 (const uint64_t *)e->exp_meta.p, (int)P, e->exp_buf.p);
        CK(cudaMemcpyAsync(out, e->exp_buf.p, tot, cudaMemcpyDeviceToHost, e->st));
        CK(cudaStreamSynchronize(e->st));
    });
}

qcsim_status qcsim_engine_export_slices_device(qcsim_engine *e, const uint64_t *slices, uint64_t count, void *out,
                                               uint64_t capacity, uint64_t *len, uint64_t *plane_offsets) {
    return guarded([&] {
        if (!e || !len || !plane_offsets || (count && !slices)) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (!e->compressed) raise(QCSIM_INVALID_ARGUMENT, "engine is not compressed");
        const uint64_t P = 2 * count;
        std::vector<uint64_t> meta(3 * P);
        uint64_t tot = 0;
        for (uint64_t k = 0; k < count; ++k) {
            if (slices[k] < e->s0 || slices[k] >= e->s0 + e->ns) raise(QCSIM_INVALID_ARGUMENT, "slice not owned by this rank");
            const uint64_t j = slices[k] - e->s0;
            for (int p = 0; p < 2; ++p) {
                plane_offsets[2 * k + p] = tot;
                meta[2 * k + p] = e->blk_off_h[2 * j + p];
                meta[P + 2 * k + p] = tot;
                meta[2 * P + 2 * k + p] = e->blk_bytes_h[2 * j + p];
                tot += e->blk_bytes_h[2 * j + p];
            }
        }
        plane_offsets[P] = tot;
        *len = tot;
        if (!out || !count) return;
        if (capacity < tot) raise(QCSIM_INVALID_ARGUMENT, "output capacity too small");
        CK(cudaSetDevice(e->cfg.device));
        e->exp_meta.ensure(3 * P);
        CK(cudaMemcpyAsync(e->exp_meta.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, e->st));
        launch_k(gather_blocks, (unsigned)P, 256, 0, e->st, (const uint8_t *)e->arena[e->cur].p,
                 (const uint64_t *)e->exp_meta.p, (int)P, (uint8_t *)out);
        CK(cudaStreamSynchronize(e->st));
    });
}

qcsim_status qcsim_engine_import_partners_device(qcsim_engine *e, const uint64_t *slices, uint64_t count,
                                                 const void *blocks, const uint64_t *plane_offsets) {
    return guarded([&] {
        if (!e || (count && (!slices || !blocks || !plane_offsets))) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        e->dev_imp = (const uint8_t *)blocks;
        for (uint64_t k = 0; k < count; ++k) {
            if (slices[k] >= e->S) raise(QCSIM_INVALID_ARGUMENT, "slice out of range");
            const uint64_t a = plane_offsets[2 * k], b = plane_offsets[2 * k + 1], c = plane_offsets[2 * k + 2];
            if (b < a || c < b) raise(QCSIM_INVALID_ARGUMENT, "plane offsets must be non-decreasing");
            e->dev_imp_at[slices[k]] = {a, b, b - a, c - b};
        }
    });
}

qcsim_status qcsim_engine_import_partner(qcsim_engine *e, uint64_t slice, const uint8_t *blocks, uint64_t len) {
    return guarded([&] {
        if (!e || !blocks) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (slice >= e->S) raise(QCSIM_INVALID_ARGUMENT, "slice out of range");
        e->imported.emplace_back(slice, std::vector<uint8_t>(blocks, blocks + len));
    });
}

qcsim_status qcsim_engine_set_global_norms(qcsim_engine *e, const double *norms, uint64_t count) {
    return guarded([&] {
        if (!e || !norms) raise(QCSIM_INVALID_ARGUMENT, "null argument");
        if (count != e->S) raise(QCSIM_INVALID_ARGUMENT, "norm table must hold every slice");
        std::memcpy(e->sq_norm.data(), norms, count * sizeof(double));
    });
}

} // extern "C"
