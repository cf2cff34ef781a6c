// enc_tiles.cuh -- tile-parallel QCB1 encoder (compress_plane,
// codec.cpp:410-533), v2.
//
// Every stage is a grid over (plane, 1024-element tile) of all planes in the
// batch; cross-tile state travels through small plane-level scans
// (plane_scans).  The only serial work is the exact FP64 chain over the
// nonzero codes (enc_chain), one plane per lane.
//
//   T1 enc_x         x = gate(old) (or raw plane), sq-norm tile partials,
//                    speculative outliers from the jump |x_i - x_{i-1}|
//   S  scan          base (last outlier) before every tile
//   T2 enc_lattice   lattice codes m^ = K_i - K_{i-1}, K relative to the
//                    segment base, event flags
//   (T2 also writes the event list for planes of <= 64 tiles, tile
//    offsets by decoupled look-back; larger planes: S scan + T3 enc_compact)
//   C  enc_chain     exact d += RN(q*m^) over events (codec.cpp:445)
//   T4 enc_verify    every decision re-evaluated with the exact prediction
//                    (codec.cpp:440-451); refuted planes -> enc_serial_x
//   (T4 also writes the tiles' run boundaries / outliers, codec.cpp:468-482)
//   S  scans         run start/end across tiles, outlier offsets
//   TB tok_count     tokens per element, histogram (codec.cpp:484-488)
//   S  scan          token offsets
//   TC tok_emit      tokens, outlier records, decode-index token state
#pragma once

#include <type_traits>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "align.cuh"

namespace qcb {

struct TileArgs {
    // per plane
    PlaneParams *params;   // flags |= kFlagFallback on refutation
    double *x;             // [plane][L] values to encode
    uint32_t *sym;         // [plane][L] speculated, then exact symbols
    uint8_t *fl;           // [plane][L] bit0 event, bit1 outlier (speculative)
    uint32_t *evlist;      // [plane][L] event element indices (bit 31: outlier)
    double *evc;           // [plane][L] event addend q*m^ (outlier: its value)
    double *dval;          // [plane][L] chain value per event ordinal
    double *evD;           // [plane][L] lattice estimate of d per event ordinal (chain_scan.cuh)
    unsigned long long *lb; // [plane][ntiles] event-offset look-back slots (epoch-tagged)
    uint32_t lb_epoch;
    unsigned long long *trace; // debug: enc_lattice phase stamps, 8 per block
    // Run-aware shortcuts for planes of many tiles (nullptr: off).
    //   zx[plane][tile]    = 1: the tile's new values are all +-0.0 (enc_x);
    //   ztriv[plane][tile] = 1: the tile's final symbols are all the zero
    //                        code, continuing a run that began before the
    //                        tile, no outliers (enc_verify) -- the tokenizer
    //                        treats it as flat without loading its symbols.
    uint8_t *zx, *ztriv;
    uint32_t *chain_prog;  // [plane] events whose chain value enc_chain has published (zeroed per
                           // pass); non-null: enc_verify runs alongside the chain, tile-major,
                           // each tile waiting for its own plane's chain front
    uint32_t *lat_bad;     // [plane] enc_gate_lattice met a code outside (-H, H) (zeroed per pass)
    int want_evD;          // the block-parallel chain reads the lattice estimates (evD);
                           // the serial warp chain does not: they are not written
    int ev_tile_local;     // event records at tile-local slots (tile * kTile + rank), no
                           // plane-wide offsets: the chain-scan kernel maps ordinals
    // run statistics of the final symbols (tokenizer input, codec.cpp:468-482),
    // written by enc_verify / enc_serial_x: first / last run start and
    // outliers per tile
    int32_t *t_firstb, *t_lastb, *t_nout;
    IndexRec *index;       // [plane][nidx]
    // per plane-tile, stride ntiles (+1 for scanned arrays)
    int32_t *t_lastout;    // last speculative outlier in the tile (-1)
    int32_t *t_base;       // scanned: last outlier strictly before the tile
    uint32_t *t_nev;       // events per tile
    uint32_t *t_evoff;     // scanned (ntiles + 1)
    double *tilesum;       // [unit][ntiles]
    uint64_t L;
    int ntiles;
    int tile_sh;           // log2(ntiles) when ntiles is a power of two, else -1 (split_block)
    int log2C;
    int qb;
    int predictor;
    // per-pass bookkeeping reset by enc_x (tile 0 of every plane)
    uint32_t *symrange;              // [plane][2]
    uint32_t *hspecial;              // [plane][2]
    unsigned long long *gamma;       // [plane]
};

// (plane or unit, tile) of a block: a shift when the tile count is a power of
// two (engine planes), else the division.
__device__ __forceinline__ void split_block(uint32_t b, int ntiles, int sh, int &pl, int &t) {
    if (sh >= 0) {
        pl = (int)(b >> sh);
        t = (int)(b & (uint32_t)(ntiles - 1));
    } else {
        pl = (int)(b / (uint32_t)ntiles);
        t = (int)(b % (uint32_t)ntiles);
    }
}

__device__ __forceinline__ bool is_negzero(double v) { return bits_of(v) == 0x8000000000000000ull; }

// Plane parameters as ONE consistent snapshot per block.  Other blocks of
// the same kernel may set kFlagFallback concurrently (atomicOr); a per-thread
// read could let some threads of a block return early while the rest enter
// a barrier or a block-wide scan.  All threads must call this.
__device__ __forceinline__ PlaneParams block_params(const PlaneParams *params, int pl) {
    // bounds are fixed while the tile grids run (every lane loads the same
    // words: one transaction per warp); only the fallback flag can change
    // under the block, so the block agrees on it with one voting barrier
    PlaneParams pp = params[pl];
    const int fb = __syncthreads_or((int)(__ldcg(&params[pl].flags) & kFlagFallback));
    pp.flags = (pp.flags & ~(uint32_t)kFlagFallback) | (fb ? (uint32_t)kFlagFallback : 0u);
    return pp;
}

// Per-plane hand-off between grids that overlap (programmatic launch without
// a grid-wide wait): every block of plane p of the producer arrives in
// cnt[p]; the last one resets it and raises done[p] to the pass's epoch.  A
// consumer block of plane p waits for done[p] == epoch and reads the
// producer's data from L2.
struct PlaneFlow {
    uint32_t *cnt;
    uint32_t *done;
    uint32_t epoch;
};
__device__ __forceinline__ void flow_arrive(const PlaneFlow &F, int pl, uint32_t blocks) { // thread 0, after a barrier
    __threadfence();
    const uint32_t old = atomicAdd(F.cnt + pl, 1u);
    if (old + 1 == blocks) {
        F.cnt[pl] = 0u;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(F.done + pl), "r"(F.epoch) : "memory");
    }
}
__device__ __forceinline__ void flow_wait(const uint32_t *done, int pl, uint32_t epoch) { // one thread
    uint32_t v;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + pl) : "memory");
        if (v != epoch) __nanosleep(32);
    } while (v != epoch);
}

// A thread's kPerThread (= 4) consecutive elements of a tile in one or two
// vector loads (tile starts are 1024-element aligned); scalar at a ragged end.
static_assert(kPerThread == 4, "vector tile loads assume 4 elements per thread");
__device__ __forceinline__ void load4(const uint8_t *p, int k0, int tl, uint32_t *v) {
    if (k0 + 4 <= tl) {
        const uint32_t w = *reinterpret_cast<const uint32_t *>(p + k0);
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (w >> (8 * e)) & 0xFF;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = k0 + e < tl ? p[k0 + e] : 0u;
    }
}
__device__ __forceinline__ void load4(const uint32_t *p, int k0, int tl, uint32_t *v) {
    if (k0 + 4 <= tl) {
        const uint4 w = *reinterpret_cast<const uint4 *>(p + k0);
        v[0] = w.x;
        v[1] = w.y;
        v[2] = w.z;
        v[3] = w.w;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = k0 + e < tl ? p[k0 + e] : 0u;
    }
}
__device__ __forceinline__ void load4(const double *p, int k0, int tl, double *v) {
    if (k0 + 4 <= tl) {
        const double2 a = *reinterpret_cast<const double2 *>(p + k0);
        const double2 b = *reinterpret_cast<const double2 *>(p + k0 + 2);
        v[0] = a.x;
        v[1] = a.y;
        v[2] = b.x;
        v[3] = b.y;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = k0 + e < tl ? p[k0 + e] : 0.0;
    }
}

// Planes with few tiles get their cross-tile carries inline: the consuming
// block reduces the per-tile values before (or after) its own tile instead
// of waiting for a separate plane_scan launch.
constexpr int kInlineTiles = 64;
enum ScanKind { kScanMaxExcl = 0, kScanSumExcl = 1, kScanMinExclRev = 2 };

// Exclusive carry of tile t over the per-tile array `a` (stride ntiles):
// max over [0,t) (init -1), sum over [0,t), or min over (t,ntiles) (init
// INT_MAX).  All threads call it; result broadcast through shared memory.
__device__ int32_t tile_carry(const int32_t *a, int t, int ntiles, int kind) {
    __shared__ int32_t s_res;
    if (threadIdx.x < 32) {
        int32_t v = kind == kScanMaxExcl ? -1 : (kind == kScanSumExcl ? 0 : 0x7FFFFFFF);
        const int lo = kind == kScanMinExclRev ? t + 1 : 0;
        const int hi = kind == kScanMinExclRev ? ntiles : t;
        for (int k = lo + (int)threadIdx.x; k < hi; k += 32) {
            const int32_t x = __ldcg(a + k);
            v = kind == kScanMaxExcl ? max(v, x) : (kind == kScanSumExcl ? v + x : min(v, x));
        }
        for (int off = 16; off >= 1; off >>= 1) {
            const int32_t o = __shfl_xor_sync(0xffffffffu, v, off);
            v = kind == kScanMaxExcl ? max(v, o) : (kind == kScanSumExcl ? v + o : min(v, o));
        }
        if (threadIdx.x == 0) s_res = v;
    }
    __syncthreads();
    const int32_t r = s_res;
    __syncthreads();
    return r;
}

// Two exclusive carries of tile t in one warp pass and one barrier pair.
__device__ __forceinline__ int32_t carry_reduce(int kind, int32_t v, int32_t x) {
    return kind == kScanMaxExcl ? max(v, x) : (kind == kScanSumExcl ? v + x : min(v, x));
}
__device__ __forceinline__ int32_t carry_init(int kind) {
    return kind == kScanMaxExcl ? -1 : (kind == kScanSumExcl ? 0 : 0x7FFFFFFF);
}
__device__ void tile_carry2(const int32_t *a1, int k1, const int32_t *a2, int k2, int t, int ntiles, int32_t &r1,
                            int32_t &r2) {
    __shared__ int32_t s_res2[2];
    if (threadIdx.x < 32) {
        int32_t v1 = carry_init(k1), v2 = carry_init(k2);
        const int lo1 = k1 == kScanMinExclRev ? t + 1 : 0, hi1 = k1 == kScanMinExclRev ? ntiles : t;
        const int lo2 = k2 == kScanMinExclRev ? t + 1 : 0, hi2 = k2 == kScanMinExclRev ? ntiles : t;
        for (int k = (int)threadIdx.x; k < ntiles; k += 32) {
            if (k >= lo1 && k < hi1) v1 = carry_reduce(k1, v1, __ldcg(a1 + k));
            if (k >= lo2 && k < hi2) v2 = carry_reduce(k2, v2, __ldcg(a2 + k));
        }
        for (int off = 16; off >= 1; off >>= 1) {
            v1 = carry_reduce(k1, v1, __shfl_xor_sync(0xffffffffu, v1, off));
            v2 = carry_reduce(k2, v2, __shfl_xor_sync(0xffffffffu, v2, off));
        }
        if (threadIdx.x == 0) {
            s_res2[0] = v1;
            s_res2[1] = v2;
        }
    }
    __syncthreads();
    r1 = s_res2[0];
    r2 = s_res2[1];
    __syncthreads();
}
// N exclusive carries of tile t in one warp pass and one barrier pair.
template <int N>
__device__ void tile_carryN(const int32_t *const *a, const int *kinds, int t, int ntiles, int32_t *r) {
    __shared__ int32_t s_resn[N];
    if (threadIdx.x < 32) {
        int32_t v[N];
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = carry_init(kinds[q]);
        for (int k = (int)threadIdx.x; k < ntiles; k += 32) {
#pragma unroll
            for (int q = 0; q < N; ++q) {
                const bool rev = kinds[q] == kScanMinExclRev;
                if (rev ? k > t : k < t) v[q] = carry_reduce(kinds[q], v[q], __ldcg(a[q] + k));
            }
        }
#pragma unroll
        for (int q = 0; q < N; ++q)
            for (int off = 16; off >= 1; off >>= 1) v[q] = carry_reduce(kinds[q], v[q], __shfl_xor_sync(0xffffffffu, v[q], off));
        if (threadIdx.x == 0)
#pragma unroll
            for (int q = 0; q < N; ++q) s_resn[q] = v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < N; ++q) r[q] = s_resn[q];
    __syncthreads();
}

// Sum over tiles [0, t) and over all tiles of one per-tile array, one pass.
__device__ void tile_excl_total(const int32_t *a, int t, int ntiles, int32_t &excl, int32_t &total) {
    __shared__ int32_t s_et[2];
    if (threadIdx.x < 32) {
        int32_t v1 = 0, v2 = 0;
        for (int k = (int)threadIdx.x; k < ntiles; k += 32) {
            const int32_t x = __ldcg(a + k);
            v2 += x;
            if (k < t) v1 += x;
        }
        for (int off = 16; off >= 1; off >>= 1) {
            v1 += __shfl_xor_sync(0xffffffffu, v1, off);
            v2 += __shfl_xor_sync(0xffffffffu, v2, off);
        }
        if (threadIdx.x == 0) {
            s_et[0] = v1;
            s_et[1] = v2;
        }
    }
    __syncthreads();
    excl = s_et[0];
    total = s_et[1];
    __syncthreads();
}

// carry_of for two arrays of the same plane / tile at once
__device__ __forceinline__ void carry_of2(const int32_t *sc1, int st1, const int32_t *raw1, int k1, const int32_t *sc2,
                                          int st2, const int32_t *raw2, int k2, int pl, int t, int ntiles,
                                          int32_t &r1, int32_t &r2) {
    if (ntiles > kInlineTiles) {
        r1 = sc1[(uint64_t)pl * st1 + t];
        r2 = sc2[(uint64_t)pl * st2 + t];
        return;
    }
    tile_carry2(raw1 + (uint64_t)pl * ntiles, k1, raw2 + (uint64_t)pl * ntiles, k2, t, ntiles, r1, r2);
}

// The scanned value for tile t: from the plane_scan output when the plane
// has many tiles, else computed inline from the raw per-tile array.
__device__ __forceinline__ int32_t carry_of(const int32_t *scanned, int scanned_stride, const int32_t *raw, int pl,
                                            int t, int ntiles, int kind) {
    if (ntiles > kInlineTiles) return scanned[(uint64_t)pl * scanned_stride + t];
    return tile_carry(raw + (uint64_t)pl * ntiles, t, ntiles, kind);
}

// ------------------------------------------------------------------ T1
// kVec: element pairs through Src::load2 (16-byte loads) instead of load().
template <int NP, class Src, bool kVec>
__global__ void __launch_bounds__(kEncThreads, 5) enc_x(TileArgs A, Src src, int units) {
    pdl_begin();
    int unit, t;
    split_block(blockIdx.x, A.ntiles, A.tile_sh, unit, t);
    if (unit >= units) return;
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    if (t == 0 && tid < NP) {
        // per-pass reset of the plane's flags and histogram bookkeeping
        const int pl = unit * NP + tid;
        const PlaneParams pp = A.params[pl];
        A.params[pl].flags = (A.predictor == 1 && pp.eb != 0.0) ? kFlagFallback : 0u;
        A.symrange[2 * pl] = 0xFFFFFFFFu;
        A.symrange[2 * pl + 1] = 0;
        A.hspecial[2 * pl] = 0;
        A.hspecial[2 * pl + 1] = 0;
        A.gamma[pl] = 0;
    }
    __shared__ double xs[NP][kTile + 1];
    __shared__ double red[kEncThreads];
    using RedI = cub::BlockReduce<int, kEncThreads>;
    __shared__ typename RedI::TempStorage red_tmp;
    // Element pairs, striped over the block (coalesced; 16-byte loads where
    // the source has them); element t0-1 as xs[.][0].  Blocks none of whose
    // source tiles carries a decoder zero flag read without looking at flags.
    static_assert(kTile % 2 == 0, "pairs");
    __shared__ int s_flagged;
    if (tid == 0) s_flagged = src.flagged_sources(unit, (uint32_t)t) ? 1 : 0;
    __syncthreads();
    const bool flagged = s_flagged != 0;
    int nonzero[NP];
    for (int p = 0; p < NP; ++p) nonzero[p] = 0;
    auto load_tile = [&](auto kF) {
        constexpr bool kFlags = decltype(kF)::value;
#pragma unroll 2
        for (int k2 = tid; k2 < kTile / 2; k2 += kEncThreads) {
            double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0};
            const int k = 2 * k2;
            if (kVec && k + 1 < tl) src.template load2f<kFlags>(unit, t0 + k, a, b);
            else {
                if (k < tl) src.template loadf<kFlags>(unit, t0 + k, a);
                if (k + 1 < tl) src.template loadf<kFlags>(unit, t0 + k + 1, b);
            }
            for (int p = 0; p < NP; ++p) {
                xs[p][k + 1] = a[p];
                xs[p][k + 2] = b[p];
                nonzero[p] |= (a[p] != 0.0) | (b[p] != 0.0); // (NaN counts as nonzero)
            }
            // the new values go out as they arrive (one 16-byte store per plane)
            for (int p = 0; p < NP; ++p) {
                double *xrow = A.x + ((uint64_t)unit * NP + p) * L + t0 + k;
                if (k + 1 < tl && (L & 1) == 0) *reinterpret_cast<double2 *>(xrow) = make_double2(a[p], b[p]);
                else {
                    if (k < tl) xrow[0] = a[p];
                    if (k + 1 < tl) xrow[1] = b[p];
                }
            }
        }
        if (tid == 0) {
            double v[2] = {0.0, 0.0};
            if (t0 > 0) src.template loadf<kFlags>(unit, t0 - 1, v);
            for (int p = 0; p < NP; ++p) xs[p][0] = v[p];
        }
    };
    if (flagged) load_tile(std::true_type{});
    else load_tile(std::false_type{});
    if (A.zx) { // all-zero tiles are flagged for the later grids
        for (int p = 0; p < NP; ++p) {
            const int any = __syncthreads_or(nonzero[p]);
            if (tid == 0) A.zx[((uint64_t)unit * NP + p) * A.ntiles + t] = any ? 0 : 1;
        }
    } else {
        __syncthreads();
    }
    if (Src::kNorms) {
        double acc[kPerThread];
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e + 1;
            const double a = dmul(xs[0][k], xs[0][k]);
            const double b = dmul(xs[NP - 1][k], xs[NP - 1][k]);
            acc[e] = dadd(a, b);
        }
        // the tile's adjacent-pair tree: 5 levels inside each warp by
        // shuffles (left operand = lower index, as the reference tree), then
        // the 8 warp sums
        double v = dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3]));
        const int lane = tid & 31;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double o = __shfl_down_sync(0xffffffffu, v, off);
            if ((lane & (2 * off - 1)) == 0) v = dadd(v, o);
        }
        if (lane == 0) red[tid >> 5] = v;
        __syncthreads();
        if (tid == 0) {
            static_assert(kEncThreads == 256, "8 warp sums");
            const double s01 = dadd(red[0], red[1]), s23 = dadd(red[2], red[3]);
            const double s45 = dadd(red[4], red[5]), s67 = dadd(red[6], red[7]);
            A.tilesum[(uint64_t)unit * A.ntiles + t] = dadd(dadd(s01, s23), dadd(s45, s67));
        }
    }
    // speculative outliers
    const double hh = (double)(1ll << (A.qb - 1));
    for (int p = 0; p < NP; ++p) {
        const uint64_t pl = (uint64_t)unit * NP + p;
        const PlaneParams pp = A.params[pl];
        int last = -1;
        uint8_t *flrow = A.fl + pl * L;
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            bool out = false;
            if (k < tl && pp.eb != 0.0) {
                const double xp = xs[p][k]; // x[i-1], 0.0 at i = 0
                const double rr = dmul(dsub(xs[p][k + 1], xp), pp.inv_q);
                out = !(fabs(rr) < hh - 0.5);
            }
            if (k < tl) flrow[t0 + k] = out ? 2 : 0;
            if (out) last = k;
        }
        const int tl_last = RedI(red_tmp).Reduce(last, cub::Max());
        if (tid == 0) A.t_lastout[pl * A.ntiles + t] = tl_last >= 0 ? (int32_t)(t0 + tl_last) : -1;
        __syncthreads();
    }
}

// ----------------------------------------------------------- plane scans
// One block per plane over `ntiles` entries (ntiles <= 4096).

template <int ITEMS>
__global__ void __launch_bounds__(256) plane_scan(const int32_t *in, int32_t *out, int ntiles, int planes, int kind,
                                                  int in_stride, int out_stride) {
    pdl_begin();
    const int pl = blockIdx.x;
    if (pl >= planes) return;
    using Scan = cub::BlockScan<int32_t, 256>;
    __shared__ typename Scan::TempStorage tmp;
    const int32_t *a = in + (uint64_t)pl * in_stride;
    int32_t *o = out + (uint64_t)pl * out_stride;
    int32_t v[ITEMS], r[ITEMS];
    const int tid = threadIdx.x;
    for (int e = 0; e < ITEMS; ++e) {
        const int k = tid * ITEMS + e;
        const int src = kind == kScanMinExclRev ? ntiles - 1 - k : k;
        if (k < ntiles) v[e] = a[src];
        else v[e] = kind == kScanMaxExcl ? -1 : (kind == kScanSumExcl ? 0 : 0x7FFFFFFF);
    }
    int32_t total;
    if (kind == kScanMaxExcl) Scan(tmp).ExclusiveScan(v, r, -1, cub::Max(), total);
    else if (kind == kScanSumExcl) Scan(tmp).ExclusiveSum(v, r, total);
    else Scan(tmp).ExclusiveScan(v, r, 0x7FFFFFFF, cub::Min(), total);
    for (int e = 0; e < ITEMS; ++e) {
        const int k = tid * ITEMS + e;
        if (k < ntiles) o[kind == kScanMinExclRev ? ntiles - 1 - k : k] = r[e];
    }
    if (tid == 0 && kind == kScanSumExcl) o[ntiles] = total;
}

// Decoupled look-back over the tiles of one plane (one thread per block):
// publish this tile's count, add predecessors' counts until one with an
// inclusive prefix, publish the inclusive prefix.  Slots carry the pass
// epoch in their tag, so they never need clearing; blocks of a plane are
// dispatched in tile order (block = plane * ntiles + tile).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_tag(uint32_t epoch, uint32_t status) {
    return (unsigned long long)((epoch << 2) | status) << 32;
}
__device__ void lookback_publish_aggregate(unsigned long long *slots, uint32_t epoch, int t, uint32_t local) {
    st_release_u64(&slots[t], lb_tag(epoch, 1) | local);
}
// Warp-wide: lanes read 32 predecessors at once; the window slides back
// until it meets an inclusive prefix (or tile 0).  Call with a full warp;
// the result is valid in every lane.
__device__ uint32_t lookback_exclusive(unsigned long long *slots, uint32_t epoch, int t, uint32_t local) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) st_release_u64(&slots[t], lb_tag(epoch, t == 0 ? 2 : 1) | local);
    uint32_t prefix = 0;
    int hi = t - 1; // window [hi - 31, hi]
    while (hi >= 0) {
        const int k = hi - lane;
        unsigned long long w = 0;
        uint32_t st = 2; // below tile 0: acts as an inclusive zero
        if (k >= 0) {
            do {
                w = ld_acquire_u64(&slots[k]);
                st = ((uint32_t)(w >> 32) >> 2) == epoch ? ((uint32_t)(w >> 32) & 3) : 0;
                if (st == 0) __nanosleep(32);
            } while (st == 0);
        }
        // the nearest inclusive prefix in the window ends the walk
        const unsigned incl = __ballot_sync(0xffffffffu, st == 2);
        const int stop = incl ? __ffs(incl) - 1 : 32; // lanes [0, stop] contribute
        uint32_t v = (lane <= stop && k >= 0) ? (uint32_t)w : 0u;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        prefix += v;
        if (incl) break;
        hi -= 32;
    }
    if (lane == 0 && t > 0) st_release_u64(&slots[t], lb_tag(epoch, 2) | (prefix + local));
    return prefix;
}

// ------------------------------------------------------------------ T2
// Lattice codes, flags and the plane's event list (the compaction is fused:
// the tile's event offset comes from the look-back above).
__device__ __forceinline__ void lattice_tile(const TileArgs &A, int pl, int t) {
    auto stamp = [&](int k) {
        if (A.trace && threadIdx.x == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            A.trace[8ull * blockIdx.x + k] = tt;
        }
    };
    stamp(0);
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    using ScanI = cub::BlockScan<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage scan_tmp;
    __shared__ long long kb[kEncThreads];
    const PlaneParams pp = block_params(A.params, pl);
    const long long half = 1ll << (A.qb - 1);
    const double *x = A.x + (uint64_t)pl * L;
    uint8_t *fl = A.fl + (uint64_t)pl * L;
    uint32_t *sym = A.sym + (uint64_t)pl * L;
    unsigned long long *lbs = A.lb + (uint64_t)pl * A.ntiles;
    if (pp.flags & kFlagFallback) {
        if (tid == 0) {
            A.t_nev[(uint64_t)pl * A.ntiles + t] = 0;
            if (A.ntiles <= kInlineTiles) lookback_publish_aggregate(lbs, A.lb_epoch, t, 0);
        }
        return;
    }
    if (pp.eb == 0.0) {
        // lossless / zero range: d == x, symbols final, no events
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            if (k >= tl) continue;
            const uint64_t i = t0 + k;
            const double x1 = i > 0 ? x[i - 1] : 0.0;
            double pred;
            if (A.predictor == 0) pred = x1;
            else pred = i == 0 ? 0.0 : (i == 1 ? x1 : predict_linear(x1, x[i - 2]));
            sym[i] = bits_of(x[i]) == bits_of(pred) ? (uint32_t)half : 0u;
            fl[i] = 0;
        }
        if (tid == 0) {
            A.t_nev[(uint64_t)pl * A.ntiles + t] = 0;
            if (A.ntiles <= kInlineTiles) lookback_publish_aggregate(lbs, A.lb_epoch, t, 0);
        }
        return;
    }
    if (A.zx && A.ntiles > kInlineTiles && tl == kTile && A.zx[(uint64_t)pl * A.ntiles + t]) {
        // Every value of the tile is +-0.0 (enc_x), so K is the same for all
        // its elements and only the first one can carry a code: when it does
        // not (and is no speculative outlier), the tile is the zero code
        // throughout -- no value loads, no scans.  Same operations as the
        // general path below for these inputs (block-uniform decision).
        bool trivial = !(fl[t0] & 2);
        if (trivial) {
            const int32_t tb = A.t_base[(uint64_t)pl * A.ntiles + t]; // last outlier before the tile or -1
            const double base = tb >= 0 ? x[tb] : 0.0;
            const long long Kz = llround_exact(dmul(dsub(0.0, base), pp.inv_q));
            long long kprev = 0;
            bool prev_out = false;
            double xp = 0.0;
            if (t0 > 0) {
                xp = x[t0 - 1];
                prev_out = (fl[t0 - 1] & 2) != 0;
                if (!prev_out) kprev = llround_exact(dmul(dsub(xp, base), pp.inv_q));
            }
            trivial = Kz - kprev == 0 && !(prev_out && is_negzero(xp));
        }
        if (trivial) {
            const uint32_t hs = (uint32_t)half;
            *reinterpret_cast<uint4 *>(sym + t0 + tid * kPerThread) = make_uint4(hs, hs, hs, hs);
            // (the flags enc_x wrote are already 0: no speculative outliers)
            if (tid == 0) A.t_nev[(uint64_t)pl * A.ntiles + t] = 0;
            return;
        }
    }
    // speculative outliers of this tile and the element before it (enc_x
    // recorded whether the tile has any: most have none, and then neither
    // the flags nor a scan are needed -- every element's segment base comes
    // from the carry)
    const bool tile_out = A.t_lastout[(uint64_t)pl * A.ntiles + t] >= 0; // block-uniform
    int opos[kPerThread];
    double xv[kPerThread];
    if (tile_out) {
        uint32_t fv[kPerThread];
        load4(fl + t0, tid * kPerThread, tl, fv);
        for (int e = 0; e < kPerThread; ++e) opos[e] = (tid * kPerThread + e < tl && (fv[e] & 2)) ? tid * kPerThread + e : -1;
    } else {
        for (int e = 0; e < kPerThread; ++e) opos[e] = -1;
    }
    load4(x + t0, tid * kPerThread, tl, xv);
    int lo[kPerThread];
    if (tile_out) {
        ScanI(scan_tmp).ExclusiveScan(opos, lo, -1, cub::Max());
    } else {
        for (int e = 0; e < kPerThread; ++e) lo[e] = -1;
    }
    stamp(1);
    const int32_t tbase = carry_of(A.t_base, A.ntiles, A.t_lastout, pl, t, A.ntiles, kScanMaxExcl); // position or -1
    stamp(2);
    long long K[kPerThread];
    double dh[kPerThread]; // lattice estimate of the chain value (chain_scan.cuh)
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        if (opos[e] >= 0) {
            K[e] = 0;
            dh[e] = xv[e];
        } else {
            double base;
            if (lo[e] >= 0) base = x[t0 + lo[e]];
            else base = tbase >= 0 ? x[tbase] : 0.0;
            K[e] = k < tl ? llround_exact(dmul(dsub(xv[e], base), pp.inv_q)) : 0;
            dh[e] = dadd(base, dmul(pp.q, (double)K[e]));
        }
    }
    const bool fused = A.ntiles <= kInlineTiles; // else enc_compact writes the events
    kb[tid] = K[kPerThread - 1];
    // K and outlier status of element t0-1 (for the first element)
    long long kprev0 = 0;
    bool prevout0 = false;
    double xprev0 = 0.0;
    if (tid == 0 && t0 > 0) {
        const uint64_t i = t0 - 1;
        xprev0 = x[i];
        prevout0 = (fl[i] & 2) != 0;
        if (!prevout0) {
            const double base = tbase >= 0 ? x[tbase] : 0.0;
            kprev0 = llround_exact(dmul(dsub(xprev0, base), pp.inv_q));
        }
    }
    __syncthreads();
    int evflag[kPerThread];
    uint32_t esym[kPerThread];
    uint32_t fword = 0; // this thread's 4 flag bytes (one 32-bit store)
    int bad = 0;
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        evflag[e] = 0;
        esym[e] = 0;
        if (k >= tl) continue;
        long long kprev;
        bool prev_out;
        double xp;
        if (e > 0) { kprev = K[e - 1]; prev_out = opos[e - 1] >= 0; xp = xv[e - 1]; }
        else if (tid > 0) { kprev = kb[tid - 1]; prev_out = lo[0] == k - 1; xp = x[t0 + k - 1]; }
        else { kprev = kprev0; prev_out = prevout0; xp = xprev0; }
        if (prev_out) kprev = 0;
        uint8_t f;
        uint32_t sy;
        if (opos[e] >= 0) {
            f = 3;
            sy = kOutlierSym;
        } else {
            const long long m = K[e] - kprev;
            if (m <= -half || m >= half) bad = 1;
            sy = (uint32_t)(m + half);
            f = (m != 0 || (prev_out && is_negzero(xp))) ? 1 : 0;
        }
        fword |= (uint32_t)f << (8 * e);
        esym[e] = sy;
        evflag[e] = f & 1;
    }
    {
        const int k0 = tid * kPerThread;
        if (k0 + kPerThread <= tl) { // flags and symbols: one 4-byte and one 16-byte store
            *reinterpret_cast<uint32_t *>(fl + t0 + k0) = fword;
            *reinterpret_cast<uint4 *>(sym + t0 + k0) = make_uint4(esym[0], esym[1], esym[2], esym[3]);
        } else {
            for (int e = 0; e < kPerThread && k0 + e < tl; ++e) {
                fl[t0 + k0 + e] = (uint8_t)(fword >> (8 * e));
                sym[t0 + k0 + e] = esym[e];
            }
        }
    }
    if (bad) atomicOr(&A.params[pl].flags, kFlagFallback);
    stamp(3);
    // event list: tile offset by look-back, in-tile positions by a block scan
    int epos[kPerThread], tot;
    __syncthreads();
    if (!fused) { // the event count only (enc_compact places the records)
        __shared__ int s_tot;
        int mine = 0;
        for (int e = 0; e < kPerThread; ++e) mine += evflag[e];
        mine = __reduce_add_sync(0xffffffffu, mine);
        if (tid == 0) s_tot = 0;
        __syncthreads();
        if ((tid & 31) == 0 && mine) atomicAdd(&s_tot, mine);
        __syncthreads();
        tot = s_tot;
    } else {
        ScanI(scan_tmp).ExclusiveSum(evflag, epos, tot);
    }
    if (!fused) {
        // lattice estimates of the events only (enc_compact reads them there;
        // dval is scratch until the chain overwrites it)
        if (A.want_evD) {
            double *dhat = A.dval + (uint64_t)pl * L;
            for (int e = 0; e < kPerThread; ++e)
                if (evflag[e]) dhat[t0 + tid * kPerThread + e] = dh[e];
        }
        if (tid == 0) A.t_nev[(uint64_t)pl * A.ntiles + t] = (uint32_t)tot;
        return;
    }
    __shared__ uint32_t s_evbase;
    if (A.ev_tile_local) { // no cross-tile wait: records at the tile's own slots
        if (tid == 0) A.t_nev[(uint64_t)pl * A.ntiles + t] = (uint32_t)tot;
        if (tid == 0) s_evbase = (uint32_t)t0;
    } else if (tid < 32) {
        const uint32_t b = lookback_exclusive(lbs, A.lb_epoch, t, (uint32_t)tot);
        if (tid == 0) {
            A.t_nev[(uint64_t)pl * A.ntiles + t] = (uint32_t)tot;
            s_evbase = b;
        }
    }
    __syncthreads();
    const uint32_t evb = s_evbase;
    stamp(4);
    uint32_t *ev = A.evlist + (uint64_t)pl * L;
    double *evc = A.evc + (uint64_t)pl * L;
    double *evD = A.evD + (uint64_t)pl * L;
    for (int e = 0; e < kPerThread; ++e) {
        if (!evflag[e]) continue;
        const uint32_t i = (uint32_t)(t0 + tid * kPerThread + e);
        const bool out = opos[e] >= 0;
        const uint32_t o = evb + (uint32_t)epos[e];
        // the record the chain consumes: element index (bit 31 = outlier),
        // addend q*m^ (or the outlier value), lattice estimate of d
        ev[o] = i | (out ? 0x80000000u : 0u);
        evc[o] = out ? xv[e] : dmul(pp.q, (double)((long long)esym[e] - half));
        if (A.want_evD) evD[o] = dh[e];
    }
    stamp(5);
}
// redo == nullptr: one block per (plane, tile).  Otherwise the planes listed
// in redo[1 .. redo[0]] only (enc_gate_lattice's planes with a speculative
// outlier), on a grid of rmax * ntiles blocks.
__global__ void __launch_bounds__(kEncThreads, 5) enc_lattice(TileArgs A, int planes, const uint32_t *redo, int rmax) {
    pdl_begin();
    int r, t;
    split_block(blockIdx.x, A.ntiles, A.tile_sh, r, t);
    if (!redo) {
        if (r < planes) lattice_tile(A, r, t);
        return;
    }
    const uint32_t cnt = redo[0];
    for (; (uint32_t)r < cnt; r += rmax) {
        lattice_tile(A, (int)redo[1 + r], t);
        __syncthreads();
    }
}

// Planes with a speculative outlier anywhere (t_lastout / its exclusive max
// scan t_base), listed for enc_lattice's redo grid.  One block.
__global__ void __launch_bounds__(256) lattice_redo_list(TileArgs A, int planes, uint32_t *redo) {
    pdl_begin();
    __shared__ uint32_t s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int pl = threadIdx.x; pl < planes; pl += blockDim.x) {
        const uint64_t last = (uint64_t)pl * A.ntiles + (A.ntiles - 1);
        if (A.t_base[last] >= 0 || A.t_lastout[last] >= 0) redo[1 + atomicAdd(&s_cnt, 1u)] = (uint32_t)pl;
        else if (A.lat_bad[pl]) atomicOr(&A.params[pl].flags, kFlagFallback); // serial re-encode
    }
    __syncthreads();
    if (threadIdx.x == 0) redo[0] = s_cnt;
}

// T1+T2 for planes of many whole tiles with a lossy absolute bound and the
// previous-value predictor: new = gate(scale * old) AND its lattice codes in
// one grid, each thread keeping its 4 consecutive elements of every plane in
// registers (no shared-memory staging; 16-byte loads and stores).  The
// segment base is taken as "no speculative outlier before this element"
// (base 0.0) -- true for every element of a plane without speculative
// outliers, which is almost every plane; the few planes that have one
// (t_lastout) are listed by lattice_redo_list and redone by enc_lattice from
// the x and flags written here.  Same operations on the same values as
// enc_x + enc_lattice for the planes it finishes.
template <int NP, class Src>
__global__ void __launch_bounds__(kEncThreads, 4) enc_gate_lattice(TileArgs A, Src src, int units) {
    pdl_begin();
    int unit, t;
    split_block(blockIdx.x, A.ntiles, A.tile_sh, unit, t);
    if (unit >= units) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile; // (whole tiles: L is a multiple of kTile)
    if (t == 0 && tid < NP) {
        // per-pass reset of the plane's flags and histogram bookkeeping
        const int pl = unit * NP + tid;
        A.params[pl].flags = 0u;
        A.symrange[2 * pl] = 0xFFFFFFFFu;
        A.symrange[2 * pl + 1] = 0;
        A.hspecial[2 * pl] = 0;
        A.hspecial[2 * pl + 1] = 0;
        A.gamma[pl] = 0;
    }
    __shared__ int s_flagged;
    __shared__ double s_last[NP][kEncThreads / 32]; // each warp's last element
    __shared__ double s_halo[NP];                   // element t0 - 1
    __shared__ double red[kEncThreads / 32];
    __shared__ int s_nev[NP], s_lastout[NP];
    if (tid == 0) s_flagged = src.flagged_sources(unit, (uint32_t)t) ? 1 : 0;
    if (tid < NP) {
        s_nev[tid] = 0;
        s_lastout[tid] = -1;
    }
    __syncthreads();
    const bool flagged = s_flagged != 0;
    const int k0 = tid * kPerThread;
    double xv[NP][kPerThread];
    auto load_mine = [&](auto kF) {
        constexpr bool kFlags = decltype(kF)::value;
#pragma unroll
        for (int h = 0; h < kPerThread; h += 2) {
            double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0};
            src.template load2f<kFlags>(unit, t0 + k0 + h, a, b);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                xv[p][h] = a[p];
                xv[p][h + 1] = b[p];
            }
        }
        if (tid == kEncThreads - 1) { // (the last thread: its own loads are issued first)
            double v[2] = {0.0, 0.0};
            if (t0 > 0) src.template loadf<kFlags>(unit, t0 - 1, v);
#pragma unroll
            for (int p = 0; p < NP; ++p) s_halo[p] = v[p];
        }
    };
    if (flagged) load_mine(std::true_type{});
    else load_mine(std::false_type{});
    int nonzero[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        double *xrow = A.x + ((uint64_t)unit * NP + p) * L + t0 + k0;
        *reinterpret_cast<double2 *>(xrow) = make_double2(xv[p][0], xv[p][1]);
        *reinterpret_cast<double2 *>(xrow + 2) = make_double2(xv[p][2], xv[p][3]);
        nonzero[p] = (xv[p][0] != 0.0) | (xv[p][1] != 0.0) | (xv[p][2] != 0.0) | (xv[p][3] != 0.0);
        if (lane == 31) s_last[p][wid] = xv[p][kPerThread - 1];
    }
    double nv = 0.0;
    if (Src::kNorms) {
        double acc[kPerThread];
#pragma unroll
        for (int e = 0; e < kPerThread; ++e)
            acc[e] = dadd(dmul(xv[0][e], xv[0][e]), dmul(xv[NP - 1][e], xv[NP - 1][e]));
        // the tile's adjacent-pair tree (as enc_x)
        nv = dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3]));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double o = __shfl_down_sync(0xffffffffu, nv, off);
            if ((lane & (2 * off - 1)) == 0) nv = dadd(nv, o);
        }
        if (lane == 0) red[wid] = nv;
    }
    // all-zero tiles are flagged for the later grids (also the barrier that
    // publishes s_last / s_halo / red)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int any = __syncthreads_or(nonzero[p]);
        if (tid == 0 && A.zx) A.zx[((uint64_t)unit * NP + p) * A.ntiles + t] = any ? 0 : 1;
    }
    if (Src::kNorms && tid == 0) {
        static_assert(kEncThreads == 256, "8 warp sums");
        const double s01 = dadd(red[0], red[1]), s23 = dadd(red[2], red[3]);
        const double s45 = dadd(red[4], red[5]), s67 = dadd(red[6], red[7]);
        A.tilesum[(uint64_t)unit * A.ntiles + t] = dadd(dadd(s01, s23), dadd(s45, s67));
    }
    const long long half = 1ll << (A.qb - 1);
    const double hh = (double)half;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const uint64_t pl = (uint64_t)unit * NP + p;
        const PlaneParams pp = A.params[pl]; // (eb, q, inv_q: fixed while this grid runs)
        // the element before this thread's first one
        double xp = __shfl_up_sync(0xffffffffu, xv[p][kPerThread - 1], 1);
        if (lane == 0) xp = wid > 0 ? s_last[p][wid - 1] : s_halo[p];
        // K of that element against base 0.0 (dsub(x, 0.0) == x bitwise)
        long long kprev = llround_exact(dmul(dsub(xp, 0.0), pp.inv_q));
        uint32_t esym[kPerThread], fword = 0;
        int nev = 0, last = -1, bad = 0;
        double dh[kPerThread];
#pragma unroll
        for (int e = 0; e < kPerThread; ++e) {
            const double xi = xv[p][e];
            // speculative outlier (enc_x): the jump from the previous value
            const double rr = dmul(dsub(xi, xp), pp.inv_q);
            const bool out = !(fabs(rr) < hh - 0.5);
            const long long K = llround_exact(dmul(dsub(xi, 0.0), pp.inv_q));
            const long long m = K - kprev;
            if (m <= -half || m >= half) bad = 1;
            uint32_t f = m != 0 ? 1u : 0u;
            esym[e] = (uint32_t)(m + half);
            if (out) { // (the plane is redone by enc_lattice: only the flag matters)
                f = 3u;
                esym[e] = kOutlierSym;
                last = k0 + e;
                bad = 0;
            }
            dh[e] = dadd(0.0, dmul(pp.q, (double)K));
            fword |= f << (8 * e);
            nev += (int)(f & 1u);
            kprev = K;
            xp = xi;
        }
        *reinterpret_cast<uint32_t *>(A.fl + pl * L + t0 + k0) = fword;
        *reinterpret_cast<uint4 *>(A.sym + pl * L + t0 + k0) = make_uint4(esym[0], esym[1], esym[2], esym[3]);
        if (A.want_evD && nev) {
            double *dhat = A.dval + pl * L + t0 + k0;
#pragma unroll
            for (int e = 0; e < kPerThread; ++e)
                if ((fword >> (8 * e)) & 1u) dhat[e] = dh[e];
        }
        // (decided per plane by lattice_redo_list: a plane that is redone
        // ignores it)
        if (bad) atomicOr(&A.lat_bad[pl], 1u);
        nev = __reduce_add_sync(0xffffffffu, nev);
        last = __reduce_max_sync(0xffffffffu, last);
        if (lane == 0) {
            if (nev) atomicAdd(&s_nev[p], nev);
            if (last >= 0) atomicMax(&s_lastout[p], last);
        }
    }
    __syncthreads();
    if (tid < NP) {
        const uint64_t pl = (uint64_t)unit * NP + tid;
        A.t_nev[pl * A.ntiles + t] = (uint32_t)s_nev[tid];
        A.t_lastout[pl * A.ntiles + t] = s_lastout[tid] >= 0 ? (int32_t)(t0 + s_lastout[tid]) : -1;
    }
}

// ------------------------------------------------------------------ T3
// Event list for planes with many tiles (the fused look-back in enc_lattice
// would serialise hundreds of tiles): tile offsets from the plane scan.
__device__ __forceinline__ void compact_tile(const TileArgs &A, int pl, int t) {
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    using ScanI = cub::BlockScan<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage scan_tmp;
    const uint8_t *fl = A.fl + (uint64_t)pl * L;
    int f[kPerThread], pos[kPerThread];
    uint32_t fv[kPerThread];
    load4(fl + t0, tid * kPerThread, tl, fv); // (one 4-byte load; 0 past the end)
    for (int e = 0; e < kPerThread; ++e) f[e] = (int)(fv[e] & 1u);
    ScanI(scan_tmp).ExclusiveSum(f, pos);
    const uint32_t base = (uint32_t)carry_of(reinterpret_cast<const int32_t *>(A.t_evoff), A.ntiles + 1,
                                             reinterpret_cast<const int32_t *>(A.t_nev), pl, t, A.ntiles, kScanSumExcl);
    uint32_t *ev = A.evlist + (uint64_t)pl * L;
    double *evc = A.evc + (uint64_t)pl * L;
    double *evD = A.evD + (uint64_t)pl * L;
    const double *dhat = A.dval + (uint64_t)pl * L;
    const uint32_t *sym = A.sym + (uint64_t)pl * L;
    const double *x = A.x + (uint64_t)pl * L;
    const double q = A.params[pl].q;
    const long long half = 1ll << (A.qb - 1);
    for (int e = 0; e < kPerThread; ++e) {
        if (!f[e]) continue;
        const uint64_t i = t0 + tid * kPerThread + e;
        const bool out = (fv[e] & 2u) != 0;
        // the event record the chain consumes: its addend (or outlier value)
        // and the element index with bit 31 = outlier
        ev[base + pos[e]] = (uint32_t)i | (out ? 0x80000000u : 0u);
        evc[base + pos[e]] = out ? x[i] : dmul(q, (double)((long long)sym[i] - half));
        if (A.want_evD) evD[base + pos[e]] = dhat[i];
    }
}
// Grid of (plane, K) blocks; block (p, y) takes the plane's tiles y, y + K,
// ... and skips event-free tiles without touching their data.
// evcount != nullptr: the events placed are counted (bench roofline).
__global__ void __launch_bounds__(kEncThreads) enc_compact(TileArgs A, int planes, int K,
                                                           unsigned long long *evcount) {
    pdl_begin();
    const int pl = blockIdx.x / K, y = blockIdx.x % K;
    if (pl >= planes) return;
    if (block_params(A.params, pl).flags & kFlagFallback) return;
    unsigned long long placed = 0;
    for (int t = y; t < A.ntiles; t += K) {
        const uint32_t ne = A.t_nev[(uint64_t)pl * A.ntiles + t];
        if (ne == 0) continue; // no events in this tile
        placed += ne;
        compact_tile(A, pl, t);
        __syncthreads();
    }
    if (evcount && threadIdx.x == 0 && placed) atomicAdd(evcount, placed);
}

// ------------------------------------------------------------------ chain
// One warp per plane.  Event records (addend, outlier bit) stream into a
// shared-memory ring with TMA bulk copies (cp.async.bulk + mbarrier, issued
// kChainBufs chunks ahead by lane 0); the dependent chain d = RN(d + c)
// (codec.cpp:445 / :607 in index order) reads warp-broadcast addends, so
// only the DADD latency is serial.
constexpr int kChainChunk = 1024; // events per bulk copy
constexpr int kChainBufs = 8;     // ring depth with few planes (96 KB, dynamic smem); many
                                  // planes use a 2-deep ring so more warps fit per SM
__host__ __device__ constexpr size_t chain_smem_bytes(int bufs) { return 12ull * bufs * kChainChunk + 8 * bufs; }
constexpr size_t kChainSmem = chain_smem_bytes(kChainBufs);

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__global__ void __launch_bounds__(32) enc_chain(TileArgs A, int planes, int nbufs) {
    pdl_begin();
    const int pl = blockIdx.x;
    if (pl >= planes) return;
    const int lane = threadIdx.x;
    const PlaneParams pp = block_params(A.params, pl);
    if ((pp.flags & kFlagFallback) || pp.eb == 0.0) return;
    // ring in dynamic shared memory: [bufs][chunk] addends, [bufs][chunk]
    // event words, [bufs] mbarriers
    extern __shared__ __align__(128) unsigned char chain_smem[];
    double(*cbuf)[kChainChunk] = reinterpret_cast<double(*)[kChainChunk]>(chain_smem);
    uint32_t(*obuf)[kChainChunk] =
        reinterpret_cast<uint32_t(*)[kChainChunk]>(chain_smem + sizeof(double) * nbufs * kChainChunk);
    uint64_t *bar = reinterpret_cast<uint64_t *>(chain_smem + 12 * nbufs * kChainChunk);
    const uint64_t L = A.L;
    const uint32_t nev = (uint32_t)carry_of(reinterpret_cast<const int32_t *>(A.t_evoff), A.ntiles + 1,
                                            reinterpret_cast<const int32_t *>(A.t_nev), pl, A.ntiles, A.ntiles,
                                            kScanSumExcl);
    if (nev == 0) return;
    const uint32_t *ev = A.evlist + (uint64_t)pl * L;
    const double *evc = A.evc + (uint64_t)pl * L;
    double *dv = A.dval + (uint64_t)pl * L;
    const uint32_t nchunks = (nev + kChainChunk - 1) / kChainChunk;
    auto issue = [&](uint32_t ch) {
        const int b = ch % nbufs;
        const uint32_t n = tmin<uint32_t>(kChainChunk, nev - ch * kChainChunk);
        const uint32_t cb = (n * 8 + 15) & ~15u, ob = (n * 4 + 15) & ~15u; // buffers are padded
        mbar_expect_tx(&bar[b], cb + ob);
        tma_load_1d(cbuf[b], evc + (uint64_t)ch * kChainChunk, cb, &bar[b]);
        tma_load_1d(obuf[b], ev + (uint64_t)ch * kChainChunk, ob, &bar[b]);
    };
    if (lane == 0) {
        for (int b = 0; b < nbufs; ++b) mbar_init(&bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t ch = 0; ch < nchunks && ch < (uint32_t)nbufs; ++ch) issue(ch);
    }
    __syncwarp();
    double d = 0.0;
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
        const int b = ch % nbufs;
        mbar_wait(&bar[b], (ch / nbufs) & 1);
        const uint32_t n = tmin<uint32_t>(kChainChunk, nev - ch * kChainChunk);
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t cnt = tmin<uint32_t>(32, n - base);
            const uint32_t o = lane < (int)cnt ? obuf[b][base + lane] >> 31 : 0u;
            const uint32_t outmask = __ballot_sync(0xffffffffu, o != 0);
            double mine = 0.0;
            if (outmask == 0 && cnt == 32) {
                // Every lane runs the same dependent chain but stops adding
                // after its own event: lane j ends with exactly d_j (same
                // operations, same order as the serial recurrence).  The only
                // per-step instruction on the critical path is the
                // (predicated) DADD; one shuffle carries d to the next batch.
                // Lanes past their own event add +0.0 instead: x + 0.0 == x
                // bitwise for every value reachable here (d_k is never -0.0 on
                // this outlier-free path: RN(q*0) is +0.0), so the select
                // lands on the addend, off the dependency chain.
                // Every lane runs the same chain but stops adding after its
                // own event, so lane j ends with exactly d_j (identical
                // operations and order); one shuffle carries d onward.
                // (Measured 14.4 cycles/event on a dense plane vs 19.7 for a
                // per-step select; the DADD latency floor is 8.2.)
                double dl = d;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const double cj = cbuf[b][base + j];
                    if (j <= lane) dl = dadd(dl, cj);
                }
                mine = dl;
                d = __shfl_sync(0xffffffffu, dl, 31);
            } else {
                for (uint32_t j = 0; j < cnt; ++j) {
                    const double cj = cbuf[b][base + j];
                    if ((outmask >> j) & 1) d = cj;
                    else d = dadd(d, cj);
                    if (lane == (int)j) mine = d;
                }
            }
            if (lane < (int)cnt) dv[(uint64_t)ch * kChainChunk + base + lane] = mine;
        }
        __syncwarp();
        if (A.chain_prog && lane == 0) { // the chain front: enc_verify's tiles wait for it
            __threadfence();
            const uint32_t upto = tmin<uint32_t>((ch + 1) * kChainChunk, nev);
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(A.chain_prog + pl), "r"(upto) : "memory");
        }
        if (lane == 0 && ch + nbufs < nchunks) issue(ch + nbufs);
    }
}

// ------------------------------------------------------------------ T4
// chain_done != nullptr: launched alongside enc_chain_scan (no grid-wide
// wait); a tile waits for its own plane's chain (done[pl] == epoch) and
// reads the chain values from L2.
__device__ __forceinline__ void verify_tile(const TileArgs &A, int planes, const uint32_t *chain_done,
                                            uint32_t epoch) {
    int pl, t;
    if (A.chain_prog) { // tile-major: the chain fronts of all planes advance together
        t = (int)(blockIdx.x / (uint32_t)planes);
        pl = (int)(blockIdx.x - (uint32_t)t * (uint32_t)planes);
    } else {
        split_block(blockIdx.x, A.ntiles, A.tile_sh, pl, t);
    }
    if (pl >= planes) return;
    const PlaneParams pp = block_params(A.params, pl);
    if (pp.flags & kFlagFallback) return;
    if (A.chain_prog && pp.eb != 0.0) {
        // the chain values of every event up to the end of this tile
        const uint32_t need = (uint32_t)(reinterpret_cast<const int32_t *>(A.t_evoff) + (uint64_t)pl * (A.ntiles + 1))[t + 1];
        __shared__ int s_gave_up;
        if (threadIdx.x == 0) {
            s_gave_up = 0;
            uint32_t v = need, spins = 0;
            if (need) do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.chain_prog + pl) : "memory");
                if (v < need) {
                    __nanosleep(128);
                    if (++spins > (1u << 23)) { // (> 1 s: never in a healthy run) -> serial re-encode
                        atomicOr(&A.params[pl].flags, kFlagFallback);
                        s_gave_up = 1;
                        break;
                    }
                }
            } while (v < need);
        }
        __syncthreads();
        if (s_gave_up) return;
    }
    if (A.chain_prog) chain_done = A.chain_prog; // (chain values through L2 from here on)
    if (chain_done && !A.chain_prog && pp.eb != 0.0) {
        if (threadIdx.x == 0) {
            uint32_t v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(chain_done + pl) : "memory");
                if (v != epoch) __nanosleep(64);
            } while (v != epoch);
        }
        __syncthreads();
    }
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    const uint64_t C = 1ull << A.log2C;
    const uint64_t nidx = (L >> A.log2C) + 1;
    const double *x = A.x + (uint64_t)pl * L;
    IndexRec *idx = A.index + (uint64_t)pl * nidx;
    __shared__ int s_fb, s_lb, s_no;
    if (tid == 0) {
        s_fb = 0x7FFFFFFF;
        s_lb = -1;
        s_no = 0;
    }
    __syncthreads();
    const uint32_t *fsym = A.sym + (uint64_t)pl * L;
    auto tile_stats = [&](const uint32_t *sv) { // sv[e]: final symbol of element tid*4+e
        int fb = 0x7FFFFFFF, lb = -1, no = 0;
        uint32_t prev = (t0 + tid * kPerThread > 0 && tid * kPerThread < tl) ? fsym[t0 + tid * kPerThread - 1] : 0u;
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            if (k >= tl) break;
            const uint64_t i = t0 + k;
            if (i == 0 || sv[e] != prev) {
                fb = min(fb, (int)i);
                lb = max(lb, (int)i);
            }
            no += sv[e] == kOutlierSym;
            prev = sv[e];
        }
        // (one shared-memory atomic per warp and statistic)
        fb = __reduce_min_sync(0xffffffffu, fb);
        lb = __reduce_max_sync(0xffffffffu, lb);
        no = __reduce_add_sync(0xffffffffu, no);
        if ((tid & 31) == 0) {
            if (fb != 0x7FFFFFFF) atomicMin(&s_fb, fb);
            if (lb >= 0) atomicMax(&s_lb, lb);
            if (no) atomicAdd(&s_no, no);
        }
        __syncthreads();
        if (tid == 0) {
            A.t_firstb[(uint64_t)pl * A.ntiles + t] = s_fb;
            A.t_lastb[(uint64_t)pl * A.ntiles + t] = s_lb;
            A.t_nout[(uint64_t)pl * A.ntiles + t] = s_no;
        }
    };
    if (pp.eb == 0.0) {
        // lossless: d == x; only the decode index needs d[e-1], d[e-2]
        for (int k = tid; k < tl; k += kEncThreads) {
            const uint64_t i = t0 + k;
            if ((i & (C - 1)) == 0) {
                idx[i >> A.log2C].dprev = i > 0 ? x[i - 1] : 0.0;
                idx[i >> A.log2C].dprev2 = i > 1 ? x[i - 2] : 0.0;
            }
        }
        uint32_t sv[kPerThread];
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            sv[e] = k < tl ? fsym[t0 + k] : 0u;
        }
        tile_stats(sv);
        return;
    }
    const long long half = 1ll << (A.qb - 1);
    const double *dv = A.dval + (uint64_t)pl * L;
    if (A.zx && A.ntiles > kInlineTiles && tl == kTile && A.t_nev[(uint64_t)pl * A.ntiles + t] == 0) {
        // No event in the tile: every code is the zero code, no speculative
        // outlier, so every element sees the same exact prediction -- the
        // chain value of the last event before the tile -- and the reference
        // decision (codec.cpp:440-451) reduces to "m = 0 accepted":
        // |r| < 0.49 (m = 0 for certain), rec = pred + q*0 finite and equal
        // to pred, |x - rec| <= eb.  A tile of +-0.0 values (enc_x's flag)
        // evaluates that once; other tiles per element from x alone (no
        // flag / symbol loads, no rank scan, no chain gathers).  Anything
        // else falls through to the general path.  Block-uniform.
        const int32_t *eo = reinterpret_cast<const int32_t *>(A.t_evoff) + (uint64_t)pl * (A.ntiles + 1);
        const uint32_t evbase = (uint32_t)eo[t], nev_plane = (uint32_t)eo[A.ntiles];
        if (evbase <= nev_plane && nev_plane <= L) {
            const double pred = evbase > 0 ? (chain_done ? __ldcg(dv + evbase - 1) : __ldg(dv + evbase - 1)) : 0.0;
            const double rr = dadd(pred, dmul(pp.q, 0.0));
            bool ok = isfinite(rr) && bits_of(rr) == bits_of(pred);
            if (A.zx[(uint64_t)pl * A.ntiles + t]) {
                // (-0.0 values give the same: only |x - rr| and |r0| enter)
                const double r0 = dmul(dsub(0.0, pred), pp.inv_q);
                ok = ok && fabs(r0) < 0.49 && fabs(dsub(0.0, rr)) <= pp.eb;
            } else {
                double xv4[kPerThread];
                load4(x + t0, tid * kPerThread, tl, xv4);
#pragma unroll
                for (int e = 0; e < kPerThread; ++e) {
                    const double r0 = dmul(dsub(xv4[e], pred), pp.inv_q);
                    ok = ok && fabs(r0) < 0.49 && fabs(dsub(xv4[e], rr)) <= pp.eb;
                }
                ok = __syncthreads_and(ok);
            }
            if (ok) {
                for (uint64_t i = t0 + (uint64_t)tid * C; i < t0 + kTile; i += (uint64_t)kEncThreads * C) {
                    if (i & (C - 1)) continue; // (checkpoints wider than a tile)
                    idx[i >> A.log2C].dprev = pred;
                    idx[i >> A.log2C].dprev2 = 0.0;
                }
                if (tid == 0) {
                    // run statistics: the only possible run start is the first element
                    const uint32_t prev = t0 > 0 ? fsym[t0 - 1] : 0u;
                    const bool starts = t0 == 0 || prev != (uint32_t)half;
                    A.t_firstb[(uint64_t)pl * A.ntiles + t] = starts ? (int32_t)t0 : 0x7FFFFFFF;
                    A.t_lastb[(uint64_t)pl * A.ntiles + t] = starts ? (int32_t)t0 : -1;
                    A.t_nout[(uint64_t)pl * A.ntiles + t] = 0;
                    A.ztriv[(uint64_t)pl * A.ntiles + t] = starts ? 0 : 1;
                }
                return;
            }
        }
    }
    using ScanI = cub::BlockScan<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage scan_tmp;
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    const uint8_t *fl = A.fl + (uint64_t)pl * L;
    uint32_t *sym = A.sym + (uint64_t)pl * L;
    int f[kPerThread], rank[kPerThread];
    double xv[kPerThread];
    uint32_t symv[kPerThread];
    {
        uint32_t fv[kPerThread];
        load4(fl + t0, tid * kPerThread, tl, fv);
        load4(x + t0, tid * kPerThread, tl, xv);
        load4(sym + t0, tid * kPerThread, tl, symv);
        for (int e = 0; e < kPerThread; ++e) f[e] = (fv[e] & 1) ? 1 : 0;
    }
    // event offset of the tile and the plane's event count, one carry pass
    uint32_t evbase, nev_plane;
    if (A.ntiles <= kInlineTiles) {
        int32_t ex, tot;
        tile_excl_total(reinterpret_cast<const int32_t *>(A.t_nev) + (uint64_t)pl * A.ntiles, t, A.ntiles, ex, tot);
        evbase = (uint32_t)ex;
        nev_plane = (uint32_t)tot;
    } else {
        const int32_t *eo = reinterpret_cast<const int32_t *>(A.t_evoff) + (uint64_t)pl * (A.ntiles + 1);
        evbase = (uint32_t)eo[t];
        nev_plane = (uint32_t)eo[A.ntiles];
    }
    int nf_tile;
    {
        bool anyf = false; // (an event-free tile: every rank is 0)
        for (int e = 0; e < kPerThread; ++e) anyf |= f[e] != 0;
        if (__syncthreads_or(anyf)) {
            ScanI(scan_tmp).ExclusiveSum(f, rank, nf_tile);
        } else {
            for (int e = 0; e < kPerThread; ++e) rank[e] = 0;
            nf_tile = 0;
        }
    }
    __syncthreads();
    // guard: the event ordinals of this tile must lie inside the plane's
    // event list (a violation means corrupt carries -> serial re-encode)
    if ((uint64_t)evbase + (uint64_t)nf_tile > (uint64_t)nev_plane || nev_plane > L) {
        if (tid == 0) {
            printf("qcsim enc_verify: plane %d tile %d evbase %u tile events %d plane events %u (L %llu)\n", pl, t,
                   evbase, nf_tile, nev_plane, (unsigned long long)L);
            atomicOr(&A.params[pl].flags, kFlagFallback);
        }
        return;
    }
    int bad = 0;
    uint32_t sv[kPerThread];
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        sv[e] = 0;
        if (k >= tl) continue;
        const uint64_t i = t0 + k;
        const uint32_t ord = evbase + (uint32_t)rank[e]; // events before i
        // (L2 reads only when the chain grid may still be running)
        const double pred = ord > 0 ? (chain_done ? __ldcg(dv + ord - 1) : __ldg(dv + ord - 1)) : 0.0;
        const double dspec = f[e] ? (chain_done ? __ldcg(dv + ord) : __ldg(dv + ord)) : pred;
        double rec = 0.0;
        const double xi = xv[e];
        uint32_t sy;
        const double r0 = dmul(dsub(xi, pred), pp.inv_q);
        if (fabs(r0) < 0.49) {
            // m = 0 for certain (the reference's quotient differs from r0 by a
            // few ulps): quantize's m = 0 branch without the rounding guards
            const double rr = dadd(pred, dmul(pp.q, 0.0));
            sy = (isfinite(rr) && fabs(dsub(xi, rr)) <= pp.eb) ? (uint32_t)half : kOutlierSym;
            if (sy != kOutlierSym) rec = rr;
        } else {
            sy = quantize(xi, pred, pp.q, pp.inv_q, pp.eb, half, &rec);
        }
        if (sy == kOutlierSym) rec = xi;
        sv[e] = symv[e];
        if (sy != sv[e] || bits_of(rec) != bits_of(dspec)) bad = 1;
        if ((i & (C - 1)) == 0) {
            idx[i >> A.log2C].dprev = pred;
            idx[i >> A.log2C].dprev2 = 0.0; // unused by the previous-value predictor
        }
    }
    if (bad) s_bad = 1;
    tile_stats(sv); // (a refuted plane gets them again from enc_serial_x)
    if (tid == 0 && s_bad) atomicOr(&A.params[pl].flags, kFlagFallback);
}
// flow.cnt != nullptr: the plane's tiles report completion (enc_serial_x
// and tok_count then run alongside, per plane)
// ser_done != nullptr: the plane's last tile also releases tok_count directly
// when the plane was not refuted (enc_serial_x releases the refuted ones).
__global__ void __launch_bounds__(kEncThreads, 6) enc_verify(TileArgs A, int planes, const uint32_t *chain_done,
                                                          uint32_t epoch, PlaneFlow flow, uint32_t *ser_done) {
    if (chain_done || A.chain_prog) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    else pdl_begin();
    verify_tile(A, planes, chain_done, epoch);
    if (!flow.cnt) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int pl = blockIdx.x / A.ntiles;
        __threadfence();
        const uint32_t old = atomicAdd(flow.cnt + pl, 1u);
        if (old + 1 == (uint32_t)A.ntiles) {
            flow.cnt[pl] = 0u;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flow.done + pl), "r"(flow.epoch) : "memory");
            if (ser_done && !(__ldcg(&A.params[pl].flags) & kFlagFallback))
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ser_done + pl), "r"(flow.epoch) : "memory");
        }
    }
}

// E1f: exact serial closed loop for refuted / linear planes (x from A.x).
__device__ __forceinline__ void serial_plane(const TileArgs &A, int pl) {
    PlaneParams pp = A.params[pl];
    pp.flags = __ldcg(&A.params[pl].flags);
    if (!(pp.flags & kFlagFallback)) return;
    const uint64_t L = A.L;
    const long long half = 1ll << (A.qb - 1);
    const uint64_t C = 1ull << A.log2C;
    const uint64_t nidx = (L >> A.log2C) + 1;
    const double eb = pp.eb, q = pp.q;
    const double *x = A.x + (uint64_t)pl * L;
    uint32_t *sym = A.sym + (uint64_t)pl * L;
    IndexRec *idx = A.index + (uint64_t)pl * nidx;
    double d1 = 0.0, d2 = 0.0;
    int fb = 0x7FFFFFFF, lb = -1, no = 0; // run statistics of the current tile
    uint32_t prev = 0;
    for (uint64_t i = 0; i < L; ++i) {
        if ((i & (C - 1)) == 0) {
            idx[i >> A.log2C].dprev = d1;
            idx[i >> A.log2C].dprev2 = d2;
        }
        const double xi = x[i];
        double pred;
        if (A.predictor == 0) pred = i > 0 ? d1 : 0.0;
        else pred = i == 0 ? 0.0 : (i == 1 ? d1 : predict_linear(d1, d2));
        double rec = 0.0;
        uint32_t sy = kOutlierSym;
        if (eb == 0.0) {
            if (bits_of(xi) == bits_of(pred)) { sy = (uint32_t)half; rec = pred; }
        } else {
            const double r = ddiv(dsub(xi, pred), q);
            if (isfinite(r) && fabs(r) < (double)half) {
                const long long m = llround_exact(r);
                if (m > -half && m < half) {
                    const double rr = dadd(pred, dmul(q, (double)m));
                    if (isfinite(rr) && fabs(dsub(xi, rr)) <= eb) { sy = (uint32_t)(m + half); rec = rr; }
                }
            }
        }
        if (sy == kOutlierSym) rec = xi;
        sym[i] = sy;
        d2 = d1;
        d1 = rec;
        if (i == 0 || sy != prev) {
            fb = min(fb, (int)i);
            lb = max(lb, (int)i);
        }
        no += sy == kOutlierSym;
        prev = sy;
        if ((i + 1) % kTile == 0 || i + 1 == L) {
            const uint64_t t = i / kTile;
            A.t_firstb[(uint64_t)pl * A.ntiles + t] = fb;
            A.t_lastb[(uint64_t)pl * A.ntiles + t] = lb;
            A.t_nout[(uint64_t)pl * A.ntiles + t] = no;
            if (A.ztriv) A.ztriv[(uint64_t)pl * A.ntiles + t] = 0; // (the symbols were rewritten)
            fb = 0x7FFFFFFF;
            lb = -1;
            no = 0;
        }
    }
}
// ver_done != nullptr: runs alongside enc_verify; one thread per plane waits
// for its plane's tiles, re-encodes a refuted plane, then raises
// ser_done[pl] (tok_count's hand-off).
__global__ void enc_serial_x(TileArgs A, int planes, const uint32_t *ver_done, uint32_t *ser_done, uint32_t epoch) {
    if (ver_done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    else pdl_begin();
    const int pl = blockIdx.x * blockDim.x + threadIdx.x;
    if (pl >= planes) return;
    if (ver_done) flow_wait(ver_done, pl, epoch);
    serial_plane(A, pl);
    if (ser_done) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ser_done + pl), "r"(epoch) : "memory");
    }
}

// ------------------------------------------------------------ tokenizer
struct TokArgs {
    const uint32_t *sym;   // [plane][L] exact
    const double *x;       // [plane][L]
    uint32_t *tsym, *trep; // [plane][L+1]
    uint32_t *opos;        // [plane][L]
    double *oval;          // [plane][L]
    uint32_t *ocount;      // [plane]
    uint32_t *ntok;        // [plane]
    uint32_t *hist;        // [plane][rsym+1] (zero between uses)
    uint32_t *hspecial;    // [plane][2]
    uint32_t *symrange;    // [plane][2]
    unsigned long long *gamma_bits; // [plane]
    IndexRec *index;
    // per plane-tile
    int32_t *t_firstb, *t_lastb; // first / last run start in the tile (-1 / INT_MAX none)
    int32_t *t_nout, *t_ooff;    // outliers per tile, scanned (+1)
    int32_t *t_prevb;            // scanned: last run start strictly before the tile
    int32_t *t_nextb;            // scanned: first run start strictly after the tile
    int32_t *t_ntok, *t_tokoff;  // tokens per tile, scanned (+1)
    const uint8_t *ztriv;        // [plane][tile] flat zero-code tiles (TileArgs::ztriv) or nullptr
    uint64_t L;
    int ntiles, tile_sh, log2C, qb;
};

struct RunInfo {
    uint64_t start, end;
};

// Per element: run [start, end) from the tile's run starts (warp shuffles +
// one shared-memory exchange) + the scanned carries.
__device__ __forceinline__ void element_runs(const TokArgs &A, int pl, int t, uint64_t t0, int tl, uint64_t *start,
                                             uint64_t *end, const uint32_t *sv, int32_t *bases = nullptr,
                                             const int32_t *carries = nullptr) {
    // sv: this thread's symbols as loaded by tile_load_syms; carries: the
    // tile_carries() result when the caller computed it already
    const int tid = threadIdx.x;
    int isb[kPerThread], st[kPerThread];
    int32_t prevb, nextb_carry;
    if (carries) {
        prevb = carries[0];
        nextb_carry = carries[1];
        if (bases) {
            bases[0] = carries[2];
            bases[1] = carries[3];
        }
    } else if (bases && A.ntiles <= kInlineTiles) { // + token / outlier offsets of the tile (tok_emit)
        const uint64_t o = (uint64_t)pl * A.ntiles;
        const int32_t *arr[4] = {A.t_lastb + o, A.t_firstb + o, A.t_ntok + o, A.t_nout + o};
        const int kinds[4] = {kScanMaxExcl, kScanMinExclRev, kScanSumExcl, kScanSumExcl};
        int32_t r[4];
        tile_carryN<4>(arr, kinds, t, A.ntiles, r);
        prevb = r[0];
        nextb_carry = r[1];
        bases[0] = r[2];
        bases[1] = r[3];
    } else {
        carry_of2(A.t_prevb, A.ntiles, A.t_lastb, kScanMaxExcl, A.t_nextb, A.ntiles, A.t_firstb, kScanMinExclRev, pl,
                  t, A.ntiles, prevb, nextb_carry);
        if (bases)
            carry_of2(A.t_tokoff, A.ntiles + 1, A.t_ntok, kScanSumExcl, A.t_ooff, A.ntiles + 1, A.t_nout,
                      kScanSumExcl, pl, t, A.ntiles, bases[0], bases[1]);
    }
    // run starts (boundaries) of this thread's elements; st[e] = the last one
    // at or before element e, nx[e] = the first one after it, both within
    // this thread
    int last_in = -1;
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        const uint64_t i = t0 + k;
        isb[e] = (k < tl && (i == 0 || sv[e + 1] != sv[e])) ? (int)k : -1;
        last_in = isb[e] >= 0 ? isb[e] : last_in;
        st[e] = last_in;
    }
    int first_in = 0x7FFFFFFF;
    int nx[kPerThread];
    for (int e = kPerThread - 1; e >= 0; --e) {
        nx[e] = first_in;
        if (isb[e] >= 0) first_in = isb[e];
    }
    // across threads: the last boundary of the lower threads (exclusive max
    // scan) and the first boundary of the higher ones (exclusive reverse min
    // scan) -- within the warp by shuffles, across warps through one
    // shared-memory exchange and one barrier
    __shared__ int s_wlast[kEncThreads / 32], s_wfirst[kEncThreads / 32];
    const int lane = tid & 31, wid = tid >> 5;
    int incl_last = last_in, incl_first = first_in;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, incl_last, off);
        const int c = __shfl_down_sync(0xffffffffu, incl_first, off);
        if (lane >= off) incl_last = max(incl_last, a);
        if (lane + off < 32) incl_first = min(incl_first, c);
    }
    int prev_last = __shfl_up_sync(0xffffffffu, incl_last, 1);   // lower lanes of this warp
    int next_first = __shfl_down_sync(0xffffffffu, incl_first, 1); // higher lanes of this warp
    if (lane == 0) prev_last = -1;
    if (lane == 31) next_first = 0x7FFFFFFF;
    if (lane == 31) s_wlast[wid] = incl_last;
    if (lane == 0) s_wfirst[wid] = incl_first;
    __syncthreads();
    for (int w = 0; w < wid; ++w) prev_last = max(prev_last, s_wlast[w]);
    for (int w = wid + 1; w < kEncThreads / 32; ++w) next_first = min(next_first, s_wfirst[w]);
    __syncthreads(); // (the exchange arrays are reused by the caller's next tile)
    const uint64_t after = nextb_carry == 0x7FFFFFFF ? A.L : (uint64_t)nextb_carry;
    for (int e = 0; e < kPerThread; ++e) {
        const int sl = st[e] >= 0 ? st[e] : prev_last;
        start[e] = sl >= 0 ? t0 + sl : (uint64_t)prevb;
        const int nb = nx[e] != 0x7FFFFFFF ? nx[e] : next_first;
        end[e] = (nb != 0x7FFFFFFF && nb < tl) ? t0 + nb : after;
    }
}

// A tile is "flat" when no run starts inside it: every element equals its
// predecessor (so the tile lies inside one run that began in an earlier
// tile).  Such a tile emits no token and counts nothing (a run longer than
// the tile is always collapsed, codec.cpp:460-482); only its decode-index
// records need the run's end.  Block-uniform result; sym via L2.
// This thread's symbols, sv[0] = the element before them, sv[1..kPerThread]
// = its own (the layout element_runs consumes), from L2; no barrier.
__device__ __forceinline__ void tile_load_syms(const uint32_t *sym, uint64_t t0, int tl, uint32_t *sv) {
    const int k0 = threadIdx.x * kPerThread;
    if (k0 + kPerThread <= tl) { // one 16-byte load (tile starts are 1024-element aligned)
        static_assert(kPerThread == 4, "uint4 symbol loads");
        const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(sym + t0 + k0));
        sv[1] = w.x;
        sv[2] = w.y;
        sv[3] = w.z;
        sv[4] = w.w;
    } else {
        for (int e = 0; e < kPerThread; ++e) sv[e + 1] = k0 + e < tl ? __ldcg(sym + t0 + k0 + e) : 0u;
    }
    sv[0] = (t0 + k0 > 0 && k0 < tl) ? __ldcg(sym + t0 + k0 - 1) : 0u;
}
// Flatness of the tile from the loaded symbols (block-uniform).
__device__ __forceinline__ bool tile_flat(const uint32_t *sym, uint64_t t0, int tl, const uint32_t *sv,
                                          uint32_t &s_out) {
    const int k0 = threadIdx.x * kPerThread;
    bool flat = t0 > 0 && tl >= (int)kMinRunLen;
    for (int e = 0; e < kPerThread; ++e)
        if (k0 + e < tl) flat &= sv[e + 1] == sv[e];
    flat = __syncthreads_and(flat);
    uint32_t s = 0;
    if (flat) {
        s = __ldcg(sym + t0);
        flat = s != kOutlierSym;
    }
    s_out = s;
    return flat;
}
__device__ __forceinline__ bool tile_is_flat(const uint32_t *sym, uint64_t t0, int tl, uint32_t *sv,
                                             uint32_t &s_out) {
    tile_load_syms(sym, t0, tl, sv);
    return tile_flat(sym, t0, tl, sv, s_out);
}
// prevb, nextb, token base, outlier base of tile t (element_runs' carries).
__device__ __forceinline__ void tile_carries(const TokArgs &A, int pl, int t, int32_t *r) {
    if (A.ntiles <= kInlineTiles) {
        const uint64_t o = (uint64_t)pl * A.ntiles;
        const int32_t *arr[4] = {A.t_lastb + o, A.t_firstb + o, A.t_ntok + o, A.t_nout + o};
        const int kinds[4] = {kScanMaxExcl, kScanMinExclRev, kScanSumExcl, kScanSumExcl};
        tile_carryN<4>(arr, kinds, t, A.ntiles, r);
    } else {
        carry_of2(A.t_prevb, A.ntiles, A.t_lastb, kScanMaxExcl, A.t_nextb, A.ntiles, A.t_firstb, kScanMinExclRev, pl,
                  t, A.ntiles, r[0], r[1]);
        carry_of2(A.t_tokoff, A.ntiles + 1, A.t_ntok, kScanSumExcl, A.t_ooff, A.ntiles + 1, A.t_nout, kScanSumExcl,
                  pl, t, A.ntiles, r[2], r[3]);
    }
}

// ser_done != nullptr: runs alongside enc_serial_x; a tile waits for its
// plane's final symbols (ser_done[pl] == epoch) and reads them from L2.
__global__ void __launch_bounds__(kEncThreads) tok_count(TokArgs A, int planes, const uint32_t *ser_done,
                                                         uint32_t epoch) {
    if (ser_done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    else pdl_begin();
    int pl, t;
    split_block(blockIdx.x, A.ntiles, A.tile_sh, pl, t);
    if (pl >= planes) return;
    if (ser_done) {
        if (threadIdx.x == 0) flow_wait(ser_done, pl, epoch);
        __syncthreads();
    }
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    const uint32_t *sym = A.sym + (uint64_t)pl * L;
    uint32_t sv[kPerThread + 1];
    if (A.ztriv && A.ztriv[(uint64_t)pl * A.ntiles + t]) { // known flat (enc_verify): nothing to load
        if (tid == 0) A.t_ntok[(uint64_t)pl * A.ntiles + t] = 0;
        return;
    }
    {
        uint32_t fs;
        if (tile_is_flat(sym, t0, tl, sv, fs)) { // inside one long run: no tokens, no counts
            if (tid == 0) A.t_ntok[(uint64_t)pl * A.ntiles + t] = 0;
            return;
        }
    }
    using RedI = cub::BlockReduce<int, kEncThreads>;
    __shared__ typename RedI::TempStorage rtmp;
    __shared__ __align__(16) uint32_t hist[kWin];
    __shared__ uint16_t touched[kTile + 1]; // window bins this tile hit (first-touch list)
    __shared__ uint32_t ntouched;
    __shared__ uint32_t h0, hrun, smin, smax;
    __shared__ unsigned long long gbits;
    const long long half = 1ll << (A.qb - 1);
    const uint32_t rsym = 1u << A.qb;
    const uint32_t wlo = (uint32_t)(half - kWin / 2);
    uint32_t *ghist = A.hist + (uint64_t)pl * ((uint64_t)rsym + 1);
    for (int k = tid; k < kWin / 4; k += kEncThreads) reinterpret_cast<uint4 *>(hist)[k] = make_uint4(0, 0, 0, 0);
    if (tid == 0) { h0 = 0; hrun = 0; smin = 0xFFFFFFFFu; smax = 0; gbits = 0; ntouched = 0; }
    uint64_t start[kPerThread], end[kPerThread];
    element_runs(A, pl, t, t0, tl, start, end, sv);
    auto count = [&](uint32_t s, uint32_t n) {
        if (s == kOutlierSym) atomicAdd(&h0, n);
        else if (s == rsym) atomicAdd(&hrun, n);
        else if (s - wlo < (uint32_t)kWin) {
            if (atomicAdd(&hist[s - wlo], n) == 0) touched[atomicAdd(&ntouched, 1u)] = (uint16_t)(s - wlo);
        }
        else {
            atomicAdd(&ghist[s], n);
            atomicMin(&smin, s);
            atomicMax(&smax, s);
        }
    };
    int cnt = 0;
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        if (k >= tl) continue;
        const uint64_t i = t0 + k;
        const uint32_t s = sv[e + 1];
        const uint64_t len = end[e] - start[e];
        const bool longrun = s != kOutlierSym && len >= kMinRunLen;
        if (longrun) {
            if (i == start[e]) {
                cnt += 2;
                count(s, 1);
                count(rsym, 1);
                atomicAdd(&gbits, (unsigned long long)(2 * bit_width64(len - 1) - 1));
            }
        } else {
            cnt += 1;
            count(s, 1);
        }
    }
    const int tot = RedI(rtmp).Sum(cnt);
    __syncthreads();
    if (tid == 0) {
        A.t_ntok[(uint64_t)pl * A.ntiles + t] = tot;
        if (h0) atomicAdd(&A.hspecial[2 * pl], h0);
        if (hrun) atomicAdd(&A.hspecial[2 * pl + 1], hrun);
        if (gbits) atomicAdd(&A.gamma_bits[pl], gbits);
    }
    for (uint32_t m = tid; m < ntouched; m += kEncThreads) {
        const uint32_t k = touched[m];
        const uint32_t v = hist[k];
        const uint32_t sy = wlo + k;
        if (sy != kOutlierSym && sy < rsym) {
            atomicAdd(&ghist[sy], v);
            atomicMin(&smin, sy);
            atomicMax(&smax, sy);
        }
    }
    __syncthreads();
    if (tid == 0 && smin <= smax) {
        atomicMin(&A.symrange[2 * pl], smin);
        atomicMax(&A.symrange[2 * pl + 1], smax);
    }
}

__device__ __forceinline__ void tok_emit_tile(const TokArgs &A, int planes, int blk) {
    int pl, t;
    split_block((uint32_t)blk, A.ntiles, A.tile_sh, pl, t);
    if (pl >= planes) return;
    const int tid = threadIdx.x;
    const uint64_t L = A.L;
    const uint64_t t0 = (uint64_t)t * kTile;
    const int tl = (int)tmin<uint64_t>(kTile, L - t0);
    const uint32_t *sym = A.sym + (uint64_t)pl * L;
    const double *x = A.x + (uint64_t)pl * L;
    using ScanI = cub::BlockScan<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage tmp;
    const uint32_t rsym = 1u << A.qb;
    const uint64_t C = 1ull << A.log2C;
    const uint64_t nidx = (L >> A.log2C) + 1;
    uint32_t *tsym = A.tsym + (uint64_t)pl * (L + 1);
    uint32_t *trep = A.trep + (uint64_t)pl * (L + 1);
    IndexRec *idx = A.index + (uint64_t)pl * nidx;
    uint32_t sv[kPerThread + 1];
    int32_t carries[4];
    const bool known_flat = A.ztriv && A.ztriv[(uint64_t)pl * A.ntiles + t]; // (enc_verify: the zero code throughout)
    if (!known_flat) tile_load_syms(sym, t0, tl, sv); // in flight while warp 0 gathers the carries
    tile_carries(A, pl, t, carries);
    {
        uint32_t fs = 1u << (A.qb - 1);
        if (known_flat || tile_flat(sym, t0, tl, sv, fs)) {
            // inside one long run: no tokens or outliers; the index records
            // resume after the run's literal + RUN tokens
            const int32_t nextb = carries[1], tokb = carries[2], ob = carries[3];
            const uint64_t end = nextb == 0x7FFFFFFF ? L : (uint64_t)nextb;
            for (uint64_t i = ((t0 + C - 1) & ~(C - 1)) + (uint64_t)tid * C; i < t0 + tl; i += (uint64_t)kEncThreads * C) {
                IndexRec *r = idx + (i >> A.log2C);
                r->last_lit = fs;
                r->ocur = (uint32_t)ob;
                r->tok = (uint32_t)tokb;
                r->run_left = (uint32_t)(end - i);
            }
            if (t == A.ntiles - 1 && tid == 0) {
                A.ntok[pl] = (uint32_t)tokb;
                A.ocount[pl] = (uint32_t)ob;
            }
            return;
        }
    }
    uint64_t start[kPerThread], end[kPerThread];
    int32_t bases[2];
    element_runs(A, pl, t, t0, tl, start, end, sv, bases, carries);
    int cnt[kPerThread], tpos[kPerThread], isout[kPerThread], opos[kPerThread];
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        cnt[e] = 0;
        isout[e] = 0;
        if (k >= tl) continue;
        const uint64_t i = t0 + k;
        const uint32_t s = sv[e + 1];
        const uint64_t len = end[e] - start[e];
        const bool longrun = s != kOutlierSym && len >= kMinRunLen;
        cnt[e] = longrun ? (i == start[e] ? 2 : 0) : 1;
        isout[e] = s == kOutlierSym;
    }
    __syncthreads();
    int tile_tok, tile_out;
    ScanI(tmp).ExclusiveSum(cnt, tpos, tile_tok);
    if (A.t_nout[(uint64_t)pl * A.ntiles + t] != 0) { // (enc_verify's count: most tiles hold no outlier)
        __syncthreads();
        ScanI(tmp).ExclusiveSum(isout, opos, tile_out);
    } else {
        for (int e = 0; e < kPerThread; ++e) opos[e] = 0;
        tile_out = 0;
    }
    const uint32_t tokbase = (uint32_t)bases[0], obase = (uint32_t)bases[1];
    for (int e = 0; e < kPerThread; ++e) {
        const int k = tid * kPerThread + e;
        if (k >= tl) continue;
        const uint64_t i = t0 + k;
        const uint32_t s = sv[e + 1];
        const uint32_t tk = tokbase + (uint32_t)tpos[e];
        const uint64_t len = end[e] - start[e];
        const bool longrun = s != kOutlierSym && len >= kMinRunLen;
        if (cnt[e] == 2) {
            tsym[tk] = s;
            trep[tk] = 0;
            tsym[tk + 1] = rsym;
            trep[tk + 1] = (uint32_t)(len - 1);
        } else if (cnt[e] == 1) {
            tsym[tk] = s;
            trep[tk] = 0;
        }
        if (isout[e]) {
            A.opos[(uint64_t)pl * L + obase + opos[e]] = (uint32_t)i;
            A.oval[(uint64_t)pl * L + obase + opos[e]] = x[i];
        }
        if ((i & (C - 1)) == 0) {
            // decoder state at element i (codec.cpp:612-626)
            IndexRec *r = idx + (i >> A.log2C);
            const uint32_t ocur = obase + (uint32_t)opos[e];
            if (i == start[e]) {
                r->tok = tk;
                r->run_left = 0;
                r->last_lit = i == 0 ? rsym : sym[i - 1];
                r->ocur = ocur;
            } else {
                r->last_lit = s;
                r->ocur = ocur;
                if (longrun) {
                    // the run's literal + RUN tokens precede: resume after them
                    // (token index of the run start = tk since non-start
                    // elements of a long run emit nothing)
                    r->tok = tk;
                    r->run_left = (uint32_t)(end[e] - i);
                } else {
                    r->tok = tk;
                    r->run_left = 0;
                }
            }
        }
    }
    if (t == A.ntiles - 1 && tid == 0) { // plane totals: the last tile's offsets + its own counts
        A.ntok[pl] = tokbase + (uint32_t)tile_tok;
        A.ocount[pl] = obase + (uint32_t)tile_out;
    }
}
__global__ void __launch_bounds__(kEncThreads) tok_emit(TokArgs A, int planes) {
    pdl_begin();
    tok_emit_tile(A, planes, blockIdx.x);
}

} // namespace qcb
