// chain_scan.cuh -- block-parallel exact evaluation of the encoder's FP64
// chain d_k = RN(d_{k-1} + c_k) over a plane's events (codec.cpp:445; the
// decoder's codec.cpp:607 is the same recurrence).
//
// Why it can be parallel.  Write every chain value as an integer multiple of
// a power of two, d_k = K_k * 2^A_k.  A_k (the "alignment") is speculated per
// event by enc_lattice: A_k = max(ulp(d^_k), mu) where d^_k is the lattice
// estimate of d_k and mu = min(ulp(q), lowbit(segment base)).  Every c_k =
// RN(q*m) is a multiple of 2^ulp(q), so every d_k is a multiple of 2^mu, and
// the rounding of one step happens at 2^A_k.  A step K_{k-1} -> K_k is then
// an integer map that depends on K_{k-1} only through its low W bits:
//
//     K_k = floor(K_{k-1} / 2^W) * 2^E + T[K_{k-1} mod 2^W],
//     W = max(0, A_k + 1 - A_{k-1}),  E = W + A_{k-1} - A_k,
//     T[r] = RNE((r * 2^A_{k-1} + c_k) / 2^A_k).
//
// Maps of this shape are closed under composition (the composed W only
// grows with the net rise in magnitude), so a thread folds its events into
// one map (W <= kMaxW = 2: 4-entry tables), the block scans the maps, and each
// thread gets its exact start value.  Steps a map cannot express (a jump up
// by several binades, huge cancellations) "poison" their thread: a serial
// resolver pass computes those threads with plain FP64 once their start is
// known.  Finally every thread recomputes its own events with the real FP64
// additions from its start value, and adjacent threads compare end and start
// values: if all boundaries agree, every value is exact by induction.  A
// disagreement (a mis-speculated alignment) sends the rest of the plane to the
// serial warp chain.  The result is therefore bit-identical to the serial
// recurrence in every case; the speculation only decides the speed.
#pragma once

#include "align.cuh"
#include "enc_tiles.cuh"

namespace qcb {

// ------------------------------------------------------ integer maps
struct ChainFn {
    int W, E;          // K -> (K >> W) * 2^E + T[K & (2^W - 1)]
    long long T[kTab];
};
constexpr long long kTLimit = 1ll << 62;

// T[r] without dynamic register indexing (a select tree)
__device__ __forceinline__ long long fn_T(const ChainFn &F, int r) {
    long long v[kTab];
#pragma unroll
    for (int i = 0; i < kTab; ++i) v[i] = F.T[i];
#pragma unroll
    for (int bit = 0, w = kTab; w > 1; ++bit, w >>= 1) {
#pragma unroll
        for (int i = 0; i < w / 2; ++i) v[i] = ((r >> bit) & 1) ? v[2 * i + 1] : v[2 * i];
    }
    return v[0];
}
// Ring-exact (mod 2^64): correct whenever the true result fits in int64.
__device__ __forceinline__ long long fn_apply(const ChainFn &F, long long K) {
    const long long H = K >> F.W;
    return (long long)((unsigned long long)H << F.E) + fn_T(F, (int)(K & ((1 << F.W) - 1)));
}

// One chain step on an exact K (units 2^a) with addend c: RNE((K * 2^a + c)
// / 2^b), computed in units of 2^(b-2) with a sticky bit for the part of c
// below that.  int64 when the shifts are small (the common case), else
// int128.
struct StepC {
    int sa;          // a - (b - 2)
    int sc;          // ec - (b - 2) when >= 0
    long long Mc;    // c = Mc * 2^ec
    long long qc;    // floor(c / 2^(b-2)) when sc < 0
    bool sticky;     // c has bits below 2^(b-2)
    bool fast;
};
__device__ __forceinline__ StepC step_consts(int a, int b, double c) {
    StepC k;
    int ec;
    k.Mc = sig_of(c, ec);
    const int u = b - 2;
    k.sa = a - u;
    k.sc = ec - u;
    k.sticky = false;
    k.qc = 0;
    if (k.sc < 0) {
        const int sh = -k.sc;
        if (sh >= 62) {
            k.qc = k.Mc < 0 ? -1 : 0;
            k.sticky = k.Mc != 0;
        } else {
            k.qc = k.Mc >> sh;
            k.sticky = (k.Mc - k.qc * (1ll << sh)) != 0;
        }
    }
    k.fast = k.sa >= 0 && k.sa <= 8 && k.sc <= 8;
    return k;
}
__device__ __forceinline__ bool step_eval(const StepC &k, long long K, long long &out) {
    if (k.fast && K < (1ll << 54) && K > -(1ll << 54)) {
        const long long N = K * (1ll << k.sa) + (k.sc >= 0 ? k.Mc * (1ll << k.sc) : k.qc);
        long long R = N >> 2;
        const int rm = (int)(N & 3);
        if (rm == 3 || (rm == 2 && (k.sticky || (R & 1)))) R += 1;
        out = R;
        return true;
    }
    if (k.sa < 0 || k.sa > 70 || k.sc > 70) return false;
    __int128 N = (__int128)K << k.sa;
    N += k.sc >= 0 ? ((__int128)k.Mc << k.sc) : (__int128)k.qc;
    __int128 R = N >> 2;
    const int rm = (int)(N & 3);
    if (rm == 3 || (rm == 2 && (k.sticky || (R & 1)))) R += 1;
    if (R >= (__int128)kTLimit || R <= -(__int128)kTLimit) return false;
    out = (long long)R;
    return true;
}

// F <- (step a->b with addend c) o F, on deviations: F maps the deviation
// entering the thread to the deviation from reference khp (units 2^a); the
// result maps it to the deviation from kh (units 2^b).  Adding m * 2^W_G to
// K adds m * 2^E_G to the step's result, so after widening F until its high
// part moves in whole multiples of 2^W_G, every residue class is the step
// evaluated on one representative K.
__device__ __forceinline__ bool compose_step(ChainFn &F, int a, long long khp, int b, long long kh, double c) {
    int WG = b + 1 - a;
    if (WG < 0) WG = 0;
    if (WG > kMaxW) return false;
    const int EG = WG + a - b;
    if (EG > 62) return false;
    if (F.E < WG) {
        const int d = WG - F.E;
        const int nw = F.W + d;
        if (nw > kMaxW) return false;
        long long T[kTab];
#pragma unroll
        for (int r = 0; r < kTab; ++r)
            T[r] = r < (1 << nw) ? fn_T(F, r & ((1 << F.W) - 1)) + (long long)(r >> F.W) * (1ll << F.E) : 0;
#pragma unroll
        for (int r = 0; r < kTab; ++r) F.T[r] = T[r];
        F.W = nw;
        F.E = WG;
    }
    const StepC k = step_consts(a, b, c);
#pragma unroll
    for (int r = 0; r < kTab; ++r) {
        if (r >= (1 << F.W)) break;
        long long R;
        if (!step_eval(k, khp + F.T[r], R)) return false;
        R -= kh;
        if (R >= kTLimit || R <= -kTLimit) return false;
        F.T[r] = R;
    }
    F.E = F.E - WG + EG;
    return F.E <= 62;
}

// F <- G o F
__device__ __forceinline__ bool fn_compose(const ChainFn &G, ChainFn &F) {
    if (F.E < G.W) { // widen F so that its high part carries whole G-inputs
        const int d = G.W - F.E;
        const int nw = F.W + d;
        if (nw > kMaxW) return false;
        long long T[kTab];
#pragma unroll
        for (int r = 0; r < kTab; ++r)
            T[r] = r < (1 << nw) ? fn_T(F, r & ((1 << F.W) - 1)) + (long long)(r >> F.W) * (1ll << F.E) : 0;
#pragma unroll
        for (int r = 0; r < kTab; ++r) F.T[r] = T[r];
        F.W = nw;
        F.E = G.W;
    }
    const long long mask = (1ll << G.W) - 1;
#pragma unroll
    for (int r = 0; r < kTab; ++r) {
        if (r >= (1 << F.W)) continue;
        const long long v = F.T[r];
        const long long hi = v >> G.W;
        const long long top = G.E >= 62 ? hi : (hi >> (62 - G.E));
        if (top != 0 && top != -1) return false;
        const long long t = (long long)((unsigned long long)hi << G.E) + fn_T(G, (int)(v & mask));
        if (t >= kTLimit || t <= -kTLimit) return false;
        F.T[r] = t;
    }
    F.E = F.E - G.W + G.E;
    return F.E <= 62;
}

// ------------------------------------------------------ alignment maps
// A_k = max(ulp(d^_k), min(A_{k-1}, ulp(c_k))) is a lower bound on the
// alignment of d_k (c_k is a multiple of 2^ulp(c_k), the exact sum of two
// multiples of 2^m is one, and rounding to 2^ulp(d_k) keeps it).  Each step
// is a clamp a -> min(max(a, lo), hi); clamps compose, so the A_k of a chunk
// come from one block scan.  An outlier resets A to lowbit(x).
constexpr int kAInf = 30000;
struct Clamp {
    int lo, hi;
};
__device__ __forceinline__ int clamp_apply(Clamp f, int a) { return min(max(a, f.lo), f.hi); }
__device__ __forceinline__ Clamp clamp_then(Clamp f, Clamp g) { // g o f
    return Clamp{clamp_apply(g, f.lo), clamp_apply(g, f.hi)};
}
__device__ __forceinline__ Clamp event_clamp(bool outlier, double c, double dh, int uq) {
    if (outlier) {
        const int a = c == 0.0 ? uq : low_bit(c);
        return Clamp{a, a};
    }
    const int g = ulp_exp(dh);
    const int u = c == 0.0 ? kAInf : ulp_exp(c);
    return g <= u ? Clamp{g, u} : Clamp{g, g};
}

// ------------------------------------------------------ the kernel
#ifndef QCSIM_CS_THREADS
#define QCSIM_CS_THREADS 256
#endif
constexpr int kCsThreads = QCSIM_CS_THREADS;        // (512, i.e. 8192-event chunks, measured slower: 39.3 vs 37.2 ms)
constexpr int kCsEpt = 16;                        // events per thread
constexpr int kCsChunk = kCsThreads * kCsEpt;     // events per block pass
constexpr int kCsPad = kCsEpt + 1;                // bank-conflict-free rows
constexpr int kCsWarps = kCsThreads / 32;
constexpr uint32_t kCsSerialMax = 256;            // planes with fewer events run serially
constexpr int kCsResolveMax = 48 * kCsThreads / 256; // more resolve points: the chunk runs serially

struct ChainElem {
    int kind; // 0 map of the chunk carry, 1 constant (T[0] = delta), 2 map of resolved thread `base`
    int base;
    ChainFn f;
};
#ifndef QCSIM_CS_WARPSCAN
#define QCSIM_CS_WARPSCAN 0  // warp-shuffle map scan: correct, measured slower (38.9 vs 37.2 ms per 500 passes)
#endif
__device__ __forceinline__ long long shfl_up_ll(long long v, int off) {
    const int lo = __shfl_up_sync(0xffffffffu, (int)(v & 0xffffffff), off);
    const int hi = __shfl_up_sync(0xffffffffu, (int)(v >> 32), off);
    return (long long)(((unsigned long long)(unsigned)hi << 32) | (unsigned)lo);
}
__device__ __forceinline__ ChainElem shfl_up_elem(const ChainElem &x, int off) {
    ChainElem p;
    p.kind = __shfl_up_sync(0xffffffffu, x.kind, off);
    p.base = __shfl_up_sync(0xffffffffu, x.base, off);
    p.f.W = __shfl_up_sync(0xffffffffu, x.f.W, off);
    p.f.E = __shfl_up_sync(0xffffffffu, x.f.E, off);
#pragma unroll
    for (int r = 0; r < kTab; ++r) p.f.T[r] = shfl_up_ll(x.f.T[r], off);
    return p;
}
struct ChainScanSmem {
    double c[kCsThreads * kCsPad];     // addend / outlier value, then the chain value
    long long kh[kCsThreads * kCsPad]; // lattice estimate of d, then the reference K
    ChainElem el[kCsThreads];
    long long resd[kCsThreads];        // resolved delta at the end of a resolve point
    double dend[kCsThreads];
    int16_t A[kCsThreads * kCsPad];
    uint8_t out[kCsThreads * kCsPad];
    Clamp wclamp[kCsWarps];
    ChainElem wagg[kCsWarps];          // warp aggregates of the map scan
    uint32_t pmask[kCsWarps];          // resolve points
    int fail;
    int firstbad;
    int tent;                          // a tentative last value was published
};
constexpr size_t kChainScanSmem = sizeof(ChainScanSmem);

// Serial chain for one warp over events [from, to) (same recurrence, same
// order); returns the last value on every lane.  Outlier-free batches of 32
// use the per-lane prefix form of enc_chain: lane j runs the same chain and
// stops adding after event j, so only the DADD latency is serial.
struct IdentitySlot {
    __device__ uint64_t operator()(uint32_t ord) const { return ord; }
};
template <class Slot = IdentitySlot>
__device__ double chain_serial_warp(const double *evc, const uint32_t *ev, double *dv, uint32_t from, uint32_t to,
                                    double d, int lane, Slot slot = Slot()) {
    for (uint32_t base = from; base < to; base += 32) {
        const uint32_t cnt = tmin<uint32_t>(32, to - base);
        const uint64_t g = lane < (int)cnt ? slot(base + lane) : 0;
        const double cl = lane < (int)cnt ? evc[g] : 0.0;
        const uint32_t o = lane < (int)cnt ? ev[g] >> 31 : 0u;
        const unsigned om = __ballot_sync(0xffffffffu, o != 0);
        double mine = 0.0;
        if (om == 0 && cnt == 32) {
            double dl = d;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const double cj = __shfl_sync(0xffffffffu, cl, j);
                if (j <= lane) dl = dadd(dl, cj);
            }
            mine = dl;
            d = __shfl_sync(0xffffffffu, dl, 31);
        } else {
            for (uint32_t j = 0; j < cnt; ++j) {
                const double cj = __shfl_sync(0xffffffffu, cl, j);
                d = ((om >> j) & 1) ? cj : dadd(d, cj);
                if (lane == (int)j) mine = d;
            }
        }
        if (lane < (int)cnt) dv[base + lane] = mine;
    }
    return d;
}

// The same for a chunk already staged in shared memory (slot layout of
// ChainScanSmem): events [0, n) of the chunk, values written to dv[0, n).
template <class Smem>
__device__ double chain_serial_smem(const Smem &S, double *dv, int n, double d, int lane) {
    for (int base = 0; base < n; base += 32) {
        const int cnt = min(32, n - base);
        const int j = base + lane;
        const int sj = (j / kCsEpt) * kCsPad + (j % kCsEpt);
        const bool o = lane < cnt && S.out[sj];
        const unsigned om = __ballot_sync(0xffffffffu, o);
        double mine = 0.0;
        if (om == 0 && cnt == 32) {
            double dl = d;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int b = base + k;
                const double ck = S.c[(b / kCsEpt) * kCsPad + (b % kCsEpt)];
                if (k <= lane) dl = dadd(dl, ck);
            }
            mine = dl;
            d = __shfl_sync(0xffffffffu, dl, 31);
        } else {
            for (int k = 0; k < cnt; ++k) {
                const int b = base + k;
                const double ck = S.c[(b / kCsEpt) * kCsPad + (b % kCsEpt)];
                d = ((om >> k) & 1) ? ck : dadd(d, ck);
                if (lane == k) mine = d;
            }
        }
        if (lane < cnt) dv[j] = mine;
    }
    return d;
}

// d = (kh + delta) * 2^A
__device__ __forceinline__ bool delta_to_d(long long kh, long long delta, int A, double &d) {
    return k_to_d(kh + delta, A, d);
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Chunk-to-chunk hand-off of the exact chain value (decoupled look-back):
// chunk k of a plane publishes its last value and raises its flag to the
// launch's epoch; chunk k+1 does all of its map building first and only then
// waits.  Blocks are numbered chunk-major (block = chunk * planes + plane), so
// a waiter's predecessor always has a smaller block index (dispatched
// earlier) and the resident blocks advance every plane's chain at once.
struct ChainLink {
    double *carry;   // [plane][cmax] exact last value of a chunk ...
    uint32_t *flag;  // [plane][cmax] ... released when it is final (epoch)
    double *tcarry;  // [plane][cmax] tentative last value (from the maps, before the
    uint32_t *tflag; //   chunk's own verification): the successor starts on it
    int cmax;        // chunks per plane in the grid
    uint32_t epoch;  // this launch's flag value
    unsigned long long *trace; // debug: per block 8 phase times (%globaltimer ns), see CS_TRACE
    // per-plane completion for the consumer grid (enc_verify runs alongside,
    // waiting per plane instead of for the whole grid): every block of plane
    // p counts itself in cnt[p]; the last one resets it and raises done[p]
    // to the epoch (nullptr: the consumer waits for the grid)
    uint32_t *cnt;
    uint32_t *done;
};
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// phases: 0 start, 4 loaded, 5 alignments, 6 folded, 1 maps scanned,
// 2 carry in, 3 end
#define CS_TRACE(k) \
    if (link.trace && threadIdx.x == 0) link.trace[8ull * blockIdx.x + (k)] = gtimer()

#define CS_FAIL(code) atomicOr(&S.fail, 1 << (code))
__device__ __forceinline__ void chain_chunk(const TileArgs &A, int planes, const ChainLink &link, uint32_t *stats,
                                            int debug) {
    const int pl = blockIdx.x % planes, ck = blockIdx.x / planes; // chunk-major: every plane's chain advances
    const PlaneParams pp = block_params(A.params, pl);
    if ((pp.flags & kFlagFallback) || pp.eb == 0.0) return;
    const uint64_t L = A.L;
    const uint32_t nev = (uint32_t)carry_of(reinterpret_cast<const int32_t *>(A.t_evoff), A.ntiles + 1,
                                            reinterpret_cast<const int32_t *>(A.t_nev), pl, A.ntiles, A.ntiles,
                                            kScanSumExcl);
    const uint32_t c0 = (uint32_t)ck * kCsChunk;
    if (c0 >= nev) return;
    if (ck == 0 && threadIdx.x == 0 && stats) // events of the pass (bench roofline)
        atomicAdd(reinterpret_cast<unsigned long long *>(stats + 6), (unsigned long long)nev);

    extern __shared__ __align__(16) unsigned char cs_raw[];
    ChainScanSmem &S = *reinterpret_cast<ChainScanSmem *>(cs_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    CS_TRACE(0);
    const uint32_t *ev = A.evlist + (uint64_t)pl * L;
    const double *evc = A.evc + (uint64_t)pl * L;
    const double *evD = A.evD + (uint64_t)pl * L;
    double *dv = A.dval + (uint64_t)pl * L;
    const int uq = ulp_exp(pp.q);
    const int n = (int)tmin<uint32_t>(kCsChunk, nev - c0);
    const int nthr = (n + kCsEpt - 1) / kCsEpt;
    // event ordinal -> record slot (tile-local records, enc_lattice)
    __shared__ uint32_t s_tpre[kInlineTiles + 1];
    if (A.ev_tile_local && tid < 32) {
        const int32_t *tn = reinterpret_cast<const int32_t *>(A.t_nev) + (uint64_t)pl * A.ntiles;
        uint32_t carry = 0;
        for (int b0 = 0; b0 < A.ntiles; b0 += 32) {
            const uint32_t v = b0 + tid < A.ntiles ? (uint32_t)tn[b0 + tid] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (tid >= off) incl += o;
            }
            if (b0 + tid < A.ntiles) s_tpre[b0 + tid] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (tid == 0) s_tpre[A.ntiles] = carry;
    }
    __syncthreads();
    auto slot_of = [&](uint32_t ord) -> uint64_t {
        if (!A.ev_tile_local) return ord;
        int lo = 0, hi = A.ntiles; // last tile with prefix <= ord
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_tpre[mid] <= ord) lo = mid;
            else hi = mid;
        }
        return (uint64_t)lo * kTile + (ord - s_tpre[lo]);
    };
    if (nev <= kCsSerialMax) { // a handful of events: the plain recurrence is cheaper
        if (threadIdx.x < 32) chain_serial_warp(evc, ev, dv, 0, nev, 0.0, threadIdx.x, slot_of);
        return;
    }

    if (tid == 0) {
        S.fail = 0;
        S.firstbad = kCsThreads;
    }
    if (tid < kCsWarps) S.pmask[tid] = tid == 0 ? 1u : 0u; // thread 0 starts from the carry
    CS_TRACE(7);
    {
        // ordinals rise by kCsThreads per iteration: walk the tile prefix forward
        int tile = 0;
        if (A.ev_tile_local) {
            int lo = 0, hi = A.ntiles;
            const uint32_t o0 = c0 + tid;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_tpre[mid] <= o0) lo = mid;
                else hi = mid;
            }
            tile = lo;
        }
        // slots first, then every load in flight at once, then the stores
        uint64_t g[kCsEpt];
#pragma unroll
        for (int i = 0; i < kCsEpt; ++i) {
            const int j = tid + i * kCsThreads;
            g[i] = c0 + j;
            if (A.ev_tile_local && j < n) {
                while (tile + 1 < A.ntiles && s_tpre[tile + 1] <= c0 + j) ++tile;
                g[i] = (uint64_t)tile * kTile + (c0 + j - s_tpre[tile]);
            }
        }
        double cv[kCsEpt];
        long long dv2[kCsEpt];
        uint32_t evv[kCsEpt];
#pragma unroll
        for (int i = 0; i < kCsEpt; ++i) {
            const int j = tid + i * kCsThreads;
            if (j < n) {
                cv[i] = __ldg(evc + g[i]);
                dv2[i] = __double_as_longlong(__ldg(evD + g[i]));
                evv[i] = __ldg(ev + g[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < kCsEpt; ++i) {
            const int j = tid + i * kCsThreads;
            if (j < n) {
                const int s = (j / kCsEpt) * kCsPad + (j % kCsEpt);
                S.c[s] = cv[i];
                S.kh[s] = dv2[i];
                S.out[s] = (uint8_t)(evv[i] >> 31);
            }
        }
    }
    __syncthreads();

    CS_TRACE(4);
    // ---- alignments: clamp scan from the weakest claim about the carry
    const int k0 = tid * kCsEpt;
    const int cnt = max(0, min(kCsEpt, n - k0));
    Clamp cf{-kAInf, kAInf};
    for (int k = 0; k < cnt; ++k) {
        const int s = tid * kCsPad + k;
        cf = clamp_then(cf, event_clamp(S.out[s], S.c[s], __longlong_as_double(S.kh[s]), uq));
    }
    Clamp inc = cf; // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int lo = __shfl_up_sync(0xffffffffu, inc.lo, off), hi = __shfl_up_sync(0xffffffffu, inc.hi, off);
        if (lane >= off) inc = clamp_then(Clamp{lo, hi}, inc);
    }
    if (lane == 31) S.wclamp[warp] = inc;
    __syncthreads();
    {
        Clamp pre{-kAInf, kAInf};
        for (int w = 0; w < warp; ++w) pre = clamp_then(pre, S.wclamp[w]);
        Clamp ex{__shfl_up_sync(0xffffffffu, inc.lo, 1), __shfl_up_sync(0xffffffffu, inc.hi, 1)};
        if (lane > 0) pre = clamp_then(pre, ex);
        int a = clamp_apply(pre, -1074); // every double is a multiple of 2^-1074
        for (int k = 0; k < cnt; ++k) {
            const int s = tid * kCsPad + k;
            const double dh = __longlong_as_double(S.kh[s]);
            a = clamp_apply(event_clamp(S.out[s], S.c[s], dh, uq), a);
            S.A[s] = (int16_t)a;
            S.kh[s] = S.out[s] ? ref_k(S.c[s], a) : ref_k(dh, a);
        }
    }
    __syncthreads();

    CS_TRACE(5);
    // ---- fold my events into one map on deviations (thread 0 is resolved
    // from the carry instead)
    const int lsl = (tid - 1) * kCsPad + kCsEpt - 1; // left neighbour's last slot
    const int a_in = tid == 0 ? 0 : S.A[lsl];
    const long long kh_in = tid == 0 ? 0 : S.kh[lsl];
    ChainFn F;
    F.W = 0;
    F.E = 0;
#pragma unroll
    for (int r = 0; r < kTab; ++r) F.T[r] = 0;
    bool known = false, poison = tid == 0;
    double val = 0.0;
    int a = a_in;
    long long kp = kh_in;
    for (int k = 0; k < cnt; ++k) {
        const int s = tid * kCsPad + k;
        const double c = S.c[s];
        const int b = S.A[s];
        const long long kb = S.kh[s];
        if (S.out[s]) {
            known = true;
            poison = false;
            val = c;
        } else if (known) {
            val = dadd(val, c);
        } else if (!poison) {
            if (!compose_step(F, a, kp, b, kb, c)) poison = true;
        }
        a = b;
        kp = kb;
    }
    ChainElem e;
    e.base = tid;
    e.f = F;
    e.kind = 0;
    if (tid == 0 || (cnt > 0 && poison && !known)) {
        e.kind = 2; // identity after my own (resolved) end
        e.f.W = 0;
        e.f.E = 0;
        e.f.T[0] = 0;
    } else if (cnt > 0 && known) {
        long long K = 0;
        if (!d_to_k(val, a, K)) CS_FAIL(1);
        e.kind = 1;
        e.f.T[0] = K - kp;
    }
    S.el[tid] = e;
    const unsigned pm = __ballot_sync(0xffffffffu, cnt > 0 && !known && poison);
    if (lane == 0 && pm) atomicOr(&S.pmask[warp], pm);
    __syncthreads();

    CS_TRACE(6);
    if (debug && stats && cnt > 0) atomicAdd(&stats[8 + min(e.kind == 0 ? e.f.W : 4 + e.kind, 7)], 1u); // W histogram
    int npts = 0;
#pragma unroll
    for (int w = 0; w < kCsWarps; ++w) npts += __popc(S.pmask[w]);
    const bool serial_chunk = npts > kCsResolveMax; // the maps do not fit this stretch

    // ---- inclusive segmented scan of the maps.  A composition that does not
    // fit turns the left range's last thread into a resolve point.
#if QCSIM_CS_WARPSCAN
    // Warp level by shuffles (5 steps, no block barrier), then the warp
    // aggregates (3 steps in warp 0), then one composition per thread with
    // its warp's exclusive prefix.
    if (!serial_chunk) {
        auto combine = [&](ChainElem &x, const ChainElem &p, int pt) { // x <- x o p (x.kind == 0)
            if (p.kind == 1) {
                x.kind = 1;
                x.f.T[0] = fn_apply(x.f, p.f.T[0]);
            } else {
                ChainFn g = p.f;
                if (fn_compose(x.f, g)) {
                    x.f = g;
                    x.kind = p.kind;
                    x.base = p.base;
                } else {
                    x.kind = 2;
                    x.base = pt;
                    atomicOr(&S.pmask[pt >> 5], 1u << (pt & 31));
                }
            }
        };
        ChainElem x = e;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const ChainElem p = shfl_up_elem(x, off);
            if (lane >= off && tid < nthr && x.kind == 0) combine(x, p, tid - off);
        }
        if (lane == 31) S.wagg[warp] = x;
        __syncthreads();
        if (warp == 0) { // inclusive scan over the warp aggregates (lanes < kCsWarps)
            ChainElem y = lane < kCsWarps ? S.wagg[lane] : ChainElem{};
#pragma unroll
            for (int off = 1; off < kCsWarps; off <<= 1) {
                const ChainElem p = shfl_up_elem(y, off);
                if (lane >= off && lane < kCsWarps && y.kind == 0) combine(y, p, 32 * (lane - off) + 31);
            }
            if (lane < kCsWarps) S.wagg[lane] = y;
        }
        __syncthreads();
        if (warp > 0 && tid < nthr && x.kind == 0) combine(x, S.wagg[warp - 1], 32 * warp - 1);
        S.el[tid] = x;
        __syncthreads();
    }
#else
    for (int off = 1; off < (serial_chunk ? 1 : nthr); off <<= 1) {
        ChainElem x = S.el[tid];
        const int pt = tid - off;
        const bool act = tid >= off && tid < nthr && x.kind == 0;
        ChainElem p;
        if (act) p = S.el[pt];
        __syncthreads();
        if (act) {
            if (p.kind == 1) {
                x.kind = 1;
                x.f.T[0] = fn_apply(x.f, p.f.T[0]);
            } else {
                ChainFn g = p.f;
                if (fn_compose(x.f, g)) {
                    x.f = g;
                    x.kind = p.kind;
                    x.base = p.base;
                } else {
                    x.kind = 2;
                    x.base = pt;
                    atomicOr(&S.pmask[pt >> 5], 1u << (pt & 31));
                }
            }
        }
        S.el[tid] = x;
        __syncthreads();
    }
#endif
    const ChainElem *P = S.el;
    auto delta_before = [&](int t) -> long long { // deviation entering thread t >= 1
        const ChainElem &q = P[t - 1];
        if (q.kind == 1) return q.f.T[0];
        return fn_apply(q.f, S.resd[q.base]);
    };

    // ---- the exact value before this chunk
    CS_TRACE(1);
    // (the map path starts on the predecessor's tentative value and checks
    // it against the final one before publishing its own final value; a
    // serial chunk waits for the final value)
    const uint64_t lk = (uint64_t)pl * link.cmax + ck;
    if (tid == 0) {
        double cd = 0.0;
        if (ck > 0) {
            const uint32_t *fp = (serial_chunk ? link.flag : link.tflag) + lk - 1;
            while (ld_acquire(fp) != link.epoch) {
            }
            cd = serial_chunk ? link.carry[lk - 1] : link.tcarry[lk - 1];
        }
        S.dend[kCsThreads - 1] = cd; // parked until the final pass overwrites it
    }
    __syncthreads();
    const double carry_d = S.dend[kCsThreads - 1];
    CS_TRACE(2);

    if (serial_chunk) {
        if (tid < 32) {
            const double d = chain_serial_smem(S, dv + c0, n, carry_d, tid);
            if (tid == 0) {
                if (c0 + n < nev) {
                    link.carry[lk] = d;
                    link.tcarry[lk] = d;
                    st_release(link.flag + lk, link.epoch);
                    st_release(link.tflag + lk, link.epoch);
                }
                if (stats) atomicAdd(&stats[4], 1u);
            }
        }
        return;
    }

    // ---- serial resolver over the resolve points (in order)
    uint32_t nresolve = 0;
    if (tid == 0) {
        for (int w = 0; w < kCsWarps; ++w) {
            unsigned m = S.pmask[w];
            while (m) {
                const int p = w * 32 + __ffs(m) - 1;
                m &= m - 1;
                if (p >= nthr) break;
                ++nresolve;
                double d = carry_d;
                if (p > 0) {
                    const int pls = (p - 1) * kCsPad + kCsEpt - 1;
                    if (!delta_to_d(S.kh[pls], delta_before(p), S.A[pls], d)) CS_FAIL(3);
                }
                const int cp = min(kCsEpt, n - p * kCsEpt);
                for (int k = 0; k < cp; ++k) {
                    const int s = p * kCsPad + k;
                    d = S.out[s] ? S.c[s] : dadd(d, S.c[s]);
                }
                const int ls = p * kCsPad + cp - 1;
                long long K = 0;
                if (!d_to_k(d, S.A[ls], K)) CS_FAIL(4);
                S.resd[p] = K - S.kh[ls];
            }
        }
        // tentative last value from the maps: the successor starts on it
        // while this chunk verifies itself
        if (c0 + n < nev) {
            const int lls = (nthr - 1) * kCsPad + (n - (nthr - 1) * kCsEpt) - 1;
            double dt = 0.0;
            if (S.fail == 0 && delta_to_d(S.kh[lls], delta_before(nthr), S.A[lls], dt)) {
                link.tcarry[lk] = dt;
                st_release(link.tflag + lk, link.epoch);
                S.tent = 1;
            } else {
                S.tent = 0;
            }
        }
    }
    __syncthreads();

    // ---- every thread: exact FP64 recomputation from its start value
    double dstart = 0.0;
    if (cnt > 0) {
        if (tid == 0) dstart = carry_d;
        else if (!delta_to_d(kh_in, delta_before(tid), a_in, dstart)) CS_FAIL(5);
        double d = dstart;
        for (int k = 0; k < cnt; ++k) {
            const int s = tid * kCsPad + k;
            d = S.out[s] ? S.c[s] : dadd(d, S.c[s]);
            S.c[s] = d;
        }
        S.dend[tid] = d;
    }
    __syncthreads();
    // boundaries: my start must equal my left neighbour's end (== so that
    // -0.0 / +0.0 agree: the next addend is never -0.0)
    if (cnt > 0 && tid > 0 && !(dstart == S.dend[tid - 1])) {
        CS_FAIL(6);
        if (debug) atomicMin(&S.firstbad, tid);
    }
    if (debug) {
        __syncthreads();
        if (tid == S.firstbad && atomicAdd(&stats[2], 1u) < 3) {
            const ChainElem &q = P[tid - 1];
            printf("chain_scan: plane %d chunk %u thread %d start %.17g left end %.17g | kind %d base %d W %d E %d "
                   "T %lld %lld | a_in %d kh_in %lld resd[base] %lld fail %x\n",
                   pl, c0, tid, dstart, S.dend[tid - 1], q.kind, q.base, q.f.W, q.f.E, q.f.T[0], q.f.T[1], a_in,
                   kh_in, q.kind == 2 ? S.resd[q.base] : -1ll, S.fail);
        }
    }
    // the carry this chunk started from must be the predecessor's final value
    if (tid == 0 && ck > 0) {
        const uint32_t *fp = link.flag + lk - 1;
        while (ld_acquire(fp) != link.epoch) {
        }
        const double fin = link.carry[lk - 1];
        if (bits_of(fin) != bits_of(carry_d)) {
            CS_FAIL(7);
            S.dend[kCsThreads - 1] = fin; // (read back below as the redo's start)
        }
    }
    __syncthreads();
    const bool failed = S.fail != 0;
    const double carry_fin = (failed && ck > 0 && (S.fail & (1 << 7))) ? S.dend[kCsThreads - 1] : carry_d;
    // publish the exact last value for the next chunk first (its hand-off is
    // the critical path), then store this chunk's values
    if (!failed && tid == 0 && c0 + n < nev) {
        link.carry[lk] = S.dend[nthr - 1];
        st_release(link.flag + lk, link.epoch);
        if (!S.tent) { // nothing tentative went out: the final value serves both
            link.tcarry[lk] = S.dend[nthr - 1];
            st_release(link.tflag + lk, link.epoch);
        }
    }
    if (!failed) {
        for (int j = tid; j < n; j += kCsThreads) dv[c0 + j] = S.c[(j / kCsEpt) * kCsPad + (j % kCsEpt)];
    } else if (tid < 32) { // redo this chunk with the serial recurrence
        if (debug && tid == 0 && atomicAdd(&stats[3], 1u) < 16)
            printf("chain_scan: plane %d chunk %u fail mask %x\n", pl, c0, S.fail);
        const double d = chain_serial_warp(evc, ev, dv, c0, c0 + n, carry_fin, tid, slot_of);
        if (tid == 0) S.dend[nthr - 1] = d;
    }
    if (tid == 0) {
        if (failed && c0 + n < nev) {
            link.carry[lk] = S.dend[nthr - 1];
            st_release(link.flag + lk, link.epoch);
            if (!S.tent) {
                link.tcarry[lk] = S.dend[nthr - 1];
                st_release(link.tflag + lk, link.epoch);
            }
        }
        CS_TRACE(3);
        if (stats) {
            atomicAdd(&stats[0], nresolve);
            if (failed) atomicAdd(&stats[1], 1u);
        }
    }
}
__global__ void __launch_bounds__(kCsThreads, kCsThreads * kCsEpt > 4096 ? 1 : 2) enc_chain_scan(TileArgs A, int planes, ChainLink link, uint32_t *stats,
                                                                int debug) {
    pdl_begin();
    chain_chunk(A, planes, link, stats, debug);
    if (!link.done) return;
    __syncthreads(); // every chain value of this block is written
    if (threadIdx.x == 0) {
        const int pl = blockIdx.x % planes;
        __threadfence();
        const uint32_t old = atomicAdd(link.cnt + pl, 1u);
        if (old + 1 == (uint32_t)link.cmax) { // the plane's last block
            link.cnt[pl] = 0u;
            __threadfence(); // acquire the other blocks' counts (and their values)
            st_release(link.done + pl, link.epoch);
        }
    }
}
#undef CS_FAIL
#undef CS_TRACE
} // namespace qcb
