// encode_kernels.cuh -- QCB1 encoder kernels (compress_plane, codec.cpp:410-533).
//
// Pipeline per batch of planes:
//   E1  enc_quantize   speculative closed-loop quantization, one block per
//                      unit (1 plane, or a slice = re+im planes), streaming
//                      1024-element tiles in index order:
//                        spec   lattice decisions m^ in parallel
//                        chain  one thread: exact d += RN(q*m^) over the
//                               nonzero codes only (the serial floor)
//                        verify every decision re-evaluated in parallel with
//                               the exact prediction; any mismatch sends the
//                               plane to E1f
//   E1f enc_serial     exact serial closed loop (codec.cpp:430-458), one
//                      thread per refuted / linear-predictor plane
//   E2  enc_tokenize   run collapse (codec.cpp:460-482) + histogram, fully
//                      parallel per tile (runs carried across tiles)
//   E3  enc_codebook   two-queue Huffman + canonical codes (codec.cpp:160-249)
//   E5  enc_pack       header, table, MSB-first stream, outliers, index
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace qcb {

// ------------------------------------------------------------ arguments
struct EncPlanes {
    PlaneParams *params;       // [plane] eb/q/flags (flags written by E1)
    uint32_t *sym;             // [plane][L] exact symbols
    uint32_t *opos;            // [plane][L] outlier positions (compact)
    double *oval;              // [plane][L] outlier values
    uint32_t *ocount;          // [plane] outliers
    IndexRec *index;           // [plane][nidx]
    double *tilesum;           // [unit][ntiles] sq-norm tree partials (engine)
    uint64_t L;
    int log2C;                 // checkpoint every 2^log2C elements
    int qb;
    int predictor;
};

// Source of plane values: raw planes (codec mode).
struct RawSrc {
    const double *const *x;    // per plane
    __device__ __forceinline__ void load(int unit, uint64_t i, double *v) const { v[0] = x[unit][i]; }
    static constexpr bool kNorms = false;
};

// Source of plane values: the engine's gate pass.  New
// amplitude of global index g = action applied to the scaled old values.
struct GateSrc {
    const double *old;          // dense old planes, [slot][re|im][L]
    const int32_t *slot_of;     // global slice -> slot in `old`
    const uint64_t *unit_slice; // unit -> global slice
    const double *scale;        // device scalar 1/sqrt(G); nullptr = none
    DevAction act;
    int s;
    uint64_t L;
    static constexpr bool kNorms = true;

    __device__ __forceinline__ void fetch(uint64_t g, double sc, bool apply, double &re, double &im) const {
        const int32_t slot = slot_of[g >> s];
        const uint64_t off = g & (L - 1);
        const double *p = old + (uint64_t)slot * 2 * L;
        re = p[off];
        im = p[L + off];
        if (apply) {
            re = dmul(re, sc);
            im = dmul(im, sc);
        }
    }
    __device__ __forceinline__ void load(int unit, uint64_t i, double *v) const {
        const uint64_t g = (unit_slice[unit] << s) | i;
        const bool apply = scale != nullptr;
        const double sc = apply ? *scale : 1.0;
        if (act.kind == 0) {
            double r, m;
            fetch(g, sc, apply, r, m);
            if ((g & act.mask) == act.mask) cmul(act.f[0], act.f[1], r, m, v[0], v[1]);
            else { v[0] = r; v[1] = m; }
        } else if (act.kind == 1) {
            if ((g & act.mask) != act.mask) { fetch(g, sc, apply, v[0], v[1]); return; }
            const uint64_t tb = 1ull << act.target;
            double v0r, v0i, v1r, v1i, p0r, p0i, p1r, p1i;
            fetch(g & ~tb, sc, apply, v0r, v0i);
            fetch(g | tb, sc, apply, v1r, v1i);
            const double *u = (g & tb) ? act.u + 4 : act.u;
            cmul(u[0], u[1], v0r, v0i, p0r, p0i);
            cmul(u[2], u[3], v1r, v1i, p1r, p1i);
            v[0] = dadd(p0r, p1r);
            v[1] = dadd(p0i, p1i);
        } else {
            const uint64_t ba = (g >> act.a) & 1, bb = (g >> act.b) & 1;
            const uint64_t src = ba != bb ? g ^ ((1ull << act.a) | (1ull << act.b)) : g;
            fetch(src, sc, apply, v[0], v[1]);
        }
    }
};

// ------------------------------------------------------------ E1 smem
template <int NP> struct E1Smem {
    double x[NP][kTile];
    double c[NP][kTile];       // q*m^ (x for outliers); reused for final d
    double d[NP][kTile];       // chain values at events
    uint32_t ssym[NP][kTile];  // speculated symbol
    uint16_t ev[NP][kTile];    // compact event list
    uint8_t fl[NP][kTile];     // bit0 event, bit1 outlier
    long long kb[NP][kEncThreads]; // K of each thread's last element
    double red[kEncThreads];
    // carry (per plane)
    double dlast[NP], d2last[NP], xlast[NP], x2last[NP], base[NP];
    long long klast[NP];
    uint32_t ocount[NP];
    int nev[NP];
    int fail[NP];
    int prevout[NP];  // last element of the previous tile was an outlier
    int tilelast[NP]; // tile-local index of the tile's last outlier (-1 none)
};

template <int NP, class Src>
__global__ void __launch_bounds__(kEncThreads)
enc_quantize(EncPlanes P, Src src, int units) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E1Smem<NP> &S = *reinterpret_cast<E1Smem<NP> *>(smem_raw);
    using ScanI = cub::BlockScan<int, kEncThreads>;
    using RedI = cub::BlockReduce<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage scan_tmp;
    __shared__ typename RedI::TempStorage red_tmp;

    const int unit = blockIdx.x;
    if (unit >= units) return;
    const int tid = threadIdx.x;
    const uint64_t L = P.L;
    const long long half = 1ll << (P.qb - 1);
    const double hh = (double)half;
    const uint64_t C = 1ull << P.log2C;
    const uint64_t nidx = (L >> P.log2C) + 1;
    const int ntiles = (int)((L + kTile - 1) / kTile);

    PlaneParams prm[NP];
    for (int p = 0; p < NP; ++p) prm[p] = P.params[unit * NP + p];

    if (tid < NP) {
        S.dlast[tid] = 0.0;
        S.d2last[tid] = 0.0;
        S.xlast[tid] = 0.0;
        S.x2last[tid] = 0.0;
        S.base[tid] = 0.0;
        S.klast[tid] = 0;
        S.ocount[tid] = 0;
        S.prevout[tid] = 0;
        S.tilelast[tid] = -1;
        S.nev[tid] = 0;
        // linear predictor with eb > 0: no speculation model -> serial path
        S.fail[tid] = (P.predictor == 1 && prm[tid].eb != 0.0) ? 1 : 0;
    }
    __syncthreads();

    for (int t = 0; t < ntiles; ++t) {
        const uint64_t t0 = (uint64_t)t * kTile;
        const int tl = (int)tmin<uint64_t>(kTile, L - t0);
        // ---------------------------------------------------- load (striped)
        for (int k = tid; k < kTile; k += kEncThreads) {
            double v[2] = {0.0, 0.0};
            if (k < tl) src.load(unit, t0 + k, v);
            for (int p = 0; p < NP; ++p) S.x[p][k] = v[p];
        }
        __syncthreads();
        // ------------------------- sq-norm: adjacent-pair tree over the tile
        if (Src::kNorms) {
            double acc[kPerThread];
            for (int e = 0; e < kPerThread; ++e) {
                const int k = tid * kPerThread + e;
                const double a = dmul(S.x[0][k], S.x[0][k]);
                const double b = dmul(S.x[NP - 1][k], S.x[NP - 1][k]);
                acc[e] = dadd(a, b);
            }
            S.red[tid] = dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3]));
            __syncthreads();
            for (int w = kEncThreads / 2; w >= 1; w >>= 1) {
                double v = 0.0;
                if (tid < w) v = dadd(S.red[2 * tid], S.red[2 * tid + 1]);
                __syncthreads();
                if (tid < w) S.red[tid] = v;
                __syncthreads();
            }
            if (tid == 0) P.tilesum[(uint64_t)unit * ntiles + t] = S.red[0];
        }
        // ------------------------------------------------------- speculation
        for (int p = 0; p < NP; ++p) {
            if (S.fail[p]) continue; // uniform: read after a barrier
            const PlaneParams pp = prm[p];
            if (pp.eb == 0.0) {
                // Lossless / zero-range planes: d == x, symbols fully parallel.
                for (int e = 0; e < kPerThread; ++e) {
                    const int k = tid * kPerThread + e;
                    const uint64_t i = t0 + k;
                    const double x1 = k > 0 ? S.x[p][k - 1] : S.xlast[p];
                    const double x2 = k > 1 ? S.x[p][k - 2] : (k == 1 ? S.xlast[p] : S.x2last[p]);
                    double pred;
                    if (P.predictor == 0) pred = i > 0 ? x1 : 0.0;
                    else pred = i == 0 ? 0.0 : (i == 1 ? x1 : predict_linear(x1, x2));
                    S.ssym[p][k] = (k < tl && bits_of(S.x[p][k]) == bits_of(pred)) ? (uint32_t)half : 0u;
                }
                __syncthreads();
                continue;
            }
            // 1) speculative outliers from the jump size
            int opos[kPerThread];
            for (int e = 0; e < kPerThread; ++e) {
                const int k = tid * kPerThread + e;
                const double xp = k > 0 ? S.x[p][k - 1] : S.xlast[p];
                const double rr = dmul(dsub(S.x[p][k], xp), pp.inv_q);
                opos[e] = (k < tl && !(fabs(rr) < hh - 0.5)) ? k : -1;
            }
            // 2) last outlier strictly before each element
            int lo[kPerThread];
            ScanI(scan_tmp).ExclusiveScan(opos, lo, -1, cub::Max());
            // 3) lattice index relative to the segment base (an outlier is
            //    its own base, K = 0)
            long long K[kPerThread];
            for (int e = 0; e < kPerThread; ++e) {
                const int k = tid * kPerThread + e;
                if (opos[e] >= 0) {
                    K[e] = 0;
                } else {
                    const double base = lo[e] >= 0 ? S.x[p][lo[e]] : S.base[p];
                    K[e] = llround_exact(dmul(dsub(S.x[p][k], base), pp.inv_q));
                }
            }
            S.kb[p][tid] = K[kPerThread - 1];
            int mylast = -1;
            for (int e = 0; e < kPerThread; ++e) mylast = max(mylast, opos[e]);
            const int tile_last = RedI(red_tmp).Reduce(mylast, cub::Max());
            if (tid == 0) S.tilelast[p] = tile_last;
            __syncthreads();
            // 4) codes, events
            int evflag[kPerThread];
            for (int e = 0; e < kPerThread; ++e) {
                const int k = tid * kPerThread + e;
                uint8_t f = 0;
                uint32_t sy = 0;
                double c = 0.0;
                if (k < tl) {
                    long long kprev;
                    bool prev_out;
                    if (e > 0) { kprev = K[e - 1]; prev_out = opos[e - 1] >= 0; }
                    else if (tid > 0) { kprev = S.kb[p][tid - 1]; prev_out = lo[0] == k - 1; }
                    else { kprev = S.klast[p]; prev_out = S.prevout[p] != 0; }
                    if (prev_out) kprev = 0;
                    if (opos[e] >= 0) {
                        f = 3;
                        c = S.x[p][k];
                    } else {
                        const long long m = K[e] - kprev;
                        if (m <= -half || m >= half) atomicExch(&S.fail[p], 1);
                        sy = (uint32_t)(m + half);
                        c = dmul(pp.q, (double)m);
                        const double xp = k > 0 ? S.x[p][k - 1] : S.xlast[p];
                        // after a -0.0 outlier an m = 0 step yields +0.0
                        const bool negz = prev_out && bits_of(xp) == 0x8000000000000000ull;
                        f = (m != 0 || negz) ? 1 : 0;
                    }
                }
                S.fl[p][k] = f;
                S.ssym[p][k] = sy;
                S.c[p][k] = c;
                evflag[e] = f & 1;
            }
            // 5) compact the event list
            int epos[kPerThread];
            int total;
            ScanI(scan_tmp).ExclusiveSum(evflag, epos, total);
            for (int e = 0; e < kPerThread; ++e)
                if (evflag[e]) S.ev[p][epos[e]] = (uint16_t)(tid * kPerThread + e);
            if (tid == 0) S.nev[p] = total;
            __syncthreads();
        }
        // -------------------------------------------------------------- chain
        // One thread walks the planes' event lists; the independent chains
        // interleave so their DADD latencies overlap.
        if (tid == 0) {
            double dd[NP];
            int k[NP], ne[NP];
            for (int p = 0; p < NP; ++p) {
                dd[p] = S.dlast[p];
                k[p] = 0;
                ne[p] = (!S.fail[p] && prm[p].eb != 0.0) ? S.nev[p] : 0;
            }
            bool more = true;
            while (more) {
                more = false;
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    if (k[p] < ne[p]) {
                        const int i = S.ev[p][k[p]];
                        const double c = S.c[p][i];
                        const double sum = dadd(dd[p], c);
                        dd[p] = (S.fl[p][i] & 2) ? c : sum;
                        S.d[p][i] = dd[p];
                        ++k[p];
                        more |= k[p] < ne[p];
                    }
                }
            }
        }
        __syncthreads();
        // ------------------------------------------------- fill + verify
        for (int p = 0; p < NP; ++p) {
            if (S.fail[p]) continue;
            const PlaneParams pp = prm[p];
            const bool lossless = pp.eb == 0.0;
            double dfin[kPerThread];
            uint32_t esym[kPerThread];
            int isout[kPerThread];
            if (lossless) {
                for (int e = 0; e < kPerThread; ++e) {
                    const int k = tid * kPerThread + e;
                    dfin[e] = S.x[p][k];
                    esym[e] = S.ssym[p][k];
                    isout[e] = (k < tl && esym[e] == 0) ? 1 : 0;
                }
            } else {
                int evp[kPerThread], lev[kPerThread];
                for (int e = 0; e < kPerThread; ++e) {
                    const int k = tid * kPerThread + e;
                    evp[e] = (S.fl[p][k] & 1) ? k : -1;
                }
                ScanI(scan_tmp).ExclusiveScan(evp, lev, -1, cub::Max());
                int bad = 0;
                for (int e = 0; e < kPerThread; ++e) {
                    const int k = tid * kPerThread + e;
                    const double pred = lev[e] >= 0 ? S.d[p][lev[e]] : S.dlast[p];
                    const double dspec = evp[e] >= 0 ? S.d[p][k] : pred;
                    double rec = 0.0;
                    uint32_t sy = 0;
                    if (k < tl) {
                        sy = quantize(S.x[p][k], pred, pp.q, pp.inv_q, pp.eb, half, &rec);
                        if (sy == kOutlierSym) rec = S.x[p][k];
                        if (sy != S.ssym[p][k] || bits_of(rec) != bits_of(dspec)) bad = 1;
                    }
                    dfin[e] = rec;
                    esym[e] = sy;
                    isout[e] = (k < tl && sy == 0) ? 1 : 0;
                }
                if (bad) atomicExch(&S.fail[p], 1);
            }
            __syncthreads();
            if (S.fail[p]) continue; // uniform after the barrier
            int opos2[kPerThread];
            int ntot;
            ScanI(scan_tmp).ExclusiveSum(isout, opos2, ntot);
            const uint64_t pl = (uint64_t)unit * NP + p;
            uint32_t *symrow = P.sym + pl * L;
            for (int e = 0; e < kPerThread; ++e) {
                const int k = tid * kPerThread + e;
                if (k < tl) symrow[t0 + k] = esym[e];
                if (isout[e]) {
                    const uint64_t o = S.ocount[p] + (uint32_t)opos2[e];
                    P.opos[pl * L + o] = (uint32_t)(t0 + k);
                    P.oval[pl * L + o] = S.x[p][k];
                }
                S.c[p][k] = dfin[e]; // final reconstruction
            }
            __syncthreads();
            // checkpoints: dprev / dprev2 of every element e = j*C in the tile
            for (int k = tid; k < tl; k += kEncThreads) {
                const uint64_t i = t0 + k;
                if ((i & (C - 1)) == 0) {
                    IndexRec *r = P.index + pl * nidx + (i >> P.log2C);
                    r->dprev = k > 0 ? S.c[p][k - 1] : S.dlast[p];
                    r->dprev2 = k > 1 ? S.c[p][k - 2] : (k == 1 ? S.dlast[p] : S.d2last[p]);
                }
            }
            __syncthreads();
            if (tid == 0) {
                S.ocount[p] += (uint32_t)ntot;
                if (!lossless) {
                    const int lo = S.tilelast[p];
                    if (lo >= 0) S.base[p] = S.x[p][lo];
                    S.klast[p] = S.kb[p][kEncThreads - 1];
                    S.prevout[p] = (lo == tl - 1) ? 1 : 0;
                }
                S.d2last[p] = tl > 1 ? S.c[p][tl - 2] : S.dlast[p];
                S.dlast[p] = S.c[p][tl - 1];
                S.x2last[p] = tl > 1 ? S.x[p][tl - 2] : S.xlast[p];
                S.xlast[p] = S.x[p][tl - 1];
            }
            __syncthreads();
        }
    }
    if (tid < NP) {
        const uint64_t pl = (uint64_t)unit * NP + tid;
        P.ocount[pl] = S.ocount[tid];
        uint32_t f = P.params[pl].flags & ~kFlagFallback;
        if (S.fail[tid]) f |= kFlagFallback;
        P.params[pl].flags = f;
        if (!S.fail[tid] && (L & (C - 1)) == 0) {
            IndexRec *r = P.index + pl * nidx + (L >> P.log2C);
            r->dprev = S.dlast[tid];
            r->dprev2 = S.d2last[tid];
        }
    }
}

// ----------------------------------------------------------- E1f serial
// codec.cpp:430-458 verbatim, one thread per plane that needs it.
template <int NP, class Src>
__global__ void enc_serial(EncPlanes P, Src src, int units) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= units * NP) return;
    const int unit = gid / NP, p = gid % NP;
    const uint64_t pl = (uint64_t)gid;
    const PlaneParams pp = P.params[pl];
    if (!(pp.flags & kFlagFallback)) return;
    const uint64_t L = P.L;
    const long long half = 1ll << (P.qb - 1);
    const uint64_t C = 1ull << P.log2C;
    const uint64_t nidx = (L >> P.log2C) + 1;
    const double eb = pp.eb, q = pp.q;
    double d1 = 0.0, d2 = 0.0;
    uint32_t no = 0;
    uint32_t *symrow = P.sym + pl * L;
    for (uint64_t i = 0; i < L; ++i) {
        if ((i & (C - 1)) == 0) {
            IndexRec *r = P.index + pl * nidx + (i >> P.log2C);
            r->dprev = d1;
            r->dprev2 = d2;
        }
        double v[2];
        src.load(unit, i, v);
        const double x = v[p];
        double pred;
        if (P.predictor == 0) pred = i > 0 ? d1 : 0.0;
        else pred = i == 0 ? 0.0 : (i == 1 ? d1 : predict_linear(d1, d2));
        double rec = 0.0;
        uint32_t sy = kOutlierSym;
        if (eb == 0.0) {
            if (bits_of(x) == bits_of(pred)) { sy = (uint32_t)half; rec = pred; }
        } else {
            const double r = ddiv(dsub(x, pred), q);
            if (isfinite(r) && fabs(r) < (double)half) {
                const long long m = llround_exact(r);
                if (m > -half && m < half) {
                    const double rr = dadd(pred, dmul(q, (double)m));
                    if (isfinite(rr) && fabs(dsub(x, rr)) <= eb) { sy = (uint32_t)(m + half); rec = rr; }
                }
            }
        }
        if (sy == kOutlierSym) {
            rec = x;
            P.opos[pl * L + no] = (uint32_t)i;
            P.oval[pl * L + no] = x;
            ++no;
        }
        symrow[i] = sy;
        d2 = d1;
        d1 = rec;
    }
    if ((L & (C - 1)) == 0) {
        IndexRec *r = P.index + pl * nidx + (L >> P.log2C);
        r->dprev = d1;
        r->dprev2 = d2;
    }
    P.ocount[pl] = no;
}

// ----------------------------------------------------------- E2 tokenize
struct TokPlanes {
    const uint32_t *sym;     // [plane][L]
    uint32_t *tsym;          // [plane][L+1] token symbols
    uint32_t *trep;          // [plane][L+1] repeats (RUN tokens)
    uint32_t *ntok;          // [plane]
    uint32_t *hist;          // [plane][nbins]  nbins = 2^qb + 1 (kept zeroed)
    uint32_t *hspecial;      // [plane][2] counts of the outlier and RUN symbols
    uint32_t *symrange;      // [plane][2] min/max symbol seen
    uint64_t *gamma_bits;    // [plane]
    IndexRec *index;
    uint64_t L;
    int log2C;
    int qb;
};

struct TokSmem {
    uint32_t hist[kWin];
    uint32_t ssym[kTile];
    uint32_t tstart[kTile];
    uint32_t opre[kTile];
    uint16_t bl[kTile + 1];
    uint32_t h0, hrun;
    // carry: the open run
    uint32_t runsym, prevsym, runtok, ocur_start;
    uint64_t runstart;
    uint32_t ntok, ocount;
    unsigned long long gamma;
    uint32_t smin, smax;
    int nb;
};

// Checkpoint record for element e inside run [s, s+len) of symbol `sym`
// whose first token is `tok0` (codec.cpp:612-626 decoder state).
__device__ __forceinline__ void write_ckpt(IndexRec *r, uint64_t e, uint64_t s, uint64_t len, uint32_t sym,
                                           uint32_t prevsym, uint32_t tok0, uint32_t ocur_start) {
    const bool longrun = sym != kOutlierSym && len >= kMinRunLen;
    if (e == s) {
        r->tok = tok0;
        r->run_left = 0;
        r->last_lit = prevsym;
        r->ocur = ocur_start;
    } else {
        r->last_lit = sym;
        r->ocur = ocur_start + (sym == kOutlierSym ? (uint32_t)(e - s) : 0u);
        if (longrun) {
            r->tok = tok0 + 2;
            r->run_left = (uint32_t)(s + len - e);
        } else {
            r->tok = tok0 + (uint32_t)(e - s);
            r->run_left = 0;
        }
    }
}

__global__ void __launch_bounds__(kEncThreads) enc_tokenize(TokPlanes T, int planes) {
    const int pl = blockIdx.x;
    if (pl >= planes) return;
    const int tid = threadIdx.x;
    using ScanI = cub::BlockScan<int, kEncThreads>;
    __shared__ typename ScanI::TempStorage scan_tmp;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TokSmem &S = *reinterpret_cast<TokSmem *>(smem_raw);

    const uint64_t L = T.L;
    const long long half = 1ll << (T.qb - 1);
    const uint32_t rsym = 1u << T.qb;
    const uint64_t C = 1ull << T.log2C;
    const uint64_t nidx = (L >> T.log2C) + 1;
    const uint32_t *sym = T.sym + (uint64_t)pl * L;
    uint32_t *tsym = T.tsym + (uint64_t)pl * (L + 1);
    uint32_t *trep = T.trep + (uint64_t)pl * (L + 1);
    uint32_t *ghist = T.hist + (uint64_t)pl * ((uint64_t)rsym + 1);
    IndexRec *idx = T.index + (uint64_t)pl * nidx;
    const uint32_t wlo = (uint32_t)(half - kWin / 2);

    for (int k = tid; k < kWin; k += kEncThreads) S.hist[k] = 0;
    if (tid == 0) {
        S.runsym = sym[0];
        S.prevsym = rsym; // "no literal yet" sentinel
        S.runstart = 0;
        S.runtok = 0;
        S.ocur_start = 0;
        S.ntok = 0;
        S.ocount = 0;
        S.gamma = 0;
        S.smin = 0xFFFFFFFFu;
        S.smax = 0;
        S.h0 = 0;
        S.hrun = 0;
    }
    __syncthreads();

    auto count_sym = [&](uint32_t s, uint32_t n) {
        if (s == kOutlierSym) atomicAdd(&S.h0, n);
        else if (s == rsym) atomicAdd(&S.hrun, n);
        else if (s - wlo < (uint32_t)kWin) atomicAdd(&S.hist[s - wlo], n);
        else {
            atomicAdd(&ghist[s], n);
            atomicMin(&S.smin, s);
            atomicMax(&S.smax, s);
        }
    };

    const int ntiles = (int)((L + kTile - 1) / kTile);
    for (int t = 0; t < ntiles; ++t) {
        const uint64_t t0 = (uint64_t)t * kTile;
        const int tl = (int)tmin<uint64_t>(kTile, L - t0);
        const bool last_tile = t == ntiles - 1;
        for (int k = tid; k < tl; k += kEncThreads) S.ssym[k] = sym[t0 + k];
        __syncthreads();
        // boundaries: element k starts a new run
        int bflag[kPerThread], bpos[kPerThread], isout[kPerThread], opre[kPerThread];
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            const uint32_t prev = k > 0 ? S.ssym[k - 1] : S.runsym;
            bflag[e] = (k < tl && t0 + k > 0 && S.ssym[k] != prev) ? 1 : 0;
            isout[e] = (k < tl && S.ssym[k] == kOutlierSym) ? 1 : 0;
        }
        int nb, nout;
        ScanI(scan_tmp).ExclusiveSum(bflag, bpos, nb);
        __syncthreads();
        ScanI(scan_tmp).ExclusiveSum(isout, opre, nout);
        for (int e = 0; e < kPerThread; ++e)
            if (bflag[e]) S.bl[bpos[e]] = (uint16_t)(tid * kPerThread + e);
        if (tid == 0) S.nb = nb;
        __syncthreads();
        // The run carried in from earlier tiles closes here when the tile has
        // a boundary (or is the last tile); its tokens go first, through
        // element 0's scan slot (element 0 may itself start a new run).
        const bool carry_closes = nb > 0 || last_tile;
        const uint64_t carry_len = carry_closes ? t0 + (nb > 0 ? S.bl[0] : tl) - S.runstart : 0;
        const bool carry_long = S.runsym != kOutlierSym && carry_len >= kMinRunLen;
        const int carry_cnt = carry_closes ? (carry_long ? 2 : (int)carry_len) : 0;
        // per element: its run (ri = -1 is the carried run) and own tokens
        int cnt[kPerThread], tpos[kPerThread], ri[kPerThread];
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            ri[e] = bpos[e] + bflag[e] - 1; // boundaries at or before k, minus one
            cnt[e] = 0;
            if (k >= tl || ri[e] < 0) continue;
            const bool closed = ri[e] + 1 < nb || last_tile;
            if (!closed) continue;
            const uint32_t s = S.ssym[k];
            const int rs = S.bl[ri[e]];
            const uint64_t end = t0 + (ri[e] + 1 < nb ? S.bl[ri[e] + 1] : tl);
            const uint64_t len = end - (t0 + rs);
            const bool longrun = s != kOutlierSym && len >= kMinRunLen;
            cnt[e] = longrun ? (k == rs ? 2 : 0) : 1;
        }
        int scnt[kPerThread];
        for (int e = 0; e < kPerThread; ++e) scnt[e] = cnt[e] + ((tid == 0 && e == 0) ? carry_cnt : 0);
        int ntile;
        ScanI(scan_tmp).ExclusiveSum(scnt, tpos, ntile);
        __syncthreads();
        // own-token position of every element (carried tokens precede k = 0's)
        for (int e = 0; e < kPerThread; ++e) tpos[e] += (tid == 0 && e == 0) ? carry_cnt : 0;
        // emit the carried run
        if (tid == 0 && carry_cnt > 0) {
            const uint32_t tk = S.ntok;
            const uint32_t s = S.runsym;
            if (carry_long) {
                tsym[tk] = s;
                trep[tk] = 0;
                tsym[tk + 1] = rsym;
                trep[tk + 1] = (uint32_t)(carry_len - 1);
                count_sym(s, 1);
                count_sym(rsym, 1);
                atomicAdd(&S.gamma, (unsigned long long)(2 * bit_width64(carry_len - 1) - 1));
            } else {
                for (int r = 0; r < carry_cnt; ++r) {
                    tsym[tk + r] = s;
                    trep[tk + r] = 0;
                }
                count_sym(s, (uint32_t)carry_cnt);
            }
        }
        // emit runs that start and close in this tile
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            if (k >= tl || cnt[e] == 0) continue;
            const uint32_t s = S.ssym[k];
            const int rs = S.bl[ri[e]];
            const uint64_t end = t0 + (ri[e] + 1 < nb ? S.bl[ri[e] + 1] : tl);
            const uint64_t len = end - (t0 + rs);
            const bool longrun = s != kOutlierSym && len >= kMinRunLen;
            const uint32_t tk = S.ntok + (uint32_t)tpos[e];
            if (longrun) {
                tsym[tk] = s;
                trep[tk] = 0;
                tsym[tk + 1] = rsym;
                trep[tk + 1] = (uint32_t)(len - 1);
                count_sym(s, 1);
                count_sym(rsym, 1);
                atomicAdd(&S.gamma, (unsigned long long)(2 * bit_width64(len - 1) - 1));
            } else {
                tsym[tk] = s;
                trep[tk] = 0;
                count_sym(s, 1u);
            }
        }
        __syncthreads();
        // Resolve checkpoints with full run information (second sweep so
        // that start-element token positions are visible through smem).
        uint32_t *s_tpos_start = S.tstart;
        uint32_t *s_opre = S.opre;
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            s_tpos_start[k] = S.ntok + (uint32_t)tpos[e];
            s_opre[k] = S.ocount + (uint32_t)opre[e];
        }
        __syncthreads();
        for (int e = 0; e < kPerThread; ++e) {
            const int k = tid * kPerThread + e;
            const uint64_t i = t0 + k;
            if (k >= tl || (i & (C - 1)) != 0) continue;
            const bool closed = ri[e] + 1 < nb || last_tile;
            if (!closed) continue;
            const uint32_t s = S.ssym[k];
            const int rs = ri[e] >= 0 ? S.bl[ri[e]] : -1;
            const uint64_t start = ri[e] >= 0 ? t0 + rs : S.runstart;
            const uint64_t end = t0 + (ri[e] + 1 < nb ? S.bl[ri[e] + 1] : tl);
            const uint32_t tok0 = ri[e] >= 0 ? s_tpos_start[rs] : S.ntok;
            const uint32_t prevsym = ri[e] >= 0 ? (rs > 0 ? S.ssym[rs - 1] : S.runsym) : S.prevsym;
            const uint32_t ocs = ri[e] >= 0 ? s_opre[rs] : S.ocur_start;
            write_ckpt(&idx[i >> T.log2C], i, start, end - start, s, prevsym, tok0, ocs);
        }
        // checkpoints of the carried run that lie in earlier tiles
        const bool carried_closes = nb > 0 || last_tile;
        if (carried_closes && t > 0) {
            const uint64_t start = S.runstart;
            const uint64_t end = t0 + (nb > 0 ? S.bl[0] : tl);
            const uint64_t first_e = (start + C - 1) & ~(C - 1);
            for (uint64_t e = first_e + (uint64_t)tid * C; e < t0; e += (uint64_t)kEncThreads * C)
                write_ckpt(&idx[e >> T.log2C], e, start, end - start, S.runsym, S.prevsym, S.ntok, S.ocur_start);
        }
        __syncthreads();
        // carry update
        if (tid == 0) {
            if (nb > 0) {
                const int lb = S.bl[nb - 1];
                S.prevsym = lb > 0 ? S.ssym[lb - 1] : S.runsym;
                S.runsym = S.ssym[lb];
                S.runstart = t0 + lb;
                S.ocur_start = s_opre[lb];
            }
            S.ntok += (uint32_t)ntile;
            S.ocount += (uint32_t)nout;
        }
        __syncthreads();
    }
    // flush the window histogram into the dense per-plane histogram
    for (int k = tid; k < kWin; k += kEncThreads) {
        const uint32_t v = S.hist[k];
        const uint32_t sy = wlo + k;
        if (v && sy != kOutlierSym && sy < rsym) {
            ghist[sy] += v;
            atomicMin(&S.smin, sy);
            atomicMax(&S.smax, sy);
        }
    }
    __syncthreads();
    if (tid == 0) {
        T.ntok[pl] = S.ntok;
        T.gamma_bits[pl] = S.gamma;
        T.symrange[2 * pl] = S.smin;
        T.symrange[2 * pl + 1] = S.smax;
        T.hspecial[2 * pl] = S.h0;
        T.hspecial[2 * pl + 1] = S.hrun;
    }
}

} // namespace qcb
