// foreign_kernels.cuh -- chunk-parallel decode of QCB1 blocks that carry no
// decode index (decompress_plane / decompress_planes_device / partner
// imports; codec.cpp:535-633), the fast path in front of the validating
// token walk fd_scan (decode_kernels.cuh).
//
// The stream is cut into segments of kFpBits bits.  Prefix codes
// resynchronise: a decode started at an arbitrary bit soon falls onto the
// true token boundaries.  So:
//   fp_spec    one thread per segment decodes speculatively from the
//              segment's first bit to the first token boundary at or past its
//              end, recording its first kFpM boundaries with running element /
//              outlier / literal counts;
//   fp_resolve one thread per plane walks the segments: the true entry of
//              segment t is the exit of segment t-1; it must be one of t's
//              recorded boundaries (else the plane takes the serial path);
//              counts after it give every segment's element and outlier start
//              and the last literal before it;
//   fp_events  one thread per segment re-decodes its true tokens (twice:
//              count, then write) into the plane's event list -- the chain
//              addends RN(q*m) of nonzero codes, the outlier values, the
//              +0.0 step after a -0.0 outlier -- checking every condition of
//              codec.cpp:591-632 on the way (any failure: serial path);
//   fp_chain   one warp per plane runs the exact FP64 chain over the events
//              (codec.cpp:607) and writes the decoder record of every segment
//              entry; dec_chunks then decodes the segments in parallel.
// Blocks the fast path declines (sync failure, any check failing, the
// linear predictor) are decoded by fd_scan, whose serial walk reports the
// reference's exact first error.
#pragma once

#include "common.cuh"
#include "decode_kernels.cuh"

namespace qcb {

constexpr uint64_t kFpBits = 4096;   // segment length in stream bits
constexpr uint64_t kFpLead = 2048;   // a speculative decode starts this far before its segment (to resync)
constexpr uint64_t kFpSpan = 192;    // a token spans < 57 + 127 bits: the true entry lies within this of the start
constexpr int kFpM = 64;             // boundaries recorded per segment (in [start, start + kFpSpan))

struct FpBound {
    uint64_t bp;
    uint32_t elem, outl, lits, pad;
};
struct FpSeg {
    uint64_t exit;    // first boundary at or past the segment end (speculative path)
    uint64_t err_at;  // token start of the first decode failure (~0: none)
    uint32_t elem, outl, lits, last; // totals from the segment start; last literal symbol
    uint32_t nb;      // boundaries recorded
    uint32_t pad;
};
struct FpEntry {      // the true decoder state at a segment's entry
    uint64_t bp;
    uint32_t elem, outl, last, nev;
    uint32_t ev0;     // first event of the segment
    uint32_t pad;
};

struct FpArgs {
    const uint8_t *arena;
    const uint64_t *blk_off;
    uint32_t *err;        // [plane] != 0: header/table error (fd_head)
    uint32_t *slow;       // [plane] out: 1 = take the serial path
    uint64_t stride;      // segments per plane (max)
    FpBound *bnd;         // [plane][stride][kFpM]
    FpSeg *seg;           // [plane][stride]
    FpEntry *ent;         // [plane][stride]
    uint32_t *nseg;       // [plane]
    double *ev;           // [plane][n] event values
    uint8_t *evk;         // [plane][n] 1 = outlier value, 0 = addend
    IndexRec *rec;        // [plane][rec_stride] out
    uint32_t *nrec;       // [plane] out
    uint64_t rec_stride;
    uint64_t n;
};

// Per-plane view of a block (header already validated by fd_head).
struct FpPlane {
    const uint32_t *stream;
    const uint8_t *orec;
    uint64_t sbits, sbytes, n, nout;
    double eb, q;
    long long half;
    uint32_t rsym;
    int pred;
    const uint32_t *lut;
    const uint64_t *first;
    const uint32_t *count, *basei, *sorted;
    uint32_t maxlen;
    __device__ void init(const uint8_t *blk, const DecTables &T, int pl) {
        pred = blk[6];
        const int qb = blk[7];
        n = load_le(blk + 8, 8);
        eb = __longlong_as_double((long long)load_le(blk + 16, 8));
        q = dmul(2.0, eb);
        nout = load_le(blk + 24, 8);
        const uint64_t plen = load_le(blk + 32, 8);
        half = 1ll << (qb - 1);
        rsym = 1u << qb;
        const uint32_t tc = (uint32_t)load_le(blk + kHeaderBytes, 4);
        const uint64_t table_bytes = 4 + 5ull * tc;
        sbytes = plen - table_bytes - 16 * nout;
        sbits = sbytes * 8;
        stream = reinterpret_cast<const uint32_t *>(blk + kHeaderBytes + table_bytes);
        orec = blk + kHeaderBytes + table_bytes + sbytes;
        lut = T.lut + (uint64_t)pl * (1u << kLutBits);
        first = T.first + (uint64_t)pl * (kMaxCodeLen + 1);
        count = T.count + (uint64_t)pl * (kMaxCodeLen + 1);
        basei = T.basei + (uint64_t)pl * (kMaxCodeLen + 1);
        sorted = T.sorted + (uint64_t)pl * T.cap;
        maxlen = T.meta[4 * pl];
    }
    // One token at bp: its symbol, the bits it takes (code + gamma) and its
    // repeat count (RUN: the gamma value, else 1).  Returns false on a
    // decode failure (invalid / truncated code or gamma).
    __device__ __forceinline__ bool token(BitWindow &bw, uint64_t &bp, uint32_t &s, uint64_t &reps) const {
        const uint32_t le = lut[bw.acc >> (64 - kLutBits)];
        uint32_t l = le & 63;
        s = le >> 6;
        if (!l) {
            const uint64_t w = (int)maxlen <= bw.n ? bw.acc : peek64<false>(stream, bp);
            for (uint32_t ll = kLutBits + 1; ll <= maxlen; ++ll) {
                if (!count[ll]) continue;
                const uint64_t c = w >> (64 - ll);
                if (c >= first[ll] && c - first[ll] < count[ll]) {
                    s = sorted[basei[ll] + (uint32_t)(c - first[ll])];
                    l = ll;
                    break;
                }
            }
            if (!l) return false;
        }
        if (bp + l > sbits) return false;
        if ((int)l <= bw.n) bw.skip((int)l);
        else bw.init(stream, bp + l);
        bp += l;
        reps = 1;
        if (s == rsym) {
            const uint64_t g = peek64<false>(stream, bp);
            const int z = g ? __clzll((long long)g) : 64;
            if (z > 63 || bp + 2 * (uint64_t)z + 1 > sbits) return false;
            reps = z == 0 ? 1 : (peek64<false>(stream, bp + z) >> (63 - z));
            bp += 2 * (uint64_t)z + 1;
            bw.init(stream, bp);
        }
        return true;
    }
};

__global__ void __launch_bounds__(128) fp_spec(FpArgs A, DecTables T, int planes) {
    pdl_begin();
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int pl = (int)(gid / A.stride);
    const uint64_t t = gid % A.stride;
    if (pl >= planes || A.err[pl]) return;
    FpPlane P;
    P.init(A.arena + A.blk_off[pl], T, pl);
    const uint64_t nseg = (P.sbits + kFpBits - 1) / kFpBits;
    if (t == 0) A.nseg[pl] = (uint32_t)tmax<uint64_t>(nseg, 1);
    if (t >= nseg) return;
    FpBound *bnd = A.bnd + ((uint64_t)pl * A.stride + t) * kFpM;
    FpSeg S{};
    S.err_at = ~0ull;
    S.last = P.rsym;
    const uint64_t seg0 = t * kFpBits;
    // start early: by the segment's first bit the decode has fallen onto the
    // true token boundaries (prefix codes resynchronise)
    uint64_t bp = seg0 > kFpLead ? seg0 - kFpLead : 0;
    const uint64_t stop = (t + 1) * kFpBits;
    BitWindow bw;
    bw.init(P.stream, bp);
    uint32_t nb = 0, elem = 0, outl = 0, lits = 0;
    while (bp < stop && bp < P.sbits) {
        if (bp >= seg0 && bp < seg0 + kFpSpan && nb < (uint32_t)kFpM) bnd[nb++] = FpBound{bp, elem, outl, lits, 0};
        const uint64_t b0 = bp;
        uint32_t s;
        uint64_t reps;
        if (!P.token(bw, bp, s, reps)) {
            S.err_at = b0;
            break;
        }
        if (s == P.rsym) {
            elem += (uint32_t)tmin<uint64_t>(reps, 0xFFFFFFFFull);
        } else {
            ++elem;
            ++lits;
            S.last = s;
            if (s == kOutlierSym) ++outl;
        }
    }
    S.exit = bp;
    S.elem = elem;
    S.outl = outl;
    S.lits = lits;
    S.nb = nb;
    A.seg[(uint64_t)pl * A.stride + t] = S;
}

__global__ void fp_resolve(FpArgs A, DecTables T, int planes) {
    pdl_begin();
    const int pl = blockIdx.x * blockDim.x + threadIdx.x;
    if (pl >= planes || A.err[pl]) return;
    const uint8_t *blk = A.arena + A.blk_off[pl];
    FpPlane P;
    P.init(blk, T, pl);
    const uint32_t rsym = 1u << blk[7];
    // linear predictor (every element is an event) and lossless blocks take
    // the serial path
    const double heb = __longlong_as_double((long long)load_le(blk + 16, 8));
    uint32_t slow = (blk[6] != 0 || heb == 0.0) ? 1u : 0u;
    const uint32_t nseg = A.nseg[pl];
    uint64_t e = 0;
    uint32_t elem = 0, outl = 0, last = rsym;
    for (uint32_t t = 0; t < nseg && !slow; ++t) {
        const FpSeg S = A.seg[(uint64_t)pl * A.stride + t];
        const FpBound *bnd = A.bnd + ((uint64_t)pl * A.stride + t) * kFpM;
        // the true entry among the speculative path's first boundaries
        int b = -1;
        for (uint32_t k = 0; k < S.nb; ++k)
            if (bnd[k].bp == e) {
                b = (int)k;
                break;
            }
        FpEntry &E = A.ent[(uint64_t)pl * A.stride + t];
        E.bp = e;
        E.elem = elem;
        E.outl = outl;
        E.last = last;
        if (b < 0) {
            // the speculative decode did not resynchronise in time: walk this
            // segment from its true entry here
            if (t + 1 == nseg) break; // (fp_events walks the last one anyway)
            BitWindow bw;
            bw.init(P.stream, e);
            uint64_t bp = e;
            const uint64_t stop = (uint64_t)(t + 1) * kFpBits;
            while (bp < stop) {
                uint32_t sy;
                uint64_t reps;
                if (!P.token(bw, bp, sy, reps)) {
                    slow = 1;
                    break;
                }
                if (sy == P.rsym) {
                    elem += (uint32_t)tmin<uint64_t>(reps, 0xFFFFFFFFull);
                } else {
                    ++elem;
                    last = sy;
                    if (sy == kOutlierSym) ++outl;
                }
            }
            e = bp;
        } else {
            if (S.err_at != ~0ull && S.err_at >= e && t + 1 < nseg) {
                slow = 1; // a failure on the true path
                break;
            }
            elem += S.elem - bnd[b].elem;
            outl += S.outl - bnd[b].outl;
            if (S.lits > bnd[b].lits) last = S.last;
            e = S.exit;
        }
        if (elem > A.n) { // (the last segment may count padding as tokens: fp_events decides)
            if (t + 1 < nseg) slow = 1;
        }
    }
    A.slow[pl] = slow;
}

// Re-decodes segment t from its true entry.  write = false: counts events
// (into ent.nev); write = true: stores them at ent.ev0.  Any failure marks
// the plane slow.
__device__ __forceinline__ void fp_segment(const FpArgs &A, const DecTables &T, int pl, uint64_t t, bool write) {
    const uint32_t nseg = A.nseg[pl];
    if (t >= nseg) return;
    FpPlane P;
    P.init(A.arena + A.blk_off[pl], T, pl);
    FpEntry &E = A.ent[(uint64_t)pl * A.stride + t];
    const bool lastseg = t + 1 == nseg;
    const uint64_t stop = lastseg ? ~0ull : A.ent[(uint64_t)pl * A.stride + t + 1].bp;
    uint64_t bp = E.bp, i = E.elem, ocur = E.outl;
    uint32_t last = E.last;
    // d == -0.0 before the entry: only an outlier literal can leave it
    bool negz = last == kOutlierSym && ocur > 0 &&
                bits_of(__longlong_as_double((long long)load_le(P.orec + 16 * (ocur - 1) + 8, 8))) ==
                    0x8000000000000000ull;
    uint32_t nev = 0;
    double *ev = A.ev + (uint64_t)pl * A.n + E.ev0;
    uint8_t *evk = A.evk + (uint64_t)pl * A.n + E.ev0;
    auto bad = [&]() { atomicExch(&A.slow[pl], 1u); };
    BitWindow bw;
    bw.init(P.stream, bp);
    while (bp < stop && i < P.n) {
        uint32_t s;
        uint64_t reps;
        if (!P.token(bw, bp, s, reps)) return bad();
        if (s == P.rsym) {
            if (last == P.rsym || last == kOutlierSym) return bad();
            if (reps > P.n - i) return bad();
            const long long m = (long long)last - P.half;
            if (m != 0) {
                if (write) {
                    const double a = dmul(P.q, (double)m);
                    for (uint64_t k = 0; k < reps; ++k) {
                        ev[nev + k] = a;
                        evk[nev + k] = 0;
                    }
                }
                nev += (uint32_t)reps;
            } else if (negz && P.eb != 0.0) { // -0.0 + 0.0 = +0.0, then constant
                if (write) {
                    ev[nev] = dmul(P.q, 0.0);
                    evk[nev] = 0;
                }
                ++nev;
            }
            negz = false;
            i += reps;
            continue;
        }
        last = s;
        if (s == kOutlierSym) {
            if (ocur >= P.nout) return bad();
            if (load_le(P.orec + 16 * ocur, 8) != i) return bad();
            const double v = __longlong_as_double((long long)load_le(P.orec + 16 * ocur + 8, 8));
            if (write) {
                ev[nev] = v;
                evk[nev] = 1;
            }
            ++nev;
            ++ocur;
            negz = bits_of(v) == 0x8000000000000000ull;
        } else {
            const long long m = (long long)s - P.half;
            if (m != 0 || (negz && P.eb != 0.0)) {
                if (write) {
                    ev[nev] = dmul(P.q, (double)m);
                    evk[nev] = 0;
                }
                ++nev;
            }
            negz = false;
        }
        ++i;
    }
    if (lastseg) { // the reference's trailing checks (codec.cpp:628-632)
        if (i != P.n || ocur != P.nout || (bp + 7) / 8 != P.sbytes) return bad();
    } else if (bp != stop || i != A.ent[(uint64_t)pl * A.stride + t + 1].elem) {
        return bad();
    }
    if (!write) E.nev = nev;
}

__global__ void __launch_bounds__(128) fp_count(FpArgs A, DecTables T, int planes) {
    pdl_begin();
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int pl = (int)(gid / A.stride);
    if (pl >= planes || A.err[pl] || A.slow[pl]) return;
    fp_segment(A, T, pl, gid % A.stride, false);
}

__global__ void fp_evscan(FpArgs A, int planes) {
    pdl_begin();
    const int pl = blockIdx.x * blockDim.x + threadIdx.x;
    if (pl >= planes || A.err[pl] || A.slow[pl]) return;
    uint32_t acc = 0;
    for (uint32_t t = 0; t < A.nseg[pl]; ++t) {
        FpEntry &E = A.ent[(uint64_t)pl * A.stride + t];
        E.ev0 = acc;
        acc += E.nev;
    }
}

__global__ void __launch_bounds__(128) fp_events(FpArgs A, DecTables T, int planes) {
    pdl_begin();
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int pl = (int)(gid / A.stride);
    if (pl >= planes || A.err[pl] || A.slow[pl]) return;
    fp_segment(A, T, pl, gid % A.stride, true);
}

// The exact chain d = RN(d + RN(q*m)) / d = outlier over the plane's events,
// segment by segment; the decoder record of every segment entry (k >= 1).
// One warp per plane: the warp stages 1024 events at a time in shared
// memory, lane 0 runs the dependent additions.
__global__ void __launch_bounds__(32) fp_chain(FpArgs A, int planes) {
    pdl_begin();
    const int pl = blockIdx.x;
    if (pl >= planes || A.err[pl] || A.slow[pl]) return;
    constexpr int kStage = 2048;
    __shared__ double sv[kStage];
    __shared__ __align__(16) uint8_t sk[kStage];
    __shared__ uint32_t smask[kStage / 32]; // outlier flags of 32 staged events
    const int lane = threadIdx.x;
    const uint32_t nseg = A.nseg[pl];
    const double *ev = A.ev + (uint64_t)pl * A.n;
    const uint8_t *evk = A.evk + (uint64_t)pl * A.n;
    IndexRec *rec = A.rec + (uint64_t)pl * A.rec_stride;
    const FpEntry *ent = A.ent + (uint64_t)pl * A.stride;
    const uint64_t tot = (uint64_t)ent[nseg - 1].ev0 + ent[nseg - 1].nev;
    double d = 0.0;
    uint64_t staged0 = 0, staged1 = 0; // events [staged0, staged1) are in sv
    for (uint32_t t = 0; t < nseg; ++t) {
        const FpEntry E = ent[t];
        if (t > 0 && lane == 0) rec[t - 1] = IndexRec{d, 0.0, E.bp, 0u, E.outl, E.last, E.elem};
        uint64_t k = E.ev0;
        const uint64_t kend = (uint64_t)E.ev0 + E.nev;
        while (k < kend) {
            if (k >= staged1) { // stage the next events, 32-aligned groups (coalesced)
                __syncwarp();
                staged0 = k & ~31ull;
                staged1 = tmin<uint64_t>(staged0 + kStage, tot);
                // independent loads (many in flight), then the flag masks
#pragma unroll 16
                for (int j = lane; j < kStage; j += 32) {
                    const uint64_t x = staged0 + j;
                    sv[j] = x < staged1 ? __ldg(ev + x) : 0.0;
                    sk[j] = x < staged1 ? __ldg(evk + x) : 0;
                }
                __syncwarp();
                for (int g = lane; g < kStage / 32; g += 32) {
                    const uint4 a = *reinterpret_cast<const uint4 *>(sk + 32 * g);
                    const uint4 b = *reinterpret_cast<const uint4 *>(sk + 32 * g + 16);
                    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                    uint32_t m = 0;
#pragma unroll
                    for (int q = 0; q < 32; ++q)
                        if ((w[q >> 2] >> (8 * (q & 3))) & 0xFF) m |= 1u << q;
                    smask[g] = m;
                }
                __syncwarp();
            }
            const uint64_t hi = tmin<uint64_t>(kend, staged1);
            if (lane == 0) {
                uint64_t kk = k;
                while (kk < hi) {
                    const uint64_t r = kk - staged0;
                    const uint32_t m = smask[r >> 5] >> (r & 31);
                    if (m == 0 && (r & 31) == 0 && kk + 32 <= hi) {
                        // 32 addends, no outlier: the bare dependent additions
#pragma unroll
                        for (int u = 0; u < 32; ++u) d = dadd(d, sv[r + u]);
                        kk += 32;
                        continue;
                    }
                    const double v = sv[r];
                    d = (m & 1u) ? v : dadd(d, v);
                    ++kk;
                }
            }
            k = hi;
        }
    }
    if (lane == 0) A.nrec[pl] = nseg > 0 ? nseg - 1 : 0;
}

} // namespace qcb
