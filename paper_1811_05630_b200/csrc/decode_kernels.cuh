// decode_kernels.cuh -- QCB1 decoder kernels (decompress_plane,
// codec.cpp:535-633).
//
// D1 dec_prepare  one block per plane: parse the code table, canonical
//                 codes (codec.cpp:233-249), an 11-bit lookup table plus
//                 first-code/count/base arrays for longer codes
//                 (PrefixDecoder, codec.cpp:251-286).
// D2 dec_chunks   one thread per (plane, checkpoint chunk): resumes from the
//                 encoder's IndexRec and reproduces codec.cpp:591-626 for
//                 C elements -- chunk-parallel and bit-exact.
// FD fd_head / fd_scan (below) + foreign_kernels.cuh: blocks without a decode
//                 index (host API, partner imports), every check and error of
//                 codec.cpp:535-633 in the reference's order.
#pragma once

#include "common.cuh"
#include "norm.cuh"

namespace qcb {

struct DecTables {
    uint32_t *lut;       // [plane][1 << kLutBits]: sym << 6 | len (0 = long code)
    uint64_t *first;     // [plane][kMaxCodeLen + 1]
    uint32_t *count;     // [plane][kMaxCodeLen + 1]
    uint32_t *basei;     // [plane][kMaxCodeLen + 1]
    uint32_t *sorted;    // [plane][cap] symbols in (len, sym) order
    uint32_t *meta;      // [plane][4]: maxlen, nsym, table bytes lo, -
    uint64_t cap;
};

struct DecPlanes {
    const uint8_t *arena;
    const uint64_t *blk_off;   // [plane] block start in the arena (its decode index follows it)
    double *const *out;        // [plane] output plane
    uint64_t L;
    int log2C;                 // fine checkpoint spacing (index_records, common.cuh)
    // foreign blocks (no index in a slot): records built by fd_scan
    const IndexRec *ext_index = nullptr; // [plane][ext_stride]
    const uint32_t *ext_nrec = nullptr;  // [plane]
    uint64_t ext_stride = 0;
    // fine > 0: ext_index holds the ENCODER's fine checkpoints of the pass
    // that wrote these blocks (one every 2^(fine) elements, still in the
    // engine's scratch inside one run()): record k (1-based) is the decoder
    // state at element k << fine, every plane has ext_fixed_nrec of them
    // (ext_nrec unused).  Small planes carry only a few stored records
    // (7.8% of a ~2.5 KB block); the scratch checkpoints give the deferred
    // loop its chunk parallelism back without enlarging the stored state.
    int fine = 0;
    uint32_t ext_fixed_nrec = 0;
    const uint32_t *skip = nullptr;      // [plane] != 0: not decoded (a codec error was found)
    // Zero-tile flags (run-aware gate pass, SURVEY.md §7 H1 "run-aware
    // shortcut"): an encoder tile (kTile elements) that lies inside one long
    // run of +0.0 is not written at all; zflag[plane * ztiles + tile] = 1
    // tells the gate kernel that the tile's values are +0.0.  The flags are
    // cleared before the grid runs.  nullptr: every element is written.
    uint8_t *zflag = nullptr;
    uint32_t ztiles = 0;
};

__device__ __forceinline__ uint64_t load_le(const uint8_t *p, int bytes) {
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

__global__ void __launch_bounds__(256) dec_prepare(DecPlanes D, DecTables T, int planes) {
    pdl_begin();
    const int pl = blockIdx.x;
    if (pl >= planes) return;
    if (D.skip && D.skip[pl]) return; // invalid table: never parsed
    const int tid = threadIdx.x;
    __shared__ uint32_t cnt[kMaxCodeLen + 1];
    __shared__ uint64_t first[kMaxCodeLen + 1];
    __shared__ uint32_t basei[kMaxCodeLen + 1];
    __shared__ uint32_t s_n;
    const uint8_t *blk = D.arena + D.blk_off[pl];
    const uint8_t *tab = blk + kHeaderBytes + 4;
    if (tid == 0) s_n = (uint32_t)load_le(blk + kHeaderBytes, 4);
    if (tid <= kMaxCodeLen) cnt[tid] = 0;
    uint32_t *lut = T.lut + (uint64_t)pl * (1u << kLutBits);
    for (int k = tid; k < (1 << kLutBits); k += 256) lut[k] = 0;
    __syncthreads();
    const uint32_t n = s_n;
    for (uint32_t r = tid; r < n; r += 256) atomicAdd(&cnt[tab[5ull * r + 4]], 1u);
    __syncthreads();
    if (tid == 0) {
        uint64_t c = 0;
        int prev = -1;
        uint32_t b = 0;
        uint32_t maxlen = 0;
        for (int l = 1; l <= kMaxCodeLen; ++l) {
            first[l] = 0;
            basei[l] = b;
            if (!cnt[l]) continue;
            if (prev >= 0) c <<= (l - prev);
            first[l] = c;
            c += cnt[l];
            b += cnt[l];
            prev = l;
            maxlen = l;
        }
        // symbols in (len, sym) order: the table is in symbol order, so a
        // stable pass by length keeps symbol order inside each length
        uint32_t next[kMaxCodeLen + 1];
        for (int l = 0; l <= kMaxCodeLen; ++l) next[l] = basei[l];
        uint32_t *sorted = T.sorted + (uint64_t)pl * T.cap;
        for (uint32_t r = 0; r < n; ++r) {
            const uint8_t l = tab[5ull * r + 4];
            sorted[next[l]++] = (uint32_t)load_le(tab + 5ull * r, 4);
        }
        for (int l = 0; l <= kMaxCodeLen; ++l) {
            T.first[(uint64_t)pl * (kMaxCodeLen + 1) + l] = first[l];
            T.count[(uint64_t)pl * (kMaxCodeLen + 1) + l] = cnt[l];
            T.basei[(uint64_t)pl * (kMaxCodeLen + 1) + l] = basei[l];
        }
        T.meta[4 * pl] = maxlen;
        T.meta[4 * pl + 1] = n;
    }
    __syncthreads();
    // short codes -> LUT
    const uint32_t *sorted = T.sorted + (uint64_t)pl * T.cap;
    for (uint32_t r = tid; r < n; r += 256) {
        // r-th entry in (len, sym) order
        int l = 1;
        while (l < kMaxCodeLen && !(r >= basei[l] && r < basei[l] + cnt[l])) ++l;
        if (l > kLutBits) continue;
        const uint64_t code = first[l] + (r - basei[l]);
        const uint32_t lo = (uint32_t)(code << (kLutBits - l));
        const uint32_t hi = (uint32_t)((code + 1) << (kLutBits - l));
        const uint32_t e = (sorted[r] << 6) | (uint32_t)l;
        for (uint32_t k = lo; k < hi; ++k) lut[k] = e;
    }
}

// 64-bit MSB-first window at stream bit `bp` of big-endian-ordered words
// (the block's stream starts 16-byte aligned in the arena; the arena and
// the shared staging buffer are padded, so reading 3 words ahead is safe).
template <bool kShared>
__device__ __forceinline__ uint64_t peek64(const uint32_t *w, uint64_t bp) {
    const uint64_t wi = bp >> 5;
    const uint32_t b = (uint32_t)(bp & 31);
    uint32_t w0, w1, w2;
    if (kShared) {
        w0 = w[wi];
        w1 = w[wi + 1];
        w2 = w[wi + 2];
    } else {
        w0 = __ldg(w + wi);
        w1 = __ldg(w + wi + 1);
        w2 = __ldg(w + wi + 2);
    }
    const uint64_t hi = ((uint64_t)bswap32(w0) << 32) | bswap32(w1);
    if (b == 0) return hi;
    return (hi << b) | (bswap32(w2) >> (32 - b));
}

// MSB-first bit window over a word stream: `acc` holds the next n valid bits
// (32 < n <= 64 between symbols), `pre` the next word, loaded one refill
// ahead, so a symbol costs shifts instead of dependent word loads.
struct BitWindow {
    uint64_t acc;
    int n;
    const uint32_t *src; // next word after `pre`
    uint32_t pre;
    __device__ __forceinline__ void init(const uint32_t *words, uint64_t bitpos) {
        const uint64_t wi = bitpos >> 5;
        const int b = (int)(bitpos & 31);
        acc = (((uint64_t)bswap32(words[wi]) << 32) | bswap32(words[wi + 1])) << b;
        n = 64 - b;
        pre = words[wi + 2];
        src = words + wi + 3;
        refill();
    }
    __device__ __forceinline__ void refill() {
        while (n <= 32) {
            acc |= (uint64_t)bswap32(pre) << (32 - n);
            n += 32;
            pre = *src++;
        }
    }
    __device__ __forceinline__ void skip(int l) { // l <= n
        acc = l < 64 ? acc << l : 0ull;
        n -= l;
        refill();
    }
};

constexpr int kDecThreads = 128;             // chunks per block (one per thread)
constexpr int kDecStageWords = 4096;         // 16 KB of stream staged per block
constexpr int kDecBatch = 8;                 // listed (long) runs per lane per batch
constexpr int kDecTokBatch = 64;             // tokens per lane per batch
constexpr int kDecFills = 64;                // block-wide fills per block
constexpr uint32_t kDecBlockFill = 4096;     // runs at least this long are filled by the whole block
constexpr uint32_t kDecWarpRun = 32;         // runs at least this long are written by the whole warp
struct DecFill {
    uint64_t start;
    uint64_t len;
    double v;
};
struct DecRun {          // elements [start, end) take `v`
    uint32_t start;
    uint32_t end;
    double v;
};
struct DecSmem {
    uint32_t lut[1 << kLutBits];
    uint32_t sw[kDecStageWords + 4];
    DecRun runs[kDecBatch][kDecThreads];          // entry-major: a warp's lanes write adjacent entries
    DecFill fill[kDecFills];
    uint32_t nfill;
};
constexpr size_t kDecSmem = sizeof(DecSmem);

// One block per (plane, group of kDecThreads index chunks).  The plane's
// chunk count follows from its block size (index_records), the records come
// from the index stored after the block in its slot; blocks past the plane's
// chunk count exit.  The plane's 11-bit LUT and the group's stream words
// are staged in shared memory.
//
// Decoding reproduces codec.cpp:591-626 in two alternating phases per warp:
//  1. every lane decodes its own chunk, token by token, from its record.  A
//     literal is one element (d = p + (2eb)m, or the outlier), written at
//     once by the lane; a RUN token of a zero code with the previous-value
//     predictor is ONE constant run of d (d + 0.0 == d, the first element
//     canonicalises -0.0): shorter than kDecWarpRun elements it is written
//     by the lane, longer it goes to the lane's run list, and from
//     kDecBlockFill elements on to the block list; other RUN tokens (nonzero
//     code, linear predictor) emit one element per step, as the reference's
//     serial loop does.  The FP64 work is per token, in the reference's order;
//  2. the warp writes the listed runs of its lanes in turn, 32 consecutive
//     elements per store (coalesced).  The block list is written by all
//     threads at the end (whole tiles of +0.0 are flagged instead, zflag).
// N.enabled: the grid's last block runs the engine's normalization for this
// gate pass instead (it needs only the previous pass's norms; the gate kernel
// that applies the scale runs after this grid).
__global__ void __launch_bounds__(kDecThreads, 5) dec_chunks(DecPlanes D, DecTables T, int planes, NormArgs N) {
    pdl_begin();
    if (N.enabled && blockIdx.x == gridDim.x - 1) {
        engine_norm_body(N);
        return;
    }
    extern __shared__ __align__(16) unsigned char dec_raw[];
    DecSmem &S = *reinterpret_cast<DecSmem *>(dec_raw);
    const uint64_t nchunks_max = D.ext_index ? D.ext_stride + 1 : ((D.L + (1ull << D.log2C) - 1) >> D.log2C);
    const uint32_t groups = (uint32_t)((nchunks_max + kDecThreads - 1) / kDecThreads);
    const int pl = (int)(blockIdx.x / groups);
    if (pl >= planes) return;
    if (D.skip && D.skip[pl]) return;
    const uint8_t *blk = D.arena + D.blk_off[pl];
    const uint64_t payload = load_le(blk + 32, 8);
    const uint64_t bbytes = kHeaderBytes + payload;
    const uint64_t nchunks =
        (D.ext_index ? (D.fine ? D.ext_fixed_nrec : D.ext_nrec[pl]) : index_records(D.L, bbytes, D.log2C)) + 1;
    const uint64_t j0 = (uint64_t)(blockIdx.x % groups) * kDecThreads;
    if (j0 >= nchunks) return;
    const uint64_t j = j0 + threadIdx.x;
    const uint64_t jend = tmin<uint64_t>(j0 + kDecThreads, nchunks);
    const uint8_t pred_kind = blk[6];
    const int qb = blk[7];
    const long long half = 1ll << (qb - 1);
    const uint32_t rsym = 1u << qb;
    const double eb = __longlong_as_double((long long)load_le(blk + 16, 8));
    const double q = dmul(2.0, eb);
    const uint64_t nout = load_le(blk + 24, 8);
    const uint32_t n = T.meta[4 * pl + 1];
    const uint32_t maxlen = T.meta[4 * pl];
    const uint64_t table_bytes = 4 + 5ull * n;
    const uint64_t sbytes = payload - table_bytes - 16 * nout;
    const uint32_t *stream = reinterpret_cast<const uint32_t *>(blk + kHeaderBytes + table_bytes);
    const uint8_t *orec = blk + kHeaderBytes + table_bytes + sbytes;
    const uint32_t *glut = T.lut + (uint64_t)pl * (1u << kLutBits);
    const uint64_t *first = T.first + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *count = T.count + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *basei = T.basei + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *sorted = T.sorted + (uint64_t)pl * T.cap;
    const IndexRec *sidx = D.ext_index ? D.ext_index + (uint64_t)pl * D.ext_stride
                                       : reinterpret_cast<const IndexRec *>(D.arena + index_offset(D.blk_off[pl], bbytes));
    auto rec_bitpos = [&](uint64_t jj) -> uint64_t { return jj == 0 ? 0ull : sidx[jj - 1].bitpos; };

    {
        const uint4 *g4 = reinterpret_cast<const uint4 *>(glut);
        uint4 *s4 = reinterpret_cast<uint4 *>(S.lut);
#pragma unroll
        for (int k = threadIdx.x; k < (1 << kLutBits) / 4; k += kDecThreads) s4[k] = g4[k];
    }
    if (threadIdx.x == 0) S.nfill = 0;
    // stream words this group reads: [bitpos(j0), bitpos(jend)) + lookahead
    const uint64_t w_lo = rec_bitpos(j0) >> 5;
    const uint64_t bit_hi = jend < nchunks ? rec_bitpos(jend) : sbytes * 8;
    const uint64_t w_hi = (bit_hi >> 5) + 3;
    const bool staged = w_hi - w_lo <= (uint64_t)kDecStageWords;
    if (staged)
        for (uint64_t w = w_lo + threadIdx.x; w < w_hi; w += kDecThreads) S.sw[w - w_lo] = __ldg(stream + w);
    __syncthreads();

    const bool active = j < jend;
    const int lane = threadIdx.x & 31;
    IndexRec r{};
    if (active && j > 0) r = sidx[j - 1];
    if (j == 0) r.last_lit = rsym; // initial decoder state (codec.cpp:587-590)
    uint64_t bp = r.bitpos;
    uint32_t run_left = r.run_left;
    const uint32_t *wsrc = staged ? S.sw : stream; // the window's word source ...
    const uint64_t wbase = staged ? w_lo * 32 : 0;  // ... and its first bit
    const uint64_t sbase = wbase;
    // the lane's next bits in a register window (refilled one 32-bit word at
    // a time from the staged words or the stream): one LUT probe per token
    BitWindow bw;
    if (active) bw.init(wsrc, bp - wbase);
    uint32_t last = r.last_lit;
    uint64_t ocur = r.ocur;
    double d1 = r.dprev, d2 = r.dprev2;
    // chunk j: from record j to record j + 1 (element indices in `tok`)
    const uint64_t e0 = j == 0 ? 0 : (D.fine ? j << D.fine : (uint64_t)r.tok);
    const uint64_t e1 = !active ? e0 : (j + 1 < nchunks ? (D.fine ? (j + 1) << D.fine : (uint64_t)sidx[j].tok) : D.L);
    double *out = D.out[pl];
    const int wbase_t = threadIdx.x & ~31; // first thread of this warp

    uint64_t i = e0;
    bool dead = !active;
    // value of the element at i for symbol s (codec.cpp:605-611)
    auto value_of = [&](uint32_t s) -> double {
        if (s == kOutlierSym) {
            const double v = __longlong_as_double((long long)load_le(orec + 16 * ocur + 8, 8));
            ++ocur;
            return v;
        }
        double pred;
        if (pred_kind == 0) pred = i > 0 ? d1 : 0.0;
        else pred = i == 0 ? 0.0 : (i == 1 ? d1 : predict_linear(d1, d2));
        const long long m = (long long)s - half;
        return eb == 0.0 ? pred : dadd(pred, dmul(q, (double)m));
    };
    while (__any_sync(0xffffffffu, !dead && i < e1)) {
        // ---- phase 1: up to kDecTokBatch tokens of this lane's chunk.
        // Literals and constant runs shorter than kDecWarpRun elements are
        // written at once by their own lane; longer runs go to the lane's
        // run list (whole warp, phase 2) or the block list (>= kDecBlockFill)
        int nr = 0, ntok = 0;
        while (!dead && i < e1 && nr < kDecBatch && ntok < kDecTokBatch) {
            ++ntok;
            if (run_left > 0) {
                const double v = value_of(last);
                if (pred_kind == 0 && bits_of(v) == bits_of(d1) && i > 0) {
                    // a constant run: the rest of the RUN (within the chunk)
                    const uint64_t take = tmin<uint64_t>(run_left, e1 - i);
                    bool placed = false;
                    if (take >= kDecBlockFill) {
                        const uint32_t slot = atomicAdd(&S.nfill, 1u);
                        if (slot < (uint32_t)kDecFills) {
                            S.fill[slot] = DecFill{i, take, v};
                            placed = true;
                        }
                    }
                    if (!placed) {
                        if (take >= kDecWarpRun) S.runs[nr++][threadIdx.x] = DecRun{(uint32_t)i, (uint32_t)(i + take), v};
                        else
                            for (uint64_t e = i; e < i + take; ++e) out[e] = v;
                    }
                    i += take;
                    run_left -= (uint32_t)take;
                    d2 = v;
                    continue;
                }
                // one element of the run (first element of a -0.0 run, a
                // nonzero code, the linear predictor)
                out[i] = v;
                d2 = d1;
                d1 = v;
                ++i;
                --run_left;
                continue;
            }
            const uint64_t wtop = bw.acc;
            const uint32_t le = S.lut[wtop >> (64 - kLutBits)];
            uint32_t s, l;
            if (le & 63) {
                l = le & 63;
                s = le >> 6;
                bw.skip((int)l);
            } else {
                // a code longer than the LUT: from the window when it holds
                // maxlen bits, else from the words (then the window restarts)
                const bool inwin = (int)maxlen <= bw.n;
                const uint64_t w = inwin ? wtop : (staged ? peek64<true>(S.sw, bp - sbase) : peek64<false>(stream, bp));
                s = 0;
                l = 0;
                for (uint32_t ll = kLutBits + 1; ll <= maxlen; ++ll) {
                    if (!count[ll]) continue;
                    const uint64_t c = w >> (64 - ll);
                    if (c >= first[ll] && c - first[ll] < count[ll]) {
                        s = sorted[basei[ll] + (uint32_t)(c - first[ll])];
                        l = ll;
                        break;
                    }
                }
                if (l == 0) { // corrupt (never for encoder-produced blocks)
                    dead = true;
                    break;
                }
                if (inwin) bw.skip((int)l);
                else bw.init(wsrc, bp + l - wbase);
            }
            bp += l;
            if (s == rsym) {
                // Elias gamma: z zeros, then the value in z + 1 bits
                const int z = __clzll((long long)bw.acc);
                if (2 * z + 1 <= bw.n) {
                    run_left = (uint32_t)(bw.acc >> (64 - (2 * z + 1)));
                    bw.skip(2 * z + 1);
                    bp += 2 * z + 1;
                } else {
                    const uint64_t g = staged ? peek64<true>(S.sw, bp - sbase) : peek64<false>(stream, bp);
                    const int zz = __clzll((long long)g);
                    run_left = (uint32_t)(g >> (64 - (2 * zz + 1)));
                    bp += 2 * zz + 1;
                    bw.init(wsrc, bp - wbase);
                }
            } else {
                const double v = value_of(s);
                out[i] = v;
                d2 = d1;
                d1 = v;
                ++i;
                last = s;
            }
        }
        // ---- phase 2: the listed runs (>= kDecWarpRun elements), each by the
        // whole warp, 32 consecutive elements per store (coalesced)
        __syncwarp();
        unsigned lanes = __ballot_sync(0xffffffffu, nr > 0);
        while (lanes) {
            const int rr = __ffs(lanes) - 1;
            lanes &= lanes - 1;
            const int n = __shfl_sync(0xffffffffu, nr, rr);
            const int col = wbase_t + rr;
            for (int c = 0; c < n; ++c) {
                const DecRun R = S.runs[c][col];
                for (uint64_t e = (uint64_t)R.start + (uint64_t)lane; e < (uint64_t)R.end; e += 32) out[e] = R.v;
            }
        }
        __syncwarp();
    }
    __syncthreads();
    // long constant runs, coalesced by the whole block
    const uint32_t nf = tmin<uint32_t>(S.nfill, (uint32_t)kDecFills);
    auto fill_range = [&](uint64_t st, uint64_t len, double v) {
        if (len == 0) return;
        if (st & 1) { // 16-byte aligned vector stores after an odd head
            if (threadIdx.x == 0) out[st] = v;
            ++st;
            --len;
        }
        double4 *o4 = reinterpret_cast<double4 *>(out + st);
        const uint64_t n4 = (st & 3) ? 0 : len / 4; // 32-byte stores when aligned
        const double4 v4 = make_double4(v, v, v, v);
        for (uint64_t k = threadIdx.x; k < n4; k += kDecThreads) o4[k] = v4;
        double2 *o2 = reinterpret_cast<double2 *>(out + st + 4 * n4);
        const uint64_t rest = len - 4 * n4;
        const double2 v2 = make_double2(v, v);
        for (uint64_t k = threadIdx.x; k < rest / 2; k += kDecThreads) o2[k] = v2;
        if ((rest & 1) && threadIdx.x == 0) out[st + 4 * n4 + rest - 1] = v;
    };
    for (uint32_t f = 0; f < nf; ++f) {
        const DecFill F = S.fill[f];
        if (D.zflag && bits_of(F.v) == 0ull) {
            // whole tiles of +0.0: flagged, not written (the gate kernel
            // reads the flag); the ragged head and tail are written
            const uint64_t t_lo = (F.start + kTile - 1) >> kTileLog2, t_hi = (F.start + F.len) >> kTileLog2;
            if (t_hi > t_lo) {
                uint8_t *zf = D.zflag + (uint64_t)pl * D.ztiles;
                for (uint64_t t = t_lo + threadIdx.x; t < t_hi; t += kDecThreads) zf[t] = 1;
                fill_range(F.start, (t_lo << kTileLog2) - F.start, F.v);
                fill_range(t_hi << kTileLog2, F.start + F.len - (t_hi << kTileLog2), F.v);
                continue;
            }
        }
        fill_range(F.start, F.len, F.v);
    }
}

// ------------------------------------------------------------ validating
enum DecErr : uint32_t {
    kDecOk = 0,
    kDecPayloadSmall,     // "payload smaller than code table header"
    kDecTableEmpty,       // "empty prefix-code table"
    kDecTableTrunc,       // "code table truncated"
    kDecSymOrder,         // "code table symbols not strictly increasing"
    kDecSymRange,         // "code table symbol out of range"
    kDecLenRange,         // "code length out of range"
    kDecOverfull,         // "prefix code table overfull"
    kDecLenMismatch,      // "payload/header length mismatch"
    kDecStreamTrunc,      // "code stream truncated"
    kDecInvalidCode,      // "invalid prefix code in stream"
    kDecRunNoCode,        // "run escape without preceding code"
    kDecRunRange,         // "run length out of range"
    kDecRunOverflow,      // "run overflows element count"
    kDecOutExhausted,     // "outlier list exhausted early"
    kDecOutPos,           // "outlier position mismatch"
    kDecOutUnused,        // "unused trailing outliers"
    kDecStreamLen,        // "code stream length mismatch"
    kDecNoMem,            // scratch too small
    // header checks (from_bytes, codec.cpp:366-408) for device-resident
    // blocks whose headers the host never saw (engine partner imports)
    kDecHdrTrunc,         // "block header truncated"
    kDecMagic,            // "bad block magic"
    kDecVersion,          // "unsupported block version"
    kDecModeByte,         // "bad codec mode byte"
    kDecPredByte,         // "bad predictor byte"
    kDecQbRange,          // "quant_code_bits out of range"
    kDecCount0,           // "element_count must be at least 1"
    kDecOutCount,         // "outlier_count exceeds element_count"
    kDecEbBad,            // "bad effective_abs_bound"
    kDecPayTrunc,         // "block payload truncated"
    kDecWrongLen,         // element_count differs from the destination plane
};


// ------------------------------------------------------- foreign blocks
// QCB1 blocks that carry no decode index (decompress_plane, partner
// imports): fd_head validates header and code table (codec.cpp:366-408,
// 535-583, the reference's order), dec_prepare builds the tables, fd_scan
// walks every token once -- one thread per plane, every check of
// codec.cpp:585-632 in order, no element stores -- and leaves a decode
// record (the decoder state at a token boundary) every kFdBits stream bits;
// dec_chunks then writes the elements chunk-parallel from those records.
constexpr uint64_t kFdBits = 4096;

struct FdArgs {
    const uint8_t *arena;      // staged blocks (code streams 16-byte aligned, padded)
    const uint64_t *blk_off;   // [plane]
    const uint64_t *avail;     // [plane] bytes available (header checks)
    uint32_t *err;             // [plane] out: first error (kDec*), 0 = ok
    uint64_t n_expected;       // element_count every block must have
    uint64_t cap;              // code-table capacity of the decode tables
    IndexRec *rec;             // [plane][stride] out
    uint32_t *nrec;            // [plane] out
    uint64_t stride;
    const uint32_t *only = nullptr; // fd_scan: [plane] != 0 selects the planes to walk
};

__global__ void fd_head(FdArgs A, int planes) {
    pdl_begin();
    const int pl = blockIdx.x * blockDim.x + threadIdx.x;
    if (pl >= planes) return;
    const uint8_t *blk = A.arena + A.blk_off[pl];
    auto fail = [&](uint32_t e) { A.err[pl] = e; };
    A.err[pl] = kDecOk;
    const uint64_t len = A.avail[pl];
    if (len < kHeaderBytes) return fail(kDecHdrTrunc);
    if (blk[0] != 'Q' || blk[1] != 'C' || blk[2] != 'B' || blk[3] != '1') return fail(kDecMagic);
    if (blk[4] != 1) return fail(kDecVersion);
    if (blk[5] > 2) return fail(kDecModeByte);
    if (blk[6] > 1) return fail(kDecPredByte);
    if (blk[7] < 4 || blk[7] > 24) return fail(kDecQbRange);
    const uint64_t n = load_le(blk + 8, 8), nout = load_le(blk + 24, 8), plen = load_le(blk + 32, 8);
    const double heb = __longlong_as_double((long long)load_le(blk + 16, 8));
    if (n == 0) return fail(kDecCount0);
    if (nout > n) return fail(kDecOutCount);
    if (!(heb >= 0.0) || !isfinite(heb)) return fail(kDecEbBad);
    if (plen > len - kHeaderBytes) return fail(kDecPayTrunc);
    if (A.n_expected && n != A.n_expected) return fail(kDecWrongLen);
    const uint32_t rsym = 1u << blk[7];
    const uint8_t *pl_ = blk + kHeaderBytes;
    if (plen < 4) return fail(kDecPayloadSmall);
    const uint32_t tc = (uint32_t)load_le(pl_, 4);
    const uint64_t table_bytes = 4 + (uint64_t)tc * 5;
    if (tc == 0) return fail(kDecTableEmpty);
    if (plen < table_bytes) return fail(kDecTableTrunc);
    if (tc > A.cap) return fail(kDecNoMem);
    uint32_t cnt[kMaxCodeLen + 1];
    for (int l = 0; l <= kMaxCodeLen; ++l) cnt[l] = 0;
    uint32_t prev = 0;
    for (uint32_t i = 0; i < tc; ++i) {
        const uint32_t sy = (uint32_t)load_le(pl_ + 4 + 5ull * i, 4);
        const uint8_t l = pl_[4 + 5ull * i + 4];
        if (i > 0 && sy <= prev) return fail(kDecSymOrder);
        if (sy > rsym) return fail(kDecSymRange);
        if (l < 1 || l > kMaxCodeLen) return fail(kDecLenRange);
        ++cnt[l];
        prev = sy;
    }
    double kraft = 0.0;
    for (int l = 1; l <= kMaxCodeLen; ++l) {
        const double term = ldexp(1.0, -l);
        for (uint32_t k = 0; k < cnt[l]; ++k) kraft = dadd(kraft, term);
    }
    if (kraft > 1.0 + 1e-9) return fail(kDecOverfull);
    if (plen < table_bytes + nout * 16) return fail(kDecLenMismatch);
}

__global__ void fd_scan(FdArgs A, DecTables T, int planes) {
    pdl_begin();
    const int pl = blockIdx.x * blockDim.x + threadIdx.x;
    if (pl >= planes || A.err[pl] || (A.only && !A.only[pl])) return;
    const uint8_t *blk = A.arena + A.blk_off[pl];
    auto fail = [&](uint32_t e) { A.err[pl] = e; };
    const uint8_t pred_kind = blk[6];
    const int qb = blk[7];
    const uint64_t n = load_le(blk + 8, 8);
    const double eb = __longlong_as_double((long long)load_le(blk + 16, 8));
    const double q = dmul(2.0, eb);
    const uint64_t nout = load_le(blk + 24, 8);
    const uint64_t plen = load_le(blk + 32, 8);
    const long long half = 1ll << (qb - 1);
    const uint32_t rsym = 1u << qb;
    const uint32_t tc = (uint32_t)load_le(blk + kHeaderBytes, 4);
    const uint64_t table_bytes = 4 + 5ull * tc;
    const uint64_t sbytes = plen - table_bytes - 16 * nout;
    const uint64_t sbits = sbytes * 8;
    const uint32_t *stream = reinterpret_cast<const uint32_t *>(blk + kHeaderBytes + table_bytes);
    const uint8_t *orec = blk + kHeaderBytes + table_bytes + sbytes;
    const uint32_t *lut = T.lut + (uint64_t)pl * (1u << kLutBits);
    const uint64_t *first = T.first + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *count = T.count + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *basei = T.basei + (uint64_t)pl * (kMaxCodeLen + 1);
    const uint32_t *sorted = T.sorted + (uint64_t)pl * T.cap;
    const uint32_t maxlen = T.meta[4 * pl];
    IndexRec *rec = A.rec + (uint64_t)pl * A.stride;
    uint32_t nr = 0;
    uint64_t next_mark = kFdBits;
    BitWindow bw;
    bw.init(stream, 0);
    uint64_t bp = 0, i = 0, ocur = 0;
    uint32_t last = rsym;
    double d1 = 0.0, d2 = 0.0;
    // the reference's value of element i for symbol es (codec.cpp:605-611)
    auto value = [&](uint32_t es) -> double {
        double pred;
        if (pred_kind == 0) pred = i > 0 ? d1 : 0.0;
        else pred = i == 0 ? 0.0 : (i == 1 ? d1 : predict_linear(d1, d2));
        const long long m = (long long)es - half;
        return eb == 0.0 ? pred : dadd(pred, dmul(q, (double)m));
    };
    while (i < n) {
        if (bp >= next_mark) { // a record at this token boundary
            if (nr < A.stride) rec[nr++] = IndexRec{d1, d2, bp, 0u, (uint32_t)ocur, last, (uint32_t)i};
            next_mark = (bp / kFdBits + 1) * kFdBits;
        }
        // prefix code (PrefixDecoder, codec.cpp:251-286): LUT, then long codes
        const uint64_t remain = sbits - bp;
        const uint32_t le = lut[bw.acc >> (64 - kLutBits)];
        uint32_t s = 0, l = le & 63;
        if (l) {
            s = le >> 6;
        } else {
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
        }
        if (l == 0) return fail(remain < maxlen ? kDecStreamTrunc : kDecInvalidCode);
        if (l > remain) return fail(kDecStreamTrunc);
        if ((int)l <= bw.n) bw.skip((int)l);
        else bw.init(stream, bp + l);
        bp += l;
        if (s == rsym) {
            if (last == rsym || last == kOutlierSym) return fail(kDecRunNoCode);
            // Elias gamma: zeros, a one, then the value's low bits
            const uint64_t g = peek64<false>(stream, bp);
            int zeros = g ? __clzll((long long)g) : 64;
            if (zeros > 63 || (g == 0 && sbits - bp > 64)) { // more than 63 zeros before the terminating one
                if (sbits - bp <= 63) return fail(kDecStreamTrunc);
                return fail(kDecRunRange);
            }
            if ((uint64_t)zeros + 1 > sbits - bp) return fail(kDecStreamTrunc);
            uint64_t v;
            if (zeros == 0) {
                v = 1;
            } else {
                const uint64_t vb = bp + zeros; // the value: the one + `zeros` bits
                if (vb + zeros + 1 > sbits) return fail(kDecStreamTrunc);
                const uint64_t h = peek64<false>(stream, vb);
                v = h >> (63 - zeros);
            }
            bp += 2 * (uint64_t)zeros + 1;
            bw.init(stream, bp);
            if (v > n - i) return fail(kDecRunOverflow);
            // v repeats of `last`: a constant run needs no per-element work
            if (pred_kind == 0) {
                uint64_t k = 0;
                while (k < v) {
                    const double x = value(last);
                    if (bits_of(x) == bits_of(d1) && i > 0) { // constant from here on
                        d2 = d1;
                        i += v - k;
                        k = v;
                        break;
                    }
                    d2 = d1;
                    d1 = x;
                    ++i;
                    ++k;
                }
            } else {
                for (uint64_t k = 0; k < v; ++k) {
                    const double x = value(last);
                    d2 = d1;
                    d1 = x;
                    ++i;
                }
            }
            continue;
        }
        last = s;
        double x;
        if (s == kOutlierSym) {
            if (ocur >= nout) return fail(kDecOutExhausted);
            if (load_le(orec + 16 * ocur, 8) != i) return fail(kDecOutPos);
            x = __longlong_as_double((long long)load_le(orec + 16 * ocur + 8, 8));
            ++ocur;
        } else {
            x = value(s);
        }
        d2 = d1;
        d1 = x;
        ++i;
    }
    if (ocur != nout) return fail(kDecOutUnused);
    if ((bp + 7) / 8 != sbytes) return fail(kDecStreamLen);
    A.nrec[pl] = nr;
}

} // namespace qcb
