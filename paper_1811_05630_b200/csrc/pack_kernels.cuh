// pack_kernels.cuh -- codebook construction and QCB1 block assembly.
//
// E3 enc_codebook: histogram -> freq (sorted by symbol, codec.cpp:484-488)
//    -> two-queue Huffman lengths (codec.cpp:168-229) -> canonical codes
//    (codec.cpp:233-249) -> exact block size.
// E5 enc_pack: header (codec.cpp:343-357), table (codec.cpp:508-512),
//    MSB-first code stream with Elias-gamma run lengths (codec.cpp:513-520),
//    outlier records (codec.cpp:521-524), decode index bit positions.
#pragma once

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "decode_kernels.cuh" // DecTables
#include "enc_tiles.cuh" // carry_of / tile_carry
#include "chain_scan.cuh"

namespace qcb {

struct CodeBook {
    // inputs (from E2 / E1)
    uint32_t *hist;            // [plane][rsym+1], zeroed again by E3
    const uint32_t *hspecial;  // [plane][2]
    const uint32_t *symrange;  // [plane][2]
    const uint64_t *gamma_bits;// [plane]
    const uint32_t *ocount;    // [plane]
    // scratch, [plane][cap]
    uint32_t *sym;             // symbols in ascending order
    uint64_t *cnt;             // their counts
    uint8_t *len;              // code lengths
    uint64_t *code;            // canonical codes
    uint64_t *key;             // sort keys (count << 25 | sym)
    uint64_t *ncnt;            // [plane][2cap] node counts
    int32_t *parent;           // [plane][2cap]
    // outputs, [plane]
    uint32_t *nsym;
    uint64_t *stream_bits;
    uint64_t *block_bytes;
    uint64_t *slot_bytes;      // 16 + round_up(block_bytes, 16) + decode index (common.cuh)
    uint32_t *err;             // nonzero: codec error code
    uint64_t cap;
    int qb;
    uint64_t L;                // plane length
    int log2C;                 // fine checkpoint spacing (the slot keeps a subset, index_select)
    DecTables dec;             // optional: decode tables of the new blocks
    uint8_t *zero_arena = nullptr; // fixed slots (plane p at p * zero_W): zero the plane's slot for the packer
    uint64_t zero_W = 0;
    unsigned long long *trace = nullptr; // debug phase stamps
};

enum : uint32_t { kErrDepth = 1 };

// Bitonic sort of n keys (n <= len of `a`, padded with ~0 to a power of two).
__device__ void block_bitonic(uint64_t *a, uint32_t n) {
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t i = n + threadIdx.x; i < m; i += blockDim.x) a[i] = ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

constexpr uint32_t kSmallN = 1024; // alphabets up to this size stay in shared memory

// Decode tables of a block (PrefixDecoder, codec.cpp:251-273) written by the
// encoder itself, so the next gate pass needs no table-parsing kernel.
// entries: n symbols in ascending order with code lengths and canonical codes.
__device__ void emit_dec_tables(const DecTables &T, int pl, uint32_t n, const uint32_t *sym, const uint8_t *len,
                                const uint64_t *code, const uint32_t *lcount, const uint64_t *lfirst0) {
    uint32_t *lut = T.lut + (uint64_t)pl * (1u << kLutBits);
    __shared__ uint32_t basei[kMaxCodeLen + 2];
    __shared__ uint32_t s_maxlen;
    if (threadIdx.x == 0) { // shared memory only; the tables are written in parallel below
        uint32_t b = 0, maxlen = 0;
        basei[0] = 0;
        for (int l = 1; l <= kMaxCodeLen; ++l) {
            basei[l] = b;
            b += lcount[l];
            if (lcount[l]) maxlen = l;
        }
        s_maxlen = maxlen;
        T.meta[4 * pl] = maxlen;
        T.meta[4 * pl + 1] = n;
    }
    __syncthreads();
    for (int l = threadIdx.x; l <= kMaxCodeLen; l += blockDim.x) {
        const bool any = l > 0 && lcount[l];
        T.first[(uint64_t)pl * (kMaxCodeLen + 1) + l] = any ? lfirst0[l] : 0;
        T.count[(uint64_t)pl * (kMaxCodeLen + 1) + l] = l > 0 ? lcount[l] : 0;
        T.basei[(uint64_t)pl * (kMaxCodeLen + 1) + l] = basei[l];
    }
    const int lmax = (int)min((uint32_t)kLutBits, s_maxlen);
    uint32_t *sorted = T.sorted + (uint64_t)pl * T.cap;
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
        const int l = len[r];
        // (len, sym) order: position within the length = code - first code
        sorted[basei[l] + (uint32_t)(code[r] - lfirst0[l])] = sym[r];
    }
    __syncthreads();
    // short codes -> LUT: every entry decodes its own kLutBits-bit window
    // (canonical first/count per length), one store per entry
    for (uint32_t k = threadIdx.x; k < (1u << kLutBits); k += blockDim.x) {
        uint32_t e = 0;
        for (int l = 1; l <= lmax; ++l) {
            const uint32_t c = lcount[l];
            if (!c) continue;
            const uint64_t w = (uint64_t)(k >> (kLutBits - l));
            if (w >= lfirst0[l] && w - lfirst0[l] < c) {
                e = (sorted[basei[l] + (uint32_t)(w - lfirst0[l])] << 6) | (uint32_t)l;
                break;
            }
        }
        lut[k] = e;
    }
}

// Two-queue Huffman merge (codec.cpp:168-229; ties prefer the leaf queue) by
// one thread, with both queue heads held in 4-deep register windows that
// are refilled three picks ahead, so the shared-memory latency stays off the
// serial compare/select path.  nc[0, n) = leaf counts (sorted by (count,
// sym)); internal node counts are appended at nc[n...]; par[] receives the
// parent of every node (root: -1).  Returns the node count.
template <class U32P, class I32P>
__device__ uint32_t huff_merge_serial(U32P nc, I32P par, uint32_t n) {
    uint32_t lp = 0, ip = n, nodes = n;
    uint32_t L[4], I[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        L[k] = lp + k < n ? nc[lp + k] : 0u;
        I[k] = 0u;
    }
    while ((n - lp) + (nodes - ip) >= 2) {
        uint32_t v[2], q[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const bool leaf = lp < n && (ip >= nodes || L[0] <= I[0]);
            if (leaf) {
                v[k] = L[0];
                q[k] = lp;
                ++lp;
                L[0] = L[1];
                L[1] = L[2];
                L[2] = L[3];
                L[3] = lp + 3 < n ? nc[lp + 3] : 0u;
            } else {
                v[k] = I[0];
                q[k] = ip;
                ++ip;
                I[0] = I[1];
                I[1] = I[2];
                I[2] = I[3];
                I[3] = ip + 3 < nodes ? nc[ip + 3] : 0u;
            }
        }
        const uint32_t sum = v[0] + v[1];
        nc[nodes] = sum;
        par[q[0]] = (int32_t)nodes;
        par[q[1]] = (int32_t)nodes;
        // the new node joins the internal window if it lands inside it
        const uint32_t d = nodes - ip;
        if (d == 0) I[0] = sum;
        else if (d == 1) I[1] = sum;
        else if (d == 2) I[2] = sum;
        else if (d == 3) I[3] = sum;
        ++nodes;
    }
    par[nodes - 1] = -1;
    return nodes;
}

// The same merge for larger alphabets (nc[0, n) = leaf counts, par[0, n) =
// -1 on entry) by one warp, up to 32 picks per round.  Internal nodes are
// appended in non-decreasing order behind every node that already exists, so
// as long as a round only takes internal nodes that existed when it started,
// its picks are the plain merge of two sorted lists (leaves, known internal
// nodes): lane j finds pick j by a merge-path search.  The round stops at the
// first pick that would need a node created in the same round; picks are
// paired in order into new nodes.
template <class U32P, class I32P>
__device__ void huff_merge_batched(U32P nc, I32P par, uint32_t n, int tid) {
    uint32_t lp = 0, ip = n, nodes = n;
    while ((n - lp) + (nodes - ip) >= 2) {
        const uint32_t nA = n - lp, nB = nodes - ip, j = (uint32_t)tid;
        // leaves among the first j picks (ties: the leaf goes first)
        uint32_t lo = j > nB ? j - nB : 0u, hi = tmin<uint32_t>(j, nA);
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (nc[lp + mid] <= nc[ip + j - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        const uint32_t cL = lo, cI = j - lo;
        // pick j exists among the known nodes, and no node created in this
        // round can be the internal head yet (j < 2: none exists)
        const bool valid = j < nA + nB && (cI < nB || j < 2);
        const bool take_leaf = cL < nA && (cI >= nB || nc[lp + cL] <= nc[ip + cI]);
        const uint32_t idx = valid ? (take_leaf ? lp + cL : ip + cI) : 0u;
        const uint32_t val = valid ? nc[idx] : 0u;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        uint32_t P = vm == 0xffffffffu ? 32u : (uint32_t)(__ffs(~vm) - 1); // leading valid picks
        P &= ~1u;
        const uint32_t pidx = __shfl_xor_sync(0xffffffffu, idx, 1);
        const uint32_t pval = __shfl_xor_sync(0xffffffffu, val, 1);
        const unsigned lm = __ballot_sync(0xffffffffu, valid && take_leaf) & (P >= 32 ? 0xffffffffu : ((1u << P) - 1u));
        __syncwarp(); // every lane has read nc before the new nodes land
        if (j < P && (j & 1) == 0) {
            const uint32_t k = nodes + (j >> 1);
            nc[k] = val + pval;
            par[idx] = (int32_t)k;
            par[pidx] = (int32_t)k;
        }
        const uint32_t nl = (uint32_t)__popc(lm);
        lp += nl;
        ip += P - nl;
        nodes += P >> 1;
        __syncwarp();
    }
    if (tid == 0) par[nodes - 1] = -1;
    __syncwarp();
}
constexpr uint32_t kDepthSerialN = 64; // larger (shared-memory) alphabets: depths by pointer jumping

// One block per plane.  Working arrays live in shared memory for alphabets of
// up to kSmallN symbols (the serial two-queue merge then runs on smem), in
// per-plane global scratch beyond that.
__device__ __forceinline__ void codebook_plane(const CodeBook &B, int planes, int pl) {
    if (pl >= planes) return;
    const int tid = threadIdx.x;
    auto stamp = [&](int k) { // debug phase trace (B.trace: 16 stamps per plane)
        if (B.trace && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            B.trace[16ull * pl + k] = t;
        }
    };
    stamp(0);
    using Scan = cub::BlockScan<int, 256>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint64_t k_s[kSmallN];
    __shared__ uint32_t sym_s[kSmallN], cnt_s[kSmallN];
    __shared__ uint32_t nc_s[2 * kSmallN];
    __shared__ int32_t par_s[2 * kSmallN];
    __shared__ uint8_t len_s[kSmallN];
    __shared__ uint64_t code_s[kSmallN];
    __shared__ uint32_t s_n, s_nodes, s_lmax;
    __shared__ uint32_t lcount[kMaxCodeLen + 2];
    __shared__ uint64_t lfirst[kMaxCodeLen + 2], lfirst0[kMaxCodeLen + 2];
    __shared__ unsigned long long s_bits;
    __shared__ uint32_t s_err;
    __shared__ uint64_t s_slotb;

    const uint32_t rsym = 1u << B.qb;
    uint32_t *hist = B.hist + (uint64_t)pl * ((uint64_t)rsym + 1);
    const uint64_t cap = B.cap;
    const uint32_t h0 = B.hspecial[2 * pl], hrun = B.hspecial[2 * pl + 1];
    const uint32_t smin = B.symrange[2 * pl], smax = B.symrange[2 * pl + 1];
    // alphabet size first (decides smem vs global working arrays): every
    // thread owns a contiguous slice of the symbol range, counts its nonzero
    // bins, and one block scan places each slice in the ascending list
    const uint64_t R = smin <= smax ? (uint64_t)smax - smin + 1 : 0;
    const uint64_t per = (R + 255) / 256;
    const uint64_t b0 = (uint64_t)smin + tid * per, b1 = tmin<uint64_t>(b0 + per, (uint64_t)smin + R);
    int mine = 0;
    for (uint64_t s2 = b0; s2 < b1; ++s2) mine += hist[s2] != 0;
    int pos_r = 0, tot_r = 0;
    Scan(scan_tmp).ExclusiveSum(mine, pos_r, tot_r);
    if (tid < kMaxCodeLen + 2) lcount[tid] = 0;
    const uint32_t n = (h0 ? 1u : 0u) + (uint32_t)tot_r + (hrun ? 1u : 0u);
    const bool small = n <= kSmallN;
    if (B.trace && tid == 0) B.trace[16ull * pl + 15] = n; // debug: alphabet size
    uint32_t *sym = small ? sym_s : B.sym + pl * cap;
    uint32_t *cnt = small ? cnt_s : reinterpret_cast<uint32_t *>(B.cnt + pl * cap);
    uint8_t *len = small ? len_s : B.len + pl * cap;
    uint64_t *code = small ? code_s : B.code + pl * cap;
    uint64_t *keys = small ? k_s : B.key + pl * cap * 2;
    uint32_t *nc = small ? nc_s : reinterpret_cast<uint32_t *>(B.ncnt + pl * cap * 2);
    int32_t *par = small ? par_s : B.parent + pl * cap * 2;

    if (tid == 0) {
        s_n = (h0 ? 1u : 0u) + (uint32_t)tot_r;
        s_lmax = 0;
        s_bits = 0;
        s_err = 0;
        if (h0) {
            sym[0] = kOutlierSym;
            cnt[0] = h0;
        }
    }
    stamp(1);
    // 1) compaction of the symbol range, ascending (freq, codec.cpp:484-488)
    {
        uint32_t o = (h0 ? 1u : 0u) + (uint32_t)pos_r;
        for (uint64_t s2 = b0; s2 < b1; ++s2) {
            const uint32_t v = hist[s2];
            if (v) {
                sym[o] = (uint32_t)s2;
                cnt[o] = v;
                ++o;
                hist[s2] = 0; // restore the zero invariant
            }
        }
    }
    __syncthreads();
    if (tid == 0 && hrun) {
        sym[s_n] = rsym;
        cnt[s_n] = hrun;
        s_n += 1;
    }
    __syncthreads();
    if (n == 0) { // unreachable for L >= 1
        if (tid == 0) B.err[pl] = 0;
        return;
    }
    stamp(2);
    // 2) leaves sorted by (count, symbol)
    for (uint32_t i = tid; i < n; i += 256) keys[i] = ((uint64_t)cnt[i] << 25) | sym[i];
    __syncthreads();
    if (n > 1) block_bitonic(keys, n);
    stamp(3);
    // 3) two-queue merge (codec.cpp:168-229; ties prefer the leaf queue).
    if (tid < 32) {
        if (n == 1) {
            if (tid == 0) par[0] = -1;
        } else {
            for (uint32_t i = tid; i < n; i += 32) {
                nc[i] = (uint32_t)(keys[i] >> 25);
                par[i] = -1;
            }
            __syncwarp();
            // small alphabets (skewed trees, one pick pair per step): one
            // thread; larger ones: the warp-batched merge
            if (n <= 64) {
                if (tid == 0) huff_merge_serial(nc, par, n);
                __syncwarp();
            } else {
                huff_merge_batched(nc, par, n, tid);
            }
        }
        if (tid == 0 && n > 1) {
            const uint32_t nodes = 2 * n - 1;
            s_nodes = nodes;
            if (!small || n <= kDepthSerialN) { // large or tiny alphabet: depths top-down, serially
                nc[nodes - 1] = 0;
                for (int64_t v = (int64_t)nodes - 2; v >= 0; --v) nc[v] = nc[par[v]] + 1;
            }
        }
    }
    __syncthreads();
    // depths by pointer jumping (parents have larger indices; root -> 0),
    // stored in nc
    if (n > kDepthSerialN && small) {
        const uint32_t nodes = s_nodes;
        for (uint32_t v = tid; v < nodes; v += 256) {
            nc[v] = par[v] < 0 ? 0u : 1u; // distance to the current ancestor
        }
        __syncthreads();
        for (int round = 0; round < 32; ++round) {
            int changed = 0;
            for (uint32_t v = tid; v < nodes; v += 256) {
                const int32_t a = par[v];
                if (a >= 0 && par[a] >= 0) changed = 1;
            }
            if (!__syncthreads_or(changed)) break;
            // one jump: read everything first, then write (separate phases)
            uint32_t nd[(2 * kSmallN + 255) / 256];
            int32_t na[(2 * kSmallN + 255) / 256];
            int q = 0;
            for (uint32_t v = tid; v < nodes && q < (2 * kSmallN + 255) / 256; v += 256, ++q) {
                const int32_t a = par[v];
                if (a >= 0 && par[a] >= 0) { // stop at the root: -1 marks only the root itself
                    nd[q] = nc[v] + nc[a];
                    na[q] = par[a];
                } else {
                    nd[q] = nc[v];
                    na[q] = a;
                }
            }
            __syncthreads();
            q = 0;
            for (uint32_t v = tid; v < nodes && q < (2 * kSmallN + 255) / 256; v += 256, ++q) {
                nc[v] = nd[q];
                par[v] = na[q];
            }
            __syncthreads();
        }
    }
    __syncthreads();
    stamp(4);
    // 4) lengths in symbol order
    for (uint32_t i = tid; i < n; i += 256) {
        const uint32_t s = (uint32_t)(keys[i] & ((1ull << 25) - 1));
        const uint32_t depth = n == 1 ? 1u : nc[i];
        if (depth < 1 || depth > (uint32_t)kMaxCodeLen) atomicExch(&s_err, kErrDepth);
        uint32_t lo = 0, hi = n; // rank of s in the ascending symbol list
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (sym[mid] < s) lo = mid + 1;
            else hi = mid;
        }
        const uint8_t l = (uint8_t)tmin<uint32_t>(depth, kMaxCodeLen);
        len[lo] = l;
        atomicAdd(&lcount[l], 1u);
        atomicMax(&s_lmax, (uint32_t)l);
        atomicAdd(&s_bits, (unsigned long long)cnt[lo] * l);
    }
    __syncthreads();
    stamp(5);
    // 5) canonical codes (codec.cpp:233-249): (len, sym) order == symbol
    //    order within a length
    if (tid == 0) {
        uint64_t c = 0;
        int prev = -1;
        const int lm = (int)s_lmax;
        for (int l = 0; l <= kMaxCodeLen; ++l) lfirst[l] = 0;
        for (int l = 1; l <= lm; ++l) {
            if (!lcount[l]) continue;
            if (prev >= 0) c <<= (l - prev);
            lfirst[l] = c;
            c += lcount[l];
            prev = l;
        }
        for (int l = 0; l <= kMaxCodeLen; ++l) lfirst0[l] = lfirst[l];
        const uint64_t bits = s_bits + B.gamma_bits[pl];
        // outliers are never run-collapsed: one outlier token (symbol 0) per
        // outlier, so h0 is the plane's outlier count (codec.cpp:460-488)
        const uint64_t payload = 4 + 5ull * n + (bits + 7) / 8 + 16ull * h0;
        const uint64_t bytes = kHeaderBytes + payload;
        B.nsym[pl] = n;
        B.stream_bits[pl] = bits;
        B.block_bytes[pl] = bytes;
        const uint64_t slotb =
            16 + ((bytes + 15) & ~15ull) + ((index_records(B.L, bytes, B.log2C) * sizeof(IndexRec) + 15) & ~15ull);
        B.slot_bytes[pl] = slotb;
        B.err[pl] = s_err;
        s_slotb = slotb;
    }
    __syncthreads();
    if (B.zero_arena) { // stream words are OR-combined at chunk seams
        uint4 *w = reinterpret_cast<uint4 *>(B.zero_arena + (uint64_t)pl * B.zero_W);
        for (uint64_t k = tid; k < s_slotb / 16; k += 256) w[k] = make_uint4(0, 0, 0, 0);
    }
    // canonical codes in symbol order, one warp: a symbol's code is its
    // length's next free code plus its rank among equal lengths in the group
    if (tid < 32) {
        for (uint32_t g0 = 0; g0 < n; g0 += 32) {
            const uint32_t r = g0 + tid;
            const int l = r < n ? len[r] : 0;
            const unsigned peers = __match_any_sync(0xffffffffu, l);
            const uint32_t rank = __popc(peers & ((1u << tid) - 1));
            if (r < n) code[r] = lfirst[l] + rank;
            __syncwarp();
            if (r < n && rank == 0) lfirst[l] += __popc(peers);
            __syncwarp();
        }
    }
    __syncthreads();
    stamp(6);
    if (small) { // publish the codebook for the packer
        for (uint32_t r = tid; r < n; r += 256) {
            B.sym[pl * cap + r] = sym_s[r];
            B.len[pl * cap + r] = len_s[r];
            B.code[pl * cap + r] = code_s[r];
        }
    }
    stamp(7);
    if (B.dec.lut) emit_dec_tables(B.dec, pl, n, sym, len, code, lcount, lfirst0);
    stamp(8);
    if (B.trace && tid == 0) B.trace[16ull * pl + 9] = n;
}
__global__ void __launch_bounds__(256) enc_codebook(CodeBook B, int planes) {
    pdl_begin();
    codebook_plane(B, planes, blockIdx.x);
}
// Tokens (tok_emit) and codebooks in one grid: both consume only tok_count's
// outputs, so the codebook blocks (first in the grid, one per plane, short
// serial phases) overlap the tile-parallel token emission.
__global__ void __launch_bounds__(256) tok_emit_codebook(TokArgs A, CodeBook B, int planes) {
    pdl_begin();
    if ((int)blockIdx.x < planes) codebook_plane(B, planes, blockIdx.x);
    else tok_emit_tile(A, planes, (int)blockIdx.x - planes);
}

// ------------------------------------------------------------------ E5
struct PackArgs {
    const uint32_t *tsym, *trep, *ntok;   // tokens [plane][L+1]
    const uint32_t *cb_sym;               // [plane][cap]
    const uint8_t *cb_len;
    const uint64_t *cb_code;
    const uint32_t *nsym;
    const uint64_t *stream_bits, *block_bytes, *slot_off;
    const uint32_t *opos;                 // [plane][L]
    const double *oval;
    const uint32_t *ocount;
    const PlaneParams *params;
    IndexRec *index;                      // [plane][nidx]
    uint8_t *arena;
    uint64_t arena_cap;                   // bytes usable in `arena`
    uint32_t *overflow;                   // set when the batch does not fit
    uint64_t *blk_off;                    // out: block start in the arena
    uint64_t L, cap;
    int log2C, qb, mode, predictor;
    int planes_total;                     // slot_off[planes_total] = bytes needed
    unsigned long long *lb;               // != nullptr: chunk bit offsets by decoupled look-back
    uint32_t lb_epoch;                    //   (no pack_count pass; slots pre-zeroed)
};

__device__ __forceinline__ void put_bits_smem(uint32_t *w, uint32_t o, uint64_t v, int n) {
    // MSB-first: the first bit of v (bit n-1) lands at stream bit o
    while (n > 0) {
        const uint32_t wi = o >> 5, b = o & 31;
        const int take = min(n, 32 - (int)b);
        const uint32_t chunk = (uint32_t)((v >> (n - take)) & ((1ull << take) - 1));
        atomicOr(&w[wi], chunk << (32 - b - take));
        o += take;
        n -= take;
    }
}

__device__ __forceinline__ void store_le(uint8_t *p, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

constexpr int kPackTok = 1024;                 // tokens per pack block
constexpr int kPackWords = kPackTok * 120 / 32 + 2;
constexpr int kCodeWin = 2048;                 // dense shared codebook window

// Per-block view of a plane's codebook (codec.cpp:493-496 code_of): a dense
// shared-memory window over the symbol range when it is narrow, else a
// binary search over the sorted symbol list.
struct SCodebook {
    uint64_t code[kCodeWin];
    uint8_t len[kCodeWin];
    uint64_t code0, coderun;
    uint8_t len0, lenrun;
    uint32_t lo, span, n;
    bool dense;
};

__device__ void load_codebook(SCodebook &C, const PackArgs &A, int pl) {
    const uint32_t n = A.nsym[pl];
    const uint32_t *cs = A.cb_sym + pl * A.cap;
    const uint8_t *cl = A.cb_len + pl * A.cap;
    const uint64_t *cc = A.cb_code + pl * A.cap;
    const uint32_t rsym = 1u << A.qb;
    // literal symbols occupy ranks [r0, r1): 0 first, RUN last when present
    const uint32_t r0 = (n && cs[0] == kOutlierSym) ? 1 : 0;
    const uint32_t r1 = (n && cs[n - 1] == rsym) ? n - 1 : n;
    if (threadIdx.x == 0) {
        C.n = n;
        C.len0 = 0;
        C.lenrun = 0;
        if (r0) { C.code0 = cc[0]; C.len0 = cl[0]; }
        if (r1 < n) { C.coderun = cc[n - 1]; C.lenrun = cl[n - 1]; }
        C.lo = r1 > r0 ? cs[r0] : 0;
        C.span = r1 > r0 ? cs[r1 - 1] - cs[r0] + 1 : 0;
        C.dense = C.span <= (uint32_t)kCodeWin;
    }
    __syncthreads();
    if (C.dense) {
        for (uint32_t k = threadIdx.x; k < C.span; k += blockDim.x) C.len[k] = 0;
        __syncthreads();
        for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            C.code[cs[r] - C.lo] = cc[r];
            C.len[cs[r] - C.lo] = cl[r];
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void lookup_code(const SCodebook &C, const PackArgs &A, int pl, uint32_t s,
                                            uint64_t &code, int &len) {
    const uint32_t rsym = 1u << A.qb;
    if (s == kOutlierSym) { code = C.code0; len = C.len0; return; }
    if (s == rsym) { code = C.coderun; len = C.lenrun; return; }
    if (C.dense) { code = C.code[s - C.lo]; len = C.len[s - C.lo]; return; }
    const uint32_t *cs = A.cb_sym + pl * A.cap;
    uint32_t lo = 0, hi = C.n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cs[mid] < s) lo = mid + 1;
        else hi = mid;
    }
    code = A.cb_code[pl * A.cap + lo];
    len = A.cb_len[pl * A.cap + lo];
}

// token -> (code, code length, gamma length): codec.cpp:513-520
__device__ __forceinline__ uint32_t token_bits(const SCodebook &C, const PackArgs &A, int pl, uint32_t s,
                                               uint32_t rep, uint64_t &code, int &len, int &glen) {
    lookup_code(C, A, pl, s, code, len);
    glen = s == (1u << A.qb) ? 2 * bit_width64(rep) - 1 : 0;
    return (uint32_t)(len + glen);
}

// P1: bits of every 1024-token chunk (grid: planes x chunks).
__device__ __forceinline__ void pack_count_item(const PackArgs &A, int planes, int nck, int32_t *cbits, int pl, int c) {
    if (pl >= planes) return;
    // zero this block's share of the plane's arena slot (stream words are
    // OR-combined at chunk seams by pack_write); skipped when the batch
    // does not fit -- pack_write then reports the overflow
    if (A.slot_off[A.planes_total] + 64 <= A.arena_cap) {
        const uint64_t s0 = A.slot_off[pl], s1 = A.slot_off[pl + 1]; // 16-byte aligned slots
        const uint64_t nw = (s1 - s0) / 16, per = (nw + nck - 1) / nck;
        uint4 *w = reinterpret_cast<uint4 *>(A.arena + s0);
        for (uint64_t k = (uint64_t)c * per + threadIdx.x; k < tmin<uint64_t>(nw, (uint64_t)(c + 1) * per);
             k += blockDim.x)
            w[k] = make_uint4(0, 0, 0, 0);
    }
    const uint32_t ntok = A.ntok[pl];
    const uint32_t t0 = (uint32_t)c * kPackTok;
    if (t0 >= ntok) {
        if (threadIdx.x == 0) cbits[(uint64_t)pl * nck + c] = 0;
        return;
    }
    __shared__ SCodebook C;
    load_codebook(C, A, pl);
    const uint32_t tn = tmin<uint32_t>(kPackTok, ntok - t0);
    const uint32_t *ts = A.tsym + (uint64_t)pl * (A.L + 1);
    const uint32_t *tr = A.trep + (uint64_t)pl * (A.L + 1);
    uint32_t bits = 0;
    for (uint32_t k = threadIdx.x; k < tn; k += blockDim.x) {
        uint64_t code;
        int len, glen;
        bits += token_bits(C, A, pl, ts[t0 + k], tr[t0 + k], code, len, glen);
    }
    using Red = cub::BlockReduce<uint32_t, 256>;
    __shared__ typename Red::TempStorage rt;
    const uint32_t tot = Red(rt).Sum(bits);
    if (threadIdx.x == 0) cbits[(uint64_t)pl * nck + c] = (int32_t)tot;
}

// Zero the batch's arena range (stream words are OR-combined at chunk seams).
__global__ void arena_zero(uint8_t *arena, uint64_t cap, const uint64_t *total_ptr) {
    pdl_begin();
    const uint64_t total = *total_ptr + 64;
    if (total > cap) return;
    uint4 *w = reinterpret_cast<uint4 *>(arena);
    const uint64_t nw = (total + 15) / 16;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nw; k += (uint64_t)gridDim.x * blockDim.x)
        w[k] = make_uint4(0, 0, 0, 0);
}


// P2: header + table (chunk 0), stream bits of every chunk, outlier records,
// decode-index bit positions (grid: planes x chunks).
__device__ __forceinline__ void pack_write_item(const PackArgs &A, int planes, int nck, const int32_t *coff,
                                                const int32_t *cbits, int pl, int c) {
    if (pl >= planes) return;
    const int tid = threadIdx.x;
    if (A.slot_off[A.planes_total] + 64 > A.arena_cap) {
        if (tid == 0) atomicExch(A.overflow, 1u);
        return;
    }
    const uint32_t ntok = A.ntok[pl];
    const uint32_t t0 = (uint32_t)c * kPackTok;
    const uint32_t nchk = (ntok + kPackTok - 1) / kPackTok;
    if (c >= (int)nchk) return;
    __shared__ SCodebook C;
    __shared__ uint32_t words[kPackWords];
    __shared__ uint32_t toff[kPackTok + 1];
    __shared__ uint32_t s_jlo, s_jhi;
    using Scan = cub::BlockScan<uint32_t, 256>;
    __shared__ typename Scan::TempStorage scan_tmp;

    const uint32_t n = A.nsym[pl];
    const uint64_t pre = kHeaderBytes + 4 + 5ull * n;
    const uint64_t shift = (16 - (pre & 15)) & 15;
    const uint64_t off = A.slot_off[pl] + shift;
    uint8_t *blk = A.arena + off;
    uint8_t *stream = blk + pre; // 16-byte aligned
    const uint64_t bits = A.stream_bits[pl];
    const uint64_t sbytes = (bits + 7) / 8;
    const uint32_t nout = A.ocount[pl];
    const uint32_t rsym = 1u << A.qb;
    const uint64_t nidx = (A.L >> A.log2C) + 1;
    const uint32_t nchunks_idx = (uint32_t)((A.L + (1ull << A.log2C) - 1) >> A.log2C);
    IndexRec *idx = A.index + pl * nidx;
    auto put_rec = [&](uint32_t j, uint64_t bitpos) { idx[j].bitpos = bitpos; };

    if (c == 0) {
        const uint64_t payload = 4 + 5ull * n + sbytes + 16ull * nout;
        const uint32_t *cs = A.cb_sym + pl * A.cap;
        const uint8_t *cl = A.cb_len + pl * A.cap;
        if (tid == 0) {
            A.blk_off[pl] = off;
            blk[0] = 'Q'; blk[1] = 'C'; blk[2] = 'B'; blk[3] = '1';
            blk[4] = 1;
            blk[5] = (uint8_t)A.mode;
            blk[6] = (uint8_t)A.predictor;
            blk[7] = (uint8_t)A.qb;
            store_le(blk + 8, A.L, 8);
            store_le(blk + 16, bits_of(A.params[pl].eb), 8);
            store_le(blk + 24, nout, 8);
            store_le(blk + 32, payload, 8);
            store_le(blk + 40, n, 4);
            idx[0].bitpos = 0;
            idx[0].tok = 0;
            idx[0].run_left = 0;
            idx[0].ocur = 0;
            idx[0].last_lit = rsym;
        }
        for (uint32_t r = tid; r < n; r += 256) {
            store_le(blk + 44 + 5ull * r, cs[r], 4);
            blk[44 + 5ull * r + 4] = cl[r];
        }
        // outlier records (u64 pos, f64 value), LE, after the stream
        uint8_t *orec = stream + sbytes;
        const uint32_t *op = A.opos + pl * A.L;
        const double *ov = A.oval + pl * A.L;
        for (uint32_t k = tid; k < nout; k += 256) {
            store_le(orec + 16ull * k, op[k], 8);
            store_le(orec + 16ull * k + 8, bits_of(ov[k]), 8);
        }
    }
    load_codebook(C, A, pl);
    const uint32_t tn = tmin<uint32_t>(kPackTok, ntok - t0);
    const uint32_t *ts = A.tsym + (uint64_t)pl * (A.L + 1);
    const uint32_t *tr = A.trep + (uint64_t)pl * (A.L + 1);
    uint64_t tcode[4];
    int tlen[4], glen[4];
    uint32_t tbits[4];
    for (int e = 0; e < 4; ++e) {
        const uint32_t k = tid * 4 + e;
        tbits[e] = 0;
        tlen[e] = glen[e] = 0;
        tcode[e] = 0;
        if (k < tn) tbits[e] = token_bits(C, A, pl, ts[t0 + k], tr[t0 + k], tcode[e], tlen[e], glen[e]);
    }
    uint32_t pos[4], tot;
    Scan(scan_tmp).ExclusiveSum(tbits, pos, tot);
    uint64_t base_bit;
    // the word buffer (bounded for any bit offset) and the token offsets do
    // not depend on where the chunk starts: the other warps fill them while
    // warp 0 looks back
    const uint32_t nw_max = (tot + 62) / 32;
    for (int e = 0; e < 4; ++e) {
        const uint32_t k = tid * 4 + e;
        if (k <= tn) toff[k] = pos[e];
    }
    if (tid == 255) toff[tn] = tot;
    if (A.lb) { // this chunk's bits -> look-back over the plane's earlier chunks
        __shared__ uint32_t s_base;
        if (tid < 32) {
            const uint32_t b = lookback_exclusive(A.lb + (uint64_t)pl * nck, A.lb_epoch, c, tot);
            if (tid == 0) s_base = b;
        } else {
            for (uint32_t w = tid - 32; w < nw_max; w += 224) words[w] = 0;
        }
        __syncthreads();
        base_bit = s_base;
    } else {
        for (uint32_t w = tid; w < nw_max; w += 256) words[w] = 0;
        base_bit = (uint64_t)(uint32_t)carry_of(coff, nck + 1, cbits, pl, c, nck, kScanSumExcl);
    }
    const uint32_t b0 = (uint32_t)(base_bit & 31);
    const uint32_t nwords = (b0 + tot + 31) / 32;
    __syncthreads();
    for (int e = 0; e < 4; ++e) {
        const uint32_t k = tid * 4 + e;
        if (k < tn) {
            put_bits_smem(words, b0 + pos[e], tcode[e], tlen[e]);
            if (glen[e]) put_bits_smem(words, b0 + pos[e] + tlen[e], tr[t0 + k], glen[e]);
        }
    }
    __syncthreads();
    // words -> global (big-endian byte order); the first and last words may
    // be shared with the neighbouring chunks (or outlier bytes): OR them
    uint32_t *gw = reinterpret_cast<uint32_t *>(stream);
    const uint64_t w0 = base_bit / 32;
    for (uint32_t w = tid; w < nwords; w += 256) {
        const uint32_t v = bswap32(words[w]);
        if (w == 0 || w == nwords - 1) atomicOr(&gw[w0 + w], v);
        else gw[w0 + w] = v;
    }
    // decode-index bit positions for checkpoints resuming in this chunk
    const bool last_chunk = c == (int)nchk - 1;
    if (nchunks_idx <= 16u * 256u) { // few records: every thread filters its share in parallel
        for (uint32_t j = 1 + tid; j < nchunks_idx; j += 256) {
            const uint32_t tk = idx[j].tok;
            if (tk >= t0 && (last_chunk || tk < t0 + tn))
                put_rec(j, tk >= t0 + tn ? base_bit + tot : base_bit + toff[tk - t0]);
        }
        return;
    }
    if (tid == 0) {
        uint32_t lo = 1, hi = nchunks_idx;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (idx[mid].tok < t0) lo = mid + 1;
            else hi = mid;
        }
        s_jlo = lo;
        hi = nchunks_idx;
        uint32_t lo2 = lo;
        while (lo2 < hi) {
            const uint32_t mid = (lo2 + hi) >> 1;
            if (last_chunk || idx[mid].tok < t0 + tn) lo2 = mid + 1;
            else hi = mid;
        }
        s_jhi = last_chunk ? nchunks_idx : lo2;
    }
    __syncthreads();
    for (uint32_t j = s_jlo + tid; j < s_jhi; j += 256) {
        const uint32_t tk = idx[j].tok;
        put_rec(j, tk >= t0 + tn ? base_bit + tot : base_bit + toff[tk - t0]);
    }
}

// Both packer grids are (plane, K) blocks; block (p, y) takes the plane's
// chunks y, y + K, ... and stops after the last chunk holding tokens (or
// slot words to zero).  A 2^20-element plane has 1025 chunk slots, but a
// well-compressed plane fills a handful: looping replaces hundreds of
// thousands of empty blocks.  A block takes its chunks in increasing order,
// and a plane's blocks are dispatched in order, so a look-back wait
// (pack_write) always targets a dispatched chunk.
__global__ void __launch_bounds__(256) pack_count(PackArgs A, int planes, int nck, int K, int32_t *cbits) {
    pdl_begin();
    const int pl = blockIdx.x / K, y = blockIdx.x % K;
    if (pl >= planes) return;
    const uint32_t ntok = A.ntok[pl];
    int cend = (int)((ntok + kPackTok - 1) / kPackTok); // chunks with tokens
    if (A.slot_off[A.planes_total] + 64 <= A.arena_cap) { // chunks with slot words to zero
        const uint64_t nw = (A.slot_off[pl + 1] - A.slot_off[pl]) / 16, per = (nw + nck - 1) / nck;
        if (per) cend = max(cend, (int)((nw + per - 1) / per));
    }
    for (int c = y; c < nck; c += K) {
        if (c >= cend) { // nothing to zero or count: a zero bit count
            cbits[(uint64_t)pl * nck + c] = 0;
            continue;
        }
        pack_count_item(A, planes, nck, cbits, pl, c);
        __syncthreads();
    }
}
// The slot's decode index (common.cuh): record k = the first fine
// checkpoint at or past k * B stream bits.  One thread per fine checkpoint j
// writes the records k with bitpos(j - 1) < k * B <= bitpos(j); the last one
// also writes the end markers.  After pack_write (bit positions final).
__global__ void __launch_bounds__(256) index_select(PackArgs A, int planes) {
    pdl_begin();
    const uint64_t nfine = (A.L + (1ull << A.log2C) - 1) >> A.log2C;
    const uint32_t per = (uint32_t)((nfine + 255) / 256);
    const int pl = blockIdx.x / per;
    if (pl >= planes) return;
    const uint64_t j = (uint64_t)(blockIdx.x % per) * 256 + threadIdx.x;
    if (j >= nfine) return;
    if (A.slot_off[A.planes_total] + 64 > A.arena_cap) return; // arena overflow: nothing was packed
    const uint32_t n = A.nsym[pl];
    const uint64_t bits = A.stream_bits[pl];
    const uint64_t nout = A.ocount[pl];
    const uint64_t bbytes = kHeaderBytes + 4 + 5ull * n + (bits + 7) / 8 + 16ull * nout;
    const int sh = index_shift(A.L, bbytes, A.log2C);
    const uint64_t nrec = bbytes >> sh;
    if (!nrec) return;
    const uint64_t B = 8ull << sh; // bits per record
    const uint64_t nidx = (A.L >> A.log2C) + 1;
    const IndexRec *fine = A.index + (uint64_t)pl * nidx;
    const uint64_t pre = kHeaderBytes + 4 + 5ull * n;
    const uint64_t off = A.slot_off[pl] + ((16 - (pre & 15)) & 15);
    IndexRec *sidx = reinterpret_cast<IndexRec *>(A.arena + index_offset(off, bbytes));
    const uint64_t bj = j == 0 ? 0 : fine[j].bitpos;
    const uint64_t bprev = j == 0 ? 0 : (j == 1 ? 0 : fine[j - 1].bitpos);
    // k in (bprev / B, bj / B]  (j = 0: k = 0 only, not stored)
    uint64_t k0 = j == 0 ? 1 : bprev / B + 1, k1 = j == 0 ? 0 : bj / B;
    if (j > 0 && bprev == bj) k1 = k0 - 1; // no new multiple crossed
    if (k1 > nrec) k1 = nrec;
    if (j > 0) {
        IndexRec r = fine[j];
        r.tok = (uint32_t)(j << A.log2C);
        for (uint64_t k = k0; k <= k1; ++k) sidx[k - 1] = r;
    }
    if (j == nfine - 1) { // records past the last checkpoint: end markers
        IndexRec e{};
        e.bitpos = bits;
        e.tok = (uint32_t)A.L;
        for (uint64_t k = (j == 0 ? 1 : tmax<uint64_t>(k1 + 1, k0)); k <= nrec; ++k) sidx[k - 1] = e;
    }
}

__global__ void __launch_bounds__(256) pack_write(PackArgs A, int planes, int nck, int K, const int32_t *coff,
                                                  const int32_t *cbits) {
    pdl_begin();
    const int pl = blockIdx.x / K, y = blockIdx.x % K;
    if (pl >= planes) return;
    const int nchk = (int)((A.ntok[pl] + kPackTok - 1) / kPackTok);
    for (int c = y; c < nchk; c += K) {
        pack_write_item(A, planes, nck, coff, cbits, pl, c);
        __syncthreads();
    }
}

} // namespace qcb
