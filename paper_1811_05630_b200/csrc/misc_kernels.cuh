// misc_kernels.cuh -- small kernels around the codec / engine pipeline.
#pragma once

#include <cfloat>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "norm.cuh"

namespace qcb {

// Effective bound per plane (codec.cpp:309-327) and reciprocal.
// mode: 0 RangeRelative, 1 Absolute, 2 Lossless.  One block per unit.
template <int NP, class Src>
__global__ void __launch_bounds__(256) init_params(PlaneParams *params, Src src, int units, uint64_t L,
                                                   int mode, double bound, int predictor, uint32_t *nonfinite,
                                                   uint32_t *symrange, uint32_t *hspecial,
                                                   unsigned long long *gamma_bits) {
    pdl_begin();
    const int unit = blockIdx.x;
    if (unit >= units) return;
    __shared__ double smin[NP][256], smax[NP][256];
    __shared__ int sbad;
    const int tid = threadIdx.x;
    double lo[NP], hi[NP];
    for (int p = 0; p < NP; ++p) { lo[p] = INFINITY; hi[p] = -INFINITY; }
    if (tid == 0) sbad = 0;
    __syncthreads();
    const bool need_range = mode == 0;
    const bool need_scan = nonfinite != nullptr;
    if (need_range || need_scan) {
        int bad = 0;
        for (uint64_t i = tid; i < L; i += 256) {
            double v[2];
            src.load(unit, i, v);
            for (int p = 0; p < NP; ++p) {
                if (!isfinite(v[p])) bad = 1;
                lo[p] = fmin(lo[p], v[p]);
                hi[p] = fmax(hi[p], v[p]);
            }
        }
        if (bad) sbad = 1;
    }
    for (int p = 0; p < NP; ++p) { smin[p][tid] = lo[p]; smax[p][tid] = hi[p]; }
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        if (tid < w)
            for (int p = 0; p < NP; ++p) {
                smin[p][tid] = fmin(smin[p][tid], smin[p][tid + w]);
                smax[p][tid] = fmax(smax[p][tid], smax[p][tid + w]);
            }
        __syncthreads();
    }
    if (tid < NP) {
        double eb;
        if (mode == 2) eb = 0.0;
        else if (mode == 1) eb = bound;
        else {
            eb = dmul(bound, dsub(smax[tid][0], smin[tid][0]));
            if (!isfinite(eb)) eb = DBL_MAX;
            if (eb == 0.0) eb = 0.0;
        }
        PlaneParams pp;
        pp.eb = eb;
        pp.q = dmul(2.0, eb);
        pp.inv_q = ddiv(1.0, pp.q);
        // the linear predictor with eb > 0 has no lattice model: serial path
        pp.flags = (predictor == 1 && eb != 0.0) ? kFlagFallback : 0u;
        pp.pad = 0;
        params[unit * NP + tid] = pp;
        const int pl = unit * NP + tid;
        symrange[2 * pl] = 0xFFFFFFFFu;
        symrange[2 * pl + 1] = 0;
        hspecial[2 * pl] = 0;
        hspecial[2 * pl + 1] = 0;
        gamma_bits[pl] = 0;
        if (nonfinite && sbad) atomicExch(nonfinite, 1u);
    }
}

// Exclusive scan of the per-plane arena slot sizes (16-byte aligned slots):
// out[p] = sum(in[0..p)), out[planes] = total.  One 1024-thread block.
// (also clears the packer's arena-overflow flag for this batch: a kernel
// instead of a memset keeps the launch chain programmatic)
__global__ void __launch_bounds__(256) slot_scan(const uint64_t *in, uint64_t *out, int planes, uint32_t *overflow) {
    pdl_begin();
    if (threadIdx.x == 0) *overflow = 0u;
    using Scan = cub::BlockScan<unsigned long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < planes; base += 256) {
        const int k = base + (int)threadIdx.x;
        const unsigned long long v = k < planes ? in[k] : 0ull;
        unsigned long long r, tot;
        Scan(tmp).ExclusiveSum(v, r, tot);
        if (k < planes) out[k] = carry + r;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[planes] = carry;
}

// Packs blocks scattered over an arena (fixed slots) back to back:
// meta = [src offset x P | dst offset x P | length x P], one block per block.
__global__ void gather_blocks(const uint8_t *arena, const uint64_t *meta, int P, uint8_t *out) {
    pdl_begin();
    const int k = blockIdx.x;
    if (k >= P) return;
    const uint8_t *src = arena + meta[k];
    uint8_t *dst = out + meta[P + k];
    for (uint64_t i = threadIdx.x; i < meta[2 * P + k]; i += blockDim.x) dst[i] = src[i];
}

// Per-slice sq_norm: adjacent-pair tree over the tile partials (the tile
// partials are themselves the lower levels of the same tree).
// One block per slice for slices of many tiles: the same adjacent-pair tree
// (levels in shared memory), ntiles <= 4096.
__global__ void __launch_bounds__(256) slice_norms_block(const double *tilesum, int ntiles, int units, double *out) {
    pdl_begin();
    __shared__ double buf[4096];
    const int u = blockIdx.x;
    if (u >= units) return;
    const double *t = tilesum + (uint64_t)u * ntiles;
    for (int k = threadIdx.x; k < ntiles; k += blockDim.x) buf[k] = t[k];
    __syncthreads();
    for (int w = ntiles / 2; w >= 1; w >>= 1) {
        double v[16];
        int n = 0;
        for (int k = threadIdx.x; k < w; k += blockDim.x) v[n++] = dadd(buf[2 * k], buf[2 * k + 1]);
        __syncthreads();
        n = 0;
        for (int k = threadIdx.x; k < w; k += blockDim.x) buf[k] = v[n++];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[u] = buf[0];
}
__global__ void slice_norms(const double *tilesum, int ntiles, int units, double *out) {
    pdl_begin();
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= units) return;
    // ntiles is a power of two (L and kTile are); iterative pairwise levels
    double buf[64];
    const double *t = tilesum + (uint64_t)u * ntiles;
    if (ntiles <= 64) {
        for (int k = 0; k < ntiles; ++k) buf[k] = t[k];
        for (int w = ntiles / 2; w >= 1; w >>= 1)
            for (int k = 0; k < w; ++k) buf[k] = dadd(buf[2 * k], buf[2 * k + 1]);
        out[u] = buf[0];
        return;
    }
    // larger: reduce groups of 64 recursively (tree shape preserved since
    // every group is an aligned power-of-two range)
    double acc[64];
    int groups = ntiles / 64;
    for (int gidx = 0; gidx < groups && gidx < 64; ++gidx) {
        for (int k = 0; k < 64; ++k) buf[k] = t[gidx * 64 + k];
        for (int w = 32; w >= 1; w >>= 1)
            for (int k = 0; k < w; ++k) buf[k] = dadd(buf[2 * k], buf[2 * k + 1]);
        acc[gidx] = buf[0];
    }
    // groups <= 64 for ntiles <= 4096 (L <= 2^22); larger slices use
    // slice_norms_large
    for (int w = groups / 2; w >= 1; w >>= 1)
        for (int k = 0; k < w; ++k) acc[k] = dadd(acc[2 * k], acc[2 * k + 1]);
    out[u] = acc[0];
}

// Dense gate step for compression-off engines: new = gate(old),
// plus the same per-tile sq-norm partials the encoder produces.
template <class Src>
__global__ void __launch_bounds__(256) dense_gate(Src src, int units, uint64_t L, double *out, double *tilesum) {
    pdl_begin();
    const int ntiles = (int)((L + kTile - 1) / kTile);
    const int unit = blockIdx.x / ntiles, t = blockIdx.x % ntiles;
    if (unit >= units) return;
    __shared__ double red[256];
    const int tid = threadIdx.x;
    double acc[4];
    for (int e = 0; e < 4; ++e) {
        const uint64_t i = (uint64_t)t * kTile + tid * 4 + e;
        acc[e] = 0.0;
        if (i < L) {
            double v[2];
            src.load(unit, i, v);
            out[(uint64_t)unit * 2 * L + i] = v[0];
            out[(uint64_t)unit * 2 * L + L + i] = v[1];
            acc[e] = dadd(dmul(v[0], v[0]), dmul(v[1], v[1]));
        }
    }
    red[tid] = dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3]));
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        double v = 0.0;
        if (tid < w) v = dadd(red[2 * tid], red[2 * tid + 1]);
        __syncthreads();
        if (tid < w) red[tid] = v;
        __syncthreads();
    }
    if (tid == 0) tilesum[(uint64_t)unit * ntiles + t] = red[0];
}

// Per gate pass: compression ratio min / sum (plane order, as the host's
// record_sizes), current and peak bytes, fallback planes, latched errors.
// Fused with the slot-offset scan of the packer (one block, both read the
// codebook's per-plane results).
__global__ void __launch_bounds__(256) slot_scan_stats(const uint64_t *slot_bytes, uint64_t *slot_off,
                                                       const uint64_t *bytes, const uint32_t *err,
                                                       const PlaneParams *params, int planes, uint64_t L,
                                                       unsigned long long gate, EngineDevStats *st,
                                                       uint32_t *overflow, GateRowDev *rows,
                                                       unsigned long long row0, unsigned long long nrows,
                                                       int log2C) {
    pdl_begin();
    if (threadIdx.x == 0) *overflow = 0u;
    using Scan = cub::BlockScan<unsigned long long, 256>;
    using Red = cub::BlockReduce<unsigned long long, 256>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Red::TempStorage red;
    } tmp;
    __shared__ unsigned long long carry;
    __shared__ double ratio[1024];
    const int tid = threadIdx.x;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < planes; base += 256) {
        const int k = base + tid;
        const unsigned long long v = k < planes ? slot_bytes[k] : 0ull;
        unsigned long long r, tot;
        Scan(tmp.scan).ExclusiveSum(v, r, tot);
        if (k < planes) slot_off[k] = carry + r;
        __syncthreads();
        if (tid == 0) carry += tot;
        __syncthreads();
    }
    if (tid == 0) slot_off[planes] = carry;
    const double in_bytes = (double)(8 * L);
    unsigned long long tsum = 0, fb = 0, isum = 0;
    int bad = 0;
    double rmin = 0.0, rsum = 0.0, pmin = INFINITY, psum = 0.0;
    if (tid == 0) {
        rmin = st->ratio_min;
        rsum = st->ratio_sum;
    }
    for (int base = 0; base < planes; base += 1024) {
        const int m = min(1024, planes - base);
        for (int k = tid; k < m; k += 256) {
            const uint64_t b = bytes[base + k];
            ratio[k] = ddiv(in_bytes, (double)b);
            tsum += b;
            isum += index_records(L, b, log2C) * sizeof(IndexRec);
            fb += (params[base + k].flags & kFlagFallback) ? 1 : 0;
            bad |= err[base + k] != 0;
        }
        __syncthreads();
        if (tid == 0) // plane order, in registers
            for (int k = 0; k < m; ++k) {
                const double r = ratio[k];
                if (r < rmin) rmin = r;
                rsum = dadd(rsum, r);
                if (r < pmin) pmin = r;
                psum = dadd(psum, r);
            }
        __syncthreads();
    }
    tsum = Red(tmp.red).Sum(tsum);
    __syncthreads();
    fb = Red(tmp.red).Sum(fb);
    __syncthreads();
    isum = Red(tmp.red).Sum(isum);
    bad = __syncthreads_or(bad);
    if (tid == 0) {
        write_gate_row(rows, row0, nrows, gate, pmin, psum, (unsigned long long)planes, tsum, isum);
        st->ratio_min = rmin;
        st->ratio_sum = rsum;
        st->calls += (unsigned long long)planes;
        st->current = tsum;
        if (tsum > st->peak) st->peak = tsum;
        st->fallback += fb;
        if (st->status == kEngOk && bad) {
            st->status = kEngDepth;
            st->status_gate = gate;
        }
    }
}

// ------------------------------------------------ on-device state comparison
// Two decoded states ([slot][re|im][L], same layout): per 1024-element tile,
// pairwise trees of conj(a).b (re, im), |a|^2, |b|^2 and the max |a - b|
// (statevec.cpp:199-247 semantics; the host finishes the tile trees).
__global__ void __launch_bounds__(256) state_compare(const double *a, const double *b, uint64_t L, int units,
                                                     double *part) {
    pdl_begin();
    const int ntiles = (int)((L + kTile - 1) / kTile);
    const int unit = blockIdx.x / ntiles, t = blockIdx.x % ntiles;
    if (unit >= units) return;
    __shared__ double red[4][256];
    __shared__ double mx[256];
    const int tid = threadIdx.x;
    double s[4][4], m = 0.0;
    for (int e = 0; e < 4; ++e) {
        const uint64_t i = (uint64_t)t * kTile + tid * 4 + e;
        s[0][e] = s[1][e] = s[2][e] = s[3][e] = 0.0;
        if (i < L) {
            const double ar = a[(uint64_t)unit * 2 * L + i], ai = a[(uint64_t)unit * 2 * L + L + i];
            const double br = b[(uint64_t)unit * 2 * L + i], bi = b[(uint64_t)unit * 2 * L + L + i];
            s[0][e] = dadd(dmul(ar, br), dmul(ai, bi));
            s[1][e] = dsub(dmul(ar, bi), dmul(ai, br));
            s[2][e] = dadd(dmul(ar, ar), dmul(ai, ai));
            s[3][e] = dadd(dmul(br, br), dmul(bi, bi));
            const double dr = dsub(ar, br), di = dsub(ai, bi);
            m = fmax(m, __dsqrt_rn(dadd(dmul(dr, dr), dmul(di, di))));
        }
    }
    for (int q = 0; q < 4; ++q) red[q][tid] = dadd(dadd(s[q][0], s[q][1]), dadd(s[q][2], s[q][3]));
    mx[tid] = m;
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        double v[4], vm = 0.0;
        if (tid < w) {
            for (int q = 0; q < 4; ++q) v[q] = dadd(red[q][2 * tid], red[q][2 * tid + 1]);
            vm = fmax(mx[2 * tid], mx[2 * tid + 1]);
        }
        __syncthreads();
        if (tid < w) {
            for (int q = 0; q < 4; ++q) red[q][tid] = v[q];
            mx[tid] = vm;
        }
        __syncthreads();
    }
    if (tid == 0) {
        double *o = part + 5 * ((uint64_t)unit * ntiles + t);
        for (int q = 0; q < 4; ++q) o[q] = red[q][0];
        o[4] = mx[0];
    }
}

} // namespace qcb
