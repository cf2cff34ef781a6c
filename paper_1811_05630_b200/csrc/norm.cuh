// norm.cuh -- gate-pass normalization of the deferred engine loop
// (DESIGN.md §3.2): shared by the standalone engine_norm kernel
// and the decoder grid's extra block.
#pragma once

#include "common.cuh"

namespace qcb {

// ------------------------------------------------ deferred engine bookkeeping
// Gate passes that never wait for the host: the normalization scale and the
// run metrics live on the device; errors are latched (first one wins) and
// raised by the host when the run returns.
enum : uint32_t { kEngOk = 0, kEngNumeric = 1, kEngDepth = 2, kEngOverflow = 3 };

struct EngineDevStats {
    double ratio_min, ratio_sum, norm_G;
    unsigned long long calls, current, peak, fallback, status_gate;
    uint32_t status, pad;
};

// Per-gate row of a deferred run (index gate - row0 + 1; row 0 holds the
// run's start stamp): this pass's min ratio, ratio sum in plane order, calls,
// block bytes, decode-index bytes and a %globaltimer stamp taken when the
// pass's metrics are settled.
struct GateRowDev {
    double min_ratio, ratio_sum;
    unsigned long long calls, bytes, index_bytes, t_ns;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct NormArgs {
    int norm;              // run the normalization (norm_every)
    const double *tilesum; // [slice][ntiles] partial trees of the previous pass (nullptr: sq holds the norms)
    int ntiles;
    double *sq, *b0, *b1;  // slice norms, tree buffers
    uint64_t S;
    double tol10;
    unsigned long long gate;
    double *scale;
    const uint32_t *overflow;
    EngineDevStats *st;
    int enabled;           // the extra block runs at all (norm or stats)
    // run metrics of the previous encode pass (fixed-slot deferred loop: no
    // slot scan), accumulated before the normalization
    int stats;
    const uint64_t *bytes;
    const uint32_t *err;
    const PlaneParams *params;
    int planes;
    uint64_t L;
    int log2C;             // finest decode-index chunk (index bytes per plane, common.cuh)
    unsigned long long stats_gate;
    GateRowDev *rows;      // per-gate rows of the run (nullptr: none)
    unsigned long long row0;
    unsigned long long nrows;
    int stamp;             // first pass of a run: stamp rows[0]
};

__device__ __forceinline__ void write_gate_row(GateRowDev *rows, unsigned long long row0, unsigned long long nrows,
                                               unsigned long long gate, double pmin, double psum,
                                               unsigned long long calls, unsigned long long bytes,
                                               unsigned long long ibytes) {
    if (!rows || gate < row0 || gate - row0 >= nrows) return;
    GateRowDev &r = rows[gate - row0 + 1];
    r.min_ratio = pmin;
    r.ratio_sum = psum;
    r.calls = calls;
    r.bytes = bytes;
    r.index_bytes = ibytes;
    r.t_ns = global_ns();
}

// Per encode pass: compression ratio min / sum in plane order (as the
// host's record_sizes), current and peak bytes, fallback planes, latched
// codec errors.  The whole block: ratios in parallel, the plane-order sum
// by thread 0.
__device__ void pass_stats(const uint64_t *bytes, const uint32_t *err, const PlaneParams *params, int planes,
                           uint64_t L, unsigned long long gate, EngineDevStats *st, const NormArgs &N) {
    __shared__ double s_r[256];
    __shared__ unsigned long long s_tsum, s_fb, s_isum;
    __shared__ int s_bad;
    const int tid = threadIdx.x, nt = min((int)blockDim.x, 256);
    const double in_bytes = (double)(8 * L);
    if (tid == 0) {
        s_tsum = 0;
        s_fb = 0;
        s_isum = 0;
        s_bad = 0;
    }
    double rmin = 0.0, rsum = 0.0, pmin = INFINITY, psum = 0.0;
    if (tid == 0) {
        rmin = st->ratio_min;
        rsum = st->ratio_sum;
    }
    __syncthreads();
    for (int base = 0; base < planes; base += nt) {
        const int k = base + tid;
        if (tid < nt && k < planes) {
            const uint64_t b = bytes[k];
            s_r[tid] = ddiv(in_bytes, (double)b);
            atomicAdd(&s_tsum, (unsigned long long)b);
            atomicAdd(&s_isum, (unsigned long long)(index_records(L, b, N.log2C) * sizeof(IndexRec)));
            if (params[k].flags & kFlagFallback) atomicAdd(&s_fb, 1ull);
            if (err[k] != 0) s_bad = 1;
        }
        __syncthreads();
        if (tid == 0)
            for (int j = 0; j < nt && base + j < planes; ++j) {
                const double r = s_r[j];
                if (r < rmin) rmin = r;
                rsum = dadd(rsum, r);
                if (r < pmin) pmin = r;
                psum = dadd(psum, r);
            }
        __syncthreads();
    }
    if (tid == 0) {
        write_gate_row(N.rows, N.row0, N.nrows, gate, pmin, psum, (unsigned long long)planes, s_tsum, s_isum);
        st->ratio_min = rmin;
        st->ratio_sum = rsum;
        st->calls += (unsigned long long)planes;
        st->current = s_tsum;
        if (s_tsum > st->peak) st->peak = s_tsum;
        st->fallback += s_fb;
        if (st->status == kEngOk && s_bad) {
            st->status = kEngDepth;
            st->status_gate = gate;
        }
    }
    __syncthreads();
}
__global__ void pass_stats_kernel(NormArgs N) {
    pdl_begin();
    pass_stats(N.bytes, N.err, N.params, N.planes, N.L, N.stats_gate, N.st, N);
}


// Gate-pass prologue of the deferred loop: per-slice sq_norm of the previous
// pass from its tile partials (the slice_norms tree), G = pairwise tree over
// the S slice norms (the association of the host's tree_sum_host /
// DESIGN.md §3.2), drift check, scale = 1/sqrt(G); also latches an arena
// overflow of the previous pass.
__device__ void engine_norm_body(const NormArgs &N) {
    const double *tilesum = N.tilesum;
    const int ntiles = N.ntiles;
    double *sq = N.sq, *b0 = N.b0, *b1 = N.b1;
    const uint64_t S = N.S;
    const double tol10 = N.tol10;
    const unsigned long long gate = N.gate;
    double *scale = N.scale;
    const uint32_t *overflow = N.overflow;
    EngineDevStats *st = N.st;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (N.stats) pass_stats(N.bytes, N.err, N.params, N.planes, N.L, N.stats_gate, st, N);
    if (N.stamp && N.rows && tid == 0) N.rows[0].t_ns = global_ns();
    if (!N.norm) return;
    // slice norms: one thread per slice over its (aligned power-of-two) tiles
    // (tilesum == nullptr: `sq` already holds them)
    for (uint64_t u = tid; tilesum && u < S; u += nt) {
        const double *t = tilesum + u * ntiles;
        double acc[64], buf[64];
        if (ntiles <= 64) {
            for (int k = 0; k < ntiles; ++k) buf[k] = t[k];
            for (int w = ntiles / 2; w >= 1; w >>= 1)
                for (int k = 0; k < w; ++k) buf[k] = dadd(buf[2 * k], buf[2 * k + 1]);
            sq[u] = buf[0];
        } else {
            const int groups = ntiles / 64;
            for (int g = 0; g < groups && g < 64; ++g) {
                for (int k = 0; k < 64; ++k) buf[k] = t[g * 64 + k];
                for (int w = 32; w >= 1; w >>= 1)
                    for (int k = 0; k < w; ++k) buf[k] = dadd(buf[2 * k], buf[2 * k + 1]);
                acc[g] = buf[0];
            }
            for (int w = groups / 2; w >= 1; w >>= 1)
                for (int k = 0; k < w; ++k) acc[k] = dadd(acc[2 * k], acc[2 * k + 1]);
            sq[u] = acc[0];
        }
    }
    __syncthreads();
    for (uint64_t k = tid; k < S; k += nt) b0[k] = sq[k];
    __syncthreads();
    double *in = b0, *out = b1;
    for (uint64_t w = S / 2; w >= 1; w /= 2) {
        for (uint64_t k = tid; k < w; k += nt) out[k] = dadd(in[2 * k], in[2 * k + 1]);
        __syncthreads();
        double *t = in;
        in = out;
        out = t;
    }
    if (tid == 0) {
        if (overflow && *overflow && st->status == kEngOk) {
            st->status = kEngOverflow;
            st->status_gate = gate - 1;
        }
        const double G = in[0];
        if (!isfinite(G) || fabs(dsub(G, 1.0)) > tol10) {
            if (st->status == kEngOk) {
                st->status = kEngNumeric;
                st->status_gate = gate;
                st->norm_G = G;
            }
            *scale = 1.0;
        } else {
            *scale = ddiv(1.0, __dsqrt_rn(G));
        }
    }
}

__global__ void __launch_bounds__(256) engine_norm(NormArgs N) {
    pdl_begin();
    engine_norm_body(N);
}

} // namespace qcb
