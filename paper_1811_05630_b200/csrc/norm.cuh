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

struct NormArgs {
    const double *tilesum; // [slice][ntiles] partial trees of the previous pass (nullptr: sq holds the norms)
    int ntiles;
    double *sq, *b0, *b1;  // slice norms, tree buffers
    uint64_t S;
    double tol10;
    unsigned long long gate;
    double *scale;
    const uint32_t *overflow;
    EngineDevStats *st;
    int enabled;
};


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
