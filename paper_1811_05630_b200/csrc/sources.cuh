// sources.cuh -- where the encoder's plane values come from.
//
// RawSrc : caller planes (compress_plane, codec.hpp:98-99).
// GateSrc: the engine gate pass: the new
//          amplitude of global index g is the lowered action (circuit.cpp:
//          392-427) applied to the scaled old amplitudes of g's slice and its
//          partner slice, with the pinned product/sum order shared with
//          oracle/qcsim_oracle.c (apply_one).
#pragma once

#include "common.cuh"

namespace qcb {

// Source of plane values: raw planes (codec mode).
struct RawSrc {
    const double *const *x;    // per plane
    __device__ __forceinline__ void load(int unit, uint64_t i, double *v) const { v[0] = x[unit][i]; }
    static constexpr bool kNorms = false;
};

// Which local slices a batch of encoder units covers, and where each
// unit's partner slice sits among the decoded old planes.
//   identity: unit u = local slice gbase + u (gbase = 0 when all local
//             slices are one batch: the partner of u is u ^ hm, slot u ^ hm);
//   grouped:  a wave of `nunits` slices closed under the partner mask: unit
//             u is member (u mod G) of group gbase + u / G, G = 2^popcount(hm),
//             the member bits sitting at hm's positions; the partner is
//             member (u mod G) ^ (G - 1) of the same group, slot u ^ (G - 1);
//   remote:   identity, but every partner lives on another rank; imported
//             partners are decoded at slot nunits + u.
struct SliceMap {
    uint64_t s0 = 0;    // first local slice (global index)
    uint64_t hm = 0;    // partner XOR mask over slice indices (relative to s0)
    uint64_t gbase = 0; // grouped: first group of the batch
    uint32_t gsh = 0;   // grouped: log2(G) = popcount(hm)
    uint32_t mode = 0;  // 0 identity, 1 grouped, 2 remote
    uint32_t nunits = 0;
    __host__ __device__ __forceinline__ uint64_t slice_rel(uint32_t unit) const {
        if (mode != 1) return gbase + unit;
        uint64_t r = gbase + (unit >> gsh);
        uint32_t m = unit & ((1u << gsh) - 1);
        uint64_t h = hm;
        while (h) { // deposit the member bits at hm's positions, lowest first
            const int b = ctz64(h);
            r = ((r >> b) << (b + 1)) | (r & ((1ull << b) - 1)) | ((uint64_t)(m & 1u) << b);
            m >>= 1;
            h &= h - 1;
        }
        return r;
    }
    __host__ __device__ __forceinline__ uint32_t partner_slot(uint32_t unit) const {
        if (mode == 0) return unit ^ (uint32_t)hm;
        if (mode == 1) return unit ^ ((1u << gsh) - 1);
        return nunits + unit;
    }
    __host__ __device__ static __forceinline__ int ctz64(uint64_t v) {
#ifdef __CUDA_ARCH__
        return __ffsll((long long)v) - 1;
#else
        return __builtin_ctzll(v);
#endif
    }
};

// Source of plane values: the engine's gate pass.  New
// amplitude of global index g = action applied to the scaled old values.
struct GateSrc {
    const double *old;          // dense old planes, [slot][re|im][L]
    SliceMap map;               // unit -> slice, partner slot
    double scale;               // 1/sqrt(G) (host-computed) ...
    const double *scale_dev;    // ... or device-computed (engine_norm) when set
    int apply_scale;            // 0: normalization skipped for this gate
    DevAction act;
    int s;
    uint64_t L;
    static constexpr bool kNorms = true;

    __device__ __forceinline__ void fetch(uint64_t g, uint64_t own, uint32_t unit, double sc, bool apply,
                                          double &re, double &im) const {
        const uint32_t slot = (g >> s) == own ? unit : map.partner_slot(unit);
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
        const uint64_t own = map.s0 + map.slice_rel((uint32_t)unit);
        const uint64_t g = (own << s) | i;
        const bool apply = apply_scale != 0;
        const double sc = scale_dev ? *scale_dev : scale;
        if (act.kind == 0) {
            double r, m;
            fetch(g, own, unit, sc, apply, r, m);
            if ((g & act.mask) == act.mask) cmul(act.f[0], act.f[1], r, m, v[0], v[1]);
            else { v[0] = r; v[1] = m; }
        } else if (act.kind == 1) {
            if ((g & act.mask) != act.mask) { fetch(g, own, unit, sc, apply, v[0], v[1]); return; }
            const uint64_t tb = 1ull << act.target;
            double v0r, v0i, v1r, v1i, p0r, p0i, p1r, p1i;
            fetch(g & ~tb, own, unit, sc, apply, v0r, v0i);
            fetch(g | tb, own, unit, sc, apply, v1r, v1i);
            const double *u = (g & tb) ? act.u + 4 : act.u;
            cmul(u[0], u[1], v0r, v0i, p0r, p0i);
            cmul(u[2], u[3], v1r, v1i, p1r, p1i);
            v[0] = dadd(p0r, p1r);
            v[1] = dadd(p0i, p1i);
        } else {
            const uint64_t ba = (g >> act.a) & 1, bb = (g >> act.b) & 1;
            const uint64_t src = ba != bb ? g ^ ((1ull << act.a) | (1ull << act.b)) : g;
            fetch(src, own, unit, sc, apply, v[0], v[1]);
        }
    }
};

} // namespace qcb
