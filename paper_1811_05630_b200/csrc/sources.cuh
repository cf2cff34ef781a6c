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

// Source of plane values: the engine's gate pass.  New
// amplitude of global index g = action applied to the scaled old values.
struct GateSrc {
    const double *old;          // dense old planes, [slot][re|im][L]
    const int32_t *slot_of;     // global slice -> slot in `old`
    const uint64_t *unit_slice; // unit -> global slice
    double scale;               // 1/sqrt(G) (host-computed) ...
    const double *scale_dev;    // ... or device-computed (engine_norm) when set
    int apply_scale;            // 0: normalization skipped for this gate
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
        const bool apply = apply_scale != 0;
        const double sc = scale_dev ? *scale_dev : scale;
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

} // namespace qcb
