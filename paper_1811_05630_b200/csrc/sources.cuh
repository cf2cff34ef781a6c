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
    // elements i (even) and i + 1: caller planes carry no alignment promise
    __device__ __forceinline__ void load2(int unit, uint64_t i, double *a, double *b) const {
        a[0] = x[unit][i];
        b[0] = x[unit][i + 1];
    }
    static constexpr bool kNorms = false;
    template <bool> __device__ __forceinline__ void loadf(int unit, uint64_t i, double *v) const { load(unit, i, v); }
    template <bool> __device__ __forceinline__ void load2f(int unit, uint64_t i, double *a, double *b) const {
        load2(unit, i, a, b);
    }
    __device__ __forceinline__ bool flagged_sources(int, uint32_t) const { return false; }
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
    const uint8_t *zold = nullptr; // zero-tile flags of `old`, [slot plane][ztiles] (decode_kernels.cuh)
    uint32_t ztiles = 0;
    static constexpr bool kNorms = true;

    // kFlags: consult the decoder's zero-tile flags (a flagged tile may not be
    // written).  enc_x takes the flag-free instantiation for blocks none of
    // whose source tiles is flagged (flagged_sources).
    template <bool kFlags>
    __device__ __forceinline__ void fetch(uint64_t g, uint64_t own, uint32_t unit, double sc, bool apply,
                                          double &re, double &im) const {
        const uint32_t slot = (g >> s) == own ? unit : map.partner_slot(unit);
        const uint64_t off = g & (L - 1);
        const double *p = old + (uint64_t)slot * 2 * L;
        bool zr = false, zi = false; // tile flagged +0.0 by the decoder (possibly not written)
        if (kFlags && zold) {
            const uint64_t tt = off >> kTileLog2;
            zr = zold[(uint64_t)(2 * slot) * ztiles + tt] != 0;
            zi = zold[(uint64_t)(2 * slot + 1) * ztiles + tt] != 0;
        }
        re = zr ? 0.0 : p[off];
        im = zi ? 0.0 : p[L + off];
        if (apply) {
            re = dmul(re, sc);
            im = dmul(im, sc);
        }
    }
    // Elements g (even offset) and g + 1 of one slice: one 16-byte load per
    // plane (the planes are 16-byte aligned: cudaMalloc base, even L).
    template <bool kFlags>
    __device__ __forceinline__ void fetch2(uint64_t g, uint64_t own, uint32_t unit, double sc, bool apply,
                                           double2 &re, double2 &im) const {
        const uint32_t slot = (g >> s) == own ? unit : map.partner_slot(unit);
        const uint64_t off = g & (L - 1);
        const double *p = old + (uint64_t)slot * 2 * L;
        bool zr = false, zi = false;
        if (kFlags && zold) {
            const uint64_t tt = off >> kTileLog2;
            zr = zold[(uint64_t)(2 * slot) * ztiles + tt] != 0;
            zi = zold[(uint64_t)(2 * slot + 1) * ztiles + tt] != 0;
        }
        re = zr ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(p + off);
        im = zi ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(p + L + off);
        if (apply) {
            re.x = dmul(re.x, sc);
            re.y = dmul(re.y, sc);
            im.x = dmul(im.x, sc);
            im.y = dmul(im.y, sc);
        }
    }
    // load() of elements i (even) and i + 1 (< L) with vector fetches: the
    // same operations per element, in the same order.
    template <bool kFlags>
    __device__ __forceinline__ void load2f(int unit, uint64_t i, double *a, double *b) const {
        const uint64_t own = map.s0 + map.slice_rel((uint32_t)unit);
        const uint64_t g = (own << s) | i;
        const bool apply = apply_scale != 0;
        const double sc = scale_dev ? *scale_dev : scale;
        double2 r, m;
        if (act.kind == 0) {
            fetch2<kFlags>(g, own, unit, sc, apply, r, m);
            if ((g & act.mask) == act.mask) cmul(act.f[0], act.f[1], r.x, m.x, a[0], a[1]);
            else { a[0] = r.x; a[1] = m.x; }
            if (((g | 1) & act.mask) == act.mask) cmul(act.f[0], act.f[1], r.y, m.y, b[0], b[1]);
            else { b[0] = r.y; b[1] = m.y; }
        } else if (act.kind == 1) {
            const uint64_t tb = 1ull << act.target;
            const bool on0 = (g & act.mask) == act.mask, on1 = ((g | 1) & act.mask) == act.mask;
            double p0r, p0i, p1r, p1i;
            if (act.target == 0) { // the pair itself: v0 = element g, v1 = element g + 1
                fetch2<kFlags>(g, own, unit, sc, apply, r, m);
                if (on0) {
                    cmul(act.u[0], act.u[1], r.x, m.x, p0r, p0i);
                    cmul(act.u[2], act.u[3], r.y, m.y, p1r, p1i);
                    a[0] = dadd(p0r, p1r);
                    a[1] = dadd(p0i, p1i);
                } else { a[0] = r.x; a[1] = m.x; }
                if (on1) {
                    cmul(act.u[4], act.u[5], r.x, m.x, p0r, p0i);
                    cmul(act.u[6], act.u[7], r.y, m.y, p1r, p1i);
                    b[0] = dadd(p0r, p1r);
                    b[1] = dadd(p0i, p1i);
                } else { b[0] = r.y; b[1] = m.y; }
                return;
            }
            if (!on0 && !on1) {
                fetch2<kFlags>(g, own, unit, sc, apply, r, m);
                a[0] = r.x; a[1] = m.x; b[0] = r.y; b[1] = m.y;
                return;
            }
            double2 r1, m1; // r, m: the bit-clear partner's pair; r1, m1: the bit-set one's
            fetch2<kFlags>(g & ~tb, own, unit, sc, apply, r, m);
            fetch2<kFlags>(g | tb, own, unit, sc, apply, r1, m1);
            const double *u = (g & tb) ? act.u + 4 : act.u;
            if (on0) {
                cmul(u[0], u[1], r.x, m.x, p0r, p0i);
                cmul(u[2], u[3], r1.x, m1.x, p1r, p1i);
                a[0] = dadd(p0r, p1r);
                a[1] = dadd(p0i, p1i);
            } else if (g & tb) { a[0] = r1.x; a[1] = m1.x; }
            else { a[0] = r.x; a[1] = m.x; }
            if (on1) {
                cmul(u[0], u[1], r.y, m.y, p0r, p0i);
                cmul(u[2], u[3], r1.y, m1.y, p1r, p1i);
                b[0] = dadd(p0r, p1r);
                b[1] = dadd(p0i, p1i);
            } else if (g & tb) { b[0] = r1.y; b[1] = m1.y; }
            else { b[0] = r.y; b[1] = m.y; }
        } else {
            if (act.a == 0 || act.b == 0) { // the swap moves bit 0: element-wise
                loadf<kFlags>(unit, i, a);
                loadf<kFlags>(unit, i + 1, b);
                return;
            }
            const uint64_t ba = (g >> act.a) & 1, bb = (g >> act.b) & 1;
            const uint64_t src = ba != bb ? g ^ ((1ull << act.a) | (1ull << act.b)) : g;
            fetch2<kFlags>(src, own, unit, sc, apply, r, m);
            a[0] = r.x; a[1] = m.x; b[0] = r.y; b[1] = m.y;
        }
    }
    template <bool kFlags>
    __device__ __forceinline__ void loadf(int unit, uint64_t i, double *v) const {
        const uint64_t own = map.s0 + map.slice_rel((uint32_t)unit);
        const uint64_t g = (own << s) | i;
        const bool apply = apply_scale != 0;
        const double sc = scale_dev ? *scale_dev : scale;
        if (act.kind == 0) {
            double r, m;
            fetch<kFlags>(g, own, unit, sc, apply, r, m);
            if ((g & act.mask) == act.mask) cmul(act.f[0], act.f[1], r, m, v[0], v[1]);
            else { v[0] = r; v[1] = m; }
        } else if (act.kind == 1) {
            if ((g & act.mask) != act.mask) { fetch<kFlags>(g, own, unit, sc, apply, v[0], v[1]); return; }
            const uint64_t tb = 1ull << act.target;
            double v0r, v0i, v1r, v1i, p0r, p0i, p1r, p1i;
            fetch<kFlags>(g & ~tb, own, unit, sc, apply, v0r, v0i);
            fetch<kFlags>(g | tb, own, unit, sc, apply, v1r, v1i);
            const double *u = (g & tb) ? act.u + 4 : act.u;
            cmul(u[0], u[1], v0r, v0i, p0r, p0i);
            cmul(u[2], u[3], v1r, v1i, p1r, p1i);
            v[0] = dadd(p0r, p1r);
            v[1] = dadd(p0i, p1i);
        } else {
            const uint64_t ba = (g >> act.a) & 1, bb = (g >> act.b) & 1;
            const uint64_t src = ba != bb ? g ^ ((1ull << act.a) | (1ull << act.b)) : g;
            fetch<kFlags>(src, own, unit, sc, apply, v[0], v[1]);
        }
    }
    __device__ __forceinline__ void load(int unit, uint64_t i, double *v) const { loadf<true>(unit, i, v); }
    __device__ __forceinline__ void load2(int unit, uint64_t i, double *a, double *b) const {
        load2f<true>(unit, i, a, b);
    }
    // True when a plane-tile that the new tile `t` of `unit` (or its halo
    // element, the last one of tile t - 1) may read is flagged: own and
    // partner slot, tiles t and t - 1 and their images under the action's
    // tile-index bits.  Conservative; one thread per block evaluates it.
    __device__ __forceinline__ bool flagged_sources(int unit, uint32_t t) const {
        if (!zold) return false;
        uint32_t tm = 0;
        if (act.kind == 1) {
            if (act.target >= kTileLog2 && act.target < s) tm = 1u << (act.target - kTileLog2);
        } else if (act.kind == 2) {
            if (act.a >= kTileLog2 && act.a < s) tm |= 1u << (act.a - kTileLog2);
            if (act.b >= kTileLog2 && act.b < s) tm |= 1u << (act.b - kTileLog2);
        }
        const uint32_t slots[2] = {(uint32_t)unit, map.hm ? map.partner_slot((uint32_t)unit) : (uint32_t)unit};
        const uint32_t tiles[4] = {t, t ^ tm, t ? t - 1 : t, (t ? t - 1 : t) ^ tm};
        uint32_t any = 0;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 4; ++b)
                any |= zold[(uint64_t)(2 * slots[a]) * ztiles + tiles[b]] | zold[(uint64_t)(2 * slots[a] + 1) * ztiles + tiles[b]];
        return any != 0;
    }
};

} // namespace qcb
