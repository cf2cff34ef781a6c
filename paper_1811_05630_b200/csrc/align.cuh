// align.cuh -- exponent helpers for the alignment speculation of the
// parallel FP64 chain (see chain_scan.cuh).
#pragma once

#include "common.cuh"

namespace qcb {

// ------------------------------------------------------ exponent helpers
__device__ __forceinline__ int ulp_exp(double v) {
    const int e = (int)((bits_of(v) >> 52) & 0x7FF);
    return e == 0 ? -1074 : e - 1075;
}
// exponent of the lowest set bit (4096 for zero)
__device__ __forceinline__ int low_bit(double v) {
    const uint64_t b = bits_of(v);
    const int e = (int)((b >> 52) & 0x7FF);
    uint64_t m = b & ((1ull << 52) - 1);
    if (e) m |= 1ull << 52;
    if (!m) return 4096;
    return (e ? e - 1075 : -1074) + __ffsll((long long)m) - 1;
}
// v = sig * 2^ex exactly (sig signed, |sig| < 2^53)
__device__ __forceinline__ long long sig_of(double v, int &ex) {
    const uint64_t b = bits_of(v);
    const int e = (int)((b >> 52) & 0x7FF);
    long long m = (long long)(b & ((1ull << 52) - 1));
    if (e) m |= 1ll << 52;
    ex = e ? e - 1075 : -1074;
    return (b >> 63) ? -m : m;
}
__device__ __forceinline__ double pow2i(int e) { // e in [-1074, 1023]
    if (e >= -1022) return __longlong_as_double((long long)(e + 1023) << 52);
    return __longlong_as_double(1ll << (e + 1074));
}
// d = K * 2^A exactly (false if not representable that way)
__device__ __forceinline__ bool k_to_d(long long K, int A, double &d) {
    if (K > (1ll << 53) || K < -(1ll << 53) || A < -1074 || A > 970) return false;
    d = dmul((double)K, pow2i(A)); // exact: the product is representable
    return true;
}
__device__ __forceinline__ bool d_to_k(double d, int A, long long &K) {
    int ex;
    const long long M = sig_of(d, ex);
    if (M == 0) { K = 0; return true; }
    const int sh = ex - A;
    if (sh >= 0) {
        if (sh > 9) return false;
        K = M * (1ll << sh);
        return true;
    }
    if (sh <= -62) return false;
    if (M & ((1ll << -sh) - 1)) return false;
    K = M >> -sh;
    return true;
}

// Alignment exponent of a lattice event (estimate dhat, segment mu) and of
// an outlier value x (its own mu' = min(ulp(q), lowbit(x))).
__device__ __forceinline__ int16_t event_align(double dhat, int mu) { return (int16_t)max(ulp_exp(dhat), mu); }
__device__ __forceinline__ int segment_mu(double base, int uq) { return min(uq, low_bit(base)); }
__device__ __forceinline__ int16_t outlier_align(double x, int uq) {
    return (int16_t)max(ulp_exp(x), segment_mu(x, uq));
}

#ifndef QCSIM_CS_MAXW
#define QCSIM_CS_MAXW 2
#endif
constexpr int kMaxW = QCSIM_CS_MAXW;  // chain map tables of up to 2^kMaxW entries
constexpr int kTab = 1 << kMaxW;

// Reference K for an estimate dh at alignment A (A >= ulp(dh)): floor to a
// multiple of 2^kMaxW.
__device__ __forceinline__ long long ref_k(double dh, int A) {
    int ex;
    const long long M = sig_of(dh, ex);
    const int sh = A - ex; // >= 0
    long long K = sh >= 62 ? (M < 0 ? -1 : 0) : (M >> sh);
    return K & ~(long long)(kTab - 1);
}

} // namespace qcb
