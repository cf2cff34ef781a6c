// Microbenchmark: two-queue Huffman merge (codec.cpp:168-229) on a small
// skewed alphabet in shared memory -- serial (one thread) vs warp-batched,
// through generic pointers vs direct shared arrays.  Cycles per plane.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <class T> __device__ T tmin(T a, T b) { return a < b ? a : b; }

template <class P>
__device__ uint32_t merge_serial(P nc, int32_t *par, uint32_t n) {
    uint32_t lp = 0, ip = n, nodes = n;
    uint32_t lv = nc[0], iv = 0;
    while ((n - lp) + (nodes - ip) >= 2) {
        uint32_t pick[2], pv[2];
        for (int k = 0; k < 2; ++k) {
            const bool leaf_ok = lp < n, int_ok = ip < nodes;
            const bool take_leaf = leaf_ok && (!int_ok || lv <= iv);
            if (take_leaf) { pick[k] = lp; pv[k] = lv; ++lp; lv = lp < n ? nc[lp] : 0u; }
            else { pick[k] = ip; pv[k] = iv; ++ip; iv = ip < nodes ? nc[ip] : 0u; }
        }
        const uint32_t sum = pv[0] + pv[1];
        nc[nodes] = sum;
        par[pick[0]] = (int32_t)nodes;
        par[pick[1]] = (int32_t)nodes;
        if (ip == nodes) iv = sum;
        ++nodes;
    }
    return nodes;
}
template <class P>
__device__ uint32_t merge_warp(P nc, int32_t *par, uint32_t n, int tid) {
    uint32_t lp = 0, ip = n, nodes = n;
    while ((n - lp) + (nodes - ip) >= 2) {
        const uint32_t nA = n - lp, nB = nodes - ip, j = (uint32_t)tid;
        uint32_t lo = j > nB ? j - nB : 0u, hi = min(j, nA);
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (nc[lp + mid] <= nc[ip + j - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        const uint32_t cL = lo, cI = j - lo;
        const bool valid = j < nA + nB && (cI < nB || j < 2);
        const bool take_leaf = cL < nA && (cI >= nB || nc[lp + cL] <= nc[ip + cI]);
        const uint32_t idx = valid ? (take_leaf ? lp + cL : ip + cI) : 0u;
        const uint32_t val = valid ? nc[idx] : 0u;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        uint32_t P2 = vm == 0xffffffffu ? 32u : (uint32_t)(__ffs(~vm) - 1);
        P2 &= ~1u;
        const uint32_t pidx = __shfl_xor_sync(0xffffffffu, idx, 1);
        const uint32_t pval = __shfl_xor_sync(0xffffffffu, val, 1);
        const unsigned lm = __ballot_sync(0xffffffffu, valid && take_leaf) & (P2 >= 32 ? 0xffffffffu : ((1u << P2) - 1u));
        __syncwarp();
        if (j < P2 && (j & 1) == 0) {
            const uint32_t k = nodes + (j >> 1);
            nc[k] = val + pval; par[idx] = (int32_t)k; par[pidx] = (int32_t)k;
        }
        const uint32_t nl = (uint32_t)__popc(lm);
        lp += nl; ip += P2 - nl; nodes += P2 >> 1;
        __syncwarp();
    }
    return nodes;
}

__device__ __forceinline__ uint32_t wsel(uint32_t lo, uint32_t hi, uint32_t i) {
    return __shfl_sync(0xffffffffu, i >= 32 ? hi : lo, i & 31);
}
__device__ void huff_merge_regs(const uint64_t *keys, uint32_t n, int32_t *par, int lane) {
    const uint32_t L0 = (uint32_t)lane < n ? (uint32_t)(keys[lane] >> 25) : 0u;
    const uint32_t L1 = (uint32_t)lane + 32 < n ? (uint32_t)(keys[lane + 32] >> 25) : 0u;
    uint32_t I0 = 0, I1 = 0;                         // internal node counts
    int32_t lp0 = -1, lp1 = -1, ip0 = -1, ip1 = -1;  // parents (global node index)
    uint32_t lp = 0, ip = 0, ni = 0;                 // leaf head, internal head, internal nodes
    uint32_t lv = wsel(L0, L1, 0), iv = 0;
    while ((n - lp) + (ni - ip) >= 2) {
        const uint32_t l1 = wsel(L0, L1, min(lp + 1, 63u)), l2 = wsel(L0, L1, min(lp + 2, 63u));
        const uint32_t i1 = wsel(I0, I1, min(ip + 1, 63u)), i2 = wsel(I0, I1, min(ip + 2, 63u));
        uint32_t pk[2], pv[2];
        bool pl_[2];
        uint32_t ln = l1, in = i1; // the heads after the current ones
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const bool take_leaf = lp < n && (ip >= ni || lv <= iv);
            pl_[k] = take_leaf;
            if (take_leaf) {
                pk[k] = lp;
                pv[k] = lv;
                ++lp;
                lv = ln;
                ln = l2;
            } else {
                pk[k] = ip;
                pv[k] = iv;
                ++ip;
                iv = in;
                in = i2;
            }
        }
        const uint32_t sum = pv[0] + pv[1];
        const int32_t node = (int32_t)(n + ni);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t q = pk[k];
            if ((uint32_t)lane == (q & 31)) {
                if (pl_[k]) {
                    if (q < 32) lp0 = node; else lp1 = node;
                } else {
                    if (q < 32) ip0 = node; else ip1 = node;
                }
            }
        }
        if ((uint32_t)lane == (ni & 31)) {
            if (ni < 32) I0 = sum; else I1 = sum;
        }
        if (ip == ni) iv = sum; // the internal queue was empty
        ++ni;
    }
    if ((uint32_t)lane < n) par[lane] = lp0;
    if ((uint32_t)lane + 32 < n) par[lane + 32] = lp1;
    if ((uint32_t)lane < ni) par[n + lane] = ip0;
    if ((uint32_t)lane + 32 < ni) par[n + lane + 32] = ip1;
    __syncwarp();
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

__global__ void bench(int mode, uint32_t n, uint32_t *gscratch, long long *cyc, unsigned long long *ns, uint32_t *out) {
    __shared__ uint32_t nc_s[2048];
    __shared__ int32_t par_s[2048];
    const int tid = threadIdx.x;
    uint32_t *nc = (mode & 4) ? gscratch + blockIdx.x * 4096 : nc_s;
    int32_t *par = (mode & 4) ? (int32_t *)(gscratch + blockIdx.x * 4096 + 2048) : par_s;
    // skewed sorted counts: geometric-ish
    for (uint32_t i = tid; i < n; i += blockDim.x) { nc[i] = 1u + (i * i * i) / 7u + (i > n - 3 ? 100000u * i : 0u); par[i] = -1; }
    __syncthreads();
    long long t0 = clock64();
    unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    uint32_t nodes = 0;
    if ((mode & 3) == 0) { if (tid == 0) nodes = merge_serial(nc, par, n); }
    else if ((mode & 3) == 1) { if (tid < 32) nodes = merge_warp(nc, par, n, tid); }
    else if ((mode & 3) == 2) { if (tid == 0) nodes = huff_merge_serial(nc_s, par_s, n); }
    else { if (tid < 32) nodes = merge_warp(nc_s, par_s, n, tid); }
    __syncthreads();
    long long t1 = clock64();
    unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (tid == 0) { cyc[blockIdx.x] = t1 - t0; ns[blockIdx.x] = g1 - g0; out[blockIdx.x] = nodes + nc[nodes - 1]; }
}

int main() {
    uint32_t *g, *out; long long *cyc; unsigned long long *ns;
    cudaMalloc(&g, 128 * 4096 * 4); cudaMalloc(&out, 128 * 4); cudaMalloc(&cyc, 128 * 8); cudaMalloc(&ns, 128 * 8);
    const char *names[] = {"serial/generic", "warp/generic", "serial/prefetch", "warp/smem"};
    for (uint32_t n : {8u, 38u, 200u, 1000u})
        for (int mode = 0; mode < 8; ++mode) {
            for (int rep = 0; rep < 3; ++rep) bench<<<128, 256>>>(mode, n, g, cyc, ns, out);
            cudaDeviceSynchronize();
            long long hc[128]; unsigned long long hn[128]; uint32_t ho[128];
            cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
            cudaMemcpy(hn, ns, sizeof hn, cudaMemcpyDeviceToHost);
            cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
            double c = 0, t = 0; for (int i = 0; i < 128; ++i) { c += hc[i]; t += hn[i]; }
            printf("n=%4u %-16s %s cycles %9.0f  ns %9.0f  check %u\n", n, names[mode & 3], (mode & 4) ? "gmem" : "    ", c / 128, t / 128, ho[0]);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
