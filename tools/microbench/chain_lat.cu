// Dependent FP64 add chains with different operand sources (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_const(double *out, long long *cyc, int iters) {
    double d = threadIdx.x, b = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 32; ++j) d = __dadd_rn(d, b);
    }
    *cyc = clock64() - t0; out[threadIdx.x] = d;
}
__global__ void k_regs(double *out, long long *cyc, int iters) {
    double c[32];
    for (int j = 0; j < 32; ++j) c[j] = 1e-9 * (j + threadIdx.x);
    double d = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 32; ++j) d = __dadd_rn(d, c[j]);
    }
    *cyc = clock64() - t0; out[threadIdx.x] = d;
}
__global__ void k_smem(double *out, long long *cyc, int iters) {
    __shared__ double s[1024];
    for (int j = threadIdx.x; j < 1024; j += 32) s[j] = 1e-9 * j;
    __syncwarp();
    double d = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int base = (i * 32) & 1023;
#pragma unroll
        for (int j = 0; j < 32; ++j) d = __dadd_rn(d, s[base + j]);
    }
    *cyc = clock64() - t0; out[threadIdx.x] = d;
}
__global__ void k_smem_store(double *out, long long *cyc, int iters) {
    __shared__ double s[1024];
    for (int j = threadIdx.x; j < 1024; j += 32) s[j] = 1e-9 * j;
    __syncwarp();
    double d = threadIdx.x, mine = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int base = (i * 32) & 1023;
        double dd[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { d = __dadd_rn(d, s[base + j]); dd[j] = d; }
#pragma unroll
        for (int j = 0; j < 32; ++j) if ((int)threadIdx.x == j) mine = dd[j];
        out[(i & 63) * 32 + threadIdx.x] = mine;
    }
    *cyc = clock64() - t0; out[threadIdx.x] += d;
}
int main() {
    double *out; long long *cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    const char *names[] = {"const b", "regs c[j]", "smem s[j]", "smem + store"};
    for (int v = 0; v < 4; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) k_const<<<1, 32>>>(out, cyc, iters);
            if (v == 1) k_regs<<<1, 32>>>(out, cyc, iters);
            if (v == 2) k_smem<<<1, 32>>>(out, cyc, iters);
            if (v == 3) k_smem_store<<<1, 32>>>(out, cyc, iters);
            cudaDeviceSynchronize();
        }
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-14s %.2f cycles per dependent DADD\n", names[v], (double)c / (iters * 32.0));
    }
    return 0;
}
