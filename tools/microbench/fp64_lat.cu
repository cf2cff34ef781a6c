// Microbenchmark: dependent-chain latency of FP64 ops on sm_100a (B200).
// Used to size the serial predictor chain of the encoder.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double *out, long long *cyc, double a, double b, int iters) {
    double x = a + threadIdx.x * 1e-30;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = __dadd_rn(x, b);
        if (OP == 1) x = __dmul_rn(x, b);
        if (OP == 2) x = __ddiv_rn(x, b);
        if (OP == 3) x = __dadd_rn(x, (double)llround(__ddiv_rn(__dadd_rn(x, -a), b)));
        if (OP == 4) { // full closed-loop quantizer step (T1)
            double r = __ddiv_rn(__dadd_rn(a, -x), b);
            long long m = llround(r);
            double rec = __dadd_rn(x, __dmul_rn(b, (double)m));
            x = fabs(__dadd_rn(a, -rec)) <= b ? rec : a + 1e-3 * i;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x + blockIdx.x * blockDim.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *out; long long *cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    const char *names[] = {"dadd", "dmul", "ddiv", "sub+div+llround+add", "T1 quantizer step"};
    int iters = 1 << 16;
    for (int op = 0; op < 5; ++op) {
        for (int warps : {1, 4, 16, 64}) {
            long long c = 0;
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto launch = [&](int blocks) {
                switch (op) {
                case 0: chain<0><<<blocks, 32 * (warps > 32 ? 32 : warps)>>>(out, cyc, 1.0, 1e-9, iters); break;
                case 1: chain<1><<<blocks, 32 * (warps > 32 ? 32 : warps)>>>(out, cyc, 1.0, 1.0000001, iters); break;
                case 2: chain<2><<<blocks, 32 * (warps > 32 ? 32 : warps)>>>(out, cyc, 1.0, 1.0000001, iters); break;
                case 3: chain<3><<<blocks, 32 * (warps > 32 ? 32 : warps)>>>(out, cyc, 1.0, 3.0, iters); break;
                case 4: chain<4><<<blocks, 32 * (warps > 32 ? 32 : warps)>>>(out, cyc, 0.3, 2e-5, iters); break;
                }
            };
            int blocks = warps > 32 ? 148 * (warps / 32) : 1;
            launch(blocks); cudaDeviceSynchronize();
            cudaEventRecord(e0); launch(blocks); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            double thr = (double)blocks * 32 * (warps > 32 ? 32 : warps) * iters / (ms * 1e-3);
            printf("%-24s warps/blk=%2d blocks=%4d  cyc/iter(thread0)=%7.2f  chip ops/s=%.3e\n", names[op],
                   warps > 32 ? 32 : warps, blocks, (double)c / iters, thr);
        }
    }
    return 0;
}
