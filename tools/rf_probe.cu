// rf_probe.cu -- dev microbenchmark: FP64 throughput vs number of distinct register operands.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(long iters, const double* in, double* out) {
    double a[8], b[8], c[8];
    for (int q = 0; q < 8; ++q) { a[q] = in[q] + threadIdx.x; b[q] = in[8 + q] * 0.5 + threadIdx.x * 1e-9; c[q] = in[16 + q] * 1e-3 + threadIdx.x * 1e-9; }
    const double bb = in[24];
    for (long i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (MODE == 0) a[q] = fma(b[q], c[q], a[q]);        // 3 distinct registers
                if (MODE == 1) a[q] = fma(a[q], b[q], a[q]);        // 2 distinct
                if (MODE == 2) a[q] = fma(bb, c[q], a[q]);          // shared B operand (reuse candidate)
                if (MODE == 3) a[q] = a[q] * b[q];                  // DMUL 2 distinct
                if (MODE == 4) a[q] = fma(b[q], 0.999, a[q]);      // reg, imm, reg
            }
    }
    double s = 0; for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 1234.5) out[0] = s;
}
template <int MODE> void run(const char* nm) {
    double h[32]; for (int q = 0; q < 32; ++q) h[q] = 1.0 + q * 1e-3;
    double *d, *o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long iters = 20000; dim3 g(sms * 4), b(512);
    k<MODE><<<g, b>>>(iters / 10, d, o);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<MODE><<<g, b>>>(iters, d, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_iters = (double)iters * g.x * b.x / 32.0 / sms / 4.0;
    printf("%-34s %.3f ms  SMSP cycles per FP64 instr %.3f\n", nm, ms, ms * 1e-3 * 1.965e9 / warp_iters / 16.0);
}
int main() {
    run<0>("DFMA b,c,a (3 distinct)"); run<1>("DFMA a,b,a (2 distinct)"); run<2>("DFMA bb,c,a (shared B)");
    run<3>("DMUL a,b"); run<4>("DFMA b,imm,a");
    return 0;
}
