// pipe_probe.cu -- dev microbenchmarks of the sm_100a FP64 pipe vs MUFU.RSQ64H (not product code).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq(double x) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

// K DFMA per iteration per chain, 8 chains; R rsqrt per iteration (independent chains)
template <int NF, int NR>
__global__ void mix(long iters, double* out) {
    double a[8], r[4];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
    for (int k = 0; k < 4; ++k) r[k] = 1.0 + threadIdx.x * 1e-7 + k;
    const double b = 0.999999999, c = 1e-12;
    for (long i = 0; i < iters; ++i) {
#pragma unroll
        for (int f = 0; f < NF; ++f) a[f & 7] = fma(a[f & 7], b, c);
#pragma unroll
        for (int q = 0; q < NR; ++q) r[q & 3] = rsq(r[q & 3]) + 0.5;  // DADD keeps it > 0
    }
    double s = 0; for (int k = 0; k < 8; ++k) s += a[k]; for (int k = 0; k < 4; ++k) s += r[k];
    if (s == 1234.5) out[0] = s;
}

template <int NF, int NR>
void run(const char* name) {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long iters = 20000;
    dim3 g(sms * 4), b(512);
    mix<NF, NR><<<g, b>>>(iters / 10, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<NF, NR><<<g, b>>>(iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_iters = (double)iters * g.x * b.x / 32.0 / sms / 4.0;   // per SMSP
    double clk = 1.965e9;
    double cyc = ms * 1e-3 * clk / warp_iters;  // SMSP cycles per warp-iteration
    printf("%-28s NF=%2d NR=%d  %.3f ms  SMSP cycles per warp-iter %.2f  (DFMA-only bound %.1f)\n", name, NF, NR, ms,
           cyc, 2.0 * NF);
    cudaFree(d);
}

int main() {
    run<16, 0>("dfma only");
    run<0, 4>("rsq64h (+dadd) only");
    run<0, 1>("rsq64h (+dadd) x1");
    run<24, 1>("24 dfma + 1 rsq(+dadd)");
    run<26, 1>("26 dfma + 1 rsq(+dadd)");
    run<24, 2>("24 dfma + 2 rsq(+dadd)");
    return 0;
}
