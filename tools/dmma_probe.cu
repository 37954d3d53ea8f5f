// dmma_probe.cu -- dev microbenchmark: do DMMA (FP64 tensor) and DFMA (FP64 pipe) throughputs add?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NF, int NM>
__global__ void k(long iters, const double* in, double* out) {
    double a[8], c0[4], c1[4];
    for (int q = 0; q < 8; ++q) a[q] = in[q] + threadIdx.x * 1e-9;
    for (int q = 0; q < 4; ++q) { c0[q] = 0; c1[q] = 0; }
    const double b = in[9], c = in[10], ma = in[11] + threadIdx.x * 1e-9, mb = in[12] + threadIdx.x * 1e-9;
    for (long i = 0; i < iters; ++i) {
#pragma unroll
        for (int f = 0; f < NF; ++f) a[f & 7] = fma(a[f & 7], b, c);
#pragma unroll
        for (int m = 0; m < NM; ++m) dmma(c0[m & 3], c1[m & 3], ma, mb);
    }
    double s = 0; for (int q = 0; q < 8; ++q) s += a[q]; for (int q = 0; q < 4; ++q) s += c0[q] + c1[q];
    if (s == 1234.5) out[0] = s;
}
template <int NF, int NM> void run(const char* nm) {
    double h[16]; for (int q = 0; q < 16; ++q) h[q] = 1.0 + q * 1e-3; h[9] = 0.999999; h[10] = 1e-12;
    double *d, *o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long iters = 20000; dim3 g(sms * 4), bl(512);
    k<NF, NM><<<g, bl>>>(iters / 10, d, o);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<NF, NM><<<g, bl>>>(iters, d, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_iters = (double)iters * g.x * bl.x / 32.0 / sms / 4.0;
    double cyc = ms * 1e-3 * 1.965e9 / warp_iters;
    double fl = (2.0 * NF * 32 + 512.0 * NM) * warp_iters * sms * 4 / (ms * 1e-3) / 1e12;
    printf("%-26s NF=%2d NM=%2d  %.3f ms  SMSP cyc/warp-iter %.2f  (DFMA-only %.0f)  %.2f TFLOP/s\n", nm, NF, NM, ms, cyc,
           2.0 * NF, fl);
}
int main() {
    run<16, 0>("dfma only");
    run<0, 4>("dmma only");
    run<0, 8>("dmma only");
    run<16, 4>("dfma + dmma");
    run<16, 2>("dfma + dmma");
    run<16, 1>("dfma + dmma");
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
