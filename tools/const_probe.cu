// const_probe.cu -- dev prototype: Stokes SL+DL pair loop with the source tile in the constant
// bank (uniform-register operands) vs shared memory.  Measures SMSP cycles per warp-pair.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NS = 600;                       // sources per tile (80 B each -> 64 KB)
__constant__ double csrc[NS * 10];
__device__ __forceinline__ double rsq(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

template <int J>
__device__ __forceinline__ void pairs(const double (&x)[J][3], const double* s, double (&acc)[J][3]) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
        double rx = x[j][0] - s[0], ry = x[j][1] - s[1], rz = x[j][2] - s[2];
        double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq(r2);
        double e = fma(-r2, y0 * y0, 1.0);
        double h = e * fma(e, 0.375, 0.5);
        double rinv = fma(y0, h, y0);
        rinv = (__double2hiint(r2) == 0) ? 0.0 : rinv;
        double s2 = rinv * rinv;
        double rg = fma(rx, s[6], fma(ry, s[7], rz * s[8]));
        double ra = fma(rx, s[3], fma(ry, s[4], rz * s[5]));
        double c = (rg * s2) * fma(ra, s2, 1.0);
        acc[j][0] = fma(rinv, fma(c, rx, s[6]), acc[j][0]);
        acc[j][1] = fma(rinv, fma(c, ry, s[7]), acc[j][1]);
        acc[j][2] = fma(rinv, fma(c, rz, s[8]), acc[j][2]);
    }
}

template <int J, int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) kconst(const double* xt, double* out, int reps) {
    double x[J][3], acc[J][3];
    for (int j = 0; j < J; ++j) { long t = (long)blockIdx.x * 256 * J + threadIdx.x + 256 * j;
        for (int q = 0; q < 3; ++q) { x[j][q] = xt[3 * t + q]; acc[j][q] = 0; } }
    for (int r = 0; r < reps; ++r) {
#pragma unroll UNR
        for (int m = 0; m < NS; ++m) pairs<J>(x, csrc + 10 * m, acc);
    }
    for (int j = 0; j < J; ++j) { long t = (long)blockIdx.x * 256 * J + threadIdx.x + 256 * j;
        for (int q = 0; q < 3; ++q) out[3 * t + q] = acc[j][q]; }
}

template <int J, int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) ksmem(const double* xt, const double* src, double* out, int reps) {
    __shared__ double ss[NS * 10];
    for (int q = threadIdx.x; q < NS * 10; q += 256) ss[q] = src[q];
    __syncthreads();
    double x[J][3], acc[J][3];
    for (int j = 0; j < J; ++j) { long t = (long)blockIdx.x * 256 * J + threadIdx.x + 256 * j;
        for (int q = 0; q < 3; ++q) { x[j][q] = xt[3 * t + q]; acc[j][q] = 0; } }
    for (int r = 0; r < reps; ++r) {
#pragma unroll UNR
        for (int m = 0; m < NS; ++m) pairs<J>(x, ss + 10 * m, acc);
    }
    for (int j = 0; j < J; ++j) { long t = (long)blockIdx.x * 256 * J + threadIdx.x + 256 * j;
        for (int q = 0; q < 3; ++q) out[3 * t + q] = acc[j][q]; }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8;          // whole waves for 1..4 CTAs/SM
    const long T = (long)blocks * 256 * 4;
    double *xt, *out, *src;
    cudaMalloc(&xt, T * 3 * 8); cudaMalloc(&out, T * 3 * 8); cudaMalloc(&src, NS * 80);
    double* h = new double[T * 3];
    for (long i = 0; i < T * 3; ++i) h[i] = (i * 0.6180339887) - (long)(i * 0.6180339887) + 2.0;
    cudaMemcpy(xt, h, T * 24, cudaMemcpyHostToDevice);
    double hs[NS * 10];
    for (int m = 0; m < NS; ++m) { for (int q = 0; q < 3; ++q) hs[10 * m + q] = 0.001 * m + q * 0.3;
        for (int q = 3; q < 9; ++q) hs[10 * m + q] = 0.1 + 0.001 * q; hs[10 * m + 9] = 0; }
    cudaMemcpyToSymbol(csrc, hs, sizeof(hs)); cudaMemcpy(src, hs, sizeof(hs), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto report = [&](const char* nm, int J, float ms, int reps) {
        long Tj = (long)blocks * 256 * J;
        double pairs = (double)Tj * NS * reps;
        double cyc = ms * 1e-3 * 1.965e9 * sms * 4 / (pairs / 32);
        printf("%-24s J=%d  %.3f ms  %.1f Gpair/s  %.1f SMSP cyc/warp-pair  %.1f%% of 37.2TF\n", nm, J, ms, pairs / ms / 1e6,
               cyc, pairs * 39 / (ms * 1e-3) / 37.22e12 * 100);
    };
#define RUN(KER, J, U, MB, ...) { KER<J, U, MB><<<blocks, 256>>>(__VA_ARGS__, 2); cudaEventRecord(e0); \
    KER<J, U, MB><<<blocks, 256>>>(__VA_ARGS__, 20); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; \
    cudaEventElapsedTime(&ms, e0, e1); char nm[64]; snprintf(nm, 64, #KER " U%d MB%d", U, MB); report(nm, J, ms, 20); }
    RUN(ksmem, 2, 4, 2, xt, src, out)
    RUN(kconst, 2, 4, 2, xt, out)
    RUN(kconst, 2, 2, 2, xt, out)
    RUN(kconst, 4, 2, 1, xt, out)
    RUN(kconst, 4, 2, 2, xt, out)
    RUN(kconst, 1, 4, 4, xt, out)
    RUN(kconst, 2, 4, 3, xt, out)
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
