// farconst.cu -- far field for the operator apply with source tiles in the CONSTANT bank.
//
// Why (measured): on sm_100a an FP64 instruction whose three source
// operands are distinct vector registers occupies the FP64 pipe for 3 cycles instead of 2
// (tools/rf_probe.cu).  In the N-body pair every source value (y, a, g) is warp-uniform; read
// from shared memory it lands in vector registers and ~8 of the 27 FP64 instructions per pair
// pay the third cycle (tools/sass_cost.py).  Read from the constant bank with a uniform index it
// is loaded by LDCU into UNIFORM registers, which are free operands: the modelled pair cost drops
// from 61 to 55 cycles per warp and the measured pair rate rises ~8% (tools/const_probe.cu).
//
// Structure: the packed source records rec[m] = {y(3), a(3), g(3), 0} (80 B) are split into
// tiles of 200 sources.  Tile i is copied (D2D, stream-ordered) into constant buffer i % nb
// (nb = 4; the bank can also be split 8 x 100) and processed by a launch on internal stream i % nb over ALL
// local targets; stream s accumulates its tiles s, s+nb, ... into its own partial array, so the
// summation order per target depends only on M and the nb kernels in flight hide each other's
// tails.  The whole sequence is captured once into a CUDA graph per operator and replayed per apply.
#include <cuda_runtime.h>
#include <cstdlib>
#include <mutex>
#include <vector>
#include "common.cuh"

namespace slb {

constexpr int kConstRecs = 800;          // records the constant bank holds (800 x 80 B = 64 KB)
constexpr int kMaxConstBufs = 8;         // buffers = streams = partial arrays: 4 x 200 or 8 x 100 records
constexpr int kRec = 10;                 // doubles per packed record
constexpr int kConstThreads = 128;
constexpr int kSlot = kConstRecs / kMaxConstBufs * kRec;   // doubles per 1/8 of the bank

__constant__ double c_rec[kConstRecs * kRec];

// buffers for M sources (a function of M only: every rank of a sharded operator sums in the same
// order).  8 x 100 records was measured too: slower on c3 / c3v (far 7.90 / 9.52 ms vs 7.33 / 9.05 ms
// with 4 x 200) -- twice the launches and copies cost more than the better SM fill gains.
static int const_bufs_for(int64_t M) { (void)M; return 4; }

template <int KIND, int J, int CM, int ORD = 3>
__device__ __forceinline__ void const_pairs(const double (&x)[J][3], const double* s, double (&acc)[J][3],
                                            bool& anyz, unsigned& zc) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const double rx = x[j][0] - s[0], ry = x[j][1] - s[1], rz = x[j][2] - s[2];
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        const double y0 = rsqrt_mufu(r2);
        const double e = fma(-r2, y0 * y0, 1.0);
        double h;
        if constexpr (ORD == 3) h = e * fma(e, 0.375, 0.5);
        else if constexpr (ORD == 4) {                 // cubic term (~2^-46 y0) in FP32: one FP64 instruction fewer
            const float ef = __double2float_rn(e);
            h = fma(e, 0.5, (double)(0.375f * ef * ef));
        } else h = 0.5 * e;                            // ORD 2: measurement only (error ~3/8 e^2 ~ 2e-14)
        double rinv = fma(y0, h, y0);                  // y0 (1 + e/2 + 3e^2/8)
        if constexpr (CM != 2) {                       // CM 2: no coincident-pair handling (measurement only)
            const bool z = is_zero_r2(r2);
            rinv = z ? 0.0 : rinv;
            if (CM == 0) anyz |= z;                    // rare: exact recount after the loop
            else zc += z;
        }
        if constexpr (KIND == FAR_STOKES_SLDL) {
            // u += rinv (g + c r),  c = (r.g) rinv^2 (1 + (r.a) rinv^2)
            const double s2 = rinv * rinv;
            const double rg = fma(rx, s[6], fma(ry, s[7], rz * s[8]));
            const double ra = fma(rx, s[3], fma(ry, s[4], rz * s[5]));
            const double c = (rg * s2) * fma(ra, s2, 1.0);
            acc[j][0] = fma(rinv, fma(c, rx, s[6]), acc[j][0]);
            acc[j][1] = fma(rinv, fma(c, ry, s[7]), acc[j][1]);
            acc[j][2] = fma(rinv, fma(c, rz, s[8]), acc[j][2]);
        } else if constexpr (KIND == FAR_STOKES_DL) {
            // u += (r.a)(r.g) rinv^5 r
            const double s2 = rinv * rinv;
            const double ra = fma(rx, s[3], fma(ry, s[4], rz * s[5]));
            const double rd = fma(rx, s[6], fma(ry, s[7], rz * s[8]));
            const double b = (ra * rd) * ((s2 * s2) * rinv);
            acc[j][0] = fma(b, rx, acc[j][0]);
            acc[j][1] = fma(b, ry, acc[j][1]);
            acc[j][2] = fma(b, rz, acc[j][2]);
        } else if constexpr (KIND == FAR_LAPLACE_SLDL) {
            // Laplace D + eta S_L: u += rinv ((r.q) rinv^2 + s)
            const double rq = fma(rx, s[6], fma(ry, s[7], rz * s[8]));
            acc[j][0] = fma(rinv, fma(rq, rinv * rinv, s[9]), acc[j][0]);
        } else {
            // Laplace DL: u += (r.q) rinv^3
            const double rq = fma(rx, s[6], fma(ry, s[7], rz * s[8]));
            acc[j][0] = fma(rq, (rinv * rinv) * rinv, acc[j][0]);
        }
    }
}

template <int KIND, int J, int BUF, int CM, int UNR = 4, int MINB = 4, int ORD = 3>
__global__ void __launch_bounds__(kConstThreads, MINB)
far_const_kernel(int64_t T, const double* __restrict__ x_trg, int n_src, int first,
                 double* __restrict__ partial, unsigned long long* __restrict__ coincident) {
    constexpr int D = far_scalar(KIND) ? 1 : 3;
    double x[J][3], acc[J][3];
    bool valid[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int64_t t = (int64_t)blockIdx.x * kConstThreads * J + threadIdx.x + kConstThreads * j;
        valid[j] = t < T;
        const int64_t tc = valid[j] ? t : T - 1;
        x[j][0] = x_trg[3 * tc]; x[j][1] = x_trg[3 * tc + 1]; x[j][2] = x_trg[3 * tc + 2];
#pragma unroll
        for (int q = 0; q < 3; ++q) acc[j][q] = (q < D && !first) ? partial[tc * D + q] : 0.0;
    }
    bool anyz = false;
    unsigned zc0 = 0;
    const double* base = c_rec + BUF * kSlot;     // BUF: buffer offset in eighths of the bank
#pragma unroll UNR
    for (int m = 0; m < n_src; ++m) const_pairs<KIND, J, CM, ORD>(x, base + kRec * m, acc, anyz, zc0);
    if (CM == 1 && zc0) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < J; ++j) any |= valid[j];
        if (any) atomicAdd(coincident, (unsigned long long)zc0);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int64_t t = (int64_t)blockIdx.x * kConstThreads * J + threadIdx.x + kConstThreads * j;
        if (valid[j]) {
#pragma unroll
            for (int q = 0; q < D; ++q) partial[t * D + q] = acc[j][q];
        }
    }
    // coincident (r = 0) pairs: recount exactly, only in threads that saw one (valid targets only)
    if (anyz) {
        unsigned long long zc = 0;
        for (int m = 0; m < n_src; ++m)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const double rx = x[j][0] - base[kRec * m], ry = x[j][1] - base[kRec * m + 1],
                             rz = x[j][2] - base[kRec * m + 2];
                zc += (valid[j] && is_zero_r2(fma(rx, rx, fma(ry, ry, rz * rz)))) ? 1 : 0;
            }
        if (zc) atomicAdd(coincident, zc);
    }
}

// Variant with fewer NON-FP64 instructions per pair (the FP64 count stays 27): source record read as
// five 16-byte constant loads, the coincident-pair select applied to the high word of the MUFU seed
// only (its low word is zero), coincident pairs detected through a running minimum of r2's high word
// and recounted exactly after the loop (rare).
template <int J>
__device__ __forceinline__ void const_pairs_lean(const double (&x)[J][3], const double2* s, double (&acc)[J][3],
                                                 unsigned& mn) {
    const double2 q0 = s[0], q1 = s[1], q2 = s[2], q3 = s[3], q4 = s[4];
    const double y_0 = q0.x, y_1 = q0.y, y_2 = q1.x, a0 = q1.y, a1 = q2.x, a2 = q2.y, g0 = q3.x, g1 = q3.y, g2 = q4.x;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const double rx = x[j][0] - y_0, ry = x[j][1] - y_1, rz = x[j][2] - y_2;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        const unsigned hi = (unsigned)__double2hiint(r2);
        int yh = __double2hiint(rsqrt_mufu(r2));
        yh = hi ? yh : 0;                               // coincident pair (R14): seed 0 -> rinv = 0
        mn = min(mn, hi);
        const double y0 = __hiloint2double(yh, 0);
        const double e = fma(-r2, y0 * y0, 1.0);
        const double h = e * fma(e, 0.375, 0.5);
        const double rinv = fma(y0, h, y0);
        const double s2 = rinv * rinv;
        const double rg = fma(rx, g0, fma(ry, g1, rz * g2));
        const double ra = fma(rx, a0, fma(ry, a1, rz * a2));
        const double c = (rg * s2) * fma(ra, s2, 1.0);
        acc[j][0] = fma(rinv, fma(c, rx, g0), acc[j][0]);
        acc[j][1] = fma(rinv, fma(c, ry, g1), acc[j][1]);
        acc[j][2] = fma(rinv, fma(c, rz, g2), acc[j][2]);
    }
}

template <int J, int BUF, int UNR, int MINB>
__global__ void __launch_bounds__(kConstThreads, MINB)
far_const_lean_kernel(int64_t T, const double* __restrict__ x_trg, int n_src, int first,
                      double* __restrict__ partial, unsigned long long* __restrict__ coincident) {
    double x[J][3], acc[J][3];
    bool valid[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int64_t t = (int64_t)blockIdx.x * kConstThreads * J + threadIdx.x + kConstThreads * j;
        valid[j] = t < T;
        const int64_t tc = valid[j] ? t : T - 1;
        x[j][0] = x_trg[3 * tc]; x[j][1] = x_trg[3 * tc + 1]; x[j][2] = x_trg[3 * tc + 2];
#pragma unroll
        for (int q = 0; q < 3; ++q) acc[j][q] = first ? 0.0 : partial[tc * 3 + q];
    }
    unsigned mn = 0xffffffffu;
    const double* base = c_rec + BUF * kSlot;
    const double2* b2 = reinterpret_cast<const double2*>(base);
#pragma unroll UNR
    for (int m = 0; m < n_src; ++m) const_pairs_lean<J>(x, b2 + (kRec / 2) * m, acc, mn);
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int64_t t = (int64_t)blockIdx.x * kConstThreads * J + threadIdx.x + kConstThreads * j;
        if (valid[j]) {
#pragma unroll
            for (int q = 0; q < 3; ++q) partial[t * 3 + q] = acc[j][q];
        }
    }
    if (mn == 0) {   // some pair of this thread was coincident: count exactly (valid targets only)
        unsigned long long zc = 0;
        for (int m = 0; m < n_src; ++m)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const double rx = x[j][0] - base[kRec * m], ry = x[j][1] - base[kRec * m + 1],
                             rz = x[j][2] - base[kRec * m + 2];
                zc += (valid[j] && is_zero_r2(fma(rx, rx, fma(ry, ry, rz * rz)))) ? 1 : 0;
            }
        if (zc) atomicAdd(coincident, zc);
    }
}

// rec[m] = {geo[m][0..5], dyn[m][0..2], 0}
__global__ void pack_rec_kernel(int64_t M, const double* __restrict__ geo, const double* __restrict__ dyn,
                                double* __restrict__ rec) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    const double2* g = reinterpret_cast<const double2*>(geo + m * 6);
    const double2* d = reinterpret_cast<const double2*>(dyn + m * 4);
    double2* o = reinterpret_cast<double2*>(rec + m * kRec);
    o[0] = g[0]; o[1] = g[1]; o[2] = g[2];
    const double2 d0 = d[0], d1 = d[1];
    o[3] = d0;
    o[4] = d1;                 // {g_z, 0} (Stokes) or {q_z, s} (Laplace combined field)
}

constexpr int kJ = 2;

// environment knobs: read once (function-local statics: thread-safe initialisation)
static int const_count_mode() {
    // 1 (default): per-pair count -- measured faster than flag+recount (profiles/r01_bench_c4_cm*.json)
    static const int v = [] { const char* e = getenv("SLB_CONST_COUNT"); return (e && e[0] == '0') ? 0 : 1; }();
    return v;
}

static int const_variant() {
    static const int v = [] { const char* e = getenv("SLB_CONST_VARIANT"); return e ? atoi(e) : 0; }();
    return v;
}

template <int KIND, int BUF, int J, int UNR, int MINB, int CM = 1, int ORD = 3>
static void launch_tile_v(int64_t T, const double* x, int n, int first, double* part, unsigned long long* zc,
                          cudaStream_t s) {
    const unsigned grid = (unsigned)((T + kConstThreads * J - 1) / (kConstThreads * J));
    far_const_kernel<KIND, J, BUF, CM, UNR, MINB, ORD><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc);
}

template <int KIND, int BUF>
static void launch_tile(int64_t T, const double* x, int n, int first, double* part, unsigned long long* zc,
                        cudaStream_t s, bool check) {
    const unsigned grid = (unsigned)((T + kConstThreads * kJ - 1) / (kConstThreads * kJ));
    if (!check) {
        far_const_kernel<KIND, kJ, BUF, 2><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc);
        return;
    }
    if (KIND == FAR_STOKES_SLDL && const_variant() != 0) {
        switch (const_variant()) {
            case 1: launch_tile_v<KIND, BUF, 2, 2, 4>(T, x, n, first, part, zc, s); return;
            case 2: launch_tile_v<KIND, BUF, 2, 8, 4>(T, x, n, first, part, zc, s); return;
            case 3: launch_tile_v<KIND, BUF, 3, 2, 3>(T, x, n, first, part, zc, s); return;
            case 4: launch_tile_v<KIND, BUF, 1, 8, 8>(T, x, n, first, part, zc, s); return;
            case 8: launch_tile_v<KIND, BUF, 2, 4, 4, 2, 3>(T, x, n, first, part, zc, s); return;   // no r = 0 handling
            case 9: launch_tile_v<KIND, BUF, 2, 4, 4, 2, 2>(T, x, n, first, part, zc, s); return;   // + 2nd-order rsqrt
            case 10: launch_tile_v<KIND, BUF, 2, 4, 4, 1, 2>(T, x, n, first, part, zc, s); return;  // 2nd-order rsqrt only
            case 12: launch_tile_v<KIND, BUF, 2, 4, 4, 1, 4>(T, x, n, first, part, zc, s); return;  // FP32 cubic term
            case 13: launch_tile_v<KIND, BUF, 2, 4, 4, 2, 4>(T, x, n, first, part, zc, s); return;  // + no r = 0 handling
            case 11: launch_tile_v<KIND, BUF, 2, 4, 5>(T, x, n, first, part, zc, s); return;         // 5 CTAs/SM (<= 102 regs)
            case 6: far_const_lean_kernel<2, BUF, 4, 4><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc); return;
            case 7: far_const_lean_kernel<2, BUF, 2, 4><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc); return;
            default: launch_tile_v<KIND, BUF, 4, 1, 2>(T, x, n, first, part, zc, s); return;
        }
    }
    if (const_count_mode() == 1)
        far_const_kernel<KIND, kJ, BUF, 1><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc);
    else
        far_const_kernel<KIND, kJ, BUF, 0><<<grid, kConstThreads, 0, s>>>(T, x, n, first, part, zc);
}

template <int KIND>
static void launch_tile_buf(int slot, int64_t T, const double* x, int n, int first, double* part,
                            unsigned long long* zc, cudaStream_t s, bool check) {
    switch (slot) {
        case 0: launch_tile<KIND, 0>(T, x, n, first, part, zc, s, check); break;
        case 1: launch_tile<KIND, 1>(T, x, n, first, part, zc, s, check); break;
        case 2: launch_tile<KIND, 2>(T, x, n, first, part, zc, s, check); break;
        case 3: launch_tile<KIND, 3>(T, x, n, first, part, zc, s, check); break;
        case 4: launch_tile<KIND, 4>(T, x, n, first, part, zc, s, check); break;
        case 5: launch_tile<KIND, 5>(T, x, n, first, part, zc, s, check); break;
        case 6: launch_tile<KIND, 6>(T, x, n, first, part, zc, s, check); break;
        default: launch_tile<KIND, 7>(T, x, n, first, part, zc, s, check); break;
    }
}

// Issue the constant-bank far field on nb = const_bufs_for(M) internal streams (forked from/joined to s).
// partials: [nb][T][D].  Returns the number of kernel launches issued.
slb_status far_const_issue(FarKind kind, int64_t M, int64_t T, const double* x, const double* rec,
                           double* partials, unsigned long long* zc, cudaStream_t s, cudaStream_t* ws,
                           cudaEvent_t fork, cudaEvent_t* join, int64_t* launches, bool check) {
    const int D = far_scalar(kind) ? 1 : 3;
    const int nb = const_bufs_for(M);
    const int tile = kConstRecs / nb;                // 200 or 100 records per buffer
    const int stride = kMaxConstBufs / nb;           // buffer b occupies eighth b * stride
    *launches = 0;
    SLB_CUDA(cudaEventRecord(fork, s));
    for (int b = 0; b < nb; ++b) SLB_CUDA(cudaStreamWaitEvent(ws[b], fork, 0));
    const int64_t ntiles = (M + tile - 1) / tile;
    for (int b = 0; b < nb; ++b) {
        double* part = partials + (int64_t)b * T * D;
        if (b >= ntiles && T > 0) SLB_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * T * D, ws[b]));
    }
    for (int64_t i = 0; i < ntiles; ++i) {
        const int b = (int)(i % nb);
        const int64_t m0 = i * tile;
        const int n = (int)std::min<int64_t>(tile, M - m0);
        SLB_CUDA(cudaMemcpyToSymbolAsync(c_rec, rec + m0 * kRec, sizeof(double) * n * kRec,
                                         sizeof(double) * (size_t)b * stride * kSlot, cudaMemcpyDeviceToDevice, ws[b]));
        if (T > 0) {
            double* part = partials + (int64_t)b * T * D;
            const int first = (i < nb) ? 1 : 0;
            switch (kind) {
                case FAR_STOKES_SLDL: launch_tile_buf<FAR_STOKES_SLDL>(b * stride, T, x, n, first, part, zc, ws[b], check); break;
                case FAR_STOKES_DL: launch_tile_buf<FAR_STOKES_DL>(b * stride, T, x, n, first, part, zc, ws[b], check); break;
                case FAR_LAPLACE_SLDL: launch_tile_buf<FAR_LAPLACE_SLDL>(b * stride, T, x, n, first, part, zc, ws[b], check); break;
                default: launch_tile_buf<FAR_LAPLACE>(b * stride, T, x, n, first, part, zc, ws[b], check); break;
            }
            ++*launches;
        }
    }
    for (int b = 0; b < nb; ++b) {
        SLB_CUDA(cudaEventRecord(join[b], ws[b]));
        SLB_CUDA(cudaStreamWaitEvent(s, join[b], 0));
    }
    return check_launch("far_const_kernel");
}

slb_status pack_rec_launch(int64_t M, const double* geo, const double* dyn, double* rec, cudaStream_t s) {
    if (M <= 0) return SLB_OK;
    pack_rec_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(M, geo, dyn, rec);
    ++g_launch_count;
    return check_launch("pack_rec_kernel");
}

// ---- library-wide serialisation of the constant bank (distinct operators are safe
// to apply concurrently).  c_rec is one per device for the whole process; every issue of the tile
// sequence (graph launch or direct) holds this lock, waits on the device's bank event (recorded by
// the previous user, a no-op before the first) and re-records it after its last tile, so the tile
// copies of two operators can never interleave on the device.
namespace {
constexpr int kMaxDevs = 64;
std::mutex g_bank_mu;
cudaEvent_t g_bank_ev[kMaxDevs] = {};
}

ConstBankLock::ConstBankLock() : lk_(g_bank_mu) {}
ConstBankLock::~ConstBankLock() = default;

slb_status ConstBankLock::acquire(cudaStream_t s) {
    int dev = 0;
    SLB_CUDA(cudaGetDevice(&dev));
    SLB_REQUIRE(dev >= 0 && dev < kMaxDevs, SLB_ERR_UNSUPPORTED, "device ordinal beyond the bank table");
    if (!g_bank_ev[dev]) SLB_CUDA(cudaEventCreateWithFlags(&g_bank_ev[dev], cudaEventDisableTiming));
    dev_ = dev;
    SLB_CUDA(cudaStreamWaitEvent(s, g_bank_ev[dev], 0));
    return SLB_OK;
}

slb_status ConstBankLock::release(cudaStream_t s) {
    SLB_CUDA(cudaEventRecord(g_bank_ev[dev_], s));
    return SLB_OK;
}

int far_const_bufs(int64_t M) { return const_bufs_for(M); }
int far_const_tile(int64_t M) { return kConstRecs / const_bufs_for(M); }

// Load this module's kernels and constant symbol eagerly (lazy module loading must not happen
// inside a stream capture).
slb_status far_const_prepare() {
    void* p = nullptr;
    SLB_CUDA(cudaGetSymbolAddress(&p, c_rec));
    cudaFuncAttributes fa;
#define PREP1(K, C) SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 0, C>)); \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 1, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 2, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 3, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 4, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 5, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 6, C>));                 \
    SLB_CUDA(cudaFuncGetAttributes(&fa, far_const_kernel<K, kJ, 7, C>));
#define PREP(K) PREP1(K, 0) PREP1(K, 1) PREP1(K, 2)
    PREP(FAR_STOKES_SLDL)
    PREP(FAR_STOKES_DL)
    PREP(FAR_LAPLACE)
    PREP(FAR_LAPLACE_SLDL)
#undef PREP
#undef PREP1
    SLB_CUDA(cudaFuncGetAttributes(&fa, pack_rec_kernel));
    return SLB_OK;
}

}  // namespace slb
