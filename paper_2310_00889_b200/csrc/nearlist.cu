// nearlist.cu -- (NEXT N3) near-list construction on the GPU.
//
// Stands in for the paper's near-region search (§3.3: spheres around the nodes
// of each element, Morton-sorted, overlap search): here the rule of DESIGN.md R15,
//     near(t) = { k : sqrt(min_j |x_t - y_kj|^2) < radius_k }  U  { own_panel[t] },
// evaluated exactly in fp64 with the distance written as ((dx*dx + dy*dy) + dz*dz) without FMA
// contraction, so decisions are bit-identical to the input generator's CPU rule.
// One warp per target scans all panels: a bounding-sphere test (panel centroid + max node
// distance, conservative by a relative 1e-9) prunes, survivors get the exact node minimum;
// warp ballots emit the panel ids in ascending order.  Two passes (count, fill) around an
// exclusive scan; output is the CSR the operator consumes.
#include <algorithm>
#include "common.cuh"

namespace slb {

__global__ void panel_sphere_kernel(int64_t P, int Nn, const double* __restrict__ y, double* __restrict__ sph) {
    const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= P) return;
    const double* yk = y + k * Nn * 3;
    double c[3] = {0, 0, 0};
    for (int j = lane; j < Nn; j += 32)
        for (int q = 0; q < 3; ++q) c[q] += yk[3 * j + q];
    for (int q = 0; q < 3; ++q) {
        for (int off = 16; off > 0; off >>= 1) c[q] += __shfl_xor_sync(0xffffffffu, c[q], off);
        c[q] /= Nn;
    }
    double r = 0.0;
    for (int j = lane; j < Nn; j += 32) {
        const double dx = yk[3 * j] - c[0], dy = yk[3 * j + 1] - c[1], dz = yk[3 * j + 2] - c[2];
        r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
    }
    for (int off = 16; off > 0; off >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, off));
    if (lane == 0) {
        sph[4 * k] = c[0]; sph[4 * k + 1] = c[1]; sph[4 * k + 2] = c[2];
        sph[4 * k + 3] = r * (1.0 + 1e-12) + 1e-300;
    }
}

template <bool FILL>
__global__ void __launch_bounds__(256)
near_build_kernel(int64_t T, const double* __restrict__ x, int64_t P, int Nn, const double* __restrict__ y,
                  const double* __restrict__ radius, const double* __restrict__ sph,
                  const int64_t* __restrict__ own, int64_t* __restrict__ counts_or_rowptr,
                  int32_t* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= T) return;
    const double x0 = x[3 * t], x1 = x[3 * t + 1], x2 = x[3 * t + 2];
    const int64_t ow = own ? own[t] : -1;
    int64_t base = FILL ? counts_or_rowptr[t] : 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t k0 = 0; k0 < P; k0 += 32) {
        const int64_t k = k0 + lane;
        bool near = false;
        if (k < P) {
            const double lim = radius[k];
            if (k == ow) {
                near = true;
            } else {
                const double cx = x0 - sph[4 * k], cy = x1 - sph[4 * k + 1], cz = x2 - sph[4 * k + 2];
                const double dc = sqrt(cx * cx + cy * cy + cz * cz);
                if (dc - sph[4 * k + 3] < lim * (1.0 + 1e-9)) {
                    const double* yk = y + k * Nn * 3;
                    double m = __longlong_as_double(0x7ff0000000000000ll);
                    for (int j = 0; j < Nn; ++j) {
                        const double dx = __dsub_rn(x0, yk[3 * j]);
                        const double dy = __dsub_rn(x1, yk[3 * j + 1]);
                        const double dz = __dsub_rn(x2, yk[3 * j + 2]);
                        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                        m = fmin(m, d2);
                    }
                    near = __dsqrt_rn(m) < lim;
                }
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, near);
        if (FILL && near) out[base + __popc(mask & lt)] = (int32_t)k;
        base += __popc(mask);
    }
    if (!FILL && lane == 0) counts_or_rowptr[t] = base;
}

// exclusive scan of counts[0..n) into row_ptr[0..n] (single CTA, chunked; setup-time only)
__global__ void __launch_bounds__(1024) scan_kernel(int64_t n, const int64_t* __restrict__ counts,
                                                    int64_t* __restrict__ row_ptr) {
    __shared__ int64_t s[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < n; c0 += 1024) {
        const int64_t i = c0 + threadIdx.x;
        const int64_t v = i < n ? counts[i] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const int64_t a = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += a;
            __syncthreads();
        }
        if (i < n) row_ptr[i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) row_ptr[n] = carry;
}

}  // namespace slb

using namespace slb;

extern "C" slb_status slb_near_build(int64_t n_trg, const double* x_trg, int64_t n_panels, int nodes_per_panel,
                                     const double* y_nodes, const double* radius, const int64_t* own_panel,
                                     int64_t* row_ptr, int32_t* panel_idx, int64_t capacity, int64_t* nnz_out,
                                     cudaStream_t s) {
    SLB_REQUIRE(n_trg >= 0 && n_panels >= 0 && nodes_per_panel > 0, SLB_ERR_INVALID_ARG, "bad sizes");
    SLB_REQUIRE(row_ptr && nnz_out, SLB_ERR_INVALID_ARG, "row_ptr and nnz_out are required");
    SLB_REQUIRE(n_trg == 0 || (x_trg && (n_panels == 0 || (y_nodes && radius))), SLB_ERR_INVALID_ARG, "null input");
    SLB_REQUIRE(n_panels <= 2147483647LL, SLB_ERR_UNSUPPORTED, "panel ids must fit int32");
    SLB_REQUIRE(check_sticky("slb_near_build") == SLB_OK, SLB_ERR_CUDA, slb_last_error());
    double* sph = nullptr;
    int64_t* counts = nullptr;
    SLB_CUDA(cudaMallocAsync(&sph, sizeof(double) * 4 * std::max<int64_t>(n_panels, 1), s));
    SLB_CUDA(cudaMallocAsync(&counts, sizeof(int64_t) * std::max<int64_t>(n_trg, 1), s));
    if (n_panels > 0) {
        panel_sphere_kernel<<<(unsigned)((n_panels + 7) / 8), 256, 0, s>>>(n_panels, nodes_per_panel, y_nodes, sph);
        ++g_launch_count;
    }
    const unsigned grid = (unsigned)std::max<int64_t>(1, (n_trg + 7) / 8);
    if (n_trg > 0) {
        near_build_kernel<false><<<grid, 256, 0, s>>>(n_trg, x_trg, n_panels, nodes_per_panel, y_nodes, radius, sph,
                                                      own_panel, counts, nullptr);
        ++g_launch_count;
    }
    scan_kernel<<<1, 1024, 0, s>>>(n_trg, counts, row_ptr);
    ++g_launch_count;
    slb_status st = check_launch("slb_near_build (count)");
    int64_t nnz = 0;
    if (st == SLB_OK) {
        cudaError_t e = cudaMemcpyAsync(&nnz, row_ptr + n_trg, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error(std::string("slb_near_build: ") + cudaGetErrorString(e));
            st = SLB_ERR_CUDA;
        }
    }
    if (st == SLB_OK) {
        *nnz_out = nnz;
        if (panel_idx) {
            if (capacity < nnz) {
                set_error("slb_near_build: capacity < nnz");
                st = SLB_ERR_INVALID_ARG;
            } else if (n_trg > 0) {
                near_build_kernel<true><<<grid, 256, 0, s>>>(n_trg, x_trg, n_panels, nodes_per_panel, y_nodes, radius,
                                                             sph, own_panel, row_ptr, panel_idx);
                ++g_launch_count;
                st = check_launch("slb_near_build (fill)");
            }
        }
    }
    cudaFreeAsync(sph, s);
    cudaFreeAsync(counts, s);
    return st;
}
