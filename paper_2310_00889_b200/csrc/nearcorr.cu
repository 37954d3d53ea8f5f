// nearcorr.cu -- (c) block-sparse near-field correction, its setup fold, and the fused
// finalize of the operator apply.
//
// PAPER.md Eq. e:nystrom-correction: u(x) += sum_{k: x in N_k} sum_ij E_ij^(k)(x) sigma_ij,
// E = (special quadrature) - G w, stored as a sparse matrix
// "whose product with the current density vector is added to the result of the FMM".
//
// Apply: one warp per target row; each lane streams 16-byte slices of the row's blocks
// (ld.global.cs: evict-first, the blocks are touched once per apply) and reads the matching
// slices of the coarse density (L2-resident, ld.global.nc); lane partial sums are combined
// with a fixed xor-butterfly, so the result is deterministic.  HBM-bound: bytes per (t,k) =
// 8 tdim sdim N_n (+4 index).
#include <algorithm>
#include <cstdlib>
#include "common.cuh"

namespace slb {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Streaming near apply (B200): one warp per target row; the row's blocks (t_dim x cols doubles,
// contiguous) are pulled into a per-warp STG-deep shared-memory ring by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) issued by lane 0, so several KB per warp are in flight
// with no per-thread address arithmetic; lanes then read the slot (LDS.128) against sigma'_k
// (L2-resident, ld.global.nc).  Lane partials are combined with a fixed xor butterfly.
//   MODE 0 (slb_nearcorr_apply):  u[t] += near(t)
//   MODE 1 (slb_matvec finalize): u[t]  = (sum_c partials[c][t] + near(t)) + c_id sigma'_t [t < n_on] + (L sigma)_t
constexpr int kNearStages = 3;
constexpr int kNearWarps = 4;

// Each warp owns G consecutive targets (G chosen so a warp streams ~48 blocks); the TMA ring runs
// continuously across the group's row boundaries (block i of the group always goes to slot
// i % STG), so short rows do not drain the pipeline, while CTAs still run in target order --
// the warps active at any moment read a narrow window of the block array (a persistent,
// range-partitioned variant spread 1184 concurrent streams over 125 GB and thrashed the TLB).
template <int TD, int MODE>
__global__ void __launch_bounds__(kNearWarps * 32)
near_stream_kernel(int64_t T, int cols2, const int64_t* __restrict__ row_ptr,
                   const int32_t* __restrict__ panel_idx, const double* __restrict__ blocks,
                   const double* __restrict__ sigma_c, const double* __restrict__ partials, int64_t n_chunks,
                   int64_t n_on, double c_id, const double* __restrict__ sig_local,
                   const double* __restrict__ Lsig, double* __restrict__ u, int G) {
    extern __shared__ __align__(128) double2 ring[];      // [warps][STG][TD*cols2]
    __shared__ __align__(8) uint64_t bars[kNearWarps * kNearStages];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = TD * cols2;                          // double2 per block
    const uint32_t bytes = (uint32_t)slot * 16u;
    double2* myring = ring + (size_t)w * kNearStages * slot;
    uint64_t* mybar = bars + w * kNearStages;
    if (lane == 0) {
        for (int q = 0; q < kNearStages; ++q) mbar_init(&mybar[q], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * kNearWarps + w;
    const int64_t ta = gw * G;
    const int64_t tb = ta + G < T ? ta + G : T;
    if (ta >= tb) return;
    const int64_t pa = row_ptr[ta], pb = row_ptr[tb];
    const double2* B = reinterpret_cast<const double2*>(blocks);
    if (lane == 0) {
        for (int q = 0; q < kNearStages && pa + q < pb; ++q) {
            mbar_expect_tx(&mybar[q], bytes);
            bulk_g2s(myring + (size_t)q * slot, B + (pa + q) * slot, bytes, &mybar[q]);
        }
    }
    const double2* S2 = reinterpret_cast<const double2*>(sigma_c);
    int64_t i = 0;                                        // block counter within [pa, pb)
    for (int64_t t = ta; t < tb; ++t) {
        double acc[TD];
#pragma unroll
        for (int r = 0; r < TD; ++r) acc[r] = 0.0;
        const int64_t p1 = row_ptr[t + 1];
        for (int64_t p = row_ptr[t]; p < p1; ++p, ++i) {
            const int st = (int)(i % kNearStages);
            const int64_t k = panel_idx[p];
            const double2* Sk = S2 + k * cols2;
            mbar_wait(&mybar[st], (uint32_t)((i / kNearStages) & 1));
            const double2* R = myring + (size_t)st * slot;
#pragma unroll 2
            for (int c = lane; c < cols2; c += 32) {
                const double2 sv = __ldg(Sk + c);
#pragma unroll
                for (int r = 0; r < TD; ++r) {
                    const double2 bv = R[r * cols2 + c];
                    acc[r] = fma(bv.x, sv.x, fma(bv.y, sv.y, acc[r]));
                }
            }
            __syncwarp();
            if (lane == 0 && pa + i + kNearStages < pb) {
                fence_proxy_async_smem();
                mbar_expect_tx(&mybar[st], bytes);
                bulk_g2s(myring + (size_t)st * slot, B + (pa + i + kNearStages) * slot, bytes, &mybar[st]);
            }
        }
        double far[TD];
#pragma unroll
        for (int r = 0; r < TD; ++r) far[r] = 0.0;
        if (MODE == 1)
            for (int64_t c = lane; c < n_chunks; c += 32)
#pragma unroll
                for (int r = 0; r < TD; ++r) far[r] += partials[(c * T + t) * TD + r];
#pragma unroll
        for (int r = 0; r < TD; ++r) {
            const double nv = warp_sum(acc[r]);
            const double fv = MODE == 1 ? warp_sum(far[r]) : 0.0;
            if (lane == r) {
                if (MODE == 0) {
                    u[t * TD + r] += nv;
                } else {
                    double v = fv + nv;
                    if (t < n_on) {
                        v += c_id * sig_local[t * TD + r];
                        if (Lsig) v += Lsig[t * TD + r];
                    }
                    u[t * TD + r] = v;
                }
            }
        }
    }
}

static slb_status near_stream_launch(int mode, int64_t T, int tdim, int cols, const int64_t* row_ptr,
                                     const int32_t* panel_idx, const double* blocks, const double* sigma_c,
                                     const double* partials, int64_t n_chunks, int64_t n_on, double c_id,
                                     const double* sig_local, const double* Lsig, double* u, int G, cudaStream_t s) {
    if (T <= 0) return SLB_OK;
    const int cols2 = cols / 2;
    const size_t smem = (size_t)kNearWarps * kNearStages * tdim * cols2 * 16;
    SLB_REQUIRE(smem <= 227 * 1024, SLB_ERR_UNSUPPORTED, "near blocks too large for the smem ring");
    G = std::max(1, G);
    const unsigned grid = (unsigned)std::max<int64_t>(1, (T + (int64_t)G * kNearWarps - 1) / ((int64_t)G * kNearWarps));
#define NEAR_LAUNCH(TD, MODE)                                                                               \
    do {                                                                                                    \
        { slb_status st_ = smem_optin((const void*)near_stream_kernel<TD, MODE>); if (st_ != SLB_OK) return st_; } \
        near_stream_kernel<TD, MODE><<<grid, kNearWarps * 32, smem, s>>>(T, cols2, row_ptr, panel_idx, blocks,  \
                                                                         sigma_c, partials, n_chunks, n_on, c_id, \
                                                                         sig_local, Lsig, u, G);            \
    } while (0)
    if (tdim == 1) {
        if (mode == 0) NEAR_LAUNCH(1, 0); else NEAR_LAUNCH(1, 1);
    } else {
        if (mode == 0) NEAR_LAUNCH(3, 0); else NEAR_LAUNCH(3, 1);
    }
#undef NEAR_LAUNCH
    ++g_launch_count;
    return check_launch("near_stream_kernel");
}


// Ragged angular orders (NEXT N4): block p = [TD][ck] doubles at boff[p] (ck = its panel's nodes x
// sdim, panel k's density at coarse node cn0[k]), blocks of very different widths (c3v: 10-55 KB).
// The TMA ring holds fixed slots of S double2; a block streams through ceil(TD ck2 / S) slots
// (chunks of its flat [row][col] layout).  Lane 0 produces chunks in the same (block, chunk) order
// the warp consumes them.  Per row, every lane visits the columns c = lane (mod 32) in increasing
// order exactly as near_stream_kernel does, so a ragged operator whose orders happen to be equal
// returns the uniform operator's result bit for bit.
template <int TD, int MODE>
__global__ void __launch_bounds__(kNearWarps * 32)
near_stream_ragged_kernel(int64_t T, int S, const int64_t* __restrict__ row_ptr,
                          const int32_t* __restrict__ panel_idx, const double* __restrict__ blocks,
                          const double* __restrict__ sigma_c, const double* __restrict__ partials, int64_t n_chunks,
                          int64_t n_on, double c_id, const double* __restrict__ sig_local,
                          const double* __restrict__ Lsig, double* __restrict__ u, int G,
                          const int64_t* __restrict__ cn0, const int64_t* __restrict__ boff, int sdim, int ucols2,
                          const int64_t* __restrict__ bmeta) {
    // uniform panels (cn0 = boff = NULL): every block is TD x ucols2 double2
    extern __shared__ __align__(128) double2 ring[];      // [warps][STG][S]
    __shared__ __align__(8) uint64_t bars[kNearWarps * kNearStages];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* myring = ring + (size_t)w * kNearStages * S;
    uint64_t* mybar = bars + w * kNearStages;
    if (lane == 0) {
        for (int q = 0; q < kNearStages; ++q) mbar_init(&mybar[q], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * kNearWarps + w;
    const int64_t ta = gw * G;
    const int64_t tb = ta + G < T ? ta + G : T;
    if (ta >= tb) return;
    const int64_t pa = row_ptr[ta], pb = row_ptr[tb];
    const double2* B = reinterpret_cast<const double2*>(blocks);
    // producer cursor (lane 0): block pp, first double2 qq of the next chunk
    int64_t pp = pa, qq = 0;
    auto produce = [&](int st) {
        if (pp >= pb) return;
        const int64_t len2 = boff ? (boff[pp + 1] - boff[pp]) / 2 : (int64_t)TD * ucols2;
        const int64_t b0 = boff ? boff[pp] / 2 : pp * (int64_t)TD * ucols2;
        const int64_t n2 = (len2 - qq) < S ? (len2 - qq) : S;
        mbar_expect_tx(&mybar[st], (uint32_t)(n2 * 16));
        bulk_g2s(myring + (size_t)st * S, B + b0 + qq, (uint32_t)(n2 * 16), &mybar[st]);
        qq += n2;
        if (qq >= len2) { ++pp; qq = 0; }
    };
    if (lane == 0)
        for (int q = 0; q < kNearStages; ++q) produce(q);
    const double2* S2 = reinterpret_cast<const double2*>(sigma_c);
    int64_t i = 0;                                        // chunk counter
    for (int64_t t = ta; t < tb; ++t) {
        double acc[TD];
#pragma unroll
        for (int r = 0; r < TD; ++r) acc[r] = 0.0;
        const int64_t p1 = row_ptr[t + 1];
        for (int64_t p = row_ptr[t]; p < p1; ++p) {
            int ck;
            const double2* Sk;
            if (bmeta) {
                const int64_t bm = bmeta[p];
                ck = (int)(bm & 4095);
                Sk = S2 + (bm >> 12);
            } else {
                const int64_t k = panel_idx[p];
                ck = cn0 ? (int)((cn0[k + 1] - cn0[k]) * sdim / 2) : ucols2;
                Sk = cn0 ? S2 + cn0[k] * sdim / 2 : S2 + k * (int64_t)ucols2;
            }
            const int len2 = TD * ck;
            for (int q0 = 0; q0 < len2; q0 += S, ++i) {
                const int st = (int)(i % kNearStages);
                const int n2 = (len2 - q0) < S ? (len2 - q0) : S;
                mbar_wait(&mybar[st], (uint32_t)((i / kNearStages) & 1));
                const double2* R = myring + (size_t)st * S - q0;   // R[f] = block flat index f
#pragma unroll
                for (int r = 0; r < TD; ++r) {
                    const int lo = max(q0 - r * ck, 0), hi = min(q0 + n2 - r * ck, ck);
                    if (lo >= hi) continue;
                    for (int c = lo + ((lane - lo) & 31); c < hi; c += 32) {
                        const double2 sv = __ldg(Sk + c);
                        const double2 bv = R[r * ck + c];
                        acc[r] = fma(bv.x, sv.x, fma(bv.y, sv.y, acc[r]));
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_smem();
                    produce(st);
                }
            }
        }
        double far[TD];
#pragma unroll
        for (int r = 0; r < TD; ++r) far[r] = 0.0;
        if (MODE == 1)
            for (int64_t c = lane; c < n_chunks; c += 32)
#pragma unroll
                for (int r = 0; r < TD; ++r) far[r] += partials[(c * T + t) * TD + r];
#pragma unroll
        for (int r = 0; r < TD; ++r) {
            const double nv = warp_sum(acc[r]);
            const double fv = MODE == 1 ? warp_sum(far[r]) : 0.0;
            if (lane == r) {
                if (MODE == 0) {
                    u[t * TD + r] += nv;
                } else {
                    double v = fv + nv;
                    if (t < n_on) {
                        v += c_id * sig_local[t * TD + r];
                        if (Lsig) v += Lsig[t * TD + r];
                    }
                    u[t * TD + r] = v;
                }
            }
        }
    }
}

// Chunked streaming for ragged blocks: slots of S <= kChunk2 double2.  Measured on c3v (blocks of
// 10-74 KB): S = 320 (5 KB slots, 3 CTAs = 12 streaming warps per SM) 1.73 ms = 85 % of HBM;
// 240: 1.89, 480: 1.96, 640: 2.78, 800: 2.75, 1152: 4.13 ms -- more warps per SM beat bigger copies.
constexpr int kChunk2 = 320;

static slb_status near_ragged_launch(int mode, int64_t T, int tdim, const int64_t* row_ptr, const int32_t* panel_idx,
                                     const double* blocks, const double* sigma_c, const double* partials,
                                     int64_t n_chunks, int64_t n_on, double c_id, const double* sig_local,
                                     const double* Lsig, double* u, int G, cudaStream_t s, const RagNear& rag,
                                     int ucols = 0) {
    if (T <= 0) return SLB_OK;
    const int widest2 = tdim * (rag.boff ? rag.max_cols : ucols) / 2;
    static const int chunk = [] {
        const char* e = getenv("SLB_NEAR_CHUNK");
        return e ? std::max(64, atoi(e)) : kChunk2;
    }();
    const int S = std::min(widest2, chunk);
    const size_t smem = (size_t)kNearWarps * kNearStages * S * 16;
    G = std::max(1, G);
    const unsigned grid = (unsigned)std::max<int64_t>(1, (T + (int64_t)G * kNearWarps - 1) / ((int64_t)G * kNearWarps));
#define RAG_LAUNCH(TD, MODE)                                                                                  \
    do {                                                                                                      \
        { slb_status st_ = smem_optin((const void*)near_stream_ragged_kernel<TD, MODE>); if (st_ != SLB_OK) return st_; } \
        near_stream_ragged_kernel<TD, MODE><<<grid, kNearWarps * 32, smem, s>>>(                              \
            T, S, row_ptr, panel_idx, blocks, sigma_c, partials, n_chunks, n_on, c_id, sig_local, Lsig, u, G,  \
            rag.cn0, rag.boff, tdim, ucols / 2, rag.bmeta);                                                   \
    } while (0)
    if (tdim == 1) {
        if (mode == 0) RAG_LAUNCH(1, 0); else RAG_LAUNCH(1, 1);
    } else {
        if (mode == 0) RAG_LAUNCH(3, 0); else RAG_LAUNCH(3, 1);
    }
#undef RAG_LAUNCH
    ++g_launch_count;
    return check_launch("near_stream_ragged_kernel");
}

slb_status near_apply_launch(int64_t T, int tdim, int cols, const int64_t* row_ptr, const int32_t* panel_idx,
                             const double* blocks, const double* sigma_c, double* u, cudaStream_t s) {
    // same width rule as finalize_launch: blocks wider than 600 double2 (and every block the whole-block
    // ring cannot hold, e.g. Stokes 12 x 32 or 16 x 64 panels) stream through the chunked kernel
    if (tdim * cols / 2 > 600)
        return near_ragged_launch(0, T, tdim, row_ptr, panel_idx, blocks, sigma_c, nullptr, 0, 0, 0.0, nullptr,
                                  nullptr, u, 4, s, RagNear(), cols);
    return near_stream_launch(0, T, tdim, cols, row_ptr, panel_idx, blocks, sigma_c, nullptr, 0, 0, 0.0, nullptr,
                              nullptr, u, 4, s);
}

slb_status finalize_launch(const FarPlan& plan, int64_t T, int tdim, int cols, const double* partials,
                           const int64_t* row_ptr, const int32_t* panel_idx, const double* blocks,
                           const double* sigma_c_global, int64_t n_on, double c_id, const double* sig_local,
                           const double* Lsig, double* u, int G, cudaStream_t s, const RagNear& rag) {
    // uniform blocks wider than 600 double2 (c2: 11.5 KB, c3: 17 KB) also stream through the chunked
    // kernel: c3 near 0.78 -> 0.62 ms, c2 0.150 -> 0.120 ms; c4/c5's 8.6 KB blocks stay on the plain
    // ring (chunking them: c4 2.46 -> 2.84 ms)
    static const int chunk_uniform = [] {
        const char* e = getenv("SLB_NEAR_CHUNKED_UNIFORM");
        return e ? atoi(e) : 600;
    }();
    if (rag.boff || (chunk_uniform && tdim * cols / 2 > chunk_uniform))
        return near_ragged_launch(1, T, tdim, row_ptr, panel_idx, blocks, sigma_c_global, partials, plan.n_chunks,
                                  n_on, c_id, sig_local, Lsig, u, G, s, rag, cols);
    return near_stream_launch(1, T, tdim, cols, row_ptr, panel_idx, blocks, sigma_c_global, partials, plan.n_chunks,
                              n_on, c_id, sig_local, Lsig, u, G, s);
}

// ------------------------------------------------------------------ fold (setup)
// For each target t (one CTA) and each near panel k = panel_idx[p]:
//   G[ij][m] = K_ij(x_t - y_m; n_m) w_m over panel k's fine nodes m (K symmetric: 6 entries),
//   H[ij][a][b] = sum_{mt} G[ij][a][mt] F[mt][b]        (theta adjoint, ms x nt)
//   blocks[p][i][(a' b) j] -= sum_{a} Ps[a][a'] H[ij][a][b]
__global__ void __launch_bounds__(128)
fold_kernel(int kind, int64_t T, const double* __restrict__ x_trg, const int64_t* __restrict__ row_ptr,
            const int32_t* __restrict__ panel_idx, const __grid_constant__ InterpParams ip,
            const double* __restrict__ y_f, const double* __restrict__ n_f, const double* __restrict__ w_f,
            const double* __restrict__ eta_f, double eta, double* __restrict__ blocks,
            const int32_t* __restrict__ pbucket, int bucket, const int64_t* __restrict__ fn0,
            const int64_t* __restrict__ boff, int rch) {
    // rch: fine GL rows (a) per pass -- ms unless a (32 x 128) panel's G would not fit shared memory
    extern __shared__ double sm[];
    const int ns = ip.ns, nt = ip.nt, ms = ip.ms, mt = ip.mt;
    const double* Ps = ip.vg ? ip.vg : ip.v;
    const double* F = Ps + ms * ns;
    const int Mn = ms * mt, Nn = ns * nt;
    const int NG = far_scalar(kind) ? 1 : 6;
    const int TD = far_scalar(kind) ? 1 : 3;
    const int Mc = rch * mt;        // fine nodes per pass
    double* G = sm;                 // [NG][rch * mt]
    double* H = sm + NG * Mc;       // [NG][rch][nt]
    const int64_t t = blockIdx.x;
    if (t >= T) return;
    const double x0 = x_trg[3 * t], x1 = x_trg[3 * t + 1], x2 = x_trg[3 * t + 2];
    for (int64_t p = row_ptr[t]; p < row_ptr[t + 1]; ++p) {
        const int64_t k = panel_idx[p];
        if (pbucket && pbucket[k] != bucket) continue;          // ragged: another launch's orders
        const int64_t mk0 = fn0 ? fn0[k] : k * (int64_t)Mn;
        double* Bp = blocks + (boff ? boff[p] : p * (int64_t)TD * Nn * TD);
        for (int a0 = 0; a0 < ms; a0 += rch) {
            const int ra = min(rch, ms - a0);
            for (int q = threadIdx.x; q < ra * mt; q += blockDim.x) {
                const int64_t m = mk0 + (int64_t)a0 * mt + q;
                double r[3] = {x0 - y_f[3 * m], x1 - y_f[3 * m + 1], x2 - y_f[3 * m + 2]};
                double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
                double nn[3] = {n_f[3 * m], n_f[3 * m + 1], n_f[3 * m + 2]};
                double w = w_f[m];
                if (r2 == 0.0) {
                    for (int g = 0; g < NG; ++g) G[g * Mc + q] = 0.0;
                    continue;
                }
                double ir = 1.0 / sqrt(r2);
                double rn = r[0] * nn[0] + r[1] * nn[1] + r[2] * nn[2];
                if (far_scalar(kind)) {
                    const double e = (kind == FAR_LAPLACE_SLDL) ? (eta_f ? eta_f[m] : eta) : 0.0;
                    G[q] = (rn * ir * ir * ir + e * ir) / (4.0 * kPi) * w;
                } else {
                    double e = (kind == FAR_STOKES_SLDL) ? (eta_f ? eta_f[m] : eta) : 0.0;
                    double ir3 = ir * ir * ir;
                    double sl = e / (8.0 * kPi);
                    double dl = 3.0 / (4.0 * kPi) * rn * ir3 * ir * ir;
                    int g = 0;
                    for (int i = 0; i < 3; ++i)
                        for (int j = i; j < 3; ++j, ++g) {
                            double v = sl * ((i == j ? ir : 0.0) + r[i] * r[j] * ir3) + dl * r[i] * r[j];
                            G[g * Mc + q] = v * w;
                        }
                }
            }
            __syncthreads();
            const int nH = NG * ra * nt;
            for (int q = threadIdx.x; q < nH; q += blockDim.x) {
                int b = q % nt, a = (q / nt) % ra, g = q / (nt * ra);
                const double* Gr = G + g * Mc + a * mt;
                double acc = 0.0;
                for (int c = 0; c < mt; ++c) acc = fma(Gr[c], F[c * nt + b], acc);
                H[(g * rch + a) * nt + b] = acc;
            }
            __syncthreads();
            const int nE = TD * Nn * TD;
            for (int q = threadIdx.x; q < nE; q += blockDim.x) {
                int j = q % TD, node = (q / TD) % Nn, i = q / (TD * Nn);
                int a2 = node / nt, b = node % nt;
                int lo = i < j ? i : j, hi = i < j ? j : i;
                int g = (TD == 1) ? 0 : (lo == 0 ? hi : (lo == 1 ? 2 + hi : 5));
                const double* Hg = H + g * rch * nt;
                double acc = 0.0;
                for (int a = 0; a < ra; ++a) acc = fma(Ps[(a0 + a) * ns + a2], Hg[a * nt + b], acc);
                Bp[q] -= acc;
            }
            __syncthreads();
        }
    }
}

slb_status fold_launch(FarKind kind, int64_t T, const double* x_trg, const int64_t* row_ptr,
                       const int32_t* panel_idx, const InterpParams& ip, const double* y_fine,
                       const double* n_fine, const double* w_fine, const double* eta_fine, double eta,
                       double* blocks, cudaStream_t s, const int32_t* pbucket, int bucket, const int64_t* fn0,
                       const int64_t* boff) {
    if (T <= 0) return SLB_OK;
    SLB_REQUIRE(T <= 2147483647LL, SLB_ERR_UNSUPPORTED, "too many targets for fold");
    const int NG = far_scalar(kind) ? 1 : 6;
    auto smem_of = [&](int r) { return sizeof(double) * (size_t)(NG * r * ip.mt + NG * r * ip.nt); };
    int rch = ip.ms;
    while (rch > 1 && smem_of(rch) > 227 * 1024) rch = (rch + 1) / 2;
    const size_t smem = smem_of(rch);
    SLB_REQUIRE(smem <= 227 * 1024, SLB_ERR_UNSUPPORTED, "fold: grid too large for shared memory");
    { slb_status st_ = smem_optin((const void*)fold_kernel); if (st_ != SLB_OK) return st_; }
    fold_kernel<<<(unsigned)T, 128, smem, s>>>((int)kind, T, x_trg, row_ptr, panel_idx, ip, y_fine, n_fine,
                                              w_fine, eta_fine, eta, blocks, pbucket, bucket, fn0, boff, rch);
    ++g_launch_count;
    return check_launch("fold_kernel");
}

// ------------------------------------------------------------------ synthetic blocks
__global__ void fill_blocks_kernel(uint64_t seed, uint64_t first, int64_t count, double s_blk,
                                   double* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += stride) {
        double u01 = (double)(splitmix64(seed, first + (uint64_t)q) >> 11) * (1.0 / 9007199254740992.0);
        double v = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u01), 1.0), 1.7320508075688772);
        out[q] = __dmul_rn(v, s_blk);
    }
}

}  // namespace slb

using namespace slb;

extern "C" slb_status slb_fill_blocks(uint64_t seed, uint64_t first, int64_t count, double s_blk,
                                      double* blocks, cudaStream_t s) {
    SLB_REQUIRE(count >= 0, SLB_ERR_INVALID_ARG, "count < 0");
    if (count == 0) return SLB_OK;
    SLB_REQUIRE(blocks, SLB_ERR_INVALID_ARG, "null blocks");
    int64_t want = (count + 255) / 256;
    unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)num_sms() * 16);
    fill_blocks_kernel<<<grid, 256, 0, s>>>(seed, first, count, s_blk, blocks);
    ++g_launch_count;
    return check_launch("fill_blocks_kernel");
}

namespace slb {
// targets per warp for the streaming near kernel: ~420 KB of blocks streamed per warp (48 blocks of
// 8.6 KB at c4/c5), but at least ~8 CTAs' worth of warp groups per SM so the last wave's tail stays
// short (c3, 30 k targets with 17 KB blocks: G = 2 -> 0.81 ms vs G = 9 -> 1.07 ms).
int near_group_size(int64_t T, int64_t nnz, double block_bytes) {
    if (const char* e = getenv("SLB_NEAR_G")) return std::max(1, atoi(e));
    if (T <= 0 || nnz <= 0) return 1;
    const double per_target = (double)nnz / (double)T * block_bytes;
    double G = std::round(420e3 / std::max(per_target, 1.0));
    G = std::min(G, std::floor((double)T / (4.0 * 148.0 * 8.0)));
    return (int)std::min<double>(16.0, std::max<double>(1.0, G));
}
}  // namespace slb

namespace slb {
// CSR sanity check (setup): flags[0] |= 1 if row_ptr[0] != 0 or not monotone, |= 2 if a panel id is
// outside [0, n_panels).
__global__ void csr_check_kernel(int64_t T, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ panel_idx,
                                 int64_t n_panels, int* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && row_ptr[0] != 0) atomicOr(flags, 1);
    if (i < T && row_ptr[i + 1] < row_ptr[i]) atomicOr(flags, 1);
    const int64_t nnz = row_ptr[T];
    if (i < T && (row_ptr[i + 1] > nnz || row_ptr[i] < 0)) atomicOr(flags, 1);
    if (i < T && row_ptr[i] >= 0 && row_ptr[i + 1] <= nnz) {
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int64_t k = panel_idx[p];
            if (k < 0 || k >= n_panels) { atomicOr(flags, 2); break; }
        }
    }
}

slb_status csr_check(int64_t T, const int64_t* row_ptr, const int32_t* panel_idx, int64_t n_panels) {
    int* f = nullptr;
    SLB_CUDA(cudaMalloc(&f, sizeof(int)));
    SLB_CUDA(cudaMemset(f, 0, sizeof(int)));
    csr_check_kernel<<<(unsigned)((T + 256) / 256), 256>>>(T, row_ptr, panel_idx, n_panels, f);
    ++g_launch_count;
    int h = 0;
    cudaError_t e = cudaMemcpy(&h, f, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(f);
    if (e != cudaSuccess) { set_error(std::string("csr_check: ") + cudaGetErrorString(e)); return SLB_ERR_CUDA; }
    if (h & 1) { set_error("row_ptr must start at 0 and be nondecreasing"); return SLB_ERR_INVALID_ARG; }
    if (h & 2) { set_error("panel_idx entry outside [0, n_panels_global)"); return SLB_ERR_INVALID_ARG; }
    return SLB_OK;
}
}  // namespace slb
