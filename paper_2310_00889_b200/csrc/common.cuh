// common.cuh -- internal helpers of libslb (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <mutex>
#include <string>
#include "../../include/slb.h"

namespace slb {

void set_error(const std::string& msg);

#define SLB_REQUIRE(cond, code, msg)                                   \
    do {                                                               \
        if (!(cond)) {                                                 \
            ::slb::set_error(std::string(__func__) + ": " + (msg));    \
            return (code);                                             \
        }                                                              \
    } while (0)

#define SLB_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            ::slb::set_error(std::string(__func__) + ": " #call ": " +              \
                             cudaGetErrorString(e_));                               \
            return e_ == cudaErrorMemoryAllocation ? SLB_ERR_OOM : SLB_ERR_CUDA;    \
        }                                                                           \
    } while (0)

// check for launch errors (and sticky asynchronous faults) after a launch
slb_status check_launch(const char* what);
slb_status check_sticky(const char* what);

constexpr double kPi = 3.141592653589793238462643383279502884;

// ---- host-side interpolation operators (own implementation; shares nothing with oracle/) ----
// Gauss-Legendre nodes (ascending) and weights on [-1,1].
void gl_nodes(int n, double* x, double* w);
// Barycentric Lagrange interpolation matrix from nodes xs[0..nf) to points xt[0..nt): P[m][i].
void bary_matrix(int nf, const double* xs, int nt, const double* xt, double* P);
// Trigonometric interpolation matrix F[b][j] = (1/N)[1 + 2 sum_{l=1}^{N/2-1} cos(l d) + cos(N d / 2)],
// d = 2 pi b / M - 2 pi j / N  (the real interpolant with the Nyquist cosine; N even).
void trig_matrix(int N, int M, double* F);

// Interpolation matrices passed BY VALUE as a kernel parameter (<= 32 KB param space); larger
// grids (e.g. N_th = 64 -> M_th = 128) keep them in a device buffer pointed to by vg.
constexpr int kMaxInterp = 3600;   // doubles: ms*ns + mt*nt
struct InterpParams {
    int ns, nt, ms, mt;
    const double* vg;              // device copy when the matrices exceed kMaxInterp, else nullptr
    const double* mats_d;          // device copy (P_s then F_th) whenever make_interp was given `owned`
    double v[kMaxInterp];          // P_s [ms][ns] followed by F [mt][nt]
};
// Fills ip.  If the matrices do not fit the parameter budget and `owned` is given, they are copied
// into a new device buffer (*owned; the caller frees it after the kernels using ip completed);
// returns false if they do not fit and owned == nullptr, or on allocation failure.
bool make_interp(int ns, int nt, int ms, int mt, InterpParams* ip, double** owned = nullptr);

// ---- device helpers ----
#ifdef __CUDACC__
__device__ __forceinline__ double rsqrt_mufu(double x) {
    // raw MUFU.RSQ64H approximation (ftz); refined by the caller
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

// 1/sqrt(r2) to ~1 ulp: MUFU seed + one cubic (3rd-order) correction
//   y = y0 (1 + e/2 + 3 e^2/8),  e = 1 - r2 y0^2.   5 FP64-pipe instructions.
__device__ __forceinline__ double rsqrt_refined(double r2) {
    double y0 = rsqrt_mufu(r2);
    double e = fma(-r2, y0 * y0, 1.0);
    double p = fma(e, 0.375, 0.5);
    double ye = y0 * e;
    return fma(ye, p, y0);
}

__device__ __forceinline__ bool is_zero_r2(double r2) {
    // r2 >= 0 always; hi word == 0  <=>  r2 < 2^-1022 (0 or subnormal): coincident pair (R14)
    return __double2hiint(r2) == 0;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}


// ---- mbarrier / TMA bulk-copy PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte store through a multicast (NVLS) mapping: replicated by the switch into every bound copy.
// multimem.st has no .v2.f64 form; the two doubles travel as four 32-bit lanes (a store: bits unchanged).
__device__ __forceinline__ void multimem_st2(double* p, double a, double b) {
    const unsigned long long ua = (unsigned long long)__double_as_longlong(a);
    const unsigned long long ub = (unsigned long long)__double_as_longlong(b);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "f"(__int_as_float((int)(ua & 0xffffffffull))), "f"(__int_as_float((int)(ua >> 32))),
                 "f"(__int_as_float((int)(ub & 0xffffffffull))), "f"(__int_as_float((int)(ub >> 32)))
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
#endif  // __CUDACC__

// Kernel launch bookkeeping for launch accounting.
extern std::atomic<unsigned long long> g_launch_count;

// Raise a kernel's dynamic shared-memory limit to the device maximum, once per kernel (thread-safe).
slb_status smem_optin(const void* fn);

int num_sms();

// ---- far-field engine (farfield.cu) ----
// FAR_LAPLACE_SLDL: the Laplace combined field D + eta S_L, records {q = w sigma n/4pi, s = eta w sigma/4pi}
enum FarKind { FAR_LAPLACE = 0, FAR_STOKES_SLDL = 1, FAR_STOKES_DL = 2, FAR_LAPLACE_SLDL = 3 };
__host__ __device__ constexpr bool far_scalar(int k) { return k == FAR_LAPLACE || k == FAR_LAPLACE_SLDL; }

// Summation plan; depends ONLY on the source count M (bitwise determinism across ranks).
struct FarPlan {
    int64_t M;
    int64_t chunk;     // sources per chunk (multiple of 256)
    int64_t n_chunks;
    int split;         // warps sharing one target group inside a CTA (1 or 4)
};
FarPlan far_plan(int64_t M);

// Packed source records: geo[m] = {y(3), a(3)}, dyn[m] = {d(3), 0}
//   Laplace:     a unused,              d = w sigma n / (4 pi)
//   Stokes SLDL: a = (3/(4 pi e)) n,     d = e w sigma,   e = eta/(8 pi)
//   Stokes DL:   a = (3/(4 pi)) n,       d = w sigma
slb_status far_partials(FarKind kind, const FarPlan& plan, int64_t n_trg, const double* x_trg,
                        const double* geo, const double* dyn, double* partials,
                        unsigned long long* coincident, cudaStream_t s);
slb_status far_reduce(const FarPlan& plan, int64_t n_trg, int tdim, const double* partials,
                      double* u, cudaStream_t s);
unsigned long long* coincident_counter();

// ---- constant-bank far field (farconst.cu) ----
slb_status far_const_issue(FarKind kind, int64_t M, int64_t T, const double* x, const double* rec,
                           double* partials, unsigned long long* zc, cudaStream_t s, cudaStream_t* ws,
                           cudaEvent_t fork, cudaEvent_t* join, int64_t* launches, bool check = true);
// check = false: the kernels without the r = 0 select and count -- only for operators whose create-time
// prescan found no coincident (target, source) pair (bitwise-identical results in that case)
slb_status pack_rec_launch(int64_t M, const double* geo, const double* dyn, double* rec, cudaStream_t s);
int far_const_bufs(int64_t M);   // streams / partial arrays for M sources
// Scoped host lock + device event chain serialising all users of the constant bank (farconst.cu).
class ConstBankLock {
  public:
    ConstBankLock();
    ~ConstBankLock();
    slb_status acquire(cudaStream_t s);   // s waits for the previous user's last tile
    slb_status release(cudaStream_t s);   // record: the next user waits for s's work so far
  private:
    std::unique_lock<std::mutex> lk_;
    int dev_ = 0;
};
int far_const_tile(int64_t M);   // sources per constant-bank tile
slb_status far_const_prepare();

// ---- packing kernels (farfield.cu) ----
slb_status pack_geo(FarKind kind, int64_t M, const double* y, const double* n, const double* eta_src,
                    double eta, double* geo, cudaStream_t s);
// per-source scale used by the dyn packing: Stokes -> sc[m] = e_m w_m (SLDL) or w_m (DL), 1 double;
// Laplace -> sc[m] = {w_m n_m / (4 pi), eta_m w_m / (4 pi)}, 4 doubles
slb_status pack_scale(FarKind kind, int64_t M, const double* n, const double* w, const double* eta_src,
                      double eta, double* sc, cudaStream_t s);
slb_status pack_dyn(FarKind kind, int64_t M, const double* sc, const double* sigma, double* dyn,
                    cudaStream_t s);

// ---- upsample (upsample.cu) ----
// sigma_fine: written as plain values (dyn == nullptr) or packed into dyn records with sc.
// Ragged panels (NEXT N4): plist = the bucket's panel ids (NULL: 0..n_panels-1), c_off / f_off =
// first coarse / fine node of each panel id (NULL: uniform p*ns*nt / p*ms*mt).
slb_status upsample_launch(FarKind kind, int64_t n_panels, const InterpParams& ip, int ncomp,
                           const double* sigma_coarse, double* sigma_fine, const double* sc,
                           double* dyn, cudaStream_t s, const int32_t* plist = nullptr,
                           const int64_t* c_off = nullptr, const int64_t* f_off = nullptr,
                           double* copy_out = nullptr, double* dyn_mc = nullptr);

// true when upsample_launch takes the streaming warp-per-panel kernel for this grid (which can also
// write the staged coarse density to copy_out, for any plist)
bool upsample_streams(FarKind kind, const InterpParams& ip, int nc, bool records, const double* sigma_coarse,
                      const double* sc);

// ---- near (nearcorr.cu) ----
slb_status near_apply_launch(int64_t n_trg, int tdim, int cols, const int64_t* row_ptr,
                             const int32_t* panel_idx, const double* blocks, const double* sigma_c,
                             double* u, cudaStream_t s);
// Ragged near blocks (NEXT N4): device offsets, all NULL for uniform panels.
struct RagNear {
    const int64_t* cn0 = nullptr;    // [P_global+1] first coarse node of each panel
    const int64_t* boff = nullptr;   // [nnz+1] first double of each block (CSR order)
    int max_cols = 0;                // largest nodes_per_panel * sdim
    const int64_t* bmeta = nullptr;  // [nnz] (sigma double2 offset << 12) | (block width / 2): one
                                     // independent load per block instead of panel_idx -> cn0
};
// fused finalize: u[t] = sum_c partials[c][t] + near(t) + c_id * sig_loc[t] (t < n_on) + Lsig[t]
slb_status finalize_launch(const FarPlan& plan, int64_t n_trg, int tdim, int cols,
                           const double* partials, const int64_t* row_ptr, const int32_t* panel_idx,
                           const double* blocks, const double* sigma_c_global, int64_t n_on,
                           double c_id, const double* sig_local, const double* Lsig, double* u,
                           int G, cudaStream_t s, const RagNear& rag = RagNear());
int near_group_size(int64_t T, int64_t nnz, double block_bytes);   // block_bytes: mean near block size
slb_status csr_check(int64_t T, const int64_t* row_ptr, const int32_t* panel_idx, int64_t n_panels);
// Ragged (NEXT N4): only pairs whose panel has pbucket[k] == bucket are folded (pbucket NULL: all);
// fn0 = first fine node of each global panel, boff = block offsets (NULL: uniform).
slb_status fold_launch(FarKind kind, int64_t n_trg, const double* x_trg, const int64_t* row_ptr,
                       const int32_t* panel_idx, const InterpParams& ip, const double* y_fine,
                       const double* n_fine, const double* w_fine, const double* eta_fine,
                       double eta, double* blocks, cudaStream_t s, const int32_t* pbucket = nullptr,
                       int bucket = 0, const int64_t* fn0 = nullptr, const int64_t* boff = nullptr);

// ---- projector (projector.cu) ----
slb_status body_moments_launch(int64_t n_bodies, const int64_t* node_begin, const double* y,
                               const double* w, double* mom /*[nb][16]*/, cudaStream_t s);
slb_status proj_launch(int64_t n_bodies, const int64_t* node_begin, const double* y,
                       const double* w, const double* bodyc /*[nb][16]*/, const double* sigma,
                       double* coef /*[nb][6]*/, double* sigma_p, double* Lsig,
                       int64_t max_nodes_per_body, cudaStream_t s);

slb_status completion_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* bodyc,
                             const double* ft /*[nb][6]*/, double* nu, int64_t max_nodes_per_body, cudaStream_t s);
slb_status proj_coef_launch(int64_t n_bodies, const int64_t* nb0, const double* y, const double* w,
                            const double* bodyc, const double* sigma, double* coef /*[nb][6]*/, cudaStream_t s);

}  // namespace slb
