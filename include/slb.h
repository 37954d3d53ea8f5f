/*
 * slb.h -- C-ABI of the B200-native slender-body Nystrom layer-potential operator apply
 * (Malhotra & Barnett, arXiv 2310.00889, "Efficient convergent boundary integral methods
 * for slender bodies").  Implemented by libslb.so (hand-written CUDA for sm_100a + NCCL).
 *
 * The operator (PAPER.md line numbers "P:L"):
 *
 *   u_t = c_I [t < n_on] sigma'_t                                    identity term
 *       + sum_m K(x_t - y_m; n_m) w_m (U sigma')_m                    far field, Eq. e:nystrom-no-correction P:L862-872
 *       + sum_{k in near(t)} E_{t,k} sigma'_k                         local corrections, Eq. e:nystrom-correction P:L935-961
 *     E_{t,k} = B_{t,k} - sum_{m in fine(k)} K(x_t - y_m; n_m) w_m U_{m,:}
 *   with sigma' = sigma, or sigma' = (I - L) sigma and + L sigma for the mobility operator
 *   (K(I-L) + L) (Eq. e:new-mobility-bie P:L2009, projector Eq. L).
 *
 *   Kernels (r = x - y, n the outward unit normal at the source):
 *     Laplace DL   K = (r.n) / (4 pi |r|^3)
 *     Stokes       K = eta S(r) + D(r; n),
 *                  S = (1/8pi)(I/|r| + r r^T/|r|^3)                      (Eq. e:stokes-sl P:L538)
 *                  D = +(3/4pi)(r.n) r r^T/|r|^5                         (Eq. e:stokes-dl P:L551; sign: DESIGN.md R1)
 *   U = upsampling: P_s (Lagrange, N_s GL -> M_s GL per panel) x F_th (trigonometric,
 *       N_th -> M_th uniform).  Pairs with r = 0 contribute 0 (R14).
 *
 * Conventions for every function:
 *   - all floating point is fp64; integer index arrays are int64 (row_ptr) / int32 (panel ids);
 *   - array pointers are DEVICE pointers (except *_host variants and slb_comm ids), row-major,
 *     contiguous, 16-byte aligned (cudaMalloc / torch allocations satisfy this);
 *   - the caller owns every array argument; the library never frees caller memory;
 *   - every call is asynchronous on the given stream and returns after launch; nothing
 *     throws across the boundary; argument errors return SLB_ERR_INVALID_ARG or
 *     SLB_ERR_UNSUPPORTED before anything is launched; launch/CUDA errors return
 *     SLB_ERR_CUDA; asynchronous device faults surface as SLB_ERR_CUDA on a later call;
 *   - slb_last_error() gives a human-readable message for the last failing call on this thread;
 *   - node layout: [panel][i (s, GL ascending)][j (theta_j = 2 pi j / N)][component].
 * Determinism: for fixed inputs every function is bitwise reproducible, and slb_matvec gives
 * bitwise-identical u for any number of ranks (the per-target summation order depends only
 * on the global source count M).
 * Concurrency: one operator must not be used from two threads at once; DISTINCT operators and the
 *   stand-alone calls may run concurrently on any streams and host threads.  The one library-wide
 *   device resource -- the 64 KB __constant__ source-tile bank of the large-M far field -- is
 *   serialised inside the library: each slb_matvec that uses it takes a host lock, makes its stream
 *   wait on the device's "bank" event (recorded by the previous user), launches its tile graph and
 *   re-records the event, so users of the bank run one after another on the device in issue order.
 *   (Consequence: two large operators applied "concurrently" overlap everything except their far
 *   fields.)  Kernel shared-memory limits are raised once per kernel to the device maximum.
 */
#ifndef SLB_H
#define SLB_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLB_ABI_VERSION 2

typedef enum {
    SLB_OK = 0,
    SLB_ERR_INVALID_ARG = 1,
    SLB_ERR_CUDA = 2,
    SLB_ERR_NCCL = 3,
    SLB_ERR_OOM = 4,
    SLB_ERR_UNSUPPORTED = 5
} slb_status;

/* SLB_LAPLACE_DL also carries the Laplace combined field D + eta S_L when eta / eta_fine /
 * eta_panel is given.  SLB_STOKES_SL / SLB_LAPLACE_SL (pure single layers, weight 1) are accepted by
 * slb_nearcorr_quad[_ragged] only; the operator evaluates them as the combined kernels with eta = 1
 * and zero normals. */
typedef enum { SLB_LAPLACE_DL = 1, SLB_STOKES_SLDL = 2, SLB_STOKES_SL = 3, SLB_LAPLACE_SL = 4 } slb_kernel;

/* Compiled limits (SLB_ERR_UNSUPPORTED beyond them). */
#define SLB_MAX_NS 32
#define SLB_MAX_NT 64
#define SLB_MAX_MS 64
#define SLB_MAX_MT 128

int slb_abi_version(void);
const char* slb_last_error(void);

/* CFIE single-layer mixing parameter eta = 1 / (2 rho ln(1/rho)), 0 < rho < 1
 * (R11).  Returns NaN outside (0,1). Host function. */
double slb_eta_cfie(double rho);

/* Number of coincident (r == 0) target/source pairs skipped by far-field launches since
 * the last reset (device counter; synchronises the device).  R14.
 * Operators on the constant-bank far path (M >= 2^16) decide once, at slb_operator_create, whether
 * any such pair exists between their targets and sources (one extra far-field pass with zero
 * strengths, not counted here); if none does, their applies run kernels without the r == 0 test --
 * same results bit for bit, nothing to count.  SLB_CONST_PRESCAN=0 keeps the test in every apply. */
long long slb_coincident_count(void);
void slb_coincident_reset(void);

/* Number of kernels this library has launched since it was loaded (launch accounting). */
unsigned long long slb_launch_count(void);

/* (a, NEXT N4) Ragged upsample: panel p is ns[p] x nt[p] -> ms[p] x mt[p] (HOST arrays [n_panels]),
 * nodes of consecutive panels back to back in both arrays.  Otherwise as
 * slb_upsample.  Synchronises s (uploads the panel tables). */
slb_status slb_upsample_ragged(int64_t n_panels, const int32_t* ns, const int32_t* nt, const int32_t* ms,
                               const int32_t* mt, int ncomp, const double* sigma_coarse, double* sigma_fine,
                               cudaStream_t s);

/* (a) Upsample a density from the coarse Nystrom grid to the fine smooth-quadrature grid,
 *   sigma_fine[p][a][b][c] = sum_i sum_j P_s[a][i] F_th[b][j] sigma_coarse[p][i][j][c],
 *   P_s = barycentric Lagrange from the ns GL nodes to the ms GL nodes of [-1,1],
 *   F_th[b][j] = C_nt(2 pi b / mt - 2 pi j / nt), C_N the real trigonometric cardinal
 *   function with the Nyquist cosine (R3).  Requires nt, mt even, ms >= 1.
 *   sigma_coarse: [n_panels][ns][nt][ncomp]; sigma_fine: [n_panels][ms][mt][ncomp] (written). */
slb_status slb_upsample(int64_t n_panels, int ns, int nt, int ms, int mt, int ncomp,
                        const double* sigma_coarse, double* sigma_fine, cudaStream_t s);

/* (b) Far field, Laplace double layer, exact all-pairs sum:
 *   u[t] = sum_m (x_t - y_m).n_m / (4 pi |x_t - y_m|^3) w_m sigma[m].
 *   x_trg: [n_trg][3]; y, n: [n_src][3]; w, sigma: [n_src]; u: [n_trg] (written). */
slb_status slb_farfield_laplace_dl(int64_t n_trg, const double* x_trg, int64_t n_src,
                                   const double* y, const double* n, const double* w,
                                   const double* sigma, double* u, cudaStream_t s);

/* (b) Far field, Stokes single + double layer, exact all-pairs sum:
 *   u[t] = sum_m (eta_m S(x_t - y_m) + D(x_t - y_m; n_m)) w_m sigma[m]   (3-vectors).
 *   eta_src: [n_src] per-source eta (every entry must be > 0; an entry <= 0 poisons the result
 *   with NaN) or NULL, in which case the scalar eta (>= 0) is used for all sources; eta == 0
 *   with eta_src == NULL evaluates the pure double layer.  Pure single layer: pass n = zeros.
 *   sigma: [n_src][3]; u: [n_trg][3] (written). */
slb_status slb_farfield_stokes_sldl(int64_t n_trg, const double* x_trg, int64_t n_src,
                                    const double* y, const double* n, const double* w,
                                    const double* eta_src, double eta, const double* sigma,
                                    double* u, cudaStream_t s);

/* (c) Near-field correction apply, u[t] += sum_{p in [row_ptr[t], row_ptr[t+1])}
 *   blocks[p] (tdim x nodes_per_panel*sdim) . sigma_coarse[panel_idx[p]] (nodes_per_panel*sdim).
 *   row_ptr: [n_trg+1] int64 (monotone, row_ptr[0] = 0); panel_idx: [nnz] int32;
 *   blocks: [nnz][tdim][nodes_per_panel*sdim]; sigma_coarse: [n_panels][nodes_per_panel][sdim];
 *   u: [n_trg][tdim] ACCUMULATED.  tdim, sdim in {1,3}; nodes_per_panel*sdim even. */
slb_status slb_nearcorr_apply(int64_t n_trg, int tdim, int sdim, int nodes_per_panel,
                              const int64_t* row_ptr, const int32_t* panel_idx,
                              const double* blocks, const double* sigma_coarse, double* u,
                              cudaStream_t s);

/* (c, setup) Fold the smooth-rule subtraction into the blocks in place:
 *   blocks[p] <- blocks[p] - G_{t,k} U_k, G_{t,k}[i][(m,j)] = K_ij(x_t - y_m; n_m) w_m over the
 *   ms*mt fine nodes m of panel k = panel_idx[p], U_k the per-panel upsampling (as slb_upsample).
 *   After folding, slb_nearcorr_apply applies E = B - G U (the paper's E).
 *   kernel: SLB_LAPLACE_DL (tdim = sdim = 1) or SLB_STOKES_SLDL (3); y_fine, n_fine: [M][3],
 *   w_fine: [M], eta_fine: [M] (Stokes; may be NULL -> eta). */
slb_status slb_nearcorr_fold(slb_kernel kernel, int64_t n_trg, const double* x_trg,
                             const int64_t* row_ptr, const int32_t* panel_idx, int ns, int nt,
                             int ms, int mt, const double* y_fine, const double* n_fine,
                             const double* w_fine, const double* eta_fine, double eta,
                             double* blocks, cudaStream_t s);

/* (NEXT N1, setup) Special-quadrature blocks B for the CSR pairs (§3.2.3-3.2.4,
 * P:L1195-1354): B_{t,k}[r][(i,j,c)] = int int_{Gamma_k} K_rc(x_t - y; n) l_i(s) C_j(th) J ds dth, the
 * exact action of the layer potential on panel k's interpolant, by a singularity-resolving
 * adaptive rule: geometry interpolated from the panel's coarse nodes
 * y_coarse [n_panels][ns][nt][3]; trg_node[t] = global coarse node id if target t is that node
 * (on-surface, singular) else -1 (may be NULL: all off-surface); eta_panel [n_panels]: single-layer
 * weight (required for SLB_STOKES_SLDL: eta S + D; optional for SLB_LAPLACE_DL: D + eta S_L; for the
 * pure single layers SLB_STOKES_SL / SLB_LAPLACE_SL NULL means weight 1); order = GL points per cell direction (4..24), beta = accepted
 * distance / cell diameter.  blocks [nnz][tdim][ns*nt*sdim] written (unfolded B).  Synchronises s.
 * SLB_ERR_UNSUPPORTED if a target is too close for the cell budget, or if a panel's working set
 * exceeds shared memory (Stokes: N_s N_th <= 1024, e.g. 16 x 64). */
slb_status slb_nearcorr_quad(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                             const int64_t* row_ptr, const int32_t* panel_idx, int ns, int nt,
                             const double* y_coarse, const double* eta_panel, int order, double beta,
                             double* blocks, cudaStream_t s);

/* (NEXT N1 + N4) Same for ragged orders: panel k has panel_ns[k] x panel_nt[k] nodes (HOST arrays
 * [n_panels]; N_s <= 32, N_th even <= 64), y_coarse is the per-panel node blocks back to back
 * (P:L770-781), block p = [tdim][N_n^(k) sdim] packed back to back in CSR order.  Synchronises s. */
slb_status slb_nearcorr_quad_ragged(slb_kernel kernel, int64_t n_trg, const double* x_trg, const int64_t* trg_node,
                                    const int64_t* row_ptr, const int32_t* panel_idx, int64_t n_panels,
                                    const int32_t* panel_ns, const int32_t* panel_nt, const double* y_coarse,
                                    const double* eta_panel, int order, double beta, double* blocks, cudaStream_t s);

/* Synthetic special-quadrature blocks (input generation, R10):
 *   blocks[q] = ((2 u_q - 1) sqrt(3)) s_blk,  u_q = (splitmix64(seed, first + q) >> 11) 2^-53,
 *   q in [0, count).  Bit-identical to the oracle's definition. */
slb_status slb_fill_blocks(uint64_t seed, uint64_t first, int64_t count, double s_blk,
                           double* blocks, cudaStream_t s);

/* (NEXT N3, setup) Near-list construction: CSR over targets of
 *   near(t) = { k : sqrt(min_j |x_t - y_kj|^2) < radius[k] }  U  { own_panel[t] }   (R15;
 *   stands in for the paper's sphere/Morton near-region search, §3.3),
 *   distances evaluated exactly in fp64 as ((dx*dx + dy*dy) + dz*dz), panels ascending per row.
 *   x_trg: [n_trg][3]; y_nodes: [n_panels][nodes_per_panel][3]; radius: [n_panels];
 *   own_panel: [n_trg] (-1 = none) or NULL.  row_ptr: [n_trg+1] (written).  panel_idx: NULL to
 *   only count, else [capacity] (written when capacity >= nnz).  *nnz_out (host) = nnz.
 *   Synchronises s (the count is returned to the host). */
slb_status slb_near_build(int64_t n_trg, const double* x_trg, int64_t n_panels, int nodes_per_panel,
                          const double* y_nodes, const double* radius, const int64_t* own_panel,
                          int64_t* row_ptr, int32_t* panel_idx, int64_t capacity, int64_t* nnz_out,
                          cudaStream_t s);

/* ---------------- full operator (single- or multi-GPU) ---------------- */
typedef struct slb_comm slb_comm;
typedef struct slb_operator slb_operator;

/* NCCL communicator over one process per GPU.  The 128-byte id is created on one rank with
 * slb_comm_unique_id and broadcast by the caller (e.g. through torch.distributed). */
slb_status slb_comm_unique_id(unsigned char id[128]);
slb_status slb_comm_create(const unsigned char id[128], int nranks, int rank, slb_comm** out);
slb_status slb_comm_destroy(slb_comm* c);
/* Collectives issued through c so far: out[0] = ncclAllGather calls (create-time panel-range gather
 * and the per-apply in-place gathers of the fine records and the coarse density), out[1] =
 * ncclBroadcast calls (the grouped in-place broadcasts that replace the all-gather when the rank
 * shards are unequal, or when SLB_FORCE_GROUPED_GATHER=1), out[2] = ncclAllReduce calls (slb_gmres
 * dot products).  Every operator/solver holding a communicator issues them, a one-rank
 * communicator included (NCCL's gather is then an identity, the offsets and counts are the
 * multi-rank ones).  Host counters; no synchronisation. */
slb_status slb_comm_collective_counts(const slb_comm* c, long long out[3]);

typedef struct {
    slb_kernel kernel;
    int ns, nt, ms, mt;
    int64_t n_panels_global;
    int64_t panel_begin, panel_end;     /* this rank's source panels [begin, end) */
    int64_t n_trg_local;                /* local targets */
    int64_t n_on_local;                 /* first n_on_local local targets = local panels' coarse nodes */
    double c_identity;                  /* 0.5 for the BIE operator (exterior limit), 0 for potential evaluation */
    const double* x_trg;                /* [n_trg_local][3] */
    const double* y_fine;               /* [M][3] global fine nodes, M = n_panels_global*ms*mt */
    const double* n_fine;               /* [M][3] */
    const double* w_fine;               /* [M] */
    const double* eta_fine;             /* [M] single-layer weight (Stokes: entries > 0; Laplace: the
                                           combined field D + eta S_L) or NULL -> eta */
    double eta;                         /* scalar eta when eta_fine == NULL (0 -> pure DL, either kernel) */
    const int64_t* row_ptr;             /* [n_trg_local+1] local CSR */
    const int32_t* panel_idx;           /* [nnz] GLOBAL panel ids */
    double* blocks;                     /* [nnz][tdim][ns*nt*sdim]; folded in place at create unless blocks_folded */
    int blocks_folded;                  /* 1: blocks already hold E = B - G U */
    /* mobility projector (Eq. L): n_bodies_local = 0 disables.  Bodies must be whole on a rank. */
    int64_t n_bodies_local;
    const int32_t* body_of_panel_local; /* [panel_end-panel_begin] local body id, nondecreasing */
    const double* y_coarse;             /* [local nodes][3] */
    const double* w_coarse;             /* [local nodes] */
    /* (NEXT N4) ragged orders, §3.1 P:L770-781 ("element k ... polynomial order N_s^(k),
     * Fourier order N_th^(k)"): HOST arrays [n_panels_global]; each pair (panel_nt, panel_mt) and
     * (panel_ns, panel_ms) is given together or both NULL (then the scalar nt, mt / ns, ms apply).
     * Panel k has panel_ns[k] x panel_nt[k] coarse and panel_ms[k] x panel_mt[k] fine nodes
     * (N_th, M_th even; all within the compiled limits).  Every node array is the per-panel
     * blocks back to back in panel order; near block p is [tdim][N_n^(k) sdim] with k =
     * panel_idx[p], the blocks packed back to back in CSR order.  Read during create only. */
    const int32_t* panel_nt;
    const int32_t* panel_mt;
    const int32_t* panel_ns;
    const int32_t* panel_ms;
} slb_operator_desc;

/* Borrows every descriptor pointer (they must outlive the operator); owns only its scratch
 * and packed source records.  Synchronises the device once (setup). comm NULL -> 1 GPU. */
slb_status slb_operator_create(const slb_operator_desc* d, slb_comm* comm, slb_operator** out);

/* One operator apply on this rank: sigma_local [local panels][ns][nt][sdim] ->
 * u_local [n_trg_local][tdim] (written).  Collective across the communicator's ranks. */
slb_status slb_matvec(slb_operator* op, const double* sigma_local, double* u_local, cudaStream_t s);

/* Same, with HOST buffers: copies sigma in and u out on stream s (pinned memory gives
 * asynchronous copies), then synchronises s before returning. */
slb_status slb_matvec_host(slb_operator* op, const double* sigma_local_host, double* u_local_host,
                           cudaStream_t s);

/* Stage 1 of an apply alone: the projector (mobility operators) and
 * the upsample of sigma_local into the operator's fine source records, exactly the kernels slb_matvec
 * launches first; nothing else (no gather, far field or finalize).  For per-kernel timing (bench.py's
 * upsample roofline); the records it writes are the next apply's inputs, so it leaves the operator valid.
 * Errors: SLB_ERR_INVALID_ARG (null operator, null density with local nodes), SLB_ERR_CUDA. */
slb_status slb_operator_prepare(slb_operator* op, const double* sigma_local, cudaStream_t s);

/* Stage timing of the last slb_matvec (ms, CUDA events on s; -1 if unavailable):
 * [0] projector+upsample, [1] all-gather, [2] far field, [3] finalize (reduce+near+identity). */
slb_status slb_operator_last_timings(slb_operator* op, float out_ms[4]);

/* (NEXT N4) 1 if the operator gathers the fine source records through an NVLink-SHARP multicast object
 * (environment SLB_NVLS=1 at creation, a communicator, a multicast-capable device, the streaming
 * upsample): the upsample epilogue stores every record with multimem.st into all ranks' copies and the
 * per-apply ncclAllGather of the records is dropped (a one-int all-reduce barrier remains for > 1 rank;
 * more ranks exchange the multicast handle as a fabric handle).  0: the NCCL all-gather path. */
int slb_operator_nvls(const slb_operator* op);

/* 1 if this device supports multicast objects: CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and a probe
 * cuMulticastCreate succeeds (some single-GPU containers report the attribute but reject creation). */
int slb_nvls_supported(void);

/* Number of kernel launches slb_matvec issues on this rank (for launch accounting). */
int slb_operator_launches_per_matvec(const slb_operator* op);

slb_status slb_operator_destroy(slb_operator* op);

/* (NEXT N2) Restarted GMRES(restart) for  A x = rhs  with A = slb_matvec,
 * e.g. the CFIEs (I/2 + D + eta S) sigma = u0 and the mobility BIE (K(I-L) + L) sigma = rhs.
 * Requires a square operator (targets = the local nodes).  rhs, x: [local nodes][sdim] device;
 * x holds the initial guess on entry and the solution on return.  Stops when the true residual
 * ||rhs - A x|| <= tol ||rhs|| (checked at restarts) or after max_iters matvecs.  CGS2
 * orthogonalisation, fixed-order reductions (NCCL all-reduce across ranks): reproducible.
 * Collective across the operator's ranks; synchronises s.  iters_out, relres_out: host, may be NULL. */
slb_status slb_gmres(slb_operator* op, const double* rhs, double* x, int restart, int max_iters,
                     double tol, int* iters_out, double* relres_out, cudaStream_t s);

/* (NEXT N2) Stokes mobility solve, PAPER.md "Stokes slender mobility CFIE":
 * given per-body force F_b and torque T_b (about the body's quadrature-weighted centroid c_b),
 *   nu = alpha_b + beta_b x (x - c_b), int nu = F_b, int nu x (x - c_b) = T_b    (completion flow, P:L1903-1912;
 *        closed form alpha_b = F_b / |Omega_b|, beta_b = -I_b^-1 T_b with the projector's moments)
 *   (K(I - L) + L) sigma = -S[nu]                                                  (Eq. e:new-mobility-bie)
 *   V = -L sigma = v_b + omega_b x (x - c_b)                                       (Eq. e:recover-rigidbody-motion)
 * mob: mobility operator (Stokes CFIE kernel, projector enabled, square); sl: operator of the
 * same local nodes and targets evaluating the pure single layer S (SLB_STOKES_SLDL, eta = 1, zero
 * normals, c_identity = 0, blocks from slb_nearcorr_quad(SLB_STOKES_SL, ...)).
 * force_torque: HOST [n_bodies_local][6] = (F, T); rigid_out: HOST [n_bodies_local][6] = (v, omega)
 * written; sigma: device [local nodes][3], initial guess in, density out.  Other arguments as
 * slb_gmres.  Collective across the ranks; synchronises s. */
slb_status slb_mobility_solve(slb_operator* mob, slb_operator* sl, const double* force_torque, double* rigid_out,
                              double* sigma, int restart, int max_iters, double tol, int* iters_out,
                              double* relres_out, cudaStream_t s);

/* Microbenchmark: sustained FP64 FMA throughput (GFLOP/s, FMA = 2 flops) of this device,
 * measured with dependent-chain-free DFMA streams over all SMs for ~iters iterations. */
slb_status slb_bench_dfma(int64_t iters, double* gflops, cudaStream_t s);

#ifdef __cplusplus
}
#endif
#endif /* SLB_H */
