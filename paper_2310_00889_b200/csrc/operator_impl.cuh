// operator_impl.cuh -- internal definition of slb_operator / slb_comm and the NCCL loader
// (shared by operator.cu and gmres.cu; not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <dlfcn.h>
#include <mutex>
#include <nccl.h>
#include <string>
#include <vector>
#include "common.cuh"

namespace slb {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

inline NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
#define LOADSYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(AllGather, "ncclAllGather");
    LOADSYM(Broadcast, "ncclBroadcast");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(GetErrorString, "ncclGetErrorString");
#undef LOADSYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Broadcast &&
             api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
    return api;
}

#define SLB_NCCL(call)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            ::slb::set_error(std::string(__func__) + ": " #call ": " + nccl().GetErrorString(r_)); \
            return SLB_ERR_NCCL;                                                              \
        }                                                                                     \
    } while (0)

}  // namespace slb

struct slb_comm;

namespace slb {
// (NEXT N4) multicast buffer: one physical copy per rank, a unicast and a multicast mapping (nvls.cu)
struct NvlsBuf {
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUdeviceptr uc_va = 0, mc_va = 0;
    size_t size = 0;
    CUdevice dev = 0;
    bool bound = false;
};
bool nvls_supported();
slb_status nvls_alloc(slb_comm* c, size_t bytes, NvlsBuf* b);
void nvls_free(NvlsBuf* b);
slb_status matvec_direct(slb_operator* op, const double* sigma_local, double* u_local, cudaStream_t s);
}  // namespace slb

struct slb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    // collectives issued through this communicator (slb_comm_collective_counts)
    std::atomic<long long> n_allgather{0}, n_broadcast{0}, n_allreduce{0};
};

struct slb_operator {
    slb_operator_desc d;
    slb_comm* comm = nullptr;
    slb::FarKind kind;
    int tdim = 1, sdim = 1;
    slb::FarPlan plan;
    slb::InterpParams ip;
    double* ip_buf = nullptr;           // device interpolation matrices (large grids)
    int64_t P_loc = 0, N_loc = 0, Nn = 0, Mn = 0, M = 0, cols = 0;
    std::vector<int64_t> ranges;        // panel offsets of all ranks [R+1]
    bool equal_shards = true;
    // device buffers owned by the operator
    double* geo = nullptr;              // [M][6]
    double* sc = nullptr;               // local fine scales [M_loc] or [M_loc][3]
    double* dyn = nullptr;              // [M][4] global fine records
    double* coarse = nullptr;           // [P_global][Nn][sdim] global sigma'
    double* partials = nullptr;         // [n_chunks][T_loc][tdim]
    double* Lsig = nullptr;             // [N_loc][3]
    int64_t* nb0 = nullptr;             // [nb+1] local node offsets of bodies
    double* bodyc = nullptr;            // [nb][16]
    double* coef = nullptr;             // [nb][6]
    int64_t max_nodes_body = 0;
    double* sig_dev = nullptr;          // host-variant staging
    double* u_dev = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool timed = false;
    // constant-bank far field (large M): packed records, 4 worker streams, captured graph
    bool use_const = false;
    double* rec = nullptr;              // [M][10]
    cudaStream_t ws[8] = {};
    cudaEvent_t fork = nullptr, join[8] = {};
    cudaGraphExec_t graph = nullptr;
    int64_t const_launches = 0;
    bool far_check = true;              // false: create-time prescan found no r = 0 pair (R14) -> unchecked kernels
    unsigned long long prescan_pairs = 0;
    int near_G = 1;                     // targets per warp in the near stream kernel
    // ragged angular orders (NEXT N4): per-(nt, mt) buckets; all empty / NULL for uniform panels
    bool ragged = false;
    std::vector<int64_t> cn0, fn0;      // host [P_global+1] first coarse / fine node of each panel
    int64_t* cn0_d = nullptr;           // device copy of cn0
    int64_t* fn0_d = nullptr;           // device copy of fn0
    int64_t* lc0_d = nullptr;           // [P_loc+1] local coarse offsets (cn0 - cn0[begin])
    int64_t* lf0_d = nullptr;           // [P_loc+1] local fine offsets (fn0 - fn0[begin])
    int64_t* boff_d = nullptr;          // [nnz+1] block offsets (doubles)
    int32_t* pbucket_d = nullptr;       // [P_global] bucket of each panel
    struct Bucket {
        int nt, mt, ns, ms;
        slb::InterpParams ip;
        int64_t n_loc = 0;              // local panels in this bucket
        int32_t* plist_d = nullptr;     // their local panel ids
        double* ip_buf = nullptr;       // device interpolation matrices when too large for ip.v
    };
    std::vector<Bucket> buckets;
    int max_cols = 0;                   // widest block (nodes * sdim)
    int64_t blk_total = 0;              // doubles in all local blocks (ragged)
    int64_t* bmeta_d = nullptr;         // [nnz] packed sigma offset / width per block (ragged)
    // (NEXT N4) fused upsample + gather: dyn lives in a multicast object, the upsample writes through dyn_mc
    bool nvls_on = false;
    slb::NvlsBuf nvls;
    double* dyn_mc = nullptr;
    // whole-apply CUDA graphs keyed by the (sigma, u) pointers (slb_matvec)
    struct ApplyGraph {
        const double* sigma;
        double* u;
        cudaGraphExec_t exec;
        unsigned long long launches;
    };
    std::vector<ApplyGraph> apply_graphs;
    cudaStream_t cap_stream = nullptr;
    bool seen_direct = false;
    int* barrier_d = nullptr;           // one int for the NVLS barrier all-reduce
    int* coincident_dummy() {
        if (!barrier_d) { cudaMalloc(&barrier_d, sizeof(int)); cudaMemset(barrier_d, 0, sizeof(int)); }
        return barrier_d;
    }
};

