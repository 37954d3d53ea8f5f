// nvls.cu -- (NEXT N4) NVLink-SHARP multicast buffers for the fused upsample + gather.
//
// The fine source records (the only per-apply exchange) can live in a multicast object:
// every rank binds its own physical copy, reads it through an ordinary (unicast) mapping, and the
// upsample epilogue WRITES through the multicast mapping (multimem.st), which the NVSwitch replicates
// into every rank's copy -- the all-gather becomes part of the upsample's stores and the separate
// collective disappears (only a tiny barrier remains so no rank reads before all have written).
// The driver API is reached through cudaGetDriverEntryPoint (libslb does not link libcuda).  A one-rank
// team is exercised on one GPU; more ranks exchange the multicast handle as a FABRIC handle broadcast
// over the NCCL communicator (needs an NVSwitch system with fabric handles; otherwise the operator keeps
// the NCCL all-gather).
#include <cuda.h>
#include <cstring>
#include <string>
#include "operator_impl.cuh"

namespace slb {

struct DrvApi {
    bool ok = false;
    CUresult (*DeviceGet)(CUdevice*, int);
    CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
    CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
    CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                                 unsigned long long);
    CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
    CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*MemRelease)(CUmemGenericAllocationHandle);
    CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*MemAddressFree)(CUdeviceptr, size_t);
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*MemUnmap)(CUdeviceptr, size_t);
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                           unsigned long long);
    CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
};

static DrvApi& drv() {
    static DrvApi api;
    static bool tried = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (tried) return api;
    tried = true;
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
            !*fn)
            ok = false;
    };
#define GET(field, name) get(name, reinterpret_cast<void**>(&api.field))
    GET(DeviceGet, "cuDeviceGet");
    GET(DeviceGetAttribute, "cuDeviceGetAttribute");
    GET(MulticastCreate, "cuMulticastCreate");
    GET(MulticastAddDevice, "cuMulticastAddDevice");
    GET(MulticastBindMem, "cuMulticastBindMem");
    GET(MulticastUnbind, "cuMulticastUnbind");
    GET(MulticastGetGranularity, "cuMulticastGetGranularity");
    GET(MemCreate, "cuMemCreate");
    GET(MemRelease, "cuMemRelease");
    GET(MemAddressReserve, "cuMemAddressReserve");
    GET(MemAddressFree, "cuMemAddressFree");
    GET(MemMap, "cuMemMap");
    GET(MemUnmap, "cuMemUnmap");
    GET(MemSetAccess, "cuMemSetAccess");
    GET(MemExportToShareableHandle, "cuMemExportToShareableHandle");
    GET(MemImportFromShareableHandle, "cuMemImportFromShareableHandle");
#undef GET
    api.ok = ok;
    return api;
}

#define DRV(call, what)                                                                          \
    do {                                                                                         \
        CUresult r_ = (call);                                                                    \
        if (r_ != CUDA_SUCCESS) {                                                                \
            set_error(std::string("nvls: ") + what + " failed (CUresult " + std::to_string((int)r_) + ")"); \
            nvls_free(b);                                                                        \
            return SLB_ERR_UNSUPPORTED;                                                          \
        }                                                                                        \
    } while (0)

void nvls_free(NvlsBuf* b) {
    if (!b) return;
    DrvApi& A = drv();
    if (!A.ok) return;
    if (b->mc_va) { A.MemUnmap(b->mc_va, b->size); A.MemAddressFree(b->mc_va, b->size); }
    if (b->uc_va) { A.MemUnmap(b->uc_va, b->size); A.MemAddressFree(b->uc_va, b->size); }
    if (b->bound) A.MulticastUnbind(b->mc, b->dev, 0, b->size);
    if (b->mem) A.MemRelease(b->mem);
    if (b->mc) A.MemRelease(b->mc);
    *b = NvlsBuf();
}

// The attribute alone is not enough: on some systems (e.g. one GPU of an NVSwitch box exposed to a
// container) CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 1 but cuMulticastCreate returns
// CUDA_ERROR_INVALID_VALUE (tools/nvls_probe.py).  Probe a minimal object once.
bool nvls_supported() {
    DrvApi& A = drv();
    if (!A.ok) return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    CUdevice cd;
    if (A.DeviceGet(&cd, dev) != CUDA_SUCCESS) return false;
    int v = 0;
    if (A.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !v) return false;
    static std::mutex mu;
    static int probed[64];                       // 0 unknown, 1 yes, 2 no (per device)
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return false;
    if (!probed[dev]) {
        CUmulticastObjectProp mp;
        std::memset(&mp, 0, sizeof(mp));
        mp.numDevices = 1;
        mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        size_t gran = 0;
        mp.size = 1 << 21;
        CUmemGenericAllocationHandle h = 0;
        bool ok = A.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS;
        if (ok && gran > mp.size) mp.size = gran;
        ok = ok && A.MulticastCreate(&h, &mp) == CUDA_SUCCESS;
        if (h) A.MemRelease(h);
        probed[dev] = ok ? 1 : 2;
    }
    return probed[dev] == 1;
}

// Multicast buffer of >= bytes shared by the communicator's ranks (c == NULL or one rank: a team of one).
slb_status nvls_alloc(slb_comm* c, size_t bytes, NvlsBuf* b) {
    *b = NvlsBuf();
    DrvApi& A = drv();
    SLB_REQUIRE(A.ok, SLB_ERR_UNSUPPORTED, "nvls: driver multicast API not available");
    SLB_REQUIRE(nvls_supported(), SLB_ERR_UNSUPPORTED, "nvls: device does not support multicast");
    int dev = 0;
    SLB_CUDA(cudaGetDevice(&dev));
    DRV(A.DeviceGet(&b->dev, dev), "cuDeviceGet");
    const int R = c ? c->nranks : 1;
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)R;
    // a shareable handle type is required even for a team of one (NONE is rejected)
    mp.handleTypes = R > 1 ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    size_t gran = 0;
    DRV(A.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    const size_t size = (bytes + gran - 1) / gran * gran;
    mp.size = size;
    b->size = size;
    if (R == 1 || c->rank == 0) DRV(A.MulticastCreate(&b->mc, &mp), "cuMulticastCreate");
    if (R > 1) {
        // rank 0 exports a fabric handle, NCCL broadcasts its 64 bytes, the others import it
        CUmemFabricHandle fh;
        std::memset(&fh, 0, sizeof(fh));
        if (c->rank == 0) DRV(A.MemExportToShareableHandle(&fh, b->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0), "export");
        void* dbuf = nullptr;
        if (cudaMalloc(&dbuf, sizeof(fh)) != cudaSuccess) { nvls_free(b); set_error("nvls: staging alloc"); return SLB_ERR_OOM; }
        cudaMemcpy(dbuf, &fh, sizeof(fh), cudaMemcpyHostToDevice);
        ncclResult_t nr = nccl().Broadcast(dbuf, dbuf, sizeof(fh), ncclUint8, 0, c->comm, 0);
        cudaMemcpy(&fh, dbuf, sizeof(fh), cudaMemcpyDeviceToHost);
        cudaFree(dbuf);
        if (nr != ncclSuccess) { nvls_free(b); set_error("nvls: handle broadcast"); return SLB_ERR_NCCL; }
        if (c->rank != 0) DRV(A.MemImportFromShareableHandle(&b->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC), "import");
    }
    DRV(A.MulticastAddDevice(b->mc, b->dev), "cuMulticastAddDevice");
    if (R > 1) {                                  // every device joins before anyone binds memory
        int* flag = nullptr;
        cudaMalloc(&flag, sizeof(int));
        ncclResult_t nr = nccl().AllReduce(flag, flag, 1, ncclInt32, ncclSum, c->comm, 0);
        cudaStreamSynchronize(0);
        cudaFree(flag);
        if (nr != ncclSuccess) { nvls_free(b); set_error("nvls: join barrier"); return SLB_ERR_NCCL; }
    }
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = R > 1 ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    DRV(A.MemCreate(&b->mem, size, &ap, 0), "cuMemCreate");
    DRV(A.MulticastBindMem(b->mc, 0, b->mem, 0, size, 0), "cuMulticastBindMem");
    b->bound = true;
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV(A.MemAddressReserve(&b->uc_va, size, gran, 0, 0), "reserve (unicast)");
    DRV(A.MemMap(b->uc_va, size, 0, b->mem, 0), "map (unicast)");
    DRV(A.MemSetAccess(b->uc_va, size, &acc, 1), "access (unicast)");
    DRV(A.MemAddressReserve(&b->mc_va, size, gran, 0, 0), "reserve (multicast)");
    DRV(A.MemMap(b->mc_va, size, 0, b->mc, 0), "map (multicast)");
    DRV(A.MemSetAccess(b->mc_va, size, &acc, 1), "access (multicast)");
    return SLB_OK;
}

}  // namespace slb

extern "C" int slb_nvls_supported(void) { return slb::nvls_supported() ? 1 : 0; }
