// multicast.cu -- NVLS multicast buffers for generator DP replicas (NEXT f1:
// "N gen replicas receive one write each").
//
// One multicast object per generator rank position (TP rank x PP stage); its
// team is every GPU of the job.  Each replica GPU binds its generator buffer
// (VMM memory created here) at offset 0; every other GPU binds a scratch
// allocation of the same size (the NVSwitch delivers every multicast store to
// every team member).  A sender maps the multicast VA and stores once; the
// switch replicates to all replicas, so the sender's NVLink egress is one copy
// instead of dp_gen copies.  Driver API calls go through cudaGetDriverEntryPoint
// (no libcuda link dependency; the library still loads on GPU-less hosts).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <unistd.h>

#include "internal.h"

using namespace llrl;

namespace {

struct Drv {
    CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long);
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*mcGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
    CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*addrFree)(CUdeviceptr, size_t);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
    CUresult (*exportHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
    CUresult (*importHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
    CUresult (*deviceGet)(CUdevice *, int);
    bool ok = false;
};

Drv &drv() {
    static Drv d;
    static bool tried = false;
    if (tried) return d;
    tried = true;
    auto get = [](const char *name, void **fn) {
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
               q == cudaDriverEntryPointSuccess && *fn;
    };
    d.ok = get("cuMulticastCreate", (void **)&d.mcCreate) && get("cuMulticastAddDevice", (void **)&d.mcAddDevice) &&
           get("cuMulticastBindMem", (void **)&d.mcBindMem) && get("cuMulticastUnbind", (void **)&d.mcUnbind) &&
           get("cuMulticastGetGranularity", (void **)&d.mcGranularity) && get("cuMemCreate", (void **)&d.memCreate) &&
           get("cuMemRelease", (void **)&d.memRelease) && get("cuMemAddressReserve", (void **)&d.addrReserve) &&
           get("cuMemAddressFree", (void **)&d.addrFree) && get("cuMemMap", (void **)&d.memMap) &&
           get("cuMemUnmap", (void **)&d.memUnmap) && get("cuMemSetAccess", (void **)&d.setAccess) &&
           get("cuMemExportToShareableHandle", (void **)&d.exportHandle) &&
           get("cuMemImportFromShareableHandle", (void **)&d.importHandle) && get("cuDeviceGet", (void **)&d.deviceGet);
    return d;
}

llrl_status cu_fail(CUresult r, const char *what) {
    set_error("%s failed (CUresult %d)", what, int(r));
    return LLRL_E_CUDA;
}

#define CUK(call, what)                                   \
    do {                                                  \
        CUresult r_ = (call);                             \
        if (r_ != CUDA_SUCCESS) return cu_fail(r_, what); \
    } while (0)

}  // namespace

struct llrl_mcbuf {
    CUmemGenericAllocationHandle mc = 0;
    size_t size = 0, gran = 0;
    int n_devices = 0;
    int device = -1;                         // the local device (bound / mapped)
    CUmemGenericAllocationHandle mem = 0;    // local physical memory bound to the object
    CUdeviceptr local = 0, mcva = 0;         // unicast VA of the local memory, multicast VA
    bool bound = false;
    std::vector<std::pair<CUdeviceptr, CUmemGenericAllocationHandle>> peers;   // peers' memory mapped here
};

extern "C" {

llrl_status llrl_mc_create(int n_devices, int64_t bytes, int *fd_out, int64_t *size_out, llrl_mcbuf **out) {
    if (n_devices < 1 || bytes <= 0 || !fd_out || !out) { set_error("llrl_mc_create: invalid argument"); return LLRL_E_INVALID; }
    Drv &d = drv();
    if (!d.ok) { set_error("multicast driver entry points unavailable"); return LLRL_E_UNSUPPORTED; }
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = unsigned(n_devices);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = size_t(bytes);
    size_t gran = 0;
    CUK(d.mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    mp.size = (size_t(bytes) + gran - 1) / gran * gran;
    llrl_mcbuf *m = new (std::nothrow) llrl_mcbuf();
    if (!m) { set_error("out of host memory"); return LLRL_E_NOMEM; }
    CUresult r = d.mcCreate(&m->mc, &mp);
    if (r != CUDA_SUCCESS) { delete m; return cu_fail(r, "cuMulticastCreate"); }
    int fd = -1;
    r = d.exportHandle(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) { d.memRelease(m->mc); delete m; return cu_fail(r, "cuMemExportToShareableHandle"); }
    m->size = mp.size;
    m->gran = gran;
    m->n_devices = n_devices;
    *fd_out = fd;
    if (size_out) *size_out = int64_t(mp.size);
    *out = m;
    return LLRL_OK;
}

llrl_status llrl_mc_import(int fd, int n_devices, int64_t size, llrl_mcbuf **out) {
    if (fd < 0 || n_devices < 1 || size <= 0 || !out) { set_error("llrl_mc_import: invalid argument"); return LLRL_E_INVALID; }
    Drv &d = drv();
    if (!d.ok) { set_error("multicast driver entry points unavailable"); return LLRL_E_UNSUPPORTED; }
    llrl_mcbuf *m = new (std::nothrow) llrl_mcbuf();
    if (!m) { set_error("out of host memory"); return LLRL_E_NOMEM; }
    CUresult r = d.importHandle(&m->mc, reinterpret_cast<void *>(intptr_t(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) { delete m; return cu_fail(r, "cuMemImportFromShareableHandle"); }
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = unsigned(n_devices);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = size_t(size);
    size_t gran = 0;
    r = d.mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) { d.memRelease(m->mc); delete m; return cu_fail(r, "cuMulticastGetGranularity"); }
    m->size = size_t(size);
    m->gran = gran;
    m->n_devices = n_devices;
    *out = m;
    return LLRL_OK;
}

// Add `device` to the team, create its physical memory (the whole object size),
// bind it at offset 0, map it at a unicast VA (*local_ptr) and map the
// multicast VA (*mc_ptr).  Blocks until every team member has joined.
llrl_status llrl_mc_join(llrl_mcbuf *m, int device, void **local_ptr, void **mc_ptr) {
    if (!m || device < 0 || !local_ptr || !mc_ptr || m->bound) { set_error("llrl_mc_join: invalid argument"); return LLRL_E_INVALID; }
    Drv &d = drv();
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) {
        set_error("llrl_mc_join: cannot use device %d", device);
        return LLRL_E_CUDA;
    }
    CUdevice dev;
    CUK(d.deviceGet(&dev, device), "cuDeviceGet");
    CUK(d.mcAddDevice(m->mc, dev), "cuMulticastAddDevice");
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUK(d.memCreate(&m->mem, m->size, &ap, 0), "cuMemCreate");
    CUK(d.mcBindMem(m->mc, 0, m->mem, 0, m->size, 0), "cuMulticastBindMem");
    CUmemAccessDesc ad;
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = device;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUK(d.addrReserve(&m->local, m->size, m->gran, 0, 0), "cuMemAddressReserve");
    CUK(d.memMap(m->local, m->size, 0, m->mem, 0), "cuMemMap");
    CUK(d.setAccess(m->local, m->size, &ad, 1), "cuMemSetAccess");
    CUK(d.addrReserve(&m->mcva, m->size, m->gran, 0, 0), "cuMemAddressReserve(mc)");
    CUK(d.memMap(m->mcva, m->size, 0, m->mc, 0), "cuMemMap(mc)");
    CUK(d.setAccess(m->mcva, m->size, &ad, 1), "cuMemSetAccess(mc)");
    m->device = device;
    m->bound = true;
    *local_ptr = reinterpret_cast<void *>(m->local);
    *mc_ptr = reinterpret_cast<void *>(m->mcva);
    cudaSetDevice(prev);
    return LLRL_OK;
}

llrl_status llrl_mc_export_local(const llrl_mcbuf *m, int *fd_out) {
    if (!m || !fd_out || !m->bound) { set_error("llrl_mc_export_local: invalid argument (join first)"); return LLRL_E_INVALID; }
    int fd = -1;
    CUK(drv().exportHandle(&fd, m->mem, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
    *fd_out = fd;
    return LLRL_OK;
}

llrl_status llrl_mc_map_peer(llrl_mcbuf *m, int fd, int device, void **ptr) {
    if (!m || fd < 0 || device < 0 || !ptr) { set_error("llrl_mc_map_peer: invalid argument"); return LLRL_E_INVALID; }
    Drv &d = drv();
    if (!d.ok) { set_error("multicast driver entry points unavailable"); return LLRL_E_UNSUPPORTED; }
    CUmemGenericAllocationHandle h = 0;
    CUK(d.importHandle(&h, reinterpret_cast<void *>(intptr_t(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
        "cuMemImportFromShareableHandle(peer)");
    CUdeviceptr va = 0;
    CUresult r = d.addrReserve(&va, m->size, m->gran, 0, 0);
    if (r == CUDA_SUCCESS) r = d.memMap(va, m->size, 0, h, 0);
    if (r == CUDA_SUCCESS) {
        CUmemAccessDesc ad;
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = device;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = d.setAccess(va, m->size, &ad, 1);
    }
    if (r != CUDA_SUCCESS) {
        if (va) { d.memUnmap(va, m->size); d.addrFree(va, m->size); }
        d.memRelease(h);
        return cu_fail(r, "llrl_mc_map_peer");
    }
    m->peers.push_back({va, h});
    *ptr = reinterpret_cast<void *>(va);
    return LLRL_OK;
}

void llrl_mc_destroy(llrl_mcbuf *m) {
    if (!m) return;
    Drv &d = drv();
    if (d.ok) {
        for (auto &pv : m->peers) {
            d.memUnmap(pv.first, m->size);
            d.addrFree(pv.first, m->size);
            d.memRelease(pv.second);
        }
        if (m->mcva) { d.memUnmap(m->mcva, m->size); d.addrFree(m->mcva, m->size); }
        if (m->local) { d.memUnmap(m->local, m->size); d.addrFree(m->local, m->size); }
        if (m->bound) {
            CUdevice dev;
            if (d.deviceGet(&dev, m->device) == CUDA_SUCCESS) d.mcUnbind(m->mc, dev, 0, m->size);
        }
        if (m->mem) d.memRelease(m->mem);
        if (m->mc) d.memRelease(m->mc);
    }
    delete m;
}

llrl_status llrl_plan_set_multicast(llrl_plan *p, int device, void *const *dst_mc_ptrs) {
    if (!p || device < 0 || device >= p->n_devices || !dst_mc_ptrs) { set_error("invalid argument"); return LLRL_E_INVALID; }
    DeviceWork &W = p->dev[size_t(device)];
    W.dst_mc.assign(dst_mc_ptrs, dst_mc_ptrs + p->n_dst);
    return LLRL_OK;
}

}  // extern "C"
