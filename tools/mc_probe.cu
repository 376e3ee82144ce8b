// mc_probe.cu -- feasibility probe for NVLS multicast on this box (single
// process, 2 GPUs): create a multicast object, bind one VMM allocation per
// GPU, map the multicast VA on GPU 0, store through it with st.global and
// multimem.st, and check that both GPUs received the data.  Also reports
// whether FABRIC / POSIX-FD shareable handles can be exported.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x)                                                                  \
    do {                                                                       \
        CUresult r_ = (x);                                                     \
        if (r_ != CUDA_SUCCESS) {                                              \
            const char *s_ = nullptr;                                          \
            cuGetErrorString(r_, &s_);                                         \
            printf("FAIL %s: %d %s\n", #x, int(r_), s_ ? s_ : "?");            \
            return 1;                                                          \
        }                                                                      \
    } while (0)

__global__ void store_plain(unsigned *mc, unsigned n, unsigned v) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) mc[i] = v + i;
}
__global__ void store_multimem(float *mc, unsigned n4) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        float a = float(4 * i), b = a + 1, c = a + 2, d = a + 3;
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(a), "f"(b),
                     "f"(c), "f"(d)
                     : "memory");
    }
    __threadfence_system();
}

int main() {
    CU(cuInit(0));
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    printf("devices %d\n", ndev);
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    CUdevice dev[2];
    CUcontext ctx[2];
    for (int i = 0; i < 2; i++) {
        CU(cuDeviceGet(&dev[i], i));
        CU(cuDevicePrimaryCtxRetain(&ctx[i], dev[i]));
    }
    CU(cuCtxSetCurrent(ctx[0]));
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = 2;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = 64ull << 20;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("mc granularity %zu\n", gran);
    mp.size = (mp.size + gran - 1) / gran * gran;
    const size_t size = mp.size;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int i = 0; i < 2; i++) CU(cuMulticastAddDevice(mc, dev[i]));
    CUmemGenericAllocationHandle mem[2];
    CUdeviceptr uva[2];
    for (int i = 0; i < 2; i++) {
        CU(cuCtxSetCurrent(ctx[i]));
        CUmemAllocationProp ap;
        memset(&ap, 0, sizeof ap);
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = i;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CU(cuMemCreate(&mem[i], size, &ap, 0));
        CU(cuMulticastBindMem(mc, 0, mem[i], 0, size, 0));
        CU(cuMemAddressReserve(&uva[i], size, gran, 0, 0));
        CU(cuMemMap(uva[i], size, 0, mem[i], 0));
        CUmemAccessDesc ad;
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = i;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CU(cuMemSetAccess(uva[i], size, &ad, 1));
        CU(cuMemsetD8(uva[i], 0, size));
    }
    CU(cuCtxSetCurrent(ctx[0]));
    CUdeviceptr mcva;
    CU(cuMemAddressReserve(&mcva, size, gran, 0, 0));
    CU(cuMemMap(mcva, size, 0, mc, 0));
    CUmemAccessDesc ad0;
    ad0.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad0.location.id = 0;
    ad0.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(mcva, size, &ad0, 1));
    const unsigned n = 1u << 20;
    store_plain<<<148, 256>>>(reinterpret_cast<unsigned *>(mcva), n, 7);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("FAIL plain store kernel\n"); return 1; }
    std::vector<unsigned> h(n);
    for (int i = 0; i < 2; i++) {
        CU(cuCtxSetCurrent(ctx[i]));
        CU(cuMemcpyDtoH(h.data(), uva[i], n * 4));
        unsigned bad = 0;
        for (unsigned k = 0; k < n; k++) bad += h[k] != 7 + k;
        printf("st.global via MC VA -> device %d: %u mismatches\n", i, bad);
    }
    CU(cuCtxSetCurrent(ctx[0]));
    store_multimem<<<148, 256>>>(reinterpret_cast<float *>(mcva + (16u << 20)), n / 4);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("FAIL multimem kernel\n"); return 1; }
    std::vector<float> f(n);
    for (int i = 0; i < 2; i++) {
        CU(cuCtxSetCurrent(ctx[i]));
        CU(cuMemcpyDtoH(f.data(), uva[i] + (16u << 20), n * 4));
        unsigned bad = 0;
        for (unsigned k = 0; k < n; k++) bad += f[k] != float(k);
        printf("multimem.st -> device %d: %u mismatches\n", i, bad);
    }
    // shareable handle export of the multicast object
    int fd = -1;
    CUresult r = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    printf("export POSIX fd: %d (fd %d)\n", int(r), fd);
    // fabric handles need a separate object created with the FABRIC type
    CUmulticastObjectProp mp2 = mp;
    mp2.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    CUmemGenericAllocationHandle mc2;
    r = cuMulticastCreate(&mc2, &mp2);
    printf("create FABRIC mc: %d\n", int(r));
    if (r == CUDA_SUCCESS) {
        CUmemFabricHandle fh;
        r = cuMemExportToShareableHandle(&fh, mc2, CU_MEM_HANDLE_TYPE_FABRIC, 0);
        printf("export FABRIC: %d\n", int(r));
    }
    printf("PROBE_DONE\n");
    return 0;
}
