// mc_bulk_probe.cu -- can anything but multimem.st feed an NVLS multicast object
// faster than ~570 GB/s (C9's multicast bound)?  Single process, every visible GPU
// in the multicast team (as in C9: GPU 0 writes, the others receive; GPU 0 binds
// memory too).  GPU 0 writes `bytes` through the multicast VA with
//   (a) multimem.st.relaxed.sys.global.v4.f32  (the shipped path)
//   (b) st.global.v4 (plain stores to the multicast VA)
//   (c) cp.async.bulk.global.shared::cta       (TMA bulk stores, 32 KiB stages)
//   (d) cudaMemcpyAsync device -> multicast VA (copy engine)
// checks that every GPU received the data and prints GB/s of user bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_bulk_probe mc_bulk_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
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

__device__ __forceinline__ uint4 pattern(size_t i, unsigned salt) {
    const unsigned v = unsigned(i) * 2654435761u + salt;
    return make_uint4(v, v + 1, v + 2, v + 3);
}

__global__ void k_multimem(char *mc, size_t n16, unsigned salt) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = pattern(i, salt);
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 16 * i),
                     "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
                     "f"(__uint_as_float(v.w))
                     : "memory");
    }
}

__global__ void k_plain(char *mc, size_t n16, unsigned salt) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = pattern(i, salt);
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 16 * i), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w)
                     : "memory");
    }
}

// TMA bulk stores: each CTA fills a 32 KiB shared stage with the pattern, then
// cp.async.bulk's it to consecutive 32 KiB blocks of the destination (2 stages).
constexpr int kStage = 32 * 1024;
__global__ void __launch_bounds__(256) k_bulk(char *mc, size_t nblk, unsigned salt) {
    extern __shared__ __align__(128) unsigned char sm[];
    int buf = 0;
    for (size_t b = blockIdx.x; b < nblk; b += gridDim.x, buf ^= 1) {
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        uint4 *s = reinterpret_cast<uint4 *>(sm + buf * kStage);
        for (int j = threadIdx.x; j < kStage / 16; j += blockDim.x) s[j] = pattern(b * (kStage / 16) + j, salt);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned saddr = unsigned(__cvta_generic_to_shared(s));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(mc + b * kStage),
                         "r"(saddr), "r"(kStage)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill(char *p, size_t n16, unsigned salt) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        reinterpret_cast<uint4 *>(p)[i] = pattern(i, salt);
}

__global__ void k_check(const char *p, size_t n16, unsigned salt, unsigned long long *bad) {
    unsigned long long b = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = reinterpret_cast<const uint4 *>(p)[i], w = pattern(i, salt);
        b += (v.x != w.x) | (v.y != w.y) | (v.z != w.z) | (v.w != w.w);
    }
    if (b) atomicAdd(bad, b);
}

int main(int argc, char **argv) {
    CU(cuInit(0));
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    printf("devices %d\n", ndev);
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t want = (argc > 1 ? size_t(atoll(argv[1])) : 2048ull) << 20;   // bytes per write
    std::vector<CUdevice> dev(ndev);
    std::vector<CUcontext> ctx(ndev);
    for (int i = 0; i < ndev; i++) {
        CU(cuDeviceGet(&dev[i], i));
        CU(cuDevicePrimaryCtxRetain(&ctx[i], dev[i]));
    }
    CU(cuCtxSetCurrent(ctx[0]));
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = ndev;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = want;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    mp.size = (want + gran - 1) / gran * gran;
    const size_t size = mp.size;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int i = 0; i < ndev; i++) CU(cuMulticastAddDevice(mc, dev[i]));
    std::vector<CUmemGenericAllocationHandle> mem(ndev);
    std::vector<CUdeviceptr> uva(ndev);
    for (int i = 0; i < ndev; i++) {
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
    char *srcbuf = nullptr;
    cudaSetDevice(0);
    cudaMalloc(&srcbuf, size);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStage);
    unsigned long long *bad = nullptr;
    cudaMallocManaged(&bad, sizeof *bad);
    const size_t n16 = size / 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[4] = {"multimem.st.v4", "st.global.v4 to MC VA", "cp.async.bulk to MC VA", "cudaMemcpyAsync to MC VA"};
    for (int m = 0; m < 4; m++) {
        const unsigned salt = 1000u * (m + 1);
        for (int i = 0; i < ndev; i++) {
            CU(cuCtxSetCurrent(ctx[i]));
            CU(cuMemsetD8(uva[i], 0, size));
            cudaDeviceSynchronize();
        }
        CU(cuCtxSetCurrent(ctx[0]));
        if (m == 3) {
            k_fill<<<296, 512>>>(srcbuf, n16, salt);
            cudaDeviceSynchronize();
        }
        float best = 1e30f;
        cudaError_t err = cudaSuccess;
        for (int rep = 0; rep < 4 && err == cudaSuccess; rep++) {
            cudaEventRecord(e0);
            if (m == 0) k_multimem<<<296, 512>>>(reinterpret_cast<char *>(mcva), n16, salt);
            if (m == 1) k_plain<<<296, 512>>>(reinterpret_cast<char *>(mcva), n16, salt);
            if (m == 2) k_bulk<<<148, 256, 2 * kStage>>>(reinterpret_cast<char *>(mcva), size / kStage, salt);
            if (m == 3) err = cudaMemcpyAsync(reinterpret_cast<void *>(mcva), srcbuf, size, cudaMemcpyDeviceToDevice);
            cudaEventRecord(e1);
            cudaError_t e2 = cudaEventSynchronize(e1);
            if (err == cudaSuccess) err = e2;
            if (err == cudaSuccess) err = cudaGetLastError();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        if (err != cudaSuccess) {
            printf("%-28s FAILED: %s\n", names[m], cudaGetErrorString(err));
            if (err == cudaErrorIllegalAddress || err == cudaErrorLaunchFailure) return 1;   // context is gone
            cudaGetLastError();
            continue;
        }
        printf("%-28s %.3f ms for %.2f GB -> %.1f GB/s;", names[m], best, size / 1e9, size / best / 1e6);
        for (int i = 0; i < ndev; i++) {
            cudaSetDevice(i);
            *bad = 0;
            k_check<<<296, 512>>>(reinterpret_cast<const char *>(uva[i]), n16, salt, bad);
            cudaDeviceSynchronize();
            printf(" dev%d bad=%llu", i, *bad);
        }
        printf("\n");
        cudaSetDevice(0);
        CU(cuCtxSetCurrent(ctx[0]));
    }
    printf("PROBE_DONE\n");
    return 0;
}
