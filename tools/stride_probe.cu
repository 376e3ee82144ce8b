// stride_probe.cu -- HBM read rate of strided row segments (the o / down column
// bands of FSDP row chunks that C2 / C3 / C12 read) vs contiguous reads, with the
// same TMA bulk-copy pipeline the sync kernels use: one CTA per SM, 4 x 32 KiB
// shared-memory stages filled by cp.async.bulk (one copy per row segment), the
// stage discarded once landed.  Reads `total` bytes as segments of `seg` bytes
// at a pitch of `pitch` bytes (pitch = seg: contiguous), CTA b taking stage
// blocks b, b + grid, ...
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stride_probe stride_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int kStage = 32 * 1024, kStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(64) k_read(const char *base, int64_t nrows, int64_t seg, int64_t pitch,
                                             int64_t nbands, int band_major) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[kStages];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; s++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // a stage = rows_per segments of one band: rows r0.., band b (column offset b * seg)
    const int64_t rows_per = kStage / seg;
    const int64_t blocks_per_band = (nrows + rows_per - 1) / rows_per, nblk = blocks_per_band * nbands;
    int n = 0;
    for (int64_t k = blockIdx.x; k < nblk; k += gridDim.x, n++) {
        const int st = n % kStages;
        if (n >= kStages) {   // wait for the stage's previous fill (phase of its last use)
            const uint32_t ph = ((n / kStages) - 1) & 1;
            asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
                         ::"r"(smem_u32(&full[st])), "r"(ph) : "memory");
        }
        // row-major: concurrent CTAs read sibling bands of the same rows; band-major:
        // one band's row blocks in sequence (the plan's tile order)
        const int64_t band = band_major ? k / blocks_per_band : k % nbands;
        const int64_t r0 = (band_major ? k % blocks_per_band : k / nbands) * rows_per;
        const int64_t nr = r0 + rows_per <= nrows ? rows_per : nrows - r0;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])),
                         "r"(uint32_t(nr * seg)) : "memory");
        __syncwarp();
        for (int64_t r = lane; r < nr; r += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + st * kStage + r * seg)), "l"(base + (r0 + r) * pitch + band * seg),
                         "r"(uint32_t(seg)), "r"(smem_u32(&full[st]))
                         : "memory");
    }
    for (int j = 0; j < kStages && j < n; j++) {   // drain
        const int m = n - 1 - j, st = m % kStages;
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
                     ::"r"(smem_u32(&full[st])), "r"(uint32_t((m / kStages) & 1)) : "memory");
    }
}

int main() {
    const int64_t total = 16ll << 30;
    char *buf = nullptr;
    if (cudaMalloc(&buf, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(buf, 1, total);
    cudaFuncSetAttribute(k_read, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // (segment bytes, bands per row): pitch = seg * bands.  bands = 1: contiguous rows
    const int64_t cases[][2] = {{32768, 1}, {16384, 1}, {2048, 1}, {2048, 8},  {4096, 4},  {7168, 8},
                                {14336, 4}, {1024, 8},  {2048, 4}, {8192, 8},  {2048, 16}, {3584, 8}};
    for (int bm = 0; bm < 2; bm++)
    for (auto &c : cases) {
        const int64_t seg = c[0], bands = c[1], pitch = seg * bands, nrows = total / pitch;
        if (bm && bands == 1) continue;
        float best = 1e30f;
        for (int rep = 0; rep < 4; rep++) {
            cudaEventRecord(a);
            k_read<<<sms, 64, kStages * kStage>>>(buf, nrows, seg, pitch, bands, bm);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const cudaError_t e = cudaGetLastError();
        printf("%s seg %6lld B x %2lld bands (pitch %6lld B): %.3f ms, %.1f GB/s %s\n", bm ? "band-major" : "row-major ",
               (long long)seg, (long long)bands,
               (long long)pitch, best, nrows * pitch / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
