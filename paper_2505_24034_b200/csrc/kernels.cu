// kernels.cu -- the hot path for sm_100a.
//
// K1 relayout + cast + move   (a3; §5.2: each GPU sends its
//                               own shards straight into the generator's CUDA
//                               memory over NVLink, no CPU, no PS hop)
// K2 fp8 128x128 block quant  (a4; "quantization ... on the inference side",
//                               P:145; arithmetic = DESIGN.md R7)
// K3 completion               (a6; release/acquire epoch counters, R10)
//
// One persistent kernel per device and sync executes every work item that
// device owns (push items for tiles it sources, pull items for multi-source fp8
// blocks landing on it).  The work is a memory-movement problem with ~1 ALU op
// per element: no tensor cores; the design targets HBM and NVLink bandwidth:
// 16-byte vector loads (L1 no-allocate, read-only path) and 16-byte stores to
// local or peer-mapped addresses, several independent loads in flight per
// thread, and a grid of (#SMs x resident CTAs) CTAs striding over work items
// that the planner interleaved across destinations.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "kernels.h"

namespace llrl {

namespace {

__device__ __forceinline__ uint4 ld_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// RNE fp32 -> bf16 of two values; `lo` lands in the low half (lower address).
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ uint16_t bf16_rn(float x) {
    uint16_t r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x));
    return r;
}

// RN + satfinite fp32 -> e4m3 of two values; `lo` lands in the low byte.
__device__ __forceinline__ uint32_t e4m3x2_rn(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// ---- K1: relayout + cast ----------------------------------------------------

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

// 8 elements (one 16-byte destination vector for bf16) per vector step.
template <bool SRC_F32>
__device__ __forceinline__ void cast_item(const Item &it, const KParams &P) {
    const char *src = static_cast<const char *>(P.src[it.src_rank]);
    char *dst = static_cast<char *>(P.dst[it.dst_rank]);
    constexpr int es = SRC_F32 ? 4 : 2;
    const bool dst_f32 = it.flags & F_DST_F32;
    if (it.flags & F_VEC) {
        const int vpr = it.cols >> 3;
        const int nvec = it.rows * vpr;
        for (int v0 = threadIdx.x; v0 < nvec; v0 += kThreads * kUnroll) {
            uint4 a[kUnroll], b[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                const int v = v0 + u * kThreads;
                if (v < nvec) {
                    const int r = v / vpr, c = (v - r * vpr) << 3;
                    const char *s = src + (it.src_off + int64_t(r) * it.src_ld + c) * es;
                    a[u] = ld_stream(s);
                    if (SRC_F32) b[u] = ld_stream(s + 16);
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                const int v = v0 + u * kThreads;
                if (v < nvec) {
                    const int r = v / vpr, c = (v - r * vpr) << 3;
                    const int64_t doff = it.dst_off + int64_t(r) * it.dst_ld + c;
                    if (SRC_F32) {
                        if (dst_f32) {
                            st_v4(dst + doff * 4, a[u]);
                            st_v4(dst + doff * 4 + 16, b[u]);
                        } else {
                            uint4 o;
                            o.x = bf16x2_rn(__uint_as_float(a[u].x), __uint_as_float(a[u].y));
                            o.y = bf16x2_rn(__uint_as_float(a[u].z), __uint_as_float(a[u].w));
                            o.z = bf16x2_rn(__uint_as_float(b[u].x), __uint_as_float(b[u].y));
                            o.w = bf16x2_rn(__uint_as_float(b[u].z), __uint_as_float(b[u].w));
                            st_v4(dst + doff * 2, o);
                        }
                    } else {
                        st_v4(dst + doff * 2, a[u]);
                    }
                }
            }
        }
    } else {
        const int n = it.rows * it.cols;
        for (int e = threadIdx.x; e < n; e += kThreads) {
            const int r = e / it.cols, c = e - r * it.cols;
            const int64_t so = it.src_off + int64_t(r) * it.src_ld + c;
            const int64_t dof = it.dst_off + int64_t(r) * it.dst_ld + c;
            if (SRC_F32) {
                const uint32_t x = *reinterpret_cast<const uint32_t *>(src + so * 4);
                if (dst_f32) *reinterpret_cast<uint32_t *>(dst + dof * 4) = x;
                else *reinterpret_cast<uint16_t *>(dst + dof * 2) = bf16_rn(__uint_as_float(x));
            } else {
                *reinterpret_cast<uint16_t *>(dst + dof * 2) = *reinterpret_cast<const uint16_t *>(src + so * 2);
            }
        }
    }
}

// ---- K2: fp8 block quantisation (R7) ------------------------------------------

// Block-wide max of non-negative fp32 bit patterns (order-preserving as u32).
__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t *s_red) {
    v = __reduce_max_sync(0xffffffffu, v);
    __syncthreads();                       // s_red reuse across items
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t m = s_red[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; w++) m = max(m, s_red[w]);
    return m;
}

__device__ __forceinline__ void fp8_scales(uint32_t amax_bits, float *inv, float *scale) {
    const float amax_c = fmaxf(__uint_as_float(amax_bits), 0x1p-64f);
    *inv = __fdiv_rn(448.0f, amax_c);
    *scale = __fdiv_rn(amax_c, 448.0f);
}

// Single-source block, vector path: thread t covers rows (t/8) + 32k, k < 4,
// columns [(t%8)*16, +16).  Raw source words stay in registers between the
// amax pass and the quantise pass (one HBM read per element).
template <bool SRC_F32>
__device__ __forceinline__ void fp8_item_vec(const Item &it, const KParams &P, uint32_t *s_red) {
    constexpr int W = SRC_F32 ? 4 : 2;           // 16-byte words per 16 elements
    const char *src = static_cast<const char *>(P.src[it.src_rank]);
    char *dst = static_cast<char *>(P.dst[it.dst_rank]);
    const int rg = threadIdx.x >> 3;
    const int cc = (threadIdx.x & 7) * 16;
    const bool col_ok = cc < it.cols;
    uint4 w[4][W];
    uint32_t amax = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = rg + 32 * k;
        if (col_ok && r < it.rows) {
            const char *s = src + (it.src_off + int64_t(r) * it.src_ld + cc) * (SRC_F32 ? 4 : 2);
#pragma unroll
            for (int j = 0; j < W; j++) w[k][j] = ld_stream(s + 16 * j);
        } else {
#pragma unroll
            for (int j = 0; j < W; j++) w[k][j] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < W; j++) {
            const uint32_t q[4] = {w[k][j].x, w[k][j].y, w[k][j].z, w[k][j].w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (SRC_F32) {
                    amax = max(amax, q[e] & 0x7FFFFFFFu);
                } else {
                    amax = max(amax, (q[e] << 16) & 0x7FFFFFFFu);
                    amax = max(amax, q[e] & 0x7FFF0000u);
                }
            }
        }
    }
    amax = block_max_u32(amax, s_red);
    float inv, scale;
    fp8_scales(amax, &inv, &scale);
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = rg + 32 * k;
        if (col_ok && r < it.rows) {
            float x[16];
#pragma unroll
            for (int j = 0; j < W; j++) {
                const uint32_t q[4] = {w[k][j].x, w[k][j].y, w[k][j].z, w[k][j].w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if (SRC_F32) {
                        x[4 * j + e] = __uint_as_float(q[e]);
                    } else {
                        x[8 * j + 2 * e] = bf16_lo(q[e]);
                        x[8 * j + 2 * e + 1] = bf16_hi(q[e]);
                    }
                }
            }
            uint32_t ow[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t lo = e4m3x2_rn(__fmul_rn(x[4 * i], inv), __fmul_rn(x[4 * i + 1], inv));
                const uint32_t hi = e4m3x2_rn(__fmul_rn(x[4 * i + 2], inv), __fmul_rn(x[4 * i + 3], inv));
                ow[i] = lo | (hi << 16);
            }
            st_v4(dst + it.dst_off + int64_t(r) * it.dst_ld + cc, make_uint4(ow[0], ow[1], ow[2], ow[3]));
        }
    }
    if (threadIdx.x == 0) *reinterpret_cast<float *>(dst + it.aux) = scale;
}

template <bool SRC_F32>
__device__ __forceinline__ float load_elem(const char *base, int64_t idx) {
    if (SRC_F32) return *reinterpret_cast<const float *>(base + idx * 4);
    return __uint_as_float(uint32_t(*reinterpret_cast<const uint16_t *>(base + idx * 2)) << 16);
}

// Generic block (unaligned single source, or several sources = pull, R8):
// two element-strided passes over the block's segments.
template <bool SRC_F32>
__device__ void fp8_item_generic(const Item &it, const KParams &P, uint32_t *s_red) {
    char *dst = static_cast<char *>(P.dst[it.dst_rank]);
    Seg one;
    const Seg *segs;
    int nseg;
    if (it.kind == K_FP8) {
        one.src_off = it.src_off; one.src_ld = it.src_ld; one.src_rank = it.src_rank;
        one.r0 = 0; one.c0 = 0; one.rows = it.rows; one.cols = it.cols;
        segs = &one;
        nseg = 1;
    } else {
        segs = P.segs + it.src_off;
        nseg = it.src_rank;
    }
    uint32_t amax = 0;
    for (int s = 0; s < nseg; s++) {
        const Seg sg = segs[s];
        const char *src = static_cast<const char *>(P.src[sg.src_rank]);
        const int n = sg.rows * sg.cols;
        for (int e = threadIdx.x; e < n; e += kThreads) {
            const int r = e / sg.cols, c = e - r * sg.cols;
            amax = max(amax, __float_as_uint(load_elem<SRC_F32>(src, sg.src_off + int64_t(r) * sg.src_ld + c)) & 0x7FFFFFFFu);
        }
    }
    amax = block_max_u32(amax, s_red);
    float inv, scale;
    fp8_scales(amax, &inv, &scale);
    for (int s = 0; s < nseg; s++) {
        const Seg sg = segs[s];
        const char *src = static_cast<const char *>(P.src[sg.src_rank]);
        const int n = sg.rows * sg.cols;
        for (int e = threadIdx.x; e < n; e += kThreads) {
            const int r = e / sg.cols, c = e - r * sg.cols;
            const float x = load_elem<SRC_F32>(src, sg.src_off + int64_t(r) * sg.src_ld + c);
            const uint8_t q = uint8_t(e4m3x2_rn(__fmul_rn(x, inv), 0.0f) & 0xFF);
            dst[it.dst_off + int64_t(sg.r0 + r) * it.dst_ld + sg.c0 + c] = q;
        }
    }
    if (threadIdx.x == 0) *reinterpret_cast<float *>(dst + it.aux) = scale;
}

// ---- the persistent sync kernel + K3 signal -------------------------------------

// MODE 0: relayout + cast items only (low register count -> full occupancy);
// MODE 1: fp8 block items.  The planner sorts a device's items as
// [cast items | fp8 items]; each launch covers one contiguous range.
template <bool SRC_F32, int MODE>
__global__ void __launch_bounds__(kThreads) llrl_k_sync(const __grid_constant__ KParams P) {
    __shared__ uint32_t s_red[kThreads / 32];
    for (int i = P.item_begin + blockIdx.x; i < P.item_end; i += gridDim.x) {
        const Item it = P.items[i];
        if (MODE == 0) {
            cast_item<SRC_F32>(it, P);
        } else if (it.kind == K_FP8 && (it.flags & F_VEC)) {
            fp8_item_vec<SRC_F32>(it, P, s_red);
        } else {
            fp8_item_generic<SRC_F32>(it, P, s_red);
        }
    }
    if (P.done != nullptr) {
        // Completion (a6): every thread orders its stores at system scope, the CTA
        // joins, one thread counts the CTA in; the last CTA of this launch
        // publishes one arrival to every destination device with a release add.
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long prev = atomicAdd(P.done, 1ULL);
            if (prev + 1 == P.done_target) {
                __threadfence_system();
                for (int s = 0; s < P.n_signal; s++)
                    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(P.signal[s]) : "memory");
            }
        }
    }
}

// K3 receiver: spin (acquire, system scope) until `target` arrivals, bounded by
// a timeout so a missing peer cannot hang the GPU; on timeout flag[1] = 1.
__global__ void llrl_k_wait(unsigned long long *flag, unsigned long long target, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    unsigned long long t0, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= target) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > timeout_ns) {
            atomicExch(flag + 1, 1ULL);
            return;
        }
        __nanosleep(256);
    }
}

}  // namespace

template <int MODE>
static cudaError_t launch_mode(const KParams &P, bool src_f32, int grid, cudaStream_t stream) {
    if (src_f32) llrl_k_sync<true, MODE><<<grid, kThreads, 0, stream>>>(P);
    else llrl_k_sync<false, MODE><<<grid, kThreads, 0, stream>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_sync(const KParams &P, int mode, bool src_f32, int grid, cudaStream_t stream) {
    return mode == 0 ? launch_mode<0>(P, src_f32, grid, stream) : launch_mode<1>(P, src_f32, grid, stream);
}

cudaError_t launch_wait(unsigned long long *flag, unsigned long long target, cudaStream_t stream) {
    llrl_k_wait<<<1, 32, 0, stream>>>(flag, target, 30ull * 1000 * 1000 * 1000);
    return cudaGetLastError();
}

int sync_threads() { return kThreads; }

cudaError_t sync_occupancy(int mode, bool src_f32, int *blocks_per_sm) {
    const void *fn = mode == 0 ? (src_f32 ? (const void *)llrl_k_sync<true, 0> : (const void *)llrl_k_sync<false, 0>)
                               : (src_f32 ? (const void *)llrl_k_sync<true, 1> : (const void *)llrl_k_sync<false, 1>);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, kThreads, 0);
}

}  // namespace llrl
