// kernels.cu -- the hot path for sm_100a.
//
// K1  llrl_k_cast_tma  relayout + cast + move (a3; §5.2: each
//                      GPU sends its own shards straight into the generator's
//                      CUDA memory over NVLink, no CPU, no PS hop), plus the
//                      MXFP8 / MXFP4 / NVFP4 row-group quantisation (R13, R15,
//                      R16).
//                      Warp-specialised: a producer warp stages rows with
//                      cp.async.bulk (TMA) into a 4-deep shared-memory ring,
//                      worker warps convert in shared memory, a storer warp
//                      writes back with bulk copies to local or peer HBM.
// K1r llrl_k_cast<U,M> register variant of K1 (16-byte LDG / STG, U loads in
//                      flight per thread); used for NVLS multicast stores (f1).
// K2  llrl_k_fp8_tma   fp8 128x128 block quantisation (a4; R7): 2-D tensor-map
//                      TMA box per block, warp-specialised like K1.
// K2r llrl_k_fp8       register variant of K2.
// K3  completion       (a6): last CTA of a launch publishes a release add to every
//                      destination GPU's per-sender counter; llrl_k_wait spins
//                      with acquire loads (R10).
// K4  llrl_k_nv_amax   NVFP4 per-tensor partial amax (bulk-copy staged), the
// K5  llrl_k_nv_scale / llrl_k_nv_fetch  cross-GPU amax handshake (R16).
//
// The work is memory movement with about one ALU op per element: no dense
// contraction, no tensor cores; the design targets HBM and NVLink bandwidth.
// Every launch is a persistent grid (one or two CTAs per SM for the TMA
// kernels) striding over work items the planner interleaved across destinations.
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

__device__ __forceinline__ void st_v2(void *p, uint32_t x, uint32_t y) {
    asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(x), "r"(y) : "memory");
}

__device__ __forceinline__ void st_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// NVLS multicast stores (f1): one store, replicated by the NVSwitch to every
// GPU bound to the multicast object.  Bit patterns pass through unchanged
// (no arithmetic on a store).
__device__ __forceinline__ void mc_st_v4(void *p, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(v.x)),
                 "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
}
__device__ __forceinline__ void mc_st_v2(void *p, uint32_t x, uint32_t y) {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(__uint_as_float(x)),
                 "f"(__uint_as_float(y))
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

// One "unit" = 16 bytes of SOURCE (4 fp32 or 8 bf16 elements).  Thread t of a
// CTA handles units t, t + 256, ... so every warp-wide load instruction reads
// 512 contiguous bytes and every store instruction writes 256 (f32->bf16,
// 8-byte stores) or 512 contiguous bytes: full 32-byte sectors both ways.
// U units per thread are loaded before any is stored (U x 16 B in flight).
template <bool SRC_F32, int U>
__device__ __forceinline__ void cast_item(const Item &it, const KParams &P) {
    const char *src = static_cast<const char *>(P.src[it.src_rank]);
    char *dst = static_cast<char *>(P.dst[it.dst_rank]);
    constexpr int es = SRC_F32 ? 4 : 2;
    constexpr int E = 16 / es;                       // elements per unit
    const bool dst_f32 = it.flags & F_DST_F32;
    if (it.flags & F_VEC) {                          // planner: offsets, lds, cols multiples of 8 elements
        const int upr = it.cols / E;                 // units per row
        const int nunits = it.rows * upr;
        const bool one_d = it.rows == 1;
        const bool mc = it.flags & F_MC;
        if (mc) dst = static_cast<char *>(P.dst_mc[it.dst_rank]);
        const char *sbase = src + it.src_off * es;
        char *dbase = dst + it.dst_off * (dst_f32 ? 4 : 2);
        for (int u0 = threadIdx.x; u0 < nunits; u0 += kThreads * U) {
            uint4 a[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int u = u0 + k * kThreads;
                if (u < nunits) {
                    int r = 0, c = u * E;
                    if (!one_d) { r = u / upr; c = (u - r * upr) * E; }
                    a[k] = ld_stream(sbase + (int64_t(r) * it.src_ld + c) * es);
                }
            }
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int u = u0 + k * kThreads;
                if (u >= nunits) break;
                int r = 0, c = u * E;
                if (!one_d) { r = u / upr; c = (u - r * upr) * E; }
                const int64_t doff = int64_t(r) * it.dst_ld + c;
                if (SRC_F32 && !dst_f32) {
                    const uint32_t lo = bf16x2_rn(__uint_as_float(a[k].x), __uint_as_float(a[k].y));
                    const uint32_t hi = bf16x2_rn(__uint_as_float(a[k].z), __uint_as_float(a[k].w));
                    if (mc) mc_st_v2(dbase + doff * 2, lo, hi);
                    else st_v2(dbase + doff * 2, lo, hi);
                } else if (mc) {
                    mc_st_v4(dbase + doff * es, a[k]);
                } else {
                    st_v4(dbase + doff * es, a[k]);   // identity (f32->f32, bf16->bf16)
                }
            }
        }
    } else {
        if (it.flags & F_MC) dst = static_cast<char *>(P.dst_mc[it.dst_rank]);   // plain stores to the MC VA
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

// Named barrier over the 256 threads that process blocks (barrier 1): the TMA
// producer warp of llrl_k_fp8_tma never joins it.
__device__ __forceinline__ void workers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Block-wide max of non-negative fp32 bit patterns (order-preserving as u32).
// Callers alternate between two 8-word s_red buffers from item to item, so one
// barrier per item suffices (a warp can run at most one item ahead).
__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t *s_red) {
    v = __reduce_max_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    workers_sync();
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

// |x| bit patterns of one 16-byte word of source elements, max-accumulated
// (as fp32 bit patterns: order-preserving for non-negative values).  bf16
// words: |x| on both halves with one mask, pairwise max.bf16x2, then the two
// halves -- about one instruction per element.
__device__ __forceinline__ uint32_t max_bf16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// max(|a|, |b|) per bf16 half; the sign bits are junk (xor of the inputs'),
// cleared by the caller.  NaN inputs lose to numbers, as with max.bf16x2.
__device__ __forceinline__ uint32_t maxabs_bf16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// |x| max of two 16-byte words of bf16 (16 elements) as an fp32 bit pattern.
__device__ __forceinline__ uint32_t amax16_bf16(const uint4 &a, const uint4 &b) {
    const uint32_t m = maxabs_bf16x2(maxabs_bf16x2(maxabs_bf16x2(a.x, a.y), maxabs_bf16x2(a.z, a.w)),
                                     maxabs_bf16x2(maxabs_bf16x2(b.x, b.y), maxabs_bf16x2(b.z, b.w))) &
                       0x7FFF7FFFu;
    return max(m << 16, m & 0xFFFF0000u);
}

template <bool SRC_F32>
__device__ __forceinline__ uint32_t word_amax(uint4 w, uint32_t amax) {
    if (SRC_F32) {
        amax = max(amax, w.x & 0x7FFFFFFFu);
        amax = max(amax, w.y & 0x7FFFFFFFu);
        amax = max(amax, w.z & 0x7FFFFFFFu);
        return max(amax, w.w & 0x7FFFFFFFu);
    }
    constexpr uint32_t m = 0x7FFF7FFFu;
    const uint32_t p = max_bf16x2(max_bf16x2(w.x & m, w.y & m), max_bf16x2(w.z & m, w.w & m));
    return max(amax, max(p << 16, p & 0xFFFF0000u));
}

// (a, b) * r on the packed fp32x2 datapath (sm_100: one instruction, both
// products fp32 RN, identical to two __fmul_rn).
__device__ __forceinline__ void mul2_rn(float &a, float &b, float r) {
    asm("{\n .reg .b64 x, s;\n mov.b64 x, {%0, %1};\n mov.b64 s, {%2, %2};\n"
        " mul.rn.f32x2 x, x, s;\n mov.b64 {%0, %1}, x;\n}"
        : "+f"(a), "+f"(b)
        : "f"(r));
}

// 8 products -> 4 bytes of e2m1 codes (element 2i in the low nibble of byte i).
__device__ __forceinline__ uint32_t e2m1x8_rn(const float *y) {
    uint32_t d;
    asm("{\n .reg .b8 c0, c1, c2, c3;\n"
        " cvt.rn.satfinite.e2m1x2.f32 c0, %2, %1;\n"
        " cvt.rn.satfinite.e2m1x2.f32 c1, %4, %3;\n"
        " cvt.rn.satfinite.e2m1x2.f32 c2, %6, %5;\n"
        " cvt.rn.satfinite.e2m1x2.f32 c3, %8, %7;\n"
        " mov.b32 %0, {c0, c1, c2, c3};\n}"
        : "=r"(d)
        : "f"(y[0]), "f"(y[1]), "f"(y[2]), "f"(y[3]), "f"(y[4]), "f"(y[5]), "f"(y[6]), "f"(y[7]));
    return d;
}

// 16 source elements (W words) -> 16 e4m3 codes (one 16-byte word).
template <bool SRC_F32, int W>
__device__ __forceinline__ uint4 quant16(const uint4 *w, float inv) {
    float x[16];
#pragma unroll
    for (int j = 0; j < W; j++) {
        const uint32_t q[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
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
#pragma unroll
    for (int i = 0; i < 8; i++) mul2_rn(x[2 * i], x[2 * i + 1], inv);
    uint32_t ow[4];
#pragma unroll
    for (int i = 0; i < 4; i++) ow[i] = e4m3x2_rn(x[4 * i], x[4 * i + 1]) | (e4m3x2_rn(x[4 * i + 2], x[4 * i + 3]) << 16);
    return make_uint4(ow[0], ow[1], ow[2], ow[3]);
}

// Exact value of an E4M3FN code (finite codes only).
__device__ __forceinline__ float e4m3_value(uint32_t code) {
    const uint32_t E = (code >> 3) & 0xF, m = code & 0x7;
    const float v = E == 0 ? float(m) * 0x1p-9f : __uint_as_float(((E + 120u) << 23) | (m << 20));
    return (code & 0x80) ? -v : v;
}

// x / 6 correctly rounded (fp32 RN) for x >= 0: q = x * RN(1/6) and one fma
// correction (Markstein), exact for every float in [2^-100, FLT_MAX] (it is
// not near the subnormal range: those, inf and NaN take the full division).
// Exhaustively checked against the RN quotient by tests/test_arith_cpu.py.
__device__ __forceinline__ float div6_rn(float x) {
    constexpr float y = 0x1.555556p-3f;              // RN(1/6)
    if (!(x >= 0x1p-100f && x <= 0x1.fffffep127f)) return __fdiv_rn(x, 6.0f);
    const float q = __fmul_rn(x, y);
    const float r = __fmaf_rn(-6.0f, q, x);
    return __fmaf_rn(r, y, q);
}

// 16 source elements (W words) -> 16 e2m1 codes, two per byte, the even
// element in the low nibble (cvt.e2m1x2 puts its first operand in the high nibble).
template <bool SRC_F32, int W>
__device__ __forceinline__ uint2 quant16_e2m1(const uint4 *w, float inv) {
    float x[16];
#pragma unroll
    for (int j = 0; j < W; j++) {
        const uint32_t q[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
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
#pragma unroll
    for (int i = 0; i < 8; i++) mul2_rn(x[2 * i], x[2 * i + 1], inv);
    return make_uint2(e2m1x8_rn(x), e2m1x8_rn(x + 8));
}

// Single-source block, thread t covers rows (t/8) + 32k, k < 4, columns
// [(t%8)*16, +16).  Raw source words stay in registers between the amax pass
// and the quantise pass (one HBM read per element).  FROM_SMEM: the block was
// staged by TMA into `stage` (row pitch 128 elements); else loaded from HBM.
template <bool SRC_F32, bool FROM_SMEM>
__device__ __forceinline__ void fp8_block(const Item &it, const KParams &P, const unsigned char *stage,
                                          uint32_t *s_red) {
    constexpr int es = SRC_F32 ? 4 : 2;
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
            if (FROM_SMEM) {
                const uint4 *s = reinterpret_cast<const uint4 *>(stage + (r * 128 + cc) * es);
#pragma unroll
                for (int j = 0; j < W; j++) w[k][j] = s[j];
            } else {
                const char *s = src + (it.src_off + int64_t(r) * it.src_ld + cc) * es;
#pragma unroll
                for (int j = 0; j < W; j++) w[k][j] = ld_stream(s + 16 * j);
            }
        } else {
#pragma unroll
            for (int j = 0; j < W; j++) w[k][j] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < W; j++) amax = word_amax<SRC_F32>(w[k][j], amax);
    }
    amax = block_max_u32(amax, s_red);
    float inv, scale;
    fp8_scales(amax, &inv, &scale);
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = rg + 32 * k;
        if (col_ok && r < it.rows)
            st_v4(dst + it.dst_off + int64_t(r) * it.dst_ld + cc, quant16<SRC_F32, W>(w[k], inv));
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

// Completion (a6): every thread orders its stores at system scope, the CTA
// joins, one thread counts the CTA in; the last CTA of the launch resets the
// counter for the next launch on the stream and publishes one arrival to every
// destination device with a release add at system scope.  No per-call host
// state: the launch parameters are the same on every call, so a sync can be
// captured once in a CUDA graph and replayed.
// Programmatic dependent launch: a cast launch lets the fp8 launch queued
// behind it start at once (the two touch disjoint items); the fp8 grid then
// waits for the cast grid's completion before it completes or signals.
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Debug timeline (LLRL_TIMELINE=1): %globaltimer at CTA start / after its last
// store, per CTA of the cast launch (llrl_debug_timeline).
__device__ __forceinline__ void timeline_mark(const KParams &P, int which) {
    if (P.timeline == nullptr) return;
    if (which) __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.timeline[2 * blockIdx.x + which] = t;
    }
}

__device__ __forceinline__ void complete(const KParams &P) {
    timeline_mark(P, 1);
    if (P.queue) {
        // dynamic item queue (llrl_k_cast_tma): the last CTA out -- every claim
        // made -- resets it for the next launch (graph-replayable)
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(P.queue + 1, 1u) + 1 == gridDim.x) {
            atomicExch(P.queue, 0u);
            atomicExch(P.queue + 1, 0u);
        }
    }
    if (P.pdl_wait) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (P.done == nullptr) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long prev = atomicAdd(P.done, 1ULL);
        if (prev + 1 == gridDim.x) {
            atomicExch(P.done, 0ULL);
            __threadfence_system();
            for (int s = 0; s < P.n_signal; s++)
                asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(P.signal[s]) : "memory");
        }
    }
}

// K1 launch: relayout + cast items [item_begin, item_end), persistent CTAs.
template <bool SRC_F32, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) llrl_k_cast(const __grid_constant__ KParams P) {
    pdl_release();
    timeline_mark(P, 0);
    for (int i = P.item_begin + blockIdx.x; i < P.item_end; i += gridDim.x) {
        const Item it = P.items[i];
        cast_item<SRC_F32, U>(it, P);
    }
    complete(P);
}

// K2 launch, register variant: fp8 block items loaded straight from HBM.
template <bool SRC_F32>
__global__ void __launch_bounds__(kThreads) llrl_k_fp8(const __grid_constant__ KParams P) {
    __shared__ uint32_t s_red[2][kThreads / 32];
    int k = 0;
    for (int i = P.item_begin + blockIdx.x; i < P.item_end; i += gridDim.x, ++k) {
        const Item it = P.items[i];
        if (it.kind == K_FP8 && (it.flags & F_VEC)) fp8_block<SRC_F32, false>(it, P, nullptr, s_red[k & 1]);
        else fp8_item_generic<SRC_F32>(it, P, s_red[k & 1]);
    }
    complete(P);
}

// ---- K2 TMA pipeline -------------------------------------------------------------
// Warp-specialised: warp 8 (producer) stages each block's rows into shared
// memory with cp.async.bulk (one bulk copy per row, completion counted in
// bytes on the stage's mbarrier), up to fp8_stages() blocks ahead; warps 0-7
// (workers) reduce amax and quantise from shared memory and release the stage.
// Loads of the next blocks overlap the reduction of the current one.

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok)
                     : "r"(smem_u32(b)), "r"(parity)
                     : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 2-D tensor TMA: one 128x128 box of the piece's tensor map at (x, y); rows /
// columns outside the piece are zero-filled (never used: workers mask).
__device__ __forceinline__ void tma_box_g2s(void *dst_smem, const void *tmap, int x, int y, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(dst_smem)), "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
                 : "memory");
}

// 3-D tensor TMA: box of a strided cast band's map at row `row` (kernels' own
// [rows][n1][b0] 8-byte-unit view, runtime.cu ensure_cast_tmaps).
__device__ __forceinline__ void tma_box3_g2s(void *dst_smem, const void *tmap, int row, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(dst_smem)), "l"(tmap), "r"(0), "r"(0), "r"(row), "r"(smem_u32(bar))
                 : "memory");
}

template <bool SRC_F32>
__host__ __device__ constexpr int fp8_stages() { return SRC_F32 ? 3 : 3; }
template <bool SRC_F32>
__host__ __device__ constexpr int fp8_stage_bytes() { return 128 * 128 * (SRC_F32 ? 4 : 2); }

template <bool SRC_F32, int NST = fp8_stages<SRC_F32>(), int MINB = 2>
__global__ void __launch_bounds__(kThreads + 32, MINB) llrl_k_fp8_tma(const __grid_constant__ KParams P) {
    constexpr int S = NST;
    constexpr int kStage = fp8_stage_bytes<SRC_F32>();
    constexpr int es = SRC_F32 ? 4 : 2;
    extern __shared__ __align__(128) unsigned char stages[];
    __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S];
    __shared__ Item slot[S];
    __shared__ uint32_t s_red[2][kThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kThreads / 32) {
        // producer
        int k = 0;
        for (int i = P.item_begin + blockIdx.x; i < P.item_end; i += gridDim.x, ++k) {
            const int st = k % S;
            mbar_wait(&empty_bar[st], ((k / S) & 1) ^ 1);
            const Item it = P.items[i];
            const bool tma = it.kind == K_FP8 && (it.flags & F_VEC);
            const TmaRef ref = tma ? P.tma_refs[i - P.fp8_base] : TmaRef{-1, 0, 0, 0};
            if (lane == 0) {
                slot[st] = it;
                if (tma && ref.map >= 0) {
                    // the whole 128x128 box lands (zero-filled outside the piece)
                    mbar_arrive_tx(&full_bar[st], uint32_t(kStage));
                    tma_box_g2s(stages + st * kStage, static_cast<const unsigned char *>(P.tmaps) + 128 * ref.map,
                                ref.x, ref.y, &full_bar[st]);
                } else if (tma) {
                    mbar_arrive_tx(&full_bar[st], uint32_t(it.rows * it.cols * es));
                } else {
                    mbar_arrive(&full_bar[st]);
                }
            }
            __syncwarp();
            if (tma && ref.map < 0) {
                const char *src = static_cast<const char *>(P.src[it.src_rank]) + it.src_off * es;
                for (int r = lane; r < it.rows; r += 32)
                    bulk_g2s(stages + st * kStage + r * 128 * es, src + int64_t(r) * it.src_ld * es,
                             uint32_t(it.cols * es), &full_bar[st]);
            }
        }
    } else {
        // workers
        int k = 0;
        for (int i = P.item_begin + blockIdx.x; i < P.item_end; i += gridDim.x, ++k) {
            const int st = k % S;
            mbar_wait(&full_bar[st], (k / S) & 1);
            const Item it = slot[st];
            if (it.kind == K_FP8 && (it.flags & F_VEC))
                fp8_block<SRC_F32, true>(it, P, stages + st * kStage, s_red[k & 1]);
            else
                fp8_item_generic<SRC_F32>(it, P, s_red[k & 1]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
        }
    }
    complete(P);
}

// ---- K1: TMA-staged relayout + cast / quantisation ------------------------------
// Warp-specialised: warp 0 (producer) stages each item's rows into an NST-deep
// ring of SB-byte shared-memory stages with cp.async.bulk (mbarrier tx-count
// completion); warp 1 (storer) writes each converted stage back with
// cp.async.bulk shared -> global (local HBM or a peer GPU's HBM over NVLink)
// and releases it once the bulk store has read it; warps 2.. (NWK workers)
// convert in shared memory (fp32 -> bf16, MXFP8 / MXFP4 / NVFP4 groups).  Data
// never passes through registers on identity copies (bf16 -> bf16).

// TMA cast kernel configurations: (stage bytes, stages, worker threads, CTAs/SM)
#define LLRL_TMA_A 32 * 1024, 4, 512, 1
#define LLRL_TMA_B 16 * 1024, 4, 256, 2
#define LLRL_TMA_C 32 * 1024, 4, 256, 1

// Chunk k of a cast item: `nr` rows x `nc` columns starting at (r0, c0) of the
// item, at most kCastStageBytes of source.  Same enumeration on both roles.
struct Chunk {
    int r0, nr, c0, nc;
};
template <int SB>
__device__ __forceinline__ int cast_chunks(const Item &it, int es, int *rows_per, int *segs_per_row) {
    const int row_bytes = it.cols * es;
    if (row_bytes <= SB) {
        *rows_per = SB / row_bytes;
        *segs_per_row = 1;
        return (it.rows + *rows_per - 1) / *rows_per;
    }
    *rows_per = 1;
    *segs_per_row = (row_bytes + SB - 1) / SB;
    return it.rows * *segs_per_row;
}
template <int SB>
__device__ __forceinline__ Chunk cast_chunk(const Item &it, int es, int rows_per, int segs_per_row, int k) {
    Chunk c;
    if (it.rows == 1) {                 // one (long) row: segments, no division
        const int seg_elems = SB / es;
        c.r0 = 0;
        c.nr = 1;
        c.c0 = k * seg_elems;
        c.nc = min(seg_elems, it.cols - c.c0);
    } else if (segs_per_row == 1) {
        c.r0 = k * rows_per;
        c.nr = min(rows_per, it.rows - c.r0);
        c.c0 = 0;
        c.nc = it.cols;
    } else {
        const int seg_elems = SB / es;
        c.r0 = k / segs_per_row;
        c.nr = 1;
        c.c0 = (k % segs_per_row) * seg_elems;
        c.nc = min(seg_elems, it.cols - c.c0);
    }
    return c;
}

// The item sequence of a CTA, which its three roles walk in lockstep, each role
// looping over an item's chunks (stages) inside its item loop -- per-item work
// (descriptor load, flags, chunk geometry, NVFP4 tensor table) stays out of the
// per-stage path, which matters for the quantising variant's 16 KiB stages
// (two 16-element units per worker thread per stage).
// Static phase, items [item_begin, static_end): striding (CTA b takes items b,
// b + gridDim.x, ...) or, with P.static_block, a contiguous block of them per
// CTA (the plan interleaves destinations in proportion to their bytes, so a
// block carries every destination's share while a stride can alias with the
// interleave period); every role walks this sequence itself.
// Claimed phase, items [static_end, item_end) (only with P.queue): the producer
// claims each item with one atomicAdd (the next claim in flight while the
// current item's copies are issued) and hands the item to the other roles in
// shared memory at the item's first stage (index -1: end of work).  The claimed
// tail absorbs the spread of per-SM and per-link speeds, so all CTAs finish
// together.
struct ItemWalk {
    int i, step, static_hi;
    unsigned claimed;
    bool dyn;
};
__device__ __forceinline__ void walk_init(ItemWalk &w, const KParams &P, bool producer, int lane) {
    if (P.static_block) {
        const int64_t n = P.static_end - P.item_begin;
        w.step = 1;
        w.i = P.item_begin + int(n * blockIdx.x / gridDim.x) - 1;
        w.static_hi = P.item_begin + int(n * (blockIdx.x + 1) / gridDim.x);
    } else {
        w.step = int(gridDim.x);
        w.i = P.item_begin + int(blockIdx.x) - int(gridDim.x);
        w.static_hi = P.static_end;
    }
    w.claimed = 0;
    w.dyn = false;
    if (producer && P.queue && lane == 0) w.claimed = atomicAdd(P.queue, 1u);   // first claim, in flight
}
// Static phase: the next item (>= 0), or -1 at its end; sets w.dyn when a
// claimed phase follows.
__device__ __forceinline__ int walk_static(ItemWalk &w, const KParams &P) {
    w.i += w.step;
    if (w.i < w.static_hi) return w.i;
    w.dyn = P.queue != nullptr;
    return -1;
}
// Producer, claimed phase: the next claimed item, or -1 when the queue is empty.
__device__ __forceinline__ int walk_claim(ItemWalk &w, const KParams &P, int lane) {
    const int i = P.static_end + int(__shfl_sync(0xffffffffu, w.claimed, 0));
    if (i >= P.item_end) return -1;
    if (lane == 0) w.claimed = atomicAdd(P.queue, 1u);   // the next item, in flight
    return i;
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <bool SRC_F32, int SB, int NST, int NWK, int MINB>
__global__ void __launch_bounds__(64 + NWK, MINB) llrl_k_cast_tma(const __grid_constant__ KParams P) {
    constexpr int kCastStageBytes = SB, kCastStages = NST, kCastWorkers = NWK;
    pdl_release();
    timeline_mark(P, 0);
    // warp 0: producer (bulk loads global -> shared), warp 1: storer (bulk stores
    // shared -> global), warps 2..: workers (conversion in shared memory).  A stage
    // moves full (producer -> workers) -> converted (workers -> storer) -> empty
    // (storer -> producer, once its bulk store has read the stage).
    constexpr int es = SRC_F32 ? 4 : 2;
    constexpr int kWorkerWarps = kCastWorkers / 32;
    extern __shared__ __align__(128) unsigned char stages[];   // kCastStages x (in 32 KiB + out 16 KiB)
    constexpr int kOut = kCastStageBytes / 2;   // bf16, MXFP8 or MXFP4 codes of a chunk
    constexpr int kStride = kCastStageBytes + kOut;
    __shared__ __align__(8) uint64_t full_bar[kCastStages], conv_bar[kCastStages], empty_bar[kCastStages];
    __shared__ float nv_r[2][128], nv_senc[2];   // NVFP4: r per E4M3 code, S_enc (R16)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kCastStages; s++) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&conv_bar[s], kWorkerWarps);
            mbar_init(&empty_bar[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // claimed phase: the item (index, -1: end of work; descriptor) each stage
    // starts, written by the producer before its arrive on the stage's full
    // barrier (release -> acquire; the storer sees it through the workers' arrive)
    __shared__ int s_item[kCastStages];
    __shared__ Item s_it[kCastStages];
    ItemWalk w;
    walk_init(w, P, warp == 0, lane);
    if (warp == 0) {
        // producer: stages the rows of every vector item; scalar items pass a token
        int n = 0;
        for (;;) {
            int i = w.dyn ? -1 : walk_static(w, P);
            if (i < 0 && w.dyn) i = walk_claim(w, P, lane);
            if (i < 0) {
                if (w.dyn) {                      // end-of-work token for the other roles
                    const int st = n % kCastStages;
                    mbar_wait(&empty_bar[st], ((n / kCastStages) & 1) ^ 1);
                    if (lane == 0) {
                        s_item[st] = -1;
                        mbar_arrive(&full_bar[st]);
                    }
                }
                break;
            }
            const Item it = P.items[i];
            const bool vec = it.flags & F_VEC;
            int rows_per = 1, segs = 1;
            const int nch = vec ? cast_chunks<SB>(it, es, &rows_per, &segs) : 1;
            int band = -1, band_row = 0, band_rows = 0;   // strided-source band map (LLRL_CAST_TMAP)
            if (P.cast_refs) {
                const CastRef r = P.cast_refs[i];
                if (r.map >= 0 && (band_rows = P.cast_box[r.map]) > 0) {
                    band = r.map;
                    band_row = r.row;
                }
            }
            const char *src = static_cast<const char *>(P.src[it.src_rank]) + it.src_off * es;
            for (int k = 0; k < nch; k++, n++) {
                const int st = n % kCastStages;
                mbar_wait(&empty_bar[st], ((n / kCastStages) & 1) ^ 1);
                if (w.dyn && k == 0 && lane == 0) {
                    s_item[st] = i;
                    s_it[st] = it;
                }
                if (!vec) {
                    if (lane == 0) mbar_arrive(&full_bar[st]);
                    continue;
                }
                const Chunk c = cast_chunk<SB>(it, es, rows_per, segs, k);
                if (lane == 0) mbar_arrive_tx(&full_bar[st], uint32_t(c.nr * c.nc * es));
                __syncwarp();
                unsigned char *dst = stages + st * kStride;
                if (c.nc == it.src_ld) {          // rows contiguous in the source: one bulk copy
                    if (lane == 0)
                        bulk_g2s(dst, src + int64_t(c.r0) * it.src_ld * es, uint32_t(c.nr * c.nc * es), &full_bar[st]);
                } else if (band >= 0 && c.nc == it.cols && c.nr == band_rows) {
                    // strided whole rows: one 3-D tensor box (the band's map) instead of a copy per row
                    if (lane == 0)
                        tma_box3_g2s(dst, static_cast<const unsigned char *>(P.cast_tmaps) + 128 * band, band_row + c.r0,
                                     &full_bar[st]);
                } else {
                    for (int r = lane; r < c.nr; r += 32)
                        bulk_g2s(dst + r * c.nc * es, src + (int64_t(c.r0 + r) * it.src_ld + c.c0) * es,
                                 uint32_t(c.nc * es), &full_bar[st]);
                }
            }
        }
    } else if (warp == 1) {
        // storer: write each converted stage back, release it once read.  One item
        // body, inlined into the static loop (item from the plan table) and into
        // the claimed loop (item handed over in shared memory, its first stage's
        // barrier already passed).  The item is taken BY VALUE: its shared-memory
        // slot is rewritten once the producer recycles the item's first stage.
        int n = 0, pend = -1;
        auto item = [&](const Item it, const bool first_waited) {
            const bool vec = it.flags & F_VEC;
            int rows_per = 1, segs = 1;
            const int nch = vec ? cast_chunks<SB>(it, es, &rows_per, &segs) : 1;
            const bool mx = it.flags & F_MX, fp4 = it.flags & F_FP4;
            const bool cast = SRC_F32 && !(it.flags & F_DST_F32) && !mx;
            const int des = mx ? 1 : cast ? 2 : es;
            // F_MC: the position's multicast VA (bulk stores through NVLS, LLRL_MC_TMA=1)
            char *dbase = static_cast<char *>((it.flags & F_MC) ? P.dst_mc[it.dst_rank] : P.dst[it.dst_rank]);
            for (int k = 0; k < nch; k++, n++) {
                const int st = n % kCastStages;
                if (!(first_waited && k == 0)) mbar_wait(&conv_bar[st], (n / kCastStages) & 1);
                if (!vec) {                       // scalar item: workers wrote global memory directly
                    if (lane == 0) {
                        // release the deferred stage now: the producer may need it before
                        // another vector chunk arrives (deadlock with few CTAs otherwise)
                        if (pend >= 0) {
                            bulk_wait_read<0>();
                            mbar_arrive(&empty_bar[pend]);
                            pend = -1;
                        }
                        mbar_arrive(&empty_bar[st]);
                    }
                    continue;
                }
                if (lane == 0) {
                    const Chunk c = cast_chunk<SB>(it, es, rows_per, segs, k);
                    const unsigned char *out = stages + st * kStride + ((cast || mx) ? kCastStageBytes : 0);
                    // rows contiguous in the destination (chunk spans whole rows): one bulk store
                    const int nrow = c.nc == it.dst_ld ? 1 : c.nr, nel = c.nc == it.dst_ld ? c.nr * c.nc : c.nc;
                    for (int r = 0; r < nrow; r++) {
                        const int64_t e = it.dst_off + int64_t(c.r0 + r) * it.dst_ld + c.c0;   // element offset
                        if (fp4) bulk_s2g(dbase + e / 2, out + r * c.nc / 2, uint32_t(nel / 2));
                        else bulk_s2g(dbase + e * des, out + r * c.nc * des, uint32_t(nel * des));
                    }
                    bulk_commit();
                    bulk_wait_read<1>();              // the previous group has read its stage
                    if (pend >= 0) mbar_arrive(&empty_bar[pend]);
                    pend = st;
                }
            }
        };
        for (int i; (i = walk_static(w, P)) >= 0;) item(P.items[i], false);
        while (w.dyn) {                           // claimed phase: the item arrives with its first stage
            const int st = n % kCastStages;
            mbar_wait(&conv_bar[st], (n / kCastStages) & 1);
            if (s_item[st] < 0) break;
            item(s_it[st], true);
        }
        if (lane == 0) {
            bulk_wait_all();                      // every bulk store complete before the signal
            if (pend >= 0) mbar_arrive(&empty_bar[pend]);
        }
    } else {
        // workers: one item body, inlined into the static and the claimed loop (as
        // for the storer)
        const int wt = threadIdx.x - 64;
        int n = 0;
        int nv_tid = -1, nv_buf = 0;
        auto item = [&](const Item it, const bool first_waited) {
            const bool dst_f32 = it.flags & F_DST_F32;
            char *dbase = static_cast<char *>((it.flags & F_MC) ? P.dst_mc[it.dst_rank] : P.dst[it.dst_rank]);
            if (!(it.flags & F_VEC)) {
                const int st = n % kCastStages;
                if (!first_waited) mbar_wait(&full_bar[st], (n / kCastStages) & 1);
                const char *src = static_cast<const char *>(P.src[it.src_rank]);
                const int ne = it.rows * it.cols;
                for (int e = wt; e < ne; e += kCastWorkers) {
                    const int r = e / it.cols, c = e - r * it.cols;
                    const int64_t so = it.src_off + int64_t(r) * it.src_ld + c;
                    const int64_t dof = it.dst_off + int64_t(r) * it.dst_ld + c;
                    if (SRC_F32) {
                        const uint32_t x = *reinterpret_cast<const uint32_t *>(src + so * 4);
                        if (dst_f32) *reinterpret_cast<uint32_t *>(dbase + dof * 4) = x;
                        else *reinterpret_cast<uint16_t *>(dbase + dof * 2) = bf16_rn(__uint_as_float(x));
                    } else {
                        *reinterpret_cast<uint16_t *>(dbase + dof * 2) = *reinterpret_cast<const uint16_t *>(src + so * 2);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv_bar[st]);
                n++;
                return;
            }
            int rows_per, segs;
            const int nch = cast_chunks<SB>(it, es, &rows_per, &segs);
            const bool mx = it.flags & F_MX;
            const bool fp4 = it.flags & F_FP4;
            const bool nv = it.flags & F_NV;
            const bool cast = SRC_F32 && !dst_f32 && !mx;
            if (nv && it.tid != nv_tid) {
                // R16, per generator tensor: S_enc = 2688 / max(A, 2^-64), and for every
                // E4M3 group-scale code c the element multiplier r(c) = S_enc / s_q(c)
                // (0 for s_q = 0) -- one exact division per code instead of per group.
                // Double-buffered: a worker one tensor ahead writes the other table.
                nv_tid = it.tid;
                nv_buf ^= 1;
                const float A = fmaxf(__uint_as_float(P.nv_amax[it.tid]), 0x1p-64f);
                const float s_enc = __fdiv_rn(2688.0f, A);
                if (wt < 128) {
                    const float sq = e4m3_value(uint32_t(wt));
                    nv_r[nv_buf][wt] = (wt == 0 || wt == 127) ? 0.0f : __fdiv_rn(s_enc, sq);
                }
                if (wt == 0) nv_senc[nv_buf] = s_enc;
                asm volatile("bar.sync 1, %0;" ::"n"(NWK) : "memory");
            }
            for (int k = 0; k < nch; k++, n++) {
                const int st = n % kCastStages;
                if (!(first_waited && k == 0)) mbar_wait(&full_bar[st], (n / kCastStages) & 1);
                unsigned char *in = stages + st * kStride;
                unsigned char *out = in + kCastStageBytes;
                if (cast || mx) {
                    const Chunk c = cast_chunk<SB>(it, es, rows_per, segs, k);
                    if (cast) {
                        const int nunits = c.nr * c.nc / 4;          // 4 fp32 -> 4 bf16 per unit
                        for (int u = wt; u < nunits; u += kCastWorkers) {
                            const uint4 a = reinterpret_cast<const uint4 *>(in)[u];
                            reinterpret_cast<uint2 *>(out)[u] =
                                make_uint2(bf16x2_rn(__uint_as_float(a.x), __uint_as_float(a.y)),
                                           bf16x2_rn(__uint_as_float(a.z), __uint_as_float(a.w)));
                        }
                    } else {
                        // MX (R13 / R15): lanes (2j, 2j+1) hold the two halves of one 1x32 group;
                        // NVFP4 (R16): each thread's 16 elements are one 1x16 group
                        const int nunits = c.nr * c.nc / 16;         // 16 elements per thread
                        // NVFP4 scale byte of unit u: nv_s0 + u, plus nv_gap per chunk row
                        // (the row of unit u is floor((u + 0.5) / upr) through a float reciprocal:
                        // exact for upr <= 1024 units per chunk row, error < 2^-12)
                        const int gsh = nv ? 4 : 5;                  // log2 of the group size (offsets >= 0)
                        char *sb = dbase + it.aux + ((it.dst_off + int64_t(c.r0) * it.dst_ld + c.c0) >> gsh);
                        const int gap = c.nr > 1 ? int((it.dst_ld - c.nc) >> gsh) : 0;
                        const float inv_upr = __frcp_rn(float(c.nc / 16));
                        for (int u0 = 0; u0 < nunits; u0 += kCastWorkers) {
                            const int u = u0 + wt;
                            const bool live = u < nunits;
                            constexpr int W = SRC_F32 ? 4 : 2;
                            uint4 wd[W];
                            uint32_t amax = 0;
#pragma unroll
                            for (int j = 0; j < W; j++)
                                wd[j] = live ? reinterpret_cast<const uint4 *>(in + u * 16 * es)[j] : make_uint4(0, 0, 0, 0);
                            if (SRC_F32) {
#pragma unroll
                                for (int j = 0; j < W; j++) amax = word_amax<SRC_F32>(wd[j], amax);
                            } else {
                                amax = amax16_bf16(wd[0], wd[W - 1]);
                            }
                            if (nv) {
                                // group scale s = (amax / 6) * S_enc -> E4M3 code; r = S_enc / s_q
                                const float t6 = div6_rn(__uint_as_float(amax));
                                const uint32_t sc = e4m3x2_rn(__fmul_rn(t6, nv_senc[nv_buf]), 0.0f) & 0xFFu;
                                const float r = nv_r[nv_buf][sc];
                                if (live) {
                                    reinterpret_cast<uint2 *>(out)[u] = quant16_e2m1<SRC_F32, W>(wd, r);
                                    // scale byte: sb[u], plus gap per chunk row (dst_off, dst_ld, c0: whole groups)
                                    int g = u;
                                    if (gap) g += __float2int_rz((float(u) + 0.5f) * inv_upr) * gap;
                                    sb[g] = static_cast<char>(sc);
                                }
                                continue;
                            }
                            amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
                            // shared exponent floor(log2 amax) - emax (8 for E4M3, 2 for E2M1),
                            // clamped at -127: E8M0 code max(E - emax, 0)
                            const int code = max(int(amax >> 23) - (fp4 ? 2 : 8), 0);
                            const float inv = __uint_as_float(uint32_t(254 - code) << 23);   // 2^-(code - 127)
                            if (live) {
                                if (fp4) reinterpret_cast<uint2 *>(out)[u] = quant16_e2m1<SRC_F32, W>(wd, inv);
                                else reinterpret_cast<uint4 *>(out)[u] = quant16<SRC_F32, W>(wd, inv);
                                if ((u & 1) == 0) {   // group index as for NVFP4, 32-element groups
                                    int g = u >> 1;
                                    if (gap) g += __float2int_rz((float(u) + 0.5f) * inv_upr) * gap;
                                    sb[g] = static_cast<char>(code);
                                }
                            }
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv_bar[st]);
            }
        };
        for (int i; (i = walk_static(w, P)) >= 0;) item(P.items[i], false);
        while (w.dyn) {                           // claimed phase: the item arrives with its first stage
            const int st = n % kCastStages;
            mbar_wait(&full_bar[st], (n / kCastStages) & 1);
            if (s_item[st] < 0) {                 // end of work: pass the token to the storer
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv_bar[st]);
                break;
            }
            item(s_it[st], true);
        }
    }
    complete(P);
}

// ---- NVFP4 (R16) per-tensor amax: a max-reduction across the GPUs that feed
// each generator tensor, run inside the sync before the quantisation.
// Phase A (llrl_k_nv_amax, every contributing GPU): block max |x| of every
// NVFP4 item -> atomicMax into a local partial per tensor; the last CTA
// writes each partial into row [tensor][my device] of the owning GPU's table
// and signals it.  Phase B (llrl_k_nv_scale, owning GPU, after all partials
// arrived): global amax = max of the row, kept in the row's last word; the
// fp32 tensor scale A / 2688 goes into the generator buffer; partial words are
// cleared for the next sync; contributors are signalled.  Phase C
// (llrl_k_nv_fetch, contributors): copy the global amax of each contributed
// tensor into a local array the quantising kernel reads.
// Phase A streams the source through shared memory with bulk copies (one
// producer warp keeps kNvStages x 32 KiB in flight across item boundaries, as
// in llrl_k_cast_tma) and 8 reducer warps take max |x|.  Each CTA owns a
// contiguous range of items: consecutive items mostly belong to one tensor, so
// a CTA publishes one partial per tensor run (one atomic per warp) -- no
// same-address atomic storms.
constexpr int kNvStageBytes = 32 * 1024, kNvStages = 4;
template <bool SRC_F32>
__global__ void __launch_bounds__(kThreads + 32, 1) llrl_k_nv_amax(const __grid_constant__ NvAmaxParams P) {
    constexpr int es = SRC_F32 ? 4 : 2;
    extern __shared__ __align__(128) unsigned char stages[];
    __shared__ __align__(8) uint64_t full_bar[kNvStages], empty_bar[kNvStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kNvStages; st++) {
            mbar_init(&full_bar[st], 1);
            mbar_init(&empty_bar[st], kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // Each CTA takes one contiguous item range (P.run = 0, the default) or runs of
    // P.run items striped over the CTAs (LLRL_NV_RUN; a run is mostly one tensor,
    // so one atomic per warp per run either way).
    const int run = P.run > 0 ? P.run : (P.n_items + gridDim.x - 1) / gridDim.x;
    if (warp == kThreads / 32) {
        // producer
        int n = 0;
        for (int r0 = blockIdx.x * run; r0 < P.n_items; r0 += gridDim.x * run)
        for (int i = r0, i1 = min(P.n_items, r0 + run); i < i1; i++) {
            const Item it = P.items[i];
            if (!(it.flags & F_NV)) continue;
            int rows_per, segs;
            const int nch = cast_chunks<kNvStageBytes>(it, es, &rows_per, &segs);
            const char *src = static_cast<const char *>(P.src[it.src_rank]) + it.src_off * es;
            for (int k = 0; k < nch; k++, n++) {
                const int st = n % kNvStages;
                mbar_wait(&empty_bar[st], ((n / kNvStages) & 1) ^ 1);
                const Chunk c = cast_chunk<kNvStageBytes>(it, es, rows_per, segs, k);
                if (lane == 0) mbar_arrive_tx(&full_bar[st], uint32_t(c.nr * c.nc * es));
                __syncwarp();
                unsigned char *dst = stages + st * kNvStageBytes;
                if (c.nc == it.src_ld) {          // rows contiguous in the source: one bulk copy
                    if (lane == 0)
                        bulk_g2s(dst, src + int64_t(c.r0) * it.src_ld * es, uint32_t(c.nr * c.nc * es), &full_bar[st]);
                } else {
                    for (int r = lane; r < c.nr; r += 32)
                        bulk_g2s(dst + r * c.nc * es, src + (int64_t(c.r0 + r) * it.src_ld + c.c0) * es,
                                 uint32_t(c.nc * es), &full_bar[st]);
                }
            }
        }
    } else {
        // reducers
        uint32_t amax = 0;
        int cur = -1, n = 0;
        for (int r0 = blockIdx.x * run; r0 < P.n_items; r0 += gridDim.x * run)
        for (int i = r0, i1 = min(P.n_items, r0 + run); i < i1; i++) {
            const Item it = P.items[i];
            if (!(it.flags & F_NV)) continue;
            if (it.tid != cur) {
                if (cur >= 0) {
                    amax = __reduce_max_sync(0xffffffffu, amax);
                    if (lane == 0 && amax) atomicMax(P.partial + cur, amax);
                }
                amax = 0;
                cur = it.tid;
            }
            int rows_per, segs;
            const int nch = cast_chunks<kNvStageBytes>(it, es, &rows_per, &segs);
            for (int k = 0; k < nch; k++, n++) {
                const int st = n % kNvStages;
                const Chunk c = cast_chunk<kNvStageBytes>(it, es, rows_per, segs, k);
                const int nw = c.nr * c.nc * es / 16;
                mbar_wait(&full_bar[st], (n / kNvStages) & 1);
                const uint4 *w = reinterpret_cast<const uint4 *>(stages + st * kNvStageBytes);
                for (int v = threadIdx.x; v < nw; v += kThreads) amax = word_amax<SRC_F32>(w[v], amax);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[st]);
            }
        }
        if (cur >= 0) {
            amax = __reduce_max_sync(0xffffffffu, amax);
            if (lane == 0 && amax) atomicMax(P.partial + cur, amax);
        }
    }
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        const unsigned long long prev = atomicAdd(P.done, 1ULL);
        last = prev + 1 == gridDim.x;
        if (last) atomicExch(P.done, 0ULL);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int j = threadIdx.x; j < P.n_contrib; j += blockDim.x) {
        const int tid = P.contrib[j];
        const uint32_t v = atomicAdd(P.partial + tid, 0u);      // coherent read of the partial
        P.tables[P.tensor_dev[tid]][tid * kNvTableStride + P.my_dev] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < P.n_signal; s++)
            asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(P.signal[s]) : "memory");
}

__global__ void __launch_bounds__(kThreads) llrl_k_nv_scale(const __grid_constant__ NvScaleParams P) {
    const auto *loc = static_cast<const DeviceWork::NvLocal *>(P.locals);
    for (int j = threadIdx.x; j < P.n_local; j += kThreads) {
        uint32_t *row = P.table + loc[j].tid * kNvTableStride;
        uint32_t a = 0;
        for (int s = 0; s < kMaxDevices; s++) {
            a = max(a, row[s]);
            row[s] = 0;                                   // ready for the next sync
        }
        row[kMaxDevices] = a;
        const float A = fmaxf(__uint_as_float(a), 0x1p-64f);
        *reinterpret_cast<float *>(static_cast<char *>(P.dst[loc[j].dst_rank]) + loc[j].tscale_off) =
            __fdiv_rn(A, 2688.0f);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < P.n_signal; s++)
            asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(P.signal[s]) : "memory");
}

__global__ void __launch_bounds__(kThreads) llrl_k_nv_fetch(const __grid_constant__ NvFetchParams P) {
    for (int j = threadIdx.x; j < P.n_contrib; j += kThreads) {
        const int tid = P.contrib[j];
        P.amax_out[tid] = P.tables[P.tensor_dev[tid]][tid * kNvTableStride + kMaxDevices];
    }
}

// llrl_sync_nv_amax: the fp32 tensor scale A / 2688 of every local tensor from
// the caller-supplied amax (the same formula as llrl_k_nv_scale, R16).
__global__ void __launch_bounds__(kThreads) llrl_k_nv_tscale(const __grid_constant__ NvTscaleParams P) {
    const auto *loc = static_cast<const DeviceWork::NvLocal *>(P.locals);
    for (int j = threadIdx.x + blockIdx.x * kThreads; j < P.n_local; j += kThreads * gridDim.x) {
        const float A = fmaxf(__uint_as_float(P.amax[loc[j].tid]), 0x1p-64f);
        *reinterpret_cast<float *>(static_cast<char *>(P.dst[loc[j].dst_rank]) + loc[j].tscale_off) =
            __fdiv_rn(A, 2688.0f);
    }
}

// K3 receiver: thread s spins (acquire, system scope) until flag slot s reaches
// its target (0 = not waited on): slot ranges as in kernels.h (data arrivals,
// staging announcements, NVFP4 amax / ready per device).  One counter
// per sender, so a fast sender's later arrivals can never stand in for a slow
// sender's.  Bounded by a timeout so a missing peer cannot hang the GPU; on
// timeout flag[2 * kMaxDevices] = 1.
__global__ void llrl_k_wait(unsigned long long *flags, WaitTargets t, unsigned long long timeout_ns) {
    const int s = threadIdx.x;
    if (s >= kNumSlots || t.count[s] == 0) return;
    // expected arrivals live on the device (flags[kExpected + s]): graph-replayable
    unsigned long long *expected = flags + kFlagExpected + s;
    const unsigned long long target = *expected + t.count[s];
    *expected = target;
    unsigned long long t0, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + s) : "memory");
        if (v >= target) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > timeout_ns) {
            atomicExch(flags + kFlagTimeout, 1ULL);
            return;
        }
        __nanosleep(256);
    }
}

// Announce (release, system scope) that everything ordered before this kernel
// on its stream -- e.g. the H2D copy of a layer group -- is visible.
__global__ void llrl_k_signal(SignalTargets t) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int i = 0; i < t.n; i++) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(t.slot[i]) : "memory");
}

}  // namespace

// Cast-kernel variants: 0-5 = register kernel llrl_k_cast<U, MINB> (units in
// flight per thread, min resident CTAs per SM), 6 = TMA-staged llrl_k_cast_tma
// (default).  LLRL_CAST_VARIANT selects one for tuning.
struct CastVariant {
    const void *f32, *bf16;
};
#define LLRL_CV(U, M) {(const void *)llrl_k_cast<true, U, M>, (const void *)llrl_k_cast<false, U, M>}
static const CastVariant kCastVariants[] = {LLRL_CV(4, 1), LLRL_CV(8, 1), LLRL_CV(8, 4), LLRL_CV(4, 8),
                                            LLRL_CV(16, 1), LLRL_CV(2, 8)};
#undef LLRL_CV
constexpr int kNumCastVariants = int(sizeof(kCastVariants) / sizeof(kCastVariants[0]));

static const void *kernel_for(int mode, int variant, bool src_f32) {
    if (mode == 0 && variant == kCastTmaVariant)
        return src_f32 ? (const void *)llrl_k_cast_tma<true, LLRL_TMA_A> : (const void *)llrl_k_cast_tma<false, LLRL_TMA_A>;
    if (mode == 0 && variant == kCastTmaVariant + 1)
        return src_f32 ? (const void *)llrl_k_cast_tma<true, LLRL_TMA_B> : (const void *)llrl_k_cast_tma<false, LLRL_TMA_B>;
    if (mode == 0 && variant == kCastTmaVariant + 2)
        return src_f32 ? (const void *)llrl_k_cast_tma<true, LLRL_TMA_C> : (const void *)llrl_k_cast_tma<false, LLRL_TMA_C>;
    if (mode == 1) {
        if (variant == 0) return src_f32 ? (const void *)llrl_k_fp8<true> : (const void *)llrl_k_fp8<false>;
        if (variant == 2) return src_f32 ? (const void *)llrl_k_fp8_tma<true> : (const void *)llrl_k_fp8_tma<false, 6, 1>;
        if (variant == 3) return src_f32 ? (const void *)llrl_k_fp8_tma<true> : (const void *)llrl_k_fp8_tma<false, 2, 3>;
        return src_f32 ? (const void *)llrl_k_fp8_tma<true> : (const void *)llrl_k_fp8_tma<false>;
    }
    if (variant < 0 || variant >= kNumCastVariants)   // out of range: the default TMA variant
        return src_f32 ? (const void *)llrl_k_cast_tma<true, LLRL_TMA_A> : (const void *)llrl_k_cast_tma<false, LLRL_TMA_A>;
    return src_f32 ? kCastVariants[variant].f32 : kCastVariants[variant].bf16;
}

// Block size and dynamic shared memory of a launch (fp8 TMA: 256 workers + 1 producer warp).
static void launch_shape(int mode, int variant, bool src_f32, int *threads, size_t *smem) {
    *threads = kThreads;
    *smem = 0;
    if (mode == 0 && variant == kCastTmaVariant) {
        *threads = 64 + 512;
        *smem = size_t(4) * (32 * 1024 + 16 * 1024);
    }
    if (mode == 0 && variant == kCastTmaVariant + 1) {
        *threads = 64 + 256;
        *smem = size_t(4) * (16 * 1024 + 8 * 1024);
    }
    if (mode == 0 && variant == kCastTmaVariant + 2) {
        *threads = 64 + 256;
        *smem = size_t(4) * (32 * 1024 + 16 * 1024);
    }
    if (mode == 1 && variant != 0) {   // fp8 TMA variants (bf16 source): 1 = 3 stages x 2 CTAs/SM,
        *threads = kThreads + 32;      // 2 = 6 stages x 1 CTA/SM, 3 = 2 stages x 3 CTAs/SM
        const int st = src_f32 ? fp8_stages<true>() : variant == 2 ? 6 : variant == 3 ? 2 : fp8_stages<false>();
        *smem = size_t(st) * (src_f32 ? fp8_stage_bytes<true>() : fp8_stage_bytes<false>());
    }
}

static cudaError_t prepare(const void *fn, size_t smem) {
    if (smem == 0) return cudaSuccess;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

cudaError_t launch_sync(const KParams &P, int mode, int variant, bool src_f32, int grid, cudaStream_t stream) {
    const void *fn = kernel_for(mode, variant, src_f32);
    int threads;
    size_t smem;
    launch_shape(mode, variant, src_f32, &threads, &smem);
    void *args[] = {const_cast<KParams *>(&P)};
    if (!P.pdl_wait) return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, stream);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_nv_amax(const NvAmaxParams &P, bool src_f32, int grid, cudaStream_t stream) {
    constexpr int smem = kNvStages * kNvStageBytes;
    const void *fn = src_f32 ? (const void *)llrl_k_nv_amax<true> : (const void *)llrl_k_nv_amax<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (src_f32) llrl_k_nv_amax<true><<<grid, kThreads + 32, smem, stream>>>(P);
    else llrl_k_nv_amax<false><<<grid, kThreads + 32, smem, stream>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_nv_scale(const NvScaleParams &P, cudaStream_t stream) {
    llrl_k_nv_scale<<<1, kThreads, 0, stream>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_nv_fetch(const NvFetchParams &P, cudaStream_t stream) {
    llrl_k_nv_fetch<<<1, kThreads, 0, stream>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_nv_tscale(const NvTscaleParams &P, cudaStream_t stream) {
    const int grid = std::max(1, std::min(64, (P.n_local + kThreads - 1) / kThreads));
    llrl_k_nv_tscale<<<grid, kThreads, 0, stream>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_signal(const SignalTargets &t, cudaStream_t stream) {
    llrl_k_signal<<<1, 32, 0, stream>>>(t);
    return cudaGetLastError();
}

cudaError_t launch_wait(unsigned long long *flags, const WaitTargets &t, cudaStream_t stream) {
    llrl_k_wait<<<1, kNumSlots, 0, stream>>>(flags, t, 30ull * 1000 * 1000 * 1000);
    return cudaGetLastError();
}


cudaError_t sync_occupancy(int mode, int variant, bool src_f32, int *blocks_per_sm) {
    const void *fn = kernel_for(mode, variant, src_f32);
    int threads;
    size_t smem;
    launch_shape(mode, variant, src_f32, &threads, &smem);
    cudaError_t e = prepare(fn, smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, threads, smem);
}

int num_cast_variants() { return kNumCastVariants + 3; }   // + the three TMA variants

int cast_stage_bytes(int variant) {
    if (variant == kCastTmaVariant + 1) return 16 * 1024;   // LLRL_TMA_B
    return 32 * 1024;                                       // LLRL_TMA_A, LLRL_TMA_C
}

}  // namespace llrl
