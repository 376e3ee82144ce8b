// init.cu -- K0: synthetic trainer weights (harness support).
//
// Counter-based: the value of element (param, global row, col) depends only on
// (seed, param, row, col), so every trainer layout of a model holds the same
// full tensors.  Integer operations only; bit-identical to synth.weight_bits
// (pinned by tests/test_gpu_parity.py::test_fill_matches_synth).
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"

namespace llrl {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ uint64_t hash64(uint64_t seed, uint64_t param, uint64_t row, uint64_t col) {
    return mix64(seed * 0x9E3779B97F4A7C15ull + param * 0xD1B54A32D192ED03ull + row * 0xABC98388FB8FAC03ull +
                 col * 0x8CB92BA72F3D8DD7ull);
}

// Geometric draw in [0, 8]: trailing zeros of (t | 0x100), t = low 8 hash bits.
__device__ __forceinline__ uint32_t geo8(uint64_t h) { return __ffs(uint32_t(h & 0xFF) | 0x100u) - 1; }

__global__ void llrl_k_fill(char *base, const FillPiece *pieces, bool f32, uint64_t seed) {
    const FillPiece pc = pieces[blockIdx.y];
    const int64_t n = pc.rows * pc.cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / pc.cols, c = e - r * pc.cols;
        const uint64_t h = hash64(seed, uint64_t(pc.param), uint64_t(pc.r0 + r), uint64_t(pc.c0 + c));
        const uint64_t sign = h >> 63, exp = 127 - 6 - geo8(h);
        if (f32) {
            const uint32_t v = pc.is_norm ? uint32_t(0x3F800000u | ((h >> 8) & 0x3FFFFu))
                                          : uint32_t((sign << 31) | (exp << 23) | ((h >> 8) & 0x7FFFFFu));
            reinterpret_cast<uint32_t *>(base + pc.byte_off)[e] = v;
        } else {
            const uint16_t v = pc.is_norm ? uint16_t(0x3F80u | ((h >> 8) & 0x3u))
                                          : uint16_t((sign << 15) | (exp << 7) | ((h >> 8) & 0x7Fu));
            reinterpret_cast<uint16_t *>(base + pc.byte_off)[e] = v;
        }
    }
}

}  // namespace

cudaError_t launch_fill(void *base, const FillPiece *pieces_dev, int n_pieces, int64_t max_elems, bool f32,
                        uint64_t seed, cudaStream_t stream) {
    if (n_pieces == 0 || max_elems == 0) return cudaSuccess;
    int64_t bx = (max_elems + 255) / 256;
    if (bx > 4096) bx = 4096;
    for (int y0 = 0; y0 < n_pieces; y0 += 65535) {
        const int ny = n_pieces - y0 < 65535 ? n_pieces - y0 : 65535;
        llrl_k_fill<<<dim3(unsigned(bx), unsigned(ny)), 256, 0, stream>>>(static_cast<char *>(base), pieces_dev + y0,
                                                                         f32, seed);
    }
    return cudaGetLastError();
}

}  // namespace llrl
