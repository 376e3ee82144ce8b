/*
 * synth.c -- the seeded input generator of synth/__init__.py (weight_bits)
 * written in plain C, for filling full-size trainer buffers fast on the host.
 *
 * Holds NO arithmetic of the method (no re-layout, no cast, no quantisation):
 * it only turns (seed, param id, global row, global col) into a trainer weight
 * BIT PATTERN with integer operations.  Pinned bit
 * for bit against the numpy definition by tests/test_synth_cpu.py.  Shared by
 * the oracle side and the CUDA side of the tests (and bench.py's CPU legs);
 * includes nothing from oracle/ or from the product.
 */
#include <stdint.h>

static uint64_t mix(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

/* Trailing zeros of (t | 0x100), t = the low 8 hash bits: a geometric draw in [0, 8]. */
static uint64_t ctz8(uint64_t h)
{
    return (uint64_t)__builtin_ctzll((h & 0xFF) | 0x100);
}

/* Rows [r0, r1) x cols [c0, c1) of parameter `param` (global coordinates),
 * written row-major to out (uint32 patterns if f32, else uint16 bf16 patterns). */
void synth_fill(uint64_t seed, int64_t param, int is_norm, int f32,
                int64_t r0, int64_t r1, int64_t c0, int64_t c1, void *out)
{
    uint32_t *o32 = (uint32_t *)out;
    uint16_t *o16 = (uint16_t *)out;
    int64_t i = 0;
    uint64_t base = seed * 0x9E3779B97F4A7C15ull + (uint64_t)param * 0xD1B54A32D192ED03ull;
    for (int64_t r = r0; r < r1; r++) {
        uint64_t br = base + (uint64_t)r * 0xABC98388FB8FAC03ull;
        for (int64_t c = c0; c < c1; c++, i++) {
            uint64_t h = mix(br + (uint64_t)c * 0x8CB92BA72F3D8DD7ull);
            uint64_t sign = h >> 63, e = 127 - 6 - ctz8(h);
            if (f32)
                o32[i] = is_norm ? (uint32_t)(0x3F800000u | ((h >> 8) & 0x3FFFFu))
                                 : (uint32_t)((sign << 31) | (e << 23) | ((h >> 8) & 0x7FFFFFu));
            else
                o16[i] = is_norm ? (uint16_t)(0x3F80u | ((h >> 8) & 0x3u))
                                 : (uint16_t)((sign << 15) | (e << 7) | ((h >> 8) & 0x7Fu));
        }
    }
}
