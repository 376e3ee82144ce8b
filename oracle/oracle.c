/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the DDMA weight
 * synchronisation of LlamaRL (arxiv 2505.24034, §5.2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product path in
 * paper_2505_24034_b200/ and neither side includes the other.
 *
 * What it computes:
 *   for every parameter p:  full(p) = the unique tensor reassembled from the
 *   trainer shards ("each GPU only stores or updates its assigned
 *   shards"), and generator rank g receives its slice -- fused as QKV /
 *   gate_up -- of cast(full(p)) ("different parallelisms and data
 *   precision"; "quantization (fp8 or fp4) on the inference side").
 *   Post-condition: generator parameters byte-identical to the cast trainer
 *   parameters.
 *
 * Every convention the paper leaves open is a numbered DESIGN.md reading
 * (R1..R16); the comments below cite them.  Algorithm order:
 *   1. per layer, materialise each full parameter from all trainer shards,
 *      asserting replicas are bitwise equal and every element is covered;
 *   2. for each generator rank build its local (fused) tensors;
 *   3. cast: RNE bf16, identity f32, or 128x128-block fp8 e4m3;
 *   4. write into the generator rank's flat buffer, asserting every byte of
 *      it is written at most once.
 *
 * Parity pins (tests/test_oracle_pins.py): bf16 RNE vs ml_dtypes/torch over
 * all 2^32 patterns; e4m3 vs ml_dtypes; fp8 block vs numpy fp32 + ml_dtypes;
 * layout + sync vs an independent numpy/torch brute force (torch.chunk,
 * torch.cat) over the toy sweep; closed-form provenance; exactly-once
 * coverage.  No function of this file is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_E_INVALID -1
#define ORC_E_INDIVISIBLE -2
#define ORC_E_MISMATCH -3     /* replicas of one element differ */
#define ORC_E_UNSUPPORTED -4
#define ORC_E_UNCOVERED -8    /* an element of full(p) is held by no trainer rank */
#define ORC_E_OVERLAP -9      /* a generator byte would be written twice */
#define ORC_E_NOMEM -7

enum { ORC_F32 = 0, ORC_BF16 = 1, ORC_FP8 = 2, ORC_MXFP8 = 3, ORC_MXFP4 = 4, ORC_NVFP4 = 5 };

typedef struct {
    int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ffn, vocab, with_embed;
} orc_model;

typedef struct {
    int32_t fsdp, tp_train, tp_gen, src_dtype, dst_dtype, fsdp_inner;
    int32_t dp_gen;             /* generator data-parallel replicas (R12) */
    int32_t pp_train, pp_gen;   /* pipeline stages on each side (R14) */
} orc_cfg;
/* Rank numbering (R3, R12, R14): trainer rank = stage*(fsdp*tp_train) + mesh
 * rank; generator rank q = d*(pp_gen*tp_gen) + stage*tp_gen + g. */

/* ------------------------------------------------------------------------ */
/* Scalar casts                                                              */
/* ------------------------------------------------------------------------ */

/* fp32 -> bf16, IEEE round-to-nearest-even on the bit pattern (R6): keep the
 * upper 16 bits, round up when the dropped 16 bits exceed half an ulp, or
 * equal half an ulp and the kept part is odd.  A carry out of the mantissa
 * moves to the next binade (or to Inf) as the definition requires.
 * Subnormals are rounded like any other value (no flush).  NaN: quiet NaN
 * with the sign kept; the payload is unspecified (R6), tests compare NaN as a
 * class. */
uint16_t orc_bf16_rne(uint32_t b)
{
    if ((b & 0x7FFFFFFFu) > 0x7F800000u)
        return (uint16_t)((b >> 16) | 0x0040u);
    uint32_t upper = b >> 16;
    uint32_t dropped = b & 0xFFFFu;
    if (dropped > 0x8000u || (dropped == 0x8000u && (upper & 1u)))
        upper += 1;
    return (uint16_t)upper;
}

/* fp32 -> fp8 E4M3FN (bias 7, max 448, no Inf, NaN = S.1111.111), round to
 * nearest even, saturating to +-448 (PTX cvt.rn.satfinite semantics; R7).
 * Written from the format definition: find the quantum of the binade of |v|
 * (2^(e-3) for normals, 2^-9 for subnormals), round |v|/quantum to the
 * nearest integer (ties to even) and encode the rounded value. */
static uint8_t e4m3_encode(double a, uint8_t sign);

uint8_t orc_e4m3_rn_satfinite(float v)
{
    uint32_t vb;
    memcpy(&vb, &v, 4);
    uint8_t sign = (uint8_t)((vb >> 31) << 7);
    if (isnan(v))
        return (uint8_t)(sign | 0x7F);
    return e4m3_encode(fabs((double)v), sign);
}

/* |value| a (exact, double) -> E4M3FN code, RN-even, saturating. */
static uint8_t e4m3_encode(double a, uint8_t sign)
{
    if (a == 0.0)
        return sign;
    if (a > 448.0)
        return (uint8_t)(sign | 0x7E);           /* satfinite */
    double quantum;
    if (a < ldexp(1.0, -6)) {
        quantum = ldexp(1.0, -9);                /* subnormal grid m * 2^-9 */
    } else {
        int e;
        frexp(a, &e);                            /* a = f * 2^e, f in [0.5,1) */
        quantum = ldexp(1.0, (e - 1) - 3);       /* 3 mantissa bits */
    }
    double q = a / quantum;                      /* exact: power-of-two divide */
    double n = floor(q);
    double rem = q - n;
    if (rem > 0.5 || (rem == 0.5 && fmod(n, 2.0) != 0.0))
        n += 1.0;
    double r = n * quantum;                      /* rounded magnitude */
    if (r > 448.0)
        r = 448.0;                               /* satfinite */
    if (r == 0.0)
        return sign;
    if (r < ldexp(1.0, -6))
        return (uint8_t)(sign | (uint8_t)(r / ldexp(1.0, -9)));   /* exp field 0 */
    int e;
    double f = frexp(r, &e);                     /* r = f*2^e, f in [0.5,1) */
    int E = (e - 1) + 7;                         /* biased exponent */
    int m = (int)((f * 2.0 - 1.0) * 8.0);        /* exact: 3-bit mantissa */
    return (uint8_t)(sign | (uint8_t)(E << 3) | (uint8_t)m);
}

/* |value| a (exact, double) -> E2M1 (FP4: bias 1, 2 exponent bits, 1 mantissa
 * bit; magnitudes {0, 0.5, 1, 1.5, 2, 3, 4, 6}) code, RN-even, saturating at 6
 * (cvt.rn.satfinite.e2m1x2 semantics; R15).  sign is 0 or 8. */
static uint8_t e2m1_encode(double a, uint8_t sign)
{
    if (a == 0.0)
        return sign;
    if (a > 6.0)
        return (uint8_t)(sign | 0x7);
    double quantum;
    if (a < 1.0) {
        quantum = 0.5;                           /* subnormal grid m * 0.5 */
    } else {
        int e;
        frexp(a, &e);                            /* a = f * 2^e, f in [0.5,1) */
        quantum = ldexp(1.0, (e - 1) - 1);       /* 1 mantissa bit */
    }
    double q = a / quantum;
    double n = floor(q);
    double rem = q - n;
    if (rem > 0.5 || (rem == 0.5 && fmod(n, 2.0) != 0.0))
        n += 1.0;
    double r = n * quantum;
    if (r > 6.0)
        r = 6.0;
    if (r == 0.0)
        return sign;
    if (r < 1.0)
        return (uint8_t)(sign | 0x1);            /* 0.5: exponent field 0, mantissa 1 */
    int e;
    double f = frexp(r, &e);                     /* r = f*2^e */
    int E = (e - 1) + 1;                         /* biased exponent */
    int m = (int)((f * 2.0 - 1.0) * 2.0);        /* exact: 1-bit mantissa */
    return (uint8_t)(sign | (uint8_t)(E << 1) | (uint8_t)m);
}

uint8_t orc_e2m1_rn_satfinite(float v)
{
    uint32_t vb;
    memcpy(&vb, &v, 4);
    return e2m1_encode(fabs((double)v), (uint8_t)((vb >> 31) << 3));
}

void orc_e2m1_array(const float *in, int64_t n, uint8_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = orc_e2m1_rn_satfinite(in[i]);
}

/* One MXFP4 block (OCP MX v1.0 with E2M1 elements, reading R15): as
 * orc_mx_block with emax_elem = 2 (E2M1's largest exponent): X =
 * floor(log2 amax) - 2 clamped below at -127; q = e2m1_rn_satfinite(v / 2^X)
 * (exact quotient, one rounding); one code per output byte (the caller packs
 * two per byte, even element in the low nibble). */
void orc_mx4_block(const float *x, int64_t n, uint8_t *q, uint8_t *scale)
{
    float amax = 0.0f;
    for (int64_t i = 0; i < n; i++)
        if (fabsf(x[i]) > amax)
            amax = fabsf(x[i]);
    int X = -127;
    if (amax > 0.0f) {
        int e;
        frexp((double)amax, &e);
        X = (e - 1) - 2;
        if (X < -127)
            X = -127;
    }
    for (int64_t i = 0; i < n; i++) {
        uint32_t vb;
        memcpy(&vb, &x[i], 4);
        q[i] = e2m1_encode(fabs(ldexp((double)x[i], -X)), (uint8_t)((vb >> 31) << 3));
    }
    *scale = (uint8_t)(X + 127);
}

/* E4M3FN code -> its exact value (used to decode NVFP4 block scales). */
static double e4m3_decode(uint8_t code)
{
    int sign = code >> 7, E = (code >> 3) & 0xF, m = code & 0x7;
    double v = E == 0 ? ldexp((double)m, -9) : ldexp(1.0 + m / 8.0, E - 7);
    return sign ? -v : v;
}

/* NVFP4 (reading R16): E2M1 elements in 1x16 row groups with an E4M3 scale per
 * group and one fp32 scale per generator tensor.  Per tensor: amax_t over the
 * whole generator-local tensor, A = max(amax_t, 2^-64), S_enc = 2688 / A,
 * S_dec = A / 2688 (fp32 RN; 2688 = 448 * 6).  Per group: s = (amax_g / 6) *
 * S_enc (two fp32 RN operations), its E4M3 code sb = e4m3_rn_satfinite(s) and
 * decoded value s_q; r = S_enc / s_q (fp32 RN; r = 0 when s_q = 0); element
 * q = e2m1_rn_satfinite(x * r) (fp32 RN product).  Stored: packed codes, the
 * group scale codes, S_dec. */
float orc_nv_tensor_scales(const float *x, int64_t n, float *s_enc)
{
    float amax = 0.0f;
    for (int64_t i = 0; i < n; i++)
        if (fabsf(x[i]) > amax)
            amax = fabsf(x[i]);
    const float A = amax > 0x1p-64f ? amax : 0x1p-64f;
    volatile float enc = 2688.0f / A;
    volatile float dec = A / 2688.0f;
    *s_enc = enc;
    return dec;
}

void orc_nv_group(const float *x, int64_t n, float s_enc, uint8_t *q, uint8_t *scale)
{
    float amax = 0.0f;
    for (int64_t i = 0; i < n; i++)
        if (fabsf(x[i]) > amax)
            amax = fabsf(x[i]);
    volatile float t = amax / 6.0f;
    volatile float sv = t * s_enc;
    const uint8_t code = orc_e4m3_rn_satfinite(sv);
    const float sq = (float)e4m3_decode(code);     /* exact: e4m3 values are fp32-representable */
    volatile float r = sq == 0.0f ? 0.0f : s_enc / sq;
    for (int64_t i = 0; i < n; i++) {
        volatile float y = x[i] * r;
        q[i] = orc_e2m1_rn_satfinite(y);
    }
    *scale = code;
}

/* One MXFP8 block (OCP Microscaling Formats v1.0, E4M3 elements; DESIGN.md
 * reading R13): n <= 32 consecutive elements of one row share the scale
 * X = 2^(floor(log2(amax)) - emax_elem) with emax_elem = 8 (E4M3), the shared
 * exponent clamped below at -127 (E8M0's smallest value; amax = 0 gives -127);
 * each element is q = e4m3_rn_satfinite(v / X), the quotient taken exactly
 * (one rounding).  The scale byte is the E8M0 code (shared exponent + 127). */
void orc_mx_block(const float *x, int64_t n, uint8_t *q, uint8_t *scale)
{
    float amax = 0.0f;
    for (int64_t i = 0; i < n; i++)
        if (fabsf(x[i]) > amax)
            amax = fabsf(x[i]);
    int X = -127;
    if (amax > 0.0f) {
        int e;
        frexp((double)amax, &e);                 /* amax = f * 2^e, f in [0.5, 1) */
        X = (e - 1) - 8;                         /* floor(log2(amax)) - emax_elem */
        if (X < -127)
            X = -127;
    }
    for (int64_t i = 0; i < n; i++) {
        uint32_t vb;
        memcpy(&vb, &x[i], 4);
        q[i] = e4m3_encode(fabs(ldexp((double)x[i], -X)), (uint8_t)((vb >> 31) << 7));
    }
    *scale = (uint8_t)(X + 127);
}

/* Vectorised wrappers for the exhaustive pins. */
void orc_bf16_rne_array(const uint32_t *in, int64_t n, uint16_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = orc_bf16_rne(in[i]);
}

void orc_e4m3_array(const float *in, int64_t n, uint8_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = orc_e4m3_rn_satfinite(in[i]);
}

/* One fp8 block (reading R7): amax of |x| over the block,
 * amax_c = max(amax, 2^-64), inv = 448/amax_c and scale = amax_c/448 in fp32
 * round-to-nearest, q = e4m3_rn_satfinite(x * inv) with an fp32 RN product.
 * Compiled with -ffp-contract=off: no fused operations. */
void orc_fp8_block(const float *x, int64_t rows, int64_t cols, int64_t ld,
                   uint8_t *q, int64_t qld, float *scale)
{
    float amax = 0.0f;
    for (int64_t r = 0; r < rows; r++)
        for (int64_t c = 0; c < cols; c++) {
            float a = fabsf(x[r * ld + c]);
            if (a > amax)
                amax = a;
        }
    const float floor_amax = 0x1p-64f;
    float amax_c = amax > floor_amax ? amax : floor_amax;
    volatile float inv = 448.0f / amax_c;
    volatile float sc = amax_c / 448.0f;
    for (int64_t r = 0; r < rows; r++)
        for (int64_t c = 0; c < cols; c++) {
            volatile float y = x[r * ld + c] * inv;
            q[r * qld + c] = orc_e4m3_rn_satfinite(y);
        }
    *scale = sc;
}

/* ------------------------------------------------------------------------ */
/* Parameters                                                                */
/* ------------------------------------------------------------------------ */

/* Trainer-side (source) parameter list, canonical order (R0):
 *   [embed] ; per layer: attn_norm q k v o mlp_norm gate up down ; [final_norm lm_head]
 * Shapes W[out, in] (Llama-3.1 [ext]); norms are [d, 1].
 * kind: 0 = column-parallel (split rows: q k v gate up embed lm_head),
 *       1 = row-parallel (split columns: o down), 2 = norm (replicated). */
enum { SLOT_ATTN_NORM, SLOT_Q, SLOT_K, SLOT_V, SLOT_O, SLOT_MLP_NORM,
       SLOT_GATE, SLOT_UP, SLOT_DOWN, SLOT_EMBED, SLOT_FINAL_NORM, SLOT_LM_HEAD };
enum { KIND_COL = 0, KIND_ROW = 1, KIND_NORM = 2 };

int orc_num_src_params(const orc_model *m)
{
    return 9 * m->n_layers + (m->with_embed ? 3 : 0);
}

static void slot_shape(const orc_model *m, int slot, int64_t *rows, int64_t *cols, int *kind)
{
    int64_t d = m->d_model, qd = (int64_t)m->n_heads * m->head_dim;
    int64_t kvd = (int64_t)m->n_kv_heads * m->head_dim, f = m->d_ffn, V = m->vocab;
    switch (slot) {
    case SLOT_ATTN_NORM: case SLOT_MLP_NORM: case SLOT_FINAL_NORM:
        *rows = d; *cols = 1; *kind = KIND_NORM; break;
    case SLOT_Q: *rows = qd; *cols = d; *kind = KIND_COL; break;
    case SLOT_K: case SLOT_V: *rows = kvd; *cols = d; *kind = KIND_COL; break;
    case SLOT_O: *rows = d; *cols = qd; *kind = KIND_ROW; break;
    case SLOT_GATE: case SLOT_UP: *rows = f; *cols = d; *kind = KIND_COL; break;
    case SLOT_DOWN: *rows = d; *cols = f; *kind = KIND_ROW; break;
    case SLOT_EMBED: case SLOT_LM_HEAD: *rows = V; *cols = d; *kind = KIND_COL; break;
    default: *rows = 0; *cols = 0; *kind = -1;
    }
}

/* src param id -> (slot, layer); layer -1 for embed/final_norm/lm_head. */
static int src_param_slot(const orc_model *m, int p, int *layer)
{
    int P = orc_num_src_params(m);
    if (p < 0 || p >= P)
        return -1;
    if (m->with_embed) {
        if (p == 0) { *layer = -1; return SLOT_EMBED; }
        if (p == P - 2) { *layer = -1; return SLOT_FINAL_NORM; }
        if (p == P - 1) { *layer = -1; return SLOT_LM_HEAD; }
        p -= 1;
    }
    *layer = p / 9;
    return p % 9;
}

static int layer_slot_to_src_param(const orc_model *m, int layer, int slot)
{
    int base = m->with_embed ? 1 : 0;
    if (slot == SLOT_EMBED) return 0;
    if (slot == SLOT_FINAL_NORM) return orc_num_src_params(m) - 2;
    if (slot == SLOT_LM_HEAD) return orc_num_src_params(m) - 1;
    return base + 9 * layer + slot;
}

/* R14: decoder layers split evenly and contiguously over pp stages; embed
 * lives on the first stage, final_norm and lm_head on the last. */
static int layer_stage(const orc_model *m, int layer, int first_or_last, int pp)
{
    if (layer >= 0)
        return layer / (m->n_layers / pp);
    return first_or_last ? pp - 1 : 0;
}

static int src_param_stage(const orc_model *m, int p, int pp)
{
    int layer = -1, slot = src_param_slot(m, p, &layer);
    return layer_stage(m, layer, slot != SLOT_EMBED, pp);
}

int orc_src_param_info(const orc_model *m, int p, int64_t *rows, int64_t *cols, int *kind)
{
    int layer, slot = src_param_slot(m, p, &layer);
    if (slot < 0)
        return ORC_E_INVALID;
    slot_shape(m, slot, rows, cols, kind);
    return ORC_OK;
}

static int64_t dtype_size(int dt)
{
    return dt == ORC_F32 ? 4 : dt == ORC_BF16 ? 2 : 1;
}

static int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

static int check_model(const orc_model *m, const orc_cfg *c)
{
    if (m->n_layers < 0 || m->d_model <= 0 || m->n_heads <= 0 || m->n_kv_heads <= 0 ||
        m->head_dim <= 0 || m->d_ffn <= 0 || (m->with_embed && m->vocab <= 0))
        return ORC_E_INVALID;
    if (c->fsdp <= 0 || c->tp_train <= 0 || c->tp_gen <= 0 || c->dp_gen <= 0 ||
        c->pp_train <= 0 || c->pp_gen <= 0)
        return ORC_E_INVALID;
    /* R14: whole layers per stage */
    if (m->n_layers % c->pp_train || m->n_layers % c->pp_gen)
        return ORC_E_INDIVISIBLE;
    if (c->src_dtype != ORC_F32 && c->src_dtype != ORC_BF16)
        return ORC_E_UNSUPPORTED;
    if (c->dst_dtype < ORC_F32 || c->dst_dtype > ORC_NVFP4)
        return ORC_E_UNSUPPORTED;
    if (c->dst_dtype == ORC_F32 && c->src_dtype != ORC_F32)
        return ORC_E_UNSUPPORTED;
    /* R1: trainer TP splits evenly (rows of column-parallel, columns of row-parallel) */
    int P = orc_num_src_params(m);
    for (int p = 0; p < P; p++) {
        int64_t R, C; int kind;
        orc_src_param_info(m, p, &R, &C, &kind);
        if (kind == KIND_COL && R % c->tp_train) return ORC_E_INDIVISIBLE;
        if (kind == KIND_ROW && C % c->tp_train) return ORC_E_INDIVISIBLE;
    }
    /* R4: generator TP -- whole query heads, whole or replicated KV heads, even ffn / vocab */
    int T = c->tp_gen;
    if (m->n_heads % T) return ORC_E_INDIVISIBLE;
    if (m->n_kv_heads % T && T % m->n_kv_heads) return ORC_E_INDIVISIBLE;
    if (m->d_ffn % T) return ORC_E_INDIVISIBLE;
    if (m->with_embed && m->vocab % T) return ORC_E_INDIVISIBLE;
    /* R15: MXFP4 packs two elements per byte: every quantised generator tensor has
     * an even number of columns (and, for whole 1x32 groups, a multiple of 32);
     * R16 likewise with 1x16 groups.  Checked after the divisibility rules
     * (DESIGN R21: these rules are stated on the generator-local column counts,
     * which exist only once the split divides; a layout that violates both
     * reports INDIVISIBLE). */
    if (c->dst_dtype == ORC_MXFP4 && (m->d_model % 32 || (m->n_heads * m->head_dim / c->tp_gen) % 32 ||
                                      (m->d_ffn / c->tp_gen) % 32))
        return ORC_E_UNSUPPORTED;
    if (c->dst_dtype == ORC_NVFP4 && (m->d_model % 16 || (m->n_heads * m->head_dim / c->tp_gen) % 16 ||
                                      (m->d_ffn / c->tp_gen) % 16))
        return ORC_E_UNSUPPORTED;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Trainer layout (R1 Megatron TP, R2 FSDP2 Shard(0) torch.chunk, R3 mesh)   */
/* ------------------------------------------------------------------------ */

/* Rectangle [r0,r1) x [c0,c1) of full(p) that trainer rank `rank` holds. */
static void src_rect(const orc_model *m, const orc_cfg *c, int rank, int p,
                     int64_t *r0, int64_t *r1, int64_t *c0, int64_t *c1)
{
    int F = c->fsdp, Tt = c->tp_train;
    int stage = rank / (F * Tt);
    rank %= F * Tt;
    int f, t;
    if (c->fsdp_inner) { t = rank / F; f = rank % F; }   /* rank = t*F + f */
    else               { f = rank / Tt; t = rank % Tt; } /* rank = f*Tt + t (default) */
    int64_t R, C; int kind;
    orc_src_param_info(m, p, &R, &C, &kind);
    if (src_param_stage(m, p, c->pp_train) != stage) {   /* R14: not on this stage */
        *r0 = *r1 = *c0 = *c1 = 0;
        return;
    }
    /* TP-local shard */
    int64_t tr0 = 0, tr1 = R, tc0 = 0, tc1 = C;
    if (kind == KIND_COL) { tr0 = t * (R / Tt); tr1 = tr0 + R / Tt; }
    if (kind == KIND_ROW) { tc0 = t * (C / Tt); tc1 = tc0 + C / Tt; }
    /* FSDP: torch.chunk(dim 0) of the TP-local shard: chunk = ceil(rows / F) */
    int64_t lrows = tr1 - tr0;
    int64_t chunk = (lrows + F - 1) / F;
    int64_t a = (int64_t)f * chunk, b = a + chunk;
    if (a > lrows) a = lrows;
    if (b > lrows) b = lrows;
    *r0 = tr0 + a; *r1 = tr0 + b; *c0 = tc0; *c1 = tc1;
}

/* Byte offset of param p's piece in trainer rank `rank`'s flat buffer: pieces
 * in canonical order, each starting at a 256-byte boundary (R0). */
int64_t orc_src_piece(const orc_model *m, const orc_cfg *c, int rank, int p,
                      int64_t *r0, int64_t *r1, int64_t *c0, int64_t *c1)
{
    int64_t es = dtype_size(c->src_dtype), off = 0;
    for (int q = 0; q <= p; q++) {
        int64_t a0, a1, b0, b1;
        src_rect(m, c, rank, q, &a0, &a1, &b0, &b1);
        off = align256(off);
        if (q == p) {
            *r0 = a0; *r1 = a1; *c0 = b0; *c1 = b1;
            return off;
        }
        off += (a1 - a0) * (b1 - b0) * es;
    }
    return -1;
}

int64_t orc_src_rank_bytes(const orc_model *m, const orc_cfg *c, int rank)
{
    int P = orc_num_src_params(m);
    if (P == 0)
        return 0;
    int64_t r0, r1, c0, c1;
    int64_t off = orc_src_piece(m, c, rank, P - 1, &r0, &r1, &c0, &c1);
    return align256(off + (r1 - r0) * (c1 - c0) * dtype_size(c->src_dtype));
}

/* ------------------------------------------------------------------------ */
/* Generator layout (R4 vLLM-style fused packing, R7 fp8, R9 scale placement) */
/* ------------------------------------------------------------------------ */

/* Generator parameter list, canonical order:
 *   [embed] ; per layer: attn_norm qkv o mlp_norm gate_up down ; [final_norm lm_head] */
enum { G_ATTN_NORM, G_QKV, G_O, G_MLP_NORM, G_GATE_UP, G_DOWN, G_EMBED, G_FINAL_NORM, G_LM_HEAD };

int orc_num_dst_params(const orc_model *m)
{
    return 6 * m->n_layers + (m->with_embed ? 3 : 0);
}

static int dst_param_slot(const orc_model *m, int gp, int *layer)
{
    int P = orc_num_dst_params(m);
    if (gp < 0 || gp >= P)
        return -1;
    if (m->with_embed) {
        if (gp == 0) { *layer = -1; return G_EMBED; }
        if (gp == P - 2) { *layer = -1; return G_FINAL_NORM; }
        if (gp == P - 1) { *layer = -1; return G_LM_HEAD; }
        gp -= 1;
    }
    *layer = gp / 6;
    return gp % 6;
}

/* A part: rows [fr0, fr0+nr) x cols [fc0, fc0+nc) of full(src_param), placed
 * at local rows [lr0, lr0+nr), cols [0, nc) of the generator tensor. */
typedef struct { int src_param; int64_t fr0, fc0, nr, nc, lr0; } part_t;

/* Local shape of generator param gp on rank g and its parts (<= 3). */
static int dst_parts(const orc_model *m, const orc_cfg *c, int g, int stage, int gp,
                     int64_t *rows, int64_t *cols, int *quant, part_t *parts)
{
    int T = c->tp_gen, layer, gs = dst_param_slot(m, gp, &layer);
    int64_t d = m->d_model, hd = m->head_dim;
    int64_t qrows = (int64_t)m->n_heads * hd / T;
    int n = 0;
    *quant = 0;
    switch (gs) {
    case G_ATTN_NORM: case G_MLP_NORM: case G_FINAL_NORM: {
        int slot = gs == G_ATTN_NORM ? SLOT_ATTN_NORM : gs == G_MLP_NORM ? SLOT_MLP_NORM : SLOT_FINAL_NORM;
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, slot), 0, 0, d, 1, 0};
        *rows = d; *cols = 1;
        break;
    }
    case G_QKV: {
        /* q rows [g*qrows, (g+1)*qrows); k and v: KV % T == 0 -> rows
         * [g*kvrows, ...); T > KV -> whole head g / (T/KV) (replicated). */
        int64_t kvrows, kv0;
        if (m->n_kv_heads % T == 0) {
            kvrows = (int64_t)m->n_kv_heads * hd / T;
            kv0 = g * kvrows;
        } else {
            kvrows = hd;
            kv0 = (int64_t)(g / (T / m->n_kv_heads)) * hd;
        }
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_Q), g * qrows, 0, qrows, d, 0};
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_K), kv0, 0, kvrows, d, qrows};
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_V), kv0, 0, kvrows, d, qrows + kvrows};
        *rows = qrows + 2 * kvrows; *cols = d; *quant = 1;
        break;
    }
    case G_O: {
        int64_t oc = (int64_t)m->n_heads * hd / T;
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_O), 0, g * oc, d, oc, 0};
        *rows = d; *cols = oc; *quant = 1;
        break;
    }
    case G_GATE_UP: {
        int64_t fr = m->d_ffn / T;
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_GATE), g * fr, 0, fr, d, 0};
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_UP), g * fr, 0, fr, d, fr};
        *rows = 2 * fr; *cols = d; *quant = 1;
        break;
    }
    case G_DOWN: {
        int64_t fc = m->d_ffn / T;
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, SLOT_DOWN), 0, g * fc, d, fc, 0};
        *rows = d; *cols = fc; *quant = 1;
        break;
    }
    case G_EMBED: case G_LM_HEAD: {
        int64_t vr = m->vocab / T;
        int slot = gs == G_EMBED ? SLOT_EMBED : SLOT_LM_HEAD;
        parts[n++] = (part_t){layer_slot_to_src_param(m, layer, slot), g * vr, 0, vr, d, 0};
        *rows = vr; *cols = d;
        break;
    }
    default:
        return -1;
    }
    if (c->dst_dtype != ORC_FP8 && c->dst_dtype != ORC_MXFP8 && c->dst_dtype != ORC_MXFP4 &&
        c->dst_dtype != ORC_NVFP4)
        *quant = 0;
    if (stage >= 0 && layer_stage(m, layer, gs != G_EMBED, c->pp_gen) != stage) {
        *rows = 0; *cols = 0;          /* R14: not on this generator stage */
        return 0;
    }
    return n;
}

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* Bytes of a generator tensor's data: fp32 4, bf16 2, fp8 / MXFP8 1 per
 * element; MXFP4 two elements per byte (R15; C even). */
static int64_t data_bytes(const orc_cfg *c, int64_t R, int64_t C, int qt)
{
    if (qt)
        return (c->dst_dtype == ORC_MXFP4 || c->dst_dtype == ORC_NVFP4) ? R * C / 2 : R * C;
    return R * C * (c->dst_dtype == ORC_F32 ? 4 : 2);
}

/* Bytes of a quantised weight's scale grid (R9, R13): fp8 blocks: fp32
 * [ceil(R/128), ceil(C/128)]; MXFP8: E8M0 bytes [R, ceil(C/32)]. */
static int64_t scale_grid_bytes(const orc_cfg *c, int64_t R, int64_t C)
{
    if (c->dst_dtype == ORC_MXFP8 || c->dst_dtype == ORC_MXFP4)
        return R * cdiv(C, 32);
    if (c->dst_dtype == ORC_NVFP4)
        return R * cdiv(C, 16);
    return cdiv(R, 128) * cdiv(C, 128) * 4;
}

/* Byte offsets of generator param gp on rank g (R0, R9): params in canonical
 * order at 256-byte boundaries; a quantised weight's fp32 scale grid
 * [ceil(R/128), ceil(C/128)] follows it at the next 256-byte boundary. */
int orc_dst_param(const orc_model *m, const orc_cfg *c, int g, int gp,
                  int64_t *rows, int64_t *cols, int *quant,
                  int64_t *byte_off, int64_t *scale_off)
{
    /* R12 / R14: generator rank -> (TP rank, pipeline stage); replicas repeat */
    int stage = (g / c->tp_gen) % c->pp_gen;
    g %= c->tp_gen;
    int64_t off = 0;
    for (int q = 0; q <= gp; q++) {
        part_t parts[3];
        int64_t R, C; int qt;
        if (dst_parts(m, c, g, stage, q, &R, &C, &qt, parts) < 0)
            return ORC_E_INVALID;
        off = align256(off);
        int64_t data_off = off;
        off += data_bytes(c, R, C, qt);
        int64_t s_off = -1;
        if (qt) {
            off = align256(off);
            s_off = off;
            off += scale_grid_bytes(c, R, C);
            if (c->dst_dtype == ORC_NVFP4) {   /* R16: fp32 tensor scale at the next 256-byte boundary */
                off = align256(off);
                off += 4;
            }
        }
        if (q == gp) {
            *rows = R; *cols = C; *quant = qt; *byte_off = data_off; *scale_off = s_off;
            return ORC_OK;
        }
    }
    return ORC_E_INVALID;
}

int64_t orc_dst_rank_bytes(const orc_model *m, const orc_cfg *c, int g)
{
    int P = orc_num_dst_params(m);
    if (P == 0)
        return 0;
    int64_t R, C, off, soff; int qt;
    orc_dst_param(m, c, g, P - 1, &R, &C, &qt, &off, &soff);
    int64_t end = off + data_bytes(c, R, C, qt);
    if (qt)
        end = soff + scale_grid_bytes(c, R, C);
    if (qt && c->dst_dtype == ORC_NVFP4)
        end = align256(end) + 4;
    return align256(end);
}

/* R16: byte offset of an NVFP4 tensor's fp32 scale (-1 if none). */
int64_t orc_dst_tensor_scale_off(const orc_model *m, const orc_cfg *c, int g, int gp)
{
    int64_t R, C, off, soff; int qt;
    if (orc_dst_param(m, c, g, gp, &R, &C, &qt, &off, &soff) || !qt || c->dst_dtype != ORC_NVFP4)
        return -1;
    return align256(soff + scale_grid_bytes(c, R, C));
}

/* For point checks at full size: generator element (g, gp, lr, lc) comes
 * from element (row, col) of source param *src_param. */
int orc_dst_element_source(const orc_model *m, const orc_cfg *c, int g, int gp,
                           int64_t lr, int64_t lc, int *src_param, int64_t *row, int64_t *col)
{
    int stage = (g / c->tp_gen) % c->pp_gen;
    g %= c->tp_gen;
    part_t parts[3];
    int64_t R, C; int qt;
    int n = dst_parts(m, c, g, stage, gp, &R, &C, &qt, parts);
    if (n < 0 || lr < 0 || lr >= R || lc < 0 || lc >= C)
        return ORC_E_INVALID;
    for (int i = 0; i < n; i++)
        if (lr >= parts[i].lr0 && lr < parts[i].lr0 + parts[i].nr) {
            *src_param = parts[i].src_param;
            *row = parts[i].fr0 + (lr - parts[i].lr0);
            *col = parts[i].fc0 + lc;
            return ORC_OK;
        }
    return ORC_E_INVALID;
}

/* orc_dst_element_source for every element of generator param gp on rank g,
 * row-major (R*C entries in each output array).  A plain loop, for the
 * exhaustive pin in tests/test_oracle_pins.py. */
int orc_dst_param_sources(const orc_model *m, const orc_cfg *c, int g, int gp,
                          int32_t *src_param, int64_t *row, int64_t *col)
{
    int64_t R, C, off, soff; int qt;
    int rc = orc_dst_param(m, c, g, gp, &R, &C, &qt, &off, &soff);
    if (rc)
        return rc;
    for (int64_t lr = 0; lr < R; lr++)
        for (int64_t lc = 0; lc < C; lc++) {
            int p;
            int64_t i = lr * C + lc;
            if ((rc = orc_dst_element_source(m, c, g, gp, lr, lc, &p, &row[i], &col[i])))
                return rc;
            src_param[i] = p;
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* The sync                                                                  */
/* ------------------------------------------------------------------------ */

static float load_src(const void *buf, int dt, int64_t i, uint32_t *bits)
{
    float v;
    if (dt == ORC_F32) {
        memcpy(bits, (const uint8_t *)buf + 4 * i, 4);
    } else {
        uint16_t h;
        memcpy(&h, (const uint8_t *)buf + 2 * i, 2);
        *bits = (uint32_t)h << 16;              /* bf16 widens exactly */
    }
    memcpy(&v, bits, 4);
    return v;
}

/* Step 1: materialise full(p) from every trainer rank. */
static int materialise(const orc_model *m, const orc_cfg *c, const void *const *src,
                       int p, float **out)
{
    int64_t R, C; int kind;
    orc_src_param_info(m, p, &R, &C, &kind);
    float *full = (float *)malloc((size_t)(R * C > 0 ? R * C : 1) * sizeof(float));
    uint8_t *seen = (uint8_t *)calloc((size_t)(R * C > 0 ? R * C : 1), 1);
    if (!full || !seen) { free(full); free(seen); return ORC_E_NOMEM; }
    int nsrc = c->fsdp * c->tp_train * c->pp_train;
    for (int s = 0; s < nsrc; s++) {
        int64_t r0, r1, c0, c1;
        int64_t off = orc_src_piece(m, c, s, p, &r0, &r1, &c0, &c1);
        int64_t lc = c1 - c0;
        const uint8_t *base = (const uint8_t *)src[s] + off;
        for (int64_t r = r0; r < r1; r++)
            for (int64_t col = c0; col < c1; col++) {
                uint32_t bits;
                float v = load_src(base, c->src_dtype, (r - r0) * lc + (col - c0), &bits);
                int64_t i = r * C + col;
                if (seen[i]) {
                    uint32_t prev;
                    memcpy(&prev, &full[i], 4);
                    if (prev != bits) { free(full); free(seen); return ORC_E_MISMATCH; }
                } else {
                    full[i] = v;
                    seen[i] = 1;
                }
            }
    }
    for (int64_t i = 0; i < R * C; i++)
        if (!seen[i]) { free(full); free(seen); return ORC_E_UNCOVERED; }
    free(seen);
    *out = full;
    return ORC_OK;
}

static int mark_written(uint8_t *written, int64_t off, int64_t nbytes)
{
    for (int64_t i = off; i < off + nbytes; i++) {
        if (written[i])
            return ORC_E_OVERLAP;
        written[i] = 1;
    }
    return ORC_OK;
}

/* Steps 2-4 for one generator param on rank g, given full tensors of its sources. */
static int write_dst_param(const orc_model *m, const orc_cfg *c, int g, int gp,
                           float *const *full_by_src, uint8_t *dst, uint8_t *written)
{
    part_t parts[3];
    int64_t R, C, off, soff; int qt;
    int n = dst_parts(m, c, g % c->tp_gen, (g / c->tp_gen) % c->pp_gen, gp, &R, &C, &qt, parts);
    orc_dst_param(m, c, g, gp, &R, &C, &qt, &off, &soff);
    /* Step 2: the generator-local (fused) tensor */
    float *local = (float *)malloc((size_t)(R * C > 0 ? R * C : 1) * sizeof(float));
    if (!local)
        return ORC_E_NOMEM;
    for (int i = 0; i < n; i++) {
        int64_t fullC, fullR; int kind;
        orc_src_param_info(m, parts[i].src_param, &fullR, &fullC, &kind);
        const float *full = full_by_src[parts[i].src_param];
        for (int64_t r = 0; r < parts[i].nr; r++)
            for (int64_t col = 0; col < parts[i].nc; col++)
                local[(parts[i].lr0 + r) * C + col] = full[(parts[i].fr0 + r) * fullC + parts[i].fc0 + col];
    }
    /* Step 3-4: cast and store */
    int rc = ORC_OK;
    if (qt && c->dst_dtype == ORC_NVFP4) {
        int64_t nsc = cdiv(C, 16);
        int64_t ts = align256(soff + R * nsc);
        if ((rc = mark_written(written, off, R * C / 2)) || (rc = mark_written(written, soff, R * nsc)) ||
            (rc = mark_written(written, ts, 4)))
            goto out;
        float s_enc;
        float s_dec = orc_nv_tensor_scales(local, R * C, &s_enc);
        memcpy(dst + ts, &s_dec, 4);
        uint8_t codes[16];
        for (int64_t r = 0; r < R; r++)
            for (int64_t j = 0; j < nsc; j++) {
                int64_t n = C - j * 16 < 16 ? C - j * 16 : 16;
                orc_nv_group(local + r * C + j * 16, n, s_enc, codes, dst + soff + r * nsc + j);
                for (int64_t k = 0; k < n; k += 2)   /* even element -> low nibble */
                    dst[off + (r * C + j * 16 + k) / 2] = (uint8_t)(codes[k] | (codes[k + 1] << 4));
            }
    } else if (qt && c->dst_dtype == ORC_MXFP4) {
        int64_t nsc = cdiv(C, 32);
        if ((rc = mark_written(written, off, R * C / 2)) || (rc = mark_written(written, soff, R * nsc)))
            goto out;
        uint8_t codes[32];
        for (int64_t r = 0; r < R; r++)
            for (int64_t j = 0; j < nsc; j++) {
                int64_t n = C - j * 32 < 32 ? C - j * 32 : 32;
                orc_mx4_block(local + r * C + j * 32, n, codes, dst + soff + r * nsc + j);
                for (int64_t k = 0; k < n; k += 2)   /* even element -> low nibble */
                    dst[off + (r * C + j * 32 + k) / 2] = (uint8_t)(codes[k] | (codes[k + 1] << 4));
            }
    } else if (qt && c->dst_dtype == ORC_MXFP8) {
        int64_t nsc = cdiv(C, 32);
        if ((rc = mark_written(written, off, R * C)) || (rc = mark_written(written, soff, R * nsc)))
            goto out;
        for (int64_t r = 0; r < R; r++)
            for (int64_t j = 0; j < nsc; j++) {
                int64_t n = C - j * 32 < 32 ? C - j * 32 : 32;
                orc_mx_block(local + r * C + j * 32, n, dst + off + r * C + j * 32, dst + soff + r * nsc + j);
            }
    } else if (qt) {
        int64_t nbr = cdiv(R, 128), nbc = cdiv(C, 128);
        if ((rc = mark_written(written, off, R * C)) || (rc = mark_written(written, soff, nbr * nbc * 4)))
            goto out;
        for (int64_t bi = 0; bi < nbr; bi++)
            for (int64_t bj = 0; bj < nbc; bj++) {
                int64_t br = R - bi * 128 < 128 ? R - bi * 128 : 128;
                int64_t bc = C - bj * 128 < 128 ? C - bj * 128 : 128;
                float s;
                orc_fp8_block(local + bi * 128 * C + bj * 128, br, bc, C,
                              dst + off + bi * 128 * C + bj * 128, C, &s);
                memcpy(dst + soff + (bi * nbc + bj) * 4, &s, 4);
            }
    } else if (c->dst_dtype == ORC_F32) {
        if ((rc = mark_written(written, off, R * C * 4)))
            goto out;
        memcpy(dst + off, local, (size_t)(R * C * 4));
    } else {
        if ((rc = mark_written(written, off, R * C * 2)))
            goto out;
        for (int64_t i = 0; i < R * C; i++) {
            uint32_t b;
            memcpy(&b, &local[i], 4);
            uint16_t h = orc_bf16_rne(b);
            memcpy(dst + off + 2 * i, &h, 2);
        }
    }
out:
    free(local);
    return rc;
}

/* The sync restricted to generator params [gp_begin, gp_end): src[s] =
 * trainer rank s's flat buffer, dst[g] = generator rank g's flat buffer (host
 * memory, sizes orc_*_rank_bytes).  Bytes of dst covered by no param
 * (alignment padding) are left untouched.  Walks the generator params in
 * order; materialises each source param on first use and frees it once the
 * generator param that consumes it is written (every source param feeds
 * exactly one generator param). */
int orc_sync_range(const orc_model *m, const orc_cfg *c, const void *const *src,
                   void *const *dst, int gp_begin, int gp_end)
{
    int rc = check_model(m, c);
    if (rc)
        return rc;
    int P = orc_num_src_params(m), ND = c->tp_gen * c->pp_gen * c->dp_gen;
    float **full = (float **)calloc((size_t)(P > 0 ? P : 1), sizeof(float *));
    uint8_t **written = (uint8_t **)calloc((size_t)ND, sizeof(uint8_t *));
    if (!full || !written) { free(full); free(written); return ORC_E_NOMEM; }
    for (int q = 0; q < ND; q++) {
        written[q] = (uint8_t *)calloc((size_t)orc_dst_rank_bytes(m, c, q) + 1, 1);
        if (!written[q]) { rc = ORC_E_NOMEM; goto done; }
    }
    for (int gp = gp_begin; gp < gp_end && rc == ORC_OK; gp++) {
        part_t parts[3];
        int64_t R, C; int qt;
        int n = dst_parts(m, c, 0, -1, gp, &R, &C, &qt, parts);
        for (int i = 0; i < n && rc == ORC_OK; i++)
            if (!full[parts[i].src_param])
                rc = materialise(m, c, src, parts[i].src_param, &full[parts[i].src_param]);
        for (int q = 0; q < ND && rc == ORC_OK; q++)   /* every stage rank / replica writes its own copy */
            rc = write_dst_param(m, c, q, gp, full, (uint8_t *)dst[q], written[q]);
        for (int i = 0; i < n; i++) {
            free(full[parts[i].src_param]);
            full[parts[i].src_param] = NULL;
        }
    }
done:
    for (int p = 0; p < P; p++)
        free(full[p]);
    for (int q = 0; q < ND; q++)
        free(written[q]);
    free(full);
    free(written);
    return rc;
}

/* The whole sync (all generator params). */
int orc_sync(const orc_model *m, const orc_cfg *c, const void *const *src, void *const *dst)
{
    return orc_sync_range(m, c, src, dst, 0, orc_num_dst_params(m));
}

int orc_check(const orc_model *m, const orc_cfg *c) { return check_model(m, c); }
