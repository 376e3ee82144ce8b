// layout.cpp -- step a1: trainer and generator layouts.
//
// PAPER.md §5.2: "each GPU only stores or updates its assigned shards,
// leveraging the same tensor and parallel groups used during training"
// trainer and generator "can use different parallelisms and data precision".
// The concrete conventions are DESIGN.md readings R0-R4, R7, R9.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "internal.h"

namespace llrl {

static thread_local char g_err[512];

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int64_t dtype_bytes(int dt) { return dt == LLRL_F32 ? 4 : dt == LLRL_BF16 ? 2 : 1; }

int64_t data_bytes(int dt, int64_t elems) {
    return (dt == LLRL_MXFP4 || dt == LLRL_NVFP4) ? elems / 2 : elems * dtype_bytes(dt);
}

// R9 / R13 / R15: fp8 blocks -> fp32 [ceil(R/128), ceil(C/128)]; MX -> E8M0 bytes [R, ceil(C/32)].
int64_t scale_grid_bytes(int dt, int64_t rows, int64_t cols) {
    if (dt == LLRL_MXFP8 || dt == LLRL_MXFP4) return rows * ((cols + kMxGroup - 1) / kMxGroup);
    if (dt == LLRL_NVFP4) return rows * ((cols + kNvGroup - 1) / kNvGroup);
    return ((rows + kFp8Block - 1) / kFp8Block) * ((cols + kFp8Block - 1) / kFp8Block) * 4;
}

static int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// R0: canonical source-parameter list.
std::vector<SrcParam> enumerate_src_params(const llrl_model &m) {
    const int64_t d = m.d_model, qd = int64_t(m.n_heads) * m.head_dim;
    const int64_t kvd = int64_t(m.n_kv_heads) * m.head_dim, f = m.d_ffn, V = m.vocab;
    std::vector<SrcParam> ps;
    auto add = [&](int kind, int layer, int64_t r, int64_t c, int split) {
        ps.push_back(SrcParam{kind, layer, r, c, split, split == 2});
    };
    if (m.with_embed) add(LLRL_P_EMBED, -1, V, d, 0);
    for (int l = 0; l < m.n_layers; l++) {
        add(LLRL_P_ATTN_NORM, l, d, 1, 2);
        add(LLRL_P_Q, l, qd, d, 0);
        add(LLRL_P_K, l, kvd, d, 0);
        add(LLRL_P_V, l, kvd, d, 0);
        add(LLRL_P_O, l, d, qd, 1);
        add(LLRL_P_MLP_NORM, l, d, 1, 2);
        add(LLRL_P_GATE, l, f, d, 0);
        add(LLRL_P_UP, l, f, d, 0);
        add(LLRL_P_DOWN, l, d, f, 1);
    }
    if (m.with_embed) {
        add(LLRL_P_FINAL_NORM, -1, d, 1, 2);
        add(LLRL_P_LM_HEAD, -1, V, d, 0);
    }
    return ps;
}

}  // namespace llrl

using namespace llrl;

namespace {

// Trainer rank -> (fsdp index, tp index), R3.
void mesh_coords(int rank, int fsdp, int tp, uint32_t flags, int *f, int *t) {
    if (flags & LLRL_MESH_FSDP_INNER) { *t = rank / fsdp; *f = rank % fsdp; }
    else { *f = rank / tp; *t = rank % tp; }
}

// R14: pipeline stage of a layer (-1: embed -> first stage; -2: head -> last).
int stage_of(const llrl_model &m, int kind, int layer, int pp) {
    if (layer >= 0) return layer / (m.n_layers / pp);
    return kind == LLRL_P_EMBED ? 0 : pp - 1;
}

// R1 then R2: Megatron TP rectangle, then torch.chunk of its rows over FSDP.
Rect trainer_rect(const SrcParam &p, int f, int t, int fsdp, int tp) {
    Rect r{0, p.rows, 0, p.cols};
    if (p.split == 0) { int64_t n = p.rows / tp; r.r0 = t * n; r.r1 = r.r0 + n; }
    if (p.split == 1) { int64_t n = p.cols / tp; r.c0 = t * n; r.c1 = r.c0 + n; }
    const int64_t lrows = r.rows();
    const int64_t chunk = (lrows + fsdp - 1) / fsdp;
    const int64_t a = std::min<int64_t>(int64_t(f) * chunk, lrows);
    const int64_t b = std::min<int64_t>(a + chunk, lrows);
    return Rect{r.r0 + a, r.r0 + b, r.c0, r.c1};
}

int find_src(const std::vector<SrcParam> &ps, int kind, int layer) {
    for (size_t i = 0; i < ps.size(); i++)
        if (ps[i].kind == kind && ps[i].layer == layer) return int(i);
    return -1;
}

llrl_status build_src(llrl_layout *L) {
    const auto &ps = L->src_params;
    for (const auto &p : ps) {
        if (p.split == 0 && p.rows % L->tp_train) return LLRL_E_INDIVISIBLE;
        if (p.split == 1 && p.cols % L->tp_train) return LLRL_E_INDIVISIBLE;
    }
    if (L->model.n_layers % L->pp_train) return LLRL_E_INDIVISIBLE;
    const int mesh = L->fsdp * L->tp_train;
    L->n_ranks = mesh * L->pp_train;
    const int64_t es = dtype_bytes(L->dtype);
    L->pieces.assign(L->n_ranks, {});
    L->rank_bytes.assign(L->n_ranks, 0);
    for (int r = 0; r < L->n_ranks; r++) {
        int f, t;
        const int stage = r / mesh;
        mesh_coords(r % mesh, L->fsdp, L->tp_train, L->flags, &f, &t);
        int64_t off = 0;
        for (size_t i = 0; i < ps.size(); i++) {
            Piece pc;
            pc.param = int(i);
            pc.rect = stage_of(L->model, ps[i].kind, ps[i].layer, L->pp_train) == stage
                          ? trainer_rect(ps[i], f, t, L->fsdp, L->tp_train)
                          : Rect{};
            pc.rows = pc.rect.rows();
            pc.cols = pc.rect.cols();
            off = align_up(off);
            pc.byte_off = off;
            pc.dtype = L->dtype;
            off += pc.rows * pc.cols * es;
            L->pieces[r].push_back(pc);
        }
        L->rank_bytes[r] = align_up(off);
    }
    return LLRL_OK;
}

// R4: generator-local tensors of rank g; R7/R9 quantisation and scale grid.
llrl_status build_dst(llrl_layout *L) {
    const llrl_model &m = L->model;
    const int T = L->tp_gen;
    if (m.n_heads % T) return LLRL_E_INDIVISIBLE;
    if (m.n_kv_heads % T && T % m.n_kv_heads) return LLRL_E_INDIVISIBLE;
    if (m.d_ffn % T) return LLRL_E_INDIVISIBLE;
    if (m.with_embed && m.vocab % T) return LLRL_E_INDIVISIBLE;
    if (m.n_layers % L->pp_gen) return LLRL_E_INDIVISIBLE;
    // R15: MXFP4 packs two elements per byte -- quantised tensors keep whole 1x32 groups
    if (L->dtype == LLRL_MXFP4 && (m.d_model % kMxGroup || (int64_t(m.n_heads) * m.head_dim / T) % kMxGroup ||
                                   (m.d_ffn / T) % kMxGroup))
        return LLRL_E_UNSUPPORTED;
    if (L->dtype == LLRL_NVFP4 && (m.d_model % kNvGroup || (int64_t(m.n_heads) * m.head_dim / T) % kNvGroup ||
                                   (m.d_ffn / T) % kNvGroup))
        return LLRL_E_UNSUPPORTED;
    const auto &ps = L->src_params;
    auto &dp = L->dst_params;
    dp.clear();
    if (m.with_embed) dp.push_back({LLRL_P_EMBED, -1, false});
    for (int l = 0; l < m.n_layers; l++) {
        dp.push_back({LLRL_P_ATTN_NORM, l, false});
        dp.push_back({LLRL_P_QKV, l, true});
        dp.push_back({LLRL_P_O, l, true});
        dp.push_back({LLRL_P_MLP_NORM, l, false});
        dp.push_back({LLRL_P_GATE_UP, l, true});
        dp.push_back({LLRL_P_DOWN, l, true});
    }
    if (m.with_embed) {
        dp.push_back({LLRL_P_FINAL_NORM, -1, false});
        dp.push_back({LLRL_P_LM_HEAD, -1, false});
    }
    const int64_t d = m.d_model, hd = m.head_dim;
    const int64_t q_local = int64_t(m.n_heads) * hd / T;
    const bool kv_split = m.n_kv_heads % T == 0;
    const int64_t kv_local = kv_split ? int64_t(m.n_kv_heads) * hd / T : hd;
    const int64_t f_local = m.d_ffn / T;
    const int64_t v_local = m.with_embed ? m.vocab / T : 0;

    const int NS = T * L->pp_gen;           // ranks of one replica: stage*T + g
    L->n_ranks = NS;
    L->pieces.assign(size_t(NS), {});
    L->rank_bytes.assign(size_t(NS), 0);
    for (int sg = 0; sg < NS; sg++) {
        const int stage = sg / T, g = sg % T;
        const int64_t kv_row0 = kv_split ? g * kv_local : int64_t(g / (T / m.n_kv_heads)) * hd;
        int64_t off = 0;
        for (size_t i = 0; i < dp.size(); i++) {
            Piece pc;
            pc.param = int(i);
            const int l = dp[i].layer;
            auto src = [&](int kind) { return find_src(ps, kind, l); };
            switch (dp[i].kind) {
            case LLRL_P_ATTN_NORM: case LLRL_P_MLP_NORM: case LLRL_P_FINAL_NORM:
                pc.rows = d; pc.cols = 1;
                pc.parts = {{src(dp[i].kind), 0, 0, d, 1, 0}};
                break;
            case LLRL_P_QKV:
                pc.rows = q_local + 2 * kv_local; pc.cols = d;
                pc.parts = {{src(LLRL_P_Q), g * q_local, 0, q_local, d, 0},
                            {src(LLRL_P_K), kv_row0, 0, kv_local, d, q_local},
                            {src(LLRL_P_V), kv_row0, 0, kv_local, d, q_local + kv_local}};
                break;
            case LLRL_P_O:
                pc.rows = d; pc.cols = q_local;
                pc.parts = {{src(LLRL_P_O), 0, g * q_local, d, q_local, 0}};
                break;
            case LLRL_P_GATE_UP:
                pc.rows = 2 * f_local; pc.cols = d;
                pc.parts = {{src(LLRL_P_GATE), g * f_local, 0, f_local, d, 0},
                            {src(LLRL_P_UP), g * f_local, 0, f_local, d, f_local}};
                break;
            case LLRL_P_DOWN:
                pc.rows = d; pc.cols = f_local;
                pc.parts = {{src(LLRL_P_DOWN), 0, g * f_local, d, f_local, 0}};
                break;
            case LLRL_P_EMBED: case LLRL_P_LM_HEAD:
                pc.rows = v_local; pc.cols = d;
                pc.parts = {{src(dp[i].kind), g * v_local, 0, v_local, d, 0}};
                break;
            default:
                return LLRL_E_INVALID;
            }
            if (stage_of(m, dp[i].kind, l, L->pp_gen) != stage) {   // R14: another stage's tensor
                pc.rows = 0;
                pc.cols = 0;
                pc.parts.clear();
            }
            pc.rect = Rect{0, pc.rows, 0, pc.cols};
            pc.quantised = (L->dtype == LLRL_FP8_E4M3 || L->dtype == LLRL_MXFP8 || L->dtype == LLRL_MXFP4 ||
                            L->dtype == LLRL_NVFP4) && dp[i].quantisable;
            pc.dtype = pc.quantised ? L->dtype : (L->dtype == LLRL_F32 ? LLRL_F32 : LLRL_BF16);
            off = align_up(off);
            pc.byte_off = off;
            off += data_bytes(pc.dtype, pc.rows * pc.cols);
            if (pc.quantised) {
                off = align_up(off);
                pc.scale_off = off;
                off += scale_grid_bytes(L->dtype, pc.rows, pc.cols);
                if (L->dtype == LLRL_NVFP4) {      // R16: fp32 tensor scale at the next 256-byte boundary
                    off = align_up(off);
                    pc.tscale_off = off;
                    off += 4;
                }
            }
            L->pieces[size_t(sg)].push_back(pc);
        }
        L->rank_bytes[size_t(sg)] = align_up(off);
    }
    // R12: generator DP replicas -- rank d*NS + q is laid out exactly like rank q
    for (int rep = 1; rep < L->dp_gen; rep++)
        for (int q = 0; q < NS; q++) {
            L->pieces.push_back(L->pieces[size_t(q)]);
            L->rank_bytes.push_back(L->rank_bytes[size_t(q)]);
        }
    L->n_ranks = NS * L->dp_gen;
    return LLRL_OK;
}

bool model_ok(const llrl_model *m) {
    return m && m->n_layers >= 0 && m->d_model > 0 && m->n_heads > 0 && m->n_kv_heads > 0 &&
           m->head_dim > 0 && m->d_ffn > 0 && (!m->with_embed || m->vocab > 0);
}

}  // namespace

extern "C" {

const char *llrl_last_error(void) { return llrl::g_err; }
const char *llrl_version(void) { return "llrl 0.1 (sm_100a)"; }

llrl_status llrl_layout_describe_ex(const llrl_model *m, const llrl_layout_opts *o, llrl_layout **src_out,
                                    llrl_layout **dst_out) {
    if (!o || !src_out || !dst_out || !model_ok(m) || o->fsdp <= 0 || o->tp_train <= 0 || o->tp_gen <= 0 ||
        o->dp_gen <= 0 || o->pp_train <= 0 || o->pp_gen <= 0) {
        set_error("llrl_layout_describe: invalid argument");
        return LLRL_E_INVALID;
    }
    if (o->fsdp * o->tp_train * o->pp_train > kMaxRanks || o->tp_gen * o->dp_gen * o->pp_gen > kMaxRanks) {
        set_error("llrl_layout_describe: at most %d ranks per side", kMaxRanks);
        return LLRL_E_INVALID;
    }
    const int src_dtype = o->src_dtype, dst_dtype = o->dst_dtype;
    if ((src_dtype != LLRL_F32 && src_dtype != LLRL_BF16) ||
        (dst_dtype != LLRL_F32 && dst_dtype != LLRL_BF16 && dst_dtype != LLRL_FP8_E4M3 && dst_dtype != LLRL_MXFP8 &&
         dst_dtype != LLRL_MXFP4 && dst_dtype != LLRL_NVFP4) ||
        (dst_dtype == LLRL_F32 && src_dtype != LLRL_F32)) {
        set_error("llrl_layout_describe: unsupported dtypes src=%d dst=%d", src_dtype, dst_dtype);
        return LLRL_E_UNSUPPORTED;
    }
    llrl_layout *S = new (std::nothrow) llrl_layout();
    llrl_layout *D = new (std::nothrow) llrl_layout();
    if (!S || !D) { delete S; delete D; set_error("out of host memory"); return LLRL_E_NOMEM; }
    for (llrl_layout *L : {S, D}) {
        L->model = *m;
        L->fsdp = o->fsdp; L->tp_train = o->tp_train; L->tp_gen = o->tp_gen; L->dp_gen = o->dp_gen;
        L->pp_train = o->pp_train; L->pp_gen = o->pp_gen;
        L->flags = o->flags;
        L->src_params = enumerate_src_params(*m);
    }
    S->is_src = true;  S->dtype = src_dtype;
    D->is_src = false; D->dtype = dst_dtype;
    llrl_status st = build_src(S);
    if (st == LLRL_OK) st = build_dst(D);
    if (st != LLRL_OK) {
        set_error(st == LLRL_E_INDIVISIBLE ? "a tensor-parallel split does not divide a dimension (R1/R4)"
                                           : "layout construction failed");
        delete S; delete D;
        return st;
    }
    *src_out = S; *dst_out = D;
    return LLRL_OK;
}

llrl_status llrl_layout_describe(const llrl_model *m, int fsdp, int tp_train, int tp_gen,
                                 llrl_dtype src_dtype, llrl_dtype dst_dtype, uint32_t flags,
                                 llrl_layout **src_out, llrl_layout **dst_out) {
    const llrl_layout_opts o{fsdp, tp_train, tp_gen, 1, 1, 1, src_dtype, dst_dtype, flags, 0};
    return llrl_layout_describe_ex(m, &o, src_out, dst_out);
}

llrl_status llrl_layout_num_ranks(const llrl_layout *l, int *n) {
    if (!l || !n) { set_error("NULL argument"); return LLRL_E_INVALID; }
    *n = l->n_ranks;
    return LLRL_OK;
}

llrl_status llrl_layout_num_params(const llrl_layout *l, int *n) {
    if (!l || !n) { set_error("NULL argument"); return LLRL_E_INVALID; }
    *n = l->is_src ? int(l->src_params.size()) : int(l->dst_params.size());
    return LLRL_OK;
}

llrl_status llrl_layout_rank_bytes(const llrl_layout *l, int rank, int64_t *bytes) {
    if (!l || !bytes || rank < 0 || rank >= l->n_ranks) { set_error("invalid rank"); return LLRL_E_INVALID; }
    *bytes = l->rank_bytes[rank];
    return LLRL_OK;
}

llrl_status llrl_layout_param_view(const llrl_layout *l, int rank, int param, llrl_param_view *out) {
    if (!l || !out || rank < 0 || rank >= l->n_ranks || param < 0 || param >= int(l->pieces[rank].size())) {
        set_error("llrl_layout_param_view: invalid rank/param");
        return LLRL_E_INVALID;
    }
    const Piece &pc = l->pieces[rank][param];
    std::memset(out, 0, sizeof *out);
    if (l->is_src) {
        const SrcParam &sp = l->src_params[param];
        out->kind = sp.kind; out->layer = sp.layer; out->is_norm = sp.is_norm;
        out->src_param = param;
        out->full_r0 = pc.rect.r0; out->full_c0 = pc.rect.c0;
    } else {
        const DstParamDesc &dp = l->dst_params[param];
        out->kind = dp.kind; out->layer = dp.layer;
        out->is_norm = dp.kind == LLRL_P_ATTN_NORM || dp.kind == LLRL_P_MLP_NORM || dp.kind == LLRL_P_FINAL_NORM;
        out->src_param = -1;
    }
    out->dtype = pc.dtype;
    out->quantised = pc.quantised;
    out->rows = pc.rows; out->cols = pc.cols;
    out->byte_off = pc.byte_off;
    out->scale_off = pc.scale_off;
    out->tensor_scale_off = pc.tscale_off;
    return LLRL_OK;
}

void llrl_layout_destroy(llrl_layout *l) { delete l; }

}  // extern "C"
