// plan.cpp -- step a2: the routing plan.
//
// "Re-sharding ... computed by byte-range intersection", made
// 2-D: every generator part (a rectangle of a full source tensor, R4) is
// intersected with every trainer piece (R1-R3) holding that tensor.  Each
// non-empty intersection is a tile (param, src rank, dst rank, rows x cols,
// src/dst offsets and leading dimensions).  Replicated trainer pieces (norms
// under trainer TP) contribute one tile from one chosen holder (R5).  Tiles
// become device work items:
//   - bf16 / f32 destinations: K_CAST items of <= chunk_elems() elements, executed by
//     the SOURCE GPU (push: cast before the transfer, so NVLink carries the
//     destination width);
//   - fp8 destinations: one item per 128x128 block of the generator-local
//     tensor (R7); single-source blocks are pushed (K_FP8 on the source GPU),
//     multi-source blocks are pulled (K_FP8_MULTI on the destination GPU, R8).
// Each device's items are interleaved across destination devices in
// proportion to their bytes so that every NVLink peer and the local HBM copy
// progress together.  The plan also records the traffic matrix and the
// algorithmic HBM / NVLink bytes that bench.py's roofline uses.
#include <cstdlib>
#include <cstring>
#include <new>
#include <tuple>

#include "internal.h"

using namespace llrl;

namespace {

// elements per K_CAST item (64 KiB of bf16: keeps the grid's working window small);
// LLRL_CHUNK_ELEMS overrides (tuning knob)
int64_t chunk_elems() {
    static const int64_t c = [] {
        const char *v = getenv("LLRL_CHUNK_ELEMS");
        const int64_t x = v ? atoll(v) : 0;
        return x >= 1024 ? x / 8 * 8 : int64_t(32 * 1024);
    }();
    return c;
}

struct Builder {
    const llrl_layout *S, *D;
    llrl_plan *P;
    int64_t es_src, es_dst;

    // Generator DP replicas (R12): rank q = d*NS + position.  A position is
    // multicast-eligible when the plan asks for it and its replicas sit on
    // pairwise different GPUs.
    int n_pos() const { return D->n_ranks / D->dp_gen; }
    bool mc_position(int pos) const {
        if (!P->multicast || D->dp_gen < 2) return false;
        for (int a = 0; a < D->dp_gen; a++)
            for (int b = a + 1; b < D->dp_gen; b++)
                if (P->dst_device[size_t(a * n_pos() + pos)] == P->dst_device[size_t(b * n_pos() + pos)]) return false;
        return true;
    }
    std::vector<std::vector<std::vector<int>>> mc_extra;   // [exec dev][group] -> replica devices to signal
    uint64_t mc_counter = 0;
    // elements per cast item: chunk_elems(), or 8 Ki for tiny syncs (< 64 MB of
    // cast source in the plan: latency-bound, so every CTA of the register kernel
    // takes at most one item -- one dependent round trip, all its loads in
    // flight at once; C1: 11.2 us per isolated sync vs 12.0 at 4 Ki and 12.9 at
    // 1 Ki, profiles/r02/ab/c1_chunk.txt)
    int64_t chunk = chunk_elems();
    void size_chunks() {
        if (getenv("LLRL_CHUNK_ELEMS")) return;
        int64_t bytes = 0;
        for (const Tile &t : P->tiles) bytes += t.rows * t.cols * es_src;
        if (bytes < (int64_t(64) << 20)) chunk = 8192;
    }
    // multicast egress split: every k-th multicast item is pushed to each replica
    // instead (0 = all multicast, the default); LLRL_MC_UNICAST_PERIOD=k opts in.
    // Measured on C9 at 4 GPUs (profiles/r02/survey4.txt): k = 0 28.2 ms, 9 29.9,
    // 5 33.2, 3 39.3 -- the NVLS stores already occupy the egress links, so the
    // unicast share adds time instead of filling headroom.
    static int mc_unicast_period() {
        static const int k = [] {
            const char *v = getenv("LLRL_MC_UNICAST_PERIOD");
            return v ? std::max(0, atoi(v)) : 0;
        }();
        return k;
    }

    // a5 broadcast (R17): replica d >= 1 of a rank position whose replicas sit on
    // pairwise different GPUs is a byte copy of replica 0 -- left to ncclBroadcast.
    bool nccl_replica(int g) const {
        if (P->nccl_mode != 1) return false;
        const int pos = g % n_pos();
        if (g / n_pos() == 0) return false;
        for (int a = 0; a < D->dp_gen; a++)
            for (int b = a + 1; b < D->dp_gen; b++)
                if (P->dst_device[size_t(a * n_pos() + pos)] == P->dst_device[size_t(b * n_pos() + pos)]) return false;
        return true;
    }

    // a5 all-gather (R18): the whole sync is a plain replication of FSDP chunks.
    bool allgather_eligible() const {
        const int F = S->fsdp;
        if (F < 2 || S->tp_train != 1 || S->pp_train != 1 || D->tp_gen != 1 || D->pp_gen != 1 || D->dp_gen != F) return false;
        if (S->dtype != D->dtype || (D->dtype != LLRL_BF16 && D->dtype != LLRL_F32)) return false;
        for (int f = 0; f < F; f++) {
            if (P->src_device[size_t(f)] != P->dst_device[size_t(f)]) return false;
            for (int h = f + 1; h < F; h++)
                if (P->src_device[size_t(f)] == P->src_device[size_t(h)]) return false;
        }
        for (const SrcParam &sp : S->src_params)
            if (sp.rows % F) return false;
        return true;
    }

    int nccl_set(std::vector<int> devs) {
        std::sort(devs.begin(), devs.end());
        for (size_t k = 0; k < P->nccl_sets.size(); k++)
            if (P->nccl_sets[k] == devs) return int(k);
        P->nccl_sets.push_back(devs);
        return int(P->nccl_sets.size()) - 1;
    }

    void account_copy(int from, int to, int64_t bytes) {
        P->dev[size_t(to)].hbm_write += bytes;
        P->dev[size_t(from)].hbm_read += bytes;
        if (from != to) {
            P->dev[size_t(from)].nvl_tx += bytes;
            P->dev[size_t(to)].nvl_rx += bytes;
        }
        P->traffic[size_t(from) * P->n_devices + to] += bytes;
        P->stats.src_bytes += bytes;
        P->stats.dst_bytes += bytes;
    }

    void make_nccl_ops() {
        if (P->nccl_mode == 2) {
            const int F = S->fsdp;
            P->nccl_elem_bytes = int(es_src);
            std::vector<int> devs(P->src_device.begin(), P->src_device.begin() + F);
            nccl_set(devs);
            for (size_t p = 0; p < S->src_params.size(); p++) {
                const Piece &sp0 = S->pieces[0][p];
                // where the part of source param p lands in the generator (tp_gen = 1: whole rows)
                int64_t doff = -1;
                for (const Piece &pc : D->pieces[0])
                    for (const DstPart &part : pc.parts)
                        if (part.src_param == int(p)) doff = pc.byte_off + part.lr0 * pc.cols * es_src;
                llrl_plan::NcclGather og;
                og.src_param = int(p);
                og.count = sp0.rows * sp0.cols;
                for (int f = 0; f < F; f++) {
                    og.src_off.push_back(S->pieces[size_t(f)][p].byte_off);
                    og.dst_off.push_back(doff);
                }
                for (int f = 0; f < F; f++)
                    for (int h = 0; h < F; h++) account_copy(devs[size_t(h)], devs[size_t(f)], og.count * es_src);
                P->nccl_gather.push_back(og);
            }
            return;
        }
        for (int pos = 0; pos < n_pos(); pos++) {
            if (!nccl_replica(n_pos() + pos)) continue;
            std::vector<int> devs;
            for (int d = 0; d < D->dp_gen; d++) devs.push_back(P->dst_device[size_t(d * n_pos() + pos)]);
            llrl_plan::NcclBcast b;
            b.set = nccl_set(devs);
            b.root_dev = P->dst_device[size_t(pos)];
            b.bytes = D->rank_bytes[size_t(pos)];
            for (int dev : P->nccl_sets[size_t(b.set)])
                for (int d = 0; d < D->dp_gen; d++)
                    if (P->dst_device[size_t(d * n_pos() + pos)] == dev) b.dst_rank.push_back(d * n_pos() + pos);
            for (int d = 1; d < D->dp_gen; d++) account_copy(b.root_dev, P->dst_device[size_t(d * n_pos() + pos)], b.bytes);
            P->nccl_bcast.push_back(b);
        }
    }

    int holder(const std::vector<int> &members, int g) const {
        for (int r : members)
            if (P->src_device[r] == P->dst_device[g]) return r;   // same GPU first (R5)
        return members[size_t(g) % members.size()];              // else rotate by dst rank
    }

    llrl_status make_tiles() {
        const int nsrc = S->n_ranks;
        for (int g = 0; g < D->n_ranks; g++) {
            if (P->nccl_mode == 2 || nccl_replica(g)) continue;   // a5: filled by NCCL (R17, R18)
            for (const Piece &pc : D->pieces[g]) {
                const int64_t es_d = dtype_bytes(pc.dtype);
                for (const DstPart &part : pc.parts) {
                    const Rect F{part.fr0, part.fr0 + part.nr, part.fc0, part.fc0 + part.nc};
                    // group trainer pieces with identical rectangles (replicas)
                    std::vector<Rect> rects;
                    std::vector<std::vector<int>> members;
                    for (int s = 0; s < nsrc; s++) {
                        const Rect &r = S->pieces[s][part.src_param].rect;
                        if (intersect(r, F).empty()) continue;
                        size_t k = 0;
                        while (k < rects.size() && !(rects[k] == r)) k++;
                        if (k == rects.size()) { rects.push_back(r); members.push_back({}); }
                        members[k].push_back(s);
                    }
                    int64_t covered = 0;
                    for (size_t a = 0; a < rects.size(); a++) {
                        covered += intersect(rects[a], F).area();
                        for (size_t b = a + 1; b < rects.size(); b++)
                            if (!intersect(rects[a], rects[b]).empty()) {
                                set_error("trainer pieces of param %d overlap without being replicas", part.src_param);
                                return LLRL_E_INVALID;
                            }
                    }
                    if (covered != F.area()) {
                        set_error("param %d: trainer shards cover %lld of %lld elements", part.src_param,
                                  (long long)covered, (long long)F.area());
                        return LLRL_E_INVALID;
                    }
                    for (size_t a = 0; a < rects.size(); a++) {
                        const int h = holder(members[a], g);
                        const Piece &sp = S->pieces[h][part.src_param];
                        const Rect I = intersect(rects[a], F);
                        Tile t;
                        t.src_param = part.src_param;
                        t.dst_param = pc.param;
                        t.src_rank = h;
                        t.dst_rank = g;
                        t.rows = I.rows();
                        t.cols = I.cols();
                        t.src_ld = sp.cols;
                        t.src_off = sp.byte_off / es_src + (I.r0 - sp.rect.r0) * sp.cols + (I.c0 - sp.rect.c0);
                        t.lr0 = part.lr0 + (I.r0 - F.r0);
                        t.lc0 = I.c0 - F.c0;
                        t.dst_ld = pc.cols;
                        // element offset in the rank buffer (MXFP4: 4-bit elements)
                        t.dst_off = ((pc.dtype == LLRL_MXFP4 || pc.dtype == LLRL_NVFP4) ? 2 * pc.byte_off : pc.byte_off / es_d) +
                                    t.lr0 * pc.cols + t.lc0;
                        t.quant = pc.quantised;
                        P->tiles.push_back(t);
                    }
                }
            }
        }
        return LLRL_OK;
    }

    void add_cast_items(const Tile &t, std::vector<Item> &out) {
        Item base{};
        base.kind = K_CAST;
        base.src_rank = uint8_t(t.src_rank);
        base.dst_rank = uint8_t(t.dst_rank);
        base.tid = -1;
        const uint16_t fl = D->dtype == LLRL_F32 ? F_DST_F32 : 0;
        const bool contiguous = t.rows == 1 || (t.cols == t.src_ld && t.cols == t.dst_ld);
        if (contiguous) {
            // one 1-D run: scalar head up to a 16-byte destination boundary, vector body, scalar tail
            int64_t n = t.rows * t.cols, so = t.src_off, dof = t.dst_off;
            auto emit = [&](int64_t s, int64_t d, int64_t len, bool vec) {
                for (int64_t i = 0; i < len; i += chunk) {
                    Item it = base;
                    it.src_off = s + i; it.dst_off = d + i;
                    it.rows = 1; it.cols = int32_t(std::min(chunk, len - i));
                    it.src_ld = it.cols; it.dst_ld = it.cols;
                    it.flags = uint8_t(fl | (vec ? F_VEC : 0));
                    out.push_back(it);
                }
            };
            if ((so & 7) == (dof & 7)) {
                int64_t head = std::min<int64_t>((8 - (dof & 7)) & 7, n);
                int64_t body = (n - head) / 8 * 8;
                int64_t tail = n - head - body;
                if (head) emit(so, dof, head, false);
                if (body) emit(so + head, dof + head, body, true);
                if (tail) emit(so + head + body, dof + head + body, tail, false);
            } else {
                emit(so, dof, n, false);
            }
            return;
        }
        const bool vec = (t.src_off % 8 == 0) && (t.dst_off % 8 == 0) && (t.cols % 8 == 0) &&
                         (t.src_ld % 8 == 0) && (t.dst_ld % 8 == 0);
        const int64_t rows_per = std::max<int64_t>(1, chunk / t.cols);
        for (int64_t r = 0; r < t.rows; r += rows_per) {
            Item it = base;
            it.rows = int32_t(std::min(rows_per, t.rows - r));
            it.cols = int32_t(t.cols);
            it.src_ld = int32_t(t.src_ld);
            it.dst_ld = int32_t(t.dst_ld);
            it.src_off = t.src_off + r * t.src_ld;
            it.dst_off = t.dst_off + r * t.dst_ld;
            it.flags = uint8_t(fl | (vec ? F_VEC : 0));
            out.push_back(it);
        }
    }

    // MXFP8 tile -> cast items with F_MX.  Every 1x32 group must lie inside one
    // tile and one item: the tile's columns (or, for a run contiguous on both
    // sides, its whole length) start and end on 32-element group boundaries.
    std::map<std::pair<int, int>, int32_t> nv_tid;   // (dst rank, dst param) -> NVFP4 tensor id

    llrl_status add_mx_items(const Tile &t) {
        const Piece &pc = D->pieces[size_t(t.dst_rank)][size_t(t.dst_param)];
        const bool nv = pc.dtype == LLRL_NVFP4;
        const bool fp4 = pc.dtype == LLRL_MXFP4 || nv;
        const int64_t grp = nv ? kNvGroup : kMxGroup;
        const int64_t base = fp4 ? 2 * pc.byte_off : pc.byte_off;   // element offset of the tensor
        const bool contiguous = t.rows == 1 || (t.cols == t.src_ld && t.cols == t.dst_ld);
        const bool ok = (t.dst_off - base) % grp == 0 && (contiguous ? (t.rows * t.cols) % grp == 0
                                                                     : t.cols % grp == 0) &&
                        t.src_off % 8 == 0 && t.src_ld % 8 == 0 && pc.cols % grp == 0;
        if (!ok) {
            set_error("MX/NVFP4: tile of generator param %d is not aligned to whole row groups", t.dst_param);
            return LLRL_E_UNSUPPORTED;
        }
        int32_t tid = -1;
        if (nv) {
            auto key = std::make_pair(t.dst_rank, t.dst_param);
            auto f = nv_tid.find(key);
            if (f == nv_tid.end()) {
                tid = int32_t(P->nv_tensors.size());
                nv_tid[key] = tid;
                P->nv_tensors.push_back({int32_t(t.dst_rank), int32_t(t.dst_param),
                                         int32_t(P->dst_device[size_t(t.dst_rank)]), pc.tscale_off});
                P->dev[size_t(P->dst_device[size_t(t.dst_rank)])].hbm_write += 4;   // the fp32 tensor scale
                P->stats.dst_bytes += 4;
            } else {
                tid = f->second;
            }
            if (P->nv_sources.size() <= size_t(tid)) P->nv_sources.resize(size_t(tid) + 1);
            P->nv_sources[size_t(tid)].push_back(
                llrl_nv_source{int32_t(t.src_rank), int32_t(t.src_param), t.src_off, t.rows, t.cols, t.src_ld});
            DeviceWork &E = P->dev[size_t(P->src_device[size_t(t.src_rank)])];
            if (std::find(E.nv_contrib.begin(), E.nv_contrib.end(), tid) == E.nv_contrib.end())
                E.nv_contrib.push_back(tid);
        }
        std::vector<Item> tmp;
        add_cast_items(t, tmp);
        const int sd = P->src_device[size_t(t.src_rank)], dd = P->dst_device[size_t(t.dst_rank)];
        const SrcParam &sp = S->src_params[size_t(t.src_param)];
        auto &L = lists[size_t(sd)][size_t(dd)][size_t(group_of(sp.kind, sp.layer))];
        for (Item it : tmp) {
            it.flags = uint8_t((it.flags & F_VEC) | F_MX | (fp4 ? F_FP4 : 0) | (nv ? F_NV : 0));
            if (!(it.flags & F_VEC) || it.dst_off % grp != 0) {
                set_error("MX/NVFP4: unaligned cast item");
                return LLRL_E_UNSUPPORTED;
            }
            it.aux = pc.scale_off - base / grp;           // scale byte of element o: aux + o / group
            it.tid = tid;
            L.push_back(it);
        }
        const int64_t n = t.rows * t.cols;
        account(sd, sd, dd, n * es_src, (fp4 ? n / 2 : n) + n / grp, false);
        // R16: the two-pass sync's per-tensor amax pass reads the source once more.
        // Not algorithmic bytes (a sync given the amax reads it once): tracked apart.
        if (nv) P->dev[size_t(sd)].nv_amax_read += n * es_src;
        return LLRL_OK;
    }

    // work lists per executing device, per destination device, per layer group
    std::vector<std::vector<std::vector<std::vector<Item>>>> lists;   // [exec dev][dst dev][group]
    std::vector<std::vector<Seg>> seglists;                           // [exec dev] (pull blocks)
    int n_groups = 0;

    // Layer groups (llrl_sync_group): [embed] | layer 0 | ... | layer L-1 | [final_norm + lm_head].
    int group_of(int kind, int layer) const {
        const int base = S->model.with_embed ? 1 : 0;
        if (layer >= 0) return base + layer;
        if (kind == LLRL_P_EMBED) return 0;
        return n_groups - 1;
    }

    void account(int exec, int sdev, int ddev, int64_t src_bytes, int64_t dst_bytes, bool pull) {
        const int G = P->n_devices;
        P->dev[sdev].hbm_read += src_bytes;
        P->dev[ddev].hbm_write += dst_bytes;
        const int64_t wire = pull ? src_bytes : dst_bytes;
        if (sdev != ddev) {
            P->dev[sdev].nvl_tx += wire;
            P->dev[ddev].nvl_rx += wire;
        }
        if (pull) P->traffic[size_t(sdev) * G + ddev] += src_bytes;   // read by ddev from sdev
        else P->traffic[size_t(exec) * G + ddev] += dst_bytes;
        P->stats.src_bytes += src_bytes;
        P->stats.dst_bytes += dst_bytes;
    }

    // For every single-source vector fp8 block: the trainer piece it reads
    // (one TMA tensor map per piece) and its coordinates inside the piece.
    void make_tma_refs(DeviceWork &W) {
        std::map<std::pair<int, int>, int> piece_map;   // (src rank, piece index) -> map index
        W.tma_refs.assign(W.items.size() - size_t(W.n_cast), TmaRef{-1, 0, 0, 0});
        for (size_t i = size_t(W.n_cast); i < W.items.size(); i++) {
            const Item &it = W.items[i];
            if (it.kind != K_FP8 || !(it.flags & F_VEC)) continue;
            const auto &pcs = S->pieces[it.src_rank];
            // the piece containing element src_off (pieces are in increasing offset order)
            size_t lo = 0, hi = pcs.size();
            while (hi - lo > 1) {
                const size_t mid = (lo + hi) / 2;
                if (pcs[mid].byte_off / es_src <= it.src_off) lo = mid; else hi = mid;
            }
            while (lo > 0 && pcs[lo].rows * pcs[lo].cols == 0) lo--;
            const Piece &pc = pcs[lo];
            const int64_t rel = it.src_off - pc.byte_off / es_src;
            if ((pc.cols * es_src) % 16 != 0 || rel < 0 || rel >= pc.rows * pc.cols) continue;
            auto key = std::make_pair(int(it.src_rank), int(lo));
            auto f = piece_map.find(key);
            int m;
            if (f == piece_map.end()) {
                m = int(W.tma_pieces.size());
                piece_map[key] = m;
                W.tma_pieces.push_back(TmaPiece{int(it.src_rank), pc.byte_off, pc.rows, pc.cols});
            } else {
                m = f->second;
            }
            W.tma_refs[i - size_t(W.n_cast)] = TmaRef{m, int32_t(rel % pc.cols), int32_t(rel / pc.cols), 0};
        }
    }

    // For every vector cast item whose source rows are strided (a column band of
    // a wider trainer piece, e.g. o / down from FSDP row chunks into a column-
    // parallel generator): the band's 3-D tensor map and the item's first row in
    // it, so that each stage is one TMA box instead of one bulk copy per row.
    void make_cast_refs(DeviceWork &W) {
        std::map<std::tuple<int, int64_t, int64_t>, int> band_map;   // (src rank, band byte off, row bytes)
        W.cast_refs.assign(size_t(W.n_cast), CastRef{-1, 0});
        for (size_t i = 0; i < size_t(W.n_cast); i++) {
            const Item &it = W.items[i];
            if (it.kind != K_CAST || !(it.flags & F_VEC) || (it.flags & F_MC) || it.rows < 2 || it.cols == it.src_ld)
                continue;
            const auto &pcs = S->pieces[it.src_rank];
            size_t lo = 0, hi = pcs.size();
            while (hi - lo > 1) {
                const size_t mid = (lo + hi) / 2;
                if (pcs[mid].byte_off / es_src <= it.src_off) lo = mid; else hi = mid;
            }
            while (lo > 0 && pcs[lo].rows * pcs[lo].cols == 0) lo--;
            const Piece &pc = pcs[lo];
            const int64_t rel = it.src_off - pc.byte_off / es_src;
            if (pc.cols != it.src_ld || rel < 0 || rel >= pc.rows * pc.cols) continue;
            const int64_t row = rel / pc.cols, col = rel % pc.cols;
            const int64_t off = pc.byte_off + col * es_src, rb = int64_t(it.cols) * es_src;
            auto key = std::make_tuple(int(it.src_rank), off, rb);
            auto f = band_map.find(key);
            int m;
            if (f == band_map.end()) {
                m = int(W.cast_bands.size());
                band_map[key] = m;
                W.cast_bands.push_back(CastBand{int(it.src_rank), off, pc.rows, rb, pc.cols * es_src});
            } else {
                m = f->second;
            }
            W.cast_refs[i] = CastRef{m, int32_t(row)};
        }
        if (W.cast_bands.empty()) W.cast_refs.clear();
    }

    llrl_status make_items() {
        const int G = P->n_devices;
        n_groups = S->model.n_layers + (S->model.with_embed ? 2 : 0);
        P->n_groups = n_groups;
        P->model_with_embed = S->model.with_embed != 0;
        lists.assign(G, std::vector<std::vector<std::vector<Item>>>(G, std::vector<std::vector<Item>>(n_groups)));
        mc_extra.assign(size_t(G), std::vector<std::vector<int>>(size_t(n_groups)));
        seglists.assign(G, {});
        // bf16 / f32 tiles, and MXFP8 tiles (row-wise 1x32 groups ride on cast items, R13)
        const bool mx = D->dtype == LLRL_MXFP8 || D->dtype == LLRL_MXFP4 || D->dtype == LLRL_NVFP4;
        for (const Tile &t : P->tiles) {
            if (t.quant && !mx) continue;
            if (t.quant) {
                llrl_status st = add_mx_items(t);
                if (st != LLRL_OK) return st;
                continue;
            }
            const int sd = P->src_device[t.src_rank], dd = P->dst_device[t.dst_rank];
            const SrcParam &sp = S->src_params[size_t(t.src_param)];
            const size_t grp = size_t(group_of(sp.kind, sp.layer));
            const int pos = t.dst_rank % n_pos(), rep = t.dst_rank / n_pos();
            if (!mc_position(pos)) {
                add_cast_items(t, lists[sd][dd][grp]);
                account(sd, sd, dd, t.rows * t.cols * es_src, t.rows * t.cols * es_dst, false);
                continue;
            }
            // multicast: replica 0's items go through the multicast VA (one NVLink
            // egress copy for all replicas); the other replicas' tiles emit nothing
            if (rep != 0) continue;
            std::vector<Item> tmp;
            add_cast_items(t, tmp);
            for (Item it : tmp) {
                const int64_t n = int64_t(it.rows) * it.cols;
                // egress split: NVLS multicast stores top out below the link rate
                // (~560 of ~770 GB/s), so one item in mc_unicast_period() goes to
                // every replica as plain peer pushes, filling the link's headroom
                if (mc_unicast_period() > 0 && (mc_counter++ % uint64_t(mc_unicast_period())) == 0) {
                    for (int d = 0; d < D->dp_gen; d++) {
                        Item u = it;
                        u.dst_rank = uint8_t(d * n_pos() + pos);   // replicas share replica 0's layout (R12)
                        const int rd = P->dst_device[size_t(u.dst_rank)];
                        lists[sd][rd][grp].push_back(u);
                        account(sd, sd, rd, n * es_src, n * es_dst, false);
                    }
                    continue;
                }
                {
                    it.flags = uint8_t(it.flags | F_MC);
                    lists[sd][dd][grp].push_back(it);
                    P->dev[size_t(sd)].has_mc = true;
                    account(sd, sd, dd, n * es_src, n * es_dst, false);
                    for (int d = 1; d < D->dp_gen; d++) {
                        const int rd = P->dst_device[size_t(d * n_pos() + pos)];
                        P->dev[size_t(rd)].hbm_write += n * es_dst;
                        if (rd != sd) P->dev[size_t(rd)].nvl_rx += n * es_dst;
                        P->traffic[size_t(sd) * P->n_devices + rd] += n * es_dst;
                        P->stats.dst_bytes += n * es_dst;
                        if (rd != sd) {
                            auto &ex = mc_extra[size_t(sd)][grp];
                            if (std::find(ex.begin(), ex.end(), rd) == ex.end()) ex.push_back(rd);
                        }
                    }
                }
            }
        }
        // fp8 blocks: group quantised tiles by (dst rank, dst param)
        std::map<std::pair<int, int>, std::vector<size_t>> by_param;
        for (size_t i = 0; i < P->tiles.size(); i++)
            if (P->tiles[i].quant && !mx) by_param[{P->tiles[i].dst_rank, P->tiles[i].dst_param}].push_back(i);
        for (auto &kv : by_param) {
            const int g = kv.first.first;
            const Piece &pc = D->pieces[g][kv.first.second];
            const int dd = P->dst_device[g];
            const DstParamDesc &dpd = D->dst_params[size_t(kv.first.second)];
            const size_t grp = size_t(group_of(dpd.kind, dpd.layer));
            const int64_t nbr = (pc.rows + kFp8Block - 1) / kFp8Block, nbc = (pc.cols + kFp8Block - 1) / kFp8Block;
            for (int64_t bi = 0; bi < nbr; bi++)
                for (int64_t bj = 0; bj < nbc; bj++) {
                    const Rect B{bi * kFp8Block, std::min(pc.rows, (bi + 1) * kFp8Block),
                                 bj * kFp8Block, std::min(pc.cols, (bj + 1) * kFp8Block)};
                    std::vector<std::pair<size_t, Rect>> segs;
                    for (size_t ti : kv.second) {
                        const Tile &t = P->tiles[ti];
                        const Rect I = intersect(Rect{t.lr0, t.lr0 + t.rows, t.lc0, t.lc0 + t.cols}, B);
                        if (!I.empty()) segs.push_back({ti, I});
                    }
                    Item it{};
                    it.dst_rank = uint8_t(g);
                    it.tid = -1;
                    it.rows = int32_t(B.rows());
                    it.cols = int32_t(B.cols());
                    it.dst_off = pc.byte_off + B.r0 * pc.cols + B.c0;
                    it.dst_ld = int32_t(pc.cols);
                    it.aux = pc.scale_off + (bi * nbc + bj) * 4;
                    P->stats.n_fp8_blocks++;
                    if (segs.size() == 1 && segs[0].second == B) {
                        const Tile &t = P->tiles[segs[0].first];
                        const int sd = P->src_device[t.src_rank];
                        it.kind = K_FP8;
                        it.src_rank = uint8_t(t.src_rank);
                        it.src_off = t.src_off + (B.r0 - t.lr0) * t.src_ld + (B.c0 - t.lc0);
                        it.src_ld = int32_t(t.src_ld);
                        const bool vec = it.cols % 16 == 0 && it.src_off % 8 == 0 && it.src_ld % 8 == 0 &&
                                         it.dst_off % 16 == 0 && it.dst_ld % 16 == 0;
                        it.flags = vec ? F_VEC : 0;
                        lists[sd][dd][grp].push_back(it);
                        account(sd, sd, dd, B.area() * es_src, B.area() + 4, false);
                    } else {
                        it.kind = K_FP8_MULTI;
                        P->stats.n_fp8_pull_blocks++;
                        auto &sl = seglists[dd];
                        it.src_off = int64_t(sl.size());
                        it.src_rank = uint8_t(segs.size());   // segment count
                        for (auto &s : segs) {
                            const Tile &t = P->tiles[s.first];
                            const Rect &I = s.second;
                            Seg sg{};
                            sg.src_rank = t.src_rank;
                            sg.src_ld = int32_t(t.src_ld);
                            sg.src_off = t.src_off + (I.r0 - t.lr0) * t.src_ld + (I.c0 - t.lc0);
                            sg.r0 = int32_t(I.r0 - B.r0);
                            sg.c0 = int32_t(I.c0 - B.c0);
                            sg.rows = int32_t(I.rows());
                            sg.cols = int32_t(I.cols());
                            sl.push_back(sg);
                            account(dd, P->src_device[t.src_rank], dd, I.area() * es_src, 0, true);
                        }
                        account(dd, dd, dd, 0, B.area() + 4, false);
                        lists[dd][dd][grp].push_back(it);
                    }
                }
        }
        // Per executing device and layer group: interleave the destination lists by
        // fractional progress (every NVLink peer and the local copy advance
        // together), then lay the items out as [cast items | fp8 items], each
        // class group-major, with per-group offsets for llrl_sync_group.
        auto item_bytes = [](const Item &it) { return double(it.rows) * double(it.cols); };
        for (int e = 0; e < G; e++) {
            DeviceWork &W = P->dev[e];
            W.segs = std::move(seglists[e]);
            std::vector<std::vector<Item>> cast_g(static_cast<size_t>(n_groups)), fp8_g(static_cast<size_t>(n_groups));
            W.group_signal.assign(size_t(n_groups), {});
            std::vector<char> sends(size_t(G), 0);
            for (int grp = 0; grp < n_groups; grp++) {
                struct Cursor { int dst; size_t pos; double total, done; };
                std::vector<Cursor> cur;
                for (int d = 0; d < G; d++) {
                    const auto &L = lists[e][d][size_t(grp)];
                    if (L.empty()) continue;
                    double tot = 0;
                    for (auto &it : L) tot += item_bytes(it);
                    cur.push_back({d, 0, tot, 0});
                    if (d != e) { W.group_signal[size_t(grp)].push_back(d); sends[size_t(d)] = 1; }
                }
                for (int d : mc_extra[size_t(e)][size_t(grp)]) {      // multicast replicas are written too
                    auto &gs = W.group_signal[size_t(grp)];
                    if (std::find(gs.begin(), gs.end(), d) == gs.end()) { gs.push_back(d); sends[size_t(d)] = 1; }
                }
                // rotate the start by the executing device so senders spread over receivers
                if (!cur.empty()) std::rotate(cur.begin(), cur.begin() + size_t(e) % cur.size(), cur.end());
                size_t n_total = 0, n_done = 0;
                for (auto &c : cur) n_total += lists[e][c.dst][size_t(grp)].size();
                while (n_done < n_total) {
                    Cursor *best = nullptr;
                    double best_frac = 2.0;
                    for (auto &c : cur) {
                        if (c.pos >= lists[e][c.dst][size_t(grp)].size()) continue;
                        const double f = c.done / c.total;
                        if (f < best_frac) { best_frac = f; best = &c; }
                    }
                    const Item &it = lists[e][best->dst][size_t(grp)][best->pos++];
                    best->done += item_bytes(it);
                    (it.kind == K_CAST ? cast_g : fp8_g)[size_t(grp)].push_back(it);
                    n_done++;
                }
            }
            W.cast_off.assign(size_t(n_groups) + 1, 0);
            W.fp8_off.assign(size_t(n_groups) + 1, 0);
            for (int grp = 0; grp < n_groups; grp++) {
                W.cast_off[size_t(grp)] = int64_t(W.items.size());
                W.items.insert(W.items.end(), cast_g[size_t(grp)].begin(), cast_g[size_t(grp)].end());
            }
            W.n_cast = int64_t(W.items.size());
            W.cast_off[size_t(n_groups)] = W.n_cast;
            for (int grp = 0; grp < n_groups; grp++) {
                W.fp8_off[size_t(grp)] = int64_t(W.items.size());
                W.items.insert(W.items.end(), fp8_g[size_t(grp)].begin(), fp8_g[size_t(grp)].end());
            }
            W.fp8_off[size_t(n_groups)] = int64_t(W.items.size());
            for (int d = 0; d < G; d++)
                if (sends[size_t(d)]) W.signal_devices.push_back(d);
            make_tma_refs(W);
            make_cast_refs(W);
            P->stats.n_items += int64_t(W.items.size());
        }
        for (int e = 0; e < G; e++) {
            P->dev[size_t(e)].group_senders_in.assign(size_t(n_groups), 0);
            P->dev[size_t(e)].group_senders.assign(size_t(n_groups), {});
        }
        for (int e = 0; e < G; e++) {
            for (int d : P->dev[size_t(e)].signal_devices) {
                P->dev[size_t(d)].n_senders_in++;
                P->dev[size_t(d)].senders.push_back(e);
            }
            for (int grp = 0; grp < n_groups; grp++)
                for (int d : P->dev[size_t(e)].group_signal[size_t(grp)]) {
                    P->dev[size_t(d)].group_senders_in[size_t(grp)]++;
                    if (P->dev[size_t(d)].group_senders.empty())
                        P->dev[size_t(d)].group_senders.assign(size_t(n_groups), {});
                    P->dev[size_t(d)].group_senders[size_t(grp)].push_back(e);
                }
        }
        // pull dependencies per group (multi-source fp8 blocks read peers' trainer bytes)
        for (int e = 0; e < G; e++) {
            P->dev[size_t(e)].pull_from.assign(size_t(n_groups), {});
            P->dev[size_t(e)].pull_to.assign(size_t(n_groups), {});
        }
        for (int e = 0; e < G; e++) {
            DeviceWork &W = P->dev[size_t(e)];
            for (int grp = 0; grp < n_groups; grp++) {
                std::vector<char> from(size_t(G), 0);
                for (int64_t i = W.fp8_off[size_t(grp)]; i < W.fp8_off[size_t(grp) + 1]; i++) {
                    const Item &it = W.items[size_t(i)];
                    if (it.kind != K_FP8_MULTI) continue;
                    for (int k = 0; k < it.src_rank; k++) {
                        const int sd = P->src_device[size_t(W.segs[size_t(it.src_off) + size_t(k)].src_rank)];
                        if (sd != e) from[size_t(sd)] = 1;
                    }
                }
                for (int sd = 0; sd < G; sd++)
                    if (from[size_t(sd)]) {
                        W.pull_from[size_t(grp)].push_back(sd);
                        P->dev[size_t(sd)].pull_to[size_t(grp)].push_back(e);
                    }
            }
        }
        // NVFP4 handshake sets: tensors held per device, contributors per device
        for (int32_t tid = 0; tid < int32_t(P->nv_tensors.size()); tid++)
            P->dev[size_t(P->nv_tensors[size_t(tid)].device)].nv_local.push_back(tid);
        for (int e = 0; e < G; e++)
            for (int32_t tid : P->dev[size_t(e)].nv_contrib) {
                const int d = P->nv_tensors[size_t(tid)].device;
                auto &tg = P->dev[size_t(e)].nv_targets;
                if (std::find(tg.begin(), tg.end(), d) == tg.end()) tg.push_back(d);
                auto &sn = P->dev[size_t(d)].nv_senders;
                if (std::find(sn.begin(), sn.end(), e) == sn.end()) sn.push_back(e);
            }
        // per-group byte ranges of every rank buffer (host <-> device streaming)
        P->src_group_range.assign(size_t(S->n_ranks), std::vector<std::pair<int64_t, int64_t>>(size_t(n_groups), {-1, -1}));
        P->dst_group_range.assign(size_t(D->n_ranks), std::vector<std::pair<int64_t, int64_t>>(size_t(n_groups), {-1, -1}));
        auto widen = [](std::pair<int64_t, int64_t> &r, int64_t lo, int64_t hi) {
            if (hi <= lo) return;
            if (r.first < 0) r = {lo, hi};
            else r = {std::min(r.first, lo), std::max(r.second, hi)};
        };
        for (int r = 0; r < S->n_ranks; r++)
            for (const Piece &pc : S->pieces[size_t(r)]) {
                const SrcParam &sp = S->src_params[size_t(pc.param)];
                widen(P->src_group_range[size_t(r)][size_t(group_of(sp.kind, sp.layer))], pc.byte_off,
                      pc.byte_off + pc.rows * pc.cols * es_src);
            }
        for (int g = 0; g < D->n_ranks; g++)
            for (const Piece &pc : D->pieces[size_t(g)]) {
                const DstParamDesc &dpd = D->dst_params[size_t(pc.param)];
                auto &rg = P->dst_group_range[size_t(g)][size_t(group_of(dpd.kind, dpd.layer))];
                widen(rg, pc.byte_off, pc.byte_off + data_bytes(pc.dtype, pc.rows * pc.cols));
                if (pc.quantised) widen(rg, pc.scale_off, pc.scale_off + scale_grid_bytes(pc.dtype, pc.rows, pc.cols));
                if (pc.tscale_off >= 0) widen(rg, pc.tscale_off, pc.tscale_off + 4);   // NVFP4 tensor scale
            }
        return LLRL_OK;
    }
};

bool same_model(const llrl_model &a, const llrl_model &b) { return std::memcmp(&a, &b, sizeof a) == 0; }

}  // namespace

llrl_plan::~llrl_plan() = default;   // device tables are released by llrl_plan_destroy (runtime.cu)

extern "C" {

llrl_status llrl_plan_create(const llrl_layout *src, const llrl_layout *dst, const int *src_device,
                             const int *dst_device, uint32_t flags, llrl_plan **out) {
    if (!src || !dst || !src_device || !dst_device || !out || !src->is_src || dst->is_src) {
        set_error("llrl_plan_create: invalid argument");
        return LLRL_E_INVALID;
    }
    if (!same_model(src->model, dst->model) || src->src_params.size() != dst->src_params.size()) {
        set_error("llrl_plan_create: src and dst describe different models");
        return LLRL_E_MISMATCH;
    }
    llrl_plan *P = new (std::nothrow) llrl_plan();
    if (!P) { set_error("out of host memory"); return LLRL_E_NOMEM; }
    P->n_src = src->n_ranks;
    P->n_dst = dst->n_ranks;
    P->multicast = (flags & LLRL_PLAN_MULTICAST) != 0;
    P->nv = dst->dtype == LLRL_NVFP4;
    P->src_dtype = src->dtype;
    P->dst_dtype = dst->dtype;
    P->src_device.assign(src_device, src_device + P->n_src);
    P->dst_device.assign(dst_device, dst_device + P->n_dst);
    P->src_rank_bytes = src->rank_bytes;
    P->dst_rank_bytes = dst->rank_bytes;
    int maxdev = 0;
    for (int d : P->src_device) maxdev = std::max(maxdev, d);
    for (int d : P->dst_device) maxdev = std::max(maxdev, d);
    for (int d : P->src_device) if (d < 0) maxdev = kMaxDevices;
    for (int d : P->dst_device) if (d < 0) maxdev = kMaxDevices;
    if (maxdev >= kMaxDevices) {
        delete P;
        set_error("llrl_plan_create: device ordinals must be in [0, %d)", kMaxDevices);
        return LLRL_E_INVALID;
    }
    P->n_devices = maxdev + 1;
    P->dev.resize(P->n_devices);
    P->traffic.assign(size_t(P->n_devices) * P->n_devices, 0);
    std::memset(&P->stats, 0, sizeof P->stats);
    // es_dst: element size of NON-quantised generator tensors (quantised formats keep
    // embed / lm_head / norms in bf16, R7 / R13 / R15)
    Builder b{};
    b.S = src;
    b.D = dst;
    b.P = P;
    b.es_src = dtype_bytes(src->dtype);
    b.es_dst = dtype_bytes(dst->dtype == LLRL_F32 ? LLRL_F32 : LLRL_BF16);
    if (flags & LLRL_PLAN_NCCL) {
        if (P->multicast) {
            delete P;
            set_error("llrl_plan_create: LLRL_PLAN_NCCL and LLRL_PLAN_MULTICAST are exclusive");
            return LLRL_E_INVALID;
        }
        P->nccl_mode = b.allgather_eligible() ? 2 : dst->dp_gen >= 2 ? 1 : 0;
    }
    llrl_status st = b.make_tiles();
    if (st == LLRL_OK) {
        b.size_chunks();
        st = b.make_items();
    }
    if (st == LLRL_OK) b.make_nccl_ops();
    if (st == LLRL_OK && P->nccl_mode == 1 && P->nccl_bcast.empty()) P->nccl_mode = 0;
    if (st != LLRL_OK) { delete P; return st; }
    P->stats.n_devices = P->n_devices;
    P->stats.n_src_ranks = P->n_src;
    P->stats.n_dst_ranks = P->n_dst;
    P->stats.n_tiles = int64_t(P->tiles.size());
    *out = P;
    return LLRL_OK;
}

static int64_t tile_runs(const Tile &t) {
    return (t.rows == 1 || (t.cols == t.src_ld && t.cols == t.dst_ld)) ? 1 : t.rows;
}

llrl_status llrl_plan_num_runs(const llrl_plan *p, int64_t *n) {
    if (!p || !n) { set_error("NULL argument"); return LLRL_E_INVALID; }
    int64_t s = 0;
    for (const Tile &t : p->tiles) s += tile_runs(t);
    *n = s;
    return LLRL_OK;
}

llrl_status llrl_plan_get_runs(const llrl_plan *p, int64_t first, int64_t count, llrl_run *out) {
    if (!p || (!out && count) || first < 0 || count < 0) { set_error("invalid argument"); return LLRL_E_INVALID; }
    int64_t idx = 0, w = 0;
    for (const Tile &t : p->tiles) {
        const int64_t nr = tile_runs(t);
        if (idx + nr <= first) { idx += nr; continue; }
        for (int64_t k = std::max<int64_t>(0, first - idx); k < nr && w < count; k++) {
            llrl_run &r = out[w++];
            r.src_param = t.src_param;
            r.src_rank = t.src_rank;
            r.dst_rank = t.dst_rank;
            r.flags = t.quant ? 1 : 0;
            if (nr == 1) { r.src_off = t.src_off; r.dst_off = t.dst_off; r.len = t.rows * t.cols; }
            else { r.src_off = t.src_off + k * t.src_ld; r.dst_off = t.dst_off + k * t.dst_ld; r.len = t.cols; }
        }
        idx += nr;
        if (w == count) break;
    }
    if (w != count) { set_error("run range out of bounds"); return LLRL_E_INVALID; }
    return LLRL_OK;
}

llrl_status llrl_plan_stats_get(const llrl_plan *p, llrl_plan_stats *out) {
    if (!p || !out) { set_error("NULL argument"); return LLRL_E_INVALID; }
    *out = p->stats;
    return LLRL_OK;
}

llrl_status llrl_plan_traffic(const llrl_plan *p, int64_t *bytes) {
    if (!p || !bytes) { set_error("NULL argument"); return LLRL_E_INVALID; }
    std::copy(p->traffic.begin(), p->traffic.end(), bytes);
    return LLRL_OK;
}

llrl_status llrl_plan_device_bytes(const llrl_plan *p, int device, int64_t *hbm_read, int64_t *hbm_write,
                                   int64_t *nvl_tx, int64_t *nvl_rx) {
    if (!p || device < 0 || device >= p->n_devices) { set_error("invalid device"); return LLRL_E_INVALID; }
    const DeviceWork &W = p->dev[device];
    if (hbm_read) *hbm_read = W.hbm_read;
    if (hbm_write) *hbm_write = W.hbm_write;
    if (nvl_tx) *nvl_tx = W.nvl_tx;
    if (nvl_rx) *nvl_rx = W.nvl_rx;
    return LLRL_OK;
}

}  // extern "C"
