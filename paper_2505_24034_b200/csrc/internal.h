// internal.h -- library-private types of libllrl (host C++ + CUDA).
// Nothing here is shared with oracle/ (independent paths).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "llrl.h"

namespace llrl {

constexpr int kMaxRanks = 64;      // per side; kernel parameter tables are sized by it
constexpr int kMaxDevices = 16;
constexpr int64_t kAlign = 256;    // R0: every piece starts at a 256-byte boundary
constexpr int kFp8Block = 128;     // R7
constexpr int kMxGroup = 32;       // R13
constexpr int kNvGroup = 16;       // R16

void set_error(const char *fmt, ...);
int64_t dtype_bytes(int dt);
int64_t scale_grid_bytes(int dt, int64_t rows, int64_t cols);
int64_t data_bytes(int dt, int64_t elems);   // MXFP4: elems / 2

// A rectangle [r0, r1) x [c0, c1) of a full parameter tensor.
struct Rect {
    int64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
    int64_t rows() const { return r1 - r0; }
    int64_t cols() const { return c1 - c0; }
    int64_t area() const { return rows() * cols(); }
    bool empty() const { return r1 <= r0 || c1 <= c0; }
    bool operator==(const Rect &o) const { return r0 == o.r0 && r1 == o.r1 && c0 == o.c0 && c1 == o.c1; }
};
inline Rect intersect(const Rect &a, const Rect &b) {
    Rect r{std::max(a.r0, b.r0), std::min(a.r1, b.r1), std::max(a.c0, b.c0), std::min(a.c1, b.c1)};
    if (r.empty()) r = Rect{};
    return r;
}

// Full (unsharded) source parameter.
struct SrcParam {
    int kind;      // LLRL_P_*
    int layer;
    int64_t rows, cols;
    int split;     // 0 = rows (column-parallel), 1 = cols (row-parallel), 2 = replicated (norm)
    bool is_norm;
};

// One contribution of a source parameter to a generator tensor:
// full rows [fr0, fr0+nr) x cols [fc0, fc0+nc) land at local rows [lr0, ...), cols [0, nc).
struct DstPart {
    int src_param;
    int64_t fr0, fc0, nr, nc, lr0;
};

struct Piece {          // one parameter on one rank
    int param;          // index in this side's param list
    Rect rect;          // src side: rectangle of the full tensor; dst side: local [0,R)x[0,C)
    int64_t rows, cols; // local shape
    int64_t byte_off;
    int64_t scale_off = -1;
    int64_t tscale_off = -1;      // NVFP4 fp32 tensor scale (R16)
    bool quantised = false;
    int dtype;
    std::vector<DstPart> parts;   // dst side only
};

struct DstParamDesc {
    int kind, layer;
    bool quantisable;   // linear weight (qkv / o / gate_up / down)
};

}  // namespace llrl

struct llrl_layout {
    bool is_src;
    llrl_model model;
    int fsdp, tp_train, tp_gen, dp_gen, pp_train, pp_gen;
    int dtype;          // src: data dtype; dst: target dtype (F32/BF16/FP8)
    uint32_t flags;
    int n_ranks;
    std::vector<llrl::SrcParam> src_params;      // canonical source params (both sides keep it)
    std::vector<llrl::DstParamDesc> dst_params;  // dst side only
    std::vector<std::vector<llrl::Piece>> pieces;   // [rank][param]
    std::vector<int64_t> rank_bytes;
};

namespace llrl {
// layout.cpp
std::vector<SrcParam> enumerate_src_params(const llrl_model &m);
}

// ---- plan ----------------------------------------------------------------

namespace llrl {

enum ItemKind : uint8_t {
    K_CAST = 0,        // 2-D (or 1-D when rows == 1) relayout + cast to bf16 / copy to f32
    K_FP8 = 1,         // one 128x128 (or edge) fp8 block, single source
    K_FP8_MULTI = 2,   // one fp8 block gathered from several sources (pull, R8)
};
enum ItemFlag : uint8_t {
    F_VEC = 1,         // 16-byte vector path legal (offsets / lds / cols aligned)
    F_DST_F32 = 2,     // destination dtype f32 (identity), else bf16 (K_CAST)
    F_MX = 4,          // K_CAST into MXFP8 codes (1 byte); aux = scale byte base (R13)
    F_MC = 8,          // K_CAST stored through the NVLS multicast VA of dst_rank's position (f1)
    F_FP4 = 16,        // with F_MX: MXFP4 (E2M1 codes, two per byte; dst offsets in 4-bit elements) (R15)
    F_NV = 32,         // with F_MX | F_FP4: NVFP4 1x16 groups, E4M3 group scales, per-tensor scale (R16)
};

// Device work item (48 bytes).  Offsets in elements of each side's dtype, except
// fp8 items: dst_off = byte offset of the block's top-left code, aux = byte
// offset of its scale.  K_FP8_MULTI: src_off = first segment index, src_rank =
// segment count.
struct alignas(16) Item {
    int64_t src_off;
    int64_t dst_off;
    int64_t aux;
    int32_t rows, cols;
    int32_t src_ld, dst_ld;
    uint8_t src_rank, dst_rank;   // < kMaxRanks (K_FP8_MULTI: src_rank = segment count)
    uint8_t kind, flags;
    int32_t tid;                  // NVFP4 (F_NV): generator tensor id (amax table row), else -1
};
static_assert(sizeof(Item) == 48, "Item layout");

// Segment of a multi-source fp8 block (block-local rectangle + its source).
struct alignas(16) Seg {
    int64_t src_off;
    int32_t src_ld;
    int32_t src_rank;
    int32_t r0, c0, rows, cols;
};
static_assert(sizeof(Seg) == 32, "Seg layout");

// fp8 block source as a 2-D TMA tile: tensor map `map` (one per source piece)
// and the block's top-left (x = column, y = row) inside that piece.  map < 0:
// no tensor map (stride not 16-byte aligned); the kernel stages row by row.
struct TmaRef {
    int32_t map, x, y, pad;
};
struct TmaPiece {            // a trainer piece that fp8 blocks read through a tensor map
    int src_rank;
    int64_t byte_off, rows, cols;
};
// A column band of a trainer piece that strided cast items read through a 3-D
// tensor map: rows of `row_bytes` at a pitch of `ld_bytes`, starting at byte_off
// of the src rank buffer (each stage of an item = one box of whole rows).
struct CastBand {
    int src_rank;
    int64_t byte_off, rows, row_bytes, ld_bytes;
};
struct CastRef {             // per cast item: its band's map (-1: none) and first row in the band
    int32_t map, row;
};

// Host-side tile: one rectangle intersection (param part, src rank, dst rank).
struct Tile {
    int src_param;
    int dst_param;
    int src_rank, dst_rank;
    int64_t rows, cols;
    int64_t src_off, src_ld;   // elements
    int64_t dst_off, dst_ld;   // elements (fp8: bytes)
    int64_t lr0, lc0;          // top-left in the generator-local tensor
    bool quant;
};

struct DeviceWork {
    std::vector<Item> items;
    std::vector<Seg> segs;
    std::vector<TmaRef> tma_refs;      // one per fp8 item (index i - n_cast)
    std::vector<CastRef> cast_refs;    // one per cast item (strided source rows: 3-D tensor map)
    std::vector<CastBand> cast_bands;
    std::vector<void *> dst_mc;        // multicast VA per dst rank (llrl_plan_set_multicast)
    // NVFP4 (R16) per-tensor amax handshake
    std::vector<int32_t> nv_contrib;   // tensor ids this device's items quantise
    std::vector<int> nv_targets;       // devices holding those tensors (amax -> them, ready <- them)
    std::vector<int32_t> nv_local;     // tensor ids held by this device
    std::vector<int> nv_senders;       // devices contributing to them
    uint32_t *d_nv_partial = nullptr;  // [n_tensors] local partial amax (u32 bits)
    uint32_t *d_nv_amax = nullptr;     // [n_tensors] global amax fetched for the quantiser
    int32_t *d_nv_contrib = nullptr, *d_nv_tensor_dev = nullptr;
    struct NvLocal { int32_t tid, dst_rank; int64_t tscale_off; };
    NvLocal *d_nv_local = nullptr;
    unsigned long long *d_nv_done = nullptr;
    int64_t nv_table_off = -1;         // this plan's region of the comm's amax table (byte offset)
    llrl_comm *own_comm = nullptr;     // library-owned comm of a one-device NVFP4 plan called with comm = NULL
    std::vector<char> src_touched, dst_touched;   // ranks this device's items read / write
    bool touched_valid = false;
    bool has_mc = false;
    std::vector<TmaPiece> tma_pieces;
    std::vector<int> signal_devices;   // devices this device writes into (excl. itself)
    int n_senders_in = 0;              // other devices writing into this device
    // layer groups: items [cast_off[g], cast_off[g+1]) and [fp8_off[g], fp8_off[g+1])
    std::vector<int64_t> cast_off, fp8_off;
    std::vector<std::vector<int>> group_signal;   // per group: devices written (excl. itself)
    std::vector<int> group_senders_in;            // per group: other devices writing here
    std::vector<int> senders;                     // devices writing here (whole sync)
    std::vector<std::vector<int>> group_senders;  // per group
    // pull items (multi-source fp8 blocks) read peers' trainer buffers: in
    // llrl_sync_host those peers announce "group g staged" (src-ready counters)
    std::vector<std::vector<int>> pull_from;      // per group: devices this device reads from
    std::vector<std::vector<int>> pull_to;        // per group: devices that read from this device
    int64_t hbm_read = 0, hbm_write = 0, nvl_tx = 0, nvl_rx = 0;
    int64_t nv_amax_read = 0;          // NVFP4 two-pass: bytes the amax pre-pass re-reads (not algorithmic)
    // device-side state (lazily created by the runtime)
    int uploaded_device = -1;
    Item *d_items = nullptr;
    Seg *d_segs = nullptr;
    TmaRef *d_tma_refs = nullptr;
    CastRef *d_cast_refs = nullptr;         // null: no strided cast items (or LLRL_CAST_TMAP=0)
    void *d_cast_tmaps = nullptr;           // CUtensorMap[cast_bands.size()]
    std::vector<unsigned char> h_cast_tmaps;
    int32_t *d_cast_box = nullptr;          // per band: rows per box, 0 = per-row copies
    std::vector<int32_t> h_cast_box;
    std::vector<const void *> cast_tmap_src;   // src base pointers the cast maps were encoded for
    int cast_tmap_sb = 0;                      // stage bytes the boxes were sized for
    void *d_tmaps = nullptr;                // CUtensorMap[tma_pieces.size()] (64-byte aligned)
    std::vector<unsigned char> h_tmaps;     // host copy (kept alive for the async upload)
    std::vector<const void *> tmap_src;     // src base pointers the maps were encoded for
    unsigned long long *d_done = nullptr;   // last-CTA counter (cumulative)
    unsigned long long *d_timeline = nullptr;   // LLRL_TIMELINE: per-CTA start / end of the cast launch
    unsigned int *d_queue = nullptr;            // dynamic item queue of the TMA cast launch
    double static_frac = 0.9;                   // TMA cast launches: share of items striped (rest claimed)
    int static_block = 0;                       // ... as one contiguous block per CTA instead of a stride
    int nv_run = 0;                             // NVFP4 amax pass: items per run striped over CTAs (0: one range per CTA)
    void *h2d_stream = nullptr, *d2h_stream = nullptr;   // llrl_sync_host pipeline (cudaStream_t)
    std::vector<void *> events;                           // cudaEvent_t pool for the pipeline
    int64_t n_cast = 0;                // items [0, n_cast) are K_CAST, the rest fp8
    int grid_cast = 0, grid_fp8 = 0;
    bool no_pdl = false;               // LLRL_PDL=0: plain stream order between the launches
    int variant = 0;                   // cast-kernel variant (kernels.cu)
    int max_ctas = 0;                  // grid cap (0 = all SMs); llrl_plan_set_max_ctas
    int fp8_variant = 1;               // 0: register kernel, 1: TMA pipeline
};

}  // namespace llrl

struct llrl_plan {
    int n_src, n_dst, n_devices;
    bool multicast = false;
    bool nv = false;                     // NVFP4 destination (R16)
    struct NvTensor { int32_t dst_rank, dst_param, device; int64_t tscale_off; };
    std::vector<NvTensor> nv_tensors;    // tensor id -> generator tensor
    std::vector<std::vector<llrl_nv_source>> nv_sources;   // tensor id -> trainer regions (its tiles)
    // a5: NCCL for plain replication (LLRL_PLAN_NCCL; R17, R18)
    int nccl_mode = 0;                   // 0 kernels only, 1 kernels + broadcast, 2 all-gather only
    struct NcclBcast {                   // replica 0 of a rank position -> the other replicas
        int set;                         // index in nccl_sets (its sub-communicator)
        int root_dev;
        std::vector<int> dst_rank;       // per member device (nccl_sets[set] order)
        int64_t bytes;
    };
    struct NcclGather {                  // one source parameter: F row chunks -> every replica
        int src_param;
        int64_t count;                   // elements per trainer rank
        std::vector<int64_t> src_off, dst_off;   // bytes, per FSDP rank f / replica f
    };
    std::vector<NcclBcast> nccl_bcast;
    std::vector<NcclGather> nccl_gather;
    std::vector<std::vector<int>> nccl_sets;     // distinct device sets (sorted): one sub-communicator each
    int nccl_elem_bytes = 0;
    struct NcclState {
        void *parent = nullptr;
        std::vector<void *> sub;         // per set: ncclComm_t, or null if not a member
        int rank = -1;
    };
    std::map<int, NcclState> nccl;       // per device (this process)
    int src_dtype, dst_dtype;
    std::vector<int> src_device, dst_device;
    std::vector<int64_t> src_rank_bytes, dst_rank_bytes;
    int n_groups = 0;
    bool model_with_embed = false;       // groups: 0 = embed, 1..L = layers, L+1 = final_norm + lm_head
    std::vector<std::vector<std::pair<int64_t, int64_t>>> src_group_range, dst_group_range;   // [rank][group]
    std::vector<llrl::Tile> tiles;
    std::vector<llrl::DeviceWork> dev;   // indexed by device ordinal
    std::vector<int64_t> traffic;        // G x G
    llrl_plan_stats stats;
    ~llrl_plan();
};

struct llrl_comm {
    int device;
    // 1 MiB device buffer: completion counters, expected counts and the NVFP4
    // amax table; layout in kernels.h (kSlot*, kFlag*, kNvTableOffset).
    unsigned long long *flags = nullptr;
    unsigned long long *peer_flags[llrl::kMaxDevices] = {};
    bool ipc_opened[llrl::kMaxDevices] = {};
    int64_t nv_next = -1;                // next free byte of the NVFP4 amax table (per-plan regions)
};

namespace llrl {
// nccl.cpp (a5): this device's NCCL operations of one sync on `stream`; free the plan's communicators.
llrl_status nccl_enqueue(llrl_plan *p, int device, void *const *src_ptrs, void *const *dst_ptrs, void *stream);
void nccl_destroy(llrl_plan *p);
}  // namespace llrl
