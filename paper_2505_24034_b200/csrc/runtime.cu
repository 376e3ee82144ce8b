// runtime.cu -- host runtime behind llrl_sync: device table
// upload, kernel launch, completion flags (comm), IPC mapping, the host-buffer
// end-to-end entry, and the K0 fill entry.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"
#include "kernels.h"

using namespace llrl;

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

llrl_status cuda_fail(cudaError_t e, const char *what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return LLRL_E_CUDA;
}

#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// Upload the device's work tables on first use (setup; not on the per-step path).
llrl_status ensure_uploaded(llrl_plan *p, int device) {
    DeviceWork &W = p->dev[device];
    if (W.uploaded_device == device) return LLRL_OK;
    if (!W.items.empty()) {
        CK(cudaMalloc(&W.d_items, W.items.size() * sizeof(Item)));
        CK(cudaMemcpy(W.d_items, W.items.data(), W.items.size() * sizeof(Item), cudaMemcpyHostToDevice));
    }
    if (!W.segs.empty()) {
        CK(cudaMalloc(&W.d_segs, W.segs.size() * sizeof(Seg)));
        CK(cudaMemcpy(W.d_segs, W.segs.data(), W.segs.size() * sizeof(Seg), cudaMemcpyHostToDevice));
    }
    if (!W.tma_refs.empty()) {
        CK(cudaMalloc(&W.d_tma_refs, W.tma_refs.size() * sizeof(TmaRef)));
        CK(cudaMemcpy(W.d_tma_refs, W.tma_refs.data(), W.tma_refs.size() * sizeof(TmaRef), cudaMemcpyHostToDevice));
    }
    // 3-D tensor-map boxes for strided cast sources: opt-in (LLRL_CAST_TMAP=1).
    // Measured slower than per-row bulk copies (C2 7.34 vs 6.93 ms, C12 27.94
    // vs 27.56 ms on 1 GPU), kept as the experiment's record.
    const char *ct = getenv("LLRL_CAST_TMAP");
    if (!W.cast_bands.empty() && ct && atoi(ct) != 0) {
        CK(cudaMalloc(&W.d_cast_refs, W.cast_refs.size() * sizeof(CastRef)));
        CK(cudaMemcpy(W.d_cast_refs, W.cast_refs.data(), W.cast_refs.size() * sizeof(CastRef), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&W.d_cast_tmaps, W.cast_bands.size() * 128));
        CK(cudaMalloc(&W.d_cast_box, W.cast_bands.size() * 4));
        CK(cudaMemset(W.d_cast_box, 0, W.cast_bands.size() * 4));
    }
    if (!W.tma_pieces.empty()) {
        CK(cudaMalloc(&W.d_tmaps, W.tma_pieces.size() * 128));
        W.h_tmaps.assign(W.tma_pieces.size() * 128, 0);
    }
    if (p->nv && !p->nv_tensors.empty()) {
        const size_t nt = p->nv_tensors.size();
        CK(cudaMalloc(&W.d_nv_partial, nt * 4));
        CK(cudaMalloc(&W.d_nv_amax, nt * 4));
        CK(cudaMemset(W.d_nv_amax, 0, nt * 4));
        std::vector<int32_t> tdev(nt);
        for (size_t t = 0; t < nt; t++) tdev[t] = p->nv_tensors[t].device;
        CK(cudaMalloc(&W.d_nv_tensor_dev, nt * 4));
        CK(cudaMemcpy(W.d_nv_tensor_dev, tdev.data(), nt * 4, cudaMemcpyHostToDevice));
        if (!W.nv_contrib.empty()) {
            CK(cudaMalloc(&W.d_nv_contrib, W.nv_contrib.size() * 4));
            CK(cudaMemcpy(W.d_nv_contrib, W.nv_contrib.data(), W.nv_contrib.size() * 4, cudaMemcpyHostToDevice));
        }
        if (!W.nv_local.empty()) {
            std::vector<DeviceWork::NvLocal> loc;
            for (int32_t t : W.nv_local)
                loc.push_back({t, p->nv_tensors[size_t(t)].dst_rank, p->nv_tensors[size_t(t)].tscale_off});
            CK(cudaMalloc(&W.d_nv_local, loc.size() * sizeof(DeviceWork::NvLocal)));
            CK(cudaMemcpy(W.d_nv_local, loc.data(), loc.size() * sizeof(DeviceWork::NvLocal), cudaMemcpyHostToDevice));
        }
        CK(cudaMalloc(&W.d_nv_done, 256));
        CK(cudaMemset(W.d_nv_done, 0, 256));
    }
    CK(cudaMalloc(&W.d_done, 256));
    CK(cudaMemset(W.d_done, 0, 256));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int64_t n_cast = W.n_cast, n_fp8 = int64_t(W.items.size()) - W.n_cast;
    // Cast kernel: TMA-staged (G->S->G bulk copies, local or peer) by default --
    // with its dedicated storer warp it matched or beat the register kernel on
    // every HBM- and NVLink-bound config measured (profiles/r01_y_bench_*).
    // Quantising plans (MX / NVFP4) take the 16 KiB-stage variant with two CTAs
    // per SM: their workers are instruction-bound and the second CTA hides the
    // per-chunk setup (C7/C10/C11: 2-3% faster, profiles/r01_var_*); plain
    // casts keep one CTA with 32 KiB stages (C2: 2.5% faster).
    bool has_mx = false;
    for (const Item &it : W.items)
        if (it.flags & F_MX) { has_mx = true; break; }
    W.variant = has_mx ? kCastTmaVariant + 1 : kDefaultCastVariant;
    // Tiny syncs (< 64 MB of cast source on this device, e.g. C1) are latency-bound:
    // the register kernel starts moving bytes sooner than the TMA pipeline
    // (C1: 15.4 vs 18.8 us per sync; profiles/r01_final/c1v_*).
    if (!has_mx) {
        const int64_t es = p->src_dtype == LLRL_F32 ? 4 : 2;
        int64_t bytes = 0;
        for (int64_t i = 0; i < n_cast; i++) bytes += int64_t(W.items[size_t(i)].rows) * W.items[size_t(i)].cols * es;
        if (bytes < (int64_t(64) << 20)) W.variant = 1;
    }
    if (const char *v = getenv("LLRL_CAST_VARIANT")) W.variant = atoi(v);   // tuning knob
    if (has_mx && W.variant < kCastTmaVariant) W.variant = kCastTmaVariant + 1;   // MX: TMA kernels only
    // multicast: register kernel (multimem.st); LLRL_MC_TMA=1 keeps the TMA kernel,
    // whose storer bulk-stores F_MC stages through the multicast VA
    const char *mct = getenv("LLRL_MC_TMA");
    if (W.has_mc && !(mct && atoi(mct)) && (W.variant < 0 || W.variant >= kCastTmaVariant)) W.variant = 1;
    if (W.variant < 0 || W.variant >= num_cast_variants()) W.variant = kDefaultCastVariant;
    W.fp8_variant = 1;                                                       // TMA pipeline
    if (const char *v = getenv("LLRL_PDL")) W.no_pdl = atoi(v) == 0;
    if (const char *v = getenv("LLRL_FP8_VARIANT")) W.fp8_variant = std::min(std::max(atoi(v), 0), 3);
    for (int mode = 0; mode < 2; mode++) {
        int per_sm = 0;
        CK(sync_occupancy(mode, mode == 0 ? W.variant : W.fp8_variant, p->src_dtype == LLRL_F32, &per_sm));
        if (per_sm < 1) per_sm = 1;
        const int64_t n = mode == 0 ? n_cast : n_fp8;
        int64_t cap = int64_t(sms) * per_sm;
        if (W.max_ctas > 0) cap = std::min<int64_t>(cap, W.max_ctas);           // llrl_plan_set_max_ctas
        const int g = int(std::min<int64_t>(cap, std::max<int64_t>(1, n)));
        (mode == 0 ? W.grid_cast : W.grid_fp8) = g;
    }
    CK(cudaMalloc(&W.d_queue, 256));
    CK(cudaMemset(W.d_queue, 0, 256));
    // Item order of the TMA cast launch (kernels.cu ItemWalk): the first
    // static_frac of a launch's items striped over the CTAs, the rest claimed
    // dynamically.  Striped items need no hand-off (each role reads the plan
    // table itself); the claimed tail lets every CTA finish together whatever
    // its SM's speed.  Measured (profiles/r02/ab/): with
    // pushes to peer GPUs, all claimed (C3 13.13 vs 13.88 ms at 0.9 striped, C8
    // 29.24 vs 30.66, C2 11.20 vs 11.43 at 4 GPUs: a CTA's share of each link
    // follows the plan's interleave, whatever the per-link speeds); local-only
    // syncs: 0.9 (C3 21.5 vs 22.2 ms fully striped, C10 16.2 vs 16.5), and
    // plans with an fp8 launch behind the cast launch (C4) run 7% faster fully
    // striped -- CTAs that finish early hand their SM to the programmatically
    // dependent fp8 grid.
    // Quantising syncs that push but are HBM-bound (the device's plan bytes over
    // the HBM rate exceed its NVLink bytes over the peer-copy rate; C12 at 2 and
    // 4 GPUs: 2.6 GB over NVLink, 43 GB through HBM per GPU at 4) keep the
    // local-only order: 13.03 vs 13.91 ms all claimed at 4 GPUs, supplied amax
    // 7.96 vs 8.80 (profiles/r02/ab/c12_4gpu_order.txt); NVLink-bound syncs
    // lose with it (C3 at 4 GPUs 13.63 vs 13.14 ms) and plain casts that push
    // keep claiming (C3 at 2 GPUs, HBM-bound: 20.92 ms claimed).
    bool pushes_remote = false;
    for (int64_t i = 0; i < n_cast && !pushes_remote; i++)
        pushes_remote = p->dst_device[size_t(W.items[size_t(i)].dst_rank)] != device;
    const double t_nvl = double(std::max(W.nvl_tx, W.nvl_rx)) / 770e9,
                 t_hbm = double(W.hbm_read + W.hbm_write) / 6533e9;   // measured peer copy / HBM copy rates
    const bool nvlink_bound = pushes_remote && t_nvl > t_hbm;
    W.static_frac = (pushes_remote && (nvlink_bound || !has_mx)) ? 0.0 : n_fp8 > 0 ? 1.0 : 0.9;
    // Static items of quantising (MX / NVFP4) plans as one contiguous block per
    // CTA: consecutive items then share their generator tensor and tile (fewer
    // NVFP4 table rebuilds, each a barrier across the workers): C7 / C10 / C11 /
    // C12 1-2% faster at 1 GPU, while plain casts lose 0.8% (C2), profiles/r02/ab/block.txt
    W.static_block = has_mx ? 1 : 0;
    if (const char *v = getenv("LLRL_STATIC_FRAC")) W.static_frac = std::min(1.0, std::max(0.0, atof(v)));
    if (const char *v = getenv("LLRL_STATIC_BLOCK")) W.static_block = atoi(v) != 0;
    // NVFP4 amax pass: one contiguous item range per CTA, or -- when quantised
    // sources arrive as strided rows (FSDP chunks into column-split tensors,
    // C12) -- runs of 32 items striped over the CTAs, so that no CTA's range is
    // heavy in the slower strided rows (kernels.cu llrl_k_nv_amax): C12's amax
    // pass 2.6% faster, its sync 0.8%, while contiguous plans (C11) lose 0.8%
    // with runs (profiles/r02/ab/nv_amax_runs.txt).  LLRL_NV_RUN=k overrides.
    W.nv_run = 0;
    for (int64_t i = 0; i < n_cast; i++) {
        const Item &it = W.items[size_t(i)];
        if ((it.flags & F_NV) && it.rows > 1 && it.cols != it.src_ld) { W.nv_run = 32; break; }
    }
    if (const char *v = getenv("LLRL_NV_RUN")) W.nv_run = std::max(0, atoi(v));
    if (const char *v = getenv("LLRL_TIMELINE"))
        if (atoi(v) && W.grid_cast > 0) {
            CK(cudaMalloc(&W.d_timeline, size_t(W.grid_cast) * 16));
            CK(cudaMemset(W.d_timeline, 0, size_t(W.grid_cast) * 16));
        }
    W.uploaded_device = device;
    return LLRL_OK;
}

typedef CUresult (*PFN_encode_tiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                     const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// (Re-)encode the device's TMA tensor maps when the trainer base pointers
// change (first sync, or new buffers): one 2-D map per trainer piece read by
// fp8 blocks, box 128x128 elements; uploaded on the sync stream.
llrl_status ensure_tmaps(llrl_plan *p, DeviceWork &W, void *const *src_ptrs, cudaStream_t s) {
    if (W.tma_pieces.empty()) return LLRL_OK;
    bool same = W.tmap_src.size() == size_t(p->n_src);
    for (int r = 0; same && r < p->n_src; r++) same = W.tmap_src[size_t(r)] == src_ptrs[r];
    if (same) return LLRL_OK;
    static PFN_encode_tiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) { set_error("cuTensorMapEncodeTiled unavailable"); return LLRL_E_CUDA; }
        encode = reinterpret_cast<PFN_encode_tiled>(fn);
    }
    const int64_t es = dtype_bytes(p->src_dtype);
    for (size_t m = 0; m < W.tma_pieces.size(); m++) {
        const TmaPiece &tp = W.tma_pieces[m];
        void *base = static_cast<char *>(src_ptrs[tp.src_rank]) + tp.byte_off;
        const cuuint64_t dims[2] = {cuuint64_t(tp.cols), cuuint64_t(tp.rows)};
        const cuuint64_t strides[1] = {cuuint64_t(tp.cols * es)};
        const cuuint32_t box[2] = {128, 128}, estr[2] = {1, 1};
        CUresult r = encode(reinterpret_cast<CUtensorMap *>(W.h_tmaps.data() + 128 * m),
                            es == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d) for piece %zu", int(r), m); return LLRL_E_CUDA; }
    }
    CK(cudaMemcpyAsync(W.d_tmaps, W.h_tmaps.data(), W.h_tmaps.size(), cudaMemcpyHostToDevice, s));
    W.tmap_src.assign(src_ptrs, src_ptrs + p->n_src);
    return LLRL_OK;
}

// (Re-)encode the 3-D tensor maps of the strided cast bands (plan.cpp
// make_cast_refs) when the trainer base pointers or the kernel's stage size
// change.  A band is viewed as [rows][n1][b0] 8-byte units (b0 <= 256, n1 <= 256:
// TMA box dimensions), box = [rows per stage][n1][b0] -- in shared memory the
// same bytes as the packed rows.  Bands that do not fit a stage stay on per-row
// copies (their refs are cleared on the device copy).
llrl_status ensure_cast_tmaps(llrl_plan *p, DeviceWork &W, void *const *src_ptrs, int stage_bytes, cudaStream_t s) {
    if (W.cast_bands.empty() || !W.d_cast_refs) return LLRL_OK;
    bool same = W.cast_tmap_sb == stage_bytes && W.cast_tmap_src.size() == size_t(p->n_src);
    for (int r = 0; same && r < p->n_src; r++) same = W.cast_tmap_src[size_t(r)] == src_ptrs[r];
    if (same) return LLRL_OK;
    static PFN_encode_tiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) { set_error("cuTensorMapEncodeTiled unavailable"); return LLRL_E_CUDA; }
        encode = reinterpret_cast<PFN_encode_tiled>(fn);
    }
    W.h_cast_tmaps.assign(W.cast_bands.size() * 128, 0);
    std::vector<int32_t> box_rows_of(W.cast_bands.size(), 0);   // 0: band not usable (per-row copies)
    for (size_t m = 0; m < W.cast_bands.size(); m++) {
        const CastBand &b = W.cast_bands[m];
        CUtensorMap *tm = reinterpret_cast<CUtensorMap *>(W.h_cast_tmaps.data() + 128 * m);
        const int64_t units = b.row_bytes / 8;
        int64_t b0 = 0;
        for (int64_t d = std::min<int64_t>(256, units); d >= 2; d--)
            if (units % d == 0 && d % 2 == 0) { b0 = d; break; }
        const int64_t n1 = b0 ? units / b0 : 0, box_rows = stage_bytes / b.row_bytes;
        void *base = static_cast<char *>(src_ptrs[b.src_rank]) + b.byte_off;
        if (b.row_bytes % 16 || b0 == 0 || n1 > 256 || box_rows < 1 || (reinterpret_cast<uintptr_t>(base) & 15)) continue;
        const cuuint64_t dims[3] = {cuuint64_t(b0), cuuint64_t(n1), cuuint64_t(b.rows)};
        const cuuint64_t strides[2] = {cuuint64_t(b0 * 8), cuuint64_t(b.ld_bytes)};
        const cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(n1), cuuint32_t(std::min<int64_t>(256, box_rows))},
                         estr[3] = {1, 1, 1};
        CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d) for cast band %zu", int(r), m); return LLRL_E_CUDA; }
        box_rows_of[m] = int32_t(std::min<int64_t>(256, box_rows));
    }
    W.h_cast_box = box_rows_of;
    CK(cudaMemcpyAsync(W.d_cast_tmaps, W.h_cast_tmaps.data(), W.h_cast_tmaps.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(W.d_cast_box, W.h_cast_box.data(), W.h_cast_box.size() * 4, cudaMemcpyHostToDevice, s));
    W.cast_tmap_src.assign(src_ptrs, src_ptrs + p->n_src);
    W.cast_tmap_sb = stage_bytes;
    return LLRL_OK;
}

// Which ranks a device's items touch (pointer validation); computed once.
void touched_ranks(const llrl_plan *p, DeviceWork &W) {
    if (W.touched_valid) return;
    W.src_touched.assign(size_t(p->n_src), 0);
    W.dst_touched.assign(size_t(p->n_dst), 0);
    for (int32_t tid : W.nv_local)   // NVFP4: the fp32 tensor scale is written on the holder's device
        W.dst_touched[size_t(p->nv_tensors[size_t(tid)].dst_rank)] = 1;
    for (const Item &it : W.items) {
        if (it.kind == K_FP8_MULTI) {
            for (int s = 0; s < it.src_rank; s++) W.src_touched[size_t(W.segs[size_t(it.src_off) + s].src_rank)] = 1;
        } else {
            W.src_touched[it.src_rank] = 1;
        }
        if (!(it.flags & F_MC)) W.dst_touched[it.dst_rank] = 1;   // multicast items use the MC VA
    }
    W.touched_valid = true;
}

}  // namespace

extern "C" {

// Common prologue of llrl_sync / llrl_sync_group / llrl_sync_host: validate,
// fill the pointer tables, upload on first use.
// nv_table: the NVFP4 two-pass handshake needs the comm's amax table even on one
// device; a one-device plan called with comm = NULL gets a library-owned comm.
static llrl_status prologue(llrl_plan *p, llrl_comm *&comm, int device, void *const *src_ptrs,
                            void *const *dst_ptrs, KParams *kp, bool nv_table) {
    if (!p || !src_ptrs || !dst_ptrs || device < 0 || device >= p->n_devices) {
        set_error("llrl_sync: invalid argument (device %d of %d)", device, p ? p->n_devices : 0);
        return LLRL_E_INVALID;
    }
    DeviceWork &W = p->dev[size_t(device)];
    bool cross = !W.signal_devices.empty() || W.n_senders_in > 0;
    for (size_t g = 0; g < W.pull_from.size(); g++) cross = cross || !W.pull_from[g].empty() || !W.pull_to[g].empty();
    if (nv_table) {
        bool remote = false;
        for (int d : W.nv_targets) remote = remote || d != device;
        for (int d : W.nv_senders) remote = remote || d != device;
        if (!comm && !cross && !remote) {
            if (!W.own_comm) {
                llrl_status st = llrl_comm_create(device, &W.own_comm);
                if (st != LLRL_OK) return st;
            }
            comm = W.own_comm;
        }
        cross = cross || remote || !comm;
    }
    if (cross) {
        if (!comm || comm->device != device) {
            set_error("llrl_sync: device %d exchanges data with peers and needs its comm", device);
            return LLRL_E_NOPEER;
        }
        for (int d : W.signal_devices)
            if (!comm->peer_flags[d]) {
                set_error("llrl_sync: no flag mapping for peer device %d", d);
                return LLRL_E_NOPEER;
            }
    }
    touched_ranks(p, W);
    const std::vector<char> &su = W.src_touched, &du = W.dst_touched;
    std::memset(kp, 0, sizeof *kp);
    for (int r = 0; r < p->n_src; r++) {
        if (su[size_t(r)] && !src_ptrs[r]) { set_error("llrl_sync: src_ptrs[%d] is NULL", r); return LLRL_E_NOPEER; }
        kp->src[r] = src_ptrs[r];
    }
    for (int g = 0; g < p->n_dst; g++) {
        if (du[size_t(g)] && !dst_ptrs[g]) { set_error("llrl_sync: dst_ptrs[%d] is NULL", g); return LLRL_E_NOPEER; }
        kp->dst[g] = dst_ptrs[g];
    }
    llrl_status st = ensure_uploaded(p, device);
    if (st != LLRL_OK) return st;
    if (W.has_mc) {
        if (W.dst_mc.size() != size_t(p->n_dst)) {
            set_error("llrl_sync: device %d multicasts but llrl_plan_set_multicast was not called", device);
            return LLRL_E_NOPEER;
        }
        for (int g = 0; g < p->n_dst; g++) kp->dst_mc[g] = W.dst_mc[size_t(g)];
    }
    kp->items = W.d_items;
    kp->segs = W.d_segs;
    kp->nv_amax = W.d_nv_amax;
    kp->tma_refs = W.d_tma_refs;
    kp->tmaps = W.d_tmaps;
    kp->fp8_base = int(W.n_cast);
    return LLRL_OK;
}

// Enqueue cast items [c0, c1) and fp8 items [f0, f1); the last launch signals
// every device in `sig` (its last CTA, after all CTAs' stores are fenced).
// Every device table ensure_uploaded allocates (plan destroy, re-upload).
static void free_device_tables(DeviceWork &W) {
    void **ptrs[] = {reinterpret_cast<void **>(&W.d_items), reinterpret_cast<void **>(&W.d_segs),
                     reinterpret_cast<void **>(&W.d_done), reinterpret_cast<void **>(&W.d_tma_refs),
                     reinterpret_cast<void **>(&W.d_tmaps), reinterpret_cast<void **>(&W.d_nv_partial),
                     reinterpret_cast<void **>(&W.d_nv_amax), reinterpret_cast<void **>(&W.d_nv_contrib),
                     reinterpret_cast<void **>(&W.d_nv_tensor_dev), reinterpret_cast<void **>(&W.d_nv_local),
                     reinterpret_cast<void **>(&W.d_nv_done), reinterpret_cast<void **>(&W.d_timeline),
                     reinterpret_cast<void **>(&W.d_queue), reinterpret_cast<void **>(&W.d_cast_refs),
                     reinterpret_cast<void **>(&W.d_cast_tmaps), reinterpret_cast<void **>(&W.d_cast_box)};
    for (void **q : ptrs) {
        cudaFree(*q);
        *q = nullptr;
    }
}

static llrl_status launch_ranges(llrl_plan *p, DeviceWork &W, llrl_comm *comm, KParams &kp, int64_t c0, int64_t c1,
                                 int64_t f0, int64_t f1, const std::vector<int> &sig, cudaStream_t s) {
    const bool has_fp8 = f1 > f0;
    if (has_fp8 && W.fp8_variant >= 1) {
        llrl_status st = ensure_tmaps(p, W, const_cast<void *const *>(kp.src), s);
        if (st != LLRL_OK) return st;
    }
    if (c1 > c0 && W.d_cast_refs && W.variant >= kCastTmaVariant) {
        llrl_status st = ensure_cast_tmaps(p, W, const_cast<void *const *>(kp.src), cast_stage_bytes(W.variant), s);
        if (st != LLRL_OK) return st;
    }
    for (int mode = 0; mode < 2; mode++) {
        const int64_t b = mode == 0 ? c0 : f0, e = mode == 0 ? c1 : f1;
        if (e <= b) continue;
        const bool last = mode == 1 || !has_fp8;
        const int grid = int(std::min<int64_t>(mode == 0 ? W.grid_cast : W.grid_fp8, e - b));
        kp.item_begin = int(b);
        kp.item_end = int(e);
        kp.done = nullptr;
        kp.n_signal = 0;
        if (last && !sig.empty()) {
            kp.done = W.d_done;
            kp.n_signal = int(sig.size());
            for (int i = 0; i < kp.n_signal; i++) kp.signal[i] = comm->peer_flags[sig[size_t(i)]] + comm->device;
        }
        kp.pdl_wait = (mode == 1 && c1 > c0 && !W.no_pdl) ? 1 : 0;   // fp8 launch overlaps the cast tail
        kp.timeline = mode == 0 ? W.d_timeline : nullptr;
        kp.static_end = int(e);
        kp.static_block = 0;
        kp.queue = nullptr;
        kp.cast_refs = nullptr;
        if (mode == 0 && W.variant >= kCastTmaVariant && W.d_cast_refs) {
            kp.cast_refs = W.d_cast_refs;
            kp.cast_tmaps = W.d_cast_tmaps;
            kp.cast_box = W.d_cast_box;
        }
        if (mode == 0 && W.variant >= kCastTmaVariant) {
            kp.static_end = int(b + int64_t(W.static_frac * double(e - b)));
            kp.static_block = W.static_block;
            if (kp.static_end < e) kp.queue = W.d_queue;
        }
        CK(launch_sync(kp, mode, mode == 0 ? W.variant : W.fp8_variant, p->src_dtype == LLRL_F32, grid, s));
        kp.pdl_wait = 0;
    }
    return LLRL_OK;
}

// One arrival is expected in slot base + d for every device d in `devs`.
static llrl_status wait_arrivals(llrl_comm *comm, const std::vector<int> &devs, cudaStream_t s, int base = 0) {
    if (devs.empty()) return LLRL_OK;
    WaitTargets t;
    std::memset(&t, 0, sizeof t);
    for (int d : devs) t.count[base + d] = 1;
    CK(launch_wait(comm->flags, t, s));
    return LLRL_OK;
}

// NVFP4 (R16) per-tensor amax handshake (see kernels.cu): partials -> owners,
// owners reduce and publish, contributors fetch; all device-side, stream-ordered.
// Each plan has its own table region (assigned on its first sync on a comm, in
// the same order on every process -- the same-sequence rule of llrl.h).
static uint32_t *nv_table(llrl_comm *comm, int dev, const DeviceWork &W) {
    return reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(comm->peer_flags[dev]) + W.nv_table_off);
}

static llrl_status nv_handshake(llrl_plan *p, DeviceWork &W, llrl_comm *comm, int device, const KParams &kp,
                                cudaStream_t s) {
    if (W.nv_table_off < 0) {
        const int64_t need = (int64_t(p->nv_tensors.size()) * kNvTableStride * 4 + 255) / 256 * 256;
        if (comm->nv_next < 0) comm->nv_next = kNvTableOffset;
        if (comm->nv_next + need > kCommBytes) {
            set_error("NVFP4: %zu generator tensors exceed the comm's free amax table space", p->nv_tensors.size());
            return LLRL_E_UNSUPPORTED;
        }
        W.nv_table_off = comm->nv_next;
        comm->nv_next += need;
    }
    for (int d : W.nv_targets)
        if (!comm->peer_flags[d]) { set_error("NVFP4: no comm mapping for device %d", d); return LLRL_E_NOPEER; }
    for (int d : W.nv_senders)
        if (!comm->peer_flags[d]) { set_error("NVFP4: no comm mapping for device %d", d); return LLRL_E_NOPEER; }
    if (!W.nv_contrib.empty()) {
        NvAmaxParams a;
        std::memset(&a, 0, sizeof a);
        a.items = W.d_items;
        a.n_items = int(W.n_cast);
        a.run = W.nv_run;
        a.partial = W.d_nv_partial;
        a.done = W.d_nv_done;
        a.contrib = W.d_nv_contrib;
        a.n_contrib = int(W.nv_contrib.size());
        a.tensor_dev = W.d_nv_tensor_dev;
        for (int d = 0; d < p->n_devices; d++)
            if (comm->peer_flags[d]) a.tables[d] = nv_table(comm, d, W);
        a.my_dev = device;
        a.n_signal = int(W.nv_targets.size());
        for (int i = 0; i < a.n_signal; i++) a.signal[i] = comm->peer_flags[W.nv_targets[size_t(i)]] + kSlotNvAmax + device;
        for (int r = 0; r < p->n_src; r++) a.src[r] = kp.src[r];
        CK(cudaMemsetAsync(W.d_nv_partial, 0, p->nv_tensors.size() * 4, s));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(sms), W.n_cast)));   // 1 CTA / SM
        CK(launch_nv_amax(a, p->src_dtype == LLRL_F32, grid, s));
    }
    if (!W.nv_local.empty()) {
        llrl_status st = wait_arrivals(comm, W.nv_senders, s, kSlotNvAmax);
        if (st != LLRL_OK) return st;
        NvScaleParams c;
        std::memset(&c, 0, sizeof c);
        c.locals = W.d_nv_local;
        c.n_local = int(W.nv_local.size());
        c.table = nv_table(comm, device, W);
        for (int g = 0; g < p->n_dst; g++) c.dst[g] = kp.dst[g];
        c.n_signal = int(W.nv_senders.size());
        for (int i = 0; i < c.n_signal; i++) c.signal[i] = comm->peer_flags[W.nv_senders[size_t(i)]] + kSlotNvReady + device;
        CK(launch_nv_scale(c, s));
    }
    if (!W.nv_contrib.empty()) {
        llrl_status st = wait_arrivals(comm, W.nv_targets, s, kSlotNvReady);
        if (st != LLRL_OK) return st;
        NvFetchParams f;
        std::memset(&f, 0, sizeof f);
        f.contrib = W.d_nv_contrib;
        f.n_contrib = int(W.nv_contrib.size());
        f.tensor_dev = W.d_nv_tensor_dev;
        for (int d = 0; d < p->n_devices; d++)
            if (comm->peer_flags[d]) f.tables[d] = nv_table(comm, d, W);
        f.amax_out = W.d_nv_amax;
        CK(launch_nv_fetch(f, s));
    }
    return LLRL_OK;
}

static llrl_status sync_body(llrl_plan *p, llrl_comm *comm, int device, KParams &kp, cudaStream_t s);

llrl_status llrl_sync(llrl_plan *p, llrl_comm *comm, int device, void *const *src_ptrs, void *const *dst_ptrs,
                      void *stream) {
    DeviceGuard guard(device >= 0 ? device : 0);
    KParams kp;
    llrl_status st = prologue(p, comm, device, src_ptrs, dst_ptrs, &kp, p && p->nv);
    if (st != LLRL_OK) return st;
    st = sync_body(p, comm, device, kp, static_cast<cudaStream_t>(stream));
    if (st != LLRL_OK) return st;
    // a5: replicas by ncclBroadcast once replica 0 is complete here (stream order
    // after the completion wait), or the whole sync as ncclAllGathers (R17, R18)
    return nccl_enqueue(p, device, src_ptrs, dst_ptrs, stream);
}

// The whole-sync launch sequence (llrl_sync; llrl_sync_host for NVFP4).
static llrl_status sync_body(llrl_plan *p, llrl_comm *comm, int device, KParams &kp, cudaStream_t s) {
    llrl_status st = LLRL_OK;
    DeviceWork &W = p->dev[size_t(device)];
    if (p->nv) {
        st = nv_handshake(p, W, comm, device, kp, s);
        if (st != LLRL_OK) return st;
    }
    st = launch_ranges(p, W, comm, kp, 0, W.n_cast, W.n_cast, int64_t(W.items.size()), W.signal_devices, s);
    if (st != LLRL_OK) return st;
    return wait_arrivals(comm, W.senders, s);
}

// ---- NVFP4 with a caller-supplied tensor amax (one pass) ----------------------

llrl_status llrl_plan_nv_num_tensors(const llrl_plan *p, int *n) {
    if (!p || !n) { set_error("NULL argument"); return LLRL_E_INVALID; }
    *n = int(p->nv_tensors.size());
    return LLRL_OK;
}

llrl_status llrl_plan_nv_tensor(const llrl_plan *p, int tid, llrl_nv_tensor *out) {
    if (!p || !out || tid < 0 || size_t(tid) >= p->nv_tensors.size()) {
        set_error("llrl_plan_nv_tensor: invalid argument");
        return LLRL_E_INVALID;
    }
    const llrl_plan::NvTensor &t = p->nv_tensors[size_t(tid)];
    out->dst_rank = t.dst_rank;
    out->dst_param = t.dst_param;
    out->device = t.device;
    out->n_sources = int32_t(p->nv_sources[size_t(tid)].size());
    return LLRL_OK;
}

llrl_status llrl_plan_nv_tensor_sources(const llrl_plan *p, int tid, int first, int count, llrl_nv_source *out) {
    if (!p || tid < 0 || size_t(tid) >= p->nv_tensors.size() || first < 0 || count < 0 || (count && !out) ||
        size_t(first) + size_t(count) > p->nv_sources[size_t(tid)].size()) {
        set_error("llrl_plan_nv_tensor_sources: invalid argument");
        return LLRL_E_INVALID;
    }
    std::copy(p->nv_sources[size_t(tid)].begin() + first, p->nv_sources[size_t(tid)].begin() + first + count, out);
    return LLRL_OK;
}

llrl_status llrl_sync_nv_amax(llrl_plan *p, llrl_comm *comm, int device, const float *amax_dev,
                              void *const *src_ptrs, void *const *dst_ptrs, void *stream) {
    if (!p || !p->nv || !amax_dev) { set_error("llrl_sync_nv_amax: needs an NVFP4 plan and an amax array"); return LLRL_E_INVALID; }
    DeviceGuard guard(device >= 0 ? device : 0);
    KParams kp;
    llrl_status st = prologue(p, comm, device, src_ptrs, dst_ptrs, &kp, false);
    if (st != LLRL_OK) return st;
    DeviceWork &W = p->dev[size_t(device)];
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    kp.nv_amax = reinterpret_cast<const uint32_t *>(amax_dev);
    if (!W.nv_local.empty()) {
        NvTscaleParams t;
        std::memset(&t, 0, sizeof t);
        t.locals = W.d_nv_local;
        t.n_local = int(W.nv_local.size());
        t.amax = kp.nv_amax;
        for (int g = 0; g < p->n_dst; g++) t.dst[g] = kp.dst[g];
        CK(launch_nv_tscale(t, s));
    }
    st = launch_ranges(p, W, comm, kp, 0, W.n_cast, W.n_cast, int64_t(W.items.size()), W.signal_devices, s);
    if (st != LLRL_OK) return st;
    return wait_arrivals(comm, W.senders, s);
}

llrl_status llrl_plan_num_groups(const llrl_plan *p, int *n) {
    if (!p || !n) { set_error("NULL argument"); return LLRL_E_INVALID; }
    *n = p->n_groups;
    return LLRL_OK;
}

llrl_status llrl_plan_set_max_ctas(llrl_plan *p, int device, int max_ctas) {
    if (!p || device < 0 || device >= p->n_devices || max_ctas < 0) { set_error("invalid argument"); return LLRL_E_INVALID; }
    DeviceWork &W = p->dev[size_t(device)];
    W.max_ctas = max_ctas;
    if (W.uploaded_device >= 0) {           // re-upload (grid sizes) at the next sync
        DeviceGuard guard(W.uploaded_device);
        free_device_tables(W);
        W.tmap_src.clear();
        W.cast_tmap_src.clear();
        W.uploaded_device = -1;
    }
    return LLRL_OK;
}

llrl_status llrl_plan_group_range(const llrl_plan *p, int side, int rank, int group, int64_t *lo, int64_t *hi) {
    if (!p || !lo || !hi || group < 0 || group >= p->n_groups || (side != 0 && side != 1) || rank < 0 ||
        rank >= (side == 0 ? p->n_src : p->n_dst)) {
        set_error("llrl_plan_group_range: invalid argument");
        return LLRL_E_INVALID;
    }
    const auto &r = (side == 0 ? p->src_group_range : p->dst_group_range)[size_t(rank)][size_t(group)];
    *lo = r.first;
    *hi = r.second;
    return LLRL_OK;
}

llrl_status llrl_sync_group(llrl_plan *p, llrl_comm *comm, int device, int group, void *const *src_ptrs,
                            void *const *dst_ptrs, void *stream) {
    if (!p || group < 0 || group >= p->n_groups) { set_error("llrl_sync_group: invalid group"); return LLRL_E_INVALID; }
    if (p->nv) { set_error("llrl_sync_group: NVFP4 needs whole-tensor amax -- use llrl_sync"); return LLRL_E_UNSUPPORTED; }
    if (p->nccl_mode) { set_error("llrl_sync_group: NCCL replication is per rank buffer -- use llrl_sync"); return LLRL_E_UNSUPPORTED; }
    DeviceGuard guard(device >= 0 ? device : 0);
    KParams kp;
    llrl_status st = prologue(p, comm, device, src_ptrs, dst_ptrs, &kp, false);
    if (st != LLRL_OK) return st;
    DeviceWork &W = p->dev[size_t(device)];
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t g = size_t(group);
    st = launch_ranges(p, W, comm, kp, W.cast_off[g], W.cast_off[g + 1], W.fp8_off[g], W.fp8_off[g + 1],
                       W.group_signal[g], s);
    if (st != LLRL_OK) return st;
    return wait_arrivals(comm, W.group_senders[g], s);
}

llrl_status llrl_debug_timeline(const llrl_plan *p, int device, uint64_t *out, int max_ctas, int *n_ctas) {
    if (!p || !out || !n_ctas || device < 0 || device >= p->n_devices) { set_error("invalid argument"); return LLRL_E_INVALID; }
    const DeviceWork &W = p->dev[size_t(device)];
    *n_ctas = 0;
    if (!W.d_timeline) return LLRL_OK;
    DeviceGuard guard(device);
    const int n = std::min(max_ctas, W.grid_cast);
    CK(cudaMemcpy(out, W.d_timeline, size_t(n) * 16, cudaMemcpyDeviceToHost));
    *n_ctas = n;
    return LLRL_OK;
}

llrl_status llrl_sync_num_launches(const llrl_plan *p, int device, int *n) {
    if (!p || !n || device < 0 || device >= p->n_devices) { set_error("invalid argument"); return LLRL_E_INVALID; }
    const DeviceWork &W = p->dev[device];
    *n = (W.n_cast > 0 ? 1 : 0) + (int64_t(W.items.size()) > W.n_cast ? 1 : 0) + (W.n_senders_in > 0 ? 1 : 0);
    if (p->nv)   // amax, scale (+ wait), fetch (+ wait)
        *n += (W.nv_contrib.empty() ? 0 : 3) + (W.nv_local.empty() ? 0 : 2);
    return LLRL_OK;
}

llrl_status llrl_plan_device_info(const llrl_plan *p, int device, llrl_device_info *out) {
    if (!p || !out || device < 0 || device >= p->n_devices) { set_error("invalid argument"); return LLRL_E_INVALID; }
    const DeviceWork &W = p->dev[device];
    std::memset(out, 0, sizeof *out);
    out->n_items = int64_t(W.items.size());
    out->n_cast_items = W.n_cast;
    out->n_fp8_items = out->n_items - W.n_cast;
    for (const Item &it : W.items) out->n_fp8_pull_items += it.kind == K_FP8_MULTI;
    out->n_signal = int32_t(W.signal_devices.size());
    out->n_senders_in = W.n_senders_in;
    out->nv_amax_read_bytes = W.nv_amax_read;
    return llrl_sync_num_launches(p, device, &out->n_launches);
}

// Host-buffer entry: per layer group, H2D of the group's trainer bytes (copy
// stream) -> the group's kernels (+ completion) on `stream` -> D2H of the
// group's generator bytes (second copy stream), so PCIe traffic in both
// directions overlaps the kernels of neighbouring groups.
llrl_status llrl_sync_host(llrl_plan *p, llrl_comm *comm, int device, const void *const *host_src,
                           void *const *host_dst, void *const *src_ptrs, void *const *dst_ptrs, void *stream) {
    if (!host_src || !host_dst) { set_error("llrl_sync_host: invalid argument"); return LLRL_E_INVALID; }
    if (p && p->nccl_mode) { set_error("llrl_sync_host: not for LLRL_PLAN_NCCL plans -- use llrl_sync"); return LLRL_E_UNSUPPORTED; }
    DeviceGuard guard(device >= 0 ? device : 0);
    KParams kp;
    llrl_status st = prologue(p, comm, device, src_ptrs, dst_ptrs, &kp, p && p->nv);
    if (st != LLRL_OK) return st;
    DeviceWork &W = p->dev[size_t(device)];
    const int G = p->n_groups;
    if (!W.h2d_stream) {
        cudaStream_t a, b;
        CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        W.h2d_stream = a;
        W.d2h_stream = b;
        W.events.resize(size_t(2 * G + 2));
        for (auto &e : W.events) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            e = ev;
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaStream_t h2d = static_cast<cudaStream_t>(W.h2d_stream), d2h = static_cast<cudaStream_t>(W.d2h_stream);
    auto ev = [&](size_t i) { return static_cast<cudaEvent_t>(W.events[i]); };
    // copies must not overtake work already queued on `stream` (previous sync)
    CK(cudaEventRecord(ev(size_t(2 * G)), s));
    CK(cudaStreamWaitEvent(h2d, ev(size_t(2 * G)), 0));
    CK(cudaStreamWaitEvent(d2h, ev(size_t(2 * G)), 0));
    if (p->nv) {
        // NVFP4 (R16): a tensor's scale needs its whole amax, so no per-group
        // pipelining: every trainer byte in, the whole sync, every generator byte out
        for (int r = 0; r < p->n_src; r++)
            if (p->src_device[size_t(r)] == device && host_src[r])
                CK(cudaMemcpyAsync(src_ptrs[r], host_src[r], size_t(p->src_rank_bytes[size_t(r)]),
                                   cudaMemcpyHostToDevice, s));
        st = sync_body(p, comm, device, kp, s);
        if (st != LLRL_OK) return st;
        for (int q = 0; q < p->n_dst; q++)
            if (p->dst_device[size_t(q)] == device && host_dst[q])
                CK(cudaMemcpyAsync(host_dst[q], dst_ptrs[q], size_t(p->dst_rank_bytes[size_t(q)]),
                                   cudaMemcpyDeviceToHost, s));
        return LLRL_OK;
    }
    // Group order: the first group's H2D and the last group's D2H are not
    // overlapped with anything, so the (large) embedding and lm_head groups go
    // to the middle of the pipeline and decoder layers open and close it.  Every
    // device uses the same order (per-sender arrival counts stay paired).
    std::vector<int> order;
    if (p->model_with_embed && G >= 4) {
        for (int g = 1; g < G - 1; g++) {
            order.push_back(g);
            if (g == G / 2) {
                order.push_back(0);
                order.push_back(G - 1);
            }
        }
    } else {
        for (int g = 0; g < G; g++) order.push_back(g);
    }
    for (int g : order) {
        for (int r = 0; r < p->n_src; r++) {
            const auto &rg = p->src_group_range[size_t(r)][size_t(g)];
            if (p->src_device[size_t(r)] != device || !host_src[r] || rg.first < 0) continue;
            CK(cudaMemcpyAsync(static_cast<char *>(src_ptrs[r]) + rg.first,
                               static_cast<const char *>(host_src[r]) + rg.first, size_t(rg.second - rg.first),
                               cudaMemcpyHostToDevice, h2d));
        }
        const size_t gg = size_t(g);
        if (!W.pull_to[gg].empty()) {            // peers pull this group's trainer bytes
            SignalTargets t;
            std::memset(&t, 0, sizeof t);
            for (int d : W.pull_to[gg]) {
                if (!comm || !comm->peer_flags[d]) { set_error("llrl_sync_host: no flag mapping for %d", d); return LLRL_E_NOPEER; }
                t.slot[t.n++] = comm->peer_flags[d] + kSlotStaged + device;
            }
            CK(launch_signal(t, h2d));
        }
        CK(cudaEventRecord(ev(size_t(2 * g)), h2d));
        CK(cudaStreamWaitEvent(s, ev(size_t(2 * g)), 0));
        st = wait_arrivals(comm, W.pull_from[gg], s, kSlotStaged);   // their bytes staged
        if (st != LLRL_OK) return st;
        st = launch_ranges(p, W, comm, kp, W.cast_off[gg], W.cast_off[gg + 1], W.fp8_off[gg], W.fp8_off[gg + 1],
                           W.group_signal[gg], s);
        if (st != LLRL_OK) return st;
        st = wait_arrivals(comm, W.group_senders[gg], s);
        if (st != LLRL_OK) return st;
        CK(cudaEventRecord(ev(size_t(2 * g + 1)), s));
        CK(cudaStreamWaitEvent(d2h, ev(size_t(2 * g + 1)), 0));
        for (int q = 0; q < p->n_dst; q++) {
            const auto &rg = p->dst_group_range[size_t(q)][gg];
            if (p->dst_device[size_t(q)] != device || !host_dst[q] || rg.first < 0) continue;
            CK(cudaMemcpyAsync(static_cast<char *>(host_dst[q]) + rg.first,
                               static_cast<const char *>(dst_ptrs[q]) + rg.first, size_t(rg.second - rg.first),
                               cudaMemcpyDeviceToHost, d2h));
        }
    }
    CK(cudaEventRecord(ev(size_t(2 * G + 1)), d2h));
    CK(cudaStreamWaitEvent(s, ev(size_t(2 * G + 1)), 0));
    return LLRL_OK;
}

void llrl_plan_destroy(llrl_plan *p) {
    if (!p) return;
    nccl_destroy(p);
    for (size_t d = 0; d < p->dev.size(); d++) {
        DeviceWork &W = p->dev[d];
        if (W.uploaded_device < 0) continue;
        DeviceGuard guard(W.uploaded_device);
        free_device_tables(W);
        for (void *e : W.events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
        if (W.h2d_stream) cudaStreamDestroy(static_cast<cudaStream_t>(W.h2d_stream));
        if (W.d2h_stream) cudaStreamDestroy(static_cast<cudaStream_t>(W.d2h_stream));
        if (W.own_comm) llrl_comm_destroy(W.own_comm);
    }
    delete p;
}

// ---- comm -------------------------------------------------------------------

llrl_status llrl_comm_create(int device, llrl_comm **out) {
    if (!out || device < 0 || device >= kMaxDevices) { set_error("llrl_comm_create: invalid argument"); return LLRL_E_INVALID; }
    llrl_comm *c = new (std::nothrow) llrl_comm();
    if (!c) { set_error("out of host memory"); return LLRL_E_NOMEM; }
    c->device = device;
    DeviceGuard guard(device);
    cudaError_t e = cudaMalloc(&c->flags, kCommBytes);
    if (e == cudaSuccess) e = cudaMemset(c->flags, 0, kCommBytes);
    if (e != cudaSuccess) { delete c; return cuda_fail(e, "llrl_comm_create"); }
    c->peer_flags[device] = c->flags;
    c->nv_next = kNvTableOffset;
    *out = c;
    return LLRL_OK;
}

llrl_status llrl_comm_export(const llrl_comm *c, void *handle64) {
    if (!c || !handle64) { set_error("invalid argument"); return LLRL_E_INVALID; }
    DeviceGuard guard(c->device);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->flags));
    std::memcpy(handle64, &h, sizeof h);
    return LLRL_OK;
}

llrl_status llrl_comm_import(llrl_comm *c, int peer_device, const void *handle64) {
    if (!c || !handle64 || peer_device < 0 || peer_device >= kMaxDevices) { set_error("invalid argument"); return LLRL_E_INVALID; }
    if (peer_device == c->device) return LLRL_OK;
    DeviceGuard guard(c->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    void *ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer_flags[peer_device] = static_cast<unsigned long long *>(ptr);
    c->ipc_opened[peer_device] = true;
    return LLRL_OK;
}

llrl_status llrl_comm_flag_ptr(const llrl_comm *c, void **dev_ptr) {
    if (!c || !dev_ptr) { set_error("invalid argument"); return LLRL_E_INVALID; }
    *dev_ptr = c->flags;
    return LLRL_OK;
}

llrl_status llrl_comm_set_peer(llrl_comm *c, int peer_device, void *peer_flag_dev_ptr) {
    if (!c || peer_device < 0 || peer_device >= kMaxDevices || !peer_flag_dev_ptr) { set_error("invalid argument"); return LLRL_E_INVALID; }
    if (peer_device != c->device) {
        DeviceGuard guard(c->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
    c->peer_flags[peer_device] = static_cast<unsigned long long *>(peer_flag_dev_ptr);
    return LLRL_OK;
}

llrl_status llrl_comm_timed_out(const llrl_comm *c, int *timed_out) {
    if (!c || !timed_out) { set_error("invalid argument"); return LLRL_E_INVALID; }
    DeviceGuard guard(c->device);
    unsigned long long v = 0;
    CK(cudaMemcpy(&v, c->flags + kFlagTimeout, sizeof v, cudaMemcpyDeviceToHost));
    *timed_out = v != 0;
    return LLRL_OK;
}

void llrl_comm_destroy(llrl_comm *c) {
    if (!c) return;
    DeviceGuard guard(c->device);
    for (int d = 0; d < kMaxDevices; d++)
        if (c->ipc_opened[d]) cudaIpcCloseMemHandle(c->peer_flags[d]);
    cudaFree(c->flags);
    delete c;
}

// ---- IPC for caller buffers -------------------------------------------------------

typedef CUresult (*PFN_addr_range)(CUdeviceptr *, size_t *, CUdeviceptr);

llrl_status llrl_ipc_handle(const void *dev_ptr, void *handle64, int64_t *offset) {
    if (!dev_ptr || !handle64 || !offset) { set_error("invalid argument"); return LLRL_E_INVALID; }
    static PFN_addr_range get_range = nullptr;
    if (!get_range) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) { set_error("cuMemGetAddressRange unavailable"); return LLRL_E_CUDA; }
        get_range = reinterpret_cast<PFN_addr_range>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, CUdeviceptr(dev_ptr)) != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed");
        return LLRL_E_CUDA;
    }
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    std::memcpy(handle64, &h, sizeof h);
    *offset = int64_t(CUdeviceptr(dev_ptr) - base);
    return LLRL_OK;
}

llrl_status llrl_ipc_open(const void *handle64, int64_t offset, void **dev_ptr) {
    if (!handle64 || !dev_ptr || offset < 0) { set_error("invalid argument"); return LLRL_E_INVALID; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    void *base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<char *>(base) + offset;
    return LLRL_OK;
}

llrl_status llrl_ipc_close(void *dev_ptr, int64_t offset) {
    if (!dev_ptr) { set_error("invalid argument"); return LLRL_E_INVALID; }
    CK(cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - offset));
    return LLRL_OK;
}

// ---- K0 ----------------------------------------------------------------------------

llrl_status llrl_fill_synthetic(const llrl_layout *src, int rank, void *dev_ptr, uint64_t seed, void *stream) {
    if (!src || !src->is_src || rank < 0 || rank >= src->n_ranks || !dev_ptr) {
        set_error("llrl_fill_synthetic: invalid argument");
        return LLRL_E_INVALID;
    }
    std::vector<FillPiece> fp;
    int64_t mx = 0;
    for (const Piece &pc : src->pieces[rank]) {
        if (pc.rows * pc.cols == 0) continue;
        fp.push_back(FillPiece{pc.byte_off, pc.rows, pc.cols, pc.rect.r0, pc.rect.c0, pc.param,
                               src->src_params[size_t(pc.param)].is_norm ? 1 : 0});
        mx = std::max(mx, pc.rows * pc.cols);
    }
    if (fp.empty()) return LLRL_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FillPiece *d = nullptr;
    CK(cudaMallocAsync(&d, fp.size() * sizeof(FillPiece), s));
    CK(cudaMemcpyAsync(d, fp.data(), fp.size() * sizeof(FillPiece), cudaMemcpyHostToDevice, s));
    CK(launch_fill(dev_ptr, d, int(fp.size()), mx, src->dtype == LLRL_F32, seed, s));
    CK(cudaFreeAsync(d, s));
    CK(cudaStreamSynchronize(s));   // the host vector is released on return
    return LLRL_OK;
}

}  // extern "C"
