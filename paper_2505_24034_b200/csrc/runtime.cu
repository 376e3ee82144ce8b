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
    CK(cudaMalloc(&W.d_done, 256));
    CK(cudaMemset(W.d_done, 0, 256));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int64_t n_cast = W.n_cast, n_fp8 = int64_t(W.items.size()) - W.n_cast;
    W.variant = kDefaultCastVariant;
    if (const char *v = getenv("LLRL_CAST_VARIANT")) W.variant = atoi(v);   // tuning knob
    if (W.variant < 0 || W.variant >= num_cast_variants()) W.variant = kDefaultCastVariant;
    for (int mode = 0; mode < 2; mode++) {
        int per_sm = 0;
        CK(sync_occupancy(mode, W.variant, p->src_dtype == LLRL_F32, &per_sm));
        if (per_sm < 1) per_sm = 1;
        const int64_t n = mode == 0 ? n_cast : n_fp8;
        const int g = int(std::min<int64_t>(int64_t(sms) * per_sm, std::max<int64_t>(1, n)));
        (mode == 0 ? W.grid_cast : W.grid_fp8) = g;
    }
    W.epoch = 0;
    W.uploaded_device = device;
    return LLRL_OK;
}

// Which ranks a device's items touch (for pointer validation).
void touched_ranks(const DeviceWork &W, std::vector<char> &src, std::vector<char> &dst) {
    for (const Item &it : W.items) {
        if (it.kind == K_FP8_MULTI) {
            for (int s = 0; s < it.src_rank; s++) src[size_t(W.segs[size_t(it.src_off) + s].src_rank)] = 1;
        } else {
            src[it.src_rank] = 1;
        }
        dst[it.dst_rank] = 1;
    }
}

}  // namespace

extern "C" {

llrl_status llrl_sync(llrl_plan *p, llrl_comm *comm, int device, void *const *src_ptrs, void *const *dst_ptrs,
                      void *stream) {
    if (!p || !src_ptrs || !dst_ptrs || device < 0 || device >= p->n_devices) {
        set_error("llrl_sync: invalid argument (device %d of %d)", device, p ? p->n_devices : 0);
        return LLRL_E_INVALID;
    }
    DeviceWork &W = p->dev[device];
    const bool cross = !W.signal_devices.empty() || W.n_senders_in > 0;
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
    std::vector<char> su(size_t(p->n_src), 0), du(size_t(p->n_dst), 0);
    touched_ranks(W, su, du);
    KParams kp;
    std::memset(&kp, 0, sizeof kp);
    for (int r = 0; r < p->n_src; r++) {
        if (su[r] && !src_ptrs[r]) { set_error("llrl_sync: src_ptrs[%d] is NULL", r); return LLRL_E_NOPEER; }
        kp.src[r] = src_ptrs[r];
    }
    for (int g = 0; g < p->n_dst; g++) {
        if (du[g] && !dst_ptrs[g]) { set_error("llrl_sync: dst_ptrs[%d] is NULL", g); return LLRL_E_NOPEER; }
        kp.dst[g] = dst_ptrs[g];
    }
    DeviceGuard guard(device);
    llrl_status st = ensure_uploaded(p, device);
    if (st != LLRL_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!W.items.empty()) {
        W.epoch++;
        kp.items = W.d_items;
        kp.segs = W.d_segs;
        const int64_t n = int64_t(W.items.size());
        const bool has_cast = W.n_cast > 0, has_fp8 = n > W.n_cast;
        for (int mode = 0; mode < 2; mode++) {
            if (mode == 0 ? !has_cast : !has_fp8) continue;
            const bool last = mode == 1 || !has_fp8;
            const int grid = mode == 0 ? W.grid_cast : W.grid_fp8;
            kp.item_begin = mode == 0 ? 0 : int(W.n_cast);
            kp.item_end = mode == 0 ? int(W.n_cast) : int(n);
            kp.done = nullptr;
            kp.n_signal = 0;
            if (last && !W.signal_devices.empty()) {
                kp.done = W.d_done;
                kp.done_target = W.epoch * uint64_t(grid);
                kp.n_signal = int(W.signal_devices.size());
                for (int i = 0; i < kp.n_signal; i++) kp.signal[i] = comm->peer_flags[W.signal_devices[i]];
            }
            CK(launch_sync(kp, mode, W.variant, p->src_dtype == LLRL_F32, grid, s));
        }
    }
    if (W.n_senders_in > 0) {
        comm->expected += uint64_t(W.n_senders_in);
        CK(launch_wait(comm->flags, comm->expected, s));
    }
    return LLRL_OK;
}

llrl_status llrl_sync_num_launches(const llrl_plan *p, int device, int *n) {
    if (!p || !n || device < 0 || device >= p->n_devices) { set_error("invalid argument"); return LLRL_E_INVALID; }
    const DeviceWork &W = p->dev[device];
    *n = (W.n_cast > 0 ? 1 : 0) + (int64_t(W.items.size()) > W.n_cast ? 1 : 0) + (W.n_senders_in > 0 ? 1 : 0);
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
    return llrl_sync_num_launches(p, device, &out->n_launches);
}

llrl_status llrl_sync_host(llrl_plan *p, llrl_comm *comm, int device, const void *const *host_src,
                           void *const *host_dst, void *const *src_ptrs, void *const *dst_ptrs, void *stream) {
    if (!p || !host_src || !host_dst || !src_ptrs || !dst_ptrs || device < 0 || device >= p->n_devices) {
        set_error("llrl_sync_host: invalid argument");
        return LLRL_E_INVALID;
    }
    DeviceGuard guard(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int r = 0; r < p->n_src; r++)
        if (p->src_device[r] == device && host_src[r])
            CK(cudaMemcpyAsync(src_ptrs[r], host_src[r], size_t(p->src_rank_bytes[r]), cudaMemcpyHostToDevice, s));
    llrl_status st = llrl_sync(p, comm, device, src_ptrs, dst_ptrs, stream);
    if (st != LLRL_OK) return st;
    for (int g = 0; g < p->n_dst; g++)
        if (p->dst_device[g] == device && host_dst[g])
            CK(cudaMemcpyAsync(host_dst[g], dst_ptrs[g], size_t(p->dst_rank_bytes[g]), cudaMemcpyDeviceToHost, s));
    return LLRL_OK;
}

void llrl_plan_destroy(llrl_plan *p) {
    if (!p) return;
    for (size_t d = 0; d < p->dev.size(); d++) {
        DeviceWork &W = p->dev[d];
        if (W.uploaded_device < 0) continue;
        DeviceGuard guard(W.uploaded_device);
        cudaFree(W.d_items);
        cudaFree(W.d_segs);
        cudaFree(W.d_done);
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
    cudaError_t e = cudaMalloc(&c->flags, 256);
    if (e == cudaSuccess) e = cudaMemset(c->flags, 0, 256);
    if (e != cudaSuccess) { delete c; return cuda_fail(e, "llrl_comm_create"); }
    c->peer_flags[device] = c->flags;
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
