// nccl.cpp -- step a5: NCCL where the trainer -> generator
// mapping is a plain replication (north_star; BROADCAST semantics, "sent
// identically to each inbound process").  The plan decides which case
// applies (plan.cpp, readings R17 / R18); this file owns the communicators and
// enqueues the collectives.  libnccl.so.2 is loaded with dlopen on first use
// (the one torch already loaded, if any), so the library has no link-time
// NCCL dependency and every non-NCCL path works without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "internal.h"

using namespace llrl;

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](const char *n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommSplit && a.CommDestroy && a.Broadcast && a.AllGather &&
               a.GroupStart && a.GroupEnd && a.GetErrorString;
    });
    return a;
}

llrl_status nccl_fail(ncclResult_t r, const char *what) {
    set_error("%s: %s", what, api().GetErrorString ? api().GetErrorString(r) : "NCCL error");
    return LLRL_E_CUDA;
}

#define NK(call)                                         \
    do {                                                 \
        ncclResult_t r_ = (call);                        \
        if (r_ != ncclSuccess) return nccl_fail(r_, #call); \
    } while (0)

llrl_status need_api() {
    if (!api().ok) {
        set_error("NCCL unavailable: libnccl.so.2 could not be loaded (%s)", dlerror() ? dlerror() : "missing symbols");
        return LLRL_E_UNSUPPORTED;
    }
    return LLRL_OK;
}

}  // namespace

namespace llrl {

// Enqueue this device's NCCL operations of one sync on `stream` (after the
// kernels and the completion wait for the broadcast case; alone for the
// all-gather case).  Grouped: one NCCL launch sequence per sync.
llrl_status nccl_enqueue(llrl_plan *p, int device, void *const *src_ptrs, void *const *dst_ptrs, void *stream) {
    if (p->nccl_mode == 0) return LLRL_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto f = p->nccl.find(device);
    if (f == p->nccl.end() || !f->second.parent) {
        set_error("llrl_sync: NCCL plan used on device %d before llrl_nccl_attach", device);
        return LLRL_E_NOPEER;
    }
    const llrl_plan::NcclState &st = f->second;
    const NcclApi &A = api();
    NK(A.GroupStart());
    if (p->nccl_mode == 1) {
        for (const auto &b : p->nccl_bcast) {
            ncclComm_t c = static_cast<ncclComm_t>(st.sub[size_t(b.set)]);
            if (!c) continue;
            const auto &devs = p->nccl_sets[size_t(b.set)];
            int me = -1, root = -1;
            for (size_t k = 0; k < devs.size(); k++) {
                if (devs[k] == device) me = int(k);
                if (devs[k] == b.root_dev) root = int(k);
            }
            void *buf = dst_ptrs[b.dst_rank[size_t(me)]];
            if (!buf) { NK(A.GroupEnd()); set_error("llrl_sync: dst_ptrs[%d] is NULL", b.dst_rank[size_t(me)]); return LLRL_E_NOPEER; }
            NK(A.Broadcast(buf, buf, size_t(b.bytes), ncclUint8, root, c, s));
        }
    } else {
        ncclComm_t c = static_cast<ncclComm_t>(st.sub[0]);
        const auto &devs = p->nccl_sets[0];
        // FSDP rank f on device src_device[f]; NCCL rank = index in the sorted device set
        int f = -1;
        for (int r = 0; r < p->n_src; r++)
            if (p->src_device[size_t(r)] == device) f = r;
        if (c && f >= 0) {
            const char *sb = static_cast<const char *>(src_ptrs[f]);
            char *db = static_cast<char *>(dst_ptrs[f]);
            if (!sb || !db) { NK(A.GroupEnd()); set_error("llrl_sync: NULL rank buffer for FSDP rank %d", f); return LLRL_E_NOPEER; }
            (void)devs;
            const ncclDataType_t dt = p->nccl_elem_bytes == 4 ? ncclFloat32 : ncclBfloat16;
            for (const auto &g : p->nccl_gather)
                NK(A.AllGather(sb + g.src_off[size_t(f)], db + g.dst_off[size_t(f)], size_t(g.count), dt, c, s));
        }
    }
    NK(A.GroupEnd());
    return LLRL_OK;
}

void nccl_destroy(llrl_plan *p) {
    if (!api().ok) return;
    for (auto &kv : p->nccl) {
        for (void *c : kv.second.sub)
            if (c) api().CommDestroy(static_cast<ncclComm_t>(c));
        if (kv.second.parent) api().CommDestroy(static_cast<ncclComm_t>(kv.second.parent));
    }
    p->nccl.clear();
}

}  // namespace llrl

extern "C" {

llrl_status llrl_nccl_unique_id(void *id128) {
    if (!id128) { set_error("llrl_nccl_unique_id: NULL"); return LLRL_E_INVALID; }
    llrl_status s = need_api();
    if (s != LLRL_OK) return s;
    ncclUniqueId id;
    NK(api().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
    return LLRL_OK;
}

llrl_status llrl_nccl_attach(llrl_plan *p, int device, const void *id128, int rank, int nranks) {
    if (!p || !id128 || device < 0 || device >= kMaxDevices || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("llrl_nccl_attach: invalid argument");
        return LLRL_E_INVALID;
    }
    llrl_status s = need_api();
    if (s != LLRL_OK) return s;
    if (p->nccl.count(device)) { set_error("llrl_nccl_attach: device %d already attached", device); return LLRL_E_INVALID; }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    llrl_plan::NcclState st;
    st.rank = rank;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t parent = nullptr;
    ncclResult_t r = api().CommInitRank(&parent, nranks, id, rank);
    if (r == ncclSuccess) {
        st.parent = parent;
        // one sub-communicator per device set, created collectively in plan order
        // (every process walks the same list; non-members pass NOCOLOR)
        for (const auto &devs : p->nccl_sets) {
            int key = -1;
            for (size_t k = 0; k < devs.size(); k++)
                if (devs[k] == device) key = int(k);
            if (p->nccl_mode == 2 && key >= 0)   // all-gather: NCCL rank = FSDP rank (chunk order)
                for (int f = 0; f < p->n_src; f++)
                    if (p->src_device[size_t(f)] == device) key = f;
            ncclComm_t sub = nullptr;
            r = api().CommSplit(parent, key >= 0 ? 0 : NCCL_SPLIT_NOCOLOR, key >= 0 ? key : 0, &sub, nullptr);
            if (r != ncclSuccess) break;
            st.sub.push_back(sub);
        }
    }
    if (prev >= 0) cudaSetDevice(prev);
    p->nccl[device] = st;
    if (r != ncclSuccess) return nccl_fail(r, "llrl_nccl_attach");
    return LLRL_OK;
}

llrl_status llrl_plan_nccl_info(const llrl_plan *p, int device, llrl_nccl_info *out) {
    if (!p || !out || device < 0 || device >= p->n_devices) { set_error("llrl_plan_nccl_info: invalid argument"); return LLRL_E_INVALID; }
    std::memset(out, 0, sizeof *out);
    out->mode = p->nccl_mode;
    if (p->nccl_mode == 1) {
        for (const auto &b : p->nccl_bcast) {
            const auto &devs = p->nccl_sets[size_t(b.set)];
            if (std::find(devs.begin(), devs.end(), device) == devs.end()) continue;
            out->n_broadcasts++;
            if (device != b.root_dev) out->bytes += b.bytes;
        }
    } else if (p->nccl_mode == 2) {
        const auto &devs = p->nccl_sets[0];
        if (std::find(devs.begin(), devs.end(), device) != devs.end()) {
            out->n_allgathers = int32_t(p->nccl_gather.size());
            for (const auto &g : p->nccl_gather) out->bytes += g.count * p->nccl_elem_bytes * int64_t(devs.size() - 1);
        }
    }
    return LLRL_OK;
}

}  // extern "C"
