// kernels.h -- launch interface between the runtime (runtime.cu) and the
// sm_100a kernels (kernels.cu, init.cu).  Library-private.
#pragma once

#include <cuda_runtime.h>

#include "internal.h"

namespace llrl {

// Kernel parameters, passed by value (__grid_constant__): no per-step host->device
// copy of the pointer tables.
struct KParams {
    const Item *items;
    const Seg *segs;
    const TmaRef *tma_refs;            // fp8 items: index i - fp8_base
    const void *tmaps;                 // CUtensorMap array (global memory)
    const uint32_t *nv_amax;           // NVFP4: global amax (u32 bits) per tensor id, fetched locally
    int fp8_base;
    unsigned long long *done;          // per (plan, device) CTA completion counter (self-resetting), or null
    int item_begin, item_end;          // [begin, end) of this launch
    int static_end;                    // TMA cast launch: items [item_begin, static_end) striped, the rest claimed (queue)
    int static_block;                  // static items as one contiguous block per CTA instead of a stride
    int n_signal;
    unsigned long long *signal[kMaxDevices];   // arrival counters of destination devices
    const void *src[kMaxRanks];
    void *dst[kMaxRanks];
    void *dst_mc[kMaxRanks];           // multicast VA per dst rank (F_MC items)
    unsigned long long *timeline;      // debug (LLRL_TIMELINE): [grid][start, end] of the cast launch, or null
    unsigned int *queue;               // TMA cast launch: [next item, CTAs done] (dynamic claims), or null
    const CastRef *cast_refs;          // TMA cast launch: per item band map + row (strided sources), or null
    const void *cast_tmaps;            // CUtensorMap per band (3-D)
    const int32_t *cast_box;           // per band: rows per box (0 = per-row copies)
    int pdl_wait;                      // launched as a programmatic dependent of the previous
                                       // launch: wait for it before completing / signalling
};

constexpr int kCastTmaVariant = 6;      // llrl_k_cast_tma (TMA-staged)
constexpr int kDefaultCastVariant = kCastTmaVariant;
cudaError_t launch_sync(const KParams &P, int mode, int variant, bool src_f32, int grid, cudaStream_t stream);
int cast_stage_bytes(int variant);     // stage bytes of a TMA cast variant

// NVFP4 (R16) per-tensor amax handshake kernels.
struct NvAmaxParams {
    const Item *items;
    int n_items;                       // scan items [0, n_items) (the cast range), F_NV ones count
    int run;                           // items per run, runs striped over the CTAs (0: one range per CTA)
    uint32_t *partial;                 // [n_tensors] local partial amax
    unsigned long long *done;          // self-resetting CTA counter
    const int32_t *contrib;            // tensor ids this device contributes to
    int n_contrib;
    const int32_t *tensor_dev;         // tensor id -> device
    uint32_t *tables[kMaxDevices];     // amax table of every device (peer-mapped)
    int my_dev;
    int n_signal;
    unsigned long long *signal[kMaxDevices];
    const void *src[kMaxRanks];
};
struct NvScaleParams {
    const void *locals;                // DeviceWork::NvLocal[n_local]
    int n_local;
    uint32_t *table;                   // this device's amax table
    void *dst[kMaxRanks];
    int n_signal;
    unsigned long long *signal[kMaxDevices];
};
struct NvFetchParams {
    const int32_t *contrib;
    int n_contrib;
    const int32_t *tensor_dev;
    const uint32_t *tables[kMaxDevices];
    uint32_t *amax_out;                // [n_tensors]
};
cudaError_t launch_nv_amax(const NvAmaxParams &P, bool src_f32, int grid, cudaStream_t stream);
cudaError_t launch_nv_scale(const NvScaleParams &P, cudaStream_t stream);
cudaError_t launch_nv_fetch(const NvFetchParams &P, cudaStream_t stream);
// llrl_sync_nv_amax: the fp32 tensor scale of every local tensor from a supplied amax.
struct NvTscaleParams {
    const void *locals;                // DeviceWork::NvLocal[n_local]
    int n_local;
    const uint32_t *amax;              // [n_tensors] (fp32 bits)
    void *dst[kMaxRanks];
};
cudaError_t launch_nv_tscale(const NvTscaleParams &P, cudaStream_t stream);
// comm buffer (u64 words): slot ranges of kMaxDevices counters each --
// [0,16) data arrivals per sender, [16,32) "layer group staged" per device,
// [32,48) NVFP4 partial amax arrivals per sender, [48,64) NVFP4 "tensor scales
// ready" per receiver; [64] timeout flag; [128,192) expected counts per slot
// (device-side, local); from byte kNvTableOffset: the NVFP4 amax tables, one
// region per plan (17 u32 per tensor: one partial per sender device, then the
// global amax).
constexpr int kSlotData = 0, kSlotStaged = 16, kSlotNvAmax = 32, kSlotNvReady = 48, kNumSlots = 64;
constexpr int kFlagTimeout = 64;
constexpr int kFlagExpected = 128;
constexpr int64_t kNvTableOffset = 4096;
constexpr int64_t kCommBytes = 4 << 20;
constexpr int kNvTableStride = kMaxDevices + 1;   // u32 per tensor
struct WaitTargets {
    unsigned long long count[kNumSlots];   // arrivals to wait for per flag slot; 0 = none
};
struct SignalTargets {
    unsigned long long *slot[kMaxDevices];
    int n;
};
cudaError_t launch_signal(const SignalTargets &t, cudaStream_t stream);
cudaError_t launch_wait(unsigned long long *flags, const WaitTargets &t, cudaStream_t stream);
cudaError_t sync_occupancy(int mode, int variant, bool src_f32, int *blocks_per_sm);
int num_cast_variants();

// K0 (init.cu): synthetic trainer weights of one piece.
struct FillPiece {
    int64_t byte_off, rows, cols, r0, c0;
    int param, is_norm;
};
cudaError_t launch_fill(void *base, const FillPiece *pieces_dev, int n_pieces, int64_t max_elems, bool f32,
                        uint64_t seed, cudaStream_t stream);

}  // namespace llrl
