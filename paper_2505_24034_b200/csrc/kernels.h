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
    int fp8_base;
    unsigned long long *done;          // per (plan, device) CTA completion counter (self-resetting), or null
    int item_begin, item_end;          // [begin, end) of this launch
    int n_signal;
    unsigned long long *signal[kMaxDevices];   // arrival counters of destination devices
    const void *src[kMaxRanks];
    void *dst[kMaxRanks];
    void *dst_mc[kMaxRanks];           // multicast VA per dst rank (F_MC items)
};

constexpr int kCastTmaVariant = 6;      // llrl_k_cast_tma (TMA-staged)
constexpr int kDefaultCastVariant = kCastTmaVariant;
cudaError_t launch_sync(const KParams &P, int mode, int variant, bool src_f32, int grid, cudaStream_t stream);
// comm flag buffer words: [0, 16) data arrivals per sender, [16, 32) staging
// announcements per device, [32] timeout flag, [64, 96) expected counts
// (device-side, local only).
constexpr int kFlagTimeout = 2 * kMaxDevices;
constexpr int kFlagExpected = 4 * kMaxDevices;
constexpr int kFlagBytes = 8 * 8 * kMaxDevices;
struct WaitTargets {
    unsigned long long count[2 * kMaxDevices];   // arrivals to wait for per flag slot; 0 = none
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
