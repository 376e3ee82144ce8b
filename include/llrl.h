/*
 * llrl.h -- C ABI of libllrl: B200-native DDMA weight synchronisation
 * (LlamaRL, arxiv 2505.24034, §5.2 "Distributed Direct Memory Access
 * (DDMA) Weights Update").
 *
 * The problem: "sending updated policy parameters from a training
 * executor to an inference executor", where "each GPU only stores or updates
 * its assigned shards, leveraging the same tensor and parallel groups used
 * during training", by "direct memory transfers between CUDA memory
 * regions across devices -- bypassing CPU memory".  Trainer and
 * generator "can use different parallelisms and data precision",
 * including "quantization (fp8 ...) on the inference side".
 *
 * Three calls carry the method:
 *   llrl_layout_describe  -- step a1: both sides' per-rank flat-buffer layouts
 *   llrl_plan_create      -- step a2: the integer routing plan (tiles -> runs)
 *   llrl_sync             -- steps a3-a6: the hot path on one device's stream
 * Conventions that the paper leaves open are DESIGN.md readings R0-R11.
 *
 * General rules
 *   - Every call returns llrl_status (0 = OK, negative = error) unless noted;
 *     on error llrl_last_error() returns a thread-local message.  No C++
 *     exception or abort crosses the ABI.
 *   - Offsets in llrl_param_view are BYTES from the rank buffer base.  Offsets
 *     in llrl_run are ELEMENTS of that side's data dtype (MXFP4: 4-bit
 *     elements, i.e. twice the byte offset).
 *   - Rank buffers must be 256-byte aligned device allocations owned by the
 *     caller.  The library owns layouts, plans and comms until *_destroy,
 *     including their device-side tables and flag buffers.
 *   - `cudaStream_t` is passed as `void *` so this header has no CUDA
 *     dependency.
 */
#ifndef LLRL_H
#define LLRL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LLRL_OK = 0,
    LLRL_E_INVALID = -1,      /* bad argument / NULL / out of range          */
    LLRL_E_INDIVISIBLE = -2,  /* a TP split does not divide a dimension (R1, R4) */
    LLRL_E_MISMATCH = -3,     /* src and dst layouts describe different models */
    LLRL_E_UNSUPPORTED = -4,  /* dtype combination not supported             */
    LLRL_E_CUDA = -5,         /* CUDA runtime error (message has cudaGetErrorString) */
    LLRL_E_NOPEER = -6,       /* a device the plan needs has no comm peer mapping */
    LLRL_E_NOMEM = -7         /* host or device allocation failed            */
} llrl_status;

/* LLRL_MXFP8: OCP MX E4M3 elements with one E8M0 scale byte per 1x32 row
 * group (NEXT f2, "quantization (fp8 or fp4) on the inference side", P:145;
 * reading R13); scale grid [R, ceil(C/32)] bytes after each quantised weight. */
/* LLRL_MXFP4: OCP MX E2M1 elements (two per byte, even element in the low
 * nibble) with one E8M0 scale byte per 1x32 row group (reading R15). */
/* LLRL_NVFP4: E2M1 elements (packed like MXFP4) with one E4M3 scale per 1x16
 * row group and one fp32 scale per generator tensor (reading R16); the tensor
 * scale needs the tensor's global amax, a cross-GPU max-reduction inside the
 * sync (llrl_sync_group returns UNSUPPORTED -- a layer group never holds whole
 * tensors' contributions; llrl_sync_host copies whole buffers in, runs the whole
 * sync, copies whole buffers out, without per-group pipelining). */
typedef enum { LLRL_F32 = 0, LLRL_BF16 = 1, LLRL_FP8_E4M3 = 2, LLRL_MXFP8 = 3, LLRL_MXFP4 = 4,
               LLRL_NVFP4 = 5 } llrl_dtype;

/* Llama-style decoder shapes (Llama-3.1 config.json fields [ext]). */
typedef struct {
    int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ffn, vocab, with_embed;
} llrl_model;

/* flags of llrl_layout_describe */
#define LLRL_MESH_FSDP_INNER 1u   /* trainer rank = t*fsdp + f (default f*tp + t), R3 */

/* parameter kinds reported by llrl_layout_param_view */
enum {
    LLRL_P_ATTN_NORM = 0, LLRL_P_Q, LLRL_P_K, LLRL_P_V, LLRL_P_O, LLRL_P_MLP_NORM,
    LLRL_P_GATE, LLRL_P_UP, LLRL_P_DOWN, LLRL_P_EMBED, LLRL_P_FINAL_NORM, LLRL_P_LM_HEAD,
    LLRL_P_QKV, LLRL_P_GATE_UP
};

typedef struct llrl_layout llrl_layout;
typedef struct llrl_plan llrl_plan;
typedef struct llrl_comm llrl_comm;

/* One parameter piece on one rank. */
typedef struct {
    int32_t kind;        /* LLRL_P_* */
    int32_t layer;       /* -1 for embed / final_norm / lm_head */
    int32_t dtype;       /* llrl_dtype of the data */
    int32_t quantised;   /* 1: fp8 data followed by its scale grid (R7, R9, R13) */
    int64_t rows, cols;  /* local shape, row-major, leading dimension = cols */
    int64_t byte_off;    /* data offset in the rank buffer */
    int64_t scale_off;   /* scale grid offset, -1 if not quantised */
    int64_t full_r0, full_c0;  /* src side: top-left of the piece in the full tensor; dst: 0 */
    int32_t src_param;   /* src side: canonical source-param id; dst side: -1 */
    int32_t is_norm;
    int64_t tensor_scale_off;  /* NVFP4: byte offset of the fp32 tensor scale, else -1 */
} llrl_param_view;

/* ---- a1: layouts ------------------------------------------------------------
 * Describe the trainer (src) and generator (dst) layouts of `m` for a trainer
 * mesh fsdp x tp_train (fsdp*tp_train ranks, R1-R3) and a generator with
 * tp_gen ranks (R4).  src_dtype in {F32, BF16}; dst_dtype in {F32 (only from
 * F32: identity/provenance mode), BF16, FP8_E4M3 (R7), MXFP8 (R13), MXFP4 (R15),
 * NVFP4 (R16)}.
 * Errors: INVALID (NULL, non-positive sizes), INDIVISIBLE, UNSUPPORTED.
 * Ownership: *src_out and *dst_out belong to the caller (llrl_layout_destroy). */
llrl_status llrl_layout_describe(const llrl_model *m, int fsdp, int tp_train, int tp_gen,
                                 llrl_dtype src_dtype, llrl_dtype dst_dtype, uint32_t flags,
                                 llrl_layout **src_out, llrl_layout **dst_out);
/* Same, with generator data parallelism and pipeline stages on either side
 * (decoupled DP / PP; readings R12, R14): pp_* stages split the
 * decoder layers evenly and contiguously (embed on the first stage,
 * final_norm + lm_head on the last; n_layers % pp != 0 -> INDIVISIBLE);
 * trainer rank = stage*(fsdp*tp_train) + mesh rank, generator rank
 * q = d*(pp_gen*tp_gen) + stage*tp_gen + g, replica d holding exactly what
 * replica 0 holds.  Parameters of other stages are empty pieces (0 bytes).
 * llrl_layout_describe == this with dp_gen = pp_train = pp_gen = 1. */
typedef struct {
    int32_t fsdp, tp_train, tp_gen, dp_gen, pp_train, pp_gen;
    int32_t src_dtype, dst_dtype;   /* llrl_dtype */
    uint32_t flags;
    int32_t reserved;
} llrl_layout_opts;
llrl_status llrl_layout_describe_ex(const llrl_model *m, const llrl_layout_opts *opts,
                                    llrl_layout **src_out, llrl_layout **dst_out);
llrl_status llrl_layout_num_ranks(const llrl_layout *l, int *n);
llrl_status llrl_layout_num_params(const llrl_layout *l, int *n);
/* Bytes of rank `rank`'s flat buffer (a multiple of 256). */
llrl_status llrl_layout_rank_bytes(const llrl_layout *l, int rank, int64_t *bytes);
/* Where parameter `param` (canonical index of that side, R0) lives on `rank`. */
llrl_status llrl_layout_param_view(const llrl_layout *l, int rank, int param, llrl_param_view *out);
void llrl_layout_destroy(llrl_layout *l);

/* ---- a2: plan --------------------------------------------------------------
 * Build the routing plan from src to dst (same model; else MISMATCH).
 * src_device[r] / dst_device[g] = GPU ordinal hosting trainer rank r /
 * generator rank g (any mapping; several ranks may share a GPU).  Host-only:
 * no CUDA call is made; device tables are uploaded on the first llrl_sync
 * that needs them.  flags: 0 (reserved).
 * Ownership: the plan copies what it needs; the layouts may be destroyed. */
llrl_status llrl_plan_create(const llrl_layout *src, const llrl_layout *dst,
                             const int *src_device, const int *dst_device, uint32_t flags,
                             llrl_plan **out);
/* flags of llrl_plan_create */
#define LLRL_PLAN_MULTICAST 1u   /* NEXT f1: write generator DP replicas once through NVLS
                                    multicast (see llrl_mc_*); positions whose replicas share
                                    a GPU fall back to per-replica pushes */
void llrl_plan_destroy(llrl_plan *p);

/* A canonical 1-D run: `len` consecutive elements (verification view). */
typedef struct {
    int32_t src_param;   /* canonical source-param id */
    int32_t src_rank, dst_rank;
    int32_t flags;       /* bit0: quantised destination (fp8 bytes) */
    int64_t src_off, dst_off, len;   /* elements of each side's data dtype */
} llrl_run;
llrl_status llrl_plan_num_runs(const llrl_plan *p, int64_t *n);
llrl_status llrl_plan_get_runs(const llrl_plan *p, int64_t first, int64_t count, llrl_run *out);

typedef struct {
    int32_t n_devices;          /* 1 + the largest device ordinal used      */
    int32_t n_src_ranks, n_dst_ranks;
    int64_t n_tiles;            /* rectangle intersections (param, src, dst) */
    int64_t n_items;            /* work items over all devices              */
    int64_t n_fp8_blocks, n_fp8_pull_blocks;
    int64_t src_bytes, dst_bytes;   /* algorithmic bytes read / written (whole sync) */
} llrl_plan_stats;
llrl_status llrl_plan_stats_get(const llrl_plan *p, llrl_plan_stats *out);
/* bytes_GxG[s*G + d] = bytes written by device s's work into device d's memory
 * (wire bytes when s != d; local HBM writes when s == d).  G = n_devices. */
llrl_status llrl_plan_traffic(const llrl_plan *p, int64_t *bytes_GxG);
/* Algorithmic HBM bytes of one device for one sync: reads of everything sourced
 * there plus writes of everything landing there; and NVLink egress/ingress. */
llrl_status llrl_plan_device_bytes(const llrl_plan *p, int device, int64_t *hbm_read,
                                   int64_t *hbm_write, int64_t *nvl_tx, int64_t *nvl_rx);

/* Per-device share of one sync. */
typedef struct {
    int64_t n_items, n_cast_items, n_fp8_items, n_fp8_pull_items;
    int32_t n_signal;      /* devices this device writes into (and signals) */
    int32_t n_senders_in;  /* other devices writing into this device (it waits for them) */
    int32_t n_launches;    /* kernels llrl_sync enqueues on this device */
    int32_t reserved;
    int64_t nv_amax_read_bytes;   /* NVFP4 two-pass sync: source bytes the per-tensor amax
                                     pass re-reads on this device (on top of the algorithmic
                                     hbm_read of llrl_plan_device_bytes; 0 with
                                     llrl_sync_nv_amax) */
} llrl_device_info;
llrl_status llrl_plan_device_info(const llrl_plan *p, int device, llrl_device_info *out);

/* ---- completion comm (a6) --------------------------------------------------
 * A comm owns one 1 MiB buffer on `device`: per-sender-device counters of data
 * arrivals, "trainer bytes staged" announcements (llrl_sync_host with pull
 * items) and the NVFP4 amax / scale handshake, a timeout flag (a wait gave up
 * after 30 s), the arrivals expected so far, and the NVFP4 amax table.
 * All counters are cumulative and live on the device: llrl_sync /
 * llrl_sync_group launch identical parameters on every call, so after one
 * warm-up call they can be captured in a CUDA graph and replayed.
 * Devices that exchange data in a plan must know each other's flag buffers:
 *   multi-process: llrl_comm_export on each, exchange the 64-byte handles
 *                  (e.g. torch.distributed.all_gather_object), llrl_comm_import;
 *   single process: llrl_comm_flag_ptr + llrl_comm_set_peer (peer access is
 *                  enabled by the library).
 * One comm per device per process; it may serve any number of plans, provided
 * every process issues the same sequence of llrl_sync calls.  Each NVFP4 plan
 * takes its own region of the comm's amax table on its first llrl_sync on that
 * device (regions are assigned in first-sync order, which the same-sequence
 * rule makes identical on every process; they are not reused after
 * llrl_plan_destroy); the table holds about 60k NVFP4 tensors per comm
 * lifetime (UNSUPPORTED beyond). */
llrl_status llrl_comm_create(int device, llrl_comm **out);
llrl_status llrl_comm_export(const llrl_comm *c, void *handle64);
llrl_status llrl_comm_import(llrl_comm *c, int peer_device, const void *handle64);
llrl_status llrl_comm_flag_ptr(const llrl_comm *c, void **dev_ptr);
llrl_status llrl_comm_set_peer(llrl_comm *c, int peer_device, void *peer_flag_dev_ptr);
/* ---- NVLS multicast buffers (NEXT f1) -----------------------------------------
 * One multicast object per generator rank position (TP rank x PP stage) whose
 * replicas live on different GPUs; its team is every GPU of the job.  The
 * creating process calls llrl_mc_create (size rounded up to the multicast
 * granularity; *fd_out is a POSIX file descriptor to pass to the other
 * processes, e.g. over a Unix socket with SCM_RIGHTS), the others
 * llrl_mc_import; then every process calls llrl_mc_join for its GPU, which
 * creates and binds that GPU's physical memory and maps it at a unicast VA
 * (*local_ptr: use it as the generator rank buffer on replica GPUs; scratch
 * elsewhere) and maps the multicast VA (*mc_ptr).  llrl_plan_set_multicast
 * gives a device the multicast VA of every generator rank (NULL where none).
 * Errors: UNSUPPORTED (no multicast driver support), CUDA. */
typedef struct llrl_mcbuf llrl_mcbuf;
llrl_status llrl_mc_create(int n_devices, int64_t bytes, int *fd_out, int64_t *size_out, llrl_mcbuf **out);
llrl_status llrl_mc_import(int fd, int n_devices, int64_t size, llrl_mcbuf **out);
llrl_status llrl_mc_join(llrl_mcbuf *m, int device, void **local_ptr, void **mc_ptr);
void llrl_mc_destroy(llrl_mcbuf *m);
/* Unicast access to a peer GPU's memory of the same multicast object (for the
 * plan's egress split: a share of a replica position's items is pushed to every
 * replica as plain peer stores, the rest multicast): llrl_mc_export_local gives a
 * POSIX fd of this process's bound memory (after llrl_mc_join), llrl_mc_map_peer
 * maps a peer's fd into this process for `device` (*ptr: that replica's rank
 * buffer as seen here).  Unmapped by llrl_mc_destroy. */
llrl_status llrl_mc_export_local(const llrl_mcbuf *m, int *fd_out);
llrl_status llrl_mc_map_peer(llrl_mcbuf *m, int fd, int device, void **ptr);
llrl_status llrl_plan_set_multicast(llrl_plan *p, int device, void *const *dst_mc_ptrs);

/* ---- NVFP4 with a caller-supplied tensor amax (R16 in one pass) ----------------
 * llrl_sync on an NVFP4 plan reads every quantised source twice: a per-tensor
 * amax pass (a max-reduction across every GPU feeding the tensor, done inside
 * the sync) and the quantising pass.  A caller that already knows each
 * generator tensor's amax -- e.g. its optimizer epilogue took max |w| while
 * writing the updated shards ("stream layer l as soon as the optimizer updates
 * it", NEXT f3) -- passes it to llrl_sync_nv_amax, which reads each
 * source byte once (no amax pass, no handshake).
 * The plan's NVFP4 generator tensors are numbered 0..n-1.  Tensor `tid` is
 * generator param `dst_param` (canonical generator index) on generator rank
 * `dst_rank`, held by GPU `device`; its elements are exactly the trainer
 * regions llrl_plan_nv_tensor_sources lists (src_rank's buffer, element offset
 * src_off, rows x cols with leading dimension src_ld; replicated pieces are
 * listed once).  Errors: INVALID (not an NVFP4 plan, tid / range out of bounds). */
typedef struct {
    int32_t dst_rank, dst_param, device, n_sources;
} llrl_nv_tensor;
typedef struct {
    int32_t src_rank, src_param;
    int64_t src_off, rows, cols, src_ld;   /* elements of the trainer dtype */
} llrl_nv_source;
llrl_status llrl_plan_nv_num_tensors(const llrl_plan *p, int *n);
llrl_status llrl_plan_nv_tensor(const llrl_plan *p, int tid, llrl_nv_tensor *out);
llrl_status llrl_plan_nv_tensor_sources(const llrl_plan *p, int tid, int first, int count, llrl_nv_source *out);
/* As llrl_sync, for an NVFP4 plan, with amax_dev[tid] (device memory on
 * `device`, fp32, one per plan tensor id) = max |x| over generator tensor tid:
 * the same array on every device; it must be +0 or a positive finite value.
 * When `stream` passes the call, the device's generator shards are complete
 * (codes, group scales and each local tensor's fp32 scale A / 2688 with
 * A = max(amax, 2^-64)); the result is byte-identical to llrl_sync's when the
 * supplied amax is the exact one.  `comm` may be NULL iff the device exchanges
 * no data with peers. */
llrl_status llrl_sync_nv_amax(llrl_plan *p, llrl_comm *comm, int device, const float *amax_dev,
                              void *const *src_ptrs, void *const *dst_ptrs, void *stream);

/* ---- a5: NCCL where the mapping is a plain replication ---------------------------
 * north_star: "a fallback that uses NCCL broadcast/all-gather only where the
 * trainer->generator mapping is a plain shard replication"; the paper's
 * replication semantics are BROADCAST, "sent identically to each inbound
 * process".  A plan created with LLRL_PLAN_NCCL takes the NCCL path in
 * the two cases that are pure replication (readings R17, R18 of DESIGN.md):
 *   broadcast: generator DP replicas (R12) whose replicas of a rank position
 *     sit on pairwise different GPUs: the fused kernels write replica 0 only,
 *     then ncclBroadcast copies replica 0's whole rank buffer to the others;
 *   all-gather: an FSDP-only trainer (tp_train = pp = 1, fsdp = F >= 2, every
 *     parameter's rows divisible by F) synced without a cast (same dtype) into
 *     F generator replicas of tp_gen = 1 placed on the trainer ranks' GPUs
 *     (replica f with trainer rank f): every generator tensor part is the
 *     concatenation of the F row chunks, i.e. one ncclAllGather per source
 *     parameter into its offset in the generator buffer -- no kernel of ours.
 * Otherwise (or without the flag) the fused kernels do everything.
 * llrl_nccl_unique_id: one process makes the id (128 bytes) and shares it;
 * llrl_nccl_attach: EVERY process of the job calls it once per plan, with its
 * GPU, its rank in [0, nranks) and nranks (a collective: it creates the
 * library-owned NCCL communicator and the sub-communicators the plan needs);
 * the communicators are destroyed with the plan.  Then llrl_sync enqueues the
 * NCCL operations after (broadcast) or instead of (all-gather) the kernels.
 * llrl_plan_nccl_info: the operations one device takes part in.
 * Errors: UNSUPPORTED (libnccl.so.2 not loadable), CUDA (NCCL error text),
 * NOPEER (llrl_sync on an NCCL plan before llrl_nccl_attach). */
#define LLRL_PLAN_NCCL 2u
typedef struct {
    int32_t n_broadcasts;   /* ncclBroadcast calls per sync on this device (member of) */
    int32_t n_allgathers;   /* ncclAllGather calls per sync on this device */
    int64_t bytes;          /* bytes this device receives through them per sync */
    int32_t mode;           /* 0 = kernels only, 1 = kernels + broadcast, 2 = all-gather only */
    int32_t reserved;
} llrl_nccl_info;
llrl_status llrl_nccl_unique_id(void *id128);
llrl_status llrl_nccl_attach(llrl_plan *p, int device, const void *id128, int rank, int nranks);
llrl_status llrl_plan_nccl_info(const llrl_plan *p, int device, llrl_nccl_info *out);

/* Synchronous check of the timeout flag (1 if any wait on this device gave up). */
llrl_status llrl_comm_timed_out(const llrl_comm *c, int *timed_out);
void llrl_comm_destroy(llrl_comm *c);

/* ---- IPC helpers for caller-owned buffers ----------------------------------
 * handle64 + byte offset of `dev_ptr` inside its cudaMalloc allocation, and
 * the reverse mapping in another process (peer access over NVLink). */
llrl_status llrl_ipc_handle(const void *dev_ptr, void *handle64, int64_t *offset);
llrl_status llrl_ipc_open(const void *handle64, int64_t offset, void **dev_ptr);
llrl_status llrl_ipc_close(void *dev_ptr, int64_t offset);

/* ---- a3-a6: the hot path ----------------------------------------------------
 * Enqueue on `stream` (a cudaStream_t of device comm->device) every work item
 * this device executes: push items for tiles sourced here (cast before the
 * transfer: wire bytes at the destination width), pull items for multi-source
 * fp8 blocks landing here (R8); then signal each destination device this device
 * wrote to; then wait until every device writing into this device's
 * destinations has signalled.  When `stream` passes that point, every
 * generator shard resident on this device is complete.  Asynchronous to the
 * host; no host round trip on the per-step path.
 * src_ptrs[r] (r < n_src_ranks), dst_ptrs[g] (g < n_dst_ranks): rank buffer
 * base pointers valid in this process (local or peer/IPC-mapped); entries this
 * device never touches may be NULL.  `comm` may be NULL iff the plan uses one
 * device.  Preconditions (step boundary): no one writes the src
 * buffers or reads the dst buffers during the sync.  Syncs of one plan on one
 * device are stream-ordered: issue them on one stream (or order the streams),
 * since a plan's per-device completion counters are reused from sync to sync;
 * every process issues the same sequence of syncs (per-sender arrival counts).
 * A device that holds no rank of the plan has nothing to do (the call is a
 * no-op below the plan's highest device ordinal, INVALID above it).
 * Errors: INVALID, NOPEER (a needed peer flag buffer or pointer missing), CUDA. */
llrl_status llrl_sync(llrl_plan *p, llrl_comm *comm, int device,
                      void *const *src_ptrs, void *const *dst_ptrs, void *stream);

/* Layer-group streaming (NEXT f3: "stream layer l as soon as the optimizer
 * updates it"): the plan's work split by layer group -- group 0 = embed (if
 * any), then one group per decoder layer, then final_norm + lm_head.
 * llrl_sync_group enqueues exactly the work of one group (push, signal, wait),
 * so group g can be synced while the trainer still updates later layers.  All
 * processes must issue the same sequence of llrl_sync / llrl_sync_group calls;
 * running every group once is equivalent to one llrl_sync. */
llrl_status llrl_plan_num_groups(const llrl_plan *p, int *n);
/* Byte range [*lo, *hi) of layer group `group` in rank `rank`'s buffer on the
 * trainer (side 0) or generator (side 1) side; *lo = *hi = -1 if the rank holds
 * nothing of that group.  Lets a caller update / consume one group at a time. */
llrl_status llrl_plan_group_range(const llrl_plan *p, int side, int rank, int group, int64_t *lo, int64_t *hi);
llrl_status llrl_sync_group(llrl_plan *p, llrl_comm *comm, int device, int group,
                            void *const *src_ptrs, void *const *dst_ptrs, void *stream);

/* Same as llrl_sync, with the trainer shards hosted on this device first
 * copied from HOST buffers host_src[r] and, after the sync, the generator
 * shards resident on this device copied back to host_dst[g] (entries of ranks
 * on other devices are ignored; host buffers should be pinned).  Pipelined per
 * layer group on two library-owned copy streams: H2D of group g+1 and D2H of
 * group g-1 overlap the kernels of group g (decoder layers open and close the
 * pipeline; the embedding and lm_head groups run in its middle).  NVFP4 plans
 * are not pipelined (whole buffers in, the whole sync, whole buffers out on
 * `stream`: a tensor's scale needs its whole amax).  When `stream` passes the
 * end of the call, every host_dst byte of this device's generator ranks is
 * written. */
llrl_status llrl_sync_host(llrl_plan *p, llrl_comm *comm, int device,
                           const void *const *host_src, void *const *host_dst,
                           void *const *src_ptrs, void *const *dst_ptrs, void *stream);

/* Cap the CTAs (≈ SMs) the sync kernels of `device` use (0 = all).  An
 * NVLink-bound device saturates its links with a fraction of the SMs, leaving
 * the rest to overlapping compute (f3).  Must be called before the first sync
 * on that device or between syncs (tables are re-uploaded). */
llrl_status llrl_plan_set_max_ctas(llrl_plan *p, int device, int max_ctas);

/* Number of kernels llrl_sync enqueues on `device` (for launch accounting). */
llrl_status llrl_sync_num_launches(const llrl_plan *p, int device, int *n);

/* ---- harness support (tests / bench only; not part of the method) ----------
 * K0: fill trainer rank `rank`'s buffer with the counter-based synthetic
 * weights of DESIGN.md §4 (bit-identical to synth.weight_bits). */
llrl_status llrl_fill_synthetic(const llrl_layout *src, int rank, void *dev_ptr, uint64_t seed,
                                void *stream);

/* Debug timeline (set LLRL_TIMELINE=1 before the plan's first sync on `device`):
 * out[2c], out[2c+1] = %globaltimer (ns) when CTA c of the last cast launch
 * started / finished its last store; *n_ctas = CTAs copied (0 when disabled).
 * Synchronous. */
llrl_status llrl_debug_timeline(const llrl_plan *p, int device, uint64_t *out, int max_ctas, int *n_ctas);

const char *llrl_last_error(void);
const char *llrl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LLRL_H */
