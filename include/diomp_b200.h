/*
 * diomp_b200.h -- C ABI of libdiomp_b200.so, the B200-native data plane of the
 * DiOMP-Offloading hot path (global memory, one-sided put/get, fence/barrier,
 * OMPCCL bcast/reduce/allreduce, Minimod stencil, row-stripe DGEMM).
 *
 * Conventions
 *   - Plain integers and pointers only: device addresses are uint64_t (UVA),
 *     streams/events are opaque pointers (cudaStream_t / cudaEvent_t).
 *   - Every entry point returns an int status: the reference's wire status
 *     vocabulary (reference/pkg/src/diomp/wire.py:46-52) extended with host
 *     allocator outcomes, or DIOMP_CUDA_ERROR_BASE + cudaError_t.
 *   - Entry points are reentrant on distinct streams (runtime.py put/get may be
 *     called from any thread).  Heap handles are NOT thread-safe:
 *     allocation is a single-flow collective in the reference.
 *
 * Each function names the reference interface it replaces (file:line, paths
 * relative to reference/pkg/src/diomp/).
 */
#ifndef DIOMP_B200_H
#define DIOMP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (wire.py:46-52 Status + allocator errors) ------------- */
#define DIOMP_OK 0
#define DIOMP_INVALID_ADDRESS 1  /* wire.Status.INVALID_ADDRESS -> errors.InvalidAddress */
#define DIOMP_BAD_REQUEST 2      /* wire.Status.BAD_REQUEST                            */
#define DIOMP_INTERNAL 3         /* wire.Status.INTERNAL                               */
#define DIOMP_PENDING 4          /* event/handle not complete yet (HandleState.Pending) */
#define DIOMP_OUT_OF_SEGMENT 10  /* errors.OutOfSegment (allocators.py)                */
#define DIOMP_DOUBLE_FREE 11     /* errors.DoubleFree   (allocators.py)                */
#define DIOMP_CUDA_ERROR_BASE 100

#define DIOMP_MAX_TEAM 64        /* max endpoints in one team / flag array slots       */

const char *diomp_status_string(int status);
int diomp_version(void);
int diomp_device_count(int *count);
int diomp_device_sync(int device);
/* Device-side wait timeouts (see diomp_wait) are recorded, not trapped:
 * returns DIOMP_INTERNAL (and clears it) if any wait on `device` timed out. */
int diomp_device_error(int device);
/* Sets the device wait timeout (default 30 s) and maps a pinned mirror of the
 * error word, after which diomp_device_error is a host load, not a CUDA call. */
int diomp_set_wait_timeout(int device, double seconds);

/* ---- segments: global_memory.py:190-206 (GlobalMemory.__init__ arenas),
 *      segment_create global_memory.py:391-393.  A segment is one zero-filled
 *      cudaMalloc per device; peers map it by CUDA IPC (one process per GPU)
 *      or peer access (one process, several GPUs).                          */
int diomp_seg_create(int device, uint64_t bytes, uint64_t *base_out);
int diomp_seg_destroy(int device, uint64_t base);
int diomp_seg_ipc_export(int device, uint64_t base, uint8_t handle_out[64]);
int diomp_seg_ipc_import(int device, const uint8_t handle[64], uint64_t *base_out);
int diomp_seg_ipc_close(int device, uint64_t base);
int diomp_peer_enable(int device, int peer_device);

/* ---- heaps: allocators.py:36-190 (LinearAllocator, BuddyAllocator,
 *      ReverseBumpAllocator).  Offsets are bit-identical to the reference.  */
#define DIOMP_HEAP_LINEAR 0  /* (capacity, alignment)                    allocators.py:36-72   */
#define DIOMP_HEAP_BUDDY 1   /* (capacity, reserve_from; UINT64_MAX=none) allocators.py:75-150 */
#define DIOMP_HEAP_REVERSE 2 /* (floor=arg, capacity, alignment)         allocators.py:153-190 */
int diomp_heap_create(int kind, uint64_t capacity, uint64_t arg, uint64_t alignment,
                      void **heap_out);
int diomp_heap_destroy(void *heap);
int diomp_heap_alloc(void *heap, uint64_t size, uint64_t *offset_out);
int diomp_heap_free(void *heap, uint64_t offset, uint64_t *size_out);
int diomp_heap_block_size(void *heap, uint64_t size, uint64_t *block_out);
/* live map in insertion order (the reference's `live` dict); n_inout = capacity in, count out */
int diomp_heap_live(void *heap, uint64_t *offsets, uint64_t *sizes, uint64_t *n_inout);

/* ---- streams / events: streams.py:56-121 (Stream), runtime.py:472-484
 *      (_maybe_stream), runtime.py:535-556 (fence = drain of the ledgers). */
int diomp_stream_create(int device, void **stream_out);
int diomp_stream_destroy(void *stream);
int diomp_stream_sync(void *stream);
int diomp_event_create(int device, void **event_out);
int diomp_event_create_sync(int device, void **event_out); /* no timing: cheaper record */
int diomp_event_record(void *event, void *stream);
int diomp_event_query(void *event); /* DIOMP_OK when complete, DIOMP_PENDING otherwise */
int diomp_event_sync(void *event);
int diomp_event_destroy(void *event);
int diomp_event_elapsed_ms(void *start, void *stop, float *ms_out);
int diomp_stream_wait_event(void *stream, void *event);
int diomp_stream_query(void *stream); /* DIOMP_OK idle, DIOMP_PENDING busy */


/* ---- one-sided data plane: runtime.py:371-470 (put/get) replacing
 *      transport.py:508-566 (rma_put/rma_get frames).  D2D transfers are an
 *      SM-issued copy kernel launched on `device` (put: the source's device,
 *      stores cross NVLink; get: the destination's device, loads cross
 *      NVLink).  dst/src may be peer-mapped addresses.                       */
int diomp_copy(int device, uint64_t dst, uint64_t src, uint64_t nbytes, void *stream);
/* Runtime.put / Runtime.get D2D legs (runtime.py:371-419 / 421-470).  `remote`
 * = the far side is another GPU.  Engine per size (DIOMP_PUT_ENGINE /
 * DIOMP_GET_ENGINE override): remote put >= 64 KiB on the copy engine (SM
 * stores to a peer cap at ~715 GB/s, CE reaches 779), remote get >= 16 MiB on
 * the bulk-async TMA kernel, everything else on the SM copy kernel.          */
int diomp_put(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int remote, void *stream);
int diomp_get(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int remote, void *stream);
/* ---- rank-addressed RMA context: what a C / Cython caller binds
 *      to reach the global address space without Python.
 *      A context holds the peer table -- every endpoint's segment base as
 *      mapped in this process (CUDA IPC / peer access; global_memory.py:73-84
 *      GlobalAddress -> arena) -- and the ops in flight.  An endpoint is
 *      rank * devices_per_rank + dev (topology.py endpoint index).
 *      put/get replace runtime.py:371-470 -> transport.py:508-566 and return
 *      an op handle (transport.py:58-101 CompletionHandle): op_query ->
 *      DIOMP_OK (RemoteDone) / DIOMP_PENDING, op_wait blocks (DIOMP_INTERNAL on
 *      timeout), fence_group(mask) = runtime.py:535-556 fence toward a set of
 *      endpoints.  Ranges are checked against the segment extent
 *      (DIOMP_INVALID_ADDRESS); allocation-level checks (global_memory.py:
 *      306-333) stay with the caller, as in the reference.                  */
int diomp_rma_ctx_create(int32_t nranks, int32_t devices_per_rank, void **ctx_out);
int diomp_rma_ctx_destroy(void *ctx);
/* local device index -> CUDA device ordinal; phys_gpu = box-wide GPU id
 * (two endpoints on the same phys_gpu are local copies, others cross NVLink) */
int diomp_rma_set_local(void *ctx, int32_t local_dev, int32_t cuda_device, int32_t phys_gpu);
int diomp_rma_set_force_remote(void *ctx, int32_t on); /* test knob: take the NVLink engines */
int diomp_peer_table_set(void *ctx, int32_t rank, int32_t dev, uint64_t base, uint64_t bytes,
                         int32_t phys_gpu);
/* kind DIOMP_H2D (src = host pointer) or DIOMP_D2D (src = device pointer on local_dev) */
int diomp_rma_put(void *ctx, int32_t dst_rank, int32_t dst_dev, uint64_t dst_off, uint64_t src,
                  uint64_t nbytes, int32_t kind, int32_t local_dev, void *stream,
                  uint64_t *op_out);
/* kind DIOMP_D2H (dst = host pointer) or DIOMP_D2D (dst = device pointer on local_dev) */
int diomp_rma_get(void *ctx, int32_t src_rank, int32_t src_dev, uint64_t src_off, uint64_t dst,
                  uint64_t nbytes, int32_t kind, int32_t local_dev, void *stream,
                  uint64_t *op_out);
int diomp_op_query(void *ctx, uint64_t op);
int diomp_op_wait(void *ctx, uint64_t op, double timeout_s);   /* timeout_s < 0: no limit */
int diomp_fence_group(void *ctx, uint64_t endpoint_mask);
int diomp_rma_outstanding(void *ctx, uint64_t endpoint_mask, uint64_t *count_out);

/* host<->device legs of H2D put / D2H get (TransferKind, global_memory.py:52-70) */
#define DIOMP_H2D 1
#define DIOMP_D2H 2
#define DIOMP_D2D 3
int diomp_memcpy_async(uint64_t dst, uint64_t src, uint64_t nbytes, int kind, void *stream);
int diomp_memset_async(uint64_t dst, int value, uint64_t nbytes, void *stream);
/* blocking copy with `device` current (cell reads/writes, host views) */
int diomp_memcpy_sync(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int kind);

/* ---- device-side synchronisation (replaces the 2 ms host polling of
 *      runtime.py:535-556 and the TCP dissemination barrier runtime.py:493-513
 *      inside hot loops).  Flags are u64 counters in symmetric memory:
 *      signal = st.release.sys, wait = ld.acquire.sys until >= value.       */
int diomp_signal(int device, uint64_t flag_addr, uint64_t value, void *stream);
int diomp_wait(int device, uint64_t flag_addr, uint64_t value, void *stream);

/* A team is a communicator as seen by one launching endpoint
 * (collectives.py:102-143 Communicator / bootstrap: ring order = members
 * rotated to the root).  base[p] is position p's segment base as addressable
 * from `device`; flags of endpoint p live at base[p] + flag_off, slot index =
 * slot[q] (the global endpoint index of the signalling position q).
 * epoch_to[q] / epoch_from[q]: signals already sent to / received from q on
 * this pair.  Every collective call consumes ONE signal per pair -- its entry
 * handshake (block 0 signals +1 at kernel start, every CTA waits for the
 * peers' +1) -- and the caller advances both epochs by 1.  There is no exit
 * handshake inside the kernels: the next call's entry certifies the previous
 * one's completion toward each peer (the peer's stream has moved past it).
 * Where the caller itself needs the result, diomp_team_barrier behind the
 * kernel is the exit (one more signal, +1 again).  sync=0 skips all flag
 * traffic (the caller orders the endpoints with host barriers; used when
 * several endpoints share one GPU).                                           */
typedef struct {
    int32_t k;
    int32_t pos;
    int32_t device;
    int32_t sync;
    uint64_t flag_off;
    uint64_t counter_off; /* u32 scratch in own segment for last-CTA detection */
    uint64_t base[DIOMP_MAX_TEAM];
    uint32_t slot[DIOMP_MAX_TEAM];
    uint64_t epoch_to[DIOMP_MAX_TEAM];
    uint64_t epoch_from[DIOMP_MAX_TEAM];
} diomp_team;

int diomp_team_barrier(const diomp_team *team, void *stream);

/* ---- OMPCCL collectives (collectives.py:232-405).  Offsets are symmetric
 *      (same on every position).  Results are bit-identical to the
 *      reference's ring folds:
 *        reduce:    root gets ((v_root op v_root+1) op ...) op v_root-1
 *        allreduce: block b=[b*count/k,(b+1)*count/k) folded from position b.
 * allreduce is one kernel (fold, store the block to every member); bcast:
 * every non-root pulls its 1/(k-1) block from the root and pushes it to the
 * other non-roots.                                                           */
#define DIOMP_F32 0
#define DIOMP_F64 1
#define DIOMP_I32 2
#define DIOMP_I64 3
#define DIOMP_SUM 0
#define DIOMP_MIN 1
#define DIOMP_MAX 2
int diomp_bcast(const diomp_team *team, uint64_t offset, uint64_t nbytes, int32_t root,
                void *stream);
int diomp_reduce(const diomp_team *team, uint64_t send_off, uint64_t recv_off, uint64_t count,
                 int32_t dtype, int32_t op, int32_t root, void *stream);
int diomp_allreduce(const diomp_team *team, uint64_t send_off, uint64_t recv_off,
                    uint64_t count, int32_t dtype, int32_t op, void *stream);

/* Small messages: one-shot low-latency (LL) allreduce / bcast for teams of
 * k <= 8 on distinct GPUs.  Every 4-byte payload word travels with its flag
 * in one 8-byte store, (epoch << 32) | word, into the receiver's LL slot for
 * the sender (two parities per slot), so a call needs no entry or exit
 * handshake: allreduce = every position stores its vector to every peer,
 * then folds all k in the reference order (bit-identical); bcast = the root
 * stores to every non-root.  epoch_to[q] / epoch_from[q] = this call's epoch
 * for the pair (both ends count every LL call between them, from 1); the
 * LL region is `ll_off` in every member's segment, slot_bytes per (source
 * endpoint, parity), at least 2x the payload.  The 4 KiB below `ll_off`
 * (zero at start) hold the acknowledgement bank: a consumer acknowledges
 * each call to its writers, and a writer reuses a parity slot only after the
 * peer acknowledged the call that used it last (so a bcast root, which gets
 * no words back, can never overwrite a slot a slow peer has not read).      */
typedef struct {
    int32_t k, pos, device, dtype, op, root, mode;  /* mode 0 allreduce, 1 bcast (bytes) */
    int32_t _pad;
    uint64_t base[DIOMP_MAX_TEAM];
    uint32_t slot[DIOMP_MAX_TEAM];
    uint32_t epoch_to[DIOMP_MAX_TEAM];
    uint32_t epoch_from[DIOMP_MAX_TEAM];
    uint64_t ll_off, slot_bytes;
    uint64_t send_off, recv_off, count;
} diomp_ll_args;
int diomp_ll_collective(const diomp_ll_args *args, void *stream);
/* The same call as the runtime issues it, in one C call (replaces the
 * per-call Python of collectives.py:326-405's small-message path): epochs
 * taken from -- and advanced in -- the RMA context's per-pair LL table
 * (args->epoch_* are outputs), `stream` ordered after `after` (the caller's
 * stream, by an event; NULL = no ordering), and with blocking != 0 the
 * stream drained and the device error word checked (DIOMP_INTERNAL = a
 * device-side wait timed out: TransportFailure).                          */
int diomp_ll_call(void *rma_ctx, diomp_ll_args *args, void *stream, void *after,
                  int32_t blocking);

#ifdef DIOMP_EXPERIMENTS
/* ---- Experiments build only (-DDIOMP_EXPERIMENTS; measured slower than the
 *      defaults on B200, kept out of the product library).
 * bcast chain (root -> root+1 -> ... pipelined in chunks with per-CTA
 * progress flags) from `bytes` for teams of k >= 3; pull flavour = every hop
 * loads from its predecessor.  allreduce with the copy engine pushing each
 * folded block from `bytes`.  Same bytes as the defaults.                    */
int diomp_set_bcast_chain_min(uint64_t bytes);
int diomp_set_bcast_pullchain(int32_t on);
int diomp_set_allreduce_ce_min(uint64_t bytes);
/* NVSwitch multicast (NVLS) allreduce: the switch reduces (multimem.ld_reduce)
 * and one multimem.st fans the result out.  Float sums agree with the
 * reference fold within rounding (not bitwise); integer sum/min/max exact;
 * float min/max refused.  Setup is collective over the communicator
 * (position 0 creates the multicast object, exports a POSIX fd, members
 * import, add their GPU, bind a window of their HBM).                      */
int diomp_mc_supported(int device, int *out);
int diomp_mc_window_bytes(int nmembers, uint64_t want, uint64_t *total_out);
int diomp_mc_create(int nmembers, uint64_t total, int *fd_out, uint64_t *mc_out);
int diomp_mc_import(int fd, uint64_t *mc_out);
int diomp_mc_add_device(uint64_t mc, int device);
int diomp_mc_bind(uint64_t mc, int device, uint64_t total, uint64_t *uc_out, uint64_t *mc_va_out,
                  uint64_t *phys_out);
int diomp_mc_release(uint64_t mc, int device, uint64_t total, uint64_t uc, uint64_t mc_va,
                     uint64_t phys);
typedef struct {
    int32_t device, k, pos, dtype, op, _pad;
    uint64_t uc, mc;      /* window: own unicast VA / multicast VA (2 MiB flag header first) */
    uint64_t window;      /* data bytes per round (window size minus the header) */
    uint64_t send, recv;  /* own device pointers, 16 B aligned; recv may equal send */
    uint64_t count;       /* elements */
    uint64_t epoch;       /* rounds completed on this window so far (all members equal) */
    uint64_t counter;     /* u32 last-CTA counter in own memory */
} diomp_nvls_args;
int diomp_allreduce_nvls(const diomp_nvls_args *args, void *stream);
int diomp_nvls_rounds(uint64_t count, int dtype, uint64_t window, uint64_t *rounds_out);
#endif /* DIOMP_EXPERIMENTS */

/* ---- Minimod stencil: kernels/__init__.py:30 seam `stencil_update`
 *      (reference.py:14-31 / _core.pyx:9-32).  One interior update of
 *      (NX, NY, NZ) C-order f64 arrays, ghost width `radius` (<= 8); u_next may
 *      alias u_prev.  Bit-identical to the reference (no FMA, fixed order).  */
typedef struct {
    uint64_t u_next, u_cur, u_prev;
    int64_t NX, NY, NZ;
    int32_t radius;
    int32_t _pad;
    double center;
    double wx[9], wy[9], wz[9];
} diomp_stencil_args;
int diomp_stencil_update(int device, const diomp_stencil_args *args, void *stream);

/* Fused driver step (apps/stencil.py:113-126 + apps/halo_onesided.py:12-25):
 * update + point source + halo planes stored straight into the neighbours'
 * ghost planes + per-step neighbour flags.  field[0]/field[1] are the two
 * local buffers (field_a / field_b of stencil.py:85-86); left/right are the
 * neighbours' same buffers as addressable from `device` (0 = no neighbour).
 * Step s uses prev=field[s%2], cur=field[(s+1)%2].                            */
typedef struct {
    int32_t device;
    int32_t radius;       /* must be 4 */
    int64_t NX, NY, NZ;   /* local extents incl. ghosts: NX = nxl + 2R */
    uint64_t field[2];
    uint64_t left_field[2];
    uint64_t right_field[2];
    int64_t src_i, src_j, src_k; /* local index of the point source, src_i < 0: none */
    double amp;
    double center;
    double w[5];
    /* device sync (sync != 0): wait own flag slots, signal neighbours' slots */
    int32_t sync;
    int32_t _pad;
    uint64_t wait_left, wait_right;     /* own flag addresses written by the neighbours */
    uint64_t sig_left, sig_right;       /* neighbours' flag addresses I write            */
    uint64_t from_left, from_right;     /* signals already received per neighbour         */
    uint64_t to_left, to_right;         /* signals already sent per neighbour             */
    uint64_t counter;                   /* u32 in own segment (last-CTA detection)        */
} diomp_stencil_plan;
/* Launch steps [step0, step0+nsteps) on `stream`.  With sync, every call
 * raises nsteps + 1 signals per neighbour (an entry signal, then one per
 * finished step) and waits for as many; the caller advances the from/to
 * counters by nsteps + 1.  The entry handshake means no halo store of this
 * call can land in a neighbour's ghost planes before the neighbour's stream
 * reached the call (its field initialisation / H2D copies are complete).
 * sync = 0 with neighbour fields set is the host-ordered fused mode (one
 * step per call, host barrier between calls); it needs the TMA fast path
 * (R = 4, even NZ, 16 B aligned) and returns DIOMP_BAD_REQUEST otherwise. */
int diomp_stencil_run(const diomp_stencil_plan *plan, int64_t step0, int64_t nsteps,
                      void *stream);

/* ---- matmul: kernels/__init__.py:31 seam `matmul_f64` (_core.pyx:35-46):
 *      c = a @ b with a k-ordered left fold per element, no FMA (bit-exact). */
int diomp_matmul_f64(int device, int64_t n, int64_t k, int64_t m, uint64_t a, uint64_t b,
                     uint64_t c, void *stream);

/* Row-stripe ring DGEMM step (apps/cannon.py:119-145): C += A_blk @ B on the
 * FP64 tensor cores (DMMA), row-major, FMA accumulation (tolerance, not
 * bit-pinned -- the reference uses BLAS here).  fwd != 0: the kernel also
 * stores every B element exactly once to fwd (the predecessor's spare stripe,
 * peer-mapped), fusing the stripe shift of cannon.py:124-131 into the GEMM.
 * Optional device sync as in the stencil plan (wait on own flags before
 * reading B / writing fwd, last CTA signals).                                */
typedef struct {
    int32_t device;
    int32_t sync;
    int64_t M, N, K;
    uint64_t A, B, C, fwd;
    int64_t lda, ldb, ldc, ldf;
    uint64_t wait_addr[2];
    uint64_t wait_value[2];
    uint64_t sig_addr[2];
    uint64_t sig_value[2];
    uint64_t counter;
} diomp_dgemm_args;
int diomp_dgemm(const diomp_dgemm_args *args, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DIOMP_B200_H */
