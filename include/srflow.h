/*
 * srflow.h - C ABI of the B200-native transfer hot path (libsrflow.so).
 *
 * The reference (rdmaflow, /root/reference/pkg/src/rdmaflow) has no FFI: its
 * boundary is a Python class API.  Every entry point below replaces one
 * reference method on that path; the citation after each declaration names
 * the method (paths relative to pkg/src/rdmaflow/).  All functions return an
 * srf_status (0 = OK); the message of the last failure on the calling thread
 * is available from srf_last_error().  Status codes map 1:1 onto the
 * reference exception classes in errors.py (see SRF_E_* below).
 *
 * Addresses are space-relative byte offsets, exactly like the reference's
 * flat-space addresses (memspace.py:89-133); the device pointer of an address
 * is base + addr.  No torch types cross this boundary.
 */
#ifndef SRFLOW_H
#define SRFLOW_H

#include <stddef.h>
#include <stdint.h>
#include <sys/types.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py class each maps onto) ---------------------- */
enum srf_status {
    SRF_OK = 0,
    SRF_PENDING = 1,             /* not an error: event / flag not ready yet   */
    SRF_E_ZERO_LENGTH = 10,      /* errors.ZeroLength          errors.py:9      */
    SRF_E_OUT_OF_MEMORY = 11,    /* errors.OutOfMemory         errors.py:13     */
    SRF_E_OUT_OF_BOUNDS = 12,    /* errors.OutOfBounds         errors.py:21     */
    SRF_E_NOT_REGISTERED = 13,   /* errors.NotRegistered       errors.py:35     */
    SRF_E_BAD_TOKEN = 14,        /* errors.BadToken            errors.py:39     */
    SRF_E_REMOTE_OOB = 15,       /* errors.RemoteOutOfBounds   errors.py:43     */
    SRF_E_INVALID_LENGTH = 16,   /* errors.InvalidLength       errors.py:47     */
    SRF_E_TIMEOUT = 17,          /* errors.Timeout             errors.py:59     */
    SRF_E_PEER_UNREACHABLE = 18, /* errors.PeerUnreachable     errors.py:31     */
    SRF_E_INVALID_CONFIG = 19,   /* errors.InvalidConfig       errors.py:103    */
    SRF_E_SHAPE_MISMATCH = 20,   /* errors.ShapeMismatch       errors.py:95     */
    SRF_E_PROTOCOL = 21,         /* errors.ProtocolError       errors.py:116    */
    SRF_E_DEVICE = 22            /* CUDA failure -> errors.RdmaFlowError        */
};

typedef struct srf_space  *srf_space_t;   /* one server's HBM pool          */
typedef struct srf_stream *srf_stream_t;  /* one queue pair's CUDA stream   */
typedef struct srf_event  *srf_event_t;   /* one verb's completion          */

/* ---- library -------------------------------------------------------------- */
const char *srf_last_error(void);
int srf_version(void);
int srf_device_count(int *count);
/* pinned host staging (async H2D of metadata blocks, e2e inputs) */
int srf_host_alloc(uint64_t nbytes, void **out);
int srf_host_free(void *ptr);
/* number of sm_100a kernels this library launched since load */
uint64_t srf_launch_count(void);
/* launch-geometry knobs of the copy kernels: 0 = CTAs per SM (1..32),
 * 1 = threads per CTA (128/256/512), 2 = copy implementation (0 vector,
 * 1 TMA bulk), 3 = pool allocator (0 cudaMalloc + CUDA IPC, 1 VMM + fd),
 * 4 = 16-B vectors in flight per thread (4 or 8), 5 = 32-B vectors (0/1),
 * 6 = cross-device bodies >= value KiB move on the copy engine, the tail
 *     flag still released by an SM store after them (0 = never, the default),
 * 7 = force system-scope puts/gets on one device (tests), 8 = credit/flag
 *     timeout in ms, 9 = pipelined-edge CTAs per SM (1..4), 10 = pipelined-
 *     edge chunk KiB (0 = automatic), 11 = flag-only edge consumer threads,
 * 12 = GenGrad work-unit KiB, 13 = flag-only edge consumer clears with a
 *     system-scope release (1) instead of a relaxed store (0, the default),
 * 14 = pipelined-edge CTAs in total (0: knob 9 per SM) */
int srf_tune(int knob, int value);

/* ---- memory spaces (memspace.py) ----------------------------------------- */
/* MemorySpace.__init__ (memspace.py:98-113): one cudaMalloc(capacity) on
 * cuda_device, zero-filled like np.zeros. */
int srf_space_create(int server_id, int cuda_device, uint64_t capacity,
                     uint32_t max_regions, srf_space_t *out);
int srf_space_destroy(srf_space_t space);
int srf_space_info(srf_space_t space, int *server_id, int *cuda_device,
                   uint64_t *capacity, void **device_base);
/* the space's default stream (local compute, byte IO) as cudaStream_t */
void *srf_space_cuda_stream(srf_space_t space);

/* MemorySpace.allocate_region (memspace.py:116-133): bump allocation, 8-B
 * aligned base.  The 64-bit access token is supplied by the host so its
 * random stream stays identical to the reference's. */
int srf_region_alloc(srf_space_t space, uint64_t length, int registered,
                     uint64_t token, int64_t *region_id, uint64_t *base);
int srf_region_count(srf_space_t space, uint32_t *count);
int srf_next_addr(srf_space_t space, uint64_t *next_addr);
/* MemorySpace.check_remote_access (memspace.py:145-157) */
int srf_check_remote(srf_space_t space, uint64_t addr, uint64_t length,
                     uint64_t token);
/* MemorySpace.check_registered (memspace.py:159-167) */
int srf_check_registered(srf_space_t space, uint64_t addr, uint64_t length,
                         uint64_t token);

/* MemorySpace.read_at/read_raw (memspace.py:180-198), D2H, synchronous */
int srf_read(srf_space_t space, uint64_t addr, uint64_t length, void *host_dst);
/* MemorySpace.write_at/write_raw (memspace.py:184-219), H2D, synchronous */
int srf_write(srf_space_t space, uint64_t addr, uint64_t length,
              const void *host_src);
/* H2D from caller-pinned memory, asynchronous on `stream` (NULL = default) */
int srf_write_async(srf_space_t space, uint64_t addr, uint64_t length,
                    const void *host_src, srf_stream_t stream);
int srf_read_async(srf_space_t space, uint64_t addr, uint64_t length,
                   void *host_dst, srf_stream_t stream);
/* MemorySpace.view (memspace.py:188-194): device pointer of an address */
int srf_device_ptr(srf_space_t space, uint64_t addr, void **dptr);
/* wait for all work on the space's default stream; reports device timeouts */
int srf_space_sync(srf_space_t space);

/* ---- peers (fabric.py RdmaDevice.connect, fabric.py:286-303) ----------- */
/* enable NVLink peer access between the two spaces' GPUs (both directions) */
int srf_connect(srf_space_t a, srf_space_t b);
/* multi-process: export the pool (cudaIpcGetMemHandle, 64 bytes) and map a
 * peer's exported pool as a remote space proxy; the proxy's region table is
 * filled with srf_region_import so remote checks stay identical. */
int srf_space_export(srf_space_t space, void *handle64);
/* enable direct peer access from `device` to `peer_device` (same process) */
int srf_enable_peer(int device, int peer_device);
int srf_space_import(const void *handle64, int server_id, int local_device,
                     uint64_t capacity, srf_space_t *out);
/* VMM pools (knob 3 = 1): export the allocation as a POSIX fd and map a
 * peer's fd (obtained through pidfd_getfd / SCM_RIGHTS) as a proxy */
int srf_space_export_fd(srf_space_t space, int *fd);
int srf_space_import_fd(int fd, int server_id, int local_device, uint64_t capacity,
                        srf_space_t *out);
int srf_region_import(srf_space_t proxy, int64_t region_id, uint64_t base,
                      uint64_t length, int registered, uint64_t token);

/* ---- streams and completions (fabric.py CompletionQueue/_finish_verb) --- */
int srf_stream_create(srf_space_t space, srf_stream_t *out);
int srf_stream_destroy(srf_stream_t stream);
void *srf_stream_cuda(srf_stream_t stream);
int srf_stream_sync(srf_stream_t stream);
int srf_event_record(srf_space_t space, srf_stream_t stream, srf_event_t *out);
/* SRF_OK when complete, SRF_PENDING otherwise (Channel.take_completion poll) */
int srf_event_query(srf_event_t ev);
int srf_event_wait(srf_event_t ev);
int srf_event_wait_free(srf_event_t ev);  /* take_completion: wait, then release */
int srf_event_free(srf_event_t ev);

/* CUDA-graph capture of a stream's launches (many-small-transfer steps are
 * launch-bound: SURVEY.md H5) and timing events for the benchmark. */
int srf_graph_begin(srf_stream_t stream);
int srf_graph_end(srf_stream_t stream, void **graph_exec);
int srf_graph_launch(void *graph_exec, srf_stream_t stream);
int srf_graph_destroy(void *graph_exec);
int srf_stream_wait_event(srf_stream_t stream, srf_event_t ev);
/* Order the space's own stream after an event (BufferRef frees: a block
 * freed while device work may still use it carries a fence event; the next
 * allocation that reuses those bytes makes the space's stream wait on it -
 * memspace.py:315-357 frees at refcount 0, which stays host-immediate so the
 * first-fit addresses equal the reference's). */
int srf_space_wait_event(srf_space_t space, srf_event_t ev);
int srf_timing_event_create(srf_space_t space, srf_event_t *out);
int srf_event_record_on(srf_event_t ev, srf_stream_t stream);
int srf_event_elapsed_ms(srf_event_t start, srf_event_t end, float *ms);

/* ---- verbs: the hot path ------------------------------------------------- */
/* Channel.one_sided_write (fabric.py:349-369) + _deliver_chunks (:391-421).
 * K1 static_put / K3 meta_put.  Gathers nseg local registered ranges
 * (src_addr[i], src_len[i], src_token[i]) of src_space into
 * [dst_addr, dst_addr + sum(len)) of dst_space.  Every byte but the last is
 * written by 16-B vector stores from all CTAs; after a system-scope fence and
 * a grid arrival count the last CTA writes the final byte (the tail flag of
 * wire.py:74-76 / :112-116) with st.release.sys, so an observed flag implies a
 * complete payload - the guarantee ascending delivery gave the reference.
 * flags: SRF_PUT_WAIT_EMPTY makes every CTA acquire-spin until the remote
 * tail byte reads 0x00 (receiver consumed) before writing.
 * ev_out may be NULL. */
#define SRF_PUT_WAIT_EMPTY 0x1
int srf_put(srf_space_t src_space, const uint64_t *src_addr,
            const uint64_t *src_len, const uint64_t *src_token, int nseg,
            srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
            int flags, srf_stream_t stream, srf_event_t *ev_out);
/* srf_put + this rank's own receive poll in ONE launch (device loops where
 * each rank sends and receives every round): after the tail release, the
 * last CTA acquire-spins on rcv_flag_addr of rcv_space (local) and clears it
 * (K2 fused). */
int srf_put_consume(srf_space_t src_space, const uint64_t *src_addr, const uint64_t *src_len,
                    const uint64_t *src_token, int nseg, srf_space_t dst_space,
                    uint64_t dst_addr, uint64_t dst_token, int flags, srf_space_t rcv_space,
                    uint64_t rcv_flag_addr, srf_stream_t stream, srf_event_t *ev_out);
/* Channel.one_sided_read (fabric.py:371-389).  K4 peer_pull: launched on the
 * reader's GPU, loads [src_addr, +length) from the peer pool, stores into the
 * local registered range dst_addr. */
/* K3 with the block inline: DynSender.send's metadata (runtime/protocol.py:
 * 163-201).  The `len` (<= 1024) bytes are a kernel parameter - no staging
 * copy from the host - and one launch writes them into the sender's
 * registered stage block [stage_addr, +len) (write_at(meta_stage)) and into
 * [dst_addr, +len) of dst_space, last byte released last (and mirrored to the
 * receiver's host doorbell).  Same checks and flags as srf_put. */
int srf_put_inline(srf_space_t src_space, uint64_t stage_addr, uint64_t stage_token,
                   const void *bytes, uint32_t len, srf_space_t dst_space, uint64_t dst_addr,
                   uint64_t dst_token, int flags, srf_stream_t stream, srf_event_t *ev_out);
int srf_get(srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
            srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
            uint64_t length, srf_stream_t stream, srf_event_t *ev_out);
/* MemorySpace.copy_bytes (memspace.py:223-236).  K5 stage_copy, local D2D. */
int srf_copy(srf_space_t space, uint64_t src_addr, uint64_t dst_addr,
             uint64_t length, srf_stream_t stream, srf_event_t *ev_out);
/* StaticReceiver.poll (runtime/protocol.py:124-138) as a device consumer
 * prologue.  K2 flag_wait: one warp acquire-spins on the byte at flag_addr
 * until it equals `expect`, then (clear != 0) stores 0x00.  Bounded by
 * timeout_ns; a timeout is reported by the next srf_space_sync. */
int srf_flag_wait(srf_space_t space, uint64_t flag_addr, uint8_t expect,
                  int clear, uint64_t timeout_ns, srf_stream_t stream);

/* Device consumer used by the release/acquire stress test and the
 * microbenchmark: thread 0 acquire-spins on flag_addr (== 0x01), then the
 * CTA computes sum(data[i] * (i % 251 + 1)) over n bytes into the u64 at
 * out_addr and clears the flag.  Same bounded-timeout reporting as K2. */
int srf_consume_checksum(srf_space_t space, uint64_t flag_addr, uint64_t data_addr,
                         uint64_t n, uint64_t out_addr, uint64_t timeout_ns,
                         srf_stream_t stream);

/* ---- host doorbells (polling without a CUDA call) -------
 * srf_doorbell_bind gives a receive region (static payload||flag, or a
 * metadata block with mirror != 0) a pinned, host-mapped shadow.  Every
 * srf_put from this process into that region also writes the shadow from its
 * last CTA (the block, then the flag, st.release.sys), so
 * StaticReceiver.poll / DynReceiver.poll (protocol.py:124-138, :234-242) read
 * host memory instead of copying from the device.  srf_flag_read falls back
 * to a device read when no doorbell is bound or the space was exported to
 * other processes.  srf_flag_clear clears the shadow and (asynchronously, on
 * the space's stream) the device byte; the next srf_put into the region waits
 * for that clear. */
int srf_doorbell_bind(srf_space_t space, uint64_t region_addr, uint64_t region_len,
                      int mirror);
int srf_flag_read(srf_space_t space, uint64_t tail_addr, uint64_t len, void *host_out);
int srf_flag_clear(srf_space_t space, uint64_t tail_addr);

/* graph.py apply_in_place (graph.py:392-405) for W workers in one pass.
 * K6 ps_apply:  op SRF_APPLY_XOR: var ^= g_0 ^ ... ^ g_{W-1} (bytewise)
 *               op SRF_APPLY_SGD: var = (((var - lr*g_0) - lr*g_1) ...) fp32,
 *                                 every product and difference rounded
 *                                 separately (no FMA contraction).
 * Gradients may live in peer pools (fused pull + apply). */
#define SRF_APPLY_XOR 0
#define SRF_APPLY_SGD 1
#define SRF_MAX_WORKERS 16
int srf_apply(srf_space_t var_space, uint64_t var_addr, uint64_t nbytes,
              srf_space_t const *grad_spaces, const uint64_t *grad_addrs,
              int nworkers, int op, float lr, srf_stream_t stream,
              srf_event_t *ev_out);

/* GenGrad / Input values on the device (graph.py:333-350 node_rng +
 * synthesize_values, used by compute_node graph.py:363-370): elements
 * [elem_offset, elem_offset + nelems) of
 *   Generator(PCG64(((seed & 0xFFFFFFFF)*1000003 + node)*1000033 + iteration))
 *     .random(n, dtype=float32)
 * bit-exact (numpy's SeedSequence seeding, PCG64 XSL-RR, 24-bit floats), into
 * fp32 elements at addr (4-B aligned) of the space, on its stream. */
int srf_gen_reference(srf_space_t space, uint64_t addr, uint64_t nelems, uint64_t elem_offset,
                      uint64_t seed, uint64_t node, uint64_t iteration, srf_stream_t stream,
                      srf_event_t *ev_out);

/* ---- batched PS step (configs[2..4]) ------------------------------------
 * One launch per phase per step over descriptor lists that are validated
 * once at creation (registration, token and bounds checks of every edge, the
 * same gates srf_put applies per verb).  Phases of one PS iteration
 * (runtime/session.py:606-629 over workloads.py:59-94):
 *   put batch   - K1 weight pushes shard -> workers (static placement) and
 *                 K3 metadata writes workers -> shards (dynamic allocation);
 *                 body then tail byte released last; flags SRF_PUT_WAIT_EMPTY
 *   gen batch   - per worker x variable: acquire the weight flag (consume +
 *                 clear, StaticReceiver.poll), wait for the shard's credit
 *                 (meta flag clear), then (mode 1) produce the gradient
 *                 on the device - the reference's own PCG64 GenGrad stream
 *                 (graph.py:333-350), bit-exact, as srf_gen_reference - or
 *                 (mode 0) keep a host-uploaded one
 *   apply batch - per variable: DynReceiver.poll + decode_meta + validation
 *                 on the device, then K4+K6 fused: the update reads every
 *                 remote gradient straight through the peer mapping (no
 *                 local copy) and folds all workers in ascending order
 *                 (XOR or SGD); clears the meta flags.
 * Descriptor arrays are parallel; for the apply batch the per-(variable,
 * worker) arrays are flattened in ascending worker order. */
typedef struct srf_batch *srf_batch_t;
int srf_batch_put_create(int n, srf_space_t const *src_space, const uint64_t *src_addr,
                         const uint64_t *body_len, const uint64_t *src_token,
                         const uint64_t *tail_addr, srf_space_t const *dst_space,
                         const uint64_t *dst_addr, const uint64_t *dst_token, int flags,
                         srf_batch_t *out);
int srf_batch_gen_create(int n, srf_space_t const *space, const uint64_t *grad_addr,
                         const uint64_t *nbytes, const uint64_t *weight_flag_addr,
                         srf_space_t const *credit_space, const uint64_t *credit_addr,
                         const uint64_t *node_id, uint64_t seed, srf_batch_t *out);
int srf_batch_apply_create(srf_space_t space, int nvars, const uint64_t *var_addr,
                           const uint64_t *nbytes, const int *nworkers, const int *rank,
                           srf_space_t const *src_space, const uint64_t *src_addr,
                           const int *is_meta, srf_space_t const *peer_space,
                           const uint64_t *peer_lo, const uint64_t *peer_hi,
                           const uint64_t *peer_token, int op, float lr, srf_batch_t *out);
/* grid_cap > 0 bounds the grid (CTAs loop over the batch's work units) */
int srf_batch_launch(srf_batch_t batch, srf_stream_t stream, uint64_t iteration, int mode,
                     int grid_cap);
int srf_batch_destroy(srf_batch_t batch);
/* graph-replayed PS steps: a gen batch launched with iteration == UINT64_MAX
 * reads the iteration from the u64 at addr of space; srf_counter_add bumps it
 * (one thread, stream-ordered) at the end of each captured step */
int srf_batch_set_iteration_source(srf_batch_t batch, srf_space_t space, uint64_t addr);
int srf_counter_add(srf_space_t space, uint64_t addr, uint64_t delta, srf_stream_t stream);
/* `iters` PS iterations (it0, it0+1, ...) in ONE cooperative launch when every
 * server lives on this GPU: the four phases run back to back separated by
 * grid-wide barriers; flags and credits are used exactly as in the per-phase
 * launches (latency-bound configs: the MLP parity set) */
int srf_ps_persistent(srf_batch_t push, srf_batch_t gen, srf_batch_t meta,
                      srf_batch_t const *apply, int napply, srf_stream_t stream, uint64_t it0,
                      uint32_t iters, int mode);

/* Exchange schedule: one launch per PS iteration in which persistent CTAs
 * claim the work units of this GPU's push, gen and apply batches from ONE
 * queue ordered by a per-edge key (every rank derives the same keys from the
 * variable, e.g. push(v) < gen(v) < apply(v) < ...).  A unit waits only on
 * units earlier in that global order, so any grid makes progress, and a shard
 * pulls variable v while later weights are still in flight.  The gen batch
 * must carry its metadata puts (srf_batch_gen_set_meta: gen edge
 * gen_index[i] sends meta edge i from its last CTA - DynSender.send after the
 * producer, runtime/protocol.py:163-201). */
typedef struct srf_exchange *srf_exchange_t;
int srf_batch_gen_set_meta(srf_batch_t gen, int n, const int *gen_index, srf_batch_t meta);
/* co-located worker/shard (the apply reads the gradient in place): gen edge i
 * releases the byte at ready_addr[i] of space[i] to 1 when its gradient is
 * complete and waits for 0 before overwriting it; the apply waits for 1 and
 * clears it (srf_batch_apply_set_ready, one entry per (variable, worker) edge
 * in creation order, UINT64_MAX = none).  Needed by the exchange schedule,
 * where an apply unit may be claimed while the gradient is still produced. */
int srf_batch_gen_set_ready(srf_batch_t gen, srf_space_t const *space,
                            const uint64_t *ready_addr);
int srf_batch_apply_set_ready(srf_batch_t apply, srf_space_t space, const uint64_t *ready_addr);
/* static gradient pushes (the reference's mechanism_override="static",
 * runtime/session.py:368): put edge i first waits until the byte at
 * ready_addr[i] of space[i] (same GPU) reads 1 - its gen released the
 * gradient - and clears it to 0 once the body is copied, the gen's credit.
 * UINT64_MAX = none. */
/* Fused weight push (extension, ps.PsStep(fuse_push=True)): apply batch
 * descriptor v also writes its updated variable into nfwd[v] workers' static
 * receive regions (fwd_*: space / payload address / token, flag after the
 * payload) and releases their flags with the byte at tail_addr - the next
 * iteration's StaticSender.send of the weights (runtime/protocol.py:63-91)
 * folded into this iteration's ApplyGrad (graph.py:392-405).  Active only in
 * srf_batch_launch calls with mode bit 0 set. */
int srf_batch_apply_set_forward(srf_batch_t apply, const int *nfwd,
                                srf_space_t const *fwd_space, const uint64_t *fwd_addr,
                                const uint64_t *fwd_token, srf_space_t tail_space,
                                uint64_t tail_addr);
int srf_batch_put_set_src_ready(srf_batch_t put, srf_space_t const *space,
                                const uint64_t *ready_addr);
/* partitioned variables (extension): gen edge i produces elements
 * elem_offset[i] ... of its model variable's gradient stream */
int srf_batch_gen_set_offsets(srf_batch_t gen, const uint64_t *elem_offset);
int srf_ps_exchange_create(srf_batch_t push, const uint64_t *push_key, srf_batch_t gen,
                           const uint64_t *gen_key, srf_batch_t const *apply, int napply,
                           const uint64_t *apply_key, srf_exchange_t *out);
int srf_ps_exchange_launch(srf_exchange_t exchange, srf_stream_t stream, uint64_t iteration,
                           int regen);
/* iterations iteration, iteration+1, ... in ONE launch: the queue repeats,
 * and push edge i of a later iteration first waits until its variable's
 * apply (global apply descriptor push_apply_index[i] across the apply
 * batches in creation order, -1: none) completed for the previous one
 * (srf_ps_exchange_link must have been called). */
int srf_ps_exchange_link(srf_exchange_t exchange, const int *push_apply_index);
/* regen bit 0: GenGrad regenerates; bit 1: the apply units also write the
 * next weights (srf_batch_apply_set_forward; the exchange then carries no
 * weight pushes - build it without them). */
int srf_ps_exchange_launch_n(srf_exchange_t exchange, srf_stream_t stream, uint64_t iteration,
                             uint32_t iterations, int regen);
int srf_ps_exchange_destroy(srf_exchange_t exchange);

/* Device-side DynReceiver.poll + fetch (runtime/protocol.py:224-254): acquire
 * the metadata flag of the block at meta_addr (rank-D layout, wire.py:79-142),
 * validate it like decode_meta + check_remote_access (token, [peer_lo,
 * peer_hi) of peer, payload_len == prod(dims) * elem size, <= dst_cap),
 * pull the bytes into [dst_addr, +len) (K4), store len at len_out_addr
 * (UINT64_MAX: none; all ones on a rejected block) and clear the flag.
 * Rejections raise SRF_E_BAD_TOKEN at the next sync. */
int srf_dyn_recv(srf_space_t receiver, uint64_t meta_addr, int rank, srf_space_t peer,
                 uint64_t peer_lo, uint64_t peer_hi, uint64_t peer_token, uint64_t dst_addr,
                 uint64_t dst_cap, uint64_t len_out_addr, srf_stream_t stream);

/* Registered pool behind torch's CUDA allocator (torch.cuda.memory.
 * CUDAPluggableAllocator over srf_torch_malloc / srf_torch_free): every torch
 * tensor of that GPU lives in [region_addr, +length) of the space, so it can
 * be sent or received zero-copy (analyzer.py:226-272).
 * Freed blocks are reused only after the freeing stream passed them.  A GPU
 * without a pool, or a request the pool cannot hold, gets plain cudaMalloc
 * memory (torch works; zero-copy verbs on it are refused as NotRegistered). */
int srf_torch_pool_attach(srf_space_t space, uint64_t region_addr, uint64_t length);
int srf_torch_pool_stats(int cuda_device, uint64_t *in_use, uint64_t *peak,
                         uint64_t *capacity);
void *srf_torch_malloc(ssize_t size, int cuda_device, void *cuda_stream);
void srf_torch_free(void *ptr, ssize_t size, int cuda_device, void *cuda_stream);

/* RPC-style serialize/copy baseline (runtime/protocol.py:257-448) on the
 * device - the comparator the north star reports zero-copy against.  The
 * stream metadata||payload moves in 4096-B fragments (16-B header + 4080 B)
 * through a 16-slot ring of posted 4-KiB receive slots in dst: a sender CTA
 * serialises each fragment into its staging slot (counted copy 1) and writes
 * it into a free ring slot; a receiver CTA checks the header, copies it out
 * into meta_out / tensor_out (counted copy 2) and re-posts the slot.  Same
 * GPU: one cooperative launch; two GPUs: one launch per side. */
int srf_rpc_transfer(srf_space_t src, uint64_t meta_addr, uint32_t meta_len,
                     uint64_t payload_addr, uint64_t payload_len, uint64_t stage_addr,
                     srf_space_t dst, uint64_t ring_addr, uint64_t ring_flags_addr,
                     uint64_t meta_out_addr, uint64_t tensor_out_addr, uint64_t msg_id,
                     srf_stream_t src_stream, srf_stream_t dst_stream);

/* MatMul compute kind of Session graphs (graph.py:371-372) on the device,
 * bit-identical to numpy's `a @ b`: an ascending-k FMA chain per output
 * (floats), wrapping sums (integers).  Plain device pointers (row-major
 * a[m,k], b[k,n], c[m,n]), element type code as wire.ElemType (0 F32, 1 F64,
 * 2 I32, 3 I64, 4 U8), launched on cuda_stream. */
int srf_matmul(int elem, uint64_t a_ptr, uint64_t b_ptr, uint64_t c_ptr, uint64_t m, uint64_t k,
               uint64_t n, void *cuda_stream);

/* The compute kinds of Session graphs on the device, operands and result in
 * one space (graph.py:371-377): kind 0 MatMul a[m,k] @ b[k,n] (as srf_matmul),
 * kind 1 Add a + b over n elements of equal shape (integers wrap), kind 2
 * Sigmoid (1 / (1 + exp(-x as float64))) rounded to the float type.  The
 * result is written straight into the output block (no staging). */
int srf_compute(srf_space_t space, int kind, int elem, uint64_t a_addr, uint64_t b_addr,
                uint64_t out_addr, uint64_t m, uint64_t k, uint64_t n, srf_stream_t stream);

/* Add with numpy broadcasting (graph.py:373-374, compute_node ADD): a[a_dims] +
 * b[b_dims], equal rank <= 8, each dimension pair equal or one of them 1;
 * the result has the broadcast shape. */
int srf_add_bcast(srf_space_t space, int elem, uint64_t a_addr, const uint64_t *a_dims,
                  uint64_t b_addr, const uint64_t *b_dims, int rank, uint64_t out_addr,
                  srf_stream_t stream);

/* ConcatDyn (graph.py:383-389, compute_node): the n_in inputs (space addresses, byte
 * lengths; 1..8 of them, not all empty) concatenated and repeated to fill
 * out_len bytes at out_addr, on the device. */
int srf_concat_tile(srf_space_t space, int n_in, const uint64_t *in_addr,
                    const uint64_t *in_len, uint64_t out_addr, uint64_t out_len,
                    srf_stream_t stream);

/* ReduceMax consumer of the microbenchmark (graph.py:378-382) on the
 * receiving GPU: out_addr receives max over n fp32 at in_addr. */
int srf_reduce_max_f32(srf_space_t space, uint64_t in_addr, uint64_t n,
                       uint64_t out_addr, srf_stream_t stream);

/* ---- pipelined static edge (EXTENSION of static placement) ---------------
 * One edge, `slots` pre-placed receive regions (slot i = payload || flag at
 * dst_addr + i * slot_stride, allocated and published by the receiver like
 * the reference's static region, analyzer.py:149-220).  srf_edge_send queues
 * `rounds` transfers in ONE persistent launch: round j (counting continues
 * across calls) puts payload j % nsrc (src_addr + (j % nsrc) * src_stride)
 * into slot j % slots with the reference's per-round protocol - the credit
 * (the slot's flag was cleared by its consumer, runtime/protocol.py:102-111),
 * the body, the flag byte released last (fabric.py:349-356) - but rounds
 * overlap: chunks of round j+1 stream while round j is published and
 * consumed (device_stream.cuh).  srf_edge_consume is the receiver's
 * StaticReceiver.poll for rounds [first, first + rounds) on the device (one
 * CTA; mode 1 also stores a weighted byte checksum of every round's payload
 * at sums_addr, 8 B per round).  Creation checks registration and token and
 * bounds of the whole source and slot spans, like srf_put per verb.
 * credit_addr (UINT64_MAX: none): 4 * slots bytes of the SENDER's pool; the
 * consumer, given the same words (credit_space = its mapping of the sender's
 * pool), stores each slot's consumed-use count there right after clearing
 * the flag, and the sender reads that local copy of the credit instead of
 * loading the remote flag over NVLink every round. */
typedef struct srf_edge *srf_edge_t;
int srf_edge_create(srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
                    uint64_t nbytes, uint32_t nsrc, uint64_t src_stride,
                    srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
                    uint32_t slots, uint64_t slot_stride, uint64_t credit_addr,
                    srf_edge_t *out);
int srf_edge_info(srf_edge_t edge, uint64_t *chunk, uint32_t *nchunks, int *ctas,
                  uint64_t *next_round);
/* diagnostics: released[slots] | arrival[slots] | credit[slots] | claim | exit */
int srf_edge_state(srf_edge_t edge, uint32_t *host_out, uint32_t nwords);
int srf_edge_send(srf_edge_t edge, uint32_t rounds, srf_stream_t stream, srf_space_t src_space);
int srf_edge_consume(srf_space_t receiver, uint64_t slots_addr, uint32_t slots,
                     uint64_t slot_stride, uint64_t nbytes, uint64_t first_round,
                     uint32_t rounds, int mode, uint64_t sums_addr, srf_space_t credit_space,
                     uint64_t credit_addr, srf_stream_t stream);
int srf_edge_destroy(srf_edge_t edge);

/* Pull edge (EXTENSION, same per-slot protocol driven by the receiver): the
 * receiver's GPU pulls round j's payload from the sender's source j % nsrc
 * (src_space: the receiver's mapping of the sender's pool) straight into its
 * pre-placed slot j % slots - peer loads, or TMA bulk copies with tma = 1 -
 * and releases the slot's flag last, like StaticSender.send's final byte
 * (fabric.py:349-356); consumers are the same srf_edge_consume.  Round j
 * starts once the sender posted it: srf_edge_post raises the 8-B word at
 * posted_addr of the receiver's pool (one system-scope release store,
 * the role of the write's arrival in runtime/protocol.py:63-91), optionally
 * after waiting until the source it reuses was fully pulled (pulled_addr:
 * 4 * nsrc B of the sender's pool receiving each source's pulled-use count,
 * UINT64_MAX: none - the same credit as the slot flag, for the sender's
 * buffer; fabric.py:371-389 is the one-sided read these pulls replace). */
int srf_edge_create_pull(srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
                         uint64_t nbytes, uint32_t nsrc, uint64_t src_stride,
                         srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
                         uint32_t slots, uint64_t slot_stride, uint64_t posted_addr,
                         uint64_t pulled_addr, int tma, srf_edge_t *out);
int srf_edge_recv(srf_edge_t edge, uint32_t rounds, srf_stream_t stream, srf_space_t dst_space);
int srf_edge_post(srf_space_t snd_space, srf_space_t rcv_space, uint64_t posted_addr,
                  uint64_t count, uint64_t wait_addr, uint32_t need, srf_stream_t stream);

/* Pipelined dynamic edge (EXTENSION of dynamic allocation, runtime/protocol.py
 * :147-254): `slots` metadata blocks on the receiver (8D+33 B each, the
 * layout of encode_meta, wire.py:109-119).  srf_dyn_edge_send (sender GPU,
 * one thread) writes round j's block into slot j % slots once its flag reads
 * 0 - dims, element code, the payload's space address (src_addr + (j % nsrc) *
 * src_stride), token and length, flag released last.  srf_dyn_edge_recv (one
 * persistent TMA launch on the receiver) acquires each block, validates it
 * like decode_meta + check_remote_access (wire.py:122-144,
 * memspace.py:145-157; a bad block sets the space's error), allocates the
 * round's block on demand from a device ring arena in round order, and pulls
 * the payload from the sender's pool into it (fabric.py:371-389).
 * srf_dyn_edge_consume consumes rounds in order (mode 1: byte checksums),
 * frees their ring blocks and clears the metadata flags (the credits). */
typedef struct srf_dyn_edge *srf_dyn_edge_t;
int srf_dyn_edge_create(srf_space_t src_space, uint64_t lo, uint64_t hi, uint64_t token,
                        uint64_t max_bytes, uint32_t rank, srf_space_t dst_space,
                        uint64_t meta_addr, uint64_t meta_stride, uint32_t slots,
                        uint64_t ring_addr, uint64_t ring_cap, srf_dyn_edge_t *out);
int srf_dyn_edge_recv(srf_dyn_edge_t edge, uint32_t rounds, srf_stream_t stream,
                      srf_space_t dst_space);
int srf_dyn_edge_consume(srf_dyn_edge_t edge, srf_space_t dst_space, uint64_t first_round,
                         uint32_t rounds, int mode, uint64_t sums_addr, srf_stream_t stream);
int srf_dyn_edge_send(srf_space_t snd_space, srf_space_t rcv_space, uint64_t meta_addr,
                      uint64_t meta_stride, uint32_t slots, uint32_t rank, int elem,
                      const uint64_t *dims, uint64_t src_addr, uint64_t src_stride,
                      uint32_t nsrc, uint64_t src_token, uint64_t first_round, uint32_t rounds,
                      srf_stream_t stream);
int srf_dyn_edge_destroy(srf_dyn_edge_t edge);

/* ---- Session iteration recording and replay (runtime/session.py:606-629) --
 * srf_record_begin / srf_record_end capture every device launch the library
 * makes in between (puts, pulls, inline metadata puts, GenGrad, updates,
 * ReduceMax, MatMul, receivers' flag clears) with their exact arguments;
 * *replayable is 0 when something outside that set happened (a host write into
 * device memory, a copy-engine body, another kernel, a second GPU).
 * srf_oplist_same: 1 when b repeats a with every GenGrad iteration advanced by
 * gen_delta.  srf_oplist_replay: `count` more iterations of the recording as
 * one CUDA graph each on `stream` (a stream of the recording's GPU), GenGrad
 * iterations advanced by first_offset, first_offset + 1, ...; the stream
 * serialises what the host path serialised with its completion waits. */
typedef struct srf_oplist *srf_oplist_t;
int srf_record_begin(void);
int srf_record_end(srf_oplist_t *out, int *replayable);
/* the caller launched device work outside the library during the recording */
int srf_record_taint(const char *why);
int srf_oplist_info(srf_oplist_t list, uint32_t *nops, int *cuda_device, char *why,
                    uint32_t why_len);
int srf_oplist_same(srf_oplist_t a, srf_oplist_t b, int64_t gen_delta);
/* diagnostics: where b stops repeating a, as text */
int srf_oplist_diff(srf_oplist_t a, srf_oplist_t b, int64_t gen_delta, char *out, uint32_t len);
int srf_oplist_replay(srf_oplist_t list, uint64_t first_offset, uint32_t count,
                      srf_stream_t stream);
int srf_oplist_destroy(srf_oplist_t list);
/* All phases of a steady-state period behind ONE instantiated graph: lists[p]
 * recorded at iteration iters[p]; edges = the union of every phase's byte-range
 * conflicts; srf_replay_set_launch updates only the nodes whose arguments
 * differ from the phase last launched, then launches (runtime/session.py:
 * 606-629 replayed for periods too long to instantiate one graph each). */
typedef struct srf_replay_set *srf_replay_set_t;
int srf_replay_set_create(srf_oplist_t *lists, const int64_t *iters, uint32_t nphase,
                          srf_replay_set_t *out);
int srf_replay_set_launch(srf_replay_set_t set, uint32_t phase, uint64_t iteration,
                          srf_stream_t stream);
int srf_replay_set_info(srf_replay_set_t set, uint32_t *nodes, uint32_t *edges,
                        uint32_t *classes, uint64_t *updates);
int srf_replay_set_destroy(srf_replay_set_t set);

#ifdef __cplusplus
}
#endif
#endif /* SRFLOW_H */
