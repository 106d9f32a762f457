// abi_stream.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// C ABI: the pipelined static edge (device_stream.cuh).

struct srf_edge {
  int device;
  StreamEdgeArgs a;        // fixed fields; first_round / rounds set per launch
  unsigned int *state;     // released[slots] | arrival[slots] | credit[slots] | claim | exit
  uint64_t next_round;
  int ctas;
  int pull = 0;            // 1: a pull edge (k_pull_stream on the receiver's GPU)
  int pre = 0;             // 1: few slots - k_pull_stream_pre stages chunks early
};


extern "C" {

int srf_edge_create(srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
                    uint64_t nbytes, uint32_t nsrc, uint64_t src_stride,
                    srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
                    uint32_t slots, uint64_t slot_stride, uint64_t credit_addr,
                    srf_edge_t *out) {
  DeviceGuard device_guard;
  if (nbytes < 1) return fail(SRF_E_INVALID_LENGTH, "zero-length edge");
  if (slots < 1 || nsrc < 1) return fail(SRF_E_INVALID_CONFIG, "slots and nsrc must be >= 1");
  if (slot_stride < nbytes + 1 || (nsrc > 1 && src_stride < nbytes))
    return fail(SRF_E_INVALID_CONFIG, "slot/source stride shorter than the payload");
  if (src_space->imported) return fail(SRF_E_INVALID_CONFIG, "the sender's payloads are local");
  const uint64_t src_span = (uint64_t)(nsrc - 1) * src_stride + nbytes;
  const uint64_t dst_span = (uint64_t)(slots - 1) * slot_stride + nbytes + 1;
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    int rc = check_registered_locked(src_space, src_addr, src_span, src_token);
    if (rc) return rc;
  }
  {
    std::lock_guard<std::mutex> g(dst_space->mu);
    int rc = check_remote_locked(dst_space, dst_addr, dst_span, dst_token);
    if (rc) return rc;
  }
  srf_edge *e = new srf_edge();
  e->device = src_space->device;
  memset(&e->a, 0, sizeof e->a);
  e->a.src = src_space->base + src_addr;
  e->a.src_stride = src_stride;
  e->a.nsrc = nsrc;
  e->a.dst = dst_space->base + dst_addr;
  e->a.slot_stride = slot_stride;
  e->a.slots = slots;
  e->a.nbytes = nbytes;
  // chunk: S/16 within [64 KiB, 256 KiB] - large enough to amortise a work
  // item's claim, credit check and system-scope arrival, small enough that a
  // round spreads over many CTAs (tools/edge_probe.py sweep,
  // profiles/r2s_edge_slots.jsonl)
  const int sms = sm_count_of(e->device);
  e->ctas = g_edge_ctas ? g_edge_ctas : std::max(1, sms * g_edge_ctas_per_sm);
  uint64_t chunk = g_edge_chunk ? (g_edge_chunk << 10)
                                : std::min<uint64_t>(256 << 10,
                                                     std::max<uint64_t>(64 << 10, nbytes / 16));
  chunk = (chunk + 4095) & ~4095ull;
  if (chunk > nbytes) chunk = nbytes;
  e->a.chunk = chunk;
  e->a.nchunks = (uint32_t)((nbytes + chunk - 1) / chunk);
  e->a.sys = (g_force_sys || dst_space->imported || dst_space->device != src_space->device) ? 1 : 0;
  e->a.timeout_ns = g_put_timeout_ns;
  e->a.err = src_space->err;
  if (credit_addr != UINT64_MAX) {
    int rc = check_raw(src_space, credit_addr, 4ull * slots, "credit mirror");
    if (rc) {
      delete e;
      return rc;
    }
    if (credit_addr % 4) {
      delete e;
      return fail(SRF_E_INVALID_CONFIG, "credit mirror must be 4-B aligned");
    }
    e->a.credit_mirror = (const unsigned int *)(src_space->base + credit_addr);
  }
  e->next_round = 0;
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t words = 3 * (size_t)slots + 2;
  cudaError_t err = cudaMalloc(&e->state, words * sizeof(unsigned));
  if (err == cudaSuccess) err = cudaMemset(e->state, 0, words * sizeof(unsigned));
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    delete e;
    return fail(SRF_E_DEVICE, "edge state: %s", cudaGetErrorString(err));
  }
  e->a.released = e->state;
  e->a.arrival = e->state + slots;
  e->a.credit = e->state + 2 * slots;
  e->a.claim = e->state + 3 * slots;
  e->a.exit_count = e->state + 3 * slots + 1;
  *out = e;
  return SRF_OK;
}

// Pull edge: the receiver's GPU runs the edge (k_pull_stream).  src_space
// may be the receiver's mapping of the sender's pool (imported); dst_space is
// the receiver's own pool.  posted_addr: 8 B in dst_space (zeroed here) that
// the sender's srf_edge_post raises; pulled_addr (UINT64_MAX: none): 4*nsrc
// B of the sender's pool (through src_space) receiving each source's
// fully-pulled use count.
int srf_edge_create_pull(srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
                         uint64_t nbytes, uint32_t nsrc, uint64_t src_stride,
                         srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
                         uint32_t slots, uint64_t slot_stride, uint64_t posted_addr,
                         uint64_t pulled_addr, int tma, srf_edge_t *out) {
  DeviceGuard device_guard;
  if (nbytes < 1) return fail(SRF_E_INVALID_LENGTH, "zero-length edge");
  if (slots < 1 || nsrc < 1) return fail(SRF_E_INVALID_CONFIG, "slots and nsrc must be >= 1");
  if (slot_stride < nbytes + 1 || (nsrc > 1 && src_stride < nbytes))
    return fail(SRF_E_INVALID_CONFIG, "slot/source stride shorter than the payload");
  if (dst_space->imported) return fail(SRF_E_INVALID_CONFIG, "a pull edge's slots are local");
  const uint64_t src_span = (uint64_t)(nsrc - 1) * src_stride + nbytes;
  const uint64_t dst_span = (uint64_t)(slots - 1) * slot_stride + nbytes + 1;
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    int rc = check_remote_locked(src_space, src_addr, src_span, src_token);
    if (rc) return rc;
  }
  {
    std::lock_guard<std::mutex> g(dst_space->mu);
    int rc = check_registered_locked(dst_space, dst_addr, dst_span, dst_token);
    if (rc) return rc;
  }
  int rc = check_raw(dst_space, posted_addr, 8, "posted word");
  if (rc) return rc;
  if (posted_addr % 8) return fail(SRF_E_INVALID_CONFIG, "posted word must be 8-B aligned");
  if (pulled_addr != UINT64_MAX) {
    rc = check_raw(src_space, pulled_addr, 4ull * nsrc, "pulled counts");
    if (rc) return rc;
    if (pulled_addr % 4) return fail(SRF_E_INVALID_CONFIG, "pulled counts must be 4-B aligned");
  }
  if (!src_space->imported && src_space->device != dst_space->device) {
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, dst_space->device, src_space->device));
    if (!can) return fail(SRF_E_PEER_UNREACHABLE, "no peer path");
  }
  srf_edge *e = new srf_edge();
  e->device = dst_space->device;
  e->pull = 1;
  memset(&e->a, 0, sizeof e->a);
  e->a.src = src_space->base + src_addr;
  e->a.src_stride = src_stride;
  e->a.nsrc = nsrc;
  e->a.dst = dst_space->base + dst_addr;
  e->a.slot_stride = slot_stride;
  e->a.slots = slots;
  e->a.nbytes = nbytes;
  const bool aligned = ((uintptr_t)e->a.src % 16 == 0) && ((uintptr_t)e->a.dst % 16 == 0) &&
                       (nsrc == 1 || src_stride % 16 == 0) && slot_stride % 16 == 0;
  e->a.tma = (tma && aligned) ? 1 : 0;
  // one or two slots: stage the next round's chunks before the slot is free
  // (k_pull_stream_pre; chunks fit the 6 x 16 KiB stages)
  e->pre = (e->a.tma && slots <= 2 && !g_pull_no_prefetch) ? 1 : 0;
  const int sms = sm_count_of(e->device);
  // TMA: one CTA per SM keeps 6 x 16 KiB loads in flight from one issuing
  // thread; SM loads: the push edge's geometry
  e->ctas = g_edge_ctas ? g_edge_ctas
                        : std::max(1, e->a.tma ? sms - 1 : sms * g_edge_ctas_per_sm);
  uint64_t chunk = g_edge_chunk ? (g_edge_chunk << 10)
                  : e->pre ? std::min<uint64_t>(64 << 10, std::max<uint64_t>(16 << 10,
                                                                             nbytes / 128))
                           : std::min<uint64_t>(256 << 10,
                                                std::max<uint64_t>(64 << 10, nbytes / 16));
  chunk = (chunk + 4095) & ~4095ull;
  if (e->pre && chunk > (uint64_t)kBulkChunk * kBulkStages)
    chunk = (uint64_t)kBulkChunk * kBulkStages;
  if (chunk > nbytes) chunk = nbytes;
  e->a.chunk = chunk;
  e->a.nchunks = (uint32_t)((nbytes + chunk - 1) / chunk);
  e->a.sys = 0;
  e->a.timeout_ns = g_put_timeout_ns;
  e->a.err = dst_space->err;
  e->a.posted = (const unsigned long long *)(dst_space->base + posted_addr);
  e->a.pulled = pulled_addr == UINT64_MAX ? nullptr
                                          : (unsigned int *)(src_space->base + pulled_addr);
  e->next_round = 0;
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t words = 3 * (size_t)slots + 2;
  cudaError_t err = cudaMalloc(&e->state, words * sizeof(unsigned));
  if (err == cudaSuccess) err = cudaMemset(e->state, 0, words * sizeof(unsigned));
  if (err == cudaSuccess) err = cudaMemset((void *)e->a.posted, 0, 8);
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    delete e;
    return fail(SRF_E_DEVICE, "edge state: %s", cudaGetErrorString(err));
  }
  e->a.released = e->state;
  e->a.arrival = e->state + slots;
  e->a.credit = e->state + 2 * slots;
  e->a.claim = e->state + 3 * slots;
  e->a.exit_count = e->state + 3 * slots + 1;
  *out = e;
  return SRF_OK;
}

// the receiver pulls its next `rounds` rounds (one persistent launch)
int srf_edge_recv(srf_edge_t e, uint32_t rounds, srf_stream_t st, srf_space_t dst_space) {
  DeviceGuard device_guard;
  if (!e->pull) return fail(SRF_E_INVALID_CONFIG, "srf_edge_recv needs a pull edge");
  if (rounds == 0) return SRF_OK;
  if ((uint64_t)rounds * e->a.nchunks > 0xFFFFFFFFull)
    return fail(SRF_E_INVALID_CONFIG, "too many work items in one launch");
  srf_stream *s = stream_or_default(dst_space, st);
  if (s->device != e->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  StreamEdgeArgs a = e->a;
  a.first_round = e->next_round;
  a.rounds = rounds;
  const uint64_t items = (uint64_t)rounds * a.nchunks;
  const int grid = (int)std::min<uint64_t>((uint64_t)e->ctas, items);
  CUDA_TRY(cudaSetDevice(e->device));
  if (a.tma) {
    static bool attr_set[64] = {false};
    if (e->device >= 0 && e->device < 64 && !attr_set[e->device]) {
      CUDA_TRY(cudaFuncSetAttribute(k_pull_stream<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem));
      CUDA_TRY(cudaFuncSetAttribute(k_pull_stream_pre,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem));
      attr_set[e->device] = true;
    }
    if (e->pre)
      k_pull_stream_pre<<<grid, 256, kBulkSmem, s->s>>>(a);
    else
      k_pull_stream<true><<<grid, 256, kBulkSmem, s->s>>>(a);
  } else {
    k_pull_stream<false><<<grid, 512, 0, s->s>>>(a);
  }
  int rc = launch_check("k_pull_stream");
  if (rc) return rc;
  e->next_round += rounds;
  return SRF_OK;
}

// The sender's half of a pull edge: raise the receiver's posted-round word
// to `count` (rounds [0, count) are in their sources).  rcv_space: the
// sender's mapping of the receiver's pool.  wait_addr (UINT64_MAX: none) /
// need: first wait until the 4-B pulled count at wait_addr of the sender's
// own pool reaches need (the source about to be reused was fully pulled).
int srf_edge_post(srf_space_t snd_space, srf_space_t rcv_space, uint64_t posted_addr,
                  uint64_t count, uint64_t wait_addr, uint32_t need, srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(rcv_space, posted_addr, 8, "posted word");
  if (rc) return rc;
  if (posted_addr % 8) return fail(SRF_E_INVALID_CONFIG, "posted word must be 8-B aligned");
  const unsigned int *wp = nullptr;
  if (wait_addr != UINT64_MAX) {
    rc = check_raw(snd_space, wait_addr, 4, "pulled count");
    if (rc) return rc;
    wp = (const unsigned int *)(snd_space->base + wait_addr);
  }
  srf_stream *s = stream_or_default(snd_space, st);
  CUDA_TRY(cudaSetDevice(s->device));
  k_post_rounds<<<1, 1, 0, s->s>>>((unsigned long long *)(rcv_space->base + posted_addr), count,
                                   wp, need, g_put_timeout_ns, snd_space->err);
  return launch_check("k_post_rounds");
}

int srf_edge_info(srf_edge_t e, uint64_t *chunk, uint32_t *nchunks, int *ctas,
                  uint64_t *next_round) {
  if (chunk) *chunk = e->a.chunk;
  if (nchunks) *nchunks = e->a.nchunks;
  if (ctas) *ctas = e->ctas;
  if (next_round) *next_round = e->next_round;
  return SRF_OK;
}

// released[slots] | arrival[slots] | credit[slots] | claim | exit (diagnostics)
int srf_edge_state(srf_edge_t e, uint32_t *host_out, uint32_t nwords) {
  DeviceGuard device_guard;
  const uint32_t words = 3 * e->a.slots + 2;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaMemcpy(host_out, e->state, sizeof(uint32_t) * std::min(words, nwords),
                      cudaMemcpyDeviceToHost));
  return SRF_OK;
}

int srf_edge_send(srf_edge_t e, uint32_t rounds, srf_stream_t st, srf_space_t src_space) {
  DeviceGuard device_guard;
  if (e->pull) return fail(SRF_E_INVALID_CONFIG, "a pull edge runs on the receiver: srf_edge_recv");
  if (rounds == 0) return SRF_OK;
  if ((uint64_t)rounds * e->a.nchunks > 0xFFFFFFFFull)
    return fail(SRF_E_INVALID_CONFIG, "too many work items in one launch");
  srf_stream *s = stream_or_default(src_space, st);
  if (s->device != e->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  StreamEdgeArgs a = e->a;
  a.first_round = e->next_round;
  a.rounds = rounds;
  const uint64_t items = (uint64_t)rounds * a.nchunks;
  const int grid = (int)std::min<uint64_t>((uint64_t)e->ctas, items);
  CUDA_TRY(cudaSetDevice(e->device));
  k_put_stream<<<grid, 512, 0, s->s>>>(a);
  int rc = launch_check("k_put_stream");
  if (rc) return rc;
  e->next_round += rounds;
  return SRF_OK;
}

int srf_edge_consume(srf_space_t rcv, uint64_t slots_addr, uint32_t slots, uint64_t slot_stride,
                     uint64_t nbytes, uint64_t first_round, uint32_t rounds, int mode,
                     uint64_t sums_addr, srf_space_t credit_space, uint64_t credit_addr,
                     srf_stream_t st) {
  DeviceGuard device_guard;
  if (rcv->imported) return fail(SRF_E_INVALID_CONFIG, "the receiver consumes its own slots");
  if (slots < 1 || slot_stride < nbytes + 1)
    return fail(SRF_E_INVALID_CONFIG, "bad slot geometry");
  int rc = check_raw(rcv, slots_addr, (uint64_t)(slots - 1) * slot_stride + nbytes + 1, "slots");
  if (rc) return rc;
  if (mode == 1) {
    rc = check_raw(rcv, sums_addr, 8ull * rounds, "checksums");
    if (rc) return rc;
    if (sums_addr % 8) return fail(SRF_E_INVALID_CONFIG, "checksums must be 8-B aligned");
  }
  unsigned int *mirror = nullptr;
  if (credit_space) {
    rc = check_raw(credit_space, credit_addr, 4ull * slots, "credit mirror");
    if (rc) return rc;
    if (credit_addr % 4) return fail(SRF_E_INVALID_CONFIG, "credit mirror must be 4-B aligned");
    mirror = (unsigned int *)(credit_space->base + credit_addr);
  }
  if (rounds == 0) return SRF_OK;
  srf_stream *s = stream_or_default(rcv, st);
  CUDA_TRY(cudaSetDevice(s->device));
  // a pinned, mapped word per device: the consumer stamps it when it runs
  static std::mutex mu;
  static uint32_t *started_host[64] = {nullptr}, *started_dev[64] = {nullptr};
  static uint32_t tickets[64] = {0};
  uint32_t *sh = nullptr, *sd = nullptr, ticket = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    const int dev = s->device;
    if (dev >= 0 && dev < 64) {
      if (!started_host[dev]) {
        CUDA_TRY(cudaHostAlloc((void **)&started_host[dev], 64,
                               cudaHostAllocMapped | cudaHostAllocPortable));
        CUDA_TRY(cudaHostGetDevicePointer((void **)&started_dev[dev], started_host[dev], 0));
        *(volatile uint32_t *)started_host[dev] = 0;
      }
      sh = started_host[dev];
      sd = started_dev[dev];
      ticket = ++tickets[dev];
      if (ticket == 0) ticket = ++tickets[dev];
    }
  }
  k_consume_stream<<<1, mode == 1 ? 1024 : g_consume_threads, 0, s->s>>>(
      rcv->base + slots_addr, slot_stride, slots, nbytes, first_round, rounds,
      mode == 1 ? 1 : (g_consume_release ? 2 : 0),
      (unsigned long long *)(rcv->base + sums_addr), mirror, sd, ticket, g_put_timeout_ns,
      rcv->err);
  rc = launch_check("k_consume_stream");
  if (rc || !sh) return rc;
  // wait until the consumer CTA is resident (work queued before it on the
  // stream delays it; the wait is bounded by the put timeout)
  const auto t0 = std::chrono::steady_clock::now();
  while (*(volatile uint32_t *)sh != ticket) {
    if (cudaStreamQuery(s->s) == cudaSuccess) break;  // already finished
    if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(g_put_timeout_ns))
      return fail(SRF_E_TIMEOUT, "edge consumer did not start");
  }
  return SRF_OK;
}

// ---- pipelined dynamic edge (device_stream.cuh, k_dyn_*) -------------------
struct srf_dyn_edge {
  int device;
  DynEdgeArgs a;
  void *state = nullptr;
  uint64_t next_round = 0;
  int ctas = 0;
};

// Receiver side: metadata slots (slots x meta_stride bytes at meta_addr of
// dst_space, flag bytes zeroed here), a ring arena of ring_cap bytes at
// ring_addr (256-B aligned), and the sender's payload region [lo, hi) with its
// token as seen through src_space (the receiver's mapping of the sender).
int srf_dyn_edge_create(srf_space_t src_space, uint64_t lo, uint64_t hi, uint64_t token,
                        uint64_t max_bytes, uint32_t rank, srf_space_t dst_space,
                        uint64_t meta_addr, uint64_t meta_stride, uint32_t slots,
                        uint64_t ring_addr, uint64_t ring_cap, srf_dyn_edge_t *out) {
  DeviceGuard device_guard;
  if (rank < 1 || rank > (uint32_t)kDynMaxRank)
    return fail(SRF_E_INVALID_CONFIG, "rank 1..%d", kDynMaxRank);
  if (slots < 1) return fail(SRF_E_INVALID_CONFIG, "slots >= 1");
  if (dst_space->imported) return fail(SRF_E_INVALID_CONFIG, "the receiver's slots are local");
  if (meta_stride < 8ull * rank + 33 || meta_stride % 8 || meta_addr % 8)
    return fail(SRF_E_INVALID_CONFIG, "metadata slots: 8-B aligned, >= 8D+33 B apart");
  if (ring_addr % 256 || ring_cap < ((max_bytes + 255) & ~255ull) || ring_cap == 0)
    return fail(SRF_E_INVALID_CONFIG, "ring arena: 256-B aligned, >= one round");
  int rc = check_raw(dst_space, meta_addr, (uint64_t)slots * meta_stride, "metadata slots");
  if (!rc) rc = check_raw(dst_space, ring_addr, ring_cap, "ring arena");
  if (rc) return rc;
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    rc = check_remote_locked(src_space, lo, hi - lo, token);
    if (rc) return rc;
  }
  srf_dyn_edge *e = new srf_dyn_edge();
  e->device = dst_space->device;
  DynEdgeArgs &a = e->a;
  memset(&a, 0, sizeof a);
  a.meta = dst_space->base + meta_addr;
  a.meta_stride = meta_stride;
  a.slots = slots;
  a.rank = rank;
  a.peer_base = src_space->base;
  a.lo = lo;
  a.hi = hi;
  a.token = token;
  a.max_bytes = max_bytes;
  uint64_t chunk = g_edge_chunk ? (g_edge_chunk << 10)
                                : std::min<uint64_t>(256 << 10,
                                                     std::max<uint64_t>(32 << 10, max_bytes / 16));
  chunk = (chunk + 4095) & ~4095ull;
  if (chunk > max_bytes && max_bytes) chunk = (max_bytes + 15) & ~15ull;
  if (chunk == 0) chunk = 16;
  a.chunk = chunk;
  a.nchunks = (uint32_t)std::max<uint64_t>(1, (max_bytes + chunk - 1) / chunk);
  a.ring = dst_space->base + ring_addr;
  a.ring_cap = ring_cap;
  a.timeout_ns = g_put_timeout_ns;
  a.err = dst_space->err;
  e->ctas = g_edge_ctas ? g_edge_ctas : std::max(1, sm_count_of(e->device) - 2);
  CUDA_TRY(cudaSetDevice(e->device));
  // arrival[slots] claim exit alloc_seq consumed | alloc_head freed out[3 slots] | ready[slots]
  const size_t words32 = (size_t)slots + 5, words64 = 2 + 3 * (size_t)slots;
  const size_t bytes = 8 * ((words32 * 4 + 7) / 8) + 8 * words64 + slots;
  cudaError_t err = cudaMalloc(&e->state, bytes);
  if (err == cudaSuccess) err = cudaMemset(e->state, 0, bytes);
  for (uint32_t i = 0; err == cudaSuccess && i < slots; ++i)
    err = cudaMemset(a.meta + (uint64_t)i * meta_stride + 8ull * rank + 32, 0, 1);
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    if (e->state) cudaFree(e->state);
    delete e;
    return fail(SRF_E_DEVICE, "dynamic edge state: %s", cudaGetErrorString(err));
  }
  unsigned int *w32 = (unsigned int *)e->state;
  a.arrival = w32;
  a.claim = w32 + slots;
  a.exit_count = w32 + slots + 1;
  a.alloc_seq = w32 + slots + 2;
  a.consumed = w32 + slots + 3;
  unsigned long long *w64 = (unsigned long long *)((uint8_t *)e->state + 8 * ((words32 * 4 + 7) / 8));
  a.alloc_head = w64;
  a.freed = w64 + 1;
  a.out = w64 + 2;
  a.ready = (uint8_t *)(w64 + words64);
  *out = e;
  return SRF_OK;
}

// the receiver pulls its next `rounds` rounds (one persistent TMA launch)
int srf_dyn_edge_recv(srf_dyn_edge_t e, uint32_t rounds, srf_stream_t st, srf_space_t dst_space) {
  DeviceGuard device_guard;
  if (rounds == 0) return SRF_OK;
  if ((uint64_t)rounds * e->a.nchunks > 0xFFFFFFFFull)
    return fail(SRF_E_INVALID_CONFIG, "too many work items in one launch");
  srf_stream *s = stream_or_default(dst_space, st);
  if (s->device != e->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  DynEdgeArgs a = e->a;
  a.first_round = e->next_round;
  a.rounds = rounds;
  const int grid = (int)std::min<uint64_t>((uint64_t)e->ctas, (uint64_t)rounds * a.nchunks);
  CUDA_TRY(cudaSetDevice(e->device));
  static bool attr_set[64] = {false};
  if (e->device >= 0 && e->device < 64 && !attr_set[e->device]) {
    CUDA_TRY(cudaFuncSetAttribute(k_dyn_pull_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kBulkSmem));
    attr_set[e->device] = true;
  }
  k_dyn_pull_stream<<<grid, 256, kBulkSmem, s->s>>>(a);
  int rc = launch_check("k_dyn_pull_stream");
  if (rc) return rc;
  e->next_round += rounds;
  return SRF_OK;
}

// the receiver's consumer for rounds [first_round, +rounds) (mode 1: 8-B
// checksum per round at sums_addr of dst_space); returns once it is resident
int srf_dyn_edge_consume(srf_dyn_edge_t e, srf_space_t dst_space, uint64_t first_round,
                         uint32_t rounds, int mode, uint64_t sums_addr, srf_stream_t st) {
  DeviceGuard device_guard;
  if (mode == 1) {
    int rc = check_raw(dst_space, sums_addr, 8ull * rounds, "checksums");
    if (rc) return rc;
    if (sums_addr % 8) return fail(SRF_E_INVALID_CONFIG, "checksums must be 8-B aligned");
  }
  if (rounds == 0) return SRF_OK;
  srf_stream *s = stream_or_default(dst_space, st);
  if (s->device != e->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  CUDA_TRY(cudaSetDevice(s->device));
  // a pinned, mapped word per device the consumer stamps when it runs
  static std::mutex mu;
  static uint32_t *hs[64] = {nullptr}, *ds[64] = {nullptr}, tickets[64] = {0};
  const int dev = s->device;
  if (dev < 0 || dev >= 64) return fail(SRF_E_INVALID_CONFIG, "device index %d", dev);
  uint32_t ticket, *sh, *sd;
  {
    std::lock_guard<std::mutex> g(mu);
    if (!hs[dev]) {
      CUDA_TRY(cudaHostAlloc((void **)&hs[dev], 64, cudaHostAllocMapped | cudaHostAllocPortable));
      CUDA_TRY(cudaHostGetDevicePointer((void **)&ds[dev], hs[dev], 0));
      *(volatile uint32_t *)hs[dev] = 0;
    }
    sh = hs[dev];
    sd = ds[dev];
    ticket = ++tickets[dev];
    if (ticket == 0) ticket = ++tickets[dev];
  }
  k_dyn_consume_stream<<<1, mode == 1 ? 1024 : 32, 0, s->s>>>(
      e->a, first_round, rounds, mode, (unsigned long long *)(dst_space->base + sums_addr), sd,
      ticket);
  int rc = launch_check("k_dyn_consume_stream");
  if (rc) return rc;
  const auto t0 = std::chrono::steady_clock::now();
  while (*(volatile uint32_t *)sh != ticket) {
    if (cudaStreamQuery(s->s) == cudaSuccess) break;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(g_put_timeout_ns))
      return fail(SRF_E_TIMEOUT, "dynamic edge consumer did not start");
  }
  return SRF_OK;
}

// Sender side: rounds [first_round, +rounds), round j announcing payload
// src_addr + (j % nsrc) * src_stride (registered, token) of nbytes with the
// given dims / element code.  rcv_space: the sender's mapping of the receiver.
int srf_dyn_edge_send(srf_space_t snd_space, srf_space_t rcv_space, uint64_t meta_addr,
                      uint64_t meta_stride, uint32_t slots, uint32_t rank, int elem,
                      const uint64_t *dims, uint64_t src_addr, uint64_t src_stride,
                      uint32_t nsrc, uint64_t src_token, uint64_t first_round, uint32_t rounds,
                      srf_stream_t st) {
  DeviceGuard device_guard;
  if (rank < 1 || rank > (uint32_t)kDynMaxRank || slots < 1 || nsrc < 1)
    return fail(SRF_E_INVALID_CONFIG, "rank / slots / nsrc");
  if (elem < 0 || elem > 4) return fail(SRF_E_INVALID_CONFIG, "element code %d", elem);
  const uint64_t esz = elem == 0 || elem == 2 ? 4 : elem == 4 ? 1 : 8;
  uint64_t nbytes = esz;
  for (uint32_t k = 0; k < rank; ++k) nbytes *= dims[k];
  int rc = check_raw(rcv_space, meta_addr, (uint64_t)slots * meta_stride, "metadata slots");
  if (rc) return rc;
  if (meta_stride % 8 || meta_addr % 8 || meta_stride < 8ull * rank + 33)
    return fail(SRF_E_INVALID_CONFIG, "metadata slot geometry");
  {
    std::lock_guard<std::mutex> g(snd_space->mu);
    rc = check_registered_locked(snd_space, src_addr, (uint64_t)(nsrc - 1) * src_stride + nbytes,
                                 src_token);
    if (rc) return rc;
  }
  if (rounds == 0) return SRF_OK;
  DynSendArgs a;
  memset(&a, 0, sizeof a);
  a.meta = rcv_space->base + meta_addr;
  a.meta_stride = meta_stride;
  a.slots = slots;
  a.rank = rank;
  a.code = (uint32_t)elem;
  a.nsrc = nsrc;
  for (uint32_t k = 0; k < rank; ++k) a.dims[k] = dims[k];
  a.src_addr = src_addr;
  a.src_stride = src_stride;
  a.token = src_token;
  a.nbytes = nbytes;
  a.first_round = first_round;
  a.rounds = rounds;
  a.timeout_ns = g_put_timeout_ns;
  a.err = snd_space->err;
  srf_stream *s = stream_or_default(snd_space, st);
  CUDA_TRY(cudaSetDevice(s->device));
  k_dyn_send_stream<<<1, 1024, 0, s->s>>>(a);
  return launch_check("k_dyn_send_stream");
}

int srf_dyn_edge_destroy(srf_dyn_edge_t e) {
  DeviceGuard device_guard;
  if (!e) return SRF_OK;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  cudaFree(e->state);
  delete e;
  return SRF_OK;
}

int srf_edge_destroy(srf_edge_t e) {
  DeviceGuard device_guard;
  if (!e) return SRF_OK;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  cudaFree(e->state);
  delete e;
  return SRF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Session iteration recording and replay (host_record.cuh)
// ---------------------------------------------------------------------------
extern "C" {

int srf_record_begin(void) {
  std::lock_guard<std::mutex> g(g_rec_mu);
  if (g_rec) return fail(SRF_E_INVALID_CONFIG, "a recording is already active");
  g_rec = new srf_oplist();
  g_rec_expected = false;
  return SRF_OK;
}

int srf_record_end(srf_oplist_t *out, int *replayable) {
  std::lock_guard<std::mutex> g(g_rec_mu);
  if (!g_rec) return fail(SRF_E_INVALID_CONFIG, "no active recording");
  srf_oplist *l = g_rec;
  g_rec = nullptr;
  g_rec_expected = false;
  if (replayable) *replayable = (!l->dirty && !l->ops.empty() && l->device >= 0) ? 1 : 0;
  *out = l;
  return SRF_OK;
}

int srf_record_taint(const char *why) {
  rec_dirty(why ? why : "device work outside the library");
  return SRF_OK;
}

int srf_oplist_info(srf_oplist_t l, uint32_t *nops, int *device, char *why, uint32_t why_len) {
  if (nops) *nops = (uint32_t)l->ops.size();
  if (why && why_len && l->exec) {
    snprintf(why, why_len, "graph: %u nodes, %u dependency edges", l->nodes, l->edges);
    if (device) *device = l->device;
    return SRF_OK;
  }
  if (device) *device = l->device;
  if (why && why_len) {
    snprintf(why, why_len, "%s", l->dirty ? l->why.c_str() : "");
  }
  return SRF_OK;
}

int srf_oplist_same(srf_oplist_t a, srf_oplist_t b, int64_t gen_delta) {
  if (a->dirty || b->dirty || a->ops.size() != b->ops.size() || a->device != b->device) return 0;
  for (size_t i = 0; i < a->ops.size(); ++i)
    if (!rec_same(a->ops[i], b->ops[i], gen_delta)) return 0;
  return 1;
}

// diagnostics: where b stops repeating a (first differing op, kinds, counts)
int srf_oplist_diff(srf_oplist_t a, srf_oplist_t b, int64_t gen_delta, char *out, uint32_t len) {
  if (a->ops.size() != b->ops.size()) {
    snprintf(out, len, "op count %zu vs %zu", a->ops.size(), b->ops.size());
    return SRF_OK;
  }
  for (size_t i = 0; i < a->ops.size(); ++i) {
    if (!rec_same(a->ops[i], b->ops[i], gen_delta)) {
      const RecOp &x = a->ops[i], &y = b->ops[i];
      char extra[256] = "";
      if (x.kind == REC_PUT && y.kind == REC_PUT)
        snprintf(extra, sizeof extra, " put dst %p/%p seg0 %p/%p len %llu/%llu",
                 (void *)x.put.dst, (void *)y.put.dst, (const void *)x.put.seg[0].src,
                 (const void *)y.put.seg[0].src, (unsigned long long)x.put.total,
                 (unsigned long long)y.put.total);
      else if (x.kind == REC_APPLY && y.kind == REC_APPLY)
        snprintf(extra, sizeof extra, " apply var %p/%p g0 %p/%p", (void *)x.apply.var,
                 (void *)y.apply.var, (const void *)x.apply.g[0], (const void *)y.apply.g[0]);
      else if (x.kind == REC_GEN && y.kind == REC_GEN)
        snprintf(extra, sizeof extra, " gen dst %p/%p it %llu/%llu", (void *)x.gen.dst,
                 (void *)y.gen.dst, (unsigned long long)x.gen.iteration,
                 (unsigned long long)y.gen.iteration);
      snprintf(out, len, "op %zu kind %d/%d%s", i, x.kind, y.kind, extra);
      return SRF_OK;
    }
  }
  snprintf(out, len, "same");
  return SRF_OK;
}

int srf_oplist_replay(srf_oplist_t l, uint64_t first_offset, uint32_t count, srf_stream_t st) {
  DeviceGuard device_guard;
  if (l->dirty || l->ops.empty()) return fail(SRF_E_INVALID_CONFIG, "recording not replayable");
  if (st->device != l->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  if (count == 0) return SRF_OK;
  CUDA_TRY(cudaSetDevice(l->device));
  if (!l->exec) {
    // one CUDA graph of the recorded iteration with data dependencies
    // (host_record.cuh); GenGrad reads its iteration offset from a device
    // word set before each launch
    int rc = rec_build_graph(l);
    if (rc) return rc;
  }
  if (!l->done) CUDA_TRY(cudaEventCreateWithFlags(&l->done, cudaEventDisableTiming));
  for (uint32_t i = 0; i < count; ++i) {
    // relaunch an exec only after its previous launch finished: relaunching
    // one still in flight stalled the host ~3.5 ms per launch (host_record.cuh,
    // replay set); with a period of p phases the host stays p launches ahead
    CUDA_TRY(cudaEventSynchronize(l->done));
    k_set_u64<<<1, 1, 0, st->s>>>(l->iter_add, first_offset + i);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaGraphLaunch(l->exec, st->s));
    CUDA_TRY(cudaEventRecord(l->done, st->s));
  }
  g_launches.fetch_add((uint64_t)count * (l->ops.size() + 1), std::memory_order_relaxed);
  return SRF_OK;
}

// One graph for all phases of a period (host_record.cuh, "Replay set").
// lists[p] is the recording of phase p, made at iteration iters[p]; fails
// with SRF_E_INVALID_CONFIG when the phases do not share one op sequence.
int srf_replay_set_create(srf_oplist_t *lists, const int64_t *iters, uint32_t nphase,
                          srf_replay_set_t *out) {
  DeviceGuard device_guard;
  if (nphase == 0) return fail(SRF_E_INVALID_CONFIG, "no phases");
  const srf_oplist *l0 = lists[0];
  for (uint32_t p = 0; p < nphase; ++p) {
    const srf_oplist *l = lists[p];
    if (l->dirty || l->ops.empty() || l->device != l0->device || l->ops.size() != l0->ops.size())
      return fail(SRF_E_INVALID_CONFIG, "phases differ in device or op count");
    for (size_t i = 0; i < l->ops.size(); ++i)
      if (!rec_same_function(l0->ops[i], l->ops[i]))
        return fail(SRF_E_INVALID_CONFIG, "phase %u op %zu launches another kernel", p, i);
  }
  CUDA_TRY(cudaSetDevice(l0->device));
  srf_replay_set *rs = new srf_replay_set();
  rs->device = l0->device;
  rs->nphase = nphase;
  rs->n = (uint32_t)l0->ops.size();
  int rc = rec_set_build(rs, lists, iters);
  if (rc) {
    for (auto &v : rs->ops)
      for (RecOp &op : v) delete op.inl;
    delete rs;
    return rc;
  }
  *out = rs;
  return SRF_OK;
}

// replay iteration `iteration` with phase `phase`'s recording (stream order)
int srf_replay_set_launch(srf_replay_set_t rs, uint32_t phase, uint64_t iteration,
                          srf_stream_t st) {
  DeviceGuard device_guard;
  if (phase >= rs->nphase) return fail(SRF_E_INVALID_CONFIG, "phase out of range");
  if (st->device != rs->device) return fail(SRF_E_INVALID_CONFIG, "stream on another GPU");
  CUDA_TRY(cudaSetDevice(rs->device));
  int rc = rec_set_launch(rs, phase, iteration, st->s);
  if (rc) return rc;
  g_launches.fetch_add((uint64_t)rs->n + 1, std::memory_order_relaxed);
  return SRF_OK;
}

int srf_replay_set_info(srf_replay_set_t rs, uint32_t *nodes, uint32_t *edges,
                        uint32_t *classes, uint64_t *updates) {
  if (nodes) *nodes = rs->n;
  if (edges) *edges = rs->edges;
  if (classes) {
    uint32_t c = 0;
    for (size_t k = 0; k < rs->cls.size(); ++k) c += rs->cls[k] == k / rs->n ? 1 : 0;
    *classes = c;
  }
  if (updates) *updates = rs->updates;
  return SRF_OK;
}

int srf_replay_set_destroy(srf_replay_set_t rs) {
  DeviceGuard device_guard;
  if (!rs) return SRF_OK;
  cudaSetDevice(rs->device);
  cudaDeviceSynchronize();
  for (auto &v : rs->ops)
    for (RecOp &op : v) delete op.inl;
  delete rs;
  return SRF_OK;
}

int srf_oplist_destroy(srf_oplist_t l) {
  DeviceGuard device_guard;
  if (!l) return SRF_OK;
  if (l->device >= 0) cudaSetDevice(l->device);
  delete l;
  return SRF_OK;
}

}  // extern "C"
