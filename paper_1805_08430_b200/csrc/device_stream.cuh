// device_stream.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Pipelined static edge: many static-placement transfers of one edge in ONE
// persistent launch (EXTENSION of the reference's static placement).
//
// The reference's static edge has one pre-placed receive region per edge and
// a flag credit (runtime/protocol.py:49-138, analyzer.py:149-220), so round
// k+1 cannot start before round k was consumed, and on the GPU every round
// pays a kernel launch, a grid-wide arrival, a system-scope release and the
// consumer's poll (~9 us over NVLink) - 4 MiB rounds reached only
// 0.32 of the link.  Here the receiver pre-places `slots` regions for the
// edge (slot i = payload || flag at dst + i * slot_stride); round j writes
// slot j % slots; each slot keeps the reference protocol exactly (flag byte
// released last, consumer clears it = the credit).  The sender kernel is a
// persistent work queue of (round, chunk) items claimed in order: a CTA copies
// one chunk and arrives on the slot's counter; the last arriver releases the
// slot's flag (st.release.sys) - no grid barrier, no kernel boundary between
// rounds, so chunks of round j+1 stream while round j's tail is published and
// consumed.  Item (j, c) waits only on (a) the previous use of its slot being
// fully released (sender-local counter) and (b) the consumer's credit for that
// previous use (the remote flag read 0; the first CTA that sees it caches it
// locally so the other chunks skip the NVLink round trip).  The earliest
// unfinished item never waits on a later one: no deadlock for any grid.

struct StreamEdgeArgs {
  const uint8_t *src;      // nsrc payloads, src_stride apart (round j sends j % nsrc)
  uint64_t src_stride;
  uint32_t nsrc;
  uint8_t *dst;            // slot 0 (a peer's pool or this GPU's)
  uint64_t slot_stride;
  uint32_t slots;
  uint64_t nbytes;         // payload bytes S; the flag is at slot + S
  uint64_t chunk;          // bytes per work item
  uint32_t nchunks;
  uint64_t first_round;    // rounds continue across launches
  uint32_t rounds;
  unsigned int *released;  // [slots] uses of the slot released (sender-local)
  unsigned int *arrival;   // [slots] chunk arrivals of the slot's current use
  unsigned int *credit;    // [slots] uses whose predecessor was consumed (cached credit)
  unsigned int *claim;     // work queue head
  unsigned int *exit_count;
  // credit mirror (nullptr: none): [slots] words in the SENDER's memory that
  // the consumer stores the slot's consumed-use count into (a posted write
  // over NVLink) right after clearing the flag - the same credit as the
  // cleared flag, read locally instead of by a remote load per round, which
  // queues behind payload traffic when both link directions are busy
  const unsigned int *credit_mirror;
  int sys;                 // destination is a peer's memory
  uint64_t timeout_ns;
  int *err;
  // pull edges (k_pull_stream, launched on the RECEIVER's GPU): src is the
  // sender's memory, dst the receiver's own slots
  const unsigned long long *posted;  // receiver-local: rounds the sender posted
  unsigned int *pulled;    // [nsrc] in the SENDER's memory: uses of each source
                           // fully pulled (nullptr: none)
  int tma;                 // 1: chunks move through TMA bulk copies
};

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const unsigned int *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u32(unsigned int *p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys_u32(unsigned int *p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_release_gpu_max(unsigned int *p, unsigned v) {
  asm volatile("red.release.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(512) k_put_stream(const __grid_constant__ StreamEdgeArgs a) {
  __shared__ uint32_t s_i;
  __shared__ int s_last;
  const uint32_t total = a.rounds * a.nchunks;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(a.claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= total) break;
    const uint32_t jr = i / a.nchunks;
    const uint32_t c = i - jr * a.nchunks;
    const uint64_t j = a.first_round + jr;
    const uint32_t slot = (uint32_t)(j % a.slots);
    const uint32_t m = (uint32_t)(j / a.slots);  // use index of the slot
    uint8_t *d = a.dst + (uint64_t)slot * a.slot_stride;
    if (threadIdx.x == 0 && *(volatile int *)a.err == 0) {
      // (a) the slot's previous use is fully released (its tail published)
      // (after any timeout the remaining items skip their waits: the launch
      // drains in microseconds and the host raises the error)
      wait_count(a.released + slot, m, a.timeout_ns, a.err);
      // (b) ... and consumed: the receiver cleared its flag (the reference's
      // credit, protocol.py:102-111); cached once seen
      if (m > 0 && a.credit_mirror) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_sys_u32(a.credit_mirror + slot) < m) {
          if (globaltimer_ns() - t0 > a.timeout_ns) {
            atomicExch(a.err, 2);
            break;
          }
          __nanosleep(20);
        }
      } else if (m > 0 && ld_acquire_gpu_u32(a.credit + slot) < m) {
        if (c == 0) {
          // the round's first chunk polls the receiver's flag; the others
          // wait on the cached credit (one remote poll per round, not one
          // per chunk: under two-way load every remote read queues behind
          // the payload in both link directions)
          if (!spin_until(d + a.nbytes, 0, a.timeout_ns, a.sys)) atomicExch(a.err, 2);
          red_release_gpu_max(a.credit + slot, m);
        } else {
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_gpu_u32(a.credit + slot) < m && *(volatile int *)a.err == 0) {
            if (globaltimer_ns() - t0 > a.timeout_ns) {
              atomicExch(a.err, 2);
              break;
            }
            __nanosleep(20);
          }
        }
      }
    }
    __syncthreads();
    if (c == 0 && !a.credit_mirror && a.slots > 1 && threadIdx.x == 32 &&
        *(volatile int *)a.err == 0) {
      // credit look-ahead: one non-blocking poll for the use half the ring
      // ahead, so by the time its chunks are claimed the credit is cached
      // (a flag read 0 after that slot's previous use was released means
      // the consumer cleared it - the same test as the demand path)
      const uint64_t jn = j + a.slots / 2;
      const uint32_t sn = (uint32_t)(jn % a.slots), mn = (uint32_t)(jn / a.slots);
      if (mn > 0 && ld_acquire_gpu_u32(a.credit + sn) < mn &&
          ld_acquire_gpu_u32(a.released + sn) >= mn) {
        const uint8_t *fn = a.dst + (uint64_t)sn * a.slot_stride + a.nbytes;
        if ((a.sys ? ld_acquire_sys_u8(fn) : ld_acquire_gpu_u8(fn)) == 0)
          red_release_gpu_max(a.credit + sn, mn);
      }
    }
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t n = a.nbytes - off < a.chunk ? a.nbytes - off : a.chunk;
    const uint8_t *s = a.src + (j % a.nsrc) * a.src_stride;
    copy_bytes_grid<8>(d + off, s + off, n, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(a.arrival + slot, a.nchunks - 1, a.sys);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      atomicExch(a.arrival + slot, 0u);    // re-armed before anything is published
      release_tail(d + a.nbytes, 1, a.sys);  // flag last: the round is delivered
      count_done(a.released + slot);
    }
  }
  // the last CTA out re-arms the queue for the next launch
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    *a.exit_count = 0;
  }
}

// Receiver side of the pipelined edge (StaticReceiver.poll per round, on the
// device): one CTA walks rounds in order, acquire-spins on the slot's flag,
// optionally checksums the payload the flag guards, then clears the flag
// (release: the sender may overwrite the slot only after these reads).
// mode 0: consume the flag only; 1: also store a weighted byte checksum of
// the round's payload into sums[r] (tests); 2: flag only, cleared with a
// system-scope release anyway (knob consume_release, for comparison).
__global__ void __launch_bounds__(1024) k_consume_stream(uint8_t *slots_base, uint64_t slot_stride,
                                                          uint32_t slots, uint64_t nbytes,
                                                          uint64_t first_round, uint32_t rounds,
                                                          int mode, unsigned long long *sums,
                                                          unsigned int *credit_mirror,
                                                          uint32_t *started, uint32_t ticket,
                                                          uint64_t timeout_ns, int *err) {
  __shared__ unsigned long long acc;
  __shared__ int ok;
  // residency handshake: the host launches the sender only after this CTA is
  // running, so a full-GPU sender grid can never keep it from being scheduled
  if (threadIdx.x == 0 && started) {
    *(volatile uint32_t *)started = ticket;
    __threadfence_system();
  }
  if (!(mode & 1)) {
    // flag-only: lane 0 of warp w consumes the slots s with s % W == w, each
    // slot's rounds in order - W slots' polls and clears proceed at once (one
    // thread walking every round capped small rounds at ~0.5 us each); a
    // slot stays on one warp, so a flag read 1 is always that round's
    const uint32_t W = blockDim.x / 32, w = threadIdx.x / 32;
    if (threadIdx.x % 32 != 0) return;
    for (uint32_t r = 0; r < rounds; ++r) {
      const uint64_t j = first_round + r;
      const uint32_t slot = (uint32_t)(j % slots);
      if (slot % W != w) continue;
      uint8_t *d = slots_base + (uint64_t)slot * slot_stride;
      if (!spin_until(d + nbytes, 1, timeout_ns, 1)) {
        atomicExch(err, 1);
        return;
      }
      if (mode == 2) release_tail(d + nbytes, 0, 1);
      else st_relaxed_sys_u8(d + nbytes, 0);
      if (credit_mirror) {
        if (mode == 2) st_release_sys_u32(credit_mirror + slot, (unsigned)(j / slots) + 1);
        else st_relaxed_sys_u32(credit_mirror + slot, (unsigned)(j / slots) + 1);
      }
    }
    return;
  }
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint64_t j = first_round + r;
    uint8_t *d = slots_base + (j % slots) * slot_stride;
    if (threadIdx.x == 0) {
      acc = 0;
      ok = spin_until(d + nbytes, 1, timeout_ns, 1) ? 1 : 0;
      if (!ok) atomicExch(err, 1);
    }
    __syncthreads();
    if (!ok) return;
    if (mode & 1) {
      unsigned long long sum = 0;
      for (uint64_t i = threadIdx.x; i < nbytes; i += blockDim.x)
        sum += (unsigned long long)__ldcg(d + i) * (i % 251 + 1);  // L2: the slot is rewritten
      atomicAdd(&acc, sum);
      __syncthreads();
      if (threadIdx.x == 0) sums[r] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // StaticReceiver.poll's clear = the credit.  With a checksum the clear
      // must be a system-scope release (the sender may overwrite the slot
      // only after these reads); flag-only consumption read nothing to order,
      // and a release.sys costs a MEMBAR.SYS that, on a GPU also sending over
      // NVLink, waits behind its own outbound stores (~4-8 us per round)
      if (mode) release_tail(d + nbytes, 0, 1);
      else st_relaxed_sys_u8(d + nbytes, 0);
      if (credit_mirror) {             // ... mirrored to the sender (posted write)
        if (mode) st_release_sys_u32(credit_mirror + j % slots, (unsigned)(j / slots) + 1);
        else st_relaxed_sys_u32(credit_mirror + j % slots, (unsigned)(j / slots) + 1);
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Pull edge (k_pull_stream): the same pipelined static edge, driven by the
// RECEIVER.  The sender posts "round j's payload is in source j % nsrc" by
// storing the posted-round count into a word of the receiver's pool
// (k_post_rounds, one posted store over NVLink per batch of rounds); the
// receiver's SMs pull each (round, chunk) item from the sender's memory
// straight into the pre-placed slot (peer loads, or TMA bulk copies peer
// global -> shared -> local global) and the last arriver of a round releases
// the slot's flag exactly as the push edge does (flag last, the consumer
// clears it = the credit).  Why: one GPU's NVLink read responses carry user
// data at 751-765 GB/s one way against 700-719 for its SM stores
// (profiles/r2_pull_ring.jsonl: the write packets' header overhead); the
// credit checks become local loads.  When the sender may rewrite a source,
// the last arriver also publishes the source's pulled-use count into the
// sender's memory (red.max.release.sys), the sender's licence to reuse it.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const unsigned long long *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 only: [src, src + n) -> [dst, ...) through shared memory with
// kBulkStages 16-KiB stages (n a multiple of 16, both 16-B aligned); seq
// continues across calls so every stage's mbarrier phase is (use / stages) & 1
__device__ void bulk_copy_range(uint8_t *dst, const uint8_t *src, uint64_t n, uint8_t *stage,
                                uint64_t *bars, uint32_t &seq) {
  const uint32_t np = (uint32_t)((n + kBulkChunk - 1) / kBulkChunk);
  auto bytes_of = [&](uint32_t p) {
    const uint64_t off = (uint64_t)p * kBulkChunk;
    return (uint32_t)(n - off < (uint64_t)kBulkChunk ? n - off : kBulkChunk);
  };
  const uint32_t pre = np < (uint32_t)kBulkStages ? np : kBulkStages;
  for (uint32_t p = 0; p < pre; ++p) {
    const uint32_t st = (seq + p) % kBulkStages;
    mbar_expect_tx(&bars[st], bytes_of(p));
    bulk_g2s(stage + st * kBulkChunk, src + (uint64_t)p * kBulkChunk, bytes_of(p), &bars[st]);
  }
  for (uint32_t p = 0; p < np; ++p) {
    const uint32_t q = seq + p, st = q % kBulkStages;
    mbar_wait(&bars[st], (q / kBulkStages) & 1);
    bulk_s2g(dst + (uint64_t)p * kBulkChunk, stage + st * kBulkChunk, bytes_of(p));
    if (p >= 1 && p - 1 + kBulkStages < np) {
      bulk_wait_read<1>();  // piece p-1's store has read its stage: refill it
      const uint32_t pp = p - 1 + kBulkStages, s2 = (seq + pp) % kBulkStages;
      mbar_expect_tx(&bars[s2], bytes_of(pp));
      bulk_g2s(stage + s2 * kBulkChunk, src + (uint64_t)pp * kBulkChunk, bytes_of(pp),
               &bars[s2]);
    }
  }
  bulk_wait_all();
  seq += np;
}

template <bool kTma>
__global__ void __launch_bounds__(512) k_pull_stream(const __grid_constant__ StreamEdgeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_i;
  __shared__ int s_last;
  uint64_t *bars = (uint64_t *)(smem + kBulkChunk * kBulkStages);
  uint32_t seq = 0;
  if (kTma && threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t total = a.rounds * a.nchunks;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(a.claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= total) break;
    const uint32_t jr = i / a.nchunks;
    const uint32_t c = i - jr * a.nchunks;
    const uint64_t j = a.first_round + jr;
    const uint32_t slot = (uint32_t)(j % a.slots);
    const uint32_t m = (uint32_t)(j / a.slots);
    uint8_t *d = a.dst + (uint64_t)slot * a.slot_stride;
    if (threadIdx.x == 0 && *(volatile int *)a.err == 0) {
      // the sender posted round j (its payload is in place) ...
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u64(a.posted) < j + 1) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          break;
        }
        __nanosleep(32);
      }
      // ... the slot's previous use was released, and consumed (its flag
      // read 0 again: the consumer's clear, a local load here)
      wait_count(a.released + slot, m, a.timeout_ns, a.err);
      if (m > 0 && !spin_until(d + a.nbytes, 0, a.timeout_ns, 0)) atomicExch(a.err, 2);
    }
    __syncthreads();
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t n = a.nbytes - off < a.chunk ? a.nbytes - off : a.chunk;
    const uint8_t *s = a.src + (j % a.nsrc) * a.src_stride + off;
    if (*(volatile int *)a.err == 0) {
      if (kTma) {
        const uint64_t mid = n & ~15ull;  // create() checked 16-B alignment
        if (threadIdx.x == 0 && mid) bulk_copy_range(d + off, s, mid, smem, bars, seq);
        for (uint64_t k = mid + threadIdx.x; k < n; k += blockDim.x)
          d[off + k] = ld_byte<true>(s + k);
        if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
      } else {
        // coherent loads: a source may be rewritten between rounds
        copy_bytes_grid<8, true, true>(d + off, s, n, threadIdx.x, blockDim.x, false);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(a.arrival + slot, a.nchunks - 1, 0);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      atomicExch(a.arrival + slot, 0u);
      if (*(volatile int *)a.err == 0) release_tail(d + a.nbytes, 1, 0);  // flag last
      count_done(a.released + slot);
      if (a.pulled) {
        // the source's use is fully read: the sender may rewrite it
        const unsigned v = (unsigned)(j / a.nsrc) + 1;
        asm volatile("red.release.sys.global.max.u32 [%0], %1;" ::"l"(a.pulled + j % a.nsrc),
                     "r"(v)
                     : "memory");
      }
    }
  }
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    *a.exit_count = 0;
  }
}

// Few-slot pull edges (the reference's ONE region per edge, or two):
// k_pull_stream_pre stages an item's whole chunk (<= kBulkStages x 16 KiB) in
// shared memory as soon as its round is posted, and stores it into the slot
// only once the slot is free.  With one slot the next round's NVLink reads
// then overlap the consumer's poll of this round instead of starting after
// its clear - the round-trip latency is what caps a single region.
__global__ void __launch_bounds__(256) k_pull_stream_pre(const __grid_constant__ StreamEdgeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_i;
  __shared__ int s_last;
  uint64_t *bars = (uint64_t *)(smem + kBulkChunk * kBulkStages);
  uint32_t uses[kBulkStages];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) {
      mbar_init(&bars[i], 1);
      uses[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t total = a.rounds * a.nchunks;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(a.claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= total) break;
    const uint32_t jr = i / a.nchunks;
    const uint32_t c = i - jr * a.nchunks;
    const uint64_t j = a.first_round + jr;
    const uint32_t slot = (uint32_t)(j % a.slots);
    const uint32_t m = (uint32_t)(j / a.slots);
    uint8_t *d = a.dst + (uint64_t)slot * a.slot_stride;
    const uint64_t off = (uint64_t)c * a.chunk;
    const uint64_t n = a.nbytes - off < a.chunk ? a.nbytes - off : a.chunk;
    const uint8_t *src = a.src + (j % a.nsrc) * a.src_stride + off;
    const uint64_t mid = n & ~15ull;
    const uint32_t np = (uint32_t)((mid + kBulkChunk - 1) / kBulkChunk);
    uint32_t issued = 0;   // (thread 0) stages whose loads are in flight
    if (threadIdx.x == 0 && *(volatile int *)a.err == 0) {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u64(a.posted) < j + 1) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          break;
        }
        __nanosleep(32);
      }
      // stage the chunk now ...
      if (*(volatile int *)a.err == 0)
        for (uint32_t p = 0; p < np; ++p, ++issued) {
          const uint32_t b = (uint32_t)((mid - (uint64_t)p * kBulkChunk) < kBulkChunk
                                            ? mid - (uint64_t)p * kBulkChunk : kBulkChunk);
          mbar_expect_tx(&bars[p], b);
          bulk_g2s(smem + p * kBulkChunk, src + (uint64_t)p * kBulkChunk, b, &bars[p]);
        }
      // ... and wait for the slot only before writing it
      wait_count(a.released + slot, m, a.timeout_ns, a.err);
      if (m > 0 && !spin_until(d + a.nbytes, 0, a.timeout_ns, 0)) atomicExch(a.err, 2);
    }
    __syncthreads();
    const bool ok = *(volatile int *)a.err == 0;
    if (threadIdx.x == 0) {
      for (uint32_t p = 0; p < issued; ++p) {
        mbar_wait(&bars[p], uses[p] & 1);   // (issued loads complete either way)
        ++uses[p];
        if (ok) {
          const uint32_t b = (uint32_t)((mid - (uint64_t)p * kBulkChunk) < kBulkChunk
                                            ? mid - (uint64_t)p * kBulkChunk : kBulkChunk);
          bulk_s2g(d + off + (uint64_t)p * kBulkChunk, smem + p * kBulkChunk, b);
        }
      }
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (ok)
      for (uint64_t k = mid + threadIdx.x; k < n; k += blockDim.x) d[off + k] = ld_byte<true>(src + k);
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(a.arrival + slot, a.nchunks - 1, 0);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      atomicExch(a.arrival + slot, 0u);
      if (*(volatile int *)a.err == 0) release_tail(d + a.nbytes, 1, 0);
      count_done(a.released + slot);
      if (a.pulled) {
        const unsigned v = (unsigned)(j / a.nsrc) + 1;
        asm volatile("red.release.sys.global.max.u32 [%0], %1;" ::"l"(a.pulled + j % a.nsrc),
                     "r"(v)
                     : "memory");
      }
    }
  }
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    *a.exit_count = 0;
  }
}

// Sender side of a pull edge: publish "rounds [.., count) are posted" into
// the receiver's word (one posted store, system-scope release: the payload
// writes that preceded it on this stream are visible to the receiver's
// pulls).  With wait_pulled, first wait until the source the first new round
// reuses was fully pulled (pulled[src] >= need): a sender that rewrites its
// sources between posts never overwrites bytes a pull may still read.
__global__ void k_post_rounds(unsigned long long *posted, unsigned long long count,
                              const unsigned int *wait_pulled, uint32_t need,
                              uint64_t timeout_ns, int *err) {
  if (wait_pulled && need) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys_u32(wait_pulled) < need) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicExch(err, 2);
        return;
      }
      __nanosleep(64);
    }
  }
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(posted), "l"(count) : "memory");
}

// ---------------------------------------------------------------------------
// Pipelined DYNAMIC edge (extension of dynamic allocation, runtime/protocol.py
// :147-254): `slots` metadata blocks on the receiver instead of one.  The
// sender (k_dyn_send_stream, one thread) writes round j's 8D+33-byte block -
// byte-identical to encode_meta (wire.py:109-119): element code, rank, dims,
// the payload's space address, token, length, flag last with a system-scope
// release - into slot j % slots once that slot's flag reads 0 (the credit).
// The receiver (k_dyn_pull_stream, persistent, TMA) acquires the flag, decodes
// and validates the block like decode_meta + check_remote_access
// (wire.py:122-144, memspace.py:145-157), allocates the round's block on
// demand from a device ring arena (in round order: the chunk-0 CTA bumps the
// head, waiting while the ring is full), pulls the payload from the sender's
// pool into it (the one-sided read of fabric.py:371-389) and marks it ready.
// The consumer (k_dyn_consume_stream) reads the block, frees it (ring tail)
// and clears the metadata flag - the sender's credit for the slot.
// ---------------------------------------------------------------------------
static constexpr int kDynMaxRank = 8;

struct DynEdgeArgs {
  uint8_t *meta;                  // receiver: slot 0's metadata block (local)
  uint64_t meta_stride;
  uint32_t slots, rank;
  const uint8_t *peer_base;       // receiver's mapping of the sender's pool
  uint64_t lo, hi, token;         // the sender's payload region (its space coordinates)
  uint64_t max_bytes, chunk;
  uint32_t nchunks;
  uint8_t *ring;
  uint64_t ring_cap;
  unsigned long long *alloc_head, *freed;  // bytes allocated / freed (monotonic)
  unsigned int *alloc_seq;        // rounds allocated
  unsigned int *consumed;         // rounds consumed (their flags cleared)
  unsigned long long *out;        // [slots][3]: offset, length, allocation end
  uint8_t *ready;                 // [slots]: round's block complete
  unsigned int *arrival, *claim, *exit_count;
  uint64_t first_round;
  uint32_t rounds;
  uint64_t timeout_ns;
  int *err;
};

__device__ __forceinline__ uint64_t ld_volatile_u64(const void *p) {
  return *(const volatile uint64_t *)p;
}

struct DynSendArgs {
  uint8_t *meta;                  // the receiver's slot 0 (through the sender's mapping)
  uint64_t meta_stride;
  uint32_t slots, rank, code, nsrc;
  uint64_t dims[kDynMaxRank];
  uint64_t src_addr, src_stride, token, nbytes;  // payload j % nsrc (space coordinates)
  uint64_t first_round;
  uint32_t rounds;
  uint64_t timeout_ns;
  int *err;
};

// up to 32 warps: warp t owns the slots s with s % L == t (L = min(32, slots)) and
// writes their rounds in order, so up to L rounds' credit polls and metadata
// writes are in flight at once (one thread spent ~4 us per round on the
// remote flag read and the system-scope release, which capped 1 MiB rounds at
// ~260 GB/s); a slot's rounds stay on one lane, so a credit read 0 can only
// be the slot's previous round's
__global__ void k_dyn_send_stream(const __grid_constant__ DynSendArgs a) {
  // one active lane per warp: lanes of one warp spinning on different flags
  // would serialise their divergent polls
  const uint32_t warps = blockDim.x / 32, me = threadIdx.x / 32;
  const uint32_t L = a.slots < warps ? a.slots : warps;
  if (threadIdx.x % 32 != 0 || me >= L) return;
  for (uint32_t r = 0; r < a.rounds; ++r) {
    const uint64_t j = a.first_round + r;
    if ((uint32_t)(j % a.slots) % L != me) continue;
    uint8_t *m = a.meta + (j % a.slots) * a.meta_stride;
    uint8_t *flag = m + 8ull * a.rank + 32;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys_u8(flag) != 0) {       // the consumer's credit
      if (globaltimer_ns() - t0 > a.timeout_ns) {
        atomicExch(a.err, 2);
        return;
      }
      __nanosleep(32);
    }
    uint64_t *w = (uint64_t *)m;
    w[0] = (uint64_t)a.code | ((uint64_t)a.rank << 8);
    for (uint32_t k = 0; k < a.rank; ++k) w[1 + k] = a.dims[k];
    w[1 + a.rank] = a.src_addr + (j % a.nsrc) * a.src_stride;
    w[2 + a.rank] = a.token;
    w[3 + a.rank] = a.nbytes;
    release_tail(flag, 1, 1);                     // flag last
  }
}

__global__ void __launch_bounds__(256) k_dyn_pull_stream(const __grid_constant__ DynEdgeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_i;
  __shared__ int s_last, s_bad;
  __shared__ uint64_t s_off, s_len, s_src;
  uint64_t *bars = (uint64_t *)(smem + kBulkChunk * kBulkStages);
  uint32_t seq = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t total = a.rounds * a.nchunks;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(a.claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= total) break;
    const uint32_t jr = i / a.nchunks;
    const uint32_t c = i - jr * a.nchunks;
    const uint64_t j = a.first_round + jr;
    const uint32_t slot = (uint32_t)(j % a.slots);
    const uint8_t *m = a.meta + (uint64_t)slot * a.meta_stride;
    if (threadIdx.x == 0) {
      s_bad = *(volatile int *)a.err != 0;
      const uint64_t t0 = globaltimer_ns();
      // the slot's previous round must have been consumed (its flag cleared):
      // a flag still set from round j - slots is not round j's
      while (!s_bad && j >= a.slots &&
             ld_acquire_gpu_u32(a.consumed) < (uint32_t)(j - a.slots + 1)) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          s_bad = 1;
        }
        __nanosleep(32);
      }
      while (!s_bad && ld_acquire_sys_u8(m + 8ull * a.rank + 32) != 1) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          s_bad = 1;
        }
        __nanosleep(32);
      }
      uint64_t addr = 0, plen = 0;
      if (!s_bad) {
        // decode_meta + check_remote_access on the device
        const uint32_t code = ((const volatile uint8_t *)m)[0];
        const uint32_t rk = ((const volatile uint8_t *)m)[1];
        const uint64_t esz = code == 0 ? 4 : code == 1 ? 8 : code == 2 ? 4 : code == 3 ? 8
                           : code == 4 ? 1 : 0;
        uint64_t prod = esz;
        for (uint32_t k = 0; k < a.rank; ++k) prod *= ld_volatile_u64(m + 8 + 8 * k);
        addr = ld_volatile_u64(m + 8 + 8 * a.rank);
        const uint64_t tok = ld_volatile_u64(m + 16 + 8 * a.rank);
        plen = ld_volatile_u64(m + 24 + 8 * a.rank);
        if (rk != a.rank || esz == 0 || prod != plen || plen > a.max_bytes || tok != a.token ||
            addr < a.lo || addr + plen > a.hi) {
          atomicExch(a.err, 6);
          s_bad = 1;
        }
      }
      uint64_t off = 0;
      if (!s_bad && c == 0) {
        // on-demand allocation from the ring arena, in round order
        const uint64_t t1 = globaltimer_ns();
        while (ld_acquire_gpu_u32(a.alloc_seq) != (uint32_t)j && !s_bad) {
          if (globaltimer_ns() - t1 > a.timeout_ns) { atomicExch(a.err, 7); s_bad = 1; }
          __nanosleep(20);
        }
        uint64_t head = ld_volatile_u64(a.alloc_head);
        const uint64_t need = plen ? (plen + 255) & ~255ull : 256;
        if (head % a.ring_cap + need > a.ring_cap) head += a.ring_cap - head % a.ring_cap;
        const uint64_t end = head + need;
        while (!s_bad) {   // wait until the consumer freed enough of the ring
          uint64_t fr;
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(fr) : "l"(a.freed) : "memory");
          if (fr + a.ring_cap >= end) break;
          if (globaltimer_ns() - t1 > a.timeout_ns) { atomicExch(a.err, 7); s_bad = 1; }
          __nanosleep(32);
        }
        off = head % a.ring_cap;
        unsigned long long *o = a.out + 3ull * slot;
        o[0] = off;
        o[1] = plen;
        o[2] = end;
        *(volatile unsigned long long *)a.alloc_head = end;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.alloc_seq),
                     "r"((unsigned)j + 1) : "memory");
      } else if (!s_bad) {
        const uint64_t t1 = globaltimer_ns();
        while (ld_acquire_gpu_u32(a.alloc_seq) < (uint32_t)j + 1 && !s_bad) {
          if (globaltimer_ns() - t1 > a.timeout_ns) { atomicExch(a.err, 7); s_bad = 1; }
          __nanosleep(20);
        }
        off = ld_volatile_u64(a.out + 3ull * slot);
      }
      s_off = off;
      s_len = plen;
      s_src = (uint64_t)(a.peer_base + addr);
    }
    __syncthreads();
    const uint64_t coff = (uint64_t)c * a.chunk;
    if (!s_bad && coff < s_len) {
      const uint64_t n = s_len - coff < a.chunk ? s_len - coff : a.chunk;
      uint8_t *d = a.ring + s_off + coff;
      const uint8_t *s = (const uint8_t *)s_src + coff;
      if ((((uintptr_t)d | (uintptr_t)s) & 15) == 0) {
        const uint64_t mid = n & ~15ull;
        if (threadIdx.x == 0 && mid) bulk_copy_range(d, s, mid, smem, bars, seq);
        for (uint64_t k = mid + threadIdx.x; k < n; k += blockDim.x) d[k] = ld_byte<true>(s + k);
        if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
      } else {
        copy_bytes_grid<8, true, true>(d, s, n, threadIdx.x, blockDim.x, false);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(a.arrival + slot, a.nchunks - 1, 0);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      atomicExch(a.arrival + slot, 0u);
      if (*(volatile int *)a.err == 0) release_tail(a.ready + slot, 1, 0);
    }
  }
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    *a.exit_count = 0;
  }
}

// The receiver's consumer: round j's block, in order; mode 1 stores a weighted
// byte checksum per round (tests); then frees the block (ring tail) and clears
// the metadata flag (the sender's credit, DynReceiver.poll's clear).
__global__ void __launch_bounds__(1024) k_dyn_consume_stream(DynEdgeArgs a, uint64_t first_round,
                                                              uint32_t rounds, int mode,
                                                              unsigned long long *sums,
                                                              uint32_t *started, uint32_t ticket) {
  __shared__ unsigned long long acc;
  __shared__ int ok;
  if (threadIdx.x == 0 && started) {
    *(volatile uint32_t *)started = ticket;
    __threadfence_system();
  }
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint64_t j = first_round + r;
    const uint32_t slot = (uint32_t)(j % a.slots);
    if (threadIdx.x == 0) {
      acc = 0;
      ok = spin_until(a.ready + slot, 1, a.timeout_ns, 0) ? 1 : 0;
      if (!ok) atomicExch(a.err, 1);
    }
    __syncthreads();
    if (!ok) return;
    const uint64_t off = ld_volatile_u64(a.out + 3ull * slot);
    const uint64_t len = ld_volatile_u64(a.out + 3ull * slot + 1);
    const uint64_t end = ld_volatile_u64(a.out + 3ull * slot + 2);
    if (mode & 1) {
      unsigned long long sum = 0;
      const uint8_t *b = a.ring + off;
      for (uint64_t i = threadIdx.x; i < len; i += blockDim.x)
        sum += (unsigned long long)__ldcg(b + i) * (i % 251 + 1);
      atomicAdd(&acc, sum);
      __syncthreads();
      if (threadIdx.x == 0) sums[r] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      a.ready[slot] = 0;
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.freed), "l"(end) : "memory");
      if (mode & 1) __threadfence_system();  // checksummed reads before the credit
      // the credit: a relaxed store - the consumer read nothing the sender
      // will rewrite (a system-scope release here is a MEMBAR.SYS per round
      // in the one serial thread; device_stream.cuh k_consume_stream)
      st_relaxed_sys_u8(a.meta + (uint64_t)slot * a.meta_stride + 8ull * a.rank + 32, 0);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.consumed),
                   "r"((unsigned)j + 1) : "memory");
    }
    __syncthreads();
  }
}
