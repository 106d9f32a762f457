// host_launch.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Launch geometry, copy-engine K1 variant, DeviceGuard.

// ---------------------------------------------------------------------------
// launch geometry
// ---------------------------------------------------------------------------
static void copy_geometry(int device, uint64_t bytes, int *grid, int *block) {
  const int threads = g_copy_threads;
  // one CTA per 16 KiB (small puts spread over many SMs: latency), capped at
  // k CTAs/SM (large puts: fewer CTAs polling the credit and arriving)
  const uint64_t per_cta = 16 << 10;
  uint64_t want = (bytes + per_cta - 1) / per_cta;
  uint64_t cap = (uint64_t)sm_count_of(device) * g_ctas_per_sm;
  if (want < 1) want = 1;
  if (want > cap) want = cap;
  *grid = (int)want;
  *block = threads;
}

// Completion events (one per verb) are recycled through a per-device pool:
// cudaEventCreate/Destroy per verb cost more host time than the record.
static std::mutex g_event_pool_mu;
static std::vector<srf_event *> g_event_pool[64];

static int record_event(int device, cudaStream_t s, srf_event_t *ev_out) {
  if (!ev_out) return SRF_OK;
  srf_event *ev = nullptr;
  if (device >= 0 && device < 64) {
    std::lock_guard<std::mutex> g(g_event_pool_mu);
    if (!g_event_pool[device].empty()) {
      ev = g_event_pool[device].back();
      g_event_pool[device].pop_back();
    }
  }
  cudaError_t e = cudaSuccess;
  if (!ev) {
    ev = new srf_event();
    ev->device = device;
    ev->pooled = device >= 0 && device < 64;
    e = cudaEventCreateWithFlags(&ev->e, cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventRecord(ev->e, s);
  if (e != cudaSuccess) {
    delete ev;
    return fail(SRF_E_DEVICE, "event: %s", cudaGetErrorString(e));
  }
  *ev_out = ev;
  return SRF_OK;
}

static void release_event(srf_event *ev) {
  if (ev->pooled) {
    std::lock_guard<std::mutex> g(g_event_pool_mu);
    if (g_event_pool[ev->device].size() < 4096) {
      g_event_pool[ev->device].push_back(ev);
      return;
    }
  }
  cudaEventDestroy(ev->e);
  delete ev;
}

static int launch_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(SRF_E_DEVICE, "%s launch: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  rec_check_launch(what);
  return SRF_OK;
}

static int g_put_impl = 0;  // 0 = vector LDG/STG, 1 = TMA bulk (large segments)
static int g_unroll = 8;    // 16-B vectors in flight per thread (4 or 8)
// knob 6: cross-device bodies of at least this many bytes move on the copy
// engine (0: never, the default - every byte moves in a kernel).  Kept as a
// labelled comparator: round 1 used it from 32 MiB because one-slot K1
// rounds got ~616 GB/s per direction in the ring vs the engine's 713; the
// pipelined edge (srf_edge_*) reaches ~707 with SM stores alone
// (profiles/r2_edge_probe.jsonl).
static uint64_t g_peer_ce_bytes = 0;
static int g_force_sys = 0;  // knob 7 (tests): every put/get takes the cross-device path
static uint64_t g_put_timeout_ns = 5000000000ull;  // knob 8: credit wait limit of a put
static int g_edge_ctas_per_sm = 2;   // knob 9: pipelined edge CTAs per SM
static int g_edge_ctas = 0;          // knob 14: pipelined edge CTAs in total (0: per-SM knob)
static uint64_t g_edge_chunk = 0;    // knob 10: pipelined edge chunk (KiB; 0 = automatic)
static int g_consume_threads = 256;  // knob 11: flag-only edge consumer CTA size (warps in parallel)
static int g_consume_release = 0;    // knob 13: flag-only consumer clears with release.sys
static int g_pull_no_prefetch = 0;   // knob 16: few-slot pull edges without early staging
// knob 12: GenGrad work-unit size.  A unit's thread 0 derives the PCG64 stream
// and jumps to the unit's first element (~150 dependent 128-bit multiplies)
// before the CTA generates, so units must be large enough to amortise that.
static uint64_t g_gen_unit_bytes = 128 << 10;

// launch K1/K4/K5 with the configured implementation
static int launch_copy(const PutArgs &a, srf_stream *s, const char *what) {
  uint64_t big = 0;
  for (int i = 0; i < a.nseg; ++i) big = std::max<uint64_t>(big, a.seg[i].len);
  // the TMA variant has no fused consume (its non-bulk remainder keeps the
  // pull's source-aligned sectors)
  if (g_put_impl == 1 && big >= (uint64_t)4 * kBulkChunk && !a.consume) {
    static bool attr_set[64] = {false};
    if (s->device >= 0 && s->device < 64 && !attr_set[s->device]) {
      CUDA_TRY(cudaFuncSetAttribute(k_put_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kBulkSmem));
      attr_set[s->device] = true;
    }
    uint64_t chunks = (a.total + kBulkChunk - 1) / kBulkChunk;
    uint64_t cap = (uint64_t)sm_count_of(s->device) * 2;
    int grid = (int)std::max<uint64_t>(1, std::min(chunks, cap));
    k_put_bulk<<<grid, 256, kBulkSmem, s->s>>>(a);
    if (recording()) rec_put(a, s, grid, 256, 4);
  } else {
    int grid, block;
    copy_geometry(s->device, a.total, &grid, &block);
    // a large segment whose ends are not co-aligned mod 32 takes the
    // sector-realigning kernel; everything else the lean one
    bool sectors = false;
    for (int i = 0; i < a.nseg; ++i)
      if (a.seg[i].len >= 4096 &&
          (((uintptr_t)(a.dst + a.seg[i].dst_off) ^ (uintptr_t)a.seg[i].src) & 31) != 0)
        sectors = true;
    if (g_unroll == 8) {
      if (sectors)
        k_put<8, true><<<grid, block, 0, s->s>>>(a);
      else
        k_put<8, false><<<grid, block, 0, s->s>>>(a);
    } else {
      if (sectors)
        k_put<4, true><<<grid, block, 0, s->s>>>(a);
      else
        k_put<4, false><<<grid, block, 0, s->s>>>(a);
    }
    if (recording())
      rec_put(a, s, grid, block, (g_unroll == 8 ? 0 : 2) + (sectors ? 1 : 0));
  }
  return launch_check(what);
}

// K1 with a copy-engine body: body copies -> a one-thread K1 that releases
// the tail byte.  Stream order starts the tail kernel only after the copies
// have completed, so a consumer that acquires the flag sees the body
// (release/acquire stress test, tests/test_gpu_kernels.py).  Only for puts
// without a credit wait: a DMA copy cannot be skipped when a credit times
// out, so credit-gated puts stay on the kernel (put_impl).
static int put_via_copy_engine(const PutArgs &a, srf_stream *s) {
  if (recording()) rec_dirty("copy-engine body");
  const uint64_t body = a.total - 1;
  for (int i = 0; i < a.nseg; ++i) {
    const Seg &sg = a.seg[i];
    if (sg.dst_off >= body) break;
    const uint64_t n = std::min<uint64_t>(sg.len, body - sg.dst_off);
    CUDA_TRY(cudaMemcpyAsync(a.dst + sg.dst_off, sg.src, n, cudaMemcpyDeviceToDevice, s->s));
  }
  PutArgs t = a;
  const Seg &ls = a.seg[a.nseg - 1];
  t.nseg = 1;
  t.seg[0].src = ls.src + ls.len - 1;
  t.seg[0].dst_off = a.total - 1;
  t.seg[0].len = 1;
  t.wait_empty = 0;
  k_put<4, false><<<1, 32, 0, s->s>>>(t);
  return launch_check("k_put(tail)");
}

// Restores the caller's current device when an API call returns: entry
// points switch to the device of the objects they touch, and a caller (torch
// with device="cuda") must not see that switch.
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  }
  ~DeviceGuard() {
    int now = -1;
    if (dev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != dev) cudaSetDevice(dev);
  }
};
