// abi_core.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// C ABI: knobs, spaces, regions, verbs (put/get/copy/flag/apply), torch pool, streams.

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *srf_last_error(void) { return g_last_error.c_str(); }
int srf_version(void) { return 1; }

int srf_tune(int knob, int value) {
  DeviceGuard device_guard;
  switch (knob) {
    case 0:
      if (value < 1 || value > 32) return fail(SRF_E_INVALID_CONFIG, "ctas_per_sm");
      g_ctas_per_sm = value;
      return SRF_OK;
    case 1:
      if (value != 128 && value != 256 && value != 512)
        return fail(SRF_E_INVALID_CONFIG, "copy threads must be 128, 256 or 512");
      g_copy_threads = value;
      return SRF_OK;
    case 2:
      if (value != 0 && value != 1) return fail(SRF_E_INVALID_CONFIG, "put impl 0|1");
      g_put_impl = value;
      return SRF_OK;
    case 3:
      if (value != 0 && value != 1) return fail(SRF_E_INVALID_CONFIG, "alloc 0=cudaMalloc|1=vmm");
      g_alloc_vmm = value;
      return SRF_OK;
    case 4:
      if (value != 4 && value != 8) return fail(SRF_E_INVALID_CONFIG, "unroll 4|8");
      g_unroll = value;
      return SRF_OK;
    case 5: {
      if (value != 0 && value != 1) return fail(SRF_E_INVALID_CONFIG, "vec32 0|1");
      int ndev = 0;
      cudaGetDeviceCount(&ndev);
      int cur = 0;
      cudaGetDevice(&cur);
      for (int dev = 0; dev < ndev; ++dev) {
        CUDA_TRY(cudaSetDevice(dev));
        CUDA_TRY(cudaMemcpyToSymbol(g_vec32, &value, sizeof value));
      }
      cudaSetDevice(cur);
      return SRF_OK;
    }
    case 6:
      if (value < 0) return fail(SRF_E_INVALID_CONFIG, "peer_ce_kib >= 0");
      g_peer_ce_bytes = (uint64_t)value << 10;
      return SRF_OK;
    case 7:
      // test knob: treat every destination/source as a peer's memory -
      // system-scope arrival/release and the copy-engine body path - so a
      // one-GPU box exercises the cross-device code
      if (value != 0 && value != 1) return fail(SRF_E_INVALID_CONFIG, "force_sys 0|1");
      g_force_sys = value;
      return SRF_OK;
    case 8:
      if (value < 1) return fail(SRF_E_INVALID_CONFIG, "put_timeout_ms >= 1");
      g_put_timeout_ns = (uint64_t)value * 1000000ull;
      return SRF_OK;
    case 9:
      if (value < 1 || value > 4) return fail(SRF_E_INVALID_CONFIG, "edge_ctas_per_sm 1..4");
      g_edge_ctas_per_sm = value;
      return SRF_OK;
    case 10:
      if (value < 0) return fail(SRF_E_INVALID_CONFIG, "edge_chunk_kib >= 0");
      g_edge_chunk = (uint64_t)value;
      return SRF_OK;
    case 12:
      if (value < 16) return fail(SRF_E_INVALID_CONFIG, "gen_unit_kib >= 16");
      g_gen_unit_bytes = (uint64_t)value << 10;
      return SRF_OK;
    case 13:
      g_consume_release = value ? 1 : 0;
      return SRF_OK;
    case 16:
      g_pull_no_prefetch = value ? 1 : 0;
      return SRF_OK;
    case 14:
      if (value < 0 || value > 4096) return fail(SRF_E_INVALID_CONFIG, "edge_ctas 0..4096");
      g_edge_ctas = value;
      return SRF_OK;
    case 11:
      if (value < 32 || value > 1024 || value % 32)
        return fail(SRF_E_INVALID_CONFIG, "consume_threads: a multiple of 32 in [32, 1024]");
      g_consume_threads = value;
      return SRF_OK;
    default:
      return fail(SRF_E_INVALID_CONFIG, "unknown knob %d", knob);
  }
}
uint64_t srf_launch_count(void) { return g_launches.load(); }

int srf_host_alloc(uint64_t nbytes, void **out) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaHostAlloc(out, nbytes ? nbytes : 1, cudaHostAllocPortable));
  memset(*out, 0, nbytes ? nbytes : 1);
  return SRF_OK;
}

int srf_host_free(void *p) {
  DeviceGuard device_guard;
  if (p) cudaFreeHost(p);
  return SRF_OK;
}

// ---------------------------------------------------------------------------
// Registered pool for torch's CUDA allocator: torch tensors
// are born inside a registered region, so any of them is a zero-copy source
// or destination of a one-sided verb (analyzer.py:226-272 generalised beyond
// the synthetic producers).  First fit over an offset-ordered free map with
// coalescing; a freed block returns to the map only once the work queued on
// the freeing stream has passed it (event), like the caching allocator's
// stream-ordered reuse.
// ---------------------------------------------------------------------------
struct TorchPool {
  srf_space *sp = nullptr;
  uint64_t base = 0, cap = 0;  // region [base, base + cap) of sp
  std::map<uint64_t, uint64_t> free_;        // offset -> length
  std::unordered_map<uint64_t, uint64_t> live;
  struct Pending { uint64_t off, len; cudaEvent_t ev; };
  std::vector<Pending> pending;
  uint64_t in_use = 0, peak = 0;
  std::mutex mu;
};
static TorchPool *g_tpool[64] = {nullptr};
static constexpr uint64_t kTorchAlign = 512;

static void tpool_insert_free(TorchPool *p, uint64_t off, uint64_t len) {
  auto it = p->free_.emplace(off, len).first;
  auto nx = std::next(it);
  if (nx != p->free_.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    p->free_.erase(nx);
  }
  if (it != p->free_.begin()) {
    auto pv = std::prev(it);
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      p->free_.erase(it);
    }
  }
}

static void tpool_reclaim(TorchPool *p, bool wait) {
  size_t k = 0;
  for (auto &q : p->pending) {
    if (wait) cudaEventSynchronize(q.ev);
    if (cudaEventQuery(q.ev) == cudaSuccess) {
      cudaEventDestroy(q.ev);
      tpool_insert_free(p, q.off, q.len);
    } else {
      p->pending[k++] = q;
    }
  }
  p->pending.resize(k);
}

int srf_torch_pool_attach(srf_space_t sp, uint64_t region_addr, uint64_t length) {
  DeviceGuard device_guard;
  if (!sp || sp->imported) return fail(SRF_E_INVALID_CONFIG, "torch pool needs a local space");
  int rc = check_raw(sp, region_addr, length, "torch pool");
  if (rc) return rc;
  if (sp->device < 0 || sp->device >= 64 || g_tpool[sp->device])
    return fail(SRF_E_INVALID_CONFIG, "GPU %d already has a torch pool", sp->device);
  TorchPool *p = new TorchPool();
  p->sp = sp;
  const uint64_t a0 = (region_addr + kTorchAlign - 1) / kTorchAlign * kTorchAlign;
  p->base = a0;
  p->cap = (region_addr + length - a0) / kTorchAlign * kTorchAlign;
  p->free_.emplace(0, p->cap);
  g_tpool[sp->device] = p;
  return SRF_OK;
}

int srf_torch_pool_stats(int device, uint64_t *in_use, uint64_t *peak, uint64_t *capacity) {
  DeviceGuard device_guard;
  if (device < 0 || device >= 64 || !g_tpool[device])
    return fail(SRF_E_INVALID_CONFIG, "no torch pool on GPU %d", device);
  TorchPool *p = g_tpool[device];
  std::lock_guard<std::mutex> g(p->mu);
  *in_use = p->in_use;
  *peak = p->peak;
  *capacity = p->cap;
  return SRF_OK;
}

void *srf_torch_malloc(ssize_t size, int device, void *stream) {
  (void)stream;
  if (size < 0 || device < 0 || device >= 64) return nullptr;
  if (!g_tpool[device]) {
    // a GPU without a pool: plain device memory (torch works, nothing registered)
    void *q = nullptr;
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&q, std::max<ssize_t>(size, 1)) !=
        cudaSuccess)
      return nullptr;
    return q;
  }
  TorchPool *p = g_tpool[device];
  const uint64_t len = std::max<uint64_t>(kTorchAlign,
                                          ((uint64_t)size + kTorchAlign - 1) / kTorchAlign *
                                              kTorchAlign);
  std::lock_guard<std::mutex> g(p->mu);
  for (int attempt = 0; attempt < 2; ++attempt) {
    tpool_reclaim(p, attempt == 1);
    for (auto it = p->free_.begin(); it != p->free_.end(); ++it) {
      if (it->second < len) continue;
      const uint64_t off = it->first, rest = it->second - len;
      p->free_.erase(it);
      if (rest) p->free_.emplace(off + len, rest);
      p->live[off] = len;
      p->in_use += len;
      p->peak = std::max(p->peak, p->in_use);
      return p->sp->base + p->base + off;
    }
  }
  // pool exhausted: ordinary device memory (the tensor works; a zero-copy
  // verb on it is refused as NotRegistered by the region checks)
  void *q = nullptr;
  if (cudaSetDevice(device) == cudaSuccess && cudaMalloc(&q, (size_t)size) == cudaSuccess)
    return q;
  if (getenv("SRFLOW_TPOOL_DEBUG")) {
    uint64_t largest = 0, total = 0;
    for (auto &kv : p->free_) { largest = std::max(largest, kv.second); total += kv.second; }
    fprintf(stderr, "srf_torch_malloc(%zd): no block; free %llu in %zu blocks (largest %llu), "
            "pending %zu, in use %llu\n", size, (unsigned long long)total, p->free_.size(),
            (unsigned long long)largest, p->pending.size(), (unsigned long long)p->in_use);
  }
  return nullptr;
}

void srf_torch_free(void *ptr, ssize_t size, int device, void *stream_) {
  DeviceGuard device_guard;
  cudaStream_t stream = (cudaStream_t)stream_;
  (void)size;
  if (!ptr || device < 0 || device >= 64) return;
  TorchPool *p = g_tpool[device];
  if (!p || (uint8_t *)ptr < p->sp->base + p->base ||
      (uint8_t *)ptr >= p->sp->base + p->base + p->cap) {
    cudaSetDevice(device);
    cudaFree(ptr);  // plain memory of a GPU without a pool
    return;
  }
  const uint64_t off = (uint64_t)((uint8_t *)ptr - (p->sp->base + p->base));
  std::lock_guard<std::mutex> g(p->mu);
  auto it = p->live.find(off);
  if (it == p->live.end()) return;
  const uint64_t len = it->second;
  p->live.erase(it);
  p->in_use -= len;
  cudaEvent_t ev = nullptr;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
      cudaEventRecord(ev, stream) == cudaSuccess) {
    p->pending.push_back({off, len, ev});
  } else {
    if (ev) cudaEventDestroy(ev);
    cudaStreamSynchronize(stream);
    tpool_insert_free(p, off, len);
  }
  cudaSetDevice(cur);
}

int srf_device_count(int *count) {
  DeviceGuard device_guard;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(SRF_E_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return SRF_OK;
}

int srf_space_create(int server_id, int cuda_device, uint64_t capacity,
                     uint32_t max_regions, srf_space_t *out) {
  DeviceGuard device_guard;
  if (capacity == 0) return fail(SRF_E_ZERO_LENGTH, "capacity must be >= 1");
  CUDA_TRY(cudaSetDevice(cuda_device));
  int rc_load = preload_kernels(cuda_device);
  if (rc_load) return rc_load;
  srf_space *sp = new srf_space();
  sp->server_id = server_id;
  sp->device = cuda_device;
  sp->capacity = capacity;
  sp->max_regions = max_regions;
  sp->imported = false;
  sp->next_addr = 0;
  sp->stream = nullptr;
  sp->err = nullptr;
  sp->vmm = g_alloc_vmm != 0;
  sp->export_fd = -1;
  sp->map_size = 0;
  if (sp->vmm) {
    cudaFree(0);  // make the primary context current for the driver calls
    int rc0 = vmm_alloc(sp);
    if (rc0 != SRF_OK) {
      delete sp;
      return rc0;
    }
  } else {
    cudaError_t e0 = cudaMalloc(&sp->base, capacity);
    if (e0 != cudaSuccess) {
      delete sp;
      return fail(SRF_E_OUT_OF_MEMORY, "server %d: cudaMalloc(%llu): %s",
                  server_id, (unsigned long long)capacity, cudaGetErrorString(e0));
    }
  }
  cudaError_t e;
  int rc = make_stream(cuda_device, true, nullptr, &sp->stream);
  if (rc == SRF_OK) {
    e = cudaMalloc(&sp->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(sp->err, 0, sizeof(int), sp->stream->s);
    // np.zeros semantics: the whole space reads as zero bytes (SM stores, see
    // k_zero_fill)
    if (e == cudaSuccess) {
      const int grid = sm_count_of(cuda_device) * 4;
      k_zero_fill<<<grid, 256, 0, sp->stream->s>>>(sp->base, capacity);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(sp->stream->s);
    if (e != cudaSuccess) rc = fail(SRF_E_DEVICE, "space init: %s", cudaGetErrorString(e));
  }
  if (rc != SRF_OK) {
    free_stream(sp->stream);
    if (sp->vmm)
      vmm_free(sp);
    else
      cudaFree(sp->base);
    if (sp->err) cudaFree(sp->err);
    delete sp;
    return rc;
  }
  *out = sp;
  return SRF_OK;
}

int srf_space_destroy(srf_space_t sp) {
  DeviceGuard device_guard;
  if (!sp) return SRF_OK;
  cudaSetDevice(sp->device);
  free_stream(sp->stream);
  if (sp->db) {
    for (auto &kv : *sp->db) cudaEventDestroy(kv.second.clear_ev);
    delete sp->db;
    cudaFreeHost(sp->db_host);
  }
  if (sp->vmm)
    vmm_free(sp);
  else if (sp->imported)
    cudaIpcCloseMemHandle(sp->base);
  else
    cudaFree(sp->base);
  if (sp->err) cudaFree(sp->err);
  delete sp;
  return SRF_OK;
}

int srf_space_info(srf_space_t sp, int *server_id, int *cuda_device,
                   uint64_t *capacity, void **device_base) {
  DeviceGuard device_guard;
  if (server_id) *server_id = sp->server_id;
  if (cuda_device) *cuda_device = sp->device;
  if (capacity) *capacity = sp->capacity;
  if (device_base) *device_base = sp->base;
  return SRF_OK;
}

void *srf_space_cuda_stream(srf_space_t sp) { return (void *)sp->stream->s; }

int srf_region_alloc(srf_space_t sp, uint64_t length, int registered,
                     uint64_t token, int64_t *region_id, uint64_t *base) {
  DeviceGuard device_guard;
  if (length < 1)
    return fail(SRF_E_ZERO_LENGTH, "region length must be >= 1, got %llu",
                (unsigned long long)length);
  std::lock_guard<std::mutex> g(sp->mu);
  if (sp->regions.size() >= sp->max_regions)
    return fail(SRF_E_OUT_OF_MEMORY, "server %d: region table full (%u)",
                sp->server_id, sp->max_regions);
  uint64_t b = (sp->next_addr + kAlign - 1) & ~(kAlign - 1);
  if (b + length > sp->capacity)
    return fail(SRF_E_OUT_OF_MEMORY,
                "server %d: need %llu bytes at %llu, capacity %llu",
                sp->server_id, (unsigned long long)length,
                (unsigned long long)b, (unsigned long long)sp->capacity);
  Region r{(int64_t)sp->regions.size(), b, length, registered != 0,
           registered ? token : 0};
  sp->regions.push_back(r);
  sp->next_addr = b + length;
  *region_id = r.id;
  *base = b;
  return SRF_OK;
}

int srf_region_import(srf_space_t proxy, int64_t region_id, uint64_t base,
                      uint64_t length, int registered, uint64_t token) {
  DeviceGuard device_guard;
  std::lock_guard<std::mutex> g(proxy->mu);
  if (base + length > proxy->capacity)
    return fail(SRF_E_OUT_OF_BOUNDS, "imported region escapes space");
  proxy->regions.push_back(Region{region_id, base, length, registered != 0,
                                  registered ? token : 0});
  proxy->next_addr = std::max(proxy->next_addr, base + length);
  return SRF_OK;
}

int srf_region_count(srf_space_t sp, uint32_t *count) {
  DeviceGuard device_guard;
  std::lock_guard<std::mutex> g(sp->mu);
  *count = (uint32_t)sp->regions.size();
  return SRF_OK;
}

int srf_next_addr(srf_space_t sp, uint64_t *next_addr) {
  DeviceGuard device_guard;
  std::lock_guard<std::mutex> g(sp->mu);
  *next_addr = sp->next_addr;
  return SRF_OK;
}

int srf_check_remote(srf_space_t sp, uint64_t addr, uint64_t length,
                     uint64_t token) {
  DeviceGuard device_guard;
  std::lock_guard<std::mutex> g(sp->mu);
  return check_remote_locked(sp, addr, length, token);
}

int srf_check_registered(srf_space_t sp, uint64_t addr, uint64_t length,
                         uint64_t token) {
  DeviceGuard device_guard;
  std::lock_guard<std::mutex> g(sp->mu);
  return check_registered_locked(sp, addr, length, token);
}

int srf_read(srf_space_t sp, uint64_t addr, uint64_t length, void *host_dst) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, length, "read");
  if (rc) return rc;
  if (length == 0) return SRF_OK;
  CUDA_TRY(cudaSetDevice(sp->device));
  CUDA_TRY(cudaMemcpyAsync(host_dst, sp->base + addr, length,
                           cudaMemcpyDeviceToHost, sp->stream->s));
  CUDA_TRY(cudaStreamSynchronize(sp->stream->s));
  return SRF_OK;
}

int srf_write(srf_space_t sp, uint64_t addr, uint64_t length,
              const void *host_src) {
  if (recording()) rec_dirty("host write into device memory");
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, length, "write");
  if (rc) return rc;
  if (length == 0) return SRF_OK;
  CUDA_TRY(cudaSetDevice(sp->device));
  CUDA_TRY(cudaMemcpyAsync(sp->base + addr, host_src, length,
                           cudaMemcpyHostToDevice, sp->stream->s));
  CUDA_TRY(cudaStreamSynchronize(sp->stream->s));
  return SRF_OK;
}

int srf_write_async(srf_space_t sp, uint64_t addr, uint64_t length,
                    const void *host_src, srf_stream_t st) {
  if (recording()) rec_dirty("host write into device memory");
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, length, "write");
  if (rc) return rc;
  if (length == 0) return SRF_OK;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  CUDA_TRY(cudaMemcpyAsync(sp->base + addr, host_src, length,
                           cudaMemcpyHostToDevice, s->s));
  return SRF_OK;
}

int srf_read_async(srf_space_t sp, uint64_t addr, uint64_t length,
                   void *host_dst, srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, length, "read");
  if (rc) return rc;
  if (length == 0) return SRF_OK;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  CUDA_TRY(cudaMemcpyAsync(host_dst, sp->base + addr, length,
                           cudaMemcpyDeviceToHost, s->s));
  return SRF_OK;
}

int srf_device_ptr(srf_space_t sp, uint64_t addr, void **dptr) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, 0, "view");
  if (rc) return rc;
  *dptr = sp->base + addr;
  return SRF_OK;
}

int srf_space_sync(srf_space_t sp) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(sp->device));
  CUDA_TRY(cudaStreamSynchronize(sp->stream->s));
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, sp->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) {
    cudaMemsetAsync(sp->err, 0, sizeof(int), sp->stream->s);
    cudaStreamSynchronize(sp->stream->s);
    if (err == 8)
      return fail(SRF_E_PROTOCOL, "server %d: RPC fragment out of order (ReassemblyGap)",
                  sp->server_id);
    if (err == 6)
      return fail(SRF_E_BAD_TOKEN,
                  "server %d: device-side metadata validation failed (token/bounds/length)",
                  sp->server_id);
    return fail(SRF_E_TIMEOUT, "server %d: device flag wait timed out (code %d)",
                sp->server_id, err);
  }
  return SRF_OK;
}

int srf_connect(srf_space_t a, srf_space_t b) {
  DeviceGuard device_guard;
  if (a->device == b->device) return SRF_OK;
  int can_ab = 0, can_ba = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can_ab, a->device, b->device));
  CUDA_TRY(cudaDeviceCanAccessPeer(&can_ba, b->device, a->device));
  if (!can_ab || !can_ba)
    return fail(SRF_E_PEER_UNREACHABLE, "GPU %d and GPU %d have no peer path",
                a->device, b->device);
  const int pairs[2][2] = {{a->device, b->device}, {b->device, a->device}};
  for (auto &p : pairs) {
    CUDA_TRY(cudaSetDevice(p[0]));
    cudaError_t e = cudaDeviceEnablePeerAccess(p[1], 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      cudaGetLastError();
    else if (e != cudaSuccess)
      return fail(SRF_E_PEER_UNREACHABLE, "enable peer %d->%d: %s", p[0], p[1],
                  cudaGetErrorString(e));
  }
  return SRF_OK;
}

int srf_enable_peer(int device, int peer_device) {
  DeviceGuard device_guard;
  if (device == peer_device) return SRF_OK;
  CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SRF_OK;
  }
  if (e != cudaSuccess)
    return fail(SRF_E_PEER_UNREACHABLE, "enable peer %d->%d: %s", device, peer_device,
                cudaGetErrorString(e));
  return SRF_OK;
}

int srf_space_export_fd(srf_space_t sp, int *fd) {
  DeviceGuard device_guard;
  if (!sp->vmm || sp->imported)
    return fail(SRF_E_INVALID_CONFIG, "fd export needs a VMM-allocated local space");
  sp->exported = true;
  if (sp->export_fd < 0) {
    auto exp = drv<PFN_export>("cuMemExportToShareableHandle");
    if (!exp) return fail(SRF_E_DEVICE, "cuMemExportToShareableHandle unavailable");
    int f = -1;
    DRV_TRY(exp(&f, sp->mh, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
            "cuMemExportToShareableHandle");
    sp->export_fd = f;
  }
  *fd = sp->export_fd;
  return SRF_OK;
}

int srf_space_import_fd(int fd, int server_id, int local_device, uint64_t capacity,
                        srf_space_t *out) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(local_device));
  cudaFree(0);
  auto imp = drv<PFN_import>("cuMemImportFromShareableHandle");
  if (!imp) return fail(SRF_E_DEVICE, "cuMemImportFromShareableHandle unavailable");
  srf_space *sp = new srf_space();
  sp->vmm = true;
  sp->imported = true;
  sp->export_fd = -1;
  sp->server_id = server_id;
  sp->device = local_device;
  sp->capacity = capacity;
  sp->max_regions = 1u << 30;
  sp->next_addr = 0;
  sp->err = nullptr;
  size_t g = vmm_granularity(local_device);
  sp->map_size = (capacity + g - 1) / g * g;
  CUresult r = imp(&sp->mh, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    delete sp;
    return fail(SRF_E_DEVICE, "cuMemImportFromShareableHandle (CUresult %d)", (int)r);
  }
  int rc = vmm_map(sp->mh, sp->map_size, local_device, false, &sp->base);
  if (rc == SRF_OK) rc = make_stream(local_device, true, nullptr, &sp->stream);
  if (rc == SRF_OK) {
    cudaError_t e = cudaMalloc(&sp->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(sp->err, 0, sizeof(int), sp->stream->s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(sp->stream->s);
    if (e != cudaSuccess) rc = fail(SRF_E_DEVICE, "proxy: %s", cudaGetErrorString(e));
  }
  if (rc != SRF_OK) {
    delete sp;
    return rc;
  }
  *out = sp;
  return SRF_OK;
}

int srf_space_export(srf_space_t sp, void *handle64) {
  DeviceGuard device_guard;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  if (sp->imported) return fail(SRF_E_INVALID_CONFIG, "cannot re-export a proxy");
  if (sp->vmm) return fail(SRF_E_INVALID_CONFIG, "VMM pools export by fd (srf_space_export_fd)");
  sp->exported = true;
  CUDA_TRY(cudaSetDevice(sp->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, sp->base));
  memcpy(handle64, &h, sizeof h);
  return SRF_OK;
}

int srf_space_import(const void *handle64, int server_id, int local_device,
                     uint64_t capacity, srf_space_t *out) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(local_device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  void *p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  srf_space *sp = new srf_space();
  sp->vmm = false;
  sp->export_fd = -1;
  sp->map_size = 0;
  sp->server_id = server_id;
  sp->device = local_device;  // work on the proxy is issued from this GPU
  sp->capacity = capacity;
  sp->max_regions = 1u << 30;
  sp->base = (uint8_t *)p;
  sp->imported = true;
  sp->next_addr = 0;
  sp->err = nullptr;
  int rc = make_stream(local_device, true, nullptr, &sp->stream);
  if (rc == SRF_OK) {
    cudaError_t e = cudaMalloc(&sp->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(sp->err, 0, sizeof(int), sp->stream->s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(sp->stream->s);
    if (e != cudaSuccess) rc = fail(SRF_E_DEVICE, "proxy: %s", cudaGetErrorString(e));
  }
  if (rc != SRF_OK) {
    cudaIpcCloseMemHandle(p);
    delete sp;
    return rc;
  }
  *out = sp;
  return SRF_OK;
}

int srf_stream_create(srf_space_t sp, srf_stream_t *out) {
  DeviceGuard device_guard;
  return make_stream(sp->device, true, nullptr, out);
}

int srf_stream_destroy(srf_stream_t st) {
  DeviceGuard device_guard;
  free_stream(st);
  return SRF_OK;
}

void *srf_stream_cuda(srf_stream_t st) { return (void *)st->s; }

int srf_stream_sync(srf_stream_t st) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  CUDA_TRY(cudaStreamSynchronize(st->s));
  return SRF_OK;
}

int srf_event_record(srf_space_t sp, srf_stream_t st, srf_event_t *out) {
  DeviceGuard device_guard;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  return record_event(s->device, s->s, out);
}

int srf_event_query(srf_event_t ev) {
  DeviceGuard device_guard;
  cudaError_t e = cudaEventQuery(ev->e);
  if (e == cudaSuccess) return SRF_OK;
  if (e == cudaErrorNotReady) return SRF_PENDING;
  return fail(SRF_E_DEVICE, "event query: %s", cudaGetErrorString(e));
}

int srf_event_wait(srf_event_t ev) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaEventSynchronize(ev->e));
  return SRF_OK;
}

int srf_event_wait_free(srf_event_t ev) {
  DeviceGuard device_guard;
  if (!ev) return SRF_OK;
  cudaError_t e = cudaEventSynchronize(ev->e);
  release_event(ev);
  if (e != cudaSuccess) return fail(SRF_E_DEVICE, "event wait: %s", cudaGetErrorString(e));
  return SRF_OK;
}

int srf_event_free(srf_event_t ev) {
  DeviceGuard device_guard;
  if (!ev) return SRF_OK;
  release_event(ev);  // a pooled completion event is reused by a later verb
  return SRF_OK;
}

static int put_impl(srf_space_t src_space, const uint64_t *src_addr, const uint64_t *src_len,
                    const uint64_t *src_token, int nseg, srf_space_t dst_space,
                    uint64_t dst_addr, uint64_t dst_token, int flags, srf_stream_t st,
                    srf_event_t *ev_out, uint8_t *consume);

int srf_put(srf_space_t src_space, const uint64_t *src_addr,
            const uint64_t *src_len, const uint64_t *src_token, int nseg,
            srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
            int flags, srf_stream_t st, srf_event_t *ev_out) {
  return put_impl(src_space, src_addr, src_len, src_token, nseg, dst_space, dst_addr, dst_token,
                  flags, st, ev_out, nullptr);
}

int srf_put_consume(srf_space_t src_space, const uint64_t *src_addr, const uint64_t *src_len,
                    const uint64_t *src_token, int nseg, srf_space_t dst_space,
                    uint64_t dst_addr, uint64_t dst_token, int flags, srf_space_t rcv_space,
                    uint64_t rcv_flag_addr, srf_stream_t st, srf_event_t *ev_out) {
  DeviceGuard device_guard;
  int rc = check_raw(rcv_space, rcv_flag_addr, 1, "receive flag");
  if (rc) return rc;
  if (rcv_space->imported) return fail(SRF_E_INVALID_CONFIG, "the receive flag is this rank's");
  return put_impl(src_space, src_addr, src_len, src_token, nseg, dst_space, dst_addr, dst_token,
                  flags, st, ev_out, rcv_space->base + rcv_flag_addr);
}

static int put_impl(srf_space_t src_space, const uint64_t *src_addr, const uint64_t *src_len,
                    const uint64_t *src_token, int nseg, srf_space_t dst_space,
                    uint64_t dst_addr, uint64_t dst_token, int flags, srf_stream_t st,
                    srf_event_t *ev_out, uint8_t *consume) {
  DeviceGuard device_guard;
  if (nseg < 1 || nseg > kMaxSeg)
    return fail(SRF_E_INVALID_CONFIG, "gather list of %d segments (max %d)",
                nseg, kMaxSeg);
  uint64_t total = 0;
  for (int i = 0; i < nseg; ++i) total += src_len[i];
  if (total < 1) return fail(SRF_E_INVALID_LENGTH, "zero-length write");
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    for (int i = 0; i < nseg; ++i) {
      int rc = check_registered_locked(src_space, src_addr[i], src_len[i],
                                       src_token[i]);
      if (rc) return rc;
    }
  }
  {
    std::lock_guard<std::mutex> g(dst_space->mu);
    int rc = check_remote_locked(dst_space, dst_addr, total, dst_token);
    if (rc) return rc;
  }
  srf_stream *s = stream_or_default(src_space, st);
  PutArgs a;
  memset(&a, 0, sizeof a);
  uint64_t off = 0;
  int k = 0;
  for (int i = 0; i < nseg; ++i) {
    if (src_len[i] == 0) continue;
    a.seg[k].src = src_space->base + src_addr[i];
    a.seg[k].dst_off = off;
    a.seg[k].len = src_len[i];
    off += src_len[i];
    ++k;
  }
  a.nseg = k;
  a.dst = dst_space->base + dst_addr;
  a.total = total;
  a.tail_release = 1;
  a.sys_scope = (g_force_sys || dst_space->imported || dst_space->device != s->device) ? 1 : 0;
  a.db = nullptr;
  a.db_len = 0;
  if (dst_space->db && !dst_space->imported) {
    std::lock_guard<std::mutex> g(dst_space->mu);
    auto it = dst_space->db->find(dst_addr + total - 1);
    if (it != dst_space->db->end()) {
      Doorbell &d = it->second;
      const uint64_t n = std::min<uint64_t>(total, d.shadow_len);
      a.db = dst_space->db_dev + d.host_off + (d.shadow_len - n);
      a.db_len = (uint32_t)n;
      if (d.clear_pending) {
        // the receiver's clear of the device flag precedes this write
        CUDA_TRY(cudaSetDevice(s->device));
        CUDA_TRY(cudaStreamWaitEvent(s->s, d.clear_ev, 0));
        d.clear_pending = false;
      }
    }
  }
  a.wait_empty = (flags & SRF_PUT_WAIT_EMPTY) ? 1 : 0;
  a.timeout_ns = g_put_timeout_ns;
  a.counter = s->counter;
  a.err = src_space->err;
  a.consume = consume;
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  if (a.sys_scope && g_peer_ce_bytes && total - 1 >= g_peer_ce_bytes && a.db_len <= 1 &&
      !a.wait_empty && !a.consume)
    rc = put_via_copy_engine(a, s);
  else
    rc = launch_copy(a, s, "k_put");
  if (rc) return rc;
  return record_event(s->device, s->s, ev_out);
}

int srf_put_inline(srf_space_t src_space, uint64_t stage_addr, uint64_t stage_token,
                   const void *bytes, uint32_t len, srf_space_t dst_space, uint64_t dst_addr,
                   uint64_t dst_token, int flags, srf_stream_t st, srf_event_t *ev_out) {
  DeviceGuard device_guard;
  if (len < 1) return fail(SRF_E_INVALID_LENGTH, "zero-length write");
  if (len > (uint32_t)kInlineMax)
    return fail(SRF_E_INVALID_CONFIG, "inline block of %u bytes (max %d)", len, kInlineMax);
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    int rc = check_registered_locked(src_space, stage_addr, len, stage_token);
    if (rc) return rc;
  }
  {
    std::lock_guard<std::mutex> g(dst_space->mu);
    int rc = check_remote_locked(dst_space, dst_addr, len, dst_token);
    if (rc) return rc;
  }
  srf_stream *s = stream_or_default(src_space, st);
  InlineArgs a;
  memset(&a, 0, sizeof a);
  memcpy(a.bytes, bytes, len);
  a.len = len;
  a.stage = src_space->base + stage_addr;
  a.dst = dst_space->base + dst_addr;
  a.sys_scope = (g_force_sys || dst_space->imported || dst_space->device != s->device) ? 1 : 0;
  a.wait_empty = (flags & SRF_PUT_WAIT_EMPTY) ? 1 : 0;
  a.timeout_ns = g_put_timeout_ns;
  a.err = src_space->err;
  if (dst_space->db && !dst_space->imported) {
    std::lock_guard<std::mutex> g(dst_space->mu);
    auto it = dst_space->db->find(dst_addr + len - 1);
    if (it != dst_space->db->end()) {
      Doorbell &d = it->second;
      const uint64_t n = std::min<uint64_t>(len, d.shadow_len);
      a.db = dst_space->db_dev + d.host_off + (d.shadow_len - n);
      a.db_len = (uint32_t)n;
      if (d.clear_pending) {
        CUDA_TRY(cudaSetDevice(s->device));
        CUDA_TRY(cudaStreamWaitEvent(s->s, d.clear_ev, 0));
        d.clear_pending = false;
      }
    }
  }
  CUDA_TRY(cudaSetDevice(s->device));
  k_put_inline<<<1, 256, 0, s->s>>>(a);
  if (recording()) rec_inline(a, s->device);
  int rc = launch_check("k_put_inline");
  if (rc) return rc;
  return record_event(s->device, s->s, ev_out);
}

int srf_get(srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
            srf_space_t src_space, uint64_t src_addr, uint64_t src_token,
            uint64_t length, srf_stream_t st, srf_event_t *ev_out) {
  DeviceGuard device_guard;
  if (length < 1) return fail(SRF_E_INVALID_LENGTH, "zero-length read");
  {
    std::lock_guard<std::mutex> g(dst_space->mu);
    int rc = check_registered_locked(dst_space, dst_addr, length, dst_token);
    if (rc) return rc;
  }
  {
    std::lock_guard<std::mutex> g(src_space->mu);
    int rc = check_remote_locked(src_space, src_addr, length, src_token);
    if (rc) return rc;
  }
  srf_stream *s = stream_or_default(dst_space, st);
  PutArgs a;
  memset(&a, 0, sizeof a);
  a.seg[0].src = src_space->base + src_addr;
  a.seg[0].dst_off = 0;
  a.seg[0].len = length;
  a.nseg = 1;
  a.dst = dst_space->base + dst_addr;
  a.total = length;
  a.tail_release = 0;
  const bool cross = g_force_sys || src_space->imported || src_space->device != s->device;
  a.src_remote = cross ? 1 : 0;
  a.counter = s->counter;
  a.err = dst_space->err;
  CUDA_TRY(cudaSetDevice(s->device));
  int rc = SRF_OK;
  if (cross && g_peer_ce_bytes && length >= g_peer_ce_bytes)
    CUDA_TRY(cudaMemcpyAsync(a.dst, a.seg[0].src, length, cudaMemcpyDeviceToDevice, s->s));
  else
    rc = launch_copy(a, s, "k_put(get)");
  if (rc) return rc;
  return record_event(s->device, s->s, ev_out);
}

int srf_copy(srf_space_t sp, uint64_t src_addr, uint64_t dst_addr,
             uint64_t length, srf_stream_t st, srf_event_t *ev_out) {
  DeviceGuard device_guard;
  if (length == 0) return SRF_OK;
  int rc = check_raw(sp, src_addr, length, "copy src");
  if (!rc) rc = check_raw(sp, dst_addr, length, "copy dst");
  if (rc) return rc;
  srf_stream *s = stream_or_default(sp, st);
  PutArgs a;
  memset(&a, 0, sizeof a);
  a.seg[0].src = sp->base + src_addr;
  a.seg[0].len = length;
  a.nseg = 1;
  a.dst = sp->base + dst_addr;
  a.total = length;
  a.counter = s->counter;
  a.err = sp->err;
  CUDA_TRY(cudaSetDevice(s->device));
  rc = launch_copy(a, s, "k_put(copy)");
  if (rc) return rc;
  return record_event(s->device, s->s, ev_out);
}

int srf_flag_wait(srf_space_t sp, uint64_t flag_addr, uint8_t expect,
                  int clear, uint64_t timeout_ns, srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, flag_addr, 1, "flag");
  if (rc) return rc;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  k_flag_wait<<<1, 32, 0, s->s>>>(sp->base + flag_addr, expect, clear,
                                  timeout_ns, sp->err);
  return launch_check("k_flag_wait");
}

int srf_dyn_recv(srf_space_t rcv, uint64_t meta_addr, int rank, srf_space_t peer,
                 uint64_t peer_lo, uint64_t peer_hi, uint64_t peer_token, uint64_t dst_addr,
                 uint64_t dst_cap, uint64_t len_out_addr, srf_stream_t st) {
  DeviceGuard device_guard;
  if (rank < 0 || rank > 64) return fail(SRF_E_INVALID_CONFIG, "rank %d", rank);
  int rc = check_raw(rcv, meta_addr, 8 * (uint64_t)rank + 33, "meta block");
  if (!rc && dst_cap) rc = check_raw(rcv, dst_addr, dst_cap, "receive block");
  if (!rc && len_out_addr != UINT64_MAX) {
    rc = check_raw(rcv, len_out_addr, 8, "length word");
    if (!rc && len_out_addr % 8) rc = fail(SRF_E_INVALID_CONFIG, "length word must be 8-B aligned");
  }
  if (rc) return rc;
  if (peer_hi < peer_lo || peer_hi > peer->capacity)
    return fail(SRF_E_OUT_OF_BOUNDS, "peer region escapes its space");
  srf_stream *s = stream_or_default(rcv, st);
  DynRecvArgs a;
  a.meta = rcv->base + meta_addr;
  a.rank = rank;
  a.peer_base = peer->base;
  a.peer_lo = peer_lo;
  a.peer_hi = peer_hi;
  a.peer_token = peer_token;
  a.dst = rcv->base + dst_addr;
  a.dst_cap = dst_cap;
  a.len_out = len_out_addr == UINT64_MAX ? nullptr : (uint64_t *)(rcv->base + len_out_addr);
  a.counter = s->counter;
  a.timeout_ns = 10ull * 1000 * 1000 * 1000;
  a.err = rcv->err;
  a.sys = (peer->imported || peer->device != s->device) ? 1 : 0;
  int grid, block;
  copy_geometry(s->device, std::max<uint64_t>(dst_cap, 1), &grid, &block);
  CUDA_TRY(cudaSetDevice(s->device));
  k_dyn_recv<<<grid, block, 0, s->s>>>(a);
  return launch_check("k_dyn_recv");
}

int srf_consume_checksum(srf_space_t sp, uint64_t flag_addr, uint64_t data_addr,
                         uint64_t n, uint64_t out_addr, uint64_t timeout_ns,
                         srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, flag_addr, 1, "flag");
  if (!rc) rc = check_raw(sp, data_addr, n, "payload");
  if (!rc) rc = check_raw(sp, out_addr, 8, "checksum");
  if (rc) return rc;
  if (out_addr % 8) return fail(SRF_E_INVALID_CONFIG, "checksum slot must be 8-B aligned");
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  k_consume_sum<<<1, 1024, 0, s->s>>>(sp->base + flag_addr, sp->base + data_addr, n,
                                      (uint64_t *)(sp->base + out_addr), timeout_ns,
                                      sp->err);
  return launch_check("k_consume_sum");
}

int srf_apply(srf_space_t var_space, uint64_t var_addr, uint64_t nbytes,
              srf_space_t const *grad_spaces, const uint64_t *grad_addrs,
              int nworkers, int op, float lr, srf_stream_t st,
              srf_event_t *ev_out) {
  DeviceGuard device_guard;
  if (nworkers < 1 || nworkers > SRF_MAX_WORKERS)
    return fail(SRF_E_INVALID_CONFIG, "nworkers %d outside [1, %d]", nworkers,
                SRF_MAX_WORKERS);
  if (op != SRF_APPLY_XOR && op != SRF_APPLY_SGD)
    return fail(SRF_E_INVALID_CONFIG, "unknown apply op %d", op);
  if (op == SRF_APPLY_SGD && (nbytes % 4 || var_addr % 4))
    return fail(SRF_E_SHAPE_MISMATCH, "SGD needs whole fp32 elements");
  int rc = check_raw(var_space, var_addr, nbytes, "variable");
  if (rc) return rc;
  ApplyArgs a;
  memset(&a, 0, sizeof a);
  a.var = var_space->base + var_addr;
  a.nw = nworkers;
  a.n = nbytes;
  a.lr = lr;
  for (int w = 0; w < nworkers; ++w) {
    rc = check_raw(grad_spaces[w], grad_addrs[w], nbytes, "gradient");
    if (rc) return rc;
    if (op == SRF_APPLY_SGD && grad_addrs[w] % 4)
      return fail(SRF_E_SHAPE_MISMATCH, "SGD gradient not fp32 aligned");
    a.g[w] = grad_spaces[w]->base + grad_addrs[w];
  }
  srf_stream *s = stream_or_default(var_space, st);
  if (nbytes == 0) return record_event(s->device, s->s, ev_out);
  int grid, block;
  copy_geometry(s->device, nbytes, &grid, &block);
  CUDA_TRY(cudaSetDevice(s->device));
  if (op == SRF_APPLY_XOR)
    k_apply_xor<<<grid, block, 0, s->s>>>(a);
  else
    k_apply_sgd<<<grid, block, 0, s->s>>>(a);
  if (recording()) rec_apply(s->device, grid, block, a, op == SRF_APPLY_SGD);
  rc = launch_check("k_apply");
  if (rc) return rc;
  return record_event(s->device, s->s, ev_out);
}

int srf_gen_reference(srf_space_t sp, uint64_t addr, uint64_t nelems, uint64_t elem_offset,
                      uint64_t seed, uint64_t node, uint64_t iteration, srf_stream_t st,
                      srf_event_t *ev_out) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, nelems * 4, "generated tensor");
  if (rc) return rc;
  if (addr % 4) return fail(SRF_E_INVALID_CONFIG, "generated fp32 tensor must be 4-B aligned");
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  if (nelems) {
    const uint64_t want = (nelems * 4 + (128 << 10) - 1) / (128 << 10);
    const uint64_t cap = (uint64_t)sm_count_of(s->device) * 4;
    const int grid = (int)std::max<uint64_t>(1, std::min(want, cap));
    k_gen_reference<<<grid, 512, 0, s->s>>>((float *)(sp->base + addr), nelems, elem_offset,
                                            seed, node, iteration, nullptr);
    if (recording())
      rec_gen(s->device, grid, (float *)(sp->base + addr), nelems, elem_offset, seed, node,
              iteration);
    rc = launch_check("k_gen_reference");
    if (rc) return rc;
  }
  return record_event(s->device, s->s, ev_out);
}

int srf_reduce_max_f32(srf_space_t sp, uint64_t in_addr, uint64_t n,
                       uint64_t out_addr, srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, in_addr, n * 4, "reduce input");
  if (!rc) rc = check_raw(sp, out_addr, 4, "reduce output");
  if (rc) return rc;
  srf_stream *s = stream_or_default(sp, st);
  uint64_t want = (n + 256 * 64 - 1) / (256 * 64);
  uint64_t cap = std::min<uint64_t>((uint64_t)sm_count_of(s->device) * 6, kScratchBlocks);
  int grid = (int)std::max<uint64_t>(1, std::min(want, cap));
  CUDA_TRY(cudaSetDevice(s->device));
  k_reduce_max<<<grid, 256, 0, s->s>>>((const float *)(sp->base + in_addr), n,
                                       (float *)(sp->base + out_addr),
                                       s->scratch, s->counter + 1);
  if (recording())
    rec_reduce(s->device, grid, (const float *)(sp->base + in_addr), n,
               (float *)(sp->base + out_addr), s->scratch, s->counter + 1);
  return launch_check("k_reduce_max");
}

}  // extern "C"
