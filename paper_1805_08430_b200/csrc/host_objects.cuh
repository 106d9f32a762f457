// host_objects.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Error plumbing, host-side objects (spaces, regions, streams, events), CUDA VMM pools.

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                        \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess)                                                    \
      return fail(SRF_E_DEVICE, "%s: %s (%s:%d)", #expr,                      \
                  cudaGetErrorString(_e), __FILE__, __LINE__);                \
  } while (0)

// ---------------------------------------------------------------------------
// host-side objects
// ---------------------------------------------------------------------------
struct Region {
  int64_t id;
  uint64_t base, length;
  bool registered;
  uint64_t token;
};

struct srf_stream {
  int device;
  cudaStream_t s;
  bool owned;
  unsigned int *counter;  // grid arrival counter for tail-release kernels
  float *scratch;         // per-block partials for reductions
};

struct srf_space {
  bool vmm;                        // allocated with cuMemCreate (VMM) instead of cudaMalloc
  CUmemGenericAllocationHandle mh; // VMM allocation (own or imported)
  size_t map_size;
  int export_fd;                   // POSIX fd of the exported VMM allocation (-1: none)
  int server_id;
  int device;
  uint64_t capacity;
  uint32_t max_regions;
  uint8_t *base;       // device pointer (own cudaMalloc or IPC mapping)
  bool imported;       // remote proxy mapped through cudaIpcOpenMemHandle
  std::mutex mu;       // region table, next_addr
  std::vector<Region> regions;
  uint64_t next_addr;
  srf_stream *stream;  // default stream (local work + byte IO)
  int *err;            // device error word (flag-wait timeouts)
  // host-visible doorbells: pinned, mapped shadows of receive
  // flags / metadata blocks that K1/K3 update next to the device bytes
  uint8_t *db_host = nullptr;   // pinned host page(s)
  uint8_t *db_dev = nullptr;    // the same memory, device address
  uint64_t db_cap = 0, db_used = 0;
  bool exported = false;        // producers may live in other processes
  std::unordered_map<uint64_t, struct Doorbell> *db = nullptr;  // tail addr -> entry
};

struct Doorbell {
  uint64_t region_addr, region_len;  // shadowed device bytes
  uint64_t host_off;                 // offset of the shadow in db_host
  uint64_t shadow_len;               // last shadow_len bytes of the region (flag last)
  bool mirror;                       // whole region (metadata) or only the tail flag
  cudaEvent_t clear_ev;              // receiver's device-flag clear
  bool clear_pending;
};

struct srf_event {
  int device;
  cudaEvent_t e;
  bool pooled = false;  // a completion event from the per-device pool (no timing)
};

static constexpr uint64_t kAlign = 8;  // memspace.py:31 (_ALIGN)
static constexpr int kMaxSeg = 8;
static constexpr int kScratchBlocks = 1024;

// launch-geometry knobs (srf_tune): CTAs per SM and threads per CTA of the
// copy kernels.  Large puts: one 512-thread CTA per SM - the same threads as
// 2 x 256 and the same 256 MiB HBM put (0.924 of the copy peak), but half the
// CTAs that each poll the credit and arrive on the counter: NVLink puts of 4 /
// 16 MiB per round 20.3 -> 16.5 / 40.3 -> 36.2 us (A/B on one box,
// profiles/r1_geometry_probe.txt); small puts keep one CTA per 16 KiB.
static int g_ctas_per_sm = 1;
static int g_copy_threads = 512;

static int sm_count_of(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) !=
            cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

static int make_stream(int device, bool create, cudaStream_t existing,
                       srf_stream **out) {
  CUDA_TRY(cudaSetDevice(device));
  srf_stream *st = new srf_stream();
  st->device = device;
  st->owned = create;
  if (create) {
    cudaError_t e = cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete st;
      return fail(SRF_E_DEVICE, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
  } else {
    st->s = existing;
  }
  cudaError_t e = cudaMalloc(&st->counter, sizeof(unsigned int) + 16);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->counter, 0, sizeof(unsigned int) + 16, st->s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st->s);
  if (e == cudaSuccess) e = cudaMalloc(&st->scratch, sizeof(float) * kScratchBlocks);
  if (e != cudaSuccess) {
    if (create) cudaStreamDestroy(st->s);
    delete st;
    return fail(SRF_E_DEVICE, "stream scratch: %s", cudaGetErrorString(e));
  }
  *out = st;
  return SRF_OK;
}

static void free_stream(srf_stream *st) {
  if (!st) return;
  cudaSetDevice(st->device);
  cudaStreamSynchronize(st->s);
  cudaFree(st->counter);
  cudaFree(st->scratch);
  if (st->owned) cudaStreamDestroy(st->s);
  delete st;
}

static srf_stream *stream_or_default(srf_space *sp, srf_stream *st) {
  return st ? st : sp->stream;
}

// memspace.py:139-143 (_find_registered): linear scan, first containing
// registered region.
static const Region *find_registered(const srf_space *sp, uint64_t addr,
                                     uint64_t len) {
  for (const Region &r : sp->regions)
    if (r.registered && r.base <= addr && addr + len <= r.base + r.length)
      return &r;
  return nullptr;
}

static int check_remote_locked(srf_space *sp, uint64_t addr, uint64_t len,
                               uint64_t token) {
  const Region *r = find_registered(sp, addr, len);
  if (!r)
    return fail(SRF_E_REMOTE_OOB,
                "server %d: [%llu, %llu) is not inside a registered region",
                sp->server_id, (unsigned long long)addr,
                (unsigned long long)(addr + len));
  if (r->token != token)
    return fail(SRF_E_BAD_TOKEN, "server %d: token mismatch for region %lld",
                sp->server_id, (long long)r->id);
  return SRF_OK;
}

static int check_registered_locked(srf_space *sp, uint64_t addr, uint64_t len,
                                   uint64_t token) {
  const Region *r = find_registered(sp, addr, len);
  if (!r || r->token != token)
    return fail(SRF_E_NOT_REGISTERED,
                "server %d: [%llu, %llu) is not registered", sp->server_id,
                (unsigned long long)addr, (unsigned long long)(addr + len));
  return SRF_OK;
}

static int check_raw(const srf_space *sp, uint64_t addr, uint64_t len,
                     const char *what) {
  if (addr > sp->capacity || len > sp->capacity - addr)
    return fail(SRF_E_OUT_OF_BOUNDS, "%s [%llu, %llu) escapes space of %llu",
                what, (unsigned long long)addr,
                (unsigned long long)(addr + len),
                (unsigned long long)sp->capacity);
  return SRF_OK;
}


// ---------------------------------------------------------------------------
// CUDA VMM pools (cuMemCreate + POSIX-fd export), the alternative to CUDA IPC
// handles the multi-process path can select (SRFLOW_ALLOC_VMM=1; both measure
// the same over NVLink).  Driver entry points are resolved at run time
// through cudaGetDriverEntryPoint, so no libcuda link is needed.
// ---------------------------------------------------------------------------
static int g_alloc_vmm = 0;

template <typename F>
static F drv(const char *name) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (F)p;
}

#define DRV_TRY(expr, what)                                                   \
  do {                                                                        \
    CUresult _r = (expr);                                                     \
    if (_r != CUDA_SUCCESS)                                                   \
      return fail(SRF_E_DEVICE, "%s failed (CUresult %d)", what, (int)_r);     \
  } while (0)

typedef CUresult (*PFN_memCreate)(CUmemGenericAllocationHandle *, size_t,
                                  const CUmemAllocationProp *, unsigned long long);
typedef CUresult (*PFN_memGran)(size_t *, const CUmemAllocationProp *,
                                CUmemAllocationGranularity_flags);
typedef CUresult (*PFN_addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr,
                                    unsigned long long);
typedef CUresult (*PFN_memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                               unsigned long long);
typedef CUresult (*PFN_setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
typedef CUresult (*PFN_export)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                               unsigned long long);
typedef CUresult (*PFN_import)(CUmemGenericAllocationHandle *, void *,
                               CUmemAllocationHandleType);
typedef CUresult (*PFN_unmap)(CUdeviceptr, size_t);
typedef CUresult (*PFN_release)(CUmemGenericAllocationHandle);
typedef CUresult (*PFN_addrFree)(CUdeviceptr, size_t);

static size_t vmm_granularity(int device) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 2 << 20;
  auto gran = drv<PFN_memGran>("cuMemGetAllocationGranularity");
  if (gran) gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  return g;
}

// map `h` (size bytes) at a fresh VA and grant `local` (+ every peer that
// can reach it when all_peers) read/write access
static int vmm_map(CUmemGenericAllocationHandle h, size_t size, int local, bool all_peers,
                   uint8_t **out) {
  auto reserve = drv<PFN_addrReserve>("cuMemAddressReserve");
  auto map = drv<PFN_memMap>("cuMemMap");
  auto access = drv<PFN_setAccess>("cuMemSetAccess");
  if (!reserve || !map || !access) return fail(SRF_E_DEVICE, "VMM entry points missing");
  CUdeviceptr va = 0;
  DRV_TRY(reserve(&va, size, 2 << 20, 0, 0), "cuMemAddressReserve");
  DRV_TRY(map(va, size, 0, h, 0), "cuMemMap");
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  std::vector<CUmemAccessDesc> acc;
  for (int d = 0; d < ndev; ++d) {
    int ok = (d == local);
    if (!ok && all_peers) cudaDeviceCanAccessPeer(&ok, d, local);
    if (!ok) continue;
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = d;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc.push_back(a);
  }
  DRV_TRY(access(va, size, acc.data(), acc.size()), "cuMemSetAccess");
  *out = (uint8_t *)va;
  return SRF_OK;
}

static int vmm_alloc(srf_space *sp) {
  auto create = drv<PFN_memCreate>("cuMemCreate");
  if (!create) return fail(SRF_E_DEVICE, "cuMemCreate unavailable");
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = sp->device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = vmm_granularity(sp->device);
  sp->map_size = (sp->capacity + g - 1) / g * g;
  DRV_TRY(create(&sp->mh, sp->map_size, &prop, 0), "cuMemCreate");
  return vmm_map(sp->mh, sp->map_size, sp->device, true, &sp->base);
}

static void vmm_free(srf_space *sp) {
  auto unmap = drv<PFN_unmap>("cuMemUnmap");
  auto release = drv<PFN_release>("cuMemRelease");
  auto afree = drv<PFN_addrFree>("cuMemAddressFree");
  if (unmap) unmap((CUdeviceptr)sp->base, sp->map_size);
  if (afree) afree((CUdeviceptr)sp->base, sp->map_size);
  if (release) release(sp->mh);
  if (sp->export_fd >= 0) close(sp->export_fd);
}
