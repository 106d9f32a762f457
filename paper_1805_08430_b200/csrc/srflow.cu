// srflow.cu - libsrflow.so: the B200-native (sm_100a) transfer hot path.
//
// Host half: per-server HBM pools with the reference's region table, token
// and bounds gates (memspace.py:89-236), streams/events standing in for queue
// pairs and completion queues (fabric.py:113-143, :423-428), and the verb
// entry points (fabric.py:349-389).  Device half: the kernels K1..K6 of
// SURVEY.md section 2.2.  The reference moves bytes with a Python loop of
// 1-4096 B ascending chunks (fabric.py:391-421); here every byte moves through
// 16-byte vector loads/stores issued by all SMs, and the "final byte lands
// last" guarantee is rebuilt from a system-scope fence, a grid arrival count
// and one st.release.sys of the tail byte.
//
// Declarations and reference citations: include/srflow.h.

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/srflow.h"

namespace cg = cooperative_groups;

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
};

static constexpr uint64_t kAlign = 8;  // memspace.py:31 (_ALIGN)
static constexpr int kMaxSeg = 8;
static constexpr int kScratchBlocks = 1024;

// launch-geometry knobs (srf_tune): CTAs per SM and threads per CTA of the
// copy kernels; defaults chosen from the NVLink/HBM probes (profiles/).
static int g_ctas_per_sm = 2;
static int g_copy_threads = 256;

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
// CUDA VMM pools (cuMemCreate + POSIX-fd export).  Cross-process SM stores
// through cudaIpcOpenMemHandle mappings measured ~500 GB/s vs ~690 GB/s
// in-process (profiles/); VMM mappings are the alternative the multi-process
// path can select (SRFLOW_ALLOC=vmm).  Driver entry points are resolved at
// run time through cudaGetDriverEntryPoint, so no libcuda link is needed.
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

// ---------------------------------------------------------------------------
// device helpers (inline PTX: system-scope acquire/release on peer memory)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys_u8(const uint8_t *p) {
  uint16_t v;
  asm volatile("ld.acquire.sys.global.u8 %0, [%1];"
               : "=h"(v)
               : "l"(p)
               : "memory");
  return v & 0xff;
}

__device__ __forceinline__ void st_release_sys_u8(uint8_t *p, uint32_t v) {
  uint16_t x = (uint16_t)v;
  asm volatile("st.release.sys.global.u8 [%0], %1;" ::"l"(p), "h"(x)
               : "memory");
}

__device__ __forceinline__ void st_relaxed_sys_u8(uint8_t *p, uint32_t v) {
  uint16_t x = (uint16_t)v;
  asm volatile("st.relaxed.sys.global.u8 [%0], %1;" ::"l"(p), "h"(x)
               : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


// Grid arrival for the flag-last release.  Every CTA's threads finish their
// stores; bar.sync orders them before thread 0, whose acq_rel RMW on the
// arrival counter is cumulative at the chosen scope (gpu when the destination
// is this GPU's own HBM, sys when it is a peer's).  The CTA that observes
// count-1 then owns the release store of the tail byte.
__device__ __forceinline__ bool grid_arrive(unsigned int *counter, unsigned expected_last,
                                            int sys_scope) {
  unsigned prev;
  if (sys_scope)
    asm volatile("atom.add.acq_rel.sys.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
  else
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
  return prev == expected_last;
}

__device__ __forceinline__ void release_tail(uint8_t *p, uint32_t v, int sys_scope) {
  uint16_t x = (uint16_t)v;
  if (sys_scope)
    asm volatile("st.release.sys.global.u8 [%0], %1;" ::"l"(p), "h"(x) : "memory");
  else
    asm volatile("st.release.gpu.global.u8 [%0], %1;" ::"l"(p), "h"(x) : "memory");
}

// 16-byte streaming load, no L1 allocation (source is read exactly once)
__device__ __forceinline__ uint4 ld_stream_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(uint4 *p, const uint4 &v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 32-B vectors: sm_100 has 256-bit global loads/stores (LDG/STG.E.ENL2.256)
struct __align__(32) u256 {
  uint32_t v[8];
};

__device__ __forceinline__ u256 ld_v8(const u256 *p) {
  u256 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                 "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7])
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v8(u256 *p, const u256 &r) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.v[0]),
               "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]),
               "r"(r.v[7])
               : "memory");
}

template <typename V>
__device__ __forceinline__ V ld_stream(const V *p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ u256 ld_stream<u256>(const u256 *p) {
  return ld_v8(p);
}
template <>
__device__ __forceinline__ uint4 ld_stream<uint4>(const uint4 *p) {
  return ld_stream_v4(p);
}
template <typename V>
__device__ __forceinline__ void st_plain(V *p, const V &v) {
  *p = v;
}
template <>
__device__ __forceinline__ void st_plain<uint4>(uint4 *p, const uint4 &v) {
  st_v4(p, v);
}
template <>
__device__ __forceinline__ void st_plain<u256>(u256 *p, const u256 &v) {
  st_v8(p, v);
}

// Grid-wide copy of nv vectors: all loads of an unrolled batch are issued
// before its stores so every thread keeps U requests in flight (the latency of
// a peer access is ~2000 cycles, B300_MICROARCH.md "NVLink").
template <typename V, int U>
__device__ __forceinline__ void vec_copy(V *__restrict__ dst,
                                         const V *__restrict__ src,
                                         uint64_t nv, uint64_t t,
                                         uint64_t nth) {
  uint64_t i = t;
  for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_stream<V>(src + i + u * nth);
#pragma unroll
    for (int u = 0; u < U; ++u) st_plain<V>(dst + i + u * nth, r[u]);
  }
  for (; i < nv; i += nth) st_plain<V>(dst + i, ld_stream<V>(src + i));
}

// Copy n bytes with the widest vector both pointers allow.  Arena blocks are
// 8-byte aligned (memspace.py:31), so the 16-B path needs equal (p mod 16).
__constant__ int g_vec32 = 1;  // knob 5: 32-B vectors when co-aligned mod 32

template <int U16 = 4>
__device__ void copy_bytes_grid(uint8_t *dst, const uint8_t *src, uint64_t n,
                                uint64_t t, uint64_t nth) {
  if (n == 0) return;
  uintptr_t d = (uintptr_t)dst, s = (uintptr_t)src;
  uint64_t head, nv;
  if (g_vec32 && ((d ^ s) & 31) == 0 && n >= 4096) {
    head = (32 - (d & 31)) & 31;
    if (head > n) head = n;
    nv = (n - head) / 32;
    vec_copy<u256, (U16 > 4 ? U16 / 2 : 2)>((u256 *)(dst + head), (const u256 *)(src + head),
                                            nv, t, nth);
    nv *= 32;
  } else if (((d ^ s) & 15) == 0) {
    head = (16 - (d & 15)) & 15;
    if (head > n) head = n;
    nv = (n - head) / 16;
    vec_copy<uint4, U16>((uint4 *)(dst + head), (const uint4 *)(src + head), nv,
                         t, nth);
    nv *= 16;
  } else if (((d ^ s) & 7) == 0) {
    head = (8 - (d & 7)) & 7;
    if (head > n) head = n;
    nv = (n - head) / 8;
    vec_copy<uint2, 8>((uint2 *)(dst + head), (const uint2 *)(src + head), nv,
                       t, nth);
    nv *= 8;
  } else if (((d ^ s) & 3) == 0) {
    head = (4 - (d & 3)) & 3;
    if (head > n) head = n;
    nv = (n - head) / 4;
    vec_copy<uint32_t, 8>((uint32_t *)(dst + head),
                          (const uint32_t *)(src + head), nv, t, nth);
    nv *= 4;
  } else {
    // no common 4-B alignment (e.g. payload behind a 41-B metadata prefix):
    // aligned 4-B destination words assembled from two aligned source words
    // with a funnel shift, so loads and stores stay word-wide and coalesced
    head = (4 - (d & 3)) & 3;
    if (head > n) head = n;
    const uint64_t words = (n - head) / 4;
    // word j reads source words at floor((s+head)/4)+j and +1; the last one
    // may extend up to 3 bytes past the range, so keep one word for the tail
    nv = words > 0 ? words - 1 : 0;
    const uint8_t *sp = src + head;
    const uint32_t m = (uint32_t)((uintptr_t)sp & 3);
    const uint32_t *sw = (const uint32_t *)((uintptr_t)sp - m);
    uint32_t *dw = (uint32_t *)(dst + head);
    uint64_t j = t;
    for (; j + 3 * nth < nv; j += 4 * nth) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = __ldg(sw + j + u * nth);
        b[u] = __ldg(sw + j + u * nth + 1);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dw[j + u * nth] = __funnelshift_r(a[u], b[u], 8 * m);
    }
    for (; j < nv; j += nth) dw[j] = __funnelshift_r(__ldg(sw + j), __ldg(sw + j + 1), 8 * m);
    nv *= 4;
  }
  // scalar head and tail bytes
  for (uint64_t i = t; i < head; i += nth) dst[i] = src[i];
  for (uint64_t i = head + nv + t; i < n; i += nth) dst[i] = src[i];
}

struct Seg {
  const uint8_t *src;
  uint64_t dst_off;
  uint64_t len;
};

struct PutArgs {
  Seg seg[kMaxSeg];
  int nseg;
  uint8_t *dst;          // destination base (peer or local device pointer)
  uint64_t total;        // bytes in the gather list
  int tail_release;      // 1: last byte written last with st.release.sys
  int wait_empty;        // 1: spin until dst[total-1] == 0 before writing
  int sys_scope;         // 1: destination is a peer's memory (system-scope release)
  uint8_t *db;           // host-mapped doorbell shadow (nullptr: none)
  uint32_t db_len;       // bytes mirrored (1: tail flag only; total: whole block)
  uint64_t timeout_ns;
  unsigned int *counter; // arrival counter (per stream, reset by last CTA)
  int *err;
};

// K1 static_put / K3 meta_put / K4 peer_pull / K5 stage_copy.
template <int U16>
__global__ void __launch_bounds__(512) k_put(PutArgs a) {
  __shared__ int s_last;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t *tail = a.dst + a.total - 1;

  if (a.wait_empty) {
    // credit check of the iteration barrier (runtime/protocol.py:102-111):
    // the receiver must have cleared the previous transfer's flag.
    if (threadIdx.x == 0) {
      uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u8(tail) != 0) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
  }

  // body: every byte except the tail one when tail_release is set
  uint64_t body = a.tail_release ? a.total - 1 : a.total;
  for (int i = 0; i < a.nseg; ++i) {
    const Seg &sg = a.seg[i];
    if (sg.dst_off >= body) break;
    uint64_t n = sg.len;
    if (sg.dst_off + n > body) n = body - sg.dst_off;
    copy_bytes_grid<U16>(a.dst + sg.dst_off, sg.src, n, t, nth);
  }

  if (!a.tail_release) return;
  // flag-last: all CTAs publish, the last to arrive releases the tail byte.
  __syncthreads();
  if (threadIdx.x == 0) s_last = grid_arrive(a.counter, gridDim.x - 1, a.sys_scope);
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    const Seg &ls = a.seg[a.nseg - 1];
    const uint32_t v = ls.src[ls.len - 1];
    release_tail(tail, v, a.sys_scope);
    if (a.db) {
      // host doorbell: mirror the block (metadata) and then its flag, release
      // at system scope so a host load that sees the flag sees the block
      for (uint32_t i = 0; i + 1 < a.db_len; ++i) {
        const uint64_t off = a.total - a.db_len + i;
        uint64_t acc = 0;
        const uint8_t *b = nullptr;
        for (int k = 0; k < a.nseg; ++k) {
          if (off < acc + a.seg[k].len) { b = a.seg[k].src + (off - acc); break; }
          acc += a.seg[k].len;
        }
        a.db[i] = b ? *b : 0;
      }
      __threadfence_system();
      st_release_sys_u8(a.db + a.db_len - 1, v);
    }
    atomicExch(a.counter, 0u);
  }
}


// ---------------------------------------------------------------------------
// TMA bulk-copy variant of K1/K4 (cp.async.bulk): one elected thread per CTA
// streams 16 KB chunks global -> shared (mbarrier complete_tx) -> global
// (bulk_group), kBulkStages chunks in flight.  Used for large 16-B co-aligned
// segments; everything else takes the vector path.
// ---------------------------------------------------------------------------
static constexpr int kBulkChunk = 16384;
static constexpr int kBulkStages = 6;
static constexpr int kBulkSmem = kBulkChunk * kBulkStages + 64;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *smem, const void *gsrc,
                                         uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
      "[%1], %2, [%3];" ::"r"(smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *gdst, const void *smem,
                                         uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   gdst),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Thread 0 of every CTA: chunks blockIdx.x, +gridDim.x, ... of [src, src+n),
// n a multiple of 16, both pointers 16-B aligned.
__device__ void bulk_copy_cta(uint8_t *dst, const uint8_t *src, uint64_t n,
                              uint8_t *stage, uint64_t *bars, uint32_t &use) {
  const uint64_t nchunks = (n + kBulkChunk - 1) / kBulkChunk;
  const uint64_t first = blockIdx.x, step = gridDim.x;
  if (first >= nchunks) return;
  const uint64_t mine = (nchunks - first + step - 1) / step;
  auto chunk_of = [&](uint64_t k) { return first + k * step; };
  auto bytes_of = [&](uint64_t c) {
    uint64_t off = c * kBulkChunk;
    return (uint32_t)((n - off) < (uint64_t)kBulkChunk ? (n - off) : kBulkChunk);
  };
  // prologue: fill all stages
  const uint64_t pre = mine < (uint64_t)kBulkStages ? mine : kBulkStages;
  for (uint64_t k = 0; k < pre; ++k) {
    uint64_t c = chunk_of(k);
    int slot = (int)(k % kBulkStages);
    mbar_expect_tx(&bars[slot], bytes_of(c));
    bulk_g2s(stage + slot * kBulkChunk, src + c * kBulkChunk, bytes_of(c), &bars[slot]);
  }
  for (uint64_t k = 0; k < mine; ++k) {
    uint64_t c = chunk_of(k);
    int slot = (int)(k % kBulkStages);
    uint32_t parity = (uint32_t)((use + k / kBulkStages) & 1);
    mbar_wait(&bars[slot], parity);
    bulk_s2g(dst + c * kBulkChunk, stage + slot * kBulkChunk, bytes_of(c));
    // refill the slot of chunk k-1 once its store has read shared memory
    if (k >= 1 && k - 1 + kBulkStages < mine) {
      bulk_wait_read<1>();
      uint64_t kk = k - 1 + kBulkStages;
      uint64_t cc = chunk_of(kk);
      int s2 = (int)(kk % kBulkStages);
      mbar_expect_tx(&bars[s2], bytes_of(cc));
      bulk_g2s(stage + s2 * kBulkChunk, src + cc * kBulkChunk, bytes_of(cc), &bars[s2]);
    }
  }
  bulk_wait_all();
  // each barrier completed ceil-or-floor(mine / stages) phases; track per slot
  // parity by the total number of uses (all slots advance together except
  // the tail: keep slot phases in sync by counting uses per slot)
  use += (uint32_t)((mine + kBulkStages - 1) / kBulkStages);
}

__global__ void __launch_bounds__(256) k_put_bulk(PutArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int s_last;
  uint64_t *bars = (uint64_t *)(smem + kBulkChunk * kBulkStages);
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t *tail = a.dst + a.total - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (a.wait_empty) {
    if (threadIdx.x == 0) {
      uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u8(tail) != 0) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 2);
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
  }
  uint64_t body = a.tail_release ? a.total - 1 : a.total;
  uint32_t use = 0;  // uses per barrier so far (same for every slot: see below)
  for (int i = 0; i < a.nseg; ++i) {
    const Seg &sg = a.seg[i];
    if (sg.dst_off >= body) break;
    uint64_t n = sg.len;
    if (sg.dst_off + n > body) n = body - sg.dst_off;
    uint8_t *d = a.dst + sg.dst_off;
    const uint8_t *s = sg.src;
    uintptr_t dp = (uintptr_t)d, sp = (uintptr_t)s;
    if (n >= (uint64_t)4 * kBulkChunk && ((dp ^ sp) & 15) == 0) {
      uint64_t head = (16 - (dp & 15)) & 15;
      uint64_t mid = ((n - head) / 16) * 16;
      for (uint64_t j = t; j < head; j += nth) d[j] = s[j];
      for (uint64_t j = head + mid + t; j < n; j += nth) d[j] = s[j];
      if (threadIdx.x == 0) {
        // barriers are reused across segments: realign every slot's phase by
        // running complete rounds only (mine is rounded inside), so track use
        bulk_copy_cta(d + head, s + head, mid, smem, bars, use);
      }
      __syncthreads();
      // re-initialise the barriers for the next segment (phases may differ
      // between slots after a partial round)
      if (threadIdx.x == 0) {
        for (int b = 0; b < kBulkStages; ++b) {
          asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[b])));
          mbar_init(&bars[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        use = 0;
      }
      __syncthreads();
    } else {
      copy_bytes_grid(d, s, n, t, nth);
    }
  }
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (!a.tail_release) return;
  __syncthreads();
  if (threadIdx.x == 0) s_last = grid_arrive(a.counter, gridDim.x - 1, a.sys_scope);
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    const Seg &ls = a.seg[a.nseg - 1];
    const uint32_t v = ls.src[ls.len - 1];
    release_tail(tail, v, a.sys_scope);
    if (a.db) {
      // host doorbell: mirror the block (metadata) and then its flag, release
      // at system scope so a host load that sees the flag sees the block
      for (uint32_t i = 0; i + 1 < a.db_len; ++i) {
        const uint64_t off = a.total - a.db_len + i;
        uint64_t acc = 0;
        const uint8_t *b = nullptr;
        for (int k = 0; k < a.nseg; ++k) {
          if (off < acc + a.seg[k].len) { b = a.seg[k].src + (off - acc); break; }
          acc += a.seg[k].len;
        }
        a.db[i] = b ? *b : 0;
      }
      __threadfence_system();
      st_release_sys_u8(a.db + a.db_len - 1, v);
    }
    atomicExch(a.counter, 0u);
  }
}

// Pool zero-fill with plain SM stores.  cudaMemsetAsync(0) on a fresh
// multi-GiB cudaMalloc pool left it in a state where later peer (NVLink)
// stores from another GPU were partly not visible to local reads (~1.3 % of
// the bytes of a > 2 GiB put, reproducible; tests/test_gpu_kernels.py
// ::test_transfers_beyond_4gib_indexing); writing real zeros from the SMs
// avoids it.
__global__ void __launch_bounds__(256) k_zero_fill(uint8_t *p, uint64_t n) {
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t head = ((16 - ((uintptr_t)p & 15)) & 15) < n ? ((16 - ((uintptr_t)p & 15)) & 15) : n;
  const uint64_t nv = (n - head) / 16;
  uint4 *v = (uint4 *)(p + head);
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (uint64_t i = t; i < nv; i += nth) v[i] = z;
  for (uint64_t i = t; i < head; i += nth) p[i] = 0;
  for (uint64_t i = head + nv * 16 + t; i < n; i += nth) p[i] = 0;
}

// K2 flag_wait: device-side consumer prologue of StaticReceiver.poll.
__global__ void k_flag_wait(uint8_t *flag, uint32_t expect, int clear,
                            uint64_t timeout_ns, int *err) {
  if (threadIdx.x != 0) return;
  uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys_u8(flag) != expect) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return;
    }
    __nanosleep(32);
  }
  if (clear) st_relaxed_sys_u8(flag, 0);
}


// Device consumer for release/acquire checks: thread 0 acquire-spins on the
// flag, the CTA then checksums the payload it guards and clears the flag.
__global__ void __launch_bounds__(1024) k_consume_sum(uint8_t *flag,
                                                      const uint8_t *data,
                                                      uint64_t n, uint64_t *out,
                                                      uint64_t timeout_ns,
                                                      int *err) {
  __shared__ unsigned long long acc;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    acc = 0;
    ok = 1;
    uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys_u8(flag) != 1) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicExch(err, 1);
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  if (!ok) return;
  unsigned long long s = 0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) s += data[i] * (i % 251 + 1);
  atomicAdd(&acc, s);
  __syncthreads();
  if (threadIdx.x == 0) {
    *out = acc;
    st_relaxed_sys_u8(flag, 0);
  }
}

// K6 ps_apply
struct ApplyArgs {
  uint8_t *var;
  const uint8_t *g[SRF_MAX_WORKERS];
  int nw;
  uint64_t n;  // bytes
  float lr;
};

// plain (coherent) 16-B load: gradients may be peer memory
__device__ __forceinline__ uint4 ld_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float sgd1(float v, float lr, float g) {
  return __fsub_rn(v, __fmul_rn(lr, g));
}

// One element group of the update: XOR (bytewise, any alignment class) or
// SGD (fp32).  `g` points at an array of nw gradient base pointers (shared
// memory in the batch kernel, grid-constant parameters in K6) - indexing it
// never spills a pointer array to local memory.
struct XorOp {
  __device__ static uint4 fold(uint4 a, uint4 b, float) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
  }
  __device__ static uint2 fold2(uint2 a, uint2 b, float) { return make_uint2(a.x ^ b.x, a.y ^ b.y); }
};
struct SgdOp {
  __device__ static uint4 fold(uint4 a, uint4 b, float lr) {
    return make_uint4(__float_as_uint(sgd1(__uint_as_float(a.x), lr, __uint_as_float(b.x))),
                      __float_as_uint(sgd1(__uint_as_float(a.y), lr, __uint_as_float(b.y))),
                      __float_as_uint(sgd1(__uint_as_float(a.z), lr, __uint_as_float(b.z))),
                      __float_as_uint(sgd1(__uint_as_float(a.w), lr, __uint_as_float(b.w))));
  }
  __device__ static uint2 fold2(uint2 a, uint2 b, float lr) {
    return make_uint2(__float_as_uint(sgd1(__uint_as_float(a.x), lr, __uint_as_float(b.x))),
                      __float_as_uint(sgd1(__uint_as_float(a.y), lr, __uint_as_float(b.y))));
  }
};

// 16-B vectors [0, nv) at byte offset off, U vectors in flight per thread,
// workers folded in ascending order.
template <class Op, int U>
__device__ __forceinline__ void fold_v4(uint8_t *varb, const uint8_t *const *g, int nw,
                                        uint64_t off, uint64_t nv, uint64_t t, uint64_t nth,
                                        float lr) {
  uint4 *var = (uint4 *)(varb + off);
  uint64_t i = t;
  for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
    uint4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = var[i + u * nth];
    for (int w = 0; w < nw; ++w) {
      const uint4 *gw = (const uint4 *)(g[w] + off);
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = ld_v4(gw + i + u * nth);
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = Op::fold(acc[u], r[u], lr);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) var[i + u * nth] = acc[u];
  }
  for (; i < nv; i += nth) {
    uint4 acc = var[i];
    for (int w = 0; w < nw; ++w) acc = Op::fold(acc, ld_v4((const uint4 *)(g[w] + off) + i), lr);
    var[i] = acc;
  }
}

template <class Op>
__device__ __forceinline__ void fold_v2(uint8_t *varb, const uint8_t *const *g, int nw,
                                        uint64_t off, uint64_t nv, uint64_t t, uint64_t nth,
                                        float lr) {
  uint2 *var = (uint2 *)(varb + off);
  for (uint64_t i = t; i < nv; i += nth) {
    uint2 acc = var[i];
    for (int w = 0; w < nw; ++w) acc = Op::fold2(acc, ((const uint2 *)(g[w] + off))[i], lr);
    var[i] = acc;
  }
}

// The whole update of one variable over threads [t, +nth) of some grid.
// XOR works on bytes: 16-B vectors when every pointer shares (p mod 16), 8-B
// when they share (p mod 8) (arena blocks are 8-B aligned), bytes otherwise.
// SGD works on fp32: same vector classes in whole floats.
template <bool SGD>
__device__ void apply_range(uint8_t *var, const uint8_t *const *g, int nw, uint64_t n,
                            float lr, uint64_t t, uint64_t nth) {
  const uintptr_t m = (uintptr_t)var;
  bool same16 = true, same8 = true;
  for (int w = 0; w < nw; ++w) {
    const uintptr_t p = (uintptr_t)g[w];
    same16 &= ((p ^ m) & 15) == 0;
    same8 &= ((p ^ m) & 7) == 0;
  }
  const uint64_t unit = SGD ? 4 : 1;  // scalar element size
  uint64_t head = 0, body = 0;
  if (same16) {
    head = ((16 - (m & 15)) & 15);
    if (head > n) head = n;
    const uint64_t nv = (n - head) / 16;
    if (SGD) fold_v4<SgdOp, 4>(var, g, nw, head, nv, t, nth, lr);
    else fold_v4<XorOp, 4>(var, g, nw, head, nv, t, nth, lr);
    body = nv * 16;
  } else if (same8) {
    head = ((8 - (m & 7)) & 7);
    if (head > n) head = n;
    const uint64_t nv = (n - head) / 8;
    if (SGD) fold_v2<SgdOp>(var, g, nw, head, nv, t, nth, lr);
    else fold_v2<XorOp>(var, g, nw, head, nv, t, nth, lr);
    body = nv * 8;
  }
  // scalar elements outside the vector body: [0, head) and [head + body, n)
  const uint64_t rest = (n - body) / unit;
  for (uint64_t j = t; j < rest; j += nth) {
    const uint64_t e = j * unit < head ? j * unit : j * unit + body;  // byte offset
    if (SGD) {
      float v = *(float *)(var + e);
      for (int w = 0; w < nw; ++w) v = sgd1(v, lr, *(const float *)(g[w] + e));
      *(float *)(var + e) = v;
    } else {
      uint8_t acc = var[e];
      for (int w = 0; w < nw; ++w) acc ^= g[w][e];
      var[e] = acc;
    }
  }
}

__global__ void __launch_bounds__(512) k_apply_xor(const __grid_constant__ ApplyArgs a) {
  apply_range<false>(a.var, a.g, a.nw, a.n, a.lr,
                     (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                     (uint64_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(512) k_apply_sgd(const __grid_constant__ ApplyArgs a) {
  apply_range<true>(a.var, a.g, a.nw, a.n, a.lr,
                    (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                    (uint64_t)gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------------------
// Batched PS step kernels (one launch per phase per step; descriptors live in
// device memory, validated once at creation like a registered verb list).
// ---------------------------------------------------------------------------
struct BatchPut {        // K1/K3 over many edges
  const uint8_t *src;    // body source
  uint8_t *dst;          // destination (peer or local)
  uint64_t body;         // bytes before the tail
  const uint8_t *tail;   // tail byte source (flag cell / meta flag)
  uint32_t cta_begin, cta_count;
  uint32_t wait_empty, pad;
};

struct BatchGen {        // worker: consume weight, (re)produce gradient
  uint8_t *grad;
  uint64_t n;            // bytes (fp32 elements * 4)
  uint8_t *weight_flag;  // local static region tail (nullptr: local variable)
  const uint8_t *credit; // shard-side meta tail that must read 0 (nullptr: none)
  uint64_t node;         // GenGrad node id (RNG stream key)
  uint32_t cta_begin, cta_count;
  // K3 fused into the gen's last CTA (exchange schedule): the DynSender.send
  // of this gradient's metadata block (nullptr: none / separate meta batch)
  const uint8_t *meta_src;
  uint8_t *meta_dst;
  const uint8_t *meta_tail;
  uint64_t meta_body;
  uint64_t elem_offset;  // first element's index in its model variable (slices)
  // gradient read in place by a shard on this server (co-located worker):
  // released to 1 when the gradient is complete, cleared by that apply; the
  // gen waits for 0 (credit) before overwriting it.  nullptr: none.
  uint8_t *ready;
};

struct BatchApply {      // shard: fused dynamic receive (meta decode + peer
  uint8_t *var;          // reads) + ApplyGrad of all workers, ascending
  uint64_t n;
  const uint8_t *src[SRF_MAX_WORKERS];   // local gradient, or meta block
  const uint8_t *peer_base[SRF_MAX_WORKERS];
  uint64_t peer_lo[SRF_MAX_WORKERS], peer_hi[SRF_MAX_WORKERS];
  uint64_t peer_token[SRF_MAX_WORKERS];
  uint32_t is_meta;      // bit w: src[w] is a meta block
  int nw, rank;
  uint32_t cta_begin, cta_count;
  const uint8_t *ready[SRF_MAX_WORKERS];  // in-place gradient w complete (nullptr: none)
};

template <typename D>
__device__ __forceinline__ int find_desc(const D *d, int n, uint32_t u) {
  // largest i with d[i].cta_begin <= u (work units are CTA-sized slices)
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (d[mid].cta_begin <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu_u8(const uint8_t *p) {
  uint16_t v;
  asm volatile("ld.acquire.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return v & 0xff;
}

__device__ __forceinline__ bool spin_until(const uint8_t *p, uint32_t want,
                                           uint64_t timeout_ns, int sys_scope = 1) {
  uint64_t t0 = globaltimer_ns();
  while ((sys_scope ? ld_acquire_sys_u8(p) : ld_acquire_gpu_u8(p)) != want) {
    if (globaltimer_ns() - t0 > timeout_ns) return false;
    __nanosleep(20);
  }
  return true;
}

// One work unit (a CTA-sized slice of one descriptor) of each batch kind; the
// batch kernels loop over units, the exchange kernel claims them from a queue.
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const unsigned int *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Several iterations per exchange launch: a descriptor's units of iteration
// k start only after its iteration k-1 completed (its per-launch completion
// count reached k) - flags alone do not tell iterations apart, and the
// arrival counter must not mix them.
__device__ __forceinline__ void wait_count(const unsigned int *p, uint32_t want,
                                           uint64_t timeout_ns, int *err) {
  if (!p || want == 0) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_gpu_u32(p) < want) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(err, 7);
      return;
    }
    __nanosleep(20);
  }
}

__device__ __forceinline__ void count_done(unsigned int *p) {
  if (p) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// seq: per-descriptor completion counts of this launch (nullptr: one
// iteration per launch); k: iteration index in the launch; wait_done /
// wait_index: the pushed variable must have been updated k times before its
// weights are read again
__device__ __forceinline__ void put_unit(const BatchPut *descs, int n, uint32_t u,
                                         unsigned int *counters, uint64_t timeout_ns, int *err,
                                         int sys, const unsigned int *wait_done = nullptr,
                                         const int *wait_index = nullptr, uint32_t k = 0,
                                         unsigned int *seq = nullptr) {
  __shared__ int s_desc, s_last;
  {
    if (threadIdx.x == 0) {
      s_desc = find_desc(descs, n, u);
      if (seq) wait_count(seq + s_desc, k, timeout_ns, err);
      if (k && wait_index[s_desc] >= 0) wait_count(wait_done + wait_index[s_desc], k, timeout_ns, err);
    }
    __syncthreads();
    const BatchPut d = descs[s_desc];
    const uint32_t lb = u - d.cta_begin;
    if (d.wait_empty) {
      if (threadIdx.x == 0 && !spin_until(d.dst + d.body, 0, timeout_ns, sys)) atomicExch(err, 2);
      __syncthreads();
    }
    copy_bytes_grid<8>(d.dst, d.src, d.body, (uint64_t)lb * blockDim.x + threadIdx.x,
                       (uint64_t)d.cta_count * blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(&counters[s_desc], d.cta_count - 1, sys);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      // re-arm the arrival counter BEFORE publishing: whoever acquires the
      // flag (and, downstream, the next use of this edge) sees it at zero
      atomicExch(&counters[s_desc], 0u);
      release_tail(d.dst + d.body, *d.tail, sys);
      if (seq) count_done(seq + s_desc);
    }
    __syncthreads();  // shared state is reused by the next unit
  }
}

__device__ __forceinline__ void put_batch_units(const BatchPut *descs, int n,
                                                uint32_t total_units, unsigned int *counters,
                                                uint64_t timeout_ns, int *err, int sys) {
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x)
    put_unit(descs, n, u, counters, timeout_ns, err, sys);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

// uniform [0,1) fp32 of a counter-based stream keyed on (seed, node, iteration)
__device__ __forceinline__ float unit_f32(uint32_t k0, uint32_t k1, uint32_t i) {
  return (float)((fmix32(i * 0x9E3779B1u + k0) ^ k1) >> 8) * (1.0f / 16777216.0f);
}

__device__ __forceinline__ void gen_unit(const BatchGen *descs, int n, uint32_t u,
                                         unsigned int *counters, uint64_t seed,
                                         uint64_t iteration, int regen, int fuse_meta,
                                         uint64_t timeout_ns, int *err, int sys,
                                         uint32_t k = 0, unsigned int *seq = nullptr) {
  __shared__ int s_desc, s_last;
  {
    if (threadIdx.x == 0) {
      s_desc = find_desc(descs, n, u);
      if (seq) wait_count(seq + s_desc, k, timeout_ns, err);
    }
    __syncthreads();
    const BatchGen d = descs[s_desc];
    const uint32_t lb = u - d.cta_begin;
    if (threadIdx.x == 0) {
      if (d.weight_flag && !spin_until(d.weight_flag, 1, timeout_ns, sys)) atomicExch(err, 3);
      if (d.credit && !spin_until(d.credit, 0, timeout_ns, sys)) atomicExch(err, 4);
    }
    __syncthreads();
    if (regen) {
      const uint64_t key = mix64(seed * 0x9E3779B97F4A7C15ull ^ mix64(d.node + 0x51ED) ^
                                 mix64(iteration * 0xD1B54A32D192ED03ull));
      const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
      const uint64_t nf = d.n / 4;
      const uint64_t nth = (uint64_t)d.cta_count * blockDim.x;
      float4 *g4 = (float4 *)d.grad;  // gradient blocks are 16-B aligned by layout
      const uint32_t e0 = (uint32_t)d.elem_offset;
      for (uint64_t q = (uint64_t)lb * blockDim.x + threadIdx.x; q < nf / 4; q += nth) {
        const uint32_t i = (uint32_t)(4 * q) + e0;
        g4[q] = make_float4(unit_f32(k0, k1, i), unit_f32(k0, k1, i + 1),
                            unit_f32(k0, k1, i + 2), unit_f32(k0, k1, i + 3));
      }
      float *g = (float *)d.grad;
      for (uint64_t i = (nf / 4) * 4 + (uint64_t)lb * blockDim.x + threadIdx.x; i < nf; i += nth)
        g[i] = unit_f32(k0, k1, (uint32_t)i + e0);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(&counters[s_desc], d.cta_count - 1, sys);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      atomicExch(&counters[s_desc], 0u);  // re-armed before anything is published
      // the weight was consumed: clear its flag (StaticReceiver.poll semantics)
      if (d.weight_flag) release_tail(d.weight_flag, 0, sys);
      // the in-place gradient is complete (read directly by the co-located apply)
      if (d.ready) release_tail(d.ready, 1, sys);
      if (fuse_meta && d.meta_dst) {
        // K3: the gradient's metadata block, flag last; the acq_rel arrival
        // above made every CTA's gradient stores visible before this release
        for (uint64_t b = 0; b < d.meta_body; ++b) d.meta_dst[b] = d.meta_src[b];
        release_tail(d.meta_dst + d.meta_body, *d.meta_tail, sys);
      }
      if (seq) count_done(seq + s_desc);
    }
    __syncthreads();  // shared state is reused by the next unit
  }
}

__device__ __forceinline__ void gen_batch_units(const BatchGen *descs, int n,
                                                uint32_t total_units, unsigned int *counters,
                                                uint64_t seed, uint64_t iteration_arg,
                                                const uint64_t *iteration_ptr, int regen,
                                                uint64_t timeout_ns, int *err, int sys) {
  // iteration from a device counter when given (graph-replayed steps)
  const uint64_t iteration = iteration_ptr ? *(const volatile uint64_t *)iteration_ptr
                                           : iteration_arg;
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x)
    gen_unit(descs, n, u, counters, seed, iteration, regen, 0, timeout_ns, err, sys);
}

__device__ __forceinline__ void apply_unit(const BatchApply *descs, int n, uint32_t u,
                                           unsigned int *counters, int op, float lr,
                                           uint64_t timeout_ns, int *err, int sys,
                                           unsigned int *done = nullptr, uint32_t k = 0) {
  __shared__ int s_desc, s_last, s_bad;
  __shared__ const uint8_t *s_g[SRF_MAX_WORKERS];
  {
    if (threadIdx.x == 0) {
      s_desc = find_desc(descs, n, u);
      s_bad = 0;
      if (done) wait_count(done + s_desc, k, timeout_ns, err);
    }
    __syncthreads();
    const BatchApply &d = descs[s_desc];
    const uint32_t lb = u - d.cta_begin;
    const int r = d.rank;
    if (threadIdx.x < (unsigned)d.nw) {
      // DynReceiver.poll + decode_meta + validation (protocol.py:234-242,
      // wire.py:120-142, memspace.py:145-157): one lane per worker, in parallel
      const int w = threadIdx.x;
      const uint8_t *m = d.src[w];
      if (!((d.is_meta >> w) & 1)) {
        s_g[w] = m;  // co-located worker: its gradient block directly
        if (d.ready[w] && !spin_until(d.ready[w], 1, timeout_ns, sys)) {
          atomicExch(err, 5);
          s_bad = 1;
        }
      } else if (!spin_until(m + 8 * r + 32, 1, timeout_ns, sys)) {
        atomicExch(err, 5);
        s_bad = 1;
      } else {
        const uint64_t addr = *(const volatile uint64_t *)(m + 8 + 8 * r);  // after the dims
        const uint64_t tok = *(const volatile uint64_t *)(m + 16 + 8 * r);
        const uint64_t plen = *(const volatile uint64_t *)(m + 24 + 8 * r);
        // decode_meta's consistency check: payload_len == prod(dims) * elem size
        const uint32_t code = m[0];
        const uint64_t esz = code == 0 ? 4 : code == 1 ? 8 : code == 2 ? 4 : code == 3 ? 8
                           : code == 4 ? 1 : 0;
        uint64_t prod = esz;
        for (int k = 0; k < r; ++k) prod *= *(const volatile uint64_t *)(m + 8 + 8 * k);
        if (m[1] != r || esz == 0 || prod != plen || plen != d.n || tok != d.peer_token[w] ||
            addr < d.peer_lo[w] || addr + plen > d.peer_hi[w]) {
          atomicExch(err, 6);
          s_bad = 1;
        }
        s_g[w] = d.peer_base[w] + addr;  // one-sided read through the peer mapping
      }
    }
    __syncthreads();
    if (!s_bad) {
      const uint64_t t = (uint64_t)lb * blockDim.x + threadIdx.x;
      const uint64_t nth = (uint64_t)d.cta_count * blockDim.x;
      if (op == SRF_APPLY_XOR)
        apply_range<false>(d.var, s_g, d.nw, d.n, lr, t, nth);
      else
        apply_range<true>(d.var, s_g, d.nw, d.n, lr, t, nth);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(&counters[s_desc], d.cta_count - 1, sys);
    __syncthreads();
    // re-arm the arrival counter before any credit is published (thread 0,
    // ordered before the lanes' releases by the barrier)
    if (s_last && threadIdx.x == 0) atomicExch(&counters[s_desc], 0u);
    __syncthreads();
    // gradients consumed: the last CTA clears the meta flags (credit for the
    // next send; DynReceiver.poll's clear)
    if (s_last && threadIdx.x < (unsigned)d.nw && ((d.is_meta >> threadIdx.x) & 1))
      release_tail((uint8_t *)d.src[threadIdx.x] + 8 * r + 32, 0, sys);
    if (s_last && threadIdx.x < (unsigned)d.nw && d.ready[threadIdx.x])
      release_tail((uint8_t *)d.ready[threadIdx.x], 0, sys);
    if (s_last && threadIdx.x == 0) {
      // one more update of this variable completed (multi-iteration exchange)
      if (done) count_done(done + s_desc);
    }
    __syncthreads();  // shared state is reused by the next unit
  }
}

__device__ __forceinline__ void apply_batch_units(const BatchApply *descs, int n,
                                                  uint32_t total_units, unsigned int *counters,
                                                  int op, float lr, uint64_t timeout_ns,
                                                  int *err, int sys) {
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x)
    apply_unit(descs, n, u, counters, op, lr, timeout_ns, err, sys);
}


__global__ void __launch_bounds__(512) k_put_batch(const BatchPut *descs, int n,
                                                   uint32_t total_units, unsigned int *counters,
                                                   uint64_t timeout_ns, int *err, int sys) {
  put_batch_units(descs, n, total_units, counters, timeout_ns, err, sys);
}

__global__ void __launch_bounds__(512) k_gen_batch(const BatchGen *descs, int n,
                                                   uint32_t total_units, unsigned int *counters,
                                                   uint64_t seed, uint64_t iteration_arg,
                                                   const uint64_t *iteration_ptr, int regen,
                                                   uint64_t timeout_ns, int *err, int sys) {
  gen_batch_units(descs, n, total_units, counters, seed, iteration_arg, iteration_ptr, regen,
                  timeout_ns, err, sys);
}

__global__ void __launch_bounds__(256) k_apply_batch(const BatchApply *descs, int n,
                                                     uint32_t total_units, unsigned int *counters,
                                                     int op, float lr, uint64_t timeout_ns,
                                                     int *err, int sys) {
  apply_batch_units(descs, n, total_units, counters, op, lr, timeout_ns, err, sys);
}

// Device-side DynReceiver (runtime/protocol.py:224-254) for device-resident
// loops: acquire the metadata flag, decode and validate the block exactly as
// decode_meta + check_remote_access do (wire.py:114-142, memspace.py:145-157),
// pull the announced bytes into a pre-allocated block (K4), publish the length,
// and clear the flag (the poll's clear = the sender's next credit).
struct DynRecvArgs {
  uint8_t *meta;            // receiver's metadata block
  int rank;
  const uint8_t *peer_base;
  uint64_t peer_lo, peer_hi, peer_token;
  uint8_t *dst;
  uint64_t dst_cap;
  uint64_t *len_out;        // nullptr: none
  unsigned int *counter;
  uint64_t timeout_ns;
  int *err;
  int sys;
};

__global__ void __launch_bounds__(256) k_dyn_recv(const __grid_constant__ DynRecvArgs a) {
  __shared__ const uint8_t *s_src;
  __shared__ uint64_t s_len;
  __shared__ int s_ok, s_last;
  const int r = a.rank;
  if (threadIdx.x == 0) {
    s_ok = 0;
    s_len = 0;
    const uint8_t *m = a.meta;
    if (!spin_until(m + 8 * r + 32, 1, a.timeout_ns, 1)) {
      atomicExch(a.err, 5);
    } else {
      const uint64_t addr = *(const volatile uint64_t *)(m + 8 + 8 * r);
      const uint64_t tok = *(const volatile uint64_t *)(m + 16 + 8 * r);
      const uint64_t plen = *(const volatile uint64_t *)(m + 24 + 8 * r);
      const uint32_t code = m[0];
      const uint64_t esz = code == 0 ? 4 : code == 1 ? 8 : code == 2 ? 4 : code == 3 ? 8
                         : code == 4 ? 1 : 0;
      uint64_t prod = esz;
      for (int k = 0; k < r; ++k) prod *= *(const volatile uint64_t *)(m + 8 + 8 * k);
      if (m[1] != r || esz == 0 || prod != plen || tok != a.peer_token || addr < a.peer_lo ||
          addr + plen > a.peer_hi || plen > a.dst_cap) {
        atomicExch(a.err, 6);
      } else {
        s_src = a.peer_base + addr;
        s_len = plen;
        s_ok = 1;
      }
    }
  }
  __syncthreads();
  if (s_ok)
    copy_bytes_grid<8>(a.dst, s_src, s_len, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                       (uint64_t)gridDim.x * blockDim.x);
  __syncthreads();
  if (threadIdx.x == 0) s_last = grid_arrive(a.counter, gridDim.x - 1, a.sys);
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    if (a.len_out) *(volatile uint64_t *)a.len_out = s_ok ? s_len : ~0ull;
    release_tail(a.meta + 8 * r + 32, 0, a.sys);
    atomicExch(a.counter, 0u);
  }
}

// One PS iteration loop in a single cooperative launch (all servers on this
// GPU): the four phases back to back, separated by grid-wide barriers, for
// `iters` iterations.  The device flags and credits are still set and
// consumed exactly as in the per-phase launches; only the launch gaps go.
static constexpr int kMaxApply = 8;

struct PsPersistArgs {
  const BatchPut *push; int npush; uint32_t upush; unsigned int *cpush;
  const BatchGen *gen; int ngen; uint32_t ugen; unsigned int *cgen; uint64_t seed;
  const BatchPut *meta; int nmeta; uint32_t umeta; unsigned int *cmeta;
  const BatchApply *apply[kMaxApply]; int napply[kMaxApply]; uint32_t uapply[kMaxApply];
  unsigned int *capply[kMaxApply]; int nbatches;
  int op; float lr;
  uint64_t it0; uint32_t iters; int regen; uint64_t timeout_ns; int *err;
  int sys;  // every buffer is this GPU's own HBM -> 0 (gpu-scope ordering)
};

__global__ void __launch_bounds__(256) k_ps_persistent(const __grid_constant__ PsPersistArgs a) {
  cg::grid_group grid = cg::this_grid();
  for (uint32_t i = 0; i < a.iters; ++i) {
    if (a.push) put_batch_units(a.push, a.npush, a.upush, a.cpush, a.timeout_ns, a.err, a.sys);
    grid.sync();
    if (a.gen)
      gen_batch_units(a.gen, a.ngen, a.ugen, a.cgen, a.seed, a.it0 + i, nullptr, a.regen,
                      a.timeout_ns, a.err, a.sys);
    grid.sync();
    if (a.meta) put_batch_units(a.meta, a.nmeta, a.umeta, a.cmeta, a.timeout_ns, a.err, a.sys);
    grid.sync();
    for (int b = 0; b < a.nbatches; ++b)
      apply_batch_units(a.apply[b], a.napply[b], a.uapply[b], a.capply[b], a.op, a.lr,
                        a.timeout_ns, a.err, a.sys);
    grid.sync();
  }
}


// Dependency-driven PS step (the exchange schedule): every unit of this GPU's
// push, gen (+ fused meta) and apply batches sits in one queue, ordered by a
// key every rank derives from the variable, and persistent CTAs claim units
// in queue order with one atomic.  A unit only waits on units that precede it
// in that global order (weights before their gradient, gradients before their
// apply, the previous step before this one), so the earliest unfinished unit
// can always run: no deadlock whatever the grid, and a shard starts pulling
// variable v while its later weights are still being pushed.
struct ExItem {
  uint32_t unit;
  uint16_t kind;   // 0 push, 1 gen, 2 apply
  uint16_t batch;  // apply batch index
};

struct ExArgs {
  const BatchPut *push; int npush; unsigned int *cpush; int push_sys;
  const BatchGen *gen; int ngen; unsigned int *cgen; uint64_t seed; int gen_sys;
  const BatchApply *apply[kMaxApply]; int napply[kMaxApply]; unsigned int *capply[kMaxApply];
  int apply_sys[kMaxApply];
  int op; float lr;
  const ExItem *items; uint32_t nitems; unsigned int *claim; unsigned int *exit_count;
  uint64_t iteration; int regen; uint64_t timeout_ns; int *err;
  // several iterations per launch: the queue repeats `iters` times (iteration
  // k's units after iteration k-1's); done[] counts completed applies per
  // apply descriptor in this launch, push_done[i] maps push edge i to its
  // variable's counter (-1: none)
  uint32_t iters;
  unsigned int *done; int apply_base[kMaxApply]; const int *push_done;
  unsigned int *seq_push, *seq_gen;  // per-descriptor completion counts (this launch)
};

__global__ void __launch_bounds__(512) k_ps_exchange(const __grid_constant__ ExArgs a) {
  __shared__ uint32_t s_i;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(a.claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= a.nitems * a.iters) break;
    const uint32_t k = i / a.nitems;
    const ExItem x = a.items[i - k * a.nitems];
    if (x.kind == 0)
      put_unit(a.push, a.npush, x.unit, a.cpush, a.timeout_ns, a.err, a.push_sys, a.done,
               a.push_done, k, a.seq_push);
    else if (x.kind == 1)
      gen_unit(a.gen, a.ngen, x.unit, a.cgen, a.seed, a.iteration + k, a.regen, 1,
               a.timeout_ns, a.err, a.gen_sys, k, a.seq_gen);
    else
      apply_unit(a.apply[x.batch], a.napply[x.batch], x.unit, a.capply[x.batch], a.op, a.lr,
                 a.timeout_ns, a.err, a.apply_sys[x.batch], a.done + a.apply_base[x.batch], k);
  }
  // the last CTA out re-arms the queue for the next launch
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    *a.exit_count = 0;
  }
}

// ---------------------------------------------------------------------------
// RPC-style baseline on the device (runtime/protocol.py:257-448, FORMATS.md
// "RPC baseline fragment"): the stream metadata||payload is cut into 4096-B
// fragments (16-B header msg_id u64, index u32, count u32 + 4080 B); the
// sender serialises each fragment into a staging slot (counted copy 1) and
// writes it into one of the receiver's 16 posted 4-KiB ring slots; the
// receiver checks the header, copies the bytes out (counted copy 2) and
// re-posts the slot.  Warp w owns ring slot w (fragments w, w+16, ...), so the
// ring's 16-deep pipeline is kept and fragments land in order per slot.
// ---------------------------------------------------------------------------
static constexpr int kFrag = 4096, kFragHdr = 16, kFragPay = kFrag - kFragHdr, kRing = 16;

struct RpcArgs {
  const uint8_t *meta;  uint32_t meta_len;   // sender: metadata stage
  const uint8_t *payload; uint64_t pay_len;  // sender: tensor bytes
  uint8_t *stage;                            // sender: 16 x 4096 staging
  uint8_t *ring;                             // receiver: 16 x 4096 posted slots
  uint8_t *ring_flags;                       // receiver: 16 slot states (1 full)
  uint8_t *meta_out;                         // receiver: reassembled metadata
  uint8_t *tensor_out;                       // receiver: tensor buffer
  uint64_t msg_id;
  uint64_t timeout_ns;
  int *err;
  int role;                                  // -1: both (block 0 sender, 1 receiver)
};

// 64 threads (a warp pair) move one fragment
static constexpr int kSlotThreads = 64;

__device__ __forceinline__ void slot_copy(uint8_t *dst, const uint8_t *src, uint64_t n) {
  copy_bytes_grid<4>(dst, src, n, threadIdx.x % kSlotThreads, kSlotThreads);
}

__device__ __forceinline__ void slot_sync() {
  // the two warps of a slot: named barrier = slot index (0..15; the kernel
  // never uses __syncthreads)
  asm volatile("bar.sync %0, %1;" ::"r"((int)(threadIdx.x / kSlotThreads)),
               "r"(kSlotThreads));
}

// bytes [off, off + n) of the message stream into dst
__device__ __forceinline__ void stream_gather(const RpcArgs &a, uint8_t *dst, uint64_t off,
                                              uint64_t n) {
  if (off < a.meta_len) {
    uint64_t k = a.meta_len - off < n ? a.meta_len - off : n;
    slot_copy(dst, a.meta + off, k);
    dst += k; off += k; n -= k;
  }
  if (n) slot_copy(dst, a.payload + (off - a.meta_len), n);
}

__device__ __forceinline__ void stream_scatter(const RpcArgs &a, const uint8_t *src,
                                               uint64_t off, uint64_t n) {
  if (off < a.meta_len) {
    uint64_t k = a.meta_len - off < n ? a.meta_len - off : n;
    slot_copy(a.meta_out + off, src, k);
    src += k; off += k; n -= k;
  }
  if (n) slot_copy(a.tensor_out + (off - a.meta_len), src, n);
}

__global__ void __launch_bounds__(1024) k_rpc(RpcArgs a) {
  const int role = a.role >= 0 ? a.role : (int)blockIdx.x;
  const int w = threadIdx.x / kSlotThreads;            // ring slot of this warp pair
  const bool leader = (threadIdx.x % kSlotThreads) == 0;
  const uint64_t total = a.meta_len + a.pay_len;
  const uint32_t count = (uint32_t)((total + kFragPay - 1) / kFragPay);
  uint8_t *slot = a.ring + (uint64_t)w * kFrag;
  uint8_t *flag = a.ring_flags + w;
  uint8_t *st = a.stage + (uint64_t)w * kFrag;
  for (uint32_t f = w; f < count; f += kRing) {
    const uint64_t off = (uint64_t)f * kFragPay;
    const uint64_t n = total - off < (uint64_t)kFragPay ? total - off : (uint64_t)kFragPay;
    if (role == 0) {
      // sender: serialise into the staging slot (counted copy 1) - this
      // overlaps the receiver draining the previous fragment of the slot -
      // then wait for the posted ring slot and send
      if (leader) {
        *(uint64_t *)st = a.msg_id;
        *(uint32_t *)(st + 8) = f;
        *(uint32_t *)(st + 12) = count;
      }
      stream_gather(a, st + kFragHdr, off, n);
      if (leader && !spin_until(flag, 0, a.timeout_ns)) atomicExch(a.err, 7);
      slot_sync();
      slot_copy(slot, st, kFragHdr + n);  // the send verb
      slot_sync();
      if (leader) {
        __threadfence_system();
        st_release_sys_u8(flag, 1);
      }
    } else {
      // receiver: drain the slot in order, copy out (counted copy 2), re-post
      if (leader && !spin_until(flag, 1, a.timeout_ns)) atomicExch(a.err, 7);
      slot_sync();
      if (leader && (*(volatile uint64_t *)slot != a.msg_id ||
                     *(volatile uint32_t *)(slot + 8) != f))
        atomicExch(a.err, 8);  // ReassemblyGap
      stream_scatter(a, slot + kFragHdr, off, n);
      slot_sync();
      if (leader) {
        __threadfence_system();
        st_release_sys_u8(flag, 0);
      }
    }
    slot_sync();
  }
}

// ReduceMax (graph.py:378-382): per-block max, last block folds partials.
__device__ __forceinline__ float fmax_nan(float a, float b) {
  // numpy max propagates NaN
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}

__global__ void __launch_bounds__(256) k_reduce_max(const float *x, uint64_t n,
                                                    float *out, float *part,
                                                    unsigned int *counter) {
  __shared__ float sm[32];
  __shared__ int s_last;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  float m = -INFINITY;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (((uintptr_t)x & 15) == 0) {
    // 16-B loads, four in flight per thread
    const float4 *x4 = (const float4 *)x;
    const uint64_t n4 = n / 4;
    uint64_t i = t0;
    for (; i + 3 * nth < n4; i += 4 * nth) {
      float4 a = __ldg(x4 + i), b = __ldg(x4 + i + nth), c = __ldg(x4 + i + 2 * nth),
             d = __ldg(x4 + i + 3 * nth);
      m = fmax_nan(m, fmax_nan(fmax_nan(a.x, a.y), fmax_nan(a.z, a.w)));
      m = fmax_nan(m, fmax_nan(fmax_nan(b.x, b.y), fmax_nan(b.z, b.w)));
      m = fmax_nan(m, fmax_nan(fmax_nan(c.x, c.y), fmax_nan(c.z, c.w)));
      m = fmax_nan(m, fmax_nan(fmax_nan(d.x, d.y), fmax_nan(d.z, d.w)));
    }
    for (; i < n4; i += nth) {
      float4 a = __ldg(x4 + i);
      m = fmax_nan(m, fmax_nan(fmax_nan(a.x, a.y), fmax_nan(a.z, a.w)));
    }
    for (uint64_t j = n4 * 4 + t0; j < n; j += nth) m = fmax_nan(m, x[j]);
  } else {
    for (uint64_t i = t0; i < n; i += nth) m = fmax_nan(m, x[i]);
  }
  for (int o = 16; o; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(~0u, m, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(~0u, m, o));
    if (threadIdx.x == 0) {
      part[blockIdx.x] = m;
      __threadfence();
      s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float r = -INFINITY;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x)
    r = fmax_nan(r, ((volatile float *)part)[i]);
  for (int o = 16; o; o >>= 1) r = fmax_nan(r, __shfl_xor_sync(~0u, r, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    r = -INFINITY;
    for (unsigned i = 0; i < (blockDim.x >> 5); ++i) r = fmax_nan(r, sm[i]);
    *out = (n == 0) ? 0.0f : r;
    atomicExch(counter, 0u);
  }
}

// ---------------------------------------------------------------------------
// launch geometry
// ---------------------------------------------------------------------------
static void copy_geometry(int device, uint64_t bytes, int *grid, int *block) {
  const int threads = g_copy_threads;
  // one CTA moves threads * 16 B * 4 per unrolled batch; cap at k CTAs/SM
  uint64_t per_cta = (uint64_t)threads * 16 * 4;
  uint64_t want = (bytes + per_cta - 1) / per_cta;
  uint64_t cap = (uint64_t)sm_count_of(device) * g_ctas_per_sm;
  if (want < 1) want = 1;
  if (want > cap) want = cap;
  *grid = (int)want;
  *block = threads;
}

static int record_event(int device, cudaStream_t s, srf_event_t *ev_out) {
  if (!ev_out) return SRF_OK;
  srf_event *ev = new srf_event();
  ev->device = device;
  cudaError_t e = cudaEventCreateWithFlags(&ev->e, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev->e, s);
  if (e != cudaSuccess) {
    delete ev;
    return fail(SRF_E_DEVICE, "event: %s", cudaGetErrorString(e));
  }
  *ev_out = ev;
  return SRF_OK;
}

static int launch_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(SRF_E_DEVICE, "%s launch: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SRF_OK;
}

static int g_put_impl = 0;  // 0 = vector LDG/STG, 1 = TMA bulk (large segments)
static int g_unroll = 8;    // 16-B vectors in flight per thread (4 or 8)
// knob 6: cross-device bodies of at least this many bytes move on the copy
// engine (0: never).  32 MiB: the engine's extra ~15 us per put (credit wait
// launch, copy, tail launch) pays off only above ~20 MB (NVLink sweep).  SM stores into a peer's pool are capped near 496 GB/s
// across processes; the DMA engine reaches ~750 GB/s through the same mapping
// (profiles/r1_ring_probe.json, r1_xproc_store_probe*.jsonl).
static uint64_t g_peer_ce_bytes = 32ull << 20;

// launch K1/K4/K5 with the configured implementation
static int launch_copy(const PutArgs &a, srf_stream *s, const char *what) {
  uint64_t big = 0;
  for (int i = 0; i < a.nseg; ++i) big = std::max<uint64_t>(big, a.seg[i].len);
  if (g_put_impl == 1 && big >= (uint64_t)4 * kBulkChunk) {
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
  } else {
    int grid, block;
    copy_geometry(s->device, a.total, &grid, &block);
    if (g_unroll == 8)
      k_put<8><<<grid, block, 0, s->s>>>(a);
    else
      k_put<4><<<grid, block, 0, s->s>>>(a);
  }
  return launch_check(what);
}

// K1 with a copy-engine body: [credit wait] -> body copies -> a one-thread K1
// that releases the tail byte.  Stream order starts the tail kernel only after
// the copies have completed, so a consumer that acquires the flag sees the
// body (release/acquire stress test, tests/test_gpu_kernels.py).
static int put_via_copy_engine(const PutArgs &a, srf_stream *s) {
  uint8_t *tail = a.dst + a.total - 1;
  if (a.wait_empty) {
    k_flag_wait<<<1, 32, 0, s->s>>>(tail, 0, 0, a.timeout_ns, a.err);
    int rc = launch_check("k_flag_wait(credit)");
    if (rc) return rc;
  }
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
  k_put<4><<<1, 32, 0, s->s>>>(t);
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

int srf_event_free(srf_event_t ev) {
  DeviceGuard device_guard;
  if (!ev) return SRF_OK;
  cudaEventDestroy(ev->e);
  delete ev;
  return SRF_OK;
}

int srf_put(srf_space_t src_space, const uint64_t *src_addr,
            const uint64_t *src_len, const uint64_t *src_token, int nseg,
            srf_space_t dst_space, uint64_t dst_addr, uint64_t dst_token,
            int flags, srf_stream_t st, srf_event_t *ev_out) {
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
  a.sys_scope = (dst_space->imported || dst_space->device != s->device) ? 1 : 0;
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
  a.timeout_ns = 5ull * 1000 * 1000 * 1000;
  a.counter = s->counter;
  a.err = src_space->err;
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  if (a.sys_scope && g_peer_ce_bytes && total - 1 >= g_peer_ce_bytes && a.db_len <= 1)
    rc = put_via_copy_engine(a, s);
  else
    rc = launch_copy(a, s, "k_put");
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
  a.counter = s->counter;
  a.err = dst_space->err;
  CUDA_TRY(cudaSetDevice(s->device));
  int rc = SRF_OK;
  const bool cross = src_space->imported || src_space->device != s->device;
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
  k_dyn_recv<<<grid, 256, 0, s->s>>>(a);
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
  if (nbytes == 0) return record_event(var_space->device, var_space->stream->s, ev_out);
  srf_stream *s = stream_or_default(var_space, st);
  int grid, block;
  copy_geometry(s->device, nbytes, &grid, &block);
  CUDA_TRY(cudaSetDevice(s->device));
  if (op == SRF_APPLY_XOR)
    k_apply_xor<<<grid, block, 0, s->s>>>(a);
  else
    k_apply_sgd<<<grid, block, 0, s->s>>>(a);
  rc = launch_check("k_apply");
  if (rc) return rc;
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
  return launch_check("k_reduce_max");
}

// ---------------------------------------------------------------------------
// batches (PS step phases)
// ---------------------------------------------------------------------------
struct srf_batch {
  int kind;  // 0 put, 1 gen, 2 apply
  int device;
  const uint64_t *iter_ptr = nullptr;  // gen: device iteration counter (graphs)
  int sys = 1;  // 0 when every buffer of the batch is on the launching GPU
  void *descs;
  int n;
  unsigned int *counters;
  int grid;
  int op;
  float lr;
  uint64_t seed;
  int *err;
  std::vector<uint8_t> host;  // host copy of the descriptors
};

static uint32_t ctas_for(int device, uint64_t bytes, uint64_t per_cta) {
  // work units of ~per_cta bytes each (large enough to amortise the per-unit
  // flag acquire / metadata decode), at most 8 units per SM per descriptor
  uint64_t want = (bytes + per_cta - 1) / per_cta;
  uint64_t cap = (uint64_t)sm_count_of(device) * 8;  // batch phases: up to 8 units/SM
  return (uint32_t)std::max<uint64_t>(1, std::min(want, cap));
}

}  // extern "C"

template <typename D>
static int finish_batch(int kind, int device, std::vector<D> &host, int *err, srf_batch_t *out) {
  srf_batch *b = new srf_batch();
  b->kind = kind;
  b->device = device;
  b->n = (int)host.size();
  b->err = err;
  b->op = 0;
  b->lr = 0;
  b->seed = 0;
  uint32_t total = 0;
  for (auto &d : host) total = d.cta_begin + d.cta_count;
  b->grid = (int)total;
  b->host.assign((const uint8_t *)host.data(), (const uint8_t *)(host.data() + host.size()));
  CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMalloc(&b->descs, sizeof(D) * std::max<size_t>(1, host.size()));
  if (e == cudaSuccess && !host.empty())
    e = cudaMemcpy(b->descs, host.data(), sizeof(D) * host.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&b->counters, sizeof(unsigned) * std::max<size_t>(1, host.size()));
  if (e == cudaSuccess) e = cudaMemset(b->counters, 0, sizeof(unsigned) * std::max<size_t>(1, host.size()));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // counters zero before any launch
  if (e != cudaSuccess) {
    delete b;
    return fail(SRF_E_DEVICE, "batch upload: %s", cudaGetErrorString(e));
  }
  *out = b;
  return SRF_OK;
}


extern "C" {

int srf_batch_put_create(int n, srf_space_t const *src_space, const uint64_t *src_addr,
                         const uint64_t *body_len, const uint64_t *src_token,
                         const uint64_t *tail_addr, srf_space_t const *dst_space,
                         const uint64_t *dst_addr, const uint64_t *dst_token, int flags,
                         srf_batch_t *out) {
  DeviceGuard device_guard;
  if (n < 1) return fail(SRF_E_INVALID_CONFIG, "empty batch");
  int device = src_space[0]->device;
  std::vector<BatchPut> host(n);
  uint32_t next = 0;
  for (int i = 0; i < n; ++i) {
    srf_space *ss = src_space[i], *ds = dst_space[i];
    if (ss->device != device)
      return fail(SRF_E_INVALID_CONFIG, "batch spans GPUs %d and %d", device, ss->device);
    {
      std::lock_guard<std::mutex> g(ss->mu);
      int rc = check_registered_locked(ss, src_addr[i], body_len[i], src_token[i]);
      if (!rc) rc = check_registered_locked(ss, tail_addr[i], 1, src_token[i]);
      if (rc) return rc;
    }
    {
      std::lock_guard<std::mutex> g(ds->mu);
      int rc = check_remote_locked(ds, dst_addr[i], body_len[i] + 1, dst_token[i]);
      if (rc) return rc;
    }
    BatchPut &d = host[i];
    d.src = ss->base + src_addr[i];
    d.dst = ds->base + dst_addr[i];
    d.body = body_len[i];
    d.tail = ss->base + tail_addr[i];
    d.cta_begin = next;
    d.cta_count = ctas_for(device, body_len[i], 128 << 10);
    d.wait_empty = (flags & SRF_PUT_WAIT_EMPTY) ? 1 : 0;
    d.pad = 0;
    next += d.cta_count;
  }
  int rc0 = finish_batch(0, device, host, src_space[0]->err, out);
  if (rc0 == SRF_OK) {
    int sys = 0;
    for (int i = 0; i < n; ++i)
      sys |= (dst_space[i]->imported || dst_space[i]->device != device) ? 1 : 0;
    (*out)->sys = sys;
  }
  return rc0;
}

int srf_batch_gen_create(int n, srf_space_t const *space, const uint64_t *grad_addr,
                         const uint64_t *nbytes, const uint64_t *weight_flag_addr,
                         srf_space_t const *credit_space, const uint64_t *credit_addr,
                         const uint64_t *node_id, uint64_t seed, srf_batch_t *out) {
  DeviceGuard device_guard;
  if (n < 1) return fail(SRF_E_INVALID_CONFIG, "empty batch");
  const int device = space[0]->device;
  std::vector<BatchGen> host(n);
  uint32_t next = 0;
  for (int i = 0; i < n; ++i) {
    srf_space *sp = space[i];
    if (sp->device != device)
      return fail(SRF_E_INVALID_CONFIG, "batch spans GPUs %d and %d", device, sp->device);
    int rc = check_raw(sp, grad_addr[i], nbytes[i], "gradient");
    if (rc) return rc;
    if (grad_addr[i] % 16 || nbytes[i] % 4)
      return fail(SRF_E_SHAPE_MISMATCH, "gradient blocks must be 16-B aligned fp32");
    if (nbytes[i] / 4 > 0xFFFFFFFFull)
      return fail(SRF_E_SHAPE_MISMATCH, "gradient larger than 2^32 elements");
    BatchGen &d = host[i];
    d.grad = sp->base + grad_addr[i];
    d.n = nbytes[i];
    d.weight_flag = weight_flag_addr[i] == UINT64_MAX ? nullptr : sp->base + weight_flag_addr[i];
    d.credit = (credit_space[i] == nullptr || credit_addr[i] == UINT64_MAX)
                   ? nullptr : credit_space[i]->base + credit_addr[i];
    d.node = node_id[i];
    d.cta_begin = next;
    d.cta_count = ctas_for(device, nbytes[i], 128 << 10);
    next += d.cta_count;
  }
  int rc = finish_batch(1, device, host, space[0]->err, out);
  if (rc == SRF_OK) {
    (*out)->seed = seed;
    int sys = 0;
    for (int i = 0; i < n; ++i)
      if (credit_space[i])
        sys |= (credit_space[i]->imported || credit_space[i]->device != device) ? 1 : 0;
    (*out)->sys = sys;
  }
  return rc;
}

int srf_batch_apply_create(srf_space_t sp, int nvars, const uint64_t *var_addr,
                           const uint64_t *nbytes, const int *nworkers, const int *rank,
                           srf_space_t const *src_space, const uint64_t *src_addr,
                           const int *is_meta, srf_space_t const *peer_space,
                           const uint64_t *peer_lo, const uint64_t *peer_hi,
                           const uint64_t *peer_token, int op, float lr, srf_batch_t *out) {
  DeviceGuard device_guard;
  if (nvars < 1) return fail(SRF_E_INVALID_CONFIG, "empty batch");
  if (op != SRF_APPLY_XOR && op != SRF_APPLY_SGD)
    return fail(SRF_E_INVALID_CONFIG, "unknown apply op %d", op);
  std::vector<BatchApply> host(nvars);
  uint32_t next = 0;
  int k = 0;
  for (int v = 0; v < nvars; ++v) {
    BatchApply &d = host[v];
    memset(&d, 0, sizeof d);
    int rc = check_raw(sp, var_addr[v], nbytes[v], "variable");
    if (rc) return rc;
    if (nworkers[v] < 1 || nworkers[v] > SRF_MAX_WORKERS)
      return fail(SRF_E_INVALID_CONFIG, "nworkers %d", nworkers[v]);
    if (op == SRF_APPLY_SGD && (nbytes[v] % 4 || var_addr[v] % 4))
      return fail(SRF_E_SHAPE_MISMATCH, "SGD needs whole fp32 elements");
    d.var = sp->base + var_addr[v];
    d.n = nbytes[v];
    d.nw = nworkers[v];
    d.rank = rank[v];
    for (int w = 0; w < d.nw; ++w, ++k) {
      srf_space *ss = src_space[k];
      if (is_meta[k]) {
        rc = check_raw(ss, src_addr[k], 8 * rank[v] + 33, "meta block");
        if (rc) return rc;
        d.is_meta |= 1u << w;
        d.peer_base[w] = peer_space[k]->base;
        d.peer_lo[w] = peer_lo[k];
        d.peer_hi[w] = peer_hi[k];
        d.peer_token[w] = peer_token[k];
        if (peer_hi[k] > peer_space[k]->capacity)
          return fail(SRF_E_OUT_OF_BOUNDS, "peer region escapes its space");
      } else {
        rc = check_raw(ss, src_addr[k], nbytes[v], "gradient");
        if (rc) return rc;
      }
      d.src[w] = ss->base + src_addr[k];
    }
    d.cta_begin = next;
    d.cta_count = ctas_for(sp->device, nbytes[v] * (uint64_t)(d.nw + 2), 512 << 10);
    next += d.cta_count;
  }
  int rc = finish_batch(2, sp->device, host, sp->err, out);
  if (rc == SRF_OK) {
    (*out)->op = op;
    (*out)->lr = lr;
    int sys = 0;
    for (int i = 0; i < k; ++i)
      if (is_meta[i])
        sys |= (peer_space[i]->imported || peer_space[i]->device != sp->device) ? 1 : 0;
    (*out)->sys = sys;
  }
  return rc;
}

int srf_batch_launch(srf_batch_t b, srf_stream_t st, uint64_t iteration, int mode,
                     int grid_cap) {
  DeviceGuard device_guard;
  const uint64_t timeout = 10ull * 1000 * 1000 * 1000;
  const uint32_t units = (uint32_t)b->grid;
  const int grid = (int)(grid_cap > 0 ? std::min<uint32_t>(units, (uint32_t)grid_cap) : units);
  CUDA_TRY(cudaSetDevice(st->device));
  switch (b->kind) {
    case 0:
      k_put_batch<<<grid, 512, 0, st->s>>>((const BatchPut *)b->descs, b->n, units,
                                           b->counters, timeout, b->err, b->sys);
      return launch_check("k_put_batch");
    case 1:
      k_gen_batch<<<grid, 512, 0, st->s>>>((const BatchGen *)b->descs, b->n, units,
                                           b->counters, b->seed, iteration,
                                           iteration == UINT64_MAX ? b->iter_ptr : nullptr,
                                           mode, timeout, b->err, b->sys);
      return launch_check("k_gen_batch");
    default:
      k_apply_batch<<<grid, 256, 0, st->s>>>((const BatchApply *)b->descs, b->n, units,
                                             b->counters, b->op, b->lr, timeout, b->err, b->sys);
      return launch_check("k_apply_batch");
  }
}

// Device iteration counter for graph-captured PS steps: a gen batch launched
// with iteration == UINT64_MAX reads *counter; srf_counter_add bumps it in
// stream order at the end of a step.
__global__ void k_counter_add(uint64_t *p, uint64_t delta) { *p += delta; }

int srf_batch_set_iteration_source(srf_batch_t b, srf_space_t sp, uint64_t addr) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, 8, "iteration counter");
  if (rc) return rc;
  if (addr % 8) return fail(SRF_E_INVALID_CONFIG, "counter must be 8-B aligned");
  b->iter_ptr = (const uint64_t *)(sp->base + addr);
  return SRF_OK;
}

int srf_counter_add(srf_space_t sp, uint64_t addr, uint64_t delta, srf_stream_t st) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, addr, 8, "counter");
  if (rc) return rc;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  k_counter_add<<<1, 1, 0, s->s>>>((uint64_t *)(sp->base + addr), delta);
  return launch_check("k_counter_add");
}

int srf_ps_persistent(srf_batch_t push, srf_batch_t gen, srf_batch_t meta,
                      srf_batch_t const *apply, int napply, srf_stream_t st, uint64_t it0,
                      uint32_t iters, int mode) {
  DeviceGuard device_guard;
  if (napply < 0 || napply > kMaxApply)
    return fail(SRF_E_INVALID_CONFIG, "at most %d apply batches", kMaxApply);
  srf_batch *all[3] = {push, gen, meta};
  for (srf_batch *b : all)
    if (b && b->device != st->device)
      return fail(SRF_E_INVALID_CONFIG, "persistent PS step needs every batch on one GPU");
  PsPersistArgs a;
  memset(&a, 0, sizeof a);
  if (push) { a.push = (const BatchPut *)push->descs; a.npush = push->n; a.upush = push->grid; a.cpush = push->counters; }
  if (gen) { a.gen = (const BatchGen *)gen->descs; a.ngen = gen->n; a.ugen = gen->grid; a.cgen = gen->counters; a.seed = gen->seed; }
  if (meta) { a.meta = (const BatchPut *)meta->descs; a.nmeta = meta->n; a.umeta = meta->grid; a.cmeta = meta->counters; }
  for (int i = 0; i < napply; ++i) {
    if (apply[i]->device != st->device)
      return fail(SRF_E_INVALID_CONFIG, "persistent PS step needs every batch on one GPU");
    a.apply[i] = (const BatchApply *)apply[i]->descs;
    a.napply[i] = apply[i]->n;
    a.uapply[i] = apply[i]->grid;
    a.capply[i] = apply[i]->counters;
    a.op = apply[i]->op;
    a.lr = apply[i]->lr;
  }
  a.nbatches = napply;
  a.it0 = it0;
  a.iters = iters;
  a.regen = mode;
  a.timeout_ns = 10ull * 1000 * 1000 * 1000;
  a.err = (push ? push : gen ? gen : meta)->err;
  a.sys = 0;
  for (srf_batch *b : all) a.sys |= b ? b->sys : 0;
  for (int i = 0; i < napply; ++i) a.sys |= apply[i]->sys;
  CUDA_TRY(cudaSetDevice(st->device));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ps_persistent, 256, 0));
  if (per_sm < 1) return fail(SRF_E_DEVICE, "persistent PS kernel does not fit an SM");
  // no more CTAs than the busiest phase has work units: grid barriers of a
  // small grid are cheaper (latency-bound configs)
  uint32_t most = 1;
  for (srf_batch *b : all) most = std::max<uint32_t>(most, b ? (uint32_t)b->grid : 0u);
  for (int i = 0; i < napply; ++i) most = std::max<uint32_t>(most, (uint32_t)apply[i]->grid);
  const int grid = (int)std::min<uint32_t>(most, (uint32_t)(per_sm * sm_count_of(st->device)));
  void *params[] = {&a};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_ps_persistent, dim3(grid), dim3(256),
                                       params, 0, st->s));
  return launch_check("k_ps_persistent");
}

int srf_batch_gen_set_ready(srf_batch_t gen, srf_space_t const *space,
                            const uint64_t *ready_addr) {
  if (!gen || gen->kind != 1) return fail(SRF_E_INVALID_CONFIG, "not a gen batch");
  BatchGen *g = (BatchGen *)gen->host.data();
  for (int i = 0; i < gen->n; ++i) {
    if (ready_addr[i] == UINT64_MAX) {
      g[i].ready = nullptr;
      continue;
    }
    int rc = check_raw(space[i], ready_addr[i], 1, "ready flag");
    if (rc) return rc;
    if (g[i].credit) return fail(SRF_E_INVALID_CONFIG, "gen edge %d already has a credit", i);
    g[i].ready = space[i]->base + ready_addr[i];
    g[i].credit = g[i].ready;  // overwrite only after the apply consumed it
  }
  CUDA_TRY(cudaSetDevice(gen->device));
  CUDA_TRY(cudaMemcpy(gen->descs, gen->host.data(), gen->host.size(), cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_batch_apply_set_ready(srf_batch_t apply, srf_space_t space, const uint64_t *ready_addr) {
  if (!apply || apply->kind != 2) return fail(SRF_E_INVALID_CONFIG, "not an apply batch");
  BatchApply *d = (BatchApply *)apply->host.data();
  int k = 0;
  for (int v = 0; v < apply->n; ++v) {
    for (int w = 0; w < d[v].nw; ++w, ++k) {
      if (ready_addr[k] == UINT64_MAX) {
        d[v].ready[w] = nullptr;
        continue;
      }
      if ((d[v].is_meta >> w) & 1)
        return fail(SRF_E_INVALID_CONFIG, "ready flag on a metadata edge (%d)", k);
      int rc = check_raw(space, ready_addr[k], 1, "ready flag");
      if (rc) return rc;
      d[v].ready[w] = space->base + ready_addr[k];
    }
  }
  CUDA_TRY(cudaSetDevice(apply->device));
  CUDA_TRY(cudaMemcpy(apply->descs, apply->host.data(), apply->host.size(),
                      cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_batch_gen_set_offsets(srf_batch_t gen, const uint64_t *elem_offset) {
  DeviceGuard device_guard;
  if (!gen || gen->kind != 1) return fail(SRF_E_INVALID_CONFIG, "not a gen batch");
  BatchGen *g = (BatchGen *)gen->host.data();
  for (int i = 0; i < gen->n; ++i) {
    if (elem_offset[i] + g[i].n / 4 > 0xFFFFFFFFull)
      return fail(SRF_E_SHAPE_MISMATCH, "gradient element index beyond 2^32");
    g[i].elem_offset = elem_offset[i];
  }
  CUDA_TRY(cudaSetDevice(gen->device));
  CUDA_TRY(cudaMemcpy(gen->descs, gen->host.data(), gen->host.size(), cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_batch_gen_set_meta(srf_batch_t gen, int n, const int *gen_index, srf_batch_t meta) {
  DeviceGuard device_guard;
  if (!gen || gen->kind != 1 || !meta || meta->kind != 0 || n != meta->n)
    return fail(SRF_E_INVALID_CONFIG, "gen_set_meta: a gen batch and a put batch of n edges");
  BatchGen *g = (BatchGen *)gen->host.data();
  const BatchPut *m = (const BatchPut *)meta->host.data();
  for (int i = 0; i < n; ++i) {
    if (gen_index[i] < 0 || gen_index[i] >= gen->n)
      return fail(SRF_E_INVALID_CONFIG, "gen_set_meta: index %d out of range", gen_index[i]);
    BatchGen &d = g[gen_index[i]];
    d.meta_src = m[i].src;
    d.meta_dst = m[i].dst;
    d.meta_tail = m[i].tail;
    d.meta_body = m[i].body;
  }
  gen->sys |= meta->sys;
  CUDA_TRY(cudaSetDevice(gen->device));
  CUDA_TRY(cudaMemcpy(gen->descs, gen->host.data(), gen->host.size(), cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_batch_destroy(srf_batch_t b) {
  DeviceGuard device_guard;
  if (!b) return SRF_OK;
  cudaSetDevice(b->device);
  cudaFree(b->descs);
  cudaFree(b->counters);
  delete b;
  return SRF_OK;
}

// ---------------------------------------------------------------------------
// exchange schedule (k_ps_exchange)
// ---------------------------------------------------------------------------
struct srf_exchange {
  int device;
  ExArgs args;
  ExItem *items = nullptr;
  unsigned int *ctr = nullptr;  // [claim, exit_count]
  unsigned int *done = nullptr; // completions per descriptor this launch: [apply|push|gen]
  int ndone = 0, napply_descs = 0;
  int *push_done = nullptr;
  int grid = 0;
};

int srf_ps_exchange_create(srf_batch_t push, const uint64_t *push_key, srf_batch_t gen,
                           const uint64_t *gen_key, srf_batch_t const *apply, int napply,
                           const uint64_t *apply_key, srf_exchange_t *out) {
  DeviceGuard device_guard;
  if (napply < 0 || napply > kMaxApply)
    return fail(SRF_E_INVALID_CONFIG, "at most %d apply batches", kMaxApply);
  if ((push && push->kind != 0) || (gen && gen->kind != 1))
    return fail(SRF_E_INVALID_CONFIG, "exchange: batch kinds");
  int device = push ? push->device : gen ? gen->device : napply ? apply[0]->device : -1;
  if (device < 0) return fail(SRF_E_INVALID_CONFIG, "exchange: no batches");
  struct K { uint64_t key; uint32_t kind, batch, desc, unit; };
  std::vector<K> ks;
  auto add = [&](srf_batch *b, const uint64_t *key, uint32_t kind, uint32_t batch) -> int {
    if (!b) return SRF_OK;
    if (b->device != device) return fail(SRF_E_INVALID_CONFIG, "exchange spans GPUs");
    for (int i = 0; i < b->n; ++i) {
      uint32_t begin, count;
      if (kind == 0) {
        const BatchPut &d = ((const BatchPut *)b->host.data())[i];
        begin = d.cta_begin; count = d.cta_count;
      } else if (kind == 1) {
        const BatchGen &d = ((const BatchGen *)b->host.data())[i];
        begin = d.cta_begin; count = d.cta_count;
        if (d.credit && d.credit != d.ready && !d.meta_dst)
          return fail(SRF_E_INVALID_CONFIG, "exchange: gen edge %d has no fused meta", i);
      } else {
        const BatchApply &d = ((const BatchApply *)b->host.data())[i];
        begin = d.cta_begin; count = d.cta_count;
      }
      for (uint32_t u = 0; u < count; ++u) ks.push_back({key[i], kind, batch, (uint32_t)i, begin + u});
    }
    return SRF_OK;
  };
  int rc = add(push, push_key, 0, 0);
  if (!rc) rc = add(gen, gen_key, 1, 0);
  uint64_t off = 0;
  for (int b = 0; !rc && b < napply; ++b) {
    if (apply[b]->kind != 2) return fail(SRF_E_INVALID_CONFIG, "exchange: batch kinds");
    rc = add(apply[b], apply_key + off, 2, (uint32_t)b);
    off += apply[b]->n;
  }
  if (rc) return rc;
  std::stable_sort(ks.begin(), ks.end(), [](const K &x, const K &y) {
    if (x.key != y.key) return x.key < y.key;
    if (x.kind != y.kind) return x.kind < y.kind;
    if (x.batch != y.batch) return x.batch < y.batch;
    return x.desc < y.desc;
  });
  std::vector<ExItem> items(ks.size());
  for (size_t i = 0; i < ks.size(); ++i)
    items[i] = {ks[i].unit, (uint16_t)ks[i].kind, (uint16_t)ks[i].batch};
  srf_exchange *x = new srf_exchange();
  x->device = device;
  memset(&x->args, 0, sizeof x->args);
  ExArgs &a = x->args;
  if (push) { a.push = (const BatchPut *)push->descs; a.npush = push->n; a.cpush = push->counters; a.push_sys = push->sys; }
  if (gen) { a.gen = (const BatchGen *)gen->descs; a.ngen = gen->n; a.cgen = gen->counters; a.seed = gen->seed; a.gen_sys = gen->sys; }
  int nd = 0;
  for (int b = 0; b < napply; ++b) {
    a.apply_base[b] = nd;
    nd += apply[b]->n;
    a.apply[b] = (const BatchApply *)apply[b]->descs;
    a.napply[b] = apply[b]->n;
    a.capply[b] = apply[b]->counters;
    a.apply_sys[b] = apply[b]->sys;
    a.op = apply[b]->op;
    a.lr = apply[b]->lr;
  }
  a.err = push ? push->err : gen ? gen->err : apply[0]->err;
  a.nitems = (uint32_t)items.size();
  a.timeout_ns = 10ull * 1000 * 1000 * 1000;
  CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMalloc(&x->items, sizeof(ExItem) * std::max<size_t>(1, items.size()));
  if (e == cudaSuccess && !items.empty())
    e = cudaMemcpy(x->items, items.data(), sizeof(ExItem) * items.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&x->ctr, 2 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(x->ctr, 0, 2 * sizeof(unsigned int));
  const int np = a.npush, ng = a.ngen;
  x->ndone = std::max(nd + np + ng, 1);
  if (e == cudaSuccess) e = cudaMalloc(&x->done, sizeof(unsigned int) * x->ndone);
  if (e == cudaSuccess) e = cudaMemset(x->done, 0, sizeof(unsigned int) * x->ndone);
  if (e == cudaSuccess) e = cudaMalloc(&x->push_done, sizeof(int) * std::max(1, a.npush));
  if (e == cudaSuccess) e = cudaMemset(x->push_done, 0xff, sizeof(int) * std::max(1, a.npush));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  int per_sm = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ps_exchange, 512, 0);
  if (e != cudaSuccess) {
    cudaFree(x->items);
    cudaFree(x->ctr);
    cudaFree(x->done);
    cudaFree(x->push_done);
    delete x;
    return fail(SRF_E_DEVICE, "exchange: %s", cudaGetErrorString(e));
  }
  a.items = x->items;
  a.claim = x->ctr;
  a.exit_count = x->ctr + 1;
  a.done = x->done;
  a.push_done = x->push_done;
  a.seq_push = np ? x->done + nd : nullptr;
  a.seq_gen = ng ? x->done + nd + np : nullptr;
  x->napply_descs = nd;
  a.iters = 1;
  x->grid = sm_count_of(device) * std::max(1, per_sm);
  *out = x;
  return SRF_OK;
}

int srf_ps_exchange_link(srf_exchange_t x, const int *push_apply_index) {
  DeviceGuard device_guard;
  std::vector<int> m(std::max(1, x->args.npush));
  for (int i = 0; i < x->args.npush; ++i) {
    if (push_apply_index[i] < -1 || push_apply_index[i] >= x->napply_descs)
      return fail(SRF_E_INVALID_CONFIG, "exchange_link: index %d", push_apply_index[i]);
    m[i] = push_apply_index[i];
  }
  CUDA_TRY(cudaSetDevice(x->device));
  CUDA_TRY(cudaMemcpy(x->push_done, m.data(), sizeof(int) * m.size(), cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_ps_exchange_launch_n(srf_exchange_t x, srf_stream_t st, uint64_t iteration,
                             uint32_t iterations, int regen) {
  DeviceGuard device_guard;
  if (st->device != x->device) return fail(SRF_E_INVALID_CONFIG, "exchange: stream GPU");
  if (iterations < 1) return fail(SRF_E_INVALID_CONFIG, "exchange: iterations >= 1");
  if ((uint64_t)x->args.nitems * iterations > 0xFFFFFFFFull)
    return fail(SRF_E_INVALID_CONFIG, "exchange: too many units for one launch");
  x->args.iteration = iteration;
  x->args.regen = regen;
  x->args.iters = iterations;
  CUDA_TRY(cudaSetDevice(x->device));
  if (iterations > 1)
    CUDA_TRY(cudaMemsetAsync(x->done, 0, sizeof(unsigned int) * x->ndone, st->s));
  k_ps_exchange<<<x->grid, 512, 0, st->s>>>(x->args);
  return launch_check("k_ps_exchange");
}

int srf_ps_exchange_launch(srf_exchange_t x, srf_stream_t st, uint64_t iteration, int regen) {
  return srf_ps_exchange_launch_n(x, st, iteration, 1, regen);
}

int srf_ps_exchange_destroy(srf_exchange_t x) {
  DeviceGuard device_guard;
  if (!x) return SRF_OK;
  cudaSetDevice(x->device);
  cudaFree(x->items);
  cudaFree(x->ctr);
  cudaFree(x->done);
  cudaFree(x->push_done);
  delete x;
  return SRF_OK;
}

// ---------------------------------------------------------------------------
// doorbells (host-visible receive flags)
// ---------------------------------------------------------------------------
int srf_doorbell_bind(srf_space_t sp, uint64_t region_addr, uint64_t region_len, int mirror) {
  DeviceGuard device_guard;
  if (region_len < 1) return fail(SRF_E_ZERO_LENGTH, "doorbell region must be >= 1 byte");
  int rc = check_raw(sp, region_addr, region_len, "doorbell region");
  if (rc) return rc;
  if (sp->imported) return fail(SRF_E_INVALID_CONFIG, "doorbells live with the receiver");
  std::lock_guard<std::mutex> g(sp->mu);
  if (!sp->db) {
    sp->db_cap = 1 << 20;
    CUDA_TRY(cudaSetDevice(sp->device));
    CUDA_TRY(cudaHostAlloc((void **)&sp->db_host, sp->db_cap,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    memset(sp->db_host, 0, sp->db_cap);
    CUDA_TRY(cudaHostGetDevicePointer((void **)&sp->db_dev, sp->db_host, 0));
    sp->db = new std::unordered_map<uint64_t, Doorbell>();
  }
  const uint64_t tail = region_addr + region_len - 1;
  if (sp->db->count(tail)) return SRF_OK;
  const uint64_t need = mirror ? region_len : 1;
  if (sp->db_used + need > sp->db_cap) return fail(SRF_E_OUT_OF_MEMORY, "doorbell page full");
  Doorbell d;
  d.region_addr = region_addr;
  d.region_len = region_len;
  d.mirror = mirror != 0;
  d.shadow_len = need;
  d.host_off = sp->db_used;
  d.clear_pending = false;
  CUDA_TRY(cudaSetDevice(sp->device));  // the event lives on the space's GPU
  CUDA_TRY(cudaEventCreateWithFlags(&d.clear_ev, cudaEventDisableTiming));
  // initial shadow = current device bytes
  std::vector<uint8_t> cur(need);
  CUDA_TRY(cudaMemcpy(cur.data(), sp->base + tail + 1 - need, need, cudaMemcpyDeviceToHost));
  memcpy(sp->db_host + sp->db_used, cur.data(), need);
  sp->db_used += need;
  (*sp->db)[tail] = d;
  return SRF_OK;
}

// Read `len` bytes ending at tail_addr + 1: from the doorbell shadow when one
// is bound and every producer is in this process, else from the device.
int srf_flag_read(srf_space_t sp, uint64_t tail_addr, uint64_t len, void *host_out) {
  DeviceGuard device_guard;
  if (sp->db && !sp->exported) {
    std::lock_guard<std::mutex> g(sp->mu);
    auto it = sp->db->find(tail_addr);
    if (it != sp->db->end()) {
      const Doorbell &d = it->second;
      if (len <= d.shadow_len) {
        const volatile uint8_t *src = sp->db_host + d.host_off + (d.shadow_len - len);
        // flag byte first (acquire), then the rest
        uint8_t *o = (uint8_t *)host_out;
        o[len - 1] = src[len - 1];
        std::atomic_thread_fence(std::memory_order_acquire);
        for (uint64_t i = 0; i + 1 < len; ++i) o[i] = src[i];
        return SRF_OK;
      }
    }
  }
  return srf_read(sp, tail_addr + 1 - len, len, host_out);
}

// Clear a receive flag (StaticReceiver/DynReceiver.poll): shadow now, device
// byte asynchronously on the space's stream; the next srf_put into the region
// waits for that clear.
int srf_flag_clear(srf_space_t sp, uint64_t tail_addr) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, tail_addr, 1, "flag");
  if (rc) return rc;
  if (sp->db) {
    std::lock_guard<std::mutex> g(sp->mu);
    auto it = sp->db->find(tail_addr);
    if (it != sp->db->end()) {
      Doorbell &d = it->second;
      volatile uint8_t *flag = sp->db_host + d.host_off + d.shadow_len - 1;
      *flag = 0;
      CUDA_TRY(cudaSetDevice(sp->device));
      CUDA_TRY(cudaMemsetAsync(sp->base + tail_addr, 0, 1, sp->stream->s));
      CUDA_TRY(cudaEventRecord(d.clear_ev, sp->stream->s));
      d.clear_pending = true;
      return SRF_OK;
    }
  }
  const uint8_t z = 0;
  return srf_write(sp, tail_addr, 1, &z);
}

int srf_rpc_transfer(srf_space_t src, uint64_t meta_addr, uint32_t meta_len,
                     uint64_t payload_addr, uint64_t payload_len, uint64_t stage_addr,
                     srf_space_t dst, uint64_t ring_addr, uint64_t ring_flags_addr,
                     uint64_t meta_out_addr, uint64_t tensor_out_addr, uint64_t msg_id,
                     srf_stream_t st_src, srf_stream_t st_dst) {
  DeviceGuard device_guard;
  int rc = check_raw(src, meta_addr, meta_len, "rpc meta");
  if (!rc) rc = check_raw(src, payload_addr, payload_len, "rpc payload");
  if (!rc) rc = check_raw(src, stage_addr, (uint64_t)kRing * kFrag, "rpc stage");
  if (!rc) rc = check_raw(dst, ring_addr, (uint64_t)kRing * kFrag, "rpc ring");
  if (!rc) rc = check_raw(dst, ring_flags_addr, kRing, "rpc ring flags");
  if (!rc) rc = check_raw(dst, meta_out_addr, meta_len, "rpc meta out");
  if (!rc) rc = check_raw(dst, tensor_out_addr, payload_len, "rpc tensor out");
  if (rc) return rc;
  RpcArgs a;
  a.meta = src->base + meta_addr;
  a.meta_len = meta_len;
  a.payload = src->base + payload_addr;
  a.pay_len = payload_len;
  a.stage = src->base + stage_addr;
  a.ring = dst->base + ring_addr;
  a.ring_flags = dst->base + ring_flags_addr;
  a.meta_out = dst->base + meta_out_addr;
  a.tensor_out = dst->base + tensor_out_addr;
  a.msg_id = msg_id;
  a.timeout_ns = 10ull * 1000 * 1000 * 1000;
  a.err = src->err;
  srf_stream *ss = stream_or_default(src, st_src);
  srf_stream *ds = stream_or_default(dst, st_dst);
  if (ss->device == ds->device) {
    // both roles in one cooperative launch: the two CTAs are co-resident
    a.role = -1;
    CUDA_TRY(cudaSetDevice(ss->device));
    void *params[] = {&a};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_rpc, dim3(2), dim3(1024), params, 0,
                                         ss->s));
    return launch_check("k_rpc");
  }
  // two GPUs: receiver first (it waits for the sender over NVLink)
  a.role = 1;
  a.err = dst->err;
  CUDA_TRY(cudaSetDevice(ds->device));
  k_rpc<<<1, 1024, 0, ds->s>>>(a);
  rc = launch_check("k_rpc(recv)");
  if (rc) return rc;
  a.role = 0;
  a.err = src->err;
  CUDA_TRY(cudaSetDevice(ss->device));
  k_rpc<<<1, 1024, 0, ss->s>>>(a);
  return launch_check("k_rpc(send)");
}

int srf_graph_begin(srf_stream_t st) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  CUDA_TRY(cudaStreamBeginCapture(st->s, cudaStreamCaptureModeThreadLocal));
  return SRF_OK;
}

int srf_graph_end(srf_stream_t st, void **graph_exec) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamEndCapture(st->s, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess)
    return fail(SRF_E_DEVICE, "graph instantiate: %s", cudaGetErrorString(e));
  *graph_exec = (void *)ex;
  return SRF_OK;
}

int srf_graph_launch(void *graph_exec, srf_stream_t st) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)graph_exec, st->s));
  return SRF_OK;
}

int srf_graph_destroy(void *graph_exec) {
  DeviceGuard device_guard;
  if (graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)graph_exec);
  return SRF_OK;
}

int srf_stream_wait_event(srf_stream_t st, srf_event_t ev) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  CUDA_TRY(cudaStreamWaitEvent(st->s, ev->e, 0));
  return SRF_OK;
}

int srf_timing_event_create(srf_space_t sp, srf_event_t *out) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(sp->device));
  srf_event *ev = new srf_event();
  ev->device = sp->device;
  cudaError_t e = cudaEventCreate(&ev->e);
  if (e != cudaSuccess) {
    delete ev;
    return fail(SRF_E_DEVICE, "event: %s", cudaGetErrorString(e));
  }
  *out = ev;
  return SRF_OK;
}

int srf_event_record_on(srf_event_t ev, srf_stream_t st) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(st->device));
  CUDA_TRY(cudaEventRecord(ev->e, st->s));
  return SRF_OK;
}

int srf_event_elapsed_ms(srf_event_t start, srf_event_t end, float *ms) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaEventElapsedTime(ms, start->e, end->e));
  return SRF_OK;
}

}  // extern "C"
