// device_copy.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Device helpers (acquire/release PTX, grid arrival, 256-bit vectors) and the transfer kernels: K1 put (+ TMA bulk variant), pool zero-fill, K2 flag wait, release/acquire consumer.

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

// Arrival that also counts aborted CTAs (a timed-out credit): an aborted CTA
// adds kAbortUnit, so the last arriver knows whether any CTA skipped its
// share - then the tail byte is NOT released (the put did not happen as a
// whole; the host sees the timeout).  Grids stay far below 2^20 CTAs.
static constexpr unsigned kAbortUnit = 1u << 20;

// Acquire-spin until the receive region's flag reads 0 (the receiver's
// credit); false (and err = 2) on timeout.
__device__ __forceinline__ bool credit_wait(const uint8_t *flag, uint64_t timeout_ns, int *err) {
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys_u8(flag) != 0) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(err, 2);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

__device__ __forceinline__ bool grid_arrive_abort(unsigned int *counter, unsigned expected_last,
                                                  int sys_scope, bool aborted, bool *any_abort) {
  const unsigned inc = 1u + (aborted ? kAbortUnit : 0u);
  unsigned prev;
  if (sys_scope)
    asm volatile("atom.add.acq_rel.sys.u32 %0, [%1], %2;" : "=r"(prev) : "l"(counter), "r"(inc) : "memory");
  else
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(prev) : "l"(counter), "r"(inc) : "memory");
  *any_abort = aborted || (prev >= kAbortUnit);
  return (prev & (kAbortUnit - 1)) == expected_last;
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

// Coherent (L2, .cg) 256-bit load: for sources written earlier in the same
// launch (the multi-iteration PS exchange pushes variables its own apply
// units updated) or by another agent while the kernel runs (RPC ring slots).
// The non-coherent .nc path is only valid for data read-only for the launch.
__device__ __forceinline__ u256 ld_cg_v8(const u256 *p) {
  u256 r;
  asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                 "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7])
               : "l"(p));
  return r;
}

// Source loads: kCoh = false -> read-only-for-the-launch paths (.nc / __ldg);
// kCoh = true -> coherent at L2 (__ldcg / ld.global.cg).
template <typename V, bool kCoh = false>
__device__ __forceinline__ V ld_stream(const V *p) {
  if (kCoh) return __ldcg(p);
  return __ldg(p);
}
template <>
__device__ __forceinline__ u256 ld_stream<u256, false>(const u256 *p) {
  return ld_v8(p);
}
template <>
__device__ __forceinline__ u256 ld_stream<u256, true>(const u256 *p) {
  return ld_cg_v8(p);
}
template <>
__device__ __forceinline__ uint4 ld_stream<uint4, false>(const uint4 *p) {
  return ld_stream_v4(p);
}
template <bool kCoh>
__device__ __forceinline__ uint8_t ld_byte(const uint8_t *p) {
  if (kCoh) return (uint8_t)__ldcg((const unsigned char *)p);
  return *p;
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
template <typename V, int U, bool kCoh = false>
__device__ __forceinline__ void vec_copy(V *__restrict__ dst,
                                         const V *__restrict__ src,
                                         uint64_t nv, uint64_t t,
                                         uint64_t nth) {
  uint64_t i = t;
  for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_stream<V, kCoh>(src + i + u * nth);
#pragma unroll
    for (int u = 0; u < U; ++u) st_plain<V>(dst + i + u * nth, r[u]);
  }
  for (; i < nv; i += nth) st_plain<V>(dst + i, ld_stream<V, kCoh>(src + i));
}

__device__ __forceinline__ u256 pack8(const uint2 (&a)[4]) {
  u256 r;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r.v[2 * k] = a[k].x;
    r.v[2 * k + 1] = a[k].y;
  }
  return r;
}

// Destination-aligned copy for large ranges whose ends are not co-aligned mod
// 32 (arena blocks are only 8-B aligned, memspace.py:31): every store is one
// whole, aligned 32-B sector - partial-sector stores cost NVLink bandwidth
// (K1 at a destination 8 B off a sector: 495 vs 694 GB/s, 4 B off: 378;
// profiles/r1_align_probe.txt) - and the source is read at its own alignment
// class (8-B, 4-B, or aligned words funnel-shifted) and reassembled in
// registers.  U chunks of 32 B in flight per thread.
template <int U, bool kCoh = false>
__device__ void copy_dst_aligned(uint8_t *dst, const uint8_t *src, uint64_t n, uint64_t t,
                                 uint64_t nth) {
  uint64_t head = (32 - ((uintptr_t)dst & 31)) & 31;
  if (head > n) head = n;
  const uint8_t *sp = src + head;
  u256 *D = (u256 *)(dst + head);
  uint64_t nv = (n - head) / 32;
  const uint32_t sa = (uint32_t)((uintptr_t)sp & 7);
  if (sa == 0) {
    const uint2 *S8 = (const uint2 *)sp;
    uint64_t i = t;
    for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
      uint2 a[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k) a[u][k] = ld_stream<uint2, kCoh>(S8 + 4 * (i + u * nth) + k);
#pragma unroll
      for (int u = 0; u < U; ++u) st_v8(D + i + u * nth, pack8(a[u]));
    }
    for (; i < nv; i += nth) {
      uint2 a[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] = ld_stream<uint2, kCoh>(S8 + 4 * i + k);
      st_v8(D + i, pack8(a));
    }
  } else {
    // 4-B aligned source: plain words; otherwise aligned words funnel-shifted
    // by m bytes (chunk i reads words 8i .. 8i+8, the ninth reaching up to 3
    // bytes past the chunk: the last chunk is left to the scalar tail)
    const uint32_t m = (uint32_t)((uintptr_t)sp & 3);
    const uint32_t *sw = (const uint32_t *)((uintptr_t)sp - m);
    if (m && nv) nv -= 1;
    uint64_t i = t;
    for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
      uint32_t w[U][9];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < 9; ++k)
          w[u][k] = (k < 8 || m) ? ld_stream<uint32_t, kCoh>(sw + 8 * (i + u * nth) + k) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        u256 r;
#pragma unroll
        for (int k = 0; k < 8; ++k) r.v[k] = __funnelshift_r(w[u][k], w[u][k + 1], 8 * m);
        st_v8(D + i + u * nth, r);
      }
    }
    for (; i < nv; i += nth) {
      uint32_t w[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) w[k] = (k < 8 || m) ? ld_stream<uint32_t, kCoh>(sw + 8 * i + k) : 0u;
      u256 r;
#pragma unroll
      for (int k = 0; k < 8; ++k) r.v[k] = __funnelshift_r(w[k], w[k + 1], 8 * m);
      st_v8(D + i, r);
    }
  }
  for (uint64_t j = t; j < head; j += nth) dst[j] = ld_byte<kCoh>(src + j);
  for (uint64_t j = head + 32 * nv + t; j < n; j += nth) dst[j] = ld_byte<kCoh>(src + j);
}

// Source-aligned twin for pulls (the source is a peer's memory): whole
// aligned 32-B sector loads, stores at the destination's alignment (8-B or
// 4-B words; callers guarantee (dst - src) % 4 == 0).  A pull whose source
// sat 8 B off a sector ran at 571 GB/s instead of 736 (r1_align_probe.txt).
template <int U, bool kCoh = false>
__device__ void copy_src_aligned(uint8_t *dst, const uint8_t *src, uint64_t n, uint64_t t,
                                 uint64_t nth) {
  uint64_t head = (32 - ((uintptr_t)src & 31)) & 31;
  if (head > n) head = n;
  const u256 *S = (const u256 *)(src + head);
  uint8_t *dp = dst + head;
  const uint64_t nv = (n - head) / 32;
  const bool w8 = ((uintptr_t)dp & 7) == 0;
  uint64_t i = t;
  for (; i + (uint64_t)(U - 1) * nth < nv; i += (uint64_t)U * nth) {
    u256 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_stream<u256, kCoh>(S + i + u * nth);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (w8) {
        uint2 *D8 = (uint2 *)dp + 4 * (i + u * nth);
#pragma unroll
        for (int k = 0; k < 4; ++k) D8[k] = make_uint2(r[u].v[2 * k], r[u].v[2 * k + 1]);
      } else {
        uint32_t *D4 = (uint32_t *)dp + 8 * (i + u * nth);
#pragma unroll
        for (int k = 0; k < 8; ++k) D4[k] = r[u].v[k];
      }
    }
  }
  for (; i < nv; i += nth) {
    const u256 r = ld_stream<u256, kCoh>(S + i);
    if (w8) {
      uint2 *D8 = (uint2 *)dp + 4 * i;
#pragma unroll
      for (int k = 0; k < 4; ++k) D8[k] = make_uint2(r.v[2 * k], r.v[2 * k + 1]);
    } else {
      uint32_t *D4 = (uint32_t *)dp + 8 * i;
#pragma unroll
      for (int k = 0; k < 8; ++k) D4[k] = r.v[k];
    }
  }
  for (uint64_t j = t; j < head; j += nth) dst[j] = ld_byte<kCoh>(src + j);
  for (uint64_t j = head + 32 * nv + t; j < n; j += nth) dst[j] = ld_byte<kCoh>(src + j);
}

// Copy n bytes with the widest vector both pointers allow.  Arena blocks are
// 8-byte aligned (memspace.py:31), so the 16-B path needs equal (p mod 16).
// Large copies that are not co-aligned mod 32 keep one side in whole aligned
// 32-B sectors: the destination for puts (align_dst, often a peer's memory),
// the source for pulls (!align_dst, reading a peer's memory).
// kSectors = false compiles only the co-aligned classes (PS blocks).
__constant__ int g_vec32 = 1;  // knob 5: 32-B vectors when co-aligned mod 32

template <int U16 = 4, bool kSectors = true, bool kCoh = false>
__device__ void copy_bytes_grid(uint8_t *dst, const uint8_t *src, uint64_t n,
                                uint64_t t, uint64_t nth, bool align_dst = true) {
  if (n == 0) return;
  uintptr_t d = (uintptr_t)dst, s = (uintptr_t)src;
  uint64_t head, nv;
  if (kSectors && g_vec32 && ((d ^ s) & 31) != 0 && n >= 4096) {
    if (align_dst) {
      copy_dst_aligned<(U16 > 4 ? U16 / 2 : 2), kCoh>(dst, src, n, t, nth);
      return;
    }
    if (((d ^ s) & 3) == 0) {
      copy_src_aligned<(U16 > 4 ? U16 / 2 : 2), kCoh>(dst, src, n, t, nth);
      return;
    }
  }
  if (g_vec32 && ((d ^ s) & 31) == 0 && n >= 4096) {
    head = (32 - (d & 31)) & 31;
    if (head > n) head = n;
    nv = (n - head) / 32;
    vec_copy<u256, (U16 > 4 ? U16 / 2 : 2), kCoh>((u256 *)(dst + head), (const u256 *)(src + head),
                                            nv, t, nth);
    nv *= 32;
  } else if (((d ^ s) & 15) == 0) {
    head = (16 - (d & 15)) & 15;
    if (head > n) head = n;
    nv = (n - head) / 16;
    vec_copy<uint4, U16, kCoh>((uint4 *)(dst + head), (const uint4 *)(src + head), nv,
                         t, nth);
    nv *= 16;
  } else if (((d ^ s) & 7) == 0) {
    head = (8 - (d & 7)) & 7;
    if (head > n) head = n;
    nv = (n - head) / 8;
    vec_copy<uint2, 8, kCoh>((uint2 *)(dst + head), (const uint2 *)(src + head), nv,
                       t, nth);
    nv *= 8;
  } else if (((d ^ s) & 3) == 0) {
    head = (4 - (d & 3)) & 3;
    if (head > n) head = n;
    nv = (n - head) / 4;
    vec_copy<uint32_t, 8, kCoh>((uint32_t *)(dst + head),
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
        a[u] = ld_stream<uint32_t, kCoh>(sw + j + u * nth);
        b[u] = ld_stream<uint32_t, kCoh>(sw + j + u * nth + 1);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dw[j + u * nth] = __funnelshift_r(a[u], b[u], 8 * m);
    }
    for (; j < nv; j += nth)
      dw[j] = __funnelshift_r(ld_stream<uint32_t, kCoh>(sw + j), ld_stream<uint32_t, kCoh>(sw + j + 1),
                              8 * m);
    nv *= 4;
  }
  // scalar head and tail bytes
  for (uint64_t i = t; i < head; i += nth) dst[i] = ld_byte<kCoh>(src + i);
  for (uint64_t i = head + nv + t; i < n; i += nth) dst[i] = ld_byte<kCoh>(src + i);
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
  int src_remote;        // 1: a pull (K4) - keep the peer-side source reads aligned
  int wait_empty;        // 1: spin until dst[total-1] == 0 before writing
  int sys_scope;         // 1: destination is a peer's memory (system-scope release)
  uint8_t *db;           // host-mapped doorbell shadow (nullptr: none)
  uint32_t db_len;       // bytes mirrored (1: tail flag only; total: whole block)
  uint64_t timeout_ns;
  unsigned int *counter; // arrival counter (per stream, reset by last CTA)
  int *err;
  uint8_t *consume;      // srf_put_consume: this rank's receive flag to poll and clear
};

// K1 static_put / K3 meta_put / K4 peer_pull / K5 stage_copy.
// kSectors: the variant for gather lists that are not co-aligned mod 32
// (whole-sector realignment, copy_dst_aligned / copy_src_aligned); the
// co-aligned variant keeps the lean register budget of the plain paths.
template <int U16, bool kSectors>
__device__ __forceinline__ void put_body(const PutArgs &a) {
  __shared__ int s_last, s_abort;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t *tail = a.dst + a.total - 1;

  if (threadIdx.x == 0) {
    s_abort = 0;
    // credit check of the iteration barrier (runtime/protocol.py:102-111):
    // the receiver must have cleared the previous transfer's flag.  A CTA
    // whose wait times out writes nothing, and the tail is then withheld.
    if (a.wait_empty) s_abort = credit_wait(tail, a.timeout_ns, a.err) ? 0 : 1;
  }
  __syncthreads();

  // body: every byte except the tail one when tail_release is set
  if (!s_abort) {
    uint64_t body = a.tail_release ? a.total - 1 : a.total;
    for (int i = 0; i < a.nseg; ++i) {
      const Seg &sg = a.seg[i];
      if (sg.dst_off >= body) break;
      uint64_t n = sg.len;
      if (sg.dst_off + n > body) n = body - sg.dst_off;
      copy_bytes_grid<U16, kSectors>(a.dst + sg.dst_off, sg.src, n, t, nth, !a.src_remote);
    }
  }

  if (!a.tail_release) return;
  // flag-last: all CTAs publish, the last to arrive releases the tail byte.
  __syncthreads();
  if (threadIdx.x == 0) {
    bool any_abort;
    s_last = grid_arrive_abort(a.counter, gridDim.x - 1, a.sys_scope, s_abort, &any_abort);
    if (s_last && any_abort) {
      atomicExch(a.counter, 0u);  // re-armed; no tail, no doorbell, no consume
      s_last = 0;
    }
  }
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
    if (a.consume) {
      // K2 fused: this rank's receive flag (StaticReceiver.poll on the device)
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u8(a.consume) != 1) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicExch(a.err, 1);
          break;
        }
        __nanosleep(32);
      }
      st_relaxed_sys_u8(a.consume, 0);
    }
  }
}

template <int U16, bool kSectors>
__global__ void __launch_bounds__(512) k_put(const __grid_constant__ PutArgs a) {
  put_body<U16, kSectors>(a);
}


// K3 with the metadata block inline (DynSender.send, protocol.py:163-201):
// the 8D+33 bytes travel as a kernel parameter - no host-to-device staging
// copy - and one CTA writes them into the sender's registered meta stage
// (write_at(meta_stage), as the reference keeps them) and into the
// receiver's block, flag byte released last (plus the host doorbell mirror).
static constexpr int kInlineMax = 1024;

struct InlineArgs {
  uint8_t bytes[kInlineMax];
  uint32_t len;
  uint8_t *stage;         // sender's meta stage (local)
  uint8_t *dst;           // receiver's block (peer or local)
  int sys_scope;
  int wait_empty;
  uint8_t *db;            // host-mapped doorbell shadow (nullptr: none)
  uint32_t db_len;
  uint64_t timeout_ns;
  int *err;
};

__device__ __forceinline__ void put_inline_body(const InlineArgs &a) {
  __shared__ int s_abort;
  uint8_t *tail = a.dst + a.len - 1;
  if (threadIdx.x == 0) s_abort = (a.wait_empty && !credit_wait(tail, a.timeout_ns, a.err)) ? 1 : 0;
  __syncthreads();
  if (s_abort) return;
  for (uint32_t i = threadIdx.x; i < a.len; i += blockDim.x) {
    a.stage[i] = a.bytes[i];
    if (i + 1 < a.len) a.dst[i] = a.bytes[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // release is cumulative over the CTA's stores ordered before it by bar.sync
    const uint32_t v = a.bytes[a.len - 1];
    release_tail(tail, v, a.sys_scope);
    if (a.db) {
      for (uint32_t i = 0; i + 1 < a.db_len; ++i) a.db[i] = a.bytes[a.len - a.db_len + i];
      __threadfence_system();
      st_release_sys_u8(a.db + a.db_len - 1, v);
    }
  }
}

__global__ void __launch_bounds__(256) k_put_inline(const __grid_constant__ InlineArgs a) {
  put_inline_body(a);
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
  __shared__ int s_last, s_abort;
  uint64_t *bars = (uint64_t *)(smem + kBulkChunk * kBulkStages);
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t *tail = a.dst + a.total - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_abort = (a.wait_empty && !credit_wait(tail, a.timeout_ns, a.err)) ? 1 : 0;
  }
  __syncthreads();
  uint64_t body = a.tail_release ? a.total - 1 : a.total;
  if (s_abort) body = 0;  // timed-out credit: write nothing
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
      copy_bytes_grid(d, s, n, t, nth, !a.src_remote);
    }
  }
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (!a.tail_release) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    bool any_abort;
    s_last = grid_arrive_abort(a.counter, gridDim.x - 1, a.sys_scope, s_abort, &any_abort);
    if (s_last && any_abort) {
      atomicExch(a.counter, 0u);
      s_last = 0;
    }
  }
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
