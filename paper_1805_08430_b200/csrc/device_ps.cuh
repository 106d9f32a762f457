// device_ps.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Parameter-server kernels: K6 apply (XOR / SGD), batched push / GenGrad / fused pull+apply units, device DynReceiver, persistent and exchange schedules.

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
// fwd / nfwd: copies of the updated variable to write besides var (the fused
// push of the next iteration's weights, apply_unit; nfwd = 0 elsewhere)
template <class Op, int U>
__device__ __forceinline__ void fold_v4(uint8_t *varb, const uint8_t *const *g, int nw,
                                        uint64_t off, uint64_t nv, uint64_t t, uint64_t nth,
                                        float lr, uint8_t *const *fwd = nullptr,
                                        int nfwd = 0) {
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
    for (int f = 0; f < nfwd; ++f) {
      uint4 *fw = (uint4 *)(fwd[f] + off);
#pragma unroll
      for (int u = 0; u < U; ++u) fw[i + u * nth] = acc[u];
    }
  }
  for (; i < nv; i += nth) {
    uint4 acc = var[i];
    for (int w = 0; w < nw; ++w) acc = Op::fold(acc, ld_v4((const uint4 *)(g[w] + off) + i), lr);
    var[i] = acc;
    for (int f = 0; f < nfwd; ++f) ((uint4 *)(fwd[f] + off))[i] = acc;
  }
}

template <class Op>
__device__ __forceinline__ void fold_v2(uint8_t *varb, const uint8_t *const *g, int nw,
                                        uint64_t off, uint64_t nv, uint64_t t, uint64_t nth,
                                        float lr, uint8_t *const *fwd = nullptr,
                                        int nfwd = 0) {
  uint2 *var = (uint2 *)(varb + off);
  for (uint64_t i = t; i < nv; i += nth) {
    uint2 acc = var[i];
    for (int w = 0; w < nw; ++w) acc = Op::fold2(acc, ((const uint2 *)(g[w] + off))[i], lr);
    var[i] = acc;
    for (int f = 0; f < nfwd; ++f) ((uint2 *)(fwd[f] + off))[i] = acc;
  }
}

// The whole update of one variable over threads [t, +nth) of some grid.
// XOR works on bytes: 16-B vectors when every pointer shares (p mod 16), 8-B
// when they share (p mod 8) (arena blocks are 8-B aligned), bytes otherwise.
// SGD works on fp32: same vector classes in whole floats.
template <bool SGD>
__device__ void apply_range(uint8_t *var, const uint8_t *const *g, int nw, uint64_t n,
                            float lr, uint64_t t, uint64_t nth, uint8_t *const *fwd = nullptr,
                            int nfwd = 0) {
  const uintptr_t m = (uintptr_t)var;
  bool same16 = true, same8 = true;
  for (int w = 0; w < nw; ++w) {
    const uintptr_t p = (uintptr_t)g[w];
    same16 &= ((p ^ m) & 15) == 0;
    same8 &= ((p ^ m) & 7) == 0;
  }
  for (int f = 0; f < nfwd; ++f) {
    const uintptr_t p = (uintptr_t)fwd[f];
    same16 &= ((p ^ m) & 15) == 0;
    same8 &= ((p ^ m) & 7) == 0;
  }
  const uint64_t unit = SGD ? 4 : 1;  // scalar element size
  uint64_t head = 0, body = 0;
  if (same16) {
    head = ((16 - (m & 15)) & 15);
    if (head > n) head = n;
    const uint64_t nv = (n - head) / 16;
    if (SGD) fold_v4<SgdOp, 4>(var, g, nw, head, nv, t, nth, lr, fwd, nfwd);
    else fold_v4<XorOp, 4>(var, g, nw, head, nv, t, nth, lr, fwd, nfwd);
    body = nv * 16;
  } else if (same8) {
    head = ((8 - (m & 7)) & 7);
    if (head > n) head = n;
    const uint64_t nv = (n - head) / 8;
    if (SGD) fold_v2<SgdOp>(var, g, nw, head, nv, t, nth, lr, fwd, nfwd);
    else fold_v2<XorOp>(var, g, nw, head, nv, t, nth, lr, fwd, nfwd);
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
      for (int f = 0; f < nfwd; ++f) *(float *)(fwd[f] + e) = v;
    } else {
      uint8_t acc = var[e];
      for (int w = 0; w < nw; ++w) acc ^= g[w][e];
      var[e] = acc;
      for (int f = 0; f < nfwd; ++f) fwd[f][e] = acc;
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
  // source produced in-device (a static gradient push): wait until the
  // producer released it to 1, clear it to 0 once copied (the producer's
  // credit).  nullptr: none.
  uint8_t *src_ready;
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
  // fused push of the NEXT iteration's weights (PsStep(fuse_push=True)): the
  // updated variable is also stored into these workers' static receive
  // regions (payload || flag), and the last arriver releases their flags
  // with the value at fwd_tail - the StaticSender.send of the weights the
  // next iteration would otherwise issue as a separate K1 (one read of the
  // variable saved).  The credit is implied: every worker's gen cleared its
  // flag before producing the gradient this apply consumed.
  uint8_t *fwd[SRF_MAX_WORKERS];
  const uint8_t *fwd_tail;
  int nfwd, pad_fwd;
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
                                         unsigned int *seq = nullptr, bool coherent_src = false) {
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
    if (d.wait_empty || d.src_ready) {
      if (threadIdx.x == 0) {
        if (d.wait_empty && !spin_until(d.dst + d.body, 0, timeout_ns, sys)) atomicExch(err, 2);
        if (d.src_ready && !spin_until(d.src_ready, 1, timeout_ns, sys)) atomicExch(err, 3);
      }
      __syncthreads();
    }
    // (PS blocks are 256-B aligned: always co-aligned, no destination realignment).
    // Coherent source loads when the source may have been written earlier in
    // this launch: a variable updated by this launch's apply units (several
    // iterations per exchange launch) or a gradient produced in-device
    // (src_ready) - .nc loads are only defined for launch-read-only data.
    const uint64_t t0 = (uint64_t)lb * blockDim.x + threadIdx.x;
    const uint64_t nt = (uint64_t)d.cta_count * blockDim.x;
    if (coherent_src || d.src_ready)
      copy_bytes_grid<8, false, true>(d.dst, d.src, d.body, t0, nt);
    else
      copy_bytes_grid<8, false>(d.dst, d.src, d.body, t0, nt);
    __syncthreads();
    if (threadIdx.x == 0) s_last = grid_arrive(&counters[s_desc], d.cta_count - 1, sys);
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      // re-arm the arrival counter BEFORE publishing: whoever acquires the
      // flag (and, downstream, the next use of this edge) sees it at zero
      atomicExch(&counters[s_desc], 0u);
      release_tail(d.dst + d.body, *d.tail, sys);
      if (d.src_ready) release_tail(d.src_ready, 0, sys);  // source copied: credit
      if (seq) count_done(seq + s_desc);
    }
    __syncthreads();  // shared state is reused by the next unit
  }
}

__device__ __forceinline__ void put_batch_units(const BatchPut *descs, int n,
                                                uint32_t total_units, unsigned int *counters,
                                                uint64_t timeout_ns, int *err, int sys,
                                                bool coherent_src = false) {
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x)
    put_unit(descs, n, u, counters, timeout_ns, err, sys, nullptr, nullptr, 0, nullptr,
             coherent_src);
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
      // GenGrad = synthesize_values(dims, F32, node_rng(seed, node, iteration))
      // (graph.py:333-350, :363-370): the reference's PCG64 stream, bit-exact,
      // at the slice's global element indices (device_pcg.cuh)
      pcg_fill_f32_cta((float *)d.grad, d.n / 4, d.elem_offset, seed, d.node, iteration, lb,
                       d.cta_count);
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

// fwd: also store the updated variable into the descriptor's forward
// destinations (the fused next-iteration weight push; only the batch launch
// of a PsStep(fuse_push=True) sets it)
__device__ __forceinline__ void apply_unit(const BatchApply *descs, int n, uint32_t u,
                                           unsigned int *counters, int op, float lr,
                                           uint64_t timeout_ns, int *err, int sys,
                                           unsigned int *done = nullptr, uint32_t k = 0,
                                           int fwd = 0) {
  __shared__ int s_desc, s_last, s_bad;
  __shared__ const uint8_t *s_g[SRF_MAX_WORKERS];
  __shared__ uint8_t *s_fwd[SRF_MAX_WORKERS];
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
    const int nfwd = fwd ? d.nfwd : 0;
    if (threadIdx.x < (unsigned)nfwd) s_fwd[threadIdx.x] = d.fwd[threadIdx.x];
    __syncthreads();
    if (!s_bad) {
      const uint64_t t = (uint64_t)lb * blockDim.x + threadIdx.x;
      const uint64_t nth = (uint64_t)d.cta_count * blockDim.x;
      if (op == SRF_APPLY_XOR)
        apply_range<false>(d.var, s_g, d.nw, d.n, lr, t, nth, s_fwd, nfwd);
      else
        apply_range<true>(d.var, s_g, d.nw, d.n, lr, t, nth, s_fwd, nfwd);
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
    // the fused weight push: flags last, after every CTA's stores (the grid
    // arrival above is cumulative at the batch's scope)
    if (s_last && threadIdx.x < (unsigned)nfwd && !s_bad)
      release_tail(s_fwd[threadIdx.x] + d.n, *d.fwd_tail, sys);
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
                                                  int *err, int sys, int fwd = 0) {
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x)
    apply_unit(descs, n, u, counters, op, lr, timeout_ns, err, sys, nullptr, 0, fwd);
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
                                                     int *err, int sys, int fwd) {
  apply_batch_units(descs, n, total_units, counters, op, lr, timeout_ns, err, sys, fwd);
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

__global__ void __launch_bounds__(512) k_dyn_recv(const __grid_constant__ DynRecvArgs a) {
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
    copy_bytes_grid<8>(a.dst, s_src, s_len,  // pull: peer-side (source) sectors aligned
                       (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                       (uint64_t)gridDim.x * blockDim.x, false);
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
    // (iteration i pushes variables iteration i-1 of this launch updated)
    if (a.push)
      put_batch_units(a.push, a.npush, a.upush, a.cpush, a.timeout_ns, a.err, a.sys, true);
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
  int fwd;  // applies also write the next weights (PsStep(fuse_push=True))
  // several iterations per launch: the queue repeats `iters` times (iteration
  // k's units after iteration k-1's); done[] counts completed applies per
  // apply descriptor in this launch, push_done[i] maps push edge i to its
  // variable's counter (-1: none)
  uint32_t iters;
  unsigned int *done; int apply_base[kMaxApply]; const int *push_done;
  unsigned int *seq_push, *seq_gen;  // per-descriptor completion counts (this launch)
  // two lanes (lane_ctas > 0): CTAs [0, lane_ctas) claim the peer pushes
  // (`items`), the others GenGrad and apply (`items1`), each lane in the same
  // global order - pushes then occupy one CTA slot on lane_ctas SMs (the link
  // saturates with ~96 pushing CTAs) while the compute units fill the rest,
  // instead of the whole grid pushing, then the whole grid computing
  const ExItem *items1; uint32_t nitems1; unsigned int *claim1; uint32_t lane_ctas;
};

// kMinBlocks 3: 40 registers, 3 CTAs per SM - more bytes in flight for
// bandwidth-bound iterations (FCN-5 N=2 1517 -> 1693 it/s); kMinBlocks 2: the
// spill-free build (60 registers) for tiny, latency-bound iterations.
template <int kMinBlocks>
__global__ void __launch_bounds__(512, kMinBlocks) k_ps_exchange(const __grid_constant__ ExArgs a) {
  __shared__ uint32_t s_i;
  const bool lane1 = a.lane_ctas && blockIdx.x >= a.lane_ctas;
  const ExItem *items = lane1 ? a.items1 : a.items;
  const uint32_t nitems = lane1 ? a.nitems1 : a.nitems;
  unsigned int *claim = lane1 ? a.claim1 : a.claim;
  for (;;) {
    if (threadIdx.x == 0) s_i = atomicAdd(claim, 1u);
    __syncthreads();
    const uint32_t i = s_i;
    __syncthreads();
    if (i >= nitems * a.iters) break;
    const uint32_t k = i / nitems;
    const ExItem x = items[i - k * nitems];
    if (x.kind == 0)
      put_unit(a.push, a.npush, x.unit, a.cpush, a.timeout_ns, a.err, a.push_sys, a.done,
               a.push_done, k, a.seq_push, true);
    else if (x.kind == 1)
      gen_unit(a.gen, a.ngen, x.unit, a.cgen, a.seed, a.iteration + k, a.regen, 1,
               a.timeout_ns, a.err, a.gen_sys, k, a.seq_gen);
    else
      apply_unit(a.apply[x.batch], a.napply[x.batch], x.unit, a.capply[x.batch], a.op, a.lr,
                 a.timeout_ns, a.err, a.apply_sys[x.batch], a.done + a.apply_base[x.batch], k,
                 a.fwd);
  }
  // the last CTA out re-arms the queue for the next launch
  if (threadIdx.x == 0 && atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
    *a.claim = 0;
    if (a.claim1) *a.claim1 = 0;
    *a.exit_count = 0;
  }
}

// graph-replayed PS steps: advance the device iteration counter
__global__ void k_counter_add(uint64_t *p, uint64_t delta) { *p += delta; }
