// device_rpc.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// RPC-style fragment ring baseline and ReduceMax.

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

// Coherent source loads: ring slots and staging slots are rewritten by the
// other side (or this warp pair) every round within one launch.
__device__ __forceinline__ void slot_copy(uint8_t *dst, const uint8_t *src, uint64_t n) {
  copy_bytes_grid<4, true, true>(dst, src, n, threadIdx.x % kSlotThreads, kSlotThreads);
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
// MatMul compute kind of the Session's graphs (graph.py:371-372: numpy
// `a @ b`), bit-identical to numpy: numpy's float matmul (OpenBLAS sgemm /
// dgemm) accumulates each output as an ascending-k FMA chain from 0 (checked
// for k <= 64 in tests), integer matmul wraps in the element type.  Not on
// the transfer path (compute kinds are graph plumbing): one
// thread per output element.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T mm_step(T acc, T a, T b);
template <>
__device__ __forceinline__ float mm_step<float>(float acc, float a, float b) {
  return __fmaf_rn(a, b, acc);
}
template <>
__device__ __forceinline__ double mm_step<double>(double acc, double a, double b) {
  return __fma_rn(a, b, acc);
}
template <>
__device__ __forceinline__ int32_t mm_step<int32_t>(int32_t acc, int32_t a, int32_t b) {
  return (int32_t)((uint32_t)acc + (uint32_t)a * (uint32_t)b);
}
template <>
__device__ __forceinline__ int64_t mm_step<int64_t>(int64_t acc, int64_t a, int64_t b) {
  return (int64_t)((uint64_t)acc + (uint64_t)a * (uint64_t)b);
}
template <>
__device__ __forceinline__ uint8_t mm_step<uint8_t>(uint8_t acc, uint8_t a, uint8_t b) {
  return (uint8_t)(acc + a * b);
}

template <typename T>
__global__ void __launch_bounds__(256) k_matmul(const T *a, const T *b, T *c, uint64_t m,
                                                uint64_t k, uint64_t n) {
  const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * n) return;
  const uint64_t i = idx / n, j = idx - i * n;
  T acc = T(0);
  for (uint64_t t = 0; t < k; ++t) acc = mm_step<T>(acc, a[i * k + t], b[t * n + j]);
  c[idx] = acc;
}

// Add and Sigmoid compute kinds (graph.py:373-377): numpy `a + b` on equal
// shapes (integers wrap), and (1 / (1 + exp(-x.astype(float64)))).astype(x's
// type) - computed in double like the reference, then rounded once.
template <typename T>
__device__ __forceinline__ T ew_add(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ int32_t ew_add<int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
template <>
__device__ __forceinline__ int64_t ew_add<int64_t>(int64_t a, int64_t b) {
  return (int64_t)((uint64_t)a + (uint64_t)b);
}
template <>
__device__ __forceinline__ float ew_add<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double ew_add<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) k_add(const T *a, const T *b, T *out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = ew_add<T>(a[i], b[i]);
}

// Add with numpy broadcasting (operands of equal rank; a dimension of 1
// against a larger one repeats): element i of the output at coordinates c
// reads a[sum c_k * sa_k] and b[sum c_k * sb_k], strides 0 where broadcast
struct BcastArgs {
  int rank;
  uint64_t dims[8], sa[8], sb[8];
};

template <typename T>
__global__ void __launch_bounds__(256) k_add_bcast(const T *a, const T *b, T *out, uint64_t n,
                                                   const __grid_constant__ BcastArgs g) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t rem = i, oa = 0, ob = 0;
    for (int k = g.rank - 1; k >= 0; --k) {
      const uint64_t c = rem % g.dims[k];
      rem /= g.dims[k];
      oa += c * g.sa[k];
      ob += c * g.sb[k];
    }
    out[i] = ew_add<T>(a[oa], b[ob]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_sigmoid(const T *x, T *out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[i];
    out[i] = (T)(1.0 / (1.0 + exp(-v)));
  }
}

// ConcatDyn (graph.py compute_node CONCAT_DYN): the inputs' elements
// concatenated in order (they share trailing dims, so concatenating along
// dim 0 is concatenating their flat storage), repeated to fill the output:
// out[i] = cat[i % total].  Words of `unit` bytes (4 when every length and
// address allows it, else 1).
static constexpr int kConcatMax = 8;
struct ConcatArgs {
  const uint8_t *src[kConcatMax];
  uint64_t len[kConcatMax];   // bytes
  int nsrc;
  uint64_t total;             // bytes of the concatenation (> 0)
  uint8_t *out;
  uint64_t out_len;           // bytes
  int unit;
};

__global__ void __launch_bounds__(256) k_concat_tile(const __grid_constant__ ConcatArgs a) {
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t words = a.out_len / a.unit;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += nth) {
    uint64_t b = (w * a.unit) % a.total;
    int k = 0;
    while (k + 1 < a.nsrc && b >= a.len[k]) b -= a.len[k++];
    if (a.unit == 4)
      *(uint32_t *)(a.out + w * 4) = *(const uint32_t *)(a.src[k] + b);
    else
      a.out[w] = a.src[k][b];
  }
}
