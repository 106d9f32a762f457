// abi_doorbell.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// C ABI: doorbells, RPC transfer, reduce, events.

extern "C" {
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
// waits for that clear.  An exported space's producers live in other
// processes and cannot wait on that event: the device byte is written
// synchronously there (their credit check reads it over NVLink).
int srf_flag_clear(srf_space_t sp, uint64_t tail_addr) {
  DeviceGuard device_guard;
  int rc = check_raw(sp, tail_addr, 1, "flag");
  if (rc) return rc;
  if (sp->db && !sp->exported) {
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
      if (recording())  // the doorbell byte through its device mapping
        rec_clear(sp->device, sp->base + tail_addr, sp->db_dev + d.host_off + d.shadow_len - 1);
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

int srf_space_wait_event(srf_space_t sp, srf_event_t ev) {
  DeviceGuard device_guard;
  CUDA_TRY(cudaSetDevice(sp->stream->device));
  CUDA_TRY(cudaStreamWaitEvent(sp->stream->s, ev->e, 0));
  return SRF_OK;
}

int srf_matmul(int elem, uint64_t a_ptr, uint64_t b_ptr, uint64_t c_ptr, uint64_t m, uint64_t k,
               uint64_t n, void *cuda_stream) {
  DeviceGuard device_guard;
  if (m * n == 0) return SRF_OK;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const unsigned grid = (unsigned)((m * n + 255) / 256);
  switch (elem) {
    case 0: k_matmul<float><<<grid, 256, 0, s>>>((const float *)a_ptr, (const float *)b_ptr,
                                                   (float *)c_ptr, m, k, n); break;
    case 1: k_matmul<double><<<grid, 256, 0, s>>>((const double *)a_ptr, (const double *)b_ptr,
                                                    (double *)c_ptr, m, k, n); break;
    case 2: k_matmul<int32_t><<<grid, 256, 0, s>>>((const int32_t *)a_ptr, (const int32_t *)b_ptr,
                                                     (int32_t *)c_ptr, m, k, n); break;
    case 3: k_matmul<int64_t><<<grid, 256, 0, s>>>((const int64_t *)a_ptr, (const int64_t *)b_ptr,
                                                     (int64_t *)c_ptr, m, k, n); break;
    case 4: k_matmul<uint8_t><<<grid, 256, 0, s>>>((const uint8_t *)a_ptr, (const uint8_t *)b_ptr,
                                                     (uint8_t *)c_ptr, m, k, n); break;
    default: return fail(SRF_E_INVALID_CONFIG, "unknown element type %d", elem);
  }
  if (recording()) {
    int dev = 0;
    cudaGetDevice(&dev);
    rec_matmul(dev, elem, a_ptr, b_ptr, c_ptr, m, k, n);
  }
  return launch_check("k_matmul");
}

int srf_compute(srf_space_t sp, int kind, int elem, uint64_t a_addr, uint64_t b_addr,
                uint64_t out_addr, uint64_t m, uint64_t k, uint64_t n, srf_stream_t st) {
  DeviceGuard device_guard;
  if (elem < 0 || elem > 4) return fail(SRF_E_INVALID_CONFIG, "unknown element type %d", elem);
  const uint64_t es = elem == 0 || elem == 2 ? 4 : elem == 4 ? 1 : 8;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  uint8_t *base = sp->base;
  if (kind == 0) {  // MatMul: a[m,k] @ b[k,n] -> out[m,n]
    int rc = check_raw(sp, a_addr, es * m * k, "matmul a");
    if (!rc) rc = check_raw(sp, b_addr, es * k * n, "matmul b");
    if (!rc) rc = check_raw(sp, out_addr, es * m * n, "matmul out");
    if (rc) return rc;
    return srf_matmul(elem, (uint64_t)(base + a_addr), (uint64_t)(base + b_addr),
                      (uint64_t)(base + out_addr), m, k, n, (void *)s->s);
  }
  if (kind != 1 && kind != 2) return fail(SRF_E_INVALID_CONFIG, "unknown compute kind %d", kind);
  if (kind == 2 && elem != 0 && elem != 1)
    return fail(SRF_E_INVALID_CONFIG, "sigmoid of a non-float type");
  int rc = check_raw(sp, a_addr, es * n, "operand");
  if (!rc && kind == 1) rc = check_raw(sp, b_addr, es * n, "operand");
  if (!rc) rc = check_raw(sp, out_addr, es * n, "result");
  if (rc) return rc;
  if (n == 0) return SRF_OK;
  const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count_of(s->device) * 8);
  const void *a = base + a_addr, *b = kind == 1 ? base + b_addr : nullptr;
  void *o = base + out_addr;
  if (kind == 1) {
    switch (elem) {
      case 0: k_add<float><<<grid, 256, 0, s->s>>>((const float *)a, (const float *)b, (float *)o, n); break;
      case 1: k_add<double><<<grid, 256, 0, s->s>>>((const double *)a, (const double *)b, (double *)o, n); break;
      case 2: k_add<int32_t><<<grid, 256, 0, s->s>>>((const int32_t *)a, (const int32_t *)b, (int32_t *)o, n); break;
      case 3: k_add<int64_t><<<grid, 256, 0, s->s>>>((const int64_t *)a, (const int64_t *)b, (int64_t *)o, n); break;
      default: k_add<uint8_t><<<grid, 256, 0, s->s>>>((const uint8_t *)a, (const uint8_t *)b, (uint8_t *)o, n); break;
    }
  } else if (elem == 0) {
    k_sigmoid<float><<<grid, 256, 0, s->s>>>((const float *)a, (float *)o, n);
  } else {
    k_sigmoid<double><<<grid, 256, 0, s->s>>>((const double *)a, (double *)o, n);
  }
  if (recording()) rec_ewise(s->device, grid, kind, elem, a, b, o, n);
  return launch_check(kind == 1 ? "k_add" : "k_sigmoid");
}

// Add with numpy broadcasting: a[a_dims] + b[b_dims] (equal rank <= 8, every
// dimension pair equal or one of them 1) into out (the broadcast shape)
int srf_add_bcast(srf_space_t sp, int elem, uint64_t a_addr, const uint64_t *a_dims,
                  uint64_t b_addr, const uint64_t *b_dims, int rank, uint64_t out_addr,
                  srf_stream_t st) {
  DeviceGuard device_guard;
  if (elem < 0 || elem > 4) return fail(SRF_E_INVALID_CONFIG, "unknown element type %d", elem);
  if (rank < 1 || rank > 8) return fail(SRF_E_INVALID_CONFIG, "broadcast rank 1..8");
  const uint64_t es = elem == 0 || elem == 2 ? 4 : elem == 4 ? 1 : 8;
  BcastArgs g;
  memset(&g, 0, sizeof g);
  g.rank = rank;
  uint64_t na = 1, nb = 1, n = 1;
  for (int k = 0; k < rank; ++k) {
    const uint64_t x = a_dims[k], y = b_dims[k];
    if (x != y && x != 1 && y != 1)
      return fail(SRF_E_SHAPE_MISMATCH, "operands not broadcastable in dimension %d", k);
    g.dims[k] = x == 1 ? y : x;
    na *= x;
    nb *= y;
    n *= g.dims[k];
  }
  uint64_t ra = 1, rb = 1;  // row-major element strides, 0 where broadcast
  for (int k = rank - 1; k >= 0; --k) {
    g.sa[k] = (a_dims[k] == 1 && g.dims[k] != 1) ? 0 : ra;
    g.sb[k] = (b_dims[k] == 1 && g.dims[k] != 1) ? 0 : rb;
    ra *= a_dims[k];
    rb *= b_dims[k];
  }
  int rc = check_raw(sp, a_addr, es * na, "operand");
  if (!rc) rc = check_raw(sp, b_addr, es * nb, "operand");
  if (!rc) rc = check_raw(sp, out_addr, es * n, "result");
  if (rc) return rc;
  if (n == 0) return SRF_OK;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count_of(s->device) * 8);
  const void *a = sp->base + a_addr, *b = sp->base + b_addr;
  void *o = sp->base + out_addr;
  switch (elem) {
    case 0: k_add_bcast<float><<<grid, 256, 0, s->s>>>((const float *)a, (const float *)b, (float *)o, n, g); break;
    case 1: k_add_bcast<double><<<grid, 256, 0, s->s>>>((const double *)a, (const double *)b, (double *)o, n, g); break;
    case 2: k_add_bcast<int32_t><<<grid, 256, 0, s->s>>>((const int32_t *)a, (const int32_t *)b, (int32_t *)o, n, g); break;
    case 3: k_add_bcast<int64_t><<<grid, 256, 0, s->s>>>((const int64_t *)a, (const int64_t *)b, (int64_t *)o, n, g); break;
    default: k_add_bcast<uint8_t><<<grid, 256, 0, s->s>>>((const uint8_t *)a, (const uint8_t *)b, (uint8_t *)o, n, g); break;
  }
  return launch_check("k_add_bcast");
}

// ConcatDyn into the output block: the n_in inputs (space addresses and byte
// lengths, total > 0) concatenated and repeated to out_len bytes
int srf_concat_tile(srf_space_t sp, int n_in, const uint64_t *in_addr, const uint64_t *in_len,
                    uint64_t out_addr, uint64_t out_len, srf_stream_t st) {
  DeviceGuard device_guard;
  if (n_in < 1 || n_in > kConcatMax)
    return fail(SRF_E_INVALID_CONFIG, "concat of 1..%d inputs", kConcatMax);
  ConcatArgs a;
  memset(&a, 0, sizeof a);
  bool words = out_addr % 4 == 0 && out_len % 4 == 0;
  for (int i = 0; i < n_in; ++i) {
    int rc = check_raw(sp, in_addr[i], in_len[i], "concat input");
    if (rc) return rc;
    a.src[i] = sp->base + in_addr[i];
    a.len[i] = in_len[i];
    a.total += in_len[i];
    words = words && in_addr[i] % 4 == 0 && in_len[i] % 4 == 0;
  }
  if (a.total == 0) return fail(SRF_E_INVALID_LENGTH, "concat of empty inputs");
  int rc = check_raw(sp, out_addr, out_len, "concat output");
  if (rc) return rc;
  if (out_len == 0) return SRF_OK;
  a.nsrc = n_in;
  a.out = sp->base + out_addr;
  a.out_len = out_len;
  a.unit = words ? 4 : 1;
  srf_stream *s = stream_or_default(sp, st);
  CUDA_TRY(cudaSetDevice(s->device));
  const uint64_t n = out_len / a.unit;
  const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count_of(s->device) * 8);
  k_concat_tile<<<grid, 256, 0, s->s>>>(a);
  // (not recorded: a dynamic shape never repeats, launch_check marks any
  // active recording unusable)
  return launch_check("k_concat_tile");
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
