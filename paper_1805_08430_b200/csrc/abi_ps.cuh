// abi_ps.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// C ABI: PS batches, persistent launch, exchange schedule.

extern "C" {
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
    d.src_ready = nullptr;
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
    // gradients of >= 64 MiB (VGG-16's fc6/fc7) in >= 512 KiB units: fewer
    // per-unit stream derivations (~150 dependent 128-bit multiplies each);
    // smaller tensors keep finer units for overlap (profiles/r2_gen_unit_sweep.jsonl)
    const uint64_t unit = nbytes[i] >= (64ull << 20)
                              ? std::max<uint64_t>(g_gen_unit_bytes, 512 << 10)
                              : g_gen_unit_bytes;
    d.cta_count = ctas_for(device, nbytes[i], unit);
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
                                             b->counters, b->op, b->lr, timeout, b->err, b->sys,
                                             mode & 1);
      return launch_check("k_apply_batch");
  }
}

// Device iteration counter for graph-captured PS steps: a gen batch launched
// with iteration == UINT64_MAX reads *counter; srf_counter_add bumps it in
// stream order at the end of a step.

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

// Fused weight push (PsStep(fuse_push=True)): descriptor v of the apply
// batch also stores its updated variable into nfwd[v] workers' static
// receive regions (space fwd_space[k], payload at fwd_addr[k], flag right
// after it, token fwd_token[k]) and releases their flags with the byte at
// tail_addr of the batch's space.  Only launches with mode bit 0 set forward.
int srf_batch_apply_set_forward(srf_batch_t apply, const int *nfwd,
                                srf_space_t const *fwd_space, const uint64_t *fwd_addr,
                                const uint64_t *fwd_token, srf_space_t tail_space,
                                uint64_t tail_addr) {
  DeviceGuard device_guard;
  if (!apply || apply->kind != 2) return fail(SRF_E_INVALID_CONFIG, "not an apply batch");
  int rc = check_raw(tail_space, tail_addr, 1, "forward flag value");
  if (rc) return rc;
  BatchApply *d = (BatchApply *)apply->host.data();
  int k = 0, sys = apply->sys;
  for (int v = 0; v < apply->n; ++v) {
    if (nfwd[v] < 0 || nfwd[v] > SRF_MAX_WORKERS)
      return fail(SRF_E_INVALID_CONFIG, "nfwd %d", nfwd[v]);
    d[v].nfwd = nfwd[v];
    d[v].fwd_tail = tail_space->base + tail_addr;
    for (int f = 0; f < nfwd[v]; ++f, ++k) {
      srf_space *fs = fwd_space[k];
      {
        std::lock_guard<std::mutex> g(fs->mu);
        rc = check_remote_locked(fs, fwd_addr[k], d[v].n + 1, fwd_token[k]);
        if (rc) return rc;
      }
      d[v].fwd[f] = fs->base + fwd_addr[k];
      sys |= (fs->imported || fs->device != apply->device) ? 1 : 0;
    }
  }
  apply->sys = sys;
  CUDA_TRY(cudaSetDevice(apply->device));
  CUDA_TRY(cudaMemcpy(apply->descs, apply->host.data(), apply->host.size(),
                      cudaMemcpyHostToDevice));
  return SRF_OK;
}

int srf_batch_put_set_src_ready(srf_batch_t put, srf_space_t const *space,
                                const uint64_t *ready_addr) {
  DeviceGuard device_guard;
  if (!put || put->kind != 0) return fail(SRF_E_INVALID_CONFIG, "not a put batch");
  BatchPut *d = (BatchPut *)put->host.data();
  for (int i = 0; i < put->n; ++i) {
    if (ready_addr[i] == UINT64_MAX) {
      d[i].src_ready = nullptr;
      continue;
    }
    if (space[i]->device != put->device)
      return fail(SRF_E_INVALID_CONFIG, "source-ready byte of edge %d on another GPU", i);
    int rc = check_raw(space[i], ready_addr[i], 1, "source-ready flag");
    if (rc) return rc;
    d[i].src_ready = space[i]->base + ready_addr[i];
  }
  CUDA_TRY(cudaSetDevice(put->device));
  CUDA_TRY(cudaMemcpy(put->descs, put->host.data(), put->host.size(), cudaMemcpyHostToDevice));
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
  bool lean = false;  // tiny iteration: the spill-free kernel build
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
  // peer pushes get their own lane of CTAs (SRFLOW_PS_PUSH_CTAS, default 128;
  // 0: one queue); same-GPU pushes are HBM copies and keep the one queue.
  // VGG-16 N=2, static gradients in 8 MiB slices: 853 it/s with one queue,
  // 1208 with 128 push CTAs (96: 1072, 160: 1022; profiles/r2_ps_push_lane.jsonl)
  int lane = (push && push->sys) ? 128 : 0;
  if (const char *l = getenv("SRFLOW_PS_PUSH_CTAS")) lane = std::max(0, atoi(l));
  size_t npush_items = 0;
  for (const K &k : ks) npush_items += k.kind == 0;
  if (npush_items == 0 || npush_items == ks.size()) lane = 0;
  if (const char *g = getenv("SRFLOW_PS_EXCHANGE_GRID"))
    if (atoi(g) < 2) lane = 0;  // one CTA: one queue
  std::vector<ExItem> items;
  items.reserve(ks.size());
  for (int pass = 0; pass < (lane ? 2 : 1); ++pass)
    for (const K &k : ks)
      if (!lane || (pass == 0) == (k.kind == 0))
        items.push_back({k.unit, (uint16_t)k.kind, (uint16_t)k.batch});
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
  if (e == cudaSuccess) e = cudaMalloc(&x->ctr, 3 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(x->ctr, 0, 3 * sizeof(unsigned int));
  const int np = a.npush, ng = a.ngen;
  x->ndone = std::max(nd + np + ng, 1);
  if (e == cudaSuccess) e = cudaMalloc(&x->done, sizeof(unsigned int) * x->ndone);
  if (e == cudaSuccess) e = cudaMemset(x->done, 0, sizeof(unsigned int) * x->ndone);
  if (e == cudaSuccess) e = cudaMalloc(&x->push_done, sizeof(int) * std::max(1, a.npush));
  if (e == cudaSuccess) e = cudaMemset(x->push_done, 0xff, sizeof(int) * std::max(1, a.npush));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  // fewer work units than SMs: a latency-bound iteration (the MLP parity set)
  x->lean = items.size() < (size_t)sm_count_of(device);
  int per_sm = 0;
  if (e == cudaSuccess)
    e = x->lean ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ps_exchange<2>, 512, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ps_exchange<3>, 512, 0);
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
  if (lane) {
    a.nitems = (uint32_t)npush_items;
    a.items1 = x->items + npush_items;
    a.nitems1 = (uint32_t)(items.size() - npush_items);
    a.claim1 = x->ctr + 2;
  }
  a.done = x->done;
  a.push_done = x->push_done;
  a.seq_push = np ? x->done + nd : nullptr;
  a.seq_gen = ng ? x->done + nd + np : nullptr;
  x->napply_descs = nd;
  a.iters = 1;
  x->grid = sm_count_of(device) * std::max(1, per_sm);
  if (const char *g = getenv("SRFLOW_PS_EXCHANGE_GRID")) x->grid = std::max(1, atoi(g));
  // each lane keeps at least one CTA
  if (lane) a.lane_ctas = (uint32_t)std::min(lane, x->grid - 1);
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
  x->args.regen = regen & 1;
  x->args.fwd = (regen >> 1) & 1;  // mode bit 1: the fused weight push
  x->args.iters = iterations;
  CUDA_TRY(cudaSetDevice(x->device));
  if (iterations > 1)
    CUDA_TRY(cudaMemsetAsync(x->done, 0, sizeof(unsigned int) * x->ndone, st->s));
  if (x->lean)
    k_ps_exchange<2><<<x->grid, 512, 0, st->s>>>(x->args);
  else
    k_ps_exchange<3><<<x->grid, 512, 0, st->s>>>(x->args);
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

}  // extern "C"
