// host_record.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Recording and replay of one Session iteration's device work.
//
// The reference's Session.run (runtime/session.py:606-629) drives every verb
// from a Python executor: a synchronous host round trip per put, poll, pull and
// update.  Once the session is in steady state (tracing frozen, two
// consecutive iterations issuing exactly the same device work and producing
// identical RunReport rows), the later iterations are that same work with
// only the GenGrad iteration advanced.  The recorder captures, per iteration,
// every launch the library makes on the session's behalf - K1/K4/K5 puts and
// pulls, the inline K3 metadata put, GenGrad, K6 updates, ReduceMax, MatMul
// and the receivers' flag clears (device byte + host doorbell) - with their
// exact arguments; anything it cannot replay (a host write into device memory,
// a copy-engine body, an uninstrumented kernel, a second device) marks the
// recording unusable.  Replay builds one CUDA graph of the recorded iteration
// on a single stream (the host path serialised every verb anyway), with
// GenGrad reading its iteration offset from a device counter the graph's
// last node advances, and launches it once per remaining iteration.

enum RecKind : int {
  REC_PUT = 1,
  REC_INLINE = 2,
  REC_GEN = 3,
  REC_APPLY = 4,
  REC_REDUCE = 5,
  REC_CLEAR = 6,
  REC_MATMUL = 7,
  REC_EWISE = 8,   // Add / Sigmoid compute kinds
};

struct RecOp {
  int kind = 0;
  int device = -1;
  int grid = 0, block = 0, variant = 0;
  PutArgs put;
  InlineArgs *inl = nullptr;  // heap (the block is up to 1 KiB)
  ApplyArgs apply;
  int apply_sgd = 0;
  struct {
    float *dst;
    uint64_t nf, e0, seed, node, iteration;
  } gen;
  struct {
    const float *in;
    uint64_t n;
    float *out;
    float *scratch;
    unsigned int *counter;
  } red;
  struct {
    uint8_t *dev;
    uint8_t *shadow;
  } clr;
  struct {
    int elem;
    uint64_t a, b, c, m, k, n;
  } mm;
  struct {
    int op, elem;      // op 1 add, 2 sigmoid
    const void *a, *b;
    void *out;
    uint64_t n;
  } ew;
};

struct srf_oplist {
  std::vector<RecOp> ops;
  int device = -1;
  bool dirty = false;
  std::string why;
  // replay state
  cudaGraphExec_t exec = nullptr;
  uint64_t *iter_add = nullptr;  // device counter: GenGrad iteration offset
  unsigned int *priv = nullptr;  // private arrival counters / reduction scratch
  int graph_device = -1;
  uint32_t nodes = 0, edges = 0;
  ~srf_oplist() {
    for (RecOp &op : ops) delete op.inl;
    if (exec) cudaGraphExecDestroy(exec);
    if (iter_add) cudaFree(iter_add);
    if (priv) cudaFree(priv);
  }
};

static std::mutex g_rec_mu;
static srf_oplist *g_rec = nullptr;          // the active recording (one at a time)
static thread_local bool g_rec_expected = false;

static bool recording() { return g_rec != nullptr; }

static void rec_dirty(const char *why) {
  std::lock_guard<std::mutex> g(g_rec_mu);
  if (g_rec && !g_rec->dirty) {
    g_rec->dirty = true;
    g_rec->why = why;
  }
}

static void rec_push(RecOp &&op) {
  std::lock_guard<std::mutex> g(g_rec_mu);
  if (!g_rec) {
    delete op.inl;
    return;
  }
  if (g_rec->device < 0) g_rec->device = op.device;
  if (op.device != g_rec->device && !g_rec->dirty) {
    g_rec->dirty = true;
    g_rec->why = "work on a second device";
  }
  g_rec->ops.push_back(std::move(op));
  g_rec_expected = true;  // the launch_check that follows belongs to this op
}

// every kernel launch passes launch_check: one no instrumented path claimed
// makes the recording unusable
static void rec_check_launch(const char *what) {
  if (!recording()) return;
  if (g_rec_expected) {
    g_rec_expected = false;
    return;
  }
  rec_dirty(what);
}

static void rec_put(const PutArgs &a, const srf_stream *s, int grid, int block, int variant) {
  RecOp op;
  op.kind = REC_PUT;
  op.device = s->device;
  op.grid = grid;
  op.block = block;
  op.variant = variant;
  op.put = a;
  rec_push(std::move(op));
}

static void rec_inline(const InlineArgs &a, int device) {
  RecOp op;
  op.kind = REC_INLINE;
  op.device = device;
  op.grid = 1;
  op.block = 256;
  op.inl = new InlineArgs(a);
  rec_push(std::move(op));
}

static void rec_gen(int device, int grid, float *dst, uint64_t nf, uint64_t e0, uint64_t seed,
                    uint64_t node, uint64_t iteration) {
  RecOp op;
  op.kind = REC_GEN;
  op.device = device;
  op.grid = grid;
  op.block = 512;
  op.gen = {dst, nf, e0, seed, node, iteration};
  rec_push(std::move(op));
}

static void rec_apply(int device, int grid, int block, const ApplyArgs &a, int sgd) {
  RecOp op;
  op.kind = REC_APPLY;
  op.device = device;
  op.grid = grid;
  op.block = block;
  op.apply = a;
  op.apply_sgd = sgd;
  rec_push(std::move(op));
}

static void rec_reduce(int device, int grid, const float *in, uint64_t n, float *out,
                       float *scratch, unsigned int *counter) {
  RecOp op;
  op.kind = REC_REDUCE;
  op.device = device;
  op.grid = grid;
  op.block = 256;
  op.red = {in, n, out, scratch, counter};
  rec_push(std::move(op));
}

static void rec_matmul(int device, int elem, uint64_t a, uint64_t b, uint64_t c, uint64_t m,
                       uint64_t k, uint64_t n) {
  RecOp op;
  op.kind = REC_MATMUL;
  op.device = device;
  op.grid = (int)((m * n + 255) / 256);
  op.block = 256;
  op.mm = {elem, a, b, c, m, k, n};
  rec_push(std::move(op));
}

static void rec_ewise(int device, int grid, int op, int elem, const void *a, const void *b,
                      void *out, uint64_t n) {
  RecOp o;
  o.kind = REC_EWISE;
  o.device = device;
  o.grid = grid;
  o.block = 256;
  o.ew = {op, elem, a, b, out, n};
  rec_push(std::move(o));
}

// a receiver's flag clear (memset of the device byte; the host doorbell was
// cleared on the host): no kernel launch follows
static void rec_clear(int device, uint8_t *dev, uint8_t *shadow) {
  RecOp op;
  op.kind = REC_CLEAR;
  op.device = device;
  op.clr = {dev, shadow};
  rec_push(std::move(op));
  g_rec_expected = false;
}

__global__ void k_set_u64(uint64_t *p, uint64_t v) { *p = v; }

// Replayed flag clear: the device byte and its host doorbell, in stream order.
__global__ void k_clear_flag(uint8_t *dev, uint8_t *shadow) {
  *(volatile uint8_t *)dev = 0;
  if (shadow) *(volatile uint8_t *)shadow = 0;
}

static bool rec_same(const RecOp &x, const RecOp &y, int64_t gen_delta) {
  if (x.kind != y.kind || x.device != y.device || x.grid != y.grid || x.block != y.block ||
      x.variant != y.variant)
    return false;
  switch (x.kind) {
    case REC_PUT: return memcmp(&x.put, &y.put, sizeof x.put) == 0;
    case REC_INLINE: return memcmp(x.inl, y.inl, sizeof(InlineArgs)) == 0;
    case REC_GEN:
      return x.gen.dst == y.gen.dst && x.gen.nf == y.gen.nf && x.gen.e0 == y.gen.e0 &&
             x.gen.seed == y.gen.seed && x.gen.node == y.gen.node &&
             (int64_t)(y.gen.iteration - x.gen.iteration) == gen_delta;
    case REC_APPLY:
      return x.apply_sgd == y.apply_sgd && memcmp(&x.apply, &y.apply, sizeof x.apply) == 0;
    case REC_REDUCE: return memcmp(&x.red, &y.red, sizeof x.red) == 0;
    case REC_CLEAR: return x.clr.dev == y.clr.dev && x.clr.shadow == y.clr.shadow;
    case REC_MATMUL: return memcmp(&x.mm, &y.mm, sizeof x.mm) == 0;
    case REC_EWISE: return memcmp(&x.ew, &y.ew, sizeof x.ew) == 0;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Replay graph with data dependencies instead of one chain: the host path
// serialised every verb, but only ops whose byte ranges conflict (read after
// write, write after read or write) need ordering - different variables'
// pushes, GenGrads, pulls and updates may run side by side, as the device PS
// engine runs them.  Each op's footprint: the ranges it reads and writes
// (device pointers and host-mapped doorbell bytes live in one address space);
// arrival counters and reduction scratch are made private per op.
// ---------------------------------------------------------------------------
struct Span {
  uintptr_t lo, hi;  // [lo, hi)
  bool write;
};

static void rec_footprint(const RecOp &op, std::vector<Span> &out) {
  auto add = [&](const void *p, uint64_t n, bool w) {
    if (p && n) out.push_back({(uintptr_t)p, (uintptr_t)p + n, w});
  };
  switch (op.kind) {
    case REC_PUT: {
      const PutArgs &a = op.put;
      for (int i = 0; i < a.nseg; ++i) add(a.seg[i].src, a.seg[i].len, false);
      add(a.dst, a.total, true);
      if (a.db) add(a.db, a.db_len, true);
      if (a.consume) add(a.consume, 1, true);
      break;
    }
    case REC_INLINE:
      add(op.inl->stage, op.inl->len, true);
      add(op.inl->dst, op.inl->len, true);
      if (op.inl->db) add(op.inl->db, op.inl->db_len, true);
      break;
    case REC_GEN: add(op.gen.dst, 4 * op.gen.nf, true); break;
    case REC_APPLY:
      for (int w = 0; w < op.apply.nw; ++w) add(op.apply.g[w], op.apply.n, false);
      add(op.apply.var, op.apply.n, true);
      break;
    case REC_REDUCE:
      add(op.red.in, 4 * op.red.n, false);
      add(op.red.out, 4, true);
      break;
    case REC_CLEAR:
      add(op.clr.dev, 1, true);
      if (op.clr.shadow) add(op.clr.shadow, 1, true);
      break;
    case REC_EWISE: {
      const uint64_t es = op.ew.elem == 0 || op.ew.elem == 2 ? 4 : op.ew.elem == 4 ? 1 : 8;
      add(op.ew.a, es * op.ew.n, false);
      if (op.ew.b) add(op.ew.b, es * op.ew.n, false);
      add(op.ew.out, es * op.ew.n, true);
      break;
    }
    case REC_MATMUL: {
      const uint64_t es = op.mm.elem == 0 || op.mm.elem == 2 ? 4 : op.mm.elem == 4 ? 1 : 8;
      add((const void *)op.mm.a, es * op.mm.m * op.mm.k, false);
      add((const void *)op.mm.b, es * op.mm.k * op.mm.n, false);
      add((const void *)op.mm.c, es * op.mm.m * op.mm.n, true);
      break;
    }
  }
}

static bool rec_conflict(const std::vector<Span> &a, const std::vector<Span> &b) {
  for (const Span &x : a)
    for (const Span &y : b)
      if ((x.write || y.write) && x.lo < y.hi && y.lo < x.hi) return true;
  return false;
}

// Build l->exec: one kernel node per op, edges from every earlier op it
// conflicts with (transitively redundant edges kept; the graph is small).
static int rec_build_graph(srf_oplist *l) {
  const size_t n = l->ops.size();
  // private arrival counters (PutArgs.counter, reduction counter) and scratch
  const size_t words = 2 * n + (size_t)kScratchBlocks * n;
  CUDA_TRY(cudaMalloc(&l->iter_add, sizeof(uint64_t)));
  CUDA_TRY(cudaMemset(l->iter_add, 0, sizeof(uint64_t)));
  CUDA_TRY(cudaMalloc(&l->priv, sizeof(unsigned int) * words));
  CUDA_TRY(cudaMemset(l->priv, 0, sizeof(unsigned int) * words));
  std::vector<RecOp> ops = l->ops;  // patched copies (kernel params are copied at add time)
  std::vector<std::vector<Span>> fp(n);
  for (size_t i = 0; i < n; ++i) {
    if (ops[i].kind == REC_PUT) ops[i].put.counter = l->priv + 2 * i;
    if (ops[i].kind == REC_REDUCE) {
      ops[i].red.counter = l->priv + 2 * i + 1;
      ops[i].red.scratch = (float *)(l->priv + 2 * n + (size_t)kScratchBlocks * i);
    }
    rec_footprint(ops[i], fp[i]);
  }
  cudaGraph_t graph;
  CUDA_TRY(cudaGraphCreate(&graph, 0));
  std::vector<cudaGraphNode_t> node(n);
  uint32_t edges = 0;
  for (size_t j = 0; j < n; ++j) {
    std::vector<cudaGraphNode_t> deps;
    for (size_t i = 0; i < j; ++i)
      if (rec_conflict(fp[i], fp[j])) deps.push_back(node[i]);
    edges += (uint32_t)deps.size();
    RecOp &op = ops[j];
    cudaKernelNodeParams kp;
    memset(&kp, 0, sizeof kp);
    kp.gridDim = dim3((unsigned)op.grid);
    kp.blockDim = dim3((unsigned)op.block);
    void *args[8];
    const auto &m = op.mm;
    switch (op.kind) {
      case REC_PUT:
        args[0] = &op.put;
        kp.func = op.variant == 0   ? (void *)k_put<8, false>
                  : op.variant == 1 ? (void *)k_put<8, true>
                  : op.variant == 2 ? (void *)k_put<4, false>
                  : op.variant == 3 ? (void *)k_put<4, true>
                                    : (void *)k_put_bulk;
        if (op.variant == 4) kp.sharedMemBytes = kBulkSmem;
        break;
      case REC_INLINE:
        args[0] = op.inl;
        kp.func = (void *)k_put_inline;
        break;
      case REC_GEN:
        args[0] = &op.gen.dst; args[1] = &op.gen.nf; args[2] = &op.gen.e0;
        args[3] = &op.gen.seed; args[4] = &op.gen.node; args[5] = &op.gen.iteration;
        args[6] = &l->iter_add;
        kp.func = (void *)k_gen_reference;
        break;
      case REC_APPLY:
        args[0] = &op.apply;
        kp.func = op.apply_sgd ? (void *)k_apply_sgd : (void *)k_apply_xor;
        break;
      case REC_REDUCE:
        args[0] = &op.red.in; args[1] = &op.red.n; args[2] = &op.red.out;
        args[3] = &op.red.scratch; args[4] = &op.red.counter;
        kp.func = (void *)k_reduce_max;
        break;
      case REC_CLEAR:
        args[0] = &op.clr.dev; args[1] = &op.clr.shadow;
        kp.func = (void *)k_clear_flag;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        break;
      case REC_EWISE: {
        const auto &w = op.ew;
        if (w.op == 1) {
          args[0] = (void *)&w.a; args[1] = (void *)&w.b; args[2] = (void *)&w.out;
          args[3] = (void *)&w.n;
          kp.func = w.elem == 0   ? (void *)k_add<float>
                    : w.elem == 1 ? (void *)k_add<double>
                    : w.elem == 2 ? (void *)k_add<int32_t>
                    : w.elem == 3 ? (void *)k_add<int64_t>
                                  : (void *)k_add<uint8_t>;
        } else {
          args[0] = (void *)&w.a; args[1] = (void *)&w.out; args[2] = (void *)&w.n;
          kp.func = w.elem == 0 ? (void *)k_sigmoid<float> : (void *)k_sigmoid<double>;
        }
        break;
      }
      case REC_MATMUL:
        args[0] = (void *)&m.a; args[1] = (void *)&m.b; args[2] = (void *)&m.c;
        args[3] = (void *)&m.m; args[4] = (void *)&m.k; args[5] = (void *)&m.n;
        kp.func = m.elem == 0   ? (void *)k_matmul<float>
                  : m.elem == 1 ? (void *)k_matmul<double>
                  : m.elem == 2 ? (void *)k_matmul<int32_t>
                  : m.elem == 3 ? (void *)k_matmul<int64_t>
                                : (void *)k_matmul<uint8_t>;
        break;
    }
    kp.kernelParams = args;
    cudaError_t e = cudaGraphAddKernelNode(&node[j], graph, deps.data(), deps.size(), &kp);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      return fail(SRF_E_DEVICE, "replay graph node %zu: %s", j, cudaGetErrorString(e));
    }
  }
  cudaError_t e = cudaGraphInstantiate(&l->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(SRF_E_DEVICE, "replay instantiate: %s", cudaGetErrorString(e));
  l->nodes = (uint32_t)n;
  l->edges = edges;
  return SRF_OK;
}
