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
  cudaEvent_t done = nullptr;    // after the exec's latest launch
  ~srf_oplist() {
    for (RecOp &op : ops) delete op.inl;
    if (done) cudaEventDestroy(done);
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

// Kernel node parameters of one recorded op (args point into op, which must
// outlive the call that consumes kp).
static void rec_kernel_params(RecOp &op, uint64_t *const *iter_add,
                              cudaKernelNodeParams &kp, void **args) {
  memset(&kp, 0, sizeof kp);
  kp.gridDim = dim3((unsigned)op.grid);
  kp.blockDim = dim3((unsigned)op.block);
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
      args[6] = (void *)iter_add;
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
}

// Build l->exec: one kernel node per op, an edge from every earlier op it
// conflicts with that is not already an ancestor.
static int rec_build_graph(srf_oplist *l) {
  const size_t n = l->ops.size();
  static const bool timing = getenv("SRFLOW_REPLAY_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return (long long)std::chrono::duration_cast<std::chrono::microseconds>(b - a).count();
  };
  const auto t_begin = now();
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
  const auto t_alloc = now();
  cudaGraph_t graph;
  CUDA_TRY(cudaGraphCreate(&graph, 0));
  std::vector<cudaGraphNode_t> node(n);
  uint32_t edges = 0;
  // transitive reduction on the fly: walking earlier ops newest first, a
  // conflicting op that is already an ancestor (through a newer dependency)
  // needs no edge of its own.  Ancestor sets are bitsets; without this, the
  // ~600-op iterations of a 7-worker graph carried O(n^2) edges and took
  // ~120 ms per graph to build and instantiate.
  const size_t words64 = (n + 63) / 64;
  std::vector<uint64_t> anc(n * words64, 0);
  for (size_t j = 0; j < n; ++j) {
    std::vector<cudaGraphNode_t> deps;
    uint64_t *aj = &anc[j * words64];
    for (size_t i = j; i-- > 0;) {
      if ((aj[i / 64] >> (i % 64)) & 1) continue;
      if (!rec_conflict(fp[i], fp[j])) continue;
      deps.push_back(node[i]);
      const uint64_t *ai = &anc[i * words64];
      for (size_t w = 0; w < words64; ++w) aj[w] |= ai[w];
      aj[i / 64] |= 1ull << (i % 64);
    }
    edges += (uint32_t)deps.size();
    RecOp &op = ops[j];
    void *args[8];
    cudaKernelNodeParams kp;
    rec_kernel_params(op, &l->iter_add, kp, args);
    cudaError_t e = cudaGraphAddKernelNode(&node[j], graph, deps.data(), deps.size(), &kp);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      return fail(SRF_E_DEVICE, "replay graph node %zu: %s", j, cudaGetErrorString(e));
    }
  }
  const auto t_nodes = now();
  cudaError_t e = cudaGraphInstantiate(&l->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (timing)
    fprintf(stderr, "[srflow] replay graph: %zu ops, %u edges: alloc %lld us, nodes %lld us, "
            "instantiate %lld us\n", n, edges, us(t_begin, t_alloc), us(t_alloc, t_nodes),
            us(t_nodes, now()));
  if (e != cudaSuccess) return fail(SRF_E_DEVICE, "replay instantiate: %s", cudaGetErrorString(e));
  l->nodes = (uint32_t)n;
  l->edges = edges;
  return SRF_OK;
}


// Indirect replay kernels: node parameters that never change (the argument
// table, the phase word, the op index); the op's arguments for the current
// phase are read from device memory - table[phase * n + i] - so switching
// phases costs one device word, not a host update of every changed node
// (cudaGraphExecKernelNodeSetParams + relaunch measured ~13 us per node).
struct IndArgs {
  const void *const *table;
  const uint32_t *phase;
  uint32_t n, i;
};
struct GenArgs {
  float *dst;
  uint64_t nf, e0, seed, node, iteration;
};

__device__ __forceinline__ const void *ind_args(const IndArgs &ia) {
  const uint32_t p = *(const volatile uint32_t *)ia.phase;
  return ia.table[(size_t)p * ia.n + ia.i];
}

// the CTA stages its argument blob in shared memory first: the bodies then
// read arguments that no global store can alias (from global memory, every
// field - the apply's gradient pointers per element - would be reloaded)
template <typename A>
__device__ __forceinline__ const A &ind_stage(const IndArgs &ia, A *smem) {
  static_assert(sizeof(A) % 4 == 0, "argument blobs are word-sized");
  const uint32_t *src = (const uint32_t *)ind_args(ia);
  uint32_t *dst = (uint32_t *)smem;
  for (uint32_t k = threadIdx.x; k < sizeof(A) / 4; k += blockDim.x) dst[k] = src[k];
  __syncthreads();
  return *smem;
}

template <int U16, bool kSectors>
__global__ void __launch_bounds__(512) k_put_ind(const __grid_constant__ IndArgs ia) {
  __shared__ __align__(16) PutArgs sa;
  put_body<U16, kSectors>(ind_stage(ia, &sa));
}

__global__ void __launch_bounds__(256) k_put_inline_ind(const __grid_constant__ IndArgs ia) {
  __shared__ __align__(16) InlineArgs sa;
  put_inline_body(ind_stage(ia, &sa));
}

__global__ void __launch_bounds__(512) k_gen_ind(const __grid_constant__ IndArgs ia,
                                                 const uint64_t *iter_add) {
  __shared__ __align__(16) GenArgs sa;
  const GenArgs &g = ind_stage(ia, &sa);
  pcg_fill_f32_cta(g.dst, g.nf, g.e0, g.seed, g.node,
                   g.iteration + *(const volatile uint64_t *)iter_add, blockIdx.x, gridDim.x);
}

template <bool kSgd>
__global__ void __launch_bounds__(512) k_apply_ind(const __grid_constant__ IndArgs ia) {
  __shared__ __align__(16) ApplyArgs sa;
  const ApplyArgs &a = ind_stage(ia, &sa);
  apply_range<kSgd>(a.var, a.g, a.nw, a.n, a.lr, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                    (uint64_t)gridDim.x * blockDim.x);
}

__global__ void k_set_replay(uint64_t *iter_add, uint64_t it, uint32_t *phase, uint32_t p) {
  *iter_add = it;
  *phase = p;
}

// the indirect twin of an op's kernel, or nullptr (the op keeps a direct node)
static const void *rec_ind_func(const RecOp &op) {
  switch (op.kind) {
    case REC_PUT:
      return op.variant == 0   ? (const void *)k_put_ind<8, false>
             : op.variant == 1 ? (const void *)k_put_ind<8, true>
             : op.variant == 2 ? (const void *)k_put_ind<4, false>
             : op.variant == 3 ? (const void *)k_put_ind<4, true>
                               : nullptr;
    case REC_INLINE: return (const void *)k_put_inline_ind;
    case REC_GEN: return (const void *)k_gen_ind;
    case REC_APPLY: return op.apply_sgd ? (const void *)k_apply_ind<true>
                                        : (const void *)k_apply_ind<false>;
  }
  return nullptr;
}

// the argument blob an indirect kernel reads
static size_t rec_ind_blob(const RecOp &op, uint8_t *out) {
  switch (op.kind) {
    case REC_PUT: memcpy(out, &op.put, sizeof op.put); return sizeof op.put;
    case REC_INLINE: memcpy(out, op.inl, sizeof(InlineArgs)); return sizeof(InlineArgs);
    case REC_GEN: {
      GenArgs g{op.gen.dst, op.gen.nf, op.gen.e0, op.gen.seed, op.gen.node, op.gen.iteration};
      memcpy(out, &g, sizeof g);
      return sizeof g;
    }
    case REC_APPLY: memcpy(out, &op.apply, sizeof op.apply); return sizeof op.apply;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Replay set: the recordings of ALL phases of a steady-state period behind ONE
// instantiated graph.  A long period (the 7-worker LSTM graph repeats its
// arena state every 168 iterations) would otherwise instantiate one graph per
// phase (~25-75 ms each for ~700 nodes).  Phases have the same op sequence
// (kinds, functions, launch shapes); only some arguments differ (the arena
// blocks a dynamic edge cycles through).  The graph's edges are the union of
// every phase's conflicts (transitively reduced); before each launch the
// nodes whose parameters differ from the phase last loaded are updated with
// cudaGraphExecKernelNodeSetParams (launches already queued keep their own
// parameters).  GenGrad nodes store their iteration relative to their phase's
// recorded iteration; the device word adds the replayed iteration.
// ---------------------------------------------------------------------------
struct srf_replay_set {
  int device = -1;
  uint32_t nphase = 0, n = 0, edges = 0;
  std::vector<std::vector<RecOp>> ops;   // [phase][op], patched (private counters)
  std::vector<uint32_t> cls;             // [phase * n + op]: parameter class
  // kExecs instantiations of the same graph used round robin: updating and
  // launching an exec whose previous launch is still running serialises the
  // host with the device (measured ~4 ms per 700-node launch); with several
  // copies the one being updated finished long ago
  static constexpr int kExecs = 4;
  std::vector<uint32_t> loaded[kExecs];  // [op]: class loaded in exec k
  std::vector<cudaGraphNode_t> node;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec[kExecs] = {};
  cudaEvent_t done[kExecs] = {};         // after each exec's latest launch
  uint32_t next_exec = 0;
  uint64_t *iter_add = nullptr;
  unsigned int *priv = nullptr;
  uint32_t *phase = nullptr;             // device word: the phase being replayed
  uint8_t *blobs = nullptr;              // device: argument blobs of indirect ops
  const void **table = nullptr;          // device: [phase * n + op] -> blob
  std::vector<uint8_t> indirect;         // [op]: 1 when its node reads the table
  uint64_t updates = 0;
  ~srf_replay_set() {
    if (phase) cudaFree(phase);
    if (blobs) cudaFree(blobs);
    if (table) cudaFree((void *)table);
    for (auto &e : exec)
      if (e) cudaGraphExecDestroy(e);
    for (auto &e : done)
      if (e) cudaEventDestroy(e);
    if (graph) cudaGraphDestroy(graph);
    if (iter_add) cudaFree(iter_add);
    if (priv) cudaFree(priv);
  }
};

static bool rec_same_function(const RecOp &x, const RecOp &y) {
  if (x.kind != y.kind || x.device != y.device || x.grid != y.grid || x.block != y.block ||
      x.variant != y.variant)
    return false;
  switch (x.kind) {
    case REC_APPLY: return x.apply_sgd == y.apply_sgd;
    case REC_MATMUL: return x.mm.elem == y.mm.elem;
    case REC_EWISE: return x.ew.op == y.ew.op && x.ew.elem == y.ew.elem;
  }
  return true;
}

static int rec_set_build(srf_replay_set *rs, srf_oplist *const *lists, const int64_t *iters) {
  const uint32_t P = rs->nphase, n = rs->n;
  const size_t words = 2 * (size_t)n + (size_t)kScratchBlocks * n;
  CUDA_TRY(cudaMalloc(&rs->iter_add, sizeof(uint64_t)));
  CUDA_TRY(cudaMemset(rs->iter_add, 0, sizeof(uint64_t)));
  CUDA_TRY(cudaMalloc(&rs->priv, sizeof(unsigned int) * words));
  CUDA_TRY(cudaMemset(rs->priv, 0, sizeof(unsigned int) * words));
  rs->ops.resize(P);
  for (uint32_t p = 0; p < P; ++p) {
    std::vector<RecOp> &ops = rs->ops[p];
    ops = lists[p]->ops;
    for (uint32_t i = 0; i < n; ++i) {
      RecOp &op = ops[i];
      if (op.inl) op.inl = new InlineArgs(*op.inl);  // owned copies (freed in destroy)
      if (op.kind == REC_PUT) op.put.counter = rs->priv + 2 * i;
      if (op.kind == REC_REDUCE) {
        op.red.counter = rs->priv + 2 * i + 1;
        op.red.scratch = (float *)(rs->priv + 2 * (size_t)n + (size_t)kScratchBlocks * i);
      }
      if (op.kind == REC_GEN) op.gen.iteration -= (uint64_t)iters[p];
    }
  }
  // parameter classes per op: the first phase with identical parameters
  // (only class representatives are compared: an op cycles through a few)
  rs->cls.assign((size_t)P * n, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t p = 0; p < P; ++p) {
      uint32_t c = p;
      for (uint32_t q = 0; q < p; ++q)
        if (rs->cls[(size_t)q * n + i] == q && rec_same(rs->ops[q][i], rs->ops[p][i], 0)) {
          c = q;
          break;
        }
      rs->cls[(size_t)p * n + i] = c;
    }
  // conflicts: phase 0's, plus, per later phase, the pairs involving an op
  // whose parameters differ from phase 0's (other pairs conflict identically)
  const size_t words64 = (n + 63) / 64;
  std::vector<uint64_t> conf((size_t)n * words64, 0);  // bit i of row j: i < j conflict
  auto set_conf = [&](uint32_t i, uint32_t j) {
    if (i > j) std::swap(i, j);
    conf[(size_t)j * words64 + i / 64] |= 1ull << (i % 64);
  };
  std::vector<std::vector<Span>> fp0(n), fpp(n);
  for (uint32_t i = 0; i < n; ++i) rec_footprint(rs->ops[0][i], fp0[i]);
  for (uint32_t j = 0; j < n; ++j)
    for (uint32_t i = 0; i < j; ++i)
      if (rec_conflict(fp0[i], fp0[j])) set_conf(i, j);
  for (uint32_t p = 1; p < P; ++p) {
    std::vector<uint32_t> diff;
    for (uint32_t i = 0; i < n; ++i) {
      fpp[i].clear();
      if (rs->cls[(size_t)p * n + i] != rs->cls[i]) diff.push_back(i);
    }
    if (diff.empty()) continue;
    for (uint32_t i = 0; i < n; ++i) rec_footprint(rs->ops[p][i], fpp[i]);
    for (uint32_t d : diff)
      for (uint32_t i = 0; i < n; ++i)
        if (i != d && rec_conflict(fpp[d], fpp[i])) set_conf(i, d);
  }
  // ops whose arguments vary across phases read them from the device table
  constexpr size_t kBlob =
      (std::max(std::max(sizeof(PutArgs), sizeof(InlineArgs)),
                std::max(sizeof(ApplyArgs), sizeof(GenArgs))) + 63) & ~(size_t)63;
  rs->indirect.assign(n, 0);
  std::vector<size_t> blob_off((size_t)P * n, SIZE_MAX);  // [class phase * n + op]
  size_t blob_bytes = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const bool all_ind = getenv("SRFLOW_REPLAY_ALL_INDIRECT") != nullptr;  // probes
    const char *kinds = getenv("SRFLOW_REPLAY_IND_KINDS");  // probes: bitmask of RecKind
    bool varies = all_ind;
    for (uint32_t p = 1; p < P && !varies; ++p) varies = rs->cls[(size_t)p * n + i] != 0;
    if (!varies || !rec_ind_func(rs->ops[0][i])) continue;
    if (kinds && !((atoi(kinds) >> rs->ops[0][i].kind) & 1)) continue;
    rs->indirect[i] = 1;
    for (uint32_t p = 0; p < P; ++p)
      if (rs->cls[(size_t)p * n + i] == p) {
        blob_off[(size_t)p * n + i] = blob_bytes;
        blob_bytes += kBlob;
      }
  }
  CUDA_TRY(cudaMalloc(&rs->phase, sizeof(uint32_t)));
  CUDA_TRY(cudaMemset(rs->phase, 0, sizeof(uint32_t)));
  if (blob_bytes) {
    std::vector<uint8_t> host(blob_bytes, 0);
    CUDA_TRY(cudaMalloc(&rs->blobs, blob_bytes));
    std::vector<const void *> tab((size_t)P * n, nullptr);
    for (uint32_t i = 0; i < n; ++i) {
      if (!rs->indirect[i]) continue;
      for (uint32_t p = 0; p < P; ++p) {
        const uint32_t c = rs->cls[(size_t)p * n + i];
        const size_t off = blob_off[(size_t)c * n + i];
        if (c == p) rec_ind_blob(rs->ops[p][i], host.data() + off);
        tab[(size_t)p * n + i] = rs->blobs + off;
      }
    }
    CUDA_TRY(cudaMemcpy(rs->blobs, host.data(), blob_bytes, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc((void **)&rs->table, sizeof(void *) * tab.size()));
    CUDA_TRY(cudaMemcpy((void *)rs->table, tab.data(), sizeof(void *) * tab.size(),
                        cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaGraphCreate(&rs->graph, 0));
  rs->node.resize(n);
  std::vector<uint64_t> anc((size_t)n * words64, 0);
  for (uint32_t j = 0; j < n; ++j) {
    std::vector<cudaGraphNode_t> deps;
    uint64_t *aj = &anc[(size_t)j * words64];
    const uint64_t *cj = &conf[(size_t)j * words64];
    for (uint32_t i = j; i-- > 0;) {
      if (!((cj[i / 64] >> (i % 64)) & 1) || ((aj[i / 64] >> (i % 64)) & 1)) continue;
      deps.push_back(rs->node[i]);
      const uint64_t *ai = &anc[(size_t)i * words64];
      for (size_t w = 0; w < words64; ++w) aj[w] |= ai[w];
      aj[i / 64] |= 1ull << (i % 64);
    }
    rs->edges += (uint32_t)deps.size();
    void *args[8];
    cudaKernelNodeParams kp;
    rec_kernel_params(rs->ops[0][j], &rs->iter_add, kp, args);
    IndArgs ia{rs->table, rs->phase, n, j};
    if (rs->indirect[j]) {
      kp.func = (void *)rec_ind_func(rs->ops[0][j]);
      kp.sharedMemBytes = 0;
      args[0] = &ia;
      args[1] = &rs->iter_add;  // k_gen_ind only
    }
    CUDA_TRY(cudaGraphAddKernelNode(&rs->node[j], rs->graph, deps.data(), deps.size(), &kp));
  }
  const auto t_inst = std::chrono::steady_clock::now();
  for (int k = 0; k < srf_replay_set::kExecs; ++k) {
    CUDA_TRY(cudaGraphInstantiate(&rs->exec[k], rs->graph, 0));
    CUDA_TRY(cudaEventCreateWithFlags(&rs->done[k], cudaEventDisableTiming));
    if (k == 0 && getenv("SRFLOW_REPLAY_TIMING")) {
      uint32_t nind = 0;
      for (uint8_t x : rs->indirect) nind += x;
      fprintf(stderr, "[srflow] replay set: %u phases, %u ops (%u indirect), %u edges; "
              "one instantiate %lld us\n", P, n, nind, rs->edges,
              (long long)std::chrono::duration_cast<std::chrono::microseconds>(
                  std::chrono::steady_clock::now() - t_inst).count());
    }
    rs->loaded[k].assign(n, 0);  // phase 0's parameters
  }
  return SRF_OK;
}

static int rec_set_launch(srf_replay_set *rs, uint32_t phase, uint64_t iteration, cudaStream_t st) {
  const uint32_t n = rs->n;
  static const bool timing = getenv("SRFLOW_REPLAY_TIMING") != nullptr;
  static uint64_t t_upd = 0, t_launch = 0, calls = 0, upd0 = 0;
  const auto t0 = std::chrono::steady_clock::now();
  const uint32_t *c = &rs->cls[(size_t)phase * n];
  static const int nexec = getenv("SRFLOW_REPLAY_EXECS")
                               ? std::max(1, std::min(srf_replay_set::kExecs,
                                                      atoi(getenv("SRFLOW_REPLAY_EXECS"))))
                               : srf_replay_set::kExecs;
  const int k = (int)(rs->next_exec++ % nexec);
  std::vector<uint32_t> &loaded = rs->loaded[k];
  // an exec is reused only after its previous launch finished (waiting here
  // is cheap; relaunching an exec that is still in flight stalled the host
  // ~3 ms per launch)
  static const bool no_wait = getenv("SRFLOW_REPLAY_NO_EXEC_WAIT") != nullptr;
  if (!no_wait) CUDA_TRY(cudaEventSynchronize(rs->done[k]));
  for (uint32_t i = 0; i < n; ++i) {
    if (loaded[i] == c[i] || rs->indirect[i]) continue;
    void *args[8];
    cudaKernelNodeParams kp;
    rec_kernel_params(rs->ops[c[i]][i], &rs->iter_add, kp, args);
    CUDA_TRY(cudaGraphExecKernelNodeSetParams(rs->exec[k], rs->node[i], &kp));
    loaded[i] = c[i];
    ++rs->updates;
  }
  const auto t1 = std::chrono::steady_clock::now();
  k_set_replay<<<1, 1, 0, st>>>(rs->iter_add, iteration, rs->phase, phase);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaGraphLaunch(rs->exec[k], st));
  CUDA_TRY(cudaEventRecord(rs->done[k], st));
  if (timing) {
    const auto t2 = std::chrono::steady_clock::now();
    t_upd += std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count();
    t_launch += std::chrono::duration_cast<std::chrono::microseconds>(t2 - t1).count();
    if (++calls % 128 == 0) {
      fprintf(stderr, "[srflow] replay set: %llu launches, %llu node updates, update %llu us, "
              "launch %llu us (cumulative)\n", (unsigned long long)calls,
              (unsigned long long)(rs->updates - upd0), (unsigned long long)t_upd,
              (unsigned long long)t_launch);
    }
  }
  return SRF_OK;
}
