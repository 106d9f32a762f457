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
};

struct srf_oplist {
  std::vector<RecOp> ops;
  int device = -1;
  bool dirty = false;
  std::string why;
  // replay state
  cudaGraphExec_t exec = nullptr;
  uint64_t *iter_add = nullptr;  // device counter: GenGrad iteration offset
  int graph_device = -1;
  ~srf_oplist() {
    for (RecOp &op : ops) delete op.inl;
    if (exec) cudaGraphExecDestroy(exec);
    if (iter_add) cudaFree(iter_add);
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
  }
  return false;
}

// Issue one recorded iteration on stream s (GenGrad iteration = recorded +
// *iter_add, read on the device).
static cudaError_t rec_issue(const srf_oplist *l, cudaStream_t s, const uint64_t *iter_add) {
  for (const RecOp &op : l->ops) {
    switch (op.kind) {
      case REC_PUT:
        switch (op.variant) {
          case 0: k_put<8, false><<<op.grid, op.block, 0, s>>>(op.put); break;
          case 1: k_put<8, true><<<op.grid, op.block, 0, s>>>(op.put); break;
          case 2: k_put<4, false><<<op.grid, op.block, 0, s>>>(op.put); break;
          case 3: k_put<4, true><<<op.grid, op.block, 0, s>>>(op.put); break;
          default: k_put_bulk<<<op.grid, op.block, kBulkSmem, s>>>(op.put); break;
        }
        break;
      case REC_INLINE: k_put_inline<<<1, 256, 0, s>>>(*op.inl); break;
      case REC_GEN:
        k_gen_reference<<<op.grid, 512, 0, s>>>(op.gen.dst, op.gen.nf, op.gen.e0, op.gen.seed,
                                                 op.gen.node, op.gen.iteration, iter_add);
        break;
      case REC_APPLY:
        if (op.apply_sgd)
          k_apply_sgd<<<op.grid, op.block, 0, s>>>(op.apply);
        else
          k_apply_xor<<<op.grid, op.block, 0, s>>>(op.apply);
        break;
      case REC_REDUCE:
        k_reduce_max<<<op.grid, 256, 0, s>>>(op.red.in, op.red.n, op.red.out, op.red.scratch,
                                             op.red.counter);
        break;
      case REC_CLEAR: k_clear_flag<<<1, 1, 0, s>>>(op.clr.dev, op.clr.shadow); break;
      case REC_MATMUL: {
        const unsigned g = (unsigned)op.grid;
        const auto &m = op.mm;
        switch (m.elem) {
          case 0: k_matmul<float><<<g, 256, 0, s>>>((const float *)m.a, (const float *)m.b, (float *)m.c, m.m, m.k, m.n); break;
          case 1: k_matmul<double><<<g, 256, 0, s>>>((const double *)m.a, (const double *)m.b, (double *)m.c, m.m, m.k, m.n); break;
          case 2: k_matmul<int32_t><<<g, 256, 0, s>>>((const int32_t *)m.a, (const int32_t *)m.b, (int32_t *)m.c, m.m, m.k, m.n); break;
          case 3: k_matmul<int64_t><<<g, 256, 0, s>>>((const int64_t *)m.a, (const int64_t *)m.b, (int64_t *)m.c, m.m, m.k, m.n); break;
          default: k_matmul<uint8_t><<<g, 256, 0, s>>>((const uint8_t *)m.a, (const uint8_t *)m.b, (uint8_t *)m.c, m.m, m.k, m.n); break;
        }
        break;
      }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
