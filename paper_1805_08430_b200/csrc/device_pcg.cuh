// device_pcg.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// The reference's GenGrad value stream on the device, bit-exact.
//
// The reference draws every synthetic tensor as
//   Generator(PCG64(mix)).random(n, dtype=float32),
//   mix = ((seed & 0xFFFFFFFF) * 1000003 + node) * 1000033 + iteration  (mod 2^64)
// (graph.py:333-350, node_rng + synthesize_values).  numpy pins the algorithm:
//   * PCG64(int) seeds through SeedSequence(int).generate_state(4, uint64)
//     (32-bit hash mixing of the integer's 32-bit words) and
//     pcg64_set_seed(initstate = s0:s1, initseq = s2:s3);
//   * PCG64 is the 128-bit LCG  s <- s * MULT + inc  whose 64-bit output is
//     XSL-RR of the NEW state;
//   * random(float32) takes 32-bit halves of consecutive outputs, low half
//     first, and maps h -> (h >> 8) * 2^-24.
// So element i of the tensor is the (i & 1) half of raw output i >> 1, and a
// thread can start anywhere: the LCG jumps d steps in O(log d) with the table
// in pcg_table.cuh.  Each thread writes 8-float (32-B) chunks, grid-strided,
// re-using one precomputed stride jump per chunk; the kernel is HBM-store
// bound like the reference's np.random fill it replaces.
// tools/gen_pcg_table.py; tests/test_gpu_pcg.py checks it against numpy.

#include "pcg_table.cuh"

// Host+device so tools/pcg_host_check.cu can run the same code on the CPU.
#ifdef __CUDA_ARCH__
#define SRF_PCG_TABLE kPcgJump
#define SRF_HD __device__ __forceinline__
#else
#define SRF_PCG_TABLE kPcgJumpHost
#define SRF_HD __host__ __device__ inline
#endif

struct u128 {
  uint64_t lo, hi;
};

SRF_HD uint64_t umul64hi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

SRF_HD u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

SRF_HD u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

SRF_HD u128 mad128(u128 a, u128 b, u128 c) { return add128(mul128(a, b), c); }

static constexpr uint64_t kPcgMultLo = 4865540595714422341ull;
static constexpr uint64_t kPcgMultHi = 2549297995355413924ull;

struct PcgStream {
  u128 state;  // state before the first output
  u128 inc;
};

// One LCG step and the XSL-RR output of the new state (pcg64_random_r).
SRF_HD uint64_t pcg_next(u128 &s, const u128 &inc) {
  s = mad128(s, u128{kPcgMultLo, kPcgMultHi}, inc);
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// (A_d, G_d) of a d-step jump: s_{+d} = A_d * s + G_d * inc.
SRF_HD void pcg_jump_coeffs(uint64_t d, u128 &A, u128 &G) {
  A = u128{1, 0};
  G = u128{0, 0};
  for (int k = 0; d; ++k, d >>= 1) {
    if (d & 1) {
      const u128 Ak{SRF_PCG_TABLE[k][0], SRF_PCG_TABLE[k][1]};
      const u128 Gk{SRF_PCG_TABLE[k][2], SRF_PCG_TABLE[k][3]};
      G = mad128(G, Ak, Gk);
      A = mul128(A, Ak);
    }
  }
}

SRF_HD void pcg_advance(u128 &s, const u128 &inc, uint64_t d) {
  for (int k = 0; d; ++k, d >>= 1) {
    if (d & 1) {
      const u128 Ak{SRF_PCG_TABLE[k][0], SRF_PCG_TABLE[k][1]};
      const u128 Gk{SRF_PCG_TABLE[k][2], SRF_PCG_TABLE[k][3]};
      s = add128(mul128(Ak, s), mul128(Gk, inc));
    }
  }
}

// numpy SeedSequence(entropy).generate_state(4, np.uint64) for an entropy
// integer < 2^64 (its 32-bit words, least significant first; 0 -> [0]),
// pool size 4, no spawn key.
SRF_HD uint32_t ss_hashmix(uint32_t v, uint32_t &hc) {
  v ^= hc;
  hc *= 0x931e8875u;  // MULT_A
  v *= hc;
  v ^= v >> 16;
  return v;
}

SRF_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;  // MIX_MULT_L, MIX_MULT_R
  r ^= r >> 16;
  return r;
}

SRF_HD void seed_sequence4(uint64_t entropy, uint64_t out[4]) {
  const uint32_t w0 = (uint32_t)entropy, w1 = (uint32_t)(entropy >> 32);
  uint32_t hc = 0x43b0d7e5u;  // INIT_A
  uint32_t pool[4];
  pool[0] = ss_hashmix(w0, hc);
  pool[1] = ss_hashmix(w1, hc);  // 0 when the entropy has one word: same as padding
  pool[2] = ss_hashmix(0u, hc);
  pool[3] = ss_hashmix(0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  uint32_t h = 0x8b51f9ddu;  // INIT_B
  uint32_t st[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= h;
    h *= 0x58f38dedu;  // MULT_B
    v *= h;
    v ^= v >> 16;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}

// Generator(PCG64(mix)) of node_rng(seed, node, iteration) (graph.py:333-336).
SRF_HD PcgStream pcg_node_stream(uint64_t seed, uint64_t node, uint64_t iteration) {
  const uint64_t mix = ((seed & 0xFFFFFFFFull) * 1000003ull + node) * 1000033ull + iteration;
  uint64_t s[4];
  seed_sequence4(mix, s);
  PcgStream p;
  // pcg64_set_seed: initstate = s0:s1 (hi:lo), initseq = s2:s3; srandom_r
  p.inc = u128{(s[3] << 1) | 1ull, (s[2] << 1) | (s[3] >> 63)};
  u128 st = p.inc;                    // 0 * MULT + inc
  st = add128(st, u128{s[1], s[0]});  // += initstate
  p.state = mad128(st, u128{kPcgMultLo, kPcgMultHi}, p.inc);
  return p;
}

SRF_HD float pcg_half_to_f32(uint32_t h) {
  return (float)(h >> 8) * (1.0f / 16777216.0f);  // exact: h >> 8 < 2^24
}

// 8-float chunks c = t, t+nth, ... of dst (elements e0 + 8c ..).  kOdd: e0 is
// odd, so a chunk starts on the high half of raw r and ends on the low half
// of raw r+4.
template <int kOdd>
SRF_HD void pcg_fill_chunks(float *dst, uint64_t nchunks, uint64_t e0, const PcgStream &p,
                            uint64_t t, uint64_t nth) {
  u128 s = p.state;
  pcg_advance(s, p.inc, (e0 + 8 * t) >> 1);
  u128 A, G;
  pcg_jump_coeffs(4 * (nth - 1), A, G);  // from raw r+4 to the next chunk's r
  const u128 C = mul128(G, p.inc);
  for (uint64_t c = t; c < nchunks; c += nth) {
    uint32_t h[10];
    for (int j = 0; j < 4; ++j) {
      const uint64_t r = pcg_next(s, p.inc);
      h[2 * j] = (uint32_t)r;
      h[2 * j + 1] = (uint32_t)(r >> 32);
    }
    if (kOdd) {  // the 5th raw from a copy: s stays at r+4
      u128 s5 = s;
      const uint64_t r = pcg_next(s5, p.inc);
      h[8] = (uint32_t)r;
      h[9] = (uint32_t)(r >> 32);
    }
    float4 a, b;
    a.x = pcg_half_to_f32(h[kOdd + 0]);
    a.y = pcg_half_to_f32(h[kOdd + 1]);
    a.z = pcg_half_to_f32(h[kOdd + 2]);
    a.w = pcg_half_to_f32(h[kOdd + 3]);
    b.x = pcg_half_to_f32(h[kOdd + 4]);
    b.y = pcg_half_to_f32(h[kOdd + 5]);
    b.z = pcg_half_to_f32(h[kOdd + 6]);
    b.w = pcg_half_to_f32(h[kOdd + 7]);
    float4 *d4 = (float4 *)(dst + 8 * c);
    d4[0] = a;
    d4[1] = b;
    s = mad128(A, s, C);
  }
}

// Fill dst[0, nf) with elements e0 .. e0+nf-1 of the stream (floats of the
// whole tensor; e0 > 0 for a slice), threads [t, +nth) of some grid.
// dst must be 16-B aligned.
SRF_HD void pcg_fill_f32(float *dst, uint64_t nf, uint64_t e0, const PcgStream &p, uint64_t t,
                         uint64_t nth) {
  const uint64_t nchunks = nf / 8;
  if (t < nchunks) {
    if (e0 & 1)
      pcg_fill_chunks<1>(dst, nchunks, e0, p, t, nth);
    else
      pcg_fill_chunks<0>(dst, nchunks, e0, p, t, nth);
  }
  // tail elements (nf % 8 < 8), one per thread
  const uint64_t rem = nf - 8 * nchunks;
  for (uint64_t j = t; j < rem; j += nth) {
    const uint64_t e = e0 + 8 * nchunks + j;
    u128 s = p.state;
    pcg_advance(s, p.inc, e >> 1);
    const uint64_t r = pcg_next(s, p.inc);
    dst[8 * nchunks + j] = pcg_half_to_f32((e & 1) ? (uint32_t)(r >> 32) : (uint32_t)r);
  }
}

#ifdef __CUDACC__
// CTA-cooperative fill for CTA `cta` of `ctas` covering one tensor slice,
// leapfrogged: a thread keeps the 4 (odd start: 5) LCG states whose outputs
// fill its current 8-float chunk and jumps each of them straight to its next
// chunk (M^(4 nth) and the matching increment), so the states advance as
// independent chains - ILP 4-5 and one 128-bit multiply-add per 64-bit output.
// Thread 0 derives the stream (SeedSequence + seeding), the CTA's base state
// and the jump once; the other threads advance by 4 * tid raws (<= 11 jump
// bits).  Same values as pcg_fill_f32.
template <int kOdd>
__device__ __forceinline__ void pcg_chunks_leapfrog(float *dst, uint64_t nchunks, uint64_t t,
                                                    uint64_t nth, u128 s0, const u128 &inc,
                                                    const u128 &A, const u128 &C) {
  constexpr int NR = 4 + kOdd;
  u128 st[NR];  // st[j]: the state whose XSL-RR is raw r0 + j (already stepped)
  st[0] = s0;
#pragma unroll
  for (int j = 1; j < NR; ++j) st[j] = mad128(st[j - 1], u128{kPcgMultLo, kPcgMultHi}, inc);
  for (uint64_t c = t; c < nchunks; c += nth) {
    uint32_t h[2 * NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const uint64_t x = st[j].hi ^ st[j].lo;
      const unsigned rot = (unsigned)(st[j].hi >> 58);
      const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
      h[2 * j] = (uint32_t)r;
      h[2 * j + 1] = (uint32_t)(r >> 32);
      st[j] = mad128(A, st[j], C);
    }
    float4 a = make_float4(pcg_half_to_f32(h[kOdd + 0]), pcg_half_to_f32(h[kOdd + 1]),
                           pcg_half_to_f32(h[kOdd + 2]), pcg_half_to_f32(h[kOdd + 3]));
    float4 b = make_float4(pcg_half_to_f32(h[kOdd + 4]), pcg_half_to_f32(h[kOdd + 5]),
                           pcg_half_to_f32(h[kOdd + 6]), pcg_half_to_f32(h[kOdd + 7]));
    float4 *d4 = (float4 *)(dst + 8 * c);
    d4[0] = a;
    d4[1] = b;
  }
}

__device__ void pcg_fill_f32_cta(float *dst, uint64_t nf, uint64_t e0, uint64_t seed,
                                 uint64_t node, uint64_t iteration, uint64_t cta,
                                 uint64_t ctas) {
  __shared__ u128 s_base, s_inc, s_A, s_C, s_state0;
  const uint64_t nth = ctas * blockDim.x;
  // dst may be only 4-B aligned (arena blocks are 8-B aligned,
  // memspace.py:31): the first `head` floats take the scalar path and the
  // vector path starts at the first 16-B boundary
  uint64_t head = ((16 - ((uintptr_t)dst & 15)) & 15) / 4;
  if (head > nf) head = nf;
  float *vdst = dst + head;
  const uint64_t vnf = nf - head, ve0 = e0 + head;
  if (threadIdx.x == 0) {
    const PcgStream p = pcg_node_stream(seed, node, iteration);
    u128 b = p.state;
    // stepped state of the CTA's first raw: (ve0 >> 1) + 4 * cta * blockDim + 1 steps
    pcg_advance(b, p.inc, ((ve0 >> 1) + 4 * cta * blockDim.x) + 1);
    u128 A, G;
    pcg_jump_coeffs(4 * nth, A, G);
    s_base = b;
    s_inc = p.inc;
    s_A = A;
    s_C = mul128(G, p.inc);
    s_state0 = p.state;
  }
  __syncthreads();
  const uint64_t t = cta * blockDim.x + threadIdx.x;
  const uint64_t nchunks = vnf / 8;
  const u128 inc = s_inc;
  if (t < nchunks) {
    u128 s = s_base;
    pcg_advance(s, inc, 4 * (uint64_t)threadIdx.x);
    if (ve0 & 1)
      pcg_chunks_leapfrog<1>(vdst, nchunks, t, nth, s, inc, s_A, s_C);
    else
      pcg_chunks_leapfrog<0>(vdst, nchunks, t, nth, s, inc, s_A, s_C);
  }
  // scalar floats: the unaligned head, then the tail of the vector range
  const uint64_t rem = vnf - 8 * nchunks;
  for (uint64_t j = t; j < head + rem; j += nth) {
    const uint64_t local = j < head ? j : head + 8 * nchunks + (j - head);
    const uint64_t e = e0 + local;
    u128 s = s_state0;
    pcg_advance(s, inc, e >> 1);
    const uint64_t r = pcg_next(s, inc);
    dst[local] = pcg_half_to_f32((e & 1) ? (uint32_t)(r >> 32) : (uint32_t)r);
  }
  __syncthreads();  // the shared stream state is reused by the CTA's next unit
}

// Standalone GenGrad / Input on the device: synthesize_values(dims, F32,
// node_rng(seed, node, iteration)) elements [e0, e0 + nf) into dst.
// iter_add (nullptr: none): a device counter added to `iteration` - a
// replayed Session iteration (host_record.cuh) advances it per replay.
__global__ void __launch_bounds__(512) k_gen_reference(float *dst, uint64_t nf, uint64_t e0,
                                                       uint64_t seed, uint64_t node,
                                                       uint64_t iteration,
                                                       const uint64_t *iter_add) {
  if (iter_add) iteration += *(const volatile uint64_t *)iter_add;
  pcg_fill_f32_cta(dst, nf, e0, seed, node, iteration, blockIdx.x, gridDim.x);
}
#endif
