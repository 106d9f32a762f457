// K1 body-copy variants on one GPU (same-device put, 256 MiB): access pattern
// and cache-hint experiments against cudaMemcpyAsync D2D.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

struct __align__(32) u256 { uint32_t v[8]; };

template <int HINT>
__device__ __forceinline__ u256 ld(const u256 *p) {
  u256 r;
  if (HINT == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                   "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  else if (HINT == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                   "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                   "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  return r;
}
template <int HINT>
__device__ __forceinline__ void st(u256 *p, const u256 &r) {
  if (HINT == 2)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]),
                 "r"(r.v[6]), "r"(r.v[7]) : "memory");
  else if (HINT == 3)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]),
                 "r"(r.v[6]), "r"(r.v[7]) : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]),
                 "r"(r.v[6]), "r"(r.v[7]) : "memory");
}

// grid-stride, U vectors in flight per thread (current K1)
template <int U, int LH, int SH>
__global__ void k_stride(u256 *dst, const u256 *src, uint64_t nv) {
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * nth < nv; i += U * nth) {
    u256 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld<LH>(src + i + u * nth);
#pragma unroll
    for (int u = 0; u < U; ++u) st<SH>(dst + i + u * nth, r[u]);
  }
  for (; i < nv; i += nth) st<SH>(dst + i, ld<LH>(src + i));
}

// tile-stride: CTA b copies contiguous tiles b, b+grid, ... of blockDim*U vectors
template <int U, int LH, int SH>
__global__ void k_tile(u256 *dst, const u256 *src, uint64_t nv) {
  const uint64_t tile = (uint64_t)blockDim.x * U;
  const uint64_t ntiles = nv / tile;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * tile + threadIdx.x;
    u256 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld<LH>(src + base + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) st<SH>(dst + base + u * blockDim.x, r[u]);
  }
  for (uint64_t i = ntiles * tile + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
       i += (uint64_t)gridDim.x * blockDim.x)
    st<SH>(dst + i, ld<LH>(src + i));
}

int main() {
  const uint64_t S = 256ull << 20, nv = S / 32;
  const int reps = 20;
  uint8_t *a, *b, *flush;
  cudaMalloc(&a, S);
  cudaMalloc(&b, S);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(a, 7, S);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9, tot = 0;
    for (int r = 0; r < reps; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);  // evict L2 between runs
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
      tot += ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"variant\": \"%s\", \"avg_us\": %.2f, \"best_us\": %.2f, \"hbm_gbs_avg\": %.1f, \"err\": \"%s\"}\n",
           name, tot / reps * 1e3, best * 1e3, 2.0 * S / (tot / reps * 1e-3) / 1e9,
           cudaGetErrorString(e));
  };
  timeit("cudaMemcpyAsync D2D", [&] { cudaMemcpyAsync(b, a, S, cudaMemcpyDeviceToDevice); });
  char name[128];
#define RUN(K, U, LH, SH, G, T)                                                            \
  snprintf(name, sizeof name, #K " U=%d ld%d st%d grid=%dx%d", U, LH, SH, G, T);            \
  timeit(name, [&] { K<U, LH, SH><<<G, T>>>((u256 *)b, (const u256 *)a, nv); });
  for (int g : {1, 2, 4}) {
    RUN(k_stride, 4, 0, 0, sms * g, 256);
    RUN(k_stride, 4, 1, 0, sms * g, 256);
    RUN(k_stride, 4, 2, 2, sms * g, 256);
    RUN(k_stride, 4, 0, 3, sms * g, 256);
    RUN(k_tile, 4, 0, 0, sms * g, 256);
    RUN(k_tile, 8, 0, 0, sms * g, 256);
    RUN(k_tile, 4, 1, 0, sms * g, 256);
    RUN(k_tile, 4, 2, 2, sms * g, 256);
    RUN(k_tile, 8, 1, 3, sms * g, 256);
    RUN(k_tile, 4, 0, 0, sms * g, 512);
  }
  // verify one variant
  cudaMemset(b, 0, S);
  k_tile<4, 1, 0><<<sms * 2, 256>>>((u256 *)b, (const u256 *)a, nv);
  std::vector<uint8_t> h(4096);
  cudaMemcpy(h.data(), b + S - 4096, 4096, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (auto x : h) bad += x != 7;
  printf("{\"verify_tail_bad\": %d}\n", bad);
  return 0;
}
