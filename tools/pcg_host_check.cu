// Host run of the device PCG64 GenGrad code (csrc/device_pcg.cuh) over a
// simulated grid of nth threads, for checking against numpy without a GPU:
//   nvcc -std=c++17 -o /tmp/pcg_host tools/pcg_host_check.cu
//   /tmp/pcg_host seed node iteration nf e0 nth out.bin
// tests/test_host.py::test_device_pcg_stream_on_host drives it.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1805_08430_b200/csrc/device_pcg.cuh"

int main(int argc, char **argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: seed node iteration nf e0 nth out\n");
    return 2;
  }
  const uint64_t seed = strtoull(argv[1], 0, 0), node = strtoull(argv[2], 0, 0);
  const uint64_t it = strtoull(argv[3], 0, 0), nf = strtoull(argv[4], 0, 0);
  const uint64_t e0 = strtoull(argv[5], 0, 0), nth = strtoull(argv[6], 0, 0);
  std::vector<float> out(nf + 4, -1.0f);
  const PcgStream p = pcg_node_stream(seed, node, it);
  for (uint64_t t = 0; t < nth; ++t) pcg_fill_f32(out.data(), nf, e0, p, t, nth);
  FILE *f = fopen(argv[7], "wb");
  fwrite(out.data(), 4, nf, f);
  fclose(f);
  return 0;
}
