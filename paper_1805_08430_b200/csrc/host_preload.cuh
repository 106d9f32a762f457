// host_preload.cuh - part of libsrflow (included by srflow.cu, one translation unit).
// Eager loading of every kernel of the library on a device.
//
// CUDA 12 loads kernels lazily (CUDA_MODULE_LOADING=LAZY, the default): the
// first launch of a kernel loads it, and that load can wait for work already
// running on the device.  The flag protocols here run a spinning consumer
// kernel (K2, srf_edge_consume, the PS exchange) beside its producer on the
// same GPU; if the producer's first-ever launch has to load its module while
// the consumer spins, the two never run together and the consumer times out
// (observed: the first same-GPU pipelined edge of a process).  So the first
// space created on a device forces every kernel to load
// (cudaFuncGetAttributes), before any verb can launch.

static int preload_kernels(int device) {
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> g(mu);
  if (device < 0 || device >= 64 || done[device]) return SRF_OK;
  CUDA_TRY(cudaSetDevice(device));
  const void *kernels[] = {
      (const void *)k_counter_add, (const void *)k_put<8, true>, (const void *)k_put<8, false>,
      (const void *)k_put<4, true>, (const void *)k_put<4, false>, (const void *)k_put_bulk,
      (const void *)k_zero_fill, (const void *)k_flag_wait, (const void *)k_consume_sum,
      (const void *)k_gen_reference, (const void *)k_apply_xor, (const void *)k_apply_sgd,
      (const void *)k_put_batch, (const void *)k_gen_batch, (const void *)k_apply_batch,
      (const void *)k_dyn_recv, (const void *)k_ps_persistent, (const void *)k_ps_exchange<2>,
      (const void *)k_ps_exchange<3>, (const void *)k_rpc, (const void *)k_reduce_max,
      (const void *)k_matmul<float>, (const void *)k_matmul<double>,
      (const void *)k_matmul<int32_t>, (const void *)k_matmul<int64_t>,
      (const void *)k_matmul<uint8_t>, (const void *)k_put_stream,
      (const void *)k_consume_stream, (const void *)k_put_inline, (const void *)k_clear_flag,
      (const void *)k_set_u64, (const void *)k_add<float>, (const void *)k_add<double>,
      (const void *)k_add<int32_t>, (const void *)k_add<int64_t>, (const void *)k_add<uint8_t>,
      (const void *)k_sigmoid<float>, (const void *)k_sigmoid<double>,
      (const void *)k_pull_stream<true>, (const void *)k_pull_stream<false>,
      (const void *)k_post_rounds, (const void *)k_put_ind<8, false>,
      (const void *)k_put_ind<8, true>, (const void *)k_put_ind<4, false>,
      (const void *)k_put_ind<4, true>, (const void *)k_put_inline_ind, (const void *)k_gen_ind,
      (const void *)k_apply_ind<true>, (const void *)k_apply_ind<false>,
      (const void *)k_set_replay, (const void *)k_dyn_send_stream,
      (const void *)k_dyn_pull_stream, (const void *)k_dyn_consume_stream,
      (const void *)k_pull_stream_pre, (const void *)k_concat_tile,
      (const void *)k_add_bcast<float>, (const void *)k_add_bcast<double>,
      (const void *)k_add_bcast<int32_t>, (const void *)k_add_bcast<int64_t>,
      (const void *)k_add_bcast<uint8_t>};
  for (const void *k : kernels) {
    cudaFuncAttributes attr;
    cudaError_t e = cudaFuncGetAttributes(&attr, k);
    if (e != cudaSuccess) return fail(SRF_E_DEVICE, "kernel preload: %s", cudaGetErrorString(e));
  }
  done[device] = true;
  return SRF_OK;
}
