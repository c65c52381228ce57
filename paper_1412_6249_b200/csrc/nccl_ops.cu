// NCCL over NVLink/NVSwitch for the lowered parameter exchange (exchange.py):
// per bucket a reduce-scatter of the gradient sum, a fused mean+SGD on the
// owned shard (bf_sgd_mean_update) and an all-gather of the updated shard.
// Replaces the reference's up-copy -> aggregate -> sgd -> down-copy server
// subgraph (builders.py:581-611) for one process per GPU.
#include <nccl.h>

#include "common.cuh"

#define BF_NCCL(call, what)                                          \
  do {                                                               \
    ncclResult_t _r = (call);                                        \
    if (_r != ncclSuccess) {                                         \
      ::bf::set_error("%s: %s", what, ncclGetErrorString(_r));       \
      return 3;                                                      \
    }                                                                \
  } while (0)

extern "C" {

int bf_nccl_unique_id(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  BF_NCCL(ncclGetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, 128);
  return 0;
}

int bf_nccl_init(void** comm, int nranks, int rank, const unsigned char id[128]) {
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t c = nullptr;
  BF_NCCL(ncclCommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  *comm = c;
  return 0;
}

int bf_nccl_destroy(void* comm) {
  if (comm) BF_NCCL(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return 0;
}

int bf_nccl_reduce_scatter(void* comm, const float* send, float* recv, int64_t recv_count,
                           bf_stream_t s) {
  BF_NCCL(ncclReduceScatter(send, recv, (size_t)recv_count, ncclFloat32, ncclSum,
                            reinterpret_cast<ncclComm_t>(comm), bf::as_stream(s)),
          "ncclReduceScatter");
  return 0;
}

int bf_nccl_all_gather(void* comm, const float* send, float* recv, int64_t send_count,
                       bf_stream_t s) {
  BF_NCCL(ncclAllGather(send, recv, (size_t)send_count, ncclFloat32,
                        reinterpret_cast<ncclComm_t>(comm), bf::as_stream(s)),
          "ncclAllGather");
  return 0;
}

int bf_nccl_all_reduce(void* comm, const float* send, float* recv, int64_t count,
                       bf_stream_t s) {
  BF_NCCL(ncclAllReduce(send, recv, (size_t)count, ncclFloat32, ncclSum,
                        reinterpret_cast<ncclComm_t>(comm), bf::as_stream(s)),
          "ncclAllReduce");
  return 0;
}

}  // extern "C"
