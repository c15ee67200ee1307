// gcdf_comm.h -- internal interface of the exchange backends (gcdf_comm.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "gcdf.h"

namespace gcdf {

constexpr int kCommNone = 0, kCommNccl = 1, kCommHost = 2;
constexpr int kCommErrNccl = 1, kCommErrCuda = 2;

struct Comm {
  int kind = kCommNone;
  int rank = 0, world = 1;
  void *nccl = nullptr;            // ncclComm_t
  int nccl_version = 0;
  gcdf_host_allgather_fn fn = nullptr;  // host backend (tests only)
  void *user = nullptr;
  void *h_send = nullptr, *h_recv = nullptr;
  int64_t h_bytes = 0;
};

int comm_unique_id(unsigned char out[128], std::string *err);
int comm_init_nccl(Comm &c, const unsigned char id[128], int rank, int world, std::string *err);
int comm_init_host(Comm &c, int rank, int world, gcdf_host_allgather_fn fn, void *user);
void comm_destroy(Comm &c);
// One all-gather group of n pieces: rank r's bytes[i] bytes of send[i] land at
// recv[i] + r * bytes[i] on every rank; enqueued on s (NCCL) or synchronous (host backend).
int comm_allgather(Comm &c, int n, const void *const *send, void *const *recv, const int64_t *bytes, cudaStream_t s,
                   std::string *err);
// rank 0's `bytes` bytes of buf (device) to every rank's buf, in place; enqueued on s (NCCL,
// ncclBroadcast) or synchronous (host backend: an all-gather of which rank 0's piece is kept)
int comm_broadcast(Comm &c, void *buf, int64_t bytes, cudaStream_t s, std::string *err);

}  // namespace gcdf
