// gcdf_comm.cpp -- the exchange step of the sharded detect:
// one all-gather group over the ranks' per-waypoint headers and compacted records, on the
// detect call's stream.
//
// Backends:
//   * NCCL (product): libnccl.so.2 is opened at gcdf_dist_init time with dlopen (the copy
//     torch already loaded, same soname, or the system one), so libgcdf.so carries no
//     link-time NCCL dependency and shares the process's NCCL.  Both all-gathers are issued
//     in one ncclGroupStart/End on the caller's stream: no host synchronization, graph
//     capturable.  Over NVLink 5 / NVSwitch NCCL picks its own algorithm (NVLS when the
//     switch can multicast).
//   * host callback (TESTS ONLY): the caller supplies a blocking host all-gather (the tests
//     wrap torch.distributed gloo); the library synchronizes the stream, stages through
//     pinned host memory and copies the gathered bytes back.  It lets two processes on ONE
//     GPU run the whole multi-rank detect (local detect -> exchange -> merge kernel) with
//     no kernel of one rank waiting on another rank's kernel.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "gcdf_comm.h"

namespace gcdf {
namespace {

struct NcclApi {
  void *handle = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
};

const NcclApi *nccl_api(std::string *err) {
  static NcclApi api;
  static bool tried = false;
  if (tried) {
    if (!api.handle && err) *err = "libnccl.so.2 could not be opened";
    return api.handle ? &api : nullptr;
  }
  tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    if (err) *err = std::string("dlopen libnccl.so.2: ") + dlerror();
    return nullptr;
  }
  auto sym = [&](const char *name) { return dlsym(h, name); };
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
  api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
  api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
  if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_gather || !api.broadcast ||
      !api.group_start ||
      !api.group_end || !api.error_string) {
    if (err) *err = "libnccl.so.2 lacks an expected symbol";
    return nullptr;
  }
  api.handle = h;
  return &api;
}

int nccl_fail(const NcclApi *api, ncclResult_t r, const char *what, std::string *err) {
  if (err) *err = std::string(what) + ": " + (api ? api->error_string(r) : "nccl");
  return kCommErrNccl;
}

}  // namespace

int comm_unique_id(unsigned char out[128], std::string *err) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  const NcclApi *api = nccl_api(err);
  if (!api) return kCommErrNccl;
  ncclUniqueId id;
  const ncclResult_t r = api->get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId", err);
  std::memcpy(out, &id, 128);
  return 0;
}

int comm_init_nccl(Comm &c, const unsigned char id[128], int rank, int world, std::string *err) {
  const NcclApi *api = nccl_api(err);
  if (!api) return kCommErrNccl;
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api->comm_init_rank(&comm, world, uid, rank);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommInitRank", err);
  c.kind = kCommNccl;
  c.rank = rank;
  c.world = world;
  c.nccl = comm;
  if (api->get_version) api->get_version(&c.nccl_version);
  return 0;
}

int comm_init_host(Comm &c, int rank, int world, gcdf_host_allgather_fn fn, void *user) {
  c.kind = kCommHost;
  c.rank = rank;
  c.world = world;
  c.fn = fn;
  c.user = user;
  return 0;
}

void comm_destroy(Comm &c) {
  if (c.kind == kCommNccl && c.nccl) {
    const NcclApi *api = nccl_api(nullptr);
    if (api) api->comm_destroy(static_cast<ncclComm_t>(c.nccl));
  }
  if (c.h_send) cudaFreeHost(c.h_send);
  if (c.h_recv) cudaFreeHost(c.h_recv);
  c = Comm{};
}

int comm_allgather(Comm &c, int n, const void *const *send, void *const *recv, const int64_t *bytes, cudaStream_t s,
                   std::string *err) {
  if (c.kind == kCommNccl) {
    const NcclApi *api = nccl_api(err);
    if (!api) return kCommErrNccl;
    ncclComm_t comm = static_cast<ncclComm_t>(c.nccl);
    ncclResult_t r = api->group_start();
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGroupStart", err);
    for (int i = 0; i < n; ++i) {
      r = api->all_gather(send[i], recv[i], (size_t)bytes[i], ncclUint8, comm, s);
      if (r != ncclSuccess) {
        api->group_end();
        return nccl_fail(api, r, "ncclAllGather", err);
      }
    }
    r = api->group_end();
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGroupEnd", err);
    return 0;
  }
  if (c.kind != kCommHost) {
    if (err) *err = "no communicator";
    return kCommErrNccl;
  }
  // test backend: pack the pieces, one blocking host all-gather, unpack per rank
  int64_t per = 0;
  for (int i = 0; i < n; ++i) per += bytes[i];
  const int64_t need = per * c.world;
  if (need > c.h_bytes) {
    if (c.h_send) cudaFreeHost(c.h_send);
    if (c.h_recv) cudaFreeHost(c.h_recv);
    c.h_send = c.h_recv = nullptr;
    c.h_bytes = 0;
    if (cudaHostAlloc(&c.h_send, per > 0 ? per : 1, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&c.h_recv, need > 0 ? need : 1, cudaHostAllocDefault) != cudaSuccess) {
      if (err) *err = "host backend: pinned staging";
      return kCommErrCuda;
    }
    c.h_bytes = need;
  }
  char *hs = static_cast<char *>(c.h_send), *hr = static_cast<char *>(c.h_recv);
  int64_t o = 0;
  for (int i = 0; i < n; ++i) {
    if (bytes[i] && cudaMemcpyAsync(hs + o, send[i], bytes[i], cudaMemcpyDeviceToHost, s) != cudaSuccess) {
      if (err) *err = "host backend: D2H";
      return kCommErrCuda;
    }
    o += bytes[i];
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    if (err) *err = "host backend: sync";
    return kCommErrCuda;
  }
  if (c.fn(hs, hr, per, c.user) != 0) {
    if (err) *err = "host backend: the all-gather callback failed";
    return kCommErrNccl;
  }
  for (int r = 0; r < c.world; ++r) {
    o = 0;
    for (int i = 0; i < n; ++i) {
      if (bytes[i] && cudaMemcpyAsync(static_cast<char *>(recv[i]) + (int64_t)r * bytes[i], hr + (int64_t)r * per + o,
                                      bytes[i], cudaMemcpyHostToDevice, s) != cudaSuccess) {
        if (err) *err = "host backend: H2D";
        return kCommErrCuda;
      }
      o += bytes[i];
    }
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) {  // the pinned staging is reused by the next call
    if (err) *err = "host backend: sync";
    return kCommErrCuda;
  }
  return 0;
}

int comm_broadcast(Comm &c, void *buf, int64_t bytes, cudaStream_t s, std::string *err) {
  if (bytes <= 0) return 0;
  if (c.kind == kCommNccl) {
    const NcclApi *api = nccl_api(err);
    if (!api) return kCommErrNccl;
    const ncclResult_t r = api->broadcast(buf, buf, (size_t)bytes, ncclUint8, 0, static_cast<ncclComm_t>(c.nccl), s);
    return r == ncclSuccess ? 0 : nccl_fail(api, r, "ncclBroadcast", err);
  }
  if (c.kind != kCommHost) {
    if (err) *err = "no communicator";
    return kCommErrNccl;
  }
  // test backend: every rank's bytes are gathered, rank 0's piece is copied back into buf
  void *tmp = nullptr;
  if (cudaMallocAsync(&tmp, (size_t)bytes * c.world, s) != cudaSuccess) {
    if (err) *err = "host backend: broadcast staging";
    return kCommErrCuda;
  }
  const void *send[1] = {buf};
  void *recv[1] = {tmp};
  const int64_t b[1] = {bytes};
  int r = comm_allgather(c, 1, send, recv, b, s, err);
  if (r == 0 && cudaMemcpyAsync(buf, tmp, (size_t)bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
    if (err) *err = "host backend: broadcast copy";
    r = kCommErrCuda;
  }
  cudaFreeAsync(tmp, s);
  return r;
}

}  // namespace gcdf
