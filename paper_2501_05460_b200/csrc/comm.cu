// NCCL legs of the stage handoff, behind the C ABI (include/epd.h "stage handoff over NCCL").
//
// Reference seams (relative to /root/reference/pkg/src/disaggsim/):
//   * EP migration: _send_ready_shards / _schedule_transfer (engine.py:511-526) move each IRP
//     shard of post-projector MM tokens (tiles * tokens_per_patch * mm_bytes_per_token bytes)
//     to the prefill instance; _on_transfer_end("ep") (engine.py:424-435) starts prefill only
//     when every shard has landed.                                  -> epd_gather_tokens
//   * PD migration: _try_reserve_decode (engine.py:542-555) + _on_transfer_end("pd")
//     (engine.py:436-439) move total_tokens * kv_bytes_per_token bytes of KV into blocks the
//     decode instance reserved.                        -> epd_kv_handoff_send / _recv
//
// NCCL is resolved at run time (dlopen), not at link time: a process that already loaded
// NCCL (PyTorch's libnccl.so.2, 2.28.9 here) shares that copy -- one NCCL per process, so a
// communicator created here and torch.distributed's can coexist -- and libepd.so still loads
// on hosts without NCCL (only epd_comm_* then fail, with EPD_ERR_UNSUPPORTED).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "epd.h"

epd_status_t epd_detail_fail(epd_status_t code, const std::string& msg);  // capi.cu

namespace {

// The few NCCL entry points used here (ABI of nccl.h 2.x: ncclResult_t / ncclDataType_t are
// int enums, ncclUniqueId is 128 opaque bytes passed by value, ncclComm_t a pointer).
struct NcclUid {
  char internal[EPD_COMM_ID_BYTES];
};
typedef int (*GetUniqueId_t)(NcclUid*);
typedef int (*CommInitRank_t)(void**, int, NcclUid, int);
typedef int (*CommDestroy_t)(void*);
typedef int (*Send_t)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*Recv_t)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*Group_t)();
typedef const char* (*ErrStr_t)(int);
typedef int (*GetVersion_t)(int*);
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8

struct Nccl {
  GetUniqueId_t get_unique_id = nullptr;
  CommInitRank_t comm_init_rank = nullptr;
  CommDestroy_t comm_destroy = nullptr;
  Send_t send = nullptr;
  Recv_t recv = nullptr;
  Group_t group_start = nullptr;
  Group_t group_end = nullptr;
  ErrStr_t error_string = nullptr;
  GetVersion_t get_version = nullptr;
  bool ok = false;
  std::string why;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* env = std::getenv("EPD_NCCL_LIB");
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy the process already has
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<GetUniqueId_t>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<CommInitRank_t>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<CommDestroy_t>(dlsym(h, "ncclCommDestroy"));
    n.send = reinterpret_cast<Send_t>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<Recv_t>(dlsym(h, "ncclRecv"));
    n.group_start = reinterpret_cast<Group_t>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<Group_t>(dlsym(h, "ncclGroupEnd"));
    n.error_string = reinterpret_cast<ErrStr_t>(dlsym(h, "ncclGetErrorString"));
    n.get_version = reinterpret_cast<GetVersion_t>(dlsym(h, "ncclGetVersion"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.send && n.recv && n.group_start &&
           n.group_end && n.error_string && n.get_version;
    if (!n.ok) n.why = "libnccl.so.2 lacks a required symbol";
  });
  return n;
}

epd_status_t nccl_status(int rc, const char* what) {
  if (rc == 0) return EPD_OK;
  return epd_detail_fail(EPD_ERR_RUNTIME, std::string(what) + ": NCCL error " + std::to_string(rc) + " (" +
                                              nccl().error_string(rc) + ")");
}

epd_status_t need_nccl() {
  if (!nccl().ok) return epd_detail_fail(EPD_ERR_UNSUPPORTED, "NCCL unavailable: " + nccl().why);
  return EPD_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

struct epd_comm {
  void* comm = nullptr;
  int nranks = 0;
  int rank = 0;
  int device = 0;
};

extern "C" {

epd_status_t epd_comm_version(int32_t* version) {
  if (epd_status_t st = need_nccl()) return st;
  if (!version) return epd_detail_fail(EPD_ERR_VALUE, "version is null");
  int v = 0;
  if (epd_status_t st = nccl_status(nccl().get_version(&v), "ncclGetVersion")) return st;
  *version = v;
  return EPD_OK;
}

epd_status_t epd_comm_unique_id(uint8_t* id) {
  if (epd_status_t st = need_nccl()) return st;
  if (!id) return epd_detail_fail(EPD_ERR_VALUE, "id is null");
  NcclUid u;
  if (epd_status_t st = nccl_status(nccl().get_unique_id(&u), "ncclGetUniqueId")) return st;
  std::memcpy(id, u.internal, EPD_COMM_ID_BYTES);
  return EPD_OK;
}

epd_status_t epd_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, epd_comm_t** out) {
  if (epd_status_t st = need_nccl()) return st;
  if (!id || !out) return epd_detail_fail(EPD_ERR_VALUE, "comm init: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return epd_detail_fail(EPD_ERR_VALUE, "comm init: bad rank / size");
  if (cudaSetDevice(device) != cudaSuccess) return epd_detail_fail(EPD_ERR_CUDA, "comm init: cudaSetDevice failed");
  NcclUid u;
  std::memcpy(u.internal, id, EPD_COMM_ID_BYTES);
  auto* c = new epd_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (epd_status_t st = nccl_status(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank")) {
    delete c;
    return st;
  }
  *out = c;
  return EPD_OK;
}

void epd_comm_destroy(epd_comm_t* comm) {
  if (!comm) return;
  if (comm->comm && nccl().ok) nccl().comm_destroy(comm->comm);
  delete comm;
}

epd_status_t epd_gather_tokens(epd_comm_t* comm, const void* shard, int64_t n_tiles, int64_t tile_bytes,
                               void* packed, int32_t root, void* stream) {
  if (!comm) return epd_detail_fail(EPD_ERR_VALUE, "gather: null comm");
  if (n_tiles < 0 || tile_bytes <= 0) return epd_detail_fail(EPD_ERR_VALUE, "gather: bad sizes");
  if (root < 0 || root >= comm->nranks) return epd_detail_fail(EPD_ERR_VALUE, "gather: root out of range");
  std::vector<int64_t> first(comm->nranks), count(comm->nranks);
  if (epd_status_t st = epd_irp_ranges(n_tiles, comm->nranks, first.data(), count.data())) return st;
  const int me = comm->rank;
  if (me == root) {
    if (n_tiles && !packed) return epd_detail_fail(EPD_ERR_VALUE, "gather: null packed buffer on the root");
    // the root's own shard is already in place when shard aliases its slice of packed
    char* dst = static_cast<char*>(packed);
    if (count[me] && shard && shard != dst + first[me] * tile_bytes) {
      cudaError_t e = cudaMemcpyAsync(dst + first[me] * tile_bytes, shard, count[me] * tile_bytes,
                                      cudaMemcpyDeviceToDevice, S(stream));
      if (e != cudaSuccess) return epd_detail_fail(EPD_ERR_CUDA, "gather: local copy failed");
    }
  } else if (count[me] && !shard) {
    return epd_detail_fail(EPD_ERR_VALUE, "gather: null shard on an encode rank");
  }
  bool any = me == root ? false : count[me] > 0;
  for (int k = 0; k < comm->nranks && me == root; ++k) any |= (k != root && count[k] > 0);
  if (!any) return EPD_OK;
  Nccl& n = nccl();
  if (epd_status_t st = nccl_status(n.group_start(), "ncclGroupStart")) return st;
  int rc = 0;
  if (me == root) {
    for (int k = 0; k < comm->nranks && !rc; ++k)
      if (k != root && count[k] > 0)
        rc = n.recv(static_cast<char*>(packed) + first[k] * tile_bytes, (size_t)(count[k] * tile_bytes), kNcclUint8,
                    k, comm->comm, S(stream));
  } else {
    rc = n.send(shard, (size_t)(count[me] * tile_bytes), kNcclUint8, root, comm->comm, S(stream));
  }
  const int rc2 = n.group_end();
  if (epd_status_t st = nccl_status(rc, "gather: ncclSend/Recv")) return st;
  return nccl_status(rc2, "ncclGroupEnd");
}

epd_status_t epd_comm_send(epd_comm_t* comm, const void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || bytes < 0 || (bytes && !buf)) return epd_detail_fail(EPD_ERR_VALUE, "comm send: bad arguments");
  if (peer < 0 || peer >= comm->nranks) return epd_detail_fail(EPD_ERR_VALUE, "comm send: peer out of range");
  if (!bytes) return EPD_OK;
  return nccl_status(nccl().send(buf, (size_t)bytes, kNcclUint8, peer, comm->comm, S(stream)), "ncclSend");
}

epd_status_t epd_comm_recv(epd_comm_t* comm, void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || bytes < 0 || (bytes && !buf)) return epd_detail_fail(EPD_ERR_VALUE, "comm recv: bad arguments");
  if (peer < 0 || peer >= comm->nranks) return epd_detail_fail(EPD_ERR_VALUE, "comm recv: peer out of range");
  if (!bytes) return EPD_OK;
  return nccl_status(nccl().recv(buf, (size_t)bytes, kNcclUint8, peer, comm->comm, S(stream)), "ncclRecv");
}

epd_status_t epd_comm_group_start(void) {
  if (epd_status_t st = need_nccl()) return st;
  return nccl_status(nccl().group_start(), "ncclGroupStart");
}

epd_status_t epd_comm_group_end(void) {
  if (epd_status_t st = need_nccl()) return st;
  return nccl_status(nccl().group_end(), "ncclGroupEnd");
}

epd_status_t epd_kv_handoff_send(epd_comm_t* comm, const void* cache, int32_t segments, int64_t segment_stride,
                                 int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* staging,
                                 int32_t peer, void* stream) {
  if (!comm) return epd_detail_fail(EPD_ERR_VALUE, "kv send: null comm");
  if (peer < 0 || peer >= comm->nranks || peer == comm->rank)
    return epd_detail_fail(EPD_ERR_VALUE, "kv send: peer must be another rank");
  if (nblocks == 0) return EPD_OK;
  if (!staging) return epd_detail_fail(EPD_ERR_VALUE, "kv send: null staging buffer");
  if (epd_status_t st = epd_kv_pack(cache, segments, segment_stride, block_bytes, block_ids, nblocks, staging, stream))
    return st;
  const size_t bytes = (size_t)nblocks * segments * block_bytes;
  return nccl_status(nccl().send(staging, bytes, kNcclUint8, peer, comm->comm, S(stream)), "kv send: ncclSend");
}

epd_status_t epd_kv_handoff_recv(epd_comm_t* comm, void* cache, int32_t segments, int64_t segment_stride,
                                 int64_t block_bytes, const int32_t* block_ids, int32_t nblocks, void* staging,
                                 int32_t peer, void* stream) {
  if (!comm) return epd_detail_fail(EPD_ERR_VALUE, "kv recv: null comm");
  if (peer < 0 || peer >= comm->nranks || peer == comm->rank)
    return epd_detail_fail(EPD_ERR_VALUE, "kv recv: peer must be another rank");
  if (nblocks == 0) return EPD_OK;
  if (!staging) return epd_detail_fail(EPD_ERR_VALUE, "kv recv: null staging buffer");
  if (segments < 1 || block_bytes <= 0 || nblocks < 0) return epd_detail_fail(EPD_ERR_VALUE, "kv recv: bad geometry");
  const size_t bytes = (size_t)nblocks * segments * block_bytes;
  if (epd_status_t st =
          nccl_status(nccl().recv(staging, bytes, kNcclUint8, peer, comm->comm, S(stream)), "kv recv: ncclRecv"))
    return st;
  return epd_kv_unpack(staging, segments, segment_stride, block_bytes, block_ids, nblocks, cache, stream);
}

}  // extern "C"
