// extern "C" surface declared in include/epd.h: argument checking, error
// strings, and thin forwarding to the kernels / encoder executor.
#include <cstring>
#include <string>

#include "epd.h"
#include "encoder.h"
#include "kernels.h"
#include "mmcache.h"

namespace {

thread_local std::string g_err;

epd_status_t fail(epd_status_t code, const std::string& msg) {
  g_err = msg;
  return code;
}

epd_status_t cuda_status(int rc, const char* what) {
  if (rc == 0) return EPD_OK;
  std::string m = std::string(what) + ": ";
  if (rc < 1000)
    m += cudaGetErrorString((cudaError_t)rc);
  else
    m += "invalid shape/alignment (code " + std::to_string(rc) + ")";
  return fail(rc < 1000 ? EPD_ERR_CUDA : EPD_ERR_VALUE, m);
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

// shared with the other translation units of the ABI (comm.cu)
epd_status_t epd_detail_fail(epd_status_t code, const std::string& msg) { return fail(code, msg); }

namespace {

// Two-level record copy used by the KV handoff:
//   pack:   out[i][s] = cache[s][ids[i]]
//   unpack: cache[s][ids[i]] = in[i][s]
__global__ void kv_copy_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int segments,
                               long long seg_stride, long long block_bytes, const int32_t* __restrict__ ids,
                               int pack) {
  const int i = blockIdx.z;
  const int s = blockIdx.y;
  const long long cache_off = (long long)s * seg_stride + (long long)ids[i] * block_bytes;
  const long long packed_off = ((long long)i * segments + s) * block_bytes;
  const uint4* a = reinterpret_cast<const uint4*>(src + (pack ? cache_off : packed_off));
  uint4* b = reinterpret_cast<uint4*>(dst + (pack ? packed_off : cache_off));
  const long long vecs = block_bytes / 16;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < vecs;
       v += (long long)gridDim.x * blockDim.x)
    b[v] = a[v];
}

// Block-to-block KV move (handoff without a staging buffer): for block pair i and segment
// s, dst[s][dst_ids[i]] = src[s][src_ids[i]]. dst may be a peer mapping of another GPU's
// pool, so the copy is the NVLink transfer itself.
__global__ void kv_move_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, long long src_stride,
                               long long dst_stride, long long block_bytes, const int32_t* __restrict__ src_ids,
                               const int32_t* __restrict__ dst_ids) {
  const int i = blockIdx.z;
  const int s = blockIdx.y;
  const uint4* a = reinterpret_cast<const uint4*>(src + (long long)s * src_stride + (long long)src_ids[i] * block_bytes);
  uint4* b = reinterpret_cast<uint4*>(dst + (long long)s * dst_stride + (long long)dst_ids[i] * block_bytes);
  const long long vecs = block_bytes / 16;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < vecs;
       v += (long long)gridDim.x * blockDim.x)
    b[v] = a[v];
  __threadfence_system();  // dst may be a peer GPU's pool: the signal that follows must not overtake
}

__global__ void scatter_records_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ index,
                                       size_t vecs, uint4* __restrict__ dst) {
  const int rec = blockIdx.y;
  const uint4* s = src + (size_t)rec * vecs;
  uint4* d = dst + (size_t)index[rec] * vecs;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < vecs;
       i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
  __threadfence_system();  // dst may be the prefill GPU's MM pool mapped over IPC (runtime.py)
}

__global__ void timestamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

epd_status_t kv_copy(const void* src, void* dst, int32_t segments, int64_t seg_stride, int64_t block_bytes,
                     const int32_t* ids, int32_t nblocks, int pack, void* stream) {
  if (segments < 1 || block_bytes <= 0 || nblocks < 0 || seg_stride < block_bytes)
    return fail(EPD_ERR_VALUE, "kv handoff: bad geometry");
  if (block_bytes % 16 || seg_stride % 16 ||
      ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15))
    return fail(EPD_ERR_VALUE, "kv handoff: blocks must be 16-byte aligned");
  if (nblocks == 0) return EPD_OK;
  if (segments > 65535 || nblocks > 65535) return fail(EPD_ERR_VALUE, "kv handoff: too many blocks");
  long long vecs = block_bytes / 16;
  int bx = (int)((vecs + 255) / 256);
  if (bx > 8) bx = 8;
  dim3 grid(bx, segments, nblocks);
  kv_copy_kernel<<<grid, 256, 0, S(stream)>>>(reinterpret_cast<const uint8_t*>(src),
                                              reinterpret_cast<uint8_t*>(dst), segments, seg_stride,
                                              block_bytes, ids, pack);
  return cuda_status((int)cudaGetLastError(), "kv handoff");
}

}  // namespace

struct epd_encoder {
  epd::Encoder impl;
  epd_encoder(const epd_encoder_desc_t& d, int dev) : impl(d, dev) {}
};

struct epd_mmcache {
  epd::DeviceTable t;
  epd::DevicePlanner p;
  void* mem = nullptr;
  void* pmem = nullptr;
  int device = 0;
};

extern "C" {

int32_t epd_abi_version(void) { return EPD_ABI_VERSION; }
const char* epd_last_error(void) { return g_err.c_str(); }

epd_status_t epd_irp_shard(int64_t patches, int32_t width, int64_t* counts) {
  // engine.py:55-62
  if (width < 1) return fail(EPD_ERR_VALUE, "shard width must be >= 1");
  if (patches < 0) return fail(EPD_ERR_VALUE, "patch count must be non-negative");
  if (!counts) return fail(EPD_ERR_VALUE, "counts is null");
  const int64_t base = patches / width, rem = patches % width;
  for (int32_t k = 0; k < width; ++k) counts[k] = base + (k < rem ? 1 : 0);
  return EPD_OK;
}

epd_status_t epd_irp_ranges(int64_t patches, int32_t width, int64_t* first, int64_t* counts) {
  epd_status_t st = epd_irp_shard(patches, width, counts);
  if (st != EPD_OK) return st;
  if (!first) return fail(EPD_ERR_VALUE, "first is null");
  int64_t acc = 0;
  for (int32_t k = 0; k < width; ++k) {
    first[k] = acc;
    acc += counts[k];
  }
  return EPD_OK;
}

// ------------------------------------------------------------------ encoder

epd_status_t epd_encoder_create(const epd_encoder_desc_t* desc, int32_t device, epd_encoder_t** out) {
  if (!desc || !out) return fail(EPD_ERR_VALUE, "null argument");
  *out = nullptr;
  // Schema construction is host-only; device memory is touched from finalize on.
  auto* enc = new epd_encoder(*desc, device);
  std::string msg = enc->impl.validate_and_build_schema();
  if (!msg.empty()) {
    delete enc;
    return fail(EPD_ERR_UNSUPPORTED, msg);
  }
  *out = enc;
  return EPD_OK;
}

void epd_encoder_destroy(epd_encoder_t* enc) { delete enc; }

int32_t epd_encoder_num_weights(const epd_encoder_t* enc) {
  return enc ? (int32_t)enc->impl.slots.size() : 0;
}

epd_status_t epd_encoder_weight_info(const epd_encoder_t* enc, int32_t index, const char** name,
                                     int32_t* ndim, int64_t* shape) {
  if (!enc || index < 0 || index >= (int32_t)enc->impl.slots.size())
    return fail(EPD_ERR_VALUE, "weight index out of range");
  const auto& s = enc->impl.slots[index];
  if (name) *name = s.name.c_str();
  if (ndim) *ndim = (int32_t)s.shape.size();
  if (shape)
    for (size_t i = 0; i < 4; ++i) shape[i] = i < s.shape.size() ? s.shape[i] : 1;
  return EPD_OK;
}

epd_status_t epd_encoder_set_weight(epd_encoder_t* enc, int32_t index, const float* host_values,
                                    int64_t numel) {
  if (!enc || index < 0 || index >= (int32_t)enc->impl.slots.size())
    return fail(EPD_ERR_VALUE, "weight index out of range");
  if (enc->impl.finalized) return fail(EPD_ERR_RUNTIME, "encoder already finalized");
  if (!host_values || numel != enc->impl.numel(index))
    return fail(EPD_ERR_VALUE, "weight " + enc->impl.slots[index].name + ": numel mismatch");
  auto& s = enc->impl.slots[index];
  s.host.assign(host_values, host_values + numel);
  s.set = true;
  return EPD_OK;
}

epd_status_t epd_encoder_finalize(epd_encoder_t* enc, void* stream) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  if (enc->impl.finalized) return fail(EPD_ERR_RUNTIME, "encoder already finalized");
  cudaError_t e = cudaSetDevice(enc->impl.dev);
  if (e != cudaSuccess) return fail(EPD_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  std::string err;
  int rc = enc->impl.finalize(S(stream), err);
  if (rc) return fail((epd_status_t)rc, err);
  return EPD_OK;
}

epd_status_t epd_encode_tiles(epd_encoder_t* enc, const uint8_t* tiles, int32_t n, void* out, void* stream) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  if (n > 0 && (!tiles || !out)) return fail(EPD_ERR_VALUE, "null tile or output buffer");
  std::string err;
  int rc = enc->impl.encode(tiles, n, reinterpret_cast<epd::bf16*>(out), S(stream), err);
  if (rc) return fail((epd_status_t)rc, err);
  return EPD_OK;
}

epd_status_t epd_encoder_enable_fp32_check(epd_encoder_t* enc) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  if (enc->impl.finalized) return fail(EPD_ERR_RUNTIME, "fp32 check mode must be enabled before finalize");
  enc->impl.check_f32 = true;
  return EPD_OK;
}

epd_status_t epd_encode_tiles_f32(epd_encoder_t* enc, const uint8_t* tiles, int32_t n, float* out, void* stream) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  if (n > 0 && (!tiles || !out)) return fail(EPD_ERR_VALUE, "null tile or output buffer");
  std::string err;
  int rc = enc->impl.encode_f32(tiles, n, out, S(stream), err);
  if (rc) return fail((epd_status_t)rc, err);
  return EPD_OK;
}

double epd_encoder_flops_per_tile(const epd_encoder_t* enc) { return enc ? enc->impl.flops_per_tile() : 0.0; }
int32_t epd_encoder_launches(const epd_encoder_t* enc, int32_t n) { return enc ? enc->impl.launches(n) : 0; }

epd_status_t epd_encoder_set_graphs(epd_encoder_t* enc, int32_t on) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  enc->impl.use_graphs = on != 0;
  return EPD_OK;
}

epd_status_t epd_encoder_profile(epd_encoder_t* enc, int32_t on) {
  if (!enc) return fail(EPD_ERR_VALUE, "null encoder");
  enc->impl.prof_on = on != 0;
  return EPD_OK;
}

epd_status_t epd_encoder_profile_read(epd_encoder_t* enc, double* ms, double* flops, double* bytes,
                                      int64_t* launches, int32_t nclass) {
  if (!enc || !ms || !flops || !bytes || !launches || nclass < 1)
    return fail(EPD_ERR_VALUE, "profile_read: bad arguments");
  return cuda_status(enc->impl.prof_read(ms, flops, bytes, launches, nclass), "profile_read");
}

int32_t epd_encoder_profile_launches(const epd_encoder_t* enc, int32_t* cls, float* ms, double* flops, int32_t cap) {
  if (!enc) return -1;
  const auto& v = enc->impl.prof_last;
  const int32_t n = (int32_t)v.size();
  for (int32_t i = 0; i < n && i < cap; ++i) {
    if (cls) cls[i] = v[i].cls;
    if (ms) ms[i] = v[i].ms;
    if (flops) flops[i] = v[i].flops;
  }
  return n;
}

// ------------------------------------------------------------------ cache

epd_status_t epd_hash_records(const void* data, int32_t n, int64_t rec_bytes, int64_t rec_stride,
                              uint64_t* keys, void* scratch, void* stream) {
  return epd_hash_records_keyed(data, n, rec_bytes, rec_stride, 0, 0, keys, scratch, stream);
}

epd_status_t epd_hash_records_keyed(const void* data, int32_t n, int64_t rec_bytes, int64_t rec_stride,
                                    uint64_t secret0, uint64_t secret1, uint64_t* keys, void* scratch,
                                    void* stream) {
  if (n < 0 || rec_bytes < 0 || rec_stride < rec_bytes) return fail(EPD_ERR_VALUE, "hash: bad geometry");
  if (rec_bytes % 8) return fail(EPD_ERR_VALUE, "hash: record length must be a multiple of 8 bytes");
  if (n == 0) return EPD_OK;
  if (!data || !keys || !scratch) return fail(EPD_ERR_VALUE, "hash: null buffer");
  if (n > 65535) return fail(EPD_ERR_VALUE, "hash: at most 65535 records per call");
  int rc = epd::hash_records(data, n, (size_t)rec_bytes, (size_t)rec_stride,
                             reinterpret_cast<unsigned long long*>(scratch),
                             reinterpret_cast<unsigned long long*>(keys), S(stream), secret0, secret1);
  return cuda_status(rc, "hash_records");
}

epd_status_t epd_mmcache_create(int64_t capacity, int32_t device, epd_mmcache_t** out) {
  if (!out || capacity < 1) return fail(EPD_ERR_VALUE, "cache capacity must be >= 1");
  if (capacity > epd::planner_max_capacity())
    return fail(EPD_ERR_UNSUPPORTED, "cache capacity above " + std::to_string(epd::planner_max_capacity()));
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return fail(EPD_ERR_CUDA, "cudaSetDevice failed");
  unsigned long long slots = 16;
  while (slots < 2ull * (unsigned long long)capacity) slots <<= 1;
  auto* c = new epd_mmcache();
  c->device = device;
  const size_t bytes = slots * 16 + slots * 4 + 256;
  cudaError_t e = cudaMalloc(&c->mem, bytes);
  const size_t C = (size_t)capacity;
  const size_t pbytes = C * 16 + 3 * C * 4 + 64;
  if (e == cudaSuccess) e = cudaMalloc(&c->pmem, pbytes);
  if (e != cudaSuccess) {
    if (c->mem) cudaFree(c->mem);
    delete c;
    return fail(EPD_ERR_CUDA, std::string("cudaMalloc(cache table): ") + cudaGetErrorString(e));
  }
  cudaMemset(c->mem, 0, bytes);
  c->t.capacity = slots;
  c->t.keys = reinterpret_cast<unsigned long long*>(c->mem);
  c->t.vals = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(c->mem) + slots * 16);
  c->t.status = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(c->mem) + slots * 20);
  uint8_t* pm = reinterpret_cast<uint8_t*>(c->pmem);
  c->p.capacity = (int32_t)capacity;
  c->p.entry_key = reinterpret_cast<unsigned long long*>(pm);
  c->p.prev = reinterpret_cast<int32_t*>(pm + C * 16);
  c->p.next = c->p.prev + C;
  c->p.free_stack = c->p.next + C;
  c->p.state = c->p.free_stack + C;
  int rc = epd::planner_reset(c->t, c->p, 0);
  if (!rc) rc = (int)cudaDeviceSynchronize();
  if (rc) {
    cudaFree(c->mem);
    cudaFree(c->pmem);
    delete c;
    return cuda_status(rc, "mmcache_create");
  }
  *out = c;
  return EPD_OK;
}

void epd_mmcache_destroy(epd_mmcache_t* cache) {
  if (!cache) return;
  if (cache->mem) cudaFree(cache->mem);
  if (cache->pmem) cudaFree(cache->pmem);
  delete cache;
}

epd_status_t epd_mmcache_plan(epd_mmcache_t* cache, const uint64_t* keys, int32_t n, int32_t* entries,
                              int32_t* kinds, int32_t* miss_tiles, int32_t* miss_entries, uint64_t* victim_keys,
                              int32_t* counts, void* stream) {
  if (!cache || n < 0 || (n && (!keys || !entries || !kinds || !miss_tiles || !miss_entries || !victim_keys)) ||
      !counts)
    return fail(EPD_ERR_VALUE, "mmcache_plan: bad arguments");
  if ((size_t)n > epd::planner_max_tiles())
    return fail(EPD_ERR_UNSUPPORTED, "mmcache_plan: more than " + std::to_string(epd::planner_max_tiles()) +
                                         " tiles in one request");
  epd::PlanOut o{entries, kinds, miss_tiles, miss_entries, reinterpret_cast<unsigned long long*>(victim_keys),
                 counts};
  int rc = epd::planner_plan(cache->t, cache->p, reinterpret_cast<const unsigned long long*>(keys), n, o,
                             S(stream));
  return cuda_status(rc, "mmcache_plan");
}

epd_status_t epd_mmcache_lookup(epd_mmcache_t* cache, const uint64_t* keys, int32_t n, int32_t* entry,
                                int32_t* dup, void* stream) {
  if (!cache || n < 0) return fail(EPD_ERR_VALUE, "lookup: bad arguments");
  if (n == 0) return EPD_OK;
  auto k = reinterpret_cast<const unsigned long long*>(keys);
  int rc = epd::table_lookup(cache->t, k, n, entry, S(stream));
  if (!rc && dup) rc = epd::table_dedup(k, entry, n, dup, S(stream));
  return cuda_status(rc, "mmcache_lookup");
}

epd_status_t epd_mmcache_insert(epd_mmcache_t* cache, const uint64_t* keys, const int32_t* entries, int32_t n,
                                void* stream) {
  if (!cache || n < 0) return fail(EPD_ERR_VALUE, "insert: bad arguments");
  if (n == 0) return EPD_OK;
  int rc = epd::table_insert(cache->t, reinterpret_cast<const unsigned long long*>(keys), entries, n, S(stream));
  return cuda_status(rc, "mmcache_insert");
}

epd_status_t epd_mmcache_erase(epd_mmcache_t* cache, const uint64_t* keys, int32_t n, void* stream) {
  if (!cache || n < 0) return fail(EPD_ERR_VALUE, "erase: bad arguments");
  if (n == 0) return EPD_OK;
  int rc = epd::table_erase(cache->t, reinterpret_cast<const unsigned long long*>(keys), n, S(stream));
  return cuda_status(rc, "mmcache_erase");
}

epd_status_t epd_mmcache_clear(epd_mmcache_t* cache, void* stream) {
  if (!cache) return fail(EPD_ERR_VALUE, "clear: null cache");
  return cuda_status(epd::planner_reset(cache->t, cache->p, S(stream)), "mmcache_clear");
}

epd_status_t epd_mmcache_check(epd_mmcache_t* cache, void* stream) {
  if (!cache) return fail(EPD_ERR_VALUE, "check: null cache");
  int32_t st = 0;
  cudaError_t e = cudaMemcpyAsync(&st, cache->t.status, 4, cudaMemcpyDeviceToHost, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) return cuda_status((int)e, "mmcache_check");
  if (st) return fail(EPD_ERR_CAPACITY, "multimodal cache table is full");
  return EPD_OK;
}

// ------------------------------------------------------------------ packing / handoff

epd_status_t epd_gather_records(const void* src, const int32_t* index, int32_t n, int64_t rec_bytes, void* dst,
                                void* stream) {
  if (n < 0 || rec_bytes <= 0) return fail(EPD_ERR_VALUE, "gather: bad geometry");
  if (n > 65535) return fail(EPD_ERR_VALUE, "gather: at most 65535 records per call");
  return cuda_status(epd::gather_records(src, index, n, (size_t)rec_bytes, dst, S(stream)), "gather_records");
}

epd_status_t epd_scatter_records(const void* src, const int32_t* index, int32_t n, int64_t rec_bytes, void* dst,
                                 void* stream) {
  if (n < 0 || rec_bytes <= 0) return fail(EPD_ERR_VALUE, "scatter: bad geometry");
  if (n == 0) return EPD_OK;
  if (n > 65535) return fail(EPD_ERR_VALUE, "scatter: at most 65535 records per call");
  if (rec_bytes % 16 || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15))
    return fail(EPD_ERR_VALUE, "scatter: records must be 16-byte aligned");
  const size_t vecs = (size_t)rec_bytes / 16;
  int bx = (int)((vecs + 255) / 256);
  if (bx > 64) bx = 64;
  scatter_records_kernel<<<dim3(bx, n), 256, 0, S(stream)>>>(reinterpret_cast<const uint4*>(src), index, vecs,
                                                               reinterpret_cast<uint4*>(dst));
  return cuda_status((int)cudaGetLastError(), "scatter_records");
}

epd_status_t epd_peer_alloc(int64_t bytes, void** ptr) {
  if (bytes <= 0 || !ptr) return fail(EPD_ERR_VALUE, "peer_alloc: bytes must be > 0");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return cuda_status((int)e, "peer_alloc");
  }
  *ptr = p;
  return EPD_OK;
}

epd_status_t epd_peer_free(void* ptr) { return cuda_status((int)cudaFree(ptr), "peer_free"); }

epd_status_t epd_peer_export(void* ptr, void* handle) {
  if (!ptr || !handle) return fail(EPD_ERR_VALUE, "peer_export: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return cuda_status((int)e, "peer_export (cudaIpcGetMemHandle)");
  std::memcpy(handle, &h, sizeof(h));
  return EPD_OK;
}

epd_status_t epd_peer_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return fail(EPD_ERR_VALUE, "peer_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return cuda_status((int)e, "peer_open (cudaIpcOpenMemHandle)");
}

epd_status_t epd_peer_close(void* ptr) { return cuda_status((int)cudaIpcCloseMemHandle(ptr), "peer_close"); }

epd_status_t epd_peer_put(const void* src, void* dst, int64_t bytes, uint32_t* flag, uint32_t value,
                          void* stream) {
  if (bytes < 0) return fail(EPD_ERR_VALUE, "peer_put: negative size");
  return cuda_status(epd::peer_put(src, dst, (size_t)bytes, flag, value, S(stream)), "peer_put");
}

epd_status_t epd_peer_signal(uint32_t* flag, uint32_t value, void* stream) {
  if (!flag) return fail(EPD_ERR_VALUE, "peer_signal: null flag");
  return cuda_status(epd::peer_signal(flag, value, S(stream)), "peer_signal");
}

epd_status_t epd_stream_wait_geq(const uint32_t* flag, uint32_t value, void* stream) {
  if (!flag) return fail(EPD_ERR_VALUE, "stream_wait_geq: null flag");
  return cuda_status(epd::stream_wait_geq(flag, value, S(stream)), "stream_wait_geq (cuStreamWaitValue32)");
}

epd_status_t epd_timestamp(uint64_t* slot, void* stream) {
  if (!slot) return fail(EPD_ERR_VALUE, "timestamp: null slot");
  timestamp_kernel<<<1, 1, 0, S(stream)>>>(reinterpret_cast<unsigned long long*>(slot));
  return cuda_status((int)cudaGetLastError(), "timestamp");
}

epd_status_t epd_kv_move(const void* src_cache, int64_t src_segment_stride, void* dst_cache,
                         int64_t dst_segment_stride, int32_t segments, int64_t block_bytes, const int32_t* src_ids,
                         const int32_t* dst_ids, int32_t nblocks, void* stream) {
  if (segments < 1 || block_bytes <= 0 || nblocks < 0 || src_segment_stride < block_bytes ||
      dst_segment_stride < block_bytes)
    return fail(EPD_ERR_VALUE, "kv move: bad geometry");
  if (block_bytes % 16 || src_segment_stride % 16 || dst_segment_stride % 16 ||
      ((reinterpret_cast<uintptr_t>(src_cache) | reinterpret_cast<uintptr_t>(dst_cache)) & 15))
    return fail(EPD_ERR_VALUE, "kv move: blocks must be 16-byte aligned");
  if (nblocks == 0) return EPD_OK;
  if (segments > 65535 || nblocks > 65535) return fail(EPD_ERR_VALUE, "kv move: too many blocks");
  const long long vecs = block_bytes / 16;
  int bx = (int)((vecs + 255) / 256);
  if (bx > 8) bx = 8;
  kv_move_kernel<<<dim3(bx, segments, nblocks), 256, 0, S(stream)>>>(
      reinterpret_cast<const uint8_t*>(src_cache), reinterpret_cast<uint8_t*>(dst_cache), src_segment_stride,
      dst_segment_stride, block_bytes, src_ids, dst_ids);
  return cuda_status((int)cudaGetLastError(), "kv move");
}

epd_status_t epd_kv_pack(const void* cache, int32_t segments, int64_t segment_stride, int64_t block_bytes,
                         const int32_t* block_ids, int32_t nblocks, void* out, void* stream) {
  return kv_copy(cache, out, segments, segment_stride, block_bytes, block_ids, nblocks, 1, stream);
}

epd_status_t epd_kv_unpack(const void* in, int32_t segments, int64_t segment_stride, int64_t block_bytes,
                           const int32_t* block_ids, int32_t nblocks, void* cache, void* stream) {
  return kv_copy(in, cache, segments, segment_stride, block_bytes, block_ids, nblocks, 0, stream);
}

// ------------------------------------------------------------------ kernel-level ops

epd_status_t epd_linear_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M, int32_t N,
                             int32_t K, const void* bias, int32_t act, const void* resid, int32_t ldr,
                             int32_t r_mod, const void* lscale, void* out, int32_t ldo, int32_t bn,
                             void* stream) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(EPD_ERR_VALUE, "linear: empty shape");
  if (act < 0 || act > 3) return fail(EPD_ERR_VALUE, "linear: unknown activation");
  if (ldo % 8 || (resid && ldr % 8) || ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(bias) |
                                          reinterpret_cast<uintptr_t>(resid) | reinterpret_cast<uintptr_t>(lscale)) & 15))
    return fail(EPD_ERR_VALUE, "linear: epilogue tensors must be 16-byte aligned");
  epd::EpiParams ep;
  ep.act = act;
  ep.bias = reinterpret_cast<const epd::bf16*>(bias);
  ep.resid = reinterpret_cast<const epd::bf16*>(resid);
  ep.ldr = ldr;
  ep.r_mod = r_mod > 0 ? r_mod : 0x7fffffff;
  ep.lscale = reinterpret_cast<const epd::bf16*>(lscale);
  ep.out = reinterpret_cast<epd::bf16*>(out);
  ep.ldo = ldo;
  int rc = epd::gemm_bf16(reinterpret_cast<const epd::bf16*>(A), lda, reinterpret_cast<const epd::bf16*>(W), ldw,
                          M, N, K, ep, S(stream), bn);
  return cuda_status(rc, "linear_bf16");
}

epd_status_t epd_set_gemm_cta_group(int32_t policy) {
  if (policy != 0 && policy != 1 && policy != 2 && policy != 4)
    return fail(EPD_ERR_VALUE, "cta group policy must be 0, 1, 2 or 4");
  epd::set_gemm_cta_group(policy);
  return EPD_OK;
}

epd_status_t epd_linear_acc_f32(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M, int32_t N,
                                int32_t K, const void* bias, const void* lscale, float* h, int32_t ldh, int32_t bn,
                                void* stream) {
  return epd_linear_acc_f32_split(A, lda, W, ldw, M, N, K, bias, lscale, h, ldh, bn, 0, stream);
}

epd_status_t epd_linear_acc_f32_split(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M,
                                      int32_t N, int32_t K, const void* bias, const void* lscale, float* h,
                                      int32_t ldh, int32_t bn, int32_t max_split, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || !h) return fail(EPD_ERR_VALUE, "linear_acc: empty shape or null output");
  if (max_split < 0 || max_split > 16) return fail(EPD_ERR_VALUE, "linear_acc: max_split must be 0..16");
  if (ldh % 4 || (reinterpret_cast<uintptr_t>(h) & 15)) return fail(EPD_ERR_VALUE, "linear_acc: h must be 16-byte aligned");
  epd::EpiParams ep;
  ep.bias = reinterpret_cast<const epd::bf16*>(bias);
  ep.lscale = reinterpret_cast<const epd::bf16*>(lscale);
  ep.resid_f = h;
  ep.out_f = h;
  ep.ldr = ldh;
  ep.ldo = ldh;
  ep.max_split = max_split;
  int rc = epd::gemm_bf16(reinterpret_cast<const epd::bf16*>(A), lda, reinterpret_cast<const epd::bf16*>(W), ldw,
                          M, N, K, ep, S(stream), bn);
  return cuda_status(rc, "linear_acc_f32");
}

epd_status_t epd_linear_heads_bf16(const void* A, int32_t lda, const void* W, int32_t ldw, int32_t M,
                                   int32_t N, int32_t K, const void* bias, const void* resid, int32_t ldr,
                                   int32_t r_mod, int32_t H, int32_t Dp, int32_t T, int32_t Tpad,
                                   int32_t sec_cols, void* out0, void* out1, void* out2, int32_t trans_mask,
                                   void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || H <= 0 || T <= 0 || sec_cols <= 0)
    return fail(EPD_ERR_VALUE, "linear_heads: empty shape");
  epd::EpiParams ep;
  ep.mode = epd::EPI_HEADS;
  ep.bias = reinterpret_cast<const epd::bf16*>(bias);
  ep.resid = reinterpret_cast<const epd::bf16*>(resid);
  ep.ldr = ldr;
  ep.r_mod = r_mod > 0 ? r_mod : 0x7fffffff;
  ep.H = H; ep.Dp = Dp; ep.T = T; ep.Tpad = Tpad; ep.sec_cols = sec_cols;
  void* outs[3] = {out0, out1, out2};
  for (int s = 0; s < 3; ++s) {
    ep.sec_out[s] = reinterpret_cast<epd::bf16*>(outs[s]);
    ep.sec_trans[s] = (trans_mask >> s) & 1;
  }
  int rc = epd::gemm_bf16(reinterpret_cast<const epd::bf16*>(A), lda, reinterpret_cast<const epd::bf16*>(W), ldw,
                          M, N, K, ep, S(stream), 0);
  return cuda_status(rc, "linear_heads_bf16");
}

epd_status_t epd_attention_bf16(const void* q, int32_t ldq, const void* k, int32_t ldk, const void* v,
                                int32_t ldv, void* out, int32_t ldo, int32_t B, int32_t H, int32_t kv_heads,
                                int32_t Tq, int32_t Tk, int32_t Dp, int32_t Dv, int32_t head_stride,
                                int32_t flags, float scale, void* stream) {
  if (kv_heads < 0 || (kv_heads > 0 && (H % kv_heads))) return fail(EPD_ERR_VALUE, "attention: H % kv_heads != 0");
  epd::AttnParams p;
  p.q = reinterpret_cast<const epd::bf16*>(q);
  p.k = reinterpret_cast<const epd::bf16*>(k);
  p.v = reinterpret_cast<const epd::bf16*>(v);
  p.out = reinterpret_cast<epd::bf16*>(out);
  p.ldq = ldq; p.ldk = ldk; p.ldv = ldv; p.hs = head_stride;
  p.B = B; p.H = H; p.Tq = Tq; p.Tk = Tk; p.Dp = Dp; p.Dv = Dv; p.ldo = ldo;
  p.kv_group = kv_heads > 0 ? H / kv_heads : 1;
  p.q_shared = (flags & EPD_ATTN_Q_SHARED) != 0;
  p.causal = (flags & EPD_ATTN_CAUSAL) != 0;
  p.scale = scale;
  return cuda_status(epd::attention_bf16(p, S(stream)), "attention_bf16");
}

epd_status_t epd_layernorm_bf16(const void* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                const void* beta, int32_t rows, int32_t D, float eps, void* stream) {
  return cuda_status(epd::layernorm_bf16(reinterpret_cast<const epd::bf16*>(in), ld_in,
                                         reinterpret_cast<epd::bf16*>(out), ld_out,
                                         reinterpret_cast<const epd::bf16*>(gamma),
                                         reinterpret_cast<const epd::bf16*>(beta), rows, D, eps, S(stream)),
                     "layernorm_bf16");
}

epd_status_t epd_layernorm_f32_bf16(const float* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                    const void* beta, int32_t rows, int32_t D, float eps, void* stream) {
  return cuda_status(epd::layernorm_f32in(in, ld_in, reinterpret_cast<epd::bf16*>(out), ld_out,
                                          reinterpret_cast<const epd::bf16*>(gamma),
                                          reinterpret_cast<const epd::bf16*>(beta), rows, D, eps, nullptr, 1,
                                          S(stream)),
                     "layernorm_f32_bf16");
}

epd_status_t epd_patchify_u8(const uint8_t* tiles, int32_t n, int32_t Sz, int32_t C, int32_t p, int32_t Kpad,
                             int32_t row_offset, int32_t rows_per_tile, const float* mean3, const float* std3,
                             void* out, void* stream) {
  if (!mean3 || !std3) return fail(EPD_ERR_VALUE, "patchify: null mean/std");
  return cuda_status(epd::patchify_u8(tiles, n, Sz, C, p, Kpad, row_offset, rows_per_tile, mean3, std3,
                                      reinterpret_cast<epd::bf16*>(out), S(stream)),
                     "patchify_u8");
}

// ------------------------------------------------------------------ prefill consumer

epd_status_t epd_rmsnorm_f32_bf16(const float* in, int32_t ld_in, void* out, int32_t ld_out, const void* gamma,
                                  int32_t rows, int32_t D, float eps, void* stream) {
  return cuda_status(epd::rmsnorm_f32(in, ld_in, reinterpret_cast<epd::bf16*>(out), ld_out,
                                      reinterpret_cast<const epd::bf16*>(gamma), rows, D, eps, S(stream)),
                     "rmsnorm_f32_bf16");
}

epd_status_t epd_rope_bf16(void* x, int32_t ld, int32_t rows, int32_t col0, int32_t nheads, int32_t hd,
                           int32_t pos0, float theta, const float* cos_sin, void* stream) {
  return cuda_status(epd::rope_bf16(reinterpret_cast<epd::bf16*>(x), ld, rows, col0, nheads, hd, pos0, theta,
                                    cos_sin, S(stream)),
                     "rope_bf16");
}

epd_status_t epd_rope_table(float* cos_sin, int32_t rows, int32_t hd, int32_t pos0, float theta, void* stream) {
  return cuda_status(epd::rope_table(cos_sin, rows, hd, pos0, theta, S(stream)), "rope_table");
}

epd_status_t epd_silu_mul_bf16(const void* gu, int32_t ld_in, void* out, int32_t ld_out, int32_t rows, int32_t F,
                               void* stream) {
  return cuda_status(epd::silu_mul_bf16(reinterpret_cast<const epd::bf16*>(gu), ld_in,
                                        reinterpret_cast<epd::bf16*>(out), ld_out, rows, F, S(stream)),
                     "silu_mul_bf16");
}

epd_status_t epd_kv_write_paged(const void* src, int32_t ld_src, int32_t v_off, int32_t rows, int32_t row_elems,
                                const int32_t* block_ids, int32_t block_size, void* pool, int64_t seg_elems,
                                int32_t seg0, void* stream) {
  return cuda_status(epd::kv_write_paged(reinterpret_cast<const epd::bf16*>(src), ld_src, v_off, rows, row_elems,
                                         block_ids, block_size, reinterpret_cast<epd::bf16*>(pool),
                                         (size_t)seg_elems, seg0, S(stream)),
                     "kv_write_paged");
}

epd_status_t epd_gather_rows_f32(const void* src, int32_t ld_src, const int32_t* index, int32_t rows, int32_t D,
                                 float* dst, int32_t ld_dst, void* stream) {
  return cuda_status(epd::gather_rows_f32(reinterpret_cast<const epd::bf16*>(src), ld_src, index, rows, D, dst,
                                          ld_dst, S(stream)),
                     "gather_rows_f32");
}

epd_status_t epd_argmax_bf16(const void* x, int32_t n, int32_t* out, void* stream) {
  return cuda_status(epd::argmax_bf16(reinterpret_cast<const epd::bf16*>(x), n, out, S(stream)), "argmax_bf16");
}


epd_status_t epd_tile_image(const uint8_t* src, int32_t H, int32_t W, int32_t C, int32_t cols, int32_t rows,
                            int32_t thumb, int32_t thumb_first, int32_t tile, uint8_t* out, void* stream) {
  if (!src || !out) return fail(EPD_ERR_VALUE, "tile_image: null buffer");
  return cuda_status(epd::tile_image_u8(src, H, W, C, cols, rows, thumb, thumb_first, tile, out, S(stream)),
                     "tile_image");
}

epd_status_t epd_blocks_init(int32_t* stack, int32_t* top, int32_t total, void* stream) {
  return cuda_status(epd::blocks_init(stack, top, total, S(stream)), "blocks_init");
}

epd_status_t epd_blocks_alloc(int32_t* stack, int32_t* top, int32_t need, int32_t* out_ids, void* stream) {
  return cuda_status(epd::blocks_alloc(stack, top, need, out_ids, S(stream)), "blocks_alloc");
}

epd_status_t epd_blocks_free(int32_t* stack, int32_t* top, const int32_t* ids, int32_t n, void* stream) {
  return cuda_status(epd::blocks_free(stack, top, ids, n, S(stream)), "blocks_free");
}

}  // extern "C"
