// Internal interface of the multimodal-token cache kernels (see mmcache.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace epd {

struct DeviceTable {
  unsigned long long* keys = nullptr;  // [capacity][2]
  int32_t* vals = nullptr;             // [capacity]
  int32_t* status = nullptr;           // [1], set to 1 if an insert found no free slot
  unsigned long long capacity = 0;     // power of two
};

// Device-side cache planner state (see mmcache.cu "planner"): the LRU order of entries as a
// doubly linked list, the LIFO free stack of entry ids and each entry's key.
struct DevicePlanner {
  int32_t capacity = 0;                   // entries
  int32_t* prev = nullptr;                // [capacity]
  int32_t* next = nullptr;                // [capacity]
  int32_t* free_stack = nullptr;          // [capacity]
  int32_t* state = nullptr;               // [8]: head, tail, free_top, tombstones
  unsigned long long* entry_key = nullptr;  // [capacity][2]
};

// Outputs of one plan (device, caller-owned; n = tiles of the request):
//   entries[n], kinds[n] (0 hit / 1 miss / 2 dup), miss_tiles[n] and miss_entries[n] (first
//   counts[0] valid), victim_keys[n][2] (first counts[3] valid), counts[5] = misses, hits,
//   dups, victims, status (1 = more distinct tiles than the cache holds; nothing changed).
struct PlanOut {
  int32_t* entries;
  int32_t* kinds;
  int32_t* miss_tiles;
  int32_t* miss_entries;
  unsigned long long* victim_keys;
  int32_t* counts;
};

int planner_reset(const DeviceTable& t, const DevicePlanner& p, cudaStream_t stream);
int planner_plan(const DeviceTable& t, const DevicePlanner& p, const unsigned long long* keys, int n,
                 const PlanOut& out, cudaStream_t stream);
size_t planner_max_tiles();
int32_t planner_max_capacity();

int hash_records(const void* data, int n, size_t rec_bytes, size_t rec_stride,
                 unsigned long long* acc_scratch, unsigned long long* keys, cudaStream_t stream,
                 unsigned long long s0 = 0, unsigned long long s1 = 0);
int table_lookup(const DeviceTable& t, const unsigned long long* keys, int n, int32_t* out,
                 cudaStream_t stream);
int table_dedup(const unsigned long long* keys, const int32_t* lookup, int n, int32_t* dup,
                cudaStream_t stream);
int table_insert(const DeviceTable& t, const unsigned long long* keys, const int32_t* vals, int n,
                 cudaStream_t stream);
int table_erase(const DeviceTable& t, const unsigned long long* keys, int n, cudaStream_t stream);

}  // namespace epd
