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

int hash_records(const void* data, int n, size_t rec_bytes, size_t rec_stride,
                 unsigned long long* acc_scratch, unsigned long long* keys, cudaStream_t stream);
int table_lookup(const DeviceTable& t, const unsigned long long* keys, int n, int32_t* out,
                 cudaStream_t stream);
int table_dedup(const unsigned long long* keys, const int32_t* lookup, int n, int32_t* dup,
                cudaStream_t stream);
int table_insert(const DeviceTable& t, const unsigned long long* keys, const int32_t* vals, int n,
                 cudaStream_t stream);
int table_erase(const DeviceTable& t, const unsigned long long* keys, int n, cudaStream_t stream);

}  // namespace epd
