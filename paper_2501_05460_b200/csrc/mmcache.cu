// Multimodal-token cache: tile-content hash (K11) and a GPU-resident
// open-addressing hash table keyed by that hash (K12).
//
// Content hash (the cache key) of a byte record of length L (L % 8 == 0):
//   w_i  = little-endian u64 word i
//   x_i  = w_i ^ (i * 0x9E3779B97F4A7C15 + 0x243F6A8885A308D3)
//   a_i  = fmix64(x_i);  b_i = fmix64(a_i + 0x632BE59BD9B4E019)
//   key0 = fmix64((sum a_i) ^ L);  key1 = fmix64((sum b_i) + L * 0xD6E8FEB86659FD93)
//   if key0 == 0: key0 = 1          (key0 == 0 marks empty / tombstone slots)
// Sums are mod 2^64 and order-independent, so any thread/block decomposition
// produces identical keys (bit-exact with oracle/hashing.py).
//
// Table: capacity C = 2^k slots of {key0, key1, value}; linear probing from
// key0 & (C-1). Empty = (0,0), tombstone = (0,1).
#include "common.cuh"
#include "kernels.h"
#include "mmcache.h"

namespace epd {

namespace {

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kSeed = 0x243F6A8885A308D3ull;
constexpr unsigned long long kLaneB = 0x632BE59BD9B4E019ull;
constexpr unsigned long long kLenMul = 0xD6E8FEB86659FD93ull;

__device__ __forceinline__ unsigned long long fmix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb53fe5d4a1a3ull;
  k ^= k >> 33;
  return k;
}

__global__ void __launch_bounds__(256) hash_accum_kernel(const uint8_t* __restrict__ data,
                                                         size_t rec_bytes, size_t rec_stride,
                                                         unsigned long long* __restrict__ acc) {
  const int rec = blockIdx.y;
  const size_t nwords = rec_bytes / 8;
  const uint8_t* base = data + (size_t)rec * rec_stride;
  unsigned long long sa = 0, sb = 0;
  // 16-byte loads: two words per thread-iteration when aligned.
  const size_t npairs = nwords / 2;
  const bool aligned = ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  if (aligned) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(base);
    for (size_t i = tid; i < npairs; i += nth) {
      ulonglong2 w = p[i];
      const unsigned long long i0 = 2 * i, i1 = 2 * i + 1;
      unsigned long long a0 = fmix64(w.x ^ (i0 * kGolden + kSeed));
      unsigned long long a1 = fmix64(w.y ^ (i1 * kGolden + kSeed));
      sa += a0 + a1;
      sb += fmix64(a0 + kLaneB) + fmix64(a1 + kLaneB);
    }
    if (tid == 0 && (nwords & 1)) {
      const size_t i = nwords - 1;
      unsigned long long w = reinterpret_cast<const unsigned long long*>(base)[i];
      unsigned long long a = fmix64(w ^ (i * kGolden + kSeed));
      sa += a;
      sb += fmix64(a + kLaneB);
    }
  } else {
    for (size_t i = tid; i < nwords; i += nth) {
      unsigned long long w = 0;
      for (int j = 7; j >= 0; --j) w = (w << 8) | base[i * 8 + j];
      unsigned long long a = fmix64(w ^ (i * kGolden + kSeed));
      sa += a;
      sb += fmix64(a + kLaneB);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  __shared__ unsigned long long red[2][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][warp] = sa;
    red[1][warp] = sb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ta = 0, tb = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      ta += red[0][w];
      tb += red[1][w];
    }
    atomicAdd(&acc[2 * rec + 0], ta);
    atomicAdd(&acc[2 * rec + 1], tb);
  }
}

__global__ void hash_finalize_kernel(const unsigned long long* __restrict__ acc, int n,
                                     unsigned long long len, unsigned long long* __restrict__ keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k0 = fmix64(acc[2 * i] ^ len);
  unsigned long long k1 = fmix64(acc[2 * i + 1] + len * kLenMul);
  if (k0 == 0) k0 = 1;
  keys[2 * i] = k0;
  keys[2 * i + 1] = k1;
}

__global__ void table_lookup_kernel(const unsigned long long* __restrict__ tkeys,
                                    const int32_t* __restrict__ tvals, unsigned long long mask,
                                    const unsigned long long* __restrict__ keys, int n,
                                    int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k0 = keys[2 * i], k1 = keys[2 * i + 1];
  unsigned long long s = k0 & mask;
  int32_t v = -1;
  for (unsigned long long probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    const unsigned long long a = tkeys[2 * s], b = tkeys[2 * s + 1];
    if (a == 0 && b == 0) break;  // empty: chain ends
    if (a == k0 && b == k1) {
      v = tvals[s];
      break;
    }
  }
  out[i] = v;
}

// For entries with lookup miss, point later duplicates at their first
// occurrence within the batch: dup[i] = smallest j < i with equal key and
// lookup[j] < 0, else -1. Hits get dup = -1.
__global__ void batch_dedup_kernel(const unsigned long long* __restrict__ keys,
                                   const int32_t* __restrict__ lookup, int n,
                                   int32_t* __restrict__ dup) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t d = -1;
    if (lookup[i] < 0) {
      const unsigned long long k0 = keys[2 * i], k1 = keys[2 * i + 1];
      for (int j = 0; j < i; ++j) {
        if (keys[2 * j] == k0 && keys[2 * j + 1] == k1) {
          d = j;
          break;
        }
      }
    }
    dup[i] = d;
  }
}

__global__ void table_insert_kernel(unsigned long long* __restrict__ tkeys, int32_t* __restrict__ tvals,
                                    unsigned long long mask, const unsigned long long* __restrict__ keys,
                                    const int32_t* __restrict__ vals, int n, int32_t* __restrict__ status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k0 = keys[2 * i], k1 = keys[2 * i + 1];
  unsigned long long s = k0 & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    // claim an empty or tombstoned slot (key0 == 0)
    if (atomicCAS(&tkeys[2 * s], 0ull, k0) == 0ull) {
      tkeys[2 * s + 1] = k1;
      tvals[s] = vals[i];
      return;
    }
  }
  atomicExch(status, 1);  // table full
}

__global__ void table_erase_kernel(unsigned long long* __restrict__ tkeys, int32_t* __restrict__ tvals,
                                   unsigned long long mask, const unsigned long long* __restrict__ keys,
                                   int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k0 = keys[2 * i], k1 = keys[2 * i + 1];
  unsigned long long s = k0 & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    const unsigned long long a = tkeys[2 * s], b = tkeys[2 * s + 1];
    if (a == 0 && b == 0) return;
    if (a == k0 && b == k1) {
      tkeys[2 * s + 1] = 1ull;  // tombstone = (0, 1)
      tkeys[2 * s] = 0ull;
      tvals[s] = -1;
      return;
    }
  }
}

}  // namespace

int hash_records(const void* data, int n, size_t rec_bytes, size_t rec_stride,
                 unsigned long long* acc_scratch, unsigned long long* keys, cudaStream_t stream) {
  if (n <= 0) return 0;
  if (rec_bytes % 8) return 1002;
  cudaError_t e = cudaMemsetAsync(acc_scratch, 0, sizeof(unsigned long long) * 2 * n, stream);
  if (e != cudaSuccess) return (int)e;
  const size_t words = rec_bytes / 8;
  int bx = (int)((words / 2 + 256 * 8 - 1) / (256 * 8));
  if (bx < 1) bx = 1;
  if (bx > 16) bx = 16;
  hash_accum_kernel<<<dim3(bx, n), 256, 0, stream>>>(reinterpret_cast<const uint8_t*>(data), rec_bytes,
                                                     rec_stride, acc_scratch);
  hash_finalize_kernel<<<(n + 127) / 128, 128, 0, stream>>>(acc_scratch, n, (unsigned long long)rec_bytes,
                                                            keys);
  return (int)cudaGetLastError();
}

int table_lookup(const DeviceTable& t, const unsigned long long* keys, int n, int32_t* out,
                 cudaStream_t stream) {
  if (n <= 0) return 0;
  table_lookup_kernel<<<(n + 127) / 128, 128, 0, stream>>>(t.keys, t.vals, t.capacity - 1, keys, n, out);
  return (int)cudaGetLastError();
}

int table_dedup(const unsigned long long* keys, const int32_t* lookup, int n, int32_t* dup,
                cudaStream_t stream) {
  if (n <= 0) return 0;
  batch_dedup_kernel<<<(n + 255) / 256, 256, 0, stream>>>(keys, lookup, n, dup);
  return (int)cudaGetLastError();
}

int table_insert(const DeviceTable& t, const unsigned long long* keys, const int32_t* vals, int n,
                 cudaStream_t stream) {
  if (n <= 0) return 0;
  table_insert_kernel<<<(n + 127) / 128, 128, 0, stream>>>(t.keys, t.vals, t.capacity - 1, keys, vals, n,
                                                           t.status);
  return (int)cudaGetLastError();
}

int table_erase(const DeviceTable& t, const unsigned long long* keys, int n, cudaStream_t stream) {
  if (n <= 0) return 0;
  table_erase_kernel<<<(n + 127) / 128, 128, 0, stream>>>(t.keys, t.vals, t.capacity - 1, keys, n);
  return (int)cudaGetLastError();
}

}  // namespace epd
