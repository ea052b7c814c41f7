// Device-side block free list: the LIFO id semantics of the
// reference BlockManager (blocks.py:29, 52, 61) on device memory, so the paged MM / KV
// pools get their block ids without a host round trip. stack[0, *top) holds the free ids,
// stack[*top - 1] is handed out next; a fresh pool hands out 0, 1, 2, ...; freed ids go
// back in reverse so the next allocation returns them in their original order. One block
// per call, stream-ordered; capacity checks are the caller's (the host tracks the counts).
#include "common.cuh"
#include "kernels.h"

namespace epd {

namespace {

__global__ void blocks_init_kernel(int32_t* __restrict__ stack, int32_t* __restrict__ top, int total) {
  for (int i = threadIdx.x; i < total; i += blockDim.x) stack[i] = total - 1 - i;
  if (threadIdx.x == 0) *top = total;
}

__global__ void blocks_alloc_kernel(int32_t* __restrict__ stack, int32_t* __restrict__ top, int need,
                                    int32_t* __restrict__ out) {
  const int t = *top;
  for (int i = threadIdx.x; i < need; i += blockDim.x) out[i] = stack[t - 1 - i];
  __syncthreads();
  if (threadIdx.x == 0) *top = t - need;
}

__global__ void blocks_free_kernel(int32_t* __restrict__ stack, int32_t* __restrict__ top,
                                   const int32_t* __restrict__ ids, int n) {
  const int t = *top;
  for (int i = threadIdx.x; i < n; i += blockDim.x) stack[t + i] = ids[n - 1 - i];
  __syncthreads();
  if (threadIdx.x == 0) *top = t + n;
}

}  // namespace

int blocks_init(int32_t* stack, int32_t* top, int total, cudaStream_t s) {
  if (total < 0) return 1001;
  blocks_init_kernel<<<1, 256, 0, s>>>(stack, top, total);
  return (int)cudaGetLastError();
}

int blocks_alloc(int32_t* stack, int32_t* top, int need, int32_t* out, cudaStream_t s) {
  if (need < 0) return 1001;
  if (need == 0) return 0;
  blocks_alloc_kernel<<<1, 256, 0, s>>>(stack, top, need, out);
  return (int)cudaGetLastError();
}

int blocks_free(int32_t* stack, int32_t* top, const int32_t* ids, int n, cudaStream_t s) {
  if (n < 0) return 1001;
  if (n == 0) return 0;
  blocks_free_kernel<<<1, 256, 0, s>>>(stack, top, ids, n);
  return (int)cudaGetLastError();
}

}  // namespace epd
