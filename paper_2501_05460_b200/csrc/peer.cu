// EP gather over NVLink peer memory (the B200-native replacement of the NCCL grouped P2P
// in stage._gather; reference: engine._send_ready_shards / _schedule_transfer,
// engine.py:511-526, and _on_transfer_end("ep"), engine.py:424-435).
//
// Every encode rank maps the prefill rank's packed-token slots (CUDA IPC) and stores its
// shard of post-projector MM tokens straight into them at the shard's tile offset, then
// raises a per-rank sequence flag in the prefill rank's memory. The prefill rank's
// stream waits on its LOCAL flags with a stream memory operation (no spinning kernel),
// so the transfer needs no host round trip and no collective launch.
//
// Ordering: the put kernel's threads issue their 16-byte peer stores and then a
// system-scope fence; the signal kernel runs after the put kernel on the same stream and
// stores the flag with release semantics, so the data has reached the destination GPU
// before the flag does. The prefill rank's wait (GEQ on the flag) then orders every
// later kernel on its stream after the data.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace epd {

namespace {

__global__ void peer_put_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t vecs) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < vecs; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
}

__global__ void peer_signal_kernel(uint32_t* flag, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitFn wait_fn() {
  static WaitFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (WaitFn) nullptr;
    return reinterpret_cast<WaitFn>(p);
  }();
  return fn;
}

}  // namespace

int peer_put(const void* src, void* dst, size_t bytes, uint32_t* flag, uint32_t value, cudaStream_t s) {
  if (bytes % 16 || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)) return 1003;
  const size_t vecs = bytes / 16;
  if (vecs) {
    // one 16 B store per thread per pass; enough CTAs to keep the NVLink ingress busy
    // without taking SMs from the next encode for long
    size_t blocks = (vecs + 255) / 256;
    if (blocks > 2 * 148) blocks = 2 * 148;
    peer_put_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(src),
                                                      reinterpret_cast<uint4*>(dst), vecs);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  return flag ? peer_signal(flag, value, s) : 0;
}

int peer_signal(uint32_t* flag, uint32_t value, cudaStream_t s) {
  peer_signal_kernel<<<1, 1, 0, s>>>(flag, value);
  return (int)cudaGetLastError();
}

int stream_wait_geq(const uint32_t* flag, uint32_t value, cudaStream_t s) {
  WaitFn fn = wait_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorNotSupported;
}

}  // namespace epd
