// Micro-benchmark: cycles per tcgen05.mma for the operand layouts the attention kernel uses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include "common.cuh"
using namespace epd;

__device__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) tmem_alloc(&holder, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(smem);
    const uint64_t a128 = make_sdesc(base, 1024, 2), b128 = make_sdesc(base + 16384, 1024, 2);
    const uint64_t a32 = make_sdesc(base, 256, 6), b32 = make_sdesc(base + 16384, 256, 6);
    const uint64_t vmn = make_sdesc_lbo(base + 32768, 4096, 256, 6);
    const uint32_t id_s = make_idesc_bf16(128, 128);
    const uint32_t id_o = make_idesc_bf16(128, 80) | (1u << 16);
    const uint32_t id_256 = make_idesc_bf16(128, 256);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0) umma_bf16(tm, a128 + (i & 3) * 2, b128 + (i & 3) * 2, id_s, 1);        // S main: SS SW128 N=128
      if (MODE == 1) umma_bf16(tm, a32, b32, id_s, 1);                                      // S tail: SS SW32 N=128
      if (MODE == 2) umma_ts(tm + 256, tm + (i & 7) * 8, vmn + (i & 7) * 32, id_o, 1);     // PV: TS, V MN-major SW32 N=80
      if (MODE == 3) umma_bf16(tm, a128 + (i & 3) * 2, b128 + (i & 3) * 2, id_256, 1);     // GEMM-like N=256
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[MODE] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int iters = 4096;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<0><<<1, 128, 65536>>>(d, iters);
  k<1><<<1, 128, 65536>>>(d, iters);
  k<2><<<1, 128, 65536>>>(d, iters);
  k<3><<<1, 128, 65536>>>(d, iters);
  unsigned long long h[4];
  cudaError_t e = cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  const char* names[4] = {"S main SS SW128 M128 N128", "S tail SS SW32 M128 N128", "PV TS P-tmem V-MN-SW32 N80",
                          "SS SW128 M128 N256"};
  for (int m = 0; m < 4; ++m) printf("%-30s %.1f cycles/MMA\n", names[m], (double)h[m] / iters);
  return 0;
}
