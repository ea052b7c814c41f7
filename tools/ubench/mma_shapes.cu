// Micro-benchmark: cycles per tcgen05.mma (M = 128, K = 16, bf16, cta_group::1) as a function
// of N, of where A lives (TMEM: TS form, or SMEM: SS form) and of B's layout (K-major SW128,
// or MN-major SW32 as the attention's V). Answers: which of the attention's MMAs run above
// the floor 128*N/256 cycles, and why.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc mma_shapes.cu -o mma_shapes
#include <cstdio>
#include "common.cuh"
using namespace epd;

__device__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// TS: A from TMEM; BMN: B MN-major SW32 (else K-major SW128); AMN: A MN-major SW32 (SS only)
template <bool TS, bool BMN, int N, bool AMN = false>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) tmem_alloc(&holder, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3E003E00u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (threadIdx.x < 32) {
    const uint32_t base = smem_u32(smem);
    uint64_t bdesc = BMN ? make_sdesc_lbo(base + 32768, 2048, 256, 6) : make_sdesc(base + 32768, 1024, 2);
    uint64_t adesc = AMN ? make_sdesc_lbo(base, 2048, 256, 6) : make_sdesc(base, 1024, 2);
    uint32_t idesc = make_idesc_bf16(128, N) | (BMN ? (1u << 16) : 0u) | (AMN ? (1u << 15) : 0u);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
        if (TS) umma_ts(tm + 256, tm + (i & 3) * 8, bdesc + (BMN ? (i & 3) * 32 : (i & 3) * 2), idesc, 1);
        else umma_bf16(tm + 256, adesc + (AMN ? (i & 3) * 32 : (i & 3) * 2), bdesc + (BMN ? (i & 3) * 32 : (i & 3) * 2), idesc, 1);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <bool TS, bool BMN, int N, bool AMN = false>
void run(unsigned long long* d, const char* name) {
  const int iters = 8192;
  cudaFuncSetAttribute(k<TS, BMN, N, AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  k<TS, BMN, N, AMN><<<148, 128, 98304>>>(d, iters);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  printf("%-8s B %-10s N %3d: %6.1f cyc/MMA (floor %5.1f)\n", name, BMN ? "MN-SW32" : "K-SW128", N, (double)h / iters,
         128.0 * N / 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
#define ALLN(TS, BMN, NAME) \
  run<TS, BMN, 32>(d, NAME); run<TS, BMN, 48>(d, NAME); run<TS, BMN, 64>(d, NAME); run<TS, BMN, 80>(d, NAME); \
  run<TS, BMN, 96>(d, NAME); run<TS, BMN, 128>(d, NAME); run<TS, BMN, 160>(d, NAME); run<TS, BMN, 256>(d, NAME);
  ALLN(true, false, "TS")
  ALLN(false, false, "SS")
  ALLN(true, true, "TS")
  ALLN(false, true, "SS")
  run<false, true, 80, true>(d, "SS A-MN");
  run<false, false, 80, true>(d, "SS A-MN");
  return 0;
}
