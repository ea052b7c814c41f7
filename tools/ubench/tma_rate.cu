// Micro-benchmark: TMA load throughput per SM (the GEMM producer's pattern: 2-D SW128 boxes
// of 64 bf16 columns x R rows into a ring of S stages, one elected thread issuing, one
// consumer thread releasing each stage as soon as it lands). Reports bytes per SM-cycle and
// aggregate TB/s for a source that fits in L2 and one that streams from HBM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc tma_rate.cu -o tma_rate -lcuda
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "tmap.h"
using namespace epd;

template <int ROWS, int STAGES, int BOXES>
__global__ void __launch_bounds__(64, 1) tma_rate(const __grid_constant__ CUtensorMap tm, int iters, int kblocks,
                                                  int rowblocks, int share, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int BOX = ROWS * 128;
  constexpr int STAGE = BOX * BOXES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm);
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&full[stage], STAGE);
      const int kb = i % kblocks;
      for (int b = 0; b < BOXES; ++b) {
        const int rb = ((blockIdx.x / share) * BOXES + b + (i / kblocks) * (gridDim.x / share + 1) * BOXES) % rowblocks;
        tma_load_2d(smem + stage * STAGE + b * BOX, &tm, &full[stage], kb * 64, rb * ROWS);
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ROWS, int STAGES, int BOXES>
void run(const void* base, uint64_t K, uint64_t rows, int grid, const char* src, int share = 1) {
  CUtensorMap tm;
  if (make_tmap_2d(&tm, base, K, rows, K * 2, 64, ROWS, CU_TENSOR_MAP_SWIZZLE_128B)) {
    printf("tmap failed\n");
    return;
  }
  const int smem = STAGES * ROWS * 128 * BOXES + 1024 + 256;
  auto k = tma_rate<ROWS, STAGES, BOXES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, grid * sizeof(unsigned long long));
  const int iters = 4000;
  const int kblocks = (int)(K / 64), rowblocks = (int)(rows / ROWS);
  k<<<grid, 64, smem>>>(tm, 200, kblocks, rowblocks, share, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, 64, smem>>>(tm, iters, kblocks, rowblocks, share, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto c : h) mx = c > mx ? c : mx;
  const double bytes = (double)iters * ROWS * 128 * BOXES * grid;
  printf("%-4s grid %3d share %3d box %3d rows x%d stages %2d (%3d KB in flight): %6.1f B/clk/SM  %5.2f TB/s\n", src,
         grid, share, ROWS, BOXES, STAGES, STAGES * ROWS * 128 * BOXES / 1024, bytes / grid / mx, bytes / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main() {
  const uint64_t K = 4096;
  void* mid;
  const uint64_t rows_mid = 8192;  // 64 MB: L2-resident, larger than one die's half
  cudaMalloc(&mid, K * rows_mid * 2);
  cudaMemset(mid, 1, K * rows_mid * 2);
  for (int share : {1, 2, 4, 8, 13, 37, 148}) run<128, 6, 2>(mid, K, rows_mid, 148, "L2", share);
  for (int share : {1, 13}) run<256, 3, 2>(mid, K, rows_mid, 148, "L2", share);
  return 0;
}

int main_old() {
  const uint64_t K = 4096;
  void *small, *big;
  const uint64_t rows_small = 2048, rows_big = 131072;  // 16 MB (L2) and 1 GB (HBM)
  cudaMalloc(&small, K * rows_small * 2);
  cudaMalloc(&big, K * rows_big * 2);
  cudaMemset(small, 1, K * rows_small * 2);
  cudaMemset(big, 1, K * rows_big * 2);
  for (const char* src : {"L2", "HBM"}) {
    const void* base = src[0] == 'L' ? small : big;
    const uint64_t rows = src[0] == 'L' ? rows_small : rows_big;
    for (int grid : {72, 148}) {
      run<128, 6, 2>(base, K, rows, grid, src);   // the pair GEMM's stage: A 16 KB + B 16 KB
      run<128, 4, 2>(base, K, rows, grid, src);
      run<128, 12, 1>(base, K, rows, grid, src);
      run<128, 6, 1>(base, K, rows, grid, src);
      run<64, 8, 3>(base, K, rows, grid, src);
      run<256, 3, 2>(base, K, rows, grid, src);
    }
  }
  return 0;
}
