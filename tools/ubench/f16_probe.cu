// Probes for a half-precision softmax: (1) MUFU throughput of ex2.approx.f16x2 against
// ex2.approx.f32 (exponentials per cycle per SM), (2) whether tcgen05.mma kind::f16 takes a
// f16 A operand (from TMEM) with a bf16 B operand (from SMEM) — checked numerically.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc f16_probe.cu -o f16_probe
#include <cstdio>
#include <cuda_fp16.h>
#include "common.cuh"
using namespace epd;

template <bool HALF>
__global__ void mufu(unsigned long long* out, float* sink, int iters) {
  uint32_t r[16];
  for (int j = 0; j < 16; ++j) r[j] = HALF ? 0xBC00BC00u - j : __float_as_uint(-1.0f - j * 0.01f);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (HALF) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[j]));
      else asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[j]));
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  uint32_t acc = 0;
  for (int j = 0; j < 16; ++j) acc ^= r[j];
  sink[threadIdx.x] = __uint_as_float(acc);
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void mixed_mma(float* d_out, int a_f16) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&holder, 128);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  // B: 64 rows (n) x 16 k, K-major SW128: row n at (n/8)*1024 + (n%8)*128, 16-B chunk c at c ^ (n%8)
  for (int idx = threadIdx.x; idx < 64 * 16; idx += blockDim.x) {
    const int n = idx / 16, k = idx % 16;
    const float v = (float)((n % 8) + k);
    const int chunk = (k * 2) / 16, within = (k * 2) % 16;
    const int off = (n / 8) * 1024 + (n % 8) * 128 + ((chunk ^ (n % 8)) * 16) + within;
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16(v);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  // A in TMEM (columns 64..71): row m = lane quarter * 32 + lane; A[m][k] = 1 if k == m % 16
  {
    const int m = warp * 32 + lane;
    uint32_t a[8];
    for (int c = 0; c < 8; ++c) {
      const int k0 = 2 * c, k1 = 2 * c + 1;
      uint16_t h0, h1;
      if (a_f16) {
        h0 = (k0 == m % 16) ? 0x3C00 : 0;
        h1 = (k1 == m % 16) ? 0x3C00 : 0;
      } else {
        h0 = (k0 == m % 16) ? 0x3F80 : 0;
        h1 = (k1 == m % 16) ? 0x3F80 : 0;
      }
      a[c] = h0 | ((uint32_t)h1 << 16);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + ((warp * 32) << 16) + 64),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = make_idesc_bf16(128, 64);
    if (a_f16) idesc &= ~(7u << 7);  // A format f16 (0), B stays bf16 (1)
    const uint64_t bdesc = make_sdesc(smem_u32(smem), 1024, 2);
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;" ::"r"(tm), "r"(tm + 64), "l"(bdesc), "r"(idesc) : "memory");
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const int m = warp * 32 + lane;
    uint32_t v[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld32(tm + ((warp * 32) << 16) + c0, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) d_out[m * 64 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 128); }
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 1 << 20);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    mufu<false><<<148, warps * 32>>>(d, sink, iters);
    unsigned long long h32 = 0, h16 = 0;
    cudaMemcpy(&h32, d, 8, cudaMemcpyDeviceToHost);
    mufu<true><<<148, warps * 32>>>(d, sink, iters);
    cudaMemcpy(&h16, d, 8, cudaMemcpyDeviceToHost);
    const double n = (double)warps * 32 * 16 * iters;
    printf("warps %2d: f32 ex2 %.2f exp/clk/SM   f16x2 ex2 %.2f exp/clk/SM\n", warps, n / h32, 2 * n / h16);
  }
  float* dout;
  cudaMalloc(&dout, 128 * 64 * 4);
  float* h = new float[128 * 64];
  for (int af16 : {0, 1}) {
    cudaFuncSetAttribute(mixed_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaMemset(dout, 0, 128 * 64 * 4);
    mixed_mma<<<1, 128, 16384>>>(dout, af16);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mma error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, dout, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        const float want = (float)((n % 8) + (m % 16));
        if (h[m * 64 + n] != want) {
          if (bad < 4) printf("  A %s: D[%d][%d] = %g want %g\n", af16 ? "f16" : "bf16", m, n, h[m * 64 + n], want);
          ++bad;
        }
      }
    printf("A %s x B bf16: %d mismatches of %d\n", af16 ? "f16" : "bf16", bad, 128 * 64);
  }
  return 0;
}
