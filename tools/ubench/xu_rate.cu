// Issue-rate probe for the softmax / GELU instruction mix on one B200 SM (148 blocks, one per
// SM): results per clock per SM of MUFU.EX2, MUFU.RCP, F2FP.BF16.F32.PACK_AB and FFMA2.
// Each thread runs 16 independent chains, so the rate is the pipe's throughput, not latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 xu_rate.cu -o xu_rate
#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void rate(unsigned long long* out, uint32_t* sink, int iters) {
  uint32_t r[16];
  for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(-1.0f - 0.01f * (j + threadIdx.x % 7));
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[j]));
      if (OP == 2) asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(r[j]) : "r"(r[(j + 1) & 15]));
      if (OP == 3)
        asm volatile("{.reg .b64 a; mov.b64 a, {%0,%1}; fma.rn.f32x2 a, a, a, a; mov.b64 {%0,%1}, a;}"
                     : "+r"(r[j]), "+r"(r[(j + 8) & 15]));
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
  for (int j = 0; j < 16; ++j) acc ^= r[j];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int OP>
double run(int warps, unsigned long long* d, uint32_t* sink) {
  const int iters = 2048;
  rate<OP><<<148, warps * 32>>>(d, sink, iters);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  return (double)warps * 32 * 16 * iters / (double)c;  // lane-results per clock per SM
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 148 * 1024 * 4);
  for (int warps : {8, 16, 32}) {
    printf("warps %2d: ex2 %.1f  f2fp(bf16x2) %.1f  ffma2 %.1f  (lane ops / clk / SM)\n", warps,
           run<0>(warps, d, sink), run<2>(warps, d, sink), run<3>(warps, d, sink));
  }
  return 0;
}
