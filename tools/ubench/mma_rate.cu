// Micro-benchmark: cycles per tcgen05.mma for the operand layouts the attention kernel
// uses, alone and under concurrent TMEM load/store traffic from other warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include "common.cuh"
using namespace epd;

__device__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// MODE: 0 S SS SW128 N128 | 1 S SS SW32 N128 | 2 PV TS N80 | 3 SS N256 | 4 S TS SW128 N128
//       5 S TS SW32 N128 | 6 attention block mix 2x(4 S-TS-SW128 + 1 S-TS-SW32 + 8 PV-TS) per iter
// NOISE: warps 4..11 stream tcgen05.ld x32 / st x32 over TMEM columns 0..255 (softmax-like)
__device__ int g_rand;
template <int MODE, int NOISE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  __shared__ uint64_t dbar[8];
  __shared__ volatile int stop;
  if (threadIdx.x < 32) tmem_alloc(&holder, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&dbar[i], 1);
    fence_barrier_init();
    stop = 0;
  }
  // random bf16 operands in (-1, 1): exponent 0x3F/0x3E/0xBF..., random mantissas
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u + 12345u);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const uint32_t lo = 0x3E00u | (x & 0x81FFu), hi = 0x3E00u | ((x >> 16) & 0x81FFu);
    reinterpret_cast<uint32_t*>(smem)[i] = g_rand ? (lo | (hi << 16)) : 0u;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  const int warp = threadIdx.x / 32;
  if (g_rand && warp < 4) {  // random A operands / accumulators in TMEM too
    uint32_t v[32];
    for (int c = 0; c < 512; c += 32) {
      for (int j = 0; j < 32; ++j) v[j] = reinterpret_cast<uint32_t*>(smem)[(c + j + threadIdx.x * 7) & 16383];
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + ((warp * 32) << 16) + c),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
          "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
          "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
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
      if (MODE == 0) umma_bf16(tm, a128 + (i & 3) * 2, b128 + (i & 3) * 2, id_s, 1);
      if (MODE == 1) umma_bf16(tm, a32, b32, id_s, 1);
      if (MODE == 2) umma_ts(tm + 256, tm + (i & 7) * 8, vmn + (i & 7) * 32, id_o, 1);
      if (MODE == 3) umma_bf16(tm, a128 + (i & 3) * 2, b128 + (i & 3) * 2, id_256, 1);
      if (MODE == 4) umma_ts(tm, tm + 336 + (i & 3) * 8, b128 + (i & 3) * 2, id_s, 1);
      if (MODE == 5) umma_ts(tm, tm + 336 + 32, b32, id_s, 1);
      if (MODE == 7) umma_ts(tm, tm + 336 + (i & 3) * 8, b128 + (i & 3) * 2, make_idesc_bf16(128, 64), 1);
      if (MODE == 8) umma_ts(tm + 256, tm + (i & 3) * 8, vmn + (i & 3) * 32, id_o, 1);
      if (MODE == 9 || MODE == 10) {  // KB=64 kernel sequence per block, with commits (+ fences)
        const uint32_t id_s64 = make_idesc_bf16(128, 64);
        for (int g = 0; g < 2; ++g) {
          if (MODE == 10) tc_fence_after();
          for (int kk = 0; kk < 4; ++kk) umma_ts(tm + 256 + g * 128, tm + (2 * g) * 64 + kk * 8, vmn + kk * 32, id_o, 1);
          tc_commit(&dbar[g]);
          if (MODE == 10) tc_fence_after();
          for (int kk = 0; kk < 4; ++kk) umma_ts(tm + (2 * g + 1) * 64, tm + 336 + g * 128 + kk * 8, b128 + kk * 2, id_s64, kk);
          umma_ts(tm + (2 * g + 1) * 64, tm + 336 + g * 128 + 32, b32, id_s64, 1);
          tc_commit(&dbar[2 + g]);
        }
        tc_commit(&dbar[4]);
        tc_commit(&dbar[5]);
      }
      if (MODE == 6) {
        for (int g = 0; g < 2; ++g) {
          for (int kk = 0; kk < 4; ++kk) umma_ts(tm + g * 128, tm + 336 + g * 128 + kk * 8, b128 + kk * 2, id_s, kk);
          umma_ts(tm + g * 128, tm + 336 + g * 128 + 32, b32, id_s, 1);
          for (int kk = 0; kk < 8; ++kk) umma_ts(tm + 256 + g * 128, tm + g * 128 + kk * 8, vmn + kk * 32, id_o, 1);
        }
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (t1 - t0);
    stop = 1;
  } else if (NOISE >= 2 && warp >= 4 && warp < 12) {
    float a[16];
    for (int j = 0; j < 16; ++j) a[j] = -1.f * (j + threadIdx.x) / 1000.f;
    while (!stop) {
      if (NOISE == 2) {  // MUFU-heavy (softmax exps)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int j = 0; j < 16; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      } else if (NOISE == 3) {  // FMA-heavy
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], 0.999f, 0.001f);
      } else {  // large straight-line body: instruction-cache pressure
#pragma unroll
        for (int r = 0; r < 256; ++r)
#pragma unroll
          for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], 0.999f + r * 1e-6f, j * 1e-3f);
      }
    }
    if (a[0] == 12345.f) out[1] = 1;
  } else if (NOISE == 1 && warp >= 4 && warp < 12) {
    const uint32_t q = (warp & 3) * 32;
    const uint32_t col = ((warp - 4) >> 2) * 128;
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = j;
    while (!stop) {
      tmem_ld32(tm + (q << 16) + col, v);
      tmem_ld_wait();
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + (q << 16) + col + 64),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
          "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
          "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

int g_grid = 1;
template <int MODE, int NOISE>
double run(unsigned long long* d, int iters) {
  cudaFuncSetAttribute(k<MODE, NOISE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<MODE, NOISE><<<g_grid, 384, 65536>>>(d, iters);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
  return (double)h / iters;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int iters = 4096;
  for (int pass = 0; pass < 3; ++pass) {
  g_grid = pass ? 148 : 1;
  const int rnd = pass == 2;
  cudaMemcpyToSymbol(g_rand, &rnd, sizeof(int));
  printf("---- grid %d CTAs, %s operands\n", g_grid, rnd ? "random" : "zero");
  printf("%-40s %8.1f cycles/MMA\n", "S SS SW128 M128 N128", run<0, 0>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "S SS SW32 M128 N128", run<1, 0>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "PV TS V-MN-SW32 N80", run<2, 0>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "SS SW128 M128 N256", run<3, 0>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "S TS SW128 N128", run<4, 0>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "S TS SW32 N128", run<5, 0>(d, iters));
  printf("%-40s %8.1f cycles/block (26 MMAs)\n", "attention block mix", run<6, 0>(d, iters / 16));
  printf("%-40s %8.1f cycles/MMA\n", "S TS SW128 N64", run<7, 0>(d, iters));
  printf("%-40s %8.1f cycles/block (18 MMAs, ideal %.0f)\n", "KB64 block seq + commits", run<9, 0>(d, iters / 16), 2 * (4 * 60.3 + 5 * 45.6));
  printf("%-40s %8.1f cycles/block\n", "KB64 block seq + commits + fences", run<10, 0>(d, iters / 16));
  printf("%-40s %8.1f cycles/block\n", "KB64 seq + MUFU noise", run<9, 2>(d, iters / 16));
  printf("%-40s %8.1f cycles/block\n", "KB64 seq + FMA noise", run<9, 3>(d, iters / 16));
  printf("%-40s %8.1f cycles/block\n", "KB64 seq + icache noise", run<9, 4>(d, iters / 16));
  printf("%-40s %8.1f cycles/MMA\n", "S TS SW128 N128 + TMEM ld/st noise", run<4, 1>(d, iters));
  printf("%-40s %8.1f cycles/MMA\n", "PV TS N80 + TMEM ld/st noise", run<2, 1>(d, iters));
  printf("%-40s %8.1f cycles/block\n", "attention block mix + noise", run<6, 1>(d, iters / 16));
  }
  // sustained: all SMs, random operands, ~100x longer
  g_grid = 148;
  const int rnd = 1;
  cudaMemcpyToSymbol(g_rand, &rnd, sizeof(int));
  for (int rep = 0; rep < 3; ++rep)
    printf("%-40s %8.1f cycles/block\n", "SUSTAINED KB64 seq (148 CTAs, random)", run<9, 0>(d, iters * 8));
  for (int rep = 0; rep < 2; ++rep)
    printf("%-40s %8.1f cycles/MMA\n", "SUSTAINED SS N256 (148 CTAs, random)", run<3, 0>(d, iters * 100));
  return 0;
}
