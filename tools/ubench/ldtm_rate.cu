// Micro-benchmark: TMEM load / store throughput per SM (tcgen05.ld / st 32x32b), as the
// attention softmax uses them (each warp reads 64 fp32 columns of its lane quarter, then
// writes 32 packed columns back).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_05460_b200/csrc ldtm_rate.cu -o ldtm_rate
#include <cstdio>
#include "common.cuh"
using namespace epd;

// MODE 0: ld x32 twice + wait | 1: + st x32 + wait (softmax pattern) | 2: st only | 3: ld x64 once
template <int MODE>
__global__ void k(unsigned long long* out, int iters, int nwarps) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t q = (warp & 3) * 32;
    const uint32_t col = ((warp >> 2) & 3) * 128;
    uint32_t v[64];
    for (int j = 0; j < 64; ++j) v[j] = j + threadIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
      if (MODE != 2) {
        if (MODE == 3) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
              "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%"
              "46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
                "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
                "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
                "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
                "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
              : "r"(tm + (q << 16) + col));
        } else {
          tmem_ld32(tm + (q << 16) + col, *reinterpret_cast<uint32_t(*)[32]>(v));
          tmem_ld32(tm + (q << 16) + col + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        }
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 64; ++j) acc += v[j];
      }
      if (MODE == 1 || MODE == 2) {
        for (int j = 0; j < 32; ++j) v[j] += acc;
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
    if (acc == 0x12345678u) out[1] = acc;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int MODE>
void run(unsigned long long* d, int nw, int grid) {
  const int iters = 4096;
  k<MODE><<<grid, 512>>>(d, iters, nw);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  const double cyc = (double)h / iters;
  const double ldb = MODE == 2 ? 0 : nw * 32.0 * 64 * 4, stb = (MODE == 1 || MODE == 2) ? nw * 32.0 * 32 * 4 : 0;
  printf("mode %d warps %2d grid %3d: %7.1f cyc/iter  ld %6.1f B/cyc  st %6.1f B/cyc\n", MODE, nw, grid, cyc,
         ldb / cyc, stb / cyc);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  for (int grid : {1, 148})
    for (int nw : {4, 8, 16}) {
      run<0>(d, nw, grid);
      run<3>(d, nw, grid);
      run<1>(d, nw, grid);
      run<2>(d, nw, grid);
    }
  return 0;
}
