// Persistent, warp-specialized bf16 GEMM for sm_100a: TMA -> smem ring ->
// tcgen05.mma (accumulator in TMEM, double-buffered) -> fused epilogue.
//
//   C[M,N] = A[M,K] * B[N,K]^T      (both operands K-major, nn.Linear layout)
//
// Roles (192 threads / CTA, 1 CTA per SM):
//   warp 0      : TMA producer (one elected lane)
//   warp 1      : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  : epilogue (TMEM -> regs -> bias/GELU/residual -> global)
// The epilogue of tile i overlaps the MMAs of tile i+1 (two TMEM accumulators).
#include "common.cuh"
#include "kernels.h"
#include "tmap.h"

namespace epd {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

EPD_DEVICE void store8(bf16* dst, const float* x) {
  uint4 v;
  v.x = pack_bf16x2(x[0], x[1]);
  v.y = pack_bf16x2(x[2], x[3]);
  v.z = pack_bf16x2(x[4], x[5]);
  v.w = pack_bf16x2(x[6], x[7]);
  *reinterpret_cast<uint4*>(dst) = v;
}
EPD_DEVICE void load8(const bf16* src, float* x) {
  uint4 v = *reinterpret_cast<const uint4*>(src);
  float2 a = unpack_bf16x2(v.x), b = unpack_bf16x2(v.y), c = unpack_bf16x2(v.z),
         d = unpack_bf16x2(v.w);
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
  x[4] = c.x; x[5] = c.y; x[6] = d.x; x[7] = d.y;
}

// Apply the fused epilogue to 32 consecutive columns [n, n+32) of one row.
EPD_DEVICE void epilogue_chunk(const EpiParams& ep, int row, int n, int N, const uint32_t (&v)[32]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int col = n + g * 8;
    if (col >= N) break;
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __uint_as_float(v[g * 8 + j]);
    if (ep.bias) {
      float b[8];
      load8(ep.bias + col, b);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] += b[j];
    }
    if (ep.act == ACT_GELU_TANH) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = gelu_tanh(x[j]);
    } else if (ep.act == ACT_GELU_ERF) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = gelu_erf(x[j]);
    }
    if (ep.resid || ep.resid_f) {
      if (ep.lscale) {
        float s[8];
        load8(ep.lscale + col, s);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] *= s[j];
      }
      float r[8];
      const size_t roff = (size_t)(row % ep.r_mod) * ep.ldr + col;
      if (ep.resid_f) {
        const float4 r0 = *reinterpret_cast<const float4*>(ep.resid_f + roff);
        const float4 r1 = *reinterpret_cast<const float4*>(ep.resid_f + roff + 4);
        r[0] = r0.x; r[1] = r0.y; r[2] = r0.z; r[3] = r0.w;
        r[4] = r1.x; r[5] = r1.y; r[6] = r1.z; r[7] = r1.w;
      } else {
        load8(ep.resid + roff, r);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] += r[j];
    }
    if (ep.mode == EPI_ROWS) {
      if (ep.out_f) {
        float* o = ep.out_f + (size_t)row * ep.ldo + col;
        *reinterpret_cast<float4*>(o) = make_float4(x[0], x[1], x[2], x[3]);
        *reinterpret_cast<float4*>(o + 4) = make_float4(x[4], x[5], x[6], x[7]);
      } else {
        store8(ep.out + (size_t)row * ep.ldo + col, x);
      }
    } else {
      const int s = col / ep.sec_cols;
      const int within = col - s * ep.sec_cols;
      const int h = within / ep.Dp;
      const int d = within - h * ep.Dp;
      const int b = row / ep.T;
      const int t = row - b * ep.T;
      const size_t bh = (size_t)b * ep.H + h;
      bf16* base = ep.sec_out[s];
      if (!ep.sec_trans[s]) {
        store8(base + (bh * ep.T + t) * ep.Dp + d, x);
      } else {
        bf16* p = base + (bh * ep.Dp + d) * ep.Tpad + t;
#pragma unroll
        for (int j = 0; j < 8; ++j) p[(size_t)j * ep.Tpad] = __float2bfloat16_rn(x[j]);
      }
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     int M, int N, int K, const EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + Cfg::STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int nk = (K + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / num_n) * kBM;
        const int n0 = (tile % num_n) * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, m0);
          tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * kBK, n0);
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t dtmem = tmem_base + as * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adesc = make_sdesc(a_addr + k * 32, 1024, 2);
            const uint64_t bdesc = make_sdesc(b_addr + k * 32, 1024, 2);
            umma_bf16(dtmem, adesc, bdesc, idesc, (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[as]);
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r_in_tile = q * 32 + lane;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const int m0 = (tile / num_n) * kBM;
      const int n0 = (tile % num_n) * BN;
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const int row = m0 + r_in_tile;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (n0 + c >= N) break;
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c, v);
        tmem_ld_wait();
        if (row < M) epilogue_chunk(ep, row, n0 + c, N, v);
      }
      tc_fence_before();
      mbar_arrive(&tempty[as]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN>
int launch(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
           const EpiParams& ep, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ta, tb;
  int rc = make_tmap_2d(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, kBK, kBM,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, kBK, BN,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  int grid = num_sms();
  if (tiles < grid) grid = tiles;
  gemm_bf16_kernel<BN><<<grid, 192, Cfg::SMEM, stream>>>(ta, tb, M, N, K, ep);
  return (int)cudaGetLastError();
}

}  // namespace

int gemm_bf16(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
              const EpiParams& ep, cudaStream_t stream, int bn_hint) {
  if (M <= 0 || N <= 0 || K <= 0) return 1001;
  if (N % 8 != 0 || (lda * 2) % 16 != 0 || (ldb * 2) % 16 != 0) return 1002;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return 1003;
  int bn = bn_hint;
  if (bn == 0) {
    // Pick the N tile that minimises the last-wave tail for this shape.
    const int sms = num_sms();
    double best = 1e30;
    const int cands[3] = {256, 192, 128};
    for (int i = 0; i < 3; ++i) {
      const int c = cands[i];
      const long tiles = (long)((M + kBM - 1) / kBM) * ((N + c - 1) / c);
      const long waves = (tiles + sms - 1) / sms;
      // cost ~ waves * per-tile time (~ c) with a mild penalty for narrow tiles
      const double cost = (double)waves * c * (c == 128 ? 1.12 : (c == 192 ? 1.03 : 1.0));
      if (cost < best) { best = cost; bn = c; }
    }
  }
  switch (bn) {
    case 256: return launch<256>(A, lda, B, ldb, M, N, K, ep, stream);
    case 192: return launch<192>(A, lda, B, ldb, M, N, K, ep, stream);
    case 128: return launch<128>(A, lda, B, ldb, M, N, K, ep, stream);
    default: return 1004;
  }
}

}  // namespace epd
