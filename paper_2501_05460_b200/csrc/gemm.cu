// Persistent, warp-specialized bf16 GEMM for sm_100a: TMA -> smem ring ->
// tcgen05.mma (accumulator in TMEM, double-buffered) -> fused epilogue.
//
//   C[M,N] = A[M,K] * B[N,K]^T      (both operands K-major, nn.Linear layout)
//
// Roles (320 threads / CTA, 1 CTA per SM, persistent over output tiles):
//   warp 0      : TMA producer (one elected lane)
//   warp 1      : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9  : epilogue, two halves of 4 warps (one per TMEM lane quarter),
//                 each half owning half of the tile's columns: TMEM -> regs ->
//                 bias/GELU/layer-scale -> swizzled smem -> TMA store (or TMA
//                 reduce-add into the fp32 residual stream).
// The epilogue of tile i overlaps the MMAs of tile i+1 (two TMEM accumulators).
#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "tmap.h"

namespace epd {

namespace {

constexpr int kBM = 128;
// Clusters of 4 (two pairs multicasting B) halve B's L2->SM traffic, but only 33 such
// clusters are co-resident on a B200 (132 of 148 SMs); measured net 2-8 % slower than
// pairs on the encoder shapes, so the auto policy never picks them (policy 4 forces them).
#ifndef EPD_CL4_MIN_M
#define EPD_CL4_MIN_M (1 << 30)
#endif

constexpr int kBK = 64;

EPD_DEVICE void load8(const bf16* src, float* x) {
  uint4 v = *reinterpret_cast<const uint4*>(src);
  float2 a = unpack_bf16x2(v.x), b = unpack_bf16x2(v.y), c = unpack_bf16x2(v.z),
         d = unpack_bf16x2(v.w);
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
  x[4] = c.x; x[5] = c.y; x[6] = d.x; x[7] = d.y;
}

// Both GELU epilogues are relative-accurate on the negative tail, where 0.5 x (1 + t)
// with a hardware tanh (abs error ~5e-4) cancels: at x = -3 that form is off by several
// bf16 ulps. The FMA-pipe arithmetic runs on packed pairs (FFMA2 / FMUL2), two elements
// per instruction.
EPD_DEVICE float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\nmov.b64 rc, {%6,%7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0,%1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
EPD_DEVICE float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\n"
      "mul.rn.f32x2 rd, ra, rb;\nmov.b64 {%0,%1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
EPD_DEVICE float2 f2s(float v) { return make_float2(v, v); }
EPD_DEVICE float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

EPD_DEVICE float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The GELUs run over the NP packed pairs of an epilogue chunk stage by stage, so that the NP
// dependency chains interleave (per-pair calls left the compiler ~2 chains in flight and
// the epilogue warps, two per SM sub-partition, latency-bound: profiles/r02/ab.txt).
//
// GELU-tanh, 0.5 x (1 + tanh u) with u = k0 (x + k1 x^3), written as x * sigma(2u):
// e = 2^(-2 u(|x|) log2 e) and r = 1 / (1 + e) on the MUFU (ex2; one rcp per pair), then
// phi = r for x >= 0 and e r for x < 0.
template <int NP>
EPD_DEVICE void gelu_tanh_chunk(float* x) {
  float2 a[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float2 z = make_float2(fabsf(x[2 * p]), fabsf(x[2 * p + 1]));
    // -2 log2(e) k0 (z + k1 z^3) = z (C0 + C1 z^2)
    a[p] = f2mul(z, f2fma(f2mul(z, z), f2s(-0.10294324159622192f), f2s(-2.302208185195923f)));
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) a[p] = make_float2(ex2f(a[p].x), ex2f(a[p].y));  // e
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float2 y = f2fma(a[p], f2s(1.f), f2s(1.f));
    // both reciprocals from one MUFU op: 1/y0 = y1 / (y0 y1), 1/y1 = y0 / (y0 y1)
    const float2 r = f2mul(f2s(rcpf(y.x * y.y)), make_float2(y.y, y.x));
    const float2 er = f2mul(a[p], r);
    const float2 xv = make_float2(x[2 * p], x[2 * p + 1]);
    const float2 g = f2mul(xv, make_float2(xv.x >= 0.f ? r.x : er.x, xv.y >= 0.f ? r.y : er.y));
    x[2 * p] = g.x;
    x[2 * p + 1] = g.y;
  }
}
// GELU-erf, x Phi(x): Phi(-z) = 2^-F(z) for z = min(|x|, 8), F a degree-8 polynomial in
// v = z/4 - 1 (tools/fit_gelu.py: max rel err 8.5e-6 against x Phi(x) on [-8, 8]; 0.025 %
// of bf16 outputs round differently from the exact erf form, fp32 noise). Beyond |x| = 8
// the result is x (x > 0) or below 1e-14 in magnitude. The polynomial carries -F.
template <int NP>
EPD_DEVICE void gelu_erf_chunk(float* x) {
  float2 f[NP], v[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    v[p] = f2fma(make_float2(fminf(fabsf(x[2 * p]), 8.f), fminf(fabsf(x[2 * p + 1]), 8.f)), f2s(0.25f), f2s(-1.f));
    f[p] = f2fma(f2s(5.421509966e-03f), v[p], f2s(-2.080199681e-02f));
  }
  constexpr float c[7] = {4.194424301e-02f, -7.617540658e-02f, 1.449510306e-01f, -2.748279572e-01f,
                          -1.100269699e+01f, -2.438505554e+01f, -1.494647121e+01f};
#pragma unroll
  for (int k = 0; k < 7; ++k)
#pragma unroll
    for (int p = 0; p < NP; ++p) f[p] = f2fma(f[p], v[p], f2s(c[k]));
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float qx = ex2f(f[p].x), qy = ex2f(f[p].y);
    const float2 xv = make_float2(x[2 * p], x[2 * p + 1]);
    const float2 g = f2mul(xv, make_float2(xv.x >= 0.f ? 1.f - qx : qx, xv.y >= 0.f ? 1.f - qy : qy));
    x[2 * p] = g.x;
    x[2 * p + 1] = g.y;
  }
}

// Epilogue kinds (the output side of C = A B^T):
//   ROWS_BF16 : out bf16 row-major                 (TMA store, 64 B rows, SW64, 32-col chunks)
//   ROWS_F32  : out fp32 row-major                 (TMA store, 128 B rows, SW128, 32-col chunks)
//   ACC_F32   : out fp32 += result (residual stream, in place)  (TMA reduce-add, SW128)
//   HEADS     : per-head Q/K/V [bh][T][Dp] (SW32) or keys-major V^T [bh][Dp][Tpad] (no swizzle):
//               each 32-column chunk leaves as two 16-column 3-D TMA boxes; tiles that
//               straddle two images store from registers.
//   SWIGLU    : 64-column groups (gate 32 | up 32) -> 32 bf16 columns at n/2 (as ROWS_BF16)
enum EpiKind : int { EK_ROWS_BF16 = 0, EK_ROWS_F32 = 1, EK_ACC_F32 = 2, EK_HEADS = 3, EK_SWIGLU = 4 };

#ifndef EPD_GEMM_EXP
#define EPD_GEMM_EXP 0  // A/B experiments only (tools/build_variant.sh -DEPD_GEMM_EXP=n)
#endif

constexpr int kEpiStageBytes = 16384;  // per epilogue half: 128 rows x 128 B
#ifndef EPD_GEMM_BPREFETCH
#define EPD_GEMM_BPREFETCH 1  // producer fetches the first item's B tiles before the PDL wait
#endif
#ifndef EPD_EPI_PERWARP
#define EPD_EPI_PERWARP 1  // row kinds: one TMA box per warp (32 rows) instead of per 4-warp half
#endif
#ifndef EPD_GEMM_EPI_WARPS
#define EPD_GEMM_EPI_WARPS 8  // epilogue warps: 8 = two column halves x 4 lane quarters; 4 = one half
#endif
constexpr int kEpiWarps = EPD_GEMM_EPI_WARPS;
constexpr int kEpiHalves = kEpiWarps / 4;

template <int BN, int CG>
struct GemmCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = (BN / CG) * kBK * 2;  // with CTA pairs each CTA holds half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (227 * 1024 - 2 * kEpiStageBytes - 2048) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * kEpiStageBytes + 1024 + 256;
  static constexpr int THREADS = 64 + 32 * kEpiWarps;
};

EPD_DEVICE uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
EPD_DEVICE void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Map a local shared::cta address to the same offset in CTA `rank` of the cluster.
EPD_DEVICE uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Relaxed arrive on the pair leader's accumulator-empty barrier: it only hands TMEM back
// to the MMA warp, which the tcgen05 fences around the barrier order. A release.cluster
// arrive compiles to MEMBAR.ALL.GPU + ERRBAR, a stall of every epilogue warp once per tile
// that cost 3-8 % on every GEMM (profiles/r02/ab.txt).
EPD_DEVICE void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load issued by either CTA of a pair; the transaction bytes land on the leader's barrier.
EPD_DEVICE void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
EPD_DEVICE void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// As tma_load_2d_pair, delivered to every CTA in `mask` (same smem offset); each
// destination's transaction bytes land on its own pair leader's barrier.
EPD_DEVICE void tma_load_2d_pair_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                    uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu), "h"(mask)
      : "memory");
}
// Arrive on the same barrier offset in every CTA of `mask` once the pair's MMAs complete.
EPD_DEVICE void tc_commit_pair_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// Arrive on the same barrier offset in both CTAs of the pair once the pair's MMAs complete.
EPD_DEVICE void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
EPD_DEVICE void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
EPD_DEVICE void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

EPD_DEVICE void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EPD_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
EPD_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
EPD_DEVICE void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// tx bytes without an arrival (the arrival comes with the stage's other loads)
EPD_DEVICE void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
EPD_DEVICE int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
EPD_DEVICE void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
EPD_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
EPD_DEVICE void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
EPD_DEVICE void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
EPD_DEVICE void tma_store_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}

// Persistent tile schedule. Tiles are (M tile, N offset, width): full BN-wide tiles first
// (M-major, so consecutive tiles share A rows), then half-width tiles -- the last f_keep..
// full tiles split in two, so the final round holds only halves, and the ragged last N
// tile of every M row when its valid width fits in BN/2 (half-width MMAs, no wasted N).
// Decoded arithmetically by every role (no tile table: graph capture safe).
struct TileSched {
  int nf;       // full-width N tiles per M row
  int ragged;   // 1: one extra half-width N tile per M row at nf * BN
  int f_keep;   // full tiles kept whole (the rest of the num_m * nf are split)
  int f_total;  // num_m * nf
  int total;    // f_keep + 2 (f_total - f_keep) + num_m * ragged
  int num_m;    // M tiles
  int mfast;    // 1: consecutive full tiles walk down M (B, the larger operand, is read
                // from HBM once and reused from L2 by every M tile); 0: along N
};
struct TileAt {
  int mt, n0, w;
};
EPD_DEVICE TileAt tile_at(const TileSched& s, int t, int BN) {
  TileAt x;
  if (t < s.f_keep) {
    int nt;
    if (s.mfast) {
      nt = t / s.num_m;
      x.mt = t - nt * s.num_m;
    } else {
      x.mt = t / s.nf;
      nt = t - x.mt * s.nf;
    }
    x.n0 = nt * BN;
    x.w = BN;
    return x;
  }
  int k = t - s.f_keep;
  const int nsplit = s.f_total - s.f_keep;
  if (k < 2 * nsplit) {
    const int ft = s.f_keep + (k >> 1);
    int nt;
    if (s.mfast) {
      nt = ft / s.num_m;
      x.mt = ft - nt * s.num_m;
    } else {
      x.mt = ft / s.nf;
      nt = ft - x.mt * s.nf;
    }
    x.n0 = nt * BN + (k & 1) * (BN / 2);
  } else {
    x.mt = k - 2 * nsplit;
    x.n0 = s.nf * BN;
  }
  x.w = BN / 2;
  return x;
}

// CG = 1: one CTA per 128 x BN tile. CG = 2: a CTA pair (cluster of 2) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2 -- each CTA loads its 128 rows of A
// and half of B, the leader issues M=256 MMAs, both CTAs drain their own TMEM.
// CL = cluster size: 1 (single CTA), 2 (one CTA pair) or 4 (two CTA pairs stacked along M
// that share every B tile: pair 0 multicasts each half of B into both pairs, so the
// cluster streams B from L2 once for 512 rows -- the big GEMMs are L2-bandwidth bound).
template <int BN, int KIND, int CG, int CL>
__global__ void __launch_bounds__(GemmCfg<BN, CG>::THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmBh,
                     const __grid_constant__ CUtensorMap tmO0, const __grid_constant__ CUtensorMap tmO1,
                     const __grid_constant__ CUtensorMap tmO2, int M, int N, int K, const EpiParams ep,
                     const TileSched sched) {
  using Cfg = GemmCfg<BN, CG>;
  constexpr bool kPerWarpStore = EPD_EPI_PERWARP && KIND != EK_HEADS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* sEpi = sB + Cfg::STAGES * Cfg::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + 2 * kEpiStageBytes);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  static_assert(CL == CG || (CL == 4 && CG == 2), "cluster shape");
  const uint32_t crank_full = CL > 1 ? cluster_rank() : 0;  // CTA rank in the cluster
  const uint32_t crank = crank_full & 1;                     // rank within the CTA pair
  const uint32_t pair = crank_full >> 1;
  const int pid = blockIdx.x / CL;     // cluster index
  const int npid = gridDim.x / CL;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL == 4 ? 2 : 1);  // one MMA commit per pair reading the stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);  // one arrive per epilogue warp of every CTA in the pair
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmBh);
  }
  if (warp == 1) {
    if (CG == 2) tmem_alloc_pair(tmem_holder, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if (CL > 1) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();
  // A, the residual stream and the outputs belong to the previous kernels; the producer
  // waits only after it has started fetching the first item's weights (B), which no kernel
  // writes -- with programmatic dependent launch that fetch overlaps the previous kernel's tail
  if (warp != 0 || !EPD_GEMM_BPREFETCH) pdl_wait();

  const int nk = (K + kBK - 1) / kBK;
  // split-K (fp32 reduce-add only): work item = (tile, split), the splits of a tile adjacent
  const int nsplit = (KIND == EK_ACC_F32 && ep.ksplit > 1) ? ep.ksplit : 1;
  const int num_tiles = sched.total * nsplit;

  if (warp == 0) {
    // TMA producer: the whole warp walks the schedule (uniform operands), one elected lane issues
    int stage = 0;
    uint32_t phase = 0;
    int pre = 0;  // k-blocks of this CTA's first item whose B tiles were fetched before the wait
#if EPD_GEMM_BPREFETCH
    if (CL <= 2 && pid < num_tiles) {
      const int tile = pid / nsplit, sp = pid - tile * nsplit;
      const int kb_lo = sp * nk / nsplit, kb_hi = (sp + 1) * nk / nsplit;
      const TileAt x = tile_at(sched, tile, BN);
      const int n0 = x.n0 + crank * (x.w / CG);
      const bool hw = x.w != BN;
      const CUtensorMap* tb = hw ? &tmBh : &tmB;
      const uint32_t b_bytes = hw ? Cfg::B_BYTES / 2 : Cfg::B_BYTES;
      pre = kb_hi - kb_lo < Cfg::STAGES ? kb_hi - kb_lo : Cfg::STAGES;
      for (int i = 0; i < pre; ++i) {  // fresh stages: no empty wait
        if (elect_one()) {
          if (CG == 1) {
            mbar_expect_tx(&full[i], b_bytes);
            tma_load_2d(sB + i * Cfg::B_BYTES, tb, &full[i], (kb_lo + i) * kBK, n0);
          } else {
            if (crank == 0) mbar_expect_tx(&full[i], 2 * b_bytes);
            tma_load_2d_pair(sB + i * Cfg::B_BYTES, tb, &full[i], (kb_lo + i) * kBK, n0);
          }
        }
        __syncwarp();
      }
    }
    pdl_wait();
#endif
    bool first = true;
    for (int item = pid; item < num_tiles; item += npid, first = false) {
      const int tile = item / nsplit, sp = item - tile * nsplit;
      const int kb_lo = sp * nk / nsplit, kb_hi = (sp + 1) * nk / nsplit;
      const TileAt x = tile_at(sched, tile, BN);
      const int m0 = x.mt * (kBM * CL) + crank_full * kBM;
      // each CTA of a pair holds half of the tile's B rows; a half-width tile loads only
      // the first half of each CTA's box (tmBh), which is all its MMAs read
      const int n0 = x.n0 + crank * (x.w / CG);
      const bool hw = x.w != BN;
      const CUtensorMap* tb = hw ? &tmBh : &tmB;
      const uint32_t stage_bytes = Cfg::A_BYTES + (hw ? Cfg::B_BYTES / 2 : Cfg::B_BYTES);
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        const bool b_done = first && kb - kb_lo < pre;  // B already in flight (prefetch)
        const uint32_t bytes = b_done ? (uint32_t)Cfg::A_BYTES : stage_bytes;
#if EPD_GEMM_EXP == 1  // experiment: no operand loads (MMA + epilogue alone)
        if (elect_one() && crank == 0) mbar_arrive(&full[stage]);
        if (false) {
#else
        if (elect_one()) {
#endif
          if (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, m0);
            if (!b_done) tma_load_2d(sB + stage * Cfg::B_BYTES, tb, &full[stage], kb * kBK, n0);
          } else {
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
            tma_load_2d_pair(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, m0);
            if (b_done) {
            } else if (CL == 2)
              tma_load_2d_pair(sB + stage * Cfg::B_BYTES, tb, &full[stage], kb * kBK, n0);
            else if (pair == 0)  // this half of B, for both pairs
              tma_load_2d_pair_mc(sB + stage * Cfg::B_BYTES, tb, &full[stage], kb * kBK, n0,
                                  (uint16_t)((1u << crank) | (1u << (crank + 2))));
          }
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (crank == 0) {
      // MMA issuer: whole warp, elected lane issues (see elect_one)
      constexpr uint32_t idesc_full = make_idesc_bf16(kBM * CG, BN);
      constexpr uint32_t idesc_half = make_idesc_bf16(kBM * CG, BN / 2);
      const uint64_t a0 = make_sdesc(smem_u32(sA), 1024, 2);
      const uint64_t b0 = make_sdesc(smem_u32(sB), 1024, 2);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int item = pid; item < num_tiles; item += npid, ++local) {
        const int tile = item / nsplit, sp = item - tile * nsplit;
        const int kb_lo = sp * nk / nsplit, kb_hi = (sp + 1) * nk / nsplit;
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        const uint32_t idesc = tile_at(sched, tile, BN).w == BN ? idesc_full : idesc_half;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t dtmem = tmem_base + as * BN;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ao = a0 + (uint64_t)((stage * Cfg::A_BYTES) >> 4);
          const uint64_t bo = b0 + (uint64_t)((stage * Cfg::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < (EPD_GEMM_EXP == 2 ? 0 : kBK / 16); ++k) {  // EXP 2: no MMAs
              if (CG == 2) umma_bf16_pair(dtmem, ao + 2 * k, bo + 2 * k, idesc, kb != kb_lo || k != 0);
              else umma_bf16(dtmem, ao + 2 * k, bo + 2 * k, idesc, kb != kb_lo || k != 0);
            }
            if (CL == 4) tc_commit_pair_mask(&empty[stage], 0xF);  // the stage is free in all 4 CTAs
            else if (CG == 2) tc_commit_pair(&empty[stage]);
            else tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if (CL == 4) tc_commit_pair_mask(&tfull[as], (uint16_t)(3u << (2 * pair)));
          else if (CG == 2) tc_commit_pair(&tfull[as]);
          else tc_commit(&tfull[as]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: 8 warps = 2 halves x 4 TMEM lane quarters
    const int half = kEpiHalves == 2 ? (warp - 2) >> 2 : 0;
    const int q = warp & 3;
    const int r = q * 32 + lane;  // row within the tile (TMEM lane)
    const bool leader = ((warp - 2) & 3) == 0 && lane == 0;
    uint8_t* stg = sEpi + half * kEpiStageBytes;
    const int bar_id = 1 + half;
    const uint32_t tempty_leader = mapa_rank(smem_u32(&tempty[0]), crank_full & ~1u);  // pair leader
    int local = 0;
    for (int item = pid; item < num_tiles; item += npid, ++local) {
      const int tile = item / nsplit, sp = item - tile * nsplit;
      const bf16* bias_p = sp == 0 ? ep.bias : nullptr;  // the first split adds the bias
      // split-K: this warp's slab of the tile is reduce-added in split order; the counter
      // holds the number of splits done (reset to 0 by the last one, so graph replays start clean)
      int* slab_flag = nsplit > 1 ? ep.split_flags + (size_t)tile * (kEpiWarps * CL) + crank_full * kEpiWarps + (warp - 2)
                                  : nullptr;
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const TileAt x = tile_at(sched, tile, BN);
      const int m0 = x.mt * (kBM * CL) + crank_full * kBM;
      const int n0 = x.n0;
      const int hw = x.w / kEpiHalves;  // columns per epilogue half (a multiple of 32)
      const int row = m0 + r;
      // Heads bookkeeping, once per tile-half (no divisions inside the chunk loop):
      // section / head / head-dim of this half's first column, image and token of m0.
      int hsec = 0, hh = 0, hd = 0, img0 = 0, tok0 = 0;
      bool straddle = false;
      if (KIND == EK_HEADS) {
        const int nn = n0 + half * hw;
        hsec = nn / ep.sec_cols;
        const int within = nn - hsec * ep.sec_cols;
        hh = within / ep.Dp;
        hd = within - hh * ep.Dp;
        img0 = m0 / ep.T;
        tok0 = m0 - img0 * ep.T;
        // a tile that straddles two images (T % 128 != 0) cannot be one TMA box
        straddle = tok0 + kBM > ep.T;
      }
      // Per-column epilogue vectors (bias, layer scale) of the next 32-column chunk are loaded
      // one chunk ahead, so their global-load latency overlaps the accumulator wait and the
      // current chunk's arithmetic instead of stalling it.
      uint4 bias_nx[4], ls_nx[4];
      auto prefetch_vec = [&](int n) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int col = n + g * 8;
          const bool ok = KIND != EK_SWIGLU && col < N;
          bias_nx[g] = ok && bias_p ? *reinterpret_cast<const uint4*>(bias_p + col) : make_uint4(0, 0, 0, 0);
          ls_nx[g] = ok && ep.lscale ? *reinterpret_cast<const uint4*>(ep.lscale + col) : make_uint4(0, 0, 0, 0);
        }
      };
      prefetch_vec(n0 + half * hw);
      if (nsplit > 1 && sp > 0) {  // the previous split's adds into this slab come first
        if (lane == 0) {
          while (ld_acquire_gpu(slab_flag) < sp) __nanosleep(64);
          fence_proxy_async_global();
        }
        __syncwarp();
      }
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int c = half * hw; c < (EPD_GEMM_EXP == 3 ? 0 : (half + 1) * hw);  // EXP 3: no epilogue
           c += (KIND == EK_SWIGLU ? 64 : 32)) {
        const int n = n0 + c;
        if (n >= N) break;  // warp-uniform
        uint4 bias_cur[4], ls_cur[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          bias_cur[g] = bias_nx[g];
          ls_cur[g] = ls_nx[g];
        }
        if (KIND != EK_SWIGLU && c + 32 < (half + 1) * hw) prefetch_vec(n + 32);
        float x[32];
        {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(v[j]);
        }
        if (KIND == EK_SWIGLU) {
          // x = gate columns [n, n+32), u = up columns [n+32, n+64) of this 64-column group
          uint32_t u[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c + 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float bg[8] = {0, 0, 0, 0, 0, 0, 0, 0}, bu[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (ep.bias) {
              load8(ep.bias + n + g * 8, bg);
              load8(ep.bias + n + 32 + g * 8, bu);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float a = x[g * 8 + j] + bg[j];
              x[g * 8 + j] = a / (1.f + __expf(-a)) * (__uint_as_float(u[g * 8 + j]) + bu[j]);
            }
          }
        }
#pragma unroll
        for (int g = 0; g < 4 && KIND != EK_SWIGLU; ++g) {
          const int col = n + g * 8;
          float* xg = x + g * 8;
          if (col < N) {
            if (bias_p) {
              const uint4 bv = bias_cur[g];
              const float2 b0 = unpack_bf16x2(bv.x), b1 = unpack_bf16x2(bv.y), b2 = unpack_bf16x2(bv.z),
                           b3 = unpack_bf16x2(bv.w);
              const float2 bb[4] = {b0, b1, b2, b3};
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // packed adds (FFMA2 with 1)
                const float2 v = f2fma(make_float2(xg[2 * j], xg[2 * j + 1]), f2s(1.f), bb[j]);
                xg[2 * j] = v.x;
                xg[2 * j + 1] = v.y;
              }
            }
          }
        }
        if (KIND != EK_SWIGLU) {
          if (ep.act == ACT_GELU_TANH) gelu_tanh_chunk<16>(x);
          else if (ep.act == ACT_GELU_ERF) gelu_erf_chunk<16>(x);
        }
#pragma unroll
        for (int g = 0; g < 4 && KIND != EK_SWIGLU; ++g) {
          const int col = n + g * 8;
          float* xg = x + g * 8;
          if (col < N) {
            if (ep.lscale) {
              const uint4 sv = ls_cur[g];
              const float2 s0 = unpack_bf16x2(sv.x), s1 = unpack_bf16x2(sv.y), s2 = unpack_bf16x2(sv.z),
                           s3 = unpack_bf16x2(sv.w);
              xg[0] *= s0.x; xg[1] *= s0.y; xg[2] *= s1.x; xg[3] *= s1.y;
              xg[4] *= s2.x; xg[5] *= s2.y; xg[6] *= s3.x; xg[7] *= s3.y;
            }
            if (KIND != EK_ACC_F32 && ep.resid && row < M) {  // generic (direct-load) residual
              float rr[8];
              load8(ep.resid + (size_t)(row % ep.r_mod) * ep.ldr + col, rr);
#pragma unroll
              for (int j = 0; j < 8; ++j) xg[j] += rr[j];
            }
          }
        }
        // HEADS: the 32 columns are two 16-wide head-dim pieces (Dp % 16 == 0), each with its
        // own (section, head, dim) -- advanced incrementally -- and its own 4 KB staging slot.
        int psec[2] = {0, 0}, ph[2] = {0, 0}, pd[2] = {0, 0};
        bool pon[2] = {false, false}, pdirect[2] = {false, false};
        if (KIND == EK_HEADS) {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            pon[sub] = n + sub * 16 < N;
            psec[sub] = hsec; ph[sub] = hh; pd[sub] = hd;
            if ((hd += 16) == ep.Dp) {
              hd = 0;
              if (++hh == ep.H) { hh = 0; ++hsec; }
            }
            const int trans = psec[sub] == 0 ? ep.sec_trans[0] : (psec[sub] == 1 ? ep.sec_trans[1] : ep.sec_trans[2]);
            // a keys-major V^T piece must start at a 16-byte aligned token offset for TMA
            pdirect[sub] = straddle || ((tok0 & 7) && trans);
            if (pon[sub] && pdirect[sub] && row < M) {
              const int bimg = row / ep.T;
              const int t = row - bimg * ep.T;
              const size_t bh = (size_t)bimg * ep.H + ph[sub];
              bf16* base = psec[sub] == 0 ? ep.sec_out[0] : (psec[sub] == 1 ? ep.sec_out[1] : ep.sec_out[2]);
              const float* xs = x + sub * 16;
              if (!trans) {
                bf16* pp = base + (bh * ep.T + t) * ep.Dp + pd[sub];
#pragma unroll
                for (int j = 0; j < 2; ++j)
                  *reinterpret_cast<uint4*>(pp + 8 * j) =
                      make_uint4(pack_bf16x2(xs[8 * j + 0], xs[8 * j + 1]), pack_bf16x2(xs[8 * j + 2], xs[8 * j + 3]),
                                 pack_bf16x2(xs[8 * j + 4], xs[8 * j + 5]), pack_bf16x2(xs[8 * j + 6], xs[8 * j + 7]));
              } else {
                bf16* pp = base + (bh * ep.Dp + pd[sub]) * ep.Tpad + t;
#pragma unroll
                for (int j = 0; j < 16; ++j) pp[(size_t)j * ep.Tpad] = __float2bfloat16_rn(xs[j]);
              }
            }
          }
          if (!(pon[0] && !pdirect[0]) && !(pon[1] && !pdirect[1])) continue;  // nothing staged
        }
        // the previous TMA store(s) must have finished reading the staging buffer
        // (double-buffering the bf16 chunks measured neutral)
        uint8_t* sbuf = stg;
        if (kPerWarpStore) {  // each warp waits only for its own previous store
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        } else {
          if (leader) bulk_wait_read0();
          named_bar(bar_id, 128);
        }
        if (KIND == EK_ROWS_BF16 || KIND == EK_SWIGLU) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int phys = j ^ ((r >> 1) & 3);
            *reinterpret_cast<uint4*>(sbuf + r * 64 + phys * 16) =
                make_uint4(pack_bf16x2(x[8 * j + 0], x[8 * j + 1]), pack_bf16x2(x[8 * j + 2], x[8 * j + 3]),
                           pack_bf16x2(x[8 * j + 4], x[8 * j + 5]), pack_bf16x2(x[8 * j + 6], x[8 * j + 7]));
          }
        } else if (KIND == EK_ROWS_F32 || KIND == EK_ACC_F32) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int phys = j ^ (r & 7);
            *reinterpret_cast<float4*>(stg + r * 128 + phys * 16) =
                make_float4(x[4 * j + 0], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
          }
        } else {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            if (!pon[sub] || pdirect[sub]) continue;
            uint8_t* slot = stg + sub * 4096;
            const float* xs = x + sub * 16;
            const int trans = psec[sub] == 0 ? ep.sec_trans[0] : (psec[sub] == 1 ? ep.sec_trans[1] : ep.sec_trans[2]);
            if (!trans) {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int phys = j ^ ((r >> 2) & 1);
                *reinterpret_cast<uint4*>(slot + r * 32 + phys * 16) =
                    make_uint4(pack_bf16x2(xs[8 * j + 0], xs[8 * j + 1]), pack_bf16x2(xs[8 * j + 2], xs[8 * j + 3]),
                               pack_bf16x2(xs[8 * j + 4], xs[8 * j + 5]), pack_bf16x2(xs[8 * j + 6], xs[8 * j + 7]));
              }
            } else {
              bf16* t16 = reinterpret_cast<bf16*>(slot);
#pragma unroll
              for (int j = 0; j < 16; ++j) t16[j * 128 + r] = __float2bfloat16_rn(xs[j]);
            }
          }
        }
        fence_proxy_async_smem();
        if (kPerWarpStore) {
          // the warp's 32 rows leave as their own TMA box (no cross-warp barrier per chunk)
          __syncwarp();
          if (lane == 0 && m0 + q * 32 < M) {
            constexpr int slab = (KIND == EK_ROWS_F32 || KIND == EK_ACC_F32) ? 4096 : 2048;
            uint8_t* wb = stg + q * slab;
            if (KIND == EK_ROWS_BF16 || KIND == EK_ROWS_F32) tma_store_2d(&tmO0, wb, n, m0 + q * 32);
            else if (KIND == EK_SWIGLU) tma_store_2d(&tmO0, wb, n / 2, m0 + q * 32);
            else tma_reduce_add_2d(&tmO0, wb, n, m0 + q * 32);
            bulk_commit();
          }
          continue;
        }
        named_bar(bar_id, 128);
        if (leader) {
          if (KIND == EK_ROWS_BF16 || KIND == EK_ROWS_F32) {
            tma_store_2d(&tmO0, sbuf, n, m0);
          } else if (KIND == EK_SWIGLU) {
            tma_store_2d(&tmO0, sbuf, n / 2, m0);
          } else if (KIND == EK_ACC_F32) {
            tma_reduce_add_2d(&tmO0, stg, n, m0);
          } else {
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              if (!pon[sub] || pdirect[sub]) continue;
              uint8_t* slot = stg + sub * 4096;
              const int trans = psec[sub] == 0 ? ep.sec_trans[0] : (psec[sub] == 1 ? ep.sec_trans[1] : ep.sec_trans[2]);
              const int bh = img0 * ep.H + ph[sub];
              const int c0 = trans ? tok0 : pd[sub], c1 = trans ? pd[sub] : tok0;
              if (psec[sub] == 0) tma_store_3d(&tmO0, slot, c0, c1, bh);
              else if (psec[sub] == 1) tma_store_3d(&tmO1, slot, c0, c1, bh);
              else tma_store_3d(&tmO2, slot, c0, c1, bh);
            }
          }
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(tempty_leader + as * 8);
        else mbar_arrive(&tempty[as]);
      }
      if (nsplit > 1) {
        if (lane == 0) {
          bulk_wait_all0();  // this warp's reduce-adds of the item are complete in memory
          fence_proxy_async_global();
          st_release_gpu(slab_flag, sp + 1 == nsplit ? 0 : sp + 1);
        }
        __syncwarp();
      }
    }
    if (kPerWarpStore ? lane == 0 : leader) bulk_wait_all0();
  }

  tc_fence_before();
  if (CL > 1) cluster_sync_all(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// Persistent units that can be co-resident: SMs / CL, capped by how many clusters of CL
// CTAs (227 KB of smem each) the GPCs can host at once -- a persistent grid larger than
// that runs its last clusters as a second wave.
int cluster_units(int CL) {
  static int cache[5] = {0, 0, 0, 0, 0};
  if (cache[CL]) return cache[CL];
  int units = num_sms() / CL;
  if (CL > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(units * CL);
    cfg.blockDim = dim3(GemmCfg<256, 2>::THREADS);
    cfg.dynamicSmemBytes = GemmCfg<256, 2>::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const void* k = CL == 4 ? (const void*)gemm_bf16_kernel<256, EK_ROWS_BF16, 2, 4>
                            : (const void*)gemm_bf16_kernel<256, EK_ROWS_BF16, 2, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<256, 2>::SMEM);
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) == cudaSuccess && n > 0 && n < units) units = n;
    cudaGetLastError();
  }
  cache[CL] = units;
  return units;
}

// Tile schedule for `units` = SMs / CL persistent clusters (a tile spans kBM * CL rows).
// Half tiles need BN/4 to be a multiple of 32 (the epilogue's chunk width), i.e. BN in
// {128, 256}.
TileSched make_sched(int M, int N, int BN, int CL, bool halves_ok, int units) {
  const int num_m = (M + kBM * CL - 1) / (kBM * CL);
  const int num_n = (N + BN - 1) / BN;
  const bool halves = halves_ok && (BN == 256 || BN == 128);
  TileSched t;
  t.ragged = (halves && N - (num_n - 1) * BN <= BN / 2) ? 1 : 0;
  t.nf = num_n - t.ragged;
  t.f_total = num_m * t.nf;
  t.f_keep = t.f_total;
  if (halves) {
    const int w2 = 2 * t.f_total + num_m * t.ragged;  // work in half tiles
    const int r2 = (w2 + units - 1) / units;           // rounds, in half-tile units
    const int keep = units * (r2 / 2);                 // whole rounds of full tiles
    if (keep < t.f_keep) t.f_keep = keep;
  }
  t.total = t.f_keep + 2 * (t.f_total - t.f_keep) + num_m * t.ragged;
  t.num_m = num_m;
  // Walk down M when B (N x K) outweighs A (M x K): one pass over the weights from HBM,
  // shared through L2 by the few M tiles. (Walking N, a prefill's 662-row activations
  // against the 271 MB gate/up weight re-read the weights from HBM once per M tile.)
  t.mfast = (N > M && num_m > 1) ? 1 : 0;
  static const int force = [] {
    const char* e = getenv("EPD_GEMM_MFAST");  // A/B override: 0 / 1
    return e ? atoi(e) : -1;
  }();
  if (force >= 0) t.mfast = force;
  return t;
}

// Rounds (in full-tile time) the schedule takes on the persistent grid.
double sched_rounds(const TileSched& t, int units) {
  const int halves = t.total - t.f_keep;
  const int r_full = (t.f_keep + units - 1) / units;
  const int r_half = (halves + units - 1) / units;
  return r_full + 0.5 * r_half;
}

template <int BN, int KIND, int CL>
int launch(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K, const EpiParams& ep,
           cudaStream_t stream) {
  constexpr int CG = CL == 1 ? 1 : 2;
  using Cfg = GemmCfg<BN, CG>;
  CUtensorMap ta, tb, tbh, t0, t1, t2;
  int rc = make_tmap_2d(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, kBK, kBM,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc)
    rc = make_tmap_2d(&tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, kBK, BN / CG, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc)  // half-width tiles (BN in {128, 256}; otherwise never used)
    rc = make_tmap_2d(&tbh, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, kBK, BN / CG / 2,
                      CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  if (KIND == EK_ROWS_BF16 || KIND == EK_SWIGLU) {
    rc = make_tmap_2d(&t0, ep.out, (uint64_t)(KIND == EK_SWIGLU ? N / 2 : N), (uint64_t)M, (uint64_t)ep.ldo * 2,
                      32, EPD_EPI_PERWARP ? 32 : kBM, CU_TENSOR_MAP_SWIZZLE_64B);
    t1 = t2 = t0;
  } else if (KIND == EK_ROWS_F32 || KIND == EK_ACC_F32) {
    rc = make_tmap_2d_f32(&t0, ep.out_f, (uint64_t)N, (uint64_t)M, (uint64_t)ep.ldo * 4, 32,
                          EPD_EPI_PERWARP ? 32 : kBM, CU_TENSOR_MAP_SWIZZLE_128B);
    t1 = t2 = t0;
  } else {
    const uint64_t nb = (uint64_t)(M + ep.T - 1) / ep.T;
    CUtensorMap* maps[3] = {&t0, &t1, &t2};
    for (int s = 0; s < 3 && !rc; ++s) {
      if (!ep.sec_out[s] || (uint64_t)s * ep.sec_cols >= (uint64_t)N) {
        *maps[s] = ta;
        continue;
      }
      const uint64_t Dp = ep.Dp;
      if (!ep.sec_trans[s])
        rc = make_tmap_3d(maps[s], ep.sec_out[s], Dp, ep.T, nb * ep.H, Dp * 2, Dp * 2 * ep.T, 16, kBM, 1,
                          CU_TENSOR_MAP_SWIZZLE_32B);
      else
        rc = make_tmap_3d(maps[s], ep.sec_out[s], ep.T, Dp, nb * ep.H, (uint64_t)ep.Tpad * 2,
                          (uint64_t)ep.Tpad * 2 * Dp, kBM, 16, 1, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
  }
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_kernel<BN, KIND, CG, CL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  const int cap = cluster_units(CL);
  const TileSched sched = make_sched(M, N, BN, CL, KIND != EK_HEADS, cap);
  int units = cap;
  const int items = sched.total * (KIND == EK_ACC_F32 && ep.ksplit > 1 ? ep.ksplit : 1);
  if (items < units) units = items;
  const int rc2 = launch_kernel(gemm_bf16_kernel<BN, KIND, CG, CL>, dim3(units * CL), dim3(Cfg::THREADS),
                                Cfg::SMEM, stream, CL, ta, tb, tbh, t0, t1, t2, M, N, K, ep, sched);
  if (rc2) return rc2;
  return (int)cudaGetLastError();
}

template <int BN, int CL>
int launch_kind(int kind, const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
                const EpiParams& ep, cudaStream_t stream) {
  switch (kind) {
    case EK_ROWS_BF16: return launch<BN, EK_ROWS_BF16, CL>(A, lda, B, ldb, M, N, K, ep, stream);
    case EK_ROWS_F32: return launch<BN, EK_ROWS_F32, CL>(A, lda, B, ldb, M, N, K, ep, stream);
    case EK_ACC_F32: return launch<BN, EK_ACC_F32, CL>(A, lda, B, ldb, M, N, K, ep, stream);
    case EK_SWIGLU: return launch<BN, EK_SWIGLU, CL>(A, lda, B, ldb, M, N, K, ep, stream);
    default: return launch<BN, EK_HEADS, CL>(A, lda, B, ldb, M, N, K, ep, stream);
  }
}

int g_cta_group_policy = 0;  // 0 auto; else the cluster size: 1 single CTAs, 2 CTA pairs, 4 pairs sharing B

}  // namespace

void set_gemm_cta_group(int policy) { g_cta_group_policy = policy; }

// Zeroed split-K progress counters (grown, never freed: queued kernels may still use an old
// buffer). Not allocated during stream capture -- the GEMM then runs unsplit. One buffer per
// device: split launches must not run concurrently on two streams of the same device.
static int* split_flags(int need, cudaStream_t stream) {
  static int* buf[16] = {};
  static int cap[16] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  if (buf[dev] && need <= cap[dev]) return buf[dev];
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) return nullptr;
  const int n = need < (1 << 16) ? (1 << 16) : need;
  int* p = nullptr;
  if (cudaMalloc(&p, (size_t)n * sizeof(int)) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  if (cudaMemsetAsync(p, 0, (size_t)n * sizeof(int), stream) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  buf[dev] = p;
  cap[dev] = n;
  return p;
}

int gemm_bf16(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
              const EpiParams& ep, cudaStream_t stream, int bn_hint) {
  if (M <= 0 || N <= 0 || K <= 0) return 1001;
  if (N % 8 != 0 || (lda * 2) % 16 != 0 || (ldb * 2) % 16 != 0) return 1002;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return 1003;
  // Cluster size: CTA pairs (256-row tiles, each SM streaming half of B) once there are two
  // 128-row M tiles; single CTAs for M <= 256 (LM head, resampler query precompute);
  // two pairs multicasting B (512-row tiles) when M fills them. All variants compute the
  // same K-ordered sums, so the choice never changes results.
  int cl = g_cta_group_policy ? g_cta_group_policy : (M > 256 ? (M >= EPD_CL4_MIN_M ? 4 : 2) : 1);
  if (cl != 1 && cl != 2 && cl != 4) return 1001;
  if (ep.mode == EPI_HEADS && cl == 4) cl = 2;
  int bn = bn_hint, nsplit = 1;
  // split-K only where the caller allows it (fp32 reduce-add, per-warp stores)
  const bool can_split = ep.max_split > 1 && ep.out_f && ep.resid_f && ep.mode != EPI_HEADS && EPD_EPI_PERWARP;
  if (bn == 0 || can_split) {
    // Wide tiles amortise the epilogue and operand traffic best; step down only when the
    // schedule's rounds (half tiles included) favour a narrower tile. With split-K allowed,
    // S splits of every tile run as separate work items: rounds ceil(S T / U) of 1/S the
    // K each, plus ~8 % per extra split for the ordered epilogue chain.
    double best = 1e30;
    const int cands[3] = {256, 192, 128};
    const int nkb = (K + kBK - 1) / kBK;
    for (int i = 0; i < 3; ++i) {
      const int c = cands[i];
      if (bn_hint && c != bn_hint) continue;
      if (cl > 1 && c == 128) continue;
      const int u = cluster_units(cl);
      const TileSched t = make_sched(M, N, c, cl, ep.mode != EPI_HEADS, u);
      const double eff = c == 128 ? 1.35 : (c == 192 ? 1.12 : 1.0);
      for (int sp = 1; sp <= (can_split ? ep.max_split : 1); ++sp) {
        // >= 64 k-blocks (4096 of K) per split: below that the ordered fp32 reduce-add chain
        // costs more than the idle pairs (tools/split_ab.py: the 662 x 3584 x 3584 O
        // projection 26 -> 37 us at 3 splits; the 18944-deep down projection 97 -> 87 us)
        if (sp > 1 && nkb / sp < 64) break;
        const double rounds = sp == 1 ? sched_rounds(t, u) : (double)((t.total * sp + u - 1) / u) / sp;
        const double cost = rounds * c * eff * (1.0 + 0.08 * (sp - 1));
        if (cost < best - 1e-9) { best = cost; bn = c; nsplit = sp; }
      }
    }
  }
  if (ep.act == ACT_SWIGLU) {
    // every epilogue half must hold whole 64-column gate|up groups: BN = 256 (halves 128/64)
    if (bn_hint && bn_hint != 256) return 1004;
    bn = 256;
  }
  if (cl > 1 && bn == 128) cl = 1;
  int kind;
  if (ep.mode == EPI_HEADS) {
    if (ep.Dp % 16 || ep.sec_cols % ep.Dp || ep.T <= 0) return 1005;
    for (int s = 0; s < 3; ++s)
      if (ep.sec_out[s] && ep.sec_trans[s] && (ep.Tpad % 8 || ep.Tpad < ep.T)) return 1005;
    kind = EK_HEADS;
  } else if (ep.out_f) {
    if (ep.resid_f && ep.resid_f != ep.out_f) return 1005;  // fp32 residual only in place
    if (ep.resid_f && ep.resid) return 1005;
    kind = ep.resid_f ? EK_ACC_F32 : EK_ROWS_F32;
    if (ep.ldo % 4) return 1002;
  } else if (ep.act == ACT_SWIGLU) {
    if (!ep.out || ep.resid || ep.resid_f || ep.lscale || N % 64) return 1005;
    kind = EK_SWIGLU;
  } else {
    if (!ep.out || ep.resid_f) return 1005;
    kind = EK_ROWS_BF16;
  }
  static const int force_split = [] {
    const char* e = getenv("EPD_GEMM_SPLIT");  // A/B override of the split count
    return e ? atoi(e) : 0;
  }();
  if (can_split && force_split > 0) nsplit = force_split;
  EpiParams epx = ep;
  epx.ksplit = 1;
  epx.split_flags = nullptr;
  if (nsplit > 1 && kind == EK_ACC_F32) {
    const int u = cluster_units(cl);
    const TileSched t = make_sched(M, N, bn, cl, true, u);
    epx.split_flags = split_flags(t.total * kEpiWarps * cl, stream);
    if (epx.split_flags) epx.ksplit = nsplit;
  }
  const EpiParams& epl = epx;
  if (cl == 4) {
    switch (bn) {
      case 256: return launch_kind<256, 4>(kind, A, lda, B, ldb, M, N, K, epl, stream);
      case 192: return launch_kind<192, 4>(kind, A, lda, B, ldb, M, N, K, epl, stream);
      default: return 1004;
    }
  }
  if (cl == 2) {
    switch (bn) {
      case 256: return launch_kind<256, 2>(kind, A, lda, B, ldb, M, N, K, epl, stream);
      case 192: return launch_kind<192, 2>(kind, A, lda, B, ldb, M, N, K, epl, stream);
      default: return 1004;
    }
  }
  switch (bn) {
    case 256: return launch_kind<256, 1>(kind, A, lda, B, ldb, M, N, K, epl, stream);
    case 192: return launch_kind<192, 1>(kind, A, lda, B, ldb, M, N, K, epl, stream);
    case 128: return launch_kind<128, 1>(kind, A, lda, B, ldb, M, N, K, epl, stream);
    default: return 1004;
  }
}

}  // namespace epd
