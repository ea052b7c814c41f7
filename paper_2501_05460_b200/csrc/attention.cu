// Fused multi-head attention (bidirectional) for sm_100a.
//
// One CTA = NQ (1 or 2) tiles of 128 query rows of one (batch, head); the tiles
// share every K/V block. Per 64-key block j and query tile g:
//   S_g(j) = Q_g K_j^T        tcgen05.mma, A = Q_g resident in TMEM, B = K from smem,
//                             M=128 N=64 K=Dp -> fp32 S in TMEM buffer j & 1
//   P_g(j) = exp2(S*c - m_g)  softmax warps (one thread per query row): TMEM -> regs ->
//                             bf16 P written back over the first 32 columns of S
//   O_g   += P_g(j) V_j       tcgen05.mma, A = P from TMEM, B = V from smem (MN-major)
// S is double-buffered per tile, so S_g(j+1) is computed while the softmax of
// block j runs and the softmax warps never wait for the tensor core. (With one S
// buffer -- FA4's layout, right for head dim 128 -- a head dim of 72..80 leaves
// the softmax -> PV -> S chain serial and the tensor pipe ~60% idle.) TMEM:
// 4 x 64 columns of S, then O_g and Q_g in a 128-column slot each.
// The softmax is MUFU-bound: a quarter of the exponentials run as a cubic on the
// FMA pipe. The running max m_g is only raised (and O_g rescaled, after waiting
// for the in-flight PV) when a row max grows by more than 2^8.
//
// Warps: 0 TMA (lane 0: Q, K; lane 1: V), 1 MMA issue (whole warp, elected lane),
// 2..5 softmax tile 0, 6..9 tile 1.
// Layouts: Q, K, V are read in place from the row-major projection outputs through
// 2-D tensor maps (head h = columns [h*hs, h*hs + Dp) of the section; see AttnParams).
// Q/K are K-major smem operands (64-wide SW128 atoms + a 16-wide SW32 tail when
// Dp % 64 != 0); V is the MN-major B operand from 16-wide SW32 atoms (LBO = 2 KB
// between atoms, SBO = 256 B between 8-key groups).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "tmap.h"


namespace epd {

namespace {

EPD_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (FA4's MUFU offload): round-to-nearest split x = k + f,
// f in [-0.5, 0.5], cubic minimax for 2^f (max rel err 7.5e-5, far below the bf16
// rounding of P), k added straight into the exponent bits. Inputs below -126 clamp
// (the result is then ~1e-38, i.e. zero for P).
EPD_DEVICE float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) lands in the low mantissa bits
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517133f, f, 0.2426105f), f, 0.693261f), f, 0.9999281f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// Packed fp32 pairs (sm_100 FFMA2 / FADD2): two lanes of softmax arithmetic per instruction.
EPD_DEVICE float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\nmov.b64 rc, {%6,%7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0,%1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
EPD_DEVICE float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\n"
      "add.rn.f32x2 rd, ra, rb;\nmov.b64 {%0,%1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// ex2_poly on a pair, the arithmetic packed
EPD_DEVICE float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 K = make_float2(12582912.f, 12582912.f), nK = make_float2(-12582912.f, -12582912.f);
  const float2 t = add2(x, K);
  const float2 r = add2(t, nK);
  const float2 f = add2(x, make_float2(-r.x, -r.y));
  float2 q = fma2(make_float2(0.05517133f, 0.05517133f), f, make_float2(0.2426105f, 0.2426105f));
  q = fma2(q, f, make_float2(0.693261f, 0.693261f));
  q = fma2(q, f, make_float2(0.9999281f, 0.9999281f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
#ifndef EPD_ATTN_TRACE
#define EPD_ATTN_TRACE 0
#endif
#if EPD_ATTN_TRACE
// Timeline of CTA 0's first 3 items, experiment builds only (tools/attn_trace.py):
// [event][softmax warp or MMA tile][item * 16 + block] = SM clock.
__device__ uint32_t g_attn_trace[8][8][48];
#define ATR(what, unit, it, j)                                                   \
  do {                                                                         \
    if (blockIdx.x == 0 && (it) < 3 && (j) < 16 && lane == 0)                  \
      g_attn_trace[what][unit][(it) * 16 + (j)] = (uint32_t)clock64();         \
  } while (0)
#else
#define ATR(what, unit, it, j) \
  do {                         \
  } while (0)
#endif
// Pairs (of every 8) whose exponentials run on the FMA pipe, per head-dim padding. Same-box
// A/B (profiles/r02/ab.txt, tools/attn_ab.py): SigLIP (Dp 80) 2/8 74.7 us, 3/8 73.7 us, 4/8
// 78.3 us; InternViT (Dp 64) 2/8 97.3 us, 3/8 95.3 us, 4/8 103 us.
#ifndef EPD_POLY_EIGHTHS
#define EPD_POLY_EIGHTHS 3
#endif
#ifndef EPD_POLY_EIGHTHS_64
#define EPD_POLY_EIGHTHS_64 3
#endif

EPD_DEVICE float fmax3(float a, float b, float c) {
  float m;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a), "f"(b), "f"(c));  // FMNMX3
  return m;
}

EPD_DEVICE void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
EPD_DEVICE void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
EPD_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Warp-wide issue helpers: every lane executes the call with identical (warp-uniform)
// operands, so the compiler keeps them in uniform registers; elect.sync picks the one
// lane that issues. (A single-lane `if (lane == 0)` issuer instead costs two R2UR moves
// plus an elect loop per MMA -- ~70-80 issue cycles, more than a 64-key MMA executes in.)
EPD_DEVICE void umma_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
EPD_DEVICE void tc_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}


template <int DP, int NQ>
struct Cfg {
  static constexpr int KB = 64;                        // keys per block
  static constexpr int KS = 4;                         // K pipeline stages
  static constexpr int KVS = 4;                        // V pipeline stages
  static constexpr int MAIN = DP / 64;                 // 64-wide SW128 atoms of Q/K
  static constexpr bool TAIL = (DP % 64) != 0;         // 16-wide SW32 tail (DP % 64 == 16)
  static constexpr int Q_ATOM = 128 * 128;             // 128 rows x 128 B
  static constexpr int Q_AL = (128 * DP * 2 + 1023) / 1024 * 1024;
  static constexpr int K_ATOM = KB * 128;              // 64 keys x 128 B
  static constexpr int K_BYTES = KB * DP * 2;
  static constexpr int K_AL = (K_BYTES + 1023) / 1024 * 1024;
  static constexpr int V_ATOM = KB * 32;               // 64 keys x 16 dims x 2 B
  static constexpr int V_BYTES = (DP / 16) * V_ATOM;
  static constexpr int V_AL = (V_BYTES + 1023) / 1024 * 1024;
  static constexpr int OFF_Q = 0;                      // [2 buffers][NQ tiles]: next item's Q prefetched
  static constexpr int OFF_K = OFF_Q + 2 * NQ * Q_AL;
  static constexpr int OFF_V = OFF_K + KS * K_AL;
  static constexpr int OFF_BAR = OFF_V + KVS * V_AL;
  static constexpr int BAR_BYTES = 34 * 8 + 8;         // 34 mbarriers + the TMEM holder
  static constexpr int SMEM = OFF_BAR + 512 + 1024;     // + slack for the 1024 B base alignment
  static_assert(BAR_BYTES <= 512, "barrier region");
  static constexpr int THREADS = 64 + NQ * 128;
  // TMEM columns: S_{g,b} (fp32, 64 wide) at (2g + b) * 64, P_{g,b} = bf16 pairs in its first
  // 32 columns; O_g at 256 + 128 g (DP wide); Q_g (bf16 pairs, DP/2 wide) right after O_g.
  __host__ __device__ static constexpr uint32_t s_col(int g, int b) { return (uint32_t)((2 * g + b) * 64); }
  __host__ __device__ static constexpr uint32_t o_col(int g) { return (uint32_t)(256 + 128 * g); }
  __host__ __device__ static constexpr uint32_t q_col(int g) { return (uint32_t)(256 + 128 * g + DP); }
  static_assert(DP + DP / 2 <= 128 || NQ == 1, "O_g and Q_g must share a 128-column slot");
  static_assert(DP + DP / 2 <= 256, "O and Q must fit above the S buffers");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// Work items: (query-tile pair, head, image), consecutive pairs sharing (image, head)
// (causal: the last query tiles of every head first).
// Pairs that would form a last, partial round over the persistent CTAs are split into
// single 128-row tiles, so that round takes about half as long; a single tile past Tq
// is an empty item (nq = 0) that every role skips without touching a barrier.
struct AttnItem {
  int b, h, q0, nq, nkb;  // nkb: 64-key blocks this item reads (causal items stop at their last row)
};
template <int NQ>
EPD_DEVICE AttnItem attn_item(const AttnParams& p, int w, int nqp, int npairs_main) {
  int pair = w, half = -1;
  if (w >= npairs_main) {
    pair = npairs_main + ((w - npairs_main) >> 1);
    half = (w - npairs_main) & 1;
  }
  AttnItem it;
  int qp = pair % nqp;
  int bh = pair / nqp;
  if (p.causal) {
    // causal items differ in work (query tile i reads ~i + 1 key blocks): hand them out
    // longest first, so a CTA's second item is one of the short ones
    const int nbh = p.H * p.B;
    qp = nqp - 1 - pair / nbh;
    bh = pair % nbh;
  }
  it.h = bh % p.H;
  it.b = bh / p.H;
  it.q0 = qp * (NQ * 128);
  if (half < 0 || NQ == 1) {
    it.nq = p.Tq - it.q0 > 128 ? NQ : 1;  // query tiles with at least one valid row
    if (NQ == 1 && half > 0) it.nq = 0;
  } else {
    it.q0 += half * 128;
    it.nq = p.Tq > it.q0 ? 1 : 0;
  }
  int kend = p.Tk;
  if (p.causal) {
    const int last_row = min(p.Tq, it.q0 + it.nq * 128) - 1;
    kend = min(p.Tk, last_row + 1 + (p.Tk - p.Tq));
  }
  it.nkb = (kend + 63) / 64;
  return it;
}
// Number of items and pairs kept whole for a persistent grid of G CTAs. The r pairs of a
// last, partial round are split only when their 2r single tiles still fit in one round: a
// single-tile item takes ~0.6 of a pair's time (its softmax is latency-bound), so two
// rounds of singles would be slower than the one round of pairs (a 2-tile IRP shard:
// 128 pairs on 148 SMs). The host passes the schedule (pairs kept whole) to the kernel.
// EPD_ATTN_SPLIT=0 keeps every pair whole, =1 always splits the partial round (A/B runs).
inline void attn_sched(int npairs, int G, int nq_max, int* main_pairs, int* nitems) {
  static const int mode = [] {
    const char* e = std::getenv("EPD_ATTN_SPLIT");
    return e && e[0] ? atoi(e) : -1;
  }();
  int m = nq_max > 1 ? (npairs / G) * G : npairs;
  if (mode == 0 || (mode < 0 && 2 * (npairs - m) > G)) m = npairs;
  *main_pairs = m;
  *nitems = m + 2 * (npairs - m);
}

// Persistent: one CTA per SM loops over the work items. Barrier phases are tracked per
// role and per (tile, buffer) so that tail items with a single query tile keep both sides
// of every barrier in step.
template <int DP, int NQ>
__global__ void __launch_bounds__(Cfg<DP, NQ>::THREADS, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQt,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKt,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p, const int pmain) {
  using C = Cfg<DP, NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;    // [2] Q buffer landed
  uint64_t* q_empty = bars + 2;   // [2] Q buffer copied into TMEM by every softmax thread
  uint64_t* k_full = bars + 4;    // [KS]
  uint64_t* k_empty = bars + 8;   // [KS]
  uint64_t* v_full = bars + 12;   // [KVS]
  uint64_t* v_empty = bars + 16;  // [KVS]
  uint64_t* s_full = bars + 20;   // [NQ][2] S_g(j) landed in buffer j & 1
  // [NQ][2] P_g(j) written to TMEM buffer j & 1. One barrier per buffer: a softmax group
  // may finish blocks j and j+1 before the MMA warp consumes P_g(j), which would alias
  // the phase parity of a single barrier.
  uint64_t* p_ready = bars + 24;
  uint64_t* pv_done = bars + 28;  // [NQ] PV_g(j) complete (O_g stable up to block j)
  uint64_t* q_tm = bars + 30;     // [NQ] Q_g copied into TMEM
  uint64_t* o_done = bars + 32;   // [NQ] the item's last PV_g complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 34);

  const int warp = warp_id();
  const int lane = lane_id();
  const int nqp = (p.Tq + NQ * 128 - 1) / (NQ * 128);
  const int nitems = pmain + 2 * (nqp * p.H * p.B - pmain);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], NQ * 128);
    }
    for (int i = 0; i < C::KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < C::KVS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int g = 0; g < NQ; ++g) {
      mbar_init(&s_full[2 * g], 1);
      mbar_init(&s_full[2 * g + 1], 1);
      mbar_init(&p_ready[2 * g], 128);
      mbar_init(&p_ready[2 * g + 1], 128);
      mbar_init(&pv_done[g], 1);
      mbar_init(&o_done[g], 1);
      mbar_init(&q_tm[g], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_trigger();
  pdl_wait();  // Q, K, V come from the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      // Q of each item (double-buffered, so the next item's Q is fetched during this one)
      // followed by its K blocks; the K ring runs on across items.
      int kc = 0, it = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const AttnItem x = attn_item<NQ>(p, w, nqp, pmain);
        const int qb = it & 1;
        const int hcol = x.h * p.hs;
        mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], x.nq * 128 * DP * 2);
        for (int g = 0; g < x.nq; ++g) {
          uint8_t* qd = smem + C::OFF_Q + (qb * NQ + g) * C::Q_AL;
          const int qr = (p.q_shared ? 0 : x.b * p.Tq) + x.q0 + g * 128;
          for (int a = 0; a < C::MAIN; ++a) tma_load_2d(qd + a * C::Q_ATOM, &tmQ, &q_full[qb], hcol + a * 64, qr);
          if (C::TAIL) tma_load_2d(qd + C::MAIN * C::Q_ATOM, &tmQt, &q_full[qb], hcol + C::MAIN * 64, qr);
        }
        if (x.nq == 0) continue;  // empty item: Q buffer handed over with no bytes, no K blocks
        const int krow0 = x.b * p.Tk;
        const int kvcol = (x.h / p.kv_group) * p.hs;
        for (int j = 0; j < x.nkb; ++j, ++kc) {
          const int s = kc % C::KS;
          mbar_wait(&k_empty[s], ((kc / C::KS) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[s], C::K_BYTES);
          uint8_t* kd = smem + C::OFF_K + s * C::K_AL;
          for (int a = 0; a < C::MAIN; ++a)
            tma_load_2d(kd + a * C::K_ATOM, &tmK, &k_full[s], kvcol + a * 64, krow0 + j * C::KB);
          if (C::TAIL) tma_load_2d(kd + C::MAIN * C::K_ATOM, &tmKt, &k_full[s], kvcol + C::MAIN * 64, krow0 + j * C::KB);
        }
      }
    } else if (lane == 1) {
      int vc = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        const AttnItem x = attn_item<NQ>(p, w, nqp, pmain);
        if (x.nq == 0) continue;
        const int hcol = (x.h / p.kv_group) * p.hs, krow0 = x.b * p.Tk;
        for (int j = 0; j < x.nkb; ++j, ++vc) {
          const int s = vc % C::KVS;
          mbar_wait(&v_empty[s], ((vc / C::KVS) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[s], C::V_BYTES);
          uint8_t* vd = smem + C::OFF_V + s * C::V_AL;
          for (int a = 0; a < DP / 16; ++a)
            tma_load_2d(vd + a * C::V_ATOM, &tmV, &v_full[s], hcol + a * 16, krow0 + j * C::KB);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform operands, elected issue
      constexpr uint32_t idesc_s = make_idesc_bf16(128, C::KB);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DP) | (1u << 16);  // B (V) is MN-major
      const uint64_t k_main0 = make_sdesc(smem_u32(smem + C::OFF_K), 1024, 2);
      const uint64_t k_tail0 = make_sdesc(smem_u32(smem + C::OFF_K + C::MAIN * C::K_ATOM), 256, 6);
      const uint64_t v_base0 = make_sdesc_lbo(smem_u32(smem + C::OFF_V), C::V_ATOM, 256, 6);
      int kc = 0, vc = 0;
      uint32_t qtm_ph = 0, pr_ph = 0;  // phase bits: q_tm bit g, p_ready bit 2g + buffer
      // S_g(j) = Q_g K_j^T into buffer j & 1; K block j sits in ring slot kslot.
      auto issue_s = [&](int g, int j, int kslot) {
        const uint64_t ko = (uint64_t)((kslot * C::K_AL) >> 4);
        const uint32_t d = tmem + C::s_col(g, j & 1);
        const uint32_t qa = tmem + C::q_col(g);
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) {
          const int atom = kk >> 2;
          if (atom < C::MAIN) {
            const uint64_t off = (uint64_t)((atom * C::K_ATOM + (kk & 3) * 32) >> 4);
            umma_ts_warp(d, qa + kk * 8, k_main0 + ko + off, idesc_s, kk != 0);
          } else {
            umma_ts_warp(d, qa + kk * 8, k_tail0 + ko, idesc_s, kk != 0);
          }
        }
        tc_commit_warp(&s_full[2 * g + (j & 1)]);
      };
      for (int w = blockIdx.x, mit = 0; w < nitems; w += gridDim.x, ++mit) {
        const AttnItem x = attn_item<NQ>(p, w, nqp, pmain);
        if (x.nq == 0) continue;
        for (int g = 0; g < x.nq; ++g) {
          mbar_wait(&q_tm[g], (qtm_ph >> g) & 1);
          qtm_ph ^= 1u << g;
        }
        tc_fence_after();
        // two blocks of S in flight per query tile: softmax(j) overlaps S(j+1)
        const int nkb = x.nkb;
        for (int j = 0; j < 2 && j < nkb; ++j) {
          const int ks = (kc + j) % C::KS;
          mbar_wait(&k_full[ks], ((kc + j) / C::KS) & 1);
          tc_fence_after();
          for (int g = 0; g < x.nq; ++g) issue_s(g, j, ks);
          tc_commit_warp(&k_empty[ks]);
        }
        for (int j = 0; j < nkb; ++j) {
          const int sv = (vc + j) % C::KVS;
          bool v_ok = false, k_ok = false;
          uint32_t pending = (1u << x.nq) - 1u;
          for (int n_served = 0; n_served < x.nq; ++n_served) {
            const int g = __ffs(pending) - 1;
            pending &= ~(1u << g);
            const int pb = 2 * g + (j & 1);
            mbar_wait(&p_ready[pb], (pr_ph >> pb) & 1);
            ATR(2, g, mit, j);
            pr_ph ^= 1u << pb;
            if (!v_ok) {
              mbar_wait(&v_full[sv], ((vc + j) / C::KVS) & 1);
              v_ok = true;
            }
            tc_fence_after();
            const uint64_t vb = v_base0 + (uint64_t)((sv * C::V_AL) >> 4);
            const uint32_t od = tmem + C::o_col(g), pa = tmem + C::s_col(g, j & 1);
#pragma unroll
            for (int kk = 0; kk < C::KB / 16; ++kk) {
              // A = P from TMEM: keys 16kk..16kk+15 are bf16 pairs in columns 8kk..8kk+7
              // B = V, MN-major SW32: key row kk*16 (512 B), LBO = 2 KB (next 16 dims), SBO = 256 B
              umma_ts_warp(od, pa + kk * 8, vb + (uint64_t)(kk * 32), idesc_o, (j | kk) != 0);
            }
            tc_commit_warp(&pv_done[g]);
            if (j + 1 == nkb) tc_commit_warp(&o_done[g]);
            if (j + 2 < nkb) {
              // S_g(j+2) overwrites P_g(j) only after PV_g(j) (in-order tensor pipe)
              const int ks = (kc + j + 2) % C::KS;
              if (!k_ok) {
                mbar_wait(&k_full[ks], ((kc + j + 2) / C::KS) & 1);
                k_ok = true;
              }
              tc_fence_after();
              issue_s(g, j + 2, ks);
              ATR(3, g, mit, j);
            }
          }
          tc_commit_warp(&v_empty[sv]);
          if (j + 2 < nkb) tc_commit_warp(&k_empty[(kc + j + 2) % C::KS]);
        }
        kc += nkb;
        vc += nkb;
      }
    }
  } else {
    // ---------------- softmax: 4 warps per query tile, one thread per query row (TMEM lane)
    const int wi = warp - 2;
    const int g = wi >> 2;
    const int qq = warp & 3;  // TMEM lane quarter this warp may access
    const int r = qq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
    const uint32_t o_tm = tmem + lane_off + C::o_col(g);
    const float c = p.scale * 1.4426950408889634f;
    uint32_t sf_ph = 0, od_ph = 0;  // s_full phase bit per buffer
    int pv_count = 0;  // PV_g commits so far (pv_done phase bookkeeping)
    // Wait for item `it`'s Q buffer; tiles of this warp's group copy their Q rows into TMEM
    // as bf16 pairs (column c = head dims 2c, 2c+1: the TS-MMA A layout), zeroing dims >= Dv.
    // Every thread releases the buffer. Called only once all S MMAs of the previous item
    // are complete (its last s_full was observed).
    auto take_q = [&](int it, int nq) {
      const int qb = it & 1;
      mbar_wait(&q_full[qb], (it >> 1) & 1);
      if (g < nq) {
        const uint8_t* qs = smem + C::OFF_Q + (qb * NQ + g) * C::Q_AL;
        const uint32_t q_tm_addr = tmem + lane_off + C::q_col(g);
#pragma unroll
        for (int c8 = 0; c8 < DP / 8; ++c8) {
          const int d = c8 * 8;
          uint4 u = make_uint4(0u, 0u, 0u, 0u);  // dims >= Dv (the neighbouring head's columns) -> 0
          if (d >= p.Dv) {
          } else if (d < C::MAIN * 64) {
            const int atom = d >> 6, ch = (d & 63) >> 3;
            u = *reinterpret_cast<const uint4*>(qs + atom * C::Q_ATOM + r * 128 + ((ch ^ (r & 7)) * 16));
          } else {
            const int ch = (d - C::MAIN * 64) >> 3;
            u = *reinterpret_cast<const uint4*>(qs + C::MAIN * C::Q_ATOM + r * 32 + ((ch ^ ((r >> 2) & 1)) * 16));
          }
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(q_tm_addr + c8 * 4),
                       "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                       : "memory");
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&q_tm[g]);
      }
      mbar_arrive(&q_empty[qb]);
    };
    int it = 0;
    if ((int)blockIdx.x < nitems) take_q(0, attn_item<NQ>(p, blockIdx.x, nqp, pmain).nq);
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
      const AttnItem x = attn_item<NQ>(p, w, nqp, pmain);
      float l = 0.f;
      const int nkb = x.nkb;
      // keys this thread's query row may see (causal: up to its own position)
      const int klim = p.causal ? min(p.Tk, x.q0 + g * 128 + r + 1 + (p.Tk - p.Tq)) : p.Tk;
      if (g < x.nq) {
        float m_used = -INFINITY;
        for (int j = 0; j < nkb; ++j) {
          const int kvalid = klim - j * C::KB;
          mbar_wait(&s_full[2 * g + (j & 1)], (sf_ph >> (j & 1)) & 1);
          ATR(0, wi, it, j);
          sf_ph ^= 1u << (j & 1);
          tc_fence_after();
          const uint32_t s_tm = tmem + lane_off + C::s_col(g, j & 1);
          uint32_t sv[64];
          tmem_ld32(s_tm, *reinterpret_cast<uint32_t(*)[32]>(sv));
          tmem_ld32(s_tm + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
          tmem_ld_wait();
          ATR(4, wi, it, j);
          if (kvalid < 64) {
#pragma unroll
            for (int i = 0; i < 64; ++i)
              if (i >= kvalid) sv[i] = __float_as_uint(-INFINITY);
          }
          float mx;
          {
            float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < 64; i += 8)
#pragma unroll
              for (int u = 0; u < 4; ++u)
                m4[u] = fmax3(m4[u], __uint_as_float(sv[i + 2 * u]), __uint_as_float(sv[i + 2 * u + 1]));
            mx = fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
          }
          const float m_new = fmaxf(m_used, mx * c);
          if (j == 0) {
            m_used = m_new;
          } else {
            // Lazy rescale: only when a row max grows by more than 2^8. PV_g(j-1) may still
            // be accumulating into O_g, so wait for it first (rare path).
            const bool need = m_new > m_used + 8.f;
            ATR(5, wi, it, j);
            if (__any_sync(0xffffffffu, need)) {
              mbar_wait(&pv_done[g], (pv_count - 1) & 1);
              tc_fence_after();
              const float alpha = need ? ex2(m_used - m_new) : 1.f;
#pragma unroll
              for (int c0 = 0; c0 < DP; c0 += 16) {
                uint32_t o[16];
                tmem_ld16(o_tm + c0, o);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st8(o_tm + c0, o);
                tmem_st8(o_tm + c0 + 8, o + 8);
              }
              tmem_st_wait();
              if (need) {
                l *= alpha;
                m_used = m_new;
              }
            }
          }
          const float nm = -m_used;
          float2 rs0 = make_float2(0.f, 0.f), rs1 = rs0;
          uint32_t pk[32];
          const float2 c2 = make_float2(c, c), nm2 = make_float2(nm, nm);
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            // The softmax is MUFU-bound (16 ex2/clk/SM): a share of the pairs goes to the FMA
            // pipe; the pair arithmetic runs as packed FFMA2 / FADD2.
            const bool poly = ((i >> 1) & 7) < (DP == 64 ? EPD_POLY_EIGHTHS_64 : EPD_POLY_EIGHTHS);
            const float2 a = fma2(make_float2(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), c2, nm2);
            const float2 e = poly ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
            if ((i >> 1) & 1) rs1 = add2(rs1, e);
            else rs0 = add2(rs0, e);
            pk[i >> 1] = pack_bf16x2(e.x, e.y);
          }
          ATR(6, wi, it, j);
          tmem_st32(s_tm, pk);  // P_g(j) over the first 32 columns of S_g(j)
          tmem_st_wait();
          ATR(7, wi, it, j);
          const float2 rs = add2(rs0, rs1);
          l += rs.x + rs.y;
          tc_fence_before();
          ATR(1, wi, it, j);
          mbar_arrive(&p_ready[2 * g + (j & 1)]);
          ++pv_count;
        }
      }
      // All S MMAs of this item are complete: hand the next item's Q to the tensor core
      // before the O epilogue, so its first S blocks overlap the epilogue.
      const int wn = w + gridDim.x;
      if (wn < nitems) take_q(it + 1, attn_item<NQ>(p, wn, nqp, pmain).nq);
      if (g < x.nq) {
        mbar_wait(&o_done[g], od_ph);
        od_ph ^= 1;
        tc_fence_after();
        const int qrow = x.q0 + g * 128 + r;
        const float inv = 1.f / l;
        bf16* dst = p.out + ((size_t)x.b * p.Tq + qrow) * p.ldo + (size_t)x.h * p.Dv;
#pragma unroll
        for (int c0 = 0; c0 < DP; c0 += 16) {
          uint32_t o[16];
          tmem_ld16(o_tm + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (qrow < p.Tq && c0 + hh * 8 < p.Dv) {
              const uint32_t* oo = o + hh * 8;
              uint4 v;
              v.x = pack_bf16x2(__uint_as_float(oo[0]) * inv, __uint_as_float(oo[1]) * inv);
              v.y = pack_bf16x2(__uint_as_float(oo[2]) * inv, __uint_as_float(oo[3]) * inv);
              v.z = pack_bf16x2(__uint_as_float(oo[4]) * inv, __uint_as_float(oo[5]) * inv);
              v.w = pack_bf16x2(__uint_as_float(oo[6]) * inv, __uint_as_float(oo[7]) * inv);
              *reinterpret_cast<uint4*>(dst + c0 + hh * 8) = v;
            }
          }
        }
        // O_g is read: the next item's PV_g(0) (issued after its P_g(0), i.e. after this
        // thread's next p_ready arrival) may overwrite it.
        tc_fence_before();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int DP, int NQ>
int launch_attn(const AttnParams& p, cudaStream_t stream) {
  using C = Cfg<DP, NQ>;
  // 2-D maps over each section (H heads x hs columns); rows = tokens of all images. Boxes
  // that run past the last head or the last row are zero-filled by the TMA.
  const uint64_t width = (uint64_t)p.H * p.hs;
  const uint64_t kv_width = (uint64_t)(p.H / p.kv_group) * p.hs;
  const uint64_t qrows = p.q_shared ? p.Tq : (uint64_t)p.B * p.Tq;
  const uint64_t krows = (uint64_t)p.B * p.Tk;
  CUtensorMap mq, mqt, mk, mkt, mv;
  int rc = make_tmap_2d(&mq, p.q, width, qrows, (uint64_t)p.ldq * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_2d(&mqt, p.q, width, qrows, (uint64_t)p.ldq * 2, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
  if (!rc) rc = make_tmap_2d(&mk, p.k, kv_width, krows, (uint64_t)p.ldk * 2, 64, C::KB, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_2d(&mkt, p.k, kv_width, krows, (uint64_t)p.ldk * 2, 16, C::KB, CU_TENSOR_MAP_SWIZZLE_32B);
  if (!rc) rc = make_tmap_2d(&mv, p.v, kv_width, krows, (uint64_t)p.ldv * 2, 16, C::KB, CU_TENSOR_MAP_SWIZZLE_32B);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<DP, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  const int npairs = ((p.Tq + NQ * 128 - 1) / (NQ * 128)) * p.H * p.B;
  int pmain = 0, nitems = 0;
  attn_sched(npairs, num_sms(), NQ, &pmain, &nitems);
  const int grid = nitems < num_sms() ? nitems : num_sms();
  return launch_kernel(attention_kernel<DP, NQ>, dim3(grid), dim3(C::THREADS), C::SMEM, stream, 1, mq, mqt, mk, mkt,
                       mv, p, pmain);
}

}  // namespace

#if EPD_ATTN_TRACE
extern "C" int epd_debug_attn_trace(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_attn_trace, sizeof(g_attn_trace));
}
#endif

int attention_bf16(const AttnParams& p, cudaStream_t stream) {
  if (p.B <= 0 || p.H <= 0 || p.Tq <= 0 || p.Tk <= 0 || p.Dv <= 0 || p.Dv > p.Dp) return 1001;
  if ((p.ldo % 8) != 0 || (p.Dv % 8) != 0) return 1002;
  if (p.hs < p.Dv || p.ldq % 8 || p.ldk % 8 || p.ldv % 8 || p.hs % 8) return 1002;
  if (p.kv_group < 1 || p.H % p.kv_group) return 1001;
  if (p.causal && (p.Tk < p.Tq || p.q_shared)) return 1001;
  if ((reinterpret_cast<uintptr_t>(p.q) | reinterpret_cast<uintptr_t>(p.k) | reinterpret_cast<uintptr_t>(p.v)) & 15)
    return 1003;
  const bool two = p.Tq > 128;
  switch (p.Dp) {
    case 64: return two ? launch_attn<64, 2>(p, stream) : launch_attn<64, 1>(p, stream);
    case 80: return two ? launch_attn<80, 2>(p, stream) : launch_attn<80, 1>(p, stream);
    case 128: return launch_attn<128, 1>(p, stream);
    default: return 1004;
  }
}

}  // namespace epd
