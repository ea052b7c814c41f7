// Fused multi-head attention (bidirectional) for sm_100a, FA4-style.
//
// One CTA = NQ (1 or 2) tiles of 128 query rows of one (batch, head); the
// tiles share every K/V block. Per 128-key block j and query tile g:
//   S_g  = Q_g K_j^T          tcgen05.mma (A, B from smem)  M=128 N=128 K=Dp -> TMEM fp32
//   P_g  = exp2(S_g*c - m_g)  softmax warps: TMEM -> regs -> bf16 P written back to TMEM,
//                             aliasing the first 64 columns of S_g (no smem round trip)
//   O_g += P_g V_j            tcgen05.mma (A = P from TMEM, B = V from smem, MN-major)
// The running max m_g is only raised (and O_g rescaled in TMEM) when a row's
// max grows by more than 2^8, so most blocks need no correction pass. Because
// S_g(j+1) is issued after PV_g(j), the arrival of S_g(j) also means O_g is
// stable and P_g(j-1) has been consumed. While one tile runs its softmax the
// tensor core works on the other tile's PV and S.
//
// Warps: 0 TMA (lane 0: Q, K; lane 1: V), 1 TMEM alloc + MMA issue,
// 2..9 softmax tile 0, 10..17 tile 1 (two warps per TMEM lane quarter, each
// owning half of the key columns and half of the head dims).
// Layouts: Q, K, V all [bh][T][Dp] bf16 (Dp = head dim zero-padded to a
// multiple of 16). Q/K are K-major smem operands (64-wide SW128 atoms + a
// 16-wide SW32 tail when Dp % 64 != 0); V is the MN-major B operand from
// 16-wide SW32 atoms (LBO = 4 KB between atoms, SBO = 256 B between 8-key groups).
#include "common.cuh"
#include "kernels.h"
#include "tmap.h"

namespace epd {

namespace {

EPD_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

EPD_DEVICE void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
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
EPD_DEVICE void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EPD_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T (A operand from tensor memory).
EPD_DEVICE void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int DP, int NQ>
struct Cfg {
  static constexpr int KB = 128;                       // keys per block
  static constexpr int KS = 3;                         // K pipeline stages
  static constexpr int KVS = DP <= 80 ? 3 : 2;         // V pipeline stages (smem permitting)
  static constexpr int MAIN = DP / 64;                 // 64-wide SW128 atoms of Q/K
  static constexpr bool TAIL = (DP % 64) != 0;         // 16-wide SW32 tail (DP % 64 == 16)
  static constexpr int QK_ATOM = 128 * 128;            // 128 rows x 128 B
  static constexpr int QK_BYTES = 128 * DP * 2;
  static constexpr int QK_AL = (QK_BYTES + 1023) / 1024 * 1024;
  static constexpr int V_ATOM = 128 * 32;              // 128 keys x 16 dims x 2 B
  static constexpr int V_BYTES = (DP / 16) * V_ATOM;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * QK_AL;
  static constexpr int OFF_V = OFF_K + KS * QK_AL;
  static constexpr int OFF_RED = OFF_V + KVS * V_BYTES;     // [NQ][2][2][128] fp32 row exchange
  static constexpr int OFF_BAR = OFF_RED + NQ * 2 * 2 * 128 * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int THREADS = 64 + NQ * 256;
  // TMEM column of Q_0 (bf16 pairs, DP/2 columns) right after O_0; Q_g at QT_COL + 128 g
  static constexpr int QT_COL = 256 + DP;
  static_assert(DP + DP / 2 <= 128 || NQ == 1, "O_g and Q_g must share a 128-column slot");
};

template <int DP, int NQ>
__global__ void __launch_bounds__(Cfg<DP, NQ>::THREADS, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQt,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKt,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Cfg<DP, NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [KS]
  uint64_t* k_empty = bars + 4;   // [KS]
  uint64_t* v_full = bars + 7;    // [KVS]
  uint64_t* v_empty = bars + 10;  // [KVS]
  uint64_t* s_full = bars + 13;   // [NQ] S_g(j) in TMEM (and, by issue order, PV_g(j-1) complete)
  uint64_t* p_ready = bars + 15;  // [NQ] P_g(j) written to TMEM
  uint64_t* o_done = bars + 17;   // [NQ] last PV_g complete
  uint64_t* q_tm = bars + 19;     // [NQ] Q_g copied into TMEM
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 21);

  const int warp = warp_id();
  const int lane = lane_id();
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int bh = b * p.H + h;
  const int qbatch = p.q_shared ? h : bh;
  const int q0 = blockIdx.x * (NQ * 128);
  const int rem = p.Tq - q0;
  const int nq = rem > 128 ? NQ : 1;  // query tiles with at least one valid row
  const int nkb = (p.Tk + C::KB - 1) / C::KB;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < C::KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < C::KVS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int g = 0; g < NQ; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_ready[g], 256);
      mbar_init(&o_done[g], 1);
      mbar_init(&q_tm[g], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // TMEM columns: S_g / P_g at [g*128, g*128+128) (P = bf16 pairs in the first 64),
  // O_g at [256 + g*128, 256 + g*128 + DP)

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, nq * C::QK_BYTES);
      for (int g = 0; g < nq; ++g) {
        uint8_t* qd = smem + C::OFF_Q + g * C::QK_AL;
        for (int a = 0; a < C::MAIN; ++a) tma_load_3d(qd + a * C::QK_ATOM, &tmQ, q_full, a * 64, q0 + g * 128, qbatch);
        if (C::TAIL) tma_load_3d(qd + C::MAIN * C::QK_ATOM, &tmQt, q_full, C::MAIN * 64, q0 + g * 128, qbatch);
      }
      for (int j = 0; j < nkb; ++j) {
        const int s = j % C::KS;
        mbar_wait(&k_empty[s], ((j / C::KS) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], C::QK_BYTES);
        uint8_t* kd = smem + C::OFF_K + s * C::QK_AL;
        for (int a = 0; a < C::MAIN; ++a) tma_load_3d(kd + a * C::QK_ATOM, &tmK, &k_full[s], a * 64, j * C::KB, bh);
        if (C::TAIL) tma_load_3d(kd + C::MAIN * C::QK_ATOM, &tmKt, &k_full[s], C::MAIN * 64, j * C::KB, bh);
      }
    } else if (lane == 1) {
      for (int j = 0; j < nkb; ++j) {
        const int s = j % C::KVS;
        mbar_wait(&v_empty[s], ((j / C::KVS) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[s], C::V_BYTES);
        uint8_t* vd = smem + C::OFF_V + s * C::V_BYTES;
        for (int a = 0; a < DP / 16; ++a) tma_load_3d(vd + a * C::V_ATOM, &tmV, &v_full[s], a * 16, j * C::KB, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, C::KB);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DP) | (1u << 16);  // B (V) is MN-major
      mbar_wait(q_full, 0);
      // Descriptors are precomputed: per MMA the issuing thread only adds a constant
      // (start address >> 4) to a base descriptor -- at N = 80..128 the tensor core
      // finishes an MMA in 40..64 cycles, so a serial descriptor build would starve it.
      const uint64_t k_main0 = make_sdesc(smem_u32(smem + C::OFF_K), 1024, 2);
      const uint64_t k_tail0 = make_sdesc(smem_u32(smem + C::OFF_K + C::MAIN * C::QK_ATOM), 256, 6);
      const uint64_t v_base0 = make_sdesc_lbo(smem_u32(smem + C::OFF_V), C::V_ATOM, 256, 6);
      // S = Q K^T with Q resident in TMEM (A operand): only K is read from smem, so the
      // S MMAs are no longer smem-bandwidth bound (A+B from smem = 8 KB per 64 cycles).
      auto issue_s = [&](int g, int j) {
        const uint64_t ko = (uint64_t)(((j % C::KS) * C::QK_AL) >> 4);
        const uint32_t d = tmem + g * 128;
        const uint32_t qa = tmem + C::QT_COL + g * 128;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) {
          const int atom = kk >> 2;
          if (atom < C::MAIN) {
            const uint64_t off = (uint64_t)((atom * C::QK_ATOM + (kk & 3) * 32) >> 4);
            umma_bf16_ts(d, qa + kk * 8, k_main0 + ko + off, idesc_s, kk != 0);
          } else {
            umma_bf16_ts(d, qa + kk * 8, k_tail0 + ko, idesc_s, kk != 0);
          }
        }
        tc_commit(&s_full[g]);
      };
      mbar_wait(&k_full[0], 0);
      for (int g = 0; g < nq; ++g) mbar_wait(&q_tm[g], 0);
      tc_fence_after();
      for (int g = 0; g < nq; ++g) issue_s(g, 0);
      tc_commit(&k_empty[0]);
      for (int j = 0; j < nkb; ++j) {
        const int sv = j % C::KVS;
        for (int g = 0; g < nq; ++g) {
          mbar_wait(&p_ready[g], j & 1);
          if (g == 0) mbar_wait(&v_full[sv], (j / C::KVS) & 1);
          tc_fence_after();
          const uint64_t vb = v_base0 + (uint64_t)((sv * C::V_BYTES) >> 4);
          const uint32_t od = tmem + 256 + g * 128, pa = tmem + g * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // A = P from TMEM: keys 16kk..16kk+15 are bf16 pairs in columns 8kk..8kk+7
            // B = V, MN-major SW32: key row kk*16 (512 B), LBO = 4 KB (next 16 dims), SBO = 256 B
            umma_bf16_ts(od, pa + kk * 8, vb + (uint64_t)(kk * 32), idesc_o, (j | kk) != 0);
          }
          if (j + 1 == nkb) {
            tc_commit(&o_done[g]);
          } else {
            // S_g(j+1) overwrites P_g(j) only after PV_g(j) (in-order tensor pipe)
            if (g == 0) mbar_wait(&k_full[(j + 1) % C::KS], ((j + 1) / C::KS) & 1);
            tc_fence_after();
            issue_s(g, j + 1);
          }
        }
        tc_commit(&v_empty[sv]);
        if (j + 1 < nkb) tc_commit(&k_empty[(j + 1) % C::KS]);
      }
    }
  } else {
    // ---------------- softmax: per query tile g, 8 warps = 2 per TMEM lane quarter;
    // thread (row r, half hf) owns key columns [hf*64, hf*64+64) of S and head dims
    // [hf*DP/2, (hf+1)*DP/2) of O. Row maxima are combined through smem each block.
    const int wi = warp - 2;
    const int g = wi >> 3;
    const int hf = (wi >> 2) & 1;
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
    const uint32_t s_tm = tmem + lane_off + g * 128 + hf * 64;
    const uint32_t p_tm = tmem + lane_off + g * 128 + hf * 32;
    constexpr int OH = DP / 2;  // O columns per half (multiple of 8)
    const uint32_t o_tm = tmem + lane_off + 256 + g * 128 + hf * OH;
    // [2 block parity][2 hf][128]: row-max exchange; the final row sums reuse a slot
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED) + g * (2 * 2 * 128);
    const float c = p.scale * 1.4426950408889634f;
    const int bar_id = 1 + g;
    if (g < nq) {
      {
        // copy this thread's half of its Q row (K-major swizzled smem) into TMEM as bf16
        // pairs: column c of Q_g holds head dims 2c, 2c+1 (the TS-MMA A-operand layout)
        mbar_wait(q_full, 0);
        const uint8_t* qs = smem + C::OFF_Q + g * C::QK_AL;
        const uint32_t q_tm_addr = tmem + lane_off + C::QT_COL + g * 128 + hf * (DP / 4);
#pragma unroll
        for (int c8 = 0; c8 < DP / 16; ++c8) {  // 8-dim chunks of this half
          const int d = hf * (DP / 2) + c8 * 8;
          uint4 u;
          if (d < C::MAIN * 64) {
            const int atom = d >> 6, ch = (d & 63) >> 3;
            u = *reinterpret_cast<const uint4*>(qs + atom * C::QK_ATOM + r * 128 + ((ch ^ (r & 7)) * 16));
          } else {
            const int ch = (d - C::MAIN * 64) >> 3;
            u = *reinterpret_cast<const uint4*>(qs + C::MAIN * C::QK_ATOM + r * 32 + ((ch ^ ((r >> 2) & 1)) * 16));
          }
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(q_tm_addr + c8 * 4),
                       "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                       : "memory");
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&q_tm[g]);
      }
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkb; ++j) {
        const int kvalid = p.Tk - j * C::KB - hf * 64;  // valid keys among this thread's 64
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
        uint32_t sv[64];
        tmem_ld32(s_tm, *reinterpret_cast<uint32_t(*)[32]>(sv));
        tmem_ld32(s_tm + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
        tmem_ld_wait();
        float mx = -INFINITY;
        if (kvalid >= 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i) mx = fmaxf(mx, __uint_as_float(sv[i]));
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            if (i >= kvalid) sv[i] = __float_as_uint(-INFINITY);
            mx = fmaxf(mx, __uint_as_float(sv[i]));
          }
        }
        float* rb = red + (j & 1) * 256;
        rb[hf * 128 + r] = mx;
        // Both halves have read their S columns before either writes P over them.
        named_bar_sync(bar_id, 256);
        mx = fmaxf(mx, rb[(hf ^ 1) * 128 + r]);
        const float m_new = fmaxf(m_used, mx * c);
        if (j == 0) {
          m_used = m_new;
        } else {
          // S_g(j) was issued after PV_g(j-1): O_g is stable here.
          const bool need = m_new > m_used + 8.f;
          if (__any_sync(0xffffffffu, need)) {
            const float alpha = need ? ex2(m_used - m_new) : 1.f;
#pragma unroll
            for (int c0 = 0; c0 < OH; c0 += 8) {
              uint32_t o[8];
              tmem_ld8(o_tm + c0, o);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st8(o_tm + c0, o);
            }
            if (need) {
              l *= alpha;
              m_used = m_new;
            }
          }
        }
        const float nm = -m_used;
        float rs0 = 0.f, rs1 = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          const float e0 = ex2(fmaf(__uint_as_float(sv[i]), c, nm));
          const float e1 = ex2(fmaf(__uint_as_float(sv[i + 1]), c, nm));
          rs0 += e0;
          rs1 += e1;
          pk[i >> 1] = pack_bf16x2(e0, e1);
        }
        tmem_st32(p_tm, pk);
        tmem_st_wait();
        l += rs0 + rs1;
        tc_fence_before();
        mbar_arrive(&p_ready[g]);
      }
      // combine the two halves' row sums
      // the parity slot of block nkb was last read during block nkb-2's exchange, which
      // every thread of the group has passed (block nkb-1's barrier): safe to reuse
      float* lb = red + (nkb & 1) * 256;
      lb[hf * 128 + r] = l;
      named_bar_sync(bar_id, 256);
      l += lb[(hf ^ 1) * 128 + r];
      mbar_wait(&o_done[g], 0);
      tc_fence_after();
      const int qrow = q0 + g * 128 + r;
      const float inv = 1.f / l;
      bf16* dst = p.out + ((size_t)b * p.Tq + qrow) * p.ldo + (size_t)h * p.Dv + hf * OH;
#pragma unroll
      for (int c0 = 0; c0 < OH; c0 += 8) {
        uint32_t o[8];
        tmem_ld8(o_tm + c0, o);
        tmem_ld_wait();
        if (qrow < p.Tq && hf * OH + c0 < p.Dv) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv);
          v.y = pack_bf16x2(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv);
          v.z = pack_bf16x2(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv);
          v.w = pack_bf16x2(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv);
          *reinterpret_cast<uint4*>(dst + c0) = v;
        }
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
  const uint64_t Bq = p.q_shared ? p.H : (uint64_t)p.B * p.H;
  const uint64_t Bk = (uint64_t)p.B * p.H;
  const uint64_t pitch = (uint64_t)DP * 2;
  CUtensorMap mq, mqt, mk, mkt, mv;
  int rc = make_tmap_3d(&mq, p.q, DP, p.Tq, Bq, pitch, pitch * p.Tq, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_3d(&mk, p.k, DP, p.Tk, Bk, pitch, pitch * p.Tk, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_3d(&mqt, p.q, DP, p.Tq, Bq, pitch, pitch * p.Tq, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  if (!rc) rc = make_tmap_3d(&mkt, p.k, DP, p.Tk, Bk, pitch, pitch * p.Tk, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  if (!rc) rc = make_tmap_3d(&mv, p.v, DP, p.Tk, Bk, pitch, pitch * p.Tk, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<DP, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  dim3 grid((p.Tq + NQ * 128 - 1) / (NQ * 128), p.H, p.B);
  attention_kernel<DP, NQ><<<grid, C::THREADS, C::SMEM, stream>>>(mq, mqt, mk, mkt, mv, p);
  return (int)cudaGetLastError();
}

}  // namespace

int attention_bf16(const AttnParams& p, cudaStream_t stream) {
  if (p.B <= 0 || p.H <= 0 || p.Tq <= 0 || p.Tk <= 0 || p.Dv <= 0 || p.Dv > p.Dp) return 1001;
  if ((p.ldo % 8) != 0 || (p.Dv % 8) != 0) return 1002;
  const bool two = p.Tq > 128;
  switch (p.Dp) {
    case 64: return two ? launch_attn<64, 2>(p, stream) : launch_attn<64, 1>(p, stream);
    case 80: return two ? launch_attn<80, 2>(p, stream) : launch_attn<80, 1>(p, stream);
    case 128: return launch_attn<128, 1>(p, stream);
    default: return 1004;
  }
}

}  // namespace epd
