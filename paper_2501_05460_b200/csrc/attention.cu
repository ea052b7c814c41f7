// Fused multi-head attention (bidirectional, no causal mask) for sm_100a.
//
// One CTA = 128 query rows of one (batch, head). Per 128-key block j:
//   S_j  = Q K_j^T           tcgen05.mma, M=128 N=128 K=Dp, fp32 in TMEM
//   P_j  = exp2(S_j*c - m_j) softmax warps: TMEM -> regs -> bf16 P in smem (SW128)
//   O_j  = P_j V_j           tcgen05.mma, M=128 N=Dp K=128, fp32 in TMEM
//   acc  = acc*alpha_j + O_j softmax warps, fp32 registers (online softmax)
// S_{j+1} is issued before O_j so the tensor core overlaps the softmax.
//
// Roles (192 threads): warp 0 TMA, warp 1 TMEM alloc + MMA issue, warps 2..5 softmax.
// Head dims that are not a multiple of 64 (SigLIP 72 -> padded 80) are split
// into a 64-wide 128B-swizzled atom plus a 16-wide 32B-swizzled atom.
#include "common.cuh"
#include "kernels.h"
#include "tmap.h"

namespace epd {

namespace {

template <int DP>
struct AttnCfg {
  static constexpr int QROWS = 128;
  static constexpr int KB = 128;  // keys per block
  static constexpr bool TAIL32 = (DP % 64) != 0;          // 16-wide 32B-swizzled tail atom
  static constexpr int MAIN_ATOMS = DP / 64;              // full 64-wide SW128 atoms
  static constexpr int QK_ATOM_BYTES = 128 * 128;         // 128 rows x 128 B
  static constexpr int QK_TAIL_BYTES = TAIL32 ? 128 * 32 : 0;
  static constexpr int QK_BYTES = MAIN_ATOMS * QK_ATOM_BYTES + QK_TAIL_BYTES;  // = 128*DP*2
  static constexpr int QK_BYTES_AL = (QK_BYTES + 1023) / 1024 * 1024;
  static constexpr int V_ATOM_BYTES = DP * 128;           // DP rows x 64 keys x 2 B
  static constexpr int V_BYTES = 2 * V_ATOM_BYTES;
  static constexpr int P_ATOM_BYTES = 128 * 128;
  static constexpr int P_BYTES = 2 * P_ATOM_BYTES;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + QK_BYTES_AL;
  static constexpr int OFF_V = OFF_K + 2 * QK_BYTES_AL;
  static constexpr int OFF_P = OFF_V + 2 * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS_QK = DP / 16;
};

template <int DP>
__global__ void __launch_bounds__(192, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQt,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKt,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = AttnCfg<DP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sP = smem + C::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_free = bars + 11;  // [2]
  uint64_t* p_full = bars + 13;  // [2]
  uint64_t* p_free = bars + 15;  // [2]
  uint64_t* o_full = bars + 17;  // [2]
  uint64_t* o_free = bars + 19;  // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 21);

  const int warp = warp_id();
  const int lane = lane_id();
  const int qtile = blockIdx.x;
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int bh = b * p.H + h;
  const int qbatch = p.q_shared ? h : bh;
  const int q0 = qtile * C::QROWS;
  const int nkb = (p.Tk + C::KB - 1) / C::KB;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&p_free[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // TMEM columns: S buffers at [0,128) and [128,256); O buffers at 256 and 384.

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, C::QK_BYTES);
      for (int a = 0; a < C::MAIN_ATOMS; ++a)
        tma_load_3d(sQ + a * C::QK_ATOM_BYTES, &tmQ, q_full, a * 64, q0, qbatch);
      if (C::TAIL32) tma_load_3d(sQ + C::MAIN_ATOMS * C::QK_ATOM_BYTES, &tmQt, q_full, C::MAIN_ATOMS * 64, q0, qbatch);
      for (int j = 0; j < nkb; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[s], C::QK_BYTES);
        uint8_t* kd = sK + s * C::QK_BYTES_AL;
        for (int a = 0; a < C::MAIN_ATOMS; ++a)
          tma_load_3d(kd + a * C::QK_ATOM_BYTES, &tmK, &k_full[s], a * 64, j * C::KB, bh);
        if (C::TAIL32) tma_load_3d(kd + C::MAIN_ATOMS * C::QK_ATOM_BYTES, &tmKt, &k_full[s], C::MAIN_ATOMS * 64, j * C::KB, bh);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[s], C::V_BYTES);
        uint8_t* vd = sV + s * C::V_BYTES;
        tma_load_3d(vd, &tmV, &v_full[s], j * C::KB, 0, bh);
        tma_load_3d(vd + C::V_ATOM_BYTES, &tmV, &v_full[s], j * C::KB + 64, 0, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, C::KB);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DP);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_full[s], ph);
        mbar_wait(&s_free[s], ph ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * C::QK_BYTES_AL);
#pragma unroll
        for (int kk = 0; kk < C::KSTEPS_QK; ++kk) {
          const int atom = kk >> 2;
          uint64_t ad, bd;
          if (atom < C::MAIN_ATOMS) {
            ad = make_sdesc(q_addr + atom * C::QK_ATOM_BYTES + (kk & 3) * 32, 1024, 2);
            bd = make_sdesc(k_addr + atom * C::QK_ATOM_BYTES + (kk & 3) * 32, 1024, 2);
          } else {
            ad = make_sdesc(q_addr + C::MAIN_ATOMS * C::QK_ATOM_BYTES, 256, 6);
            bd = make_sdesc(k_addr + C::MAIN_ATOMS * C::QK_ATOM_BYTES, 256, 6);
          }
          umma_bf16(tmem + s * 128, ad, bd, idesc_s, kk != 0);
        }
        tc_commit(&s_full[s]);
        tc_commit(&k_empty[s]);
      };
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) issue_s(j + 1);
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&p_full[s], ph);
        mbar_wait(&v_full[s], ph);
        mbar_wait(&o_free[s], ph ^ 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sP + s * C::P_BYTES);
        const uint32_t v_addr = smem_u32(sV + s * C::V_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int atom = kk >> 2;
          const uint64_t ad = make_sdesc(p_addr + atom * C::P_ATOM_BYTES + (kk & 3) * 32, 1024, 2);
          const uint64_t bd = make_sdesc(v_addr + atom * C::V_ATOM_BYTES + (kk & 3) * 32, 1024, 2);
          umma_bf16(tmem + 256 + s * 128, ad, bd, idesc_o, kk != 0);
        }
        tc_commit(&o_full[s]);
        tc_commit(&v_empty[s]);
        tc_commit(&p_free[s]);
      }
    }
  } else {
    // ---------------- softmax / correction warps: one query row per thread
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
    const float c = p.scale * 1.4426950408889634f;
    float m = -INFINITY, l = 0.f, alpha_pend = 0.f;
    float acc[DP];
#pragma unroll
    for (int i = 0; i < DP; ++i) acc[i] = 0.f;

    auto consume_o = [&](int j, float alpha) {
      const int s = j & 1;
      mbar_wait(&o_full[s], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < DP; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + 256 + s * 128 + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[c0 + i] = acc[c0 + i] * alpha + __uint_as_float(v[i]);
      }
      tc_fence_before();
      mbar_arrive(&o_free[s]);
    };

    for (int j = 0; j < nkb; ++j) {
      const int s = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      const int kvalid = p.Tk - j * C::KB;  // keys >= kvalid are padding
      mbar_wait(&s_full[s], ph);
      tc_fence_after();
      const uint32_t sbase = tmem + lane_off + s * 128;
      float mx = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(sbase + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < kvalid) mx = fmaxf(mx, __uint_as_float(v[i]));
      }
      const float m_new = fmaxf(m, mx * c);
      const float alpha = exp2f(m - m_new);  // 0 on the first block
      mbar_wait(&p_free[s], ph ^ 1);
      float rs = 0.f;
      uint8_t* prow = sP + s * C::P_BYTES + r * 128;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(sbase + c0, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float e0 = (c0 + i < kvalid) ? exp2f(__uint_as_float(v[i]) * c - m_new) : 0.f;
          const float e1 = (c0 + i + 1 < kvalid) ? exp2f(__uint_as_float(v[i + 1]) * c - m_new) : 0.f;
          rs += e0 + e1;
          pk[i >> 1] = pack_bf16x2(e0, e1);
        }
        const int atom = c0 >> 6;
        uint8_t* arow = prow + atom * C::P_ATOM_BYTES;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int chunk = ((c0 & 63) >> 3) + q4;  // 16-byte chunk within the 128 B row
          const int phys = chunk ^ (r & 7);
          *reinterpret_cast<uint4*>(arow + phys * 16) =
              make_uint4(pk[q4 * 4 + 0], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_free[s]);
      fence_proxy_async_smem();
      mbar_arrive(&p_full[s]);
      l = l * alpha + rs;
      m = m_new;
      if (j >= 1) consume_o(j - 1, alpha_pend);
      alpha_pend = alpha;
    }
    consume_o(nkb - 1, alpha_pend);

    const int qrow = q0 + r;
    if (qrow < p.Tq) {
      const float inv = 1.f / l;
      bf16* dst = p.out + ((size_t)b * p.Tq + qrow) * p.ldo + (size_t)h * p.Dv;
#pragma unroll
      for (int d = 0; d < DP; d += 8) {
        if (d < p.Dv) {
          uint4 v;
          v.x = pack_bf16x2(acc[d + 0] * inv, acc[d + 1] * inv);
          v.y = pack_bf16x2(acc[d + 2] * inv, acc[d + 3] * inv);
          v.z = pack_bf16x2(acc[d + 4] * inv, acc[d + 5] * inv);
          v.w = pack_bf16x2(acc[d + 6] * inv, acc[d + 7] * inv);
          *reinterpret_cast<uint4*>(dst + d) = v;
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

template <int DP>
int launch_attn(const AttnParams& p, cudaStream_t stream) {
  using C = AttnCfg<DP>;
  const int Bq = p.q_shared ? p.H : p.B * p.H;
  CUtensorMap mq, mqt, mk, mkt, mv;
  const uint64_t qk_pitch1 = (uint64_t)DP * 2;
  int rc = make_tmap_3d(&mq, p.q, DP, p.Tq, Bq, qk_pitch1, qk_pitch1 * p.Tq, 64, 128, 1,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_3d(&mk, p.k, DP, p.Tk, (uint64_t)p.B * p.H, qk_pitch1, qk_pitch1 * p.Tk,
                             64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc && C::TAIL32) {
    rc = make_tmap_3d(&mqt, p.q, DP, p.Tq, Bq, qk_pitch1, qk_pitch1 * p.Tq, 16, 128, 1,
                      CU_TENSOR_MAP_SWIZZLE_32B);
    if (!rc) rc = make_tmap_3d(&mkt, p.k, DP, p.Tk, (uint64_t)p.B * p.H, qk_pitch1,
                               qk_pitch1 * p.Tk, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    mqt = mq;
    mkt = mk;
  }
  if (!rc) rc = make_tmap_3d(&mv, p.vt, p.Tk, DP, (uint64_t)p.B * p.H, (uint64_t)p.Tkpad * 2,
                             (uint64_t)p.Tkpad * 2 * DP, 64, DP, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<DP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  dim3 grid((p.Tq + 127) / 128, p.H, p.B);
  attention_kernel<DP><<<grid, 192, C::SMEM, stream>>>(mq, mqt, mk, mkt, mv, p);
  return (int)cudaGetLastError();
}

}  // namespace

int attention_bf16(const AttnParams& p, cudaStream_t stream) {
  if (p.B <= 0 || p.H <= 0 || p.Tq <= 0 || p.Tk <= 0 || p.Dv <= 0 || p.Dv > p.Dp) return 1001;
  if (p.Tkpad < p.Tk || (p.Tkpad % 8) != 0 || (p.ldo % 8) != 0 || (p.Dv % 8) != 0) return 1002;
  switch (p.Dp) {
    case 64: return launch_attn<64>(p, stream);
    case 80: return launch_attn<80>(p, stream);
    case 128: return launch_attn<128>(p, stream);
    default: return 1004;
  }
}

}  // namespace epd
