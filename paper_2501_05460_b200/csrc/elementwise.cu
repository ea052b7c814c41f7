// HBM-bound kernels: LayerNorm (warp per row, vectorised 16 B accesses,
// shuffle reductions), patchify (uint8 HWC tiles -> normalised bf16 im2col
// rows for the conv-as-GEMM patch embedding), record gather (MM-token
// packing) and the pixel-shuffle gather used by the InternVL projector.
#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "tmap.h"

namespace epd {

namespace {

// One warp per row; each lane holds up to MAXV 8-element vectors in registers.
// Optional row gather: logical row o = concat over seg of src rows
// gidx[o*segs + seg] (each D/segs wide) -- fuses the InternVL pixel shuffle.
template <typename Tin>
EPD_DEVICE void load_row8(const Tin* src, float* x);
template <>
EPD_DEVICE void load_row8<bf16>(const bf16* src, float* x) {
  uint4 u = *reinterpret_cast<const uint4*>(src);
  float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), c = unpack_bf16x2(u.z), d = unpack_bf16x2(u.w);
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
  x[4] = c.x; x[5] = c.y; x[6] = d.x; x[7] = d.y;
}
template <>
EPD_DEVICE void load_row8<float>(const float* src, float* x) {
  const float4 a = *reinterpret_cast<const float4*>(src);
  const float4 b = *reinterpret_cast<const float4*>(src + 4);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

template <int MAXV, typename Tin>
__global__ void __launch_bounds__(256) layernorm_kernel(const Tin* __restrict__ in, int ld_in,
                                                        bf16* __restrict__ out, int ld_out,
                                                        const bf16* __restrict__ gamma,
                                                        const bf16* __restrict__ beta, int rows,
                                                        int D, float eps,
                                                        const int32_t* __restrict__ gidx, int segs) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + warp;
  if (row >= rows) return;
  const int nvec = D >> 3;
  const int seg_vec = gidx ? nvec / segs : nvec;
  float x[MAXV][8];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int v = lane + i * 32;
    if (v < nvec) {
      const Tin* src;
      if (gidx) {
        const int seg = v / seg_vec;
        src = in + (size_t)gidx[(size_t)row * segs + seg] * ld_in + (v - seg * seg_vec) * 8;
      } else {
        src = in + (size_t)row * ld_in + v * 8;
      }
      load_row8<Tin>(src, x[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) sum += x[i][j];
    }
  }
  const float mean = warp_sum(sum) / (float)D;
  float var = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int v = lane + i * 32;
    if (v < nvec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float t = x[i][j] - mean;
        var += t * t;
      }
    }
  }
  const float rstd = rsqrtf(warp_sum(var) / (float)D + eps);
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int v = lane + i * 32;
    if (v < nvec) {
      float g[8], bb[8];
      uint4 ug = *reinterpret_cast<const uint4*>(gamma + v * 8);
      uint4 ub = *reinterpret_cast<const uint4*>(beta + v * 8);
      float2 t;
      t = unpack_bf16x2(ug.x); g[0] = t.x; g[1] = t.y;
      t = unpack_bf16x2(ug.y); g[2] = t.x; g[3] = t.y;
      t = unpack_bf16x2(ug.z); g[4] = t.x; g[5] = t.y;
      t = unpack_bf16x2(ug.w); g[6] = t.x; g[7] = t.y;
      t = unpack_bf16x2(ub.x); bb[0] = t.x; bb[1] = t.y;
      t = unpack_bf16x2(ub.y); bb[2] = t.x; bb[3] = t.y;
      t = unpack_bf16x2(ub.z); bb[4] = t.x; bb[5] = t.y;
      t = unpack_bf16x2(ub.w); bb[6] = t.x; bb[7] = t.y;
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = (x[i][j] - mean) * rstd * g[j] + bb[j];
      uint4 o;
      o.x = pack_bf16x2(y[0], y[1]);
      o.y = pack_bf16x2(y[2], y[3]);
      o.z = pack_bf16x2(y[4], y[5]);
      o.w = pack_bf16x2(y[6], y[7]);
      *reinterpret_cast<uint4*>(out + (size_t)row * ld_out + v * 8) = o;
    }
  }
}

// Residual-stream LayerNorm (fp32 in, bf16 out, no gather): gamma/beta are staged once
// per block in shared memory and the grid is one resident wave of warps striding over
// rows, so no row waits on a dependent gamma/beta load and there is no partial wave.
// RPW rows per warp are processed together (their loads in flight at once).
#ifndef EPD_LN_MINB
// Min resident 256-thread blocks per SM for the residual LayerNorm: 4 caps it at 64
// registers (32 warps in flight instead of 24 at 71 registers; the kernel is latency-bound):
// 12.3 -> 10.3 us per launch alone, LN share of the C2 step 0.94 -> 0.85 ms; 5 spills.
#define EPD_LN_MINB 4
#endif
template <int MAXV, int RPW>
__global__ void __launch_bounds__(256, EPD_LN_MINB) layernorm_resid_kernel(const float* __restrict__ in, int ld_in,
                                                              bf16* __restrict__ out, int ld_out,
                                                              const bf16* __restrict__ gamma,
                                                              const bf16* __restrict__ beta, int rows, int D,
                                                              float eps) {
  extern __shared__ uint4 gb[];  // [2][D/8] gamma then beta, 8 bf16 per uint4
  const int nvec = D >> 3;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    gb[i] = reinterpret_cast<const uint4*>(gamma)[i];
    gb[nvec + i] = reinterpret_cast<const uint4*>(beta)[i];
  }
  pdl_trigger();
  pdl_wait();  // gamma/beta are weights; the rows come from the previous kernel
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const float inv_d = 1.f / (float)D;
  for (int row0 = (blockIdx.x * wpb + warp) * RPW; row0 < rows; row0 += gridDim.x * wpb * RPW) {
    float x[RPW][MAXV][8];
    float sum[RPW];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
      sum[rr] = 0.f;
      const int row = row0 + rr;
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int v = lane + i * 32;
        if (v < nvec && row < rows) load_row8<float>(in + (size_t)row * ld_in + v * 8, x[rr][i]);
      }
    }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
      for (int i = 0; i < MAXV; ++i)
        if (lane + i * 32 < nvec)
#pragma unroll
          for (int j = 0; j < 8; ++j) sum[rr] += x[rr][i][j];
    float mean[RPW], var[RPW];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
      mean[rr] = warp_sum(sum[rr]) * inv_d;
      var[rr] = 0.f;
#pragma unroll
      for (int i = 0; i < MAXV; ++i)
        if (lane + i * 32 < nvec)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float t = x[rr][i][j] - mean[rr];
            var[rr] += t * t;
          }
    }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
      const int row = row0 + rr;
      const float rstd = rsqrtf(warp_sum(var[rr]) * inv_d + eps);
      if (row >= rows) continue;
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int v = lane + i * 32;
        if (v < nvec) {
          const uint4 ug = gb[v], ub = gb[nvec + v];
          const uint32_t gw[4] = {ug.x, ug.y, ug.z, ug.w}, bw[4] = {ub.x, ub.y, ub.z, ub.w};
          uint32_t o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 g2 = unpack_bf16x2(gw[j]), b2 = unpack_bf16x2(bw[j]);
            o[j] = pack_bf16x2((x[rr][i][2 * j] - mean[rr]) * rstd * g2.x + b2.x,
                               (x[rr][i][2 * j + 1] - mean[rr]) * rstd * g2.y + b2.y);
          }
          *reinterpret_cast<uint4*>(out + (size_t)row * ld_out + v * 8) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
    }
  }
}

// One block per (tile, patch row). Stage p image rows in smem, then emit
// S/p patches x Kpad columns in (c, ky, kx) order.
// uint8 HWC tiles -> normalized bf16 im2col rows (K padded to Kpad, zeros beyond C*p*p).
// One block per (tile, strip of p image rows): the strip is staged in shared memory with
// 16-byte loads, a per-block table maps each of the Kpad columns to its strip offset and
// channel, and every thread emits 8 consecutive columns as one 16-byte store.
__global__ void __launch_bounds__(256) patchify_kernel(const uint8_t* __restrict__ tiles, int S, int C, int p,
                                                     int Kpad, int row_offset, int rows_per_tile, float m0,
                                                     float m1, float m2, float s0, float s1, float s2,
                                                     bf16* __restrict__ out) {
  extern __shared__ uint8_t strip[];  // p * S * C bytes, then Kpad int32 column offsets
  const size_t strip_bytes = (size_t)p * S * C;
  int32_t* tab = reinterpret_cast<int32_t*>(strip + ((strip_bytes + 15) & ~size_t(15)));
  const int kreal = C * p * p;
  for (int col = threadIdx.x; col < Kpad; col += blockDim.x) {
    int t = -1;
    if (col < kreal) {
      const int c = col / (p * p);
      const int r = col - c * p * p;
      const int ky = r / p, kx = r - ky * p;
      t = ((ky * S + kx) * C + c) | (c << 28);  // strip offset (< 2^28) and channel
    }
    tab[col] = t;
  }
  pdl_trigger();
  pdl_wait();
  const int tile = blockIdx.y;
  const int py = blockIdx.x;
  const int np = S / p;
  const uint8_t* src = tiles + (size_t)tile * S * S * C + (size_t)py * strip_bytes;
  for (size_t i = threadIdx.x * 16; i < strip_bytes; i += blockDim.x * 16) {
    if (i + 16 <= strip_bytes && ((reinterpret_cast<uintptr_t>(src + i) & 15) == 0))
      *reinterpret_cast<uint4*>(strip + i) = *reinterpret_cast<const uint4*>(src + i);
    else
      for (size_t j = i; j < i + 16 && j < strip_bytes; ++j) strip[j] = src[j];
  }
  __syncthreads();
  const float mean[3] = {m0, m1, m2};
  const float inv[3] = {1.f / s0, 1.f / s1, 1.f / s2};
  const int kv = Kpad >> 3;
  bf16* dst = out + ((size_t)tile * rows_per_tile + row_offset + (size_t)py * np) * Kpad;
  for (int o = threadIdx.x; o < np * kv; o += blockDim.x) {
    const int px = o / kv;
    const int c8 = (o - px * kv) * 8;
    const uint8_t* sp = strip + px * p * C;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = tab[c8 + j];
      v[j] = 0.f;
      if (t >= 0) {
        const int c = t >> 28;
        v[j] = ((float)sp[t & 0x0FFFFFFF] * (1.f / 255.f) - mean[c]) * inv[c];
      }
    }
    *reinterpret_cast<uint4*>(dst + (size_t)o * 8) =
        make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
  }
}

__global__ void gather_records_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ index,
                                      int n, size_t vecs, uint4* __restrict__ dst) {
  const int rec = blockIdx.y;
  const uint4* s = src + (size_t)index[rec] * vecs;
  uint4* d = dst + (size_t)rec * vecs;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < vecs;
       i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

}  // namespace

template <typename Tin>
int layernorm_any(const Tin* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                  const bf16* beta, int rows, int D, float eps, const int32_t* gidx,
                  int segs, cudaStream_t stream) {
  if (rows <= 0) return 0;
  if (D % 8 || ld_in % 8 || ld_out % 8) return 1002;
  if (gidx && (segs <= 0 || (D / 8) % segs)) return 1002;
  const int nvec = D / 8;
  const dim3 block(256);
  const dim3 grid((rows + 7) / 8);
  if (nvec <= 32 * 5)
    return launch_kernel(layernorm_kernel<5, Tin>, grid, block, 0, stream, 1, in, ld_in, out, ld_out, gamma, beta, rows,
                         D, eps, gidx, segs);
  else if (nvec <= 32 * 16)
    return launch_kernel(layernorm_kernel<16, Tin>, grid, block, 0, stream, 1, in, ld_in, out, ld_out, gamma, beta,
                         rows, D, eps, gidx, segs);
  return 1004;
}

int layernorm_bf16_gather(const bf16* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                          const bf16* beta, int rows, int D, float eps, const int32_t* gidx,
                          int segs, cudaStream_t stream) {
  return layernorm_any<bf16>(in, ld_in, out, ld_out, gamma, beta, rows, D, eps, gidx, segs, stream);
}

#ifndef EPD_LN_RPW
#define EPD_LN_RPW 1
#endif

template <int MAXV, int RPW>
int launch_ln_resid(const float* in, int ld_in, bf16* out, int ld_out, const bf16* gamma, const bf16* beta,
                    int rows, int D, float eps, cudaStream_t stream) {
  auto k = layernorm_resid_kernel<MAXV, RPW>;
  const size_t smem = (size_t)2 * D * 2;
  static int resident = 0;  // blocks per SM at this register/smem footprint
  if (!resident) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k, 256, smem);
    if (resident < 1) resident = 1;
  }
  const int need = (rows + 8 * RPW - 1) / (8 * RPW);
  const int grid = need < resident * num_sms() ? need : resident * num_sms();
  return launch_kernel(k, dim3(grid), dim3(256), smem, stream, 1, in, ld_in, out, ld_out, gamma, beta, rows, D, eps);
}

int layernorm_f32in(const float* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                    const bf16* beta, int rows, int D, float eps, const int32_t* gidx, int segs,
                    cudaStream_t stream) {
#if EPD_LN_RPW > 0
  if (!gidx && D % 8 == 0 && ld_in % 4 == 0 && ld_out % 8 == 0 && rows > 0 && D / 8 <= 32 * 5)
    return launch_ln_resid<5, EPD_LN_RPW>(in, ld_in, out, ld_out, gamma, beta, rows, D, eps, stream);
#endif
  return layernorm_any<float>(in, ld_in, out, ld_out, gamma, beta, rows, D, eps, gidx, segs, stream);
}

int layernorm_bf16(const bf16* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                   const bf16* beta, int rows, int D, float eps, cudaStream_t stream) {
  return layernorm_bf16_gather(in, ld_in, out, ld_out, gamma, beta, rows, D, eps, nullptr, 1, stream);
}

int patchify_u8(const uint8_t* tiles, int n, int S, int C, int p, int Kpad, int row_offset,
                int rows_per_tile, const float* mean, const float* stdv, bf16* out,
                cudaStream_t stream) {
  if (n <= 0) return 0;
  if (S % p || C > 3 || Kpad < C * p * p || Kpad % 8) return 1002;
  const size_t smem = (((size_t)p * S * C + 15) & ~size_t(15)) + (size_t)Kpad * 4;
  dim3 grid(S / p, n);
  return launch_kernel(patchify_kernel, grid, dim3(256), smem, stream, 1, tiles, S, C, p, Kpad, row_offset,
                       rows_per_tile, mean[0], C > 1 ? mean[1] : 0.f, C > 2 ? mean[2] : 0.f, stdv[0],
                       C > 1 ? stdv[1] : 1.f, C > 2 ? stdv[2] : 1.f, out);
}

int gather_records(const void* src_base, const int32_t* index, int n, size_t bytes, void* dst,
                   cudaStream_t stream) {
  if (n <= 0) return 0;
  if (bytes % 16 || (reinterpret_cast<uintptr_t>(src_base) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return 1002;
  const size_t vecs = bytes / 16;
  int bx = (int)((vecs + 255) / 256);
  if (bx > 64) bx = 64;
  dim3 grid(bx, n);
  gather_records_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const uint4*>(src_base), index, n,
                                                  vecs, reinterpret_cast<uint4*>(dst));
  return (int)cudaGetLastError();
}

}  // namespace epd
