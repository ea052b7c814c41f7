// Prefill-side kernels for the LLM consumer of the packed MM tokens (SURVEY.md 8(f)
// item 1): the decoder layers reuse the tcgen05 GEMM and attention kernels; these are
// the HBM/L2-bound pieces around them. All rows are row-major with explicit pitches.
#include "common.cuh"
#include "kernels.h"

namespace epd {

namespace {

// RMSNorm of fp32 rows into bf16: y = x * rsqrt(mean(x^2) + eps) * gamma. One block of
// 256 threads per row, the row held in registers (VPT float4 per thread: D <= 4096).
template <int VPT>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ in, int ld_in,
                                                      bf16* __restrict__ out, int ld_out,
                                                      const bf16* __restrict__ gamma, int D, float eps) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const float* x = in + (size_t)row * ld_in;
  float4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = (threadIdx.x + i * 256) * 4;
    v[i] = c < D ? *reinterpret_cast<const float4*>(x + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = threadIdx.x < 8 ? red[threadIdx.x] : 0.f;
  if (threadIdx.x < 32) {
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)D + eps);
  bf16* y = out + (size_t)row * ld_out;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = (threadIdx.x + i * 256) * 4;
    if (c < D) {
      const float2 g01 = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(gamma + c));
      const float2 g23 = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(gamma + c + 2));
      uint2 o;
      o.x = pack_bf16x2(v[i].x * r * g01.x, v[i].y * r * g01.y);
      o.y = pack_bf16x2(v[i].z * r * g23.x, v[i].w * r * g23.y);
      *reinterpret_cast<uint2*>(y + c) = o;
    }
  }
}

// Rotary position embedding, rotate-half convention (Qwen2 / InternLM2): for head dims
// i < hd/2, (x_i, x_{i+hd/2}) <- (x_i cos - x_{i+hd/2} sin, x_{i+hd/2} cos + x_i sin),
// angle = pos * theta^(-2i/hd), pos = pos0 + row. In place on heads [0, nheads) starting at
// column col0 of each row. cs (optional): precomputed [rows][hd/2] (cos, sin) pairs for
// positions pos0.. -- the prefill builds it once per prompt length.
__global__ void rope_kernel(bf16* __restrict__ x, int ld, int rows, int col0, int nheads, int hd, int pos0,
                            float log2_theta, const float2* __restrict__ cs) {
  const int half = hd >> 1;
  const size_t total = (size_t)rows * nheads * half;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(i % half);
    const size_t rh = i / half;
    const int h = (int)(rh % nheads);
    const int row = (int)(rh / nheads);
    float s, c;
    if (cs) {
      const float2 t = cs[(size_t)row * half + d];
      c = t.x;
      s = t.y;
    } else {
      const float inv_freq = exp2f(-log2_theta * (2.f * d) / (float)hd);
      sincosf((float)(pos0 + row) * inv_freq, &s, &c);
    }
    bf16* p = x + (size_t)row * ld + col0 + h * hd + d;
    const float a = __bfloat162float(p[0]), b = __bfloat162float(p[half]);
    p[0] = __float2bfloat16_rn(a * c - b * s);
    p[half] = __float2bfloat16_rn(b * c + a * s);
  }
}

// Same rotation, 8 head dims per thread: 16-byte loads/stores of x (and 64 bytes of the
// cos/sin table), 32-bit index math. Per element the arithmetic is rope_kernel's.
__global__ void rope8_kernel(bf16* __restrict__ x, int ld, int rows, int col0, int nheads, int hd, int pos0,
                             float log2_theta, const float2* __restrict__ cs) {
  const int half = hd >> 1, hv = half >> 3;
  const int total = rows * nheads * hv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % hv;
    const int rh = i / hv;
    const int h = rh % nheads;
    const int row = rh / nheads;
    const int d0 = g * 8;
    float c[8], sn[8];
    if (cs) {
      const float4* t = reinterpret_cast<const float4*>(cs + (size_t)row * half + d0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = t[q];
        c[2 * q] = v.x;
        sn[2 * q] = v.y;
        c[2 * q + 1] = v.z;
        sn[2 * q + 1] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float inv_freq = exp2f(-log2_theta * (2.f * (d0 + j)) / (float)hd);
        sincosf((float)(pos0 + row) * inv_freq, &sn[j], &c[j]);
      }
    }
    bf16* p = x + (size_t)row * ld + col0 + h * hd + d0;
    uint4 ua = *reinterpret_cast<const uint4*>(p), ub = *reinterpret_cast<const uint4*>(p + half);
    const uint32_t aw[4] = {ua.x, ua.y, ua.z, ua.w}, bw[4] = {ub.x, ub.y, ub.z, ub.w};
    uint32_t oa[4], ob[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 a = unpack_bf16x2(aw[q]), b = unpack_bf16x2(bw[q]);
      const int j = 2 * q;
      oa[q] = pack_bf16x2(a.x * c[j] - b.x * sn[j], a.y * c[j + 1] - b.y * sn[j + 1]);
      ob[q] = pack_bf16x2(b.x * c[j] + a.x * sn[j], b.y * c[j + 1] + a.y * sn[j + 1]);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
    *reinterpret_cast<uint4*>(p + half) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
  }
}

__global__ void rope_table_kernel(float2* __restrict__ cs, int rows, int hd, int pos0, float log2_theta) {
  const int half = hd >> 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * half; i += gridDim.x * blockDim.x) {
    const int d = i % half, row = i / half;
    const float inv_freq = exp2f(-log2_theta * (2.f * d) / (float)hd);
    float s, c;
    sincosf((float)(pos0 + row) * inv_freq, &s, &c);
    cs[i] = make_float2(c, s);
  }
}

// SwiGLU: out[r][c] = silu(gu[r][c]) * gu[r][F + c] (gate | up halves of one GEMM output).
__global__ void silu_mul_kernel(const bf16* __restrict__ gu, int ld_in, bf16* __restrict__ out, int ld_out,
                                int rows, int F) {
  const int vecs = F / 8;
  const size_t total = (size_t)rows * vecs;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vecs);
    const size_t r = i / vecs;
    const uint4 g = *reinterpret_cast<const uint4*>(gu + r * ld_in + v * 8);
    const uint4 u = *reinterpret_cast<const uint4*>(gu + r * ld_in + F + v * 8);
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w}, uw[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 a = unpack_bf16x2(gw[j]), b = unpack_bf16x2(uw[j]);
      o[j] = pack_bf16x2(a.x / (1.f + __expf(-a.x)) * b.x, a.y / (1.f + __expf(-a.y)) * b.y);
    }
    *reinterpret_cast<uint4*>(out + r * ld_out + v * 8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Paged KV write: row t's `row_elems` values at src + t*ld_src (+ seg_stride_src for the
// second segment, V) go to block block_ids[t / block_size], slot t % block_size of segment
// seg0 (K) and seg0 + 1 (V) of the pool [segments][num_blocks][block_size * row_elems].
__global__ void kv_write_kernel(const bf16* __restrict__ src, int ld_src, int v_off, int rows, int row_elems,
                                const int32_t* __restrict__ block_ids, int block_size, bf16* __restrict__ pool,
                                size_t seg_elems, int seg0) {
  const int vecs = row_elems / 8;
  const size_t total = (size_t)rows * vecs * 2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vecs);
    const size_t rs = i / vecs;
    const int kv = (int)(rs & 1);
    const int t = (int)(rs >> 1);
    const uint4 val = *reinterpret_cast<const uint4*>(src + (size_t)t * ld_src + kv * v_off + v * 8);
    const size_t blk = (size_t)block_ids[t / block_size];
    bf16* dst = pool + (size_t)(seg0 + kv) * seg_elems + (blk * block_size + t % block_size) * row_elems + v * 8;
    *reinterpret_cast<uint4*>(dst) = val;
  }
}

// dst[r][:] = float(src[index[r]][:]) (D % 4 == 0): MM tokens / embedding rows into the
// fp32 residual stream.
__global__ void gather_rows_f32_kernel(const bf16* __restrict__ src, int ld_src, const int32_t* __restrict__ index,
                                       int rows, int D, float* __restrict__ dst, int ld_dst) {
  const int vecs = D / 4;
  const size_t total = (size_t)rows * vecs;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vecs);
    const size_t r = i / vecs;
    const uint2 u = *reinterpret_cast<const uint2*>(src + (size_t)index[r] * ld_src + v * 4);
    const float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y);
    *reinterpret_cast<float4*>(dst + r * ld_dst + v * 4) = make_float4(a.x, a.y, b.x, b.y);
  }
}

// argmax over n bf16 values (first index on ties), one block.
__global__ void __launch_bounds__(1024) argmax_kernel(const bf16* __restrict__ x, int n, int32_t* __restrict__ out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  float best = -INFINITY;
  int bi = 0x7fffffff;
  // 16-byte loads (8 values) while the pointer is 16-byte aligned; each thread walks its
  // chunks in increasing index order, so within a thread the first index wins ties
  const int head = (int)(((16 - (reinterpret_cast<uintptr_t>(x) & 15)) & 15) / 2);
  const int h = head < n ? head : n;
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const float v = __bfloat162float(x[i]);
    if (v > best) { best = v; bi = i; }
  }
  const int nv = (n - h) / 8;
  const uint4* xv = reinterpret_cast<const uint4*>(x + h);
  for (int k = threadIdx.x; k < nv; k += blockDim.x) {
    const uint4 u = xv[k];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(w[j]);
      const int i = h + k * 8 + 2 * j;
      if (f.x > best) { best = f.x; bi = i; }
      if (f.y > best) { best = f.y; bi = i + 1; }
    }
  }
  for (int i = h + nv * 8 + threadIdx.x; i < n; i += blockDim.x) {
    const float v = __bfloat162float(x[i]);
    if (v > best) { best = v; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? sv[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (threadIdx.x == 0) *out = bi;
  }
}

int grid_for(size_t work) {
  size_t g = (work + 255) / 256;
  return (int)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}

}  // namespace

int rmsnorm_f32(const float* in, int ld_in, bf16* out, int ld_out, const bf16* gamma, int rows, int D, float eps,
                cudaStream_t s) {
  if (rows <= 0) return 0;
  if (D % 4 || ld_in % 4 || ld_out % 4 || D > 4096) return 1002;
  if (D <= 2048)
    rmsnorm_kernel<2><<<rows, 256, 0, s>>>(in, ld_in, out, ld_out, gamma, D, eps);
  else
    rmsnorm_kernel<4><<<rows, 256, 0, s>>>(in, ld_in, out, ld_out, gamma, D, eps);
  return (int)cudaGetLastError();
}

int rope_bf16(bf16* x, int ld, int rows, int col0, int nheads, int hd, int pos0, float theta, const float* cs,
              cudaStream_t s) {
  if (rows <= 0) return 0;
  if (hd % 2 || theta <= 1.f) return 1002;
  const bool vec = hd % 16 == 0 && ld % 8 == 0 && col0 % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (!cs || (reinterpret_cast<uintptr_t>(cs) & 15) == 0) && (size_t)rows * nheads * hd < (1u << 31);
  if (vec)
    rope8_kernel<<<grid_for((size_t)rows * nheads * (hd / 16)), 256, 0, s>>>(
        x, ld, rows, col0, nheads, hd, pos0, log2f(theta), reinterpret_cast<const float2*>(cs));
  else
    rope_kernel<<<grid_for((size_t)rows * nheads * (hd / 2)), 256, 0, s>>>(
        x, ld, rows, col0, nheads, hd, pos0, log2f(theta), reinterpret_cast<const float2*>(cs));
  return (int)cudaGetLastError();
}

int rope_table(float* cs, int rows, int hd, int pos0, float theta, cudaStream_t s) {
  if (rows <= 0) return 0;
  if (hd % 2 || theta <= 1.f) return 1002;
  rope_table_kernel<<<grid_for((size_t)rows * hd / 2), 256, 0, s>>>(reinterpret_cast<float2*>(cs), rows, hd, pos0,
                                                                    log2f(theta));
  return (int)cudaGetLastError();
}

int silu_mul_bf16(const bf16* gu, int ld_in, bf16* out, int ld_out, int rows, int F, cudaStream_t s) {
  if (rows <= 0) return 0;
  if (F % 8 || ld_in % 8 || ld_out % 8) return 1002;
  silu_mul_kernel<<<grid_for((size_t)rows * F / 8), 256, 0, s>>>(gu, ld_in, out, ld_out, rows, F);
  return (int)cudaGetLastError();
}

int kv_write_paged(const bf16* src, int ld_src, int v_off, int rows, int row_elems, const int32_t* block_ids,
                   int block_size, bf16* pool, size_t seg_elems, int seg0, cudaStream_t s) {
  if (rows <= 0) return 0;
  if (row_elems % 8 || ld_src % 8 || v_off % 8 || block_size <= 0) return 1002;
  kv_write_kernel<<<grid_for((size_t)rows * row_elems / 4), 256, 0, s>>>(src, ld_src, v_off, rows, row_elems,
                                                                         block_ids, block_size, pool, seg_elems, seg0);
  return (int)cudaGetLastError();
}

int gather_rows_f32(const bf16* src, int ld_src, const int32_t* index, int rows, int D, float* dst, int ld_dst,
                    cudaStream_t s) {
  if (rows <= 0) return 0;
  if (D % 4 || ld_src % 4 || ld_dst % 4) return 1002;
  gather_rows_f32_kernel<<<grid_for((size_t)rows * D / 4), 256, 0, s>>>(src, ld_src, index, rows, D, dst, ld_dst);
  return (int)cudaGetLastError();
}

int argmax_bf16(const bf16* x, int n, int32_t* out, cudaStream_t s) {
  if (n <= 0) return 1001;
  argmax_kernel<<<1, 1024, 0, s>>>(x, n, out);
  return (int)cudaGetLastError();
}

}  // namespace epd
