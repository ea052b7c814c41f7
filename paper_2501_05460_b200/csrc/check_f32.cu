// fp32 check mode: plain CUDA-core (SIMT) fp32 kernels that run the encoder
// pipeline with the same B200 weight layouts (head padding, fused QKV, folded
// position terms, pixel-shuffle gather) but without bf16 rounding anywhere.
// Not a performance path: it exists so the layout transforms and fusions of the
// tensor-core path can be checked against the fp32 CPU oracle at 1e-4.
#include "common.cuh"
#include "kernels.h"

namespace epd {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

// C = A[M,K] W[N,K]^T with the fused epilogue of EpiF32 (16x16 threads, 4x4 outputs each).
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int lda,
                                                       const float* __restrict__ W, int ldw, int M, int N,
                                                       int K, EpiF32 ep) {
  __shared__ float As[TK][TM + 1];
  __shared__ float Ws[TK][TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      const int mm = i / TK, kk = i % TK;
      As[kk][mm] = (m0 + mm < M && k0 + kk < K) ? A[(size_t)(m0 + mm) * lda + k0 + kk] : 0.f;
      Ws[kk][mm] = (n0 + mm < N && k0 + kk < K) ? W[(size_t)(n0 + mm) * ldw + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col >= N) continue;
      float x = acc[i][j];
      if (ep.bias) x += ep.bias[col];
      if (ep.act == ACT_GELU_TANH) x = gelu_tanh(x);
      else if (ep.act == ACT_GELU_ERF) x = gelu_erf(x);
      if (ep.lscale) x *= ep.lscale[col];
      if (ep.resid) x += ep.resid[(size_t)(row % ep.r_mod) * ep.ldr + col];
      if (ep.mode == EPI_ROWS) {
        float* o = ep.out + (size_t)row * ep.ldo + col;
        *o = ep.accumulate ? *o + x : x;
      } else {
        const int s = col / ep.sec_cols;
        const int within = col - s * ep.sec_cols;
        const int hw = ep.dh ? ep.dh : ep.Dp;
        const int h = within / hw, d = within - h * hw;
        const int b = row / ep.T, t = row - b * ep.T;
        ep.sec_out[s][(((size_t)b * ep.H + h) * ep.T + t) * ep.Dp + d] = x;
      }
    }
  }
}

// One warp per query row: scores in smem, exact softmax, then P V with lanes over dims.
__global__ void __launch_bounds__(128) attention_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                            const float* __restrict__ v, float* __restrict__ out,
                                                            int H, int Tq, int Tk, int Dp, int Dv, int ldo,
                                                            int q_shared, float scale) {
  extern __shared__ float sc[];  // [4 warps][Tk]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qi = blockIdx.x * 4 + warp;
  const int h = blockIdx.y, b = blockIdx.z;
  if (qi >= Tq) return;
  const size_t bh = (size_t)b * H + h;
  const float* qr = q + ((q_shared ? (size_t)h : bh) * Tq + qi) * Dp;
  const float* kb = k + bh * Tk * Dp;
  const float* vb = v + bh * Tk * Dp;
  float* s = sc + warp * Tk;
  float mx = -INFINITY;
  for (int key = lane; key < Tk; key += 32) {
    float d = 0.f;
    for (int j = 0; j < Dv; ++j) d = fmaf(qr[j], kb[(size_t)key * Dp + j], d);
    d *= scale;
    s[key] = d;
    mx = fmaxf(mx, d);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int key = lane; key < Tk; key += 32) {
    const float e = expf(s[key] - mx);
    s[key] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.f / sum;
  for (int d = lane; d < Dv; d += 32) {
    float o = 0.f;
    for (int key = 0; key < Tk; ++key) o = fmaf(s[key], vb[(size_t)key * Dp + d], o);
    out[((size_t)b * Tq + qi) * ldo + (size_t)h * Dv + d] = o * inv;
  }
}

// LayerNorm fp32 -> fp32, one warp per row (two-pass in registers via smem-free loops),
// optional row gather (pixel shuffle): logical row o = concat of gidx[o*segs + s].
__global__ void __launch_bounds__(128) layernorm_f32_kernel(const float* __restrict__ in, int ld_in,
                                                            float* __restrict__ out, int ld_out,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta, int rows, int D,
                                                            float eps, const int32_t* __restrict__ gidx, int segs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + warp;
  if (row >= rows) return;
  const int seg_w = gidx ? D / segs : D;
  auto at = [&](int c) -> float {
    if (!gidx) return in[(size_t)row * ld_in + c];
    const int sg = c / seg_w;
    return in[(size_t)gidx[(size_t)row * segs + sg] * ld_in + (c - sg * seg_w)];
  };
  double sum = 0.0;
  for (int c = lane; c < D; c += 32) sum += at(c);
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = (float)(sum / D);
  double var = 0.0;
  for (int c = lane; c < D; c += 32) {
    const float t = at(c) - mean;
    var += (double)t * t;
  }
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float rstd = (float)(1.0 / sqrt(var / D + eps));
  for (int c = lane; c < D; c += 32) out[(size_t)row * ld_out + c] = (at(c) - mean) * rstd * gamma[c] + beta[c];
}

__global__ void patchify_f32_kernel(const uint8_t* __restrict__ tiles, int n, int S, int C, int p, int Kdim,
                                    int row_offset, int rows_per_tile, float m0, float m1, float m2, float s0,
                                    float s1, float s2, float* __restrict__ out) {
  const int np = S / p;
  const size_t total = (size_t)n * np * np * Kdim;
  const float mean[3] = {m0, m1, m2}, stdv[3] = {s0, s1, s2};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int col = (int)(i % Kdim);
    const size_t pr = i / Kdim;
    const int tile = (int)(pr / (np * np));
    const int pi = (int)(pr % (np * np));
    const int py = pi / np, px = pi % np;
    float x = 0.f;  // columns past C*p*p pad K to the GEMM tile
    if (col < C * p * p) {
      const int c = col / (p * p), rr = col % (p * p), ky = rr / p, kx = rr % p;
      const float u = tiles[(((size_t)tile * S + py * p + ky) * S + px * p + kx) * C + c];
      x = (u / 255.f - mean[c]) / stdv[c];
    }
    out[((size_t)tile * rows_per_tile + row_offset + pi) * Kdim + col] = x;
  }
}

}  // namespace

int gemm_f32(const float* A, int lda, const float* W, int ldw, int M, int N, int K, const EpiF32& ep,
             cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0) return 1001;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
  gemm_f32_kernel<<<grid, 256, 0, s>>>(A, lda, W, ldw, M, N, K, ep);
  return (int)cudaGetLastError();
}

int attention_f32(const float* q, const float* k, const float* v, float* out, int B, int H, int Tq, int Tk, int Dp,
                  int Dv, int ldo, int q_shared, float scale, cudaStream_t s) {
  const size_t smem = 4 * (size_t)Tk * sizeof(float);
  if (smem > 200 * 1024) return 1004;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid((Tq + 3) / 4, H, B);
  attention_f32_kernel<<<grid, 128, smem, s>>>(q, k, v, out, H, Tq, Tk, Dp, Dv, ldo, q_shared, scale);
  return (int)cudaGetLastError();
}

int layernorm_f32_check(const float* in, int ld_in, float* out, int ld_out, const float* gamma, const float* beta,
                        int rows, int D, float eps, const int32_t* gidx, int segs, cudaStream_t s) {
  if (rows <= 0) return 0;
  layernorm_f32_kernel<<<(rows + 3) / 4, 128, 0, s>>>(in, ld_in, out, ld_out, gamma, beta, rows, D, eps, gidx,
                                                      segs);
  return (int)cudaGetLastError();
}

int patchify_f32(const uint8_t* tiles, int n, int S, int C, int p, int Kdim, int row_offset, int rows_per_tile,
                 const float* mean, const float* stdv, float* out, cudaStream_t s) {
  if (n <= 0) return 0;
  patchify_f32_kernel<<<1184, 256, 0, s>>>(tiles, n, S, C, p, Kdim, row_offset, rows_per_tile, mean[0],
                                           C > 1 ? mean[1] : 0.f, C > 2 ? mean[2] : 0.f, stdv[0],
                                           C > 1 ? stdv[1] : 1.f, C > 2 ? stdv[2] : 1.f, out);
  return (int)cudaGetLastError();
}

}  // namespace epd
