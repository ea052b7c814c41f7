// Internal (C++) launch interface of the sm_100a kernels. The public, C-ABI
// surface lives in include/epd.h and csrc/capi.cu; nothing here crosses the
// shared-library boundary.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace epd {

using bf16 = __nv_bfloat16;

enum EpiMode : int { EPI_ROWS = 0, EPI_HEADS = 1 };
// ACT_SWIGLU: the weight rows come in 32-row groups alternating gate / up (group g of the
// output = rows [64g, 64g+32) gate, [64g+32, 64g+64) up); the GEMM writes
// silu(gate + b) * (up + b) to N/2 bf16 output columns (no residual / layer scale).
enum Act : int { ACT_NONE = 0, ACT_GELU_TANH = 1, ACT_GELU_ERF = 2, ACT_SWIGLU = 3 };

// Epilogue of C = A[M,K] * B[N,K]^T, fused on the TMEM accumulator:
//   x = act(acc + bias[n]);  if (resid) x = resid[row % r_mod][n] + lscale[n] * x
// EPI_ROWS : out[row * ldo + n] = x
// EPI_HEADS: column n splits into section s = n / sec_cols (q/k/v), head
//   h = (n % sec_cols) / Dp, dim d = n % Dp; row = b * T + t. Section s writes
//   sec_out[s][((b*H + h)*T + t)*Dp + d]            (sec_trans[s] == 0)
//   sec_out[s][((b*H + h)*Dp + d)*Tpad + t]         (sec_trans[s] == 1, keys-major V^T)
struct EpiParams {
  int mode = EPI_ROWS;
  int act = ACT_NONE;
  const bf16* bias = nullptr;
  const bf16* resid = nullptr;
  int ldr = 0;
  int r_mod = 0x7fffffff;
  const bf16* lscale = nullptr;
  const float* resid_f = nullptr;  // fp32 residual stream (takes precedence over resid)
  bf16* out = nullptr;
  float* out_f = nullptr;          // fp32 output (takes precedence over out)
  int ldo = 0;
  int H = 0, Dp = 0, T = 0, Tpad = 0, sec_cols = 0;
  bf16* sec_out[3] = {nullptr, nullptr, nullptr};
  int sec_trans[3] = {0, 0, 0};
  // fp32 reduce-add only: allow splitting K over up to max_split work items per output tile
  // (chosen when the tiles alone leave SMs idle). The splits add into the output in a fixed
  // order (run-to-run deterministic), but the split count depends on M, so results are not
  // batch invariant -- the encoder never sets it.
  int max_split = 0;
  int ksplit = 1;        // internal: chosen split count
  int* split_flags = nullptr;  // internal: per (tile, epilogue warp) progress counters
};

// Returns a cudaError_t-compatible code (0 = success); 1000+ for argument errors.
// GEMM CTA-group policy for subsequent launches: 0 auto, 1 single CTAs, 2 CTA pairs.
void set_gemm_cta_group(int policy);
int gemm_bf16(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
              const EpiParams& ep, cudaStream_t stream, int bn_hint = 0);

// Fused multi-head attention O = softmax(Q K^T * scale) V on tcgen05, reading Q, K, V
// straight from row-major projection outputs (no per-head relayout):
//   Q : q[(b * Tq + t) * ldq + h * hs + d]      (q_shared: q[t * ldq + h * hs + d])
//   K : k[(b * Tk + t) * ldk + (h / kv_group) * hs + d]
//   V : v[(b * Tk + t) * ldv + (h / kv_group) * hs + d]        for d < Dv
//   O : out[(b * Tq + t) * ldo + h * Dv + d]      for d < Dv
// hs = column stride between heads (Dv for packed heads). The MMAs run Dp = Dv rounded up
// to a multiple of 16 (64, 80 or 128) dims: dims beyond Dv read the neighbouring head's
// columns (or TMA zero fill past the last head); the kernel zeroes Q's dims >= Dv, so S is
// exact, and O's dims >= Dv are never stored. ld* * 2 bytes and the pointers must be
// 16-byte aligned.
struct AttnParams {
  const bf16* q = nullptr;
  const bf16* k = nullptr;
  const bf16* v = nullptr;
  bf16* out = nullptr;
  int ldq = 0, ldk = 0, ldv = 0, hs = 0;
  int B = 0, H = 0, Tq = 0, Tk = 0, Dp = 0, Dv = 0, ldo = 0;
  int q_shared = 0;
  float scale = 1.f;
  int causal = 0;    // query row t (of Tq) sees keys <= t + (Tk - Tq)
  int kv_group = 1;  // query heads per K/V head (grouped-query attention): K/V head = h / kv_group
};
int attention_bf16(const AttnParams& p, cudaStream_t stream);

// Row-wise LayerNorm over D (bf16 in/out, fp32 statistics), optional fused
// residual-free affine (gamma, beta). in/out may alias. Rows are contiguous
// with stride ld (elements).
int layernorm_bf16(const bf16* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                   const bf16* beta, int rows, int D, float eps, cudaStream_t stream);
// Same, but logical row o is the concatenation of `segs` source rows
// gidx[o*segs + s] (each D/segs wide, pitch ld_in): fuses a row gather such
// as the InternVL pixel shuffle into the normalisation.
// fp32-input variant (the residual stream is kept in fp32).
int layernorm_f32in(const float* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                    const bf16* beta, int rows, int D, float eps, const int32_t* gidx, int segs,
                    cudaStream_t stream);
int layernorm_bf16_gather(const bf16* in, int ld_in, bf16* out, int ld_out, const bf16* gamma,
                          const bf16* beta, int rows, int D, float eps, const int32_t* gidx,
                          int segs, cudaStream_t stream);

// uint8 HWC tiles [n][S][S][C] -> normalized bf16 patch rows
// [n*(S/p)^2 (+cls)][Kpad] (im2col of the conv-as-GEMM patch embedding).
// Column order = (c, ky, kx) to match Conv2d weight.view(D, C*p*p).
// Normalization: x = (u8 / 255 - mean[c]) / std[c].
int patchify_u8(const uint8_t* tiles, int n, int S, int C, int p, int Kpad, int row_offset,
                int rows_per_tile, const float* mean, const float* stdv, bf16* out,
                cudaStream_t stream);

// Gather equal-sized byte records: dst[i] = src_base[index[i]] (record = bytes).
// EP gather over NVLink peer memory (peer.cu): 16 B copy into a (possibly peer-mapped)
// destination + system fence, then *flag = value (release, system scope) when flag != 0.
int peer_put(const void* src, void* dst, size_t bytes, uint32_t* flag, uint32_t value, cudaStream_t s);
int peer_signal(uint32_t* flag, uint32_t value, cudaStream_t s);
// The stream waits until *flag >= value (cuStreamWaitValue32, GEQ; flag in local memory).
int stream_wait_geq(const uint32_t* flag, uint32_t value, cudaStream_t s);

int gather_records(const void* src_base, const int32_t* index, int n, size_t bytes, void* dst,
                   cudaStream_t stream);

// ---- prefill consumer (llm.cu): the LLM layers around the GEMM / attention kernels.
int rmsnorm_f32(const float* in, int ld_in, bf16* out, int ld_out, const bf16* gamma, int rows, int D, float eps,
                cudaStream_t s);
int rope_bf16(bf16* x, int ld, int rows, int col0, int nheads, int hd, int pos0, float theta, const float* cs,
              cudaStream_t s);
int rope_table(float* cs, int rows, int hd, int pos0, float theta, cudaStream_t s);
int silu_mul_bf16(const bf16* gu, int ld_in, bf16* out, int ld_out, int rows, int F, cudaStream_t s);
int kv_write_paged(const bf16* src, int ld_src, int v_off, int rows, int row_elems, const int32_t* block_ids,
                   int block_size, bf16* pool, size_t seg_elems, int seg0, cudaStream_t s);
int gather_rows_f32(const bf16* src, int ld_src, const int32_t* index, int rows, int D, float* dst, int ld_dst,
                    cudaStream_t s);
int argmax_bf16(const bf16* x, int n, int32_t* out, cudaStream_t s);

// ---- device block free list (blocks.cu): LIFO ids as blocks.py hands them out.
int blocks_init(int32_t* stack, int32_t* top, int total, cudaStream_t s);
int blocks_alloc(int32_t* stack, int32_t* top, int need, int32_t* out, cudaStream_t s);
int blocks_free(int32_t* stack, int32_t* top, const int32_t* ids, int n, cudaStream_t s);

// ---- image tiling (tiler.cu): grid tiles of the image resized to (cols*S, rows*S) plus an
// optional S x S thumbnail (first or last), antialiased bilinear, uint8 HWC.
int tile_image_u8(const uint8_t* src, int H, int W, int C, int cols, int rows, int thumb, int thumb_first, int S,
                  uint8_t* out, cudaStream_t s);

// ---- fp32 check mode (check_f32.cu): CUDA-core fp32 twins of the kernels above.
// Epilogue: x = act(acc + bias[n]) * lscale[n] + resid[row % r_mod][n]; ROWS writes
// (or, with accumulate, adds to) out[row*ldo + n]; HEADS scatters like EpiParams
// (natural [b*H+h][T][Dp] layout for every section).
struct EpiF32 {
  int mode = EPI_ROWS;
  int act = ACT_NONE;
  const float* bias = nullptr;
  const float* lscale = nullptr;
  const float* resid = nullptr;
  int ldr = 0;
  int r_mod = 0x7fffffff;
  int accumulate = 0;
  float* out = nullptr;
  int ldo = 0;
  int H = 0, Dp = 0, T = 0, sec_cols = 0;
  float* sec_out[3] = {nullptr, nullptr, nullptr};
  int dh = 0;  // head width of the columns (0 = Dp): dims [0, dh) of each Dp-wide head
};
int gemm_f32(const float* A, int lda, const float* W, int ldw, int M, int N, int K, const EpiF32& ep,
             cudaStream_t s);
int attention_f32(const float* q, const float* k, const float* v, float* out, int B, int H, int Tq, int Tk,
                  int Dp, int Dv, int ldo, int q_shared, float scale, cudaStream_t s);
int layernorm_f32_check(const float* in, int ld_in, float* out, int ld_out, const float* gamma,
                        const float* beta, int rows, int D, float eps, const int32_t* gidx, int segs,
                        cudaStream_t s);
int patchify_f32(const uint8_t* tiles, int n, int S, int C, int p, int Kdim, int row_offset, int rows_per_tile,
                 const float* mean, const float* stdv, float* out, cudaStream_t s);

}  // namespace epd
