// Encoder executor object behind the epd_encoder_* C ABI (see encoder.cu).
#pragma once

#include <cuda_runtime.h>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "epd.h"
#include "kernels.h"

namespace epd {

struct WeightSlot {
  std::string name;
  std::vector<int64_t> shape;
  std::vector<float> host;
  bool set = false;
};

struct LayerSlots {
  int ln1w = -1, ln1b = -1, qw = -1, qb = -1, kw = -1, kb = -1, vw = -1, vb = -1, ow = -1, ob = -1;
  int ls1 = -1, ln2w = -1, ln2b = -1, f1w = -1, f1b = -1, f2w = -1, f2b = -1, ls2 = -1;
};

// Device weight pointers; T = bf16 for the tensor-core path, float for the
// fp32 check mode (same B200 layouts, no rounding).
template <typename T>
struct LayerWT {
  T *ln1w = nullptr, *ln1b = nullptr, *qkv = nullptr, *qkvb = nullptr, *ow = nullptr, *ob = nullptr;
  T *ls1 = nullptr, *ln2w = nullptr, *ln2b = nullptr, *f1w = nullptr, *f1b = nullptr;
  T *f2w = nullptr, *f2b = nullptr, *ls2 = nullptr;
};
using LayerW = LayerWT<bf16>;

template <typename T>
struct GlobalWT {
  T *pe = nullptr, *pe_b = nullptr, *pos = nullptr, *post_w = nullptr, *post_b = nullptr;
  T *r_kv = nullptr, *r_lnkv_w = nullptr, *r_lnkv_b = nullptr, *r_kvin = nullptr, *r_kvin_b = nullptr;
  T *r_ow = nullptr, *r_ob = nullptr, *r_lnp_w = nullptr, *r_lnp_b = nullptr, *r_projT = nullptr;
  T *r_qheads = nullptr, *r_posk = nullptr;  // bf16: r_qheads row-major [Q][RH*RDp]
  T *m_ln_w = nullptr, *m_ln_b = nullptr, *m_f1w = nullptr, *m_f1b = nullptr, *m_f2w = nullptr,
    *m_f2b = nullptr;
  int32_t* ps_idx = nullptr;
};
using GlobalW = GlobalWT<bf16>;

struct Workspace {
  float* h = nullptr;  // fp32 residual stream
  bf16 *xp = nullptr, *xn = nullptr, *ao = nullptr, *qkv = nullptr, *f = nullptr;  // qkv: [M][3*H*dh]
  bf16 *r1 = nullptr, *r2 = nullptr, *rkv = nullptr, *rao = nullptr, *rr = nullptr;   // rkv: [M][2*RH*RDp]
};

// fp32 check-mode workspace (allocated on first use, chunks of f32_chunk tiles).
struct Workspace32 {
  float *xp = nullptr, *h = nullptr, *xn = nullptr, *ao = nullptr, *q = nullptr, *k = nullptr, *v = nullptr,
        *f = nullptr, *r2 = nullptr, *rk = nullptr, *rv = nullptr, *rao = nullptr, *rr = nullptr;
};

enum ProfClass : int { PROF_PATCHIFY = 0, PROF_GEMM = 1, PROF_ATTN = 2, PROF_LN = 3, PROF_OTHER = 4, PROF_NCLASS = 5 };

struct ProfRec {
  int cls;
  int ev;
  double flops;
  double bytes;
};

class Encoder {
 public:
  Encoder(const epd_encoder_desc_t& desc, int device);
  ~Encoder();
  std::string validate_and_build_schema();
  int finalize(cudaStream_t stream, std::string& err);
  int encode(const uint8_t* tiles, int n, bf16* out, cudaStream_t s, std::string& err);
  // fp32 check mode (enable before finalize): same pipeline on fp32 CUDA cores.
  int encode_f32(const uint8_t* tiles, int n, float* out, cudaStream_t s, std::string& err);
  bool check_f32 = false;
  int launches(int n) const;
  double flops_per_tile() const;
  int64_t numel(int i) const;
  int prof_read(double* ms, double* flops, double* bytes, int64_t* count, int nclass);
  // Per-launch records of the last drained profile: (class, ms, flops).
  struct ProfLaunch {
    int cls;
    float ms;
    double flops;
  };
  std::vector<ProfLaunch> prof_last;
  bool prof_on = false;
  bool use_graphs = true;

  epd_encoder_desc_t d;
  int dev;
  std::vector<WeightSlot> slots;
  bool finalized = false;

 private:
  int add(const std::string& name, std::vector<int64_t> shape);
  const float* host(int i) const;
  int forward_chunk(const uint8_t* tiles, int nt, bf16* out, cudaStream_t s);
  int forward_graph(const uint8_t* tiles, int nt, bf16* out, cudaStream_t s);
  int forward_f32(const uint8_t* tiles, int nt, float* out, cudaStream_t s);
  using GraphKey = std::tuple<int, const uint8_t*, bf16*>;  // chunk size, input, output
  std::map<GraphKey, cudaGraphExec_t> graphs;
  cudaStream_t cap_stream = nullptr;
  uint8_t* in_buf = nullptr;
  bf16* out_buf = nullptr;
  int prof_begin(cudaStream_t s);
  void prof_end(cudaStream_t s, int ev, int cls, double flops, double bytes);
  std::vector<cudaEvent_t> prof_events;
  size_t prof_used = 0;
  std::vector<ProfRec> prof_recs;

  // geometry
  int grid = 0, npatch = 0, T = 0, Tpad = 0, D = 0, H = 0, dh = 0, Dp = 0, F = 0;
  int Kreal = 0, Kpad = 0, E = 0, Q = 0, RH = 0, rdh = 0, RDp = 0;
  // schema indices
  int w_pe = -1, b_pe = -1, w_cls = -1, w_pos = -1, w_post_w = -1, w_post_b = -1;
  int r_query = -1, r_kv = -1, r_lnq_w = -1, r_lnq_b = -1, r_lnkv_w = -1, r_lnkv_b = -1;
  int r_qw = -1, r_qb = -1, r_kw = -1, r_kb = -1, r_vw = -1, r_vb = -1, r_ow = -1, r_ob = -1;
  int r_lnp_w = -1, r_lnp_b = -1, r_proj = -1, r_pos = -1;
  int m_ln_w = -1, m_ln_b = -1, m_f1w = -1, m_f1b = -1, m_f2w = -1, m_f2b = -1;
  std::vector<LayerSlots> lslots;
  // device state
  void* blob = nullptr;
  void* work = nullptr;
  GlobalW dw;
  std::vector<LayerW> dl;
  Workspace ws;
  // fp32 check mode state
  void* blob32 = nullptr;
  void* work32 = nullptr;
  int f32_chunk = 0;
  GlobalWT<float> dw32;
  std::vector<LayerWT<float>> dl32;
  Workspace32 ws32;
};

}  // namespace epd
