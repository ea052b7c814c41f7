// Vision encoder + resampler/projector executor (host C++ driving the sm_100a
// kernels). Owns the bf16 weights in the B200 layout and the activation
// workspace; one instance per GPU process.
//
// Families (public model definitions restated in oracle/encoders.py):
//   1  MiniCPM-V 2.6: SigLIP-so400m ViT (pre-LN, GELU-tanh, post-LN)
//      + perceiver resampler (kv_proj, ln_kv, 64 learned queries, MHA with
//        2-D sincos key positions, ln_post, proj)
//   2  InternVL2: InternViT-300M (CLS token, layer scale, GELU-erf, no post-LN)
//      + pixel shuffle 0.5 + mlp1 (LN, Linear, GELU, Linear)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "encoder.h"
#include "kernels.h"
#include "launch.h"
#include "tmap.h"

namespace epd {

// Largest chunk whose forward is launched with PDL in auto mode (launch.h): every chunk size
// since round 2 (same-box A/B, profiles/r02/ab.txt: 1-3 tile shards 4-6 % faster, C5 +0.9 %,
// C2 +0.2 %; round 1's erratic C5 under PDL was the attention barrier-region overlap, since fixed).
constexpr int kPdlMaxTiles = 1 << 30;

namespace {

uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

Encoder::Encoder(const epd_encoder_desc_t& desc, int device) : d(desc), dev(device) {}

Encoder::~Encoder() {
  if (blob) cudaFree(blob);
  if (work) cudaFree(work);
  if (blob32) cudaFree(blob32);
  if (work32) cudaFree(work32);
  for (auto e : prof_events) cudaEventDestroy(e);
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  if (cap_stream) cudaStreamDestroy(cap_stream);
}

int Encoder::add(const std::string& name, std::vector<int64_t> shape) {
  WeightSlot s;
  s.name = name;
  s.shape = std::move(shape);
  slots.push_back(std::move(s));
  return (int)slots.size() - 1;
}

int64_t Encoder::numel(int i) const {
  int64_t n = 1;
  for (auto v : slots[i].shape) n *= v;
  return n;
}

std::string Encoder::validate_and_build_schema() {
  const auto& x = d;
  if (x.family != EPD_FAMILY_SIGLIP_RESAMPLER && x.family != EPD_FAMILY_INTERNVIT_MLP)
    return "unknown encoder family";
  if (x.image_size <= 0 || x.patch_size <= 0 || x.image_size % x.patch_size)
    return "image_size must be a positive multiple of patch_size";
  if (x.channels < 1 || x.channels > 3) return "channels must be 1..3";
  if (x.hidden <= 0 || x.heads <= 0 || x.hidden % x.heads) return "hidden must divide into heads";
  if (x.hidden % 8 || x.mlp % 8 || x.out_dim % 8) return "hidden, mlp and out_dim must be multiples of 8";
  if (x.layers < 0 || x.max_tiles <= 0) return "layers >= 0 and max_tiles > 0 required";
  grid = x.image_size / x.patch_size;
  npatch = grid * grid;
  D = x.hidden;
  H = x.heads;
  dh = D / H;
  Dp = dh <= 64 ? 64 : (dh <= 80 ? 80 : (dh <= 128 ? 128 : 0));
  if (!Dp) return "head_dim > 128 is not supported";
  if (dh % 8) return "head_dim must be a multiple of 8";
  Kreal = x.channels * x.patch_size * x.patch_size;
  Kpad = (Kreal + 63) / 64 * 64;
  F = x.mlp;
  if (x.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    T = npatch;
    E = x.out_dim;
    Q = x.out_tokens;
    if (x.out_heads <= 0 || E % x.out_heads) return "out_dim must divide into out_heads";
    RH = x.out_heads;
    rdh = E / RH;
    RDp = rdh <= 64 ? 64 : (rdh <= 80 ? 80 : (rdh <= 128 ? 128 : 0));
    if (!RDp || rdh % 8) return "resampler head_dim must be a multiple of 8 and <= 128";
  } else {
    T = npatch + 1;
    E = x.out_dim;
    if (grid % 2) return "pixel shuffle needs an even patch grid";
    Q = npatch / 4;
    if (x.out_tokens != Q) return "InternVL out_tokens must equal (grid/2)^2";
  }
  Tpad = (T + 7) / 8 * 8;

  const int L = x.layers;
  w_pe = add("patch_embed.weight", {D, x.channels, x.patch_size, x.patch_size});
  b_pe = add("patch_embed.bias", {D});
  if (x.family == EPD_FAMILY_INTERNVIT_MLP) w_cls = add("cls_token", {D});
  w_pos = add("pos_embed", {T, D});
  for (int l = 0; l < L; ++l) {
    LayerSlots ls;
    const std::string p = "layers." + std::to_string(l) + ".";
    ls.ln1w = add(p + "ln1.weight", {D});
    ls.ln1b = add(p + "ln1.bias", {D});
    if (x.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
      ls.qw = add(p + "attn.q.weight", {D, D});
      ls.qb = add(p + "attn.q.bias", {D});
      ls.kw = add(p + "attn.k.weight", {D, D});
      ls.kb = add(p + "attn.k.bias", {D});
      ls.vw = add(p + "attn.v.weight", {D, D});
      ls.vb = add(p + "attn.v.bias", {D});
    } else {
      ls.qw = add(p + "attn.qkv.weight", {3 * D, D});
      ls.qb = add(p + "attn.qkv.bias", {3 * D});
    }
    ls.ow = add(p + "attn.o.weight", {D, D});
    ls.ob = add(p + "attn.o.bias", {D});
    if (x.family == EPD_FAMILY_INTERNVIT_MLP) ls.ls1 = add(p + "ls1", {D});
    ls.ln2w = add(p + "ln2.weight", {D});
    ls.ln2b = add(p + "ln2.bias", {D});
    ls.f1w = add(p + "mlp.fc1.weight", {F, D});
    ls.f1b = add(p + "mlp.fc1.bias", {F});
    ls.f2w = add(p + "mlp.fc2.weight", {D, F});
    ls.f2b = add(p + "mlp.fc2.bias", {D});
    if (x.family == EPD_FAMILY_INTERNVIT_MLP) ls.ls2 = add(p + "ls2", {D});
    lslots.push_back(ls);
  }
  if (x.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    w_post_w = add("post_ln.weight", {D});
    w_post_b = add("post_ln.bias", {D});
    r_query = add("rs.query", {Q, E});
    r_kv = add("rs.kv_proj.weight", {E, D});
    r_lnq_w = add("rs.ln_q.weight", {E});
    r_lnq_b = add("rs.ln_q.bias", {E});
    r_lnkv_w = add("rs.ln_kv.weight", {E});
    r_lnkv_b = add("rs.ln_kv.bias", {E});
    r_qw = add("rs.attn.q.weight", {E, E});
    r_qb = add("rs.attn.q.bias", {E});
    r_kw = add("rs.attn.k.weight", {E, E});
    r_kb = add("rs.attn.k.bias", {E});
    r_vw = add("rs.attn.v.weight", {E, E});
    r_vb = add("rs.attn.v.bias", {E});
    r_ow = add("rs.attn.o.weight", {E, E});
    r_ob = add("rs.attn.o.bias", {E});
    r_lnp_w = add("rs.ln_post.weight", {E});
    r_lnp_b = add("rs.ln_post.bias", {E});
    r_proj = add("rs.proj", {E, E});
    r_pos = add("rs.pos_embed", {T, E});
  } else {
    const int C4 = 4 * D;
    m_ln_w = add("mlp1.ln.weight", {C4});
    m_ln_b = add("mlp1.ln.bias", {C4});
    m_f1w = add("mlp1.fc1.weight", {E, C4});
    m_f1b = add("mlp1.fc1.bias", {E});
    m_f2w = add("mlp1.fc2.weight", {E, E});
    m_f2b = add("mlp1.fc2.bias", {E});
  }
  return "";
}

const float* Encoder::host(int i) const { return slots[i].host.data(); }

// ------------------------------------------------------------ finalize

namespace {

struct Arena {
  uint8_t* base = nullptr;
  size_t off = 0, cap = 0;
  void* take(size_t bytes) {
    void* p = base + off;
    off += align256(bytes);
    return p;
  }
};

}  // namespace

int Encoder::finalize(cudaStream_t stream, std::string& err) {
  for (size_t i = 0; i < slots.size(); ++i)
    if (!slots[i].set) {
      err = "weight not set: " + slots[i].name;
      return EPD_ERR_VALUE;
    }
  // ---- build the device images on the host (B200 layouts). Each image is
  // uploaded as bf16 and, in fp32 check mode, also as an fp32 twin.
  struct Image {
    bf16** dst;
    float** dst32;
    std::vector<float> v;
  };
  std::vector<Image> images;
  auto plain = [&](bf16** dst, float** dst32, int slot) {
    images.push_back({dst, dst32, std::vector<float>(host(slot), host(slot) + numel(slot))});
  };
  auto transposed = [&](bf16** dst, float** dst32, int slot, int rows, int cols) {  // out[c][r] = in[r][c]
    std::vector<float> v((size_t)rows * cols);
    const float* h = host(slot);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) v[(size_t)c * rows + r] = h[(size_t)r * cols + c];
    images.push_back({dst, dst32, std::move(v)});
  };
  // head-padded projection rows: sections s (source slot, row offset), heads nh of dim hd -> pad hp
  auto headpad_w = [&](bf16** dst, float** dst32, const std::vector<std::pair<int, int>>& secs, int nh, int hd,
                       int hp, int K) {
    std::vector<float> v((size_t)secs.size() * nh * hp * K, 0.f);
    for (size_t s = 0; s < secs.size(); ++s) {
      const float* h = host(secs[s].first) + (size_t)secs[s].second * K;
      for (int hh = 0; hh < nh; ++hh)
        for (int dd = 0; dd < hd; ++dd) {
          const float* src = h + (size_t)(hh * hd + dd) * K;
          std::copy(src, src + K, v.data() + ((s * nh + hh) * (size_t)hp + dd) * K);
        }
    }
    images.push_back({dst, dst32, std::move(v)});
  };
  auto headpad_b = [&](bf16** dst, float** dst32, const std::vector<std::pair<int, int>>& secs, int nh, int hd,
                       int hp) {
    std::vector<float> v((size_t)secs.size() * nh * hp, 0.f);
    for (size_t s = 0; s < secs.size(); ++s) {
      const float* h = host(secs[s].first) + secs[s].second;
      for (int hh = 0; hh < nh; ++hh)
        for (int dd = 0; dd < hd; ++dd) v[(s * nh + hh) * hp + dd] = h[hh * hd + dd];
    }
    images.push_back({dst, dst32, std::move(v)});
  };
#define EPD_G(field) &dw.field, &dw32.field
#define EPD_L(field) &o.field, &o32.field

  // patch embedding [D][C*p*p] padded to Kpad columns
  {
    std::vector<float> v((size_t)D * Kpad, 0.f);
    const float* h = host(w_pe);
    for (int r = 0; r < D; ++r) std::copy(h + (size_t)r * Kreal, h + (size_t)(r + 1) * Kreal, v.data() + (size_t)r * Kpad);
    images.push_back({EPD_G(pe), std::move(v)});
  }
  plain(EPD_G(pe_b), b_pe);
  {
    // additive table applied in the patch-embed epilogue as resid[row % T]:
    // rows carry the position embedding; InternViT's CLS row (whose patch row
    // is zero, so the GEMM yields just the bias) carries cls + pos0 - bias.
    std::vector<float> pos(host(w_pos), host(w_pos) + (size_t)T * D);
    if (d.family == EPD_FAMILY_INTERNVIT_MLP)
      for (int c = 0; c < D; ++c) pos[c] += host(w_cls)[c] - host(b_pe)[c];
    images.push_back({EPD_G(pos), std::move(pos)});
  }
  dl.resize(lslots.size());
  dl32.resize(lslots.size());
  for (size_t l = 0; l < lslots.size(); ++l) {
    const auto& s = lslots[l];
    auto& o = dl[l];
    auto& o32 = dl32[l];
    plain(EPD_L(ln1w), s.ln1w);
    plain(EPD_L(ln1b), s.ln1b);
    // Fused QKV [3*H*dh, D] with packed heads: the projection computes no padding and
    // writes row-major [M][3*H*dh]; attention reads its heads in place.
    if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
      headpad_w(EPD_L(qkv), {{s.qw, 0}, {s.kw, 0}, {s.vw, 0}}, H, dh, dh, D);
      headpad_b(EPD_L(qkvb), {{s.qb, 0}, {s.kb, 0}, {s.vb, 0}}, H, dh, dh);
    } else {
      headpad_w(EPD_L(qkv), {{s.qw, 0}, {s.qw, D}, {s.qw, 2 * D}}, H, dh, dh, D);
      headpad_b(EPD_L(qkvb), {{s.qb, 0}, {s.qb, D}, {s.qb, 2 * D}}, H, dh, dh);
    }
    plain(EPD_L(ow), s.ow);
    plain(EPD_L(ob), s.ob);
    plain(EPD_L(ln2w), s.ln2w);
    plain(EPD_L(ln2b), s.ln2b);
    plain(EPD_L(f1w), s.f1w);
    plain(EPD_L(f1b), s.f1b);
    plain(EPD_L(f2w), s.f2w);
    plain(EPD_L(f2b), s.f2b);
    if (d.family == EPD_FAMILY_INTERNVIT_MLP) {
      plain(EPD_L(ls1), s.ls1);
      plain(EPD_L(ls2), s.ls2);
    }
  }
  // inputs of the weight-only precomputations below (bf16 and fp32 twins)
  struct RsTmp {
    bf16 *query = nullptr, *lnq_w = nullptr, *lnq_b = nullptr, *qw = nullptr, *qb = nullptr, *kw = nullptr,
         *pos = nullptr;
  } rs;
  struct RsTmp32 {
    float *query = nullptr, *lnq_w = nullptr, *lnq_b = nullptr, *qw = nullptr, *qb = nullptr, *kw = nullptr,
          *pos = nullptr;
  } rs32;
#define EPD_R(field) &rs.field, &rs32.field
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    plain(EPD_G(post_w), w_post_w);
    plain(EPD_G(post_b), w_post_b);
    plain(EPD_G(r_kv), r_kv);
    plain(EPD_G(r_lnkv_w), r_lnkv_w);
    plain(EPD_G(r_lnkv_b), r_lnkv_b);
    headpad_w(EPD_G(r_kvin), {{r_kw, 0}, {r_vw, 0}}, RH, rdh, RDp, E);
    headpad_b(EPD_G(r_kvin_b), {{r_kb, 0}, {r_vb, 0}}, RH, rdh, RDp);
    plain(EPD_G(r_ow), r_ow);
    plain(EPD_G(r_ob), r_ob);
    plain(EPD_G(r_lnp_w), r_lnp_w);
    plain(EPD_G(r_lnp_b), r_lnp_b);
    transposed(EPD_G(r_projT), r_proj, E, E);
    plain(EPD_R(query), r_query);
    plain(EPD_R(lnq_w), r_lnq_w);
    plain(EPD_R(lnq_b), r_lnq_b);
    headpad_w(EPD_R(qw), {{r_qw, 0}}, RH, rdh, RDp, E);
    headpad_b(EPD_R(qb), {{r_qb, 0}}, RH, rdh, RDp);
    headpad_w(EPD_R(kw), {{r_kw, 0}}, RH, rdh, RDp, E);
    plain(EPD_R(pos), r_pos);
  } else {
    plain(EPD_G(m_ln_w), m_ln_w);
    plain(EPD_G(m_ln_b), m_ln_b);
    plain(EPD_G(m_f1w), m_f1w);
    plain(EPD_G(m_f1b), m_f1b);
    plain(EPD_G(m_f2w), m_f2w);
    plain(EPD_G(m_f2b), m_f2b);
  }
#undef EPD_G
#undef EPD_L
#undef EPD_R

  // ---- derived device tensors and workspace sizes
  const size_t nt = d.max_tiles;
  const size_t M = nt * T;
  size_t derived = 0;
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    derived += align256((size_t)RH * Q * RDp * 2);            // q heads
    derived += align256((size_t)T * 2 * RH * RDp * 2);        // pos_k table
  } else {
    derived += align256(nt * Q * 4 * sizeof(int32_t));        // pixel-shuffle gather index
  }
  size_t wbytes = derived, wbytes32 = 0;
  for (auto& im : images) wbytes += align256(im.v.size() * 2);
  if (check_f32) {
    wbytes32 = derived * 2;
    for (auto& im : images) wbytes32 += align256(im.v.size() * 4);
  }
  cudaError_t e = cudaMalloc(&blob, wbytes);
  if (e == cudaSuccess && check_f32) e = cudaMalloc(&blob32, wbytes32);
  if (e != cudaSuccess) {
    err = std::string("cudaMalloc(weights): ") + cudaGetErrorString(e);
    return EPD_ERR_CUDA;
  }
  Arena a{reinterpret_cast<uint8_t*>(blob), 0, wbytes};
  Arena a32{reinterpret_cast<uint8_t*>(blob32), 0, wbytes32};
  for (auto& im : images) {
    std::vector<uint16_t> hb(im.v.size());
    for (size_t i = 0; i < hb.size(); ++i) hb[i] = f2bf(im.v[i]);
    void* p = a.take(hb.size() * 2);
    e = cudaMemcpy(p, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
    *im.dst = reinterpret_cast<bf16*>(p);
    if (e == cudaSuccess && check_f32) {
      void* p32 = a32.take(im.v.size() * 4);
      e = cudaMemcpy(p32, im.v.data(), im.v.size() * 4, cudaMemcpyHostToDevice);
      *im.dst32 = reinterpret_cast<float*>(p32);
    }
    if (e != cudaSuccess) {
      err = std::string("cudaMemcpy(weights): ") + cudaGetErrorString(e);
      return EPD_ERR_CUDA;
    }
    std::vector<float>().swap(im.v);
  }
  if (check_f32 && d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    dw32.r_qheads = reinterpret_cast<float*>(a32.take((size_t)RH * Q * RDp * 4));
    dw32.r_posk = reinterpret_cast<float*>(a32.take((size_t)T * 2 * RH * RDp * 4));
  }
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    dw.r_qheads = reinterpret_cast<bf16*>(a.take((size_t)RH * Q * RDp * 2));
    dw.r_posk = reinterpret_cast<bf16*>(a.take((size_t)T * 2 * RH * RDp * 2));
  } else {
    dw.ps_idx = reinterpret_cast<int32_t*>(a.take(nt * Q * 4 * sizeof(int32_t)));
    // InternVL pixel_shuffle(0.5), ps_version v2, after dropping CLS:
    // out token (a2, b2), channel segment s <- patch (2*a2 + s/2, 2*b2 + s%2)
    std::vector<int32_t> idx(nt * Q * 4);
    const int g2 = grid / 2;
    for (size_t t = 0; t < nt; ++t)
      for (int a2 = 0; a2 < g2; ++a2)
        for (int b2 = 0; b2 < g2; ++b2)
          for (int s = 0; s < 4; ++s) {
            const int pa = 2 * a2 + s / 2, pb = 2 * b2 + s % 2;
            idx[((t * Q) + a2 * g2 + b2) * 4 + s] = (int32_t)(t * T + 1 + pa * grid + pb);
          }
    cudaMemcpy(dw.ps_idx, idx.data(), idx.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    dw32.ps_idx = dw.ps_idx;
  }

  // workspace
  size_t wsz = 0;
  auto plan = [&](size_t bytes) {
    size_t o = wsz;
    wsz += align256(bytes);
    return o;
  };
  const size_t o_xp = plan(M * Kpad * 2);
  const size_t o_h = plan(M * D * 4);
  const size_t o_xn = plan(M * D * 2);
  const size_t o_ao = plan(M * D * 2);
  const size_t o_qkv = plan(M * 3 * (size_t)H * dh * 2);
  size_t big = M * F * 2;
  size_t o_r1 = 0, o_r2 = 0, o_rkv = 0, o_rao = 0, o_rr = 0;
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    big = std::max(big, M * (size_t)E * 2);
  }
  const size_t o_f = plan(big);
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    o_r2 = plan(M * (size_t)E * 2);  // ln_kv output
    o_rkv = plan(M * 2 * (size_t)RH * RDp * 2);
    o_rao = plan(nt * Q * (size_t)E * 2);
    o_rr = plan(nt * Q * (size_t)E * 2);
    o_r1 = o_f;  // kv_proj output reuses the MLP buffer
  } else {
    o_r2 = plan(nt * Q * (size_t)4 * D * 2);  // shuffled + LN rows
    o_rr = plan(nt * Q * (size_t)E * 2);      // fc1 output
  }
  const size_t o_in = plan(nt * (size_t)d.image_size * d.image_size * d.channels);
  const size_t o_out = plan(nt * (size_t)Q * E * 2);
  e = cudaMalloc(&work, wsz);
  if (e != cudaSuccess) {
    err = std::string("cudaMalloc(workspace): ") + cudaGetErrorString(e);
    return EPD_ERR_CUDA;
  }
  uint8_t* wb = reinterpret_cast<uint8_t*>(work);
  in_buf = wb + o_in;
  out_buf = reinterpret_cast<bf16*>(wb + o_out);
  ws.xp = reinterpret_cast<bf16*>(wb + o_xp);
  ws.h = reinterpret_cast<float*>(wb + o_h);
  ws.xn = reinterpret_cast<bf16*>(wb + o_xn);
  ws.ao = reinterpret_cast<bf16*>(wb + o_ao);
  ws.qkv = reinterpret_cast<bf16*>(wb + o_qkv);
  ws.f = reinterpret_cast<bf16*>(wb + o_f);
  ws.r1 = reinterpret_cast<bf16*>(wb + o_r1);
  ws.r2 = reinterpret_cast<bf16*>(wb + o_r2);
  ws.rkv = reinterpret_cast<bf16*>(wb + o_rkv);
  ws.rao = reinterpret_cast<bf16*>(wb + o_rao);
  ws.rr = reinterpret_cast<bf16*>(wb + o_rr);
  // Padded head dims / key padding are read by the attention TMA and must be finite.
  cudaMemsetAsync(work, 0, wsz, stream);

  // ---- weight-only precomputation (resampler queries and key positions)
  int rc = 0;
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    // temporaries live in the (not yet used) MLP buffer
    bf16* qn = ws.f;
    rc = layernorm_bf16(rs.query, E, qn, E, rs.lnq_w, rs.lnq_b, Q, E, 1e-6f, stream);
    if (!rc) {
      // resampler queries, row-major [Q][RH*RDp] (attention reads them as shared queries)
      EpiParams ep;
      ep.bias = rs.qb;
      ep.out = dw.r_qheads;
      ep.ldo = RH * RDp;
      rc = gemm_bf16(qn, E, rs.qw, E, Q, RH * RDp, E, ep, stream);
    }
    if (!rc) {
      // pos_k[t][0:RH*RDp] = pos[t] @ Wk^T (head padded); second half (V section) = 0
      cudaMemsetAsync(dw.r_posk, 0, (size_t)T * 2 * RH * RDp * 2, stream);
      EpiParams ep;
      ep.out = dw.r_posk;
      ep.ldo = 2 * RH * RDp;
      rc = gemm_bf16(rs.pos, E, rs.kw, E, T, RH * RDp, E, ep, stream);
    }
    if (!rc && check_f32) {
      // fp32 twins; temporaries in the (unused) fp32 blob tail would cost memory,
      // so borrow a cudaMalloc scratch for the normalised queries.
      float* qn32 = nullptr;
      rc = (int)cudaMalloc(&qn32, (size_t)Q * E * 4);
      if (!rc) rc = layernorm_f32_check(rs32.query, E, qn32, E, rs32.lnq_w, rs32.lnq_b, Q, E, 1e-6f, nullptr, 1, stream);
      if (!rc) {
        EpiF32 ep;
        ep.mode = EPI_HEADS;
        ep.bias = rs32.qb;
        ep.H = RH; ep.Dp = RDp; ep.T = Q; ep.sec_cols = RH * RDp;
        ep.sec_out[0] = dw32.r_qheads;
        rc = gemm_f32(qn32, E, rs32.qw, E, Q, RH * RDp, E, ep, stream);
      }
      if (!rc) {
        cudaMemsetAsync(dw32.r_posk, 0, (size_t)T * 2 * RH * RDp * 4, stream);
        EpiF32 ep;
        ep.out = dw32.r_posk;
        ep.ldo = 2 * RH * RDp;
        rc = gemm_f32(rs32.pos, E, rs32.kw, E, T, RH * RDp, E, ep, stream);
      }
      if (!rc) rc = (int)cudaStreamSynchronize(stream);
      if (qn32) cudaFree(qn32);
    }
  }
  if (!rc) rc = (int)cudaStreamSynchronize(stream);
  if (rc) {
    err = "finalize precompute failed (code " + std::to_string(rc) + "): " +
          (rc < 1000 ? cudaGetErrorString((cudaError_t)rc) : "argument");
    return EPD_ERR_CUDA;
  }
  for (auto& s : slots) std::vector<float>().swap(s.host);
  finalized = true;
  return EPD_OK;
}

// ------------------------------------------------------------ forward

int Encoder::launches(int n) const {
  if (n <= 0) return 0;
  const int chunks = (n + d.max_tiles - 1) / d.max_tiles;
  int per = 1 /*patchify*/ + 1 /*patch GEMM*/ + 7 * d.layers;
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER)
    per += 1 /*post LN*/ + 1 /*kv_proj*/ + 1 /*ln_kv*/ + 1 /*kv in-proj*/ + 1 /*attn*/ + 1 /*o*/ +
           1 /*ln_post*/ + 1 /*proj*/;
  else
    per += 1 /*shuffle+LN*/ + 2 /*fc1, fc2*/;  // (+ a cudaMemset of the CLS rows, not a kernel of ours)
  return chunks * per;
}

double Encoder::flops_per_tile() const {
  const double t = npatch, Dd = D, Ff = F;
  double f = 2.0 * npatch * Kreal * Dd;  // patch embedding
  const double tt = T;
  const double layer = 2.0 * tt * Dd * 3 * Dd + 2.0 * 2.0 * tt * tt * Dd + 2.0 * tt * Dd * Dd +
                       2.0 * 2.0 * tt * Dd * Ff;
  f += d.layers * layer;
  const double Ee = E, Qq = Q;
  if (d.family == EPD_FAMILY_SIGLIP_RESAMPLER) {
    f += 2.0 * t * Dd * Ee;             // kv_proj
    f += 2.0 * 2.0 * t * Ee * Ee;       // k, v in-projections
    f += 2.0 * Qq * Ee * Ee;            // q in-projection (weight-only; precomputed once here)
    f += 2.0 * 2.0 * Qq * t * Ee;       // cross attention
    f += 2.0 * 2.0 * Qq * Ee * Ee;      // out-proj + proj
  } else {
    f += 2.0 * Qq * 4 * Dd * Ee + 2.0 * Qq * Ee * Ee;  // mlp1
  }
  return f;
}

int Encoder::encode(const uint8_t* tiles, int n, bf16* out, cudaStream_t s, std::string& err) {
  if (!finalized) {
    err = "encoder not finalized";
    return EPD_ERR_RUNTIME;
  }
  if (n < 0) {
    err = "tile count must be non-negative";
    return EPD_ERR_VALUE;
  }
  const size_t tile_bytes = (size_t)d.image_size * d.image_size * d.channels;
  for (int c0 = 0; c0 < n; c0 += d.max_tiles) {
    const int nt = std::min(d.max_tiles, n - c0);
    const uint8_t* src = tiles + (size_t)c0 * tile_bytes;
    bf16* dst = out + (size_t)c0 * Q * E;
    int rc;
    if (prof_on || !use_graphs)
      rc = forward_chunk(src, nt, dst, s);
    else
      rc = forward_graph(src, nt, dst, s);
    if (rc) {
      err = "kernel launch failed (code " + std::to_string(rc) + "): " +
            (rc < 1000 ? cudaGetErrorString((cudaError_t)rc) : "argument/shape");
      return EPD_ERR_CUDA;
    }
  }
  return EPD_OK;
}

#define EPD_TRY(x)            \
  do {                        \
    int _rc = (x);            \
    if (_rc) return _rc;      \
  } while (0)

// One CUDA graph per (chunk size, input, output): the ~200 launches of a forward pass replay
// with a single cudaGraphLaunch that reads the caller's tiles and writes the caller's token
// buffer in place (the stage's double-buffered rings keep the set of pointers small). Past
// kMaxGraphs the graphs for new pointer pairs run on the encoder-owned staging buffers
// (in_buf / out_buf) at the cost of two device copies.
int Encoder::forward_graph(const uint8_t* tiles, int nt, bf16* out, cudaStream_t s) {
  constexpr size_t kMaxGraphs = 24;
  const size_t in_bytes = (size_t)nt * d.image_size * d.image_size * d.channels;
  const size_t out_bytes = (size_t)nt * Q * E * 2;
  GraphKey key{nt, tiles, out};
  auto it = graphs.find(key);
  const bool staged = it == graphs.end() && graphs.size() >= kMaxGraphs;
  if (staged) {
    key = GraphKey{nt, in_buf, out_buf};
    it = graphs.find(key);
  }
  if (it == graphs.end()) {
    if (!cap_stream) EPD_TRY((int)cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    EPD_TRY((int)cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = forward_chunk(std::get<1>(key), nt, std::get<2>(key), cap_stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return (int)e;
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return (int)e;
    it = graphs.emplace(key, ex).first;
  }
  if (staged) EPD_TRY((int)cudaMemcpyAsync(in_buf, tiles, in_bytes, cudaMemcpyDeviceToDevice, s));
  EPD_TRY((int)cudaGraphLaunch(it->second, s));
  if (staged) EPD_TRY((int)cudaMemcpyAsync(out, out_buf, out_bytes, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// Launch with optional per-launch CUDA-event profiling (class, algorithmic FLOPs, bytes).
#define EPD_LAUNCH(cls, flops, bytes, x)        \
  do {                                          \
    const int _ev = prof_begin(s);              \
    int _rc = (x);                              \
    if (_rc) return _rc;                        \
    prof_end(s, _ev, (cls), (flops), (bytes));  \
  } while (0)

int Encoder::prof_begin(cudaStream_t s) {
  if (!prof_on) return -1;
  if (prof_used + 2 > prof_events.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      prof_events.push_back(e);
    }
  }
  const int i = (int)prof_used;
  cudaEventRecord(prof_events[i], s);
  prof_used += 2;
  return i;
}

void Encoder::prof_end(cudaStream_t s, int ev, int cls, double flops, double bytes) {
  if (ev < 0) return;
  cudaEventRecord(prof_events[ev + 1], s);
  prof_recs.push_back({cls, ev, flops, bytes});
}

int Encoder::prof_read(double* ms, double* flops, double* bytes, int64_t* count, int nclass) {
  for (int c = 0; c < nclass; ++c) ms[c] = flops[c] = bytes[c] = 0, count[c] = 0;
  if (!prof_recs.empty()) {
    cudaError_t e = cudaEventSynchronize(prof_events[prof_recs.back().ev + 1]);
    if (e != cudaSuccess) return (int)e;
  }
  prof_last.clear();
  for (const auto& r : prof_recs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, prof_events[r.ev], prof_events[r.ev + 1]);
    prof_last.push_back({r.cls, t, r.flops});
    if (r.cls < 0 || r.cls >= nclass) continue;
    ms[r.cls] += t;
    flops[r.cls] += r.flops;
    bytes[r.cls] += r.bytes;
    count[r.cls] += 1;
  }
  prof_recs.clear();
  prof_used = 0;
  return 0;
}

int Encoder::forward_chunk(const uint8_t* tiles, int nt, bf16* out, cudaStream_t s) {
  // PDL (auto mode); scheduling only, results are identical
  PdlScope pdl(nt <= kPdlMaxTiles);
  const int M = nt * T;
  const float eps = d.ln_eps;
  const bool internvl = d.family == EPD_FAMILY_INTERNVIT_MLP;
  const double dM = M, dD = D, dF = F, dE = E, dQ = (double)nt * Q, dT = T;
  const double ln_bytes_f32 = dM * dD * (4 + 2), ln_bytes = dM * dE * (2 + 2);
  // 1. patchify (+ zero CLS rows) and patch-embedding GEMM (+bias +pos)
  if (internvl)
    EPD_LAUNCH(PROF_OTHER, 0, (double)M * Kpad * 2, (int)cudaMemsetAsync(ws.xp, 0, (size_t)M * Kpad * 2, s));
  EPD_LAUNCH(PROF_PATCHIFY, 0, (double)nt * d.image_size * d.image_size * d.channels + (double)nt * npatch * Kpad * 2,
             patchify_u8(tiles, nt, d.image_size, d.channels, d.patch_size, Kpad, internvl ? 1 : 0, T,
                         d.mean, d.std, ws.xp, s));
  {
    EpiParams ep;
    ep.bias = dw.pe_b;
    ep.resid = dw.pos;
    ep.ldr = D;
    ep.r_mod = T;
    ep.out_f = ws.h;
    ep.ldo = D;
    EPD_LAUNCH(PROF_GEMM, 2.0 * nt * npatch * Kreal * dD, 0, gemm_bf16(ws.xp, Kpad, dw.pe, Kpad, M, D, Kpad, ep, s));
  }
  // 2. transformer blocks
  const int act = internvl ? ACT_GELU_ERF : ACT_GELU_TANH;
  for (size_t l = 0; l < dl.size(); ++l) {
    const auto& w = dl[l];
    EPD_LAUNCH(PROF_LN, 0, ln_bytes_f32, layernorm_f32in(ws.h, D, ws.xn, D, w.ln1w, w.ln1b, M, D, eps, nullptr, 1, s));
    {
      EpiParams ep;
      ep.bias = w.qkvb;
      ep.out = ws.qkv; ep.ldo = 3 * H * dh;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dM * dD * 3 * dD, 0, gemm_bf16(ws.xn, D, w.qkv, D, M, 3 * H * dh, D, ep, s));
    }
    {
      // heads read in place from the row-major QKV (columns: Q | K | V, head h at h*dh)
      AttnParams ap;
      ap.q = ws.qkv; ap.k = ws.qkv + H * dh; ap.v = ws.qkv + 2 * H * dh; ap.out = ws.ao;
      ap.ldq = ap.ldk = ap.ldv = 3 * H * dh; ap.hs = dh;
      ap.B = nt; ap.H = H; ap.Tq = T; ap.Tk = T; ap.Dp = Dp; ap.Dv = dh;
      ap.ldo = D;
      ap.scale = 1.f / std::sqrt((float)dh);
      EPD_LAUNCH(PROF_ATTN, 4.0 * nt * dT * dT * dD, 0, attention_bf16(ap, s));
    }
    {
      EpiParams ep;
      ep.bias = w.ob;
      ep.resid_f = ws.h; ep.ldr = D; ep.lscale = w.ls1;
      ep.out_f = ws.h; ep.ldo = D;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dM * dD * dD, 0, gemm_bf16(ws.ao, D, w.ow, D, M, D, D, ep, s));
    }
    EPD_LAUNCH(PROF_LN, 0, ln_bytes_f32, layernorm_f32in(ws.h, D, ws.xn, D, w.ln2w, w.ln2b, M, D, eps, nullptr, 1, s));
    {
      EpiParams ep;
      ep.bias = w.f1b;
      ep.act = act;
      ep.out = ws.f; ep.ldo = F;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dM * dD * dF, 0, gemm_bf16(ws.xn, D, w.f1w, D, M, F, D, ep, s));
    }
    {
      EpiParams ep;
      ep.bias = w.f2b;
      ep.resid_f = ws.h; ep.ldr = D; ep.lscale = w.ls2;
      ep.out_f = ws.h; ep.ldo = D;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dM * dD * dF, 0, gemm_bf16(ws.f, F, w.f2w, F, M, D, F, ep, s));
    }
  }
  // 3. resampler / projector
  if (!internvl) {
    EPD_LAUNCH(PROF_LN, 0, ln_bytes_f32,
               layernorm_f32in(ws.h, D, ws.xn, D, dw.post_w, dw.post_b, M, D, eps, nullptr, 1, s));
    {
      EpiParams ep;
      ep.out = ws.r1; ep.ldo = E;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dM * dD * dE, 0, gemm_bf16(ws.xn, D, dw.r_kv, D, M, E, D, ep, s));
    }
    EPD_LAUNCH(PROF_LN, 0, ln_bytes, layernorm_bf16(ws.r1, E, ws.r2, E, dw.r_lnkv_w, dw.r_lnkv_b, M, E, 1e-6f, s));
    {
      // k = (x + pos) Wk^T + bk  ==  x Wk^T + bk + (pos Wk^T)   [pos_k table, rows % T]
      // row-major [M][K | V] with RH heads of RDp each
      EpiParams ep;
      ep.bias = dw.r_kvin_b;
      ep.resid = dw.r_posk; ep.ldr = 2 * RH * RDp; ep.r_mod = T;
      ep.out = ws.rkv; ep.ldo = 2 * RH * RDp;
      EPD_LAUNCH(PROF_GEMM, 4.0 * dM * dE * dE, 0, gemm_bf16(ws.r2, E, dw.r_kvin, E, M, 2 * RH * RDp, E, ep, s));
    }
    {
      AttnParams ap;
      ap.q = dw.r_qheads; ap.k = ws.rkv; ap.v = ws.rkv + RH * RDp; ap.out = ws.rao;
      ap.ldq = RH * RDp; ap.ldk = ap.ldv = 2 * RH * RDp; ap.hs = RDp;
      ap.B = nt; ap.H = RH; ap.Tq = Q; ap.Tk = T; ap.Dp = RDp; ap.Dv = rdh;
      ap.ldo = E; ap.q_shared = 1;
      ap.scale = 1.f / std::sqrt((float)rdh);
      EPD_LAUNCH(PROF_ATTN, 4.0 * dQ * dT * dE, 0, attention_bf16(ap, s));
    }
    {
      EpiParams ep;
      ep.bias = dw.r_ob;
      ep.out = ws.rr; ep.ldo = E;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dQ * dE * dE, 0, gemm_bf16(ws.rao, E, dw.r_ow, E, nt * Q, E, E, ep, s));
    }
    EPD_LAUNCH(PROF_LN, 0, dQ * dE * 4,
               layernorm_bf16(ws.rr, E, ws.rao, E, dw.r_lnp_w, dw.r_lnp_b, nt * Q, E, 1e-6f, s));
    {
      EpiParams ep;
      ep.out = out; ep.ldo = E;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dQ * dE * dE, 0, gemm_bf16(ws.rao, E, dw.r_projT, E, nt * Q, E, E, ep, s));
    }
  } else {
    const int C4 = 4 * D;
    EPD_LAUNCH(PROF_LN, 0, dQ * C4 * (4 + 2),
               layernorm_f32in(ws.h, D, ws.r2, C4, dw.m_ln_w, dw.m_ln_b, nt * Q, C4, 1e-5f, dw.ps_idx, 4, s));
    {
      EpiParams ep;
      ep.bias = dw.m_f1b;
      ep.act = ACT_GELU_ERF;
      ep.out = ws.rr; ep.ldo = E;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dQ * C4 * dE, 0, gemm_bf16(ws.r2, C4, dw.m_f1w, C4, nt * Q, E, C4, ep, s));
    }
    {
      EpiParams ep;
      ep.bias = dw.m_f2b;
      ep.out = out; ep.ldo = E;
      EPD_LAUNCH(PROF_GEMM, 2.0 * dQ * dE * dE, 0, gemm_bf16(ws.rr, E, dw.m_f2w, E, nt * Q, E, E, ep, s));
    }
  }
  return 0;
}

// ------------------------------------------------------------ fp32 check mode

int Encoder::encode_f32(const uint8_t* tiles, int n, float* out, cudaStream_t s, std::string& err) {
  if (!finalized || !check_f32) {
    err = "fp32 check mode: enable it before finalize";
    return EPD_ERR_RUNTIME;
  }
  if (n < 0) {
    err = "tile count must be non-negative";
    return EPD_ERR_VALUE;
  }
  if (!work32) {
    f32_chunk = std::min(d.max_tiles, 4);
    const size_t nt = f32_chunk, M = nt * T;
    size_t wsz = 0;
    auto plan = [&](size_t floats) {
      size_t o = wsz;
      wsz += align256(floats * 4);
      return o;
    };
    const size_t o_xp = plan(M * Kpad), o_h = plan(M * D), o_xn = plan(M * D), o_ao = plan(M * D);
    const size_t o_q = plan(nt * H * T * Dp), o_k = plan(nt * H * T * Dp), o_v = plan(nt * H * T * Dp);
    const size_t o_f = plan(M * std::max(F, E));
    const bool siglip = d.family == EPD_FAMILY_SIGLIP_RESAMPLER;
    const size_t o_r2 = plan(siglip ? M * E : nt * Q * 4 * (size_t)D);
    const size_t o_rk = plan(siglip ? nt * RH * T * RDp : 0), o_rv = plan(siglip ? nt * RH * T * RDp : 0);
    const size_t o_rao = plan(nt * Q * (size_t)E), o_rr = plan(nt * Q * (size_t)E);
    cudaError_t e = cudaMalloc(&work32, wsz);
    if (e != cudaSuccess) {
      err = std::string("cudaMalloc(fp32 workspace): ") + cudaGetErrorString(e);
      return EPD_ERR_CUDA;
    }
    cudaMemsetAsync(work32, 0, wsz, s);
    float* b = reinterpret_cast<float*>(work32);
    auto at = [&](size_t off) { return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(b) + off); };
    ws32 = {at(o_xp), at(o_h), at(o_xn), at(o_ao), at(o_q), at(o_k), at(o_v),
            at(o_f), at(o_r2), at(o_rk), at(o_rv), at(o_rao), at(o_rr)};
  }
  const size_t tile_bytes = (size_t)d.image_size * d.image_size * d.channels;
  for (int c0 = 0; c0 < n; c0 += f32_chunk) {
    const int nt = std::min(f32_chunk, n - c0);
    const int rc = forward_f32(tiles + (size_t)c0 * tile_bytes, nt, out + (size_t)c0 * Q * E, s);
    if (rc) {
      err = "fp32 check launch failed (code " + std::to_string(rc) + ")";
      return EPD_ERR_CUDA;
    }
  }
  return EPD_OK;
}

// Same schedule and fusions as forward_chunk, every tensor fp32.
int Encoder::forward_f32(const uint8_t* tiles, int nt, float* out, cudaStream_t s) {
  const int M = nt * T;
  const float eps = d.ln_eps;
  const bool internvl = d.family == EPD_FAMILY_INTERNVIT_MLP;
  const auto& W = dw32;
  const auto& X = ws32;
  if (internvl) EPD_TRY((int)cudaMemsetAsync(X.xp, 0, (size_t)M * Kpad * 4, s));
  EPD_TRY(patchify_f32(tiles, nt, d.image_size, d.channels, d.patch_size, Kpad, internvl ? 1 : 0, T, d.mean,
                       d.std, X.xp, s));
  {
    EpiF32 ep;
    ep.bias = W.pe_b;
    ep.resid = W.pos; ep.ldr = D; ep.r_mod = T;
    ep.out = X.h; ep.ldo = D;
    EPD_TRY(gemm_f32(X.xp, Kpad, W.pe, Kpad, M, D, Kpad, ep, s));
  }
  const int act = internvl ? ACT_GELU_ERF : ACT_GELU_TANH;
  for (const auto& w : dl32) {
    EPD_TRY(layernorm_f32_check(X.h, D, X.xn, D, w.ln1w, w.ln1b, M, D, eps, nullptr, 1, s));
    {
      EpiF32 ep;
      ep.mode = EPI_HEADS;
      ep.bias = w.qkvb;
      ep.H = H; ep.Dp = Dp; ep.T = T; ep.dh = dh; ep.sec_cols = H * dh;  // packed QKV image
      ep.sec_out[0] = X.q; ep.sec_out[1] = X.k; ep.sec_out[2] = X.v;
      EPD_TRY(gemm_f32(X.xn, D, w.qkv, D, M, 3 * H * dh, D, ep, s));
    }
    EPD_TRY(attention_f32(X.q, X.k, X.v, X.ao, nt, H, T, T, Dp, dh, D, 0, 1.f / std::sqrt((float)dh), s));
    {
      EpiF32 ep;
      ep.bias = w.ob; ep.lscale = w.ls1;
      ep.accumulate = 1;
      ep.out = X.h; ep.ldo = D;
      EPD_TRY(gemm_f32(X.ao, D, w.ow, D, M, D, D, ep, s));
    }
    EPD_TRY(layernorm_f32_check(X.h, D, X.xn, D, w.ln2w, w.ln2b, M, D, eps, nullptr, 1, s));
    {
      EpiF32 ep;
      ep.bias = w.f1b; ep.act = act;
      ep.out = X.f; ep.ldo = F;
      EPD_TRY(gemm_f32(X.xn, D, w.f1w, D, M, F, D, ep, s));
    }
    {
      EpiF32 ep;
      ep.bias = w.f2b; ep.lscale = w.ls2;
      ep.accumulate = 1;
      ep.out = X.h; ep.ldo = D;
      EPD_TRY(gemm_f32(X.f, F, w.f2w, F, M, D, F, ep, s));
    }
  }
  if (!internvl) {
    EPD_TRY(layernorm_f32_check(X.h, D, X.xn, D, W.post_w, W.post_b, M, D, eps, nullptr, 1, s));
    {
      EpiF32 ep;
      ep.out = X.f; ep.ldo = E;
      EPD_TRY(gemm_f32(X.xn, D, W.r_kv, D, M, E, D, ep, s));
    }
    EPD_TRY(layernorm_f32_check(X.f, E, X.r2, E, W.r_lnkv_w, W.r_lnkv_b, M, E, 1e-6f, nullptr, 1, s));
    {
      EpiF32 ep;
      ep.mode = EPI_HEADS;
      ep.bias = W.r_kvin_b;
      ep.resid = W.r_posk; ep.ldr = 2 * RH * RDp; ep.r_mod = T;
      ep.H = RH; ep.Dp = RDp; ep.T = T; ep.sec_cols = RH * RDp;
      ep.sec_out[0] = X.rk; ep.sec_out[1] = X.rv;
      EPD_TRY(gemm_f32(X.r2, E, W.r_kvin, E, M, 2 * RH * RDp, E, ep, s));
    }
    EPD_TRY(attention_f32(W.r_qheads, X.rk, X.rv, X.rao, nt, RH, Q, T, RDp, rdh, E, 1, 1.f / std::sqrt((float)rdh), s));
    {
      EpiF32 ep;
      ep.bias = W.r_ob;
      ep.out = X.rr; ep.ldo = E;
      EPD_TRY(gemm_f32(X.rao, E, W.r_ow, E, nt * Q, E, E, ep, s));
    }
    EPD_TRY(layernorm_f32_check(X.rr, E, X.rao, E, W.r_lnp_w, W.r_lnp_b, nt * Q, E, 1e-6f, nullptr, 1, s));
    {
      EpiF32 ep;
      ep.out = out; ep.ldo = E;
      EPD_TRY(gemm_f32(X.rao, E, W.r_projT, E, nt * Q, E, E, ep, s));
    }
  } else {
    const int C4 = 4 * D;
    EPD_TRY(layernorm_f32_check(X.h, D, X.r2, C4, W.m_ln_w, W.m_ln_b, nt * Q, C4, 1e-5f, W.ps_idx, 4, s));
    {
      EpiF32 ep;
      ep.bias = W.m_f1b; ep.act = ACT_GELU_ERF;
      ep.out = X.rr; ep.ldo = E;
      EPD_TRY(gemm_f32(X.r2, C4, W.m_f1w, C4, nt * Q, E, C4, ep, s));
    }
    {
      EpiF32 ep;
      ep.bias = W.m_f2b;
      ep.out = out; ep.ldo = E;
      EPD_TRY(gemm_f32(X.rr, E, W.m_f2w, E, nt * Q, E, E, ep, s));
    }
  }
  return 0;
}

}  // namespace epd
