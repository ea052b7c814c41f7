// On-device image tiling (grid rules in tiler.py): one launch cuts
// every tile of an image -- the grid tiles of the image resized to (cols*S, rows*S) and the
// S x S thumbnail -- with antialiased bilinear resampling (the triangle filter widened by the
// downscale factor; weights as torch / PIL compute them for antialias=True), uint8 HWC in
// and out, in the model's tile order.
#include "common.cuh"
#include "kernels.h"

namespace epd {

namespace {

// Source window and normalisation of output coordinate i along one axis (in -> out size).
struct AxisAA {
  float center, invscale;
  int lo, hi;  // taps [lo, hi)
  float norm;
};

EPD_DEVICE AxisAA axis_aa(int i, int in_size, int out_size) {
  AxisAA a;
  const float scale = (float)in_size / (float)out_size;
  const float support = scale >= 1.f ? scale : 1.f;
  a.invscale = scale >= 1.f ? 1.f / scale : 1.f;
  a.center = scale * (i + 0.5f);
  a.lo = max((int)(a.center - support + 0.5f), 0);
  a.hi = min((int)(a.center + support + 0.5f), in_size);
  float tot = 0.f;
  for (int j = a.lo; j < a.hi; ++j) tot += fmaxf(0.f, 1.f - fabsf((j - a.center + 0.5f) * a.invscale));
  a.norm = tot > 0.f ? 1.f / tot : 0.f;
  return a;
}

EPD_DEVICE float tap(const AxisAA& a, int j) { return fmaxf(0.f, 1.f - fabsf((j - a.center + 0.5f) * a.invscale)); }

__global__ void tile_image_kernel(const uint8_t* __restrict__ src, int H, int W, int C, int cols, int rows,
                                  int thumb, int thumb_first, int S, uint8_t* __restrict__ out) {
  const int t = blockIdx.z;  // output tile
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= S) return;
  const int ngrid = cols * rows;
  const bool is_thumb = thumb && (thumb_first ? t == 0 : t == ngrid);
  int Wr, Hr, X, Y;
  if (is_thumb) {
    Wr = S; Hr = S; X = x; Y = y;
  } else {
    const int g = thumb && thumb_first ? t - 1 : t;
    Wr = cols * S; Hr = rows * S;
    X = (g % cols) * S + x;
    Y = (g / cols) * S + y;
  }
  const AxisAA ax = axis_aa(X, W, Wr), ay = axis_aa(Y, H, Hr);
  float acc[3] = {0.f, 0.f, 0.f};
  for (int j = ay.lo; j < ay.hi; ++j) {
    const float wy = tap(ay, j);
    if (wy == 0.f) continue;
    float row[3] = {0.f, 0.f, 0.f};
    const uint8_t* sp = src + (size_t)j * W * C;
    for (int i = ax.lo; i < ax.hi; ++i) {
      const float wx = tap(ax, i);
      for (int c = 0; c < C; ++c) row[c] = fmaf(wx, (float)sp[(size_t)i * C + c], row[c]);
    }
    for (int c = 0; c < C; ++c) acc[c] = fmaf(wy, row[c], acc[c]);
  }
  uint8_t* op = out + (((size_t)t * S + y) * S + x) * C;
  const float nrm = ax.norm * ay.norm;
  for (int c = 0; c < C; ++c) op[c] = (uint8_t)fminf(fmaxf(rintf(acc[c] * nrm), 0.f), 255.f);
}

}  // namespace

int tile_image_u8(const uint8_t* src, int H, int W, int C, int cols, int rows, int thumb, int thumb_first, int S,
                  uint8_t* out, cudaStream_t s) {
  if (H <= 0 || W <= 0 || C < 1 || C > 3 || S <= 0 || cols < 0 || rows < 0) return 1001;
  const int n = cols * rows + (thumb ? 1 : 0);
  if (n <= 0) return 1001;
  dim3 grid((S + 127) / 128, S, n);
  tile_image_kernel<<<grid, 128, 0, s>>>(src, H, W, C, cols, rows, thumb, thumb_first, S, out);
  return (int)cudaGetLastError();
}

}  // namespace epd
