// Kernel launch helper: every encoder-forward kernel is launched with programmatic
// dependent launch (PDL). A kernel triggers its dependents as soon as it starts, so the
// next kernel's CTAs are scheduled onto SMs as this one drains and run their prologue
// (barrier init, TMEM allocation, tensor-map prefetch, weight staging) early; each
// kernel executes griddepcontrol.wait (pdl_wait) before it touches memory the previous
// kernel produced or consumes. Because every kernel waits before completing, the
// ordering is transitive along the stream. Opt-in (EPD_PDL=1): it measured neutral on the
// power-capped C2 step and made the InternViT (C5) step erratic (671-900 vs 1135 tiles/s).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace epd {

inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("EPD_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v != 0;
}

template <typename... KArgs, typename... Args>
int launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int cluster,
                  Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return (int)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace epd
