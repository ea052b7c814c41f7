// Kernel launch helper: every encoder-forward kernel is launched with programmatic
// dependent launch (PDL). A kernel triggers its dependents as soon as it starts, so the
// next kernel's CTAs are scheduled onto SMs as this one drains and run their prologue
// (barrier init, TMEM allocation, tensor-map prefetch, weight staging) early; each
// kernel executes griddepcontrol.wait (pdl_wait) before it touches memory the previous
// kernel produced or consumes. Because every kernel waits before completing, the
// ordering is transitive along the stream. EPD_PDL=1 forces it on, EPD_PDL=0 off; by default
// (auto) the encoder turns it on for its forward (PdlScope): a 1-3 tile IRP shard runs 4-6 %
// faster, a 13-tile C5 request ~1 %. (Round 1 measured 10-tile chunks slower and C5 erratic
// under PDL; that was the attention kernel's barrier region overlapping its TMEM holder.)
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace epd {

// -1 auto, 0 off, 1 on
inline int pdl_mode() {
  static int v = -2;
  if (v == -2) {
    const char* e = std::getenv("EPD_PDL");
    v = (e && e[0]) ? (e[0] == '1' ? 1 : 0) : -1;
  }
  return v;
}

// auto-mode decision for the launches this thread is issuing (set by PdlScope)
inline thread_local bool g_pdl_auto = false;

inline bool pdl_enabled() {
  const int m = pdl_mode();
  return m < 0 ? g_pdl_auto : m == 1;
}

// Scoped auto-mode choice (restores the previous one on exit).
struct PdlScope {
  bool prev;
  explicit PdlScope(bool on) : prev(g_pdl_auto) { g_pdl_auto = on; }
  ~PdlScope() { g_pdl_auto = prev; }
};

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
