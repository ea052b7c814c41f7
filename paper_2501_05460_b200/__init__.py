"""B200-native encode-stage hot path of EPD disaggregated multimodal serving.

The host API mirrors the reference simulator's encode-worker, MM-token cache
and stage-handoff interfaces (disaggsim, /root/reference/pkg/src/disaggsim);
the arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/epd.h (libepd.so).
"""
__version__ = "0.1.0"
