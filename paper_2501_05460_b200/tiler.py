"""On-device image tiling: the step before the encode path.

The reference only looks tile counts up (``models.patches_for_image``, models.py:138-143,
``patch_table`` in models.cfg). This module implements the public tiling rules the
catalog's counts come from and cuts the tiles on the GPU:

* InternVL2 ``dynamic_preprocess``: the grid (cols, rows) with 1 <= cols*rows <= 12 whose
  aspect ratio is closest to the image's (ties -> the larger grid if the image has more
  than half its area), the image resized to (cols*448, rows*448) and cut row-major, plus
  a 448x448 thumbnail of the whole image when the grid has more than one tile.
* MiniCPM-V 2.6 slicing (``get_sliced_grid``): multiple = min(ceil(area / 448^2), 9); no
  slicing when it is 1; otherwise among the factorisations of multiple-1, multiple,
  multiple+1 (<= 9, > 1) the grid whose log aspect ratio is closest to the image's. The
  whole image comes first (as a 448x448 tile), then the slices. (MiniCPM keeps each
  slice's aspect ratio with a variable patch grid; here every slice is 448x448 -- the
  encoder's fixed tile -- so counts match and shapes are the encoder's.)

Pixels: antialiased bilinear resampling (the triangle filter widened by the downscale
factor, as torch.nn.functional.interpolate(..., antialias=True) and PIL use), one kernel
for all tiles of an image, uint8 HWC in and out.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from ._lib import call


def internvl_grid(width: int, height: int, max_num: int = 12, min_num: int = 1, tile: int = 448):
    """(cols, rows, thumbnail) of InternVL2 dynamic_preprocess."""
    aspect = width / height
    ratios = sorted({(i, j) for n in range(min_num, max_num + 1) for i in range(1, n + 1) for j in range(1, n + 1)
                     if min_num <= i * j <= max_num}, key=lambda x: x[0] * x[1])
    best_diff, best = float("inf"), (1, 1)
    area = width * height
    for r in ratios:
        diff = abs(aspect - r[0] / r[1])
        if diff < best_diff:
            best_diff, best = diff, r
        elif diff == best_diff and area > 0.5 * tile * tile * r[0] * r[1]:
            best = r
    return best[0], best[1], best[0] * best[1] != 1


def minicpm_grid(width: int, height: int, max_slice_nums: int = 9, tile: int = 448):
    """(cols, rows) of MiniCPM-V 2.6 get_sliced_grid, or None when the image is not sliced."""
    log_ratio = math.log(width / height)
    multiple = min(math.ceil(width * height / (tile * tile)), max_slice_nums)
    if multiple <= 1:
        return None
    grids = []
    for n in (multiple - 1, multiple, multiple + 1):
        if n == 1 or n > max_slice_nums:
            continue
        grids += [(m, n // m) for m in range(1, n + 1) if n % m == 0]
    best, best_err = (1, 1), float("inf")
    for g in grids:
        err = abs(log_ratio - math.log(g[0] / g[1]))
        if err < best_err:
            best, best_err = g, err
    return best


def plan(model: str, width: int, height: int):
    """(cols, rows, thumbnail, thumbnail_first) for a catalog model name."""
    if model.startswith("internvl"):
        cols, rows, thumb = internvl_grid(width, height)
        return cols, rows, thumb, False
    if model.startswith("minicpm"):
        g = minicpm_grid(width, height)
        if g is None:
            return 0, 0, True, True  # the whole image only
        return g[0], g[1], True, True
    raise KeyError(f"no tiling rule for {model}")


def tiles_for_image(model: str, width: int, height: int) -> int:
    cols, rows, thumb, _ = plan(model, width, height)
    return cols * rows + (1 if thumb else 0)


def tile_image(image: torch.Tensor, model: str, tile: int = 448, out: torch.Tensor | None = None) -> torch.Tensor:
    """uint8 HWC image on the device -> uint8 [n, tile, tile, C] tiles in the model's order."""
    if image.device.type != "cuda" or image.dtype != torch.uint8 or image.dim() != 3:
        raise ValueError("image must be a uint8 HWC tensor on a CUDA device")
    H, W, Cc = image.shape
    cols, rows, thumb, thumb_first = plan(model, W, H)
    n = cols * rows + (1 if thumb else 0)
    if out is None:
        out = torch.empty(n, tile, tile, Cc, dtype=torch.uint8, device=image.device)
    img = image.contiguous()
    call("epd_tile_image", C.c_void_p(img.data_ptr()), H, W, Cc, cols, rows, int(thumb), int(thumb_first), tile,
         C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream(image.device).cuda_stream))
    return out


__all__ = ["internvl_grid", "minicpm_grid", "plan", "tiles_for_image", "tile_image"]
