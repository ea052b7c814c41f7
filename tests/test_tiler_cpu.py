"""Tiling rules reproduce the reference catalog's tile counts
(models.cfg patch_table, pinned by test_models.py in the reference)."""
from paper_2501_05460_b200.configs import INTERNVL2_8B, MINICPM_V26
from paper_2501_05460_b200.tiler import internvl_grid, minicpm_grid, tiles_for_image


def test_tile_counts_match_reference_patch_table():
    for geom in (MINICPM_V26, INTERNVL2_8B):
        for (w, h), n in geom.patch_table.items():
            assert tiles_for_image(geom.name, w, h) == n, (geom.name, w, h)


def test_grids():
    assert minicpm_grid(4032, 3024) == (3, 3)
    assert minicpm_grid(787, 444) == (2, 1)
    assert minicpm_grid(313, 234) is None
    assert internvl_grid(4032, 3024) == (4, 3, True)
    assert internvl_grid(787, 444) == (2, 1, True)
    assert internvl_grid(448, 448)[:2] == (1, 1) and internvl_grid(448, 448)[2] is False
