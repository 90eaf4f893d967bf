"""Seeded synthetic inputs (workloads/): determinism, shapes, ranges, and that a
row band regenerates exactly the same rows as the full image."""
import numpy as np
import pytest

from workloads import CONFIGS, make_image, make_image_rows


def test_config_table_matches_baseline():
    c = CONFIGS
    assert [(c[i].H, c[i].W, c[i].d) for i in range(1, 6)] == \
        [(64, 64, 3), (512, 512, 3), (1080, 1920, 3), (1024, 1024, 8), (8192, 8192, 3)]
    assert [c[i].radius for i in range(1, 6)] == [6, 15, 30, 24, 48]
    assert [(c[i].N, c[i].M, c[i].seed) for i in range(1, 6)] == \
        [(20, 32, 0), (30, 64, 1), (40, 128, 2), (30, 256, 3), (40, 512, 4)]
    assert c[3].C_array[0, 1] == 35.0 ** 2 * 0.5 and c[3].C_array[0, 2] == 35.0 ** 2 * 0.3


@pytest.mark.parametrize("i", [1, 2])
def test_full_image_properties(i):
    cfg = CONFIGS[i]
    img = make_image(cfg)
    assert img.shape == (cfg.d, cfg.H, cfg.W) and img.dtype == np.float32
    assert img.min() >= 0.0 and img.max() <= cfg.value_range
    assert np.array_equal(img, make_image(cfg))
    band = make_image_rows(cfg, 37, 61)
    assert np.array_equal(band, img[:, 37:61])


def test_band_of_large_configs():
    for i in (3, 4, 5):
        cfg = CONFIGS[i]
        a = make_image_rows(cfg, 60, 70)
        b = make_image_rows(cfg, 64, 66)
        assert a.shape == (cfg.d, 10, cfg.W)
        assert np.array_equal(a[:, 4:6], b)
        assert a.min() >= 0 and a.max() <= cfg.value_range
