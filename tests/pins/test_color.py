"""Pins for the sRGB <-> CIE-Lab oracle (reading R18):
  * the derived RGB->XYZ matrix maps (1,1,1) to the D65 white and has Y-row sum 1, and agrees
    with the IEC 61966-2-1 matrix as commonly tabulated to 4 decimals;
  * white -> (100, 0, 0), black -> (0, 0, 0) exactly; every neutral grey has a* = b* = 0;
  * L* of mid-grey from the closed forms (sRGB 119 is close to L* = 50);
  * published Lab values of the sRGB primaries (D65) to 0.01;
  * round trip sRGB -> Lab -> sRGB is the identity to 1e-9 over random colours.
"""
import numpy as np
import pytest

from oracle import color


def test_matrix_against_tabulated_and_white():
    M = color.rgb_to_xyz_matrix()
    tab = np.array([[0.4124, 0.3576, 0.1805], [0.2126, 0.7152, 0.0722], [0.0193, 0.1192, 0.9505]])
    assert np.abs(M - tab).max() < 2e-4
    np.testing.assert_allclose(M @ np.ones(3), color.white(), rtol=1e-14)
    assert abs(M[1].sum() - 1.0) < 1e-14


def test_white_black_and_greys():
    lab = color.srgb_to_lab(np.array([[255.0, 0.0], [255.0, 0.0], [255.0, 0.0]]))
    np.testing.assert_allclose(lab[:, 0], [100.0, 0.0, 0.0], atol=1e-12)
    np.testing.assert_allclose(lab[:, 1], [0.0, 0.0, 0.0], atol=1e-12)
    g = np.arange(256.0)
    lab = color.srgb_to_lab(np.stack([g, g, g]))
    assert np.abs(lab[1:]).max() < 1e-12
    assert np.all(np.diff(lab[0]) > 0)
    assert abs(lab[0, 119] - 50.0) < 0.5


@pytest.mark.parametrize("rgb,lab", [((255, 0, 0), (53.2408, 80.0925, 67.2032)),
                                     ((0, 255, 0), (87.7347, -86.1827, 83.1793)),
                                     ((0, 0, 255), (32.2970, 79.1875, -107.8602))])
def test_primaries_published_values(rgb, lab):
    got = color.srgb_to_lab(np.array(rgb, dtype=np.float64).reshape(3, 1))[:, 0]
    np.testing.assert_allclose(got, lab, atol=0.01)


def test_round_trip():
    rgb = np.random.default_rng(0).uniform(0, 255, (3, 5000))
    np.testing.assert_allclose(color.lab_to_srgb(color.srgb_to_lab(rgb)), rgb, atol=1e-9)
