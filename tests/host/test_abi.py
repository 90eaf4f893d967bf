"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/bfvec.h declares, and its host-side logic (Philox block function,
diagonalisation, validation) is right. No kernel is launched."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT, golden_lines

HEADER = os.path.join(ROOT, "include", "bfvec.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bf_vec_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1605_02164_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES)


def test_philox_host_block_known_answers():
    from paper_1605_02164_b200 import philox4x64_10
    for ln in golden_lines("philox4x64_10_kat.txt"):
        h = [int(x, 16) for x in ln.split()]
        assert philox4x64_10(h[0:4], h[4:6]) == h[6:10]


def test_philox_host_matches_numpy_stream():
    from paper_1605_02164_b200 import philox4x64_10
    seed = 4
    words = [int(w) for w in np.random.Philox(key=seed).random_raw(12)]
    for b in range(3):
        assert philox4x64_10([b + 1, 0, 0, 0], [seed, 0]) == words[4 * b:4 * b + 4]


@pytest.mark.parametrize("d,seed", [(2, 0), (3, 1), (5, 2), (8, 3)])
def test_plan_diagonalisation_matches_oracle(d, seed):
    from oracle import plan as oplan
    from paper_1605_02164_b200 import Plan
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(d, d))
    C = 900.0 * (A @ A.T / d + np.eye(d))
    p = Plan(32, 32, d, 1.0, C, 10, 4, 0)
    _, _, Q, a = p.get_draws(with_samples=False)
    Qo, ao = oplan.diagonalize(C)
    np.testing.assert_allclose(a, ao, rtol=1e-12)
    np.testing.assert_allclose(Q, Qo, atol=1e-10)


def test_plan_validation_errors():
    from paper_1605_02164_b200 import BfVecError, Plan
    C = np.eye(3) * 100.0
    for args in [(0, 8, 3, 1.0, C, 10, 4, 0), (8, 8, 3, 0.0, C, 10, 4, 0), (8, 8, 3, 1.0, C, 11, 4, 0),
                 (8, 8, 3, 1.0, C, 10, 0, 0), (8, 8, 9, 1.0, np.eye(9), 10, 4, 0),
                 (8, 8, 3, 4e5, C, 10, 4, 0)]:
        with pytest.raises(BfVecError):
            Plan(*args)
    with pytest.raises(BfVecError) as e:
        Plan(8, 8, 2, 1.0, np.array([[1.0, 0.5], [0.4, 1.0]]), 10, 4, 0)
    assert e.value.status == -2
    with pytest.raises(BfVecError) as e:
        Plan(8, 8, 2, 1.0, np.array([[1.0, 2.0], [2.0, 1.0]]), 10, 4, 0)
    assert e.value.status == -3


def test_filter_requires_sampling_first():
    torch = pytest.importorskip("torch")
    from paper_1605_02164_b200 import BfVecError, Plan
    p = Plan(8, 8, 3, 1.0, np.eye(3) * 100.0, 10, 4, 0)
    with pytest.raises(BfVecError):
        p.get_draws(with_samples=True)


def test_alias_warning_static():
    from paper_1605_02164_b200 import Plan
    # alpha R = 255/30 = 8.5 > (pi/2) sqrt(4) = 3.14 -> aliasing; N = 40 -> 9.93 > 8.5: fine
    assert Plan(8, 8, 1, 1.0, [[900.0]], 4, 4, 0).info("alias") == 1
    assert Plan(8, 8, 1, 1.0, [[900.0]], 40, 4, 0).info("alias") == 0


def test_large_radius_plan_is_recursive_only():
    """r = ceil(3 sigma_s) > 64: the plan is valid (the recursive engine runs it) but the
    truncated-window engine reports itself unsupported."""
    from paper_1605_02164_b200 import Plan
    p = Plan(16, 16, 3, 30.0, np.eye(3) * 100.0, 10, 4, 0)
    assert p.info("radius") == 90 and p.info("fir_supported") == 0
    p.set_option("engine", 1)
    assert p.info("engine") == 1
    assert Plan(16, 16, 3, 2.0, np.eye(3) * 100.0, 10, 4, 0).info("fir_supported") == 1


def test_options_validate_without_gpu():
    from paper_1605_02164_b200 import BfVecError, Plan
    p = Plan(16, 16, 3, 2.0, np.eye(3) * 100.0, 10, 4, 0)
    for name, v in [("engine", 1), ("engine", 0), ("spatial_kernel", 2), ("rec_batch", 3)]:
        p.set_option(name, v)
    for name, v in [("engine", 2), ("spatial_kernel", 5), ("rec_batch", -1), ("no_such_option", 1)]:
        with pytest.raises(BfVecError):
            p.set_option(name, v)


def test_new_entry_points_validate_arguments_without_gpu():
    """bf_vec_mse_sweep / _filter_partial_p2p / _normalize_slots / colour transforms reject bad
    arguments before touching a device (no GPU in the CPU suite)."""
    import ctypes
    from paper_1605_02164_b200 import _lib
    lib = _lib.load()
    assert lib.bf_vec_srgb_to_lab(None, None, 10, None) == -1
    assert lib.bf_vec_lab_to_srgb(None, None, 10, None) == -1
    h = ctypes.c_void_p()
    C = np.eye(3) * 100.0
    assert lib.bf_vec_plan(16, 16, 3, 1.0, C.ctypes.data_as(ctypes.c_void_p), 10, 4, 0, ctypes.byref(h)) == 0
    try:
        seeds = (ctypes.c_uint64 * 1)(1)
        tl = (ctypes.c_int * 2)(2, 1)                       # not increasing
        mse = (ctypes.c_double * 2)()
        dummy = ctypes.c_void_p(16)
        assert lib.bf_vec_mse_sweep(h, dummy, dummy, 1, seeds, 2, tl, mse, None) == -1
        peers = (ctypes.c_void_p * 1)(16)
        assert lib.bf_vec_filter_partial_p2p(h, dummy, 0, 4, peers, 9, 0, 1, None) == -1      # world > 8
        assert lib.bf_vec_filter_partial_p2p(h, dummy, 0, 2, peers, 1, 0, 3, None) == -1      # slots > samples
        assert lib.bf_vec_filter_partial_p2p(h, dummy, 0, 4, peers, 1, 0, 2, None) == -6      # not sampled yet
        assert lib.bf_vec_normalize_slots(h, dummy, 0, 0, 4, dummy, None) == -1
        # pipelined host frames: null buffers are refused; before a device is bound, BF_E_STATE
        assert lib.bf_vec_filter_host_async(h, None, dummy, None) == -1
        assert lib.bf_vec_filter_host_async(None, dummy, dummy, None) == -1
        assert lib.bf_vec_filter_host_async(h, dummy, dummy, None) == -1     # in == out
        assert lib.bf_vec_filter_host_async(h, dummy, ctypes.c_void_p(32), None) == -6
        assert lib.bf_vec_host_sync(None) == -1
        assert lib.bf_vec_host_sync(h) == -6
        # new options: documented values accepted, others refused
        for name, good, bad in (("persistent", 2, 3), ("direct_rows", 8, 5), ("rec_store", 1, 2)):
            assert lib.bf_vec_set_option(h, name.encode(), float(good)) == 0
            assert lib.bf_vec_set_option(h, name.encode(), float(bad)) == -1
    finally:
        lib.bf_vec_plan_destroy(h)


def test_plan_info_reports_every_documented_key():
    from paper_1605_02164_b200 import Plan
    p = Plan(16, 16, 3, 2.0, np.eye(3) * 100.0, 10, 4, 0)
    for k in ["radius", "d", "H", "W", "M", "N", "tile_rows", "groups", "ctas", "launches_per_filter",
              "smem_bytes", "threads", "kernel_D", "kernel_R", "regs", "occupancy", "alias", "variant",
              "spatial_kernel", "engine", "rec_batch", "fir_supported", "sampler", "colorspace"]:
        p.info(k)
    assert p.info("radius") == 6 and p.info("M") == 4
