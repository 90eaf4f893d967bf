"""CPU checks of the v6 kernel's persistent schedule (`persistent_items` in
csrc/plan.cu, reached through the test-only export bfvec_test_persistent_items): for many shapes
(strips nx, chunks per pass nf, passes P, CTAs nC, classic sample groups Gc)

* every strip's work line [0, P * nf) (two-sample pass x 16-row chunk) is covered by its items
  exactly once -- no chunk-step is lost or done twice;
* a strip's items use slots 0 .. nslot - 1, each once (the normaliser sums exactly those);
* items are well formed (non-empty, inside the strip) and the per-CTA offsets are monotone;
* the busiest CTA's modelled cost is within one pass (plus the fills of its item starts) of the
  ideal equal share -- the point of the schedule;
* whole rounds of classic units: in every round the CTAs' units are consecutive strips (the L2
  reuse of f's halo columns)."""
import ctypes

import numpy as np
import pytest

from paper_1605_02164_b200 import _lib


def _items(nx, nf, P, nC, Gc, fill=3.0):
    lib = _lib.load()
    fn = lib.bfvec_test_persistent_items
    fn.restype = ctypes.c_int
    cap = 4 * nC * (nx // max(1, nC) + 8) + 4 * nx * Gc + 64
    items = (ctypes.c_int * (4 * cap))()
    off = (ctypes.c_int * (nC + 1))()
    nslot = (ctypes.c_int * nx)()
    t = ctypes.c_double()
    n = fn(nx, nf, P, nC, Gc, ctypes.c_double(fill), items, cap, off, nslot, ctypes.byref(t))
    assert n >= 0, "capacity"
    it = np.frombuffer(items, dtype=np.int32)[: 4 * n].reshape(n, 4)
    return it, np.array(off[:]), np.array(nslot[:]), t.value


def _shapes():
    rng = np.random.default_rng(7)
    out = [(16, 32, 32, 148, 8), (256, 512, 256, 148, 4), (60, 68, 64, 148, 32), (32, 64, 128, 148, 32),
           (1, 1, 1, 148, 1), (3, 4, 5, 148, 2), (10, 3, 750, 148, 40), (300, 10, 3, 148, 3)]
    for _ in range(40):
        P = int(rng.integers(1, 300))
        out.append((int(rng.integers(1, 300)), int(rng.integers(1, 100)), P, int(rng.choice([1, 7, 148, 296])),
                    int(rng.integers(1, min(P, 64) + 1))))
    return out


@pytest.mark.parametrize("shape", _shapes())
def test_persistent_items_cover_each_strip_once(shape):
    nx, nf, P, nC, Gc = shape
    it, off, nslot, t_pers = _items(nx, nf, P, nC, Gc)
    assert off[0] == 0 and off[-1] == len(it) and np.all(np.diff(off) >= 0)
    assert np.all(it[:, 1] < it[:, 2]) and np.all(it[:, 1] >= 0) and np.all(it[:, 2] <= P * nf)
    assert np.all((it[:, 0] >= 0) & (it[:, 0] < nx))
    for x in range(nx):
        mine = it[it[:, 0] == x]
        cover = np.zeros(P * nf, dtype=np.int32)
        for _, a, b, _ in mine:
            cover[a:b] += 1
        assert np.all(cover == 1), f"strip {x}: coverage {np.unique(cover)}"
        assert sorted(mine[:, 3].tolist()) == list(range(nslot[x])), f"strip {x}: slots"
    # load balance: the busiest CTA is within one pass of chunk steps plus the fills of its item
    # starts (<= 3 items per CTA beyond whole rounds) of the equal share
    total = nx * P * nf
    fill = 3.0
    ideal = total / nC
    assert t_pers <= ideal + nf + (total / nC / nf + 2 * (it.shape[0] / nC + 3)) * fill + 1e-9


def test_whole_rounds_keep_neighbouring_strips_together():
    """Config 5's shape: 256 strips x 4 groups on 148 CTAs -> 6 whole rounds; in round r CTA c works
    on strip (r * 148 + c) mod 256, so concurrently running CTAs hold consecutive strips."""
    nx, nf, P, nC, Gc = 256, 512, 256, 148, 4
    it, off, nslot, _ = _items(nx, nf, P, nC, Gc)
    for c in range(nC):
        mine = it[off[c]:off[c + 1]]
        for r in range(6):
            u = r * nC + c
            assert mine[r][0] == u % nx and mine[r][1] == (P * (u // nx) // Gc) * nf
    assert nslot.max() <= Gc + 2          # a strip's tail is split into at most two extra pieces here
