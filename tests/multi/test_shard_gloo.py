"""World-size-2 gloo tests of the multi-GPU orchestration (paper_1605_02164_b200.shard)
on CPU. The CUDA kernels are replaced by the oracle as a stand-in backend, so what is
tested is the partition arithmetic, the band-major PZ layout and the reduce-scatter."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import draws, native
from oracle import plan as oplan
from workloads.configs import random_image

H, W, D, SIG, N, M, SEED = 23, 18, 3, 1.5, 10, 9, 5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Plan:
    H, W, d, M = H, W, D, M


def _setup():
    f = random_image(H, W, D, seed=3)
    C = 900.0 * np.array([[1.0, 0.3, 0.1], [0.3, 1.0, 0.2], [0.1, 0.2, 1.0]])
    Q, a = oplan.diagonalize(C)
    Y = draws.y_draws(SEED, M, D, N)
    return f, Q, a, Y


def _oracle_partial(f, Q, a, Y):
    def partial(f_, k0, k1, rpb):
        _, P, Z = native.mcsf_full(f, Q, a, N, Y[k0:k1], SIG) if k1 > k0 else (None, np.zeros((D, H, W)), np.zeros((H, W)))
        blocks = []
        for b0 in range(0, H, rpb):
            b1 = min(H, b0 + rpb)
            blocks.append(np.concatenate([P[:, b0:b1], Z[None, b0:b1]], 0).ravel())
        return torch.from_numpy(np.concatenate(blocks))
    return partial


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1605_02164_b200 import shard
    f, Q, a, Y = _setup()
    plan = _Plan()
    if mode == "samples":
        def normalize(PZ_band, y0, y1):
            blk = PZ_band.reshape(D + 1, y1 - y0, W)
            return blk[:D] / blk[D]
        out, y0, y1 = shard.filter_samples(plan, None, partial_fn=_oracle_partial(f, Q, a, Y),
                                           normalize_fn=normalize)
        full = shard.gather_bands(out, H, band_fn=shard.sample_band)
    else:
        y0, y1 = shard.band(H, world, rank)
        s0, s1 = shard.slab_for_band(H, oplan.radius(SIG), y0, y1)
        band = native.mcsf_alg1(f[:, s0:s1], H, s0, y0, y1 - y0, Q, a, N, Y, SIG)[0]
        full = shard.gather_bands(torch.from_numpy(band), H)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["samples", "bands"])
def test_two_rank_gloo_matches_single_process(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    out = q.get(timeout=10)
    f, Q, a, Y = _setup()
    S, P, Z = native.mcsf_full(f, Q, a, N, Y, SIG)
    ok = Z / M >= 0.05
    assert out.shape == S.shape
    assert np.abs(out - S)[:, ok].max() < 1e-9


def test_partition_arithmetic():
    from paper_1605_02164_b200 import shard
    for Hh in (1, 7, 64, 8192):
        for world in (1, 2, 3, 8):
            bands = [shard.band(Hh, world, g) for g in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == Hh
            assert all(bands[g][1] == bands[g + 1][0] for g in range(world - 1))
            ks = [shard.sample_range(512, world, g) for g in range(world)]
            assert ks[0][0] == 0 and ks[-1][1] == 512 and sum(b - a for a, b in ks) == 512
            rpb, counts = shard.band_layout(Hh, 5, 3, world)
            assert sum(counts) == 4 * Hh * 5
    for (Hh, r, y0, y1) in [(100, 6, 0, 10), (100, 6, 40, 60), (100, 6, 95, 100), (5, 7, 1, 3), (1, 3, 0, 1)]:
        s0, s1 = shard.slab_for_band(Hh, r, y0, y1)
        assert (s0, s1) == native.slab_bounds(Hh, y0, y1 - y0, r)


def test_band_sharded_oracle_equals_full():
    """Band algebra without processes: bands computed from their slabs equal the full image."""
    from paper_1605_02164_b200 import shard
    f, Q, a, Y = _setup()
    S = native.mcsf_full(f, Q, a, N, Y, SIG)[0]
    r = oplan.radius(SIG)
    for world in (2, 3, 5):
        parts = []
        for g in range(world):
            y0, y1 = shard.band(H, world, g)
            s0, s1 = shard.slab_for_band(H, r, y0, y1)
            parts.append(native.mcsf_alg1(f[:, s0:s1], H, s0, y0, y1 - y0, Q, a, N, Y, SIG)[0])
        np.testing.assert_array_equal(np.concatenate(parts, 1), S)


def test_sample_shards_sum_to_full():
    from paper_1605_02164_b200 import shard
    f, Q, a, Y = _setup()
    _, P, Z = native.mcsf_full(f, Q, a, N, Y, SIG)
    for world in (2, 4):
        Ps = np.zeros_like(P)
        Zs = np.zeros_like(Z)
        for g in range(world):
            k0, k1 = shard.sample_range(M, world, g)
            if k1 > k0:
                _, p_, z_ = native.mcsf_full(f, Q, a, N, Y[k0:k1], SIG)
                Ps += p_
                Zs += z_
        np.testing.assert_allclose(Zs, Z, atol=1e-10)
        np.testing.assert_allclose(Ps, P, atol=1e-8)
