"""The fused peer-store exchange (bf_vec_filter_partial_p2p + bf_vec_normalize_slots, SURVEY
§8(e) sample sharding) with TWO ranks: two processes on the one GPU of the test
box, each mapping the other's receive buffer through CUDA IPC (P2PSlots), host collectives over
gloo. The kernels never wait on each other (each rank's kernel only stores; the owners normalise
after a host barrier), so sharing one device changes timing only, not the protocol. The bands
the two ranks produce must equal the single-process bf_vec_filter output up to fp32 summation
order (conditioned pixels, reading R5), and each rank's band must come from both ranks' samples."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from workloads import CONFIGS, make_image

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, outdir):
    import torch.distributed as dist
    from paper_1605_02164_b200 import Plan, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS[2]
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed, value_range=cfg.value_range)
    p.sample_freqs()
    f = torch.from_numpy(make_image(cfg)).cuda()
    spr = 4
    slots = shard.P2PSlots(p, world, rank, slots_per_rank=spr)
    try:
        # frame-by-frame use: three calls, different images; rank 1 is made slow
        # (a GPU sleep queued ahead of its normalise) so rank 0's next kernel stores into rank 1's
        # buffer while rank 1 still has to normalise the previous call -- the alternating slot
        # sets must keep the calls apart
        for call, img in enumerate((f.flip(2).contiguous(), f.flip(1).contiguous())):
            k0, k1 = shard.sample_range(p.M, world, rank)
            peers, mine = slots.next_set()
            p.filter_partial_p2p(img, k0, k1, peers, world, rank, slots.slots_per_rank)
            torch.cuda.current_stream().synchronize()
            dist.barrier()
            if rank == 1:
                torch.cuda._sleep(200_000_000)
            ob = p.normalize_slots(mine, world * spr, rank * slots.rows, (rank + 1) * slots.rows, device=f.device)
            np.save(os.path.join(outdir, f"frame{call}_band{rank}.npy"), ob.cpu().numpy())
        out, y0, y1 = shard.filter_samples_p2p(p, f, slots)
        np.save(os.path.join(outdir, f"band{rank}.npy"), out.cpu().numpy())
        np.save(os.path.join(outdir, f"rows{rank}.npy"), np.array([y0, y1]))
        # the raw receive buffer: slot (src * spr + g) holds source rank src's group g sums of
        # this rank's band, planes 0..D-1 then Z (plane D)
        from cuda.bindings import runtime as rt
        D = p.info("kernel_D")
        raw = np.empty((world * spr, D + 1, slots.rows, cfg.W), dtype=np.float32)
        err, = rt.cudaMemcpy(raw.ctypes.data, slots.last_ptr, raw.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        assert err == rt.cudaError_t.cudaSuccess
        np.save(os.path.join(outdir, f"zslots{rank}.npy"), raw[:, D].reshape(world, spr, slots.rows, cfg.W))
        dist.barrier()            # nobody unmaps a buffer a peer may still be reading
    finally:
        slots.close()
        p.close()
        dist.destroy_process_group()


def test_two_rank_peer_exchange_matches_single_process():
    from tests.gpu import helpers as H
    cfg = CONFIGS[2]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = H.gpu_plan(cfg)
    ref = p.filter(f).cpu().numpy()
    frames = [f.flip(2).contiguous(), f.flip(1).contiguous()]
    frame_ref = [p.filter(g).cpu().numpy() for g in frames]
    frame_ok = [p.filter_partial(g, 0, cfg.M).cpu().numpy().reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d] / cfg.M
                >= H.Z_FLOOR for g in frames]
    Z = p.filter_partial(f, 0, cfg.M).cpu().numpy().reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d]
    half = p.filter_partial(f, 0, cfg.M // 2).cpu().numpy().reshape(cfg.d + 1, cfg.H, cfg.W)
    p.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(2, _free_port(), d), nprocs=2, join=True)
        bands = [np.load(os.path.join(d, f"band{r}.npy")) for r in range(2)]
        rows = [tuple(np.load(os.path.join(d, f"rows{r}.npy"))) for r in range(2)]
        zslots = [np.load(os.path.join(d, f"zslots{r}.npy")) for r in range(2)]
        fr = [np.concatenate([np.load(os.path.join(d, f"frame{c}_band{r}.npy")) for r in range(2)], axis=1)
              for c in range(2)]
    for c in range(2):
        e = np.abs(fr[c] - frame_ref[c])[:, frame_ok[c]].max()
        print(f"frame {c}: two-rank P2P vs single process max |diff| = {e:.2e}")
        assert e < 2e-3
    assert rows == [(0, cfg.H // 2), (cfg.H // 2, cfg.H)]
    got = np.concatenate(bands, axis=1)
    ok = Z / cfg.M >= H.Z_FLOOR
    err = np.abs(got - ref)[:, ok].max()
    print(f"two-rank P2P exchange vs single process: max |diff| = {err:.2e} on conditioned pixels")
    assert err < 2e-3
    # the exchange itself: owner o's slots from source rank s sum to Z over s's samples
    # [s M / 2, (s+1) M / 2) on o's band (reading R10) -- each rank filtered only its half
    Zh = [half[cfg.d], Z - half[cfg.d]]
    for o in range(2):
        y0, y1 = rows[o]
        for src in range(2):
            np.testing.assert_allclose(zslots[o][src].sum(axis=0), Zh[src][y0:y1], atol=1e-5 * cfg.M)
