"""Multi-GPU partitions of the MCSF path, one process per GPU.

Two ways to split one image over G ranks:

* **row bands** (`filter_bands`): rank g computes output rows
  [g H / G, (g+1) H / G) from an input slab that holds every row within r of its
  band (half-sample reflection at the true image edges, reading R1) through
  `bf_vec_filter_rows`. No communication.
* **sample shards, fused exchange** (`filter_samples_p2p`): as below, but the fused kernel's
  last pass stores each finished partial tile straight into the band owner's receive slot in
  peer memory (CUDA IPC mapping, NVLink), so the exchange overlaps the computation of the other
  CTAs and there is no separate collective; owners normalise their slots.
* **sample shards** (`filter_samples`): rank g owns samples
  [floor(g M / G), floor((g+1) M / G)) (reading R10), computes raw (P, Z) sums over
  the whole image with `bf_vec_filter_partial` in band-major layout, one
  `reduce_scatter` (NCCL over NVLink on the GPU box) sums them and leaves each
  rank the (d+1) planes of its own row band, and `bf_vec_normalize` divides.

The arithmetic happens in libbfvec's kernels; this module only computes ranges
and layouts and issues the collective. The callables can be replaced (tests run
the orchestration on CPU with gloo and a stand-in backend).
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


@contextlib.contextmanager
def nvtx(name: str):
    """NVTX range on the host timeline (the C ABI marks its own calls "bfvec:<call>"): the
    exchange step of a multi-GPU run shows up by name next to them. No-op without CUDA."""
    if torch.cuda.is_available():
        torch.cuda.nvtx.range_push(name)
        try:
            yield
        finally:
            torch.cuda.nvtx.range_pop()
    else:
        yield


def band(H: int, world: int, rank: int) -> tuple:
    """Output rows [y0, y1) of rank `rank` (balanced, contiguous)."""
    return H * rank // world, H * (rank + 1) // world


def reflect(i: int, n: int) -> int:
    """Half-sample symmetric reflection into [0, n) (reading R1)."""
    p = 2 * n
    i %= p
    return i if i < n else p - 1 - i


def slab_for_band(H: int, r: int, y0: int, y1: int) -> tuple:
    """Smallest input row range [s0, s1) holding every (reflected) row within r of [y0, y1)."""
    rows = [reflect(y, H) for y in range(y0 - r, y1 + r)]
    return min(rows), max(rows) + 1


def sample_range(M: int, world: int, rank: int) -> tuple:
    """Samples [k0, k1) of rank `rank` (reading R10)."""
    return M * rank // world, M * (rank + 1) // world


def band_layout(H: int, W: int, d: int, world: int) -> tuple:
    """(rows_per_band, element counts per band) of the band-major (d+1)-plane PZ buffer
    written by bf_vec_filter_partial(..., rows_per_band)."""
    rpb = -(-H // world)
    counts = []
    for g in range(world):
        b0 = g * rpb
        b1 = min(H, b0 + rpb)
        counts.append(max(0, b1 - b0) * (d + 1) * W)
    return rpb, counts


def filter_bands(plan, slab: torch.Tensor, slab_row0: int, group=None, out=None):
    """Row-band sharding: this rank's output band from its slab (no communication).
    Returns (out_band, y0, y1)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    y0, y1 = band(plan.H, world, rank)
    return plan.filter_rows(slab, slab_row0, y0, y1, out=out), y0, y1


def filter_samples(plan, f: torch.Tensor, group=None, partial_fn=None, normalize_fn=None, out=None):
    """Sample sharding: partial sums over this rank's samples, one reduce-scatter,
    normalisation of this rank's band. Returns (out_band, y0, y1).

    partial_fn(f, k0, k1, rows_per_band) -> flat band-major PZ (default plan.filter_partial)
    normalize_fn(PZ_band, y0, y1) -> (d, y1-y0, W)     (default plan.normalize)
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H, W, d, M = plan.H, plan.W, plan.d, plan.M
    k0, k1 = sample_range(M, world, rank)
    rpb, counts = band_layout(H, W, d, world)
    if partial_fn is None:
        partial_fn = lambda f_, a, b, rows: plan.filter_partial(f_, a, b, rows_per_band=rows)  # noqa: E731
    if normalize_fn is None:
        normalize_fn = lambda PZb, a, b: plan.normalize(PZb, a, b, out=out)  # noqa: E731
    PZ = partial_fn(f, k0, k1, rpb).reshape(-1)
    PZ_band = torch.empty(counts[rank], dtype=PZ.dtype, device=PZ.device)
    with nvtx("bfvec:reduce_scatter"):
        dist.reduce_scatter(PZ_band, list(torch.split(PZ, counts)), op=dist.ReduceOp.SUM, group=group)
    y0 = min(H, rank * rpb)
    y1 = min(H, y0 + rpb)
    if y1 <= y0:
        return torch.empty((d, 0, W), dtype=PZ.dtype, device=PZ.device), y0, y1
    return normalize_fn(PZ_band, y0, y1), y0, y1


class P2PSlots:
    """This rank's receive buffer for `bf_vec_filter_partial_p2p` (world * slots_per_rank slots of
    (D+1, H/world, W) fp32) and the device pointers of every rank's buffer, mapped through CUDA IPC
    (cuda-python runtime bindings; the buffer is a plain cudaMalloc so its IPC handle covers it
    exactly). world == 1 needs no IPC.

    Reuse rule: there are TWO slot sets, used by alternate calls. After call n's
    barrier a fast rank may start call n+1's kernel, storing into its peers' buffers while a slow
    owner's normalise of call n is still queued; with one set that overwrote the partials being
    normalised. Call n+1 writes the other set, and a rank can only reach call n+2 (which reuses
    call n's set) after every owner passed call n+1's barrier -- by which point each owner has
    synchronised its stream, so its normalise of call n has finished."""

    def __init__(self, plan, world: int, rank: int, slots_per_rank: int = 4, group=None):
        from cuda.bindings import runtime as rt
        self._rt = rt
        self.world, self.rank, self.slots_per_rank = world, rank, slots_per_rank
        D = plan.info("kernel_D")
        if plan.H % world:
            raise ValueError("P2P sample sharding needs H divisible by the world size")
        self.rows = plan.H // world
        self.set_bytes = world * slots_per_rank * (D + 1) * self.rows * plan.W * 4
        self.calls = 0
        nbytes = 2 * self.set_bytes
        err, ptr = rt.cudaMalloc(nbytes)
        if err != rt.cudaError_t.cudaSuccess:
            raise MemoryError(f"cudaMalloc({nbytes}) failed: {err}")
        self.ptr = int(ptr)
        self._opened = []
        if world == 1:
            self.peers = [self.ptr]
            return
        err, h = rt.cudaIpcGetMemHandle(ptr)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaIpcGetMemHandle failed: {err}")
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h.reserved), group=group)
        peers = []
        for r, hb in enumerate(handles):
            if r == rank:
                peers.append(self.ptr)
                continue
            hh = rt.cudaIpcMemHandle_t()
            hh.reserved = hb
            err, pp = rt.cudaIpcOpenMemHandle(hh, rt.cudaIpcMemLazyEnablePeerAccess)
            if err != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaIpcOpenMemHandle(rank {r}) failed: {err}")
            self._opened.append(pp)
            peers.append(int(pp))
        self.peers = peers

    def next_set(self):
        """(peer pointers, own pointer) of the slot set this call uses; alternates per call."""
        off = (self.calls & 1) * self.set_bytes
        self.calls += 1
        return [p + off for p in self.peers], self.ptr + off

    def close(self):
        for pp in self._opened:
            self._rt.cudaIpcCloseMemHandle(pp)
        self._opened = []
        if self.ptr:
            self._rt.cudaFree(self.ptr)
            self.ptr = 0


def filter_samples_p2p(plan, f: torch.Tensor, slots: P2PSlots, group=None, out=None):
    """Sample sharding with the exchange fused into the MC kernel: partial sums over this rank's
    samples are stored by the kernel's last pass straight into the band owners' receive slots
    (NVLink peer stores), then -- once every rank's kernel has completed -- each rank normalises
    its own band from its slots. Returns (out_band, y0, y1)."""
    world, rank = slots.world, slots.rank
    k0, k1 = sample_range(plan.M, world, rank)
    peers, mine = slots.next_set()            # alternate slot sets: see P2PSlots' reuse rule
    plan.filter_partial_p2p(f, k0, k1, peers, world, rank, slots.slots_per_rank)
    if world > 1:
        with nvtx("bfvec:p2p_barrier"):
            torch.cuda.current_stream().synchronize()   # this rank's peer stores are complete ...
            dist.barrier(group)                          # ... and so are everyone else's
    y0 = rank * slots.rows
    y1 = y0 + slots.rows
    slots.last_ptr = mine
    return plan.normalize_slots(mine, world * slots.slots_per_rank, y0, y1, out=out, device=f.device), y0, y1


def gather_bands(out_band: torch.Tensor, H: int, group=None, band_fn=band) -> torch.Tensor:
    """All-gather the per-rank bands into the full (d, H, W) image (for checking)."""
    world = dist.get_world_size(group)
    d, _, W = out_band.shape
    bands = [band_fn(H, world, g) for g in range(world)]
    rmax = max(b1 - b0 for b0, b1 in bands)          # equal-size gather (gloo), trimmed after
    mine = torch.zeros((d, rmax, W), dtype=out_band.dtype, device=out_band.device)
    mine[:, :out_band.shape[1]] = out_band
    parts = [torch.empty_like(mine) for _ in bands]
    dist.all_gather(parts, mine, group=group)
    return torch.cat([p[:, :b1 - b0] for p, (b0, b1) in zip(parts, bands)], dim=1)


def sample_band(H: int, world: int, rank: int) -> tuple:
    """Row band a rank normalises in sample sharding (bands of ceil(H / world) rows)."""
    rpb = -(-H // world)
    y0 = min(H, rank * rpb)
    return y0, min(H, y0 + rpb)


__all__ = ["band", "reflect", "slab_for_band", "sample_range", "band_layout", "filter_bands",
           "filter_samples", "P2PSlots", "filter_samples_p2p", "gather_bands", "sample_band"]
