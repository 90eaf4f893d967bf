"""Python binding of the C ABI (include/bfvec.h) with the same names.

torch is used only for device buffers and streams: every step of the filter
runs in libbfvec's CUDA kernels. Tensors must be contiguous float32 on a CUDA
device, planar (d, rows, W).
"""
import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import BfVecError, check

BF_W_ALIAS = 1
BF_W_SMALL_Z = 2


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, shape, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 \
            or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return ctypes.c_void_p(t.data_ptr())


def philox4x64_10(ctr, key):
    """Host evaluation of the sampler's Philox4x64-10 block function (no GPU needed)."""
    lib = _lib.load()
    c = (ctypes.c_uint64 * 4)(*[int(x) & 0xFFFFFFFFFFFFFFFF for x in ctr])
    k = (ctypes.c_uint64 * 2)(*[int(x) & 0xFFFFFFFFFFFFFFFF for x in key])
    o = (ctypes.c_uint64 * 4)()
    check(lib.bf_vec_philox4x64_10(c, k, o), "bf_vec_philox4x64_10")
    return [int(v) for v in o]


class Plan:
    """bf_vec_plan(H, W, d, sigma_s, C, N, M, seed) and the calls on it."""

    def __init__(self, H, W, d, sigma_s, C, N, M, seed, value_range=255.0):
        self._lib = _lib.load()
        C = np.ascontiguousarray(np.asarray(C, dtype=np.float64).reshape(d, d))
        h = ctypes.c_void_p()
        check(self._lib.bf_vec_plan(int(H), int(W), int(d), float(sigma_s),
                                    C.ctypes.data_as(ctypes.c_void_p), int(N), int(M),
                                    ctypes.c_uint64(int(seed)), ctypes.byref(h)), "bf_vec_plan")
        self._h = h
        self.H, self.W, self.d, self.N, self.M = int(H), int(W), int(d), int(N), int(M)
        self.sigma_s, self.seed = float(sigma_s), int(seed)
        self.set_option("value_range", value_range)

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.bf_vec_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- options / info ----------------------------------------------------
    def set_option(self, name, value):
        check(self._lib.bf_vec_set_option(self._h, name.encode(), float(value)), "bf_vec_set_option")

    def info(self, name):
        v = ctypes.c_longlong()
        check(self._lib.bf_vec_plan_info(self._h, name.encode(), ctypes.byref(v)), "bf_vec_plan_info")
        return int(v.value)

    # -- sampler -----------------------------------------------------------
    def sample_freqs(self, stream=None):
        check(self._lib.bf_vec_sample_freqs(self._h, _stream_ptr(stream)), "bf_vec_sample_freqs")
        return self

    def get_draws(self, with_samples=True):
        """(X (M,d) int32, t (M,d) float32, Q (d,d), alpha (d)); X and t are None
        if with_samples is False (works without a GPU)."""
        d, M = self.d, self.M
        Q = np.empty((d, d), dtype=np.float64)
        a = np.empty(d, dtype=np.float64)
        X = np.empty((M, d), dtype=np.int32) if with_samples else None
        t = np.empty((M, d), dtype=np.float32) if with_samples else None
        ptr = lambda arr: arr.ctypes.data_as(ctypes.c_void_p) if arr is not None else None
        check(self._lib.bf_vec_get_draws(self._h, ptr(X), ptr(t), ptr(Q), ptr(a)), "bf_vec_get_draws")
        return X, t, Q, a

    # -- filters -----------------------------------------------------------
    def filter(self, f, out=None, stream=None):
        shp = (self.d, self.H, self.W)
        if out is None:
            out = torch.empty(shp, dtype=torch.float32, device=f.device)
        self.last_status = check(self._lib.bf_vec_filter(self._h, _dev(f, shp, "f"), _dev(out, shp, "out"),
                                                         _stream_ptr(stream)), "bf_vec_filter")
        return out

    def filter_batch(self, f, out=None, stream=None):
        """bf_vec_filter_batch: f (nimg, d, H, W) device tensor -> (nimg, d, H, W)."""
        nimg = f.shape[0]
        shp = (nimg, self.d, self.H, self.W)
        if out is None:
            out = torch.empty(shp, dtype=torch.float32, device=f.device)
        self.last_status = check(self._lib.bf_vec_filter_batch(self._h, _dev(f, shp, "f"), _dev(out, shp, "out"),
                                                               int(nimg), _stream_ptr(stream)), "bf_vec_filter_batch")
        return out

    def filter_host(self, f_host, out_host=None, stream=None):
        """bf_vec_filter_host: host (pinned) tensors in and out; synchronous."""
        shp = (self.d, self.H, self.W)
        if out_host is None:
            out_host = torch.empty(shp, dtype=torch.float32, pin_memory=True)
        for t, n in ((f_host, "f_host"), (out_host, "out_host")):
            if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous() or tuple(t.shape) != shp:
                raise ValueError(f"{n} must be a contiguous float32 host tensor of shape {shp}")
        self.last_status = check(self._lib.bf_vec_filter_host(
            self._h, ctypes.c_void_p(f_host.data_ptr()), ctypes.c_void_p(out_host.data_ptr()),
            _stream_ptr(stream)), "bf_vec_filter_host")
        return out_host

    def filter_host_async(self, f_host, out_host, stream=None):
        """bf_vec_filter_host_async: enqueue one frame (pinned host tensors in and out) and return;
        the result is in out_host after host_sync(). Keep f_host / out_host alive until then."""
        shp = (self.d, self.H, self.W)
        for t, n in ((f_host, "f_host"), (out_host, "out_host")):
            if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous() or tuple(t.shape) != shp:
                raise ValueError(f"{n} must be a contiguous float32 host tensor of shape {shp}")
        self.last_status = check(self._lib.bf_vec_filter_host_async(
            self._h, ctypes.c_void_p(f_host.data_ptr()), ctypes.c_void_p(out_host.data_ptr()),
            _stream_ptr(stream)), "bf_vec_filter_host_async")
        return out_host

    def host_sync(self):
        """bf_vec_host_sync: every enqueued filter_host_async frame is in its out_host."""
        check(self._lib.bf_vec_host_sync(self._h), "bf_vec_host_sync")

    def filter_partial(self, f, k0, k1, PZ=None, rows_per_band=None, stream=None):
        rpb = self.H if rows_per_band is None else int(rows_per_band)
        n = (self.d + 1) * self.H * self.W
        if PZ is None:
            PZ = torch.empty(n, dtype=torch.float32, device=f.device)
        # validated BEFORE the call: the kernel writes n floats through the raw pointer
        if not isinstance(PZ, torch.Tensor) or PZ.numel() != n:
            raise ValueError(f"PZ must hold (d+1)*H*W = {n} floats")
        pz_ptr = _dev(PZ, tuple(PZ.shape), "PZ")
        check(self._lib.bf_vec_filter_partial(self._h, _dev(f, (self.d, self.H, self.W), "f"), int(k0), int(k1),
                                              pz_ptr, rpb, _stream_ptr(stream)), "bf_vec_filter_partial")
        return PZ

    def filter_partial_p2p(self, f, k0, k1, peer_slots, world, rank, slots_per_rank, stream=None):
        """bf_vec_filter_partial_p2p: peer_slots = list of `world` device pointers (ints)."""
        arr = (ctypes.c_void_p * world)(*[ctypes.c_void_p(int(x)) for x in peer_slots])
        check(self._lib.bf_vec_filter_partial_p2p(self._h, _dev(f, (self.d, self.H, self.W), "f"), int(k0), int(k1),
                                                  arr, int(world), int(rank), int(slots_per_rank),
                                                  _stream_ptr(stream)), "bf_vec_filter_partial_p2p")

    def normalize_slots(self, slots_ptr, nslots, row0, row1, out=None, device=None, stream=None):
        """bf_vec_normalize_slots on a raw device pointer to (nslots, D+1, rows, W) slots."""
        rows = int(row1) - int(row0)
        if out is None:
            out = torch.empty((self.d, rows, self.W), dtype=torch.float32, device=device or "cuda")
        check(self._lib.bf_vec_normalize_slots(self._h, ctypes.c_void_p(int(slots_ptr)), int(nslots), int(row0),
                                               int(row1), _dev(out, (self.d, rows, self.W), "out"),
                                               _stream_ptr(stream)), "bf_vec_normalize_slots")
        return out

    def normalize(self, PZ_band, row0, row1, out=None, stream=None):
        rows = int(row1) - int(row0)
        if PZ_band.numel() != (self.d + 1) * rows * self.W:
            raise ValueError("PZ_band must hold (d+1)*(row1-row0)*W floats")
        if out is None:
            out = torch.empty((self.d, rows, self.W), dtype=torch.float32, device=PZ_band.device)
        check(self._lib.bf_vec_normalize(self._h, _dev(PZ_band, tuple(PZ_band.shape), "PZ_band"), int(row0),
                                         int(row1), _dev(out, (self.d, rows, self.W), "out"),
                                         _stream_ptr(stream)), "bf_vec_normalize")
        return out

    def filter_rows(self, slab, slab_row0, row0, row1, out=None, stream=None):
        rows = int(row1) - int(row0)
        slab_rows = slab.shape[1]
        if out is None:
            out = torch.empty((self.d, rows, self.W), dtype=torch.float32, device=slab.device)
        self.last_status = check(self._lib.bf_vec_filter_rows(
            self._h, _dev(slab, (self.d, slab_rows, self.W), "slab"), int(slab_row0), int(slab_rows),
            int(row0), int(row1), _dev(out, (self.d, rows, self.W), "out"), _stream_ptr(stream)),
            "bf_vec_filter_rows")
        return out

    def direct(self, f, out=None, stream=None):
        shp = (self.d, self.H, self.W)
        if out is None:
            out = torch.empty(shp, dtype=torch.float32, device=f.device)
        check(self._lib.bf_vec_direct(self._h, _dev(f, shp, "f"), _dev(out, shp, "out"), _stream_ptr(stream)),
              "bf_vec_direct")
        return out

    def mse_sweep(self, f, ref, seeds, t_list, stream=None):
        """bf_vec_mse_sweep: (len(seeds), len(t_list)) array of Eq. (20) MSEs between ref and the
        MC filter over the first T samples of realisation seeds[r] (Fig. 5)."""
        shp = (self.d, self.H, self.W)
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        tl = np.ascontiguousarray(np.asarray(t_list, dtype=np.int32))
        out = np.empty((len(sd), len(tl)), dtype=np.float64)
        check(self._lib.bf_vec_mse_sweep(self._h, _dev(f, shp, "f"), _dev(ref, shp, "ref"), len(sd),
                                         sd.ctypes.data_as(ctypes.c_void_p), len(tl),
                                         tl.ctypes.data_as(ctypes.c_void_p),
                                         out.ctypes.data_as(ctypes.c_void_p), _stream_ptr(stream)),
              "bf_vec_mse_sweep")
        return out

    def diag(self):
        zm = ctypes.c_float()
        n = ctypes.c_longlong()
        check(self._lib.bf_vec_diag(self._h, ctypes.byref(zm), ctypes.byref(n)), "bf_vec_diag")
        return float(zm.value), int(n.value)


def _color(fn_name, x, out, stream):
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous() \
            or x.shape[0] != 3:
        raise ValueError("expected a contiguous float32 CUDA tensor of shape (3, ...)")
    if out is None:
        out = torch.empty_like(x)
    n = x.numel() // 3
    check(getattr(_lib.load(), fn_name)(ctypes.c_void_p(x.data_ptr()), _dev(out, tuple(x.shape), "out"), n,
                                        _stream_ptr(stream)), fn_name)
    return out


def srgb_to_lab(rgb, out=None, stream=None):
    """bf_vec_srgb_to_lab: planar (3, ...) sRGB in [0, 255] -> CIE-Lab."""
    return _color("bf_vec_srgb_to_lab", rgb, out, stream)


def lab_to_srgb(lab, out=None, stream=None):
    """bf_vec_lab_to_srgb: planar (3, ...) CIE-Lab -> sRGB in [0, 255] (no clipping)."""
    return _color("bf_vec_lab_to_srgb", lab, out, stream)


def plan_for_config(cfg):
    """Plan for a workloads.Config (BASELINE.json configs)."""
    return Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed,
                value_range=cfg.value_range)


__all__ = ["Plan", "BfVecError", "philox4x64_10", "plan_for_config", "srgb_to_lab", "lab_to_srgb", "BF_W_ALIAS",
           "BF_W_SMALL_Z"]
