"""Thin Python binding of libfbs.so — the B200 fast bilateral stereo (FBS) hot path.

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the C ABI declared in ``include/fbs.h``.  PyTorch supplies device
memory and streams.  There is no CPU fallback: if the extension is missing or
no CUDA device is present, calls raise.

Functions keep the C names (``fbs_create``, ``fbs_compute``, ...); the
``FBS`` class is a convenience owner of one handle.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBS_LIB", os.path.join(_HERE, "libfbs.so"))  # FBS_LIB: A/B experiments
ROOT = os.path.dirname(_HERE)

FBS_OK = 0
FBS_E_ARG, FBS_E_PARAM, FBS_E_DIM, FBS_E_UNSUPPORTED, FBS_E_CUDA, FBS_E_OOM = -1, -2, -3, -4, -5, -6
FBS_INVALID = -1.0
FBS_SENTINEL = -2.0
FBS_MAX_RADIUS = 10  # volume path; the fused path stops at 6
FBS_FUSED_MAX_RADIUS = 6
FBS_PATH_VOLUME, FBS_PATH_FUSED = 0, 1
PATHS = {"volume": FBS_PATH_VOLUME, "fused": FBS_PATH_FUSED}

# every symbol include/fbs.h declares
EXPORTS = ("fbs_create", "fbs_create_ex", "fbs_create_band", "fbs_compute_rows_scatter", "fbs_compute_keys", "fbs_finalize_keys", "fbs_suggest_ranges", "fbs_compute_ranged", "fbs_destroy", "fbs_last_error", "fbs_compute", "fbs_compute_rows",
           "fbs_compute_batch", "fbs_compute_host", "fbs_compute_host_batch", "fbs_debug_volumes", "fbs_debug_select",
           "fbs_debug_maps", "fbs_stats", "fbs_profile_enable", "fbs_profile_read", "fbs_tile_stats")
FBS_NSTAGES = 3
STAGES = ("prep", "main", "finalize")  # volume path: k_cost, k_agg, k_finalize; fused: k_prep, k_fbs, k_final

_lib = None


class FbsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"FBS error {code}: {msg}")
        self.code = code


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfbs.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    lib.fbs_create.argtypes = [I, I, I, I, I, F, F]
    lib.fbs_create.restype = P
    lib.fbs_create_ex.argtypes = [I, I, I, I, I, F, F, I]
    lib.fbs_create_ex.restype = P
    lib.fbs_create_band.argtypes = [I, I, I, I, I, F, F, I, I, I]
    lib.fbs_create_band.restype = P
    lib.fbs_compute_keys.argtypes = [P, P, P, I, I, P, P, P, P]
    lib.fbs_compute_keys.restype = I
    lib.fbs_finalize_keys.argtypes = [I, I, I, I, P, P, P, P, P]
    lib.fbs_finalize_keys.restype = I
    lib.fbs_suggest_ranges.argtypes = [P, P, I, P, P, P]
    lib.fbs_suggest_ranges.restype = I
    lib.fbs_compute_ranged.argtypes = [P, P, P, P, P, P, P]
    lib.fbs_compute_ranged.restype = I
    lib.fbs_destroy.argtypes = [P]
    lib.fbs_destroy.restype = None
    lib.fbs_last_error.argtypes = []
    lib.fbs_last_error.restype = ctypes.c_char_p
    lib.fbs_compute.argtypes = [P, P, P, P, P]
    lib.fbs_compute_rows.argtypes = [P, P, P, I, I, P, P]
    lib.fbs_compute_rows_scatter.argtypes = [P, P, P, I, I, P, I, P]
    lib.fbs_compute_rows_scatter.restype = I
    lib.fbs_compute_batch.argtypes = [P, P, P, I, P, P]
    lib.fbs_compute_host.argtypes = [P, P, P, P, P]
    lib.fbs_compute_host_batch.argtypes = [P, P, P, I, P, P]
    lib.fbs_debug_volumes.argtypes = [P, P, P, P, P, P, P, P, P, P, P]
    lib.fbs_debug_select.argtypes = [P, P, P, P, P, P, P]
    lib.fbs_debug_maps.argtypes = [P, P, P, P, P, P, P]
    lib.fbs_stats.argtypes = [P, ctypes.POINTER(I)]
    lib.fbs_profile_enable.argtypes = [P, I]
    lib.fbs_profile_read.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I)]
    lib.fbs_tile_stats.argtypes = [P] + [ctypes.POINTER(ctypes.c_longlong)] * 4
    for name in ("fbs_compute", "fbs_compute_rows", "fbs_compute_batch", "fbs_compute_host", "fbs_compute_host_batch",
                 "fbs_debug_volumes", "fbs_debug_select", "fbs_debug_maps", "fbs_stats",
                 "fbs_profile_enable", "fbs_profile_read", "fbs_tile_stats"):
        getattr(lib, name).restype = I
    _lib = lib
    return lib


def last_error() -> str:
    return load_library().fbs_last_error().decode()


def _check(rc: int):
    if rc != FBS_OK:
        raise FbsError(rc, last_error())


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ---------------------------------------------------------------------------
# C-named wrappers

def fbs_create(W: int, H: int, d_min: int, d_max: int, radius: int, sigma_s: float, sigma_r: float):
    h = load_library().fbs_create(W, H, d_min, d_max, radius, sigma_s, sigma_r)
    if not h:
        raise FbsError(FBS_E_PARAM, last_error())
    return ctypes.c_void_p(h)


def fbs_create_ex(W: int, H: int, d_min: int, d_max: int, radius: int, sigma_s: float, sigma_r: float,
                  path: int):
    h = load_library().fbs_create_ex(W, H, d_min, d_max, radius, sigma_s, sigma_r, path)
    if not h:
        raise FbsError(FBS_E_PARAM, last_error())
    return ctypes.c_void_p(h)


def fbs_create_band(W: int, H: int, d_min: int, d_max: int, radius: int, sigma_s: float, sigma_r: float,
                    path: int, row_begin: int, row_end: int):
    h = load_library().fbs_create_band(W, H, d_min, d_max, radius, sigma_s, sigma_r, path, row_begin, row_end)
    if not h:
        raise FbsError(FBS_E_PARAM, last_error())
    return ctypes.c_void_p(h)


def fbs_compute_keys(h, left, right, c_lo: int, c_hi: int, keys_l, keys_r, rec_l, stream=None) -> None:
    _check(load_library().fbs_compute_keys(h, _ptr(left), _ptr(right), c_lo, c_hi, _ptr(keys_l), _ptr(keys_r),
                                           _ptr(rec_l), _stream(stream)))


def fbs_finalize_keys(W: int, H: int, d_min: int, d_max: int, keys_l, keys_r, rec_l, disp_out,
                      stream=None) -> None:
    _check(load_library().fbs_finalize_keys(W, H, d_min, d_max, _ptr(keys_l), _ptr(keys_r), _ptr(rec_l),
                                            _ptr(disp_out), _stream(stream)))


def fbs_suggest_ranges(h, seed_disp, margin: int, ranges_l, ranges_r, stream=None) -> None:
    _check(load_library().fbs_suggest_ranges(h, _ptr(seed_disp), margin, _ptr(ranges_l), _ptr(ranges_r),
                                             _stream(stream)))


def fbs_compute_ranged(h, left, right, ranges_l, ranges_r, disp_out, stream=None) -> None:
    _check(load_library().fbs_compute_ranged(h, _ptr(left), _ptr(right), _ptr(ranges_l), _ptr(ranges_r),
                                             _ptr(disp_out), _stream(stream)))


def finalize_keys(W: int, H: int, d_min: int, d_max: int, keys_l, keys_r, rec_l, out=None, stream=None):
    """LRC + subpixel from reduced keys (int64 [H, W] holding the uint64 bits) and
    records (float32 [H, W, 4]) on their device."""
    import torch
    for t, dt, shp in ((keys_l, torch.int64, (H, W)), (keys_r, torch.int64, (H, W)), (rec_l, torch.float32, (H, W, 4))):
        if t.dtype != dt or tuple(t.shape) != shp or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"finalize_keys: expected contiguous {dt} {shp} device tensors")
    if out is None:
        out = torch.empty((H, W), dtype=torch.float32, device=keys_l.device)
    fbs_finalize_keys(W, H, d_min, d_max, keys_l, keys_r, rec_l, out, stream)
    return out


def fbs_destroy(h) -> None:
    load_library().fbs_destroy(h)


def fbs_compute(h, left, right, disp_out, stream=None) -> None:
    _check(load_library().fbs_compute(h, _ptr(left), _ptr(right), _ptr(disp_out), _stream(stream)))


def fbs_compute_rows(h, left, right, row_begin: int, row_end: int, disp_band, stream=None) -> None:
    _check(load_library().fbs_compute_rows(h, _ptr(left), _ptr(right), row_begin, row_end,
                                           _ptr(disp_band), _stream(stream)))


def fbs_compute_rows_scatter(h, left, right, row_begin: int, row_end: int, out_ptrs, stream=None) -> None:
    """out_ptrs: device addresses (ints) of full-frame float32 [H][W] buffers."""
    arr = (ctypes.c_void_p * len(out_ptrs))(*[ctypes.c_void_p(int(p)) for p in out_ptrs])
    _check(load_library().fbs_compute_rows_scatter(h, _ptr(left), _ptr(right), row_begin, row_end, arr,
                                                   len(out_ptrs), _stream(stream)))


def fbs_compute_batch(h, left, right, n: int, disp_out, stream=None) -> None:
    _check(load_library().fbs_compute_batch(h, _ptr(left), _ptr(right), n, _ptr(disp_out),
                                            _stream(stream)))


def fbs_compute_host(h, left, right, disp_out, stream=None) -> None:
    """Host (CPU, ideally pinned) uint8 inputs and float output; blocking."""
    _check(load_library().fbs_compute_host(h, _ptr(left), _ptr(right), _ptr(disp_out),
                                           _stream(stream)))


def fbs_compute_host_batch(h, left, right, n: int, disp_out, stream=None) -> None:
    """n host frames back to back (pinned for asynchronous copies); pipelined, blocking."""
    _check(load_library().fbs_compute_host_batch(h, _ptr(left), _ptr(right), n, _ptr(disp_out),
                                                 _stream(stream)))


def fbs_debug_volumes(h, left, right, cost_l=None, cost_r=None, agg_l=None, agg_r=None,
                      disp_out=None, disp_l=None, disp_r=None, stream=None) -> None:
    _check(load_library().fbs_debug_volumes(h, _ptr(left), _ptr(right), _ptr(cost_l), _ptr(cost_r),
                                            _ptr(agg_l), _ptr(agg_r), _ptr(disp_out), _ptr(disp_l),
                                            _ptr(disp_r), _stream(stream)))


def fbs_debug_select(h, agg_l, agg_r, disp_l=None, disp_r=None, disp_out=None, stream=None) -> None:
    _check(load_library().fbs_debug_select(h, _ptr(agg_l), _ptr(agg_r), _ptr(disp_l), _ptr(disp_r),
                                           _ptr(disp_out), _stream(stream)))


def fbs_debug_maps(h, left, right, disp_out, disp_l=None, disp_r=None, stream=None) -> None:
    _check(load_library().fbs_debug_maps(h, _ptr(left), _ptr(right), _ptr(disp_out), _ptr(disp_l),
                                         _ptr(disp_r), _stream(stream)))


def fbs_stats(h) -> dict:
    n = ctypes.c_int(0)
    _check(load_library().fbs_stats(h, ctypes.byref(n)))
    return {"launches": n.value}


def fbs_profile_enable(h, n: int) -> None:
    _check(load_library().fbs_profile_enable(h, n))


def fbs_profile_read(h) -> tuple[dict, int]:
    """Summed milliseconds per stage over the profiled frames, and their count."""
    arr = (ctypes.c_double * FBS_NSTAGES)()
    n = ctypes.c_int(0)
    _check(load_library().fbs_profile_read(h, arr, ctypes.byref(n)))
    return dict(zip(STAGES, list(arr))), n.value


def fbs_tile_stats(h) -> dict:
    """(warp sub-tile, d-block) counts per denominator form since the last call."""
    v = [ctypes.c_longlong(0) for _ in range(4)]
    _check(load_library().fbs_tile_stats(h, *(ctypes.byref(x) for x in v)))
    return dict(zip(("fast", "edge", "general", "empty"), (x.value for x in v)))


# ---------------------------------------------------------------------------
class FBS:
    """Owner of one handle (one per stream).  Inputs/outputs are torch tensors
    on the handle's device: uint8 [H, W] pairs in, float32 [H, W] map out."""

    def __init__(self, W: int, H: int, d_min: int, d_max: int, radius: int, sigma_s: float,
                 sigma_r: float, device=None, path: str = "volume", rows=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1807_02044_b200 needs a CUDA device (sm_100a); no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.W, self.H, self.d_min, self.d_max, self.radius = W, H, d_min, d_max, radius
        self.sigma_s, self.sigma_r = sigma_s, sigma_r
        self.D = d_max - d_min + 1
        if path not in PATHS:
            raise ValueError(f"path must be one of {sorted(PATHS)}")
        self.path = path
        self.rows = (0, H) if rows is None else (int(rows[0]), int(rows[1]))
        with torch.cuda.device(self.device):
            if rows is None:
                self.h = fbs_create_ex(W, H, d_min, d_max, radius, sigma_s, sigma_r, PATHS[path])
            else:  # band handle: serves compute_rows within `rows` only (fbs_create_band)
                self.h = fbs_create_band(W, H, d_min, d_max, radius, sigma_s, sigma_r, PATHS[path], *self.rows)

    def close(self):
        if getattr(self, "h", None):
            fbs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk_pair(self, left, right, n=None, host=False):
        """Validate an input pair: uint8, contiguous, [H, W] (or [n, H, W]), on the
        handle's device (or on the host for the *_host calls)."""
        import torch
        shape = (self.H, self.W) if n is None else (n, self.H, self.W)
        for name, t in (("left", left), ("right", right)):
            if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8 or not t.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous uint8 tensor")
            if tuple(t.shape) != shape:
                raise ValueError(f"{name}: expected shape {shape}, got {tuple(t.shape)}")
            if host and t.is_cuda:
                raise ValueError(f"{name}: expected a host tensor")
            if not host and (not t.is_cuda or t.device != self.device):
                raise ValueError(f"{name}: expected a tensor on {self.device}")

    def _out(self, out, shape, dtype=None, host=False):
        import torch
        dtype = dtype or torch.float32
        if out is None:
            if host:
                return torch.empty(shape, dtype=dtype, pin_memory=True)
            return torch.empty(shape, dtype=dtype, device=self.device)
        if out.dtype != dtype or tuple(out.shape) != tuple(shape) or not out.is_contiguous():
            raise ValueError(f"out: expected a contiguous {dtype} tensor of shape {tuple(shape)}")
        if host == out.is_cuda or (not host and out.device != self.device):
            raise ValueError("out: on the wrong device")
        return out

    def compute(self, left, right, out=None, stream=None):
        self._chk_pair(left, right)
        out = self._out(out, (self.H, self.W))
        fbs_compute(self.h, left, right, out, stream)
        return out

    def compute_rows(self, left, right, r0: int, r1: int, out=None, stream=None):
        self._chk_pair(left, right)
        if not self.rows[0] <= r0 < r1 <= self.rows[1]:
            raise ValueError(f"compute_rows: need {self.rows[0]} <= r0 < r1 <= {self.rows[1]}")
        out = self._out(out, (r1 - r0, self.W))
        fbs_compute_rows(self.h, left, right, r0, r1, out, stream)
        return out

    def compute_rows_scatter(self, left, right, r0: int, r1: int, out_ptrs, stream=None):
        """Rows [r0, r1) stored into every full-frame buffer of out_ptrs (device
        addresses of float32 [H, W] buffers, e.g. symmetric-memory peers)."""
        self._chk_pair(left, right)
        if not self.rows[0] <= r0 < r1 <= self.rows[1]:
            raise ValueError(f"compute_rows_scatter: need {self.rows[0]} <= r0 < r1 <= {self.rows[1]}")
        if not 1 <= len(out_ptrs) <= 8:
            raise ValueError("compute_rows_scatter: 1..8 destination buffers")
        fbs_compute_rows_scatter(self.h, left, right, r0, r1, out_ptrs, stream)

    def compute_batch(self, left, right, out=None, stream=None):
        n = left.shape[0]
        self._chk_pair(left, right, n=n)
        out = self._out(out, (n, self.H, self.W))
        fbs_compute_batch(self.h, left, right, n, out, stream)
        return out

    def compute_host(self, left, right, out=None, stream=None):
        self._chk_pair(left, right, host=True)
        out = self._out(out, (self.H, self.W), host=True)
        fbs_compute_host(self.h, left, right, out, stream)
        return out

    def compute_host_batch(self, left, right, out=None, stream=None):
        """left/right: host uint8 [n][H][W] (pinned); returns host float [n][H][W]."""
        n = left.shape[0]
        self._chk_pair(left, right, n=n, host=True)
        out = self._out(out, (n, self.H, self.W), host=True)
        fbs_compute_host_batch(self.h, left, right, n, out, stream)
        return out

    def volumes(self, left, right, stream=None, maps=False):
        """Debug export: cost_l, cost_r, agg_l, agg_r ([H][W][D], SENT = undefined);
        with maps=True also (disp, d_L, d_R) of the same (exporting) launch."""
        import torch
        self._chk_pair(left, right)
        shp = (self.H, self.W, self.D)
        vols = [torch.empty(shp, dtype=torch.float32, device=self.device) for _ in range(4)]
        out = dl = dr = None
        if maps:
            out = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
            dl = torch.empty((self.H, self.W), dtype=torch.int32, device=self.device)
            dr = torch.empty_like(dl)
        fbs_debug_volumes(self.h, left, right, *vols, disp_out=out, disp_l=dl, disp_r=dr, stream=stream)
        return (vols, (out, dl, dr)) if maps else vols

    def maps(self, left, right, stream=None):
        import torch
        self._chk_pair(left, right)
        out = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
        dl = torch.empty((self.H, self.W), dtype=torch.int32, device=self.device)
        dr = torch.empty_like(dl)
        fbs_debug_maps(self.h, left, right, out, dl, dr, stream)
        return out, dl, dr

    def compute_keys(self, left, right, c_lo: int, c_hi: int, stream=None):
        """Disparity-range split (volume path): the WTA over [c_lo, c_hi] only.
        Returns keys_l, keys_r (int64 [H, W] holding the uint64 keys) and rec_l
        (float32 [H, W, 4]: c(d*-1), c(d*), c(d*+1), 0)."""
        import torch
        self._chk_pair(left, right)
        kl = torch.empty((self.H, self.W), dtype=torch.int64, device=self.device)
        kr = torch.empty_like(kl)
        rec = torch.empty((self.H, self.W, 4), dtype=torch.float32, device=self.device)
        fbs_compute_keys(self.h, left, right, c_lo, c_hi, kl, kr, rec, stream)
        return kl, kr, rec

    def suggest_ranges(self, seed_disp, margin: int, stream=None):
        """NEXT-4: per-pixel suggested ranges (int16 [H, W, 2] left, right) from a
        seed disparity map (float32 [H, W], values >= 0 are feature points)."""
        import torch
        if seed_disp.dtype != torch.float32 or tuple(seed_disp.shape) != (self.H, self.W) or not seed_disp.is_cuda:
            raise ValueError("suggest_ranges: expected a float32 [H, W] device seed map")
        rl = torch.empty((self.H, self.W, 2), dtype=torch.int16, device=self.device)
        rr = torch.empty_like(rl)
        fbs_suggest_ranges(self.h, seed_disp.contiguous(), margin, rl, rr, stream)
        return rl, rr

    def compute_ranged(self, left, right, ranges_l, ranges_r, out=None, stream=None):
        """NEXT-4: fbs_compute with each pixel's WTA restricted to its range."""
        import torch
        self._chk_pair(left, right)
        for t in (ranges_l, ranges_r):
            if t.dtype != torch.int16 or tuple(t.shape) != (self.H, self.W, 2) or not t.is_cuda:
                raise ValueError("compute_ranged: expected int16 [H, W, 2] device ranges")
        out = self._out(out, (self.H, self.W))
        fbs_compute_ranged(self.h, left, right, ranges_l.contiguous(), ranges_r.contiguous(), out, stream)
        return out

    def select(self, agg_l, agg_r, stream=None):
        import torch
        for t in (agg_l, agg_r):
            if t.dtype != torch.float32 or tuple(t.shape) != (self.H, self.W, self.D) or not t.is_cuda:
                raise ValueError("select: expected device float32 [H, W, D] volumes")
        out = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
        dl = torch.empty((self.H, self.W), dtype=torch.int32, device=self.device)
        dr = torch.empty_like(dl)
        fbs_debug_select(self.h, agg_l.contiguous(), agg_r.contiguous(), dl, dr, out, stream)
        return out, dl, dr

    def profile_enable(self, n: int):
        fbs_profile_enable(self.h, n)

    def profile_read(self):
        return fbs_profile_read(self.h)

    def tile_stats(self):
        return fbs_tile_stats(self.h)

    def launches_per_frame(self) -> int:
        return fbs_stats(self.h)["launches"]
