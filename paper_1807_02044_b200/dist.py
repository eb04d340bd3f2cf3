"""Multi-GPU partitioning of the FBS hot path.

Two ways, one process per GPU under torchrun (torch.distributed process groups;
NCCL over NVLink on the GPU box, gloo in the CPU tests):

* Row bands (one large frame, BASELINE config 4): output rows are split into
  equal bands of ceil(H/G) rows.  Each rank computes its band with
  fbs_compute_rows, which reads the input rows it needs (a ρ+ϱ = ρ+1 row halo)
  straight from the full frame, so no intermediate is exchanged: LRC and
  subpixel are row-local (Eq.(9)(10)).  The one exchange step is an
  all-gather of the float bands.  Because per-output arithmetic does not
  depend on the band origin, the stitched map is bit-identical to 1 GPU.
* Frame sharding (a stream of frames, BASELINE config 5): frame i goes to rank
  i mod G; no collective on the data path.
* Disparity-range split (NEXT-3, SURVEY §8(e) "Alternative"): rank k owns a
  contiguous sub-range of [d_min, d_max] and runs the WTA over it only
  (fbs_compute_keys); the per-pixel 64-bit keys (value bits << 32 | (2^32-1-d))
  are reduced with all_reduce(MAX) — ties resolve to the smallest d exactly as in
  the single-GPU WTA — and the winner's record (c(d*-1), c(d*), c(d*+1)) with a
  masked MAX; every rank then applies LRC + subpixel (fbs_finalize_keys).  Each
  rank's handle covers its sub-range plus one disparity on each side (subpixel
  neighbours).  Useful for wide-D frames.
"""
from __future__ import annotations

from typing import Callable


def band_rows(H: int, world: int) -> int:
    """Rows per band (the last band may be shorter)."""
    return -(-H // world)


def band_range(H: int, rank: int, world: int) -> tuple[int, int]:
    """[r0, r1) output rows of ``rank``; empty (r0 == r1) if the frame is short."""
    B = band_rows(H, world)
    r0 = min(H, rank * B)
    return r0, min(H, r0 + B)


def compute_banded(compute_rows: Callable, H: int, W: int, rank: int, world: int, group=None,
                   out=None, device=None):
    """Each rank runs ``compute_rows(r0, r1, band)`` on its band (band is a
    float32 [B, W] tensor view), then the bands are all-gathered into the full
    [H, W] map, returned on every rank.  ``compute_rows`` must write rows
    [r0, r1) of the map into ``band[: r1 - r0]``."""
    import torch
    import torch.distributed as dist

    B = band_rows(H, world)
    r0, r1 = band_range(H, rank, world)
    if device is not None:
        dev = torch.device(device)
    elif out is not None:
        dev = out.device
    elif world > 1 and dist.get_backend(group) != "nccl":
        dev = torch.device("cpu")
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
    full = torch.empty((B * world, W), dtype=torch.float32, device=dev)
    band = full[rank * B:(rank + 1) * B]  # compute in place: rank's slot of the gather buffer
    if r1 > r0:
        compute_rows(r0, r1, band)
    if world > 1:
        if full.is_cuda and dist.get_backend(group) != "nccl":  # gloo gathers host tensors
            host = full.cpu()
            dist.all_gather_into_tensor(host, host[rank * B:(rank + 1) * B].clone(), group=group)
            full.copy_(host)
        else:
            dist.all_gather_into_tensor(full, band.contiguous() if not band.is_contiguous() else band,
                                        group=group)
    res = full[:H]
    if out is not None:
        out.copy_(res)
        return out
    return res


_SYMM = {}


def compute_banded_scatter(m, left, right, H: int, W: int, rank: int, world: int, group=None):
    """Row bands without the all-gather (NEXT-3 band scatter): every rank's final-map
    kernel stores its band directly into all ranks' frame buffers, which live in
    symmetric memory (torch.distributed._symmetric_memory: one [H, W] float32
    buffer per rank, peers mapped into each GPU's address space, stores over
    NVLink), then a symmetric-memory barrier.  Returns this rank's full map (a
    view of its symmetric buffer, valid until the next call).  `m` is the rank's
    FBS handle (fbs_create_band or full frame)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    key = (H, W, id(group))
    if key not in _SYMM:
        buf = symm.empty((H, W), dtype=torch.float32, device=left.device)
        hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
        _SYMM[key] = (buf, hdl)
    buf, hdl = _SYMM[key]
    r0, r1 = band_range(H, rank, world)
    hdl.barrier(channel=0)  # every rank is done reading the previous frame's map
    if r1 > r0:
        m.compute_rows_scatter(left, right, r0, r1, list(hdl.buffer_ptrs))
    hdl.barrier(channel=0)  # every band has landed in every buffer
    return buf


def shard_frames(n_frames: int, rank: int, world: int) -> list[int]:
    """Frame indices owned by ``rank`` (frame i -> rank i mod world)."""
    return list(range(rank, n_frames, world))


def drange_split(d_min: int, d_max: int, world: int) -> list[tuple[int, int]]:
    """Contiguous competing sub-ranges [lo, hi] of [d_min, d_max], one per rank
    (empty ranges, lo > hi, when world > D)."""
    D = d_max - d_min + 1
    out = []
    for r in range(world):
        lo = d_min + (r * D) // world
        hi = d_min + ((r + 1) * D) // world - 1
        out.append((lo, hi))
    return out


def handle_range(d_min: int, d_max: int, lo: int, hi: int) -> tuple[int, int]:
    """The disparity range of the handle serving competing range [lo, hi]: one
    disparity beyond each end (subpixel neighbours), clipped to [d_min, d_max],
    at least two disparities whenever d_max > d_min (fbs_create needs that)."""
    return max(d_min, lo - 1), min(d_max, hi + 1)


_SIGN = -(1 << 63)  # flips the top bit: unsigned key order == signed int64 order


def reduce_keys_local(keys: list, recs: list):
    """The reduction of the disparity-range split on one process (the same
    arithmetic the all_reduce performs across ranks): keys int64 [H, W] holding
    uint64 bits, recs float32 [H, W, 4].  Returns (keys, rec) of the winners."""
    import torch
    flipped = torch.stack([k ^ _SIGN for k in keys])
    best = flipped.max(dim=0).values
    rec = torch.full_like(recs[0], float("-inf"))
    for k, r in zip(flipped, recs):
        rec = torch.maximum(rec, torch.where((k == best).unsqueeze(-1), r, torch.full_like(r, float("-inf"))))
    return best ^ _SIGN, rec


def reduce_keys_dist(keys_l, keys_r, rec_l, group=None):
    """all_reduce(MAX) of the keys (sign-flipped int64) and of the winners'
    records across the ranks of `group`, in place.  Returns (keys_l, keys_r, rec_l)."""
    import torch
    import torch.distributed as dist
    kl, kr = keys_l ^ _SIGN, keys_r ^ _SIGN
    local_l = kl.clone()
    dist.all_reduce(kl, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(kr, op=dist.ReduceOp.MAX, group=group)
    rec = torch.where((local_l == kl).unsqueeze(-1), rec_l, torch.full_like(rec_l, float("-inf")))
    dist.all_reduce(rec, op=dist.ReduceOp.MAX, group=group)
    return kl ^ _SIGN, kr ^ _SIGN, rec


def compute_drange_split(make_handle: Callable, left, right, W: int, H: int, d_min: int, d_max: int,
                         rank: int, world: int, group=None):
    """Disparity-range split of one frame across the ranks (NEXT-3).
    make_handle(dlo, dhi) -> a volume-path FBS handle for disparities [dlo, dhi].
    Returns the final map (float32 [H, W]) on every rank."""
    import torch
    import paper_1807_02044_b200 as fbs
    lo, hi = drange_split(d_min, d_max, world)[rank]
    if lo <= hi:
        a, b = handle_range(d_min, d_max, lo, hi)
        m = make_handle(a, b)
        kl, kr, rec = m.compute_keys(left, right, lo, hi)
    else:  # more ranks than disparities: contribute nothing
        kl = torch.zeros((H, W), dtype=torch.int64, device=left.device)
        kr = torch.zeros_like(kl)
        rec = torch.full((H, W, 4), float("-inf"), device=left.device)
    if world > 1:
        kl, kr, rec = reduce_keys_dist(kl, kr, rec, group)
    return fbs.finalize_keys(W, H, d_min, d_max, kl, kr, rec.contiguous())
