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
        dist.all_gather_into_tensor(full, band.contiguous() if not band.is_contiguous() else band,
                                    group=group)
    res = full[:H]
    if out is not None:
        out.copy_(res)
        return out
    return res


def shard_frames(n_frames: int, rank: int, world: int) -> list[int]:
    """Frame indices owned by ``rank`` (frame i -> rank i mod world)."""
    return list(range(rank, n_frames, world))
