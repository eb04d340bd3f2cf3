"""Multi-process (gloo, CPU) tests of the row-band partitioner and the frame
sharder in paper_1807_02044_b200/dist.py.  The per-band compute here is the
oracle on the band's input rows (+ the rho+1-row halo), so the test checks the
partition / halo / gather logic independently of the GPU: the gathered map
must equal the single-process full-frame oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_02044_b200 import dist as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("H,G", [(48, 1), (48, 2), (375, 3), (1988, 8), (7, 8), (10, 4)])
def test_band_ranges_partition_rows(H, G):
    got = [fdist.band_range(H, r, G) for r in range(G)]
    rows = [y for a, b in got for y in range(a, b)]
    assert rows == list(range(H))
    B = fdist.band_rows(H, G)
    assert all(b - a <= B for a, b in got)


def test_shard_frames():
    owned = [fdist.shard_frames(10, r, 3) for r in range(3)]
    assert sorted(sum(owned, [])) == list(range(10))
    assert owned[1] == [1, 4, 7]


def _worker(rank, world, port, W, H, cfgp, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import stereo_synth as synth
    d_min, d_max, rho, gd, gr, seed = cfgp
    L, R, _, _ = synth.layered(W, H, d_min, d_max, seed, p_flat=0.3)
    halo = rho + 1

    def compute_rows(r0, r1, band):
        a, b = max(0, r0 - halo), min(H, r1 + halo)
        res = oracle.fbs(L[a:b], R[a:b], d_min, d_max, rho, gd, gr, threads=1, volumes=False)
        band[: r1 - r0] = torch.from_numpy(res.disp[r0 - a: r1 - a].astype(np.float32))

    full = fdist.compute_banded(compute_rows, H, W, rank, world, device="cpu")
    if rank == 0:
        q.put(full.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H", [(2, 40, 29), (3, 36, 20)])
def test_banded_gather_matches_single_process(world, W, H):
    import oracle
    import stereo_synth as synth
    cfgp = (0, 9, 2, 4.0, 30.0, 123)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, cfgp, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    L, R, _, _ = synth.layered(W, H, 0, 9, 123, p_flat=0.3)
    ref = oracle.fbs(L, R, 0, 9, 2, 4.0, 30.0, threads=1).disp.astype(np.float32)
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _keys_from_agg(agg, d_min, lo, hi):
    """uint64 WTA keys of an aggregated volume [H, W, D] restricted to [lo, hi]
    (value order bits << 32 | 2^32-1-d; 0 when no defined value), numpy."""
    H, W, D = agg.shape
    sub = agg[:, :, lo - d_min: hi - d_min + 1].astype(np.float32)
    valid = sub > -2.0
    v = np.where(valid, sub, -np.inf)
    idx = np.argmax(v, axis=2)  # first maximum = smallest d on ties
    best = np.take_along_axis(sub, idx[..., None], 2)[..., 0]
    bits = best.view(np.uint32).astype(np.uint64)
    order = np.where(bits >> np.uint64(31), ~bits & np.uint64(0xFFFFFFFF), bits | np.uint64(0x80000000))
    d = (lo + idx).astype(np.uint64)
    keys = (order << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - d)
    keys[~valid.any(axis=2)] = 0
    return keys


def _drange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import stereo_synth as synth
    W, H, d_min, d_max = 40, 24, 2, 29
    L, R, _, _ = synth.layered(W, H, d_min, d_max, 5, p_flat=0.3)
    res = oracle.fbs(L, R, d_min, d_max, 2, 5.0, 32.0, threads=1)
    lo, hi = fdist.drange_split(d_min, d_max, world)[rank]
    kl = torch.from_numpy(_keys_from_agg(res.agg_l, d_min, lo, hi).view(np.int64).copy())
    kr = torch.from_numpy(_keys_from_agg(res.agg_r, d_min, lo, hi).view(np.int64).copy())
    rec = torch.full((H, W, 4), float(rank))
    kl, kr, rec = fdist.reduce_keys_dist(kl, kr, rec)
    if rank == 0:
        full_l = _keys_from_agg(res.agg_l, d_min, d_min, d_max)
        full_r = _keys_from_agg(res.agg_r, d_min, d_min, d_max)
        owner = np.searchsorted([h for _, h in fdist.drange_split(d_min, d_max, world)],
                                (0xFFFFFFFF - (full_l & 0xFFFFFFFF)).astype(np.int64))
        q.put((np.array_equal(kl.numpy().view(np.uint64), full_l), np.array_equal(kr.numpy().view(np.uint64), full_r),
               np.array_equal(rec[..., 0].numpy()[full_l != 0], owner[full_l != 0].astype(np.float32))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_drange_split_reduction_gloo(world):
    """NEXT-3 host logic: sub-range keys built from the oracle's aggregated volumes,
    all_reduce(MAX) over gloo ranks == the full-range WTA keys (ties to the smallest
    d), and the masked record reduction picks the winning rank's record."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_drange_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    ok_l, ok_r, ok_rec = q.get(timeout=60)
    assert ok_l and ok_r and ok_rec


def test_drange_split_ranges():
    for d_min, d_max, G in ((0, 59, 1), (0, 59, 2), (3, 100, 5), (0, 255, 8), (0, 3, 8)):
        rs = fdist.drange_split(d_min, d_max, G)
        ds = [d for lo, hi in rs for d in range(lo, hi + 1)]
        assert ds == list(range(d_min, d_max + 1))
        for lo, hi in rs:
            if lo <= hi:
                a, b = fdist.handle_range(d_min, d_max, lo, hi)
                assert a <= lo and b >= hi and b > a and a >= d_min and b <= d_max
