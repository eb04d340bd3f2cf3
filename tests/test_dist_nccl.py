"""Multi-GPU (NCCL) test of the row-band partitioner with the CUDA path: one
process per GPU (world = min(8, device count)), each rank computes its band with
fbs_compute_rows on its own GPU, the bands are NCCL all-gathered, and the
stitched map must equal the single-GPU fbs_compute map bit for bit (SURVEY §4,
§8(e)).  Skipped when fewer than 2 GPUs are visible (the round-end GPU tier has
one; the 1-GPU band stitching is tested in test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfgname, path, q):
    import torch.distributed as dist
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    from paper_1807_02044_b200 import dist as fdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    cfg = synth.CONFIGS[cfgname]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    r0, r1 = fdist.band_range(cfg.H, rank, world)
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=path,
                rows=(r0, r1) if r1 > r0 else None)
    full = fdist.compute_banded(lambda a, b, band: m.compute_rows(L, R, a, b, out=band[: b - a]),
                                cfg.H, cfg.W, rank, world)
    if rank == 0:
        q.put(full.cpu().numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("path", ["volume", "fused"])
@pytest.mark.parametrize("cfgname", ["teddy", "kitti"])
def test_nccl_bands_bit_identical(cfgname, path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for an NCCL process group")
    import torch.multiprocessing as mp
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    from paper_1807_02044_b200 import build
    build.build()
    world = min(8, torch.cuda.device_count())
    cfg = synth.CONFIGS[cfgname]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    ref = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r,
                  path=path).compute(L, R).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), cfgname, path, q), nprocs=world, join=True)
    got = q.get(timeout=60)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _drange_worker(rank, world, port, q):
    import torch.distributed as dist
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    from paper_1807_02044_b200 import dist as fdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    cfg = synth.CONFIGS["kitti"]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    out = fdist.compute_drange_split(
        lambda a, b: fbs.FBS(cfg.W, cfg.H, a, b, cfg.radius, cfg.gamma_d, cfg.gamma_r),
        L, R, cfg.W, cfg.H, cfg.d_min, cfg.d_max, rank, world)
    if rank == 0:
        q.put(out.cpu().numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_drange_split():
    """NEXT-3 over NCCL: the disparity-range split of a KITTI frame across the GPUs
    gives the single-GPU map (near-tie pixels aside)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for an NCCL process group")
    import torch.multiprocessing as mp
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    world = min(8, torch.cuda.device_count())
    cfg = synth.CONFIGS["kitti"]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    ref = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r).compute(L, R).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_drange_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    got = q.get(timeout=60)
    assert np.mean(got.view(np.uint32) == ref.view(np.uint32)) > 0.995


def _scatter_worker(rank, world, port, q):
    import torch.distributed as dist
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    from paper_1807_02044_b200 import dist as fdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    cfg = synth.CONFIGS["mb2014"]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    r0, r1 = fdist.band_range(cfg.H, rank, world)
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, rows=(r0, r1))
    full = fdist.compute_banded_scatter(m, L, R, cfg.H, cfg.W, rank, world)
    torch.cuda.synchronize()
    q.put((rank, full.cpu().numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_symmetric_memory_band_scatter():
    """NEXT-3 band scatter over NVLink: every rank's map assembled by peer stores
    into symmetric memory equals the single-GPU map bit for bit, on every rank."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for symmetric memory over NVLink")
    import torch.multiprocessing as mp
    import stereo_synth as synth
    import paper_1807_02044_b200 as fbs
    world = min(8, torch.cuda.device_count())
    cfg = synth.CONFIGS["mb2014"]
    L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
    ref = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r).compute(L, R).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_scatter_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    for _ in range(world):
        _, got = q.get(timeout=120)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
