"""The bin-slab reduce over peer memory (PeerSlabReduce, peer.cu) with two and three ranks.

Both ranks run on cuda:0 (the GPU boxes of this run have one GPU): the IPC mappings,
the cross-process flags and the slot double-buffering are the same code as across
GPUs, only the NVLink hop is missing.  Ranks >= 1 write their slabs' partial maps into
rank 0's slot buffer; rank 0 finalises.  Over several epochs (frames) the map
must equal the single-GPU map of the full histogram (FP64, slab-sum rounding only).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frames(n, w, h):
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, (h, w), dtype=np.uint8)
    return [np.roll(base, 3 * i, axis=1) for i in range(n)]


def _worker(rank, world, port, out_path, nbins, kw, kh, p, mode="root"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1711_01656_b200 as P
    from paper_1711_01656_b200.sharding import PeerBandReduce, PeerSlabReduce, slab_bounds

    w, h = 300, 170
    frames = _frames(5, w, h)
    crop = (frames[0][40:40 + kh, 70:70 + kw].astype(np.int64) * nbins) >> 8
    tmpl = np.bincount(crop.reshape(-1), minlength=nbins).astype(np.float64) / crop.size
    k0, k1 = slab_bounds(nbins, world, rank)
    red = PeerSlabReduce(w - kw + 1, h - kh + 1) if mode == "root" else PeerBandReduce(w, h, kw, kh)
    got = []
    try:
        for f in frames:
            src = torch.from_numpy(f).cuda()
            red.begin()
            P.build_and_match(src, nbins, tmpl, kw, kh, p, bin0=k0, bins=k1 - k0, partial=red.slot())
            red.publish()
            if mode == "band":
                red.finalize(p)
                if rank == 0:
                    got.append(red.map.cpu().numpy())
            elif rank == 0:
                lmap = torch.empty((h, w), dtype=torch.float64, device="cuda")
                red.finalize(lmap, w, h, kw, kh, p)
                got.append(lmap.cpu().numpy())
        assert not red.error(), "peer wait timed out"
        if rank == 0:
            want = [P.build_and_match_map(torch.from_numpy(f).cuda(), nbins, tmpl, kw, kh, p)[1].cpu().numpy()
                    for f in frames]
            np.save(out_path, np.stack([np.stack(got), np.stack(want)]))
    finally:
        red.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["root", "band"])
@pytest.mark.parametrize("world,nbins,kw,kh,p", [(2, 64, 33, 21, 1.0), (2, 40, 16, 16, 2.0), (3, 50, 20, 9, 1.0)])
def test_peer_slab_reduce(tmp_path, world, nbins, kw, kh, p, mode):
    """root: every partial into the root's slots, the root finalises; band: partials stay
    local, each rank finalises a band of rows into the root's map."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "maps.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, nbins, kw, kh, p, mode), nprocs=world, join=True)
    got, want = np.load(out)
    assert got.shape == want.shape
    err = np.abs(got - want)
    assert np.all(err <= 1e-5 * np.maximum(np.abs(want), 1e-12) + 1e-12), err.max()


def _c4_worker(rank, world, port, out_path, reduce):
    """BASELINE config 4 on `world` ranks (bin slabs of the 8192^2 x 256-bin histogram,
    strong scaling) through sharding.ShardedMapStep, the class bench.py times."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1711_01656_b200 as P
    from paper_1711_01656_b200.sharding import ShardedMapStep

    side, nbins, kw, kh = 8192, 256, 64, 64
    img = np.random.default_rng(4).integers(0, 256, size=(side, side), dtype=np.uint8)
    y0 = x0 = (side - 64) // 2
    crop = (img[y0:y0 + kh, x0:x0 + kw].astype(np.int64) * nbins) >> 8
    tmpl = np.bincount(crop.reshape(-1), minlength=nbins).astype(np.float64) / crop.size
    frame = torch.from_numpy(img).cuda()
    s = ShardedMapStep(side, side, nbins, tmpl, kw, kh, 1.0, reduce=reduce)
    try:
        assert s.bin1 - s.bin0 == nbins // world
        for _ in range(2):  # two epochs: the double-buffered partials and flags turn over
            s.step(frame)
        torch.cuda.synchronize()
        assert not s.error(), "peer wait timed out"
        if rank == 0:
            got = s.map.cpu().numpy()
            # the single-GPU map of the whole histogram (tensor not stored: fused no-store sweep)
            t = P.IntegralHistogramTensor(side, side, nbins, store=False)
            want = P.build_and_match_map(frame, nbins, tmpl, kw, kh, 1.0, out=t)[1].cpu().numpy()
            np.save(out_path, np.stack([got, want]))
        dist.barrier()
    finally:
        s.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("reduce", ["band", "root"])
def test_c4_two_ranks_match_single_gpu(tmp_path, reduce):
    """Verdict r1: the 2-rank C4 path (two 128-bin slabs, 34 GB of tensor each, both ranks
    on cuda:0 through the same IPC / flag code as across GPUs) equals the N = 1 map."""
    import torch.multiprocessing as mp

    if torch.cuda.mem_get_info()[0] < 90e9:
        pytest.skip("needs ~75 GB of device memory")
    out = str(tmp_path / "c4.npy")
    mp.spawn(_c4_worker, args=(2, _free_port(), out, reduce), nprocs=2, join=True)
    got, want = np.load(out)
    err = np.abs(got - want)
    assert np.all(err <= 1e-5 * np.maximum(np.abs(want), 1e-12)), err.max()
