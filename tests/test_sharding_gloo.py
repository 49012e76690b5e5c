"""Multi-rank host logic of the bin-slab sharding, on CPU with gloo (world size 2 and 3).

Each rank computes its slab's partial window sums (with the CPU oracle standing in for
the CUDA kernel, which these CPU tests cannot launch), the partials are reduced with
the same helper bench.py uses, and the destination rank's finalised map must equal the
single-rank map.  The GPU equivalence of slab partials is covered by
tests/test_gpu_parity.py::test_slab_partials_recompose / test_fused_sources_and_slabs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_01656_b200.sharding import max_over_ranks, reduce_partials, slab_bounds


def test_slab_bounds_partition():
    for nbins in (1, 7, 128, 256, 1000):
        for world in (1, 2, 3, 4, 8):
            if world > nbins:
                continue
            spans = [slab_bounds(nbins, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nbins
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [k1 - k0 for k0, k1 in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_bounds(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, p):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = oracle.smooth_image(60, 44, 17)
        bins, kw, kh = 23, 13, 9
        qb = oracle.quantize(img, bins)
        crop = qb[10:10 + kh, 20:20 + kw]
        tmpl = np.bincount(crop.reshape(-1), minlength=bins).astype(np.float64) / crop.size
        k0, k1 = slab_bounds(bins, world, rank)
        part = torch.from_numpy(oracle.hist_partial(qb, bins, tmpl, kw, kh, p, k0, k1))
        reduce_partials(part, dst=0)
        slowest = max_over_ranks(float(rank + 1))
        if rank == 0:
            got = oracle.hist_finalize(part.numpy(), 60, 44, kw, kh, p)
            want = oracle.hist_match_map_direct(qb, bins, tmpl, kw, kh, p)
            np.save(out_path, np.stack([got, want]))
            assert slowest == float(world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p", [(2, 1.0), (3, 2.0)])
def test_reduce_of_slab_partials_matches_single_rank(tmp_path, world, p):
    out = str(tmp_path / "maps.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, p), nprocs=world, join=True)
    got, want = np.load(out)
    assert np.all(np.abs(got - want) <= 1e-5 * np.abs(want) + 1e-12)


def test_peer_slot_schedule():
    """PeerSlabReduce bookkeeping: slots of consecutive epochs never overlap, every slot
    lies inside the 2 * world slot buffer, and a rank waits for exactly the epoch that
    last used its slot."""
    from paper_1711_01656_b200.sharding import ack_needed, slot_offset

    for world in (1, 2, 3, 8):
        stride = 96
        for e in range(1, 7):
            cur = {slot_offset(e, r, world, stride) for r in range(world)}
            nxt = {slot_offset(e + 1, r, world, stride) for r in range(world)}
            assert len(cur) == world and not cur & nxt
            assert all(0 <= o and o + stride <= 2 * world * stride for o in cur)
            need = ack_needed(e)
            if need:
                assert slot_offset(need, 0, world, stride) == slot_offset(e, 0, world, stride)
            else:
                assert e <= 2
    with pytest.raises(ValueError):
        slot_offset(0, 0, 2, 8)


def test_band_rows_partition():
    """PeerBandReduce's row bands tile the valid rows exactly once, in rank order."""
    from paper_1711_01656_b200.sharding import band_rows

    for nv in (1, 7, 100, 4033):
        for world in (1, 2, 3, 8):
            spans = [band_rows(nv, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nv
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(v0 <= v1 for v0, v1 in spans)
    with pytest.raises(ValueError):
        band_rows(10, 2, 2)
