"""N>1 host logic on CPU: band / view partitioning and the band gather over a
world_size-2 gloo group (the GPU box only ever has one GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_07967_b200 import sharding


def test_band_partition_examples():
    assert [b - a + 1 for a, b in sharding.band_partition(270, 8)] == [34] * 6 + [33] * 2
    bands = sharding.band_partition(270, 8)
    assert bands[0][0] == 0 and bands[-1][1] == 269
    assert all(bands[i][1] + 1 == bands[i + 1][0] for i in range(7))
    assert sharding.band_partition(3, 4) == [(0, 0), (1, 1), (2, 2), (3, 2)]   # empty last band
    assert sharding.band_pixel_rows((3, 2), 40) == (0, 0)
    assert sharding.band_pixel_rows((2, 2), 42) == (32, 42)                    # ragged bottom edge
    with pytest.raises(ValueError):
        sharding.band_partition(0, 2)


def test_views_for_rank_cover_once():
    for world in (1, 2, 4, 8):
        seen = sorted(v for r in range(world) for v in sharding.views_for_rank(64, world, r))
        assert seen == list(range(64))
    assert sharding.views_for_rank(3, 4, 3) == []


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, height, width, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid_h = -(-height // 16)
        bands = sharding.band_partition(grid_h, world)
        # every rank can build the same deterministic "frame"; it only owns its band
        frame = torch.arange(height * width * 3, dtype=torch.float32).reshape(height, width, 3)
        y0, y1 = sharding.band_pixel_rows(bands[rank], height)
        full = sharding.gather_bands(frame[y0:y1].clone(), bands, height, dist, rank, 0)
        # the in-place variant render_bands uses: dst's frame already holds its own rows
        mine = frame[y0:y1].clone()
        inplace = None
        if rank == 0:
            inplace = torch.full_like(frame, -1.0)
            inplace[y0:y1] = mine
        for w in sharding.gather_band_rows(inplace, mine, bands, height, rank, 0):
            w.wait()
        assert rank != 0 or torch.equal(inplace, frame)
        # views: weak scaling, no collective on the data path; only the max-over-ranks timing
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((bool(torch.equal(full, frame)), float(t.item())))
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("height,width", [(70, 42), (1080, 64)])
def test_band_gather_world2_gloo(height, width):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, height, width, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    ok, tmax = q.get(timeout=10)
    assert ok and tmax == 2.0


def test_band_render_union_equals_full_frame_oracle():
    """Same property the GPU test checks, stated with the oracle: rendering each
    band's tiles independently reproduces the full frame (tiles are independent,
    render.py:276-279)."""
    import paper_2408_07967_b200.scene as S
    from oracle import oracle as orc
    act = S.activate(S.gen_synthetic("mixed", 2000, 3))
    cam = S.orbit_cameras(1, 20.0, 160, 100)[0]
    img, _ = orc.render(act, cam)
    bands = sharding.band_partition(-(-100 // 16), 2)
    out = np.zeros_like(img)
    for b in bands:
        y0, y1 = sharding.band_pixel_rows(b, 100)
        out[y0:y1] = img[y0:y1]
    assert np.array_equal(out, img)


def test_balanced_band_partition_properties():
    """Work-balanced bands: contiguous, cover every row once, every rank gets a row while
    rows remain, and the heaviest band is never worse than with equal heights."""
    rng = np.random.default_rng(5)
    for grid_h, world in [(270, 8), (68, 4), (135, 2), (7, 8), (16, 1), (5, 5)]:
        for trial in range(20):
            w = rng.integers(0, 1000, grid_h)
            if trial % 3 == 0:                      # a bump in the middle, empty borders
                w = (1000 * np.exp(-0.5 * ((np.arange(grid_h) - grid_h / 2) / (grid_h / 8 + 1)) ** 2)).astype(int)
            bands = sharding.balanced_band_partition(w, world)
            assert len(bands) == world
            rows = [y for a, b in bands for y in range(a, b + 1)]
            assert rows == list(range(grid_h))
            nonempty = [b for b in bands if b[1] >= b[0]]
            assert len(nonempty) == min(world, grid_h)
            heavy = max(int(w[a:b + 1].sum()) for a, b in nonempty)
            equal = max(int(w[a:b + 1].sum()) for a, b in sharding.band_partition(grid_h, world) if b >= a)
            assert heavy <= max(equal, int(w.max()) + int(w.sum()) // world)
    # the bump: equal heights leave the middle band with most of the work
    w = np.zeros(270, int)
    w[100:170] = 100
    bal = max(int(w[a:b + 1].sum()) for a, b in sharding.balanced_band_partition(w, 8))
    eq = max(int(w[a:b + 1].sum()) for a, b in sharding.band_partition(270, 8))
    assert bal <= 900 and eq >= 3300
    assert sharding.balanced_band_partition([0, 0, 0], 2) == sharding.band_partition(3, 2)
    with pytest.raises(ValueError):
        sharding.balanced_band_partition([], 2)
