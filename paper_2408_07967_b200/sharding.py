"""Multi-GPU partitioning of the path; one process per GPU.

* views: frames share only the immutable scene, so view ``v`` goes to rank
  ``v mod world`` and no collective touches the data path;
* row bands of one frame: the tile rows are cut into ``world`` contiguous
  bands on 16-pixel boundaries; each rank renders its band (global tile
  indices, so the union of band pair lists equals the single-GPU list) and the
  bands are gathered on rank 0 with point-to-point sends (bands are unequal,
  so this is a grouped send/recv, not a padded all-gather).

Only ``torch.distributed`` is used, so the same code runs over NCCL on GPUs
and over gloo in the CPU tests.
"""

from __future__ import annotations

TILE = 16


def band_partition(grid_h: int, world: int) -> list:
    """Inclusive tile-row bands [(ty0, ty1)] per rank; earlier ranks take the
    remainder (8 GPUs x 270 rows -> 34,34,34,34,34,34,33,33).  Ranks beyond
    the number of rows get an empty band (ty0 > ty1)."""
    if grid_h < 1 or world < 1:
        raise ValueError("grid_h and world must be positive")
    per, extra = divmod(grid_h, world)
    out, y = [], 0
    for r in range(world):
        n = per + (1 if r < extra else 0)
        out.append((y, y + n - 1))
        y += n
    return out


def balanced_band_partition(row_weights, world: int, fixed_rows: float = 0.0) -> list:
    """Inclusive tile-row bands [(ty0, ty1)] per rank with (nearly) equal summed weight
    instead of equal height.  ``row_weights[ty]`` is the load estimate of tile row ``ty``
    (``Pipeline.row_weights``: in-frustum Gaussians centred in the row -- integers that every
    rank computes identically, so all ranks cut the same bands without communicating);
    ``fixed_rows`` adds a per-row cost in the same unit (pixels cost something even where no
    Gaussian lands).  Band k ends at the first row where the running weight reaches
    (k+1)/world of the total; every rank gets at least one row while rows remain.  The
    rendered frame does not depend on the cut (bands are independent)."""
    w = [float(v) + float(fixed_rows) for v in row_weights]
    grid_h = len(w)
    if grid_h < 1 or world < 1:
        raise ValueError("row_weights must be non-empty and world positive")
    total = sum(w)
    if total <= 0.0:
        return band_partition(grid_h, world)
    out, y, run = [], 0, 0.0
    for r in range(world):
        left = world - r - 1                      # ranks still to be served after this one
        if y >= grid_h:
            out.append((grid_h, grid_h - 1))      # empty band
            continue
        if left == 0:
            out.append((y, grid_h - 1))
            y = grid_h
            continue
        target = total * (r + 1) / world
        y1 = y
        run += w[y1]
        # extend while below the target, leaving at least one row for each later rank
        while run < target and y1 + 1 < grid_h - left:
            # stop early if adding the next row overshoots by more than stopping undershoots
            if run + w[y1 + 1] - target > target - run:
                break
            y1 += 1
            run += w[y1]
        out.append((y, y1))
        y = y1 + 1
    return out


def band_pixel_rows(band, height: int) -> tuple:
    """Pixel-row slice [y0, y1) covered by an inclusive tile-row band."""
    ty0, ty1 = band
    if ty1 < ty0:
        return (0, 0)
    return (ty0 * TILE, min((ty1 + 1) * TILE, height))


def views_for_rank(n_views: int, world: int, rank: int) -> list:
    """View indices rendered by ``rank`` (round robin)."""
    return list(range(rank, n_views, world))


def gather_bands(local_rows, bands, height: int, dist, rank: int, dst: int = 0):
    """Assemble the frame on ``dst`` from every rank's band rows.

    ``local_rows`` is this rank's ``(rows, W, 3)`` tensor (rows may be 0).
    Returns the full ``(H, W, 3)`` tensor on ``dst`` and ``None`` elsewhere.
    """
    import torch
    world = len(bands)
    if rank == dst:
        full = torch.empty((height,) + tuple(local_rows.shape[1:]), dtype=local_rows.dtype,
                           device=local_rows.device)
        y0, y1 = band_pixel_rows(bands[dst], height)
        full[y0:y1] = local_rows
        ops = []
        for r in range(world):
            y0, y1 = band_pixel_rows(bands[r], height)
            if r != dst and y1 > y0:
                ops.append(dist.P2POp(dist.irecv, full[y0:y1], r))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return full
    if local_rows.shape[0] > 0:
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local_rows.contiguous(), dst)]):
            w.wait()
    return None


def gather_band_rows(full, local_rows, bands, height: int, rank: int, dst: int = 0, group=None):
    """In-place band gather (what ``Pipeline.render_bands`` issues behind its blend): on
    ``dst``, ``full`` is the ``(H, W, 3)`` frame whose own band rows are already written and
    every other rank's rows are received straight into their place (row slices of a
    contiguous frame are contiguous, so no staging copy); elsewhere ``local_rows`` -- this
    rank's ``(rows, W, 3)`` band -- is sent to ``dst``.  Point-to-point because bands are
    unequal.  Returns the work handles; the caller waits on them (on CUDA tensors ``wait``
    orders the current stream behind the transfer, it does not block the host)."""
    import torch.distributed as dist
    world = len(bands)
    ops = []
    if rank == dst:
        for r in range(world):
            y0, y1 = band_pixel_rows(bands[r], height)
            if r != dst and y1 > y0:
                peer = r if group is None else dist.get_global_rank(group, r)
                ops.append(dist.P2POp(dist.irecv, full[y0:y1], peer, group))
    elif local_rows is not None and local_rows.shape[0] > 0:
        peer = dst if group is None else dist.get_global_rank(group, dst)
        ops.append(dist.P2POp(dist.isend, local_rows, peer, group))
    return dist.batch_isend_irecv(ops) if ops else []
