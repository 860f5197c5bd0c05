"""Host side of the B200 rasterizer: the reference's Python call surface.

Mirrors ``tilesplat.pipeline`` (reference ``pipeline.py``) name for name:

* ``Pipeline(scene, sh_degree=3).render(camera, strategy, tau, background,
  workers, initial_capacity, pipelined) -> (Framebuffer, FrameStats)``
  -- ``pipeline.py:65-111``
* ``run_frame`` -- ``pipeline.py:114-119``; ``psnr`` / ``max_abs_diff`` --
  ``pipeline.py:122-139``
* stage entry points ``preprocess_and_bin`` (``binning.py:197``),
  ``sort_pairs`` (``sorting.py:101``), ``tile_range_table`` (``sorting.py:139``),
  ``render_frame`` (``render.py:273``), ``power_cutoffs`` (``extent.py:19``)
  so intermediates can be diffed stage by stage.

All compute happens in ``libflashgs_b200.so`` (hand-written sm_100a CUDA)
through the C ABI in ``include/flashgs_b200.h``; torch only owns device
memory and streams.  There is no CPU fallback: without the library or a CUDA
device these functions raise.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import time
import weakref
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _capi
from .scene import activate, is_activated_scene, is_raw_scene

TAU_DEFAULT = 1.0 / 255.0          # constants.py:8
TILE_SIZE = 16                     # constants.py:4
STRATEGIES = _capi.STRATEGIES


class UnsortedPairsError(ValueError):
    """Range extraction was handed keys that are not nondecreasing
    (reference ``sorting.py:25-26``)."""


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_07967_b200 needs a CUDA device (no CPU fallback)")
    return torch


@dataclass
class FrameStats:
    """Same fields as the reference's FrameStats (``pipeline.py:28-48``); the
    stage times are CUDA-event times of the kernels of each stage."""

    strategy: str
    tau: float
    workers: int
    preprocess_bin_ns: int = 0
    sort_ns: int = 0
    render_ns: int = 0
    total_ns: int = 0
    pairs_emitted: int = 0
    pairs_contributing: int = 0
    gaussians_retained: int = 0
    gaussians_degenerate: int = 0
    tiles_nonempty: int = 0
    pair_buffer_bytes: int = 0
    buffer_regrows: int = 0
    # extras (not in the reference)
    candidate_tiles: int = 0
    e2e_ns: int = 0                # host wall clock of the call incl. the D2H copy
    front_tiles: int = 0           # lazy_sort: heavy tiles whose nearest pairs only were sorted
    redo_tiles: int = 0            # ... of which sorted in full and blended again (not saturated)

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class Framebuffer:
    image: object                  # (H, W, 3) float32: numpy (default) or CUDA tensor
    background: np.ndarray         # (3,) float32
    alpha: object = None           # (H, W) = 1 - T_final           (extras=True)
    depth: object = None           # (H, W) = sum blend weight * z  (extras=True)
    rows: tuple = None             # pixel rows [y0, y1) of the frame the arrays hold
                                   # (the whole frame unless a band was rendered)

    @property
    def width(self) -> int:
        return int(self.image.shape[1])

    @property
    def height(self) -> int:
        return int(self.image.shape[0])


def _strategy_id(strategy):
    if strategy not in _capi.STRATEGY_ID:
        raise ValueError(f"unknown strategy {strategy!r}, expected one of {STRATEGIES}")
    return _capi.STRATEGY_ID[strategy]


def _check_sh_degree(d):
    if not 0 <= int(d) <= 3:
        raise ValueError("SH degree must be in 0..3")
    return int(d)


def _stream_ptr(torch, device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _fill_counters(stats, s):
    """Device fgs_stats record -> the reference's FrameStats counters (pipeline.py:103-110)."""
    stats.pairs_emitted = int(s["pairs_emitted"])
    stats.pairs_contributing = int(s["pairs_contributing"])
    stats.gaussians_retained = int(s["gaussians_retained"])
    stats.gaussians_degenerate = int(s["gaussians_degenerate"])
    stats.tiles_nonempty = int(s["tiles_nonempty"])
    stats.pair_buffer_bytes = 12 * stats.pairs_emitted
    stats.candidate_tiles = int(s["candidate_tiles_lo"]) | (int(s["candidate_tiles_hi"]) << 32)
    stats.front_tiles = int(s["front_tiles"])
    stats.redo_tiles = int(s["redo_tiles"])


LAZY_MIN_TILES = 512     # heavy tiles a frame must have for lazy_sort to be armed for the next one
LAZY_REDO_MAX = 8        # fronts of tiles below 4097 pairs redone in a frame before level 2 is given up


class _PinnedPool:
    """Recycles pinned host frames: a frame handed to the caller returns to the
    pool when the caller's ndarray is garbage-collected."""

    def __init__(self):
        self._free = {}
        # re-entrant: give() runs from a weakref finalizer, i.e. possibly from a garbage
        # collection that starts while this very thread holds the lock in take() / give()
        self._lock = threading.RLock()

    def take(self, torch, shape, dtype):
        key = (tuple(shape), str(dtype))
        with self._lock:
            lst = self._free.get(key)
            if lst:
                return lst.pop()
        return torch.empty(shape, dtype=dtype, pin_memory=True)

    def give(self, t):
        key = (tuple(t.shape), str(t.dtype))
        with self._lock:
            lst = self._free.setdefault(key, [])
            if len(lst) < 8:
                lst.append(t)

    def as_numpy(self, t):
        arr = t.numpy()
        weakref.finalize(arr, self.give, t)
        return arr


_pinned = _PinnedPool()


class _Workspace:
    """Per-frame device buffers for one (P, W, H, capacity): allocated once,
    reused every frame (the paper's static allocation)."""

    def __init__(self, torch, device, P, width, height, capacity):
        self.lay = _capi.layout(P, width, height, capacity)
        self.capacity = int(capacity)
        self.buf = torch.empty(int(self.lay.total_bytes), dtype=torch.uint8, device=device)
        self.base = self.buf.data_ptr()
        self.rgb = torch.empty((height, width, 3), dtype=torch.float32, device=device)
        self.alpha = None
        self.depthmap = None
        self.rgb8 = None               # (H, W, 3) uint8, allocated on first quantized render
        self.h_stats = torch.empty(_capi.STATS_BYTES, dtype=torch.uint8, pin_memory=True)
        self.h_stats_np = self.h_stats.numpy().view(_capi.STATS_DTYPE)   # same pinned bytes
        self.kcut_ptr = None
        self._events = None
        self.epoch = 1
        _capi.check(_capi.lib().fgs_workspace_init(C.c_void_p(self.base), C.byref(self.lay),
                                                   _stream_ptr(torch, device)))
        # The workspace may be used on another stream next (render_iter's lanes): its
        # initialisation must not still be running then.  Creation is rare; wait here.
        torch.cuda.current_stream(device).synchronize()

    def events(self, torch):
        """The four stage-boundary events of a timed frame, created once per workspace."""
        if self._events is None:
            self._events = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        return self._events

    def set_mode(self, sort_mode, keep_sorted_keys=False, lazy_sort=False):
        _capi.check(_capi.lib().fgs_layout_set_sort_mode(C.byref(self.lay), int(sort_mode)))
        self.lay.keep_sorted_keys = 1 if keep_sorted_keys else 0
        self.lay.lazy_sort = int(lazy_sort)            # 0 off, 1: tiles > 4096 pairs, 2: > 2048

    def next_epoch(self):
        e = self.epoch
        self.epoch += 16
        if self.epoch > 0xfffffff0:
            raise RuntimeError("workspace epoch exhausted; create a new Pipeline")
        return e

    def view(self, torch, off, nbytes, dtype):
        return self.buf[int(off):int(off) + int(nbytes)].view(dtype)

    def stats_tensor(self):
        return self.buf[int(self.lay.off_stats):int(self.lay.off_stats) + _capi.STATS_BYTES]


class Pipeline:
    """Holds a scene resident in HBM; renders frames for arbitrary cameras.

    ``scene`` may be a raw ``Scene`` or an ``ActivatedScene`` -- ours or the
    reference's own dataclasses (matched on field names), as ``pipeline.py:68-75``.
    ``render`` is safe to call from several threads on one object (each call
    takes its own workspace, SURVEY.md §8(b) threading row).

    ``sort_mode``: "tile-bucket" (default; counting pass on the tile field fused
    into emission + per-tile shared-memory sort) or "onesweep" (global LSD radix
    sort on the packed tile|depth key).  Both give the bit-identical sorted list.
    """

    def __init__(self, scene, sh_degree=3, device=None, sort_mode="tile-bucket",
                 spatial_order=None, device_activate=False, lazy_sort=True):
        if sort_mode not in _capi.SORT_MODES:
            raise ValueError(f"unknown sort_mode {sort_mode!r}, expected one of {tuple(_capi.SORT_MODES)}")
        self.sort_mode = sort_mode
        # Slots in Morton order make a CTA's Gaussians hit the same few tiles: the binning
        # kernels then reserve bucket ranges per (CTA, tile) and write contiguous runs, and
        # the blend's gathers get denser.  Results do not depend on it.  The one-sweep
        # sort's tie order needs the identity order.
        if spatial_order is None:
            spatial_order = sort_mode == "tile-bucket"
        if spatial_order and sort_mode != "tile-bucket":
            raise ValueError("spatial_order needs sort_mode='tile-bucket'")
        self.spatial_order = bool(spatial_order)
        # ``lazy_sort`` (tile-bucket only): a heavy tile is opaque long before its pair list
        # ends, so the sort orders only the nearest ~1024 pairs of each heavy tile and the
        # blend falls back to a full sort of the tiles that were not saturated by then
        # (fgs_layout.lazy_sort; level 1: tiles beyond 4096 pairs, level 2: beyond 2048).
        # Frames and counters are unchanged.  The level follows the frames (_note_fronts): off
        # while a frame has too few heavy tiles to pay for the two extra launches, capped at 1
        # when fronts of the lighter class fail, and off for good when fronts mostly fail
        # (translucent clouds).
        self._lazy_cap = 2 if (lazy_sort and sort_mode == "tile-bucket") else 0
        self.lazy_sort = self._lazy_cap             # the next frame's level (see _note_fronts)
        # ``device_activate``: a raw Scene is activated by the library (fgs_scene_activate)
        # instead of on the host.  Opacities / scales may then differ from the reference's
        # NumPy activation by 1 ulp (see the header), so frames agree within the pixel
        # tolerance but pair lists are no longer guaranteed bit-identical to the reference.
        from .scene_io import DeviceScene
        resident = isinstance(scene, DeviceScene)     # arrays already in HBM (load_ply_device)
        raw = is_raw_scene(scene) and not resident
        on_device = (bool(device_activate) and raw) or resident
        if resident:
            act = None
        elif raw:
            act = None if on_device else activate(scene)
        elif is_activated_scene(scene):
            act = scene
        else:
            raise TypeError("scene must be a Scene or ActivatedScene")
        torch = _torch()
        self.sh_degree = int(sh_degree)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        src = scene if on_device else act
        self.count = int(src.means.shape[0]) if resident else int(np.asarray(src.means).shape[0])
        L = _capi.lib()
        with torch.cuda.device(self.device):
            if resident:
                f32 = lambda a, shape: a.to(self.device, torch.float32).reshape(shape).contiguous()
            else:
                f32 = lambda a, shape: torch.from_numpy(
                    np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(shape))).to(self.device)
            P = self.count
            st = _stream_ptr(torch, self.device)
            means, sh = f32(src.means, (P, 3)), f32(src.sh, (P, 48))
            if on_device:
                logit, logs = f32(scene.logit_opacities, (P,)), f32(scene.log_scales, (P, 3))
                rawrot = f32(scene.rotations, (P, 4))
                opac, scales, rots = (torch.empty_like(logit), torch.empty_like(logs),
                                      torch.empty_like(rawrot))
                _capi.check(L.fgs_scene_activate(logit.data_ptr(), logs.data_ptr(), rawrot.data_ptr(),
                                                 P, opac.data_ptr(), scales.data_ptr(),
                                                 rots.data_ptr(), st))
                from .scene import ActivatedScene
                if resident:
                    # the host copy of a device-ingested scene is made on first use only
                    parts = (means, opac, scales, rots, sh)
                    self._activated_lazy = lambda: ActivatedScene(
                        parts[0].cpu().numpy(), parts[1].cpu().numpy(), parts[2].cpu().numpy(),
                        parts[3].cpu().numpy(), parts[4].cpu().numpy().reshape(P, 16, 3))
                else:
                    act = ActivatedScene(np.asarray(scene.means, dtype=np.float32), opac.cpu().numpy(),
                                         scales.cpu().numpy(), rots.cpu().numpy(),
                                         np.asarray(scene.sh, dtype=np.float32))
            else:
                opac = f32(act.opacities, (P,))
                scales, rots = f32(act.scales, (P, 3)), f32(act.rotations, (P, 4))
            self._activated = act
            self.scene_bytes = int(L.fgs_scene_bytes(P))
            self.packed = torch.empty(max(self.scene_bytes, 16), dtype=torch.uint8, device=self.device)
            order = None
            if self.spatial_order and P:
                order = torch.empty(P, dtype=torch.int32, device=self.device)
                nbytes = int(L.fgs_scene_order_scratch_bytes(P))
                scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
                _capi.check(L.fgs_scene_order(means.data_ptr(), P, order.data_ptr(),
                                              scratch.data_ptr(), nbytes, st))
            _capi.check(L.fgs_scene_pack(means.data_ptr(), opac.data_ptr(), scales.data_ptr(),
                                         rots.data_ptr(), sh.data_ptr(),
                                         order.data_ptr() if order is not None else None, P,
                                         self.packed.data_ptr(), st))
            torch.cuda.current_stream(self.device).synchronize()
            # slot -> caller index, for mapping slot-indexed results back at the boundary
            self.slot_order = (order.cpu().numpy().view(np.uint32).astype(np.int64)
                               if order is not None else None)
            del order
        self._kcut = {}
        self._free = {}
        self._lock = threading.Lock()
        self._last_pairs = 0

    @property
    def activated(self):
        """The activated scene as host arrays (for a device-ingested scene: copied back
        on first use)."""
        if self._activated is None:
            self._activated = self._activated_lazy()
            self._activated_lazy = None
        return self._activated

    @classmethod
    def from_ply(cls, path, **kw):
        """Scene ingest on the device: ``load_ply_device`` +
        on-device activation + packing; the host never re-lays the scene out."""
        from .scene_io import load_ply_device
        return cls(load_ply_device(path, kw.get("device")), **kw)

    def row_weights(self, camera, tau=TAU_DEFAULT):
        """Load estimate per tile row for the multi-GPU row-band split:
        in-frustum Gaussians whose projected centre lies in the row (``fgs_row_histogram``),
        as a NumPy int64 array of ``ceil(height / 16)`` counts.  Exact integers: every rank
        of a band job gets the same array and hence the same
        ``sharding.balanced_band_partition``."""
        torch = _torch()
        gh = -(-int(camera.height) // TILE_SIZE)
        cam = _capi.camera_struct(camera)
        with torch.cuda.device(self.device):
            hist = torch.empty(gh, dtype=torch.int32, device=self.device)
            _capi.check(_capi.lib().fgs_row_histogram(self.packed.data_ptr(), self.count, C.byref(cam),
                                                      float(tau), hist.data_ptr(),
                                                      _stream_ptr(torch, self.device)))
            return hist.cpu().numpy().view(np.uint32).astype(np.int64)

    # -- per-tau cutoff table (extent.py:19-30), cached -------------------------
    def _cutoffs(self, torch, tau):
        key = float(tau)
        with self._lock:
            k = self._kcut.get(key)
        if k is None:
            k = torch.empty(max(self.count, 1), dtype=torch.float32, device=self.device)
            _capi.check(_capi.lib().fgs_power_cutoffs(self.packed.data_ptr(), self.count, key,
                                                      k.data_ptr(), _stream_ptr(torch, self.device)))
            with self._lock:
                if len(self._kcut) > 8:
                    self._kcut.clear()
                self._kcut[key] = k
        return k

    # -- workspace pool ---------------------------------------------------------
    def _default_capacity(self):
        return int(max(1 << 16, 8 * self.count, 1.25 * self._last_pairs + 4096))

    def _take_ws(self, torch, width, height, capacity):
        key = (int(width), int(height))
        with self._lock:
            lst = self._free.get(key, [])
            for i, ws in enumerate(lst):
                if ws.capacity >= capacity:
                    return lst.pop(i)
            if lst:
                lst.pop()          # too small: drop one, allocate a bigger one
        return _Workspace(torch, self.device, self.count, width, height, capacity)

    def _give_ws(self, ws):
        key = (int(ws.lay.width), int(ws.lay.height))
        with self._lock:
            lst = self._free.setdefault(key, [])
            if len(lst) < 4:
                lst.append(ws)

    def _note_fronts(self, stats, level, s):
        """What the next frame's ``lazy_sort`` level is, from what this one showed (it was
        rendered at ``level``; ``s`` = its device stats).  A front pays only while heavy tiles
        saturate inside it, and only on frames with enough heavy tiles to cover the two extra
        kernel launches (~10 us).  Level 2 also takes the tiles of 2049..4096 pairs: those that
        fail are long tiles blended alone at the end of the frame, so a handful of them is
        already a net loss and caps the level at 1."""
        if not self._lazy_cap:
            return
        heavy1 = stats.front_tiles
        heavy2 = heavy1 + int(s["medium_tiles"])
        used, redo = (heavy2 if level >= 2 else heavy1), stats.redo_tiles
        if level and used >= 16 and 4 * redo > used:
            self._lazy_cap = 0                          # fronts mostly fail: stop guessing
        elif level >= 2 and redo > LAZY_REDO_MAX:
            self._lazy_cap = 1
        if self._lazy_cap >= 2 and heavy2 >= LAZY_MIN_TILES:
            self.lazy_sort = 2
        elif self._lazy_cap >= 1 and heavy1 >= LAZY_MIN_TILES:
            self.lazy_sort = 1
        else:
            self.lazy_sort = 0

    # -- the hot path -----------------------------------------------------------
    def _issue(self, torch, L, ws, cam, tau, deg, sid, bg_c, flags, b0, b1, out_ptr, a_ptr, d_ptr,
               st, timing):
        """Enqueue one frame on stream ``st``.  Without stage timing it is ONE C call
        (``fgs_render``: the kernels chain by programmatic dependent launch); with it, the
        stage entry points with an event at each of the reference's three stage boundaries
        (pipeline.py:84-102)."""
        base, lay = C.c_void_p(ws.base), C.byref(ws.lay)
        if not timing:
            _capi.check(L.fgs_render(self.packed.data_ptr(), ws.kcut_ptr, self.count, C.byref(cam),
                                     float(tau), deg, sid, bg_c, flags, b0, b1, ws.next_epoch(),
                                     out_ptr, a_ptr, d_ptr, base, lay, st))
            return None
        ev = ws.events(torch)
        ev[0].record()
        _capi.check(L.fgs_preprocess(self.packed.data_ptr(), ws.kcut_ptr, self.count,
                                     C.byref(cam), float(tau), deg, sid, b0, b1, base, lay, st))
        _capi.check(L.fgs_scan(base, lay, st))
        _capi.check(L.fgs_emit(self.packed.data_ptr(), C.byref(cam), sid, b0, b1, base, lay, st))
        ev[1].record()
        _capi.check(L.fgs_sort(base, lay, ws.next_epoch(), st))
        _capi.check(L.fgs_ranges(base, lay, st))
        ev[2].record()
        _capi.check(L.fgs_blend(self.packed.data_ptr(), bg_c, float(tau), flags, b0, b1,
                                out_ptr, a_ptr, d_ptr, base, lay, st))
        ev[3].record()
        return ev

    def render(self, camera, strategy="precise", tau=TAU_DEFAULT,
               background=(0.0, 0.0, 0.0), workers=1, initial_capacity=None,
               pipelined=True, *, exact=False, extras=False, contrib=True,
               as_numpy=True, band=None, timing=True, quantized=False):
        """bin -> sort -> render on the GPU; returns (Framebuffer, FrameStats).

        ``workers`` and ``pipelined`` are accepted for signature compatibility
        and do not change the result (the reference guarantees the same).
        Keyword-only extras: ``exact`` (bit-identical frame, FP64 expf),
        ``extras`` (alpha + depth maps), ``contrib`` (pairs_contributing),
        ``as_numpy`` (False: CUDA tensors, no D2H), ``timing`` (False: no stage
        times in the stats; the frame is then a single C call), ``quantized`` (the
        image comes back as uint8, quantised on the device exactly like
        ``images.py:12-15``; a quarter of the bytes to read back), and
        ``band=(ty0, ty1)``: only that tile-row band is rendered (multi-GPU row
        splitting, see ``render_bands``) and the returned image holds just the
        band's pixel rows, ``Framebuffer.rows = (y0, y1)``.
        """
        torch = _torch()
        t_host0 = time.perf_counter_ns()
        sid = _strategy_id(strategy)
        deg = _check_sh_degree(self.sh_degree)
        L = _capi.lib()
        cam = _capi.camera_struct(camera)
        W, H = int(camera.width), int(camera.height)
        gh = -(-H // TILE_SIZE)
        b0, b1 = (0, gh - 1) if band is None else (int(band[0]), int(band[1]))
        if not (0 <= b0 <= b1 < gh):
            raise ValueError(f"band {band!r} outside the {gh} tile rows")
        y0, y1 = b0 * TILE_SIZE, min((b1 + 1) * TILE_SIZE, H)      # pixel rows rendered
        bg = np.asarray(background, dtype=np.float32).reshape(3)
        bg_c = (C.c_float * 3)(*bg.tolist())
        flags = (_capi.BLEND_EXACT if exact else 0) | (_capi.BLEND_CONTRIB if contrib else 0)
        stats = FrameStats(strategy=strategy, tau=float(tau), workers=max(1, int(workers)))
        capacity = int(initial_capacity) if initial_capacity is not None else self._default_capacity()
        capacity = max(capacity, 1)

        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            st = C.c_void_p(stream.cuda_stream)
            kcut = self._cutoffs(torch, tau)
            while True:
                ws = self._take_ws(torch, W, H, capacity)
                lazy_level = int(self.lazy_sort)
                ws.set_mode(_capi.SORT_MODES[self.sort_mode], lazy_sort=lazy_level)
                ws.kcut_ptr = kcut.data_ptr()
                if extras:
                    if ws.alpha is None:
                        ws.alpha = torch.empty((H, W), dtype=torch.float32, device=self.device)
                        ws.depthmap = torch.empty((H, W), dtype=torch.float32, device=self.device)
                    a_ptr, d_ptr = ws.alpha.data_ptr(), ws.depthmap.data_ptr()
                else:
                    a_ptr = d_ptr = None
                ev = self._issue(torch, L, ws, cam, tau, deg, sid, bg_c, flags, b0, b1,
                                 ws.rgb.data_ptr(), a_ptr, d_ptr, st, timing)
                out_img = ws.rgb
                if quantized:
                    if ws.rgb8 is None:
                        ws.rgb8 = torch.empty((H, W, 3), dtype=torch.uint8, device=self.device)
                    _capi.check(L.fgs_quantize_rgb8(ws.rgb[y0:y1].data_ptr(), (y1 - y0) * W * 3,
                                                    ws.rgb8[y0:y1].data_ptr(), st))
                    out_img = ws.rgb8
                ws.h_stats.copy_(ws.stats_tensor(), non_blocking=True)
                h_rgb = None
                if as_numpy:
                    h_rgb = _pinned.take(torch, (y1 - y0, W, 3), out_img.dtype)
                    h_rgb.copy_(out_img[y0:y1], non_blocking=True)
                    if extras:
                        h_a = _pinned.take(torch, (y1 - y0, W), torch.float32)
                        h_d = _pinned.take(torch, (y1 - y0, W), torch.float32)
                        h_a.copy_(ws.alpha[y0:y1], non_blocking=True)
                        h_d.copy_(ws.depthmap[y0:y1], non_blocking=True)
                stream.synchronize()
                s = ws.h_stats_np[0]
                if int(s["overflow"]):
                    # binning.py:134-143: grow, never truncate; counted in the stats
                    stats.buffer_regrows += 1
                    need = max(int(s["pairs_emitted"]), 2 * int(s["list_used"]))
                    capacity = max(int(capacity * 1.5) + 16, need + need // 8 + 4096)
                    if h_rgb is not None:
                        _pinned.give(h_rgb)
                    continue
                break
            if int(s["bad_depth"]):
                self._give_ws(ws)
                raise ValueError("depths must be positive and finite (cull failed upstream)")
            if timing:
                stats.preprocess_bin_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
                stats.sort_ns = int(ev[1].elapsed_time(ev[2]) * 1e6)
                stats.render_ns = int(ev[2].elapsed_time(ev[3]) * 1e6)
                stats.total_ns = int(ev[0].elapsed_time(ev[3]) * 1e6)
            _fill_counters(stats, s)
            self._note_fronts(stats, lazy_level, s)
            self._last_pairs = max(self._last_pairs, stats.pairs_emitted)
            if as_numpy:
                fb = Framebuffer(_pinned.as_numpy(h_rgb), bg)
                if extras:
                    fb.alpha, fb.depth = _pinned.as_numpy(h_a), _pinned.as_numpy(h_d)
            else:
                fb = Framebuffer(out_img[y0:y1].clone(), bg)
                if extras:
                    fb.alpha, fb.depth = ws.alpha[y0:y1].clone(), ws.depthmap[y0:y1].clone()
            fb.rows = (y0, y1)
            self._give_ws(ws)
        stats.e2e_ns = time.perf_counter_ns() - t_host0
        return fb, stats

    def render_bands(self, camera, group=None, strategy="precise", tau=TAU_DEFAULT,
                     background=(0.0, 0.0, 0.0), *, bands=None, dst=0, out=None, exact=False,
                     contrib=True, as_numpy=True, sync=True, quantized=False):
        """ONE frame split into tile-row bands over the ranks of ``group`` (a
        ``torch.distributed`` process group, default: the world), gathered on rank ``dst``
        (the reference splits a frame's tiles over its worker pool the same
        way, render.py:293-309).  Call it on every rank with the same arguments.

        Every rank holds the whole scene and renders the band ``bands[rank]`` -- by default
        the work-balanced bands of ``sharding.balanced_band_partition(self.row_weights(camera))``,
        which every rank derives identically without communicating.  The blend writes the
        band straight into the buffer that is sent: on ``dst`` the full ``(H, W, 3)`` frame
        (``out`` or a fresh tensor) in which the other ranks' rows are received in place, on
        the other ranks a band-sized buffer.  The receives are posted on a side stream before
        ``dst``'s own band is rendered, the sends are issued right behind each band's blend;
        NCCL send/recv over NVLink, no other collective.  The frame is bit-identical to
        ``render(camera)`` on one GPU (tiles are independent).  ``quantized=True`` gathers the
        frame as uint8 (each rank quantises its band on the device, ``images.py:12-15``):
        a quarter of the bytes into ``dst``, whose NVLink ingress is what bounds a frame of
        many bands.

        Returns ``(Framebuffer, FrameStats)``: on ``dst`` the whole frame (host array, or the
        device tensor with ``as_numpy=False``), elsewhere the rank's own band rows
        (``Framebuffer.rows``).  The counters are those of the rank's band.  ``sync=False``
        (device tensors only) leaves the gather enqueued on the current stream and skips the
        stats read-back, for callers that time a sequence of frames on the device."""
        torch = _torch()
        import torch.distributed as dist
        from . import sharding
        t_host0 = time.perf_counter_ns()
        if not dist.is_initialized():
            raise RuntimeError("render_bands needs an initialised torch.distributed process group")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        sid = _strategy_id(strategy)
        deg = _check_sh_degree(self.sh_degree)
        L = _capi.lib()
        cam = _capi.camera_struct(camera)
        W, H = int(camera.width), int(camera.height)
        gh = -(-H // TILE_SIZE)
        if bands is None:
            if world == 1:
                bands = [(0, gh - 1)]
            else:
                rw = self.row_weights(camera, tau)
                bands = sharding.balanced_band_partition(rw, world, fixed_rows=0.3 * float(rw.mean()))
        if len(bands) != world:
            raise ValueError(f"{len(bands)} bands for {world} ranks")
        b0, b1 = int(bands[rank][0]), int(bands[rank][1])
        y0, y1 = sharding.band_pixel_rows((b0, b1), H)
        if sync is False and as_numpy:
            raise ValueError("sync=False needs as_numpy=False")
        bg = np.asarray(background, dtype=np.float32).reshape(3)
        bg_c = (C.c_float * 3)(*bg.tolist())
        flags = (_capi.BLEND_EXACT if exact else 0) | (_capi.BLEND_CONTRIB if contrib else 0)
        stats = FrameStats(strategy=strategy, tau=float(tau), workers=world)
        capacity = self._default_capacity()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            st = C.c_void_p(stream.cuda_stream)
            kcut = self._cutoffs(torch, tau)
            fdt = torch.uint8 if quantized else torch.float32
            band_f32 = None
            if rank == dst:
                full = out if out is not None else torch.empty((H, W, 3), dtype=fdt, device=self.device)
                if tuple(full.shape) != (H, W, 3) or full.dtype != fdt or not full.is_contiguous():
                    raise ValueError(f"out must be a contiguous {fdt} (H, W, 3) CUDA tensor")
                rows = None
                if quantized:      # blend into a float band, quantise it into the frame's rows
                    band_f32 = torch.empty((max(y1 - y0, 0), W, 3), dtype=torch.float32, device=self.device)
                    frame_ptr = band_f32.data_ptr() - y0 * W * 12
                else:
                    frame_ptr = full.data_ptr()
                # the peers' rows land in place while this rank renders its own band: the
                # receives go on a side stream that does not wait for the render stream
                side = self._side_streams(torch, 1)[0]
                side.wait_stream(stream)          # `full` may still be in use by earlier work
                with torch.cuda.stream(side):
                    works = sharding.gather_band_rows(full, None, bands, H, rank, dst, group)
            else:
                full = None
                rows = torch.empty((max(y1 - y0, 0), W, 3), dtype=fdt, device=self.device)
                band_f32 = torch.empty_like(rows, dtype=torch.float32) if quantized else rows
                # the blend addresses pixels by their frame row: shift the base so that row y0
                # of the frame is row 0 of the band buffer (only rows y0..y1 are written)
                frame_ptr = band_f32.data_ptr() - y0 * W * 12
                works = None
            while True:
                ws = self._take_ws(torch, W, H, capacity)
                ws.set_mode(_capi.SORT_MODES[self.sort_mode], lazy_sort=self.lazy_sort)
                ws.kcut_ptr = kcut.data_ptr()
                if b1 >= b0:
                    self._issue(torch, L, ws, cam, tau, deg, sid, bg_c, flags, b0, b1,
                                C.c_void_p(frame_ptr), None, None, st, False)
                    if quantized:
                        q_dst = full[y0:y1] if rank == dst else rows
                        _capi.check(L.fgs_quantize_rgb8(band_f32.data_ptr(), (y1 - y0) * W * 3,
                                                        q_dst.data_ptr(), st))
                if not sync:
                    break
                ws.h_stats.copy_(ws.stats_tensor(), non_blocking=True)
                stream.synchronize()
                s = ws.h_stats_np[0]
                if b1 >= b0 and int(s["overflow"]):
                    stats.buffer_regrows += 1
                    need = max(int(s["pairs_emitted"]), 2 * int(s["list_used"]))
                    capacity = max(int(capacity * 1.5) + 16, need + need // 8 + 4096)
                    self._give_ws(ws)
                    continue
                if b1 >= b0:
                    if int(s["bad_depth"]):
                        self._give_ws(ws)
                        raise ValueError("depths must be positive and finite (cull failed upstream)")
                    _fill_counters(stats, s)
                    self._last_pairs = max(self._last_pairs, stats.pairs_emitted)
                break
            self._give_ws(ws)
            if rank != dst:
                works = sharding.gather_band_rows(None, rows, bands, H, rank, dst, group)
                for w_ in works:
                    w_.wait()
                img = rows
            else:
                with torch.cuda.stream(side):
                    for w_ in works:
                        w_.wait()
                stream.wait_stream(side)          # the frame is complete behind this point
                img = full
            fb_rows = (0, H) if rank == dst else (y0, y1)
            if as_numpy:
                h = _pinned.take(torch, tuple(img.shape), img.dtype)
                h.copy_(img, non_blocking=True)
                stream.synchronize()
                fb = Framebuffer(_pinned.as_numpy(h), bg)
            else:
                fb = Framebuffer(img, bg)
            fb.rows = fb_rows
        stats.e2e_ns = time.perf_counter_ns() - t_host0
        return fb, stats

    def render_many(self, cameras, strategy="precise", tau=TAU_DEFAULT,
                    background=(0.0, 0.0, 0.0), *, exact=False, contrib=True, depth=6, streams=3,
                    quantized=False):
        """``list(render_iter(...))``: every view's ``(Framebuffer, FrameStats)``."""
        return list(self.render_iter(cameras, strategy, tau, background, exact=exact,
                                     contrib=contrib, depth=depth, streams=streams,
                                     quantized=quantized))

    def _side_streams(self, torch, n):
        pool = getattr(self, "_streams", None)
        if pool is None:
            pool = self._streams = []
        while len(pool) < n:
            pool.append(torch.cuda.Stream(device=self.device))
        return pool[:n]

    def render_iter(self, cameras, strategy="precise", tau=TAU_DEFAULT,
                    background=(0.0, 0.0, 0.0), *, exact=False, contrib=True, depth=6, streams=3,
                    quantized=False):
        """Throughput path for a batch of views (BASELINE config 5; the reference's
        ``bench_frames`` loop, ``pipeline.py:212-233``): same frames and stats as calling
        ``render`` per camera, but up to ``depth`` frames are in flight, issued round-robin
        on ``streams`` CUDA streams, each frame one C-ABI call (``fgs_render``) followed by
        its device->host copy on the same stream.  Frames on different streams overlap on
        the GPU: the latency-bound binning kernels of one view fill the issue slots the
        blend of the previous view leaves idle, and the copy engine works in parallel
        (measured on C2: 450 us per view against 570 us back to back).  Yields
        ``(Framebuffer, FrameStats)`` in camera order; host frames are pinned buffers that
        return to a pool when the caller drops them."""
        torch = _torch()
        from collections import deque
        sid = _strategy_id(strategy)
        deg = _check_sh_degree(self.sh_degree)
        L = _capi.lib()
        bg = np.asarray(background, dtype=np.float32).reshape(3)
        bg_c = (C.c_float * 3)(*bg.tolist())
        flags = (_capi.BLEND_EXACT if exact else 0) | (_capi.BLEND_CONTRIB if contrib else 0)
        nstreams = max(1, int(streams))
        depth = max(nstreams, int(depth))
        inflight = deque()

        def finish(job):
            cam_obj, ws, h_rgb, done, t0, lazy_level = job
            done.synchronize()
            s = np.frombuffer(ws.h_stats.numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
            self._give_ws(ws)
            if int(s["overflow"]) or int(s["bad_depth"]):
                _pinned.give(h_rgb)          # grow-and-rerun / raise through the plain path
                return self.render(cam_obj, strategy, tau, background, exact=exact,
                                   contrib=contrib, timing=False, quantized=quantized)
            st = FrameStats(strategy=strategy, tau=float(tau), workers=1)
            _fill_counters(st, s)
            self._note_fronts(st, lazy_level, s)
            self._last_pairs = max(self._last_pairs, st.pairs_emitted)
            st.e2e_ns = time.perf_counter_ns() - t0
            return Framebuffer(_pinned.as_numpy(h_rgb), bg), st

        with torch.cuda.device(self.device):
            caller = torch.cuda.current_stream(self.device)
            kcut = self._cutoffs(torch, tau)
            lanes = self._side_streams(torch, nstreams)
            fork = torch.cuda.Event()
            fork.record(caller)                     # scene upload / cutoffs happen-before
            for st_ in lanes:
                st_.wait_event(fork)
            issued = 0
            try:
                for cam_obj in cameras:
                    while len(inflight) >= depth:
                        yield finish(inflight.popleft())
                    t0 = time.perf_counter_ns()
                    cam = _capi.camera_struct(cam_obj)
                    W, H = int(cam_obj.width), int(cam_obj.height)
                    gh = -(-H // TILE_SIZE)
                    ws = self._take_ws(torch, W, H, self._default_capacity())
                    lazy_level = int(self.lazy_sort)
                    ws.set_mode(_capi.SORT_MODES[self.sort_mode], lazy_sort=lazy_level)
                    lane = lanes[issued % nstreams]
                    issued += 1
                    _capi.check(L.fgs_render(self.packed.data_ptr(), kcut.data_ptr(), self.count,
                                             C.byref(cam), float(tau), deg, sid, bg_c, flags, 0, gh - 1,
                                             ws.next_epoch(), ws.rgb.data_ptr(), None, None,
                                             C.c_void_p(ws.base), C.byref(ws.lay),
                                             C.c_void_p(lane.cuda_stream)))
                    out_img = ws.rgb
                    if quantized:
                        if ws.rgb8 is None:
                            ws.rgb8 = torch.empty((H, W, 3), dtype=torch.uint8, device=self.device)
                        _capi.check(L.fgs_quantize_rgb8(ws.rgb.data_ptr(), H * W * 3,
                                                        ws.rgb8.data_ptr(),
                                                        C.c_void_p(lane.cuda_stream)))
                        out_img = ws.rgb8
                    h_rgb = _pinned.take(torch, (H, W, 3), out_img.dtype)
                    with torch.cuda.stream(lane):
                        h_rgb.copy_(out_img, non_blocking=True)
                        ws.h_stats.copy_(ws.stats_tensor(), non_blocking=True)
                        done = torch.cuda.Event()
                        done.record(lane)
                    inflight.append((cam_obj, ws, h_rgb, done, t0, lazy_level))
                while inflight:
                    yield finish(inflight.popleft())
            finally:
                for st_ in lanes:                   # later work on the caller's stream is ordered
                    caller.wait_stream(st_)


def sorted_pairs(pipe, camera, strategy="precise", tau=TAU_DEFAULT, band=None):
    """K1..K5 of the frame path for one camera; returns the device-sorted
    (keys uint64, values uint32, starts int64) as numpy -- what the blend consumes."""
    torch = _torch()
    sid = _strategy_id(strategy)
    L = _capi.lib()
    cam = _capi.camera_struct(camera)
    W, H = int(camera.width), int(camera.height)
    gh = -(-H // TILE_SIZE)
    b0, b1 = (0, gh - 1) if band is None else (int(band[0]), int(band[1]))
    capacity = pipe._default_capacity()
    with torch.cuda.device(pipe.device):
        st = _stream_ptr(torch, pipe.device)
        kcut = pipe._cutoffs(torch, tau)
        while True:
            ws = pipe._take_ws(torch, W, H, capacity)
            ws.set_mode(_capi.SORT_MODES[pipe.sort_mode], keep_sorted_keys=True)
            lay, base = C.byref(ws.lay), C.c_void_p(ws.base)
            _capi.check(L.fgs_preprocess(pipe.packed.data_ptr(), kcut.data_ptr(), pipe.count,
                                         C.byref(cam), float(tau), _check_sh_degree(pipe.sh_degree),
                                         sid, b0, b1, base, lay, st))
            _capi.check(L.fgs_scan(base, lay, st))
            _capi.check(L.fgs_emit(pipe.packed.data_ptr(), C.byref(cam), sid, b0, b1, base, lay, st))
            _capi.check(L.fgs_sort(base, lay, ws.next_epoch(), st))
            _capi.check(L.fgs_ranges(base, lay, st))
            s = np.frombuffer(ws.stats_tensor().cpu().numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
            if int(s["overflow"]):
                capacity = max(int(capacity * 1.5) + 16,
                               max(int(s["pairs_emitted"]), 2 * int(s["list_used"])) + 4096)
                continue
            break
        M, lay = int(s["pairs_emitted"]), ws.lay
        keys = ws.view(torch, lay.off_keys[lay.sorted_keys_in], M * 8, torch.int64) \
            .cpu().numpy().view(np.uint64).copy()
        vals = ws.view(torch, lay.off_vals[lay.sorted_vals_in], M * 4, torch.int32) \
            .cpu().numpy().view(np.uint32).copy()
        starts = ws.view(torch, lay.off_starts, (lay.tiles + 1) * 4, torch.int32) \
            .cpu().numpy().astype(np.int64)
        pipe._give_ws(ws)
    return keys, vals, starts


# FP32 operations of one (pixel, pair) evaluation by where the reference's loop leaves it
# (render.py:106-129, counted as SURVEY.md 8(d) does): rectangle-rejected 2 sub + 4 compare;
# cutoff-rejected + 9 for the quadratic form + 1 compare; alpha-rejected + neg, exp, mul, min,
# compare; blended + alpha*T, 3 FMA (= 6), 1 - alpha, T *=, compare.
EVAL_FLOPS = {"rect_rejected": 6, "cutoff_rejected": 16, "alpha_rejected": 21, "blended": 31}


def blend_eval_counts(pipe, camera, strategy="precise", tau=TAU_DEFAULT):
    """Measurement aid for the blend's FP32 roofline: renders ``camera`` and re-blends the
    frame's sorted pairs with the counting variant of the exact kernel (``fgs_blend_counts``).
    Returns the (pixel, pair) evaluation counts of the reference's naive loop by outcome,
    ``pairs_processed`` (M_proc: pairs visited before their tile's last pixel stopped),
    ``pixels``, ``pairs_emitted`` and ``flops`` (EVAL_FLOPS-weighted)."""
    torch = _torch()
    sid = _strategy_id(strategy)
    L = _capi.lib()
    cam = _capi.camera_struct(camera)
    W, H = int(camera.width), int(camera.height)
    gh = -(-H // TILE_SIZE)
    bg_c = (C.c_float * 3)(0.0, 0.0, 0.0)
    capacity = pipe._default_capacity()
    with torch.cuda.device(pipe.device):
        st = _stream_ptr(torch, pipe.device)
        kcut = pipe._cutoffs(torch, tau)
        while True:
            ws = pipe._take_ws(torch, W, H, capacity)
            ws.set_mode(_capi.SORT_MODES[pipe.sort_mode])
            lay, base = C.byref(ws.lay), C.c_void_p(ws.base)
            _capi.check(L.fgs_render(pipe.packed.data_ptr(), kcut.data_ptr(), pipe.count, C.byref(cam),
                                     float(tau), _check_sh_degree(pipe.sh_degree), sid, bg_c, 0, 0,
                                     gh - 1, ws.next_epoch(), ws.rgb.data_ptr(), None, None, base,
                                     lay, st))
            s = np.frombuffer(ws.stats_tensor().cpu().numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
            if int(s["overflow"]):
                capacity = max(int(capacity * 1.5) + 16,
                               max(int(s["pairs_emitted"]), 2 * int(s["list_used"])) + 4096)
                continue
            break
        ev = torch.zeros(8, dtype=torch.int64, device=pipe.device)
        _capi.check(L.fgs_blend_counts(pipe.packed.data_ptr(), bg_c, float(tau), 0, gh - 1,
                                       ws.rgb.data_ptr(), ev.data_ptr(), base, lay, st))
        c = ev.cpu().numpy()
        pipe._give_ws(ws)
    out = {k: int(c[i]) for i, k in enumerate(EVAL_FLOPS)}
    out["flops"] = sum(EVAL_FLOPS[k] * out[k] for k in EVAL_FLOPS)
    out["pairs_processed"], out["pixels"] = int(c[4]), int(c[5])
    out["pairs_emitted"] = int(s["pairs_emitted"])
    return out


def run_frame(scene, camera, strategy="precise", tau=TAU_DEFAULT,
              background=(0.0, 0.0, 0.0), workers=1, sh_degree=3, **kwargs):
    """One-shot convenience wrapper (``pipeline.py:114-119``)."""
    return Pipeline(scene, sh_degree=sh_degree).render(
        camera, strategy, tau, background, workers, **kwargs)


def _img(a):
    x = a.image if isinstance(a, Framebuffer) else a
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.asarray(x)


def psnr(a, b):
    """PSNR in dB over [0, 1] channels; "identical" when MSE is 0 (``pipeline.py:122-131``)."""
    ia, ib = _img(a), _img(b)
    if ia.shape != ib.shape:
        raise ValueError(f"shape mismatch: {ia.shape} vs {ib.shape}")
    mse = float(np.mean((ia.astype(np.float64) - ib.astype(np.float64)) ** 2))
    if mse == 0.0:
        return "identical"
    return 10.0 * math.log10(1.0 / mse)


def max_abs_diff(a, b) -> float:
    ia, ib = _img(a), _img(b)
    if ia.size == 0:
        return 0.0
    return float(np.max(np.abs(ia.astype(np.float64) - ib.astype(np.float64))))


# ----------------------------------------------------------------------------
# stage-level entry points (numpy in / numpy out), for stage-by-stage diffs
# ----------------------------------------------------------------------------

@dataclass
class BinOutput:
    """Same fields as the reference's BinOutput (``binning.py:150-173``)."""

    splat: np.ndarray
    depth: np.ndarray
    retained: np.ndarray
    tile_rects: np.ndarray
    tile_counts: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    emitted_count: int
    gaussians_retained: int
    gaussians_degenerate: int
    buffer_regrows: int
    capacity: int
    grid_w: int
    grid_h: int
    strategy: str
    tau: float
    pair_counts: np.ndarray = field(default=None, repr=False)

    @property
    def pair_buffer_bytes(self) -> int:
        return self.emitted_count * 12


def power_cutoffs(alpha0, tau=TAU_DEFAULT):
    """(k float32, keep mask) on the GPU (``extent.py:19-30``)."""
    torch = _torch()
    a = np.ascontiguousarray(np.atleast_1d(alpha0), dtype=np.float32)
    n = a.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    L = _capi.lib()
    # pack a throw-away scene whose only live field is the opacity
    z3, z4, zs = np.zeros((n, 3), np.float32), np.zeros((n, 4), np.float32), np.zeros((n, 48), np.float32)
    t = [torch.from_numpy(x).to(dev) for x in (z3, a, z3, z4, zs)]
    packed = torch.empty(max(int(L.fgs_scene_bytes(n)), 16), dtype=torch.uint8, device=dev)
    st = _stream_ptr(torch, dev)
    _capi.check(L.fgs_scene_pack(*[x.data_ptr() for x in t], None, n, packed.data_ptr(), st))
    k = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    _capi.check(L.fgs_power_cutoffs(packed.data_ptr(), n, float(tau), k.data_ptr(), st))
    return k[:n].cpu().numpy(), a > np.float32(tau)


def preprocess_and_bin(scene, camera, strategy="precise", tau=TAU_DEFAULT, workers=1,
                       sh_degree=3, chunk_size=None, initial_capacity=None,
                       band=None, sort_mode=None) -> BinOutput:
    """K1 + K2 + K3 for one camera; pairs come back unsorted (``binning.py:197-372``):
    in ascending Gaussian index with ``sort_mode="onesweep"``, bucketed by tile
    (arbitrary order inside a bucket) with ``"tile-bucket"``."""
    torch = _torch()
    sid = _strategy_id(strategy)
    deg = _check_sh_degree(sh_degree)
    pipe = scene if isinstance(scene, Pipeline) else Pipeline(scene, sh_degree=deg)
    mode = pipe.sort_mode if sort_mode is None else sort_mode
    if mode not in _capi.SORT_MODES:
        raise ValueError(f"unknown sort_mode {mode!r}")
    L = _capi.lib()
    cam = _capi.camera_struct(camera)
    W, H = int(camera.width), int(camera.height)
    gw, gh = -(-W // TILE_SIZE), -(-H // TILE_SIZE)
    b0, b1 = (0, gh - 1) if band is None else (int(band[0]), int(band[1]))
    capacity = max(1, int(initial_capacity) if initial_capacity is not None
                   else pipe._default_capacity())
    regrows = 0
    P = pipe.count
    with torch.cuda.device(pipe.device):
        st = _stream_ptr(torch, pipe.device)
        kcut = pipe._cutoffs(torch, tau)
        while True:
            ws = pipe._take_ws(torch, W, H, capacity)
            ws.set_mode(_capi.SORT_MODES[mode])
            lay, base = C.byref(ws.lay), C.c_void_p(ws.base)
            _capi.check(L.fgs_preprocess(pipe.packed.data_ptr(), kcut.data_ptr(), P, C.byref(cam),
                                         float(tau), deg, sid, b0, b1, base, lay, st))
            _capi.check(L.fgs_scan(base, lay, st))
            _capi.check(L.fgs_emit(pipe.packed.data_ptr(), C.byref(cam), sid, b0, b1, base, lay, st))
            s = np.frombuffer(ws.stats_tensor().cpu().numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
            if int(s["overflow"]):
                regrows += 1
                need = max(int(s["pairs_emitted"]), 2 * int(s["list_used"]))
                capacity = max(int(capacity * 1.5) + 16, need)
                continue
            break
        if int(s["bad_depth"]):
            raise ValueError("depths must be positive and finite (cull failed upstream)")
        M = int(s["pairs_emitted"])
        lay = ws.lay
        flags = ws.view(torch, lay.off_flags, P, torch.uint8).cpu().numpy()
        retained = (flags & 1).astype(bool)
        splat = ws.view(torch, lay.off_splat, P * 48, torch.float32).cpu().numpy().reshape(P, 12).copy()
        splat[~retained] = 0.0                           # binning.py:208 zero rows
        depth = ws.view(torch, lay.off_depth, P * 4, torch.float32).cpu().numpy().copy()
        rects = ws.view(torch, lay.off_rects, P * 8, torch.int16).cpu().numpy() \
            .view(np.uint16).reshape(P, 4).astype(np.int32)
        counts = ws.view(torch, lay.off_counts, P * 4, torch.int32).cpu().numpy().view(np.uint32).copy()
        keys = ws.view(torch, lay.off_keys[0], M * 8, torch.int64).cpu().numpy().view(np.uint64).copy()
        # a band frame writes splat rows only for Gaussians with candidate tiles in the band
        splat[(rects[:, 3] < b0) | (rects[:, 1] > b1)] = 0.0
        if mode == "tile-bucket":
            # records are (depth bits << 32 | index), bucketed by tile: rebuild the
            # reference's (tile << 32 | depth bits, index) pairs from the range table
            starts = ws.view(torch, lay.off_starts, (lay.tiles + 1) * 4, torch.int32).cpu().numpy()
            tile_of = np.repeat(np.arange(lay.tiles, dtype=np.uint64), np.diff(starts.astype(np.int64)))
            vals = (keys & np.uint64(0xffffffff)).astype(np.uint32)
            keys = (tile_of << np.uint64(32)) | (keys >> np.uint64(32))
        else:
            vals = ws.view(torch, lay.off_vals[0], M * 4, torch.int32).cpu().numpy().view(np.uint32).copy()
        cap = ws.capacity
        pipe._give_ws(ws)
    if pipe.slot_order is not None:
        # per-Gaussian frame buffers are indexed by slot: row of Gaussian slot_order[slot]
        def by_index(a):
            out = np.empty_like(a)
            out[pipe.slot_order] = a
            return out
        flags, retained, splat, depth, rects, counts = (
            by_index(x) for x in (flags, retained, splat, depth, rects, counts))
    nx = rects[:, 2] - rects[:, 0] + 1
    ny = rects[:, 3] - rects[:, 1] + 1
    return BinOutput(
        splat=splat, depth=depth, retained=retained, tile_rects=rects,
        tile_counts=np.where(retained, (nx * ny).astype(np.int64), 0),
        keys=keys, values=vals, emitted_count=M,
        gaussians_retained=int(s["gaussians_retained"]),
        gaussians_degenerate=int(s["gaussians_degenerate"]),
        buffer_regrows=regrows, capacity=int(cap), grid_w=gw, grid_h=gh,
        strategy=strategy, tau=float(tau), pair_counts=counts.astype(np.int64))


def _byte_width(max_exclusive: int) -> int:
    if max_exclusive <= 1:
        return 0
    return ((int(max_exclusive) - 1).bit_length() + 7) // 8


_sort_epoch = [1]


def sort_pairs(keys, values, workers=1, grid_tiles=None, max_value=None):
    """Sort pairs by key, ties by ascending value, on the GPU (``sorting.py:101-136``).
    Inputs are not mutated; returns new numpy arrays."""
    torch = _torch()
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    values = np.ascontiguousarray(values, dtype=np.uint32)
    n = keys.shape[0]
    if values.shape[0] != n:
        raise ValueError("keys and values must have equal length")
    if n == 0:
        return keys.copy(), values.copy()
    value_bits = 32 if max_value is None else 8 * _byte_width(int(max_value))
    tile_bits = 32 if grid_tiles is None else 8 * _byte_width(int(grid_tiles))
    dev = torch.device("cuda", torch.cuda.current_device())
    L = _capi.lib()
    k_in = torch.from_numpy(keys.view(np.int64)).to(dev)
    v_in = torch.from_numpy(values.view(np.int32)).to(dev)
    k_out, v_out = torch.empty_like(k_in), torch.empty_like(v_in)
    nbytes = int(L.fgs_sort_pairs_scratch_bytes(n))
    scratch = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    _sort_epoch[0] += 64
    _capi.check(L.fgs_sort_pairs(k_in.data_ptr(), v_in.data_ptr(), n, tile_bits, value_bits,
                                 k_out.data_ptr(), v_out.data_ptr(), scratch.data_ptr(), nbytes,
                                 _sort_epoch[0], _stream_ptr(torch, dev)))
    return k_out.cpu().numpy().view(np.uint64), v_out.cpu().numpy().view(np.uint32)


def tile_range_table(sorted_keys, grid_w, grid_h) -> np.ndarray:
    """Half-open per-tile ranges as a (tiles + 1,) int64 array (``sorting.py:139-152``)."""
    torch = _torch()
    keys = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
    tiles = int(grid_w) * int(grid_h)
    dev = torch.device("cuda", torch.cuda.current_device())
    k = torch.from_numpy(keys.view(np.int64)).to(dev)
    starts = torch.empty(tiles + 1, dtype=torch.int32, device=dev)
    stats = torch.zeros(_capi.STATS_BYTES, dtype=torch.uint8, device=dev)
    _capi.check(_capi.lib().fgs_tile_ranges(k.data_ptr() if keys.size else None, keys.shape[0],
                                            tiles, starts.data_ptr(), stats.data_ptr(),
                                            _stream_ptr(torch, dev)))
    s = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=_capi.STATS_DTYPE)[0]
    if int(s["unsorted"]):
        raise UnsortedPairsError("pair keys are not nondecreasing")
    if int(s["tile_out_of_grid"]):
        raise ValueError("tile index exceeds the grid")
    return starts.cpu().numpy().astype(np.int64)


def render_frame(splat, sorted_values, starts, width, height, background, tau,
                 workers=1, pipelined=True, *, exact=False, gaussian_depth=None):
    """K6 on caller-supplied arrays (``render.py:273-310``).  Returns
    (image (H,W,3) float32, contrib flags per pair, nonempty tile count), plus
    (alpha, depth) maps when ``gaussian_depth`` is given."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    sp = torch.from_numpy(np.ascontiguousarray(splat, dtype=np.float32)).to(dev)
    vals_np = np.ascontiguousarray(sorted_values, dtype=np.uint32)
    vals = torch.from_numpy(vals_np.view(np.int32)).to(dev)
    st_np = np.ascontiguousarray(starts, dtype=np.int64)
    st32 = torch.from_numpy(st_np.astype(np.int32)).to(dev)
    bg = np.asarray(background, dtype=np.float32).reshape(3)
    bg_c = (C.c_float * 3)(*bg.tolist())
    rgb = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
    contrib = torch.zeros(max(vals_np.shape[0], 1), dtype=torch.uint8, device=dev)
    stats = torch.zeros(_capi.STATS_BYTES, dtype=torch.uint8, device=dev)
    extras = gaussian_depth is not None
    if extras:
        gd = torch.from_numpy(np.ascontiguousarray(gaussian_depth, dtype=np.float32)).to(dev)
        alpha = torch.empty((height, width), dtype=torch.float32, device=dev)
        dmap = torch.empty((height, width), dtype=torch.float32, device=dev)
    gh = -(-int(height) // TILE_SIZE)
    flags = (_capi.BLEND_EXACT if exact else 0) | _capi.BLEND_CONTRIB
    _capi.check(_capi.lib().fgs_blend_tiles(
        sp.data_ptr() if sp.numel() else None, gd.data_ptr() if extras else None,
        vals.data_ptr() if vals.numel() else None, st32.data_ptr(), int(width), int(height),
        bg_c, float(tau), flags, 0, gh - 1, rgb.data_ptr(),
        alpha.data_ptr() if extras else None, dmap.data_ptr() if extras else None,
        contrib.data_ptr(), stats.data_ptr(), _stream_ptr(torch, dev)))
    nonempty = int(np.count_nonzero(np.diff(st_np) > 0))
    out = (rgb.cpu().numpy(), contrib[:vals_np.shape[0]].cpu().numpy(), nonempty)
    if extras:
        out = out + (alpha.cpu().numpy(), dmap.cpu().numpy())
    return out
