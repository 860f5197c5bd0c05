#!/usr/bin/env python
"""Benchmark of the rasterizer hot path (contract: see the task's bench.py rules).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload c4-4k|c1|c2|c2-dense|c3|c4|c5] [--mode views|bands]

A *step* is one frame: one pass of preprocess -> tile scan -> emit -> tile sort ->
blend over one camera view of a synthetic scene that is already resident in HBM.
Default workload = the north-star frame of BASELINE.json: 10M Gaussians (generator
`mixed`, seed 1, density-scaled per SURVEY.md 8(d)), SH degree 3, 3840x2160 -- the
largest configuration the metric ("ms/frame at 1080p & 4K by Gaussian count") is quoted
on that fits one GPU.  The line also carries a short run of configs[1] (1M Gaussians,
1920x1080) under `also.c2`.  Metric = views/sec (whole job, all GPUs); `ms_per_step` is
its inverse per GPU, `ms_per_frame` the latency of one frame issued alone.  The timed
views are DISTINCT cameras of an orbit (16, or the 64 of configs[4]); with N > 1
(torchrun, one rank per GPU) every rank holds the whole scene and renders its own views
-- independent units, no data-path collective ("scaling": "weak"); `--mode bands`
instead splits ONE frame into tile-row bands whose gather (NCCL) is inside the timed
region.

The frames are rendered the way `Pipeline.render` renders them, i.e. with `lazy_sort` at the
level the pipeline settled on during the warm-up frames (`config.lazy_sort`; `--no-lazy` = every
tile sorted in full): same frames, contrib flags and counters either way (tests/test_lazy_sort.py).

One JSON line is printed by rank 0.
  value      device-timed: K views issued round-robin on 3 CUDA streams, one start event,
             one end event per stream, longest span, max over ranks.  No L2 flush in this
             pass: every view re-reads the packed scene (2.4 GB at 10M) and rewrites its
             own workspace, all far larger than the 126 MB L2.
  ms_per_frame / kernels / roofline
             a separate pass, one frame (view 0) at a time with a 256 MiB buffer written
             between frames (L2 flush, untimed), CUDA events recorded between the kernel
             launches on the launch stream (fgs_profile_begin).
  roofline   the longest kernel of the frame against the roof that bounds it: HBM
             (MEASURED_PEAKS.json) for preprocess / emit / tile sort on algorithmic bytes,
             FP32 (SMs x 128 lanes x 2 x clock) for the blend on the flops of the
             reference loop's evaluations, counted by outcome on the device
             (fgs_blend_counts, equal to the instrumented oracle loop: tests).
             `rooflines` lists the same for every kernel of the frame.
  e2e        the same metric through the public API with HOST frames out (float32
             (H,W,3), pinned D2H inside the timed region): `Pipeline.render_iter` over the
             views, and `e2e.render_call_*` for blocking `Pipeline.render(camera)` calls.
  cpu_baseline  the CPU oracle (C/OpenMP restatement of the reference, bit-identical to it
             on tests/golden) on the same view on this box's host cores.

`--impl reference` times that CPU path alone (rank 0 only).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (gaussians, width, height, density_scale, description)
    "c1": (10_000, 256, 256, False, "BASELINE configs[0]: 10K Gaussians, SH3, 256x256 single view"),
    "c2": (1_000_000, 1920, 1080, True,
           "BASELINE configs[1]: 1M Gaussians (mixed, seed 1, density-scaled), SH3, 1920x1080 single view"),
    "c2-dense": (1_000_000, 1920, 1080, False,
                 "1M Gaussians as generated (33.5M pairs, sort-heavy stress), SH3, 1920x1080"),
    "c3": (3_000_000, 3840, 2160, True,
           "BASELINE configs[2]: 3M Gaussians (density-scaled), SH3, 3840x2160 single view"),
    "c4": (10_000_000, 7680, 4320, True,
           "BASELINE configs[3]: 10M Gaussians (density-scaled), SH3, 7680x4320"),
    "c4-4k": (10_000_000, 3840, 2160, True,
              "north_star target: 10M Gaussians (density-scaled), SH3, 3840x2160"),
    "c5": (3_000_000, 1920, 1080, True,
           "BASELINE configs[4]: 64-view batch of a 3M-Gaussian scene (density-scaled), SH3, "
           "1920x1080, views sharded over the ranks"),
}
VIEWS = {"c5": 64}       # workloads that are a batch of 64 distinct views (orbit cameras)
DEFAULT_WORKLOAD = "c4-4k"
METRIC, UNIT = "views_per_sec", "views/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


def profiled_kernels(workload):
    """Per-kernel numbers of the newest committed ncu capture of `workload`."""
    import glob
    best = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if d.get("workload") == workload:
            best = dict(d.get("kernels", {}))
            best["_file"] = os.path.relpath(path, ROOT)
    return best


class ClockSampler:
    """Samples SM clock / throttle reasons through NVML while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40,
                 "sw_thermal_slowdown": 0x20, "hw_power_brake": 0x80, "sync_boost": 0x10,
                 "applications_clocks": 0x2}
        while not self._stop.is_set():
            try:
                self.samples.append(int(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()

    def stop(self):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()
        med = int(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_scene(fgs, name):
    n, w, h, dens, desc = WORKLOADS[name]
    act = fgs.activate(fgs.gen_synthetic("mixed", n, 1, density_scale=dens))
    return act, w, h, desc


def cpu_arm(act, cam, steps, warmup, budget_s=30.0):
    """The CPU path (oracle port of the reference) on this box's host cores."""
    from oracle import oracle as orc
    cores = orc.max_threads()
    for _ in range(max(1, min(warmup, 2))):
        orc.render(act, cam)
    times, stages = [], []
    t_begin = time.perf_counter()
    for _ in range(max(1, steps)):
        _, st = orc.render(act, cam)
        times.append(st["total_ns"] / 1e9)
        stages.append((st["preprocess_bin_ns"], st["sort_ns"], st["render_ns"]))
        if time.perf_counter() - t_begin > budget_s:
            break
    t = float(np.mean(times))
    sm = np.mean(np.asarray(stages, dtype=np.float64), axis=0) / 1e6
    return {"value": 1.0 / t, "unit": UNIT, "cores": cores, "kind": "port",
            "ms_per_frame": t * 1e3, "frames_timed": len(times),
            "stage_ms": {"preprocess_bin": sm[0], "sort": sm[1], "render": sm[2]},
            "sample": f"{len(times)} whole frame(s) of the same workload, OpenMP on {cores} threads "
                      "(oracle/fgs_oracle.c: C restatement of the reference, bit-identical to it on "
                      "tests/golden)"}


def tilesplat_arm(scene_mod, names=("c1", "c2"), budget_s=40.0):
    """The UNMODIFIED reference package (`tilesplat`, pure Python + numba) timed through its own
    public call, `Pipeline(scene).render(camera, workers=...)`, on BASELINE configs[0] and
    configs[1] -- when it is installed under baseline/_ref (git-ignored; `python
    __graft_entry__.py` installs it from /root/reference where that exists, and the directory
    travels to the GPU box with the snapshot).  Beside each time: the oracle port on the same
    input, and whether the two frames are bit-identical on this box."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "tilesplat")):
        return {"unavailable": "baseline/_ref/tilesplat is not installed on this box"}
    try:
        sys.path.insert(0, ref_dir)
        import tilesplat
    except Exception as e:                                   # numba missing, ...
        return {"unavailable": f"import tilesplat failed: {e!r}"[:200]}
    from oracle import oracle as orc
    import dataclasses
    cores = os.cpu_count() or 1
    out = {"package": f"tilesplat {getattr(tilesplat, '__version__', '?')} from baseline/_ref",
           "workers": cores, "os_cpu_count": os.cpu_count()}
    for name in names:
        act, w, h, desc = make_scene(scene_mod, name)
        cam = scene_mod.orbit_cameras(1, 24.0, w, h)[0]
        r_scene = tilesplat.ActivatedScene(**{f.name: getattr(act, f.name)
                                              for f in dataclasses.fields(tilesplat.ActivatedScene)})
        r_cam = tilesplat.Camera(**{f.name: getattr(cam, f.name)
                                    for f in dataclasses.fields(tilesplat.Camera)})
        pipe = tilesplat.Pipeline(r_scene)
        pipe.render(r_cam, workers=cores)                     # numba JIT + warm-up
        rec = {"workload": desc}
        for label, wk in (("ms_per_frame", cores), ("ms_per_frame_workers1", 1)):
            ts, best, t0 = [], None, time.perf_counter()
            while len(ts) < 5 and (not ts or time.perf_counter() - t0 < budget_s / 4):
                t = time.perf_counter()
                fb, st = pipe.render(r_cam, "precise", workers=wk)
                ts.append(time.perf_counter() - t)
                if best is None or st.total_ns < best.total_ns:
                    best = st
            rec[label] = 1e3 * float(np.median(ts))
            # best frame's FrameStats.total_ns and its three stage times
            rec[label.replace("ms_per_frame", "best_stats_ms")] = {
                "total": best.total_ns / 1e6, "preprocess_bin": best.preprocess_bin_ns / 1e6,
                "sort": best.sort_ns / 1e6, "render": best.render_ns / 1e6, "frames": len(ts)}
        oimg, ost = orc.render(act, cam)
        _, ost = orc.render(act, cam)
        rec["oracle_port_ms_per_frame"] = ost["total_ns"] / 1e6
        rec["port_frame_bit_identical_to_reference"] = bool(
            np.array_equal(np.asarray(fb.image).view(np.uint32), np.asarray(oimg).view(np.uint32)))
        rec["pairs_emitted"] = int(st.pairs_emitted)
        out[name] = rec
    return out


def run_reference(args, rank):
    if rank != 0:
        return
    import paper_2408_07967_b200.scene as scene_mod
    act, w, h, desc = make_scene(scene_mod, args.workload)
    cam = scene_mod.orbit_cameras(1, 24.0, w, h)[0]           # view 0 of the orbit
    cb = cpu_arm(act, cam, min(args.steps, 20), args.warmup, budget_s=120.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": cb["frames_timed"], "warmup": args.warmup,
        "ms_per_step": cb["ms_per_frame"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "strategy": "precise", "tau": 1.0 / 255.0, "sh_degree": 3},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["tilesplat"] = tilesplat_arm(scene_mod)
    except Exception as e:                                   # never lose the arm's own line
        line["tilesplat"] = {"unavailable": f"{e!r}"[:200]}
    print(json.dumps(line), flush=True)


NVIEWS_DEFAULT = 16      # distinct orbit views the timed steps cycle through


def launches_per_frame(bucket, npass, tiles, lazy=False):
    """Kernels of this library one frame launches (tile-bucket: preprocess, [slice totals on
    grids above 12 K tiles], tile scan, tile order, run scatter, fallback placement, four sort
    classes, blend; lazy_sort: + the full sort and the second blend pass of the redo list)."""
    if bucket:      # k_preprocess, k_scan_tiles, k_tile_order, k_scatter_runs, k_place, k_tile_sort_medium,
                    # k_tile_sort_large | k_tile_front, k_tile_sort, k_tile_sort_tail, k_blend2
                    # (+ k_tile_blocksums) (+ k_tile_sort_redo, k_blend2<redo>)
        return 10 + (1 if (tiles + 1023) // 1024 > 12 else 0) + (2 if lazy else 0)
    return 6 + npass


def measure(env, name, steps, warmup, args, with_cpu, short=False):
    """All measurements of one workload on this rank; rank 0 returns the JSON record."""
    torch, dist, fgs, _capi, sharding = env["torch"], env["dist"], env["fgs"], env["_capi"], env["sharding"]
    dev, rank, world, local_rank = env["dev"], env["rank"], env["world"], env["local_rank"]
    act, W, H, desc = make_scene(fgs, name)
    P = act.count
    nv_total = VIEWS.get(name, NVIEWS_DEFAULT)
    cams = fgs.orbit_cameras(nv_total, 24.0, W, H)
    bands_mode = args.mode == "bands"
    cam0 = cams[0]                          # the "single view" of BASELINE's configs
    my_ids = [0] if bands_mode else (sharding.views_for_rank(nv_total, world, rank) or [rank % nv_total])
    my_cams = [cams[v] for v in my_ids]
    gh, gw = -(-H // 16), -(-W // 16)

    pipe = fgs.Pipeline(act, sort_mode=args.sort_mode,
                        spatial_order=False if args.no_spatial else None,
                        lazy_sort=not args.no_lazy)
    L = _capi.lib()
    hbm_peak, peak_src, sm_max = peaks()
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count

    band, bands = None, sharding.band_partition(gh, world)
    if bands_mode and world > 1:
        if args.band_split == "balanced":
            rw = pipe.row_weights(cam0)
            bands = sharding.balanced_band_partition(rw, world, fixed_rows=0.3 * float(rw.mean()))
        band = bands[rank]

    # ---- warm-up through the public API (also sizes the workspace) -------------
    pairs_by_view = []
    for i in range(max(warmup, len(my_cams) if not short else 1)):
        fb, st = pipe.render(my_cams[i % len(my_cams)], exact=args.exact, band=band)
        pairs_by_view.append(st.pairs_emitted)
    fb, st = pipe.render(cam0, exact=args.exact, band=band)
    M, R = st.pairs_emitted, int(st.gaussians_retained)
    del fb
    stream = torch.cuda.current_stream(dev)
    bucket = args.sort_mode == "tile-bucket"
    lazy = int(pipe.lazy_sort)              # level the pipeline settled on during the warm-up frames
    if args.lazy_level is not None:
        lazy = pipe.lazy_sort = args.lazy_level
        pipe._lazy_cap = 0                  # (frozen: _note_fronts leaves the level alone)
    front_tiles, redo_tiles = int(st.front_tiles), int(st.redo_tiles)
    nlanes = max(1, args.streams)
    lanes = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nlanes - 1)]
    wss = []
    for _ in range(nlanes):
        w_ = pipe._take_ws(torch, W, H, pipe._default_capacity())
        w_.set_mode(_capi.SORT_MODES[args.sort_mode], lazy_sort=lazy)
        wss.append(w_)
    lay = wss[0].lay
    T_tiles = int(lay.tiles)
    npass = 0 if bucket else int(lay.sort_passes)
    n_marks = (10 if lazy else 8) if bucket else 6 + npass
    camcs = [_capi.camera_struct(c) for c in my_cams]
    cam0c = _capi.camera_struct(cam0)
    kcut = pipe._cutoffs(torch, 1.0 / 255.0)
    bg = (C.c_float * 3)(0.0, 0.0, 0.0)
    flags = (_capi.BLEND_EXACT if args.exact else 0) | _capi.BLEND_CONTRIB
    b0, b1 = band if band is not None else (0, gh - 1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)      # > 126 MB L2

    def frame(lane=0, camc=cam0c):
        w_ = wss[lane]
        _capi.check(L.fgs_render(pipe.packed.data_ptr(), kcut.data_ptr(), P, C.byref(camc),
                                 1.0 / 255.0, 3, 0, bg, flags, b0, b1, w_.next_epoch(),
                                 w_.rgb.data_ptr(), None, None, C.c_void_p(w_.base),
                                 C.byref(w_.lay), C.c_void_p(lanes[lane].cuda_stream)))

    for i in range(max(warmup, 2 * nlanes)):
        frame(i % nlanes, camcs[i % len(camcs)])
    torch.cuda.synchronize(dev)

    # ---- pass A: view 0, one frame at a time, per-kernel CUDA events -------------
    KA = min(steps, 12 if short else 30)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(KA)]
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(n_marks)] for _ in range(KA)]
    for e in ev0:
        e.record(stream)               # materialise the handles
    for row in marks:
        for e in row:
            e.record(stream)
    handles = [(C.c_void_p * n_marks)(*[e.cuda_event for e in row]) for row in marks]
    torch.cuda.synchronize(dev)
    for i in range(KA):
        flush.fill_(i & 0xff)          # evict L2 between frames (not timed)
        ev0[i].record(stream)
        L.fgs_profile_begin(handles[i], n_marks)
        frame(0)
        got = L.fgs_profile_end()
        assert got == n_marks, (got, n_marks)
    torch.cuda.synchronize(dev)
    lat_prof_ms = np.array([ev0[i].elapsed_time(marks[i][-1]) for i in range(KA)])
    # the same, without the per-kernel events: kernels then chain by programmatic dependent
    # launch and the sort size classes overlap, so this -- not the sum of the kernels -- is
    # the latency of a frame
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(KA)]
    eve = [torch.cuda.Event(enable_timing=True) for _ in range(KA)]
    for i in range(KA):
        flush.fill_(i & 0xff)
        evs[i].record(stream)
        frame(0)
        eve[i].record(stream)
    torch.cuda.synchronize(dev)
    lat_ms = np.array([evs[i].elapsed_time(eve[i]) for i in range(KA)])
    kern = np.zeros((KA, n_marks))
    for i in range(KA):
        prev = ev0[i]
        for j in range(n_marks):
            kern[i, j] = prev.elapsed_time(marks[i][j])
            prev = marks[i][j]

    # ---- pass B: the timed steps.  K frames over this rank's DISTINCT views, round-robin
    # over `nlanes` streams (each with its own workspace) so consecutive views overlap on the
    # GPU, exactly like the public batch API.  Bands: every step is the rank's band of the
    # one frame followed by the gather on rank 0 (NCCL send/recv), all inside the timed region.
    K = steps
    t_begin = torch.cuda.Event(enable_timing=True)
    t_ends = [torch.cuda.Event(enable_timing=True) for _ in range(nlanes)]
    gather_ms = None
    full_frame = None
    if bands_mode and world > 1:
        full_frame = torch.empty((H, W, 3), dtype=torch.float32, device=dev) if rank == 0 else None
        for _ in range(2):
            pipe.render_bands(cam0, dist, bands=bands, out=full_frame, exact=args.exact, as_numpy=False)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.cuda.synchronize(dev)
    t_wall0 = time.perf_counter()
    t_begin.record(stream)
    if bands_mode and world > 1:
        for i in range(K):
            pipe.render_bands(cam0, dist, bands=bands, out=full_frame, exact=args.exact,
                              as_numpy=False, sync=False)
        t_ends[0].record(stream)
        t_ends = t_ends[:1]
    else:
        for ln in lanes[1:]:
            ln.wait_event(t_begin)
        for i in range(K):
            frame(i % nlanes, camcs[i % len(camcs)])
        for ln, e in zip(lanes, t_ends):
            e.record(ln)
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = max(t_begin.elapsed_time(e) for e in t_ends)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    views_per_step = 1 if bands_mode else world
    value = views_per_step * K / (total_ms / 1e3)

    # ---- end to end through the public API (host frame out every step) -----------
    if band is None:
        for fb, _ in pipe.render_iter([my_cams[i % len(my_cams)] for i in range(8)],
                                      exact=args.exact, streams=nlanes):   # warm the pinned pool
            pass
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # views/s of a pipelined batch: measured over at least 60 views so that the fill of the
    # pipeline (the first frame's kernels before the first read-back can start, ~2 frame times)
    # is amortised as it is in the device-timed value's streams; `e2e.steps` says how many
    Ke = max(K, 60) if not short else min(K, 32)
    t0 = time.perf_counter()
    if band is None:
        # the batch call a views/s user makes: the views through Pipeline.render_iter
        # (frame i's read-back overlaps frame i+1's kernels)
        nfr = 0
        for fb, st_e in pipe.render_iter([my_cams[i % len(my_cams)] for i in range(Ke)],
                                         exact=args.exact, streams=nlanes):
            assert fb.image.shape == (H, W, 3) and isinstance(fb.image, np.ndarray)   # host frame
            nfr += 1
        assert nfr == Ke
    else:
        for _ in range(Ke):
            fbb, _ = pipe.render_bands(cam0, dist, bands=bands, exact=args.exact)   # host frame on rank 0
            assert rank != 0 or fbb.image.shape == (H, W, 3)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = views_per_step * Ke / e2e_s
    # the reference's own entry point, one blocking call per view: Pipeline.render(camera)
    nsingle = min(K, 10 if short else 20)
    render_call = {}
    if band is None:
        for key, kw in (("float32", {}), ("quantized", {"quantized": True})):
            pipe.render(my_cams[0], exact=args.exact, timing=False, **kw)
            t1 = time.perf_counter()
            for i in range(nsingle):
                pipe.render(my_cams[i % len(my_cams)], exact=args.exact, timing=False, **kw)
            render_call[key] = (time.perf_counter() - t1) / nsingle * 1e3

    if rank != 0:
        return None

    # ---- per-kernel records and rooflines ------------------------------------------
    if bucket:
        # launch order of the size classes: persistent kernels first (fgs_launch_tile_sort)
        names = ["preprocess", "scan", "emit", "tile_sort_medium",
                 "tile_front" if lazy else "tile_sort_large",
                 "tile_sort", "tile_sort_tail", "blend"] + (["redo_sort", "redo_blend"] if lazy else [])
    else:
        names = ["preprocess", "scan", "emit", "sort_hist"] \
            + [f"sort_pass{p}" for p in range(npass)] + ["ranges", "blend"]
    kmean = kern.mean(axis=0)
    ncu_name = {"preprocess": "k_preprocess", "scan": "k_scan_tiles", "emit": "k_scatter_runs",
                "tile_sort": "k_tile_sort", "tile_sort_medium": "k_tile_sort_medium",
                "tile_sort_large": "k_tile_sort_large", "tile_sort_tail": "k_tile_sort_tail",
                "tile_front": "k_tile_front", "redo_sort": "k_tile_sort_redo",
                "blend": "k_blend" if args.exact else "k_blend2"}
    prof_all = profiled_kernels(name)
    kernels = []
    for nme, ms in zip(names, kmean):
        ent = {"name": nme, "ms": float(ms), "share": float(ms / kmean.sum())}
        for k, v in prof_all.items():
            if isinstance(v, dict) and k.split("<")[0] == ncu_name.get(nme):
                ent["ncu_dram_bytes"] = v["dram_bytes"]
                ent["ncu_issue_slots_busy_pct"] = v.get("issue_slots_busy_pct")
        kernels.append(ent)

    # evaluation counts of the compositing loop for this view (device pass, untimed; equal
    # to the instrumented oracle loop -- tests/test_gpu_parity.py)
    evals = fgs.blend_eval_counts(pipe, cam0) if band is None else None
    M_proc = evals["pairs_processed"] if evals else M
    # algorithmic bytes per launch
    alg = {
        # scene in, splat row + depth out; tile-bucket: + the 8 B record of every pair, staged
        # by run
        "preprocess": 236.0 * P + 52.0 * R + (8.0 * M if bucket else 0.0),
        # bucket: the staged records in, the bucketed records out (a copy); onesweep: 12 B pair out
        "emit": 16.0 * M if bucket else 12.0 * M + 4.0 * P,
        "tile_sort_all": 12.0 * M,          # 8 B record in, 4 B index out, all four classes
        "sort_pass": 24.0 * M,
        "blend": 52.0 * M_proc + 12.0 * W * H,
    }
    ib = names.index("blend")
    # lazy_sort: the redo list's full sort counts with the sort, its second blend pass with the blend
    ms_of = {"preprocess": float(kmean[0]), "emit": float(kmean[2]),
             "blend": float(kmean[ib] + (kmean[ib + 2] if lazy and bucket else 0.0))}
    if bucket:
        ms_of["tile_sort_all"] = float(kmean[3:ib].sum() + (kmean[ib + 1] if lazy else 0.0))
    else:
        ms_of["sort_pass"] = float(sum(k["ms"] for k in kernels if k["name"].startswith("sort_pass"))) / max(npass, 1)
    clock_mhz = float(props.clock_rate) / 1e3 if getattr(props, "clock_rate", 0) else sm_max
    fp32_peak = sms * 128 * 2 * sm_max * 1e6 / 1e12            # TFLOP/s at the max SM clock
    kname = {"preprocess": "k_preprocess", "emit": "k_scatter_runs" if bucket else "k_emit",
             "tile_sort_all": "k_tile_sort{,_medium,_tail} + k_tile_front + k_tile_sort_redo" if lazy
                              else "k_tile_sort{,_medium,_large,_tail}", "sort_pass": "k_sort_pass",
             "blend": ncu_name["blend"]}

    def roof_of(key):
        ms = ms_of[key]
        hit = [v for k, v in prof_all.items()
               if isinstance(v, dict) and k.split("<")[0] == kname[key]]
        if key == "blend" and evals is not None:
            ach = evals["flops"] / (ms * 1e-3) / 1e12
            r = {"kernel": kname[key], "bound": "fp32", "achieved": ach, "peak": fp32_peak,
                 "unit": "TFLOP/s", "frac": ach / fp32_peak, "traffic": None,
                 "launches_per_step": 1, "ms_per_launch": ms,
                 "flops_per_launch": evals["flops"],
                 "evaluations": {k: evals[k] for k in fgs.EVAL_FLOPS},
                 "flops_per_evaluation": dict(fgs.EVAL_FLOPS),
                 "pairs_processed": M_proc, "alg_bytes_per_launch": alg["blend"],
                 "hbm_view_gbs": alg["blend"] / (ms * 1e-3) / 1e9,
                 "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (max SM clock)",
                 "note": "flops = the reference loop's own operations per (pixel, pair) evaluation "
                         "(render.py:106-129: 6 / 16 / 21 / 31 by outcome), counted on the device; the "
                         "kernel culls pairs per 8x8 block and evaluates two pixels per packed "
                         "instruction, so it executes fewer instructions than that count implies"}
            if hit:
                inst = hit[0]["warp_instructions"]
                peak_issue = 4.0 * sms * (clocks.get("sm_mhz") or sm_max) * 1e6
                r["issue"] = {"warp_instructions_per_launch": inst,
                              "achieved_ginst_s": inst / (ms * 1e-3) / 1e9,
                              "peak_ginst_s": peak_issue / 1e9, "frac": inst / (ms * 1e-3) / peak_issue,
                              "ncu_issue_slots_busy_pct": hit[0].get("issue_slots_busy_pct"),
                              "ncu_fma_pipe_busy_pct": hit[0].get("fma_pipe_busy_pct"),
                              "ncu_alu_pipe_busy_pct": hit[0].get("alu_pipe_busy_pct"),
                              "ncu_xu_pipe_busy_pct": hit[0].get("xu_pipe_busy_pct")}
        else:
            ach = alg[key] / (ms * 1e-3) / 1e9
            r = {"kernel": kname[key], "bound": "hbm", "achieved": ach, "peak": hbm_peak,
                 "unit": "GB/s", "frac": ach / hbm_peak, "traffic": None,
                 "launches_per_step": {"tile_sort_all": 5 if lazy else 4, "sort_pass": npass}.get(key, 1),
                 "ms_per_launch": ms, "alg_bytes_per_launch": alg[key], "peak_source": peak_src}
        if hit:
            r["traffic"] = hit[0]["dram_bytes"]
            r["traffic_source"] = prof_all.get("_file")
        return r

    rooflines = {k: roof_of(k) for k in ms_of}
    dom = max(ms_of, key=lambda k: ms_of[k] * ({"sort_pass": npass}.get(k, 1)))
    roof = rooflines[dom]
    for ent in kernels:
        key = ent["name"]
        if key in rooflines and key != "blend":
            ent["alg_bytes"], ent["gbs"], ent["frac_hbm"] = alg[key], rooflines[key]["achieved"], rooflines[key]["frac"]
        elif key == "blend":
            ent["alg_bytes"], ent["frac_fp32"] = alg["blend"], rooflines["blend"]["frac"] if evals else None
    if bucket:
        kernels.append({"name": "tile_sort_all", "ms": ms_of["tile_sort_all"],
                        "share": float(ms_of["tile_sort_all"] / kmean.sum()),
                        "alg_bytes": alg["tile_sort_all"], "gbs": rooflines["tile_sort_all"]["achieved"],
                        "frac_hbm": rooflines["tile_sort_all"]["frac"],
                        "note": "sum of the four size-class launches"})

    cpu = cpu_arm(act, cam0, 3, 1, budget_s=25.0) if with_cpu else None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": warmup, "ms_per_step": ms_per_step, "ms_per_frame": float(lat_ms.mean()),
        "higher_is_better": True,
        "scaling": "weak" if not bands_mode else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "mode": args.mode,
                   "band_split": (args.band_split if bands_mode else None), "strategy": "precise",
                   "tau": 1.0 / 255.0, "sh_degree": 3, "gaussians": P, "width": W, "height": H,
                   "pairs": M, "pairs_processed": M_proc, "retained": R, "tiles": T_tiles,
                   "sort_mode": args.sort_mode, "sort_passes": npass,
                   "lazy_sort": lazy, "front_tiles": front_tiles, "redo_tiles": redo_tiles,
                   "blend": "exact" if args.exact else "ex2.approx+guard",
                   "streams": nlanes,
                   "distinct_views": 1 if bands_mode else len(my_cams) * world,
                   "views": "orbit_cameras(%d, 24.0, %d, %d); rank r times views r, r+N, ...; "
                            "kernels / roofline / cpu_baseline are view 0" % (nv_total, W, H),
                   "pairs_by_view": {"min": int(min(pairs_by_view)), "max": int(max(pairs_by_view))},
                   "l2": "timed steps: inputs larger than L2 -- every view re-reads the %d MB "
                         "packed scene and rewrites its own workspace, %d views in flight, 126 MB "
                         "L2, no flush; latency / per-kernel pass: 256 MiB buffer written between "
                         "frames (flush, untimed)" % (pipe.scene_bytes >> 20, nlanes),
                   "timing": "CUDA events on the launch streams: one start event, one end event "
                             "per stream, longest span; max over ranks"},
        "clocks": clocks,
        "frame_latency_ms": float(lat_ms.mean()),
        "frame_latency_profiled_ms": float(lat_prof_ms.mean()),
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_s / Ke * 1e3, "steps": Ke,
                "h2d_bytes_per_step": C.sizeof(_capi.FgsCamera) + 12,
                "d2h_bytes_per_step": W * H * 12 + 64,
                "d2h_floor_ms": (W * H * 12) / 55e9 * 1e3,
                "api": ("Pipeline.render_iter(cameras) -> per view a host numpy float32 frame "
                        "(pinned D2H behind the view's kernels on its stream; views round-robin "
                        "on %d streams) + FrameStats" % nlanes) if band is None else
                       "Pipeline.render_bands(camera, dist) -> host frame on rank 0",
                "render_call_ms": render_call.get("float32"),
                "render_call_quantized_ms": render_call.get("quantized"),
                "render_call_api": "blocking Pipeline.render(camera) per view (the reference's entry "
                                   "point): float32 host frame / uint8 host frame"},
        "gpu_launches": int(launches_per_frame(bucket, npass, T_tiles, lazy) * K),
        "roofline": roof,
        "rooflines": rooflines,
        "cpu_baseline": cpu,
        "kernels": kernels,
        "kernels_note": "per-kernel times are from the one-frame-at-a-time pass (%d frames of view "
                        "0, L2 flushed between frames); `value` overlaps consecutive views" % KA,
        "stage_ms": {"preprocess_bin": float(kmean[0:3].sum()),
                     "sort": float(kmean[3:-1].sum()), "render": float(kmean[-1])},
        "wall_s_timed_region": t_wall,
    }
    del wss, pipe, flush
    torch.cuda.empty_cache()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="views", choices=["views", "bands"])
    ap.add_argument("--band-split", default="balanced", choices=["balanced", "equal"],
                    help="--mode bands: bands of equal estimated work (default) or equal height")
    ap.add_argument("--exact", action="store_true", help="bit-exact blend mode")
    ap.add_argument("--sort-mode", default="tile-bucket", choices=["tile-bucket", "onesweep"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-also", action="store_true", help="skip the extra configs[1] run")
    ap.add_argument("--no-lazy", action="store_true",
                    help="sort every tile in full (fgs_layout.lazy_sort = 0)")
    ap.add_argument("--lazy-level", type=int, default=None, choices=[0, 1, 2],
                    help="force the lazy_sort level instead of letting the pipeline choose (A/B runs)")
    ap.add_argument("--no-spatial", action="store_true",
                    help="keep the scene in the caller's order (no Morton slot order)")
    ap.add_argument("--streams", type=int, default=3,
                    help="CUDA streams the timed views are issued on round-robin (1 = back to back)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2408_07967_b200 as fgs
    from paper_2408_07967_b200 import _capi, sharding

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product has no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    env = dict(torch=torch, dist=dist, fgs=fgs, _capi=_capi, sharding=sharding, dev=dev,
               rank=rank, world=world, local_rank=local_rank)

    line = measure(env, args.workload, args.steps, args.warmup, args,
                   with_cpu=not args.no_cpu and world == 1)
    if args.workload == DEFAULT_WORKLOAD and args.mode == "views" and not args.no_also:
        # BASELINE configs[1] beside the headline, short: value, latency, e2e, kernels
        c2 = measure(env, "c2", min(args.steps, 64), 3, args, with_cpu=False, short=True)
        if rank == 0:
            keep = ("value", "unit", "ms_per_step", "ms_per_frame", "e2e", "kernels", "roofline",
                    "rooflines", "stage_ms", "steps")
            line["also"] = {"c2": dict({k: c2[k] for k in keep},
                                       workload=c2["config"]["workload"], pairs=c2["config"]["pairs"],
                                       pairs_processed=c2["config"]["pairs_processed"],
                                       distinct_views=c2["config"]["distinct_views"])}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
