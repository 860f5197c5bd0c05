"""Report emitters driven by the GPU path.

Same call signatures and the same versioned JSON shapes as the reference's
``compare_modes`` (``pipeline.py:171-209``) and ``bench_frames``
(``pipeline.py:212-269``; field definitions in ``docs/report-schema.md:11-74``),
so a report written by this package diffs cleanly against one written by the
reference: every non-timing field is identical for the same scene, cameras and
flags.  Stage times are CUDA-event times of the kernels of each stage.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .pipeline import STRATEGIES, TAU_DEFAULT, Pipeline, max_abs_diff, psnr

REPORT_SCHEMA_VERSION = 1          # docs/report-schema.md:3


def _frame_id(cam, index):
    return getattr(cam, "cam_id", index)


@dataclass
class CompareReport:
    """Per-frame stats of every strategy plus the pairwise image metrics
    (``pipeline.py:140-168``)."""

    strategies: list
    frames: list = field(default_factory=list)

    def aggregate(self) -> dict:
        agg = {}
        for name in self.strategies:
            per_frame = [fr["stats"][name] for fr in self.frames]
            agg[name] = {
                "frames": len(per_frame),
                "pairs_emitted_total": sum(p["pairs_emitted"] for p in per_frame),
                "pairs_contributing_total": sum(p["pairs_contributing"] for p in per_frame),
                "pair_buffer_bytes_total": sum(p["pair_buffer_bytes"] for p in per_frame),
            }
        return agg

    def to_dict(self) -> dict:
        return {"schema_version": REPORT_SCHEMA_VERSION, "kind": "compare",
                "strategies": list(self.strategies), "frames": self.frames,
                "aggregate": self.aggregate()}


def _reference_stats_dict(st) -> dict:
    """FrameStats -> exactly the reference's frame-stats object (report-schema.md:11-28)."""
    d = st.to_dict()
    for extra in ("candidate_tiles", "e2e_ns", "front_tiles", "redo_tiles"):
        d.pop(extra, None)
    return d


def compare_modes(scene, cameras, strategies=STRATEGIES, tau=TAU_DEFAULT,
                  background=(0.0, 0.0, 0.0), workers=1, sh_degree=3, *,
                  exact=False) -> CompareReport:
    """Every camera under every strategy; full symmetric PSNR / max-abs-diff
    matrices per frame and the emitted-pair ratio against the first strategy."""
    names = list(strategies)
    if len(names) < 2:
        raise ValueError("compare_modes needs at least two strategies")
    pipe = scene if isinstance(scene, Pipeline) else Pipeline(scene, sh_degree=sh_degree)
    report = CompareReport(strategies=names)
    for index, cam in enumerate(cameras):
        images, stats = {}, {}
        for name in names:
            fb, st = pipe.render(cam, name, tau, background, workers, exact=exact)
            images[name] = fb
            stats[name] = _reference_stats_dict(st)
        quality, diff = {}, {}
        for i, a in enumerate(names):
            for b in names[i:]:
                same = a == b
                q = "identical" if same else psnr(images[a], images[b])
                d = 0.0 if same else max_abs_diff(images[a], images[b])
                quality[f"{a}|{b}"] = quality[f"{b}|{a}"] = q
                diff[f"{a}|{b}"] = diff[f"{b}|{a}"] = d
        first = stats[names[0]]["pairs_emitted"]
        report.frames.append({
            "frame_id": _frame_id(cam, index),
            "stats": stats,
            "psnr": quality,
            "max_abs_diff": diff,
            "pairs_emitted_ratio_vs_first": {
                n: (stats[n]["pairs_emitted"] / first if first else 0.0) for n in names},
        })
    return report


def bench_frames(scene, cameras, strategy="precise", repeat=3, tau=TAU_DEFAULT,
                 background=(0.0, 0.0, 0.0), workers=1, sh_degree=3, *, exact=False) -> dict:
    """Timing report: one untimed warm-up round, then ``repeat`` rounds over the
    camera set; aborts when the deterministic counters differ between repeats."""
    if repeat < 1:
        raise ValueError("repeat must be >= 1")
    cameras = list(cameras)
    pipe = scene if isinstance(scene, Pipeline) else Pipeline(scene, sh_degree=sh_degree)
    for cam in cameras:                       # sizes the workspace, warms the pinned pool
        pipe.render(cam, strategy, tau, background, workers, exact=exact)
    all_stats, round_totals, seen = [], [], {}
    for _ in range(repeat):
        acc = 0
        for index, cam in enumerate(cameras):
            _, st = pipe.render(cam, strategy, tau, background, workers, exact=exact)
            all_stats.append(st)
            acc += st.total_ns
            sig = (st.pairs_emitted, st.pairs_contributing, st.gaussians_retained,
                   st.tiles_nonempty)
            if seen.setdefault(_frame_id(cam, index), sig) != sig:
                raise AssertionError("non-deterministic counters across repeats")
        round_totals.append(acc)
    n = len(cameras)
    totals = np.asarray([s.total_ns for s in all_stats], dtype=np.float64)
    rounds = np.asarray(round_totals, dtype=np.float64)
    stage_ns = {
        "preprocess_bin": np.asarray([s.preprocess_bin_ns for s in all_stats], dtype=np.float64),
        "sort": np.asarray([s.sort_ns for s in all_stats], dtype=np.float64),
        "render": np.asarray([s.render_ns for s in all_stats], dtype=np.float64),
    }
    in_stages = float(sum(v.sum() for v in stage_ns.values()))
    frame_ms = {}
    for index, cam in enumerate(cameras):
        mine = totals[index::n] / 1e6
        frame_ms[_frame_id(cam, index)] = {"avg_ms": float(mine.mean()), "max_ms": float(mine.max()),
                                           "min_ms": float(mine.min())}
    return {
        "schema_version": REPORT_SCHEMA_VERSION,
        "kind": "bench",
        "strategy": strategy,
        "tau": float(tau),
        "workers": int(workers),
        "repeat": int(repeat),
        "frames_per_repeat": n,
        "avg_ms": float(rounds.mean() / 1e6),
        "max_ms": float(rounds.max() / 1e6),
        "min_ms": float(rounds.min() / 1e6),
        "frame_ms": frame_ms,
        "stage_ms": {k: float(v.mean() / 1e6) for k, v in stage_ns.items()},
        "stage_percent": {k: float(100.0 * v.sum() / in_stages) if in_stages else 0.0
                          for k, v in stage_ns.items()},
        "stage_coverage_percent": float(100.0 * in_stages / totals.sum()) if totals.sum() else 0.0,
        "pairs_emitted": [int(s.pairs_emitted) for s in all_stats[:n]],
        "pairs_contributing": [int(s.pairs_contributing) for s in all_stats[:n]],
    }
