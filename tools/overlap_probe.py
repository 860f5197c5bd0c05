#!/usr/bin/env python
"""Probe: throughput of C2 frames issued round-robin on S lanes (each with its own workspace).

mode "one":   the whole frame is one fgs_render call on the lane's stream
mode "split": the binning chain (preprocess..ranges) runs on a HIGH-priority stream, the blend
              on a LOW-priority stream behind an event, so the next view's binning CTAs are
              dispatched ahead of the pending blend CTAs of the previous view
"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2408_07967_b200 as fgs
from paper_2408_07967_b200 import _capi

n, W, H = 1_000_000, 1920, 1080
act = fgs.activate(fgs.gen_synthetic("mixed", n, 1, density_scale=True))
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
for _ in range(3):
    pipe.render(cam)
L = _capi.lib()
dev = torch.device("cuda", 0)
kcut = pipe._cutoffs(torch, 1 / 255)
camc = _capi.camera_struct(cam)
bg = (C.c_float * 3)(0, 0, 0)
gh = -(-H // 16)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
for mode in ("one", "split"):
    for S in (1, 2, 3):
        hs = [torch.cuda.Stream(priority=-1) for _ in range(S)]
        ls = [torch.cuda.Stream(priority=0) for _ in range(S)]
        binned = [torch.cuda.Event() for _ in range(S)]
        blended = [torch.cuda.Event() for _ in range(S)]
        wss = [fgs.pipeline._Workspace(torch, dev, n, W, H, pipe._default_capacity()) for _ in range(S)]
        for ws in wss:
            ws.set_mode(1)

        def frame(i):
            k = i % S
            ws = wss[k]
            if mode == "one":
                _capi.check(L.fgs_render(pipe.packed.data_ptr(), kcut.data_ptr(), n, C.byref(camc), 1 / 255, 3, 0,
                                         bg, 2, 0, gh - 1, ws.next_epoch(), ws.rgb.data_ptr(), None, None,
                                         C.c_void_p(ws.base), C.byref(ws.lay), C.c_void_p(ls[k].cuda_stream)))
                return
            h, l = hs[k], ls[k]
            hp, lp = C.c_void_p(h.cuda_stream), C.c_void_p(l.cuda_stream)
            wsp, lay = C.c_void_p(ws.base), C.byref(ws.lay)
            h.wait_event(blended[k])
            _capi.check(L.fgs_preprocess(pipe.packed.data_ptr(), kcut.data_ptr(), n, C.byref(camc), 1 / 255, 3, 0,
                                         0, gh - 1, wsp, lay, hp))
            _capi.check(L.fgs_scan(wsp, lay, hp))
            _capi.check(L.fgs_emit(pipe.packed.data_ptr(), C.byref(camc), 0, 0, gh - 1, wsp, lay, hp))
            _capi.check(L.fgs_sort(wsp, lay, ws.next_epoch(), hp))
            _capi.check(L.fgs_ranges(wsp, lay, hp))
            binned[k].record(h)
            l.wait_event(binned[k])
            _capi.check(L.fgs_blend(pipe.packed.data_ptr(), bg, 1 / 255, 2, 0, gh - 1, ws.rgb.data_ptr(), None,
                                    None, wsp, lay, lp))
            blended[k].record(l)

        for i in range(8):
            frame(i)
        torch.cuda.synchronize()
        K = 200
        t0 = time.perf_counter()
        for i in range(K):
            frame(i)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"mode={mode} lanes={S}: {dt / K * 1e6:.1f} us/frame  {K / dt:.0f} views/s  "
              f"(host issue {(t1 - t0) / K * 1e6:.1f} us/frame)", flush=True)
