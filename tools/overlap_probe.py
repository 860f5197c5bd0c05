#!/usr/bin/env python
"""Probe: throughput of C2 frames issued round-robin on S streams (each with its own workspace)."""
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
for S in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(S)]
    wss = [fgs.pipeline._Workspace(torch, dev, n, W, H, pipe._default_capacity()) for _ in range(S)]
    for ws in wss:
        ws.set_mode(1)

    def frame(i):
        ws, st = wss[i % S], streams[i % S]
        _capi.check(L.fgs_render(pipe.packed.data_ptr(), kcut.data_ptr(), n, C.byref(camc), 1 / 255, 3, 0,
                                 bg, 2, 0, gh - 1, ws.next_epoch(), ws.rgb.data_ptr(), None, None,
                                 C.c_void_p(ws.base), C.byref(ws.lay), C.c_void_p(st.cuda_stream)))
    for i in range(8):
        frame(i)
    torch.cuda.synchronize()
    K = 200
    t0 = time.perf_counter()
    for i in range(K):
        frame(i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams={S}: {dt / K * 1e6:.1f} us/frame  {K / dt:.0f} views/s", flush=True)
