"""Probe: internal work counters of one frame (regular / fallback preprocess CTAs, staged records)."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2408_07967_b200 as fgs
from paper_2408_07967_b200 import _capi

wl = sys.argv[1] if len(sys.argv) > 1 else "c4-4k"
act, W, H, desc = bench.make_scene(fgs, wl)
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
fb, st = pipe.render(cam)
ws = pipe._take_ws(torch, W, H, pipe._default_capacity())
L = _capi.lib()
camc = _capi.camera_struct(cam)
kcut = pipe._cutoffs(torch, 1 / 255)
bg = (C.c_float * 3)(0, 0, 0)
gh = -(-H // 16)
_capi.check(L.fgs_render(pipe.packed.data_ptr(), kcut.data_ptr(), pipe.count, C.byref(camc), 1 / 255, 3, 0, bg, 2,
                         0, gh - 1, ws.next_epoch(), ws.rgb.data_ptr(), None, None, C.c_void_p(ws.base),
                         C.byref(ws.lay), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
raw = ws.buf[int(ws.lay.off_stats):int(ws.lay.off_stats) + 256].cpu().numpy().view(np.uint32)
print(desc)
print("stats", raw[:16])
print("work", raw[16:32])
blocks = int(ws.lay.preprocess_blocks)
print(f"preprocess CTAs {blocks}, fallback {raw[16 + 9]} ({100.0 * raw[16 + 9] / blocks:.2f}%), staged records {raw[16 + 8]} of {raw[0]} pairs, list entries {raw[15]}")
info = ws.buf[int(ws.lay.off_ctainfo):int(ws.lay.off_ctainfo) + blocks * 16].cpu().numpy().view(np.uint32).reshape(blocks, 4)
reg = info[:, 3] != 0xffffffff
print("regular CTAs", int(reg.sum()), "entries/CTA mean", info[:, 1].mean(), "max", info[:, 1].max(), "records/CTA mean", info[reg, 2].mean() if reg.any() else 0, "max", info[:, 2].max())
