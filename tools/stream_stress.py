import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2408_07967_b200 as fgs
n = int(sys.argv[1]); W, H = int(sys.argv[2]), int(sys.argv[3]); streams = int(sys.argv[4])
act = fgs.activate(fgs.gen_synthetic("mixed", n, 1, density_scale=True))
cam = fgs.orbit_cameras(1, 24.0, W, H)[0]
pipe = fgs.Pipeline(act)
fb, st = pipe.render(cam); print("single", st.pairs_emitted, st.buffer_regrows, flush=True)
fb, st = pipe.render(cam); print("single", st.pairs_emitted, st.buffer_regrows, flush=True)
for rep in range(3):
    out = pipe.render_many([cam] * 6, streams=streams, depth=2 * streams)
    torch.cuda.synchronize()
    print("many", rep, [s.pairs_emitted for _, s in out][:3], float(out[-1][0].image.sum()), flush=True)
