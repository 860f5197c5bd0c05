"""Test helpers shared by the CPU and GPU suites (imported as a top-level
module; `tests` itself is not a package name we can rely on)."""

import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDEN_CASES = ("c1_mixed10k_256", "mixed800_256x192", "elongated800_256x192",
                "edge3000_70x42")


class GoldenCase:
    """One .npz written by tests/golden/make_golden.py (reference outputs)."""

    def __init__(self, name):
        self.name = name
        self.z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        from paper_2408_07967_b200.scene import ActivatedScene
        self.act = ActivatedScene(self.z["means"], self.z["opacities"], self.z["scales"],
                                  self.z["rotations"], self.z["sh"])
        self.tau = float(self.z["tau"])
        self.bg = tuple(float(v) for v in self.z["bg"])
        self.sh_degree = int(self.z["sh_degree"])
        self.ncam = int(self.z["ncam"])

    def camera(self, i):
        from paper_2408_07967_b200.scene import Camera
        z, p = self.z, f"c{i}_"
        w, h = (int(v) for v in z[p + "wh"])
        tx, ty, fx, fy = (float(v) for v in z[p + "intr"])
        return Camera(w, h, z[p + "position"], z[p + "view"], z[p + "proj"],
                      tx, ty, fx, fy, cam_id=str(i))

    def get(self, cam_i, field, strategy="precise"):
        q = f"c{cam_i}_" + ("" if strategy == "precise" else strategy + "_")
        return self.z[q + field]

    def has(self, cam_i, field, strategy="precise"):
        q = f"c{cam_i}_" + ("" if strategy == "precise" else strategy + "_")
        return (q + field) in self.z.files

    def retained(self, cam_i, strategy="precise"):
        n = self.act.count
        return np.unpackbits(self.get(cam_i, "retained", strategy))[:n].astype(bool)

    def contrib(self, cam_i, strategy="precise"):
        m = self.get(cam_i, "keys", strategy).shape[0]
        return np.unpackbits(self.get(cam_i, "contrib", strategy))[:m]



def make_raw_scene(means, scales, opacities, quats=None, dc=None, rest=None):
    """Raw Scene from activated target values (same contract as the reference's
    tests/conftest.py:9-35 helper: inverts the activations)."""
    from paper_2408_07967_b200.scene import Scene
    means = np.atleast_2d(np.asarray(means, dtype=np.float64))
    n = means.shape[0]
    scales = np.broadcast_to(np.asarray(scales, dtype=np.float64), (n, 3))
    opacities = np.broadcast_to(np.asarray(opacities, dtype=np.float64), (n,))
    if quats is None:
        quats = np.tile(np.array([1.0, 0, 0, 0]), (n, 1))
    quats = np.broadcast_to(np.asarray(quats, dtype=np.float64), (n, 4))
    sh = np.zeros((n, 16, 3), dtype=np.float32)
    if dc is None:
        dc = np.tile(np.array([0.8, 0.8, 0.8]), (n, 1))
    sh[:, 0, :] = np.broadcast_to(np.asarray(dc, dtype=np.float64), (n, 3))
    if rest is not None:
        sh[:, 1:, :] = rest
    return Scene(means=means.astype(np.float32),
                 normals=np.zeros((n, 3), dtype=np.float32), sh=sh,
                 logit_opacities=np.log(opacities / (1.0 - opacities)).astype(np.float32),
                 log_scales=np.log(scales).astype(np.float32),
                 rotations=quats.astype(np.float32))


def identity_camera(width=64, height=64, focal=None, position=(0.0, 0.0, 0.0)):
    from paper_2408_07967_b200.scene import make_camera
    focal = focal if focal is not None else width / 2
    return make_camera(width, height, position, np.eye(3), focal, focal)


_TILESPLAT = []


def load_tilesplat():
    """The UNMODIFIED reference package, or None: from a scratch copy of /root/reference (build
    container; nothing is written under the read-only tree), else from baseline/_ref (the
    git-ignored `pip install --target` of the same tree that travels to the GPU box)."""
    if _TILESPLAT:
        return _TILESPLAT[0]
    import importlib
    import shutil
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = "/root/reference/pkg/src/tilesplat"
    mod = None
    if os.path.isdir(src):
        d = tempfile.mkdtemp(prefix="fgs_ref_")
        shutil.copytree(src, os.path.join(d, "tilesplat"), ignore=shutil.ignore_patterns("__pycache__"))
        os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(d, "numba_cache"))
        where = d
    elif os.path.isdir(os.path.join(root, "baseline", "_ref", "tilesplat")):
        where = os.path.join(root, "baseline", "_ref")
    else:
        _TILESPLAT.append(None)
        return None
    old = sys.dont_write_bytecode
    sys.dont_write_bytecode = True
    sys.path.insert(0, where)
    try:
        mod = importlib.import_module("tilesplat")
    except Exception:                              # numba / pillow missing on this box
        mod = None
    finally:
        sys.path.remove(where)
        sys.dont_write_bytecode = old
    _TILESPLAT.append(mod)
    return mod
