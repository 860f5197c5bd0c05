"""Frame export, the format side after the path (reference ``images.py:12-55``).

``write_ppm`` is the reference's canonical bit-exact output (binary P6 of the
8-bit quantised frame, ``q = floor(clip(c, 0, 1) * 255 + 0.5)``).  A frame that is
still on the device (a CUDA tensor, e.g. ``Framebuffer.image`` from
``render(..., as_numpy=False)``) is quantised there (``fgs_quantize_rgb8``) so only
3 bytes per pixel cross PCIe; a NumPy frame is quantised on the host with the
same rule.  ``read_ppm`` reads such a file back; PNG needs Pillow.
"""

from __future__ import annotations

import numpy as np

from .service import png_bytes as _png_of_rgb8
from .service import ppm_bytes as _ppm_of_rgb8
from .service import quantize as _quantize_host


def quantize(image) -> np.ndarray:
    """float32 (H, W, 3) linear -> uint8 (``images.py:12-15``); device frames are
    quantised by the library, host frames by NumPy -- both give the same bytes."""
    if hasattr(image, "is_cuda") and image.is_cuda:
        import ctypes as C

        import torch

        from . import _capi
        img = image.contiguous().to(torch.float32)
        out = torch.empty(img.shape, dtype=torch.uint8, device=img.device)
        with torch.cuda.device(img.device):
            _capi.check(_capi.lib().fgs_quantize_rgb8(
                C.c_void_p(img.data_ptr()), img.numel(), C.c_void_p(out.data_ptr()),
                C.c_void_p(torch.cuda.current_stream(img.device).cuda_stream)))
        return out.cpu().numpy()
    return _quantize_host(image)


def write_ppm(image, path) -> None:
    """Binary P6, maxval 255 (``images.py:18-24``)."""
    with open(path, "wb") as f:
        f.write(_ppm_of_rgb8(quantize(image)))


def read_ppm(path) -> np.ndarray:
    """A binary P6 file with maxval 255, as ``write_ppm`` writes it, back as an
    ``(H, W, 3)`` uint8 array (the reference's reader: ``images.py:27-39``)."""
    with open(path, "rb") as f:
        blob = f.read()
    # header = three whitespace-separated fields after the magic, then ONE whitespace byte
    fields, pos = [], 0
    while len(fields) < 4:
        while pos < len(blob) and blob[pos:pos + 1].isspace():
            pos += 1
        end = pos
        while end < len(blob) and not blob[end:end + 1].isspace():
            end += 1
        fields.append(blob[pos:end])
        pos = end
    if fields[0] != b"P6":
        raise ValueError(f"not a P6 PPM: {fields[0]!r}")
    width, height, maxval = (int(v) for v in fields[1:])
    if maxval != 255:
        raise ValueError(f"unsupported maxval {maxval}")
    body = blob[pos + 1:pos + 1 + width * height * 3]
    if len(body) != width * height * 3:
        raise ValueError("truncated PPM body")
    return np.frombuffer(body, dtype=np.uint8).reshape(height, width, 3)


def png_bytes(image) -> bytes:
    """``images.py:46-55``."""
    return _png_of_rgb8(quantize(image))


def write_png(image, path) -> None:
    """``images.py:42-45``."""
    with open(path, "wb") as f:
        f.write(png_bytes(image))
