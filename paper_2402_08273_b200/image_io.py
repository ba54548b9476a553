"""PFM image I/O of the reference (core/image_io.cpp:15-56), for the images the
engine produces (``RenderResult.image``) and reference images for the metrics
rRMSE (``Engine.set_reference``): colour PFM, little-endian (scale -1.0), rows
stored bottom to top; reading also accepts big-endian files (scale > 0).
Errors are the reference's ``std::runtime_error`` messages as RuntimeError."""
from __future__ import annotations

import numpy as np


def write_pfm(image: np.ndarray, path: str) -> None:
    """write_pfm (core/image_io.cpp:15-25): ``image`` is (H, W, 3), row 0 at the top."""
    img = np.ascontiguousarray(image, np.float32)
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("write_pfm: image must be (H, W, 3)")
    h, w = img.shape[:2]
    try:
        with open(path, "wb") as f:
            f.write(f"PF\n{w} {h}\n-1.0\n".encode())
            f.write(img[::-1].astype("<f4").tobytes())
    except OSError:
        raise RuntimeError(f"cannot open '{path}' for writing") from None


def read_pfm(path: str) -> np.ndarray:
    """read_pfm (core/image_io.cpp:27-56): returns (H, W, 3) float32, row 0 at the top."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"cannot open '{path}'") from None
    toks, pos = [], 0
    while len(toks) < 4:   # magic, width, height, scale (whitespace separated, like operator>>)
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            break
        toks.append(data[start:pos].decode("latin-1"))
        if toks[0] != "PF":
            raise RuntimeError(f"'{path}' is not a color PFM file")
    try:
        w, h, scale = int(toks[1]), int(toks[2]), float(toks[3])
    except (IndexError, ValueError):
        raise RuntimeError(f"'{path}': malformed PFM header") from None
    if w <= 0 or h <= 0 or scale == 0.0:
        raise RuntimeError(f"'{path}': malformed PFM header")
    pos += 1   # single whitespace after the scale
    n = w * h * 3
    raw = data[pos:pos + 4 * n]
    if len(raw) < 4 * n:
        raise RuntimeError(f"'{path}': truncated PFM data")
    arr = np.frombuffer(raw, ">f4" if scale > 0 else "<f4").astype(np.float32).reshape(h, w, 3)
    return np.ascontiguousarray(arr[::-1])
