"""Synthetic MNIST-shaped data for config 3.

Real MNIST is not available offline, so config 3 uses a seeded synthetic IDX3
file in the reference's format (proj/src/instances.cpp:80-103: big-endian
magic 0x00000803, count, 28, 28, then count*784 uint8 pixels).

Generator (deterministic, numpy PCG64): every image is one filled ellipse
"digit stroke" centred in the middle of the frame (centre row/col uniform in
12..16, semi-axes uniform in [4.5, 8.5]) with pixel intensities uniform in
1..255 inside it and 0 outside.  All supports overlap around the frame
centre, so no pair of images has disjoint support — the reference rejects
such pairs because roundoff pushes L1/2 just above 1.0 — and no
image is blank (instances.cpp:121-123 would throw).
"""
from __future__ import annotations

import struct

import numpy as np


def synth_images(count: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(np.random.PCG64(0x5EED0003 + seed))
    yy, xx = np.mgrid[0:28, 0:28]
    out = np.zeros((count, 28, 28), np.uint8)
    cy = rng.integers(12, 17, count)
    cx = rng.integers(12, 17, count)
    ry = rng.uniform(4.5, 8.5, count)
    rx = rng.uniform(4.5, 8.5, count)
    for i in range(count):
        mask = ((yy - cy[i]) / ry[i]) ** 2 + ((xx - cx[i]) / rx[i]) ** 2 <= 1.0
        out[i][mask] = rng.integers(1, 256, int(mask.sum()), dtype=np.uint8)
    return out.reshape(count, 784)


def write_idx3(path: str, images: np.ndarray) -> None:
    images = np.ascontiguousarray(images, np.uint8).reshape(-1, 784)
    with open(path, "wb") as f:
        f.write(struct.pack(">IIII", 0x00000803, images.shape[0], 28, 28))
        f.write(images.tobytes())


def make_synthetic_mnist(path: str, count: int = 20000, seed: int = 0) -> str:
    """Write the config-3 IDX3 file (count images) and return its path."""
    write_idx3(path, synth_images(count, seed))
    return path
