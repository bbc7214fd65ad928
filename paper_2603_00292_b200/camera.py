"""Pinhole camera with radial distortion (camera.py:24-97 of the reference).

Only the parameters live on the host; the ray generation itself runs inside
the CUDA raygen / megakernel (``rt_raygen`` in csrc/render.cu), in fp32.
"""

import math
from dataclasses import dataclass, field

import numpy as np


class CameraError(ValueError):
    pass


def _vec3(v, name):
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise ValueError(f"{name} must have shape (3,), got {a.shape}")
    return a


@dataclass
class Camera:
    origin: np.ndarray
    right: np.ndarray
    up: np.ndarray
    distortion: float = 0.0
    forward: np.ndarray = field(init=False)

    def __post_init__(self):
        self.origin = _vec3(self.origin, "origin")
        self.right = _vec3(self.right, "right")
        self.up = _vec3(self.up, "up")
        fwd = np.cross(self.up, self.right)
        if not np.any(fwd != 0.0):
            raise CameraError("right and up are parallel, film is degenerate")
        n = math.sqrt(float(np.dot(fwd, fwd)))
        self.forward = np.asarray(fwd, dtype=np.float64) / n

    def validate_distortion(self):
        """camera.py:40-52: 1 + d*|p|^2 must stay positive on the whole film."""
        c1 = float(np.dot(self.right + self.up, self.right + self.up))
        c2 = float(np.dot(self.right - self.up, self.right - self.up))
        if 1.0 + self.distortion * max(c1, c2) <= 0.0:
            raise CameraError(
                f"distortion {self.distortion} collapses the lens mapping at the film corner")

    def as_tuple(self):
        """integrators.py:397-402 order: origin, right, up, forward, distortion."""
        return (*map(float, self.origin), *map(float, self.right), *map(float, self.up),
                *map(float, self.forward), float(self.distortion))


def pixel_to_uv(xi, yi, width, height, jitter_u=0.0, jitter_v=0.0):
    return (xi + jitter_u) / width, (yi + jitter_v) / height
