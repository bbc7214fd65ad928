"""Instance frames: SRT -> 3x4 affine and its inverse (accel.py:290-336).

Host-side float64, identical numpy operation order to the reference so the
matrices (and hence the reference-style world normals) match it
bit for bit.
"""

import math
from dataclasses import dataclass, field

import numpy as np

FULL_MASK = 0xFFFFFFFF


def _vec3(v, name):
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise ValueError(f"{name} must have shape (3,), got {a.shape}")
    return a


@dataclass
class SrtFrame:
    """Scale, axis-angle rotation, translation; composed as T * R * S."""

    scale: np.ndarray = field(default_factory=lambda: np.ones(3))
    rotation_axis: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    rotation_angle: float = 0.0
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.scale = _vec3(self.scale, "scale")
        self.rotation_axis = _vec3(self.rotation_axis, "rotation_axis")
        self.translation = _vec3(self.translation, "translation")
        if np.any(self.scale == 0.0):
            raise ValueError("scale components must be nonzero")
        if self.rotation_angle != 0.0:
            alen = math.sqrt(float(np.dot(self.rotation_axis, self.rotation_axis)))
            if abs(alen - 1.0) > 1e-6:
                raise ValueError("rotation axis must be unit length")


def frame_to_matrix(frame: SrtFrame) -> np.ndarray:
    a = frame.rotation_axis
    k = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    rot = np.eye(3) + math.sin(frame.rotation_angle) * k + (1.0 - math.cos(frame.rotation_angle)) * (k @ k)
    m = np.empty((3, 4))
    m[:, :3] = rot * frame.scale[None, :]
    m[:, 3] = frame.translation
    return m


def invert_affine(m) -> np.ndarray:
    a = np.asarray(m, dtype=np.float64)
    if abs(np.linalg.det(a[:, :3])) <= 1e-12:
        raise ValueError("affine matrix is not invertible")
    inv3 = np.linalg.inv(a[:, :3])
    out = np.empty((3, 4))
    out[:, :3] = inv3
    out[:, 3] = -inv3 @ a[:, 3]
    return out
