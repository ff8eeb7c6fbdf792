"""Load the golden fixtures in tests/golden/ (made by make_golden.py from the
reference itself) into light-weight cloud / camera records."""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Cam:
    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    @property
    def position(self) -> np.ndarray:
        return -self.rotation.T @ self.translation


@dataclass
class Cloud:
    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    opacity_logits: np.ndarray
    sh_coeffs: np.ndarray
    degree: int = 1

    @property
    def count(self) -> int:
        return self.positions.shape[0]

    def copy(self) -> "Cloud":
        return Cloud(self.positions.copy(), self.log_scales.copy(), self.rotations.copy(),
                     self.opacity_logits.copy(), self.sh_coeffs.copy(), self.degree)


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def cam_from(d: dict, prefix: str = "cam_") -> Cam:
    intr = d[prefix + "intr"]
    size = d[prefix + "size"]
    return Cam(rotation=np.asarray(d[prefix + "R"], dtype=np.float64),
               translation=np.asarray(d[prefix + "t"], dtype=np.float64),
               fx=float(intr[0]), fy=float(intr[1]), cx=float(intr[2]), cy=float(intr[3]),
               width=int(size[0]), height=int(size[1]))


def cloud_from(d: dict, prefix: str = "") -> Cloud:
    return Cloud(positions=d[prefix + "positions"], log_scales=d[prefix + "log_scales"],
                 rotations=d[prefix + "rotations"],
                 opacity_logits=d[prefix + "opacity_logits"],
                 sh_coeffs=d[prefix + "sh_coeffs"], degree=int(d[prefix + "degree"]))


RENDER_CASES = ["random60", "fd8", "rect150_f32", "sphere_init"]
