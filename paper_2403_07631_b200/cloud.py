"""PointCloud: the input type of the hot path (tomoplan/cloud_io.py:19-50).

Same constructor, validation and error types as the reference.  One
deliberate difference: float32 input is kept as float32 (the reference
up-casts to float64; float32 -> float64 is exact, so every result is
identical) so the device path moves 12 instead of 24 bytes per point.
``bounds`` is computed on the GPU (and by the build itself, which never
reads this cache).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class CloudFormatError(ValueError):
    """Unreadable file, malformed header, or zero valid points."""


@dataclass
class PointCloud:
    xyz: np.ndarray
    dropped: int = 0

    def __post_init__(self):
        arr = np.asarray(self.xyz)
        if arr.dtype != np.float32:
            arr = np.asarray(arr, dtype=np.float64)
        arr = np.ascontiguousarray(arr)
        if arr.ndim != 2 or arr.shape[1] != 3:
            raise ValueError(f"expected (N, 3) point array, got shape {arr.shape}")
        if arr.shape[0] == 0:
            raise CloudFormatError("zero valid points")
        if not np.isfinite(arr).all():
            raise ValueError("point cloud contains non-finite coordinates")
        self.xyz = arr
        self._bounds = None

    def __len__(self):
        return self.xyz.shape[0]

    @property
    def bounds(self):
        """Axis-aligned (min, max) corners as float64, computed on the device."""
        if self._bounds is None:
            from .tomogram import device_bounds
            self._bounds = device_bounds(self.xyz)
        return self._bounds
