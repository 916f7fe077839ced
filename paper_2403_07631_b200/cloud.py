"""PointCloud: the input type of the hot path (tomoplan/cloud_io.py:19-50).

Same constructor, validation, error types and attribute types as the
reference: ``cloud.xyz`` is an (N, 3) C-contiguous float64 array
(cloud_io.py:35).  The device path does not need that copy: the array the
caller passed is kept as ``cloud.points`` (float32 stays float32, anything
else becomes float64), the build uploads it directly (12 B/point for
float32 instead of 24), and ``xyz`` is materialised on first access only.
float32 -> float64 is exact, so every result is identical either way.
``bounds`` is computed on the GPU (and by the build itself, which never
reads this cache).
"""

from __future__ import annotations

import numpy as np


class CloudFormatError(ValueError):
    """Unreadable file, malformed header, or zero valid points."""


class PointCloud:
    """Unordered 3D points in meters (cloud_io.py:23-50).

    ``PointCloud(xyz, dropped=0)``; ``dropped`` counts non-finite rows
    removed at load time.  Treat instances as immutable once constructed.
    """

    __slots__ = ("points", "dropped", "_xyz64", "_bounds", "__weakref__")

    def __init__(self, xyz, dropped: int = 0):
        arr = np.asarray(xyz)
        if arr.dtype != np.float32:
            arr = np.asarray(arr, dtype=np.float64)
        arr = np.ascontiguousarray(arr)
        if arr.ndim != 2 or arr.shape[1] != 3:
            raise ValueError(f"expected (N, 3) point array, got shape {arr.shape}")
        if arr.shape[0] == 0:
            raise CloudFormatError("zero valid points")
        if not np.isfinite(arr).all():
            raise ValueError("point cloud contains non-finite coordinates")
        self.points = arr
        self.dropped = dropped
        self._xyz64 = arr if arr.dtype == np.float64 else None
        self._bounds = None

    @property
    def xyz(self) -> np.ndarray:
        """(N, 3) float64, as the reference stores it (cloud_io.py:35)."""
        if self._xyz64 is None:
            self._xyz64 = self.points.astype(np.float64)
        return self._xyz64

    def __len__(self):
        return self.points.shape[0]

    def __repr__(self):
        return f"PointCloud(n={len(self)}, dtype={self.points.dtype}, dropped={self.dropped})"

    def __eq__(self, other):
        if not hasattr(other, "xyz"):
            return NotImplemented
        return self.dropped == getattr(other, "dropped", 0) and np.array_equal(
            self.points, np.asarray(getattr(other, "points", other.xyz)))

    __hash__ = None

    @property
    def bounds(self):
        """Axis-aligned (min, max) corners as float64, computed on the device."""
        if self._bounds is None:
            from .tomogram import device_bounds
            self._bounds = device_bounds(self.points)
        return self._bounds


def source_points(cloud) -> np.ndarray:
    """The array the device path uploads: ``points`` of our PointCloud (no
    float64 copy), ``xyz`` of the reference's, or the array itself."""
    pts = getattr(cloud, "points", None)
    if isinstance(pts, np.ndarray):
        return pts
    return np.asarray(cloud.xyz if hasattr(cloud, "xyz") else cloud)
