"""B200-native point-cloud tomography hot path (arXiv 2403.07631).

Drop-in replacement for the build -> evaluate -> simplify path of the
reference package ``tomoplan`` (same names, signatures, object model and
errors), executed by hand-written sm_100a CUDA kernels in libpct.so through
a C ABI (include/pct.h).  There is no CPU fallback.
"""

from .archive import load_tomogram, save_tomogram
from . import cloud_io
from .cloud import CloudFormatError, PointCloud
from .cloud_io import DeviceCloud, load_cloud, sniff_format
from .simplify import DEFAULT_EPS_E, simplify_tomogram, unique_cells
from .tomogram import (
    GRID_SIDE_LIMIT,
    GridSizeError,
    Layer,
    Tomogram,
    TomogramSlice,
    build_tomogram,
    rasterize_index,
)
from .traversability import (
    InflationKernel,
    TravParams,
    build_kernel,
    evaluate_slice,
    evaluate_tomogram,
    fuse_costs,
    gentle_fraction,
    ground_cost,
    inflate,
    interval_cost,
    slope_magnitudes,
    terrain_cost_values,
)

__version__ = "0.1.0"

__all__ = [
    "CloudFormatError", "PointCloud", "DEFAULT_EPS_E", "simplify_tomogram", "unique_cells",
    "GRID_SIDE_LIMIT", "GridSizeError", "Layer", "Tomogram", "TomogramSlice", "build_tomogram",
    "rasterize_index", "InflationKernel", "TravParams", "build_kernel", "evaluate_slice",
    "evaluate_tomogram", "fuse_costs", "gentle_fraction", "ground_cost", "inflate",
    "interval_cost", "slope_magnitudes", "terrain_cost_values", "save_tomogram", "load_tomogram",
    "cloud_io", "DeviceCloud", "load_cloud", "sniff_format",
]
