"""CPU oracle for the tomogram hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `tomoplan` algorithm for
the three stages on the hot path:

  tomography.py      build_tomogram           tomoplan/tomogram.py:127-213
  traversability.py  evaluate_tomogram & ops  tomoplan/traversability.py:59-236
  simplify.py        simplify_tomogram        tomoplan/simplify.py:18-73
  archive.py         LGA archive bytes        tomoplan/tomogram.py:219-276
  planner_ctx.py     canonical-node arrays    tomoplan/planner.py:62-93
  cloud_io.py        binary PCD payload       tomoplan/cloud_io.py:53-55,123-146
  trajectory.py      ceiling inflation        tomoplan/trajectory.py:277-317
  fast.py + c/       build / evaluate /       the same three stages restated in
                     simplify in C            multi-threaded C (full-size maps)

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the reference
package (only available in the build container, /root/reference) and records
its outputs on seeded inputs as fixtures under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this oracle bit-for-bit against them,
``tests/test_oracle_c.py`` the C restatement (plus the config-3 pins of
``golden_r2.json``, written by ``make_golden_r2.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / CPU baseline.  The product package
``paper_2403_07631_b200`` never imports it: there is no CPU fallback.
"""

from .tomography import bounds, build, frame, rasterize_index  # noqa: F401
from .traversability import (  # noqa: F401
    evaluate,
    evaluate_slice,
    fuse_costs,
    gentle_fraction,
    ground_cost,
    inflate,
    interval_cost,
    kernel_weights,
    slope_magnitudes,
    terrain_cost_values,
)
from .simplify import simplify, unique_mask  # noqa: F401
