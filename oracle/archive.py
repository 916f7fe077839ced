"""Oracle: the LGA archive bytes (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates the reference's "layered grid archive" writer, tomogram.py:219-244
(format notes README.md:111-121): little-endian header <4sIIIfdddfI (magic
b"LGA1", version 1, rows, cols, float32 resolution, float64 origin x/y,
float64 z_min, float32 d_s, slice count), then per slice <dB (float64 plane
height, layer mask 1|2|4) followed by the float32 ground, ceiling and (if
present) cost layers."""

import struct

import numpy as np

HEADER = struct.Struct("<4sIIIfdddfI")
SLICE = struct.Struct("<dB")


def lga_bytes(ground, ceiling, cost, heights, origin, r_g, z_min, d_s):
    S, rows, cols = ground.shape
    out = bytearray(HEADER.pack(b"LGA1", 1, rows, cols, np.float32(r_g), float(origin[0]),
                                float(origin[1]), float(z_min), np.float32(d_s), S))
    for k in range(S):
        out += SLICE.pack(float(heights[k]), 1 | 2 | (4 if cost is not None else 0))
        out += np.ascontiguousarray(ground[k], "<f4").tobytes()
        out += np.ascontiguousarray(ceiling[k], "<f4").tobytes()
        if cost is not None:
            out += np.ascontiguousarray(cost[k], "<f4").tobytes()
    return bytes(out)
