"""Seeded synthetic point clouds for the five BASELINE.json configurations.

The reference's scene generator (`tomoplan/scenes.py:275-291`) has none of
these scene kinds, so each configuration gets its own generator here.  All
generators draw from ``numpy.random.default_rng(seed)`` (PCG64), sample every
surface uniformly at random by area, add isotropic Gaussian noise, and return
a C-contiguous ``(N, 3)`` float32 array.  They are inputs only: the GPU path
and the CPU oracle consume the same array, so parity does not depend on how
realistic the geometry is.

Config index -> generator:
  0  two_storey   250k pts, 20x20 m, floor/slab/roof, 15 deg ramp, walls with doors
  1  spiral_ramp  5M pts, 60x60 m, 5 decks, 10 deg helical ramp, pillars, low beams
  2  rough_terrain 20M pts, 100x100 m fBm terrain, stairs, 200 floating boxes,
                 log-normal density
  3  campus      200M pts, 400x400 m, 16 three-storey buildings, walkways
  4  batch       256 x config 0 with per-seed layout jitter
"""

from __future__ import annotations

import math

import numpy as np

# (n_points, r_g, d_s, seed) per config, from BASELINE.json "configs"
CONFIGS = {
    0: dict(name="two_storey", n_points=250_000, r_g=0.10, d_s=0.5, seed=0),
    1: dict(name="spiral_ramp", n_points=5_000_000, r_g=0.10, d_s=0.4, seed=1),
    2: dict(name="rough_terrain", n_points=20_000_000, r_g=0.05, d_s=0.3, seed=2),
    3: dict(name="campus", n_points=200_000_000, r_g=0.10, d_s=0.5, seed=3),
    4: dict(name="batch_two_storey", n_points=250_000, r_g=0.10, d_s=0.5, seed=1000,
            n_maps=256),
}


# ---------------------------------------------------------------------------
# surface primitives: each returns (area, sampler(rng, n) -> (n, 3) float64,
# xy bounding box (x_lo, y_lo, x_hi, y_hi))


def _bb(xs, ys):
    return (min(xs), min(ys), max(xs), max(ys))

def _hrect(x0, y0, lx, ly, z):
    """Horizontal rectangle; z is a constant or a callable z(x, y)."""
    def draw(rng, n):
        x = x0 + rng.random(n) * lx
        y = y0 + rng.random(n) * ly
        zz = np.full(n, float(z)) if not callable(z) else z(x, y)
        return np.column_stack([x, y, zz])
    return abs(lx * ly), draw, _bb((x0, x0 + lx), (y0, y0 + ly))


def _vrect(x0, y0, x1, y1, z0, z1):
    """Vertical rectangle spanning the segment (x0,y0)-(x1,y1) and [z0, z1]."""
    length = math.hypot(x1 - x0, y1 - y0)

    def draw(rng, n):
        s = rng.random(n)
        return np.column_stack([x0 + s * (x1 - x0), y0 + s * (y1 - y0),
                                z0 + rng.random(n) * (z1 - z0)])
    return length * abs(z1 - z0), draw, _bb((x0, x1), (y0, y1))


def _incline(x0, y0, lx, ly, z0, slope_x):
    """Rectangle rising along +x with dz/dx = slope_x (area is the true area)."""
    def draw(rng, n):
        u = rng.random(n) * lx
        return np.column_stack([x0 + u, y0 + rng.random(n) * ly, z0 + u * slope_x])
    return lx * ly * math.sqrt(1.0 + slope_x * slope_x), draw, _bb((x0, x0 + lx), (y0, y0 + ly))


def _helix(cx, cy, r_in, r_out, z0, rise_per_rad, theta_total):
    """Helical ramp surface between radii r_in and r_out."""
    area = 0.5 * theta_total * (r_out ** 2 - r_in ** 2)

    def draw(rng, n):
        th = rng.random(n) * theta_total
        r = np.sqrt(r_in ** 2 + rng.random(n) * (r_out ** 2 - r_in ** 2))
        return np.column_stack([cx + r * np.cos(th), cy + r * np.sin(th),
                                z0 + th * rise_per_rad])
    return area, draw, (cx - r_out, cy - r_out, cx + r_out, cy + r_out)


def _box_faces(x0, y0, z0, sx, sy, sz, faces="tbs"):
    out = []
    if "t" in faces:
        out.append(_hrect(x0, y0, sx, sy, z0 + sz))
    if "b" in faces:
        out.append(_hrect(x0, y0, sx, sy, z0))
    if "s" in faces:
        x1, y1, z1 = x0 + sx, y0 + sy, z0 + sz
        out += [_vrect(x0, y0, x1, y0, z0, z1), _vrect(x1, y0, x1, y1, z0, z1),
                _vrect(x1, y1, x0, y1, z0, z1), _vrect(x0, y1, x0, y0, z0, z1)]
    return out


def _wall_with_door(x0, y0, x1, y1, z0, z1, thick, door_at, door_w, door_h):
    """Two faces of a wall of the given thickness with one door gap (both faces)."""
    length = math.hypot(x1 - x0, y1 - y0)
    ux, uy = (x1 - x0) / length, (y1 - y0) / length
    nx, ny = -uy * thick, ux * thick
    parts = []
    a, b = door_at, door_at + door_w
    for ox, oy in ((0.0, 0.0), (nx, ny)):
        def seg(s0, s1, za, zb):
            return _vrect(x0 + ox + ux * s0, y0 + oy + uy * s0,
                          x0 + ox + ux * s1, y0 + oy + uy * s1, za, zb)
        parts.append(seg(0.0, a, z0, z1))
        parts.append(seg(b, length, z0, z1))
        parts.append(seg(a, b, z0 + door_h, z1))     # lintel above the door
    # wall top
    parts.append(_incline_strip(x0, y0, x1, y1, nx, ny, z1))
    return parts


def _incline_strip(x0, y0, x1, y1, nx, ny, z):
    length = math.hypot(x1 - x0, y1 - y0)
    thick = math.hypot(nx, ny)

    def draw(rng, n):
        s = rng.random(n)
        t = rng.random(n)
        return np.column_stack([x0 + s * (x1 - x0) + t * nx,
                                y0 + s * (y1 - y0) + t * ny, np.full(n, z)])
    return length * thick, draw, _bb((x0, x1, x0 + nx, x1 + nx), (y0, y1, y0 + ny, y1 + ny))


def _hrect_with_hole(x0, y0, lx, ly, z, hx0, hy0, hlx, hly):
    """Horizontal rectangle minus an axis-aligned opening (four pieces)."""
    return [_hrect(x0, y0, lx, hy0 - y0, z),
            _hrect(x0, hy0 + hly, lx, y0 + ly - hy0 - hly, z),
            _hrect(x0, hy0, hx0 - x0, hly, z),
            _hrect(hx0 + hlx, hy0, x0 + lx - hx0 - hlx, hly, z)]


def _stair(x0, y0, width, z0, steps, rise, tread):
    """Straight flight rising along +x: `steps` treads and their risers."""
    parts = []
    for s in range(steps):
        z = z0 + (s + 1) * rise
        parts.append(_hrect(x0 + s * tread, y0, tread, width, z))
        parts.append(_vrect(x0 + s * tread, y0, x0 + s * tread, y0 + width, z - rise, z))
    return parts


def _sample(parts, n_points, sigma, rng, weights=None):
    areas = np.array([p[0] for p in parts], dtype=np.float64)
    if weights is not None:
        areas = areas * weights
    counts = rng.multinomial(n_points, areas / areas.sum())
    out = np.empty((n_points, 3), dtype=np.float32)
    pos = 0
    for (_, draw, _), c in zip(parts, counts):
        if c:
            out[pos:pos + c] = draw(rng, int(c))
            pos += c
    if sigma > 0:
        # noise in chunks to bound float64 temporaries on the 200M config
        step = 1 << 24
        for a in range(0, n_points, step):
            b = min(n_points, a + step)
            out[a:b] += rng.normal(0.0, sigma, (b - a, 3)).astype(np.float32)
    return out


def _sample_seeded(parts, n_points, sigma, seed, box=None, workers=8, share=None):
    """Like _sample, but part i draws its points and noise from its own
    generator ``default_rng([seed, i])``.  The cloud is the same whichever
    parts are drawn and in whatever order, so (a) the parts are drawn in
    parallel threads and (b) ``box = (x_lo, y_lo, x_hi, y_hi)`` yields
    exactly the points of the full cloud inside the box (half-open) while
    drawing only the parts whose footprint comes near it, and (c) ``share =
    (r, n)`` draws only the parts i with i % n == r: n such shares are a
    partition of the cloud (one per rank of a sharded run)."""
    from concurrent.futures import ThreadPoolExecutor
    areas = np.array([p[0] for p in parts], dtype=np.float64)
    counts = np.random.default_rng([seed, len(parts)]).multinomial(n_points, areas / areas.sum())
    pad = 8.0 * sigma + 1e-6  # noise never moves a point further than this (p < 1e-15)
    todo = []
    for i, (p, c) in enumerate(zip(parts, counts)):
        if c == 0 or (share is not None and i % share[1] != share[0]):
            continue
        if box is not None:
            bx = p[2]
            if bx[0] > box[2] + pad or bx[2] < box[0] - pad or bx[1] > box[3] + pad \
                    or bx[3] < box[1] - pad:
                continue
        todo.append((i, p[1], int(c)))
    offs = np.concatenate([[0], np.cumsum([c for _, _, c in todo])]).astype(np.int64)
    out = np.empty((int(offs[-1]), 3), dtype=np.float32)

    def one(t):
        i, draw, c = todo[t]
        rng = np.random.default_rng([seed, i])
        dst = out[offs[t]:offs[t + 1]]
        step = 1 << 22
        for a in range(0, c, step):
            b = min(c, a + step)
            dst[a:b] = draw(rng, b - a)
            if sigma > 0:
                dst[a:b] += rng.normal(0.0, sigma, (b - a, 3)).astype(np.float32)

    with ThreadPoolExecutor(max(1, workers)) as ex:
        list(ex.map(one, range(len(todo))))
    if box is not None:
        m = (out[:, 0] >= box[0]) & (out[:, 0] < box[2]) & (out[:, 1] >= box[1]) & \
            (out[:, 1] < box[3])
        out = np.ascontiguousarray(out[m])
    return out


# ---------------------------------------------------------------------------
# fBm value noise (vectorised; lattice drawn from the scene rng)

class _Fbm:
    def __init__(self, rng, extent, octaves=4, amplitude=2.0, lacunarity=2.0,
                 base_wavelength=25.0, gain=0.5):
        self.octs = []
        freq = 1.0 / base_wavelength
        amp = amplitude
        for _ in range(octaves):
            n = int(math.ceil(extent * freq)) + 3
            self.octs.append((freq, amp, rng.uniform(-1.0, 1.0, (n, n))))
            freq *= lacunarity
            amp *= gain

    def __call__(self, x, y):
        z = np.zeros_like(x, dtype=np.float64)
        for freq, amp, lat in self.octs:
            u = x * freq
            v = y * freq
            i = np.floor(u).astype(np.int64)
            j = np.floor(v).astype(np.int64)
            fu = u - i
            fv = v - j
            fu = fu * fu * (3 - 2 * fu)
            fv = fv * fv * (3 - 2 * fv)
            n = lat.shape[0]
            i = np.clip(i, 0, n - 2)
            j = np.clip(j, 0, n - 2)
            a = lat[i, j] * (1 - fu) + lat[i + 1, j] * fu
            b = lat[i, j + 1] * (1 - fu) + lat[i + 1, j + 1] * fu
            z += amp * (a * (1 - fv) + b * fv)
        return z


# ---------------------------------------------------------------------------
# config generators

def two_storey(n_points=250_000, seed=0, jitter=False, sigma=0.02):
    """Config 0: floor z=0, slab z=3 (top+bottom), roof z=6 over 20x20 m,
    a 4 m wide 15 degree ramp floor->slab, four 0.3 m walls with door gaps."""
    rng = np.random.default_rng(seed)
    L = 20.0
    ox = oy = 0.0
    ramp_x0, ramp_y0 = 4.0, 14.0
    doors = [3.0, 8.0, 12.0, 5.0]
    if jitter:
        ox, oy = rng.uniform(-2.0, 2.0, 2)
        ramp_x0 += rng.uniform(-1.5, 1.5)
        ramp_y0 += rng.uniform(-1.0, 1.0)
        doors = list(rng.uniform(1.0, 16.0, 4))
    run = 3.0 / math.tan(math.radians(15.0))
    rw = 4.0
    parts = [_hrect(ox, oy, L, L, 0.0), _hrect(ox, oy, L, L, 6.0)]
    # slab with the ramp opening [ramp_x0, ramp_x0+run] x [ramp_y0, ramp_y0+rw]
    rx0, rx1 = ox + ramp_x0, ox + ramp_x0 + run
    ry0, ry1 = oy + ramp_y0, oy + ramp_y0 + rw
    for z in (3.0, 2.8):
        parts += [_hrect(ox, oy, L, ry0 - oy, z),
                  _hrect(ox, ry1, L, oy + L - ry1, z),
                  _hrect(ox, ry0, rx0 - ox, rw, z),
                  _hrect(rx1, ry0, ox + L - rx1, rw, z)]
    parts.append(_incline(rx0, ry0, run, rw, 0.0, math.tan(math.radians(15.0))))
    t = 0.3
    corners = [(ox, oy), (ox + L, oy), (ox + L, oy + L), (ox, oy + L)]
    for w in range(4):
        (xa, ya), (xb, yb) = corners[w], corners[(w + 1) % 4]
        parts += _wall_with_door(xa, ya, xb, yb, 0.0, 6.0, t, doors[w], 1.2, 2.2)
    return _sample(parts, n_points, sigma, rng)


def spiral_ramp(n_points=5_000_000, seed=1, sigma=0.02):
    """Config 1: five decks every 3 m over 60x60 m joined by a 6 m wide 10 degree
    helical ramp; 0.5 m pillars every 8 m; low beams 2.2 m above each deck."""
    rng = np.random.default_rng(seed)
    half = 30.0
    hole = 9.0
    r_in, r_out = 2.5, 8.5
    r_mid = 0.5 * (r_in + r_out)
    rise_per_rad = math.tan(math.radians(10.0)) * r_mid
    levels = [0.0, 3.0, 6.0, 9.0, 12.0]
    parts = []
    for li, z in enumerate(levels):
        for zz in ((z,) if li == 0 else (z, z - 0.25)):
            if li == 0:
                parts.append(_hrect(-half, -half, 2 * half, 2 * half, zz))
            else:
                # deck with a square opening around the helix
                parts += [_hrect(-half, -half, 2 * half, half - hole, zz),
                          _hrect(-half, hole, 2 * half, half - hole, zz),
                          _hrect(-half, -hole, half - hole, 2 * hole, zz),
                          _hrect(hole, -hole, half - hole, 2 * hole, zz)]
    theta_total = (levels[-1] - levels[0]) / rise_per_rad
    parts.append(_helix(0.0, 0.0, r_in, r_out, 0.0, rise_per_rad, theta_total))
    posts = np.arange(-28.0, 28.1, 8.0)
    for px in posts:
        for py in posts:
            if abs(px) < hole + 1 and abs(py) < hole + 1:
                continue
            parts += _box_faces(px - 0.25, py - 0.25, 0.0, 0.5, 0.5, levels[-1], faces="s")
    # low beams: 0.4 m wide, 0.4 m deep, bottom 2.2 m above each deck, along x
    for z in levels:
        for py in posts[1::2]:
            for x0, x1 in ((-half, -hole), (hole, half)):
                parts += _box_faces(x0, py - 0.2, z + 2.2, x1 - x0, 0.4, 0.4, faces="tb")
    return _sample(parts, n_points, sigma, rng)


def rough_terrain(n_points=20_000_000, seed=2, sigma=0.02, extent=100.0,
                  n_boxes=200, n_stairs=24):
    """Config 2: fBm heightfield (4 octaves, amplitude 2 m, lacunarity 2) with
    stairs of 0.17 m risers and floating boxes 0.6-2.5 m above ground;
    terrain density is log-normal (sigma 0.5) over 2x2 m patches."""
    rng = np.random.default_rng(seed)
    fbm = _Fbm(rng, extent)
    parts = []
    weights = []
    patch = 2.0
    npatch = int(extent / patch)
    dens = rng.lognormal(0.0, 0.5, (npatch, npatch))
    for a in range(npatch):
        for b in range(npatch):
            parts.append(_hrect(a * patch, b * patch, patch, patch, fbm))
            weights.append(dens[a, b])
    for _ in range(n_stairs):
        x0, y0 = rng.uniform(5.0, extent - 10.0, 2)
        base = float(fbm(np.array([x0]), np.array([y0]))[0])
        width, run, rise, steps = 2.0, 0.3, 0.17, 10
        for s in range(steps):
            z = base + (s + 1) * rise
            parts.append(_hrect(x0 + s * run, y0, run, width, z))
            parts.append(_vrect(x0 + s * run, y0, x0 + s * run, y0 + width, z - rise, z))
            weights += [1.0, 1.0]
    for _ in range(n_boxes):
        sx, sy = rng.uniform(1.0, 4.0, 2)
        x0 = rng.uniform(0.0, extent - sx)
        y0 = rng.uniform(0.0, extent - sy)
        g = float(fbm(np.array([x0 + sx / 2]), np.array([y0 + sy / 2]))[0])
        z0 = g + rng.uniform(0.6, 2.5)
        faces = _box_faces(x0, y0, z0, sx, sy, 0.3)
        parts += faces
        weights += [1.0] * len(faces)
    return _sample(parts, n_points, sigma, rng, weights=np.asarray(weights))


def campus(n_points=200_000_000, seed=3, sigma=0.03, extent=400.0, box=None, share=None):
    """Config 3: 400x400 m sloped terrain, 16 three-storey buildings (floors
    every 4 m, roof, perimeter walls with doors, internal ramps between the
    floors, a stair of 0.167 m risers from the top floor to the roof),
    walkways at 5 m between neighbouring buildings, rooftop plant rooms.
    Every surface draws from its own seeded generator (_sample_seeded), so
    ``box`` cheaply yields the exact crop of the full cloud and ``share =
    (rank, world)`` one rank's part of it."""
    rng = np.random.default_rng(seed)
    fbm = _Fbm(rng, extent, amplitude=0.5, base_wavelength=40.0)

    def ground(x, y):
        return 0.01 * x + 0.005 * y + fbm(x, y)

    parts = []
    bsz = 40.0
    pitch = extent / 4
    sites = []
    # terrain in strips around the building footprints (coarse 10 m patches)
    for a in range(int(extent / 10)):
        for b in range(int(extent / 10)):
            x0, y0 = a * 10.0, b * 10.0
            inside = False
            for bi in range(4):
                for bj in range(4):
                    bx = bi * pitch + (pitch - bsz) / 2
                    by = bj * pitch + (pitch - bsz) / 2
                    if bx <= x0 < bx + bsz and by <= y0 < by + bsz:
                        inside = True
            if not inside:
                parts.append(_hrect(x0, y0, 10.0, 10.0, ground))
    for bi in range(4):
        for bj in range(4):
            bx = bi * pitch + (pitch - bsz) / 2
            by = bj * pitch + (pitch - bsz) / 2
            base = float(ground(np.array([bx + bsz / 2]), np.array([by + bsz / 2]))[0])
            sites.append((bx, by, base))
            run = 4.0 / math.tan(math.radians(15.0))
            rx0, ry0 = bx + 4.0, by + 30.0
            st_steps, st_tread = 24, 0.3
            sx0, sy0 = bx + 20.0, by + 4.0
            for f in range(4):       # ground floor, 2 upper floors, roof
                z = base + 4.0 * f
                surfaces = (z,) if f == 0 else (z, z - 0.3)
                for zz in surfaces:
                    if f in (1, 2):   # opening above the ramp from the floor below
                        parts += _hrect_with_hole(bx, by, bsz, bsz, zz, rx0, ry0, run, 3.0)
                    elif f == 3:      # opening above the stair
                        parts += _hrect_with_hole(bx, by, bsz, bsz, zz, sx0, sy0,
                                                  st_steps * st_tread, 2.0)
                    else:
                        parts.append(_hrect(bx, by, bsz, bsz, zz))
                if f < 2:
                    parts.append(_incline(rx0, ry0, run, 3.0, z, 4.0 / run))
            parts += _stair(sx0, sy0, 2.0, base + 8.0, st_steps, 4.0 / st_steps, st_tread)
            corners = [(bx, by), (bx + bsz, by), (bx + bsz, by + bsz), (bx, by + bsz)]
            for w in range(4):
                (xa, ya), (xb, yb) = corners[w], corners[(w + 1) % 4]
                parts += _wall_with_door(xa, ya, xb, yb, base, base + 12.0, 0.3,
                                         float(rng.uniform(2.0, 36.0)), 2.0, 2.6)
            # rooftop plant room
            px, py = bx + rng.uniform(5.0, 25.0), by + rng.uniform(5.0, 25.0)
            parts += _box_faces(px, py, base + 12.0, 8.0, 8.0, 4.0, faces="ts")
    for bi in range(3):
        for bj in range(4):
            bx, by, base = sites[bi * 4 + bj]
            nx_, _, nbase = sites[(bi + 1) * 4 + bj]
            z = 0.5 * (base + nbase) + 5.0
            x0 = bx + bsz
            parts += [_hrect(x0, by + 18.0, nx_ - x0, 3.0, z),
                      _hrect(x0, by + 18.0, nx_ - x0, 3.0, z - 0.4)]
    return _sample_seeded(parts, n_points, sigma, seed, box=box, share=share)


def generate(config: int, n_points: int | None = None, seed: int | None = None):
    """The seeded float32 (N, 3) cloud of a BASELINE.json config (index 0-4).

    ``n_points`` / ``seed`` override the config's values (tests use reduced
    point counts).  Config 4 returns one map; pass ``seed=1000 + m`` for map m.
    """
    c = CONFIGS[config]
    n = c["n_points"] if n_points is None else int(n_points)
    s = c["seed"] if seed is None else int(seed)
    if config == 0:
        return two_storey(n, s)
    if config == 1:
        return spiral_ramp(n, s)
    if config == 2:
        return rough_terrain(n, s)
    if config == 3:
        return campus(n, s)
    if config == 4:
        return two_storey(n, s, jitter=True)
    raise ValueError(f"unknown config {config}")
