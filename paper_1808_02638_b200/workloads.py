"""Seeded synthetic workloads (patch layouts + initial conditions).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle: it builds patch descriptor lists and initial data and holds none of
the method's arithmetic (no Riemann solver, limiter, update or ghost rule).
It imports nothing from the rest of the package.

Shapes follow BASELINE.json's configs and the paper's benchmark (P:445-504:
radial acoustics, ring-shaped pressure perturbation, outflow boundaries,
fp64).  The ring itself is not printed in the paper; we use Clawpack's
public acoustics_2d_radial qinit (reading R11):
    p = 1 + cos(pi (r - 0.5) / 0.2)   if |r - 0.5| <= 0.2,   else 0;  u = v = 0.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# C layout of claw_patch_desc / oracle_patch_desc (natural alignment, 64 B).
PATCH_DTYPE = np.dtype(
    [("mx", "<i4"), ("my", "<i4"), ("dx", "<f8"), ("dy", "<f8"),
     ("xlower", "<f8"), ("ylower", "<f8"), ("mbc", "<i4"),
     ("rho", "<f8"), ("K", "<f8")], align=True)
assert PATCH_DTYPE.itemsize == 64

DOMAIN = (-1.0, 1.0, -1.0, 1.0)
EXTRAP = (1, 1, 1, 1)
PERIODIC = (2, 2, 2, 2)


@dataclass
class Level:
    descs: np.ndarray            # PATCH_DTYPE records
    ratio: int | None = None     # refinement ratio to the coarser level

    @property
    def cells(self) -> int:
        return int((self.descs["mx"].astype(np.int64) * self.descs["my"]).sum())


@dataclass
class Workload:
    name: str
    levels: list
    domain: tuple = DOMAIN
    bc: tuple = EXTRAP
    limiter: int = 4
    order_trans: int = 2
    cfl: float = 0.9
    steps: int = 20
    note: str = ""
    extra: dict = field(default_factory=dict)

    def dt0(self) -> float:
        """dt = nu * min(dx, dy) / c on the coarsest level (eq:cfl);
        c = the fastest sound speed of a heterogeneous medium (extra["cmax"])."""
        d = self.levels[0].descs
        c = self.extra.get("cmax") or math.sqrt(float(d["K"][0]) / float(d["rho"][0]))
        return self.cfl * min(float(d["dx"][0]), float(d["dy"][0])) / c


def make_descs(i0, j0, mx, my, dx, dy, domain=DOMAIN, rho=1.0, K=1.0) -> np.ndarray:
    """Descriptors from integer boxes (lower-left global index i0, j0)."""
    i0 = np.asarray(i0, dtype=np.int64)
    n = i0.size
    d = np.zeros(n, dtype=PATCH_DTYPE)
    d["mx"] = mx
    d["my"] = my
    d["dx"] = dx
    d["dy"] = dy
    d["xlower"] = domain[0] + i0 * dx
    d["ylower"] = domain[2] + np.asarray(j0, dtype=np.int64) * dy
    d["mbc"] = 2
    d["rho"] = rho
    d["K"] = K
    return d


def uniform_level(npx: int, npy: int, mx: int, my: int, domain=DOMAIN,
                  rho=1.0, K=1.0) -> np.ndarray:
    """npx x npy patches of mx x my tiling the domain, row-major order."""
    nx, ny = npx * mx, npy * my
    dx = (domain[1] - domain[0]) / nx
    dy = (domain[3] - domain[2]) / ny
    jj, ii = np.meshgrid(np.arange(npy), np.arange(npx), indexing="ij")
    return make_descs(ii.ravel() * mx, jj.ravel() * my, mx, my, dx, dy, domain, rho, K)


def ring_pressure(x, y):
    r = np.sqrt(x * x + y * y)
    return np.where(np.abs(r - 0.5) <= 0.2, 1.0 + np.cos(np.pi * (r - 0.5) / 0.2), 0.0)


def ring_ic(descs: np.ndarray, out: np.ndarray | None = None, chunk: int = 4096) -> np.ndarray:
    """Ring pressure, u = v = 0, point-sampled at cell centres.
    Returns the flat [patch][3][my][mx] array (optionally into `out`)."""
    sizes = 3 * descs["mx"].astype(np.int64) * descs["my"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    if out is None:
        out = np.zeros(int(offs[-1]))
    else:
        out[...] = 0.0
    uniform = (descs["mx"] == descs["mx"][0]).all() and (descs["my"] == descs["my"][0]).all()
    if uniform:
        mx, my = int(descs["mx"][0]), int(descs["my"][0])
        view = out.reshape(len(descs), 3, my, mx)
        ii = np.arange(mx) + 0.5
        jj = np.arange(my) + 0.5
        for s in range(0, len(descs), chunk):
            d = descs[s:s + chunk]
            x = d["xlower"][:, None, None] + ii[None, None, :] * d["dx"][:, None, None]
            y = d["ylower"][:, None, None] + jj[None, :, None] * d["dy"][:, None, None]
            view[s:s + chunk, 0] = ring_pressure(x, y)
    else:
        for p, d in enumerate(descs):
            mx, my = int(d["mx"]), int(d["my"])
            x = d["xlower"] + (np.arange(mx) + 0.5) * d["dx"]
            y = d["ylower"] + (np.arange(my) + 0.5) * d["dy"]
            X, Y = np.meshgrid(x, y)
            out[offs[p]:offs[p] + mx * my] = ring_pressure(X, Y).ravel()
    return out


def random_ic(descs: np.ndarray, seed: int) -> np.ndarray:
    """i.i.d. uniform[-1, 1] for every component (numpy default_rng(seed))."""
    n = 3 * int((descs["mx"].astype(np.int64) * descs["my"]).sum())
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def level_offsets(descs: np.ndarray) -> np.ndarray:
    sizes = 3 * descs["mx"].astype(np.int64) * descs["my"]
    return np.concatenate([[0], np.cumsum(sizes)])


# ---------------------------------------------------------------------------
# Heterogeneous media (NEXT-4 variable-coefficient acoustics, P:66, P:640;
# DESIGN.md R20): per-cell (rho, K) arrays, [patch][2][my][mx] flat.
# ---------------------------------------------------------------------------

# Layers of the layered medium: (upper y bound, rho, K), bottom to top.  The
# impedance jumps by up to 4x and the sound speed by 2x between layers.
LAYERS = ((-0.5, 1.0, 1.0), (0.0, 2.0, 0.5), (0.5, 0.5, 2.0), (np.inf, 4.0, 4.0))


def layered_medium(x, y):
    """(rho, K) at points: horizontal layers LAYERS, plus a vertical inclusion
    band 0.25 <= x < 0.5 with rho = 3, K = 0.75 (so the medium varies in both
    directions)."""
    y = np.asarray(y, dtype=np.float64) + np.zeros_like(x, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64) + np.zeros_like(y)
    rho = np.empty_like(y)
    K = np.empty_like(y)
    lo = -np.inf
    for top, r, k in LAYERS:
        m = (y >= lo) & (y < top)
        rho[m] = r
        K[m] = k
        lo = top
    inc = (x >= 0.25) & (x < 0.5)
    rho[inc] = 3.0
    K[inc] = 0.75
    return rho, K


def media_field(descs: np.ndarray, fn=layered_medium, out: np.ndarray | None = None,
                chunk: int = 4096) -> np.ndarray:
    """(rho, K) = fn(x, y) at every cell centre of the level, flat
    [patch][2][my][mx]."""
    sizes = 2 * descs["mx"].astype(np.int64) * descs["my"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    if out is None:
        out = np.zeros(int(offs[-1]))
    uniform = (descs["mx"] == descs["mx"][0]).all() and (descs["my"] == descs["my"][0]).all()
    if uniform:
        mx, my = int(descs["mx"][0]), int(descs["my"][0])
        view = out.reshape(len(descs), 2, my, mx)
        ii = np.arange(mx) + 0.5
        jj = np.arange(my) + 0.5
        for s in range(0, len(descs), chunk):
            d = descs[s:s + chunk]
            x = d["xlower"][:, None, None] + ii[None, None, :] * d["dx"][:, None, None]
            y = d["ylower"][:, None, None] + jj[None, :, None] * d["dy"][:, None, None]
            view[s:s + chunk, 0], view[s:s + chunk, 1] = fn(x, y)
    else:
        for p, d in enumerate(descs):
            mx, my = int(d["mx"]), int(d["my"])
            X, Y = np.meshgrid(d["xlower"] + (np.arange(mx) + 0.5) * d["dx"],
                               d["ylower"] + (np.arange(my) + 0.5) * d["dy"])
            r, k = fn(X, Y)
            out[offs[p]:offs[p + 1]] = np.concatenate([np.ravel(r), np.ravel(k)])
    return out


def random_media(descs: np.ndarray, seed: int, lo: float = 0.5, hi: float = 2.0) -> np.ndarray:
    """i.i.d. uniform[lo, hi] rho and K per cell (numpy default_rng(seed))."""
    n = 2 * int((descs["mx"].astype(np.int64) * descs["my"]).sum())
    return np.random.default_rng(seed).uniform(lo, hi, n)


def max_sound_speed(aux: np.ndarray, descs: np.ndarray) -> float:
    """max sqrt(K / rho) over the cells of a flat media array (for dt0)."""
    m = 0.0
    off = 0
    for p in range(len(descs)):
        n = int(descs["mx"][p]) * int(descs["my"][p])
        r, k = aux[off:off + n], aux[off + n:off + 2 * n]
        m = max(m, float(np.sqrt(k / r).max()))
        off += 2 * n
    return m


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------

def c1() -> Workload:
    """configs[0]: single 64x64 patch, ring, rho=K=1, MC, 20 steps, CFL 0.9."""
    return Workload("c1_single_64", [Level(uniform_level(1, 1, 64, 64))], steps=20,
                    note="single 64x64 uniform patch, ring pulse, MC, extrapolation BCs")


def c4(patches_per_side: int = 256, mx: int = 32) -> Workload:
    """configs[3]: 256x256 patches of 32x32 (8192^2 = 67,108,864 cells)."""
    n = patches_per_side
    return Workload(f"c4_{n}x{n}_patches_{mx}x{mx}",
                    [Level(uniform_level(n, n, mx, mx))], steps=100,
                    note=f"{n*n} patches of {mx}x{mx} on one level ({n*mx}^2 cells)")


def c5(patches_per_side: int = 256, mx: int = 64) -> Workload:
    """configs[4]: 16,384^2 cells as 256x256 patches of 64x64."""
    n = patches_per_side
    return Workload(f"c5_{n*mx}sq_patches_{mx}x{mx}",
                    [Level(uniform_level(n, n, mx, mx))], steps=100,
                    note=f"{n*mx}^2 cells as {n}x{n} patches of {mx}x{mx}")


def c5_layered(patches_per_side: int = 256, mx: int = 64) -> Workload:
    """configs[4]'s layout (16,384^2 cells as 64x64 patches) in the layered
    heterogeneous medium (NEXT-4, R20); ring pulse, MC, CFL 0.9 of
    the fastest layer (c = 2)."""
    n = patches_per_side
    return Workload(f"c5vc_{n*mx}sq_patches_{mx}x{mx}_layered",
                    [Level(uniform_level(n, n, mx, mx))], steps=100,
                    note=f"{n*mx}^2 cells, layered medium (4 layers + inclusion), per-cell rho, K",
                    extra={"media": layered_medium, "cmax": 2.0})


def ragged_level(seed: int, nx: int = 40, ny: int = 36, max_w: int = 13) -> np.ndarray:
    """A level of irregular rectangles tiling an nx x ny index space (guillotine
    cuts), exercising ragged sizes, T-junction neighbours and corners."""
    rng = np.random.default_rng(seed)
    boxes = []

    def cut(i0, j0, w, h):
        if w <= max_w and h <= max_w and (w * h <= 60 or rng.random() < 0.3):
            boxes.append((i0, j0, w, h))
            return
        if (w >= h and w > 1) or h == 1:
            k = int(rng.integers(1, w))
            cut(i0, j0, k, h)
            cut(i0 + k, j0, w - k, h)
        else:
            k = int(rng.integers(1, h))
            cut(i0, j0, w, k)
            cut(i0, j0 + k, w, h - k)

    cut(0, 0, nx, ny)
    dx = (DOMAIN[1] - DOMAIN[0]) / nx
    dy = (DOMAIN[3] - DOMAIN[2]) / ny
    d = np.zeros(len(boxes), dtype=PATCH_DTYPE)
    for k, (i0, j0, w, h) in enumerate(boxes):
        d[k] = make_descs([i0], [j0], w, h, dx, dy)[0]
    return d


# ---------------------------------------------------------------------------
# Multi-level fixed hierarchies (configs[1], configs[2]); SURVEY 8(d)
# ---------------------------------------------------------------------------

def _annulus_test(x0, x1, y0, y1, w, r0=0.5):
    """(misses, fully_inside) of the box against |r - r0| <= w."""
    # exact min/max distance from the origin over the box
    dxmin = 0.0 if x0 <= 0.0 <= x1 else min(abs(x0), abs(x1))
    dymin = 0.0 if y0 <= 0.0 <= y1 else min(abs(y0), abs(y1))
    rmin = math.hypot(dxmin, dymin)
    rmax = math.hypot(max(abs(x0), abs(x1)), max(abs(y0), abs(y1)))
    misses = not (rmin <= r0 + w and rmax >= r0 - w)
    inside = rmin >= r0 - w and rmax <= r0 + w
    return misses, inside


def _cover_map(nx, ny, boxes):
    m = np.zeros((ny, nx), dtype=bool)
    for i0, j0, w, h in boxes:
        m[j0:j0 + h, i0:i0 + w] = True
    return m


def _nest_ok(box, fine_cover, coarse_cover, R):
    """Every ghost cell of `box` is covered on its own level or has its coarse
    parent's 5-point cross covered on the coarser level (clamped indices)."""
    i0, j0, w, h = box
    ny, nx = fine_cover.shape
    cny, cnx = coarse_cover.shape
    for j in range(j0 - 2, j0 + h + 2):
        for i in range(i0 - 2, i0 + w + 2):
            if i0 <= i < i0 + w and j0 <= j < j0 + h:
                continue
            I, J = min(max(i, 0), nx - 1), min(max(j, 0), ny - 1)
            if fine_cover[J, I]:
                continue
            Ic, Jc = I // R, J // R
            for a, b in ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)):
                ci, cj = min(max(Ic + a, 0), cnx - 1), min(max(Jc + b, 0), cny - 1)
                if not coarse_cover[cj, ci]:
                    return False
    return True


def _descs_from_boxes(boxes, dx, dy, domain=DOMAIN):
    return np.concatenate([make_descs([a], [b], w, h, dx, dy, domain) for a, b, w, h in boxes])


def c2() -> Workload:
    """configs[1]: 2 levels, R = 4; L1 128^2 as 2x2 patches of 64^2; L2 a
    quadtree of 16..64-wide blocks following the ring in the first quadrant."""
    l1 = uniform_level(2, 2, 64, 64)
    R = 4
    nf = 128 * R
    dxf = 2.0 / nf
    w = 0.25
    boxes = []

    def rec(i0, j0, s):
        x0, x1 = -1 + i0 * dxf, -1 + (i0 + s) * dxf
        y0, y1 = -1 + j0 * dxf, -1 + (j0 + s) * dxf
        miss, inside = _annulus_test(x0, x1, y0, y1, w)
        if miss:
            return
        if inside or s == 16:
            boxes.append((i0, j0, s, s))
            return
        h = s // 2
        for dj in (0, h):
            for di in (0, h):
                rec(i0 + di, j0 + dj, h)

    for bj in range(nf // 2, nf, 64):
        for bi in range(nf // 2, nf, 64):
            rec(bi, bj, 64)
    l2 = _descs_from_boxes(boxes, dxf, dxf)
    return Workload("c2_2level_r4", [Level(l1), Level(l2, ratio=R)], steps=200,
                    note=f"2 levels R=4: 4 + {len(boxes)} patches (16..64 wide)")


def c3(w2: float = 0.45, w3: float = 0.40) -> Workload:
    """configs[2]: 3 levels R = (2, 4); L1 200^2 as 7x7 patches (29/28 wide),
    L2 32^2 tiles near the ring, L3 aligned 32^2 tiles near the ring."""
    n1 = 200
    cuts = [0, 29, 58, 87, 115, 143, 171, 200]   # 3 x 29 + 4 x 28
    b1 = [(cuts[a], cuts[b], cuts[a + 1] - cuts[a], cuts[b + 1] - cuts[b])
          for b in range(7) for a in range(7)]
    l1 = _descs_from_boxes(b1, 2.0 / n1, 2.0 / n1)
    n2, n3 = 2 * n1, 8 * n1
    dx2, dx3 = 2.0 / n2, 2.0 / n3
    b2 = []
    for j in range(0, n2, 32):
        for i in range(0, n2, 32):
            w_, h_ = min(32, n2 - i), min(32, n2 - j)
            miss, _ = _annulus_test(-1 + i * dx2, -1 + (i + w_) * dx2, -1 + j * dx2, -1 + (j + h_) * dx2, w2)
            if not miss:
                b2.append((i, j, w_, h_))
    cover2 = _cover_map(n2, n2, b2)
    b3 = []
    for j in range(0, n3, 32):
        for i in range(0, n3, 32):
            miss, _ = _annulus_test(-1 + i * dx3, -1 + (i + 32) * dx3, -1 + j * dx3, -1 + (j + 32) * dx3, w3)
            if not miss:
                b3.append((i, j, 32, 32))
    while True:  # drop L3 tiles that violate nesting, to a fixed point
        cover3 = _cover_map(n3, n3, b3)
        keep = [b for b in b3 if _nest_ok(b, cover3, cover2, 4)]
        if len(keep) == len(b3):
            break
        b3 = keep
    l2 = _descs_from_boxes(b2, dx2, dx2)
    l3 = _descs_from_boxes(b3, dx3, dx3)
    return Workload("c3_3level_r2_r4", [Level(l1), Level(l2, ratio=2), Level(l3, ratio=4)], steps=100,
                    note=f"3 levels R=(2,4): {len(b1)} + {len(b2)} + {len(b3)} patches")


def paper(n1: int = 1000, npx: int = 4) -> Workload:
    """NEXT-4, the paper's own benchmark shape: 3 levels
    with refinement ratio 2 between levels, a 1000 x 1000 base level in
    patches of at most 260 x 260 (here 4 x 4 patches of 250^2), the van Leer
    limiter with corner transport (order_trans 2), the ring, double precision.
    Levels 2 and 3 are not fixed: they are created by flagging and
    Berger-Rigoutsos clustering (cutoff 0.7) at t = 0 and re-created every 8
    coarse steps (regrid interval 8), with a buffer of 8 coarse cells
    (R19).  Flag: pressure jump to a neighbour above
    tol_per_dx * dx of the flagged level (a gradient threshold)."""
    l1 = uniform_level(npx, npx, n1 // npx, n1 // npx)
    return Workload(f"paper_3level_r2_vanleer_{n1}", [Level(l1)], limiter=3, order_trans=2, steps=40,
                    note=f"paper-shaped dynamic AMR: base {n1}^2 ({npx}x{npx} patches), 3 levels R=2, "
                         "van Leer, regrid every 8 coarse steps (cutoff 0.7)",
                    extra={"ratios": [2, 2], "regrid_every": 8, "cutoff": 0.7, "max_dim": 130, "min_dim": 8,
                           "tol_per_dx": 2.0, "buffer_coarse_cells": 8})


def hierarchy_ic(wl: Workload) -> list:
    """Ring initial data point-sampled on every level."""
    return [ring_ic(L.descs) for L in wl.levels]
