"""CPU oracle for the AMR-level advance of arXiv 1808.02638 (2D acoustics).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It wraps ``claw_oracle.c`` (plain C99, fp64, no FMA contraction) via
ctypes and shares no code with the CUDA path in ``paper_1808_02638_b200``.

Every function documents the PAPER.md passage it follows (P:a-b = line range
of /root/reference/PAPER.md).  Pins: tests/test_oracle_pins.py,
tests/test_oracle_brute.py, tests/test_oracle_ghost.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "claw_oracle.c")
_HDR = os.path.join(_HERE, "claw_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

# Mirror of oracle_patch_desc (C layout, natural alignment).
ORACLE_PATCH_DTYPE = np.dtype(
    [("mx", "<i4"), ("my", "<i4"), ("dx", "<f8"), ("dy", "<f8"),
     ("xlower", "<f8"), ("ylower", "<f8"), ("mbc", "<i4"),
     ("rho", "<f8"), ("K", "<f8")], align=True)
assert ORACLE_PATCH_DTYPE.itemsize == 64


class _Config(ctypes.Structure):
    _fields_ = [("xlo", ctypes.c_double), ("xhi", ctypes.c_double),
                ("ylo", ctypes.c_double), ("yhi", ctypes.c_double),
                ("bc", ctypes.c_int32 * 4), ("limiter", ctypes.c_int32),
                ("order_trans", ctypes.c_int32), ("nthreads", ctypes.c_int32)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -std=c11 -ffp-contract=off -fopenmp)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _HDR))
    if force or stale:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
               "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        vp = ctypes.c_void_p
        L.oracle_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(vp)]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_last_error.argtypes = [vp]
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_set_level.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, dp]
        L.oracle_fill_ghost.argtypes = [vp, ctypes.c_int, ctypes.c_double]
        L.oracle_advance_level.argtypes = [vp, ctypes.c_int, ctypes.c_double, dp]
        for f in ("oracle_read", "oracle_read_padded"):
            getattr(L, f).argtypes = [vp, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_write.argtypes = [vp, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_patch_cfl.argtypes = [vp, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_level_time.argtypes = [vp, ctypes.c_int, dp, dp]
        L.oracle_update_level.argtypes = [vp, ctypes.c_int]
        L.oracle_set_reflux.argtypes = [vp, ctypes.c_int]
        L.oracle_flag.argtypes = [vp, ctypes.c_int, ctypes.c_double, vp]
        L.oracle_buffer_flags.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp]
        L.oracle_buffer_flags.restype = None
        L.oracle_cluster.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_int, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.oracle_regrid.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int]
        L.oracle_level_count.argtypes = [vp, ctypes.c_int]
        L.oracle_level_desc.argtypes = [vp, ctypes.c_int, vp]
        L.oracle_reflux_count.argtypes = [vp, ctypes.c_int]
        L.oracle_reflux_read.argtypes = [vp, ctypes.c_int, vp, vp]
        L.oracle_step_patch.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int, dp, dp]
        L.oracle_rpn2.argtypes = [ctypes.c_int, dp, dp, ctypes.c_double, ctypes.c_double,
                                  dp, dp, dp, dp]
        L.oracle_rpt2.argtypes = [ctypes.c_int, dp, ctypes.c_double, ctypes.c_double, dp, dp]
        L.oracle_set_aux.argtypes = [vp, ctypes.c_int, dp]
        L.oracle_rpn2_vc.argtypes = [ctypes.c_int, dp, dp] + [ctypes.c_double] * 4 + [dp] * 4
        L.oracle_rpn2_vc.restype = None
        L.oracle_rpt2_vc.argtypes = [ctypes.c_int, dp] + [ctypes.c_double] * 6 + [dp, dp]
        L.oracle_rpt2_vc.restype = None
        L.oracle_step_patch_vc.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                           ctypes.c_int, dp, dp]
        L.oracle_philim.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oracle_philim.restype = ctypes.c_double
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    pass


class Oracle:
    """One AMR hierarchy on the CPU.  Mirrors the C-ABI call shapes
    (create / set_level / fill_ghost / advance_level / read)."""

    def __init__(self, domain=(-1.0, 1.0, -1.0, 1.0), bc=(1, 1, 1, 1), limiter=4,
                 order_trans=2, nthreads=0, reflux=False):
        cfg = _Config(*[float(v) for v in domain], (ctypes.c_int32 * 4)(*bc),
                      int(limiter), int(order_trans), int(nthreads))
        self._h = ctypes.c_void_p()
        rc = lib().oracle_create(ctypes.byref(cfg), ctypes.byref(self._h))
        if rc != 0:
            raise OracleError(f"oracle_create failed ({rc})")
        self._descs = {}
        self._dom = tuple(float(v) for v in domain)
        if reflux:
            self._check(lib().oracle_set_reflux(self._h, 1))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_destroy(self._h)
            self._h = None

    def _check(self, rc):
        if rc != 0:
            raise OracleError(f"rc={rc}: {lib().oracle_last_error(self._h).decode()}")

    def set_level(self, level: int, descs: np.ndarray, q0: np.ndarray | None = None):
        d = np.ascontiguousarray(descs.astype(ORACLE_PATCH_DTYPE))
        q = None if q0 is None else np.ascontiguousarray(q0, dtype=np.float64)
        if q is not None:
            assert q.size == 3 * int((d["mx"].astype(np.int64) * d["my"]).sum())
        self._descs[level] = d
        self._check(lib().oracle_set_level(self._h, level, len(d), d.ctypes.data,
                                           None if q is None else _dp(q)))

    def set_aux(self, level: int, aux: np.ndarray):
        """Variable media of the single level 1 (R20): aux =
        [patch][2][my][mx] (rho, K) flat, every value finite and > 0."""
        a = np.ascontiguousarray(aux, dtype=np.float64)
        d = self._descs[level]
        assert a.size == 2 * int((d["mx"].astype(np.int64) * d["my"]).sum())
        self._check(lib().oracle_set_aux(self._h, level, _dp(a)))

    def fill_ghost(self, level: int, t: float = 0.0):
        self._check(lib().oracle_fill_ghost(self._h, level, float(t)))

    def advance_level(self, level: int, dt: float) -> float:
        c = ctypes.c_double()
        self._check(lib().oracle_advance_level(self._h, level, float(dt), ctypes.byref(c)))
        return c.value

    def update_level(self, level: int):
        """Average `level` onto `level - 1` where fully covered."""
        self._check(lib().oracle_update_level(self._h, level))

    def reflux_registers(self, level: int):
        """(edges [n, 8] int32, acc [n, 3]) of level `level`'s conservation-fix
        registers (see oracle_reflux_read)."""
        n = lib().oracle_reflux_count(self._h, level)
        if n < 0:
            raise OracleError("bad level")
        e = np.zeros((n, 8), np.int32)
        a = np.zeros((n, 3))
        self._check(lib().oracle_reflux_read(self._h, level, e.ctypes.data, a.ctypes.data))
        return e, a

    def level_shape(self, level: int):
        d = self.descs(level)
        dx = float(d["dx"][0])
        return (int(round((self._dom[1] - self._dom[0]) / dx)),
                int(round((self._dom[3] - self._dom[2]) / float(d["dy"][0]))))

    def descs(self, level: int) -> np.ndarray:
        n = lib().oracle_level_count(self._h, level)
        d = np.zeros(max(n, 0), ORACLE_PATCH_DTYPE)
        if n > 0:
            self._check(lib().oracle_level_desc(self._h, level, d.ctypes.data))
        return d

    def flag(self, level: int, tol: float) -> np.ndarray:
        """Undivided-gradient flags of `level` over its index space [ny, nx] (uint8)."""
        nx, ny = self.level_shape(level)
        f = np.zeros((ny, nx), np.uint8)
        self._check(lib().oracle_flag(self._h, level, float(tol), f.ctypes.data))
        return f

    def regrid(self, level: int, boxes, R: int):
        """Replace level+1 by `boxes` ([n, 4] i0, j0, w, h in level index space) x R."""
        b = np.ascontiguousarray(np.asarray(boxes, np.int32).reshape(-1, 4))
        self._check(lib().oracle_regrid(self._h, level, len(b), b.ctypes.data, int(R)))
        self._descs[level + 1] = self.descs(level + 1)
        for l in list(self._descs):
            if l > level + 1:
                del self._descs[l]

    def read(self, level: int, patch: int) -> np.ndarray:
        d = self._descs[level][patch]
        out = np.empty((3, int(d["my"]), int(d["mx"])))
        self._check(lib().oracle_read(self._h, level, patch, _dp(out)))
        return out

    def read_level(self, level: int) -> np.ndarray:
        """All patches concatenated as [patch][3][my][mx] (flat)."""
        return np.concatenate([self.read(level, p).ravel()
                               for p in range(len(self._descs[level]))])

    def write(self, level: int, patch: int, q: np.ndarray):
        q = np.ascontiguousarray(q, dtype=np.float64)
        self._check(lib().oracle_write(self._h, level, patch, _dp(q)))

    def read_padded(self, level: int, patch: int) -> np.ndarray:
        d = self._descs[level][patch]
        out = np.empty((3, int(d["my"]) + 4, int(d["mx"]) + 4))
        self._check(lib().oracle_read_padded(self._h, level, patch, _dp(out)))
        return out

    def patch_cfl(self, level: int, patch: int) -> float:
        c = ctypes.c_double()
        self._check(lib().oracle_patch_cfl(self._h, level, patch, ctypes.byref(c)))
        return c.value

    def level_time(self, level: int):
        a, b = ctypes.c_double(), ctypes.c_double()
        self._check(lib().oracle_level_time(self._h, level, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


def step_patch(qpad: np.ndarray, dx, dy, dt, rho=1.0, K=1.0, limiter=4, order_trans=2):
    """One step of eq. (W) on a padded [3][my+4][mx+4] patch; returns
    (qout_pad, cfl)."""
    qpad = np.ascontiguousarray(qpad, dtype=np.float64)
    _, py, px = qpad.shape
    out = np.empty_like(qpad)
    c = ctypes.c_double()
    rc = lib().oracle_step_patch(px - 4, py - 4, _dp(qpad), dx, dy, dt, rho, K,
                                 limiter, order_trans, _dp(out), ctypes.byref(c))
    if rc != 0:
        raise OracleError("oracle_step_patch failed")
    return out, c.value


def step_patch_vc(qpad: np.ndarray, auxpad: np.ndarray, dx, dy, dt, limiter=4, order_trans=2):
    """One step with per-cell media: auxpad = [2][my+4][mx+4] (rho, K) with
    its ghost frame set; returns (qout_pad, cfl)."""
    qpad = np.ascontiguousarray(qpad, dtype=np.float64)
    auxpad = np.ascontiguousarray(auxpad, dtype=np.float64)
    _, py, px = qpad.shape
    assert auxpad.shape == (2, py, px)
    out = np.empty_like(qpad)
    c = ctypes.c_double()
    rc = lib().oracle_step_patch_vc(px - 4, py - 4, _dp(qpad), _dp(auxpad), dx, dy, dt,
                                    limiter, order_trans, _dp(out), ctypes.byref(c))
    if rc != 0:
        raise OracleError("oracle_step_patch_vc failed")
    return out, c.value


def rpn2_vc(ixy, ql, qr, rhol, Kl, rhor, Kr):
    ql = np.ascontiguousarray(ql, dtype=np.float64)
    qr = np.ascontiguousarray(qr, dtype=np.float64)
    wave = np.empty((2, 3)); s = np.empty(2); am = np.empty(3); ap = np.empty(3)
    lib().oracle_rpn2_vc(ixy, _dp(ql), _dp(qr), rhol, Kl, rhor, Kr, _dp(wave), _dp(s), _dp(am), _dp(ap))
    return wave, s, am, ap


def rpt2_vc(ixy, asdq, rho_m, K_m, rho, K, rho_p, K_p):
    a = np.ascontiguousarray(asdq, dtype=np.float64)
    bm = np.empty(3); bp = np.empty(3)
    lib().oracle_rpt2_vc(ixy, _dp(a), rho_m, K_m, rho, K, rho_p, K_p, _dp(bm), _dp(bp))
    return bm, bp


def rpn2(ixy, ql, qr, rho=1.0, K=1.0):
    ql = np.ascontiguousarray(ql, dtype=np.float64)
    qr = np.ascontiguousarray(qr, dtype=np.float64)
    wave = np.empty((2, 3)); s = np.empty(2); am = np.empty(3); ap = np.empty(3)
    lib().oracle_rpn2(ixy, _dp(ql), _dp(qr), rho, K, _dp(wave), _dp(s), _dp(am), _dp(ap))
    return wave, s, am, ap


def rpt2(ixy, asdq, rho=1.0, K=1.0):
    a = np.ascontiguousarray(asdq, dtype=np.float64)
    bm = np.empty(3); bp = np.empty(3)
    lib().oracle_rpt2(ixy, _dp(a), rho, K, _dp(bm), _dp(bp))
    return bm, bp


def philim(limiter: int, r: float) -> float:
    return lib().oracle_philim(limiter, float(r))


def buffer_flags(flags: np.ndarray, b: int, mask: np.ndarray | None = None) -> np.ndarray:
    """Chebyshev dilation of a [ny, nx] uint8 flag map by b cells."""
    f = np.ascontiguousarray(flags, np.uint8)
    out = np.zeros_like(f)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    lib().oracle_buffer_flags(f.ctypes.data, f.shape[1], f.shape[0], int(b),
                              None if m is None else m.ctypes.data, out.ctypes.data)
    return out


def cluster(flags: np.ndarray, cutoff: float, max_dim: int, min_dim: int) -> np.ndarray:
    """Berger-Rigoutsos boxes [n, 4] = (i0, j0, w, h) of a [ny, nx] flag map."""
    f = np.ascontiguousarray(flags, np.uint8)
    n = ctypes.c_int()
    rc = lib().oracle_cluster(f.ctypes.data, f.shape[1], f.shape[0], float(cutoff), int(max_dim),
                              int(min_dim), None, 0, ctypes.byref(n))
    if rc not in (0, -3):
        raise OracleError(f"oracle_cluster rc={rc}")
    b = np.zeros((max(n.value, 1), 4), np.int32)
    rc = lib().oracle_cluster(f.ctypes.data, f.shape[1], f.shape[0], float(cutoff), int(max_dim),
                              int(min_dim), b.ctypes.data, len(b), ctypes.byref(n))
    if rc != 0:
        raise OracleError(f"oracle_cluster rc={rc}")
    return b[:n.value]


# ---------------------------------------------------------------------------
# Regridding driver (R18/R19): the oracle's composition of the
# pinned pieces above -- plain numpy loops over the definitions, no sharing
# with libclaw's claw_regrid_auto.
# ---------------------------------------------------------------------------
def cover_map(descs: np.ndarray, domain, nx: int, ny: int) -> np.ndarray:
    """[ny, nx] uint8: 1 on the cells of the level's patches."""
    m = np.zeros((ny, nx), np.uint8)
    for e in descs:
        i0 = int(round((e["xlower"] - domain[0]) / e["dx"]))
        j0 = int(round((e["ylower"] - domain[2]) / e["dy"]))
        m[j0:j0 + e["my"], i0:i0 + e["mx"]] = 1
    return m


def nest_mask(on: np.ndarray) -> np.ndarray:
    """Nesting mask (R18): cells of the level whose in-domain neighbours
    within Chebyshev distance 2 all belong to the level."""
    ny, nx = on.shape
    off = np.pad(1 - on.astype(np.uint8), 2, constant_values=0)   # out of domain: never a veto
    bad = np.zeros((ny, nx), np.uint8)
    for dj in range(5):
        for di in range(5):
            bad |= off[dj:dj + ny, di:di + nx]
    return (on.astype(np.uint8) & (1 - bad)).astype(np.uint8)


def split_boxes(boxes, M: np.ndarray, f: np.ndarray) -> np.ndarray:
    """R18 nesting split: inside each box, the maximal runs of M in every row;
    a run identical to one of the row below extends that rectangle; pieces
    without a flag are dropped; pieces of a box ordered by (y0, x0)."""
    out = []
    for x0, y0, w, h in np.asarray(boxes, np.int64).reshape(-1, 4).tolist():
        x1, y1 = x0 + w, y0 + h
        opened, done = {}, []
        for J in range(y0, y1 + 1):
            runs = []
            if J < y1:
                I = x0
                while I < x1:
                    if not M[J, I]:
                        I += 1
                        continue
                    e = I
                    while e < x1 and M[J, e]:
                        e += 1
                    runs.append((I, e))
                    I = e
            for key in sorted(opened):
                if key not in runs:
                    done.append((key[0], opened.pop(key), key[1], J))
            for r in runs:
                opened.setdefault(r, J)
        done.sort(key=lambda r: (r[1], r[0]))
        out += [(a, y, e - a, J - y) for a, y, e, J in done if f[y:J, a:e].any()]
    return np.array(out, np.int32).reshape(-1, 4)


def regrid_auto(o: "Oracle", level: int, tol: float, buffer: int, cutoff: float, max_dim: int,
                min_dim: int, R: int) -> int:
    """flag -> buffer (clipped to the nesting mask) -> cluster -> nesting
    split -> regrid, on the oracle; the ghost frames of `level` must be
    filled.  Returns the number of new patches."""
    nx, ny = o.level_shape(level)
    M = nest_mask(cover_map(o.descs(level), o._dom, nx, ny))
    f = buffer_flags(o.flag(level, tol), buffer, M)
    pieces = split_boxes(cluster(f, cutoff, max_dim, min_dim), M, f) if f.any() else np.zeros((0, 4), np.int32)
    o.regrid(level, pieces, R)
    return len(pieces)
