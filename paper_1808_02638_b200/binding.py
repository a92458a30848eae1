"""Thin ctypes binding of libclaw.so (include/claw.h) -- argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
never computes anything of the method.  It fails loudly (ClawError) when the
shared library is missing: there is no CPU fallback.

PyTorch enters only as plumbing: the binding can adopt torch's current CUDA
stream (`stream=torch.cuda.current_stream().cuda_stream`) and torch.distributed
broadcasts the NCCL unique id (see `parallel_context`).
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from .workloads import PATCH_DTYPE

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CLAW_LIB") or os.path.join(_PKG, "libclaw.so")

CLAW_OK, CLAW_EINVAL, CLAW_ESTATE, CLAW_ENOMEM = 0, -1, -2, -3
CLAW_ECUDA, CLAW_ENCCL, CLAW_ENEST, CLAW_ENODEV = -4, -5, -6, -8
ERR_NAMES = {-1: "EINVAL", -2: "ESTATE", -3: "ENOMEM", -4: "ECUDA", -5: "ENCCL", -6: "ENEST", -7: "ENONFINITE",
             -8: "ENODEV"}
CLAW_ENONFINITE = -7

EXPORTS = [
    "claw_create", "claw_destroy", "claw_last_error", "claw_partition", "claw_set_level",
    "claw_fill_ghost", "claw_advance_level", "claw_advance_level_async", "claw_wait_cfl",
    "claw_read", "claw_write", "claw_read_level", "claw_write_level", "claw_read_padded",
    "claw_patch_cfl", "claw_owner", "claw_level_owned", "claw_debug_ghost_sources",
    "claw_debug_halo_counts", "claw_debug_halo_send", "claw_set_profiling", "claw_get_stats",
    "claw_reset_stats", "claw_synchronize", "claw_nccl_unique_id", "claw_version",
    "claw_level_mode", "claw_advance_hierarchy", "claw_halo_pack", "claw_halo_unpack",
    "claw_update_level", "claw_reflux_registers", "claw_level_extent", "claw_level_count",
    "claw_level_descs", "claw_flag", "claw_cluster", "claw_regrid", "claw_regrid_auto",
    "claw_pool_stats", "claw_pool_trim", "claw_comm_info", "claw_set_aux", "claw_advance_hierarchy_n",
    "claw_update_pack", "claw_update_unpack", "claw_debug_update_counts",
]
CLAW_HIER_UPDATE = 1


class ClawError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class ClawConfig(ctypes.Structure):
    _fields_ = [("xlo", ctypes.c_double), ("xhi", ctypes.c_double),
                ("ylo", ctypes.c_double), ("yhi", ctypes.c_double),
                ("bc", ctypes.c_int32 * 4), ("limiter", ctypes.c_int32),
                ("order_trans", ctypes.c_int32), ("device", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("tile_rows", ctypes.c_int32), ("path", ctypes.c_int32),
                ("exchange", ctypes.c_int32), ("reflux", ctypes.c_int32),
                ("check_finite", ctypes.c_int32), ("arena", ctypes.c_void_p),
                ("arena_bytes", ctypes.c_uint64), ("dist_level", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 3)]


class ClawStats(ctypes.Structure):
    _fields_ = [("step_launches", ctypes.c_int64), ("step_ms", ctypes.c_double),
                ("ghost_launches", ctypes.c_int64), ("ghost_ms", ctypes.c_double),
                ("cells_advanced", ctypes.c_int64), ("halo_bytes_sent", ctypes.c_int64)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libclaw.so from the package directory (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ClawError(CLAW_ENODEV, f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                     "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, dp, i32, i64, d = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, \
        ctypes.POINTER(ctypes.c_int64), ctypes.c_double
    L.claw_create.argtypes = [ctypes.POINTER(ClawConfig), ctypes.POINTER(vp)]
    L.claw_destroy.argtypes = [vp]
    L.claw_last_error.argtypes = [vp]
    L.claw_last_error.restype = ctypes.c_char_p
    L.claw_version.restype = ctypes.c_char_p
    L.claw_partition.argtypes = [i32, vp, i32, ctypes.POINTER(ctypes.c_int32)]
    L.claw_set_level.argtypes = [vp, i32, i32, vp, dp]
    L.claw_set_aux.argtypes = [vp, i32, dp]
    L.claw_fill_ghost.argtypes = [vp, i32, d]
    L.claw_advance_level.argtypes = [vp, i32, d, dp]
    L.claw_advance_level_async.argtypes = [vp, i32, d]
    L.claw_wait_cfl.argtypes = [vp, i32, dp]
    for f in ("claw_read", "claw_read_padded", "claw_patch_cfl"):
        getattr(L, f).argtypes = [vp, i32, i32, dp]
    L.claw_write.argtypes = [vp, i32, i32, dp]
    L.claw_read_level.argtypes = [vp, i32, dp]
    L.claw_write_level.argtypes = [vp, i32, dp]
    L.claw_owner.argtypes = [vp, i32, i32, ctypes.POINTER(ctypes.c_int32)]
    L.claw_level_owned.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int32), i64, i64]
    L.claw_debug_ghost_sources.argtypes = [vp, i32, i32, i64, i64]
    L.claw_debug_halo_counts.argtypes = [vp, i32, i32, i64, i64]
    L.claw_debug_halo_send.argtypes = [vp, i32, i32, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    L.claw_set_profiling.argtypes = [vp, i32]
    L.claw_get_stats.argtypes = [vp, ctypes.POINTER(ClawStats)]
    L.claw_reset_stats.argtypes = [vp]
    L.claw_synchronize.argtypes = [vp]
    L.claw_nccl_unique_id.argtypes = [vp]
    L.claw_level_mode.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int32)]
    L.claw_advance_hierarchy.argtypes = [vp, d, d, i32, dp]
    L.claw_advance_hierarchy_n.argtypes = [vp, d, d, i32, i32, dp]
    L.claw_update_level.argtypes = [vp, i32]
    L.claw_reflux_registers.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int64), vp, vp]
    L.claw_level_extent.argtypes = [vp, i32, i64, i64]
    L.claw_level_count.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int32)]
    L.claw_level_descs.argtypes = [vp, i32, vp]
    L.claw_flag.argtypes = [vp, i32, d, i32, i32, vp, i64]
    L.claw_cluster.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, d, i32, i32, vp, i32,
                               ctypes.POINTER(ctypes.c_int32)]
    L.claw_regrid.argtypes = [vp, i32, i32, vp, i32]
    L.claw_regrid_auto.argtypes = [vp, i32, d, i32, d, i32, i32, i32, ctypes.POINTER(ctypes.c_int32)]
    L.claw_pool_stats.argtypes = [i64, i64, i64]
    L.claw_comm_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                 ctypes.POINTER(ctypes.c_int32)]
    L.claw_halo_pack.argtypes = [vp, i32, i32, dp]
    L.claw_halo_unpack.argtypes = [vp, i32, i32, dp]
    L.claw_update_pack.argtypes = [vp, i32, dp]
    L.claw_update_unpack.argtypes = [vp, i32, i32, dp]
    L.claw_debug_update_counts.argtypes = [vp, i32, i32, i64, i64]
    _lib = L
    return L


def _dptr(a):
    if hasattr(a, "data_ptr"):  # torch tensor (host memory; checked by _host_f64)
        return ctypes.cast(ctypes.c_void_p(a.data_ptr()), ctypes.POINTER(ctypes.c_double))
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _host_f64(a, n: int, what: str, writable: bool = False):
    """Check that `a` is a C-contiguous float64 HOST buffer of exactly n
    elements (numpy array or CPU torch tensor, pinned or not) before its raw
    pointer crosses the C-ABI, which copies n doubles from / to it: an
    undersized, float32, strided or device buffer raises ClawError(EINVAL)
    instead of reading or writing out of bounds."""
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64:
            raise ClawError(CLAW_EINVAL, f"{what}: dtype {a.dtype}, need torch.float64")
        if a.device.type != "cpu":
            raise ClawError(CLAW_EINVAL, f"{what}: tensor on {a.device}, need a host (CPU) tensor")
        if not a.is_contiguous():
            raise ClawError(CLAW_EINVAL, f"{what}: tensor is not contiguous")
        size = a.numel()
    else:
        if not isinstance(a, np.ndarray):
            raise ClawError(CLAW_EINVAL, f"{what}: need a numpy array or torch tensor, got {type(a).__name__}")
        if a.dtype != np.float64:
            raise ClawError(CLAW_EINVAL, f"{what}: dtype {a.dtype}, need float64")
        if not a.flags["C_CONTIGUOUS"]:
            raise ClawError(CLAW_EINVAL, f"{what}: array is not C-contiguous")
        if writable and not a.flags["WRITEABLE"]:
            raise ClawError(CLAW_EINVAL, f"{what}: array is read-only")
        size = a.size
    if size != n:
        raise ClawError(CLAW_EINVAL, f"{what}: {size} elements, need {n}")
    return _dptr(a)


def _as_f64(q):
    """numpy input -> C-contiguous float64 copy if needed; torch tensors pass
    through unchanged (and are then checked, never silently converted)."""
    return q if hasattr(q, "data_ptr") else np.ascontiguousarray(q, dtype=np.float64)


def _descs(descs) -> np.ndarray:
    d = np.ascontiguousarray(np.asarray(descs).astype(PATCH_DTYPE))
    return d


def partition(descs, world: int) -> np.ndarray:
    d = _descs(descs)
    out = np.zeros(len(d), dtype=np.int32)
    rc = load().claw_partition(len(d), d.ctypes.data, world,
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if rc:
        raise ClawError(rc, "claw_partition failed")
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().claw_nccl_unique_id(buf)
    if rc:
        raise ClawError(rc, "NCCL unique id")
    return buf.raw


def cluster(flags: np.ndarray, cutoff: float, max_dim: int, min_dim: int) -> np.ndarray:
    """Berger-Rigoutsos boxes [n, 4] = (i0, j0, w, h) of a [ny, nx] flag map
    (claw_cluster; host-only)."""
    f = np.ascontiguousarray(flags, np.uint8)
    n = ctypes.c_int32()
    L = load()
    rc = L.claw_cluster(f.ctypes.data, f.shape[1], f.shape[0], float(cutoff), int(max_dim), int(min_dim),
                        None, 0, ctypes.byref(n))
    if rc:
        raise ClawError(rc, "claw_cluster: bad arguments")
    out = np.zeros((n.value, 4), np.int32)
    rc = L.claw_cluster(f.ctypes.data, f.shape[1], f.shape[0], float(cutoff), int(max_dim), int(min_dim),
                        out.ctypes.data, n.value, ctypes.byref(n))
    if rc:
        raise ClawError(rc, "claw_cluster failed")
    return out


def pool_stats() -> dict:
    h, m, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    load().claw_pool_stats(ctypes.byref(h), ctypes.byref(m), ctypes.byref(c))
    return {"hits": h.value, "misses": m.value, "cached_bytes": c.value}


def version() -> str:
    return load().claw_version().decode()


class Claw:
    """One libclaw context (one device, one rank)."""

    def __init__(self, domain=(-1.0, 1.0, -1.0, 1.0), bc=(1, 1, 1, 1), limiter=4,
                 order_trans=2, device=0, rank=0, world=1, nccl_id: bytes | None = None,
                 stream: int | None = None, tile_rows: int = 0, path: int = 0, exchange: int = 0,
                 reflux: bool = False, check_finite: bool = False, arena=None, dist_level: int = 0):
        """arena: None, or device memory the context carves every buffer from
        (claw_config.arena): a CUDA torch tensor (kept referenced by this
        object) or a (device pointer, bytes) pair.  dist_level (world > 1):
        the level partitioned across ranks (claw_config.dist_level; 0 = level
        1, K >= 2 = levels below K replicated, level K partitioned)."""
        L = load()
        self._idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        self._arena = arena
        if arena is None:
            aptr, abytes = None, 0
        elif hasattr(arena, "data_ptr"):
            if arena.device.type != "cuda":
                raise ClawError(CLAW_EINVAL, f"arena: tensor on {arena.device}, need a CUDA tensor")
            aptr, abytes = arena.data_ptr(), arena.numel() * arena.element_size()
        else:
            aptr, abytes = int(arena[0]), int(arena[1])
        cfg = ClawConfig(*[float(v) for v in domain], (ctypes.c_int32 * 4)(*bc), int(limiter),
                         int(order_trans), int(device), int(rank), int(world),
                         ctypes.cast(self._idbuf, ctypes.c_void_p) if self._idbuf else None,
                         stream, int(tile_rows), int(path), int(exchange), int(bool(reflux)),
                         int(bool(check_finite)), aptr, abytes, int(dist_level))
        self._h = ctypes.c_void_p()
        rc = L.claw_create(ctypes.byref(cfg), ctypes.byref(self._h))
        if rc:
            msg = L.claw_last_error(self._h).decode() if self._h else ""
            if self._h:
                L.claw_destroy(self._h)
                self._h = None
            raise ClawError(rc, msg or "claw_create failed")
        self.world, self.rank = world, rank
        self._descs = {}

    # -- lifecycle -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            load().claw_destroy(self._h)
            self._h = None
        self._arena = None   # the arena outlives claw_destroy (borrowed by the context)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc:
            raise ClawError(rc, load().claw_last_error(self._h).decode())

    # -- the five calls of north_star -----------------------------------
    def set_level(self, level: int, descs, q0=None):
        """q0: the owned patches' level array (3 * owned cells doubles), or None
        (zeros).  With world > 1 ownership is known only once the level is
        planned, so the level is set with zeros and q0 written after the size
        check."""
        d = _descs(descs)
        self._descs[level] = d
        if q0 is not None:
            q0 = _as_f64(q0)
        if q0 is None or self.world > 1:
            self._check(load().claw_set_level(self._h, level, len(d), d.ctypes.data, None))
            if q0 is not None:
                self.write_level(level, q0)
            return
        n = 3 * int((d["mx"].astype(np.int64) * d["my"].astype(np.int64)).sum())
        self._check(load().claw_set_level(self._h, level, len(d), d.ctypes.data,
                                          _host_f64(q0, n, "set_level q0")))

    def set_aux(self, level: int, aux):
        """Per-cell media of the level (claw_set_aux): aux = [patch][2][my][mx]
        (rho, K) for ALL patches, flat float64 (2 * level cells doubles)."""
        d = self._descs[level]
        n = 2 * int((d["mx"].astype(np.int64) * d["my"].astype(np.int64)).sum())
        self._check(load().claw_set_aux(self._h, level, _host_f64(_as_f64(aux), n, "set_aux aux")))

    def fill_ghost(self, level: int, t: float = 0.0):
        self._check(load().claw_fill_ghost(self._h, level, float(t)))

    def advance_level(self, level: int, dt: float) -> float:
        c = ctypes.c_double()
        self._check(load().claw_advance_level(self._h, level, float(dt), ctypes.byref(c)))
        return c.value

    def advance_level_async(self, level: int, dt: float):
        self._check(load().claw_advance_level_async(self._h, level, float(dt)))

    def wait_cfl(self, level: int) -> float:
        c = ctypes.c_double()
        self._check(load().claw_wait_cfl(self._h, level, ctypes.byref(c)))
        return c.value

    def read(self, level: int, patch: int) -> np.ndarray:
        d = self._descs[level][patch]
        out = np.empty((3, int(d["my"]), int(d["mx"])))
        self._check(load().claw_read(self._h, level, patch, _host_f64(out, out.size, "read", True)))
        return out

    def write(self, level: int, patch: int, q):
        d = self._descs[level][patch]
        q = _as_f64(q)
        self._check(load().claw_write(self._h, level, patch,
                                      _host_f64(q, 3 * int(d["mx"]) * int(d["my"]), "write")))

    # -- level-wide I/O --------------------------------------------------
    def owned_patches(self, level: int) -> np.ndarray:
        return np.array([p for p in range(len(self._descs[level])) if self.owner(level, p) == self.rank],
                        dtype=np.int64)

    def level_size(self, level: int) -> int:
        n, cells, b = self.level_owned(level)
        return 3 * cells

    def read_level(self, level: int, out=None):
        n = self.level_size(level)
        if out is None:
            out = np.empty(n)
        self._check(load().claw_read_level(self._h, level, _host_f64(out, n, "read_level out", True)))
        return out

    def write_level(self, level: int, q):
        q = _as_f64(q)
        self._check(load().claw_write_level(self._h, level, _host_f64(q, self.level_size(level), "write_level")))

    def read_padded(self, level: int, patch: int) -> np.ndarray:
        d = self._descs[level][patch]
        out = np.empty((3, int(d["my"]) + 4, int(d["mx"]) + 4))
        self._check(load().claw_read_padded(self._h, level, patch, _host_f64(out, out.size, "read_padded", True)))
        return out

    def patch_cfl(self, level: int, patch: int) -> float:
        c = ctypes.c_double()
        self._check(load().claw_patch_cfl(self._h, level, patch, ctypes.byref(c)))
        return c.value

    def owner(self, level: int, patch: int) -> int:
        r = ctypes.c_int32()
        self._check(load().claw_owner(self._h, level, patch, ctypes.byref(r)))
        return r.value

    def level_mode(self, level: int) -> str:
        m = ctypes.c_int32()
        self._check(load().claw_level_mode(self._h, level, ctypes.byref(m)))
        return {1: "grid", 2: "sparse"}.get(m.value, "generic")

    def advance_hierarchy(self, t: float, dt: float, update: bool = False) -> float:
        """One coarse step of every level with subcycling (and, with update,
        fine->coarse averaging after each fine cycle), natively."""
        c = ctypes.c_double()
        self._check(load().claw_advance_hierarchy(self._h, float(t), float(dt),
                                                  CLAW_HIER_UPDATE if update else 0, ctypes.byref(c)))
        return c.value

    def advance_hierarchy_n(self, t: float, dt: float, nsteps: int, update: bool = False) -> np.ndarray:
        """nsteps coarse steps at fixed dt with one host synchronisation;
        returns the per-step max Courant numbers (claw_advance_hierarchy_n)."""
        out = np.zeros(int(nsteps))
        self._check(load().claw_advance_hierarchy_n(self._h, float(t), float(dt), int(nsteps),
                                                    CLAW_HIER_UPDATE if update else 0, _dptr(out)))
        return out

    def update_level(self, level: int):
        """Average `level` onto `level - 1` where fully covered;
        with reflux on, then apply the conservation fix."""
        self._check(load().claw_update_level(self._h, level))

    def reflux_registers(self, level: int, values: bool = True):
        """(edges [n, 8] int32, acc [n, 3] or None): conservation-fix
        registers of fine level `level` (see claw_reflux_registers)."""
        n = ctypes.c_int64()
        self._check(load().claw_reflux_registers(self._h, level, ctypes.byref(n), None, None))
        e = np.zeros((n.value, 8), np.int32)
        a = np.zeros((n.value, 3)) if values else None
        self._check(load().claw_reflux_registers(self._h, level, ctypes.byref(n), e.ctypes.data,
                                                 a.ctypes.data if values else None))
        return e, a

    def level_owned(self, level: int):
        n, c, b = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        self._check(load().claw_level_owned(self._h, level, ctypes.byref(n), ctypes.byref(c), ctypes.byref(b)))
        return n.value, c.value, b.value

    # -- regridding -----------------------------------------
    def level_extent(self, level: int):
        nx, ny = ctypes.c_int64(), ctypes.c_int64()
        self._check(load().claw_level_extent(self._h, level, ctypes.byref(nx), ctypes.byref(ny)))
        return nx.value, ny.value

    def descs(self, level: int) -> np.ndarray:
        """The level's current patch descriptors (after regridding too)."""
        n = ctypes.c_int32()
        self._check(load().claw_level_count(self._h, level, ctypes.byref(n)))
        d = np.zeros(n.value, dtype=PATCH_DTYPE)
        if n.value:
            self._check(load().claw_level_descs(self._h, level, d.ctypes.data))
        return d

    def flag(self, level: int, tol: float, buffer: int = 0, clip: int = 0) -> np.ndarray:
        """Device flag map [ny, nx] (uint8) of `level` (claw_flag)."""
        nx, ny = self.level_extent(level)
        f = np.zeros((ny, nx), np.uint8)
        cnt = ctypes.c_int64()
        self._check(load().claw_flag(self._h, level, float(tol), int(buffer), int(clip), f.ctypes.data,
                                     ctypes.byref(cnt)))
        assert int(f.sum()) == cnt.value
        return f

    def regrid(self, level: int, boxes, R: int):
        b = np.ascontiguousarray(np.asarray(boxes, dtype=np.int32).reshape(-1, 4))
        self._check(load().claw_regrid(self._h, level, len(b), b.ctypes.data if len(b) else None, int(R)))
        self._refresh_descs(level + 1)

    def regrid_auto(self, level: int, tol: float, buffer: int, cutoff: float, max_dim: int, min_dim: int,
                    R: int) -> int:
        n = ctypes.c_int32()
        self._check(load().claw_regrid_auto(self._h, level, float(tol), int(buffer), float(cutoff),
                                            int(max_dim), int(min_dim), int(R), ctypes.byref(n)))
        self._refresh_descs(level + 1)
        return n.value

    def _refresh_descs(self, level: int):
        for l in list(self._descs):
            if l >= level:
                del self._descs[l]
        d = self.descs(level)
        if len(d):
            self._descs[level] = d

    # -- introspection ---------------------------------------------------
    def debug_ghost_sources(self, level: int, patch: int):
        d = self._descs[level][patch]
        n = (int(d["mx"]) + 4) * (int(d["my"]) + 4)
        a = np.zeros(n, dtype=np.int64)
        b = np.zeros(n, dtype=np.int64)
        self._check(load().claw_debug_ghost_sources(
            self._h, level, patch, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            b.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        shape = (int(d["my"]) + 4, int(d["mx"]) + 4)
        return a.reshape(shape), b.reshape(shape)

    def halo_pack(self, level: int, peer: int) -> np.ndarray:
        ns, _ = self.debug_halo_counts(level, peer)
        out = np.empty(3 * ns)
        if ns:
            self._check(load().claw_halo_pack(self._h, level, peer, _host_f64(out, 3 * ns, "halo_pack", True)))
        return out

    def halo_unpack(self, level: int, peer: int, buf: np.ndarray):
        buf = np.ascontiguousarray(buf, dtype=np.float64)
        _, nr = self.debug_halo_counts(level, peer)
        if buf.size or nr:
            self._check(load().claw_halo_unpack(self._h, level, peer, _host_f64(buf, 3 * nr, "halo_unpack")))

    def debug_halo_counts(self, level: int, peer: int):
        s, r = ctypes.c_int64(), ctypes.c_int64()
        self._check(load().claw_debug_halo_counts(self._h, level, peer, ctypes.byref(s), ctypes.byref(r)))
        return s.value, r.value

    def update_pack(self, level: int) -> np.ndarray:
        """The level-(level-1) cells this rank's patches of the partitioned
        level `level` averaged in the last claw_update_level ([3][n];
        claw_update_pack, exchange = 1)."""
        ns, _ = self.debug_update_counts(level, self.rank)
        out = np.empty(3 * ns)
        if ns:
            self._check(load().claw_update_pack(self._h, level, _host_f64(out, 3 * ns, "update_pack", True)))
        return out

    def update_unpack(self, level: int, peer: int, buf: np.ndarray):
        """Write rank `peer`'s averaged cells (its update_pack) into this
        rank's replica of level `level` - 1 (claw_update_unpack)."""
        buf = np.ascontiguousarray(buf, dtype=np.float64)
        _, nr = self.debug_update_counts(level, peer)
        if buf.size or nr:
            self._check(load().claw_update_unpack(self._h, level, peer, _host_f64(buf, 3 * nr, "update_unpack")))

    def debug_update_counts(self, level: int, peer: int):
        """(cells this rank sends, cells rank `peer` sends) of the update
        exchange of the partitioned level `level`."""
        s, r = ctypes.c_int64(), ctypes.c_int64()
        self._check(load().claw_debug_update_counts(self._h, level, peer, ctypes.byref(s), ctypes.byref(r)))
        return s.value, r.value

    def debug_halo_send(self, level: int, peer: int, k: int):
        p, i, j = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self._check(load().claw_debug_halo_send(self._h, level, peer, k, ctypes.byref(p),
                                                ctypes.byref(i), ctypes.byref(j)))
        return p.value, i.value, j.value

    def comm_info(self):
        """(nranks, rank, cuda_device) of the context's NCCL communicator as
        NCCL reports it, or None when there is none (world 1 / external)."""
        n, r, d = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        rc = load().claw_comm_info(self._h, ctypes.byref(n), ctypes.byref(r), ctypes.byref(d))
        if rc == CLAW_ESTATE:
            return None
        self._check(rc)
        return n.value, r.value, d.value

    def set_profiling(self, on: bool = True):
        self._check(load().claw_set_profiling(self._h, int(on)))

    def stats(self) -> dict:
        s = ClawStats()
        self._check(load().claw_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in ClawStats._fields_}

    def reset_stats(self):
        self._check(load().claw_reset_stats(self._h))

    def synchronize(self):
        self._check(load().claw_synchronize(self._h))


def berger_oliger(claw: Claw, level: int, t: float, dt: float, ratios: dict, nlevels: int) -> float:
    """Advance `level` from t by dt, then recursively the finer level R_L times
    with dt / R_L, coarse level first.  ratios[L] = R_L between
    levels L and L+1.  Returns the max CFL number seen."""
    claw.fill_ghost(level, t)
    cfl = claw.advance_level(level, dt)
    if level < nlevels:
        R = ratios[level]
        dtf = dt / R
        for k in range(R):
            cfl = max(cfl, berger_oliger(claw, level + 1, t + k * dtf, dtf, ratios, nlevels))
    return cfl
