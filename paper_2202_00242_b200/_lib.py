"""ctypes binding of libvgicp.so (include/vgicp.h).

The shared library is the only compute path: importing a product module never falls back
to NumPy.  If the library is missing or no B200 is visible, the first call raises
:class:`VgicpUnavailable` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint8, c_void_p, c_char_p
from pathlib import Path

import numpy as np

from . import errors

LIB_PATH = Path(os.environ.get("VGICP_LIB") or
                Path(__file__).resolve().parent / "lib" / "libvgicp.so")  # VGICP_LIB: A/B builds

VG_OK = 0
VG_ERR_INVALID = 1
VG_ERR_CUDA = 2
VG_ERR_DEGENERATE = 3
VG_ERR_TOO_SPARSE = 4
VG_ERR_NOMEM = 5

MODE_LINEARIZE = 0
MODE_COST = 1
MODE_COMPACT = 2
MODE_INLIERS = 3
RECORD_SIZE = {MODE_LINEARIZE: 92, MODE_COST: 2, MODE_COMPACT: 29, MODE_INLIERS: 2}
REC_LINEARIZE_F32 = 94  # 4-byte words: fp32 blocks (90), fp64 cost (2 words), int32 inliers, pad
FACTOR_UNARY = 1


class VgicpUnavailable(RuntimeError):
    """libvgicp.so is not built or cannot run here (it needs an sm_100 GPU)."""


class vg_factor_spec(ctypes.Structure):
    _fields_ = [("source", c_void_p), ("target", c_void_p), ("flags", c_int32),
                ("min_inliers", c_int32), ("var_source", c_int32), ("var_target", c_int32)]


_P_D = POINTER(c_double)
_P_I64 = POINTER(c_int64)
_P_U8 = POINTER(c_uint8)
_PP = POINTER(c_void_p)

_SIGNATURES = {
    "vg_abi_version": ([], c_int),
    "vg_last_error": ([], c_char_p),
    "vg_ctx_create": ([c_int, _PP], c_int),
    "vg_ctx_destroy": ([c_void_p], c_int),
    "vg_ctx_set_stream": ([c_void_p, c_void_p], c_int),
    "vg_ctx_synchronize": ([c_void_p], c_int),
    "vg_ctx_launch_count": ([c_void_p, _P_I64], c_int),
    "vg_pack_voxel_keys": ([c_void_p, _P_D, c_int64, c_double, _P_I64], c_int),
    "vg_deskew_points": ([c_void_p, _P_D, _P_D, c_int64, _P_D, _P_D, _P_D, c_int64, _P_D],
                         c_int),
    "vg_voxel_downsample": ([c_void_p, _P_D, _P_D, c_int64, c_double, c_double, _P_D, _P_D,
                             _P_I64], c_int),
    "vg_cloud_create": ([c_void_p, _P_D, _P_D, c_int64, _PP], c_int),
    "vg_cloud_info": ([c_void_p, _P_I64, POINTER(c_int32), POINTER(c_int32)], c_int),
    "vg_cloud_destroy": ([c_void_p], c_int),
    "vg_map_build": ([c_void_p, c_void_p, c_double, _PP], c_int),
    "vg_map_from_arrays": ([c_void_p, c_double, _P_I64, _P_D, _P_D, _P_I64, c_int64, _PP], c_int),
    "vg_map_info": ([c_void_p, _P_I64, _P_D, _P_I64], c_int),
    "vg_map_export": ([c_void_p, c_void_p, _P_I64, _P_D, _P_D, _P_I64], c_int),
    "vg_map_destroy": ([c_void_p], c_int),
    "vg_map_lookup": ([c_void_p, c_void_p, _P_D, c_int64, _P_I64, _P_I64], c_int),
    "vg_cloud_lookup": ([c_void_p, c_void_p, c_void_p, _P_D, _P_I64, _P_I64], c_int),
    "vg_match_terms": ([c_void_p, c_void_p, c_void_p, _P_D, _P_I64, _P_D, _P_D, _P_D, _P_D,
                        _P_D, _P_I64], c_int),
    "vg_linearize_terms": ([c_void_p, _P_D, _P_D, _P_D, _P_D, c_int64, c_double, c_int64,
                            c_int32, c_int32, _P_D], c_int),
    "vg_batch_create": ([c_void_p, POINTER(vg_factor_spec), c_int64, _PP], c_int),
    "vg_batch_info": ([c_void_p, _P_I64, _P_I64, _P_I64], c_int),
    "vg_batch_destroy": ([c_void_p], c_int),
    "vg_batch_linearize": ([c_void_p, _P_D, c_int, _P_D], c_int),
    "vg_batch_linearize_poses": ([c_void_p, _P_D, c_int64, c_int, _P_D], c_int),
    "vg_batch_linearize_poses_device": ([c_void_p, c_void_p, c_int64, c_int, c_void_p], c_int),
    "vg_batch_lookup_rows": ([c_void_p, _P_D, c_int64, _P_I64, _P_I64], c_int),
    "vg_batch_linearize_f32": ([c_void_p, _P_D, c_int, c_void_p], c_int),
    "vg_batch_linearize_poses_f32": ([c_void_p, _P_D, c_int64, c_int, c_void_p], c_int),
    "vg_host_alloc": ([ctypes.c_size_t, _PP], c_int),
    "vg_host_free": ([c_void_p], c_int),
    "vg_batch_compose_device": ([c_void_p, c_void_p, c_int64], c_int),
    "vg_batch_accumulate_device": ([c_void_p, c_int], c_int),
    "vg_batch_finalize_device": ([c_void_p, c_int, c_void_p], c_int),
    "vg_batch_graph_capture": ([c_void_p, c_void_p, c_int64, c_int, c_void_p], c_int),
    "vg_batch_graph_launch": ([c_void_p], c_int),
    "vg_batch_graph_capture_assemble": ([c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int32],
                                        c_int),
    "vg_batch_assemble_setup": ([c_void_p, c_int64, _P_I64, _P_I64], c_int),
    "vg_batch_assemble_setup_pairs": ([c_void_p, c_int64, POINTER(c_int32), c_int64, _P_I64],
                                      c_int),
    "vg_batch_assemble_setup_mapped": ([c_void_p, c_int64, POINTER(c_int32), c_int64,
                                        POINTER(c_int32), c_int64, _P_I64], c_int),
    "vg_batch_assemble_pairs": ([c_void_p, POINTER(c_int32)], c_int),
    "vg_batch_assemble_poses": ([c_void_p, _P_D, c_int64, _P_D], c_int),
    "vg_batch_assemble_poses_device": ([c_void_p, c_void_p, c_int64, c_void_p], c_int),
    "vg_batch_assemble_records_device": ([c_void_p, c_void_p, c_void_p], c_int),
    "vg_solver_create": ([c_void_p, c_int64, _PP], c_int),
    "vg_solver_destroy": ([c_void_p], c_int),
    "vg_solver_reset": ([c_void_p], c_int),
    "vg_solver_add_batch": ([c_void_p, c_void_p, _P_D, c_int64, _P_I64, _P_D], c_int),
    "vg_solver_add_blocks": ([c_void_p, c_int64, _P_I64, _P_D, _P_D], c_int),
    "vg_solver_factor": ([c_void_p, c_double, c_double, c_int32, _P_I64], c_int),
    "vg_solver_solve": ([c_void_p, _P_D, c_int64, _P_D], c_int),
    "vg_solver_export": ([c_void_p, _P_D, _P_D, _P_D], c_int),
    "vg_solver_diagonal": ([c_void_p, _P_D], c_int),
    "vg_knn": ([c_void_p, c_void_p, c_int32, _P_I64], c_int),
    "vg_covariances": ([c_void_p, c_void_p, _P_I64, c_int32, c_double, _P_D, _P_U8], c_int),
    "vg_cloud_estimate_covariances": ([c_void_p, c_void_p, c_int32, c_double, _P_I64, _P_D,
                                       _P_U8], c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None):
    """Load libvgicp.so and declare every entry point (no GPU needed for this step)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise VgicpUnavailable(
                f"{p} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; "
                "g.build()'` (the CUDA library is the only compute path)")
        lib = ctypes.CDLL(str(p))
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.vg_abi_version() != 1:
            raise VgicpUnavailable("libvgicp ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status code to the reference's exception types."""
    if rc == VG_OK:
        return
    msg = (_lib.vg_last_error() or b"").decode(errors="replace") if _lib else ""
    if what:
        msg = f"{what}: {msg}"
    if rc == VG_ERR_DEGENERATE:
        raise errors.DegenerateConstraint(msg)
    if rc == VG_ERR_TOO_SPARSE:
        raise errors.FrameTooSparse(msg)
    if rc == VG_ERR_INVALID:
        raise ValueError(msg)
    if rc == VG_ERR_NOMEM:
        raise MemoryError(msg)
    raise VgicpUnavailable(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_P_D) if a is not None else None


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_P_I64) if a is not None else None


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One CUDA device context of the library (one per process and device)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = c_void_p()
        check(lib.vg_ctx_create(int(device), ctypes.byref(h)), "vg_ctx_create")
        self.lib = lib
        self.device = int(device)
        self.handle = h
        self._fin = weakref.finalize(self, lib.vg_ctx_destroy, h)

    def set_stream(self, stream_ptr: int | None) -> None:
        check(self.lib.vg_ctx_set_stream(self.handle, c_void_p(stream_ptr or 0)))

    def synchronize(self) -> None:
        check(self.lib.vg_ctx_synchronize(self.handle))

    def launch_count(self) -> int:
        n = c_int64()
        check(self.lib.vg_ctx_launch_count(self.handle, ctypes.byref(n)))
        return int(n.value)


_contexts: dict[int, Context] = {}
_default_device = int(os.environ.get("VGICP_DEVICE", "0"))


def set_device(device: int) -> None:
    """Select the CUDA device used by subsequent calls (e.g. LOCAL_RANK under torchrun)."""
    global _default_device
    _default_device = int(device)


def context(device: int | None = None) -> Context:
    dev = _default_device if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        _contexts[dev] = ctx
    return ctx


class _PinnedOwner:
    """Owner of one page-locked buffer; numpy views of it keep it alive (array interface)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3}


class PinnedPool:
    """Page-locked host buffers (vg_host_alloc) for record outputs.  A device->host copy into
    pinned memory overlaps the staged computation (vg_batch_linearize*: each stage's records
    cross PCIe while the next stage computes); into pageable memory it does not.  A buffer
    goes back to the pool when the last numpy view of it dies, so callers may keep the
    returned arrays (the factor shim caches per-factor rows of them)."""

    def __init__(self):
        self._free: dict[int, list[int]] = {}
        self._lock = threading.Lock()

    def empty(self, shape, dtype=np.float64) -> np.ndarray:
        lib = load_library()
        dtype = np.dtype(dtype)
        nbytes = max(int(np.prod(shape)) * dtype.itemsize, 1)
        with self._lock:
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
        if ptr is None:
            p = c_void_p()
            check(lib.vg_host_alloc(nbytes, ctypes.byref(p)), "vg_host_alloc")
            ptr = p.value
        owner = _PinnedOwner(ptr, nbytes)
        weakref.finalize(owner, self._release, ptr, nbytes)
        return np.asarray(owner)[: int(np.prod(shape)) * dtype.itemsize].view(dtype).reshape(shape)

    def _release(self, ptr: int, nbytes: int) -> None:
        with self._lock:
            lst = self._free.setdefault(nbytes, [])
            if len(lst) < 4:
                lst.append(ptr)
                return
        if _lib is not None:
            _lib.vg_host_free(c_void_p(ptr))


PINNED = PinnedPool()


def record_cost_inliers_f32(rec: np.ndarray):
    """(cost, inliers) of compact fp32 linearization records (..., 94) -> fp64, int64."""
    words = np.ascontiguousarray(rec[..., 90:93])
    cost = words[..., 0:2].copy().view(np.float64)[..., 0]
    inl = words[..., 2].view(np.int32).astype(np.int64)
    return cost, inl


class DeviceCloud:
    """Device copy of a Frame's points (+ covariances): 64 B/point SoA in HBM (float4 xyz,
    fp64 covariance rows); non-fp32-exact points keep an extra fp64 xyz copy."""

    def __init__(self, points, covs=None, ctx: Context | None = None):
        ctx = ctx or context()
        pts = f64(points).reshape(-1, 3)
        cov = None if covs is None else f64(covs).reshape(-1, 9)
        if cov is not None and cov.shape[0] != pts.shape[0]:
            raise ValueError("covariances and points differ in length")
        h = c_void_p()
        check(ctx.lib.vg_cloud_create(ctx.handle, dptr(pts), dptr(cov), pts.shape[0],
                                      ctypes.byref(h)), "vg_cloud_create")
        self.ctx = ctx
        self.handle = h
        self.n = pts.shape[0]
        self.has_cov = cov is not None
        self._fin = weakref.finalize(self, ctx.lib.vg_cloud_destroy, h)

    def estimate_covariances(self, k: int, plane_eps: float, want_neighbors=True):
        """Fused device kNN + covariance; results stay attached to this cloud."""
        lib = self.ctx.lib
        # page-locked outputs: the device -> host copies run at PCIe speed (config 2: 131k
        # points, 0.59 vs 1.0 ms with pageable arrays)
        nbrs = PINNED.empty((self.n, k), np.int64) if want_neighbors else None
        covs = PINNED.empty((self.n, 3, 3))
        degen = PINNED.empty((self.n,), np.uint8)
        check(lib.vg_cloud_estimate_covariances(self.ctx.handle, self.handle, int(k),
                                                float(plane_eps), iptr(nbrs), dptr(covs),
                                                degen.ctypes.data_as(_P_U8)))
        self.has_cov = True
        return nbrs, covs, degen.astype(bool)


class DeviceMap:
    """Device Gaussian voxel map: 64 B hash slots + the reference fp64 arrays."""

    def __init__(self, handle, ctx: Context):
        self.ctx = ctx
        self.handle = handle
        m = c_int64()
        res = c_double()
        cap = c_int64()
        check(ctx.lib.vg_map_info(handle, ctypes.byref(m), ctypes.byref(res), ctypes.byref(cap)))
        self.m = int(m.value)
        self.resolution = float(res.value)
        self.capacity = int(cap.value)
        self._fin = weakref.finalize(self, ctx.lib.vg_map_destroy, handle)

    @classmethod
    def build(cls, cloud: DeviceCloud, resolution: float) -> "DeviceMap":
        h = c_void_p()
        check(cloud.ctx.lib.vg_map_build(cloud.ctx.handle, cloud.handle, float(resolution),
                                         ctypes.byref(h)), "vg_map_build")
        return cls(h, cloud.ctx)

    @classmethod
    def from_arrays(cls, resolution, keys, means, covs, counts, ctx: Context | None = None):
        ctx = ctx or context()
        keys = np.ascontiguousarray(keys, dtype=np.int64)
        m = keys.shape[0]
        means = f64(means).reshape(m, 3)
        covs = f64(covs).reshape(m, 9)
        counts = None if counts is None else np.ascontiguousarray(counts, dtype=np.int64)
        h = c_void_p()
        check(ctx.lib.vg_map_from_arrays(ctx.handle, float(resolution), iptr(keys), dptr(means),
                                         dptr(covs), iptr(counts), m, ctypes.byref(h)),
              "vg_map_from_arrays")
        return cls(h, ctx)

    def export(self):
        m = self.m
        keys = np.empty(m, dtype=np.int64)
        means = np.empty((m, 3))
        covs = np.empty((m, 3, 3))
        counts = np.empty(m, dtype=np.int64)
        check(self.ctx.lib.vg_map_export(self.ctx.handle, self.handle, iptr(keys), dptr(means),
                                         dptr(covs), iptr(counts)))
        return keys, means, covs, counts


class DeviceBatch:
    """A flattened set of matching-cost factors resident in HBM (vg_batch)."""

    def __init__(self, clouds, maps, unary, min_inliers, var_source=None, var_target=None,
                 ctx: Context | None = None):
        ctx = ctx or context()
        F = len(clouds)
        specs = (vg_factor_spec * max(F, 1))()
        for f in range(F):
            s = specs[f]
            s.source = clouds[f].handle.value
            s.target = maps[f].handle.value
            s.flags = FACTOR_UNARY if unary[f] else 0
            s.min_inliers = int(min_inliers[f])
            s.var_source = int(var_source[f]) if var_source is not None else 0
            s.var_target = int(var_target[f]) if var_target is not None else 0
        h = c_void_p()
        check(ctx.lib.vg_batch_create(ctx.handle, specs, F, ctypes.byref(h)), "vg_batch_create")
        self.ctx = ctx
        self.handle = h
        self.num_factors = F
        # keep the device objects alive as long as the batch references them
        self._keep = (list(clouds), list(maps))
        nf, ni, npnt = c_int64(), c_int64(), c_int64()
        check(ctx.lib.vg_batch_info(h, ctypes.byref(nf), ctypes.byref(ni), ctypes.byref(npnt)))
        self.num_items = int(ni.value)
        self.num_points = int(npnt.value)
        self._fin = weakref.finalize(self, ctx.lib.vg_batch_destroy, h)

    def linearize(self, T: np.ndarray, mode: int = MODE_LINEARIZE) -> np.ndarray:
        T = f64(T).reshape(self.num_factors, 12)
        out = PINNED.empty((self.num_factors, RECORD_SIZE[mode]))
        check(self.ctx.lib.vg_batch_linearize(self.handle, dptr(T), int(mode), dptr(out)),
              "vg_batch_linearize")
        return out

    def linearize_poses(self, poses: np.ndarray, mode: int = MODE_LINEARIZE,
                        out: np.ndarray | None = None) -> np.ndarray:
        """Records at the pose table (fp64, RECORD_SIZE[mode] per factor).  Without `out` the
        result lives in pinned memory, so its staged device->host copies overlap the compute."""
        poses = f64(poses).reshape(-1, 8)
        if out is None:
            out = PINNED.empty((self.num_factors, RECORD_SIZE[mode]))
        check(self.ctx.lib.vg_batch_linearize_poses(self.handle, dptr(poses), poses.shape[0],
                                                    int(mode), dptr(out)),
              "vg_batch_linearize_poses")
        return out

    def linearize_poses_f32(self, poses: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Compact linearization records (F, 94) float32 words (VG_REC_LINEARIZE_F32): fp32
        blocks in words 0-89, fp64 cost in 90-91, int32 inliers in 92 — half the PCIe bytes of
        linearize_poses.  Decode cost/inliers with record_cost_inliers_f32."""
        poses = f64(poses).reshape(-1, 8)
        if out is None:
            out = PINNED.empty((self.num_factors, REC_LINEARIZE_F32), np.float32)
        assert out.dtype == np.float32 and out.shape == (self.num_factors, REC_LINEARIZE_F32)
        check(self.ctx.lib.vg_batch_linearize_poses_f32(self.handle, dptr(poses), poses.shape[0],
                                                        MODE_LINEARIZE, out.ctypes.data),
              "vg_batch_linearize_poses_f32")
        return out

    def linearize_f32(self, T: np.ndarray) -> np.ndarray:
        """Explicit-transform variant of linearize_poses_f32."""
        T = f64(T).reshape(self.num_factors, 12)
        out = PINNED.empty((self.num_factors, REC_LINEARIZE_F32), np.float32)
        check(self.ctx.lib.vg_batch_linearize_f32(self.handle, dptr(T), MODE_LINEARIZE,
                                                  out.ctypes.data), "vg_batch_linearize_f32")
        return out

    def lookup_rows(self, poses: np.ndarray):
        """(rows, inliers): every factor's per-point reference row (-1 = miss), concatenated
        in factor order, and its hit count — the correspondences K4a hands to K4b."""
        poses = f64(poses).reshape(-1, 8)
        rows = np.empty(self.num_points, dtype=np.int64)
        inl = np.empty(self.num_factors, dtype=np.int64)
        check(self.ctx.lib.vg_batch_lookup_rows(self.handle, dptr(poses), poses.shape[0],
                                                iptr(rows), iptr(inl)), "vg_batch_lookup_rows")
        return rows, inl

    def linearize_poses_device(self, poses_dev_ptr: int | None, num_poses: int, mode: int,
                               out_dev_ptr: int) -> None:
        check(self.ctx.lib.vg_batch_linearize_poses_device(
            self.handle, c_void_p(poses_dev_ptr or 0), int(num_poses), int(mode),
            c_void_p(out_dev_ptr)), "vg_batch_linearize_poses_device")

    def compose_device(self, poses_dev_ptr: int, num_poses: int) -> None:
        check(self.ctx.lib.vg_batch_compose_device(self.handle, c_void_p(poses_dev_ptr),
                                                   int(num_poses)))

    def accumulate_device(self, mode: int) -> None:
        check(self.ctx.lib.vg_batch_accumulate_device(self.handle, int(mode)))

    def finalize_device(self, mode: int, out_dev_ptr: int) -> None:
        check(self.ctx.lib.vg_batch_finalize_device(self.handle, int(mode),
                                                    c_void_p(out_dev_ptr)))

    def capture_graph(self, poses_dev_ptr: int, num_poses: int, mode: int, out_dev_ptr: int):
        check(self.ctx.lib.vg_batch_graph_capture(self.handle, c_void_p(poses_dev_ptr),
                                                  int(num_poses), int(mode),
                                                  c_void_p(out_dev_ptr)))

    def capture_assemble_graph(self, poses_dev_ptr: int, num_poses: int, records_dev_ptr: int,
                               out_dev_ptr: int, zero_out: bool = False) -> None:
        """Capture compose + K4 + K5 + [zero] + K6 as the batch's graph (launch_graph)."""
        check(self.ctx.lib.vg_batch_graph_capture_assemble(
            self.handle, c_void_p(poses_dev_ptr), int(num_poses), c_void_p(records_dev_ptr),
            c_void_p(out_dev_ptr), int(bool(zero_out))), "vg_batch_graph_capture_assemble")

    def launch_graph(self) -> None:
        check(self.ctx.lib.vg_batch_graph_launch(self.handle))

    # ---- normal equations (FactorGraph._assemble_dense, factor_graph.py:522-536) ----------
    def assemble_setup(self, num_vars: int, pairs: np.ndarray | None = None) -> np.ndarray:
        """Variables are pose-table rows < num_vars; returns the (P, 2) variable pairs whose
        off-diagonal blocks the assembly produces — the batch's own pairs, or `pairs` (a
        sorted global list shared by all ranks of a sharded graph)."""
        P, total = c_int64(), c_int64()
        if pairs is None:
            check(self.ctx.lib.vg_batch_assemble_setup(self.handle, int(num_vars),
                                                       ctypes.byref(P), ctypes.byref(total)),
                  "vg_batch_assemble_setup")
            pairs = np.empty((int(P.value), 2), dtype=np.int32)
            if P.value:
                check(self.ctx.lib.vg_batch_assemble_pairs(
                    self.handle, pairs.ctypes.data_as(POINTER(c_int32))),
                    "vg_batch_assemble_pairs")
        else:
            pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
            check(self.ctx.lib.vg_batch_assemble_setup_pairs(
                self.handle, int(num_vars), pairs.ctypes.data_as(POINTER(c_int32)), len(pairs),
                ctypes.byref(total)), "vg_batch_assemble_setup_pairs")
        self.asm_vars = int(num_vars)
        self.asm_pairs = pairs
        self.asm_size = int(total.value)
        return pairs

    def assemble_setup_mapped(self, num_vars: int, pairs: np.ndarray, out_index: np.ndarray,
                              out_pairs: int) -> int:
        """Assembly over this batch's `pairs` (sorted), pair p's block written at slot
        out_index[p] of a layout with out_pairs slots; returns that layout's size (doubles)."""
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        idx = np.ascontiguousarray(out_index, dtype=np.int32)
        total = c_int64()
        check(self.ctx.lib.vg_batch_assemble_setup_mapped(
            self.handle, int(num_vars), pairs.ctypes.data_as(POINTER(c_int32)), len(pairs),
            idx.ctypes.data_as(POINTER(c_int32)), int(out_pairs), ctypes.byref(total)),
            "vg_batch_assemble_setup_mapped")
        self.asm_vars = int(num_vars)
        self.asm_pairs = pairs
        self.asm_size = int(total.value)
        return self.asm_size

    def assemble_poses(self, poses: np.ndarray, out: np.ndarray | None = None,
                       unpack: bool = True):
        """Normal equations at the pose table; `unpack=False` returns the flat C-ABI layout
        (cost, count, diag V x 21, grad V x 6, pair blocks P x 36) in `out`."""
        poses = f64(poses).reshape(-1, 8)
        if out is None:
            out = np.empty(self.asm_size)
        check(self.ctx.lib.vg_batch_assemble_poses(self.handle, dptr(poses), poses.shape[0],
                                                   dptr(out)), "vg_batch_assemble_poses")
        return NormalEquations.from_flat(out, self.asm_vars, self.asm_pairs) if unpack else out

    def assemble_records_device(self, records_dev_ptr: int, out_dev_ptr: int) -> None:
        """K6 over records written by finalize_device(MODE_LINEARIZE) on this batch."""
        check(self.ctx.lib.vg_batch_assemble_records_device(
            self.handle, c_void_p(records_dev_ptr), c_void_p(out_dev_ptr)),
            "vg_batch_assemble_records_device")

    def assemble_poses_device(self, poses_dev_ptr: int, num_poses: int, out_dev_ptr: int) -> None:
        check(self.ctx.lib.vg_batch_assemble_poses_device(
            self.handle, c_void_p(poses_dev_ptr), int(num_poses), c_void_p(out_dev_ptr)),
            "vg_batch_assemble_poses_device")


SOLVE_CHOLESKY, SOLVE_CHOLESKY_LU = 0, 1


class DeviceSolver:
    """Dense normal equations of a graph on the device and their damped solve (vg_solver_*,
    SURVEY §8f row 3): the replacement of optimize_lm's per-attempt host factorization
    (factor_graph.py:565-576) and marginal_covariance's (:707-722)."""

    def __init__(self, dim: int, ctx: "Context | None" = None):
        self.ctx = ctx or context()
        self.dim = int(dim)
        h = c_void_p()
        check(self.ctx.lib.vg_solver_create(self.ctx.handle, self.dim, ctypes.byref(h)),
              "vg_solver_create")
        self.handle = h
        self._fin = weakref.finalize(self, self.ctx.lib.vg_solver_destroy, h)

    def reset(self) -> None:
        check(self.ctx.lib.vg_solver_reset(self.handle), "vg_solver_reset")

    def add_batch(self, batch: "DeviceBatch", poses: np.ndarray, offsets) -> float:
        """Scatter the batch's device-assembled normal equations (assemble_setup first) at the
        pose table; variable v's 6x6 block at tangent offset offsets[v].  Returns its cost."""
        poses = f64(poses).reshape(-1, 8)
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        if len(offs) != batch.asm_vars:
            raise ValueError("one tangent offset per assembled variable")
        cost = c_double()
        check(self.ctx.lib.vg_solver_add_batch(self.handle, batch.handle, dptr(poses),
                                               poses.shape[0], iptr(offs), ctypes.byref(cost)),
              "vg_solver_add_batch")
        return float(cost.value)

    def add_blocks(self, blocks, g: np.ndarray | None = None) -> None:
        """Add host blocks [(row0, col0, array)] (non-overlapping) and a gradient vector."""
        if blocks:
            desc = np.array([(r, c, a.shape[0], a.shape[1]) for r, c, a in blocks],
                            dtype=np.int64)
            vals = np.concatenate([f64(a).ravel() for _, _, a in blocks])
        else:
            desc, vals = None, None
        gg = None if g is None else f64(g)
        check(self.ctx.lib.vg_solver_add_blocks(self.handle, 0 if desc is None else len(desc),
                                                iptr(desc), dptr(vals), dptr(gg)),
              "vg_solver_add_blocks")

    def factor(self, lam: float = 0.0, jitter: float = 0.0,
               method: int = SOLVE_CHOLESKY) -> int:
        """Factor H + lam diag(H) + jitter I; 0 on success, else the failing minor / pivot."""
        info = c_int64()
        check(self.ctx.lib.vg_solver_factor(self.handle, float(lam), float(jitter), int(method),
                                            ctypes.byref(info)), "vg_solver_factor")
        return int(info.value)

    def solve(self, rhs: np.ndarray | None = None) -> np.ndarray:
        """X with A X = rhs (dim or dim x k); rhs None solves A x = -g."""
        if rhs is None:
            x = np.empty(self.dim)
            check(self.ctx.lib.vg_solver_solve(self.handle, None, 1, dptr(x)), "vg_solver_solve")
            return x
        rhs = np.asarray(rhs, dtype=np.float64)
        k = 1 if rhs.ndim == 1 else rhs.shape[1]
        b = np.asfortranarray(rhs.reshape(self.dim, k))
        x = np.empty((self.dim, k), order="F")
        check(self.ctx.lib.vg_solver_solve(self.handle, b.ctypes.data_as(_P_D), k,
                                           x.ctypes.data_as(_P_D)), "vg_solver_solve")
        return x.reshape(rhs.shape)

    def diagonal(self) -> np.ndarray:
        d = np.empty(self.dim)
        check(self.ctx.lib.vg_solver_diagonal(self.handle, dptr(d)), "vg_solver_diagonal")
        return d

    def export(self, h: bool = True):
        """(H or None, g, accumulated batch cost)."""
        hh = np.empty((self.dim, self.dim)) if h else None
        g = np.empty(self.dim)
        cost = c_double()
        check(self.ctx.lib.vg_solver_export(self.handle, dptr(hh), dptr(g), ctypes.byref(cost)),
              "vg_solver_export")
        return hh, g, float(cost.value)


_UPPER6 = np.triu_indices(6)


class NormalEquations:
    """Block-sparse H, g and cost of a batch's factors (vg_batch_assemble_*): 6x6 diagonal
    blocks per variable, the gradient per variable, and H blocks (a, b) for pairs a < b."""

    def __init__(self, cost, count, diag, grad, pairs, off):
        self.cost, self.count = cost, count
        self.diag, self.grad, self.pairs, self.off = diag, grad, pairs, off

    @classmethod
    def from_flat(cls, flat: np.ndarray, V: int, pairs: np.ndarray) -> "NormalEquations":
        P = len(pairs)
        up = flat[2:2 + 21 * V].reshape(V, 21)
        diag = np.zeros((V, 6, 6))
        diag[:, _UPPER6[0], _UPPER6[1]] = up
        diag[:, _UPPER6[1], _UPPER6[0]] = up
        grad = flat[2 + 21 * V:2 + 27 * V].reshape(V, 6).copy()
        off = flat[2 + 27 * V:2 + 27 * V + 36 * P].reshape(P, 6, 6).copy()
        return cls(float(flat[0]), int(flat[1]), diag, grad, pairs, off)

    def dense(self, offsets=None, dim=None):
        """Dense H, g; variable v's 6x6 block at rows offsets[v]:offsets[v]+6 (default 6v)."""
        V = len(self.diag)
        offsets = np.arange(V) * 6 if offsets is None else np.asarray(offsets)
        dim = 6 * V if dim is None else dim
        h = np.zeros((dim, dim))
        g = np.zeros(dim)
        rows = offsets[:, None] + np.arange(6)          # (V, 6); blocks are disjoint
        h[rows[:, :, None], rows[:, None, :]] += self.diag
        g[rows] += self.grad
        if len(self.pairs):
            ra = rows[self.pairs[:, 0]]
            rb = rows[self.pairs[:, 1]]
            h[ra[:, :, None], rb[:, None, :]] += self.off
            h[rb[:, :, None], ra[:, None, :]] += self.off.transpose(0, 2, 1)
        return h, g
