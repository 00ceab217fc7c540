"""ctypes binding of include/yy.h (names follow the C ABI one to one).

Marshalling only: shapes are checked, arrays are made C-contiguous fp64 and
handed to libyy.so.  Device memory, kernels and the Schwarz loop live in the
library.  See include/yy.h for argument meaning, layout and errors.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

YY_OK, YY_ENOCONV = 0, 4
YY_CHI, YY_MAX_ITERS, YY_FIXED_ITERS, YY_PROFILE, YY_SCHWARZ, YY_HEAT_ONLY, YY_FLUX_FIX = 1, 2, 3, 4, 5, 6, 7
YY_INTERP_ORDER = 8
YY_ADVECTION = 9
TF_ONE, TF_COS, TF_SIN, TF_COS2 = 0, 1, 2, 3
SCHWARZ = {"additive": 0, "multiplicative": 1, "none": 2}

EXPORTS = ("yy_create", "yy_set_fields", "yy_get_fields", "yy_set_wall", "yy_set_source",
           "yy_set_param", "yy_set_stream", "yy_step", "yy_get_stats", "yy_time",
           "yy_last_error", "yy_destroy", "yy_debug_get", "yy_line_solve", "yy_line_prepare", "yy_launch_count",
           "yy_profile_report", "yy_set_allocator", "yy_energy")


class YYError(RuntimeError):
    pass


class yy_grid(ctypes.Structure):
    _fields_ = [("nr", c_int32), ("ntheta", c_int32), ("nphi", c_int32)]


_DP = POINTER(c_double)


class yy_fields(ctypes.Structure):
    _fields_ = [("ur", _DP), ("ut", _DP), ("up", _DP), ("p", _DP), ("T", _DP)]


ALLOC_FN = ctypes.CFUNCTYPE(c_void_p, ctypes.c_size_t, c_void_p)   # yy_set_allocator callbacks
FREE_FN = ctypes.CFUNCTYPE(None, c_void_p, c_void_p)


def lib_path() -> str:
    # YY_LIB: an alternative build of the same library (tuning experiments only)
    return os.environ.get("YY_LIB") or os.path.join(_HERE, "libyy.so")


_lib = None


def load_library():
    """Load libyy.so (in-tree).  Raises YYError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    p = lib_path()
    if not os.path.exists(p):
        raise YYError(f"{p} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(p)
    ctx = c_void_p
    L.yy_create.argtypes = [POINTER(yy_grid), c_double, c_double, c_double, c_double, c_double, POINTER(ctx)]
    L.yy_set_fields.argtypes = [ctx, c_int32, c_int32, c_int32, POINTER(yy_fields)]
    L.yy_get_fields.argtypes = [ctx, c_int32, c_int32, c_int32, POINTER(yy_fields)]
    L.yy_set_wall.argtypes = [ctx, c_int32, c_int32, POINTER(c_int32), POINTER(yy_fields)]
    L.yy_set_source.argtypes = [ctx, c_int32, c_int32, POINTER(c_int32), POINTER(yy_fields)]
    L.yy_set_param.argtypes = [ctx, c_int32, c_double]
    L.yy_set_stream.argtypes = [ctx, c_void_p]
    L.yy_step.argtypes = [ctx, c_int32, c_double]
    L.yy_get_stats.argtypes = [ctx, c_int32, POINTER(c_int32), POINTER(c_double), POINTER(c_int32)]
    L.yy_time.argtypes = [ctx]
    L.yy_time.restype = c_double
    L.yy_last_error.argtypes = [ctx]
    L.yy_last_error.restype = c_char_p
    L.yy_destroy.argtypes = [ctx]
    L.yy_destroy.restype = None
    L.yy_debug_get.argtypes = [ctx, c_char_p, c_int32, _DP]
    L.yy_line_solve.argtypes = [ctx, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]
    L.yy_line_prepare.argtypes = [ctx, c_void_p, c_void_p, c_void_p]
    L.yy_set_allocator.argtypes = [ctx, ALLOC_FN, FREE_FN, c_void_p]
    L.yy_set_allocator.restype = c_int32
    L.yy_launch_count.argtypes = [ctx]
    L.yy_launch_count.restype = ctypes.c_int64
    L.yy_profile_report.argtypes = [ctx, ctypes.c_char_p, c_int32]
    L.yy_create_pair.argtypes = [POINTER(yy_grid), c_double, c_double, c_double, c_double, c_double, c_void_p]
    L.yy_create_slabs.argtypes = [POINTER(yy_grid), c_double, c_double, c_double, c_double, c_double, c_int32,
                                  c_void_p]
    L.yy_create_dist.argtypes = [POINTER(yy_grid), c_double, c_double, c_double, c_double, c_double,
                                 c_int32, c_int32, c_void_p, c_int32, POINTER(ctx)]
    L.yy_nccl_unique_id.argtypes = [c_void_p]
    L.yy_energy.argtypes = [ctx, _DP]
    for name in ("yy_create_pair", "yy_create_slabs", "yy_create_dist", "yy_nccl_unique_id", "yy_create", "yy_set_fields", "yy_get_fields", "yy_set_wall", "yy_set_source",
                 "yy_set_param", "yy_set_stream", "yy_step", "yy_get_stats", "yy_debug_get", "yy_line_solve", "yy_line_prepare",
                 "yy_profile_report", "yy_set_allocator", "yy_energy"):
        getattr(L, name).restype = c_int32
    _lib = L
    return L


def _ptr(a):
    return a.ctypes.data_as(_DP) if a is not None else None


class Shell:
    """One Yin-Yang shell context (include/yy.h `yy_ctx`)."""

    def __init__(self, nr, ntheta, nphi, R1=1.0, R2=2.0, Pr=1.0, Ra=0.0, dt=1e-3,
                 chi=None, max_iters=None, fixed_iters=None, stream=None, heat_only=False, flux_fix_eps=None,
                 schwarz=None, advection=None, _handle=None, _patches=(0, 1)):
        self.L = load_library()
        self.nr, self.nt, self.np_ = nr, ntheta, nphi
        self.patches = tuple(_patches)        # patches this context holds
        if _handle is None:
            g = yy_grid(nr, ntheta, nphi)
            h = c_void_p()
            st = self.L.yy_create(ctypes.byref(g), R1, R2, Pr, Ra, dt, ctypes.byref(h))
            if st != YY_OK:
                raise YYError(f"yy_create failed with status {st}")
            _handle = h
        self.h = _handle
        if chi is not None:
            self.set_param(YY_CHI, chi)
        if max_iters is not None:
            self.set_param(YY_MAX_ITERS, max_iters)
        if fixed_iters is not None:
            self.set_param(YY_FIXED_ITERS, fixed_iters)
        if stream is not None:
            self.set_stream(stream)
        if heat_only:
            self.set_param(YY_HEAT_ONLY, 1)
        if flux_fix_eps is not None:
            self.set_param(YY_FLUX_FIX, flux_fix_eps)
        if schwarz is not None:
            self.set_param(YY_SCHWARZ, SCHWARZ[schwarz])
        if advection is not None:
            self.set_param(YY_ADVECTION, {"split": 0, "imex": 1}[advection])

    @classmethod
    def pair(cls, nr, ntheta, nphi, R1=1.0, R2=2.0, Pr=1.0, Ra=0.0, dt=1e-3, **kw):
        """yy_create_pair (include/yy_test.h): (Yin, Yang) one-patch contexts on this
        device exchanging through device copies — the yy_create_dist data path."""
        L = load_library()
        g = yy_grid(nr, ntheta, nphi)
        hs = (c_void_p * 2)()
        st = L.yy_create_pair(ctypes.byref(g), R1, R2, Pr, Ra, dt, hs)
        if st != YY_OK:
            raise YYError(f"yy_create_pair failed with status {st}")
        out = [cls(nr, ntheta, nphi, _handle=c_void_p(hs[p]), _patches=(p,)) for p in range(2)]
        for sh in out:
            sh._configure(**kw)
        return out

    @classmethod
    def slabs(cls, nr, ntheta, nphi, R1=1.0, R2=2.0, Pr=1.0, Ra=0.0, dt=1e-3, nslab=2, **kw):
        """yy_create_slabs (include/yy_test.h): 2*nslab radial-slab contexts
        [rank = patch*nslab + slab] on this device exchanging through device
        copies — the yy_create_dist layout of 2*nslab GPUs."""
        L = load_library()
        g = yy_grid(nr, ntheta, nphi)
        hs = (c_void_p * (2 * nslab))()
        st = L.yy_create_slabs(ctypes.byref(g), R1, R2, Pr, Ra, dt, nslab, hs)
        if st != YY_OK:
            raise YYError(f"yy_create_slabs failed with status {st}")
        out = [cls(nr, ntheta, nphi, _handle=c_void_p(hs[r]), _patches=(r // nslab,)) for r in range(2 * nslab)]
        for sh in out:
            sh._configure(**kw)
        return out

    @classmethod
    def dist(cls, nr, ntheta, nphi, R1, R2, Pr, Ra, dt, world, rank, nccl_id, device, **kw):
        """yy_create_dist: rank `rank` of `world` (2: one patch per rank) over NCCL."""
        L = load_library()
        g = yy_grid(nr, ntheta, nphi)
        h = c_void_p()
        idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
        st = L.yy_create_dist(ctypes.byref(g), R1, R2, Pr, Ra, dt, world, rank, idb, device, ctypes.byref(h))
        if st != YY_OK:
            raise YYError(f"yy_create_dist failed with status {st}")
        sh = cls(nr, ntheta, nphi, _handle=h, _patches=(rank // (world // 2),) if world > 1 else (0, 1))
        sh._configure(**kw)
        return sh

    def _configure(self, chi=None, max_iters=None, fixed_iters=None, stream=None, schwarz=None, flux_fix_eps=None,
                   advection=None):
        if advection is not None:
            self.set_param(YY_ADVECTION, {"split": 0, "imex": 1}[advection])
        if chi is not None:
            self.set_param(YY_CHI, chi)
        if max_iters is not None:
            self.set_param(YY_MAX_ITERS, max_iters)
        if fixed_iters is not None:
            self.set_param(YY_FIXED_ITERS, fixed_iters)
        if stream is not None:
            self.set_stream(stream)
        if schwarz is not None:
            self.set_param(YY_SCHWARZ, SCHWARZ[schwarz])
        if flux_fix_eps is not None:
            self.set_param(YY_FLUX_FIX, flux_fix_eps)

    # shapes of include/yy.h
    def shape(self, name):
        nr, nt, npp = self.nr, self.nt, self.np_
        return {"ur": (nr + 1, nt, npp), "ut": (nr, nt + 1, npp), "up": (nr, nt, npp + 1),
                "p": (nr, nt, npp), "T": (nr, nt, npp)}[name]

    def wall_shape(self, name):
        return (2,) + self.shape(name)[1:]

    def _check(self, st, what):
        if st < 0:
            msg = self.L.yy_last_error(self.h).decode(errors="replace")
            raise YYError(f"{what}: status {st}: {msg}")
        return st

    def close(self):
        if getattr(self, "h", None):
            self.L.yy_destroy(self.h)
            self.h = None

    __del__ = close

    def set_param(self, key, value):
        self._check(self.L.yy_set_param(self.h, key, float(value)), "yy_set_param")

    def set_stream(self, stream):
        """stream: an int cudaStream_t handle (e.g. torch.cuda.current_stream().cuda_stream)."""
        self._check(self.L.yy_set_stream(self.h, c_void_p(int(stream))), "yy_set_stream")

    def _fields(self, arrays, shape_fn):
        keep = {}
        f = yy_fields()
        for name in ("ur", "ut", "up", "p", "T"):
            a = arrays.get(name)
            if a is None:
                continue
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.shape != shape_fn(name):
                raise YYError(f"{name}: shape {a.shape} != {shape_fn(name)}")
            keep[name] = a
            setattr(f, name, _ptr(a))
        return f, keep

    def set_fields(self, patch, level, system, **arrays):
        f, keep = self._fields(arrays, self.shape)
        self._check(self.L.yy_set_fields(self.h, patch, level, system, ctypes.byref(f)), "yy_set_fields")

    def get_fields(self, patch, level=0, system=2, names=("ur", "ut", "up", "p", "T"), out=None):
        """out: optional dict of full-patch arrays to fill (a radial slab writes the
        rows it owns, so passing the same dict to every slab assembles the patch)."""
        if out is None:
            out = {n: np.empty(self.shape(n)) for n in names if not (n == "p" and level == 1)}
        f = yy_fields()
        for n, a in out.items():
            setattr(f, n, _ptr(a))
        self._check(self.L.yy_get_fields(self.h, patch, level, system, ctypes.byref(f)), "yy_get_fields")
        return out

    def _terms(self, fn, patch, terms, shape_fn, what):
        n = len(terms)
        tfs = (c_int32 * max(n, 1))(*[int(t) for t, _ in terms])
        arr = (yy_fields * max(n, 1))()
        keep = []
        for m, (_, d) in enumerate(terms):
            f, k = self._fields(d, shape_fn)
            arr[m] = f
            keep.append(k)
        self._check(fn(self.h, patch, n, tfs, arr), what)

    def set_wall(self, patch, terms):
        """terms: [(timefn, {"T","ur","ut","up": (2, ., .) arrays})]"""
        self._terms(self.L.yy_set_wall, patch, terms, self.wall_shape, "yy_set_wall")

    def set_source(self, patch, terms):
        """terms: [(timefn, {"T","ur","ut","up": full 3-D arrays})]"""
        self._terms(self.L.yy_set_source, patch, terms, self.shape, "yy_set_source")

    def step(self, nsteps=1, tol=1e-10):
        return self._check(self.L.yy_step(self.h, int(nsteps), float(tol)), "yy_step")

    def stats(self, cap=100000):
        it = (c_int32 * cap)()
        rs = (c_double * cap)()
        n = c_int32()
        self._check(self.L.yy_get_stats(self.h, cap, it, rs, ctypes.byref(n)), "yy_get_stats")
        return [(it[q], rs[q]) for q in range(n.value)]

    def time(self):
        return self.L.yy_time(self.h)

    def launch_count(self):
        return int(self.L.yy_launch_count(self.h))

    def profile(self, on=True):
        self.set_param(YY_PROFILE, 1.0 if on else 0.0)

    def profile_report(self):
        """{kernel class: (launches, total_ms)} since profile(True)."""
        buf = ctypes.create_string_buffer(1 << 16)
        self._check(self.L.yy_profile_report(self.h, buf, len(buf)), "yy_profile_report")
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split()
            out[name] = (int(n), float(ms))
        return out

    def energy(self):
        """yy_energy: (1/2 (-L T, T)_w, 1/4 ||dT||^2_D, ||dT||^2_w) of eq:Stability."""
        out = (c_double * 3)()
        self._check(self.L.yy_energy(self.h, out), "yy_energy")
        return tuple(out)

    def debug_get(self, name, patch):
        kind = {"astar_r": "ur", "astar_t": "ut", "astar_p": "up", "G_T": "T"}.get(name)
        if kind is None:
            kind = name[2:4]
        out = np.empty(self.shape(kind))
        self._check(self.L.yy_debug_get(self.h, name.encode(), patch, _ptr(out)), "yy_debug_get")
        return out

    def line_solve(self, axis, ar, at, ap, x):
        """C4 kernel-only sweep on device tensors (torch, float64, contiguous).
        ar = at = ap = None: the row weights of the last line_prepare."""
        for t in (ar, at, ap, x):
            if t is not None and not (t.is_cuda and t.dtype.is_floating_point and t.is_contiguous()):
                raise YYError("line_solve needs contiguous CUDA float64 tensors")
        p = lambda t: c_void_p(t.data_ptr()) if t is not None else None
        self._check(self.L.yy_line_solve(self.h, axis, p(ar), p(at), p(ap), p(x)), "yy_line_solve")

    def line_prepare(self, ar, at, ap):
        """Row weights of a* for line_solve(axis, None, None, None, x)."""
        for t in (ar, at, ap):
            if not (t.is_cuda and t.dtype.is_floating_point and t.is_contiguous()):
                raise YYError("line_prepare needs contiguous CUDA float64 tensors")
        self._check(self.L.yy_line_prepare(self.h, c_void_p(ar.data_ptr()), c_void_p(at.data_ptr()),
                                           c_void_p(ap.data_ptr())), "yy_line_prepare")

    def load_workload(self, wl):
        """Upload a workloads.make_workload() dict (levels, walls, sources)."""
        for patch, pd in enumerate(wl["patches"]):
            if patch not in self.patches:
                continue
            n = pd["n"]
            # both systems from one host copy of u (u1 = u2 at the start), then p2
            self.set_fields(patch, 0, 0, ur=n["ur"], ut=n["ut"], up=n["up"], T=n["T"], p=n["p1"])
            self.set_fields(patch, 0, 2, p=n["p2"])
            m = pd["nm1"]
            self.set_fields(patch, 1, 0, **{k: m[k] for k in ("ur", "ut", "up", "T")})
            self.set_wall(patch, pd["walls"])
            self.set_source(patch, pd["sources"])


def nccl_unique_id():
    """128-byte NCCL unique id for yy_create_dist (call on rank 0, broadcast it)."""
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    st = L.yy_nccl_unique_id(buf)
    if st != YY_OK:
        raise YYError(f"yy_nccl_unique_id failed with status {st} (NCCL not loadable?)")
    return buf.raw


_alloc_keep = []   # every callback pair ever installed: contexts created with it free through it


def use_torch_allocator(enable: bool = True, device=None):
    """Route the device buffers of every context created from now on through
    PyTorch's caching allocator (yy_set_allocator(NULL, ...)); enable=False
    restores cudaMalloc for later contexts.  The callbacks stay alive for the
    life of the process (a context frees through the pair it was created with)."""
    L = load_library()
    if not enable:
        st = L.yy_set_allocator(None, ALLOC_FN(), FREE_FN(), None)
    else:
        import torch
        dev = torch.cuda.current_device() if device is None else device

        def alloc(nbytes, user):
            try:
                return torch.cuda.caching_allocator_alloc(nbytes, dev)
            except Exception:   # -> NULL -> YY_ENOMEM
                return None

        def free(ptr, user):
            try:
                torch.cuda.caching_allocator_delete(ptr)
            except Exception:   # interpreter shutdown: torch already gone
                pass

        keep = (ALLOC_FN(alloc), FREE_FN(free))
        _alloc_keep.append(keep)
        st = L.yy_set_allocator(None, keep[0], keep[1], None)
    if st != YY_OK:
        raise YYError(f"yy_set_allocator failed with status {st}")
