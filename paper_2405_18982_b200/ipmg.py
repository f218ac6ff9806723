"""Thin ctypes binding of libipmg.so (include/ipmg.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  PyTorch
tensors provide device memory and the CUDA stream.

The library is loaded from this package directory; if it is missing the
import of the product API raises (there is no CPU fallback).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPMG_LIB", os.path.join(_HERE, "libipmg.so"))   # IPMG_LIB: A/B variants

IPMG_OK = 0
IPMG_ERR_NOT_CONVERGED = 7
FP64, FP32 = 0, 1
MULTIPLICATIVE, ADDITIVE = 0, 1
KERNEL_FULL, KERNEL_DIRICHLET, KERNEL_CLAMPED = 0, 1, 2
BASIS_LAGRANGE, BASIS_HERMITE = 0, 1
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "SIZE_MISMATCH", 4: "OUT_OF_MEMORY",
          5: "CUDA", 6: "NCCL", 7: "NOT_CONVERGED"}

# every symbol include/ipmg.h declares
EXPORTS = ["ipmg_config_default", "ipmg_create", "ipmg_destroy", "ipmg_level_info", "ipmg_vmult",
           "ipmg_smooth", "ipmg_smooth_colour", "ipmg_residual_restrict", "ipmg_prolongate_add",
           "ipmg_coarse_solve", "ipmg_vcycle", "ipmg_cg_solve", "ipmg_gmres_solve", "ipmg_rhs", "ipmg_to_cellwise",
           "ipmg_from_cellwise", "ipmg_synchronize", "ipmg_last_error", "ipmg_tables_1d",
           "ipmg_profile", "ipmg_profile_read", "ipmg_launch_count", "ipmg_level_partition", "ipmg_partition",
           "ipmg_nccl_unique_id", "ipmg_comm_create_nccl", "ipmg_comm_create_local", "ipmg_comm_destroy", "ipmg_alu_peak"]

KERNEL_CLASSES = {"smooth": 0, "vmult": 1, "restrict": 2, "prolong": 3, "coarse": 4, "blas": 5, "additive": 6,
                  "levels_below": 7}


class Config(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("degree", ctypes.c_int), ("coarse_cells", ctypes.c_int * 3),
                ("n_levels", ctypes.c_int), ("h0", ctypes.c_double), ("kernel", ctypes.c_int),
                ("smoother", ctypes.c_int), ("additive_omega", ctypes.c_double),
                ("post_smooth_reverse", ctypes.c_int), ("vcycle_precision", ctypes.c_int),
                ("penalty_scale", ctypes.c_double), ("device", ctypes.c_int),
                ("cuda_stream", ctypes.c_void_p), ("comm", ctypes.c_void_p), ("basis", ctypes.c_int),
                ("dist_min_dofs", ctypes.c_int64), ("boundary_penalty_scale", ctypes.c_double)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("nu", ctypes.c_double), ("rel_residual", ctypes.c_double),
                ("seconds", ctypes.c_double), ("history_len", ctypes.c_int),
                ("history", ctypes.POINTER(ctypes.c_double)), ("history_cap", ctypes.c_int)]


_lib = None


def load():
    """Load libipmg.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libipmg.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    sig = {
        "ipmg_config_default": (None, [ctypes.POINTER(Config)]),
        "ipmg_create": (i, [ctypes.POINTER(Config), ctypes.POINTER(vp)]),
        "ipmg_destroy": (i, [vp]),
        "ipmg_level_info": (i, [vp, i, ctypes.POINTER(ctypes.c_int64), ctypes.c_int * 3,
                                ctypes.POINTER(ctypes.c_double)]),
        "ipmg_vmult": (i, [vp, i, i, vp, vp]),
        "ipmg_smooth": (i, [vp, i, i, vp, vp, i]),
        "ipmg_smooth_colour": (i, [vp, i, i, vp, vp, vp, i]),
        "ipmg_residual_restrict": (i, [vp, i, i, vp, vp, vp]),
        "ipmg_prolongate_add": (i, [vp, i, i, vp, vp]),
        "ipmg_coarse_solve": (i, [vp, i, vp, vp]),
        "ipmg_vcycle": (i, [vp, vp, vp]),
        "ipmg_cg_solve": (i, [vp, vp, vp, d, i, ctypes.POINTER(SolveInfo)]),
        "ipmg_gmres_solve": (i, [vp, vp, vp, d, i, ctypes.POINTER(SolveInfo)]),
        "ipmg_rhs": (i, [vp, i, i, vp]),
        "ipmg_to_cellwise": (i, [vp, i, i, vp, vp]),
        "ipmg_from_cellwise": (i, [vp, i, i, vp, vp]),
        "ipmg_synchronize": (i, [vp]),
        "ipmg_last_error": (ctypes.c_char_p, [vp]),
        "ipmg_tables_1d": (i, [i, d, i, ctypes.POINTER(ctypes.c_double), i, ctypes.POINTER(ctypes.c_int)]),
        "ipmg_profile": (i, [vp, i]),
        "ipmg_profile_read": (i, [vp, i, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]),
        "ipmg_launch_count": (i, [vp, ctypes.POINTER(ctypes.c_int64)]),
        "ipmg_level_partition": (i, [vp, i, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int)]),
        "ipmg_partition": (i, [i, ctypes.c_int * 3, i, i, i, i, i, ctypes.c_int64, ctypes.c_int * 4]),
        "ipmg_nccl_unique_id": (i, [ctypes.c_char_p]),
        "ipmg_comm_create_nccl": (i, [ctypes.c_char_p, i, i, i, ctypes.POINTER(vp)]),
        "ipmg_comm_create_local": (i, [i, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp)]),
        "ipmg_comm_destroy": (i, [vp]),
        "ipmg_alu_peak": (i, [i, i, i, ctypes.POINTER(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class IpmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("ipmg status %s: %s" % (STATUS.get(status, status), msg))
        self.status = status


def tables_1d(k, what, penalty_scale=1.0):
    """Host-only: unit 1D tables the kernels use (see ipmg_tables_1d)."""
    lib = load()
    buf = (ctypes.c_double * 4096)()
    n = ctypes.c_int(0)
    st = lib.ipmg_tables_1d(k, penalty_scale, what, buf, 4096, ctypes.byref(n))
    if st != IPMG_OK:
        raise IpmgError(st, "ipmg_tables_1d")
    return np.array(buf[:n.value])


def alu_peak(device=0, kind="ffma2", reps=5):
    """Measured CUDA-core peak in TFLOP/s (ipmg_alu_peak): kind 'ffma2', 'ffma' or 'dfma'."""
    lib = load()
    out = ctypes.c_double()
    st = lib.ipmg_alu_peak(device, {"ffma2": 0, "ffma": 1, "dfma": 2}[kind], reps, ctypes.byref(out))
    if st != IPMG_OK:
        raise IpmgError(st, "ipmg_alu_peak")
    return out.value


def partition(dim, coarse_cells, n_levels, nranks, rank, level, degree=1, min_local_dofs=0):
    """Host-only slab partition rule (ipmg_partition): (distributed, zoff, local_layers, global_layers)."""
    lib = load()
    cc = (ctypes.c_int * 3)(*(list(coarse_cells) + [1] * (3 - len(coarse_cells))))
    out = (ctypes.c_int * 4)()
    st = lib.ipmg_partition(dim, cc, n_levels, nranks, rank, level, degree, min_local_dofs, out)
    if st != IPMG_OK:
        raise IpmgError(st, "ipmg_partition")
    return tuple(out)


class Comm:
    """A rank's communicator of the slab decomposition (ipmg_comm_*)."""

    def __init__(self, ptr, rank, nranks, kind):
        self.ptr, self.rank, self.nranks, self.kind = ptr, rank, nranks, kind

    @staticmethod
    def nccl_unique_id():
        lib = load()
        buf = ctypes.create_string_buffer(128)
        st = lib.ipmg_nccl_unique_id(buf)
        if st != IPMG_OK:
            raise IpmgError(st, lib.ipmg_last_error(None).decode())
        return buf.raw

    @classmethod
    def nccl(cls, rank, nranks, device, unique_id):
        """unique_id: the 128 bytes rank 0 got from nccl_unique_id(), broadcast to all ranks."""
        lib = load()
        c = ctypes.c_void_p()
        st = lib.ipmg_comm_create_nccl(unique_id, rank, nranks, device, ctypes.byref(c))
        if st != IPMG_OK:
            raise IpmgError(st, lib.ipmg_last_error(None).decode())
        return cls(c, rank, nranks, "nccl")

    @classmethod
    def from_torch_distributed(cls, device):
        """NCCL communicator over the default torch.distributed process group
        (the unique id travels through the group, gloo or nccl)."""
        import torch.distributed as dist
        rank, n = dist.get_rank(), dist.get_world_size()
        obj = [cls.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.nccl(rank, n, device, obj[0])

    @classmethod
    def local_team(cls, nranks, devices=None):
        """In-process team: one member per host thread (tests the distributed path on one GPU)."""
        lib = load()
        arr = (ctypes.c_void_p * nranks)()
        devs = (ctypes.c_int * nranks)(*(devices or [0] * nranks))
        st = lib.ipmg_comm_create_local(nranks, devs, ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)))
        if st != IPMG_OK:
            raise IpmgError(st, lib.ipmg_last_error(None).decode())
        return [cls(ctypes.c_void_p(arr[r]), r, nranks, "local") for r in range(nranks)]

    def close(self):
        if self.ptr:
            load().ipmg_comm_destroy(self.ptr)
            self.ptr = None


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class Handle:
    """One solver instance (ipmg_create/ipmg_destroy); methods mirror the C ABI."""

    def __init__(self, dim, degree, n_levels, coarse_cells=None, h0=0.5, smoother=MULTIPLICATIVE,
                 additive_omega=0.0, post_smooth_reverse=1, vcycle_precision=FP32, penalty_scale=1.0,
                 device=0, stream=None, comm=None, kernel=KERNEL_FULL, basis=None, dist_min_dofs=0,
                 boundary_penalty_scale=1.0):
        import torch
        self.lib = load()
        cfg = Config()
        self.lib.ipmg_config_default(ctypes.byref(cfg))
        cfg.dim, cfg.degree, cfg.n_levels, cfg.h0 = dim, degree, n_levels, h0
        cc = coarse_cells or (2,) * dim
        for a in range(3):
            cfg.coarse_cells[a] = cc[a] if a < dim else 1
        cfg.smoother, cfg.additive_omega = smoother, additive_omega
        cfg.post_smooth_reverse, cfg.vcycle_precision = post_smooth_reverse, vcycle_precision
        cfg.penalty_scale, cfg.device = penalty_scale, device
        cfg.kernel = kernel
        cfg.dist_min_dofs = dist_min_dofs
        cfg.boundary_penalty_scale = boundary_penalty_scale
        # the clamped kernel lives on the Hermite-type basis (the whole hierarchy)
        cfg.basis = (BASIS_HERMITE if kernel == KERNEL_CLAMPED else BASIS_LAGRANGE) if basis is None else basis
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        cfg.cuda_stream = ctypes.c_void_p(stream.cuda_stream)
        cfg.comm = comm.ptr if comm is not None else None
        self.comm = comm
        self.cfg = cfg
        h = ctypes.c_void_p()
        st = self.lib.ipmg_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != IPMG_OK:
            raise IpmgError(st, self.lib.ipmg_last_error(None).decode())
        self.h = h
        self.dim, self.degree, self.n_levels = dim, degree, n_levels

    def close(self):
        if getattr(self, "h", None):
            self.lib.ipmg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != IPMG_OK:
            raise IpmgError(st, "%s: %s" % (what, self.lib.ipmg_last_error(self.h).decode()))

    def level_info(self, level):
        n = ctypes.c_int64(0)
        cells = (ctypes.c_int * 3)()
        hs = ctypes.c_double(0)
        self._check(self.lib.ipmg_level_info(self.h, level, ctypes.byref(n), cells, ctypes.byref(hs)),
                    "level_info")
        return n.value, tuple(cells), hs.value

    def level_partition(self, level):
        """(distributed, zoff, nglob) of a level on this rank."""
        d, z, g = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
        self._check(self.lib.ipmg_level_partition(self.h, level, ctypes.byref(d), ctypes.byref(z), ctypes.byref(g)),
                    "level_partition")
        return d.value, z.value, g.value

    def ndofs(self, level):
        return self.level_info(level)[0]

    @staticmethod
    def _prec(t):
        import torch
        if t.dtype == torch.float64:
            return FP64
        if t.dtype == torch.float32:
            return FP32
        raise TypeError("tensor must be float64 or float32")

    def _vec(self, t, level, prec=None):
        if t is None:
            return
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("vectors must be contiguous CUDA tensors")
        if t.numel() != self.ndofs(level):
            raise ValueError("vector length %d != level %d size %d" % (t.numel(), level, self.ndofs(level)))
        if prec is not None and self._prec(t) != prec:
            raise TypeError("precision mismatch")

    def vmult(self, level, x, y):
        p = self._prec(x)
        self._vec(x, level, p), self._vec(y, level, p)
        self._check(self.lib.ipmg_vmult(self.h, level, p, _ptr(x), _ptr(y)), "vmult")

    def smooth(self, level, x, b, reverse=False):
        p = self._prec(x)
        self._vec(x, level, p), self._vec(b, level, p)
        self._check(self.lib.ipmg_smooth(self.h, level, p, _ptr(x), _ptr(b), int(reverse)), "smooth")

    def smooth_colour(self, level, x_in, b, x_out, colour):
        p = self._prec(b)
        self._vec(x_in, level, p), self._vec(b, level, p), self._vec(x_out, level, p)
        self._check(self.lib.ipmg_smooth_colour(self.h, level, p, _ptr(x_in), _ptr(b), _ptr(x_out), colour),
                    "smooth_colour")

    def residual_restrict(self, fine_level, x, b, r_c):
        p = self._prec(b)
        self._vec(x, fine_level, p), self._vec(b, fine_level, p), self._vec(r_c, fine_level - 1, p)
        self._check(self.lib.ipmg_residual_restrict(self.h, fine_level, p, _ptr(x), _ptr(b), _ptr(r_c)),
                    "residual_restrict")

    def prolongate_add(self, fine_level, e_c, x_f):
        p = self._prec(x_f)
        self._vec(e_c, fine_level - 1, p), self._vec(x_f, fine_level, p)
        self._check(self.lib.ipmg_prolongate_add(self.h, fine_level, p, _ptr(e_c), _ptr(x_f)), "prolongate_add")

    def coarse_solve(self, b0, x0):
        p = self._prec(b0)
        self._vec(b0, 0, p), self._vec(x0, 0, p)
        self._check(self.lib.ipmg_coarse_solve(self.h, p, _ptr(b0), _ptr(x0)), "coarse_solve")

    def vcycle(self, r, z):
        L = self.n_levels - 1
        self._vec(r, L, FP64), self._vec(z, L, FP64)
        self._check(self.lib.ipmg_vcycle(self.h, _ptr(r), _ptr(z)), "vcycle")

    def cg_solve(self, b, x, rtol=1e-8, max_it=100):
        """PCG (ipmg_cg_solve).  Returns dict(iterations, nu, rel_residual, seconds, history, converged)."""
        return self._solve(self.lib.ipmg_cg_solve, "cg_solve", b, x, rtol, max_it)

    def gmres_solve(self, b, x, rtol=1e-8, max_it=100):
        """Right-preconditioned GMRES (ipmg_gmres_solve); same result dict as cg_solve."""
        return self._solve(self.lib.ipmg_gmres_solve, "gmres_solve", b, x, rtol, max_it)

    def _solve(self, fn, what, b, x, rtol, max_it):
        L = self.n_levels - 1
        self._vec(b, L, FP64), self._vec(x, L, FP64)
        cap = max_it + 2
        hist = (ctypes.c_double * cap)()
        info = SolveInfo()
        info.history = hist
        info.history_cap = cap
        st = fn(self.h, _ptr(b), _ptr(x), rtol, max_it, ctypes.byref(info))
        if st not in (IPMG_OK, IPMG_ERR_NOT_CONVERGED):
            self._check(st, what)
        return dict(iterations=info.iterations, nu=info.nu, rel_residual=info.rel_residual,
                    seconds=info.seconds, history=list(hist[:info.history_len]),
                    converged=(st == IPMG_OK))

    def rhs(self, level, b, kind=0):
        """b = int f phi_i: kind 0 f == 1, kind 1 the manufactured sin solution (ipmg_rhs)."""
        self._vec(b, level, FP64)
        self._check(self.lib.ipmg_rhs(self.h, level, kind, _ptr(b)), "rhs")

    def to_cellwise(self, level, x_lib, x_cw):
        p = self._prec(x_lib)
        self._vec(x_lib, level, p), self._vec(x_cw, level, p)
        self._check(self.lib.ipmg_to_cellwise(self.h, level, p, _ptr(x_lib), _ptr(x_cw)), "to_cellwise")

    def from_cellwise(self, level, x_cw, x_lib):
        p = self._prec(x_cw)
        self._vec(x_lib, level, p), self._vec(x_cw, level, p)
        self._check(self.lib.ipmg_from_cellwise(self.h, level, p, _ptr(x_cw), _ptr(x_lib)), "from_cellwise")

    def profile(self, enable=True):
        self._check(self.lib.ipmg_profile(self.h, int(enable)), "profile")

    def profile_read(self, kernel_class):
        """(launches, total_ms, total_algorithmic_bytes) of a kernel class on the finest level."""
        n = ctypes.c_int64(0)
        ms = ctypes.c_double(0)
        by = ctypes.c_double(0)
        cls = KERNEL_CLASSES.get(kernel_class, kernel_class)
        self._check(self.lib.ipmg_profile_read(self.h, cls, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)),
                    "profile_read")
        return n.value, ms.value, by.value

    def launch_count(self):
        n = ctypes.c_int64(0)
        self._check(self.lib.ipmg_launch_count(self.h, ctypes.byref(n)), "launch_count")
        return n.value

    def synchronize(self):
        self._check(self.lib.ipmg_synchronize(self.h), "synchronize")
