"""paper_2506_05793_b200 -- B200-native FastILU (arXiv 2506.05793, Section 5).

Thin ctypes binding over the C ABI in include/fastilu.h (libfastilu_b200.so).  This module only
marshals arguments: every step of the hot path runs in the library's CUDA kernels, and there is
no CPU fallback -- if the shared library is missing the import of any entry point raises.
PyTorch is used by callers for device memory and streams (tensor.data_ptr(), stream handles).

ABI names are re-exported unchanged (fastilu_create, fastilu_compute, fastilu_apply, ...); the
`FastILU` class is a convenience wrapper around one handle.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libfastilu_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "fastilu.h")

STATUS_NAMES = ["OK", "INVALID_ARG", "BAD_MATRIX", "MISSING_DIAG", "ZERO_DIAG", "ZERO_PIVOT",
                "STATE", "CUDA", "NCCL", "OOM", "UNSUPPORTED"]
COMM_NONE, COMM_NCCL, COMM_LOCAL = 0, 1, 2


class FastILUError(RuntimeError):
    def __init__(self, code: int, index: int = -1, what: str = ""):
        self.code = code
        self.status = STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else str(code)
        self.index = index
        super().__init__(f"{what}: FASTILU_ERR_{self.status} (index {index})")


class Options(C.Structure):
    """Mirror of fastilu_options (include/fastilu.h)."""
    _fields_ = [("omega", C.c_double), ("omega_tri", C.c_double), ("device", C.c_int),
                ("stream", C.c_void_p), ("num_threads", C.c_int), ("rank", C.c_int),
                ("nranks", C.c_int), ("comm_kind", C.c_int), ("nccl_unique_id", C.c_void_p),
                ("group", C.c_void_p), ("global_n", C.c_int64), ("row_begin", C.c_int64),
                ("n_lead", C.c_int64), ("shift", C.c_double)]


I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
I8P = C.POINTER(C.c_int8)
F64P = C.POINTER(C.c_double)
H = C.c_void_p

_SIGS = {
    "fastilu_default_options": (None, [C.POINTER(Options)]),
    "fastilu_create": (C.c_int, [C.POINTER(H), C.c_int64, I64P, I32P, F64P, C.c_int,
                                 C.POINTER(Options)]),
    "fastilu_required_lead_rows": (C.c_int64, [C.c_int64, C.c_int]),
    "fastilu_set_values": (C.c_int, [H, F64P]),
    "fastilu_set_values_device": (C.c_int, [H, C.c_void_p]),
    "fastilu_compute": (C.c_int, [H, C.c_int]),
    "fastilu_compute_tol": (C.c_int, [H, C.c_double, C.c_int, C.POINTER(C.c_int)]),
    "fastilu_compute_warmup": (C.c_int, [H, C.c_int]),
    "fastilu_compute_async": (C.c_int, [H, C.c_int]),
    "fastilu_compute_async_block": (C.c_int, [H, C.c_int, C.c_int]),
    "fastilu_compute_host": (C.c_int, [H, F64P, C.c_int]),
    "fastilu_solve_host": (C.c_int, [H, F64P, C.c_int, F64P, F64P, C.c_int]),
    "fastilu_apply": (C.c_int, [H, C.c_void_p, C.c_void_p, C.c_int]),
    "fastilu_apply_host": (C.c_int, [H, F64P, F64P, C.c_int]),
    "fastilu_destroy": (C.c_int, [H]),
    "fastilu_gmres": (C.c_int, [H, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int,
                                C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "fastilu_get_sizes": (C.c_int, [H, I64P, I64P, I64P]),
    "fastilu_get_device": (C.c_int, [H, C.POINTER(C.c_int)]),
    "fastilu_get_pattern": (C.c_int, [H, I64P, I32P, I8P]),
    "fastilu_get_factors": (C.c_int, [H, F64P, F64P]),
    "fastilu_set_factors": (C.c_int, [H, F64P, F64P]),
    "fastilu_get_residual_history": (C.c_int, [H, F64P, C.c_int, C.POINTER(C.c_int)]),
    "fastilu_get_timings": (C.c_int, [H, F64P]),
    "fastilu_get_sweep_split": (C.c_int, [H, F64P]),
    "fastilu_get_info": (C.c_int, [H, C.c_char_p, C.c_int]),
    "fastilu_status_string": (C.c_char_p, [C.c_int]),
    "fastilu_error_index": (C.c_int64, [H]),
    "fastilu_symbolic": (C.c_int, [C.c_int64, I64P, I32P, C.c_int, C.c_int, I64P, I64P, I32P,
                                   I8P, I64P]),
    "fastilu_symbolic_window": (C.c_int, [C.c_int64, I64P, I32P, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_int64, C.c_int, C.c_int, I64P, I64P, I32P, I8P,
                                          I64P]),
    "fastilu_group_create": (C.c_int, [C.POINTER(H), C.c_int]),
    "fastilu_group_destroy": (C.c_int, [H]),
    "fastilu_nccl_unique_id": (C.c_int, [C.c_void_p]),
}

_lib = None


def lib():
    """Load libfastilu_b200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2506_05793_b200.build` "
                              "(the FastILU hot path exists only as CUDA kernels)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def header_functions() -> list[str]:
    """Function names declared in include/fastilu.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fastilu_[a-z_0-9]+)\s*\(", txt)))


def _p(a, t):
    return a.ctypes.data_as(t)


def _check(code, what, h=None):
    if code != 0:
        idx = lib().fastilu_error_index(h) if h else -1
        raise FastILUError(code, idx, what)


def _ptr(t):
    """Device pointer of a torch tensor or an int."""
    return t if isinstance(t, int) else t.data_ptr()


def _host_in(a, count: int, what: str):
    """A host input as a C-contiguous float64 array of exactly `count` entries (the C side reads
    exactly that many)."""
    v = np.ascontiguousarray(a, dtype=np.float64)
    if v.ndim != 1 or v.shape[0] != count:
        raise ValueError(f"{what}: expected {count} float64 values, got shape {v.shape}")
    return v


def _host_out(out, count: int, what: str):
    """A caller-supplied host output buffer: float64, C-contiguous, writeable, `count` entries."""
    if out is None:
        return np.empty(count, dtype=np.float64)
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.ndim == 1 and
            out.shape[0] == count and out.flags.c_contiguous and out.flags.writeable):
        raise ValueError(f"{what}: `out` must be a writeable C-contiguous float64 array of "
                         f"{count} entries")
    return out


def _dev_arg(t, count: int, device: int, what: str):
    """Device pointer of a CUDA tensor after checking dtype (float64), device, contiguity and
    length; raw integer pointers are passed through unchecked (the caller's contract)."""
    if isinstance(t, int):
        return t
    if str(getattr(t, "dtype", "")) != "torch.float64":
        raise ValueError(f"{what}: expected a float64 tensor, got {getattr(t, 'dtype', type(t))}")
    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{what}: expected a CUDA tensor")
    if device >= 0 and t.device.index != device:
        raise ValueError(f"{what}: tensor on cuda:{t.device.index}, handle on cuda:{device}")
    if not t.is_contiguous() or t.numel() != count:
        raise ValueError(f"{what}: expected a contiguous tensor of {count} entries, got "
                         f"{tuple(t.shape)}")
    return t.data_ptr()


# ---------------------------------------------------------------- ABI names (thin wrappers)
def fastilu_default_options() -> Options:
    o = Options()
    lib().fastilu_default_options(C.byref(o))
    return o


def fastilu_required_lead_rows(bandwidth: int, level_k: int) -> int:
    return int(lib().fastilu_required_lead_rows(int(bandwidth), int(level_k)))


def fastilu_symbolic(row_ptr, col_idx, level_k: int, num_threads: int = 0):
    """Host-only symbolic ILU(k) -> (row_ptr int64, col_idx int32, level int8)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    n = rp.shape[0] - 1
    nnz = C.c_int64(0)
    bad = C.c_int64(-1)
    st = lib().fastilu_symbolic(n, _p(rp, I64P), _p(ci, I32P), int(level_k), int(num_threads),
                                C.byref(nnz), None, None, None, C.byref(bad))
    if st:
        raise FastILUError(st, bad.value, "fastilu_symbolic")
    orp = np.empty(n + 1, dtype=np.int64)
    oci = np.empty(max(nnz.value, 1), dtype=np.int32)
    olev = np.empty(max(nnz.value, 1), dtype=np.int8)
    st = lib().fastilu_symbolic(n, _p(rp, I64P), _p(ci, I32P), int(level_k), int(num_threads),
                                C.byref(nnz), _p(orp, I64P), _p(oci, I32P), _p(olev, I8P),
                                C.byref(bad))
    if st:
        raise FastILUError(st, bad.value, "fastilu_symbolic")
    return orp, oci[:nnz.value], olev[:nnz.value]


def fastilu_symbolic_window(row_ptr, col_idx, row0: int, ncols: int, out_begin: int,
                            out_end: int, level_k: int, num_threads: int = 0):
    """Host-only symbolic ILU(k) of global rows [out_begin, out_end) from the supplied rows
    [row0, row0 + nrows) -> (row_ptr, col_idx (global), level)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    nrows = rp.shape[0] - 1
    nnz = C.c_int64(0)
    bad = C.c_int64(-1)
    args = (nrows, _p(rp, I64P), _p(ci, I32P), int(row0), int(ncols), int(out_begin),
            int(out_end), int(level_k), int(num_threads), C.byref(nnz))
    st = lib().fastilu_symbolic_window(*args, None, None, None, C.byref(bad))
    if st:
        raise FastILUError(st, bad.value, "fastilu_symbolic_window")
    no = out_end - out_begin
    orp = np.empty(no + 1, dtype=np.int64)
    oci = np.empty(max(nnz.value, 1), dtype=np.int32)
    olev = np.empty(max(nnz.value, 1), dtype=np.int8)
    st = lib().fastilu_symbolic_window(*args, _p(orp, I64P), _p(oci, I32P), _p(olev, I8P),
                                       C.byref(bad))
    if st:
        raise FastILUError(st, bad.value, "fastilu_symbolic_window")
    return orp, oci[:nnz.value], olev[:nnz.value]


def fastilu_group_create(nranks: int):
    g = H()
    st = lib().fastilu_group_create(C.byref(g), int(nranks))
    if st:
        raise FastILUError(st, -1, "fastilu_group_create")
    return g


def fastilu_group_destroy(g) -> None:
    lib().fastilu_group_destroy(g)


def fastilu_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().fastilu_nccl_unique_id(buf)
    if st:
        raise FastILUError(st, -1, "fastilu_nccl_unique_id")
    return buf.raw


def fastilu_status_string(code: int) -> str:
    return lib().fastilu_status_string(int(code)).decode()


class FastILU:
    """One fastilu_handle: create (symbolic + layouts) / compute / apply / destroy."""

    def __init__(self, row_ptr, col_idx, values, level_k: int, *, omega: float = 1.0,
                 omega_tri: float = 1.0, device: int = -1, stream=None, num_threads: int = 0,
                 rank: int = 0, nranks: int = 1, comm_kind: int = COMM_NONE,
                 nccl_unique_id: bytes | None = None, group=None, global_n: int = -1,
                 row_begin: int = 0, n_lead: int = 0, n: int | None = None,
                 shift: float = 0.0):
        L = lib()
        self._h = H()
        o = fastilu_default_options()
        o.omega, o.omega_tri, o.device = float(omega), float(omega_tri), int(device)
        o.stream = stream
        o.num_threads = int(num_threads)
        o.rank, o.nranks, o.comm_kind = int(rank), int(nranks), int(comm_kind)
        self._uid = C.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id else None
        o.nccl_unique_id = C.cast(self._uid, C.c_void_p) if self._uid is not None else None
        o.group = group
        o.global_n, o.row_begin, o.n_lead = int(global_n), int(row_begin), int(n_lead)
        o.shift = float(shift)
        self._rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self._ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        if self._rp.ndim != 1 or self._rp.shape[0] < 1:
            raise ValueError("row_ptr: expected a 1-D array of n + 1 offsets")
        self._nnz_in = int(self._rp[-1])  # values the C side reads (lead rows included)
        if self._ci.ndim != 1 or self._ci.shape[0] < self._nnz_in:
            raise ValueError(f"col_idx: expected {self._nnz_in} entries, got {self._ci.shape}")
        vals = None if values is None else _host_in(values, self._nnz_in, "values")
        nrows = (self._rp.shape[0] - 1 - int(n_lead)) if n is None else int(n)
        st = L.fastilu_create(C.byref(self._h), nrows, _p(self._rp, I64P), _p(self._ci, I32P),
                              None if vals is None else _p(vals, F64P), int(level_k),
                              C.byref(o))
        if st:
            idx = L.fastilu_error_index(self._h)
            L.fastilu_destroy(self._h)
            self._h = None
            raise FastILUError(st, idx, "fastilu_create")
        n_, s_, a_ = C.c_int64(), C.c_int64(), C.c_int64()
        L.fastilu_get_sizes(self._h, C.byref(n_), C.byref(s_), C.byref(a_))
        self.n, self.nnz_S, self.nnz_A = n_.value, s_.value, a_.value
        self.level_k = level_k
        d_ = C.c_int(-1)
        L.fastilu_get_device(self._h, C.byref(d_))
        self.device = d_.value

    # -- numeric phase
    def set_values(self, values):
        v = _host_in(values, self._nnz_in, "values")
        _check(lib().fastilu_set_values(self._h, _p(v, F64P)), "fastilu_set_values", self._h)

    def set_values_device(self, values_dev):
        _check(lib().fastilu_set_values_device(
            self._h, _dev_arg(values_dev, self._nnz_in, self.device, "values")),
            "fastilu_set_values_device", self._h)

    def compute(self, nsweeps: int):
        _check(lib().fastilu_compute(self._h, int(nsweeps)), "fastilu_compute", self._h)

    def compute_host(self, values, nsweeps: int):
        """fastilu_compute_host: new host values + nsweeps sweeps, upload pipelined with the
        numeric phase (pass a pinned array for overlap)."""
        v = _host_in(values, self._nnz_in, "values")
        _check(lib().fastilu_compute_host(self._h, _p(v, F64P), int(nsweeps)),
               "fastilu_compute_host", self._h)

    def solve_host(self, values, nsweeps: int, b, ntrisweeps: int, out=None):
        """fastilu_solve_host: new host values, nsweeps sweeps, x = M^-1 b (host arrays)."""
        v = _host_in(values, self._nnz_in, "values")
        bb = _host_in(b, self.n, "b")
        x = _host_out(out, self.n, "solve_host")
        _check(lib().fastilu_solve_host(self._h, _p(v, F64P), int(nsweeps), _p(bb, F64P),
                                        _p(x, F64P), int(ntrisweeps)), "fastilu_solve_host",
               self._h)
        return x

    def compute_async(self, nsweeps: int, nnz_per_thread: int | None = None):
        """The paper's asynchronous in-place sweeps (non-deterministic; fastilu_compute_async),
        optionally with its "Block Size" option (nonzeros per thread)."""
        if nnz_per_thread is None:
            _check(lib().fastilu_compute_async(self._h, int(nsweeps)), "fastilu_compute_async",
                   self._h)
        else:
            _check(lib().fastilu_compute_async_block(self._h, int(nsweeps), int(nnz_per_thread)),
                   "fastilu_compute_async_block", self._h)

    def compute_warmup(self, nsweeps: int):
        """Warm-up option: FastILU(0..k) with nsweeps each (fastilu_compute_warmup)."""
        _check(lib().fastilu_compute_warmup(self._h, int(nsweeps)), "fastilu_compute_warmup",
               self._h)

    def compute_tol(self, rtol: float, max_sweeps: int = 100) -> int:
        """Sweeps until r(s-1) <= rtol ||Ahat|_S||_F (or max_sweeps); returns s."""
        d = C.c_int(0)
        _check(lib().fastilu_compute_tol(self._h, float(rtol), int(max_sweeps), C.byref(d)),
               "fastilu_compute_tol", self._h)
        return d.value

    def apply(self, b, x, ntrisweeps: int):
        """b, x: float64 CUDA tensors (or raw device pointers) of length n; x may alias b."""
        _check(lib().fastilu_apply(self._h, _dev_arg(b, self.n, self.device, "b"),
                                   _dev_arg(x, self.n, self.device, "x"), int(ntrisweeps)),
               "fastilu_apply", self._h)

    def apply_host(self, b, ntrisweeps: int, out=None):
        b = _host_in(b, self.n, "b")
        x = _host_out(out, self.n, "apply_host")
        _check(lib().fastilu_apply_host(self._h, _p(b, F64P), _p(x, F64P), int(ntrisweeps)),
               "fastilu_apply_host", self._h)
        return x

    def gmres(self, b, x, restart: int = 60, rtol: float = 1e-6, max_iters: int = 1000,
              ntrisweeps: int = 5):
        """Right-preconditioned GMRES(restart) on A x = b (device arrays); returns
        (inner iterations, relative residual)."""
        it = C.c_int(0)
        rr = C.c_double(0.0)
        _check(lib().fastilu_gmres(self._h, _dev_arg(b, self.n, self.device, "b"),
                                   _dev_arg(x, self.n, self.device, "x"), int(restart), float(rtol),
                                   int(max_iters), int(ntrisweeps), C.byref(it), C.byref(rr)),
               "fastilu_gmres", self._h)
        return it.value, rr.value

    # -- introspection
    def pattern(self):
        rp = np.empty(self.n + 1, dtype=np.int64)
        ci = np.empty(max(self.nnz_S, 1), dtype=np.int32)
        lev = np.empty(max(self.nnz_S, 1), dtype=np.int8)
        _check(lib().fastilu_get_pattern(self._h, _p(rp, I64P), _p(ci, I32P), _p(lev, I8P)),
               "fastilu_get_pattern", self._h)
        return rp, ci[:self.nnz_S], lev[:self.nnz_S]

    def factors(self):
        v = np.empty(max(self.nnz_S, 1))
        s = np.empty(max(self.n, 1))
        _check(lib().fastilu_get_factors(self._h, _p(v, F64P), _p(s, F64P)),
               "fastilu_get_factors", self._h)
        return v[:self.nnz_S], s[:self.n]

    def set_factors(self, vals, s):
        """fastilu_set_factors: external factors (S row order of the owned rows, as factors()
        returns them) and scaling vector s; apply / gmres then use them (config 5 arm B)."""
        v = _host_in(vals, self.nnz_S, "vals")
        sv = _host_in(s, self.n, "s")
        _check(lib().fastilu_set_factors(self._h, _p(v, F64P), _p(sv, F64P)),
               "fastilu_set_factors", self._h)

    def residual_history(self, cap: int = 4096):
        h = np.empty(cap)
        c = C.c_int(0)
        _check(lib().fastilu_get_residual_history(self._h, _p(h, F64P), cap, C.byref(c)),
               "fastilu_get_residual_history", self._h)
        return h[:c.value].copy()

    def timings(self):
        t = np.zeros(3)
        _check(lib().fastilu_get_timings(self._h, _p(t, F64P)), "fastilu_get_timings", self._h)
        u = np.zeros(2)
        _check(lib().fastilu_get_sweep_split(self._h, _p(u, F64P)), "fastilu_get_sweep_split",
               self._h)
        return {"init_ms": t[0], "sweeps_ms": t[1], "apply_ms": t[2], "sweep1_ms": u[0],
                "sweeps_rest_ms": u[1]}

    def info(self) -> str:
        """Kernel configuration of this handle (fastilu_get_info)."""
        buf = C.create_string_buffer(1024)
        _check(lib().fastilu_get_info(self._h, buf, 1024), "fastilu_get_info", self._h)
        return buf.value.decode()

    def close(self):
        if getattr(self, "_h", None):
            lib().fastilu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
