"""Python binding of the FastDOG B200 hot path (include/fastdog.h).

Argument marshalling only: every step of the path runs in libfastdog.so
(host C++ BDD compiler + packer, sm_100a CUDA kernels).  There is no CPU
fallback: if the extension is missing, importing the solver raises.

Names follow the C ABI:  Plan (fdog_plan_*), Solver (fdog_create / iterate /
pass_ / lower_bound / get_lambda / min_marginals / finalize / ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (FDOG_LIB: another build of the same library, for same-box A/B runs)
LIB_PATH = os.environ.get("FDOG_LIB") or os.path.join(_HERE, "libfastdog.so")

STATUS = {0: "OK", 1: "EINVAL", 2: "EINFEASIBLE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ESTATE",
          7: "ETOOBIG", 8: "ENOSOLUTION"}


def ipc_handle(dev_ptr: int) -> bytes:
    """CUDA IPC handle (64 bytes) of a device allocation, e.g. an exchange region."""
    lib = load()
    buf = C.create_string_buffer(64)
    _check(lib.fdog_ipc_handle(C.c_void_p(dev_ptr), buf), "fdog_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation (peer access enabled); returns the device pointer."""
    lib = load()
    ptr = C.c_void_p()
    _check(lib.fdog_ipc_open(C.c_char_p(bytes(handle)), C.byref(ptr)), "fdog_ipc_open")
    return ptr.value


def ipc_close(dev_ptr: int):
    _check(load().fdog_ipc_close(C.c_void_p(dev_ptr)), "fdog_ipc_close")


class FastdogError(RuntimeError):
    def __init__(self, code, what, msg):
        super().__init__(f"{what}: FDOG_{STATUS.get(code, code)}: {msg}")
        self.code = code


class Problem(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("cost", C.c_void_p), ("n_cons", C.c_int32),
                ("row_ptr", C.c_void_p), ("col_var", C.c_void_p), ("col_coef", C.c_void_p),
                ("rel", C.c_void_p), ("rhs", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("precision", C.c_int32), ("device", C.c_int32), ("clamp", C.c_double),
                ("record_mm", C.c_int32), ("profile", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("nccl_unique_id", C.c_void_p), ("nccl_library", C.c_char_p),
                ("stream", C.c_void_p), ("host_threads", C.c_int32),
                ("row_owner", C.c_void_p), ("lifted", C.c_int32),
                ("dev_alloc", C.c_void_p), ("dev_free", C.c_void_p), ("alloc_ctx", C.c_void_p)]


# fdog_options::dev_alloc / dev_free: the solver's device memory from torch's
# caching allocator, stream-ordered on the solver's stream.
_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p)
_live_solvers = None  # weak set of solvers holding torch memory (closed at exit, before torch)


@_ALLOC_FN
def _torch_alloc(nbytes, device, stream, ctx):
    # The block is associated with torch's current stream, not the solver's
    # own one: the library synchronises its stream before it returns memory,
    # so the block can serve any later allocation on that stream -- e.g. the
    # next solver's (blocks of a destroyed solver-owned stream would never be
    # reused, and a fresh 2.7 GB cudaMalloc costs MRF-LP's create ~55 ms).
    # (a block torch freed on that stream may still be in use by its queued
    # work; the solver's stream is another one, so that work is waited for)
    import torch
    try:
        cur = torch.cuda.current_stream(int(device))
        ptr = torch.cuda.caching_allocator_alloc(int(nbytes), int(device), cur)
        cur.synchronize()
        return ptr
    except (RuntimeError, torch.OutOfMemoryError):
        return None  # -> FDOG_ENOMEM


@_FREE_FN
def _torch_free(ptr, device, stream, ctx):
    import torch
    torch.cuda.caching_allocator_delete(int(ptr))


def _torch_memory(solver):
    """Register a solver whose memory comes from torch; returns the two callbacks."""
    global _live_solvers
    if _live_solvers is None:
        import atexit
        import weakref
        import torch  # noqa: F401  (imported first: its exit handlers run after ours)
        _live_solvers = weakref.WeakSet()
        atexit.register(lambda: [x.close() for x in list(_live_solvers)])
    _live_solvers.add(solver)
    return C.cast(_torch_alloc, C.c_void_p), C.cast(_torch_free, C.c_void_p)


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("bdds", "nodes", "arcs", "slots", "vars_local", "vars_shared",
                                          "free_vars", "shapes", "tiles", "tiles_shared_topology",
                                          "padded_slots", "device_bytes", "launches")] + \
               [("max_hops", C.c_int32), ("max_width", C.c_int32), ("staged_tiles", C.c_int64),
                ("sweep_grid", C.c_int32), ("sweep_block", C.c_int32), ("sweep_smem_per_warp", C.c_int64),
                ("sweep_streaming", C.c_int32), ("h2d_bytes", C.c_int64),
                ("fused_small", C.c_int32), ("sweep_recompute", C.c_int32), ("tile_pairs", C.c_int64),
                ("interior_tiles", C.c_int64), ("coop_tiles", C.c_int64), ("tmem_cols", C.c_int32)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class PrimalOptions(C.Structure):
    _fields_ = [("delta0", C.c_double), ("alpha", C.c_double), ("inner", C.c_int32), ("max_rounds", C.c_int32),
                ("seed", C.c_uint64), ("omega", C.c_double), ("keep_state", C.c_int32)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char_p), ("ms", C.c_double), ("launches", C.c_int64),
                ("bytes_per_launch", C.c_double)]


EXPORTS = ["fdog_default_options", "fdog_plan_create", "fdog_plan_destroy", "fdog_plan_stats", "fdog_plan_slot_map",
           "fdog_plan_tiles", "fdog_plan_digest", "fdog_debug_trace",
           "fdog_plan_bdd", "fdog_plan_owner", "fdog_plan_shared_vars", "fdog_create",
           "fdog_create_from_plan", "fdog_destroy", "fdog_iterate", "fdog_pass", "fdog_pass_seq", "fdog_iterate_seq",
           "fdog_lower_bound",
           "fdog_finalize", "fdog_finalize_averaged", "fdog_num_slots", "fdog_slot_index", "fdog_get_lambda",
           "fdog_get_deferred", "fdog_get_lifted", "fdog_min_marginals", "fdog_set_state", "fdog_stats",
           "fdog_profile", "fdog_profile_reset", "fdog_profile_enable", "fdog_pass_begin", "fdog_pass_end",
           "fdog_exchange_size", "fdog_exchange_read", "fdog_exchange_write", "fdog_exchange_region",
           "fdog_set_peer_regions", "fdog_peer_error", "fdog_ipc_handle", "fdog_ipc_open", "fdog_ipc_close",
           "fdog_default_primal_options",
           "fdog_primal_step", "fdog_round_primal", "fdog_last_error", "fdog_version"]

_lib = None


def load():
    """Load libfastdog.so (built by __graft_entry__.build() / make); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                          "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
    sig = {
        "fdog_default_options": ([P], None),
        "fdog_plan_create": ([P, P, C.POINTER(P)], C.c_int),
        "fdog_plan_destroy": ([P], None),
        "fdog_plan_stats": ([P, P], C.c_int),
        "fdog_plan_bdd": ([P, i32, P, P, P, P, P, i32, i32], C.c_int),
        "fdog_plan_owner": ([P, P, i64], C.c_int),
        "fdog_plan_slot_map": ([P, P, i64], C.c_int),
        "fdog_plan_tiles": ([P, P, i64, P], C.c_int),
        "fdog_plan_digest": ([P, P], C.c_int),
        "fdog_debug_trace": ([P, P, i64, P], C.c_int),
        "fdog_plan_shared_vars": ([P, P, i64, P], C.c_int),
        "fdog_create": ([P, P, C.POINTER(P)], C.c_int),
        "fdog_create_from_plan": ([P, P, C.POINTER(P)], C.c_int),
        "fdog_destroy": ([P], None),
        "fdog_iterate": ([P, i32, dbl], C.c_int),
        "fdog_pass": ([P, i32, dbl], C.c_int),
        "fdog_pass_seq": ([P, i32, dbl], C.c_int),
        "fdog_iterate_seq": ([P, i32, dbl], C.c_int),
        "fdog_lower_bound": ([P, P], C.c_int),
        "fdog_finalize": ([P], C.c_int),
        "fdog_finalize_averaged": ([P], C.c_int),
        "fdog_num_slots": ([P, P], C.c_int),
        "fdog_slot_index": ([P, P, P, i64], C.c_int),
        "fdog_get_lambda": ([P, P, i64], C.c_int),
        "fdog_get_deferred": ([P, P, i64], C.c_int),
        "fdog_get_lifted": ([P, P, P, i64], C.c_int),
        "fdog_min_marginals": ([P, P, P, i64], C.c_int),
        "fdog_set_state": ([P, P, P, i64], C.c_int),
        "fdog_stats": ([P, P], C.c_int),
        "fdog_profile": ([P, P, i32, P], C.c_int),
        "fdog_profile_reset": ([P], C.c_int),
        "fdog_profile_enable": ([P, i32], C.c_int),
        "fdog_pass_begin": ([P, i32, dbl], C.c_int),
        "fdog_pass_end": ([P, i32, dbl], C.c_int),
        "fdog_exchange_size": ([P, P], C.c_int),
        "fdog_exchange_read": ([P, P, i64], C.c_int),
        "fdog_exchange_write": ([P, P, i64], C.c_int),
        "fdog_exchange_region": ([P, C.POINTER(P), P], C.c_int),
        "fdog_set_peer_regions": ([P, i32, P, dbl], C.c_int),
        "fdog_peer_error": ([P, P], C.c_int),
        "fdog_ipc_handle": ([P, P], C.c_int),
        "fdog_ipc_open": ([P, C.POINTER(P)], C.c_int),
        "fdog_ipc_close": ([P], C.c_int),
        "fdog_default_primal_options": ([P], None),
        "fdog_primal_step": ([P, i32, dbl, C.c_uint64, P, P, i64], C.c_int),
        "fdog_round_primal": ([P, P, P, i64, P, P], C.c_int),
        "fdog_last_error": ([], C.c_char_p),
        "fdog_version": ([], C.c_int32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc, what):
    if rc:
        raise FastdogError(rc, what, load().fdog_last_error().decode())


class _ProblemArrays:
    """Keeps contiguous host copies alive and builds the fdog_problem struct."""

    def __init__(self, problem):
        self.arrays = [np.ascontiguousarray(problem.cost, dtype=np.float64),
                       np.ascontiguousarray(problem.row_ptr, dtype=np.int64),
                       np.ascontiguousarray(problem.col_var, dtype=np.int32),
                       np.ascontiguousarray(problem.col_coef, dtype=np.int32),
                       np.ascontiguousarray(problem.rel, dtype=np.int8),
                       np.ascontiguousarray(problem.rhs, dtype=np.int64)]
        c, rp, cv, cc, rel, rhs = self.arrays
        self.struct = Problem(int(problem.n_vars), _ptr(c), int(rp.size - 1), _ptr(rp), _ptr(cv),
                              _ptr(cc), _ptr(rel), _ptr(rhs))


def make_options(precision=32, device=0, clamp=0.0, record_mm=False, profile=False, rank=0, world=1,
                 nccl_unique_id=None, nccl_library=None, stream=None, host_threads=0, row_owner=None,
                 lifted=False):
    lib = load()
    o = Options()
    lib.fdog_default_options(C.byref(o))
    o.precision = int(precision)
    o.device = int(device)
    o.clamp = float(clamp)
    o.record_mm = int(bool(record_mm))
    o.profile = int(bool(profile))
    o.rank = int(rank)
    o.world = int(world)
    o._uid = None
    if nccl_unique_id is not None:
        o._uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
        o.nccl_unique_id = C.cast(o._uid, C.c_void_p)
    o._lib = nccl_library.encode() if nccl_library else None
    o.nccl_library = o._lib
    o.stream = stream
    o.host_threads = int(host_threads)
    o._owner = None
    if row_owner is not None:
        o._owner = np.ascontiguousarray(row_owner, dtype=np.int32)
        o.row_owner = o._owner.ctypes.data
    o.lifted = int(bool(lifted))
    return o


class Plan:
    """Host-side compiled + packed problem (no GPU needed)."""

    def __init__(self, problem, rank=0, world=1, host_threads=0, precision=32, row_owner=None, lifted=False):
        lib = load()
        self._pa = _ProblemArrays(problem)
        self._opts = make_options(precision=precision, rank=rank, world=world, host_threads=host_threads,
                                  row_owner=row_owner, lifted=lifted)
        h = C.c_void_p()
        _check(lib.fdog_plan_create(C.byref(self._pa.struct), C.byref(self._opts), C.byref(h)),
               "fdog_plan_create")
        self._h = h
        self._lib = lib
        self.n_cons = int(problem.row_ptr.size - 1)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fdog_plan_destroy(self._h)
            self._h = None

    __del__ = close

    def stats(self) -> dict:
        s = Stats()
        _check(self._lib.fdog_plan_stats(self._h, C.byref(s)), "fdog_plan_stats")
        return s.as_dict()

    def bdd(self, j):
        """(hop_start, lo, hi) of row j; codes: node index, -1 bottom, -2 top."""
        k = C.c_int32(); n = C.c_int32()
        rc = self._lib.fdog_plan_bdd(self._h, int(j), C.byref(k), C.byref(n), None, None, None, 0, 0)
        if rc not in (0, 1):
            _check(rc, "fdog_plan_bdd")
        hs = np.empty(k.value + 1, np.int32)
        lo = np.empty(max(n.value, 1), np.int32)
        hi = np.empty(max(n.value, 1), np.int32)
        _check(self._lib.fdog_plan_bdd(self._h, int(j), C.byref(k), C.byref(n), _ptr(hs), _ptr(lo),
                                       _ptr(hi), k.value, n.value), "fdog_plan_bdd")
        return hs, lo[:n.value], hi[:n.value]

    def slot_map(self):
        """Device slot of every canonical slot (j ascending, h ascending)."""
        n = self.stats()["slots"]
        out = np.empty(max(n, 1), np.int64)
        _check(self._lib.fdog_plan_slot_map(self._h, _ptr(out), out.size), "fdog_plan_slot_map")
        return out[:n]

    def digest(self) -> int:
        """FNV-1a digest of the packed arrays and the device image."""
        x = C.c_uint64()
        _check(self._lib.fdog_plan_digest(self._h, C.byref(x)), "fdog_plan_digest")
        return x.value

    def tiles(self):
        """Tile descriptors [n, 6]: kind bits, K, lanes, valid lanes, nodes per lane, first device slot."""
        n = C.c_int64()
        _check(self._lib.fdog_plan_tiles(self._h, None, 0, C.byref(n)), "fdog_plan_tiles")
        out = np.empty((max(n.value, 1), 6), np.int64)
        _check(self._lib.fdog_plan_tiles(self._h, _ptr(out), n.value, C.byref(n)), "fdog_plan_tiles")
        return out[:n.value]

    def owner(self):
        o = np.empty(max(self.n_cons, 1), np.int32)
        _check(self._lib.fdog_plan_owner(self._h, _ptr(o), o.size), "fdog_plan_owner")
        return o[:self.n_cons]

    def shared_vars(self):
        n = C.c_int64()
        _check(self._lib.fdog_plan_shared_vars(self._h, None, 0, C.byref(n)), "fdog_plan_shared_vars")
        v = np.empty(max(n.value, 1), np.int32)
        _check(self._lib.fdog_plan_shared_vars(self._h, _ptr(v), n.value, C.byref(n)),
               "fdog_plan_shared_vars")
        return v[:n.value]


class Solver:
    """Device-resident solver (fdog_create ... fdog_destroy)."""

    def __init__(self, problem=None, *, plan: Plan | None = None, precision=32, device=0, clamp=0.0,
                 record_mm=False, profile=False, rank=0, world=1, nccl_unique_id=None,
                 nccl_library=None, stream=None, host_threads=0, row_owner=None, lifted=False,
                 allocator="torch"):
        """allocator: "torch" (device memory from torch's caching allocator, the
        default) or "cuda" (the library's own cudaMalloc)."""
        lib = load()
        self._lib = lib
        self._opts = make_options(precision, device, clamp, record_mm, profile, rank, world,
                                  nccl_unique_id, nccl_library, stream, host_threads, row_owner, lifted)
        if allocator == "torch":
            self._opts.dev_alloc, self._opts.dev_free = _torch_memory(self)
        elif allocator != "cuda":
            raise ValueError(f"allocator must be 'torch' or 'cuda', not {allocator!r}")
        h = C.c_void_p()
        if plan is not None:
            _check(lib.fdog_create_from_plan(plan._h, C.byref(self._opts), C.byref(h)),
                   "fdog_create_from_plan")
        else:
            pa = _ProblemArrays(problem)
            _check(lib.fdog_create(C.byref(pa.struct), C.byref(self._opts), C.byref(h)), "fdog_create")
        self._h = h
        self.precision = precision
        self.n_vars = int(plan._pa.struct.n_vars) if plan is not None else int(problem.n_vars)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fdog_destroy(self._h)
            self._h = None

    __del__ = close

    def iterate(self, n: int, omega: float = 0.5):
        _check(self._lib.fdog_iterate(self._h, int(n), float(omega)), "fdog_iterate")

    def pass_(self, forward: bool, omega: float = 0.5):
        _check(self._lib.fdog_pass(self._h, 1 if forward else 0, float(omega)), "fdog_pass")

    def debug_trace(self):
        """[warps, 4]: start / end (ns), tiles, SM of the last TMA-staged sweep (FDOG_TRACE=1)."""
        n = C.c_int64()
        _check(self._lib.fdog_debug_trace(self._h, None, 0, C.byref(n)), "fdog_debug_trace")
        out = np.zeros((max(n.value, 1), 4), np.uint64)
        _check(self._lib.fdog_debug_trace(self._h, _ptr(out), n.value, C.byref(n)), "fdog_debug_trace")
        return out[:n.value]

    def pass_seq(self, forward: bool, omega: float = 0.5):
        """Non-deferred (sequential) min-marginal averaging pass."""
        _check(self._lib.fdog_pass_seq(self._h, 1 if forward else 0, float(omega)), "fdog_pass_seq")

    def iterate_seq(self, n: int, omega: float = 0.5):
        _check(self._lib.fdog_iterate_seq(self._h, int(n), float(omega)), "fdog_iterate_seq")

    def lower_bound(self) -> float:
        x = C.c_double()
        _check(self._lib.fdog_lower_bound(self._h, C.byref(x)), "fdog_lower_bound")
        return x.value

    def finalize(self, averaged: bool = False):
        """P:650-652 per-slot correction, or the averaged reading of P:673."""
        if averaged:
            _check(self._lib.fdog_finalize_averaged(self._h), "fdog_finalize_averaged")
        else:
            _check(self._lib.fdog_finalize(self._h), "fdog_finalize")

    def num_slots(self) -> int:
        x = C.c_int64()
        _check(self._lib.fdog_num_slots(self._h, C.byref(x)), "fdog_num_slots")
        return x.value

    def slot_index(self):
        n = self.num_slots()
        con = np.empty(max(n, 1), np.int32); pos = np.empty(max(n, 1), np.int32)
        _check(self._lib.fdog_slot_index(self._h, _ptr(con), _ptr(pos), n), "fdog_slot_index")
        return con[:n], pos[:n]

    def _get(self, fn, out=None):
        n = self.num_slots()
        if out is None:
            out = np.empty(max(n, 1), np.float64)
        elif out.dtype != np.float64 or not out.flags.c_contiguous or out.size < n:
            raise ValueError("out: a contiguous float64 array of at least num_slots() elements")
        _check(getattr(self._lib, fn)(self._h, _ptr(out), n), fn)
        return out[:n]

    def lam(self, out=None):
        """Current lambda per slot (canonical order); `out` (optional): a
        caller-owned float64 buffer to fill, e.g. pinned host memory."""
        return self._get("fdog_get_lambda", out)

    def deferred(self, out=None):
        return self._get("fdog_get_deferred", out)

    def lifted(self):
        """(lambda^{j,0}, lambda^{j,1}) per slot, canonical order (lifted mode)."""
        n = self.num_slots()
        a, b = np.empty(max(n, 1)), np.empty(max(n, 1))
        _check(self._lib.fdog_get_lifted(self._h, _ptr(a), _ptr(b), a.size), "fdog_get_lifted")
        return a[:n], b[:n]

    def min_marginals(self):
        n = self.num_slots()
        m0 = np.empty(max(n, 1)); m1 = np.empty(max(n, 1))
        _check(self._lib.fdog_min_marginals(self._h, _ptr(m0), _ptr(m1), n), "fdog_min_marginals")
        return m0[:n], m1[:n]

    def set_state(self, lam=None, delta=None):
        n = self.num_slots()
        a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
        b = None if delta is None else np.ascontiguousarray(delta, dtype=np.float64)
        _check(self._lib.fdog_set_state(self._h, None if a is None else _ptr(a),
                                        None if b is None else _ptr(b), n), "fdog_set_state")

    def stats(self) -> dict:
        s = Stats()
        _check(self._lib.fdog_stats(self._h, C.byref(s)), "fdog_stats")
        return s.as_dict()

    def profile(self) -> dict:
        cap = 16
        arr = (KernelTime * cap)()
        n = C.c_int32()
        _check(self._lib.fdog_profile(self._h, arr, cap, C.byref(n)), "fdog_profile")
        return {arr[i].name.decode(): {"ms": arr[i].ms, "launches": arr[i].launches,
                                       "bytes_per_launch": arr[i].bytes_per_launch}
                for i in range(min(n.value, cap))}

    def profile_reset(self):
        _check(self._lib.fdog_profile_reset(self._h), "fdog_profile_reset")

    def pass_begin(self, forward: bool, omega: float = 0.5):
        _check(self._lib.fdog_pass_begin(self._h, 1 if forward else 0, float(omega)), "fdog_pass_begin")

    def pass_end(self, forward: bool, omega: float = 0.5):
        _check(self._lib.fdog_pass_end(self._h, 1 if forward else 0, float(omega)), "fdog_pass_end")

    def exchange_read(self):
        n = C.c_int64()
        _check(self._lib.fdog_exchange_size(self._h, C.byref(n)), "fdog_exchange_size")
        out = np.empty(max(n.value, 1), np.float64)
        _check(self._lib.fdog_exchange_read(self._h, _ptr(out), n.value), "fdog_exchange_read")
        return out[:n.value]

    def exchange_write(self, x):
        a = np.ascontiguousarray(x, dtype=np.float64)
        _check(self._lib.fdog_exchange_write(self._h, _ptr(a), a.size), "fdog_exchange_write")

    def exchange_region(self):
        """(device pointer, bytes) of this rank's exchange region (peer-memory mode)."""
        ptr, n = C.c_void_p(), C.c_int64()
        _check(self._lib.fdog_exchange_region(self._h, C.byref(ptr), C.byref(n)), "fdog_exchange_region")
        return ptr.value, n.value

    def set_peer_regions(self, regions, timeout_s: float = 20.0):
        """regions[k]: rank k's exchange region as a device pointer valid in this
        process (regions[rank] = own).  Passes then exchange over peer memory."""
        arr = (C.c_void_p * len(regions))(*[int(r) for r in regions])
        _check(self._lib.fdog_set_peer_regions(self._h, len(regions), arr, float(timeout_s)),
               "fdog_set_peer_regions")

    def peer_error(self) -> int:
        e = C.c_int32()
        _check(self._lib.fdog_peer_error(self._h, C.byref(e)), "fdog_peer_error")
        return e.value

    def primal_step(self, round_: int, delta: float, seed: int = 0):
        """One classification (+ perturbation) step of Alg. 2: (undecided, x)."""
        n = self.n_vars
        x = np.zeros(max(n, 1), np.uint8)
        u = C.c_int64()
        _check(self._lib.fdog_primal_step(self._h, int(round_), float(delta), int(seed), C.byref(u), _ptr(x), n),
               "fdog_primal_step")
        return u.value, x[:n]

    def round_primal(self, delta0=1.0, alpha=1.2, inner=5, max_rounds=100, seed=0, omega=0.5, keep_state=False):
        """Alg. 2: returns (x, rounds, objective); FastdogError(8) without consensus."""
        o = PrimalOptions()
        self._lib.fdog_default_primal_options(C.byref(o))
        o.delta0, o.alpha, o.inner, o.max_rounds = float(delta0), float(alpha), int(inner), int(max_rounds)
        o.seed, o.omega, o.keep_state = int(seed), float(omega), int(bool(keep_state))
        n = self.n_vars
        x = np.zeros(max(n, 1), np.uint8)
        r = C.c_int32()
        obj = C.c_double()
        _check(self._lib.fdog_round_primal(self._h, C.byref(o), _ptr(x), n, C.byref(r), C.byref(obj)),
               "fdog_round_primal")
        return x[:n], r.value, obj.value

    def profile_enable(self, on: bool):
        _check(self._lib.fdog_profile_enable(self._h, 1 if on else 0), "fdog_profile_enable")
