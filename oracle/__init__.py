"""ctypes binding of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
module.  The product path (``paper_2111_10270_b200``) never imports it and
shares no code with it.

The library is built by ``__graft_entry__.build()`` (or ``make oracle``) into
``oracle/liboracle.so``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

_ERRORS = {1: "invalid argument", 2: "infeasible constraint", 3: "out of memory", 6: "bad state",
           7: "no consensus within max_rounds"}


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: {_ERRORS.get(code, code)} ({code})")
        self.code = code


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp); plain C, no GPU."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _Problem(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("cost", C.c_void_p), ("n_cons", C.c_int32),
                ("row_ptr", C.c_void_p), ("col_var", C.c_void_p), ("col_coef", C.c_void_p),
                ("rel", C.c_void_p), ("rhs", C.c_void_p)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        lib.oracle_create.argtypes = [P, C.c_double, C.c_int, C.POINTER(P)]
        lib.oracle_destroy.argtypes = [P]
        lib.oracle_destroy.restype = None
        lib.oracle_pass.argtypes = [P, C.c_int, C.c_double]
        lib.oracle_iterate.argtypes = [P, C.c_int, C.c_double]
        lib.oracle_pass_seq.argtypes = [P, C.c_int, C.c_double]
        lib.oracle_iterate_seq.argtypes = [P, C.c_int, C.c_double]
        lib.oracle_lower_bound.argtypes = [P, P]
        lib.oracle_dual_energy.argtypes = [P, P]
        lib.oracle_finalize.argtypes = [P]
        lib.oracle_finalize_avg.argtypes = [P]
        lib.oracle_num_slots.argtypes = [P, P]
        for f in ("oracle_get_lambda", "oracle_get_deferred", "oracle_set_lambda"):
            getattr(lib, f).argtypes = [P, P, C.c_int64]
        lib.oracle_min_marginals.argtypes = [P, P, P, C.c_int64]
        lib.oracle_bdd_size.argtypes = [P, C.c_int32, P, P]
        lib.oracle_bdd_get.argtypes = [P, C.c_int32, P, P, P, P]
        lib.oracle_total_nodes.argtypes = [P, P]
        lib.oracle_num_threads.argtypes = [P]
        lib.oracle_set_lifted.argtypes = [P]
        lib.oracle_get_lifted.argtypes = [P, P, P, C.c_int64]
        lib.oracle_primal_step.argtypes = [P, C.c_int32, C.c_double, C.c_uint64, P, P]
        lib.oracle_round_primal.argtypes = [P, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_uint64,
                                            C.c_double, P, P]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def default_clamp(cost) -> float:
    """Reading A5: C = 1e4 * (1 + max_i |c_i|), identical to the product default."""
    c = np.asarray(cost, dtype=np.float64)
    return 1e4 * (1.0 + (float(np.max(np.abs(c))) if c.size else 0.0))


class Oracle:
    """fp64 oracle solver over a problem dict (see synth.Problem)."""

    def __init__(self, problem, clamp: float | None = None, n_threads: int = 0):
        lib = _load()
        self._keep = [np.ascontiguousarray(problem.cost, dtype=np.float64),
                      np.ascontiguousarray(problem.row_ptr, dtype=np.int64),
                      np.ascontiguousarray(problem.col_var, dtype=np.int32),
                      np.ascontiguousarray(problem.col_coef, dtype=np.int32),
                      np.ascontiguousarray(problem.rel, dtype=np.int8),
                      np.ascontiguousarray(problem.rhs, dtype=np.int64)]
        cost, row_ptr, col_var, col_coef, rel, rhs = self._keep
        p = _Problem(int(problem.n_vars), _ptr(cost), int(problem.n_cons), _ptr(row_ptr),
                     _ptr(col_var), _ptr(col_coef), _ptr(rel), _ptr(rhs))
        h = C.c_void_p()
        if clamp is None:
            clamp = default_clamp(cost)
        rc = lib.oracle_create(C.byref(p), float(clamp), int(n_threads), C.byref(h))
        if rc:
            raise OracleError(rc, "create")
        self._h = h
        self._lib = lib
        self.n_cons = int(problem.n_cons)
        self.n_vars = int(problem.n_vars)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def _chk(self, rc, what):
        if rc:
            raise OracleError(rc, what)

    @property
    def threads(self) -> int:
        return self._lib.oracle_num_threads(self._h)

    def pass_(self, forward: bool, omega: float = 0.5):
        self._chk(self._lib.oracle_pass(self._h, 1 if forward else 0, float(omega)), "pass")

    def iterate(self, n: int, omega: float = 0.5):
        self._chk(self._lib.oracle_iterate(self._h, int(n), float(omega)), "iterate")

    def pass_seq(self, forward: bool, omega: float = 0.5):
        """Non-deferred (sequential) min-marginal averaging pass."""
        self._chk(self._lib.oracle_pass_seq(self._h, 1 if forward else 0, float(omega)), "pass_seq")

    def iterate_seq(self, n: int, omega: float = 0.5):
        self._chk(self._lib.oracle_iterate_seq(self._h, int(n), float(omega)), "iterate_seq")

    def lower_bound(self) -> float:
        x = C.c_double()
        self._chk(self._lib.oracle_lower_bound(self._h, C.byref(x)), "lower_bound")
        return x.value

    def dual_energy(self) -> float:
        x = C.c_double()
        self._chk(self._lib.oracle_dual_energy(self._h, C.byref(x)), "dual_energy")
        return x.value

    def set_lifted(self):
        """Switch to the lifted representation before the first pass."""
        self._chk(self._lib.oracle_set_lifted(self._h), "set_lifted")

    def lifted(self):
        """(lambda^{j,0}, lambda^{j,1}) per slot, canonical order (lifted mode)."""
        n = self.num_slots()
        a, b = np.empty(max(n, 1)), np.empty(max(n, 1))
        self._chk(self._lib.oracle_get_lifted(self._h, _ptr(a), _ptr(b), a.size), "get_lifted")
        return a[:n], b[:n]

    def finalize(self, averaged: bool = False):
        fn = self._lib.oracle_finalize_avg if averaged else self._lib.oracle_finalize
        self._chk(fn(self._h), "finalize")

    def num_slots(self) -> int:
        x = C.c_int64()
        self._chk(self._lib.oracle_num_slots(self._h, C.byref(x)), "num_slots")
        return x.value

    def _get(self, fn):
        n = self.num_slots()
        out = np.empty(max(n, 1), dtype=np.float64)
        self._chk(getattr(self._lib, fn)(self._h, _ptr(out), n), fn)
        return out[:n]

    def lam(self):
        return self._get("oracle_get_lambda")

    def deferred(self):
        return self._get("oracle_get_deferred")

    def set_lambda(self, lam):
        a = np.ascontiguousarray(lam, dtype=np.float64)
        self._chk(self._lib.oracle_set_lambda(self._h, _ptr(a), a.size), "set_lambda")

    def min_marginals(self):
        n = self.num_slots()
        m0 = np.empty(max(n, 1)); m1 = np.empty(max(n, 1))
        self._chk(self._lib.oracle_min_marginals(self._h, _ptr(m0), _ptr(m1), n), "min_marginals")
        return m0[:n], m1[:n]

    def total_nodes(self) -> int:
        x = C.c_int64()
        self._chk(self._lib.oracle_total_nodes(self._h, C.byref(x)), "total_nodes")
        return x.value

    def bdd(self, j: int):
        """Return (vars, hop_start, lo, hi) of BDD j (-1 bottom, -2 top)."""
        k = C.c_int32(); n = C.c_int32()
        self._chk(self._lib.oracle_bdd_size(self._h, int(j), C.byref(k), C.byref(n)), "bdd_size")
        vars_ = np.empty(max(k.value, 1), np.int32)
        hs = np.empty(k.value + 1, np.int32)
        lo = np.empty(max(n.value, 1), np.int32)
        hi = np.empty(max(n.value, 1), np.int32)
        self._chk(self._lib.oracle_bdd_get(self._h, int(j), _ptr(vars_), _ptr(hs), _ptr(lo), _ptr(hi)),
                  "bdd_get")
        return vars_[:k.value], hs, lo[:n.value], hi[:n.value]

    def primal_step(self, round_: int, delta: float, seed: int = 0):
        """One classification + perturbation step of Alg. 2; returns (conflicts, x)."""
        x = np.zeros(max(self.n_vars, 1), np.uint8)
        nc = C.c_int64()
        self._chk(self._lib.oracle_primal_step(self._h, int(round_), float(delta), int(seed), C.byref(nc),
                                               _ptr(x)), "primal_step")
        return nc.value, x[:self.n_vars]

    def round_primal(self, delta0=1.0, alpha=1.2, inner=5, max_rounds=100, seed=0, omega=0.5):
        """Alg. 2; returns (x, rounds); raises OracleError(7) without consensus."""
        x = np.zeros(max(self.n_vars, 1), np.uint8)
        r = C.c_int32()
        self._chk(self._lib.oracle_round_primal(self._h, float(delta0), float(alpha), int(inner), int(max_rounds),
                                                int(seed), float(omega), _ptr(x), C.byref(r)), "round_primal")
        return x[:self.n_vars], r.value

    def hop_widths(self, j: int):
        _, hs, _, _ = self.bdd(j)
        return np.diff(hs)
