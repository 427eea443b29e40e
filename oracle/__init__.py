"""TEST INFRASTRUCTURE ONLY — ctypes loader for the plain fp64 CPU oracle (chap_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package. The product path (paper_2605_05086_b200) never imports it, and
this package never imports the product path: the two share nothing but the seeded input
generators in synth/.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "chap_oracle.c")

ORC_OK, ORC_ERR_INVALID_ARG, ORC_ERR_INFEASIBLE_BOUNDS = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle: plain C, -O2, no FMA contraction, no fast-math, OpenMP over j."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "chap_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


class Record(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("j", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("v", ctypes.c_double), ("s", ctypes.c_double), ("violated", ctypes.c_int64),
                ("obj", ctypes.c_double)]


RECORD_DTYPE = np.dtype([("k", "<i8"), ("j", "<i4"), ("flags", "<i4"), ("v", "<f8"), ("s", "<f8"),
                         ("violated", "<i8"), ("obj", "<f8")])


class Params(ctypes.Structure):
    _fields_ = [("tenure", ctypes.c_int32), ("weight_cap", ctypes.c_float),
                ("cutoff_delta", ctypes.c_double), ("aspiration", ctypes.c_int32), ("perturb", ctypes.c_int32),
                ("perturb_radius", ctypes.c_int32), ("smooth_prob", ctypes.c_float), ("rng_seed", ctypes.c_uint64)]


class Walker(ctypes.Structure):
    _fields_ = [("x", ctypes.POINTER(ctypes.c_double)), ("w", ctypes.POINTER(ctypes.c_float)),
                ("tabu_until", ctypes.POINTER(ctypes.c_int64)),
                ("best_x", ctypes.POINTER(ctypes.c_double)), ("k", ctypes.c_int64),
                ("cutoff_rhs", ctypes.c_double), ("best_obj", ctypes.c_double),
                ("has_incumbent", ctypes.c_int32), ("initialised", ctypes.c_int32), ("id", ctypes.c_int64),
                ("force_j", ctypes.c_int32), ("pad", ctypes.c_int32), ("force_v", ctypes.c_double)]


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L.orc_problem_create.restype = ctypes.c_int
        L.orc_problem_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64] + [P] * 9 + [
            ctypes.POINTER(ctypes.c_void_p)]
        L.orc_problem_free.argtypes = [P]
        L.orc_problem_sizes.argtypes = [P, P, P, P]
        L.orc_problem_row_map.argtypes = [P, P, P]
        L.orc_problem_vars.argtypes = [P, P, P, P]
        L.orc_auto_delta.argtypes = [P]
        L.orc_auto_delta.restype = ctypes.c_double
        L.orc_penalty.argtypes = [ctypes.c_double] * 3
        L.orc_penalty.restype = ctypes.c_double
        L.orc_breakpoint.argtypes = [ctypes.c_double] * 3 + [ctypes.c_int]
        L.orc_breakpoint.restype = ctypes.c_double
        L.orc_residuals.argtypes = [P, P, ctypes.c_double, P]
        L.orc_best_shift.argtypes = [P, P, P, ctypes.c_double, P, P, P, P, P, ctypes.c_int]
        L.orc_best_shift.restype = ctypes.c_int
        L.orc_best_shift_range.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P,
                                           ctypes.c_int]
        L.orc_best_shift_range.restype = ctypes.c_int
        L.orc_walker_init.argtypes = [P, ctypes.POINTER(Params), P, ctypes.POINTER(Walker)]
        L.orc_walker_init.restype = ctypes.c_int
        L.orc_tabu_run.argtypes = [P, ctypes.POINTER(Params), ctypes.POINTER(Walker), ctypes.c_int64, P,
                                   ctypes.c_int]
        L.orc_tabu_run.restype = ctypes.c_int
        L.orc_walker_restart.argtypes = [P, ctypes.POINTER(Params), ctypes.POINTER(Walker), P]
        L.orc_walker_restart.restype = ctypes.c_int
        L.orc_walker_set_cutoff.argtypes = [P, ctypes.POINTER(Params), ctypes.POINTER(Walker), ctypes.c_double]
        L.orc_walker_summary.argtypes = [P, ctypes.POINTER(Walker), P, P]
        L.orc_run_walkers.argtypes = [P, ctypes.POINTER(Params), P, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int]
        L.orc_run_walkers.restype = ctypes.c_int
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_draw.argtypes = [ctypes.c_uint64] * 4
        L.orc_draw.restype = ctypes.c_uint64
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def penalty(w, r_old, r_new) -> float:
    return lib().orc_penalty(float(w), float(r_old), float(r_new))


def splitmix64(state: int) -> int:
    """g(state): the first output of SplitMix64 seeded with state (R21)."""
    return lib().orc_splitmix64(state & (2**64 - 1))


def draw(seed: int, a: int, b: int, c: int) -> int:
    """The counter-based draw H(seed, a, b, c) = g(g(g(g(seed) ^ a) ^ b) ^ c) of R21."""
    M = 2**64 - 1
    return lib().orc_draw(seed & M, a & M, b & M, c & M)


def breakpoint(x_j, r_i, a_ij, is_integer) -> float:
    return lib().orc_breakpoint(float(x_j), float(r_i), float(a_ij), int(bool(is_integer)))


class Problem:
    """Normalised problem held by the oracle."""

    def __init__(self, n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c):
        L = lib()
        self._keep = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                      np.ascontiguousarray(val, np.float64), np.ascontiguousarray(lhs, np.float64),
                      np.ascontiguousarray(rhs, np.float64), np.ascontiguousarray(lb, np.float64),
                      np.ascontiguousarray(ub, np.float64), np.ascontiguousarray(is_int, np.uint8),
                      np.ascontiguousarray(c, np.float64)]
        h = ctypes.c_void_p()
        k = self._keep
        st = L.orc_problem_create(int(n), int(m), int(k[0][-1]) if m > 0 else 0,
                                  *[a.ctypes.data for a in k], ctypes.byref(h))
        if st != ORC_OK:
            raise OracleError(st)
        self.h = h
        self.n = int(n)
        mn = ctypes.c_int32(); zn = ctypes.c_int64(); zc = ctypes.c_int64()
        L.orc_problem_sizes(h, ctypes.byref(mn), ctypes.byref(zn), ctypes.byref(zc))
        self.m_norm, self.nnz_norm, self.nnz_cut = mn.value, zn.value, zc.value
        self.auto_delta = L.orc_auto_delta(h)

    @classmethod
    def from_instance(cls, inst):
        return cls(*inst.arrays())

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_problem_free(self.h)
            self.h = None

    def row_map(self):
        o = np.zeros(max(self.m_norm - 1, 1), np.int32)
        s = np.zeros(max(self.m_norm - 1, 1), np.int8)
        lib().orc_problem_row_map(self.h, o.ctypes.data, s.ctypes.data)
        return o[: self.m_norm - 1], s[: self.m_norm - 1]

    def vars(self):
        lb = np.zeros(self.n); ub = np.zeros(self.n); vc = np.zeros(self.n, np.uint8)
        lib().orc_problem_vars(self.h, lb.ctypes.data, ub.ctypes.data, vc.ctypes.data)
        return lb, ub, vc

    def residuals(self, x, cutoff_rhs=math.inf):
        x = np.ascontiguousarray(x, np.float64)
        r = np.zeros(self.m_norm)
        lib().orc_residuals(self.h, x.ctypes.data, float(cutoff_rhs), r.ctypes.data)
        return r

    def best_shift(self, x, w=None, cutoff_rhs=math.inf, threads=0):
        """Per-variable (xhat, score) and the best move (j, v, s) of Eq. (1), brute force."""
        x = np.ascontiguousarray(x, np.float64)
        wp = None
        if w is not None:
            w = np.ascontiguousarray(w, np.float32)
            assert w.shape[0] == self.m_norm
            wp = w.ctypes.data
        xhat = np.zeros(self.n); score = np.zeros(self.n)
        bj = ctypes.c_int32(); bv = ctypes.c_double(); bs = ctypes.c_double()
        st = lib().orc_best_shift(self.h, x.ctypes.data, wp, float(cutoff_rhs), xhat.ctypes.data,
                                  score.ctypes.data, ctypes.byref(bj), ctypes.byref(bv),
                                  ctypes.byref(bs), int(threads))
        if st != ORC_OK:
            raise OracleError(st)
        return xhat, score, (bj.value, bv.value, bs.value)

    def best_shift_range(self, x, j0, j1, w=None, cutoff_rhs=math.inf, threads=0, out=None):
        """The same for the variables [j0, j1) only (a bounded sample; activities from scratch)."""
        x = np.ascontiguousarray(x, np.float64)
        wp = None
        if w is not None:
            w = np.ascontiguousarray(w, np.float32)
            wp = w.ctypes.data
        xhat, score = out if out is not None else (np.zeros(self.n), np.zeros(self.n))
        bj = ctypes.c_int32(); bv = ctypes.c_double(); bs = ctypes.c_double()
        st = lib().orc_best_shift_range(self.h, x.ctypes.data, wp, float(cutoff_rhs), int(j0), int(j1),
                                        xhat.ctypes.data, score.ctypes.data, ctypes.byref(bj), ctypes.byref(bv),
                                        ctypes.byref(bs), int(threads))
        if st != ORC_OK:
            raise OracleError(st)
        return xhat, score, (bj.value, bv.value, bs.value)


@dataclass
class TabuParams:
    tenure: int = 10
    weight_cap: float = 1e6
    cutoff_delta: float = math.nan
    aspiration: int = 0
    perturb: int = 0
    perturb_radius: int = 16
    smooth_prob: float = 0.0
    rng_seed: int = 0

    def c(self):
        return Params(self.tenure, self.weight_cap, self.cutoff_delta, self.aspiration, self.perturb,
                      self.perturb_radius, self.smooth_prob, self.rng_seed)


class TabuWalker:
    """One oracle walker (own solution, tabu list and weights)."""

    def __init__(self, prob: Problem, x0, params: TabuParams = TabuParams(), walker_id: int = 0):
        self.prob = prob
        self.params = params
        self._prm = params.c()
        n, mn = prob.n, prob.m_norm
        self.x = np.zeros(max(n, 1)); self.w = np.ones(mn, np.float32)
        self.tabu_until = np.zeros(max(n, 1), np.int64); self.best_x = np.zeros(max(n, 1))
        self.S = Walker(_p(self.x, ctypes.c_double), _p(self.w, ctypes.c_float),
                        _p(self.tabu_until, ctypes.c_int64), _p(self.best_x, ctypes.c_double),
                        0, math.inf, math.inf, 0, 0, int(walker_id), -1, 0, 0.0)
        x0 = np.ascontiguousarray(x0, np.float64)
        st = lib().orc_walker_init(prob.h, ctypes.byref(self._prm), x0.ctypes.data, ctypes.byref(self.S))
        if st != ORC_OK:
            raise OracleError(st)

    def run(self, n_iters: int, threads: int = 0) -> np.ndarray:
        log = np.zeros(n_iters, RECORD_DTYPE)
        st = lib().orc_tabu_run(self.prob.h, ctypes.byref(self._prm), ctypes.byref(self.S), int(n_iters),
                                log.ctypes.data, int(threads))
        if st != ORC_OK:
            raise OracleError(st)
        return log

    def restart(self, x):
        x = np.ascontiguousarray(x, np.float64)
        st = lib().orc_walker_restart(self.prob.h, ctypes.byref(self._prm), ctypes.byref(self.S), x.ctypes.data)
        if st != ORC_OK:
            raise OracleError(st)

    def set_cutoff(self, z: float):
        lib().orc_walker_set_cutoff(self.prob.h, ctypes.byref(self._prm), ctypes.byref(self.S), float(z))

    def summary(self):
        """(violated active rows, sum of positive residuals over non-cutoff rows)"""
        v = ctypes.c_int64(); s = ctypes.c_double()
        lib().orc_walker_summary(self.prob.h, ctypes.byref(self.S), ctypes.byref(v), ctypes.byref(s))
        return v.value, s.value

    @property
    def k(self):
        return self.S.k

    @property
    def cutoff_rhs(self):
        return self.S.cutoff_rhs

    @property
    def best_obj(self):
        return self.S.best_obj

    @property
    def has_incumbent(self):
        return bool(self.S.has_incumbent)


def run_walkers(prob: Problem, walkers, K: int, n_epochs: int, n_elite: int, n_restart: int, threads: int = 0):
    """orc_run_walkers: the single-process portfolio with the every-K exchange over
    already-initialised TabuWalker objects (their states are updated in place)."""
    arr = (Walker * len(walkers))(*[w.S for w in walkers])
    prm = walkers[0]._prm
    st = lib().orc_run_walkers(prob.h, ctypes.byref(prm), ctypes.cast(arr, ctypes.c_void_p), len(walkers), int(K),
                               int(n_epochs), int(n_elite), int(n_restart), int(threads))
    if st != ORC_OK:
        raise OracleError(st)
    for w, a in zip(walkers, arr):
        w.S = a
    return walkers
