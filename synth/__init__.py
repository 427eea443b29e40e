"""Seeded synthetic MIP instances shaped like the paper's workloads.

This module is shared by the oracle side (tests, bench cpu_baseline) and the CUDA
side (tests, bench, smoke). It holds NONE of the method's arithmetic: it only draws
random instances in the problem form of PAPER.md:269 (§3.1, "Our MIPs have the form
min c^T x : Ax <= b, l <= x <= u, x_i in Z"), generalised to two-sided rows
lhs <= Ax <= rhs as BASELINE.json's north star states, plus start points.

Every generator is a pure function of its seed (numpy PCG64), so both sides see
bit-identical arrays. Recipes follow SURVEY.md §8(d) "Synthetic instance family"
and are restated in DESIGN.md §"Input recipe". All data are integers (the exactness
domain of DESIGN.md reading R11), magnitudes |a| <= 100, |rhs| < 1e7.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

INF = float("inf")


@dataclasses.dataclass
class Instance:
    """Raw (un-normalised) MIP in CSR form: lhs <= A x <= rhs, lb <= x <= ub."""

    name: str
    n: int
    m: int
    row_ptr: np.ndarray  # int64 [m+1]
    col_idx: np.ndarray  # int32 [nnz]
    val: np.ndarray      # float64 [nnz]
    lhs: np.ndarray      # float64 [m], -inf = absent
    rhs: np.ndarray      # float64 [m], +inf = absent
    lb: np.ndarray       # float64 [n]
    ub: np.ndarray       # float64 [n]
    is_int: np.ndarray   # uint8 [n]
    c: np.ndarray        # float64 [n]
    x_star: Optional[np.ndarray] = None  # planted feasible point (float64 [n])

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def arrays(self):
        return (self.n, self.m, self.row_ptr, self.col_idx, self.val, self.lhs, self.rhs,
                self.lb, self.ub, self.is_int, self.c)


def _csr_from_coo(m: int, n: int, rows: np.ndarray, cols: np.ndarray, vals: np.ndarray):
    """Sort COO triples by (row, col) and build CSR. Duplicate (row, col) pairs must not occur."""
    key = rows.astype(np.int64) * np.int64(n) + cols.astype(np.int64)
    order = np.argsort(key)  # keys are unique
    rows = rows[order]
    cols = cols[order].astype(np.int32)
    vals = vals[order].astype(np.float64)
    counts = np.bincount(rows, minlength=m).astype(np.int64)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, cols, vals


def _row_activity(m, rows, cols, vals, x):
    return np.bincount(rows, weights=vals * x[cols], minlength=m)


def _columns_to_coo(rng, m: int, deg: np.ndarray):
    """Column j gets deg[j] distinct rows, uniformly at random."""
    n = deg.shape[0]
    cols = np.repeat(np.arange(n, dtype=np.int64), deg)
    rows = rng.integers(0, m, size=cols.shape[0], dtype=np.int64)
    key = _sorted_unique(cols * np.int64(m) + rows)  # drops the rare duplicate (col, row)
    return (key % m), (key // m)


def _sorted_unique(key: np.ndarray) -> np.ndarray:
    key = np.sort(key)
    keep = np.empty(key.shape[0], dtype=bool)
    keep[:1] = True
    np.not_equal(key[1:], key[:-1], out=keep[1:])
    return key[keep]


# --------------------------------------------------------------------------------------
# Config T (BASELINE.json configs[0]): tiny MIP, 40 vars x 25 rows, knapsack + cover + general
# --------------------------------------------------------------------------------------
def tiny(seed: int) -> Instance:
    rng = np.random.default_rng([0xC0, seed])
    n_bin, n_int = 30, 10
    n = n_bin + n_int
    lb = np.zeros(n)
    ub = np.concatenate([np.ones(n_bin), np.full(n_int, 7.0)])
    is_int = np.ones(n, dtype=np.uint8)
    x_star = np.concatenate([(rng.random(n_bin) < 0.3).astype(np.float64),
                             rng.integers(0, 4, n_int).astype(np.float64)])
    rows_l, cols_l, vals_l, kinds = [], [], [], []
    for i in range(10):  # knapsack rows, 5-12 vars each, a in U{1..20}
        k = int(rng.integers(5, 13))
        cols = rng.choice(n, size=k, replace=False)
        rows_l.append(np.full(k, len(kinds))); cols_l.append(cols)
        vals_l.append(rng.integers(1, 21, k).astype(np.float64)); kinds.append("knap")
    for i in range(10):  # cover rows, |S| in [3, 8]
        k = int(rng.integers(3, 9))
        cols = rng.choice(n, size=k, replace=False)
        rows_l.append(np.full(k, len(kinds))); cols_l.append(cols)
        vals_l.append(np.ones(k)); kinds.append("cover")
    for i in range(5):  # general rows, a in U{+-1..+-5}
        k = int(rng.integers(3, 9))
        cols = rng.choice(n, size=k, replace=False)
        a = rng.integers(1, 6, k) * rng.choice([-1, 1], k)
        rows_l.append(np.full(k, len(kinds))); cols_l.append(cols)
        vals_l.append(a.astype(np.float64)); kinds.append("general")
    m = len(kinds)
    rows = np.concatenate(rows_l).astype(np.int64)
    cols = np.concatenate(cols_l).astype(np.int64)
    vals = np.concatenate(vals_l)
    # make the planted point cover every cover row
    for i, kd in enumerate(kinds):
        if kd == "cover":
            sel = cols[rows == i]
            if x_star[sel].sum() < 1:
                x_star[sel[int(rng.integers(0, sel.size))]] = 1.0
    act = _row_activity(m, rows, cols, vals, x_star)
    lhs = np.full(m, -INF)
    rhs = np.full(m, INF)
    for i, kd in enumerate(kinds):
        if kd == "knap":
            sel = rows == i
            rhs[i] = max(np.floor((vals[sel] * ub[cols[sel]]).sum() / 3.0), act[i])
        elif kd == "cover":
            lhs[i] = 1.0
        else:
            sense = int(rng.integers(0, 3))
            if sense == 0:
                rhs[i] = act[i] + rng.integers(0, 4)
            elif sense == 1:
                lhs[i] = act[i] - rng.integers(0, 4)
            else:
                lhs[i] = rhs[i] = act[i]
    c = rng.integers(-10, 11, n).astype(np.float64)
    row_ptr, col_idx, val = _csr_from_coo(m, n, rows, cols, vals)
    return Instance(f"T{seed}", n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, x_star)


# --------------------------------------------------------------------------------------
# Config S (configs[1]): set cover, 10k rows x 50k binaries, deg ~ 1 + Poisson(9)
# --------------------------------------------------------------------------------------
def setcover(seed: int = 1, m: int = 10_000, n: int = 50_000) -> Instance:
    rng = np.random.default_rng([0x5C, seed])
    deg = 1 + rng.poisson(9, n)
    rows, cols = _columns_to_coo(rng, m, deg)
    empty = np.setdiff1d(np.arange(m), rows)
    if empty.size:  # empty rows get one random column
        rows = np.concatenate([rows, empty])
        cols = np.concatenate([cols, rng.integers(0, n, empty.size)])
        key = _sorted_unique(cols * np.int64(m) + rows)
        rows, cols = key % m, key // m
    vals = np.ones(rows.shape[0])
    lhs = np.ones(m)
    rhs = np.full(m, INF)
    lb = np.zeros(n); ub = np.ones(n)
    is_int = np.ones(n, dtype=np.uint8)
    c = rng.integers(1, 101, n).astype(np.float64)
    row_ptr, col_idx, val = _csr_from_coo(m, n, rows, cols, vals)
    return Instance(f"S{seed}", n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, np.ones(n))


# --------------------------------------------------------------------------------------
# Config G (configs[2]): mixed general-integer MIP, 2e5 rows x 1e6 vars, ~1e7 nnz, 100 long columns
# --------------------------------------------------------------------------------------
LONG_KINDS = {
    "bin": "binary",
    "bkt": "integer [0, 64] (bounded domain: counting sort)",
    "unb": "integer [0, inf) (unbounded: sorted)",
    "big": "integer [0, 10000] (domain > 4096: sorted)",
    "cont": "continuous [0, 50] (sorted; tolerance mode)",
}


def mixed(seed: int = 2, n: int = 1_000_000, m: int = 200_000, n_long: int = 100,
          long_lo: float = 1e3, long_hi: float = 1e5, short_mean: float = 7.0,
          p_binary: float = 0.70, p_bounded: float = 0.25, long_kinds=("bin", "bkt")) -> Instance:
    """Config G's generator. The long columns are split into equal consecutive groups, one per
    entry of `long_kinds` (LONG_KINDS); the default (50 binary + 50 integer [0, 64]) is config G."""
    rng = np.random.default_rng([0x6E, seed])
    # variable classes: 70% binary, 25% integer [0, U] with U log-uniform{2..1000}, 5% integer [0, inf)
    u = rng.random(n)
    vclass = np.where(u < p_binary, 0, np.where(u < p_binary + p_bounded, 1, 2))
    U = np.floor(np.exp(rng.uniform(np.log(2), np.log(1001), n)))
    lb = np.zeros(n)
    ub = np.where(vclass == 0, 1.0, np.where(vclass == 1, U, INF))
    # long columns: 50 binary + 50 integer [0, 64]; unbounded integers only on short columns
    long_idx = rng.choice(n, size=n_long, replace=False)
    is_int = np.ones(n, dtype=np.uint8)
    for q, j in enumerate(long_idx):
        kind = long_kinds[q * len(long_kinds) // n_long]
        vclass[j], ub[j] = {"bin": (0, 1.0), "bkt": (1, 64.0), "unb": (2, INF), "big": (1, 10000.0),
                            "cont": (1, 50.0)}[kind]
        if kind == "cont":
            is_int[j] = 0
    deg = 1 + rng.poisson(short_mean, n)
    deg[long_idx] = 0
    rows, cols = _columns_to_coo(rng, m, deg)
    lr, lc = [], []
    for j in long_idx:
        d = int(np.floor(np.exp(rng.uniform(np.log(long_lo), np.log(long_hi)))))
        d = min(d, m)
        lr.append(rng.choice(m, size=d, replace=False).astype(np.int64))
        lc.append(np.full(d, j, dtype=np.int64))
    if n_long:
        rows = np.concatenate([rows] + lr)
        cols = np.concatenate([cols] + lc)
    # row kinds: 40% knapsack, 20% cover, 30% general, 10% packing
    rk = rng.choice(4, size=m, p=[0.4, 0.2, 0.3, 0.1])
    kind = rk[rows]
    vals = np.ones(rows.shape[0])
    kn = kind == 0
    vals[kn] = rng.integers(1, 51, int(kn.sum()))
    ge = kind == 2
    vals[ge] = rng.integers(1, 101, int(ge.sum())) * rng.choice([-1.0, 1.0], int(ge.sum()))
    # planted point
    x_star = np.where(vclass == 0, (rng.random(n) < 0.3).astype(np.float64),
                      np.minimum(rng.integers(0, 6, n), ub).astype(np.float64))
    act = _row_activity(m, rows, cols, vals, x_star)
    cov_unmet = np.where((rk == 1) & (act < 1))[0]
    if cov_unmet.size:
        # set one (the first in COO order) column of each unmet cover row to 1
        in_unmet = np.isin(rows, cov_unmet)
        r_sel, first = np.unique(rows[in_unmet], return_index=True)
        x_star[cols[in_unmet][first]] = np.maximum(x_star[cols[in_unmet][first]], 1.0)
        act = _row_activity(m, rows, cols, vals, x_star)
    ub_cap = np.minimum(ub, 10.0)
    cap_act = np.bincount(rows, weights=vals * ub_cap[cols], minlength=m)
    lhs = np.full(m, -INF)
    rhs = np.full(m, INF)
    # knapsack: a x <= max(floor(0.3 sum a min(u,10)), a x*)
    sel = rk == 0
    rhs[sel] = np.maximum(np.floor(0.3 * cap_act[sel]), act[sel])
    # cover: sum x >= 1
    lhs[rk == 1] = 1.0
    # general: <= / >= / = / ranged around a x*
    sel = np.where(rk == 2)[0]
    sense = rng.integers(0, 4, sel.size)
    s1 = rng.integers(0, 21, sel.size).astype(np.float64)
    s2 = rng.integers(0, 21, sel.size).astype(np.float64)
    a = act[sel]
    rhs[sel] = np.where(sense == 0, a + s1, np.where(sense == 1, INF, np.where(sense == 2, a, a + s1)))
    lhs[sel] = np.where(sense == 0, -INF, np.where(sense == 1, a - s2, np.where(sense == 2, a, a - s2)))
    # packing: sum x <= max(1, a x*)
    sel = rk == 3
    rhs[sel] = np.maximum(1.0, act[sel])
    c = rng.integers(-100, 101, n).astype(np.float64)
    row_ptr, col_idx, val = _csr_from_coo(m, n, rows, cols, vals)
    return Instance(f"G{seed}_n{n}", n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, x_star)


def scaled(nnz: int, seed: int = 4) -> Instance:
    """Config X (configs[4]): generator G with n = nnz/10, m = nnz/50, ~1% of nnz in long columns."""
    n = max(nnz // 10, 10)
    m = max(nnz // 50, 5)
    n_long = max(2, int(round(nnz * 0.01 / 1e4)))
    hi = max(min(1e5, m / 2), 20.0)
    lo = min(1e3, hi / 2)
    return mixed(seed, n=n, m=m, n_long=n_long, long_lo=lo, long_hi=hi, short_mean=8.0)


# --------------------------------------------------------------------------------------
# Config P (configs[3]): portfolio packing, 1e5 binaries x 2e4 rows, ~1e6 nnz
# --------------------------------------------------------------------------------------
def packing(seed: int = 3, n: int = 100_000, m: int = 20_000) -> Instance:
    rng = np.random.default_rng([0x9A, seed])
    deg = 1 + rng.poisson(9, n)
    rows, cols = _columns_to_coo(rng, m, deg)
    vals = rng.integers(1, 21, rows.shape[0]).astype(np.float64)
    rowsum = np.bincount(rows, weights=vals, minlength=m)
    rhs = np.floor(0.3 * rowsum)
    lhs = np.full(m, -INF)
    lb = np.zeros(n); ub = np.ones(n)
    is_int = np.ones(n, dtype=np.uint8)
    c = -rng.integers(1, 101, n).astype(np.float64)
    row_ptr, col_idx, val = _csr_from_coo(m, n, rows, cols, vals)
    return Instance(f"P{seed}", n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, np.zeros(n))


# --------------------------------------------------------------------------------------
# Start points and evaluation points
# --------------------------------------------------------------------------------------
def x_lower(inst: Instance) -> np.ndarray:
    """x0 = the in-domain value closest to 0 (0 for every config above)."""
    x = np.clip(np.zeros(inst.n), inst.lb, inst.ub)
    return np.where(inst.is_int.astype(bool), np.ceil(x), x)


def x_bernoulli(inst: Instance, key, p: float = 0.5) -> np.ndarray:
    """Binary start point keyed by (config seed, walker id) as SURVEY §8(d) config P states."""
    rng = np.random.default_rng(list(key))
    x = (rng.random(inst.n) < p).astype(np.float64)
    return np.clip(x, inst.lb, inst.ub)


def x_perturbed(inst: Instance, key, frac: float = 0.01) -> np.ndarray:
    """x_lower with a fraction `frac` of the variables (chosen keyed by `key`) raised by one unit
    where the upper bound allows it: a start point per weak-scaling replica."""
    rng = np.random.default_rng(list(key))
    x = x_lower(inst)
    up = (rng.random(inst.n) < frac) & (x + 1.0 <= inst.ub)
    x[up] += 1.0
    return x


def x_random(inst: Instance, seed: int, spread: int = 10) -> np.ndarray:
    """Random in-bounds point, integral on integer variables (an evaluation point for parity)."""
    rng = np.random.default_rng([0xE7, seed])
    lb = np.where(np.isfinite(inst.lb), inst.lb, -spread)
    ub = np.where(np.isfinite(inst.ub), inst.ub, lb + spread)
    ub = np.minimum(ub, lb + spread)
    x = lb + np.floor(rng.random(inst.n) * (ub - lb + 1))
    x = np.minimum(x, ub)
    cont = ~inst.is_int.astype(bool)
    x[cont] = (lb + rng.random(inst.n) * (ub - lb))[cont]
    return x


def weights_random(m_norm: int, seed: int, hi: int = 5) -> np.ndarray:
    """Integer-valued float32 weights in [1, hi] (reading R11)."""
    rng = np.random.default_rng([0x3E, seed])
    return rng.integers(1, hi + 1, m_norm).astype(np.float32)


# --------------------------------------------------------------------------------------
# Tiny random instances for property tests (SPEC.md:231 sizes)
# --------------------------------------------------------------------------------------
def random_tiny(seed: int, n_max: int = 6, m_max: int = 8, coef: int = 3, bound: int = 4,
                p_inf_bound: float = 0.0, p_binary: float = 0.3, p_cont: float = 0.0) -> Instance:
    rng = np.random.default_rng([0x71, seed])
    n = int(rng.integers(1, n_max + 1))
    m = int(rng.integers(1, m_max + 1))
    lb = rng.integers(-bound, bound + 1, n).astype(np.float64)
    ub = lb + rng.integers(0, bound + 1, n)
    ub = np.minimum(ub, bound).astype(np.float64)
    ub = np.maximum(ub, lb)
    binary = rng.random(n) < p_binary
    lb[binary] = 0.0
    ub[binary] = 1.0
    if p_inf_bound > 0:
        lb[rng.random(n) < p_inf_bound] = -INF
        ub[rng.random(n) < p_inf_bound] = INF
    is_int = (rng.random(n) >= p_cont).astype(np.uint8)
    is_int[binary] = 1
    dens = rng.random((m, n)) < 0.6
    A = rng.integers(-coef, coef + 1, (m, n)).astype(np.float64) * dens
    rows, cols = np.nonzero(A)
    vals = A[rows, cols]
    lhs = np.full(m, -INF)
    rhs = np.full(m, INF)
    for i in range(m):
        sense = int(rng.integers(0, 4))
        b = float(rng.integers(-coef * 2, coef * 2 + 1))
        if sense == 0:
            rhs[i] = b
        elif sense == 1:
            lhs[i] = b
        elif sense == 2:
            lhs[i] = rhs[i] = b
        else:
            lhs[i] = b
            rhs[i] = b + float(rng.integers(0, 4))
    c = rng.integers(-5, 6, n).astype(np.float64)
    row_ptr, col_idx, val = _csr_from_coo(m, n, rows.astype(np.int64), cols.astype(np.int64), vals)
    return Instance(f"R{seed}", n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, None)


def random_point_tiny(inst: Instance, seed: int, spread: int = 4) -> np.ndarray:
    rng = np.random.default_rng([0x72, seed])
    lo = np.where(np.isfinite(inst.lb), inst.lb, -spread)
    hi = np.where(np.isfinite(inst.ub), inst.ub, spread)
    hi = np.maximum(hi, lo)
    x = lo + np.floor(rng.random(inst.n) * (hi - lo + 1))
    x = np.minimum(x, hi)
    cont = ~inst.is_int.astype(bool)
    if cont.any():
        x[cont] = (lo + rng.integers(0, 4, inst.n) * (hi - lo) / 3.0)[cont]
    return x


CONFIGS = {
    "T": "tiny synthetic MIP: 40 binary/integer vars, 25 rows (knapsack+cover)",
    "S": "synthetic set-cover 10k rows x 50k binaries, ~500k nnz, single walker",
    "G": "synthetic mixed general-integer MIP 200k rows x 1M vars, ~10M nnz, long dense columns",
    "P": "competition-shaped portfolio: 64 tabu walkers on 1M-nnz packing MIP",
    "X": "scaling sweep: nnz 1e5 to 5e7",
}
