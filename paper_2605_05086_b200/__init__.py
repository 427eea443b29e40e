"""paper_2605_05086_b200 — B200-native best-shift tabu core of CHAP (arxiv 2605.05086).

A thin ctypes binding over libchap.so, whose C ABI is include/chap.h. The functions keep the
C names (chap_problem_create, chap_eval_best_shift, chap_tabu_step, chap_run_walkers, ...);
the small classes below only marshal arguments: every step of the method runs in the CUDA
kernels of csrc/. PyTorch is used for device memory and streams only. There is no CPU
fallback: importing this package without the built extension raises ImportError.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libchap.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libchap.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA path has no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------------------------------
# ABI structs (field order and sizes as in include/chap.h)
# ------------------------------------------------------------------------------------------
c_i32, c_i64, c_f32, c_f64, c_u8, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double,
                                          ctypes.c_uint8, ctypes.c_void_p)


class chap_problem_info(ctypes.Structure):
    _fields_ = [("n", c_i32), ("m", c_i32), ("m_norm", c_i32), ("cutoff_row", c_i32), ("nnz_norm", c_i64),
                ("nnz_cut", c_i64), ("n_fixed", c_i32), ("n_binary", c_i32), ("n_integer", c_i32),
                ("n_continuous", c_i32), ("exact_integer_data", c_i32), ("n_long_columns", c_i32),
                ("auto_cutoff_delta", c_f64), ("device_bytes", c_i64), ("model_bytes_A", c_i64),
                ("model_bytes_pass", c_i64), ("model_bytes_kernel", c_i64 * 3), ("nnz_kernel", c_i64 * 3),
                ("eval_launches", c_i32), ("n_sorted_columns", c_i32), ("model_bytes_walker_kernel", c_i64 * 3),
                ("n_gridsort_columns", c_i32), ("pad_info", c_i32), ("exchange_point_bytes", c_i64)]


class chap_move(ctypes.Structure):
    _fields_ = [("j", c_i32), ("pad", c_i32), ("v", c_f64), ("s", c_f64)]


class chap_params(ctypes.Structure):
    _fields_ = [("tenure", c_i32), ("weight_cap", c_f32), ("cutoff_delta", c_f64), ("exchange_K", c_i32),
                ("n_elite", c_i32), ("n_restart", c_i32), ("graph_iters", c_i32),
                ("binary_kernel", c_i32), ("pdl", c_i32), ("l2_persist", c_i32), ("aspiration", c_i32),
                ("lazy", c_i32), ("perturb", c_i32), ("perturb_radius", c_i32), ("smooth_prob", c_f32),
                ("rng_seed", ctypes.c_uint64)]


class chap_step_record(ctypes.Structure):
    _fields_ = [("k", c_i64), ("j", c_i32), ("flags", c_i32), ("v", c_f64), ("s", c_f64), ("violated", c_i64),
                ("obj", c_f64)]


class chap_walker_stats(ctypes.Structure):
    _fields_ = [("k", c_i64), ("violated", c_i64), ("obj", c_f64), ("best_obj", c_f64), ("cutoff_rhs", c_f64),
                ("has_incumbent", c_i32), ("pad", c_i32), ("n_moves", c_i64), ("n_stuck", c_i64)]


class chap_result(ctypes.Structure):
    _fields_ = [("best_obj", c_f64), ("has_incumbent", c_i32), ("best_walker", c_i32), ("iterations", c_i64),
                ("epochs", c_i64), ("seconds", c_f64)]


class chap_walker_summary(ctypes.Structure):
    _fields_ = [("best_obj", c_f64), ("violated", c_i64), ("sumviol", c_f64), ("gid", c_i32), ("flags", c_i32)]


SUMMARY_DTYPE = np.dtype([("best_obj", "<f8"), ("violated", "<i8"), ("sumviol", "<f8"), ("gid", "<i4"),
                          ("flags", "<i4")])
MOVE_DTYPE = np.dtype([("j", "<i4"), ("pad", "<i4"), ("v", "<f8"), ("s", "<f8")])
RECORD_DTYPE = np.dtype([("k", "<i8"), ("j", "<i4"), ("flags", "<i4"), ("v", "<f8"), ("s", "<f8"),
                         ("violated", "<i8"), ("obj", "<f8")])
STATS_DTYPE = np.dtype([("k", "<i8"), ("violated", "<i8"), ("obj", "<f8"), ("best_obj", "<f8"),
                        ("cutoff_rhs", "<f8"), ("has_incumbent", "<i4"), ("pad", "<i4"), ("n_moves", "<i8"),
                        ("n_stuck", "<i8")])
assert ctypes.sizeof(chap_move) == 24 and ctypes.sizeof(chap_step_record) == 48
assert ctypes.sizeof(chap_walker_stats) == 64

STATUS = {0: "CHAP_OK", 1: "CHAP_ERR_INVALID_ARG", 2: "CHAP_ERR_INFEASIBLE_BOUNDS", 3: "CHAP_ERR_CUDA",
          4: "CHAP_ERR_OOM", 5: "CHAP_ERR_NCCL", 6: "CHAP_ERR_STATE", 7: "CHAP_ERR_UNSUPPORTED"}

_P = c_vp
_SIGS = {
    "chap_last_error": (ctypes.c_char_p, []),
    "chap_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "chap_abi_version": (c_i32, []),
    "chap_problem_create": (ctypes.c_int, [c_i32, c_i32, c_i64] + [_P] * 9 + [c_i32, ctypes.POINTER(c_vp)]),
    "chap_problem_info_get": (ctypes.c_int, [_P, ctypes.POINTER(chap_problem_info)]),
    "chap_problem_row_map": (ctypes.c_int, [_P, _P, _P]),
    "chap_problem_destroy": (ctypes.c_int, [_P]),
    "chap_eval_best_shift": (ctypes.c_int, [_P, _P, _P, c_f64, _P, _P, _P, _P]),
    "chap_eval_best_shift_host": (ctypes.c_int, [_P, _P, _P, c_f64, _P, _P, _P, _P]),
    "chap_params_default": (ctypes.c_int, [ctypes.POINTER(chap_params)]),
    "chap_walkers_create": (ctypes.c_int, [_P, c_i32, _P, ctypes.POINTER(chap_params), _P, ctypes.POINTER(c_vp)]),
    "chap_tabu_step": (ctypes.c_int, [_P, c_i32, _P, _P]),
    "chap_walkers_get": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "chap_walkers_set_cutoff": (ctypes.c_int, [_P, c_f64, _P]),
    "chap_walkers_restart": (ctypes.c_int, [_P, c_i32, _P, _P]),
    "chap_lp_pdhg": (ctypes.c_int, [_P, _P, c_i32, ctypes.c_double, c_i32, _P, _P, _P]),
    "chap_lp_round": (ctypes.c_int, [_P, _P, _P, _P]),
    "chap_walkers_destroy": (ctypes.c_int, [_P]),
    "chap_walkers_profile": (ctypes.c_int, [_P, c_i32, _P, _P]),
    "chap_walkers_timing": (ctypes.c_int, [_P, c_i32, _P, _P]),
    "chap_walkers_launches_per_iter": (ctypes.c_int, [_P, _P]),
    "chap_walkers_exchange": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "chap_walkers_epoch": (ctypes.c_int, [_P, _P, c_i32, _P, _P, _P]),
    "chap_exchange_plan_device": (ctypes.c_int, [c_i32, c_i32, c_i32, _P, c_i32, c_i32, _P, _P, _P, _P, _P, _P,
                                                  _P, _P, _P]),
    "chap_comm_unique_id": (ctypes.c_int, [_P]),
    "chap_comm_create": (ctypes.c_int, [_P, c_i32, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "chap_comm_destroy": (ctypes.c_int, [_P]),
    "chap_run_walkers": (ctypes.c_int, [_P, c_i32, _P, ctypes.POINTER(chap_params), _P, c_i64, c_f64, _P,
                                        ctypes.POINTER(chap_result), _P]),
    "chap_exchange_plan": (ctypes.c_int, [c_i32, c_i32, _P, c_i32, c_i32, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_SIGS)


class ChapError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != 0:
        raise ChapError(st, _lib.chap_last_error().decode(errors="replace"))


def _ptr(t) -> Optional[int]:
    """Device/host address of a torch tensor or numpy array (None passes NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def default_params(**kw) -> chap_params:
    p = chap_params()
    _check(chap_params_default(ctypes.byref(p)))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


# ------------------------------------------------------------------------------------------
# thin object wrappers
# ------------------------------------------------------------------------------------------
class Problem:
    """chap_problem: normalised, device-resident instance."""

    def __init__(self, n, m, row_ptr, col_idx, val, lhs, rhs, lb, ub, is_int, c, device: int = 0):
        arrs = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                np.ascontiguousarray(val, np.float64), np.ascontiguousarray(lhs, np.float64),
                np.ascontiguousarray(rhs, np.float64), np.ascontiguousarray(lb, np.float64),
                np.ascontiguousarray(ub, np.float64), np.ascontiguousarray(is_int, np.uint8),
                np.ascontiguousarray(c, np.float64)]
        h = c_vp()
        nnz = int(arrs[0][-1]) if m > 0 else 0
        _check(chap_problem_create(int(n), int(m), nnz, *[a.ctypes.data for a in arrs], int(device), ctypes.byref(h)))
        self.h = h
        self.device = device
        self.info = chap_problem_info()
        _check(chap_problem_info_get(h, ctypes.byref(self.info)))
        self.n = self.info.n
        self.m_norm = self.info.m_norm

    @classmethod
    def from_instance(cls, inst, device: int = 0):
        return cls(*inst.arrays(), device=device)

    def close(self):
        if getattr(self, "h", None):
            chap_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def row_map(self):
        k = max(self.m_norm - 1, 0)
        o = np.zeros(max(k, 1), np.int32)
        s = np.zeros(max(k, 1), np.int8)
        _check(chap_problem_row_map(self.h, o.ctypes.data, s.ctypes.data))
        return o[:k], s[:k]

    def eval_best_shift(self, x, w=None, cutoff_rhs: float = math.inf, outputs: bool = True, stream=None):
        """chap_eval_best_shift on device tensors; returns (xhat, score, move) device tensors."""
        import torch
        dev = x.device
        xhat = torch.empty(self.n, dtype=torch.float64, device=dev) if outputs else None
        score = torch.empty(self.n, dtype=torch.float64, device=dev) if outputs else None
        best = torch.empty(MOVE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        _check(chap_eval_best_shift(self.h, _ptr(x), _ptr(w), float(cutoff_rhs), _ptr(xhat), _ptr(score),
                                    _ptr(best), _stream(stream)))
        return xhat, score, best

    def eval_best_shift_host(self, x: np.ndarray, w: Optional[np.ndarray] = None, cutoff_rhs: float = math.inf,
                             outputs: bool = True, stream=None, out=None):
        """chap_eval_best_shift_host: HOST numpy buffers in and out (copies inside the call).
        `out` = (xhat, score) float64 [n] arrays to fill (e.g. page-locked, copied by DMA directly)."""
        x = np.ascontiguousarray(x, np.float64)
        w = None if w is None else np.ascontiguousarray(w, np.float32)
        if out is not None:
            xhat, score = out
            assert xhat.dtype == np.float64 and score.dtype == np.float64 and xhat.flags.c_contiguous \
                and score.flags.c_contiguous and xhat.size == self.n and score.size == self.n
        else:
            xhat = np.empty(self.n) if outputs else None
            score = np.empty(self.n) if outputs else None
        best = np.zeros(1, MOVE_DTYPE)
        _check(chap_eval_best_shift_host(self.h, _ptr(x), _ptr(w), float(cutoff_rhs), _ptr(xhat), _ptr(score),
                                         _ptr(best), _stream(stream)))
        return xhat, score, best[0]


def move_from_bytes(t) -> np.void:
    return np.frombuffer(t.cpu().numpy().tobytes(), MOVE_DTYPE)[0]


class Walkers:
    """chap_walkers: W independent tabu walkers."""

    def __init__(self, problem: Problem, x0, params: Optional[chap_params] = None, stream=None):
        self.problem = problem
        self.W = int(x0.shape[0]) if x0.dim() == 2 else 1
        self.params = params if params is not None else default_params()
        h = c_vp()
        _check(chap_walkers_create(problem.h, self.W, _ptr(x0.contiguous()), ctypes.byref(self.params),
                                   _stream(stream), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            chap_walkers_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, n_iters: int, log: bool = False, stream=None):
        """chap_tabu_step; returns the log as a uint8 device tensor [n_iters * W * 48] (or None)."""
        import torch
        buf = None
        if log:
            buf = torch.empty(n_iters * self.W * RECORD_DTYPE.itemsize, dtype=torch.uint8,
                              device=f"cuda:{self.problem.device}")
        _check(chap_tabu_step(self.h, int(n_iters), _ptr(buf), _stream(stream)))
        return buf

    def get(self, stream=None):
        """chap_walkers_get into fresh device tensors; returns a dict of host numpy arrays."""
        import torch
        dev = f"cuda:{self.problem.device}"
        n, mn, W = self.problem.n, self.problem.m_norm, self.W
        x = torch.empty((W, n), dtype=torch.float64, device=dev)
        r = torch.empty((W, mn), dtype=torch.float64, device=dev)
        w = torch.empty((W, mn), dtype=torch.float32, device=dev)
        tabu = torch.empty((W, n), dtype=torch.int64, device=dev)
        bx = torch.empty((W, n), dtype=torch.float64, device=dev)
        st = torch.empty(W * STATS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        _check(chap_walkers_get(self.h, _ptr(x), _ptr(r), _ptr(w), _ptr(tabu), _ptr(bx), _ptr(st), _stream(stream)))
        torch.cuda.synchronize(dev)
        return {"x": x.cpu().numpy(), "r": r.cpu().numpy(), "w": w.cpu().numpy(), "tabu_until": tabu.cpu().numpy(),
                "best_x": bx.cpu().numpy(),
                "stats": np.frombuffer(st.cpu().numpy().tobytes(), STATS_DTYPE).copy()}

    def profile(self, n_iters: int, stream=None) -> np.ndarray:
        """chap_walkers_profile: average ms per iteration of [warp eval, block eval, long eval, select, apply]."""
        ms = np.zeros(5)
        _check(chap_walkers_profile(self.h, int(n_iters), ms.ctypes.data, _stream(stream)))
        return ms

    def launches_per_iter(self) -> int:
        """chap_walkers_launches_per_iter: kernel launches of one tabu iteration."""
        out = ctypes.c_int32()
        _check(chap_walkers_launches_per_iter(self.h, ctypes.addressof(out)))
        return int(out.value)

    def timing(self, mode: int, stream=None) -> np.ndarray:
        """chap_walkers_timing: the accumulated [bin, gen, eval, apply, span] ns and iteration count;
        then mode 1 = on and zeroed, 0 = off, -1 = read only."""
        out = np.zeros(6, np.uint64)
        _check(chap_walkers_timing(self.h, int(mode), out.ctypes.data, _stream(stream)))
        return out

    def exchange(self, comm: Optional["Comm"] = None, result: bool = True, stream=None):
        """chap_walkers_exchange: one portfolio exchange (on the device); with result=True returns (best
        objective, its global walker id) (synchronising), else None (stream-ordered, no sync)."""
        z = ctypes.c_double()
        g = ctypes.c_int32()
        _check(chap_walkers_exchange(self.h, comm.h if comm is not None else None,
                                     ctypes.addressof(z) if result else None, ctypes.addressof(g) if result else None,
                                     _stream(stream)))
        return (z.value, g.value) if result else None

    def epoch(self, n_iters: int, comm: Optional["Comm"] = None, result: bool = False, stream=None):
        """chap_walkers_epoch: n_iters tabu iterations + one exchange as one CUDA graph; with result=True
        returns (best objective, its global walker id) (synchronising), else None."""
        z = ctypes.c_double()
        g = ctypes.c_int32()
        _check(chap_walkers_epoch(self.h, comm.h if comm is not None else None, int(n_iters),
                                  ctypes.addressof(z) if result else None, ctypes.addressof(g) if result else None,
                                  _stream(stream)))
        return (z.value, g.value) if result else None

    def set_cutoff(self, z_best: float, stream=None):
        _check(chap_walkers_set_cutoff(self.h, float(z_best), _stream(stream)))

    def restart(self, walker: int, x, stream=None):
        _check(chap_walkers_restart(self.h, int(walker), _ptr(x.contiguous()), _stream(stream)))


def records(buf) -> np.ndarray:
    """Decode a chap_step_record log tensor."""
    return np.frombuffer(buf.cpu().numpy().tobytes(), RECORD_DTYPE).copy()


def comm_unique_id() -> bytes:
    b = (ctypes.c_uint8 * 128)()
    _check(chap_comm_unique_id(ctypes.addressof(b)))
    return bytes(b)


class Comm:
    """chap_comm: an NCCL communicator owned by the library (bootstrapped via torch.distributed)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        b = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = c_vp()
        _check(chap_comm_create(ctypes.addressof(b), int(nranks), int(rank), int(device), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            chap_comm_destroy(self.h)
            self.h = None


def run_walkers(problem: Problem, x0, params: Optional[chap_params] = None, comm: Optional[Comm] = None,
                max_iters: int = 1000, time_limit_s: float = 0.0, stream=None):
    """chap_run_walkers; returns (chap_result, best_x device tensor)."""
    import torch
    params = params if params is not None else default_params()
    res = chap_result()
    bx = torch.empty(problem.n, dtype=torch.float64, device=x0.device)
    _check(chap_run_walkers(problem.h, int(x0.shape[0]), _ptr(x0.contiguous()), ctypes.byref(params),
                            comm.h if comm is not None else None, int(max_iters), float(time_limit_s), _ptr(bx),
                            ctypes.byref(res), _stream(stream)))
    return res, bx


def exchange_plan_device(summaries: np.ndarray, W_local: int, rank: int, n_elite: int, n_restart: int,
                         device: int = 0) -> dict:
    """chap_exchange_plan_device: the exchange decisions as the device exchange computes them (for
    rank `rank`), returned as host arrays (the same keys as exchange_plan, plus local_rank and
    restart_slot)."""
    import torch
    s = np.ascontiguousarray(summaries, SUMMARY_DTYPE)
    W = int(s.shape[0])
    dev = torch.device("cuda", device)
    ds = torch.from_numpy(s.view(np.uint8).copy()).to(dev)
    E = max(2 * n_elite, 1)
    z = torch.empty(1, dtype=torch.float64, device=dev)
    cnt = torch.zeros(4, dtype=torch.int32, device=dev)
    eg = torch.full((E,), -1, dtype=torch.int32, device=dev)
    es = torch.full((E,), -1, dtype=torch.int32, device=dev)
    lr = torch.full((2 * W_local,), -2, dtype=torch.int32, device=dev)
    rg = torch.full((W,), -1, dtype=torch.int32, device=dev)
    rs = torch.full((W,), -1, dtype=torch.int32, device=dev)
    sl = torch.full((W_local,), -2, dtype=torch.int32, device=dev)
    _check(chap_exchange_plan_device(W, int(W_local), int(rank), _ptr(ds), int(n_elite), int(n_restart), _ptr(z),
                                     _ptr(cnt), _ptr(eg), _ptr(es), _ptr(lr), _ptr(rg), _ptr(rs), _ptr(sl),
                                     _stream(None)))
    torch.cuda.synchronize(dev)
    c = cnt.cpu().numpy()
    ne, nr = int(c[1]), int(c[2])
    nf = int(np.count_nonzero(s["flags"] & 1))
    nf = min(nf, n_elite)
    return {"z_best": float(z.item()), "best_gid": int(c[0]), "elite_gid": eg.cpu().numpy()[:ne],
            "elite_kind": (np.arange(ne) >= nf).astype(np.int8), "elite_slot": es.cpu().numpy()[:ne],
            "restart_gid": rg.cpu().numpy()[:nr], "restart_src": rs.cpu().numpy()[:nr],
            "local_rank": lr.cpu().numpy().reshape(2, W_local), "restart_slot": sl.cpu().numpy()}


def exchange_plan(summaries: np.ndarray, W_local: int, n_elite: int, n_restart: int) -> dict:
    """chap_exchange_plan (host only): the deterministic exchange decisions from gathered summaries
    (a SUMMARY_DTYPE array indexed by global walker id)."""
    s = np.ascontiguousarray(summaries, SUMMARY_DTYPE)
    W = int(s.shape[0])
    z = ctypes.c_double(); bg = ctypes.c_int32(); ne = ctypes.c_int32(); nr = ctypes.c_int32()
    eg = np.zeros(max(2 * n_elite, 1), np.int32); ek = np.zeros(max(2 * n_elite, 1), np.int8)
    es = np.zeros(max(2 * n_elite, 1), np.int32)
    rg = np.zeros(max(n_restart, 1), np.int32); rs = np.zeros(max(n_restart, 1), np.int32)
    _check(chap_exchange_plan(W, int(W_local), s.ctypes.data, int(n_elite), int(n_restart), ctypes.addressof(z),
                              ctypes.addressof(bg), ctypes.addressof(ne), eg.ctypes.data, ek.ctypes.data,
                              es.ctypes.data, ctypes.addressof(nr), rg.ctypes.data, rs.ctypes.data))
    return {"z_best": z.value, "best_gid": bg.value, "elite_gid": eg[:ne.value].copy(),
            "elite_kind": ek[:ne.value].copy(), "elite_slot": es[:ne.value].copy(),
            "restart_gid": rg[:nr.value].copy(), "restart_src": rs[:nr.value].copy()}


def lp_pdhg(problem: Problem, checkpoints=(100, 1000, 10000), step: float = 0.0, restart_period: int = 400,
            stream=None):
    """chap_lp_pdhg: the streamed PDHG snapshots of the LP relaxation.
    Returns (x [n_cp][n] device tensor, info numpy [n_cp][4] = iteration, c.x, max violation, step)."""
    import torch
    cps = np.ascontiguousarray(checkpoints, np.int64)
    x = torch.empty((len(cps), problem.n), dtype=torch.float64, device=f"cuda:{problem.device}")
    info = np.zeros((len(cps), 4))
    _check(chap_lp_pdhg(problem.h, cps.ctypes.data, int(len(cps)), float(step), int(restart_period), _ptr(x),
                        info.ctypes.data, _stream(stream)))
    return x, info


def lp_round(problem: Problem, x_lp, stream=None):
    """chap_lp_round: an LP point to a tabu start point (integers rounded, bounds clamped)."""
    import torch
    out = torch.empty_like(x_lp)
    _check(chap_lp_round(problem.h, _ptr(x_lp.contiguous()), _ptr(out), _stream(stream)))
    return out
