"""CPU-only: the C-ABI library loads and exports every function include/chap.h declares; the
binding's struct layouts match the header; the oracle and the product path share no code."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "chap.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chap_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    so = os.path.join(ROOT, "paper_2605_05086_b200", "libchap.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = set(re.findall(r" T (chap_\w+)", out))
    declared = _declared()
    assert len(declared) >= 18
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    import paper_2605_05086_b200 as chap
    assert set(declared) <= set(chap.EXPORTED)
    assert chap.chap_abi_version() == 4
    assert chap.chap_status_string(7) == b"CHAP_ERR_UNSUPPORTED"


def test_struct_sizes_match_header():
    import ctypes
    import paper_2605_05086_b200 as chap
    assert ctypes.sizeof(chap.chap_move) == 24
    assert ctypes.sizeof(chap.chap_step_record) == 48
    assert ctypes.sizeof(chap.chap_walker_stats) == 64
    p = chap.default_params()
    assert (p.tenure, p.weight_cap, p.exchange_K, p.n_elite, p.n_restart) == (10, 1e6, 1000, 4, -1)
    assert (p.graph_iters, p.binary_kernel, p.pdl) == (16, 0, 0)


def test_invalid_args_fail_loudly_without_gpu():
    import numpy as np
    import paper_2605_05086_b200 as chap
    # validation happens on the host before any device work
    with pytest.raises(chap.ChapError) as e:
        chap.Problem(1, 1, np.array([0, 2]), np.array([0, 0]), np.array([1.0, 1.0]), np.array([-np.inf]),
                     np.array([1.0]), np.zeros(1), np.ones(1), np.ones(1, np.uint8), np.zeros(1))
    assert e.value.status == 1 and "duplicate" in str(e.value)
    with pytest.raises(chap.ChapError) as e:
        chap.Problem(1, 0, np.array([0]), np.zeros(0, np.int32), np.zeros(0), np.zeros(0), np.zeros(0),
                     np.array([0.2]), np.array([0.8]), np.ones(1, np.uint8), np.zeros(1))
    assert e.value.status in (2, 3)   # infeasible bounds (or no device on a CPU box)


def test_oracle_and_cuda_path_share_nothing():
    prod = os.path.join(ROOT, "paper_2605_05086_b200")
    orc = os.path.join(ROOT, "oracle")
    for d, forbidden in ((prod, ("oracle", "chap_oracle")), (orc, ("paper_2605_05086_b200", "chap.h", "common.cuh"))):
        for root, _, files in os.walk(d):
            for f in files:
                if f.endswith((".py", ".c", ".h", ".cu", ".cuh")):
                    txt = open(os.path.join(root, f)).read()
                    for bad in forbidden:
                        pat = (r'^\s*(#\s*include\s*[<"][^>"]*' + re.escape(bad) + r'|import\s+' + re.escape(bad) +
                               r'|from\s+' + re.escape(bad) + r')')
                        assert not re.search(pat, txt, flags=re.M), (f, bad)


def test_binding_structs_match_header_layout(tmp_path):
    """Every ABI struct of include/chap.h: size and field offsets as gcc lays them out equal the
    ctypes binding's (catches header/binding drift without a GPU)."""
    import ctypes
    import paper_2605_05086_b200 as chap
    structs = ["chap_problem_info", "chap_move", "chap_params", "chap_step_record", "chap_walker_stats",
               "chap_result", "chap_walker_summary"]
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "chap.h"', "int main(void) {"]
    for sname in structs:
        src.append(f'  printf("{sname} size %zu\\n", sizeof({sname}));')
        for fname, _ in getattr(chap, sname)._fields_:
            src.append(f'  printf("{sname} {fname} %zu\\n", offsetof({sname}, {fname}));')
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    got = {}
    for line in subprocess.check_output([str(exe)]).decode().splitlines():
        sname, field, val = line.split()
        got[(sname, field)] = int(val)
    for sname in structs:
        cls = getattr(chap, sname)
        assert got[(sname, "size")] == ctypes.sizeof(cls), sname
        for fname, _ in cls._fields_:
            assert got[(sname, fname)] == getattr(cls, fname).offset, (sname, fname)
