"""CPU: the C-ABI library builds, loads and exports every symbol include/*.h
declares; host-only entry points behave; the engine refuses to run without a
GPU (no silent CPU fallback)."""
import ctypes
import glob
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(dfm_\w+)\s*\(", text, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("dfm_sort_pr", "dfm_naive_pr", "dfm_naive_pr_cas", "dfm_expand_alphabet",
              "dfm_trans_pr", "dfm_trans_minimize", "dfm_run_algorithm", "dfm_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    path = dfm.lib_path()
    assert os.path.exists(path), "libdfm.so not built"
    lib = ctypes.CDLL(path)
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert declared_symbols() <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", dfm.lib_path()], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_formulas_match_the_reference(pins):
    lib = dfm._load()
    for n, lv in pins["transpr"]["power_levels"]["values"].items():
        assert lib.dfm_power_levels(int(n)) == lv == dfm.power_levels(int(n))
    assert lib.dfm_expand_required_bytes(256, 1) == 9 * 256 * 4
    for n, b in pins["trans"]["required_bytes"]["values"].items():
        assert lib.dfm_trans_required_bytes(int(n)) == b == dfm.trans_required_bytes(int(n))
    assert lib.dfm_trans_required_bytes(1 << 20) == 2 ** 64 - 1  # saturates


def test_host_generator_bit_exact():
    for n, k, seed, p in ((1, 1, 3, 0.5), (1000, 3, 7, 0.3), (70000, 2, 1, 0.5)):
        d = dfm.random_dfa(n, k, seed, p)
        od, oa = O.random_dfa(n, k, seed, p)
        assert (d.delta == od).all() and (d.accepting == oa).all()


def test_host_canonicalize_and_equal():
    raw = np.array([7, 7, 3, 9, 3, 7], np.uint32)
    p = dfm.canonicalize(raw)
    assert p.block.tolist() == [0, 0, 1, 2, 1, 0] and p.num_blocks == 3
    assert p.block.tolist() == O.canonicalize(raw)[0].tolist()
    assert dfm.partitions_equal(dfm.Partition(raw, 3), p)
    with pytest.raises(ValueError):
        dfm.partitions_equal(p, dfm.Partition(raw[:2], 1))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU refusal")
def test_engine_refuses_without_gpu():
    with pytest.raises(dfm.EngineUnavailable):
        dfm.Engine(0)
