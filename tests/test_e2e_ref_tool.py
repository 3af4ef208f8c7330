"""tools/cpp/e2e_ref.cpp (the C++ drop-in e2e on the reference's own types, built
where the reference headers exist): its inputs are the same DFAs as the Python
generators (FNV-1a digest), and on the GPU it minimizes to the oracle's result."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from paper_2410_22764_b200 import generators as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "build", "e2e_ref")
pytestmark = pytest.mark.skipif(not os.path.exists(TOOL), reason="build/e2e_ref not built")


def fnv(d) -> str:
    h = 0xcbf29ce484222325
    data = np.ascontiguousarray(d.delta, dtype="<u4").tobytes() + d.accepting.tobytes()
    arr = np.frombuffer(data, np.uint8)
    for b in arr.tolist():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def run(*args):
    r = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_inputs_match_python_generators():
    assert run("vlts", 100, 2000, 5, -1)["digest"] == fnv(G.vlts_dfa(100, 2000, 5))
    assert run("random", 1000, 3, 7, -1)["digest"] == fnv(dfm.random_dfa(1000, 3, 7, 0.5))


@pytest.mark.gpu
def test_minimizes_like_the_oracle():
    from oracle import oracle as O
    for args, pair in ((("vlts", 200, 20000, 10), O.vlts_dfa(200, 20000, 10)),
                       (("random", 30000, 3, 5), O.random_dfa(30000, 3, 5, 0.5))):
        out = run(*args, 2)
        ref = O.sort_pr(*pair)
        assert (out["blocks"], out["passes"]) == (ref.num_blocks, ref.iterations)


def part_digest(block) -> str:
    b = np.asarray(block, dtype=np.uint64)
    i = np.arange(b.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return f"{int((b * (np.uint64(2654435761) * i + np.uint64(1))).sum(dtype=np.uint64)):016x}"


@pytest.mark.gpu
def test_large_partitions_through_the_output_hook():
    """Partitions of >= 64 MB are prepared on a helper thread while the library works
    and handed over through the out-ready hook (dfm_ctx_set_out_ready_hook): the C++
    result equals the Python host-buffer result — an identity one (written by the
    speculative iota thread) and a non-identity one (D2H)."""
    eng = dfm.Engine(0)
    for args, d in ((("random", 20_000_000, 2, 3), dfm.random_dfa(20_000_000, 2, 3, 0.5)),
                    (("vlts", 1000, 20_000_000, 4), G.vlts_dfa(1000, 20_000_000, 4))):
        out = run(*args, 1)
        r = eng.sort_pr(d)
        assert (out["blocks"], out["passes"]) == (r.partition.num_blocks, r.stats.iterations)
        assert out["partition_digest"] == part_digest(r.partition.block), args
