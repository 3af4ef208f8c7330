"""GPU parity at the BASELINE.json config sizes: the CUDA
path, called through the C-ABI, against the UNMODIFIED reference's results
recorded in tests/golden/config_vectors.json (tests/golden/make_config_golden.py,
oracle/_ref run multi-threaded in the CPU container).

Bar: bit-exact — sha256 of the canonical partition, block count, pass count,
closure steps, the reference's peak-memory estimate and (sortPR) the per-pass
block counts.  Inputs are regenerated here (device generator for random_dfa,
the oracle's C generators otherwise) and their sha256 is checked against the
digest of the reference-generated input first, so a mismatch in the result can
never be an input mismatch.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from tests.helpers import digest, gen, to_dfa

pytestmark = pytest.mark.gpu
MIN = dfm.RacePolicy.deterministic_min
ALGO = {"sort": dfm.Algo.sort, "naive_min": dfm.Algo.naive, "transpr_min": dfm.Algo.transpr,
        "trans": dfm.Algo.trans}

with open(os.path.join(os.path.dirname(__file__), "golden", "config_vectors.json")) as _f:
    VECTORS = json.load(_f)["vectors"]


def _input_digest(delta: np.ndarray, acc: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(delta, dtype="<u4").data)
    h.update(np.ascontiguousarray(acc, dtype=np.uint8).data)
    return h.hexdigest()


def _device_input(eng, rec):
    spec = rec["spec"]
    if spec[0] == "random" and rec["n"] >= 1_000_000:
        _, n, k, seed, p = spec
        dd = eng.random_dfa_device(n, k, seed, p)
        host = dd.download()
        assert _input_digest(host.delta, host.accepting) == rec["input_sha256"]
        return dd
    delta, acc = gen(spec)
    assert _input_digest(delta, acc) == rec["input_sha256"], rec["name"]
    return eng.upload(to_dfa((delta, acc)))


def _run(eng, algo, dd, n):
    import torch
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = eng.run_device(ALGO[algo], dd, dfm.AlgoRunConfig(policy=MIN),
                            block_out_ptr=out.data_ptr())
    torch.cuda.synchronize()
    return nb, st, out.cpu().numpy().view(np.uint32)


def _check(rec, algo, nb, st, labels):
    exp = rec[algo]
    what = (rec["name"], algo)
    assert st.status == dfm.RunStatus.ok, what
    assert nb == exp["num_blocks"], what
    assert st.iterations == exp["iterations"], what
    assert st.closure_steps == exp["closure_steps"], what
    assert st.peak_memory_estimate == exp["peak_memory_estimate"], what
    assert digest(labels) == exp["sha256"], what


@pytest.mark.parametrize("rec", VECTORS, ids=[v["name"] for v in VECTORS])
def test_config_vector(eng, eng_radix, rec):
    dd = _device_input(eng, rec)
    try:
        for algo in ("sort", "naive_min", "transpr_min", "trans"):
            if algo not in rec:
                continue
            engines = (eng, eng_radix) if algo == "sort" else (eng,)
            for e in engines:
                nb, st, labels = _run(e, algo, dd, rec["n"])
                _check(rec, algo, nb, st, labels)
            if algo == "sort" and rec["n"] <= 10_000_000:
                # the host-buffer entry point (dfm_sort_pr) with its per-pass trace
                host = dd.download()
                tr = dfm.SortTrace()
                r = eng.sort_pr(host, dfm.SortOptions(trace=tr))
                assert tr.block_counts == rec["sort"]["trace_counts"], rec["name"]
                assert digest(r.partition.block) == rec["sort"]["sha256"], rec["name"]
    finally:
        dd.free()
