"""CPU: pin the oracle restatement against the reference's golden vectors and
known-answer tests (tests/golden/*), and against the reference itself
(oracle/_ref) on seeded random inputs when it is built."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import digest, gen


def test_generators_match_pins(pins):
    g = pins["generators"]
    d, a = O.bit_splitter(3)
    assert d.tolist() == g["bits3"]["delta"]
    d, a = O.fib_dfa(5)
    assert np.flatnonzero(a).tolist() == g["fib5_acc_states"]["value"]
    assert O.fib_dfa(4)[1].tolist() == g["fib4_acc"]["value"]
    assert [O.fib_len(i) for i in range(12)] == g["fib_lengths"]["value"]
    for b in range(1, 11):
        d, a = O.bit_splitter(b)
        assert d.shape == (b - 1, 1 << b)
        assert (a == (np.arange(1 << b) >= (1 << (b - 1)))).all()


@pytest.mark.parametrize("idx", range(9))
def test_golden_vectors(golden, idx):
    # the 61 vectors are checked in 9 interleaved slices to keep each test short
    for rec in golden["vectors"][idx::9]:
        delta, acc = gen(rec["spec"])
        assert delta.shape == (rec["k"], rec["n"])
        runs = {"sort": lambda: O.sort_pr(delta, acc, trace=(tr := [])),
                "naive_min": lambda: O.naive_pr(delta, acc, "min"),
                "naive_max": lambda: O.naive_pr(delta, acc, "max"),
                "transpr_min": lambda: O.trans_pr(delta, acc, "min")}
        for key, run in runs.items():
            if key not in rec:
                continue
            if key == "naive_min" and rec["n"] > 5000:
                continue  # CPU-suite budget; the GPU suite covers these sizes
            exp = rec[key]
            tr = []
            r = O.sort_pr(delta, acc, trace=tr) if key == "sort" else run()
            assert r.num_blocks == exp["num_blocks"], (rec["name"], key)
            assert r.iterations == exp["iterations"], (rec["name"], key)
            assert r.closure_steps == exp["closure_steps"], (rec["name"], key)
            assert r.peak_memory_estimate == exp["peak_memory_estimate"], (rec["name"], key)
            assert digest(r.block) == exp["sha256"], (rec["name"], key)
            if key == "sort":
                assert [c for c, _ in tr] == exp["trace_counts"]
        if "trans" in rec:
            ins = {}
            r = O.trans_minimize(delta, acc, inspect=ins)
            assert r.block.tolist() == rec["trans"]["block"]
            assert r.iterations == rec["trans"]["iterations"]
            assert ins["apart_popcounts"].tolist() == rec["trans"]["apart_popcounts"]


def test_known_answers(pins):
    for idx in pins["fib_law"]["indices"]:
        d, a = O.fib_dfa(idx)
        N = a.size
        for r in (O.sort_pr(d, a), O.naive_pr(d, a, "min")):
            assert r.num_blocks == N and r.iterations == N - 1
    for b in pins["bits_law"]["bits"]:
        d, a = O.bit_splitter(b)
        for r in (O.sort_pr(d, a), O.naive_pr(d, a, "min")):
            assert r.num_blocks == 1 << b and r.iterations == max(b, 1)
    for f in pins["flat"]:
        d, a = O.random_dfa(*f["random"])
        r = {"sort": lambda: O.sort_pr(d, a), "naive_min": lambda: O.naive_pr(d, a, "min"),
             "transpr_min": lambda: O.trans_pr(d, a, "min"),
             "trans": lambda: O.trans_minimize(d, a)}[f["algo"]]()
        assert (r.num_blocks, r.iterations) == (f["blocks"], f["iterations"]), f
    for fp in pins["sort_first_pass_counts"]:
        if fp["family"] == "bits":
            d, a = O.bit_splitter(fp["arg"])
        else:
            d, a = np.array(fp["delta"], np.uint32), np.array(fp["acc"], np.uint8)
        tr = []
        O.sort_pr(d, a, trace=tr)
        assert tr[0][0] == fp["first_count"]
        counts = [c for c, _ in tr]
        assert all(x < y for x, y in zip(counts[:-2], counts[1:-1])) and counts[-1] == counts[-2]


def test_transpr_pins(pins):
    t = pins["transpr"]
    for n, lv in t["power_levels"]["values"].items():
        assert O.power_levels(int(n)) == lv
    rows, levels = O.expand_alphabet(*O.chain_dfa(10))
    assert levels == t["chain10"]["levels"] and rows[3 * 1 + 0][0] == t["chain10"]["row_0_3_at_0"]
    assert O.trans_pr(*O.chain_dfa(1024)).closure_steps == t["chain1024_closure_steps"]["value"]
    with pytest.raises(MemoryError) as ei:
        O.expand_alphabet(*O.chain_dfa(t["guard"]["chain"]), max_memory_bytes=t["guard"]["limit"])
    assert ei.value.required_bytes == t["guard"]["required"]
    r = O.trans_pr(*O.chain_dfa(256), max_memory_bytes=64)
    assert r.status == "capacity-exceeded" and r.block.size == 0
    assert [O.trans_pr(*O.fib_dfa(i)).iterations for i in range(5, 13)] == t["fib_5_12"]["iterations"]
    for k in t["chain_pow2"]["k"][:6]:
        r = O.trans_pr(*O.chain_dfa(1 << k))
        assert (r.iterations, r.closure_steps) == (k + 1, k)
    c = pins["comb"]
    for L in ("64", "1024"):
        d, a = O.comb_dfa(int(L), c["t"])
        e = c["L"][L]
        assert O.moore(d, a).num_blocks == e["blocks"]
        assert O.sort_pr(d, a).iterations == e["sort"]
        assert O.naive_pr(d, a).iterations == e["naive"]
        r = O.trans_pr(d, a)
        assert (r.iterations, r.closure_steps) == (e["transpr"], e["closure"])


def test_trans_pins(pins):
    t = pins["trans"]
    for idx, passes in t["fib_passes"]["values"].items():
        d, a = O.fib_dfa(int(idx))
        r = O.trans_minimize(d, a)
        assert r.iterations == passes and r.num_blocks == a.size
    d, a = O.random_dfa(*t["guard"]["random"])
    r = O.trans_minimize(d, a, max_memory_bytes=t["guard"]["limit"])
    assert r.status == "capacity-exceeded" and r.peak_memory_estimate == t["guard"]["peak"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_equals_reference_random():
    R = O.Reference()
    R.set_threads(1)
    rng = np.random.default_rng(1001)
    for t in range(120):
        n = int(rng.integers(1, 200))
        k = int(rng.integers(1, 5))
        p = [0.0, 0.1, 0.5, 1.0][t % 4]
        d, a = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), p)
        for mine, ref in ((O.sort_pr(d, a), R.sort_pr(d, a)),
                          (O.naive_pr(d, a, "min"), R.naive_pr(d, a, "min")),
                          (O.naive_pr(d, a, "max"), R.naive_pr(d, a, "max")),
                          (O.trans_pr(d, a, "min"), R.trans_pr(d, a, "min"))):
            assert (mine.block == ref.block).all()
            assert (mine.num_blocks, mine.iterations, mine.closure_steps) == \
                (ref.num_blocks, ref.iterations, ref.closure_steps)
        assert (O.moore(d, a).block == R.moore(d, a).block).all()
        if n <= 24:
            assert (O.trans_minimize(d, a).block == R.trans_minimize(d, a).block).all()


def test_post_processing_vs_reference():
    """quotient / remove_unreachable restated (dfm_oracle.c) == the reference itself."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    R = O.Reference()
    rng = np.random.default_rng(5)
    for t in range(200):
        n = int(rng.integers(1, 60))
        k = int(rng.integers(0, 4))
        d, a = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), [0, 0.1, 0.5, 1][t % 4])
        ini = int(rng.integers(0, n))
        x, y = O.remove_unreachable(d, a, ini), R.remove_unreachable(d, a, ini)
        assert (x[0] == y[0]).all() and (x[1] == y[1]).all() and x[2] == y[2]
        r = O.sort_pr(d, a)
        x, y = O.quotient(d, a, r.block, r.num_blocks, ini), R.quotient(d, a, r.block, r.num_blocks, ini)
        assert (x[0] == y[0]).all() and (x[1] == y[1]).all() and x[2] == y[2]
        bad = rng.integers(0, 3, n).astype(np.uint32)
        c, nb = O.canonicalize(bad)
        for blk, nbb in ((bad, 3), (c, nb), (c, nb + 1)):
            e1 = e2 = None
            try:
                O.quotient(d, a, blk, nbb, ini)
            except O.QuotientError as e:
                e1 = str(e)
            try:
                R.quotient(d, a, blk, nbb, ini)
            except O.QuotientError as e:
                e2 = str(e)
            assert e1 == e2
