"""GPU parity: libdfm (sm_100a kernels, called through the C-ABI) against the
oracle, the reference's golden vectors and its known-answer tests.  Bar:
bit-exact canonical partition, block count, pass count and closure steps."""
import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O
from tests.helpers import digest, gen, to_dfa

pytestmark = pytest.mark.gpu
MIN, MAX, ARB = (dfm.RacePolicy.deterministic_min, dfm.RacePolicy.deterministic_max,
                 dfm.RacePolicy.arbitrary_winner)


def check(r, exp, what):
    assert r.stats.status == dfm.RunStatus.ok, what
    assert r.partition.num_blocks == exp["num_blocks"], what
    assert r.stats.iterations == exp["iterations"], what
    assert r.stats.closure_steps == exp["closure_steps"], what
    assert r.stats.peak_memory_estimate == exp["peak_memory_estimate"], what
    assert digest(r.partition.block) == exp["sha256"], what


def test_golden_vectors(eng, eng_radix, golden):
    for rec in golden["vectors"]:
        d = to_dfa(gen(rec["spec"]))
        for e in (eng, eng_radix):
            tr = dfm.SortTrace()
            check(e.sort_pr(d, dfm.SortOptions(trace=tr)), rec["sort"], (rec["name"], "sort"))
            assert tr.block_counts == rec["sort"]["trace_counts"], rec["name"]
        if "naive_min" in rec:
            check(eng.naive_pr(d, dfm.PrOptions(policy=MIN)), rec["naive_min"], (rec["name"], "min"))
            check(eng.naive_pr(d, dfm.PrOptions(policy=MAX)), rec["naive_max"], (rec["name"], "max"))
            check(eng.trans_pr(d, dfm.PrOptions(policy=MIN)), rec["transpr_min"],
                  (rec["name"], "transpr"))
            # scheduling-dependent pass counts: only the partition is pinned
            assert digest(eng.naive_pr(d, dfm.PrOptions(policy=ARB)).partition.block) == \
                rec["naive_min"]["sha256"]
            assert digest(eng.naive_pr_cas(d).partition.block) == rec["naive_min"]["sha256"]
        if "trans" in rec:
            ins = dfm.TransInspect()
            r = eng.trans_minimize(d, inspect=ins)
            assert r.partition.block.tolist() == rec["trans"]["block"], rec["name"]
            assert r.stats.iterations == rec["trans"]["iterations"], rec["name"]
            assert ins.apart_popcounts == rec["trans"]["apart_popcounts"], rec["name"]


def test_oracle_agreement_500(eng, eng_radix):
    """acceptance.cpp:40-79 grid, checked against the C oracle."""
    rng = np.random.default_rng(1001)
    for rnd in range(500):
        n = int(rng.integers(1, 513))
        k = int(rng.integers(1, 5))
        p = [0.0, 0.1, 0.5, 1.0][rnd % 4]
        pair = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), p)
        d = to_dfa(pair)
        ref = O.sort_pr(*pair)
        for e in (eng, eng_radix):
            r = e.sort_pr(d)
            assert r.partition.block.tolist() == ref.block.tolist() and \
                r.stats.iterations == ref.iterations, (rnd, n, k)
        ref_min = O.naive_pr(*pair, "min")
        r = eng.naive_pr(d, dfm.PrOptions(policy=MIN))
        assert (r.partition.block == ref_min.block).all() and \
            r.stats.iterations == ref_min.iterations, (rnd, n, k)
        assert (eng.naive_pr_cas(d).partition.block == ref.block).all()
        ref_tp = O.trans_pr(*pair, "min")
        r = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
        assert (r.partition.block == ref_tp.block).all()
        assert (r.stats.iterations, r.stats.closure_steps) == (ref_tp.iterations, ref_tp.closure_steps)
        if n <= 64:
            ref_t = O.trans_minimize(*pair)
            r = eng.trans_minimize(d)
            assert (r.partition.block == ref_t.block).all() and \
                r.stats.iterations == ref_t.iterations, (rnd, n, k)


def test_iteration_laws(eng, pins):
    for idx in pins["fib_law"]["indices"]:
        d = to_dfa(O.fib_dfa(idx))
        N = d.num_states
        for r in (eng.sort_pr(d), eng.naive_pr(d, dfm.PrOptions(policy=MIN))):
            assert (r.partition.num_blocks, r.stats.iterations) == (N, N - 1)
    for b in pins["bits_law"]["bits"]:
        d = to_dfa(O.bit_splitter(b))
        for r in (eng.sort_pr(d), eng.naive_pr(d, dfm.PrOptions(policy=MIN))):
            assert (r.partition.num_blocks, r.stats.iterations) == (1 << b, max(b, 1))
    for f in pins["flat"]:
        d = to_dfa(O.random_dfa(*f["random"]))
        r = {"sort": lambda: eng.sort_pr(d),
             "naive_min": lambda: eng.naive_pr(d, dfm.PrOptions(policy=MIN)),
             "transpr_min": lambda: eng.trans_pr(d, dfm.PrOptions(policy=MIN)),
             "trans": lambda: eng.trans_minimize(d)}[f["algo"]]()
        assert (r.partition.num_blocks, r.stats.iterations) == (f["blocks"], f["iterations"]), f
    for fp in pins["sort_first_pass_counts"]:
        pair = O.bit_splitter(fp["arg"]) if fp["family"] == "bits" else \
            (np.array(fp["delta"], np.uint32), np.array(fp["acc"], np.uint8))
        tr = dfm.SortTrace()
        eng.sort_pr(to_dfa(pair), dfm.SortOptions(trace=tr))
        c = tr.block_counts
        assert c[0] == fp["first_count"]
        assert all(x < y for x, y in zip(c[:-2], c[1:-1])) and c[-1] == c[-2]


def test_edge_cases(eng):
    lone = dfm.Dfa.from_rows([[0]], [1])
    for r in (eng.sort_pr(lone), eng.naive_pr(lone, dfm.PrOptions(policy=MIN)),
              eng.naive_pr_cas(lone), eng.trans_pr(lone, dfm.PrOptions(policy=MIN)),
              eng.trans_minimize(lone)):
        assert (r.partition.num_blocks, r.stats.iterations) == (1, 1)
    b1 = to_dfa(O.bit_splitter(1))  # empty alphabet: keys reduce to the block label
    assert b1.alphabet_size == 0
    r = eng.sort_pr(b1)
    assert r.partition.num_blocks == 2 and r.stats.iterations == 1
    bad = dfm.Dfa.from_rows([[0, 5]], [0, 1])
    with pytest.raises(dfm.EngineError):
        eng.sort_pr(bad)
    with pytest.raises(dfm.EngineError):
        eng.run_algorithm(dfm.Algo.oracle, lone)
    # the context survives a rejected call
    assert eng.sort_pr(lone).partition.num_blocks == 1


def test_transpr_pins(eng, pins):
    t = pins["transpr"]
    d = to_dfa(O.chain_dfa(10))
    e = eng.expand_alphabet(d)
    assert e.levels == t["chain10"]["levels"] and e.row(0, 3)[0] == t["chain10"]["row_0_3_at_0"]
    assert (e.row(0, 0) == d.delta[0]).all()
    ident = dfm.Dfa(10, 2, np.vstack([d.delta, np.arange(10, dtype=np.uint32)]), d.accepting)
    e2 = eng.expand_alphabet(ident)
    assert all((e2.row(1, lv) == np.arange(10)).all() for lv in range(e2.levels))
    rng = np.random.default_rng(71)
    for _ in range(15):
        pair = O.random_dfa(int(rng.integers(1, 65)), int(rng.integers(1, 4)),
                            int(rng.integers(1, 2 ** 62)), 0.5)
        rows, levels = O.expand_alphabet(*pair)
        e = eng.expand_alphabet(to_dfa(pair))
        assert e.levels == levels and (e.delta == rows).all()
    tiny = dfm.Limits(max_memory_bytes=t["guard"]["limit"])
    with pytest.raises(dfm.CapacityError) as ei:
        eng.expand_alphabet(to_dfa(O.chain_dfa(256)), tiny)
    assert ei.value.required_bytes() == t["guard"]["required"]
    r = eng.trans_pr(to_dfa(O.chain_dfa(256)), dfm.PrOptions(policy=MIN), tiny)
    assert r.stats.status == dfm.RunStatus.capacity_exceeded and r.partition.block.size == 0
    assert r.stats.peak_memory_estimate == t["guard"]["required"]
    assert eng.trans_pr(to_dfa(O.chain_dfa(1024)), dfm.PrOptions(policy=MIN)).stats.closure_steps == 10
    c64 = to_dfa(O.chain_dfa(64))
    plain = eng.naive_pr(c64, dfm.PrOptions(policy=MIN))
    closed = eng.trans_pr(c64, dfm.PrOptions(policy=MIN))
    assert plain.stats.iterations == 63 and closed.stats.iterations <= 14
    assert closed.partition.num_blocks == 64
    r = eng.trans_pr(to_dfa(O.fib_dfa(21)), dfm.PrOptions(policy=MIN))
    f = t["fib21"]
    assert (r.stats.iterations, r.stats.closure_steps, r.partition.num_blocks) == \
        (f["iterations"], f["closure_steps"], f["blocks"])
    assert [eng.trans_pr(to_dfa(O.fib_dfa(i)), dfm.PrOptions(policy=MIN)).stats.iterations
            for i in range(5, 13)] == t["fib_5_12"]["iterations"]
    for k in t["chain_pow2"]["k"]:
        r = eng.trans_pr(to_dfa(O.chain_dfa(1 << k)), dfm.PrOptions(policy=MIN))
        assert (r.stats.iterations, r.stats.closure_steps) == (k + 1, k)


def test_trans_pins(eng, pins):
    t = pins["trans"]
    for idx, passes in {**t["fib_passes"]["values"], **t["fib_10_11"]["values"]}.items():
        d = to_dfa(O.fib_dfa(int(idx)))
        r = eng.trans_minimize(d)
        assert (r.stats.iterations, r.partition.num_blocks) == (passes, d.num_states)
    d = to_dfa(O.random_dfa(*t["guard"]["random"]))
    r = eng.trans_minimize(d, dfm.Limits(max_memory_bytes=t["guard"]["limit"]))
    assert r.stats.status == dfm.RunStatus.capacity_exceeded
    assert r.stats.peak_memory_estimate == t["guard"]["peak"] and r.partition.block.size == 0
    # apartness invariants (test_min_trans.cpp:65-113)
    rng = np.random.default_rng(82)
    for _ in range(20):
        n = int(rng.integers(2, 13))
        k = int(rng.integers(1, 4))
        pair = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), 0.4)
        ins = dfm.TransInspect()
        eng.trans_minimize(to_dfa(pair), inspect=ins)
        A = ins.apart.reshape(n, n).astype(bool)
        assert not A.diagonal().any() and (A == A.T).all()
        notA = ~A
        assert not (notA.astype(int) @ notA.astype(int) > 0)[A].any()  # transitivity of not-apart
        delta = pair[0]
        for a in range(k):
            assert not (A[np.ix_(delta[a], delta[a])] & notA).any()  # edge-closed
        assert all(x <= y for x, y in zip(ins.apart_popcounts, ins.apart_popcounts[1:]))


def test_timeouts_report_status(eng):
    r = eng.sort_pr(to_dfa(O.fib_dfa(18)), 1)
    assert r.stats.status == dfm.RunStatus.timeout and r.partition.block.size == 0
    r = eng.naive_pr(to_dfa(O.fib_dfa(18)), dfm.PrOptions(policy=MIN, timeout_ms=1))
    assert r.stats.status == dfm.RunStatus.timeout and r.partition.block.size == 0
    r = eng.trans_minimize(to_dfa(O.fib_dfa(11)), dfm.Limits(timeout_ms=1))
    assert r.stats.status == dfm.RunStatus.timeout and r.partition.block.size == 0


def test_c1_and_comb_pins(eng, eng_radix, pins):
    c = pins["c1"]
    for seed, exp in c["seeds"].items():
        d = to_dfa(O.random_dfa(c["n"], c["k"], int(seed), c["p"]))
        for e in (eng, eng_radix):
            tr = dfm.SortTrace()
            r = e.sort_pr(d, dfm.SortOptions(trace=tr) if seed == "1" else None)
            assert (r.stats.iterations, r.partition.num_blocks) == (exp["sort"], c["blocks"])
            if seed == "1":
                assert tr.block_counts == c["seed1_sort_trace"]
        r = eng.naive_pr(d, dfm.PrOptions(policy=MIN))
        assert (r.stats.iterations, r.partition.num_blocks) == (exp["naive_min"], c["blocks"])
    for L, e in pins["comb"]["L"].items():
        d = to_dfa(O.comb_dfa(int(L), pins["comb"]["t"]))
        assert eng.sort_pr(d).stats.iterations == e["sort"]
        assert eng_radix.sort_pr(d).stats.iterations == e["sort"]
        assert eng.naive_pr(d, dfm.PrOptions(policy=MIN)).stats.iterations == e["naive"]
        r = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
        assert (r.stats.iterations, r.stats.closure_steps, r.partition.num_blocks) == \
            (e["transpr"], e["closure"], e["blocks"])


def test_larger_inputs_vs_oracle(eng, eng_radix):
    for name, pair in (("random", O.random_dfa(1_000_000, 4, 5, 0.5)),
                       ("vlts", O.vlts_dfa(1000, 1_000_000, 10)),
                       ("random-k1", O.random_dfa(300_000, 1, 9, 0.5))):
        ref = O.sort_pr(*pair)
        d = to_dfa(pair)
        for e in (eng, eng_radix):
            r = e.sort_pr(d)
            assert r.stats.iterations == ref.iterations, name
            assert (r.partition.block == ref.block).all(), name
        if name == "vlts":  # transPR pass counts explode on random DFAs
            rt = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
            assert (rt.partition.block == ref.block).all()


def test_device_generator_bit_exact(eng):
    for n, k, seed in ((1, 1, 4), (12345, 3, 99), (1 << 20, 4, 1)):
        dd = eng.random_dfa_device(n, k, seed, 0.5)
        got = dd.download()
        od, oa = O.random_dfa(n, k, seed, 0.5)
        assert (got.delta == od).all() and (got.accepting == oa).all()
        dd.free()


def test_full_size_properties(eng, eng_radix):
    """1e8 states, k=4, seed 2 (the seed-1 north-star input is pinned bit-exactly against
    the reference in test_gpu_configs.py): size-independent checks of a congruence —
    labels canonical (first occurrences increasing), acceptance constant on blocks and
    every block's successor blocks a function of the block — and the hash and radix
    engines agree on partition and pass count."""
    import torch
    n, k = 100_000_000, 4
    dd = eng.random_dfa_device(n, k, 2, 0.5)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = eng.run_device(dfm.Algo.sort, dd, block_out_ptr=out.data_ptr())
    assert st.status == dfm.RunStatus.ok and 1 <= nb <= n
    out_r = torch.empty(n, dtype=torch.int32, device="cuda")
    nbr, str_ = eng_radix.run_device(dfm.Algo.sort, dd, block_out_ptr=out_r.data_ptr())
    assert (nbr, str_.iterations) == (nb, st.iterations)
    assert bool((out == out_r).all())
    del out_r
    host = dd.download()
    delta = torch.from_numpy(host.delta.view(np.int32)).cuda()
    acc = torch.from_numpy(host.accepting).cuda()
    lab = out.long()
    first = torch.full((nb,), n, dtype=torch.long, device="cuda").scatter_reduce(
        0, lab, torch.arange(n, device="cuda"), reduce="amin")
    assert bool((first[1:] > first[:-1]).all())
    acc_b = torch.zeros(nb, dtype=torch.uint8, device="cuda").scatter_(0, lab, acc)
    assert bool((acc_b[lab] == acc).all())
    for a in range(k):
        succ = lab[delta[a].long()]
        assert bool((succ == succ[first][lab]).all())
    dd.free()


def _device_labels(e, dd, n):
    import torch
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = e.run_device(dfm.Algo.sort, dd, block_out_ptr=out.data_ptr())
    assert st.status == dfm.RunStatus.ok
    return nb, st.iterations, out


@pytest.mark.parametrize("n,k,seed", [(12_000_000, 4, 3), (30_000_000, 2, 4),
                                      (12_000_000, 3, 5), (9_000_000, 9, 6),
                                      (12_000_001, 3, 7), (9_000_003, 5, 8)])
def test_blocked_signature_builder(eng, eng_radix, monkeypatch, n, k, seed):
    """The blocked (target-range bucketed) signature builder takes over the
    passes whose id mirror exceeds the L2 share; it must give the exact same
    canonical partition and pass count as the direct-gather path and the radix
    engine (both pinned against the oracle at smaller sizes)."""
    dd = eng.random_dfa_device(n, k, seed, 0.5)
    nb, it, lab = _device_labels(eng, dd, n)
    monkeypatch.setenv("DFM_SORTPR_BLOCKED", "0")
    nb0, it0, lab0 = _device_labels(eng, dd, n)
    monkeypatch.delenv("DFM_SORTPR_BLOCKED")
    nbr, itr, labr = _device_labels(eng_radix, dd, n)
    assert (nb, it) == (nb0, it0) == (nbr, itr)
    assert bool((lab == lab0).all()) and bool((lab == labr).all())
    dd.free()


@pytest.mark.parametrize("n,k,seed,wc", [(12_000_000, 4, 3, 97), (9_000_003, 5, 8, 1000),
                                         (17_000_000, 2, 11, 31)])
def test_chunked_layout(eng, monkeypatch, n, k, seed, wc):
    """Chunk-major layout (the pipelined upload builds it chunk by chunk as the
    rows arrive): forced chunking of wc windows gives the unchunked result."""
    dd = eng.random_dfa_device(n, k, seed, 0.5)
    nb, it, lab = _device_labels(eng, dd, n)
    monkeypatch.setenv("DFM_LAYOUT_CHUNK_WINDOWS", str(wc))
    nb1, it1, lab1 = _device_labels(eng, dd, n)
    monkeypatch.delenv("DFM_LAYOUT_CHUNK_WINDOWS")
    monkeypatch.setenv("DFM_SORTPR_TILE24", "0")  # 4-byte window tiles throughout
    nb2, it2, lab2 = _device_labels(eng, dd, n)
    assert (nb, it) == (nb1, it1) == (nb2, it2)
    assert bool((lab == lab1).all()) and bool((lab == lab2).all())
    dd.free()


def test_blocked_builder_vs_oracle(eng):
    """One blocked-path size checked straight against the CPU oracle."""
    pair = O.random_dfa(17_000_000, 2, 11, 0.5)
    ref = O.sort_pr(*pair)
    r = eng.sort_pr(to_dfa(pair))
    assert r.stats.iterations == ref.iterations
    assert (r.partition.block == ref.block).all()


@pytest.mark.parametrize("n,k,seed", [(12_000_000, 4, 3), (9_000_000, 12, 8)])
def test_partitioned_grouping(eng, monkeypatch, n, k, seed):
    """The opt-in partitioned shared-memory grouping gives the global-table result."""
    dd = eng.random_dfa_device(n, k, seed, 0.5)
    nb, it, lab = _device_labels(eng, dd, n)
    monkeypatch.setenv("DFM_SORTPR_PARTITION", "1")
    nb1, it1, lab1 = _device_labels(eng, dd, n)
    assert (nb, it) == (nb1, it1) and bool((lab == lab1).all())
    dd.free()


@pytest.mark.parametrize("case", [
    ("random", 100_000, 2, 1, 0.5),    # C1: every pass inside the persistent kernel
    ("random", 50_000, 8, 3, 0.5),     # keys outgrow 62 bits: the host loop takes over
    ("random", 3_000, 70, 4, 0.3),     # (k+1) > 62: host loop from the first pass
    ("random", 1 << 20, 1, 5, 0.5),    # largest small-kernel size, 8 states per thread
    ("random", 777, 3, 6, 0.0),        # one initial block
    ("fib", 20, 0, 0, 0.0),            # 10,945 states, N-1 passes over several launches
    ("chain", 5_000, 0, 0, 0.0),
    ("comb", 2_000, 3, 0, 0.0),
])
def test_small_persistent_sortpr(eng, monkeypatch, case):
    """sortPR's single-kernel path for n <= 2^20 (sortpr_small.cuh) against the
    oracle and against the host-driven loop (DFM_SORTPR_SMALL=0)."""
    kind, n, k, seed, p = case
    pair = {"random": lambda: O.random_dfa(n, k, seed, p), "fib": lambda: O.fib_dfa(n),
            "chain": lambda: O.chain_dfa(n), "comb": lambda: O.comb_dfa(n, k)}[kind]()
    d = to_dfa(pair)
    ref = O.sort_pr(*pair)
    r = eng.sort_pr(d)
    assert r.stats.status == dfm.RunStatus.ok
    assert (r.partition.num_blocks, r.stats.iterations) == (ref.num_blocks, ref.iterations)
    assert (r.partition.block == ref.block).all()
    monkeypatch.setenv("DFM_SORTPR_SMALL", "0")
    r2 = eng.sort_pr(d)
    assert r2.stats.iterations == r.stats.iterations
    assert (r2.partition.block == r.partition.block).all()


@pytest.mark.parametrize("policy", [MIN, MAX])
@pytest.mark.parametrize("case", [
    ("random", 100_000, 2, 1, 0.5),
    ("random", 20_000, 5, 7, 0.3),
    ("fib", 16, 0, 0, 0.0),
    ("vlts", 300_000, 10, 0, 0.0),
])
def test_naive_one_barrier_kernel(eng, monkeypatch, policy, case):
    """naivePR's one-barrier-per-pass persistent kernel (labels of the previous
    pass formed on the fly) against the oracle and the two-phase kernel."""
    kind, n, k, seed, p = case
    pair = {"random": lambda: O.random_dfa(n, k, seed, p), "fib": lambda: O.fib_dfa(n),
            "vlts": lambda: O.vlts_dfa(300, n, k)}[kind]()
    d = to_dfa(pair)
    ref = O.naive_pr(*pair, "min" if policy == MIN else "max")
    r = eng.naive_pr(d, dfm.PrOptions(policy=policy))
    assert r.stats.status == dfm.RunStatus.ok
    assert r.stats.iterations == ref.iterations
    assert (r.partition.block == ref.block).all()
    monkeypatch.setenv("DFM_NAIVE_FUSED", "0")
    r2 = eng.naive_pr(d, dfm.PrOptions(policy=policy))
    assert r2.stats.iterations == r.stats.iterations
    assert (r2.partition.block == r.partition.block).all()


def test_hashed_blocked_pass_with_repeated_keys(eng, eng_radix, monkeypatch):
    """vlts(1000, 2e7, 8): hashed (9 x 10-bit ids) blocked passes whose keys are
    mostly repeated — the signature rows deferred to the filter's candidates are
    then produced by a second window pass; same result as the direct path."""
    delta, acc = O.vlts_dfa(1000, 20_000_000, 8)
    dd = eng.upload(dfm.Dfa(20_000_000, 8, delta, acc, 0))
    nb, it, lab = _device_labels(eng, dd, 20_000_000)
    monkeypatch.setenv("DFM_SORTPR_BLOCKED", "0")
    nb0, it0, lab0 = _device_labels(eng, dd, 20_000_000)
    monkeypatch.delenv("DFM_SORTPR_BLOCKED")
    nbr, itr, labr = _device_labels(eng_radix, dd, 20_000_000)
    assert (nb, it) == (nb0, it0) == (nbr, itr) and nb <= 1000
    assert bool((lab == lab0).all()) and bool((lab == labr).all())
    dd.free()


def test_host_loop_relabel_in_place_vs_oracle(eng, monkeypatch):
    """The host-driven pass loop (small-n kernel off) with relabel-in-place direct
    passes (slot = new id) against the oracle, and against resolve/apply passes."""
    monkeypatch.setenv("DFM_SORTPR_SMALL", "0")
    rng = np.random.default_rng(4242)
    for rnd in range(120):
        n = int(rng.integers(1, 3000))
        k = int(rng.integers(0, 6))
        pair = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), [0.0, 0.1, 0.5, 1.0][rnd % 4])
        d = to_dfa(pair)
        ref = O.sort_pr(*pair)
        r = eng.sort_pr(d)
        assert (r.partition.num_blocks, r.stats.iterations) == (ref.num_blocks, ref.iterations), rnd
        assert (r.partition.block == ref.block).all(), rnd
    for pair in (O.fib_dfa(14), O.bit_splitter(9), O.comb_dfa(300, 3), O.random_dfa(200_000, 3, 9)):
        d = to_dfa(pair)
        ref = O.sort_pr(*pair)
        r = eng.sort_pr(d)
        monkeypatch.setenv("DFM_SORTPR_RIP", "0")
        r0 = eng.sort_pr(d)
        monkeypatch.delenv("DFM_SORTPR_RIP")
        for x in (r, r0):
            assert (x.partition.num_blocks, x.stats.iterations) == (ref.num_blocks, ref.iterations)
            assert (x.partition.block == ref.block).all()


@pytest.mark.parametrize("engine", ["hash", "radix"])
@pytest.mark.parametrize("n,k,seed", [(200_000, 4, 3), (12_000_000, 4, 3)])
def test_forced_hash_collisions_retry_exactly(eng, eng_radix, monkeypatch, n, k, seed, engine):
    """DFM_SORTPR_WEAK_HASH truncates the first seed's hashed keys to 10 bits: every
    hashed pass collides, is voided and redone under the next seed (direct passes,
    the filtered relabel-in-place pass, the radix engine's gather and blocked-builder
    keys and its leader-flag relabel included) — same result as without."""
    eng = eng if engine == "hash" else eng_radix
    monkeypatch.setenv("DFM_SORTPR_SMALL", "0")
    dd = eng.random_dfa_device(n, k, seed, 0.5)
    nb, it, lab = _device_labels(eng, dd, n)
    monkeypatch.setenv("DFM_SORTPR_WEAK_HASH", "10")
    nb1, it1, lab1 = _device_labels(eng, dd, n)
    monkeypatch.delenv("DFM_SORTPR_WEAK_HASH")
    _device_labels(eng, dd, n)  # mask restored
    assert (nb, it) == (nb1, it1)
    assert bool((lab == lab1).all())
    dd.free()


@pytest.mark.parametrize("name,pair", [
    ("vlts_k10", lambda: O.vlts_dfa(500, 200_000, 10)),
    ("vlts_k33", lambda: O.vlts_dfa(300, 60_000, 33)),
    ("random_k7", lambda: O.random_dfa(300_000, 7, 9, 0.5)),
    ("random_k40", lambda: O.random_dfa(20_000, 40, 10, 0.5)),
    ("random_k5", lambda: O.random_dfa(300_000, 5, 12, 0.5)),
    ("random_k3", lambda: O.random_dfa(300_000, 3, 11, 0.5)),  # compile-time k: rows unpacked
])
def test_packed_signature_rows(eng, monkeypatch, name, pair):
    """Direct hashed passes with a runtime alphabet (k > 4) pack their signature rows
    at the pass's mirror width (1/4/8/16/32-bit fields); compile-time alphabets
    (k <= 4) keep one word per field: the oracle's partition and pass count,
    also with every hashed pass forced to collide and retry (DFM_SORTPR_WEAK_HASH) so
    the packed rows are what verifies the groups."""
    delta, acc = pair()
    d = to_dfa((delta, acc))
    ref = O.sort_pr(delta, acc)
    monkeypatch.setenv("DFM_SORTPR_SMALL", "0")
    for weak in (None, "10"):
        if weak:
            monkeypatch.setenv("DFM_SORTPR_WEAK_HASH", weak)
        r = eng.sort_pr(d)
        monkeypatch.delenv("DFM_SORTPR_WEAK_HASH", raising=False)
        assert r.stats.iterations == ref.iterations, (name, weak)
        assert (r.partition.block == ref.block).all(), (name, weak)


def test_layout_built_beside_pass_one(eng, monkeypatch):
    """The blocked layout built on the side stream during pass 1 (device-resident
    input) gives the result of building it at pass 2."""
    n, k = 40_000_000, 4
    dd = eng.random_dfa_device(n, k, 12, 0.5)
    nb, it, lab = _device_labels(eng, dd, n)
    monkeypatch.setenv("DFM_SORTPR_LAYOUT_OVERLAP", "0")
    nb0, it0, lab0 = _device_labels(eng, dd, n)
    assert (nb, it) == (nb0, it0) and bool((lab == lab0).all())
    dd.free()



def test_one_barrier_kernel_all_policies_partition(eng):
    """Every election policy through the one-barrier kernel (a thread per state and
    grid-stride sizes) reaches the reference partition; det-min/max pass counts
    match the oracle's."""
    for pair in (O.random_dfa(50_000, 3, 31, 0.5), O.random_dfa(400_000, 2, 32, 0.5)):
        d = to_dfa(pair)
        ref = O.sort_pr(*pair)
        for pol in (MIN, MAX, ARB):
            r = eng.naive_pr(d, dfm.PrOptions(policy=pol))
            assert r.stats.status == dfm.RunStatus.ok
            assert (r.partition.block == ref.block).all(), pol
        if pair[0].shape[1] == 50_000:
            for pol, name in ((MIN, "min"), (MAX, "max")):
                assert eng.naive_pr(d, dfm.PrOptions(policy=pol)).stats.iterations == \
                    O.naive_pr(*pair, name).iterations


@pytest.mark.parametrize("name,pair", [
    ("vlts_k12", lambda: O.vlts_dfa(300, 60_000, 12)),
    ("random_k9", lambda: O.random_dfa(20_000, 9, 77, 0.5)),
    ("fib14_k1", lambda: O.fib_dfa(14)),
    ("comb_k2", lambda: O.comb_dfa(3000, 3)),
])
def test_naive_work_efficient_passes(eng, monkeypatch, name, pair):
    """The work-efficient fused pass (predecessor marks: a state re-evaluates only when
    a label it compares changed) gives the reference's partition AND pass count —
    forced on (DFM_NAIVE_DIRTY=1) for small alphabets too, and against it off."""
    delta, acc = pair()
    d = to_dfa((delta, acc))
    for pol, name_ in ((MIN, "min"), (MAX, "max")):
        ref = O.naive_pr(delta, acc, name_)
        for flag in ("1", "0"):
            monkeypatch.setenv("DFM_NAIVE_DIRTY", flag)
            r = eng.naive_pr(d, dfm.PrOptions(policy=pol))
            assert r.stats.iterations == ref.iterations, (name, name_, flag)
            assert (r.partition.block == ref.block).all(), (name, name_, flag)
    monkeypatch.setenv("DFM_NAIVE_DIRTY", "1")
    rt = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
    ref_t = O.trans_pr(delta, acc, "min")
    assert rt.stats.iterations == ref_t.iterations and (rt.partition.block == ref_t.block).all()
    assert (eng.naive_pr(d, dfm.PrOptions(policy=ARB)).partition.block ==
            O.naive_pr(delta, acc, "min").block).all()


@pytest.mark.parametrize("name,pair", [
    ("vlts_k12", lambda: O.vlts_dfa(300, 60_000, 12)),
    ("random_k9", lambda: O.random_dfa(20_000, 9, 77, 0.5)),
    ("random_k2", lambda: O.random_dfa(20_000, 2, 3, 0.5)),
])
def test_naive_dynamic_rows_and_queue(eng, monkeypatch, name, pair):
    """The kernels for inputs above the resident threads — dynamic round-robin rows of
    fused_pr_kernel (plain and letter-mask instances) and the opt-in queue_pr_kernel —
    forced on small inputs (DFM_NAIVE_ONE=0, marks from the first pass): the reference's
    partition and pass count under min and max; transPR too."""
    delta, acc = pair()
    d = to_dfa((delta, acc))
    monkeypatch.setenv("DFM_NAIVE_ONE", "0")
    for pol, name_ in ((MIN, "min"), (MAX, "max")):
        ref = O.naive_pr(delta, acc, name_)
        for dirty, queue in (("0", "0"), ("1", "0"), ("1", "1")):
            monkeypatch.setenv("DFM_NAIVE_DIRTY", dirty)
            monkeypatch.setenv("DFM_NAIVE_DIRTY_AFTER", "0")
            monkeypatch.setenv("DFM_NAIVE_QUEUE", queue)
            r = eng.naive_pr(d, dfm.PrOptions(policy=pol))
            assert r.stats.iterations == ref.iterations, (name, name_, dirty, queue)
            assert (r.partition.block == ref.block).all(), (name, name_, dirty, queue)
    rt = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
    ref_t = O.trans_pr(delta, acc, "min")
    assert rt.stats.iterations == ref_t.iterations and (rt.partition.block == ref_t.block).all()


@pytest.mark.parametrize("name,pair", [
    ("vlts_k12", lambda: O.vlts_dfa(300, 60_000, 12)),
    ("vlts_k20", lambda: O.vlts_dfa(200, 40_000, 20)),
    ("random_k9", lambda: O.random_dfa(20_000, 9, 77, 0.5)),
    ("random_k33", lambda: O.random_dfa(5_000, 33, 5, 0.5)),
])
def test_naive_lane_groups(eng, monkeypatch, name, pair):
    """4 or 8 lanes per state (fused_group_kernel, forced with DFM_NAIVE_GROUP=2 on
    inputs the thread-per-state kernel would take): the reference's partition and pass
    count under min / max, with and without the work-efficient marks; transPR too."""
    delta, acc = pair()
    d = to_dfa((delta, acc))
    monkeypatch.setenv("DFM_NAIVE_GROUP", "2")
    for pol, name_ in ((MIN, "min"), (MAX, "max")):
        ref = O.naive_pr(delta, acc, name_)
        for flag in ("1", "0"):
            monkeypatch.setenv("DFM_NAIVE_DIRTY", flag)
            r = eng.naive_pr(d, dfm.PrOptions(policy=pol))
            assert r.stats.iterations == ref.iterations, (name, name_, flag)
            assert (r.partition.block == ref.block).all(), (name, name_, flag)
    rt = eng.trans_pr(d, dfm.PrOptions(policy=MIN))
    ref_t = O.trans_pr(delta, acc, "min")
    assert rt.stats.iterations == ref_t.iterations and (rt.partition.block == ref_t.block).all()
