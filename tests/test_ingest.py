"""LTS ingestion: libdfm's parse_lts / determinize / complete against
the reference's own (ingest.hpp:130-284, oracle/_ref) — the known answers of
test_ingest.cpp, seeded random transition systems (quoting, whitespace, CRLF,
blank lines, duplicates), errors (line and message), the subset budget, large
inputs that the parser splits over several threads, and the pipeline into the
minimizer.  Host code only: no GPU needed."""
import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def ours(text, budget=1 << 22):
    try:
        lts = dfm.parse_lts(text)
    except dfm.ParseError as e:
        return {"status": "parse", "line": e.line(), "what": str(e)}
    try:
        p = dfm.determinize(lts, budget)
    except dfm.SubsetBudgetExceeded as e:
        return {"status": "budget", "line": e.budget(), "what": str(e)}
    d = dfm.complete(p)
    return {"status": "ok", "lts": lts, "pdfa": p, "dfa": d}


def same(text, budget=1 << 22):
    a, r = ours(text, budget), O.ref_ingest(text, budget)
    assert a["status"] == r["status"], (a, r)
    if r["status"] != "ok":
        assert (a["line"], a["what"]) == (r["line"], r["what"])
        return a
    n, init, labels, src, lab, dst = r["lts"]
    lts = a["lts"]
    assert (lts.num_states, lts.initial, lts.labels) == (n, init, labels)
    assert (lts.src == src).all() and (lts.label == lab).all() and (lts.dst == dst).all()
    assert (a["pdfa"].delta == r["pdfa"]).all()
    assert (a["dfa"].delta == r["dfa"][0]).all() and (a["dfa"].accepting == r["dfa"][1]).all()
    return a


def test_reference_known_answers():  # test_ingest.cpp:32-139
    lts = dfm.parse_lts('des (0, 1, 2)\n(0, "a", 1)\n')
    assert (lts.num_states, lts.initial, lts.labels, lts.transitions) == (2, 0, ["a"], [(0, 0, 1)])
    assert dfm.parse_lts('des (0, 2, 3)\n(0, tau, 1)\n(1, "send!x", 2)\n').labels == ["tau", "send!x"]
    dup = dfm.parse_lts('des (0, 3, 2)\n(0, "b", 1)\n(0, "a", 1)\n(0, "b", 1)\n')
    assert len(dup.transitions) == 3 and dup.labels == ["b", "a"]
    with pytest.raises(dfm.ParseError):
        dfm.parse_lts('des (0, 2, 2)\n(0, "a", 1)\n')
    with pytest.raises(dfm.ParseError) as e:
        dfm.parse_lts('des (0, 1, 2)\n(0, "a", 1)\n(1, "a", 0)\n')
    assert e.value.line() == 3
    with pytest.raises(dfm.ParseError) as e:
        dfm.parse_lts('des (0, 1, 2)\n(0, "a" 1)\n')
    assert e.value.line() == 2
    for bad in ('des (0, 1, 2)\n(0, "a", 5)\n', "des (9, 0, 2)\n", ""):
        with pytest.raises(dfm.ParseError):
            dfm.parse_lts(bad)
    det = dfm.parse_lts('des (0, 4, 2)\n(0, "a", 1)\n(1, "a", 0)\n(0, "b", 0)\n(1, "b", 1)\n')
    p = dfm.determinize(det)
    assert (p.num_states, p.alphabet_size) == (2, 2)
    assert p.delta[0].tolist() == [1, 0] and p.delta[1].tolist() == [0, 1]
    q = dfm.determinize(dfm.parse_lts('des (0, 2, 3)\n(0, "a", 1)\n(0, "a", 2)\n'))
    assert q.num_states == 2 and q.delta[0][0] == 1 and q.delta[0][1] == dfm.K_MISSING
    m = dfm.determinize(dfm.parse_lts(
        'des (0, 4, 3)\n(0, "a", 1)\n(0, "a", 2)\n(1, "b", 0)\n(2, "b", 2)\n'))
    M = dfm.K_MISSING
    assert m.num_states == 4
    assert m.delta[0].tolist() == [1, M, 1, M] and m.delta[1].tolist() == [M, 2, 3, 3]
    wide = dfm.parse_lts('des (0, 6, 4)\n(0, "a", 1)\n(0, "a", 2)\n(1, "a", 0)\n(1, "a", 3)\n'
                         '(2, "a", 3)\n(3, "a", 1)\n')
    with pytest.raises(dfm.SubsetBudgetExceeded):
        dfm.determinize(wide, 2)
    full = dfm.complete(dfm.determinize(det))
    assert full.num_states == 2 and full.accepting.tolist() == [1, 1]
    sink = dfm.complete(dfm.determinize(dfm.parse_lts('des (0, 1, 2)\n(1, "a", 1)\n')))
    assert sink.num_states == 2 and sink.accepting.tolist() == [1, 0]
    assert sink.delta[0].tolist() == [1, 1]


def random_lts_text(rng, n, m, nlab, style):
    labels = [f"l{i}" if i % 3 else f"act!{i}?x" for i in range(nlab)]
    lines = [f"des ({int(rng.integers(0, n))}, {m}, {n})"]
    for _ in range(m):
        s, d = int(rng.integers(0, n)), int(rng.integers(0, n))
        a = labels[int(min(nlab - 1, rng.exponential(nlab / 4)))]
        q = f'"{a}"' if (style & 1) or "!" in a else a
        sp = " " * int(rng.integers(0, 3)) if style & 2 else " "
        lines.append(f"({s},{sp}{q},{sp}{d})")
        if style & 4 and rng.random() < 0.05:
            lines.append("   \t")
    eol = "\r\n" if style & 8 else "\n"
    return eol.join(lines) + eol


def test_random_systems_match_reference():
    rng = np.random.default_rng(2410)
    for case in range(120):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(0, 120))
        nlab = int(rng.integers(1, 6))
        same(random_lts_text(rng, n, m, nlab, case % 16))


def test_errors_match_reference():
    base = 'des (0, 3, 4)\n(0, "a", 1)\n(1, b, 2)\n(2, "a", 3)\n'
    variants = [base, base.replace("(1, b, 2)", "(1, , 2)"), base.replace('"a", 3', '"a 3'),
                base.replace("(2,", "(7,"), base.replace("des (0, 3, 4)", "des (0, 3, 0)"),
                base.replace("des (0", "dse (0"), base + "(3, a, 0)\n", base + "junk\n",
                base.replace("(0, \"a\", 1)", "(0, \"a\", 1) x"), "\n\n  \n" + base,
                base.replace("(1, b, 2)", "(1, b, 99999999999)"), "des (0, 0, 1)\n", "  \n\t\n"]
    for v in variants:
        same(v)
    same(base, budget=2)


def det_lts_text(rng, n, nlab, extra):
    """A deterministic transition system (every (state, label) once, shuffled) plus
    `extra` repeated transitions (kept, as the format allows): the subset construction
    stays at the reachable singletons."""
    src = np.repeat(np.arange(n), nlab)
    lab = np.tile(np.arange(nlab), n)
    dst = rng.integers(0, n, size=n * nlab)
    pick = rng.integers(0, n * nlab, size=extra)
    src = np.concatenate([src, src[pick]])
    lab = np.concatenate([lab, lab[pick]])
    dst = np.concatenate([dst, dst[pick]])
    order = rng.permutation(src.size)
    body = "\n".join(f'({s}, "a{a}", {d})' for s, a, d in zip(src[order], lab[order], dst[order]))
    return f"des (0, {src.size}, {n})\n{body}\n"


def test_large_system_parallel_parse_matches_reference():
    """~6 MB of text: the parser cuts it into several chunks (threads); labels first
    seen in late chunks, an error in a late chunk, and a count mismatch."""
    rng = np.random.default_rng(7)
    text = det_lts_text(rng, 20_000, 15, 40)
    r = same(text)
    assert r["status"] == "ok" and r["lts"].src.size == 300_040
    lines = text.split("\n")
    bad = lines.copy()
    bad[250_000] = "(1, x 2)"
    same("\n".join(bad))
    same(text.replace("300040", "300039", 1))


def test_pipeline_into_the_minimizer_matches_reference_partition():
    rng = np.random.default_rng(11)
    text = random_lts_text(rng, 30, 90, 3, 0)
    d = dfm.complete(dfm.determinize(dfm.parse_lts(text)))
    r = O.ref_ingest(text)
    ref = O.sort_pr(*r["dfa"])
    assert d.num_states == r["dfa"][1].size
    assert O.sort_pr(d.delta, d.accepting).num_blocks == ref.num_blocks
