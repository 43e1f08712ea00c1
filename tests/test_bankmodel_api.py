"""bankmodel drop-in: paper_2405_11353_b200.bankmodel
against fixtures made by the reference itself (tests/golden/make_bank_golden.py)
plus the reference test-suite's properties (pkg/tests/test_bankmodel.py),
re-parametrised."""
import hashlib
import json
import os

import pytest

import paper_2405_11353_b200 as P
from paper_2405_11353_b200 import bankmodel as B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bankmodel_vectors.json")))


def _digest(conflicts):
    return hashlib.sha256(json.dumps([list(x) for x in conflicts]).encode()).hexdigest()[:16]


def _map(kind, par):
    return B.interleave(par) if kind == "interleave" else B.blocksize(par)


def test_schedule_matches_reference_vectors():
    keys = GOLD["schedule_keys"]
    bad = []
    for row in GOLD["schedule"]:
        c = dict(zip(keys, row))
        cfg = B.BankConfig(_map(c["kind"], c["param"]), ports=c["ports"], unroll=c["unroll"],
                           rw_overlap=c["rw_overlap"], depth=c["depth"])
        r = B.schedule(B.gen_trace(c["algo"], c["log_n"]), cfg, target_ii=c["target_ii"])
        got = (r.achieved_ii, r.feasible, len(r.conflicts), _digest(r.conflicts))
        if got != (c["achieved_ii"], c["feasible"], c["n_conflicts"], c["conflicts_sha"]):
            bad.append((c, got))
    assert not bad, bad[:3]
    assert len(GOLD["schedule"]) == 6480


def test_feasible_partition_matches_reference_vectors():
    for c in GOLD["partition"]:
        tr = B.gen_trace(c["algo"], c["log_n"])
        try:
            p = B.feasible_partition(tr, c["banks"], ports=c["ports"], unroll=c["unroll"], node_budget=200_000)
            got = None if p is None else {k: [m.kind, m.param, list(m.table) if m.table is not None else None]
                                          for k, m in sorted(p.items())}
            err = None
        except P.SearchBudgetExceeded:
            got, err = None, "budget"
        assert (got, err) == (c["result"], c["error"]), c


def test_conflict_graph_and_partners_match_reference_vectors():
    for c in GOLD["graph"]:
        g = B.conflict_graph(B.gen_trace(c["algo"], c["log_n"]), unroll=c["unroll"])
        assert {k: sorted(sorted(x) for x in v) for k, v in sorted(g.items())} == c["groups"], c
    for c in GOLD["partners"]:
        sp = B.separation_partners(B.gen_trace(c["algo"], c["log_n"]), c["addr"], "x", ports=2, unroll=c["unroll"])
        assert sorted(sp) == c["partners"], c


def test_pease_nc_partition_check_matches_reference_vectors():
    for c in GOLD["pease_nc"]:
        r = B.pease_nc_partition_check(c["log_n"], c["units"], c["ports"])
        t = B.report_text(r)
        assert (r.achieved_ii, r.swap_safe) == (c["achieved_ii"], c["swap_safe"]), c
        assert B.report_csv_row(r) == c["csv"]
        assert hashlib.sha256(t.encode()).hexdigest()[:16] == c["text_sha"]
        assert t.split("\n")[:3] == c["text_head"]


# -- properties of the reference suite, re-parametrised -----------------------

@pytest.mark.parametrize("log_n", [3, 5, 7])
def test_trace_shapes(log_n):
    n = 1 << log_n
    dit, dif, flat = (B.gen_trace(a, log_n) for a in ("dit", "dif", "flat"))
    assert [it.reads for it in dit.stages[0].iterations][:2] == [(0, 1), (2, 3)]
    assert [it.reads for it in dit.stages[-1].iterations][0] == (0, n // 2)
    assert dif.stages[0] == dit.stages[-1] and dif.stages[-1] == dit.stages[0]
    assert flat.stages == dit.stages and all(len(s.iterations) == n // 2 for s in flat.stages)
    pe, nc = B.gen_trace("pease", log_n), B.gen_trace("pease_nc", log_n)
    assert all((s.read_array, s.write_array) == ("x", "y") for s in pe.stages)
    assert [(s.read_array, s.write_array) for s in nc.stages] == [("x", "y"), ("y", "x")] * (log_n // 2) + \
        [("x", "y")] * (log_n % 2)
    for r, it in enumerate(pe.stages[0].iterations):
        assert it.reads == (2 * r, 2 * r + 1) and it.writes == (r, r + n // 2)
    assert dit.in_place and not nc.in_place


@pytest.mark.parametrize("algo", ["stockham", "sixstep", "naive"])
def test_untraced_variants(algo):
    with pytest.raises(P.UnsupportedVariant):
        B.gen_trace(algo, 4)


def test_mappings_and_validation():
    cfg = B.BankConfig(B.interleave(4))
    assert [B.bank_of(a, cfg) for a in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    m = B.blocksize(3)
    assert [m.bank_of(a) for a in range(7)] == [0, 0, 0, 1, 1, 1, 2] and m.n_banks(7) == 3
    e = B.explicit({0: 1, 1: 0, 2: 1})
    assert e.table == (1, 0, 1) and e.n_banks(3) == 2 and B.explicit([]).n_banks(0) == 1
    for bad in (lambda: B.interleave(0), lambda: B.blocksize(0), lambda: B.BankConfig(B.interleave(1), ports=0),
                lambda: B.BankConfig(B.interleave(1), depth=0),
                lambda: B.schedule(B.gen_trace("dit", 2), B.BankConfig(B.interleave(1)), target_ii=0),
                lambda: B.gen_trace("dit", 17), lambda: B.pease_nc_partition_check(4, 3),
                lambda: B.pease_nc_partition_check(3, 8),
                lambda: B.conflict_graph(B.gen_trace("dit", 9))):
        with pytest.raises(ValueError):
            bad()


def test_ii_monotone_and_budget():
    tr = B.gen_trace("dit", 4)
    for ports in (1, 2):
        last = None
        for m in (1, 2, 4, 8, 16):
            ii = B.schedule(tr, B.BankConfig(B.interleave(m), ports=ports, unroll=2)).achieved_ii
            assert last is None or ii <= last
            last = ii
    with pytest.raises(P.SearchBudgetExceeded):
        B.feasible_partition(B.gen_trace("dit", 3), 7, ports=2, unroll=4, node_budget=10)
    part = B.feasible_partition(B.gen_trace("pease", 4), 4, ports=2, unroll=4)
    assert part is not None
    assert B.schedule(B.gen_trace("pease", 4), B.BankConfig(part, ports=2, unroll=4)).conflicts == ()


def test_b200_warp_config():
    # 32 one-port banks, one butterfly per lane: pease_nc's {2r, 2r+1} reads of a
    # 32-lane step cover 64 consecutive words -> 2 per bank (II 2), as a warp sees it
    cfg = B.b200_smem_config()
    assert B.schedule(B.gen_trace("pease_nc", 10), cfg).achieved_ii >= 2
    assert B.schedule(B.gen_trace("pease_nc", 10), B.BankConfig(B.interleave(32), ports=1, unroll=16)).achieved_ii >= 1


def test_package_exports():
    for name in ("AccessTrace", "BankConfig", "BankMap", "ConflictReport", "bank_of", "blocksize", "conflict_graph",
                 "explicit", "feasible_partition", "gen_trace", "interleave", "pease_nc_partition_check", "schedule",
                 "separation_partners"):
        assert getattr(P, name) is getattr(B, name)


def test_cli_banks_matches_reference_output(capsys):
    from paper_2405_11353_b200 import cli
    assert cli.main(["banks", "--algo", "dit", "--log-n", "3", "--interleave", "1"]) == 0
    out = capsys.readouterr().out
    assert out.startswith("achieved II = 2 (target 1): infeasible at target")
    assert cli.main(["banks", "--algo", "pease_nc", "--log-n", "6", "--units", "4"]) == 0
    assert "swap-safe: yes" in capsys.readouterr().out
    assert cli.main(["banks", "--algo", "dit", "--log-n", "3", "--banks", "8", "--search", "--unroll", "4"]) == 0
    assert capsys.readouterr().out.strip().endswith("feasible: II=1")
    assert cli.main(["banks", "--algo", "dit", "--log-n", "3", "--units", "2"]) == 1
    assert cli.main(["banks", "--algo", "dit", "--log-n", "3", "--search"]) == 1
