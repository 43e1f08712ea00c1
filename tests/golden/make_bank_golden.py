"""Generate tests/golden/bankmodel_vectors.json by running the REFERENCE
bankmodel (nttkit/bankmodel.py) in this container.  The fixture pins
paper_2405_11353_b200.bankmodel (tests/test_bankmodel_api.py); the GPU box
never needs /root/reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_bank_golden.py
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from nttkit import bankmodel as R  # noqa: E402


def sched_cases():
    for algo in R.TRACE_VARIANTS:
        for log_n in (1, 2, 3, 4, 5, 6):
            for kind, par in (("interleave", 1), ("interleave", 2), ("interleave", 4), ("interleave", 8),
                              ("blocksize", 2), ("blocksize", 4)):
                for ports in (1, 2):
                    for unroll in (1, 2, 4):
                        for rw, depth in ((True, 1), (True, 2), (False, 1)):
                            for tii in (1, 2):
                                yield dict(algo=algo, log_n=log_n, kind=kind, param=par, ports=ports,
                                           unroll=unroll, rw_overlap=rw, depth=depth, target_ii=tii)


def conflicts_digest(conflicts):
    # sha256 of the conflict tuples' JSON (the full lists would make the fixture megabytes)
    return hashlib.sha256(json.dumps([list(x) for x in conflicts]).encode()).hexdigest()[:16]


def mk_map(kind, par):
    return R.interleave(par) if kind == "interleave" else R.blocksize(par)


def main():
    out = {"schedule": [], "partition": [], "graph": [], "partners": [], "pease_nc": []}
    for c in sched_cases():
        tr = R.gen_trace(c["algo"], c["log_n"])
        cfg = R.BankConfig(mk_map(c["kind"], c["param"]), ports=c["ports"], unroll=c["unroll"],
                           rw_overlap=c["rw_overlap"], depth=c["depth"])
        r = R.schedule(tr, cfg, target_ii=c["target_ii"])
        out["schedule"].append(dict(c, achieved_ii=r.achieved_ii, feasible=r.feasible,
                                    n_conflicts=len(r.conflicts), conflicts_sha=conflicts_digest(r.conflicts)))
    for algo in R.TRACE_VARIANTS:
        for log_n in (1, 2, 3, 4):
            for banks in (1, 2, 3, 4, 6, 8):
                for ports in (1, 2):
                    for unroll in (1, 2, 4):
                        tr = R.gen_trace(algo, log_n)
                        try:
                            p = R.feasible_partition(tr, banks, ports=ports, unroll=unroll, node_budget=200_000)
                            res = None if p is None else {
                                k: [m.kind, m.param, list(m.table) if m.table is not None else None]
                                for k, m in sorted(p.items())}
                            err = None
                        except R.SearchBudgetExceeded:
                            res, err = None, "budget"
                        out["partition"].append(dict(algo=algo, log_n=log_n, banks=banks, ports=ports,
                                                     unroll=unroll, result=res, error=err))
    for algo in R.TRACE_VARIANTS:
        for log_n in (1, 2, 3, 4):
            for unroll in (1, 2, 4):
                g = R.conflict_graph(R.gen_trace(algo, log_n), unroll=unroll)
                out["graph"].append(dict(algo=algo, log_n=log_n, unroll=unroll,
                                         groups={k: sorted(sorted(x) for x in v) for k, v in sorted(g.items())}))
                for addr in range(1 << log_n):
                    sp = R.separation_partners(R.gen_trace(algo, log_n), addr, "x", ports=2, unroll=unroll)
                    out["partners"].append(dict(algo=algo, log_n=log_n, unroll=unroll, addr=addr,
                                                partners=sorted(sp)))
    for log_n in range(1, 11):
        for units in (1, 2, 4, 8, 16, 32):
            if units > 1 << (log_n - 1):
                continue
            for ports in (1, 2):
                r = R.pease_nc_partition_check(log_n, units, ports)
                out["pease_nc"].append(dict(log_n=log_n, units=units, ports=ports, achieved_ii=r.achieved_ii,
                                            swap_safe=r.swap_safe, csv=R.report_csv_row(r),
                                            text_sha=hashlib.sha256(R.report_text(r).encode()).hexdigest()[:16],
                                            text_head=R.report_text(r).split("\n")[:3]))
    keys = ["algo", "log_n", "kind", "param", "ports", "unroll", "rw_overlap", "depth", "target_ii",
            "achieved_ii", "feasible", "n_conflicts", "conflicts_sha"]
    out["schedule_keys"] = keys
    out["schedule"] = [[row[k] for k in keys] for row in out["schedule"]]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bankmodel_vectors.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(path, {k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
