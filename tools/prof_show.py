"""Show metrics, stall reasons, opcode mix, top stalled SASS per launch of a
profile exported by tools/prof_one.sh.  usage: python tools/prof_show.py NAME"""
import collections, csv, gzip, io, sys
name = sys.argv[1]
base = f"gpurun_out/p1/{name}"
rows = list(csv.reader(open(base + "_raw.csv")))
h, u = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
        "sm__inst_executed.sum.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum"]
for li, v in enumerate(rows[2:]):
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    print(f"== launch {li}: {d['Kernel Name'][0][:100]}")
    for k in KEYS:
        if k in d:
            print(f"   {k:66s} {d[k][0]:>14} {d[k][1]}")
    st = [(h[i], float(v[i] or 0)) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    print("   stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*x/tot:.0f}%" for k, x in sorted(st, key=lambda t: -t[1])[:7]))
srows = list(csv.reader(io.TextIOWrapper(gzip.open(base + "_sass.csv.gz"), encoding="utf-8")))
his = [i for i, r in enumerate(srows) if r and r[0] == "Address"]
for si, hi in enumerate(his):
    hdr = srows[hi]; ix = {x: i for i, x in enumerate(hdr)}
    end = his[si + 1] - 1 if si + 1 < len(his) else len(srows)
    ops = collections.Counter(); tot = 0; stl = []
    for r in srows[hi + 1:end]:
        if len(r) != len(hdr):
            continue
        src = r[ix["Source"]].strip(); n = int(float(r[ix["Instructions Executed"]] or 0))
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        ops[op.split(".")[0]] += n; tot += n
        stl.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), n, src[:72]))
    print(f"== sass {si}: total {tot}: " + ", ".join(f"{o} {100*n/tot:.1f}" for o, n in ops.most_common(12)))
    for x in sorted(stl, reverse=True)[:8]:
        print("     ", x)
