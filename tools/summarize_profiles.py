"""Turn gpurun_out/prof/*_raw.csv + launches.csv into profiles/<round>/ summaries
and profiles/ncu_summary.json (read by bench.py for roofline.traffic)."""
import csv
import gzip
import io
import json
import os
import sys
import collections

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
RND = sys.argv[2] if len(sys.argv) > 2 else "r1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", RND)
os.makedirs(OUT, exist_ok=True)
sys.path.insert(0, ROOT)
from paper_2405_11353_b200.configs import CONFIGS  # noqa: E402

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__inst_executed.sum", "sm__inst_executed.sum.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "nsecond": 1e-9}
CASES = {"c2_pease_nc": (2, "config2_pease_nc", 1), "c2_dit": (2, "config2_dit", 1), "c3_dif": (3, "config3_dif", 2),
         "c4_pease_nc": (4, "config4_pease_nc", 2), "c5_sixstep": (5, "config5_sixstep", 4)}


def load_raw(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    return [{h[i]: (v[i], u[i]) for i in range(len(h))} for v in rows[2:]]


def num(d, k):
    v, unit = d[k]
    return float(v.replace(",", "")) * UNIT.get(unit, 1.0)


summary = {}
md = [f"# ncu summaries ({RND})", "",
      "Captured by `tools/profile_round.sh` under gpurun on one B200 (`ncu --set full --clock-control none`, "
      "cold-cache replays of one launch; compare SHARES and counters, not absolute times).", ""]
for case, (cfg, key, npass) in CASES.items():
    p = os.path.join(SRC, f"{case}_raw.csv")
    if not os.path.exists(p):
        continue
    ks = load_raw(p)
    w = CONFIGS[cfg]
    alg = w.algorithmic_bytes()
    tot_t = sum(num(d, "gpu__time_duration.sum") for d in ks)
    tot_dram = sum(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum") for d in ks)
    summary[key] = {"kernels": [d["Kernel Name"][0][:160] for d in ks], "launches_per_step": len(ks),
                    "ncu_time_s_per_step": tot_t, "dram_bytes_per_launch": tot_dram / len(ks),
                    "dram_bytes_per_step": tot_dram, "algorithmic_bytes_per_step": alg,
                    "traffic_over_algorithmic": tot_dram / alg}
    if len(ks) < npass:     # only the first launches of the step captured (-c in profile_round.sh)
        line = (f"- captured {len(ks)} of the {npass} launches per step (the column passes); ncu time of those "
                f"{tot_t*1e6:.1f} us, DRAM {tot_dram/1e6:.1f} MB (whole-step traffic: profiles/r1/traffic_steady.json)")
    else:
        line = (f"- launches per step: {len(ks)}; ncu time per step {tot_t*1e6:.1f} us; DRAM bytes per step "
                f"{tot_dram/1e6:.1f} MB vs algorithmic {alg/1e6:.1f} MB (ratio {tot_dram/alg:.2f})")
    md += [f"## {key}: {w.batch} x 2^{w.log2n}, p={w.p}", "", line, ""]
    md.append("| metric | " + " | ".join(f"launch {i}" for i in range(len(ks))) + " |")
    md.append("|---|" + "---|" * len(ks))
    for k in KEYS:
        if k in ks[0]:
            md.append(f"| {k} | " + " | ".join(f"{d[k][0]} {d[k][1]}" for d in ks) + " |")
    md.append("")
    sp = os.path.join(SRC, f"{case}_sass.csv.gz")
    if os.path.exists(sp):
        rows = list(csv.reader(io.TextIOWrapper(gzip.open(sp), encoding="utf-8")))
        his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
        ops = collections.Counter()
        tot = 0
        for si, hi in enumerate(his):
            hdr = rows[hi]
            ix = {h: i for i, h in enumerate(hdr)}
            end = his[si + 1] - 1 if si + 1 < len(his) else len(rows)
            for r in rows[hi + 1:end]:
                if len(r) != len(hdr):
                    continue
                src = r[ix["Source"]].strip()
                n = int(float(r[ix["Instructions Executed"]] or 0))
                op = src.split()[0] if src else "?"
                if op.startswith("@"):
                    op = src.split()[1]
                ops[op.split(".")[0]] += n
                tot += n
        if tot:
            md.append("SASS opcode mix (executed warp instructions): " +
                      ", ".join(f"{o} {100*n/tot:.1f}%" for o, n in ops.most_common(12)))
            md.append("")
lp = os.path.join(SRC, "launches.csv")
if os.path.exists(lp):
    rows = [r for r in csv.reader(open(lp)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    kern = collections.Counter()
    ktime = collections.Counter()
    for r in rows[1:]:
        if len(r) != len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]][:90]
        kern[name] += 1
        ktime[name] += float(r[ix["Metric Value"]].replace(",", ""))
    tot = sum(ktime.values())
    md += ["## bench.py launch list (`ncu --metrics gpu__time_duration.sum`, serialised, cold)", "",
           "| kernel | launches | total time | share |", "|---|---|---|---|"]
    for k, n in kern.most_common():
        md.append(f"| `{k}` | {n} | {ktime[k]:.0f} | {100*ktime[k]/tot:.1f}% |")
    md.append("")
    import shutil
    shutil.copy(lp, os.path.join(OUT, "bench_launches.csv"))
open(os.path.join(OUT, "summary.md"), "w").write("\n".join(md))
json.dump(summary, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
for f in os.listdir(SRC):
    if f.endswith("_raw.csv"):
        import shutil
        shutil.copy(os.path.join(SRC, f), os.path.join(OUT, f))
print("\n".join(md[:60]))
