"""Summarise an .ncu-rep: key metrics (+ optional SASS opcode mix).
usage: python tools/ncu_summary.py REP [--sass] [--json OUT KEY ALG_BYTES]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__inst_executed.sum.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "sass__inst_executed_local_loads", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "sm__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {h[i]: (v[i], u[i]) for i in range(len(h))}
        res.append(d)
    return res


def main():
    rep = sys.argv[1]
    for d in raw(rep):
        print("kernel:", d.get("Kernel Name", ("?",))[0][:120])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][0]:>16} {d[k][1]}")
        if "--json" in sys.argv:
            i = sys.argv.index("--json")
            out, key, alg = sys.argv[i + 1], sys.argv[i + 2], float(sys.argv[i + 3])
            t_us = float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1)
            def mb(k):
                v, unit = d[k]
                f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]
                return float(v) * f
            try:
                js = json.load(open(out))
            except Exception:
                js = {}
            js[key] = {"kernel": d["Kernel Name"][0][:200], "ncu_duration_us": t_us,
                       "dram_bytes_per_launch": (mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")) * 1e6,
                       "dram_read_MB": mb("dram__bytes_read.sum"), "dram_write_MB": mb("dram__bytes_write.sum"),
                       "algorithmic_bytes": alg,
                       "ipc_per_sm": float(d["sm__inst_executed.sum.per_cycle_active"][0]) / 148,
                       "note": "ncu --set full --clock-control none; cold-cache single replayed launch"}
            json.dump(js, open(out, "w"), indent=1)
    if "--sass" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        open("/tmp/_sass.csv", "w").write(out)
        subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "sass_mix.py"), "/tmp/_sass.csv"])


if __name__ == "__main__":
    main()
