"""gpurun_out/traffic/*.csv (tools/traffic_all.sh) -> profiles/<round>/traffic_steady.json"""
import csv, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_11353_b200.configs import CONFIGS
rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
K = 16
LAUNCHES = {"config2_pease_nc": 1, "config2_dit": 1, "config3_dif": 2, "config4_pease_nc": 2, "config5_sixstep": 4}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
out = {"_method": "ncu --replay-mode app-range over 16 back-to-back steps (tools/traffic_all.sh, tools/traffic_range.py, "
                  "rotating buffer sets > L2), divided by 16: steady-state DRAM bytes and time per step.  A single-launch "
                  "capture under-reads the writes still in L2 when the launch ends and times a cold launch.  "
                  "range_time_us_per_step is the whole range / 16 and so includes the eager Python launch gaps "
                  "(~8 us per launch): it matches the bench's graph replays for the millisecond steps (configs 4, 5), "
                  "not for config 2, whose 32 us steps bench.py times as CUDA-graph replays."}
for name, nl in LAUNCHES.items():
    p = f"gpurun_out/traffic/{name}.csv"
    if not os.path.exists(p):
        continue
    rows = [r for r in csv.reader(open(p)) if len(r) > 8]
    h = rows[0]
    im, iu, iv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    m = {}
    for r in rows[1:]:
        m[r[im]] = m.get(r[im], 0.0) + float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
    cfg = int(name[6])
    alg = CONFIGS[cfg].algorithmic_bytes()
    rd, wr = m.get("dram__bytes_read.sum", 0) / K, m.get("dram__bytes_write.sum", 0) / K
    out[name] = {"dram_bytes_per_step": rd + wr, "read": rd, "write": wr, "algorithmic": alg,
                 "ratio": round((rd + wr) / alg, 3), "launches_per_step": nl,
                 "range_time_us_per_step": round(m.get("gpu__time_duration.sum", 0) / K * 1e6, 2)}
os.makedirs(f"profiles/{rnd}", exist_ok=True)
json.dump(out, open(f"profiles/{rnd}/traffic_steady.json", "w"), indent=1)
print(json.dumps(out, indent=1))
