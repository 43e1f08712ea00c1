"""Split a kernel's SASS (tools/prof_one.sh export) at barriers and report,
per region, executed warp instructions, the MIO-op mix and the PC-sampled
stall reasons.  usage: python tools/sass_regions.py NAME [launch_index]"""
import collections, csv, gzip, io, sys
name = sys.argv[1]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
srows = list(csv.reader(io.TextIOWrapper(gzip.open(f"gpurun_out/p1/{name}_sass.csv.gz"), encoding="utf-8")))
his = [i for i, r in enumerate(srows) if r and r[0] == "Address"]
hi = his[which]
hdr = srows[hi]; ix = {x: i for i, x in enumerate(hdr)}
end = his[which + 1] - 1 if which + 1 < len(his) else len(srows)
SK = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
regions = []
cur = None
def newreg(start):
    return {"start": start, "n": 0, "ops": collections.Counter(), "st": collections.Counter(), "len": 0}
cur = newreg(0)
for li, r in enumerate(srows[hi + 1:end]):
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    n = int(float(r[ix["Instructions Executed"]] or 0))
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    cur["n"] += n; cur["len"] += 1
    cur["ops"][op.split(".")[0]] += n
    for k in SK:
        cur["st"][k[6:]] += int(r[ix[k]] or 0)
    if op.startswith("BAR") or op.startswith("EXIT"):
        regions.append(cur); cur = newreg(li + 1)
regions.append(cur)
tot_n = sum(g["n"] for g in regions) or 1
tot_s = sum(sum(g["st"].values()) for g in regions) or 1
for g in regions:
    s = sum(g["st"].values())
    if g["n"] * 100 < tot_n and s * 100 < tot_s:
        continue
    mio = sum(g["ops"][o] for o in ("LDS", "STS", "LDGSTS", "LDG", "STG", "LDSM", "SHFL"))
    print(f"[{g['start']:5d} +{g['len']:4d}] instr {100*g['n']/tot_n:5.1f}%  samples {100*s/tot_s:5.1f}%  mio-ops {100*mio/max(g['n'],1):4.1f}%  "
          + " ".join(f"{k}:{100*v/max(s,1):.0f}" for k, v in g["st"].most_common(5)))
    print("        ops: " + ", ".join(f"{o} {v//max(1,min(x for x in g['ops'].values() if x>0))}" for o, v in g["ops"].most_common(8)))
