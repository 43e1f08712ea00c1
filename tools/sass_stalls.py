"""Per-kernel stall breakdown from an `ncu --page source --csv --print-source sass`
dump: samples by stall reason, grouped by the opcode class of the stalled
instruction.  usage: python tools/sass_stalls.py FILE.csv[.gz] [TOP]"""
import collections, csv, gzip, io, sys
fn = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = gzip.open(fn, "rt").read() if fn.endswith(".gz") else open(fn).read()
sections = raw.split('"Kernel Name",')
for sec in sections[1:]:
    lines = sec.splitlines()
    name = lines[0].strip().strip('",')[:100]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    byop = collections.defaultdict(collections.Counter)
    ninstr = 0
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ninstr += int(float(r[ix["Instructions Executed"]] or 0))
        for h in reasons:
            v = int(float(r[ix[h]] or 0))
            tot[h] += v
            byop[op][h] += v
    S = sum(tot.values()) or 1
    print(f"== {name}  warp-instr {ninstr}  samples {S}")
    print("   " + "  ".join(f"{h[6:]}={100*v/S:.1f}%" for h, v in tot.most_common(8)))
    ops = sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:top]
    for op, c in ops:
        s = sum(c.values())
        print(f"   {op:10s} {100*s/S:5.1f}%  " + " ".join(f"{h[6:]}={100*v/S:.1f}" for h, v in c.most_common(4)))
