"""Static SASS opcode histogram of one kernel in an object file.
usage: python tools/sass_hist.py OBJ NAME_SUBSTRING [--dump]"""
import collections, re, subprocess, sys
obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = collections.Counter()
    lines = []
    for l in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
        if m:
            op = m.group(3)
            ops[op.split(".")[0]] += 1
            lines.append(l.strip())
    tot = sum(ops.values())
    print(name, "total", tot)
    print("  ".join(f"{k}:{v}" for k, v in ops.most_common(40)))
    if "--dump" in sys.argv:
        print("\n".join(lines))
