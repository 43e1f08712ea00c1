"""Static SASS opcode histogram + FMA/ALU pipe-cycle estimate for kernels whose
mangled name matches a regex (straight-line kernels: static ~ per-warp dynamic).
usage: python tools/sass_static.py OBJ_OR_SO REGEX
Pipe costs per warp instruction measured by tools/ubench_pipes.cu on B200:
IMAD/IMAD.IADD/IMAD.MOV 2, IMAD.HI/IMAD.WIDE 4 (fma pipe); IADD3/LOP3/
VIADDMNMX/SHF/... 2 (alu pipe); issue 1 per instruction."""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
FMA = {"IMAD": 2, "IMAD.IADD": 2, "IMAD.MOV": 2, "IMAD.MOV.U32": 2, "IMAD.U32": 2, "IMAD.SHL": 2, "IMAD.SHL.U32": 2,
       "IMAD.HI.U32": 4, "IMAD.HI": 4, "IMAD.WIDE.U32": 4, "IMAD.WIDE": 4, "IMAD.X": 2}
ALU = ("IADD3", "LOP3", "VIADDMNMX", "VIMNMX", "SHF", "LEA", "ISETP", "SEL", "PRMT", "VIADD", "MOV", "IABS", "BREV")
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(pat, name):
        continue
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops[m.group(2)] += 1
    tot = sum(ops.values())
    fma = sum(n * FMA.get(op, 0) for op, n in ops.items())
    alu = sum(2 * n for op, n in ops.items() if op.split(".")[0] in ALU)
    print(f"== {dem[:120]}\n   {tot} instr, fma-pipe {fma} cyc, alu-pipe {alu} cyc")
    print("   " + ", ".join(f"{op} {n}" for op, n in ops.most_common(18)))
