"""Register-operand tally of the FP64 instructions of one kernel (development aid): how many
DFMA/DMUL/DADD read 1, 2 or 3 distinct registers without a `.reuse` hit, per MUFU.RSQ64H
(= per kernel evaluation), and the cycle estimate from profiles/r02b_micro_operand.md.

    python tools/sass_operands.py <lib.so> <kernel substring> [first_line last_line]
"""
import collections
import re
import subprocess
import sys

lib, key = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
blocks = out.split("Function : ")
body = next(b for b in blocks if key in b.split("\n", 1)[0])
L = [re.sub(r"/\* 0x[0-9a-f]+ \*/", "", m.group(1)).strip()
     for m in re.finditer(r"^\s+/\*[0-9a-f]{4,5}\*/\s+(.*)$", body, re.M)]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, len(L))
c = collections.Counter()
prev = {}
for l in L[lo:hi]:
    l = re.sub(r"^@!?U?P\d+\s+", "", l)
    op = l.split()[0].split(".")[0] if l else ""
    if op in ("DFMA", "DMUL", "DADD"):
        ops = [o.strip() for o in l.split(None, 1)[1].rstrip(" ;").split(",")[1:]]
        fresh = set()
        for slot, o in enumerate(ops):
            m = re.match(r"^-?\|?(R\d+)", o)
            if m and prev.get(slot) != m.group(1):
                fresh.add(m.group(1))
        prev = {slot: re.match(r"^-?\|?(R\d+)", o).group(1) for slot, o in enumerate(ops)
                if ".reuse" in o and re.match(r"^-?\|?(R\d+)", o)}
        c[len(fresh)] += 1
    elif op == "MUFU":
        c["mufu"] += 1
    elif op:
        c["other"] += 1
        if op not in ("IMAD", "MOV", "LDS", "NOP"):
            prev = {}
ev = max(c["mufu"], 1)
cost = {0: 2.04, 1: 2.08, 2: 2.2, 3: 3.02}
cyc = sum(cost[k] * v for k, v in c.items() if isinstance(k, int)) / ev
print(f"{key} [{lo}:{hi}] evaluations {ev}: per evaluation " +
      " ".join(f"{k}-reg {c[k] / ev:.2f}" for k in (0, 1, 2, 3)) +
      f" other {c['other'] / ev:.2f} -> ~{cyc:.1f} FP64-pipe cycles per warp evaluation")
