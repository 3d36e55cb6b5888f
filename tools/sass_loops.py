"""List the loops (backward branches) of a cuobjdump -sass listing with their
instruction mix: python tools/sass_loops.py file.sass"""
import re
import sys
from collections import Counter

lines = [l for l in open(sys.argv[1]) if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for addr, txt in ins:
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < addr:
        lo = int(m.group(1), 16)
        body = [t for a, t in ins if lo <= a <= addr]
        ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
        ff = ops["FFMA"]
        print(f"loop {lo:#x}-{addr:#x}: {len(body)} instr, FFMA {ff} ({100 * ff / len(body):.0f}%), "
              + ", ".join(f"{k} {v}" for k, v in ops.most_common(6)))
