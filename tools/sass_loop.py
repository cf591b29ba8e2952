"""Opcode histogram of the hottest loop of a kernel in a built library:
the backward branch whose body holds the most shared atomics, normalised to
one 48-atomic (512-pixel) step.  python tools/sass_loop.py LIB [kernel-substr]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "walk_kernelILb1ELb1ELb0E"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if f.startswith("_Z") and kname in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, t in ins:
    m = re.search(r"BRA.*0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a:
            loop = [x for x in ins if tgt <= x[0] <= a]
            na = sum("ATOMS" in x[1] for x in loop)
            if na >= 48 and (best is None or len(loop) < len(best)):
                best = loop
c = collections.Counter()
for _, t in best:
    t2 = re.sub(r"^@!?U?P\w+\s+", "", t)
    c[t2.split()[0]] += 1
na = sum(v for k, v in c.items() if k.startswith("ATOMS"))
scale = 48.0 / na
print(f"loop: {len(best)} instructions, {na} shared atomics -> {len(best) * scale:.1f} per 48-atomic step")
for k, v in c.most_common():
    print(f"  {v * scale:6.1f} {k}")
