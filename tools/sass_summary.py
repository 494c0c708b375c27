"""Instruction-class census of the built library's SASS per kernel
(cuobjdump -sass): the tcgen05 MMAs (UTCHMMA / UTCHMMA.2CTA), TMEM loads /
stores (LDTM / STTM), bulk copies and reductions (UBLKCP / UBLKRED), MUFU
ops, and the conversions.  usage: python tools/sass_summary.py > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2310_20285_b200/libncgp_b200.so"
CLASSES = ["UTCHMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UBLKCP", "UBLKRED", "UTMALDG",
           "SYNCS", "MUFU.EX2", "MUFU.SQRT", "MUFU.RSQ", "F2I", "F2FP", "HMMA", "DMMA", "FFMA",
           "DFMA", "RED", "ATOM"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m:
        op = m.group(1)
        for c in CLASSES:
            if op == c or op.startswith(c + "."):
                per[cur][c] += 1
                break
tot = collections.Counter()
print(f"# SASS instruction classes per kernel of {LIB} (cuobjdump -sass, sm_100a)")
print("# kernel | " + " ".join(CLASSES))
for k, cnt in per.items():
    if not any(cnt.values()):
        continue
    tot.update(cnt)
    short = re.sub(r"_ZN\d+_GLOBAL__N__\w+?\d+(\w+?)E", r"\1", k)[:90]
    print(short, {c: cnt[c] for c in CLASSES if cnt[c]})
print("# total", {c: tot[c] for c in CLASSES if tot[c]})
