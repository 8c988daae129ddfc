"""Per-kernel SASS opcode census of libsglb200.so (cuobjdump -sass): the
instructions that prove the B200 paths -- DMMA.8x8x4 (fp64 tensor core),
UTMALDG (TMA tensor loads), LDGSTS (cp.async), SYNCS (mbarrier), DFMA/DADD/DMUL
(FFT arithmetic), BAR -- per kernel.  usage: python tools/sass_census.py [lib] > profiles/rNN_sass_census.txt"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "paper_1604_05140_b200", "libsglb200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
demangled = {}
names = re.findall(r"Function : (\S+)", sass)
if names:
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    demangled = dict(zip(names, out))
KEYS = ["DMMA", "UTMALDG", "UTMASTG", "LDGSTS", "SYNCS", "DFMA", "DADD", "DMUL", "LDS", "STS", "LDG", "STG",
        "BAR", "RED", "ATOM", "CCTL"]
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = demangled.get(m.group(1), m.group(1))
        per[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Za-z0-9_.]+)?", line)
    if m and cur is not None:
        op = m.group(1)
        full = op + (m.group(2) or "")
        for k in KEYS:
            if op.startswith(k):
                per[cur][full if k in ("DMMA", "UTMALDG", "SYNCS") else k] += 1
print(f"# SASS opcode census of {os.path.relpath(lib, REPO)} (static instruction counts per kernel; sm_100a)")
for fn, c in per.items():
    short = fn.replace("sglk::", "").split("(")[0]
    if not c:
        continue
    body = ", ".join(f"{k} {v}" for k, v in sorted(c.items(), key=lambda kv: (-kv[1], kv[0])))
    print(f"{short}\n    {body}")
