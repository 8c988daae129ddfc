"""Summarise an `ncu --page source --csv --print-source sass` export: stall samples
per opcode and per reason, and the hottest instructions (read here, not on the box)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
by_op = collections.Counter()
by_reason = collections.Counter()
by_op_reason = collections.defaultdict(collections.Counter)
execd = collections.Counter()
for r in data:
    op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].strip().split()[1]
    op = op.split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    by_op[op] += s
    execd[op] += int(r[ix["Instructions Executed"]] or 0)
    for k in reasons:
        v = int(r[ix[k]] or 0)
        by_reason[k] += v
        by_op_reason[op][k] += v
print(f"total samples {tot}")
print("by reason:", ", ".join(f"{k[6:]}={v / tot:.3f}" for k, v in by_reason.most_common(10)))
print("by opcode (share of samples, warp-level instructions executed, top reasons):")
for op, v in by_op.most_common(14):
    top = ", ".join(f"{k[6:]}={c / tot:.3f}" for k, c in by_op_reason[op].most_common(3))
    print(f"  {op:10s} {v / tot:6.3f}  exec={execd[op]:>10d}  {top}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("hottest instructions:")
hot = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in hot:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:2]
    print(f"  {r[ix['Address']][-5:]} {s / tot:6.3f} {r[ix['Source']].strip()[:60]:60s} {top}")
