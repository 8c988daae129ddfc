"""Summarise an `ncu --page source --csv --print-source sass` export of ONE kernel
(read here, not on the box): stall samples per code region and per opcode.

Instructions with the same execution count belong to the same region of the
kernel (prologue / per-chunk issue / MMA body / barrier / epilogue), so grouping
by execution count shows where the warps spend their samples.
usage: python tools/sass_stalls.py export.csv [top]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    seen, data = set(), []
    for r in rows[2:]:
        if len(r) == len(h) and r[0].startswith("0x") and r[0] not in seen:  # the export repeats rows
            seen.add(r[0])
            data.append(r)
    return h, data


def opcode(src):
    t = src.strip().split()
    if not t:
        return "?"
    return (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]


def main(path, top=10):
    h, data = load(path)
    ix = {k: i for i, k in enumerate(h)}
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot_s = tot_i = 0
    smp, ninstr = collections.Counter(), collections.Counter()
    rs, ops = collections.defaultdict(collections.Counter), collections.defaultdict(collections.Counter)
    for r in data:
        e = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        tot_s += s
        tot_i += e
        smp[e] += s
        ninstr[e] += 1
        ops[e][opcode(r[ix["Source"]])] += 1
        for k in reasons:
            rs[e][k[6:]] += int(r[ix[k]] or 0)
    print(f"warp instructions executed {tot_i}, stall samples {tot_s}")
    print("regions (instructions sharing an execution count), by share of samples:")
    for e, s in smp.most_common(top):
        print(f"  exec={e:9d} x {ninstr[e]:4d} instr  samples={s / max(tot_s, 1):.3f}  instr={e * ninstr[e] / max(tot_i, 1):.3f}  "
              f"{dict(rs[e].most_common(3))}  {dict(ops[e].most_common(5))}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 10)
