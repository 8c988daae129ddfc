"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel of this repo,
launch count, mean duration and share of the summed duration."""
import csv
import sys
from collections import defaultdict

OURS = ("az_", "gemm_dmma_kernel", "sglk::")


def main(path, header=""):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("void ", "").split("(")[0].replace("sglk::", "")
        if not any(o in r[ki] for o in OURS):
            continue
        v = float(r[vi].replace(",", ""))
        unit = h[vi + 1] if False else None
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    if header:
        print(header)
    print(f"{'kernel':58s} {'launches':>8s} {'mean us':>9s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:58s} {cnt[k]:8d} {tot[k] / cnt[k] / 1000:9.1f} {100 * tot[k] / s:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
