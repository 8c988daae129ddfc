"""Top SASS lines by stall samples from `ncu --page source --csv --print-source=sass`."""
import csv
import sys


def main(path, kernel_filter="", top=25):
    lines = open(path).read().splitlines()
    blocks, cur = [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    for b in blocks:
        name = b[0]
        if kernel_filter not in name:
            continue
        rows = list(csv.reader(b[1:]))
        h = rows[0]
        si = h.index("Warp Stall Sampling (All Samples)")
        src = h.index("Source")
        data = []
        tot = 0
        for r in rows[1:]:
            try:
                v = int(r[si])
            except (ValueError, IndexError):
                continue
            tot += v
            data.append((v, r[src].strip(), r[0]))
        print(name[:100], "total samples", tot)
        for v, s, a in sorted(data, reverse=True)[:top]:
            print(f"  {v:6d} {100.0 * v / max(tot, 1):5.1f}%  {a[-5:]}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 25)
