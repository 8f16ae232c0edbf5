"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total ms, launches and share (optionally only the last N launches)."""
import csv
import re
import sys


def main(path, last=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = []
    for r in rows:
        name = re.sub(r"^void ", "", r[ki])
        name = re.split(r"[(<]", name.replace("<unnamed>::", ""))[0]
        seq.append((name, float(r[vi].replace(",", "")) / 1e6))
    if last:
        seq = seq[-int(last):]
    agg = {}
    for k, v in seq:
        a = agg.setdefault(k, [0.0, 0])
        a[0] += v
        a[1] += 1
    tot = sum(v for v, _ in agg.values())
    print(f"{len(seq)} launches, {tot:.3f} ms")
    for k, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} {c:5d} {v:10.3f} ms {100 * v / tot:6.2f} %")


if __name__ == "__main__":
    main(*sys.argv[1:])
