"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by
source line: warp instructions executed, thread instructions, stall samples."""
import csv
import sys


def main(path, top=45):
    top = int(top)
    rows = list(csv.reader(open(path)))
    fname, agg, cur = "?", {}, None
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 10:
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:70])
            continue
        if cur is None or r[2] in ("...", "-"):
            continue
        try:
            smp = float(r[4]); ins = float(r[7]); thr = float(r[8])
        except ValueError:
            continue
        a = agg.setdefault(cur, [0.0, 0.0, 0.0])
        a[0] += ins; a[1] += thr; a[2] += smp
    tot = [sum(v[k] for v in agg.values()) for k in range(3)]
    print(f"total warp instr {tot[0]:.3e}  thread instr {tot[1]:.3e}  samples {tot[2]:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{v[2]/tot[2]*100:5.1f}% smp {v[0]/tot[0]*100:5.1f}% ins {v[1]/max(v[0],1):5.1f}thr  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
