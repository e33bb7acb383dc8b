"""Top source lines of an ncu source-page export by warp-stall samples.

    python tools/ncu_lines.py source.csv [N]

source.csv: ncu -i rep --page source --csv --print-source cuda,sass.
Prints file:line, share of samples, dominant stall reasons and the source text."""
import csv
import sys
from collections import defaultdict


def main(path, n=40):
    n = int(n)
    f = None
    cur = None
    hdr = None
    text = {}
    rows = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name":
            continue
        if r[0] != "":
            cur = (f, int(r[0]))
            text[cur] = r[1]
            continue
        if r[2].startswith("0x"):
            rows.setdefault(int(r[2], 16), (cur, r))
    col = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: defaultdict(float))
    for c, r in rows.values():
        a = agg[c]
        a["samples"] += float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        a["inst"] += float(r[col["Instructions Executed"]] or 0)
        for s in stalls:
            v = r[col[s]]
            a[s] += float(v) if v not in ("", "-") else 0.0
    ts = sum(a["samples"] for a in agg.values())
    ti = sum(a["inst"] for a in agg.values())
    for c, a in sorted(agg.items(), key=lambda t: -t[1]["samples"])[:n]:
        top = sorted(((a[s], s) for s in stalls), reverse=True)[:3]
        why = ", ".join(f"{s[6:]} {100 * v / max(a['samples'], 1):.0f}%" for v, s in top)
        print(f"{c[0][:14]:14s}:{c[1]:<4d} {100 * a['samples'] / ts:5.2f}% inst {100 * a['inst'] / ti:5.2f}%  "
              f"{why:45s} {text.get(c, '').strip()[:70]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
