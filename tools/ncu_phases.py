"""Attribute an ncu source-page export (--page source --csv --print-source
cuda,sass) of the tracker kernel to its phases.

    python tools/ncu_phases.py report.csv

Each SASS instruction is mapped to its source line; inlined helpers
(nid_common.cuh, homotopy.cuh ...) inherit the phase of the last tracker
line before them in address order.  Prints per-phase share of warp-stall
samples, executed instructions, and the top stall reasons of each phase."""

import csv
import sys
from collections import defaultdict

# (file, first line, last line, phase) -- track_ctl.cuh line ranges are read
# from markers in the source instead of hard-coding numbers
PHASE_FILES = {"track_rows.cuh": "eval", "track_ptab.cuh": "eval"}


def ctl_ranges(path):
    marks = {}
    for i, l in enumerate(open(path), 1):
        for key in ("NID_TP(0)", "NID_TP(1)", "NID_TP(2)", "NID_TP(3)", "NID_TP(4)", "NID_TP(5)", "NID_TP(6)"):
            if key in l and "define" not in l:
                marks[key] = i
    return marks


def main(csvp, ctl_src="paper_1804_03807_b200/csrc/track_ctl.cuh"):
    marks = ctl_ranges(ctl_src)
    order = [("control", 0, marks["NID_TP(0)"]), ("barrier", marks["NID_TP(0)"], marks["NID_TP(1)"]),
             ("eval", marks["NID_TP(1)"], marks["NID_TP(2)"]), ("barrier", marks["NID_TP(2)"], marks["NID_TP(3)"]),
             ("post_eval", marks["NID_TP(3)"], marks["NID_TP(4)"]), ("lu", marks["NID_TP(4)"], marks["NID_TP(5)"]),
             ("backsub", marks["NID_TP(5)"], marks["NID_TP(6)"]), ("tail", marks["NID_TP(6)"], 10 ** 9)]
    ctl_fn_end = None
    lu_lo = lu_hi = None
    for i, l in enumerate(open(ctl_src), 1):
        if "void track_body(" in l:
            ctl_fn_end = i
        if ("NID_D int lu_pivot" in l or "NID_D void lu_step" in l) and lu_lo is None:
            lu_lo = i
        if "// blocks per SM" in l:
            lu_hi = i

    def phase_of(f, line):
        if f == "track_ctl.cuh":
            if lu_lo and lu_lo <= line < lu_hi:
                return "lu"
            if ctl_fn_end and line < ctl_fn_end:
                return "control"
            for name, a, b in order:
                if a <= line < b:
                    return name
        if f in PHASE_FILES:
            return PHASE_FILES[f]
        return None

    by_addr = {}
    hdr = None
    f = None
    cur = None
    for r in csv.reader(open(csvp)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] != "":
            cur = (f, int(r[0]))
            continue
        if hdr is None or not r[2].startswith("0x"):
            continue
        e = by_addr.setdefault(int(r[2], 16), [[], r])
        e[0].append(cur)
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: defaultdict(float))
    last = "control"
    for addr in sorted(by_addr):
        lines, r = by_addr[addr]
        # an inlined instruction is listed under every line of its call chain:
        # the kernel body's line decides, then the evaluator, then control
        ph = None
        for fl, line in lines:
            if fl == "track_ctl.cuh" and lu_lo and lu_lo <= line < lu_hi:
                ph = "lu"
        for fl, line in lines:
            if ph is None and fl == "track_ctl.cuh" and ctl_fn_end and line >= ctl_fn_end:
                ph = phase_of(fl, line)
        if ph is None:
            for fl, line in lines:
                if fl in PHASE_FILES:
                    ph = PHASE_FILES[fl]
        if ph is None:
            for fl, line in lines:
                if fl == "track_ctl.cuh":
                    ph = "control"
        if ph is None:
            ph = last
        else:
            last = ph
        a = agg[ph]
        a["samples"] += float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        a["inst"] += float(r[col["Instructions Executed"]] or 0)
        for s in stall_cols:
            v = r[col[s]]
            a[s] += float(v) if v not in ("", "-") else 0.0
    ts = sum(a["samples"] for a in agg.values())
    ti = sum(a["inst"] for a in agg.values())
    for ph, a in sorted(agg.items(), key=lambda t: -t[1]["samples"]):
        top = sorted(((a[s], s) for s in stall_cols), reverse=True)[:5]
        print(f"{ph:10s} samples {100 * a['samples'] / ts:5.1f}%  inst {100 * a['inst'] / ti:5.1f}%  " +
              ", ".join(f"{s[6:]} {100 * v / max(a['samples'], 1):.0f}%" for v, s in top))


if __name__ == "__main__":
    main(*sys.argv[1:])
