"""Summarise an ncu --set full capture of the tracker kernel into JSON.

    python tools/ncu_summary.py report.ncu-rep paths_in_capture out.json

Records duration, DRAM bytes, FP64-pipe and issue utilisation, occupancy,
registers, shared memory, the warp-stall breakdown and the per-phase split
(tools/ncu_phases.py) -- the numbers DESIGN.md and bench.py's roofline cite."""

import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main(rep, paths, outp):
    d, units = raw(rep)
    m = {k: d.get(k) for k in KEYS}
    st = {}
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    stalls = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda t: -t[1]) if v / tot >= 0.01}

    def nbytes(k):
        return float(d[k].replace(",", "")) * SCALE.get(units.get(k, "byte"), 1)

    dram = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = outp + ".src.csv"
    open(tmp, "w").write(src)
    sys.path.insert(0, "tools")
    import ncu_phases
    buf = io.StringIO()
    old = sys.stdout
    sys.stdout = buf
    try:
        ncu_phases.main(tmp)
    finally:
        sys.stdout = old
    import os
    os.remove(tmp)
    json.dump({"source": f"ncu --set full --clock-control none --import-source on -k regex:track_ -c 1, "
                         f"tools/probe_c5.py {paths} (C5 paths 0..{int(paths) - 1})",
               "metrics": m, "units": {k: units.get(k) for k in KEYS},
               "dram_bytes": dram, "dram_bytes_per_path": dram / float(paths),
               "stall_fractions": stalls, "phases": buf.getvalue().strip().splitlines()},
              open(outp, "w"), indent=1)
    print(open(outp).read())


if __name__ == "__main__":
    main(*sys.argv[1:])
