"""Summarise ncu reports into profiles/ (run here, on the CPU box, after gpurun brings the .ncu-rep back).

    python tools/ncu_summary.py gpurun_out/gemm.ncu-rep [more.ncu-rep ...] --out profiles/round1_ncu_summary.json

Per profiled launch: kernel, grid, duration, DRAM bytes read/written (the
`traffic` numerator of bench.py's roofline), tensor-pipe and issue
utilisation, and the top warp-stall reasons.
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_mb",
    "dram__bytes_write.sum": "dram_write_mb",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg": "cycles",
}


def summarize(rep: str) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        rec = {"report": Path(rep).name, "kernel": d.get("Kernel Name", "")[:80], "grid": d.get("Grid Size"),
               "block": d.get("Block Size")}
        for k, name in KEYS.items():
            v = d.get(k)
            if v in (None, ""):
                continue
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            unit = u.get(k, "")
            if name.endswith("_mb"):
                f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
            if name == "duration_us":
                f = f * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
            rec[name] = round(f, 3)
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "")))
                  for h, v in d.items()
                  if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")
                  and v.replace(",", "").replace(".", "").isdigit()]
        stalls.sort(key=lambda x: -x[1])
        tot = sum(s for _, s in stalls) or 1.0
        rec["top_stalls"] = {k: round(v / tot, 3) for k, v in stalls[:5]}
        out.append(rec)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out_path = None
    if "--out" in args:
        i = args.index("--out")
        out_path = args[i + 1]
        args = args[:i] + args[i + 2:]
    recs = [r for rep in args for r in summarize(rep)]
    text = json.dumps(recs, indent=1)
    if out_path:
        Path(out_path).write_text(text + "\n")
    print(text)
