"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python tools/launch_share.py gpurun_out/launches.csv [--last-step N] --out profiles/roundX_launches.json

ncu serialises launches and runs them cold-cache, so absolute times differ from
bench.py's CUDA-event numbers; the SHARE of each kernel in the step is what is
compared.  ``--last-step N`` keeps only the last N launches of our kernels
(one timed step: bench.py --profile --steps 1 --warmup 1 runs two steps).
"""

import csv
import io
import json
import re
import sys
from collections import OrderedDict
from pathlib import Path


def short(name: str) -> str:
    m = re.match(r"(?:void )?([\w:]+)(<[^()]*>)?", name)
    base = m.group(1) if m else name[:60]
    tmpl = m.group(2) if m and m.group(2) else ""
    return (base.split("::")[-1] + tmpl)[:70]


def main(argv):
    path = argv[0]
    out = None
    last = None
    if "--out" in argv:
        out = argv[argv.index("--out") + 1]
    if "--last-step" in argv:
        last = int(argv[argv.index("--last-step") + 1])
    text = Path(path).read_text()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    recs = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        recs.append((short(r["Kernel Name"]), ns, r["Grid Size"]))
    if last:
        recs = recs[-last:]
    agg = OrderedDict()
    for name, ns, grid in recs:
        a = agg.setdefault(name, {"launches": 0, "ms": 0.0})
        a["launches"] += 1
        a["ms"] += ns * 1e-6
    tot = sum(a["ms"] for a in agg.values())
    res = {"source": Path(path).name, "launches": len(recs), "total_ms": round(tot, 3), "kernels": {}}
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        res["kernels"][name] = {"launches": a["launches"], "ms": round(a["ms"], 3), "share": round(a["ms"] / tot, 4)}
    s = json.dumps(res, indent=1)
    if out:
        Path(out).write_text(s + "\n")
    print(s)


if __name__ == "__main__":
    main(sys.argv[1:])
