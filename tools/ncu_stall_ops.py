"""Stall-reason totals per SASS opcode (and per execution-count class) of one kernel in an ncu report.

    python tools/ncu_stall_ops.py report.ncu-rep kernel_regex [min_exec]
Rows with Instructions Executed >= min_exec only (e.g. the per-chunk hot loop)."""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
min_ex = int(sys.argv[3]) if len(sys.argv) > 3 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ie = hdr.index("Instructions Executed")
by_op = collections.defaultdict(collections.Counter)
tot = collections.Counter()
n_ex = collections.Counter()
for r in data:
    ex = float(r[ie] or 0)
    if ex < min_ex:
        continue
    src = r[1].strip()
    tok = src.split()
    op = tok[0] if not tok[0].startswith("@") else tok[1]
    op = op.split(".")[0]
    n_ex[op] += ex
    for h in stalls:
        v = float(r[hdr.index(h)] or 0)
        by_op[op][h] += v
        tot[h] += v
T = sum(tot.values()) or 1
print("total samples", T, {k[6:]: round(v / T, 3) for k, v in tot.most_common(8)})
for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
    s = sum(c.values())
    print(f"{op:10s} {s / T:6.3f} exec {n_ex[op]:12.0f}  " + " ".join(f"{k[6:]}={v / T:.3f}" for k, v in c.most_common(4)))
