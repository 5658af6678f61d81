"""Top warp-stall SASS lines of one kernel from an ncu report (ncu -i ... --page source --csv --print-source=sass).

    python tools/ncu_hot_sass.py report.ncu-rep kernel_regex [launch_index] [n]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
li = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}",
                      "--launch-skip", str(li), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(txt))]
hdr = next(r for r in rows if "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data) or 1
print(f"{len(data)} SASS lines, {tot:.0f} samples")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    print(f"{float(r[i_s]) / tot:6.3f} {r[0][-5:]} ex={r[i_e]:>9} {r[1].strip()[:100]}")
