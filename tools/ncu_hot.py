"""Top stalled source lines of one kernel in an ncu report.

python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [--sass]

Default: CUDA source lines (needs -lineinfo and --import-source on), summed
warp-stall samples per (file, line).  --sass: per SASS instruction.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
sass = "--sass" in sys.argv
mode = "sass" if sass else "cuda,sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode,
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg: dict = {}
cur_file = "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Address", "#"):
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        si = hdr.index("Warp Stall Sampling (All Samples)")
        v = float(r[si] or 0)
    except (ValueError, IndexError):
        continue
    if sass:
        key = (r[0][-6:], r[hdr.index("Source")].strip()[:100])
    else:
        if not r[0].isdigit():
            continue
        key = (f"{cur_file}:{r[0]}", r[1].strip()[:100])
    agg[key] = agg.get(key, 0.0) + v
tot = sum(agg.values())
print(f"total samples {tot:.0f}")
for (loc, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v:8.0f} {100 * v / max(tot, 1):5.1f}%  {loc:>22} {src}")
