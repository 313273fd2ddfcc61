"""Top stalled source lines of one kernel in an ncu report:
python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [--sass]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
mode = "sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode,
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"#"') or l.startswith('"Address"') or l.startswith('"Line"'))
rd = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rd[0]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
def val(r):
    try:
        return float(r[si] or 0)
    except (ValueError, IndexError):
        return 0.0
body = [r for r in rd[1:] if len(r) > si and r[0] != h[0]]
tot = sum(val(r) for r in body)
rows = sorted(body, key=lambda r: -val(r))[:n]
print(f"total samples {tot:.0f}")
for r in rows:
    print(f"{val(r):8.0f} {100*val(r)/max(tot,1):5.1f}%  {r[0][:6]:>6} {r[src].strip()[:110]}")
