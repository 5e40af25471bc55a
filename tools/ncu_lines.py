"""Top CUDA source lines of an ncu --import-source capture by warp-stall samples
(the cuda,sass source view: one row per source line with its SASS summed).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows = "?", []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No", "") or len(r) < 8:
        continue
    rows.append((fname, r))
hdr = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Line No":
        hdr = r
        break
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
agg = {}
for f, r in rows:
    if r[iS] in ("-", "") or not r[iS].replace(".", "").isdigit():
        continue
    key = (f, r[0], r[1].strip()[:100])
    s, i = agg.get(key, (0.0, 0.0))
    agg[key] = (s + float(r[iS]), i + float(r[iI] or 0))
tot = sum(v[0] for v in agg.values()) or 1
totI = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f}, warp instructions {totI:.0f}")
for (f, ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s / tot * 100:5.1f}% stall {i / totI * 100:5.1f}% inst  {f}:{ln:<5} {src}")
