mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/frame_c3.csv python tools/probe_frame.py c3 > /dev/null 2>&1; echo c3=$?
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/frame_c3.csv")))
st = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[st]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
ks = [(r[ki].split("(")[0].replace("void ", "")[:48], float(r[vi]) / 1e3) for r in rows[st + 1:] if len(r) > vi]
n = len(ks)
# the last frame: kernels after the 4th occurrence of the screen kernel
idx = [i for i, (nm, _) in enumerate(ks) if "knn_tc2_kernel" in nm]
last = ks[idx[-1] - 2:] if idx else ks[-20:]
tot = 0
for nm, us in last:
    tot += us
    print(f"{nm:50s} {us:8.1f} us")
print("total", round(tot, 1))
PY
