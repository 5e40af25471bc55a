"""Per-source-line cost of one kernel from an ncu report (--set full,
-lineinfo build): joins ncu's SASS page (per-address executed instructions
and stall samples) with nvdisasm's line table of the same cubin.

    python tools/sass_lines.py REPORT.ncu-rep CUBIN MANGLED_NAME [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def line_table(cubin, fn):
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    start = out.find(f".text.{fn}:")
    if start < 0:
        raise SystemExit(f"{fn} not in {cubin}")
    body = out[start:]
    end = body.find("\n.text.", 10)
    body = body if end < 0 else body[:end]
    cur = ("?", 0)
    table = {}
    for ln in body.splitlines():
        m = re.search(r'line (\d+)', ln) if "//##" in ln else None
        if m:
            f = re.search(r'File "([^"]+)"', ln)
            cur = (f.group(1).split("/")[-1] if f else "?", int(m.group(1)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return table


def main():
    rep, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(cubin, fn)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ai, ie, ss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[hdr_i + 1:] if len(r) > ie and r[ai].startswith("0x")]
    base = int(data[0][ai], 16)
    by_line = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    tot_i = tot_s = 0
    for r in data:
        off = int(r[ai], 16) - base
        key, ins = table.get(off, (("?", 0), r[1]))
        n = int(float(r[ie] or 0))
        smp = int(float(r[ss] or 0))
        e = by_line[key]
        e[0] += n
        e[1] += smp
        e[2][ins.split()[0] if not ins.startswith("@") else ins.split()[1]] += n
        tot_i += n
        tot_s += smp
    print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
    for key, (n, smp, ops) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{key[0]}:{key[1]:<5} inst {100 * n / tot_i:5.1f}%  stall {100 * smp / max(1, tot_s):5.1f}%  "
              + " ".join(f"{o}:{c * 100 // max(1, n)}" for o, c in ops.most_common(5)))


if __name__ == "__main__":
    main()
