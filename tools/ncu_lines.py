"""Per-CUDA-source-line instruction and stall attribution of one kernel in an ncu report.

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [inst|stall]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
by = sys.argv[4] if len(sys.argv) > 4 else "inst"  # or "stall"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    try:
        inst = float(d.get("Instructions Executed", "0") or 0)
        st = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, r[1].strip()[:70]])
    a[0] += inst
    a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("total warp-inst %.3e" % ti)
for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0 if by == "inst" else 1])[:top]:
    print("%5.1f%% inst %5.1f%% stall  %s:%d  %s" % (100 * i / ti, 100 * s / ts, f, ln, src))
