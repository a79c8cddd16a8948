"""Per-source-line stall samples and instruction counts of one kernel from an
ncu report (--page source --print-source cuda,sass), top lines first.

    python tools/ncu_lines.py report.ncu-rep function_substring [top] [nth]

``nth`` picks the n-th function (0-based) whose name contains the substring.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
nth = int(sys.argv[4]) if len(sys.argv) > 4 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname = func = None
hdr = None
funcs = []   # distinct matching function names in order
rows = {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        func = r[1]
        if kern in func and (not funcs or funcs[-1] != func):
            if func not in funcs:
                funcs.append(func)
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit() or func is None or kern not in func:
        continue
    if len(funcs) <= nth or func != funcs[nth]:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    stalls = {k[6:]: int(v) for k, v in d.items()
              if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
    key = f"{fname}:{r[0]}"
    if key in rows:
        continue
    rows[key] = (samples, inst, key, r[1].strip()[:90], stalls)
vals = list(rows.values())
tot_s = sum(x[0] for x in vals) or 1
tot_i = sum(x[1] for x in vals) or 1
print(f"{funcs[nth][:100] if funcs else '?'}\ntotal samples {tot_s}, instructions {tot_i}")
for s, i, loc, src, st in sorted(vals, key=lambda x: -x[0])[:top]:
    top_st = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% ins  {loc:16s} {src}  {top_st}")
