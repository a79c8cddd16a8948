"""Per-source-line instruction counts and stall samples of one kernel from an
ncu report (--page source --print-source cuda,sass), top lines first.
    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = []
fname = None
agg = {}
tot_i = tot_s = 0
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    try:
        samples = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    if r[2] != "-":   # sass row
        continue
    key = f"{fname}:{r[0]}"
    a = agg.setdefault(key, [0, 0, r[1].strip()[:80]])
    a[0] += inst; a[1] += samples
    tot_i += inst; tot_s += samples
print(f"total inst {tot_i:,}  samples {tot_s:,}")
for k, (i, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{i/tot_i*100:5.1f}% inst {s/tot_s*100:5.1f}% smp  {k:22s} {src}")
