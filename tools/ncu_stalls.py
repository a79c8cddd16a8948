"""Per-source-line stall samples (long scoreboard, wait, short scoreboard, ...)
of one kernel: python tools/ncu_stalls.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
hdr = None
fname = ""
agg = {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    key = f"{fname}:{r[0]}"
    d = agg.setdefault(key, {"src": r[1].strip()[:70]})
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                d[h] = d.get(h, 0) + int(r[i])
            except ValueError:
                pass
tot = sum(v for d in agg.values() for k, v in d.items() if k != "src")
print("total samples", tot)
rows = sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "src"))
for k, d in rows[:top]:
    s = sum(v for kk, v in d.items() if kk != "src")
    tops = sorted(((v, kk[6:]) for kk, v in d.items() if kk != "src" and v), reverse=True)[:3]
    print(f"{s/tot*100:5.1f}% {k:22s} {' '.join(f'{n}={v/tot*100:.1f}' for v, n in tops):45s} {d['src']}")
