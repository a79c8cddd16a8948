"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
python tools/launches.py launches.csv [n_show]"""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg, seq = {}, []
for r in rows[1:]:
    name, v = r[ki][:70], float(r[vi].replace(",", "")) / 1000
    agg[name] = agg.get(name, 0) + v
    seq.append((name, v))
tot = sum(v for _, v in seq)
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:9.1f} us {v / tot * 100:5.1f}%  {k}")
print(f"total {tot:.1f} us over {len(seq)} launches")
for n, v in seq[:int(sys.argv[2]) if len(sys.argv) > 2 else 0]:
    print(f"{v:8.1f} {n}")
