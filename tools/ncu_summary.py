"""Summarise an ncu --set full report (per kernel: duration, DRAM bytes, SM /
FP64 / issue utilisation, occupancy, warp efficiency, top stall reasons) into
profiles/<name>.json and .md.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_composite
"""
import csv, io, json, subprocess, sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d["Kernel Name"].split("(")[0]}
        for name, m in METRICS.items():
            v = d.get(m)
            try:
                v = float(str(v).replace(",", ""))
            except (TypeError, ValueError):
                v = None
            u = unit.get(m, "").lower()
            if v is not None and name.endswith("_mb"):
                v *= {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1.0, "gbyte": 1e3, "tbyte": 1e6}.get(u, 1.0)
            if v is not None and name == "duration_us":
                v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                      "msecond": 1e3}.get(u, 1.0)
            k[name] = v
        stalls = []
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), key.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        k["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:5]}
        res.append(k)
    with open(out + ".json", "w") as f:
        json.dump({"report": rep, "kernels": res}, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu summary: `{rep}`\n\n")
        cols = ["kernel", "duration_us", "dram_read_mb", "dram_write_mb", "dram_throughput_pct",
                "fp64_pipe_pct", "issue_active_pct", "warps_active_pct", "threads_per_inst",
                "registers", "top_stalls_pct"]
        f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for k in res:
            f.write("| " + " | ".join(str(k.get(c) if not isinstance(k.get(c), float)
                                          else round(k.get(c), 2)) for c in cols) + " |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
