"""Summarise ncu reports (--set full) into the numbers DESIGN.md and bench.py quote:
duration, DRAM bytes read/written, DRAM / L2 throughput, L2 hit rate, issue-slot use,
occupancy, registers, instructions.  python scripts/ncu_summary.py report.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

WANT = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum":
        "dram_write", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_nominal",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_pct", "sm__inst_executed.sum": "instructions",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "launch__registers_per_thread": "registers", "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct"}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, name in WANT.items():
            if k in hdr:
                v, u = r[hdr.index(k)], units[hdr.index(k)]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if k.startswith("dram__bytes"):
                    x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if k == "gpu__time_duration.sum":
                    x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
                d[name] = x
        if "dram_read" in d and "duration_us" in d:
            d["dram_gbs"] = (d["dram_read"] + d.get("dram_write", 0)) / (d["duration_us"] * 1e-6) / 1e9
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarise(p):
            print(json.dumps({"report": p.split("/")[-1], **d}))
