"""Write profiles/ncu_traffic.json from the round's `ncu --set full` captures:
dram__bytes_read.sum + dram__bytes_write.sum of the captured attention launch, per workload
(bench.py reports it as roofline.traffic).
  python scripts/ncu_traffic.py r01 c2_sharegpt c2_alpaca c5_beam"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep: str) -> int:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    total = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = head.index(name)
        total += float(vals[i].replace(",", "")) * UNIT[units[i]]
    return int(round(total))


def main():
    tag, cfgs = sys.argv[1], sys.argv[2:]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel of bench.py's "
                  "default path for the workload (paged_attention_coop_kernel; paged_attention_shared_kernel for "
                  "c5_beam, whose coop figure is c5_beam_coop), one ncu --set full capture per round "
                  f"(profiles/{tag}_<workload>[_coop]_attention_ncu_details.txt); keyed by workload then n_gpus")
    for c in cfgs:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_attn_{c}_{tag}.ncu-rep")
        if os.path.exists(rep):
            d.setdefault(c, {})["1"] = dram_bytes(rep)
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
