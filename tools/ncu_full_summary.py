"""Summarise an `ncu --set full` report (per launch: time, DRAM bytes, tensor-pipe and DRAM
utilisation, SM clock, registers) as a markdown table.  Usage: ncu_full_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread"]
HEAD = ["ms", "DRAM read GB", "DRAM write GB", "tensor active %", "DRAM %", "L2 hit %", "SM GHz", "regs"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = rows[0], rows[1], rows[2:]
    print("| launch | " + " | ".join(HEAD) + " |")
    print("|---" * (len(HEAD) + 1) + "|")
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("probe::", "")
        vals = []
        for m in METRICS:
            i = hdr.index(m) if m in hdr else -1
            v = r[i] if i >= 0 else "n/a"
            u = units[i] if i >= 0 else ""
            if m == "gpu__time_duration.sum" and u == "us":
                v = f"{float(v.replace(',', '')) / 1000:.4f}"
            elif m == "gpu__time_duration.sum" and u == "ns":
                v = f"{float(v.replace(',', '')) / 1e6:.4f}"
            elif m.startswith("dram__bytes") and u == "Mbyte":
                v = f"{float(v.replace(',', '')) / 1000:.4f}"
            vals.append(v)
        print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
