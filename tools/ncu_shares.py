"""Summarise an ncu launch list (gpu__time_duration.sum CSV) into per-kernel shares (markdown)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, bi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Block Size")
    agg = collections.OrderedDict()
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "").replace("probe::", "")
        key = f"{name} {r[bi]}"
        agg.setdefault(key, []).append(float(r[vi].replace(",", "")) / 1000.0)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel (block size) | launches | mean µs | share of kernel time |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
