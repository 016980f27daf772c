"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum and,
when present, dram__bytes_read.sum / dram__bytes_write.sum)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    idi = hdr.index("ID")
    per = collections.defaultdict(dict)  # launch id -> metric -> value
    name = {}
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per[r[idi]][r[mi]] = v
        name[r[idi]] = r[ki].split("(")[0]
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, d in per.items():
        t = tot[name[lid]]
        t[0] += 1
        t[1] += d.get("gpu__time_duration.sum", 0.0)
        t[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    allt = sum(t[1] for t in tot.values()) or 1.0
    for k, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        extra = f"  dram {b / n / 1e6:10.1f} MB/launch" if b else ""
        print(f"{k[:70]:70s} {n:5d} {t / n / 1e3:10.1f} us/launch  share {t / allt:.3f}{extra}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
