"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum and,
when present, dram__bytes_read.sum / dram__bytes_write.sum)."""
import collections
import csv
import sys


def base_name(k):
    """Kernel name without its trailing (argument list), template arguments kept."""
    k = k.strip()
    if k.endswith(")"):
        depth = 0
        for i in range(len(k) - 1, -1, -1):
            depth += k[i] == ")"
            depth -= k[i] == "("
            if depth == 0:
                k = k[:i]
                break
    return k.replace("void ", "").replace("rimdp_dev::", "").replace("(bool)", "").replace("(int)", "")


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
        name[r[idi]] = base_name(r[ki])
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, d in per.items():
        t = tot[name[lid]]
        t[0] += 1
        t[1] += d.get("gpu__time_duration.sum", 0.0)
        t[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    allt = sum(t[1] for t in tot.values()) or 1.0
    for k, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        extra = f"  dram {b / n / 1e6:10.1f} MB/launch" if b else ""
        print(f"{k[:60]:60s} {n:5d} {t / n / 1e3:10.1f} us/launch  share {t / allt:.3f}{extra}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
