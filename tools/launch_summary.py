"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, collections, sys

def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0]
        tot[k][0] += 1
        tot[k][1] += v
    allt = sum(t for _, t in tot.values())
    for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {n:5d} {t / n / 1e3:10.1f} us/launch  share {t / allt:.3f}")

if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
