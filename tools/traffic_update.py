"""Update profiles/ncu_traffic.json from an ncu launch list of one config:
DRAM bytes (read + write) of one iteration's column phase = the sum over the
distinct omax_* kernels of their average bytes per launch (cold cache)."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def column_bytes(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per, name = collections.defaultdict(float), {}
    for r in rows[1:]:
        if r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        try:
            per[r[idi]] += float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name[r[idi]] = r[ki].split("(")[0].replace("rimdp_dev::", "").replace("void ", "")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for lid, b in per.items():
        if name[lid].startswith("omax_") or name[lid].startswith("bellman_short"):
            tot[name[lid]][0] += 1
            tot[name[lid]][1] += b
    return sum(b / n for n, b in tot.values()), sorted(tot)


def main(key, path):
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(f)) if os.path.exists(f) else {}
    b, ks = column_bytes(path)
    d[key] = {"dram_bytes_per_launch": b, "kernels": ks,
              "source": f"{os.path.relpath(path, ROOT)} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                        "dram__bytes_write.sum; sum over the column-phase kernels of one iteration, cold cache)"}
    json.dump(d, open(f, "w"), indent=1)
    print(key, f"{b / 1e6:.1f} MB per iteration over {len(ks)} column kernels")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
