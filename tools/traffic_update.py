"""Update profiles/ncu_traffic.json from an ncu launch list of one config:
DRAM bytes (read + write) of one iteration's column phase = the sum over the
distinct omax_* kernels of their average bytes per launch (cold cache)."""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import base_name  # noqa: E402

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
        name[r[idi]] = base_name(r[ki])
    tot = collections.defaultdict(lambda: [0, 0.0])
    for lid, b in per.items():
        if name[lid].startswith(("omax_", "bellman_short", "exact_", "value_")):
            tot[name[lid]][0] += 1
            tot[name[lid]][1] += b
    return sum(b / n for n, b in tot.values()), sorted(tot)


def per_kernel(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per, name = collections.defaultdict(dict), {}
    for r in rows[1:]:
        try:
            per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name[r[idi]] = base_name(r[ki])
    out = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, d in per.items():
        t = out[name[lid]]
        t[0] += 1
        t[1] += d.get("gpu__time_duration.sum", 0.0)
        t[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    return {k: {"launches": n, "us_per_launch": t / n / 1e3, "dram_bytes_per_launch": b / n}
            for k, (n, t, b) in out.items() if not k.startswith("<unnamed>")}


def main(key, path):
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(f)) if os.path.exists(f) else {}
    b, ks = column_bytes(path)
    d[key] = {"dram_bytes_per_launch": b, "kernels": ks,
              "source": f"{os.path.relpath(path, ROOT)} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                        "dram__bytes_write.sum; sum over the column-phase kernels of one iteration, cold cache)",
              "per_kernel": {k: v for k, v in sorted(per_kernel(path).items())}}
    json.dump(d, open(f, "w"), indent=1)
    print(key, f"{b / 1e6:.1f} MB per iteration over {len(ks)} column kernels")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
