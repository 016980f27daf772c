"""Per-instruction execution counts and stall samples from an ncu report (SASS view)."""
import csv, subprocess, sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ai, si, ei, wi = (hdr.index(x) for x in ('Address', 'Source', 'Instructions Executed', 'Warp Stall Sampling (All Samples)'))
tot = 0
lines = []
for r in rows[2:]:
    try:
        n = int(r[ei] or 0)
    except ValueError:
        continue
    tot += n
    lines.append((r[ai][-5:], r[si][:64], n, r[wi]))
print('total warp-instructions', tot, 'per unit', tot / norm)
for a, s, n, w in lines:
    if n:
        print(f'{a} {s:64s} {n / norm:8.3f} {w}')
