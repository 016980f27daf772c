"""Summarise an ncu report: key metrics, stall reasons, per-kernel launch shares."""
import csv, subprocess, sys, collections

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'lts__t_sector_hit_rate.pct', 'sm__cycles_elapsed.avg.per_second',
        'smsp__inst_executed.sum', 'l1tex__t_sector_hit_rate.pct', 'lts__t_bytes.sum']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        res.append(d)
    return res


def main(rep):
    for d in raw(rep):
        print('kernel:', d.get('Kernel Name', ('?',))[0][:100])
        for k in KEYS:
            if k in d:
                print(f'  {k:60s} {d[k][0]:>16s} {d[k][1]}')
        st = [(h, float(v[0])) for h, v in d.items() if h.startswith('smsp__pcsamp_warps_issue_stalled')
              and not h.endswith('not_issued') and v[0] not in ('', 'n/a')]
        st.sort(key=lambda x: -x[1])
        tot = sum(v for _, v in st) or 1
        print('  stalls:', ', '.join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.0%}" for h, v in st[:8]))


if __name__ == '__main__':
    main(sys.argv[1])
