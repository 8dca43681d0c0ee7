"""Summarise ncu captures into profiles/ (key metrics + launch-list shares)."""
import csv, io, json, subprocess, sys, collections

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'lts__t_sectors.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__inst_executed.sum',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard', 'launch__occupancy_limit_registers']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {'kernel': r[hdr.index('Kernel Name')]}
        for k in KEYS:
            if k in hdr:
                d[k] = (r[hdr.index(k)], units[hdr.index(k)])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(',', ''))
    return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)


def launches(csvfile):
    rows = list(csv.reader(open(csvfile)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == 'ID')
    hdr = rows[i]
    tot = collections.Counter(); cnt = collections.Counter()
    for r in rows[i + 1:]:
        if len(r) != len(hdr) or r[hdr.index('Metric Name')] != 'gpu__time_duration.sum':
            continue
        k = r[hdr.index('Kernel Name')]
        tot[k] += float(r[hdr.index('Metric Value')].replace(',', '')); cnt[k] += 1
    T = sum(tot.values())
    return {k: {'launches': cnt[k], 'total_ns': tot[k], 'share': tot[k] / T,
                'avg_us': tot[k] / cnt[k] / 1e3} for k in sorted(tot, key=lambda x: -tot[x])}


if __name__ == '__main__':
    out = {}
    for a in sys.argv[2:]:
        if a.endswith('.ncu-rep'):
            out[a] = raw(a)
            for d in out[a]:
                if 'dram__bytes_read.sum' in d:
                    d['traffic_bytes'] = to_bytes(*d['dram__bytes_read.sum']) + to_bytes(*d['dram__bytes_write.sum'])
        elif a.endswith('.csv'):
            out[a] = launches(a)
    json.dump(out, open(sys.argv[1], 'w'), indent=1)
    print(json.dumps(out, indent=1)[:3000])
