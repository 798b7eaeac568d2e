"""Print the last call's K5 launches from tools/k5_launches.sh CSVs: python tools/k5_launch_table.py gpurun_out/k5l_*.csv"""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0].isdigit()]
    calls, cur = [], []
    for r in rows:
        name, t = r[4], float(r[-1]) / 1000
        if 'hist<false>' in name or 'hist<(bool)0>' in name or 'upsweep' in name:
            if cur:
                calls.append(cur)
            cur = []
        tag = 'up' if ('upsweep' in name or 'hist<false>' in name or 'hist<(bool)0>' in name) else (
            'ih' if 'hist' in name else 'p')
        cur.append((tag, t))
    calls.append(cur)
    c = calls[-1]
    print(f.split('/')[-1], ' '.join('%s%.1f' % x for x in c), 'sum %.1f' % sum(x[1] for x in c))
