"""Summarise an ncu report: key raw metrics + top SASS stall lines.  python tools/ncu_summary.py rep.ncu-rep [nlines]"""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg',
        'launch__shared_mem_per_block_dynamic', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print('kernel:', v[h.index('Kernel Name')][:100])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f'  {w} = {v[i]} {u[i]}')
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]
    si = h.index('Warp Stall Sampling (All Samples)')
    cols = [i for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
    tot = {h[i]: 0 for i in cols}
    lines, total = [], 0
    for r in rows[2:]:
        try:
            s = int(r[si])
        except (ValueError, IndexError):
            continue
        total += s
        for i in cols:
            try:
                tot[h[i]] += int(r[i])
            except ValueError:
                pass
        lines.append((s, r[0], r[1]))
    print('stall samples', total)
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
        print(f'  {k} {v} ({100.0 * v / max(total, 1):.1f}%)')
    lines.sort(reverse=True)
    for s, a, src in lines[:n]:
        print(f'  {s:6d} {a[-5:]} {src}')


if __name__ == '__main__':
    main()
