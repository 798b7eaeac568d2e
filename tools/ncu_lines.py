"""Per-source-line warp-stall samples and instruction counts of an ncu report (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py rep.ncu-rep [nlines] [kernel-substring]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, hdr, acc = '', None, {}
    tot_s = tot_i = 0
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            cur_file = r[1].split('/')[-1]
            continue
        if r[0] == 'Line No':
            hdr = r
            si = hdr.index('Warp Stall Sampling (All Samples)')
            ii = hdr.index('Instructions Executed')
            continue
        if hdr is None or r[0] in ('Function Name',) or len(r) <= ii:
            continue
        if r[0]:  # a source line row: aggregate of its SASS
            try:
                s, i = int(r[si] or 0), int(r[ii] or 0)
            except ValueError:
                continue
            key = (cur_file, int(r[0]))
            a = acc.setdefault(key, [0, 0, r[1].strip()[:90]])
            a[0] += s
            a[1] += i
            tot_s += s
            tot_i += i
    print(f'samples {tot_s}  warp-instructions {tot_i}')
    for (f, ln), (s, i, src) in sorted(acc.items(), key=lambda x: -x[1][0])[:n]:
        print(f'{100.0 * s / max(tot_s, 1):5.1f}% samp {100.0 * i / max(tot_i, 1):5.1f}% inst  {f}:{ln}  {src}')


if __name__ == '__main__':
    main()
