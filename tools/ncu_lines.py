"""Instructions executed per source line of one kernel in an ncu report, with file attribution; prints
per-file totals and the top lines, or the total over a file's line range (`file:a-b`)."""
import csv
import io
import subprocess
import sys


def load(path, kernel):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '-k', f'regex:{kernel}',
                          '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
    fname, hdr, tot = '?', None, {}
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr is None or len(r) < 5 or not r[0].isdigit():
            continue
        v = r[hdr.index('Instructions Executed')]
        e = int(v) if v.isdigit() else 0
        tot[(fname, int(r[0]), r[1].strip()[:90])] = tot.get((fname, int(r[0]), r[1].strip()[:90]), 0) + e
    return tot


def main(path, kernel, *ranges):
    tot = load(path, kernel)
    allv = sum(tot.values()) or 1
    byf = {}
    for (f, _, _), e in tot.items():
        byf[f] = byf.get(f, 0) + e
    print('total', allv, {f: round(100 * e / allv, 1) for f, e in sorted(byf.items(), key=lambda x: -x[1])})
    for rg in ranges:
        f, ab = rg.split(':')
        a, b = (int(x) for x in ab.split('-'))
        e = sum(v for (ff, ln, _), v in tot.items() if ff == f and a <= ln <= b)
        print(f'{rg}: {e} ({100 * e / allv:.1f}%)')
    if not ranges:
        for (f, ln, src), e in sorted(tot.items(), key=lambda x: -x[1])[:30]:
            print(f'{100 * e / allv:5.1f}% {e:9d} {f}:{ln}: {src}')


if __name__ == '__main__':
    main(*sys.argv[1:])
