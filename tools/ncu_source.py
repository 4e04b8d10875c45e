"""Top source lines of one kernel in an ncu report by warp-stall samples (`--page source`)."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '-k', f'regex:{kernel}',
                          '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = []
    fname = '?'
    for r in rows:
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if len(r) == 2:
            fname = r[1].split('/')[-1][:24]
            continue
        if hdr is None or len(r) < 5 or not r[0].isdigit():
            continue
        si = hdr.index('Warp Stall Sampling (All Samples)')
        ei = hdr.index('Instructions Executed') if 'Instructions Executed' in hdr else None
        s = int(r[si]) if r[si].isdigit() else 0
        e = int(r[ei]) if ei is not None and r[ei].isdigit() else 0
        lines.append((s, e, fname, int(r[0]), r[1].strip()[:100]))
    tot = sum(x[0] for x in lines) or 1
    print(f'total samples {tot}')
    for s, e, f, ln, src in sorted(lines, reverse=True)[:top]:
        print(f'{100 * s / tot:5.1f}% {e:9d} {f}:{ln}: {src}')


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
