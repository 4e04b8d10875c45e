"""Source lines of one kernel in an ncu report ranked by instructions executed (`--page source`)."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=30):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '-k', f'regex:{kernel}',
                          '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, lines, fname, per_file = None, [], "?", {}
    for r in rows:
        if len(r) == 2 and r[0] in ('File Name', 'File Path'):
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if len(r) == 2 or hdr is None or len(r) < 5 or not r[0].isdigit():
            continue
        ei = hdr.index('Instructions Executed')
        e = int(r[ei]) if r[ei].isdigit() else 0
        lines.append((e, int(r[0]), fname + ': ' + r[1].strip()[:100]))
        per_file[fname] = per_file.get(fname, 0) + e
    tot = sum(x[0] for x in lines) or 1
    print(f'total instructions {tot}; per file:', {k: f'{100 * v / tot:.1f}%' for k, v in per_file.items()})
    for e, ln, src in sorted(lines, reverse=True)[:top]:
        print(f'{100 * e / tot:5.1f}% {e:9d} {ln}: {src}')


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
