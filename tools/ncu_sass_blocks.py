"""Hottest SASS basic blocks of one kernel in an ncu report (instructions executed x block length)."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=12, show=30):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '-k', f'regex:{kernel}',
                          '--print-source', 'sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == 'Address')
    ei, si = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
    blocks, cur = [], None
    for r in rows:
        if len(r) <= ei or not r[ei].isdigit():
            continue
        cnt, samp = int(r[ei]), int(r[si]) if r[si].isdigit() else 0
        if cur and cur['cnt'] == cnt:
            cur['ins'].append(r[1]); cur['samp'] += samp
        else:
            cur = {'start': r[0], 'cnt': cnt, 'ins': [r[1]], 'samp': samp}
            blocks.append(cur)
    tot = sum(b['cnt'] * len(b['ins']) for b in blocks)
    totS = sum(b['samp'] for b in blocks) or 1
    print(f'total {tot / 1e6:.2f}M instructions, {totS} samples')
    for b in sorted(blocks, key=lambda b: -b['cnt'] * len(b['ins']))[:top]:
        print(f"== {b['start']} cnt={b['cnt']} len={len(b['ins'])} {b['cnt'] * len(b['ins']) / 1e6:.2f}M "
              f"samples {100 * b['samp'] / totS:.1f}%")
        for i in b['ins'][:show]:
            print('      ', i)


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], *(int(a) for a in sys.argv[3:]))
