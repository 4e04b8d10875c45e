"""Write profiles/<tag>_* summaries from a round's gpurun_out/ captures (see tools/gpu_round.sh).

    python tools/profile_summary.py r01
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE_OF = {"k_predict_sort": "predict_sort", "k_predict": "predict", "k_tilesort": "tilesort", "k_cells": "cells", "k_list_scan": "list_scan",
            "k_pair_fill": "pairs", "k_pair_sort": "pairs", "k_resample_tiles": "resample", "k_moments": "moments",
            "k_births": "births"}


def short(name):
    return name.split('(')[0].replace('void ', '').replace('dog::', '').split('<')[0]


def main(tag):
    go, pr = os.path.join(ROOT, 'gpurun_out'), os.path.join(ROOT, 'profiles')
    # launch list
    rows = [r for r in csv.reader(open(os.path.join(go, f'launches_{tag}.csv'))) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(short(r[ki]), []).append(float(r[vi].replace(',', '')) / 1000.0)
    ncyc = max(len(v) for v in per.values())
    tot = sum(sum(v) for v in per.values()) / ncyc
    with open(os.path.join(pr, f'{tag}_launches.txt'), 'w') as f:
        f.write(f'# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none, cfgT, {ncyc} cycles after '
                f'33 warm cycles (cold-cache, serialised: compare shares)\n')
        f.write('# kernel | launches | mean us | share of cycle\n')
        for k, v in per.items():
            f.write(f'{k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / ncyc / tot:.1f}%\n')
        f.write(f'# sum per cycle: {tot:.1f} us\n')
    # full captures
    out = subprocess.run(['ncu', '-i', os.path.join(go, f'full_{tag}.ncu-rep'), '--page', 'raw', '--csv'],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    H, U = rr[0], rr[1]
    keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
            'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
            'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']
    scale = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
    traffic = {}
    with open(os.path.join(pr, f'{tag}_full.txt'), 'w') as f:
        f.write(f'# {tag}: ncu --set full --clock-control none captures of the bench command (cfgT)\n')
        for row in rr[2:]:
            d, u = dict(zip(H, row)), dict(zip(H, U))
            name = short(d['Kernel Name'])
            f.write(f'## {name}\n')
            for k in keys:
                if k in d:
                    f.write(f'   {k:58s} {d[k]:>16s} {u.get(k, "")}\n')
            stalls = []
            for k, v in d.items():
                if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
                    try:
                        stalls.append((float(v), k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            f.write('   top stalls (warps per issue): ' + ', '.join(f'{n} {v:.2f}' for v, n in stalls[:5]) + '\n')
            b = float(d['dram__bytes_read.sum']) * scale[u['dram__bytes_read.sum']] + \
                float(d['dram__bytes_write.sum']) * scale[u['dram__bytes_write.sum']]
            st = STAGE_OF.get(name)
            if st and st not in traffic:
                traffic[st] = b
    tp = os.path.join(pr, 'ncu_traffic.json')
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old.update({k: v for k, v in traffic.items()})
    old['_source'] = f'profiles/{tag}_full.txt (dram__bytes_read.sum + dram__bytes_write.sum per launch)'
    json.dump(old, open(tp, 'w'), indent=1)
    print(open(os.path.join(pr, f'{tag}_launches.txt')).read())
    print(open(os.path.join(pr, f'{tag}_full.txt')).read())


if __name__ == '__main__':
    main(sys.argv[1])
