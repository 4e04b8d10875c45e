"""Summarise an ncu report: one block of key metrics per profiled kernel (reads `ncu -i ... --page details`)."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'Executed Instructions',
        'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Issue Slots Busy', 'No Eligible', 'Dynamic Shared Memory Per Block', 'Static Shared Memory Per Block',
        'Waves Per SM', 'Eligible Warps Per Scheduler', 'Grid Size', 'Block Size']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'ID', 'Metric Name', 'Metric Value', 'Metric Unit'))
    cur = None
    for r in rows[1:]:
        key = (r[ii], r[ki])
        if key != cur:
            cur = key
            print(f"== [{r[ii]}] {r[ki].split('(')[0]}")
        if r[mi] in WANT:
            print(f"   {r[mi]:34s} {r[vi]:>14s} {r[ui]}")


if __name__ == '__main__':
    main(sys.argv[1])
