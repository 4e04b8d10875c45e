"""Print the bench stage times and the warm per-kernel launch list of the last tools/gpu_cycle.sh run."""
import csv
import json

d = json.loads(open('gpurun_out/bench_cur.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['stages_ms'])
rows = [r for r in csv.reader(open('gpurun_out/launches_warm.csv')) if len(r) > 10]
h = rows[0]
tot = 0
for r in rows[1:]:
    v = float(r[h.index('Metric Value')].replace(',', ''))
    tot += v
    print(f"{r[h.index('Kernel Name')].split('(')[0][:30]:30s} {v / 1000:8.1f} us")
print(f"sum {tot / 1000:.1f} us")
