"""Per-kernel device times of a few cycles at steady state (torch.profiler / CUPTI), for the modes of the
cycle: plain | exact | exact_lik | doppler.  Usage: python tools/kernel_times.py [mode] [config] [n]"""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "exact_lik"
cfg = I.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "cfgT"]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
for k in range(30):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)


def inputs(k):
    m = sc.frame(k, device="cuda").contiguous()
    if mode == "exact":
        return (I.Scene.exact_obs(m),)
    if mode == "exact_lik":
        return tuple(t.cuda().contiguous() for t in sc.exact_lik(k, m.cpu()))
    if mode == "doppler":
        d, p = sc.doppler(k, m.cpu())
        return (m, d.cuda().contiguous(), p.cuda().contiguous())
    return (m,)


step = {"plain": f.step, "exact": f.step_exact, "exact_lik": f.step_exact_lik, "doppler": f.step_doppler}[mode]
if mode in ("exact", "exact_lik"):
    for k in range(30, 42):
        f.step_exact(I.Scene.exact_obs(sc.frame(k, device="cuda").contiguous()), cfg.dt)
ins = [inputs(k) for k in range(42, 42 + n + 3)]
for x in ins[:3]:
    step(*x, cfg.dt)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for x in ins[3:]:
        step(*x, cfg.dt)
    torch.cuda.synchronize()
if len(sys.argv) > 4 and sys.argv[4] == "timeline":   # start / end of every kernel of the last cycle
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start)
    last = ev[-(len(ev) // n):]
    t0 = last[0].time_range.start
    for e in last:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  "
              f"{e.name.split('(')[0].replace('void dog::', '')[:50]}")
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0].replace("void dog::", "")[:60]
        tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / n:9.1f} us/cycle  x{cnt[k] / n:4.1f}  {k}")
print(f"{s / n:9.1f} us/cycle total kernel time ({mode}, {n} cycles)")
