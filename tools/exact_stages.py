"""cfg T exact PHD/MIB (NEXT-3) at steady state: settle with plain cycles, run exact cycles until the cycle
time converges, then per-stage device times of a few more (dog_profile_*).  Usage:
python tools/exact_stages.py [config] [n_exact_before] [n_profiled]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I  # noqa: E402

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfgT"]
n_before = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n_prof = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
for k in range(30):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
for k in range(30, 30 + n_before):
    f.step_exact(I.Scene.exact_obs(sc.frame(k, device="cuda").contiguous()), cfg.dt)
torch.cuda.synchronize()
obs = [I.Scene.exact_obs(sc.frame(k, device="cuda").contiguous()) for k in range(30 + n_before, 30 + n_before + n_prof)]
f.profile_begin(n_prof)
for o in obs:
    f.step_exact(o, cfg.dt)
torch.cuda.synchronize()
st, n = f.profile_end()
print({k: round(v / n * 1000, 1) for k, v in st.items()}, "us per cycle; total", round(sum(st.values()) / n, 3), "ms")
