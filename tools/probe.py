"""Run N plain cycles of a config with a synchronize after each (diagnostics: find the failing cycle)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfgT"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 35
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
for k in range(n):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
    torch.cuda.synchronize()
    print("cycle", k, "ok", flush=True)
