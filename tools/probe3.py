"""The bench's frame sequence (settle + warm-up + timed, then the timed frames again) with a synchronize
after each cycle (diagnostics)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS["cfgT"]
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
seq = list(range(53)) + list(range(33, 53))
for i, k in enumerate(seq):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
    torch.cuda.synchronize()
    print("cycle", i, "frame", k, "ok", flush=True)
