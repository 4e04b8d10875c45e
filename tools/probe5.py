"""N plain cycles of a config, synchronising after each (diagnostics)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS[sys.argv[1]]
n = int(sys.argv[2])
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
for k in range(n):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
    torch.cuda.synchronize()
print("ok", n, flush=True)
