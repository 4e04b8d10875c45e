"""probe3's frame sequence back to back (no synchronize between cycles)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS["cfgT"]
sc = I.scene(cfg)
frames = [sc.frame(k, device="cuda").contiguous() for k in range(53)]
f = dog.Filter.from_config(cfg)
seq = list(range(53)) + list(range(33, 53))
sync_every = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for i, k in enumerate(seq):
    f.step(frames[k], cfg.dt)
    if sync_every and i % sync_every == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("ok", flush=True)
