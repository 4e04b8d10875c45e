"""Back-to-back cycles without host synchronisation (diagnostics for launch-overlap races)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfgT"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 35
sc = I.scene(cfg)
frames = [sc.frame(k, device="cuda").contiguous() for k in range(n)]
f = dog.Filter.from_config(cfg)
for k in range(n):
    f.step(frames[k], cfg.dt)
torch.cuda.synchronize()
print("back-to-back ok", flush=True)
