"""cfg T with the radar overlay: settle with plain cycles, then a few Doppler cycles (for ncu launch lists
of the NEXT-1 path).  Usage: python tools/doppler_run.py [n_doppler_cycles]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I  # noqa: E402

cfg = I.CONFIGS["cfgT"]
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
for k in range(30):
    f.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for k in range(30, 30 + n):
    m = sc.frame(k, device="cuda").contiguous()
    dop, pA = sc.doppler(k, m, frac=0.5, p_assoc=0.8, sd=0.25, device="cuda")
    torch.cuda.synchronize()
    last = k == 30 + n - 1
    if last:
        torch.cuda.nvtx.range_push("capture")   # ncu --nvtx --nvtx-include "capture/": the last cycle only
    f.step_doppler(m, dop.contiguous(), pA.contiguous(), cfg.dt)
    if last:
        torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", int((pA > 0).sum()))
