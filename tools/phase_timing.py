"""Per-phase block times of the instrumented kernels (diagnostics build: DOG_NVCC_EXTRA=-DDOG_TIMING).

Runs the cfgT filter for 30 settle cycles, then 10 cycles with the phase counters reset; prints the
average per-block microseconds of each phase slot.  With a second argument "exact": 30 plain cycles, 8
exact PHD/MIB cycles, then 10 exact cycles measured (the run-heavy regime of NEXT-3)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

NAMES = {0: "rs A (loads)", 1: "rs B (moments, runof)", 2: "rs R (spanning segments)", 3: "rs C (F, copies)",
         4: "rs long runs", 8: "ps predict", 9: "ps radix passes", 10: "ps runs", 11: "ps lperm"}
cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfgT"]
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg)
frames = [sc.frame(k, device="cuda") for k in range(40)]
exact = len(sys.argv) > 2 and sys.argv[2] == "exact"
if exact:
    frames = frames + [sc.frame(k, device="cuda") for k in range(40, 48)]
    for k in range(30, 48):
        frames[k] = I.Scene.exact_obs(frames[k].contiguous())


def cycle(k):
    if exact and k >= 30:
        f.step_exact(frames[k], cfg.dt)
    else:
        f.step(frames[k], cfg.dt)


for k in range(38 if exact else 30):
    cycle(k)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 64)()
dog._lib.dog_timing_dump(buf, 64, 1)
for k in range(38, 48) if exact else range(30, 40):
    cycle(k)
torch.cuda.synchronize()
dog._lib.dog_timing_dump(buf, 64, 0)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.float64)
blocks = (cfg.nu + 4095) // 4096 * 10
print("windows", int(t[21]), "slow windows", int(t[20]), "radix passes per tile", t[30] / max(t[31], 1))
for i, nm in NAMES.items():
    print(f"{nm:28s} {t[i] / blocks / 1000:8.2f} us per block")
