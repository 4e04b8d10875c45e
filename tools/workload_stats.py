"""Workload statistics of a warmed-up filter (runs per sort tile, cell occupancy) -- diagnostics only."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1605_02406_b200 import dog, inputs as I

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfgT"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sc = I.scene(cfg)
f = dog.Filter.from_config(cfg, debug=True)
n_exact = int(sys.argv[3]) if len(sys.argv) > 3 else 0      # then this many exact PHD/MIB cycles (NEXT-3)
for k in range(steps):
    f.step(sc.frame(k, device="cuda"), cfg.dt)
for k in range(steps, steps + n_exact):
    f.step_exact(I.Scene.exact_obs(sc.frame(k, device="cuda")), cfg.dt)
key = f.debug("KEY")
off = f.debug("OFFSETS")
n = np.diff(off.astype(np.int64))
T = (cfg.nu + 4095) // 4096
runs = []
for t in range(T):
    kt = np.sort(key[t * 4096:(t + 1) * 4096])
    runs.append(1 + int(np.count_nonzero(np.diff(kt))))
runs = np.array(runs)
occ = n[n > 0]
print(f"cfg={cfg.name} steps={steps} n_in={int(off[-1])} cells_with_particles={occ.size}")
print(f"particles per occupied cell: mean={occ.mean():.1f} median={np.median(occ):.0f} p90={np.percentile(occ,90):.0f} max={occ.max()}")
print(f"runs per 4096-tile: mean={runs.mean():.1f} median={np.median(runs):.0f} p90={np.percentile(runs,90):.0f} max={runs.max()}")
print(f"total runs={runs.sum()} mean run length={cfg.nu / runs.sum():.1f}")
print("particles-per-cell histogram (1..8, >8):", [int(np.count_nonzero(occ == i)) for i in range(1, 9)],
      int(np.count_nonzero(occ > 8)))
s = f.scalars()
print("W mass", s["W"] * 2.0 ** -40, "A", s["A"] * 2.0 ** -40)
nb = f.debug("NB")
Rb = f.debug("RB")
print(f"cells with nb>0: {int(np.count_nonzero(nb))}  cells with Rb>0: {int(np.count_nonzero(Rb))}  "
      f"active (n>0 or Rb>0): {int(np.count_nonzero((n > 0) | (Rb > 0)))}")
