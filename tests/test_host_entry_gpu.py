"""The host entry points (include/dog.h: dog_step_host, dog_step_host_async) produce exactly what the
device entry produces -- same state, same occupancy readout per cycle.  Requires a CUDA device."""
import numpy as np
import pytest
import torch

from paper_1605_02406_b200 import inputs as I

pytestmark = pytest.mark.gpu


def test_async_host_entry_matches_device_entry():
    from paper_1605_02406_b200 import dog
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    cfg = I.config("cfg2", width=128, height=128, nu=60_000, nu_b=6_000, beams=300, movers=3, peds=2, boxes=6)
    sc = I.scene(cfg)
    frames = [sc.frame(k).contiguous() for k in range(6)]
    g_dev, g_sync, g_async = (dog.Filter.from_config(cfg) for _ in range(3))
    occ_dev = []
    for fr in frames:
        g_dev.step(fr.cuda(), cfg.dt)
        occ_dev.append(g_dev.read_cells()["occ"].cpu().numpy())
    occ_sync = torch.empty(cfg.C, dtype=torch.float32).pin_memory()
    for k, fr in enumerate(frames):
        g_sync.step_host(fr.pin_memory(), cfg.dt, occ_sync)
        assert np.array_equal(occ_sync.numpy().view(np.uint32), occ_dev[k].view(np.uint32)), k
    pinned = [fr.pin_memory() for fr in frames]
    outs = [torch.empty(cfg.C, dtype=torch.float32).pin_memory() for _ in frames]
    for k in range(len(frames)):                # all cycles enqueued back to back, one sync at the end
        g_async.step_host_async(pinned[k], cfg.dt, outs[k])
    g_async.sync()
    for k in range(len(frames)):
        assert np.array_equal(outs[k].numpy().view(np.uint32), occ_dev[k].view(np.uint32)), k
    a, b = g_dev.get_state(), g_async.get_state()
    for key in ("x", "y", "vx", "vy", "m_free"):
        assert np.array_equal(a[key].view(np.uint32), b[key].view(np.uint32)), key
