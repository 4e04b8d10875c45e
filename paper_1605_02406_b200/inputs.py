"""Seeded synthetic inputs shared by the tests, the bench and smoke() -- measurement grids and states.

This module holds NONE of the filter's arithmetic (no Dempster rule, no prediction, no resampling):
it only synthesises measurement grids of occupied/free masses with the structure of the paper's
workload (section VIII: a vehicle at the centre of a 120 m grid of 0.1 m cells, a front
laser and radars, movers among parked cars) and simple injected
particle states.  Recipe: DESIGN.md section 5.

Measurement synthesis (an inverse sensor model, the method's INPUT -- P:1272-1273 cites Homm2010):
  * 2-D ray cast from the sensor through axis-aligned boxes at half-cell steps;
  * a cell crossed by k distinct beams before their first hit gets free mass 1 - 0.3^k (per-beam
    free mass 0.7, S:149 / S:187);
  * a hit cell gets occupied mass 0.95; cells beyond a hit stay unknown (0, 0);
  * radar sectors re-detect mover cells: a laser-hit mover cell becomes (0.98, 0), an
    unobserved mover cell inside the radar sector (0.6, 0).
These masses are configuration values, not paper values.

Everything is seeded: the scene layout by numpy PCG64 ``default_rng(1605 + cfg_index)``; frame k is
a pure function of (layout, k).  Frames are built with torch ops so the bench can synthesise them
on the GPU outside the timed region; tests build them on the CPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    nu: int
    nu_b: int
    scene: str                 # "box", "front", "urban", "stress"
    cycles: int = 10
    cell_size: float = 0.1     # m (Table I)
    dt: float = 0.1            # s
    p_s: float = 0.99          # Table I
    p_b: float = 0.02          # best value in P:1786 (range 0.005..0.1)
    sigma_pos: float = 0.02    # Table I
    sigma_vel: float = 0.8     # Table I
    sigma_birth_vel: float = 4.0  # Table I
    free_tau: float = 2.0      # A-9 default
    occ_max: float = 1.0       # A-7
    v_max: float = 0.0         # A-16 (off)
    seed: int = 2406
    scene_seed: int = 1605
    # scene knobs
    beams: int = 0
    fov_deg: float = 360.0
    range_m: float = 50.0
    movers: int = 0
    peds: int = 0
    boxes: int = 0
    walls: bool = False
    poles: int = 0             # 1-2 cell static clutter (posts, trees)
    radar: bool = False
    meas_density: float = 0.0  # stress scene: fraction of cells measured i.i.d.

    @property
    def C(self) -> int:
        return self.width * self.height

    def filter_params(self) -> dict:
        return dict(p_s=self.p_s, p_b=self.p_b, sigma_pos=self.sigma_pos, sigma_vel=self.sigma_vel,
                    sigma_birth_vel=self.sigma_birth_vel, free_tau=self.free_tau,
                    occ_max=self.occ_max, v_max=self.v_max)


# The configurations of BASELINE.json (cfg 1-5) plus the north-star 1-GPU target "T"
# (SURVEY.md 8(d)).  Filter seed = 2406 + index, scene seed = 1605 + index.
CONFIGS: dict[str, Config] = {
    "cfg1": Config("cfg1", 32, 32, 10_000, 1_000, "box", cycles=10, seed=2407, scene_seed=1606),
    "cfg2": Config("cfg2", 512, 512, 2_000_000, 200_000, "front", beams=1200, fov_deg=120.0,
                   range_m=50.0, movers=6, peds=4, boxes=40, radar=True, seed=2408, scene_seed=1607),
    "cfg3": Config("cfg3", 1024, 1024, 8_000_000, 800_000, "urban", beams=4096, range_m=50.0,
                   movers=30, peds=20, boxes=300, poles=800, walls=True, seed=2409, scene_seed=1608),
    "cfgT": Config("cfgT", 2048, 2048, 8_000_000, 800_000, "urban", beams=8192, range_m=100.0,
                   movers=120, peds=80, boxes=1200, poles=3000, walls=True, seed=2412, scene_seed=1611),
    "cfg4": Config("cfg4", 2048, 2048, 32_000_000, 3_200_000, "urban", beams=8192, range_m=100.0,
                   movers=120, peds=80, boxes=1200, poles=3000, walls=True, seed=2410, scene_seed=1609),
    "cfg5": Config("cfg5", 1024, 1024, 8_000_000, 2_000_000, "stress", p_b=0.1, sigma_pos=0.08,
                   sigma_vel=3.2, movers=30, peds=20, meas_density=0.9, seed=2411,
                   scene_seed=1610),
}


def config(name: str, **over) -> Config:
    return replace(CONFIGS[name], **over)


@dataclass
class _Box:
    x0: float   # cell units, lower-left corner at frame 0
    y0: float
    w: float    # extent in cells
    h: float
    vx: float = 0.0  # cells per frame
    vy: float = 0.0
    mover: bool = False


@dataclass
class Scene:
    cfg: Config
    boxes: list = field(default_factory=list)
    sensor: tuple = (0.0, 0.0)
    stress_u: np.ndarray | None = None

    # ------------------------------------------------------------------ layout
    @staticmethod
    def build(cfg: Config) -> "Scene":
        rng = np.random.default_rng(cfg.scene_seed)
        W, H, cs, dt = cfg.width, cfg.height, cfg.cell_size, cfg.dt
        sc = Scene(cfg=cfg, sensor=(W / 2.0, H / 2.0))
        if cfg.scene == "box":
            # cfg 1: one 4x4-cell box at x 4-7, y 14-17 moving +1 cell/step (1 m/s at 0.1 m, 0.1 s)
            sc.boxes.append(_Box(4.0, 14.0, 4.0, 4.0, 1.0, 0.0, True))
            return sc
        if cfg.scene == "stress":
            sc.stress_u = rng.random(W * H).astype(np.float32)

        def add_movers(n, lmin, lmax, wmin, wmax, vmin, vmax):
            for _ in range(n):
                ang = rng.uniform(0, 2 * math.pi)
                sp = rng.uniform(vmin, vmax) * dt / cs     # cells per frame
                L = rng.uniform(lmin, lmax) / cs; Wd = rng.uniform(wmin, wmax) / cs
                horiz = abs(math.cos(ang)) >= abs(math.sin(ang))
                w, h = (L, Wd) if horiz else (Wd, L)
                x0 = rng.uniform(0, W - w); y0 = rng.uniform(0, H - h)
                sc.boxes.append(_Box(x0, y0, w, h, sp * math.cos(ang), sp * math.sin(ang), True))

        add_movers(cfg.movers, 4.0, 5.0, 1.7, 2.0, 5.0, 15.0)       # cars
        add_movers(cfg.peds, 0.5, 0.8, 0.5, 0.8, 1.0, 6.0 if cfg.scene != "front" else 2.0)
        for _ in range(cfg.boxes):                                  # parked cars / clutter
            L = rng.uniform(3.5, 5.0) / cs; Wd = rng.uniform(1.6, 2.0) / cs
            w, h = (L, Wd) if rng.random() < 0.5 else (Wd, L)
            sc.boxes.append(_Box(rng.uniform(0, W - w), rng.uniform(0, H - h), w, h))
        for _ in range(cfg.poles):                                  # posts / vegetation clutter
            d = rng.uniform(1.0, 2.0)
            sc.boxes.append(_Box(rng.uniform(0, W - d), rng.uniform(0, H - d), d, d))
        if cfg.walls:                                               # building walls y = +-15 m
            for yw in (H / 2 - 15.0 / cs, H / 2 + 15.0 / cs):
                x = 0.0
                while x < W:
                    seg = rng.uniform(10.0, 40.0) / cs
                    sc.boxes.append(_Box(x, yw, min(seg, W - x), 3.0))
                    x += seg + rng.uniform(5.0, 15.0) / cs
        # keep the sensor surroundings clear (vehicle at the centre)
        cx, cy = sc.sensor
        sc.boxes = [b for b in sc.boxes if b.mover or not (
            b.x0 - 3 / cs < cx < b.x0 + b.w + 3 / cs and b.y0 - 3 / cs < cy < b.y0 + b.h + 3 / cs)]
        return sc

    # ------------------------------------------------------------------ frames
    def _pos(self, b: _Box, k: int):
        """Constant-velocity motion reflected at the grid edges (triangle wave)."""
        W, H = self.cfg.width, self.cfg.height

        def refl(p0, v, lo, hi):
            if v == 0.0 or hi <= lo:
                return p0
            span = hi - lo
            t = (p0 - lo + v * k) % (2 * span)
            return lo + (t if t <= span else 2 * span - t)

        return refl(b.x0, b.vx, 0.0, W - b.w), refl(b.y0, b.vy, 0.0, H - b.h)

    def frame(self, k: int, device="cpu") -> torch.Tensor:
        """Measurement grid of frame k: float32 [H, W, 2] = (m_zO, m_zF), row-major (x = column)."""
        cfg = self.cfg
        W, H = cfg.width, cfg.height
        dev = torch.device(device)
        occ_obj = torch.zeros(H, W, dtype=torch.bool, device=dev)
        mov = torch.zeros(H, W, dtype=torch.bool, device=dev)
        for b in self.boxes:
            x, y = self._pos(b, k)
            c0, c1 = int(math.floor(x)), int(math.ceil(x + b.w))
            r0, r1 = int(math.floor(y)), int(math.ceil(y + b.h))
            c0, r0 = max(c0, 0), max(r0, 0)
            c1, r1 = min(c1, W), min(r1, H)
            if c1 > c0 and r1 > r0:
                occ_obj[r0:r1, c0:c1] = True
                if b.mover:
                    mov[r0:r1, c0:c1] = True
        out = torch.zeros(H, W, 2, dtype=torch.float32, device=dev)
        if cfg.scene == "box":
            out[..., 1] = 0.6
            out[occ_obj] = torch.tensor([0.9, 0.0], device=dev)
            return out
        if cfg.scene == "stress":
            u = torch.from_numpy(self.stress_u).to(dev).view(H, W)
            out[(u < 0.2)] = torch.tensor([0.9, 0.0], device=dev)
            out[(u >= 0.2) & (u < 0.9)] = torch.tensor([0.0, 0.7], device=dev)
            out[occ_obj & mov] = torch.tensor([0.9, 0.0], device=dev)
            return out
        return self._raycast(occ_obj, mov, out)

    def _raycast(self, occ_obj, mov, out):
        cfg = self.cfg
        W, H = cfg.width, cfg.height
        dev = out.device
        cx, cy = self.sensor
        rng_c = cfg.range_m / cfg.cell_size
        nb = cfg.beams
        fov = math.radians(cfg.fov_deg)
        th = (torch.arange(nb, device=dev, dtype=torch.float64) + 0.5) / nb * fov - fov / 2.0
        ns = int(rng_c / 0.5)
        r = (torch.arange(ns, device=dev, dtype=torch.float64) + 1.0) * 0.5
        px = cx + torch.cos(th)[:, None] * r[None, :]
        py = cy + torch.sin(th)[:, None] * r[None, :]
        ix = torch.floor(px).long(); iy = torch.floor(py).long()
        inside = (ix >= 0) & (ix < W) & (iy >= 0) & (iy < H)
        lin = torch.where(inside, iy * W + ix, torch.zeros_like(ix))
        hit = occ_obj.view(-1)[lin] & inside
        any_hit = hit.any(dim=1)
        first = torch.where(any_hit, hit.float().argmax(dim=1), torch.full_like(any_hit, ns, dtype=torch.long))
        sidx = torch.arange(ns, device=dev)[None, :]
        free = (sidx < first[:, None]) & inside
        # count each (beam, cell) once: drop consecutive repeats along the beam
        prev = torch.cat([torch.full_like(lin[:, :1], -1), lin[:, :-1]], dim=1)
        free &= lin != prev
        k_free = torch.bincount(lin[free], minlength=W * H).view(H, W)
        hit_cells = torch.zeros(W * H, dtype=torch.bool, device=dev)
        bi = torch.nonzero(any_hit).squeeze(1)
        hit_cells[lin[bi, first[bi]]] = True
        # a return marks the hit cell and the next cell along the beam (range noise spot)
        nxt = torch.clamp(first[bi] + 2, max=ns - 1)
        ok = inside[bi, nxt] & occ_obj.view(-1)[lin[bi, nxt]]
        hit_cells[lin[bi[ok], nxt[ok]]] = True
        hit_cells = hit_cells.view(H, W)
        mF = 1.0 - torch.pow(torch.tensor(0.3, device=dev, dtype=torch.float64), k_free.double())
        out[..., 1] = torch.where(k_free > 0, mF.float(), torch.zeros_like(out[..., 1]))
        out[hit_cells] = torch.tensor([0.95, 0.0], device=dev)
        if cfg.radar:
            yy, xx = torch.meshgrid(torch.arange(H, device=dev), torch.arange(W, device=dev), indexing="ij")
            dx = (xx + 0.5 - cx) * cfg.cell_size; dy = (yy + 0.5 - cy) * cfg.cell_size
            d = torch.sqrt(dx * dx + dy * dy)
            a = torch.rad2deg(torch.atan2(dy, dx)).abs()
            sector = (d <= 30.0) & (a >= 30.0) & (a <= 90.0)
            out[mov & sector & hit_cells] = torch.tensor([0.98, 0.0], device=dev)
            unobs = mov & sector & (~hit_cells) & (out[..., 1] == 0)
            out[unobs] = torch.tensor([0.6, 0.0], device=dev)
        return out

    def doppler(self, k: int, meas: torch.Tensor, frac: float = 0.5, p_assoc: float = 0.8, sd: float = 0.25,
                device="cpu"):
        """Radar Doppler overlay of frame k (NEXT-1 input; SPEC S:151-159 radar_overlay, S:440 defaults):
        a seeded fraction `frac` of the cells with m_zO > 0 carry a radial-velocity measurement --
        unit direction from the sensor to the cell centre, radial speed = the true object velocity (a
        mover covering the cell, else 0) projected on it plus N(0, sd^2) noise, SD sd -- and association
        probability p_assoc.  Returns (doppler [H, W, 4] f32 = (u_x, u_y, v_r, sd), p_A [H, W] f32)."""
        cfg = self.cfg
        W, H, cs, dt = cfg.width, cfg.height, cfg.cell_size, cfg.dt
        rng = np.random.default_rng((cfg.scene_seed * 1_000_003 + k) & 0xFFFFFFFF)
        vel = np.zeros((H, W, 2), np.float64)
        for b in self.boxes:
            if not b.mover:
                continue
            x, y = self._pos(b, k)
            c0, c1 = max(int(math.floor(x)), 0), min(int(math.ceil(x + b.w)), W)
            r0, r1 = max(int(math.floor(y)), 0), min(int(math.ceil(y + b.h)), H)
            if c1 > c0 and r1 > r0:
                vel[r0:r1, c0:c1] = (b.vx * cs / dt, b.vy * cs / dt)
        yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        dx = xx + 0.5 - self.sensor[0]; dy = yy + 0.5 - self.sensor[1]
        d = np.sqrt(dx * dx + dy * dy)
        d[d == 0] = 1.0
        ux, uy = dx / d, dy / d
        vr = vel[..., 0] * ux + vel[..., 1] * uy + rng.normal(0.0, sd, (H, W))
        occ = meas.detach().cpu().numpy().reshape(H, W, 2)[..., 0] > 0
        has = occ & (rng.random((H, W)) < frac)
        dop = np.stack([ux, uy, vr, np.full((H, W), sd)], -1).astype(np.float32)
        pA = np.where(has, np.float32(p_assoc), np.float32(0.0)).astype(np.float32)
        return torch.from_numpy(dop).to(device), torch.from_numpy(pA).to(device)

    @staticmethod
    def exact_obs(meas: torch.Tensor, kappa: float = 0.9) -> torch.Tensor:
        """Observation grid of the exact PHD/MIB filter (NEXT-3 input) from a measurement grid
        [..., 2] = (m_zO, m_zF), A-37 input recipe: a cell with a return (m_zO > 0) has a
        measurement (occurred = 1) with p_TP = kappa and p_FP = kappa (1 - m_zO) / m_zO capped at kappa
        (likelihood ratio m_zO / (1 - m_zO)); a cell seen free has none, with p_TP = m_zF and p_FP = 0.01;
        an unobserved cell has none with p_TP = p_FP = 0.05 (ratio 1: uninformative).  Returns f32
        [..., 4] = (occurred, p_TP, p_FP, 0) on the input's device."""
        mO, mF = meas[..., 0], meas[..., 1]
        hit = mO > 0
        seen = (~hit) & (mF > 0)
        out = torch.zeros(meas.shape[:-1] + (4,), dtype=torch.float32, device=meas.device)
        out[..., 0] = hit.float()
        pfp_hit = torch.clamp(kappa * (1.0 - mO) / torch.clamp(mO, min=1e-6), max=kappa)
        out[..., 1] = torch.where(hit, torch.full_like(mO, kappa), torch.where(seen, mF, torch.full_like(mO, 0.05)))
        out[..., 2] = torch.where(hit, pfp_hit, torch.where(seen, torch.full_like(mO, 0.01), torch.full_like(mO, 0.05)))
        return out.contiguous()

    def exact_lik(self, k: int, meas: torch.Tensor, p_cl: float = 0.02, frac: float = 0.5, p_assoc: float = 0.8,
                  sd: float = 0.25):
        """Inputs of the exact filter with a single-object likelihood (NEXT-3 general form; A-38
        input recipe): the observation grid of exact_obs with the clutter density p_cl in its 4th column --
        a clutter return's radial speed uniform over +-25 m/s, 0.02 per m/s -- and the Doppler overlay of
        `doppler` (same seeded fraction of the cells with a return) as the measurement's likelihood.
        Returns (obs [H, W, 4], lik [H, W, 4] = (u_x, u_y, v_r, sd), p_A [H, W]), f32 on the CPU."""
        obs = Scene.exact_obs(meas.detach().cpu())
        obs[..., 3] = p_cl
        lik, pA = self.doppler(k, meas, frac=frac, p_assoc=p_assoc, sd=sd)
        return obs.contiguous(), lik, pA

    def frames(self, k0: int, n: int, device="cpu") -> torch.Tensor:
        return torch.stack([self.frame(k0 + i, device) for i in range(n)])


def scene(cfg: Config | str) -> Scene:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return Scene.build(cfg)


# ---------------------------------------------------------------------- injected states
SENTINEL_POS = np.float32(-1073741824.0)   # -2^30 cells: the empty-world particle position (A-19)


def empty_state(cfg: Config):
    nu = cfg.nu
    return dict(x=np.full(nu, SENTINEL_POS, np.float32), y=np.full(nu, SENTINEL_POS, np.float32),
                vx=np.zeros(nu, np.float32), vy=np.zeros(nu, np.float32), w_bar=np.float32(0.0),
                m_free=np.zeros(cfg.C, np.float32), k=0)


def cells_state(cfg: Config, counts: np.ndarray, w_bar: float, vel=(0.0, 0.0), rng=None,
                vel_sd: float = 0.0, m_free=None, k: int = 0):
    """Particles placed cell by cell in canonical (cell-sorted) order: counts[c] particles in cell
    c at uniform positions inside the cell; the remainder of the nu slots at the sentinel."""
    rng = rng if rng is not None else np.random.default_rng(0)
    W = cfg.width
    counts = np.asarray(counts, np.int64)
    n = int(counts.sum())
    assert n <= cfg.nu, (n, cfg.nu)
    cell = np.repeat(np.arange(cfg.C, dtype=np.int64), counts)
    st = empty_state(cfg)
    col = (cell % W).astype(np.float32); row = (cell // W).astype(np.float32)
    fx = rng.random(n).astype(np.float32) * np.float32(0.999); fy = rng.random(n).astype(np.float32) * np.float32(0.999)
    st["x"][:n] = col + fx
    st["y"][:n] = row + fy
    st["vx"][:n] = np.float32(vel[0]) + np.float32(vel_sd) * rng.standard_normal(n).astype(np.float32)
    st["vy"][:n] = np.float32(vel[1]) + np.float32(vel_sd) * rng.standard_normal(n).astype(np.float32)
    st["w_bar"] = np.float32(w_bar)
    if m_free is not None:
        st["m_free"][:] = np.asarray(m_free, np.float32)
    st["k"] = k
    return st
